"""PCIe copy-shape probe: 6 arrays x n fp32 host<->device as many 1-D copies
vs one cudaMemcpy2DAsync per chunk (rows = arrays, pitch = n*4), one
direction and both at once. CUDA events; pinned host memory."""
import ctypes
import json

import torch

n = 11689512 // 4 * 4
A, CH = 6, 8
dev = torch.device("cuda:0")
h_in = torch.empty(A, n).pin_memory()
h_out = torch.empty(A, n).pin_memory()
h_in.normal_()
d_in = torch.empty(A, n, device=dev)
d_out = torch.empty(A, n, device=dev)
rt = ctypes.CDLL("libcudart.so.12") if False else None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = ctypes.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    import glob, os
    p = glob.glob(os.path.dirname(torch.__file__) + "/../nvidia/cuda_runtime/lib/libcudart.so*")
    rt = ctypes.CDLL(p[0])
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
H2D, D2H = 1, 2
cuts = [n * i // CH // 1024 * 1024 for i in range(CH)] + [n]
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def copies(direction, mode, stream):
    with torch.cuda.stream(stream):
        for c in range(CH):
            lo, hi = cuts[c], cuts[c + 1]
            if mode == "1d":
                for a in range(A):
                    if direction == H2D:
                        d_in[a, lo:hi].copy_(h_in[a, lo:hi], non_blocking=True)
                    else:
                        h_out[a, lo:hi].copy_(d_out[a, lo:hi], non_blocking=True)
            else:
                if direction == H2D:
                    dst, src = d_in.data_ptr() + lo * 4, h_in.data_ptr() + lo * 4
                else:
                    dst, src = h_out.data_ptr() + lo * 4, d_out.data_ptr() + lo * 4
                rc = rt.cudaMemcpy2DAsync(dst, n * 4, src, n * 4, (hi - lo) * 4, A, direction,
                                          ctypes.c_void_p(stream.cuda_stream))
                assert rc == 0, rc


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


cur = torch.cuda.current_stream(dev)
for mode in ("1d", "2d"):
    def h2d():
        s1.wait_stream(cur); copies(H2D, mode, s1); cur.wait_stream(s1)

    def d2h():
        s2.wait_stream(cur); copies(D2H, mode, s2); cur.wait_stream(s2)

    def both():
        s1.wait_stream(cur); s2.wait_stream(cur)
        copies(H2D, mode, s1); copies(D2H, mode, s2)
        cur.wait_stream(s1); cur.wait_stream(s2)

    out = {"mode": mode, "chunks": CH, "h2d_ms": timed(h2d), "d2h_ms": timed(d2h),
           "both_ms": timed(both)}
    out["mb_each_way"] = A * n * 4 / 1e6
    print(json.dumps(out))
torch.cuda.synchronize()
assert torch.equal(d_in.cpu(), h_in)
print("ok")
