"""PCIe ceiling and HostStreamedAdam chunk / slot sweep for the e2e line
(C2-sized tree, 6 x 4 B in and 6 x 4 B out per element).

    python tools/e2e_sweep.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_06934_b200.offload import IN_KEYS, OUT_KEYS, HostStreamedAdam  # noqa: E402

N = 11_689_512
HP = (1e-3, 0.9, 0.999, 1e-8, 0.0)


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda", 0)
    nbytes = 6 * 4 * N
    h_src = torch.empty(nbytes // 4).pin_memory()
    h_dst = torch.empty(nbytes // 4).pin_memory()
    d_a = torch.empty(nbytes // 4, device=dev)
    d_b = torch.empty(nbytes // 4, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}
    res["h2d_gbs"] = nbytes / timed(lambda: d_a.copy_(h_src, non_blocking=True)) / 1e6
    res["d2h_gbs"] = nbytes / timed(lambda: h_dst.copy_(d_b, non_blocking=True)) / 1e6

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    res["bidir_gbs_each"] = nbytes / timed(both) / 1e6
    res["bidir_floor_ms"] = nbytes / (res["bidir_gbs_each"] * 1e6)
    print(json.dumps(res), flush=True)
    g = torch.Generator(device=dev).manual_seed(0)
    # packed host rows (one strided DMA per chunk and direction), as bench.py
    h_in, h_out = HostStreamedAdam.alloc_host(N)
    for k in IN_KEYS:
        h_in[k].copy_(torch.randn(N, device=dev, generator=g).abs())
    alg = 60 * N
    cands = [dict(chunks=c, slots=sl) for c in (8, 10, 12, 14) for sl in (2, 3, 4, 6)]
    cands += [dict(ramp=r) for r in ((1, 2, 4, 4, 4, 4, 2, 1), (1, 2, 2, 2, 2, 2, 2, 2, 2, 1),
                                      (1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 1, 1))]
    for kw in cands:
        hs = HostStreamedAdam(N, dev, **kw)
        ms = timed(lambda: hs.run(h_in, h_out, 10, HP, inputs_on_host=True))
        print(json.dumps({**{k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                          "ms": round(ms, 3), "e2e_gbs": round(alg / ms / 1e6, 1)}), flush=True)
        del hs
        torch.cuda.empty_cache()

if __name__ == "__main__":
    main()
