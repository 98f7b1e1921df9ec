"""Host-resident differentiable Adam step, streamed through the GPU.

For trees whose optimizer state lives in (pinned) host memory, the step is
run chunk by chunk with three streams: host->device copies of chunk c+1,
the fused forward + backward kernels of chunk c (libdiffopt.so, the same
C-ABI calls as the device-resident path) and device->host copies of chunk
c-1 overlap, so the PCIe link in both directions is the only bound. The
per-chunk hyper-gradient sums are combined in chunk order on the device
(opt_sum_rows; deterministic).
This is the end-to-end path bench.py reports as "e2e".
"""
from __future__ import annotations

import torch

from . import _lib as L

IN_KEYS = ("g", "m", "v", "du", "dm1", "dv1")
OUT_KEYS = ("u", "m1", "v1", "dg", "dm", "dv")


class HostStreamedAdam:
    """Adam fwd + bwd over pinned host arrays of n fp32 elements."""

    def __init__(self, n, device, chunks=8, compute=L.OPT_COMPUTE_DEFAULT, slots=3,
                 ramp=None):
        """chunks: number of equal chunks; or ramp = relative chunk sizes
        (e.g. (1, 2, 4, 4, 4, 4, 2, 1)): small first / last chunks shorten
        the pipeline fill (first H2D alone) and drain (last D2H alone)
        without paying per-copy overhead on every chunk."""
        self.n, self.dev, self.compute = int(n), device, compute
        align = 4096
        weights = list(ramp) if ramp else [1] * int(chunks)
        tot = float(sum(weights))
        cuts = [0]
        acc = 0.0
        for w in weights[:-1]:
            acc += w
            cut = min(self.n, -(-int(self.n * acc / tot) // align) * align)
            cuts.append(max(cut, cuts[-1]))
        cuts.append(self.n)
        self.bounds = [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a]
        per = max(b - a for a, b in self.bounds)
        self.trees = [L.Tree(numel=e - s, device=device) for s, e in self.bounds]
        self.ws = [t.workspace(device) for t in self.trees]
        self.nb = nb = max(2, min(int(slots), len(self.bounds)))  # staging slots: H2D of
        # chunk c overlaps D2H of chunks c-1 .. c-nb+1
        self.buf = [{k: torch.empty(per, device=device) for k in IN_KEYS + OUT_KEYS}
                    for _ in range(nb)]
        self.dhp = torch.empty(len(self.bounds), 4, dtype=torch.float64, device=device)
        self.dhp_total = torch.empty(4, dtype=torch.float64, device=device)
        self.h_dhp = torch.empty(4, dtype=torch.float64).pin_memory()
        self.s_h2d = torch.cuda.Stream(device)
        self.s_cmp = torch.cuda.Stream(device)
        self.s_d2h = torch.cuda.Stream(device)

    def bytes_h2d(self):
        return 4 * self.n * len(IN_KEYS)

    def bytes_d2h(self):
        return 4 * self.n * len(OUT_KEYS) + self.h_dhp.numel() * 8

    def run(self, host_in, host_out, step, hp):
        """host_in / host_out: dicts of pinned fp32 CPU tensors of n elements.
        Enqueues everything on the three streams ordered after the current
        stream; the current stream waits for completion at the end."""
        cur = torch.cuda.current_stream(self.dev)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        h2d_done, cmp_done, d2h_done = [], [], []
        for c, (lo, hi) in enumerate(self.bounds):
            b = self.buf[c % self.nb]
            k = hi - lo
            with torch.cuda.stream(self.s_h2d):
                if c >= self.nb:  # staging slot reused: wait until chunk c-nb left the device
                    self.s_h2d.wait_event(d2h_done[c - self.nb])
                for key in IN_KEYS:
                    b[key][:k].copy_(host_in[key][lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(self.s_h2d)
                h2d_done.append(e)
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(h2d_done[c])
                t = self.trees[c]
                L.opt_adam_fwd(t, step, hp, L.OPT_F32, self.compute, b["g"], b["m"], b["v"],
                               b["u"], b["m1"], b["v1"], stream=self.s_cmp)
                L.opt_adam_bwd(t, step, hp, L.OPT_F32, self.compute, b["g"], b["m"], b["v"],
                               b["du"], b["dm1"], b["dv1"], b["dg"], b["dm"], b["dv"],
                               self.dhp[c], None, self.ws[c], stream=self.s_cmp)
                e = torch.cuda.Event()
                e.record(self.s_cmp)
                cmp_done.append(e)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(cmp_done[c])
                for key in OUT_KEYS:
                    host_out[key][lo:hi].copy_(b[key][:k], non_blocking=True)
                e = torch.cuda.Event()
                e.record(self.s_d2h)
                d2h_done.append(e)
        with torch.cuda.stream(self.s_cmp):  # chunk-ordered sum on the device (row a5)
            L.opt_sum_rows(len(self.bounds), 4, self.dhp, self.dhp_total, stream=self.s_cmp)
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_stream(self.s_cmp)
            self.h_dhp.copy_(self.dhp_total, non_blocking=True)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            cur.wait_stream(s)
        return self.h_dhp  # (lr, b1, b2, eps) sums; valid once the current stream gets here
