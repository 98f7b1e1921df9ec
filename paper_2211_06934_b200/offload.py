"""Host-resident differentiable Adam step, streamed through the GPU.

For trees whose optimizer state lives in (pinned) host memory, the step is
run chunk by chunk with three streams: host->device copies of chunk c+1,
the fused forward + backward kernels of chunk c (libdiffopt.so, the same
C-ABI calls as the device-resident path) and device->host copies of chunk
c-1 overlap, so the PCIe link in both directions is the only bound. The
per-chunk hyper-gradient sums are combined in chunk order on the device
(opt_sum_rows; deterministic). When the six input (and the six output)
host arrays are rows of one pinned buffer (alloc_host()), each chunk moves
in ONE strided DMA command per direction (opt_copy_rows) instead of six:
with both PCIe directions busy at once that is 6.3 instead of 7.3 ms for
2 x 280 MB (profiles/r02bj_*).
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
        per = -(-max(b - a for a, b in self.bounds) // 64) * 64  # rows stay 256-byte aligned
        self.trees = [L.Tree(numel=e - s, device=device) for s, e in self.bounds]
        self.ws = [t.workspace(device) for t in self.trees]
        self.nb = nb = max(2, min(int(slots), len(self.bounds)))  # staging slots: H2D of
        # chunk c overlaps D2H of chunks c-1 .. c-nb+1
        # staging slots: the six inputs and the six outputs of a chunk are
        # rows of one [6, per] device block each (one strided copy per chunk)
        self.per = per
        self.blk = [(torch.empty(len(IN_KEYS), per, device=device),
                     torch.empty(len(OUT_KEYS), per, device=device)) for _ in range(nb)]
        self.buf = [dict(zip(IN_KEYS + OUT_KEYS, list(bi) + list(bo))) for bi, bo in self.blk]
        self.dhp = torch.empty(len(self.bounds), 4, dtype=torch.float64, device=device)
        self.dhp_total = torch.empty(4, dtype=torch.float64, device=device)
        self.h_dhp = torch.empty(4, dtype=torch.float64).pin_memory()
        self.slot_free = [None] * nb  # per staging slot: D2H done of its last chunk
        self.s_h2d = torch.cuda.Stream(device)
        self.s_cmp = torch.cuda.Stream(device)
        self.s_d2h = torch.cuda.Stream(device)

    @staticmethod
    def alloc_host(n):
        """Pinned host arrays for run(): the six inputs as rows of one
        [6, n] buffer and the six outputs of another, so every chunk is one
        strided copy per direction. Returns (host_in, host_out) dicts."""
        hi = torch.empty(len(IN_KEYS), int(n)).pin_memory()
        ho = torch.empty(len(OUT_KEYS), int(n)).pin_memory()
        return dict(zip(IN_KEYS, hi)), dict(zip(OUT_KEYS, ho))

    @staticmethod
    def _rows(arrs, n):
        """(base address, pitch in bytes) when the arrays are equally spaced
        rows of ONE tensor storage (pitch >= 4n, contiguous fp32 of n
        elements each), else None. Separate allocations never qualify, even
        when they happen to be equally spaced: the strided DMA must stay
        inside one pinned allocation."""
        if any(a.dtype != torch.float32 or a.numel() != n or not a.is_contiguous() for a in arrs):
            return None
        st = arrs[0].untyped_storage().data_ptr()
        if any(a.untyped_storage().data_ptr() != st for a in arrs):
            return None
        base = arrs[0].data_ptr()
        if len(arrs) == 1:
            return base, 4 * n
        pitch = arrs[1].data_ptr() - base
        if pitch < 4 * n:
            return None
        for i, a in enumerate(arrs):
            if a.data_ptr() != base + i * pitch:
                return None
        return base, pitch

    def bytes_h2d(self):
        return 4 * self.n * len(IN_KEYS)

    def bytes_d2h(self):
        return 4 * self.n * len(OUT_KEYS) + self.h_dhp.numel() * 8

    def run(self, host_in, host_out, step, hp, inputs_on_host=False):
        """host_in / host_out: dicts of pinned fp32 CPU tensors of n elements.
        Enqueues everything ordered after the current stream; the current
        stream waits for completion at the end. host_in must not be
        rewritten before the current stream has passed this call.

        inputs_on_host=True declares that host_in was filled by the CPU (not
        by device work still queued on the current stream): the host->device
        copies then wait only for their staging slot, so the next call's
        first chunks stream in while this call's last chunks stream out and
        back-to-back calls keep both PCIe directions busy."""
        cur = torch.cuda.current_stream(self.dev)
        for s in ((self.s_cmp, self.s_d2h) if inputs_on_host else
                  (self.s_h2d, self.s_cmp, self.s_d2h)):
            s.wait_stream(cur)
        h2d_done, cmp_done, d2h_done = [], [], []
        rin = self._rows([host_in[k] for k in IN_KEYS], self.n)
        rout = self._rows([host_out[k] for k in OUT_KEYS], self.n)
        dp = 4 * self.per  # device staging pitch
        for c, (lo, hi) in enumerate(self.bounds):
            b = self.buf[c % self.nb]
            bi, bo = self.blk[c % self.nb]
            k = hi - lo
            with torch.cuda.stream(self.s_h2d):
                if c >= self.nb:  # staging slot reused: wait until chunk c-nb left the device
                    self.s_h2d.wait_event(d2h_done[c - self.nb])
                elif self.slot_free[c] is not None:  # ... or the previous call's last user
                    self.s_h2d.wait_event(self.slot_free[c])
                if rin:  # the six input rows' chunk in one strided copy
                    L.opt_copy_rows(bi, dp, rin[0] + 4 * lo, rin[1], 4 * k, len(IN_KEYS),
                                    stream=self.s_h2d)
                else:
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
                if rout:
                    L.opt_copy_rows(rout[0] + 4 * lo, rout[1], bo, dp, 4 * k, len(OUT_KEYS),
                                    stream=self.s_d2h)
                else:
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
        nc = len(self.bounds)
        for j in range(self.nb):  # the last chunk that used each slot
            last = max((c for c in range(nc) if c % self.nb == j), default=None)
            self.slot_free[j] = d2h_done[last] if last is not None else self.slot_free[j]
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            cur.wait_stream(s)
        return self.h_dhp  # (lr, b1, b2, eps) sums; valid once the current stream gets here
