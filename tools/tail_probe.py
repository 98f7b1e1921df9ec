"""C2 Adam backward reduction-tail probe: run with DIFFOPT_LIB pointing at a
build with -DDOPT_TAIL_PROBE=1 (build.build(out=..., defines=["DOPT_TAIL_PROBE=1"]));
prints the median block-completion spread and the last block's tail segments
(profiles/r02ad_bwd_tail_probe_and_dyn_experiments.txt)."""
import os, sys, json, statistics
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2211_06934_b200 import _lib as L
import synth
dev = 'cuda:0'
HP = (1e-3, 0.9, 0.999, 1e-8, 0.0)
leaves = [9408,64,64,36864,64,64,36864,64,64,36864,64,64,36864,64,64,73728,128,128,147456,128,128,8192,128,128,147456,128,128,147456,128,128,294912,256,256,589824,256,256,32768,256,256,589824,256,256,589824,256,256,1179648,512,512,2359296,512,512,131072,512,512,2359296,512,512,2359296,512,512,512000,1000]
n = sum(leaves)
tree = L.Tree(numel=n, device=dev)
ws = tree.workspace(dev)
gen = torch.Generator(device=dev).manual_seed(1)
S = []
for _ in range(4):
    s = {k: torch.randn(n, device=dev, generator=gen) * 1e-2 for k in ("g", "m", "du", "dm1", "dv1")}
    s["v"] = torch.rand(n, device=dev, generator=gen) * 1e-4
    for k in ("dg", "dm", "dv"): s[k] = torch.empty(n, device=dev)
    s["dhp"] = torch.empty(4, dtype=torch.float64, device=dev)
    S.append(s)
def call(i):
    s = S[i % 4]
    L.opt_adam_bwd(tree, 10, HP, 0, 0, s["g"], s["m"], s["v"], s["du"], s["dm1"], s["dv1"], s["dg"], s["dm"], s["dv"], s["dhp"], None, ws)
for i in range(20): call(i)
torch.cuda.synchronize()
part = ws.view(-1)  # float64 view; partials start after a 256-byte counter header
off = 256 // 8
rows = []
for i in range(30):
    # previous launch in flight so this one starts PDL-overlapped like in the bench loop
    call(i); call(i + 1)
    torch.cuda.synchronize()
    w = part[off:].cpu().numpy()
    G = int(w[16384 + 5]) if w[16384 + 5] > 0 else 0
    nb = 444
    starts = w[8192:8192 + nb]; done = w[12288:12288 + nb]
    end = w[16384 + 4]
    rows.append(dict(span_us=(end - starts.min()) / 1e3, start_spread_us=(starts.max() - starts.min()) / 1e3,
                     done_spread_us=(done.max() - done.min()) / 1e3, tail_after_lastdone_us=(end - done.max()) / 1e3,
                     last_block_done_rank=int(np.argsort(np.argsort(done))[G]),
                     cyc_blocksum=w[16384], cyc_ticket=w[16385], cyc_loads=w[16386], cyc_final=w[16387]))
keys = rows[0].keys()
print(json.dumps({k: round(statistics.median(r[k] for r in rows), 3) for k in keys}))
print(json.dumps(rows[:3]))
