#!/usr/bin/env python
"""Benchmark of the fused differentiable optimizer step (BASELINE.json metric
"diff-Adam fwd+bwd GB/s & % HBM peak").

Default workload (configs[1], C2): differentiable Adam forward + backward over
a ResNet-18-shaped tree (62 leaves, 11,689,512 fp32 elements) in one
multi-tensor launch each, warm state at t = 10, all cotangents supplied and
the four hyper-gradient sums produced. One "step" = opt_adam_fwd +
opt_adam_bwd through the C ABI. value = algorithmic bytes (60 B/elem:
24 forward + 36 backward) / device time, summed over
ranks (each rank runs its own tree: weak scaling, no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--compute default|f32|f64] [--workload c2|c1|c5|c3|maml|es]

--gpus N > 1 without a torch.distributed environment re-launches this script
under ``torch.distributed.run`` with N local ranks (one process per GPU,
NCCL; rendezvous on 127.0.0.1). Under torchrun, WORLD_SIZE must equal N.
The default line also carries the other configurations as secondary keys
(``c1``, ``c3``, ``c5``, ``es`` at N = 1; ``maml_c4`` at every N), each with
its own roofline fraction, and the paper's own speedup figures as context.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

HBM_FALLBACK = 6650.0
NOMINAL_HBM = 8000.0
BYTES_FWD = 24   # g, m, v -> u, m', v'   (fp32)
BYTES_BWD = 36   # g, m, v, du, dm', dv' -> dg, dm, dv
HP = (1e-3, 0.9, 0.999, 1e-8, 0.0)
STEP_T = 10


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU works."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, val in zip(names, r[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------- workloads
def c2_inputs():
    leaves = synth.RESNET18_LEAVES
    return synth.state_tree(0xC2, leaves), synth.offsets_of(leaves), "C2 resnet18-tree"


def c1_inputs():
    x = synth.c1_inputs()
    return x, np.array([0, x["g"].size], np.int64), "C1 flat-4096"


def c5_inputs(n):
    return synth.state_tree(0xC5, None, n=n), np.array([0, n], np.int64), f"C5 flat-{n}"


class AdamWorkload:
    """Device buffers for R rotating sets of one fwd+bwd step."""

    def __init__(self, L, x, offsets, dev, sets, compute, bf16=False):
        import torch

        self.L, self.torch, self.dev, self.compute = L, torch, dev, compute
        self.tree = L.Tree(offsets=offsets, device=dev)
        self.n = self.tree.numel
        self.sd = 1 if bf16 else 0
        t = torch

        def up(a, state=False):
            if a is None:
                return None
            if state and bf16:
                bits = synth.to_bf16_bits(a)
                return t.from_numpy(bits.view(np.int16)).to(dev).view(t.bfloat16)
            return t.from_numpy(np.ascontiguousarray(a)).to(dev)

        sdt = t.bfloat16 if bf16 else t.float32
        self.sets = []
        for _ in range(sets):
            s = dict(g=up(x["g"]), m=up(x["m"], True), v=up(x["v"], True), du=up(x["du"]),
                     dm1=up(x["dm1"]), dv1=up(x["dv1"]))
            s.update(u=t.empty(self.n, device=dev), m1=t.empty(self.n, dtype=sdt, device=dev),
                     v1=t.empty(self.n, dtype=sdt, device=dev), dg=t.empty(self.n, device=dev),
                     dm=t.empty(self.n, device=dev), dv=t.empty(self.n, device=dev),
                     dhp=t.empty(4, dtype=t.float64, device=dev))
            self.sets.append(s)
        self.ws = self.tree.workspace(dev)
        bpe_state = 2 if bf16 else 4
        self.bytes_fwd = self.n * (4 + 2 * bpe_state + 4 + 2 * bpe_state)
        self.bytes_bwd = self.n * (4 + 2 * bpe_state + 12 + 12)

    def fwd(self, s):
        self.L.opt_adam_fwd(self.tree, STEP_T, HP, self.sd, self.compute, s["g"], s["m"], s["v"],
                            s["u"], s["m1"], s["v1"])

    def bwd(self, s):
        self.L.opt_adam_bwd(self.tree, STEP_T, HP, self.sd, self.compute, s["g"], s["m"], s["v"],
                            s["du"], s["dm1"], s["dv1"], s["dg"], s["dm"], s["dv"], s["dhp"],
                            None, self.ws)


def time_ours(args, workload_inputs, dev, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2211_06934_b200 import _lib as L

    x, offsets, wname = workload_inputs
    compute = {"default": 0, "f32": 1, "f64": 2}[args.compute]
    n = int(offsets[-1])
    # rotate buffer sets so no step re-reads what the previous one left in L2
    bytes_per_set = n * 4 * 12
    sets = max(2, min(8, int(np.ceil(3 * 126e6 / max(bytes_per_set, 1))) + 1))
    W = AdamWorkload(L, x, offsets, dev, sets, compute, bf16=args.bf16)
    stream = torch.cuda.current_stream()
    sampler = ClockSampler(torch.cuda.current_device())

    def step(i):
        s = W.sets[i % sets]
        W.fwd(s)
        W.bwd(s)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    sampler.start()
    # clock soak: keep the GPU busy ~0.5 s (untimed) so the sampler sees load
    t_end = time.time() + (0.3 if args.quick else 0.5)
    i = 0
    while time.time() < t_end:
        for _ in range(50):
            step(i)
            i += 1
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.opt_launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for k in range(args.steps):
        s = W.sets[k % sets]
        W.fwd(s)
        W.bwd(s)
    ev[1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.opt_launch_count() - launches0
    ms = ev[0].elapsed_time(ev[1])
    # per-kernel average launch durations for the roofline: K back-to-back
    # launches of each kernel alone (same rotating buffer sets), bracketed by
    # CUDA events on the launching stream; an event between every launch
    # would itself perturb the back-to-back scheduling being measured.
    def loop_ms(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(args.steps):
            fn(W.sets[k % sets])
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    # 5 alternating repetitions, median reported (one 20-launch sample is
    # ~1.4 ms and a transient clock dip can move it by 10%+)
    fwd_ms, bwd_ms = [], []
    for _ in range(5):
        fwd_ms.append(loop_ms(W.fwd))
        bwd_ms.append(loop_ms(W.bwd))
    clocks = sampler.stop()
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # end-to-end through the C ABI with host buffers (pinned), copies timed
    e2e = None if args.quick else time_e2e(args, W, dev)
    if e2e is not None and world > 1:  # whole-job value: slowest rank, all ranks' bytes
        tt = torch.tensor([e2e["ms_per_step"]], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e["ms_per_step"] = float(tt.item())
        e2e["value"] = round(world * (W.bytes_fwd + W.bytes_bwd) / (e2e["ms_per_step"] * 1e-3)
                             / 1e9, 2)
        e2e["h2d_bytes_per_step"] *= world
        e2e["d2h_bytes_per_step"] *= world
    return dict(ms=ms, fwd_ms=fwd_ms, bwd_ms=bwd_ms, clocks=clocks, launches=launches, W=W,
                e2e=e2e, wname=wname, sets=sets)


def time_e2e(args, W, dev):
    """End-to-end through the public API with HOST buffers: the inputs live
    in pinned host memory and the outputs land there. Primary: the streamed
    path (offload.HostStreamedAdam: chunked H2D / fused kernels / D2H on
    three streams); also reported: plain serial staging (all H2D, the two
    C-ABI calls, all D2H)."""
    import torch

    from paper_2211_06934_b200.offload import HostStreamedAdam, IN_KEYS, OUT_KEYS

    t = torch
    s0 = W.sets[0]
    ins = [k for k in ("g", "m", "v", "du", "dm1", "dv1") if s0[k] is not None]
    outs = ["u", "m1", "v1", "dg", "dm", "dv", "dhp"]
    h_in = {k: s0[k].cpu().pin_memory() for k in ins}
    h_out = {k: t.empty_like(s0[k], device="cpu").pin_memory() for k in outs}
    stream = t.cuda.current_stream()
    steps = max(3, min(args.steps, 20))

    def timed(fn):
        for _ in range(2):
            fn()
        t.cuda.synchronize()
        a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        t.cuda.synchronize()
        return a.elapsed_time(b) / steps

    def serial():
        for k in ins:
            s0[k].copy_(h_in[k], non_blocking=True)
        W.fwd(s0)
        W.bwd(s0)
        for k in outs:
            h_out[k].copy_(s0[k], non_blocking=True)

    ms_serial = timed(serial)
    out = {"serial_ms_per_step": round(ms_serial, 4)}
    if W.sd == 0 and W.n >= 1 << 16 and len(ins) == 6:
        chunks = int(os.environ.get("E2E_CHUNKS", "12"))
        hs = HostStreamedAdam(W.n, dev, chunks=chunks, compute=W.compute)
        hin, hout = HostStreamedAdam.alloc_host(W.n)  # rows of one pinned buffer per direction
        for k in IN_KEYS:
            hin[k].copy_(h_in[k])
        ms = timed(lambda: hs.run(hin, hout, STEP_T, HP, inputs_on_host=True))
        h2d, d2h = hs.bytes_h2d(), hs.bytes_d2h()
        how = ("paper_2211_06934_b200.offload.HostStreamedAdam: pinned host inputs/outputs "
               f"(rows of one buffer per direction), {chunks} chunks, one strided H2D / "
               "opt_adam_fwd+bwd / one strided D2H per chunk overlapped on 3 streams, "
               "consecutive steps pipelined (inputs_on_host=True); all copies inside the "
               "timed region")
    else:
        ms = ms_serial
        h2d = sum(h_in[k].numel() * h_in[k].element_size() for k in ins)
        d2h = sum(h_out[k].numel() * h_out[k].element_size() for k in outs)
        how = "serial staging: H2D of the inputs, opt_adam_fwd/bwd, D2H of the outputs"
    out.update({"value": round((W.bytes_fwd + W.bytes_bwd) / (ms * 1e-3) / 1e9, 2),
                "unit": "GB/s", "ms_per_step": round(ms, 4), "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "how": how})
    return out


# --------------------------------------------------- CPU oracle timing
def time_oracle(x, offsets, max_elems=None, threads=0):
    """Oracle (as it stands, fp64) fwd + VJP on a bounded sample: whole
    leaves of the same workload up to max_elems elements."""
    import oracle

    n = int(offsets[-1])
    if max_elems is not None and max_elems < n:
        n = max_elems
    sl = slice(0, n)
    xs = {k: (None if x[k] is None else x[k][sl]) for k in x}
    # all host cores (torchrun exports OMP_NUM_THREADS=1, which would cap OpenMP's default)
    used = oracle.set_num_threads(threads or len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    oracle.adam_fwd(xs["g"], xs["m"], xs["v"], STEP_T, *HP)
    oracle.adam_vjp(xs["g"], xs["m"], xs["v"], xs["du"], xs["dm1"], xs["dv1"], STEP_T, *HP)
    dt = time.perf_counter() - t0
    oracle.set_num_threads(1)
    gbs = n * (BYTES_FWD + BYTES_BWD) / dt / 1e9
    return dict(value=gbs, unit="GB/s", cores=used, kind="oracle", seconds=dt,
                sample=f"first {n} of {int(offsets[-1])} elements of the same tree "
                       f"(fwd + VJP, fp64, {used} threads)")


def workload(args):
    if args.workload == "c1":
        return c1_inputs()
    if args.workload == "c5":
        return c5_inputs(args.size)
    return c2_inputs()


def traffic_from_profiles(wname, compute):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{wname}|{compute}|bwd")


def relaunch(n):
    """Re-run this command as N local ranks under torch.distributed.run."""
    import socket

    with socket.socket() as so:  # a free rendezvous port on the loopback interface
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, world, rank):
    """Launcher / timing plumbing without a GPU (--dry-run): every rank runs a
    trivial host step, timing follows the real contract (barrier on both
    sides, max over ranks), rank 0 prints the line with the rank PIDs."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group(args.dist_backend if args.dist_backend == "gloo" else "gloo")
    x = torch.zeros(1 << 16)
    for _ in range(args.warmup):
        x.add_(1.0)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x.add_(1.0)
    ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        pids = [None] * world
        dist.all_gather_object(pids, os.getpid())
        dist.destroy_process_group()
    else:
        pids = [os.getpid()]
    if rank == 0:
        print(json.dumps({"metric": "dry-run (launcher plumbing, no GPU work)", "value": None,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(ms / max(args.steps, 1), 6), "dry_run": True,
                          "rank_pids": pids}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--compute", default="default", choices=["default", "f32", "f64"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c1", "c5", "c3", "maml", "es"])
    ap.add_argument("--tasks", type=int, default=32, help="MAML meta-batch (C4)")
    ap.add_argument("--checkpoint-every", type=int, default=None,
                    help="C3: keep only every c-th state and recompute segments (NEXT-2)")
    ap.add_argument("--no-graph", action="store_true", help="MAML without CUDA-graph capture")
    ap.add_argument("--no-fuse-glue", action="store_true",
                    help="C3: separate inner-loss glue kernels (NEXT-2 fusion off)")
    ap.add_argument("--maml-impl", default="explicit", choices=["explicit", "batched", "streams"],
                    help="MAML shard: the hand-scheduled forward-over-reverse step "
                         "(maml_explicit), the autograd task-batched network, or per-task "
                         "graph branches")
    ap.add_argument("--maml-net", default="fused", choices=["gemm", "cudnn", "fused"],
                    help="MAML task-batched network form (maml.conv4_forward_tasks)")
    ap.add_argument("--maml-streams", type=int, default=8,
                    help="MAML (--maml-impl streams): parallel task branches in the graph")
    ap.add_argument("--maml-inner", default="sgd", choices=["sgd", "adam"],
                    help="MAML inner optimizer (explicit step): SGD momentum (C4) or Adam")
    ap.add_argument("--maml-serial", action="store_true",
                    help="MAML (--maml-impl explicit): no side stream (A/B of the concurrency)")
    ap.add_argument("--maml-outer", default="adam", choices=["adam", "peer"],
                    help="MAML outer step: NCCL all-reduce + replicated fused Adam, or the "
                         "all-reduce fused into a sharded Adam over peer memory")
    ap.add_argument("--maml-groups", type=int, default=None,
                    help="MAML: task groups run as concurrent graph branches (default: explicit "
                         "-> one group per task when a rank has <= 4 tasks, else 1; batched -> 1)")
    ap.add_argument("--size", type=int, default=1 << 24)
    ap.add_argument("--bf16", action="store_true", help="bf16 optimizer state")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 plumbing test on fewer GPUs (gloo; not a bench value)")
    ap.add_argument("--no-maml", action="store_true",
                    help="default workload: skip the C4 MAML tasks/s measurement (maml_c4)")
    ap.add_argument("--quick", action="store_true", help="skip e2e and clock soak (tuning)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="default workload: skip the secondary config keys (c1, c3, c5, es)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/timing plumbing only (no GPU work; gloo)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    world, rank, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.warmup < 3:
        args.warmup = 3
    if args.dry_run:
        return dry_run(args, world, rank)

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    # one process per GPU; --dist-backend gloo with more ranks than GPUs is a
    # plumbing test only (ranks share devices; numbers are not bench values)
    gpu = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(gpu)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", gpu)
    torch.cuda.set_device(dev)
    if args.workload == "c3":
        return run_sweep(args, dev, rank, world)
    if args.workload == "maml":
        return run_maml(args, dev, rank, world)
    if args.workload == "es":
        return run_es(args, dev, rank, world)
    wl = workload(args)
    r = time_ours(args, wl, dev, rank, world)
    W = r["W"]
    ms_step = r["ms"] / args.steps
    per_rank_bytes = W.bytes_fwd + W.bytes_bwd
    value = world * per_rank_bytes * args.steps / (r["ms"] * 1e-3) / 1e9
    peak, peak_src = peaks()
    bwd_avg = statistics.median(r["bwd_ms"])
    fwd_avg = statistics.median(r["fwd_ms"])
    achieved = W.bytes_bwd / (bwd_avg * 1e-3) / 1e9
    compute_name = {"default": "f32", "f32": "f32", "f64": "f64"}[args.compute]
    from paper_2211_06934_b200 import _lib as L
    out = {
        "metric": "diff-Adam fwd+bwd GB/s",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": compute_name,
        "data": "synthetic (seeded SplitMix64/Box-Muller; DESIGN.md input recipe)",
        "config": {"workload": r["wname"] + " adam fwd+bwd", "numel": W.n,
                   "n_leaves": W.tree.n_leaves, "state": "bf16" if args.bf16 else "f32",
                   "compute": compute_name, "step_t": STEP_T,
                   "l2": f"{r['sets']} rotating buffer sets of {W.n * 48 / 1e6:.0f} MB (> 126 MB L2)",
                   "parallelism": f"replicas x{world} (no data-path collective)",
                   "alg_bytes_per_step": per_rank_bytes},
        "frac_of_measured_hbm": round(value / world / peak, 4),
        "frac_of_nominal_8tbs": round(value / world / NOMINAL_HBM, 4),
        "fwd_ms": round(fwd_avg, 5), "bwd_ms": round(bwd_avg, 5),
        "fwd_gbs": round(W.bytes_fwd / (fwd_avg * 1e-3) / 1e9, 1),
        "clocks": r["clocks"],
        "e2e": r["e2e"],
        "gpu_launches": r["launches"],
        "roofline": {"bound": "hbm", "kernel": "step_uniform<AdamBwd> (opt_adam_bwd)",
                     "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic_from_profiles(r["wname"], compute_name),
                     "alg_bytes_per_launch": W.bytes_bwd,
                     "share_of_step": round(bwd_avg / (fwd_avg + bwd_avg), 3),
                     "how": "avg duration of K back-to-back opt_adam_bwd launches (CUDA "
                            "events on the launching stream around the loop), median of 5 "
                            "repetitions"},
        "libdiffopt_abi": L.opt_abi_version(),
    }
    if not args.no_maml:  # second half of the BASELINE metric: C4 tasks/s at this N
        try:
            m = measure_maml(args, dev, rank, world, steps=10)
            out["maml_c4"] = {k: m[k] for k in ("metric", "value", "unit", "ms_per_step", "steps",
                                                "scaling", "tasks_per_rank", "allreduce_ms",
                                                "allreduce_bytes", "gpu_launches")}
            out["maml_c4"]["config"] = m["config"]
            if world == 1 and args.tasks == 32 and args.maml_impl == "explicit":
                out["maml_c4_projection"] = maml_projection(args, dev, m["ms_per_step"])
        except Exception as e:  # never lose the headline line to the secondary workload
            out["maml_c4"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if world == 1 and not args.no_secondary and args.workload == "c2":
        out.update(secondary_configs(args, dev))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x, offsets, _ = wl
        cb = {k: v for k, v in time_oracle(x, offsets).items() if k != "seconds"}
        one = time_oracle(x, offsets, max_elems=1 << 20, threads=1)
        cb["one_thread"] = {"value": round(one["value"], 4), "unit": "GB/s", "cores": 1,
                            "sample": one["sample"]}
        cb["cpu_model"] = cpu_model()
        cb["host_cores"] = len(os.sched_getaffinity(0))
        out["cpu_baseline"] = cb
    out["paper_context"] = PAPER_CONTEXT
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


PAPER_CONTEXT = {
    "gpu_vs_cpu_optimizer_speedup": "5-20x (P:39; TorchOpt's CUDA vs CPU optimizer ops; "
                                    "hardware not stated, figures stripped)",
    "distributed_maml_8gpu_speedup": "5.2x on 8 GPUs (P:10, P:39, Fig. 3(c) P:262; "
                                     "hardware not stated)",
    "note": "context only: other hardware and workloads; not the target of this line",
}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


# bytes per element per call (each non-NULL array read or written once;
# DESIGN.md "Algorithmic bytes"): (fwd, bwd) for fp32 state / bf16 state
ALG_BYTES = {"adam": ((24, 36), (16, 32)), "rmsprop": ((16, 24), (12, 22)),
             "sgd": ((16, 24), (12, 22))}


def _loop_ms(fn, k, stream):
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(k):
        fn(i)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


def c5_point(L, op, n, bf16, dev, steps, warmup):
    """One C5 point: K back-to-back forward launches, then K backward launches
    (with hyper-gradients), CUDA events on the launching stream; inputs drawn
    on the device (synth.device_state_flat: the C5 recipe); 2 rotating
    buffer sets below 2^26 elements so no launch re-reads L2-resident data."""
    import torch

    nsets = 2 if n < (1 << 26) else 1
    sdt = torch.bfloat16 if bf16 else torch.float32
    sets = []
    for k in range(nsets):
        x = synth.device_state_flat(0xC5 + k, n, dev)
        s = {"g": x["g"], "du": x["du"]}
        if op == "adam":
            s.update(s0=x["m"].to(sdt), s1=x["v"].to(sdt), c0=x["dm1"], c1=x["dv1"])
        elif op == "rmsprop":
            s.update(s0=x["v"].to(sdt), c0=x["dv1"])
        else:
            s.update(s0=x["m"].to(sdt), c0=x["dm1"])
        del x
        s["u"] = torch.empty(n, device=dev)
        s["o0"] = torch.empty(n, dtype=sdt, device=dev)
        s["dg"] = torch.empty(n, device=dev)
        s["d0"] = torch.empty(n, device=dev)
        if op == "adam":
            s["o1"] = torch.empty(n, dtype=sdt, device=dev)
            s["d1"] = torch.empty(n, device=dev)
        s["dhp"] = torch.empty(4, dtype=torch.float64, device=dev)
        sets.append(s)
    tree = L.Tree(numel=n, device=dev)
    ws = tree.workspace(dev)
    sd = 1 if bf16 else 0
    hp = {"adam": HP, "rmsprop": (1e-2, 0.99, 1e-8), "sgd": (0.1, 0.9, False)}[op]

    def fwd(i):
        s = sets[i % nsets]
        if op == "adam":
            L.opt_adam_fwd(tree, STEP_T, hp, sd, 0, s["g"], s["s0"], s["s1"], s["u"], s["o0"],
                           s["o1"])
        elif op == "rmsprop":
            L.opt_rmsprop_fwd(tree, hp, sd, 0, s["g"], s["s0"], s["u"], s["o0"])
        else:
            L.opt_sgd_fwd(tree, hp, sd, 0, s["g"], s["s0"], s["u"], s["o0"])

    def bwd(i):
        s = sets[i % nsets]
        if op == "adam":
            L.opt_adam_bwd(tree, STEP_T, hp, sd, 0, s["g"], s["s0"], s["s1"], s["du"], s["c0"],
                           s["c1"], s["dg"], s["d0"], s["d1"], s["dhp"], None, ws)
        elif op == "rmsprop":
            L.opt_rmsprop_bwd(tree, hp, sd, 0, s["g"], s["s0"], s["du"], s["c0"], s["dg"],
                              s["d0"], s["dhp"], None, ws)
        else:
            L.opt_sgd_bwd(tree, hp, sd, 0, s["g"], s["s0"], s["du"], s["c0"], s["dg"], s["d0"],
                          s["dhp"], None, ws)

    stream = torch.cuda.current_stream()
    for i in range(warmup):
        fwd(i)
        bwd(i)
    torch.cuda.synchronize()
    fms = _loop_ms(fwd, steps, stream)
    bms = _loop_ms(bwd, steps, stream)
    del sets, ws
    torch.cuda.empty_cache()
    bf, bb = ALG_BYTES[op][1 if bf16 else 0]
    peak, _ = peaks()
    fg, bg = n * bf / (fms * 1e-3) / 1e9, n * bb / (bms * 1e-3) / 1e9
    return {"n": n, "op": op, "state": "bf16" if bf16 else "f32",
            "fwd_us": round(fms * 1e3, 2), "bwd_us": round(bms * 1e3, 2),
            "fwd_gbs": round(fg, 1), "bwd_gbs": round(bg, 1),
            "fwd_frac": round(fg / peak, 4), "bwd_frac": round(bg / peak, 4)}


def secondary_configs(args, dev):
    """The other BASELINE.json configs as secondary keys of the default line
    (driver-visible), each with its own roofline fraction against the same
    measured copy peak. Failures are reported in place, never fatal."""
    import torch

    from paper_2211_06934_b200 import _lib as L

    peak, _ = peaks()
    steps, warmup = max(5, min(args.steps, 20)), max(3, args.warmup)
    res = {}
    # C1: 4096 elements, zero state, t = 1 -- launch-bound. Host-call path
    # (one C-ABI call per kernel) and the same two calls replayed from a CUDA
    # graph (device-bound: the library calls are capturable).
    try:
        x = synth.c1_inputs()
        W = AdamWorkload(L, x, np.array([0, x["g"].size], np.int64), dev, 1, 0)
        s = W.sets[0]

        def c1_step(i):
            L.opt_adam_fwd(W.tree, 1, HP, 0, 0, s["g"], None, None, s["u"], s["m1"], s["v1"])
            L.opt_adam_bwd(W.tree, 1, HP, 0, 0, s["g"], None, None, s["du"], s["dm1"], s["dv1"],
                           s["dg"], None, None, s["dhp"], None, W.ws)

        stream = torch.cuda.current_stream()
        for i in range(20):
            c1_step(i)
        torch.cuda.synchronize()
        host_ms = _loop_ms(c1_step, 1000, stream)
        # the same two calls pre-marshalled (_lib.prepare_adam_*: one ctypes call each)
        pf = L.prepare_adam_fwd(W.tree, HP, 0, 0, s["g"], None, None, s["u"], s["m1"], s["v1"])
        pb = L.prepare_adam_bwd(W.tree, HP, 0, 0, s["g"], None, None, s["du"], s["dm1"],
                                s["dv1"], s["dg"], None, None, s["dhp"], None, W.ws)

        def c1_prepared(i):
            pf(1)
            pb(1)

        for i in range(20):
            c1_prepared(i)
        prep_ms = _loop_ms(c1_prepared, 1000, stream)
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            c1_step(0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            for i in range(100):
                c1_step(i)
        g.replay()
        torch.cuda.synchronize()
        graph_ms = _loop_ms(lambda i: g.replay(), 20, stream) / 100
        nb = x["g"].size * (4 + 12) + x["g"].size * (4 + 12 + 12)  # NULL state: g, cots only
        res["c1"] = {"metric": "C1 diff-Adam fwd+bwd us/step", "unit": "us/step",
                     "host_call_us": round(host_ms * 1e3, 3),
                     "prepared_call_us": round(prep_ms * 1e3, 3),
                     "graph_replay_us": round(graph_ms * 1e3, 3), "alg_bytes_per_step": nb,
                     "roofline": {"bound": "launch latency", "achieved_gbs":
                                  round(nb / (graph_ms * 1e-3) / 1e9, 1), "peak": peak,
                                  "frac": round(nb / (graph_ms * 1e-3) / 1e9 / peak, 4)},
                     "note": "4096 elements: the HBM floor is ~40 ns, so every number is "
                             "launch/latency bound; prepared calls skip the per-call argument "
                             "marshalling, graph replay removes the host path"}
        del W, g
    except Exception as e:  # noqa: BLE001
        res["c1"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    # C5: bandwidth sweep points (Adam 2^24 / 2^28 / 2^30, RMSProp / SGD at
    # 2^28; fp32 and bf16 state)
    pts = []
    try:
        for op, n in [("adam", 1 << 24), ("adam", 1 << 28), ("adam", 1 << 30),
                      ("rmsprop", 1 << 28), ("sgd", 1 << 28)]:
            for bf16 in (False, True):
                pts.append(c5_point(L, op, n, bf16, dev, steps, warmup))
        worst = min(min(p["fwd_frac"], p["bwd_frac"]) for p in pts)
        res["c5"] = {"metric": "C5 fwd/bwd GB/s sweep", "unit": "GB/s", "points": pts,
                     "roofline": {"bound": "hbm", "peak": peak, "min_frac": worst},
                     "data": "synthetic, drawn on the device (synth.device_state_flat)"}
    except Exception as e:  # noqa: BLE001
        res["c5"] = {"error": f"{type(e).__name__}: {e}"[:300], "points": pts}
    torch.cuda.empty_cache()
    # C3: 5-step unrolled Adam + reverse sweep over the 9 x ResNet-18 tree
    try:
        from paper_2211_06934_b200.unroll import QuadraticSweep

        leaves = synth.RESNET18_LEAVES * 9
        off = synth.offsets_of(leaves)
        n = int(off[-1])
        gen = torch.Generator(device=dev).manual_seed(0xC3)
        a = 0.5 + torch.rand(n, device=dev, generator=gen)
        th0, phi, y = (torch.randn(n, device=dev, generator=gen) for _ in range(3))
        sw = QuadraticSweep(L.Tree(offsets=off, device=dev), "adam", (1e-2, 0.9, 0.999, 1e-8, 0.0),
                            5, dev, fuse_glue=True)
        ms = _timed(lambda i: sw.run(a, th0, phi, y), min(steps, 10), warmup, 1) / min(steps, 10)
        per = sw.alg_bytes()
        res["c3"] = {"metric": "C3 5-step unrolled diff-Adam sweep GB/s", "unit": "GB/s",
                     "value": round(per / (ms * 1e-3) / 1e9, 1), "ms_per_step": round(ms, 4),
                     "numel": n, "alg_bytes_per_step": per, "fused_glue": True,
                     "roofline": {"bound": "hbm", "peak": peak,
                                  "frac": round(per / (ms * 1e-3) / 1e9 / peak, 4)},
                     "data": "synthetic, drawn on the device (a ~ U[0.5,1.5]; theta0, phi, "
                             "y ~ N(0,1))"}
        del sw, a, th0, phi, y
    except Exception as e:  # noqa: BLE001
        res["c3"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    torch.cuda.empty_cache()
    # NEXT-3 ES: antithetic perturbations of a C2-sized theta (bytes written)
    try:
        n = int(sum(synth.RESNET18_LEAVES))
        ns, sigma, seed = 16, 0.01, 5
        theta = torch.randn(n, device=dev)
        pts_es = torch.empty(2 * ns, L.es_row_stride(n), device=dev)
        ms = _timed(lambda i: L.opt_es_perturb(n, ns, 0, True, sigma, seed, theta, pts_es),
                    steps, warmup, 1) / steps
        wb = (2 * ns * n + n) * 4
        res["es"] = {"metric": "NEXT-3 ES perturb GB/s", "unit": "GB/s",
                     "value": round(wb / (ms * 1e-3) / 1e9, 1), "us_per_call": round(ms * 1e3, 2),
                     "roofline": {"bound": "hbm", "peak": peak,
                                  "frac": round(wb / (ms * 1e-3) / 1e9 / peak, 4)}}
        del pts_es
    except Exception as e:  # noqa: BLE001
        res["es"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    torch.cuda.empty_cache()
    return res


def _timed(fn, steps, warmup, world):
    import torch
    import torch.distributed as dist

    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        fn(warmup + i)
    b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def run_sweep(args, dev, rank, world):
    """C3: 5-step unrolled Adam + reverse meta-gradient sweep over a
    9 x ResNet-18 tree (558 leaves, 105,205,608 elements); replicas per rank."""
    import torch

    from paper_2211_06934_b200 import _lib as L
    from paper_2211_06934_b200.unroll import QuadraticSweep

    leaves = synth.RESNET18_LEAVES * 9
    off = synth.offsets_of(leaves)
    n = int(off[-1])
    q = synth.quadratic_problem(0xC3, n)
    tree = L.Tree(offsets=off, device=dev)
    hp = (1e-2, 0.9, 0.999, 1e-8, 0.0)
    sw = QuadraticSweep(tree, "adam", hp, 5, dev, checkpoint_every=args.checkpoint_every,
                        fuse_glue=not args.no_fuse_glue)
    a, th0, phi, y = (torch.from_numpy(q[k]).to(dev) for k in ("a", "theta0", "phi", "y"))
    del q
    l0 = L.opt_launch_count()
    ms = _timed(lambda i: sw.run(a, th0, phi, y), args.steps, args.warmup, world)
    launches = (L.opt_launch_count() - l0) * args.steps // (args.steps + args.warmup)
    per = sw.alg_bytes()
    value = world * per * args.steps / (ms * 1e-3) / 1e9
    peak, src = peaks()
    out = {"metric": "diff-Adam 5-step unrolled sweep GB/s", "value": round(value, 1),
           "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": "C3 5-step unrolled Adam + reverse sweep, 9x resnet18 tree",
                      "numel": n, "n_leaves": len(leaves), "K": 5,
                      "checkpoint_every": sw.c, "saved_state_bytes": sw.saved_bytes(),
                      "fused_glue": sw.fuse,
                      "alg_bytes_per_step": per, "launches_per_step": sw.launches_per_sweep},
           "frac_of_measured_hbm": round(value / world / peak, 4),
           "gpu_launches": launches}
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_es(args, dev, rank, world):
    """NEXT-3: zero-order ES on a C2-sized parameter vector: perturbation
    generation (bytes written) and the estimate (normals regenerated / s)."""
    import torch

    from paper_2211_06934_b200 import _lib as L

    n = int(sum(synth.RESNET18_LEAVES))
    ns, sigma, seed = 16, 0.01, 5
    ld = L.es_row_stride(n)
    theta = torch.randn(n, device=dev, generator=torch.Generator(device=dev).manual_seed(0))
    pts = torch.empty(2 * ns, ld, device=dev)
    f = torch.randn(2 * ns, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
    g = torch.empty(n, device=dev)
    ms_p = _timed(lambda i: L.opt_es_perturb(n, ns, 0, True, sigma, seed, theta, pts),
                  args.steps, args.warmup, world)
    ms_g = _timed(lambda i: L.opt_es_grad(n, ns, True, sigma, seed, f, g), args.steps, args.warmup,
                  world)
    wbytes = (2 * ns * n + n) * 4
    peak, _ = peaks()
    out = {"metric": "ES perturb GB/s", "value": round(wbytes * args.steps / (ms_p * 1e-3) / 1e9, 1),
           "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms_p / args.steps, 4), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": "NEXT-3 ES antithetic, C2-sized theta", "numel": n,
                      "samples": ns, "alg_bytes_perturb": wbytes},
           "frac_of_measured_hbm": round(wbytes * args.steps / (ms_p * 1e-3) / 1e9 / peak, 4),
           "es_grad_ms": round(ms_g / args.steps, 4),
           "es_grad_gnormals_per_s": round(ns * n * args.steps / (ms_g * 1e-3) / 1e9, 2)}
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_maml(args, dev, rank, world):
    """C4: MAML meta-batch of --tasks tasks, sharded over ranks, one NCCL
    all-reduce per outer step; value = tasks/s over all ranks."""
    out = measure_maml(args, dev, rank, world)
    if rank == 0:
        print(json.dumps(out), flush=True)


def maml_projection(args, dev, t32_ms):
    """Strong-scaling projection from ONE GPU: the step time of the shard a
    rank holds at N = 2, 4, 8 GPUs (32/N tasks, that rank's default task
    groups) measured here; tasks/s(N) = 32 / t(32/N). Excludes the NCCL
    all-reduce of the 449 KB meta-gradient (~20-30 us over NVLink)."""
    import copy

    shard = {"32": round(t32_ms, 3)}
    for k in (16, 8, 4):
        a2 = copy.copy(args)
        a2.tasks, a2.maml_groups = k, None
        shard[str(k)] = measure_maml(a2, dev, 0, 1, steps=10)["ms_per_step"]
    tps = {str(n): round(32 / (shard[str(32 // n)] * 1e-3), 1) for n in (1, 2, 4, 8)}
    return {"method": "per-rank shard step times measured on this GPU (32/N tasks per rank, "
                      "default task groups); projected tasks/s(N) = 32 / t(32/N); excludes the "
                      "~20-30 us meta-gradient all-reduce; a projection, not a multi-GPU run",
            "shard_ms": shard, "projected_tasks_per_s": tps,
            "projected_scaling": {n: round(shard["32"] / shard[str(32 // int(n))], 3)
                                  for n in ("2", "4", "8")},
            "paper": "5.2x on 8 GPUs (P:10, P:39; hardware not stated)",
            "north_star_target": ">= 6x from 1 to 8 GPUs"}


def measure_maml(args, dev, rank, world, steps=None):
    import torch

    from paper_2211_06934_b200 import _lib as L
    from paper_2211_06934_b200 import maml

    cfg = maml.MamlConfig(tasks=args.tasks, net=args.maml_net, inner_opt=args.maml_inner,
                          inner_lr=0.1 if args.maml_inner == "sgd" else 0.01)
    phi = maml.init_params(0, dev)
    inner = maml.FusedSgdInner(maml.sizes_of(maml.CONV4_SHAPES), dev, cfg)
    if args.maml_outer == "peer":  # all-reduce fused into the outer step (peer memory)
        outer = maml.PeerAdamOuter(phi.numel(), world, rank, dev, cfg.outer_lr, cfg.tasks)
    else:
        outer = maml.FusedAdamOuter(phi.numel(), dev, cfg.outer_lr)
    state = {"phi": phi}
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = False   # fp32 convolutions (dtype f32)
    torch.backends.cuda.matmul.allow_tf32 = False
    shard = None
    my_tasks = len(maml.task_range(world, rank, cfg.tasks))
    if args.maml_groups is None:  # measured (profiles/r02aa_*, r02ab_*): concurrent
        # task-group chains win at <= 16 tasks per rank: 4, 8 and 16 -> 4 chains, 32 -> 1
        from paper_2211_06934_b200.maml_explicit import default_groups

        args.maml_groups = default_groups(my_tasks) if args.maml_impl == "explicit" else 1
    if args.maml_impl == "explicit":
        from paper_2211_06934_b200 import maml_explicit

        shard = maml_explicit.ExplicitShard(maml.task_range(world, rank, cfg.tasks), cfg, dev,
                                            concurrent=not args.maml_serial,
                                            groups=args.maml_groups)
    elif not args.no_graph:
        shard = maml.GraphedShard(maml.task_range(world, rank, cfg.tasks), cfg, inner, dev,
                                  streams=(args.maml_groups if args.maml_impl == "batched"
                                           else args.maml_streams),
                                  batched=args.maml_impl == "batched")

    ar = []

    def step(i):
        state["phi"], loss, _ = maml.outer_step(state["phi"], i, cfg, inner, outer, world, rank,
                                                shard=shard, allreduce_events=ar)

    steps = max(1, min(args.steps, 20)) if steps is None else steps
    l0 = L.opt_launch_count()
    ms = _timed(step, steps, args.warmup, world)
    ar_ms = [a.elapsed_time(b) for a, b in ar[-steps:]] if ar else []
    launches = (L.opt_launch_count() - l0) * steps // (steps + args.warmup)
    if shard is not None:  # library launches replayed inside the CUDA graph
        launches += shard.launches_per_replay * steps
    value = cfg.tasks * steps / (ms * 1e-3)
    out = {"metric": "MAML meta-batch tasks/s", "value": round(value, 2), "unit": "tasks/s",
           "n_gpus": world, "steps": steps, "warmup": args.warmup,
           "ms_per_step": round(ms / steps, 3), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded 5-way tasks)",
           "config": {"workload": ("C4 MAML 4-conv64, 5-way 5-shot 15-query, 5 inner "
                                   + ("SGD-mom" if cfg.inner_opt == "sgd" else "Adam") + " steps"),
                      "tasks": cfg.tasks,
                      "parallelism": (f"task-sharded x{world}, " + (
                          "all-reduce fused into the outer step (peer memory)"
                          if args.maml_outer == "peer" else
                          f"{'NCCL' if args.dist_backend == 'nccl' else 'gloo'} all-reduce")),
                      "cuda_graph": shard is not None,
                      "shard_impl": ("eager per-task" if shard is None else
                                     f"hand-scheduled forward-over-reverse graph (explicit), "
                                     f"{shard.nstreams} task group(s)"
                                     if args.maml_impl == "explicit" else
                                     f"task-batched graph ({cfg.net}), {shard.nstreams} "
                                     "concurrent group(s)" if shard.batched else
                                     f"graph, {shard.nstreams} task branches")},
           "tasks_per_rank": len(maml.task_range(world, rank, cfg.tasks)),
           "allreduce_ms": (round(statistics.mean(ar_ms), 4) if ar_ms and world > 1 else None),
           "allreduce_bytes": (phi.numel() + 1) * 4,
           "gpu_launches": launches}
    return out


def run_reference(args, world, rank):
    """Reference arm: the oracle (CPU, fp64, all host cores) on a bounded
    sample of the same workload, timed per step; rank 0 only."""
    if rank != 0:
        return
    x, offsets, wname = workload(args)
    n = int(offsets[-1])
    sample = min(n, 1 << 21)
    for _ in range(min(args.warmup, 1)):
        time_oracle(x, offsets, sample)
    times = []
    info = None
    for _ in range(args.steps if args.steps <= 5 else 5):
        info = time_oracle(x, offsets, sample)
        times.append(info["seconds"])
    sec = statistics.median(times)
    value = sample * (BYTES_FWD + BYTES_BWD) / sec / 1e9
    out = {"metric": "diff-Adam fwd+bwd GB/s", "value": round(value, 3), "unit": "GB/s",
           "impl": "reference", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
           "ms_per_step": round(sec * 1e3 * n / sample, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": wname + " adam fwd+bwd", "numel": n},
           "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": info["cores"],
                            "kind": "oracle", "sample": info["sample"]},
           "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
