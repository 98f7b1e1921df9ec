"""Build libdiffopt variants with different launch shapes for a tuning sweep:
tools/tune_build/lib_<tag>.so, tag = U_F-MINB_F-U_B-MINB_B[-extra]."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location(
    "_diffopt_build", os.path.join(ROOT, "paper_2211_06934_b200", "build.py"))
B = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(B)

OUT = os.path.join(ROOT, "tools", "tune_build")


def one(cfg):
    uf, mf, ub, mb, extra = cfg
    tag = f"{uf}-{mf}-{ub}-{mb}" + (f"-{extra}" if extra else "")
    defs = [f"DOPT_U_FWD={uf}", f"DOPT_MINB_FWD={mf}", f"DOPT_U_BWD={ub}", f"DOPT_MINB_BWD={mb}"]
    if "ub" in extra:  # e.g. ub2x2: bf16 U fwd x bwd
        spec = extra.split("ub")[1][:3]
        defs += [f"DOPT_U_FWD_BF16={spec[0]}", f"DOPT_U_BWD_BF16={spec[2]}"]
    import re
    m = re.search(r"ld(\d)", extra)
    if m:
        defs.append(f"DOPT_LD_POLICY={m.group(1)}")
    m = re.search(r"st(\d)", extra)
    if m:
        defs.append(f"DOPT_ST_POLICY={m.group(1)}")
    m = re.search(r"gm(\d+)", extra)
    if m:
        defs.append(f"DOPT_FWD_GRID_MULT={m.group(1)}")
    m = re.search(r"bm(\d+)", extra)
    if m:
        defs.append(f"DOPT_BWD_GRID_MULT={m.group(1)}")
    if "wp" in extra:
        defs.append("DOPT_WARP_PARTIALS=1")
    if "span" in extra:
        defs.append("DOPT_SPAN=1")
    if "pipeF" in extra:
        defs.append("DOPT_PIPE_FWD=1")
    if "pipeB" in extra:
        defs.append("DOPT_PIPE_BWD=1")
    if "pdl" in extra:
        defs.append("DOPT_PDL=1")
    if "ieee" in extra:
        defs.append("DOPT_IEEE_F32")
    if "tma" in extra:
        defs += ["DOPT_TMA_FWD=1", "DOPT_TMA_BWD=1"]
        # extra like tma512x1 : consumers x CTAs per SM
        spec = extra.split("tma")[1]
        if spec:
            nc, ctas = spec.split("x")
            defs += [f"DOPT_TMA_NCONS={nc}", f"DOPT_TMA_CTAS={ctas}"]
    out = os.path.join(OUT, f"lib_{tag}.so")
    B.build(force=True, out=out, defines=defs)
    return out


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    cfgs = []
    for arg in sys.argv[1:]:
        parts = arg.split("-")
        cfgs.append(tuple(int(p) for p in parts[:4]) + ((parts[4] if len(parts) > 4 else ""),))
    with ThreadPoolExecutor(8) as ex:
        for o in ex.map(one, cfgs):
            print(o)
