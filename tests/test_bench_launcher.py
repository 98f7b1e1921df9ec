"""bench.py's N-rank launcher on the CPU box (`--gpus N` must
launch N ranks itself): `--gpus 2` without a torch.distributed environment
re-launches under torch.distributed.run; the dry run exercises rendezvous,
barriers and the max-over-ranks timing with gloo, no GPU work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    if env:
        e.update(env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e,
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def _line(stdout):
    lines = [l for l in stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, stdout
    return json.loads(lines[0])


def test_gpus_2_launches_two_ranks():
    r = _run(["--gpus", "2", "--dist-backend", "gloo", "--dry-run", "--steps", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert len(set(d["rank_pids"])) == 2 and os.getpid() not in d["rank_pids"]


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0",
                                               "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_reference_arm_prints_once_from_rank_0():
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"],
             timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle"


def test_explicit_maml_default_groups_policy():
    """Task groups per shard size for the explicit MAML step (measured sweep,
    profiles/r02ab_task_groups.txt): the 1/2/4/8-GPU shards of 32 tasks."""
    from paper_2211_06934_b200.maml_explicit import default_groups

    assert [default_groups(t) for t in (32, 16, 8, 4, 2, 1)] == [1, 4, 4, 4, 2, 1]
    assert default_groups(0) == 1
