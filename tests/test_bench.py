"""bench.py's launch contract on the CPU (reference arm only: no GPU here):
`--gpus N` without a torchrun environment starts N ranks itself, rank 0
alone prints one JSON line, and a WORLD_SIZE that disagrees with --gpus is
refused."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=900, cwd=ROOT, env=e)


def test_reference_arm_relaunches_two_ranks():
    out = _run(["--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "1", "--warmup", "3"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["workload"] == "c1" and d["config"]["parallelism"] == "replicas x2"
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_is_refused():
    out = _run(["--impl", "reference", "--gpus", "2", "--config", "c1"],
               env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0
    assert "WORLD_SIZE" in out.stderr
