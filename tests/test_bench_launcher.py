"""bench.py --gpus N launches N ranks itself (one process per GPU) when no torchrun
environment is present; this CPU test runs the same launcher with the gloo plumbing
self-test (barrier, max-over-ranks time, summed work) at N = 2."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_launcher_two_ranks_gloo():
    env = dict(os.environ, PLUQ_BENCH_ALLOW_CPU_RANKS="1", PLUQ_BENCH_PORT="29731", OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--selftest-ranks",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["selftest"]
    # max over ranks (0.02 s) and summed work (2e9): 100 Gfield-op/s
    assert abs(d["value"] - 100.0) < 1e-6


def test_launcher_refuses_missing_gpus():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("PLUQ_BENCH_ALLOW_CPU_RANKS", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0 and "needs 4 GPUs" in out.stderr
