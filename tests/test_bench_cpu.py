"""bench.py's CPU pieces: the reference arm (the oracle on host cores) prints one valid JSON
line, and the oracle sampler's ratio estimator is consistent with a full oracle run."""
import json
import os
import subprocess
import sys
import time

import oracle
from paper_2405_07989_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json():
    env = dict(os.environ, FS_REF_STEP_SECONDS="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "factorizations/s"
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] == 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0


def test_oracle_sampler_estimates_full_rate(oracle_mod):
    import bench

    inst = W.C2  # small enough to run in full
    t0 = time.perf_counter()
    full = oracle.count(inst.n, inst.gens)
    rate_full = full / (time.perf_counter() - t0)
    rate, rows, secs, boxes = bench.oracle_sample(inst, 1.0)
    assert boxes >= 1 and rows > 0
    assert 0.3 < rate / rate_full < 3.0
