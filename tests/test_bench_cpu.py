"""bench.py contract pieces that run without a GPU: the reference arm prints
exactly one JSON line with the driver's keys, and helper policies."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert "workload" in d["config"]


def test_reference_arm_nonzero_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=120, cwd=ROOT, env=env)
    assert res.returncode == 0 and res.stdout.strip() == ""


def test_chain_chunk_policy():
    sys.path.insert(0, ROOT)
    from paper_2605_13276_b200.replicate import chain_chunk_bytes
    assert chain_chunk_bytes(6_600_000_000) == 1 << 20
    assert chain_chunk_bytes(1_000_000_000) == 256 << 10
    assert chain_chunk_bytes(100_000_000) == 128 << 10
    for s in (16, 10 ** 6, 10 ** 9, 10 ** 11):
        c = chain_chunk_bytes(s)
        assert (128 << 10) <= c <= (1 << 20) and c & (c - 1) == 0
