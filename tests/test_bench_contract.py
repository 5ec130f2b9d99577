"""bench.py's reference arm (the CPU oracle, tier rule) runs without a GPU and prints one
JSON line with the contract's keys; the omniloc arm's JSON assembly is exercised on the GPU
by the driver.  (CPU only; a small sample keeps it to seconds.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                          "--config", "C3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "queries/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["config"]["workload"] == "C3"


def test_gpus_n_starts_n_ranks():
    """`bench.py --gpus N` without a launcher starts N ranks itself (torchrun on 127.0.0.1),
    each seeing WORLD_SIZE = N (it used to run one rank and print n_gpus 1)."""
    env = dict(os.environ, OL_BENCH_RANK_PROBE="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "3"], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    recs = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(r["rank"] for r in recs) == [0, 1, 2]
    assert all(r["world"] == 3 and r["gpus"] == 3 for r in recs)


def test_gpus_must_match_launcher_world():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    env.pop("OL_BENCH_RANK_PROBE", None)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--no-cpu"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300, env=env)
    assert out.returncode != 0
    assert "WORLD_SIZE=1" in out.stderr
