"""bench.py reference arm (CPU only): the JSON line the driver parses.

The reference arm times the reference's own CPU path -- atamul.SharedRunner
installed unmodified into oracle/_ref by oracle/build_ref.sh, or the oracle
port when that is absent -- on a bounded sample of the config; under torchrun
only rank 0 runs and prints.  c1's sample (1024 x 1024) keeps this fast.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None):
    env = dict(os.environ)
    env.update(extra_env or {})
    return subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1",
                           "--steps", "2", "--warmup", "1"], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "AtA effective GFLOP/s (m*n^2/time)" and d["unit"] == "GFLOP/s"
    assert d["higher_is_better"] is True and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.bench_config("c1")      # the same config object as our arm
    cb = d["cpu_baseline"]
    from oracle.cpu_baseline import reference_module
    assert cb["kind"] == ("reference" if reference_module() is not None else "port")
    assert cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    r = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
