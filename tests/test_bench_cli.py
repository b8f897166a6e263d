"""bench.py's command-line contract that needs no GPU: the reference arm
(`--impl reference`: the reference's own CPU code or the oracle port on a
bounded sample, one JSON line with the contract's keys, no product library)
and the refusal to bench fewer GPUs than asked for."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600, env=e)


def test_reference_arm_line():
    r = run("--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0",
            "--cpu-threads", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "Melem/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["n_gpus"] == 1
    assert line["e2e"] == {"value": line["value"], "unit": "Melem/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] == 2 and cb["value"] == line["value"]
    assert cb["single_thread"]["cores"] == 1 and "sample" in cb and cb["nproc"] >= 1
    assert line["config"]["workload"].startswith("C1") or "300" in line["config"]["workload"]


def test_reference_arm_other_ranks_exit_quietly():
    r = run("--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "0",
            env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_more_gpus_than_visible_is_refused():
    import torch
    if torch.cuda.device_count() >= 2:
        import pytest
        pytest.skip("needs fewer than 2 visible GPUs")
    r = run("--gpus", "2", "--steps", "1", "--warmup", "1")
    assert r.returncode == 2
    assert "error" in json.loads(r.stdout.strip().splitlines()[-1])
