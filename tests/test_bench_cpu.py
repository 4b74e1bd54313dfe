"""bench.py launch contract without a GPU: --gpus N starts N ranks itself (torch.distributed.run on
127.0.0.1) or refuses a mismatching WORLD_SIZE; the reference arm prints one JSON line from rank 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env, cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_world_size_mismatch_fails():
    r = _run(["--gpus", "2", "--config", "1"], {"WORLD_SIZE": "1"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in r.stderr


def test_gpus_spawns_ranks_reference_arm():
    r = _run(["--gpus", "2", "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_without_devices_fails():
    import torch
    if torch.cuda.is_available() and torch.cuda.device_count() >= 2:
        return
    r = _run(["--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
