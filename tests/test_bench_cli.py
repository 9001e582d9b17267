"""bench.py's launch contract on CPU (no GPU needed): --gpus N without WORLD_SIZE re-launches
itself under torch.distributed.run (N ranks, rank 0 prints one JSON line with n_gpus = N),
and a run whose WORLD_SIZE differs from --gpus refuses to print a line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(kw)
    return env


def test_gpus_n_relaunches_under_torchrun():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference", "--ref-n", "16",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, env=_env(), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "relaunching under torchrun" in r.stderr


def test_world_size_mismatch_refuses_to_print():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference", "--ref-n", "16",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, env=_env(WORLD_SIZE="1", RANK="0"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
