"""bench.py's multi-GPU launcher on CPU: `--gpus N` outside torchrun re-runs
the script as N ranks (torch.distributed.run on 127.0.0.1); inside torchrun
the world size must equal --gpus.  The self-test mode exercises exactly that
plumbing with gloo (no GPU)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


def test_launcher_spawns_world_two():
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=300, env=_env())
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d == {"launcher": "ok", "world": 2, "rank_sum": 1.0}


def test_world_size_must_match_gpus():
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=120,
                         env=_env(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert out.returncode == 2
    assert "WORLD_SIZE=1" in out.stdout
