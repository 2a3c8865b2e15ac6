"""bench.py's launch contract on a host without enough GPUs (CPU test):
`--gpus N` without a torchrun environment re-launches itself as N ranks, and
must refuse loudly (non-zero exit, a message) when fewer than N devices are
visible instead of silently measuring one GPU (round-1 review: --gpus was a
no-op); under torchrun, WORLD_SIZE must match --gpus."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""          # no device, whatever the host has
    if env_extra:
        env.update(env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env,
                          capture_output=True, text=True, timeout=300, cwd=ROOT)


def test_gpus_n_refuses_without_devices():
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert r.returncode != 0
    assert "--gpus 2" in r.stderr and "device" in r.stderr


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in r.stderr
