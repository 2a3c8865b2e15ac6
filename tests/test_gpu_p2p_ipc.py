"""The peer-memory transport ACROSS PROCESSES (the one-process-per-GPU
deployment path): 2 ranks launched by torch.distributed.run (gloo for the
setup all-gather and the NCCL-id broadcast), both on cuda:0, SEM_COMM=p2p --
windows exported with cudaIpcGetMemHandle and opened with
cudaIpcOpenMemHandle, flags released / acquired at system scope.  (Two
processes on one GPU time-slice, so the spinning collectives are slow but
correct.)  Bars as tests/test_gpu_multirank.py: partitioned DSSUM
bit-identical to the rank-ordered oracle sums (both window parities), CG with
the oracle's iteration count, x within 1e-10, no transport timeout."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_p2p_ipc_two_processes(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "verdict.json"
    env = dict(os.environ, SEM_COMM="p2p", SEM_P2P_TIMEOUT_MS="60000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "_p2p_ipc_rank.py"), str(out)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = json.loads(out.read_text())
    assert len(rows) == 2
    for row in rows:
        assert row["dssum1"] and row["dssum2"], row
        assert row["ok"] and row["its"] == row["its_oracle"], row
        assert row["x_relerr"] <= 1e-10, row
