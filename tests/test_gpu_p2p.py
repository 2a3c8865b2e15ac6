"""The peer-memory transport (SEM_COMM=p2p, include/sem.h) on one GPU:
P = 2, 4, 8 in-process ranks whose interface exchange and scalar all-gathers
are device stores into the peers' windows with release / acquire flags --
no host rendezvous, so the CG chunks run as CUDA graphs.  Same bars as
tests/test_gpu_multirank.py: partitioned DSSUM bit-identical to the
rank-ordered oracle sums (twice in a row: both window parities), CG /
Jacobi PCG / single-reduction CG with the oracle's iteration count and x
within 1e-10, a repeated solve (graph replay) bit-identical, no transport
timeout (sem_status).  Runs tests/_p2p_cases.py in a fresh process with
CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS=32 (set before
CUDA starts)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_p2p_transport_cases():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, SEM_COMM="p2p", CUDA_MODULE_LOADING="EAGER",
               CUDA_DEVICE_MAX_CONNECTIONS="32", SEM_P2P_TIMEOUT_MS="5000")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_p2p_cases.py")], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rows = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(rows) == 7, r.stdout[-3000:] + r.stderr[-3000:]
    bad = [row for row in rows if not row["ok"]]
    assert not bad, bad
