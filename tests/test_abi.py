"""CPU-side checks of the C ABI (no GPU): libsem.so loads, exports every entry
point include/sem.h declares, host-only calls work, and setup rejects
malformed meshes before touching the GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen, sem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", fn)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for mm in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b((?:sem|fd|fd2d)_\w+)\s*\(", src, flags=re.M):
            names.add(mm.group(1))
    return names


@pytest.fixture(scope="module")
def L():
    from paper_1403_0968_b200 import _build
    _build.build()
    return sem.lib()


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert {"sem_setup", "sem_ax", "sem_dssum", "sem_cg", "sem_mask", "sem_free"} <= names
    for nm in sorted(names):
        assert hasattr(L, nm), f"libsem.so does not export {nm}"
    assert {"fd_weights", "fd2d_step", "fd2d_run"} <= names
    assert set(sem.EXPORTS) >= names
    assert b"sm_100a" in L.sem_version()


def test_cuda_objects_target_sm100a(L):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sem.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_library_gll_matches_closed_forms_and_oracle(L, oracle):
    for N in range(1, 16):
        xi, w = sem.gll(N)
        xo, wo = oracle.gll(N)
        np.testing.assert_allclose(xi, xo, rtol=0, atol=2e-15)
        np.testing.assert_allclose(w, wo, rtol=0, atol=2e-15)
        assert abs(w.sum() - 2.0) < 1e-14
    xi, w = sem.gll(4)
    np.testing.assert_allclose(xi, [-1, -np.sqrt(3 / 7), 0, np.sqrt(3 / 7), 1], atol=1e-16)
    np.testing.assert_allclose(w, [0.1, 49 / 90, 32 / 45, 49 / 90, 0.1], atol=3e-16)


def test_gll_rejects_bad_order(L):
    with pytest.raises(sem.SemError) as ei:
        sem.gll(0)
    assert ei.value.code == sem.SEM_EINVAL


def _mesh_struct(m, nranks=1):
    s = sem.SemMesh()
    s.nelem = m.nelem
    s.xyz = m.xyz.ctypes.data
    s.glo = m.glo.ctypes.data
    s.dirichlet = m.dirichlet.ctypes.data
    s.rank, s.nranks = 0, nranks
    s.allgather = sem.ALLGATHER_FN()
    return s


def test_workspace_bytes_and_validation(L):
    N = 7
    xi, _ = sem.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(16, 16, 16))
    s = _mesh_struct(m)
    nb = ctypes.c_size_t(0)
    assert L.sem_workspace_bytes(ctypes.byref(s), N, ctypes.byref(nb)) == 0
    Lloc = m.nlocal
    # G (6L) + B (L) + r, p, w, xw (4L) doubles dominate
    assert 88 * Lloc <= nb.value <= 110 * Lloc
    # the screened operator's mass diagonal adds one L-vector
    alpha = np.ones(m.nlocal)
    s.alpha = alpha.ctypes.data
    nb2 = ctypes.c_size_t(0)
    assert L.sem_workspace_bytes(ctypes.byref(s), N, ctypes.byref(nb2)) == 0
    assert 8 * Lloc <= nb2.value - nb.value <= 8 * Lloc + 256
    s.alpha = None
    assert L.sem_workspace_bytes(ctypes.byref(s), 0, ctypes.byref(nb)) == sem.SEM_EINVAL
    assert L.sem_workspace_bytes(ctypes.byref(s), 16, ctypes.byref(nb)) == sem.SEM_EINVAL
    s.nelem = 0
    assert L.sem_workspace_bytes(ctypes.byref(s), N, ctypes.byref(nb)) == sem.SEM_EINVAL


def _setup_rc(L, m, N, kappa=None, alpha=None):
    s = _mesh_struct(m)
    if kappa is not None:
        s.kappa = kappa.ctypes.data
    if alpha is not None:
        s.alpha = alpha.ctypes.data
    ws = ctypes.create_string_buffer(1024)  # never reached: validation fails first
    ctx = ctypes.c_void_p()
    nb = ctypes.c_size_t(0)
    L.sem_workspace_bytes(ctypes.byref(s), N, ctypes.byref(nb))
    rc = L.sem_setup(ctypes.byref(s), N, ctypes.c_void_p(256), nb.value, None, ctypes.byref(ctx))
    return rc, L.sem_last_error(None).decode()


def test_setup_rejects_malformed_meshes(L):
    N = 3
    xi, _ = sem.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(2, 2, 1))
    # inconsistent Dirichlet flag on one copy of a shared node
    bad = meshgen.box_mesh(N, xi, elems=(2, 2, 1))
    g = bad.glo.reshape(-1)
    ids, cnt = np.unique(g, return_counts=True)
    shared = ids[cnt > 1][0]
    first = np.nonzero(g == shared)[0][0]
    bad.dirichlet.reshape(-1)[first] ^= 1
    rc, msg = _setup_rc(L, bad, N)
    assert rc == sem.SEM_EINVAL and "Dirichlet" in msg
    # an element-interior node shared between two elements
    bad2 = meshgen.box_mesh(N, xi, elems=(2, 2, 1))
    n = N + 1
    q_int = 1 + n + n * n
    bad2.glo[1, q_int] = bad2.glo[0, q_int]
    rc, msg = _setup_rc(L, bad2, N)
    assert rc == sem.SEM_EINVAL and "interior" in msg
    # negative id
    bad3 = meshgen.box_mesh(N, xi, elems=(2, 2, 1))
    bad3.glo[0, 0] = -5
    rc, msg = _setup_rc(L, bad3, N)
    assert rc == sem.SEM_EINVAL
    # screened-Coulomb coefficients: kappa > 0, alpha >= 0, finite
    kappa, alpha = meshgen.coefficients(m)
    for kap, alp, what in ((kappa * 0.0, alpha, "kappa"), (kappa, -alpha, "alpha"),
                           (kappa * np.inf, alpha, "kappa"), (kappa, alpha * np.nan, "alpha")):
        rc, msg = _setup_rc(L, m, N, kap, alp)
        assert rc == sem.SEM_EINVAL and what in msg, (what, msg)
    # misaligned workspace
    s = _mesh_struct(m)
    ctx = ctypes.c_void_p()
    assert L.sem_setup(ctypes.byref(s), N, ctypes.c_void_p(8), 1 << 30, None,
                       ctypes.byref(ctx)) == sem.SEM_EINVAL


def test_null_context_calls(L):
    assert L.sem_ax(None, None, None) == sem.SEM_ESTATE
    assert L.sem_dssum(None, None) == sem.SEM_ESTATE
    assert L.sem_cg(None, None, None, 1e-8, 10, None, None) == sem.SEM_ESTATE
    assert L.sem_pcg(None, 1, None, None, 1e-8, 10, None, None) == sem.SEM_ESTATE
    assert L.sem_diag(None, None) == sem.SEM_ESTATE
    assert L.sem_launch_count(None) == -1
    L.sem_free(None)
    for c in range(6):
        assert L.sem_strerror(c)


def test_nccl_id_host_call(L):
    assert L.sem_nccl_id_bytes() == 128


def test_no_cpu_fallback_without_gpu(L):
    """On a box without a GPU the product path must fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    N = 2
    xi, _ = sem.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(1, 1, 1))
    with pytest.raises(Exception):
        sem.Context(m, N, device=0)


def test_fd_host_calls(L, oracle):
    """fd.h host side: the library's own weights (Fornberg) agree with the
    oracle's closed form; bad arguments are rejected before any GPU work."""
    from paper_1403_0968_b200 import fd
    for r in range(1, 8):
        for dx in (1.0, 0.003):
            np.testing.assert_allclose(fd.weights(r, dx), oracle.fd_weights(r, dx), rtol=1e-12,
                                       atol=1e-13 / dx ** 2)
    om = (ctypes.c_double * 3)(1.0, -2.0, 1.0)
    p = ctypes.c_void_p(256)
    assert L.fd2d_step(p, ctypes.c_void_p(512), ctypes.c_void_p(768), 16, 16, 0, om, 0.1,
                       None) == sem.SEM_EINVAL          # r = 0
    assert L.fd2d_step(p, ctypes.c_void_p(512), ctypes.c_void_p(768), 2, 16, 1, om, 0.1,
                       None) == sem.SEM_EINVAL          # w < 2r+1
    assert L.fd2d_step(p, p, ctypes.c_void_p(768), 16, 16, 1, om, 0.1,
                       None) == sem.SEM_EINVAL          # aliasing
    assert L.fd2d_step(ctypes.c_void_p(264), ctypes.c_void_p(512), ctypes.c_void_p(768), 16, 16,
                       1, om, 0.1, None) == sem.SEM_EINVAL   # misaligned
    assert L.fd_weights(0, 1.0, om) == sem.SEM_EINVAL


def test_no_undefined_internal_symbols(L):
    """Every internal (namespace sem) symbol the library references is defined
    in it: a missing one only shows at dlopen time on the GPU box."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--undefined-only", sem.LIB_PATH], capture_output=True,
                         text=True).stdout
    missing = [ln for ln in out.splitlines() if "_ZN3sem" in ln or "_ZN6sem_fd" in ln]
    assert not missing, missing


def _build_c_consumer(tmp_path):
    import shutil
    import subprocess
    from paper_1403_0968_b200 import sem
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    lib_dir = os.path.dirname(sem.LIB_PATH)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "abi_consumer")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror",
           "-I", os.path.join(root, "include"), "-isystem", os.path.join(cuda, "include"),
           os.path.join(root, "tests", "c", "abi_consumer.c"),
           "-o", exe, "-L", lib_dir, "-l:libsem.so", f"-Wl,-rpath,{lib_dir}",
           "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}",
           "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_plain_c_consumer_compiles_links_and_runs(tmp_path):
    """include/sem.h and include/fd.h are valid C99 (pedantic, -Werror), every
    declared entry point resolves against libsem.so, and the host-only calls
    behave as documented -- from C, not through ctypes."""
    import subprocess
    exe = _build_c_consumer(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_consumer ok" in r.stdout


@pytest.mark.gpu
def test_plain_c_consumer_on_gpu(tmp_path):
    """The same C program builds a context and applies A_L to a constant
    (= 0, PAPER.md eq:semOperator annihilates constants) on device 0."""
    import subprocess
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    exe = _build_c_consumer(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
