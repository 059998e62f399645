"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/sb200.h declares, and fails loudly (no CPU fallback) without a device."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

from paper_2103_08825_b200 import _abi
from paper_2103_08825_b200.build import build


@pytest.fixture(scope="module")
def lib():
    build()
    return _abi.load()


def header_symbols():
    text = open(os.path.join(REPO, "include", "sb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(sb_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert sorted(_abi.EXPORTS) == header_symbols()


def test_library_exports_every_header_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_abi_version(lib):
    assert lib.sb_abi_version() == 1


def test_device_count_never_fails(lib):
    assert lib.sb_device_count() >= 0


def _problem(d=1, r=1, nw=3, offs=(-1, 0, 1), ws=(0.25, 0.5, 0.25), dims=(64, 1, 1)):
    p = _abi.SbProblem()
    p.d, p.r, p.shape, p.nw = d, r, _abi.SB_STAR, nw
    p._o = (ctypes.c_int32 * len(offs))(*offs)
    p._w = (ctypes.c_double * len(ws))(*ws)
    p.offsets = ctypes.cast(p._o, ctypes.POINTER(ctypes.c_int32))
    p.weights = ctypes.cast(p._w, ctypes.POINTER(ctypes.c_double))
    for a in range(3):
        p.dims[a] = dims[a]
    return p


def test_spec_errors_precede_device_checks(lib):
    h = ctypes.c_void_p()
    bad = _problem(nw=2, offs=(-1, 0), ws=(0.5, 0.5))
    assert lib.sb_plan_create(ctypes.byref(h), ctypes.byref(bad)) == _abi.SB_ERR_SPEC
    assert b"needs 3 weights" in lib.sb_last_error()
    unordered = _problem(offs=(0, -1, 1))
    assert lib.sb_plan_create(ctypes.byref(h), ctypes.byref(unordered)) == _abi.SB_ERR_SPEC
    assert b"canonical" in lib.sb_last_error()
    neg = _problem(dims=(0, 1, 1))
    assert lib.sb_plan_create(ctypes.byref(h), ctypes.byref(neg)) == _abi.SB_ERR_GRID


def test_no_cpu_fallback_without_gpu(lib):
    if lib.sb_device_count() > 0:
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = lib.sb_plan_create(ctypes.byref(h), ctypes.byref(_problem()))
    assert rc == _abi.SB_ERR_CUDA
    assert b"no CUDA device" in lib.sb_last_error()
    from paper_2103_08825_b200.core import make_stencil_spec
    from paper_2103_08825_b200.plan import sweep
    with pytest.raises(_abi.CudaError):
        sweep(make_stencil_spec("1d3p"), np.zeros(10), 1)


def test_null_arguments(lib):
    assert lib.sb_plan_create(None, None) == _abi.SB_ERR_ARG
    assert lib.sb_run(None, 1, None) == _abi.SB_ERR_ARG
    assert lib.sb_upload(None, None, 0) == _abi.SB_ERR_ARG


def _build_c_client(tmp_path):
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    exe = str(tmp_path / "sweep_c1")
    libdir = os.path.join(REPO, "paper_2103_08825_b200", "lib")
    r = subprocess.run([gcc, "-O2", "-ffp-contract=off", "-Wall", "-I", os.path.join(REPO, "include"),
                        os.path.join(REPO, "examples", "sweep_c1.c"), "-L", libdir, "-lsb200",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_builds_and_fails_loudly_without_device(lib, tmp_path):
    # the C ABI is usable from plain C; without a GPU every compute call fails with SB_ERR_CUDA
    import subprocess
    if lib.sb_device_count() > 0:
        pytest.skip("a device is present")
    exe = _build_c_client(tmp_path)
    r = subprocess.run([exe, "100", "3"], capture_output=True, text=True)
    assert r.returncode == 2 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_c_client_bit_identical_on_device(lib, tmp_path):
    import subprocess
    exe = _build_c_client(tmp_path)
    r = subprocess.run([exe, "300007", "37"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("bit-identical"), r.stdout + r.stderr


def _config_problem(key, dims, arith, k=0):
    from paper_2103_08825_b200.core import config_spec
    from paper_2103_08825_b200.plan import _problem as mk
    prob, keep = mk(config_spec(key), dims, "f64", arith, k, "auto", 0)
    prob._keep = keep
    return prob


@pytest.mark.parametrize("key,dims,arith,want", [
    ("c1", (1 << 20,), "fma", 64), ("c2", (1 << 26,), "fma", 32), ("c2", (1 << 20,), "exact", 16),
    ("c3a", (512, 512), "fma", 32), ("c3b", (512, 512), "fma", 4), ("c4", (64, 64, 64), "fma", 2),
    ("c5", (64, 64, 64), "exact", 2),
])
def test_problem_k_resolves_without_a_device(lib, key, dims, arith, want):
    k = ctypes.c_int32()
    prob = _config_problem(key, dims, arith)
    assert lib.sb_problem_k(ctypes.byref(prob), ctypes.byref(k)) == _abi.SB_OK
    assert k.value == want


def test_multi_create_fails_loudly_without_devices(lib):
    if lib.sb_device_count() > 0:
        pytest.skip("a device is visible")
    h = ctypes.c_void_p()
    prob = _config_problem("c5", (64, 64, 64), "fma")
    rc = lib.sb_multi_create(ctypes.byref(h), ctypes.byref(prob), 2, None)
    assert rc in (_abi.SB_ERR_ARG, _abi.SB_ERR_CUDA) and not h.value
