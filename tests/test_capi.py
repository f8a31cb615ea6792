"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every entry point include/rc.h declares, and its pure-host logic (the
multi-GPU partitioner) is right."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rclib():
    from paper_2312_13513_b200 import build
    build.build()
    from paper_2312_13513_b200 import _rc
    return _rc


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "rc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rc_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(rclib):
    syms = declared_symbols()
    assert len(syms) >= 14
    L = ctypes.CDLL(rclib.SO)
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(rclib.EXPORTS), "binding and header disagree"


def test_version_and_error_strings(rclib):
    assert b"sm_100a" in rclib.lib().rc_version()
    assert isinstance(rclib.lib().rc_last_error(), bytes)


@pytest.mark.parametrize("n,world", [(0, 1), (1000, 1), (1000, 3), (1 << 20, 8), (16777216, 8), (100_000_000, 8),
                                     (129, 2), (12345, 7)])
def test_partition_covers_and_aligns(rclib, n, world):
    parts = [rclib.rc_partition(n, r, world) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == n
    for (b0, e0), (b1, e1) in zip(parts, parts[1:]):
        assert e0 == b1
    for b, e in parts:
        assert b <= e and b % 128 == 0
    if n >= 128 * world * 4:   # balanced to within two MLP tiles
        sizes = [e - b for b, e in parts]
        assert max(sizes) - min(sizes) < 256


def test_partition_rejects_bad_args(rclib):
    with pytest.raises(rclib.RcError):
        rclib.rc_partition(10, 2, 2)
    with pytest.raises(rclib.RcError):
        rclib.rc_partition(-1, 0, 1)


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch, rclib):
    # the product path must fail loudly if the CUDA library is missing
    monkeypatch.setattr(rclib, "SO", str(tmp_path / "missing.so"))
    monkeypatch.setattr(rclib, "_lib", None)
    with pytest.raises(ImportError):
        rclib.lib()


def test_next_row_entry_points_reject_bad_arguments_before_any_cuda_call(rclib):
    """NEXT-row calls validate on the host and return a status without touching the device (so these
    run on a CPU box): NULL handles, missing arrays, a mesh the CSR conversion cannot hold."""
    import ctypes as C
    L = rclib.lib()
    cells = rclib.rc_cells()
    mesh = rclib.rc_mesh(2, 3, 4, 1e-3, 1e-3, 1e-3)
    # rc_kinetics / rc_laplacian / rc_pack_planes with a NULL mechanism
    assert L.rc_kinetics(None, None, C.byref(cells), None) == rclib.RC_EINVAL
    assert L.rc_laplacian(None, C.byref(mesh), C.byref(cells), None, None, None, None, 0, None) == rclib.RC_EINVAL
    assert L.rc_pack_planes(None, C.byref(mesh), C.byref(cells), None, None, None) == rclib.RC_EINVAL
    # CSR needs nx, ny, nz >= 3 (7 distinct columns per row)
    assert L.rc_ldu_to_csr(C.byref(mesh), 1, None, None, None, None, None, None) == rclib.RC_EUNSUPPORTED
    big = rclib.rc_mesh(4, 4, 4, 1e-3, 1e-3, -1.0)
    assert L.rc_ldu_to_csr(C.byref(big), 1, None, None, None, None, None, None) == rclib.RC_EINVAL
    # rc_kin_create with a NULL description
    h = C.c_void_p()
    assert L.rc_kin_create(None, None, C.byref(h)) == rclib.RC_EINVAL


def test_profiling_entry_points_reject_null_output_before_any_cuda_call(rclib):
    """rc_overlap_read and rc_profile_timeline check their output arrays first (CPU-safe)."""
    L = rclib.lib()
    assert L.rc_overlap_read(None, 0) == rclib.RC_EINVAL
    assert L.rc_profile_timeline(None, None, None, 4) == rclib.RC_EINVAL
    assert L.rc_profile_timeline(None, None, None, 0) == 0  # nothing recorded, nothing asked for
