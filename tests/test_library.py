"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/ftk_cp.h declares,
and its host-only entry points (validation, face count, workspace size) behave.  No compute calls
(no GPU here)."""
import ctypes
import os
import re

import numpy as np
import torch
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ftk():
    from paper_2011_08697_b200 import build as b
    b.build()
    import paper_2011_08697_b200 as m
    m.lib()
    return m


def _declared_symbols():
    syms = set()
    for name in os.listdir(os.path.join(ROOT, "include")):
        if name.endswith(".h"):
            src = open(os.path.join(ROOT, "include", name)).read()
            syms |= set(re.findall(r"FTK_API[^;(]*?\b(ftk_\w+)\s*\(", src))
    return syms


def test_exports_every_declared_symbol(ftk):
    syms = _declared_symbols()
    assert len(syms) >= 13
    lib = ctypes.CDLL(ftk.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(ftk.EXPORTS) == syms


def test_abi_version_and_strerror(ftk):
    assert ftk.lib().ftk_abi_version() == 1
    for s in range(8):
        assert ftk.lib().ftk_strerror(s)


@pytest.mark.parametrize("shape", [(3, 4, 3), (4, 3, 5), (9, 17, 13), (3, 3, 4, 3), (2, 5, 4, 3)])
def test_num_faces_matches_oracle(ftk, oracle_lib, shape):
    field = np.zeros(shape, np.float32)
    _, nf = oracle_lib.extract(field, 0)
    desc = ftk.make_desc(shape, np.float32, 0)
    assert ftk.num_faces(desc) == nf


def test_num_faces_configs(ftk):
    # SURVEY.md 8(a)1 / 8(d) face counts
    assert ftk.num_faces(ftk.make_desc((8, 32, 32), np.float32, 26)) == 83514
    assert ftk.num_faces(ftk.make_desc((256, 1024, 1024), np.float32, 26)) == 3205515258
    assert ftk.num_faces(ftk.make_desc((32, 128, 128, 128), np.float32, 8)) == 3831282660
    assert ftk.num_faces(ftk.make_desc((512, 4096, 4096), np.float32, 26)) == 102869569530


def test_num_faces_slabs_partition(ftk):
    """owned faces of time slabs with one ghost plane sum to the single-domain count"""
    nt = 37
    full = ftk.num_faces(ftk.make_desc((nt, 20, 24), np.float32, 0))
    for G in (2, 3, 4, 8):
        bounds = [nt * g // G for g in range(G + 1)]
        tot = 0
        for g in range(G):
            a, b = bounds[g], bounds[g + 1]
            ghost = g < G - 1
            tot += ftk.num_faces(ftk.make_desc((b - a + ghost, 20, 24), np.float32, 0, t0=a, nt_global=nt, ghost=ghost))
        assert tot == full


def test_invalid_descriptors_rejected_on_host(ftk):
    L = ftk.lib()
    bad = [
        ftk.make_desc((4, 2, 8), np.float32, 0),        # ny < 3
        ftk.make_desc((4, 8, 8), np.float32, 65),       # scale out of range
        ftk.make_desc((4, 8, 8), np.float32, 0, t0=3, nt_global=5),  # t0 + nt > nt_global
    ]
    d = ftk.make_desc((4, 8, 8), np.float32, 0)
    d.ndim = 4
    bad.append(d)
    for desc in bad:
        n = ctypes.c_int64(0)
        st = L.ftk_cp_extract(ctypes.byref(desc), None, None, 0, ctypes.byref(n), None, 0, None)
        assert st == ftk.ERR_INVALID_ARG
    # null pointers with a valid descriptor
    n = ctypes.c_int64(0)
    assert L.ftk_cp_track(ctypes.byref(ftk.make_desc((4, 8, 8), np.float32, 0)), None, None, 0,
                          ctypes.byref(n), None, 0, None, None) == ftk.ERR_INVALID_ARG


def test_workspace_grows_with_capacity(ftk):
    d = ftk.make_desc((8, 32, 32), np.float32, 26)
    a, b = ftk.workspace_size(d, 1000), ftk.workspace_size(d, 100000)
    assert 0 < a < b


def test_product_does_not_import_oracle():
    """the product package must never route through the oracle (no CPU fallback)"""
    pkg = os.path.join(ROOT, "paper_2011_08697_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "ftk_oracle" not in src, f


def test_capacity_bounds(ftk):
    """record slots are int32: capacities at or beyond 2^31 - 1 are rejected on the host"""
    L = ftk.lib()
    desc = ftk.make_desc((4, 8, 8), np.float32, 0)
    b = ctypes.c_size_t(0)
    assert L.ftk_workspace_size(ctypes.byref(desc), ftk.MAX_CAPACITY, ctypes.byref(b)) == ftk.OK
    assert L.ftk_workspace_size(ctypes.byref(desc), ftk.MAX_CAPACITY + 1, ctypes.byref(b)) == ftk.ERR_INVALID_ARG
    assert L.ftk_workspace_size(ctypes.byref(desc), -1, ctypes.byref(b)) == ftk.ERR_INVALID_ARG
    assert ftk.default_capacity(torch.empty(0)) == 1 << 16


def test_debug_switches_validated_on_host(ftk):
    """ftk_set_debug (the testing switches that replaced environment variables) rejects unknown bits"""
    L = ftk.lib()
    assert L.ftk_set_debug(ftk.DEBUG_FORCE_GENERIC | ftk.DEBUG_VERIFY_LINK | ftk.DEBUG_STITCH_HOST
                           | ftk.DEBUG_NO_GRAPH | ftk.DEBUG_UF_BY_ID) == ftk.OK
    assert L.ftk_set_debug(32) == ftk.ERR_INVALID_ARG
    assert L.ftk_set_debug(0) == ftk.OK


def test_product_reads_no_environment():
    """the library takes no hidden switches from the environment (behaviour is fixed by
    the descriptor and the explicit calls)"""
    csrc = os.path.join(ROOT, "paper_2011_08697_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert "getenv" not in src, f


def test_comm_reserve_rejects_bad_args(ftk):
    L = ftk.lib()
    assert L.ftk_comm_reserve(None, 1024) == ftk.ERR_INVALID_ARG
