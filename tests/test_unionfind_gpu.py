"""Pass-2 linking rules (track.cu uf_by_prio; include/ftk_cp.h FTK_DEBUG_UF_BY_ID): up to 2^24 records
the union-find links roots by a pseudo-random index priority and gathers each component's minimum face
id at its root; beyond, and under FTK_DEBUG_UF_BY_ID, it links by face id.  Labels are the component
minimum face id either way (Alg. 1 pass 2), so both rules must return byte-identical
records -- 2D scalar (noisy woven: many short trajectories and loops), 3D, vector, a time slab, and the
isovolume's pass 2 -- while the default rule is checked against the oracle in test_parity_gpu.py."""
import numpy as np
import pytest
import torch

import ftk_inputs as fi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ftk():
    import paper_2011_08697_b200 as m
    from paper_2011_08697_b200 import build as b
    b.build()
    m.lib()
    assert torch.cuda.is_available()
    return m


def _sorted(rec, ftk):
    a = ftk.to_numpy(rec)
    return a[np.argsort(a["face_id"], kind="stable")]


def _both(ftk, fn):
    a = fn()
    ftk.set_debug(ftk.DEBUG_UF_BY_ID)
    try:
        b = fn()
    finally:
        ftk.set_debug(0)
    return a, b


CASES = [
    ("2d-woven-noise", lambda: fi.Woven(128, 96, 16, L=15.0, sigma=0.05).generate(), {}),
    ("3d-woven", lambda: fi.Woven(40, 36, 6, nz=34, scale_log2=26).generate(), {}),
    ("2d-vector", lambda: fi.DoubleGyre(96, 48, 10, scale_log2=26).generate(), {"vector": True}),
]


@pytest.mark.parametrize("name,make,kw", CASES)
def test_rules_agree(ftk, name, make, kw):
    f = make().cuda()
    a, b = _both(ftk, lambda: _sorted(ftk.track(f, 26, **kw), ftk))
    assert len(a) > 0 and a.tobytes() == b.tobytes(), name
    assert len(np.unique(a["label"])) > 1


def test_rules_agree_slab(ftk):
    f = fi.Woven(64, 64, 16, L=15.0, sigma=0.02).generate(t0=4, nt=7).cuda()
    a, b = _both(ftk, lambda: _sorted(ftk.track(f, 26, t0=4, nt_global=16, ghost=True), ftk))
    assert a.tobytes() == b.tobytes()


def test_rules_agree_isovolume(ftk):
    f = fi.Woven(96, 80, 12, L=15.0, sigma=0.02).generate().cuda()
    a, b = _both(ftk, lambda: _sorted(ftk.iso_track(f, 26, 0.25), ftk))
    assert len(a) > 0 and a.tobytes() == b.tobytes()
