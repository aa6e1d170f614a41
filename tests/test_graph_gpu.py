"""CUDA-graph replay of ftk_cp_track (include/ftk_cp.h FTK_DEBUG_NO_GRAPH): a repeated call replays
the graph captured on its first use.  The replayed calls must return exactly the records of the plain
launch path -- same faces, labels, locations, types, flags -- for 2D, 3D, vector and time-slab calls;
a graph is keyed by the call's pointers, so another field through the same buffers is a different
graph, and new contents under the same pointer are read by the replay (graphs hold pointers, not
data); a capacity retry still converges."""
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


def _plain(ftk, field, s, **kw):
    ftk.set_debug(ftk.DEBUG_NO_GRAPH)
    try:
        return _sorted(ftk.track(field, s, **kw), ftk)
    finally:
        ftk.set_debug(0)


CASES = [
    ("2d-woven", lambda: fi.Woven(96, 80, 12, L=15.0, sigma=0.02).generate(), 26, {}),
    ("3d-woven", lambda: fi.Woven(40, 36, 6, nz=34, scale_log2=26).generate(), 26, {}),
    ("2d-vector", lambda: fi.DoubleGyre(96, 48, 10, scale_log2=26).generate(), 26, {"vector": True}),
]


@pytest.mark.parametrize("name,make,s,kw", CASES)
def test_replay_matches_plain(ftk, name, make, s, kw):
    f = make().cuda()
    want = _plain(ftk, f, s, **kw)
    assert len(want) > 0
    rec, buf = ftk.track(f, s, return_buffers=True, **kw)  # captures
    got = [_sorted(rec, ftk)]
    for _ in range(3):  # replays
        got.append(_sorted(ftk.track(f, s, buffers=buf, **kw), ftk))
    for g in got:
        assert g.tobytes() == want.tobytes(), name


def test_slab_replay(ftk):
    # a time slab with its ghost plane (labels local to the slab, cross edges exported)
    w = fi.Woven(64, 64, 16, L=15.0)
    f = w.generate(t0=4, nt=7).cuda()
    kw = dict(t0=4, nt_global=16, ghost=True)
    want = _plain(ftk, f, 26, **kw)
    rec, buf = ftk.track(f, 26, return_buffers=True, **kw)
    for _ in range(3):
        rec = ftk.track(f, 26, buffers=buf, **kw)
        assert _sorted(rec, ftk).tobytes() == want.tobytes()


def test_graph_keys_and_contents(ftk):
    a = fi.Woven(64, 64, 10, L=15.0, sigma=0.02, seed=1).generate().cuda()
    b = fi.Woven(64, 64, 10, L=15.0, sigma=0.02, seed=2).generate().cuda()
    wa, wb = _plain(ftk, a, 26), _plain(ftk, b, 26)
    assert wa.tobytes() != wb.tobytes()
    _, buf = ftk.track(a, 26, return_buffers=True)
    for f, want in ((a, wa), (b, wb), (a, wa), (b, wb)):  # two graphs through the same buffers
        assert _sorted(ftk.track(f, 26, buffers=buf), ftk).tobytes() == want.tobytes()
    c = a.clone()
    assert _sorted(ftk.track(c, 26, buffers=buf), ftk).tobytes() == wa.tobytes()  # captured for c
    c.copy_(b)  # same pointer, new contents: the replay reads them
    assert _sorted(ftk.track(c, 26, buffers=buf), ftk).tobytes() == wb.tobytes()


def test_capacity_retry_with_graphs(ftk):
    f = fi.Woven(96, 80, 12, L=15.0, sigma=0.02).generate().cuda()
    want = _plain(ftk, f, 26)
    for _ in range(2):
        rec = ftk.track(f, 26, capacity=64)
        assert _sorted(rec, ftk).tobytes() == want.tobytes()
