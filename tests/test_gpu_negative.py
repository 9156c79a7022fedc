"""GPU: fault-inject negative controls (the reference's `npconv verify
--fault-inject`, tools/npconv.cpp:157-176, registered WILL_FAIL in
tests/CMakeLists.txt:35-37).  The parity harness must SEE an engine-side
indexing bug: the engines are fed a triplet list with one triplet moved to
the wrong kernel cell (or the wrong input row) while the oracle keeps the
intact list -- every arithmetic path has to diverge beyond its own bound.
A harness that still passed would be blind."""
import numpy as np
import pytest

from test_gpu_operator import T, rel

pytestmark = pytest.mark.gpu

BOUNDS = {"exact": 1e-5, "auto": 1e-5, "bf16": 1e-2}


def _case(orc, n=600, seed=3):
    xyz = orc.gen_uniform_cube(n, 1.0, seed)
    r = 1.8 * n ** (-1 / 3)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
    si, sj, sk = orc.sort_triplets(ti, tj, tk, 3, n, n, 27)
    w = orc.make_weights(3, 1, 64, 64, seed + 1)
    f = orc.gen_features(n, 1, 64, seed + 2)
    g = orc.gen_features(n, 1, 64, seed + 3)
    return n, (si, sj, sk), w, f, g


def _engines(npc, n, trip, w, f, g, math):
    tl = npc.TripletList.from_numpy(*trip, n, n, 27, 3)
    c = npc.ExecConfig(math=getattr(npc.Math, math))
    fo = npc.mvmr(T(w), T(f), tl, n, c).out.cpu()
    gi = npc.mvmr_transposed(T(w), T(g), tl, n, c).out.cpu()
    gw = npc.vvor(T(g), T(f), tl, 27, c).grad.cpu()
    return fo, gi, gw


@pytest.mark.parametrize("math", ["exact", "auto", "bf16"])
@pytest.mark.parametrize("fault", ["cell", "row"])
def test_fault_injected_engine_is_detected(npc, orc, math, fault):
    n, (si, sj, sk), w, f, g = _case(orc)
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), si, sj, sk, n,
                                g.astype(np.float64))
    # intact list: inside the bound (the positive control)
    e_ok = [rel(a, b) for a, b in zip(_engines(npc, n, (si, sj, sk), w, f, g, math), (fo, gi, gw))]
    assert max(e_ok) <= BOUNDS[math], e_ok
    # one triplet moved: the wrong cell (npconv.cpp:171-175) or the wrong input row
    bad_j, bad_k = sj.copy(), sk.copy()
    m = len(sk) // 2
    if fault == "cell":
        bad_k[m] = (bad_k[m] + 1) % 27
    else:
        bad_j[m] = (bad_j[m] + 1) % n
    e_bad = [rel(a, b) for a, b in zip(_engines(npc, n, (si, bad_j, bad_k), w, f, g, math),
                                       (fo, gi, gw))]
    print(f"{math} {fault}: intact {max(e_ok):.2e}, injected {e_bad}")
    # every pass reads the corrupted triplet: each one must fail its bound
    assert min(e_bad) > BOUNDS[math], e_bad
