"""GPU parity: MVMR forward / input gradient and VVOR weight gradient.

Tolerances (metric: rel_error = max|a-b| / max|b|, gradcheck.cpp:11-31):
  fp64 exact path vs fp64 dense oracle          <= 1e-12  (acceptance.cpp:37)
  fp32 exact path vs fp64 oracle on the same
       fp32-rounded inputs                       <= 1e-5   (acceptance.cpp:39)
  bf16 tensor-core path vs fp64 oracle on the
       bf16-rounded operands                     <= 2e-5   (accumulation only)
  bf16 tensor-core path vs fp64 oracle on the
       fp32 inputs                               <= 1e-2
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_F64 = 1e-12
TOL_F32 = 1e-5


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def T(x, dt):
    return torch.as_tensor(np.ascontiguousarray(x)).to("cuda", dt)


def cfg(npc, math="exact", **kw):
    return npc.ExecConfig(math=getattr(npc.Math, math), **kw)


def test_hand_cases(npc):
    # test_engine.cpp:75-115
    w = np.zeros((1, 1, 2, 2))
    w[0, 0, 0, 0] = w[0, 0, 1, 1] = 1.0
    tl = npc.TripletList.from_numpy([0], [0], [0], 1, 1, 1)
    out = npc.mvmr(T(w, torch.float64), T([[[3.0, 4.0]]], torch.float64), tl, 1, cfg(npc)).out
    assert out.cpu().numpy().ravel().tolist() == [3.0, 4.0]
    tl2 = npc.TripletList.from_numpy([0, 0], [0, 1], [0, 0], 1, 2, 1)
    f = T([[[1.0, 2.0]], [[3.0, 4.0]]], torch.float64)
    assert npc.mvmr(T(w, torch.float64), f, tl2, 1, cfg(npc)).out.cpu().numpy().ravel().tolist() == [4.0, 6.0]
    wt = T(np.array([1.0, 3.0, 2.0, 4.0]).reshape(1, 1, 2, 2), torch.float64)
    g = npc.mvmr_transposed(wt, T([[[1.0, 1.0]]], torch.float64), tl, 1, cfg(npc)).out
    assert g.cpu().numpy().ravel().tolist() == [4.0, 6.0]
    # test_vvor.cpp:65-89: outer product [[3,4],[6,8]]
    gv = npc.vvor(T([[[1.0, 2.0]]], torch.float64), T([[[3.0, 4.0]]], torch.float64), tl, 1,
                  cfg(npc)).grad
    assert gv.cpu().numpy().ravel().tolist() == [3.0, 4.0, 6.0, 8.0]


def test_empty_list_zeros(npc, orc):
    w = T(orc.make_weights(3, 1, 4, 4, 5, np.float64), torch.float64)
    f = T(orc.gen_features(10, 1, 4, 6, np.float64), torch.float64)
    tl = npc.TripletList.from_numpy([], [], [], 0, 0, 27)
    out = npc.mvmr(w, f, tl, 10, cfg(npc)).out
    assert out.shape == (10, 1, 4) and float(out.abs().max()) == 0.0
    g = npc.vvor(f, f, tl, 27, cfg(npc)).grad
    assert float(g.abs().max()) == 0.0


@pytest.mark.parametrize("groups", [1, 2])
@pytest.mark.parametrize("axis", [0, 1, 2, 3])
def test_engine_matches_oracle_f64(npc, orc, groups, axis):
    # test_engine.cpp:128-148 shapes
    n, cig, cog = 64, 8, 16
    w = orc.make_weights(3, groups, cig, cog, 11, np.float64)
    f = orc.gen_features(n, groups, cig, 12, np.float64)
    rng = np.random.default_rng(13)
    i = rng.integers(0, n, 2000)
    j = rng.integers(0, n, 2000)
    k = rng.integers(0, 27, 2000)
    order = np.lexsort((j, i))
    i, j, k = i[order], j[order], k[order]
    fout, _, _ = orc.dense_conv(w, f, i, j, k, n)
    si, sj, sk = orc.sort_triplets(i, j, k, axis, n, n, 27)
    tl = npc.TripletList.from_numpy(si, sj, sk, n, n, 27, axis)
    out = npc.mvmr(T(w, torch.float64), T(f, torch.float64), tl, n, cfg(npc)).out
    assert rel(out.cpu(), fout) <= TOL_F64


def _instance(orc, seed, n=None):
    rng = np.random.default_rng(1000 + seed)
    t = int(rng.choice([1, 3, 5]))
    wide = seed % 7 == 3
    G = 1 if wide else int(rng.choice([1, 2, 4]))
    cig = int(rng.integers(33, 65)) if wide else int(rng.integers(1, 17))
    cog = int(rng.integers(33, 65)) if wide else int(rng.integers(1, 17))
    n = n or int(rng.integers(20, 200))
    nt = int(rng.integers(100, 4000))
    K = t ** 3
    i = rng.integers(0, n, nt)
    j = rng.integers(0, n, nt)
    k = rng.integers(0, K, nt)
    o = np.lexsort((j, i))
    return t, G, cig, cog, n, i[o], j[o], k[o]


@pytest.mark.parametrize("seed", list(range(20)))
def test_acceptance_style_instances(npc, orc, seed):
    """acceptance.cpp:104-206: random t, G, C; fwd + both gradients, fp64 and fp32
    (fp32 inputs cast to fp64 for the oracle so both routes see identical values)."""
    t, G, cig, cog, n, i, j, k = _instance(orc, seed)
    K = t ** 3
    w = orc.make_weights(t, G, cig, cog, 2 + seed, np.float64)
    f = orc.gen_features(n, G, cig, 3 + seed, np.float64)
    go = orc.gen_features(n, G, cog, 4 + seed, np.float64)
    axis = seed % 4
    si, sj, sk = orc.sort_triplets(i, j, k, axis, n, n, K)
    tl = npc.TripletList.from_numpy(si, sj, sk, n, n, K, axis)
    for dt, tol in ((np.float64, TOL_F64), (np.float32, TOL_F32)):
        wq, fq, gq = w.astype(dt), f.astype(dt), go.astype(dt)
        fo, gi, gw = orc.dense_conv(wq.astype(np.float64), fq.astype(np.float64), i, j, k, n,
                                    gq.astype(np.float64))
        td = torch.float64 if dt == np.float64 else torch.float32
        c = cfg(npc)
        out = npc.mvmr(T(wq, td), T(fq, td), tl, n, c).out
        gin = npc.mvmr_transposed(T(wq, td), T(gq, td), tl, n, c).out
        gww = npc.vvor(T(gq, td), T(fq, td), tl, K, c).grad
        assert rel(out.cpu(), fo) <= tol, ("fwd", dt)
        assert rel(gin.cpu(), gi) <= tol, ("dgrad", dt)
        assert rel(gww.cpu(), gw) <= tol, ("wgrad", dt)


def test_validation_errors(npc, orc):
    w = T(orc.make_weights(3, 1, 4, 4, 96, np.float64), torch.float64)
    f = T(orc.gen_features(8, 1, 4, 97, np.float64), torch.float64)
    tl = npc.TripletList.from_numpy([0], [0], [0], 1, 1, 27)
    for bad in (dict(L=0), dict(workers=-1), dict(b_out=0)):
        with pytest.raises(npc.ShapeError):
            npc.mvmr(w, f, tl, 8, npc.ExecConfig(**bad))
    with pytest.raises(npc.IndexError):
        npc.mvmr(w, f, npc.TripletList.from_numpy([0], [0], [30], 1, 1, 27), 8)
    with pytest.raises(npc.IndexError):
        npc.mvmr(w, f, npc.TripletList.from_numpy([0], [9], [0], 1, 8, 27), 8)
    with pytest.raises(npc.IndexError):
        npc.mvmr(w, f, npc.TripletList.from_numpy([8], [0], [0], 8, 1, 27), 8)
    with pytest.raises(npc.ShapeError):
        npc.mvmr(w, f, npc.TripletList.from_numpy([0], [0], [0], 1, 1, 1), 8)
    with pytest.raises(npc.ShapeError):
        npc.mvmr(w, T(orc.gen_features(8, 1, 5, 98, np.float64), torch.float64), tl, 8)
    with pytest.raises(npc.ShapeError):
        npc.mvmr(w, T(orc.gen_features(8, 2, 4, 99, np.float64), torch.float64), tl, 8)
    with pytest.raises(npc.ShapeError):
        npc.mvmr(w, f, npc.TripletList.from_numpy([0], [0], [0], 9, 1, 27), 8)
    go = T(orc.gen_features(8, 1, 4, 100, np.float64), torch.float64)
    with pytest.raises(npc.IndexError):
        npc.vvor(go, f, npc.TripletList.from_numpy([0], [0], [27], 1, 1, 27), 27)
    with pytest.raises(npc.ShapeError):
        npc.vvor(go, f, tl, 0)
    with pytest.raises(npc.ShapeError):
        npc.vvor(go, f, tl, 27, npc.ExecConfig(L=0))


def test_large_channels_and_odd_widths(npc, orc):
    # test_engine.cpp:401-440
    n = 32
    rng = np.random.default_rng(103)
    i, j = np.sort(rng.integers(0, n, 500)), rng.integers(0, n, 500)
    k = np.zeros(500, dtype=np.int64)
    for (G, ci, co) in ((1, 64, 64), (3, 13, 9), (1, 200, 300)):
        w = orc.make_weights(1, G, ci, co, 101, np.float64)
        f = orc.gen_features(n, G, ci, 102, np.float64)
        go = orc.gen_features(n, G, co, 104, np.float64)
        fo, gi, gw = orc.dense_conv(w, f, i, j, k, n, go)
        tl = npc.TripletList.from_numpy(i, j, k, n, n, 1)
        assert rel(npc.mvmr(T(w, torch.float64), T(f, torch.float64), tl, n, cfg(npc)).out.cpu(), fo) <= TOL_F64
        assert rel(npc.mvmr_transposed(T(w, torch.float64), T(go, torch.float64), tl, n,
                                       cfg(npc)).out.cpu(), gi) <= TOL_F64
        assert rel(npc.vvor(T(go, torch.float64), T(f, torch.float64), tl, 1, cfg(npc)).grad.cpu(),
                   gw) <= TOL_F64


def test_deterministic_bitwise(npc, orc):
    n = 100
    t, G, cig, cog = 3, 2, 8, 8
    w = T(orc.make_weights(t, G, cig, cog, 41, np.float64), torch.float64)
    f = T(orc.gen_features(n, G, cig, 42, np.float64), torch.float64)
    rng = np.random.default_rng(43)
    i, j, k = rng.integers(0, n, 3000), rng.integers(0, n, 3000), rng.integers(0, 27, 3000)
    tl = npc.TripletList.from_numpy(i, j, k, n, n, 27)
    a = npc.mvmr(w, f, tl, n, npc.ExecConfig(deterministic=True, workers=1)).out
    for workers in (2, 4, 8):
        b = npc.mvmr(w, f, tl, n, npc.ExecConfig(deterministic=True, workers=workers)).out
        assert torch.equal(a, b)
    ga = npc.vvor(f, f, tl, 27).grad
    gb = npc.vvor(f, f, tl, 27).grad
    assert torch.equal(ga, gb)


def test_vvor_linearity(npc, orc):
    # test_vvor.cpp:91-106: 2*gout gives exactly 2*dW
    n = 50
    rng = np.random.default_rng(5)
    i, j, k = np.sort(rng.integers(0, n, 800)), rng.integers(0, n, 800), rng.integers(0, 27, 800)
    tl = npc.TripletList.from_numpy(i, j, k, n, n, 27)
    go = T(orc.gen_features(n, 1, 6, 7, np.float64), torch.float64)
    f = T(orc.gen_features(n, 1, 5, 8, np.float64), torch.float64)
    a = npc.vvor(go, f, tl, 27).grad
    b = npc.vvor(2 * go, f, tl, 27).grad
    assert torch.equal(b, 2 * a)


def test_library_dw_allreduce_single_rank(npc):
    """npcg_allreduce_dw through the library's own NCCL
    communicator: with one rank the sum is the identity, fp32 and fp64; bad
    dtype / arguments are rejected like the reference's errors."""
    from paper_2511_23227_b200.shard import DwComm
    comm = DwComm(0, 1, 0)
    for dt in (torch.float32, torch.float64):
        g = torch.randn(27, 1, 64, 64, device="cuda", dtype=dt)
        ref = g.clone()
        comm.allreduce(g)
        torch.cuda.synchronize()
        assert torch.equal(g, ref)
    with pytest.raises(npc.ShapeError):
        comm.allreduce(torch.zeros(4, device="cuda", dtype=torch.float16))
    comm.close()
