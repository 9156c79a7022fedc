"""GPU parity of the operator path (PointConvOp, conv_op.hpp) and the BASELINE
configs at parity-test sizes:
  c1: 16K uniform points, C_in = C_out = 32, t = 3, forward        (exact path)
  c2: 100K uniform points, C = 64, forward + both gradients         (exact + bf16)
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def T(x, dt=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(x)).to("cuda", dt)


def test_pointconv_state_and_shapes(npc, orc):
    w = T(orc.make_weights(3, 1, 4, 5, 1))
    op = npc.PointConvOp(w, npc.ConvGeometry(radius=0.3, t=3))
    with pytest.raises(npc.StateError):
        op.backward(T(np.zeros((3, 1, 5))))
    with pytest.raises(npc.StateError):
        op.cached_triplets()
    with pytest.raises(npc.ShapeError):
        npc.PointConvOp(w, npc.ConvGeometry(radius=0.3, t=5))
    xyz = orc.gen_uniform_cube(200, 1.0, 3)
    cl = npc.make_point_cloud(xyz)
    with pytest.raises(npc.ShapeError):
        op.forward(cl, T(np.zeros((199, 1, 4))))
    f = T(orc.gen_features(200, 1, 4, 4))
    op.forward(cl, f)
    with pytest.raises(npc.ShapeError):
        op.backward(T(np.zeros((200, 1, 4))))


def test_pointconv_matches_oracle_and_caches(npc, orc, golden):
    g = golden("conv_small.npz")
    n = len(g["xyz"])
    cl = npc.make_point_cloud(g["xyz"])
    w = T(g["w"], torch.float64)
    op = npc.PointConvOp(w, npc.ConvGeometry(radius=float(g["radius"]), t=3),
                         npc.ExecConfig(math=npc.Math.exact))
    out = op.forward(cl, T(g["fin"], torch.float64))
    assert rel(out.cpu(), g["fout"]) <= 1e-12
    res = op.backward(T(g["gout"], torch.float64))
    assert rel(res.grad_in.cpu(), g["grad_in"]) <= 1e-12
    assert rel(res.grad_w.cpu(), g["grad_w"]) <= 1e-12
    ti, tj, tk = op.cached_triplets().numpy()  # by_k (choose_sort_axis)
    assert np.array_equal(ti, g["i"]) and np.array_equal(tj, g["j"]) and np.array_equal(tk, g["k"])
    nb = op.neighbors()
    op.forward(cl, T(g["fin"], torch.float64))
    assert op.neighbors() is nb  # identity cache hit (conv_op.hpp:109-111)
    cl2 = npc.make_point_cloud(g["xyz"])
    op.forward(cl2, T(g["fin"], torch.float64))
    assert op.neighbors() is not nb


def test_pointwise_t1_identity(npc, orc):
    # test_conv_op.cpp:35-56: t=1, tiny radius -> F_out = W^T f per point
    xyz = orc.gen_uniform_cube(100, 10.0, 5)
    cl = npc.make_point_cloud(xyz)
    w = orc.make_weights(1, 1, 6, 7, 6, np.float64)
    f = orc.gen_features(100, 1, 6, 7, np.float64)
    op = npc.PointConvOp(T(w, torch.float64), npc.ConvGeometry(radius=1e-6, t=1))
    out = op.forward(cl, T(f, torch.float64)).cpu().numpy()
    want = np.einsum("ngc,gcm->ngm", f, w[0])
    assert rel(out, want) <= 1e-14


def test_strided_two_cloud_forward(npc, orc, ref):
    # conv_op.hpp:161-175, 219-225 on a clustered cloud (config-3 stand-in, small)
    xyz = ref.gen_gaussian_clusters(6000, 8, 4.0, 0.3, 17)
    cl = npc.make_point_cloud(xyz)
    w = orc.make_weights(3, 1, 16, 24, 8, np.float64)
    op = npc.PointConvOp(T(w, torch.float64), npc.ConvGeometry(radius=0.25, t=3))
    f = orc.gen_features(6000, 1, 16, 9, np.float64)
    sr = npc.strided_block(op, cl, T(f, torch.float64), 0.2)
    kept, parent, koff = ref.voxel_downsample(xyz, 0.2)
    assert np.array_equal(sr.map.kept_index.cpu().numpy(), kept)
    coarse = xyz[kept]
    ti, tj, tk = ref.build_triplets(coarse, xyz, 0.25, 3, axis=0)
    fo, _, _ = orc.dense_conv(w, f, ti, tj, tk, len(kept))
    assert rel(sr.coarse_features.cpu(), fo) <= 1e-12
    up = npc.upsample(cl, sr.map, sr.coarse_features)
    assert up.shape[0] == 6000


@pytest.mark.parametrize("math", ["auto", "exact"])
def test_c1_forward_parity(npc, orc, math):
    """BASELINE config 1: 16K points, C=32, the default fp32 contract (the
    split tensor-core path) and the exact CUDA-core engine vs the fp64 oracle."""
    n = 16384
    xyz = orc.gen_uniform_cube(n, 1.0, 1)
    r = 1.8 * n ** (-1 / 3)
    w = orc.make_weights(3, 1, 32, 32, 2)
    f = orc.gen_features(n, 1, 32, 3)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
    assert len(ti) == 385924
    fo, _, _ = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=getattr(npc.Math, math)))
    out = op.forward(npc.make_point_cloud(xyz), T(f))
    assert rel(out.cpu(), fo) <= 1e-5


@pytest.mark.slow
def test_c2_fwd_bwd_parity(npc, orc):
    """BASELINE config 2: 100K points, C=64, forward + dgrad + wgrad."""
    n = 100000
    xyz = orc.gen_uniform_cube(n, 1.0, 1)
    r = 1.8 * n ** (-1 / 3)
    w = orc.make_weights(3, 1, 64, 64, 2)
    f = orc.gen_features(n, 1, 64, 3)
    go = orc.gen_features(n, 1, 64, 4)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
    assert len(ti) == 2435886
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    cl = npc.make_point_cloud(xyz)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.exact))
    out = op.forward(cl, T(f))
    res = op.backward(T(go))
    assert rel(out.cpu(), fo) <= 1e-5
    assert rel(res.grad_in.cpu(), gi) <= 1e-5
    assert rel(res.grad_w.cpu(), gw) <= 1e-5


# ---------------------------------------------------------------------------
# bf16 tensor-core path (tcgen05): C = 64, G = 1, t = 3
# ---------------------------------------------------------------------------
def _bf16(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def _emulate_tc(ti, tj, tk, n_out, n_in, w, f, g):
    """The exact arithmetic of the tensor-core engines, in numpy: per (row, cell)
    aggregation of bf16-rounded neighbor rows with fp32 accumulation in CSR order,
    rounded to bf16, then GEMMs against bf16-rounded weights (fp64 here; the
    device accumulates in fp32, so agreement is ~1e-6)."""
    K, ci, co = w.shape[0], w.shape[2], w.shape[3]
    wb = _bf16(w[:, 0]).astype(np.float64)          # (K, Cin, Cout)
    fb, gb = _bf16(f[:, 0]), _bf16(g[:, 0])
    ti, tj, tk = ti.astype(np.int64), tj.astype(np.int64), tk.astype(np.int64)
    # forward aggregation over (i, k), CSR order = (i, j) order of the build
    A = np.zeros((n_out, K, ci), np.float32)
    np.add.at(A, (ti, tk), fb[tj])
    A = _bf16(A.reshape(-1, ci)).reshape(n_out, K, ci).astype(np.float64)
    fout = np.einsum("nkc,kcm->nm", A, wb)
    # dgrad aggregation over (j, k) in (j, i) order
    o = np.lexsort((ti, tj))
    B = np.zeros((n_in, K, co), np.float32)
    np.add.at(B, (tj[o], tk[o]), gb[ti[o]])
    B = _bf16(B.reshape(-1, co)).reshape(n_in, K, co).astype(np.float64)
    gin = np.einsum("nkm,kcm->nc", B, wb)
    if _fused_backward(K, ci, co):
        # the fused backward (one aggregation for both gradients): dW_k =
        # sum_j bf16(B_k[j]) (x) bf16(F_in[j])  (vvor.hpp:79-84)
        gw = np.einsum("nkm,nc->kmc", B, fb.astype(np.float64))
    else:
        gw = np.einsum("nm,nkc->kmc", gb.astype(np.float64), A)
    return fout, gin, gw


def _fused_backward(K, ci, co):
    """Whether the library's bf16 backward runs the fused kernel (both
    gradients, K = 27, C_in, C_out <= 64; NPCG_FUSED_BWD=0 turns it off)."""
    import os
    return (K == 27 and ci <= 64 and co <= 64 and os.environ.get("NPCG_FUSED_BWD", "1") != "0"
            and os.environ.get("NPCG_TC_ENGINE", "halo") != "gather")


def _bf16_case(npc, orc, n, seed=1):
    xyz = orc.gen_uniform_cube(n, 1.0, seed)
    r = 1.8 * n ** (-1 / 3)
    w = orc.make_weights(3, 1, 64, 64, 2)
    f = orc.gen_features(n, 1, 64, 3)
    go = orc.gen_features(n, 1, 64, 4)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
    return xyz, r, w, f, go, (ti, tj, tk)


def test_bf16_path_matches_emulation_and_oracle(npc, orc):
    n = 8192
    xyz, r, w, f, go, (ti, tj, tk) = _bf16_case(npc, orc, n)
    cl = npc.make_point_cloud(xyz)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(cl, T(f))
    res = op.backward(T(go))
    st = op.neighbors().plan_stats()
    assert all(v["overflow"] == 0 for v in st.values()), st
    efo, egi, egw = _emulate_tc(ti, tj, tk, n, n, w, f, go)
    # precision-isolated: identical bf16 operands, only accumulation order differs
    assert rel(out.cpu().numpy()[:, 0], efo) <= 2e-5
    assert rel(res.grad_in.cpu().numpy()[:, 0], egi) <= 2e-5
    assert rel(res.grad_w.cpu().numpy()[:, 0], egw) <= 2e-5
    # end-to-end bound vs the fp64 oracle on the fp32 inputs (<= 1e-2)
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    assert rel(out.cpu(), fo) <= 1e-2
    assert rel(res.grad_in.cpu(), gi) <= 1e-2
    assert rel(res.grad_w.cpu(), gw) <= 1e-2


def test_bf16_path_deterministic(npc, orc):
    n = 20000
    xyz, r, w, f, go, _ = _bf16_case(npc, orc, n, seed=5)
    cl = npc.make_point_cloud(xyz)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    a = op.forward(cl, T(f))
    ra = op.backward(T(go))
    b = op.forward(cl, T(f))
    rb = op.backward(T(go))
    assert torch.equal(a, b)
    assert torch.equal(ra.grad_in, rb.grad_in)
    assert torch.equal(ra.grad_w, rb.grad_w)


def test_bf16_raw_triplets_api(npc, orc):
    """npcg_mvmr / mvmr_transposed / vvor with math=bf16 on a raw TripletList
    (identity order, no coordinates)."""
    n = 3000
    xyz, r, w, f, go, (ti, tj, tk) = _bf16_case(npc, orc, n, seed=9)
    si, sj, sk = orc.sort_triplets(ti, tj, tk, 3, n, n, 27)
    tl = npc.TripletList.from_numpy(si, sj, sk, n, n, 27, 3)
    c = npc.ExecConfig(math=npc.Math.bf16)
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    assert rel(npc.mvmr(T(w), T(f), tl, n, c).out.cpu(), fo) <= 1e-2
    assert rel(npc.mvmr_transposed(T(w), T(go), tl, n, c).out.cpu(), gi) <= 1e-2
    assert rel(npc.vvor(T(go), T(f), tl, 27, c).grad.cpu(), gw) <= 1e-2


@pytest.mark.parametrize("cin,cout", [(64, 64), (128, 256)])
def test_bf16_clustered_cloud(npc, orc, ref, cin, cout):
    """Dense clusters stress the tile capacities; super-tiles beyond them are
    served by the exact engine, results stay within the bf16 bound."""
    xyz = ref.gen_gaussian_clusters(30000, 20, 4.0, 0.15, 21)
    r = 0.08
    w = orc.make_weights(3, 1, cin, cout, 2)
    f = orc.gen_features(30000, 1, cin, 3)
    go = orc.gen_features(30000, 1, cout, 4)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
    cl = npc.make_point_cloud(xyz)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(cl, T(f))
    res = op.backward(T(go))
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, 30000,
                                go.astype(np.float64))
    assert rel(out.cpu(), fo) <= 1e-2
    assert rel(res.grad_in.cpu(), gi) <= 1e-2
    assert rel(res.grad_w.cpu(), gw) <= 1e-2


@pytest.mark.parametrize("cin,cout", [(64, 128), (128, 64), (128, 128), (256, 256), (64, 256),
                                      (256, 128), (32, 32), (48, 80), (96, 160), (16, 256)])
def test_bf16_wide_channels(npc, orc, cin, cout):
    """C_in, C_out in {64, 128, 256} on the tensor-core engines: forward /
    input gradient gather 64-channel chunks accumulated in TMEM with up to 256
    output columns per tile; the weight gradient pairs (cell, C_in chunk) A
    tiles against G tiles of C_out columns.  Other multiples of 16 are
    zero-padded to 64 / 128 / 256 (math = bf16 forces narrow widths onto the
    tensor cores; the automatic choice runs them on the split fp32-contract path)."""
    n = 6000
    xyz = orc.gen_uniform_cube(n, 1.0, 31)
    r = 1.8 * n ** (-1 / 3)
    w = orc.make_weights(3, 1, cin, cout, 32)
    f = orc.gen_features(n, 1, cin, 33)
    go = orc.gen_features(n, 1, cout, 34)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    cl = npc.make_point_cloud(xyz)
    out = op.forward(cl, T(f))
    res = op.backward(T(go))
    assert out.shape == (n, 1, cout) and res.grad_in.shape == (n, 1, cin)
    efo, egi, egw = _emulate_tc(ti, tj, tk, n, n, w, f, go)
    assert rel(out.cpu().numpy()[:, 0], efo) <= 2e-5
    assert rel(res.grad_in.cpu().numpy()[:, 0], egi) <= 2e-5
    assert rel(res.grad_w.cpu().numpy()[:, 0], egw) <= 2e-5
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    assert rel(out.cpu(), fo) <= 1e-2
    assert rel(res.grad_in.cpu(), gi) <= 1e-2
    assert rel(res.grad_w.cpu(), gw) <= 1e-2
    assert torch.equal(op.forward(cl, T(f)), out)  # deterministic
    assert torch.equal(op.backward(T(go)).grad_w, res.grad_w)


def _voxel_for_ratio(npc, cloud, ratio):
    lo, hi = 1e-4, 100.0
    for _ in range(60):
        v = (lo * hi) ** 0.5
        coarse, _ = npc.voxel_downsample(cloud, v)
        m = coarse.n_points()
        if abs(m * ratio / cloud.n_points() - 1) < 0.05:
            break
        lo, hi = (v, hi) if m * ratio > cloud.n_points() else (lo, v)
    return v, coarse


@pytest.mark.parametrize("cout", [64, 128])
def test_bf16_strided_lidar_dense(npc, orc, cout):
    """Config-3 shape: a LiDAR-like scan, voxel-downsampled ~4x, strided
    two-cloud conv with ~50 (near the sensor: hundreds of) fine neighbors per
    coarse point.  The 128-row super-tiles exceed the halo / block capacities;
    the planner re-tiles them as smaller tiles (down to 8 rows), and 8-row
    tiles that still do not fit become rank-split records accumulated in TMEM,
    so every row stays on the tensor cores.  A rank-split (row, cell) sum is
    rounded to bf16 per record instead of once, so the emulation bound here is
    one bf16 ulp (2^-8) rather than 2e-5."""
    from paper_2511_23227_b200.synthetic import gen_lidar_scan
    n = 24000
    xyz = gen_lidar_scan(n, 7)
    fine = npc.make_point_cloud(xyz)
    v, coarse = _voxel_for_ratio(npc, fine, 4.0)
    r = 1.8 * v
    w = orc.make_weights(3, 1, 64, cout, 5)
    f = orc.gen_features(n, 1, 64, 6)
    m = coarse.n_points()
    go = orc.gen_features(m, 1, cout, 7)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(fine, coarse, T(f))
    res = op.backward(T(go))
    ti, tj, tk = op.cached_triplets().numpy()
    if cout == 64:
        st = op.neighbors().plan_stats()
        assert all(v_["overflow"] == 0 for v_ in st.values()), st
    efo, egi, egw = _emulate_tc(ti, tj, tk, m, n, w, f, go)
    assert rel(out.cpu().numpy()[:, 0], efo) <= 2 ** -8
    assert rel(res.grad_in.cpu().numpy()[:, 0], egi) <= 2 ** -8
    assert rel(res.grad_w.cpu().numpy()[:, 0], egw) <= 2 ** -8
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, m,
                                go.astype(np.float64))
    assert max(rel(out.cpu(), fo), rel(res.grad_in.cpu(), gi), rel(res.grad_w.cpu(), gw)) <= 1e-2


def test_bf16_indoor_surface(npc, orc):
    """Config-4 geometry: surface-sampled room, neighbors concentrated in the
    cells a plane crosses (up to ~10 per (row, cell)).  Super-tiles whose halo
    exceeds the cap run as items of halo-segment records (partial (row, cell)
    sums rounded per record), hence the 2^-8 emulation bound."""
    from paper_2511_23227_b200.synthetic import gen_indoor_fragment
    n = 40000
    xyz, area = gen_indoor_fragment(n, 11)
    r = (25.0 / (np.pi * n / area)) ** 0.5
    cl = npc.make_point_cloud(xyz)
    w = orc.make_weights(3, 1, 64, 64, 5)
    f = orc.gen_features(n, 1, 64, 6)
    go = orc.gen_features(n, 1, 64, 7)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(cl, T(f))
    res = op.backward(T(go))
    st = op.neighbors().plan_stats()
    assert all(v_["overflow"] == 0 for v_ in st.values()), st
    ti, tj, tk = op.cached_triplets().numpy()
    efo, egi, egw = _emulate_tc(ti, tj, tk, n, n, w, f, go)
    assert rel(out.cpu().numpy()[:, 0], efo) <= 2 ** -8
    assert rel(res.grad_in.cpu().numpy()[:, 0], egi) <= 2 ** -8
    assert rel(res.grad_w.cpu().numpy()[:, 0], egw) <= 2 ** -8
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    assert max(rel(out.cpu(), fo), rel(res.grad_in.cpu(), gi), rel(res.grad_w.cpu(), gw)) <= 1e-2


def test_bf16_wide_pipeline_repeated(npc, orc):
    """Regression: with descriptor slots shared between aggregation groups, a
    group could wait on a slot two barrier phases ahead (parity waits cannot
    tell) and read a stale descriptor -- an intermittent illegal address on
    128-channel passes.  Slots are now a multiple of the groups; repeated
    128 -> 128 fwd+bwd steps on a surface cloud must run and agree bitwise."""
    from paper_2511_23227_b200.synthetic import gen_indoor_fragment
    n = 150000
    xyz, area = gen_indoor_fragment(n, 11)
    r = 2 * (25.0 / (np.pi * n / area)) ** 0.5
    cl = npc.make_point_cloud(xyz)
    w = orc.make_weights(3, 1, 128, 128, 5)
    f, go = T(orc.gen_features(n, 1, 128, 6)), T(orc.gen_features(n, 1, 128, 7))
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    ref = None
    for _ in range(8):
        out = op.forward(cl, f)
        res = op.backward(go)
        torch.cuda.synchronize()
        cur = (out.clone(), res.grad_in.clone(), res.grad_w.clone())
        if ref is None:
            ref = cur
        assert all(torch.equal(a, b) for a, b in zip(cur, ref))


@pytest.mark.parametrize("case", ["one_point", "five_points", "partial_tile", "isolated",
                                  "empty_batch", "two_cloud_tiny"])
def test_bf16_edge_cases(npc, orc, case):
    """Tensor-core path on degenerate shapes: a single point, fewer rows than a
    tile, partial last tiles, rows with only the self-neighbor, an empty batch
    in a jagged cloud, a strided conv onto a handful of sites."""
    rng_seed = {"one_point": 1, "five_points": 2, "partial_tile": 3, "isolated": 4,
                "empty_batch": 5, "two_cloud_tiny": 6}[case]
    off = None
    if case == "one_point":
        xyz = orc.gen_uniform_cube(1, 1.0, rng_seed); r = 0.3
    elif case == "five_points":
        xyz = orc.gen_uniform_cube(5, 1.0, rng_seed); r = 0.6
    elif case == "partial_tile":
        xyz = orc.gen_uniform_cube(300, 1.0, rng_seed); r = 0.25
    elif case == "isolated":
        xyz = orc.gen_uniform_cube(700, 1.0, rng_seed); r = 1e-4  # self-neighbor only
    elif case == "empty_batch":
        xyz = orc.gen_uniform_cube(900, 1.0, rng_seed); r = 0.2
        off = np.array([0, 400, 400, 900], dtype=np.int64)
    else:
        xyz = orc.gen_uniform_cube(2000, 1.0, rng_seed); r = 0.3
    cl = npc.make_point_cloud(xyz, off)
    out_cl = npc.make_point_cloud(xyz[:7]) if case == "two_cloud_tiny" else cl
    n_in, n_out = len(xyz), out_cl.n_points()
    w = orc.make_weights(3, 1, 64, 64, 9)
    f = orc.gen_features(n_in, 1, 64, 10)
    go = orc.gen_features(n_out, 1, 64, 11)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(cl, out_cl, T(f)) if out_cl is not cl else op.forward(cl, T(f))
    res = op.backward(T(go))
    ti, tj, tk = op.cached_triplets().numpy()
    efo, egi, egw = _emulate_tc(ti, tj, tk, n_out, n_in, w, f, go)
    assert out.shape == (n_out, 1, 64) and res.grad_in.shape == (n_in, 1, 64)
    assert rel(out.cpu().numpy()[:, 0], efo) <= 2e-5
    assert rel(res.grad_in.cpu().numpy()[:, 0], egi) <= 2e-5
    assert rel(res.grad_w.cpu().numpy()[:, 0], egw) <= 2e-5


@pytest.mark.parametrize("t,cin,cout", [(5, 64, 64), (5, 128, 64), (1, 64, 128)])
def test_bf16_kernel_resolutions(npc, orc, t, cin, cout):
    """t = 5 (125 kernel cells) and t = 1 on the tensor cores (the reference's
    geometry supports any odd t; K <= 128 runs on tcgen05).  The radius here
    (~70 neighbors) overflows the 256-row halo cap and, at t = 1, puts all of
    them in one cell, so rows run as split records (partial sums rounded per
    record): emulation bound 2^-8."""
    n = 6000
    xyz = orc.gen_uniform_cube(n, 1.0, 41)
    r = (1.8 if t == 3 else 2.6) * n ** (-1 / 3)
    w = orc.make_weights(t, 1, cin, cout, 42)
    f = orc.gen_features(n, 1, cin, 43)
    go = orc.gen_features(n, 1, cout, 44)
    ti, tj, tk = orc.build_triplets(xyz, xyz, r, t)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=t), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(npc.make_point_cloud(xyz), T(f))
    res = op.backward(T(go))
    efo, egi, egw = _emulate_tc(ti, tj, tk, n, n, w, f, go)
    bound = 2 ** -8
    assert rel(out.cpu().numpy()[:, 0], efo) <= bound
    assert rel(res.grad_in.cpu().numpy()[:, 0], egi) <= bound
    assert rel(res.grad_w.cpu().numpy()[:, 0], egw) <= bound
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    assert max(rel(out.cpu(), fo), rel(res.grad_in.cpu(), gi), rel(res.grad_w.cpu(), gw)) <= 1e-2


@pytest.mark.slow
def test_c2_bf16_fwd_bwd(npc, orc):
    """BASELINE config 2 (100K, C=64) on the tensor-core path, bound 1e-2."""
    n = 100000
    xyz, r, w, f, go, (ti, tj, tk) = _bf16_case(npc, orc, n)
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                go.astype(np.float64))
    cl = npc.make_point_cloud(xyz)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=npc.Math.bf16))
    out = op.forward(cl, T(f))
    res = op.backward(T(go))
    st = op.neighbors().plan_stats()
    assert all(v["overflow"] == 0 for v in st.values()), st
    e = (rel(out.cpu(), fo), rel(res.grad_in.cpu(), gi), rel(res.grad_w.cpu(), gw))
    assert max(e) <= 1e-2, e


@pytest.mark.parametrize("pinned_mb", [None, "0"])
def test_cpp_dropin_header(npc, pinned_mb):
    """The C++ drop-in (include/npcg/npconv.hpp) passes reference-style cases,
    with its pinned tensor storage and with all tensors pageable
    (NPCG_HOST_PINNED_MAX_MB=0: the staged copy path)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_dropin")
    assert os.path.exists(exe), "run __graft_entry__.build() first"
    env = dict(os.environ)
    if pinned_mb is not None:
        env["NPCG_HOST_PINNED_MAX_MB"] = pinned_mb
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_gather_engine_parity():
    """The alternative forward / dgrad engine (A tiles gathered from L2 by
    cp.async, NPCG_TC_ENGINE=gather; the engine is chosen once per process)
    passes the bf16 emulation / oracle bounds and determinism checks.  It
    covers C = 64 at uniform density (tiles beyond its capacities go to the
    exact engine), so the wide / dense cases are not rerun under it."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, NPCG_TC_ENGINE="gather")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(here, "test_gpu_operator.py"),
                        "-k", "bf16 and not gather and not dense and not indoor and not wide"],
                       env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("math", ["bf16", "auto"])
def test_output_tiles_without_neighbors(npc, orc, math):
    """A two-cloud layer whose output cloud has whole tiles of points with no
    input neighbour (empty halos): those rows are exactly zero, the others
    match the oracle, and the backward's empty rows / gradients too."""
    rng = np.random.default_rng(3)
    xin = orc.gen_uniform_cube(3000, 1.0, 5)
    near = xin[rng.choice(3000, 200, replace=False)] + rng.normal(0, 0.01, (200, 3))
    far = rng.random((400, 3)) + 10.0  # > 128 consecutive rows with no neighbours
    xout = np.concatenate([near, far])
    r = 1.8 * 3000 ** (-1 / 3)
    w = orc.make_weights(3, 1, 64, 64, 7)
    f = orc.gen_features(3000, 1, 64, 8)
    go = orc.gen_features(len(xout), 1, 64, 9)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3), npc.ExecConfig(math=getattr(npc.Math, math)))
    out = op.forward(npc.make_point_cloud(xin), npc.make_point_cloud(xout), T(f))
    res = op.backward(T(go))
    ti, tj, tk = orc.build_triplets(xout, xin, r, 3)
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, len(xout),
                                go.astype(np.float64))
    tol = 1e-2 if math == "bf16" else 1e-5
    assert torch.count_nonzero(out[200:]) == 0
    assert rel(out.cpu(), fo) <= tol
    assert rel(res.grad_in.cpu(), gi) <= tol and rel(res.grad_w.cpu(), gw) <= tol


def test_cpp_dropin_large_tensors_pinned_equals_pageable(npc):
    """tools/cpp/bench_dropin at 200K points (51 MB tensors): results through
    the pinned tensor storage (one DMA per tensor) are bitwise those through
    pageable storage (staged copies) -- same checksum of out, grad_in, grad_w."""
    import json
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "cpp", "bench_dropin")
    assert os.path.exists(exe), "run __graft_entry__.build() first"
    sums = []
    for mb in (None, "0"):
        env = dict(os.environ)
        if mb is not None:
            env["NPCG_HOST_PINNED_MAX_MB"] = mb
        r = subprocess.run([exe, "200000", "2", "1", "auto"], capture_output=True, text=True, timeout=300, env=env)
        assert r.returncode == 0, r.stdout + r.stderr
        sums.append(json.loads(r.stdout.strip().splitlines()[-1])["checksum"])
    assert sums[0] == sums[1], sums
