"""GPU parity: degraded (voxel) mode -- build_triplets_degraded
(triplets.cpp:78-133) and the degraded PointConvOp (conv_op.hpp:133-158,
193-202), SURVEY.md §8(f) next #3.

Bars: triplets in the reference's build order, snapped sites, kept / parent
maps and site offsets byte-equal to the reference (golden fixtures from the
unmodified reference, the C oracle on fresh clouds); acceptance criterion 3
(acceptance.cpp:274-340): on voxel-centre clouds native and degraded modes
give identical triplet sets and bit-identical deterministic forwards; the
degraded forward equals the dense oracle on the gathered site rows (rel
<= 1e-13 fp64, test_conv_op.cpp:133-175) and backward scatters gradients to
the representative points only."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _geom(npc, voxel, t):
    return npc.ConvGeometry(t=t, mode=npc.ConvMode.degraded, voxel_size=voxel)


def _build(npc, xyz, voxel, t, off=None):
    cl = npc.make_point_cloud(np.asarray(xyz, dtype=np.float64), off)
    b = npc.build_triplets_degraded(cl, _geom(npc, voxel, t))
    tl = b.triplets
    return ((tl.i.cpu().numpy().astype(np.uint32), tl.j.cpu().numpy().astype(np.uint32),
             tl.k.cpu().numpy().astype(np.uint32)), b.snapped.xyz.cpu().numpy(),
            b.sites.kept_index.cpu().numpy(), b.sites.parent_of.cpu().numpy(),
            b.snapped.batch_offsets(), b)


def test_known_answers(npc, golden):
    """test_triplets.cpp:154-215."""
    h = golden("golden_hand.json")["degraded"]
    v = h["voxel"]
    c0, c1, c2, c3 = h["cases"]
    (ti, tj, tk), sn, kept, parent, so, _ = _build(npc, c0["xyz"], v, c0["t"])
    assert list(ti) == c0["i"] and list(tj) == c0["j"] and list(tk) == c0["k"]
    assert sn.tolist() == c0["snapped"]
    (ti, tj, tk), *_ = _build(npc, c1["xyz"], v, c1["t"])
    assert sorted(tk.tolist()) == c1["k_multiset"]
    assert all(tk[n] > tk[n - 1] for n in range(1, len(ti)) if ti[n] == ti[n - 1])
    (ti, tj, tk), sn, kept, parent, so, b = _build(npc, c2["xyz"], v, c2["t"])
    assert len(sn) == c2["n_sites"] and parent[0] == parent[1] != parent[2]
    assert b.triplets.n_in == 2 and b.triplets.n_out == 2
    (ti, tj, tk), *_, b = _build(npc, c3["xyz"], v, c3["t"])
    assert sorted(tk.tolist()) == c3["k_multiset"] and b.triplets.n_kernels == c3["n_kernels"]
    cl = npc.make_point_cloud(np.zeros((1, 3)))
    with pytest.raises(npc.VoxelError):
        npc.build_triplets_degraded(cl, _geom(npc, 0.0, 3))
    with pytest.raises(npc.ShapeError):
        npc.build_triplets_degraded(cl, _geom(npc, 1.0, 4))
    with pytest.raises(npc.ShapeError):  # t validated before the voxel size (triplets.cpp:79-81)
        npc.build_triplets_degraded(cl, _geom(npc, 0.0, 4))


def test_matches_reference_golden(npc, golden):
    g = golden("degraded_clusters.npz")
    for t in (3, 5):
        (ti, tj, tk), sn, kept, parent, so, _ = _build(npc, g["xyz"], float(g["voxel"]), t,
                                                     g["offsets"])
        for got, key in ((ti, "i"), (tj, "j"), (tk, "k"), (sn, "snapped"), (kept, "kept"),
                         (parent, "parent"), (so, "site_offsets")):
            assert np.array_equal(got, g[f"t{t}_{key}"]), (t, key)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_matches_oracle_random(npc, orc, seed):
    rng = np.random.default_rng(seed)
    n = 6000
    xyz = orc.gen_uniform_cube(n, 1.0, seed)
    if seed % 2 == 0:  # clustered: many points per voxel
        xyz = np.round(xyz * 12) / 12 + rng.normal(0, 0.01, xyz.shape)
    off = [0, 2000, 2000, n] if seed % 2 else None
    for v, t in ((0.05, 3), (0.08, 5), (0.13, 1)):
        a = _build(npc, xyz, v, t, off)
        b = orc.build_triplets_degraded(xyz, v, t, off)
        assert all(np.array_equal(x, y) for x, y in zip(a[0], b[0])), (v, t)
        assert all(np.array_equal(x, y) for x, y in zip(a[1:5], b[1:])), (v, t)


def test_criterion3_native_equals_degraded(npc, ref):
    """acceptance.cpp:274-340 on the GPU: voxel-centre clouds, t = 1 and 3."""
    v = 0.5
    for t in (1, 3):
        xyz = ref.gen_grid_snapped(400, 10, v, 42 + t)
        n = len(xyz)
        cl = npc.make_point_cloud(xyz)
        radius = v * np.sqrt(3.0) / 2.0 if t == 1 else 1.8 * v
        nat = npc.build_triplets_native(cl, cl, npc.ConvGeometry(radius=radius, t=t))
        deg = npc.build_triplets_degraded(cl, _geom(npc, v, t))
        assert deg.snapped.n_points() == n
        assert np.array_equal(deg.sites.kept_index.cpu().numpy(), np.arange(n))
        canon = lambda tl: sorted(zip(tl.i.cpu().tolist(), tl.j.cpu().tolist(),
                                      tl.k.cpu().tolist()))
        assert canon(nat) == canon(deg.triplets)
        w = torch.from_numpy(ref.make_weights(t, 2, 6, 8, 43, np.float64)).cuda()
        f = torch.from_numpy(ref.gen_features(n, 2, 6, 44, np.float64)).cuda()
        cfg = npc.ExecConfig(deterministic=True)
        ns = npc.sort_triplets(nat, npc.SortAxis.by_k)
        ds = npc.sort_triplets(deg.triplets, npc.SortAxis.by_k)
        a = npc.mvmr(w, f, ns, n, cfg).out
        b = npc.mvmr(w, f, ds, n, cfg).out
        assert torch.equal(a, b)


def test_degraded_pointconv_small(npc, orc):
    """test_conv_op.cpp:133-175: two points in one voxel + one isolated point."""
    xyz = np.array([[0.2, 0.2, 0.2], [0.3, 0.3, 0.3], [5, 5, 5]])
    cl = npc.make_point_cloud(xyz)
    w = torch.from_numpy(orc.make_weights(3, 1, 2, 3, 351, np.float64)).cuda()
    f = torch.from_numpy(orc.gen_features(3, 1, 2, 352, np.float64)).cuda()
    op = npc.PointConvOp(w, _geom(npc, 1.0, 3), npc.ExecConfig(deterministic=True))
    out = op.forward(cl, f)
    assert op.snapped_cloud().n_points() == 2 and out.shape[0] == 2
    kept = op.site_map().kept_index.cpu().numpy()
    site_f = f.cpu().numpy()[kept]
    tl = op.cached_triplets()
    ti, tj, tk = (x.cpu().numpy() for x in (tl.i, tl.j, tl.k))
    go = orc.gen_features(2, 1, 3, 353, np.float64)
    fo, gi, gw = orc.dense_conv(w.cpu().numpy(), site_f, ti, tj, tk, 2, go)
    assert orc.rel_error(out.cpu().numpy(), fo) <= 1e-13
    res = op.backward(torch.from_numpy(go).cuda())
    assert res.grad_in.shape[0] == 3
    g = res.grad_in.cpu().numpy()
    for p in range(3):
        mag = np.abs(g[p]).sum()
        assert (mag > 0) if p in kept else (mag == 0)
    assert orc.rel_error(g[kept], gi) <= 1e-13
    assert orc.rel_error(res.grad_w.cpu().numpy(), gw) <= 1e-13


@pytest.mark.parametrize("math,tol", [("exact", 1e-5), ("bf16", 1e-2)])
def test_degraded_pointconv_c64(npc, orc, math, tol):
    """A 30K-point cloud merged to voxel sites, C = 64: exact fp32 and the
    tensor-core path against the fp64 oracle on the gathered site rows."""
    n = 30000
    xyz = orc.gen_uniform_cube(n, 1.0, 11)
    cl = npc.make_point_cloud(xyz)
    w = orc.make_weights(3, 1, 64, 64, 2)
    f = orc.gen_features(n, 1, 64, 3)
    op = npc.PointConvOp(torch.from_numpy(w).cuda(), _geom(npc, 0.035, 3),
                         npc.ExecConfig(math=getattr(npc.Math, math)))
    out = op.forward(cl, torch.from_numpy(f).cuda())
    ns = op.snapped_cloud().n_points()
    kept = op.site_map().kept_index.cpu().numpy()
    tl = op.cached_triplets()
    ti, tj, tk = (x.cpu().numpy() for x in (tl.i, tl.j, tl.k))
    go = orc.gen_features(ns, 1, 64, 4)
    fo, gi, gw = orc.dense_conv(w.astype(np.float64), f[kept].astype(np.float64), ti, tj, tk, ns,
                                go.astype(np.float64))
    res = op.backward(torch.from_numpy(go).cuda())
    g = res.grad_in.cpu().numpy()
    mask = np.ones(n, bool)
    mask[kept] = False
    assert np.abs(g[mask]).max() == 0.0
    e = (orc.rel_error(out.cpu().numpy(), fo), orc.rel_error(g[kept], gi),
         orc.rel_error(res.grad_w.cpu().numpy(), gw))
    assert max(e) <= tol, e


def test_state_errors(npc, orc):
    w = torch.from_numpy(orc.make_weights(3, 1, 2, 2, 1, np.float64)).cuda()
    nat = npc.PointConvOp(w, npc.ConvGeometry(radius=0.5, t=3))
    with pytest.raises(npc.StateError):
        nat.snapped_cloud()
    cl = npc.make_point_cloud(orc.gen_uniform_cube(5, 1.0, 343))
    nat.forward(cl, torch.zeros((5, 1, 2), dtype=torch.float64, device="cuda"))
    with pytest.raises(npc.StateError):
        nat.site_map()
    dop = npc.PointConvOp(w, _geom(npc, 1.0, 3))
    with pytest.raises(npc.StateError):  # two-cloud forward requires native mode
        dop.forward(cl, cl, torch.zeros((5, 1, 2), dtype=torch.float64, device="cuda"))
