"""GPU: the strided path at the boundary --
upsample (spatial.cpp:154-169, npcg_upsample) and strided_block
(conv_op.hpp:219-225) checked against the unmodified reference
(oracle/_ref) on the same inputs."""
import numpy as np
import pytest
import torch

from test_gpu_operator import T, rel

pytestmark = pytest.mark.gpu


def _cloud(npc, xyz, off):
    return npc.PointCloud(torch.as_tensor(np.ascontiguousarray(xyz)).to("cuda"),
                          np.asarray(off, np.int64))


@pytest.mark.parametrize("dtype,G,C", [(np.float32, 1, 64), (np.float32, 2, 5),
                                       (np.float64, 1, 3), (np.float64, 1, 128)])
def test_upsample_matches_reference(npc, ref, dtype, G, C):
    xyz = ref.gen_gaussian_clusters(6000, 12, 2.0, 0.3, 77)
    off = np.array([0, 2500, 2500, 6000])
    v = 0.35
    coarse_cl, mp = npc.voxel_downsample(_cloud(npc, xyz, off), v)
    kept, parent = mp.kept_index.cpu().numpy(), mp.parent_of.cpu().numpy()
    rk, rp, _ = ref.voxel_downsample(xyz, v, off)
    assert np.array_equal(kept, rk) and np.array_equal(parent, rp)
    rng = np.random.default_rng(5)
    coarse = rng.uniform(-1, 1, size=(len(kept), G, C)).astype(dtype)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    fine = npc.upsample(_cloud(npc, xyz, off), mp, T(coarse, tdt))
    expect = ref.upsample(xyz, kept, parent, coarse, off)
    assert fine.shape == expect.shape
    assert np.array_equal(fine.cpu().numpy(), expect)  # a row copy: bit-identical


def test_upsample_errors(npc, orc):
    import ctypes as C
    from paper_2511_23227_b200 import _lib as L
    xyz = orc.gen_uniform_cube(500, 1.0, 2)
    cl = _cloud(npc, xyz, [0, 500])
    coarse_cl, mp = npc.voxel_downsample(cl, 0.3)
    nk = mp.kept_index.numel()
    with pytest.raises(npc.ShapeError):  # spatial.cpp:156-157
        npc.upsample(_cloud(npc, xyz[:400], [0, 400]), mp, T(np.zeros((nk, 1, 4))))
    with pytest.raises(npc.ShapeError):  # spatial.cpp:158-159
        npc.upsample(cl, mp, T(np.zeros((nk + 1, 1, 4))))
    # a parent outside the coarse rows: IndexError before any copy (the ABI)
    ctx = npc.context()
    h = ctx.bind()
    bad = mp.parent_of.clone()
    bad[7] = nk
    src = T(np.ones((nk, 4)))
    dst = torch.zeros((500, 4), device="cuda")
    st = L.lib().npcg_upsample(h, 0, bad.data_ptr(), 500, src.data_ptr(), nk, 4, dst.data_ptr())
    assert st == 6  # NPCG_ERR_INDEX
    assert float(dst.abs().sum()) == 0.0
    assert L.lib().npcg_upsample(h, 0, bad.data_ptr(), 500, src.data_ptr(), nk, 0,
                                 dst.data_ptr()) == 3  # width < 1: ShapeError
    del C


@pytest.mark.parametrize("math,tol", [("exact", 1e-5), ("bf16", 1e-2)])
def test_strided_block_matches_reference(npc, ref, orc, math, tol):
    """strided_block: voxel_downsample(cloud) then the two-cloud conv from the
    fine cloud onto the kept points; the reference chain (its downsample, its
    build_triplets_native(coarse, fine), its fp64 dense oracle) on the same
    inputs."""
    xyz = ref.gen_gaussian_clusters(8000, 20, 2.0, 0.25, 31)
    off = np.array([0, 3000, 8000])
    v = 0.2
    r = 1.8 * v
    cin, cout = 64, 128
    w = orc.make_weights(3, 1, cin, cout, 9)
    f = orc.gen_features(len(xyz), 1, cin, 10)
    op = npc.PointConvOp(T(w), npc.ConvGeometry(radius=r, t=3),
                         npc.ExecConfig(math=getattr(npc.Math, math)))
    res = npc.strided_block(op, _cloud(npc, xyz, off), T(f), v)
    rk, rp, roff = ref.voxel_downsample(xyz, v, off)
    assert np.array_equal(res.map.kept_index.cpu().numpy(), rk)
    assert np.array_equal(res.map.parent_of.cpu().numpy(), rp)
    assert np.array_equal(res.coarse_cloud.batch_offsets(), roff)
    cxyz = xyz[rk]
    ti, tj, tk = ref.build_triplets(cxyz, xyz, r, 3, out_off=roff, in_off=off)
    fo, _, _ = ref.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, len(rk))
    assert res.coarse_features.shape == (len(rk), 1, cout)
    assert rel(res.coarse_features.cpu(), fo) <= tol
    # and back up: every fine point gets its voxel's coarse row
    up = npc.upsample(_cloud(npc, xyz, off), res.map, res.coarse_features)
    expect = ref.upsample(xyz, rk, rp, res.coarse_features.cpu().numpy(), off)
    assert np.array_equal(up.cpu().numpy(), expect)
