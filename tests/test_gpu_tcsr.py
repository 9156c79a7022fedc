"""GPU: the transposed neighbor structure of same-cloud handles is taken from
the forward arrays (the radius relation is symmetric) with each entry's cell
found in the forward row (csrc/neighbors.cu, k_tcsr_cells).  It must equal
the stable radix-sort build (NPCG_TCSR_SORT=1) exactly: the exact-engine input
gradient (which walks the transposed rows in order) and the bf16 fused
backward (planned over them) are bitwise equal between the two builds, on
uniform and clustered clouds, one and several batches, t = 3 and 5."""
import os

import numpy as np
import pytest
import torch

from test_gpu_operator import T

pytestmark = pytest.mark.gpu


def _cloud(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.random((n, 3)), None
    if kind == "clusters":
        c = rng.random((12, 3)) * 4
        xyz = c[rng.integers(0, 12, n)] + rng.normal(0, 0.15, (n, 3))
        return xyz, None
    xyz = rng.random((n, 3))  # three scenes of a jagged batch
    return xyz, [0, n // 5, n // 2, n]


def _backward(npc, orc, xyz, off, r, t, math, tcsr_sort):
    old = os.environ.get("NPCG_TCSR_SORT")
    os.environ["NPCG_TCSR_SORT"] = "1" if tcsr_sort else "0"
    try:
        n = len(xyz)
        cl = npc.make_point_cloud(xyz, off)
        nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=t))
        dt = np.float64 if math == "exact" else np.float32
        w = T(orc.make_weights(t, 1, 64, 64, 3).astype(dt))
        f = T(orc.gen_features(n, 1, 64, 4).astype(dt))
        g = T(orc.gen_features(n, 1, 64, 5).astype(dt))
        gi, gw = npc.conv_backward(nb, w, f, g, npc.ExecConfig(math=getattr(npc.Math, math)))
        torch.cuda.synchronize()
        return gi, gw
    finally:
        if old is None:
            os.environ.pop("NPCG_TCSR_SORT", None)
        else:
            os.environ["NPCG_TCSR_SORT"] = old


@pytest.mark.parametrize("kind", ["uniform", "clusters", "batches"])
@pytest.mark.parametrize("t", [3, 5])
def test_same_cloud_transposed_structure_equals_sorted_build(npc, orc, kind, t):
    n = 20000
    xyz, off = _cloud(kind, n, 7 + t)
    r = 1.8 * n ** (-1 / 3) * (1.0 if kind != "clusters" else 0.5)
    for math in ("exact", "bf16"):
        a = _backward(npc, orc, xyz, off, r, t, math, tcsr_sort=True)
        b = _backward(npc, orc, xyz, off, r, t, math, tcsr_sort=False)
        assert torch.equal(a[0], b[0]), (kind, t, math, "grad_in")
        assert torch.equal(a[1], b[1]), (kind, t, math, "grad_w")


def test_fast_transposed_build_is_used(npc, orc):
    ctx = npc.context()
    ctx.profile_reset()
    ctx.profile(True)
    xyz, _ = _cloud("uniform", 5000, 1)
    cl = npc.make_point_cloud(xyz)
    nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=1.8 * 5000 ** (-1 / 3), t=3))
    ctx.profile_reset()
    w = T(orc.make_weights(3, 1, 64, 64, 3).astype(np.float64))
    g = T(orc.gen_features(5000, 1, 64, 5).astype(np.float64))
    npc.conv_backward(nb, w, None, g, npc.ExecConfig(math=npc.Math.exact), need_w=False)
    torch.cuda.synchronize()
    prof = ctx.profile_dump()
    ctx.profile(False)
    assert "tcsr_cells" in prof and "radix_scatter" not in prof, sorted(prof)
