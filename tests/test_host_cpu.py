"""Host-side logic of the mirror API and the multi-GPU sharding, on CPU.

The N>1 path of bench.py shards whole clouds of a batch across ranks and
all-reduces the weight gradient.  The rank/shard arithmetic
and the reduction are exercised here with world_size 2 over gloo, using the
oracle as the per-rank engine (CPU stand-in for the GPU engines)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_23227_b200 import npconv
from paper_2511_23227_b200 import shard


def test_validate_offsets():
    npconv.validate_offsets(3, [0, 3])
    npconv.validate_offsets(4, [0, 0, 4])
    with pytest.raises(npconv.OffsetError):
        npconv.validate_offsets(3, [0])
    with pytest.raises(npconv.OffsetError):
        npconv.validate_offsets(3, [1, 3])
    with pytest.raises(npconv.OffsetError):
        npconv.validate_offsets(3, [0, 2])
    with pytest.raises(npconv.OffsetError):
        npconv.validate_offsets(4, [0, 3, 2, 4])


def test_make_point_cloud_rejects_nonfinite_before_upload():
    with pytest.raises(npconv.NonFiniteError):
        npconv.make_point_cloud(np.array([[0.0, np.nan, 0.0]]))
    with pytest.raises(npconv.OffsetError):
        npconv.make_point_cloud(np.zeros((2, 3)), [0, 1])


def test_error_hierarchy_names():
    for cls in (npconv.OffsetError, npconv.NonFiniteError, npconv.ShapeError, npconv.RadiusError,
                npconv.VoxelError, npconv.IndexError, npconv.DomainError, npconv.StateError,
                npconv.IOError):
        assert issubclass(cls, npconv.Error)
    assert npconv.IndexError is npconv.NpcIndexError


def test_shard_ranges_cover_batch():
    for n_scenes in (1, 7, 64):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.scene_range(n_scenes, r, world) for r in range(world)]
            flat = [s for a, b in spans for s in range(a, b)]
            assert flat == list(range(n_scenes))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    orc = Oracle()
    n_scenes, n_pts, t = 4, 300, 3
    w = orc.make_weights(t, 1, 4, 5, 2, np.float64)
    gw_local = np.zeros((27, 1, 5, 4))
    a, b = shard.scene_range(n_scenes, rank, world)
    for s in range(a, b):
        xyz = orc.gen_uniform_cube(n_pts, 1.0, 1 + s)
        r = 1.8 * n_pts ** (-1 / 3)
        ti, tj, tk = orc.build_triplets(xyz, xyz, r, t)
        fin = orc.gen_features(n_pts, 1, 4, 100 + s, np.float64)
        gout = orc.gen_features(n_pts, 1, 5, 200 + s, np.float64)
        _, _, gw = orc.dense_conv(w, fin, ti, tj, tk, n_pts, gout)
        gw_local += gw
    tens = torch.from_numpy(gw_local)
    shard.allreduce_weight_grad(tens)
    q.put((rank, tens.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_weight_grad_allreduce_equals_single_process():
    from oracle import Oracle
    orc = Oracle()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: all 4 scenes summed
    w = orc.make_weights(3, 1, 4, 5, 2, np.float64)
    total = np.zeros((27, 1, 5, 4))
    for s in range(4):
        xyz = orc.gen_uniform_cube(300, 1.0, 1 + s)
        r = 1.8 * 300 ** (-1 / 3)
        ti, tj, tk = orc.build_triplets(xyz, xyz, r, 3)
        fin = orc.gen_features(300, 1, 4, 100 + s, np.float64)
        gout = orc.gen_features(300, 1, 5, 200 + s, np.float64)
        total += orc.dense_conv(w, fin, ti, tj, tk, 300, gout)[2]
    assert np.allclose(res[0], total, rtol=1e-12, atol=1e-12)
    assert np.array_equal(res[0], res[1])
