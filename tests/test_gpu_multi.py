"""GPU: the library's own multi-GPU exchange -- the NCCL
communicator of libnpcg (npcg_comm_create / npcg_allreduce_dw through
shard.DwComm) and ConvStack's dW all-reduce overlapped with the next layer's
backward.  One GPU: world size 1 (the all-reduce is the identity; the
overlap path must not change a bit).  Two GPUs (skipped on a one-GPU box):
two ranks each own half of the scenes (shard.scene_range), the summed dW
equals the single-process dW over all scenes within fp32 tolerance, and
both ranks hold identical sums."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from test_gpu_operator import T, rel

pytestmark = pytest.mark.gpu


def _stack_case(npc, orc, n=6000):
    xyz = orc.gen_uniform_cube(n, 1.0, 4)
    r = 1.8 * n ** (-1 / 3)
    ws = [T(orc.make_weights(3, 1, 64, 64, 30 + l)) for l in range(3)]
    f = T(orc.gen_features(n, 1, 64, 40))
    g = T(orc.gen_features(n, 1, 64, 41))
    return npc.make_point_cloud(xyz), r, ws, f, g


@pytest.mark.parametrize("math", ["bf16", "auto"])
def test_stack_dw_allreduce_overlap_world1(npc, orc, math):
    from paper_2511_23227_b200 import shard
    from paper_2511_23227_b200.stack import ConvStack
    cl, r, ws, f, g = _stack_case(npc, orc)
    cfg = npc.ExecConfig(math=getattr(npc.Math, math))
    geom = npc.ConvGeometry(radius=r, t=3)
    plain = ConvStack(ws, geom, cfg)
    plain.forward(cl, f)
    ref = plain.backward(g)
    comm = shard.DwComm(0, 1)
    st = ConvStack(ws, geom, cfg, comm=comm)
    st.forward(cl, f)
    got = st.backward(g)
    torch.cuda.synchronize()
    assert torch.equal(got.grad_in, ref.grad_in)
    for a, b in zip(got.grad_w, ref.grad_w):
        assert torch.equal(a, b)
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from oracle import Oracle
    from paper_2511_23227_b200 import npconv as npc
    from paper_2511_23227_b200 import shard
    orc = Oracle()
    dev = torch.device("cuda", rank)
    comm = shard.DwComm(rank, world, rank)
    w = torch.from_numpy(orc.make_weights(3, 1, 64, 64, 2)).to(dev)
    cfg = npc.ExecConfig(math=npc.Math.auto)
    a, b = shard.scene_range(4, rank, world)
    gw = torch.zeros((27, 1, 64, 64), device=dev)
    for s in range(a, b):
        n = 5000
        cl = npc.make_point_cloud(orc.gen_uniform_cube(n, 1.0, 1 + s), device=dev)
        nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=1.8 * n ** (-1 / 3), t=3))
        f = torch.from_numpy(orc.gen_features(n, 1, 64, 100 + s)).to(dev)
        g = torch.from_numpy(orc.gen_features(n, 1, 64, 200 + s)).to(dev)
        _, gws = npc.conv_backward(nb, w, f, g, cfg, need_in=False)
        gw += gws
    comm.allreduce(gw)
    torch.cuda.synchronize()
    q.put((rank, gw.cpu().numpy()))
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (the gpurun box has one)")
def test_library_allreduce_world2(npc, orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = orc.make_weights(3, 1, 64, 64, 2).astype(np.float64)
    total = np.zeros((27, 1, 64, 64))
    for s in range(4):
        n = 5000
        xyz = orc.gen_uniform_cube(n, 1.0, 1 + s)
        ti, tj, tk = orc.build_triplets(xyz, xyz, 1.8 * n ** (-1 / 3), 3)
        f = orc.gen_features(n, 1, 64, 100 + s).astype(np.float64)
        g = orc.gen_features(n, 1, 64, 200 + s).astype(np.float64)
        total += orc.dense_conv(w, f, ti, tj, tk, n, g)[2]
    assert np.array_equal(res[0], res[1])
    assert rel(res[0], total) <= 1e-5
