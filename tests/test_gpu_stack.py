"""GPU: layer stacks over one shared neighbor structure, CUDA-graph replay
(test_conv_op.cpp:270-309)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _oracle_chain(orc, ws, f, tl, n, gout):
    ti, tj, tk = (x.cpu().numpy().view(np.uint32) for x in (tl.i, tl.j, tl.k))
    acts = [f.astype(np.float64)]
    for w in ws:
        fo, _, _ = orc.dense_conv(w.astype(np.float64), acts[-1], ti, tj, tk, n)
        acts.append(fo)
    g = gout.astype(np.float64)
    gws = [None] * len(ws)
    for l in range(len(ws) - 1, -1, -1):
        _, g, gws[l] = orc.dense_conv(ws[l].astype(np.float64), acts[l], ti, tj, tk, n, g)
    return acts[-1], g, gws


def test_stacked_layers_compose_like_the_oracle(npc, orc):
    """test_conv_op.cpp:291-309 (fp64, rel <= 1e-12), plus the backward chain."""
    from paper_2511_23227_b200.stack import ConvStack
    n = 80
    cl = npc.make_point_cloud(orc.gen_uniform_cube(n, 2.0, 401))
    ws = [orc.make_weights(3, 1, 3, 5, 402, np.float64), orc.make_weights(3, 1, 5, 4, 403, np.float64)]
    f = orc.gen_features(n, 1, 3, 404, np.float64)
    gout = orc.gen_features(n, 1, 4, 405, np.float64)
    st = ConvStack([_T(w) for w in ws], npc.ConvGeometry(radius=0.6, t=3),
                   npc.ExecConfig(deterministic=True))
    out = st.forward(cl, _T(f))
    gr = st.backward(_T(gout))
    fo, gi, gws = _oracle_chain(orc, ws, f, st.ops[0].cached_triplets(), n, gout)
    assert orc.rel_error(out.cpu().numpy(), fo) <= 1e-12
    assert orc.rel_error(gr.grad_in.cpu().numpy(), gi) <= 1e-12
    for a, b in zip(gr.grad_w, gws):
        assert orc.rel_error(a.cpu().numpy(), b) <= 1e-12


def test_cache_shared_and_reused(npc, orc):
    """test_conv_op.cpp:270-289: same cloud -> the cache survives; another
    cloud rebuilds it.  All layers of a stack share one handle."""
    from paper_2511_23227_b200.stack import ConvStack
    n = 50
    cl = npc.make_point_cloud(orc.gen_uniform_cube(n, 2.0, 391))
    ws = [_T(orc.make_weights(3, 1, 3, 3, 392, np.float64)) for _ in range(3)]
    st = ConvStack(ws, npc.ConvGeometry(radius=0.5, t=3))
    st.forward(cl, _T(orc.gen_features(n, 1, 3, 393, np.float64)))
    h = st.neighbors(cl)
    assert all(op.neighbors() is h for op in st.ops)
    st.forward(cl, _T(orc.gen_features(n, 1, 3, 394, np.float64)))
    assert st.neighbors(cl) is h
    other = npc.make_point_cloud(orc.gen_uniform_cube(n, 2.0, 395))
    st.forward(other, _T(orc.gen_features(n, 1, 3, 393, np.float64)))
    assert st.neighbors(other) is not h and st.ops[0].cached_triplets().size() >= 0


def test_c64_stack_tensor_core_and_graph(npc, orc):
    """A 3-layer C=64 stack on the tcgen05 path: within the bf16 bound of the
    fp64 oracle chain; a captured CUDA graph replays bit-identically to the
    eager step, also on fresh inputs copied into its static buffers."""
    from paper_2511_23227_b200.stack import ConvStack
    n = 20000
    cl = npc.make_point_cloud(orc.gen_uniform_cube(n, 1.0, 7))
    r = 1.8 * n ** (-1 / 3)
    ws = [orc.make_weights(3, 1, 64, 64, 10 + l) for l in range(3)]
    st = ConvStack([_T(w) for w in ws], npc.ConvGeometry(radius=r, t=3),
                   npc.ExecConfig(math=npc.Math.bf16))
    f = orc.gen_features(n, 1, 64, 3)
    gout = orc.gen_features(n, 1, 64, 4)
    out = st.forward(cl, _T(f)).clone()
    gr = st.backward(_T(gout))
    gi, gws = gr.grad_in.clone(), [g.clone() for g in gr.grad_w]
    fo, ogi, ogws = _oracle_chain(orc, ws, f, st.ops[0].cached_triplets(), n, gout)
    e = [orc.rel_error(out.cpu().numpy(), fo), orc.rel_error(gi.cpu().numpy(), ogi)] + \
        [orc.rel_error(a.cpu().numpy(), b) for a, b in zip(gws, ogws)]
    assert max(e) <= 1e-2, e
    st.capture(cl, _T(f), _T(gout))
    o2, g2 = st.replay()
    torch.cuda.synchronize()
    assert torch.equal(o2, out) and torch.equal(g2.grad_in, gi)
    assert all(torch.equal(a, b) for a, b in zip(g2.grad_w, gws))
    f_new, g_new = orc.gen_features(n, 1, 64, 30), orc.gen_features(n, 1, 64, 40)
    st.static_fin.copy_(_T(f_new))
    st.static_gout.copy_(_T(g_new))
    o3, g3 = st.replay()
    o3, gi3 = o3.clone(), g3.grad_in.clone()
    eo = st.forward(cl, _T(f_new))
    eg = st.backward(_T(g_new))
    assert torch.equal(o3, eo) and torch.equal(gi3, eg.grad_in)
