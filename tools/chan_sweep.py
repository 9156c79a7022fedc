"""Channel-width sweep of the conv passes at one cloud size: per-kernel device
time (library profiler, CUDA events on the library stream) of the tensor-core
and exact engines for (C_in, C_out) pairs.

    python tools/chan_sweep.py [n_points] [iters] [cin:cout ...]

CHAN_SWEEP_TC_ONLY=1 skips the exact engines.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_2511_23227_b200 import npconv as npc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pairs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[3:]] or \
    [(64, 64), (64, 128), (128, 128), (128, 256), (256, 256)]
o = Oracle()
xyz = o.gen_uniform_cube(n, 1.0, 1)
r = 1.8 * n ** (-1 / 3)
cl = npc.make_point_cloud(xyz)
nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=3))
ctx = npc.context()


def T(x):
    return torch.from_numpy(x).cuda()


for cin, cout in pairs:
    w = T(o.make_weights(3, 1, cin, cout, 2))
    f = T(o.gen_features(n, 1, cin, 3))
    g = T(o.gen_features(n, 1, cout, 4))
    maths = (npc.Math.bf16,) if os.environ.get("CHAN_SWEEP_TC_ONLY") else (npc.Math.bf16, npc.Math.exact)
    for math in maths:
        cfg = npc.ExecConfig(math=math)
        fo = torch.empty((n, 1, cout), device="cuda")
        gi = torch.empty((n, 1, cin), device="cuda")
        gw = torch.empty((27, 1, cin, cout), device="cuda")
        for _ in range(2):
            npc.conv_forward(nb, w, f, cfg, out=fo)
            npc.conv_backward(nb, w, f, g, cfg, grad_in=gi, grad_w=gw)
        torch.cuda.synchronize()
        ctx.profile_reset()
        ctx.profile(True)
        for _ in range(iters):
            npc.conv_forward(nb, w, f, cfg, out=fo)
            npc.conv_backward(nb, w, f, g, cfg, grad_in=gi, grad_w=gw)
        torch.cuda.synchronize()
        d = ctx.profile_dump()
        ctx.profile(False)
        tot = sum(ms for _, ms in d.values()) / iters
        top = sorted(d.items(), key=lambda kv: -kv[1][1])[:5]
        print(f"{cin:4d}->{cout:<4d} {math.name:6s} step {tot:8.3f} ms | " +
              "  ".join(f"{k} {ms / c:.3f}" for k, (c, ms) in top), flush=True)
