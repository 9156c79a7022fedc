"""fwd+dgrad+wgrad device time vs cloud size (uniform cube, C=64, t=3, bf16
path), with the library's peak scratch memory: how the engines scale from a
few tiles to the size where L2 no longer holds the bf16 images."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_2511_23227_b200 import npconv as npc  # noqa: E402

o = Oracle()
cfg = npc.ExecConfig(math=npc.Math.bf16)
ctx = npc.context()
sizes = [int(x) for x in sys.argv[1:]] or [100_000, 250_000, 500_000, 1_000_000, 2_000_000, 4_000_000]
print("points,triplets,ms_per_step,Mpoints_per_s,fwd_ms,dgrad_ms,wgrad_ms,peak_scratch_GB")
for n in sizes:
    cl = npc.make_point_cloud(o.gen_uniform_cube(n, 1.0, 1))
    nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=1.8 * n ** (-1 / 3), t=3))
    nb.prepare(npc.Math.bf16)
    w = torch.from_numpy(o.make_weights(3, 1, 64, 64, 2)).cuda()
    f = torch.from_numpy(o.gen_features(n, 1, 64, 3)).cuda()
    g = torch.from_numpy(o.gen_features(n, 1, 64, 4)).cuda()
    fo, gi = torch.empty_like(f), torch.empty_like(f)
    gw = torch.empty((27, 1, 64, 64), device="cuda")
    for _ in range(3):
        npc.conv_forward(nb, w, f, cfg, out=fo)
        npc.conv_backward(nb, w, f, g, cfg, grad_in=gi, grad_w=gw)
    torch.cuda.synchronize()
    ctx.reset_peak()
    ctx.profile_reset()
    ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        npc.conv_forward(nb, w, f, cfg, out=fo)
        npc.conv_backward(nb, w, f, g, cfg, grad_in=gi, grad_w=gw)
    e1.record()
    torch.cuda.synchronize()
    d = ctx.profile_dump()
    ctx.profile(False)
    ms = e0.elapsed_time(e1) / 5
    k = lambda name: d.get(name, (1, 0.0))[1] / 5
    print(f"{n},{nb.size},{ms:.4f},{n / ms / 1e3:.1f},{k('conv_fwd_tc'):.4f},{k('conv_dgrad_tc'):.4f},"
          f"{k('conv_wgrad_tc'):.4f},{ctx.memory()[1] / 1e9:.3f}", flush=True)
    del nb, f, g, fo, gi
    torch.cuda.empty_cache()
