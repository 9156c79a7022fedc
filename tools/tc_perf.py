"""Times the tensor-core engines at the north-star size; prints plan stats and per-kernel ms.
    python tools/tc_perf.py [n] [iters] [math: bf16|f32tc|auto|exact]"""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle
from paper_2511_23227_b200 import npconv as npc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
o = Oracle()
xyz = o.gen_uniform_cube(n, 1.0, 1); r = 1.8 * n ** (-1/3)
T = lambda x: torch.from_numpy(x).cuda()
w = T(o.make_weights(3, 1, 64, 64, 2)); f = T(o.gen_features(n, 1, 64, 3)); g = T(o.gen_features(n, 1, 64, 4))
cl = npc.make_point_cloud(xyz)
nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=3))
t0 = time.time(); st = nb.plan_stats(); torch.cuda.synchronize()
print("plan", json.dumps(st), "build_s %.3f" % (time.time() - t0), flush=True)
cfg = npc.ExecConfig(math=getattr(npc.Math, sys.argv[3] if len(sys.argv) > 3 else "bf16"))
fo = torch.empty((n, 1, 64), device="cuda"); gi = torch.empty_like(fo); gw = torch.empty((27, 1, 64, 64), device="cuda")
for _ in range(2):
    npc.conv_forward(nb, w, f, cfg, out=fo); npc.conv_backward(nb, w, f, g, cfg, grad_in=gi, grad_w=gw, fin_unchanged=True)
torch.cuda.synchronize()
ctx = npc.context(); ctx.profile_reset(); ctx.profile(True)
for _ in range(iters):
    npc.conv_forward(nb, w, f, cfg, out=fo); npc.conv_backward(nb, w, f, g, cfg, grad_in=gi, grad_w=gw, fin_unchanged=True)
torch.cuda.synchronize()
d = ctx.profile_dump(); ctx.profile(False)
print("step %.4f ms" % (sum(v[1] for v in d.values()) / iters))
for k, (c, ms) in sorted(d.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:20s} {c:4d} launches  {ms / c:8.4f} ms/launch", flush=True)
