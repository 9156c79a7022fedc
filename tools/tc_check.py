"""Quick tensor-core path check: small cloud, bf16 path vs oracle (prints errors)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle
from paper_2511_23227_b200 import npconv as npc

def rel(a, b):
    a = np.asarray(a, np.float64).ravel(); b = np.asarray(b, np.float64).ravel()
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))

o = Oracle()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
xyz = o.gen_uniform_cube(n, 1.0, 1); r = 1.8 * n ** (-1/3)
w = o.make_weights(3, 1, 64, 64, 2); f = o.gen_features(n, 1, 64, 3); g = o.gen_features(n, 1, 64, 4)
ti, tj, tk = o.build_triplets(xyz, xyz, r, 3)
fo, gi, gw = o.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n, g.astype(np.float64))
cl = npc.make_point_cloud(xyz)
T = lambda x: torch.from_numpy(x).cuda()
nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=3))
print("plan", nb.plan_stats(), flush=True)
cfg = npc.ExecConfig(math=npc.Math.bf16)
t0 = time.time()
out = npc.conv_forward(nb, T(w), T(f), cfg); torch.cuda.synchronize()
print("fwd", rel(out.cpu(), fo), time.time() - t0, flush=True)
gi_, gw_ = npc.conv_backward(nb, T(w), T(f), T(g), cfg, need_w=False); torch.cuda.synchronize()
print("dgrad", rel(gi_.cpu(), gi), flush=True)
_, gw_ = npc.conv_backward(nb, T(w), T(f), T(g), cfg, need_in=False); torch.cuda.synchronize()
print("wgrad", rel(gw_.cpu(), gw), flush=True)
