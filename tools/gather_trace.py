"""Per-stage timeline of the gather-engine forward kernel (CTA 0): loader
start/issued, fixup start/done, MMA start/issued (npcg_debug_trace_forward)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle
from paper_2511_23227_b200 import npconv as npc, _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
o = Oracle(); xyz = o.gen_uniform_cube(n, 1.0, 1); r = 1.8 * n ** (-1/3)
T = lambda x: torch.from_numpy(x).cuda()
w = T(o.make_weights(3, 1, 64, 64, 2)); f = T(o.gen_features(n, 1, 64, 3))
cl = npc.make_point_cloud(xyz); nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=3))
out = torch.empty((n, 1, 64), device="cuda")
tr = np.zeros(512 * 8, dtype=np.int64)
for _ in range(2):
    h = nb.ctx.bind()
    nb.ctx.check(L.lib().npcg_debug_trace_forward(h, nb.h, C.c_void_p(w.data_ptr()), C.c_void_p(f.data_ptr()), C.c_void_p(out.data_ptr()), tr.ctypes.data_as(C.c_void_p)), "trace")
t = tr.reshape(512, 8).astype(np.float64)
t0 = t[t > 0].min()
print("st   ld_start ld_issued fix_start fix_done mma_start mma_issued | issue->fix fix mma_wait")
for s in range(60, 100):
    x = t[s]
    print(f"{s:3d} " + " ".join(f"{(v - t0 if v > 0 else -1):9.0f}" for v in x[:6]) +
          f" | {x[2]-x[1]:6.0f} {x[3]-x[2]:6.0f} {x[4]-x[3]:6.0f}")
d = lambda a, b: np.median([t[s, b] - t[s, a] for s in range(20, 500) if t[s, a] > 0 and t[s, b] > 0])
iv = lambda e: np.median(np.diff([t[s, e] for s in range(20, 500) if t[s, e] > 0]))
print("median: ld_start->issued %.0f issued->fix_start %.0f fix %.0f fix_done->mma_start %.0f mma %.0f" % (d(0,1), d(1,2), d(2,3), d(3,4), d(4,5)))
print("median stage interval at mma_start %.0f, ld_start %.0f" % (iv(4), iv(0)))
print("ld_start(s) - mma_issued(s-5) median %.0f" % np.median([t[s,0]-t[s-5,5] for s in range(25,500) if t[s,0]>0 and t[s-5,5]>0]))
