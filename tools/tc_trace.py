"""Pipeline timeline of the tensor-core forward kernel (CTA 0), from npcg_debug_trace_forward."""
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
names = ["d_issue", "d_full", "a_empty", "agg_done", "mma_start", "mma_issued", "w_full"]
print("stage " + " ".join(f"{x:>9s}" for x in names))
for s in list(range(0, 12)) + list(range(100, 112)):
    print(f"{s:5d} " + " ".join(f"{(t[s,e]-t0 if t[s,e] > 0 else -1):9.0f}" for e in range(7)))
v = lambda a, b: np.median([t[s, b] - t[s, a] for s in range(20, 400) if t[s, a] > 0 and t[s, b] > 0])
d = lambda e: np.median(np.diff([t[s, e] for s in range(20, 400) if t[s, e] > 0]))
print("median per-stage interval: mma_start %.0f  agg_done %.0f  d_issue %.0f" % (d(4), d(3), d(0)))
print("median latencies: d_issue->d_full %.0f  a_empty->agg_done %.0f  agg_done->mma_start %.0f  mma_start->mma_issued %.0f" % (v(0,1), v(2,3), v(3,4), v(4,5)))
print("median d_full->a_empty %.0f" % v(1, 2))
# halo switches: gap between consecutive MMA starts, at super-tile boundaries (54 stages per 2 x 128-row super-tile)
ms = np.array([t[s, 4] for s in range(512) if t[s, 4] > 0])
gaps = np.diff(ms)
per = 2 * 27
bnd = [gaps[i] for i in range(len(gaps)) if (i + 1) % per == 0]
inner = [gaps[i] for i in range(len(gaps)) if (i + 1) % per != 0]
print("MMA-start gaps: inner median %.0f mean %.0f | super-tile boundary median %.0f mean %.0f (n=%d)"
      % (np.median(inner), np.mean(inner), np.median(bnd), np.mean(bnd), len(bnd)))
print("boundary share of time: %.1f%%" % (100 * np.sum(bnd) / np.sum(gaps)))
