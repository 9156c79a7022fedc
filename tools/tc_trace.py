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
tr = np.zeros(512 * 16, dtype=np.int64)
for _ in range(2):
    h = nb.ctx.bind()
    nb.ctx.check(L.lib().npcg_debug_trace_forward(h, nb.h, C.c_void_p(w.data_ptr()), C.c_void_p(f.data_ptr()), C.c_void_p(out.data_ptr()), tr.ctypes.data_as(C.c_void_p)), "trace")
t = tr.reshape(512, 16).astype(np.float64)
t0 = t[t > 0].min()
names = ["d_issue", "d_full", "a_empty", "agg_done", "mma_start", "mma_issued", "w_full", "grp_done"]
print("stage " + " ".join(f"{x:>9s}" for x in names))
for s in list(range(0, 12)) + list(range(100, 112)):
    print(f"{s:5d} " + " ".join(f"{(t[s,e]-t0 if t[s,e] > 0 else -1):9.0f}" for e in range(8)))
v = lambda a, b: np.median([t[s, b] - t[s, a] for s in range(20, 400) if t[s, a] > 0 and t[s, b] > 0])
d = lambda e: np.median(np.diff([t[s, e] for s in range(20, 400) if t[s, e] > 0]))
print("median per-stage interval: mma_start %.0f  agg_done %.0f  d_issue %.0f" % (d(4), d(3), d(0)))
print("median latencies: d_issue->d_full %.0f  a_empty->agg_done %.0f  agg_done->mma_start %.0f  mma_start->mma_issued %.0f" % (v(0,1), v(2,3), v(3,4), v(4,5)))
print("median d_full->a_empty %.0f  agg_done(w0)->grp_done %.0f  grp_done->mma_start %.0f" % (v(1, 2), v(3, 7), v(7, 4)))
# halo switches: gap between consecutive MMA starts, at super-tile boundaries (54 stages per 2 x 128-row super-tile)
ms = np.array([t[s, 4] for s in range(512) if t[s, 4] > 0])
gaps = np.diff(ms)
per = 2 * 27
bnd = [gaps[i] for i in range(len(gaps)) if (i + 1) % per == 0]
inner = [gaps[i] for i in range(len(gaps)) if (i + 1) % per != 0]
print("MMA-start gaps: inner median %.0f mean %.0f | super-tile boundary median %.0f mean %.0f (n=%d)"
      % (np.median(inner), np.mean(inner), np.median(bnd), np.mean(bnd), len(bnd)))
print("boundary share of time: %.1f%%" % (100 * np.sum(bnd) / np.sum(gaps)))
# slot round trip: MMA of stage s issued -> the slot's next user (s + NSA) acquires it
w = lambda a, b, dj: np.median([t[s + dj, b] - t[s, a] for s in range(20, 400) if t[s, a] > 0 and t[s + dj, b] > 0])
print("mma_issued(s) -> a_empty(s+4) %.0f   d_full(s+4) - mma_issued(s) %.0f" % (w(5, 2, 4), w(5, 1, 4)))
# MMA-warp loop: first stage of a cell (even s) -- previous issue -> W wait passed -> first issue
ev = [s for s in range(20, 400, 2) if t[s, 6] > 0 and t[s - 1, 5] > 0]
print("MMA warp per cell: issued(s-1)->w_full(s) %.0f  w_full(s)->mma_start(s) %.0f  issued(s)->start(s+1) %.0f"
      % (np.median([t[s, 6] - t[s - 1, 5] for s in ev]), np.median([t[s, 4] - t[s, 6] for s in ev]),
         np.median([t[s + 1, 4] - t[s, 5] for s in ev])))
ev = [s for s in range(20, 400, 2) if t[s, 8] > 0 and t[s, 12] > 0 and t[s + 1, 11] > 0]
m = lambda a, b, da=0, db=0: np.median([t[s + db, b] - t[s + da, a] for s in ev])
print("cell: top->w_full %.0f  w_full->start0 %.0f  start0->fence0 %.0f  fence0->mmadone0 %.0f  mmadone0->issued0 %.0f"
      % (m(8, 6), m(6, 4), m(4, 10), m(10, 11), m(11, 5)))
print("      issued0->start1 %.0f  start1->fence1 %.0f fence1->mmadone1 %.0f  mmadone1->issued1 %.0f  issued1->cell_end %.0f  cell_end->next top %.0f"
      % (m(5, 4, 0, 1), m(4, 10, 1, 1), m(10, 11, 1, 1), m(11, 5, 1, 1), m(5, 12, 1, 0), m(12, 8, 0, 2)))
