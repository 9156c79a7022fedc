"""Times the neighbor build (search + kernel cells + CSR) and the tensor-core
plan build separately for the north-star cloud, with the per-kernel device
times of each phase (library profiler)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_2511_23227_b200 import npconv as npc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
o = Oracle()
xyz = o.gen_uniform_cube(n, 1.0, 1)
r = 1.8 * n ** (-1 / 3)
ctx = npc.context()
for rep in range(3):
    cl = npc.make_point_cloud(xyz)
    torch.cuda.synchronize()
    ctx.profile_reset()
    ctx.profile(True)
    t0 = time.perf_counter()
    nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=3))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d1 = ctx.profile_dump()
    ctx.profile_reset()
    nb.prepare(npc.Math.bf16)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    d2 = ctx.profile_dump()
    ctx.profile(False)
    print(f"rep {rep}: build {1e3 * (t1 - t0):.1f} ms (kernels {sum(v[1] for v in d1.values()):.1f}), "
          f"plans {1e3 * (t2 - t1):.1f} ms (kernels {sum(v[1] for v in d2.values()):.1f})")
for name, d in (("build", d1), ("plans", d2)):
    print(name, ", ".join(f"{k} {v[0]}x {v[1]:.2f}" for k, v in sorted(d.items(), key=lambda kv: -kv[1][1])[:12]))
