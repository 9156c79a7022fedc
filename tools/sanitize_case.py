"""One small conv layer per engine, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) over the library's kernels: neighbor build, tile
planning, the tcgen05 forward / fused backward / wgrad / split kernels and the
exact CUDA-core engines.  Results are checked against the fp64 oracle so a run
that the tool perturbs still has to be right.  tools/sanitize.sh drives it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import Oracle
from paper_2511_23227_b200 import npconv as npc


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    n = int(os.environ.get("SAN_POINTS", "3000"))
    maths = os.environ.get("SAN_MATH", "bf16,auto,exact").split(",")
    o = Oracle()
    xyz = o.gen_uniform_cube(n, 1.0, 3)
    r = 1.8 * n ** (-1 / 3)
    T = lambda x: torch.from_numpy(x).cuda()
    for math in maths:
        for cin, cout in ((64, 64), (64, 128)):
            w = o.make_weights(3, 1, cin, cout, 5)
            f = o.gen_features(n, 1, cin, 6)
            g = o.gen_features(n, 1, cout, 7)
            cl = npc.make_point_cloud(xyz)
            nb = npc.build_neighbors(cl, cl, npc.ConvGeometry(radius=r, t=3))
            cfg = npc.ExecConfig(math=getattr(npc.Math, math))
            out = npc.conv_forward(nb, T(w), T(f), cfg)
            gi, gw = npc.conv_backward(nb, T(w), T(f), T(g), cfg)
            torch.cuda.synchronize()
            ti, tj, tk = o.build_triplets(xyz, xyz, r, 3)
            fo, egi, egw = o.dense_conv(w.astype(np.float64), f.astype(np.float64), ti, tj, tk, n,
                                        g.astype(np.float64))
            tol = 1e-2 if math == "bf16" else 1e-5
            e = (rel(out.cpu(), fo), rel(gi.cpu(), egi), rel(gw.cpu(), egw))
            print(f"{math} {cin}->{cout}: rel {e[0]:.1e} {e[1]:.1e} {e[2]:.1e}")
            assert max(e) <= tol, (math, cin, cout, e)
    print("SANITIZE CASE OK")


if __name__ == "__main__":
    main()
