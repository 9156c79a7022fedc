"""Device-timed measurements of BASELINE.json configs 1-4 on one GPU
(config 5 is `bench.py --workload batch64`).  One JSON line per config.

  c1  16K uniform points, C_in = C_out = 32, forward only   (exact fp32 engine)
  c2  100K uniform points, C = 64, forward + dgrad + wgrad  (bf16-operand tcgen05)
  c3  LiDAR-like scan, 120K points: voxel downsample (~4x) + strided 64 -> 128
      conv (two-cloud build), forward + backward
  c4  1M-point indoor fragment, 7-layer encoder/decoder (64 -> 128 -> 256 -> 128 -> 64),
      strided convs down, transposed (coarse -> fine) convs up, forward + backward

The reference ships no LiDAR / indoor generators and no network stack
("builder defines"); the generators are this repo's
(paper_2511_23227_b200/synthetic.py), seeded and described in DESIGN.md.  Mpoints/s = output points of the config's
unit / device time (CUDA events on the library stream, after warm-up); the
tensor fraction counts F = 2 |T| C_in C_out per pass.

    python tools/configs_bench.py [c1 c2 c3 c4] [--steps K] [--warmup W]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_2511_23227_b200 import npconv as npc  # noqa: E402
from paper_2511_23227_b200.synthetic import gen_indoor_fragment, gen_lidar_scan  # noqa: E402


def peaks():
    p = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
    bf16 = p.get("bf16_tflops_sustained") or p.get("bf16_tflops") or 1379.2
    return float(bf16)


def voxel_for_ratio(cloud: npc.PointCloud, ratio: float) -> tuple[float, npc.PointCloud]:
    """Bisection on the voxel edge for n_coarse ~= n / ratio (GPU voxel_downsample)."""
    n = cloud.n_points()
    x = cloud.xyz
    ext = float((x.max(0).values - x.min(0).values).max())
    lo, hi = ext * 1e-6, ext
    best = None
    for _ in range(40):
        v = (lo * hi) ** 0.5
        coarse, _ = npc.voxel_downsample(cloud, v)
        m = coarse.n_points()
        best = (v, coarse)
        if abs(m * ratio / n - 1) < 0.02:
            break
        if m * ratio > n:
            lo = v
        else:
            hi = v
    return best


# ---------------------------------------------------------------------------
class Layer:
    def __init__(self, name, out_cloud, in_cloud, radius, cin, cout, seed, orc, math):
        self.name, self.cin, self.cout = name, cin, cout
        self.nb = npc.build_neighbors(out_cloud, in_cloud, npc.ConvGeometry(radius=radius, t=3))
        self.nb.prepare(math)
        self.w = torch.from_numpy(orc.make_weights(3, 1, cin, cout, seed)).cuda()
        self.n_out, self.n_in = out_cloud.n_points(), in_cloud.n_points()


def time_steps(step, steps, warmup):
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx = npc.context()
    ctx.profile_reset()
    ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    prof = ctx.profile_dump()
    ctx.profile(False)
    return e0.elapsed_time(e1) / steps, prof


def run_stack(layers, fin, math, steps, warmup):
    cfg = npc.ExecConfig(math=math)
    acts = [fin]
    outs = [torch.empty((l.n_out, 1, l.cout), device="cuda") for l in layers]
    gis = [torch.empty((l.n_in, 1, l.cin), device="cuda") for l in layers]
    gws = [torch.empty((27, 1, l.cin, l.cout), device="cuda") for l in layers]
    gtop = torch.from_numpy(Oracle().gen_features(layers[-1].n_out, 1, layers[-1].cout, 4)).cuda()

    def step():
        h = acts[0]
        for l, o in zip(layers, outs):
            npc.conv_forward(l.nb, l.w, h, cfg, out=o)
            h = o
        g = gtop
        for i in range(len(layers) - 1, -1, -1):
            l = layers[i]
            inp = acts[0] if i == 0 else outs[i - 1]
            npc.conv_backward(l.nb, l.w, inp, g, cfg, grad_in=gis[i], grad_w=gws[i])
            g = gis[i]
    return time_steps(step, steps, warmup)


def per_layer(layers, fin, math, steps):
    """Device ms of each layer's forward + backward alone (same buffers)."""
    cfg = npc.ExecConfig(math=math)
    o = Oracle()
    out = []
    h = fin
    for l in layers:
        x = h if h.shape[2] == l.cin and h.shape[0] == l.n_in else \
            torch.from_numpy(o.gen_features(l.n_in, 1, l.cin, 5)).cuda()
        y = torch.empty((l.n_out, 1, l.cout), device="cuda")
        g = torch.from_numpy(o.gen_features(l.n_out, 1, l.cout, 6)).cuda()
        gi = torch.empty((l.n_in, 1, l.cin), device="cuda")
        gw = torch.empty((27, 1, l.cin, l.cout), device="cuda")

        def step():
            npc.conv_forward(l.nb, l.w, x, cfg, out=y)
            npc.conv_backward(l.nb, l.w, x, g, cfg, grad_in=gi, grad_w=gw)
        ms, prof = time_steps(step, steps, 2)
        st = l.nb.plan_stats() if (l.cin, l.cout) == (64, 64) else None
        out.append({"name": l.name, "ms": round(ms, 4),
                    "kernels": {k: round(v[1] / steps, 4) for k, v in prof.items() if v[1] / steps > 0.01},
                    "plan": st})
        h = y
    return out


def result(name, desc, unit_points, ms, prof, layers, bf16, extra):
    flop = sum(3 * 2 * l.nb.size * l.cin * l.cout for l in layers)
    return {"config": name, "math": MATH, "workload": desc,
            "value": round(unit_points / (ms / 1e3) / 1e6, 3),
            "unit": "Mpoints/s", "ms_per_step": round(ms, 4),
            "tensor_frac": round(flop / (ms / 1e3) / 1e12 / bf16, 4),
            "algorithmic_flop_per_step": flop,
            "layers": [{"name": l.name, "n_out": l.n_out, "n_in": l.n_in, "c_in": l.cin,
                        "c_out": l.cout, "triplets": l.nb.size} for l in layers],
            "kernels_ms_per_step": {k: round(v[1] / max(1, STEPS), 4) for k, v in
                                    sorted(prof.items(), key=lambda kv: -kv[1][1])},
            **extra}


STEPS = 5
MATH = "bf16"


def main():
    global STEPS, MATH
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c4"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--math", default="bf16", choices=["bf16", "auto", "exact", "f32tc"],
                    help="arithmetic of c2-c4 (c1 always reports auto = the split fp32-contract path, exact, and bf16)")
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    STEPS = a.steps
    orc = Oracle()
    bf16 = peaks()
    auto = getattr(npc.Math, a.math)
    MATH = a.math
    for c in a.configs:
        t0 = time.time()
        if c == "c1":
            n = 16384
            cl = npc.make_point_cloud(orc.gen_uniform_cube(n, 1.0, 1))
            l = Layer("conv", cl, cl, 1.8 * n ** (-1 / 3), 32, 32, 2, orc, npc.Math.auto)
            f = torch.from_numpy(orc.gen_features(n, 1, 32, 3)).cuda()
            out = torch.empty((n, 1, 32), device="cuda")
            cfg = npc.ExecConfig(math=npc.Math.auto)
            ms, prof = time_steps(lambda: npc.conv_forward(l.nb, l.w, f, cfg, out=out),
                                  a.steps, a.warmup)
            flop = 2 * l.nb.size * 32 * 32
            cfg16 = npc.ExecConfig(math=npc.Math.bf16)
            ms16, _ = time_steps(lambda: npc.conv_forward(l.nb, l.w, f, cfg16, out=out),
                                 a.steps, a.warmup)
            cfgx = npc.ExecConfig(math=npc.Math.exact)
            msx, _ = time_steps(lambda: npc.conv_forward(l.nb, l.w, f, cfgx, out=out), a.steps, a.warmup)
            r = {"config": "c1", "workload": "16K uniform, C=32, forward (default fp32 contract: the split "
                 "tensor-core path)",
                 "exact_engine": {"ms_per_step": round(msx, 4), "value": round(n / (msx / 1e3) / 1e6, 3)},
                 "value": round(n / (ms / 1e3) / 1e6, 3), "unit": "Mpoints/s",
                 "ms_per_step": round(ms, 4), "triplets": l.nb.size,
                 "fp32_gflops": round(flop / (ms / 1e3) / 1e9, 1),
                 "kernels_ms_per_step": {k: round(v[1] / a.steps, 4) for k, v in prof.items()},
                 "bf16_forced": {"ms_per_step": round(ms16, 4),
                                 "value": round(n / (ms16 / 1e3) / 1e6, 3),
                                 "note": "math=bf16: C=32 zero-padded to 64 on tcgen05"}}
        elif c == "c2":
            n = 100_000
            cl = npc.make_point_cloud(orc.gen_uniform_cube(n, 1.0, 1))
            layers = [Layer("conv", cl, cl, 1.8 * n ** (-1 / 3), 64, 64, 2, orc, auto)]
            f = torch.from_numpy(orc.gen_features(n, 1, 64, 3)).cuda()
            ms, prof = run_stack(layers, f, auto, a.steps, a.warmup)
            r = result("c2", "100K uniform, C=64, fwd+dgrad+wgrad", n, ms, prof, layers, bf16, {})
        elif c == "c3":
            n = 120_000
            xyz = gen_lidar_scan(n, 7)
            fine = npc.make_point_cloud(xyz)
            v, coarse = voxel_for_ratio(fine, 4.0)
            r_s = 1.8 * v
            layers = [Layer("strided", coarse, fine, r_s, 64, 128, 2, orc, auto)]
            f = torch.from_numpy(orc.gen_features(n, 1, 64, 3)).cuda()
            ms, prof = run_stack(layers, f, auto, a.steps, a.warmup)
            r = result("c3", "LiDAR-like 64-beam scan (seed 7), voxel_downsample ~4x, strided "
                       "64->128 two-cloud conv fwd+bwd; Mpoints/s over output points",
                       coarse.n_points(), ms, prof, layers, bf16,
                       {"n_in": n, "n_out": coarse.n_points(), "voxel": v, "radius": r_s})
        elif c == "c4":
            n = 1_000_000
            xyz, area = gen_indoor_fragment(n, 11)
            c0 = npc.make_point_cloud(xyz)
            rho = n / area
            r0 = (25.0 / (np.pi * rho)) ** 0.5  # ~25 neighbors on a surface
            v1, c1 = voxel_for_ratio(c0, 4.0)
            v2, c2 = voxel_for_ratio(c1, 4.0)
            r1, r2 = 2 * r0, 4 * r0
            layers = [Layer("enc0", c0, c0, r0, 64, 64, 20, orc, auto),
                      Layer("down1", c1, c0, r1, 64, 128, 21, orc, auto),
                      Layer("enc1", c1, c1, r1, 128, 128, 22, orc, auto),
                      Layer("down2", c2, c1, r2, 128, 256, 23, orc, auto),
                      Layer("enc2", c2, c2, r2, 256, 256, 24, orc, auto),
                      Layer("up1", c1, c2, r2, 256, 128, 25, orc, auto),
                      Layer("up0", c0, c1, r1, 128, 64, 26, orc, auto)]
            f = torch.from_numpy(orc.gen_features(n, 1, 64, 3)).cuda()
            ms, prof = run_stack(layers, f, auto, a.steps, a.warmup)
            r = result("c4", "1M-point indoor fragment (seed 11), 7-layer encoder/decoder "
                       "64-128-256-128-64, fwd+bwd; Mpoints/s over input points",
                       n, ms, prof, layers, bf16,
                       {"levels": [c0.n_points(), c1.n_points(), c2.n_points()],
                        "radii": [r0, r1, r2], "voxels": [v1, v2],
                        "per_layer": per_layer(layers, f, auto, a.steps)})
        else:
            raise SystemExit(f"unknown config {c}")
        r["setup_s"] = round(time.time() - t0, 2)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
