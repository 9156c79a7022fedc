"""Replays a recorded triplet workload (TPL1, triplets.hpp:84-93) through the
GPU engines and, optionally, the reference's CPU engines (oracle/_ref), and
writes one CSV in the reference bench schema (npconv.cpp:290-304,
proj/README.md "Bench CSV schema") with a row per (kernel, executor,
repetition) plus the median row (repetition = -1).

    python tools/replay.py workload.tpl --c-in 64 --c-out 64 --reps 5 [--cpu] > rows.csv

GPU executors: `gpu_tc` (tcgen05 bf16-operand path; G = 1, C_in and C_out
multiples of 16 up to 256) and
`gpu_exact` (fp32 CUDA-core engines).  The access counters and closed-form
predictions of the reference's CPU executors have no GPU analogue and are
written as 0; aux_bytes is the library's peak scratch allocation."""
from __future__ import annotations

import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

HEADER = ("kernel,executor,sort_axis,L,b_out,b_in,repetition,triplets,groups,c_in,c_out,workers,"
          "deterministic,wall_time_ns,w_reads,fin_reads,fout_atomic_writes,aux_bytes,"
          "pred_naive,pred_grouped")
AXES = ["none", "by_i", "by_j", "by_k"]


def row(kernel, executor, axis, rep, n, cin, cout, workers, det, ns, aux):
    return (f"{kernel},{executor},{AXES[axis]},0,0,0,{rep},{n},1,{cin},{cout},{workers},"
            f"{int(det)},{int(ns)},0,0,0,{int(aux)},0,0")


def main():
    from oracle import Oracle
    from paper_2511_23227_b200 import formats as fm
    from paper_2511_23227_b200 import npconv as npc

    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--c-in", type=int, default=64)
    ap.add_argument("--c-out", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kernel", choices=["mvmr", "vvor", "both"], default="both")
    ap.add_argument("--cpu", action="store_true", help="also time the reference (oracle/_ref)")
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    if a.reps < 3:
        raise SystemExit("--reps must be >= 3 (median-of-repetitions timing)")

    i, j, k, n_out, n_in, nk, axis = fm.read_triplets_arrays(a.workload)
    n = len(i)
    t = round(nk ** (1 / 3))
    orc = Oracle()
    w = orc.make_weights(t, 1, a.c_in, a.c_out, a.seed)
    f = orc.gen_features(n_in, 1, a.c_in, a.seed + 1)
    g = orc.gen_features(n_out, 1, a.c_out, a.seed + 2)
    dev = torch.device("cuda", 0)
    tl = npc.TripletList.from_numpy(i, j, k, n_out, n_in, nk, axis, device=dev)
    W, F, G = (torch.from_numpy(x).to(dev) for x in (w, f, g))
    ctx = npc.context(dev)
    print(HEADER)
    kernels = ["mvmr", "vvor"] if a.kernel == "both" else [a.kernel]
    execs = [("gpu_exact", npc.Math.exact)]
    if all(c % 16 == 0 and 16 <= c <= 256 for c in (a.c_in, a.c_out)):
        execs.insert(0, ("gpu_tc", npc.Math.bf16))
    for kern in kernels:
        for name, math in execs:
            cfg = npc.ExecConfig(math=math, deterministic=True)
            run = (lambda: npc.mvmr(W, F, tl, n_out, cfg)) if kern == "mvmr" else \
                (lambda: npc.vvor(G, F, tl, nk, cfg))
            run()  # warm-up: builds and caches the plans
            torch.cuda.synchronize()
            times = []
            for rep in range(a.reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                run()
                e.record()
                torch.cuda.synchronize()
                times.append(s.elapsed_time(e) * 1e6)
                print(row(kern, name, axis, rep, n, a.c_in, a.c_out, 0, True, times[-1],
                          ctx.memory()[1]))
            print(row(kern, name, axis, -1, n, a.c_in, a.c_out, 0, True, statistics.median(times),
                      ctx.memory()[1]))
        if a.cpu:
            from oracle import Reference
            import time
            r = Reference()
            workers = r.hardware_concurrency()
            times = []
            for rep in range(a.reps):
                t0 = time.perf_counter_ns()
                if kern == "mvmr":
                    r.mvmr(w, f, i, j, k, n_out, grouped=1, det=0, workers=workers)
                else:
                    r.vvor(g, f, i, j, k, nk, grouped=1, det=0, workers=workers)
                times.append(time.perf_counter_ns() - t0)
                print(row(kern, "cpu_grouped", axis, rep, n, a.c_in, a.c_out, workers, False,
                          times[-1], 0))
            print(row(kern, "cpu_grouped", axis, -1, n, a.c_in, a.c_out, workers, False,
                      statistics.median(times), 0))


if __name__ == "__main__":
    main()
