"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libnpref.so, built from
/root/reference by `make -f oracle/Makefile`):

    python tests/golden/make_golden.py

Every array in the fixtures is an output of the reference's own public API
(build_triplets_native, sort_triplets, radius_search, dense_conv_oracle,
mvmr/mvmr_transposed/vvor, voxel_downsample) on the stated seeded inputs, so
the fixtures pin parity on the GPU box where /root/reference does not exist.
The hand-computed known answers (golden_hand.json) are transcribed from the
reference tests with their file:line.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402


def main():
    r = Reference()
    out = {}

    # 1. uniform cube, self-convolution, t=3 (test_triplets / acceptance criterion 7 style)
    n = 2000
    xyz = r.gen_uniform_cube(n, 1.0, 11)
    rad = 1.8 * n ** (-1.0 / 3.0)
    tn = r.build_triplets(xyz, xyz, rad, 3, axis=0)
    tk = r.build_triplets(xyz, xyz, rad, 3, axis=3)
    np.savez_compressed(os.path.join(HERE, "geom_uniform_2000.npz"), xyz=xyz, radius=rad, t=3,
                        i=tn[0], j=tn[1], k=tn[2], bk_i=tk[0], bk_j=tk[1], bk_k=tk[2])
    out["geom_uniform_2000"] = int(len(tn[0]))

    # 2. multi-batch with an empty batch, t=5
    xyz2 = r.gen_uniform_cube(600, 3.0, 34)
    off2 = np.array([0, 150, 150, 400, 600], dtype=np.int64)
    t2 = r.build_triplets(xyz2, xyz2, 0.6, 5, axis=0, out_off=off2, in_off=off2)
    np.savez_compressed(os.path.join(HERE, "geom_multibatch.npz"), xyz=xyz2, offsets=off2,
                        radius=0.6, t=5, i=t2[0], j=t2[1], k=t2[2])
    out["geom_multibatch"] = int(len(t2[0]))

    # 3. cross query: gaussian clusters targets, uniform queries (test_spatial.cpp:112-116)
    tgt = r.gen_gaussian_clusters(300, 5, 6.0, 0.4, 32)
    qry = r.gen_uniform_cube(150, 6.0, 33)
    oi, ii = r.radius_search(qry, tgt, 0.9)
    t3 = r.build_triplets(qry, tgt, 0.9, 3, axis=0)
    np.savez_compressed(os.path.join(HERE, "geom_cross.npz"), queries=qry, targets=tgt,
                        radius=0.9, out_index=oi, in_index=ii, i=t3[0], j=t3[1], k=t3[2])
    out["geom_cross"] = int(len(oi))

    # 4. conv values: G=2, C_in=8, C_out=12, t=3 on a 300-point cloud
    n4 = 300
    xyz4 = r.gen_uniform_cube(n4, 1.0, 41)
    rad4 = 1.8 * n4 ** (-1.0 / 3.0)
    ti, tj, tk4 = r.build_triplets(xyz4, xyz4, rad4, 3, axis=3)
    w = r.make_weights(3, 2, 8, 12, 42, dtype=np.float64)
    fin = r.gen_features(n4, 2, 8, 43, dtype=np.float64)
    gout = r.gen_features(n4, 2, 12, 44, dtype=np.float64)
    fout, gin, gw = r.dense_conv(w, fin, ti, tj, tk4, n4, gout)
    w32 = w.astype(np.float32)
    f32 = fin.astype(np.float32)
    g32 = gout.astype(np.float32)
    m32 = r.mvmr(w32, f32, ti, tj, tk4, n4)
    mt32 = r.mvmr_transposed(w32, g32, ti, tj, tk4, n4)
    v32 = r.vvor(g32, f32, ti, tj, tk4, 27)
    np.savez_compressed(os.path.join(HERE, "conv_small.npz"), xyz=xyz4, radius=rad4, i=ti, j=tj,
                        k=tk4, w=w, fin=fin, gout=gout, fout=fout, grad_in=gin, grad_w=gw,
                        mvmr_f32=m32, mvmr_t_f32=mt32, vvor_f32=v32)
    out["conv_small"] = int(len(ti))

    # 5. voxel downsample (spatial.cpp:94-152) on a clustered cloud with 2 batches
    xyz5 = r.gen_gaussian_clusters(500, 6, 5.0, 0.3, 103)
    off5 = np.array([0, 220, 500], dtype=np.int64)
    kept, parent, koff = r.voxel_downsample(xyz5, 0.45, off5)
    np.savez_compressed(os.path.join(HERE, "voxel_clusters.npz"), xyz=xyz5, offsets=off5,
                        voxel=0.45, kept=kept, parent=parent, kept_offsets=koff)
    out["voxel_clusters"] = int(len(kept))

    # 5b. degraded (voxel) build (triplets.cpp:78-133): clustered 3-batch cloud
    #     (middle batch empty), t = 3 and t = 5, build order + sites
    xyz6 = r.gen_gaussian_clusters(900, 8, 4.0, 0.35, 104)
    off6 = np.array([0, 400, 400, 900], dtype=np.int64)
    deg = {"xyz": xyz6, "offsets": off6, "voxel": 0.3}
    for t in (3, 5):
        (ti, tj, tk), snapped, kept, parent, soff = r.build_triplets_degraded(xyz6, 0.3, t, off6)
        deg.update({f"t{t}_i": ti, f"t{t}_j": tj, f"t{t}_k": tk, f"t{t}_snapped": snapped,
                    f"t{t}_kept": kept, f"t{t}_parent": parent, f"t{t}_site_offsets": soff})
        out[f"degraded_t{t}"] = int(len(ti))
    np.savez_compressed(os.path.join(HERE, "degraded_clusters.npz"), **deg)

    # 6. mt19937_64 draws + generators (random.hpp / synthetic.cpp)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), draws=r.mt_draws(5489, 64),
                        cube=r.gen_uniform_cube(8, 2.0, 7),
                        feats=r.gen_features(4, 1, 3, 9),
                        weights=r.make_weights(1, 1, 3, 2, 10))

    hand = {
        "source": "reference tests, transcribed (see each entry)",
        "radius_collinear": {"ref": "test_spatial.cpp:39-53", "xyz": [[0, 0, 0], [1, 0, 0], [2, 0, 0]],
                             "radius": 1.5,
                             "pairs": [[0, 0], [0, 1], [1, 0], [1, 1], [1, 2], [2, 1], [2, 2]]},
        "closed_ball": {"ref": "test_spatial.cpp:70-74", "q": [[0, 0, 0]], "t": [[1, 0, 0]],
                        "radius": 1.0, "count": 1},
        "batch_isolation": {"ref": "test_spatial.cpp:96-103",
                            "xyz": [[0, 0, 0], [0.5, 0, 0], [0, 0, 0], [0.5, 0, 0]],
                            "offsets": [0, 2, 4], "radius": 1.0,
                            "pairs": [[0, 0], [0, 1], [1, 0], [1, 1], [2, 2], [2, 3], [3, 2], [3, 3]]},
        "kernel_index": {"ref": "test_triplets.cpp:45-69", "cases": [
            [[0, 0, 0], [0, 0, 0], 1.0, 3, 13],
            [[5, -2, 7], [5, -2, 7], 0.25, 3, 13],
            [[0, 0, 0], [0, 0, 0], 1.0, 5, 62],
            [[0, 0, 0], [0.4, 0, 0], 0.6, 3, 22],
            [[0, 0, 0], [1.0, 0, 0], 1.0, 3, 22],
            [[0, 0, 0], [1.0, 1.0, 1.0], 1.0, 3, 26],
            [[0, 0, 0], [-1.0, -1.0, -1.0], 1.0, 3, 0],
            [[0, 0, 0], [0.9, -0.3, 0.2], 1.0, 1, 0]]},
        "collinear_native": {"ref": "test_triplets.cpp:89-101", "radius": 1.5, "t": 3,
                             "size": 7, "k_of_1_0": 4},
        "sort_by_k": {"ref": "test_triplets.cpp:218-258", "i": [2, 0, 1], "j": [5, 6, 7],
                      "k": [2, 0, 1], "sorted_k": [0, 1, 2], "sorted_j": [6, 7, 5],
                      "stab_i": [0, 1, 2, 3], "stab_k": [1, 0, 1, 0], "stab_sorted_i": [1, 3, 0, 2]},
        "choose_sort_axis": {"ref": "test_triplets.cpp:273-293", "cases": [
            [100000, 100000, 27, 3], [10, 100000, 27, 1], [100000, 5, 27, 2], [27, 27, 27, 3]]},
        "mvmr_identity": {"ref": "test_engine.cpp:75-87", "out": [3.0, 4.0]},
        "mvmr_reduce": {"ref": "test_engine.cpp:89-101", "out": [4.0, 6.0]},
        "dgrad": {"ref": "test_engine.cpp:103-115", "w": [1.0, 3.0, 2.0, 4.0], "out": [4.0, 6.0]},
        "degraded": {"ref": "test_triplets.cpp:154-215", "voxel": 1.0, "cases": [
            {"xyz": [[0.25, 0.25, 0.25]], "t": 3, "i": [0], "j": [0], "k": [13],
             "snapped": [[0.5, 0.5, 0.5]]},
            {"xyz": [[0.5, 0.5, 0.5], [1.5, 0.5, 0.5]], "t": 3, "k_multiset": [4, 13, 13, 22]},
            {"xyz": [[0.2, 0.2, 0.2], [0.8, 0.8, 0.8], [5, 5, 5]], "t": 3, "n_sites": 2},
            {"xyz": [[0.5, 0.5, 0.5], [2.5, 0.5, 0.5]], "t": 5, "k_multiset": [12, 62, 62, 112],
             "n_kernels": 125}]},
        "counts": out,
    }
    with open(os.path.join(HERE, "golden_hand.json"), "w") as f:
        json.dump(hand, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
