"""Pins the CPU oracle (oracle/npc_oracle.c) before it is trusted as the checker:
against the reference's golden vectors / known answers (tests/golden/, produced by
the unmodified reference) and, when oracle/_ref is built, against the reference
itself on fresh seeded inputs.  CPU only."""
import numpy as np
import pytest


def test_rng_matches_reference_fixture(orc, golden):
    g = golden("rng.npz")
    assert np.array_equal(orc.mt_draws(5489, 64), g["draws"])
    assert np.array_equal(orc.gen_uniform_cube(8, 2.0, 7), g["cube"])
    assert np.array_equal(orc.gen_features(4, 1, 3, 9), g["feats"])
    assert np.array_equal(orc.make_weights(1, 1, 3, 2, 10), g["weights"])


def test_known_answers(orc, golden):
    h = golden("golden_hand.json")
    c = h["radius_collinear"]
    oi, ii = orc.radius_search(np.array(c["xyz"], float), np.array(c["xyz"], float), c["radius"])
    assert [[a, b] for a, b in zip(oi, ii)] == c["pairs"]
    cb = h["closed_ball"]
    assert len(orc.radius_search(np.array(cb["q"], float), np.array(cb["t"], float),
                                 cb["radius"])[0]) == cb["count"]
    bi = h["batch_isolation"]
    x = np.array(bi["xyz"], float)
    oi, ii = orc.radius_search(x, x, bi["radius"], bi["offsets"], bi["offsets"])
    assert [[a, b] for a, b in zip(oi, ii)] == bi["pairs"]
    for center, nbr, r, t, k in h["kernel_index"]["cases"]:
        assert orc.kernel_index(center, nbr, r, t) == k
    cn = h["collinear_native"]
    xyz = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    ti, tj, tk = orc.build_triplets(xyz, xyz, cn["radius"], cn["t"])
    assert len(ti) == cn["size"]
    assert tk[[n for n in range(len(ti)) if ti[n] == 1 and tj[n] == 0][0]] == cn["k_of_1_0"]
    s = h["sort_by_k"]
    oi, oj, ok = orc.sort_triplets(s["i"], s["j"], s["k"], 3, 3, 8, 3)
    assert list(ok) == s["sorted_k"] and list(oj) == s["sorted_j"]
    oi, oj, ok = orc.sort_triplets(s["stab_i"], [9] * 4, s["stab_k"], 3, 4, 10, 2)
    assert list(oi) == s["stab_sorted_i"]
    for n_out, n_in, nk, axis in h["choose_sort_axis"]["cases"]:
        assert orc.choose_sort_axis(n_out, n_in, nk) == axis


def test_error_codes(orc):
    x = np.zeros((1, 3))
    with pytest.raises(Exception):
        orc.radius_search(x, x, 0.0)
    assert orc.kernel_index([0, 0, 0], [0, 0, 0], 1.0, 2) == -3
    assert orc.kernel_index([0, 0, 0], [0, 0, 0], 0.0, 3) == -4


@pytest.mark.parametrize("name", ["geom_uniform_2000.npz", "geom_multibatch.npz"])
def test_triplets_match_golden(orc, golden, name):
    g = golden(name)
    off = g.get("offsets")
    ti, tj, tk = orc.build_triplets(g["xyz"], g["xyz"], float(g["radius"]), int(g["t"]), off, off)
    assert np.array_equal(ti, g["i"]) and np.array_equal(tj, g["j"]) and np.array_equal(tk, g["k"])
    if "bk_i" in g:
        n = len(g["xyz"])
        si, sj, sk = orc.sort_triplets(ti, tj, tk, 3, n, n, int(g["t"]) ** 3)
        assert np.array_equal(si, g["bk_i"]) and np.array_equal(sj, g["bk_j"])
        assert np.array_equal(sk, g["bk_k"])


def test_cross_query_matches_golden(orc, golden):
    g = golden("geom_cross.npz")
    oi, ii = orc.radius_search(g["queries"], g["targets"], float(g["radius"]))
    assert np.array_equal(oi, g["out_index"]) and np.array_equal(ii, g["in_index"])
    boi, bii = orc.brute_radius(g["queries"], g["targets"], float(g["radius"]))
    assert np.array_equal(boi, g["out_index"]) and np.array_equal(bii, g["in_index"])
    ti, tj, tk = orc.build_triplets(g["queries"], g["targets"], float(g["radius"]), 3)
    assert np.array_equal(tk, g["k"])


def test_dense_oracle_matches_golden(orc, golden):
    g = golden("conv_small.npz")
    fout, gin, gw = orc.dense_conv(g["w"], g["fin"], g["i"], g["j"], g["k"], len(g["xyz"]),
                                   g["gout"])
    # literal Eq. 1 in the same storage order: identical up to the last bit
    assert orc.rel_error(fout, g["fout"]) <= 1e-15
    assert orc.rel_error(gin, g["grad_in"]) <= 1e-15
    assert orc.rel_error(gw, g["grad_w"]) <= 1e-15
    # the reference fp32 engines sit within the reference's own 1e-5 bound
    assert orc.rel_error(g["mvmr_f32"], g["fout"]) <= 1e-5
    assert orc.rel_error(g["mvmr_t_f32"], g["grad_in"]) <= 1e-5
    assert orc.rel_error(g["vvor_f32"], g["grad_w"]) <= 1e-5


def test_voxel_downsample_matches_golden(orc, golden):
    g = golden("voxel_clusters.npz")
    kept, parent, koff = orc.voxel_downsample(g["xyz"], float(g["voxel"]), g["offsets"])
    assert np.array_equal(kept, g["kept"])
    assert np.array_equal(parent, g["parent"])
    assert np.array_equal(koff, g["kept_offsets"])


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_oracle_equals_reference_fresh(orc, ref, seed):
    n = 1500 + 250 * seed
    xyz = ref.gen_uniform_cube(n, 1.0, seed)
    r = 1.8 * n ** (-1 / 3)
    a = orc.build_triplets(xyz, xyz, r, 3)
    b = ref.build_triplets(xyz, xyz, r, 3, axis=0)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))
    # cross-cloud with t=5
    q = ref.gen_uniform_cube(n // 3, 1.0, seed + 100)
    a = orc.build_triplets(q, xyz, 1.3 * r, 5)
    b = ref.build_triplets(q, xyz, 1.3 * r, 5, axis=0)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))


def test_oracle_boundary_exactness(orc, ref):
    """Points on exact cell boundaries and at exactly the radius: the FMA recipe
    must reproduce the reference's accept/reject decisions."""
    v = 0.125
    g = np.stack(np.meshgrid(*[np.arange(6) * v] * 3, indexing="ij"), -1).reshape(-1, 3)
    for r in (v, 2 * v, np.sqrt(2) * v, np.sqrt(3) * v, 0.1, 0.3):
        a = orc.build_triplets(g, g, r, 3)
        b = ref.build_triplets(g, g, r, 3, axis=0)
        assert all(np.array_equal(p, q) for p, q in zip(a, b)), r


def test_degraded_known_answers(orc, golden):
    """test_triplets.cpp:154-215 through the C oracle."""
    h = golden("golden_hand.json")["degraded"]
    v = h["voxel"]
    c0, c1, c2, c3 = h["cases"]
    (ti, tj, tk), sn, kept, parent, so = orc.build_triplets_degraded(c0["xyz"], v, c0["t"])
    assert list(ti) == c0["i"] and list(tj) == c0["j"] and list(tk) == c0["k"]
    assert sn.tolist() == c0["snapped"]
    (ti, tj, tk), *_ = orc.build_triplets_degraded(c1["xyz"], v, c1["t"])
    assert sorted(tk.tolist()) == c1["k_multiset"]
    assert all(tk[n] > tk[n - 1] for n in range(1, len(ti)) if ti[n] == ti[n - 1])
    (ti, tj, tk), sn, kept, parent, so = orc.build_triplets_degraded(c2["xyz"], v, c2["t"])
    assert len(sn) == c2["n_sites"] and parent[0] == parent[1] != parent[2]
    (ti, tj, tk), *_ = orc.build_triplets_degraded(c3["xyz"], v, c3["t"])
    assert sorted(tk.tolist()) == c3["k_multiset"]
    with pytest.raises(Exception):
        orc.build_triplets_degraded([[0, 0, 0]], 0.0, 3)
    with pytest.raises(Exception):
        orc.build_triplets_degraded([[0, 0, 0]], 1.0, 4)


def test_degraded_matches_golden(orc, golden):
    g = golden("degraded_clusters.npz")
    for t in (3, 5):
        (ti, tj, tk), sn, kept, parent, so = orc.build_triplets_degraded(
            g["xyz"], float(g["voxel"]), t, g["offsets"])
        for got, key in ((ti, "i"), (tj, "j"), (tk, "k"), (sn, "snapped"), (kept, "kept"),
                         (parent, "parent"), (so, "site_offsets")):
            assert np.array_equal(got, g[f"t{t}_{key}"]), (t, key)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_degraded_oracle_vs_reference(orc, ref, seed):
    """The C restatement against the reference's build_triplets_degraded on
    fresh seeded clouds (uniform multi-batch with an empty batch, clusters)."""
    xyz = orc.gen_uniform_cube(2500, 1.0, seed)
    off = [0, 900, 900, 2500]
    for v, t in ((0.06, 3), (0.11, 1), (0.09, 5)):
        a = orc.build_triplets_degraded(xyz, v, t, off)
        b = ref.build_triplets_degraded(xyz, v, t, off)
        assert all(np.array_equal(x, y) for x, y in zip(a[0], b[0]))
        assert all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
    xyz = ref.gen_gaussian_clusters(3000, 10, 3.0, 0.2, seed + 10)
    a = orc.build_triplets_degraded(xyz, 0.05, 3)
    b = ref.build_triplets_degraded(xyz, 0.05, 3)
    assert all(np.array_equal(x, y) for x, y in zip(a[0], b[0]))
    assert all(np.array_equal(x, y) for x, y in zip(a[1:], b[1:]))
