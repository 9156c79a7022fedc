"""Wire / disk formats (io.hpp, io.cpp:30-151; triplets.hpp:84-93; SURVEY.md
§8(f) next #4): files written here are read back bit-exactly by the
reference's own readers and vice versa; error behaviour follows io.cpp."""
import os

import numpy as np
import pytest

from paper_2511_23227_b200 import formats as fm


def _cloud(orc):
    xyz = orc.gen_uniform_cube(777, 3.0, 5) - 1.0
    return xyz, np.array([0, 300, 300, 777], dtype=np.int64)


def test_npc_roundtrip_and_reference(tmp_path, orc, ref):
    xyz, off = _cloud(orc)
    p1, p2 = str(tmp_path / "a.npc"), str(tmp_path / "b.npc")
    fm.write_npc(p1, (xyz, off))
    rx, ro = fm.read_npc_arrays(p1)
    assert np.array_equal(rx, xyz) and np.array_equal(ro, off)
    gx, go = ref.read_cloud(p1)                        # reference reads our file
    assert np.array_equal(gx, xyz) and np.array_equal(go, off)
    ref.write_cloud(p2, xyz, off)                      # and we read the reference's
    assert open(p1, "rb").read() == open(p2, "rb").read()


def test_xyz_roundtrip_and_reference(tmp_path, orc, ref):
    xyz, _ = _cloud(orc)
    xyz[0] = [1e-300, -0.1, 3.0000000000000004]
    p1, p2 = str(tmp_path / "a.xyz"), str(tmp_path / "b.xyz")
    fm.write_cloud(p1, (xyz, None))
    ref.write_cloud(p2, xyz)
    assert open(p1).read() == open(p2).read()           # same 17-digit text
    rx, ro = fm.read_xyz_arrays(p2)
    assert np.array_equal(rx, xyz) and list(ro) == [0, len(xyz)]
    with open(p1, "a") as f:
        f.write("# comment\n\n1 2 3\n")
    rx, _ = fm.read_xyz_arrays(p1)
    gx, _ = ref.read_cloud(p1)
    assert np.array_equal(rx, gx) and len(rx) == len(xyz) + 1


def test_triplets_roundtrip_and_reference(tmp_path, orc, ref):
    xyz = orc.gen_uniform_cube(1500, 1.0, 3)
    ti, tj, tk = orc.build_triplets(xyz, xyz, 0.12, 3)
    si, sj, sk = orc.sort_triplets(ti, tj, tk, 3, 1500, 1500, 27)
    p1, p2 = str(tmp_path / "a.tpl"), str(tmp_path / "b.tpl")
    fm.write_triplets(p1, (si, sj, sk, 1500, 1500, 27, 3))
    got = ref.read_triplets(p1)
    assert all(np.array_equal(a, b) for a, b in zip(got[:3], (si, sj, sk)))
    assert got[3:] == (1500, 1500, 27, 3)
    ref.write_triplets(p2, si, sj, sk, 1500, 1500, 27, 3)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    r = fm.read_triplets_arrays(p2)
    assert all(np.array_equal(a, b) for a, b in zip(r[:3], (si, sj, sk))) and r[3:] == (1500, 1500, 27, 3)


def test_errors_match_reference(tmp_path, ref):
    bad = str(tmp_path / "bad.npc")
    open(bad, "wb").write(b"NPC2" + bytes(12))
    with pytest.raises(fm.IOError_, match="bad magic"):
        fm.read_npc_arrays(bad)
    with pytest.raises(Exception):
        ref.read_cloud(bad)
    trunc = str(tmp_path / "t.npc")
    fm.write_npc(trunc, (np.zeros((4, 3)), None))
    open(trunc, "ab").truncate(os.path.getsize(trunc) - 8)
    with pytest.raises(fm.IOError_, match="truncated position block"):
        fm.read_npc_arrays(trunc)
    rng = str(tmp_path / "r.tpl")
    fm.write_triplets(rng, (np.array([0, 5]), np.array([0, 1]), np.array([0, 2]), 5, 5, 27, 0))
    with pytest.raises(fm.IOError_, match="out of declared range"):
        fm.read_triplets_arrays(rng)
    with pytest.raises(Exception):
        ref.read_triplets(rng)
    ax = str(tmp_path / "ax.tpl")
    fm.write_triplets(ax, (np.array([0]), np.array([0]), np.array([0]), 1, 1, 1, 7))
    with pytest.raises(fm.IOError_, match="invalid sort_axis"):
        fm.read_triplets_arrays(ax)
    txt = str(tmp_path / "bad.xyz")
    open(txt, "w").write("1 2 3\n1 2\n")
    with pytest.raises(fm.IOError_, match=":2: expected"):
        fm.read_xyz_arrays(txt)
    with pytest.raises(fm.IOError_, match="cannot open"):
        fm.read_npc_arrays(str(tmp_path / "missing.npc"))


@pytest.mark.gpu
def test_gpu_roundtrip_and_replay(tmp_path, npc, orc, ref):
    """A cloud read from NPC1 builds the same triplets on the GPU as the
    reference reading the same file; the TPL1 written from the GPU build
    replays through tools/replay.py into the reference CSV schema."""
    import subprocess
    import sys
    xyz, off = _cloud(orc)
    p = str(tmp_path / "c.npc")
    ref.write_cloud(p, xyz, off)
    cl = fm.read_npc(p)
    tl = npc.build_triplets_native(cl, cl, npc.ConvGeometry(radius=0.35, t=3))
    rx, ro = ref.read_cloud(p)
    ti, tj, tk = ref.build_triplets(rx, rx, 0.35, 3, out_off=ro, in_off=ro)
    got = [x.cpu().numpy().view(np.uint32) for x in (tl.i, tl.j, tl.k)]
    assert all(np.array_equal(a, b) for a, b in zip(got, (ti, tj, tk)))
    tp = str(tmp_path / "w.tpl")
    fm.write_triplets(tp, npc.sort_triplets(tl, npc.SortAxis.by_k))
    back = fm.read_triplets(tp)
    assert torch_equal(back, npc.sort_triplets(tl, npc.SortAxis.by_k))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "replay.py"), tp, "--reps", "3",
                        "--cpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("kernel,executor,sort_axis,L,b_out,b_in,repetition")
    rows = [ln.split(",") for ln in lines[1:]]
    assert all(len(x) == 20 for x in rows)
    assert {x[1] for x in rows} == {"gpu_tc", "gpu_exact", "cpu_grouped"}
    assert sum(1 for x in rows if x[6] == "-1") == 6


def torch_equal(a, b):
    return all(bool((x == y).all()) for x, y in zip((a.i, a.j, a.k), (b.i, b.j, b.k))) and \
        (a.n_out, a.n_in, a.n_kernels, int(a.sort_axis)) == (b.n_out, b.n_in, b.n_kernels,
                                                             int(b.sort_axis))
