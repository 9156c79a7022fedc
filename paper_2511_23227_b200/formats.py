"""Wire / disk formats of the reference (io.hpp, io.cpp:30-151; triplets.hpp:84-93),
so recorded clouds and triplet lists replay identically on the reference (CPU)
and here (GPU).  Host-side byte layout only; clouds come back as GPU
PointClouds through make_point_cloud (its validation applies, as the
reference's read_* end in make_point_cloud).

  XYZ   ASCII "x y z" per line, 17 significant digits, '#' comments, one batch
  NPC1  "NPC1" | u32 N | u32 B | u32 0 | u32 offsets[B+1] | f64 xyz[N][3]
  TPL1  "TPL1" | u32 size | u32 n_out | u32 n_in | u32 n_kernels | u32 sort_axis
        | u32 i[size] | u32 j[size] | u32 k[size]
All little-endian.  Errors raise IOError_ (npc::IOError, errors.hpp)."""
from __future__ import annotations

import numpy as np
import torch

from . import npconv as npc

IOError_ = npc.NpcIOError
_U32 = np.dtype("<u4")
_F64 = np.dtype("<f8")


def _host_cloud(cloud):
    """(xyz (N, 3) float64, offsets) of a PointCloud or an (xyz, offsets) pair."""
    if isinstance(cloud, tuple):
        xyz, off = cloud
        xyz = np.asarray(xyz, dtype=np.float64).reshape(-1, 3)
        return xyz, np.asarray([0, len(xyz)] if off is None else off, dtype=np.int64)
    return cloud.xyz.detach().to("cpu", torch.float64).numpy().reshape(-1, 3), cloud.batch_offsets()


def write_xyz(path: str, cloud) -> None:
    """io.cpp:32-42: '%.17g %.17g %.17g' per point (doubles round-trip)."""
    xyz, _ = _host_cloud(cloud)
    try:
        with open(path, "w") as f:
            for x, y, z in xyz:
                f.write("%.17g %.17g %.17g\n" % (x, y, z))
    except OSError as e:
        raise IOError_(f"cannot open for writing: {path}") from e


def read_xyz_arrays(path: str):
    """io.cpp:44-60: blank lines and '#' comments skipped; one batch."""
    try:
        lines = open(path).read().split("\n")
    except OSError as e:
        raise IOError_(f"cannot open: {path}") from e
    pts = []
    for no, line in enumerate(lines, 1):
        if not line or line[0] == "#":
            continue
        parts = line.split()
        try:
            pts.append([float(parts[0]), float(parts[1]), float(parts[2])])
        except (IndexError, ValueError):
            raise IOError_(f"{path}:{no}: expected 'x y z'") from None
    xyz = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    return xyz, np.array([0, len(xyz)], dtype=np.int64)


def read_xyz(path: str) -> "npc.PointCloud":
    return npc.make_point_cloud(*read_xyz_arrays(path))


def write_npc(path: str, cloud) -> None:
    xyz, off = _host_cloud(cloud)
    head = np.array([len(xyz), len(off) - 1, 0], dtype=_U32)
    try:
        with open(path, "wb") as f:
            f.write(b"NPC1")
            f.write(head.tobytes())
            f.write(np.asarray(off, dtype=_U32).tobytes())
            f.write(np.ascontiguousarray(xyz, dtype=_F64).tobytes())
    except OSError as e:
        raise IOError_(f"cannot open for writing: {path}") from e


class _Reader:
    def __init__(self, path: str):
        self.path = path
        try:
            with open(path, "rb") as f:
                self.buf = f.read()
        except OSError as e:
            raise IOError_(f"cannot open: {path}") from e
        self.pos = 0

    def magic(self, m: bytes):
        if self.buf[:4] != m:
            raise IOError_(f"{self.path}: bad magic, expected {m.decode()}")
        self.pos = 4

    def u32(self, what: str) -> int:
        if self.pos + 4 > len(self.buf):
            raise IOError_(f"truncated {what}")
        v = int(np.frombuffer(self.buf, _U32, 1, self.pos)[0])
        self.pos += 4
        return v

    def array(self, dtype, count: int, what: str) -> np.ndarray:
        nbytes = count * dtype.itemsize
        if self.pos + nbytes > len(self.buf):
            raise IOError_(f"{self.path}: truncated {what}")
        a = np.frombuffer(self.buf, dtype, count, self.pos).copy()
        self.pos += nbytes
        return a


def read_npc_arrays(path: str):
    """io.cpp:76-93 -> (xyz, offsets)."""
    r = _Reader(path)
    r.magic(b"NPC1")
    n = r.u32("point count")
    b = r.u32("batch count")
    r.u32("reserved field")
    off = np.array([r.u32("batch offset") for _ in range(b + 1)], dtype=np.int64)
    xyz = r.array(_F64, 3 * n, "position block").reshape(-1, 3)
    return xyz, off


def read_npc(path: str) -> "npc.PointCloud":
    """read_npc_arrays + make_point_cloud (offset / finiteness validation)."""
    return npc.make_point_cloud(*read_npc_arrays(path))


def write_cloud(path: str, cloud) -> None:
    """io.cpp:95-100: '.xyz' text, anything else NPC1."""
    (write_xyz if path.endswith(".xyz") else write_npc)(path, cloud)


def read_cloud(path: str) -> "npc.PointCloud":
    return read_xyz(path) if path.endswith(".xyz") else read_npc(path)


def write_triplets(path: str, t) -> None:
    """io.cpp:108-125.  t: a TripletList or (i, j, k, n_out, n_in, n_kernels, axis)."""
    if isinstance(t, tuple):
        i, j, k, n_out, n_in, nk, axis = t
        arrs = [np.asarray(x).astype(_U32) for x in (i, j, k)]
        head = np.array([len(arrs[0]), n_out, n_in, nk, int(axis)], dtype=_U32)
    else:
        head = np.array([t.size(), t.n_out, t.n_in, t.n_kernels, int(t.sort_axis)], dtype=_U32)
        arrs = [x.detach().cpu().numpy().view(np.uint32).astype(_U32) for x in (t.i, t.j, t.k)]
    try:
        with open(path, "wb") as f:
            f.write(b"TPL1")
            f.write(head.tobytes())
            for a in arrs:
                f.write(a.tobytes())
    except OSError as e:
        raise IOError_(f"cannot open for writing: {path}") from e


def read_triplets_arrays(path: str):
    """io.cpp:127-151: declared ranges are checked for every triplet ->
    (i, j, k, n_out, n_in, n_kernels, sort_axis)."""
    r = _Reader(path)
    r.magic(b"TPL1")
    n = r.u32("triplet count")
    n_out, n_in, nk = r.u32("n_out"), r.u32("n_in"), r.u32("n_kernels")
    axis = r.u32("sort_axis")
    if axis > 3:
        raise IOError_(f"{path}: invalid sort_axis value")
    i, j, k = (r.array(_U32, n, "index array") for _ in range(3))
    if n and (int(i.max()) >= n_out or int(j.max()) >= n_in or int(k.max()) >= nk):
        raise IOError_(f"{path}: triplet index out of declared range")
    return i, j, k, n_out, n_in, nk, axis


def read_triplets(path: str, device=None) -> "npc.TripletList":
    return npc.TripletList.from_numpy(*read_triplets_arrays(path), device=device)
