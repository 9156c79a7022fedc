"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

See ``oracle/__init__.py``.  All arrays are numpy; clouds are ``(N, 3)`` float64
positions plus int64 batch offsets ``[0, ..., N]``; triplets are three uint32
arrays in struct-of-arrays layout (reference ``triplets.hpp:20-30``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_D = C.c_double
_INT = C.c_int


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _offsets(n, offsets):
    if offsets is None:
        return np.array([0, n], dtype=np.int64)
    return np.ascontiguousarray(offsets, dtype=np.int64)


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing -- run `make -f oracle/Makefile`")
    return C.CDLL(path)


class Oracle:
    """The C restatement (oracle/npc_oracle.c)."""

    def __init__(self, path: str | None = None):
        self.lib = lib = _load(path or os.path.join(_HERE, "liboracle.so"))
        lib.orc_radius_search.restype = _INT
        lib.orc_brute_radius.restype = _INT
        lib.orc_pairs_size.restype = _I64
        lib.orc_kernel_index.restype = _I64
        lib.orc_build_triplets.restype = _INT
        lib.orc_triplets_size.restype = _I64
        lib.orc_choose_sort_axis.restype = _INT
        lib.orc_dense_conv.restype = _INT
        lib.orc_rel_error_f64.restype = _D
        lib.orc_rel_error_f32.restype = _D
        lib.orc_voxel_downsample.restype = _I64
        for name in ("orc_gen_uniform_cube",):
            getattr(lib, name).argtypes = [_I64, _D, _U64, _P]
        lib.orc_gen_features_f32.argtypes = [_I64, _U64, _P]
        lib.orc_gen_features_f64.argtypes = [_I64, _U64, _P]
        lib.orc_make_weights_f32.argtypes = [_I64, _I64, _I64, _I64, _U64, _P]
        lib.orc_make_weights_f64.argtypes = [_I64, _I64, _I64, _I64, _U64, _P]
        lib.orc_mt19937_64_draws.argtypes = [_U64, _I64, _P]
        search_args = [_P, _P, _I64, _P, _P, _I64, _D, C.POINTER(_P)]
        lib.orc_radius_search.argtypes = search_args
        lib.orc_brute_radius.argtypes = search_args
        lib.orc_pairs_size.argtypes = [_P]
        lib.orc_pairs_copy.argtypes = [_P, _P, _P]
        lib.orc_pairs_free.argtypes = [_P]
        lib.orc_kernel_index.argtypes = [_P, _P, _D, _I64]
        lib.orc_build_triplets.argtypes = [_P, _P, _I64, _P, _P, _I64, _D, _I64, C.POINTER(_P)]
        lib.orc_triplets_size.argtypes = [_P]
        lib.orc_triplets_copy.argtypes = [_P, _P, _P, _P]
        lib.orc_triplets_free.argtypes = [_P]
        lib.orc_sort_triplets.argtypes = [_P, _P, _P, _I64, _INT, _I64, _I64, _I64, _P, _P, _P]
        lib.orc_choose_sort_axis.argtypes = [_I64, _I64, _I64]
        lib.orc_dense_conv.argtypes = [_P, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _P, _I64,
                                       _I64, _P, _P, _P, _P]
        lib.orc_rel_error_f64.argtypes = [_P, _P, _I64, _D]
        lib.orc_rel_error_f32.argtypes = [_P, _P, _I64, _D]
        lib.orc_voxel_downsample.argtypes = [_P, _P, _I64, _D, _P, _P, _P]
        lib.orc_build_triplets_degraded.restype = _I64
        lib.orc_build_triplets_degraded.argtypes = [_P, _P, _I64, _D, _I64, _P, _P, _P, _P,
                                                    C.POINTER(_P)]

    # -- generators (random.hpp / synthetic.cpp / tensors.hpp) --------------
    def mt_draws(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self.lib.orc_mt19937_64_draws(seed, n, _ptr(out))
        return out

    def gen_uniform_cube(self, n: int, extent: float, seed: int) -> np.ndarray:
        out = np.empty((n, 3), dtype=np.float64)
        self.lib.orc_gen_uniform_cube(n, extent, seed, _ptr(out))
        return out

    def gen_features(self, n, g, c, seed, dtype=np.float32) -> np.ndarray:
        out = np.empty((n, g, c), dtype=dtype)
        fn = self.lib.orc_gen_features_f32 if dtype == np.float32 else self.lib.orc_gen_features_f64
        fn(n * g * c, seed, _ptr(out))
        return out

    def make_weights(self, t, g, cin, cout, seed, dtype=np.float32) -> np.ndarray:
        out = np.empty((t ** 3, g, cin, cout), dtype=dtype)
        fn = self.lib.orc_make_weights_f32 if dtype == np.float32 else self.lib.orc_make_weights_f64
        fn(t, g, cin, cout, seed, _ptr(out))
        return out

    # -- geometry (spatial.cpp / triplets.cpp) ------------------------------
    def _pairs(self, fn, q, q_off, t, t_off, radius):
        q = _f64(q).reshape(-1, 3)
        t = _f64(t).reshape(-1, 3)
        qo, to = _offsets(len(q), q_off), _offsets(len(t), t_off)
        h = _P()
        rc = fn(_ptr(q), _ptr(qo), len(qo) - 1, _ptr(t), _ptr(to), len(to) - 1, radius, C.byref(h))
        if rc:
            raise OracleError(rc, "radius_search")
        n = self.lib.orc_pairs_size(h)
        oi = np.empty(n, dtype=np.int64)
        ii = np.empty(n, dtype=np.int64)
        self.lib.orc_pairs_copy(h, _ptr(oi), _ptr(ii))
        self.lib.orc_pairs_free(h)
        return oi, ii

    def radius_search(self, q, t, radius, q_off=None, t_off=None):
        return self._pairs(self.lib.orc_radius_search, q, q_off, t, t_off, radius)

    def brute_radius(self, q, t, radius, q_off=None, t_off=None):
        return self._pairs(self.lib.orc_brute_radius, q, q_off, t, t_off, radius)

    def kernel_index(self, center, neighbor, radius, t) -> int:
        c = _f64(center)
        nb = _f64(neighbor)
        return int(self.lib.orc_kernel_index(_ptr(c), _ptr(nb), radius, t))

    def build_triplets(self, out_xyz, in_xyz, radius, t, out_off=None, in_off=None):
        o = _f64(out_xyz).reshape(-1, 3)
        i = _f64(in_xyz).reshape(-1, 3)
        oo, io = _offsets(len(o), out_off), _offsets(len(i), in_off)
        h = _P()
        rc = self.lib.orc_build_triplets(_ptr(o), _ptr(oo), len(oo) - 1, _ptr(i), _ptr(io),
                                         len(io) - 1, radius, t, C.byref(h))
        if rc:
            raise OracleError(rc, "build_triplets_native")
        n = self.lib.orc_triplets_size(h)
        ti, tj, tk = (np.empty(n, dtype=np.uint32) for _ in range(3))
        self.lib.orc_triplets_copy(h, _ptr(ti), _ptr(tj), _ptr(tk))
        self.lib.orc_triplets_free(h)
        return ti, tj, tk

    def sort_triplets(self, ti, tj, tk, axis, n_out, n_in, n_kernels):
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        oi, oj, ok = (np.empty_like(ti) for _ in range(3))
        self.lib.orc_sort_triplets(_ptr(ti), _ptr(tj), _ptr(tk), len(ti), axis, n_out, n_in,
                                   n_kernels, _ptr(oi), _ptr(oj), _ptr(ok))
        return oi, oj, ok

    def choose_sort_axis(self, n_out, n_in, n_kernels) -> int:
        return int(self.lib.orc_choose_sort_axis(n_out, n_in, n_kernels))

    # -- dense oracle (oracle.cpp:12-67) -------------------------------------
    def dense_conv(self, w, fin, ti, tj, tk, n_out, gout=None):
        """fp64 literal Eq. 1.  w (K,G,Cin,Cout), fin (N_in,G,Cin), gout (N_out,G,Cout).
        Returns (fout, grad_in, grad_w[(K,G,Cout,Cin)]) -- the last two None without gout."""
        w = _f64(w)
        K, G, cin, cout = w.shape
        fin = _f64(fin).reshape(-1, G, cin)
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        fout = np.zeros((n_out, G, cout))
        gin = gw = None
        if gout is not None:
            gout = _f64(gout).reshape(n_out, G, cout)
            gin = np.zeros_like(fin)
            gw = np.zeros((K, G, cout, cin))
        rc = self.lib.orc_dense_conv(_ptr(w), K, G, cin, cout, _ptr(fin), len(fin), _ptr(ti),
                                     _ptr(tj), _ptr(tk), len(ti), n_out, _ptr(gout), _ptr(fout),
                                     _ptr(gin), _ptr(gw))
        if rc:
            raise OracleError(rc, "dense_conv_oracle")
        return fout, gin, gw

    @staticmethod
    def rel_error(a, b, floor=1e-30) -> float:
        """gradcheck.cpp:11-31: max|a-b| / max(max|b|, floor)."""
        a = np.asarray(a, dtype=np.float64).ravel()
        b = np.asarray(b, dtype=np.float64).ravel()
        if a.size == 0:
            return 0.0
        return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), floor))

    def voxel_downsample(self, xyz, voxel, offsets=None):
        xyz = _f64(xyz).reshape(-1, 3)
        off = _offsets(len(xyz), offsets)
        kept = np.empty(len(xyz), dtype=np.int64)
        parent = np.empty(len(xyz), dtype=np.int64)
        out_off = np.empty(len(off), dtype=np.int64)
        m = self.lib.orc_voxel_downsample(_ptr(xyz), _ptr(off), len(off) - 1, voxel, _ptr(kept),
                                          _ptr(parent), _ptr(out_off))
        if m < 0:
            raise OracleError(-m, "voxel_downsample")
        return kept[:m].copy(), parent, out_off

    def build_triplets_degraded(self, xyz, voxel, t, offsets=None):
        """triplets.cpp:78-133: ((i, j, k) in build order, snapped xyz, kept, parent, site offsets)."""
        return _degraded(self.lib, "orc_build_triplets_degraded", "orc", xyz, voxel, t, offsets)


def _degraded(lib, fn, pfx, xyz, voxel, t, offsets):
    xyz = _f64(xyz).reshape(-1, 3)
    off = _offsets(len(xyz), offsets)
    n = len(xyz)
    snapped = np.empty((max(n, 1), 3), dtype=np.float64)
    kept = np.empty(max(n, 1), dtype=np.int64)
    parent = np.empty(max(n, 1), dtype=np.int64)
    site_off = np.empty(len(off), dtype=np.int64)
    h = _P()
    m = getattr(lib, fn)(_ptr(xyz), _ptr(off), len(off) - 1, voxel, t, _ptr(snapped), _ptr(kept),
                         _ptr(parent), _ptr(site_off), C.byref(h))
    if m < 0:
        raise OracleError(-m, "build_triplets_degraded")
    size = getattr(lib, pfx + "_triplets_size")(h)
    ti, tj, tk = (np.empty(size, dtype=np.uint32) for _ in range(3))
    getattr(lib, pfx + "_triplets_copy")(h, _ptr(ti), _ptr(tj), _ptr(tk))
    getattr(lib, pfx + "_triplets_free")(h)
    return (ti, tj, tk), snapped[:m].copy(), kept[:m].copy(), parent[:n].copy(), site_off


def reference_available(path: str | None = None) -> bool:
    return os.path.exists(path or os.path.join(_HERE, "_ref", "libnpref.so"))


class Reference:
    """The unmodified reference core (oracle/_ref/libnpref.so)."""

    def __init__(self, path: str | None = None):
        self.lib = lib = _load(path or os.path.join(_HERE, "_ref", "libnpref.so"))
        lib.ref_mt19937_64_draws.argtypes = [_U64, _I64, _P]
        lib.ref_gen_uniform_cube.argtypes = [_I64, _D, _U64, _P]
        lib.ref_gen_uniform_cube.restype = _INT
        lib.ref_gen_gaussian_clusters.argtypes = [_I64, _I64, _D, _D, _U64, _P]
        lib.ref_gen_gaussian_clusters.restype = _INT
        lib.ref_gen_grid_snapped.argtypes = [_I64, _I64, _D, _U64, _P]
        lib.ref_gen_grid_snapped.restype = _INT
        for s in ("f32", "f64"):
            getattr(lib, f"ref_gen_features_{s}").argtypes = [_I64, _I64, _I64, _U64, _P]
            getattr(lib, f"ref_make_weights_{s}").argtypes = [_I64, _I64, _I64, _I64, _U64, _P]
            getattr(lib, f"ref_mvmr_{s}").argtypes = [_P, _I64, _I64, _I64, _I64, _P, _I64, _P, _P,
                                                      _P, _I64, _I64, _I64, _I64, _INT, _INT, _I64,
                                                      _INT, _P]
            getattr(lib, f"ref_mvmr_transposed_{s}").argtypes = getattr(lib, f"ref_mvmr_{s}").argtypes
            getattr(lib, f"ref_vvor_{s}").argtypes = [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P,
                                                      _P, _I64, _I64, _I64, _I64, _INT, _INT, _I64,
                                                      _INT, _P]
            getattr(lib, f"ref_upsample_{s}").argtypes = [_P, _P, _I64, _P, _I64, _P, _P, _I64, _I64,
                                                          _P]
        search_args = [_P, _P, _I64, _P, _P, _I64, _D, C.POINTER(_P)]
        lib.ref_radius_search.argtypes = search_args
        lib.ref_brute_radius.argtypes = search_args
        lib.ref_pairs_size.argtypes = [_P]
        lib.ref_pairs_size.restype = _I64
        lib.ref_pairs_copy.argtypes = [_P, _P, _P]
        lib.ref_pairs_free.argtypes = [_P]
        lib.ref_kernel_index.argtypes = [_P, _P, _D, _I64]
        lib.ref_kernel_index.restype = _I64
        lib.ref_build_triplets.argtypes = [_P, _P, _I64, _P, _P, _I64, _D, _I64, _INT, C.POINTER(_P)]
        lib.ref_triplets_size.argtypes = [_P]
        lib.ref_triplets_size.restype = _I64
        lib.ref_triplets_axis.argtypes = [_P]
        lib.ref_triplets_copy.argtypes = [_P, _P, _P, _P]
        lib.ref_triplets_free.argtypes = [_P]
        lib.ref_sort_triplets.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I64, _INT, _P, _P, _P]
        lib.ref_dense_oracle.argtypes = [_P, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _P, _I64,
                                         _I64, _I64, _I64, _P, _P, _P, _P]
        lib.ref_voxel_downsample.argtypes = [_P, _P, _I64, _D, _P, _P, _P]
        lib.ref_voxel_downsample.restype = _I64
        lib.ref_build_triplets_degraded.argtypes = [_P, _P, _I64, _D, _I64, _P, _P, _P, _P,
                                                    C.POINTER(_P)]
        lib.ref_build_triplets_degraded.restype = _I64
        lib.ref_write_cloud.argtypes = [C.c_char_p, _P, _P, _I64]
        lib.ref_write_cloud.restype = _INT
        lib.ref_read_cloud.argtypes = [C.c_char_p, _P, _P, C.POINTER(_I64)]
        lib.ref_read_cloud.restype = _I64
        lib.ref_write_triplets.argtypes = [C.c_char_p, _P, _P, _P, _I64, _I64, _I64, _I64, _INT]
        lib.ref_write_triplets.restype = _INT
        lib.ref_read_triplets.argtypes = [C.c_char_p, _P, _P, _P, _P]
        lib.ref_read_triplets.restype = _INT
        lib.ref_conv_layer_f32.argtypes = [_P, _I64, _D, _I64, _I64, _I64, _P, _P, _P, _INT, _INT,
                                           _P, _P, _P, _P, C.POINTER(_P)]
        lib.ref_conv_cache_free.argtypes = [_P]
        lib.ref_hardware_concurrency.restype = _INT

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def mt_draws(self, seed, n):
        out = np.empty(n, dtype=np.uint64)
        self.lib.ref_mt19937_64_draws(seed, n, _ptr(out))
        return out

    def gen_uniform_cube(self, n, extent, seed):
        out = np.empty((n, 3), dtype=np.float64)
        rc = self.lib.ref_gen_uniform_cube(n, extent, seed, _ptr(out))
        if rc:
            raise OracleError(rc, "gen_uniform_cube")
        return out

    def gen_gaussian_clusters(self, n, clusters, extent, sigma, seed):
        out = np.empty((n, 3), dtype=np.float64)
        rc = self.lib.ref_gen_gaussian_clusters(n, clusters, extent, sigma, seed, _ptr(out))
        if rc:
            raise OracleError(rc, "gen_gaussian_clusters")
        return out

    def gen_grid_snapped(self, n, cells, voxel, seed):
        out = np.empty((n, 3), dtype=np.float64)
        rc = self.lib.ref_gen_grid_snapped(n, cells, voxel, seed, _ptr(out))
        if rc:
            raise OracleError(rc, "gen_grid_snapped")
        return out

    def gen_features(self, n, g, c, seed, dtype=np.float32):
        out = np.empty((n, g, c), dtype=dtype)
        s = "f32" if dtype == np.float32 else "f64"
        getattr(self.lib, f"ref_gen_features_{s}")(n, g, c, seed, _ptr(out))
        return out

    def make_weights(self, t, g, cin, cout, seed, dtype=np.float32):
        out = np.empty((t ** 3, g, cin, cout), dtype=dtype)
        s = "f32" if dtype == np.float32 else "f64"
        getattr(self.lib, f"ref_make_weights_{s}")(t, g, cin, cout, seed, _ptr(out))
        return out

    def _pairs(self, fn, q, q_off, t, t_off, radius):
        q = _f64(q).reshape(-1, 3)
        t = _f64(t).reshape(-1, 3)
        qo, to = _offsets(len(q), q_off), _offsets(len(t), t_off)
        h = _P()
        rc = fn(_ptr(q), _ptr(qo), len(qo) - 1, _ptr(t), _ptr(to), len(to) - 1, radius, C.byref(h))
        if rc:
            raise OracleError(rc, "radius_search")
        n = self.lib.ref_pairs_size(h)
        oi = np.empty(n, dtype=np.int64)
        ii = np.empty(n, dtype=np.int64)
        self.lib.ref_pairs_copy(h, _ptr(oi), _ptr(ii))
        self.lib.ref_pairs_free(h)
        return oi, ii

    def radius_search(self, q, t, radius, q_off=None, t_off=None):
        return self._pairs(self.lib.ref_radius_search, q, q_off, t, t_off, radius)

    def brute_radius(self, q, t, radius, q_off=None, t_off=None):
        return self._pairs(self.lib.ref_brute_radius, q, q_off, t, t_off, radius)

    def kernel_index(self, center, neighbor, radius, t) -> int:
        return int(self.lib.ref_kernel_index(_ptr(_f64(center)), _ptr(_f64(neighbor)), radius, t))

    def build_triplets(self, out_xyz, in_xyz, radius, t, axis=0, out_off=None, in_off=None):
        """build_triplets_native, then sort_triplets(axis) (axis=-1: choose_sort_axis)."""
        o = _f64(out_xyz).reshape(-1, 3)
        i = _f64(in_xyz).reshape(-1, 3)
        oo, io = _offsets(len(o), out_off), _offsets(len(i), in_off)
        h = _P()
        rc = self.lib.ref_build_triplets(_ptr(o), _ptr(oo), len(oo) - 1, _ptr(i), _ptr(io),
                                         len(io) - 1, radius, t, axis, C.byref(h))
        if rc:
            raise OracleError(rc, "build_triplets_native")
        n = self.lib.ref_triplets_size(h)
        ti, tj, tk = (np.empty(n, dtype=np.uint32) for _ in range(3))
        self.lib.ref_triplets_copy(h, _ptr(ti), _ptr(tj), _ptr(tk))
        self.lib.ref_triplets_free(h)
        return ti, tj, tk

    def sort_triplets(self, ti, tj, tk, axis, n_out, n_in, n_kernels):
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        oi, oj, ok = (np.empty_like(ti) for _ in range(3))
        rc = self.lib.ref_sort_triplets(_ptr(ti), _ptr(tj), _ptr(tk), len(ti), n_out, n_in,
                                        n_kernels, axis, _ptr(oi), _ptr(oj), _ptr(ok))
        if rc:
            raise OracleError(rc, "sort_triplets")
        return oi, oj, ok

    def mvmr(self, w, fin, ti, tj, tk, n_out, tl_out=None, tl_in=None, grouped=1, det=0, L=128,
             workers=0):
        dt = w.dtype
        s = "f32" if dt == np.float32 else "f64"
        K, G, cin, cout = w.shape
        t = round(K ** (1 / 3))
        fin = np.ascontiguousarray(fin, dtype=dt)
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        out = np.zeros((n_out, G, cout), dtype=dt)
        rc = getattr(self.lib, f"ref_mvmr_{s}")(
            _ptr(np.ascontiguousarray(w)), t, G, cin, cout, _ptr(fin), fin.shape[0], _ptr(ti),
            _ptr(tj), _ptr(tk), len(ti), n_out if tl_out is None else tl_out,
            fin.shape[0] if tl_in is None else tl_in, n_out, grouped, det, L, workers, _ptr(out))
        if rc:
            raise OracleError(rc, "mvmr")
        return out

    def mvmr_transposed(self, w, gout, ti, tj, tk, n_in, tl_out=None, tl_in=None, grouped=1,
                        det=0, L=128, workers=0):
        dt = w.dtype
        s = "f32" if dt == np.float32 else "f64"
        K, G, cin, cout = w.shape
        t = round(K ** (1 / 3))
        gout = np.ascontiguousarray(gout, dtype=dt)
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        out = np.zeros((n_in, G, cin), dtype=dt)
        rc = getattr(self.lib, f"ref_mvmr_transposed_{s}")(
            _ptr(np.ascontiguousarray(w)), t, G, cin, cout, _ptr(gout), gout.shape[0], _ptr(ti),
            _ptr(tj), _ptr(tk), len(ti), gout.shape[0] if tl_out is None else tl_out,
            n_in if tl_in is None else tl_in, n_in, grouped, det, L, workers, _ptr(out))
        if rc:
            raise OracleError(rc, "mvmr_transposed")
        return out

    def vvor(self, gout, fin, ti, tj, tk, n_kernels, tl_out=None, tl_in=None, grouped=1, det=0,
             L=128, workers=0):
        dt = gout.dtype
        s = "f32" if dt == np.float32 else "f64"
        gout = np.ascontiguousarray(gout)
        fin = np.ascontiguousarray(fin, dtype=dt)
        _, G, cout = gout.shape
        cin = fin.shape[2]
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        out = np.zeros((n_kernels, G, cout, cin), dtype=dt)
        rc = getattr(self.lib, f"ref_vvor_{s}")(
            _ptr(gout), gout.shape[0], _ptr(fin), fin.shape[0], G, cin, cout, _ptr(ti), _ptr(tj),
            _ptr(tk), len(ti), gout.shape[0] if tl_out is None else tl_out,
            fin.shape[0] if tl_in is None else tl_in, n_kernels, grouped, det, L, workers,
            _ptr(out))
        if rc:
            raise OracleError(rc, "vvor")
        return out

    def dense_conv(self, w, fin, ti, tj, tk, n_out, gout=None):
        w = _f64(w)
        K, G, cin, cout = w.shape
        t = round(K ** (1 / 3))
        fin = _f64(fin).reshape(-1, G, cin)
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        fout = np.zeros((n_out, G, cout))
        gin = gw = None
        if gout is not None:
            gout = _f64(gout).reshape(n_out, G, cout)
            gin = np.zeros_like(fin)
            gw = np.zeros((K, G, cout, cin))
        rc = self.lib.ref_dense_oracle(_ptr(w), t, G, cin, cout, _ptr(fin), len(fin), _ptr(ti),
                                       _ptr(tj), _ptr(tk), len(ti), n_out, len(fin), n_out,
                                       _ptr(gout), _ptr(fout), _ptr(gin), _ptr(gw))
        if rc:
            raise OracleError(rc, "dense_conv_oracle")
        return fout, gin, gw

    def voxel_downsample(self, xyz, voxel, offsets=None):
        xyz = _f64(xyz).reshape(-1, 3)
        off = _offsets(len(xyz), offsets)
        kept = np.empty(len(xyz), dtype=np.int64)
        parent = np.empty(len(xyz), dtype=np.int64)
        out_off = np.empty(len(off), dtype=np.int64)
        m = self.lib.ref_voxel_downsample(_ptr(xyz), _ptr(off), len(off) - 1, voxel, _ptr(kept),
                                          _ptr(parent), _ptr(out_off))
        if m < 0:
            raise OracleError(-m, "voxel_downsample")
        return kept[:m].copy(), parent, out_off

    def upsample(self, xyz, kept, parent, coarse, offsets=None):
        """The reference's upsample (spatial.hpp:52-54) of coarse (n_kept, G, C)."""
        xyz = _f64(xyz).reshape(-1, 3)
        off = _offsets(len(xyz), offsets)
        coarse = np.ascontiguousarray(coarse)
        s = "f32" if coarse.dtype == np.float32 else "f64"
        kept = np.ascontiguousarray(kept, np.int64)
        parent = np.ascontiguousarray(parent, np.int64)
        _, G, Cc = coarse.shape
        out = np.empty((len(xyz), G, Cc), dtype=coarse.dtype)
        rc = getattr(self.lib, f"ref_upsample_{s}")(_ptr(xyz), _ptr(off), len(off) - 1, _ptr(kept),
                                                    len(kept), _ptr(parent), _ptr(coarse), G, Cc,
                                                    _ptr(out))
        if rc:
            raise OracleError(rc, "upsample")
        return out

    def build_triplets_degraded(self, xyz, voxel, t, offsets=None):
        """The reference's build_triplets_degraded (triplets.hpp:63-76)."""
        return _degraded(self.lib, "ref_build_triplets_degraded", "ref", xyz, voxel, t, offsets)

    # -- io.hpp / triplets.hpp:84-93 through the reference's writers / readers --
    def write_cloud(self, path, xyz, offsets=None):
        xyz = _f64(xyz).reshape(-1, 3)
        off = _offsets(len(xyz), offsets)
        rc = self.lib.ref_write_cloud(path.encode(), _ptr(xyz), _ptr(off), len(off) - 1)
        if rc:
            raise OracleError(rc, "write_cloud")

    def read_cloud(self, path):
        nb = _I64()
        n = self.lib.ref_read_cloud(path.encode(), None, None, C.byref(nb))
        if n < 0:
            raise OracleError(-n, "read_cloud")
        xyz = np.empty((n, 3), dtype=np.float64)
        off = np.empty(nb.value + 1, dtype=np.int64)
        self.lib.ref_read_cloud(path.encode(), _ptr(xyz), _ptr(off), C.byref(nb))
        return xyz, off

    def write_triplets(self, path, ti, tj, tk, n_out, n_in, n_kernels, axis=0):
        ti, tj, tk = _u32(ti), _u32(tj), _u32(tk)
        rc = self.lib.ref_write_triplets(path.encode(), _ptr(ti), _ptr(tj), _ptr(tk), len(ti),
                                         n_out, n_in, n_kernels, axis)
        if rc:
            raise OracleError(rc, "write_triplets")

    def read_triplets(self, path):
        meta = np.zeros(5, dtype=np.int64)
        rc = self.lib.ref_read_triplets(path.encode(), None, None, None, _ptr(meta))
        if rc:
            raise OracleError(rc, "read_triplets")
        ti, tj, tk = (np.empty(int(meta[0]), dtype=np.uint32) for _ in range(3))
        self.lib.ref_read_triplets(path.encode(), _ptr(ti), _ptr(tj), _ptr(tk), _ptr(meta))
        return ti, tj, tk, int(meta[1]), int(meta[2]), int(meta[3]), int(meta[4])

    def conv_layer_f32(self, xyz, radius, t, w, fin, gout, workers=0, build=True, cache=None,
                       outputs=False):
        """Times the reference chain; returns (times[5], cache_handle, (fout, gin, gw)|None)."""
        xyz = _f64(xyz)
        n = len(xyz)
        K, _, cin, cout = w.shape
        times = np.zeros(5)
        h = cache if cache is not None else _P()
        fo = gi = gw = None
        if outputs:
            fo = np.empty((n, 1, cout), np.float32)
            gi = np.empty((n, 1, cin), np.float32)
            gw = np.empty((K, 1, cout, cin), np.float32)
        rc = self.lib.ref_conv_layer_f32(_ptr(xyz), n, radius, t, cin, cout,
                                         _ptr(np.ascontiguousarray(w, np.float32)),
                                         _ptr(np.ascontiguousarray(fin, np.float32)),
                                         _ptr(np.ascontiguousarray(gout, np.float32)), workers,
                                         1 if build else 0, _ptr(times), _ptr(fo), _ptr(gi),
                                         _ptr(gw), C.byref(h))
        if rc:
            raise OracleError(rc, "conv_layer")
        return times, h, ((fo, gi, gw) if outputs else None)

    def free_cache(self, h):
        if h is not None and h.value:
            self.lib.ref_conv_cache_free(h)
