"""Python mirror of the reference ``npc::`` operator API over libnpcg.so.

Same names, argument meaning and error classes as the reference headers
(``/root/reference/proj/core/include/npconv/*.hpp``); tensors are torch CUDA
tensors (device memory plumbing only -- every computation is a libnpcg.so
kernel).  Reference -> here:

    PointCloud / make_point_cloud     point_cloud.hpp:18-50
    radius_search                     spatial.hpp:39-40
    voxel_downsample / upsample       spatial.hpp:47-54
    local_voxel_kernel_index          triplets.hpp:48-49
    build_triplets_native             triplets.hpp:56-57
    sort_triplets / choose_sort_axis  triplets.hpp:78-82
    mvmr / mvmr_transposed            engine.hpp:66-76
    vvor / WeightGradient             vvor.hpp:12-88
    PointConvOp / strided_block       conv_op.hpp:32-225
    Error hierarchy                   errors.hpp:10-67

Layouts: features (N, G, C); weights (K, G, C_in, C_out); weight gradients
(K, G, C_out, C_in); triplets SoA u32 (held as int32 tensors, same bits).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

# ---------------------------------------------------------------------------
# errors (errors.hpp:10-67)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    """Base class for all npconv errors."""


class OffsetError(Error):
    pass


class NonFiniteError(Error):
    pass


class ShapeError(Error):
    pass


class RadiusError(Error):
    pass


class VoxelError(Error):
    pass


class NpcIndexError(Error):
    pass


class DomainError(Error):
    pass


class StateError(Error):
    pass


class NpcIOError(Error):
    pass


class CudaError(Error):
    pass


class OutOfMemory(Error):
    pass


class InvalidArgument(Error):
    pass


class Unsupported(Error):
    pass


# reference spellings (they shadow Python builtins only inside this namespace)
IndexError = NpcIndexError  # noqa: A001
IOError = NpcIOError  # noqa: A001

_ERRORS = {1: OffsetError, 2: NonFiniteError, 3: ShapeError, 4: RadiusError, 5: VoxelError,
           6: NpcIndexError, 7: DomainError, 8: StateError, 9: NpcIOError, 10: CudaError,
           11: OutOfMemory, 12: InvalidArgument, 13: Unsupported}


class SortAxis(enum.IntEnum):  # triplets.hpp:15
    none = 0
    by_i = 1
    by_j = 2
    by_k = 3


class Executor(enum.IntEnum):  # engine.hpp:11
    naive = 0
    grouped = 1


class Math(enum.IntEnum):  # npcg_math
    auto = 0    # the reference's fp32 contract (rel <= 1e-5): split tensor cores, else exact
    exact = 1   # CUDA cores in the API dtype
    bf16 = 2    # opt-in: bf16 operands on the tensor cores (rel ~2e-3, bound 1e-2)
    f32tc = 3   # split operands on the tensor cores (rel ~4e-6, bound 1e-5)


class ConvMode(enum.IntEnum):  # triplets.hpp:34
    native = 0
    degraded = 1


@dataclass
class ExecConfig:  # engine.hpp:22-29 (+ math)
    L: int = 128
    b_out: int = 32
    b_in: int = 32
    executor: Executor = Executor.grouped
    deterministic: bool = False
    workers: int = 0
    math: Math = Math.auto
    flags: int = 0  # npcg flags (L.FLAG_FIN_UNCHANGED)

    def _c(self, flags: int = 0):
        return L.npcg_exec_config(self.L, self.b_out, self.b_in, int(self.executor),
                                  int(bool(self.deterministic)), self.workers, int(self.math),
                                  int(self.flags) | flags, 0)


@dataclass
class ConvGeometry:  # triplets.hpp:36-41
    radius: float = 1.0
    t: int = 3
    mode: ConvMode = ConvMode.native
    voxel_size: float = 1.0


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


class Context:
    """One libnpcg context per CUDA device; follows torch's current stream."""

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        st = L.lib().npcg_context_create(device, None, C.byref(h))
        if st:
            raise _ERRORS.get(st, Error)(
                f"npcg_context_create(device={device}) failed: {L.STATUS_NAMES.get(st, st)}"
                " -- a B200 (sm_100a) is required; there is no CPU fallback")
        self.h = h

    def bind(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        L.lib().npcg_context_set_stream(self.h, C.c_void_p(s))
        return self.h

    def check(self, status: int, what: str):
        if status:
            msg = (L.lib().npcg_last_error(self.h) or b"").decode()
            raise _ERRORS.get(status, Error)(f"{what}: {msg}" if msg else what)

    def launch_count(self) -> int:
        n = C.c_int64()
        L.lib().npcg_launch_count(self.h, C.byref(n))
        return n.value

    def profile(self, enable: bool):
        L.lib().npcg_profile_enable(self.h, int(enable))

    def profile_reset(self):
        self.check(L.lib().npcg_profile_reset(self.h), "profile_reset")

    def profile_query(self, name_substr: str = ""):
        n = C.c_int64()
        ms = C.c_double()
        self.check(L.lib().npcg_profile_query(self.h, name_substr.encode(), C.byref(n),
                                              C.byref(ms)), "profile_query")
        return n.value, ms.value

    def profile_dump(self) -> dict:
        buf = C.create_string_buffer(1 << 16)
        self.check(L.lib().npcg_profile_dump(self.h, buf, len(buf)), "profile_dump")
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split("\t")
            out[name] = (int(n), float(ms))
        return out

    def memory(self):
        cur = C.c_int64()
        peak = C.c_int64()
        L.lib().npcg_memory_stats(self.h, C.byref(cur), C.byref(peak))
        return cur.value, peak.value

    def reset_peak(self):
        L.lib().npcg_memory_reset_peak(self.h)


_ctx_lock = threading.Lock()
_contexts: dict[int, Context] = {}


def context(device=None) -> Context:
    if device is None:
        device = torch.cuda.current_device()
    if isinstance(device, torch.device):
        device = device.index if device.index is not None else torch.cuda.current_device()
    with _ctx_lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else None


def _dev(t, dtype=None, device=None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.ascontiguousarray(t))
    if device is None:
        device = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
    return t.to(device=device, dtype=dtype or t.dtype).contiguous()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.float64:
        return 1
    raise ShapeError(f"unsupported feature dtype {t.dtype} (float32 / float64)")


# ---------------------------------------------------------------------------
# point clouds (point_cloud.hpp / point_cloud.cpp)
# ---------------------------------------------------------------------------


class PointCloud:
    """Batched point set: (N, 3) float64 positions on the GPU + host batch offsets."""

    def __init__(self, positions: torch.Tensor, batch_offsets: np.ndarray):
        self.xyz = positions
        self.offsets = np.ascontiguousarray(batch_offsets, dtype=np.int64)

    def n_points(self) -> int:
        return int(self.xyz.shape[0])

    def n_batches(self) -> int:
        return len(self.offsets) - 1

    def batch_offsets(self) -> np.ndarray:
        return self.offsets

    def batch_range(self, b: int):
        return int(self.offsets[b]), int(self.offsets[b + 1])

    def positions(self) -> np.ndarray:
        return self.xyz.detach().cpu().numpy()

    def _c(self):
        return L.npcg_cloud(_ptr(self.xyz), self.offsets.ctypes.data_as(C.c_void_p),
                            self.n_points(), self.n_batches())


def validate_offsets(n: int, offsets) -> np.ndarray:
    """point_cloud.cpp:20-31 (host logic, raises OffsetError)."""
    off = np.asarray(offsets, dtype=np.int64)
    if off.ndim != 1 or off.size < 2:
        raise OffsetError("batch_offsets needs at least [0, N]")
    if off[0] != 0:
        raise OffsetError("batch_offsets must start at 0")
    if off[-1] != n:
        raise OffsetError(f"batch_offsets must end at the point count ({n})")
    if np.any(np.diff(off) < 0):
        raise OffsetError("batch_offsets must be monotone non-decreasing")
    return off


def make_point_cloud(positions, batch_offsets=None, device=None) -> PointCloud:
    """point_cloud.hpp:44-50: validates offsets and finiteness, uploads to the GPU."""
    if isinstance(positions, torch.Tensor):
        pos = positions.to(torch.float64)
    else:
        pos = torch.as_tensor(np.asarray(positions, dtype=np.float64))
    pos = pos.reshape(-1, 3)
    n = int(pos.shape[0])
    off = validate_offsets(n, [0, n] if batch_offsets is None else batch_offsets)
    if n and not bool(torch.isfinite(pos).all()):
        raise NonFiniteError("point coordinate is NaN or infinite")
    return PointCloud(_dev(pos, torch.float64, device), off)


# ---------------------------------------------------------------------------
# neighbor handles, NeighborList, TripletList
# ---------------------------------------------------------------------------


class Neighbors:
    """Owns a device-resident npcg_neighbors (the PointConvOp triplet cache)."""

    def __init__(self, ctx: Context, handle: C.c_void_p, clouds=()):
        self.ctx = ctx
        self.h = handle
        self._keep = clouds  # positions must outlive nothing, but keep for identity checks
        n = C.c_int64()
        L.lib().npcg_neighbors_size(handle, C.byref(n))
        no, ni, nk = C.c_int64(), C.c_int64(), C.c_int64()
        r = C.c_double()
        L.lib().npcg_neighbors_info(handle, C.byref(no), C.byref(ni), C.byref(nk), C.byref(r))
        self.size, self.n_out, self.n_in, self.n_kernels, self.radius = (
            n.value, no.value, ni.value, nk.value, r.value)
        ns, nf, nbat = C.c_int64(), C.c_int64(), C.c_int64()
        self.degraded = L.lib().npcg_neighbors_sites(handle, C.byref(ns), C.byref(nf),
                                                     C.byref(nbat)) == 0
        # rows of the caller's input features (degraded: the original points)
        self.n_fine = nf.value if self.degraded else self.n_in
        self._sites = None

    def sites(self):
        """Degraded handles (conv_op.hpp:56-57): (snapped_cloud, DownsampleMap)."""
        if not self.degraded:
            raise StateError("PointConvOp: no degraded cache")
        if self._sites is None:
            dev = torch.device("cuda", self.ctx.device)
            nbat = C.c_int64()
            L.lib().npcg_neighbors_sites(self.h, None, None, C.byref(nbat))
            xyz = torch.empty((self.n_out, 3), dtype=torch.float64, device=dev)
            kept = torch.empty(max(self.n_out, 1), dtype=torch.int64, device=dev)
            parent = torch.empty(max(self.n_fine, 1), dtype=torch.int64, device=dev)
            off = np.zeros(nbat.value + 1, dtype=np.int64)
            h = self.ctx.bind()
            self.ctx.check(L.lib().npcg_neighbors_export_sites(
                h, self.h, _ptr(xyz), _ptr(kept), _ptr(parent),
                off.ctypes.data_as(C.c_void_p)), "export_sites")
            self._sites = (PointCloud(xyz, off),
                           DownsampleMap(kept[:self.n_out], parent[:self.n_fine]))
        return self._sites

    def __del__(self):
        try:
            if self.h:
                L.lib().npcg_neighbors_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def export_triplets(self, axis: SortAxis) -> "TripletList":
        dev = torch.device("cuda", self.ctx.device)
        i, j, k = (torch.empty(self.size, dtype=torch.int32, device=dev) for _ in range(3))
        h = self.ctx.bind()
        self.ctx.check(L.lib().npcg_neighbors_export_triplets(h, self.h, int(axis), _ptr(i),
                                                              _ptr(j), _ptr(k)),
                       "export_triplets")
        return TripletList(i, j, k, self.n_out, self.n_in, self.n_kernels, SortAxis(axis),
                           handle=self if axis == SortAxis.none else None)

    def plan_stats(self) -> dict:
        out = (C.c_int64 * 12)()
        h = self.ctx.bind()
        self.ctx.check(L.lib().npcg_neighbors_plan_stats(h, self.h, out), "plan_stats")
        v = list(out)
        # overflow = rows the tensor-core plan leaves to the exact engine
        return {name: {"super_tiles": v[4 * i], "overflow": v[4 * i + 1], "max_halo": v[4 * i + 2],
                       "mean_halo": v[4 * i + 3] / 100.0}
                for i, name in enumerate(("fwd", "dgrad", "wgrad"))}

    def prepare(self, math: Math = Math.auto):
        h = self.ctx.bind()
        self.ctx.check(L.lib().npcg_neighbors_prepare(h, self.h, int(math)), "prepare")


@dataclass
class NeighborList:  # spatial.hpp:14-20
    out_index: torch.Tensor
    in_index: torch.Tensor
    radius: float = 0.0

    def size(self) -> int:
        return int(self.out_index.numel())


@dataclass
class TripletList:  # triplets.hpp:20-30
    i: torch.Tensor
    j: torch.Tensor
    k: torch.Tensor
    n_out: int = 0
    n_in: int = 0
    n_kernels: int = 0
    sort_axis: SortAxis = SortAxis.none
    handle: Neighbors | None = field(default=None, repr=False)

    def size(self) -> int:
        return int(self.i.numel())

    def numpy(self):
        f = lambda t: t.detach().cpu().numpy().view(np.uint32)  # noqa: E731
        return f(self.i), f(self.j), f(self.k)

    def _c(self):
        return L.npcg_triplets(_ptr(self.i), _ptr(self.j), _ptr(self.k), self.size(), self.n_out,
                               self.n_in, self.n_kernels, int(self.sort_axis))

    @staticmethod
    def from_numpy(i, j, k, n_out, n_in, n_kernels, sort_axis=SortAxis.none, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        cv = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(dev)  # noqa: E731
        return TripletList(cv(i), cv(j), cv(k), int(n_out), int(n_in), int(n_kernels),
                           SortAxis(sort_axis))


def _build(out_cloud: PointCloud, in_cloud: PointCloud, radius: float, t: int) -> Neighbors:
    ctx = context(out_cloud.xyz.device)
    h = ctx.bind()
    oc, ic = out_cloud._c(), in_cloud._c()
    nb = C.c_void_p()
    if t == 0:
        st = L.lib().npcg_radius_search(h, C.byref(oc), C.byref(ic), float(radius), C.byref(nb))
    else:
        st = L.lib().npcg_build_triplets_native(h, C.byref(oc), C.byref(ic), float(radius), int(t),
                                                C.byref(nb))
    ctx.check(st, "radius_search" if t == 0 else "build_triplets_native")
    return Neighbors(ctx, nb, (out_cloud, in_cloud))


def radius_search(queries: PointCloud, targets: PointCloud, radius: float) -> NeighborList:
    """spatial.hpp:39-40."""
    nb = _build(queries, targets, radius, 0)
    dev = queries.xyz.device
    oi = torch.empty(nb.size, dtype=torch.int64, device=dev)
    ii = torch.empty(nb.size, dtype=torch.int64, device=dev)
    h = nb.ctx.bind()
    nb.ctx.check(L.lib().npcg_neighbors_export_pairs(h, nb.h, _ptr(oi), _ptr(ii)), "export_pairs")
    return NeighborList(oi, ii, float(radius))


def build_neighbors(out_cloud: PointCloud, in_cloud: PointCloud, geom: ConvGeometry) -> Neighbors:
    """Native mode: radius neighbors of out_cloud in in_cloud with kernel cells.
    Degraded mode: the voxel-site build of in_cloud (out_cloud ignored, as the
    reference's single-cloud degraded forward, conv_op.hpp:116-120)."""
    if geom.mode != ConvMode.native:
        return _build_degraded(in_cloud, geom.voxel_size, geom.t)
    return _build(out_cloud, in_cloud, geom.radius, geom.t)


def _build_degraded(in_cloud: PointCloud, voxel_size: float, t: int) -> Neighbors:
    ctx = context(in_cloud.xyz.device)
    h = ctx.bind()
    ic = in_cloud._c()
    nb = C.c_void_p()
    ctx.check(L.lib().npcg_build_triplets_degraded(h, C.byref(ic), float(voxel_size), int(t),
                                                   C.byref(nb)), "build_triplets_degraded")
    return Neighbors(ctx, nb, (in_cloud,))


@dataclass
class DegradedBuild:  # triplets.hpp:63-67
    triplets: "TripletList"
    snapped: PointCloud
    sites: "DownsampleMap"


def build_triplets_degraded(in_cloud: PointCloud, geom: ConvGeometry) -> DegradedBuild:
    """triplets.hpp:69-76: site triplets in build order (sort_axis none), the
    snapped site cloud and the site map."""
    nb = _build_degraded(in_cloud, geom.voxel_size, geom.t)
    snapped, sites = nb.sites()
    return DegradedBuild(nb.export_triplets(SortAxis.none), snapped, sites)


def build_triplets_native(out_cloud: PointCloud, in_cloud: PointCloud,
                          geom: ConvGeometry) -> TripletList:
    """triplets.hpp:56-57: (i, j)-ordered triplets, sort_axis none."""
    if geom.t < 1 or geom.t % 2 == 0:
        raise ShapeError("conv geometry: kernel resolution t must be odd and >= 1")
    return _build(out_cloud, in_cloud, geom.radius, geom.t).export_triplets(SortAxis.none)


def kernel_index_batch(centers, neighbors, radius: float, t: int) -> torch.Tensor:
    c = _dev(centers, torch.float64).reshape(-1, 3)
    nb = _dev(neighbors, torch.float64, c.device).reshape(-1, 3)
    ctx = context(c.device)
    out = torch.empty(c.shape[0], dtype=torch.int64, device=c.device)
    h = ctx.bind()
    ctx.check(L.lib().npcg_kernel_index(h, _ptr(c), _ptr(nb), c.shape[0], float(radius), int(t),
                                        _ptr(out)), "local_voxel_kernel_index")
    return out


def local_voxel_kernel_index(center, neighbor, radius: float, t: int) -> int:
    """triplets.hpp:48-49 (evaluated by the GPU kernel-cell recipe)."""
    return int(kernel_index_batch([center], [neighbor], radius, t)[0].item())


def choose_sort_axis(triplets: TripletList) -> SortAxis:
    """triplets.hpp:82."""
    return SortAxis(L.lib().npcg_choose_sort_axis(triplets.n_out, triplets.n_in,
                                                  triplets.n_kernels))


def sort_triplets(triplets: TripletList, axis: SortAxis) -> TripletList:
    """triplets.hpp:78: stable counting-sort semantics; input untouched."""
    n = triplets.size()
    dev = triplets.i.device
    oi, oj, ok = (torch.empty(n, dtype=torch.int32, device=dev) for _ in range(3))
    ctx = context(dev)
    h = ctx.bind()
    tc = triplets._c()
    ctx.check(L.lib().npcg_sort_triplets(h, C.byref(tc), int(axis), _ptr(oi), _ptr(oj), _ptr(ok)),
              "sort_triplets")
    return TripletList(oi, oj, ok, triplets.n_out, triplets.n_in, triplets.n_kernels,
                       SortAxis(axis))


# ---------------------------------------------------------------------------
# engines (engine.hpp / vvor.hpp)
# ---------------------------------------------------------------------------


@dataclass
class MvmrResult:
    out: torch.Tensor


@dataclass
class VvorResult:
    grad: torch.Tensor  # (K, G, C_out, C_in)


def _t_of(K: int) -> int:
    t = round(K ** (1.0 / 3.0))
    for c in (t - 1, t, t + 1):
        if c >= 1 and c ** 3 == K:
            return c
    raise ShapeError("WeightTensor: K must be t^3 with t odd")


def to_weight_tensor(grad: torch.Tensor) -> torch.Tensor:
    """vvor.hpp:50-62 WeightGradient::to_weight_tensor: (K,G,Cout,Cin) -> (K,G,Cin,Cout)."""
    return grad.transpose(-1, -2).contiguous()


def transposed_weights(w: torch.Tensor) -> torch.Tensor:
    """tensors.hpp:113-123 WeightTensor::transposed."""
    return w.transpose(-1, -2).contiguous()


def mvmr(weights: torch.Tensor, fin: torch.Tensor, triplets: TripletList, n_out: int,
         config: ExecConfig = ExecConfig()) -> MvmrResult:
    """engine.hpp:66-69."""
    K, G, cin, cout = weights.shape
    if fin.dim() != 3 or fin.shape[1] != G:
        raise ShapeError("mvmr: weight and feature group counts differ")
    if fin.shape[2] != cin:
        raise ShapeError("mvmr: weight C_in_g does not match feature channels")
    if fin.dtype != weights.dtype:
        raise ShapeError("mvmr: weight and feature dtypes differ")
    t = _t_of(K)
    dev = fin.device
    out = torch.empty((max(int(n_out), 0), G, cout), dtype=fin.dtype, device=dev)
    ctx = context(dev)
    h = ctx.bind()
    tc, cfg = triplets._c(), config._c()
    w = weights.contiguous()
    f = fin.contiguous()
    ctx.check(L.lib().npcg_mvmr(h, _dtype_code(f), _ptr(w), t, G, cin, cout, _ptr(f), f.shape[0],
                                C.byref(tc), int(n_out), C.byref(cfg), _ptr(out)), "mvmr")
    return MvmrResult(out)


def mvmr_transposed(weights: torch.Tensor, gout: torch.Tensor, triplets: TripletList, n_in: int,
                    config: ExecConfig = ExecConfig()) -> MvmrResult:
    """engine.hpp:73-76."""
    K, G, cin, cout = weights.shape
    if gout.dim() != 3 or gout.shape[2] != cout:
        raise ShapeError("mvmr_transposed: weight C_out_g does not match gradient channels")
    if gout.shape[1] != G:
        raise ShapeError("mvmr: weight and feature group counts differ")
    t = _t_of(K)
    dev = gout.device
    out = torch.empty((max(int(n_in), 0), G, cin), dtype=gout.dtype, device=dev)
    ctx = context(dev)
    h = ctx.bind()
    tc, cfg = triplets._c(), config._c()
    w = weights.contiguous()
    g = gout.contiguous()
    ctx.check(L.lib().npcg_mvmr_transposed(h, _dtype_code(g), _ptr(w), t, G, cin, cout, _ptr(g),
                                           g.shape[0], C.byref(tc), int(n_in), C.byref(cfg),
                                           _ptr(out)), "mvmr_transposed")
    return MvmrResult(out)


def vvor(gout: torch.Tensor, fin: torch.Tensor, triplets: TripletList, n_kernels: int,
         config: ExecConfig = ExecConfig()) -> VvorResult:
    """vvor.hpp:85-88."""
    if gout.dim() != 3 or fin.dim() != 3 or gout.shape[1] != fin.shape[1]:
        raise ShapeError("vvor: gradient and feature group counts differ")
    G, cout, cin = gout.shape[1], gout.shape[2], fin.shape[2]
    if n_kernels < 1:
        raise ShapeError("vvor: n_kernels must be >= 1")
    dev = gout.device
    grad = torch.empty((int(n_kernels), G, cout, cin), dtype=gout.dtype, device=dev)
    ctx = context(dev)
    h = ctx.bind()
    tc, cfg = triplets._c(), config._c()
    g = gout.contiguous()
    f = fin.contiguous()
    ctx.check(L.lib().npcg_vvor(h, _dtype_code(g), _ptr(g), g.shape[0], _ptr(f), f.shape[0], G, cin,
                                cout, C.byref(tc), int(n_kernels), C.byref(cfg), _ptr(grad)),
              "vvor")
    return VvorResult(grad)


# ---------------------------------------------------------------------------
# operator (conv_op.hpp)
# ---------------------------------------------------------------------------


@dataclass
class BackwardResult:
    grad_in: torch.Tensor
    grad_w: torch.Tensor


def _check_layer(nb: Neighbors, weights: torch.Tensor, rows: torch.Tensor, n_rows: int,
                 width: int, what: str):
    """The operator's shape checks (conv_op.hpp:129-131, engine.cpp:284-288)
    before any device work: weight kernel count, feature rows and widths."""
    if weights.dim() != 4 or weights.shape[0] != nb.n_kernels:
        raise ShapeError(f"{what}: weight kernel count != geometry t^3")
    if rows.dim() != 3 or rows.shape[0] != n_rows:
        raise ShapeError(f"{what}: feature rows != cloud points")
    if rows.shape[1] != weights.shape[1] or rows.shape[2] != width:
        raise ShapeError(f"{what}: weight and feature shapes differ")
    if rows.dtype != weights.dtype:
        raise ShapeError(f"{what}: weight and feature dtypes differ")


def conv_forward(nb: Neighbors, weights: torch.Tensor, fin: torch.Tensor,
                 config: ExecConfig = ExecConfig(), out: torch.Tensor | None = None):
    """npcg_conv_forward over a cached neighbor handle."""
    K, G, cin, cout = weights.shape
    _check_layer(nb, weights, fin, nb.n_fine, cin, "conv_forward")
    if out is None:
        out = torch.empty((nb.n_out, G, cout), dtype=fin.dtype, device=fin.device)
    cfg = config._c()
    h = nb.ctx.bind()
    nb.ctx.check(L.lib().npcg_conv_forward(h, nb.h, _dtype_code(fin), _ptr(weights), G, cin, cout,
                                           _ptr(fin), C.byref(cfg), _ptr(out)), "conv_forward")
    return out


def conv_backward(nb: Neighbors, weights: torch.Tensor, fin: torch.Tensor, gout: torch.Tensor,
                  config: ExecConfig = ExecConfig(), grad_in=None, grad_w=None, need_in=True,
                  need_w=True, fin_unchanged: bool = False):
    """npcg_conv_backward.  fin_unchanged: `fin` is the very buffer the last
    conv_forward on this handle read, unmodified since (the operator's saved
    input) -- its device image is then reused (NPCG_FLAG_FIN_UNCHANGED)."""
    K, G, cin, cout = weights.shape
    if fin is not None:
        _check_layer(nb, weights, fin, nb.n_fine, cin, "conv_backward")
    _check_layer(nb, weights, gout, nb.n_out, cout, "conv_backward")
    if need_in and grad_in is None:
        grad_in = torch.empty((nb.n_fine, G, cin), dtype=gout.dtype, device=gout.device)
    if need_w and grad_w is None:
        grad_w = torch.empty((K, G, cout, cin), dtype=gout.dtype, device=gout.device)
    cfg = config._c(L.FLAG_FIN_UNCHANGED if fin_unchanged else 0)
    h = nb.ctx.bind()
    nb.ctx.check(L.lib().npcg_conv_backward(h, nb.h, _dtype_code(gout), _ptr(weights), G, cin, cout,
                                            _ptr(fin), _ptr(gout), C.byref(cfg),
                                            _ptr(grad_in) if need_in else None,
                                            _ptr(grad_w) if need_w else None), "conv_backward")
    return grad_in, grad_w


class PointConvOp:
    """conv_op.hpp:32-84: owns weights + geometry, caches the neighbor structure
    per (position buffers, sizes) identity (conv_op.hpp:106-127), forward /
    backward through the GPU engines.  No bias, no activation."""

    def __init__(self, weights: torch.Tensor, geometry: ConvGeometry,
                 config: ExecConfig = ExecConfig(), copy_fin: bool = True):
        if _t_of(weights.shape[0]) != geometry.t:
            raise ShapeError("PointConvOp: weight kernel resolution != geometry t")
        self._w = weights.contiguous()
        self.geometry_ = geometry
        self.config_ = config
        self.copy_fin = copy_fin
        self._nb: Neighbors | None = None
        self._key = None
        self._sorted: TripletList | None = None
        self._fin: torch.Tensor | None = None

    def weights(self):
        return self._w

    def geometry(self):
        return self.geometry_

    def config(self):
        return self.config_

    def neighbors(self) -> Neighbors:
        if self._nb is None:
            raise StateError("PointConvOp: no triplet cache yet, run forward first")
        return self._nb

    def cached_triplets(self) -> TripletList:
        """The sorted triplet cache (sort_triplets(..., choose_sort_axis), conv_op.hpp:123)."""
        nb = self.neighbors()
        if self._sorted is None:
            axis = SortAxis(L.lib().npcg_choose_sort_axis(nb.n_out, nb.n_in, nb.n_kernels))
            self._sorted = nb.export_triplets(axis)
        return self._sorted

    def snapped_cloud(self) -> PointCloud:
        """conv_op.hpp:56: sites of the last degraded forward."""
        if self._nb is None or not self._nb.degraded:
            raise StateError("PointConvOp: no degraded cache")
        return self._nb.sites()[0]

    def site_map(self) -> "DownsampleMap":
        """conv_op.hpp:57."""
        if self._nb is None or not self._nb.degraded:
            raise StateError("PointConvOp: no degraded cache")
        return self._nb.sites()[1]

    def _build_cache(self, in_cloud: PointCloud, out_cloud: PointCloud):
        key = (in_cloud.xyz.data_ptr(), out_cloud.xyz.data_ptr(), in_cloud.n_points(),
               out_cloud.n_points())
        if self._nb is not None and key == self._key:
            return
        self._nb = build_neighbors(out_cloud, in_cloud, self.geometry_)
        self._key = key
        self._sorted = None
        self._fin = None

    def forward(self, in_cloud: PointCloud, a, b=None) -> torch.Tensor:
        """forward(in_cloud, fin) or forward(in_cloud, out_cloud, fin)."""
        if b is None:
            out_cloud, fin = in_cloud, a
        else:
            if self.geometry_.mode != ConvMode.native:
                raise StateError("PointConvOp::forward: two-cloud forward requires native mode")
            out_cloud, fin = a, b
        if fin.shape[0] != in_cloud.n_points():
            raise ShapeError("PointConvOp::forward: feature rows != cloud points")
        if fin.dim() != 3 or fin.shape[1] != self._w.shape[1] or fin.shape[2] != self._w.shape[2]:
            raise ShapeError("mvmr: weight and feature shapes differ")
        self._build_cache(in_cloud, out_cloud)
        out = conv_forward(self._nb, self._w, fin.contiguous(), self.config_)
        self._fin = fin.clone() if self.copy_fin else fin.contiguous()  # conv_op.hpp:138
        return out

    def backward(self, gout: torch.Tensor) -> BackwardResult:
        if self._fin is None:
            raise StateError("PointConvOp::backward: no cached forward inputs")
        K, G, cin, cout = self._w.shape
        if gout.dim() != 3 or gout.shape[0] != self._nb.n_out or gout.shape[1] != G or \
                gout.shape[2] != cout:
            raise ShapeError("PointConvOp::backward: gout shape mismatch")
        # the saved input is the operator's own copy (or, with copy_fin=False,
        # the caller's promise not to modify it): its device image is reused
        gi, gw = conv_backward(self._nb, self._w, self._fin, gout.contiguous(), self.config_,
                               fin_unchanged=True)
        return BackwardResult(gi, gw)


# ---------------------------------------------------------------------------
# strided path (spatial.hpp:47-54, conv_op.hpp:219-225)
# ---------------------------------------------------------------------------


@dataclass
class DownsampleMap:  # spatial.hpp:25-28
    kept_index: torch.Tensor
    parent_of: torch.Tensor


def voxel_downsample(cloud: PointCloud, voxel_size: float):
    ctx = context(cloud.xyz.device)
    n = cloud.n_points()
    dev = cloud.xyz.device
    kept = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    parent = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    out_off = np.zeros(cloud.n_batches() + 1, dtype=np.int64)
    nk = C.c_int64()
    h = ctx.bind()
    cc = cloud._c()
    ctx.check(L.lib().npcg_voxel_downsample(h, C.byref(cc), float(voxel_size), _ptr(kept),
                                            _ptr(parent), out_off.ctypes.data_as(C.c_void_p),
                                            C.byref(nk)), "voxel_downsample")
    kept = kept[:nk.value]
    coarse = PointCloud(cloud.xyz.index_select(0, kept).contiguous(), out_off)
    return coarse, DownsampleMap(kept, parent[:n])


def upsample(fine: PointCloud, mp: DownsampleMap, coarse: torch.Tensor) -> torch.Tensor:
    """spatial.hpp:52-54 (spatial.cpp:154-169) through npcg_upsample: fine row m
    = coarse row parent_of[m]."""
    if mp.parent_of.numel() != fine.n_points():
        raise ShapeError("upsample: map does not cover the fine cloud")
    if mp.kept_index.numel() != coarse.shape[0]:
        raise ShapeError("upsample: coarse features do not match the map")
    c = coarse.contiguous()
    n = fine.n_points()
    out = torch.empty((n,) + tuple(c.shape[1:]), dtype=c.dtype, device=c.device)
    width = int(np.prod(c.shape[1:])) if c.dim() > 1 else 1
    ctx = context(c.device)
    h = ctx.bind()
    par = mp.parent_of.contiguous()
    ctx.check(L.lib().npcg_upsample(h, _dtype_code(c), _ptr(par), n, _ptr(c), c.shape[0], width,
                                    _ptr(out)), "upsample")
    return out


@dataclass
class StridedResult:
    coarse_cloud: PointCloud
    coarse_features: torch.Tensor
    map: DownsampleMap


def strided_block(op: PointConvOp, cloud: PointCloud, fin: torch.Tensor,
                  voxel_size: float) -> StridedResult:
    coarse, mp = voxel_downsample(cloud, voxel_size)
    feats = op.forward(cloud, coarse, fin)
    return StridedResult(coarse, feats, mp)
