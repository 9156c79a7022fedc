// refabi_shim.cpp -- the reference's own hot-path C++ API, implemented over
// libnpcg.so.  Compiled against the UNMODIFIED reference headers
// (/root/reference/proj/core/include/npconv/*.hpp) so that the reference's
// acceptance gate (proj/tests/acceptance.cpp) and doctest suites
// (proj/tests/test_*.cpp) link against the GPU engines instead of
// engine.cpp / vvor.cpp / the search and triplet builders of spatial.cpp and
// triplets.cpp -- the "relink" a reference caller would do.  The reference's
// other translation units (point_cloud, synthetic, io, oracle, gradcheck, and
// the non-hot-path functions of engine / vvor / spatial / triplets, whose hot
// functions are renamed away at compile time) link unchanged.  Built by
// oracle/Makefile into oracle/_ref/ (test infrastructure: it needs the
// reference headers, so it is built only where /root/reference exists).
//
// Replaced functions (reference declaration -> C ABI):
//   spatial.hpp:39-40   radius_search            npcg_radius_search + export_pairs
//   spatial.hpp:47-48   voxel_downsample         npcg_voxel_downsample
//   spatial.hpp:52-54   upsample                 npcg_upsample
//   triplets.hpp:48-49  local_voxel_kernel_index npcg_kernel_index
//   triplets.hpp:56-57  build_triplets_native    npcg_build_triplets_native + export
//   triplets.hpp:63-76  build_triplets_degraded  npcg_build_triplets_degraded + export
//   triplets.hpp:78,82  sort_triplets, choose_sort_axis
//   engine.hpp:66-76    mvmr, mvmr_transposed    npcg_mvmr, npcg_mvmr_transposed
//   vvor.hpp:85-88      vvor                     npcg_vvor
// Access counters (engine.hpp:38-50) describe the CPU executors' memory
// traffic; the GPU engines report zeros (the CPU access model is out of scope).
#include <cuda_runtime.h>

#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "npcg.h"
#include "npconv/engine.hpp"
#include "npconv/errors.hpp"
#include "npconv/spatial.hpp"
#include "npconv/triplets.hpp"
#include "npconv/vvor.hpp"

namespace {

npcg_context* ctx() {
  static npcg_context* c = [] {
    npcg_context* p = nullptr;
    const int dev = std::getenv("NPCG_DEVICE") ? std::atoi(std::getenv("NPCG_DEVICE")) : 0;
    if (npcg_context_create(dev, nullptr, &p) != NPCG_OK)
      throw std::runtime_error("refabi: npcg_context_create failed (a B200 is required)");
    return p;
  }();
  return c;
}

[[noreturn]] void raise(npcg_status s, const std::string& what) {
  const std::string m = what + ": " + npcg_last_error(ctx());
  switch (s) {
    case NPCG_ERR_OFFSET: throw npc::OffsetError(m);
    case NPCG_ERR_NONFINITE: throw npc::NonFiniteError(m);
    case NPCG_ERR_SHAPE: throw npc::ShapeError(m);
    case NPCG_ERR_RADIUS: throw npc::RadiusError(m);
    case NPCG_ERR_VOXEL: throw npc::VoxelError(m);
    case NPCG_ERR_INDEX: throw npc::IndexError(m);
    case NPCG_ERR_DOMAIN: throw npc::DomainError(m);
    case NPCG_ERR_STATE: throw npc::StateError(m);
    case NPCG_ERR_IO: throw npc::IOError(m);
    default: throw std::runtime_error(m + " (" + npcg_status_string(s) + ")");
  }
}
void check(npcg_status s, const char* what) {
  if (s != NPCG_OK) raise(s, what);
}

template <typename T>
class Dev {
 public:
  explicit Dev(size_t n) : n_(n) {
    if (n && cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)) != cudaSuccess)
      throw std::runtime_error("refabi: cudaMalloc failed");
  }
  Dev(const T* h, size_t n) : Dev(n) {
    if (n) cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice);
  }
  ~Dev() {
    if (p_) cudaFree(p_);
  }
  Dev(const Dev&) = delete;
  T* get() const { return p_; }
  std::vector<T> host(size_t n) const {
    std::vector<T> v(n);
    check(npcg_context_synchronize(ctx()), "sync");
    if (n) cudaMemcpy(v.data(), p_, n * sizeof(T), cudaMemcpyDeviceToHost);
    return v;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

struct DevCloud {
  Dev<double> xyz;
  std::vector<int64_t> off;
  npcg_cloud view{};
  explicit DevCloud(const npc::PointCloud& c)
      : xyz(c.positions().empty() ? nullptr : c.positions().data()->data(), 3 * c.positions().size()),
        off(c.batch_offsets().begin(), c.batch_offsets().end()) {
    view = {xyz.get(), off.data(), c.n_points(), c.n_batches()};
  }
};

struct Handle {
  npcg_neighbors* h = nullptr;
  ~Handle() {
    if (h) npcg_neighbors_destroy(h);
  }
};

npc::TripletList export_triplets(const Handle& nb, npc::SortAxis axis) {
  int64_t n = 0, no = 0, ni = 0, nk = 0;
  check(npcg_neighbors_size(nb.h, &n), "size");
  check(npcg_neighbors_info(nb.h, &no, &ni, &nk, nullptr), "info");
  Dev<uint32_t> i(n), j(n), k(n);
  check(npcg_neighbors_export_triplets(ctx(), nb.h, static_cast<int32_t>(axis), i.get(), j.get(), k.get()),
        "export_triplets");
  npc::TripletList t;
  t.i = i.host(n);
  t.j = j.host(n);
  t.k = k.host(n);
  t.n_out = no;
  t.n_in = ni;
  t.n_kernels = nk;
  t.sort_axis = axis;
  return t;
}

struct DevTriplets {
  Dev<uint32_t> i, j, k;
  npcg_triplets view{};
  explicit DevTriplets(const npc::TripletList& t)
      : i(t.i.data(), t.i.size()), j(t.j.data(), t.j.size()), k(t.k.data(), t.k.size()) {
    view = {i.get(), j.get(), k.get(), t.size(), t.n_out, t.n_in, t.n_kernels,
            static_cast<int32_t>(t.sort_axis)};
  }
};

npcg_exec_config cfg_of(const npc::ExecConfig& c) {
  return {c.L, c.b_out, c.b_in, static_cast<int32_t>(c.executor), c.deterministic ? 1 : 0, c.workers,
          NPCG_MATH_AUTO, 0, 0};
}
template <typename T>
constexpr npcg_dtype dtype_of() {
  return std::is_same_v<T, float> ? NPCG_F32 : NPCG_F64;
}

}  // namespace

namespace npc {

NeighborList radius_search(const PointCloud& queries, const PointCloud& targets, double radius) {
  DevCloud q(queries), t(targets);
  Handle nb;
  check(npcg_radius_search(ctx(), &q.view, &t.view, radius, &nb.h), "radius_search");
  int64_t n = 0;
  check(npcg_neighbors_size(nb.h, &n), "size");
  Dev<int64_t> oi(n), ii(n);
  check(npcg_neighbors_export_pairs(ctx(), nb.h, oi.get(), ii.get()), "export_pairs");
  NeighborList out;
  out.out_index = oi.host(n);
  out.in_index = ii.host(n);
  out.radius = radius;
  return out;
}

std::pair<PointCloud, DownsampleMap> voxel_downsample(const PointCloud& cloud, double voxel_size) {
  DevCloud c(cloud);
  const int64_t n = cloud.n_points();
  Dev<int64_t> kept(std::max<int64_t>(n, 1)), parent(std::max<int64_t>(n, 1));
  std::vector<int64_t> off(cloud.n_batches() + 1);
  int64_t nk = 0;
  check(npcg_voxel_downsample(ctx(), &c.view, voxel_size, kept.get(), parent.get(), off.data(), &nk),
        "voxel_downsample");
  DownsampleMap m;
  m.kept_index = kept.host(nk);
  m.parent_of = parent.host(n);
  std::vector<Vec3> pts(nk);
  for (int64_t s = 0; s < nk; ++s) pts[s] = cloud.position(m.kept_index[s]);
  return {PointCloud(std::move(pts), std::move(off)), std::move(m)};
}

template <typename T>
FeatureTensor<T> upsample(const PointCloud& fine, const DownsampleMap& map, const FeatureTensor<T>& coarse) {
  if (static_cast<int64_t>(map.parent_of.size()) != fine.n_points())
    throw ShapeError("upsample: map does not cover the fine cloud");
  if (static_cast<int64_t>(map.kept_index.size()) != coarse.n())
    throw ShapeError("upsample: coarse features do not match the map");
  const int64_t n = fine.n_points(), w = coarse.groups() * coarse.channels();
  FeatureTensor<T> out(n, coarse.groups(), coarse.channels());
  if (n == 0) return out;
  Dev<int64_t> par(map.parent_of.data(), map.parent_of.size());
  Dev<T> dc(coarse.values().data(), coarse.values().size());
  Dev<T> dst(static_cast<size_t>(n * w));
  check(npcg_upsample(ctx(), dtype_of<T>(), par.get(), n, dc.get(), coarse.n(), w, dst.get()), "upsample");
  const auto h = dst.host(static_cast<size_t>(n * w));
  std::copy(h.begin(), h.end(), out.values_mut().begin());
  return out;
}
template FeatureTensor<float> upsample<float>(const PointCloud&, const DownsampleMap&, const FeatureTensor<float>&);
template FeatureTensor<double> upsample<double>(const PointCloud&, const DownsampleMap&,
                                                const FeatureTensor<double>&);

std::int64_t local_voxel_kernel_index(const Vec3& center, const Vec3& neighbor, double radius, std::int64_t t) {
  Dev<double> c(center.data(), 3), nb(neighbor.data(), 3);
  Dev<int64_t> k(1);
  check(npcg_kernel_index(ctx(), c.get(), nb.get(), 1, radius, t, k.get()), "local_voxel_kernel_index");
  return k.host(1)[0];
}

TripletList build_triplets_native(const PointCloud& out_cloud, const PointCloud& in_cloud,
                                  const ConvGeometry& geom) {
  DevCloud o(out_cloud), i(in_cloud);
  Handle nb;
  check(npcg_build_triplets_native(ctx(), &o.view, &i.view, geom.radius, geom.t, &nb.h),
        "build_triplets_native");
  return export_triplets(nb, SortAxis::none);
}

DegradedBuild build_triplets_degraded(const PointCloud& in_cloud, const ConvGeometry& geom) {
  DevCloud c(in_cloud);
  Handle nb;
  check(npcg_build_triplets_degraded(ctx(), &c.view, geom.voxel_size, geom.t, &nb.h), "build_triplets_degraded");
  int64_t ns = 0, nf = 0, nbat = 0;
  check(npcg_neighbors_sites(nb.h, &ns, &nf, &nbat), "sites");
  Dev<double> xyz(std::max<int64_t>(3 * ns, 1));
  Dev<int64_t> kept(std::max<int64_t>(ns, 1)), parent(std::max<int64_t>(nf, 1));
  std::vector<int64_t> off(nbat + 1);
  check(npcg_neighbors_export_sites(ctx(), nb.h, xyz.get(), kept.get(), parent.get(), off.data()),
        "export_sites");
  const auto hx = xyz.host(3 * ns);
  std::vector<Vec3> pts(ns);
  for (int64_t s = 0; s < ns; ++s) pts[s] = {hx[3 * s], hx[3 * s + 1], hx[3 * s + 2]};
  DegradedBuild b;
  b.triplets = export_triplets(nb, SortAxis::none);
  b.snapped = PointCloud(std::move(pts), std::move(off));
  b.sites.kept_index = kept.host(ns);
  b.sites.parent_of = parent.host(nf);
  return b;
}

TripletList sort_triplets(TripletList triplets, SortAxis axis) {
  if (axis == SortAxis::none || triplets.size() <= 1) {  // triplets.cpp:136-139
    triplets.sort_axis = axis;
    return triplets;
  }
  DevTriplets d(triplets);
  const int64_t n = triplets.size();
  Dev<uint32_t> i(n), j(n), k(n);
  check(npcg_sort_triplets(ctx(), &d.view, static_cast<int32_t>(axis), i.get(), j.get(), k.get()),
        "sort_triplets");
  TripletList out;
  out.i = i.host(n);
  out.j = j.host(n);
  out.k = k.host(n);
  out.n_out = triplets.n_out;
  out.n_in = triplets.n_in;
  out.n_kernels = triplets.n_kernels;
  out.sort_axis = axis;
  return out;
}

SortAxis choose_sort_axis(const TripletList& t) {
  return static_cast<SortAxis>(npcg_choose_sort_axis(t.n_out, t.n_in, t.n_kernels));
}

template <typename T>
MvmrResult<T> mvmr(const WeightTensor<T>& weights, const FeatureTensor<T>& fin, const TripletList& triplets,
                   std::int64_t n_out, const ExecConfig& config) {
  if (weights.groups() != fin.groups()) throw ShapeError("mvmr: weight and feature group counts differ");
  if (weights.c_in() != fin.channels()) throw ShapeError("mvmr: weight C_in_g does not match feature channels");
  DevTriplets d(triplets);
  Dev<T> w(weights.values().data(), weights.values().size()), f(fin.values().data(), fin.values().size());
  const int64_t nv = std::max<int64_t>(n_out, 0) * weights.groups() * weights.c_out();
  Dev<T> out(static_cast<size_t>(nv));
  const npcg_exec_config c = cfg_of(config);
  check(npcg_mvmr(ctx(), dtype_of<T>(), w.get(), weights.t(), weights.groups(), weights.c_in(), weights.c_out(),
                  f.get(), fin.n(), &d.view, n_out, &c, out.get()),
        "mvmr");
  MvmrResult<T> r{FeatureTensor<T>(n_out, weights.groups(), weights.c_out()), {}, 0};
  const auto h = out.host(static_cast<size_t>(nv));
  std::copy(h.begin(), h.end(), r.out.values_mut().begin());
  return r;
}

template <typename T>
MvmrResult<T> mvmr_transposed(const WeightTensor<T>& weights, const FeatureTensor<T>& gout,
                              const TripletList& triplets, std::int64_t n_in, const ExecConfig& config) {
  if (weights.c_out() != gout.channels())
    throw ShapeError("mvmr_transposed: weight C_out_g does not match gradient channels");
  if (weights.groups() != gout.groups()) throw ShapeError("mvmr: weight and feature group counts differ");
  DevTriplets d(triplets);
  Dev<T> w(weights.values().data(), weights.values().size()), g(gout.values().data(), gout.values().size());
  const int64_t nv = std::max<int64_t>(n_in, 0) * weights.groups() * weights.c_in();
  Dev<T> out(static_cast<size_t>(nv));
  const npcg_exec_config c = cfg_of(config);
  check(npcg_mvmr_transposed(ctx(), dtype_of<T>(), w.get(), weights.t(), weights.groups(), weights.c_in(),
                             weights.c_out(), g.get(), gout.n(), &d.view, n_in, &c, out.get()),
        "mvmr_transposed");
  MvmrResult<T> r{FeatureTensor<T>(n_in, weights.groups(), weights.c_in()), {}, 0};
  const auto h = out.host(static_cast<size_t>(nv));
  std::copy(h.begin(), h.end(), r.out.values_mut().begin());
  return r;
}

template <typename T>
VvorResult<T> vvor(const FeatureTensor<T>& gout, const FeatureTensor<T>& fin, const TripletList& triplets,
                   std::int64_t n_kernels, const ExecConfig& config) {
  if (gout.groups() != fin.groups()) throw ShapeError("vvor: gradient and feature group counts differ");
  DevTriplets d(triplets);
  Dev<T> g(gout.values().data(), gout.values().size()), f(fin.values().data(), fin.values().size());
  const int64_t nv = std::max<int64_t>(n_kernels, 0) * gout.groups() * gout.channels() * fin.channels();
  Dev<T> grad(static_cast<size_t>(std::max<int64_t>(nv, 1)));
  const npcg_exec_config c = cfg_of(config);
  check(npcg_vvor(ctx(), dtype_of<T>(), g.get(), gout.n(), f.get(), fin.n(), gout.groups(), fin.channels(),
                  gout.channels(), &d.view, n_kernels, &c, grad.get()),
        "vvor");
  VvorResult<T> r{WeightGradient<T>(n_kernels, gout.groups(), gout.channels(), fin.channels()), {}, 0};
  const auto h = grad.host(static_cast<size_t>(nv));
  std::copy(h.begin(), h.end(), r.grad.values_mut().begin());
  return r;
}

template MvmrResult<float> mvmr<float>(const WeightTensor<float>&, const FeatureTensor<float>&,
                                       const TripletList&, std::int64_t, const ExecConfig&);
template MvmrResult<double> mvmr<double>(const WeightTensor<double>&, const FeatureTensor<double>&,
                                         const TripletList&, std::int64_t, const ExecConfig&);
template MvmrResult<float> mvmr_transposed<float>(const WeightTensor<float>&, const FeatureTensor<float>&,
                                                  const TripletList&, std::int64_t, const ExecConfig&);
template MvmrResult<double> mvmr_transposed<double>(const WeightTensor<double>&, const FeatureTensor<double>&,
                                                    const TripletList&, std::int64_t, const ExecConfig&);
template VvorResult<float> vvor<float>(const FeatureTensor<float>&, const FeatureTensor<float>&,
                                       const TripletList&, std::int64_t, const ExecConfig&);
template VvorResult<double> vvor<double>(const FeatureTensor<double>&, const FeatureTensor<double>&,
                                         const TripletList&, std::int64_t, const ExecConfig&);

}  // namespace npc
