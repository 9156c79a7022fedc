// ref_capi.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie (/root/reference/proj/core/src/*.cpp) into
// oracle/_ref/libnpref.so.  It lets the Python test harness and bench.py's
// `--impl reference` arm call the reference's own public API
// (core/include/npconv/*.hpp) with plain pointers.  Nothing here re-implements
// reference behaviour; every function forwards to the npc:: call named in its
// comment.  The B200 product never links this file.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "npconv/conv_op.hpp"
#include "npconv/engine.hpp"
#include "npconv/errors.hpp"
#include "npconv/oracle.hpp"
#include "npconv/point_cloud.hpp"
#include "npconv/spatial.hpp"
#include "npconv/synthetic.hpp"
#include "npconv/tensors.hpp"
#include "npconv/io.hpp"
#include "npconv/triplets.hpp"
#include "npconv/vvor.hpp"

using namespace npc;

namespace {

// Error classes -> npcg status numbering (include/npcg.h).
int status_of(const std::exception& e) {
  if (dynamic_cast<const OffsetError*>(&e)) return 1;
  if (dynamic_cast<const NonFiniteError*>(&e)) return 2;
  if (dynamic_cast<const ShapeError*>(&e)) return 3;
  if (dynamic_cast<const RadiusError*>(&e)) return 4;
  if (dynamic_cast<const VoxelError*>(&e)) return 5;
  if (dynamic_cast<const IndexError*>(&e)) return 6;
  if (dynamic_cast<const DomainError*>(&e)) return 7;
  if (dynamic_cast<const StateError*>(&e)) return 8;
  if (dynamic_cast<const IOError*>(&e)) return 9;
  return 99;
}

PointCloud cloud_of(const double* xyz, const int64_t* off, int64_t nb) {
  const int64_t n = off[nb];
  std::vector<Vec3> pts(static_cast<std::size_t>(n));
  for (int64_t p = 0; p < n; ++p) pts[p] = {xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]};
  return make_point_cloud(std::move(pts), std::vector<int64_t>(off, off + nb + 1));
}

TripletList list_of(const uint32_t* i, const uint32_t* j, const uint32_t* k, int64_t n,
                    int64_t n_out, int64_t n_in, int64_t n_kernels, int axis) {
  TripletList t;
  t.i.assign(i, i + n);
  t.j.assign(j, j + n);
  t.k.assign(k, k + n);
  t.n_out = n_out;
  t.n_in = n_in;
  t.n_kernels = n_kernels;
  t.sort_axis = static_cast<SortAxis>(axis);
  return t;
}

ExecConfig cfg_of(int grouped, int det, int64_t L, int workers) {
  ExecConfig c;
  c.executor = grouped ? Executor::grouped : Executor::naive;
  c.deterministic = det != 0;
  c.L = L;
  c.workers = workers;
  return c;
}

struct RefTriplets {
  TripletList t;
};
struct RefPairs {
  NeighborList nl;
};

}  // namespace

extern "C" {

// std::mt19937_64 raw draws (random.hpp:56) -- pins the oracle's generator.
void ref_mt19937_64_draws(uint64_t seed, int64_t n, uint64_t* out) {
  std::mt19937_64 g(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = g();
}

// synthetic.cpp:12-23
int ref_gen_uniform_cube(int64_t n, double extent, uint64_t seed, double* xyz) {
  try {
    PointCloud c = gen_uniform_cube(n, extent, seed);
    for (int64_t p = 0; p < n; ++p)
      for (int a = 0; a < 3; ++a) xyz[3 * p + a] = c.position(p)[a];
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}

// synthetic.cpp:25-46
int ref_gen_gaussian_clusters(int64_t n, int64_t clusters, double extent, double sigma,
                              uint64_t seed, double* xyz) {
  try {
    PointCloud c = gen_gaussian_clusters(n, clusters, extent, sigma, seed);
    for (int64_t p = 0; p < n; ++p)
      for (int a = 0; a < 3; ++a) xyz[3 * p + a] = c.position(p)[a];
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}

// synthetic.cpp:48-81
int ref_gen_grid_snapped(int64_t n, int64_t cells, double voxel, uint64_t seed, double* xyz) {
  try {
    PointCloud c = gen_grid_snapped(n, cells, voxel, seed);
    for (int64_t p = 0; p < n; ++p)
      for (int a = 0; a < 3; ++a) xyz[3 * p + a] = c.position(p)[a];
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}

// synthetic.hpp:33-40
void ref_gen_features_f32(int64_t n, int64_t g, int64_t c, uint64_t seed, float* out) {
  FeatureTensor<float> f = gen_features<float>(n, g, c, seed);
  std::memcpy(out, f.values().data(), f.values().size() * sizeof(float));
}
void ref_gen_features_f64(int64_t n, int64_t g, int64_t c, uint64_t seed, double* out) {
  FeatureTensor<double> f = gen_features<double>(n, g, c, seed);
  std::memcpy(out, f.values().data(), f.values().size() * sizeof(double));
}

// tensors.hpp:142-150
void ref_make_weights_f32(int64_t t, int64_t g, int64_t ci, int64_t co, uint64_t seed,
                          float* out) {
  WeightTensor<float> w = make_weights<float>(t, g, ci, co, seed);
  std::memcpy(out, w.values().data(), w.values().size() * sizeof(float));
}
void ref_make_weights_f64(int64_t t, int64_t g, int64_t ci, int64_t co, uint64_t seed,
                          double* out) {
  WeightTensor<double> w = make_weights<double>(t, g, ci, co, seed);
  std::memcpy(out, w.values().data(), w.values().size() * sizeof(double));
}

// spatial.hpp:39-40 radius_search
int ref_radius_search(const double* q, const int64_t* qo, int64_t qnb, const double* t,
                      const int64_t* to, int64_t tnb, double r, void** out) {
  try {
    auto* h = new RefPairs{radius_search(cloud_of(q, qo, qnb), cloud_of(t, to, tnb), r)};
    *out = h;
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}
int ref_brute_radius(const double* q, const int64_t* qo, int64_t qnb, const double* t,
                     const int64_t* to, int64_t tnb, double r, void** out) {
  try {
    auto* h = new RefPairs{
        oracle::brute_radius_oracle(cloud_of(q, qo, qnb), cloud_of(t, to, tnb), r)};
    *out = h;
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}
int64_t ref_pairs_size(void* h) { return static_cast<RefPairs*>(h)->nl.size(); }
void ref_pairs_copy(void* h, int64_t* oi, int64_t* ii) {
  auto* p = static_cast<RefPairs*>(h);
  std::memcpy(oi, p->nl.out_index.data(), p->nl.out_index.size() * sizeof(int64_t));
  std::memcpy(ii, p->nl.in_index.data(), p->nl.in_index.size() * sizeof(int64_t));
}
void ref_pairs_free(void* h) { delete static_cast<RefPairs*>(h); }

// triplets.hpp:48-49
int64_t ref_kernel_index(const double* c, const double* nb, double r, int64_t t) {
  try {
    return local_voxel_kernel_index({c[0], c[1], c[2]}, {nb[0], nb[1], nb[2]}, r, t);
  } catch (const std::exception& e) { return -status_of(e); }
}

// triplets.hpp:56-57 build_triplets_native, optionally followed by
// sort_triplets(axis) (axis < 0: choose_sort_axis, as PointConvOp does).
int ref_build_triplets(const double* outp, const int64_t* oo, int64_t onb, const double* inp,
                       const int64_t* io, int64_t inb, double r, int64_t t, int axis,
                       void** out) {
  try {
    ConvGeometry g;
    g.radius = r;
    g.t = t;
    TripletList tl = build_triplets_native(cloud_of(outp, oo, onb), cloud_of(inp, io, inb), g);
    if (axis != 0) {
      const SortAxis a = axis < 0 ? choose_sort_axis(tl) : static_cast<SortAxis>(axis);
      tl = sort_triplets(std::move(tl), a);
    }
    *out = new RefTriplets{std::move(tl)};
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}
int64_t ref_triplets_size(void* h) { return static_cast<RefTriplets*>(h)->t.size(); }
int ref_triplets_axis(void* h) { return static_cast<int>(static_cast<RefTriplets*>(h)->t.sort_axis); }
void ref_triplets_copy(void* h, uint32_t* i, uint32_t* j, uint32_t* k) {
  auto& t = static_cast<RefTriplets*>(h)->t;
  std::memcpy(i, t.i.data(), t.i.size() * 4);
  std::memcpy(j, t.j.data(), t.j.size() * 4);
  std::memcpy(k, t.k.data(), t.k.size() * 4);
}
void ref_triplets_free(void* h) { delete static_cast<RefTriplets*>(h); }

// triplets.hpp:78 sort_triplets
int ref_sort_triplets(const uint32_t* i, const uint32_t* j, const uint32_t* k, int64_t n,
                      int64_t n_out, int64_t n_in, int64_t nk, int axis, uint32_t* oi,
                      uint32_t* oj, uint32_t* ok) {
  try {
    TripletList s = sort_triplets(list_of(i, j, k, n, n_out, n_in, nk, 0),
                                  static_cast<SortAxis>(axis));
    std::memcpy(oi, s.i.data(), n * 4);
    std::memcpy(oj, s.j.data(), n * 4);
    std::memcpy(ok, s.k.data(), n * 4);
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}

// engine.hpp:66-76 mvmr / mvmr_transposed; vvor.hpp:85-88 vvor.
#define NPREF_ENGINES(T, SUF)                                                              \
  int ref_mvmr_##SUF(const T* w, int64_t t, int64_t G, int64_t ci, int64_t co, const T* f,  \
                     int64_t n_in, const uint32_t* i, const uint32_t* j, const uint32_t* k, \
                     int64_t n, int64_t tl_out, int64_t tl_in, int64_t n_out, int grouped,   \
                     int det, int64_t L, int workers, T* out) {                            \
    try {                                                                                  \
      WeightTensor<T> W(t, G, ci, co, std::vector<T>(w, w + t * t * t * G * ci * co));    \
      FeatureTensor<T> F(n_in, G, ci, std::vector<T>(f, f + n_in * G * ci));               \
      auto r = mvmr(W, F, list_of(i, j, k, n, tl_out, tl_in, t * t * t, 0), n_out,         \
                    cfg_of(grouped, det, L, workers));                                     \
      std::memcpy(out, r.out.values().data(), r.out.values().size() * sizeof(T));          \
      return 0;                                                                            \
    } catch (const std::exception& e) { return status_of(e); }                             \
  }                                                                                        \
  int ref_mvmr_transposed_##SUF(const T* w, int64_t t, int64_t G, int64_t ci, int64_t co,   \
                                const T* g, int64_t n_go, const uint32_t* i,               \
                                const uint32_t* j, const uint32_t* k, int64_t n,           \
                                int64_t tl_out, int64_t tl_in, int64_t n_in, int grouped,   \
                                int det, int64_t L, int workers, T* out) {                 \
    try {                                                                                  \
      WeightTensor<T> W(t, G, ci, co, std::vector<T>(w, w + t * t * t * G * ci * co));    \
      FeatureTensor<T> Go(n_go, G, co, std::vector<T>(g, g + n_go * G * co));              \
      auto r = mvmr_transposed(W, Go, list_of(i, j, k, n, tl_out, tl_in, t * t * t, 0),    \
                               n_in, cfg_of(grouped, det, L, workers));                    \
      std::memcpy(out, r.out.values().data(), r.out.values().size() * sizeof(T));          \
      return 0;                                                                            \
    } catch (const std::exception& e) { return status_of(e); }                             \
  }                                                                                        \
  int ref_vvor_##SUF(const T* g, int64_t n_go, const T* f, int64_t n_in, int64_t G,        \
                     int64_t ci, int64_t co, const uint32_t* i, const uint32_t* j,          \
                     const uint32_t* k, int64_t n, int64_t tl_out, int64_t tl_in,           \
                     int64_t nk, int grouped, int det, int64_t L, int workers, T* out) {    \
    try {                                                                                  \
      FeatureTensor<T> Go(n_go, G, co, std::vector<T>(g, g + n_go * G * co));              \
      FeatureTensor<T> F(n_in, G, ci, std::vector<T>(f, f + n_in * G * ci));               \
      auto r = vvor(Go, F, list_of(i, j, k, n, tl_out, tl_in, nk, 0), nk,                  \
                    cfg_of(grouped, det, L, workers));                                     \
      std::memcpy(out, r.grad.values().data(), r.grad.values().size() * sizeof(T));        \
      return 0;                                                                            \
    } catch (const std::exception& e) { return status_of(e); }                             \
  }
NPREF_ENGINES(float, f32)
NPREF_ENGINES(double, f64)

// oracle.hpp:27-30 dense_conv_oracle (fp64), with gradients when gout != NULL.
int ref_dense_oracle(const double* w, int64_t t, int64_t G, int64_t ci, int64_t co,
                     const double* f, int64_t n_in, const uint32_t* i, const uint32_t* j,
                     const uint32_t* k, int64_t n, int64_t tl_out, int64_t tl_in, int64_t n_out,
                     const double* gout, double* fout, double* gin, double* gw) {
  try {
    WeightTensor<double> W(t, G, ci, co, std::vector<double>(w, w + t * t * t * G * ci * co));
    FeatureTensor<double> F(n_in, G, ci, std::vector<double>(f, f + n_in * G * ci));
    std::vector<double> gv;
    FeatureTensor<double> Go;
    if (gout) Go = FeatureTensor<double>(n_out, G, co, std::vector<double>(gout, gout + n_out * G * co));
    auto r = oracle::dense_conv_oracle(W, F, list_of(i, j, k, n, tl_out, tl_in, t * t * t, 0),
                                       n_out, gout ? &Go : nullptr);
    std::memcpy(fout, r.f_out.values().data(), r.f_out.values().size() * sizeof(double));
    if (gout) {
      std::memcpy(gin, r.grad_in->values().data(), r.grad_in->values().size() * sizeof(double));
      std::memcpy(gw, r.grad_w->values().data(), r.grad_w->values().size() * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}

// spatial.hpp:52-54 upsample (the reference checks the map against the cloud
// and the coarse tensor, then copies rows through parent_of)
#define NPREF_UPSAMPLE(T, SUF)                                                              \
  int ref_upsample_##SUF(const double* xyz, const int64_t* off, int64_t nb, const int64_t* kept, \
                         int64_t n_kept, const int64_t* parent, const T* coarse, int64_t G,    \
                         int64_t C, T* out) {                                                 \
    try {                                                                                    \
      const PointCloud fine = cloud_of(xyz, off, nb);                                        \
      DownsampleMap m;                                                                       \
      m.kept_index.assign(kept, kept + n_kept);                                              \
      m.parent_of.assign(parent, parent + fine.n_points());                                  \
      FeatureTensor<T> c(n_kept, G, C, std::vector<T>(coarse, coarse + n_kept * G * C));     \
      auto r = upsample(fine, m, c);                                                         \
      std::memcpy(out, r.values().data(), r.values().size() * sizeof(T));                    \
      return 0;                                                                              \
    } catch (const std::exception& e) { return status_of(e); }                               \
  }
NPREF_UPSAMPLE(float, f32)
NPREF_UPSAMPLE(double, f64)

// spatial.hpp:47-48 voxel_downsample
int64_t ref_voxel_downsample(const double* xyz, const int64_t* off, int64_t nb, double v,
                             int64_t* kept, int64_t* parent, int64_t* out_off) {
  try {
    auto [down, map] = voxel_downsample(cloud_of(xyz, off, nb), v);
    std::memcpy(kept, map.kept_index.data(), map.kept_index.size() * 8);
    std::memcpy(parent, map.parent_of.data(), map.parent_of.size() * 8);
    auto o = down.batch_offsets();
    std::memcpy(out_off, o.data(), o.size() * 8);
    return down.n_points();
  } catch (const std::exception& e) { return -status_of(e); }
}

// triplets.hpp:63-76 build_triplets_degraded (ConvMode::degraded geometry)
int64_t ref_build_triplets_degraded(const double* xyz, const int64_t* off, int64_t nb, double v,
                                    int64_t t, double* snapped, int64_t* kept, int64_t* parent,
                                    int64_t* site_off, void** out) {
  try {
    ConvGeometry g;
    g.mode = ConvMode::degraded;
    g.voxel_size = v;
    g.t = t;
    DegradedBuild b = build_triplets_degraded(cloud_of(xyz, off, nb), g);
    const int64_t ns = b.snapped.n_points();
    for (int64_t s = 0; s < ns; ++s)
      for (int a = 0; a < 3; ++a) snapped[3 * s + a] = b.snapped.position(s)[a];
    std::memcpy(kept, b.sites.kept_index.data(), b.sites.kept_index.size() * 8);
    std::memcpy(parent, b.sites.parent_of.data(), b.sites.parent_of.size() * 8);
    auto o = b.snapped.batch_offsets();
    std::memcpy(site_off, o.data(), o.size() * 8);
    *out = new RefTriplets{std::move(b.triplets)};
    return ns;
  } catch (const std::exception& e) { return -status_of(e); }
}

// io.hpp / triplets.hpp:84-93 file formats (NPC1, XYZ, TPL1), through the
// reference's own writers / readers
int ref_write_cloud(const char* path, const double* xyz, const int64_t* off, int64_t nb) {
  try {
    write_cloud(path, cloud_of(xyz, off, nb));
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}
// Returns the point count (xyz / off sized by the caller: query with xyz == NULL
// first, which also returns the batch count through *nb).
int64_t ref_read_cloud(const char* path, double* xyz, int64_t* off, int64_t* nb) {
  try {
    PointCloud c = read_cloud(path);
    *nb = c.n_batches();
    if (xyz) {
      for (int64_t p = 0; p < c.n_points(); ++p)
        for (int a = 0; a < 3; ++a) xyz[3 * p + a] = c.position(p)[a];
      auto o = c.batch_offsets();
      std::memcpy(off, o.data(), o.size() * 8);
    }
    return c.n_points();
  } catch (const std::exception& e) { return -status_of(e); }
}
int ref_write_triplets(const char* path, const uint32_t* i, const uint32_t* j, const uint32_t* k,
                       int64_t n, int64_t n_out, int64_t n_in, int64_t nk, int axis) {
  try {
    TripletList t;
    t.i.assign(i, i + n);
    t.j.assign(j, j + n);
    t.k.assign(k, k + n);
    t.n_out = n_out;
    t.n_in = n_in;
    t.n_kernels = nk;
    t.sort_axis = static_cast<SortAxis>(axis);
    write_triplets(path, t);
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}
// meta[0..4] = size, n_out, n_in, n_kernels, axis; arrays filled when i != NULL
int ref_read_triplets(const char* path, uint32_t* i, uint32_t* j, uint32_t* k, int64_t* meta) {
  try {
    TripletList t = read_triplets(path);
    meta[0] = t.size();
    meta[1] = t.n_out;
    meta[2] = t.n_in;
    meta[3] = t.n_kernels;
    meta[4] = static_cast<int64_t>(t.sort_axis);
    if (i) {
      std::memcpy(i, t.i.data(), t.i.size() * 4);
      std::memcpy(j, t.j.data(), t.j.size() * 4);
      std::memcpy(k, t.k.data(), t.k.size() * 4);
    }
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}

// The reference's own conv-layer chain, timed with steady_clock exactly as
// SURVEY.md §8d prescribes: build_triplets_native -> sort_triplets(by_k) ->
// mvmr -> mvmr_transposed -> vvor (ExecConfig{grouped, L=128,
// deterministic=false, workers}).  times[0..4] = build, sort, fwd, dgrad, wgrad
// in seconds.  `build` < 0 skips the geometry (pre-built triplets reused, the
// PointConvOp cache-hit case) and only runs the three engines.
int ref_conv_layer_f32(const double* xyz, int64_t n, double r, int64_t t, int64_t ci,
                       int64_t co, const float* w, const float* f, const float* gout,
                       int workers, int build, double* times, float* fout, float* gin,
                       float* gw, void** cache) {
  try {
    using Clk = std::chrono::steady_clock;
    auto secs = [](Clk::time_point a) {
      return std::chrono::duration<double>(Clk::now() - a).count();
    };
    ExecConfig cfg = cfg_of(1, 0, 128, workers);
    RefTriplets* cached = cache ? static_cast<RefTriplets*>(*cache) : nullptr;
    TripletList sorted;
    if (build || !cached) {
      const int64_t off[2] = {0, n};
      PointCloud c = cloud_of(xyz, off, 1);
      ConvGeometry g;
      g.radius = r;
      g.t = t;
      auto t0 = Clk::now();
      TripletList tl = build_triplets_native(c, c, g);
      times[0] = secs(t0);
      t0 = Clk::now();
      sorted = sort_triplets(std::move(tl), choose_sort_axis(tl));
      times[1] = secs(t0);
      if (cache) {
        delete cached;
        *cache = new RefTriplets{sorted};
      }
    } else {
      sorted = cached->t;
      times[0] = times[1] = 0.0;
    }
    WeightTensor<float> W(t, 1, ci, co, std::vector<float>(w, w + t * t * t * ci * co));
    FeatureTensor<float> F(n, 1, ci, std::vector<float>(f, f + n * ci));
    FeatureTensor<float> G(n, 1, co, std::vector<float>(gout, gout + n * co));
    auto t0 = Clk::now();
    auto a = mvmr(W, F, sorted, n, cfg);
    times[2] = secs(t0);
    t0 = Clk::now();
    auto b = mvmr_transposed(W, G, sorted, n, cfg);
    times[3] = secs(t0);
    t0 = Clk::now();
    auto c = vvor(G, F, sorted, W.kernels(), cfg);
    times[4] = secs(t0);
    if (fout) std::memcpy(fout, a.out.values().data(), n * co * sizeof(float));
    if (gin) std::memcpy(gin, b.out.values().data(), n * ci * sizeof(float));
    if (gw) std::memcpy(gw, c.grad.values().data(), c.grad.values().size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) { return status_of(e); }
}
void ref_conv_cache_free(void* h) { delete static_cast<RefTriplets*>(h); }

int ref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
