// C++ parity test of the drop-in header include/npcg/npconv.hpp: reference-style
// test cases (transcribed from /root/reference/proj/tests, cited per case)
// written against the `npc::` API, checked against the C oracle
// (oracle/npc_oracle.c) where a reference value is computed.
#include <cmath>
#include <cstdio>
#include <set>
#include <utility>
#include <vector>

#include "npcg/npconv.hpp"

extern "C" {  // oracle/npc_oracle.c (test infrastructure)
void orc_gen_uniform_cube(int64_t n, double extent, uint64_t seed, double* xyz);
void orc_gen_features_f64(int64_t count, uint64_t seed, double* out);
void orc_make_weights_f64(int64_t t, int64_t g, int64_t cin, int64_t cout, uint64_t seed, double* out);
int orc_dense_conv(const double* w, int64_t K, int64_t G, int64_t cin, int64_t cout, const double* fin,
                   int64_t n_in, const uint32_t* ti, const uint32_t* tj, const uint32_t* tk, int64_t n_t,
                   int64_t n_out, const double* gout, double* fout, double* grad_in, double* grad_w);
}

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(c)) {                                                         \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);          \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, E)                                        \
  do {                                                                  \
    ++g_checks;                                                         \
    bool ok_ = false;                                                   \
    try {                                                               \
      (void)(expr);                                                     \
    } catch (const E&) {                                                \
      ok_ = true;                                                       \
    } catch (...) {                                                     \
    }                                                                   \
    if (!ok_) {                                                         \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d  %s does not throw %s\n", __FILE__, __LINE__, #expr, #E); \
    }                                                                   \
  } while (0)

using namespace npc;

static double rel(std::span<const double> a, const std::vector<double>& b) {
  double md = 0, mr = 0;
  for (size_t i = 0; i < b.size(); ++i) {
    md = std::max(md, std::fabs(a[i] - b[i]));
    mr = std::max(mr, std::fabs(b[i]));
  }
  return md / std::max(mr, 1e-30);
}

int main() {
  // test_spatial.cpp:39-53 radius search on collinear points
  {
    PointCloud c = make_point_cloud({{0, 0, 0}, {1, 0, 0}, {2, 0, 0}});
    NeighborList nl = radius_search(c, c, 1.5);
    std::set<std::pair<int64_t, int64_t>> s, want = {{0, 0}, {0, 1}, {1, 0}, {1, 1}, {1, 2}, {2, 1}, {2, 2}};
    for (int64_t r = 0; r < nl.size(); ++r) s.insert({nl.out_index[r], nl.in_index[r]});
    CHECK(s == want);
    CHECK(nl.radius == 1.5);
  }
  // test_spatial.cpp:56-93 edge cases
  {
    PointCloud c = make_point_cloud({{0, 0, 0}});
    CHECK_THROWS_AS(radius_search(c, c, 0.0), RadiusError);
    CHECK_THROWS_AS(radius_search(c, c, -1.0), RadiusError);
    CHECK(radius_search(make_point_cloud({{0, 0, 0}}), make_point_cloud({{1, 0, 0}}), 1.0).size() == 1);
    PointCloud q = make_point_cloud({{0, 0, 0}, {1, 1, 1}}, {0, 1, 2});
    CHECK_THROWS_AS(radius_search(q, c, 1.0), ShapeError);
    CHECK_THROWS_AS(make_point_cloud({{0, 0, 0}}, {0, 2}), OffsetError);
  }
  // test_triplets.cpp:45-69 local voxel kernel index
  {
    CHECK(local_voxel_kernel_index({0, 0, 0}, {0, 0, 0}, 1.0, 3) == 13);
    CHECK(local_voxel_kernel_index({0, 0, 0}, {0, 0, 0}, 1.0, 5) == 62);
    CHECK(local_voxel_kernel_index({0, 0, 0}, {0.4, 0, 0}, 0.6, 3) == 22);
    CHECK(local_voxel_kernel_index({0, 0, 0}, {1.0, 1.0, 1.0}, 1.0, 3) == 26);
    CHECK(local_voxel_kernel_index({0, 0, 0}, {-1.0, -1.0, -1.0}, 1.0, 3) == 0);
    CHECK_THROWS_AS(local_voxel_kernel_index({0, 0, 0}, {0, 0, 0}, 1.0, 2), ShapeError);
  }
  // test_triplets.cpp:89-101 native build on collinear points
  {
    ConvGeometry g;
    g.radius = 1.5;
    PointCloud c = make_point_cloud({{0, 0, 0}, {1, 0, 0}, {2, 0, 0}});
    TripletList t = build_triplets_native(c, c, g);
    CHECK(t.size() == 7);
    for (int64_t n = 0; n < t.size(); ++n)
      if (t.i[n] == 1 && t.j[n] == 0) CHECK(t.k[n] == 4);
    CHECK(t.sort_axis == SortAxis::none);
  }
  // test_triplets.cpp:218-258 sort stability
  {
    TripletList u;
    u.i = {0, 1, 2, 3};
    u.j = {9, 9, 9, 9};
    u.k = {1, 0, 1, 0};
    u.n_out = 4;
    u.n_in = 10;
    u.n_kernels = 2;
    TripletList s = sort_triplets(u, SortAxis::by_k);
    CHECK((s.i == std::vector<uint32_t>{1, 3, 0, 2}));
    CHECK((s.k == std::vector<uint32_t>{0, 0, 1, 1}));
    CHECK(choose_sort_axis(s) == SortAxis::by_k);
  }
  // test_engine.cpp:75-115 MVMR hand cases
  {
    WeightTensor<double> w(1, 1, 2, 2);
    w.at(0, 0, 0, 0) = 1.0;
    w.at(0, 0, 1, 1) = 1.0;
    TripletList t;
    t.i = {0, 0};
    t.j = {0, 1};
    t.k = {0, 0};
    t.n_out = 1;
    t.n_in = 2;
    t.n_kernels = 1;
    FeatureTensor<double> f(2, 1, 2, {1.0, 2.0, 3.0, 4.0});
    auto r = mvmr(w, f, t, 1);
    CHECK(r.out.at(0, 0, 0) == 4.0 && r.out.at(0, 0, 1) == 6.0);
    WeightTensor<double> w2(1, 1, 2, 2, {1.0, 3.0, 2.0, 4.0});
    TripletList t1 = t;
    t1.i = {0};
    t1.j = {0};
    t1.k = {0};
    t1.n_in = 1;
    auto g = mvmr_transposed(w2, FeatureTensor<double>(1, 1, 2, {1.0, 1.0}), t1, 1);
    CHECK(g.out.at(0, 0, 0) == 4.0 && g.out.at(0, 0, 1) == 6.0);
    ExecConfig bad;
    bad.L = 0;
    CHECK_THROWS_AS(mvmr(w, f, t, 1, bad), ShapeError);
    TripletList oob = t1;
    oob.k = {5};
    CHECK_THROWS_AS(mvmr(w, f, oob, 1), IndexError);  // n_kernels matches, k out of range
  }
  // PointConvOp forward/backward vs the fp64 dense oracle (exact and bf16 math)
  {
    const int64_t n = 3000;
    std::vector<double> xyz(3 * n);
    orc_gen_uniform_cube(n, 1.0, 7, xyz.data());
    std::vector<Vec3> pts(n);
    for (int64_t p = 0; p < n; ++p) pts[p] = {xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]};
    PointCloud c = make_point_cloud(pts);
    const double r = 1.8 * std::pow(static_cast<double>(n), -1.0 / 3.0);
    std::vector<double> wv(27 * 64 * 64), fv(n * 64), gv(n * 64);
    orc_make_weights_f64(3, 1, 64, 64, 2, wv.data());
    orc_gen_features_f64(n * 64, 3, fv.data());
    orc_gen_features_f64(n * 64, 4, gv.data());
    ConvGeometry geo;
    geo.radius = r;
    TripletList tl = build_triplets_native(c, c, geo);
    std::vector<double> fo(n * 64), gi(n * 64), gw(27 * 64 * 64);
    CHECK(orc_dense_conv(wv.data(), 27, 1, 64, 64, fv.data(), n, tl.i.data(), tl.j.data(), tl.k.data(),
                         tl.size(), n, gv.data(), fo.data(), gi.data(), gw.data()) == 0);
    for (npcg_math m : {NPCG_MATH_EXACT, NPCG_MATH_BF16}) {
      ExecConfig cfg;
      cfg.math = m;
      const double tol = m == NPCG_MATH_EXACT ? 1e-12 : 1e-2;
      if (m == NPCG_MATH_EXACT) {
        PointConvOp<double> op(WeightTensor<double>(3, 1, 64, 64, wv), geo, cfg);
        CHECK_THROWS_AS(op.backward(FeatureTensor<double>(n, 1, 64)), StateError);
        auto out = op.forward(c, FeatureTensor<double>(n, 1, 64, fv));
        auto res = op.backward(FeatureTensor<double>(n, 1, 64, gv));
        CHECK(rel(out.values(), fo) <= tol);
        CHECK(rel(res.grad_in.values(), gi) <= tol);
        CHECK(rel(res.grad_w.values(), gw) <= tol);
        CHECK(op.cached_triplets().sort_axis == SortAxis::by_k);
      } else {
        std::vector<float> wf(wv.begin(), wv.end()), ff(fv.begin(), fv.end()), gf(gv.begin(), gv.end());
        PointConvOp<float> op(WeightTensor<float>(3, 1, 64, 64, wf), geo, cfg);
        auto out = op.forward(c, FeatureTensor<float>(n, 1, 64, ff));
        auto res = op.backward(FeatureTensor<float>(n, 1, 64, gf));
        std::vector<double> o(out.values().begin(), out.values().end()),
            a(res.grad_in.values().begin(), res.grad_in.values().end()),
            b(res.grad_w.values().begin(), res.grad_w.values().end());
        CHECK(rel(o, fo) <= tol);
        CHECK(rel(a, gi) <= tol);
        CHECK(rel(b, gw) <= tol);
      }
    }
  }
  std::printf("drop-in: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
