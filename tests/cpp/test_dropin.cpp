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
  // degraded (voxel) mode: test_triplets.cpp:154-215, test_conv_op.cpp:133-175
  {
    ConvGeometry dg;
    dg.mode = ConvMode::degraded;
    dg.voxel_size = 1.0;
    DegradedBuild b = build_triplets_degraded(make_point_cloud({{0.25, 0.25, 0.25}}), dg);
    CHECK(b.triplets.size() == 1 && b.triplets.k[0] == 13);
    CHECK((b.snapped.position(0) == Vec3{0.5, 0.5, 0.5}));
    b = build_triplets_degraded(make_point_cloud({{0.5, 0.5, 0.5}, {1.5, 0.5, 0.5}}), dg);
    std::vector<uint32_t> ks = b.triplets.k;
    std::sort(ks.begin(), ks.end());
    CHECK((ks == std::vector<uint32_t>{4, 13, 13, 22}));
    b = build_triplets_degraded(make_point_cloud({{0.2, 0.2, 0.2}, {0.8, 0.8, 0.8}, {5, 5, 5}}), dg);
    CHECK(b.snapped.n_points() == 2 && b.sites.parent_of[0] == b.sites.parent_of[1]);
    CHECK(b.sites.parent_of[2] != b.sites.parent_of[0]);
    ConvGeometry bad = dg;
    bad.voxel_size = 0.0;
    CHECK_THROWS_AS(build_triplets_degraded(make_point_cloud({{0, 0, 0}}), bad), VoxelError);
    bad = dg;
    bad.t = 4;
    CHECK_THROWS_AS(build_triplets_degraded(make_point_cloud({{0, 0, 0}}), bad), ShapeError);
    // degraded PointConvOp: gather representative rows, scatter gradients back
    PointCloud cloud = make_point_cloud({{0.2, 0.2, 0.2}, {0.3, 0.3, 0.3}, {5, 5, 5}});
    std::vector<double> wv(27 * 2 * 3), fv(3 * 2), gv(2 * 3);
    orc_make_weights_f64(3, 1, 2, 3, 351, wv.data());
    orc_gen_features_f64(6, 352, fv.data());
    orc_gen_features_f64(6, 353, gv.data());
    ExecConfig cfg;
    cfg.deterministic = true;
    PointConvOp<double> op(WeightTensor<double>(3, 1, 2, 3, wv), dg, cfg);
    CHECK_THROWS_AS(op.snapped_cloud(), StateError);
    auto out = op.forward(cloud, FeatureTensor<double>(3, 1, 2, fv));
    CHECK(op.snapped_cloud().n_points() == 2 && out.n() == 2);
    const auto& kept = op.site_map().kept_index;
    std::vector<double> sf(2 * 2);
    for (int m = 0; m < 2; ++m)
      for (int c = 0; c < 2; ++c) sf[2 * m + c] = fv[2 * kept[m] + c];
    const TripletList& tl = op.cached_triplets();
    std::vector<double> fo(2 * 3), gi(2 * 2), gw(27 * 3 * 2);
    CHECK(orc_dense_conv(wv.data(), 27, 1, 2, 3, sf.data(), 2, tl.i.data(), tl.j.data(), tl.k.data(),
                         tl.size(), 2, gv.data(), fo.data(), gi.data(), gw.data()) == 0);
    CHECK(rel(out.values(), fo) <= 1e-13);
    auto res = op.backward(FeatureTensor<double>(2, 1, 3, gv));
    CHECK(res.grad_in.n() == 3);
    for (int p = 0; p < 3; ++p) {
      const bool rep = p == kept[0] || p == kept[1];
      const double mag = std::abs(res.grad_in.at(p, 0, 0)) + std::abs(res.grad_in.at(p, 0, 1));
      CHECK(rep ? mag > 0.0 : mag == 0.0);
    }
    CHECK(rel(res.grad_w.values(), gw) <= 1e-13);
    CHECK_THROWS_AS(op.forward(cloud, cloud, FeatureTensor<double>(3, 1, 2, fv)), StateError);
  }
  // voxel_downsample + file formats (io.hpp; triplets.hpp:84-93)
  {
    PointCloud c = make_point_cloud({{0.1, 0.1, 0.1}, {0.2, 0.2, 0.2}, {3, 3, 3}, {0.5, 0.5, 0.5}}, {0, 3, 4});
    auto [coarse, map] = voxel_downsample(c, 1.0);
    CHECK(coarse.n_points() == 3 && coarse.n_batches() == 2 && map.parent_of.size() == 4);
    CHECK(map.parent_of[0] == map.parent_of[1]);
    const std::string dir = "/tmp";
    write_cloud(dir + "/npcg_dropin.npc", c);
    PointCloud r = read_cloud(dir + "/npcg_dropin.npc");
    CHECK(r.n_points() == 4 && r.n_batches() == 2 && r.position(2)[0] == 3.0);
    write_cloud(dir + "/npcg_dropin.xyz", c);
    PointCloud x = read_cloud(dir + "/npcg_dropin.xyz");
    CHECK(x.n_points() == 4 && x.n_batches() == 1 && x.position(1)[2] == 0.2);
    TripletList t = build_triplets_native(c, c, ConvGeometry{0.5, 3});
    write_triplets(dir + "/npcg_dropin.tpl", t);
    TripletList u = read_triplets(dir + "/npcg_dropin.tpl");
    CHECK(u.i == t.i && u.j == t.j && u.k == t.k && u.n_out == t.n_out && u.n_kernels == 27);
    {
      std::ofstream bad(dir + "/npcg_dropin_bad.npc", std::ios::binary);
      bad.write("NPC2", 4);
    }
    CHECK_THROWS_AS(read_npc(dir + "/npcg_dropin_bad.npc"), IOError);
    TripletList oob = t;
    oob.n_out = 1;
    write_triplets(dir + "/npcg_dropin_oob.tpl", oob);
    CHECK_THROWS_AS(read_triplets(dir + "/npcg_dropin_oob.tpl"), IOError);
  }
  // strided_block + upsample (conv_op.hpp:219-225; spatial.cpp:154-169)
  {
    const int64_t n = 3000;
    std::vector<double> xyz(3 * n);
    orc_gen_uniform_cube(n, 1.0, 21, xyz.data());
    std::vector<Vec3> pts(n);
    for (int64_t p = 0; p < n; ++p) pts[p] = {xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2]};
    PointCloud c = make_point_cloud(std::move(pts));
    const double v = 0.1, r = 1.8 * v;
    std::vector<double> wv(27 * 4 * 6), fv(n * 4);
    orc_make_weights_f64(3, 1, 4, 6, 22, wv.data());
    orc_gen_features_f64(n * 4, 23, fv.data());
    PointConvOp<double> op(WeightTensor<double>(3, 1, 4, 6, wv), ConvGeometry{r, 3});
    auto sr = strided_block(op, c, FeatureTensor<double>(n, 1, 4, fv), v);
    auto [coarse, map] = voxel_downsample(c, v);
    CHECK(sr.coarse_cloud.n_points() == coarse.n_points() && sr.map.kept_index == map.kept_index);
    TripletList t = build_triplets_native(coarse, c, ConvGeometry{r, 3});
    std::vector<double> fo(coarse.n_points() * 6);
    CHECK(orc_dense_conv(wv.data(), 27, 1, 4, 6, fv.data(), n, t.i.data(), t.j.data(), t.k.data(), t.size(),
                         coarse.n_points(), nullptr, fo.data(), nullptr, nullptr) == 0);
    CHECK(rel(sr.coarse_features.values(), fo) <= 1e-12);
    auto up = upsample(c, sr.map, sr.coarse_features);
    bool same = up.n() == n;
    for (int64_t p = 0; same && p < n; ++p)
      for (int64_t q = 0; q < 6; ++q)
        same &= up.at(p, 0, q) == sr.coarse_features.at(sr.map.parent_of[p], 0, q);
    CHECK(same);
    DownsampleMap bad = sr.map;
    bad.parent_of.pop_back();
    CHECK_THROWS_AS(upsample(c, bad, sr.coarse_features), ShapeError);
  }
  std::printf("drop-in: %d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
