// End-to-end timing through the torch-free C++ drop-in (include/npcg/npconv.hpp),
// the boundary a reference caller uses when it swaps npconv/conv_op.hpp for
// npcg/npconv.hpp: PointConvOp<float>::forward / backward on HOST tensors,
// host->device and device->host copies and the host result vectors inside the
// timed region (conv_op.hpp:120-206 semantics: the op caches the neighbor
// structure per cloud, saves its input, returns grad_in and grad_w by value).
//
//   bench_dropin [n=1000000] [steps=10] [warmup=3] [math=bf16|auto|exact] [c=64]
//
// Prints one JSON line: Mpoints/s over n input points per fwd+bwd step, wall
// clock (std::chrono, the host sees every result), and the bytes copied.
#include <npcg/npconv.hpp>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 1000000;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
  const int warmup = argc > 3 ? std::atoi(argv[3]) : 3;
  const std::string math = argc > 4 ? argv[4] : "bf16";
  const int64_t c = argc > 5 ? std::atoll(argv[5]) : 64;
  const int64_t t = 3;
  using namespace npc;

  // the reference's seeded generators (synthetic.hpp / tensors.hpp), served by the library
  std::vector<double> xyz(static_cast<size_t>(n) * 3);
  if (npcg_gen_uniform_cube(n, 1.0, 1, xyz.data()) != NPCG_OK) return 2;
  std::vector<Vec3> pos(static_cast<size_t>(n));
  std::memcpy(pos.data(), xyz.data(), xyz.size() * sizeof(double));
  PointCloud cloud(std::move(pos), {0, n});
  std::vector<float> wv(static_cast<size_t>(t * t * t * c * c)), fv(static_cast<size_t>(n * c)),
      gv(static_cast<size_t>(n * c));
  if (npcg_make_weights(t, 1, c, c, 2, NPCG_F32, wv.data()) != NPCG_OK) return 2;
  if (npcg_gen_features(n, 1, c, 3, NPCG_F32, fv.data()) != NPCG_OK) return 2;
  if (npcg_gen_features(n, 1, c, 4, NPCG_F32, gv.data()) != NPCG_OK) return 2;
  FeatureTensor<float> fin(n, 1, c, std::move(fv)), gout(n, 1, c, std::move(gv));

  ExecConfig cfg;
  cfg.math = math == "bf16" ? NPCG_MATH_BF16 : math == "exact" ? NPCG_MATH_EXACT : NPCG_MATH_AUTO;
  const ConvGeometry geom{1.8 * std::pow(static_cast<double>(n), -1.0 / 3.0), t, ConvMode::native, 1.0};
  PointConvOp<float> op(WeightTensor<float>(t, 1, c, c, std::move(wv)), geom, cfg);

  using clk = std::chrono::steady_clock;
  const auto b0 = clk::now();
  double check = 0;
  for (int s = 0; s < warmup; ++s) {  // the first forward builds the neighbor cache and the tile plans
    const FeatureTensor<float> out = op.forward(cloud, fin);
    const BackwardResult<float> r = op.backward(gout);
    check += out.values()[0] + r.grad_in.values()[0] + r.grad_w.values()[0];
  }
  const double warm_s = std::chrono::duration<double>(clk::now() - b0).count();
  const auto t0 = clk::now();
  for (int s = 0; s < steps; ++s) {
    const FeatureTensor<float> out = op.forward(cloud, fin);
    const BackwardResult<float> r = op.backward(gout);
    check += out.values()[0] + r.grad_in.values()[0] + r.grad_w.values()[0];
  }
  const double sec = std::chrono::duration<double>(clk::now() - t0).count();
  const double ms = 1e3 * sec / steps;
  // split: forward alone, backward alone; and, for contrast, what one fresh
  // pageable n x c std::vector<float> costs on this host (allocation + first
  // touch), which results in pooled pinned storage no longer pay
  double f_ms = 0, b_ms = 0, v_ms = 0;
  for (int s = 0; s < 3; ++s) {
    const auto a = clk::now();
    const FeatureTensor<float> out = op.forward(cloud, fin);
    const auto b = clk::now();
    const BackwardResult<float> r = op.backward(gout);
    const auto e = clk::now();
    std::vector<float> v(static_cast<size_t>(n * c));
    check += v[v.size() / 2];
    const auto g = clk::now();
    f_ms += std::chrono::duration<double, std::milli>(b - a).count() / 3;
    b_ms += std::chrono::duration<double, std::milli>(e - b).count() / 3;
    v_ms += std::chrono::duration<double, std::milli>(g - e).count() / 3;
    check += out.values()[0] + r.grad_in.values()[0];
  }
  // a full checksum of one more step's results (outside the timed region)
  {
    const FeatureTensor<float> out = op.forward(cloud, fin);
    const BackwardResult<float> r = op.backward(gout);
    double cs = 0;
    for (float v : out.values()) cs += v;
    for (float v : r.grad_in.values()) cs += 2.0 * v;
    for (float v : r.grad_w.values()) cs += 3.0 * v;
    check = cs;
  }
  // per step: fin + gout up; out, grad_in, grad_w down (the weights stay resident)
  const int64_t h2d = 2 * n * c * 4, d2h = 2 * n * c * 4 + t * t * t * c * c * 4;
  std::printf(
      "{\"impl\": \"cpp_dropin\", \"metric\": \"conv_layer_fwd_bwd_throughput\", \"value\": %.3f, "
      "\"unit\": \"Mpoints/s\", \"ms_per_step\": %.4f, \"steps\": %d, \"warmup\": %d, \"math\": \"%s\", "
      "\"n_points\": %lld, \"channels\": %lld, \"h2d_bytes_per_step\": %lld, \"d2h_bytes_per_step\": %lld, "
      "\"forward_ms\": %.3f, \"backward_ms\": %.3f, \"pageable_vector_first_touch_ms\": %.3f, "
      "\"first_steps_s\": %.3f, \"timer\": \"host wall clock (std::chrono), results in host vectors\", "
      "\"checksum\": %.17g}\n",
      n / (ms * 1e3), ms, steps, warmup, math.c_str(), static_cast<long long>(n), static_cast<long long>(c),
      static_cast<long long>(h2d), static_cast<long long>(d2h), f_ms, b_ms, v_ms, warm_s, check);
  return std::isfinite(check) ? 0 : 1;
}
