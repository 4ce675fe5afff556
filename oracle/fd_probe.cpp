// Test infrastructure (diagnostics): the reference's end-to-end gradient check
// scene of acceptance criterion C4 (acceptance.cpp:218-237: 6 random DRKs,
// 8x8 render, SH degree 1, background 0.3, finite_diff_check seed 23, step
// 1e-4) with the per-scalar analytic gradients printed, so the reference build
// and the GPU adapter build can be compared scalar by scalar.
#include <cstdio>
#include <random>

#include "drk/grad.hpp"
#include "drk/optimize.hpp"

using namespace drk;

int main() {
  std::mt19937_64 rng2(19);
  std::vector<RawDrkParams> raws = init_random(Vec3(-0.5, -0.5, 1.5), Vec3(0.5, 0.5, 2.5), 6, 8, 1, rng2);
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  for (auto& r : raws) {
    r.opacity_raw = sigmoid_inverse(0.3 + 0.5 * u01(rng2));
    r.quat_raw = Vec4(1.0, 0.4 * (u01(rng2) - 0.5), 0.4 * (u01(rng2) - 0.5), 0.4 * (u01(rng2) - 0.5));
    r.tau_raw = tau_raw_for(-0.05 + 0.7 * u01(rng2));
    r.eta_raw = sigmoid_inverse(0.2 + 0.6 * u01(rng2));
  }
  Camera cam;
  cam.width = cam.height = 8;
  cam.fx = cam.fy = 8;
  cam.cx = cam.cy = 4;
  RenderOptions opt;
  opt.sh_degree = 1;
  opt.background = Vec3(0.3, 0.3, 0.3);
  std::mt19937_64 rng(23);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  FrameGrad fg;
  fg.d_color = Image(cam.width, cam.height, 3);
  fg.d_depth = Image(cam.width, cam.height, 1);
  fg.d_alpha = Image(cam.width, cam.height, 1);
  fg.d_normal = Image(cam.width, cam.height, 3);
  for (auto& v : fg.d_color.data) v = 2.0 * unit(rng) - 1.0;
  for (auto& v : fg.d_depth.data) v = 0.1 * (2.0 * unit(rng) - 1.0);
  for (auto& v : fg.d_alpha.data) v = 0.5 * (2.0 * unit(rng) - 1.0);
  for (auto& v : fg.d_normal.data) v = 0.1 * (2.0 * unit(rng) - 1.0);
  std::vector<DrkPrimitive> prims;
  for (const auto& r : raws) prims.push_back(activate(r));
  ReplayBuffer replay;
  const FrameBuffers fb = render(prims, cam, opt, &replay);
  const ParamGrads g = backward_render(raws, prims, cam, opt, replay, fg);
  for (size_t p = 0; p < raws.size(); ++p) {
    int s = 0;
    for_each_scalar(g.raw[p], [&](const double& x, ParamClass c) {
      std::printf("%zu %d %d %.17g\n", p, s++, (int)c, x);
    });
  }
  for (size_t i = 0; i < fb.color.data.size(); ++i) std::printf("C %zu %.17g\n", i, fb.color.data[i]);
  const GradCheckReport rep = finite_diff_check(raws, cam, opt, 23, 1e-4);
  for (int c = 0; c < 8; ++c) std::printf("class %d max_rel %.3e\n", c, rep.max_rel_error[c]);
  std::printf("checked %d skipped_branch %d skipped_small %d\n", rep.checked, rep.skipped_branch, rep.skipped_small);
  return 0;
}
