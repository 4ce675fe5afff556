// Times the drop-in path: the reference's own C++ API (drk::render, drk::loss,
// drk::backward_render, reference raster.hpp:92-93, optimize.hpp:19,
// grad.hpp:58-61) served by the GPU adapter (drk_adapter.cpp), as a reference
// user who links the adapter calls it.  Host std::vector<DrkPrimitive> in,
// host Images / ParamGrads out: the conversions and host<->device copies are
// inside the timed spans.  Built by oracle/Makefile.ref (target `adapter`)
// against the reference objects with those functions weakened; run by
// bench.py's adapter leg.
//
//   adapter_bench <input.bin> <warmup> <steps>
// input.bin: int32 n, k, terms, W, H; float64 fx, fy, cx, cy, R[9], t[3];
// float32 raw[S][n] (scalar-major, for_each_scalar order); float64 target[H][W][3].
// Prints one JSON line: forward and forward+backward ms per step.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "drk/grad.hpp"
#include "drk/optimize.hpp"
#include "drk/raster.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: adapter_bench input.bin warmup steps\n");
    return 2;
  }
  std::ifstream in(argv[1], std::ios::binary);
  int32_t hdr[5];
  double camv[16];
  in.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  in.read(reinterpret_cast<char*>(camv), sizeof camv);
  const int n = hdr[0], k = hdr[1], terms = hdr[2], W = hdr[3], H = hdr[4];
  const int S = drk::scalar_count(k, terms);
  std::vector<float> raw((size_t)S * n);
  in.read(reinterpret_cast<char*>(raw.data()), sizeof(float) * raw.size());
  drk::Image target(W, H, 3);
  in.read(reinterpret_cast<char*>(target.data.data()), sizeof(double) * target.data.size());
  if (!in) {
    std::fprintf(stderr, "adapter_bench: short input\n");
    return 2;
  }
  drk::Camera cam;
  cam.fx = camv[0];
  cam.fy = camv[1];
  cam.cx = camv[2];
  cam.cy = camv[3];
  cam.width = W;
  cam.height = H;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) cam.world_to_cam_rot(r, c) = camv[4 + 3 * r + c];
  for (int r = 0; r < 3; ++r) cam.world_to_cam_trans[r] = camv[13 + r];
  int deg = 0;
  while ((deg + 1) * (deg + 1) < terms) ++deg;
  std::vector<drk::RawDrkParams> raws(n);
  for (int i = 0; i < n; ++i) {
    drk::RawDrkParams p = drk::RawDrkParams::zeros(k, deg);
    int s = 0;
    drk::for_each_scalar(p, [&](double& x, drk::ParamClass) { x = raw[(size_t)(s++) * n + i]; });
    raws[i] = p;
  }
  drk::RenderOptions opt;
  opt.sh_degree = 3;
  const int warm = std::atoi(argv[2]), steps = std::atoi(argv[3]);
  using clk = std::chrono::steady_clock;
  double fwd_ms = 0, fb_ms = 0, act_ms = 0;
  for (int it = 0; it < warm + steps; ++it) {
    const auto t0 = clk::now();
    std::vector<drk::DrkPrimitive> prims;
    prims.reserve(n);
    for (const auto& r : raws) prims.push_back(drk::activate(r));
    const auto t1 = clk::now();
    const drk::FrameBuffers fb = drk::render(prims, cam, opt);
    const auto t2 = clk::now();
    const drk::LossResult lr = drk::loss(fb.color, target, 0.0);
    drk::ReplayBuffer replay;  // the adapter keeps the forward's decisions on the device
    replay.width = W;
    replay.height = H;
    drk::FrameGrad fg;
    fg.d_color = lr.d_color;
    const drk::ParamGrads g = drk::backward_render(raws, prims, cam, opt, replay, fg);
    const auto t3 = clk::now();
    if (g.raw.size() != (size_t)n) return 1;
    if (it >= warm) {
      act_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
      fwd_ms += std::chrono::duration<double, std::milli>(t2 - t1).count();
      fb_ms += std::chrono::duration<double, std::milli>(t3 - t1).count();
    }
  }
  std::printf("{\"activate_ms\": %.3f, \"render_ms\": %.3f, \"render_loss_backward_ms\": %.3f, \"steps\": %d}\n",
              act_ms / steps, fwd_ms / steps, fb_ms / steps, steps);
  return 0;
}
