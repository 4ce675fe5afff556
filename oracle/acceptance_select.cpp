// Test infrastructure: the reference's acceptance suite
// (/root/reference/proj/tests/acceptance.cpp), compiled
// UNMODIFIED by inclusion, with a selector main: `acceptance_* C4 C5 C6 C10`
// runs those criteria (no argument: all ten) and prints the suite's own
// PASS / FAIL lines.  Linked against the reference library
// (oracle/_ref/acceptance_ref) or, with render / bin_primitives /
// backward_render / eval_sorting / losses weakened, against the GPU adapter
// (oracle/_ref/acceptance_adapter) — the drop-in proof for the hot-path
// criteria C4 (gradients), C5 (culling), C6 (sorting) and C10 (determinism).
#define main drk_reference_acceptance_main
#include "acceptance.cpp"
#undef main

#include <cstring>

int main(int argc, char** argv) {
  const Criterion criteria[] = {
      {"C1 gaussian reduction", c1_gaussian_reduction},
      {"C2 sharpening suite", c2_sharpening},
      {"C3 calibrated radius", c3_calibration},
      {"C4 gradient correctness", c4_gradients},
      {"C5 culling conservativeness", c5_culling},
      {"C6 sorting", c6_sorting},
      {"C7 teaser-scale fitting", c7_teaser_fit},
      {"C8 mesh conversion", c8_mesh},
      {"C9 density-control ordering", c9_density},
      {"C10 determinism", c10_determinism},
  };
  int failures = 0, ran = 0;
  for (const Criterion& c : criteria) {
    bool selected = argc <= 1;
    for (int i = 1; i < argc; ++i) {
      const size_t n = std::strlen(argv[i]);
      if (std::strncmp(c.label, argv[i], n) == 0 && c.label[n] == ' ') selected = true;
    }
    if (!selected) continue;
    ++ran;
    std::string detail;
    bool ok = false;
    try {
      ok = c.run(detail);
    } catch (const std::exception& e) {
      detail = std::string("exception: ") + e.what();
    }
    std::printf("%s - %s: %s\n", ok ? "PASS" : "FAIL", c.label, detail.c_str());
    std::fflush(stdout);
    failures += ok ? 0 : 1;
  }
  if (failures) std::printf("%d criteria failed\n", failures);
  else std::printf("all %d selected criteria passed\n", ran);
  return failures == 0 && ran > 0 ? 0 : 1;
}
