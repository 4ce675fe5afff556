// Test infrastructure: C entry points over the UNMODIFIED reference
// drk::save_scene / drk::load_scene (io.cpp:40-97), compiled by
// oracle/Makefile.ref into oracle/_ref/libdrk_refio.so.  Pins the scene-file
// restatement (oracle/scene_io.py) and writes the golden scene fixture.
#include <cstring>
#include <vector>

#include "drk/errors.hpp"
#include "drk/io.hpp"

namespace {
// status codes of include/drk_b200.h
int status_of(const std::exception& e) {
  if (dynamic_cast<const drk::IoError*>(&e)) return 11;
  if (dynamic_cast<const drk::CorruptFileError*>(&e)) return 12;
  if (dynamic_cast<const drk::VersionMismatchError*>(&e)) return 13;
  if (dynamic_cast<const drk::DimensionMismatchError*>(&e)) return 6;
  return 1;
}
}  // namespace

extern "C" {

// raw: f64 scalar-major [S][n] (the C-ABI order), each value stored as the
// reference stores it (double, narrowed to f32 by save_scene).
int refio_save_scene(const char* path, const double* raw, int n, int k, int sh_degree) {
  try {
    drk::Scene sc;
    sc.basis_count = k;
    sc.sh_degree = sh_degree;
    for (int i = 0; i < n; ++i) {
      drk::RawDrkParams p = drk::RawDrkParams::zeros(k, sh_degree);
      int s = 0;
      drk::for_each_scalar(p, [&](double& x, drk::ParamClass) { x = raw[(size_t)s++ * n + i]; });
      sc.params.push_back(std::move(p));
    }
    drk::save_scene(sc, path);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// hdr[4] = {K, sh_degree, count, scalar_count}; raw (may be null to query) f64 [S][count].
int refio_load_scene(const char* path, int expected_k, long long* hdr, double* raw, long long cap) {
  try {
    const drk::Scene sc = drk::load_scene(path, expected_k);
    const long long n = (long long)sc.params.size();
    int S = 0;
    if (n > 0) drk::for_each_scalar(sc.params[0], [&](const double&, drk::ParamClass) { ++S; });
    hdr[0] = sc.basis_count;
    hdr[1] = sc.sh_degree;
    hdr[2] = n;
    hdr[3] = S;
    if (raw && n <= cap) {
      for (long long i = 0; i < n; ++i) {
        int s = 0;
        drk::for_each_scalar(sc.params[i], [&](const double& x, drk::ParamClass) { raw[(size_t)s++ * n + i] = x; });
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
}
