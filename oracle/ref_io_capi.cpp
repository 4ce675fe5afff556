// Test infrastructure: C entry points over the UNMODIFIED reference
// drk::save_scene / drk::load_scene (io.cpp:40-97), compiled by
// oracle/Makefile.ref into oracle/_ref/libdrk_refio.so.  Pins the scene-file
// restatement (oracle/scene_io.py) and writes the golden scene fixture.
#include <cstring>
#include <vector>

#include "drk/errors.hpp"
#include "drk/io.hpp"
#include "drk/mesh.hpp"

namespace {
// status codes of include/drk_b200.h
int status_of(const std::exception& e) {
  if (dynamic_cast<const drk::IoError*>(&e)) return 11;
  if (dynamic_cast<const drk::CorruptFileError*>(&e)) return 12;
  if (dynamic_cast<const drk::VersionMismatchError*>(&e)) return 13;
  if (dynamic_cast<const drk::DimensionMismatchError*>(&e)) return 6;
  if (dynamic_cast<const drk::DegenerateFaceError*>(&e)) return 14;
  if (dynamic_cast<const drk::TooManyVerticesError*>(&e)) return 15;
  if (dynamic_cast<const drk::ParseError*>(&e)) return 16;
  if (dynamic_cast<const drk::EmptyMeshError*>(&e)) return 17;
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

// --- Mesh2DRK (mesh.cpp) -------------------------------------------------------
static drk::Mesh g_mesh;
static int g_warn = 0;

// load_mesh (mesh.cpp:134-217): sizes[4] = {nv, nf, n_indices, n_warnings}
int refmesh_load(const char* path, long long* sizes) {
  try {
    std::vector<std::string> w;
    g_mesh = drk::load_mesh(path, &w);
    g_warn = (int)w.size();
    long long ni = 0;
    for (const auto& f : g_mesh.faces) ni += (long long)f.indices.size();
    sizes[0] = (long long)g_mesh.vertices.size();
    sizes[1] = (long long)g_mesh.faces.size();
    sizes[2] = ni;
    sizes[3] = g_warn;
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

void refmesh_arrays(double* verts, int* off, int* idx, double* colors) {
  for (size_t v = 0; v < g_mesh.vertices.size(); ++v)
    for (int k = 0; k < 3; ++k) verts[3 * v + k] = g_mesh.vertices[v][k];
  int o = 0;
  off[0] = 0;
  for (size_t f = 0; f < g_mesh.faces.size(); ++f) {
    for (int id : g_mesh.faces[f].indices) idx[o++] = id;
    off[f + 1] = o;
    for (int k = 0; k < 3; ++k) colors[3 * f + k] = g_mesh.faces[f].color[k];
  }
}

// convert (mesh.cpp:326-343) of a mesh given as arrays -> raw f64 SoA [S][cap]
int refmesh_convert(const double* verts, long long nv, const int* off, const int* idx, const double* colors, int nf,
                    int k, double* raw, long long cap, long long* n_out, long long* n_skipped) {
  try {
    drk::Mesh m;
    for (long long v = 0; v < nv; ++v) m.vertices.emplace_back(verts[3 * v], verts[3 * v + 1], verts[3 * v + 2]);
    for (int f = 0; f < nf; ++f) {
      drk::MeshFace face;
      for (int j = off[f]; j < off[f + 1]; ++j) face.indices.push_back(idx[j]);
      face.color = drk::Vec3(colors[3 * f], colors[3 * f + 1], colors[3 * f + 2]);
      m.faces.push_back(face);
    }
    std::vector<std::string> w;
    const std::vector<drk::RawDrkParams> out = drk::convert(m, k, &w);
    *n_out = (long long)out.size();
    *n_skipped = (long long)w.size();
    if ((long long)out.size() <= cap)
      for (size_t i = 0; i < out.size(); ++i) {
        int s = 0;
        drk::for_each_scalar(out[i], [&](const double& x, drk::ParamClass) { raw[(size_t)s++ * cap + i] = x; });
      }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// shade_lambert (mesh.cpp:345-357) in place on raw f64 SoA [S][n] (SH degree 0)
int refmesh_shade(double* raw, int n, int k, const double* light, double ambient) {
  try {
    std::vector<drk::RawDrkParams> p(n);
    for (int i = 0; i < n; ++i) {
      p[i] = drk::RawDrkParams::zeros(k, 0);
      int s = 0;
      drk::for_each_scalar(p[i], [&](double& x, drk::ParamClass) { x = raw[(size_t)s++ * n + i]; });
    }
    drk::shade_lambert(p, drk::Vec3(light[0], light[1], light[2]), ambient);
    for (int i = 0; i < n; ++i) {
      int s = 0;
      drk::for_each_scalar(p[i], [&](const double& x, drk::ParamClass) { raw[(size_t)s++ * n + i] = x; });
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
}
