// Mesh2DRK (reference mesh.cpp, mesh.hpp): one DRK per mesh face, on the
// device.  k_face_to_drk runs face_to_drk_raw (mesh.cpp:219-319) with one thread
// per face — centroid, Newell normal, tangent frame, boundary points at their
// polar angles, padding to K by bisecting the widest angular gap onto the edge,
// angles_to_raw (the inverse of the angle activation), log radii over the
// sharpness calibration, quaternion of the frame — in fp64 in the reference's
// expression order (--fmad=false), rounded once to the f32 raw layout.  convert
// (mesh.cpp:326-343) keeps the faces in order and skips degenerate ones (stable
// compaction); shade_lambert (mesh.cpp:345-357) bakes Lambertian shading into
// the degree-0 SH row.  The OBJ / MTL subset loader (mesh.cpp:134-217) is host
// code: it produces the vertex / face arrays the kernels take.
#include <algorithm>
#include <array>
#include <cmath>
#include <fstream>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "drk_internal.h"

namespace drk {

int set_error(drk_ctx* c, int status, const std::string& msg);
int cuda_check(drk_ctx* c, cudaError_t e, const char* where);
template <typename T>
int exclusive_scan(drk_ctx* c, const T* in, long long n, long long* out, long long* total);

namespace {

constexpr double kSh0 = 0.28209479177387814;  // mesh.cpp:16
constexpr double kPlanarTol = 1e-5;           // mesh.cpp:17
constexpr int kMaxFaceK = 16;

enum : int { kFaceOk = 0, kFaceDegenerate = 1, kFaceTooMany = 2 };

struct FaceConsts {
  double calibration;  // mesh_radius_calibration (mesh.cpp:132)
  double eta_raw, tau_raw, opacity_raw;
};

__device__ __forceinline__ double sq3(double x, double y, double z) { return sqrt(x * x + y * y + z * z); }

// face_to_drk_raw (mesh.cpp:219-319) for face f; writes column `col` of the
// raw SoA (S = 3+4+2K+3+3 rows, stride ld) when the face converts.
__device__ int face_to_raw(int f, const double* __restrict__ V, const int* __restrict__ off,
                           const int* __restrict__ idx, const double* __restrict__ colors, int K, FaceConsts cst,
                           float* raw, long long ld, long long col) {
  const int b = off[f], n = off[f + 1] - off[f];
  if (n < 3) return kFaceDegenerate;
  if (n > K) return kFaceTooMany;
  double cx = 0, cy = 0, cz = 0;
  for (int i = 0; i < n; ++i) {
    const double* p = V + 3 * (size_t)idx[b + i];
    cx += p[0];
    cy += p[1];
    cz += p[2];
  }
  cx /= n;
  cy /= n;
  cz /= n;
  // newell_normal (mesh.cpp:46-57)
  double nx = 0, ny = 0, nz = 0;
  for (int i = 0; i < n; ++i) {
    const double* a = V + 3 * (size_t)idx[b + i];
    const double* q = V + 3 * (size_t)idx[b + (i + 1) % n];
    nx += (a[1] - q[1]) * (a[2] + q[2]);
    ny += (a[2] - q[2]) * (a[0] + q[0]);
    nz += (a[0] - q[0]) * (a[1] + q[1]);
  }
  const double nlen = sq3(nx, ny, nz);
  if (nlen < 1e-12) return kFaceDegenerate;
  nx /= nlen;
  ny /= nlen;
  nz /= nlen;
  const double* v0 = V + 3 * (size_t)idx[b];
  double rx0 = v0[0] - cx, rx1 = v0[1] - cy, rx2 = v0[2] - cz;
  const double dn = rx0 * nx + rx1 * ny + rx2 * nz;
  rx0 -= dn * nx;
  rx1 -= dn * ny;
  rx2 -= dn * nz;
  const double rl = sq3(rx0, rx1, rx2);
  if (rl < 1e-12) return kFaceDegenerate;
  rx0 /= rl;
  rx1 /= rl;
  rx2 /= rl;
  const double ry0 = ny * rx2 - nz * rx1, ry1 = nz * rx0 - nx * rx2, ry2 = nx * rx1 - ny * rx0;  // normal x rx
  double px[kMaxFaceK], py[kMaxFaceK], ang[kMaxFaceK];
  for (int i = 0; i < n; ++i) {
    const double* p = V + 3 * (size_t)idx[b + i];
    const double d0 = p[0] - cx, d1 = p[1] - cy, d2 = p[2] - cz;
    px[i] = d0 * rx0 + d1 * rx1 + d2 * rx2;
    py[i] = d0 * ry0 + d1 * ry1 + d2 * ry2;
    if (sqrt(px[i] * px[i] + py[i] * py[i]) < 1e-12) return kFaceDegenerate;
    double a = 0.0;
    if (i > 0) {
      a = atan2(py[i], px[i]);
      if (a <= 0) a += 2.0 * kPi;
    }
    ang[i] = a;
  }
  for (int i = 1; i < n; ++i)
    if (ang[i] <= ang[i - 1]) return kFaceDegenerate;
  // pad to K by bisecting the widest angular gap (mesh.cpp:262-283)
  int m = n;
  while (m < K) {
    int widest = 0;
    double best = -1;
    for (int i = 0; i < m; ++i) {
      const double next = i + 1 < m ? ang[i + 1] : 2.0 * kPi;
      const double gap = next - ang[i];
      if (gap > best + 1e-15) {
        best = gap;
        widest = i;
      }
    }
    const double next_angle = widest + 1 < m ? ang[widest + 1] : 2.0 * kPi;
    const double mid = 0.5 * (ang[widest] + next_angle);
    const double ax = px[widest], ay = py[widest];
    const int w1 = (widest + 1) % m;
    const double bx = px[w1], by = py[w1];
    const double dx = cos(mid), dy = sin(mid);
    const double ca = dx * ay - dy * ax, cb = dx * by - dy * bx;
    const double t = ca / (ca - cb);
    const double ix = ax + t * (bx - ax), iy = ay + t * (by - ay);
    for (int i = m; i > widest + 1; --i) {
      px[i] = px[i - 1];
      py[i] = py[i - 1];
      ang[i] = ang[i - 1];
    }
    px[widest + 1] = ix;
    py[widest + 1] = iy;
    ang[widest + 1] = mid;
    ++m;
  }
  // kernel ordering (mesh.cpp:285-295): first vertex carried at exactly 2 pi
  double angles[kMaxFaceK], radii[kMaxFaceK];
  for (int i = 1; i < K; ++i) {
    angles[i - 1] = ang[i];
    radii[i - 1] = sqrt(px[i] * px[i] + py[i] * py[i]);
  }
  angles[K - 1] = 2.0 * kPi;
  radii[K - 1] = sqrt(px[0] * px[0] + py[0] * py[0]);
  // angles_to_raw (mesh.cpp:101-125)
  const double residual = 1.0 / (K - 2);
  double ratios[kMaxFaceK];
  double prev = 0, rmin = 1, rmax = 0;
  for (int i = 0; i < K; ++i) {
    ratios[i] = (angles[i] - prev) / (2.0 * kPi);
    rmin = ratios[i] < rmin ? ratios[i] : rmin;
    rmax = rmax < ratios[i] ? ratios[i] : rmax;
    prev = angles[i];
  }
  const double d_lo = residual / rmin, d_hi = (1.0 + residual) / rmax;
  const bool exact = d_lo < d_hi;
  const double total = exact ? sqrt(d_lo * d_hi) : 0.5 * (d_lo + d_hi);
  // rotation_to_quat (mesh.cpp:79-97) of the frame with columns rx, ry, normal
  const double m00 = rx0, m10 = rx1, m20 = rx2, m01 = ry0, m11 = ry1, m21 = ry2, m02 = nx, m12 = ny, m22 = nz;
  double q[4];
  const double tr = m00 + m11 + m22;
  if (tr > 0) {
    const double s = sqrt(tr + 1.0) * 2.0;
    q[0] = 0.25 * s; q[1] = (m21 - m12) / s; q[2] = (m02 - m20) / s; q[3] = (m10 - m01) / s;
  } else if (m00 > m11 && m00 > m22) {
    const double s = sqrt(1.0 + m00 - m11 - m22) * 2.0;
    q[0] = (m21 - m12) / s; q[1] = 0.25 * s; q[2] = (m01 + m10) / s; q[3] = (m02 + m20) / s;
  } else if (m11 > m22) {
    const double s = sqrt(1.0 + m11 - m00 - m22) * 2.0;
    q[0] = (m02 - m20) / s; q[1] = (m01 + m10) / s; q[2] = 0.25 * s; q[3] = (m12 + m21) / s;
  } else {
    const double s = sqrt(1.0 + m22 - m00 - m11) * 2.0;
    q[0] = (m10 - m01) / s; q[1] = (m02 + m20) / s; q[2] = (m12 + m21) / s; q[3] = 0.25 * s;
  }
  if (!raw) return kFaceOk;  // status pass
  // raw record in for_each_scalar order (types.hpp:48-58), SH degree 0
  float* r = raw + col;
  r[0] = (float)cx;
  r[ld] = (float)cy;
  r[2 * ld] = (float)cz;
  for (int j = 0; j < 4; ++j) r[(3 + j) * ld] = (float)q[j];
  for (int i = 0; i < K; ++i) r[(7 + i) * ld] = (float)log(radii[i] / cst.calibration);
  for (int i = 0; i < K; ++i) {
    double s = ratios[i] * total - residual;
    s = s < 1e-9 ? 1e-9 : (1.0 - 1e-9 < s ? 1.0 - 1e-9 : s);
    r[(7 + K + i) * ld] = (float)log(s / (1.0 - s));  // sigmoid_inverse (core.cpp:82-85)
  }
  r[(7 + 2 * K) * ld] = (float)cst.eta_raw;
  r[(8 + 2 * K) * ld] = (float)cst.tau_raw;
  r[(9 + 2 * K) * ld] = (float)cst.opacity_raw;
  for (int c = 0; c < 3; ++c) r[(10 + 2 * K + c) * ld] = (float)((colors[3 * (size_t)f + c] - 0.5) / kSh0);
  return kFaceOk;
}

// pass 0: status per face; pass 1: write the kept faces at their scanned slots
__global__ void k_face_status(int nf, const double* V, const int* off, const int* idx, const double* colors, int K,
                              FaceConsts cst, int* status, int* keep) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const int st = face_to_raw(f, V, off, idx, colors, K, cst, nullptr, 0, 0);
  status[f] = st;
  keep[f] = st == kFaceOk;
}

__global__ void k_face_emit(int nf, const double* V, const int* off, const int* idx, const double* colors, int K,
                            FaceConsts cst, const int* status, const long long* pos, float* raw, long long ld) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf || status[f] != kFaceOk) return;
  face_to_raw(f, V, off, idx, colors, K, cst, raw, ld, pos[f]);
}

// shade_lambert (mesh.cpp:345-357) on raw f32 SoA [S][n]
__global__ void k_shade_lambert(int n, int K, float* raw, double lx, double ly, double lz, double ambient) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double q0 = raw[(size_t)3 * n + i], q1 = raw[(size_t)4 * n + i], q2 = raw[(size_t)5 * n + i],
               q3 = raw[(size_t)6 * n + i];
  const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
  const double c0 = 2 * (x * z + w * y), c1 = 2 * (y * z - w * x), c2 = 1 - 2 * (x * x + y * y);  // rot.col(2)
  const double d = -(lx * c0 + ly * c1 + lz * c2);
  const double lambert = 0.0 < d ? d : 0.0;
  const double factor = ambient + (1.0 - ambient) * lambert;
  for (int c = 0; c < 3; ++c) {
    float* p = raw + (size_t)(10 + 2 * K + c) * n + i;
    const double color = 0.5 + kSh0 * (double)*p;
    double shaded = color * factor;
    shaded = shaded < 0.0 ? 0.0 : (1.0 < shaded ? 1.0 : shaded);
    *p = (float)((shaded - 0.5) / kSh0);
  }
}

FaceConsts face_consts() {
  auto sigmoid_inverse = [](double y) { return std::log(y / (1.0 - y)); };  // core.cpp:82-85
  FaceConsts c;
  c.calibration = std::sqrt(2.0 * std::log(2.0));
  c.eta_raw = sigmoid_inverse(1.0 - 1e-6);
  c.tau_raw = sigmoid_inverse(((kTauHigh - 1e-6) - kTauLow) / (kTauHigh - kTauLow));  // tau_raw_for (core.cpp:87)
  c.opacity_raw = sigmoid_inverse(1.0 - 1e-6);
  return c;
}

// ---------------------------------------------------------------------------
// OBJ / MTL subset (mesh.cpp:19-44, 134-217), host
// ---------------------------------------------------------------------------
using V3 = std::array<double, 3>;

bool planar_convex(const std::vector<V3>& pts) {  // face_planar_convex (mesh.cpp:59-77)
  const int m = (int)pts.size();
  if (m == 3) return true;
  double n[3] = {0, 0, 0};
  for (int i = 0; i < m; ++i) {
    const V3& a = pts[i];
    const V3& b = pts[(i + 1) % m];
    n[0] += (a[1] - b[1]) * (a[2] + b[2]);
    n[1] += (a[2] - b[2]) * (a[0] + b[0]);
    n[2] += (a[0] - b[0]) * (a[1] + b[1]);
  }
  const double len = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
  if (len < 1e-12) return false;
  for (double& v : n) v /= len;
  double c[3] = {0, 0, 0};
  for (const V3& p : pts)
    for (int k = 0; k < 3; ++k) c[k] += p[k];
  for (double& v : c) v /= m;
  for (const V3& p : pts) {
    const double d = (p[0] - c[0]) * n[0] + (p[1] - c[1]) * n[1] + (p[2] - c[2]) * n[2];
    if (std::abs(d) > kPlanarTol) return false;
  }
  for (int i = 0; i < m; ++i) {
    const V3& p0 = pts[i];
    const V3& p1 = pts[(i + 1) % m];
    const V3& p2 = pts[(i + 2) % m];
    const double e0[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
    const double e1[3] = {p2[0] - p1[0], p2[1] - p1[1], p2[2] - p1[2]};
    const double x[3] = {e0[1] * e1[2] - e0[2] * e1[1], e0[2] * e1[0] - e0[0] * e1[2], e0[0] * e1[1] - e0[1] * e1[0]};
    if (x[0] * n[0] + x[1] * n[1] + x[2] * n[2] < -1e-12) return false;
  }
  return true;
}

}  // namespace
}  // namespace drk

struct drk_mesh {
  std::vector<double> verts;   // nv x 3
  std::vector<int32_t> off{0}; // faces CSR
  std::vector<int32_t> idx;
  std::vector<double> colors;  // nf x 3
  int n_warnings = 0;
  std::string err;
};

using namespace drk;

namespace {
int mesh_fail(drk_mesh* m, int st, const std::string& msg) {
  if (m) m->err = msg;
  return st;
}

void parse_mtl(const std::string& path, std::vector<std::pair<std::string, V3>>* mats, int* warnings) {
  std::ifstream in(path);
  if (!in) {
    ++*warnings;
    return;
  }
  std::string line, current;
  while (std::getline(in, line)) {
    std::istringstream ss(line);
    std::string tag;
    if (!(ss >> tag)) continue;
    if (tag == "newmtl") {
      ss >> current;
      mats->emplace_back(current, V3{0.7, 0.7, 0.7});
    } else if (tag == "Kd" && !mats->empty()) {
      V3 kd;
      if (ss >> kd[0] >> kd[1] >> kd[2]) mats->back().second = kd;
    }
  }
}
}  // namespace

extern "C" int drk_mesh_load(const char* path_c, drk_mesh** out) {
  if (!path_c || !out) return DRK_ERR_INVALID_ARG;
  *out = nullptr;
  auto* m = new drk_mesh();
  const std::string path(path_c);
  std::ifstream in(path);
  if (!in) {
    *out = m;
    return mesh_fail(m, DRK_ERR_IO, "cannot open mesh file: " + path);
  }
  std::vector<std::pair<std::string, V3>> mats;
  V3 color{0.7, 0.7, 0.7};
  bool warned_tex = false;
  std::string line;
  int line_no = 0;
  std::vector<std::pair<std::vector<int>, V3>> faces;
  std::vector<V3> verts;
  *out = m;
  while (std::getline(in, line)) {
    ++line_no;
    std::istringstream ss(line);
    std::string tag;
    if (!(ss >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      V3 p;
      if (!(ss >> p[0] >> p[1] >> p[2])) return mesh_fail(m, DRK_ERR_PARSE, "malformed vertex at line " + std::to_string(line_no));
      verts.push_back(p);
    } else if (tag == "vt") {
      if (!warned_tex) {
        ++m->n_warnings;
        warned_tex = true;
      }
    } else if (tag == "f") {
      std::vector<int> ids;
      std::string tok;
      while (ss >> tok) {
        const size_t slash = tok.find('/');
        const std::string head = slash == std::string::npos ? tok : tok.substr(0, slash);
        int id = 0;
        try {
          id = std::stoi(head);
        } catch (...) {
          return mesh_fail(m, DRK_ERR_PARSE, "malformed face index at line " + std::to_string(line_no));
        }
        if (id > 0) id -= 1;
        else if (id < 0) id += (int)verts.size();
        else return mesh_fail(m, DRK_ERR_PARSE, "face index 0 at line " + std::to_string(line_no));
        if (id < 0 || id >= (int)verts.size())
          return mesh_fail(m, DRK_ERR_PARSE, "face index out of range at line " + std::to_string(line_no));
        ids.push_back(id);
      }
      if (ids.size() < 3)
        return mesh_fail(m, DRK_ERR_PARSE, "face with fewer than 3 vertices at line " + std::to_string(line_no));
      faces.emplace_back(std::move(ids), color);
    } else if (tag == "mtllib") {
      std::string file;
      if (ss >> file) {
        const size_t pos = path.find_last_of("/\\");
        parse_mtl((pos == std::string::npos ? std::string() : path.substr(0, pos + 1)) + file, &mats, &m->n_warnings);
      }
    } else if (tag == "usemtl") {
      std::string name;
      ss >> name;
      color = V3{0.7, 0.7, 0.7};
      for (const auto& [mat, kd] : mats)
        if (mat == name) color = kd;
    }
  }
  if (faces.empty()) return mesh_fail(m, DRK_ERR_EMPTY_MESH, "mesh has no faces: " + path);
  for (const V3& v : verts) m->verts.insert(m->verts.end(), v.begin(), v.end());
  auto push = [&](const std::vector<int>& ids, const V3& c) {
    m->idx.insert(m->idx.end(), ids.begin(), ids.end());
    m->off.push_back((int32_t)m->idx.size());
    m->colors.insert(m->colors.end(), c.begin(), c.end());
  };
  for (const auto& [ids, c] : faces) {
    std::vector<V3> pts;
    for (int id : ids) pts.push_back(verts[id]);
    if (pts.size() > 3 && !planar_convex(pts)) {  // fan triangulation (mesh.cpp:201-212)
      ++m->n_warnings;
      for (size_t i = 1; i + 1 < ids.size(); ++i) push({ids[0], ids[i], ids[i + 1]}, c);
    } else {
      push(ids, c);
    }
  }
  return DRK_OK;
}

extern "C" int drk_mesh_info(const drk_mesh* m, int64_t* n_vertices, int64_t* n_faces, int64_t* n_indices,
                             int32_t* n_warnings) {
  if (!m) return DRK_ERR_INVALID_ARG;
  if (n_vertices) *n_vertices = (int64_t)m->verts.size() / 3;
  if (n_faces) *n_faces = (int64_t)m->off.size() - 1;
  if (n_indices) *n_indices = (int64_t)m->idx.size();
  if (n_warnings) *n_warnings = m->n_warnings;
  return DRK_OK;
}

extern "C" const char* drk_mesh_error(const drk_mesh* m) { return m ? m->err.c_str() : ""; }

extern "C" int drk_mesh_arrays(const drk_mesh* m, double* vertices, int32_t* face_offsets, int32_t* indices,
                               double* colors) {
  if (!m) return DRK_ERR_INVALID_ARG;
  if (vertices) std::copy(m->verts.begin(), m->verts.end(), vertices);
  if (face_offsets) std::copy(m->off.begin(), m->off.end(), face_offsets);
  if (indices) std::copy(m->idx.begin(), m->idx.end(), indices);
  if (colors) std::copy(m->colors.begin(), m->colors.end(), colors);
  return DRK_OK;
}

extern "C" void drk_mesh_free(drk_mesh* m) { delete m; }

extern "C" int drk_mesh_convert(drk_ctx* c, const double* vertices, int64_t n_vertices, const int32_t* face_offsets,
                                const int32_t* indices, const double* colors, int n_faces, int k, float* raw_out,
                                int64_t cap, int64_t* n_out, int64_t* n_skipped) {
  if (!c || !n_out || n_faces < 0 || n_vertices < 0) return DRK_ERR_INVALID_ARG;
  if (k < 3 || k > kMaxFaceK) return set_error(c, DRK_ERR_UNSUPPORTED, "basis_count must be in [3, 16]");
  cudaSetDevice(c->device);
  *n_out = 0;
  if (n_skipped) *n_skipped = 0;
  if (n_faces == 0) return DRK_OK;
  if (!vertices || !face_offsets || !indices || !colors) return DRK_ERR_INVALID_ARG;
  int* st = ensure<int>(c->dens_code, 2 * (size_t)n_faces);
  long long* pos = ensure<long long>(c->dens_pos, (size_t)n_faces + 1);
  if (!st || !pos) return set_error(c, DRK_ERR_OOM, "mesh scratch");
  int* keep = st + n_faces;
  cudaStream_t s = c->stream;
  const FaceConsts cst = face_consts();
  k_face_status<<<(n_faces + 127) / 128, 128, 0, s>>>(n_faces, vertices, face_offsets, indices, colors, k, cst, st,
                                                       keep);
  DRK_COUNT_LAUNCH();
  std::vector<int> hs(n_faces);
  cudaMemcpyAsync(hs.data(), st, sizeof(int) * n_faces, cudaMemcpyDeviceToHost, s);
  if (int e = cuda_check(c, cudaStreamSynchronize(s), "mesh convert")) return e;
  for (int f = 0; f < n_faces; ++f)  // TooManyVerticesError propagates out of convert (mesh.cpp:336-340)
    if (hs[f] == kFaceTooMany)
      return set_error(c, DRK_ERR_TOO_MANY_VERTICES, "face " + std::to_string(f) + " has more vertices than basis_count");
  long long total = 0;
  if (int e = exclusive_scan<int>(c, keep, n_faces, pos, &total)) return e;
  *n_out = total;
  if (n_skipped) *n_skipped = n_faces - total;
  if (!raw_out) return DRK_OK;
  if (total > cap) return set_error(c, DRK_ERR_INVALID_ARG, "output capacity below the converted face count");
  k_face_emit<<<(n_faces + 127) / 128, 128, 0, s>>>(n_faces, vertices, face_offsets, indices, colors, k, cst, st, pos,
                                                     raw_out, cap);
  DRK_COUNT_LAUNCH();
  return cuda_check(c, cudaGetLastError(), "mesh convert");
}

extern "C" int drk_shade_lambert(drk_ctx* c, float* raw, int n, int k, const double* light_dir, double ambient) {
  if (!c || !light_dir || n < 0 || (n > 0 && !raw) || k < 3) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  // light_dir.normalized() on the host (Eigen: v / |v|)
  const double ln = std::sqrt(light_dir[0] * light_dir[0] + light_dir[1] * light_dir[1] + light_dir[2] * light_dir[2]);
  if (n > 0) {
    k_shade_lambert<<<(n + 255) / 256, 256, 0, c->stream>>>(n, k, raw, light_dir[0] / ln, light_dir[1] / ln,
                                                             light_dir[2] / ln, ambient);
    DRK_COUNT_LAUNCH();
  }
  return cuda_check(c, cudaGetLastError(), "shade_lambert");
}
