// DRKSCENE v1 scene files straight to / from the device SoA layout of the
// C-ABI (reference io.cpp:40-97, format comment io.hpp:20-23).
//
// File: one text header line "DRKSCENE <version> <K> <sh_degree> <count>\n"
// followed by count little-endian f32 records, each scalar_count(K, terms)
// values in the for_each_scalar order (types.hpp:48-74).  The C-ABI keeps the
// same scalar order but scalar-major ([S][n]), so a load is: header checks in
// the reference's order -> payload read in chunks into two pinned staging
// buffers (the read of chunk i+1 overlaps the H2D copy of chunk i) -> one
// shared-memory tiled transpose AoS -> SoA on the device.  A save runs the
// inverse transpose and D2H copies in chunks to the file.
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "drk_internal.h"

namespace drk {

int set_error(drk_ctx* c, int status, const std::string& msg);
int cuda_check(drk_ctx* c, cudaError_t e, const char* where);

constexpr int kSceneVersion = 1;                  // io.cpp:22
constexpr size_t kChunk = size_t(32) << 20;       // staging chunk (bytes)
constexpr int kTrRecs = 32;                       // records per transpose tile

// AoS [n][S] -> SoA [S][n] (to_soa) or back.  One CTA per 32 records: the
// tile (32 x S floats, S <= 74) is read and written with consecutive threads
// on consecutive addresses in both layouts.
template <bool TO_SOA>
__global__ void __launch_bounds__(256) k_scene_transpose(const float* __restrict__ in, float* __restrict__ out,
                                                         long long n, int S) {
  extern __shared__ float tile[];  // [kTrRecs][S + 1]
  const long long r0 = (long long)blockIdx.x * kTrRecs;
  const int nr = (int)min((long long)kTrRecs, n - r0);
  const int ld = S + 1;
  if (TO_SOA) {
    for (int e = threadIdx.x; e < nr * S; e += blockDim.x) {
      const int r = e / S, s = e - r * S;
      tile[r * ld + s] = in[(r0 + r) * S + s];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < S * kTrRecs; e += blockDim.x) {
      const int s = e / kTrRecs, r = e - s * kTrRecs;
      if (r < nr) out[(size_t)s * n + r0 + r] = tile[r * ld + s];
    }
  } else {
    for (int e = threadIdx.x; e < S * kTrRecs; e += blockDim.x) {
      const int s = e / kTrRecs, r = e - s * kTrRecs;
      if (r < nr) tile[r * ld + s] = in[(size_t)s * n + r0 + r];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * S; e += blockDim.x) {
      const int r = e / S, s = e - r * S;
      out[(r0 + r) * S + s] = tile[r * ld + s];
    }
  }
}

static void launch_transpose(bool to_soa, const float* in, float* out, long long n, int S, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned blocks = (unsigned)((n + kTrRecs - 1) / kTrRecs);
  const size_t smem = sizeof(float) * kTrRecs * (S + 1);
  if (to_soa) k_scene_transpose<true><<<blocks, 256, smem, s>>>(in, out, n, S);
  else k_scene_transpose<false><<<blocks, 256, smem, s>>>(in, out, n, S);
  DRK_COUNT_LAUNCH();
}

// std::istream >> int / long on one whitespace-separated token: optional sign,
// at least one digit; the token must end at whitespace or the line end (a
// trailing non-digit would make the next extraction fail in the reference).
static bool next_token(const char*& p, std::string& tok) {
  while (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f') ++p;
  const char* b = p;
  while (*p && *p != ' ' && *p != '\t' && *p != '\r' && *p != '\v' && *p != '\f') ++p;
  tok.assign(b, p);
  return !tok.empty();
}
// `last`: the final extraction of the header, after which the reference reads
// nothing more, so characters after the digits are ignored there.
static bool parse_long(const char*& p, long long lo, long long hi, long long* v, bool last = false) {
  std::string t;
  if (!next_token(p, t)) return false;
  errno = 0;
  char* e = nullptr;
  const long long x = strtoll(t.c_str(), &e, 10);
  if (e == t.c_str() || (*e != '\0' && !last) || errno == ERANGE || x < lo || x > hi) return false;
  *v = x;
  return true;
}

struct SceneFile {
  FILE* f = nullptr;
  ~SceneFile() {
    if (f) fclose(f);
  }
};

// Header checks of load_scene (io.cpp:58-76) in the reference's order; on
// success the file is positioned at the payload and *payload_bytes holds the
// remaining file size.
static int read_header(drk_ctx* c, SceneFile& sf, const char* path, int expected_k, drk_scene_header* h,
                       long long* payload_bytes) {
  sf.f = fopen(path, "rb");
  if (!sf.f) return set_error(c, DRK_ERR_IO, std::string("cannot open scene file: ") + path);
  std::string line;
  int ch;
  bool any = false;
  while ((ch = fgetc(sf.f)) != EOF) {
    any = true;
    if (ch == '\n') break;
    line.push_back((char)ch);
    if (line.size() > 4096) break;  // no plausible header is this long
  }
  if (!any) return set_error(c, DRK_ERR_CORRUPT_FILE, std::string("missing scene header: ") + path);
  const char* p = line.c_str();
  std::string magic;
  long long version = 0, k = 0, deg = 0, count = -1;
  const bool ok = next_token(p, magic) && parse_long(p, INT32_MIN, INT32_MAX, &version) &&
                  parse_long(p, INT32_MIN, INT32_MAX, &k) && parse_long(p, INT32_MIN, INT32_MAX, &deg) &&
                  parse_long(p, INT64_MIN, INT64_MAX, &count, true);
  if (!ok || magic != "DRKSCENE") return set_error(c, DRK_ERR_CORRUPT_FILE, std::string("not a scene file: ") + path);
  if (version != kSceneVersion)
    return set_error(c, DRK_ERR_VERSION, "unsupported scene version " + std::to_string(version));
  if (k < 3 || deg < 0 || deg > 3 || count < 0)
    return set_error(c, DRK_ERR_CORRUPT_FILE, std::string("implausible scene header: ") + path);
  if (expected_k > 0 && k != expected_k)
    return set_error(c, DRK_ERR_VERSION, "scene has K=" + std::to_string(k) + ", pipeline expects K=" +
                                             std::to_string(expected_k));
  const long long here = ftello(sf.f);
  if (fseeko(sf.f, 0, SEEK_END) != 0) return set_error(c, DRK_ERR_IO, std::string("cannot seek: ") + path);
  const long long end = ftello(sf.f);
  fseeko(sf.f, here, SEEK_SET);
  const long long terms = (deg + 1) * (deg + 1);
  const long long rec = 4 * (3 + 4 + 2 * k + 3 + 3 * terms);
  if (count > (end - here) / rec || (end - here) != rec * count)
    return set_error(c, DRK_ERR_CORRUPT_FILE, std::string("scene payload size disagrees with the header count: ") + path);
  h->version = (int32_t)version;
  h->basis_count = (int32_t)k;
  h->sh_degree = (int32_t)deg;
  h->scalar_count = (int32_t)(rec / 4);
  h->count = count;
  *payload_bytes = end - here;
  return DRK_OK;
}

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  bool init(size_t bytes) {
    for (int i = 0; i < 2; ++i) {
      if (cudaHostAlloc(&p[i], bytes, cudaHostAllocDefault) != cudaSuccess) return false;
      if (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) return false;
    }
    return true;
  }
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventSynchronize(done[i]), cudaEventDestroy(done[i]);
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
};

}  // namespace drk

using namespace drk;

extern "C" int drk_scene_read_header(const char* path, int expected_basis_count, drk_scene_header* out) {
  if (!path || !out) return DRK_ERR_INVALID_ARG;
  SceneFile sf;
  long long bytes = 0;
  return read_header(nullptr, sf, path, expected_basis_count, out, &bytes);
}

extern "C" int drk_scene_load(drk_ctx* c, const char* path, int expected_basis_count, float* raw, int64_t capacity,
                              drk_scene_header* out) {
  if (!c || !path || !out) return DRK_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  SceneFile sf;
  long long bytes = 0;
  if (int st = read_header(c, sf, path, expected_basis_count, out, &bytes)) return st;
  const long long n = out->count;
  if (n > capacity) return set_error(c, DRK_ERR_INVALID_ARG, "device buffer holds fewer primitives than the scene");
  if (n == 0) return DRK_OK;
  if (!raw) return DRK_ERR_INVALID_ARG;
  if (n > INT32_MAX) return set_error(c, DRK_ERR_UNSUPPORTED, "more than 2^31-1 primitives");
  cudaStream_t s = c->stream;
  float* aos = ensure<float>(c->scene_aos, (size_t)bytes / 4);
  if (!aos) return set_error(c, DRK_ERR_OOM, "scene staging");
  Pinned pin;
  const size_t chunk = (size_t)std::min<long long>(bytes, (long long)kChunk);
  if (!pin.init(chunk)) return set_error(c, DRK_ERR_OOM, "pinned scene staging");
  long long done = 0;
  for (int i = 0; done < bytes; i ^= 1) {
    const size_t want = (size_t)std::min<long long>(chunk, bytes - done);
    cudaEventSynchronize(pin.done[i]);  // the copy that last used this buffer
    if (fread(pin.p[i], 1, want, sf.f) != want)
      return set_error(c, DRK_ERR_CORRUPT_FILE, std::string("short read of the scene payload: ") + path);
    cudaMemcpyAsync(reinterpret_cast<char*>(aos) + done, pin.p[i], want, cudaMemcpyHostToDevice, s);
    cudaEventRecord(pin.done[i], s);
    done += (long long)want;
  }
  launch_transpose(true, aos, raw, n, out->scalar_count, s);
  return cuda_check(c, cudaStreamSynchronize(s), "scene load");
}

extern "C" int drk_scene_save(drk_ctx* c, const char* path, const float* raw, int n, int k, int sh_degree) {
  if (!c || !path || n < 0 || (n > 0 && !raw)) return DRK_ERR_INVALID_ARG;
  if (k < 3 || k > 16 || sh_degree < 0 || sh_degree > 3)
    return set_error(c, DRK_ERR_DIMENSION, "primitive layout differs from the scene header");
  cudaSetDevice(c->device);
  const int S = 3 + 4 + 2 * k + 3 + 3 * (sh_degree + 1) * (sh_degree + 1);
  const long long bytes = 4LL * S * n;
  cudaStream_t s = c->stream;
  float* aos = nullptr;
  if (n > 0) {
    aos = ensure<float>(c->scene_aos, (size_t)S * n);
    if (!aos) return set_error(c, DRK_ERR_OOM, "scene staging");
    launch_transpose(false, raw, aos, n, S, s);
    if (int st = cuda_check(c, cudaGetLastError(), "scene transpose")) return st;
  }
  SceneFile sf;
  sf.f = fopen(path, "wb");
  if (!sf.f) return set_error(c, DRK_ERR_IO, std::string("cannot open scene file for writing: ") + path);
  if (fprintf(sf.f, "DRKSCENE %d %d %d %d\n", kSceneVersion, k, sh_degree, n) < 0)
    return set_error(c, DRK_ERR_IO, std::string("failed writing scene file: ") + path);
  if (n > 0) {
    Pinned pin;
    const size_t chunk = (size_t)std::min<long long>(bytes, (long long)kChunk);
    if (!pin.init(chunk)) return set_error(c, DRK_ERR_OOM, "pinned scene staging");
    // D2H of chunk i+1 is queued before chunk i is written to the file
    size_t len[2] = {0, 0};
    long long next = 0;
    int i = 0;
    auto issue = [&](int b) {
      len[b] = (size_t)std::min<long long>(chunk, bytes - next);
      cudaMemcpyAsync(pin.p[b], reinterpret_cast<const char*>(aos) + next, len[b], cudaMemcpyDeviceToHost, s);
      cudaEventRecord(pin.done[b], s);
      next += (long long)len[b];
    };
    issue(0);
    while (len[i] > 0) {
      if (next < bytes) issue(i ^ 1);
      else len[i ^ 1] = 0;
      if (int st = cuda_check(c, cudaEventSynchronize(pin.done[i]), "scene save")) return st;
      if (fwrite(pin.p[i], 1, len[i], sf.f) != len[i])
        return set_error(c, DRK_ERR_IO, std::string("failed writing scene file: ") + path);
      i ^= 1;
    }
  }
  if (fflush(sf.f) != 0) return set_error(c, DRK_ERR_IO, std::string("failed writing scene file: ") + path);
  return DRK_OK;
}
