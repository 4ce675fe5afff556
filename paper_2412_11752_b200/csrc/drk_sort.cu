// Device-wide exclusive scan and stable LSD radix sort (hand-written, no CUB).
//
// Sort: 8-bit digits, 2048 elements per CTA (8 warps x 32 lanes x 8 items).
// Per pass: k_rs_hist (per-CTA digit histogram, digit-major layout) ->
// exclusive scan of the 256 x nblk histogram -> k_rs_scatter (stable ranks via
// warp match_any + per-warp running counts, then warp prefix per digit).
// Pairs are (key u32, value u32): key = tile << b | b-bit monotone quantisation
// of the fp64 depth key (k_pack_keys, drk_prep.cu), value = primitive id; four
// 8-bit passes.  Runs of equal keys are ordered afterwards on the full fp64 key
// (k_tie_rank, drk_prep.cu), so the sort itself need not be stable.
#include "drk_internal.h"

namespace drk {

constexpr int kScanThreads = 256, kScanItems = 4, kScanBlock = kScanThreads * kScanItems;

template <typename T>
__global__ void k_scan_block(const T* __restrict__ in, long long n, long long* out, long long* bsum) {
  __shared__ long long sm[kScanThreads];
  const long long base = (long long)blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  long long v[kScanItems], run = 0;
  for (int k = 0; k < kScanItems; ++k) {
    const long long idx = base + k;
    v[k] = idx < n ? (long long)in[idx] : 0;
    run += v[k];
  }
  sm[threadIdx.x] = run;
  __syncthreads();
  for (int off = 1; off < kScanThreads; off <<= 1) {
    const long long t = threadIdx.x >= off ? sm[threadIdx.x - off] : 0;
    __syncthreads();
    sm[threadIdx.x] += t;
    __syncthreads();
  }
  long long ex = sm[threadIdx.x] - run;
  for (int k = 0; k < kScanItems; ++k) {
    const long long idx = base + k;
    if (idx < n) out[idx] = ex;
    ex += v[k];
  }
  if (threadIdx.x == kScanThreads - 1) bsum[blockIdx.x] = sm[threadIdx.x];
}

__global__ void k_scan_add(long long* out, long long n, const long long* __restrict__ bpre) {
  const long long base = (long long)blockIdx.x * kScanBlock;
  const long long add = bpre[blockIdx.x];
  for (int k = threadIdx.x; k < kScanBlock; k += kScanThreads) {
    const long long idx = base + k;
    if (idx < n) out[idx] += add;
  }
}

// Exclusive scan of n values into out; *total receives the sum (host value;
// synchronises the stream).  tmp must hold scan_tmp_elems(n) long longs.
size_t scan_tmp_elems(long long n) {
  size_t tot = 0;
  long long m = n;
  do {
    m = (m + kScanBlock - 1) / kScanBlock;
    tot += 2 * (size_t)m + 2;
  } while (m > 1);
  return tot + 4;
}

template <typename T>
void scan_level(const T* in, long long n, long long* out, long long* tmp, cudaStream_t s) {
  const long long nb = (n + kScanBlock - 1) / kScanBlock;
  long long* bsum = tmp;
  long long* bpre = tmp + nb + 1;
  k_scan_block<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, out, bsum);
  launch_counter() += nb > 1 ? 2 : 1;
  if (nb > 1) {
    scan_level<long long>(bsum, nb, bpre, tmp + 2 * nb + 2, s);
    k_scan_add<<<(unsigned)nb, kScanThreads, 0, s>>>(out, n, bpre);
  }
}

template <typename T>
int exclusive_scan(drk_ctx* c, const T* in, long long n, long long* out, long long* total) {
  long long* tmp = ensure<long long>(c->scan_tmp, scan_tmp_elems(n) + 1);
  if (!tmp) return set_error(c, DRK_ERR_OOM, "scan scratch");
  if (n == 0) {
    if (total) *total = 0;
    return DRK_OK;
  }
  scan_level<T>(in, n, out, tmp, c->stream);
  if (total) {
    long long last_ex = 0;
    T last_in{};
    cudaMemcpyAsync(&last_ex, out + n - 1, sizeof(long long), cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(&last_in, in + n - 1, sizeof(T), cudaMemcpyDeviceToHost, c->stream);
    if (int st = cuda_check(c, cudaStreamSynchronize(c->stream), "scan")) return st;
    *total = last_ex + (long long)last_in;
  }
  return cuda_check(c, cudaGetLastError(), "scan");
}

template int exclusive_scan<int>(drk_ctx*, const int*, long long, long long*, long long*);
template int exclusive_scan<unsigned>(drk_ctx*, const unsigned*, long long, long long*, long long*);

// ---------------------------------------------------------------------------
// radix sort
// ---------------------------------------------------------------------------
#ifndef DRK_RS_ITEMS
#define DRK_RS_ITEMS 8
#endif
constexpr int kRsWarps = 8, kRsItems = DRK_RS_ITEMS, kRsThreads = kRsWarps * 32, kRsChunk = kRsThreads * kRsItems;

// per-warp sub-histograms: after the first pass the keys arrive grouped by
// digit, and a single block-wide histogram would serialise on same-address
// shared-memory atomics
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const unsigned* __restrict__ src, long long n,
                                                        int shift, unsigned* hist, int nblk) {
  __shared__ unsigned cnt[kRsWarps][256];
  for (int d = threadIdx.x; d < kRsWarps * 256; d += kRsThreads) (&cnt[0][0])[d] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const long long base = (long long)blockIdx.x * kRsChunk;
  unsigned kk[kRsItems];
#pragma unroll
  for (int k = 0; k < kRsItems; ++k) {
    const long long i = base + k * kRsThreads + threadIdx.x;
    kk[k] = i < n ? ((src[i] >> shift) & 255u) : 256u;
  }
#pragma unroll
  for (int k = 0; k < kRsItems; ++k)
    if (kk[k] < 256u) atomicAdd(&cnt[warp][kk[k]], 1u);
  __syncthreads();
  unsigned t = 0;
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) t += cnt[w][threadIdx.x];
  hist[(size_t)threadIdx.x * nblk + blockIdx.x] = t;
}

// One stable LSD pass: per-warp match-based ranks, block-local digit order
// staged in shared memory, then written out digit run by digit run so that
// consecutive threads store consecutive addresses of one bucket.
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const unsigned* __restrict__ kin,
                                                           const unsigned* __restrict__ vin,
                                                           unsigned* kout, unsigned* vout,
                                                           long long n, int shift,
                                                           const long long* __restrict__ offs, int nblk) {
  __shared__ unsigned whist[kRsWarps][256];
  __shared__ unsigned bstart[256];
  __shared__ long long gbase[256];
  extern __shared__ unsigned rs_dyn[];  // staging: keys then values, kRsChunk each
  unsigned* sk = rs_dyn;
  unsigned* sv = rs_dyn + kRsChunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = threadIdx.x; d < kRsWarps * 256; d += kRsThreads) (&whist[0][0])[d] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kRsChunk + (long long)warp * 32 * kRsItems;
  const unsigned lt = (1u << lane) - 1u;
  unsigned kk[kRsItems], vv[kRsItems];
  int dig[kRsItems];
  unsigned rank[kRsItems];
  // a warp whose items are all valid needs only the 8 digit-bit ballots
  const bool full = base + 32 * kRsItems <= n;
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const long long i = base + r * 32 + lane;
    const bool valid = i < n;
    kk[r] = valid ? kin[i] : 0;
    vv[r] = valid ? vin[i] : 0;
  }
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const bool valid = base + r * 32 + lane < n;
    const int d = valid ? (int)((kk[r] >> shift) & 255u) : 256;
    dig[r] = d;
    // lanes with the same digit: intersection of per-bit ballots (bit 8 marks
    // invalid items)
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool bit = (d >> b) & 1;
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
    if (!full) {
      const bool bit = (d >> 8) & 1;
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
    const unsigned cur = valid ? whist[warp][d] : 0;
    rank[r] = cur + __popc(peers & lt);
    __syncwarp();
    const int leader = 31 - __clz(peers);
    if (valid && lane == leader) whist[warp][d] = cur + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    // per digit: warp offsets (in warp order) and the block total
    const int d = threadIdx.x;  // kRsThreads == 256 digits
    unsigned run = 0;
    for (int w = 0; w < kRsWarps; ++w) {
      const unsigned t = whist[w][d];
      whist[w][d] = run;
      run += t;
    }
    // block-local digit starts: exclusive scan of the totals over digits
    unsigned incl = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    bstart[d] = incl;  // warp-inclusive for now
    __syncthreads();
    unsigned wsum = 0;
    for (int w = 0; w < warp; ++w) wsum += bstart[w * 32 + 31];
    __syncthreads();
    bstart[d] = wsum + incl - run;
    gbase[d] = offs[(size_t)d * nblk + blockIdx.x];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    if (dig[r] == 256) continue;
    const unsigned pos = bstart[dig[r]] + whist[warp][dig[r]] + rank[r];
    sk[pos] = kk[r];
    sv[pos] = vv[r];
  }
  __syncthreads();
  const long long cnt_ll = n - (long long)blockIdx.x * kRsChunk;
  const int cnt = cnt_ll < kRsChunk ? (int)cnt_ll : kRsChunk;
  for (int idx = threadIdx.x; idx < cnt; idx += kRsThreads) {
    const unsigned key = sk[idx], val = sv[idx];
    const int d = (int)((key >> shift) & 255u);
    const long long pos = gbase[d] + (idx - (long long)bstart[d]);
    kout[pos] = key;
    vout[pos] = val;
  }
}

// LSD sort of (k, v) pairs by the 32-bit key (stable; four passes, so the
// result ends in the input buffers).
int sort_pairs(drk_ctx* c, unsigned* k, unsigned* v, unsigned* k2, unsigned* v2, long long n) {
  if (n <= 1) return DRK_OK;
  cudaStream_t s = c->stream;
  const int nblk = (int)((n + kRsChunk - 1) / kRsChunk);
  unsigned* hist = ensure<unsigned>(c->hist, (size_t)256 * nblk);
  long long* off = ensure<long long>(c->sortoff, (size_t)256 * nblk);
  if (!hist || !off) return set_error(c, DRK_ERR_OOM, "sort scratch");
  const size_t rs_smem = 2 * sizeof(unsigned) * kRsChunk;
  for (int d = 0; d < 4; ++d) {
    k_rs_hist<<<nblk, kRsThreads, 0, s>>>(k, n, 8 * d, hist, nblk);
    sort_trace("hist", s);
    if (int st = exclusive_scan<unsigned>(c, hist, (long long)256 * nblk, off, nullptr)) return st;
    sort_trace("scan", s);
    k_rs_scatter<<<nblk, kRsThreads, rs_smem, s>>>(k, v, k2, v2, n, 8 * d, off, nblk);
    sort_trace("scatter", s);
    launch_counter() += 2;
    std::swap(k, k2);
    std::swap(v, v2);
  }
  return cuda_check(c, cudaGetLastError(), "sort");
}

}  // namespace drk
