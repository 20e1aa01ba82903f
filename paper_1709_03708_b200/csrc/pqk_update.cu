// pqk_update.cu — histogram, sparse-voting update, empty-cluster repair and the
// numpy-exact objective sums of one PQk-means Lloyd iteration on sm_100a.
//
//   histogram : clustering.py:344-347 (bincount(labels*L + codes[:,m])) and the
//               counts of clustering.py:458, as integer atomics (order independent,
//               bit exact).
//   vote      : clustering.py:349-356.  votes_j = sum_s hist[s] * T[m][s][j] for the
//               support s of each (filled k, m); center = argmin_j, lowest j on ties.
//               Computed in fp64 (ascending s, FMA); the argmin is certified against
//               the rounding error of any summation order (the reference uses an
//               OpenBLAS dgemv whose order is kernel specific), and near ties are
//               re-decided in double-double arithmetic (exact-arithmetic argmin).
//   repair    : clustering.py:460-466.  The E empty clusters (ascending k) take the
//               codes of the E largest sd_sq (lowest index first among equal
//               values) — a radix select over the 96-bit key (sd_sq bits, ~index).
//   objective : clustering.py:448-449, float(np.mean(np.sqrt(sd))) and
//               float(np.mean(sd)), evaluated with numpy's pairwise-summation tree so
//               the sums (and hence the exact-equality stop rule at :450) match.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "pqk_common.cuh"
#include "pqk_tc.cuh"

namespace pqk {


// ---------------------------------------------------------------------------
// histogram
__global__ void histogram_kernel(const uint8_t* __restrict__ codes, int64_t n, int mp, int m, int l,
                                 const uint32_t* __restrict__ labels, uint32_t* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = labels[i];
    const uint32_t* x = reinterpret_cast<const uint32_t*>(codes + i * mp);  // mp is a multiple of 4
    uint32_t* hk = hist + k * m * l;
    for (int w = 0; 4 * w < m; ++w) {
      const uint32_t cw = __ldg(x + w);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (4 * w + b < m) atomicAdd(&hk[(4 * w + b) * l + ((cw >> (8 * b)) & 0xffu)], 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// cluster-tiled histogram.  At configs 4/5 the K x M x L table (410 MB / 1.64 GB) is far
// larger than L2, so every random global atomic of histogram_kernel costs a DRAM sector
// round trip (config 4 shard: 15.7 ms, 1% of HBM).  Instead the codes are bucketed by
// cluster tile (T consecutive clusters, T*M*L*4 B of shared memory) with a two-pass
// counting sort, and one CTA per tile counts its members in shared memory and writes
// its dense slab of the table (zeros included: no memset).  Counts are integers, so
// the result is bit-identical to the atomic kernel whatever the order.
constexpr int kHistTileBytes = 96 * 1024;    // 2 CTAs per SM in the tile pass
constexpr int kHistMaxBuckets = 40 * 1024;   // shared-memory cursors of the bucket passes
constexpr int kHistThreads = 512;

// pass 1: cnt[c][b] = members of bucket b among CTA c's contiguous element range
__global__ void __launch_bounds__(kHistThreads) hbin_count_kernel(const uint32_t* __restrict__ labels, int64_t n,
                                                                  int64_t per_cta, uint32_t tile, int nb,
                                                                  uint32_t* __restrict__ cnt, int pad4) {
  extern __shared__ uint32_t sc[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sc[b] = 0;
  __syncthreads();
  const int64_t lo = blockIdx.x * per_cta, hi = min(n, lo + per_cta);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&sc[__ldg(labels + i) / tile], 1u);
  __syncthreads();
  // pad4 (sector-staged scatter): every (CTA, bucket) run is a whole number of 32-byte
  // sectors of 8-byte records, padding records carry label word ~0
  for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[(int64_t)blockIdx.x * nb + b] = pad4 ? (sc[b] + 3u) & ~3u : sc[b];
}

// thread per bucket: cnt[c][b] -> exclusive prefix over c, tot[b] = bucket size
__global__ void hbin_colscan_kernel(uint32_t* __restrict__ cnt, int ctas, int nb, uint32_t* __restrict__ tot) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  uint32_t run = 0;
#pragma unroll 8
  for (int c = 0; c < ctas; ++c) {
    const uint32_t v = cnt[(int64_t)c * nb + b];
    cnt[(int64_t)c * nb + b] = run;
    run += v;
  }
  tot[b] = run;
}

// one CTA: base[b] = exclusive prefix of tot over buckets, base[nb] = n (in place: tot -> base)
__global__ void __launch_bounds__(1024) hbin_scan_kernel(uint32_t* __restrict__ tot, int nb) {
  __shared__ uint32_t warp_sum[32];
  const int per = (nb + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(nb, lo + per);
  uint32_t s = 0;
  for (int b = lo; b < hi; ++b) s += tot[b];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = warp_sum[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    warp_sum[lane] = wi - w;
  }
  __syncthreads();
  uint32_t run = warp_sum[wid] + incl - s;
  for (int b = lo; b < hi; ++b) {
    const uint32_t v = tot[b];
    tot[b] = run;
    run += v;
  }
  if (threadIdx.x == 1023) tot[nb] = run;
}

// pass 2: scatter records (code words, tile-local label word) into bucket order; CTA c
// writes into its reserved run base[b] + cnt[c][b] of every bucket.  Every (CTA, bucket)
// run is an open L2 line until it fills, so the host sizes the CTA count to keep
// ctas x buckets x 128 B near the L2 size (a spilled partial line costs a DRAM
// read-modify-write: 8x the algorithmic traffic at config 4 with 296 CTAs).
__global__ void __launch_bounds__(1024) hbin_scatter_kernel(
    const uint8_t* __restrict__ codes, int mw, const uint32_t* __restrict__ labels, int64_t n, int64_t per_cta,
    uint32_t tile, int nb, const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ base,
    uint32_t* __restrict__ rec) {
  extern __shared__ uint32_t cur[];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) cur[b] = base[b] + cnt[(int64_t)blockIdx.x * nb + b];
  __syncthreads();
  const int64_t lo = blockIdx.x * per_cta, hi = min(n, lo + per_cta);
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(codes);
  const int rw = mw + 1;
  if (mw == 1) {  // 4-byte codes: one 8-byte record store
    uint2* rec2 = reinterpret_cast<uint2*>(rec);
    constexpr int U = 4;
    for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)U * blockDim.x) {
      uint32_t k[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + (int64_t)u * blockDim.x;
        k[u] = i < hi ? __ldg(labels + i) : 0xffffffffu;
        c[u] = i < hi ? __ldg(cw + i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k[u] == 0xffffffffu) continue;
        const uint32_t b = k[u] / tile;
        const uint32_t p = atomicAdd(&cur[b], 1u);
        rec2[p] = make_uint2(c[u], k[u] - b * tile);
      }
    }
    return;
  }
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t k = __ldg(labels + i);
    const uint32_t b = k / tile;
    const uint32_t p = atomicAdd(&cur[b], 1u);
    uint32_t* r = rec + (int64_t)p * rw;
    for (int w = 0; w < mw; ++w) r[w] = __ldg(cw + i * mw + w);
    r[mw] = k - b * tile;
  }
}

// pass 2, sector-staged (4-byte codes, nb * 40 B of shared memory): each bucket keeps a
// 4-record (32-byte) buffer in shared memory and its CTA run cursor; a full buffer leaves
// as one whole sector (two 16-byte stores, sector-aligned: runs are padded to 4 records),
// so no partial line is ever written back to DRAM (the direct scatter's 8-byte stores to
// ~600k open runs read-modify-wrote 2.3 GB at config 4).  Elements go in rounds of one
// per thread: a slot is claimed with a shared atomic; the thread that fills slot 3 flushes
// after a barrier; threads that overflowed a full buffer retry next round.
__global__ void __launch_bounds__(1024) hbin_scatter4_kernel(
    const uint32_t* __restrict__ codes, const uint32_t* __restrict__ labels, int64_t n, int64_t per_cta,
    uint32_t tile, int nb, const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ base,
    uint2* __restrict__ rec) {
  extern __shared__ __align__(16) uint8_t hs4[];
  uint4* buf = reinterpret_cast<uint4*>(hs4);          // [nb][2] (4 records)
  uint32_t* cur = reinterpret_cast<uint32_t*>(hs4 + (size_t)nb * 32);
  uint32_t* fill = cur + nb;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    cur[b] = base[b] + cnt[(int64_t)blockIdx.x * nb + b];
    fill[b] = 0u;
  }
  __syncthreads();
  const int64_t lo = blockIdx.x * per_cta, hi = min(n, lo + per_cta);
  uint2* bufr = reinterpret_cast<uint2*>(hs4);
  for (int64_t i0 = lo; i0 < hi; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool pending = i < hi;
    uint32_t b = 0, s = 0;
    uint2 r = make_uint2(0u, 0u);
    if (pending) {
      const uint32_t k = __ldcs(labels + i);
      b = k / tile;
      r = make_uint2(__ldcs(codes + i), k - b * tile);
    }
    while (__syncthreads_or(pending)) {
      bool flusher = false;
      if (pending) {
        s = atomicAdd(&fill[b], 1u);
        if (s < 4u) {
          bufr[b * 4 + s] = r;
          pending = false;
          flusher = (s == 3u);
        }
      }
      __syncthreads();
      if (flusher) {
        const uint32_t p = cur[b];
        cur[b] = p + 4u;
        fill[b] = 0u;
        uint4* dst = reinterpret_cast<uint4*>(rec + p);
        dst[0] = buf[2 * b];
        dst[1] = buf[2 * b + 1];
      }
      __syncthreads();
    }
  }
  // partial buffers: pad to a whole sector with ~0-label records
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const uint32_t f = fill[b];
    if (f) {
      for (uint32_t q = f; q < 4u; ++q) bufr[b * 4 + q] = make_uint2(0u, 0xffffffffu);
      uint4* dst = reinterpret_cast<uint4*>(rec + cur[b]);
      dst[0] = buf[2 * b];
      dst[1] = buf[2 * b + 1];
    }
  }
}

// pass 3: one CTA per cluster tile — shared-memory counts, dense slab write, counts[k]
__global__ void __launch_bounds__(kHistThreads) hbin_tile_kernel(
    const uint32_t* __restrict__ rec, int mw, const uint32_t* __restrict__ base,
    int tile, int64_t k, int m, int l, uint32_t* __restrict__ hist, uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t sh[];
  const int b = blockIdx.x;
  const int64_t k0 = (int64_t)b * tile;
  const int tk = (int)min((int64_t)tile, k - k0);
  const int row = m * l;  // entries per cluster
  const int ent = tk * row;
  for (int e = threadIdx.x; e < ent; e += blockDim.x) sh[e] = 0;
  __syncthreads();
  const uint32_t lo = base[b], hi = base[b + 1];
  const int rw = mw + 1;
  for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
    const uint32_t* r = rec + p * rw;
    if (r[mw] == 0xffffffffu) continue;  // padding of the sector-staged scatter
    uint32_t* hk = sh + (int)r[mw] * row;
    for (int w = 0; 4 * w < m; ++w) {
      const uint32_t c = r[w];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * w + q < m) atomicAdd(&hk[(4 * w + q) * l + ((c >> (8 * q)) & 0xffu)], 1u);
    }
  }
  __syncthreads();
  uint32_t* dst = hist + k0 * row;
  if ((row & 3) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(sh);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int e = threadIdx.x; e < ent / 4; e += blockDim.x) d4[e] = s4[e];
  } else {
    for (int e = threadIdx.x; e < ent; e += blockDim.x) dst[e] = sh[e];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int t = wid; t < tk; t += blockDim.x >> 5) {
    uint32_t c = 0;
    for (int s = lane; s < l; s += 32) c += sh[t * row + s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[k0 + t] = c;
  }
}

// counts[k] = sum_s hist[k][0][s] (clustering.py:458's bincount): one warp per cluster,
// no contended per-cluster atomics in the histogram pass
__global__ void counts_from_hist_kernel(const uint32_t* __restrict__ hist, int64_t k, int m, int l,
                                        uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t kk = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (kk >= k) return;
  const uint32_t* row = hist + kk * m * l;
  uint32_t c = 0;
  for (int s = lane; s < l; s += 32) c += row[s];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) counts[kk] = c;
}

// ---------------------------------------------------------------------------
// vote
struct Best {
  double v1;
  int l1;
  double v2;
};

__device__ __forceinline__ Best merge_best(const Best& a, const Best& b) {
  Best r;
  if (b.v1 < a.v1 || (b.v1 == a.v1 && b.l1 < a.l1)) {
    r.v1 = b.v1;
    r.l1 = b.l1;
    r.v2 = fmin(a.v1, b.v2);
  } else {
    r.v1 = a.v1;
    r.l1 = a.l1;
    r.v2 = fmin(a.v2, b.v1);
  }
  return r;
}

__device__ __forceinline__ Best shfl_best(const Best& a, int off) {
  Best b;
  b.v1 = __shfl_xor_sync(0xffffffffu, a.v1, off);
  b.l1 = __shfl_xor_sync(0xffffffffu, a.l1, off);
  b.v2 = __shfl_xor_sync(0xffffffffu, a.v2, off);
  return b;
}

struct DD {
  double hi, lo;
  int l;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// a < b in (value, index) order; values closer than 2^-100 relative count as equal.
__device__ __forceinline__ bool dd_less(const DD& a, const DD& b) {
  const double diff = __dadd_rn(__dsub_rn(a.hi, b.hi), __dsub_rn(a.lo, b.lo));
  const double tol = ldexp(fmax(fabs(a.hi), fabs(b.hi)), -100);
  if (diff < -tol) return true;
  if (diff > tol) return false;
  return a.l < b.l;
}

// One warp per (filled cluster k, subspace m), m-major so that concurrently running
// warps share one subspace table.  Lane q owns candidates j = lane + 32*i (i < 8).
// Stage 1 (fp32, table t32): every term h*t >= 0 carries relative error <= 2u (count
// and table conversion) plus one FMA rounding, so a top-2 gap above 4(nnz+3)u32
// proves the exact-arithmetic argmin.  Stage 2 (fp64): any summation order of the
// nnz products is within (nnz+1)u of the exact sum, a gap above 4(nnz+2)u proves it.
// Stage 3 (double-double): near ties; values within 2^-100 relative tie -> lowest j.
constexpr int kVoteWarps = 8;

__device__ __forceinline__ void warp_best(Best& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b = merge_best(b, shfl_best(b, o));
}

// fp16 copy of the fp32 filter tables for the vote's first stage (half the L2 bytes per
// support row): T16 = fp16(T32 * 2^f) with max * 2^f < 2^15 per subspace.  Grid
// (kT16Slices, m): every block of a subspace reduces the whole subspace maximum (256 KB of
// L2 reads, float4) and converts its slice (one block per subspace took 49 us per call).
constexpr int kT16Slices = 32;
__global__ void __launch_bounds__(1024) vote_t16_kernel(const float* __restrict__ t32, int l, __half* __restrict__ t16) {
  __shared__ float s_red[32];
  __shared__ int s_f;
  const float* src = t32 + (size_t)blockIdx.y * l * l;
  __half* dst = t16 + (size_t)blockIdx.y * l * l;
  const int ll = l * l;  // l == 256: a multiple of 4 * kT16Slices
  float mx = 0.0f;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (int i = threadIdx.x; i < ll / 4; i += blockDim.x) {
    const float4 v = __ldg(s4 + i);
    mx = fmaxf(fmaxf(mx, fmaxf(v.x, v.y)), fmaxf(v.z, v.w));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = s_red[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) {
      int ex = 0;
      frexpf(v, &ex);  // v in [2^(ex-1), 2^ex)
      s_f = v > 0.0f ? 15 - ex : 0;
    }
  }
  __syncthreads();
  const int f = s_f;
  const int per = ll / kT16Slices;
  for (int i = blockIdx.x * per + threadIdx.x; i < (blockIdx.x + 1) * per; i += blockDim.x)
    dst[i] = __float2half_rn(ldexpf(src[i], f));
}

// fp16 first stage with the subspace's table staged in shared memory (l = 256).  Grid
// (CTAs per subspace, m): a CTA copies T16[m] (128 KB) once and its 32 warps vote rows
// (k, m) of a contiguous k range, so every support row is a conflict-free 512-byte
// shared read instead of an L2 read (the L2-bound warp-per-row kernel took 96 us at
// config 2).  Same arithmetic and certificate as vote_kernel's fp16 stage; rows it
// cannot certify are appended to a row list for vote_kernel, which goes straight to fp64.
constexpr int kV16Warps = 32;
constexpr size_t kV16Smem = 256 * 256 * sizeof(__half) + (size_t)kV16Warps * 256 * 8;
__global__ void __launch_bounds__(32 * kV16Warps, 1) vote16_smem_kernel(
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ counts, int64_t k, int m, int mp,
    const __half* __restrict__ t16, int64_t rows_per_cta, uint8_t* __restrict__ newc, int32_t* __restrict__ left,
    int32_t* __restrict__ left_count,
    unsigned long long* __restrict__ acc) {
  constexpr int l = 256;
  extern __shared__ __align__(16) uint8_t v16_smem[];
  __half* th = reinterpret_cast<__half*>(v16_smem);
  int* s_s_all = reinterpret_cast<int*>(v16_smem + 256 * 256 * sizeof(__half));
  uint32_t* s_h_all = reinterpret_cast<uint32_t*>(s_s_all + kV16Warps * 256);
  __shared__ unsigned long long s_acc[2];
  const int mm = blockIdx.y;
  {
    const uint4* src = reinterpret_cast<const uint4*>(t16 + (size_t)mm * l * l);
    uint4* dst = reinterpret_cast<uint4*>(th);
    for (int i = threadIdx.x; i < l * l / 8; i += blockDim.x) dst[i] = __ldg(src + i);
    if (threadIdx.x < 2) s_acc[threadIdx.x] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* ss = s_s_all + warp * 256;
  uint32_t* sh = s_h_all + warp * 256;
  const int64_t k_lo = blockIdx.x * rows_per_cta, k_hi = min(k, k_lo + rows_per_cta);
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  unsigned long long my_nnz = 0, my_fail = 0;
  for (int64_t kk = k_lo + warp; kk < k_hi; kk += kV16Warps) {
    const int64_t gw = (int64_t)mm * k + kk;
    if (counts[kk] == 0) continue;
    const uint32_t* hrow = hist + (kk * m + mm) * l;
    uint32_t hv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) hv[i] = hrow[32 * i + lane];
    int nnz = 0;
    unsigned long long hs = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t h = hv[i];
      hs += h;
      const unsigned bal = __ballot_sync(0xffffffffu, h != 0);
      if (h) {
        const int pos = nnz + __popc(bal & ((1u << lane) - 1u));
        ss[pos] = 32 * i + lane;
        sh[pos] = h;
      }
      nnz += __popc(bal);
    }
    __syncwarp();
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0f;
    for (int j = 0; j < nnz; ++j) {
      const float h = __uint2float_rn(sh[j]);
      const uint4 raw = *(reinterpret_cast<const uint4*>(th + ss[j] * l) + lane);
      const __half2* hp = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f2 = __half22float2(hp[i]);
        v[2 * i] = __fmaf_rn(h, f2.x, v[2 * i]);
        v[2 * i + 1] = __fmaf_rn(h, f2.y, v[2 * i + 1]);
      }
    }
    __syncwarp();  // ss/sh are rewritten by the next row
    Best b{inf, 0, inf};
#pragma unroll
    for (int i = 0; i < 8; ++i) b = merge_best(b, Best{(double)v[i], 8 * lane + i, inf});
    warp_best(b);
    const double eps = 4.8828125e-04 + (double)(nnz + 4) * 5.9604644775390625e-08 + 9.5367431640625e-07;
    unsigned long long ht = hs;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, o);
    const double hsum = (double)ht;
    const bool ok = (b.v2 - b.v1) > eps * (b.v1 + b.v2) + 1.1920928955078125e-07 * hsum;
    if (lane == 0) {
      if (ok) {
        newc[kk * mp + mm] = (uint8_t)b.l1;
        my_nnz += (unsigned long long)nnz;  // rows left to vote_kernel count their nnz there
      } else {
        ++my_fail;
        left[atomicAdd(left_count, 1)] = (int32_t)gw;
      }
    }
  }
  if (lane == 0 && (my_nnz | my_fail)) {
    atomicAdd(&s_acc[0], my_nnz);
    atomicAdd(&s_acc[1], my_fail);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_acc[0]) atomicAdd(&acc[0], s_acc[0]);
    if (s_acc[1]) atomicAdd(&acc[3], s_acc[1]);
  }
}

// Tensor-core first stage (l = 256): votes of 128 clusters x 256 candidates per tcgen05
// tile, D[r][j] = sum_s A[r][s] B[j][s] with A = the clusters' count rows (fp16, exact:
// counts < 2048, larger counts split as lo = h & 2047 and hi = h >> 11 into a second TMEM
// accumulator, v = lo + 2048 hi; tiles with a count >= 2^22 go to vote_kernel whole) and
// B[j][s] = T16[s][j] (fp16 tables, transposed through shared memory once per CTA).
// Products are exact in the fp32 accumulator and all addends are nonnegative, so the
// accumulation error is <= 16 instructions x 17 x 2^-23 x v (the encoder's per-instruction
// bound, tools/diag_tc_error.py); with the fp16 table rounding the winner is certified
// when v2 - v1 > eps (v1 + v2) + 2^-23 H, eps = 2^-11 + 272 2^-23 + 2^-20, else the row
// goes to vote_kernel's fp64 path (appended to the undecided-row list).  The dense contraction replaces the
// SIMT stage's sum over the support (issue bound: ~1e9 FMAs + conversions at config 2).
constexpr int kVtcThreads = 256;
constexpr size_t kVtcSmem = 1024 + 256 * 256 * 2 + 128 * 256 * 2;  // align slack + B + A
__global__ void __launch_bounds__(kVtcThreads, 1) vote_tc_kernel(
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ counts, int64_t k, int m, int mp,
    const __half* __restrict__ t16, uint8_t* __restrict__ newc, int32_t* __restrict__ left,
    int32_t* __restrict__ left_count,
    unsigned long long* __restrict__ acc) {
  extern __shared__ __align__(1024) uint8_t vtc_raw[];  // (no-swizzle operands need 16 B alignment)
  uint8_t* smem = vtc_raw;
  uint8_t* sb = smem;                  // B: 256 (j) x 256 (s) fp16, K-major canonical
  uint8_t* sa = smem + 256 * 256 * 2;  // A: 128 (rows) x 256 (s) fp16; staging for the transpose
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ uint32_t row_h[128];  // cluster sizes: < 2^32 by the API contract
  __shared__ int row_nnz[128];
  __shared__ unsigned long long s_acc[2];
  __shared__ double ep_v1[128], ep_v2[128];
  __shared__ int ep_l1[128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mm = blockIdx.y;
  const __half* tsub = t16 + (size_t)mm * 256 * 256;
  // B = T16^T in two 128-row halves staged row-major in the A buffer
  for (int half = 0; half < 2; ++half) {
    const uint4* src = reinterpret_cast<const uint4*>(tsub + (size_t)half * 128 * 256);
    uint4* stg = reinterpret_cast<uint4*>(sa);
    for (int i0 = 0; i0 < 128 * 256 / 8; i0 += 8 * kVtcThreads) {  // 8 loads in flight per thread
      uint4 t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = __ldg(src + i0 + u * kVtcThreads + tid);
#pragma unroll
      for (int u = 0; u < 8; ++u) stg[i0 + u * kVtcThreads + tid] = t[u];
    }
    __syncthreads();
    const __half* st = reinterpret_cast<const __half*>(sa);
    // item (j, g): B[j][s] for s = half*128 + 8g .. +7
    for (int q = tid; q < 256 * 16; q += kVtcThreads) {
      const int j = q & 255, g = q >> 8;
      __align__(16) __half v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = st[(8 * g + e) * 256 + j];
      *reinterpret_cast<uint4*>(sb + tc::kmajor_off(j, half * 128 + 8 * g, 256)) = *reinterpret_cast<uint4*>(v);
    }
    __syncthreads();
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    s_acc[0] = 0;
    s_acc[1] = 0;
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tacc = tbase;
  uint32_t phase = 0;
  unsigned long long my_nnz = 0, my_fail = 0;
  const int64_t ntiles = (k + 127) / 128;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t k0 = tile * 128;
    if (tid < 128) {
      row_h[tid] = 0;
      row_nnz[tid] = 0;
    }
    __syncthreads();
    // A fill: item (r, g) = 8 counts; lanes 0-7 take 8 rows of one core matrix (conflict-free stores)
    uint32_t hmax = 0;
    for (int it0 = 0; it0 < 16; it0 += 8) {  // 8 items (16 loads) in flight per thread
    uint4 ld[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = (it0 + u) * kVtcThreads + tid;
      const int wq = q >> 5, ln = q & 31;
      const int r = (wq & 15) * 8 + (ln & 7), g = (wq >> 4) * 4 + (ln >> 3);
      const int64_t kk = k0 + r;
      ld[u][0] = ld[u][1] = make_uint4(0u, 0u, 0u, 0u);
      if (kk < k) {
        const uint4* src = reinterpret_cast<const uint4*>(hist + (kk * m + mm) * 256 + 8 * g);
        ld[u][0] = __ldg(src);
        ld[u][1] = __ldg(src + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = (it0 + u) * kVtcThreads + tid;
      const int wq = q >> 5, ln = q & 31;
      const int r = (wq & 15) * 8 + (ln & 7), g = (wq >> 4) * 4 + (ln >> 3);
      const uint4 a = ld[u][0], b = ld[u][1];
      const uint32_t h[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t hs = 0;
      int nz = 0;
      __align__(16) __half v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        hs += h[e];
        nz += h[e] != 0;
        hmax = max(hmax, h[e]);
        v[e] = __uint2half_rn(h[e] & 2047u);
      }
      *reinterpret_cast<uint4*>(sa + tc::kmajor_off(r, 8 * g, 256)) = *reinterpret_cast<uint4*>(v);
      // lanes l, l+8, l+16, l+24 share row r: combine, then one shared atomic per row
      hs += __shfl_xor_sync(0xffffffffu, hs, 8);
      hs += __shfl_xor_sync(0xffffffffu, hs, 16);
      nz += __shfl_xor_sync(0xffffffffu, nz, 8);
      nz += __shfl_xor_sync(0xffffffffu, nz, 16);
      if (ln < 8 && hs) {
        atomicAdd(&row_h[r], hs);
        atomicAdd(&row_nnz[r], nz);
      }
    }
    }
    const int need_hi = __syncthreads_or(hmax >= 2048u);
    const int too_big = __syncthreads_or(hmax >= (1u << 22));
    if (too_big) {  // the whole tile to vote_kernel
      if (tid < 128 && k0 + tid < k) {
        const int64_t kk = k0 + tid;
        const bool filled = counts[kk] != 0;
        if (filled) left[atomicAdd(left_count, 1)] = (int32_t)((int64_t)mm * k + kk);
        my_fail += filled;
      }
      __syncthreads();
      continue;
    }
    for (int pass = 0; pass < 1 + need_hi; ++pass) {
      if (pass == 1) {  // refill A with the high parts (the lo MMAs have completed)
        for (int it = 0; it < 16; ++it) {
          const int q = it * kVtcThreads + tid;
          const int wq = q >> 5, ln = q & 31;
          const int r = (wq & 15) * 8 + (ln & 7), g = (wq >> 4) * 4 + (ln >> 3);
          const int64_t kk = k0 + r;
          uint32_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (kk < k) {
            const uint4* src = reinterpret_cast<const uint4*>(hist + (kk * m + mm) * 256 + 8 * g);
            const uint4 a = __ldg(src), b = __ldg(src + 1);
            h[0] = a.x; h[1] = a.y; h[2] = a.z; h[3] = a.w; h[4] = b.x; h[5] = b.y; h[6] = b.z; h[7] = b.w;
          }
          __align__(16) __half v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint2half_rn(h[e] >> 11);
          *reinterpret_cast<uint4*>(sa + tc::kmajor_off(r, 8 * g, 256)) = *reinterpret_cast<uint4*>(v);
        }
      }
      tc::fence_proxy_async();
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      if (tid == 0) {
        const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
        for (int st = 0; st < 16; ++st)
          tc::mma_f16(tacc + 256 * pass, tc::smem_desc(a0 + st * 256, 128, 4096), tc::smem_desc(b0 + st * 256, 128, 4096),
                      tc::idesc_f16_f32(128, 256), st > 0 ? 1u : 0u);
        tc::commit(&bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
      tc::fence_after();
    }
    {
      // warp w reads TMEM lanes 32 (w & 3) .. +31 and candidate columns 128 (w >> 2) .. +127
      const int r = 32 * (warp & 3) + lane, chalf = warp >> 2;
      const uint32_t lrow = tacc + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * chalf;
      double v1, v2;
      int l1;
      if (!need_hi) {  // nonnegative fp32: the bit patterns order as uint32
        uint32_t b1 = 0xffffffffu, b2 = 0xffffffffu;
        int i1 = 0;
        for (int c0 = 0; c0 < 128; c0 += 16) {
          uint32_t lo[16];
          tc::tmem_ld16(lrow + c0, lo);
          tc::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t x = lo[e];
            b2 = min(b2, max(b1, x));  // second smallest (ties keep the lower index as b1)
            if (x < b1) i1 = c0 + e;
            b1 = min(b1, x);
          }
        }
        v1 = (double)__uint_as_float(b1);
        v2 = (double)__uint_as_float(b2);
        l1 = 128 * chalf + i1;
      } else {
        v1 = __longlong_as_double(0x7ff0000000000000LL);
        v2 = v1;
        l1 = 0;
        for (int c0 = 0; c0 < 128; c0 += 16) {
          uint32_t lo[16], hi[16];
          tc::tmem_ld16(lrow + c0, lo);
          tc::tmem_ld16(lrow + 256 + c0, hi);
          tc::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const double v = (double)__uint_as_float(lo[e]) + 2048.0 * (double)__uint_as_float(hi[e]);
            if (v < v1) {
              v2 = v1;
              v1 = v;
              l1 = 128 * chalf + c0 + e;
            } else if (v < v2) {
              v2 = v;
            }
          }
        }
      }
      if (chalf == 1) {
        ep_v1[r] = v1;
        ep_v2[r] = v2;
        ep_l1[r] = l1;
      }
      __syncthreads();
      if (chalf == 0) {
        // merge with the upper half (higher indices: it wins only when strictly smaller)
        const double w1 = ep_v1[r], w2 = ep_v2[r];
        if (w1 < v1) {
          v2 = fmin(v1, w2);
          v1 = w1;
          l1 = ep_l1[r];
        } else {
          v2 = fmin(v2, w1);
        }
        const int64_t kk = k0 + r;
        if (kk < k) {
          const int64_t gw = (int64_t)mm * k + kk;
          if (counts[kk] != 0) {
            const double eps = 4.8828125e-04 + 272.0 * 1.1920928955078125e-07 + 9.5367431640625e-07;
            const bool ok = (v2 - v1) > eps * (v1 + v2) + 1.1920928955078125e-07 * (double)row_h[r];
            if (ok) {
              newc[kk * mp + mm] = (uint8_t)l1;
              my_nnz += (unsigned long long)row_nnz[r];
            } else {
              ++my_fail;
              left[atomicAdd(left_count, 1)] = (int32_t)gw;
            }
          }
        }
      }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // one shared atomic per warp (a 64-bit CAS loop each)
    my_nnz += __shfl_xor_sync(0xffffffffu, my_nnz, o);
    my_fail += __shfl_xor_sync(0xffffffffu, my_fail, o);
  }
  if (lane == 0 && (my_nnz | my_fail)) {
    atomicAdd(&s_acc[0], my_nnz);
    atomicAdd(&s_acc[1], my_fail);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tacc, 512);
  if (tid == 0) {
    if (s_acc[0]) atomicAdd(&acc[0], s_acc[0]);
    if (s_acc[1]) atomicAdd(&acc[3], s_acc[1]);
  }
}

// one (k, m) row per warp (all lanes call it with the same gw)
__device__ __forceinline__ void vote_row(int64_t gw, int* __restrict__ ss, uint32_t* __restrict__ sh,
                                         const uint32_t* __restrict__ hist, const uint32_t* __restrict__ counts,
                                         int64_t k, int m, int l, int mp, const double* __restrict__ t64,
                                         const float* __restrict__ t32, const __half* __restrict__ t16,
                                         uint8_t* __restrict__ newc, unsigned long long* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const int mm = (int)(gw / k);
  const int64_t kk = gw - (int64_t)mm * k;
  if (counts[kk] == 0) return;  // empty: left 0, repaired later
  const uint32_t* hrow = hist + (kk * m + mm) * l;
  int nnz = 0;
  unsigned long long hs = 0;  // sum of this row's counts (the fp16 stage's absolute term)
  for (int base = 0; base < l; base += 32) {
    const int s = base + lane;
    const uint32_t h = (s < l) ? hrow[s] : 0u;
    hs += h;
    const unsigned bal = __ballot_sync(0xffffffffu, h != 0);
    if (h) {
      const int pos = nnz + __popc(bal & ((1u << lane) - 1u));
      ss[pos] = s;
      sh[pos] = h;
    }
    nnz += __popc(bal);
  }
  __syncwarp();
  if (lane == 0) atomicAdd(&acc[0], (unsigned long long)nnz);
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  if (t16) {
    // stage 1 (l = 256): fp16 tables, fp32 FMA.  Lane owns columns 8 lane .. 8 lane + 7 (one
    // 16-byte load per support row).  Per product the table entry carries relative error
    // <= 2^-11 + 2^-23 (fp16 and fp32 roundings) plus 2^-25 absolute (fp16 subnormals);
    // the FMA chain adds <= (nnz + 1) 2^-24 relative.  With H = sum of the counts,
    // |v~_j - v_j| <= eps v~_j + 2^-24 H, eps = 2^-11 + (nnz + 4) 2^-24 + 2^-20; the
    // winner is certified when v~_2 - v~_1 > eps (v~_1 + v~_2) + 2^-23 H.
    const __half* th = t16 + (size_t)mm * l * l;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0f;
    for (int j = 0; j < nnz; ++j) {
      const float h = __uint2float_rn(sh[j]);
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(th + (size_t)ss[j] * l) + lane);
      const __half2* hp = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f2 = __half22float2(hp[i]);
        v[2 * i] = __fmaf_rn(h, f2.x, v[2 * i]);
        v[2 * i + 1] = __fmaf_rn(h, f2.y, v[2 * i + 1]);
      }
    }
    Best b{inf, 0, inf};
#pragma unroll
    for (int i = 0; i < 8; ++i) b = merge_best(b, Best{(double)v[i], 8 * lane + i, inf});
    warp_best(b);
    const double eps = 4.8828125e-04 + (double)(nnz + 4) * 5.9604644775390625e-08 + 9.5367431640625e-07;
    unsigned long long ht = hs;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, o);
    const double hsum = (double)ht;
    if ((b.v2 - b.v1) > eps * (b.v1 + b.v2) + 1.1920928955078125e-07 * hsum) {
      if (lane == 0) newc[kk * mp + mm] = (uint8_t)b.l1;
      return;
    }
    if (lane == 0) atomicAdd(&acc[3], 1ull);
  } else if (t32) {
    const float* tf = t32 + (size_t)mm * l * l;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0f;
    for (int j = 0; j < nnz; ++j) {
      const float h = __uint2float_rn(sh[j]);
      const float* row = tf + (size_t)ss[j] * l;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (lane + 32 * i < l) v[i] = __fmaf_rn(h, __ldg(&row[lane + 32 * i]), v[i]);
    }
    Best b{inf, 0, inf};
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (lane + 32 * i < l) b = merge_best(b, Best{(double)v[i], lane + 32 * i, inf});
    warp_best(b);
    const double margin32 = 4.0 * (double)(nnz + 3) * 5.9604644775390625e-08;
    if ((b.v2 - b.v1) > margin32 * b.v2) {
      if (lane == 0) newc[kk * mp + mm] = (uint8_t)b.l1;
      return;
    }
    if (lane == 0) atomicAdd(&acc[3], 1ull);
  }
  const double* td = t64 + (size_t)mm * l * l;
  {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0;
    for (int j = 0; j < nnz; ++j) {
      const double h = (double)sh[j];
      const double* row = td + (size_t)ss[j] * l;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (lane + 32 * i < l) v[i] = __fma_rn(h, __ldg(&row[lane + 32 * i]), v[i]);
    }
    Best b{inf, 0, inf};
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (lane + 32 * i < l) b = merge_best(b, Best{v[i], lane + 32 * i, inf});
    warp_best(b);
    const double margin = 4.0 * (double)(nnz + 2) * ldexp(1.0, -53);
    if ((b.v2 - b.v1) > margin * b.v2) {
      if (lane == 0) newc[kk * mp + mm] = (uint8_t)b.l1;
      return;
    }
  }
  // near tie: double-double sums (exact products via FMA, compensated additions)
  DD d{inf, 0.0, 0x7fffffff};
  for (int i = 0; i < 8; ++i) {
    const int c = lane + 32 * i;
    if (c >= l) break;
    double hi = 0.0, lo = 0.0;
    for (int j = 0; j < nnz; ++j) {
      const double h = (double)sh[j];
      const double t = __ldg(&td[(size_t)ss[j] * l + c]);
      const double p = __dmul_rn(h, t);
      const double pe = __fma_rn(h, t, -p);
      double s, e;
      two_sum(hi, p, s, e);
      e = __dadd_rn(e, __dadd_rn(lo, pe));
      hi = __dadd_rn(s, e);
      lo = __dsub_rn(e, __dsub_rn(hi, s));
    }
    const DD cand{hi, lo, c};
    if (dd_less(cand, d)) d = cand;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DD od;
    od.hi = __shfl_xor_sync(0xffffffffu, d.hi, o);
    od.lo = __shfl_xor_sync(0xffffffffu, d.lo, o);
    od.l = __shfl_xor_sync(0xffffffffu, d.l, o);
    if (dd_less(od, d)) d = od;
  }
  if (lane == 0) {
    newc[kk * mp + mm] = (uint8_t)d.l;
    atomicAdd(&acc[1], 1ull);
  }
}

// rows = nullptr: one warp per (k, m) row; otherwise a grid-stride loop over the *count rows
// the first stage (vote_tc_kernel / vote16_smem_kernel) could not certify
__global__ void __launch_bounds__(32 * kVoteWarps) vote_kernel(const uint32_t* __restrict__ hist,
                                                               const uint32_t* __restrict__ counts, int64_t k, int m,
                                                               int l, int mp, const double* __restrict__ t64,
                                                               const float* __restrict__ t32,
                                                               const __half* __restrict__ t16,
                                                               const int32_t* __restrict__ rows,
                                                               const int32_t* __restrict__ row_count,
                                                               uint8_t* __restrict__ newc,
                                                               unsigned long long* __restrict__ acc) {
  __shared__ int s_s[kVoteWarps][kMaxL];
  __shared__ uint32_t s_h[kVoteWarps][kMaxL];
  const int warp = threadIdx.x >> 5;
  if (rows) {
    const int64_t cnt = *row_count;
    for (int64_t i = (int64_t)blockIdx.x * kVoteWarps + warp; i < cnt; i += (int64_t)gridDim.x * kVoteWarps)
      vote_row(rows[i], s_s[warp], s_h[warp], hist, counts, k, m, l, mp, t64, t32, t16, newc, acc);
  } else {
    const int64_t gw = (int64_t)blockIdx.x * kVoteWarps + warp;
    if (gw < k * m) vote_row(gw, s_s[warp], s_h[warp], hist, counts, k, m, l, mp, t64, t32, t16, newc, acc);
  }
}

// ---------------------------------------------------------------------------
// order-preserving compaction of a flag array (two kernels; blockDim == 1024)
__global__ void empty_count_kernel(const uint32_t* __restrict__ counts, int64_t k, int32_t* __restrict__ blockcnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int f = (i < k) && counts[i] == 0;
  const int c = __syncthreads_count(f);
  if (threadIdx.x == 0) blockcnt[blockIdx.x] = c;
}

__global__ void empty_compact_kernel(const uint32_t* __restrict__ counts, int64_t k,
                                     const int32_t* __restrict__ blockcnt, int32_t* __restrict__ empty_list) {
  __shared__ int s_off;
  __shared__ int s_warp[32];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < (int)blockIdx.x; ++b) s += blockcnt[b];
    s_off = s;
  }
  const int f = (i < k) && counts[i] == 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  const int pre = __popc(bal & ((1u << lane) - 1u));
  if (lane == 31) s_warp[warp] = pre + f;
  __syncthreads();
  if (warp == 0) {
    const int v = s_warp[lane];
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_warp[lane] = x - v;
  }
  __syncthreads();
  if (f) empty_list[s_off + s_warp[warp] + pre] = (int32_t)i;
}

// number of empty clusters (acc[2]) and the public vote stats
__global__ void empties_kernel(const uint32_t* __restrict__ counts, int64_t k, unsigned long long* __restrict__ acc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c = __syncthreads_count((i < k) && counts[i] == 0);
  if (threadIdx.x == 0 && c) atomicAdd(&acc[2], (unsigned long long)c);
}

__global__ void vote_stats_kernel(int64_t k, const unsigned long long* __restrict__ acc, int64_t* __restrict__ stats) {
  stats[PQK_STAT_NNZ_TOTAL] = (int64_t)acc[0];
  stats[PQK_STAT_VOTE_EXACT] = (int64_t)acc[1];
  stats[PQK_STAT_EMPTY] = (int64_t)acc[2];
  stats[PQK_STAT_FILLED] = k - (int64_t)acc[2];
  stats[PQK_STAT_VOTE_FP64] = (int64_t)acc[3];
}

// ---------------------------------------------------------------------------
// repair: radix select of the top-E 96-bit keys (sd bits desc, index asc)
struct SelState {
  unsigned long long prefix_hi;
  unsigned int prefix_lo;
  unsigned int pad;
  long long remaining;
  unsigned long long count;
};

__device__ __forceinline__ void comp_key(const double* sd, int64_t i, int64_t base, uint64_t& hi, uint32_t& lo) {
  hi = (uint64_t)__double_as_longlong(sd[i]);
  lo = ~(uint32_t)(base + i);
}

// digit pass p (0..11): p<8 -> bits of hi from the top, else bits of lo from the top.
__device__ __forceinline__ bool sel_match(uint64_t hi, uint32_t lo, int p, const SelState& st, int& digit) {
  if (p < 8) {
    const int sh = 56 - 8 * p;
    const uint64_t mask_hi = (p == 0) ? 0ull : (~0ull << (sh + 8));
    if ((hi & mask_hi) != (st.prefix_hi & mask_hi)) return false;
    digit = (int)((hi >> sh) & 0xff);
    return true;
  }
  if (hi != st.prefix_hi) return false;
  const int q = p - 8;
  const int sh = 24 - 8 * q;
  const uint32_t mask_lo = (q == 0) ? 0u : (~0u << (sh + 8));
  if ((lo & mask_lo) != (st.prefix_lo & mask_lo)) return false;
  digit = (int)((lo >> sh) & 0xff);
  return true;
}

__global__ void sel_hist_kernel(const double* __restrict__ sd, int64_t n, int64_t base, int p,
                                const SelState* __restrict__ stp, unsigned int* __restrict__ ghist) {
  __shared__ unsigned int h[256];
  const SelState st = *stp;
  if (st.remaining <= 0) return;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t hi;
    uint32_t lo;
    comp_key(sd, i, base, hi, lo);
    int d;
    if (sel_match(hi, lo, p, st, d)) atomicAdd(&h[d], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&ghist[i], h[i]);
}

__global__ void sel_choose_kernel(int p, SelState* stp, unsigned int* ghist) {
  if (threadIdx.x == 0) {
    SelState st = *stp;
    if (st.remaining > 0) {
      long long cum = 0;
      int dstar = 0;
      for (int d = 255; d >= 0; --d) {
        const long long c = ghist[d];
        if (cum + c >= st.remaining) {
          dstar = d;
          break;
        }
        cum += c;
      }
      st.remaining -= cum;
      if (p < 8)
        st.prefix_hi |= (unsigned long long)dstar << (56 - 8 * p);
      else
        st.prefix_lo |= (unsigned int)dstar << (24 - 8 * (p - 8));
      *stp = st;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) ghist[i] = 0;
}

__global__ void sel_init_kernel(SelState* st, unsigned int* ghist, const int64_t* __restrict__ e_src, int64_t e_const,
                                int64_t n) {
  if (threadIdx.x == 0) {
    int64_t e = e_src ? e_src[PQK_STAT_EMPTY] : e_const;
    if (e > n) e = n;
    st->prefix_hi = 0;
    st->prefix_lo = 0;
    st->remaining = e;
    st->count = 0;
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) ghist[i] = 0;
}

// after 12 passes the prefix is the E-th largest key exactly (keys are unique)
__global__ void sel_collect_kernel(const double* __restrict__ sd, int64_t n, int64_t base, SelState* stp,
                                   uint64_t* __restrict__ ck_hi, uint32_t* __restrict__ ck_lo,
                                   const int64_t* __restrict__ e_src, int64_t e_const) {
  const int64_t e = e_src ? e_src[PQK_STAT_EMPTY] : e_const;
  if (e <= 0) return;
  const uint64_t th = stp->prefix_hi;
  const uint32_t tl = stp->prefix_lo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t hi;
    uint32_t lo;
    comp_key(sd, i, base, hi, lo);
    if (hi > th || (hi == th && lo >= tl)) {
      const unsigned long long pos = atomicAdd(&stp->count, 1ull);
      ck_hi[pos] = hi;
      ck_lo[pos] = lo;
    }
  }
}

// Descending sort of the (exactly E, unique) candidates: a bitonic network over P = the
// power of two >= the workspace capacity min(N, K) (fixed at launch, so the repair graph
// replays for any E), keys padded with (0, 0), which is below every real key (lo =
// ~index >= 1 since indices are < 2^32 - 1).  Stages with partner distance < 2048 run in
// shared memory (one block = 2048 keys); the longer ones are one global pass each:
// log2(P/2048) * (log2(P/2048) + 1) / 2 + log2(P/2048) + 1 launches, O(P log^2 P) work
// (E = 1e5: 28 launches, ~1e7 compare-exchanges) instead of the O(E^2) rank count.
constexpr int kSortTile = 2048;

__device__ __forceinline__ bool key_less(uint64_t ah, uint32_t al, uint64_t bh, uint32_t bl) {
  return ah < bh || (ah == bh && al < bl);
}

// compare-exchange of i and i^j inside stage k (overall order descending)
__device__ __forceinline__ void cmpx(uint64_t* hi, uint32_t* lo, int64_t gi, int i, int j, int64_t k) {
  const int p = i ^ j;
  if (p > i) {
    const bool desc = (gi & k) == 0;
    const bool sw = desc ? key_less(hi[i], lo[i], hi[p], lo[p]) : key_less(hi[p], lo[p], hi[i], lo[i]);
    if (sw) {
      const uint64_t th = hi[i];
      const uint32_t tl = lo[i];
      hi[i] = hi[p];
      lo[i] = lo[p];
      hi[p] = th;
      lo[p] = tl;
    }
  }
}

// load (with padding) and sort each 2048-key tile: stages k = 2 .. 2048
__global__ void __launch_bounds__(1024) sort_tile_kernel(const SelState* __restrict__ stp,
                                                         const uint64_t* __restrict__ ck_hi,
                                                         const uint32_t* __restrict__ ck_lo, uint64_t* __restrict__ s_hi,
                                                         uint32_t* __restrict__ s_lo) {
  __shared__ uint64_t hi[kSortTile];
  __shared__ uint32_t lo[kSortTile];
  const int64_t cnt = (int64_t)stp->count;
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    const int64_t g = base + t;
    hi[t] = g < cnt ? ck_hi[g] : 0ull;
    lo[t] = g < cnt ? ck_lo[g] : 0u;
  }
  __syncthreads();
  for (int k = 2; k <= kSortTile; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < kSortTile; t += blockDim.x) cmpx(hi, lo, base + t, t, j, k);
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    s_hi[base + t] = hi[t];
    s_lo[base + t] = lo[t];
  }
}

// one global compare-exchange pass (partner distance j >= 2048) of stage k
__global__ void sort_global_kernel(uint64_t* __restrict__ s_hi, uint32_t* __restrict__ s_lo, int64_t p, int64_t j,
                                   int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = i ^ j;
    if (q <= i) continue;
    const bool desc = (i & k) == 0;
    const uint64_t ah = s_hi[i], bh = s_hi[q];
    const uint32_t al = s_lo[i], bl = s_lo[q];
    if (desc ? key_less(ah, al, bh, bl) : key_less(bh, bl, ah, al)) {
      s_hi[i] = bh;
      s_lo[i] = bl;
      s_hi[q] = ah;
      s_lo[q] = al;
    }
  }
}

// the remaining distances j = 1024 .. 1 of stage k, in shared memory per tile
__global__ void __launch_bounds__(1024) sort_merge_tile_kernel(uint64_t* __restrict__ s_hi, uint32_t* __restrict__ s_lo,
                                                               int64_t k) {
  __shared__ uint64_t hi[kSortTile];
  __shared__ uint32_t lo[kSortTile];
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    hi[t] = s_hi[base + t];
    lo[t] = s_lo[base + t];
  }
  __syncthreads();
  for (int j = kSortTile >> 1; j > 0; j >>= 1) {
    for (int t = threadIdx.x; t < kSortTile; t += blockDim.x) cmpx(hi, lo, base + t, t, j, k);
    __syncthreads();
  }
  for (int t = threadIdx.x; t < kSortTile; t += blockDim.x) {
    s_hi[base + t] = hi[t];
    s_lo[base + t] = lo[t];
  }
}

static int64_t sort_extent(int64_t cap) {
  int64_t p = kSortTile;
  while (p < cap) p <<= 1;
  return p;
}

__global__ void repair_apply_kernel(const SelState* __restrict__ stp, const uint32_t* __restrict__ sorted_lo,
                                    const int32_t* __restrict__ empty_list, const uint8_t* __restrict__ codes,
                                    int mp, uint8_t* __restrict__ newc) {
  const int64_t cnt = (int64_t)stp->count;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < cnt; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = (int64_t)(~sorted_lo[r]);
    const int64_t kk = empty_list[r];
    for (int j = 0; j < mp; ++j) newc[kk * mp + j] = codes[idx * mp + j];
  }
}

__global__ void cand_out_kernel(const SelState* __restrict__ stp, const uint64_t* __restrict__ s_hi,
                                const uint32_t* __restrict__ s_lo, uint64_t* __restrict__ out_keys,
                                int64_t* __restrict__ out_index) {
  const int64_t cnt = (int64_t)stp->count;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < cnt; r += (int64_t)gridDim.x * blockDim.x) {
    out_keys[r] = s_hi[r];
    out_index[r] = (int64_t)(~s_lo[r]);
  }
}

// ---------------------------------------------------------------------------
// numpy pairwise-sum objective
__device__ __forceinline__ void leaf_pairwise(const double* __restrict__ a, int n, bool do_sqrt, double& res) {
  auto val = [&](int i) { return do_sqrt ? __dsqrt_rn(a[i]) : a[i]; };
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, val(i));
    res = r;
    return;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = val(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], val(i + j));
  }
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) s = __dadd_rn(s, val(i));
  res = s;
}

// Eight lanes per leaf: lane j owns numpy's accumulator r[j] (elements 8i+j), the
// three shuffle levels add ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), lane 0 adds the
// n%8 tail sequentially; leaves shorter than 8 are summed sequentially from 0.0.
__global__ void obj_leaf8_kernel(const double* __restrict__ sd, int64_t nleaves, const int64_t* __restrict__ leaf_off,
                                 const int32_t* __restrict__ leaf_len, double2* __restrict__ leafval) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, j = lane & 7;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t0 = warp * 4; t0 < nleaves; t0 += nwarps * 4) {
    const int64_t t = t0 + grp;
    const bool valid = t < nleaves;
    const int n = valid ? leaf_len[t] : 0;
    const double* a = sd + (valid ? leaf_off[t] : 0);
    double r1 = 0.0, r2 = 0.0;
    const int nb = n - (n % 8);
    if (n >= 8) {
      r2 = __ldcs(a + j);
      r1 = __dsqrt_rn(r2);
      int i = 8;
      // four loads in flight per lane, then the sequential (numpy-order) adds
      for (; i + 32 <= nb; i += 32) {
        double x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = __ldcs(a + i + 8 * q + j);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          r2 = __dadd_rn(r2, x[q]);
          r1 = __dadd_rn(r1, __dsqrt_rn(x[q]));
        }
      }
      for (; i < nb; i += 8) {
        const double x = __ldcs(a + i + j);
        r2 = __dadd_rn(r2, x);
        r1 = __dadd_rn(r1, __dsqrt_rn(x));
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const double y1 = __shfl_xor_sync(0xffffffffu, r1, o);
      const double y2 = __shfl_xor_sync(0xffffffffu, r2, o);
      r1 = __dadd_rn(r1, y1);
      r2 = __dadd_rn(r2, y2);
    }
    if (valid && j == 0) {
      if (n < 8) {
        r1 = 0.0;
        r2 = 0.0;
      }
      for (int i = (n < 8 ? 0 : nb); i < n; ++i) {
        const double x = a[i];
        r2 = __dadd_rn(r2, x);
        r1 = __dadd_rn(r1, __dsqrt_rn(x));
      }
      leafval[t] = make_double2(r1, r2);
    }
  }
}

__global__ void obj_level_kernel(int64_t start, int64_t count, int64_t child_start, const int32_t* __restrict__ na,
                                 const int32_t* __restrict__ nb, const double2* __restrict__ leafval,
                                 double2* __restrict__ nodeval) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = start + t;
    const int a = na[id], b = nb[id];
    double2 r;
    if (b < 0) {
      r = leafval[a];
    } else {
      const double2 x = nodeval[child_start + a];
      const double2 y = nodeval[child_start + b];
      r = make_double2(__dadd_rn(x.x, y.x), __dadd_rn(x.y, y.y));
    }
    nodeval[id] = r;
  }
}

struct DepthStarts {
  long long v[64];
};

// All remaining (small, <= 4096-node) levels, deepest first, in one CTA; writes the root
// sums.  Each level's values stay in shared memory for the next one (the first tail level
// reads its children from nodeval, leaves from leafval), so a level costs a barrier, not
// a global round trip.
constexpr int kObjTailMax = 4096;
__global__ void __launch_bounds__(1024) obj_levels_tail_kernel(int top_depth, DepthStarts ds,
                                                               const int32_t* __restrict__ na,
                                                               const int32_t* __restrict__ nb,
                                                               const double2* __restrict__ leafval,
                                                               const double2* __restrict__ nodeval,
                                                               double* __restrict__ out2) {
  extern __shared__ double2 s_tail[];  // [2][kObjTailMax]
  double2(*sbuf)[kObjTailMax] = reinterpret_cast<double2(*)[kObjTailMax]>(s_tail);
  int cur = 0;
  bool prev_smem = false;
  for (int d = top_depth; d >= 0; --d) {
    const int64_t start = ds.v[d], count = ds.v[d + 1] - ds.v[d], child = ds.v[d + 1];
    const double2* prev = sbuf[cur ^ 1];
    for (int64_t t = threadIdx.x; t < count; t += blockDim.x) {
      const int64_t id = start + t;
      const int a = __ldg(na + id), b = __ldg(nb + id);
      double2 r;
      if (b < 0) {
        r = __ldg(leafval + a);
      } else {
        const double2 x = prev_smem ? prev[a] : __ldg(nodeval + child + a);
        const double2 y = prev_smem ? prev[b] : __ldg(nodeval + child + b);
        r = make_double2(__dadd_rn(x.x, y.x), __dadd_rn(x.y, y.y));
      }
      sbuf[cur][t] = r;
    }
    __syncthreads();
    cur ^= 1;
    prev_smem = true;
  }
  if (threadIdx.x == 0) {
    out2[0] = sbuf[cur ^ 1][0].x;
    out2[1] = sbuf[cur ^ 1][0].y;
  }
}

// ---------------------------------------------------------------------------
struct RepairWS {
  SelState* st;
  unsigned int* ghist;
  unsigned long long* acc;
  int32_t* blockcnt;
  int32_t* empty_list;
  uint64_t* ck_hi;
  uint32_t* ck_lo;
  uint64_t* s_hi;  // sorted candidates, sort_p entries (power of two >= capacity)
  uint32_t* s_lo;
  int64_t sort_p;
  size_t total;
};

static RepairWS repair_layout(void* base, int64_t n, int64_t k) {
  RepairWS w{};
  const int64_t cap = std::max<int64_t>(1, std::min(n, k));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = align_up(off, 256);
    const size_t o = off;
    off += bytes;
    return o;
  };
  const size_t o_st = take(sizeof(SelState));
  const size_t o_gh = take(256 * sizeof(unsigned int));
  const size_t o_acc = take(4 * sizeof(unsigned long long));
  const size_t o_bc = take(((k + 1023) / 1024 + 1) * sizeof(int32_t));
  const size_t o_el = take(std::max<int64_t>(k, 1) * sizeof(int32_t));
  const size_t o_ch = take(cap * sizeof(uint64_t));
  const size_t o_cl = take(cap * sizeof(uint32_t));
  w.sort_p = sort_extent(cap);
  const size_t o_sh = take(w.sort_p * sizeof(uint64_t));
  const size_t o_sl = take(w.sort_p * sizeof(uint32_t));
  w.total = align_up(off, 256);
  char* b = static_cast<char*>(base);
  if (b) {
    w.st = reinterpret_cast<SelState*>(b + o_st);
    w.ghist = reinterpret_cast<unsigned int*>(b + o_gh);
    w.acc = reinterpret_cast<unsigned long long*>(b + o_acc);
    w.blockcnt = reinterpret_cast<int32_t*>(b + o_bc);
    w.empty_list = reinterpret_cast<int32_t*>(b + o_el);
    w.ck_hi = reinterpret_cast<uint64_t*>(b + o_ch);
    w.ck_lo = reinterpret_cast<uint32_t*>(b + o_cl);
    w.s_hi = reinterpret_cast<uint64_t*>(b + o_sh);
    w.s_lo = reinterpret_cast<uint32_t*>(b + o_sl);
  }
  return w;
}

static int run_select(const double* d_sd, int64_t n, int64_t base, const int64_t* e_src, int64_t e_const,
                      RepairWS& w, cudaStream_t stream) {
  const DevInfo& di = dev_info();
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)di.sms * 4));
  sel_init_kernel<<<1, 256, 0, stream>>>(w.st, w.ghist, e_src, e_const, n);
  PQK_LAUNCH_CHECK("sel_init_kernel");
  for (int p = 0; p < 12; ++p) {
    sel_hist_kernel<<<grid, 256, 0, stream>>>(d_sd, n, base, p, w.st, w.ghist);
    PQK_LAUNCH_CHECK("sel_hist_kernel");
    sel_choose_kernel<<<1, 256, 0, stream>>>(p, w.st, w.ghist);
    PQK_LAUNCH_CHECK("sel_choose_kernel");
  }
  sel_collect_kernel<<<grid, 256, 0, stream>>>(d_sd, n, base, w.st, w.ck_hi, w.ck_lo, e_src, e_const);
  PQK_LAUNCH_CHECK("sel_collect_kernel");
  const int64_t p = w.sort_p;
  sort_tile_kernel<<<(unsigned)(p / kSortTile), 1024, 0, stream>>>(w.st, w.ck_hi, w.ck_lo, w.s_hi, w.s_lo);
  PQK_LAUNCH_CHECK("sort_tile_kernel");
  for (int64_t k = 2 * kSortTile; k <= p; k <<= 1) {
    for (int64_t j = k >> 1; j >= kSortTile; j >>= 1) {
      sort_global_kernel<<<(unsigned)std::min<int64_t>((p + 255) / 256, (int64_t)di.sms * 8), 256, 0, stream>>>(
          w.s_hi, w.s_lo, p, j, k);
      PQK_LAUNCH_CHECK("sort_global_kernel");
    }
    sort_merge_tile_kernel<<<(unsigned)(p / kSortTile), 1024, 0, stream>>>(w.s_hi, w.s_lo, k);
    PQK_LAUNCH_CHECK("sort_merge_tile_kernel");
  }
  return PQK_OK;
}

}  // namespace pqk

using namespace pqk;

// stream-ordered allocations (cudaMallocAsync: valid inside a CUDA-graph capture) keep
// their freed blocks in the device's default pool (no OS round trip per call)
static int keep_default_pool() {
  static bool kept[64] = {};
  int dev = 0;
  PQK_CUDA_TRY(cudaGetDevice(&dev));
  if (!kept[dev & 63]) {
    cudaMemPool_t pool;
    PQK_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    PQK_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    kept[dev & 63] = true;
  }
  return PQK_OK;
}



extern "C" int pqk_histogram_device(const uint8_t* d_codes, int64_t n, int32_t m, int32_t l,
                                    const uint32_t* d_labels, int64_t k, uint32_t* d_hist, uint32_t* d_counts,
                                    void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int mp = padded_m(m);
  if (mp == 0 || l < 1 || l > kMaxL || k < 1 || n < 0) return fail(PQK_EINVAL, "pqk_histogram_device: bad arguments");
  if (n > (int64_t)UINT32_MAX) return fail(PQK_EUNSUPPORTED, "pqk_histogram_device: n must be < 2^32 (uint32 counts)");
  const int tile = std::min(255, std::max(1, kHistTileBytes / (m * l * 4)));
  const int64_t nb = (k + tile - 1) / tile;
  // PQK_HIST_MODE=atomic|tiled forces a path (tests, tools/diag_hist.py); by default tables
  // that stay L2 resident (config 2's 41 MB) use the plain atomics, which are faster there
  static const int mode = [] {
    const char* e = getenv("PQK_HIST_MODE");
    return !e ? 0 : (e[0] == 'a' ? 1 : (e[0] == 't' ? 2 : 0));
  }();
  const bool small_table = (double)k * m * l * 4 <= 64.0 * (1 << 20);
  const bool tiled_ok = nb <= kHistMaxBuckets && (int64_t)m * l * 4 <= kHistTileBytes;
  if (tiled_ok && (mode == 2 || (mode == 0 && !small_table))) {
    const DevInfo& di = dev_info();
    const int nbi = (int)nb;
    // open-line budget of the scatter: ctas x buckets x 128 B <= frontier
    static const double frontier = [] {
      const char* e = getenv("PQK_HIST_FRONTIER_MB");
      return (e ? atof(e) : 96.0) * (1 << 20);
    }();
    // (measured at config 4, 4167 buckets: 47 CTAs 4.7 ms scatter, 188 CTAs 3.9 ms, 296 CTAs
    // 8.1 ms with 13 GB of DRAM read-modify-write; the scatter is store-transaction bound)
    const int mw = mp / 4;
    // sector-staged scatter (4-byte codes, bucket buffers in shared memory, one CTA per SM);
    // PQK_HIST_STAGED=0 keeps the direct scatter (diagnostic)
    static const bool staged_on = [] {
      const char* e = getenv("PQK_HIST_STAGED");
      return !(e && e[0] == '0');
    }();
    const size_t staged_smem = (size_t)nbi * 40;
    const bool staged = staged_on && mw == 1 && staged_smem <= (size_t)di.smem_optin &&
                        (double)n + 3.0 * di.sms * nbi < 4294967295.0;
    const int ctas = staged ? di.sms
                            : (int)std::max<int64_t>(di.sms, std::min<int64_t>(di.sms * 2, (int64_t)(frontier / (128.0 * nbi))));
    const int64_t per_cta = std::max<int64_t>((n + ctas - 1) / ctas, 1);
    const size_t cnt_b = align_up((size_t)ctas * nbi * 4, 256), base_b = align_up((size_t)(nbi + 1) * 4, 256);
    const int64_t nrec = std::max<int64_t>(n, 1) + (staged ? 3LL * ctas * nbi : 0);  // + sector padding
    const size_t rec_b = align_up((size_t)nrec * (mw + 1) * 4, 256);
    { const int _rc = keep_default_pool(); if (_rc != PQK_OK) return _rc; }
    uint8_t* ws = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), cnt_b + base_b + rec_b, stream) != cudaSuccess) {
      (void)cudaGetLastError();  // no room for the bucketed records: the atomic path below
      ws = nullptr;
    }
    if (ws) {
      uint32_t* cnt = reinterpret_cast<uint32_t*>(ws);
      uint32_t* base = reinterpret_cast<uint32_t*>(ws + cnt_b);
      uint32_t* rec = reinterpret_cast<uint32_t*>(ws + cnt_b + base_b);
      const size_t sm_nb = (size_t)nbi * 4;
      static int smem_set[64] = {};
      int dev = 0;
      PQK_CUDA_TRY(cudaGetDevice(&dev));
      if (!smem_set[dev & 63]) {
        PQK_CUDA_TRY(cudaFuncSetAttribute(hbin_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistMaxBuckets * 4));
        PQK_CUDA_TRY(cudaFuncSetAttribute(hbin_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistMaxBuckets * 4));
        PQK_CUDA_TRY(cudaFuncSetAttribute(hbin_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistTileBytes));
        PQK_CUDA_TRY(cudaFuncSetAttribute(hbin_scatter4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, di.smem_optin));
        smem_set[dev & 63] = 1;
      }
      hbin_count_kernel<<<ctas, kHistThreads, sm_nb, stream>>>(d_labels, n, per_cta, (uint32_t)tile, nbi, cnt,
                                                               staged ? 1 : 0);
      PQK_LAUNCH_CHECK("hbin_count_kernel");
      hbin_colscan_kernel<<<(nbi + 255) / 256, 256, 0, stream>>>(cnt, ctas, nbi, base);
      PQK_LAUNCH_CHECK("hbin_colscan_kernel");
      hbin_scan_kernel<<<1, 1024, 0, stream>>>(base, nbi);
      PQK_LAUNCH_CHECK("hbin_scan_kernel");
      if (staged) {
        hbin_scatter4_kernel<<<ctas, 1024, staged_smem, stream>>>(reinterpret_cast<const uint32_t*>(d_codes), d_labels,
                                                                   n, per_cta, (uint32_t)tile, nbi, cnt, base,
                                                                   reinterpret_cast<uint2*>(rec));
        PQK_LAUNCH_CHECK("hbin_scatter4_kernel");
      } else {
        hbin_scatter_kernel<<<ctas, 1024, sm_nb, stream>>>(d_codes, mw, d_labels, n, per_cta, (uint32_t)tile, nbi, cnt,
                                                           base, rec);
        PQK_LAUNCH_CHECK("hbin_scatter_kernel");
      }
      hbin_tile_kernel<<<nbi, kHistThreads, (size_t)tile * m * l * 4, stream>>>(rec, mw, base, tile, k, m, l, d_hist,
                                                                               d_counts);
      PQK_LAUNCH_CHECK("hbin_tile_kernel");
      PQK_CUDA_TRY(cudaFreeAsync(ws, stream));
      return PQK_OK;
    }
  }
  PQK_CUDA_TRY(cudaMemsetAsync(d_hist, 0, (size_t)k * m * l * sizeof(int32_t), stream));
  if (n > 0) {
    const DevInfo& di = dev_info();
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)di.sms * 8);
    histogram_kernel<<<grid, 256, 0, stream>>>(d_codes, n, mp, m, l, d_labels, d_hist);
    PQK_LAUNCH_CHECK("histogram_kernel");
  }
  counts_from_hist_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, stream>>>(d_hist, k, m, l, d_counts);
  PQK_LAUNCH_CHECK("counts_from_hist_kernel");
  return PQK_OK;
}

extern "C" int pqk_vote_tables16_device(const float* d_t32, int32_t m, int32_t l, void* d_t16, void* stream) {
  if (!d_t32 || !d_t16 || m < 1 || l != 256) return fail(PQK_EINVAL, "pqk_vote_tables16_device: bad arguments");
  vote_t16_kernel<<<dim3(kT16Slices, m), 1024, 0, (cudaStream_t)stream>>>(d_t32, l, (__half*)d_t16);
  PQK_LAUNCH_CHECK("vote_t16_kernel");
  return PQK_OK;
}

static int vote_impl(const uint32_t* d_hist, const uint32_t* d_counts, int64_t k, int32_t m, int32_t l,
                     const double* d_t64, const float* d_t32, const __half* t16_given, uint8_t* d_new_centers,
                     int64_t* d_stats, void* stream_);

// d_stats has PQK_STATS_LEN slots: 0..15 public, 16..19 scratch accumulators of the vote.
extern "C" int pqk_vote_device(const uint32_t* d_hist, const uint32_t* d_counts, int64_t k, int32_t m, int32_t l,
                               const double* d_t64, const float* d_t32, uint8_t* d_new_centers, int64_t* d_stats,
                               void* stream) {
  return vote_impl(d_hist, d_counts, k, m, l, d_t64, d_t32, nullptr, d_new_centers, d_stats, stream);
}

extern "C" int pqk_vote16_device(const uint32_t* d_hist, const uint32_t* d_counts, int64_t k, int32_t m, int32_t l,
                                 const double* d_t64, const float* d_t32, const void* d_t16,
                                 uint8_t* d_new_centers, int64_t* d_stats, void* stream) {
  if (d_t16 && (!d_t32 || l != 256)) return fail(PQK_EINVAL, "pqk_vote16_device: d_t16 needs d_t32 and l == 256");
  return vote_impl(d_hist, d_counts, k, m, l, d_t64, d_t32, (const __half*)d_t16, d_new_centers, d_stats, stream);
}

static int vote_impl(const uint32_t* d_hist, const uint32_t* d_counts, int64_t k, int32_t m, int32_t l,
                     const double* d_t64, const float* d_t32, const __half* t16_given, uint8_t* d_new_centers,
                     int64_t* d_stats, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int mp = padded_m(m);
  if (mp == 0 || l < 2 || l > kMaxL || k < 1 || !d_stats) return fail(PQK_EINVAL, "pqk_vote_device: bad arguments");
  if ((int64_t)k * m >= ((int64_t)1 << 31)) return fail(PQK_EUNSUPPORTED, "pqk_vote_device: k*m too large");
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(d_stats + 16);
  PQK_CUDA_TRY(cudaMemsetAsync(acc, 0, 4 * sizeof(unsigned long long), stream));
  PQK_CUDA_TRY(cudaMemsetAsync(d_new_centers, 0, (size_t)k * mp, stream));
  // fp16 first-stage tables, rebuilt every call (the tables may differ between calls) in
  // stream-ordered memory (cudaMallocAsync: also valid inside a CUDA-graph capture)
  const __half* t16 = t16_given;  // prebuilt by pqk_vote_tables16_device (constant tables)
  __half* t16_own = nullptr;
  if (!t16 && d_t32 && l == 256) {
    { const int _rc = keep_default_pool(); if (_rc != PQK_OK) return _rc; }
    PQK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t16_own), (size_t)m * l * l * sizeof(__half), stream));
    vote_t16_kernel<<<dim3(kT16Slices, m), 1024, 0, stream>>>(d_t32, l, t16_own);
    PQK_LAUNCH_CHECK("vote_t16_kernel");
    t16 = t16_own;
  }
  int32_t* left = nullptr;  // [0] = count, then the rows the first stage left undecided
  if (t16) {
    // fp16 stage from shared-memory tables; vote_kernel then takes the uncertified rows to fp64
    static int attr_v16[64] = {};
    int dev = 0;
    PQK_CUDA_TRY(cudaGetDevice(&dev));
    if (!attr_v16[dev & 63]) {
      PQK_CUDA_TRY(cudaFuncSetAttribute(vote16_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kV16Smem));
      PQK_CUDA_TRY(cudaFuncSetAttribute(vote_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVtcSmem));
      attr_v16[dev & 63] = 1;
    }
    PQK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&left), ((size_t)k * m + 4) * sizeof(int32_t), stream));
    PQK_CUDA_TRY(cudaMemsetAsync(left, 0, sizeof(int32_t), stream));
    const int per = std::max(1, dev_info().sms / m);
    static const bool simt = [] {
      const char* e = getenv("PQK_VOTE_SIMT");
      return e && e[0] == '1';
    }();
    if (simt) {
      const int64_t rows = (k + per - 1) / per;
      vote16_smem_kernel<<<dim3(per, m), 32 * kV16Warps, kV16Smem, stream>>>(d_hist, d_counts, k, m, mp, t16, rows,
                                                                             d_new_centers, left + 4, left, acc);
      PQK_LAUNCH_CHECK("vote16_smem_kernel");
    } else {
      const int64_t tiles = (k + 127) / 128;
      const int per_tc = (int)std::min<int64_t>(per, tiles);
      vote_tc_kernel<<<dim3(per_tc, m), kVtcThreads, kVtcSmem, stream>>>(d_hist, d_counts, k, m, mp, t16,
                                                                          d_new_centers, left + 4, left, acc);
      PQK_LAUNCH_CHECK("vote_tc_kernel");
    }
  }
  if (left) {  // the undecided rows only (fp64 stage), grid-stride over the device-side count
    const int grid = (int)std::min<int64_t>((k * m + kVoteWarps - 1) / kVoteWarps, (int64_t)dev_info().sms * 8);
    vote_kernel<<<grid, 32 * kVoteWarps, 0, stream>>>(d_hist, d_counts, k, m, l, mp, d_t64, nullptr, nullptr,
                                                      left + 4, left, d_new_centers, acc);
  } else {
    vote_kernel<<<(unsigned)((k * m + kVoteWarps - 1) / kVoteWarps), 32 * kVoteWarps, 0, stream>>>(
        d_hist, d_counts, k, m, l, mp, d_t64, d_t32, t16, nullptr, nullptr, d_new_centers, acc);
  }
  PQK_LAUNCH_CHECK("vote_kernel");
  if (t16_own) PQK_CUDA_TRY(cudaFreeAsync(t16_own, stream));
  if (left) PQK_CUDA_TRY(cudaFreeAsync(left, stream));
  empties_kernel<<<(unsigned)((k + 1023) / 1024), 1024, 0, stream>>>(d_counts, k, acc);
  PQK_LAUNCH_CHECK("empties_kernel");
  vote_stats_kernel<<<1, 1, 0, stream>>>(k, acc, d_stats);
  PQK_LAUNCH_CHECK("vote_stats_kernel");
  return PQK_OK;
}

extern "C" size_t pqk_repair_workspace_bytes(int64_t n, int64_t k) {
  if (n < 0 || k < 1) return 0;
  return repair_layout(nullptr, n, k).total;
}

extern "C" int pqk_repair_device(const double* d_sd_sq, const uint8_t* d_codes, int64_t n, int32_t m,
                                 const uint32_t* d_counts, int64_t k, uint8_t* d_new_centers, void* d_ws,
                                 size_t ws_bytes, int64_t* d_stats, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int mp = padded_m(m);
  if (mp == 0 || k < 1 || n < 1 || !d_ws || !d_stats) return fail(PQK_EINVAL, "pqk_repair_device: bad arguments");
  if (n > ((int64_t)1 << 32)) return fail(PQK_EUNSUPPORTED, "pqk_repair_device: n must be <= 2^32 (32-bit key index)");
  RepairWS w = repair_layout(d_ws, n, k);
  if (ws_bytes < w.total) return fail(PQK_EINVAL, "pqk_repair_device: workspace too small");
  const int kb = (int)((k + 1023) / 1024);
  // empty clusters in ascending k; E itself is d_stats[PQK_STAT_EMPTY] from pqk_vote_device
  empty_count_kernel<<<kb, 1024, 0, stream>>>(d_counts, k, w.blockcnt);
  PQK_LAUNCH_CHECK("empty_count_kernel");
  empty_compact_kernel<<<kb, 1024, 0, stream>>>(d_counts, k, w.blockcnt, w.empty_list);
  PQK_LAUNCH_CHECK("empty_compact_kernel");
  int rc = run_select(d_sd_sq, n, 0, d_stats, 0, w, stream);
  if (rc != PQK_OK) return rc;
  const DevInfo& di = dev_info();
  repair_apply_kernel<<<di.sms, 256, 0, stream>>>(w.st, w.s_lo, w.empty_list, d_codes, mp, d_new_centers);
  PQK_LAUNCH_CHECK("repair_apply_kernel");
  return PQK_OK;
}

extern "C" int pqk_repair_candidates_device(const double* d_sd_sq, int64_t n, int64_t base_index, int64_t e,
                                            void* d_ws, size_t ws_bytes, uint64_t* d_out_keys, int64_t* d_out_index,
                                            void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n < 1 || e < 0 || base_index < 0 || !d_ws) return fail(PQK_EINVAL, "pqk_repair_candidates_device: bad arguments");
  if (base_index + n > ((int64_t)1 << 32))
    return fail(PQK_EUNSUPPORTED, "pqk_repair_candidates_device: base_index + n must be <= 2^32 (32-bit key index)");
  if (e == 0) return PQK_OK;
  RepairWS w = repair_layout(d_ws, n, std::max<int64_t>(e, 1));
  if (ws_bytes < w.total) return fail(PQK_EINVAL, "pqk_repair_candidates_device: workspace too small");
  int rc = run_select(d_sd_sq, n, base_index, nullptr, std::min(e, n), w, stream);
  if (rc != PQK_OK) return rc;
  const DevInfo& di = dev_info();
  cand_out_kernel<<<di.sms, 256, 0, stream>>>(w.st, w.s_hi, w.s_lo, d_out_keys, d_out_index);
  PQK_LAUNCH_CHECK("cand_out_kernel");
  return PQK_OK;
}

extern "C" size_t pqk_objective_workspace_bytes(int64_t nleaves, int64_t nnodes) {
  return align_up((size_t)std::max<int64_t>(nleaves, 1) * sizeof(double2), 256) +
         (size_t)std::max<int64_t>(nnodes, 1) * sizeof(double2);
}

extern "C" int pqk_objective_device(const double* d_sd_sq, int64_t n, int64_t nleaves, int32_t ndepth,
                                    const int64_t* d_leaf_off, const int32_t* d_leaf_len,
                                    const int64_t* h_depth_start, const int32_t* d_node_a,
                                    const int32_t* d_node_b, void* d_ws, size_t ws_bytes, double* d_out2,
                                    void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n < 1 || nleaves < 1 || ndepth < 1 || !h_depth_start || !d_ws)
    return fail(PQK_EINVAL, "pqk_objective_device: bad arguments");
  const int64_t nnodes = h_depth_start[ndepth];
  if (ws_bytes < pqk_objective_workspace_bytes(nleaves, nnodes))
    return fail(PQK_EINVAL, "pqk_objective_device: workspace too small");
  double2* leafval = reinterpret_cast<double2*>(d_ws);
  double2* nodeval = reinterpret_cast<double2*>(static_cast<char*>(d_ws) +
                                                align_up((size_t)nleaves * sizeof(double2), 256));
  const DevInfo& di = dev_info();
  if (ndepth > 63) return fail(PQK_EUNSUPPORTED, "pqk_objective_device: tree too deep");
  {
    const int64_t warps = (nleaves + 3) / 4;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)di.sms * 16));
    obj_leaf8_kernel<<<grid, 256, 0, stream>>>(d_sd_sq, nleaves, d_leaf_off, d_leaf_len, leafval);
    PQK_LAUNCH_CHECK("obj_leaf8_kernel");
  }
  // the tail kernel takes the top levels 0..tail_top, every one of them <= kObjTailMax nodes
  // (an unbalanced tree's deepest levels can be small while shallower ones are not)
  int tail_top = 0;
  while (tail_top + 1 < ndepth && h_depth_start[tail_top + 2] - h_depth_start[tail_top + 1] <= kObjTailMax) ++tail_top;
  int d = ndepth - 1;
  for (; d > tail_top; --d) {
    const int64_t start = h_depth_start[d];
    const int64_t count = h_depth_start[d + 1] - start;
    const int64_t child = h_depth_start[d + 1];
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)di.sms * 8));
    obj_level_kernel<<<grid, 256, 0, stream>>>(start, count, child, d_node_a, d_node_b, leafval, nodeval);
    PQK_LAUNCH_CHECK("obj_level_kernel");
  }
  DepthStarts ds{};
  for (int i = 0; i <= ndepth; ++i) ds.v[i] = h_depth_start[i];
  {
    static bool attr[64] = {};
    int dev = 0;
    PQK_CUDA_TRY(cudaGetDevice(&dev));
    if (!attr[dev & 63]) {
      PQK_CUDA_TRY(cudaFuncSetAttribute(obj_levels_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(2 * kObjTailMax * sizeof(double2))));
      attr[dev & 63] = true;
    }
  }
  obj_levels_tail_kernel<<<1, 1024, 2 * kObjTailMax * sizeof(double2), stream>>>(d, ds, d_node_a, d_node_b, leafval,
                                                                                 nodeval, d_out2);
  PQK_LAUNCH_CHECK("obj_levels_tail_kernel");
  return PQK_OK;
}
