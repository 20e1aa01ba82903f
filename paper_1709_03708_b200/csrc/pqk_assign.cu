// pqk_assign.cu — nearest-center assignment of PQ codes on sm_100a.
//
// Replaces the reference linear scan (clustering.py:167-197): for every code n,
//   labels[n] = argmin_k fl64(((0 + T_0[x^0][c_k^0]) + T_1[x^1][c_k^1]) + ...)
// (float64, ascending m, np.argmin lowest index on ties, clustering.py:183-188)
// and the winner's float64 distance sd_sq[n] (pq.py:287-290 as called at
// clustering.py:447), bit-identical to the reference.
//
// Pipeline per call (all stream-ordered, no host sync):
//   1. dedup   : distinct center codes, each represented by its lowest original
//                index, kept in ascending-index order (pos -> idx).  Identical
//                center rows tie exactly in any precision, so scanning only the
//                representatives and returning the representative index is the
//                reference tie rule.
//   2. qbuild  : the restricted tables of the distinct centers, chunked for the
//                scan:  Q[t][s][m][j] = T32[m][s][c_{t*KC+j}^m]  (fp32, scaled by a
//                power of two), KC centers per chunk.  This is the reference's
//                `restricted` (clustering.py:177-180) re-laid out for shared memory.
//   3. scan    : persistent kernel, one CTA per SM.  A producer thread streams the
//                chunks through an S-stage shared-memory ring with cp.async.bulk
//                (TMA engine) + mbarriers; 11 consumer warps hold their codes and
//                running (best, runner-up) keys in registers and do pure
//                LDS.128 + FADD + IMNMX over the chunk.  fp32 sums are a filter:
//                a code is certified when the runner-up exceeds the winner by more
//                than the fp32 error bound, which proves the fp64 winner is the same
//                center; the fp64 distance of the winner is then recomputed exactly.
//   4. rescan  : codes that were not certified (near ties) get an exact fp64 scan
//                over all distinct centers (ascending m, __dadd_rn, lowest index).
//
// Shared-memory layout and bank conflicts.  A chunk row s holds, for every
// subspace m, the KC candidate values T[m][s][c_j^m]: row = MP*KC*4 bytes, the
// m-slab at byte m*KC*4.  A lane reads one float4 (4 centers) of one subspace of
// one code per LDS.128.  An LDS.128 is served in quarter-warp phases of 8 lanes;
// the 8 lanes of a phase serve P = 8/H codes (H = KC/4 lanes per code).  Code slot
// c of the phase reads subspace m = (c + i) mod MP at step i, so the P codes of a
// phase always hit P distinct m-slabs, i.e. disjoint banks, whatever their code
// bytes are: every LDS.128 is 4 conflict-free wavefronts (128 B each).
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>

#include "pqk_common.cuh"
#include "pqk_hscan.cuh"
#include "pqk_hscan8.cuh"

namespace pqk {

// ---------------------------------------------------------------------------
// small kernels
__global__ void tables_to_f32_kernel(const double* __restrict__ t64, int m, int l, int mp, int exp2,
                                     float* __restrict__ t32) {
  const size_t ll = (size_t)l * l;
  const size_t total = (size_t)mp * ll;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t mm = i / ll;
    t32[i] = (mm < (size_t)m) ? (float)ldexp(t64[i], exp2) : 0.0f;
  }
}

__global__ void pad_codes_kernel(const uint8_t* __restrict__ raw, int64_t n, int m, int mp,
                                 uint8_t* __restrict__ out) {
  const int64_t total = n * mp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / mp;
    const int j = (int)(i - r * mp);
    out[i] = j < m ? raw[r * m + j] : (uint8_t)0;
  }
}

// ---------------------------------------------------------------------------
// center dedup (hash, lowest index per distinct code, order-preserving compaction)
__device__ __forceinline__ bool code_eq(const uint8_t* __restrict__ cs, int mp, int a, int b) {
  const uint32_t* pa = reinterpret_cast<const uint32_t*>(cs + (size_t)a * mp);
  const uint32_t* pb = reinterpret_cast<const uint32_t*>(cs + (size_t)b * mp);
  for (int w = 0; w < mp / 4; ++w)
    if (pa[w] != pb[w]) return false;
  return true;
}

__device__ __forceinline__ uint32_t code_hash(const uint8_t* __restrict__ cs, int mp, int a) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(cs + (size_t)a * mp);
  uint32_t h = 0x9e3779b9u;
  for (int w = 0; w < mp / 4; ++w) h = mix32(h ^ (p[w] + 0x85ebca6bu * (uint32_t)w));
  return h;
}

__global__ void dedup_insert_kernel(const uint8_t* __restrict__ cs, int k, int mp, int32_t* hash, uint32_t mask) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  uint32_t h = code_hash(cs, mp, i) & mask;
  while (true) {
    const int cur = atomicCAS(&hash[h], -1, i);
    if (cur == -1) return;
    if (code_eq(cs, mp, cur, i)) {
      atomicMin(&hash[h], i);
      return;
    }
    h = (h + 1) & mask;
  }
}

__global__ void dedup_mark_kernel(const uint8_t* __restrict__ cs, int k, int mp, const int32_t* __restrict__ hash,
                                  uint32_t mask, int32_t* __restrict__ rep, int32_t* __restrict__ blockcnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int is_rep = 0;
  if (i < k) {
    uint32_t h = code_hash(cs, mp, i) & mask;
    while (true) {
      const int cur = hash[h];
      if (cur >= 0 && code_eq(cs, mp, cur, i)) {
        rep[i] = cur;
        is_rep = (cur == i);
        break;
      }
      h = (h + 1) & mask;
    }
  }
  const int cnt = __syncthreads_count(is_rep);
  if (threadIdx.x == 0) blockcnt[blockIdx.x] = cnt;
}

// blockDim == 1024
__global__ void dedup_compact_kernel(const uint8_t* __restrict__ cs, int k, int mp, int kc,
                                     const int32_t* __restrict__ rep, const int32_t* __restrict__ blockcnt,
                                     int32_t* __restrict__ pos2idx, uint8_t* __restrict__ ucodes,
                                     int32_t* __restrict__ counters) {
  __shared__ int s_off;
  __shared__ int s_warp[32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < (int)blockIdx.x; ++b) s += blockcnt[b];
    s_off = s;
  }
  const int is_rep = (i < k) && (rep[i] == i);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, is_rep);
  const int pre = __popc(bal & ((1u << lane) - 1u));
  if (lane == 31) s_warp[warp] = pre + is_rep;
  __syncthreads();
  if (warp == 0) {
    const int v = s_warp[lane];
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_warp[lane] = x - v;  // exclusive
    if (lane == 31 && blockIdx.x == gridDim.x - 1) {
      const int total = s_off + x;
      counters[0] = total;
      counters[2] = (total + kc - 1) / kc;
    }
  }
  __syncthreads();
  if (is_rep) {
    const int pos = s_off + s_warp[warp] + pre;
    pos2idx[pos] = i;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(cs + (size_t)i * mp);
    uint32_t* dst = reinterpret_cast<uint32_t*>(ucodes + (size_t)pos * mp);
    for (int w = 0; w < mp / 4; ++w) dst[w] = src[w];
  }
}

// ---------------------------------------------------------------------------
// restricted-table chunks
template <int MP, int KC>
__global__ void qbuild_kernel(const float* __restrict__ t32, int l, const uint8_t* __restrict__ ucodes,
                              const int32_t* __restrict__ counters, float4* __restrict__ q,
                              const int32_t* __restrict__ gate = nullptr, int32_t gate_min = 0) {
  if (gate && *gate < gate_min) return;  // the fp32 list tier will not run
  const int U = counters[0];
  const int nchunks = (U + KC - 1) / KC;
  constexpr int Q4 = KC / 4;
  const int64_t units = (int64_t)nchunks * l * MP * Q4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < units; i += (int64_t)gridDim.x * blockDim.x) {
    const int q4 = (int)(i % Q4);
    int64_t r = i / Q4;
    const int mm = (int)(r % MP);
    r /= MP;
    const int s = (int)(r % l);
    const int t = (int)(r / l);
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int u = t * KC + q4 * 4 + j;
      v[j] = (u < U) ? t32[((size_t)mm * l + ucodes[(size_t)u * MP + mm]) * l + s] : __int_as_float(0x7f800000);
    }
    q[i] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// ---------------------------------------------------------------------------
// the scan
struct ScanParams {
  const uint8_t* codes;
  int64_t n;
  const float* q;
  int l;
  int m;
  const int32_t* counters;  // [0] U, [1] flagged, [2] nchunks
  const int32_t* pos2idx;
  const uint8_t* ucodes;
  const double* t64;
  double cert_factor;
  uint32_t* labels;
  double* sd_sq;
  int32_t* flags;
  int32_t* flag_count;
  int64_t pass_size;
  int64_t npasses;
  // list mode (second filter tier): scan the codes list[0 .. *list_count), but only when
  // *list_count >= list_min (smaller lists go to the exact rescan); pass sizes derived
  // on the device so the launch needs no host sync
  const int32_t* list;
  const int32_t* list_count;
  int32_t list_min;
};

template <int W>
__device__ __forceinline__ void load_rotated(const uint8_t* __restrict__ codes, int idx, bool valid, int c,
                                             uint32_t (&out)[W]) {
  uint32_t w[W];
  if (valid) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(codes + (size_t)idx * (4 * W));
    if constexpr (W == 1) {
      w[0] = __ldg(p);
    } else if constexpr (W == 2) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
      w[0] = v.x;
      w[1] = v.y;
    } else {
#pragma unroll
      for (int k = 0; k < W; k += 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + k / 4);
        w[k] = v.x;
        w[k + 1] = v.y;
        w[k + 2] = v.z;
        w[k + 3] = v.w;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = 0u;
  }
  // rotate left by c bytes: out byte i = code byte (c + i) mod MP (c < 8)
  const int qw = (W == 1) ? 0 : (c >> 2);
  const int rb = (W == 1) ? (c & 3) : (c & 3);
  uint32_t u[W];
#pragma unroll
  for (int k = 0; k < W; ++k) u[k] = qw ? w[(k + 1) % W] : w[k];
#pragma unroll
  for (int k = 0; k < W; ++k) out[k] = __funnelshift_r(u[k], u[(k + 1) % W], 8 * rb);
}

template <int MP, int KC, int C, int NW, int S, bool LIST = false>
__global__ void __launch_bounds__((NW + 1) * 32, 1) scan_kernel(const ScanParams p) {
  constexpr int H = KC / 4;       // lanes per code
  constexpr int OWN_W = 32 / H;   // code owners per warp
  constexpr int OWN = NW * OWN_W; // code owners per CTA
  constexpr int ROW = MP * KC * 4;
  constexpr int P = 8 / H;        // codes per LDS.128 phase
  constexpr int W = MP / 4;
  static_assert(MP % P == 0, "MP must be a multiple of the phase width");

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  uint8_t* stages = smem + 128;
  const uint32_t chunk_bytes = (uint32_t)p.l * ROW;
  const int nchunks = p.counters[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  int n;
  int pass_size;
  int64_t npasses;
  if (p.list) {
    n = *p.list_count;
    if (n < p.list_min || n == 0) return;
    pass_size = (int)min((int64_t)OWN * C, ((int64_t)n + G - 1) / G);
    npasses = ((int64_t)n + pass_size - 1) / pass_size;
  } else {
    n = (int)p.n;
    pass_size = (int)p.pass_size;
    npasses = p.npasses;
  }
  const int64_t my_passes = (npasses > blockIdx.x) ? (npasses - blockIdx.x + G - 1) / G : 0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer: stream chunks through the ring ----------------
    if (lane == 0) {
      const int64_t total = my_passes * nchunks;
      const char* src = reinterpret_cast<const char*>(p.q);
      int t = 0;
      for (int64_t g = 0; g < total; ++g) {
        const int st = (int)(g % S);
        const uint32_t ph = (uint32_t)((g / S) & 1);
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&full[st], chunk_bytes);
        bulk_g2s(stages + (size_t)st * chunk_bytes, src + (size_t)t * chunk_bytes, chunk_bytes, &full[st]);
        if (++t == nchunks) t = 0;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int o = lane / H;
  const int c = o % P;
  const int h = lane % H;
  uint32_t lc[MP];
#pragma unroll
  for (int i = 0; i < MP; ++i) lc[i] = (uint32_t)(((c + i) % MP) * (KC * 4) + h * 16);
  const uint32_t stage0 = smem_u32(stages);

  uint32_t g = 0;
  for (int pi = 0; pi < (int)my_passes; ++pi) {
    const int base = ((int)blockIdx.x + pi * (int)G) * pass_size;
    const int end = min(n, base + pass_size);
    const int my0 = base + warp * OWN_W + o;  // code of slot j: my0 + j*OWN

    uint32_t cw[C][W];
    uint32_t bk[C], sk[C], bc[C];
    int rid[C];  // code row (list mode: list[position])
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int pos = my0 + j * OWN;
      const int idx = (p.list && pos < end) ? __ldg(&p.list[pos]) : pos;
      rid[j] = idx;
      load_rotated<W>(p.codes, idx, pos < end, c, cw[j]);
      bk[j] = 0xffffffffu;
      sk[j] = 0xffffffffu;
      bc[j] = 0u;
    }

    // list tier: slots past the end of this warp's share of the list are skipped
    // (warp-uniform), so a short list costs its codes, not the full register capacity
    int jact = C;
    if (LIST) {
      const int rem = end - (base + warp * OWN_W);
      jact = rem <= 0 ? 0 : min(C, (rem + OWN - 1) / OWN);
    }
    for (int t = 0; t < nchunks; ++t, ++g) {
      const int st = (int)(g % S);
      const uint32_t ph = (g / S) & 1u;
      mbar_wait(&full[st], ph);
      const uint32_t sb = stage0 + (uint32_t)st * chunk_bytes;
      uint32_t lcs[MP];
#pragma unroll
      for (int i = 0; i < MP; ++i) lcs[i] = sb + lc[i];
      // software pipeline: the LDS.128s of code j+1 are in flight while code j is reduced
      float4 buf[2][MP];
#pragma unroll
      for (int i = 0; i < MP; ++i)
        buf[0][i] = lds128(__byte_perm(cw[0][i >> 2], 0u, 0x4440u | (uint32_t)(i & 3)) * ROW + lcs[i]);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        if (LIST && j >= jact) break;
        if (j + 1 < C && (!LIST || j + 1 < jact)) {
#pragma unroll
          for (int i = 0; i < MP; ++i)
            buf[(j + 1) & 1][i] =
                lds128(__byte_perm(cw[j + 1][i >> 2], 0u, 0x4440u | (uint32_t)(i & 3)) * ROW + lcs[i]);
        }
        float4* v = buf[j & 1];
        // pairwise tree over the MP subspace terms (any order is covered by the certificate)
#pragma unroll
        for (int w = 1; w < MP; w *= 2) {
#pragma unroll
          for (int i = 0; i + w < MP; i += 2 * w) {
            v[i].x += v[i + w].x;
            v[i].y += v[i + w].y;
            v[i].z += v[i + w].z;
            v[i].w += v[i + w].w;
          }
        }
        const uint32_t k0 = (__float_as_uint(v[0].x) & ~3u);
        const uint32_t k1 = (__float_as_uint(v[0].y) & ~3u) | 1u;
        const uint32_t k2 = (__float_as_uint(v[0].z) & ~3u) | 2u;
        const uint32_t k3 = (__float_as_uint(v[0].w) & ~3u) | 3u;
        const uint32_t lo01 = min(k0, k1), hi01 = max(k0, k1);
        const uint32_t lo23 = min(k2, k3), hi23 = max(k2, k3);
        const uint32_t lo = min(lo01, lo23);
        const uint32_t mid = min(max(lo01, lo23), min(hi01, hi23));
        bc[j] = (lo < bk[j]) ? (uint32_t)t : bc[j];
        sk[j] = min(max(bk[j], lo), min(sk[j], mid));
        bk[j] = min(bk[j], lo);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }

    // ---------------- finalize: merge lanes, certify, exact fp64 distance ----------------
#pragma unroll
    for (int j = 0; j < C; ++j) {
      uint32_t b = bk[j], s = sk[j];
      uint32_t ci = bc[j] * KC + h * 4 + (b & 3u);
      if constexpr (H == 2) {
        const uint32_t ob = __shfl_xor_sync(0xffffffffu, b, 1);
        const uint32_t os = __shfl_xor_sync(0xffffffffu, s, 1);
        const uint32_t oci = __shfl_xor_sync(0xffffffffu, ci, 1);
        const uint32_t ns = min(max(b, ob), min(s, os));
        if (ob < b || (ob == b && oci < ci)) {
          b = ob;
          ci = oci;
        }
        s = ns;
      }
      const int idx = rid[j];
      if (h == 0 && my0 + j * OWN < end) {
        const uint32_t sm = s & ~3u;
        bool cert;
        if (sm >= 0x7f800000u) {
          cert = true;  // no finite runner-up (a single distinct center)
        } else {
          const float fbh = __uint_as_float((b & ~3u) + 3u);
          const float fsl = __uint_as_float(sm);
          cert = (double)fsl > (double)fbh * p.cert_factor;
        }
        if (cert) {
          const uint8_t* xc = p.codes + (size_t)idx * MP;
          const uint8_t* cc = p.ucodes + (size_t)ci * MP;
          double acc = 0.0;
          for (int mm = 0; mm < p.m; ++mm)
            acc = dadd(acc, __ldg(&p.t64[((size_t)mm * p.l + xc[mm]) * p.l + cc[mm]]));
          p.labels[idx] = (uint32_t)__ldg(&p.pos2idx[ci]);
          p.sd_sq[idx] = acc;
        } else {
          const int f = atomicAdd(p.flag_count, 1);
          p.flags[f] = idx;
        }
      }
    }
  }
}

// exact float64 scan over all distinct centers; one warp per code.
// all_mode: every code (fp64-only tables or unsupported MP); else the flagged list.
__global__ void rescan_kernel(const uint8_t* __restrict__ codes, int64_t n, int mp, int m, int l,
                              const uint8_t* __restrict__ ucodes, const int32_t* __restrict__ counters,
                              const int32_t* __restrict__ flags, const int32_t* __restrict__ flag_count,
                              const int32_t* __restrict__ pos2idx, const double* __restrict__ t64,
                              uint32_t* __restrict__ labels, double* __restrict__ sd_sq, int all_mode,
                              int32_t max_count) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nf = all_mode ? n : (int64_t)(*flag_count);
  if (!all_mode && nf >= max_count) return;  // the list went to the fp32 list scan
  const int U = counters[0];
  for (int64_t w = gw; w < nf; w += nw) {
    const int64_t idx = all_mode ? w : (int64_t)flags[w];
    const uint8_t* xc = codes + idx * mp;
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bu = 0x7fffffff;
    for (int u = lane; u < U; u += 32) {
      const uint8_t* cc = ucodes + (size_t)u * mp;
      double d = 0.0;
      for (int mm = 0; mm < m; ++mm) d = dadd(d, __ldg(&t64[((size_t)mm * l + xc[mm]) * l + cc[mm]]));
      if (d < best) {
        best = d;
        bu = u;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int ou = __shfl_xor_sync(0xffffffffu, bu, off);
      if (ob < best || (ob == best && ou < bu)) {
        best = ob;
        bu = ou;
      }
    }
    if (lane == 0) {
      labels[idx] = (uint32_t)pos2idx[bu];
      sd_sq[idx] = best;
    }
  }
}

// Same exact scan, one CTA per code: the code's M float64 table rows T[m][x^m][:]
// are staged in shared memory, threads stride over the distinct centers.
__global__ void __launch_bounds__(256) rescan_cta_kernel(
    const uint8_t* __restrict__ codes, int64_t n, int mp, int m, int l, const uint8_t* __restrict__ ucodes,
    const int32_t* __restrict__ counters, const int32_t* __restrict__ flags, const int32_t* __restrict__ flag_count,
    const int32_t* __restrict__ pos2idx, const double* __restrict__ t64, uint32_t* __restrict__ labels,
    double* __restrict__ sd_sq, int all_mode, int32_t max_count) {
  extern __shared__ double s_rows[];  // m * l
  __shared__ double s_best[8];
  __shared__ int s_bu[8];
  const int64_t nf = all_mode ? n : (int64_t)(*flag_count);
  if (!all_mode && nf >= max_count) return;  // the list went to the fp32 list scan
  const int U = counters[0];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t f = blockIdx.x; f < nf; f += gridDim.x) {
    const int64_t idx = all_mode ? f : (int64_t)flags[f];
    const uint8_t* xc = codes + idx * mp;
    __syncthreads();
    for (int e = tid; e < m * l; e += blockDim.x) {
      const int mm = e / l, s = e - mm * l;
      s_rows[e] = __ldg(&t64[((size_t)mm * l + xc[mm]) * l + s]);
    }
    __syncthreads();
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bu = 0x7fffffff;
    // 4 centres per thread per step (independent code loads and add chains), visited in
    // ascending index order per thread, so that ties keep the lowest index
    const int bd = (int)blockDim.x;
    for (int u0 = tid; u0 < U; u0 += 4 * bd) {
      double d[4] = {0.0, 0.0, 0.0, 0.0};
      for (int w = 0; 4 * w < m; ++w) {
        uint32_t cw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int u = u0 + q * bd;
          cw[q] = u < U ? __ldg(reinterpret_cast<const uint32_t*>(ucodes + (size_t)u * mp) + w) : 0u;
        }
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          const int mm = 4 * w + bb;
          if (mm < m) {
#pragma unroll
            for (int q = 0; q < 4; ++q) d[q] = dadd(d[q], s_rows[mm * l + ((cw[q] >> (8 * bb)) & 0xffu)]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * bd;
        if (u < U && d[q] < best) {
          best = d[q];
          bu = u;
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int ou = __shfl_xor_sync(0xffffffffu, bu, off);
      if (ob < best || (ob == best && ou < bu)) {
        best = ob;
        bu = ou;
      }
    }
    if (lane == 0) {
      s_best[warp] = best;
      s_bu[warp] = bu;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (s_best[w] < best || (s_best[w] == best && s_bu[w] < bu)) {
          best = s_best[w];
          bu = s_bu[w];
        }
      labels[idx] = (uint32_t)pos2idx[bu];
      sd_sq[idx] = best;
    }
  }
}

// first window sets the statistics, later windows add their flagged codes
// kc_tier > 0: a fixed-point first tier ran (chunks of kc_tier centres, lookup_bytes per lookup)
__global__ void assign_stats_kernel(const int32_t* __restrict__ counters, int64_t* __restrict__ stats, int first,
                                    int kc_tier, int lookup_bytes, int32_t list_min) {
  stats[PQK_STAT_UNIQUE_CENTERS] = counters[0];
  stats[PQK_STAT_FLAGGED] = (first ? 0 : stats[PQK_STAT_FLAGGED]) + counters[1];
  // codes decided by the exact rescan: the first-tier list when short, else what the
  // fp32 list tier left
  const int32_t exact = !kc_tier ? counters[1] : (counters[1] < list_min ? counters[1] : counters[3]);
  stats[PQK_STAT_FLAGGED_FP64] = (first ? 0 : stats[PQK_STAT_FLAGGED_FP64]) + exact;
  stats[PQK_STAT_NCHUNKS] = kc_tier ? (counters[0] + kc_tier - 1) / kc_tier : counters[2];
  stats[PQK_STAT_LOOKUP_BYTES] = lookup_bytes;
}

__global__ void paired_distance_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                       const uint32_t* __restrict__ idx, int64_t n, int mp, int m, int l,
                                       const double* __restrict__ t64, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* xa = a + i * mp;
    const uint8_t* xb = b + (idx ? (int64_t)idx[i] : i) * mp;
    double acc = 0.0;
    for (int mm = 0; mm < m; ++mm) acc = dadd(acc, t64[((size_t)mm * l + xa[mm]) * l + xb[mm]]);
    out[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// host side
DevInfo& dev_info() {
  static DevInfo info[64];
  int dev = 0;
  cudaGetDevice(&dev);
  DevInfo& d = info[dev & 63];
  if (d.sms == 0) {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return d;
}

static inline int kc_for(int mp) { return mp == 4 ? 8 : 4; }

struct AssignWS {
  int32_t* hash;
  int32_t* rep;
  int32_t* blockcnt;
  int32_t* pos2idx;
  uint8_t* ucodes;
  float* q;
  int32_t* flags;
  int32_t* counters;
  uint32_t hash_size;
  size_t total;
  // 16-bit fixed-point first tier
  h16::Scale* scale;
  uint16_t* t16;
  uint4* q16;
  int32_t* flags2;
  uint2* keys16;
  uint32_t* keys3;
  // 8-bit first tier (padded M = 4): aliases of the 16-bit buffers (never both in a call)
  uint8_t* t8;
  uint4* q8;
  uint32_t* keys8;
};

// Rows per scan window: the scan and the flag list index rows of a window in 32 bits;
// larger shards are scanned window by window (the table chunks are built once).
constexpr int64_t kScanWindow = (int64_t)1 << 30;
// The 8-bit tier keeps T keys per code (structure of arrays, T x 4 B per code of a window):
// smaller windows bound that buffer (2^28 codes: 8 GB at T = 8).
constexpr int64_t kScanWindow8 = (int64_t)1 << 28;

static AssignWS assign_ws_layout(void* base, int64_t n, int64_t k, int mp, int l) {
  AssignWS w{};
  uint32_t hs = 64;
  while (hs < 2 * (uint64_t)k) hs <<= 1;
  w.hash_size = hs;
  const int kc = kc_for(mp);
  const int64_t nchunks_max = (k + kc - 1) / kc;
  const int64_t nblk = (k + 1023) / 1024;
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align) {
    off = align_up(off, align);
    const size_t o = off;
    off += bytes;
    return o;
  };
  const size_t o_cnt = take(16 * sizeof(int32_t), 256);
  const size_t o_hash = take(hs * sizeof(int32_t), 256);
  const size_t o_rep = take(k * sizeof(int32_t), 256);
  const size_t o_blk = take(nblk * sizeof(int32_t), 256);
  const size_t o_p2i = take(k * sizeof(int32_t), 256);
  const size_t o_uc = take((size_t)k * mp, 256);
  const size_t o_q = take((size_t)nchunks_max * l * mp * kc * sizeof(float), 1024);
  const size_t o_fl = take((size_t)std::max<int64_t>(std::min(n, kScanWindow), 1) * sizeof(int32_t), 256);
  const int kc16 = h16::kcFor(mp);
  const bool h16_ok = mp <= 16;
  const size_t o_sc = take(sizeof(h16::Scale), 256);
  const size_t o_t16 = take(h16_ok ? (size_t)mp * l * l * sizeof(uint16_t) : 0, 256);
  const size_t o_q16 = take(h16_ok ? (size_t)((k + kc16 - 1) / kc16) * l * mp * kc16 * sizeof(uint16_t) : 0, 1024);
  const size_t o_fl2 =
      take(h16_ok ? (size_t)std::max<int64_t>(std::min(n, kScanWindow), 1) * sizeof(int32_t) : 0, 256);
  // (B, Sg) per code, plus the third key when one lane owns a code (KC = 8: MP 8 / 16)
  const size_t k16_bytes =
      h16_ok ? (size_t)std::max<int64_t>(std::min(n, kScanWindow), 1) * (sizeof(uint2) + (kc16 == 8 ? 4 : 0)) : 0;
  const size_t k8_bytes =
      mp == 4 ? (size_t)std::max<int64_t>(std::min(n, kScanWindow8), 1) * h8::kMaxT * sizeof(uint32_t) : 0;
  const size_t o_k16 = take(std::max(k16_bytes, k8_bytes), 256);
  w.total = align_up(off, 256);
  char* b = static_cast<char*>(base);
  if (b) {
    w.counters = reinterpret_cast<int32_t*>(b + o_cnt);
    w.hash = reinterpret_cast<int32_t*>(b + o_hash);
    w.rep = reinterpret_cast<int32_t*>(b + o_rep);
    w.blockcnt = reinterpret_cast<int32_t*>(b + o_blk);
    w.pos2idx = reinterpret_cast<int32_t*>(b + o_p2i);
    w.ucodes = reinterpret_cast<uint8_t*>(b + o_uc);
    w.q = reinterpret_cast<float*>(b + o_q);
    w.flags = reinterpret_cast<int32_t*>(b + o_fl);
    w.scale = reinterpret_cast<h16::Scale*>(b + o_sc);
    w.t16 = reinterpret_cast<uint16_t*>(b + o_t16);
    w.q16 = reinterpret_cast<uint4*>(b + o_q16);
    w.flags2 = reinterpret_cast<int32_t*>(b + o_fl2);
    w.keys16 = reinterpret_cast<uint2*>(b + o_k16);
    w.keys3 = reinterpret_cast<uint32_t*>(b + o_k16 + (size_t)std::max<int64_t>(std::min(n, kScanWindow), 1) * sizeof(uint2));
    // q16 region: ceil(k/16) x l x 4 x 16 x 2 B >= ceil(k/32) x l x 128 B; t16: 4 l^2 x 2 B >= 4 l^2
    w.t8 = reinterpret_cast<uint8_t*>(b + o_t16);
    w.q8 = reinterpret_cast<uint4*>(b + o_q16);
    w.keys8 = reinterpret_cast<uint32_t*>(b + o_k16);
  }
  return w;
}

template <int MP, int KC, int NW, int S, int C, int... Cs>
static int launch_scan_c(int c_need, const ScanParams& p, int grid, int l, cudaStream_t stream) {
  if constexpr (sizeof...(Cs) > 0) {
    if (c_need > C) return launch_scan_c<MP, KC, NW, S, Cs...>(c_need, p, grid, l, stream);
  }
  const bool prof = p.list == nullptr;  // bench events bracket the first-tier scan only
  const DevInfo& di = dev_info();
  const size_t smem = 128 + (size_t)S * l * MP * KC * 4;
  if ((int)smem > di.smem_optin) return fail(PQK_EUNSUPPORTED, "assignment chunk ring exceeds shared memory");
  auto kern = scan_kernel<MP, KC, C, NW, S>;
  if constexpr (sizeof...(Cs) == 0) {  // the largest variant also serves the list tier
    if (p.list) kern = scan_kernel<MP, KC, C, NW, S, true>;
  }
  PQK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfileEvents& pe = profile_events();
  if (prof && pe.before) PQK_CUDA_TRY(record_profile_event(pe.before, stream));
  kern<<<grid, (NW + 1) * 32, smem, stream>>>(p);
  PQK_LAUNCH_CHECK("scan_kernel");
  if (prof && pe.after) PQK_CUDA_TRY(record_profile_event(pe.after, stream));
  return PQK_OK;
}

// Balanced persistent schedule: every CTA runs the same number of equal passes and
// the kernel variant with the smallest register slot count C that holds a pass.
template <int MP, int KC, int NW, int S, int... Cs>
static int launch_scan(const ScanParams& base_params, int l, cudaStream_t stream) {
  constexpr int H = KC / 4;
  constexpr int OWN = NW * (32 / H);
  constexpr int CMAX = std::max({Cs...});
  constexpr int NB = OWN * CMAX;  // codes per pass (register capacity of a CTA)
  const DevInfo& di = dev_info();
  ScanParams p = base_params;
  const int64_t n = p.n;
  const int64_t G = di.sms;
  const int64_t per_cta = std::max<int64_t>(1, (n + G * NB - 1) / (G * NB));
  int64_t npasses = G * per_cta;
  int64_t pass_size = (n + npasses - 1) / npasses;
  // Small inputs: fewer CTAs rather than passes below ~1/4 of the register capacity.
  const int64_t min_pass = std::max<int64_t>(1, NB / 4);
  if (pass_size < min_pass) {
    pass_size = min_pass;
    npasses = (n + pass_size - 1) / pass_size;
  }
  p.pass_size = pass_size;
  p.npasses = npasses;
  const int grid = (int)std::min<int64_t>(G, npasses);
  if (grid <= 0) return PQK_OK;
  const int c_need = (int)((pass_size + OWN - 1) / OWN);
  return launch_scan_c<MP, KC, NW, S, Cs...>(c_need, p, grid, l, stream);
}

// Second tier: the fp32 scan over a device-side list (runs only when the list holds at
// least list_min codes; pass sizes derived on the device).  Largest register variant.
template <int MP, int KC, int NW, int S, int... Cs>
static int launch_scan_list(const ScanParams& p, int l, cudaStream_t stream) {
  constexpr int CMAX = std::max({Cs...});
  return launch_scan_c<MP, KC, NW, S, Cs...>(CMAX, p, dev_info().sms, l, stream);
}

// ---------------------------------------------------------------------------
// 16-bit first tier (pqk_hscan.cuh)
template <int MP, int KC, int NW, int S, int C, int... Cs>
static int launch_hscan_c(int c_need, const h16::HScanParams& p, uint2* keys, int grid, int l,
                          cudaStream_t stream) {
  if constexpr (sizeof...(Cs) > 0) {
    if (c_need > C) return launch_hscan_c<MP, KC, NW, S, Cs...>(c_need, p, keys, grid, l, stream);
  }
  const DevInfo& di = dev_info();
  const size_t smem = 128 + (size_t)S * 256 * MP * KC * 2;  // ring stride: 256 rows (immediate offsets)
  if ((int)smem > di.smem_optin) return fail(PQK_EUNSUPPORTED, "assignment chunk ring exceeds shared memory");
  auto kern = h16::hscan_kernel<MP, KC, C, NW, S>;
  PQK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfileEvents& pe = profile_events();
  if (pe.before) PQK_CUDA_TRY(record_profile_event(pe.before, stream));
  kern<<<grid, (NW + 1) * 32, smem, stream>>>(p, keys);
  PQK_LAUNCH_CHECK("hscan_kernel");
  if (pe.after) PQK_CUDA_TRY(record_profile_event(pe.after, stream));
  const int fgrid = (int)std::min<int64_t>((p.n + 255) / 256, (int64_t)di.sms * 64);
  h16::hfinal_kernel<MP, KC><<<std::max(fgrid, 1), 256, 0, stream>>>(p, keys);
  PQK_LAUNCH_CHECK("hfinal_kernel");
  return PQK_OK;
}

template <int MP, int KC, int NW, int S, int... Cs>
static int launch_hscan(const h16::HScanParams& base_params, uint2* keys, int l, cudaStream_t stream) {
  constexpr int H = KC / 8;
  constexpr int OWN = NW * (32 / H);
  constexpr int CMAX = std::max({Cs...});
  constexpr int NB = OWN * CMAX;
  const DevInfo& di = dev_info();
  h16::HScanParams p = base_params;
  const int64_t n = p.n;
  const int64_t G = di.sms;
  const int64_t per_cta = std::max<int64_t>(1, (n + G * NB - 1) / (G * NB));
  int64_t npasses = G * per_cta;
  int64_t pass_size = (n + npasses - 1) / npasses;
  const int64_t min_pass = std::max<int64_t>(1, NB / 4);
  if (pass_size < min_pass) {
    pass_size = min_pass;
    npasses = (n + pass_size - 1) / pass_size;
  }
  p.pass_size = pass_size;
  p.npasses = npasses;
  const int grid = (int)std::min<int64_t>(G, npasses);
  if (grid <= 0) return PQK_OK;
  const int c_need = (int)((pass_size + OWN - 1) / OWN);
  return launch_hscan_c<MP, KC, NW, S, Cs...>(c_need, p, keys, grid, l, stream);
}


// ---------------------------------------------------------------------------
// 8-bit first tier (pqk_hscan8.cuh, padded M = 4)
static int h8_top() {
  static int t = [] {
    const char* e = getenv("PQK_H8_T");  // diagnostic: keys kept per code (4 or 6)
    return (e && atoi(e) == 4) ? 4 : 6;
  }();
  return t;
}

template <int NW, int S, int T, int C, int... Cs>
static int launch_hscan8_c(int c_need, const h8::H8Params& p, uint32_t* keys, int64_t kstride, int grid, int l,
                           cudaStream_t stream) {
  if constexpr (sizeof...(Cs) > 0) {
    if (c_need > C) return launch_hscan8_c<NW, S, T, Cs...>(c_need, p, keys, kstride, grid, l, stream);
  }
  const DevInfo& di = dev_info();
  const size_t smem = 128 + 1024 + (size_t)S * 256 * h8::ROW;  // ring stride: 256 rows (immediate offsets); 1 KB alignment slack
  if ((int)smem > di.smem_optin) return fail(PQK_EUNSUPPORTED, "assignment chunk ring exceeds shared memory");
  auto kern = h8::hscan8_kernel<C, NW, S, T>;
  PQK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfileEvents& pe = profile_events();
  if (pe.before) PQK_CUDA_TRY(record_profile_event(pe.before, stream));
  kern<<<grid, (NW + 1) * 32, smem, stream>>>(p, keys, kstride);
  PQK_LAUNCH_CHECK("hscan8_kernel");
  if (pe.after) PQK_CUDA_TRY(record_profile_event(pe.after, stream));
  const int fgrid = (int)std::min<int64_t>((p.n + 255) / 256, (int64_t)di.sms * 64);
  h8::hfinal8_kernel<T><<<std::max(fgrid, 1), 256, 0, stream>>>(p, keys, kstride);
  PQK_LAUNCH_CHECK("hfinal8_kernel");
  return PQK_OK;
}

template <int NW, int S, int T, int... Cs>
static int launch_hscan8(const h8::H8Params& base_params, uint32_t* keys, int64_t kstride, int l,
                         cudaStream_t stream) {
  constexpr int OWN = NW * 32;
  constexpr int CMAX = std::max({Cs...});
  constexpr int NB = OWN * CMAX;
  const DevInfo& di = dev_info();
  h8::H8Params p = base_params;
  const int64_t n = p.n;
  const int64_t G = di.sms;
  // Every CTA runs per_cta equal passes of C register slots (OWN codes each); a pass costs
  // its C slot-streams of every chunk whatever the slots' fill, plus a ring restart.  Pick
  // (per_cta, C) minimising per_cta x (C + 0.3) for the codes of a CTA: config 2 (19.2
  // slot-passes per CTA) takes 4 x 5 instead of 3 x 7 (a third of the 7th slot idle).
  int64_t per_cta = std::max<int64_t>(1, (n + G * NB - 1) / (G * NB));
  {
    double best = 1e300;
    for (int64_t pc = per_cta; pc <= per_cta + 8; ++pc) {
      const int64_t c = (n + G * pc * OWN - 1) / (G * pc * OWN);
      if (c > CMAX) continue;
      const double cost = (double)pc * ((double)c + 0.3);
      if (cost < best) {
        best = cost;
        per_cta = pc;
      }
    }
  }
  int64_t npasses = G * per_cta;
  int64_t pass_size = (n + npasses - 1) / npasses;
  const int64_t min_pass = std::max<int64_t>(1, NB / 4);
  if (pass_size < min_pass) {
    pass_size = min_pass;
    npasses = (n + pass_size - 1) / pass_size;
  }
  p.pass_size = pass_size;
  p.npasses = npasses;
  const int grid = (int)std::min<int64_t>(G, npasses);
  if (grid <= 0) return PQK_OK;
  const int c_need = (int)((pass_size + OWN - 1) / OWN);
  return launch_hscan8_c<NW, S, T, Cs...>(c_need, p, keys, kstride, grid, l, stream);
}

// 0: fixed-point first tier where it pays off (default: 8-bit for padded M = 4, 16-bit for
// 8 and 16); 1: fp32 scan only; 2: fixed-point first tier whenever supported; 3: as 2, and
// the fp32 list tier for any list length (tests); 4, 5: as 2, 3 with the 16-bit tier at
// padded M = 4 too (no 8-bit tier)
static int g_scan_mode = 0;

}  // namespace pqk

using namespace pqk;

extern "C" int32_t pqk_padded_m(int32_t m) { return padded_m(m); }

extern "C" int pqk_set_scan_mode(int32_t mode) {
  if (mode < 0 || mode > 5) return fail(PQK_EINVAL, "pqk_set_scan_mode: mode must be in [0, 5]");
  g_scan_mode = mode;
  return PQK_OK;
}

extern "C" int32_t pqk_get_scan_mode(void) { return g_scan_mode; }

extern "C" int pqk_tables_to_f32(const double* d_t64, int32_t m, int32_t l, int32_t exp2, float* d_t32,
                                 void* stream) {
  if (!d_t64 || !d_t32 || m < 1 || l < 1 || l > kMaxL) return fail(PQK_EINVAL, "pqk_tables_to_f32: bad arguments");
  const int mp = padded_m(m);
  const size_t total = (size_t)mp * l * l;
  const int grid = (int)std::min<size_t>((total + 255) / 256, 4096);
  tables_to_f32_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_t64, m, l, mp, exp2, d_t32);
  PQK_LAUNCH_CHECK("tables_to_f32_kernel");
  return PQK_OK;
}

extern "C" int pqk_pad_codes_device(const uint8_t* d_raw, int64_t n, int32_t m, uint8_t* d_padded, void* stream) {
  if (n < 0 || m < 1 || (n > 0 && (!d_raw || !d_padded))) return fail(PQK_EINVAL, "pqk_pad_codes_device: bad arguments");
  if (n == 0) return PQK_OK;
  const int mp = padded_m(m);
  const int64_t total = n * mp;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 8192);
  pad_codes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_raw, n, m, mp, d_padded);
  PQK_LAUNCH_CHECK("pad_codes_kernel");
  return PQK_OK;
}

// Side stream + fork/join events per (device, caller stream): the 16-bit tier's scale
// preparation (table maximum, sampled exact scan over the raw centers) runs beside the
// center dedup and joins before the table quantisation.  Event fork/join also captures
// into a CUDA graph as two parallel branches.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static int side_stream_for(int dev, cudaStream_t main, SideStream** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SideStream> table;
  std::lock_guard<std::mutex> lock(mu);
  SideStream& ss = table[{dev, main}];
  if (!ss.s) {
    PQK_CUDA_TRY(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    PQK_CUDA_TRY(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    PQK_CUDA_TRY(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  *out = &ss;
  return PQK_OK;
}

extern "C" size_t pqk_assign_workspace_bytes(int64_t n, int64_t k, int32_t m, int32_t l) {
  const int mp = padded_m(m);
  if (mp == 0 || k < 1 || n < 0 || l < 1) return 0;
  return assign_ws_layout(nullptr, n, k, mp, l).total;
}

extern "C" int pqk_assign_device(const uint8_t* d_codes, int64_t n, int32_t m, int32_t l, const uint8_t* d_centers,
                                 int64_t k, const double* d_t64, const float* d_t32, int32_t fp64_only, void* d_ws,
                                 size_t ws_bytes, uint32_t* d_labels, double* d_sd_sq, int64_t* d_stats,
                                 void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int mp = padded_m(m);
  if (mp == 0 || l < 2 || l > kMaxL) return fail(PQK_EINVAL, "pqk_assign_device: M must be >= 1 and L in [2, 256]");
  if (k < 1) return fail(PQK_EINVAL, "centers must be non-empty");
  if (n < 0 || k >= (int64_t)1 << 30) return fail(PQK_EUNSUPPORTED, "pqk_assign_device: k must be < 2^30");
  if (n == 0) return PQK_OK;
  if (!d_codes || !d_centers || !d_t64 || !d_labels || !d_sd_sq || !d_ws)
    return fail(PQK_EINVAL, "pqk_assign_device: null pointer");
  const bool fast = !fp64_only && mp <= 32 && d_t32 != nullptr;
  const int kc16 = h16::kcFor(mp);
  // the 16-bit tier pays off above ~2^31 lookups (its per-call table preparation and
  // finalisation cost tens of microseconds); smaller problems run the fp32 scan
  const bool tier_on = fast && g_scan_mode != 1 &&
                       (g_scan_mode >= 2 || (double)n * (double)k * (double)m >= 2147483648.0);
  const bool use8 = tier_on && mp == 4 && g_scan_mode < 4 && (k + h8::KC - 1) / h8::KC < (1 << 24) - 1;
  const bool use16 = tier_on && !use8 && mp <= 16 && (k + kc16 - 1) / kc16 <= 65535;
  const bool use_tier = use8 || use16;
  AssignWS w = assign_ws_layout(d_ws, n, k, mp, l);
  if (ws_bytes < w.total) return fail(PQK_EINVAL, "pqk_assign_device: workspace too small");

  const DevInfo& di0 = dev_info();
  SideStream* side = nullptr;
  if (use_tier) {
    // 0. scale preparation on the side branch (w.scale is free: the fork follows every
    //    earlier reader on the caller's stream)
    int dev = 0;
    PQK_CUDA_TRY(cudaGetDevice(&dev));
    { const int rc = side_stream_for(dev, stream, &side); if (rc != PQK_OK) return rc; }
    static bool attr16[64] = {};
    if (!attr16[dev & 63]) {
      PQK_CUDA_TRY(cudaFuncSetAttribute(h16::scale_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        96 * 1024));
      attr16[dev & 63] = true;
    }
    PQK_CUDA_TRY(cudaEventRecord(side->fork, stream));
    PQK_CUDA_TRY(cudaStreamWaitEvent(side->s, side->fork, 0));
    PQK_CUDA_TRY(cudaMemsetAsync(w.scale, 0, sizeof(h16::Scale), side->s));
    const int64_t cnt = (int64_t)m * l * l;
    h16::table_max_kernel<<<(int)std::min<int64_t>((cnt + 255) / 256, (int64_t)di0.sms * 4), 256, 0, side->s>>>(
        d_t64, cnt, w.scale);
    PQK_LAUNCH_CHECK("table_max_kernel");
    h16::scale_sample_kernel<<<h16::kScaleSample, 256, (size_t)m * l * sizeof(double), side->s>>>(
        d_codes, n, mp, m, l, d_centers, nullptr, d_t64, w.scale, (int)k);
    PQK_LAUNCH_CHECK("scale_sample_kernel");
    PQK_CUDA_TRY(cudaEventRecord(side->join, side->s));
  }
  // 1. dedup
  PQK_CUDA_TRY(cudaMemsetAsync(w.counters, 0, 16 * sizeof(int32_t), stream));
  PQK_CUDA_TRY(cudaMemsetAsync(w.hash, 0xff, w.hash_size * sizeof(int32_t), stream));
  const int kb = (int)((k + 1023) / 1024);
  dedup_insert_kernel<<<(int)((k + 255) / 256), 256, 0, stream>>>(d_centers, (int)k, mp, w.hash, w.hash_size - 1);
  PQK_LAUNCH_CHECK("dedup_insert_kernel");
  dedup_mark_kernel<<<kb, 1024, 0, stream>>>(d_centers, (int)k, mp, w.hash, w.hash_size - 1, w.rep, w.blockcnt);
  PQK_LAUNCH_CHECK("dedup_mark_kernel");
  dedup_compact_kernel<<<kb, 1024, 0, stream>>>(d_centers, (int)k, mp, kc_for(mp), w.rep, w.blockcnt, w.pos2idx,
                                                w.ucodes, w.counters);
  PQK_LAUNCH_CHECK("dedup_compact_kernel");

  const DevInfo& di = dev_info();
  // 2. fp32 restricted-table chunks (16-bit path: built inside the window loop, only
  //    when the first tier leaves a list long enough for the fp32 list tier)
  auto qbuild32 = [&](const int32_t* gate, int32_t gate_min) -> int {
    const int kc = kc_for(mp);
    const int64_t units = ((k + kc - 1) / kc) * l * mp * (kc / 4);
    const int qgrid = (int)std::min<int64_t>((units + 255) / 256, (int64_t)di.sms * 16);
    float4* q4 = (float4*)w.q;
    switch (mp) {
      case 4: qbuild_kernel<4, 8><<<qgrid, 256, 0, stream>>>(d_t32, l, w.ucodes, w.counters, q4, gate, gate_min); break;
      case 8: qbuild_kernel<8, 4><<<qgrid, 256, 0, stream>>>(d_t32, l, w.ucodes, w.counters, q4, gate, gate_min); break;
      case 16: qbuild_kernel<16, 4><<<qgrid, 256, 0, stream>>>(d_t32, l, w.ucodes, w.counters, q4, gate, gate_min); break;
      case 32: qbuild_kernel<32, 4><<<qgrid, 256, 0, stream>>>(d_t32, l, w.ucodes, w.counters, q4, gate, gate_min); break;
    }
    PQK_LAUNCH_CHECK("qbuild_kernel");
    return PQK_OK;
  };
  if (fast && !use_tier) {  // the fixed-point tiers build it only for a long uncertified list
    const int rc = qbuild32(nullptr, 0);
    if (rc != PQK_OK) return rc;
  }
  if (use8) {
    // 8-bit fixed-point tables and their 32-centre chunks
    const int qmax = h8::qmax_for(m);
    PQK_CUDA_TRY(cudaStreamWaitEvent(stream, side->join, 0));  // scale ready (side branch)
    const int64_t cnt4 = (int64_t)4 * l * l;
    h8::table_quantize8_kernel<<<(int)std::min<int64_t>((cnt4 + 255) / 256, (int64_t)di.sms * 8), 256, 0,
                                 stream>>>(d_t64, m, l, qmax, w.scale, w.t8);
    PQK_LAUNCH_CHECK("table_quantize8_kernel");
    const int rgrid = (int)std::min<int64_t>((k + h8::KC - 1) / h8::KC, (int64_t)di.sms * 8);
    const size_t rsm = (size_t)4 * h8::KC * (l + 4);
    h8::qbuild8_rows_kernel<<<rgrid, 256, rsm, stream>>>(w.t8, l, m, qmax, w.ucodes, w.counters, w.q8);
    PQK_LAUNCH_CHECK("qbuild8_rows_kernel");
  }
  if (use16) {
    // 16-bit fixed-point tables (scale from the table maximum) and their chunks
    const int qmax = h16::qmax_for(m);
    PQK_CUDA_TRY(cudaStreamWaitEvent(stream, side->join, 0));  // scale ready (side branch)
    const int64_t cntp = (int64_t)mp * l * l;
    h16::table_quantize_kernel<<<(int)std::min<int64_t>((cntp + 255) / 256, (int64_t)di.sms * 8), 256, 0,
                                 stream>>>(d_t64, m, l, mp, qmax, w.scale, w.t16);
    PQK_LAUNCH_CHECK("table_quantize_kernel");
    const int64_t units = ((k + kc16 - 1) / kc16) * l * mp * (kc16 / 8);
    const int qgrid = (int)std::min<int64_t>((units + 255) / 256, (int64_t)di.sms * 16);
    if (l % 8 == 0) {  // row-staged build
      const int rgrid = (int)std::min<int64_t>((k + kc16 - 1) / kc16, (int64_t)di.sms * 8);
      const size_t rsm = (size_t)mp * kc16 * (l + 2) * sizeof(uint16_t);
      static bool attr_q[64] = {};
      int dev = 0;
      cudaGetDevice(&dev);
      if (!attr_q[dev & 63]) {
        PQK_CUDA_TRY(cudaFuncSetAttribute(h16::qbuild16_rows_kernel<16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(16 * 8 * (kMaxL + 2) * sizeof(uint16_t))));
        attr_q[dev & 63] = true;
      }
      switch (mp) {
        case 4: h16::qbuild16_rows_kernel<4, 16><<<rgrid, 256, rsm, stream>>>(w.t16, l, m, qmax, w.ucodes, w.counters, w.q16); break;
        case 8: h16::qbuild16_rows_kernel<8, 8><<<rgrid, 256, rsm, stream>>>(w.t16, l, m, qmax, w.ucodes, w.counters, w.q16); break;
        case 16: h16::qbuild16_rows_kernel<16, 8><<<rgrid, 256, rsm, stream>>>(w.t16, l, m, qmax, w.ucodes, w.counters, w.q16); break;
      }
      PQK_LAUNCH_CHECK("qbuild16_rows_kernel");
    } else {
      switch (mp) {
        case 4: h16::qbuild16_kernel<4, 16><<<qgrid, 256, 0, stream>>>(w.t16, l, m, qmax, w.ucodes, w.counters, w.q16); break;
        case 8: h16::qbuild16_kernel<8, 8><<<qgrid, 256, 0, stream>>>(w.t16, l, m, qmax, w.ucodes, w.counters, w.q16); break;
        case 16: h16::qbuild16_kernel<16, 8><<<qgrid, 256, 0, stream>>>(w.t16, l, m, qmax, w.ucodes, w.counters, w.q16); break;
      }
      PQK_LAUNCH_CHECK("qbuild16_kernel");
    }
  }
  // list tier threshold: below it the exact rescan is cheaper than streaming every chunk
  // (fp32 list scan: every CTA streams all chunks, a fixed cost, so it only beats the
  // exact rescan, whose cost is per code, for lists of ~250 codes per SM and more)
  const int32_t list_min = (g_scan_mode == 3 || g_scan_mode == 5) ? 0 : di.sms * 256;
  const size_t rows_bytes = (size_t)m * l * sizeof(double);
  const bool cta_rescan = rows_bytes <= 96 * 1024;
  if (cta_rescan) {
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
      PQK_CUDA_TRY(cudaFuncSetAttribute(rescan_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
      attr_set[dev & 63] = true;
    }
  }
  const int64_t window = use8 ? kScanWindow8 : kScanWindow;
  for (int64_t w0 = 0; w0 < n; w0 += window) {
    const int64_t wn = std::min(window, n - w0);
    const uint8_t* codes = d_codes + w0 * mp;
    uint32_t* labels = d_labels + w0;
    double* sd_sq = d_sd_sq + w0;
    if (w0 > 0) PQK_CUDA_TRY(cudaMemsetAsync(w.counters + 1, 0, sizeof(int32_t), stream));
    if (w0 > 0) PQK_CUDA_TRY(cudaMemsetAsync(w.counters + 3, 0, sizeof(int32_t), stream));
    if (use8) {
      // 3a. 8-bit first tier over every code
      h8::H8Params hp{};
      hp.codes = codes;
      hp.n = wn;
      hp.q = w.q8;
      hp.l = l;
      hp.m = m;
      hp.counters = w.counters;
      hp.pos2idx = w.pos2idx;
      hp.ucodes = w.ucodes;
      hp.t64 = d_t64;
      hp.sc = w.scale;
      hp.labels = labels;
      hp.sd_sq = sd_sq;
      hp.flags = w.flags;
      hp.flag_count = w.counters + 1;
      const int rc = h8_top() == 4 ? launch_hscan8<11, 4, 4, 1, 2, 3, 4, 5, 6, 7, 8>(hp, w.keys8, wn, l, stream)
                                   : launch_hscan8<11, 4, 6, 1, 2, 3, 4, 5, 6, 7, 8>(hp, w.keys8, wn, l, stream);
      if (rc != PQK_OK) return rc;
    }
    if (use16) {
      // 3a. 16-bit first tier over every code
      h16::HScanParams hp{};
      hp.codes = codes;
      hp.n = wn;
      hp.q = w.q16;
      hp.l = l;
      hp.m = m;
      hp.counters = w.counters;
      hp.pos2idx = w.pos2idx;
      hp.ucodes = w.ucodes;
      hp.t64 = d_t64;
      hp.sc = w.scale;
      hp.labels = labels;
      hp.sd_sq = sd_sq;
      hp.flags = w.flags;
      hp.flag_count = w.counters + 1;
      hp.keys3 = w.keys3;
      int rc = PQK_OK;
      switch (mp) {
        case 4: rc = launch_hscan<4, 16, 11, 4, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>(hp, w.keys16, l, stream); break;
        case 8: rc = launch_hscan<8, 8, 11, 4, 1, 2, 3, 4, 5, 6, 7, 8>(hp, w.keys16, l, stream); break;
        case 16: rc = launch_hscan<16, 8, 11, 3, 1, 2, 3, 4>(hp, w.keys16, l, stream); break;
      }
      if (rc != PQK_OK) return rc;
    }
    if (use_tier) {
      // 3b. fp32 tier over the uncertified list when it is long
      int rc = qbuild32(w.counters + 1, list_min);
      if (rc != PQK_OK) return rc;
      ScanParams sp{};
      sp.codes = codes;
      sp.n = 0;
      sp.q = w.q;
      sp.l = l;
      sp.m = m;
      sp.counters = w.counters;
      sp.pos2idx = w.pos2idx;
      sp.ucodes = w.ucodes;
      sp.t64 = d_t64;
      sp.cert_factor = 1.0 + 4.0 * (2.0 * m) * ldexp(1.0, -24);
      sp.labels = labels;
      sp.sd_sq = sd_sq;
      sp.flags = w.flags2;
      sp.flag_count = w.counters + 3;
      sp.list = w.flags;
      sp.list_count = w.counters + 1;
      sp.list_min = list_min;
      switch (mp) {
        case 4: rc = launch_scan_list<4, 8, 11, 4, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14>(sp, l, stream); break;
        case 8: rc = launch_scan_list<8, 4, 11, 4, 1, 2, 3, 4, 5, 6, 7, 8>(sp, l, stream); break;
        case 16: rc = launch_scan_list<16, 4, 11, 3, 1, 2, 3, 4>(sp, l, stream); break;
      }
      if (rc != PQK_OK) return rc;
      // 4. exact rescans: the short first-tier list, then what the fp32 tier left
      rescan_cta_kernel<<<di.sms * 8, 256, rows_bytes, stream>>>(codes, wn, mp, m, l, w.ucodes, w.counters, w.flags,
                                                                w.counters + 1, w.pos2idx, d_t64, labels, sd_sq, 0,
                                                                list_min);
      PQK_LAUNCH_CHECK("rescan_cta_kernel");
      rescan_cta_kernel<<<di.sms * 2, 256, rows_bytes, stream>>>(codes, wn, mp, m, l, w.ucodes, w.counters,
                                                                w.flags2, w.counters + 3, w.pos2idx, d_t64, labels,
                                                                sd_sq, 0, 0x7fffffff);
      PQK_LAUNCH_CHECK("rescan_cta_kernel");
      if (d_stats) {
        assign_stats_kernel<<<1, 1, 0, stream>>>(w.counters, d_stats, w0 == 0, use8 ? h8::KC : kc16,
                                                 use8 ? 1 : 2, list_min);
        PQK_LAUNCH_CHECK("assign_stats_kernel");
      }
      continue;
    }
    if (fast) {
      // 3. scan
      ScanParams sp{};
      sp.codes = codes;
      sp.n = wn;
      sp.q = w.q;
      sp.l = l;
      sp.m = m;
      sp.counters = w.counters;
      sp.pos2idx = w.pos2idx;
      sp.ucodes = w.ucodes;
      sp.t64 = d_t64;
      sp.cert_factor = 1.0 + 4.0 * (2.0 * m) * ldexp(1.0, -24);
      sp.labels = labels;
      sp.sd_sq = sd_sq;
      sp.flags = w.flags;
      sp.flag_count = w.counters + 1;
      int rc = PQK_OK;
      switch (mp) {
        case 4: rc = launch_scan<4, 8, 11, 4, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14>(sp, l, stream); break;
        case 8: rc = launch_scan<8, 4, 11, 4, 1, 2, 3, 4, 5, 6, 7, 8>(sp, l, stream); break;
        case 16: rc = launch_scan<16, 4, 11, 3, 1, 2, 3, 4>(sp, l, stream); break;
        case 32: rc = launch_scan<32, 4, 11, 1, 1, 2>(sp, l, stream); break;
      }
      if (rc != PQK_OK) return rc;
    }
    // 4. exact rescan of uncertified codes (or every code in fp64-only mode)
    if (cta_rescan) {
      const int grid = (int)std::min<int64_t>(fast ? (int64_t)di.sms * 2 : wn, (int64_t)di.sms * 8);
      rescan_cta_kernel<<<std::max(grid, 1), 256, rows_bytes, stream>>>(
          codes, wn, mp, m, l, w.ucodes, w.counters, w.flags, w.counters + 1, w.pos2idx, d_t64, labels, sd_sq,
          fast ? 0 : 1, 0x7fffffff);
      PQK_LAUNCH_CHECK("rescan_cta_kernel");
    } else {
      const int64_t warps = fast ? (int64_t)di.sms * 32 : std::min<int64_t>(wn, (int64_t)di.sms * 64);
      const int grid = (int)std::max<int64_t>(1, (warps * 32 + 255) / 256);
      rescan_kernel<<<grid, 256, 0, stream>>>(codes, wn, mp, m, l, w.ucodes, w.counters, w.flags, w.counters + 1,
                                              w.pos2idx, d_t64, labels, sd_sq, fast ? 0 : 1, 0x7fffffff);
      PQK_LAUNCH_CHECK("rescan_kernel");
    }
    if (d_stats) {
      assign_stats_kernel<<<1, 1, 0, stream>>>(w.counters, d_stats, w0 == 0, 0, 4, 0);
      PQK_LAUNCH_CHECK("assign_stats_kernel");
    }
  }
  return PQK_OK;
}

extern "C" int pqk_paired_distance_device(const uint8_t* d_a, const uint8_t* d_b, const uint32_t* d_idx, int64_t n,
                                          int32_t m, int32_t l, const double* d_t64, double* d_out, void* stream) {
  const int mp = padded_m(m);
  if (mp == 0 || l < 1 || l > kMaxL || n < 0) return fail(PQK_EINVAL, "pqk_paired_distance_device: bad arguments");
  if (n == 0) return PQK_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 8192);
  paired_distance_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_a, d_b, d_idx, n, mp, m, l, d_t64, d_out);
  PQK_LAUNCH_CHECK("paired_distance_kernel");
  return PQK_OK;
}
