// pqk_hscan.cuh — 16-bit fixed-point assignment scan (first filter tier of the
// nearest-center assignment, clustering.py:167-197).  Included by pqk_assign.cu.
//
// Why 16 bits.  The scan is bound by shared-memory lookups (one lane read per
// (code, center, subspace)).  Storing the restricted tables as uint16 halves the
// bytes of every lookup, and integer sums of uint16 pairs packed in one 32-bit
// register are exact (IADD3 adds two centers at once: every sum of M entries is kept
// <= 65535, so no carry crosses the halves).  The only error is the quantisation of
// each table entry, q = min(QMAX, rint(t * s)) with QMAX = floor(65535 / M):
// q <= s t + 1/2 + O(2^-40) (saturation only lowers q), so a code-center sum obeys
//     s * D(u) >= Q(u) - M/2 - 0.01      (D = exact float64 reference sum).
// The scale s = QMAX / t_hi resolves the distances that decide assignments:
// t_hi = min(max(T), 2 x the largest per-subspace term of the nearest centre over a
// sample of 128 codes).  Entries above t_hi saturate; the bound above still holds, and
// a code whose decision involves saturated terms simply fails its certificate.
//
// Keys.  Each lane holds 8 centers of a KC-center chunk as 4 packed registers.  Per
// chunk it takes their minimum (VIMNMX3.U16x2, then the two halves) and forms one 32-bit
// key (value << 16 | chunk); it tracks the smallest key B and the second-smallest S
// over chunks — no per-centre index bookkeeping in the loop.
//
// Finalisation (per code, hfinal_kernel).  c* = chunk of the smallest key.  The chunk is re-read from
// the global table copy, its centres with Q(u) <= Q_min + M + 1 are re-evaluated
// exactly in float64 (ascending m, __dadd_rn) and the smallest, lowest index on ties,
// is the candidate winner w* with distance d*.  Every other centre of chunk c* has
// Q(u) >= Qn (the smallest non-candidate sum), every centre of another chunk has
// Q(u) >= Sg, the minimum over the code's lanes of (chunk(B) == c* ? S : B); the code is
// certified when min(Sg, Qn) - M/2 - 0.01 > s d* (1 + 2^-40): then w* is the float64 argmin with
// the reference's lowest-index tie rule, and d* its paired_distance_sq.  Uncertified
// codes (near ties within the quantisation error, ~0.1-2% of codes) go to the next
// tier: the fp32 scan over the list (large lists) or the exact fp64 rescan (small).
#pragma once

namespace pqk {
namespace h16 {

// packed unsigned 16-bit minimum (VIMNMX.U16x2 / VIMNMX3.U16x2 on sm_100a)
__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

constexpr int kcFor(int mp) { return mp == 4 ? 16 : 8; }
inline int qmax_for(int m) { return 65535 / m; }

// scratch block of the 16-bit path (in the assignment workspace)
struct Scale {
  unsigned long long maxbits;  // max table entry (float64 bits; entries are >= 0)
  double s;                    // quantisation scale
  int bad;                     // a negative / non-finite entry: every code goes to the next tier
  int pad;
  unsigned long long termbits;  // largest nearest-centre term over the code sample (float64 bits)
};

constexpr int kScaleSample = 128;

// Scale heuristic (never affects correctness): for kScaleSample evenly spaced codes,
// the nearest distinct centre (float64 sums over the staged table rows, first minimum)
// and the largest of its M terms; their maximum goes to sc->termbits.
__global__ void __launch_bounds__(256) scale_sample_kernel(const uint8_t* __restrict__ codes, int64_t n, int mp,
                                                           int m, int l, const uint8_t* __restrict__ ucodes,
                                                           const int32_t* __restrict__ counters,
                                                           const double* __restrict__ t64, Scale* sc, int u_fixed) {
  extern __shared__ double s_rows[];  // m * l
  __shared__ double s_best[8];
  __shared__ int s_bu[8];
  const int64_t idx = (int64_t)blockIdx.x * n / gridDim.x;
  const uint8_t* xc = codes + idx * mp;
  const int U = u_fixed >= 0 ? u_fixed : counters[0];  // u_fixed: raw centers (duplicates kept)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < m * l; e += blockDim.x) {
    const int mm = e / l, s = e - mm * l;
    s_rows[e] = t64[((size_t)mm * l + xc[mm]) * l + s];
  }
  __syncthreads();
  double best = __longlong_as_double(0x7ff0000000000000LL);
  int bu = 0x7fffffff;
  const int bd = (int)blockDim.x;
  for (int u0 = tid; u0 < U; u0 += 4 * bd) {  // 4 independent centres per step
    double d[4] = {0.0, 0.0, 0.0, 0.0};
    for (int w = 0; 4 * w < m; ++w) {
      uint32_t cw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * bd;
        cw[q] = u < U ? __ldg(reinterpret_cast<const uint32_t*>(ucodes + (size_t)u * mp) + w) : 0u;
      }
#pragma unroll
      for (int bb = 0; bb < 4; ++bb)
        if (4 * w + bb < m) {
#pragma unroll
          for (int q = 0; q < 4; ++q) d[q] += s_rows[(4 * w + bb) * l + ((cw[q] >> (8 * bb)) & 0xffu)];
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (u0 + q * bd < U && d[q] < best) {
        best = d[q];
        bu = u0 + q * bd;
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
    if (bu != 0x7fffffff) {
      double tm = 0.0;
      for (int mm = 0; mm < m; ++mm) tm = fmax(tm, s_rows[mm * l + ucodes[(size_t)bu * mp + mm]]);
      if (tm >= 0.0 && tm < __longlong_as_double(0x7ff0000000000000LL))
        atomicMax(&sc->termbits, (unsigned long long)__double_as_longlong(tm));
    }
  }
}

__global__ void table_max_kernel(const double* __restrict__ t64, int64_t count, Scale* sc) {
  unsigned long long mx = 0ull;
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = t64[i];
    if (!(v >= 0.0) || v == __longlong_as_double(0x7ff0000000000000LL)) bad = 1;
    else mx = max(mx, (unsigned long long)__double_as_longlong(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&sc->maxbits, mx);
    if (bad) atomicOr(&sc->bad, 1);
  }
}

// T16[mm][a][b] = min(QMAX, rint(T[mm][a][b] * s)) for mm < m, 0 for the padding subspaces
__global__ void table_quantize_kernel(const double* __restrict__ t64, int m, int l, int mp, int qmax, Scale* sc,
                                      uint16_t* __restrict__ t16) {
  const double tmax = __longlong_as_double((long long)sc->maxbits);
  const double tsam = 2.0 * __longlong_as_double((long long)sc->termbits);
  const double thi = (tsam > 0.0 && tsam < tmax) ? tsam : tmax;
  const double s = thi > 0.0 ? (double)qmax / thi : 1.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->s = s;
  const size_t ll = (size_t)l * l;
  const size_t total = (size_t)mp * ll;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t mm = i / ll;
    uint16_t q = 0;
    if (mm < (size_t)m) {
      const double v = rint(__dmul_rn(t64[i], s));
      q = (uint16_t)(v >= (double)qmax ? qmax : (v > 0.0 ? (int)v : 0));  // saturate (q <= s t + 1/2)
    }
    t16[i] = q;
  }
}

// Q16[t][s][mm][j] = T16[mm][s][c_{t KC + j}^mm]; padding centres (u >= U) get QMAX on the
// real subspaces (sum M QMAX <= 65535: never below a real centre) and 0 on padding ones.
template <int MP, int KC>
__global__ void qbuild16_kernel(const uint16_t* __restrict__ t16, int l, int m, int qmax,
                                const uint8_t* __restrict__ ucodes, const int32_t* __restrict__ counters,
                                uint4* __restrict__ q) {
  const int U = counters[0];
  const int nchunks = (U + KC - 1) / KC;
  constexpr int Q8 = KC / 8;  // uint4 (8 values) per (t, s, mm)
  const int64_t units = (int64_t)nchunks * l * MP * Q8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < units; i += (int64_t)gridDim.x * blockDim.x) {
    const int q8 = (int)(i % Q8);
    int64_t r = i / Q8;
    const int mm = (int)(r % MP);
    r /= MP;
    const int s = (int)(r % l);
    const int t = (int)(r / l);
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t v2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int u = t * KC + q8 * 8 + 2 * j + e;
        v2[e] = (u < U) ? (uint32_t)t16[((size_t)mm * l + ucodes[(size_t)u * MP + mm]) * l + s]
                        : (mm < m ? (uint32_t)qmax : 0u);
      }
      w[j] = v2[0] | (v2[1] << 16);
    }
    q[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Same table as qbuild16_kernel, one CTA per chunk t (grid-stride): the chunk's KC center
// rows T16[mm][c_u][*] (contiguous 2L-byte rows) are copied into shared memory with 16-byte
// loads, then written out in Q16 order with 16-byte stores.  qbuild16_kernel gathered
// every value with a 2-byte load from a random row (10M gathers, 16.5 us at config 2).
template <int MP, int KC>
__global__ void __launch_bounds__(256) qbuild16_rows_kernel(const uint16_t* __restrict__ t16, int l, int m, int qmax,
                                                            const uint8_t* __restrict__ ucodes,
                                                            const int32_t* __restrict__ counters,
                                                            uint4* __restrict__ q) {
  extern __shared__ uint16_t sq[];  // [MP * KC][l + 2] (padded rows)
  const int U = counters[0];
  const int nchunks = (U + KC - 1) / KC;
  constexpr int Q8 = KC / 8;
  const int ls = l + 2;
  const int l8 = l / 8;  // l is a multiple of 8 (checked by the caller)
  for (int t = blockIdx.x; t < nchunks; t += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < MP * KC * l8; i += blockDim.x) {
      const int c8 = i % l8, row = i / l8;
      const int mm = row / KC, j = row - mm * KC;
      const int u = t * KC + j;
      uint4 v;
      if (u < U && mm < m) {
        const int c = ucodes[(size_t)u * MP + mm];
        v = __ldg(reinterpret_cast<const uint4*>(t16 + ((size_t)mm * l + c) * l) + c8);
      } else {
        const uint32_t f = (mm < m) ? ((uint32_t)qmax | ((uint32_t)qmax << 16)) : 0u;
        v = make_uint4(f, f, f, f);
      }
      uint32_t* d = reinterpret_cast<uint32_t*>(sq + row * ls + 8 * c8);  // 4-byte aligned (ls even)
      d[0] = v.x;
      d[1] = v.y;
      d[2] = v.z;
      d[3] = v.w;
    }
    __syncthreads();
    uint4* qt = q + (size_t)t * l * MP * Q8;
    for (int i = threadIdx.x; i < l * MP * Q8; i += blockDim.x) {
      const int q8 = i % Q8;
      const int r = i / Q8;
      const int mm = r % MP, sidx = r / MP;
      const uint16_t* col = sq + (mm * KC + q8 * 8) * ls + sidx;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) w[e] = (uint32_t)col[(2 * e) * ls] | ((uint32_t)col[(2 * e + 1) * ls] << 16);
      qt[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

struct HScanParams {
  const uint8_t* codes;
  int64_t n;
  const uint4* q;
  int l;
  int m;
  const int32_t* counters;  // [0] U
  const int32_t* pos2idx;
  const uint8_t* ucodes;
  const double* t64;
  const Scale* sc;
  uint32_t* labels;
  double* sd_sq;
  int32_t* flags;
  int32_t* flag_count;
  int64_t pass_size;
  int64_t npasses;
  uint32_t* keys3;  // one lane per code (KC = 8): the third-smallest chunk key per code
};

template <int W>
__device__ __forceinline__ void load_code_rot(const uint8_t* __restrict__ codes, int idx, bool valid, int c,
                                              uint32_t (&out)[W]) {
  uint32_t w[W];
#pragma unroll
  for (int k = 0; k < W; ++k) w[k] = 0u;
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
  }
  // rotate left by c bytes (c < 8): out byte i = code byte (c + i) mod MP
  const int qw = (W == 1) ? 0 : (c >> 2);
  const int rb = c & 3;
  uint32_t u[W];
#pragma unroll
  for (int k = 0; k < W; ++k) u[k] = qw ? w[(k + 1) % W] : w[k];
#pragma unroll
  for (int k = 0; k < W; ++k) out[k] = __funnelshift_r(u[k], u[(k + 1) % W], 8 * rb);
}

// Exact pass over one chunk of a code (finalisation): the KC fixed-point sums (as in the
// scan), centres with Q <= lim re-evaluated in float64 (ascending m, __dadd_rn) into
// (best, bu) with the lowest index on ties (chunks may be visited out of index order),
// the smallest sum above lim into qn.
template <int MP, int KC>
__device__ __forceinline__ void hfinal_chunk(const HScanParams& p, const uint32_t (&xb)[MP / 4], uint32_t chunk,
                                             uint32_t lim, int U, int m, double& best, int& bu, uint32_t& qn) {
  constexpr int G8 = KC / 8;  // uint4 groups of 8 centres per (chunk, row, subspace)
  uint32_t r[G8][4];
#pragma unroll
  for (int g = 0; g < G8; ++g) r[g][0] = r[g][1] = r[g][2] = r[g][3] = 0u;
#pragma unroll
  for (int mm = 0; mm < MP; ++mm) {
    if (mm < m) {
      const uint32_t x = (xb[mm >> 2] >> (8 * (mm & 3))) & 0xffu;
#pragma unroll
      for (int g = 0; g < G8; ++g) {
        const uint4 w = __ldg(p.q + (((size_t)chunk * p.l + x) * MP + mm) * G8 + g);
        r[g][0] += w.x;
        r[g][1] += w.y;
        r[g][2] += w.z;
        r[g][3] += w.w;
      }
    }
  }
  const int u0 = (int)chunk * KC;
  const int nreal = min(KC, U - u0);  // real centres of the chunk (the last chunk is partial)
  uint32_t cand = 0u;
#pragma unroll
  for (int e = 0; e < KC; ++e) {
    const uint32_t w = r[e >> 3][(e & 7) >> 1];
    const uint32_t qv = (e < nreal) ? ((e & 1) ? (w >> 16) : (w & 0xffffu)) : 0xffffffffu;
    const bool c = qv <= lim;
    cand |= (c ? 1u : 0u) << e;
    if (!c) qn = min(qn, qv);  // padding (~0) never lowers qn
  }
  while (cand) {  // ascending centre index within the chunk
    const int e = __ffs(cand) - 1;
    cand &= cand - 1u;
    const int u = u0 + e;
    uint32_t cb[MP / 4];
#pragma unroll
    for (int w = 0; w < MP / 4; ++w) cb[w] = __ldg(reinterpret_cast<const uint32_t*>(p.ucodes + (size_t)u * MP) + w);
    double d = 0.0;
#pragma unroll
    for (int mm = 0; mm < MP; ++mm) {
      if (mm < m) {
        const uint32_t x = (xb[mm >> 2] >> (8 * (mm & 3))) & 0xffu;
        const uint32_t c = (cb[mm >> 2] >> (8 * (mm & 3))) & 0xffu;
        d = dadd(d, __ldg(&p.t64[((size_t)mm * p.l + x) * p.l + c]));
      }
    }
    if (d < best || (d == best && u < bu)) {
      best = d;
      bu = u;
    }
  }
}

// Finalisation, one thread per code (a separate, fully parallel kernel: its dependent
// global loads would otherwise stall every warp of the scan at the end of each pass).
// keys[i] = (B, Sg): B = (Q << 16 | chunk) of the smallest chunk minimum, Sg the lower
// bound of every centre outside chunk(B) (~0: none).  With one lane per code (KC = 8)
// Sg is the second-smallest chunk key and keys3[i] the third: when Sg's chunk holds
// candidates (value <= lim) it is evaluated too and the third key bounds the rest (a
// code-level top-2 of chunks left 0.5% of config 5's codes uncertified, top-3 none of
// 3,000 sampled).
template <int MP, int KC>
__global__ void __launch_bounds__(256, MP >= 16 ? 2 : 4) hfinal_kernel(const HScanParams p, const uint2* __restrict__ keys) {
  constexpr bool T3 = (KC == 8);
  const int U = p.counters[0];
  const int m = p.m;
  const double s_q = p.sc->s;
  const bool bad = p.sc->bad != 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 kv = keys[i];
    const uint32_t cstar = kv.x & 0xffffu, sg = kv.y;
    const uint8_t* xc = p.codes + (size_t)i * MP;
    uint32_t xb[MP / 4];
#pragma unroll
    for (int w = 0; w < MP / 4; ++w) xb[w] = __ldg(reinterpret_cast<const uint32_t*>(xc) + w);
    // candidates: within M + 1 units of the smallest chunk minimum; the rest bound from below
    const uint32_t lim = (kv.x >> 16) + (uint32_t)m + 1u;
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bu = 0x7fffffff;
    uint32_t qn = 0xffffffffu;  // smallest non-candidate sum of the evaluated chunks (none: ~0)
    hfinal_chunk<MP, KC>(p, xb, cstar, lim, U, m, best, bu, qn);
    // lower bound of every centre not evaluated: other chunks and the non-candidates
    uint32_t qlow;
    if (T3 && sg != 0xffffffffu && (sg >> 16) <= lim) {
      hfinal_chunk<MP, KC>(p, xb, sg & 0xffffu, lim, U, m, best, bu, qn);
      const uint32_t k3 = __ldg(p.keys3 + i);
      qlow = min(k3 == 0xffffffffu ? 0xffffffffu : (k3 >> 16), qn);
    } else {
      qlow = min(sg == 0xffffffffu ? 0xffffffffu : (sg >> 16), qn);
    }
    bool cert = !bad && bu != 0x7fffffff;
    if (cert && qlow != 0xffffffffu) {
      const double lo = (double)qlow - 0.5 * (double)m - 0.01;
      cert = lo > best * s_q * (1.0 + 0x1p-40);
    }
    if (cert) {
      p.labels[i] = (uint32_t)__ldg(&p.pos2idx[bu]);
      p.sd_sq[i] = best;
    } else {
      const int f = atomicAdd(p.flag_count, 1);
      p.flags[f] = (int32_t)i;
    }
  }
}

// Shared-memory layout: chunk row s holds, for every subspace mm, the KC uint16 values
// T16[mm][s][c_j^mm] (a 2 KC-byte m-slab); a lane reads 16 bytes (8 centres) of one slab
// per LDS.128, H = KC / 8 lanes per code.  The 8 lanes of a quarter-warp phase serve
// P = 8 / H codes; code slot c reads slab (c + i) mod MP at step i, so the slabs of a
// phase are P consecutive ones: disjoint banks whatever the code bytes (4 wavefronts per
// LDS.128, as in the fp32 scan).
template <int MP, int KC, int C, int NW, int S>
__global__ void __launch_bounds__((NW + 1) * 32, 1) hscan_kernel(const HScanParams p, uint2* __restrict__ keys) {
  constexpr int H = KC / 8;
  constexpr int OWN_W = 32 / H;
  constexpr int OWN = NW * OWN_W;
  constexpr int ROW = MP * KC * 2;
  constexpr int P = 8 / H;
  constexpr int W = MP / 4;
  static_assert(MP % P == 0, "MP must be a multiple of the phase width");

  constexpr uint32_t STAGE = 256u * ROW;  // ring stride (a chunk holds l <= 256 rows)

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  uint8_t* stages = smem + 128;
  const uint32_t chunk_bytes = (uint32_t)p.l * ROW;
  const int U = p.counters[0];
  const int nchunks = (U + KC - 1) / KC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  const int64_t my_passes = (p.npasses > blockIdx.x) ? (p.npasses - blockIdx.x + G - 1) / G : 0;

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
    if (lane == 0) {
      // every pass restarts the ring at stage 0 (chunk t -> stage t % S, so that the
      // consumers address stages with immediates); bit st of `bits` = parity of stage st
      const char* src = reinterpret_cast<const char*>(p.q);
      uint32_t bits = 0;
      for (int64_t pi = 0; pi < my_passes; ++pi) {
        for (int t = 0; t < nchunks; ++t) {
          const int st = t % S;
          mbar_wait(&empty[st], ((bits >> st) & 1u) ^ 1u);
          bits ^= 1u << st;
          mbar_arrive_expect_tx(&full[st], chunk_bytes);
          bulk_g2s(stages + (size_t)st * STAGE, src + (size_t)t * chunk_bytes, chunk_bytes, &full[st]);
        }
      }
    }
    return;
  }

  const int o = lane / H;
  const int c = o % P;
  const int h = lane % H;
  uint32_t lc[MP];
#pragma unroll
  for (int i = 0; i < MP; ++i) lc[i] = (uint32_t)(((c + i) % MP) * (KC * 2) + h * 16);
  const uint32_t stage0 = smem_u32(stages);
  const int n = (int)p.n;
  const int pass_size = (int)p.pass_size;

  uint32_t bits = 0;
  for (int pi = 0; pi < (int)my_passes; ++pi) {
    const int base = ((int)blockIdx.x + pi * (int)G) * pass_size;
    const int end = min(n, base + pass_size);
    const int my0 = base + warp * OWN_W + o;

    // per (slot, subspace step) the shared-memory address of the code's row in stage 0
    uint32_t off[C][MP];
    uint32_t bk[C], sk[C], rk[C];  // rk: third-smallest key (one lane per code only)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int idx = my0 + j * OWN;
      uint32_t cw[W];
      load_code_rot<W>(p.codes, idx, idx < end, c, cw);
#pragma unroll
      for (int i = 0; i < MP; ++i)
        off[j][i] = __byte_perm(cw[i >> 2], 0u, 0x4440u | (uint32_t)(i & 3)) * ROW + lc[i] + stage0;
      bk[j] = sk[j] = rk[j] = 0xffffffffu;
    }

    for (int t0 = 0; t0 < nchunks; t0 += S) {
#pragma unroll
    for (int st = 0; st < S; ++st) {
      const int t = t0 + st;
      if (t >= nchunks) break;
      mbar_wait(&full[st], (bits >> st) & 1u);
      bits ^= 1u << st;
      uint4 buf[2][MP];
#pragma unroll
      for (int i = 0; i < MP; ++i) buf[0][i] = lds128u(off[0][i] + st * STAGE);
#pragma unroll
      for (int j = 0; j < C; ++j) {
        if (j + 1 < C) {
#pragma unroll
          for (int i = 0; i < MP; ++i) buf[(j + 1) & 1][i] = lds128u(off[j + 1][i] + st * STAGE);
        }
        uint4* v = buf[j & 1];
        // exact packed sums (no carry across halves: every sum <= 65535)
        uint32_t r0 = v[0].x, r1 = v[0].y, r2 = v[0].z, r3 = v[0].w;
#pragma unroll
        for (int i = 1; i < MP; ++i) {
          r0 += v[i].x;
          r1 += v[i].y;
          r2 += v[i].z;
          r3 += v[i].w;
        }
        const uint32_t cm = vmin2(vmin2(r0, r1), vmin2(r2, r3));
        const uint32_t c2 = vmin2(cm, __byte_perm(cm, 0u, 0x1032));  // both halves: min of the 8
        const uint32_t kk = __byte_perm((uint32_t)t, c2, 0x5410);      // (min << 16) | chunk
        if constexpr (H == 1) rk[j] = max(sk[j], min(rk[j], kk));     // third smallest
        sk[j] = max(bk[j], min(sk[j], kk));                            // second smallest (bk <= sk)
        bk[j] = min(bk[j], kk);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    }

    // ---------------- end of pass: merge the code's lanes, store (B, Sg) ----------------
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const uint32_t k0 = bk[j], s0 = sk[j];
      uint32_t k1 = 0xffffffffu, s1 = 0xffffffffu;
      if constexpr (H == 2) {
        k1 = __shfl_xor_sync(0xffffffffu, k0, 1);
        s1 = __shfl_xor_sync(0xffffffffu, s0, 1);
      }
      const uint32_t kb = min(k0, k1);
      const uint32_t cstar = kb & 0xffffu;
      const uint32_t sg = min(((k0 & 0xffffu) == cstar) ? s0 : k0, ((k1 & 0xffffu) == cstar) ? s1 : k1);
      const int idx = my0 + j * OWN;
      if (h == 0 && idx < end) {
        keys[idx] = make_uint2(kb, sg);
        if constexpr (H == 1) p.keys3[idx] = rk[j];
      }
    }
  }
}

}  // namespace h16
}  // namespace pqk
