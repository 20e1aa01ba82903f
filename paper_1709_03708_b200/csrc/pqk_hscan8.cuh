// pqk_hscan8.cuh — 8-bit fixed-point first tier of the nearest-center assignment
// (clustering.py:167-197) for codes of at most 4 subspaces (padded M = 4: configs 1, 2
// and 4, the north-star shard).  Included by pqk_assign.cu after pqk_hscan.cuh.
//
// Why 8 bits.  The scan is bound by shared-memory lookup bandwidth (one lane read per
// (code, center, subspace)).  With one-byte table entries a 16-byte LDS.128 serves 16
// centres, twice the 16-bit tier: the same 128 B/clk/SM carry twice the lookups.  Entries
// are quantised as q = min(QMAX, rint(s t)) with QMAX = floor(255 / M) (63 at M = 4), so a
// code-centre sum of M entries fits one byte and four centres add exactly in one 32-bit
// IADD3 (no carry crosses a byte).  The bound of the 16-bit tier holds unchanged:
//     s * D(u) >= Q(u) - M/2 - 0.01       (D = the exact float64 reference sum),
// because q <= s t + 1/2 (saturation only lowers q).
//
// Why top-T.  At 8 bits the quantisation step is coarse (t_hi / 63), so the best centre
// and its near rivals often sit in different chunks.  Every lane owns one code and keeps
// the T smallest chunk-minimum keys (value << 24 | chunk), sorted, in registers: a sorted
// insert is 2T - 1 min/max.  Every chunk outside the T stored ones has a minimum >= the
// T-th key, so the finalisation evaluates only the stored chunks' candidates.  Measured
// on config-4 data (tools/diag_scan8.py): T = 4 leaves 1.1% of the codes uncertified,
// T = 6 0.07% (a code-level top-2, as in the 16-bit tier, would leave 24%).
//
// Finalisation (hfinal8_kernel, thread per code).  qmin = value of the smallest key,
// lim = qmin + M + 1.  For every stored chunk with value <= lim the code's 32 sums are
// recomputed from the chunk table, centres with Q <= lim are re-evaluated exactly in
// float64 (ascending m, __dadd_rn) and the smallest (lowest position on ties: positions
// ascend with the original index) is the winner w* with distance d*.  Every centre not
// evaluated has Q >= min(lim + 1, V_T): lim + 1 bounds the non-candidates of evaluated
// chunks and every stored chunk above lim, V_T the T-th key's value the chunks not stored
// (none when the code saw fewer than T chunks).  Certified when that bound - M/2 - 0.01 > s d* (1 + 2^-40):
// every other centre's float64 sum then exceeds d*, so w* is the reference's argmin and d*
// its paired_distance_sq.  Uncertified codes go to the next tier (fp32 list scan, exact
// fp64 rescan) exactly as after the 16-bit tier.
#pragma once

namespace pqk {
namespace h8 {

constexpr int KC = 32;         // centres per chunk
constexpr int ROW = 4 * KC;    // bytes per chunk row: 4 subspace slabs of 32 one-byte entries
constexpr int kMaxT = 8;
inline int qmax_for(int m) { return 255 / m; }

// T8[mm][a][b] = min(QMAX, rint(T[mm][a][b] * s)), s = QMAX / t_hi (t_hi as in the 16-bit
// tier: min(max T, 2 x the largest nearest-centre term of the sampled codes)); padding
// subspaces (mm >= m) are 0.  Writes s to sc->s for the finalisation.
__global__ void table_quantize8_kernel(const double* __restrict__ t64, int m, int l, int qmax, h16::Scale* sc,
                                       uint8_t* __restrict__ t8) {
  const double tmax = __longlong_as_double((long long)sc->maxbits);
  const double tsam = 2.0 * __longlong_as_double((long long)sc->termbits);
  const double thi = (tsam > 0.0 && tsam < tmax) ? tsam : tmax;
  const double s = thi > 0.0 ? (double)qmax / thi : 1.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->s = s;
  const size_t ll = (size_t)l * l;
  const size_t total = 4 * ll;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t mm = i / ll;
    uint8_t q = 0;
    if (mm < (size_t)m) {
      const double v = rint(__dmul_rn(t64[i], s));
      q = (uint8_t)(v >= (double)qmax ? qmax : (v > 0.0 ? (int)v : 0));  // saturate (q <= s t + 1/2)
    }
    t8[i] = q;
  }
}

// Q8[t][s][mm][j] = T8[mm][s][c_{32 t + j}^mm] (chunk t, row s: 4 slabs of 32 bytes).
// One CTA per chunk (grid-stride): the chunk's 4 x 32 centre rows T8[mm][c][*] are staged
// in shared memory, then written out row by row with 16-byte stores.  Padding centres
// (u >= U) get QMAX on the real subspaces (their sum M QMAX <= 255 is never below a real
// centre's... and never a candidate: the finalisation skips u >= U) and 0 elsewhere.
__global__ void __launch_bounds__(256) qbuild8_rows_kernel(const uint8_t* __restrict__ t8, int l, int m, int qmax,
                                                           const uint8_t* __restrict__ ucodes,
                                                           const int32_t* __restrict__ counters,
                                                           uint4* __restrict__ q) {
  extern __shared__ uint8_t s8[];  // [4 * KC][ls] centre rows
  const int U = counters[0];
  const int nchunks = (U + KC - 1) / KC;
  const int ls = l + 4;
  const bool vec = (l % 16) == 0;
  for (int t = blockIdx.x; t < nchunks; t += gridDim.x) {
    __syncthreads();
    if (vec) {
      const int l16 = l / 16;
      for (int i = threadIdx.x; i < 4 * KC * l16; i += blockDim.x) {
        const int c16 = i % l16, row = i / l16;
        const int mm = row / KC, j = row - mm * KC;
        const int u = t * KC + j;
        uint4 v;
        if (u < U && mm < m) {
          const int c = ucodes[(size_t)u * 4 + mm];
          v = __ldg(reinterpret_cast<const uint4*>(t8 + ((size_t)mm * l + c) * l) + c16);
        } else {
          const uint32_t f = (mm < m) ? (uint32_t)qmax * 0x01010101u : 0u;
          v = make_uint4(f, f, f, f);
        }
        uint32_t* d = reinterpret_cast<uint32_t*>(s8 + row * ls + 16 * c16);  // 4-byte aligned (ls % 4 == 0)
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
      }
    } else {
      for (int i = threadIdx.x; i < 4 * KC * l; i += blockDim.x) {
        const int sidx = i % l, row = i / l;
        const int mm = row / KC, j = row - mm * KC;
        const int u = t * KC + j;
        uint8_t v;
        if (u < U && mm < m) v = t8[((size_t)mm * l + ucodes[(size_t)u * 4 + mm]) * l + sidx];
        else v = (mm < m) ? (uint8_t)qmax : (uint8_t)0;
        s8[row * ls + sidx] = v;
      }
    }
    __syncthreads();
    uint4* qt = q + (size_t)t * l * 8;
    for (int i = threadIdx.x; i < l * 8; i += blockDim.x) {
      const int g = i & 7;  // 16-byte group of row s: slab mm = g / 2, half g % 2
      const int sidx = i >> 3;
      const uint8_t* col = s8 + ((g >> 1) * KC + (g & 1) * 16) * ls + sidx;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = (uint32_t)col[(4 * e) * ls] | ((uint32_t)col[(4 * e + 1) * ls] << 8) |
               ((uint32_t)col[(4 * e + 2) * ls] << 16) | ((uint32_t)col[(4 * e + 3) * ls] << 24);
      qt[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

struct H8Params {
  const uint8_t* codes;  // (n, 4) uint8, this window
  int64_t n;
  const uint4* q;        // Q8 chunks
  int l;
  int m;
  const int32_t* counters;  // [0] U
  const int32_t* pos2idx;
  const uint8_t* ucodes;
  const double* t64;
  const h16::Scale* sc;
  uint32_t* labels;
  double* sd_sq;
  int32_t* flags;
  int32_t* flag_count;
  int64_t pass_size;
  int64_t npasses;
};

__device__ __forceinline__ uint32_t vmin3(uint32_t a, uint32_t b, uint32_t c) {
  return h16::vmin2(h16::vmin2(a, b), c);  // VIMNMX3.U16x2
}

// Shared-memory layout: chunk row s = 4 slabs (one per subspace) of 32 one-byte entries.
// One lane per code; a lane reads a 16-byte half-slab (16 centres) per LDS.128.  Lane c of
// a quarter-warp phase (c = lane % 8) reads, at subspace step i, slab (c + i) mod 4 of its
// code's row x_{(c+i) mod 4}, half (c / 4) xor k for k = 0, 1: the 8 lanes of a phase cover
// the 8 distinct 16-byte granules of a 128-byte row, conflict-free whatever the code
// bytes (4 wavefronts per LDS.128).
template <int C, int NW, int S, int T>
__global__ void __launch_bounds__((NW + 1) * 32, 1) hscan8_kernel(const H8Params p, uint32_t* __restrict__ keys,
                                                                  int64_t kstride) {
  constexpr int OWN = NW * 32;
  constexpr uint32_t STAGE = 256u * ROW;  // ring stride (a chunk holds l <= 256 rows)

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  // the ring starts 1024-aligned in the shared window (measured: 1.381 -> 1.367 s at config 4
  // against the 128-byte alignment)
  uint8_t* stages = smem + 128 + ((1024u - ((smem_u32(smem) + 128u) & 1023u)) & 1023u);
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

  const int c = lane & 7;
  const int rot = c & 3;
  const uint32_t hsel = (uint32_t)(c >> 2) * 16u;
  uint32_t lc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) lc[i] = (uint32_t)(((rot + i) & 3) * KC);
  const uint32_t stage0 = smem_u32(stages);
  const int n = (int)p.n;
  const int pass_size = (int)p.pass_size;

  uint32_t bits = 0;
  for (int pi = 0; pi < (int)my_passes; ++pi) {
    const int base = ((int)blockIdx.x + pi * (int)G) * pass_size;
    const int end = min(n, base + pass_size);
    const int my0 = base + warp * 32 + lane;

    uint32_t off[C][2][4];
    uint32_t key[C][T];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int idx = my0 + j * OWN;
      const uint32_t w = idx < end ? __ldg(reinterpret_cast<const uint32_t*>(p.codes) + idx) : 0u;
      const uint32_t cw = __funnelshift_r(w, w, 8 * rot);  // byte i = code byte (rot + i) mod 4
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t a = __byte_perm(cw, 0u, 0x4440u | (uint32_t)i) * ROW + lc[i] + stage0;
        off[j][0][i] = a + hsel;
        off[j][1][i] = a + (hsel ^ 16u);
      }
#pragma unroll
      for (int e = 0; e < T; ++e) key[j][e] = 0xffffffffu;
    }

    for (int t0 = 0; t0 < nchunks; t0 += S) {
#pragma unroll
      for (int st = 0; st < S; ++st) {
        const int t = t0 + st;
        if (t >= nchunks) break;
        mbar_wait(&full[st], (bits >> st) & 1u);
        bits ^= 1u << st;
        uint4 buf[2][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) buf[0][i] = h16::lds128u(off[0][0][i] + st * STAGE);
        uint32_t part = 0u;
#pragma unroll
        for (int hs = 0; hs < 2 * C; ++hs) {
          const int j = hs >> 1, k = hs & 1;
          if (hs + 1 < 2 * C) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              buf[(hs + 1) & 1][i] = h16::lds128u(off[(hs + 1) >> 1][(hs + 1) & 1][i] + st * STAGE);
          }
          const uint4* v = buf[hs & 1];
          // exact byte-packed sums of 16 centres (every sum <= 255: no carry between bytes)
          const uint32_t r0 = v[0].x + v[1].x + v[2].x + v[3].x;
          const uint32_t r1 = v[0].y + v[1].y + v[2].y + v[3].y;
          const uint32_t r2 = v[0].z + v[1].z + v[2].z + v[3].z;
          const uint32_t r3 = v[0].w + v[1].w + v[2].w + v[3].w;
          // u16x2 minima: the high byte of each half of r holds the odd bytes, of r << 8 the
          // even ones; a u16 minimum carries the minimum of the high bytes
          const uint32_t a = vmin3(r0, r1, r2);
          const uint32_t b = vmin3(r0 << 8, r1 << 8, r2 << 8);
          if (k == 0) {
            part = h16::vmin2(vmin3(a, b, r3), r3 << 8);
          } else {
            const uint32_t mm = vmin3(vmin3(a, b, r3), r3 << 8, part);
            const uint32_t f = h16::vmin2(mm, mm >> 16);            // byte 1 = min of the chunk's 32
            const uint32_t kk = __byte_perm((uint32_t)t, f, 0x5210);  // (min << 24) | chunk
#pragma unroll
            for (int e = T - 1; e > 0; --e) key[j][e] = min(key[j][e], max(key[j][e - 1], kk));
            key[j][0] = min(key[j][0], kk);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    }

    // end of pass: the code's T keys, structure-of-arrays (coalesced stores)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int idx = my0 + j * OWN;
      if (idx < end) {
#pragma unroll
        for (int e = 0; e < T; ++e) __stcs(keys + (int64_t)e * kstride + idx, key[j][e]);  // evict-first: Q8 stays in L2
      }
    }
  }
}

// L2 policy for the chunk-table re-reads of the finalisation: keep Q8 (100 MB at config
// 4) resident while the keys, codes, labels and distances stream through with evict-first
// loads/stores.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ldg4_keep(const uint4* ptr, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}

// Finalisation, one thread per code (see the header comment).
template <int T>
__global__ void __launch_bounds__(256, 4) hfinal8_kernel(const H8Params p, const uint32_t* __restrict__ keys,
                                                         int64_t kstride) {
  const int U = p.counters[0];
  const int m = p.m;
  const double s_q = p.sc->s;
  const bool bad = p.sc->bad != 0;
  const uint64_t pol = l2_evict_last_policy();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k[T];
#pragma unroll
    for (int e = 0; e < T; ++e) k[e] = __ldcs(keys + (int64_t)e * kstride + i);
    const uint32_t xw = __ldcs(reinterpret_cast<const uint32_t*>(p.codes) + i);
    const uint32_t lim = (k[0] >> 24) + (uint32_t)m + 1u;
    // every chunk not stored has a minimum >= the T-th key (none: fewer than T chunks)
    uint32_t qlow = (k[T - 1] == 0xffffffffu) ? 0xffffffffu : (k[T - 1] >> 24);
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bu = 0x7fffffff;
    bool more = true;
#pragma unroll
    for (int e = 0; e < T; ++e) {
      const uint32_t ke = k[e];
      if (ke == 0xffffffffu) more = false;  // sorted: no more chunks
      if (!more) continue;
      const uint32_t v = ke >> 24;
      if (v > lim) {  // sorted: this and every later stored chunk are bounds
        qlow = min(qlow, v);
        more = false;
        continue;
      }
      const uint32_t t = ke & 0xffffffu;
      // the 32 sums of chunk t (as in the scan: rows x^mm, slab mm)
      uint32_t r[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) r[w] = 0u;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        const uint32_t x = (xw >> (8 * mm)) & 0xffu;
        const uint4* src = p.q + (((size_t)t * p.l + x) * 4 + mm) * 2;
        const uint4 a0 = ldg4_keep(src, pol), a1 = ldg4_keep(src + 1, pol);
        r[0] += a0.x;
        r[1] += a0.y;
        r[2] += a0.z;
        r[3] += a0.w;
        r[4] += a1.x;
        r[5] += a1.y;
        r[6] += a1.z;
        r[7] += a1.w;
      }
      const int u0 = (int)t * KC;
      const int nreal = min(KC, U - u0);
      // candidates (Q <= lim) word by word; every real non-candidate has Q >= lim + 1, which
      // is the bound used for them (exact minima give the same certificate rate on config-4
      // data, and cost a byte extraction per centre)
      const uint32_t lim4 = min(lim, 255u) * 0x01010101u;
      qlow = min(qlow, lim + 1u);
      uint32_t cand = 0u;  // bit j: centre j is a candidate
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int nb = min(4, max(0, nreal - 4 * w));
        const uint32_t realm = nb >= 4 ? 0xffffffffu : ((1u << (8 * nb)) - 1u);
        const uint32_t hb = __vcmpleu4(r[w], lim4) & realm & 0x80808080u;
        cand |= ((hb * 0x00204081u) >> 28) << (4 * w);  // byte flags 7/15/23/31 -> bits 28..31
      }
      while (cand) {  // ascending position within the chunk
        const int j = __ffs(cand) - 1;
        cand &= cand - 1u;
        const int u = u0 + j;
        const uint32_t cb = __ldg(reinterpret_cast<const uint32_t*>(p.ucodes) + u);
        double d = 0.0;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
          if (mm < m) {
            const uint32_t x = (xw >> (8 * mm)) & 0xffu;
            const uint32_t cc = (cb >> (8 * mm)) & 0xffu;
            d = dadd(d, __ldg(&p.t64[((size_t)mm * p.l + x) * p.l + cc]));
          }
        }
        if (d < best || (d == best && u < bu)) {  // chunks are visited out of order
          best = d;
          bu = u;
        }
      }
    }
    bool cert = !bad && bu != 0x7fffffff;
    if (cert && qlow != 0xffffffffu) {
      const double lo = (double)qlow - 0.5 * (double)m - 0.01;
      cert = lo > best * s_q * (1.0 + 0x1p-40);
    }
    if (cert) {
      __stcs(p.labels + i, (uint32_t)__ldg(&p.pos2idx[bu]));
      __stcs(p.sd_sq + i, best);
    } else {
      const int f = atomicAdd(p.flag_count, 1);
      p.flags[f] = (int32_t)i;
    }
  }
}

}  // namespace h8
}  // namespace pqk
