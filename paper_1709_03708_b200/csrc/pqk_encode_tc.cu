// pqk_encode_tc.cu — tcgen05 (5th-gen tensor core) building blocks of the PQ encoder.
//
// pqk_tc_selftest: one 128 x 256 x K fp16 tile through the full tcgen05 path
// (canonical no-swizzle K-major smem operands, UMMA descriptors, TMEM accumulator,
// tcgen05.commit -> mbarrier, tcgen05.ld epilogue).  It is the device diagnostic the
// encoder's tests run first: a wrong descriptor shows up here as a wrong product.
#include "pqk_common.cuh"
#include "pqk_tc.cuh"

namespace pqk {

__global__ void __launch_bounds__(128) tc_selftest_kernel(const __half* __restrict__ A, const __half* __restrict__ B,
                                                          float* __restrict__ C, int K) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sa = smem;
  uint8_t* sb = smem + 128 * K * 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = 0; k < K; ++k) {
    *reinterpret_cast<__half*>(sa + tc::kmajor_off(tid, k, K)) = A[tid * K + k];
    *reinterpret_cast<__half*>(sb + tc::kmajor_off(tid, k, K)) = B[tid * K + k];
    *reinterpret_cast<__half*>(sb + tc::kmajor_off(tid + 128, k, K)) = B[(tid + 128) * K + k];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t taddr = tbase;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const uint32_t sbo = (uint32_t)(K / 8) * 128;
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t da = tc::smem_desc(a0 + s * 256, 128, sbo);
      const uint64_t db = tc::smem_desc(b0 + s * 256, 128, sbo);
      tc::mma_f16(taddr, da, db, tc::idesc_f16_f32(128, 256), s > 0 ? 1u : 0u);
    }
    tc::commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c0 = 0; c0 < 256; c0 += 16) {
    uint32_t r[16];
    tc::tmem_ld16(taddr + ((uint32_t)(32 * warp) << 16) + c0, r);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) C[(size_t)(32 * warp + lane) * 256 + c0 + j] = __uint_as_float(r[j]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(taddr, 256);
}

}  // namespace pqk

using namespace pqk;

extern "C" int pqk_tc_selftest(const void* d_a, const void* d_b, float* d_c, int32_t k, void* stream) {
  if (!d_a || !d_b || !d_c || k < 16 || k % 16 != 0 || k > 256) return fail(PQK_EINVAL, "pqk_tc_selftest: bad arguments");
  const size_t smem = (size_t)(128 + 256) * k * 2;
  PQK_CUDA_TRY(cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tc_selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>((const __half*)d_a, (const __half*)d_b, d_c, k);
  PQK_LAUNCH_CHECK("tc_selftest_kernel");
  return PQK_OK;
}

// ===========================================================================
// Tensor-core PQ encoder (pq.py:205-231 on tcgen05).
//
// For subspace m and a tile of 128 vectors: S = X_m C_m^T (128 x 256) on the tensor
// cores, g_l = ||c_l||^2 - 2 x.c_l, code = argmin_l g_l (= argmin ||x - c_l||^2).
// Exactness: x and c are scaled by powers of two into fp16 range and split as
// v = hi + lo (fp16 each, ~22 significant bits); S = hi.hi + hi.lo + lo.hi in fp32
// (the lo.hi pass is skipped for tiles whose x are exactly fp16, e.g. integer SIFT
// data).  The epilogue keeps best and runner-up per row and certifies the winner
// when their gap exceeds a rigorous bound on the split/accumulation error; other
// (vector, subspace) pairs are re-decided by the exact float64 sequential sum
// (scipy cdist order) in encode_exact_kernel.
//
// Warp roles (persistent, one CTA per SM, 576 threads):
//   warp 0  TMA producer: 2-D tensor-map loads of X[128 rows x KP] per (tile, m)
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer (2 accumulators of
//           128 x 256 fp32 = all 512 TMEM columns, double-buffered)
//   warps 2-17 transform (fp32 -> fp16 hi/lo in the UMMA K-major layout) and
//           epilogue (tcgen05.ld, argmin, certificate, code store); warp w reads
//           TMEM lanes 32*(w%4).. and columns [64*h, 64*h+64), h = (w-2)/4.
// ===========================================================================
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace pqk {
namespace enc {

constexpr int kRows = 128;
constexpr int kN = 256;
constexpr int kXStages = 3;
constexpr int kWorkWarps = 16;  // transform + epilogue warps (4 per SM sub-partition)
constexpr int kThreads = (2 + kWorkWarps) * 32;

struct EncParams {
  const float* x;
  const float* cw;
  const uint8_t* bprep;  // [M][2][256 x KP] fp16, UMMA K-major
  const float* cnc;      // [M][256]  s_c * ||c||^2 (+inf for padding rows)
  const float* cstat;    // [M][4]    C2, C1, CN (scaled), s_c
  int64_t n;
  int d, m, l, ks;
  uint8_t* codes;
  int stride;
  uint32_t* flags;
  unsigned int* counters;  // [0] flagged, [1] overflow
  uint32_t flag_cap;
  int ntiles;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int KP>
__host__ __device__ constexpr size_t smem_bytes(int m) {
  return (size_t)m * 2 * kN * KP * 2          // B hi/lo
         + (size_t)kXStages * kRows * KP * 4  // X stages
         + (size_t)2 * 2 * kRows * KP * 2     // A hi/lo, double-buffered
         + (size_t)m * kN * 4 + (size_t)m * 16  // cnc, cstat
         + (size_t)4 * kRows * 16              // row stats, 4 buffers
         + (size_t)3 * kRows * 16              // column-quarter merge
         + 2 * kWorkWarps * 4 + 16 * 8 + 16;   // lo flags, barriers, tmem base
}

template <int KP>
__global__ void __launch_bounds__(kThreads, 1) encode_tc_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                const EncParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int A_PART = kRows * KP * 2;
  constexpr int B_PART = kN * KP * 2;
  constexpr int X_STAGE = kRows * KP * 4;
  const int M = p.m;
  const uint32_t bytesB = (uint32_t)M * 2 * B_PART;
  uint8_t* sB = smem;
  uint8_t* sX = smem + bytesB;
  uint8_t* sA = sX + kXStages * X_STAGE;
  float* s_cnc = reinterpret_cast<float*>(sA + 2 * 2 * A_PART);
  float* s_cstat = s_cnc + M * kN;
  float4* s_stats = reinterpret_cast<float4*>(s_cstat + M * 4);
  float4* s_merge = s_stats + 4 * kRows;                     // [3][128]
  int* s_lo = reinterpret_cast<int*>(s_merge + 3 * kRows);    // [2][kWorkWarps]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_lo + 2 * kWorkWarps);
  uint64_t* xfull = bars;
  uint64_t* xempty = bars + 3;
  uint64_t* afull = bars + 6;
  uint64_t* aempty = bars + 8;
  uint64_t* tfull = bars + 10;
  uint64_t* tempty = bars + 12;
  uint64_t* bload = bars + 14;
  uint32_t* s_tbase = reinterpret_cast<uint32_t*>(bars + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int my_tiles = (p.ntiles > (int)blockIdx.x) ? (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int items = my_tiles * M;

  if (tid == 0) {
    for (int i = 0; i < kXStages; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], kWorkWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], kWorkWarps);
      mbar_init(&aempty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kWorkWarps);
    }
    mbar_init(bload, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(s_tbase, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *s_tbase;

  // codebook operands and statistics, once per CTA
  if (tid == 0) {
    const uint32_t cbytes = (uint32_t)M * kN * 4, sbytes = (uint32_t)M * 16;
    mbar_arrive_expect_tx(bload, bytesB + cbytes + sbytes);
    for (uint32_t off = 0; off < bytesB; off += 32768)
      bulk_g2s(sB + off, p.bprep + off, min(32768u, bytesB - off), bload);
    bulk_g2s(s_cnc, p.cnc, cbytes, bload);
    bulk_g2s(s_cstat, p.cstat, sbytes, bload);
  }
  mbar_wait(bload, 0);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int w = 0; w < items; ++w) {
        const int t = (int)blockIdx.x + (w / M) * (int)gridDim.x, m = w % M;
        const int xs = w % kXStages;
        const uint32_t ph = (uint32_t)((w / kXStages) & 1);
        mbar_wait(&xempty[xs], ph ^ 1u);
        mbar_arrive_expect_tx(&xfull[xs], X_STAGE);
        tma_load_2d(sX + xs * X_STAGE, &tmap, m * KP, t * kRows, &xfull[xs]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_f16_f32(kRows, kN);
      const uint32_t sbo = (uint32_t)(KP / 8) * 128;
      for (int w = 0; w < items; ++w) {
        const int m = w % M, ab = w & 1;
        const uint32_t ph = (uint32_t)((w >> 1) & 1);
        mbar_wait(&afull[ab], ph);
        mbar_wait(&tempty[ab], ph ^ 1u);
        tc::fence_after();
        int lo_any = 0;
#pragma unroll
        for (int j = 0; j < kWorkWarps; ++j) lo_any |= s_lo[ab * kWorkWarps + j];
        const uint32_t a_hi = smem_u32(sA + (ab * 2 + 0) * A_PART), a_lo = smem_u32(sA + (ab * 2 + 1) * A_PART);
        const uint32_t b_hi = smem_u32(sB + (m * 2 + 0) * B_PART), b_lo = smem_u32(sB + (m * 2 + 1) * B_PART);
        const uint32_t tacc = tbase + (uint32_t)ab * kN;
        uint32_t acc = 0;
#pragma unroll
        for (int s = 0; s < KP / 16; ++s) {
          tc::mma_f16(tacc, tc::smem_desc(a_hi + s * 256, 128, sbo), tc::smem_desc(b_hi + s * 256, 128, sbo), idesc, acc);
          acc = 1;
        }
#pragma unroll
        for (int s = 0; s < KP / 16; ++s)
          tc::mma_f16(tacc, tc::smem_desc(a_hi + s * 256, 128, sbo), tc::smem_desc(b_lo + s * 256, 128, sbo), idesc, 1);
        if (lo_any) {
#pragma unroll
          for (int s = 0; s < KP / 16; ++s)
            tc::mma_f16(tacc, tc::smem_desc(a_lo + s * 256, 128, sbo), tc::smem_desc(b_hi + s * 256, 128, sbo), idesc, 1);
        }
        tc::commit(&aempty[ab]);
        tc::commit(&tfull[ab]);
      }
    }
  } else {
    // ---------------- transform + epilogue warps ----------------
    const int ww = warp - 2;
    constexpr int TPR = 4;                                   // transform: threads per row
    constexpr int VPT = KP / TPR;                            // floats per thread
    const int tr = (kRows / kWorkWarps) * ww + lane / TPR;  // 8 rows per warp
    const int th = lane % TPR;
    const int q = warp & 3, h = ww >> 2;                     // epilogue: TMEM lane quadrant, column quarter
    const int er = 32 * q + lane;
    const float eps = (float)(KP + 11) * 2.384185791015625e-07f;  // (KP+11) * 2^-22

    auto transform = [&](int w) {
      const int ab = w & 1, xs = w % kXStages;
      mbar_wait(&xfull[xs], (uint32_t)((w / kXStages) & 1));
      const float* xr = reinterpret_cast<const float*>(sX + xs * X_STAGE) + tr * KP + th * VPT;
      float v[VPT];
#pragma unroll
      for (int j = 0; j < VPT; j += 4) {
        const float4 f = *reinterpret_cast<const float4*>(xr + j);
        v[j] = f.x;
        v[j + 1] = f.y;
        v[j + 2] = f.z;
        v[j + 3] = f.w;
      }
      float amax = 0.f;
#pragma unroll
      for (int j = 0; j < VPT; ++j) amax = fmaxf(amax, fabsf(v[j]));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));  // every lane has consumed its loads
      if (lane == 0) mbar_arrive(&xempty[xs]);
      int ex = 0;
      const bool fin = amax > 0.f && amax <= 3.4e38f;
      if (fin) frexpf(amax, &ex);
      const float scale = fin ? ldexpf(1.0f, 14 - ex) : 1.0f;
      uint32_t hw[VPT / 2], lw[VPT / 2];
      float x2 = 0.f, x1 = 0.f;
      int lo_nz = 0;
#pragma unroll
      for (int j = 0; j < VPT; j += 2) {
        const float s0 = v[j] * scale, s1 = v[j + 1] * scale;
        const __half h0 = __float2half_rn(s0), h1 = __float2half_rn(s1);
        const __half l0 = __float2half_rn(s0 - __half2float(h0)), l1 = __float2half_rn(s1 - __half2float(h1));
        lo_nz |= ((__half_as_ushort(l0) | __half_as_ushort(l1)) & 0x7fff) != 0;
        hw[j / 2] = __half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
        lw[j / 2] = __half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
        x2 = fmaf(s0, s0, fmaf(s1, s1, x2));
        x1 += fabsf(s0) + fabsf(s1);
      }
      x2 += __shfl_xor_sync(0xffffffffu, x2, 1);
      x2 += __shfl_xor_sync(0xffffffffu, x2, 2);
      x1 += __shfl_xor_sync(0xffffffffu, x1, 1);
      x1 += __shfl_xor_sync(0xffffffffu, x1, 2);
      const unsigned bal = __ballot_sync(0xffffffffu, lo_nz);
      mbar_wait(&aempty[ab], (uint32_t)(((w >> 1) & 1) ^ 1));
      uint8_t* ahi = sA + (ab * 2 + 0) * A_PART;
      uint8_t* alo = sA + (ab * 2 + 1) * A_PART;
#pragma unroll
      for (int c = 0; c < VPT / 8; ++c) {
        const int k = th * VPT + 8 * c;
        *reinterpret_cast<uint4*>(ahi + tc::kmajor_off(tr, k, KP)) =
            make_uint4(hw[4 * c], hw[4 * c + 1], hw[4 * c + 2], hw[4 * c + 3]);
        *reinterpret_cast<uint4*>(alo + tc::kmajor_off(tr, k, KP)) =
            make_uint4(lw[4 * c], lw[4 * c + 1], lw[4 * c + 2], lw[4 * c + 3]);
      }
      if (VPT % 8) {  // KP = 16: 4 floats per thread, half a 16-byte chunk
        const int k = th * VPT;
        *reinterpret_cast<uint2*>(ahi + tc::kmajor_off(tr, k, KP)) = make_uint2(hw[0], hw[1]);
        *reinterpret_cast<uint2*>(alo + tc::kmajor_off(tr, k, KP)) = make_uint2(lw[0], lw[1]);
      }
      // 4 stats buffers: a warp can run at most 3 items ahead of the slowest epilogue
      // reader (MMA(w+2) waits for every warp's tempty arrival of item w)
      if (th == 0) s_stats[(w & 3) * kRows + tr] = make_float4(scale, sqrtf(x2) * 1.00001f, x1 * 1.00001f, 0.f);
      if (lane == 0) s_lo[ab * kWorkWarps + ww] = (bal != 0);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
    };

    auto epilogue = [&](int w) {
      const int m = w % M, ab = w & 1;
      const int t = (int)blockIdx.x + (w / M) * (int)gridDim.x;
      mbar_wait(&tfull[ab], (uint32_t)((w >> 1) & 1));
      tc::fence_after();
      const float4 st = s_stats[(w & 3) * kRows + er];
      const float4 cs = *reinterpret_cast<const float4*>(s_cstat + 4 * m);  // C2, C1, CN, s_c
      const float sr = st.x, x2 = st.y, x1 = st.z;
      // rigorous bound on |computed - exact| of g = s_r s_c (|c|^2 - 2 x.c) (see header)
      const float dS = eps * x2 * cs.x + 2.98023223876953125e-08f * (x1 + cs.y);  // 2^-25
      const float big = sr * cs.z + x2 * cs.x;
      const float dg = 2.0f * dS + 1.1920928955078125e-07f * big;                // 2^-23
      const float margin = 2.0f * dg * 1.001f + 1e-12f * big;
      // e'_l = s_c |x - c_l|^2 = cnc_l - (2/s_r) S'_l + s_c |x|^2 >= 0 (offset widened by the
      // error bound so that every computed e' is nonnegative: its bits then order as uint)
      const float nsr = -2.0f / sr;
      const float off = cs.w * (x2 * x2) / (sr * sr) * 1.0001f + 2.0f * dg / sr;
      const float* cn = s_cnc + m * kN + 64 * h;
      uint32_t k[64];
      const uint32_t tacc = tbase + (uint32_t)ab * kN + 64u * h + ((uint32_t)(32 * q) << 16);
      {
        uint32_t r0[16], r1[16], r2[16], r3[16];
        tc::tmem_ld16(tacc + 0, r0);
        tc::tmem_ld16(tacc + 16, r1);
        tc::tmem_ld16(tacc + 32, r2);
        tc::tmem_ld16(tacc + 48, r3);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          k[j] = r0[j];
          k[16 + j] = r1[j];
          k[32 + j] = r2[j];
          k[48 + j] = r3[j];
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      // keys: e' bits with the low 6 mantissa bits replaced by the column (one LOP3 each)
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const float e = fmaf(__uint_as_float(k[j]), nsr, cn[j]) + off;
        k[j] = (__float_as_uint(e) & ~63u) | (uint32_t)j;
      }
      uint32_t b = k[0];
#pragma unroll
      for (int j = 1; j + 1 < 64; j += 2) b = min(b, min(k[j], k[j + 1]));
      b = min(b, k[63]);
      // runner-up key: keys are unique, so min over (k - (b + 1)) mod 2^32 maps the winner
      // to 0xffffffff and every other key k to k - b - 1 (order preserved)
      const uint32_t bp = b + 1u;
      uint32_t rr = 0xffffffffu;
#pragma unroll
      for (int j = 0; j < 64; j += 2) rr = min(rr, min(k[j] - bp, k[j + 1] - bp));
      rr += bp;
      // merge the four column quarters of each row (warps sharing quadrant q)
      if (h > 0) s_merge[(h - 1) * kRows + er] = make_float4(__uint_as_float(b), __uint_as_float(rr), 0.f, 0.f);
      named_bar(1 + q, 128);
      if (h == 0) {
        uint32_t wb = b, wr = rr;
        int wh = 0;
        float other = __int_as_float(0x7f800000);  // min lower bound of losing quarters' winners
#pragma unroll
        for (int u = 1; u < 4; ++u) {
          const float4 o = s_merge[(u - 1) * kRows + er];
          const uint32_t ob = __float_as_uint(o.x);
          if ((ob & ~63u) < (wb & ~63u)) {  // strictly smaller value: ties keep the lower quarter
            other = fminf(other, __uint_as_float(wb & ~63u));
            wb = ob;
            wr = __float_as_uint(o.y);
            wh = u;
          } else {
            other = fminf(other, __uint_as_float(ob & ~63u));
          }
        }
        const int64_t n = (int64_t)t * kRows + er;
        if (n < p.n) {
          const float w_hi = __uint_as_float((wb & ~63u) | 63u);
          const float r_lo = fminf(__uint_as_float(wr & ~63u), other);
          // e' values are g/s_r units; a non-finite row makes the margin NaN/inf
          const bool cert = (r_lo - w_hi) * sr > margin;
          if (cert) {
            p.codes[n * p.stride + m] = (uint8_t)(64 * wh + (int)(wb & 63u));
          } else {
            const unsigned f = atomicAdd(&p.counters[0], 1u);
            if (f < p.flag_cap)
              p.flags[f] = (uint32_t)(n * M + m);
            else
              p.counters[1] = 1u;
          }
        }
      }
      named_bar(1 + q, 128);  // s_merge is reused by the next item
    };

    if (items > 0) transform(0);
    for (int w = 0; w < items; ++w) {
      if (w + 1 < items) transform(w + 1);
      epilogue(w);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tbase, 512);
  }
}

// Codebook preparation: one block of 256 threads per subspace.
template <int KP>
__global__ void __launch_bounds__(256) encode_prep_kernel(const float* __restrict__ cw, int m, int l, int ks,
                                                         uint8_t* __restrict__ bprep, float* __restrict__ cnc,
                                                         float* __restrict__ cstat) {
  __shared__ float red[8];
  __shared__ float s_scale;
  const int mm = blockIdx.x, row = threadIdx.x, lane = row & 31, warp = row >> 5;
  const float* c = cw + ((size_t)mm * l + row) * ks;
  float amax = 0.f;
  if (row < l)
    for (int k = 0; k < ks; ++k) amax = fmaxf(amax, fabsf(c[k]));
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) red[warp] = amax;
  __syncthreads();
  if (row == 0) {
    float a = 0.f;
    for (int i = 0; i < 8; ++i) a = fmaxf(a, red[i]);
    int ex = 0;
    if (a > 0.f) frexpf(a, &ex);
    s_scale = a > 0.f ? ldexpf(1.0f, 14 - ex) : 1.0f;
  }
  __syncthreads();
  const float sc = s_scale;
  uint8_t* bh = bprep + (size_t)(mm * 2 + 0) * kN * KP * 2;
  uint8_t* bl = bprep + (size_t)(mm * 2 + 1) * kN * KP * 2;
  double nn = 0.0;
  float c2 = 0.f, c1 = 0.f;
  for (int k = 0; k < KP; ++k) {
    const float v = (row < l && k < ks) ? c[k] * sc : 0.f;
    const __half hi = __float2half_rn(v);
    const __half lo = __float2half_rn(v - __half2float(hi));
    *reinterpret_cast<__half*>(bh + tc::kmajor_off(row, k, KP)) = hi;
    *reinterpret_cast<__half*>(bl + tc::kmajor_off(row, k, KP)) = lo;
    if (row < l && k < ks) {
      const double cd = (double)c[k];
      nn += cd * cd;
    }
    c2 = fmaf(v, v, c2);
    c1 += fabsf(v);
  }
  const float cn = row < l ? (float)(nn * (double)sc) : __int_as_float(0x7f800000);
  cnc[mm * kN + row] = cn;
  // block maxima of C2, C1, CN over real rows
  float v2 = row < l ? sqrtf(c2) * 1.00001f : 0.f, v1 = row < l ? c1 * 1.00001f : 0.f, vn = row < l ? cn : 0.f;
  for (int o = 16; o > 0; o >>= 1) {
    v2 = fmaxf(v2, __shfl_xor_sync(0xffffffffu, v2, o));
    v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, o));
    vn = fmaxf(vn, __shfl_xor_sync(0xffffffffu, vn, o));
  }
  __shared__ float r2[8], r1[8], rn[8];
  if (lane == 0) {
    r2[warp] = v2;
    r1[warp] = v1;
    rn[warp] = vn;
  }
  __syncthreads();
  if (row == 0) {
    float a = 0.f, b = 0.f, d = 0.f;
    for (int i = 0; i < 8; ++i) {
      a = fmaxf(a, r2[i]);
      b = fmaxf(b, r1[i]);
      d = fmaxf(d, rn[i]);
    }
    cstat[4 * mm + 0] = a;
    cstat[4 * mm + 1] = b;
    cstat[4 * mm + 2] = d * 1.00001f;
    cstat[4 * mm + 3] = sc;  // s_c: the epilogue's |x|^2 offset
  }
}

// Exact float64 decision for the pairs the certificate did not cover; one warp per pair.
__global__ void encode_exact_kernel(const float* __restrict__ x, int64_t n, int d, const float* __restrict__ cw, int m,
                                    int l, int ks, const uint32_t* __restrict__ flags,
                                    const unsigned int* __restrict__ counters, uint32_t flag_cap,
                                    uint8_t* __restrict__ codes, int stride) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool all = counters[1] != 0;
  const int64_t total = all ? n * m : (int64_t)min(counters[0], flag_cap);
  for (int64_t w = gw; w < total; w += nw) {
    const int64_t pair = all ? w : (int64_t)flags[w];
    const int64_t row = pair / m;
    const int mm = (int)(pair - row * m);
    const float* xv = x + row * d + (size_t)mm * ks;
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bl = 0x7fffffff;
    for (int c = lane; c < l; c += 32) {
      const float* cv = cw + ((size_t)mm * l + c) * ks;
      double acc = 0.0;
      for (int k = 0; k < ks; ++k) {
        const double df = __dsub_rn((double)xv[k], (double)cv[k]);
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
      if (argmin_less(acc, c, best, bl)) {
        best = acc;
        bl = c;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bl, o);
      if (argmin_less(ob, oi, best, bl)) {
        best = ob;
        bl = oi;
      }
    }
    if (lane == 0) codes[row * stride + mm] = (uint8_t)bl;
  }
}

__global__ void encode_stats_kernel(const unsigned int* __restrict__ counters, unsigned long long* __restrict__ out) {
  *out += (unsigned long long)counters[0];  // pairs not certified (all re-decided in fp64)
}

}  // namespace enc

// ---------------------------------------------------------------------------
// host side
namespace {
struct EncWS {
  std::mutex mu;
  void* p = nullptr;
  size_t bytes = 0;
};
EncWS g_encws[64];

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

template <int KP>
int launch_encode_tc(const float* d_x, int64_t n, int d, const float* d_cw, int m, int l, uint8_t* d_codes, int stride,
                     unsigned long long* flagged_out, cudaStream_t stream) {
  using namespace enc;
  const DevInfo& di = dev_info();
  const size_t smem = smem_bytes<KP>(m);
  int dev = 0;
  cudaGetDevice(&dev);
  EncWS& ws = g_encws[dev & 63];
  std::lock_guard<std::mutex> lock(ws.mu);
  const size_t b_bytes = (size_t)m * 2 * kN * KP * 2;
  const uint32_t cap = (uint32_t)std::min<int64_t>(n * m, (int64_t)(n * m) / 64 + 65536);
  const size_t need = align_up(b_bytes, 256) + align_up((size_t)m * kN * 4, 256) + align_up((size_t)m * 16, 256) +
                      align_up((size_t)cap * 4, 256) + 256;
  if (ws.bytes < need) {
    if (ws.p) cudaFree(ws.p);
    ws.p = nullptr;
    ws.bytes = 0;
    PQK_CUDA_TRY(cudaMalloc(&ws.p, need));
    ws.bytes = need;
  }
  char* base = static_cast<char*>(ws.p);
  uint8_t* bprep = reinterpret_cast<uint8_t*>(base);
  float* cnc = reinterpret_cast<float*>(base + align_up(b_bytes, 256));
  float* cstat = reinterpret_cast<float*>(reinterpret_cast<char*>(cnc) + align_up((size_t)m * kN * 4, 256));
  uint32_t* flags = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(cstat) + align_up((size_t)m * 16, 256));
  unsigned int* counters = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(flags) + align_up((size_t)cap * 4, 256));

  CUtensorMap map;
  auto encoder = tensor_map_encoder();
  if (!encoder) return fail(PQK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  const cuuint32_t box[2] = {(cuuint32_t)KP, (cuuint32_t)kRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult cr = encoder(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(d_x), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(PQK_ECUDA, "cuTensorMapEncodeTiled failed");

  PQK_CUDA_TRY(cudaMemsetAsync(counters, 0, 8, stream));
  encode_prep_kernel<KP><<<m, 256, 0, stream>>>(d_cw, m, l, KP, bprep, cnc, cstat);
  PQK_LAUNCH_CHECK("encode_prep_kernel");
  EncParams ep{};
  ep.x = d_x;
  ep.cw = d_cw;
  ep.bprep = bprep;
  ep.cnc = cnc;
  ep.cstat = cstat;
  ep.n = n;
  ep.d = d;
  ep.m = m;
  ep.l = l;
  ep.ks = KP;
  ep.codes = d_codes;
  ep.stride = stride;
  ep.flags = flags;
  ep.counters = counters;
  ep.flag_cap = cap;
  ep.ntiles = (int)((n + kRows - 1) / kRows);
  auto kern = encode_tc_kernel<KP>;
  PQK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::max(1, std::min(di.sms, ep.ntiles));
  kern<<<grid, kThreads, smem, stream>>>(map, ep);
  PQK_LAUNCH_CHECK("encode_tc_kernel");
  encode_exact_kernel<<<di.sms, 256, 0, stream>>>(d_x, n, d, d_cw, m, l, KP, flags, counters, cap, d_codes, stride);
  PQK_LAUNCH_CHECK("encode_exact_kernel");
  encode_stats_kernel<<<1, 1, 0, stream>>>(counters, flagged_out);
  PQK_LAUNCH_CHECK("encode_stats_kernel");
  return PQK_OK;
}
}  // namespace

// Tensor-core encoder eligibility and launch (called by pqk_encode_device).
int encode_tc_try(const float* d_x, int64_t n, int d, const float* d_cw, int m, int l, uint8_t* d_codes, int stride,
                  unsigned long long* flagged_out, cudaStream_t stream, bool* used) {
  *used = false;
  const int ks = d / m;
  if (n < 1 || n >= ((int64_t)1 << 31) / std::max(m, 1) || (d % 4) != 0 || (reinterpret_cast<uintptr_t>(d_x) & 15))
    return PQK_OK;
  const DevInfo& di = dev_info();
  int rc = PQK_OK;
  switch (ks) {
    case 16:
      if (enc::smem_bytes<16>(m) > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tc<16>(d_x, n, d, d_cw, m, l, d_codes, stride, flagged_out, stream);
      break;
    case 32:
      if (enc::smem_bytes<32>(m) > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tc<32>(d_x, n, d, d_cw, m, l, d_codes, stride, flagged_out, stream);
      break;
    case 64:
      if (enc::smem_bytes<64>(m) > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tc<64>(d_x, n, d, d_cw, m, l, d_codes, stride, flagged_out, stream);
      break;
    default:
      return PQK_OK;
  }
  if (rc == PQK_OK) *used = true;
  return rc;
}

}  // namespace pqk
