// pqk_encode_tc.cu — tcgen05 (5th-gen tensor core) building blocks of the PQ encoder.
//
// pqk_tc_selftest: one 128 x 256 x K fp16 tile through the full tcgen05 path
// (canonical no-swizzle K-major smem operands, UMMA descriptors, TMEM accumulator,
// tcgen05.commit -> mbarrier, tcgen05.ld epilogue).  It is the device diagnostic the
// encoder's tests run first: a wrong descriptor shows up here as a wrong product.
#include "pqk_common.cuh"
#include "pqk_tc.cuh"
#ifndef ENC_XST
#define ENC_XST 3
#endif
#ifndef FILTER_ROWS
#define FILTER_ROWS 4
#endif

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
// Each CTA owns one subspace m (blockIdx.x % M) and walks 128-vector tiles.  For a
// tile, one accumulator of 128 x 256 fp32 in TMEM receives
//
//   D_rj = s^2 |x_r|^2 - 2 s^2 x_r.c_j + s^2 |c_j|^2    (= s^2 |x_r - c_j|^2)
//
// entirely from tcgen05.mma: the x and -2c operands are scaled by one power of two s
// per subspace and split v = hi + lo into fp16 pairs (hi.hi + hi.lo [+ lo.hi when the
// tile's x are not exactly fp16]); s^2|c_j|^2 and the row's s^2|x_r|^2 enter through
// 16 extra K columns of the hi pass (three fp16 parts each, times an exact power of
// two).  The epilogue therefore has no per-distance floating-point work: accumulator
// words compare as signed int32 (so that the rare negative values produced by rounding
// next to a zero distance still sort below every positive value), and the best and
// runner-up come from group (j / 16) and class (j % 16) minima, one 3-input min per
// column.  They give a certificate: the winner is certified when the runner-up exceeds it
// by more than twice a rigorous bound on |computed - exact| (split, skipped lo.lo term,
// tensor-core accumulation).  Uncertified (vector, subspace) pairs are re-decided by
// the exact float64 sequential sum (scipy cdist order) in encode_exact_kernel.
//
// Warp roles (persistent, one CTA per SM, 576 threads):
//   warp 0   TMA producer: 2-D tensor-map loads of X[128 rows x dsub] per tile
//   warp 1   TMEM allocator + single-thread tcgen05.mma issuer (2 accumulators of
//            128 x 256 fp32 = all 512 TMEM columns, double-buffered)
//   warps 2-9 epilogue (tcgen05.ld, partition minima, certificate), whole rows: warp w
//            reads TMEM lane quadrant w % 4 of accumulator (w - 2) / 4
//   warps 10-17 transform (fp32 -> scaled fp16 hi/lo + extension columns in the UMMA
//            K-major layout), 16 rows each
// ===========================================================================
#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>

namespace pqk {
namespace enc {

// Timing experiments of tools/exp_encode.sh (results are wrong when set): bit 0 the transform
// only runs its barrier protocol, bit 1 the epilogue only reads the accumulator, bit 2 one
// MMA instruction per item.
#ifndef ENC_EXP
#define ENC_EXP 0
#endif
constexpr int kRows = 128;
constexpr int kN = 256;
constexpr int kExt = 16;       // extension K columns of the hi pass
constexpr int kEpiWarps = 8;   // 2 per TMEM lane quadrant: one per accumulator
constexpr int kTrWarps = 8;    // transform warps (16 rows each)
constexpr int kThreads = (2 + kEpiWarps + kTrWarps) * 32;
// encode_tc_kernel's transform: one thread per row (4 warps x 32 rows), the row's KP
// columns streamed in 8-column groups (no cross-lane reductions, no per-row shuffles)
constexpr int kTrWarpsR = 4;
// ENC_TRSETS transform warp sets take alternate items (measured on a B200: two sets are 3%
// slower than one, the kernel is bound by ALU-pipe issue, not by the transform's latency)
#ifndef ENC_TRSETS
#define ENC_TRSETS 1
#endif
constexpr int kTrSets = ENC_TRSETS;
constexpr int kThreadsR = (2 + kEpiWarps + kTrSets * kTrWarpsR) * 32;
constexpr int kChunk = 32;     // epilogue columns per tcgen05.ld pair
constexpr bool kMmaHalves = false;  // N=128 MMA halves (separately released) vs N=256
constexpr float kX2Limit = 1073741824.0f;  // 2^30: |s x|^2 bound for the fp16 extension parts

// per-subspace constants written by encode_prep_kernel (floats)
enum { CST_S = 0, CST_ACN = 1, CST_CB = 2, CST_CN = 3, CST_S1C = 4, CST_VALID = 5, CST_LEN = 8 };

template <int KP>
struct Geo {
  static constexpr int KE = KP + kExt;
  static constexpr int XST = KP >= 64 ? 2 : ENC_XST;  // X stages (TMA ring depth)
  static constexpr bool SWZ = KP >= 32;         // X tile loaded with the 128-byte swizzle
  static constexpr int B_HI = kN * KE * 2;
  static constexpr int B_LO = kN * KP * 2;
  static constexpr int B_BYTES = B_HI + B_LO;
  static constexpr int A_HI = kRows * KE * 2;
  static constexpr int A_LO = kRows * KP * 2;
  static constexpr int A_BYTES = A_HI + A_LO;
  static constexpr int X_STAGE = kRows * KP * 4;  // 128 x dsub floats (dsub <= KP)
  static constexpr int OFF_X = B_BYTES;           // multiple of 1024 (swizzled TMA destination)
  static constexpr int OFF_A = OFF_X + XST * X_STAGE;
  static constexpr int OFF_STATS = OFF_A + 2 * A_BYTES;        // float4 [4][128]
  static constexpr int OFF_LO = OFF_STATS + 4 * kRows * 16;    // int [2][kTrWarps]
  static constexpr int OFF_CST = OFF_LO + 2 * kTrWarps * 4;    // float [8]
  static constexpr int OFF_BAR = OFF_CST + CST_LEN * 4;        // uint64 [32]
  static constexpr int OFF_TBASE = OFF_BAR + 32 * 8;
  static constexpr int SMEM = OFF_TBASE + 16 + 1024;           // + alignment slack
};

struct EncParams {
  const uint8_t* bprep;  // [M][B_BYTES]: hi+ext (256 x KE) then lo (256 x KP), fp16 K-major
  const float* cst;      // [M][CST_LEN]
  const float* bch;      // [M][kMaxChunks] K-streamed kernel: max_j |B_j| over each 32-column chunk
  int64_t n;
  int m, ks;
  uint8_t* codes;
  int stride;
  uint32_t* flags;         // [M][flag_cap] uncertified rows per subspace
  unsigned int* counters;  // [0] flagged total, [1] overflow, [2 + m] per-subspace count
  uint32_t flag_cap;
  int ntiles;        // 128-row tiles
  int tstride;       // CTAs per subspace
  uint32_t keymask;  // ~15u, a run-time value so that key packing is one LOP3
  uint32_t one;      // 1
  uint32_t* tcmask;  // K-streamed kernel: [M][flag_cap][8] candidate codewords of each uncertified pair
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int imin3(int a, int b, int c) { return min(a, min(b, c)); }
__device__ __forceinline__ uint32_t umin3(uint32_t a, uint32_t b, uint32_t c) { return min(a, min(b, c)); }

// one lane of a converged warp (elect.sync: ptxas then knows a single thread runs the branch)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

// 32 columns (two tcgen05.ld x16) into r[0..31]
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr), "r"(taddr + 16u));
}

// tcgen05.wait::ld with the destination registers as operands, so that no use of them
// can be scheduled before the wait
__device__ __forceinline__ void tmem_wait32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// x * one + y on the FMA pipe (one = 1 at run time: keeps ptxas from fusing the add
// into an ALU VIADDMNMX, the epilogue being ALU-bound)
__device__ __forceinline__ uint32_t imad(uint32_t x, uint32_t one, uint32_t y) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(y));
  return r;
}

// Best and runner-up of a row's 256 accumulator words by two partitions of the columns:
// groups g = j / 16 and classes q = j % 16 (a group and a class share exactly one column).
// Every column other than the best lies outside the best's group or outside its class,
// so runner-up = min(second-smallest group minimum, second-smallest class minimum).
// Words compare as signed int32 (raw fp32 bits: the rare negative values next to a zero
// distance sort below every positive one; two negatives in the wrong order only make the
// certificate fail).  Per column: half a 3-input min for its class, half for its group.
__device__ __forceinline__ int tree_min16(const uint32_t (&k)[32], int o) {
  const int t0 = imin3((int)k[o], (int)k[o + 1], (int)k[o + 2]);
  const int t1 = imin3((int)k[o + 3], (int)k[o + 4], (int)k[o + 5]);
  const int t2 = imin3((int)k[o + 6], (int)k[o + 7], (int)k[o + 8]);
  const int t3 = imin3((int)k[o + 9], (int)k[o + 10], (int)k[o + 11]);
  const int t4 = imin3((int)k[o + 12], (int)k[o + 13], (int)k[o + 14]);
  return min(imin3(t0, t1, t2), imin3(t3, t4, (int)k[o + 15]));
}
// smallest two group minima (G2 = G1 on a tie, so a tie never certifies) and G1's group
__device__ __forceinline__ void fold_group(int v, int g, int& G1, int& G2, int& gi) {
  gi = v < G1 ? g : gi;
  G2 = min(G2, max(G1, v));
  G1 = min(G1, v);
}
// one 32-column chunk c: groups 2c, 2c+1; classes q and q (columns q, q+16)
__device__ __forceinline__ void chunk_fold(const uint32_t (&k)[32], int c, int (&cls)[16], int& G1, int& G2,
                                           int& gi) {
#pragma unroll
  for (int q = 0; q < 16; ++q) cls[q] = imin3(cls[q], (int)k[q], (int)k[q + 16]);
  fold_group(tree_min16(k, 0), 2 * c, G1, G2, gi);
  fold_group(tree_min16(k, 16), 2 * c + 1, G1, G2, gi);
}
// second-smallest class minimum (as a key truncated to 4 bits less, class in the low
// bits: unique keys) and the class of the smallest
__device__ __forceinline__ void class_best2(const int (&cls)[16], uint32_t kmask, uint32_t one, int& qb, int& Y,
                                            int* best_key = nullptr) {
  uint32_t ck[32];
#pragma unroll
  for (int q = 0; q < 16; ++q) ck[q] = ((uint32_t)cls[q] & kmask) | (uint32_t)q;
  const int b = tree_min16(ck, 0);
  if (best_key) *best_key = b;
  qb = b & 15;
  const uint32_t nbp = ~(uint32_t)b;  // -(b + 1): the winner maps to 0xffffffff
#pragma unroll
  for (int q = 0; q < 16; ++q) ck[q] = imad(ck[q], one, nbp);
  const uint32_t t0 = umin3(ck[0], ck[1], ck[2]), t1 = umin3(ck[3], ck[4], ck[5]);
  const uint32_t t2 = umin3(ck[6], ck[7], ck[8]), t3 = umin3(ck[9], ck[10], ck[11]);
  const uint32_t t4 = umin3(ck[12], ck[13], ck[14]);
  Y = (int)(min(umin3(t0, t1, t2), umin3(t3, t4, ck[15])) - nbp) & (int)kmask;
}

// one 32-column chunk c, group minima kept per group (encode_tc_kernel's epilogue: the
// running best / runner-up fold of fold_group cost 5 ALU-pipe instructions per group, the
// kernel's limiting pipe; the 16 minima are ranked once per row by class_best2 instead)
__device__ __forceinline__ void chunk_fold_keep(const uint32_t (&k)[32], int c, int (&cls)[16], int (&grp)[16]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) cls[q] = imin3(cls[q], (int)k[q], (int)k[q + 16]);
  grp[2 * c] = tree_min16(k, 0);
  grp[2 * c + 1] = tree_min16(k, 16);
}

// Epilogue of one 128-row item for one epilogue warp (row n of TMEM lane quadrant q):
// the 256 accumulator columns (two N=128 halves, signalled and released separately),
// best / runner-up by the group x class partitions, certificate, code store or flag.
__device__ __forceinline__ void epilogue_row(const EncParams& p, int m, int64_t n, uint32_t tacc, uint64_t* tfull2,
                                             uint64_t* tempty2, uint32_t ph, float4 st, float eps_main2,
                                             float eps_main3, float eps_ext, float cb, float cnm, float s1c,
                                             float sqrt_kp, int lane) {
  int cls[16], grp[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) cls[q] = 0x7fffffff;
  uint32_t ka[32], kb[32];
  tmem_ld32(tacc, ka);
#pragma unroll
  for (int c = 0; c < kN / kChunk; c += 2) {
    tmem_wait32(ka);
    tmem_ld32(tacc + (uint32_t)((c + 1) * kChunk), kb);
    if (!(ENC_EXP & 2)) chunk_fold_keep(ka, c, cls, grp);
    else grp[2 * c] = grp[2 * c + 1] = (int)ka[c];
    tmem_wait32(kb);
    if (c + 2 == kN / kChunk / 2 || c + 2 == kN / kChunk) {  // a column half fully read
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty2[c + 2 == kN / kChunk ? 1 : 0]);
    }
    if (c + 2 < kN / kChunk) {
      if (c + 2 == kN / kChunk / 2) {
        mbar_wait(&tfull2[1], ph);
        tc::fence_after();
      }
      tmem_ld32(tacc + (uint32_t)((c + 2) * kChunk), ka);
    }
    if (!(ENC_EXP & 2)) chunk_fold_keep(kb, c + 1, cls, grp);
    else grp[2 * c + 2] = grp[2 * c + 3] = (int)kb[c];
  }
  if (n < p.n) {
    int qb, Y, gi, G2, bk;
    class_best2(cls, p.keymask, p.one, qb, Y, &bk);
    class_best2(grp, p.keymask, p.one, gi, G2);
    const int R = min(G2, Y);
    // every key is truncated by 4 mantissa bits (within 16 ulp <= 2^-19 |v| of its value,
    // below it for v >= 0, above it for v < 0).  The best word W lies between the smallest
    // class key's two ends (low bits 0 / 15; w_hi: the larger as floats); R bounds the
    // runner-up from below after the (1 + 2^-17) step for negative words.  gi and qb can name
    // different columns only when another word shares W's upper 28 bits, i.e. lies within
    // d15 = 15 ulp of it: the d15 margin keeps such rows from certifying.
    const float w_a = __int_as_float(bk | 15), w_b = __int_as_float(bk & ~15);
    const float w_hi = fmaxf(w_a, w_b), d15 = fabsf(w_a - w_b), rv = __int_as_float(R);
    const float r_lo = rv >= 0.f ? rv : rv * 1.00000762939453125f;  // 1 + 2^-17
    // rigorous bound on |computed - exact| of any D_rj (see header)
    const float P = st.y * cb * 1.001f;  // >= sum |split products|
    const float E = (st.w != 0.f ? eps_main3 : eps_main2) * P + eps_ext * (P + cnm + st.x) * 1.001f  //
                    + 4.76837158203125e-07f * P                                 // 4 * 2^-23: split, lo.lo
                    + 2.98023223876953125e-08f * (sqrt_kp * st.y + s1c)          // 2^-25: subnormal lo parts
                    + 9.313225746154785e-10f * (cnm + st.x)                      // 2^-30: extension parts
                    + 1e-3f;
    const bool cert = ENC_EXP ? true
                              : (st.z != 0.f && (r_lo - w_hi) > 2.0f * E * 1.0001f + 1.01f * d15);
    if (cert) {
      p.codes[n * p.stride + m] = (uint8_t)(16 * gi + qb);
    } else {
      atomicAdd(&p.counters[0], 1u);
      const unsigned f = atomicAdd(&p.counters[2 + m], 1u);
      if (f < p.flag_cap)
        p.flags[(size_t)m * p.flag_cap + f] = (uint32_t)n;
      else
        p.counters[1] = 1u;
    }
  }
}

// Epilogue of the K-streamed kernel: two accumulators, H (hi . hi + extension, columns
// [0, 256)) and L (hi . lo + lo . hi, columns [256, 512)), summed per column (one fp32
// rounding) before the same partition minima and certificate.  st.w carries the row's
// prefix bound W = sum over chunks c of the running sum of |x_c| max_j |B_j,c| (bounds
// every max |addend| of H's two hi . hi instructions per chunk).
//
// Nothing of the next item can overlap this epilogue (both accumulators belong to one
// item), so each TMEM lane quadrant is served by two warps: half 0 folds codewords
// [0, 128), half 1 codewords [128, 256).  Half 1 hands its class minima and its best /
// runner-up group minima to half 0 through shared memory (ex, 20 words per row); half 0
// merges, decides and hands back the candidate threshold of its uncertified rows; both then
// build their half of the candidate mask, re-reading only the 32-column chunks whose group
// minima (kept in registers) admit a candidate.  Named barrier bar (64 threads) orders
// the three hand-overs.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])
               :
               : "memory");
}
__device__ __forceinline__ void pair_sync(int bar) { asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory"); }

constexpr int kExWords = 20;  // per row: 16 class minima, G1, G2, gi, pad (80 B: conflict-free uint4 rows)

// H + L of one 32-column chunk into ka (L read in two 16-column pieces)
__device__ __forceinline__ void load_sum32(uint32_t tacc, int c, uint32_t (&ka)[32]) {
  uint32_t kb[16];
  tmem_ld32(tacc + (uint32_t)(c * kChunk), ka);
  tmem_ld16(tacc + (uint32_t)(kN + c * kChunk), kb);
  tmem_wait32(ka);
  tmem_wait16(kb);
#pragma unroll
  for (int j = 0; j < 16; ++j) ka[j] = __float_as_uint(__fadd_rn(__uint_as_float(ka[j]), __uint_as_float(kb[j])));
  tmem_ld16(tacc + (uint32_t)(kN + c * kChunk + 16), kb);
  tmem_wait16(kb);
#pragma unroll
  for (int j = 0; j < 16; ++j)
    ka[16 + j] = __float_as_uint(__fadd_rn(__uint_as_float(ka[16 + j]), __uint_as_float(kb[j])));
}

template <bool kPair>
__device__ __forceinline__ void arrive_at_issuer(uint64_t* bar) {  // the MMA issuer's barrier (pair: in cluster rank 0)
  if (kPair) tc::mbar_arrive_rank0(bar);
  else mbar_arrive(bar);
}

template <bool kPair>
__device__ __forceinline__ void epilogue_row_split(const EncParams& p, int m, int64_t n, uint32_t tacc,
                                                   uint64_t* tempty2, float4 st, float eps_h, float eps_l,
                                                   float eps_ext, float cb, float cnm, float s1c, float sqrt_kp,
                                                   int lane, int half, uint32_t* ex_row, int bar) {
  int cls[16], grp[8];
#pragma unroll
  for (int q = 0; q < 16; ++q) cls[q] = 0x7fffffff;
  int G1 = 0x7fffffff, G2 = 0x7fffffff, gi = 0;
  uint32_t ka[32];
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) {
    const int c = 4 * half + cc;
    load_sum32(tacc, c, ka);
#pragma unroll
    for (int q = 0; q < 16; ++q) cls[q] = imin3(cls[q], (int)ka[q], (int)ka[q + 16]);
    grp[2 * cc] = tree_min16(ka, 0);
    grp[2 * cc + 1] = tree_min16(ka, 16);
    fold_group(grp[2 * cc], 2 * c, G1, G2, gi);
    fold_group(grp[2 * cc + 1], 2 * c + 1, G1, G2, gi);
  }
  uint4* ex4 = reinterpret_cast<uint4*>(ex_row);
  bool flagged = false;
  float thr = __int_as_float(0xff800000);  // -inf: no candidates
  if (half == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      ex4[i] = make_uint4((uint32_t)cls[4 * i], (uint32_t)cls[4 * i + 1], (uint32_t)cls[4 * i + 2],
                          (uint32_t)cls[4 * i + 3]);
    ex4[4] = make_uint4((uint32_t)G1, (uint32_t)G2, (uint32_t)gi, 0u);
    pair_sync(bar);  // 1: partial minima of codewords [128, 256) visible to half 0
    pair_sync(bar);  // 2: thresholds visible
    thr = __uint_as_float(ex_row[0]);
  } else {
    pair_sync(bar);  // 1
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 o = ex4[i];
      cls[4 * i] = min(cls[4 * i], (int)o.x);
      cls[4 * i + 1] = min(cls[4 * i + 1], (int)o.y);
      cls[4 * i + 2] = min(cls[4 * i + 2], (int)o.z);
      cls[4 * i + 3] = min(cls[4 * i + 3], (int)o.w);
    }
    {
      // two sorted pairs of group minima merged (a tie between the halves' smallest leaves
      // G2 = G1: never certifies; the lower group index wins as in the running fold)
      const uint4 o = ex4[4];
      const int h1 = (int)o.x, h2 = (int)o.y;
      gi = h1 < G1 ? (int)o.z : gi;
      G2 = min(max(G1, h1), min(G2, h2));
      G1 = min(G1, h1);
    }
    if (n < p.n) {
      int qb, Y;
      class_best2(cls, p.keymask, p.one, qb, Y);
      const int R = min(G2, Y);
      const float w_hi = __int_as_float(G1), rv = __int_as_float(R);
      const float r_lo = rv >= 0.f ? rv : rv * 1.00000762939453125f;
      const float P = st.y * cb * 1.001f;
      const float W = fminf(st.w, (float)(p.ks / 32) * P);  // every prefix (32-column chunks) is also <= P
      const float E = eps_h * W + eps_l * P + eps_ext * (P + cnm + st.x) * 1.001f  //
                      + 4.76837158203125e-07f * P                                 // 4 * 2^-23: split, lo.lo
                      + 2.98023223876953125e-08f * (sqrt_kp * st.y + s1c)          // 2^-25: subnormal lo parts
                      + 9.313225746154785e-10f * (cnm + st.x)                      // 2^-30: extension parts
                      + 1e-3f;
      const bool cert = st.z != 0.f && (r_lo - w_hi) > 2.0f * E * 1.0001f;
      if (cert) {
        p.codes[n * p.stride + m] = (uint8_t)(16 * gi + qb);
      } else {
        flagged = true;
        // candidates: every codeword whose exact distance can be <= the winner's, i.e. computed
        // D_j <= W + 2 E (w_hi is some computed value >= the smallest one, also when negative
        // words misorder as integers); all of them for rows outside the certified range
        const float t0 = w_hi + 2.0f * E * 1.0001f;
        const float t = t0 + fabsf(t0) * 1e-6f + 1e-30f;  // the sum rounded up
        thr = (st.z != 0.f && t == t) ? t : __int_as_float(0x7f800000);
      }
    }
    ex_row[0] = __float_as_uint(thr);
    pair_sync(bar);  // 2
  }
  // candidate mask of this half's 128 codewords, for warps with an uncertified row: only
  // the chunks holding a group minimum within the threshold are read again
  uint32_t mw[4] = {0u, 0u, 0u, 0u};
  const bool cand_row = thr != __int_as_float(0xff800000);
  if (__any_sync(0xffffffffu, cand_row)) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const bool need = cand_row && (!(__int_as_float(grp[2 * cc]) > thr) || !(__int_as_float(grp[2 * cc + 1]) > thr));
      if (__any_sync(0xffffffffu, need)) {
        load_sum32(tacc, 4 * half + cc, ka);
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) word |= !(__uint_as_float(ka[j]) > thr) ? (1u << j) : 0u;  // NaN: a candidate
        mw[cc] = word;
      }
    }
  }
  tc::fence_before();
  if (half == 1) {
    ex4[1] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    __syncwarp();
    if (lane == 0) {
      arrive_at_issuer<kPair>(&tempty2[0]);
      arrive_at_issuer<kPair>(&tempty2[1]);
    }
    pair_sync(bar);  // 3: mask words of codewords [128, 256) visible
    return;
  }
  pair_sync(bar);  // 3
  const uint4 mo = ex4[1];
  // released only after the pair's shared-memory row was read: half 1 writes it again only
  // behind the next item's accumulators, which wait for this arrive
  __syncwarp();
  if (lane == 0) {
    arrive_at_issuer<kPair>(&tempty2[0]);
    arrive_at_issuer<kPair>(&tempty2[1]);
  }
  if (flagged) {
    atomicAdd(&p.counters[0], 1u);
    const unsigned f = atomicAdd(&p.counters[2 + m], 1u);
    if (f < p.flag_cap) {
      p.flags[(size_t)m * p.flag_cap + f] = (uint32_t)n;
      uint4* dst = reinterpret_cast<uint4*>(p.tcmask + ((size_t)m * p.flag_cap + f) * 8);
      dst[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
      dst[1] = mo;
    } else {
      p.counters[1] = 1u;
    }
  }
}

template <int KP>
__global__ void __launch_bounds__(kThreadsR, 1) encode_tc_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                const EncParams p) {
  using G = Geo<KP>;
  constexpr int KE = G::KE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;
  uint8_t* sX = smem + G::OFF_X;
  uint8_t* sA = smem + G::OFF_A;
  float4* s_stats = reinterpret_cast<float4*>(smem + G::OFF_STATS);
  int* s_lo = reinterpret_cast<int*>(smem + G::OFF_LO);
  float* s_cst = reinterpret_cast<float*>(smem + G::OFF_CST);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  static_assert(G::XST <= 8, "X ring barriers");
  uint64_t* xfull = bars;         // [XST <= 8]
  uint64_t* xempty = bars + 8;    // [XST <= 8]
  uint64_t* afull = bars + 16;    // [2]
  uint64_t* aempty = bars + 18;   // [2]
  uint64_t* tfull = bars + 20;    // [2][2]: accumulator, column half
  uint64_t* tempty = bars + 24;   // [2][2]
  uint64_t* bload = bars + 28;
  uint32_t* s_tbase = reinterpret_cast<uint32_t*>(smem + G::OFF_TBASE);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = (int)blockIdx.x % p.m;
  const int t0 = (int)blockIdx.x / p.m;
  const int items = t0 < p.ntiles ? (p.ntiles - t0 + p.tstride - 1) / p.tstride : 0;
  const int ks = p.ks;

  if (tid == 0) {
    for (int i = 0; i < G::XST; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], kTrWarpsR);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], kTrWarpsR);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps / 2);
    }
    mbar_init(bload, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(s_tbase, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *s_tbase;

  // this subspace's operands and constants, once per CTA
  if (tid == 0) {
    const uint8_t* src = p.bprep + (size_t)m * G::B_BYTES;
    mbar_arrive_expect_tx(bload, (uint32_t)G::B_BYTES + CST_LEN * 4);
    for (uint32_t off = 0; off < (uint32_t)G::B_BYTES; off += 32768)
      bulk_g2s(sB + off, src + off, min(32768u, (uint32_t)G::B_BYTES - off), bload);
    bulk_g2s(s_cst, p.cst + (size_t)m * CST_LEN, CST_LEN * 4, bload);
  }
  mbar_wait(bload, 0);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint32_t xbytes = (uint32_t)(kRows * ks * 4);
      for (int w = 0; w < items; ++w) {
        const int t = t0 + w * p.tstride;
        const int xs = w % G::XST;
        mbar_wait(&xempty[xs], (uint32_t)(((w / G::XST) & 1) ^ 1));
        mbar_arrive_expect_tx(&xfull[xs], xbytes);
        uint8_t* dst = sX + xs * G::X_STAGE;
        if (KP == 64) {  // two 32-float swizzled boxes
          tma_load_2d(dst, &tmap, m * ks, t * kRows, &xfull[xs]);
          tma_load_2d(dst + kRows * 128, &tmap, m * ks + 32, t * kRows, &xfull[xs]);
        } else {
          tma_load_2d(dst, &tmap, m * ks, t * kRows, &xfull[xs]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // (one lane runs the loop: electing a lane per item with the whole warp waiting, as in
    // encode_tck_kernel, measured 1% slower here, the kernel being issue-bound)
    if (lane == 0) {
      // kMmaHalves: two N = 128 halves per accumulator, each released separately by the
      // epilogue (the next item's first half can run while the epilogue reads the second);
      // otherwise one N = 256 instruction per K step, both halves committed together
      constexpr int NH = kMmaHalves ? 2 : 1;
      const uint32_t idesc = tc::idesc_f16_f32(kRows, kN / NH);
      constexpr uint32_t sboE = (uint32_t)(KE / 8) * 128, sboP = (uint32_t)(KP / 8) * 128;
      const uint32_t b_hi0 = smem_u32(sB), b_lo0 = smem_u32(sB + G::B_HI);
      for (int w = 0; w < items; ++w) {
        const int ab = w & 1;
        const uint32_t ph = (uint32_t)((w >> 1) & 1);
        mbar_wait_spin(&afull[ab], ph);
        tc::fence_after();
        int lo_any = 0;
#pragma unroll
        for (int j = 0; j < kTrWarpsR; ++j) lo_any |= s_lo[ab * kTrWarpsR + j];
        const uint32_t a_hi = smem_u32(sA + ab * G::A_BYTES), a_lo = a_hi + G::A_HI;
#pragma unroll
        for (int hf = 0; hf < NH; ++hf) {
          mbar_wait_spin(&tempty[2 * ab + hf], ph ^ 1u);
          if (NH == 1) mbar_wait_spin(&tempty[2 * ab + 1], ph ^ 1u);
          tc::fence_after();
          const uint32_t tacc = tbase + (uint32_t)ab * kN + (uint32_t)hf * (kN / 2);
          const uint32_t b_hi = b_hi0 + (uint32_t)hf * 16u * sboE, b_lo = b_lo0 + (uint32_t)hf * 16u * sboP;
          // hi . lo, [lo . hi] first, while the accumulator is small (their truncation errors
          // scale with it, <= 2^-9 of the main terms), then hi . hi, then the |c|^2 / |x|^2
          // extension block last, so that the large extension terms enter in one instruction
#pragma unroll
          for (int s = 0; s < ((ENC_EXP & 4) ? 1 : KP / 16); ++s)
            tc::mma_f16(tacc, tc::smem_desc(a_hi + s * 256, 128, sboE), tc::smem_desc(b_lo + s * 256, 128, sboP), idesc,
                        s > 0 ? 1u : 0u);
          if (lo_any && !(ENC_EXP & 4)) {
#pragma unroll
            for (int s = 0; s < KP / 16; ++s)
              tc::mma_f16(tacc, tc::smem_desc(a_lo + s * 256, 128, sboP), tc::smem_desc(b_hi + s * 256, 128, sboE),
                          idesc, 1u);
          }
          if (!(ENC_EXP & 4)) {
#pragma unroll
            for (int s = 0; s < KP / 16; ++s)
              tc::mma_f16(tacc, tc::smem_desc(a_hi + s * 256, 128, sboE), tc::smem_desc(b_hi + s * 256, 128, sboE),
                          idesc, 1u);
            tc::mma_f16(tacc, tc::smem_desc(a_hi + (KP / 16) * 256, 128, sboE),
                        tc::smem_desc(b_hi + (KP / 16) * 256, 128, sboE), idesc, 1u);
          }
          tc::commit(&tfull[2 * ab + hf]);
          if (NH == 1) tc::commit(&tfull[2 * ab + 1]);
        }
        tc::commit(&aempty[ab]);
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ---------------- epilogue warps: whole rows of one accumulator ----------------
    const int ew = warp - 2;
    const int q = warp & 3;   // TMEM lane quadrant (warp % 4)
    const int e = ew >> 2;    // accumulator / item parity
    const int er = 32 * q + lane;
    // tensor-core accumulation model: an MMA instruction adds 16 products to the
    // accumulator with error <= 17 * 2^-23 * max(|addend|).  The lo passes run first: their
    // products and partial sums are bounded by P_L <= 2^-9 P as |lo| <= 2^-11 |hi| (plus
    // subnormal floors < 2^-24 (sqrt(KP) |s x| + S1c) P-units, far inside the 1e-3 term); the KP/16 hi . hi instructions then see
    // addends <= P + P_L; the extension instruction (7 nonzero addends) P + |c|^2 + |x|^2.
    // Total: 17 * 2^-23 * (KP/16) * (P + 3 P_L) <= 17 * (KP/16) * (1 + 3 * 2^-9) * 2^-23 * P,
    // whether or not the tile runs the lo . hi pass.
    const float eps_main2 = (float)(17 * KP / 16) * (1.0f + 3.0f / 512.0f) * 1.1920928955078125e-07f;
    const float eps_main3 = eps_main2;
    const float eps_ext = 7.0f * 1.1920928955078125e-07f;
    const float cb = s_cst[CST_CB], cnm = s_cst[CST_CN], s1c = s_cst[CST_S1C];
    for (int w = e; w < items; w += 2) {
      const int t = t0 + w * p.tstride;
      const uint32_t ph = (uint32_t)((w >> 1) & 1);
      mbar_wait(&tfull[2 * e], ph);
      tc::fence_after();
      const float4 st = s_stats[(w & 3) * kRows + er];  // x2u, |s x|, ok
      const uint32_t tacc = tbase + (uint32_t)e * kN + ((uint32_t)(32 * q) << 16);
      epilogue_row(p, m, (int64_t)t * kRows + er, tacc, &tfull[2 * e], &tempty[2 * e], ph, st, eps_main2, eps_main3,
                   eps_ext, cb, cnm, s1c, sqrtf((float)KP), lane);
    }
  } else {
    // ---------------- transform warps: one thread per row ----------------
    // 8-column groups streamed X (swizzled TMA tile) -> scaled fp16 hi / lo -> the UMMA
    // K-major A tiles (8 consecutive rows = one 128-byte core matrix per STS.128 phase);
    // |s x|^2 and the lo-nonzero flag accumulate in the row's own thread.
    const int tw = (warp - 2 - kEpiWarps) % kTrWarpsR;
    const int tset = (warp - 2 - kEpiWarps) / kTrWarpsR;  // items tset, tset + kTrSets, ...
    const int r = 32 * tw + lane;
    constexpr int NG = KP / 8;
    const float sc = s_cst[CST_S];
    const __half acn = __float2half_rn(s_cst[CST_ACN]);
    const bool valid = s_cst[CST_VALID] != 0.f;
    const uint32_t aoff_hi = tc::kmajor_off(r, 0, KE), aoff_lo = (uint32_t)G::A_HI + tc::kmajor_off(r, 0, KP);
    for (int w = tset; w < items; w += kTrSets) {
      const int ab = w & 1, xs = w % G::XST;
      // several sets: A buffer first (MMA(w - 2) done implies every earlier item was
      // transformed, so this set is never two phases ahead of the X ring, where a parity wait
      // would pass on stale data); one set: X first, its loads fly while the A buffer drains
      if (kTrSets > 1) mbar_wait(&aempty[ab], (uint32_t)(((w >> 1) & 1) ^ 1));
      mbar_wait(&xfull[xs], (uint32_t)((w / G::XST) & 1));
      const uint8_t* xb = sX + xs * G::X_STAGE;
      uint8_t* ahi = sA + ab * G::A_BYTES + aoff_hi;
      uint8_t* alo = sA + ab * G::A_BYTES + aoff_lo;
      float acc0 = 0.f, acc1 = 0.f;
      uint32_t lr = 0;
      // batches of up to 4 groups (32 floats): every load of a batch is issued before its
      // first A store (the stores could alias the loads for the compiler, which would
      // otherwise expose one shared-memory round trip per group)
      constexpr int GB = NG < 4 ? NG : 4;
      if (ENC_EXP & 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[xs]);
        if (kTrSets == 1) mbar_wait(&aempty[ab], (uint32_t)(((w >> 1) & 1) ^ 1));
      }
#pragma unroll
      for (int g0 = 0; g0 < ((ENC_EXP & 1) ? 0 : NG); g0 += GB) {
        float4 f[2 * GB];
#pragma unroll
        for (int i = 0; i < 2 * GB; ++i) {
          const int g = g0 + i / 2, h = i & 1;
          f[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (G::SWZ) {
            // 128-byte rows of 8 x 16-byte chunks, chunk index XOR (row % 8); KP = 64: two halves
            const int chunk = 2 * g + h, half = chunk >> 3, ch = chunk & 7;
            f[i] = *reinterpret_cast<const float4*>(xb + half * (kRows * 128) + r * 128 + ((ch ^ (r & 7)) << 4));
          } else if (8 * g < ks) {  // dsub = 8 < KP = 16: the upper group is zero padding
            f[i] = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xb) + r * ks + 8 * g + 4 * h);
          }
        }
        if (kTrSets == 1 && g0 == 0) mbar_wait(&aempty[ab], (uint32_t)(((w >> 1) & 1) ^ 1));
#pragma unroll
        for (int gg = 0; gg < GB; ++gg) {
          const int g = g0 + gg;
          const float v[8] = {f[2 * gg].x,     f[2 * gg].y,     f[2 * gg].z,     f[2 * gg].w,
                              f[2 * gg + 1].x, f[2 * gg + 1].y, f[2 * gg + 1].z, f[2 * gg + 1].w};
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float a0 = v[2 * j] * sc, a1 = v[2 * j + 1] * sc;
            const __half2 hh = __floats2half2_rn(a0, a1);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(a0 - hf.x, a1 - hf.y);
            hw[j] = *reinterpret_cast<const uint32_t*>(&hh);
            lw[j] = *reinterpret_cast<const uint32_t*>(&ll);
            acc0 = fmaf(a0, a0, acc0);
            acc1 = fmaf(a1, a1, acc1);
          }
          lr |= (lw[0] | lw[1]) | (lw[2] | lw[3]);
          *reinterpret_cast<uint4*>(ahi + g * 128) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          *reinterpret_cast<uint4*>(alo + g * 128) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
      }
      // the X stage is released only after the loaded values were used: releasing it right
      // after the loads were issued (before the A-buffer wait) produced wrong codes in the
      // items that follow a CTA's start (tools/diag_encode_mismatch.py)
      __syncwarp();
      if (lane == 0) mbar_arrive(&xempty[xs]);
      lr &= 0x7fff7fffu;  // -0 lo parts are zeros
      const unsigned bal = __ballot_sync(0xffffffffu, lr != 0u);
      // |s x|^2 rounded up (fp32 sum of KP products: relative error < (KP+4) 2^-24).  Rows
      // with NaN / inf / out-of-range values are not certified (stats .z = 0); their A rows
      // only reach their own accumulator row.
      const float x2u = (acc0 + acc1) * (1.0f + (float)(KP + 8) * 5.9604644775390625e-08f);
      const bool ok = valid && (x2u < kX2Limit);
      // extension columns: [acn x3, |s x|^2 parts (x 2^15), 2^15 (padding codewords), 0...]
      const float xv = ok ? x2u * 3.0517578125e-05f : 0.f;  // 2^-15, exact
      const __half x_h = __float2half_rn(xv);
      const float r1 = xv - __half2float(x_h);
      const __half x_m = __float2half_rn(r1);
      const __half x_l = __float2half_rn(r1 - __half2float(x_m));
      const __half p15 = __float2half_rn(32768.f);
      const __half z = __float2half_rn(0.f);
      *reinterpret_cast<uint4*>(ahi + NG * 128) =
          make_uint4(pack_h2(acn, acn), pack_h2(acn, x_h), pack_h2(x_m, x_l), pack_h2(p15, z));
      *reinterpret_cast<uint4*>(ahi + (NG + 1) * 128) = make_uint4(0u, 0u, 0u, 0u);
      // |s x| rounded up: sqrt.approx has relative error < 2^-21
      float xn;
      asm("sqrt.approx.f32 %0, %1;" : "=f"(xn) : "f"(x2u));
      // 4 stats buffers: transform(w + 4) waits for MMA(w + 2), which waits for every
      // epilogue warp of parity w to have read item w's stats
      s_stats[(w & 3) * kRows + r] = make_float4(x2u, xn * 1.000002f, ok ? 1.f : 0.f, lr ? 1.f : 0.f);
      if (lane == 0) s_lo[ab * kTrWarpsR + tw] = (bal != 0);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tbase, 512);
  }
}

// Codebook preparation: one block of 256 threads (one per codeword slot) per subspace.
// B = -2 s c split into fp16 hi/lo (K-major, zero-padded to KP), extension row
// [cn parts, 2^15 x3, padding, 0...] with cn = s^2 |c|^2 / acn in three fp16 parts, and
// the constants of the epilogue's error bound.
template <int KP>
__global__ void __launch_bounds__(256) encode_prep_kernel(const float* __restrict__ cw, int m, int l, int ks,
                                                         uint8_t* __restrict__ bprep, float* __restrict__ cst) {
  using G = Geo<KP>;
  constexpr int KE = G::KE;
  __shared__ float red[8];
  __shared__ int bad[8];
  __shared__ double redd[8];
  __shared__ float s_sc;
  __shared__ int s_bad;
  __shared__ double s_cn;
  const int mm = blockIdx.x, row = threadIdx.x, lane = row & 31, warp = row >> 5;
  const bool real = row < l;
  const float* c = cw + ((size_t)mm * l + (real ? row : 0)) * ks;
  float amax = 0.f;
  int nonfinite = 0;
  if (real)
    for (int k = 0; k < ks; ++k) {
      const float a = fabsf(c[k]);
      nonfinite |= !(a <= 3.4028234663852886e38f);
      amax = fmaxf(amax, a);
    }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o);
  }
  if (lane == 0) {
    red[warp] = amax;
    bad[warp] = nonfinite;
  }
  __syncthreads();
  if (row == 0) {
    float a = 0.f;
    int b = 0;
    for (int i = 0; i < 8; ++i) {
      a = fmaxf(a, red[i]);
      b |= bad[i];
    }
    int ex = 0;
    if (a > 0.f && !b) frexpf(a, &ex);  // a in [2^(ex-1), 2^ex)
    // |s c| < 2^8: vectors up to ~2^8 x the codebook's range stay inside the fp16
    // operand and |s x|^2 < 2^30 extension ranges (others take the exact path)
    s_sc = (a > 0.f && !b) ? ldexpf(1.0f, 8 - ex) : 1.0f;
    s_bad = b;
  }
  __syncthreads();
  const float sc = s_sc;
  const bool cb_ok = !s_bad;
  uint8_t* bh = bprep + (size_t)mm * G::B_BYTES;
  uint8_t* bl = bh + G::B_HI;
  double cn = 0.0, nb2 = 0.0, s1 = 0.0;
  for (int k = 0; k < KP; ++k) {
    const float cv = (real && cb_ok && k < ks) ? c[k] * sc : 0.f;  // exact (power-of-two scale)
    const float bv = -2.0f * cv;
    const __half hi = __float2half_rn(bv);
    const __half lo = __float2half_rn(bv - __half2float(hi));
    *reinterpret_cast<__half*>(bh + tc::kmajor_off(row, k, KE)) = hi;
    *reinterpret_cast<__half*>(bl + tc::kmajor_off(row, k, KP)) = lo;
    cn += (double)cv * (double)cv;
    nb2 += (double)bv * (double)bv;
    s1 += fabs((double)bv);
  }
  // block maximum of cn -> acn = 2^a with cn / acn < 2^15 (cn < KP 2^16 <= 2^22: a <= 8)
  double cmx = cn;
  for (int o = 16; o > 0; o >>= 1) cmx = fmax(cmx, __shfl_xor_sync(0xffffffffu, cmx, o));
  if (lane == 0) redd[warp] = cmx;
  __syncthreads();
  if (row == 0) {
    double a = 0.0;
    for (int i = 0; i < 8; ++i) a = fmax(a, redd[i]);
    s_cn = a;
  }
  __syncthreads();
  int ea = 0;
  if (s_cn >= 16384.0) {
    frexp(s_cn, &ea);  // s_cn < 2^ea
    ea -= 14;          // s_cn / 2^ea < 2^14
  }
  const double acn = ldexp(1.0, ea);
  const double cv = cn / acn;
  const __half c_h = __double2half(cv);
  const double r1 = cv - (double)__half2float(c_h);
  const __half c_m = __double2half(r1);
  const __half c_l = __double2half(r1 - (double)__half2float(c_m));
  const __half p15 = __float2half_rn(32768.f);
  const __half pad = __float2half_rn(real ? 0.f : 65504.f);
  const __half z = __float2half_rn(0.f);
  *reinterpret_cast<uint4*>(bh + tc::kmajor_off(row, KP, KE)) =
      make_uint4(pack_h2(c_h, c_m), pack_h2(c_l, p15), pack_h2(p15, p15), pack_h2(pad, z));
  *reinterpret_cast<uint4*>(bh + tc::kmajor_off(row, KP + 8, KE)) = make_uint4(0u, 0u, 0u, 0u);
  // block maxima of |B_j|, cn_j, sum |B_j| over real rows
  float vb = real ? (float)sqrt(nb2) : 0.f, vc = real ? (float)cn : 0.f, v1 = real ? (float)s1 : 0.f;
  for (int o = 16; o > 0; o >>= 1) {
    vb = fmaxf(vb, __shfl_xor_sync(0xffffffffu, vb, o));
    vc = fmaxf(vc, __shfl_xor_sync(0xffffffffu, vc, o));
    v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, o));
  }
  __shared__ float rb[8], rc[8], r1s[8];
  if (lane == 0) {
    rb[warp] = vb;
    rc[warp] = vc;
    r1s[warp] = v1;
  }
  __syncthreads();
  if (row == 0) {
    float a = 0.f, b2 = 0.f, d = 0.f;
    for (int i = 0; i < 8; ++i) {
      a = fmaxf(a, rb[i]);
      b2 = fmaxf(b2, rc[i]);
      d = fmaxf(d, r1s[i]);
    }
    float* o = cst + (size_t)mm * CST_LEN;
    o[CST_S] = sc;
    o[CST_ACN] = (float)acn;
    o[CST_CB] = a * 1.0001f;
    o[CST_CN] = b2 * 1.0001f;
    o[CST_S1C] = d * 1.0001f;
    o[CST_VALID] = cb_ok ? 1.f : 0.f;
    o[6] = 0.f;
    o[7] = 0.f;
  }
}

// Exact float64 decision for the (row, subspace) pairs the certificate did not cover.
// Block (x, m) holds subspace m's codebook in shared memory (row stride ks + 1: lanes
// reading different codewords hit different banks); one warp per flagged row, each
// lane owning codewords lane, lane + 32, ...; float64 (x - c)^2 summed sequentially
// without FMA (scipy cdist order), np.argmin order (first NaN, else lowest index).
__global__ void __launch_bounds__(256) encode_exact_kernel(const float* __restrict__ x, int64_t n, int d,
                                                          const float* __restrict__ cw, int m, int l, int ks,
                                                          const uint32_t* __restrict__ flags,
                                                          const unsigned int* __restrict__ counters, uint32_t flag_cap,
                                                          uint8_t* __restrict__ codes, int stride) {
  extern __shared__ float s_cb[];
  const int mm = blockIdx.y;
  const bool all = counters[1] != 0;
  const int64_t total = all ? n : (int64_t)min(counters[2 + mm], flag_cap);
  if (total == 0 || (int64_t)blockIdx.x * 8 >= total) return;
  const int sp = ks + 1;
  const float* cb = cw + (size_t)mm * l * ks;
  for (int i0 = threadIdx.x; i0 < l * ks; i0 += 8 * blockDim.x) {  // 8 loads in flight per thread
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < l * ks ? __ldg(cb + i) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < l * ks) s_cb[(i / ks) * sp + (i % ks)] = v[u];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < total; i += (int64_t)gridDim.x * 8) {
    const int64_t row = all ? i : (int64_t)flags[(size_t)mm * flag_cap + i];
    const float* xv = x + row * d + (size_t)mm * ks;
    const float x0 = lane < ks ? xv[lane] : 0.f, x1 = lane + 32 < ks ? xv[lane + 32] : 0.f;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    // codewords c >= l alias codeword l - 1 (same distance, larger index: never chosen)
    int cbase[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) cbase[u] = min(lane + 32 * u, l - 1) * sp;
    for (int k = 0; k < ks; ++k) {
      const double xk = (double)__shfl_sync(0xffffffffu, k < 32 ? x0 : x1, k & 31);
      double df[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) df[u] = __dsub_rn(xk, (double)s_cb[cbase[u] + k]);
#pragma unroll
      for (int u = 0; u < 8; ++u) df[u] = __dmul_rn(df[u], df[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = __dadd_rn(acc[u], df[u]);
    }
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bl = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = lane + 32 * u;
      if (argmin_less(acc[u], c, best, bl)) {
        best = acc[u];
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

// ===========================================================================
// K-streamed variant for long subspaces (dsub = ks a multiple of 32 in [96, 1024], e.g.
// BASELINE config 3's 512-D subspaces).  The codebook operands no longer fit in shared
// memory, so each 128-vector item streams K in 32-column chunks: X chunk by TMA (128-byte
// swizzle), B chunk (hi + lo, 32 KB) by a bulk copy from the prepared global layout, A
// chunk by the transform warps; every chunk's MMAs accumulate into the item's TMEM
// accumulator, the |c|^2 / |x|^2 extension block follows the last chunk.  Epilogue,
// certificate and fallback are the same as encode_tc_kernel's (epilogue_row), with the
// accumulation bound scaled by the instruction count (ks / 16 per pass).
// ===========================================================================
// timing-experiment switches of the K-streamed kernel (results are wrong when set):
// 1 = B chunks copied only for the first ring round, 2 = hi . hi pass only, 4 = no transform
// arithmetic / stores, 8 = no epilogue, 16 = X tiles loaded only for the first ring round
#ifndef ENC_KEXP
#define ENC_KEXP 0
#endif
constexpr int kKC = 32;
constexpr int kMaxChunks = 32;  // ks <= 1024
#ifndef ENC_KXST
#define ENC_KXST 3
#endif
#ifndef ENC_KBST
#define ENC_KBST 3
#endif
#ifndef ENC_KAST
#define ENC_KAST 2
#endif
#ifndef ENC_KTRG
#define ENC_KTRG 2
#endif
#ifndef ENC_KSPIN
#define ENC_KSPIN 0
#endif
constexpr int kXSt = ENC_KXST, kBSt = ENC_KBST, kASt = ENC_KAST;  // ring depths: X tiles, B chunks, A chunks
constexpr int kTrGroups = ENC_KTRG;                         // transform groups taking chunks in turn
constexpr int kTrGroupWarps = kTrWarps / kTrGroups;         // warps per group
constexpr int kTrPasses = kRows / (8 * kTrGroupWarps);      // 8-row passes per warp and chunk
static_assert(kTrGroups == 1 || kTrGroups == 2, "transform groups");
// the CTA pair variant's ring depths (half the B bytes per CTA leave room for deeper rings)
#ifndef ENC_KPXST
#define ENC_KPXST 4
#endif
#ifndef ENC_KPBST
#define ENC_KPBST 5
#endif
#ifndef ENC_KPAST
#define ENC_KPAST 2
#endif
#ifndef ENC_KPSEM
#define ENC_KPSEM 1
#endif

// kPair: the CTA pair variant (cta_group::2): each CTA of a 2-CTA cluster keeps 128 of the
// 256 codewords of every B chunk (half the B bytes written to and read from its shared
// memory, the kernel's limiting resource) and its own 128-row tile of X / A.
template <bool kPair>
struct GeoK {
  static constexpr int NB = kPair ? kN / 2 : kN;      // codewords held per CTA
  static constexpr int XST = kPair ? ENC_KPXST : kXSt;  // ring depths: X tiles, B chunks, A chunks
  static constexpr int BST = kPair ? ENC_KPBST : kBSt;
  static constexpr int AST = kPair ? ENC_KPAST : kASt;
  static_assert(2 * XST + 3 * BST + 2 * AST + 13 <= 48, "mbarrier slots");
  static constexpr int X_STAGE = kRows * kKC * 4;     // 16 KB (1024-aligned, swizzled)
  static constexpr int B_HI = NB * kKC * 2;           // 16 KB (pair: 8 KB)
  static constexpr int B_CHUNK = 2 * B_HI;            // hi + lo
  static constexpr int B_EXT = NB * kExt * 2;         // 8 KB (pair: 4 KB)
  static constexpr int GB_HI = kN * kKC * 2;          // prepared operands in global memory: all 256 codewords
  static constexpr int GB_CHUNK = 2 * GB_HI;
  static constexpr int GB_EXT = kN * kExt * 2;
  static constexpr int A_HI = kRows * kKC * 2;        // 8 KB
  static constexpr int A_CHUNK = 2 * A_HI;
  static constexpr int A_EXT = kRows * kExt * 2;      // 4 KB
  static constexpr int OFF_BEXT = 0;
  static constexpr int OFF_X = B_EXT;
  static constexpr int OFF_B = OFF_X + XST * X_STAGE;
  static constexpr int OFF_A = OFF_B + BST * B_CHUNK;
  static constexpr int OFF_AEXT = OFF_A + AST * A_CHUNK;
  static constexpr int OFF_STATS = OFF_AEXT + A_EXT;          // one extension buffer (see the transform warps)
  static constexpr int OFF_EX = OFF_STATS + 2 * kRows * 16;   // float4 [2][kRows] row stats
  static constexpr int OFF_PART = OFF_EX + kRows * kExWords * 4;  // (epilogue warp pairs' hand-over rows)
  static constexpr int OFF_LO = OFF_PART + 2 * kRows * 8;         // float2 [2][kRows]: group 1's row partials
  static constexpr int OFF_CST = OFF_LO + AST * kTrWarps * 4;
  static constexpr int OFF_BCH = OFF_CST + CST_LEN * 4;   // float [kMaxChunks]
  static constexpr int OFF_BAR = OFF_BCH + kMaxChunks * 4;  // uint64 [48]
  static constexpr int OFF_TBASE = OFF_BAR + 48 * 8;
  static constexpr int SMEM = OFF_TBASE + 16 + 1024;
  __host__ __device__ static size_t bprep_bytes(int ks) { return (size_t)(ks / kKC) * GB_CHUNK + GB_EXT; }
};

template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1) encode_tck_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                const EncParams p) {
  using G = GeoK<kPair>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sBext = smem + G::OFF_BEXT;
  uint8_t* sX = smem + G::OFF_X;
  uint8_t* sB = smem + G::OFF_B;
  uint8_t* sA = smem + G::OFF_A;
  uint8_t* sAext = smem + G::OFF_AEXT;
  float4* s_stats = reinterpret_cast<float4*>(smem + G::OFF_STATS);
  uint32_t* s_ex = reinterpret_cast<uint32_t*>(smem + G::OFF_EX);
  float2* s_part = reinterpret_cast<float2*>(smem + G::OFF_PART);
  int* s_lo = reinterpret_cast<int*>(smem + G::OFF_LO);
  float* s_cst = reinterpret_cast<float*>(smem + G::OFF_CST);
  float* s_bch = reinterpret_cast<float*>(smem + G::OFF_BCH);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* xfull = bars;                 // [G::XST]
  uint64_t* xempty = xfull + G::XST;        // [G::XST]
  uint64_t* bfull = xempty + G::XST;        // [G::BST]
  uint64_t* bempty = bfull + G::BST;        // [G::BST]
  uint64_t* afull = bempty + G::BST;        // [G::AST]
  uint64_t* aempty = afull + G::AST;        // [G::AST]
  uint64_t* aefull = aempty + G::AST;       // [2] extension rows of A
  uint64_t* aeempty = aefull + 2;         // [2]
  uint64_t* tfull = aeempty + 2;          // [2][2]
  uint64_t* tempty = tfull + 4;           // [2][2]
  uint64_t* bload = tempty + 4;
  uint64_t* bpeer = bload + 1;            // [G::BST] pair: the peer CTA's half of a B chunk has landed
  uint32_t* s_tbase = reinterpret_cast<uint32_t*>(smem + G::OFF_TBASE);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // pair: the two CTAs of a cluster take the two 128-row tiles of a tile pair of one subspace;
  // tstride counts tile pairs, both CTAs run the same number of items (a missing last tile
  // loads zeros past the end of X and stores nothing)
  const int cr = kPair ? (int)tc::cluster_rank() : 0;
  const int gid = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int m = gid % p.m;
  const int t0 = gid / p.m;
  const int ntl = kPair ? (p.ntiles + 1) >> 1 : p.ntiles;
  const int items = t0 < ntl ? (ntl - t0 + p.tstride - 1) / p.tstride : 0;
  const int nsig = kPair ? 2 : 1;  // CTAs signalling the issuer's barriers
  const int ks = p.ks, nk = ks / kKC;
  const uint8_t* bprep = p.bprep + (size_t)m * G::bprep_bytes(ks);

  if (tid == 0) {
    for (int i = 0; i < G::XST; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], kTrGroupWarps);
    }
    for (int i = 0; i < G::BST; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
      mbar_init(&bpeer[i], 1);
    }
    for (int i = 0; i < G::AST; ++i) {
      mbar_init(&afull[i], nsig * kTrGroupWarps);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&aefull[i], nsig * kTrGroupWarps);
      mbar_init(&aeempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], nsig * kEpiWarps);
    }
    mbar_init(bload, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if (kPair) tc::tmem_alloc_pair(s_tbase, 512);
    else tc::tmem_alloc(s_tbase, 512);
  }
  tc::fence_before();
  __syncthreads();
  if (kPair) tc::cluster_sync();  // both CTAs' barriers initialised before any remote arrive / multicast commit
  tc::fence_after();
  const uint32_t tbase = *s_tbase;
  if (tid == 0) {
    mbar_arrive_expect_tx(bload, (uint32_t)G::B_EXT + CST_LEN * 4 + kMaxChunks * 4);
    bulk_g2s(sBext, bprep + (size_t)nk * G::GB_CHUNK + (size_t)cr * G::B_EXT, G::B_EXT, bload);
    bulk_g2s(s_cst, p.cst + (size_t)m * CST_LEN, CST_LEN * 4, bload);
    bulk_g2s(s_bch, p.bch + (size_t)m * kMaxChunks, kMaxChunks * 4, bload);
  }
  mbar_wait(bload, 0);
  const int nchunks = items * nk;

  if (warp == 0) {
    // ---------------- producer: X chunks (TMA) and B chunks (bulk copies) ----------------
    // One lane polls both rings, so that the X tiles run ahead by the whole X ring (through
    // an item's epilogue) whatever the state of the B ring.
    if (lane == 0) {
      int gx = 0, gb = 0;
      while (gx < nchunks || gb < nchunks) {
        bool did = false;
        if (gx < nchunks) {
          const int xs = gx % G::XST;
          if (mbar_test(&xempty[xs], (uint32_t)(((gx / G::XST) & 1) ^ 1))) {
            const int w = gx / nk, c = gx - w * nk;
            const int t = kPair ? 2 * (t0 + w * p.tstride) + cr : t0 + w * p.tstride;
            if ((ENC_KEXP & 16) && gx >= G::XST) {
              mbar_arrive(&xfull[xs]);
            } else {
              mbar_arrive_expect_tx(&xfull[xs], (uint32_t)G::X_STAGE);
              tma_load_2d(sX + xs * G::X_STAGE, &tmap, m * ks + c * kKC, t * kRows, &xfull[xs]);
            }
            ++gx;
            did = true;
          }
        }
        if (gb < nchunks) {
          const int bs = gb % G::BST;
          if (mbar_test(&bempty[bs], (uint32_t)(((gb / G::BST) & 1) ^ 1))) {
            const int c = gb % nk;
            if ((ENC_KEXP & 1) && gb >= G::BST) {
              mbar_arrive(&bfull[bs]);
            } else {
              mbar_arrive_expect_tx(&bfull[bs], (uint32_t)G::B_CHUNK);
              if (kPair) {  // this CTA's 128 codewords of the hi and of the lo block
                const uint8_t* src = bprep + (size_t)c * G::GB_CHUNK + (size_t)cr * G::B_HI;
                bulk_g2s(sB + bs * G::B_CHUNK, src, G::B_HI, &bfull[bs]);
                bulk_g2s(sB + bs * G::B_CHUNK + G::B_HI, src + G::GB_HI, G::B_HI, &bfull[bs]);
              } else {
                bulk_g2s(sB + bs * G::B_CHUNK, bprep + (size_t)c * G::GB_CHUNK, G::B_CHUNK, &bfull[bs]);
              }
            }
            ++gb;
            did = true;
          }
        }
        if (!did) __nanosleep(32);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // One item in flight: accumulator H = TMEM columns [0, 256) takes hi . hi and the
    // extension block, L = [256, 512) the lo passes, so that the lo passes' truncation
    // errors scale with L's small magnitude, and H's with its running prefix.
    if (kPair && cr == 1) {
      // the peer CTA issues nothing: this lane reports each landed B half to rank 0
      if (lane == 0) {
        for (int g = 0; g < nchunks; ++g) {
          const int bs = g % G::BST;
          mbar_wait(&bfull[bs], (uint32_t)((g / G::BST) & 1));
          tc::mbar_arrive_rank0(&bpeer[bs]);
        }
      }
    } else {
      // The whole warp runs the loop and one elected lane issues: inside a lane == 0 branch
      // ptxas wraps every tcgen05 instruction (uniform-register operands) in a loop over the
      // active lanes, ~140 dependent instructions per chunk on the issuing thread
      auto mma = [](uint32_t d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
        if (kPair) tc::mma_f16_pair(d, da, db, id, acc);
        else tc::mma_f16(d, da, db, id, acc);
      };
      auto commit = [](uint64_t* bar) {
        if (kPair) tc::commit_pair(bar);
        else tc::commit(bar);
      };
      auto wait = [](uint64_t* bar, uint32_t par) {
        if (kPair) tc::mbar_wait_spin_cluster(bar, par);
        else mbar_wait_spin(bar, par);
      };
      const uint32_t idesc = tc::idesc_f16_f32(kPair ? 2 * kRows : kRows, kN);
      constexpr uint32_t sboC = (uint32_t)(kKC / 8) * 128, sboE = (uint32_t)(kExt / 8) * 128;
      const uint32_t tH = tbase, tL = tbase + (uint32_t)kN;
      for (int w = 0; w < items; ++w) {
        const uint32_t ph = (uint32_t)(w & 1);
        wait(&tempty[0], ph ^ 1u);
        wait(&tempty[1], ph ^ 1u);
        for (int c = 0; c < nk; ++c) {
          const int g = w * nk + c;
          const int as = g % G::AST, bs = g % G::BST;
          wait(&afull[as], (uint32_t)((g / G::AST) & 1));
          mbar_wait_spin(&bfull[bs], (uint32_t)((g / G::BST) & 1));
          if (kPair) wait(&bpeer[bs], (uint32_t)((g / G::BST) & 1));
          tc::fence_after();
          int lo_any = kPair ? 1 : 0;  // pair: the lo . hi pass always runs (no flags from the peer CTA)
#pragma unroll
          for (int j = 0; j < kTrGroupWarps; ++j) lo_any |= s_lo[as * kTrWarps + j];
          if (elect_one()) {
          const uint32_t a_hi = smem_u32(sA + as * G::A_CHUNK), a_lo = a_hi + G::A_HI;
          const uint32_t b_hi = smem_u32(sB + bs * G::B_CHUNK), b_lo = b_hi + G::B_HI;
#pragma unroll
          for (int s = 0; s < ((ENC_KEXP & 2) ? (c == 0 ? 1 : 0) : kKC / 16); ++s)
            mma(tL, tc::smem_desc(a_hi + s * 256, 128, sboC), tc::smem_desc(b_lo + s * 256, 128, sboC), idesc,
                (c > 0 || s > 0) ? 1u : 0u);
          if (lo_any && !(ENC_KEXP & 2)) {
#pragma unroll
            for (int s = 0; s < kKC / 16; ++s)
              mma(tL, tc::smem_desc(a_lo + s * 256, 128, sboC), tc::smem_desc(b_hi + s * 256, 128, sboC), idesc, 1u);
          }
#pragma unroll
          for (int s = 0; s < kKC / 16; ++s)
            mma(tH, tc::smem_desc(a_hi + s * 256, 128, sboC), tc::smem_desc(b_hi + s * 256, 128, sboC), idesc,
                (c > 0 || s > 0) ? 1u : 0u);
          commit(&aempty[as]);
          commit(&bempty[bs]);
          }
          __syncwarp();
        }
        wait(&aefull[0], ph);
        tc::fence_after();
        if (elect_one()) {
          mma(tH, tc::smem_desc(smem_u32(sAext), 128, sboE), tc::smem_desc(smem_u32(sBext), 128, sboE), idesc, 1u);
          commit(&aeempty[0]);
          commit(&tfull[0]);
          commit(&tfull[1]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ---------------- epilogue warps: two per TMEM lane quadrant (128 codewords each) ----------------
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    const int er = 32 * q + lane;
    // H: two hi . hi instructions per chunk with max |addend| <= the row's running prefix
    // (sum W over chunks, st.w); L: 4 nk instructions with addends <= 2^-9 P
    // (|lo| <= 2^-11 |hi|); the H + L addition rounds once (2^-24, folded into eps_ext)
    const float eps_h = 2.0f * 17.0f * (1.0f + 3.0f / 512.0f) * 1.1920928955078125e-07f;
    const float eps_l = (float)(4 * 17 * nk) * (1.0f / 512.0f) * 1.1920928955078125e-07f;
    const float eps_ext = 7.5f * 1.1920928955078125e-07f;
    const float cb = s_cst[CST_CB], cnm = s_cst[CST_CN], s1c = s_cst[CST_S1C];
    const float sqrt_ks = sqrtf((float)ks);
    for (int w = 0; w < items; ++w) {
      const int t = kPair ? 2 * (t0 + w * p.tstride) + cr : t0 + w * p.tstride;
      mbar_wait(&tfull[0], (uint32_t)(w & 1));
      tc::fence_after();
      const float4 st = s_stats[(w & 1) * kRows + er];
      const uint32_t tacc = tbase + ((uint32_t)(32 * q) << 16);
      if (ENC_KEXP & 8) {
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          arrive_at_issuer<kPair>(&tempty[0]);
          arrive_at_issuer<kPair>(&tempty[1]);
        }
        if (st.x == 123.456f) p.codes[((int64_t)t * kRows + er) * p.stride + m] = 0;
        continue;
      }
      epilogue_row_split<kPair>(p, m, (int64_t)t * kRows + er, tacc, tempty, st, eps_h, eps_l, eps_ext, cb, cnm, s1c, sqrt_ks,
                         lane, half, s_ex + er * kExWords, 1 + q);
    }
  } else {
    // ---------------- transform warps ----------------
    // kTrGroups groups of kTrGroupWarps warps take the chunks in turn, kTrPasses passes of 8
    // rows per warp (8 columns per lane).  With two groups a chunk's chain (X tile ->
    // registers -> fp16 split -> wait for the A stage -> stores -> proxy fence) may take two
    // chunk times, and each lane carries four independent rows through it.
    const int tw = warp - 2 - kEpiWarps;
    const int grp = tw / kTrGroupWarps, twg = tw % kTrGroupWarps;
    if constexpr (kTrGroups == 2) {
      // one lane per row (32 rows per warp, 4 warps per chunk, the two groups alternate over
      // the chunks): no cross-lane sums, eight independent 16-byte column groups per lane
      const int r = 32 * twg + lane;
      const float sc = s_cst[CST_S];
      const __half acn = __float2half_rn(s_cst[CST_ACN]);
      const bool valid = s_cst[CST_VALID] != 0.f;
      const uint32_t arow = (uint32_t)((r >> 3) * (kKC / 8) * 128 + (r & 7) * 16);  // kmajor_off(r, 0, kKC)
      int g = grp;
      for (int w = 0; w < items; ++w) {
        float x2 = 0.f, wsum = 0.f;
        const int gend = (w + 1) * nk;
        for (; g < gend; g += 2) {
          const int c = g - w * nk;
          const int xs = g % G::XST, as = g % G::AST;
          const uint32_t aph = (uint32_t)((g / G::AST) & 1);
          mbar_wait(&xfull[xs], (uint32_t)((g / G::XST) & 1));
          const uint8_t* xb = sX + xs * G::X_STAGE + r * 128;
          uint32_t hw[16], lw[16];
          uint32_t lo_nz = 0;
          float ec = 0.f;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const float4 f = *reinterpret_cast<const float4*>(xb + ((ch ^ (r & 7)) << 4));
            const float a0 = f.x * sc, a1 = f.y * sc, a2 = f.z * sc, a3 = f.w * sc;
            const __half2 h01 = __floats2half2_rn(a0, a1), h23 = __floats2half2_rn(a2, a3);
            const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
            const __half2 l01 = __floats2half2_rn(a0 - f01.x, a1 - f01.y);
            const __half2 l23 = __floats2half2_rn(a2 - f23.x, a3 - f23.y);
            hw[2 * ch] = *reinterpret_cast<const uint32_t*>(&h01);
            hw[2 * ch + 1] = *reinterpret_cast<const uint32_t*>(&h23);
            lw[2 * ch] = *reinterpret_cast<const uint32_t*>(&l01);
            lw[2 * ch + 1] = *reinterpret_cast<const uint32_t*>(&l23);
            lo_nz |= lw[2 * ch] | lw[2 * ch + 1];
            ec = fmaf(a0, a0, fmaf(a1, a1, fmaf(a2, a2, fmaf(a3, a3, ec))));
          }
          x2 += ec;
          // the row's chunk norm rounded up, times max_j |B_j,c|, counted for the nk - c prefixes holding it
          wsum = fmaf(sqrtf(ec), (float)(nk - c) * s_bch[c] * 1.000001f, wsum);
          const unsigned bal = __ballot_sync(0xffffffffu, (lo_nz & 0x7fff7fffu) != 0);
          // released after the loaded values were consumed (see encode_tc_kernel's transform)
          if (lane == 0) mbar_arrive(&xempty[xs]);
          if (ENC_KSPIN) mbar_wait_spin(&aempty[as], aph ^ 1u);
          else mbar_wait(&aempty[as], aph ^ 1u);
          uint8_t* ahi = sA + as * G::A_CHUNK + arow;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            *reinterpret_cast<uint4*>(ahi + j * 128) = make_uint4(hw[4 * j], hw[4 * j + 1], hw[4 * j + 2], hw[4 * j + 3]);
            *reinterpret_cast<uint4*>(ahi + G::A_HI + j * 128) =
                make_uint4(lw[4 * j], lw[4 * j + 1], lw[4 * j + 2], lw[4 * j + 3]);
          }
          if (lane == 0) s_lo[as * kTrWarps + twg] = (bal != 0);
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) arrive_at_issuer<kPair>(&afull[as]);
        }
        // group 1 hands its row partials to group 0, which writes the extension rows and stats
        if (grp == 1) s_part[(w & 1) * kRows + r] = make_float2(x2, wsum);
        asm volatile("bar.sync 5, %0;" ::"n"(kTrWarps * 32) : "memory");
        if (grp == 1) continue;
        mbar_wait(&aeempty[0], (uint32_t)((w & 1) ^ 1));
        {
          const float2 o = s_part[(w & 1) * kRows + r];
          const float acc = x2 + o.x;
          // |s x|^2 rounded up: fp32 sums of ks products (relative error < (ks + 4) 2^-24)
          const float x2u = acc * (1.0f + (float)(ks + 16) * 5.9604644775390625e-08f);
          const bool ok = valid && (x2u < kX2Limit);
          const float xv = ok ? x2u * 3.0517578125e-05f : 0.f;
          const __half x_h = __float2half_rn(xv);
          const float r1 = xv - __half2float(x_h);
          const __half x_m = __float2half_rn(r1);
          const __half x_l = __float2half_rn(r1 - __half2float(x_m));
          const __half p15 = __float2half_rn(32768.f);
          const __half z = __float2half_rn(0.f);
          uint8_t* ae = sAext;
          *reinterpret_cast<uint4*>(ae + tc::kmajor_off(r, 0, kExt)) =
              make_uint4(pack_h2(acn, acn), pack_h2(acn, x_h), pack_h2(x_m, x_l), pack_h2(p15, z));
          *reinterpret_cast<uint4*>(ae + tc::kmajor_off(r, 8, kExt)) = make_uint4(0u, 0u, 0u, 0u);
          float xn;
          asm("sqrt.approx.f32 %0, %1;" : "=f"(xn) : "f"(x2u));
          // w: the prefix bound with the hi/lo split's (1 + 2^-11)^2 and fp32 sum slack
          s_stats[(w & 1) * kRows + r] = make_float4(x2u, xn * 1.000002f, ok ? 1.f : 0.f, (wsum + o.y) * 1.002f);
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) arrive_at_issuer<kPair>(&aefull[0]);
      }
    } else {
    const int th = lane >> 3;  // 4 lanes per row: lanes r, r+8, r+16, r+24
    const float sc = s_cst[CST_S];
    const __half acn = __float2half_rn(s_cst[CST_ACN]);
    const bool valid = s_cst[CST_VALID] != 0.f;
    int g = grp;  // next chunk of this group, counted over all items
    for (int w = 0; w < items; ++w) {
      // row partials over this group's chunks: |s x|^2 and the prefix bound
      // sum_c sum_{c'<=c} |x_c'| B_c' = sum_c' |x_c'| B_c' (nk - c')
      float x2[kTrPasses], wsum[kTrPasses];
#pragma unroll
      for (int ps = 0; ps < kTrPasses; ++ps) x2[ps] = wsum[ps] = 0.f;
      const int gend = (w + 1) * nk;
      for (; g < gend; g += kTrGroups) {
        const int c = g - w * nk;
        const int xs = g % G::XST, as = g % G::AST;
        const uint32_t aph = (uint32_t)((g / G::AST) & 1);
        mbar_wait(&xfull[xs], (uint32_t)((g / G::XST) & 1));
        if (ENC_KEXP & 4) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&xempty[xs]);
          mbar_wait(&aempty[as], aph ^ 1u);
          if (lane == 0) s_lo[as * kTrWarps + twg] = 1;
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) arrive_at_issuer<kPair>(&afull[as]);
          continue;
        }
        float v[kTrPasses][8];
#pragma unroll
        for (int ps = 0; ps < kTrPasses; ++ps) {
          const int r = 8 * kTrPasses * twg + 8 * ps + (lane & 7);
          const uint8_t* xb = sX + xs * G::X_STAGE + r * 128;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int ch = 2 * th + cc;
            const float4 f = *reinterpret_cast<const float4*>(xb + ((ch ^ (r & 7)) << 4));
            v[ps][4 * cc] = f.x;
            v[ps][4 * cc + 1] = f.y;
            v[ps][4 * cc + 2] = f.z;
            v[ps][4 * cc + 3] = f.w;
          }
        }
        uint32_t hw[kTrPasses][4], lw[kTrPasses][4];
        uint32_t lo_nz = 0;
        const float wc = (float)(nk - c) * s_bch[c] * 1.000001f;
#pragma unroll
        for (int ps = 0; ps < kTrPasses; ++ps) {
          float ec = 0.f;
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const float a0 = v[ps][j] * sc, a1 = v[ps][j + 1] * sc;
            const __half2 hh = __floats2half2_rn(a0, a1);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(a0 - hf.x, a1 - hf.y);
            hw[ps][j / 2] = *reinterpret_cast<const uint32_t*>(&hh);
            lw[ps][j / 2] = *reinterpret_cast<const uint32_t*>(&ll);
            lo_nz |= lw[ps][j / 2];
            ec = fmaf(a0, a0, fmaf(a1, a1, ec));
          }
          x2[ps] += ec;
          // the row's chunk energy (4 lanes per row), its norm rounded up, times max_j |B_j,c|
          ec += __shfl_xor_sync(0xffffffffu, ec, 8);
          ec += __shfl_xor_sync(0xffffffffu, ec, 16);
          wsum[ps] = fmaf(sqrtf(ec), wc, wsum[ps]);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, (lo_nz & 0x7fff7fffu) != 0);
        // released after the loaded values were consumed (an arrive issued right behind the
        // loads is not ordered after their completion: see encode_tc_kernel's transform)
        if (lane == 0) mbar_arrive(&xempty[xs]);
        if (ENC_KSPIN) mbar_wait_spin(&aempty[as], aph ^ 1u);
        else mbar_wait(&aempty[as], aph ^ 1u);
        uint8_t* ahi = sA + as * G::A_CHUNK;
#pragma unroll
        for (int ps = 0; ps < kTrPasses; ++ps) {
          const int r = 8 * kTrPasses * twg + 8 * ps + (lane & 7);
          *reinterpret_cast<uint4*>(ahi + tc::kmajor_off(r, 8 * th, kKC)) =
              make_uint4(hw[ps][0], hw[ps][1], hw[ps][2], hw[ps][3]);
          *reinterpret_cast<uint4*>(ahi + G::A_HI + tc::kmajor_off(r, 8 * th, kKC)) =
              make_uint4(lw[ps][0], lw[ps][1], lw[ps][2], lw[ps][3]);
        }
        if (lane == 0) s_lo[as * kTrWarps + twg] = (bal != 0);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) arrive_at_issuer<kPair>(&afull[as]);
      }
      // the item's rows: group 1 hands its partials to group 0, which writes the extension
      // rows and the stats (whole-row |s x|^2 now known)
#pragma unroll
      for (int ps = 0; ps < kTrPasses; ++ps) {
        x2[ps] += __shfl_xor_sync(0xffffffffu, x2[ps], 8);
        x2[ps] += __shfl_xor_sync(0xffffffffu, x2[ps], 16);
      }
      if (kTrGroups == 2) {
        if (grp == 1 && th == 0) {
#pragma unroll
          for (int ps = 0; ps < kTrPasses; ++ps)
            s_part[(w & 1) * kRows + 8 * kTrPasses * twg + 8 * ps + (lane & 7)] = make_float2(x2[ps], wsum[ps]);
        }
        asm volatile("bar.sync 5, %0;" ::"n"(kTrWarps * 32) : "memory");
        if (grp == 1) continue;
      }
      // one extension buffer: the previous item's extension instruction has completed long
      // before this item's last chunks could be stored (A ring of 2 behind the in-order MMAs)
      mbar_wait(&aeempty[0], (uint32_t)((w & 1) ^ 1));
#pragma unroll
      for (int ps = 0; ps < kTrPasses; ++ps) {
        const int r = 8 * kTrPasses * twg + 8 * ps + (lane & 7);
        const float2 o = kTrGroups == 2 ? s_part[(w & 1) * kRows + r] : make_float2(0.f, 0.f);
        const float acc = x2[ps] + o.x;
        // |s x|^2 rounded up: fp32 sums of ks products (relative error < (ks + 4) 2^-24)
        const float x2u = acc * (1.0f + (float)(ks + 16) * 5.9604644775390625e-08f);
        const bool ok = valid && (x2u < kX2Limit);
        if (th == 0) {
          const float xv = ok ? x2u * 3.0517578125e-05f : 0.f;
          const __half x_h = __float2half_rn(xv);
          const float r1 = xv - __half2float(x_h);
          const __half x_m = __float2half_rn(r1);
          const __half x_l = __float2half_rn(r1 - __half2float(x_m));
          const __half p15 = __float2half_rn(32768.f);
          const __half z = __float2half_rn(0.f);
          uint8_t* ae = sAext;
          *reinterpret_cast<uint4*>(ae + tc::kmajor_off(r, 0, kExt)) =
              make_uint4(pack_h2(acn, acn), pack_h2(acn, x_h), pack_h2(x_m, x_l), pack_h2(p15, z));
          *reinterpret_cast<uint4*>(ae + tc::kmajor_off(r, 8, kExt)) = make_uint4(0u, 0u, 0u, 0u);
          float xn;
          asm("sqrt.approx.f32 %0, %1;" : "=f"(xn) : "f"(x2u));
          // w: the prefix bound with the hi/lo split's (1 + 2^-11)^2 and fp32 sum slack
          s_stats[(w & 1) * kRows + r] =
              make_float4(x2u, xn * 1.000002f, ok ? 1.f : 0.f, (wsum[ps] + o.y) * 1.002f);
        }
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) arrive_at_issuer<kPair>(&aefull[0]);
    }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (kPair) tc::cluster_sync();  // no CTA leaves (or frees TMEM) while its peer can still signal it
  if (warp == 1) {
    tc::fence_after();
    if (kPair) tc::tmem_dealloc_pair(tbase, 512);
    else tc::tmem_dealloc(tbase, 512);
  }
}

// Codebook preparation for the K-streamed kernel: per subspace, B chunks [hi | lo] of 32
// columns then the extension block (same values as encode_prep_kernel).
// Prepared-operand cache of the K-streamed path (a stream encodes a long input chunk by
// chunk with one codebook): cw is compared word for word with the copy taken at the last
// preparation; equal -> encode_prep_k_kernel keeps the prepared operands.
__global__ void encode_cb_compare_kernel(const uint32_t* __restrict__ cw, const uint32_t* __restrict__ copy,
                                         int64_t words, int* __restrict__ differs) {
  int d = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    d |= (cw[i] != copy[i]);
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(differs, 1);
}

__global__ void __launch_bounds__(256) encode_prep_k_kernel(const float* __restrict__ cw, int m, int l, int ks,
                                                           uint8_t* __restrict__ bprep, float* __restrict__ cst,
                                                           float* __restrict__ bch, const int* __restrict__ differs,
                                                           float* __restrict__ cw_copy) {
  if (differs && *differs == 0) return;  // same codebook as the last preparation
  if (cw_copy) {
    const size_t per = (size_t)l * ks;
    for (size_t i = threadIdx.x; i < per; i += blockDim.x)
      cw_copy[(size_t)blockIdx.x * per + i] = cw[(size_t)blockIdx.x * per + i];
  }
  __shared__ float red[8], rb[8], rc[8], r1s[8];
  __shared__ unsigned int s_bmax[kMaxChunks];
  __shared__ int bad[8];
  __shared__ double redd[8];
  __shared__ float s_sc;
  __shared__ int s_bad;
  __shared__ double s_cn;
  const int mm = blockIdx.x, row = threadIdx.x, lane = row & 31, warp = row >> 5;
  const bool real = row < l;
  const float* c = cw + ((size_t)mm * l + (real ? row : 0)) * ks;
  float amax = 0.f;
  int nonfinite = 0;
  if (real)
    for (int k = 0; k < ks; ++k) {
      const float a = fabsf(c[k]);
      nonfinite |= !(a <= 3.4028234663852886e38f);
      amax = fmaxf(amax, a);
    }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o);
  }
  if (lane == 0) {
    red[warp] = amax;
    bad[warp] = nonfinite;
  }
  __syncthreads();
  if (row == 0) {
    float a = 0.f;
    int b = 0;
    for (int i = 0; i < 8; ++i) {
      a = fmaxf(a, red[i]);
      b |= bad[i];
    }
    int ex = 0;
    if (a > 0.f && !b) frexpf(a, &ex);
    s_sc = (a > 0.f && !b) ? ldexpf(1.0f, 8 - ex) : 1.0f;  // |s c| < 2^8
    s_bad = b;
  }
  __syncthreads();
  const float sc = s_sc;
  const bool cb_ok = !s_bad;
  uint8_t* base = bprep + (size_t)mm * GeoK<false>::bprep_bytes(ks);
  if (row < kMaxChunks) s_bmax[row] = 0u;
  __syncthreads();
  double cn = 0.0, nb2 = 0.0, s1 = 0.0, nbc = 0.0;
  for (int k = 0; k < ks; ++k) {
    const float cv = (real && cb_ok) ? c[k] * sc : 0.f;
    const float bv = -2.0f * cv;
    const __half hi = __float2half_rn(bv);
    const __half lo = __float2half_rn(bv - __half2float(hi));
    uint8_t* chunk = base + (size_t)(k / kKC) * GeoK<false>::GB_CHUNK;
    *reinterpret_cast<__half*>(chunk + tc::kmajor_off(row, k % kKC, kKC)) = hi;
    *reinterpret_cast<__half*>(chunk + GeoK<false>::GB_HI + tc::kmajor_off(row, k % kKC, kKC)) = lo;
    cn += (double)cv * (double)cv;
    nb2 += (double)bv * (double)bv;
    s1 += fabs((double)bv);
    nbc += (double)bv * (double)bv;
    if (k % kKC == kKC - 1) {  // chunk norm, rounded up (non-negative floats order as uint)
      atomicMax(&s_bmax[k / kKC], __float_as_uint((float)sqrt(nbc) * 1.0001f));
      nbc = 0.0;
    }
  }
  __syncthreads();
  if (row < ks / kKC) bch[(size_t)mm * kMaxChunks + row] = __uint_as_float(s_bmax[row]);
  double cmx = cn;
  for (int o = 16; o > 0; o >>= 1) cmx = fmax(cmx, __shfl_xor_sync(0xffffffffu, cmx, o));
  if (lane == 0) redd[warp] = cmx;
  __syncthreads();
  if (row == 0) {
    double a = 0.0;
    for (int i = 0; i < 8; ++i) a = fmax(a, redd[i]);
    s_cn = a;
  }
  __syncthreads();
  int ea = 0;
  if (s_cn >= 16384.0) {
    frexp(s_cn, &ea);
    ea -= 14;
  }
  const double acn = ldexp(1.0, ea);
  const double cvv = cn / acn;
  const __half c_h = __double2half(cvv);
  const double r1 = cvv - (double)__half2float(c_h);
  const __half c_m = __double2half(r1);
  const __half c_l = __double2half(r1 - (double)__half2float(c_m));
  const __half p15 = __float2half_rn(32768.f);
  const __half pad = __float2half_rn(real ? 0.f : 65504.f);
  const __half z = __float2half_rn(0.f);
  uint8_t* ext = base + (size_t)(ks / kKC) * GeoK<false>::GB_CHUNK;
  *reinterpret_cast<uint4*>(ext + tc::kmajor_off(row, 0, kExt)) =
      make_uint4(pack_h2(c_h, c_m), pack_h2(c_l, p15), pack_h2(p15, p15), pack_h2(pad, z));
  *reinterpret_cast<uint4*>(ext + tc::kmajor_off(row, 8, kExt)) = make_uint4(0u, 0u, 0u, 0u);
  float vb = real ? (float)sqrt(nb2) : 0.f, vc = real ? (float)cn : 0.f, v1 = real ? (float)s1 : 0.f;
  for (int o = 16; o > 0; o >>= 1) {
    vb = fmaxf(vb, __shfl_xor_sync(0xffffffffu, vb, o));
    vc = fmaxf(vc, __shfl_xor_sync(0xffffffffu, vc, o));
    v1 = fmaxf(v1, __shfl_xor_sync(0xffffffffu, v1, o));
  }
  if (lane == 0) {
    rb[warp] = vb;
    rc[warp] = vc;
    r1s[warp] = v1;
  }
  __syncthreads();
  if (row == 0) {
    float a = 0.f, b2 = 0.f, d = 0.f;
    for (int i = 0; i < 8; ++i) {
      a = fmaxf(a, rb[i]);
      b2 = fmaxf(b2, rc[i]);
      d = fmaxf(d, r1s[i]);
    }
    float* o = cst + (size_t)mm * CST_LEN;
    o[CST_S] = sc;
    o[CST_ACN] = (float)acn;
    o[CST_CB] = a * 1.0001f;
    o[CST_CN] = b2 * 1.0001f;
    o[CST_S1C] = d * 1.0001f;
    o[CST_VALID] = cb_ok ? 1.f : 0.f;
    o[6] = 0.f;
    o[7] = 0.f;
  }
}

// Exact float64 fallback for long subspaces (the pairs the tensor-core certificate left):
// the codebook streams through shared memory in 32-column chunks converted to float64 once
// per chunk (all warps of a block in lockstep); each warp decides two rows at a time, each
// lane keeping the running sequential sums of its 8 codewords for both, so the summation
// order is scipy cdist's and the argmin np.argmin's (first NaN, else lowest index).
constexpr int kExactRows = 4;
constexpr int kFilterRows = FILTER_ROWS;  // rows per warp of the fp32 pre-filter

// Flattened (subspace, tile) schedule of the K-streamed fallback kernels: tile t of the
// concatenated per-subspace lists (subspaces leave very different numbers of pairs, so a
// fixed block range per subspace left most blocks idle).
__device__ __forceinline__ bool flat_tile(int64_t t, int m, const unsigned int* __restrict__ counters, uint32_t cap,
                                          int64_t n, int rows_per, int& mm, int64_t& i0, int64_t& total) {
  const bool all = counters[1] != 0;
  for (int q = 0; q < m; ++q) {
    const int64_t tot = all ? n : (int64_t)min(counters[2 + q], cap);
    const int64_t nt = (tot + rows_per - 1) / rows_per;
    if (t < nt) {
      mm = q;
      i0 = t * rows_per;
      total = tot;
      return true;
    }
    t -= nt;
  }
  return false;
}

__global__ void __launch_bounds__(256) encode_exact_k_kernel(const float* __restrict__ x, int64_t n, int d,
                                                            const float* __restrict__ cw, int m, int l, int ks,
                                                            const uint32_t* __restrict__ flags,
                                                            const unsigned int* __restrict__ counters,
                                                            uint32_t flag_cap, uint8_t* __restrict__ codes, int stride,
                                                            int only_all) {
  extern __shared__ float s_cbf[];  // 2 x 256 x 33 float32 (double buffer)
  const bool all = counters[1] != 0;
  if (only_all && !all) return;  // the list went to encode_exact_cand_kernel
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int cbase[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) cbase[u] = min(lane + 32 * u, l - 1) * 33;  // c >= l aliases l - 1
  constexpr int kRowsPerBlock = 8 * kExactRows;
  for (int64_t t = blockIdx.x;; t += gridDim.x) {
    int mm;
    int64_t i0, total;
    if (!flat_tile(t, m, counters, flag_cap, n, kRowsPerBlock, mm, i0, total)) break;
    const float* cb = cw + (size_t)mm * l * ks;
    bool active[kExactRows];
    int64_t row[kExactRows];
#pragma unroll
    for (int r = 0; r < kExactRows; ++r) {
      const int64_t i = i0 + warp * kExactRows + r;
      active[r] = i < total;
      row[r] = active[r] ? (all ? i : (int64_t)flags[(size_t)mm * flag_cap + i]) : 0;
    }
    double acc[kExactRows][8];
#pragma unroll
    for (int r = 0; r < kExactRows; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[r][u] = 0.0;
    // fp32 codebook chunks double-buffered through cp.async (exact in float64 on use), the
    // rows' x values one chunk ahead in registers
    auto stage = [&](int k0, int buf) {
      float* dst = s_cbf + buf * (256 * 33);
      for (int e = threadIdx.x; e < l * 32; e += blockDim.x) {
        const int c = e >> 5, k = e & 31;
        const uint32_t sa = smem_u32(dst + c * 33 + k);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(cb + (size_t)c * ks + k0 + k)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    __syncthreads();  // the previous tile's readers are done with both buffers
    stage(0, 0);
    float xn[kExactRows];
#pragma unroll
    for (int r = 0; r < kExactRows; ++r) xn[r] = active[r] ? x[row[r] * d + (size_t)mm * ks + lane] : 0.f;
    for (int k0 = 0; k0 < ks; k0 += 32) {
      const int buf = (k0 >> 5) & 1;
      if (k0 + 32 < ks) {
        stage(k0 + 32, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      float xl[kExactRows];
#pragma unroll
      for (int r = 0; r < kExactRows; ++r) xl[r] = xn[r];
      if (k0 + 32 < ks) {
#pragma unroll
        for (int r = 0; r < kExactRows; ++r)
          xn[r] = active[r] ? x[row[r] * d + (size_t)mm * ks + k0 + 32 + lane] : 0.f;
      }
      const float* scb = s_cbf + buf * (256 * 33);
#pragma unroll 2
      for (int k = 0; k < 32; ++k) {
        double c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = (double)scb[cbase[u] + k];
#pragma unroll
        for (int r = 0; r < kExactRows; ++r) {
          const double xk = (double)__shfl_sync(0xffffffffu, xl[r], k);
          double df[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) df[u] = __dsub_rn(xk, c[u]);
#pragma unroll
          for (int u = 0; u < 8; ++u) df[u] = __dmul_rn(df[u], df[u]);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[r][u] = __dadd_rn(acc[r][u], df[u]);
        }
      }
      __syncthreads();  // buffer buf is restaged two chunks later
    }
#pragma unroll
    for (int r = 0; r < kExactRows; ++r) {
      double best = __longlong_as_double(0x7ff0000000000000LL);
      int bl = 0x7fffffff;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = lane + 32 * u;
        if (argmin_less(acc[r][u], c, best, bl)) {
          best = acc[r][u];
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
      if (active[r] && lane == 0) codes[row[r] * stride + mm] = (uint8_t)bl;
    }
  }
}

// fp32 pre-filter of the K-streamed path's uncertified pairs (config 3: 512-D subspaces
// of deep features leave ~4.7% of the (vector, subspace) pairs to the exact path, whose
// float64 sums dominated the encode).  Same schedule as encode_exact_k_kernel (codebook
// chunks of 32 dimensions staged in shared memory, a warp per row, lanes over codewords)
// but in fp32: d = fma(x - c, x - c, d), sequential over the ks dimensions.  Bound: every
// term is >= 0, so the computed sum D^ and the exact real sum D of the fp32 inputs obey
// |D^ - D| <= g D + eta, g = (ks + 2) 2^-24 (x 1.01), eta = ks 2^-120 (underflowed squares);
// the reference's float64 sum D64 obeys |D64 - D| <= g64 D, g64 = (ks + 2) 2^-53.  The
// fp32 winner (b1, lowest index on ties) is certified when
//     (b1 + eta)(1 + g)(1 + g64) < (b2 - eta)(1 - g)(1 - g64)      (b2: the runner-up)
// in float64: then every other codeword's float64 distance exceeds the winner's, which is
// np.argmin over scipy's cdist row.  Rows with NaN / inf, near ties and exact ties go on
// to the float64 kernel (list flags2 / counters2, per subspace).
__global__ void __launch_bounds__(256) encode_filter32_k_kernel(
    const float* __restrict__ x, int64_t n, int d, const float* __restrict__ cw, int m, int l, int ks,
    const uint32_t* __restrict__ flags, const unsigned int* __restrict__ counters, uint32_t flag_cap,
    uint8_t* __restrict__ codes, int stride, uint32_t* __restrict__ flags2, unsigned int* __restrict__ counters2,
    uint32_t* __restrict__ cmask) {
  extern __shared__ float s_cbf[];  // 2 x 256 x 33 float32 (double buffer)
  const bool all = counters[1] != 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int cbase[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) cbase[u] = min(lane + 32 * u, l - 1) * 33;  // c >= l aliases l - 1
  constexpr int kRowsPerBlock = 8 * kFilterRows;
  const double g32 = (double)(ks + 2) * 5.9604644775390625e-08 * 1.01;
  const double g64 = (double)(ks + 2) * 1.1102230246251565e-16 * 1.01;
  const double eta = (double)ks * 7.52316384526264e-37;  // ks x 2^-120
  for (int64_t t = blockIdx.x;; t += gridDim.x) {
    int mm;
    int64_t i0, total;
    if (!flat_tile(t, m, counters, flag_cap, n, kRowsPerBlock, mm, i0, total)) break;
    const float* cb = cw + (size_t)mm * l * ks;
    bool active[kFilterRows];
    int64_t row[kFilterRows];
#pragma unroll
    for (int r = 0; r < kFilterRows; ++r) {
      const int64_t i = i0 + warp * kFilterRows + r;
      active[r] = i < total;
      row[r] = active[r] ? (all ? i : (int64_t)flags[(size_t)mm * flag_cap + i]) : 0;
    }
    float acc[kFilterRows][8];
#pragma unroll
    for (int r = 0; r < kFilterRows; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[r][u] = 0.f;
    // codebook chunks double-buffered through cp.async (chunk c + 1 in flight while chunk c
    // is consumed), the rows' x values one chunk ahead in registers
    auto stage = [&](int k0, int buf) {
      float* dst = s_cbf + buf * (256 * 33);
      for (int e = threadIdx.x; e < l * 32; e += blockDim.x) {
        const int c = e >> 5, k = e & 31;
        const uint32_t sa = smem_u32(dst + c * 33 + k);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(cb + (size_t)c * ks + k0 + k)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    __syncthreads();  // the previous tile's readers are done with both buffers
    stage(0, 0);
    float xn[kFilterRows];
#pragma unroll
    for (int r = 0; r < kFilterRows; ++r) xn[r] = active[r] ? x[row[r] * d + (size_t)mm * ks + lane] : 0.f;
    for (int k0 = 0; k0 < ks; k0 += 32) {
      const int buf = (k0 >> 5) & 1;
      if (k0 + 32 < ks) {
        stage(k0 + 32, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      float xl[kFilterRows];
#pragma unroll
      for (int r = 0; r < kFilterRows; ++r) xl[r] = xn[r];
      if (k0 + 32 < ks) {
#pragma unroll
        for (int r = 0; r < kFilterRows; ++r)
          xn[r] = active[r] ? x[row[r] * d + (size_t)mm * ks + k0 + 32 + lane] : 0.f;
      }
      const float* sc = s_cbf + buf * (256 * 33);
#pragma unroll 4
      for (int k = 0; k < 32; ++k) {
        float c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = sc[cbase[u] + k];
#pragma unroll
        for (int r = 0; r < kFilterRows; ++r) {
          const float xk = __shfl_sync(0xffffffffu, xl[r], k);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float df = __fsub_rn(xk, c[u]);
            acc[r][u] = __fmaf_rn(df, df, acc[r][u]);
          }
        }
      }
      __syncthreads();  // buffer buf is restaged two chunks later
    }
#pragma unroll
    for (int r = 0; r < kFilterRows; ++r) {
      // best (lowest index on ties) and runner-up over the 256 codewords; NaN never wins
      float b1 = __int_as_float(0x7f800000), b2 = b1;
      int l1 = 0x7fffffff;
      bool nan = false;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = lane + 32 * u;
        if (c >= l) continue;
        const float v = acc[r][u];
        nan |= (v != v);
        if (v < b1) {
          b2 = b1;
          b1 = v;
          l1 = c;
        } else {
          b2 = fminf(b2, v);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
        const float ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
        const int ol1 = __shfl_xor_sync(0xffffffffu, l1, o);
        if (ob1 < b1 || (ob1 == b1 && ol1 < l1)) {
          b2 = fminf(b1, ob2);
          b1 = ob1;
          l1 = ol1;
        } else {
          b2 = fminf(b2, ob1);
        }
      }
      nan = __any_sync(0xffffffffu, nan);
      const double lhs = ((double)b1 + eta) * (1.0 + g32) * (1.0 + g64) * (1.0 + 1e-12);
      const double rhs = ((double)b2 - eta) * (1.0 - g32) * (1.0 - g64);
      const bool finite = !nan && b1 < __int_as_float(0x7f800000);
      const bool cert = finite && lhs < rhs;  // false for inf / NaN
      if (!cert) {
        // candidates for the float64 decision: every codeword whose float64 distance can be
        // <= the winner's (lower bound <= the winner's upper bound); all of them for rows
        // with NaN / inf (np.argmin's NaN rule needs every value)
        unsigned f = 0;
        if (lane == 0 && active[r]) {
          atomicAdd(&counters2[0], 1u);
          f = atomicAdd(&counters2[2 + mm], 1u);
          if (f < flag_cap)
            flags2[(size_t)mm * flag_cap + f] = (uint32_t)row[r];
          else
            counters2[1] = 1u;
        }
        f = __shfl_sync(0xffffffffu, f, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = lane + 32 * u;
          const double lo = ((double)acc[r][u] - eta) * (1.0 - g32) * (1.0 - g64);
          const bool cand = c < l && (!finite || lo <= lhs);
          const unsigned bm = __ballot_sync(0xffffffffu, cand);
          if (lane == 0 && active[r] && f < flag_cap && cmask) cmask[((size_t)mm * flag_cap + f) * 8 + u] = bm;
        }
      } else if (active[r] && lane == 0) {
        codes[row[r] * stride + mm] = (uint8_t)l1;
      }
    }
  }
}

// fp32 filter over the tensor-core pass's candidates (K-streamed path).  encode_tck_kernel
// leaves each uncertified pair with the mask of the codewords its error bound cannot
// exclude (a handful of the 256); this kernel evaluates only those: one warp per pair,
// lanes over the dimensions (float4, coalesced codeword rows), d^ = sum (x - c)^2 in fp32.
// Every term is >= 0, so for any summation order |d^ - D| <= g D + eta with
// g = (ks + 2) 2^-24 (x 1.01), eta = ks 2^-120 (encode_filter32_k_kernel's bound, which this
// kernel replaces on the product path); the certificate and the reduced candidate mask
// handed to encode_exact_cand_kernel are the same as there.
#ifndef FILTER_GRID
#define FILTER_GRID 2  // CTAs per SM of the candidate filter's grid-stride launch: one resident wave (config 3: 126 us; 8 per SM: 134 us)
#endif
#ifndef EXACT_GRID
#define EXACT_GRID 8
#endif
#ifndef FILTER_OCC
#define FILTER_OCC 2
#endif
// (one dependent chain flag -> row -> x -> candidate rows per pair and warp; measured at
// config 3: 2 resident CTAs per SM 134 us, 3 or 4 (80 / 64 registers) 153 us)
__global__ void __launch_bounds__(256, FILTER_OCC) encode_filter32_cand_kernel(
    const float* __restrict__ x, int d, const float* __restrict__ cw, int m, int l, int ks,
    const uint32_t* __restrict__ flags, const unsigned int* __restrict__ counters, uint32_t flag_cap,
    const uint32_t* __restrict__ tcmask, uint8_t* __restrict__ codes, int stride, uint32_t* __restrict__ flags2,
    unsigned int* __restrict__ counters2, uint32_t* __restrict__ cmask2) {
  __shared__ float s_val[8][256];
  if (counters[1] != 0) {  // the pair list overflowed: every row goes to encode_exact_k_kernel
    if (blockIdx.x == 0 && threadIdx.x == 0) counters2[1] = 1u;
    return;
  }
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double g32 = (double)(ks + 2) * 5.9604644775390625e-08 * 1.01;
  const double g64 = (double)(ks + 2) * 1.1102230246251565e-16 * 1.01;
  const double eta = (double)ks * 7.52316384526264e-37;  // ks x 2^-120
  int64_t tot = 0;
  for (int q = 0; q < m; ++q) tot += min(counters[2 + q], flag_cap);
  float* val = s_val[wib];
  for (int64_t pi = gw; pi < tot; pi += nw) {
    int mm = 0;
    int64_t i = pi;
    while (i >= (int64_t)min(counters[2 + mm], flag_cap)) i -= min(counters[2 + mm], flag_cap), ++mm;
    const size_t slot = (size_t)mm * flag_cap + (size_t)i;
    const int64_t row = flags[slot];
    const float* xv = x + row * d + (size_t)mm * ks;
    const float* cb = cw + (size_t)mm * l * ks;
    // the row's x values: float4 groups lane, lane + 32, ... (ks <= 1024: at most 8 per lane)
    float4 xr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      xr[q] = (4 * (lane + 32 * q) < ks) ? __ldg(reinterpret_cast<const float4*>(xv) + lane + 32 * q)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t mword[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) mword[u] = __ldg(tcmask + slot * 8 + u);
    float b1 = __int_as_float(0x7f800000);
    int l1 = 0x7fffffff;
    bool nan = false;
    __syncwarp();
    for (int u = 0; u < 8; ++u) {
      uint32_t bm = mword[u];
      while (bm) {
        // two candidates per round (their loads overlap)
        const int j0 = __ffs(bm) - 1;
        bm &= bm - 1u;
        const int j1 = bm ? __ffs(bm) - 1 : -1;
        if (j1 >= 0) bm &= bm - 1u;
        const int c0 = min(32 * u + j0, l - 1), c1 = min(32 * u + max(j1, 0), l - 1);
        const float4* r0 = reinterpret_cast<const float4*>(cb + (size_t)c0 * ks);
        const float4* r1 = reinterpret_cast<const float4*>(cb + (size_t)c1 * ks);
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (4 * (lane + 32 * q) < ks) {
            const float4 v0 = __ldg(r0 + lane + 32 * q), v1 = __ldg(r1 + lane + 32 * q);
            float t;
            t = __fsub_rn(xr[q].x, v0.x), a0 = __fmaf_rn(t, t, a0);
            t = __fsub_rn(xr[q].y, v0.y), a0 = __fmaf_rn(t, t, a0);
            t = __fsub_rn(xr[q].z, v0.z), a0 = __fmaf_rn(t, t, a0);
            t = __fsub_rn(xr[q].w, v0.w), a0 = __fmaf_rn(t, t, a0);
            t = __fsub_rn(xr[q].x, v1.x), a1 = __fmaf_rn(t, t, a1);
            t = __fsub_rn(xr[q].y, v1.y), a1 = __fmaf_rn(t, t, a1);
            t = __fsub_rn(xr[q].z, v1.z), a1 = __fmaf_rn(t, t, a1);
            t = __fsub_rn(xr[q].w, v1.w), a1 = __fmaf_rn(t, t, a1);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a0 = __fadd_rn(a0, __shfl_xor_sync(0xffffffffu, a0, o));
          a1 = __fadd_rn(a1, __shfl_xor_sync(0xffffffffu, a1, o));
        }
        if (32 * u + j0 < l) {
          nan |= (a0 != a0);
          if (a0 < b1) b1 = a0, l1 = 32 * u + j0;  // ascending index: the first minimum stays
          if (lane == 0) val[32 * u + j0] = a0;
        }
        if (j1 >= 0 && 32 * u + j1 < l) {
          nan |= (a1 != a1);
          if (a1 < b1) b1 = a1, l1 = 32 * u + j1;
          if (lane == 0) val[32 * u + j1] = a1;
        }
      }
    }
    __syncwarp();
    // candidates whose float64 distance can be <= the winner's (the winner among them)
    const double lhs = ((double)b1 + eta) * (1.0 + g32) * (1.0 + g64) * (1.0 + 1e-12);
    const bool finite = !nan && b1 < __int_as_float(0x7f800000);
    uint32_t out[8];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = lane + 32 * u;
      const bool in = c < l && ((mword[u] >> lane) & 1u);
      bool cand = false;
      if (in) {
        const double lo = ((double)val[c] - eta) * (1.0 - g32) * (1.0 - g64);
        cand = !finite || lo <= lhs;
      }
      out[u] = __ballot_sync(0xffffffffu, cand);
      cnt += __popc(out[u]);
    }
    if (finite && cnt == 1) {
      if (lane == 0) codes[row * stride + mm] = (uint8_t)l1;
    } else {
      unsigned f = 0;
      if (lane == 0) {
        atomicAdd(&counters2[0], 1u);
        f = atomicAdd(&counters2[2 + mm], 1u);
        if (f < flag_cap)
          flags2[(size_t)mm * flag_cap + f] = (uint32_t)row;
        else
          counters2[1] = 1u;
      }
      f = __shfl_sync(0xffffffffu, f, 0);
      // an empty mask (cannot happen: the tensor-core winner is always its own candidate) or a
      // non-finite row: every codeword goes to the float64 decision
      if (f < flag_cap && lane < 8) {
        uint32_t wv = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) wv = (lane == u) ? out[u] : wv;
        if (!finite || cnt == 0) {  // codewords 32 lane .. 32 lane + 31 below l
          const int nb = min(max(l - 32 * lane, 0), 32);
          wv = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
        }
        cmask2[((size_t)mm * flag_cap + f) * 8 + lane] = wv;
      }
    }
    __syncwarp();
  }
}

// Float64 decision over the pre-filter's candidates only (typically 2-3 of the 256
// codewords per pair).  Float64 issue is the scarce resource (a warp instruction costs the
// same for one active lane as for 32), so a warp packs the (pair, candidate) entries of
// consecutive pairs onto its 32 lanes: each lane runs the sequential float64 sum of
// (x - c)^2 in scipy cdist order for its entry, a segmented reduction picks each pair's
// winner in np.argmin order (first NaN, else value, then lowest index).  Codewords outside
// the candidate set are provably farther in float64 (see encode_filter32_cand_kernel), so
// this is the argmin over all 256.  Pairs with more than 32 candidates (non-finite rows:
// all of them) take the lanes alone, in rounds.  When the pair list overflowed
// (counters2[1]) every row goes through encode_exact_k_kernel.
__device__ __forceinline__ double exact_dist64(const float* __restrict__ xv, const float* __restrict__ cv, int ks) {
  const float4* cv4 = reinterpret_cast<const float4*>(cv);
  const float4* xv4 = reinterpret_cast<const float4*>(xv);
  double acc = 0.0;
  for (int k0 = 0; k0 < ks / 4; k0 += 8) {  // 32 dimensions per batch of loads (ks % 32 == 0)
    float4 xa[8], ca[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      xa[q] = __ldg(xv4 + k0 + q);
      ca[q] = __ldg(cv4 + k0 + q);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float xs[4] = {xa[q].x, xa[q].y, xa[q].z, xa[q].w};
      const float cs[4] = {ca[q].x, ca[q].y, ca[q].z, ca[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double df = __dsub_rn((double)xs[e], (double)cs[e]);
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
    }
  }
  return acc;
}

__global__ void __launch_bounds__(256, 4) encode_exact_cand_kernel(
    const float* __restrict__ x, int d, const float* __restrict__ cw, int m, int l, int ks,
    const uint32_t* __restrict__ flags2, const unsigned int* __restrict__ counters2, uint32_t flag_cap,
    const uint32_t* __restrict__ cmask, uint8_t* __restrict__ codes, int stride) {
  if (counters2[1] != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t tot = 0;
  for (int q = 0; q < m; ++q) tot += min(counters2[2 + q], flag_cap);
  // a contiguous range of pairs per warp
  // (at least 12: ~30 candidates, so that a flush fills most lanes)
  const int64_t per = max((tot + nw - 1) / nw, (int64_t)12);
  const int64_t p0 = min(tot, gw * per), p1 = min(tot, p0 + per);
  // lane state of the batch being filled
  const float* my_x = nullptr;
  const float* my_c = nullptr;
  int my_cw = 0x7fffffff, my_seg = -1;
  int64_t my_out = -1;  // head lanes: where the pair's code goes
  int fill = 0, seg = 0;
  auto flush = [&]() {
    double acc = __longlong_as_double(0x7ff0000000000000LL);
    if (my_seg >= 0) acc = exact_dist64(my_x, my_c, ks);
    int bl = my_cw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, acc, o);
      const int oi = __shfl_down_sync(0xffffffffu, bl, o);
      const int os = __shfl_down_sync(0xffffffffu, my_seg, o);
      if (lane + o < 32 && os == my_seg && my_seg >= 0 && argmin_less(ob, oi, acc, bl)) {
        acc = ob;
        bl = oi;
      }
    }
    if (my_out >= 0) codes[my_out] = (uint8_t)bl;
    my_seg = -1;
    my_out = -1;
    my_cw = 0x7fffffff;
    fill = 0;
    seg = 0;
  };
  for (int64_t p = p0; p < p1; ++p) {
    int mm = 0;
    int64_t i = p;
    while (i >= (int64_t)min(counters2[2 + mm], flag_cap)) i -= min(counters2[2 + mm], flag_cap), ++mm;
    const size_t slot = (size_t)mm * flag_cap + (size_t)i;
    const int64_t row = flags2[slot];
    const float* xv = x + row * d + (size_t)mm * ks;
    const float* cb = cw + (size_t)mm * l * ks;
    // lane u < 8 holds mask word u (codewords 32 u ..); counts and their prefix over the words
    const uint32_t wv = lane < 8 ? __ldg(cmask + slot * 8 + lane) : 0u;
    const int pc = __popc(wv);
    int pre = pc;  // inclusive prefix over lanes
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += t;
    }
    const int cnt = __shfl_sync(0xffffffffu, pre, 7);
    if (cnt == 0) continue;  // cannot happen (the filter's winner is its own candidate)
    if (cnt > 32) {
      // rounds of 32 candidates on the whole warp
      flush();
      double best = __longlong_as_double(0x7ff0000000000000LL);
      int bl = 0x7fffffff;
      for (int t0 = 0; t0 < cnt; t0 += 32) {
        const int k = t0 + lane;  // this lane's candidate: the k-th set bit of the 256-bit mask
        int cwi = -1;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t wu = __shfl_sync(0xffffffffu, wv, u);
          const int hi = __shfl_sync(0xffffffffu, pre, u), lo = hi - __popc(wu);
          if (k < cnt && k >= lo && k < hi) cwi = 32 * u + (int)__fns(wu, 0, k - lo + 1);
        }
        if (cwi >= 0) {
          const double acc = exact_dist64(xv, cb + (size_t)cwi * ks, ks);
          if (argmin_less(acc, cwi, best, bl)) {
            best = acc;
            bl = cwi;
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bl, o);
        if (argmin_less(ob, oi, best, bl)) {
          best = ob;
          bl = oi;
        }
      }
      if (lane == 0) codes[row * stride + mm] = (uint8_t)bl;
      continue;
    }
    if (fill + cnt > 32) flush();
    // lanes fill .. fill + cnt - 1 take the pair's candidates in ascending codeword order
    {
      const int k = lane - fill;
      int cwi = -1;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t wu = __shfl_sync(0xffffffffu, wv, u);
        const int hi = __shfl_sync(0xffffffffu, pre, u), lo = hi - __popc(wu);
        if (k >= 0 && k < cnt && k >= lo && k < hi) cwi = 32 * u + (int)__fns(wu, 0, k - lo + 1);
      }
      if (cwi >= 0) {
        my_x = xv;
        my_c = cb + (size_t)cwi * ks;
        my_cw = cwi;
        my_seg = seg;
        if (k == 0) my_out = row * stride + mm;
      }
    }
    fill += cnt;
    ++seg;
  }
  flush();
}

__global__ void encode_stats_kernel(const unsigned int* __restrict__ counters, unsigned long long* __restrict__ out) {
  *out += (unsigned long long)counters[0];  // pairs not certified (all re-decided in fp64)
}

}  // namespace enc

// ---------------------------------------------------------------------------
// host side
namespace {
// Encoder workspace (prepared codebook operands, flag buckets, counters), one per
// (device, stream): launches on one stream are ordered, so a buffer is reused only after
// the previous encode on that stream has finished with it.
struct EncWS {
  void* p = nullptr;
  size_t bytes = 0;
  // K-streamed path: the codebook the prepared operands were made from (a device copy in
  // the workspace) and the shape / pointer it was prepared for
  const float* prep_cw = nullptr;
  int prep_m = 0, prep_l = 0, prep_ks = 0;
};
std::mutex g_encws_mu;
std::map<std::pair<int, cudaStream_t>, EncWS> g_encws;

EncWS& enc_workspace(cudaStream_t stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  return g_encws[{dev, stream}];
}

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
int launch_encode_tc(const float* d_x, int64_t n, int d, const float* d_cw, int m, int l, int ks, uint8_t* d_codes,
                     int stride, unsigned long long* flagged_out, cudaStream_t stream) {
  using namespace enc;
  using G = Geo<KP>;
  const DevInfo& di = dev_info();
  std::lock_guard<std::mutex> lock(g_encws_mu);
  EncWS& ws = enc_workspace(stream);
  const size_t b_bytes = (size_t)m * G::B_BYTES;
  const uint32_t cap = (uint32_t)std::min<int64_t>(n, n / 4 + 4096);  // flagged rows per subspace
  const size_t need = align_up(b_bytes, 256) + align_up((size_t)m * CST_LEN * 4, 256) +
                      align_up((size_t)m * cap * 4, 256) + align_up((size_t)(m + 2) * 4, 256);
  if (ws.bytes < need) {
    if (ws.p) cudaFree(ws.p);
    ws.p = nullptr;
    ws.bytes = 0;
    PQK_CUDA_TRY(cudaMalloc(&ws.p, need));
    ws.bytes = need;
  }
  char* base = static_cast<char*>(ws.p);
  uint8_t* bprep = reinterpret_cast<uint8_t*>(base);
  float* cst = reinterpret_cast<float*>(base + align_up(b_bytes, 256));
  uint32_t* flags = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(cst) + align_up((size_t)m * CST_LEN * 4, 256));
  unsigned int* counters =
      reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(flags) + align_up((size_t)m * cap * 4, 256));

  CUtensorMap map;
  auto encoder = tensor_map_encoder();
  if (!encoder) return fail(PQK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  const cuuint32_t box[2] = {(cuuint32_t)std::min(ks, 32), (cuuint32_t)kRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult cr = encoder(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(d_x), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              ks >= 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(PQK_ECUDA, "cuTensorMapEncodeTiled failed");

  PQK_CUDA_TRY(cudaMemsetAsync(counters, 0, (size_t)(m + 2) * 4, stream));
  encode_prep_kernel<KP><<<m, 256, 0, stream>>>(d_cw, m, l, ks, bprep, cst);
  PQK_LAUNCH_CHECK("encode_prep_kernel");
  EncParams ep{};
  ep.bprep = bprep;
  ep.cst = cst;
  ep.n = n;
  ep.m = m;
  ep.ks = ks;
  ep.codes = d_codes;
  ep.stride = stride;
  ep.flags = flags;
  ep.counters = counters;
  ep.flag_cap = cap;
  ep.ntiles = (int)((n + kRows - 1) / kRows);
  ep.tstride = std::max(1, std::min(di.sms / m, ep.ntiles));  // CTAs per subspace
  ep.keymask = ~15u;
  ep.one = 1u;
  auto kern = encode_tc_kernel<KP>;
  PQK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
  kern<<<ep.tstride * m, kThreadsR, G::SMEM, stream>>>(map, ep);
  PQK_LAUNCH_CHECK("encode_tc_kernel");
  const int exact_smem = l * (ks + 1) * 4;
  PQK_CUDA_TRY(cudaFuncSetAttribute(encode_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, exact_smem));
  const dim3 egrid((unsigned)std::max(1, 2 * di.sms / m), (unsigned)m);
  encode_exact_kernel<<<egrid, 256, exact_smem, stream>>>(d_x, n, d, d_cw, m, l, ks, flags, counters, cap, d_codes,
                                                          stride);
  PQK_LAUNCH_CHECK("encode_exact_kernel");
  encode_stats_kernel<<<1, 1, 0, stream>>>(counters, flagged_out);
  PQK_LAUNCH_CHECK("encode_stats_kernel");
  return PQK_OK;
}
// K-streamed launch for long subspaces (ks % 32 == 0, 96 <= ks <= 1024)
int launch_encode_tck(const float* d_x, int64_t n, int d, const float* d_cw, int m, int l, int ks, uint8_t* d_codes,
                      int stride, unsigned long long* flagged_out, cudaStream_t stream) {
  using namespace enc;
  using G = GeoK<false>;
  const DevInfo& di = dev_info();
  std::lock_guard<std::mutex> lock(g_encws_mu);
  EncWS& ws = enc_workspace(stream);
  const size_t b_bytes = (size_t)m * G::bprep_bytes(ks);
  const uint32_t cap = (uint32_t)std::min<int64_t>(n, n / 4 + 4096);  // flagged rows per subspace
  const size_t bch_bytes = align_up((size_t)m * kMaxChunks * 4, 256);
  const size_t need = align_up(b_bytes, 256) + align_up((size_t)m * CST_LEN * 4, 256) +
                      2 * (align_up((size_t)m * cap * 4, 256) + align_up((size_t)(m + 2) * 4, 256)) + bch_bytes +
                      2 * align_up((size_t)m * cap * 32, 256) + align_up((size_t)m * l * ks * 4, 256) + 256;
  if (ws.bytes < need) {
    if (ws.p) cudaFree(ws.p);
    ws.p = nullptr;
    ws.bytes = 0;
    ws.prep_cw = nullptr;  // the layout moves: prepare again
    PQK_CUDA_TRY(cudaMalloc(&ws.p, need));
    ws.bytes = need;
  }
  char* base = static_cast<char*>(ws.p);
  uint8_t* bprep = reinterpret_cast<uint8_t*>(base);
  float* cst = reinterpret_cast<float*>(base + align_up(b_bytes, 256));
  uint32_t* flags = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(cst) + align_up((size_t)m * CST_LEN * 4, 256));
  unsigned int* counters =
      reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(flags) + align_up((size_t)m * cap * 4, 256));
  float* bch = reinterpret_cast<float*>(reinterpret_cast<char*>(counters) + align_up((size_t)(m + 2) * 4, 256));
  // the fp32 pre-filter's output list: pairs left to the float64 kernel
  uint32_t* flags2 = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(bch) + bch_bytes);
  unsigned int* counters2 =
      reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(flags2) + align_up((size_t)m * cap * 4, 256));
  uint32_t* cmask = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(counters2) + align_up((size_t)(m + 2) * 4, 256));
  // candidate masks left by the tensor-core pass (cmask: those left by the fp32 filter)
  uint32_t* tcmask = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(cmask) + align_up((size_t)m * cap * 32, 256));
  float* cw_copy = reinterpret_cast<float*>(reinterpret_cast<char*>(tcmask) + align_up((size_t)m * cap * 32, 256));
  int* differs = reinterpret_cast<int*>(reinterpret_cast<char*>(cw_copy) + align_up((size_t)m * l * ks * 4, 256));

  CUtensorMap map;
  auto encoder = tensor_map_encoder();
  if (!encoder) return fail(PQK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kKC, (cuuint32_t)kRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult cr = encoder(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(d_x), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(PQK_ECUDA, "cuTensorMapEncodeTiled failed");

  PQK_CUDA_TRY(cudaMemsetAsync(counters, 0, (size_t)(m + 2) * 4, stream));
  PQK_CUDA_TRY(cudaMemsetAsync(counters2, 0, (size_t)(m + 2) * 4, stream));
  // prepared operands: reused when the same codebook (pointer, shape and contents) comes back
  const bool same_shape = ws.prep_cw == d_cw && ws.prep_m == m && ws.prep_l == l && ws.prep_ks == ks;
  if (same_shape) {
    PQK_CUDA_TRY(cudaMemsetAsync(differs, 0, sizeof(int), stream));
    const int64_t words = (int64_t)m * l * ks;
    encode_cb_compare_kernel<<<(int)std::min<int64_t>((words + 255) / 256, (int64_t)di.sms * 4), 256, 0, stream>>>(
        reinterpret_cast<const uint32_t*>(d_cw), reinterpret_cast<const uint32_t*>(cw_copy), words, differs);
    PQK_LAUNCH_CHECK("encode_cb_compare_kernel");
  }
  encode_prep_k_kernel<<<m, 256, 0, stream>>>(d_cw, m, l, ks, bprep, cst, bch, same_shape ? differs : nullptr,
                                              cw_copy);
  ws.prep_cw = d_cw;
  ws.prep_m = m;
  ws.prep_l = l;
  ws.prep_ks = ks;
  PQK_LAUNCH_CHECK("encode_prep_k_kernel");
  EncParams ep{};
  ep.bprep = bprep;
  ep.cst = cst;
  ep.bch = bch;
  ep.n = n;
  ep.m = m;
  ep.ks = ks;
  ep.codes = d_codes;
  ep.stride = stride;
  ep.flags = flags;
  ep.counters = counters;
  ep.flag_cap = cap;
  ep.ntiles = (int)((n + kRows - 1) / kRows);
  ep.keymask = ~15u;
  ep.one = 1u;
  ep.tcmask = tcmask;
  // CTA pairs (cta_group::2: half the B bytes through each CTA's shared memory) unless
  // PQK_ENCODE_TCK_PAIR=0 or the input is a single tile
  static const bool pair_off = [] {
    const char* e = getenv("PQK_ENCODE_TCK_PAIR");
    return e && e[0] == '0';
  }();
  if (!pair_off && ep.ntiles >= 2 && di.sms >= 2 * m) {
    using GP = GeoK<true>;
    ep.tstride = std::max(1, std::min(di.sms / 2 / m, (ep.ntiles + 1) / 2));  // tile pairs per subspace
    PQK_CUDA_TRY(cudaFuncSetAttribute(encode_tck_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GP::SMEM));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * ep.tstride * m), 1u, 1u);
    cfg.blockDim = dim3((unsigned)kThreads, 1u, 1u);
    cfg.dynamicSmemBytes = GP::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PQK_CUDA_TRY(cudaLaunchKernelEx(&cfg, encode_tck_kernel<true>, map, ep));
  } else {
    ep.tstride = std::max(1, std::min(di.sms / m, ep.ntiles));
    PQK_CUDA_TRY(
        cudaFuncSetAttribute(encode_tck_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    encode_tck_kernel<false><<<ep.tstride * m, kThreads, G::SMEM, stream>>>(map, ep);
  }
  PQK_LAUNCH_CHECK("encode_tck_kernel");
  const dim3 egrid((unsigned)(2 * di.sms), 1u);  // flattened (subspace, tile) schedule
  // fp32 filter over the candidates the tensor-core pass left for each uncertified pair, then
  // float64 for what it cannot decide (PQK_ENCODE_DENSE_FILTER=1: the earlier filter over all
  // 256 codewords of those pairs, kept for comparison runs)
  static const bool dense_filter = [] {
    const char* e = getenv("PQK_ENCODE_DENSE_FILTER");
    return e && e[0] == '1';
  }();
  if (dense_filter) {
    const int fsmem = 2 * 256 * 33 * 4;
    PQK_CUDA_TRY(cudaFuncSetAttribute(encode_filter32_k_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem));
    encode_filter32_k_kernel<<<egrid, 256, fsmem, stream>>>(d_x, n, d, d_cw, m, l, ks, flags, counters, cap, d_codes,
                                                            stride, flags2, counters2, cmask);
    PQK_LAUNCH_CHECK("encode_filter32_k_kernel");
  } else {
    encode_filter32_cand_kernel<<<di.sms * FILTER_GRID, 256, 0, stream>>>(d_x, d, d_cw, m, l, ks, flags, counters, cap, tcmask,
                                                                 d_codes, stride, flags2, counters2, cmask);
    PQK_LAUNCH_CHECK("encode_filter32_cand_kernel");
  }
  // float64 over the candidates of each remaining pair; every row (all 256 codewords) only
  // when the pair list overflowed
  encode_exact_cand_kernel<<<di.sms * EXACT_GRID, 256, 0, stream>>>(d_x, d, d_cw, m, l, ks, flags2, counters2, cap, cmask,
                                                            d_codes, stride);
  PQK_LAUNCH_CHECK("encode_exact_cand_kernel");
  const int esmem = 2 * 256 * 33 * 4;
  PQK_CUDA_TRY(cudaFuncSetAttribute(encode_exact_k_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, esmem));
  encode_exact_k_kernel<<<egrid, 256, esmem, stream>>>(d_x, n, d, d_cw, m, l, ks, flags2, counters2, cap, d_codes,
                                                       stride, 1);
  PQK_LAUNCH_CHECK("encode_exact_k_kernel");
  encode_stats_kernel<<<1, 1, 0, stream>>>(counters2, flagged_out);  // pairs decided in float64
  PQK_LAUNCH_CHECK("encode_stats_kernel");
  return PQK_OK;
}
}  // namespace

// Tensor-core encoder eligibility and launch (called by pqk_encode_device): dsub in
// {8, 16, 32, 64} (operands resident in shared memory) or a multiple of 32 in [96, 1024]
// (K-streamed), at most one CTA per subspace per SM, 16-byte aligned rows.
int encode_tc_try(const float* d_x, int64_t n, int d, const float* d_cw, int m, int l, uint8_t* d_codes, int stride,
                  unsigned long long* flagged_out, cudaStream_t stream, bool* used) {
  *used = false;
  const int ks = d / m;
  const DevInfo& di = dev_info();
  if (n < 1 || n >= ((int64_t)1 << 31) || (d % 4) != 0 || (reinterpret_cast<uintptr_t>(d_x) & 15) ||
      m > di.sms)
    return PQK_OK;
  int rc = PQK_OK;
  switch (ks) {
    case 8:
    case 16:
      if ((size_t)enc::Geo<16>::SMEM > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tc<16>(d_x, n, d, d_cw, m, l, ks, d_codes, stride, flagged_out, stream);
      break;
    case 32:
      if ((size_t)enc::Geo<32>::SMEM > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tc<32>(d_x, n, d, d_cw, m, l, ks, d_codes, stride, flagged_out, stream);
      break;
    case 64:
      if ((size_t)enc::Geo<64>::SMEM > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tc<64>(d_x, n, d, d_cw, m, l, ks, d_codes, stride, flagged_out, stream);
      break;
    default:
      // long subspaces: K-streamed kernel (codebook chunks through shared memory)
      if (ks % enc::kKC != 0 || ks < 96 || ks > 1024 || (size_t)enc::GeoK<false>::SMEM > (size_t)di.smem_optin) return PQK_OK;
      rc = launch_encode_tck(d_x, n, d, d_cw, m, l, ks, d_codes, stride, flagged_out, stream);
  }
  if (rc == PQK_OK) *used = true;
  return rc;
}

}  // namespace pqk
