// pqk_binary.cu — the Bk-means baseline on sm_100a.
//
// Reference: baselines.py (binarize :229-250, hamming_to_centers :285-288,
// bkmeans_fit :291-382, majority_center :253-282).  Codes are packed bits, MSB first
// within each byte (np.packbits); device rows are padded to wp in {4, 8, 16, 32} bytes with
// zero bytes (XOR of equal pads is 0, so Hamming distances are unchanged).
//
//   binarize   bit b of x = (x . R[:, b] >= 0) with the float64 projection.  fp32 filter
//              with a rigorous bound (|x| |R_b| (d + 4) 2^-24 + rounding of R to fp32);
//              undecided bits take the exact sign of a double-double dot product.
//   assign     labels = argmin_k popcount(code ^ center_k), lowest k on ties: packed key
//              dist << 24 | k, min over centers tiled through shared memory.
//   update     per-bit majority over a cluster's members: bit = 2 * ones > count (ties
//              give 0); empty clusters are repaired by pqk_repair_device on sd = dist^2
//              (same order as the reference's argmax over dist, lowest index first).
//   objective  pqk_objective_device on sd = dist^2: sums of sqrt(sd) = dist and of dist^2,
//              i.e. np.mean(dist) and np.mean(dist.astype(float64) ** 2).
#include "pqk_common.cuh"

namespace pqk {
namespace bin {

constexpr int kAssignThreads = 256;

// one thread per row; rotation (fp32 copy + fp64) in shared memory, 32 bits per pass
__global__ void __launch_bounds__(128) binarize_kernel(const float* __restrict__ x, int64_t n, int d,
                                                      const double* __restrict__ rot, int bits,
                                                      uint8_t* __restrict__ codes, int stride,
                                                      unsigned long long* __restrict__ exact_count) {
  extern __shared__ float s_r[];  // d x bits, fp32
  for (int i = threadIdx.x; i < d * bits; i += blockDim.x) s_r[i] = (float)rot[i];
  __syncthreads();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= n) return;
  const float* xr = x + row * d;
  float xn2 = 0.f;
  for (int k = 0; k < d; ++k) xn2 = fmaf(xr[k], xr[k], xn2);
  // |sum x_k r_k| error: fp32 FMA chain (d + 2) 2^-24 sum |x_k r32_k| plus the rounding of r to
  // fp32 (2^-24 |x_k r_k|); sum |x_k r_k| <= |x| |r| with |r| <= 1 + 1e-6 (orthonormal columns)
  const float bound = sqrtf(xn2) * 1.001f * (float)(d + 8) * 5.9604644775390625e-08f + 1e-37f;
  for (int b0 = 0; b0 < bits; b0 += 32) {
    const int nb = min(32, bits - b0);
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    for (int k = 0; k < d; ++k) {
      const float xv = xr[k];
      const float* rk = s_r + k * bits + b0;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nb) acc[j] = fmaf(xv, rk[j], acc[j]);
    }
    uint32_t word = 0;  // bit j of this pass at position 31 - j
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j >= nb) break;
      bool one;
      if (fabsf(acc[j]) > bound) {
        one = acc[j] > 0.f;
      } else {
        // exact sign: double-double accumulation (products exact via FMA)
        double s = 0.0, c = 0.0;
        for (int k = 0; k < d; ++k) {
          const double a = (double)xr[k], r = rot[(size_t)k * bits + b0 + j];
          const double p = __dmul_rn(a, r);
          const double pe = __fma_rn(a, r, -p);  // exact product error
          const double t = __dadd_rn(s, p);      // TwoSum(s, p), no contraction
          const double bp = __dsub_rn(t, s);
          const double e = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(p, bp));
          s = t;
          c = __dadd_rn(c, __dadd_rn(e, pe));
        }
        const double v = __dadd_rn(s, c);
        one = v >= 0.0;
        atomicAdd(exact_count, 1ull);
      }
      word |= (one ? 1u : 0u) << (31 - j);
    }
    // bytes b0/8 .. : MSB-first bit order within each byte (np.packbits)
    uint8_t* out = codes + row * stride + b0 / 8;
    for (int byte = 0; byte < (nb + 7) / 8; ++byte) out[byte] = (uint8_t)(word >> (24 - 8 * byte));
  }
}

// labels[i] = argmin_k popcount(codes[i] ^ centers[k]) (lowest k on ties); sd[i] = dist^2
template <int W4>
__global__ void __launch_bounds__(kAssignThreads) hamming_assign_kernel(const uint8_t* __restrict__ codes, int64_t n,
                                                                        const uint8_t* __restrict__ centers, int64_t k,
                                                                        uint32_t* __restrict__ labels,
                                                                        double* __restrict__ sd, int32_t* __restrict__ dist_out) {
  extern __shared__ uint4 s_c4[];
  uint32_t* s_c = reinterpret_cast<uint32_t*>(s_c4);
  constexpr int kTileK = (48 * 1024) / (W4 * 4);
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint32_t x[W4];
#pragma unroll
  for (int w = 0; w < W4; ++w) x[w] = i < n ? reinterpret_cast<const uint32_t*>(codes + i * (W4 * 4))[w] : 0u;
  uint32_t best = 0xffffffffu;
  for (int64_t k0 = 0; k0 < k; k0 += kTileK) {
    const int kt = (int)(k - k0 < (int64_t)kTileK ? k - k0 : (int64_t)kTileK);
    __syncthreads();
    const uint32_t* src = reinterpret_cast<const uint32_t*>(centers + k0 * (W4 * 4));
    for (int j = threadIdx.x; j < kt * W4; j += blockDim.x) s_c[j] = src[j];
    __syncthreads();
    int c = 0;
    for (; c + 1 < kt; c += 2) {
      uint32_t d0 = 0, d1 = 0;
#pragma unroll
      for (int w = 0; w < W4; ++w) {
        d0 += __popc(x[w] ^ s_c[c * W4 + w]);
        d1 += __popc(x[w] ^ s_c[(c + 1) * W4 + w]);
      }
      const uint32_t kc = (uint32_t)(k0 + c);
      best = min(best, min((d0 << 24) | kc, (d1 << 24) | (kc + 1u)));
    }
    if (c < kt) {
      uint32_t d0 = 0;
#pragma unroll
      for (int w = 0; w < W4; ++w) d0 += __popc(x[w] ^ s_c[c * W4 + w]);
      best = min(best, (d0 << 24) | (uint32_t)(k0 + c));
    }
  }
  if (i < n) {
    const uint32_t dist = best >> 24;
    labels[i] = best & 0xffffffu;
    if (sd) sd[i] = (double)(dist * dist);
    if (dist_out) dist_out[i] = (int32_t)dist;
  }
}

// dist[i][k] for every pair (hamming_to_centers); one thread per (i, k)
template <int W4>
__global__ void hamming_matrix_kernel(const uint8_t* __restrict__ codes, int64_t n, const uint8_t* __restrict__ centers,
                                      int64_t k, int32_t* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * k) return;
  const int64_t i = t / k, c = t - i * k;
  const uint32_t* a = reinterpret_cast<const uint32_t*>(codes + i * (W4 * 4));
  const uint32_t* b = reinterpret_cast<const uint32_t*>(centers + c * (W4 * 4));
  int s = 0;
#pragma unroll
  for (int w = 0; w < W4; ++w) s += __popc(a[w] ^ b[w]);
  out[t] = s;
}

// counts[label] and ones[label][b] (atomics: exact integers, order irrelevant)
__global__ void majority_count_kernel(const uint8_t* __restrict__ codes, int64_t n, int wp, int bits,
                                      const uint32_t* __restrict__ labels, int32_t* __restrict__ counts,
                                      int32_t* __restrict__ ones) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t lab = labels[i];
  atomicAdd(&counts[lab], 1);
  const uint8_t* x = codes + i * wp;
  int32_t* o = ones + (size_t)lab * bits;
  for (int byte = 0; byte < bits / 8; ++byte) {
    uint32_t v = x[byte];
    while (v) {
      const int j = 31 - __clz(v);  // bit value 2^j -> bit index 7 - j within the byte
      v &= ~(1u << j);
      atomicAdd(&o[8 * byte + (7 - j)], 1);
    }
  }
}

// new_centers[k] = packbits(2 * ones > count) for filled k, 0 for empty k; EMPTY/FILLED stats
__global__ void majority_center_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ ones, int64_t k,
                                       int wp, int bits, uint8_t* __restrict__ newc,
                                       unsigned long long* __restrict__ acc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= k * wp) return;
  const int64_t kk = t / wp;
  const int byte = (int)(t - kk * wp);
  const int32_t cnt = counts[kk];
  uint8_t v = 0;
  if (cnt > 0 && byte < bits / 8) {
    const int32_t* o = ones + (size_t)kk * bits + 8 * byte;
#pragma unroll
    for (int j = 0; j < 8; ++j) v |= (uint8_t)((2 * o[j] > cnt ? 1 : 0) << (7 - j));
  }
  newc[t] = v;
  if (byte == 0) atomicAdd(&acc[cnt > 0 ? 1 : 0], 1ull);  // [0] empty, [1] filled
}

__global__ void majority_stats_kernel(const unsigned long long* __restrict__ acc, int64_t* __restrict__ stats) {
  stats[PQK_STAT_EMPTY] = (int64_t)acc[0];
  stats[PQK_STAT_FILLED] = (int64_t)acc[1];
}

}  // namespace bin
}  // namespace pqk

using namespace pqk;

extern "C" int pqk_binarize_device(const float* d_x, int64_t n, int32_t d, const double* d_rotation, int32_t bits,
                                   uint8_t* d_codes, int32_t code_stride, int64_t* d_stats, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_x || n < 0 || d < 1 || !d_rotation || bits < 8 || bits % 8 || bits > d || !d_codes || code_stride < bits / 8 ||
      !d_stats)
    return fail(PQK_EINVAL, "pqk_binarize_device: bad arguments");
  if ((size_t)d * bits * 4 > 200 * 1024) return fail(PQK_EUNSUPPORTED, "pqk_binarize_device: rotation too large");
  unsigned long long* exact = reinterpret_cast<unsigned long long*>(d_stats + 16);
  PQK_CUDA_TRY(cudaMemsetAsync(exact, 0, 8, stream));
  if (n == 0) return PQK_OK;
  if (code_stride > bits / 8) PQK_CUDA_TRY(cudaMemsetAsync(d_codes, 0, (size_t)n * code_stride, stream));
  const size_t smem = (size_t)d * bits * 4;
  PQK_CUDA_TRY(cudaFuncSetAttribute(bin::binarize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  bin::binarize_kernel<<<(unsigned)((n + 127) / 128), 128, smem, stream>>>(d_x, n, d, d_rotation, bits, d_codes,
                                                                           code_stride, exact);
  PQK_LAUNCH_CHECK("binarize_kernel");
  PQK_CUDA_TRY(cudaMemcpyAsync(d_stats + PQK_STAT_ENCODE_FLAGGED, exact, 8, cudaMemcpyDeviceToDevice, stream));
  return PQK_OK;
}

extern "C" int pqk_hamming_assign_device(const uint8_t* d_codes, int64_t n, int32_t wp, const uint8_t* d_centers,
                                         int64_t k, uint32_t* d_labels, double* d_sd, int32_t* d_dist, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_codes || n < 0 || !d_centers || k < 1 || k > (1 << 24) || !d_labels ||
      (wp != 4 && wp != 8 && wp != 16 && wp != 32))
    return fail(PQK_EINVAL, "pqk_hamming_assign_device: bad arguments");
  if (n == 0) return PQK_OK;
  const unsigned g = (unsigned)((n + bin::kAssignThreads - 1) / bin::kAssignThreads);
  const size_t smem = 48 * 1024;
  switch (wp) {
    case 4:
      bin::hamming_assign_kernel<1><<<g, bin::kAssignThreads, smem, stream>>>(d_codes, n, d_centers, k, d_labels, d_sd, d_dist);
      break;
    case 8:
      bin::hamming_assign_kernel<2><<<g, bin::kAssignThreads, smem, stream>>>(d_codes, n, d_centers, k, d_labels, d_sd, d_dist);
      break;
    case 16:
      bin::hamming_assign_kernel<4><<<g, bin::kAssignThreads, smem, stream>>>(d_codes, n, d_centers, k, d_labels, d_sd, d_dist);
      break;
    default:
      bin::hamming_assign_kernel<8><<<g, bin::kAssignThreads, smem, stream>>>(d_codes, n, d_centers, k, d_labels, d_sd, d_dist);
  }
  PQK_LAUNCH_CHECK("hamming_assign_kernel");
  return PQK_OK;
}

extern "C" int pqk_hamming_matrix_device(const uint8_t* d_codes, int64_t n, int32_t wp, const uint8_t* d_centers,
                                         int64_t k, int32_t* d_out, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_codes || n < 0 || !d_centers || k < 0 || !d_out || (wp != 4 && wp != 8 && wp != 16 && wp != 32))
    return fail(PQK_EINVAL, "pqk_hamming_matrix_device: bad arguments");
  if (n == 0 || k == 0) return PQK_OK;
  const unsigned g = (unsigned)((n * k + 255) / 256);
  if (wp == 4)
    bin::hamming_matrix_kernel<1><<<g, 256, 0, stream>>>(d_codes, n, d_centers, k, d_out);
  else if (wp == 8)
    bin::hamming_matrix_kernel<2><<<g, 256, 0, stream>>>(d_codes, n, d_centers, k, d_out);
  else if (wp == 16)
    bin::hamming_matrix_kernel<4><<<g, 256, 0, stream>>>(d_codes, n, d_centers, k, d_out);
  else
    bin::hamming_matrix_kernel<8><<<g, 256, 0, stream>>>(d_codes, n, d_centers, k, d_out);
  PQK_LAUNCH_CHECK("hamming_matrix_kernel");
  return PQK_OK;
}

extern "C" int pqk_majority_update_device(const uint8_t* d_codes, int64_t n, int32_t wp, int32_t bits,
                                          const uint32_t* d_labels, int64_t k, int32_t* d_counts, int32_t* d_ones,
                                          uint8_t* d_new_centers, int64_t* d_stats, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_codes || n < 1 || (wp != 4 && wp != 8 && wp != 16 && wp != 32) || bits < 8 || bits % 8 || bits > 8 * wp ||
      !d_labels ||
      k < 1 || !d_counts || !d_ones || !d_new_centers || !d_stats)
    return fail(PQK_EINVAL, "pqk_majority_update_device: bad arguments");
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(d_stats + 16);
  PQK_CUDA_TRY(cudaMemsetAsync(acc, 0, 16, stream));
  PQK_CUDA_TRY(cudaMemsetAsync(d_counts, 0, (size_t)k * 4, stream));
  PQK_CUDA_TRY(cudaMemsetAsync(d_ones, 0, (size_t)k * bits * 4, stream));
  bin::majority_count_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_codes, n, wp, bits, d_labels, d_counts,
                                                                              d_ones);
  PQK_LAUNCH_CHECK("majority_count_kernel");
  bin::majority_center_kernel<<<(unsigned)((k * wp + 255) / 256), 256, 0, stream>>>(d_counts, d_ones, k, wp, bits,
                                                                                    d_new_centers, acc);
  PQK_LAUNCH_CHECK("majority_center_kernel");
  bin::majority_stats_kernel<<<1, 1, 0, stream>>>(acc, d_stats);
  PQK_LAUNCH_CHECK("majority_stats_kernel");
  return PQK_OK;
}
