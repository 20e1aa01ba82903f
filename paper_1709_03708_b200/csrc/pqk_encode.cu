// pqk_encode.cu — PQ encoder on sm_100a (replaces pq.encode, pq.py:205-231).
//
// code[n][m] = argmin_l sum_d (x_d - c_{l,d})^2 where the reference upcasts the
// float32 vector and codewords to float64 and scipy's cdist("sqeuclidean") sums
// the squares sequentially without FMA (pq.py:114-116, 226-230); lowest l wins
// ties (np.argmin).  The kernel computes the distances in fp32 as a filter and
// keeps the best and runner-up; when the runner-up is not separated from the
// winner by more than the fp32 error bound the (vector, subspace) pair is
// re-decided with the exact fp64 sequential sum.  Certified winners are exactly
// the reference's.
//
// Layout: one CTA per (128-vector tile, subspace); the subspace codebook
// (L x dsub fp32) is staged in shared memory and read as a warp-wide broadcast;
// each thread keeps its sub-vector in registers.
#include <algorithm>

#include "pqk_common.cuh"

namespace pqk {

// pqk_encode_tc.cu: tensor-core encoder; *used = false when the shape is not covered.
int encode_tc_try(const float* d_x, int64_t n, int d, const float* d_cw, int m, int l, uint8_t* d_codes, int stride,
                  unsigned long long* flagged_out, cudaStream_t stream, bool* used);


template <int MAXD>
__global__ void __launch_bounds__(128) encode_kernel(const float* __restrict__ vec, int64_t n, int d,
                                                     const float* __restrict__ cw, int m, int l, int dsub,
                                                     uint8_t* __restrict__ codes, int stride,
                                                     unsigned long long* __restrict__ flagged) {
  extern __shared__ float s_cb[];  // l * dsub (MAXD>0) ; unused for the generic path
  const int mm = blockIdx.y;
  const float* cb = cw + (size_t)mm * l * dsub;
  if (MAXD > 0) {
    for (int i = threadIdx.x; i < l * dsub; i += blockDim.x) s_cb[i] = cb[i];
    __syncthreads();
  }
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* x = vec + i * d + (size_t)mm * dsub;
  const float fmax_ = __int_as_float(0x7f7fffff);
  float b1 = __int_as_float(0x7f800000), b2 = b1;
  int l1 = 0;
  if (MAXD > 0) {
    float xr[MAXD > 0 ? MAXD : 1];
#pragma unroll
    for (int j = 0; j < MAXD; ++j) xr[j] = (j < dsub) ? x[j] : 0.f;
    for (int c = 0; c < l; ++c) {
      const float* cc = s_cb + c * dsub;
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < MAXD; ++j) {
        if (j < dsub) {
          const float df = xr[j] - cc[j];
          acc = __fmaf_rn(df, df, acc);
        }
      }
      if (acc < b1) {
        b2 = b1;
        b1 = acc;
        l1 = c;
      } else if (acc < b2) {
        b2 = acc;
      }
    }
  } else {
    for (int c = 0; c < l; ++c) {
      const float* cc = cb + (size_t)c * dsub;
      float acc = 0.f;
      for (int j = 0; j < dsub; ++j) {
        const float df = x[j] - __ldg(&cc[j]);
        acc = __fmaf_rn(df, df, acc);
      }
      if (acc < b1) {
        b2 = b1;
        b1 = acc;
        l1 = c;
      } else if (acc < b2) {
        b2 = acc;
      }
    }
  }
  // fp32 value of a sum of dsub nonnegative terms: relative error <= (dsub+3)u plus
  // an absolute term for squares flushed below the normal range.
  const double gamma = (double)(dsub + 4) * 5.9604644775390625e-08;  // 2^-24
  const double absl = (double)dsub * 2.350988701644575e-38;          // 2^-125
  // certified only with a finite winner and a finite, clearly separated runner-up
  // (l == 1: a single finite candidate); non-finite inputs go to the exact path
  bool cert = (l == 1) && b1 <= fmax_;
  if (l > 1 && b1 <= fmax_ && b2 <= fmax_) cert = (double)b2 > ((double)b1 + absl) * (1.0 + 4.0 * gamma);
  if (!cert) {
    // exact: float64 sequential sum, separate multiply and add (scipy cdist order),
    // np.argmin order (first NaN wins, else lowest index among equal values)
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bl = 0x7fffffff;
    const float* cbg = cb;
    for (int c = 0; c < l; ++c) {
      const float* cc = cbg + (size_t)c * dsub;
      double acc = 0.0;
      for (int j = 0; j < dsub; ++j) {
        const double df = __dsub_rn((double)x[j], (double)__ldg(&cc[j]));
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
      if (argmin_less(acc, c, best, bl)) {
        best = acc;
        bl = c;
      }
    }
    l1 = bl;
    atomicAdd(flagged, 1ull);
  }
  codes[i * stride + mm] = (uint8_t)l1;
}

}  // namespace pqk

using namespace pqk;

extern "C" int pqk_encode_device(const float* d_vectors, int64_t n, int32_t d, const float* d_codewords, int32_t m,
                                 int32_t l, uint8_t* d_codes, int32_t code_stride, int64_t* d_stats, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (m < 1 || d < 1 || d % m != 0 || l < 1 || l > kMaxL || n < 0 || code_stride < m || !d_stats)
    return fail(PQK_EINVAL, "pqk_encode_device: bad arguments");
  if (n == 0) return PQK_OK;
  if (m > 65535) return fail(PQK_EUNSUPPORTED, "pqk_encode_device: too many subspaces");
  const int dsub = d / m;
  unsigned long long* flagged = reinterpret_cast<unsigned long long*>(d_stats + 20);
  PQK_CUDA_TRY(cudaMemsetAsync(flagged, 0, sizeof(unsigned long long), stream));
  if (code_stride > m) PQK_CUDA_TRY(cudaMemsetAsync(d_codes, 0, (size_t)n * code_stride, stream));
  // tcgen05 path for the shapes it covers (dsub in {16,32,64}, operands fit in smem);
  // PQK_ENCODE_SIMT=1 forces the SIMT kernel (used by tests to cross-check both paths)
  static const bool force_simt = [] {
    const char* e = getenv("PQK_ENCODE_SIMT");
    return e && e[0] == '1';
  }();
  bool used_tc = false;
  if (!force_simt) {
    const int rc = encode_tc_try(d_vectors, n, d, d_codewords, m, l, d_codes, code_stride, flagged, stream, &used_tc);
    if (rc != PQK_OK) return rc;
  }
  if (used_tc) {
    PQK_CUDA_TRY(cudaMemcpyAsync(d_stats + PQK_STAT_ENCODE_FLAGGED, flagged, sizeof(int64_t),
                                 cudaMemcpyDeviceToDevice, stream));
    return PQK_OK;
  }
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)m);
  const size_t smem = (size_t)l * dsub * sizeof(float);
  if (dsub <= 8) {
    encode_kernel<8><<<grid, 128, smem, stream>>>(d_vectors, n, d, d_codewords, m, l, dsub, d_codes, code_stride, flagged);
  } else if (dsub <= 16) {
    encode_kernel<16><<<grid, 128, smem, stream>>>(d_vectors, n, d, d_codewords, m, l, dsub, d_codes, code_stride, flagged);
  } else if (dsub <= 32) {
    encode_kernel<32><<<grid, 128, smem, stream>>>(d_vectors, n, d, d_codewords, m, l, dsub, d_codes, code_stride, flagged);
  } else {
    encode_kernel<0><<<grid, 128, 0, stream>>>(d_vectors, n, d, d_codewords, m, l, dsub, d_codes, code_stride, flagged);
  }
  PQK_LAUNCH_CHECK("encode_kernel");
  // publish the count into the public slot
  PQK_CUDA_TRY(cudaMemcpyAsync(d_stats + PQK_STAT_ENCODE_FLAGGED, flagged, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                               stream));
  return PQK_OK;
}
