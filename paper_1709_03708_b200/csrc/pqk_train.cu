// pqk_train.cu — PQ codebook training on sm_100a.
//
// One Lloyd step of the reference's per-subspace k-means (pq.py:127-152,
// _lloyd_subspace), float64 throughout and bit-identical to numpy/scipy:
//   labels = _nearest(points, centers)          cdist sqeuclidean: sequential sum of
//                                               (x-c)*(x-c), separate sub/mul/add; np.argmin
//   counts = bincount(labels)
//   sums   = _cluster_sums(points, labels, L)   per-dimension bincount with weights: each
//                                               (cluster, dim) sum accumulates its members in
//                                               increasing point index from 0.0
//   centers[filled] = sums / counts
//   own    = np.sum((points - centers[labels])**2, axis=1)   numpy pairwise sum per row
// The empty-codeword reseed (farthest points, lowest index first) is finished by the
// host with pqk_repair_candidates_device over `own`.
#include "pqk_common.cuh"

namespace pqk {

// labels[i] = argmin_l ||x_i - c_l||^2 over the subspace columns [col0, col0+dsub)
template <int MAXD>
__global__ void __launch_bounds__(128) train_nearest_kernel(const float* __restrict__ x, int64_t n, int d, int col0,
                                                            int dsub, const double* __restrict__ centers, int l,
                                                            int use_smem, int32_t* __restrict__ labels) {
  extern __shared__ double s_c[];
  if (use_smem) {
    for (int i = threadIdx.x; i < l * dsub; i += blockDim.x) s_c[i] = centers[i];
    __syncthreads();
  }
  const double* cb = use_smem ? s_c : centers;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* xr = x + i * d + col0;
  double best = __longlong_as_double(0x7ff0000000000000LL);
  int bl = 0x7fffffff;
  if (MAXD > 0) {
    double xv[MAXD > 0 ? MAXD : 1];
#pragma unroll
    for (int k = 0; k < MAXD; ++k) xv[k] = k < dsub ? (double)xr[k] : 0.0;
    for (int c = 0; c < l; ++c) {
      const double* cc = cb + (size_t)c * dsub;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < MAXD; ++k) {
        if (k < dsub) {
          const double df = __dsub_rn(xv[k], cc[k]);
          acc = __dadd_rn(acc, __dmul_rn(df, df));
        }
      }
      if (argmin_less(acc, c, best, bl)) {
        best = acc;
        bl = c;
      }
    }
  } else {
    for (int c = 0; c < l; ++c) {
      const double* cc = cb + (size_t)c * dsub;
      double acc = 0.0;
      for (int k = 0; k < dsub; ++k) {
        const double df = __dsub_rn((double)xr[k], cc[k]);
        acc = __dadd_rn(acc, __dmul_rn(df, df));
      }
      if (argmin_less(acc, c, best, bl)) {
        best = acc;
        bl = c;
      }
    }
  }
  labels[i] = bl;
}

// One warp per codeword k: lanes own dimensions, members are visited in increasing
// point index (ballot over 32 labels at a time), so each (k, dim) sum has numpy's order.
__global__ void __launch_bounds__(256) train_sums_kernel(const float* __restrict__ x, int64_t n, int d, int col0,
                                                         int dsub, const int32_t* __restrict__ labels, int l,
                                                         double* __restrict__ sums, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= l) return;
  for (int d0 = 0; d0 < dsub; d0 += 32) {
    double acc = 0.0;
    int cnt = 0;
    for (int64_t base = 0; base < n; base += 32) {
      const int64_t i = base + lane;
      const int lab = i < n ? labels[i] : -1;
      unsigned bal = __ballot_sync(0xffffffffu, lab == k);
      while (bal) {
        const int j = __ffs(bal) - 1;
        bal &= bal - 1;
        if (d0 + lane < dsub) acc = __dadd_rn(acc, (double)x[(base + j) * d + col0 + d0 + lane]);
        ++cnt;
      }
    }
    if (d0 + lane < dsub) sums[(size_t)k * dsub + d0 + lane] = acc;
    if (d0 == 0 && lane == 0) counts[k] = cnt;
  }
}

__global__ void train_update_kernel(double* __restrict__ centers, const double* __restrict__ sums,
                                    const int32_t* __restrict__ counts, int l, int dsub,
                                    unsigned long long* __restrict__ empty) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= l * dsub) return;
  const int k = i / dsub;
  const int c = counts[k];
  if (c > 0)
    centers[i] = __ddiv_rn(sums[i], (double)c);
  else if (i % dsub == 0)
    atomicAdd(empty, 1ull);
}

// numpy pairwise sum of a row held in registers (loops_utils.h.src), n <= 128 per leaf
__device__ __forceinline__ double np_pairwise_leaf(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) s = __dadd_rn(s, a[i]);
  return s;
}

__device__ double np_pairwise(const double* a, int n) {
  if (n <= 128) return np_pairwise_leaf(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

// own[i] = np.sum((x_i - c_{label_i})**2) for rows of length dsub (<= 1024)
__global__ void __launch_bounds__(128) train_own_kernel(const float* __restrict__ x, int64_t n, int d, int col0,
                                                        int dsub, const double* __restrict__ centers,
                                                        const int32_t* __restrict__ labels, double* __restrict__ own,
                                                        double* __restrict__ scratch,
                                                        const unsigned long long* __restrict__ empty) {
  if (*empty == 0) return;  // only the empty-codeword reseed reads `own`
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* row = scratch + i * dsub;
  const float* xr = x + i * d + col0;
  const double* cc = centers + (size_t)labels[i] * dsub;
  for (int k = 0; k < dsub; ++k) {
    const double df = __dsub_rn((double)xr[k], cc[k]);
    row[k] = __dmul_rn(df, df);
  }
  own[i] = np_pairwise(row, dsub);
}

// DistanceTables (pq.py:254-268): t[m][i][j] = sum_d (c_i - c_j)^2 in float64, the
// difference and square rounded separately and summed in increasing d (scipy cdist /
// the numpy loop of build_distance_tables).  One thread per (i, j).
__global__ void build_tables_kernel(const float* __restrict__ cw, int l, int dsub, double* __restrict__ t) {
  const int mm = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= l * l) return;
  const int i = e / l, j = e - i * l;
  const float* ci = cw + ((size_t)mm * l + i) * dsub;
  const float* cj = cw + ((size_t)mm * l + j) * dsub;
  double acc = 0.0;
  for (int k = 0; k < dsub; ++k) {
    const double df = __dsub_rn((double)ci[k], (double)cj[k]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  t[((size_t)mm * l + i) * l + j] = acc;
}

__global__ void train_stats_kernel(const unsigned long long* __restrict__ empty, int64_t* __restrict__ stats) {
  stats[PQK_STAT_EMPTY] = (int64_t)*empty;
}

}  // namespace pqk

using namespace pqk;

extern "C" size_t pqk_train_workspace_bytes(int64_t n, int32_t dsub) {
  if (n < 1 || dsub < 1) return 0;
  return align_up((size_t)n * dsub * sizeof(double), 256) + 256;
}

extern "C" int pqk_train_step_device(const float* d_x, int64_t n, int32_t d, int32_t col0, int32_t dsub,
                                     double* d_centers, int32_t l, int32_t* d_labels, double* d_sums,
                                     int32_t* d_counts, double* d_own, void* d_ws, size_t ws_bytes, int64_t* d_stats,
                                     void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n < 1 || d < 1 || dsub < 1 || col0 < 0 || col0 + dsub > d || l < 2 || l > kMaxL || dsub > 1024 || !d_stats ||
      !d_ws)
    return fail(PQK_EINVAL, "pqk_train_step_device: bad arguments");
  if (ws_bytes < pqk_train_workspace_bytes(n, dsub)) return fail(PQK_EINVAL, "pqk_train_step_device: workspace too small");
  unsigned long long* empty = reinterpret_cast<unsigned long long*>(d_stats + 16);
  PQK_CUDA_TRY(cudaMemsetAsync(empty, 0, sizeof(unsigned long long), stream));
  const int grid = (int)((n + 127) / 128);
  const size_t cbytes = (size_t)l * dsub * sizeof(double);
  const int use_smem = cbytes <= 96 * 1024;
  const size_t smem = use_smem ? cbytes : 0;
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    PQK_CUDA_TRY(cudaFuncSetAttribute(train_nearest_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    PQK_CUDA_TRY(cudaFuncSetAttribute(train_nearest_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    PQK_CUDA_TRY(cudaFuncSetAttribute(train_nearest_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    PQK_CUDA_TRY(cudaFuncSetAttribute(train_nearest_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr[dev & 63] = true;
  }
  if (dsub <= 8)
    train_nearest_kernel<8><<<grid, 128, smem, stream>>>(d_x, n, d, col0, dsub, d_centers, l, use_smem, d_labels);
  else if (dsub <= 16)
    train_nearest_kernel<16><<<grid, 128, smem, stream>>>(d_x, n, d, col0, dsub, d_centers, l, use_smem, d_labels);
  else if (dsub <= 32)
    train_nearest_kernel<32><<<grid, 128, smem, stream>>>(d_x, n, d, col0, dsub, d_centers, l, use_smem, d_labels);
  else
    train_nearest_kernel<0><<<grid, 128, smem, stream>>>(d_x, n, d, col0, dsub, d_centers, l, use_smem, d_labels);
  PQK_LAUNCH_CHECK("train_nearest_kernel");
  train_sums_kernel<<<(l + 7) / 8, 256, 0, stream>>>(d_x, n, d, col0, dsub, d_labels, l, d_sums, d_counts);
  PQK_LAUNCH_CHECK("train_sums_kernel");
  train_update_kernel<<<(l * dsub + 255) / 256, 256, 0, stream>>>(d_centers, d_sums, d_counts, l, dsub, empty);
  PQK_LAUNCH_CHECK("train_update_kernel");
  train_own_kernel<<<grid, 128, 0, stream>>>(d_x, n, d, col0, dsub, d_centers, d_labels, d_own, (double*)d_ws,
                                              empty);
  PQK_LAUNCH_CHECK("train_own_kernel");
  train_stats_kernel<<<1, 1, 0, stream>>>(empty, d_stats);
  PQK_LAUNCH_CHECK("train_stats_kernel");
  return PQK_OK;
}

extern "C" int pqk_build_tables_device(const float* d_codewords, int32_t m, int32_t l, int32_t dsub, double* d_tables,
                                       void* stream) {
  if (!d_codewords || m < 1 || l < 1 || l > kMaxL || dsub < 1 || !d_tables)
    return fail(PQK_EINVAL, "pqk_build_tables_device: bad arguments");
  const dim3 grid((unsigned)((l * l + 255) / 256), (unsigned)m);
  build_tables_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_codewords, l, dsub, d_tables);
  PQK_LAUNCH_CHECK("build_tables_kernel");
  return PQK_OK;
}
