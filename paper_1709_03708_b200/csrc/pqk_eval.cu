// pqk_eval.cu — original-space evaluation on sm_100a.
//
// baselines.cluster_means (baselines.py:26-37) and original_space_error (:385-413),
// bit-identical to numpy:
//   counts = bincount(labels)
//   sums[k][d] = bincount(labels, weights=points[:, d])   -> each (cluster, dim) sum adds its
//                members in increasing point index, starting from 0.0, in float64
//   means = sums / counts (rows of empty clusters stay 0)
//   sq[i] = np.sum((points[i] - means[labels[i]])**2)    -> numpy pairwise sum of the row
//   error = np.mean(np.sqrt(sq))                          -> pqk_objective_device's tree
//
// The member lists come from a stable LSD radix sort of the labels (8-bit digits: per-tile
// histograms, an exclusive scan, a stable scatter ranked with __match_any_sync), so one
// warp per cluster can walk its members in index order with coalesced row reads.
#include "pqk_common.cuh"

namespace pqk {
namespace ev {

constexpr int kTile = 1024;
constexpr int kSortThreads = 256;
constexpr int kRounds = kTile / kSortThreads;
constexpr int kScanBlock = 1024;  // elements per block in the exclusive scan (256 threads x 4)
constexpr int kMeansBatch = 4;    // member rows loaded ahead of their (ordered) additions

__global__ void __launch_bounds__(kSortThreads) rs_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                              uint32_t* __restrict__ hist, int nb) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int i = threadIdx.x; i < kTile; i += kSortThreads) {
    const int64_t e = base + i;
    if (e < n) atomicAdd(&h[(keys[e] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// stable scatter of one tile: an element's rank among equal digits counts the tile's
// earlier elements (previous rounds, lower warps of this round, lower lanes of this warp)
__global__ void __launch_bounds__(kSortThreads) rs_scatter_kernel(const uint32_t* __restrict__ kin,
                                                                 const uint32_t* __restrict__ vin,
                                                                 uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                                 int64_t n, int shift, const uint32_t* __restrict__ offs,
                                                                 int nb) {
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kSortThreads / 32][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  run[tid] = offs[(size_t)tid * nb + blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int r = 0; r < kRounds; ++r) {
    for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int64_t e = base + (int64_t)r * kSortThreads + tid;
    const bool valid = e < n;
    const uint32_t key = valid ? kin[e] : 0u;
    const uint32_t val = valid ? vin[e] : 0u;
    const uint32_t dg = valid ? ((key >> shift) & 255u) : 256u + (uint32_t)lane;  // invalid lanes match nothing
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const unsigned lower = peers & ((1u << lane) - 1u);
    if (valid && lower == 0) wcnt[warp][dg] = (uint32_t)__popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pos = run[dg] + (uint32_t)__popc(lower);
      for (int w = 0; w < warp; ++w) pos += wcnt[w][dg];
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) add += wcnt[w][tid];
    run[tid] += add;
    __syncthreads();
  }
}

// exclusive scan of uint32 (counts < 2^32): per-block scans plus block offsets
__global__ void __launch_bounds__(256) scan_block_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                         int64_t n, uint32_t* __restrict__ block_sums) {
  __shared__ uint32_t s[kScanBlock];
  __shared__ uint32_t wsum[8];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kScanBlock; i += 256) s[i] = base + i < n ? in[base + i] : 0u;
  __syncthreads();
  // each thread owns 4 consecutive elements
  uint32_t v[4], t = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j] = t;
    t += s[4 * tid + j];
  }
  uint32_t incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += wsum[w];
  const uint32_t excl = woff + incl - t;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t e = base + 4 * tid + j;
    if (e < n) out[e] = excl + v[j];
  }
  if (tid == 255) block_sums[blockIdx.x] = woff + incl;
}

__global__ void scan_add_kernel(uint32_t* __restrict__ out, int64_t n, const uint32_t* __restrict__ block_offs) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) out[e] += block_offs[e / kScanBlock];
}

__global__ void iota_kernel(uint32_t* __restrict__ v, int64_t n) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) v[e] = (uint32_t)e;
}

__global__ void label_count_kernel(const int32_t* __restrict__ labels, int64_t n, uint32_t* __restrict__ counts) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) atomicAdd(&counts[labels[e]], 1u);
}

// one warp per cluster: lanes own dimensions (4 per lane per 128-dim slab), members are
// visited in increasing point index (the stably sorted order), sums start from 0.0
template <typename T>
__global__ void __launch_bounds__(256) cluster_means_kernel(const T* __restrict__ x, int d,
                                                           const uint32_t* __restrict__ order,
                                                           const uint32_t* __restrict__ seg,
                                                           const uint32_t* __restrict__ counts, int k,
                                                           double* __restrict__ means) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= k) return;
  const uint32_t start = seg[c], cnt = counts[c];
  for (int d0 = 0; d0 < d; d0 += 128) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t j0 = 0; j0 < cnt; j0 += 32) {
      const uint32_t nj = min(32u, cnt - j0);
      const uint32_t my_row = lane < (int)nj ? order[start + j0 + lane] : 0u;
      for (uint32_t j = 0; j < nj; j += kMeansBatch) {
        // rows j..j+kMeansBatch-1: loads first (memory-level parallelism), then the adds in
        // member order
        T v[kMeansBatch][4];
#pragma unroll
        for (int q = 0; q < kMeansBatch; ++q) {
          const uint32_t row = __shfl_sync(0xffffffffu, my_row, (int)min(j + q, nj - 1));
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int dim = d0 + lane + 32 * u;
            v[q][u] = (j + q < nj && dim < d) ? x[(size_t)row * d + dim] : (T)0;
          }
        }
#pragma unroll
        for (int q = 0; q < kMeansBatch; ++q)
          if (j + q < nj) {
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = __dadd_rn(acc[u], (double)v[q][u]);
          }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int dim = d0 + lane + 32 * u;
      if (dim < d) means[(size_t)c * d + dim] = cnt ? __ddiv_rn(acc[u], (double)cnt) : 0.0;
    }
  }
}

// numpy pairwise_sum of one row by a group of 8 lanes: lane j of the group owns numpy's
// accumulator r[j] (elements j, j + 8, j + 16, ... added in order), the 8 accumulators are
// combined as ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) by xor-shuffles (IEEE
// addition is commutative, so every lane ends with the same value), the tail (n % 8) and
// rows shorter than 8 are added in order; rows longer than 128 split as numpy does.
template <typename F>
__device__ double np_pairwise8(const F& f, int off, int n, int j) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(off + i));
    return r;
  }
  if (n <= 128) {
    double r = f(off + j);
    const int full = n - (n % 8);
    for (int i = 8; i < full; i += 8) r = __dadd_rn(r, f(off + i + j));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    for (int i = full; i < n; ++i) r = __dadd_rn(r, f(off + i));
    return r;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise8(f, off, n2, j), np_pairwise8(f, off + n2, n - n2, j));
}

template <typename T>
struct SqDiff {
  const T* xr;
  const double* mr;
  __device__ double operator()(int k) const {
    const double df = __dsub_rn((double)xr[k], mr[k]);
    return __dmul_rn(df, df);
  }
};

// sq[i] for 4 rows per warp (8 lanes per row; loads of 8 consecutive elements per row)
template <typename T>
__global__ void __launch_bounds__(256) assigned_sq_kernel(const T* __restrict__ x, int64_t n, int d,
                                                         const double* __restrict__ centers,
                                                         const int32_t* __restrict__ labels, double* __restrict__ sq) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
  const bool valid = row < n;
  const int64_t rr = valid ? row : n - 1;  // whole warps stay convergent for the shuffles
  const SqDiff<T> f{x + rr * d, centers + (size_t)labels[rr] * d};
  const double v = np_pairwise8(f, 0, d, lane & 7);
  if (valid && (lane & 7) == 0) sq[row] = v;
}

}  // namespace ev

namespace {
struct SortWs {
  uint32_t *k0, *v0, *k1, *v1, *hist, *scan_tmp;
  size_t hist_n;
};

size_t scan_ws_elems(int64_t n) {
  size_t total = 0;
  while (n > 1) {
    n = (n + ev::kScanBlock - 1) / ev::kScanBlock;
    total += (size_t)n + 1;
  }
  return total + 4;
}

int exclusive_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp, cudaStream_t stream) {
  using namespace ev;
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  uint32_t* sums = tmp;
  scan_block_kernel<<<(unsigned)nb, 256, 0, stream>>>(in, out, n, sums);
  PQK_LAUNCH_CHECK("scan_block_kernel");
  if (nb > 1) {
    uint32_t* offs = sums + nb;
    const int rc = exclusive_scan(sums, offs, nb, offs + nb, stream);
    if (rc != PQK_OK) return rc;
    scan_add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(out, n, offs);
    PQK_LAUNCH_CHECK("scan_add_kernel");
  }
  return PQK_OK;
}
}  // namespace

}  // namespace pqk

using namespace pqk;

namespace {
size_t means_ws_bytes(int64_t n, int32_t k) {
  const int64_t nb = (n + ev::kTile - 1) / ev::kTile;
  const size_t hist_n = (size_t)256 * nb;
  return align_up((size_t)n * 4, 256) * 4                                  // keys / values ping-pong
         + align_up(hist_n * 4, 256) * 2                                   // histograms + scanned
         + align_up((size_t)k * 4, 256) * 2                                // counts (u32) + segment starts
         + align_up(scan_ws_elems(std::max<int64_t>(hist_n, k)) * 4 * 2, 256) + 1024;
}
}  // namespace

extern "C" size_t pqk_cluster_means_workspace_bytes(int64_t n, int32_t k) {
  if (n < 1 || k < 1) return 0;
  return means_ws_bytes(n, k);
}

// means[k][d] = float64 mean of the points labelled k (0 for empty k); counts[k] optional.
// x is float32 (dtype 0) or float64 (dtype 1), row-major (n, d); labels in [0, k).
extern "C" int pqk_cluster_means_device(const void* d_x, int32_t dtype, int64_t n, int32_t d, const int32_t* d_labels,
                                        int32_t k, double* d_means, int32_t* d_counts, void* d_ws, size_t ws_bytes,
                                        void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_x || n < 1 || n > 0xffffffffLL || d < 1 || !d_labels || k < 1 || !d_means || !d_ws || (dtype != 0 && dtype != 1))
    return fail(PQK_EINVAL, "pqk_cluster_means_device: bad arguments");
  if (ws_bytes < means_ws_bytes(n, k)) return fail(PQK_EINVAL, "pqk_cluster_means_device: workspace too small");
  using namespace ev;
  const int64_t nb = (n + kTile - 1) / kTile;
  const size_t hist_n = (size_t)256 * nb;
  char* p = static_cast<char*>(d_ws);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += align_up(bytes, 256);
    return reinterpret_cast<uint32_t*>(q);
  };
  uint32_t* k0 = take((size_t)n * 4);
  uint32_t* v0 = take((size_t)n * 4);
  uint32_t* k1 = take((size_t)n * 4);
  uint32_t* v1 = take((size_t)n * 4);
  uint32_t* hist = take(hist_n * 4);
  uint32_t* hscan = take(hist_n * 4);
  uint32_t* cnt = take((size_t)k * 4);
  uint32_t* seg = take((size_t)k * 4);
  uint32_t* tmp = take(scan_ws_elems(std::max<int64_t>(hist_n, k)) * 4 * 2);

  const unsigned g256 = (unsigned)((n + 255) / 256);
  PQK_CUDA_TRY(cudaMemcpyAsync(k0, d_labels, (size_t)n * 4, cudaMemcpyDeviceToDevice, stream));
  iota_kernel<<<g256, 256, 0, stream>>>(v0, n);
  PQK_LAUNCH_CHECK("iota_kernel");
  int bits = 1;
  while (bits < 31 && ((int64_t)1 << bits) < (int64_t)k) ++bits;
  for (int shift = 0; shift < bits; shift += 8) {
    rs_hist_kernel<<<(unsigned)nb, kSortThreads, 0, stream>>>(k0, n, shift, hist, (int)nb);
    PQK_LAUNCH_CHECK("rs_hist_kernel");
    const int rc = exclusive_scan(hist, hscan, (int64_t)hist_n, tmp, stream);
    if (rc != PQK_OK) return rc;
    rs_scatter_kernel<<<(unsigned)nb, kSortThreads, 0, stream>>>(k0, v0, k1, v1, n, shift, hscan, (int)nb);
    PQK_LAUNCH_CHECK("rs_scatter_kernel");
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  PQK_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)k * 4, stream));
  label_count_kernel<<<g256, 256, 0, stream>>>(d_labels, n, cnt);
  PQK_LAUNCH_CHECK("label_count_kernel");
  const int rc = exclusive_scan(cnt, seg, k, tmp, stream);
  if (rc != PQK_OK) return rc;
  const unsigned gk = (unsigned)((k + 7) / 8);
  if (dtype == 0)
    cluster_means_kernel<float><<<gk, 256, 0, stream>>>(static_cast<const float*>(d_x), d, v0, seg, cnt, k, d_means);
  else
    cluster_means_kernel<double><<<gk, 256, 0, stream>>>(static_cast<const double*>(d_x), d, v0, seg, cnt, k, d_means);
  PQK_LAUNCH_CHECK("cluster_means_kernel");
  if (d_counts) PQK_CUDA_TRY(cudaMemcpyAsync(d_counts, cnt, (size_t)k * 4, cudaMemcpyDeviceToDevice, stream));
  return PQK_OK;
}

// sq[i] = np.sum((x[i] - centers[labels[i]])**2) (numpy pairwise order), float64
extern "C" int pqk_assigned_sq_device(const void* d_x, int32_t dtype, int64_t n, int32_t d, const double* d_centers,
                                      const int32_t* d_labels, double* d_sq, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_x || n < 1 || d < 1 || !d_centers || !d_labels || !d_sq || (dtype != 0 && dtype != 1))
    return fail(PQK_EINVAL, "pqk_assigned_sq_device: bad arguments");
  const unsigned g = (unsigned)((n * 8 + 255) / 256);  // 8 lanes per row
  if (dtype == 0)
    ev::assigned_sq_kernel<float><<<g, 256, 0, stream>>>(static_cast<const float*>(d_x), n, d, d_centers, d_labels, d_sq);
  else
    ev::assigned_sq_kernel<double><<<g, 256, 0, stream>>>(static_cast<const double*>(d_x), n, d, d_centers, d_labels, d_sq);
  PQK_LAUNCH_CHECK("assigned_sq_kernel");
  return PQK_OK;
}
