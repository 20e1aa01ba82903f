// pqk_ingest.cu — file-format ingest on the device.
//
// The streaming pipeline (paper_1709_03708_b200/io.py) copies raw file bytes into pinned
// buffers and straight to the GPU; these kernels validate and unpack them there, so the
// host never touches individual records:
//   fvecs/bvecs (io.py:50-89): records of [int32 dim | dim x float32 (or uint8)] ->
//     dense float32 rows; the first record (in file order) whose dim differs from the
//     expected one is reported (atomicMin), matching the reference's diagnostic.
//   PQKC payload (io.py:238-266): n x M subindex bytes -> device code rows of stride MP
//     (pad bytes 0); the first byte >= L (in file order) is reported.
#include "pqk_common.cuh"

namespace pqk {
namespace ing {

// err[0] = first bad record (int64 max if none), err[1] = its declared dimension
__global__ void unpack_vecs_kernel(const uint8_t* __restrict__ raw, int64_t n, int dim, int itemsize, int64_t base,
                                   float* __restrict__ out, unsigned long long* __restrict__ err) {
  const int64_t rec_bytes = 4 + (int64_t)itemsize * dim;
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    const uint8_t* rec = raw + r * rec_bytes;
    if (threadIdx.x == 0) {
      const int32_t d = (int32_t)((uint32_t)rec[0] | ((uint32_t)rec[1] << 8) | ((uint32_t)rec[2] << 16) |
                                  ((uint32_t)rec[3] << 24));  // bvecs records need not be aligned
      if (d != dim) {
        const unsigned long long idx = (unsigned long long)(base + r);
        const unsigned long long old = atomicMin(&err[0], idx);
        if (idx < old) atomicExch(&err[1], (unsigned long long)(uint32_t)d);
      }
    }
    float* o = out + r * dim;
    if (itemsize == 4) {  // records are 4 (d + 1) bytes: word aligned, little-endian
      const uint32_t* w = reinterpret_cast<const uint32_t*>(rec) + 1;
      for (int j = threadIdx.x; j < dim; j += blockDim.x) o[j] = __uint_as_float(w[j]);
    } else {
      for (int j = threadIdx.x; j < dim; j += blockDim.x) o[j] = (float)rec[4 + j];
    }
  }
}

// err[0] = first bad byte position (record * m + column) or int64 max, err[1] = its value
__global__ void unpack_codes_kernel(const uint8_t* __restrict__ raw, int64_t n, int m, int l, int64_t base,
                                    uint8_t* __restrict__ out, int stride, unsigned long long* __restrict__ err) {
  const int64_t total = n * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / stride;
    const int c = (int)(t - r * stride);
    uint8_t v = 0;
    if (c < m) {
      v = raw[r * m + c];
      if (v >= l) {
        const unsigned long long pos = (unsigned long long)((base + r) * m + c);
        const unsigned long long old = atomicMin(&err[0], pos);
        if (pos < old) atomicExch(&err[1], (unsigned long long)v);
      }
    }
    out[t] = v;
  }
}

}  // namespace ing
}  // namespace pqk

using namespace pqk;

extern "C" int pqk_unpack_vecs_device(const uint8_t* d_raw, int64_t n, int32_t dim, int32_t itemsize,
                                      int64_t base_record, float* d_out, uint64_t* d_err, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_raw || n < 0 || dim < 1 || (itemsize != 1 && itemsize != 4) || !d_out || !d_err)
    return fail(PQK_EINVAL, "pqk_unpack_vecs_device: bad arguments");
  if (n == 0) return PQK_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(n, 8 * dev_info().sms);
  ing::unpack_vecs_kernel<<<grid, 128, 0, stream>>>(d_raw, n, dim, itemsize, base_record, d_out,
                                                    reinterpret_cast<unsigned long long*>(d_err));
  PQK_LAUNCH_CHECK("unpack_vecs_kernel");
  return PQK_OK;
}

extern "C" int pqk_unpack_codes_device(const uint8_t* d_raw, int64_t n, int32_t m, int32_t l, int64_t base_record,
                                       uint8_t* d_out, int32_t stride, uint64_t* d_err, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!d_raw || n < 0 || m < 1 || l < 1 || l > 256 || !d_out || stride < m || !d_err)
    return fail(PQK_EINVAL, "pqk_unpack_codes_device: bad arguments");
  if (n == 0) return PQK_OK;
  const int64_t total = n * stride;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 8 * dev_info().sms);
  ing::unpack_codes_kernel<<<grid, 256, 0, stream>>>(d_raw, n, m, l, base_record, d_out, stride,
                                                     reinterpret_cast<unsigned long long*>(d_err));
  PQK_LAUNCH_CHECK("unpack_codes_kernel");
  return PQK_OK;
}
