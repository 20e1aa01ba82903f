// pqk_probe.cu — measured ceilings for the bench rooflines.
//
// pqk_smem_probe: shared-memory load bandwidth of the whole GPU, measured with the
// instruction mix the assignment scan's ceiling rests on: conflict-free LDS.128 from
// every warp of a CTA, one CTA of 1024 threads per SM (the scan kernels run one
// persistent CTA per SM).  A warp's LDS.128 is 512 B = 4 wavefronts of 128 B; the
// architectural ceiling is 128 B/clk/SM.  The loads are volatile (never hoisted or
// merged), the loaded words are folded into one register per thread and written out
// once so nothing is dead code.  Returns bytes/s measured with CUDA events on `stream`.
//
// pqk_tmem_probe: tensor-memory read bandwidth (tcgen05.ld), the ceiling of the encoder's
// epilogue: every 128-vector item's 128 x 256 fp32 accumulator (128 KB) is read once from
// TMEM, so at dsub = 32 the epilogue reads 8 TMEM bytes per HBM byte.  One CTA per SM
// allocates all 512 columns; 16 warps (4 per TMEM lane quadrant) read 32 lanes x 32
// columns per tcgen05.ld.32x32b.x32, two loads in flight, and fold the words into one
// register.  Returns TMEM bytes/s of the whole GPU.
#include <algorithm>

#include "pqk_common.cuh"
#include "pqk_tc.cuh"

namespace pqk {

constexpr int kProbeThreads = 1024;
constexpr int kProbeSmemBytes = 64 * 1024;  // 4096 16-byte slots

__global__ void __launch_bounds__(kProbeThreads, 1) smem_probe_kernel(int iters, uint32_t* __restrict__ sink) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* w = reinterpret_cast<uint32_t*>(smem);
  for (int i = threadIdx.x; i < kProbeSmemBytes / 4; i += blockDim.x) w[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t base = smem_u32(smem);
  // lane i of a warp reads slot (warp*32 + i + u*256 + it) mod 4096: 32 consecutive 16-byte
  // slots per instruction (conflict-free, 4 wavefronts); the 16 unrolled loads have
  // distinct addresses (identical volatile loads could be merged)
  uint32_t off = (uint32_t)threadIdx.x * 16u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t a = base + ((off + (uint32_t)u * 4096u) & (kProbeSmemBytes - 1));
      uint32_t x, y, z, v;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(v) : "r"(a) : "memory");
      acc ^= x + y + z + v;
    }
    off += 16u;  // walk the buffer (still 32 consecutive slots per warp instruction)
  }
  if (acc == 0x9e3779b9u) sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;  // practically never; keeps acc live
}


constexpr int kTmemProbeWarps = 16;

__device__ __forceinline__ void tmem_ld32x(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__global__ void __launch_bounds__(kTmemProbeWarps * 32, 1) tmem_probe_kernel(int iters, uint32_t* __restrict__ sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t q = (uint32_t)(warp & 3);              // lane quadrant of this warp
  const uint32_t col0 = (uint32_t)(warp >> 2) * 128u;   // 4 warps per quadrant, 128 columns each
  const uint32_t base = tbase + ((32u * q) << 16) + col0;
  uint32_t acc = 0, a[32], b[32];
  for (int it = 0; it < iters; ++it) {
    tmem_ld32x(base, a);
    tmem_ld32x(base + 32u, b);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= a[j] + b[j];
    tmem_ld32x(base + 64u, a);
    tmem_ld32x(base + 96u, b);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= a[j] + b[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
  if (acc == 0x9e3779b9u) sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;  // keeps the loads live
}

}  // namespace pqk

using namespace pqk;

extern "C" int pqk_smem_probe(int32_t device, int32_t iters, double* bytes_per_s, double* ms_out, void* stream) {
  if (!bytes_per_s || iters < 1) return fail(PQK_EINVAL, "pqk_smem_probe: bad arguments");
  PQK_CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  PQK_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cudaStream_t s = (cudaStream_t)stream;
  PQK_CUDA_TRY(cudaFuncSetAttribute(smem_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kProbeSmemBytes));
  uint32_t* sink = nullptr;
  PQK_CUDA_TRY(cudaMallocAsync((void**)&sink, (size_t)sms * kProbeThreads * sizeof(uint32_t), s));
  cudaEvent_t e0, e1;
  PQK_CUDA_TRY(cudaEventCreate(&e0));
  PQK_CUDA_TRY(cudaEventCreate(&e1));
  // warm-up launch (clocks ramp, module load), then the timed one
  smem_probe_kernel<<<sms, kProbeThreads, kProbeSmemBytes, s>>>(std::max(1, iters / 8), sink);
  PQK_LAUNCH_CHECK("smem_probe_kernel");
  // best of three timed launches (the peak is an upper bound: take the fastest)
  float ms = 0.f;
  for (int rep = 0; rep < 3; ++rep) {
    PQK_CUDA_TRY(cudaEventRecord(e0, s));
    smem_probe_kernel<<<sms, kProbeThreads, kProbeSmemBytes, s>>>(iters, sink);
    PQK_LAUNCH_CHECK("smem_probe_kernel");
    PQK_CUDA_TRY(cudaEventRecord(e1, s));
    PQK_CUDA_TRY(cudaEventSynchronize(e1));
    float t = 0.f;
    PQK_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
    ms = rep == 0 ? t : std::min(ms, t);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  PQK_CUDA_TRY(cudaFreeAsync(sink, s));
  PQK_CUDA_TRY(cudaStreamSynchronize(s));
  const double bytes = (double)sms * kProbeThreads * (double)iters * 16.0 * 16.0;
  *bytes_per_s = bytes / (ms * 1e-3);
  if (ms_out) *ms_out = ms;
  return PQK_OK;
}

extern "C" int pqk_tmem_probe(int32_t device, int32_t iters, double* bytes_per_s, double* ms_out, void* stream) {
  if (!bytes_per_s || iters < 1) return fail(PQK_EINVAL, "pqk_tmem_probe: bad arguments");
  PQK_CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  PQK_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* sink = nullptr;
  PQK_CUDA_TRY(cudaMallocAsync((void**)&sink, (size_t)sms * kTmemProbeWarps * 32 * sizeof(uint32_t), s));
  cudaEvent_t e0, e1;
  PQK_CUDA_TRY(cudaEventCreate(&e0));
  PQK_CUDA_TRY(cudaEventCreate(&e1));
  tmem_probe_kernel<<<sms, kTmemProbeWarps * 32, 0, s>>>(std::max(1, iters / 8), sink);
  PQK_LAUNCH_CHECK("tmem_probe_kernel");
  float ms = 0.f;
  for (int rep = 0; rep < 3; ++rep) {
    PQK_CUDA_TRY(cudaEventRecord(e0, s));
    tmem_probe_kernel<<<sms, kTmemProbeWarps * 32, 0, s>>>(iters, sink);
    PQK_LAUNCH_CHECK("tmem_probe_kernel");
    PQK_CUDA_TRY(cudaEventRecord(e1, s));
    PQK_CUDA_TRY(cudaEventSynchronize(e1));
    float t = 0.f;
    PQK_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
    ms = rep == 0 ? t : std::min(ms, t);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  PQK_CUDA_TRY(cudaFreeAsync(sink, s));
  PQK_CUDA_TRY(cudaStreamSynchronize(s));
  // per iteration every warp reads 4 x (32 lanes x 32 columns x 4 B)
  const double bytes = (double)sms * kTmemProbeWarps * (double)iters * 4.0 * 4096.0;
  *bytes_per_s = bytes / (ms * 1e-3);
  if (ms_out) *ms_out = ms;
  return PQK_OK;
}
