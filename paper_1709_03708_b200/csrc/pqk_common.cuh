// pqk_common.cuh — shared helpers for the sm_100a PQk-means kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <string>

#include "pqk_b200.h"

namespace pqk {

// ---------------------------------------------------------------------------
// error reporting (thread-local last error; entry points return pqk_status_t)
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);

#define PQK_CUDA_TRY(expr)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::pqk::cuda_fail(_e, #expr); \
  } while (0)

// every kernel launch of the library is followed by exactly one PQK_LAUNCH_CHECK,
// which also counts it (pqk_launch_count)
void count_launch();
#define PQK_LAUNCH_CHECK(what)                              \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return ::pqk::cuda_fail(_e, what); \
    ::pqk::count_launch();                                  \
  } while (0)

// optional events recorded around the assignment scan kernel (bench roofline)
struct ProfileEvents {
  cudaEvent_t before = nullptr, after = nullptr;
};
ProfileEvents& profile_events();

// Record a profile event; inside a CUDA-graph capture it becomes an external event-record
// node so the event fires on every replay.
inline cudaError_t record_profile_event(cudaEvent_t ev, cudaStream_t stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(stream, &st);
  if (e != cudaSuccess) return e;
  return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, stream, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, stream);
}

constexpr int kMaxL = 256;

// Padded subspace count of the device code layout: the assignment scan rotates the
// subspace index across the 4 (MP=4) or 8 (MP>=8) codes of a shared-memory phase, so
// MP must be a multiple of that phase width (see pqk_assign.cu).
inline int padded_m(int m) {
  if (m < 1) return 0;
  if (m <= 4) return 4;
  if (m <= 8) return 8;
  if (m <= 16) return 16;
  if (m <= 32) return 32;
  return ((m + 7) / 8) * 8;  // large M: only the fp64 path
}

// per-device attributes (cached on first use for the current device)
struct DevInfo {
  int sms = 0;
  int smem_optin = 0;
};
DevInfo& dev_info();

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// device helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// latency-critical waiters (the single MMA-issuing thread): spin without a suspend hint
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// one non-blocking test of the phase with this parity
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"  // suspend-time hint (ns)
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Exact float64 accumulate without FMA contraction: acc + t rounded once (numpy's `acc += t`).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// np.argmin order: a NaN is the minimum (the first NaN wins), otherwise value then index.
__device__ __forceinline__ bool argmin_less(double a, int ia, double b, int ib) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return na && (!nb || ia < ib);
  return a < b || (a == b && ia < ib);
}

// 32-bit mixing hash for center-code dedup.
__device__ __forceinline__ uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x7feb352dU;
  h ^= h >> 15;
  h *= 0x846ca68bU;
  h ^= h >> 16;
  return h;
}

}  // namespace pqk
