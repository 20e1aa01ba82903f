// pqk_peer.cu — single-process multi-GPU exchange over peer memory (NVLink / NVSwitch).
//
// The one bulk exchange of a sharded Lloyd iteration is the sum of the G devices'
// K x M x L member histograms and K counts (clustering.py:344-347, :458 over the whole
// job).  In a single process every device can read every other device's buffers
// directly (cudaDeviceEnablePeerAccess; UVA pointers), so the allreduce becomes one
// kernel per device that reads its slice of every peer's histogram over NVLink and
// writes the sum in place (reduce-scatter: each device then votes on its own slice of
// clusters and the new center rows are gathered with peer copies).  Traffic per device:
// (G-1)/G of the histogram bytes read over NVLink, 1/G written locally; no staging
// buffers, no NCCL communicator.  Integer sums: the result is independent of G and of
// the order (bit-identical to the single-GPU histogram).
#include "pqk_common.cuh"

namespace pqk {

constexpr int kMaxPeers = 16;

struct PeerPtrs {
  const uint32_t* p[kMaxPeers];
};

// out[i] = sum_g peers.p[g][i] for i in [0, count); 16-byte vectors when every pointer is
// 16-byte aligned (count % 4 handled by the scalar tail).  `out` may alias peers.p[self]:
// each element is read by the same thread before it is written.
__global__ void __launch_bounds__(512) peer_sum_kernel(PeerPtrs peers, int g, int64_t count, uint32_t* out,
                                                       int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = count >> 2;
    for (int64_t i = tid; i < nv; i += stride) {
      uint4 acc = __ldcv(reinterpret_cast<const uint4*>(peers.p[0]) + i);
      for (int j = 1; j < g; ++j) {
        const uint4 v = __ldcv(reinterpret_cast<const uint4*>(peers.p[j]) + i);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      reinterpret_cast<uint4*>(out)[i] = acc;
    }
    done = nv << 2;
  }
  for (int64_t i = done + tid; i < count; i += stride) {
    uint32_t acc = __ldcv(peers.p[0] + i);
    for (int j = 1; j < g; ++j) acc += __ldcv(peers.p[j] + i);
    out[i] = acc;
  }
}

}  // namespace pqk

using namespace pqk;

extern "C" int pqk_peer_sum_device(const uint32_t* const* peer_ptrs, int32_t g, int64_t count, uint32_t* d_out,
                                   void* stream) {
  if (!peer_ptrs || g < 1 || g > kMaxPeers || count < 0 || (count > 0 && !d_out))
    return fail(PQK_EINVAL, "pqk_peer_sum_device: 1 <= g <= 16 peer buffers");
  if (count == 0) return PQK_OK;
  PeerPtrs pp{};
  bool aligned = ((uintptr_t)d_out & 15) == 0;
  for (int j = 0; j < g; ++j) {
    if (!peer_ptrs[j]) return fail(PQK_EINVAL, "pqk_peer_sum_device: null peer buffer");
    pp.p[j] = peer_ptrs[j];
    aligned = aligned && ((uintptr_t)peer_ptrs[j] & 15) == 0;
  }
  const DevInfo& di = dev_info();
  const int64_t work = aligned ? (count >> 2) : count;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((work + 511) / 512, (int64_t)di.sms * 4));
  peer_sum_kernel<<<blocks, 512, 0, (cudaStream_t)stream>>>(pp, g, count, d_out, aligned ? 1 : 0);
  PQK_LAUNCH_CHECK("peer_sum_kernel");
  return PQK_OK;
}

// Enable peer access between every ordered pair of distinct devices in the list (a device
// listed twice shares its own memory).  Fails with PQK_EUNSUPPORTED if a pair cannot.
extern "C" int pqk_enable_peer_access(const int32_t* devices, int32_t g) {
  if (!devices || g < 1 || g > kMaxPeers) return fail(PQK_EINVAL, "pqk_enable_peer_access: 1 <= g <= 16 devices");
  int cur = 0;
  PQK_CUDA_TRY(cudaGetDevice(&cur));
  for (int a = 0; a < g; ++a) {
    for (int b = 0; b < g; ++b) {
      const int da = devices[a], db = devices[b];
      if (da == db) continue;
      int can = 0;
      PQK_CUDA_TRY(cudaDeviceCanAccessPeer(&can, da, db));
      if (!can) {
        cudaSetDevice(cur);
        return fail(PQK_EUNSUPPORTED, "device " + std::to_string(da) + " cannot access device " +
                                          std::to_string(db) + " (no peer path)");
      }
      PQK_CUDA_TRY(cudaSetDevice(da));
      const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        cudaSetDevice(cur);
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
  PQK_CUDA_TRY(cudaSetDevice(cur));
  return PQK_OK;
}
