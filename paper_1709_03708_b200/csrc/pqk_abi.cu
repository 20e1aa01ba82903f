// pqk_abi.cu — C-ABI glue: error state, host-side helpers (table scale, numpy
// pairwise-sum plan) and the host-buffer entry points that a binding of the
// reference's AssignStrategy plugin (clustering.py:200-216) calls.
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pqk_common.cuh"

namespace pqk {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
static ProfileEvents g_prof;

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
ProfileEvents& profile_events() { return g_prof; }

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t err, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(err);
  return err == cudaErrorMemoryAllocation ? PQK_ENOMEM : PQK_ECUDA;
}

// ---------------------------------------------------------------------------
// numpy pairwise summation plan (numpy/_core/src/umath/loops_utils.h.src):
//   n <= 128 -> leaf (8-accumulator block sum; n < 8 sequential)
//   else     -> n2 = n/2 - (n/2 % 8); sum(a[:n2]) + sum(a[n2:])
struct PlanNode {
  int64_t off, len;
};

static void plan_levels(int64_t n, std::vector<std::vector<PlanNode>>& levels, int64_t& nleaves) {
  levels.clear();
  nleaves = 0;
  levels.push_back({PlanNode{0, n}});
  while (true) {
    std::vector<PlanNode> next;
    for (const PlanNode& p : levels.back()) {
      if (p.len <= 128) {
        ++nleaves;
        continue;
      }
      int64_t n2 = p.len / 2;
      n2 -= n2 % 8;
      next.push_back(PlanNode{p.off, n2});
      next.push_back(PlanNode{p.off + n2, p.len - n2});
    }
    if (next.empty()) break;
    levels.push_back(std::move(next));
  }
}


// ---------------------------------------------------------------------------
// host-buffer context: one stream and grow-only device buffers per device
struct HostCtx {
  bool init = false;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // D2H of results that are final early (labels)
  cudaEvent_t assigned = nullptr;
  cudaEvent_t codes_ready = nullptr;  // the codes' H2D (copy stream) has landed
  std::mutex mu;
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  Buf raw, codes, centers_raw, centers, t64, t32, t16, labels, sd, ws, stats, hist, counts, newc, rws, vec, cw, obj,
      objws, plan, scale;
  // the last table set uploaded (compared by content: a caller re-running assign or fit
  // steps with the same DistanceTables skips the upload, the scale decision's host sync
  // and the fp16 vote-table build)
  std::vector<double> tab_host;
  int tab_m = 0, tab_l = 0, tab_fp64_only = 0;
  bool tab_t16 = false;
  // pinned staging for results copied out while later work runs (pageable caller buffers
  // would make cudaMemcpyAsync wait for the copy, serialising the host)
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // cached numpy-summation plan for the last n (uploaded into `plan`)
  int64_t plan_n = -1, plan_nleaves = 0, plan_nnodes = 0;
  size_t plan_o_len = 0, plan_o_na = 0, plan_o_nb = 0;
  std::vector<int64_t> plan_depth_start;
};

static HostCtx g_ctx[64];

static int ensure(HostCtx::Buf& b, size_t bytes) {
  if (bytes == 0) bytes = 1;
  if (b.bytes >= bytes) return PQK_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  PQK_CUDA_TRY(cudaMalloc(&b.p, bytes));
  b.bytes = bytes;
  return PQK_OK;
}

static int ctx_begin(int device, HostCtx*& ctx) {
  if (device < 0 || device >= 64) return fail(PQK_EINVAL, "device index out of range");
  PQK_CUDA_TRY(cudaSetDevice(device));
  ctx = &g_ctx[device];
  if (!ctx->init) {
    PQK_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    PQK_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    PQK_CUDA_TRY(cudaEventCreateWithFlags(&ctx->assigned, cudaEventDisableTiming));
    PQK_CUDA_TRY(cudaEventCreateWithFlags(&ctx->codes_ready, cudaEventDisableTiming));
    ctx->init = true;
  }
  return PQK_OK;
}

#define PQK_TRY(expr)            \
  do {                           \
    int _rc = (expr);            \
    if (_rc != PQK_OK) return _rc; \
  } while (0)

// Table statistics on the device (the host-buffer entry points upload the tables anyway):
// out[0] = bits of the largest entry, out[1] = bits of the smallest nonzero entry (both
// nonnegative doubles, so their bit patterns order as uint64), out[2] = entries that are
// NaN, negative or infinite.
__global__ void table_stats_kernel(const double* __restrict__ t, int64_t count, unsigned long long* __restrict__ out) {
  unsigned long long mx = 0ull, mn = 0x7ff0000000000000ull, bad = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = t[i];
    const bool ok = v >= 0.0 && v <= 1.7976931348623157e308;
    bad += !ok;
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    if (ok) {
      mx = b > mx ? b : mx;
      if (v > 0.0) mn = b < mn ? b : mn;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long omx = __shfl_xor_sync(0xffffffffu, mx, o), omn = __shfl_xor_sync(0xffffffffu, mn, o);
    mx = omx > mx ? omx : mx;
    mn = omn < mn ? omn : mn;
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], mx);
    atomicMin(&out[1], mn);
    if (bad) atomicAdd(&out[2], bad);
  }
}

// The exponent / fp64-only decision of pqk_table_scale from the table's extremes.
static void table_scale_decide(double mx, double mn, int32_t* e_out, int32_t* f64_out) {
  *e_out = 0;
  *f64_out = 0;
  if (mx == 0.0) return;
  // keep nonzero entries inside [2^-100, 2^100] after scaling: far from fp32
  // subnormals (relative error bound) and from overflow of sums of up to 2^20 terms.
  int e = 0;
  if (mx > ldexp(1.0, 100) || mn < ldexp(1.0, -100)) {
    int ex = 0;
    std::frexp(mx, &ex);  // mx in [2^(ex-1), 2^ex)
    e = 100 - ex;
  }
  if (ldexp(mx, e) > ldexp(1.0, 100) || ldexp(mn, e) < ldexp(1.0, -100)) {
    *f64_out = 1;
    return;
  }
  *e_out = e;
}

// Upload tables, build the scaled fp32 copy (scale decided on the device) and, for
// L = 256, the fp16 first-stage vote tables; skipped when the content is unchanged.
static int upload_tables(HostCtx* c, const double* tables, int m, int l, int& fp64_only) {
  const int mp = padded_m(m);
  const size_t cnt = (size_t)m * l * l;
  if (c->tab_m == m && c->tab_l == l && c->tab_host.size() == cnt &&
      std::memcmp(c->tab_host.data(), tables, cnt * sizeof(double)) == 0) {
    fp64_only = c->tab_fp64_only;
    return PQK_OK;
  }
  c->tab_m = 0;  // invalid until the upload below completes
  PQK_TRY(ensure(c->t64, cnt * sizeof(double)));
  PQK_TRY(ensure(c->t32, (size_t)mp * l * l * sizeof(float)));
  PQK_TRY(ensure(c->scale, 4 * sizeof(unsigned long long)));
  PQK_CUDA_TRY(cudaMemcpyAsync(c->t64.p, tables, cnt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const unsigned long long init[3] = {0ull, 0x7ff0000000000000ull, 0ull};
  PQK_CUDA_TRY(cudaMemcpyAsync(c->scale.p, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
  const DevInfo& di = dev_info();
  table_stats_kernel<<<std::max(1, std::min((int)((cnt + 255) / 256), 4 * di.sms)), 256, 0, c->stream>>>(
      (const double*)c->t64.p, (int64_t)cnt, (unsigned long long*)c->scale.p);
  PQK_LAUNCH_CHECK("table_stats_kernel");
  unsigned long long st[3];
  PQK_CUDA_TRY(cudaMemcpyAsync(st, c->scale.p, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
  PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (st[2]) return fail(PQK_EINVAL, "table entries must be finite and non-negative");
  double mx, mn;
  std::memcpy(&mx, &st[0], sizeof(double));
  std::memcpy(&mn, &st[1], sizeof(double));  // +inf when there is no nonzero entry
  int32_t e = 0, f64 = 0;
  table_scale_decide(mx, mn, &e, &f64);
  fp64_only = f64;
  PQK_TRY(pqk_tables_to_f32((const double*)c->t64.p, m, l, e, (float*)c->t32.p, c->stream));
  c->tab_t16 = false;
  if (l == 256 && !f64) {
    PQK_TRY(ensure(c->t16, cnt * 2));
    PQK_TRY(pqk_vote_tables16_device((const float*)c->t32.p, m, l, c->t16.p, c->stream));
    c->tab_t16 = true;
  }
  c->tab_host.assign(tables, tables + cnt);
  c->tab_fp64_only = f64;
  c->tab_m = m;
  c->tab_l = l;
  return PQK_OK;
}

// Device -> host copy of a result on `stream`: straight into the caller's buffer when it is
// page-locked, else into the context's pinned staging buffer (finish_d2h copies it out
// after the stream is synchronised).
static bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unknown pointer
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static int start_d2h(HostCtx* c, void* dst, const void* src, size_t bytes, cudaStream_t stream, bool& staged) {
  staged = !host_is_pinned(dst);
  if (!staged) {
    PQK_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
    return PQK_OK;
  }
  if (c->stage_bytes < bytes) {
    if (c->stage) cudaFreeHost(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    PQK_CUDA_TRY(cudaMallocHost(&c->stage, bytes));
    c->stage_bytes = bytes;
  }
  PQK_CUDA_TRY(cudaMemcpyAsync(c->stage, src, bytes, cudaMemcpyDeviceToHost, stream));
  return PQK_OK;
}

static void finish_d2h(HostCtx* c, void* dst, size_t bytes, bool staged) {
  if (staged) std::memcpy(dst, c->stage, bytes);
}

static int upload_codes(HostCtx* c, HostCtx::Buf& rawb, HostCtx::Buf& dst, const uint8_t* h, int64_t n, int m,
                        cudaStream_t stream) {
  const int mp = padded_m(m);
  PQK_TRY(ensure(dst, (size_t)std::max<int64_t>(n, 1) * mp));
  if (n == 0) return PQK_OK;
  if (mp == m) {
    PQK_CUDA_TRY(cudaMemcpyAsync(dst.p, h, (size_t)n * m, cudaMemcpyHostToDevice, stream));
    return PQK_OK;
  }
  PQK_TRY(ensure(rawb, (size_t)n * m));
  PQK_CUDA_TRY(cudaMemcpyAsync(rawb.p, h, (size_t)n * m, cudaMemcpyHostToDevice, stream));
  return pqk_pad_codes_device((const uint8_t*)rawb.p, n, m, (uint8_t*)dst.p, stream);
}
static int upload_codes(HostCtx* c, HostCtx::Buf& rawb, HostCtx::Buf& dst, const uint8_t* h, int64_t n, int m) {
  return upload_codes(c, rawb, dst, h, n, m, c->stream);
}

// The N codes go up on the copy stream first, so that their H2D overlaps the table
// upload, its scale decision (one host sync on the main stream) and the center upload;
// the main stream joins before the assignment.
static int start_codes_upload(HostCtx* c, const uint8_t* h, int64_t n, int m) {
  PQK_TRY(upload_codes(c, c->raw, c->codes, h, n, m, c->copy_stream));
  PQK_CUDA_TRY(cudaEventRecord(c->codes_ready, c->copy_stream));
  return PQK_OK;
}

static bool validate_codes_host(const uint8_t* codes, int64_t n, int m, int l) {
  if (l >= 256) return true;  // every uint8 is a valid subindex
  const size_t cnt = (size_t)n * m;
  for (size_t i = 0; i < cnt; ++i)
    if (codes[i] >= l) return false;
  return true;
}

}  // namespace pqk

using namespace pqk;

extern "C" int pqk_abi_version(void) { return PQK_ABI_VERSION; }

extern "C" const char* pqk_last_error(void) { return g_last_error.c_str(); }

extern "C" int64_t pqk_launch_count(void) { return g_launches.load(); }

extern "C" int pqk_set_profile_events(void* before_scan, void* after_scan) {
  g_prof.before = (cudaEvent_t)before_scan;
  g_prof.after = (cudaEvent_t)after_scan;
  return PQK_OK;
}

extern "C" int pqk_device_info(int32_t device, int32_t* sm_count, int32_t* smem_optin_bytes) {
  int n = 0;
  PQK_CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(PQK_EINVAL, "device index out of range");
  int v = 0;
  PQK_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (sm_count) *sm_count = v;
  PQK_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  if (smem_optin_bytes) *smem_optin_bytes = v;
  return PQK_OK;
}

extern "C" int pqk_table_scale(const double* t, int64_t count, int32_t* exp2_out, int32_t* fp64_only_out) {
  if (!t || count < 0 || !exp2_out || !fp64_only_out) return fail(PQK_EINVAL, "pqk_table_scale: bad arguments");
  // branch-free reduction (vectorises): bad counts NaN / negative / infinite entries
  double mx = 0.0, mn = INFINITY;
  int64_t bad = 0;
  for (int64_t i = 0; i < count; ++i) {
    const double v = t[i];
    bad += !(v >= 0.0 && v <= 1.7976931348623157e308);
    mx = v > mx ? v : mx;
    mn = (v > 0.0 && v < mn) ? v : mn;
  }
  if (bad) return fail(PQK_EINVAL, "table entries must be finite and non-negative");
  table_scale_decide(mx, mn, exp2_out, fp64_only_out);
  return PQK_OK;
}

extern "C" int pqk_pairwise_plan_size(int64_t n, int64_t* nleaves, int32_t* ndepth, int64_t* nnodes) {
  if (n < 1 || !nleaves || !ndepth || !nnodes) return fail(PQK_EINVAL, "pqk_pairwise_plan_size: n must be >= 1");
  std::vector<std::vector<PlanNode>> levels;
  int64_t nl = 0;
  plan_levels(n, levels, nl);
  int64_t nn = 0;
  for (auto& lv : levels) nn += (int64_t)lv.size();
  *nleaves = nl;
  *ndepth = (int32_t)levels.size();
  *nnodes = nn;
  return PQK_OK;
}

extern "C" int pqk_pairwise_plan_build(int64_t n, int64_t* leaf_off, int32_t* leaf_len, int64_t* depth_start,
                                       int32_t* node_a, int32_t* node_b) {
  if (n < 1 || !leaf_off || !leaf_len || !depth_start || !node_a || !node_b)
    return fail(PQK_EINVAL, "pqk_pairwise_plan_build: bad arguments");
  std::vector<std::vector<PlanNode>> levels;
  int64_t nl = 0;
  plan_levels(n, levels, nl);
  int64_t leaf = 0, id = 0;
  for (size_t d = 0; d < levels.size(); ++d) {
    depth_start[d] = id;
    int64_t child = 0;  // position of the next child within level d+1
    for (const PlanNode& p : levels[d]) {
      if (p.len <= 128) {
        leaf_off[leaf] = p.off;
        leaf_len[leaf] = (int32_t)p.len;
        node_a[id] = (int32_t)leaf;
        node_b[id] = -1;
        ++leaf;
      } else {
        node_a[id] = (int32_t)child;
        node_b[id] = (int32_t)(child + 1);
        child += 2;
      }
      ++id;
    }
  }
  depth_start[levels.size()] = id;
  return PQK_OK;
}

extern "C" int pqk_assign_host(const uint8_t* codes, int64_t n, int32_t m, const uint8_t* centers, int64_t k,
                               const double* tables, int32_t l, uint32_t* labels, double* sd_sq, int32_t device) {
  if (m < 1 || l < 2 || l > kMaxL || n < 0) return fail(PQK_EINVAL, "pqk_assign_host: M >= 1 and L in [2, 256]");
  if (k < 1) return fail(PQK_EINVAL, "centers must be non-empty");
  if ((n > 0 && (!codes || !labels)) || !centers || !tables) return fail(PQK_EINVAL, "pqk_assign_host: null pointer");
  if (!validate_codes_host(codes, n, m, l) || !validate_codes_host(centers, k, m, l))
    return fail(PQK_EINVAL, "code indices must lie in [0, L)");
  if (n == 0) return PQK_OK;
  HostCtx* c = nullptr;
  PQK_TRY(ctx_begin(device, c));
  std::lock_guard<std::mutex> lock(c->mu);
  int fp64_only = 0;
  PQK_TRY(start_codes_upload(c, codes, n, m));
  PQK_TRY(upload_tables(c, tables, m, l, fp64_only));
  PQK_TRY(upload_codes(c, c->centers_raw, c->centers, centers, k, m));
  PQK_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->codes_ready, 0));
  PQK_TRY(ensure(c->labels, (size_t)n * sizeof(uint32_t)));
  PQK_TRY(ensure(c->sd, (size_t)n * sizeof(double)));
  const size_t wsb = pqk_assign_workspace_bytes(n, k, m, l);
  PQK_TRY(ensure(c->ws, wsb));
  PQK_TRY(ensure(c->stats, PQK_STATS_LEN * sizeof(int64_t)));
  PQK_TRY(pqk_assign_device((const uint8_t*)c->codes.p, n, m, l, (const uint8_t*)c->centers.p, k,
                            (const double*)c->t64.p, (const float*)c->t32.p, fp64_only, c->ws.p, wsb,
                            (uint32_t*)c->labels.p, (double*)c->sd.p, (int64_t*)c->stats.p, c->stream));
  bool staged = false;
  PQK_TRY(start_d2h(c, labels, c->labels.p, (size_t)n * sizeof(uint32_t), c->stream, staged));
  if (sd_sq)
    PQK_CUDA_TRY(cudaMemcpyAsync(sd_sq, c->sd.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));
  finish_d2h(c, labels, (size_t)n * sizeof(uint32_t), staged);
  return PQK_OK;
}

extern "C" int pqk_encode_host(const float* vectors, int64_t n, int32_t d, const float* codewords, int32_t m,
                               int32_t l, uint8_t* codes, int32_t device) {
  if (m < 1 || d < 1 || d % m != 0 || l < 1 || l > kMaxL || n < 0)
    return fail(PQK_EINVAL, "pqk_encode_host: bad arguments");
  if (n == 0) return PQK_OK;
  HostCtx* c = nullptr;
  PQK_TRY(ctx_begin(device, c));
  std::lock_guard<std::mutex> lock(c->mu);
  PQK_TRY(ensure(c->vec, (size_t)n * d * sizeof(float)));
  PQK_TRY(ensure(c->cw, (size_t)l * d * sizeof(float)));
  PQK_TRY(ensure(c->codes, (size_t)n * m));
  PQK_TRY(ensure(c->stats, PQK_STATS_LEN * sizeof(int64_t)));
  PQK_CUDA_TRY(cudaMemcpyAsync(c->vec.p, vectors, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  PQK_CUDA_TRY(cudaMemcpyAsync(c->cw.p, codewords, (size_t)l * d * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  PQK_TRY(pqk_encode_device((const float*)c->vec.p, n, d, (const float*)c->cw.p, m, l, (uint8_t*)c->codes.p, m,
                            (int64_t*)c->stats.p, c->stream));
  PQK_CUDA_TRY(cudaMemcpyAsync(codes, c->codes.p, (size_t)n * m, cudaMemcpyDeviceToHost, c->stream));
  PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return PQK_OK;
}

extern "C" int pqk_lloyd_step_host(const uint8_t* codes, int64_t n, int32_t m, const uint8_t* centers, int64_t k,
                                   const double* tables, int32_t l, uint32_t* labels, uint8_t* new_centers,
                                   double* obj2, int64_t* stats, int32_t device) {
  if (m < 1 || l < 2 || l > kMaxL || n < 1) return fail(PQK_EINVAL, "pqk_lloyd_step_host: M >= 1, L in [2,256], N >= 1");
  if (k < 1 || k > n) return fail(PQK_EINVAL, "k must be in [1, N]");
  if (!codes || !centers || !tables || !labels || !new_centers || !obj2 || !stats)
    return fail(PQK_EINVAL, "pqk_lloyd_step_host: null pointer");
  HostCtx* c = nullptr;
  PQK_TRY(ctx_begin(device, c));
  std::lock_guard<std::mutex> lock(c->mu);
  const int mp = padded_m(m);
  int fp64_only = 0;
  PQK_TRY(start_codes_upload(c, codes, n, m));
  PQK_TRY(upload_tables(c, tables, m, l, fp64_only));
  PQK_TRY(upload_codes(c, c->centers_raw, c->centers, centers, k, m));
  PQK_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->codes_ready, 0));
  PQK_TRY(ensure(c->labels, (size_t)n * sizeof(uint32_t)));
  PQK_TRY(ensure(c->sd, (size_t)n * sizeof(double)));
  const size_t wsb = pqk_assign_workspace_bytes(n, k, m, l);
  PQK_TRY(ensure(c->ws, wsb));
  PQK_TRY(ensure(c->stats, PQK_STATS_LEN * sizeof(int64_t)));
  PQK_TRY(ensure(c->hist, (size_t)k * m * l * sizeof(int32_t)));
  PQK_TRY(ensure(c->counts, (size_t)k * sizeof(int32_t)));
  PQK_TRY(ensure(c->newc, (size_t)k * mp));
  const size_t rwsb = pqk_repair_workspace_bytes(n, k);
  PQK_TRY(ensure(c->rws, rwsb));
  // objective plan (depends on n only; built and uploaded once per n)
  if (c->plan_n != n) {
    int64_t nl = 0, nn = 0;
    int32_t nd = 0;
    PQK_TRY(pqk_pairwise_plan_size(n, &nl, &nd, &nn));
    std::vector<int64_t> leaf_off(nl), depth_start(nd + 1);
    std::vector<int32_t> leaf_len(nl), na(nn), nb(nn);
    PQK_TRY(pqk_pairwise_plan_build(n, leaf_off.data(), leaf_len.data(), depth_start.data(), na.data(), nb.data()));
    c->plan_o_len = align_up(nl * sizeof(int64_t), 256);
    c->plan_o_na = c->plan_o_len + align_up(nl * sizeof(int32_t), 256);
    c->plan_o_nb = c->plan_o_na + align_up(nn * sizeof(int32_t), 256);
    PQK_TRY(ensure(c->plan, c->plan_o_nb + nn * sizeof(int32_t)));
    char* p = (char*)c->plan.p;
    PQK_CUDA_TRY(cudaMemcpyAsync(p, leaf_off.data(), nl * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    PQK_CUDA_TRY(cudaMemcpyAsync(p + c->plan_o_len, leaf_len.data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice,
                                 c->stream));
    PQK_CUDA_TRY(cudaMemcpyAsync(p + c->plan_o_na, na.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    PQK_CUDA_TRY(cudaMemcpyAsync(p + c->plan_o_nb, nb.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));  // host vectors go out of scope
    c->plan_n = n;
    c->plan_nleaves = nl;
    c->plan_nnodes = nn;
    c->plan_depth_start = depth_start;
  }
  const int64_t nleaves = c->plan_nleaves, nnodes = c->plan_nnodes;
  const int32_t ndepth = (int32_t)c->plan_depth_start.size() - 1;
  const int64_t* depth_start_h = c->plan_depth_start.data();
  char* pb = (char*)c->plan.p;
  const size_t o_len = c->plan_o_len, o_na = c->plan_o_na, o_nb = c->plan_o_nb;
  const size_t owsb = pqk_objective_workspace_bytes(nleaves, nnodes);
  PQK_TRY(ensure(c->objws, owsb));
  PQK_TRY(ensure(c->obj, 2 * sizeof(double)));

  int64_t* dstats = (int64_t*)c->stats.p;
  PQK_CUDA_TRY(cudaMemsetAsync(dstats, 0, PQK_STATS_LEN * sizeof(int64_t), c->stream));
  PQK_TRY(pqk_assign_device((const uint8_t*)c->codes.p, n, m, l, (const uint8_t*)c->centers.p, k,
                            (const double*)c->t64.p, (const float*)c->t32.p, fp64_only, c->ws.p, wsb,
                            (uint32_t*)c->labels.p, (double*)c->sd.p, dstats, c->stream));
  // labels are final once assigned: copy them out on the side while the update runs
  PQK_CUDA_TRY(cudaEventRecord(c->assigned, c->stream));
  PQK_CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->assigned, 0));
  bool staged = false;
  PQK_TRY(start_d2h(c, labels, c->labels.p, (size_t)n * sizeof(uint32_t), c->copy_stream, staged));
  PQK_TRY(pqk_objective_device((const double*)c->sd.p, n, nleaves, ndepth, (const int64_t*)pb,
                               (const int32_t*)(pb + o_len), depth_start_h, (const int32_t*)(pb + o_na),
                               (const int32_t*)(pb + o_nb), c->objws.p, owsb, (double*)c->obj.p, c->stream));
  PQK_TRY(pqk_histogram_device((const uint8_t*)c->codes.p, n, m, l, (const uint32_t*)c->labels.p, k,
                               (uint32_t*)c->hist.p, (uint32_t*)c->counts.p, c->stream));
  PQK_TRY(pqk_vote16_device((const uint32_t*)c->hist.p, (const uint32_t*)c->counts.p, k, m, l,
                            (const double*)c->t64.p, fp64_only ? nullptr : (const float*)c->t32.p,
                            c->tab_t16 ? c->t16.p : nullptr, (uint8_t*)c->newc.p, dstats, c->stream));
  int64_t hstats[PQK_STATS_LEN];
  PQK_CUDA_TRY(cudaMemcpyAsync(hstats, dstats, sizeof(hstats), cudaMemcpyDeviceToHost, c->stream));
  PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (hstats[PQK_STAT_EMPTY] > 0) {
    PQK_TRY(pqk_repair_device((const double*)c->sd.p, (const uint8_t*)c->codes.p, n, m, (const uint32_t*)c->counts.p,
                              k, (uint8_t*)c->newc.p, c->rws.p, rwsb, dstats, c->stream));
  }
  PQK_CUDA_TRY(cudaMemcpyAsync(obj2, c->obj.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  PQK_CUDA_TRY(cudaMemcpyAsync(stats, dstats, PQK_STATS_LEN * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  if (mp == m) {
    PQK_CUDA_TRY(cudaMemcpyAsync(new_centers, c->newc.p, (size_t)k * m, cudaMemcpyDeviceToHost, c->stream));
    PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));
  } else {
    std::vector<uint8_t> tmp((size_t)k * mp);
    PQK_CUDA_TRY(cudaMemcpyAsync(tmp.data(), c->newc.p, tmp.size(), cudaMemcpyDeviceToHost, c->stream));
    PQK_CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < k; ++i) std::memcpy(new_centers + i * m, tmp.data() + i * mp, m);
  }
  PQK_CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
  finish_d2h(c, labels, (size_t)n * sizeof(uint32_t), staged);
  return PQK_OK;
}

extern "C" int pqk_host_release(int32_t device) {
  if (device < 0 || device >= 64) return fail(PQK_EINVAL, "device index out of range");
  HostCtx& c = g_ctx[device];
  if (!c.init) return PQK_OK;
  std::lock_guard<std::mutex> lock(c.mu);
  PQK_CUDA_TRY(cudaSetDevice(device));
  HostCtx::Buf* bufs[] = {&c.raw, &c.codes, &c.centers_raw, &c.centers, &c.t64, &c.t32,   &c.t16,
                          &c.labels, &c.sd, &c.ws,  &c.stats,       &c.hist,    &c.counts, &c.newc, &c.rws,
                          &c.vec, &c.cw,    &c.obj, &c.objws,       &c.plan,    &c.scale};
  for (auto* b : bufs) {
    if (b->p) cudaFree(b->p);
    b->p = nullptr;
    b->bytes = 0;
  }
  if (c.stage) cudaFreeHost(c.stage);
  c.stage = nullptr;
  c.stage_bytes = 0;
  c.tab_host.clear();
  c.tab_host.shrink_to_fit();
  c.tab_m = c.tab_l = 0;
  c.tab_t16 = false;
  cudaStreamDestroy(c.stream);
  cudaStreamDestroy(c.copy_stream);
  cudaEventDestroy(c.assigned);
  cudaEventDestroy(c.codes_ready);
  c.stream = c.copy_stream = nullptr;
  c.assigned = c.codes_ready = nullptr;
  c.init = false;
  c.plan_n = -1;
  c.plan_depth_start.clear();
  return PQK_OK;
}
