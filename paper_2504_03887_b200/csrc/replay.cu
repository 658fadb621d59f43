// Batched caching-allocator replay for sm_100a -- host side of the C ABI
// (include/peakmem_b200.h).  The kernels live in replay_device.cuh.

#include <cuda_runtime.h>
#include <stdint.h>

#include "peakmem_b200.h"
#include "replay_device.cuh"

// ---------------------------------------------------------------------------
// Host side of the C ABI.

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(PM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr int kWarps = 12;
constexpr size_t kBucket_host = 32;  // warps (traces in flight) per CTA, 1 CTA / SM
constexpr int kRetryWarps = 1;
constexpr int kMaxRetryWarps = 64;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// workspace = ctl | retry list | retry pools | record table
struct Layout {
  size_t retry_list, gpool, recs, total;
  int nbmax_g;
  int retry_warps;
};

Layout layout_for(int64_t total_events, int64_t max_trace_events,
                  int32_t n_traces) {
  Layout L;
  size_t off = align_up(sizeof(pmb::Ctl), 256);
  L.retry_list = off;
  off = align_up(off + 3 * sizeof(int32_t) * (size_t)(n_traces > 0 ? n_traces : 1),
                 256);
  const int64_t mx = max_trace_events > 0 ? max_trace_events : 1;
  L.nbmax_g = (int)(mx / 8 + 4);
  int warps = n_traces < kMaxRetryWarps ? n_traces : kMaxRetryWarps;
  if (warps < 1) warps = 1;
  L.retry_warps = warps;
  L.gpool = off;
  off = align_up(off + (size_t)warps * pmb::gmem_warp_bytes(L.nbmax_g), 256);
  L.recs = off;
  off = align_up(off + 32 * (size_t)(total_events > 0 ? total_events : 1), 256);
  L.total = off;
  return L;
}

struct Occupancy {
  int sms = 0, per_sm = 0, buckets = 0, warps = 0;
  size_t smem = 0;
  int per_sm1 = 0;  // tier-1 retry kernel
  size_t smem1 = 0;
  int nbmax2 = 0;   // tier-2: one warp with a shared-memory directory
  size_t smem2 = 0;
};

constexpr int kTier1Warps = 8;  // tier 1: a dedicated 32-bucket pool per warp

template <int W>
int setup_kernel(int optin, int cap, int* buckets, size_t* smem, int* per_sm) {
  int b = (int)(((size_t)optin - (size_t)W * 32 * 24 - 256) / (kBucket_host * 24));
  if (cap > 0 && cap < b) b = cap;
  if (b < 2 * W) b = 2 * W;
  *buckets = b;
  *smem = pmb::smem_cta_bytes(b, W);
  cudaError_t e = cudaFuncSetAttribute(
      pmb::replay_smem_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)*smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      per_sm, pmb::replay_smem_kernel<W>, W * 32, *smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy");
  if (*per_sm < 1) return fail(PM_ERR_CUDA, "replay kernel cannot be resident");
  return PM_SUCCESS;
}

// Main pass: one CTA of `warps` warps per SM sharing a bucket pool sized to
// the remaining shared memory (PM_POOL_BUCKETS caps it, PM_REPLAY_WARPS picks
// 12 or 16 warps; 12 measured faster on C3).  Tier 1: 8 warps x 32 dedicated buckets.
int query_occupancy(Occupancy* out) {
  static std::mutex mu;
  static int cached_dev = -1;
  static Occupancy cached;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> g(mu);
  if (cached_dev != dev) {
    Occupancy o;
    e = cudaDeviceGetAttribute(&o.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                               dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    int cap = 0;
    if (const char* env = getenv("PM_POOL_BUCKETS")) cap = atoi(env);
    o.warps = kWarps;
    if (const char* env = getenv("PM_REPLAY_WARPS")) o.warps = atoi(env);
    int rc;
    if (o.warps == 12)
      rc = setup_kernel<12>(optin, cap, &o.buckets, &o.smem, &o.per_sm);
    else {
      o.warps = 16;
      rc = setup_kernel<16>(optin, cap, &o.buckets, &o.smem, &o.per_sm);
    }
    if (rc != PM_SUCCESS) return rc;
    int b1 = 0;
    rc = setup_kernel<kTier1Warps>(optin, kTier1Warps * 32, &b1, &o.smem1,
                                   &o.per_sm1);
    if (rc != PM_SUCCESS) return rc;
    o.nbmax2 = (int)(((size_t)optin - 1024) / (kBucket_host * 24 + 32));
    while (o.nbmax2 > 8 && pmb::gmem_warp_bytes(o.nbmax2) > (size_t)optin) --o.nbmax2;
    o.smem2 = pmb::gmem_warp_bytes(o.nbmax2);
    e = cudaFuncSetAttribute(pmb::replay_dirmem_kernel<1, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)o.smem2);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute tier 2");
    cached = o;
    cached_dev = dev;
  }
  *out = cached;
  return PM_SUCCESS;
}

void keep_pool_mapped() {
  // the default release threshold (0) unmaps the stream-ordered pool at
  // every synchronisation; keep it mapped between calls
  static std::mutex mu;
  static int tuned_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> g(mu);
  if (tuned_dev == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  tuned_dev = dev;
}

}  // namespace

extern "C" {

#ifdef PM_DEBUG_UNIFORM
int pm_debug_nonuniform_line(void) {
  int v = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&v, pmb::g_nonuniform_line, sizeof(int));
  return v;
}
#endif

const char* pm_last_error(void) { return g_last_error.c_str(); }

int pm_version(void) { return 2; }

int pm_replay_workspace_bytes(int64_t total_events, int64_t max_trace_events,
                              int32_t n_traces, size_t* out_bytes) {
  if (!out_bytes || total_events < 0 || max_trace_events < 0 || n_traces < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_workspace_bytes: bad args");
  *out_bytes = layout_for(total_events, max_trace_events, n_traces).total;
  return PM_SUCCESS;
}

}  // extern "C"

namespace {

// pm_replay_batch with optional streamed input: when `ready` is non-null the
// main kernel waits, per trace, for the flag of the group (group_end[g] =
// traces consumed through group g) the copy engine writes after the group.
int replay_batch_impl(const pm_req_t* reqs, const int64_t* trace_offsets,
                      int32_t n_traces, const pm_cfg_t* cfgs,
                      const int32_t* cfg_of_trace, const int32_t* trace_order,
                      pm_result_t* results, int64_t* timeline, void* workspace,
                      size_t workspace_bytes, int64_t total_events,
                      int64_t max_trace_events, void* stream_,
                      const unsigned* group_end, int n_groups,
                      const unsigned* ready) {
  if (n_traces < 0 || total_events < 0 || max_trace_events < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_batch: negative size");
  if (n_traces == 0) return PM_SUCCESS;
  if (!trace_offsets || !cfgs || !results || !workspace ||
      (total_events > 0 && !reqs))
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_batch: null argument");
  if (max_trace_events >= (int64_t)0x7FFFFFFF)
    return fail(PM_ERR_INVALID_ARGUMENT,
                "pm_replay_batch: traces are limited to 2^31-1 requests");
  const Layout L = layout_for(total_events, max_trace_events, n_traces);
  if (workspace_bytes < L.total)
    return fail(PM_ERR_WORKSPACE_TOO_SMALL,
                "pm_replay_batch: workspace smaller than "
                "pm_replay_workspace_bytes()");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  char* base = static_cast<char*>(workspace);
  pmb::Ctl* ctl = reinterpret_cast<pmb::Ctl*>(base);
  int32_t* retry_list = reinterpret_cast<int32_t*>(base + L.retry_list);
  char* gpool = base + L.gpool;
  pmb::u64* recs = reinterpret_cast<pmb::u64*>(base + L.recs);

  Occupancy occ;
  int rc = query_occupancy(&occ);
  if (rc != PM_SUCCESS) return rc;

  cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(pmb::Ctl), stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  int32_t* list1 = retry_list;
  int32_t* list2 = retry_list + n_traces;
  long long want = ((long long)n_traces + occ.warps - 1) / occ.warps;
  long long grid = (long long)occ.per_sm * occ.sms;
  if (want < grid) grid = want;
  if (const char* cap = getenv("PM_MAX_GRID")) {  // debugging aid
    const long long g = atoll(cap);
    if (g > 0 && g < grid) grid = g;
  }
#define PM_LAUNCH_MAIN(W)                                                     \
  pmb::replay_smem_kernel<W><<<(unsigned)grid, W * 32, occ.smem, stream>>>(  \
      reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs, ctl, \
      0, trace_order, n_traces, list1, occ.buckets, group_end, n_groups, ready)
  if (occ.warps == 12)
    PM_LAUNCH_MAIN(12);
  else
    PM_LAUNCH_MAIN(16);
#undef PM_LAUNCH_MAIN
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay_smem_kernel launch");
  // tier 1: dedicated 32-bucket pools (grid sized for the worst case; idle
  // CTAs exit at once when nothing overflowed)
  long long grid1 = (long long)occ.per_sm1 * occ.sms;
  long long want1 = ((long long)n_traces + kTier1Warps - 1) / kTier1Warps;
  if (want1 < grid1) grid1 = want1;
  pmb::replay_smem_kernel<kTier1Warps>
      <<<(unsigned)grid1, kTier1Warps * 32, occ.smem1, stream>>>(
          reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs,
          ctl, 1, list1, 0, list2, kTier1Warps * 32, nullptr, 0, nullptr);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay tier-1 launch");
  {
    int32_t* list3 = retry_list + 2 * (size_t)n_traces;
    long long grid2 = occ.sms;
    if (n_traces < grid2) grid2 = n_traces;
    pmb::replay_dirmem_kernel<1, true><<<(unsigned)grid2, 32, occ.smem2, stream>>>(
        reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs, ctl,
        2, list2, list3, nullptr, occ.nbmax2);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "replay tier-2 launch");
    pmb::replay_dirmem_kernel<kRetryWarps, false>
        <<<L.retry_warps / kRetryWarps, kRetryWarps * 32, 0, stream>>>(
            reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs,
            ctl, 3, list3, nullptr, gpool, L.nbmax_g);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay tier-3 launch");
  return PM_SUCCESS;
}

}  // namespace

extern "C" {

int pm_replay_batch(const pm_req_t* reqs, const int64_t* trace_offsets,
                    int32_t n_traces, const pm_cfg_t* cfgs,
                    const int32_t* cfg_of_trace, const int32_t* trace_order,
                    pm_result_t* results, int64_t* timeline, void* workspace,
                    size_t workspace_bytes, int64_t total_events,
                    int64_t max_trace_events, void* stream_) {
  return replay_batch_impl(reqs, trace_offsets, n_traces, cfgs, cfg_of_trace,
                           trace_order, results, timeline, workspace,
                           workspace_bytes, total_events, max_trace_events,
                           stream_, nullptr, 0, nullptr);
}

int pm_replay_host(const pm_req_t* reqs, const int64_t* trace_offsets,
                   int32_t n_traces, const pm_cfg_t* cfgs, int32_t n_cfgs,
                   const int32_t* cfg_of_trace, pm_result_t* results,
                   int64_t* timeline, void* stream_) {
  if (n_traces < 0 || n_cfgs < 1)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_host: bad counts");
  if (n_traces == 0) return PM_SUCCESS;
  if (!trace_offsets || !cfgs || !results)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_host: null argument");
  const int64_t total = trace_offsets[n_traces] - trace_offsets[0];
  if (trace_offsets[0] != 0 || total < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_host: offsets must start at 0");
  if (total > 0 && !reqs)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_host: null requests");
  int64_t max_ev = 0;
  for (int32_t i = 0; i < n_traces; ++i) {
    int64_t len = trace_offsets[i + 1] - trace_offsets[i];
    if (len < 0) return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_host: offsets decrease");
    if (len > max_ev) max_ev = len;
  }
  if (cfg_of_trace)
    for (int32_t i = 0; i < n_traces; ++i)
      if (cfg_of_trace[i] < 0 || cfg_of_trace[i] >= n_cfgs)
        return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_host: cfg index out of range");
  // Streamed upload: G contiguous trace groups, each copied (copy stream)
  // and then flagged with a 4-byte DMA write; the kernel consumes groups in
  // order, longest trace first within a group, so replay overlaps the H2D.
  const size_t bytes_in = 16 * (size_t)total;
  int G = (int)(bytes_in / (256u << 20));
  if (G < 1) G = 1;
  if (G > 64) G = 64;
  if (G > n_traces) G = n_traces;
  std::vector<int32_t> gfirst(G + 1);
  for (int g = 0; g <= G; ++g) gfirst[g] = (int32_t)(((int64_t)n_traces * g) / G);
  std::vector<int32_t> order(n_traces);
  std::vector<unsigned> group_end(G);
  for (int g = 0; g < G; ++g) {
    for (int32_t i = gfirst[g]; i < gfirst[g + 1]; ++i) order[i] = i;
    std::stable_sort(order.begin() + gfirst[g], order.begin() + gfirst[g + 1],
                     [&](int32_t a, int32_t b) {
                       return trace_offsets[a + 1] - trace_offsets[a] >
                              trace_offsets[b + 1] - trace_offsets[b];
                     });
    group_end[g] = (unsigned)gfirst[g + 1];
  }
  const Layout L = layout_for(total, max_ev, n_traces);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const size_t b_reqs = align_up(16 * (size_t)(total > 0 ? total : 1), 256);
  const size_t b_offs = align_up(8 * (size_t)(n_traces + 1), 256);
  const size_t b_cfgs = align_up(sizeof(pm_cfg_t) * (size_t)n_cfgs, 256);
  const size_t b_cfgof = align_up(4 * (size_t)n_traces, 256);
  const size_t b_order = b_cfgof;
  const size_t b_res = align_up(sizeof(pm_result_t) * (size_t)n_traces, 256);
  const size_t b_tl = timeline ? align_up(16 * (size_t)(total > 0 ? total : 1), 256) : 0;
  const size_t b_grp = align_up(8 * (size_t)G, 256);
  const size_t bytes = b_reqs + b_offs + b_cfgs + b_cfgof + b_order + b_res +
                       b_tl + 2 * b_grp + L.total;
  keep_pool_mapped();
  static unsigned* one = nullptr;  // pinned source of the group flags
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (!one) {
      cudaError_t e = cudaHostAlloc((void**)&one, sizeof(unsigned), cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
      *one = 1u;
    }
  }
  cudaStream_t cs = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
  cudaEvent_t zeroed = nullptr;
  e = cudaEventCreateWithFlags(&zeroed, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    cudaStreamDestroy(cs);
    return cuda_fail(e, "cudaEventCreate");
  }
  void* dmem = nullptr;
  e = cudaMallocAsync(&dmem, bytes, stream);
  if (e != cudaSuccess) {
    cudaEventDestroy(zeroed);
    cudaStreamDestroy(cs);
    return cuda_fail(e, "cudaMallocAsync");
  }
  char* p = static_cast<char*>(dmem);
  pm_req_t* d_reqs = reinterpret_cast<pm_req_t*>(p);
  p += b_reqs;
  int64_t* d_offs = reinterpret_cast<int64_t*>(p);
  p += b_offs;
  pm_cfg_t* d_cfgs = reinterpret_cast<pm_cfg_t*>(p);
  p += b_cfgs;
  int32_t* d_cfgof = reinterpret_cast<int32_t*>(p);
  p += b_cfgof;
  int32_t* d_order = reinterpret_cast<int32_t*>(p);
  p += b_order;
  pm_result_t* d_res = reinterpret_cast<pm_result_t*>(p);
  p += b_res;
  int64_t* d_tl = timeline ? reinterpret_cast<int64_t*>(p) : nullptr;
  p += b_tl;
  unsigned* d_gend = reinterpret_cast<unsigned*>(p);
  p += b_grp;
  unsigned* d_ready = reinterpret_cast<unsigned*>(p);
  p += b_grp;
  void* d_ws = p;
  int rc = PM_SUCCESS;
#define PM_CHECK(call, what)                 \
  do {                                       \
    cudaError_t e_ = (call);                 \
    if (e_ != cudaSuccess) {                 \
      rc = cuda_fail(e_, what);              \
      goto done;                             \
    }                                        \
  } while (0)
  PM_CHECK(cudaMemcpyAsync(d_offs, trace_offsets, 8 * (size_t)(n_traces + 1),
                           cudaMemcpyHostToDevice, stream), "H2D offsets");
  PM_CHECK(cudaMemcpyAsync(d_cfgs, cfgs, sizeof(pm_cfg_t) * (size_t)n_cfgs,
                           cudaMemcpyHostToDevice, stream), "H2D cfgs");
  if (cfg_of_trace)
    PM_CHECK(cudaMemcpyAsync(d_cfgof, cfg_of_trace, 4 * (size_t)n_traces,
                             cudaMemcpyHostToDevice, stream), "H2D cfg_of");
  PM_CHECK(cudaMemcpyAsync(d_order, order.data(), 4 * (size_t)n_traces,
                           cudaMemcpyHostToDevice, stream), "H2D order");
  PM_CHECK(cudaMemcpyAsync(d_gend, group_end.data(), 4 * (size_t)G,
                           cudaMemcpyHostToDevice, stream), "H2D groups");
  PM_CHECK(cudaMemsetAsync(d_ready, 0, 4 * (size_t)G, stream), "memset flags");
  if (d_tl)  // entries past an OOM / error stay zero, as on the host side
    PM_CHECK(cudaMemsetAsync(d_tl, 0, b_tl, stream), "memset timeline");
  PM_CHECK(cudaEventRecord(zeroed, stream), "event record");
  PM_CHECK(cudaStreamWaitEvent(cs, zeroed, 0), "stream wait");
  for (int g = 0; g < G; ++g) {
    const int64_t e0 = trace_offsets[gfirst[g]], e1 = trace_offsets[gfirst[g + 1]];
    if (e1 > e0)
      PM_CHECK(cudaMemcpyAsync(d_reqs + e0, reqs + e0, 16 * (size_t)(e1 - e0),
                               cudaMemcpyHostToDevice, cs), "H2D requests");
    PM_CHECK(cudaMemcpyAsync(d_ready + g, one, sizeof(unsigned),
                             cudaMemcpyHostToDevice, cs), "H2D flag");
  }
  rc = replay_batch_impl(d_reqs, d_offs, n_traces, d_cfgs,
                         cfg_of_trace ? d_cfgof : nullptr, d_order, d_res, d_tl,
                         d_ws, L.total, total, max_ev, stream_, d_gend, G, d_ready);
  if (rc != PM_SUCCESS) goto done;
  PM_CHECK(cudaMemcpyAsync(results, d_res, sizeof(pm_result_t) * (size_t)n_traces,
                           cudaMemcpyDeviceToHost, stream), "D2H results");
  if (timeline && total > 0)
    PM_CHECK(cudaMemcpyAsync(timeline, d_tl, 16 * (size_t)total,
                             cudaMemcpyDeviceToHost, stream), "D2H timeline");
done:
#undef PM_CHECK
  {
    cudaError_t e2 = cudaStreamSynchronize(cs);
    if (rc == PM_SUCCESS && e2 != cudaSuccess) rc = cuda_fail(e2, "copy stream");
  }
  cudaFreeAsync(dmem, stream);
  e = cudaStreamSynchronize(stream);
  if (rc == PM_SUCCESS && e != cudaSuccess) rc = cuda_fail(e, "cudaStreamSynchronize");
  cudaEventDestroy(zeroed);
  cudaStreamDestroy(cs);
  return rc;
}

}  // extern "C"
