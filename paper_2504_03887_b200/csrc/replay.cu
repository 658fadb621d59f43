// Batched caching-allocator replay for sm_100a -- host side of the C ABI
// (include/peakmem_b200.h).  The kernels live in replay_device.cuh.

#include <cuda_runtime.h>
#include <stdint.h>

#include "peakmem_b200.h"
#include "replay_device.cuh"
#include "replay_narrow.cuh"

// ---------------------------------------------------------------------------
// Host side of the C ABI.

#include <algorithm>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
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

constexpr int kWarps = 12;        // wide main kernel (PM_REPLAY_WIDE=1)
constexpr int kNarrowWarps = 24;  // narrow main kernel (PM_REPLAY_WARPS: 12..32)
constexpr size_t kBucket_host = 32;  // warps (traces in flight) per CTA, 1 CTA / SM
constexpr int kRetryWarps = 1;
constexpr int kMaxRetryWarps = 64;
constexpr int kPass1Warps = 6;    // narrow pass 1: warps (private pools) per SM

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// workspace = ctl | retry list | retry pools | record table | checkpoint
// offsets | checkpoint region
struct Layout {
  size_t retry_list, gpool, recs, ck_off, ck, ck_bytes, total;
  int nbmax_g;
  int retry_warps;
};

Layout layout_for(int64_t total_events, int64_t max_trace_events,
                  int32_t n_traces) {
  Layout L;
  size_t off = align_up(sizeof(pmb::Ctl), 256);
  L.retry_list = off;
  off = align_up(off + 7 * sizeof(int32_t) * (size_t)(n_traces > 0 ? n_traces : 1),
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
  // checkpoints of traces handed between narrow passes (replay_narrow.cuh
  // NCk): ~16 B per free block; a full region only means a restart
  L.ck_off = off;
  off = align_up(off + 8 * (size_t)(n_traces > 0 ? n_traces : 1), 256);
  L.ck = off;
  size_t ckb = 4 * (size_t)(total_events > 0 ? total_events : 1) +
               256 * (size_t)(n_traces > 0 ? n_traces : 1);
  if (ckb < (64u << 20)) ckb = 64u << 20;
  if (ckb > (1ull << 30)) ckb = 1ull << 30;
  L.ck_bytes = ckb;
  off = align_up(off + ckb, 256);
  L.total = off;
  return L;
}

struct Occupancy {
  int sms = 0, per_sm = 0, buckets = 0, warps = 0;
  size_t smem = 0;
  bool narrow = true;  // main pass: replay_narrow_kernel (else the wide kernel)
  int per_sm_n = 0, buckets_n = 0;  // the narrow main kernel's launch
  size_t smem_n = 0;
  // batches under a wave: the narrowest main-kernel CTA that holds the
  // batch with one trace per warp -- 1, 12, 16 or 20 warps per CTA
  // (kSmallWidths): fewer warps share an SM's pool and issue slots, and they
  // compile to 96 registers instead of 80 (PM_REPLAY_WARPS pins the width)
  int per_sm_w[4] = {0, 0, 0, 0}, buckets_w[4] = {0, 0, 0, 0};
  size_t smem_w[4] = {0, 0, 0, 0};
  bool warps_pinned = false;
  int nbmax_m1 = 0, nbmax_m2 = 0;   // narrow memory-directory passes 2-3
  size_t smem_m1 = 0;
  int warps_s1 = 0, nbmax_s1 = 0;   // pass 1: warps per SM, buckets per warp
  size_t warp_bytes_s1 = 0;
  int per_sm1 = 0;  // tier-1 retry kernel
  size_t smem1 = 0;
  int nbmax2 = 0;   // tier-2: one warp with a shared-memory directory
  int nbmax3 = 0;   // tier-3: shared-memory directory over an HBM pool
  size_t smem3 = 0;
  size_t smem2 = 0;
};

constexpr int kTier1Warps = 8;  // tier 1: a dedicated 32-bucket pool per warp
constexpr int kSmallWidths[4] = {1, 12, 16, 20};

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

template <int W>
int setup_narrow(int optin, int cap, int* buckets, size_t* smem, int* per_sm) {
  int b = (int)(((size_t)optin - (size_t)W * pmn::kWarpStageBytes - 256) /
                (kBucket_host * 16));
  if (cap > 0 && cap < b) b = cap;
  if (b < 2 * W) b = 2 * W;
  *buckets = b;
  *smem = pmn::smem_cta_bytes(b, W);
  cudaError_t e = cudaFuncSetAttribute(
      pmn::replay_narrow_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)*smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute narrow");
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      per_sm, pmn::replay_narrow_kernel<W>, W * 32, *smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy narrow");
  if (*per_sm < 1) return fail(PM_ERR_CUDA, "narrow replay kernel cannot be resident");
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
    const char* wide = getenv("PM_REPLAY_WIDE");
    o.narrow = !(wide && atoi(wide) != 0);
    o.warps = o.narrow ? kNarrowWarps : kWarps;
    if (const char* env = getenv("PM_REPLAY_WARPS")) {
      o.warps = atoi(env);
      o.warps_pinned = true;
    }
    int rc = setup_narrow<1>(optin, cap, &o.buckets_w[0], &o.smem_w[0], &o.per_sm_w[0]);
    if (rc == PM_SUCCESS)
      rc = setup_narrow<12>(optin, cap, &o.buckets_w[1], &o.smem_w[1], &o.per_sm_w[1]);
    if (rc == PM_SUCCESS)
      rc = setup_narrow<16>(optin, cap, &o.buckets_w[2], &o.smem_w[2], &o.per_sm_w[2]);
    if (rc == PM_SUCCESS)
      rc = setup_narrow<20>(optin, cap, &o.buckets_w[3], &o.smem_w[3], &o.per_sm_w[3]);
    if (rc != PM_SUCCESS) return rc;
    // the narrow main kernel is always set up (wire-word input needs it even
    // when PM_REPLAY_WIDE selects the wide main pass)
    const int nw = o.narrow ? o.warps : kNarrowWarps;
    switch (nw) {
      // 1: one warp per CTA (no bucket hand-off between warps): the
      // configuration compute-sanitizer's racecheck can judge completely
      case 1: rc = setup_narrow<1>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n); break;
      case 12: rc = setup_narrow<12>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n); break;
      case 20: rc = setup_narrow<20>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n); break;
      case 24: rc = setup_narrow<24>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n); break;
      case 28: rc = setup_narrow<28>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n); break;
      case 32: rc = setup_narrow<32>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n); break;
      default:
        if (o.narrow) o.warps = 16;
        rc = setup_narrow<16>(optin, cap, &o.buckets_n, &o.smem_n, &o.per_sm_n);
    }
    if (rc != PM_SUCCESS) return rc;
    if (o.narrow) {
      o.buckets = o.buckets_n;
      o.smem = o.smem_n;
      o.per_sm = o.per_sm_n;
    } else if (o.warps == 12)
      rc = setup_kernel<12>(optin, cap, &o.buckets, &o.smem, &o.per_sm);
    else if (o.warps == 14)
      rc = setup_kernel<14>(optin, cap, &o.buckets, &o.smem, &o.per_sm);
    else {
      o.warps = 16;
      rc = setup_kernel<16>(optin, cap, &o.buckets, &o.smem, &o.per_sm);
    }
    if (rc != PM_SUCCESS) return rc;
    // narrow memory-directory passes: one warp per CTA, 24 B of directory
    // per bucket, + 512 B of entries per bucket in the shared-memory pass
    o.nbmax_m1 = (int)(((size_t)optin - pmn::kWarpStageBytes - 256) / (24 + 512));
    o.smem_m1 = pmn::mem_tier_smem(o.nbmax_m1, true);
    o.warps_s1 = kPass1Warps;
    if (const char* env = getenv("PM_PASS1_WARPS")) o.warps_s1 = atoi(env);
    if (o.warps_s1 < 1) o.warps_s1 = 1;
    if (o.warps_s1 > 8) o.warps_s1 = 8;
    o.nbmax_s1 = (int)(((size_t)optin / o.warps_s1 - pmn::kWarpStageBytes - 256) / (24 + 512));
    o.warp_bytes_s1 = align_up(pmn::mem_tier_smem(o.nbmax_s1, true), 128);
    e = cudaFuncSetAttribute(pmn::replay_narrow_mem_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)std::max(o.smem_m1, o.warps_s1 * o.warp_bytes_s1));
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute pass 1");
    o.nbmax_m2 = (int)(((size_t)optin - pmn::kWarpStageBytes - 256) / 24);
    e = cudaFuncSetAttribute(pmn::replay_narrow_mem_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pmn::mem_tier_smem(o.nbmax_m2, false));
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute pass 2");
    if (rc != PM_SUCCESS) return rc;
    int b1 = 0;
    rc = setup_kernel<kTier1Warps>(optin, kTier1Warps * 32, &b1, &o.smem1,
                                   &o.per_sm1);
    if (rc != PM_SUCCESS) return rc;
    o.nbmax2 = (int)(((size_t)optin - 1024) / (kBucket_host * 24 + 32));
    while (o.nbmax2 > 8 && pmb::gmem_warp_bytes(o.nbmax2) > (size_t)optin) --o.nbmax2;
    o.smem2 = pmb::gmem_warp_bytes(o.nbmax2);
    e = cudaFuncSetAttribute(pmb::replay_dirmem_kernel<1, 0>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)o.smem2);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute tier 2");
    o.nbmax3 = (int)(((size_t)optin - 32 * 24 - 256) / 32);
    o.smem3 = pmb::hybrid_smem_bytes(o.nbmax3);
    e = cudaFuncSetAttribute(pmb::replay_dirmem_kernel<1, 1>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)o.smem3);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute tier 3");
    // load every replay kernel now (lazy module loading would otherwise
    // load a retry tier at its first launch, which waits for the device --
    // and pm_replay_host's main pass waits for copies enqueued after it)
    {
      cudaFuncAttributes fa;
      const void* fns[] = {
          (const void*)pmn::replay_narrow_kernel<1>,
          (const void*)pmn::replay_narrow_kernel<12>, (const void*)pmn::replay_narrow_kernel<16>,
          (const void*)pmn::replay_narrow_kernel<20>, (const void*)pmn::replay_narrow_kernel<24>,
          (const void*)pmn::replay_narrow_kernel<28>, (const void*)pmn::replay_narrow_kernel<32>,
          (const void*)pmn::replay_narrow_mem_kernel<true>,
          (const void*)pmn::replay_narrow_mem_kernel<false>,
          (const void*)pmb::replay_smem_kernel<8>, (const void*)pmb::replay_smem_kernel<12>,
          (const void*)pmb::replay_smem_kernel<14>, (const void*)pmb::replay_smem_kernel<16>,
          (const void*)pmb::replay_dirmem_kernel<1, 0>,
          (const void*)pmb::replay_dirmem_kernel<1, 1>,
          (const void*)pmb::replay_dirmem_kernel<kRetryWarps, 2>};
      for (const void* f : fns) {
        e = cudaFuncGetAttributes(&fa, f);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
      }
    }
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

#ifdef PM_STATS
int pm_debug_stats(unsigned long long* out16) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, pmn::g_stats, 16 * sizeof(unsigned long long));
  return 0;
}
#endif

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

int pm_validate_inject(int64_t request_index, int32_t kind) {
#ifdef PM_VALIDATE
  const int v[2] = {(int)request_index, kind};
  cudaError_t e = cudaMemcpyToSymbol(pmb::g_inject, v, sizeof(v));
  return e == cudaSuccess ? PM_SUCCESS : cuda_fail(e, "pm_validate_inject");
#else
  (void)request_index;
  (void)kind;
  return fail(PM_ERR_INVALID_ARGUMENT, "pm_validate_inject: not a validating build");
#endif
}

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
                      const unsigned* ready,
                      const std::function<int()>& after_main = {},
                      const uint64_t* wire = nullptr) {
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
  long long* ck_off = reinterpret_cast<long long*>(base + L.ck_off);
  char* ck_base = base + L.ck;
  const unsigned long long ck_cap = L.ck_bytes;

  Occupancy occ;
  int rc = query_occupancy(&occ);
  if (rc != PM_SUCCESS) return rc;

  cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(pmb::Ctl), stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  // pass lists (pmn::route): narrow memory-directory tiers, then the wide
  // tiers 1-4 (an encoding limit goes straight to wide tier 1)
  const size_t nt = (size_t)n_traces;
  int32_t* list_m1 = retry_list;           // pass 1: narrow, smem, multi-warp
  int32_t* list_mb = retry_list + nt;      // pass 2: narrow, smem, one warp
  int32_t* list_m2 = retry_list + 2 * nt;  // pass 3: narrow, HBM entries
  int32_t* list_w1 = retry_list + 3 * nt;  // pass 4: wide tier 1
  int32_t* list_w2 = retry_list + 4 * nt;  // pass 5: wide tier 2
  int32_t* list_w3 = retry_list + 5 * nt;  // pass 6: wide tier 3
  int32_t* list_w4 = retry_list + 6 * nt;  // pass 7: wide tier 4
  const bool narrow = occ.narrow || wire != nullptr;  // wire words need it
  const int mwarps = narrow && !occ.narrow ? kNarrowWarps : occ.warps;
  long long want = ((long long)n_traces + mwarps - 1) / mwarps;
  const long long full = (long long)(narrow && !occ.narrow ? occ.per_sm_n : occ.per_sm) * occ.sms;
  long long grid = full;
  if (want < grid) grid = want;
  // Under half a wave (a small sweep, a rank's shard at 8 GPUs): spread the
  // traces over every SM rather than packing them into the fewest CTAs --
  // a warp's chain is shorter when fewer warps share its SM
  const char* spread_env = getenv("PM_SPREAD");
  int lwarps = mwarps;  // the narrow main kernel's width for this launch
  size_t lsmem = occ.smem_n;
  int lbuckets = occ.buckets_n;
  const bool spread_ok = !(spread_env && atoi(spread_env) == 0);
  if (narrow && 2 * (long long)n_traces <= full * mwarps && spread_ok) {
    const long long spread = n_traces < occ.sms ? n_traces : occ.sms;
    if (spread > grid) grid = spread < full ? spread : full;
  }
  // and in the narrowest CTAs that hold the batch (C3 traces: 148 traces one
  // warp per CTA 80 vs 105 ms; 600-1776 traces 12 warps per CTA 15-19 %
  // faster than 24)
  if (narrow && spread_ok && !occ.warps_pinned) {
    for (int k = 0; k < 4; ++k) {
      const long long slots = (long long)kSmallWidths[k] * occ.sms * occ.per_sm_w[k];
      if (n_traces > slots) continue;
      lwarps = kSmallWidths[k];
      lsmem = occ.smem_w[k];
      lbuckets = occ.buckets_w[k];
      grid = (long long)occ.sms * occ.per_sm_w[k];
      if (grid > n_traces) grid = n_traces;
      break;
    }
  }
  if (const char* cap = getenv("PM_MAX_GRID")) {  // debugging aid
    const long long g = atoll(cap);
    if (g > 0 && g < grid) grid = g;
  }
  // Long traces start in the main pass like any other: a trace that outgrows
  // a pass continues in the next from its checkpoint, so nothing is replayed
  // twice (the round-1 rule sent traces of >= 2^20 requests in batches of at
  // most one per SM straight to pass 2, when a hand-off restarted at request
  // 0; with checkpoints C5's lone trace is 3.68 s that way, 3.53 s through
  // the passes).  PM_LONG_SKIP=1 restores the skip.
  int long_trace = pmn::kNoSkip;
  if (const char* env = getenv("PM_LONG_SKIP"))
    if (atoi(env) != 0 && n_traces <= occ.sms) long_trace = pmn::kLongTrace;
  // Narrow pass 1 runs BESIDE the main pass: launched right behind it as a
  // programmatic dependent launch (the main pass's CTAs release it once they
  // are all resident, so it can never take SMs the main pass needs), its
  // CTAs take SMs the main pass leaves idle (a batch of less than a wave)
  // or frees as its CTAs finish, and continue hand-offs as they arrive
  // instead of after the whole main pass -- a replay that outgrows the main
  // pass early (C4's fragmenting configs) no longer waits for the slowest
  // main replay (PM_BESIDE=0: pass 1 after the main pass).
  bool beside = false;
  {
    const char* env = getenv("PM_BESIDE");
    beside = narrow && ready == nullptr && !(env && atoi(env) == 0);
  }
  if (beside) {
    e = cudaMemsetAsync(list_m1, 0xFF, 4 * nt, stream);  // slots start at -1
    if (e != cudaSuccess) return cuda_fail(e, "beside pass setup");
  }
  // A packed batch of one wave with a short tail: its long traces fill the
  // first CTAs warp-major and the tail whole CTAs, which free their SMs early
  // for the pass-1 grid beside (pmn::pos_prep_kernel; PM_TAIL_CTAS=0: the
  // atomic counter throughout).
  if (narrow && lwarps >= 24 && (long long)n_traces <= grid * lwarps) {
    const char* env = getenv("PM_TAIL_CTAS");
    if (!(env && atoi(env) == 0)) {
      // long traces per long CTA (PM_TAIL_PER_CTA, experiment)
      int per_cta = lwarps;
      if (const char* pe = getenv("PM_TAIL_PER_CTA"))
        if (atoi(pe) > 0 && atoi(pe) <= lwarps) per_cta = atoi(pe);
      pmn::pos_prep_kernel<<<1, 1024, 0, stream>>>(trace_offsets, trace_order, n_traces,
                                                   per_cta, (int)grid, ctl);
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(e, "first-wave split");
    }
  }
#define PM_LAUNCH_NARROW(W)                                                   \
  pmn::replay_narrow_kernel<W><<<(unsigned)grid, W * 32, lsmem, stream>>>(    \
      reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline,             \
      reinterpret_cast<pmb::u32*>(recs), ctl, trace_order, n_traces, list_m1, \
      lbuckets, group_end, n_groups, ready,                                   \
      reinterpret_cast<const pmb::u64*>(wire), const_cast<pm_req_t*>(reqs),   \
      list_w1, long_trace, ck_off, ck_base, ck_cap)
#define PM_LAUNCH_MAIN(W)                                                     \
  pmb::replay_smem_kernel<W><<<(unsigned)grid, W * 32, occ.smem, stream>>>(  \
      reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs, ctl, \
      0, trace_order, n_traces, list_m1, occ.buckets, group_end, n_groups, ready)
  if (narrow) {
    switch (lwarps) {
      case 1: PM_LAUNCH_NARROW(1); break;
      case 12: PM_LAUNCH_NARROW(12); break;
      case 20: PM_LAUNCH_NARROW(20); break;
      case 24: PM_LAUNCH_NARROW(24); break;
      case 28: PM_LAUNCH_NARROW(28); break;
      case 32: PM_LAUNCH_NARROW(32); break;
      default: PM_LAUNCH_NARROW(16); break;
    }
  } else if (occ.warps == 12)
    PM_LAUNCH_MAIN(12);
  else if (occ.warps == 14)
    PM_LAUNCH_MAIN(14);
  else
    PM_LAUNCH_MAIN(16);
#undef PM_LAUNCH_MAIN
#undef PM_LAUNCH_NARROW
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay main-pass launch");
  if (after_main) {
    // streamed input: the copies go in behind the main pass (which waits
    // on their flags) and before any further launch
    const int rc2 = after_main();
    if (rc2 != PM_SUCCESS) return rc2;
  }
  const long long gtraces = n_traces < occ.sms ? n_traces : occ.sms;
  if (beside) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)gtraces);
    lc.blockDim = dim3(32 * occ.warps_s1);
    lc.dynamicSmemBytes = (size_t)occ.warps_s1 * occ.warp_bytes_s1;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelEx(&lc, pmn::replay_narrow_mem_kernel<true>, reqs, trace_offsets, cfgs,
                           cfg_of_trace, results, timeline, reinterpret_cast<pmb::u32*>(recs),
                           ctl, (int)pmn::kTierMemSmem, (const int32_t*)list_m1, list_mb,
                           list_w1, (char*)nullptr, occ.nbmax_s1,
                           reinterpret_cast<const pmb::u64*>(wire), const_cast<pm_req_t*>(reqs),
                           long_trace, ck_off, ck_base, ck_cap, (size_t)occ.warp_bytes_s1, 1);
    if (e != cudaSuccess) return cuda_fail(e, "replay beside-pass launch");
  }
  // passes 1-2: narrow, shared-memory directory (entries in shared memory,
  // then in HBM: the per-CTA region fits in tier 4's, nb <= nbmax_g)
  // pass 1: several warps per SM, each with a private shared-memory pool
  // (fragmented traces replay side by side); pass 2: one warp owning the
  // SM's shared memory for the traces that outgrow those
  if (!beside) {
    pmn::replay_narrow_mem_kernel<true>
        <<<(unsigned)gtraces, 32 * occ.warps_s1, occ.warps_s1 * occ.warp_bytes_s1, stream>>>(
            reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline,
            reinterpret_cast<pmb::u32*>(recs), ctl, pmn::kTierMemSmem, list_m1, list_mb,
            list_w1, nullptr, occ.nbmax_s1, reinterpret_cast<const pmb::u64*>(wire),
            const_cast<pm_req_t*>(reqs), long_trace, ck_off, ck_base, ck_cap,
            occ.warp_bytes_s1, 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "replay pass-1 launch");
  }
  pmn::replay_narrow_mem_kernel<true><<<(unsigned)gtraces, 32, occ.smem_m1, stream>>>(
      reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline,
      reinterpret_cast<pmb::u32*>(recs), ctl, pmn::kTierMemSmemBig, list_mb, list_m2,
      list_w1, nullptr, occ.nbmax_m1, reinterpret_cast<const pmb::u64*>(wire),
      const_cast<pm_req_t*>(reqs), long_trace, ck_off, ck_base, ck_cap, 0, 0);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay pass-2 launch");
  {
    int nbm2 = occ.nbmax_m2 < L.nbmax_g ? occ.nbmax_m2 : L.nbmax_g;
    if (const char* env = getenv("PM_M2_BUCKETS")) {  // experiment
      const int c = atoi(env);
      if (c > 0 && c < nbm2) nbm2 = c;
    }
    // up to one CTA per SM, as many as the retry region holds
    long long gm2 = (long long)((L.recs - L.gpool) / pmn::mem_tier_pool_bytes(nbm2));
    if (gm2 > occ.sms) gm2 = occ.sms;
    if (gm2 > n_traces) gm2 = n_traces;
    if (gm2 < 1) gm2 = 1;
    pmn::replay_narrow_mem_kernel<false>
        <<<(unsigned)gm2, 32, pmn::mem_tier_smem(nbm2, false), stream>>>(
            reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline,
            reinterpret_cast<pmb::u32*>(recs), ctl, pmn::kTierMemHbm, list_m2,
            list_w4, list_w1, gpool, nbm2, reinterpret_cast<const pmb::u64*>(wire),
            const_cast<pm_req_t*>(reqs), pmn::kNoSkip, ck_off, ck_base, ck_cap, 0, 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "replay pass-3 launch");
  }
  // wide tier 1 (pass 3): dedicated 32-bucket pools (grid sized for the
  // worst case; idle CTAs exit at once when nothing was escalated)
  long long grid1 = (long long)occ.per_sm1 * occ.sms;
  long long want1 = ((long long)n_traces + kTier1Warps - 1) / kTier1Warps;
  if (want1 < grid1) grid1 = want1;
  pmb::replay_smem_kernel<kTier1Warps>
      <<<(unsigned)grid1, kTier1Warps * 32, occ.smem1, stream>>>(
          reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs,
          ctl, pmn::kTierWide1, list_w1, 0, list_w2, kTier1Warps * 32, nullptr,
          0, nullptr);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay tier-1 launch");
  {
    pmb::replay_dirmem_kernel<1, 0><<<(unsigned)gtraces, 32, occ.smem2, stream>>>(
        reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs, ctl,
        pmn::kTierWide1 + 1, list_w2, list_w3, nullptr, occ.nbmax2);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "replay tier-2 launch");
    // tier 3: shared-memory directory, HBM entries (the per-warp pool fits
    // in tier 4's region: nbmax3 is capped at tier 4's bucket count)
    const int nb3 = occ.nbmax3 < L.nbmax_g ? occ.nbmax3 : L.nbmax_g;
    long long grid3 = L.retry_warps < occ.sms ? L.retry_warps : occ.sms;
    pmb::replay_dirmem_kernel<1, 1><<<(unsigned)grid3, 32, pmb::hybrid_smem_bytes(nb3),
                                      stream>>>(
        reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs, ctl,
        pmn::kTierWide1 + 2, list_w3, list_w4, gpool, nb3);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "replay tier-3 launch");
    pmb::replay_dirmem_kernel<kRetryWarps, 2>
        <<<L.retry_warps / kRetryWarps, kRetryWarps * 32, 0, stream>>>(
            reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs,
            ctl, pmn::kTierWide4, list_w4, nullptr, gpool, L.nbmax_g);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay tier-4 launch");
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

}  // extern "C"

namespace {

// pm_replay_host / pm_replay_host_wire: `src` holds pm_req_t records
// (wb = 16) or wire words (wb = 8).  Wire words are replayed by the narrow
// main pass directly; d_reqs then only receives the pm_req_t expansion of
// traces escalated to the wide tiers.
int replay_host_impl(const void* src, size_t wb, const int64_t* trace_offsets,
                     int32_t n_traces, const pm_cfg_t* cfgs, int32_t n_cfgs,
                     const int32_t* cfg_of_trace, pm_result_t* results,
                     int64_t* timeline, void* stream_) {
  const char* reqs = static_cast<const char*>(src);
  const bool wire = wb == 8;
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
  // Streamed upload in longest-first order: the traces, sorted by length
  // (stable), are cut into G groups of ~equal bytes; each trace is copied to
  // its own offset on a copy stream and each group is followed by a 4-byte
  // DMA of a pinned "1" into its ready flag.  The kernel (launched first)
  // takes traces in the same order and waits for a trace's group flag, so
  // replay overlaps the H2D and the last group to land holds the shortest
  // traces.
  const size_t bytes_in = wb * (size_t)total;
  int G = (int)(bytes_in / (256u << 20));
  if (G < 1) G = 1;
  if (G > 64) G = 64;
  if (G > n_traces) G = n_traces;
  std::vector<int32_t> order(n_traces);
  for (int32_t i = 0; i < n_traces; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return trace_offsets[a + 1] - trace_offsets[a] >
           trace_offsets[b + 1] - trace_offsets[b];
  });
  std::vector<unsigned> group_end(G);
  {
    int g = 0;
    int64_t acc = 0;
    for (int32_t i = 0; i < n_traces; ++i) {
      const int32_t t = order[i];
      acc += trace_offsets[t + 1] - trace_offsets[t];
      // close group g once the groups so far hold their share of the
      // requests (the last group takes the rest; a group may be empty)
      while (g < G - 1 && acc * G >= total * (int64_t)(g + 1)) {
        group_end[g++] = (unsigned)(i + 1);
      }
    }
    while (g < G) group_end[g++] = (unsigned)n_traces;
  }
  const Layout L = layout_for(total, max_ev, n_traces);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  // Pinned source: by default the kernels read it in place (zero copy:
  // pinned memory is device-addressable, each warp's TMA bulk load pulls
  // its next chunk over PCIe one chunk ahead), so nothing is staged in HBM.
  // PM_HOST_COPY=1 streams it through the copy engines instead (launch
  // first, per-group ready flags).  A pageable source is copied before the
  // launch: its cudaMemcpyAsync synchronises with the device.
  bool pinned = false;
  void* mapped = nullptr;
  {
    cudaPointerAttributes pa;
    pinned = cudaPointerGetAttributes(&pa, reqs) == cudaSuccess &&
             pa.type == cudaMemoryTypeHost;
    cudaGetLastError();  // clear a failed query
  }
  const char* copy_env = getenv("PM_HOST_COPY");
  const bool zero_copy =
      pinned && !(copy_env && atoi(copy_env) != 0) &&
      cudaHostGetDevicePointer(&mapped, const_cast<char*>(reqs), 0) == cudaSuccess;
  cudaGetLastError();
  // d_reqs: staged pm_req_t, or (wire) the expansion of escalated traces
  const size_t b_reqs = (zero_copy && !wire)
                            ? 256
                            : align_up(16 * (size_t)(total > 0 ? total : 1), 256);
  const size_t b_wire = (wire && !zero_copy)
                            ? align_up(8 * (size_t)(total > 0 ? total : 1), 256)
                            : 0;
  const size_t b_offs = align_up(8 * (size_t)(n_traces + 1), 256);
  const size_t b_cfgs = align_up(sizeof(pm_cfg_t) * (size_t)n_cfgs, 256);
  const size_t b_cfgof = align_up(4 * (size_t)n_traces, 256);
  const size_t b_order = b_cfgof;
  const size_t b_res = align_up(sizeof(pm_result_t) * (size_t)n_traces, 256);
  const size_t b_tl = timeline ? align_up(16 * (size_t)(total > 0 ? total : 1), 256) : 0;
  const size_t b_grp = align_up(8 * (size_t)G, 256);
  const size_t bytes = b_reqs + b_wire + b_offs + b_cfgs + b_cfgof + b_order +
                       b_res + b_tl + 2 * b_grp + L.total;
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
  // PM_TRACE_PHASES=1: report when the copies and the replay finished
  const bool trace_phases = getenv("PM_TRACE_PHASES") != nullptr;
  cudaEvent_t ph[3] = {nullptr, nullptr, nullptr};
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
  char* d_src = wire ? p : reinterpret_cast<char*>(d_reqs);
  p += b_wire;
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
  if (trace_phases) {
    cudaEventCreate(&ph[0]);
    cudaEventCreate(&ph[1]);
    cudaEventCreate(&ph[2]);
    cudaEventRecord(ph[0], stream);
  }
  {
    // Pinned source: launch the main pass first (it waits on the flags) and
    // enqueue the copies behind it, before the tier launches.  A pageable
    // source makes each cudaMemcpyAsync synchronise with the device, so its
    // copies are all enqueued before the launch (no overlap, no deadlock).
    auto enqueue_copies = [&]() -> int {
      int32_t i = 0;
      for (int g = 0; g < G; ++g) {
        while (i < (int32_t)group_end[g]) {
          // one copy per run of traces adjacent in memory
          const int32_t t0 = order[i];
          int64_t e0 = trace_offsets[t0], e1 = trace_offsets[t0 + 1];
          ++i;
          while (i < (int32_t)group_end[g] && trace_offsets[order[i]] == e1) {
            e1 = trace_offsets[order[i] + 1];
            ++i;
          }
          cudaError_t ce = cudaSuccess;
          if (e1 > e0)
            ce = cudaMemcpyAsync(d_src + wb * e0, reqs + wb * e0,
                                 wb * (size_t)(e1 - e0), cudaMemcpyHostToDevice, cs);
          if (ce != cudaSuccess) {
            // release the waiting replay before failing (results unused)
            cudaMemsetAsync(d_ready, 0xFF, 4 * (size_t)G, cs);
            return cuda_fail(ce, "H2D requests");
          }
        }
        cudaError_t ce = cudaMemcpyAsync(d_ready + g, one, sizeof(unsigned),
                                         cudaMemcpyHostToDevice, cs);
        if (ce != cudaSuccess) {
          cudaMemsetAsync(d_ready, 0xFF, 4 * (size_t)G, cs);
          return cuda_fail(ce, "H2D flag");
        }
      }
      if (trace_phases) cudaEventRecord(ph[2], cs);
      return PM_SUCCESS;
    };
    if (zero_copy) {
      const pm_req_t* rsrc =
          wire ? d_reqs : reinterpret_cast<const pm_req_t*>(mapped);
      rc = replay_batch_impl(rsrc, d_offs, n_traces, d_cfgs,
                             cfg_of_trace ? d_cfgof : nullptr, d_order, d_res,
                             d_tl, d_ws, L.total, total, max_ev, stream_,
                             nullptr, 0, nullptr, std::function<int()>(),
                             wire ? reinterpret_cast<const uint64_t*>(mapped)
                                  : nullptr);
      if (trace_phases) cudaEventRecord(ph[2], stream);
      if (rc != PM_SUCCESS) goto done;
      goto launched;
    }
    if (!pinned) {
      rc = enqueue_copies();
      if (rc != PM_SUCCESS) goto done;
    }
    rc = replay_batch_impl(d_reqs, d_offs, n_traces, d_cfgs,
                           cfg_of_trace ? d_cfgof : nullptr, d_order, d_res,
                           d_tl, d_ws, L.total, total, max_ev, stream_, d_gend,
                           G, d_ready,
                           pinned ? std::function<int()>(enqueue_copies)
                                  : std::function<int()>(),
                           wire ? reinterpret_cast<const uint64_t*>(d_src) : nullptr);
    if (rc != PM_SUCCESS) goto done;
  }
launched:
  PM_CHECK(cudaMemcpyAsync(results, d_res, sizeof(pm_result_t) * (size_t)n_traces,
                           cudaMemcpyDeviceToHost, stream), "D2H results");
  if (timeline && total > 0)
    PM_CHECK(cudaMemcpyAsync(timeline, d_tl, 16 * (size_t)total,
                             cudaMemcpyDeviceToHost, stream), "D2H timeline");
  if (trace_phases) cudaEventRecord(ph[1], stream);
done:
#undef PM_CHECK
  {
    cudaError_t e2 = cudaStreamSynchronize(cs);
    if (rc == PM_SUCCESS && e2 != cudaSuccess) rc = cuda_fail(e2, "copy stream");
  }
  cudaFreeAsync(dmem, stream);
  e = cudaStreamSynchronize(stream);
  if (rc == PM_SUCCESS && e != cudaSuccess) rc = cuda_fail(e, "cudaStreamSynchronize");
  if (trace_phases && ph[1]) {
    float k = 0, c = 0;
    cudaEventElapsedTime(&k, ph[0], ph[1]);
    cudaEventElapsedTime(&c, ph[0], ph[2]);
    fprintf(stderr, "pm_replay_host: copies done %.1f ms, replay done %.1f ms after start\n", c, k);
    for (auto& x : ph) cudaEventDestroy(x);
  }
  cudaEventDestroy(zeroed);
  cudaStreamDestroy(cs);
  return rc;
}

}  // namespace

extern "C" {

int pm_replay_host(const pm_req_t* reqs, const int64_t* trace_offsets,
                   int32_t n_traces, const pm_cfg_t* cfgs, int32_t n_cfgs,
                   const int32_t* cfg_of_trace, pm_result_t* results,
                   int64_t* timeline, void* stream) {
  return replay_host_impl(reqs, 16, trace_offsets, n_traces, cfgs, n_cfgs,
                          cfg_of_trace, results, timeline, stream);
}

int pm_replay_host_wire(const uint64_t* words, const int64_t* trace_offsets,
                        int32_t n_traces, const pm_cfg_t* cfgs, int32_t n_cfgs,
                        const int32_t* cfg_of_trace, pm_result_t* results,
                        int64_t* timeline, void* stream) {
  return replay_host_impl(words, 8, trace_offsets, n_traces, cfgs, n_cfgs,
                          cfg_of_trace, results, timeline, stream);
}

int pm_wire_pack(const pm_req_t* reqs, const int64_t* trace_offsets,
                 int32_t n_traces, uint64_t* words, int64_t* first_bad) {
  if (first_bad) *first_bad = -1;
  if (n_traces < 0 || (n_traces > 0 && (!trace_offsets || !words)))
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_wire_pack: bad arguments");
  if (n_traces == 0) return PM_SUCCESS;
  // Traces are independent (each numbers its own handles), so host threads
  // pack contiguous runs of traces of ~equal request counts; the lowest bad
  // index over all threads is the one reported.
  const int64_t total = trace_offsets[n_traces] - trace_offsets[0];
  unsigned hw = std::thread::hardware_concurrency();
  int nt = (int)std::min<int64_t>(hw ? hw : 1, std::max<int64_t>(1, total >> 20));
  nt = std::min(nt, (int)n_traces);
  std::vector<int64_t> bad(nt, INT64_MAX);
  auto work = [&](int w) {
    // traces [t0, t1) of worker w: split by cumulative request count
    auto cut = [&](int k) -> int32_t {
      const int64_t target = trace_offsets[0] + total * k / nt;
      return (int32_t)(std::lower_bound(trace_offsets, trace_offsets + n_traces, target) -
                       trace_offsets);
    };
    const int32_t t0 = w == 0 ? 0 : cut(w), t1 = w == nt - 1 ? n_traces : cut(w + 1);
    for (int32_t t = t0; t < t1; ++t) {
      int64_t allocs = 0;
      for (int64_t i = trace_offsets[t]; i < trace_offsets[t + 1]; ++i) {
        const pm_req_t& r = reqs[i];
        const uint32_t kind = r.kind_stream & 3u;
        if (kind == PM_KIND_ALLOC && (r.kind_stream >> 2) == 0 &&
            r.handle == allocs && r.size >= 1 && r.size < (int64_t)(1ll << 62)) {
          words[i] = (uint64_t)r.size;
          ++allocs;
        } else if (kind == PM_KIND_FREE && r.handle >= 0) {
          words[i] = PM_WIRE_FREE | (uint64_t)(uint32_t)r.handle;
        } else {
          bad[w] = i;
          return;
        }
      }
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w) th.emplace_back(work, w);
    for (auto& x : th) x.join();
  }
  const int64_t b = *std::min_element(bad.begin(), bad.end());
  if (b != INT64_MAX) {
    if (first_bad) *first_bad = b;
    return fail(PM_ERR_INVALID_ARGUMENT,
                "pm_wire_pack: request " + std::to_string(b) + " has no wire encoding");
  }
  return PM_SUCCESS;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Batched capacity bisection: the smallest device capacity
// each trace runs in, by bisection over many replays of the whole batch.
//
// The capacity enters the reference only through `reserved + seg > cap`
// (allocator.py:258-287, 328-333), and reserved / seg are sums of segment
// sizes, all multiples of u = gcd(k_small_buffer, k_large_buffer,
// k_round_large) (segment_size_for, allocator.py:86-92).  So a run at
// capacity C equals the run at floor(C/u)*u and the answer is a multiple of
// u.  Bracket: the unbounded peak_reserved runs (that run never exceeds
// it); below, capacity 0 OOMs on the first allocation, and when every block
// is splittable (max_split_size None) so does anything below the unbounded
// peak_allocated (reserved >= allocated = the sum of rounded live sizes).
// Each round replays only the traces still bracketing, each at its own
// midpoint (one pm_cfg_t per trace), until hi - lo == u.

namespace {

__device__ __host__ inline int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

struct CapLayout {
  size_t replay, tcfg, iota, lo, hi, unit, active, count, res, total;
};

CapLayout cap_layout_for(int64_t total_events, int64_t max_trace_events,
                         int32_t n_traces) {
  CapLayout C;
  const size_t n = (size_t)(n_traces > 0 ? n_traces : 1);
  size_t off = 0;
  C.replay = off;
  off = align_up(off + layout_for(total_events, max_trace_events, n_traces).total, 256);
  C.tcfg = off;
  off = align_up(off + sizeof(pm_cfg_t) * n, 256);
  C.iota = off;
  off = align_up(off + 4 * n, 256);
  C.lo = off;
  off = align_up(off + 8 * n, 256);
  C.hi = off;
  off = align_up(off + 8 * n, 256);
  C.unit = off;
  off = align_up(off + 8 * n, 256);
  C.active = off;
  off = align_up(off + 4 * n, 256);
  C.count = off;
  off = align_up(off + 8, 256);
  C.res = off;
  off = align_up(off + sizeof(pm_result_t) * n, 256);
  C.total = off;
  return C;
}

__global__ void cap_prepare_kernel(const pm_cfg_t* __restrict__ cfgs,
                                   const int32_t* __restrict__ cfg_of,
                                   int32_t n, pm_cfg_t* __restrict__ tcfg,
                                   int32_t* __restrict__ iota,
                                   int32_t* __restrict__ n_probes) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  pm_cfg_t c = cfgs[cfg_of ? cfg_of[t] : 0];
  c.device_capacity = -1;  // round 0: unbounded
  tcfg[t] = c;
  iota[t] = t;
  n_probes[t] = 0;
}

// after round 0: bracket each trace (lo OOMs, hi runs), in units of u
__global__ void cap_bracket_kernel(const pm_result_t* __restrict__ r0,
                                   const pm_cfg_t* __restrict__ tcfg, int32_t n,
                                   int64_t* __restrict__ lo, int64_t* __restrict__ hi,
                                   int64_t* __restrict__ unit,
                                   int64_t* __restrict__ min_cap,
                                   pm_result_t* __restrict__ unbounded) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const pm_result_t r = r0[t];
  if (unbounded) unbounded[t] = r;
  const pm_cfg_t c = tcfg[t];
  const int64_t u = gcd64(gcd64(c.k_small_buffer, c.k_large_buffer), c.k_round_large);
  unit[t] = u;
  if (r.status != PM_OK) {  // malformed: no capacity answer
    lo[t] = hi[t] = 0;
    min_cap[t] = -1;
    return;
  }
  // with max_split_size None every block is split to its rounded size, so
  // allocated bytes do not depend on the capacity and any C below the
  // unbounded peak_allocated OOMs; an unsplit oversize block (max_split
  // set) makes allocated capacity-dependent, so the bracket starts at 0
  lo[t] = (c.max_split_size < 0 && r.peak_allocated > 0)
              ? (r.peak_allocated - 1) / u : -1;
  hi[t] = r.peak_reserved / u;
  min_cap[t] = 0;  // pending: cap_finish_kernel writes hi * u
}

// one block: the traces still bracketing (in LPT order) get their midpoint
__global__ void cap_select_kernel(const int32_t* __restrict__ order, int32_t n,
                                  const int64_t* __restrict__ lo,
                                  const int64_t* __restrict__ hi,
                                  const int64_t* __restrict__ unit,
                                  pm_cfg_t* __restrict__ tcfg,
                                  int32_t* __restrict__ active,
                                  int64_t* __restrict__ count) {
  __shared__ int warp_sum[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int start = 0; start < n; start += blockDim.x) {
    const int i = start + threadIdx.x;
    const int t = i < n ? (order ? order[i] : i) : -1;
    const bool on = t >= 0 && hi[t] - lo[t] > 1;
    if (on) tcfg[t].device_capacity = (lo[t] + (hi[t] - lo[t]) / 2) * unit[t];
    const unsigned m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) warp_sum[w] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      if (k < w) before += warp_sum[k];
      total += warp_sum[k];
    }
    if (on) active[base + before + __popc(m & ((1u << lane) - 1))] = t;
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

__global__ void cap_update_kernel(const int32_t* __restrict__ active, int32_t m,
                                  const pm_result_t* __restrict__ res,
                                  const pm_cfg_t* __restrict__ tcfg,
                                  const int64_t* __restrict__ unit,
                                  int64_t* __restrict__ lo, int64_t* __restrict__ hi,
                                  int64_t* __restrict__ min_cap,
                                  int32_t* __restrict__ n_probes,
                                  int64_t* __restrict__ probe_capacity,
                                  pm_result_t* __restrict__ probe_results,
                                  int32_t max_probes, int32_t n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int t = active[i];
  const pm_result_t r = res[t];
  const int64_t cap = tcfg[t].device_capacity;
  const int k = n_probes[t]++;
  if (k < max_probes) {
    if (probe_capacity) probe_capacity[(size_t)k * n + t] = cap;
    if (probe_results) probe_results[(size_t)k * n + t] = r;
  }
  if (r.status == PM_OOM) {
    lo[t] = cap / unit[t];
  } else if (r.status == PM_OK) {
    hi[t] = cap / unit[t];
  } else {  // cannot happen after a clean unbounded run; stop the search
    lo[t] = hi[t] - 1;
    min_cap[t] = -2;
  }
}

__global__ void cap_finish_kernel(int32_t n, const int64_t* __restrict__ hi,
                                  const int64_t* __restrict__ unit,
                                  int64_t* __restrict__ min_cap) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (min_cap[t] == 0) min_cap[t] = hi[t] * unit[t];
}

}  // namespace

extern "C" {

int pm_capacity_workspace_bytes(int64_t total_events, int64_t max_trace_events,
                                int32_t n_traces, size_t* out_bytes) {
  if (!out_bytes || total_events < 0 || max_trace_events < 0 || n_traces < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_capacity_workspace_bytes: bad args");
  *out_bytes = cap_layout_for(total_events, max_trace_events, n_traces).total;
  return PM_SUCCESS;
}

int pm_capacity_search(const pm_req_t* reqs, const int64_t* trace_offsets,
                       int32_t n_traces, const pm_cfg_t* cfgs,
                       const int32_t* cfg_of_trace, const int32_t* trace_order,
                       int64_t* min_capacity, int32_t* n_probes,
                       pm_result_t* unbounded, int64_t* probe_capacity,
                       pm_result_t* probe_results, int32_t max_probes,
                       void* workspace, size_t workspace_bytes,
                       int64_t total_events, int64_t max_trace_events,
                       void* stream_) {
  if (n_traces < 0 || max_probes < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_capacity_search: negative size");
  if (n_traces == 0) return PM_SUCCESS;
  if (!min_capacity || !n_probes || !cfgs || !workspace)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_capacity_search: null argument");
  const CapLayout C = cap_layout_for(total_events, max_trace_events, n_traces);
  if (workspace_bytes < C.total)
    return fail(PM_ERR_WORKSPACE_TOO_SMALL,
                "pm_capacity_search: workspace smaller than "
                "pm_capacity_workspace_bytes()");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  char* base = static_cast<char*>(workspace);
  void* rws = base + C.replay;
  const size_t rws_bytes = C.tcfg - C.replay;
  pm_cfg_t* tcfg = reinterpret_cast<pm_cfg_t*>(base + C.tcfg);
  int32_t* iota = reinterpret_cast<int32_t*>(base + C.iota);
  int64_t* lo = reinterpret_cast<int64_t*>(base + C.lo);
  int64_t* hi = reinterpret_cast<int64_t*>(base + C.hi);
  int64_t* unit = reinterpret_cast<int64_t*>(base + C.unit);
  int32_t* active = reinterpret_cast<int32_t*>(base + C.active);
  int64_t* count = reinterpret_cast<int64_t*>(base + C.count);
  pm_result_t* res = reinterpret_cast<pm_result_t*>(base + C.res);
  const unsigned blocks = (unsigned)((n_traces + 255) / 256);

  cap_prepare_kernel<<<blocks, 256, 0, stream>>>(cfgs, cfg_of_trace, n_traces,
                                                  tcfg, iota, n_probes);
  int rc = replay_batch_impl(reqs, trace_offsets, n_traces, tcfg, iota,
                             trace_order, res, nullptr, rws, rws_bytes,
                             total_events, max_trace_events, stream_, nullptr,
                             0, nullptr);
  if (rc != PM_SUCCESS) return rc;
  cap_bracket_kernel<<<blocks, 256, 0, stream>>>(res, tcfg, n_traces, lo, hi,
                                                  unit, min_capacity, unbounded);
  int64_t* h_count = nullptr;
  cudaError_t e = cudaMallocHost((void**)&h_count, sizeof(int64_t));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  for (int round = 0; round < 64; ++round) {
    cap_select_kernel<<<1, 1024, 0, stream>>>(trace_order, n_traces, lo, hi,
                                              unit, tcfg, active, count);
    e = cudaMemcpyAsync(h_count, count, sizeof(int64_t), cudaMemcpyDeviceToHost,
                        stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
      cudaFreeHost(h_count);
      return cuda_fail(e, "pm_capacity_search: round sync");
    }
    const int32_t m = (int32_t)*h_count;
    if (m == 0) break;
    rc = replay_batch_impl(reqs, trace_offsets, m, tcfg, iota, active, res,
                           nullptr, rws, rws_bytes, total_events,
                           max_trace_events, stream_, nullptr, 0, nullptr);
    if (rc != PM_SUCCESS) {
      cudaFreeHost(h_count);
      return rc;
    }
    cap_update_kernel<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(
        active, m, res, tcfg, unit, lo, hi, min_capacity, n_probes,
        probe_capacity, probe_results, max_probes, n_traces);
  }
  cudaFreeHost(h_count);
  cap_finish_kernel<<<blocks, 256, 0, stream>>>(n_traces, hi, unit, min_capacity);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pm_capacity_search launch");
  return PM_SUCCESS;
}

}  // extern "C"

