// Batched caching-allocator replay for sm_100a: one warp per trace.
//
// Restates the state machine of peakmem.allocator.AllocatorState
// (reference pkg/src/peakmem/allocator.py:155-357) and replay()
// (allocator.py:360-393) for thousands of independent traces at once.
//
// Data layout (per trace, owned by one warp):
//   * free pool   -- every free block of the trace, as an UNSORTED array of
//                    (addr, key) pairs in shared memory (capacity KS; a trace
//                    that outgrows it is re-run by the global-pool variant).
//                    key = at_start<<63 | at_end<<62 | stream<<46 | size.
//                    Best fit (allocator.py:203-221, restated in SURVEY
//                    App. B as argmin (size, addr) over same-stream blocks
//                    with rounded <= size < rounded + max_split) is a
//                    lane-parallel scan + redux argmin.
//   * records     -- one 16 B record per handle in HBM: (addr, key) of the
//                    allocated block, 0 = never used, key ~0 = freed.
//                    Handles are dense per trace (< n_events), so the table
//                    sits at the trace's own event offset.
//   * no chains   -- the reference keeps doubly linked block chains per
//                    segment (allocator.py:95-132).  Here a block only needs
//                    to know whether it touches its segment's start / end:
//                    the free neighbour that coalescing (allocator.py:
//                    301-318) merges is the pool entry ending at addr (prev)
//                    or starting at addr+size (next), which is inside the
//                    same segment exactly when the freed block is not at the
//                    segment edge on that side.  A segment is wholly free
//                    (allocator.py:131-132) iff a pool entry has both flags.
//   * scalars     -- reserved / allocated / peaks / next_base / segment
//                    counts are warp-uniform registers.
//
// Requests are read 32 at a time with one coalesced 128-bit load per lane;
// the handles' records are gathered for the whole chunk at once and staged
// in shared memory; in-chunk reuse of a handle is forwarded with a ballot
// (last earlier lane with the same handle) instead of a reload.

#include <cuda_runtime.h>
#include <stdint.h>

#include "peakmem_b200.h"

namespace pmb {

typedef unsigned long long u64;

constexpr int kSizeBits = 46;
constexpr u64 kSizeMask = (1ull << kSizeBits) - 1;
constexpr u64 kStreamMask = 0xFFFFull << kSizeBits;
constexpr u64 kAtEnd = 1ull << 62;
constexpr u64 kAtStart = 1ull << 63;
constexpr u64 kKeyMask = kAtEnd - 1;  // stream | size
constexpr u64 kBoth = kAtStart | kAtEnd;
constexpr u64 kFreed = ~0ull;
constexpr unsigned kFull = 0xffffffffu;

struct Cfg {
  long long small_size, small_buffer, min_large, large_buffer, round_large,
      alignment, max_split, capacity;
};

struct WarpState {
  long long reserved, allocated, peak_reserved, peak_allocated, next_base;
  int F, nseg, nseg_peak, maxF;
};

// argmin over lanes of (k, a) among `valid` lanes; -1 if none.  Keys and
// addresses are < 2^63 so 0xffffffff halves never collide with a winner
// once the `c` chain gates them.
__device__ __forceinline__ int warp_argmin(bool valid, u64 k, u64 a) {
  unsigned any = __ballot_sync(kFull, valid);
  if (!any) return -1;
  if ((any & (any - 1)) == 0) return __ffs(any) - 1;
  unsigned khi = valid ? (unsigned)(k >> 32) : 0xffffffffu;
  unsigned m = __reduce_min_sync(kFull, khi);
  bool c = valid && khi == m;
  unsigned klo = c ? (unsigned)k : 0xffffffffu;
  m = __reduce_min_sync(kFull, klo);
  c = c && (unsigned)k == m;
  unsigned bm = __ballot_sync(kFull, c);
  if ((bm & (bm - 1)) == 0) return __ffs(bm) - 1;
  unsigned ahi = c ? (unsigned)(a >> 32) : 0xffffffffu;
  m = __reduce_min_sync(kFull, ahi);
  c = c && (unsigned)(a >> 32) == m;
  unsigned alo = c ? (unsigned)a : 0xffffffffu;
  m = __reduce_min_sync(kFull, alo);
  c = c && (unsigned)a == m;
  bm = __ballot_sync(kFull, c);
  return __ffs(bm) - 1;
}

// allocator.py:86-92
__device__ __forceinline__ long long segment_size_for(long long rounded,
                                                      const Cfg& c) {
  if (rounded <= c.small_size) return c.small_buffer;
  if (rounded <= c.min_large) return c.large_buffer;
  return ((rounded + c.round_large - 1) / c.round_large) * c.round_large;
}

// Remove pool slot s by moving the last entry into it (single lane).
__device__ __forceinline__ void pool_remove_lane(u64* pa, u64* pk, int s,
                                                 int F) {
  pa[s] = pa[F - 1];
  pk[s] = pk[F - 1];
}

// _make_room (allocator.py:258-271): stage 1 releases wholly-free segments
// above max_split, largest first (ties: creation order == ascending base),
// stopping as soon as the new segment fits; stage 2 releases every
// wholly-free segment.
__device__ __forceinline__ void make_room(WarpState& w, u64* pa, u64* pk,
                                          long long seg, const Cfg& c,
                                          int lane) {
  if (c.max_split >= 0) {
    while (w.reserved + seg > c.capacity) {
      u64 bk = ~0ull, ba = ~0ull;
      int bs = -1;
      for (int s = lane; s < w.F; s += 32) {
        u64 k = pk[s];
        long long sz = (long long)(k & kSizeMask);
        if ((k & kBoth) == kBoth && sz > c.max_split) {
          u64 kk = kSizeMask - (u64)sz;  // min kk == max size
          u64 a = pa[s];
          if (kk < bk || (kk == bk && a < ba)) {
            bk = kk;
            ba = a;
            bs = s;
          }
        }
      }
      int wl = warp_argmin(bs >= 0, bk, ba);
      if (wl < 0) break;
      int slot = __shfl_sync(kFull, bs, wl);
      long long sz = (long long)(pk[slot] & kSizeMask);
      __syncwarp();
      if (lane == 0) pool_remove_lane(pa, pk, slot, w.F);
      __syncwarp();
      w.F -= 1;
      w.reserved -= sz;
      w.nseg -= 1;
    }
  }
  if (w.reserved + seg > c.capacity) {
    long long reserved = w.reserved;
    int F = w.F, nseg = w.nseg;
    if (lane == 0) {
      int s = 0;
      while (s < F) {
        u64 k = pk[s];
        if ((k & kBoth) == kBoth) {
          reserved -= (long long)(k & kSizeMask);
          nseg -= 1;
          pool_remove_lane(pa, pk, s, F);
          F -= 1;
        } else {
          ++s;
        }
      }
    }
    __syncwarp();
    w.reserved = __shfl_sync(kFull, reserved, 0);
    w.F = __shfl_sync(kFull, F, 0);
    w.nseg = __shfl_sync(kFull, nseg, 0);
  }
}

// One trace, replayed by the calling warp.  Returns the status; fills *res.
// pa/pk: pool arrays (shared or global), pool_cap entries.
// st_a/st_k: 32-entry per-warp staging of the chunk's records.
__device__ __forceinline__ void replay_trace(
    int tr, const pm_req_t* __restrict__ reqs,
    const int64_t* __restrict__ offs, const pm_cfg_t* __restrict__ cfgs,
    const int32_t* __restrict__ cfg_of, pm_result_t* __restrict__ results,
    int64_t* __restrict__ timeline, ulonglong2* __restrict__ rec_base,
    u64* pa, u64* pk, int pool_cap, u64* st_a, u64* st_k, int lane) {
  const long long e0 = offs[tr];
  const long long n = offs[tr + 1] - e0;
  const pm_cfg_t* cp = cfgs + (cfg_of ? cfg_of[tr] : 0);
  Cfg c;
  c.small_size = cp->k_small_size;
  c.small_buffer = cp->k_small_buffer;
  c.min_large = cp->k_min_large_alloc;
  c.large_buffer = cp->k_large_buffer;
  c.round_large = cp->k_round_large;
  c.alignment = cp->alignment;
  c.max_split = cp->max_split_size;
  c.capacity = cp->device_capacity;
  const u64 amask = (u64)c.alignment - 1;

  ulonglong2* recs = rec_base + e0;
  const ulonglong2 zero2 = make_ulonglong2(0ull, 0ull);
  for (long long i = lane; i < n; i += 32) recs[i] = zero2;
  __syncwarp();

  WarpState w;
  w.reserved = w.allocated = w.peak_reserved = w.peak_allocated = 0;
  w.next_base = 0;
  w.F = 0;
  w.nseg = w.nseg_peak = 0;
  w.maxF = 0;
  int status = PM_OK;
  long long stop = -1;

  const ulonglong2* rq = reinterpret_cast<const ulonglong2*>(reqs + e0);
  // prefetch of the next chunk's requests (one 128-bit load per lane)
  ulonglong2 nxt = make_ulonglong2(0ull, 0xFFFFFFFFull);
  if (lane < n) nxt = __ldg(rq + lane);

  for (long long cbase = 0; cbase < n; cbase += 32) {
    const ulonglong2 ev = nxt;
    if (cbase + 32 + lane < n) nxt = __ldg(rq + cbase + 32 + lane);
    const long long my_size = (long long)ev.x;
    const int my_h = (int)(unsigned)(ev.y & 0xffffffffull);
    const unsigned my_ks = (unsigned)(ev.y >> 32);
    const bool my_valid = cbase + lane < n;
    const bool hok = my_valid && my_h >= 0 && (long long)my_h < n;
    ulonglong2 r = zero2;
    if (hok) r = recs[my_h];
    st_a[lane] = r.x;
    st_k[lane] = r.y;
    const int hcmp = my_valid ? my_h : -1;  // never matches a valid handle
    __syncwarp();

    const int cnt = (int)((n - cbase) < 32 ? (n - cbase) : 32);
    long long tl_r = 0, tl_a = 0;
    int done = cnt;
    for (int j = 0; j < cnt; ++j) {
      const long long size = __shfl_sync(kFull, my_size, j);
      const int hj = __shfl_sync(kFull, my_h, j);
      const unsigned ks = __shfl_sync(kFull, my_ks, j);
      const unsigned kind = ks & 3u;
      const unsigned strm = ks >> 2;
      int st = PM_OK;
      if (kind == PM_KIND_UNKNOWN) {
        st = PM_UNKNOWN_KIND;
      } else if (kind == PM_KIND_MISSING_FIELD) {
        st = PM_MISSING_FIELD;
      } else if (hj < 0 || (long long)hj >= n) {
        st = PM_BAD_HANDLE;
      }
      unsigned m = __ballot_sync(kFull, hcmp == hj) & ((1u << j) - 1u);
      const int src = m ? 31 - __clz(m) : j;
      const u64 ra = st_a[src];
      const u64 rk = st_k[src];
      u64 out_a = 0, out_k = 0;
      if (st == PM_OK && kind == PM_KIND_ALLOC) {
        // allocate (allocator.py:273-292); precedence: duplicate, then
        // zero size (round_request, allocator.py:79-83)
        if (rk != 0) {
          st = PM_DUPLICATE_HANDLE;
        } else if (size <= 0) {
          st = PM_ZERO_SIZE;
        } else if (strm > 0xFFFFu) {
          st = PM_BAD_STREAM;
        } else {
          const u64 rounded = ((u64)size + amask) & ~amask;
          if (rounded > kSizeMask) {
            st = PM_SIZE_LIMIT;
          } else {
            const u64 sbits = (u64)strm << kSizeBits;
            const u64 lo = sbits | rounded;
            u64 span = kSizeMask + 1 - rounded;
            if (c.max_split >= 0 && (u64)c.max_split < span)
              span = (u64)c.max_split;
            // best fit: argmin (size, addr), same stream,
            // rounded <= size < rounded + max_split
            u64 bk = ~0ull, ba = ~0ull;
            int bs = -1;
            const int F = w.F;
            int s0 = lane;
            for (; s0 + 96 < F; s0 += 128) {
              u64 k4[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) k4[u] = pk[s0 + 32 * u] & kKeyMask;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                if (k4[u] - lo < span) {
                  const u64 a = pa[s0 + 32 * u];
                  if (k4[u] < bk || (k4[u] == bk && a < ba)) {
                    bk = k4[u];
                    ba = a;
                    bs = s0 + 32 * u;
                  }
                }
              }
            }
            for (; s0 < F; s0 += 32) {
              const u64 k = pk[s0] & kKeyMask;
              if (k - lo < span) {
                const u64 a = pa[s0];
                if (k < bk || (k == bk && a < ba)) {
                  bk = k;
                  ba = a;
                  bs = s0;
                }
              }
            }
            const int wl = warp_argmin(bs >= 0, bk, ba);
            if (wl >= 0) {
              // hit: _take (allocator.py:234-242) with _split (:223-232)
              const int slot = __shfl_sync(kFull, bs, wl);
              const u64 key = pk[slot];
              const u64 A = pa[slot];
              const u64 S = key & kSizeMask;
              const bool splittable =
                  c.max_split < 0 || (long long)S <= c.max_split;
              __syncwarp();
              if (splittable && S > rounded) {
                out_k = (key & (kAtStart | kStreamMask)) | rounded;
                if (lane == 0) {
                  pa[slot] = A + rounded;
                  pk[slot] = (key & (kAtEnd | kStreamMask)) | (S - rounded);
                }
              } else {
                out_k = key;
                if (lane == 0) pool_remove_lane(pa, pk, slot, w.F);
                w.F -= 1;
              }
              out_a = A;
              __syncwarp();
            } else {
              // miss: new segment (allocator.py:278-288, 244-250)
              const long long seg = segment_size_for((long long)rounded, c);
              if (c.capacity >= 0 && w.reserved + seg > c.capacity) {
                make_room(w, pa, pk, seg, c, lane);
                if (w.reserved + seg > c.capacity) st = PM_OOM;
              }
              if (st == PM_OK) {
                if ((u64)seg > kSizeMask) {
                  st = PM_SIZE_LIMIT;
                } else {
                  const u64 A = (u64)w.next_base;
                  w.next_base += seg;
                  w.reserved += seg;
                  w.nseg += 1;
                  w.nseg_peak = max(w.nseg_peak, w.nseg);
                  const bool splittable =
                      c.max_split < 0 || seg <= c.max_split;
                  if (splittable && (u64)seg > rounded) {
                    if (w.F >= pool_cap) {
                      st = PM_POOL_OVERFLOW;
                    } else {
                      out_k = kAtStart | sbits | rounded;
                      if (lane == 0) {
                        pa[w.F] = A + rounded;
                        pk[w.F] = kAtEnd | sbits | ((u64)seg - rounded);
                      }
                      w.F += 1;
                    }
                  } else {
                    out_k = kBoth | sbits | (u64)seg;
                  }
                  out_a = A;
                  __syncwarp();
                }
              }
            }
            if (st == PM_OK) {
              w.allocated += (long long)(out_k & kSizeMask);
              w.peak_reserved = max(w.peak_reserved, w.reserved);
              w.peak_allocated = max(w.peak_allocated, w.allocated);
              w.maxF = max(w.maxF, w.F);
              if (lane == j) {
                st_a[j] = out_a;
                st_k[j] = out_k;
                recs[hj] = make_ulonglong2(out_a, out_k);
              }
            }
          }
        }
      } else if (st == PM_OK) {
        // free (allocator.py:294-320): double free before unknown handle
        if (rk == kFreed) {
          st = PM_DOUBLE_FREE;
        } else if (rk == 0) {
          st = PM_UNKNOWN_HANDLE;
        } else {
          const u64 A = ra;
          const u64 S = rk & kSizeMask;
          const bool fs = (rk & kAtStart) != 0;
          const bool fe = (rk & kAtEnd) != 0;
          w.allocated -= (long long)S;
          const u64 endA = A + S;
          int ns = -1, ps = -1;
          const int F = w.F;
          int s0 = lane;
          for (; s0 + 96 < F; s0 += 128) {
            u64 a4[4], k4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              a4[u] = pa[s0 + 32 * u];
              k4[u] = pk[s0 + 32 * u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (!fe && a4[u] == endA) ns = s0 + 32 * u;
              if (!fs && a4[u] + (k4[u] & kSizeMask) == A) ps = s0 + 32 * u;
            }
          }
          for (; s0 < F; s0 += 32) {
            const u64 a = pa[s0];
            if (!fe && a == endA) ns = s0;
            if (!fs && a + (pk[s0] & kSizeMask) == A) ps = s0;
          }
          const unsigned bn = __ballot_sync(kFull, ns >= 0);
          const unsigned bp = __ballot_sync(kFull, ps >= 0);
          const int nslot = bn ? __shfl_sync(kFull, ns, __ffs(bn) - 1) : -1;
          const int pslot = bp ? __shfl_sync(kFull, ps, __ffs(bp) - 1) : -1;
          if (nslot < 0 && pslot < 0) {
            if (w.F >= pool_cap) {
              st = PM_POOL_OVERFLOW;
            } else {
              if (lane == 0) {
                pa[w.F] = A;
                pk[w.F] = rk;
              }
              w.F += 1;
              w.maxF = max(w.maxF, w.F);
            }
          } else {
            __syncwarp();
            if (lane == 0) {
              if (nslot < 0) {  // merge into prev
                pk[pslot] = (pk[pslot] + S) | (rk & kAtEnd);
              } else if (pslot < 0) {  // absorb next
                const u64 nk = pk[nslot];
                pa[nslot] = A;
                pk[nslot] = (nk + S) | (rk & kAtStart);
              } else {  // prev absorbs self and next
                const u64 nk = pk[nslot];
                pk[pslot] = (pk[pslot] + S + (nk & kSizeMask)) | (nk & kAtEnd);
                pool_remove_lane(pa, pk, nslot, w.F);
              }
            }
            if (nslot >= 0 && pslot >= 0) w.F -= 1;
          }
          __syncwarp();
          if (st == PM_OK && lane == j) {
            st_k[j] = kFreed;
            recs[hj].y = kFreed;
          }
        }
      }
      if (st != PM_OK) {
        status = st;
        stop = cbase + j;
        done = j;
        break;
      }
      if (lane == j) {
        tl_r = w.reserved;
        tl_a = w.allocated;
      }
      __syncwarp();
    }
    if (timeline != nullptr && lane < done) {
      long long gi = e0 + cbase + lane;
      reinterpret_cast<longlong2*>(timeline)[gi] = make_longlong2(tl_r, tl_a);
    }
    if (status != PM_OK) break;
  }

  if (lane == 0) {
    pm_result_t res;
    res.peak_reserved = w.peak_reserved;
    res.peak_allocated = w.peak_allocated;
    res.final_reserved = w.reserved;
    res.final_allocated = w.allocated;
    res.stop_index = stop;
    res.n_events_replayed =
        status == PM_OK ? n : (status == PM_OOM ? stop + 1 : stop);
    res.status = status;
    res.n_segments_final = w.nseg;
    res.n_segments_peak = w.nseg_peak;
    res.max_free_blocks = w.maxF;
    results[tr] = res;
  }
}

struct Ctl {
  unsigned work;        // main-kernel work counter
  unsigned n_retry;     // traces whose pool outgrew shared memory
  unsigned retry_work;  // retry-kernel work counter
  unsigned pad[61];
};

// Main kernel: persistent warps pull traces (longest first) from a global
// counter; each warp's free pool lives in dynamic shared memory
// (pool_cap entries of 16 B) next to its 32-entry record staging area.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    replay_smem_kernel(const pm_req_t* __restrict__ reqs,
                       const int64_t* __restrict__ offs, int n_traces,
                       const pm_cfg_t* __restrict__ cfgs,
                       const int32_t* __restrict__ cfg_of,
                       const int32_t* __restrict__ order,
                       pm_result_t* __restrict__ results,
                       int64_t* __restrict__ timeline,
                       ulonglong2* __restrict__ recs, Ctl* ctl,
                       int32_t* __restrict__ retry_list, int pool_cap) {
  extern __shared__ u64 smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  u64* pa = smem + (size_t)wib * (2 * pool_cap + 64);
  u64* pk = pa + pool_cap;
  u64* st_a = pk + pool_cap;
  u64* st_k = st_a + 32;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&ctl->work, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= (unsigned)n_traces) break;
    const int tr = order ? order[t] : (int)t;
    replay_trace(tr, reqs, offs, cfgs, cfg_of, results, timeline, recs, pa,
                 pk, pool_cap, st_a, st_k, lane);
    __syncwarp();
    if (lane == 0 && results[tr].status == PM_POOL_OVERFLOW) {
      unsigned k = atomicAdd(&ctl->n_retry, 1u);
      retry_list[k] = tr;
    }
  }
}

// Traces whose free pool outgrew shared memory: same replay with the pool in
// a per-warp HBM region of 2*max_events+2 entries (free blocks never exceed
// live allocations + live segments <= 2 * allocations).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    replay_gpool_kernel(const pm_req_t* __restrict__ reqs,
                        const int64_t* __restrict__ offs,
                        const pm_cfg_t* __restrict__ cfgs,
                        const int32_t* __restrict__ cfg_of,
                        pm_result_t* __restrict__ results,
                        int64_t* __restrict__ timeline,
                        ulonglong2* __restrict__ recs, Ctl* ctl,
                        const int32_t* __restrict__ retry_list,
                        u64* __restrict__ gpool, long long gpool_cap) {
  __shared__ u64 s_sa[WARPS][32];
  __shared__ u64 s_sk[WARPS][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * WARPS + wib;
  u64* pa = gpool + gw * 2 * gpool_cap;
  u64* pk = pa + gpool_cap;
  const unsigned n_retry = ctl->n_retry;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&ctl->retry_work, 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= n_retry) break;
    const int tr = retry_list[t];
    replay_trace(tr, reqs, offs, cfgs, cfg_of, results, timeline, recs, pa,
                 pk, (int)(gpool_cap < 0x7fffffff ? gpool_cap : 0x7fffffff),
                 s_sa[wib], s_sk[wib], lane);
  }
}

}  // namespace pmb

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

constexpr int kDefaultPoolCap = 1024;  // shared-memory pool entries per warp
constexpr int kWarps = 4;              // warps (traces in flight) per CTA
constexpr int kRetryWarps = 4;
constexpr int kMaxRetryCtas = 64;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// workspace = ctl | retry list | retry pools | record table
struct Layout {
  size_t retry_list, gpool, recs, total;
  long long gpool_cap;
  int retry_ctas;
};

Layout layout_for(int64_t total_events, int64_t max_trace_events,
                  int32_t n_traces) {
  Layout L;
  size_t off = align_up(sizeof(pmb::Ctl), 256);
  L.retry_list = off;
  off = align_up(off + sizeof(int32_t) * (size_t)(n_traces > 0 ? n_traces : 1),
                 256);
  L.gpool_cap = 2 * (max_trace_events > 0 ? max_trace_events : 1) + 2;
  int ctas = (n_traces + kRetryWarps - 1) / kRetryWarps;
  if (ctas > kMaxRetryCtas) ctas = kMaxRetryCtas;
  if (ctas < 1) ctas = 1;
  L.retry_ctas = ctas;
  L.gpool = off;
  off = align_up(off + (size_t)ctas * kRetryWarps * 2 * 8 * (size_t)L.gpool_cap,
                 256);
  L.recs = off;
  off = align_up(off + 16 * (size_t)(total_events > 0 ? total_events : 1), 256);
  L.total = off;
  return L;
}

struct Occupancy {
  int sms = 0, per_sm = 0, pool_cap = 0;
  size_t smem = 0;
};

int pool_cap_setting() {
  const char* env = getenv("PM_POOL_CAP");
  int cap = env ? atoi(env) : kDefaultPoolCap;
  if (cap < 32) cap = 32;
  if (cap > 4096) cap = 4096;
  return cap;
}

size_t smem_bytes_for(int pool_cap) {
  return (size_t)kWarps * (2 * (size_t)pool_cap + 64) * sizeof(pmb::u64);
}

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
    o.pool_cap = pool_cap_setting();
    o.smem = smem_bytes_for(o.pool_cap);
    e = cudaFuncSetAttribute(pmb::replay_smem_kernel<kWarps>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)o.smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &o.per_sm, pmb::replay_smem_kernel<kWarps>, kWarps * 32, o.smem);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    if (o.per_sm < 1) o.per_sm = 1;
    cached = o;
    cached_dev = dev;
  }
  *out = cached;
  return PM_SUCCESS;
}

}  // namespace

extern "C" {

const char* pm_last_error(void) { return g_last_error.c_str(); }

int pm_version(void) { return 1; }

int pm_replay_workspace_bytes(int64_t total_events, int64_t max_trace_events,
                              int32_t n_traces, size_t* out_bytes) {
  if (!out_bytes || total_events < 0 || max_trace_events < 0 || n_traces < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_workspace_bytes: bad args");
  *out_bytes = layout_for(total_events, max_trace_events, n_traces).total;
  return PM_SUCCESS;
}

int pm_replay_batch(const pm_req_t* reqs, const int64_t* trace_offsets,
                    int32_t n_traces, const pm_cfg_t* cfgs,
                    const int32_t* cfg_of_trace, const int32_t* trace_order,
                    pm_result_t* results, int64_t* timeline, void* workspace,
                    size_t workspace_bytes, int64_t total_events,
                    int64_t max_trace_events, void* stream_) {
  if (n_traces < 0 || total_events < 0 || max_trace_events < 0)
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_batch: negative size");
  if (n_traces == 0) return PM_SUCCESS;
  if (!trace_offsets || !cfgs || !results || !workspace ||
      (total_events > 0 && !reqs))
    return fail(PM_ERR_INVALID_ARGUMENT, "pm_replay_batch: null argument");
  const Layout L = layout_for(total_events, max_trace_events, n_traces);
  if (workspace_bytes < L.total)
    return fail(PM_ERR_WORKSPACE_TOO_SMALL,
                "pm_replay_batch: workspace smaller than "
                "pm_replay_workspace_bytes()");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  char* base = static_cast<char*>(workspace);
  pmb::Ctl* ctl = reinterpret_cast<pmb::Ctl*>(base);
  int32_t* retry_list = reinterpret_cast<int32_t*>(base + L.retry_list);
  pmb::u64* gpool = reinterpret_cast<pmb::u64*>(base + L.gpool);
  ulonglong2* recs = reinterpret_cast<ulonglong2*>(base + L.recs);

  Occupancy occ;
  int rc = query_occupancy(&occ);
  if (rc != PM_SUCCESS) return rc;
  cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(pmb::Ctl), stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  long long want = ((long long)n_traces + kWarps - 1) / kWarps;
  long long grid = (long long)occ.per_sm * occ.sms;
  if (want < grid) grid = want;
  pmb::replay_smem_kernel<kWarps>
      <<<(unsigned)grid, kWarps * 32, occ.smem, stream>>>(
          reqs, trace_offsets, n_traces, cfgs, cfg_of_trace, trace_order,
          results, timeline, recs, ctl, retry_list, occ.pool_cap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay_smem_kernel launch");
  pmb::replay_gpool_kernel<kRetryWarps>
      <<<L.retry_ctas, kRetryWarps * 32, 0, stream>>>(
          reqs, trace_offsets, cfgs, cfg_of_trace, results, timeline, recs,
          ctl, retry_list, gpool, L.gpool_cap);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "replay_gpool_kernel launch");
  return PM_SUCCESS;
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
  // longest trace first: the persistent warps then finish together
  std::vector<int32_t> order(n_traces);
  for (int32_t i = 0; i < n_traces; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return trace_offsets[a + 1] - trace_offsets[a] >
           trace_offsets[b + 1] - trace_offsets[b];
  });
  const Layout L = layout_for(total, max_ev, n_traces);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const size_t b_reqs = align_up(16 * (size_t)(total > 0 ? total : 1), 256);
  const size_t b_offs = align_up(8 * (size_t)(n_traces + 1), 256);
  const size_t b_cfgs = align_up(sizeof(pm_cfg_t) * (size_t)n_cfgs, 256);
  const size_t b_cfgof = align_up(4 * (size_t)n_traces, 256);
  const size_t b_order = b_cfgof;
  const size_t b_res = align_up(sizeof(pm_result_t) * (size_t)n_traces, 256);
  const size_t b_tl = timeline ? align_up(16 * (size_t)(total > 0 ? total : 1), 256) : 0;
  const size_t bytes =
      b_reqs + b_offs + b_cfgs + b_cfgof + b_order + b_res + b_tl + L.total;
  {
    // keep the stream-ordered pool's memory mapped between calls: the
    // default release threshold (0) unmaps it at every synchronisation
    static std::mutex mu;
    static int tuned_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      std::lock_guard<std::mutex> g(mu);
      if (tuned_dev != dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          uint64_t thr = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        tuned_dev = dev;
      }
    }
  }
  void* dmem = nullptr;
  cudaError_t e = cudaMallocAsync(&dmem, bytes, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
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
  if (total > 0)
    PM_CHECK(cudaMemcpyAsync(d_reqs, reqs, 16 * (size_t)total,
                             cudaMemcpyHostToDevice, stream), "H2D requests");
  PM_CHECK(cudaMemcpyAsync(d_offs, trace_offsets, 8 * (size_t)(n_traces + 1),
                           cudaMemcpyHostToDevice, stream), "H2D offsets");
  PM_CHECK(cudaMemcpyAsync(d_cfgs, cfgs, sizeof(pm_cfg_t) * (size_t)n_cfgs,
                           cudaMemcpyHostToDevice, stream), "H2D cfgs");
  if (cfg_of_trace)
    PM_CHECK(cudaMemcpyAsync(d_cfgof, cfg_of_trace, 4 * (size_t)n_traces,
                             cudaMemcpyHostToDevice, stream), "H2D cfg_of");
  PM_CHECK(cudaMemcpyAsync(d_order, order.data(), 4 * (size_t)n_traces,
                           cudaMemcpyHostToDevice, stream), "H2D order");
  rc = pm_replay_batch(d_reqs, d_offs, n_traces, d_cfgs,
                       cfg_of_trace ? d_cfgof : nullptr, d_order, d_res, d_tl,
                       d_ws, L.total, total, max_ev, stream_);
  if (rc != PM_SUCCESS) goto done;
  PM_CHECK(cudaMemcpyAsync(results, d_res, sizeof(pm_result_t) * (size_t)n_traces,
                           cudaMemcpyDeviceToHost, stream), "D2H results");
  if (timeline && total > 0)
    PM_CHECK(cudaMemcpyAsync(timeline, d_tl, 16 * (size_t)total,
                             cudaMemcpyDeviceToHost, stream), "D2H timeline");
done:
#undef PM_CHECK
  cudaFreeAsync(dmem, stream);
  e = cudaStreamSynchronize(stream);
  if (rc == PM_SUCCESS && e != cudaSuccess) rc = cuda_fail(e, "cudaStreamSynchronize");
  return rc;
}

}  // extern "C"
