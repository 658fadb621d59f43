// Narrow-encoded replay: the main pass of pm_replay_batch (sm_100a).
//
// Same state machine as replay_device.cuh (peakmem.allocator.AllocatorState,
// reference pkg/src/peakmem/allocator.py:155-393), same data structures, but
// every block size and address is held in *allocator units* as a 32-bit
// value.  Every block size and address the reference can produce is a
// multiple of
//
//     u = 2^s,  s = min(ctz(alignment), ctz(k_small_buffer),
//                       ctz(k_large_buffer), ctz(k_round_large))
//
// (rounded requests are multiples of the power-of-two alignment,
// allocator.py:79-83; segments are k_small_buffer, k_large_buffer or a
// multiple of k_round_large, :86-92; addresses are sums of both), so
// size_u = size >> s and addr_u = addr >> s are exact.  With that:
//
//  * a free block is ONE 64-bit word ka = size_u << 32 | addr_u, and the
//    best-fit order (size, addr) (allocator.py:203-221) is plain unsigned
//    order of ka: directory search, bucket split ranks and the argmin are
//    single 64-bit compares instead of (key, addr) pairs;
//  * a pool entry is 16 B (ka + links) instead of 24 B, so the CTA-shared
//    shared-memory pool holds 1.5x the entries and more traces fit per SM;
//  * an allocated-block record is 16 B (addr_u, size_u, left ref, right
//    ref): one 128-bit gather per request instead of four 64-bit loads.
//
// The encoding covers one stream (stream 0) and next_base_u < 2^32 - 1
// (2 TiB of segments ever reserved at u = 512).  A trace that leaves it
// (another stream, a larger block or address space) stops with
// PM_ENCODING_LIMIT and is replayed from the start by the wide tiers
// (replay_device.cuh); a trace whose free blocks outgrow the main pass's
// 32-bucket register directory or the CTA pool stops with PM_POOL_OVERFLOW
// and is replayed by the narrow memory-directory tiers below.  Results are
// bit-identical whichever tier finishes a trace.
//
// Per warp (one trace at a time):
//  * requests arrive 32 at a time by 1-D TMA bulk copy (cp.async.bulk +
//    mbarrier) into a shared double buffer, one chunk ahead; 8-byte wire
//    words (pm_replay_host_wire) are decoded there in place;
//  * each lane gathers its request's handle record; a per-trace handle
//    watermark says which records belong to this run (no table zeroing);
//    in-chunk reuse of a handle is forwarded with a ballot, and link
//    updates to a staged handle are mirrored into the staging copy;
//  * free blocks live in buckets of <= 32 entries with per-bucket occupancy
//    masks (a removal clears a bit; entries move only on split / merge),
//    indexed by a sorted directory in registers (lane d = position d: one
//    ballot finds a bucket) or, in the retry passes, in shared memory with
//    a register summary;
//  * the main pass's warps (24 per SM) share one shared-memory bucket pool
//    and wait for buckets when it runs dry (one victim per deadlocked CTA
//    escalates); config constants, peaks and counters that the allocation
//    path touches live in a per-warp shared record, keeping the kernel at 80
//    registers.
#pragma once

#include "replay_device.cuh"

namespace pmn {

using pmb::kBucket;
using pmb::kFreeTag;
using pmb::kFull;
using pmb::kHalf;
using pmb::kNone;
using pmb::is_free_ref;
using pmb::lanemask_lt;
using pmb::u32;
using pmb::u64;

#ifdef PM_STATS
// debug build only (tools/stats_replay.py): pool-operation counters
__device__ unsigned long long g_stats[16];
#define PM_STAT(i) \
  do {             \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_stats[i], 1ull); \
  } while (0)
#else
#define PM_STAT(i) ((void)0)
#endif

constexpr u32 kFreedU = 0xFFFFFFFFu;  // record size of a freed handle
constexpr u32 kMaxU = 0xFFFFFFFEu;    // sizes / addresses stay below this

__device__ __forceinline__ u32 hi(u64 x) { return (u32)(x >> 32); }
__device__ __forceinline__ u32 lo(u64 x) { return (u32)x; }
__device__ __forceinline__ u64 pk(u32 h, u32 l) {
  return ((u64)h << 32) | (u64)l;
}

// Free-block entries: ka = size_u << 32 | addr_u, ln = left | right << 32
// (neighbour handles or kNone).
struct NPool {
  u64* ka;
  u64* ln;
};

// Allocated-block records, 16 B per handle: x addr_u, y size_u (0 never
// allocated, kFreedU freed), z left ref, w right ref.
struct NRecs {
  uint4* base;
  __device__ __forceinline__ u32* word(u32 h, int w) const {
    return reinterpret_cast<u32*>(base + h) + w;  // w: immediate offset
  }
  __device__ __forceinline__ uint4* rec(u32 h) const { return base + h; }
};

// Directory in registers: lane d holds bucket position d -- its lower bound
// (packed ka), physical bucket and occupancy mask (bit i: slot i holds an
// entry).  Removing an entry clears its bit: entries never move between
// slots except on bucket split / merge, so their ids stay valid and the
// allocated neighbours' refs need no re-pointing.
struct NDir {
  static constexpr bool kResumes = false;  // the main pass starts traces fresh
  // find() on an empty directory gives -1, whose shuffled mask is 0
  static constexpr bool kEmptyFindSafe = true;
  // no soft size (32 positions at most)
  __device__ __forceinline__ bool soft_due() const { return false; }
  __device__ __forceinline__ void soft_failed() {}
  u64 db;
  int dp;
  unsigned dm;
  int nb;
  int lane;
  unsigned* cta_used;  // CTA-shared bitmap of physical buckets in use
  int cta_words, cta_buckets;

  __device__ __forceinline__ void init(int lane_) {
    db = ~0ull;
    dp = -1;
    dm = 0;
    nb = 0;
    lane = lane_;
  }
  // last position whose bound <= x (nb > 0: position 0's bound is 0)
  __device__ __forceinline__ int find(u64 x) const {
    return 31 - __clz(__ballot_sync(kFull, db <= x));
  }
  __device__ __forceinline__ int phys(int d) const {
    return __shfl_sync(kFull, dp, d);
  }
  __device__ __forceinline__ unsigned mask(int d) const {
    return __shfl_sync(kFull, dm, d);
  }
  __device__ __forceinline__ u64 bound(int d) const {
    return __shfl_sync(kFull, db, d);
  }
  __device__ __forceinline__ void set_bit(int d, int b) {
    if (lane == d) dm |= 1u << b;
  }
  __device__ __forceinline__ void clear_bit(int d, int b) {
    if (lane == d) dm &= ~(1u << b);
  }
  __device__ __forceinline__ void set_mask(int d, unsigned m) {
    if (lane == d) dm = m;
  }
  __device__ __forceinline__ int pos_of_phys(int p) const {
    return __ffs(__ballot_sync(kFull, dp == p)) - 1;
  }
  __device__ __forceinline__ int mergeable() const {
    const unsigned mn = __shfl_down_sync(kFull, dm, 1);
    const unsigned m = __ballot_sync(
        kFull, lane < nb - 1 && __popc(dm) + __popc(mn) <= kBucket);
    return m ? __ffs(m) - 1 : -1;
  }
  __device__ __forceinline__ void insert(int d, u64 b, int p, unsigned m) {
    const u64 ub = __shfl_up_sync(kFull, db, 1);
    const int up = __shfl_up_sync(kFull, dp, 1);
    const unsigned um = __shfl_up_sync(kFull, dm, 1);
    if (lane > d) {
      db = ub;
      dp = up;
      dm = um;
    } else if (lane == d) {
      db = b;
      dp = p;
      dm = m;
    }
    nb += 1;
  }
  __device__ __forceinline__ void erase(int d) {
    u64 nbd = __shfl_down_sync(kFull, db, 1);
    int np = __shfl_down_sync(kFull, dp, 1);
    unsigned nm = __shfl_down_sync(kFull, dm, 1);
    if (lane == 31) {
      nbd = ~0ull;
      np = -1;
      nm = 0;
    }
    if (lane >= d) {
      db = nbd;
      dp = np;
      dm = nm;
    }
    nb -= 1;
    if (d == 0 && lane == 0) db = 0;
  }
  __device__ __forceinline__ int alloc_phys() {
    int p = -1;
    PM_STAT(12);
    if (lane == 0) {
      for (int w = 0; w < cta_words && p < 0; ++w) {
        unsigned v = *(volatile unsigned*)&cta_used[w];
        while (v != 0xffffffffu) {
          const int b = __ffs(~v) - 1;
          const unsigned old = atomicOr(&cta_used[w], 1u << b);
          if (!(old & (1u << b))) {
            p = w * 32 + b;
            // acquire: the previous owner's accesses to the bucket precede ours
            __threadfence_block();
            break;
          }
          v = old | (1u << b);
        }
      }
      if (p >= cta_buckets) p = -1;
    }
    p = __shfl_sync(kFull, p, 0);
    // lane 0's acquire (atomic + fence) reaches the other lanes through the
    // warp barrier's memory ordering before any of them touches the bucket
    __syncwarp();
    return p;
  }
  // The CTA's pool is exhausted: wait for another warp to hand a bucket
  // back (buckets empty out continuously as free blocks are taken).  If
  // every warp replaying a trace in this CTA is waiting, ONE of them (the
  // holder of the victim token) returns -1: its trace escalates to the wide
  // tiers and its buckets go back to the others.  ctr[0] waiting warps,
  // ctr[1] active warps, ctr[2] victim token, after the bitmap.
  __device__ __forceinline__ int alloc_phys_wait() {
    int p = alloc_phys();
    if (p >= 0) return p;
    int* ctr = reinterpret_cast<int*>(cta_used + cta_words);
    if (lane == 0) atomicAdd(&ctr[0], 1);
    for (;;) {
      PM_STAT(13);
      __nanosleep(500);
      p = alloc_phys();
      if (p >= 0) break;
      int victim = 0;
      if (lane == 0 &&
          *(volatile int*)&ctr[0] >= *(volatile int*)&ctr[1])
        victim = atomicCAS(&ctr[2], 0, 1) == 0;
      if (__shfl_sync(kFull, victim, 0)) break;
    }
    if (lane == 0) atomicSub(&ctr[0], 1);
    return p;
  }
  // a victim hands its token back once its buckets are released
  __device__ __forceinline__ void release_victim_token() {
    int* ctr = reinterpret_cast<int*>(cta_used + cta_words);
    if (lane == 0) atomicExch(&ctr[2], 0);
  }
  // release: this warp's accesses to the bucket precede the next owner's
  // (the bucket changes hands through the CTA bitmap's atomics)
  __device__ __forceinline__ void free_phys(int p) {
    __syncwarp();
    __threadfence_block();
    if (lane == 0) atomicAnd(&cta_used[p >> 5], ~(1u << (p & 31)));
  }
  __device__ __forceinline__ void release_all() {
    __syncwarp();
    __threadfence_block();
    if (lane < nb) atomicAnd(&cta_used[dp >> 5], ~(1u << (dp & 31)));
    nb = 0;
  }
  __device__ __forceinline__ bool full() const { return nb >= 32; }
  __device__ __forceinline__ int capacity() const { return 32; }
};

struct NWarpState;
struct NCtx {
  long long reserved, allocated, peak_allocated;
  int F, maxF;  // free blocks now / high-water mark
  NWarpState* ws;
};

// Per-trace values read only on the allocation / segment paths live in the
// warp's shared staging area rather than in registers (registers set how
// many warps fit per SM).
struct __align__(16) NWarpState {
  // read together (one 128-bit load) at the top of every request
  u32 amask;      // alignment - 1 (bytes; alignment <= 2^31 in this pass)
  u32 lim;        // largest rounded request in units (0: unit too large)
  u32 span;       // best-fit window in units (0xFFFFFFFF: unbounded)
  u32 split_lim;  // splittable iff size_u <= split_lim
  const pm_cfg_t* cp;
  long long peak_reserved, peak_allocated;
  u32 next_base;  // units
  int nseg, nseg_peak, maxF;  // maxF: free-block high-water mark
  u64 stash_ka, stash_ln;     // a free entry the pool had no room for
  int abase_chunk;            // wire: allocs before the current chunk
};

// Per-warp staging area: two 512 B request buffers (TMA destinations), 512 B
// of gathered records, two mbarriers, the warp state -- a multiple of 16 B
// (the TMA destinations and uint4 records need it).
constexpr size_t kWarpStageBytes =
    (2 * 32 * 16 + 32 * 16 + 16 + sizeof(NWarpState) + 15) / 16 * 16;

// ---- record refs (global store + staged mirror) ---------------------------

__device__ __forceinline__ void set_link(const NRecs& rec, uint4* st, int hcmp,
                                         int lane, u32 g, int right, u32 val) {
  if (lane == 0) *rec.word(g, 2 + right) = val;
  if (hcmp == (int)g) {
    if (right)
      st[lane].w = val;
    else
      st[lane].z = val;
  }
}

__device__ __forceinline__ void relink_lanes(const NRecs& rec, uint4* st,
                                             int hcmp, int lane, bool moved,
                                             u64 links, int dst) {
  const u32 L = lo(links), R = hi(links);
  const u32 val = kFreeTag | (u32)dst;
  if (moved) {
    if (L != kNone) *rec.word(L, 3) = val;
    if (R != kNone) *rec.word(R, 2) = val;
  }
  unsigned m = __ballot_sync(kFull, moved);
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const u32 gl = __shfl_sync(kFull, L, src);
    const u32 gr = __shfl_sync(kFull, R, src);
    const u32 v = __shfl_sync(kFull, val, src);
    if (gl != kNone && hcmp == (int)gl) st[lane].w = v;
    if (gr != kNone && hcmp == (int)gr) st[lane].z = v;
  }
  __syncwarp();
}

// argmin of distinct packed values over the valid lanes (-1 if none)
__device__ __forceinline__ int argmin_pk(bool valid, u64 x) {
  const unsigned any = __ballot_sync(kFull, valid);
  if (!any) return -1;
  if ((any & (any - 1)) == 0) return __ffs(any) - 1;
  PM_STAT(10);
  const u32 mh = __reduce_min_sync(kFull, valid ? hi(x) : 0xffffffffu);
  const bool c = valid && hi(x) == mh;
  const unsigned bm = __ballot_sync(kFull, c);
  if ((bm & (bm - 1)) == 0) return __ffs(bm) - 1;
  PM_STAT(11);
  const u32 ml = __reduce_min_sync(kFull, c ? lo(x) : 0xffffffffu);
  return __ffs(__ballot_sync(kFull, c && lo(x) == ml)) - 1;
}

// ---- bucket maintenance -----------------------------------------------------

// Merge the first adjacent bucket pair whose entries fit in one bucket: the
// right bucket's entries move into the left one's free slots.
template <class D>
__device__ __forceinline__ bool try_merge(const NPool& P, D& dir,
                                          const NRecs& rec, uint4* st,
                                          int hcmp, int lane) {
  const int e = dir.mergeable();
  if (e < 0) return false;
  PM_STAT(7);
  const int pa = dir.phys(e), pb = dir.phys(e + 1);
  const unsigned ma = dir.mask(e), mb = dir.mask(e + 1);
  const bool mv = (mb >> lane) & 1u;
  u64 ka = 0, l = 0;
  int dst = -1;
  if (mv) {
    ka = P.ka[pb * kBucket + lane];
    l = P.ln[pb * kBucket + lane];
    // the r-th moving entry takes the r-th free slot of the left bucket
    const int r = __popc(mb & lanemask_lt());
    dst = pa * kBucket + (int)__fns(~ma, 0, r + 1);
  }
  __syncwarp();
  if (mv) {
    P.ka[dst] = ka;
    P.ln[dst] = l;
  }
  __syncwarp();
  relink_lanes(rec, st, hcmp, lane, mv, l, dst);
  dir.set_mask(e, ma | __reduce_or_sync(kFull, mv ? 1u << (dst - pa * kBucket) : 0u));
  dir.erase(e + 1);
  dir.free_phys(pb);
  return true;
}

// Split the full bucket at position d: the upper half by ka rank moves to a
// new bucket (slots 0..15), the lower half stays in place.  False if no
// bucket can be had and nothing merges (overflow).
template <class D>
__device__ __forceinline__ bool split_bucket(const NPool& P, D& dir, int d,
                                             const NRecs& rec, uint4* st,
                                             int hcmp, int lane) {
  // past the directory's soft size a merge is tried before it grows
  if (!dir.full() && dir.soft_due()) {
    if (try_merge(P, dir, rec, st, hcmp, lane)) return true;  // the caller finds again
    dir.soft_failed();
  }
  int q = dir.full() ? -1 : dir.alloc_phys();
  if (q < 0) {
    if (try_merge(P, dir, rec, st, hcmp, lane)) return true;
    if (dir.full()) return false;
    q = dir.alloc_phys_wait();
    if (q < 0) return false;
  }
  PM_STAT(6);
  const int p = dir.phys(d);
  const int base = p * kBucket;
  const u64 ka = P.ka[base + lane];  // full bucket: every slot holds one
  const u64 l = P.ln[base + lane];
  int rank = 0;
#pragma unroll 8
  for (int j = 0; j < kBucket; ++j)
    rank += __shfl_sync(kFull, ka, j) < ka ? 1 : 0;
  const bool up = rank >= kHalf;
  const int bl = __ffs(__ballot_sync(kFull, rank == kHalf)) - 1;
  const u64 bound = __shfl_sync(kFull, ka, bl);
  const int dst = up ? q * kBucket + rank - kHalf : base + lane;
  __syncwarp();
  if (up) {
    P.ka[dst] = ka;
    P.ln[dst] = l;
  }
  __syncwarp();
  dir.set_mask(d, ~__ballot_sync(kFull, up));
  dir.insert(d + 1, bound, q, 0xFFFFu);
  relink_lanes(rec, st, hcmp, lane, up, l, dst);
  return true;
}

// The pool cannot take an entry (no physical bucket, a full directory): the
// request still completes -- the entry is parked in the warp's state under
// kStashId and the trace is handed to the next pass right after this
// request, its checkpoint carrying the parked entry (save_checkpoint).
constexpr int kStashId = 0x7FFFFFF0;

__device__ __forceinline__ int stash_entry(NCtx& c, u64 ka, u64 links) {
  c.F += 1;
  c.maxF = max(c.maxF, c.F);
  __syncwarp();
  c.ws->stash_ka = ka;  // uniform stores
  c.ws->stash_ln = links;
  __syncwarp();
  return kStashId;
}

// Insert a free block; returns its id (kStashId: parked, see above).
template <class D>
__device__ __forceinline__ int pool_insert(const NPool& P, D& dir, NCtx& c,
                                           u64 ka, u64 links, const NRecs& rec,
                                           uint4* st, int hcmp, int lane) {
  // common case in one test: a directory with a bucket of room for ka
  // (the register directory's find on an empty directory gives -1 with a
  // zero mask, so the empty case folds into the same rare branch)
  int d = 0;
  unsigned m = 0;
  bool rare;
  if constexpr (D::kEmptyFindSafe) {
    d = dir.find(ka);
    m = dir.mask(d);
    rare = dir.nb == 0 || m == kFull;
  } else {
    rare = dir.nb == 0;
    if (!rare) {
      d = dir.find(ka);
      m = dir.mask(d);
      rare = m == kFull;
    }
  }
  if (rare) {
    bool room = true;
    if (dir.nb == 0) {
      const int q = dir.alloc_phys_wait();
      if (q < 0)
        room = false;
      else
        dir.insert(0, 0ull, q, 0u);
    }
    if (room) {
      d = dir.find(ka);
      m = dir.mask(d);
      while (m == kFull) {
        // a full directory whose buckets are >= 3/4 occupied would thrash
        // (merge a pair, split, merge ...) on every insert: hand the trace to
        // the next pass, which has room, instead
        if ((dir.full() && c.F >= 24 * dir.capacity()) ||
            !split_bucket(P, dir, d, rec, st, hcmp, lane)) {
          room = false;
          break;
        }
        d = dir.find(ka);
        m = dir.mask(d);
      }
    }
    if (!room) return stash_entry(c, ka, links);
  }
  const int slot = __ffs(~m) - 1;
  const int id = dir.phys(d) * kBucket + slot;
  PM_STAT(5);
  c.F += 1;
  c.maxF = max(c.maxF, c.F);  // the count grows only here
  __syncwarp();
  P.ka[id] = ka;
  P.ln[id] = links;
  dir.set_bit(d, slot);
  return id;
}

// Remove free block `id`: clear its slot (nothing moves); an emptied bucket
// leaves the directory unless it is the last one.
template <class D>
__device__ __forceinline__ void pool_remove(D& dir, NCtx& c, int id) {
  const int p = id / kBucket;
  const int d = dir.pos_of_phys(p);
  PM_STAT(2);
  dir.clear_bit(d, id % kBucket);
  c.F -= 1;
  if (dir.mask(d) == 0u && dir.nb > 1) {
    PM_STAT(4);
    dir.erase(d);
    dir.free_phys(p);
  }
}

// Rekey entry `id` to (ka, links) -- in place when it stays in its bucket
// -- or, with id < 0, insert a new entry.  Returns the entry's id (-1 on
// overflow); the caller re-points the neighbours whose refs changed.
template <class D>
__device__ __forceinline__ int pool_upsert(const NPool& P, D& dir, NCtx& c,
                                           int id, u64 ka, u64 links,
                                           const NRecs& rec, uint4* st,
                                           int hcmp, int lane) {
  if (id >= 0) {
    const int d = dir.find(ka);
    if (dir.phys(d) == id / kBucket) {
      PM_STAT(0);
      __syncwarp();
      P.ka[id] = ka;
      P.ln[id] = links;
      return id;
    }
    PM_STAT(1);
    pool_remove(dir, c, id);
  }
  return pool_insert(P, dir, c, ka, links, rec, st, hcmp, lane);
}

// Best fit (allocator.py:203-221): argmin ka over entries
// with ru <= size_u and size_u - ru < span (span 0xFFFFFFFF: no bound --
// size_u - ru <= kMaxU - 1 always).  The bucket holding ru and the next
// one are loaded together; the next one's minimum is the only candidate
// when the first holds none.
template <class D>
__device__ __forceinline__ int best_fit(const NPool& P, const D& dir,
                                        u32 ru, u32 span, int lane,
                                        u64& KA, u64& LN) {
  if (dir.nb == 0) return -1;
  const int d = dir.find((u64)ru << 32);
  const int p = dir.phys(d);
  const bool in = (dir.mask(d) >> lane) & 1u;
  const u64 ka = in ? P.ka[p * kBucket + lane] : ~0ull;
  const u64 ln = in ? P.ln[p * kBucket + lane] : 0ull;
  PM_STAT(8);
  const bool el = in && hi(ka) >= ru && hi(ka) - ru < span;
  const int w = argmin_pk(el, ka);
  if (w >= 0) {
    KA = __shfl_sync(kFull, ka, w);
    LN = __shfl_sync(kFull, ln, w);
    return p * kBucket + w;
  }
  // every key of the next bucket is >= (ru, 0): its minimum is the only
  // candidate (loaded only now: most allocations hit the first bucket)
  PM_STAT(9);
  if (d + 1 >= dir.nb) return -1;
  const int p2 = dir.phys(d + 1);
  const bool in2 = (dir.mask(d + 1) >> lane) & 1u;
  const u64 ka2 = in2 ? P.ka[p2 * kBucket + lane] : ~0ull;
  const int w2 = argmin_pk(in2, ka2);
  if (w2 >= 0) {
    const u64 kw = __shfl_sync(kFull, ka2, w2);
    if (hi(kw) - ru < span) {
      KA = kw;
      LN = P.ln[p2 * kBucket + w2];
      return p2 * kBucket + w2;
    }
  }
  return -1;
}

// Wholly-free segment (entry with no allocated neighbour) of largest size_u
// > thr (thr < 0: any), ties lowest addr; -1 if none.
template <class D>
__device__ __forceinline__ int find_release_candidate(const NPool& P,
                                                      const D& dir,
                                                      long long thr, int lane) {
  u64 best = ~0ull;
  int bid = -1;
  for (int d = 0; d < dir.nb; ++d) {
    const int p = dir.phys(d);
    const int id = p * kBucket + lane;
    if (((dir.mask(d) >> lane) & 1u) && P.ln[id] == ~0ull) {
      const u64 ka = P.ka[id];
      if ((long long)hi(ka) > thr) {
        const u64 key = pk(0xFFFFFFFFu - hi(ka), lo(ka));
        if (key < best) {
          best = key;
          bid = id;
        }
      }
    }
  }
  const int w = argmin_pk(bid >= 0, best);
  return w < 0 ? -1 : __shfl_sync(kFull, bid, w);
}

template <class D>
__device__ __forceinline__ void make_room(const NPool& P, D& dir, NCtx& c,
                                          long long seg, NWarpState* ws, int s,
                                          const NRecs& rec, uint4* st,
                                          int hcmp, int lane) {
  const long long capacity = ws->cp->device_capacity;
  const long long t = ws->cp->max_split_size;
  // stage-1 threshold in units: size > t  <=>  size_u > floor(t / u)
  const long long rel_thr = t >= 0 ? (long long)((u64)t >> s) : -1;
  int stage = t >= 0 ? 1 : 2;
  if (stage == 2 && c.reserved + seg <= capacity) return;
  for (;;) {
    if (stage == 1 && c.reserved + seg <= capacity) break;
    const int id = find_release_candidate(P, dir, stage == 1 ? rel_thr : -1,
                                          lane);
    if (id < 0) {
      if (stage == 2 || c.reserved + seg <= capacity) break;
      stage = 2;
      continue;
    }
    const long long sz = (long long)hi(P.ka[id]) << s;
    pool_remove(dir, c, id);
    c.reserved -= sz;
    const int ns = ws->nseg - 1;  // every lane reads before any lane writes
    __syncwarp();
    ws->nseg = ns;  // uniform store
    __syncwarp();
  }
}

#ifdef PM_VALIDATE
// ---- invariant checks (validating build) --------------------------------------
//
// AllocatorState.check_invariants (allocator.py:324-354) over the narrow
// state, after every applied request: every free entry and every live
// record is checked against its neighbours (mutual refs, address
// contiguity, no free-free adjacency), the index ranges, the chain heads /
// tails against the segment count, and the byte sums against reserved /
// allocated.  Returns 0 or a pm_invariant_t code.

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum32(int v) { return __reduce_add_sync(kFull, v); }
__device__ __forceinline__ bool live_u(u32 y) { return y != 0u && y != kFreedU; }

template <class D>
__device__ int validate_narrow(const NPool& P, const D& dir, const NRecs& rec,
                               int wm, const NCtx& c, const NWarpState* ws, int s,
                               int lane) {
  const long long align = ws->cp->alignment;
  const long long cap = ws->cp->device_capacity;
  int bad = 0;
  long long free_u = 0, alloc_u = 0;
  int heads = 0, tails = 0, nfree = 0, free_links = 0, free_refs = 0;
  auto flag = [&](int code) {
    if (!bad) bad = code;
  };
  // neighbour `g` of a free entry `id` at [A, A+S): an allocated handle whose
  // opposite ref names the entry
  auto check_free_nb = [&](u32 g, int id, u32 A, u32 S, bool right) {
    if (g & kFreeTag) {
      flag(PM_INV_ADJACENT_FREE);
      return;
    }
    if ((int)g > wm) {
      flag(PM_INV_LINK);
      return;
    }
    const uint4 r = *rec.rec(g);
    const bool contiguous = right ? A + S == r.x : r.x + r.y == A;
    const u32 back = right ? r.z : r.w;
    if (!live_u(r.y) || !contiguous || back != (kFreeTag | (u32)id)) flag(PM_INV_LINK);
  };
  for (int d = 0; d < dir.nb; ++d) {
    const int p = dir.phys(d);
    const unsigned m = dir.mask(d);
    const u64 lo_b = dir.bound(d);
    const bool last = d + 1 >= dir.nb;
    const u64 hi_b = last ? ~0ull : dir.bound(d + 1);
    if ((m >> lane) & 1u) {
      const int id = p * kBucket + lane;
      const u64 ka = P.ka[id], ln = P.ln[id];
      const u32 S = hi(ka), A = lo(ka), L = lo(ln), R = hi(ln);
      nfree += 1;
      free_u += S;
      if (S == 0) flag(PM_INV_BLOCK_SIZE);
      if ((((long long)S) << s) % align) flag(PM_INV_UNALIGNED);
      if (ka < lo_b || (!last && ka >= hi_b)) flag(PM_INV_POOL);
      if (L == kNone) {
        heads += 1;
      } else {
        free_links += 1;
        check_free_nb(L, id, A, S, false);
      }
      if (R == kNone) {
        tails += 1;
      } else {
        free_links += 1;
        check_free_nb(R, id, A, S, true);
      }
    }
  }
  for (int h = lane; h <= wm; h += 32) {
    const uint4 r = *rec.rec((u32)h);
    if (!live_u(r.y)) continue;
    alloc_u += r.y;
    if ((((long long)r.y) << s) % align) flag(PM_INV_UNALIGNED);
    for (int side = 0; side < 2; ++side) {
      const u32 g = side ? r.w : r.z;
      if (g == kNone) {
        if (side) tails += 1; else heads += 1;
        continue;
      }
      if (g & kFreeTag) {
        // a free neighbour: its entry must name h back and abut it
        free_refs += 1;
        const int id = (int)(g & ~kFreeTag);
        const u64 ka = P.ka[id], ln = P.ln[id];
        const bool ok = side ? (r.x + r.y == lo(ka) && lo(ln) == (u32)h)
                             : (lo(ka) + hi(ka) == r.x && hi(ln) == (u32)h);
        if (!ok) flag(PM_INV_LINK);
        continue;
      }
      if ((int)g > wm) {
        flag(PM_INV_LINK);
        continue;
      }
      const uint4 q = *rec.rec(g);
      const bool ok = side ? (r.x + r.y == q.x && q.z == (u32)h)
                           : (q.x + q.y == r.x && q.w == (u32)h);
      if (!live_u(q.y) || !ok) flag(PM_INV_LINK);
    }
  }
  const unsigned any = __ballot_sync(kFull, bad != 0);
  if (any) return __shfl_sync(kFull, bad, __ffs(any) - 1);
  heads = warp_sum32(heads);
  tails = warp_sum32(tails);
  nfree = warp_sum32(nfree);
  free_links = warp_sum32(free_links);
  free_refs = warp_sum32(free_refs);
  free_u = warp_sum64(free_u);
  alloc_u = warp_sum64(alloc_u);
  if (heads != ws->nseg || tails != ws->nseg) return PM_INV_SEGMENTS;
  if (nfree != c.F || free_links != free_refs) return PM_INV_POOL;
  if ((alloc_u << s) != c.allocated) return PM_INV_ALLOCATED;
  if (((alloc_u + free_u) << s) != c.reserved) return PM_INV_CONSERVATION;
  if (cap >= 0 && c.reserved > cap) return PM_INV_CAPACITY;
  return 0;
}
#endif

// ---- request staging: 1-D TMA bulk copies into a per-warp double buffer ----

__device__ __forceinline__ u32 smem_addr(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one lane: arm the barrier with the byte count and start the copy
__device__ __forceinline__ void bulk_load(void* dst, const void* src, u32 bytes,
                                          u64* bar) {
  // order this warp's earlier generic reads of the buffer before the
  // async-proxy write that refills it
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  u32 ok;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;"
        " selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

// Per-warp staging: two 32-request chunk buffers (TMA destinations), their
// barriers, and the chunk's gathered records.
struct NStage {
  ulonglong2* buf;  // [2][32]
  u64* bar;         // [2]
  uint4* rec;       // [32]
  NWarpState* ws;
  u32 g;            // chunks consumed by this warp (buffer g & 1)
};

__device__ __forceinline__ int ctz64(long long v) {
  return __ffsll(v) - 1;
}

// ---- checkpoints: hand a trace to the next pass mid-way ---------------------
//
// A trace handed off between requests (prepare_request) leaves its complete
// state behind: the scalars, the watermark and, bucket by bucket in
// directory order, its free entries -- the record table already lives in
// HBM.  The next narrow pass rebuilds the same bucket partition in its own
// pool (only the entries' ids change: their allocated neighbours' refs are
// re-pointed) and continues at the next request instead of replaying the
// trace again from request 0.  Space comes from a bump region of the
// workspace; when it is exhausted the trace simply restarts, as before.

struct __align__(16) NCkHeader {
  int r, wm, abase, nb;
  int F, maxF, nseg, nseg_peak;
  long long reserved, allocated, peak_allocated, peak_reserved;
  u32 next_base, pad0, pad1, pad2;
};  // 80 B

struct NCk {
  long long* off;                  // per trace: checkpoint offset or -1
  char* base;                      // bump region
  unsigned long long* used;        // bump counter (Ctl)
  unsigned long long cap;          // region bytes
  bool save, load;                 // this pass writes / resumes checkpoints
};

template <class D>
__device__ __forceinline__ void save_checkpoint(const NCk& ck, int tr, int r, int wm,
                                                int abase, const NCtx& c,
                                                const NWarpState* ws, const NPool& P,
                                                const D& dir, int lane) {
  // the parked entry (counted in c.F) joins the bucket whose key range
  // holds it -- or forms the only group of an empty directory
  const u64 sk = ws->stash_ka, sl = ws->stash_ln;
  const int groups = dir.nb > 0 ? dir.nb : 1;
  const unsigned long long bytes =
      sizeof(NCkHeader) + 16ull * (unsigned long long)groups + 16ull * (unsigned long long)c.F;
  unsigned long long off = 0;
  if (lane == 0) off = atomicAdd(ck.used, (bytes + 15) & ~15ull);
  off = __shfl_sync(kFull, off, 0);
  if (off + bytes > ck.cap) {
    if (lane == 0) ck.off[tr] = -1;  // no room: the next pass restarts it
    return;
  }
  char* b = ck.base + off;
  if (lane == 0) {
    NCkHeader h;
    h.r = r;
    h.wm = wm;
    h.abase = abase;
    h.nb = groups;
    h.F = c.F;
    h.maxF = c.maxF;
    h.nseg = ws->nseg;
    h.nseg_peak = ws->nseg_peak;
    h.reserved = c.reserved;
    h.allocated = c.allocated;
    h.peak_allocated = c.peak_allocated;
    h.peak_reserved = ws->peak_reserved;
    h.next_base = ws->next_base;
    h.pad0 = h.pad1 = h.pad2 = 0;
    *reinterpret_cast<NCkHeader*>(b) = h;
  }
  ulonglong2* desc = reinterpret_cast<ulonglong2*>(b + sizeof(NCkHeader));
  ulonglong2* ent = desc + groups;
  int e = 0;
  if (dir.nb == 0) {
    if (lane == 0) {
      desc[0] = make_ulonglong2(0ull, 1ull);
      ent[0] = make_ulonglong2(sk, sl);
    }
  }
  for (int d = 0; d < dir.nb; ++d) {
    const int p = dir.phys(d);
    const unsigned m = dir.mask(d);
    const u64 bound = dir.bound(d);
    const bool last = d + 1 >= dir.nb;
    const u64 next = last ? ~0ull : dir.bound(d + 1);
    const bool here = sk >= bound && (last || sk < next);
    const int k = __popc(m) + (here ? 1 : 0);
    if (lane == 0) desc[d] = make_ulonglong2(bound, (u64)k);
    if ((m >> lane) & 1u) {
      const int r = __popc(m & lanemask_lt());
      ent[e + r] = make_ulonglong2(P.ka[p * kBucket + lane], P.ln[p * kBucket + lane]);
    }
    if (here && lane == 0) ent[e + k - 1] = make_ulonglong2(sk, sl);
    e += k;
  }
  __threadfence();  // the next pass (a later launch) reads it
  if (lane == 0) ck.off[tr] = (long long)off;
}

// Rebuild the directory from a checkpoint (a fresh pass: empty directory,
// private pool) and re-point the entries' allocated neighbours.  Returns the
// request to continue at.
template <class D>
__device__ __forceinline__ int resume_state(const NCk& ck, int tr, NCtx& c,
                                            NWarpState* ws, const NPool& P, D& dir,
                                            const NRecs& rec, int& wm, int& abase,
                                            int lane) {
  const char* b = ck.base + ck.off[tr];
  const NCkHeader h = *reinterpret_cast<const NCkHeader*>(b);
  const ulonglong2* desc = reinterpret_cast<const ulonglong2*>(b + sizeof(NCkHeader));
  const ulonglong2* ent = desc + h.nb;
  int e = 0, pos = 0;
  auto relink = [&](const ulonglong2& x, int id) {
    const u32 L = lo(x.y), R = hi(x.y);
    const u32 val = kFreeTag | (u32)id;
    if (L != kNone) *rec.word(L, 3) = val;
    if (R != kNone) *rec.word(R, 2) = val;
  };
  for (int d = 0; d < h.nb; ++d) {
    const ulonglong2 dd = desc[d];
    const int k = (int)dd.y;
    const int p = dir.alloc_phys();  // a fresh pass holds >= nb + 1 buckets
    if (k <= kBucket) {
      const int id = p * kBucket + lane;
      if (lane < k) {
        const ulonglong2 x = ent[e + lane];
        P.ka[id] = x.x;
        P.ln[id] = x.y;
        relink(x, id);
      }
      __syncwarp();
      dir.insert(pos++, dd.x, p, k >= 32 ? kFull : ((1u << k) - 1u));
    } else {
      // a full bucket plus the parked entry: 33 keys, split at rank 16
      const ulonglong2 x = ent[e + lane];
      const ulonglong2 xe = ent[e + kBucket];
      int rank = xe.x < x.x ? 1 : 0;
#pragma unroll 8
      for (int i = 0; i < kBucket; ++i) rank += __shfl_sync(kFull, x.x, i) < x.x ? 1 : 0;
      const int rank_e = __popc(__ballot_sync(kFull, x.x < xe.x));
      const int q = dir.alloc_phys();
      const int id = rank < kHalf ? p * kBucket + rank : q * kBucket + rank - kHalf;
      P.ka[id] = x.x;
      P.ln[id] = x.y;
      relink(x, id);
      const int ide = rank_e < kHalf ? p * kBucket + rank_e : q * kBucket + rank_e - kHalf;
      if (lane == 0) {
        P.ka[ide] = xe.x;
        P.ln[ide] = xe.y;
        relink(xe, ide);
      }
      const unsigned at16 = __ballot_sync(kFull, rank == kHalf);
      const u64 bound_q = at16 ? __shfl_sync(kFull, x.x, __ffs(at16) - 1) : xe.x;
      __syncwarp();
      dir.insert(pos++, dd.x, p, 0xFFFFu);
      dir.insert(pos++, bound_q, q, (1u << (kBucket + 1 - kHalf)) - 1u);
    }
    e += k;
  }
  c.reserved = h.reserved;
  c.allocated = h.allocated;
  c.peak_allocated = h.peak_allocated;
  c.F = h.F;
  c.maxF = h.maxF;
  __syncwarp();
  if (lane == 0) {
    ws->peak_reserved = h.peak_reserved;
    ws->next_base = h.next_base;
    ws->nseg = h.nseg;
    ws->nseg_peak = h.nseg_peak;
  }
  __syncwarp();
  wm = h.wm;
  abase = h.abase;
  return h.r;
}

// ---- one trace ---------------------------------------------------------------

template <class D>
__device__ __forceinline__ void replay_trace(
    int tr, const pm_req_t* __restrict__ reqs, const int64_t* __restrict__ offs,
    const pm_cfg_t* __restrict__ cfgs, const int32_t* __restrict__ cfg_of,
    pm_result_t* __restrict__ results, int64_t* __restrict__ timeline,
    u32* rec_base, const NPool& P, D& dir, NStage& sg, int lane,
    const u64* __restrict__ wire, pm_req_t* __restrict__ expand,
    bool expand_overflow, int long_trace, const NCk& ck) {
  const long long e0 = offs[tr];
  const int n = (int)(offs[tr + 1] - e0);  // < 2^31 (pm_replay_batch)
  const pm_cfg_t* cp = cfgs + (cfg_of ? cfg_of[tr] : 0);
  NWarpState* ws = sg.ws;
  int s;
  {
    s = ctz64(cp->alignment);
    s = min(s, ctz64(cp->k_small_buffer));
    s = min(s, ctz64(cp->k_large_buffer));
    s = min(s, ctz64(cp->k_round_large));
    const long long t = cp->max_split_size;
    u32 span, split_lim;
    if (t >= 0) {
      const u64 sp = ((u64)t + ((1ull << s) - 1)) >> s;  // ceil(t / u)
      span = sp > 0xFFFFFFFEull ? 0xFFFFFFFFu : (u32)sp;
      const u64 fl = (u64)t >> s;
      split_lim = fl > 0xFFFFFFFFull ? 0xFFFFFFFFu : (u32)fl;
    } else {
      span = 0xFFFFFFFFu;
      split_lim = 0xFFFFFFFFu;
    }
    __syncwarp();
    if (lane == 0) {
      NWarpState w;
      w.cp = cp;
      w.amask = (u32)(cp->alignment - 1);
      // units above 16 MiB are left to the wide tiers altogether
      w.lim = s > 24 || cp->alignment > (1ll << 31) ? 0u : kMaxU;
      w.span = span;
      w.split_lim = split_lim;
      w.peak_reserved = w.peak_allocated = 0;
      w.next_base = 0;
      w.nseg = w.nseg_peak = w.maxF = 0;
      *ws = w;
    }
    __syncwarp();
  }

  NRecs rec;
  rec.base = reinterpret_cast<uint4*>(rec_base) + e0;
  // this trace's timeline entries (null: no timeline requested)
  longlong2* const tl =
      timeline ? reinterpret_cast<longlong2*>(timeline) + e0 : nullptr;
  // Handle watermark instead of zeroing the record table: records of
  // handles <= wm belong to this run (written by an allocation, or zeroed
  // below); a handle above it has not been touched yet, so its record is
  // "never allocated" without reading memory.  Interned handles appear in
  // first-appearance order (pack_trace, wire words), so the watermark
  // advances without gaps and nothing is zeroed; a gap is zeroed when the
  // watermark jumps over it.  Retry passes start from their own watermark,
  // so records left by an earlier pass are never trusted.
  int wm = -1;
  dir.init(lane);
  __syncwarp();

  NCtx c;
  c.reserved = c.allocated = c.peak_allocated = 0;
  c.F = c.maxF = 0;
  c.ws = ws;
  int status = PM_OK;
  int stop = -1;
  int inv = 0;  // PM_VALIDATE: the violated invariant
  // A trace of >= 2^20 requests replays at one warp's latency (~1 us per
  // request) in every pass, and long traces are the ones that outgrow the
  // earlier passes' capacity and restart: send it straight to the last
  // narrow pass.
  const bool resumed = D::kResumes && ck.load && ck.off[tr] >= 0;
  const bool skip = !resumed && n >= long_trace;

  // requests arrive as pm_req_t (16 B) or as wire words (8 B, decoded in
  // shared memory below)
  // Bulk copies need 16 B-aligned sources and sizes: a chunk of wire words
  // is fetched from the even word at or before it, rounded up to an even
  // count (a word of the neighbouring trace at either end is ignored).
  int abase = 0;  // wire: allocs before this chunk (= the next new handle)
  const int nchunks = skip ? 0 : (n + 31) / 32;
  if (skip) {
    status = PM_POOL_OVERFLOW;
    stop = 0;
  }
  int r0 = 0;  // first request to replay (a checkpoint's resume point)
  if constexpr (D::kResumes) {
    if (resumed) r0 = resume_state(ck, tr, c, ws, P, dir, rec, wm, abase, lane);
  }
  __syncwarp();
  // until a checkpoint is saved, the next pass restarts this trace
  if (ck.save && lane == 0) ck.off[tr] = -1;
  const int k0 = r0 >> 5;
  auto fetch = [&](int k, u32 buf) {
    const int cnt = min(n - 32 * k, 32);
    if (wire) {
      const long long w0 = e0 + 32 * k;
      const long long a0 = w0 & ~1ll;
      const u32 words = (u32)((w0 - a0) + cnt + 1) & ~1u;
      bulk_load(sg.buf + 32 * buf, wire + a0, words * 8, sg.bar + buf);
    } else {
      bulk_load(sg.buf + 32 * buf, reqs + e0 + 32 * k, (u32)cnt * 16,
                sg.bar + buf);
    }
  };
  if (lane == 0 && k0 < nchunks) fetch(k0, sg.g & 1);

  for (int k = k0; k < nchunks; ++k) {
    const int cbase = 32 * k;
    if (wire) {
      __syncwarp();
      ws->abase_chunk = abase;  // uniform store: a checkpoint's resume point
    }
    const u32 b = sg.g & 1;
    mbar_wait(sg.bar + b, (sg.g >> 1) & 1);
    if (lane == 0 && k + 1 < nchunks) {
      // prefetch the next chunk into the other buffer (consumed last chunk)
      fetch(k + 1, b ^ 1);
    }
    ulonglong2* cb = sg.buf + 32 * b;
    const int cnt = min(n - cbase, 32);
    if (wire) {
      // decode the chunk's wire words in place into pm_req_t form
      const int off = (int)((e0 + cbase) & 1);
      const u64 w =
          lane < cnt ? reinterpret_cast<const u64*>(cb)[off + lane] : 0ull;
      __syncwarp();
      const u32 tag = (u32)(w >> 62);
      const unsigned am = __ballot_sync(kFull, lane < cnt && tag == 0);
      if (lane < cnt) {
        ulonglong2 d;
        if (tag == 0) {  // alloc of the next new handle, stream 0
          d.x = w & ((1ull << 62) - 1);
          d.y = (u64)(u32)(abase + __popc(am & lanemask_lt()));
        } else if (tag == 1) {  // free
          d.x = 0;
          d.y = (w & 0x7FFFFFFFull) | ((u64)PM_KIND_FREE << 32);
        } else {  // not produced by pm_wire_pack
          d.x = 0;
          d.y = 0xFFFFFFFFull | ((u64)PM_KIND_UNKNOWN << 32);
        }
        cb[lane] = d;
      }
      abase += __popc(am);
      // these generic writes precede the async-proxy refill of the buffer
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    // Chunk prologue, lane-parallel (lane i = request cbase + i): decode the
    // request once, check everything that does not depend on the replay
    // state (kind, handle range, size, stream, encoding) and round the size,
    // find the latest earlier request of the chunk on the same handle (its
    // staged record is the one this request reads), and gather the handle's
    // record.  The serial loop below then reads one packed 16 B word per
    // request.
    const ulonglong2 evl = lane < cnt ? cb[lane] : make_ulonglong2(0ull, 0ull);
    const int my_h = lane < cnt ? (int)lo(evl.y) : -1;
    const bool hok = my_h >= 0 && my_h < n;
    const bool fresh = hok && my_h > wm;
    {
      const int cmax = __reduce_max_sync(kFull, hok ? my_h : -1);
      if (cmax > wm) {
        // distinct fresh handles in the chunk; fewer than cmax - wm means
        // the watermark jumps over handles this chunk does not touch
        const unsigned same = __match_any_sync(kFull, fresh ? my_h : -1);
        const bool first = fresh && (same & lanemask_lt()) == 0u;
        const int distinct = __popc(__ballot_sync(kFull, first));
        if (distinct < cmax - wm) {
          for (int h = wm + 1 + lane; h <= cmax; h += 32)
            *rec.rec((u32)h) = make_uint4(0, 0, 0, 0);
          __syncwarp();
        }
        wm = cmax;
      }
    }
    uint4 r = make_uint4(0, 0, 0, 0);
    uint4* const myrec = rec.rec((u32)(hok ? my_h : 0));
    if (hok && !fresh) r = *myrec;
#ifdef PM_VALIDATE
    // the validator reads every record <= wm: a fresh handle's record is
    // "never allocated" from the start of its chunk
    if (fresh) *myrec = r;
#endif
    uint4* st = sg.rec;
    st[lane] = r;
    const int hcmp = hok ? my_h : -1;
    {
      const unsigned kind_l = hi(evl.y) & 3u;
      int pre = PM_OK;
      u32 ru_l = 0;
      if (kind_l >= PM_KIND_UNKNOWN) {
        pre = kind_l == PM_KIND_UNKNOWN ? PM_UNKNOWN_KIND : PM_MISSING_FIELD;
      } else if (!hok) {
        pre = PM_BAD_HANDLE;
      } else if (kind_l == PM_KIND_ALLOC) {
        // checked after the duplicate-handle test at replay time
        const long long size = (long long)evl.x;
        const uint4 kc = *reinterpret_cast<const uint4*>(ws);  // amask, lim
        const u64 rounded = (((u64)size + kc.x) & ~(u64)kc.x) >> s;
        if (size <= 0)
          pre = PM_ZERO_SIZE;
        else if ((hi(evl.y) >> 2) != 0u || rounded > (u64)kc.y)
          pre = PM_ENCODING_LIMIT;  // outside the encoding: wide tiers
        else
          ru_l = (u32)rounded;
      }
      const unsigned same = __match_any_sync(kFull, hcmp);
      const unsigned earlier = same & lanemask_lt();
      const int src_l = earlier ? 31 - __clz(earlier) : lane;
      __syncwarp();
      // x ru, y handle, z kind | pre << 2 | src << 8
      if (lane < cnt)
        reinterpret_cast<uint4*>(cb)[lane] = make_uint4(
            ru_l, (u32)my_h, kind_l | ((u32)pre << 2) | ((u32)src_l << 8), 0u);
      // generic writes into a TMA destination precede its async refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();

    const int j0 = k == k0 ? (r0 & 31) : 0;
    uint4 ev_next = reinterpret_cast<const uint4*>(cb)[j0];
    for (int j = j0; j < cnt; ++j) {
      // the next request's word is loaded before this one's dependent chain
      // (clamped to the chunk's own buffer: slot 32 would be the other
      // buffer, which the prefetch's bulk copy may be writing)
      const uint4 ev = ev_next;
      ev_next = reinterpret_cast<const uint4*>(cb)[min(j + 1, 31)];
      bool handoff = false;  // an entry was parked: hand off after this request
      const int hj = (int)ev.y;
      const unsigned kind = ev.z & 3u;
      const int pre = (int)((ev.z >> 2) & 63u);
      const int src = (int)(ev.z >> 8);
      int sts = PM_OK;
      if (kind >= PM_KIND_UNKNOWN || pre == PM_BAD_HANDLE) {
        sts = pre;
      } else {
        const uint4 rj = st[src];
        // the allocation constants, loaded alongside the record
        const uint4 kc = *reinterpret_cast<const uint4*>(ws);
        const u32 k_span = kc.z, k_split = kc.w;
        int rm_id = -1;
        bool up = false;
        int up_id = -1;
        u64 up_ka = 0, up_l = 0;
        u32 f1 = kNone, f2 = kNone;
        int both_pid = -1;
        u32 both_S = 0, both_rS = 0, both_rR = kNone;
        // neighbour refs that must name the upserted entry even when it
        // keeps its id (the other side is re-pointed only if it moved)
        bool newL = false, newR = false;
        const bool is_alloc = kind == PM_KIND_ALLOC;
        bool split_out = false;
        u32 out_a = 0, out_s = 0, out_L = kNone, out_R = kNone;
        if (is_alloc) {
          // one test for the rare errors: a duplicate handle first, then the
          // prologue's zero size / encoding limit
          if (rj.y != 0 || pre != PM_OK) {
            sts = rj.y != 0 ? PM_DUPLICATE_HANDLE : pre;
          } else {
            const u32 ru = ev.x;
            const u32 split_lim = k_split;
            u64 KA = 0, Lk = 0;
            const int id = best_fit(P, dir, ru, k_span, lane, KA, Lk);
            if (id >= 0) {
              // hit: _take (allocator.py:234-242), _split (:223-232)
              const u32 Lf = lo(Lk), Rf = hi(Lk);
              const u32 S = hi(KA), A = lo(KA);
              out_a = A;
              out_L = Lf;
              f1 = Lf;
              if (S <= split_lim && S > ru) {
                up = true;
                up_id = id;
                up_ka = pk(S - ru, A + ru);
                up_l = pmb::mk_links(kNone, Rf);  // left (hj) set below
                out_s = ru;
                split_out = true;
              } else {
                rm_id = id;
                out_s = S;
                out_R = Rf;
                f2 = Rf;
              }
            } else {
              // miss: new segment (allocator.py:278-288, 244-250)
              PM_STAT(14);
              pmb::Cfg wc;
              wc.cp = ws->cp;
              const long long seg =
                  pmb::segment_size_for((long long)ru << s, wc);
              const long long capacity = wc.cp->device_capacity;
              if (capacity >= 0 && c.reserved + seg > capacity) {
                make_room(P, dir, c, seg, ws, s, rec, st, hcmp, lane);
                if (c.reserved + seg > capacity) sts = PM_OOM;
              }
              const u64 seg_u = (u64)seg >> s;
              const u32 A = ws->next_base;
              if (sts == PM_OK && (u64)A + seg_u > kMaxU)
                sts = PM_ENCODING_LIMIT;
              if (sts == PM_OK) {
                c.reserved += seg;
                {
                  const int ns = ws->nseg + 1;
                  const int np = max(ws->nseg_peak, ns);
                  const long long pr = max(ws->peak_reserved, c.reserved);
                  __syncwarp();
                  ws->next_base = A + (u32)seg_u;  // uniform stores
                  ws->nseg = ns;
                  ws->nseg_peak = np;
                  ws->peak_reserved = pr;  // reserved grows only here
                  __syncwarp();
                }
                out_a = A;
                if ((u32)seg_u <= split_lim && (u32)seg_u > ru) {
                  up = true;
                  up_ka = pk((u32)seg_u - ru, A + ru);
                  up_l = pmb::mk_links(kNone, kNone);
                  out_s = ru;
                  split_out = true;
                } else {
                  out_s = (u32)seg_u;
                }
              }
            }
          }
        } else {
          // free (allocator.py:294-320): double free before unknown handle
          if (rj.y - 1u >= kFreedU - 1u) {  // rj.y == 0 or rj.y == kFreedU
            sts = rj.y == 0 ? PM_UNKNOWN_HANDLE : PM_DOUBLE_FREE;
          } else {
            const u32 A = rj.x, S = rj.y, L = rj.z, R = rj.w;
            c.allocated -= (long long)S << s;
            const bool lf = is_free_ref(L), rf = is_free_ref(R);
            up = true;
            if (!lf && !rf) {
              PM_STAT(15);
              up_ka = pk(S, A);
              up_l = pmb::mk_links(L, R);
            } else if (lf && !rf) {
              const int pid = (int)(L & ~kFreeTag);
              up_id = pid;
              up_ka = P.ka[pid] + ((u64)S << 32);
              up_l = pmb::mk_links(lo(P.ln[pid]), R);
              newR = true;
            } else if (!lf && rf) {
              const int rid = (int)(R & ~kFreeTag);
              up_id = rid;
              up_ka = pk(hi(P.ka[rid]) + S, A);
              up_l = pmb::mk_links(L, hi(P.ln[rid]));
              newL = true;
            } else {
              const int rid = (int)(R & ~kFreeTag);
              both_pid = (int)(L & ~kFreeTag);
              both_rS = hi(P.ka[rid]);
              both_rR = hi(P.ln[rid]);
              both_S = S;
              rm_id = rid;
            }
          }
        }
        if (sts == PM_OK) {
          if (rm_id >= 0) {
            pool_remove(dir, c, rm_id);
            if (both_pid >= 0) {
              up_id = both_pid;
              up_ka = P.ka[both_pid] + ((u64)(both_S + both_rS) << 32);
              up_l = pmb::mk_links(lo(P.ln[both_pid]), both_rR);
              newR = true;
            }
          }
          if (up) {
            // a split remainder's left neighbour is hj itself: its record
            // is written whole below, so only the stored entry names it
            const u64 links = split_out ? (up_l & 0xFFFFFFFF00000000ull) | (u64)(u32)hj
                                        : up_l;
            const int nid = pool_upsert(P, dir, c, up_id, up_ka, links, rec, st,
                                        hcmp, lane);
            if (nid < 0) {
              sts = PM_POOL_OVERFLOW;
            } else {
              const bool moved = nid != up_id;
              const u32 L = lo(up_l), R = hi(up_l);
              if ((newL || moved) && L != kNone)
                set_link(rec, st, hcmp, lane, L, 1, kFreeTag | (u32)nid);
              if ((newR || moved) && R != kNone)
                set_link(rec, st, hcmp, lane, R, 0, kFreeTag | (u32)nid);
              if (split_out) out_R = kFreeTag | (u32)nid;
              handoff = nid == kStashId;
            }
          }
        }
        if (sts == PM_OK) {
          if (f2 != kNone) set_link(rec, st, hcmp, lane, f2, 0, (u32)hj);
          if (f1 != kNone) set_link(rec, st, hcmp, lane, f1, 1, (u32)hj);
          __syncwarp();
          if (is_alloc) {
            c.allocated += (long long)out_s << s;
            c.peak_allocated = max(c.peak_allocated, c.allocated);
            if (lane == j) {
              const uint4 o = make_uint4(out_a, out_s, out_L, out_R);
              st[j] = o;
              *myrec = o;
            }
          } else if (lane == j) {
            st[j].y = kFreedU;
            reinterpret_cast<u32*>(myrec)[1] = kFreedU;
          }
        }
      }
#ifdef PM_VALIDATE
      if (sts == PM_OK && pmb::g_inject[1] != 0 && cbase + j == pmb::g_inject[0]) {
        // fault injection for the validator's own tests (pm_validate_inject)
        if (pmb::g_inject[1] == 1) c.allocated += 1ll << s;
        if (pmb::g_inject[1] == 2 && lane == 0 && hj >= 0)
          *rec.word((u32)hj, 2) = (u32)hj;  // a ref that is not mutual
      }
      if (sts == PM_OK && !handoff) {
        __syncwarp();
        const int code = validate_narrow(P, dir, rec, wm, c, ws, s, lane);
        if (code) {
          sts = PM_INVARIANT_VIOLATION;
          inv = code;
        }
      }
#endif
      // one test on the common path: an error stops before the request, a
      // hand-off after it (its timeline entry is written first)
      if (sts != PM_OK || handoff) {
        if (sts != PM_OK) {
          status = sts;
          stop = cbase + j;
          break;
        }
        if (tl != nullptr && lane == j)
          tl[cbase + j] = make_longlong2(c.reserved, c.allocated);
        __syncwarp();
        // the request is complete; continue at the next one in the next pass
        status = PM_POOL_OVERFLOW;
        stop = cbase + j + 1;
        if (ck.save) {
          // records of this chunk's handles not seen yet are not state yet:
          // make them "never allocated" for the next pass
          const unsigned done_l = j == 31 ? kFull : (2u << j) - 1u;
          const unsigned same = __match_any_sync(kFull, hcmp);
          if (fresh && (done_l >> lane & 1u) == 0u && (same & done_l) == 0u)
            *myrec = make_uint4(0, 0, 0, 0);
        }
        break;  // the checkpoint is written after the chunk loop
      }
      if (tl != nullptr && lane == j)
        tl[cbase + j] = make_longlong2(c.reserved, c.allocated);
      __syncwarp();
    }
    __syncwarp();
    sg.g += 1;
    if (status != PM_OK) {
      if (k + 1 < nchunks) {
        // drain the prefetch in flight so the buffer's phase stays in step
        mbar_wait(sg.bar + (sg.g & 1), (sg.g >> 1) & 1);
        sg.g += 1;
      }
      break;
    }
  }

  if (status == PM_POOL_OVERFLOW && stop > 0 && ck.save) {
    // handed off after request stop - 1 (a parked entry): leave the state
    __syncwarp();
    save_checkpoint(ck, tr, stop, wm, ws->abase_chunk, c, ws, P, dir, lane);
  }
  if (wire != nullptr &&
      (status == PM_ENCODING_LIMIT ||
       (status == PM_POOL_OVERFLOW && expand_overflow))) {
    // the wide tiers read pm_req_t: expand this trace's words for them
    int ab = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const u64 w = i < n ? __ldg(wire + e0 + i) : 0ull;
      const u32 tag = (u32)(w >> 62);
      const unsigned am = __ballot_sync(kFull, i < n && tag == 0);
      if (i < n) {
        pm_req_t d;
        if (tag == 0) {
          d.size = (int64_t)(w & ((1ull << 62) - 1));
          d.handle = ab + __popc(am & lanemask_lt());
          d.kind_stream = PM_KIND_ALLOC;
        } else if (tag == 1) {
          d.size = 0;
          d.handle = (int32_t)(w & 0x7FFFFFFFull);
          d.kind_stream = PM_KIND_FREE;
        } else {
          d.size = 0;
          d.handle = -1;
          d.kind_stream = PM_KIND_UNKNOWN;
        }
        expand[e0 + i] = d;
      }
      ab += __popc(am);
    }
  }

  dir.release_all();
  if (lane == 0) {
    pm_result_t res;
    res.peak_reserved = ws->peak_reserved;
    res.peak_allocated = c.peak_allocated;
    res.final_reserved = c.reserved;
    res.final_allocated = c.allocated;
    res.stop_index = stop;
    res.n_events_replayed =
        status == PM_OK ? n : (status == PM_OOM ? stop + 1 : stop);
    res.status = status;
    res.n_segments_final = ws->nseg;
    res.n_segments_peak = ws->nseg_peak;
    res.max_free_blocks = status == PM_INVARIANT_VIOLATION ? inv : c.maxF;
    results[tr] = res;
  }
}

__device__ __forceinline__ NStage carve_stage(char* wst) {
  NStage sg;
  sg.buf = reinterpret_cast<ulonglong2*>(wst);
  sg.rec = reinterpret_cast<uint4*>(wst + 2 * 32 * 16);
  sg.bar = reinterpret_cast<u64*>(wst + 3 * 32 * 16);
  sg.ws = reinterpret_cast<NWarpState*>(wst + 3 * 32 * 16 + 16);
  sg.g = 0;
  return sg;
}

// ---- escalation routing ------------------------------------------------------
//
// Passes of one pm_replay_batch, in launch order (Ctl work / n_list index):
//   0 main narrow pass (register directory, CTA-shared pool)
//   1 narrow, memory directory, entries in shared memory, several warps
//     per SM with a private pool each                        (kTierMemSmem)
//   2 the same with one warp owning the SM's shared memory   (kTierMemSmemBig)
//   3 narrow, memory directory, entries in HBM              (kTierMemHbm)
//   4..7 the wide tiers 1-4 of replay_device.cuh            (kTierWide1..)
// Between narrow passes a trace moves with its checkpoint (NCk) and
// continues where it stopped.
// A capacity overflow moves a trace to the next capacity tier; an encoding
// limit sends it to the first wide tier.
// requests: with PM_LONG_SKIP=1 a trace this long goes straight to pass 2
// when the batch is too small to fill the main pass anyway (the host passes
// kNoSkip otherwise, the default)
constexpr int kLongTrace = 1 << 20;
constexpr int kNoSkip = 0x7FFFFFFF;
constexpr int kTierMemSmem = 1;
constexpr int kTierMemSmemBig = 2;
constexpr int kTierMemHbm = 3;
constexpr int kTierWide1 = 4;
constexpr int kTierWide4 = 7;

__device__ __forceinline__ void route(pmb::Ctl* ctl, int sts, int tr,
                                      int next_pass,
                                      int32_t* __restrict__ overflow_list,
                                      int32_t* __restrict__ enc_list) {
  if (sts == PM_POOL_OVERFLOW) {
    overflow_list[atomicAdd(&ctl->n_list[next_pass], 1u)] = tr;
  } else if (sts == PM_ENCODING_LIMIT) {
    enc_list[atomicAdd(&ctl->n_list[kTierWide1], 1u)] = tr;
  }
}

// Directory in shared memory (one warp per CTA, any number of buckets up
// to nbmax): bounds and physical ids by position, occupancy masks and
// positions by physical bucket, a stack of free physical buckets.  Same
// interface as NDir; find is a 32-ary warp search over the sorted bounds.
struct NDirMem {
  static constexpr bool kResumes = true;  // passes 1-3 continue checkpoints
  static constexpr bool kEmptyFindSafe = false;  // positions index memory
  // soft size: past it a full bucket first tries to merge a pair elsewhere
  // instead of growing the directory, whose inserts / erases shift O(nb)
  // positions and whose find takes one more round beyond 2048 (C5's trace:
  // 4.02 -> 3.7 s); the directory still grows to nbmax when nothing merges
  // (after a failed attempt the next one waits for 64 more positions, so a
  // dense directory is not rescanned on every split)
  static constexpr int kSoftBuckets = 2048;
  int soft_at;
  __device__ __forceinline__ bool soft_due() const { return nb >= soft_at; }
  __device__ __forceinline__ void soft_failed() { soft_at = nb + 64; }
  u64* db;          // [nbmax] bound by position
  int* dp;          // [nbmax] physical bucket by position
  unsigned* m;      // [nbmax] occupancy mask by position
  int* pos;         // [nbmax] position by physical bucket
  int* pstack;      // [nbmax] free physical buckets
  int nb, ptop, nbmax, lane;
  // register summary: lane L holds the bounds at positions 32 L and
  // 32 (L + 32)
  u64 sb, sb2;

  __device__ __forceinline__ void refresh() {
    sb = 32 * lane < nb ? db[32 * lane] : ~0ull;
    sb2 = 32 * (lane + 32) < nb ? db[32 * (lane + 32)] : ~0ull;
  }
  __device__ __forceinline__ void init(int lane_) {
    lane = lane_;
    nb = 0;
    soft_at = kSoftBuckets;
    sb = sb2 = ~0ull;
    __syncwarp();
    for (int i = lane; i < nbmax; i += 32) pstack[i] = nbmax - 1 - i;
    __syncwarp();
    ptop = nbmax;
  }
  // last position whose bound <= x.  Up to 2048 positions: the summary
  // picks the block of 32, one probe of it the position; beyond, each round
  // probes 32 evenly spaced positions of the live range, shrinking it 32x
  __device__ __forceinline__ int find(u64 x) const {
    if (nb <= 2048) {
      const unsigned hi_b = __ballot_sync(kFull, sb2 <= x);
      const int blk = hi_b ? 63 - __clz(hi_b)
                           : 31 - __clz(__ballot_sync(kFull, sb <= x));
      const int e = 32 * blk + lane;
      const unsigned b = __ballot_sync(kFull, e < nb && db[e] <= x);
      return 32 * blk + 31 - __clz(b);
    }
    int lo_ = 0, hi_ = nb;
    while (hi_ - lo_ > 32) {
      const int step = (hi_ - lo_ + 31) / 32;
      const int e = lo_ + lane * step;
      const unsigned b = __ballot_sync(kFull, e < hi_ && db[e] <= x);
      lo_ += (31 - __clz(b)) * step;  // lane 0 probes lo_: always true
      hi_ = min(lo_ + step, hi_);
    }
    const int e = lo_ + lane;
    const unsigned b = __ballot_sync(kFull, e < hi_ && db[e] <= x);
    return b ? lo_ + 31 - __clz(b) : lo_;
  }
  __device__ __forceinline__ int phys(int d) const { return dp[d]; }
  __device__ __forceinline__ unsigned mask(int d) const { return m[d]; }
  __device__ __forceinline__ u64 bound(int d) const { return db[d]; }
  __device__ __forceinline__ void set_mask(int d, unsigned v) {
    __syncwarp();
    m[d] = v;  // uniform store
    __syncwarp();
  }
  __device__ __forceinline__ void set_bit(int d, int b) {
    set_mask(d, mask(d) | (1u << b));
  }
  __device__ __forceinline__ void clear_bit(int d, int b) {
    set_mask(d, mask(d) & ~(1u << b));
  }
  __device__ __forceinline__ int pos_of_phys(int p) const { return pos[p]; }
  __device__ __forceinline__ int mergeable() const {
    for (int base = 0; base < nb - 1; base += 32) {
      const int x = base + lane;
      bool ok = false;
      if (x < nb - 1) ok = __popc(m[x]) + __popc(m[x + 1]) <= kBucket;
      const unsigned b = __ballot_sync(kFull, ok);
      if (b) return base + __ffs(b) - 1;
    }
    return -1;
  }
  __device__ __forceinline__ void insert(int d, u64 b, int p, unsigned mk) {
    // shift positions d.. up by one, 32 at a time from the top
    for (int base = ((nb - 1 - d) / 32) * 32; base >= 0; base -= 32) {
      const int e = d + base + lane;
      const bool mv = e < nb;
      u64 xb = 0;
      int xp = 0;
      unsigned xm = 0;
      if (mv) {
        xb = db[e];
        xp = dp[e];
        xm = m[e];
      }
      __syncwarp();
      if (mv) {
        db[e + 1] = xb;
        dp[e + 1] = xp;
        m[e + 1] = xm;
        pos[xp] = e + 1;
      }
      __syncwarp();
    }
    db[d] = b;
    dp[d] = p;
    m[d] = mk;
    pos[p] = d;
    __syncwarp();
    nb += 1;
    refresh();
  }
  __device__ __forceinline__ void erase(int d) {
    for (int base = 0; d + 1 + base < nb; base += 32) {
      const int e = d + 1 + base + lane;
      const bool mv = e < nb;
      u64 xb = 0;
      int xp = 0;
      unsigned xm = 0;
      if (mv) {
        xb = db[e];
        xp = dp[e];
        xm = m[e];
      }
      __syncwarp();
      if (mv) {
        db[e - 1] = xb;
        dp[e - 1] = xp;
        m[e - 1] = xm;
        pos[xp] = e - 1;
      }
      __syncwarp();
    }
    nb -= 1;
    if (d == 0) db[0] = 0;  // uniform store
    __syncwarp();
    refresh();
  }
  __device__ __forceinline__ int alloc_phys() {
    if (ptop == 0) return -1;
    ptop -= 1;
    return pstack[ptop];
  }
  __device__ __forceinline__ int alloc_phys_wait() { return alloc_phys(); }
  __device__ __forceinline__ void free_phys(int p) {
    __syncwarp();
    pstack[ptop] = p;  // uniform store
    __syncwarp();
    ptop += 1;
  }
  __device__ __forceinline__ void release_all() {
    nb = 0;
    soft_at = kSoftBuckets;
    sb = sb2 = ~0ull;
  }
  __device__ __forceinline__ void release_victim_token() {}
  __device__ __forceinline__ bool full() const { return nb >= nbmax; }
  __device__ __forceinline__ int capacity() const { return nbmax; }
};

// Shared memory of a memory-directory tier CTA (one warp): staging, the
// directory arrays (24 B per bucket) and, when SMEM_POOL, the entries
// (512 B per bucket).
__host__ __device__ __forceinline__ size_t mem_dir_bytes(int nbmax) {
  return (size_t)nbmax * 24;
}
__host__ __device__ __forceinline__ size_t mem_tier_smem(int nbmax, bool smem_pool) {
  return kWarpStageBytes + mem_dir_bytes(nbmax) +
         (smem_pool ? (size_t)nbmax * kBucket * 16 : 0);
}
__host__ __device__ __forceinline__ size_t mem_tier_pool_bytes(int nbmax) {
  return ((size_t)nbmax * kBucket * 16 + 255) / 256 * 256;
}

// Shared memory per CTA: the pool (B x 32 x 16 B), per warp a staging area
// (two 512 B request buffers, 512 B of gathered records, two barriers),
// and the pool's in-use bitmap.

__host__ __device__ __forceinline__ size_t smem_cta_bytes(int buckets,
                                                          int warps) {
  return (size_t)buckets * kBucket * 16 + (size_t)warps * kWarpStageBytes +
         (size_t)((buckets + 31) / 32) * 4 + 12;
}

// First-wave split of a packed one-wave batch (see replay_narrow_kernel):
// traces longer than a quarter of the longest are "long"; when they fill
// fewer CTAs than the grid, ctl->pos_ctas = the CTAs they fill (else 0, the
// counter).  One block; the batch is at most one wave (a few thousand).
__global__ void __launch_bounds__(1024)
    pos_prep_kernel(const int64_t* __restrict__ offs,
                    const int32_t* __restrict__ list, int n_traces, int per_cta,
                    int grid, pmb::Ctl* ctl) {
  __shared__ long long s_max;
  __shared__ int s_long;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_long = 0;
  }
  __syncthreads();
  long long mx = 0;
  for (int i = threadIdx.x; i < n_traces; i += blockDim.x) {
    const int tr = list ? list[i] : i;
    mx = max(mx, (long long)(offs[tr + 1] - offs[tr]));
  }
  atomicMax(&s_max, mx);
  __syncthreads();
  const long long thr = s_max / 4;
  int cnt = 0;
  for (int i = threadIdx.x; i < n_traces; i += blockDim.x) {
    const int tr = list ? list[i] : i;
    cnt += (offs[tr + 1] - offs[tr]) > thr;
  }
  atomicAdd(&s_long, cnt);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int g_long = (s_long + per_cta - 1) / per_cta;
    ctl->pos_ctas = g_long < grid ? g_long : 0;
  }
}

// Main pass: persistent warps pull traces (longest first) from a global
// counter; the CTA's warps share one shared-memory bucket pool.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    replay_narrow_kernel(const pm_req_t* __restrict__ reqs,
                         const int64_t* __restrict__ offs,
                         const pm_cfg_t* __restrict__ cfgs,
                         const int32_t* __restrict__ cfg_of,
                         pm_result_t* __restrict__ results,
                         int64_t* __restrict__ timeline, u32* recs,
                         pmb::Ctl* ctl, const int32_t* __restrict__ list,
                         int n_traces, int32_t* __restrict__ overflow_list,
                         int buckets, const unsigned* __restrict__ group_end,
                         int n_groups, const volatile unsigned* ready,
                         const u64* __restrict__ wire,
                         pm_req_t* __restrict__ expand,
                         int32_t* __restrict__ enc_list, int long_trace,
                         long long* __restrict__ ck_off, char* __restrict__ ck_base,
                         unsigned long long ck_cap) {
  extern __shared__ __align__(16) char smem[];
  // every CTA of this grid is resident: the pass-1 grid launched behind it
  // (a programmatic dependent launch) may start on the SMs it leaves free
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  NCk ck;
  ck.off = ck_off;
  ck.base = ck_base;
  ck.used = &ctl->ck_used;
  ck.cap = ck_cap;
  ck.save = ck_off != nullptr;
  ck.load = false;
  const size_t E = (size_t)buckets * kBucket;
  NPool P;
  P.ka = reinterpret_cast<u64*>(smem);
  P.ln = P.ka + E;
  NStage sg = carve_stage(smem + E * 16 + (size_t)wib * kWarpStageBytes);
  unsigned* used = reinterpret_cast<unsigned*>(smem + E * 16 +
                                               (size_t)WARPS * kWarpStageBytes);
  const int words = (buckets + 31) / 32;
  for (int i = threadIdx.x; i < words + 3; i += blockDim.x) used[i] = 0u;
  int* active = reinterpret_cast<int*>(used + words) + 1;
  if (lane == 0) {
    mbar_init(sg.bar);
    mbar_init(sg.bar + 1);
    mbar_fence_init();
  }
  __syncthreads();
  NDir dir;
  dir.cta_used = used;
  dir.cta_words = words;
  dir.cta_buckets = buckets;
  // First wave by position.  Batches under a wave (the narrow widths, 1-20
  // warps per CTA: a small sweep, a rank's shard at 4-8 GPUs) start
  // warp-major: SM c's warps take positions c, c + grid, c + 2 grid, ... of
  // the longest-first order, so every SM holds one trace of each length
  // class and no SM's warps are all long ones (the atomic counter hands the
  // longest traces to whichever CTAs start first, often the same SMs):
  // 1250 C3 traces 111.6 -> 97.7 ms.  A packed batch of one wave with a
  // short tail (C4: 2898 C3-length replays, 552 GPT-2-length ones) gets
  // ctl->pos_ctas = the CTAs its long traces fill (pos_prep_kernel): those
  // CTAs take the long positions warp-major, the remaining CTAs the short
  // tail CTA by CTA, so whole SMs free up early for the pass-1 grid beside
  // (the counter left that to launch timing: C4 126 or 157 ms).  Positions
  // [0, grid x WARPS) are each taken once; the counter continues after them.
  constexpr bool kByPosition = WARPS < 24;
  const unsigned wave = gridDim.x * WARPS;
  const unsigned pc = kByPosition ? gridDim.x : (unsigned)ctl->pos_ctas;
  bool first = pc > 0;
  for (;;) {
    unsigned t = 0;
    if (first) {
      const unsigned c = blockIdx.x;
      t = c < pc ? (unsigned)wib * pc + c : pc * WARPS + (c - pc) * WARPS + wib;
      first = false;
    } else {
      if (lane == 0) t = (pc > 0 ? wave : 0u) + atomicAdd(&ctl->work[0], 1u);
      t = __shfl_sync(kFull, t, 0);
    }
    if (t >= (unsigned)n_traces) break;
    if (ready != nullptr) {
      if (lane == 0) {
        int g = 0;
        while (g + 1 < n_groups && t >= group_end[g]) ++g;
        while (ready[g] == 0u) __nanosleep(2000);
      }
      __syncwarp();
    }
    const int tr = list ? list[t] : (int)t;
    if (lane == 0) atomicAdd(active, 1);
    replay_trace(tr, reqs, offs, cfgs, cfg_of, results, timeline, recs, P, dir,
                 sg, lane, wire, expand, false, long_trace, ck);
    __syncwarp();
    if (lane == 0) atomicSub(active, 1);
    const int sts = results[tr].status;
    if (sts == PM_POOL_OVERFLOW) dir.release_victim_token();
    if (lane == 0) {
      __threadfence();  // the trace's records / checkpoint before its list entry
      route(ctl, sts, tr, kTierMemSmem, overflow_list, enc_list);
    }
  }
  // a pass-1 grid running beside the main pass learns here that no more
  // traces will be handed over (every list entry precedes the flag)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->main_exited, 1u) + 1u == gridDim.x) atomicExch(&ctl->main_done, 1u);
  }
}

// Memory-directory tiers (passes 1 and 2): one warp per CTA replays the
// traces whose free blocks outgrew the main pass's register directory or
// CTA pool, with the directory in shared memory and the entries in shared
// memory (SMEM_POOL) or in a per-CTA HBM region.
template <bool SMEM_POOL>
__global__ void __launch_bounds__(256, 1)
    replay_narrow_mem_kernel(const pm_req_t* __restrict__ reqs,
                             const int64_t* __restrict__ offs,
                             const pm_cfg_t* __restrict__ cfgs,
                             const int32_t* __restrict__ cfg_of,
                             pm_result_t* __restrict__ results,
                             int64_t* __restrict__ timeline, u32* recs,
                             pmb::Ctl* ctl, int pass,
                             const int32_t* __restrict__ list,
                             int32_t* __restrict__ overflow_list,
                             int32_t* __restrict__ enc_list,
                             char* __restrict__ gpool, int nbmax,
                             const u64* __restrict__ wire,
                             pm_req_t* __restrict__ expand, int long_trace,
                             long long* __restrict__ ck_off, char* __restrict__ ck_base,
                             unsigned long long ck_cap, size_t warp_bytes,
                             int beside_main) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  // each warp of the CTA owns a slice of the shared memory (its staging,
  // directory and, in the shared-memory passes, its bucket pool)
  char* wsm = smem + (size_t)(threadIdx.x >> 5) * warp_bytes;
  NStage sg = carve_stage(wsm);
  NCk ck;
  ck.off = ck_off;
  ck.base = ck_base;
  ck.used = &ctl->ck_used;
  ck.cap = ck_cap;
  // pass 1 checkpoints for pass 2; pass 2 hands off to the wide tiers,
  // which replay from the start in their own representation
  ck.save = SMEM_POOL && ck_off != nullptr;
  ck.load = ck_off != nullptr;
  char* dbase = wsm + kWarpStageBytes;
  NDirMem dir;
  dir.nbmax = nbmax;
  dir.db = reinterpret_cast<u64*>(dbase);
  dir.dp = reinterpret_cast<int*>(dir.db + nbmax);
  dir.m = reinterpret_cast<unsigned*>(dir.dp + nbmax);
  dir.pos = reinterpret_cast<int*>(dir.m + nbmax);
  dir.pstack = dir.pos + nbmax;
  NPool P;
  char* pbase = SMEM_POOL ? dbase + mem_dir_bytes(nbmax)
                          : gpool + (size_t)blockIdx.x * mem_tier_pool_bytes(nbmax);
  P.ka = reinterpret_cast<u64*>(pbase);
  P.ln = P.ka + (size_t)nbmax * kBucket;
  if (lane == 0) {
    mbar_init(sg.bar);
    mbar_init(sg.bar + 1);
    mbar_fence_init();
  }
  __syncwarp();
  const unsigned n = beside_main ? 0u : ctl->n_list[pass];
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&ctl->work[pass], 1u);
    t = __shfl_sync(kFull, t, 0);
    int tr;
    if (!beside_main) {
      if (t >= n) break;
      tr = list[t];
    } else {
      // running beside the main pass (batches of one wave): wait until the
      // main pass has handed over entry t -- or has finished without it
      // (list slots start at -1; an entry is published after its data)
      tr = -1;
      if (lane == 0) {
        for (;;) {
          const unsigned cnt = *(volatile unsigned*)&ctl->n_list[pass];
          if (t < cnt) {
            const int v = *(volatile const int*)&list[t];
            if (v >= 0) {
              tr = v;
              break;
            }
          } else if (*(volatile unsigned*)&ctl->main_done) {
            if (t >= *(volatile unsigned*)&ctl->n_list[pass]) {
              tr = -2;
              break;
            }
            continue;
          }
          __nanosleep(4000);
        }
        __threadfence();  // acquire: the entry's records / checkpoint
      }
      tr = __shfl_sync(kFull, tr, 0);
      __syncwarp();
      if (tr == -2) break;
    }
    // the last narrow tier expands wire words for the wide tier it hands to
    replay_trace(tr, reqs, offs, cfgs, cfg_of, results, timeline, recs, P, dir,
                 sg, lane, wire, expand, !SMEM_POOL,
                 SMEM_POOL ? long_trace : kNoSkip, ck);
    __syncwarp();
    if (lane == 0)
      route(ctl, results[tr].status, tr,
            !SMEM_POOL ? kTierWide4 : pass == kTierMemSmem ? kTierMemSmemBig : kTierMemHbm,
            overflow_list, enc_list);
  }
}

}  // namespace pmn
