// Device side of the batched caching-allocator replay (sm_100a).
//
// Restates the state machine of peakmem.allocator.AllocatorState
// (reference pkg/src/peakmem/allocator.py:155-357) and replay()
// (allocator.py:360-393); one warp replays one trace.
//
// Per-trace state:
//
//  * allocated blocks -- one 32 B record per handle in HBM at the trace's
//    own event offset (handles are dense, < n_events):
//        addr | key | left ref | right ref
//    key = stream<<46 | size; key 0 = never used, key ~0 = freed.  A ref
//    names the neighbour inside the segment: kNone (segment edge), a handle
//    (allocated neighbour) or kFreeTag|id (free neighbour).  The refs replace
//    the reference's doubly linked chains (allocator.py:95-132): coalescing
//    on free (allocator.py:301-318) reads two refs and never searches.
//  * free blocks -- a bucketed index: buckets of <= 32 entries
//    (key, addr, links) cover disjoint (key, addr) ranges listed in a sorted
//    directory.  Best fit -- argmin (size, addr) over the request's stream
//    with rounded <= size < rounded + max_split (allocator.py:203-221;
//    SURVEY App. B) -- is one directory ballot plus a scan of one (rarely
//    two) buckets.  A free block's id is its bucket position phys*32+idx;
//    when an entry moves, its allocated neighbours' refs are re-pointed.
//    The directory is held in REGISTERS (lane d = position d) by the main
//    kernel (DirReg, <= 32 buckets in shared memory) and in memory by the
//    HBM retry kernel (DirMem, any size).
//  * scalars -- reserved / allocated / peaks / next_base / counts are
//    warp-uniform registers.
//
// Shared-memory discipline (independent thread scheduling gives no lockstep
// guarantee between collectives): a uniform update is stored by every lane
// with the same value, so each lane reads back its own store, and is
// preceded by __syncwarp() so no lane can overwrite a slot another lane has
// yet to read; lane-divergent writes (bucket splits / merges, staged-record
// mirrors) are fenced by __syncwarp() on both sides.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "peakmem_b200.h"

namespace pmb {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kSizeBits = 46;
constexpr u64 kSizeMask = (1ull << kSizeBits) - 1;
constexpr u64 kFreed = ~0ull;
constexpr u32 kNone = 0xFFFFFFFFu;
constexpr u32 kFreeTag = 0x80000000u;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kBucket = 32;
constexpr int kHalf = kBucket / 2;

__device__ __forceinline__ bool is_free_ref(u32 r) {
  return r != kNone && (r & kFreeTag);
}
__device__ __forceinline__ u32 lo32(u64 x) { return (u32)x; }
__device__ __forceinline__ u32 hi32(u64 x) { return (u32)(x >> 32); }
__device__ __forceinline__ u64 mk_links(u32 l, u32 r) {
  return (u64)l | ((u64)r << 32);
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ bool dir_le(u64 dk, u64 da, u64 k, u64 a) {
  return dk < k || (dk == k && da <= a);
}

#ifdef PM_DEBUG_UNIFORM
__device__ int g_nonuniform_line;
template <class T>
__device__ __forceinline__ void check_uniform(T v, int line) {
  const unsigned long long x = (unsigned long long)v;
  const unsigned long long x0 = __shfl_sync(0xffffffffu, x, 0);
  if (__ballot_sync(0xffffffffu, x != x0) && (threadIdx.x & 31) == 0)
    atomicCAS(&g_nonuniform_line, 0, line);
}
#define PM_UNIFORM(v) check_uniform((v), __LINE__)
#else
#define PM_UNIFORM(v) ((void)0)
#endif

// Allocator constants: the per-request ones in registers, the miss-path
// ones (segment sizing, capacity) read from the caller's config record.
struct Cfg {
  const pm_cfg_t* cp;
  u64 amask;
  long long max_split;
};

// Free-block entries (bucket storage), shared memory or HBM.
struct Pool {
  u64* key;    // [nbmax*32]  stream<<46 | size
  u64* addr;   // [nbmax*32]
  u64* links;  // [nbmax*32]  left | right<<32 (handles or kNone)
};

// Per-chunk staged copies of the records of the chunk's handles.
struct Stage {
  u64* a;
  u64* k;
  u32* L;
  u32* R;
};

// Allocated-block records: 4 u64 words per handle -- addr, key, left ref,
// right ref.  Every access is a u64 word access (no type punning), so the
// compiler cannot reorder a ref update past a later gather of the record.
struct Recs {
  u64* base;
  __device__ __forceinline__ u64* word(u32 h, int w) const {
    return base + 4 * (size_t)h + w;
  }
  __device__ __forceinline__ u64* link_ptr(u32 h, int right) const {
    return word(h, 2 + right);
  }
};

// ---- directory policies -----------------------------------------------------
//
// Both expose: nb, find(k, a), phys(d), count(d), add_count(d, delta),
// pos_of_phys(p), insert(d, k, a, p, c), erase(d), set_count(d, c),
// count_next(d), alloc_phys(), free_phys(p), nbmax.

// Directory in registers: lane d holds position d (nb <= 32 buckets).
struct DirReg {
  u64 dk, da;
  int dp, dc;
  int nb;
  int nbmax;
  int lane;
  unsigned* cta_used;  // CTA-shared bitmap of physical buckets in use
  int cta_words, cta_buckets;

  __device__ __forceinline__ void init(int nbmax_, int lane_) {
    dk = da = ~0ull;
    dp = -1;
    dc = 0;
    nb = 0;
    nbmax = nbmax_;
    lane = lane_;
  }
  __device__ __forceinline__ int find(u64 k, u64 a) const {
    const unsigned m = __ballot_sync(kFull, dir_le(dk, da, k, a));
    return 31 - __clz(m);
  }
  __device__ __forceinline__ int phys(int d) const {
    return __shfl_sync(kFull, dp, d);
  }
  __device__ __forceinline__ int count(int d) const {
    return __shfl_sync(kFull, dc, d);
  }
  __device__ __forceinline__ u64 bound_k(int d) const {
    return __shfl_sync(kFull, dk, d);
  }
  __device__ __forceinline__ u64 bound_a(int d) const {
    return __shfl_sync(kFull, da, d);
  }
  __device__ __forceinline__ int count_next(int d) const {
    return __shfl_sync(kFull, dc, d + 1);
  }
  __device__ __forceinline__ void add_count(int d, int delta) {
    if (lane == d) dc += delta;
  }
  __device__ __forceinline__ void set_count(int d, int c) {
    if (lane == d) dc = c;
  }
  __device__ __forceinline__ int pos_of_phys(int p) const {
    return __ffs(__ballot_sync(kFull, dp == p)) - 1;
  }
  // first position e < nb-1 with count(e) + count(e+1) <= 32, or -1
  __device__ __forceinline__ int mergeable() const {
    const int cn = __shfl_down_sync(kFull, dc, 1);
    const unsigned m =
        __ballot_sync(kFull, lane < nb - 1 && dc + cn <= kBucket);
    return m ? __ffs(m) - 1 : -1;
  }
  __device__ __forceinline__ void insert(int d, u64 k, u64 a, int p, int c) {
    const u64 uk = __shfl_up_sync(kFull, dk, 1);
    const u64 ua = __shfl_up_sync(kFull, da, 1);
    const int up = __shfl_up_sync(kFull, dp, 1);
    const int uc = __shfl_up_sync(kFull, dc, 1);
    if (lane > d) {
      dk = uk;
      da = ua;
      dp = up;
      dc = uc;
    } else if (lane == d) {
      dk = k;
      da = a;
      dp = p;
      dc = c;
    }
    nb += 1;
  }
  __device__ __forceinline__ void erase(int d) {
    u64 nk = __shfl_down_sync(kFull, dk, 1);
    u64 na = __shfl_down_sync(kFull, da, 1);
    int np = __shfl_down_sync(kFull, dp, 1);
    int nc = __shfl_down_sync(kFull, dc, 1);
    if (lane == 31) {
      nk = na = ~0ull;
      np = -1;
      nc = 0;
    }
    if (lane >= d) {
      dk = nk;
      da = na;
      dp = np;
      dc = nc;
    }
    nb -= 1;
    if (d == 0 && lane == 0) dk = da = 0;
  }
  // claim a free physical bucket of the CTA-shared pool; -1 if exhausted
  __device__ __forceinline__ int alloc_phys() {
    int p = -1;
    if (lane == 0) {
      for (int w = 0; w < cta_words && p < 0; ++w) {
        unsigned v = cta_used[w];
        while (v != 0xffffffffu) {
          const int b = __ffs(~v) - 1;
          const unsigned old = atomicOr(&cta_used[w], 1u << b);
          if (!(old & (1u << b))) {
            p = w * 32 + b;
            __threadfence_block();  // acquire the bucket from its last owner
            break;
          }
          v = old | (1u << b);
        }
      }
      if (p >= cta_buckets) p = -1;  // padding bits past the pool
    }
    return __shfl_sync(kFull, p, 0);
  }
  // release: this warp's accesses precede the next owner's
  __device__ __forceinline__ void free_phys(int p) {
    __syncwarp();
    __threadfence_block();
    if (lane == 0) atomicAnd(&cta_used[p >> 5], ~(1u << (p & 31)));
  }
  // hand every bucket of this warp back to the CTA pool
  __device__ __forceinline__ void release_all() {
    __syncwarp();
    __threadfence_block();
    if (lane < nb) atomicAnd(&cta_used[dp >> 5], ~(1u << (dp & 31)));
    nb = 0;
  }
  __device__ __forceinline__ bool full() const { return nb >= nbmax; }
};

// Directory in memory (retry tiers, any number of buckets): sorted bounds
// with a 32-ary warp-cooperative search and a physical -> position map.
struct DirMem {
  u64* dkey;
  u64* daddr;
  int* dphys;
  int* cnt;     // by physical bucket
  int* pstack;  // free physical buckets
  int* pos;     // by physical bucket: directory position
  int nb, ptop, nbmax, lane;

  __device__ __forceinline__ void init(int nbmax_, int lane_) {
    nb = 0;
    nbmax = nbmax_;
    lane = lane_;
    for (int i = lane; i < nbmax; i += 32) pstack[i] = nbmax - 1 - i;
    __syncwarp();
    ptop = nbmax;
  }
  // last position whose bound <= (k, a): each round 32 lanes probe evenly
  // spaced positions of the live range, shrinking it 32x
  __device__ __forceinline__ int find(u64 k, u64 a) const {
    int lo = 0, hi = nb;  // answer in [lo, hi), bound[lo] <= (k, a)
    while (hi - lo > 32) {
      const int step = (hi - lo + 31) / 32;
      const int e = lo + lane * step;
      const bool pr = e < hi && dir_le(dkey[e], daddr[e], k, a);
      const unsigned m = __ballot_sync(kFull, pr);
      const int t = 31 - __clz(m);  // lane 0 probes lo, always true
      lo = lo + t * step;
      hi = min(lo + step, hi);
    }
    const int e = lo + lane;
    const bool pr = e < hi && dir_le(dkey[e], daddr[e], k, a);
    const unsigned m = __ballot_sync(kFull, pr);
    return m ? lo + 31 - __clz(m) : lo;
  }
  __device__ __forceinline__ int phys(int d) const { return dphys[d]; }
  __device__ __forceinline__ int count(int d) const { return cnt[dphys[d]]; }
  __device__ __forceinline__ u64 bound_k(int d) const { return dkey[d]; }
  __device__ __forceinline__ u64 bound_a(int d) const { return daddr[d]; }
  __device__ __forceinline__ int count_next(int d) const {
    return cnt[dphys[d + 1]];
  }
  __device__ __forceinline__ void add_count(int d, int delta) {
    const int p = dphys[d];
    const int v = cnt[p] + delta;
    __syncwarp();
    cnt[p] = v;
    __syncwarp();
  }
  __device__ __forceinline__ void set_count(int d, int c) {
    const int p = dphys[d];
    __syncwarp();
    cnt[p] = c;
    __syncwarp();
  }
  __device__ __forceinline__ int pos_of_phys(int p) const { return pos[p]; }
  __device__ __forceinline__ int mergeable() const {
    for (int base = 0; base < nb - 1; base += 32) {
      const int x = base + lane;
      bool ok = false;
      if (x < nb - 1) ok = cnt[dphys[x]] + cnt[dphys[x + 1]] <= kBucket;
      const unsigned m = __ballot_sync(kFull, ok);
      if (m) return base + __ffs(m) - 1;
    }
    return -1;
  }
  __device__ __forceinline__ void insert(int d, u64 k, u64 a, int p, int c) {
    for (int base = ((nb - 1 - d) / 32) * 32; base >= 0; base -= 32) {
      const int e = d + base + lane;
      u64 xk = 0, xa = 0;
      int xp = 0;
      const bool mv = e < nb;
      if (mv) {
        xk = dkey[e];
        xa = daddr[e];
        xp = dphys[e];
      }
      __syncwarp();
      if (mv) {
        dkey[e + 1] = xk;
        daddr[e + 1] = xa;
        dphys[e + 1] = xp;
        pos[xp] = e + 1;
      }
      __syncwarp();
    }
    dkey[d] = k;
    daddr[d] = a;
    dphys[d] = p;
    cnt[p] = c;
    pos[p] = d;
    __syncwarp();
    nb += 1;
  }
  __device__ __forceinline__ void erase(int d) {
    for (int base = 0; d + 1 + base < nb; base += 32) {
      const int e = d + 1 + base + lane;
      u64 xk = 0, xa = 0;
      int xp = 0;
      const bool mv = e < nb;
      if (mv) {
        xk = dkey[e];
        xa = daddr[e];
        xp = dphys[e];
      }
      __syncwarp();
      if (mv) {
        dkey[e - 1] = xk;
        daddr[e - 1] = xa;
        dphys[e - 1] = xp;
        pos[xp] = e - 1;
      }
      __syncwarp();
    }
    nb -= 1;
    __syncwarp();
    if (d == 0) {
      dkey[0] = 0;
      daddr[0] = 0;
    }
    __syncwarp();
  }
  __device__ __forceinline__ int alloc_phys() {
    if (ptop == 0) return -1;
    ptop -= 1;
    return pstack[ptop];
  }
  __device__ __forceinline__ void release_all() { nb = 0; }
  __device__ __forceinline__ void free_phys(int p) {
    __syncwarp();
    pstack[ptop] = p;
    __syncwarp();
    ptop += 1;
  }
  __device__ __forceinline__ bool full() const { return nb >= nbmax; }
};

struct Ctx {
  long long reserved, allocated, peak_reserved, peak_allocated, next_base;
  int F, maxF, nseg, nseg_peak;
};

// ---- record refs (global store + staged mirror) ---------------------------

__device__ __forceinline__ void set_link(const Recs& rec, const Stage& st,
                                         int hcmp, int lane, u32 g, int right,
                                         u32 val) {
  if (lane == 0) *rec.link_ptr(g, right) = (u64)val;
  if (hcmp == (int)g) (right ? st.R : st.L)[lane] = val;
}

// Re-point the allocated neighbours of free entry `id` (links l) at it.
__device__ __forceinline__ void relink(const Recs& rec, const Stage& st,
                                       int hcmp, int lane, u64 l, int id) {
  const u32 L = lo32(l), R = hi32(l);
  if (L != kNone) set_link(rec, st, hcmp, lane, L, 1, kFreeTag | (u32)id);
  if (R != kNone) set_link(rec, st, hcmp, lane, R, 0, kFreeTag | (u32)id);
}

// Lane-parallel relink of entries that moved (each lane its own entry).
__device__ __forceinline__ void relink_lanes(const Recs& rec, const Stage& st,
                                             int hcmp, int lane, bool moved,
                                             u64 links, int dst) {
  const u32 L = lo32(links), R = hi32(links);
  const u32 val = kFreeTag | (u32)dst;
  if (moved) {
    if (L != kNone) *rec.link_ptr(L, 1) = (u64)val;
    if (R != kNone) *rec.link_ptr(R, 0) = (u64)val;
  }
  unsigned m = __ballot_sync(kFull, moved);
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const u32 gl = __shfl_sync(kFull, L, src);
    const u32 gr = __shfl_sync(kFull, R, src);
    const u32 v = __shfl_sync(kFull, val, src);
    if (gl != kNone && hcmp == (int)gl) st.R[lane] = v;
    if (gr != kNone && hcmp == (int)gr) st.L[lane] = v;
  }
  __syncwarp();
}

// ---- warp argmin over (k, a) with the address loaded only on key ties ----

__device__ __forceinline__ int argmin_ka(bool valid, u64 k, const u64* addr,
                                         int id) {
  const unsigned any = __ballot_sync(kFull, valid);
  if (!any) return -1;
  if ((any & (any - 1)) == 0) return __ffs(any) - 1;
  unsigned m = __reduce_min_sync(kFull, valid ? hi32(k) : 0xffffffffu);
  bool c = valid && hi32(k) == m;
  m = __reduce_min_sync(kFull, c ? lo32(k) : 0xffffffffu);
  c = c && lo32(k) == m;
  unsigned bm = __ballot_sync(kFull, c);
  if ((bm & (bm - 1)) == 0) return __ffs(bm) - 1;
  const u64 a = c ? addr[id] : ~0ull;
  m = __reduce_min_sync(kFull, c ? hi32(a) : 0xffffffffu);
  c = c && hi32(a) == m;
  m = __reduce_min_sync(kFull, c ? lo32(a) : 0xffffffffu);
  c = c && lo32(a) == m;
  bm = __ballot_sync(kFull, c);
  return __ffs(bm) - 1;
}

// ---- bucket maintenance -----------------------------------------------------

// Merge the first adjacent bucket pair whose entries fit in one bucket.
template <class D>
__device__ __forceinline__ bool try_merge(const Pool& P, D& dir,
                                          const Recs& rec, const Stage& st,
                                          int hcmp, int lane) {
  const int e = dir.mergeable();
  if (e < 0) return false;
  const int pa = dir.phys(e), pb = dir.phys(e + 1);
  const int na = dir.count(e), nbb = dir.count_next(e);
  const bool mv = lane < nbb;
  u64 k = 0, a = 0, l = 0;
  const int src = pb * kBucket + lane, dst = pa * kBucket + na + lane;
  if (mv) {
    k = P.key[src];
    a = P.addr[src];
    l = P.links[src];
  }
  __syncwarp();
  if (mv) {
    P.key[dst] = k;
    P.addr[dst] = a;
    P.links[dst] = l;
  }
  __syncwarp();
  relink_lanes(rec, st, hcmp, lane, mv, l, dst);
  dir.set_count(e, na + nbb);
  dir.erase(e + 1);
  dir.free_phys(pb);
  return true;
}

// Split the full bucket at directory position d into halves by (key, addr)
// rank.  False if the directory is full and nothing merges (overflow).
template <class D>
__device__ __forceinline__ bool split_bucket(const Pool& P, D& dir, int d,
                                             const Recs& rec, const Stage& st,
                                             int hcmp, int lane) {
  // a full directory first merges an adjacent pair; the caller re-finds
  // its bucket and retries (the merge always frees a directory slot)
  const int q = dir.full() ? -1 : dir.alloc_phys();
  if (q < 0) return try_merge(P, dir, rec, st, hcmp, lane);
  const int p = dir.phys(d);
  const int base = p * kBucket;
  const u64 k = P.key[base + lane];
  const u64 a = P.addr[base + lane];
  const u64 l = P.links[base + lane];
  int rank = 0;
#pragma unroll 8
  for (int j = 0; j < kBucket; ++j) {
    const u64 kj = __shfl_sync(kFull, k, j);
    const u64 aj = __shfl_sync(kFull, a, j);
    rank += (kj < k || (kj == k && aj < a)) ? 1 : 0;
  }
  const bool up = rank >= kHalf;
  const unsigned holes = __ballot_sync(kFull, up && lane < kHalf);
  const unsigned movers = __ballot_sync(kFull, !up && lane >= kHalf);
  int dst;
  if (up) {
    dst = q * kBucket + rank - kHalf;
  } else if (lane >= kHalf) {
    const int r = __popc(movers & lanemask_lt());
    dst = base + (int)__fns(holes, 0, r + 1);
  } else {
    dst = base + lane;
  }
  const int bl = __ffs(__ballot_sync(kFull, rank == kHalf)) - 1;
  const u64 bk = __shfl_sync(kFull, k, bl);
  const u64 ba = __shfl_sync(kFull, a, bl);
  __syncwarp();
  P.key[dst] = k;
  P.addr[dst] = a;
  P.links[dst] = l;
  __syncwarp();
  dir.set_count(d, kHalf);
  dir.insert(d + 1, bk, ba, q, kHalf);
  relink_lanes(rec, st, hcmp, lane, dst != base + lane, l, dst);
  return true;
}

// Insert a free block; returns its id or -1 on pool overflow.
template <class D>
__device__ __forceinline__ int pool_insert(const Pool& P, D& dir, Ctx& c,
                                           u64 k, u64 a, u64 links,
                                           const Recs& rec, const Stage& st,
                                           int hcmp, int lane) {
  if (dir.nb == 0) {
    const int q = dir.alloc_phys();
    if (q < 0) return -1;
    dir.insert(0, 0ull, 0ull, q, 0);
  }
  int d = dir.find(k, a);
  int cnt = dir.count(d);
  while (cnt >= kBucket) {
    if (!split_bucket(P, dir, d, rec, st, hcmp, lane)) return -1;
    d = dir.find(k, a);
    cnt = dir.count(d);
  }
  const int id = dir.phys(d) * kBucket + cnt;
  __syncwarp();  // every lane is past its reads of the slot
  P.key[id] = k;  // uniform store by every lane
  P.addr[id] = a;
  P.links[id] = links;
  dir.add_count(d, 1);
  c.F += 1;
  return id;
}

// Remove free block `id`; the bucket's last entry fills the hole (its
// neighbours re-pointed).  Returns the id that moved into `id` (-1: none).
template <class D>
__device__ __forceinline__ int pool_remove(const Pool& P, D& dir, Ctx& c,
                                           int id, const Recs& rec,
                                           const Stage& st, int hcmp,
                                           int lane) {
  const int p = id / kBucket;
  const int d = dir.pos_of_phys(p);
  const int last = dir.count(d) - 1;
  const int lid = p * kBucket + last;
  int moved = -1;
  if (lid != id) {
    const u64 lk = P.key[lid], la = P.addr[lid], ll = P.links[lid];
    __syncwarp();
    P.key[id] = lk;
    P.addr[id] = la;
    P.links[id] = ll;
    relink(rec, st, hcmp, lane, ll, id);
    moved = lid;
  }
  dir.add_count(d, -1);
  c.F -= 1;
  if (last == 0 && dir.nb > 1) {
    dir.erase(d);
    dir.free_phys(p);
  }
  return moved;
}

// Rekey entry `id` to (k, a, links) -- in place when it stays in its bucket
// -- or, with id < 0, insert a new entry.  Returns the entry's id (-1 on
// overflow).  The caller re-points the entry's neighbours (relink).  The
// single call site keeps one inlined copy of insert / split / merge.
template <class D>
__device__ __forceinline__ int pool_upsert(const Pool& P, D& dir, Ctx& c,
                                           int id, u64 k, u64 a, u64 links,
                                           const Recs& rec, const Stage& st,
                                           int hcmp, int lane) {
  if (id >= 0) {
    const int d = dir.find(k, a);
    if (dir.phys(d) == id / kBucket) {
      __syncwarp();
      P.key[id] = k;
      P.addr[id] = a;
      P.links[id] = links;
      return id;
    }
    pool_remove(P, dir, c, id, rec, st, hcmp, lane);
  }
  return pool_insert(P, dir, c, k, a, links, rec, st, hcmp, lane);
}

// Best fit (allocator.py:203-221): argmin (key, addr) with
// key - lo < span, i.e. same stream and rounded <= size < rounded + span.
template <class D>
__device__ __forceinline__ int best_fit(const Pool& P, const D& dir, u64 lo,
                                        u64 span, int lane) {
  if (dir.nb == 0) return -1;
  const int d = dir.find(lo, 0ull);
  {
    const int p = dir.phys(d);
    const int id = p * kBucket + lane;
    const bool in = lane < dir.count(d);
    const u64 k = in ? P.key[id] : ~0ull;
    const bool el = in && (k - lo) < span;
    const int w = argmin_ka(el, k, P.addr, id);
    if (w >= 0) return p * kBucket + w;
  }
  if (d + 1 < dir.nb) {
    // every key of the next bucket exceeds lo: its minimum is the only
    // remaining candidate
    const int p = dir.phys(d + 1);
    const int id = p * kBucket + lane;
    const bool in = lane < dir.count_next(d);
    const u64 k = in ? P.key[id] : ~0ull;
    const int w = argmin_ka(in, k, P.addr, id);
    if (w >= 0) {
      const u64 kw = __shfl_sync(kFull, k, w);
      if (kw - lo < span) return p * kBucket + w;
    }
  }
  return -1;
}

// allocator.py:86-92
__device__ __forceinline__ long long segment_size_for(long long rounded,
                                                      const Cfg& c) {
  const pm_cfg_t* cp = c.cp;
  if (rounded <= cp->k_small_size) return cp->k_small_buffer;
  if (rounded <= cp->k_min_large_alloc) return cp->k_large_buffer;
  const long long rl = cp->k_round_large;
  return ((rounded + rl - 1) / rl) * rl;
}

// Wholly-free segment (free entry with no allocated neighbour) of largest
// size > t, ties lowest addr; -1 if none.
template <class D>
__device__ __forceinline__ int find_release_candidate(const Pool& P,
                                                      const D& dir,
                                                      long long t, int lane) {
  u64 bk = ~0ull, ba = ~0ull;
  int bid = -1;
  for (int d = 0; d < dir.nb; ++d) {
    const int p = dir.phys(d);
    const int id = p * kBucket + lane;
    if (lane < dir.count(d) && P.links[id] == ~0ull) {
      const long long sz = (long long)(P.key[id] & kSizeMask);
      if (sz > t) {
        const u64 kk = kSizeMask - (u64)sz;
        const u64 a = P.addr[id];
        if (kk < bk || (kk == bk && a < ba)) {
          bk = kk;
          ba = a;
          bid = id;
        }
      }
    }
  }
  const unsigned any = __ballot_sync(kFull, bid >= 0);
  if (!any) return -1;
  unsigned m = __reduce_min_sync(kFull, bid >= 0 ? hi32(bk) : 0xffffffffu);
  bool cc = bid >= 0 && hi32(bk) == m;
  m = __reduce_min_sync(kFull, cc ? lo32(bk) : 0xffffffffu);
  cc = cc && lo32(bk) == m;
  m = __reduce_min_sync(kFull, cc ? hi32(ba) : 0xffffffffu);
  cc = cc && hi32(ba) == m;
  m = __reduce_min_sync(kFull, cc ? lo32(ba) : 0xffffffffu);
  cc = cc && lo32(ba) == m;
  const int w = __ffs(__ballot_sync(kFull, cc)) - 1;
  return __shfl_sync(kFull, bid, w);
}

// _make_room (allocator.py:258-271): stage 1 releases over-threshold
// wholly-free segments largest first (ties: creation order == ascending
// base) until the new segment fits; stage 2 releases every wholly-free one.
template <class D>
__device__ __forceinline__ void make_room(const Pool& P, D& dir, Ctx& c,
                                          long long seg, const Cfg& cf,
                                          const Recs& rec, const Stage& st,
                                          int hcmp, int lane) {
  const long long capacity = cf.cp->device_capacity;
  // stage 1 (max_split set): threshold max_split, stop once it fits;
  // stage 2: threshold -1 (every wholly-free segment), entered only if it
  // still does not fit, runs until no candidate is left
  int stage = cf.max_split >= 0 ? 1 : 2;
  if (stage == 2 && c.reserved + seg <= capacity) return;
  for (;;) {
    if (stage == 1 && c.reserved + seg <= capacity) break;
    const int id = find_release_candidate(
        P, dir, stage == 1 ? cf.max_split : -1, lane);
    if (id < 0) {
      if (stage == 2 || c.reserved + seg <= capacity) break;
      stage = 2;
      continue;
    }
    const long long sz = (long long)(P.key[id] & kSizeMask);
    pool_remove(P, dir, c, id, rec, st, hcmp, lane);
    c.reserved -= sz;
    c.nseg -= 1;
  }
}

#ifdef PM_VALIDATE
// fault injection for the validator's tests: {request index, kind}
__device__ int g_inject[2];

// ---- invariant checks (validating build) --------------------------------------
// AllocatorState.check_invariants (allocator.py:324-354) over the wide
// state after every applied request; see replay_narrow.cuh validate_narrow.
__device__ __forceinline__ bool live_k(u64 k) { return k != 0ull && k != kFreed; }

template <class D>
__device__ int validate_wide(const Pool& P, const D& dir, const Recs& rec,
                             long long n, const Ctx& c, const Cfg& cf, int lane) {
  const long long align = cf.cp->alignment;
  const long long cap = cf.cp->device_capacity;
  int bad = 0;
  long long free_b = 0, alloc_b = 0;
  int heads = 0, tails = 0, nfree = 0, free_links = 0, free_refs = 0;
  auto flag = [&](int code) {
    if (!bad) bad = code;
  };
  for (int d = 0; d < dir.nb; ++d) {
    const int p = dir.phys(d);
    const int cntd = dir.count(d);
    const u64 lk = dir.bound_k(d), la = dir.bound_a(d);
    const bool last = d + 1 >= dir.nb;
    const u64 hk = last ? ~0ull : dir.bound_k(d + 1);
    const u64 ha = last ? ~0ull : dir.bound_a(d + 1);
    if (lane < cntd) {
      const int id = p * kBucket + lane;
      const u64 K = P.key[id], A = P.addr[id], ln = P.links[id];
      const u64 S = K & kSizeMask;
      const u32 L = lo32(ln), R = hi32(ln);
      nfree += 1;
      free_b += (long long)S;
      if (S == 0) flag(PM_INV_BLOCK_SIZE);
      if ((long long)S % align) flag(PM_INV_UNALIGNED);
      if ((d > 0 && !dir_le(lk, la, K, A)) || (!last && dir_le(hk, ha, K, A)))
        flag(PM_INV_POOL);
      for (int side = 0; side < 2; ++side) {
        const u32 g = side ? R : L;
        if (g == kNone) {
          if (side) tails += 1; else heads += 1;
          continue;
        }
        free_links += 1;
        if (g & kFreeTag) {
          flag(PM_INV_ADJACENT_FREE);
          continue;
        }
        if ((long long)g >= n) {
          flag(PM_INV_LINK);
          continue;
        }
        const u64 ga = *rec.word(g, 0), gk = *rec.word(g, 1);
        const u32 back = (u32)*rec.word(g, side ? 2 : 3);
        const bool contiguous = side ? A + S == ga : ga + (gk & kSizeMask) == A;
        if (!live_k(gk) || !contiguous || back != (kFreeTag | (u32)id)) flag(PM_INV_LINK);
        else if ((gk >> kSizeBits) != (K >> kSizeBits)) flag(PM_INV_STREAM);
      }
    }
  }
  for (long long h = lane; h < n; h += 32) {
    const u64 A = *rec.word((u32)h, 0), K = *rec.word((u32)h, 1);
    if (!live_k(K)) continue;
    const u64 S = K & kSizeMask;
    alloc_b += (long long)S;
    if (S == 0) flag(PM_INV_BLOCK_SIZE);
    if ((long long)S % align) flag(PM_INV_UNALIGNED);
    for (int side = 0; side < 2; ++side) {
      const u32 g = (u32)*rec.word((u32)h, side ? 3 : 2);
      if (g == kNone) {
        if (side) tails += 1; else heads += 1;
        continue;
      }
      if (g & kFreeTag) {
        free_refs += 1;
        const int id = (int)(g & ~kFreeTag);
        const u64 ea = P.addr[id], ek = P.key[id], el = P.links[id];
        const bool ok = side ? (A + S == ea && lo32(el) == (u32)h)
                             : (ea + (ek & kSizeMask) == A && hi32(el) == (u32)h);
        if (!ok) flag(PM_INV_LINK);
        continue;
      }
      if ((long long)g >= n) {
        flag(PM_INV_LINK);
        continue;
      }
      const u64 qa = *rec.word(g, 0), qk = *rec.word(g, 1);
      const u32 back = (u32)*rec.word(g, side ? 2 : 3);
      const bool ok = side ? (A + S == qa) : (qa + (qk & kSizeMask) == A);
      if (!live_k(qk) || !ok || back != (u32)h) flag(PM_INV_LINK);
      else if ((qk >> kSizeBits) != (K >> kSizeBits)) flag(PM_INV_STREAM);
    }
  }
  const unsigned any = __ballot_sync(kFull, bad != 0);
  if (any) return __shfl_sync(kFull, bad, __ffs(any) - 1);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    free_b += __shfl_xor_sync(kFull, free_b, o);
    alloc_b += __shfl_xor_sync(kFull, alloc_b, o);
  }
  heads = __reduce_add_sync(kFull, heads);
  tails = __reduce_add_sync(kFull, tails);
  nfree = __reduce_add_sync(kFull, nfree);
  free_links = __reduce_add_sync(kFull, free_links);
  free_refs = __reduce_add_sync(kFull, free_refs);
  if (heads != c.nseg || tails != c.nseg) return PM_INV_SEGMENTS;
  if (nfree != c.F || free_links != free_refs) return PM_INV_POOL;
  if (alloc_b != c.allocated) return PM_INV_ALLOCATED;
  if (alloc_b + free_b != c.reserved) return PM_INV_CONSERVATION;
  if (cap >= 0 && c.reserved > cap) return PM_INV_CAPACITY;
  return 0;
}
#endif

// ---- one trace ---------------------------------------------------------------

template <class D>
__device__ __forceinline__ void replay_trace(
    int tr, const pm_req_t* __restrict__ reqs,
    const int64_t* __restrict__ offs, const pm_cfg_t* __restrict__ cfgs,
    const int32_t* __restrict__ cfg_of, pm_result_t* __restrict__ results,
    int64_t* __restrict__ timeline, u64* rec_base, const Pool& P,
    D& dir, int nbmax, const Stage& st, int lane) {
  const long long e0 = offs[tr];
  const long long n = offs[tr + 1] - e0;
  const pm_cfg_t* cp = cfgs + (cfg_of ? cfg_of[tr] : 0);
  Cfg cf;
  cf.cp = cp;
  cf.amask = (u64)cp->alignment - 1;
  cf.max_split = cp->max_split_size;
  const u64 amask = cf.amask;

  Recs rec;
  rec.base = rec_base + 4 * (size_t)e0;
  for (long long i = lane; i < 4 * n; i += 32) rec.base[i] = 0ull;
  dir.init(nbmax, lane);
  __syncwarp();

  Ctx c;
  c.reserved = c.allocated = c.peak_reserved = c.peak_allocated = 0;
  c.next_base = 0;
  c.F = c.maxF = c.nseg = c.nseg_peak = 0;
  int status = PM_OK;
  long long stop = -1;
  int inv = 0;  // PM_VALIDATE: the violated invariant

  const ulonglong2* rq = reinterpret_cast<const ulonglong2*>(reqs + e0);
  ulonglong2 nxt = make_ulonglong2(0ull, 0xFFFFFFFFull);
  if (lane < n) nxt = __ldg(rq + lane);

  for (long long cbase = 0; cbase < n; cbase += 32) {
    const ulonglong2 ev = nxt;
    if (cbase + 32 + lane < n) nxt = __ldg(rq + cbase + 32 + lane);
    const long long my_size = (long long)ev.x;
    const int my_h = (int)lo32(ev.y);
    const unsigned my_ks = hi32(ev.y);
    const bool my_valid = cbase + lane < n;
    const bool hok = my_valid && my_h >= 0 && (long long)my_h < n;
    u64 ra = 0, rk = 0, rl = 0;
    u64 rr = 0;
    if (hok) {
      const u64* rp = rec.word((u32)my_h, 0);
      ra = rp[0];
      rk = rp[1];
      rl = rp[2];
      rr = rp[3];
    }
    st.a[lane] = ra;
    st.k[lane] = rk;
    st.L[lane] = (u32)rl;
    st.R[lane] = (u32)rr;
    const int hcmp = hok ? my_h : -1;  // never matches a handle
    __syncwarp();

    const int cnt = (int)((n - cbase) < 32 ? (n - cbase) : 32);
    long long tl_r = 0, tl_a = 0;
    int done = cnt;
    for (int j = 0; j < cnt; ++j) {
      const long long size = __shfl_sync(kFull, my_size, j);
      const int hj = __shfl_sync(kFull, my_h, j);
      const unsigned ks = __shfl_sync(kFull, my_ks, j);
      const unsigned kind = ks & 3u;
      const unsigned m = __ballot_sync(kFull, hcmp == hj) & ((1u << j) - 1u);
      const int src = m ? 31 - __clz(m) : j;
      int sts = PM_OK;
      if (kind >= PM_KIND_UNKNOWN) {
        sts = kind == PM_KIND_UNKNOWN ? PM_UNKNOWN_KIND : PM_MISSING_FIELD;
      } else if ((unsigned)hj >= (unsigned long long)n) {
        sts = PM_BAD_HANDLE;
      } else {
        // Plan the pool work of this request (warp-uniform), then run it at
        // single sites: B) remove an entry, C) rekey-or-insert an entry and
        // re-point its neighbours, D) up to two further link fixes.
        int rm_id = -1;           // B
        bool up = false;          // C
        int up_id = -1;
        u64 up_k = 0, up_a = 0, up_l = 0;
        u32 f1 = kNone, f2 = kNone;  // D: (f1 right ref, f2 left ref) := hj
        int both_pid = -1;        // free merging on both sides
        u64 both_S = 0, both_rk = 0;
        u32 both_rR = kNone;
        bool is_alloc = kind == PM_KIND_ALLOC;
        bool split_out = false;   // alloc: out_R is the remainder entry
        u64 out_a = 0, out_k = 0;
        u32 out_L = kNone, out_R = kNone;
        if (is_alloc) {
          // allocate (allocator.py:273-292): duplicate, then zero size
          const unsigned strm = ks >> 2;
          const u64 rounded = ((u64)size + amask) & ~amask;
          if (st.k[src] != 0) {
            sts = PM_DUPLICATE_HANDLE;
          } else if (size <= 0) {
            sts = PM_ZERO_SIZE;
          } else if (strm > 0xFFFFu) {
            sts = PM_BAD_STREAM;
          } else if (rounded > kSizeMask) {
            sts = PM_SIZE_LIMIT;
          } else {
            const u64 sbits = (u64)strm << kSizeBits;
            const u64 lo = sbits | rounded;
            u64 span = kSizeMask + 1 - rounded;
            if (cf.max_split >= 0 && (u64)cf.max_split < span)
              span = (u64)cf.max_split;
            const int id = best_fit(P, dir, lo, span, lane);
            if (id >= 0) {
              // hit: _take (allocator.py:234-242), _split (:223-232)
              const u64 K = P.key[id];
              const u64 A = P.addr[id];
              const u64 Lk = P.links[id];
              const u32 Lf = lo32(Lk), Rf = hi32(Lk);
              const u64 S = K & kSizeMask;
              const bool splittable =
                  cf.max_split < 0 || (long long)S <= cf.max_split;
              out_a = A;
              out_L = Lf;
              f1 = Lf;
              if (splittable && S > rounded) {
                up = true;
                up_id = id;
                up_k = sbits | (S - rounded);
                up_a = A + rounded;
                up_l = mk_links((u32)hj, Rf);
                out_k = sbits | rounded;
                split_out = true;
              } else {
                rm_id = id;
                out_k = K;
                out_R = Rf;
                f2 = Rf;
              }
            } else {
              // miss: new segment (allocator.py:278-288, 244-250)
              const long long seg = segment_size_for((long long)rounded, cf);
              const long long capacity = cp->device_capacity;
              if (capacity >= 0 && c.reserved + seg > capacity) {
                make_room(P, dir, c, seg, cf, rec, st, hcmp, lane);
                if (c.reserved + seg > capacity) sts = PM_OOM;
              }
              if (sts == PM_OK && (u64)seg > kSizeMask) sts = PM_SIZE_LIMIT;
              if (sts == PM_OK) {
                const u64 A = (u64)c.next_base;
                c.next_base += seg;
                c.reserved += seg;
                c.nseg += 1;
                c.nseg_peak = max(c.nseg_peak, c.nseg);
                const bool splittable = cf.max_split < 0 || seg <= cf.max_split;
                out_a = A;
                if (splittable && (u64)seg > rounded) {
                  up = true;
                  up_k = sbits | ((u64)seg - rounded);
                  up_a = A + rounded;
                  up_l = mk_links((u32)hj, kNone);
                  out_k = sbits | rounded;
                  split_out = true;
                } else {
                  out_k = sbits | (u64)seg;
                }
              }
            }
          }
        } else {
          // free (allocator.py:294-320): double free before unknown handle
          const u64 rkj = st.k[src];
          if (rkj == kFreed) {
            sts = PM_DOUBLE_FREE;
          } else if (rkj == 0) {
            sts = PM_UNKNOWN_HANDLE;
          } else {
            const u64 A = st.a[src];
            const u32 L = st.L[src], R = st.R[src];
            const u64 S = rkj & kSizeMask;
            c.allocated -= (long long)S;
            const bool lf = is_free_ref(L), rf = is_free_ref(R);
            up = true;
            if (!lf && !rf) {
              up_k = rkj;
              up_a = A;
              up_l = mk_links(L, R);
            } else if (lf && !rf) {
              // the free block on the left absorbs this one
              const int pid = (int)(L & ~kFreeTag);
              up_id = pid;
              up_k = P.key[pid] + S;
              up_a = P.addr[pid];
              up_l = mk_links(lo32(P.links[pid]), R);
            } else if (!lf && rf) {
              // the free block on the right absorbs this one
              const int rid = (int)(R & ~kFreeTag);
              up_id = rid;
              up_k = P.key[rid] + S;
              up_a = A;
              up_l = mk_links(L, hi32(P.links[rid]));
            } else {
              // left absorbs this block and the right free block: the
              // right entry goes first (B), then the left is rekeyed (C)
              const int rid = (int)(R & ~kFreeTag);
              both_pid = (int)(L & ~kFreeTag);
              both_rk = P.key[rid];
              both_rR = hi32(P.links[rid]);
              both_S = S;
              rm_id = rid;
            }
          }
        }
        if (sts == PM_OK) {
          if (rm_id >= 0) {  // B
            const int moved = pool_remove(P, dir, c, rm_id, rec, st, hcmp, lane);
            if (both_pid >= 0) {
              const int pid = moved == both_pid ? rm_id : both_pid;
              up_id = pid;
              up_k = P.key[pid] + both_S + (both_rk & kSizeMask);
              up_a = P.addr[pid];
              up_l = mk_links(lo32(P.links[pid]), both_rR);
            }
          }
          if (up) {  // C
            const int nid = pool_upsert(P, dir, c, up_id, up_k, up_a, up_l,
                                        rec, st, hcmp, lane);
            if (nid < 0) {
              sts = PM_POOL_OVERFLOW;
            } else {
              relink(rec, st, hcmp, lane, up_l, nid);
              if (split_out) out_R = kFreeTag | (u32)nid;
            }
          }
        }
        if (sts == PM_OK) {
          // D: the taken block's allocated neighbours now point at hj
          if (f2 != kNone) set_link(rec, st, hcmp, lane, f2, 0, (u32)hj);
          if (f1 != kNone) set_link(rec, st, hcmp, lane, f1, 1, (u32)hj);
          PM_UNIFORM(dir.nb);
          PM_UNIFORM(c.F);
          c.maxF = max(c.maxF, c.F);
          __syncwarp();  // order after any mirror / link store to hj
          if (is_alloc) {
            PM_UNIFORM(out_L);
            PM_UNIFORM(out_R);
            PM_UNIFORM(out_k);
            PM_UNIFORM(out_a);
            c.allocated += (long long)(out_k & kSizeMask);
            c.peak_reserved = max(c.peak_reserved, c.reserved);
            c.peak_allocated = max(c.peak_allocated, c.allocated);
            st.a[j] = out_a;  // uniform stores
            st.k[j] = out_k;
            st.L[j] = out_L;
            st.R[j] = out_R;
            if (lane == j) {
              u64* rp = rec.word((u32)hj, 0);
              rp[0] = out_a;
              rp[1] = out_k;
              rp[2] = (u64)out_L;
              rp[3] = (u64)out_R;
            }
          } else {
            st.k[j] = kFreed;  // uniform store
            if (lane == j) *rec.word((u32)hj, 1) = kFreed;
          }
        }
      }
#ifdef PM_VALIDATE
      if (sts == PM_OK && g_inject[1] != 0 && cbase + j == g_inject[0]) {
        if (g_inject[1] == 1) c.allocated += 1;
        if (g_inject[1] == 2 && lane == 0 && hj >= 0) *rec.word((u32)hj, 2) = (u64)(u32)hj;
      }
      if (sts == PM_OK) {
        __syncwarp();
        const int code = validate_wide(P, dir, rec, n, c, cf, lane);
        if (code) {
          sts = PM_INVARIANT_VIOLATION;
          inv = code;
        }
      }
#endif
      if (sts != PM_OK) {
        status = sts;
        stop = cbase + j;
        done = j;
        break;
      }
      if (lane == j) {
        tl_r = c.reserved;
        tl_a = c.allocated;
      }
      __syncwarp();  // staged mirrors written by single lanes
    }
    if (timeline != nullptr && lane < done) {
      const long long gi = e0 + cbase + lane;
      reinterpret_cast<longlong2*>(timeline)[gi] = make_longlong2(tl_r, tl_a);
    }
    __syncwarp();
    if (status != PM_OK) break;
  }

  dir.release_all();
  if (lane == 0) {
    pm_result_t res;
    res.peak_reserved = c.peak_reserved;
    res.peak_allocated = c.peak_allocated;
    res.final_reserved = c.reserved;
    res.final_allocated = c.allocated;
    res.stop_index = stop;
    res.n_events_replayed =
        status == PM_OK ? n : (status == PM_OOM ? stop + 1 : stop);
    res.status = status;
    res.n_segments_final = c.nseg;
    res.n_segments_peak = c.nseg_peak;
    res.max_free_blocks = status == PM_INVARIANT_VIOLATION ? inv : c.maxF;
    results[tr] = res;
  }
}

// ---- kernels -------------------------------------------------------------------

struct Ctl {
  unsigned work[8];   // work counters: main pass, tiers 1..4
  unsigned n_list[8]; // traces queued for tier k (index 1..4)
  unsigned long long ck_used;  // checkpoint region bump counter (narrow passes)
  unsigned main_exited;        // main-pass CTAs finished
  unsigned main_done;          // 1 once every main-pass CTA has finished
  int pos_ctas;  // packed main pass: first wave by position (0: counter)
  unsigned pad[43];
};

// Shared-memory layout of the main kernel (per CTA): the bucket pool
// (3 x B*32 u64: key, addr, links), WARPS staging areas (32 x 24 B each) and
// the pool's in-use bitmap.  The HBM retry kernel gives each warp a private
// region: pool + staging + a memory directory (2 x nbmax u64 + 3 x nbmax int).
__host__ __device__ __forceinline__ size_t smem_cta_bytes(int buckets,
                                                          int warps) {
  return (size_t)buckets * kBucket * 24 + (size_t)warps * 32 * 24 +
         (size_t)((buckets + 31) / 32) * 4;
}
__host__ __device__ __forceinline__ size_t gmem_warp_bytes(int nbmax) {
  return ((size_t)nbmax * kBucket * 24 + 32 * 24 + (size_t)nbmax * 32 + 255) /
         256 * 256;
}

__device__ __forceinline__ void carve_pool(char* base, int nbuckets, Pool& P) {
  const size_t E = (size_t)nbuckets * kBucket;
  u64* q = reinterpret_cast<u64*>(base);
  P.key = q;
  P.addr = q + E;
  P.links = q + 2 * E;
}

__device__ __forceinline__ void carve_stage(char* base, Stage& st) {
  u64* s = reinterpret_cast<u64*>(base);
  st.a = s;
  st.k = s + 32;
  st.L = reinterpret_cast<u32*>(s + 64);
  st.R = st.L + 32;
}

// Main kernel: persistent warps pull traces (longest first) from a global
// counter.  The CTA's warps share one shared-memory bucket pool (free-block
// counts vary 10x between traces, so pooling fits far more warps per SM than
// private worst-case pools); each warp's directory lives in its registers.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    replay_smem_kernel(const pm_req_t* __restrict__ reqs,
                       const int64_t* __restrict__ offs,
                       const pm_cfg_t* __restrict__ cfgs,
                       const int32_t* __restrict__ cfg_of,
                       pm_result_t* __restrict__ results,
                       int64_t* __restrict__ timeline, u64* recs, Ctl* ctl,
                       int pass, const int32_t* __restrict__ list, int n_host,
                       int32_t* __restrict__ overflow_list, int buckets,
                       const unsigned* __restrict__ group_end, int n_groups,
                       const volatile unsigned* ready) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  Pool P;
  carve_pool(smem, buckets, P);
  Stage st;
  carve_stage(smem + (size_t)buckets * kBucket * 24 + (size_t)wib * 32 * 24,
              st);
  unsigned* used = reinterpret_cast<unsigned*>(
      smem + (size_t)buckets * kBucket * 24 + (size_t)WARPS * 32 * 24);
  const int words = (buckets + 31) / 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) used[i] = 0u;
  __syncthreads();
  DirReg dir;
  dir.cta_used = used;
  dir.cta_words = words;
  dir.cta_buckets = buckets;
  const unsigned n = pass == 0 ? (unsigned)n_host : ctl->n_list[pass];
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&ctl->work[pass], 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= n) break;
    if (ready != nullptr) {
      // streamed input: wait until the copy engine has landed this trace's
      // group (its flag is written after the group's requests, in order)
      if (lane == 0) {
        int g = 0;
        while (g + 1 < n_groups && t >= group_end[g]) ++g;
        while (ready[g] == 0u) __nanosleep(2000);
      }
      __syncwarp();
    }
    const int tr = list ? list[t] : (int)t;
    replay_trace(tr, reqs, offs, cfgs, cfg_of, results, timeline, recs, P,
                 dir, kBucket, st, lane);
    __syncwarp();
    if (lane == 0 && results[tr].status == PM_POOL_OVERFLOW) {
      const unsigned k = atomicAdd(&ctl->n_list[pass + 1], 1u);
      overflow_list[k] = tr;
    }
  }
}

// Tiers 2-4 -- traces whose free blocks outgrew a dedicated 32-bucket
// register directory: the same replay with a memory-resident directory.
//   MODE 0 (tier 2): one warp owns a whole SM's shared memory (~290
//           buckets), entries and directory both in shared memory;
//   MODE 1 (tier 3): the directory (and the chunk staging) in shared
//           memory, up to ~7k buckets, the entries in an HBM pool -- every
//           directory search stays on-chip, only entry reads go to L2/HBM;
//   MODE 2 (tier 4): everything in a per-warp HBM region sized for the
//           longest trace (free blocks never exceed live allocations + live
//           segments <= 2 x requests, and with every adjacent bucket pair
//           holding > 32 entries a directory of n/8+4 buckets always has
//           room).
__host__ __device__ __forceinline__ size_t hybrid_smem_bytes(int nbmax) {
  return 32 * 24 + (size_t)nbmax * 32;
}
__host__ __device__ __forceinline__ size_t hybrid_pool_bytes(int nbmax) {
  return ((size_t)nbmax * kBucket * 24 + 255) / 256 * 256;
}

template <int WARPS, int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1)
    replay_dirmem_kernel(const pm_req_t* __restrict__ reqs,
                         const int64_t* __restrict__ offs,
                         const pm_cfg_t* __restrict__ cfgs,
                         const int32_t* __restrict__ cfg_of,
                         pm_result_t* __restrict__ results,
                         int64_t* __restrict__ timeline, u64* recs, Ctl* ctl,
                         int pass, const int32_t* __restrict__ list,
                         int32_t* __restrict__ overflow_list,
                         char* __restrict__ gpool, int nbmax) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * WARPS + wib;
  Pool P;
  Stage st;
  char* dbase;  // staging area followed by the directory arrays
  if (MODE == 1) {
    carve_pool(gpool + (size_t)gw * hybrid_pool_bytes(nbmax), nbmax, P);
    dbase = smem + (size_t)wib * hybrid_smem_bytes(nbmax);
  } else {
    char* base = MODE == 0 ? smem + (size_t)wib * gmem_warp_bytes(nbmax)
                           : gpool + (size_t)gw * gmem_warp_bytes(nbmax);
    carve_pool(base, nbmax, P);
    dbase = base + (size_t)nbmax * kBucket * 24;
  }
  carve_stage(dbase, st);
  DirMem dir;
  {
    u64* q = reinterpret_cast<u64*>(dbase + 32 * 24);
    dir.dkey = q;
    dir.daddr = q + nbmax;
    int* ip = reinterpret_cast<int*>(q + 2 * (size_t)nbmax);
    dir.dphys = ip;
    dir.cnt = ip + nbmax;
    dir.pstack = ip + 2 * nbmax;
    dir.pos = ip + 3 * nbmax;
  }
  const unsigned n = ctl->n_list[pass];
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&ctl->work[pass], 1u);
    t = __shfl_sync(kFull, t, 0);
    if (t >= n) break;
    const int tr = list[t];
    replay_trace(tr, reqs, offs, cfgs, cfg_of, results, timeline, recs, P,
                 dir, nbmax, st, lane);
    __syncwarp();
    if (overflow_list != nullptr && lane == 0 &&
        results[tr].status == PM_POOL_OVERFLOW) {
      const unsigned k = atomicAdd(&ctl->n_list[pass + 1], 1u);
      overflow_list[k] = tr;
    }
  }
}

}  // namespace pmb
