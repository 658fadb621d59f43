/*
 * TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT PATH.
 *
 * CPU oracle for the batched replay: a line-by-line C restatement of the
 * reference's fast simulator, peakmem.allocator (reference tree
 * /root/reference/pkg/src/peakmem/allocator.py), keeping ITS data structures
 * rather than the GPU engine's:
 *   - segments with doubly linked block chains   (allocator.py:95-132)
 *   - one free pool sorted by (stream, size, addr), maintained by insort
 *     and a bisect_left                          (allocator.py:163-199)
 *   - best fit = forward walk from bisect_left((stream, rounded, 0))
 *                                                 (allocator.py:203-221)
 *   - split / take / new segment / release / make_room
 *                                                 (allocator.py:223-271)
 *   - allocate / free / replay, error precedence  (allocator.py:273-320,
 *                                                  360-393)
 * plus the segment counts the reference keeps implicitly in
 * AllocatorState.segments (len() after every request).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load
 * this library, always as the checker / the reported CPU baseline.
 * Pinned against the reference itself by tests/golden (see
 * tests/golden/make_golden.py, run in a container where the reference is
 * importable).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/peakmem_b200.h"

enum { FREE_ST = 0, ALLOC_ST = 1 };

typedef struct {
  int32_t seg;
  int64_t offset, size;
  int32_t state, stream;
  int32_t prev, next;
} OBlock;

typedef struct {
  int64_t base, size;
  int32_t stream, head;
} OSeg;

typedef struct {
  int64_t stream, size, addr;
  int32_t block;
} OPoolEnt;

typedef struct {
  pm_cfg_t cfg;
  OBlock* blocks;
  int64_t nblocks, capblocks;
  OSeg* segs;
  int64_t nsegs_all, capsegs;
  int32_t* seglist; /* live segments in creation order (Python list) */
  int64_t nseglist, capseglist;
  OPoolEnt* pool;
  int64_t npool, cappool;
  int32_t* amap;  /* handle -> block, -1 */
  uint8_t* freed; /* handle -> freed */
  int64_t next_base, reserved, allocated, peak_reserved, peak_allocated;
  int32_t nseg_peak, max_pool;
} OState;

static void* grow(void* p, int64_t* cap, int64_t need, size_t elt) {
  if (need <= *cap) return p;
  int64_t c = *cap ? *cap : 16;
  while (c < need) c *= 2;
  void* q = realloc(p, (size_t)c * elt);
  if (!q) abort();
  *cap = c;
  return q;
}

static int64_t block_addr(const OState* s, int32_t b) {
  return s->segs[s->blocks[b].seg].base + s->blocks[b].offset;
}

/* lexicographic (stream, size, addr) compare */
static int key_lt(int64_t s1, int64_t z1, int64_t a1, int64_t s2, int64_t z2,
                  int64_t a2) {
  if (s1 != s2) return s1 < s2;
  if (z1 != z2) return z1 < z2;
  return a1 < a2;
}

/* _bisect_left over the (stream, size, addr) prefix (allocator.py:191-199) */
static int64_t bisect_left(const OState* s, int64_t st, int64_t sz,
                           int64_t ad) {
  int64_t lo = 0, hi = s->npool;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    const OPoolEnt* e = &s->pool[mid];
    if (key_lt(e->stream, e->size, e->addr, st, sz, ad))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* _pool_add: insort (allocator.py:180-181); keys are unique per block */
static void pool_add(OState* s, int32_t b) {
  const OBlock* k = &s->blocks[b];
  int64_t ad = block_addr(s, b);
  int64_t i = bisect_left(s, k->stream, k->size, ad);
  s->pool = grow(s->pool, &s->cappool, s->npool + 1, sizeof(OPoolEnt));
  memmove(&s->pool[i + 1], &s->pool[i],
          (size_t)(s->npool - i) * sizeof(OPoolEnt));
  s->pool[i].stream = k->stream;
  s->pool[i].size = k->size;
  s->pool[i].addr = ad;
  s->pool[i].block = b;
  s->npool++;
}

/* _pool_remove (allocator.py:183-189) */
static void pool_remove(OState* s, int32_t b) {
  const OBlock* k = &s->blocks[b];
  int64_t i = bisect_left(s, k->stream, k->size, block_addr(s, b));
  if (i >= s->npool || s->pool[i].block != b) abort(); /* assert entry[3] is block */
  memmove(&s->pool[i], &s->pool[i + 1],
          (size_t)(s->npool - i - 1) * sizeof(OPoolEnt));
  s->npool--;
}

static int32_t new_block(OState* s, int32_t seg, int64_t off, int64_t size,
                         int32_t state) {
  s->blocks = grow(s->blocks, &s->capblocks, s->nblocks + 1, sizeof(OBlock));
  OBlock* b = &s->blocks[s->nblocks];
  b->seg = seg;
  b->offset = off;
  b->size = size;
  b->state = state;
  b->stream = s->segs[seg].stream;
  b->prev = b->next = -1;
  return (int32_t)s->nblocks++;
}

/* _find_best_fit (allocator.py:203-221) */
static int32_t find_best_fit(const OState* s, int64_t rounded, int64_t stream) {
  int64_t t = s->cfg.max_split_size;
  int64_t i = bisect_left(s, stream, rounded, 0);
  while (i < s->npool) {
    const OPoolEnt* e = &s->pool[i];
    if (e->stream != stream) return -1;
    if (t >= 0 && e->size > t && e->size - rounded >= t) {
      i++;
      continue;
    }
    return e->block;
  }
  return -1;
}

/* _split (allocator.py:223-232) */
static void split(OState* s, int32_t b, int64_t rounded) {
  int64_t remainder = s->blocks[b].size - rounded;
  int32_t tail = new_block(s, s->blocks[b].seg, s->blocks[b].offset + rounded,
                           remainder, FREE_ST);
  OBlock* B = &s->blocks[b];
  OBlock* T = &s->blocks[tail];
  T->prev = b;
  T->next = B->next;
  if (B->next >= 0) s->blocks[B->next].prev = tail;
  B->next = tail;
  B->size = rounded;
  pool_add(s, tail);
}

/* _take (allocator.py:234-242) */
static void take(OState* s, int32_t b, int64_t rounded, int32_t handle) {
  pool_remove(s, b);
  int64_t t = s->cfg.max_split_size;
  int splittable = t < 0 || s->blocks[b].size <= t;
  if (splittable && s->blocks[b].size > rounded) split(s, b, rounded);
  s->blocks[b].state = ALLOC_ST;
  s->amap[handle] = b;
  s->allocated += s->blocks[b].size;
}

/* _new_segment (allocator.py:244-250) */
static int32_t new_segment(OState* s, int64_t seg_size, int64_t stream) {
  s->segs = grow(s->segs, &s->capsegs, s->nsegs_all + 1, sizeof(OSeg));
  int32_t si = (int32_t)s->nsegs_all++;
  s->segs[si].base = s->next_base;
  s->segs[si].size = seg_size;
  s->segs[si].stream = (int32_t)stream;
  s->segs[si].head = new_block(s, si, 0, seg_size, FREE_ST);
  s->next_base += seg_size;
  s->seglist = grow(s->seglist, &s->capseglist, s->nseglist + 1, sizeof(int32_t));
  s->seglist[s->nseglist++] = si;
  s->reserved += seg_size;
  pool_add(s, s->segs[si].head);
  if (s->nseglist > s->nseg_peak) s->nseg_peak = (int32_t)s->nseglist;
  return si;
}

static int wholly_free(const OState* s, int32_t si) {
  const OBlock* h = &s->blocks[s->segs[si].head];
  return h->next < 0 && h->state == FREE_ST;
}

/* _release_segment (allocator.py:252-256): list.remove keeps order */
static void release_segment(OState* s, int32_t si) {
  pool_remove(s, s->segs[si].head);
  for (int64_t i = 0; i < s->nseglist; ++i) {
    if (s->seglist[i] == si) {
      memmove(&s->seglist[i], &s->seglist[i + 1],
              (size_t)(s->nseglist - i - 1) * sizeof(int32_t));
      s->nseglist--;
      break;
    }
  }
  s->reserved -= s->segs[si].size;
}

/* _make_room (allocator.py:258-271) */
static int make_room(OState* s, int64_t seg_size) {
  int64_t cap = s->cfg.device_capacity;
  int64_t t = s->cfg.max_split_size;
  if (t >= 0) {
    /* over = [...]; sorted(over, key=-size) is stable */
    int64_t n = 0;
    int32_t* over = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->nseglist + 1));
    for (int64_t i = 0; i < s->nseglist; ++i) {
      int32_t si = s->seglist[i];
      if (wholly_free(s, si) && s->segs[si].size > t) over[n++] = si;
    }
    /* stable insertion sort by descending size */
    for (int64_t i = 1; i < n; ++i) {
      int32_t v = over[i];
      int64_t j = i - 1;
      while (j >= 0 && s->segs[over[j]].size < s->segs[v].size) {
        over[j + 1] = over[j];
        --j;
      }
      over[j + 1] = v;
    }
    for (int64_t i = 0; i < n; ++i) {
      if (s->reserved + seg_size <= cap) break;
      release_segment(s, over[i]);
    }
    free(over);
  }
  if (s->reserved + seg_size > cap) {
    int64_t n = 0;
    int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->nseglist + 1));
    for (int64_t i = 0; i < s->nseglist; ++i)
      if (wholly_free(s, s->seglist[i])) all[n++] = s->seglist[i];
    for (int64_t i = 0; i < n; ++i) release_segment(s, all[i]);
    free(all);
  }
  return s->reserved + seg_size <= cap;
}

/* segment_size_for (allocator.py:86-92), on the ROUNDED size */
static int64_t segment_size_for(int64_t size, const pm_cfg_t* c) {
  if (size <= c->k_small_size) return c->k_small_buffer;
  if (size <= c->k_min_large_alloc) return c->k_large_buffer;
  return ((size + c->k_round_large - 1) / c->k_round_large) * c->k_round_large;
}

/* allocate (allocator.py:273-292); returns a pm_status_t */
static int allocate(OState* s, int32_t handle, int64_t size, int64_t stream) {
  if (s->amap[handle] >= 0 || s->freed[handle]) return PM_DUPLICATE_HANDLE;
  if (size <= 0) return PM_ZERO_SIZE; /* round_request (allocator.py:79-83) */
  int64_t a = s->cfg.alignment;
  int64_t rounded = ((size + a - 1) / a) * a;
  int32_t b = find_best_fit(s, rounded, stream);
  if (b < 0) {
    int64_t seg_size = segment_size_for(rounded, &s->cfg);
    int64_t cap = s->cfg.device_capacity;
    if (cap >= 0 && s->reserved + seg_size > cap) {
      if (!make_room(s, seg_size)) return PM_OOM;
    }
    int32_t si = new_segment(s, seg_size, stream);
    b = s->segs[si].head;
  }
  take(s, b, rounded, handle);
  if (s->reserved > s->peak_reserved) s->peak_reserved = s->reserved;
  if (s->allocated > s->peak_allocated) s->peak_allocated = s->allocated;
  return PM_OK;
}

/* free (allocator.py:294-320) */
static int free_handle(OState* s, int32_t handle) {
  if (s->freed[handle]) return PM_DOUBLE_FREE;
  int32_t b = s->amap[handle];
  if (b < 0) return PM_UNKNOWN_HANDLE;
  s->amap[handle] = -1;
  s->freed[handle] = 1;
  s->allocated -= s->blocks[b].size;
  s->blocks[b].state = FREE_ST;
  int32_t nxt = s->blocks[b].next;
  if (nxt >= 0 && s->blocks[nxt].state == FREE_ST) {
    pool_remove(s, nxt);
    s->blocks[b].size += s->blocks[nxt].size;
    s->blocks[b].next = s->blocks[nxt].next;
    if (s->blocks[nxt].next >= 0) s->blocks[s->blocks[nxt].next].prev = b;
  }
  int32_t prv = s->blocks[b].prev;
  if (prv >= 0 && s->blocks[prv].state == FREE_ST) {
    pool_remove(s, prv);
    s->blocks[prv].size += s->blocks[b].size;
    s->blocks[prv].next = s->blocks[b].next;
    if (s->blocks[b].next >= 0) s->blocks[s->blocks[b].next].prev = prv;
    b = prv;
  }
  pool_add(s, b);
  return PM_OK;
}

/* replay (allocator.py:360-393) over one packed trace */
int oracle_replay(const pm_req_t* reqs, int64_t n, const pm_cfg_t* cfg,
                  pm_result_t* out, int64_t* timeline) {
  OState s;
  memset(&s, 0, sizeof(s));
  s.cfg = *cfg;
  s.amap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  s.freed = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  for (int64_t i = 0; i < n; ++i) s.amap[i] = -1;
  int status = PM_OK;
  int64_t stop = -1;
  for (int64_t i = 0; i < n; ++i) {
    const pm_req_t* r = &reqs[i];
    unsigned kind = r->kind_stream & 3u;
    unsigned stream = r->kind_stream >> 2;
    int st = PM_OK;
    if (kind == PM_KIND_UNKNOWN)
      st = PM_UNKNOWN_KIND;
    else if (kind == PM_KIND_MISSING_FIELD)
      st = PM_MISSING_FIELD;
    else if (r->handle < 0 || r->handle >= n)
      st = PM_BAD_HANDLE;
    else if (kind == PM_KIND_ALLOC)
      st = allocate(&s, r->handle, r->size, (int64_t)stream);
    else
      st = free_handle(&s, r->handle);
    if (st != PM_OK) {
      status = st;
      stop = i;
      break;
    }
    if (s.npool > s.max_pool) s.max_pool = (int32_t)s.npool;
    if (timeline) {
      timeline[2 * i] = s.reserved;
      timeline[2 * i + 1] = s.allocated;
    }
  }
  out->peak_reserved = s.peak_reserved;
  out->peak_allocated = s.peak_allocated;
  out->final_reserved = s.reserved;
  out->final_allocated = s.allocated;
  out->stop_index = stop;
  out->n_events_replayed =
      status == PM_OK ? n : (status == PM_OOM ? stop + 1 : stop);
  out->status = status;
  out->n_segments_final = (int32_t)s.nseglist;
  out->n_segments_peak = s.nseg_peak;
  out->max_free_blocks = s.max_pool;
  free(s.blocks);
  free(s.segs);
  free(s.seglist);
  free(s.pool);
  free(s.amap);
  free(s.freed);
  return 0;
}

typedef struct {
  const pm_req_t* reqs;
  const int64_t* offs;
  const pm_cfg_t* cfgs;
  const int32_t* cfg_of;
  pm_result_t* out;
  int64_t* timeline;
  int32_t n_traces;
  volatile int32_t* next;
} Job;

static void* worker(void* arg) {
  Job* j = (Job*)arg;
  for (;;) {
    int32_t t = __atomic_fetch_add(j->next, 1, __ATOMIC_RELAXED);
    if (t >= j->n_traces) break;
    int64_t e0 = j->offs[t], n = j->offs[t + 1] - e0;
    const pm_cfg_t* c = j->cfgs + (j->cfg_of ? j->cfg_of[t] : 0);
    oracle_replay(j->reqs + e0, n, c, j->out + t,
                  j->timeline ? j->timeline + 2 * e0 : NULL);
  }
  return NULL;
}

/* Independent traces on `n_threads` host threads (one trace per task). */
int oracle_replay_batch(const pm_req_t* reqs, const int64_t* offs,
                        int32_t n_traces, const pm_cfg_t* cfgs,
                        const int32_t* cfg_of, pm_result_t* out,
                        int64_t* timeline, int32_t n_threads) {
  volatile int32_t next = 0;
  Job job = {reqs, offs, cfgs, cfg_of, out, timeline, n_traces, &next};
  if (n_threads <= 1) {
    worker(&job);
    return 0;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, worker, &job);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return 0;
}
