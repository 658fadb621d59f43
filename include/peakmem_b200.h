/*
 * peakmem_b200.h -- C ABI of the B200 engine for the xMem (arXiv 2504.03887)
 * data-parallel hot path: batched caching-allocator replay.
 *
 * Every entry point is plain C: pointers, sizes and an opaque CUDA stream
 * handle (cudaStream_t passed as void*).  No torch types cross the boundary.
 * Return value: 0 on success, otherwise a pm_err_t code (never aborts);
 * pm_last_error() returns a static description of the last failure on the
 * calling thread.  The library keeps no global state besides that string and
 * is re-entrant per (device, stream).
 *
 * Reference interface each entry point replaces (paths relative to the
 * reference tree /root/reference):
 *   pm_replay_batch        -> peakmem.allocator.replay(requests, cfg, validate)
 *                             pkg/src/peakmem/allocator.py:360-393, applied to
 *                             many independent traces at once (one warp each)
 *   pm_replay_host         -> same, called with HOST buffers (H2D/D2H inside);
 *                             this is what a ctypes/cgo/JNI binding of
 *                             peakmem.estimator's `replay` (estimator.py:9,152)
 *                             would call
 *   pm_cfg_t               -> peakmem.allocator.AllocatorConfig
 *                             (allocator.py:49-76)
 *   pm_result_t            -> peakmem.allocator.SimulationResult
 *                             (allocator.py:135-152) plus the segment counts
 *                             the reference keeps in AllocatorState.segments
 *                             (allocator.py:161,247,255)
 *   pm_status_t            -> the exception taxonomy of replay()
 *                             (allocator.py:371-385, errors.py:52-78)
 */
#ifndef PEAKMEM_B200_H
#define PEAKMEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- packed request record (16 B, read with one 128-bit load) ---------- */
/* kind_stream: bits 0-1 kind, bits 2-31 dense stream id (< 65536).         */
enum {
  PM_KIND_ALLOC = 0,        /* "alloc"  (allocator.py:374-375)               */
  PM_KIND_FREE = 1,         /* "free"   (allocator.py:376-377)               */
  PM_KIND_UNKNOWN = 2,      /* any other kind -> MalformedSequence (:379)    */
  PM_KIND_MISSING_FIELD = 3 /* alloc without "size" -> KeyError (:375)       */
};
typedef struct {
  int64_t size;        /* requested bytes (ignored for frees)               */
  int32_t handle;      /* dense per-trace handle, 0 <= handle < n_events    */
  uint32_t kind_stream;
} pm_req_t;

/* ---- allocator configuration (AllocatorConfig, allocator.py:49-76) ----- */
typedef struct {
  int64_t k_small_size;      /* 1 MiB  */
  int64_t k_small_buffer;    /* 2 MiB  */
  int64_t k_min_large_alloc; /* 10 MiB */
  int64_t k_large_buffer;    /* 20 MiB */
  int64_t k_round_large;     /* 2 MiB  */
  int64_t alignment;         /* 512, power of two */
  int64_t max_split_size;    /* < 0 : None (unbounded) */
  int64_t device_capacity;   /* < 0 : None (never OOM) */
} pm_cfg_t;

/* ---- per-trace status (first failure in sequence order wins) ---------- */
typedef enum {
  PM_OK = 0,
  PM_OOM = 1,              /* OutOfMemory verdict: stop_index = failing req */
  PM_UNKNOWN_HANDLE = 2,   /* -> MalformedSequence                          */
  PM_DOUBLE_FREE = 3,      /* -> MalformedSequence                          */
  PM_DUPLICATE_HANDLE = 4, /* -> MalformedSequence                          */
  PM_ZERO_SIZE = 5,        /* -> ZeroSize (propagates unwrapped)            */
  PM_UNKNOWN_KIND = 6,     /* -> MalformedSequence                          */
  PM_MISSING_FIELD = 7,    /* -> KeyError                                   */
  PM_BAD_HANDLE = 8,       /* handle outside [0, n_events): caller bug      */
  PM_SIZE_LIMIT = 9,       /* a block >= 2^46 B: outside the engine's range */
  PM_BAD_STREAM = 10,      /* stream id >= 65536                            */
  PM_POOL_OVERFLOW = 11,   /* internal; resolved by the global-pool retry   */
  PM_ENCODING_LIMIT = 12,  /* internal; the narrow pass hands the trace to
                              the wide (64-bit) tiers                       */
  PM_INVARIANT_VIOLATION = 13 /* validating build only (libpeakmem_b200_
                              validate.so, -DPM_VALIDATE): the allocator
                              state broke an invariant of check_invariants
                              (allocator.py:324-354) after request
                              stop_index; max_free_blocks holds the
                              pm_invariant_t code -> AssertionError        */
} pm_status_t;

/* Invariants the validating build checks after EVERY applied request
 * (AllocatorState.check_invariants, allocator.py:324-354, run after each
 * allocate / free when validate=True, :291-292 / :319-320), restated over
 * the engine's state (free-entry index + per-handle records with neighbour
 * refs instead of per-segment block chains): */
typedef enum {
  PM_INV_BLOCK_SIZE = 1,    /* a block of size <= 0 ("blk.size > 0")         */
  PM_INV_UNALIGNED = 2,     /* size % alignment != 0 ("unaligned block")     */
  PM_INV_LINK = 3,          /* a neighbour ref that is not mutual, not live
                               or not address-contiguous ("tiling gap /
                               overlap", "broken back-link")               */
  PM_INV_ADJACENT_FREE = 4, /* two free blocks adjacent ("adjacent free")   */
  PM_INV_SEGMENTS = 5,      /* chain heads / tails != segments              */
  PM_INV_CONSERVATION = 6,  /* free + allocated != reserved ("conservation") */
  PM_INV_ALLOCATED = 7,     /* live blocks != allocated_bytes               */
  PM_INV_POOL = 8,          /* pool entries != free blocks of the chains, or
                               an entry outside its index range ("pool and
                               segment chains disagree")                   */
  PM_INV_CAPACITY = 9,      /* reserved > device_capacity                   */
  PM_INV_STREAM = 10        /* neighbours on different streams              */
} pm_invariant_t;

typedef struct {
  int64_t peak_reserved;
  int64_t peak_allocated;
  int64_t final_reserved;
  int64_t final_allocated;
  int64_t stop_index;        /* index of the OOM / first malformed request, -1 */
  int64_t n_events_replayed; /* requests consumed, including an OOM request */
  int32_t status;            /* pm_status_t */
  int32_t n_segments_final;  /* len(AllocatorState.segments) at the end */
  int32_t n_segments_peak;   /* max len(AllocatorState.segments) */
  int32_t max_free_blocks;   /* high-water mark of the free pool (diagnostic) */
} pm_result_t;               /* 64 B */

/* ---- library-level errors (return codes) ------------------------------ */
typedef enum {
  PM_SUCCESS = 0,
  PM_ERR_INVALID_ARGUMENT = 1,
  PM_ERR_CUDA = 2,
  PM_ERR_WORKSPACE_TOO_SMALL = 3,
  PM_ERR_NO_DEVICE = 4,
  PM_ERR_CYCLIC_PARENT = 5,  /* pm_layer_tree: -> CyclicParentLink */
  PM_ERR_ENGINE_LIMIT = 6,   /* a packed key range exceeded: -> EngineLimitExceeded */
  PM_ERR_SKIPPED = 7         /* pm_pipeline_batch: the caller skipped the trace */
} pm_err_t;

const char* pm_last_error(void);
int pm_version(void);

/* Validating build only (libpeakmem_b200_validate.so): corrupt the state
 * right after request `request_index` of every trace so tests can see the
 * invariant checks fire (kind 1: allocated_bytes off by one unit; kind 2: a
 * neighbour ref that is not mutual; 0: off).  The regular build returns
 * PM_ERR_INVALID_ARGUMENT. */
int pm_validate_inject(int64_t request_index, int32_t kind);

/* Bytes of device workspace pm_replay_batch needs for a batch with
 * `total_events` requests, whose longest trace has `max_trace_events`. */
int pm_replay_workspace_bytes(int64_t total_events, int64_t max_trace_events,
                              int32_t n_traces, size_t* out_bytes);

/* Batched replay, all pointers DEVICE pointers (caller-owned):
 *   reqs            packed requests of every trace, concatenated
 *   trace_offsets   n_traces+1 int64 prefix offsets into reqs
 *   cfgs            configs; cfg_of_trace[i] indexes it (NULL -> cfgs[0])
 *   trace_order     optional processing order (e.g. longest first), NULL ok
 *   results         n_traces pm_result_t
 *   timeline        optional (NULL ok): 2 x int64 (reserved, allocated) per
 *                   request, written for every successfully applied request
 *   workspace       >= pm_replay_workspace_bytes(...) bytes
 *   total_events    == trace_offsets[n_traces] - trace_offsets[0]
 *   max_trace_events = longest trace (sizes the global-pool retry)
 * Asynchronous on `stream` (a cudaStream_t). */
int pm_replay_batch(const pm_req_t* reqs, const int64_t* trace_offsets,
                    int32_t n_traces, const pm_cfg_t* cfgs,
                    const int32_t* cfg_of_trace, const int32_t* trace_order,
                    pm_result_t* results, int64_t* timeline, void* workspace,
                    size_t workspace_bytes, int64_t total_events,
                    int64_t max_trace_events, void* stream);

/* Same replay from HOST buffers: copies inputs in, replays, copies results
 * (and the optional timeline) out, synchronously.  Device memory is taken
 * from the stream-ordered pool of the current device. */
int pm_replay_host(const pm_req_t* reqs, const int64_t* trace_offsets,
                   int32_t n_traces, const pm_cfg_t* cfgs, int32_t n_cfgs,
                   const int32_t* cfg_of_trace, pm_result_t* results,
                   int64_t* timeline, void* stream);

/* ---- 8-byte wire format for host-buffer replay --------------------------
 * replay() input (allocator.py:360-393) after the packer's handle interning
 * is, in the common case, "alloc of the next new handle with a size" or
 * "free of handle h".  Those fit one 64-bit word:
 *   bits 63..62 = 0 : alloc, handle = number of allocs before it in the
 *                     trace, stream 0, size = bits 61..0 (>= 1)
 *   bits 63..62 = 1 : free of handle bits 30..0
 * pm_wire_pack converts pm_req_t traces to wire words; it returns
 * PM_ERR_INVALID_ARGUMENT (and *first_bad = the request index) when a
 * request does not fit (an alloc of another handle, a stream, a size < 1 or
 * >= 2^62, an unknown kind), in which case the caller uses pm_replay_host.
 * pm_replay_host_wire is pm_replay_host on wire words: half the H2D bytes,
 * bit-identical results.  pm_wire_pack runs on host threads (contiguous runs
 * of traces), so packing keeps up with the zero-copy replay. */
#define PM_WIRE_FREE (1ull << 62)
int pm_wire_pack(const pm_req_t* reqs, const int64_t* trace_offsets,
                 int32_t n_traces, uint64_t* words, int64_t* first_bad);
int pm_replay_host_wire(const uint64_t* words, const int64_t* trace_offsets,
                        int32_t n_traces, const pm_cfg_t* cfgs, int32_t n_cfgs,
                        const int32_t* cfg_of_trace, pm_result_t* results,
                        int64_t* timeline, void* stream);

/* ---- batched capacity bisection ------------------------
 * The smallest device_capacity each trace replays in without OutOfMemory,
 * found by bisection over whole-batch replays.  No reference function does
 * the search; each probe is the reference's replay() with
 * AllocatorConfig(device_capacity=C) (allocator.py:358-393), and the capacity
 * enters only through `reserved + seg > cap` (allocator.py:258-287,
 * 328-333), so the answer is a multiple of u = gcd(k_small_buffer,
 * k_large_buffer, k_round_large).  Bracket: the unbounded peak_reserved
 * runs; 0 OOMs, and with max_split_size None so does every C below the
 * unbounded peak_allocated.  Bisection returns
 * the C (multiple of u) that runs while C - u OOMs; if the allocator is not
 * monotone in C a smaller runnable capacity may exist below an OOMing one.
 *
 * Device pointers; device_capacity in cfgs is ignored.  min_capacity[t]:
 * the answer, 0 for a trace without allocations, -1 when the unbounded run
 * is malformed (see unbounded[t].status).  n_probes[t]: bisection replays of
 * trace t.  unbounded (nullable): round-0 results (peak_reserved = the
 * reference's estimate).  probe_capacity / probe_results (nullable,
 * [max_probes][n_traces]): the capacity and result of probe k of trace t.
 * Synchronises `stream` once per round (to size the next round). */
int pm_capacity_workspace_bytes(int64_t total_events, int64_t max_trace_events,
                                int32_t n_traces, size_t* out_bytes);

int pm_capacity_search(const pm_req_t* reqs, const int64_t* trace_offsets,
                       int32_t n_traces, const pm_cfg_t* cfgs,
                       const int32_t* cfg_of_trace, const int32_t* trace_order,
                       int64_t* min_capacity, int32_t* n_probes,
                       pm_result_t* unbounded, int64_t* probe_capacity,
                       pm_result_t* probe_results, int32_t max_probes,
                       void* workspace, size_t workspace_bytes,
                       int64_t total_events, int64_t max_trace_events,
                       void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PEAKMEM_B200_H */
