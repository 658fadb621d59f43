/*
 * peakmem_pipeline.h -- C ABI of the GPU analysis / link / orchestration
 * stages of the xMem (arXiv 2504.03887) estimator (csrc/pipeline.cu).
 *
 * Host arrays in, host arrays out; device memory is stream-ordered scratch.
 * Return 0 or a pm_err_t code (include/peakmem_b200.h); the message is in
 * pm_pipeline_last_error().  Timestamps are integer microseconds; INT64_MIN
 * stands for Python's None (a never-freed block).
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/peakmem):
 *   pm_sort_events -> trace.parse_trace's sort + normalize (trace.py:222-236)
 *   pm_link        -> analysis.build_operator_roots (analysis.py:185-211),
 *                     analysis.group_memory_events (analysis.py:252-294) and
 *                     linking.link (linking.py:126-132) + the backward-
 *                     retained test of orchestration.tag_gradient_blocks
 *                     (orchestration.py:122-132, linking.py:40-43), as
 *                     called by orchestration.analyze (orchestration.py:107)
 *   pm_link_roots  -> linking.link on caller-given roots and blocks
 *   pm_orchestrate -> orchestration.build_sequence's per-block rewrites,
 *                     emission and total order (orchestration.py:270-387)
 *   pm_layer_tree  -> analysis.build_layer_tree's ancestor walk, child
 *                     order and walk order (analysis.py:113-182)
 *   pm_pipeline_batch -> orchestration.analyze + orchestration.build_sequence
 *                     (orchestration.py:107-116, 237-399) for B traces in one
 *                     call, device columns in, the replay batch out
 */
#ifndef PEAKMEM_PIPELINE_H
#define PEAKMEM_PIPELINE_H

#include <stdint.h>

#include "peakmem_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* pm_pipeline_last_error(void);

int pm_sort_events(const double* ts, const double* dur, int64_t n,
                   int64_t* perm, int64_t* start, int64_t* duration,
                   void* stream);

int pm_link(int64_t n_ops, const int64_t* op_start, const int64_t* op_end,
            const int64_t* op_seq, int64_t n_inst, const int64_t* in_start,
            const int64_t* in_addr, const int64_t* in_nbytes,
            int64_t n_leaves, const int64_t* l_start, const int64_t* l_end,
            int64_t* op_root, int64_t* n_roots_out, int64_t* root_op,
            int64_t* root_start, int64_t* root_end, int64_t* root_seq_off,
            int64_t* root_seq, int64_t* root_leaf, int64_t* bwd_off,
            int64_t* bwd_root, int64_t bwd_cap, int64_t* n_bwd_out,
            int64_t* n_blocks_out, int64_t* b_inst, int64_t* b_alloc,
            int64_t* b_size, int64_t* b_free, int32_t* b_role,
            int64_t* b_prof, int64_t* b_root, void* stream);

int pm_link_roots(int64_t n_roots, const int64_t* root_start,
                  const int64_t* root_end, const int64_t* root_seq_off,
                  const int64_t* root_seq, int64_t n_leaves,
                  const int64_t* l_start, const int64_t* l_end,
                  int64_t n_blocks, const int64_t* b_alloc,
                  const int64_t* b_free, int64_t* root_leaf, int64_t* bwd_off,
                  int64_t* bwd_root, int64_t bwd_cap, int64_t* n_bwd_out,
                  int32_t* b_role, int64_t* b_prof, int64_t* b_root,
                  void* stream);

int pm_orchestrate(int64_t nb, const int64_t* b_alloc, const int64_t* b_size,
                   const int64_t* b_free, const int32_t* b_role,
                   int32_t n_spans, const int64_t* span_start,
                   const int64_t* span_end, const int64_t* span_iter,
                   int32_t n_param, const int64_t* param_sizes,
                   int32_t n_windows, const int64_t* win_start,
                   const int64_t* win_end, int32_t n_zg, const int64_t* zg,
                   int32_t clones, int64_t tpl_start, int64_t tpl_end,
                   int64_t shift, int64_t n_batch, const int64_t* batch_vts,
                   const int64_t* batch_size, const int32_t* batch_kind,
                   const int64_t* batch_it, const int64_t* batch_j,
                   int64_t req_cap, int64_t* n_req_out, int64_t* n_model_out,
                   int64_t* o_raw, int32_t* o_kind, int64_t* o_size,
                   int64_t* o_vts, int32_t* o_tag, int64_t* o_a, int64_t* o_b,
                   int32_t* o_role, pm_req_t* o_packed, int32_t* fb_role,
                   int64_t* fb_free, int32_t* fb_flags, void* stream);

/* pm_layer_tree -> analysis.build_layer_tree (analysis.py:113-182), the
 * structural part: n python_function frames in event order (python id /
 * parent id, INT64_MIN = None; is_layer = the name matches a layer prefix;
 * start).  Duplicate ids keep the first frame; each layer frame's nearest
 * layer ancestor follows the reference's parent walk (a chain that revisits
 * the walker's own id, or does not terminate, returns
 * PM_ERR_CYCLIC_PARENT).  event_id (nullable) breaks start ties; NULL =
 * input order.  Outputs over the n_layers layer frames (their
 * order = event order): node_parent (index or -1 = the synthetic root),
 * child_order + child_off (n_layers+2; slot 0 = root, slot v+1 = node v):
 * children sorted by (start, event id), and walk[0..*n_walk): the pre-order
 * walk from the root (LayerNode.walk without the root).  Layer frames that
 * are each other's nearest layer ancestors (a cycle the reference's walk
 * does not flag) are reachable from no root path and not in the walk. */
int pm_layer_tree(int64_t n, const int64_t* pid, const int64_t* par,
                  const uint8_t* is_layer, const int64_t* start,
                  const int64_t* event_id, int64_t n_layers,
                  int64_t* node_parent,
                  int64_t* child_order, int64_t* child_off, int64_t* walk,
                  int64_t* n_walk, void* stream);


/* ---- the batched, device-resident pipeline ------------------------------
 *
 * pm_pipeline_batch -> orchestration.analyze (orchestration.py:107-116) then
 * orchestration.build_sequence (orchestration.py:237-399) for n_traces
 * traces at once, as PeakMemoryEstimator.estimate calls them
 * (estimator.py:146,152).  The event columns of all traces are concatenated
 * trace-major (each trace in event order, i.e. the order parse_trace sorts
 * into) and passed as DEVICE pointers with HOST per-trace offsets; the
 * per-trace orchestration parameters (a handful of values derived from the
 * trace's markers and sidecar on the host, exactly as build_sequence
 * derives them) are HOST arrays in CSR form.  The orchestrated requests of
 * all traces are written to `reqs` (DEVICE, capacity req_cap) in the layout
 * pm_replay_batch reads: trace t is reqs[req_off[t] .. req_off[t+1]) with
 * dense per-trace handles, so the replay runs on it without a host round
 * trip.  Timestamps are integer microseconds; INT64_MIN = None. */
typedef struct {
  int32_t n_traces;
  /* host offsets [n_traces + 1] into the three event columns */
  const int64_t* fn_off;  /* python_function frames */
  const int64_t* op_off;  /* cpu_op events */
  const int64_t* in_off;  /* cpu_instant_event events */
  /* device columns */
  const int64_t* fn_pid;        /* python id (INT64_MIN = None) */
  const int64_t* fn_par;        /* parent python id (INT64_MIN = None) */
  const uint8_t* fn_is_layer;   /* name starts with a layer prefix */
  const int64_t* fn_start;
  const int64_t* fn_end;
  const int64_t* op_start;
  const int64_t* op_end;
  const int64_t* op_seq;        /* sequence number, -1 = None */
  const int64_t* in_start;
  const int64_t* in_addr;
  const int64_t* in_nbytes;
  /* host, per trace (CSR offsets [n_traces + 1]) -- see build_sequence */
  const int64_t* span_off;      /* optimizer-step markers in marker order */
  const int64_t* span_start;
  const int64_t* span_end;
  const int64_t* span_iter;
  const int64_t* param_off;     /* sidecar param sizes, sorted unique */
  const int64_t* param_sizes;
  const int64_t* win_off;       /* windows of the included iterations */
  const int64_t* win_start;
  const int64_t* win_end;
  const int64_t* zg_off;        /* zero-grad starts incl. cloned markers, sorted */
  const int64_t* zg;
  const int32_t* clones;        /* [n_traces] iterations cloned */
  const int64_t* tpl_start;     /* [n_traces] clone template window */
  const int64_t* tpl_end;
  const int64_t* shift;         /* [n_traces] template width */
  const int64_t* bat_off;       /* batch requests (vts, size, kind, it, j) */
  const int64_t* bat_vts;
  const int64_t* bat_size;
  const int32_t* bat_kind;
  const int64_t* bat_it;
  const int64_t* bat_j;
  const int32_t* skip;          /* [n_traces] nullable: nonzero = emit nothing
                                   (a trace that failed a host-side check) */
} pm_pipeline_batch_t;

/* Returns 0 or a pm_err_t (PM_ERR_WORKSPACE_TOO_SMALL: req_cap is below
 * req_off[n_traces], which is filled in; PM_ERR_ENGINE_LIMIT: a packed key
 * range exceeded).  Per trace (host outputs): req_off [n_traces + 1],
 * status (0; -1 NoGradientBlocks; PM_ERR_CYCLIC_PARENT; PM_ERR_SKIPPED),
 * n_model (model-load requests), breakdown (nullable, [n_traces x 8]:
 * ALLOC bytes by role code 0 unclassified, 1 model, 2 batch, 3 gradient,
 * 4 optimizer_state, 5 temporary, 6 retained -- estimator.py:160-164). */
/* Optional per-trace views (caller-allocated DEVICE buffers except blk_off,
 * a HOST array; pass NULL to skip) -- left on the device so a caller reads
 * them only if it needs them:
 * the ordered request columns of every trace, concatenated like `reqs`
 * (capacity req_cap): raw index within the trace, kind (0 alloc, 1 free),
 * size, virtual_ts, tag (0 model / 1 batch / 2 block / 3 clone), a, b (the
 * block-id parts: model i | batch it, j | block id | clone c, id), role;
 * every block's final role and free time after orchestration (capacity
 * fb_cap >= all traces' blocks; build_sequence mutates the analyzed blocks
 * so, orchestration.py:222-223,197) and the per-trace block offsets
 * blk_off[n_traces + 1]. */
typedef struct {
  int64_t* o_raw;
  int32_t* o_kind;
  int64_t* o_size;
  int64_t* o_vts;
  int32_t* o_tag;
  int64_t* o_a;
  int64_t* o_b;
  int32_t* o_role;
  int32_t* fb_role;
  int64_t* fb_free;
  int64_t fb_cap;
  int64_t* blk_off;
} pm_pipeline_views_t;

int pm_pipeline_batch(const pm_pipeline_batch_t* in, pm_req_t* reqs,
                      int64_t req_cap, int64_t* req_off, int32_t* status,
                      int64_t* n_model, int64_t* breakdown,
                      pm_pipeline_views_t* views, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PEAKMEM_PIPELINE_H */
