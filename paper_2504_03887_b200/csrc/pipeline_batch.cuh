// Batched, device-resident analysis -> link -> orchestration (sm_100a).
//
// Included at the end of pipeline.cu (one translation unit: the stage_*
// functions, the pmp kernels and the Arena live there).
//
// pm_pipeline_batch takes the event columns of B traces, concatenated
// trace-major with per-trace offsets, as DEVICE pointers and writes the
// orchestrated pm_req_t sequences of all B traces straight into a device
// buffer laid out for pm_replay_batch (req_off = its per-trace offsets).
// Every per-event / per-op / per-block stage runs once over the whole batch:
//
//  * isolation by rebasing, not by per-trace launches.  Every stage of the
//    reference that compares timestamps (operator nesting, leaf containment,
//    block ownership, backward-op containment) only ever relates events of
//    one trace, so each trace's times are shifted into a disjoint range
//    (trace t occupies [base_t, base_t + span_t], base_{t+1} > base_t +
//    span_t): sorted by start, traces come out trace-major, prefix maxima
//    of one trace never reach the next, and every containment test across a
//    trace boundary fails exactly as it must.  Sequence numbers and python
//    ids are rebased the same way (joins by equality stay inside a trace);
//    address recurrence (analysis.py:265-290) checks the trace id.  Block
//    times are shifted back right after the link, so orchestration works on
//    each trace's own timestamps with its own parameters;
//  * orchestration (orchestration.py:135-399) runs per block with the
//    block's trace's windows / spans / zero-grad marks / clone template,
//    emission positions come from scans over the whole batch, and the total
//    order is one (virtual_ts - vmin_t, rank, index) radix sort followed by
//    a stable sort on the trace id.
//
// pm_orchestrate and pm_layer_tree (the single-trace entry points the
// Python API's per-trace views use) are the same cores with B = 1.

namespace pmp {

// trace of element i: the last t with off[t] <= i (off: B + 1 entries)
__global__ void k_trace_of(const long long* off, int B, long long n, int* tr) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  tr[i] = (int)(upper_bound_ll(off, (long long)B + 1, i) - 1);
}

// out[i] = in[i] + delta[tr[i]], `keep` values passed through unchanged
__global__ void k_rebase(const long long* in, const int* tr,
                         const long long* delta, long long n, long long keep,
                         long long* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long v = in[i];
  out[i] = v == keep ? v : v + delta[tr[i]];
}

// sequence numbers: negative = none (kept as -1), else rebased
__global__ void k_rebase_seq(const long long* in, const int* tr,
                             const long long* delta, long long n,
                             long long* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long v = in[i];
  out[i] = v < 0 ? -1 : v + delta[tr[i]];
}

__device__ __forceinline__ void atomic_min_ll(long long* a, long long v) {
  atomicMin(a, v);
}
__device__ __forceinline__ void atomic_max_ll(long long* a, long long v) {
  atomicMax(a, v);
}

// Per-trace min / max of a column (values equal to `skip` ignored; `lo_skip`
// additionally ignores values below it): each block reduces a tile of
// contiguous elements; a tile inside one trace costs one atomic pair.
constexpr int kTile = 4096;
__global__ void k_minmax_by_trace(const long long* v, const int* tr, long long n,
                                  long long skip, long long lo_skip,
                                  long long* mn, long long* mx) {
  const long long t0 = (long long)blockIdx.x * kTile;
  if (t0 >= n) return;
  const long long t1 = t0 + kTile < n ? t0 + kTile : n;
  const int ta = tr[t0], tb = tr[t1 - 1];
  long long lo = INT64_MAX, hi = INT64_MIN;
  for (long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const long long x = v[i];
    const bool ok = x != skip && x >= lo_skip;
    if (ta == tb) {
      if (ok) {
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
      }
    } else if (ok) {
      atomic_min_ll(&mn[tr[i]], x);
      atomic_max_ll(&mx[tr[i]], x);
    }
  }
  if (ta != tb) return;
  typedef cub::BlockReduce<long long, 256> BR;
  __shared__ typename BR::TempStorage s1, s2;
  const long long blo = BR(s1).Reduce(lo, MinOp());
  const long long bhi = BR(s2).Reduce(hi, MaxOp());
  if (threadIdx.x == 0 && blo <= bhi) {
    atomic_min_ll(&mn[ta], blo);
    atomic_max_ll(&mx[ta], bhi);
  }
}

__global__ void k_fill_ll(long long* a, long long n, long long v) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

// ---- orchestration, batched (orchestration.py:200-347) ----------------------

struct OrchBatch {
  int B;
  const int* trb;           // trace of each block
  const long long* blk_off;  // [B+1] first block of each trace
  const int* skip;          // [B] nonzero: trace already failed, no requests
  const long long *span_off, *span_start, *span_end, *span_iter;
  const long long *param_off, *param_sizes;  // sorted unique per trace
  const long long *win_off, *win_start, *win_end;
  const long long *zg_off, *zg;  // sorted zero-grad starts per trace
  const int* clones;
  const long long *tpl_start, *tpl_end, *shift;
};

__global__ void k_orch_blocks_b(OrchBatch p, const long long* b_alloc,
                                const long long* b_size, const long long* b_free,
                                const int* role_in, long long nb, int* role_out,
                                long long* free0, long long* free_out,
                                int* flags) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int tr = p.trb[b];
  const long long t = b_alloc[b], sz = b_size[b];
  const bool grad = role_in[b] == R_GRAD;
  int role = role_in[b];
  long long fr = b_free[b];
  bool dropped = false;
  const long long s0 = p.span_off[tr], s1 = p.span_off[tr + 1];
  const long long* ps = p.param_sizes + p.param_off[tr];
  const long long np = p.param_off[tr + 1] - p.param_off[tr];
  for (long long k = s0; k < s1; ++k) {
    const long long s = p.span_start[k], e = p.span_end[k];
    if (!(s <= t && t < e)) continue;
    if (p.span_iter[k] == 0) {
      // extract_optimizer_state (orchestration.py:200-227)
      const long long pi = lower_bound_ll(ps, np, sz);
      const bool is_param = pi < np && ps[pi] == sz;
      if (is_param && !(fr != kNoneTs && fr < e)) {
        role = R_STATE;
        fr = kNoneTs;
      }
      if (role != R_STATE) dropped = true;
    } else {
      dropped = true;
    }
  }
  const bool seq = role != R_TEMP && !dropped;
  int f = seq ? F_SEQ : 0;
  if (seq && role != R_STATE && p.clones[tr] > 0 && p.tpl_start[tr] <= t &&
      t < p.tpl_end[tr])
    f |= F_TPL;
  free0[b] = fr;  // lifetime at clone time
  const long long* zg = p.zg + p.zg_off[tr];
  const int nzg = (int)(p.zg_off[tr + 1] - p.zg_off[tr]);
  if (grad) fr = next_zg(zg, nzg, t);  // adjust_gradient_lifetimes
  const long long w0 = p.win_off[tr], w1 = p.win_off[tr + 1];
  bool inwin = false;
  if (w1 > w0) {
    if (t < p.win_start[w0]) inwin = true;
    for (long long k = w0; k < w1 && !inwin; ++k)
      if (p.win_start[k] <= t && t < p.win_end[k]) inwin = true;
  }
  if (seq && inwin) f |= F_CHOSEN;
  if (grad && w1 > w0 && p.win_start[w0] <= t && t < p.win_end[w0]) f |= F_MODEL;
  if (p.skip[tr]) f = 0;
  role_out[b] = role;
  free_out[b] = fr;
  flags[b] = f;
}

// per-block request counts: model (1), chosen (1 or 2), clone template (2)
__global__ void k_orch_counts(const int* flags, const long long* free_out,
                              long long nb, long long* cm, long long* cc,
                              long long* ct) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) {  // trailing zero: the exclusive scans end with the totals
    cm[b] = cc[b] = ct[b] = 0;
    return;
  }
  const int f = flags[b];
  cm[b] = (f & F_MODEL) ? 1 : 0;
  cc[b] = (f & F_CHOSEN) ? (free_out[b] != kNoneTs ? 2 : 1) : 0;
  ct[b] = (f & F_TPL) ? 2 : 0;
}

// per-trace totals of the three counts: [B] x 3
__global__ void k_orch_totals(const long long* blk_off, int B,
                              const long long* xm, const long long* xc,
                              const long long* xt, long long* tot) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B) return;
  const long long a = blk_off[t], z = blk_off[t + 1];
  tot[3 * t + 0] = xm[z] - xm[a];
  tot[3 * t + 1] = xc[z] - xc[a];
  tot[3 * t + 2] = xt[z] - xt[a];
}

// raw request record (pre-order): tag 0 model / 1 batch / 2 block / 3 clone;
// tr = the trace
struct RawReqB {
  long long vts, size;
  long long a, b;  // model: i | batch: iteration, j | block: id | clone: c, id
  int kind;        // 0 alloc, 1 free, -1 absent (a clone's missing free)
  int tag;
  int role;
  int tr;
};

// per trace: [0] raw base, [1] n_model, [2] n_batch, [3] n_chosen,
// [4] n_tpl, [5] clones -- long long x 6
struct Lay {
  long long base, n_model, n_batch, n_chosen, n_tpl, clones;
};

__global__ void k_raw_absent(RawReqB* raw, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) raw[i].kind = -1;
}

__global__ void k_emit_model_b(const int* flags, const int* trb,
                               const long long* blk_off, const long long* xm,
                               const long long* b_size, long long nb,
                               const Lay* lay, RawReqB* raw) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb || !(flags[b] & F_MODEL)) return;
  const int t = trb[b];
  const Lay L = lay[t];
  const long long j = xm[b] - xm[blk_off[t]];  // model index in block order
  const long long i = L.n_model - 1 - j;       // reversed backward order
  RawReqB r;
  r.vts = i - L.n_model;
  r.size = b_size[b];
  r.a = i;
  r.b = 0;
  r.kind = 0;
  r.tag = 0;
  r.role = R_MODEL;
  r.tr = t;
  raw[L.base + i] = r;
}

__global__ void k_emit_batch_b(const long long* bat_off, int B,
                               const long long* vts, const long long* size,
                               const int* kind, const long long* it,
                               const long long* jj, long long nbat,
                               const int* skip, const Lay* lay, RawReqB* raw) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= nbat) return;
  const int t = (int)(upper_bound_ll(bat_off, (long long)B + 1, k) - 1);
  if (skip[t]) return;
  const Lay L = lay[t];
  RawReqB r;
  r.vts = vts[k];
  r.size = size[k];
  r.a = it[k];
  r.b = jj[k];
  r.kind = kind[k];
  r.tag = 1;
  r.role = R_BATCH;
  r.tr = t;
  raw[L.base + L.n_model + (k - bat_off[t])] = r;
}

__global__ void k_emit_blocks_b(const int* flags, const int* trb,
                                const long long* blk_off, const long long* xc,
                                const long long* b_alloc, const long long* b_size,
                                const long long* free_out, const int* role,
                                long long nb, const Lay* lay, RawReqB* raw) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb || !(flags[b] & F_CHOSEN)) return;
  const int t = trb[b];
  const Lay L = lay[t];
  const long long o = L.base + L.n_model + L.n_batch + (xc[b] - xc[blk_off[t]]);
  RawReqB r;
  r.vts = b_alloc[b];
  r.size = b_size[b];
  r.a = b - blk_off[t];
  r.b = 0;
  r.kind = 0;
  r.tag = 2;
  r.role = role[b];
  r.tr = t;
  raw[o] = r;
  if (free_out[b] != kNoneTs) {
    r.vts = free_out[b];
    r.kind = 1;
    raw[o + 1] = r;
  }
}

__global__ void k_emit_clones_b(OrchBatch p, const int* flags,
                                const long long* xt, const long long* b_alloc,
                                const long long* b_size, const long long* free0,
                                const int* role, long long nb, const Lay* lay,
                                RawReqB* raw) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb || !(flags[b] & F_TPL)) return;
  const int t = p.trb[b];
  const Lay L = lay[t];
  const long long base = L.base + L.n_model + L.n_batch + L.n_chosen;
  const long long pos = xt[b] - xt[p.blk_off[t]];
  const long long* zg = p.zg + p.zg_off[t];
  const int nzg = (int)(p.zg_off[t + 1] - p.zg_off[t]);
  for (int c = 1; c <= p.clones[t]; ++c) {
    const long long shift = p.shift[t] * c;
    const long long o = base + (long long)(c - 1) * L.n_tpl + pos;
    const long long ta = b_alloc[b] + shift;
    long long fr = free0[b] == kNoneTs ? kNoneTs : free0[b] + shift;
    if (role[b] == R_GRAD) fr = next_zg(zg, nzg, ta);
    RawReqB r;
    r.vts = ta;
    r.size = b_size[b];
    r.a = c;
    r.b = b - p.blk_off[t];
    r.kind = 0;
    r.tag = 3;
    r.role = role[b];
    r.tr = t;
    raw[o] = r;
    if (fr != kNoneTs) {
      r.vts = fr;
      r.kind = 1;
      raw[o + 1] = r;
    }
  }
}

__global__ void k_present(const RawReqB* raw, long long n, long long* f) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i <= n) f[i] = i < n && raw[i].kind >= 0 ? 1 : 0;
}

__global__ void k_compact_raw(const RawReqB* raw, const long long* pos,
                              long long n, RawReqB* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && raw[i].kind >= 0) out[pos[i]] = raw[i];
}

// compacted per-trace offsets: off[t] = pos[base_t] (off[B] = total)
__global__ void k_compact_off(const Lay* lay, int B, long long n_raw,
                              const long long* pos, long long* off) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > B) return;
  off[t] = pos[t < B ? lay[t].base : n_raw];
}

__global__ void k_raw_vts(const RawReqB* raw, long long n, long long* v, int* tr) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v[i] = raw[i].vts;
  tr[i] = raw[i].tr;
}

// total order key within a trace (orchestration.py:368-383): (virtual_ts,
// rank, idx), rank 0 = free of an older block, 1 = alloc, 2 = free at its
// alloc's ts.  Every free directly follows its alloc in raw order.
__global__ void k_order_keys_b(const RawReqB* raw, long long n,
                               const long long* vmin, u64* keys,
                               long long* idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const RawReqB r = raw[i];
  int rank = 1;
  if (r.kind == 1) rank = raw[i - 1].vts < r.vts ? 0 : 2;
  keys[i] = ((u64)(r.vts - vmin[r.tr]) << 2) | (u64)rank;
  idx[i] = i;
}

__global__ void k_trace_keys(const RawReqB* raw, const long long* perm,
                             long long n, u64* keys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) keys[i] = (u64)raw[perm[i]].tr;
}

// packed replay records: handle = the alloc's index within its trace
__global__ void k_pack_b(const RawReqB* raw, const long long* perm,
                         const long long* roff, long long n, pm_req_t* out,
                         long long* out_raw) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = perm[i];
  const RawReqB r = raw[k];
  const long long b0 = roff[r.tr];
  pm_req_t q;
  q.size = r.size;
  q.handle = (int32_t)((r.kind == 0 ? k : k - 1) - b0);
  q.kind_stream = r.kind == 0 ? PM_KIND_ALLOC : PM_KIND_FREE;
  out[i] = q;
  if (out_raw) out_raw[i] = k - b0;
}

// phase breakdown (estimator.py:160-164): ALLOC bytes by role, per trace.
// A CTA whose tile lies in one trace sums into 8 shared counters and adds
// them once (a single trace would otherwise serialise millions of atomics
// on seven addresses).
__global__ void k_breakdown(const RawReqB* raw, long long n,
                            unsigned long long* bd) {
  __shared__ unsigned long long acc[8];
  const long long t0 = (long long)blockIdx.x * kTile;
  if (t0 >= n) return;
  const long long t1 = t0 + kTile < n ? t0 + kTile : n;
  const int ta = raw[t0].tr, tb = raw[t1 - 1].tr;
  if (threadIdx.x < 8) acc[threadIdx.x] = 0ull;
  __syncthreads();
  for (long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const RawReqB r = raw[i];
    if (r.kind != 0) continue;
    if (ta == tb)
      atomicAdd(&acc[r.role], (unsigned long long)r.size);
    else
      atomicAdd(&bd[8 * r.tr + r.role], (unsigned long long)r.size);
  }
  __syncthreads();
  if (ta == tb && threadIdx.x < 8 && acc[threadIdx.x])
    atomicAdd(&bd[8 * ta + threadIdx.x], acc[threadIdx.x]);
}

// ordered request columns for the single-trace API
__global__ void k_unpack_ordered(const RawReqB* raw, const long long* perm,
                                 long long n, int* kind, long long* size,
                                 long long* vts, int* tag, long long* a,
                                 long long* b, int* role) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const RawReqB r = raw[perm[i]];
  kind[i] = r.kind;
  size[i] = r.size;
  vts[i] = r.vts;
  tag[i] = r.tag;
  a[i] = r.a;
  b[i] = r.b;
  role[i] = r.role;
}

// ---- layer tree helpers, batched -------------------------------------------

// non-wrapper layers in walk order (linking.py:46-47): is_wrapper = has
// children
__global__ void k_leaf_flags(const long long* walk, long long nw,
                             const long long* off, int* f) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < nw) {
    const long long v = walk[i];
    f[i] = off[v + 2] > off[v + 1] ? 0 : 1;
  }
}

__global__ void k_gather_idx2(const long long* src, const long long* i1,
                              const long long* i2, long long n, long long* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[i1[i2[i]]];
}

__global__ void k_block_trace(const long long* b_inst, const int* itr,
                              long long nb, int* trb) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b < nb) trb[b] = itr[b_inst[b]];
}

// first index of each trace in a trace-sorted column (off[B] = n)
__global__ void k_trace_offsets(const int* tr, long long n, int B, long long* off) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > B) return;
  off[t] = lower_bound_ll(tr, n, t);
}

}  // namespace pmp

namespace {

using namespace pmp;

int bits_for(long long v) {
  int b = 1;
  while (b < 63 && (1ll << b) <= v) ++b;
  return b;
}

// ---- layer tree core (a4 / f4: analysis.py:113-182) --------------------------
//
// n python_function frames in event order: python id / parent id (INT64_MIN
// = None), is_layer, start, event id (nullable: input order breaks start
// ties) and, batched, the trace of each frame (nullable).  Outputs (device,
// arena-owned): the layer frames (lay), each layer's nearest layer ancestor
// (np, -1 = the synthetic root), children in (start, event) order (ord +
// off, slot 0 = root) and the pre-order walk from the root.  A parent chain
// that revisits a python id sets cyclic[trace] (the reference raises
// CyclicParentLink, analysis.py:136-151).
struct TreeDev {
  long long nl = 0;
  long long* lay = nullptr;
  long long* np = nullptr;
  long long* ord = nullptr;
  long long* off = nullptr;
  long long* walk = nullptr;
  long long n_walk = 0;
};

int layer_tree_core(Arena& A, long long n, const long long* d_pid,
                    const long long* d_par, const unsigned char* d_isl,
                    const long long* d_start, const long long* d_eid,
                    const int* d_tr, int* d_cyclic, TreeDev* T) {
  cudaStream_t s = A.s;
  T->nl = 0;
  T->n_walk = 0;
  if (n == 0) return PM_SUCCESS;
  int* lflag = A.alloc<int>(n);
  long long* lay_index = A.alloc<long long>(n);
  PM_TRY(check_arena(A, "layer tree"));
  pmp::k_u8_to_int<<<blocks_for(n), 256, 0, s>>>(d_isl, n, lflag);
  PM_TRY(excl_sum(A, lflag, lay_index, n));
  const long long nl = read_scalar(lay_index + n - 1, s) + read_scalar((const int*)lflag + n - 1, s);
  T->nl = nl;
  if (nl == 0) return PM_SUCCESS;
  // python id -> first frame
  u64* keys = A.alloc<u64>(n);
  u64* skeys = A.alloc<u64>(n);
  long long* idx = A.alloc<long long>(n);
  long long* sidx = A.alloc<long long>(n);
  int* first = A.alloc<int>(n);
  u64* ukeys = A.alloc<u64>(n);
  long long* upos = A.alloc<long long>(n);
  long long* nsel = A.alloc<long long>(1);
  long long* parent_pos = A.alloc<long long>(n);
  T->lay = A.alloc<long long>(nl);
  T->np = A.alloc<long long>(nl);
  unsigned* pkey = A.alloc<unsigned>(nl);
  unsigned* pkey2 = A.alloc<unsigned>(nl);
  u64* skey = A.alloc<u64>(nl);
  u64* skey2 = A.alloc<u64>(nl);
  long long* ord = A.alloc<long long>(nl);
  long long* ord2 = A.alloc<long long>(nl);
  T->off = A.alloc<long long>(nl + 2);
  long long* jump[2] = {A.alloc<long long>(nl), A.alloc<long long>(nl)};
  int* depth[2] = {A.alloc<int>(nl), A.alloc<int>(nl)};
  int* sdepth = A.alloc<int>(nl);
  long long* by_depth = A.alloc<long long>(nl);
  long long* nodes = A.alloc<long long>(nl);
  int* dmax = A.alloc<int>(1);
  long long* size = A.alloc<long long>(nl);
  long long* pre = A.alloc<long long>(nl);
  T->walk = A.alloc<long long>(nl);
  long long* minus1 = A.alloc<long long>(1);
  PM_TRY(check_arena(A, "layer tree"));
  size_t tmp = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, skeys, idx, sidx, (int64_t)n, 0, 64, s);
  cub::DeviceSelect::Flagged(nullptr, t2, skeys, first, ukeys, nsel, (int64_t)n, s);
  tmp = std::max(tmp, t2);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, skey, skey2, ord, ord2, (int64_t)nl, 0, 64, s);
  tmp = std::max(tmp, t2);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, depth[0], sdepth, ord, by_depth, (int64_t)nl, 0, 32, s);
  tmp = std::max(tmp, t2);
  cub::DeviceReduce::Max(nullptr, t2, depth[0], dmax, (int64_t)nl, s);
  tmp = std::max(tmp, t2);
  void* t = A.alloc<char>(tmp);
  PM_TRY(check_arena(A, "layer tree"));

  pmp::k_pid_keys<<<blocks_for(n), 256, 0, s>>>(d_pid, n, keys, idx);
  cub::DeviceRadixSort::SortPairs(t, tmp, keys, skeys, idx, sidx, (int64_t)n, 0, 64, s);
  pmp::k_pid_first<<<blocks_for(n), 256, 0, s>>>(skeys, n, first);
  cub::DeviceSelect::Flagged(t, tmp, skeys, first, ukeys, nsel, (int64_t)n, s);
  cub::DeviceSelect::Flagged(t, tmp, sidx, first, upos, nsel, (int64_t)n, s);
  const long long nu = read_scalar(nsel, s);
  pmp::k_pid_parent<<<blocks_for(n), 256, 0, s>>>(d_par, n, ukeys, upos, nu, parent_pos);
  // layer frames and their index among layers (input is in event order)
  pmp::k_scatter_flagged<<<blocks_for(n), 256, 0, s>>>(lflag, lay_index, n, T->lay);
  pmp::k_layer_anc<<<blocks_for(nl), 256, 0, s>>>(T->lay, nl, d_pid, parent_pos, d_isl,
                                                   lay_index, n, d_tr, T->np, d_cyclic);
  // children in (start, event) order per parent: stable sort by start, then
  // stable sort by parent slot (nodes are in event order to begin with)
  pmp::k_gather_u64<<<blocks_for(nl), 256, 0, s>>>(d_start, T->lay, nl,
                                                    0x8000000000000000ull, 0, skey);
  pmp::k_iota<<<blocks_for(nl), 256, 0, s>>>(ord, nl);
  if (d_eid) {
    // ties by event id rather than input order: sort by it first (LSD)
    u64* ekey = A.alloc<u64>(nl);
    u64* ekey2 = A.alloc<u64>(nl);
    long long* eord = A.alloc<long long>(nl);
    PM_TRY(check_arena(A, "layer tree"));
    pmp::k_gather_u64<<<blocks_for(nl), 256, 0, s>>>(d_eid, T->lay, nl,
                                                      0x8000000000000000ull, 0, ekey);
    cub::DeviceRadixSort::SortPairs(t, tmp, ekey, ekey2, ord, eord, (int64_t)nl, 0, 64, s);
    pmp::k_gather_u64<<<blocks_for(nl), 256, 0, s>>>(d_start, T->lay, nl, 0, 0, skey2);
    pmp::k_gather_u64_idx<<<blocks_for(nl), 256, 0, s>>>(skey2, eord, nl,
                                                          0x8000000000000000ull, skey);
    cudaMemcpyAsync(ord, eord, nl * sizeof(long long), cudaMemcpyDeviceToDevice, s);
  }
  cub::DeviceRadixSort::SortPairs(t, tmp, skey, skey2, ord, ord2, (int64_t)nl, 0, 64, s);
  pmp::k_gather_parent_key<<<blocks_for(nl), 256, 0, s>>>(T->np, ord2, nl, pkey);
  cub::DeviceRadixSort::SortPairs(t, tmp, pkey, pkey2, ord2, ord, (int64_t)nl, 0, 32, s);
  T->ord = ord;
  pmp::k_child_off<<<blocks_for(nl + 2), 256, 0, s>>>(pkey2, nl, T->off);
  // depth (pointer jumping) and nodes grouped by depth
  pmp::k_depth_init<<<blocks_for(nl), 256, 0, s>>>(T->np, nl, jump[0], depth[0]);
  int cur = 0;
  for (long long span = 1; span < 2 * nl; span *= 2) {
    pmp::k_depth_step<<<blocks_for(nl), 256, 0, s>>>(jump[cur], depth[cur], nl,
                                                     jump[cur ^ 1], depth[cur ^ 1]);
    cur ^= 1;
  }
  pmp::k_depth_final<<<blocks_for(nl), 256, 0, s>>>(jump[cur], nl, depth[cur]);
  pmp::k_iota<<<blocks_for(nl), 256, 0, s>>>(nodes, nl);
  cub::DeviceRadixSort::SortPairs(t, tmp, depth[cur], sdepth, nodes, by_depth, (int64_t)nl, 0, 32, s);
  cub::DeviceReduce::Max(t, tmp, depth[cur], dmax, (int64_t)nl, s);
  const int maxd = read_scalar(dmax, s);
  if (maxd < 0) return PM_SUCCESS;  // no frame reaches the root: empty walk
  long long* lvl = A.alloc<long long>(maxd + 2);
  PM_TRY(check_arena(A, "layer tree"));
  pmp::k_level_off<<<blocks_for(maxd + 2), 256, 0, s>>>(sdepth, nl, maxd, lvl);
  std::vector<long long> h_lvl(maxd + 2);
  PM_TRY(download(h_lvl.data(), lvl, maxd + 2, s));
  PM_TRY(sync_check(s, "layer tree: levels"));
  // subtree sizes bottom-up, pre-order positions top-down; per level the
  // nodes with more than kBigNode children go to the CTA-per-node kernels
  // (big[d]: count, then nodes -- a level holds at most nl / kBigNode of them)
  const long long bigcap = 1 + nl / pmp::kBigNode + 1;
  long long* big = A.alloc<long long>((size_t)(maxd + 1) * bigcap);
  PM_TRY(check_arena(A, "layer tree big nodes"));
  cudaMemsetAsync(big, 0, sizeof(long long) * (size_t)(maxd + 1) * bigcap, s);
  const unsigned big_grid = 148;
  for (int d = maxd; d >= 0; --d) {
    const long long a = h_lvl[d], b = h_lvl[d + 1];
    if (b > a) {
      long long* bd = big + (size_t)d * bigcap;
      pmp::k_subtree_level<<<blocks_for(32 * (b - a)), 256, 0, s>>>(by_depth + a, b - a,
                                                              ord, T->off, size, bd);
      pmp::k_subtree_big<<<big_grid, pmp::kBigThreads, 0, s>>>(bd, ord, T->off, size);
    }
  }
  (void)minus1;
  pmp::k_preorder_big<<<1, pmp::kBigThreads, 0, s>>>(nullptr, ord, T->off, size, pre);
  for (int d = 0; d < maxd; ++d) {
    const long long a = h_lvl[d], b = h_lvl[d + 1];
    if (b > a) {
      pmp::k_preorder_level<<<blocks_for(32 * (b - a)), 256, 0, s>>>(by_depth + a, b - a,
                                                               ord, T->off, size, pre);
      pmp::k_preorder_big<<<big_grid, pmp::kBigThreads, 0, s>>>(big + (size_t)d * bigcap, ord,
                                                               T->off, size, pre);
    }
  }
  // reachable nodes: depth >= 0, i.e. by_depth[h_lvl[0] ..]
  const long long r0 = h_lvl[0], nr = h_lvl[maxd + 1] - h_lvl[0];
  pmp::k_scatter_walk<<<blocks_for(nr), 256, 0, s>>>(by_depth + r0, nr, pre, T->walk);
  T->n_walk = nr;
  return PM_SUCCESS;
}

// ---- orchestration core ------------------------------------------------------
//
// Inputs (device): nb blocks trace-major (alloc, size, free, role: 3 marks
// tag_gradient_blocks' gradients), their traces and the per-trace
// parameters (OrchBatch); the batch requests (CSR by trace) and their host
// offsets; per-trace `skip`.  Outputs: per-block role / free / flags, the
// ordered sequence (raw records + permutation), packed pm_req_t, per-trace
// request offsets (host), n_model (host), status (host: 0, -1
// NoGradientBlocks, PM_ERR_INVALID_ARGUMENT timestamp range), breakdown.
struct OrchIn {
  OrchBatch p;
  long long nb = 0;
  const long long *b_alloc, *b_size, *b_free;
  const int* b_role;
  const long long* h_blk_off;  // host [B+1]
  const int* h_skip;           // host [B]
  const long long* bat_off;    // device [B+1]
  const long long* h_bat_off;  // host [B+1]
  const long long *bat_vts, *bat_size, *bat_it, *bat_j;
  const int* bat_kind;
};

struct OrchOut {
  int* role = nullptr;
  long long* free0 = nullptr;
  long long* free_out = nullptr;
  int* flags = nullptr;
  RawReqB* raw = nullptr;  // compacted, raw order
  long long* perm = nullptr;
  long long n = 0;
  long long* d_roff = nullptr;      // device [B+1]
  std::vector<long long> roff;      // host [B+1]
  std::vector<long long> n_model;   // host [B]
  std::vector<int> status;          // host [B]
  unsigned long long* bd = nullptr;  // device [B x 8]
};

int orch_core(Arena& A, const OrchIn& in, pm_req_t* packed, long long req_cap,
              long long* out_raw, OrchOut* O) {
  cudaStream_t s = A.s;
  const int B = in.p.B;
  const long long nb = in.nb;
  O->role = A.alloc<int>(nb);
  O->free0 = A.alloc<long long>(nb);
  O->free_out = A.alloc<long long>(nb);
  O->flags = A.alloc<int>(nb);
  long long* cm = A.alloc<long long>(nb + 1);
  long long* cc = A.alloc<long long>(nb + 1);
  long long* ct = A.alloc<long long>(nb + 1);
  long long* xm = A.alloc<long long>(nb + 1);
  long long* xc = A.alloc<long long>(nb + 1);
  long long* xt = A.alloc<long long>(nb + 1);
  long long* tot = A.alloc<long long>(3 * (size_t)B);
  Lay* lay = A.alloc<Lay>(B);
  O->d_roff = A.alloc<long long>(B + 1);
  O->bd = A.alloc<unsigned long long>(8 * (size_t)B);
  PM_TRY(check_arena(A, "orchestrate"));
  if (nb > 0)
    k_orch_blocks_b<<<blocks_for(nb), 256, 0, s>>>(in.p, in.b_alloc, in.b_size, in.b_free,
                                                   in.b_role, nb, O->role, O->free0,
                                                   O->free_out, O->flags);
  k_orch_counts<<<blocks_for(nb + 1), 256, 0, s>>>(O->flags, O->free_out, nb, cm, cc, ct);
  PM_TRY(excl_sum(A, cm, xm, nb + 1));
  PM_TRY(excl_sum(A, cc, xc, nb + 1));
  PM_TRY(excl_sum(A, ct, xt, nb + 1));
  k_orch_totals<<<blocks_for(B), 256, 0, s>>>(in.p.blk_off, B, xm, xc, xt, tot);
  std::vector<long long> h_tot(3 * (size_t)B);
  std::vector<int> h_clones(B);
  PM_TRY(download(h_tot.data(), tot, 3 * (size_t)B, s));
  PM_TRY(download(h_clones.data(), in.p.clones, B, s));
  PM_TRY(sync_check(s, "orchestrate counts"));
  // raw layout per trace: model | batch | chosen | clone copies
  std::vector<Lay> h_lay(B);
  O->n_model.assign(B, 0);
  O->status.assign(B, 0);
  long long n_raw = 0;
  std::vector<int> h_skip2(B);
  for (int t = 0; t < B; ++t) {
    Lay L{};
    L.base = n_raw;
    if (!in.h_skip[t]) {
      O->n_model[t] = h_tot[3 * t];
      if (h_tot[3 * t] == 0) {
        O->status[t] = -1;  // NoGradientBlocks (orchestration.py:152-153)
      } else {
        L.n_model = h_tot[3 * t];
        L.n_batch = in.h_bat_off[t + 1] - in.h_bat_off[t];
        L.n_chosen = h_tot[3 * t + 1];
        L.n_tpl = h_tot[3 * t + 2];
        L.clones = h_clones[t];
      }
    }
    // a failed or skipped trace emits nothing
    h_skip2[t] = in.h_skip[t] || O->status[t] != 0;
    h_lay[t] = L;
    n_raw += L.n_model + L.n_batch + L.n_chosen + L.clones * L.n_tpl;
  }
  int* skip2 = A.upload(h_skip2.data(), B);
  RawReqB* raw = A.alloc<RawReqB>(n_raw);
  long long* pos = A.alloc<long long>(n_raw + 1);
  long long* fl = A.alloc<long long>(n_raw + 1);
  PM_TRY(check_arena(A, "orchestrate raw"));
  cudaMemcpyAsync(lay, h_lay.data(), sizeof(Lay) * B, cudaMemcpyHostToDevice, s);
  k_raw_absent<<<blocks_for(n_raw), 256, 0, s>>>(raw, n_raw);
  OrchBatch p2 = in.p;
  p2.skip = skip2;
  if (nb > 0) {
    // flags of skipped traces' blocks: no model / chosen / template requests
    k_orch_blocks_b<<<blocks_for(nb), 256, 0, s>>>(p2, in.b_alloc, in.b_size, in.b_free,
                                                   in.b_role, nb, O->role, O->free0,
                                                   O->free_out, O->flags);
    k_emit_model_b<<<blocks_for(nb), 256, 0, s>>>(O->flags, in.p.trb, in.p.blk_off, xm,
                                                  in.b_size, nb, lay, raw);
    k_emit_blocks_b<<<blocks_for(nb), 256, 0, s>>>(O->flags, in.p.trb, in.p.blk_off, xc,
                                                   in.b_alloc, in.b_size, O->free_out,
                                                   O->role, nb, lay, raw);
    k_emit_clones_b<<<blocks_for(nb), 256, 0, s>>>(p2, O->flags, xt, in.b_alloc, in.b_size,
                                                   O->free0, O->role, nb, lay, raw);
  }
  const long long nbat = in.h_bat_off[B];
  if (nbat > 0)
    k_emit_batch_b<<<blocks_for(nbat), 256, 0, s>>>(in.bat_off, B, in.bat_vts, in.bat_size,
                                                    in.bat_kind, in.bat_it, in.bat_j, nbat,
                                                    skip2, lay, raw);
  // compact the absent clone frees out (raw order kept)
  k_present<<<blocks_for(n_raw + 1), 256, 0, s>>>(raw, n_raw, fl);
  PM_TRY(excl_sum(A, fl, pos, n_raw + 1));
  k_compact_off<<<blocks_for(B + 1), 256, 0, s>>>(lay, B, n_raw, pos, O->d_roff);
  O->roff.assign(B + 1, 0);
  PM_TRY(download(O->roff.data(), O->d_roff, B + 1, s));
  PM_TRY(sync_check(s, "orchestrate emit"));
  const long long n = O->roff[B];
  O->n = n;
  if (n > req_cap) return perr(PM_ERR_WORKSPACE_TOO_SMALL, "orchestrate: req_cap");
  O->raw = A.alloc<RawReqB>(n);
  O->perm = A.alloc<long long>(n);
  long long* v = A.alloc<long long>(n);
  int* vtr = A.alloc<int>(n);
  long long* vmin = A.alloc<long long>(B);
  long long* vmax = A.alloc<long long>(B);
  u64* keys = A.alloc<u64>(n);
  PM_TRY(check_arena(A, "orchestrate order"));
  k_compact_raw<<<blocks_for(n_raw), 256, 0, s>>>(raw, pos, n_raw, O->raw);
  cudaMemsetAsync(O->bd, 0, sizeof(unsigned long long) * 8 * B, s);
  if (n > 0) {
    // total order: per-trace (vts - vmin, rank, index), then stable by trace
    k_fill_ll<<<blocks_for(B), 256, 0, s>>>(vmin, B, INT64_MAX);
    k_fill_ll<<<blocks_for(B), 256, 0, s>>>(vmax, B, INT64_MIN);
    k_raw_vts<<<blocks_for(n), 256, 0, s>>>(O->raw, n, v, vtr);
    k_minmax_by_trace<<<(unsigned)((n + kTile - 1) / kTile), 256, 0, s>>>(
        v, vtr, n, INT64_MIN + 1, INT64_MIN, vmin, vmax);
    std::vector<long long> h_min(B), h_max(B);
    PM_TRY(download(h_min.data(), vmin, B, s));
    PM_TRY(download(h_max.data(), vmax, B, s));
    PM_TRY(sync_check(s, "orchestrate range"));
    for (int t = 0; t < B; ++t)
      if (h_min[t] <= h_max[t] && (u64)(h_max[t] - h_min[t]) >= (1ull << 61))
        return perr(PM_ERR_INVALID_ARGUMENT, "orchestrate: timestamp range too wide");
    k_order_keys_b<<<blocks_for(n), 256, 0, s>>>(O->raw, n, vmin, keys, O->perm);
    PM_TRY(sort_pairs(A, keys, O->perm, n));
    if (B > 1) {
      k_trace_keys<<<blocks_for(n), 256, 0, s>>>(O->raw, O->perm, n, keys);
      PM_TRY(sort_pairs(A, keys, O->perm, n, bits_for(B)));
    }
    k_pack_b<<<blocks_for(n), 256, 0, s>>>(O->raw, O->perm, O->d_roff, n, packed, out_raw);
    k_breakdown<<<(unsigned)((n + kTile - 1) / kTile), 256, 0, s>>>(O->raw, n, O->bd);
  }
  return PM_SUCCESS;
}

// per-trace parameter CSR built from host arrays (upload)
struct HostParams {
  std::vector<long long> span_off, param_off, win_off, zg_off, bat_off;
};

}  // namespace

extern "C" {

// a13-a19 (orchestration.py:237-399) after link, one trace: the batched
// core with B = 1.  Inputs (host):
//   blocks (block-id order): alloc, size, free (INT64_MIN = None), role
//     (3 marks the blocks tag_gradient_blocks tagged);
//   spans: optimizer-step markers in marker order (start, end, iteration);
//   param_sizes sorted unique; windows (start, end) of the included
//   iterations; zero-grad starts sorted (original + cloned markers);
//   clones, template window, shift (template width);
//   batch requests already built on the host (tiny): n_batch records of
//   (vts, size, kind, iteration, j).
// Outputs (host, capacity req_cap >= n_model + n_batch + 2 * blocks *
// (1 + clones)): the ordered sequence -- raw index, kind, size, vts, tag
// (0 model / 1 batch / 2 block / 3 clone), a, b, role -- the packed replay
// records, per-block final role / free / flags, n_model.  Status -1 in
// *n_req_out means NoGradientBlocks.
int pm_orchestrate(int64_t nb, const int64_t* b_alloc, const int64_t* b_size,
                   const int64_t* b_free, const int32_t* b_role, int32_t n_spans,
                   const int64_t* span_start, const int64_t* span_end,
                   const int64_t* span_iter, int32_t n_param,
                   const int64_t* param_sizes, int32_t n_windows,
                   const int64_t* win_start, const int64_t* win_end,
                   int32_t n_zg, const int64_t* zg, int32_t clones,
                   int64_t tpl_start, int64_t tpl_end, int64_t shift,
                   int64_t n_batch, const int64_t* batch_vts,
                   const int64_t* batch_size, const int32_t* batch_kind,
                   const int64_t* batch_it, const int64_t* batch_j,
                   int64_t req_cap, int64_t* n_req_out, int64_t* n_model_out,
                   int64_t* o_raw, int32_t* o_kind, int64_t* o_size,
                   int64_t* o_vts, int32_t* o_tag, int64_t* o_a, int64_t* o_b,
                   int32_t* o_role, pm_req_t* o_packed, int32_t* fb_role,
                   int64_t* fb_free, int32_t* fb_flags, void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  Arena A(s);
  OrchIn in;
  in.p.B = 1;
  in.nb = nb;
  const long long h_blk_off[2] = {0, nb};
  const long long h_sp[2] = {0, n_spans}, h_pa[2] = {0, n_param},
                  h_wi[2] = {0, n_windows}, h_zg[2] = {0, n_zg}, h_ba[2] = {0, n_batch};
  const int zero = 0;
  in.h_blk_off = h_blk_off;
  in.h_skip = &zero;
  in.h_bat_off = h_ba;
  int* trb0 = A.alloc<int>(nb);
  in.p.trb = trb0;
  in.p.blk_off = A.upload(h_blk_off, 2);
  in.p.skip = A.upload(&zero, 1);
  in.p.span_off = A.upload(h_sp, 2);
  in.p.span_start = A.upload((const long long*)span_start, n_spans);
  in.p.span_end = A.upload((const long long*)span_end, n_spans);
  in.p.span_iter = A.upload((const long long*)span_iter, n_spans);
  in.p.param_off = A.upload(h_pa, 2);
  in.p.param_sizes = A.upload((const long long*)param_sizes, n_param);
  in.p.win_off = A.upload(h_wi, 2);
  in.p.win_start = A.upload((const long long*)win_start, n_windows);
  in.p.win_end = A.upload((const long long*)win_end, n_windows);
  in.p.zg_off = A.upload(h_zg, 2);
  in.p.zg = A.upload((const long long*)zg, n_zg);
  const int h_cl = clones;
  const long long h_ts = tpl_start, h_te = tpl_end, h_sh = shift;
  in.p.clones = A.upload(&h_cl, 1);
  in.p.tpl_start = A.upload(&h_ts, 1);
  in.p.tpl_end = A.upload(&h_te, 1);
  in.p.shift = A.upload(&h_sh, 1);
  in.b_alloc = A.upload((const long long*)b_alloc, nb);
  in.b_size = A.upload((const long long*)b_size, nb);
  in.b_free = A.upload((const long long*)b_free, nb);
  in.b_role = A.upload((const int*)b_role, nb);
  in.bat_off = A.upload(h_ba, 2);
  in.bat_vts = A.upload((const long long*)batch_vts, n_batch);
  in.bat_size = A.upload((const long long*)batch_size, n_batch);
  in.bat_kind = A.upload((const int*)batch_kind, n_batch);
  in.bat_it = A.upload((const long long*)batch_it, n_batch);
  in.bat_j = A.upload((const long long*)batch_j, n_batch);
  pm_req_t* d_packed = A.alloc<pm_req_t>(req_cap);
  long long* d_oraw = A.alloc<long long>(req_cap);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "pm_orchestrate: alloc");
  if (nb > 0) cudaMemsetAsync(trb0, 0, sizeof(int) * nb, s);
  OrchOut O;
  int rc = orch_core(A, in, d_packed, req_cap, d_oraw, &O);
  if (rc) return rc;
  rc = download(fb_role, (const int32_t*)O.role, nb, s);
  if (!rc) rc = download(fb_free, (const int64_t*)O.free_out, nb, s);
  if (!rc) rc = download(fb_flags, (const int32_t*)O.flags, nb, s);
  if (rc) return rc;
  *n_model_out = O.n_model[0];
  if (O.status[0] != 0) {
    *n_req_out = -1;  // NoGradientBlocks
    return sync_check(s, "pm_orchestrate");
  }
  const long long n = O.n;
  int32_t* d_kind = A.alloc<int32_t>(n);
  long long* d_size = A.alloc<long long>(n);
  long long* d_vts = A.alloc<long long>(n);
  int32_t* d_tag = A.alloc<int32_t>(n);
  long long* d_a = A.alloc<long long>(n);
  long long* d_b = A.alloc<long long>(n);
  int32_t* d_role = A.alloc<int32_t>(n);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "pm_orchestrate: alloc");
  if (n > 0)
    k_unpack_ordered<<<blocks_for(n), 256, 0, s>>>(O.raw, O.perm, n, d_kind, d_size, d_vts,
                                                   d_tag, d_a, d_b, d_role);
  rc = download(o_raw, (const int64_t*)d_oraw, n, s);
  if (!rc) rc = download(o_packed, (const pm_req_t*)d_packed, n, s);
  if (!rc) rc = download(o_kind, d_kind, n, s);
  if (!rc) rc = download(o_size, (const int64_t*)d_size, n, s);
  if (!rc) rc = download(o_vts, (const int64_t*)d_vts, n, s);
  if (!rc) rc = download(o_tag, d_tag, n, s);
  if (!rc) rc = download(o_a, (const int64_t*)d_a, n, s);
  if (!rc) rc = download(o_b, (const int64_t*)d_b, n, s);
  if (!rc) rc = download(o_role, d_role, n, s);
  if (rc) return rc;
  rc = sync_check(s, "pm_orchestrate");
  if (rc) return rc;
  *n_req_out = n;
  return PM_SUCCESS;
}

// a4 / f4: the layer tree of one trace (host arrays; see the header)
int pm_layer_tree(int64_t n, const int64_t* pid, const int64_t* par,
                  const uint8_t* is_layer, const int64_t* start,
                  const int64_t* event_id, int64_t n_layers,
                  int64_t* node_parent,
                  int64_t* child_order, int64_t* child_off, int64_t* walk,
                  int64_t* n_walk, void* stream_) {
  if (n < 0 || n_layers < 0 || n_layers > n ||
      (n > 0 && (!pid || !par || !is_layer || !start)) ||
      (n_layers > 0 && (!node_parent || !child_order || !child_off || !walk)))
    return perr(PM_ERR_INVALID_ARGUMENT, "pm_layer_tree: bad arguments");
  if (child_off) {
    child_off[0] = 0;
    if (n_layers == 0) child_off[1] = 0;
  }
  if (n_walk) *n_walk = 0;
  if (n_layers == 0) return PM_SUCCESS;
  cudaStream_t s = (cudaStream_t)stream_;
  Arena A(s);
  const long long* d_pid = (const long long*)A.upload(pid, n);
  const long long* d_par = (const long long*)A.upload(par, n);
  const unsigned char* d_isl = A.upload(is_layer, n);
  const long long* d_start = (const long long*)A.upload(start, n);
  const long long* d_eid = event_id ? (const long long*)A.upload(event_id, n) : nullptr;
  int* cyclic = A.alloc<int>(1);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "pm_layer_tree: alloc");
  cudaMemsetAsync(cyclic, 0, sizeof(int), s);
  TreeDev T;
  int rc = layer_tree_core(A, n, d_pid, d_par, d_isl, d_start, d_eid, nullptr, cyclic, &T);
  if (rc) return rc;
  if (T.nl != n_layers)
    return perr(PM_ERR_INVALID_ARGUMENT, "pm_layer_tree: n_layers disagrees with is_layer");
  int h_cyc = 0;
  rc = download(&h_cyc, cyclic, 1, s);
  if (!rc) rc = sync_check(s, "pm_layer_tree");
  if (rc) return rc;
  if (h_cyc) return perr(PM_ERR_CYCLIC_PARENT, "parent chain revisits a python id");
  rc = download(node_parent, (const int64_t*)T.np, T.nl, s);
  if (!rc) rc = download(child_order, (const int64_t*)T.ord, T.nl, s);
  if (!rc) rc = download(child_off, (const int64_t*)T.off, T.nl + 2, s);
  if (!rc) rc = download(walk, (const int64_t*)T.walk, T.n_walk, s);
  if (rc) return rc;
  if (n_walk) *n_walk = T.n_walk;
  return sync_check(s, "pm_layer_tree");
}

// The batched pipeline: see peakmem_pipeline.h.
int pm_pipeline_batch(const pm_pipeline_batch_t* in, pm_req_t* reqs,
                      int64_t req_cap, int64_t* req_off, int32_t* status,
                      int64_t* n_model, int64_t* breakdown,
                      pm_pipeline_views_t* views, void* stream_) {
  if (!in || in->n_traces < 1 || !in->fn_off || !in->op_off || !in->in_off ||
      !in->span_off || !in->param_off || !in->win_off || !in->zg_off ||
      !in->bat_off || !in->clones || !in->tpl_start || !in->tpl_end ||
      !in->shift || !req_off || !status || !n_model)
    return perr(PM_ERR_INVALID_ARGUMENT, "pm_pipeline_batch: bad arguments");
  cudaStream_t s = (cudaStream_t)stream_;
  const int B = in->n_traces;
  const long long nf = in->fn_off[B], no = in->op_off[B], ni = in->in_off[B];
  for (int t = 0; t < B; ++t)
    if (in->fn_off[t + 1] < in->fn_off[t] || in->op_off[t + 1] < in->op_off[t] ||
        in->in_off[t + 1] < in->in_off[t] || in->bat_off[t + 1] < in->bat_off[t])
      return perr(PM_ERR_INVALID_ARGUMENT, "pm_pipeline_batch: offsets not monotone");
  if ((nf && (!in->fn_pid || !in->fn_par || !in->fn_is_layer || !in->fn_start ||
              !in->fn_end)) ||
      (no && (!in->op_start || !in->op_end || !in->op_seq)) ||
      (ni && (!in->in_start || !in->in_addr || !in->in_nbytes)))
    return perr(PM_ERR_INVALID_ARGUMENT, "pm_pipeline_batch: missing columns");
  Arena A(s);
  long long* d_foff = A.upload((const long long*)in->fn_off, B + 1);
  long long* d_ooff = A.upload((const long long*)in->op_off, B + 1);
  long long* d_ioff = A.upload((const long long*)in->in_off, B + 1);
  int* trf = A.alloc<int>(nf);
  int* tro = A.alloc<int>(no);
  int* tri = A.alloc<int>(ni);
  // per-trace min / max: [0] time, [1] seq, [2] python ids
  long long* mn = A.alloc<long long>(3 * (size_t)B);
  long long* mx = A.alloc<long long>(3 * (size_t)B);
  PM_TRY(check_arena(A, "pm_pipeline_batch"));
  if (nf) k_trace_of<<<blocks_for(nf), 256, 0, s>>>(d_foff, B, nf, trf);
  if (no) k_trace_of<<<blocks_for(no), 256, 0, s>>>(d_ooff, B, no, tro);
  if (ni) k_trace_of<<<blocks_for(ni), 256, 0, s>>>(d_ioff, B, ni, tri);
  k_fill_ll<<<blocks_for(3 * B), 256, 0, s>>>(mn, 3 * B, INT64_MAX);
  k_fill_ll<<<blocks_for(3 * B), 256, 0, s>>>(mx, 3 * B, INT64_MIN);
  auto mm = [&](const int64_t* col, const int* tr, long long n, long long skip,
                long long lo_skip, int which) {
    if (n > 0)
      k_minmax_by_trace<<<(unsigned)((n + kTile - 1) / kTile), 256, 0, s>>>(
          (const long long*)col, tr, n, skip, lo_skip, mn + (size_t)which * B,
          mx + (size_t)which * B);
  };
  // INT64_MIN never occurs as a timestamp or a non-None id
  mm(in->fn_start, trf, nf, INT64_MIN, INT64_MIN, 0);
  mm(in->fn_end, trf, nf, INT64_MIN, INT64_MIN, 0);
  mm(in->op_start, tro, no, INT64_MIN, INT64_MIN, 0);
  mm(in->op_end, tro, no, INT64_MIN, INT64_MIN, 0);
  mm(in->in_start, tri, ni, INT64_MIN, INT64_MIN, 0);
  mm(in->op_seq, tro, no, INT64_MIN, 0, 1);
  mm(in->fn_pid, trf, nf, INT64_MIN, INT64_MIN, 2);
  mm(in->fn_par, trf, nf, INT64_MIN, INT64_MIN, 2);
  std::vector<long long> h_mn(3 * (size_t)B), h_mx(3 * (size_t)B);
  PM_TRY(download(h_mn.data(), mn, 3 * (size_t)B, s));
  PM_TRY(download(h_mx.data(), mx, 3 * (size_t)B, s));
  PM_TRY(sync_check(s, "pm_pipeline_batch ranges"));
  // disjoint per-trace ranges: time (gap 2), seq (gap 1), python ids (gap 1)
  std::vector<long long> delta(3 * (size_t)B, 0);
  const long long lim[3] = {1ll << 61, 1ll << 31, 1ll << 61};
  for (int w = 0; w < 3; ++w) {
    unsigned long long base = w == 2 ? 1 : 0;  // ids stay clear of None
    for (int t = 0; t < B; ++t) {
      const long long lo = h_mn[(size_t)w * B + t], hi = h_mx[(size_t)w * B + t];
      if (lo > hi) continue;  // nothing of this kind in the trace
      const unsigned long long span = (unsigned long long)(hi - lo);
      if (span >= (unsigned long long)lim[w] || base + span >= (unsigned long long)lim[w])
        return perr(w == 1 ? PM_ERR_ENGINE_LIMIT : PM_ERR_INVALID_ARGUMENT,
                    w == 1 ? "pm_pipeline_batch: sequence numbers of the batch span >= 2^31"
                           : "pm_pipeline_batch: timestamps / python ids of the batch span too wide");
      delta[(size_t)w * B + t] = (long long)base - lo;
      base += span + (w == 0 ? 2 : 1);
    }
  }
  long long* d_delta = A.upload(delta.data(), 3 * (size_t)B);
  long long* fs = A.alloc<long long>(nf);
  long long* fe = A.alloc<long long>(nf);
  long long* fpid = A.alloc<long long>(nf);
  long long* fpar = A.alloc<long long>(nf);
  long long* os = A.alloc<long long>(no);
  long long* oe = A.alloc<long long>(no);
  long long* oseq = A.alloc<long long>(no);
  long long* is = A.alloc<long long>(ni);
  int* cyclic = A.alloc<int>(B);
  PM_TRY(check_arena(A, "pm_pipeline_batch"));
  cudaMemsetAsync(cyclic, 0, sizeof(int) * B, s);
  const long long* dt = d_delta;
  if (nf) {
    k_rebase<<<blocks_for(nf), 256, 0, s>>>((const long long*)in->fn_start, trf, dt, nf,
                                            INT64_MIN, fs);
    k_rebase<<<blocks_for(nf), 256, 0, s>>>((const long long*)in->fn_end, trf, dt, nf,
                                            INT64_MIN, fe);
    k_rebase<<<blocks_for(nf), 256, 0, s>>>((const long long*)in->fn_pid, trf, dt + 2 * B,
                                            nf, INT64_MIN, fpid);
    k_rebase<<<blocks_for(nf), 256, 0, s>>>((const long long*)in->fn_par, trf, dt + 2 * B,
                                            nf, INT64_MIN, fpar);
  }
  if (no) {
    k_rebase<<<blocks_for(no), 256, 0, s>>>((const long long*)in->op_start, tro, dt, no,
                                            INT64_MIN, os);
    k_rebase<<<blocks_for(no), 256, 0, s>>>((const long long*)in->op_end, tro, dt, no,
                                            INT64_MIN, oe);
    k_rebase_seq<<<blocks_for(no), 256, 0, s>>>((const long long*)in->op_seq, tro, dt + B,
                                                no, oseq);
  }
  if (ni)
    k_rebase<<<blocks_for(ni), 256, 0, s>>>((const long long*)in->in_start, tri, dt, ni,
                                            INT64_MIN, is);
  // a4: one layer forest over the batch (the traces' top-level layers all
  // hang off the synthetic root, in trace order)
  TreeDev T;
  PM_TRY(layer_tree_core(A, nf, fpid, fpar, in->fn_is_layer, fs, nullptr, trf, cyclic, &T));
  // leaves: non-wrapper layers in walk order (trace-major)
  long long nleaf = 0;
  long long* l_start = nullptr;
  long long* l_end = nullptr;
  if (T.n_walk > 0) {
    int* lf = A.alloc<int>(T.n_walk);
    long long* leaves = A.alloc<long long>(T.n_walk);
    long long* nsel = A.alloc<long long>(1);
    l_start = A.alloc<long long>(T.n_walk);
    l_end = A.alloc<long long>(T.n_walk);
    PM_TRY(check_arena(A, "pm_pipeline_batch leaves"));
    k_leaf_flags<<<blocks_for(T.n_walk), 256, 0, s>>>(T.walk, T.n_walk, T.off, lf);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, T.walk, lf, leaves, nsel, (int64_t)T.n_walk, s);
    void* t = A.alloc<char>(tmp);
    PM_TRY(check_arena(A, "pm_pipeline_batch leaves"));
    cub::DeviceSelect::Flagged(t, tmp, T.walk, lf, leaves, nsel, (int64_t)T.n_walk, s);
    nleaf = read_scalar(nsel, s);
    if (nleaf >= (1ll << 24))  // owner-list keys hold the leaf in 24 bits
      return perr(PM_ERR_ENGINE_LIMIT, "pm_pipeline_batch: >= 2^24 leaf layers in one batch");
    if (nleaf > 0) {
      k_gather_idx2<<<blocks_for(nleaf), 256, 0, s>>>(fs, T.lay, leaves, nleaf, l_start);
      k_gather_idx2<<<blocks_for(nleaf), 256, 0, s>>>(fe, T.lay, leaves, nleaf, l_end);
    }
  }
  // a5 / a7 / a8-a11 over the whole batch
  RootsDev R;
  BlocksDev Bk;
  JoinDev J;
  long long* d_op_root = A.alloc<long long>(no);
  long long* d_root_op = A.alloc<long long>(no);
  PM_TRY(check_arena(A, "pm_pipeline_batch link"));
  PM_TRY(stage_roots(A, no, os, oe, oseq, &R, d_op_root, d_root_op));
  PM_TRY(stage_group(A, ni, is, (const long long*)in->in_addr,
                     (const long long*)in->in_nbytes, &Bk, tri));
  PM_TRY(stage_join(A, R, nleaf, l_start, l_end, Bk, &J));
  // blocks back in their trace's own time; per-trace block offsets
  const long long nb = Bk.n;
  int* trb = A.alloc<int>(nb);
  long long* blk_off = A.alloc<long long>(B + 1);
  long long* b_alloc = A.alloc<long long>(nb);
  long long* b_free = A.alloc<long long>(nb);
  PM_TRY(check_arena(A, "pm_pipeline_batch blocks"));
  if (nb > 0) {
    // blocks are in instant order, i.e. trace-major: offsets by bisection
    k_block_trace<<<blocks_for(nb), 256, 0, s>>>(Bk.inst, tri, nb, trb);
    k_trace_offsets<<<blocks_for(B + 1), 256, 0, s>>>(trb, nb, B, blk_off);
    std::vector<long long> neg(B);
    for (int t = 0; t < B; ++t) neg[t] = -delta[t];
    long long* d_neg = A.upload(neg.data(), B);
    PM_TRY(check_arena(A, "pm_pipeline_batch blocks"));
    k_rebase<<<blocks_for(nb), 256, 0, s>>>(Bk.alloc, trb, d_neg, nb, INT64_MIN, b_alloc);
    k_rebase<<<blocks_for(nb), 256, 0, s>>>(Bk.free, trb, d_neg, nb, INT64_MIN, b_free);
  } else {
    cudaMemsetAsync(blk_off, 0, sizeof(long long) * (B + 1), s);
  }
  std::vector<long long> h_blk_off(B + 1);
  std::vector<int> h_cyc(B);
  PM_TRY(download(h_blk_off.data(), blk_off, B + 1, s));
  PM_TRY(download(h_cyc.data(), cyclic, B, s));
  PM_TRY(sync_check(s, "pm_pipeline_batch link"));
  // a13-a19: orchestration with each trace's own parameters
  OrchIn oi;
  oi.p.B = B;
  oi.p.trb = trb;
  oi.p.blk_off = blk_off;
  std::vector<int> h_skip(B);
  for (int t = 0; t < B; ++t)
    h_skip[t] = h_cyc[t] ? 1 : (in->skip ? in->skip[t] : 0);
  oi.p.skip = A.upload(h_skip.data(), B);
  const int64_t* so = in->span_off;
  oi.p.span_off = A.upload((const long long*)so, B + 1);
  oi.p.span_start = A.upload((const long long*)in->span_start, so[B]);
  oi.p.span_end = A.upload((const long long*)in->span_end, so[B]);
  oi.p.span_iter = A.upload((const long long*)in->span_iter, so[B]);
  oi.p.param_off = A.upload((const long long*)in->param_off, B + 1);
  oi.p.param_sizes = A.upload((const long long*)in->param_sizes, in->param_off[B]);
  oi.p.win_off = A.upload((const long long*)in->win_off, B + 1);
  oi.p.win_start = A.upload((const long long*)in->win_start, in->win_off[B]);
  oi.p.win_end = A.upload((const long long*)in->win_end, in->win_off[B]);
  oi.p.zg_off = A.upload((const long long*)in->zg_off, B + 1);
  oi.p.zg = A.upload((const long long*)in->zg, in->zg_off[B]);
  oi.p.clones = A.upload((const int*)in->clones, B);
  oi.p.tpl_start = A.upload((const long long*)in->tpl_start, B);
  oi.p.tpl_end = A.upload((const long long*)in->tpl_end, B);
  oi.p.shift = A.upload((const long long*)in->shift, B);
  oi.nb = nb;
  oi.b_alloc = b_alloc;
  oi.b_size = Bk.size;
  oi.b_free = b_free;
  oi.b_role = J.role;
  oi.h_blk_off = h_blk_off.data();
  oi.h_skip = h_skip.data();
  const int64_t* bo = in->bat_off;
  oi.bat_off = A.upload((const long long*)bo, B + 1);
  oi.h_bat_off = (const long long*)bo;
  oi.bat_vts = A.upload((const long long*)in->bat_vts, bo[B]);
  oi.bat_size = A.upload((const long long*)in->bat_size, bo[B]);
  oi.bat_kind = A.upload((const int*)in->bat_kind, bo[B]);
  oi.bat_it = A.upload((const long long*)in->bat_it, bo[B]);
  oi.bat_j = A.upload((const long long*)in->bat_j, bo[B]);
  PM_TRY(check_arena(A, "pm_pipeline_batch params"));
  OrchOut O;
  long long* d_oraw = views ? (long long*)views->o_raw : nullptr;
  int rc = orch_core(A, oi, reqs, req_cap, d_oraw, &O);
  for (int t = 0; t <= B; ++t) req_off[t] = O.roff.empty() ? 0 : O.roff[t];
  if (rc) return rc;
  if (views) {
    // the per-trace views of build_sequence, written to the caller's DEVICE
    // buffers: the ordered request columns and every block's final role /
    // lifetime (orchestration.py:222-223,197)
    if (nb > views->fb_cap) return perr(PM_ERR_WORKSPACE_TOO_SMALL, "pm_pipeline_batch: fb_cap");
    const long long n = O.n;
    if (n > 0)
      k_unpack_ordered<<<blocks_for(n), 256, 0, s>>>(
          O.raw, O.perm, n, views->o_kind, (long long*)views->o_size,
          (long long*)views->o_vts, views->o_tag, (long long*)views->o_a,
          (long long*)views->o_b, views->o_role);
    if (nb > 0) {
      cudaMemcpyAsync(views->fb_role, O.role, sizeof(int32_t) * nb, cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(views->fb_free, O.free_out, sizeof(int64_t) * nb, cudaMemcpyDeviceToDevice, s);
    }
    for (int t = 0; t <= B; ++t) views->blk_off[t] = h_blk_off[t];
  }
  std::vector<unsigned long long> h_bd(8 * (size_t)B);
  PM_TRY(download(h_bd.data(), O.bd, 8 * (size_t)B, s));
  PM_TRY(sync_check(s, "pm_pipeline_batch"));
  for (int t = 0; t < B; ++t) {
    status[t] = h_cyc[t] ? PM_ERR_CYCLIC_PARENT : (h_skip[t] ? PM_ERR_SKIPPED : O.status[t]);
    n_model[t] = O.n_model[t];
    if (breakdown)
      for (int r = 0; r < 8; ++r) breakdown[8 * t + r] = (int64_t)h_bd[8 * t + r];
  }
  return PM_SUCCESS;
}

}  // extern "C"
