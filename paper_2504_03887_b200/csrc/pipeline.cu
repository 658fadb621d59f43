// Data analysis, data link and sequence orchestration on the GPU (sm_100a).
//
// Device restatement of the reference pipeline stages between the parsed
// trace and the allocator replay (reference pkg/src/peakmem/):
//   pm_sort_events  trace.py:222-236     stable sort by raw ts, fp64 normalize
//   pm_link         analysis.py:185-211  operator roots (prefix-max nesting)
//                   analysis.py:252-294  alloc/free grouping by address
//                   linking.py:50-65     innermost-leaf ownership of roots
//                   linking.py:68-92     backward ops by sequence number
//                   linking.py:95-123    block -> owning op / layer, roles
//                   linking.py:40-43,    backward-retained = gradient blocks
//                   orchestration.py:122-132
//   pm_orchestrate  orchestration.py:135-399 (state / drop / clone /
//                   gradient lifetimes / model load / batch / total order)
// Layer-tree construction and marker typing stay on the host (string-typed,
// a few hundred nodes); everything per-event / per-block / per-op is here.
//
// All entry points take HOST arrays and return HOST arrays (the C ABI a
// Python / cgo / JNI caller binds); device memory is stream-ordered scratch.
// Sorting uses CUB's stable onesweep radix sort; joins, scans and the
// role / lifetime maps are the kernels below.

#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "peakmem_b200.h"
#include "peakmem_pipeline.h"

namespace pmp {

typedef unsigned long long u64;
constexpr long long kNoneTs = INT64_MIN;  // "None" timestamp

// ---- small device helpers ---------------------------------------------------

template <class T>
__device__ __forceinline__ long long upper_bound_ll(const T* a, long long n,
                                                    T v) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (a[mid] <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

template <class T>
__device__ __forceinline__ long long lower_bound_ll(const T* a, long long n,
                                                    T v) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// ---- a1: event sort + normalization -----------------------------------------

__global__ void k_ts_keys(const double* ts, long long n, double* keys,
                          long long* idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = ts[i];
  keys[i] = t == 0.0 ? 0.0 : t;  // -0.0 compares equal to 0.0 in Python
  idx[i] = i;
}

// start = floor(ts - t0); end = max(start, ceil((ts + dur) - t0))
// (trace.py:228-234), IEEE fp64 round-to-nearest, no contraction.
__global__ void k_normalize(const double* ts, const double* dur,
                            const long long* perm, long long n,
                            const double* t0p, long long* start,
                            long long* duration) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double t0 = *t0p;
  const long long f = perm[i];
  const double t = ts[f];
  const double e = __dadd_rn(t, dur[f]);
  const long long s = (long long)floor(__dsub_rn(t, t0));
  long long en = (long long)ceil(__dsub_rn(e, t0));
  if (en < s) en = s;
  start[i] = s;
  duration[i] = en - s;
}

// ---- a5: operator roots -----------------------------------------------------

__global__ void k_iota(long long* v, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void k_gather_u64(const long long* src, const long long* idx,
                             long long n, u64 bias, int negate, u64* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  u64 v = (u64)(src[idx[i]]) + bias;
  out[i] = negate ? ~v : v;
}

__global__ void k_gather_ll(const long long* src, const long long* idx,
                            long long n, long long* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[idx[i]];
}

struct MaxOp {
  __device__ __forceinline__ long long operator()(long long a,
                                                  long long b) const {
    return a > b ? a : b;
  }
};

// nested iff start < M and end <= M, M = exclusive prefix max of end
// (analysis.py:199-206)
__global__ void k_root_flags(const long long* s_start, const long long* s_end,
                             const long long* s_pmax, long long n, int* flag) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long M = s_pmax[i];
  const bool nested = s_start[i] < M && s_end[i] <= M;
  flag[i] = nested ? 0 : 1;
}

__global__ void k_root_assign(const long long* perm, const int* incl,
                              const int* flag, const long long* s_start,
                              const long long* s_end, long long n,
                              long long* op_root, long long* root_op,
                              long long* root_start, long long* root_end) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long r = incl[i] - 1;
  op_root[perm[i]] = r;
  if (flag[i]) {
    root_op[r] = perm[i];
    root_start[r] = s_start[i];
    root_end[r] = s_end[i];
  }
}

__global__ void k_seq_keys(const long long* op_root, const long long* seq,
                           long long n, u64* keys, int* valid) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long s = seq[i];
  valid[i] = s >= 0 ? 1 : 0;
  keys[i] = ((u64)op_root[i] << 32) | (u64)(s & 0xffffffffll);
}

// ---- a4: layer tree (analysis.py:113-182) --------------------------------------

// first occurrence of every python id: keys sorted stably by id, the first
// of each run kept (analysis.py:126-134: duplicates keep the first)
__global__ void k_pid_keys(const long long* pid, long long n, u64* keys,
                           long long* idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (u64)pid[i] ^ 0x8000000000000000ull;  // order-preserving bias
  idx[i] = i;
}

__global__ void k_pid_first(const u64* skeys, long long n, int* first) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool none = skeys[i] == 0ull;  // INT64_MIN (None) biased to 0
  first[i] = !none && (i == 0 || skeys[i] != skeys[i - 1]) ? 1 : 0;
}

__global__ void k_pid_parent(const long long* par, long long n,
                             const u64* ukeys, const long long* upos,
                             long long nu, long long* parent_pos) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long p = par[i];
  long long r = -1;
  if (p != kNoneTs && nu > 0) {
    const u64 k = (u64)p ^ 0x8000000000000000ull;
    const long long j = lower_bound_ll(ukeys, nu, k);
    if (j < nu && ukeys[j] == k) r = upos[j];
  }
  parent_pos[i] = r;
}

// nearest layer ancestor of every layer frame: the reference's walk
// (analysis.py:136-151) one parent at a time -- a chain that reaches a
// frame with the walker's own python id (its own frame included) or runs
// longer than n steps revisits an id: CyclicParentLink (flagged).
__global__ void k_layer_anc(const long long* lay, long long nl,
                            const long long* pid, const long long* parent_pos,
                            const unsigned char* is_layer,
                            const long long* lay_index, long long n,
                            const int* tr, long long* node_parent,
                            int* cyclic) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nl) return;
  const long long e = lay[v];
  const long long own = pid[e];
  long long c = parent_pos[e];
  long long steps = 0;
  long long anc = -1;
  while (c >= 0) {
    if (c == e || (own != kNoneTs && pid[c] == own) || ++steps > n) {
      atomicExch(&cyclic[tr ? tr[e] : 0], 1);
      anc = -1;
      break;
    }
    if (is_layer[c]) {
      anc = lay_index[c];
      break;
    }
    c = parent_pos[c];
  }
  node_parent[v] = anc;
}

// CSR offsets of children per parent slot (slot 0 = the synthetic root):
// off[p] = first index in the (parent, start, event)-sorted order
__global__ void k_child_off(const unsigned* sorted_parent_key, long long nl,
                            long long* off) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k > nl + 1) return;
  off[k] = lower_bound_ll(sorted_parent_key, nl, (unsigned)k);
}

// level offsets of depth-sorted nodes: lvl[d] = first node of depth >= d
__global__ void k_level_off(const int* sorted_depth, long long nl, int maxd,
                            long long* lvl) {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d > maxd + 1) return;
  lvl[d] = lower_bound_ll(sorted_depth, nl, d);
}

// depth by pointer jumping (list ranking over parent links)
__global__ void k_depth_init(const long long* node_parent, long long nl,
                             long long* jump, int* depth) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nl) return;
  jump[v] = node_parent[v];
  depth[v] = node_parent[v] >= 0 ? 1 : 0;
}

__global__ void k_depth_step(const long long* jump_in, const int* depth_in,
                             long long nl, long long* jump_out, int* depth_out) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nl) return;
  const long long j = jump_in[v];
  if (j >= 0) {
    depth_out[v] = depth_in[v] + depth_in[j];
    jump_out[v] = jump_in[j];
  } else {
    depth_out[v] = depth_in[v];
    jump_out[v] = -1;
  }
}

// a chain that never reached the root runs into a cycle of layer frames
// (each the other's nearest layer ancestor -- not an error for the
// reference): such nodes hang off no root path and are left out of the walk
__global__ void k_depth_final(const long long* jump, long long nl, int* depth) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v < nl && jump[v] != -1) depth[v] = -1;
}

// subtree sizes, one depth level at a time from the deepest
// One warp per node of the level: a node's children are read 32 at a time
// (a wrapper can have hundreds of thousands of them, which one thread would
// walk serially).
__device__ __forceinline__ long long warp_sum_ll(long long x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ long long warp_incl_scan_ll(long long x) {
  const int lane = threadIdx.x & 31;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// subtree sizes, one level at a time from the bottom.  One warp per node of
// the level; a node with more than kBigNode children (a wrapper over
// hundreds of thousands of layers) is handed to k_subtree_big, one CTA per
// node (`big` collects them: big[0] = count, then the nodes).
constexpr long long kBigNode = 2048;
__global__ void k_subtree_level(const long long* lvl_nodes, long long m,
                                const long long* child_order,
                                const long long* off, long long* size,
                                long long* big) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;  // whole warp
  const long long v = lvl_nodes[w];
  if (off[v + 2] - off[v + 1] > kBigNode) {
    if (lane == 0)
      big[1 + atomicAdd(reinterpret_cast<unsigned long long*>(big), 1ull)] = v;
    return;
  }
  long long s = 0;
  for (long long k = off[v + 1] + lane; k < off[v + 2]; k += 32)
    s += size[child_order[k]];
  s = warp_sum_ll(s);
  if (lane == 0) size[v] = s + 1;
}

constexpr int kBigThreads = 512;
__global__ void __launch_bounds__(kBigThreads)
    k_subtree_big(const long long* big, const long long* child_order,
                  const long long* off, long long* size) {
  typedef cub::BlockReduce<long long, kBigThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const long long nbig = big[0];
  for (long long i = blockIdx.x; i < nbig; i += gridDim.x) {
    const long long v = big[1 + i];
    long long s = 0;
    for (long long k = off[v + 1] + threadIdx.x; k < off[v + 2]; k += kBigThreads)
      s += size[child_order[k]];
    s = BR(tmp).Sum(s);
    if (threadIdx.x == 0) size[v] = s + 1;
    __syncthreads();
  }
}

// pre-order positions of the children of the big nodes of a level (and of
// the synthetic root, big == nullptr): one CTA per node, 512 children per
// step, a block-wide exclusive scan of their subtree sizes
__global__ void __launch_bounds__(kBigThreads)
    k_preorder_big(const long long* big, const long long* child_order,
                   const long long* off, const long long* size, long long* pre) {
  typedef cub::BlockScan<long long, kBigThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  const long long nbig = big ? big[0] : 1;
  for (long long i = blockIdx.x; i < nbig; i += gridDim.x) {
    const long long v = big ? big[1 + i] : -1;
    long long next = v >= 0 ? pre[v] + 1 : 0;
    const long long b = off[v + 2];
    for (long long base = off[v + 1]; base < b; base += kBigThreads) {
      const long long k = base + threadIdx.x;
      long long c = -1, sz = 0;
      if (k < b) {
        c = child_order[k];
        sz = size[c];
      }
      long long ex, total;
      BS(tmp).ExclusiveSum(sz, ex, total);
      if (k < b) pre[c] = next + ex;
      next += total;
      __syncthreads();
    }
  }
}

// pre-order positions, one level at a time from the top: children of v
// take consecutive ranges after pre[v] in (start, event) order (big nodes:
// k_preorder_big)
__global__ void k_preorder_level(const long long* lvl_nodes, long long m,
                                 const long long* child_order,
                                 const long long* off, const long long* size,
                                 long long* pre) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;  // whole warp
  const long long v = lvl_nodes[w];  // -1: the synthetic root
  if (off[v + 2] - off[v + 1] > kBigNode) return;
  long long next = v >= 0 ? pre[v] + 1 : 0;
  const long long b = off[v + 2];
  for (long long base = off[v + 1]; base < b; base += 32) {
    const long long k = base + lane;
    long long c = -1, sz = 0;
    if (k < b) {
      c = child_order[k];
      sz = size[c];
    }
    const long long incl = warp_incl_scan_ll(sz);
    if (k < b) pre[c] = next + incl - sz;
    next += __shfl_sync(0xffffffffu, incl, 31);
  }
}

__global__ void k_scatter_walk(const long long* nodes, long long m,
                               const long long* pre, long long* walk) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) walk[pre[nodes[i]]] = nodes[i];
}

__global__ void k_u8_to_int(const unsigned char* f, long long n, int* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = f[i] ? 1 : 0;
}

__global__ void k_scatter_flagged(const int* flag, const long long* pos,
                                  long long n, long long* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[pos[i]] = i;
}

__global__ void k_gather_parent_key(const long long* node_parent,
                                    const long long* ord, long long nl,
                                    unsigned* keys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < nl) keys[i] = (unsigned)(node_parent[ord[i]] + 1);
}

__global__ void k_gather_u64_idx(const u64* src, const long long* idx,
                                 long long n, u64 bias, u64* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[idx[i]] + bias;
}

// ---- a7: grouping -------------------------------------------------------------

__global__ void k_addr_keys(const long long* addr, long long n, u64* keys,
                            long long* idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (u64)addr[i];
  idx[i] = i;
}

// free_time of a positive instant = ts of the next instant at its address
// in (ts, event_id) order (analysis.py:265-290)
// (batched: tr = trace of each instant; an address recurs only within its
// own trace -- the stable sort keeps each trace's run of an address together)
__global__ void k_next_same_addr(const u64* skeys, const long long* sidx,
                                 long long n, const long long* start,
                                 const int* tr, long long* free_time) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = sidx[i];
  long long ft = kNoneTs;
  if (i + 1 < n && skeys[i + 1] == skeys[i] &&
      (tr == nullptr || tr[sidx[i + 1]] == tr[k]))
    ft = start[sidx[i + 1]];
  free_time[k] = ft;
}

__global__ void k_positive(const long long* nbytes, long long n, int* pos) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) pos[i] = nbytes[i] > 0 ? 1 : 0;
}

__global__ void k_blocks(const int* pos, const int* excl, long long n,
                         const long long* start, const long long* nbytes,
                         const long long* free_inst, long long* b_inst,
                         long long* b_alloc, long long* b_size,
                         long long* b_free) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n || !pos[i]) return;
  const long long b = excl[i];
  b_inst[b] = i;
  b_alloc[b] = start[i];
  b_size[b] = nbytes[i];
  b_free[b] = free_inst[i];
}

// ---- a8: innermost leaf per root ------------------------------------------

__global__ void k_leaf_keys(const long long* lstart, long long n, u64* keys,
                            long long* idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (u64)lstart[i];
  idx[i] = i;
}

// For each root: among leaves with lstart <= rstart and rend <= lend, the
// smallest duration, ties -> first in walk order (linking.py:56-64).
// One warp per root, warp-cooperative: the leaves are sorted by start with
// an inclusive prefix max of their ends; the lanes binary-search the last
// leaf starting at or before the root 32-ary (one probe per lane per round),
// then scan backwards 32 leaves per step.  The prefix max only falls going
// backwards, so the scan ends at the first step where some lane's prefix
// max is below the root's end (no earlier leaf can contain it).
__global__ void k_link_fwd(const long long* sl_start, const long long* sl_w,
                           const long long* sl_pmax_end,
                           const long long* lstart, const long long* lend,
                           long long nl, const long long* rstart,
                           const long long* rend, long long nr,
                           long long* root_leaf) {
  const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nr) return;  // whole warp
  const long long s = rstart[r], e = rend[r];
  // upper_bound(sl_start, s) by 32-ary search: [lo, hi) holds the answer
  long long lo = 0, hi = nl;
  while (hi - lo > 32) {
    const long long step = (hi - lo + 31) / 32;
    const long long k = lo + lane * step;
    const unsigned b = __ballot_sync(0xffffffffu, k < hi && sl_start[k] <= s);
    if (b == 0) {
      hi = lo;  // sl_start[lo] > s
      break;
    }
    const int last = 31 - __clz(b);
    lo += last * step;
    hi = min(lo + step, hi);
    lo += 1;  // sl_start[lo - 1] <= s
  }
  if (hi > lo) {
    const long long k = lo + lane;
    const unsigned b = __ballot_sync(0xffffffffu, k < hi && sl_start[k] <= s);
    lo += b ? 32 - __clz(b) : 0;
  }
  // lo = upper_bound: leaves [0, lo) start at or before the root
  long long best = -1, bdur = 0;
  for (long long base = lo - 1; base >= 0; base -= 32) {
    const long long i = base - lane;
    const bool ok = i >= 0 && sl_pmax_end[i] >= e;
    if (ok) {
      const long long w = sl_w[i];
      if (lend[w] >= e) {
        const long long dur = lend[w] - lstart[w];
        if (best < 0 || dur < bdur || (dur == bdur && w < best)) {
          best = w;
          bdur = dur;
        }
      }
    }
    if (!__all_sync(0xffffffffu, ok)) break;
  }
  // warp argmin of (duration, walk index) over the lanes' candidates
  for (int o = 16; o > 0; o >>= 1) {
    const long long ob = __shfl_down_sync(0xffffffffu, best, o);
    const long long od = __shfl_down_sync(0xffffffffu, bdur, o);
    if (ob >= 0 && (best < 0 || od < bdur || (od == bdur && ob < best))) {
      best = ob;
      bdur = od;
    }
  }
  if (lane == 0) root_leaf[r] = best;
}

// ---- a9: backward ops by sequence number ------------------------------------

// FS pairs (leaf, seq) for every seq of every owned root
__global__ void k_fs_count(const long long* root_leaf, const long long* rs_off,
                           long long nr, long long* cnt) {
  long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nr) return;
  cnt[r] = root_leaf[r] >= 0 ? rs_off[r + 1] - rs_off[r] : 0;
}

__global__ void k_fs_emit(const long long* root_leaf, const long long* rs_off,
                          const long long* rs_seq, const long long* fs_off,
                          long long nr, long long* fs_leaf, long long* fs_seq) {
  long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nr || root_leaf[r] < 0) return;
  long long o = fs_off[r];
  for (long long k = rs_off[r]; k < rs_off[r + 1]; ++k, ++o) {
    fs_leaf[o] = root_leaf[r];
    fs_seq[o] = rs_seq[k];
  }
}

// by-seq index: (seq, root) pairs sorted by seq
__global__ void k_join_count(const long long* fs_leaf, const long long* fs_seq,
                             long long nfs, const long long* bs_seq,
                             const long long* bs_root, long long nbs,
                             const long long* root_leaf, long long* cnt) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nfs) return;
  const long long s = fs_seq[i], P = fs_leaf[i];
  long long lo = lower_bound_ll(bs_seq, nbs, s);
  long long c = 0;
  for (long long k = lo; k < nbs && bs_seq[k] == s; ++k)
    if (root_leaf[bs_root[k]] != P) ++c;
  cnt[i] = c;
}

__global__ void k_join_emit(const long long* fs_leaf, const long long* fs_seq,
                            long long nfs, const long long* bs_seq,
                            const long long* bs_root, long long nbs,
                            const long long* root_leaf, const long long* off,
                            u64* keys, long long* seqs) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nfs) return;
  const long long s = fs_seq[i], P = fs_leaf[i];
  long long lo = lower_bound_ll(bs_seq, nbs, s);
  long long o = off[i];
  for (long long k = lo; k < nbs && bs_seq[k] == s; ++k) {
    const long long r = bs_root[k];
    if (root_leaf[r] != P) {
      keys[o] = ((u64)P << 32) | (u64)r;
      seqs[o] = s;
      ++o;
    }
  }
}

// ---- a10 / a11: block attachment and gradients ----------------------------


__global__ void k_owned_flag(const long long* owner, long long nr, int* f) {
  long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r < nr) f[r] = owner[r] >= 0 ? 1 : 0;
}

enum Role { R_UNCL = 0, R_MODEL = 1, R_BATCH = 2, R_GRAD = 3, R_STATE = 4,
            R_TEMP = 5, R_RET = 6 };

__global__ void k_unpack_pairs(const u64* keys, long long n, long long* hi,
                               long long* lo) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  hi[i] = (long long)(keys[i] >> 32);
  lo[i] = (long long)(keys[i] & 0xffffffffull);
}

__global__ void k_count_by(const long long* key, long long n, long long* cnt) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[key[i]]), 1ull);
}

// ---- exact join helpers -------------------------------------------------------

struct MinOp {
  __device__ __forceinline__ long long operator()(long long a,
                                                  long long b) const {
    return a < b ? a : b;
  }
};

// keys[i] = bias(src[idx[i]]) with idx read as root ids (u64 order of a
// signed value)
__global__ void k_gather_ll2(const long long* src, const long long* idx,
                             long long n, u64* out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (u64)src[idx[i]] + (1ull << 63);
}

// prefix max of root ends along each leaf's backward list
__global__ void k_seg_pmax_end(const long long* off, const long long* roots,
                               const long long* rend, long long nl,
                               long long* pmax) {
  long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (w >= nl) return;
  long long m = INT64_MIN;
  for (long long k = off[w]; k < off[w + 1]; ++k) {
    const long long e = rend[roots[k]];
    m = e > m ? e : m;
    pmax[k] = m;
  }
}

// owner entries: [0, nf) forward (profile, 0, root index), then backward
// (profile, 1, position within the profile's list)
__global__ void k_owner_entries(const long long* fwd_roots, long long nf,
                                const long long* root_leaf,
                                const long long* bw_leaf,
                                const long long* bw_root, long long nbw,
                                const long long* bw_off,
                                const long long* rstart, long long* ow_root,
                                long long* ow_prof, u64* key) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nf + nbw) return;
  long long P, r, kind, pos;
  if (i < nf) {
    r = fwd_roots[i];
    P = root_leaf[r];
    kind = 0;
    pos = r;
  } else {
    const long long k = i - nf;
    r = bw_root[k];
    P = bw_leaf[k];
    kind = 1;
    pos = k - bw_off[P];
  }
  ow_root[i] = r;
  ow_prof[i] = P;
  // profile (24 bits) | kind (1) | position (39)
  key[i] = ((u64)P << 40) | ((u64)kind << 39) | (u64)pos;
  (void)rstart;
}

// biased start of each entry's root, in the current permutation order
__global__ void k_entry_start_key(const long long* perm, const long long* ow_root,
                                  const long long* rstart, long long n,
                                  u64* key) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) key[i] = (u64)rstart[ow_root[perm[i]]] + (1ull << 63);
}

__global__ void k_owner_finish(const long long* perm, const long long* ow_root,
                               const long long* ow_prof,
                               const long long* rstart, long long n,
                               long long* o_start, long long* o_root,
                               long long* o_prof) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long e = perm[i];
  o_root[i] = ow_root[e];
  o_prof[i] = ow_prof[e];
  o_start[i] = rstart[ow_root[e]];
}

// attach_blocks on the sorted owner list: the last entry with start <= alloc
// (bisect_right - 1), then the half-open containment check.
__global__ void k_attach2(const long long* o_start, const long long* o_root,
                          const long long* o_prof, long long n_own,
                          const long long* rend, const long long* b_alloc,
                          const long long* b_free, long long nb, int* role,
                          long long* prof, long long* b_root) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const long long t = b_alloc[b];
  const long long i = upper_bound_ll(o_start, n_own, t) - 1;
  int rl = 0;
  long long P = -1, rr = -1;
  if (i >= 0) {
    const long long r = o_root[i];
    if (t < rend[r]) {
      const long long f = b_free[b];
      rl = (f != kNoneTs && f < rend[r]) ? 5 : 6;
      P = o_prof[i];
      rr = r;
    }
  }
  role[b] = rl;
  prof[b] = P;
  b_root[b] = rr;
}

// backward_retained_blocks (linking.py:40-43): any backward op of the
// block's profile containing alloc; backward scan bounded by prefix max.
__global__ void k_gradients2(const long long* bw_off, const long long* bw_root,
                             const long long* bw_pmax, const long long* rstart,
                             const long long* rend, const long long* b_alloc,
                             const long long* prof, long long nb, int* role) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb || role[b] != 6) return;
  const long long P = prof[b], t = b_alloc[b];
  long long lo = bw_off[P], hi = bw_off[P + 1];
  // entries are sorted by start: last with start <= t
  long long a = lo, z = hi;
  while (a < z) {
    long long mid = (a + z) >> 1;
    if (rstart[bw_root[mid]] <= t)
      a = mid + 1;
    else
      z = mid;
  }
  for (long long k = a - 1; k >= lo && bw_pmax[k] > t; --k) {
    if (rend[bw_root[k]] > t) {
      role[b] = 3;
      return;
    }
  }
}

// ---- a14-a19: orchestration ---------------------------------------------------

struct OrchParams {
  int n_spans;
  const long long* span_start;  // span markers in marker order
  const long long* span_end;
  const long long* span_iter;
  int n_param;
  const long long* param_sizes;  // sorted unique
  int n_windows;
  const long long* win_start;
  const long long* win_end;
  int n_zg;
  const long long* zg;  // sorted zero-grad starts (original + cloned)
  long long tpl_start, tpl_end;  // clone template window (if clones)
  int clones;
  long long shift;  // template width
};

enum Flags { F_SEQ = 1, F_CHOSEN = 2, F_TPL = 4, F_MODEL = 8 };

__device__ __forceinline__ long long next_zg(const long long* zg, int n,
                                             long long t) {
  long long i = upper_bound_ll(zg, (long long)n, t);
  return i < n ? zg[i] : kNoneTs;
}

// Per-block role / lifetime rewrite (orchestration.py:270-347).
__global__ void k_orch_blocks(OrchParams p, const long long* b_alloc,
                              const long long* b_size, const long long* b_free,
                              const int* role_in, const int* grad,
                              long long nb, int* role_out, long long* free0,
                              long long* free_out, int* flags) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const long long t = b_alloc[b], sz = b_size[b];
  int role = role_in[b];
  long long fr = b_free[b];
  bool dropped = false;
  for (int k = 0; k < p.n_spans; ++k) {
    const long long s = p.span_start[k], e = p.span_end[k];
    if (!(s <= t && t < e)) continue;
    if (p.span_iter[k] == 0) {
      // extract_optimizer_state (orchestration.py:200-227)
      const long long pi = lower_bound_ll(p.param_sizes, (long long)p.n_param, sz);
      const bool is_param = pi < p.n_param && p.param_sizes[pi] == sz;
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
  if (seq && role != R_STATE && p.clones > 0 && p.tpl_start <= t &&
      t < p.tpl_end)
    f |= F_TPL;
  free0[b] = fr;  // lifetime at clone time
  if (grad[b]) fr = next_zg(p.zg, p.n_zg, t);  // adjust_gradient_lifetimes
  bool inwin = false;
  if (p.n_windows > 0) {
    if (t < p.win_start[0]) inwin = true;
    for (int k = 0; k < p.n_windows && !inwin; ++k)
      if (p.win_start[k] <= t && t < p.win_end[k]) inwin = true;
  }
  if (seq && inwin) f |= F_CHOSEN;
  if (grad[b] && p.n_windows > 0 && p.win_start[0] <= t && t < p.win_end[0])
    f |= F_MODEL;
  role_out[b] = role;
  free_out[b] = fr;
  flags[b] = f;
}

// raw request record (pre-order): tag 0 model / 1 batch / 2 block / 3 clone
struct RawReq {
  long long vts, size;
  long long a, b;  // model: i | batch: iteration, j | block: id | clone: c, id
  int kind;        // 0 alloc, 1 free
  int tag;
  int role;
  int pad;
};

__global__ void k_emit_blocks(const int* flags, const long long* b_alloc,
                              const long long* b_size,
                              const long long* free_out, const int* role,
                              const long long* chosen_off, long long nb,
                              long long base, RawReq* raw) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb || !(flags[b] & F_CHOSEN)) return;
  long long o = base + chosen_off[b];
  RawReq r;
  r.vts = b_alloc[b];
  r.size = b_size[b];
  r.a = b;
  r.b = 0;
  r.kind = 0;
  r.tag = 2;
  r.role = role[b];
  r.pad = 0;
  raw[o] = r;
  if (free_out[b] != kNoneTs) {
    r.vts = free_out[b];
    r.kind = 1;
    raw[o + 1] = r;
  }
}

__global__ void k_emit_clones(const int* flags, const long long* b_alloc,
                              const long long* b_size, const long long* free0,
                              const int* role, const long long* tpl_off,
                              long long ntpl_req, long long nb, long long base,
                              OrchParams p, RawReq* raw) {
  long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nb || !(flags[b] & F_TPL)) return;
  for (int c = 1; c <= p.clones; ++c) {
    const long long shift = p.shift * c;
    long long o = base + (long long)(c - 1) * ntpl_req + tpl_off[b];
    const long long t = b_alloc[b] + shift;
    long long fr = free0[b] == kNoneTs ? kNoneTs : free0[b] + shift;
    if (role[b] == R_GRAD) fr = next_zg(p.zg, p.n_zg, t);
    RawReq r;
    r.vts = t;
    r.size = b_size[b];
    r.a = c;
    r.b = b;
    r.kind = 0;
    r.tag = 3;
    r.role = role[b];
    r.pad = 0;
    raw[o] = r;
    if (fr != kNoneTs) {
      r.vts = fr;
      r.kind = 1;
      raw[o + 1] = r;
    }
  }
}

// total order key (orchestration.py:368-383): (virtual_ts, rank, idx) with
// rank 0 = free of an older block, 1 = alloc, 2 = free at its alloc's ts.
// Every free follows its alloc in raw order, so alloc ts is raw[i-1].vts.
__global__ void k_order_keys(const RawReq* raw, long long n, long long vmin,
                             u64* keys, long long* idx) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const RawReq r = raw[i];
  int rank = 1;
  if (r.kind == 1) rank = raw[i - 1].vts < r.vts ? 0 : 2;
  keys[i] = ((u64)(r.vts - vmin) << 2) | (u64)rank;
  idx[i] = i;
}

// min / max virtual timestamp: a warp reduction, then one atomic pair per
// warp (one pair per element serialised on two addresses)
__global__ void k_minmax_vts(const RawReq* raw, long long n, long long* mm) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long lo = INT64_MAX, hi = INT64_MIN;
  if (i < n) lo = hi = raw[i].vts;
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}

// packed replay records: handle = raw index of the block's alloc
__global__ void k_pack(const RawReq* raw, const long long* perm, long long n,
                       pm_req_t* out, long long* out_raw) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long k = perm[i];
  const RawReq r = raw[k];
  pm_req_t q;
  q.size = r.size;
  q.handle = (int32_t)(r.kind == 0 ? k : k - 1);
  q.kind_stream = r.kind == 0 ? PM_KIND_ALLOC : PM_KIND_FREE;
  out[i] = q;
  out_raw[i] = k;
}

}  // namespace pmp

// ---------------------------------------------------------------------------
// Host side.

namespace {

using pmp::u64;
thread_local std::string g_err;

int perr(int code, const std::string& m) {
  g_err = m;
  return code;
}

// The default release threshold (0) hands the stream-ordered pool's memory
// back to the driver at every synchronisation, so each call would map its
// scratch (GBs at C5 scale) afresh; keep it mapped between calls.
void keep_pool_mapped() {
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

// stream-ordered scratch arena, freed on destruction
struct Arena {
  cudaStream_t s;
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  explicit Arena(cudaStream_t st) : s(st) { keep_pool_mapped(); }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), s);
    if (e != cudaSuccess) {
      err = e;
      return nullptr;
    }
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const T* h, size_t n) {
    T* d = alloc<T>(n);
    if (d && n) {
      cudaError_t e = cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) err = e;
    }
    return d;
  }
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

inline unsigned blocks_for(long long n, int t = 256) {
  return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1);
}

template <class T>
int download(T* h, const T* d, size_t n, cudaStream_t s) {
  if (n == 0) return PM_SUCCESS;
  cudaError_t e = cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return perr(PM_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
  return PM_SUCCESS;
}

int sync_check(cudaStream_t s, const char* what) {
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return perr(PM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return PM_SUCCESS;
}

// stable radix sort of (u64 key, i64 value) pairs, in place via scratch
int sort_pairs(Arena& A, u64* keys, long long* vals, long long n, int end_bit = 64) {
  if (n <= 1) return PM_SUCCESS;
  u64* k2 = A.alloc<u64>(n);
  long long* v2 = A.alloc<long long>(n);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, k2, vals, v2, (int64_t)n, 0, end_bit, A.s);
  void* t = A.alloc<char>(tmp);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "sort scratch");
  cub::DeviceRadixSort::SortPairs(t, tmp, keys, k2, vals, v2, (int64_t)n, 0, end_bit, A.s);
  cudaMemcpyAsync(keys, k2, n * sizeof(u64), cudaMemcpyDeviceToDevice, A.s);
  cudaMemcpyAsync(vals, v2, n * sizeof(long long), cudaMemcpyDeviceToDevice, A.s);
  return PM_SUCCESS;
}

template <class T, class U>
int excl_sum(Arena& A, const T* in, U* out, long long n) {
  if (n <= 0) return PM_SUCCESS;
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int64_t)n, A.s);
  void* t = A.alloc<char>(tmp);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "scan scratch");
  cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int64_t)n, A.s);
  return PM_SUCCESS;
}

template <class T>
int incl_sum(Arena& A, const T* in, T* out, long long n) {
  if (n <= 0) return PM_SUCCESS;
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, (int64_t)n, A.s);
  void* t = A.alloc<char>(tmp);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "scan scratch");
  cub::DeviceScan::InclusiveSum(t, tmp, in, out, (int64_t)n, A.s);
  return PM_SUCCESS;
}

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T h{};
  cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return h;
}

}  // namespace

extern "C" {

const char* pm_pipeline_last_error(void) { return g_err.c_str(); }

// a1 (trace.py:222-236): stable sort of events by raw ts (file order breaks
// ties) and fp64 normalization.  perm[i] = file index of the i-th event.
int pm_sort_events(const double* ts, const double* dur, int64_t n,
                   int64_t* perm, int64_t* start, int64_t* duration,
                   void* stream_) {
  if (n < 0 || (n > 0 && (!ts || !dur || !perm || !start || !duration)))
    return perr(PM_ERR_INVALID_ARGUMENT, "pm_sort_events: bad arguments");
  if (n == 0) return PM_SUCCESS;
  cudaStream_t s = (cudaStream_t)stream_;
  Arena A(s);
  double* d_ts = A.upload(ts, n);
  double* d_dur = A.upload(dur, n);
  double* keys = A.alloc<double>(n);
  double* k2 = A.alloc<double>(n);
  long long* idx = A.alloc<long long>(n);
  long long* idx2 = A.alloc<long long>(n);
  long long* d_start = A.alloc<long long>(n);
  long long* d_dur_o = A.alloc<long long>(n);
  if (A.err != cudaSuccess) return perr(PM_ERR_CUDA, "pm_sort_events: alloc");
  pmp::k_ts_keys<<<blocks_for(n), 256, 0, s>>>(d_ts, n, keys, idx);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, k2, idx, idx2, (int64_t)n, 0, 64, s);
  void* t = A.alloc<char>(tmp);
  cub::DeviceRadixSort::SortPairs(t, tmp, keys, k2, idx, idx2, (int64_t)n, 0, 64, s);
  pmp::k_normalize<<<blocks_for(n), 256, 0, s>>>(d_ts, d_dur, idx2, n, k2,
                                                 d_start, d_dur_o);
  int rc = download(perm, (const int64_t*)idx2, n, s);
  if (rc == PM_SUCCESS) rc = download(start, (const int64_t*)d_start, n, s);
  if (rc == PM_SUCCESS) rc = download(duration, (const int64_t*)d_dur_o, n, s);
  if (rc != PM_SUCCESS) return rc;
  return sync_check(s, "pm_sort_events");
}

// ---- staged link pipeline (device pointers) --------------------------------

}  // extern "C"

namespace {

using namespace pmp;

struct RootsDev {
  long long n = 0, nseq = 0;
  long long* start = nullptr;
  long long* end = nullptr;
  long long* rs_off = nullptr;   // [n+1] CSR of sorted unique seqs
  long long* rs_seq = nullptr;
  long long* rs_root = nullptr;
};

struct BlocksDev {
  long long n = 0;
  long long *inst = nullptr, *alloc = nullptr, *size = nullptr, *free = nullptr;
};

struct JoinDev {
  long long* root_leaf = nullptr;
  long long nbw = 0;
  long long* bw_off = nullptr;
  long long* bw_root = nullptr;
  int* role = nullptr;
  long long* prof = nullptr;
  long long* broot = nullptr;
};

#define PM_TRY(x)                 \
  do {                            \
    int rc_ = (x);                \
    if (rc_ != PM_SUCCESS) return rc_; \
  } while (0)

int check_arena(Arena& A, const char* w) {
  return A.err != cudaSuccess ? perr(PM_ERR_CUDA, std::string(w) + ": " +
                                                      cudaGetErrorString(A.err))
                              : PM_SUCCESS;
}

// CSR offsets from a key column sorted ascending: off[k] = first index of k
int csr_from_sorted(Arena& A, const long long* key, long long n, long long nk,
                    long long* off) {
  long long* cnt = A.alloc<long long>(nk + 1);
  PM_TRY(check_arena(A, "csr"));
  cudaMemsetAsync(cnt, 0, sizeof(long long) * (nk + 1), A.s);
  if (n > 0) k_count_by<<<blocks_for(n), 256, 0, A.s>>>(key, n, cnt);
  return excl_sum(A, cnt, off, nk + 1);
}

// sort unique u64 keys in place; returns the unique count
long long sort_unique(Arena& A, u64* keys, long long n, u64* out) {
  if (n == 0) return 0;
  long long* dummy = A.alloc<long long>(n);
  long long* nout = A.alloc<long long>(1);
  if (A.err != cudaSuccess) return -1;
  k_iota<<<blocks_for(n), 256, 0, A.s>>>(dummy, n);
  if (sort_pairs(A, keys, dummy, n)) return -1;
  size_t tmp = 0;
  cub::DeviceSelect::Unique(nullptr, tmp, keys, out, nout, (int64_t)n, A.s);
  void* t = A.alloc<char>(tmp);
  if (A.err != cudaSuccess) return -1;
  cub::DeviceSelect::Unique(t, tmp, keys, out, nout, (int64_t)n, A.s);
  return read_scalar(nout, A.s);
}

// a5 (analysis.py:185-211)
int stage_roots(Arena& A, long long no, const long long* d_ostart,
                const long long* d_oend, const long long* d_oseq,
                RootsDev* R, long long* d_op_root, long long* d_root_op) {
  cudaStream_t s = A.s;
  long long* perm = A.alloc<long long>(no);
  u64* keys = A.alloc<u64>(no);
  long long* s_start = A.alloc<long long>(no);
  long long* s_end = A.alloc<long long>(no);
  long long* s_pmax = A.alloc<long long>(no);
  int* flag = A.alloc<int>(no);
  int* incl = A.alloc<int>(no);
  R->start = A.alloc<long long>(no);
  R->end = A.alloc<long long>(no);
  PM_TRY(check_arena(A, "stage_roots"));
  long long nr = 0;
  if (no > 0) {
    k_iota<<<blocks_for(no), 256, 0, s>>>(perm, no);
    // (start asc, end desc, id asc) by two stable LSD passes
    k_gather_u64<<<blocks_for(no), 256, 0, s>>>(d_oend, perm, no, 1ull << 63, 1, keys);
    PM_TRY(sort_pairs(A, keys, perm, no));
    k_gather_u64<<<blocks_for(no), 256, 0, s>>>(d_ostart, perm, no, 1ull << 63, 0, keys);
    PM_TRY(sort_pairs(A, keys, perm, no));
    k_gather_ll<<<blocks_for(no), 256, 0, s>>>(d_ostart, perm, no, s_start);
    k_gather_ll<<<blocks_for(no), 256, 0, s>>>(d_oend, perm, no, s_end);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveScan(nullptr, tmp, s_end, s_pmax, MaxOp(), (long long)INT64_MIN, (int64_t)no, s);
    void* t = A.alloc<char>(tmp);
    PM_TRY(check_arena(A, "stage_roots scan"));
    cub::DeviceScan::ExclusiveScan(t, tmp, s_end, s_pmax, MaxOp(), (long long)INT64_MIN, (int64_t)no, s);
    k_root_flags<<<blocks_for(no), 256, 0, s>>>(s_start, s_end, s_pmax, no, flag);
    PM_TRY(incl_sum(A, flag, incl, no));
    k_root_assign<<<blocks_for(no), 256, 0, s>>>(perm, incl, flag, s_start, s_end, no,
                                                 d_op_root, d_root_op, R->start, R->end);
    nr = read_scalar(incl + no - 1, s);
  }
  R->n = nr;
  // seqs absorbed into their roots: sorted unique (root, seq)
  u64* skeys = A.alloc<u64>(no);
  int* svalid = A.alloc<int>(no);
  u64* sel = A.alloc<u64>(no);
  u64* uq = A.alloc<u64>(no);
  long long* nsel = A.alloc<long long>(1);
  R->rs_off = A.alloc<long long>(nr + 1);
  R->rs_seq = A.alloc<long long>(no);
  R->rs_root = A.alloc<long long>(no);
  PM_TRY(check_arena(A, "stage_roots seqs"));
  long long nseq = 0;
  if (no > 0) {
    k_seq_keys<<<blocks_for(no), 256, 0, s>>>(d_op_root, d_oseq, no, skeys, svalid);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, skeys, svalid, sel, nsel, (int64_t)no, s);
    void* t = A.alloc<char>(tmp);
    PM_TRY(check_arena(A, "stage_roots select"));
    cub::DeviceSelect::Flagged(t, tmp, skeys, svalid, sel, nsel, (int64_t)no, s);
    const long long nv = read_scalar(nsel, s);
    nseq = sort_unique(A, sel, nv, uq);
    if (nseq < 0) return perr(PM_ERR_CUDA, "stage_roots unique");
    if (nseq > 0) k_unpack_pairs<<<blocks_for(nseq), 256, 0, s>>>(uq, nseq, R->rs_root, R->rs_seq);
  }
  R->nseq = nseq;
  return csr_from_sorted(A, R->rs_root, nseq, nr, R->rs_off);
}

// a7 (analysis.py:252-294)
int stage_group(Arena& A, long long ni, const long long* d_istart,
                const long long* d_iaddr, const long long* d_inb, BlocksDev* B,
                const int* d_itr = nullptr) {
  cudaStream_t s = A.s;
  u64* akeys = A.alloc<u64>(ni);
  long long* aidx = A.alloc<long long>(ni);
  long long* free_inst = A.alloc<long long>(ni);
  int* pos = A.alloc<int>(ni);
  int* pexcl = A.alloc<int>(ni);
  B->inst = A.alloc<long long>(ni);
  B->alloc = A.alloc<long long>(ni);
  B->size = A.alloc<long long>(ni);
  B->free = A.alloc<long long>(ni);
  PM_TRY(check_arena(A, "stage_group"));
  long long nb = 0;
  if (ni > 0) {
    k_addr_keys<<<blocks_for(ni), 256, 0, s>>>(d_iaddr, ni, akeys, aidx);
    PM_TRY(sort_pairs(A, akeys, aidx, ni));
    k_next_same_addr<<<blocks_for(ni), 256, 0, s>>>(akeys, aidx, ni, d_istart, d_itr,
                                                    free_inst);
    k_positive<<<blocks_for(ni), 256, 0, s>>>(d_inb, ni, pos);
    PM_TRY(excl_sum(A, pos, pexcl, ni));
    nb = read_scalar(pexcl + ni - 1, s) + read_scalar(pos + ni - 1, s);
    k_blocks<<<blocks_for(ni), 256, 0, s>>>(pos, pexcl, ni, d_istart, d_inb, free_inst,
                                            B->inst, B->alloc, B->size, B->free);
  }
  B->n = nb;
  return PM_SUCCESS;
}

// a8-a11 (linking.py:50-132, orchestration.py:122-132): exact for any
// root set (unsorted or equal starts included).
int stage_join(Arena& A, const RootsDev& R, long long nl,
               const long long* d_lstart, const long long* d_lend,
               const BlocksDev& B, JoinDev* J) {
  cudaStream_t s = A.s;
  const long long nr = R.n, nseq = R.nseq, nb = B.n;
  // -- forward owner per root
  u64* lkeys = A.alloc<u64>(nl);
  long long* lidx = A.alloc<long long>(nl);
  long long* sl_start = A.alloc<long long>(nl);
  long long* sl_end = A.alloc<long long>(nl);
  long long* sl_pmax = A.alloc<long long>(nl);
  J->root_leaf = A.alloc<long long>(nr);
  PM_TRY(check_arena(A, "stage_join"));
  if (nl > 0) {
    k_leaf_keys<<<blocks_for(nl), 256, 0, s>>>(d_lstart, nl, lkeys, lidx);
    PM_TRY(sort_pairs(A, lkeys, lidx, nl));
    k_gather_ll<<<blocks_for(nl), 256, 0, s>>>(d_lstart, lidx, nl, sl_start);
    k_gather_ll<<<blocks_for(nl), 256, 0, s>>>(d_lend, lidx, nl, sl_end);
    size_t tmp = 0;
    cub::DeviceScan::InclusiveScan(nullptr, tmp, sl_end, sl_pmax, MaxOp(), (int64_t)nl, s);
    void* t = A.alloc<char>(tmp);
    PM_TRY(check_arena(A, "stage_join scan"));
    cub::DeviceScan::InclusiveScan(t, tmp, sl_end, sl_pmax, MaxOp(), (int64_t)nl, s);
  }
  if (nr > 0) {
    if (nl > 0)
      k_link_fwd<<<blocks_for(32 * nr), 256, 0, s>>>(sl_start, lidx, sl_pmax, d_lstart, d_lend,
                                                     nl, R.start, R.end, nr, J->root_leaf);
    else
      cudaMemsetAsync(J->root_leaf, 0xff, sizeof(long long) * nr, s);
  }
  // -- backward ops: (leaf, root) pairs through shared seqs
  long long* fs_cnt = A.alloc<long long>(nr + 1);
  long long* fs_off = A.alloc<long long>(nr + 1);
  PM_TRY(check_arena(A, "stage_join fs"));
  long long nfs = 0;
  if (nr > 0) {
    cudaMemsetAsync(fs_cnt, 0, sizeof(long long) * (nr + 1), s);
    k_fs_count<<<blocks_for(nr), 256, 0, s>>>(J->root_leaf, R.rs_off, nr, fs_cnt);
    PM_TRY(excl_sum(A, fs_cnt, fs_off, nr + 1));
    nfs = read_scalar(fs_off + nr, s);
  }
  long long* fs_leaf = A.alloc<long long>(nfs);
  long long* fs_seq = A.alloc<long long>(nfs);
  u64* bs_keys = A.alloc<u64>(nseq);
  long long* bs_root = A.alloc<long long>(nseq);
  long long* j_cnt = A.alloc<long long>(nfs + 1);
  long long* j_off = A.alloc<long long>(nfs + 1);
  PM_TRY(check_arena(A, "stage_join join"));
  long long nj = 0;
  if (nfs > 0) {
    k_fs_emit<<<blocks_for(nr), 256, 0, s>>>(J->root_leaf, R.rs_off, R.rs_seq, fs_off, nr,
                                             fs_leaf, fs_seq);
    cudaMemcpyAsync(bs_root, R.rs_root, sizeof(long long) * nseq, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(bs_keys, R.rs_seq, sizeof(long long) * nseq, cudaMemcpyDeviceToDevice, s);
    PM_TRY(sort_pairs(A, bs_keys, bs_root, nseq));
    cudaMemsetAsync(j_cnt, 0, sizeof(long long) * (nfs + 1), s);
    k_join_count<<<blocks_for(nfs), 256, 0, s>>>(fs_leaf, fs_seq, nfs, (const long long*)bs_keys,
                                                 bs_root, nseq, J->root_leaf, j_cnt);
    PM_TRY(excl_sum(A, j_cnt, j_off, nfs + 1));
    nj = read_scalar(j_off + nfs, s);
  }
  u64* jkeys = A.alloc<u64>(nj);
  long long* jseq = A.alloc<long long>(nj);
  u64* ukeys = A.alloc<u64>(nj);
  long long* umin = A.alloc<long long>(nj);
  long long* nrun = A.alloc<long long>(1);
  PM_TRY(check_arena(A, "stage_join pairs"));
  long long nbw = 0;
  if (nj > 0) {
    k_join_emit<<<blocks_for(nfs), 256, 0, s>>>(fs_leaf, fs_seq, nfs, (const long long*)bs_keys,
                                                bs_root, nseq, J->root_leaf, j_off, jkeys, jseq);
    PM_TRY(sort_pairs(A, jkeys, jseq, nj));
    size_t tmp = 0;
    cub::DeviceReduce::ReduceByKey(nullptr, tmp, jkeys, ukeys, jseq, umin, nrun, MinOp(),
                                   (int64_t)nj, s);
    void* t = A.alloc<char>(tmp);
    PM_TRY(check_arena(A, "stage_join reduce"));
    cub::DeviceReduce::ReduceByKey(t, tmp, jkeys, ukeys, jseq, umin, nrun, MinOp(),
                                   (int64_t)nj, s);
    nbw = read_scalar(nrun, s);
  }
  // order within a leaf: (start, first matching seq, root) -- the stable
  // found.sort(key=start) over seq-then-by_seq insertion (linking.py:83-90)
  J->nbw = nbw;
  long long* bw_leaf = A.alloc<long long>(nbw);
  J->bw_root = A.alloc<long long>(nbw);
  long long* bperm = A.alloc<long long>(nbw);
  u64* bkey = A.alloc<u64>(nbw);
  long long* tmpll = A.alloc<long long>(nbw);
  J->bw_off = A.alloc<long long>(nl + 1);
  PM_TRY(check_arena(A, "stage_join bwd"));
  if (nbw > 0) {
    k_unpack_pairs<<<blocks_for(nbw), 256, 0, s>>>(ukeys, nbw, bw_leaf, J->bw_root);
    k_iota<<<blocks_for(nbw), 256, 0, s>>>(bperm, nbw);
    // LSD passes: root (already ascending within leaf), min seq, start, leaf
    k_gather_u64<<<blocks_for(nbw), 256, 0, s>>>(umin, bperm, nbw, 1ull << 63, 0, bkey);
    PM_TRY(sort_pairs(A, bkey, bperm, nbw));
    k_gather_ll<<<blocks_for(nbw), 256, 0, s>>>(J->bw_root, bperm, nbw, tmpll);
    k_gather_ll2<<<blocks_for(nbw), 256, 0, s>>>(R.start, tmpll, nbw, bkey);
    PM_TRY(sort_pairs(A, bkey, bperm, nbw));
    k_gather_u64<<<blocks_for(nbw), 256, 0, s>>>(bw_leaf, bperm, nbw, 1ull << 63, 0, bkey);
    PM_TRY(sort_pairs(A, bkey, bperm, nbw));
    k_gather_ll<<<blocks_for(nbw), 256, 0, s>>>(J->bw_root, bperm, nbw, tmpll);
    cudaMemcpyAsync(J->bw_root, tmpll, sizeof(long long) * nbw, cudaMemcpyDeviceToDevice, s);
    k_gather_ll<<<blocks_for(nbw), 256, 0, s>>>(bw_leaf, bperm, nbw, tmpll);
    cudaMemcpyAsync(bw_leaf, tmpll, sizeof(long long) * nbw, cudaMemcpyDeviceToDevice, s);
  }
  PM_TRY(csr_from_sorted(A, bw_leaf, nbw, nl, J->bw_off));
  // prefix max of ends within each leaf's backward list
  long long* bw_pmax = A.alloc<long long>(nbw);
  PM_TRY(check_arena(A, "stage_join pmax"));
  if (nbw > 0 && nl > 0)
    k_seg_pmax_end<<<blocks_for(nl), 256, 0, s>>>(J->bw_off, J->bw_root, R.end, nl, bw_pmax);
  // -- owner list (attach_blocks, linking.py:102-108): profiles in walk
  // order, forward ops (root order) then backward ops, stable by start
  long long* nf = A.alloc<long long>(1);
  long long* fwd_roots = A.alloc<long long>(nr);
  PM_TRY(check_arena(A, "stage_join owners"));
  long long n_fwd = 0;
  if (nr > 0) {
    int* fl = A.alloc<int>(nr);
    long long* ri = A.alloc<long long>(nr);
    PM_TRY(check_arena(A, "stage_join fwd"));
    k_owned_flag<<<blocks_for(nr), 256, 0, s>>>(J->root_leaf, nr, fl);
    k_iota<<<blocks_for(nr), 256, 0, s>>>(ri, nr);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, ri, fl, fwd_roots, nf, (int64_t)nr, s);
    void* t = A.alloc<char>(tmp);
    PM_TRY(check_arena(A, "stage_join sel"));
    cub::DeviceSelect::Flagged(t, tmp, ri, fl, fwd_roots, nf, (int64_t)nr, s);
    n_fwd = read_scalar(nf, s);
  }
  const long long n_own = n_fwd + nbw;
  long long* ow_root = A.alloc<long long>(n_own);
  long long* ow_prof = A.alloc<long long>(n_own);
  long long* operm = A.alloc<long long>(n_own);
  u64* okey = A.alloc<u64>(n_own);
  long long* o_start = A.alloc<long long>(n_own);
  long long* o_root = A.alloc<long long>(n_own);
  long long* o_prof = A.alloc<long long>(n_own);
  PM_TRY(check_arena(A, "stage_join owner list"));
  if (n_own > 0) {
    k_owner_entries<<<blocks_for(n_own), 256, 0, s>>>(fwd_roots, n_fwd, J->root_leaf, bw_leaf,
                                                     J->bw_root, nbw, J->bw_off, R.start,
                                                     ow_root, ow_prof, okey);
    k_iota<<<blocks_for(n_own), 256, 0, s>>>(operm, n_own);
    PM_TRY(sort_pairs(A, okey, operm, n_own));  // pre-sort list order
    k_entry_start_key<<<blocks_for(n_own), 256, 0, s>>>(operm, ow_root, R.start, n_own, okey);
    PM_TRY(sort_pairs(A, okey, operm, n_own));  // stable by start
    k_owner_finish<<<blocks_for(n_own), 256, 0, s>>>(operm, ow_root, ow_prof, R.start, n_own,
                                                     o_start, o_root, o_prof);
  }
  // -- blocks
  J->role = A.alloc<int>(nb);
  J->prof = A.alloc<long long>(nb);
  J->broot = A.alloc<long long>(nb);
  PM_TRY(check_arena(A, "stage_join blocks"));
  if (nb > 0) {
    k_attach2<<<blocks_for(nb), 256, 0, s>>>(o_start, o_root, o_prof, n_own, R.end, B.alloc,
                                             B.free, nb, J->role, J->prof, J->broot);
    if (nl > 0)
      k_gradients2<<<blocks_for(nb), 256, 0, s>>>(J->bw_off, J->bw_root, bw_pmax, R.start, R.end,
                                                  B.alloc, J->prof, nb, J->role);
  }
  return PM_SUCCESS;
}

int download_link(cudaStream_t s, const RootsDev& R, const BlocksDev& B,
                  const JoinDev& J, long long nl, int64_t* root_seq_off,
                  int64_t* root_seq, int64_t* root_leaf, int64_t* bwd_off,
                  int64_t* bwd_root, int64_t bwd_cap, int64_t* n_bwd_out,
                  int64_t* n_blocks_out, int64_t* b_inst, int64_t* b_alloc,
                  int64_t* b_size, int64_t* b_free, int32_t* b_role,
                  int64_t* b_prof, int64_t* b_root) {
  *n_bwd_out = J.nbw;
  *n_blocks_out = B.n;
  if (J.nbw > bwd_cap) return perr(PM_ERR_WORKSPACE_TOO_SMALL, "pm_link: bwd_cap");
  int rc = PM_SUCCESS;
  if (!rc && root_seq_off) rc = download(root_seq_off, (const int64_t*)R.rs_off, R.n + 1, s);
  if (!rc && root_seq) rc = download(root_seq, (const int64_t*)R.rs_seq, R.nseq, s);
  if (!rc) rc = download(root_leaf, (const int64_t*)J.root_leaf, R.n, s);
  if (!rc) rc = download(bwd_off, (const int64_t*)J.bw_off, nl + 1, s);
  if (!rc) rc = download(bwd_root, (const int64_t*)J.bw_root, J.nbw, s);
  if (!rc && b_inst) rc = download(b_inst, (const int64_t*)B.inst, B.n, s);
  if (!rc && b_alloc) rc = download(b_alloc, (const int64_t*)B.alloc, B.n, s);
  if (!rc && b_size) rc = download(b_size, (const int64_t*)B.size, B.n, s);
  if (!rc && b_free) rc = download(b_free, (const int64_t*)B.free, B.n, s);
  if (!rc) rc = download(b_role, (const int32_t*)J.role, B.n, s);
  if (!rc) rc = download(b_prof, (const int64_t*)J.prof, B.n, s);
  if (!rc) rc = download(b_root, (const int64_t*)J.broot, B.n, s);
  return rc;
}

}  // namespace

extern "C" {

// a5 / a7 / a8 / a9 / a10 / a11 on one trace.  Inputs (host, event order):
//   ops: n_ops x (start, end, seq[-1 = none]);
//   instants: n_inst x (start, addr, nbytes);
//   leaves (non-wrapper layers in walk order): n_leaves x (start, end).
// Outputs (host, caller-allocated; capacities in brackets):
//   op_root[n_ops], root_op/root_start/root_end[n_ops] (n_roots returned),
//   root_seq_off[n_ops+1], root_seq[n_ops] (sorted unique seqs per root),
//   root_leaf[n_ops] (forward owner, -1), bwd_off[n_leaves+1],
//   bwd_root[bwd_cap] (per leaf, in the reference's order; *n_bwd returned;
//   PM_ERR_WORKSPACE_TOO_SMALL if it exceeds bwd_cap), blocks (n_blocks
//   returned, <= n_inst): b_inst, b_alloc, b_size, b_free (INT64_MIN =
//   None), b_role (0 uncl, 3 gradient, 5 temporary, 6 retained), b_prof
//   (leaf, -1), b_root (owning root, -1).
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
            int64_t* b_prof, int64_t* b_root, void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  Arena A(s);
  RootsDev R;
  BlocksDev B;
  JoinDev J;
  long long* d_ostart = A.upload((const long long*)op_start, n_ops);
  long long* d_oend = A.upload((const long long*)op_end, n_ops);
  long long* d_oseq = A.upload((const long long*)op_seq, n_ops);
  long long* d_op_root = A.alloc<long long>(n_ops);
  long long* d_root_op = A.alloc<long long>(n_ops);
  long long* d_istart = A.upload((const long long*)in_start, n_inst);
  long long* d_iaddr = A.upload((const long long*)in_addr, n_inst);
  long long* d_inb = A.upload((const long long*)in_nbytes, n_inst);
  long long* d_lstart = A.upload((const long long*)l_start, n_leaves);
  long long* d_lend = A.upload((const long long*)l_end, n_leaves);
  PM_TRY(check_arena(A, "pm_link"));
  PM_TRY(stage_roots(A, n_ops, d_ostart, d_oend, d_oseq, &R, d_op_root, d_root_op));
  PM_TRY(stage_group(A, n_inst, d_istart, d_iaddr, d_inb, &B));
  PM_TRY(stage_join(A, R, n_leaves, d_lstart, d_lend, B, &J));
  *n_roots_out = R.n;
  int rc = download(op_root, (const int64_t*)d_op_root, n_ops, s);
  if (!rc) rc = download(root_op, (const int64_t*)d_root_op, R.n, s);
  if (!rc) rc = download(root_start, (const int64_t*)R.start, R.n, s);
  if (!rc) rc = download(root_end, (const int64_t*)R.end, R.n, s);
  if (!rc)
    rc = download_link(s, R, B, J, n_leaves, root_seq_off, root_seq, root_leaf,
                       bwd_off, bwd_root, bwd_cap, n_bwd_out, n_blocks_out,
                       b_inst, b_alloc, b_size, b_free, b_role, b_prof, b_root);
  if (rc) return rc;
  return sync_check(s, "pm_link");
}

// linking.py:126-132 on GIVEN roots (any set, as the reference's link()
// accepts) and given blocks (alloc, free).  Root seqs as CSR
// (root_seq_off[n_roots+1], sorted unique per root).
int pm_link_roots(int64_t n_roots, const int64_t* root_start,
                  const int64_t* root_end, const int64_t* root_seq_off,
                  const int64_t* root_seq, int64_t n_leaves,
                  const int64_t* l_start, const int64_t* l_end,
                  int64_t n_blocks, const int64_t* b_alloc,
                  const int64_t* b_free, int64_t* root_leaf, int64_t* bwd_off,
                  int64_t* bwd_root, int64_t bwd_cap, int64_t* n_bwd_out,
                  int32_t* b_role, int64_t* b_prof, int64_t* b_root,
                  void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  Arena A(s);
  RootsDev R;
  BlocksDev B;
  JoinDev J;
  R.n = n_roots;
  R.start = A.upload((const long long*)root_start, n_roots);
  R.end = A.upload((const long long*)root_end, n_roots);
  R.rs_off = A.upload((const long long*)root_seq_off, n_roots + 1);
  const long long nseq = n_roots > 0 ? root_seq_off[n_roots] : 0;
  R.nseq = nseq;
  R.rs_seq = A.upload((const long long*)root_seq, nseq);
  std::vector<long long> rr(nseq > 0 ? nseq : 1);
  for (long long r = 0; r < n_roots; ++r)
    for (long long k = root_seq_off[r]; k < root_seq_off[r + 1]; ++k) rr[k] = r;
  R.rs_root = A.upload(rr.data(), nseq);
  B.n = n_blocks;
  B.alloc = A.upload((const long long*)b_alloc, n_blocks);
  B.free = A.upload((const long long*)b_free, n_blocks);
  long long* d_lstart = A.upload((const long long*)l_start, n_leaves);
  long long* d_lend = A.upload((const long long*)l_end, n_leaves);
  PM_TRY(check_arena(A, "pm_link_roots"));
  PM_TRY(stage_join(A, R, n_leaves, d_lstart, d_lend, B, &J));
  int64_t nbo = 0;
  int rc = download_link(s, R, B, J, n_leaves, nullptr, nullptr, root_leaf, bwd_off,
                         bwd_root, bwd_cap, n_bwd_out, &nbo, nullptr, nullptr,
                         nullptr, nullptr, b_role, b_prof, b_root);
  if (rc) return rc;
  return sync_check(s, "pm_link_roots");
}

}  // extern "C"

// orchestration and layer-tree cores, their single-trace entry points
// (pm_orchestrate, pm_layer_tree) and the batched pipeline (pm_pipeline_batch)
#include "pipeline_batch.cuh"
