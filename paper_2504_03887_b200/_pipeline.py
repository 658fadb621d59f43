"""ctypes binding of the analysis / link / orchestration kernels
(csrc/pipeline.cu, built into lib/libpeakmem_pipeline.so).  No CPU fallback:
a missing library or device raises EngineUnavailable."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import LIB_DIR, REQ_DTYPE
from .errors import EngineLimitExceeded, EngineUnavailable

LIB_PATH = LIB_DIR / "libpeakmem_pipeline.so"
EXPORTED_SYMBOLS = ("pm_pipeline_last_error", "pm_sort_events", "pm_link",
                    "pm_link_roots", "pm_orchestrate", "pm_layer_tree",
                    "pm_pipeline_batch")
PM_ERR_WORKSPACE_TOO_SMALL = 3
PM_ERR_CYCLIC_PARENT = 5
PM_ERR_ENGINE_LIMIT = 6
PM_ERR_SKIPPED = 7
NONE = np.iinfo(np.int64).min

_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise EngineUnavailable(
                f"{LIB_PATH} is not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(str(LIB_PATH))
        lib.pm_pipeline_last_error.restype = ctypes.c_char_p
        lib.pm_pipeline_last_error.argtypes = []
        for name in EXPORTED_SYMBOLS[1:]:
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(None if a is None else a.ctypes.data)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _check(rc: int, lib) -> None:
    if rc == PM_ERR_ENGINE_LIMIT:
        raise EngineLimitExceeded(lib.pm_pipeline_last_error().decode(errors="replace"))
    if rc != 0:
        msg = lib.pm_pipeline_last_error().decode(errors="replace")
        raise RuntimeError(f"peakmem_b200 pipeline error {rc}: {msg}")


def _stream():
    try:
        import torch
        return torch.cuda.current_stream().cuda_stream
    except Exception:  # pragma: no cover
        return 0


def sort_events(ts: np.ndarray, dur: np.ndarray):
    """Stable device sort by raw ts + fp64 normalization (trace.py:222-236).
    Returns (perm, start, duration) in event-id order."""
    lib = load()
    _native.require_device()
    n = len(ts)
    ts = np.ascontiguousarray(ts, dtype=np.float64)
    dur = np.ascontiguousarray(dur, dtype=np.float64)
    perm = np.empty(n, np.int64)
    start = np.empty(n, np.int64)
    duration = np.empty(n, np.int64)
    _check(lib.pm_sort_events(_p(ts), _p(dur), ctypes.c_int64(n), _p(perm),
                              _p(start), _p(duration),
                              ctypes.c_void_p(_stream())), lib)
    return perm, start, duration


def layer_tree(pid, par, is_layer, start, event_id=None):
    """Device layer tree over python_function frames in event order
    (pm_layer_tree; analysis.py:113-182).  Returns (node_parent,
    child_order, child_off, walk) over the layer frames; raises
    CyclicParentLink like the reference's walk."""
    from .errors import CyclicParentLink
    lib = load()
    _native.require_device()
    pid, par, start = _i64(pid), _i64(par), _i64(start)
    eid = None if event_id is None else _i64(event_id)
    flag = np.ascontiguousarray(is_layer, dtype=np.uint8)
    n = len(pid)
    nl = int(flag.sum())
    node_parent = np.empty(max(nl, 1), np.int64)
    child_order = np.empty(max(nl, 1), np.int64)
    child_off = np.zeros(nl + 2, np.int64)
    walk = np.empty(max(nl, 1), np.int64)
    n_walk = ctypes.c_int64(0)
    rc = lib.pm_layer_tree(ctypes.c_int64(n), _p(pid), _p(par), _p(flag),
                           _p(start), _p(eid), ctypes.c_int64(nl), _p(node_parent),
                           _p(child_order), _p(child_off), _p(walk),
                           ctypes.byref(n_walk), ctypes.c_void_p(_stream()))
    if rc == PM_ERR_CYCLIC_PARENT:
        raise CyclicParentLink(lib.pm_pipeline_last_error().decode(errors="replace"))
    _check(rc, lib)
    return node_parent[:nl], child_order[:nl], child_off, walk[:n_walk.value]


def _check_seq_range(seq, n_ops: int) -> None:
    """The sequence-number join sorts (root << 32 | seq) keys
    (csrc/pipeline.cu k_seq_keys): sequence numbers and root ids must fit in
    32 bits.  The reference keeps unbounded ints, so larger values are an
    engine limit, never a silent truncation."""
    if n_ops >= 1 << 32 or (len(seq) and int(seq.max()) >= 1 << 32):
        raise EngineLimitExceeded(
            "sequence numbers and operator counts must be below 2^32")


class LinkResult:
    """Columnar output of pm_link (see csrc/pipeline.cu)."""


def link(op_start, op_end, op_seq, in_start, in_addr, in_nbytes,
         l_start, l_end) -> LinkResult:
    _check_seq_range(_i64(op_seq), len(op_start))
    lib = load()
    _native.require_device()
    op_start, op_end, op_seq = map(_i64, (op_start, op_end, op_seq))
    in_start, in_addr, in_nbytes = map(_i64, (in_start, in_addr, in_nbytes))
    l_start, l_end = map(_i64, (l_start, l_end))
    no, ni, nl = len(op_start), len(in_start), len(l_start)
    r = LinkResult()
    r.op_root = np.empty(no, np.int64)
    root_op = np.empty(max(no, 1), np.int64)
    root_start = np.empty(max(no, 1), np.int64)
    root_end = np.empty(max(no, 1), np.int64)
    root_seq_off = np.empty(no + 1, np.int64)
    root_seq = np.empty(max(no, 1), np.int64)
    root_leaf = np.empty(max(no, 1), np.int64)
    bwd_off = np.empty(nl + 1, np.int64)
    b_inst = np.empty(max(ni, 1), np.int64)
    b_alloc = np.empty(max(ni, 1), np.int64)
    b_size = np.empty(max(ni, 1), np.int64)
    b_free = np.empty(max(ni, 1), np.int64)
    b_role = np.empty(max(ni, 1), np.int32)
    b_prof = np.empty(max(ni, 1), np.int64)
    b_root = np.empty(max(ni, 1), np.int64)
    n_roots = ctypes.c_int64(0)
    n_bwd = ctypes.c_int64(0)
    n_blocks = ctypes.c_int64(0)
    cap = max(4 * no, 16)
    while True:
        bwd_root = np.empty(cap, np.int64)
        rc = lib.pm_link(
            ctypes.c_int64(no), _p(op_start), _p(op_end), _p(op_seq),
            ctypes.c_int64(ni), _p(in_start), _p(in_addr), _p(in_nbytes),
            ctypes.c_int64(nl), _p(l_start), _p(l_end), _p(r.op_root),
            ctypes.byref(n_roots), _p(root_op), _p(root_start), _p(root_end),
            _p(root_seq_off), _p(root_seq), _p(root_leaf), _p(bwd_off),
            _p(bwd_root), ctypes.c_int64(cap), ctypes.byref(n_bwd),
            ctypes.byref(n_blocks), _p(b_inst), _p(b_alloc), _p(b_size),
            _p(b_free), _p(b_role), _p(b_prof), _p(b_root),
            ctypes.c_void_p(_stream()))
        if rc == 3 and n_bwd.value > cap:  # PM_ERR_WORKSPACE_TOO_SMALL
            cap = n_bwd.value
            continue
        _check(rc, lib)
        break
    nr, nb = n_roots.value, n_blocks.value
    r.n_roots, r.n_blocks = nr, nb
    r.root_op, r.root_start, r.root_end = root_op[:nr], root_start[:nr], root_end[:nr]
    r.root_seq_off = root_seq_off[:nr + 1]
    r.root_seq = root_seq[:int(r.root_seq_off[-1]) if nr else 0]
    r.root_leaf = root_leaf[:nr]
    r.bwd_off = bwd_off
    r.bwd_root = bwd_root[:n_bwd.value]
    r.b_inst, r.b_alloc, r.b_size = b_inst[:nb], b_alloc[:nb], b_size[:nb]
    r.b_free, r.b_role, r.b_prof, r.b_root = (b_free[:nb], b_role[:nb],
                                              b_prof[:nb], b_root[:nb])
    return r


def link_roots(root_start, root_end, root_seq_off, root_seq, l_start, l_end,
               b_alloc, b_free) -> LinkResult:
    """The join on GIVEN roots (linking.py:126-132 with any root set)."""
    _check_seq_range(_i64(root_seq), len(root_start))
    lib = load()
    _native.require_device()
    root_start, root_end, root_seq_off, root_seq = map(
        _i64, (root_start, root_end, root_seq_off, root_seq))
    l_start, l_end, b_alloc, b_free = map(_i64, (l_start, l_end, b_alloc, b_free))
    nr, nl, nb = len(root_start), len(l_start), len(b_alloc)
    r = LinkResult()
    r.root_leaf = np.empty(max(nr, 1), np.int64)
    r.bwd_off = np.empty(nl + 1, np.int64)
    r.b_role = np.empty(max(nb, 1), np.int32)
    r.b_prof = np.empty(max(nb, 1), np.int64)
    r.b_root = np.empty(max(nb, 1), np.int64)
    n_bwd = ctypes.c_int64(0)
    cap = max(4 * nr, 16)
    while True:
        bwd_root = np.empty(cap, np.int64)
        rc = lib.pm_link_roots(
            ctypes.c_int64(nr), _p(root_start), _p(root_end), _p(root_seq_off),
            _p(root_seq), ctypes.c_int64(nl), _p(l_start), _p(l_end),
            ctypes.c_int64(nb), _p(b_alloc), _p(b_free), _p(r.root_leaf),
            _p(r.bwd_off), _p(bwd_root), ctypes.c_int64(cap),
            ctypes.byref(n_bwd), _p(r.b_role), _p(r.b_prof), _p(r.b_root),
            ctypes.c_void_p(_stream()))
        if rc == 3 and n_bwd.value > cap:
            cap = n_bwd.value
            continue
        _check(rc, lib)
        break
    r.root_leaf = r.root_leaf[:nr]
    r.bwd_root = bwd_root[:n_bwd.value]
    r.b_role, r.b_prof, r.b_root = r.b_role[:nb], r.b_prof[:nb], r.b_root[:nb]
    return r


class OrchResult:
    """Ordered request sequence from pm_orchestrate."""


def orchestrate(b_alloc, b_size, b_free, b_role, spans, param_sizes, windows,
                zg, clones, tpl, shift, batch) -> OrchResult:
    """spans: (start, end, iteration) arrays; windows: (start, end) arrays;
    tpl: (start, end); batch: (vts, size, kind, iteration, j) arrays."""
    lib = load()
    _native.require_device()
    b_alloc, b_size, b_free = map(_i64, (b_alloc, b_size, b_free))
    b_role = np.ascontiguousarray(b_role, dtype=np.int32)
    sp_s, sp_e, sp_i = map(_i64, spans)
    param_sizes = _i64(param_sizes)
    w_s, w_e = map(_i64, windows)
    zg = _i64(zg)
    bv, bs, bk, bi, bj = batch
    bv, bs, bi, bj = map(_i64, (bv, bs, bi, bj))
    bk = np.ascontiguousarray(bk, dtype=np.int32)
    nb = len(b_alloc)
    cap = len(param_sizes) * 0 + nb + len(bv) + 2 * nb * (1 + max(clones, 0)) + 16
    o = OrchResult()
    o.raw = np.empty(cap, np.int64)
    o.kind = np.empty(cap, np.int32)
    o.size = np.empty(cap, np.int64)
    o.vts = np.empty(cap, np.int64)
    o.tag = np.empty(cap, np.int32)
    o.a = np.empty(cap, np.int64)
    o.b = np.empty(cap, np.int64)
    o.role = np.empty(cap, np.int32)
    o.packed = np.empty(cap, REQ_DTYPE)
    o.fb_role = np.empty(max(nb, 1), np.int32)
    o.fb_free = np.empty(max(nb, 1), np.int64)
    o.fb_flags = np.empty(max(nb, 1), np.int32)
    n_req = ctypes.c_int64(0)
    n_model = ctypes.c_int64(0)
    _check(lib.pm_orchestrate(
        ctypes.c_int64(nb), _p(b_alloc), _p(b_size), _p(b_free), _p(b_role),
        ctypes.c_int32(len(sp_s)), _p(sp_s), _p(sp_e), _p(sp_i),
        ctypes.c_int32(len(param_sizes)), _p(param_sizes),
        ctypes.c_int32(len(w_s)), _p(w_s), _p(w_e), ctypes.c_int32(len(zg)),
        _p(zg), ctypes.c_int32(clones), ctypes.c_int64(tpl[0]),
        ctypes.c_int64(tpl[1]), ctypes.c_int64(shift),
        ctypes.c_int64(len(bv)), _p(bv), _p(bs), _p(bk), _p(bi), _p(bj),
        ctypes.c_int64(cap), ctypes.byref(n_req), ctypes.byref(n_model),
        _p(o.raw), _p(o.kind), _p(o.size), _p(o.vts), _p(o.tag), _p(o.a),
        _p(o.b), _p(o.role), _p(o.packed), _p(o.fb_role), _p(o.fb_free),
        _p(o.fb_flags), ctypes.c_void_p(_stream())), lib)
    o.n_model = n_model.value
    n = n_req.value
    o.n = n
    if n >= 0:
        for f in ("raw", "kind", "size", "vts", "tag", "a", "b", "role", "packed"):
            setattr(o, f, getattr(o, f)[:n])
    o.fb_role, o.fb_free, o.fb_flags = o.fb_role[:nb], o.fb_free[:nb], o.fb_flags[:nb]
    return o


# ---- the batched, device-resident pipeline (pm_pipeline_batch) -------------

_BATCH_FIELDS = [
    ("n_traces", ctypes.c_int32),
    *[(f, ctypes.c_void_p) for f in (
        "fn_off", "op_off", "in_off",
        "fn_pid", "fn_par", "fn_is_layer", "fn_start", "fn_end",
        "op_start", "op_end", "op_seq", "in_start", "in_addr", "in_nbytes",
        "span_off", "span_start", "span_end", "span_iter", "param_off",
        "param_sizes", "win_off", "win_start", "win_end", "zg_off", "zg",
        "clones", "tpl_start", "tpl_end", "shift", "bat_off", "bat_vts",
        "bat_size", "bat_kind", "bat_it", "bat_j", "skip")],
]


class PipelineBatch(ctypes.Structure):
    """pm_pipeline_batch_t (include/peakmem_pipeline.h)."""

    _fields_ = _BATCH_FIELDS


class PipelineViews(ctypes.Structure):
    """pm_pipeline_views_t (include/peakmem_pipeline.h)."""

    _fields_ = [*[(f, ctypes.c_void_p) for f in (
        "o_raw", "o_kind", "o_size", "o_vts", "o_tag", "o_a", "o_b", "o_role",
        "fb_role", "fb_free")], ("fb_cap", ctypes.c_int64), ("blk_off", ctypes.c_void_p)]


def pipeline_batch(desc: PipelineBatch, d_reqs_ptr: int, req_cap: int,
                   n_traces: int, fb_cap: int | None = None):
    """Run pm_pipeline_batch; the host arrays `desc` points at must stay
    alive for the call.  Returns (req_off, status, n_model, breakdown,
    views) -- views (a dict of host arrays) only when fb_cap is given."""
    lib = load()
    _native.require_device()
    req_off = np.zeros(n_traces + 1, np.int64)
    status = np.zeros(n_traces, np.int32)
    n_model = np.zeros(n_traces, np.int64)
    breakdown = np.zeros((n_traces, 8), np.int64)
    views = None
    vdesc = None
    if fb_cap is not None:
        # device buffers: read back only when a view is asked for
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        cap = max(req_cap, 1)
        i64, i32 = torch.int64, torch.int32
        views = {f: torch.empty(cap, dtype=dt, device=dev) for f, dt in (
            ("raw", i64), ("kind", i32), ("size", i64), ("vts", i64), ("tag", i32),
            ("a", i64), ("b", i64), ("role", i32))}
        views["fb_role"] = torch.empty(max(fb_cap, 1), dtype=i32, device=dev)
        views["fb_free"] = torch.empty(max(fb_cap, 1), dtype=i64, device=dev)
        views["blk_off"] = np.zeros(n_traces + 1, np.int64)
        vdesc = PipelineViews()
        for f in ("raw", "kind", "size", "vts", "tag", "a", "b", "role"):
            setattr(vdesc, "o_" + f, views[f].data_ptr())
        vdesc.fb_role = views["fb_role"].data_ptr()
        vdesc.fb_free = views["fb_free"].data_ptr()
        vdesc.fb_cap = max(fb_cap, 1)
        vdesc.blk_off = views["blk_off"].ctypes.data
    rc = lib.pm_pipeline_batch(ctypes.byref(desc), ctypes.c_void_p(d_reqs_ptr),
                               ctypes.c_int64(req_cap), _p(req_off), _p(status),
                               _p(n_model), _p(breakdown),
                               ctypes.byref(vdesc) if vdesc is not None else None,
                               ctypes.c_void_p(_stream()))
    if rc == PM_ERR_WORKSPACE_TOO_SMALL:
        raise MemoryError(f"pm_pipeline_batch: {int(req_off[-1])} requests > "
                          f"capacity {req_cap}")
    _check(rc, lib)
    return req_off, status, n_model, breakdown, views
