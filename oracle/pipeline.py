"""TEST INFRASTRUCTURE -- CPU restatement of the reference's analysis -> link
-> orchestration path (reference pkg/src/peakmem/{trace,analysis,linking,
orchestration}.py), used as the checker for traces too large or too many to
keep golden vectors for.  Pinned to the reference by
tests/test_oracle_pipeline.py (same goldens the GPU path is held to).

Plain Python over dicts and tuples; each stage cites the reference lines it
restates.  Where the reference is quadratic (link_layers_to_ops,
linking.py:56-64) the restatement probes leaves sorted by start with a
prefix-max bound -- the same answer, verified against the goldens.
"""

from __future__ import annotations

import math
from bisect import bisect_right

LAYER_PREFIX = "nn.Module: "
KNOWN = ("python_function", "cpu_op", "user_annotation", "cpu_instant_event",
         "other")


def normalize(records):
    """trace.py:174-236 -> list of event dicts in event-id order."""
    rows = []
    for rec in records:
        if rec.get("ph") == "M":
            continue
        cat = rec.get("cat")
        cat = cat if cat in KNOWN else "other"
        args = rec.get("args") or {}
        ev = {"cat": cat, "name": str(rec.get("name", ""))}
        if cat == "python_function":
            ev["pid"] = _int(args.get("Python id"))
            ev["parent"] = _int(args.get("Python parent id"))
        elif cat == "cpu_op":
            s = _int(args.get("Sequence number"))
            ev["seq"] = None if s is not None and s < 0 else s
        elif cat == "cpu_instant_event":
            a, b = _int(args.get("Addr")), _int(args.get("Bytes"))
            if a is None or b is None or b == 0:
                continue
            ev["addr"], ev["bytes"] = a, b
        ts = float(rec["ts"])
        rows.append((ts, ts + float(rec.get("dur", 0) or 0), ev))
    t0 = min(r[0] for r in rows)
    order = sorted(range(len(rows)), key=lambda i: (rows[i][0], i))
    out = []
    for eid, i in enumerate(order):
        ts, te, ev = rows[i]
        s = math.floor(ts - t0)
        ev = dict(ev, id=eid, start=s, end=max(s, math.ceil(te - t0)))
        out.append(ev)
    return out


def _int(v):
    return None if v is None else int(v)


def layer_tree(events):
    """analysis.py:115-182 -> nested dict tree; leaves in walk order."""
    funcs = [e for e in events if e["cat"] == "python_function"]
    by_id = {}
    for e in funcs:
        if e["pid"] is not None and e["pid"] not in by_id:
            by_id[e["pid"]] = e

    def anc(e):
        seen = {e["pid"]} if e["pid"] is not None else set()
        cur = e
        while cur["parent"] is not None:
            p = by_id.get(cur["parent"])
            if p is None:
                return None
            if p["pid"] in seen:
                raise ValueError("CyclicParentLink")
            seen.add(p["pid"])
            if p["name"].startswith(LAYER_PREFIX):
                return p
            cur = p
        return None

    nodes = {}
    root = {"name": "<root>", "start": 0, "end": 0, "children": [], "id": -1}
    layers = [e for e in funcs if e["name"].startswith(LAYER_PREFIX)]
    for e in layers:
        nodes[e["id"]] = {"name": e["name"][len(LAYER_PREFIX):], "start": e["start"],
                          "end": e["end"], "children": [], "id": e["id"]}
    for e in layers:
        a = anc(e)
        (nodes[a["id"]] if a else root)["children"].append(nodes[e["id"]])
    for n in list(nodes.values()) + [root]:
        n["children"].sort(key=lambda c: (c["start"], c["id"]))
        n["wrapper"] = bool(n["children"])
    root["wrapper"] = True
    if root["children"]:
        root["start"] = min(c["start"] for c in root["children"])
        root["end"] = max(c["end"] for c in root["children"])
    walk = []

    def rec(n):
        walk.append(n)
        for c in n["children"]:
            rec(c)
    rec(root)
    leaves = [n for n in walk[1:] if not n["wrapper"]]
    return root, leaves


def roots_of(events):
    """analysis.py:185-211"""
    ops = sorted((e for e in events if e["cat"] == "cpu_op"),
                 key=lambda e: (e["start"], -e["end"], e["id"]))
    roots, cur = [], None
    for e in ops:
        if cur is not None and e["start"] < cur["end"] and e["end"] <= cur["end"]:
            if e["seq"] is not None:
                cur["seqs"].add(e["seq"])
            continue
        cur = {"name": e["name"], "start": e["start"], "end": e["end"],
               "seqs": set() if e["seq"] is None else {e["seq"]}}
        roots.append(cur)
    return roots


def markers_of(events):
    """analysis.py:214-249"""
    def kind(n):
        if n.startswith("ProfilerStep"):
            return "profiler_step"
        if "zero_grad" in n:
            return "zero_grad"
        if n.startswith("Optimizer.step") or n.endswith(".step"):
            return "optimizer_step"
        return None
    ann = [(e, kind(e["name"])) for e in events if e["cat"] == "user_annotation"]
    steps = sorted((e for e, k in ann if k == "profiler_step"),
                   key=lambda e: (e["start"], e["id"]))
    if not steps:
        raise ValueError("NoIterationMarkers")
    starts = [e["start"] for e in steps]
    out = [("profiler_step", e["start"], e["end"], i) for i, e in enumerate(steps)]
    for e, k in ann:
        if k in ("zero_grad", "optimizer_step"):
            out.append((k, e["start"], e["end"],
                        max(0, bisect_right(starts, e["start"]) - 1)))
    out.sort(key=lambda m: (m[1], m[0]))
    return out


def blocks_of(events):
    """analysis.py:252-294"""
    open_at, blocks = {}, []
    for e in events:
        if e["cat"] != "cpu_instant_event":
            continue
        if e["bytes"] > 0:
            stale = open_at.pop(e["addr"], None)
            if stale is not None:
                stale["free"] = e["start"]
            b = {"addr": e["addr"], "size": e["bytes"], "alloc": e["start"],
                 "free": None, "role": "unclassified"}
            open_at[e["addr"]] = b
            blocks.append(b)
        else:
            b = open_at.pop(e["addr"], None)
            if b is not None:
                b["free"] = e["start"]
    blocks.sort(key=lambda b: b["alloc"])
    for i, b in enumerate(blocks):
        b["id"] = i
    return blocks


def link(leaves, roots, blocks):
    """linking.py:50-132 (+ gradient candidates of linking.py:40-43)."""
    # innermost containing leaf; ties -> first in walk order
    order = sorted(range(len(leaves)), key=lambda w: leaves[w]["start"])
    lstarts = [leaves[w]["start"] for w in order]
    pmax, m = [], -math.inf
    for w in order:
        m = max(m, leaves[w]["end"])
        pmax.append(m)
    prof = {w: {"fwd": [], "bwd": [], "ret": [], "tmp": []} for w in range(len(leaves))}
    owner = []
    for r, op in enumerate(roots):
        best = None
        i = bisect_right(lstarts, op["start"]) - 1
        while i >= 0 and pmax[i] >= op["end"]:
            w = order[i]
            L = leaves[w]
            if L["end"] >= op["end"]:
                key = (L["end"] - L["start"], w)
                if best is None or key < best:
                    best = key
            i -= 1
        owner.append(None if best is None else best[1])
        if best is not None:
            prof[best[1]]["fwd"].append(r)
    by_seq = {}
    for r, op in enumerate(roots):
        for s in op["seqs"]:
            by_seq.setdefault(s, []).append(r)
    for w, p in prof.items():
        own = set(p["fwd"])
        seqs = sorted(set().union(*[roots[r]["seqs"] for r in p["fwd"]]) if p["fwd"] else ())
        seen, found = set(), []
        for s in seqs:
            for r in by_seq.get(s, []):
                if r in own or r in seen:
                    continue
                seen.add(r)
                found.append(r)
        found.sort(key=lambda r: roots[r]["start"])
        p["bwd"] = found
    owners = sorted(((roots[r]["start"], w, r) for w in range(len(leaves))
                     for r in prof[w]["fwd"] + prof[w]["bwd"]), key=lambda x: x[0])
    starts = [o[0] for o in owners]
    for b in blocks:
        i = bisect_right(starts, b["alloc"]) - 1
        if i < 0:
            continue
        _, w, r = owners[i]
        if not roots[r]["start"] <= b["alloc"] < roots[r]["end"]:
            continue
        if b["free"] is not None and b["free"] < roots[r]["end"]:
            b["role"] = "temporary"
            prof[w]["tmp"].append(b["id"])
        else:
            b["role"] = "retained"
            prof[w]["ret"].append(b["id"])
        b["prof"] = w
    return prof


def gradients(prof, roots, blocks):
    """backward_retained_blocks per profile in walk order (linking.py:40-43)"""
    out = []
    for w in sorted(prof):
        p = prof[w]
        for bid in p["ret"]:
            b = blocks[bid]
            if any(roots[r]["start"] <= b["alloc"] < roots[r]["end"] for r in p["bwd"]):
                out.append(bid)
    return out


def build_sequence(events, side, iterations=2):
    """orchestration.py:237-399 -> list of (kind, block_id, size, vts)."""
    root, leaves = layer_tree(events)
    roots = roots_of(events)
    markers = markers_of(events)
    blocks = blocks_of(events)
    prof = link(leaves, roots, blocks)
    steps = sorted((m for m in markers if m[0] == "profiler_step"), key=lambda m: m[3])
    n = len(steps)
    include = min(iterations, n)
    clones = iterations - include
    windows = []
    for k in range(include):
        s = steps[k][1]
        windows.append((s, steps[k + 1][1] if k + 1 < n else steps[k][2]))
    grads = gradients(prof, roots, blocks)
    for bid in grads:
        blocks[bid]["role"] = "gradient"
    grad_set = set(grads)
    dropped = set()
    psizes = set(side["param_sizes"])
    for kind, s, e, it in markers:
        if kind != "optimizer_step":
            continue
        inspan = [b for b in blocks if s <= b["alloc"] < e]
        if it == 0:
            for b in inspan:
                if b["size"] in psizes and not (b["free"] is not None and b["free"] < e):
                    b["role"] = "optimizer_state"
                    b["free"] = None
            dropped |= {b["id"] for b in inspan if b["role"] != "optimizer_state"}
        else:
            dropped |= {b["id"] for b in inspan}

    def seqd(b):
        return b["role"] != "temporary" and b["id"] not in dropped
    clone_blocks, clone_markers = [], []
    tpl = windows[-1]
    width = tpl[1] - tpl[0]
    if clones:
        template = [b for b in blocks if seqd(b) and b["role"] != "optimizer_state"
                    and tpl[0] <= b["alloc"] < tpl[1]]
        tm = [m for m in markers if m[3] == include - 1 and tpl[0] <= m[1] < tpl[1]]
        for c in range(1, clones + 1):
            sh = width * c
            for b in template:
                clone_blocks.append(dict(b, id=f"clone{c}:{b['id']}", alloc=b["alloc"] + sh,
                                         free=None if b["free"] is None else b["free"] + sh))
            for m in tm:
                clone_markers.append((m[0], m[1] + sh, m[2] + sh, include - 1 + c))
    allm = markers + clone_markers
    zg = sorted(m[1] for m in allm if m[0] == "zero_grad")
    for b in [blocks[i] for i in grads] + [b for b in clone_blocks if b["role"] == "gradient"]:
        i = bisect_right(zg, b["alloc"])
        b["free"] = zg[i] if i < len(zg) else None
    mg = sorted((blocks[i] for i in grad_set
                 if windows[0][0] <= blocks[i]["alloc"] < windows[0][1]),
                key=lambda b: (b["alloc"], b["id"]))
    if not mg:
        raise ValueError("NoGradientBlocks")
    raw = [("alloc", f"model:{i}", sz, i - len(mg))
           for i, sz in enumerate([b["size"] for b in reversed(mg)])]
    st = sorted((m for m in allm if m[0] == "profiler_step" and m[3] < iterations),
                key=lambda m: m[3])
    for m in st:
        for j, sz in enumerate(side["batch_bytes"]):
            raw.append(("alloc", f"batch:{m[3]}:{j}", sz, m[1]))
            raw.append(("free", f"batch:{m[3]}:{j}", sz, m[2]))
    chosen = [b for b in blocks if seqd(b) and (
        b["alloc"] < windows[0][0] or any(w[0] <= b["alloc"] < w[1] for w in windows))]
    for b in chosen + clone_blocks:
        raw.append(("alloc", b["id"], b["size"], b["alloc"]))
        if b["free"] is not None:
            raw.append(("free", b["id"], b["size"], b["free"]))
    ats = {r[1]: r[3] for r in raw if r[0] == "alloc"}

    def key(i):
        k, bid, _, t = raw[i]
        rank = 1 if k == "alloc" else (0 if ats.get(bid, -(1 << 62)) < t else 2)
        return (t, rank, i)
    return [raw[i] for i in sorted(range(len(raw)), key=key)]



def request_digest_rows(seq):
    """Rows the golden request-list digest is taken over."""
    return [[k, b, sz, t] for k, b, sz, t in seq]
