"""ctypes binding of the native trace reader and config digest
(csrc/ingest.cpp, lib/libpeakmem_ingest.so; host C++)."""

from __future__ import annotations

import ctypes

import numpy as np

from ._native import LIB_DIR
from .errors import EngineUnavailable

LIB_PATH = LIB_DIR / "libpeakmem_ingest.so"
EXPORTED_SYMBOLS = ("pm_ingest_last_error", "pm_ingest_json", "pm_ingest_count",
                    "pm_ingest_dropped", "pm_ingest_n_names", "pm_ingest_names_bytes",
                    "pm_ingest_columns", "pm_ingest_free", "pm_bundle_digest")
UNSUPPORTED, EMPTY = 5, 7
_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise EngineUnavailable(f"{LIB_PATH} is not built")
        lib = ctypes.CDLL(str(LIB_PATH))
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        lib.pm_ingest_json.restype = ctypes.c_int
        lib.pm_ingest_json.argtypes = [vp, i64, ctypes.c_int,
                                       ctypes.POINTER(vp)]
        for f in ("pm_ingest_count", "pm_ingest_dropped", "pm_ingest_n_names",
                  "pm_ingest_names_bytes"):
            getattr(lib, f).restype = i64
            getattr(lib, f).argtypes = [vp]
        lib.pm_ingest_columns.restype = None
        lib.pm_ingest_columns.argtypes = [vp] * 8
        lib.pm_ingest_free.restype = None
        lib.pm_ingest_free.argtypes = [vp]
        lib.pm_bundle_digest.restype = ctypes.c_int
        lib.pm_bundle_digest.argtypes = (
            [i64, vp, vp, vp, vp, vp, i64, ctypes.c_char_p, vp, ctypes.c_int, vp, i64, vp,
             i64, ctypes.c_char_p, i64, i64, i64, i64, i64, i64, i64,
             ctypes.c_char_p])
        _lib = lib
    return _lib


def parse_json(data: bytes, strict: bool):
    """-> (ts, dur, cat, ints[7, n], names NameColumn, dropped) or
    UNSUPPORTED / EMPTY (int)."""
    from .trace import NameColumn
    lib = load()
    h = ctypes.c_void_p()
    # any contiguous buffer (bytes, a read-only mmap of the file)
    buf = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    rc = lib.pm_ingest_json(ctypes.c_void_p(buf.ctypes.data), len(data),
                            1 if strict else 0, ctypes.byref(h))
    if rc != 0:
        return rc
    try:
        n = lib.pm_ingest_count(h)
        nn = lib.pm_ingest_n_names(h)
        nb = lib.pm_ingest_names_bytes(h)
        ts = np.empty(n, np.float64)
        dur = np.empty(n, np.float64)
        cat = np.empty(n, np.int8)
        ints = np.empty((7, n), np.int64)
        ids = np.empty(n, np.int32)
        off = np.empty(nn + 1, np.int64)
        blob = ctypes.create_string_buffer(max(nb, 1))
        lib.pm_ingest_columns(h, ts.ctypes.data, dur.ctypes.data, cat.ctypes.data,
                              ints.ctypes.data, ids.ctypes.data, off.ctypes.data,
                              blob)
        text = blob.raw[:nb].decode("utf-8")
        o = off.tolist()
        table = [text[o[i]:o[i + 1]] for i in range(nn)]
        return ts, dur, cat, ints, NameColumn(table, ids), lib.pm_ingest_dropped(h)
    finally:
        lib.pm_ingest_free(h)


def bundle_digest(bundle, sidecar, iterations, capacity, initial, max_split) -> str:
    """SHA-256 of the estimator payload (estimator.py:189-202), natively."""
    lib = load()
    from .trace import NameColumn
    col = NameColumn.of(bundle.names)
    tab = [t.encode("utf-8") for t in col.table]
    off = np.zeros(len(tab) + 1, np.int64)
    np.cumsum([len(t) for t in tab], out=off[1:])
    blob = b"".join(tab)
    ids = np.ascontiguousarray(col.ids, np.int32)
    keys = ("python_id", "parent_id", "sequence_number", "addr", "nbytes",
            "total_allocated", "total_reserved")
    ints = np.ascontiguousarray(np.stack([bundle.ints[k] for k in keys]), np.int64)
    cat = np.ascontiguousarray(bundle.category, np.int8)
    start = np.ascontiguousarray(bundle.start, np.int64)
    dur = np.ascontiguousarray(bundle.duration, np.int64)
    if sidecar is not None:
        ps = np.asarray(sidecar.param_sizes, np.int64)
        bb = np.asarray(sidecar.batch_bytes, np.int64)
        opt = sidecar.optimizer_name.encode("utf-8")
        scap, sini = sidecar.device_capacity, sidecar.initial_memory
    else:
        ps = bb = np.zeros(0, np.int64)
        opt, scap, sini = b"", 0, 0
    out = ctypes.create_string_buffer(65)
    lib.pm_bundle_digest(len(start), cat.ctypes.data, start.ctypes.data,
                         dur.ctypes.data, ints.ctypes.data, ids.ctypes.data,
                         len(tab), blob, off.ctypes.data,
                         1 if sidecar is not None else 0, ps.ctypes.data, len(ps),
                         bb.ctypes.data, len(bb), opt, len(opt), scap, sini,
                         iterations, capacity, initial,
                         -1 if max_split is None else max_split, out)
    return out.value.decode()
