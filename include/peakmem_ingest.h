/*
 * peakmem_ingest.h -- C ABI of the host-side trace reader and config digest
 * of the xMem (arXiv 2504.03887) estimator (csrc/ingest.cpp, plain C++17,
 * lib/libpeakmem_ingest.so).  SURVEY §8f rows f1 (ingest) and f2 (digest).
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/peakmem):
 *   pm_ingest_json .. pm_ingest_free -> trace.parse_trace's read + per-record
 *       rules (trace.py:155-221): json.loads of the file, traceEvents / bare
 *       list root, 'M' records skipped, category mapping, int() of the arg
 *       fields, sequence numbers < 0 -> None, unusable instant events
 *       dropped, EmptyTrace when nothing survives (trace.py:226).  The sort
 *       and floor/ceil normalisation (trace.py:222-236) stay on the GPU
 *       (pm_sort_events, include/peakmem_pipeline.h).
 *   pm_bundle_digest -> PeakMemoryEstimator._digest (estimator.py:189-202):
 *       SHA-256 of json.dumps(payload, sort_keys=True,
 *       separators=(",", ":")) over the bundle's re-serialisation
 *       (trace.py:116-143) and the estimator configuration.
 *
 * The reader accepts a strict subset of what Python's json + the reference
 * rules accept and returns PM_INGEST_UNSUPPORTED for everything else
 * (invalid JSON, strings where numbers belong, int fields outside int64 or
 * equal to INT64_MIN, lone surrogates, strict-mode errors); the caller then
 * runs the Python reader, which restates the reference's exact errors.  On
 * success its columns are identical (bit-exact fp64, int64 with INT64_MIN =
 * None, names) to the Python reader's (tests/test_ingest.py).
 */
#ifndef PEAKMEM_INGEST_H
#define PEAKMEM_INGEST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM_INGEST_UNSUPPORTED 5
#define PM_INGEST_EMPTY 7

const char* pm_ingest_last_error(void);

/* Parse `len` bytes of UTF-8 JSON.  0: *handle holds the columns (free with
 * pm_ingest_free); PM_INGEST_UNSUPPORTED; PM_INGEST_EMPTY (no events). */
int pm_ingest_json(const char* text, int64_t len, int strict, void** handle);

int64_t pm_ingest_count(void* handle);       /* events kept, file order     */
int64_t pm_ingest_dropped(void* handle);     /* unusable instants dropped   */
int64_t pm_ingest_n_names(void* handle);     /* distinct event names        */
int64_t pm_ingest_names_bytes(void* handle); /* UTF-8 bytes of those names  */

/* ts/dur: raw fp64 (n); cat: int8 code of EventCategory order (n); ints:
 * 7 x n field-major (python id, parent id, sequence number, addr, bytes,
 * total allocated, total reserved); name_id: n indices into the table of
 * distinct names, given as n_names+1 CODE-POINT offsets into `names`
 * (UTF-8, pm_ingest_names_bytes bytes). */
void pm_ingest_columns(void* handle, double* ts, double* dur, int8_t* cat,
                       int64_t* ints, int32_t* name_id, int64_t* name_off,
                       char* names);

void pm_ingest_free(void* handle);

/* Columns in event-id order (after the sort); name_id (n) indexes a table
 * of n_names names given as a UTF-8 blob with n_names+1 BYTE offsets; ints
 * as above; sidecar_present 0 -> "sidecar": null;
 * max_split < 0 -> null.  Writes 64 hex chars + NUL to hex_out. */
int pm_bundle_digest(int64_t n, const int8_t* cat, const int64_t* start,
                     const int64_t* dur, const int64_t* ints,
                     const int32_t* name_id, int64_t n_names,
                     const char* names, const int64_t* name_off,
                     int sidecar_present, const int64_t* param_sizes,
                     int64_t n_param, const int64_t* batch_bytes,
                     int64_t n_batch, const char* optimizer, int64_t opt_len,
                     int64_t sc_capacity, int64_t sc_initial,
                     int64_t iterations, int64_t device_capacity,
                     int64_t initial_memory, int64_t max_split, char* hex_out);

#ifdef __cplusplus
}
#endif

#endif /* PEAKMEM_INGEST_H */
