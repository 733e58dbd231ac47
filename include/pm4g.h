/* ============================================================================
 * pm4g.h -- C ABI of libpm4g, the B200-native hot path of PM4Py-GPU
 *           (Berti, Phan Nghia, van der Aalst, arXiv 2204.04898).
 *
 * Citations: P:<line> = PAPER.md, S:<line> = SPEC.md (see DESIGN.md §2 for the
 * readings R1..R19 taken where the paper is silent).
 *
 * Conventions (all entry points)
 *   - Every function returns a pm4g_status.  On failure, pm4g_last_error()
 *     returns a thread-local, human-readable message; outputs are untouched or
 *     partially written and must not be used.
 *   - Device pointers are CUDA global-memory pointers on the current device;
 *     host pointers are ordinary (preferably pinned) host memory.  Each
 *     argument says which.  No torch types cross this boundary.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All work is enqueued asynchronously on it.  Calls that must
 *     return a host-side size synchronise the stream; they say so.
 *   - Ownership: the library owns pm4g_log, pm4g_variant_table and pm4g_comm
 *     objects and the device memory behind them (freed by *_destroy).  Input
 *     columns are copied unless PM4G_BORROW is set, in which case the caller
 *     keeps them alive and unchanged until the log is destroyed or sorted.
 *     Fixed-size outputs (A*A tables, A vectors, per-case arrays) go into
 *     caller-allocated device buffers.
 *   - Logs are immutable except for pm4g_sort, which moves a log from
 *     the "ingested" to the "formatted" state in place (idempotent).
 *     Filters return a new log in the state of their input.
 *   - Empty inputs are valid everywhere: an empty log yields zero tables, zero
 *     cases and zero variants.
 * ========================================================================== */
#ifndef PM4G_H
#define PM4G_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pm4g_status {
    PM4G_OK = 0,
    PM4G_EINVAL = 1,     /* bad argument or call order (e.g. t1 > t2; log not sorted) */
    PM4G_EDATA = 2,      /* validation failure: code out of range / length mismatch */
    PM4G_ENOMEM = 3,     /* device or host allocation failed */
    PM4G_ECUDA = 4,      /* a CUDA runtime error (message carries cudaGetErrorString) */
    PM4G_ENCCL = 5,      /* an NCCL error, or NCCL could not be loaded */
    PM4G_EKEYWIDTH = 6,  /* reserved, no longer returned: logs whose case_bits + ts_bits > 64
                            take the wide path of pm4g_sort */
    PM4G_ECOLLISION = 7  /* reserved, never returned: variant-key collisions (local or across
                            ranks) are always resolved exactly by verification + re-keying */
} pm4g_status;

typedef void* pm4g_stream_t; /* cudaStream_t */

typedef struct pm4g_log pm4g_log;
typedef struct pm4g_variant_table pm4g_variant_table;
typedef struct pm4g_comm pm4g_comm;

/* ---------------------------------------------------------------- log create
 * P:93 "we assume an event log to be ingested ... into a dataframe"; the
 * columnar, dictionary-encoded table of S:27-47 (EventTable): case code u32,
 * activity code u8/u16/u32, timestamp int64 (ms since epoch, R3; may be
 * negative, R4).  Rows are in ingest order; that order is the tie-break (R2).
 */
enum {
    PM4G_BORROW = 1u << 0,      /* reference the device columns zero-copy */
    PM4G_HOST_INPUT = 1u << 1,  /* columns are HOST pointers: copied H2D on `stream` */
    PM4G_SORTED_HINT = 1u << 2  /* reserved (ignored) */
};

enum { PM4G_KIND_CODES = 0, PM4G_KIND_I64 = 1, PM4G_KIND_F64 = 2 };

/* An extra attribute column: u32 dictionary codes, int64 or f64,
 * with an optional validity mask (u8 per row, 1 = present; NULL = no nulls). */
typedef struct pm4g_column {
    int32_t kind;          /* PM4G_KIND_* */
    const void* data;      /* [n_events], device (host with PM4G_HOST_INPUT) */
    const uint8_t* valid;  /* [n_events] or NULL */
    uint64_t dict_size;    /* for PM4G_KIND_CODES: codes must be < dict_size */
} pm4g_column;

typedef struct pm4g_log_desc {
    int64_t n_events;          /* rows (>= 0) */
    const uint32_t* case_code; /* [n_events] case dictionary codes */
    const void* act;           /* [n_events] activity codes, act_bytes wide */
    int32_t act_bytes;         /* 1, 2 or 4 */
    const int64_t* ts;         /* [n_events] timestamps */
    uint64_t n_case_codes;     /* global case dictionary size (codes < this) */
    uint32_t case_lo;          /* this shard's case range [case_lo, case_hi) (R19); */
    uint32_t case_hi;          /*   case_hi == 0 means "up to n_case_codes" */
    uint32_t n_activities;     /* activity dictionary size A (codes < A), A >= 1 */
    int32_t n_extra;           /* number of extra attribute columns */
    const pm4g_column* extra;  /* [n_extra] host array of column descriptors */
    uint32_t flags;            /* PM4G_BORROW | PM4G_HOST_INPUT */
} pm4g_log_desc;

/* Validates (every case code in [case_lo, case_hi) and < n_case_codes,
 * every activity code < n_activities, extra codes < dict_size; first violation
 * -> PM4G_EDATA with the row in the message) and computes the metadata the key
 * build needs (ts_min, ts_max, key bit widths).  Synchronises `stream` once.
 * *out receives a new log in the "ingested" state. */
pm4g_status pm4g_log_create(const pm4g_log_desc* desc, pm4g_stream_t stream, pm4g_log** out);
/* pm4g_log_create followed by pm4g_filter_time(.., PM4G_TIME_EVENTS) (P:126,
 * keep rows with t1 <= ts <= t2, inclusive) in ONE pass over the
 * columns: every row is validated as pm4g_log_create does (same errors), while
 * the metadata and the radix histograms cover the kept rows only, and the
 * returned log is the lazily filtered one (pm4g_sort's first radix pass keeps
 * the rows in range; see pm4g_filter_time).  With extra columns it is exactly
 * the two calls.  EINVAL if t1 > t2.  Synchronises `stream` once. */
pm4g_status pm4g_log_create_filtered(const pm4g_log_desc* desc, int64_t t1, int64_t t2, pm4g_stream_t stream,
                                     pm4g_log** out);
pm4g_status pm4g_log_destroy(pm4g_log* log);

typedef struct pm4g_log_info {
    int64_t n_events;
    int64_t n_cases;        /* non-empty cases (R15); -1 until sorted */
    int32_t sorted;         /* 1 in the "formatted" state */
    int32_t act_bytes;
    uint32_t n_activities;
    uint32_t case_lo, case_hi;
    int64_t ts_min, ts_max; /* over the log's rows (0, -1 when empty) */
    int32_t case_bits, ts_bits, key_bits, radix_passes;
} pm4g_log_info;
pm4g_status pm4g_log_info_get(const pm4g_log* log, pm4g_log_info* info);

/* ---------------------------------------------------------------- format (sort)
 * P:108 "The dataframe is ordered based on three criteria (in order, case
 * identifier, the timestamp, and the absolute index of the event)".
 * Stable LSD radix sort of the composite key ((case - case_lo) << ts_bits) |
 * (ts - ts_min) with the activity (and a row index when extra columns exist) as
 * payload; stability realises the third criterion (R2).  Then materialises the
 * case segments (the cases dataframe's row ranges).
 * Idempotent.  Wide path (case_bits + ts_bits > 64, e.g.
 * microsecond timestamps over years with millions of cases; S:39 fixes
 * timestamps as full signed 64-bit): the key is ts - ts_min alone (up to 64
 * bits), the radix passes take their case digits from the case column through
 * the ingest-row payload, and the formatted log keeps each row's case beside
 * it; every output is identical to the narrow path's definition.
 * Synchronises `stream` once: the host learns whether any case needs the exact
 * fallback (cases longer than 1024 rows, or running > 512 rows past a 4096-row
 * tile; they are then sorted by one batched segmented radix sort, one more
 * round trip).  This is a deliberate deviation from SURVEY.md 8(b), which lets
 * only log_create and variants synchronise; pm4g_sort_analyze folds this check
 * into the analysis' own synchronisation instead. */
pm4g_status pm4g_sort(pm4g_log* log, pm4g_stream_t stream);

/* The formatted log, decoded into caller device buffers (each [n_events], any
 * may be NULL): case codes, activity codes widened to u32 and timestamps.
 * Requires the sorted state (else EINVAL). */
pm4g_status pm4g_sorted_columns(const pm4g_log* log, uint32_t* case_code, uint32_t* act,
                                int64_t* ts, pm4g_stream_t stream);

/* ---------------------------------------------------------------- aggregates
 * All require the sorted state (EINVAL otherwise).  The A x A tables also
 * require A * A < 2^32 (edge ids are 32-bit; EINVAL otherwise).  With comm != NULL the
 * tables are summed over all ranks (NCCL allreduce, exact in integers)
 * and every rank receives the global result. */

/* Directly-follows graph ("calculating the frequency/performance
 * directly-follows graph").  For every pair of
 * consecutive rows i, i+1 of the same case: cnt[a_i * A + a_{i+1}] += 1 and
 * dur_sum[..] += ts_{i+1} - ts_i (R5, int64 modulo 2^64, R8).  mean[k] =
 * (double)dur_sum[k] / (double)cnt[k] for cnt[k] > 0, else 0.0 (R6).
 * cnt, dur_sum: device [A*A] (required); mean: device [A*A] or NULL. */
pm4g_status pm4g_dfg(const pm4g_log* log, uint64_t* cnt, int64_t* dur_sum, double* mean,
                     pm4g_comm* comm, pm4g_stream_t stream);

/* Performance-DFG extremes: for
 * every edge, dur_min[k] / dur_max[k] = the smallest / largest pair duration
 * ts_{i+1} - ts_i over its occurrences, as u64 (exact: 0 <= difference < 2^64
 * after the sort, R20); 0 where cnt[k] = 0.  With comm: min / max over ranks
 * (NCCL allreduce with ncclMin / ncclMax).  dur_min, dur_max: device [A*A]
 * (one may be NULL). */
pm4g_status pm4g_dfg_minmax(const pm4g_log* log, uint64_t* dur_min, uint64_t* dur_max,
                            pm4g_comm* comm, pm4g_stream_t stream);

/* Eventually-follows graph + temporal profile (P:122
 * "discovers the eventually-follows graphs or the temporal profile";
 * S:284-291; reading R22).  For every case and every ordered row
 * pair i < j inside it (O(sum m^2) pairs): cnt[a_i * A + a_j] += 1,
 * dur_sum[..] += d (u64, modulo 2^64), dur_sumsq += d^2 as an exact unsigned
 * 128-bit value, d = ts_j - ts_i >= 0.  dur_sumsq is [2*A*A]: low words at
 * [0, A*A), high words at [A*A, 2*A*A).  mean = dur_sum / cnt and the
 * population stdev per R22 (fp64, identical formula to the oracle's); 0 where
 * cnt = 0.  Any output may be NULL (at least one required).  With comm: summed
 * over ranks (the 128-bit words as four 32-bit limbs, exact). */
pm4g_status pm4g_efg(const pm4g_log* log, uint64_t* cnt, uint64_t* dur_sum, uint64_t* dur_sumsq,
                     double* mean, double* stdev, pm4g_comm* comm, pm4g_stream_t stream);

/* Start / end activities: start[a] = number of cases whose
 * first formatted row has activity a; end[a] likewise for the last row.
 * Sum start = sum end = n_cases.  start, end: device [A]. */
pm4g_status pm4g_start_end(const pm4g_log* log, uint64_t* start, uint64_t* end, pm4g_comm* comm,
                           pm4g_stream_t stream);

/* Cases dataframe ("the number of events for the case, the
 * throughput time of the case"): one row per non-empty case of this
 * shard in ascending case code (R1, R15): case_code, n_events, dur = last ts -
 * first ts (R9).  Arrays are device [capacity]; capacity must be >= n_cases
 * (pm4g_log_info_get) else EINVAL.  *n_cases_out (host, may be NULL) receives
 * n_cases.  Any output pointer may be NULL.  Local to the shard (no comm). */
pm4g_status pm4g_case_durations(const pm4g_log* log, uint32_t* case_code, uint32_t* n_events,
                                int64_t* dur, uint64_t capacity, uint64_t* n_cases_out,
                                pm4g_stream_t stream);

/* Variants ("This requires a double aggregation: first, the events
 * need to be grouped in cases. Then this grouping is used to aggregate the
 * cases into the variants").  A variant is the exact
 * activity sequence of a case (R10).  Cases are hashed (two 64-bit polynomial
 * hashes + length), group-counted in a device hash table, and every case is
 * verified against its variant's representative sequence; a hash collision is
 * resolved exactly by re-keying the mismatching cases.  Output order: count
 * descending, then representative (= smallest) case code ascending (R11).
 * Synchronises `stream` (the result size is a host value).  With comm the
 * per-rank tables are all-gathered and merged; every rank gets the global
 * table. */
pm4g_status pm4g_variants(const pm4g_log* log, pm4g_comm* comm, pm4g_stream_t stream,
                          pm4g_variant_table** out);
/* n_variants and the total length of all variant sequences (host outputs). */
pm4g_status pm4g_variants_size(const pm4g_variant_table* v, uint64_t* n_variants, uint64_t* total_len);
/* Copies the table into caller device buffers (any may be NULL): count[V],
 * len[V], rep_case[V] (case code), seq_off[V+1] (exclusive offsets into
 * seq_act), seq_act[total_len] (activity codes as u32). */
pm4g_status pm4g_variants_get(const pm4g_variant_table* v, uint64_t* count, uint32_t* len,
                              uint32_t* rep_case, uint64_t* seq_off, uint32_t* seq_act,
                              pm4g_stream_t stream);
/* case_variant[n_cases] (device): index into the output order of the variant
 * of each local case (ascending case code); "case_to_variant". */
pm4g_status pm4g_variants_case_index(const pm4g_variant_table* v, uint32_t* case_variant,
                                     pm4g_stream_t stream);
pm4g_status pm4g_variants_destroy(pm4g_variant_table* v);

/* Upper bound on n_cases known on the host without waiting for the device:
 * min(n_events, case_max - case_min + 1) (0 for an empty log).  Any state. */
pm4g_status pm4g_case_capacity(const pm4g_log* log, uint64_t* capacity);

/* Fused pass: one read of the formatted log produces every requested output
 * (each pointer may be NULL to skip it; variants == NULL skips variants).
 * Same semantics as the separate calls above.  With capacity >=
 * pm4g_case_capacity the call does not wait for the case count (entries past
 * n_cases are left untouched); otherwise it synchronises to check it. */
typedef struct pm4g_outputs {
    uint64_t* cnt;        /* [A*A] device */
    int64_t* dur_sum;     /* [A*A] device */
    double* mean;         /* [A*A] device */
    uint64_t* start;      /* [A]   device */
    uint64_t* end;        /* [A]   device */
    uint32_t* case_code;  /* [capacity] device */
    uint32_t* n_events;   /* [capacity] device */
    int64_t* dur;         /* [capacity] device */
    uint64_t capacity;
    pm4g_variant_table** variants; /* host out-pointer */
    uint64_t* dur_min;    /* [A*A] device, optional (NEXT-2, see pm4g_dfg_minmax) */
    uint64_t* dur_max;    /* [A*A] device, optional */
} pm4g_outputs;
pm4g_status pm4g_analyze(const pm4g_log* log, const pm4g_outputs* out, pm4g_comm* comm,
                         pm4g_stream_t stream);

/* pm4g_sort then pm4g_analyze (format.apply, then the aggregates) in
 * one call, with identical results.  The sort's host check for cases the
 * in-shared-memory ranking cannot take (longer than 1024 rows, or running far
 * past a tile; S:184-192 still holds for them via an exact radix sort) is
 * folded into the analysis' own synchronisation instead of costing a separate
 * round trip: if such cases exist, they are sorted exactly and the analysis is
 * recomputed before the call returns.  Falls back to the two separate calls
 * when comm != NULL, when no variants are requested (no synchronisation to
 * share), or when the log has extra columns.  An already formatted log is only
 * analysed.  Errors: those of pm4g_sort and pm4g_analyze.
 * CUDA graphs (opt-in, environment PM4G_GRAPH=1, read once per process): the
 * launches between the call's host round trips are captured from `stream` and
 * run as one graph per segment; the executable graphs are kept per (device,
 * stream, segment) and updated in place by later calls of the same shape
 * (another shape re-instantiates them).  Results are identical.  `stream` must
 * be capturable: on the legacy default stream the call runs eagerly. */
pm4g_status pm4g_sort_analyze(pm4g_log* log, const pm4g_outputs* out, pm4g_comm* comm,
                              pm4g_stream_t stream);

/* ---------------------------------------------------------------- filters
 * Return a NEW log (in the state -- ingested or formatted -- of `in`) holding
 * the kept rows in their original relative order.  Kept cases keep
 * their codes; cases left empty disappear (R15). */
enum { PM4G_TIME_EVENTS = 0, PM4G_TIME_CASES_CONTAINED = 1, PM4G_TIME_CASES_INTERSECTING = 2 };

/* P:126 "three different types of timestamp filtering (events, cases
 * contained, cases intersecting)".  Bounds inclusive (R12).
 * EVENTS: keep rows with t1 <= ts <= t2 (cases may become partial; adjacency
 * is re-derived by the next format, R13).  CASES_CONTAINED: keep every row of
 * cases with first ts >= t1 and last ts <= t2.  CASES_INTERSECTING: keep every
 * row of cases with first ts <= t2 and last ts >= t1.  EINVAL if t1 > t2.
 * EVENTS on an ingested (unsorted) log without extra columns is LAZY (SURVEY.md
 * 8(a) A1 "fused with A2 when unsorted"): one scan of the case / ts columns
 * counts the kept rows and builds their metadata; the new log shares `in`'s
 * columns (kept alive past pm4g_log_destroy(in); borrowed columns must stay
 * valid until the new log is sorted) and pm4g_sort's first radix pass keeps
 * the rows in range while it builds the composite key.  Any other consumer of
 * the new log (filters, partition, concat, repartition) first compacts it.
 * Every filter synchronises `stream` once (the kept-row count). */
pm4g_status pm4g_filter_time(const pm4g_log* in, int64_t t1, int64_t t2, int32_t mode,
                             pm4g_stream_t stream, pm4g_log** out);

/* Whole-case filters on a FORMATTED log (P:98-103,
 * P:121-127; reading R21).  A case matches on its
 * formatted rows:
 *   START_IN / END_IN: its first / last activity is in codes[0..n_codes)
 *                      (codes >= A never match);
 *   SIZE:              lo <= n_events <= hi;
 *   THROUGHPUT:        lo <= last ts - first ts <= hi;
 *   PATHS:             some consecutive pair (a_k, a_{k+1}) equals one of the
 *                      pairs (codes[2j], codes[2j+1]).
 * Every row of the case is kept iff match == (keep != 0) (keep / remove mode,
 * S:465).  codes: HOST array.  EINVAL: unsorted input, lo > hi, odd
 * n_codes for PATHS, bad kind.  Returns a new formatted log. */
enum { PM4G_CASE_START_IN = 0, PM4G_CASE_END_IN = 1, PM4G_CASE_SIZE = 2, PM4G_CASE_THROUGHPUT = 3,
       PM4G_CASE_PATHS = 4 };
typedef struct pm4g_case_pred {
    int32_t kind;              /* PM4G_CASE_* */
    const uint32_t* codes;     /* host: activity codes, or flattened (a, b) pairs */
    int64_t n_codes;
    int64_t lo, hi;            /* SIZE / THROUGHPUT bounds, inclusive */
} pm4g_case_pred;
pm4g_status pm4g_filter_cases(const pm4g_log* in, const pm4g_case_pred* pred, int32_t keep,
                              pm4g_stream_t stream, pm4g_log** out);

/* filter_by_variants ("keeps/remove all the cases whose variant fall
 * inside the collection"): a case matches iff its exact activity
 * sequence equals one of the n_seqs sequences given in HOST CSR form
 * (seq_off[n_seqs + 1] ascending, seq_act[seq_off[n_seqs]]); unknown or empty
 * sequences never match.  Rows kept iff match == (keep != 0).  Formatted
 * input required (EINVAL otherwise).  Returns a new formatted log. */
pm4g_status pm4g_filter_variants(const pm4g_log* in, const uint64_t* seq_off, const uint32_t* seq_act,
                                 int64_t n_seqs, int32_t keep, pm4g_stream_t stream, pm4g_log** out);

enum { PM4G_COL_ACTIVITY = -1 };
enum { PM4G_PRED_IN_SET = 0, PM4G_PRED_RANGE_I64 = 1, PM4G_PRED_RANGE_F64 = 2 };
enum { PM4G_LEVEL_EVENTS = 0, PM4G_LEVEL_CASES = 1 };

typedef struct pm4g_pred {
    int32_t kind;           /* PM4G_PRED_* (must match the column kind, else EINVAL) */
    const uint32_t* codes;  /* IN_SET: HOST array of codes */
    int64_t n_codes;
    int64_t lo_i, hi_i;     /* RANGE_I64: inclusive, lo <= hi */
    double lo_f, hi_f;      /* RANGE_F64: inclusive, lo <= hi */
} pm4g_pred;

/* P:96-97 ("filtering the events/rows for which the cost is > 1000")
 * ("filtering the cases with at least one event with activity ..."), P:128;
 * S:445-453.  column = PM4G_COL_ACTIVITY or an extra-column index.  A row
 * matches if its value satisfies the predicate; nulls never match (R14).
 * level EVENTS: keep rows with match == keep.  level CASES: keep every row of
 * cases with (>= 1 matching row) == keep. */
pm4g_status pm4g_filter_attr(const pm4g_log* in, int32_t column, const pm4g_pred* pred,
                             int32_t level, int32_t keep, pm4g_stream_t stream, pm4g_log** out);

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU; the log is sharded by contiguous case-code ranges (R19,
 * S:228-231) so no case crosses a shard.  The communicator is an NCCL
 * communicator owned by the library; the caller only transports the unique id
 * (e.g. torch.distributed broadcast).  NCCL is loaded on first use
 * (PM4G_ENCCL if unavailable). */
pm4g_status pm4g_comm_unique_id(void* id_out, size_t* id_bytes); /* id_out: host, >= 128 B */
pm4g_status pm4g_comm_create(const void* id, int32_t nranks, int32_t rank, pm4g_comm** out);
pm4g_status pm4g_comm_destroy(pm4g_comm* comm);

/* ---------------------------------------------------------------- global repartition (NEXT-4)
 * a single unsorted global table, ingested in arbitrary
 * row slices on the ranks (the log as a columnar table), is moved so
 * that rank r holds exactly the rows with bounds[r] <= case < bounds[r + 1]
 * (contiguous case ranges, R19).  Rows arrive in (source rank, row)
 * order, so the destination's ingest order is the global table's order
 * restricted to its cases (the stable tie-break of R2 is preserved).
 * bounds: HOST u32[nranks + 1], ascending, covering every case code of the
 * input (EINVAL otherwise), bounds[nranks] <= n_case_codes.  `in` must be
 * ingested (not sorted).  Every column (activity, timestamp, extra columns) is
 * exchanged with grouped ncclSend / ncclRecv; the result is a new ingested
 * log with case range [bounds[rank], bounds[rank + 1]), validated. */
pm4g_status pm4g_repartition(const pm4g_log* in, const uint32_t* bounds, pm4g_comm* comm,
                             pm4g_stream_t stream, pm4g_log** out);
/* The same data movement on one device: parts[r] (r < n_parts) receives the
 * rows of `in` with bounds[r] <= case < bounds[r + 1], in their original order
 * (a stable split), as a new ingested log with case range [bounds[r],
 * bounds[r + 1]).  parts: host array of n_parts out-pointers. */
pm4g_status pm4g_partition_by_case(const pm4g_log* in, const uint32_t* bounds, int32_t n_parts,
                                   pm4g_stream_t stream, pm4g_log** parts);
/* Concatenation of ingested logs (same activity dictionary and columns) in the
 * given order -- what a rank holds after the exchange -- as a new ingested log
 * with case range [case_lo, case_hi), validated. */
pm4g_status pm4g_log_concat(const pm4g_log* const* logs, int32_t n_logs, uint32_t case_lo, uint32_t case_hi,
                            pm4g_stream_t stream, pm4g_log** out);

/* Loopback merge for R shards held by ONE process on one device (the
 * fake-collective used to test the merge logic without NCCL): combines the
 * per-shard variant tables exactly as the NCCL path does after its allgather.
 * parts: host array of R variant tables computed on disjoint case ranges.
 * local_part in [0, R): the merged table also carries the case -> variant
 * index (pm4g_variants_case_index) of that part's cases, in the merged order --
 * what every rank gets for its own cases from the NCCL path; -1: none. */
pm4g_status pm4g_variants_merge(const pm4g_variant_table* const* parts, int32_t n_parts, int32_t local_part,
                                pm4g_stream_t stream, pm4g_variant_table** out);
/* Loopback sum of R packed integer tables (device [R][len] u64 -> [len]):
 * the reduction C1 performs over NVLink, for fake-collective tests. */
pm4g_status pm4g_sum_u64(const uint64_t* parts, int32_t n_parts, uint64_t len, uint64_t* out,
                         pm4g_stream_t stream);
/* Per-shard DFG/start/end partial tables packed as [cnt A*A | sum A*A |
 * start A | end A] (device, u64) -- the exact payload C1 allreduces -- and the
 * finaliser that turns a (summed) packed table into the public outputs. */
pm4g_status pm4g_tables_partial(const pm4g_log* log, uint64_t* packed, pm4g_stream_t stream);
pm4g_status pm4g_tables_finalize(const uint64_t* packed, uint32_t n_activities, uint64_t* cnt,
                                 int64_t* dur_sum, double* mean, uint64_t* start, uint64_t* end,
                                 pm4g_stream_t stream);

/* ---------------------------------------------------------------- diagnostics */
const char* pm4g_last_error(void);
const char* pm4g_version(void);
/* Number of kernels this library has launched (process-wide counter). */
uint64_t pm4g_launch_count(void);
/* Device memory held by the library (process-wide): blocks / bytes owned by
 * live handles and scratch, and bytes of freed blocks kept in its reuse cache.
 * After every handle is destroyed, live_blocks == 0 (the leak check of
 * tests/test_gpu_sanitizer.py).  Any pointer may be NULL. */
pm4g_status pm4g_mem_stats(uint64_t* live_blocks, uint64_t* live_bytes, uint64_t* cached_bytes);
/* Return every cached (freed) block to the CUDA memory pool; synchronises the
 * device first.  Live blocks are untouched. */
pm4g_status pm4g_mem_release(void);
/* Per-kernel timing with CUDA events recorded around every launch on the
 * launching stream (enable -> run -> collect).  collect synchronises. */
pm4g_status pm4g_prof_enable(int32_t on);
pm4g_status pm4g_prof_reset(void);
/* Aggregates recorded launches by kernel name; returns the number of names.
 * For i < that number, pm4g_prof_entry gives name, launches, total ms and the
 * algorithmic bytes the library attributes to those launches. */
pm4g_status pm4g_prof_collect(int32_t* n_names);
pm4g_status pm4g_prof_entry(int32_t i, const char** name, uint64_t* launches, double* total_ms,
                            double* bytes);
/* The individual launches of the last collect, in launch order: start time
 * relative to the first recorded launch and duration (ms). */
int32_t pm4g_prof_n_records(void);
pm4g_status pm4g_prof_record(int32_t i, const char** name, double* start_ms, double* dur_ms);

#ifdef __cplusplus
}
#endif
#endif /* PM4G_H */
