/*
 * aggb200.h — C ABI of libaggb200.so, the B200-native group-by aggregation
 * hot path (arXiv 1311.0059 operators) behind the reference's operator API.
 *
 * The reference's boundary is the Python Operator plugin API
 * (/root/reference/pkg/src/aggbench/operators/base.py:126-231):
 *     op = OPERATORS[algo_id](OpContext(EngineConfig, AggSpec), DatasetStats, level)
 *     op.open(); op.push(frame)...; op.close() -> finished frames
 *     run_operator(op, source) / collect_groups(op, source)
 * Its kernels (_kernels.k_*) are internal and work on one 32 KB frame per call
 * (SURVEY.md §8(b)); this ABI replaces the operator as a whole with batched,
 * columnar, stream-ordered calls.  Every entry point below names the reference
 * interface it replaces.  No torch types cross this boundary: plain pointers,
 * sizes and POD structs only.  Device pointers unless a field says otherwise.
 *
 * Threading: one handle per (device, stream); a handle is not thread safe;
 * distinct handles may run concurrently (one OpContext per run).
 * Errors: every call returns an AGGB_* status; aggb_last_error() returns the
 * thread-local message.  The Python shim maps statuses onto the reference's
 * exception classes (core.py:28-61).
 */
#ifndef AGGB200_H
#define AGGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (core.py:28-61 exception classes) -------------------- */
#define AGGB_OK 0
#define AGGB_INVALID_BUDGET 1      /* InvalidBudget                         */
#define AGGB_BUDGET_EXHAUSTED 2    /* BudgetExhausted                       */
#define AGGB_CAPACITY_EXCEEDED 3   /* CapacityExceeded                      */
#define AGGB_SPEC_ERROR 4          /* SpecError                             */
#define AGGB_ORDER_ERROR 5         /* MergeOrderError                       */
#define AGGB_CUDA_ERROR 6          /* (new) CUDA runtime failure            */
#define AGGB_INVALID_ARG 7         /* (new) bad pointer / size / state      */
#define AGGB_INVALID_RECORD 8      /* InvalidRecord                         */

/* ---- algorithm ids (operators/__init__.py:37-58) ------------------------ */
#define AGGB_SORT_BASED 0
#define AGGB_HASH_SORT 1
#define AGGB_ORIGINAL_HH 2
#define AGGB_SHARED_HASH 3
#define AGGB_DYNAMIC_DESTAGING 4
#define AGGB_PRE_PARTITIONING 5

/* ---- aggregate functions (core.py:115-123 AGGREGATES) ------------------- */
#define AGGB_FN_SUM 0
#define AGGB_FN_COUNT 1
#define AGGB_FN_AVG 2
#define AGGB_FN_MIN 3
#define AGGB_FN_MAX 4

/* ---- column types ------------------------------------------------------- */
#define AGGB_I64 0
#define AGGB_F64 1
#define AGGB_I32 2

/* ---- input kinds -------------------------------------------------------- */
#define AGGB_INPUT_RAW 0      /* value columns; init ops applied on load (k_expand, _kernels.py:237-264) */
#define AGGB_INPUT_STATES 1   /* reference state records: per-function state columns (f64), merged */

#define AGGB_MAX_FNS 32
#define AGGB_MAX_VALS 32
#define AGGB_MAX_KEYS 2

/* EngineConfig (operators/base.py:50-65) + DatasetStats (core.py:383-404). */
typedef struct {
  int32_t algo;             /* AGGB_* algorithm id                           */
  int32_t memory_frames;    /* M: budget in frames (EngineConfig.memory_frames) */
  int32_t frame_size;       /* p: bytes per frame (EngineConfig.frame_size)  */
  int32_t input_sorted;     /* EngineConfig.input_sorted                     */
  int64_t budget_groups;    /* >0: resident-table capacity in groups, overriding the
                               frame-derived capacity (BASELINE configs state budgets in groups) */
  double fudge;             /* EngineConfig.fudge (default 1.2)              */
  double slot_ratio;        /* EngineConfig.slot_ratio (default 1.0)         */
  uint64_t seed;            /* EngineConfig.seed                             */
  double group_estimate;    /* EngineConfig.group_estimate; < 0 means None   */
  double stats_R, stats_R_t, stats_G, stats_G_t;  /* DatasetStats            */
  int32_t level;            /* Operator(..., level) (base.py:131-137)        */
  int32_t emit_partials;    /* 1: finish() leaves unfinalized state columns (multi-GPU combine
                               step; the reference's unfinalized runs, _emit_record finalize=0) */
  int32_t reserved_[6];
} aggb_config;

/* AggSpec (core.py:126-185) + an explicit key / value-column binding. */
typedef struct {
  int32_t n_fns;
  int32_t fn[AGGB_MAX_FNS];       /* AGGB_FN_*                               */
  int32_t col[AGGB_MAX_FNS];      /* RAW: value column of fn i; STATES: ignored */
  int32_t n_keys;                 /* 1 or 2 key columns (C5: int64 || int32)   */
  int32_t key_type[AGGB_MAX_KEYS];/* AGGB_I64 / AGGB_I32                       */
  int32_t n_vals;                 /* RAW: value columns; STATES: state columns */
  int32_t val_type[AGGB_MAX_VALS];/* AGGB_I64 / AGGB_F64 / AGGB_I32            */
  int32_t input_kind;             /* AGGB_INPUT_RAW / AGGB_INPUT_STATES        */
} aggb_spec;

/* One pushed batch: the columnar form of a run of input frames. */
typedef struct {
  int64_t n_rows;
  const void* key[AGGB_MAX_KEYS];
  int64_t key_stride[AGGB_MAX_KEYS];   /* bytes between rows (0: packed)       */
  const void* val[AGGB_MAX_VALS];
  int64_t val_stride[AGGB_MAX_VALS];
  int32_t on_host;                     /* 1: pointers are host memory (copied H2D on the stream;
                                          aggb_push returns once the copies out of them are done,
                                          so the caller may refill its buffers) */
  int32_t reserved_;
} aggb_input;

/* Finished groups (the decoded output frames of close()). Owned by the handle,
 * valid until the next aggb_reset / aggb_destroy (cf. reused frames, base.py:6-8). */
typedef struct {
  int64_t n_groups;
  void* key[AGGB_MAX_KEYS];            /* device, key_type per column          */
  void* out[AGGB_MAX_FNS];             /* device, one column per function      */
  int32_t out_type[AGGB_MAX_FNS];      /* AGGB_I64 / AGGB_F64                  */
  int32_t sorted;                      /* 1 when keys ascend (sort_based)      */
  int32_t reserved_;
} aggb_result;

/* Metrics (core.py:339-380), GPU edition: no comparison counts (a CPU-model
 * quantity); byte counters feed the roofline. */
typedef struct {
  int64_t records;                     /* input records pushed                 */
  int64_t output_groups;
  int64_t resident_groups;             /* groups held by the level-0 table     */
  int64_t spilled_records;             /* records written to HBM run buffers   */
  int64_t spilled_bytes;
  int64_t spilled_partitions;          /* non-empty partitions sealed          */
  int64_t recursion_depth;
  int64_t grace_levels;
  int64_t fallbacks;
  int64_t high_water_bytes;            /* device bytes held by the handle      */
  int64_t budget_groups;               /* resident-table capacity used         */
  int64_t partitions_level0;           /* spill fan-out chosen at level 0      */
  int64_t kernel_launches;             /* kernels launched since create/reset  */
  int64_t hbm_bytes_alg;               /* algorithmic bytes     */
  int64_t level0_spilled_records;      /* records spilled before recursion     */
  int64_t child_subpasses;             /* most sub-passes a child took (fan-out
                                          beyond one spill pass)               */
} aggb_metrics;

/* Operator.__init__ + open() (base.py:131-137, hash_sort.py:27-38,
 * hybrid.py:363-390 / :488-516, sort_based.py:34-52): validate the budget
 * (InvalidBudget), plan the table / partitions and allocate device state.
 * `stream` is a cudaStream_t (NULL: the handle creates its own). */
int aggb_create(int device, const aggb_config* cfg, const aggb_spec* spec,
                void* stream, void** handle);

/* Operator.push(frame) (base.py:178-179; k_table_insert _kernels.py:353-392,
 * k_pp_probe :917-962, k_hh_push :865-914, k_sort_load :544-581): aggregate one
 * batch; may partition and spill into HBM run buffers.  Asynchronous on the
 * handle's stream. */
int aggb_push(void* handle, const aggb_input* in);

/* Operator.close() (base.py:181-182; _drain_runs hybrid.py:244-277,
 * MergeDriver run_store.py:249-386, k_flush_slots _kernels.py:473-519):
 * recurse over spilled runs, finalize, and describe the result.  Synchronizes
 * the stream. */
int aggb_finish(void* handle, aggb_result* out);

/* Copy the result into caller buffers, host or device (cudaMemcpyDefault; this
 * is the decode of output frames, core.py:241-248).  keys[i]: n_groups *
 * sizeof(key_type[i]); out[j]: n_groups * 8.  NULL entries are skipped. */
int aggb_copy_result(void* handle, void* const* host_keys, void* const* host_out);

/* Multi-GPU exchange helpers (new).  After aggb_finish on a
 * handle created with emit_partials = 1, aggb_exchange_pack writes this rank's
 * partial groups as records of aggb_exchange_record_bytes() bytes (key words,
 * then state words) into the device buffer `send`, grouped by destination
 * dest = hash(key, exchange seed) % nranks, and fills counts[nranks] (host) with
 * records per destination.  The caller moves the bytes (NCCL all-to-allv via
 * torch.distributed) and merges what it received with aggb_push_partials
 * (same record layout, device pointer) on a handle of the same spec. */
int64_t aggb_exchange_record_bytes(void* handle);
int aggb_exchange_pack(void* handle, int nranks, void* send, int64_t* counts);
int aggb_push_partials(void* handle, const void* recv, int64_t n_records);

/* Raw-first exchange (new; "choose raw vs partial
 * adaptively").  When local aggregation would collapse little (C4: ~0.5N
 * distinct keys, 16 B raw < 24 B partial per record), ranks exchange input rows
 * before aggregating.  aggb_exchange_pack_raw packs the device columns of `in`
 * by dest = hash(key, exchange seed) % nranks (the seed aggb_exchange_pack
 * uses) into `send`: records of aggb_exchange_raw_record_bytes() bytes, one
 * 8-byte slot per key column then per value column (4-byte columns in the low
 * half).  The receiver pushes what it got with aggb_push, each column a
 * strided view (stride = record bytes, offset = 8 x column index). */
int64_t aggb_exchange_raw_record_bytes(void* handle);
int aggb_exchange_pack_raw(void* handle, const aggb_input* in, int nranks, void* send, int64_t* counts);

/* Bytes of the spill page pool mapped from pinned host memory (new; SURVEY.md
 * §8(f) f3): the pool is one reserved address range, HBM first, host memory once
 * HBM is exhausted (runs larger than HBM, the RunWriter/RunReader analog). */
int64_t aggb_pool_host_bytes(void* handle);

/* Metrics snapshot (Metrics.as_dict, core.py:378-380). */
int aggb_metrics_get(void* handle, aggb_metrics* out);

/* Per-kernel timing: when enabled, the handle brackets every kernel it launches
 * with CUDA events on its stream; aggb_kernel_stats reports, per kernel kind i
 * (0 .. until AGGB_INVALID_ARG), its name, launch count and summed device ms
 * since aggb_profile(h, 1).  (new; roofline evidence, no reference counterpart) */
int aggb_profile(void* handle, int enable);
int aggb_kernel_stats(void* handle, int i, const char** name, int64_t* launches, double* total_ms);

/* Reuse the handle for a fresh run (new OpContext), keeping device memory. */
int aggb_reset(void* handle);

void aggb_destroy(void* handle);

/* Thread-local message of the last failing call on this thread. */
const char* aggb_last_error(void);

/* Seeded device generator for the BASELINE configs (paper_1311_0059_b200/datagen.py
 * restated on the device; integer columns bit-identical to the host generator).
 * kind: 0 uniform int lo+x%range -> int64, 1 U[0,1) f64, 2 normal f64,
 *       3 zipf keys (cdf: device f64[K]; a, b: affine permutation), 4 uniform int -> int32. */
int aggb_generate(void* stream, int kind, uint64_t seed, uint64_t stream_id, int64_t start,
                  int64_t n, int64_t lo, int64_t range, const double* cdf, int64_t K,
                  uint64_t a, uint64_t b, void* out, int64_t out_stride);

/* Flush L2 between timed iterations (writes `bytes` of scratch). */
int aggb_l2_flush(void* stream, void* scratch, int64_t bytes);

/* Library / build identification. */
const char* aggb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AGGB200_H */
