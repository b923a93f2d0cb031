/*
 * gdvfs.h -- C ABI of the B200 (sm_100a) evaluation path for arXiv 2004.08177's
 * data-driven DVFS scheduler: batched energy/time GBT ensemble evaluation over
 * every (application x clock) candidate, the deadline-aware selection fused
 * into the same kernel, and the host EDF loop that consumes the decisions.
 *
 * Plain C, plain pointers and sizes; no C++ or torch types cross it.  Every
 * entry point returns GD_OK (0) or an error code and leaves a message in
 * gd_last_error() (thread-local).  Each function cites the reference
 * interface it replaces (paths relative to /root/reference/proj).
 *
 * Threading: one gd_ctx per (device, host thread).  Calls that take host
 * buffers are synchronous; *_device variants take device pointers, enqueue on
 * the context's stream and return without synchronising.  A context keeps
 * grow-only device scratch, a pinned staging buffer and (for small
 * decisions-only gd_grid_select calls) CUDA graphs of the whole call keyed by
 * (models, batch shape, options, stream); GDVFS_GRAPHS=0 disables the graphs.
 */
#ifndef GDVFS_H
#define GDVFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes.  The C++ facade (include/gpudvfs_b200/gpu_api.hpp) maps them
 * back onto the reference's exception types (core.hpp:14-29). */
enum {
    GD_OK = 0,
    GD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument               */
    GD_ERR_DATA = 2,             /* gpudvfs::data_error                  */
    GD_ERR_MISSING_ARTIFACT = 3, /* gpudvfs::missing_artifact_error      */
    GD_ERR_IO = 4,               /* gpudvfs::io_error                    */
    GD_ERR_CUDA = 5,             /* device failure (no CPU fallback)     */
    GD_ERR_UNSUPPORTED = 6
};

/* Model kinds / targets (models.hpp:29, core.hpp:103). */
enum { GD_KIND_OLS = 0, GD_KIND_LASSO = 1, GD_KIND_GBT = 2 };
enum { GD_TARGET_ENERGY = 0, GD_TARGET_TIME = 1 };

/* SchedulerOptions knobs (scheduler.hpp:52-67). */
enum { GD_MODE_TEXT = 0, GD_MODE_LITERAL = 1 };
enum { GD_OBJECTIVE_ENERGY = 0, GD_OBJECTIVE_POWER = 1 };
enum { GD_BUDGET_REMAINING = 0, GD_BUDGET_FULL = 1 };

/* Decision status / note (scheduler.hpp:23-32, scheduler.cpp:196,221). */
enum { GD_SCHEDULED = 0, GD_REJECTED = 1 };
enum { GD_NOTE_NONE = 0, GD_NOTE_BEST_EFFORT = 1, GD_NOTE_MISSING_DATA = 2 };

typedef struct gd_ctx gd_ctx;
typedef struct gd_model gd_model;

/* One tree ensemble as flat arrays over all trees.  Node fields are exactly
 * models::GbtNode (models.hpp:35-43): feature (< 0 = leaf), threshold,
 * tree-local left/right child indices, leaf_value.  Node order within a tree
 * is free (level order after fit_gbt, preorder after load_model); leaf ids
 * reported by gd_predict_rows are indices in THIS order. */
typedef struct gd_forest_view {
    int32_t n_trees;
    const int64_t* tree_offsets; /* n_trees + 1, node offset of each tree */
    const int32_t* feature;
    const double* threshold;
    const int32_t* left;
    const int32_t* right;
    const double* leaf_value;
} gd_forest_view;

typedef struct gd_model_info {
    int32_t kind;
    int32_t target;
    int32_t n_cols;
    int32_t n_trees;
    int64_t n_nodes;
    int32_t max_depth;
    int32_t pad;
    double base_prediction; /* GBT base / linear intercept */
    double learning_rate;
} gd_model_info;

/* 24-byte per-app decision record (ScheduleDecision minus the Job copy). */
typedef struct gd_decision {
    int32_t clock_index; /* index into the clock_catalog order, -1 = none */
    int16_t status;      /* GD_SCHEDULED / GD_REJECTED */
    int16_t note;        /* GD_NOTE_* */
    double energy_ws;    /* predicted E of the chosen clock (0 if none) */
    double time_s;       /* predicted T of the chosen clock (0 if none) */
} gd_decision;

/* The (app x clock) grid, replacing the rows ModelPredictorState::build
 * materialises (scheduler.cpp:329-370).  Row r holds the energy-encoded
 * feature row of profiled record r (ingest::apply_encoding, ingest.cpp:401-439);
 * the time model sees the same row with the n_cat categorical columns
 * cat_cols[] replaced by cat_t[r * n_cat + k].  For clock c of app a the
 * record is rec_of_clock[a * n_clocks + c] (the nearest-record substitution of
 * scheduler.cpp:341-359) or, when rec_of_clock is NULL, record a; columns
 * sm_col / mem_col (-1 = absent) are overridden with the candidate clock
 * (scheduler.cpp:352-357).  sm_clock/mem_clock list the catalog in
 * clock_catalog order (core.cpp:177-184), which fixes tie order. */
typedef struct gd_grid {
    const double* rows;
    int64_t n_records;
    int32_t n_cols;
    int32_t n_cat;
    const double* cat_t;
    const int32_t* cat_cols;
    const int32_t* rec_of_clock;
    int64_t n_apps;
    const int32_t* sm_clock;
    const int32_t* mem_clock;
    int32_t n_clocks;
    int32_t sm_col;
    int32_t mem_col;
    int32_t pad;
    const double* budgets; /* per-app time budget (deadline_s for full_deadline) */
} gd_grid;

typedef struct gd_select_opts {
    int32_t mode;        /* GD_MODE_* */
    int32_t objective;   /* GD_OBJECTIVE_* */
    int32_t best_effort; /* best_effort_fallback */
    int32_t pad;
} gd_select_opts;

/* One job of a Workload (core.hpp:89-96).  app_rank orders app_id strings
 * (std::string '<'); app_index selects the job's row of the per-app E/T
 * tables, -1 when the predictor has no data ("missing correlated data"). */
typedef struct gd_job {
    double arrival_s;
    double deadline_s;
    int64_t app_rank;
    int32_t app_index;
    int32_t pad;
} gd_job;

/* ExecutionTimeSource (scheduler.hpp:78): seconds job `job` runs at catalog
 * clock `clock_index`. */
typedef double (*gd_exec_fn)(void* user, int64_t job, int32_t clock_index);

const char* gd_last_error(void);
const char* gd_version(void);

/* Contexts ---------------------------------------------------------------- */
int gd_ctx_create(int32_t device, gd_ctx** out);
int gd_ctx_destroy(gd_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores
 * the context's own stream. */
int gd_ctx_set_stream(gd_ctx* ctx, void* cuda_stream);
int gd_ctx_synchronize(gd_ctx* ctx);
/* Number of kernels this context has launched so far. */
int64_t gd_ctx_launch_count(const gd_ctx* ctx);
/* Per-kernel timing (measurement hook, off by default): while on, every grid
 * call records CUDA events on the context stream around each kernel it
 * launches; gd_ctx_kernel_times then synchronizes on them and returns the
 * last grid call's kernel durations in launch order (ms) with their kernel
 * names ("rank", "walk", "acc" per app batch, or "general"), n = count. */
int gd_ctx_set_timing(gd_ctx* ctx, int on);
int gd_ctx_kernel_times(gd_ctx* ctx, float* ms, const char** names, int32_t max, int32_t* n);

/* Models: the packer.  Replaces holding a models::FittedModel
 * (models.hpp:63-70) for prediction.  Validates the trees (children in range,
 * every node reached once, features < n_cols) and re-lays them out on the
 * device as 16-byte nodes with adjacent children.  ctx may be NULL: the
 * model is then parsed, packed and validated on the host only (no device
 * copy; prediction calls reject it). */
int gd_model_upload_gbt(gd_ctx* ctx, const gd_forest_view* forest, double base_prediction, double learning_rate,
                        int32_t n_cols, int32_t target, gd_model** out);
int gd_model_upload_linear(gd_ctx* ctx, const double* coefficients, int32_t n_cols, double intercept,
                           int32_t kind, int32_t target, gd_model** out);
/* Parse a "gpudvfs-model 1" file (models.cpp:639-714, load_model_file) and
 * upload it.  Errors: GD_ERR_MISSING_ARTIFACT (cannot open), GD_ERR_DATA. */
int gd_model_load_file(gd_ctx* ctx, const char* path, gd_model** out);
int gd_model_info_get(const gd_model* model, gd_model_info* out);
/* Column name j of a model loaded from file (NULL for uploaded models). */
const char* gd_model_column(const gd_model* model, int32_t j);
/* Export the host copy of the trees (as given / as parsed). Arrays sized by
 * gd_model_info_get; any pointer may be NULL. */
int gd_model_export(const gd_model* model, int64_t* tree_offsets, int32_t* feature, double* threshold,
                    int32_t* left, int32_t* right, double* leaf_value);
int gd_model_free(gd_model* model);

/* K1 -- models::predict (models.cpp:395-428) over materialised rows: one
 * value per row, energy clamped at 0, leaf_ids (R x n_trees, nullable) are
 * predict_row's final node index per tree (models.cpp:71-78). */
int gd_predict_rows(gd_ctx* ctx, const gd_model* model, const double* rows, int64_t n_rows, int32_t n_cols,
                    double* out, int32_t* leaf_ids);
int gd_predict_rows_device(gd_ctx* ctx, const gd_model* model, const double* d_rows, int64_t n_rows,
                           int32_t n_cols, double* d_out, int32_t* d_leaf_ids);

/* K2+K3 -- the fused grid kernel: energy + time ensembles for every
 * (app, clock) candidate generated on the fly, then the deadline-masked
 * selection of scheduler.cpp:54-100,212-223 per app.  e_out / t_out
 * (A x C, nullable) receive the per-candidate predictions (what the
 * ClockPredictor of make_model_predictor returns). */
/* Shapes: any catalog size (above 512 clocks the kernels run in 512-clock
 * chunks and one wide selection); models or catalogs the partial-evaluation
 * pipeline cannot take -- a feature with more than 65535 distinct
 * thresholds, a tree of more than 65536 nodes, clock values above 65535 MHz,
 * or per-clock records (rec_of_clock) -- run on the general per-candidate
 * kernel, with the same results.  gd_grid_select_device cannot read the
 * catalog on the host: its clock values must lie in 1..65535 MHz unless
 * rec_of_clock is given. */
int gd_grid_select(gd_ctx* ctx, const gd_model* energy, const gd_model* time, const gd_grid* grid,
                   const gd_select_opts* opts, gd_decision* out, double* e_out, double* t_out);
int gd_grid_select_device(gd_ctx* ctx, const gd_model* energy, const gd_model* time, const gd_grid* d_grid,
                          const gd_select_opts* opts, gd_decision* d_out, double* d_e_out, double* d_t_out);

/* K3 alone -- selection over given candidate tables E/T (A x C), e.g. from a
 * non-model ClockPredictor such as make_truth_predictor (scheduler.cpp:283). */
int gd_select(gd_ctx* ctx, const double* energy, const double* time, int64_t n_apps, const int32_t* sm_clock,
              int32_t n_clocks, const double* budgets, const gd_select_opts* opts, gd_decision* out);

/* schedule_d_dvfs (scheduler.cpp:182-237) driven by run_edf_loop
 * (scheduler.cpp:105-147): arrivals in (arrival, app_id) order, EDF pick by
 * (arrival + deadline, arrival, app_id), per-job budget (remaining or full),
 * selection over the job's E/T row, clock advanced by exec time.  exec_time
 * (A x C table) or exec_fn supplies ExecutionTimeSource.  Writes one decision
 * per job in processing order and the job index of each into order[]. */
int gd_schedule_edf(const gd_job* jobs, int64_t n_jobs, const double* energy, const double* time,
                    const int32_t* sm_clock, int32_t n_clocks, int32_t budget_kind, const gd_select_opts* opts,
                    const double* exec_time, gd_exec_fn exec_fn, void* exec_user, gd_decision* out,
                    int64_t* order);

/* Selection frontier for budget queries (the remaining_time EDF
 * loop re-selects each job at a budget known only when it is dequeued).  Per
 * app: t_sorted[a][k] = the app's predicted times sorted by (T, E, catalog
 * index); best[a][k] = catalog index of select_text's choice
 * (scheduler.cpp:62-81, objective per `objective`) among the first k + 1 of
 * them; first[a] = the best-effort choice (argmin (T, E, index),
 * scheduler.cpp:215-220), or -2 when the app has a non-finite E or T (query
 * those by a scan).  A budget b is answered by k = #{t_sorted <= b}: choice
 * best[a][k-1], none if k == 0.  Host buffers; synchronous. */
int gd_frontier(gd_ctx* ctx, const double* energy, const double* time, int64_t n_apps, const int32_t* sm_clock,
                int32_t n_clocks, int32_t objective, double* t_sorted, int32_t* best, int32_t* first);

/* gd_schedule_edf with text-mode selections answered from a frontier
 * (O(log C) per job instead of O(C)); literal mode and rows flagged
 * first = -2 fall back to the scan.  Same outputs as gd_schedule_edf. */
int gd_schedule_edf_frontier(const gd_job* jobs, int64_t n_jobs, const double* energy, const double* time,
                             const double* t_sorted, const int32_t* best, const int32_t* first,
                             const int32_t* sm_clock, int32_t n_clocks, int32_t budget_kind,
                             const gd_select_opts* opts, const double* exec_time, gd_exec_fn exec_fn,
                             void* exec_user, gd_decision* out, int64_t* order);

/* Training: fit_gbt on the GPU ------------------------------
 * GBTConfig (models.hpp:18-24). */
typedef struct gd_gbt_config {
    int32_t iterations;
    int32_t depth;
    double learning_rate;
    double l2_leaf_reg;
    uint64_t seed;
} gd_gbt_config;

/* models::fit_gbt (models.cpp:381-393; GbtCore, models.cpp:161-368): the
 * level-wise exact-greedy booster over presorted columns, with the split
 * search, routing and residual updates on the device.  rows is the
 * EncodedMatrix (n_rows x n_cols, row-major), targets its targets.  The
 * returned model's trees are node for node those of fit_gbt (node order,
 * features, thresholds, leaf values -- gd_model_export reads them) and it is
 * uploaded on ctx, ready for prediction.  Errors: the reference's
 * validate_config / require_rows messages (GD_ERR_INVALID_ARGUMENT). */
int gd_fit_gbt(gd_ctx* ctx, const double* rows, int64_t n_rows, int32_t n_cols, const double* targets,
               const gd_gbt_config* config, int32_t target, gd_model** out);

/* Multi-GPU: query-row sharding ------------------------------
 * Under full_deadline apps are independent (scheduler.cpp:203-205), so the
 * grid path shards by contiguous app ranges (rank g of G owns apps
 * [A*g/G, A*(g+1)/G)) with a replica of both ensembles per device; the only
 * collective is one NCCL gather of the 24-byte decisions to the root.  NCCL
 * is loaded at first use (libnccl.so.2; GDVFS_NCCL_LIB overrides); without
 * it these calls return GD_ERR_UNSUPPORTED. */
typedef struct gd_comm gd_comm;
typedef struct gd_multi gd_multi;

/* One process per GPU (torchrun): rank 0 creates a 128-byte id, every rank
 * receives it out of band and joins with its context's device. */
int gd_comm_unique_id(void* id128);
int gd_comm_init_rank(gd_ctx* ctx, const void* id128, int32_t n_ranks, int32_t rank, gd_comm** out);
int gd_comm_destroy(gd_comm* comm);
/* The decision gather: rank r contributes counts[r] decisions (d_send, device
 * memory); root receives them in rank order at d_recv (sum of counts).  Every
 * rank calls it with the same counts; enqueued on the context stream. */
int gd_gather_decisions(gd_comm* comm, const gd_decision* d_send, const int64_t* counts, gd_decision* d_recv,
                        int32_t root);

/* One process driving several GPUs: a context per device + ncclCommInitAll. */
int gd_multi_create(const int32_t* devices, int32_t n_devices, gd_multi** out);
int gd_multi_destroy(gd_multi* multi);
int32_t gd_multi_size(const gd_multi* multi);
int gd_multi_ctx(gd_multi* multi, int32_t index, gd_ctx** out);
/* A copy of `src` (a model of any context, or host-only) on every device of
 * the group: replicas[0 .. size-1], freed with gd_model_free. */
int gd_multi_model_replicate(gd_multi* multi, const gd_model* src, gd_model** replicas);
/* gd_grid_select (host buffers) row-sharded over the group: one host thread
 * per device evaluates its app range, E/T tables (nullable) land directly in
 * the caller's arrays, decisions are gathered to the first device by one
 * NCCL gather and copied back once.  energy[i] / time[i] are the replicas on
 * device i.  Results are identical to gd_grid_select on one device. */
int gd_multi_grid_select(gd_multi* multi, gd_model* const* energy, gd_model* const* time, const gd_grid* grid,
                         const gd_select_opts* opts, gd_decision* out, double* e_out, double* t_out);

/* Measure this device's FP64 add throughput (adds/s) with independent
 * __dadd_rn chains: the peak of the path's binding roofline (in-order FP64
 * leaf sums), measured on the same box as the kernel it bounds. */
int gd_microbench_dadd(gd_ctx* ctx, double* adds_per_second);

#ifdef __cplusplus
}
#endif

#endif /* GDVFS_H */
