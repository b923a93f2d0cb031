// gd_device.cuh -- device-side data layout shared by the sm_100a kernels.
//
// Packed ensemble node (16 bytes, one LDG.128 per visited node):
//   internal: v = threshold (exact double), feat = column, aux = global index
//             of the left child; the right child is aux + 1 (the packer
//             re-lays every tree out breadth-first so siblings are adjacent).
//   leaf:     feat = -1, v = leaf_value, aux = the leaf's ORIGINAL tree-local
//             node index (what GbtTree::predict_row's `idx` ends on,
//             models.cpp:71-78) so leaf ids come out in the caller's numbering.
#pragma once

#include <cstddef>
#include <cstdint>

#include "gdvfs.h"

namespace gd {

struct __align__(16) PNode {
    double v;
    int32_t feat;
    int32_t aux;
};
static_assert(sizeof(PNode) == 16, "PNode must stay 16 bytes");

// Walk node (8 bytes), the rank form of a grid node used by the walk kernel:
//   internal: key = index of its threshold among the sorted distinct non-NaN
//             thresholds of its feature (-1 for a NaN threshold);
//   clock:    key = t16 (clamp(floor(thr), 0, 65535));
//   leaf:     key = packed (grid) index of the leaf;
//   fc = feat << 19 | 8 * child | leaf flags: feat (signed; kFeat* for leaf /
//   clock) in the top 13 bits, the byte offset of the left child within its
//   tree (right = +8) in the low 19 bits, whose 3 low bits are free: bit 0 set
//   when the left child is a leaf, bit 1 when the right one is (a walk stops
//   at the parent; the leaf's packed index is the tree's root + its position).  With rank(x) = #{thresholds of the feature < x} (NaN x:
//   their count), `x <= thr_k  <=>  rank(x) <= k` exactly.
struct __align__(8) WNode {
    int32_t key;
    int32_t fc;
};
static_assert(sizeof(WNode) == 8, "WNode must stay 8 bytes");

// In the grid variant of a packed model the clock columns are recoded so one
// `feat < 0` test stops a row-only walk: leaf -1, sm_clock -2, mem_clock -3.
constexpr int32_t kFeatLeaf = -1;
constexpr int32_t kFeatSm = -2;
constexpr int32_t kFeatMem = -3;

// Everything the fused grid kernel needs, passed as one __grid_constant__.
struct GridParams {
    const PNode* e_nodes;
    const int32_t* e_roots;
    const PNode* t_nodes;
    const int32_t* t_roots;
    const WNode* e_wnodes;  // walk nodes (rank form), trees padded to an even node count
    const WNode* t_wnodes;
    const int32_t* e_wroots;  // n_trees + 1, in walk-node units
    const int32_t* t_wroots;
    const double* e_thr;      // sorted distinct thresholds per feature, [thr_off[f], thr_off[f+1])
    const double* t_thr;
    const int32_t* e_thr_off;
    const int32_t* t_thr_off;
    double e_base, e_lr, t_base, t_lr;
    int32_t e_trees, t_trees;
    int32_t e_max_pair_nodes, t_max_pair_nodes;  // roots[] carry a sentinel roots[n_trees]
    int32_t max_tree_nodes;
    const int32_t* e_wint;  // per tree: loadable walk-node prefix (up to the last internal node, even)
    const int32_t* t_wint;
    int32_t max_wint;
    int32_t rank16;  // every feature has <= 65535 distinct thresholds (16-bit ranks)
    int32_t rank8;   // ... <= 255 (8-bit ranks: 1024-app walk tiles)

    const double* rows;    // [n_records, n_cols] energy-encoded
    const double* rows_t;  // [n_records, n_cols] time-encoded (general mode only)
    const double* cat_t;   // [n_records, n_cat]
    const int32_t* cat_cols;
    const int32_t* rec_of_clock;  // [n_apps, n_clocks] or null
    const int32_t* sm;
    const int32_t* mem;
    const double* budgets;
    gd_decision* out;
    double* e_out;
    double* t_out;
    int64_t n_apps;
    int32_t n_cols, n_cat, n_clocks, sm_col, mem_col;
    int32_t mode, objective, best_effort;
    int64_t out_stride;  // row stride of e_out / t_out (n_clocks, or the full catalog for a clock chunk)
    // Host-buffer calls of several app batches (launch_grid_select, fast
    // path, rec_of_clock null): rows / cat_t / budgets still on the host
    // (pinned); batch b's slices are copied on `copy_stream` and batch b's
    // kernels wait for `batch_ready[b]`, so the upload overlaps the compute.
    const double* h_rows = nullptr;
    const double* h_cat_t = nullptr;
    const double* h_budgets = nullptr;
    void* copy_stream = nullptr;
    void* const* batch_ready = nullptr;  // cudaEvent_t[n_batches]
};

struct SelectParams {
    const double* energy;
    const double* time;
    const int32_t* sm;
    const double* budgets;
    gd_decision* out;
    int64_t n_apps;
    int32_t n_clocks;
    int32_t mode, objective, best_effort;
};

// Launchers (gd_kernels.cu).  All enqueue on `stream` and return the
// cudaError_t of the launch.
int launch_predict_gbt(const PNode* nodes, const int32_t* roots, int32_t n_trees, double base, double lr,
                       int clamp, const double* rows, int64_t n_rows, int32_t n_cols, double* out,
                       int32_t* leaf_ids, int sm_count, void* stream);
int launch_predict_linear(const double* coef, double intercept, int clamp, const double* rows, int64_t n_rows,
                          int32_t n_cols, double* out, int sm_count, void* stream);
int launch_build_rows_t(const double* rows, const double* cat_t, const int32_t* cat_cols, int32_t n_cat,
                        int64_t n_records, int32_t n_cols, double* rows_t, void* stream);
// The grid path (gd_grid.cu).  Without rec_of_clock it runs, per app batch,
// the walk kernel then the accumulate+select kernel, using `scratch` (at
// least grid_scratch_bytes) for the per-(app, tree) records; `launches` is
// incremented per kernel launched.
int64_t grid_scratch_per_app(const GridParams& p);
int64_t grid_batch_apps(const GridParams& p);  // apps per batch of the fast path
size_t grid_scratch_bytes(const GridParams& p, bool general);
// `mark(name)`, if set, is called after each kernel launch (timing hook).
typedef void (*LaunchMark)(void* user, const char* name);
int launch_grid_select(const GridParams& p, bool general, int sm_count, void* stream, void* scratch,
                       size_t scratch_bytes, int64_t* launches, LaunchMark mark = nullptr, void* user = nullptr);
int launch_select(const SelectParams& p, int sm_count, void* stream);
// K3 for catalogs wider than kMaxClocks: a warp per app striding over the clocks.
int launch_select_wide(const SelectParams& p, int sm_count, void* stream);
// Whether the partial-evaluation pipeline (rank -> walk -> accumulate) can
// take these models: 16-bit feature ranks, trees of <= 65536 nodes and a
// walk geometry that fits shared memory.  Otherwise the general kernel runs.
bool grid_fast_path_ok(const GridParams& p);
int launch_dadd_probe(double* scratch, int blocks, int iters, void* stream);
// Selection frontier (gd_kernels.cu frontier_kernel): sorted times, prefix
// best catalog index, first (best-effort) index or -2 for non-finite rows.
int launch_frontier(const double* E, const double* T, const int32_t* sm, int64_t n_apps, int32_t n_clocks,
                    int32_t objective, double* t_sorted, int32_t* best, int32_t* first, int sm_count, void* stream);
// Copy `n` packed nodes recoding features sm_col / mem_col as kFeatSm / kFeatMem.
int launch_recode_clock_nodes(const PNode* src, PNode* dst, int64_t n, int32_t sm_col, int32_t mem_col, void* stream);

// Walk nodes (rank form) from grid nodes; `dst` must be zeroed (padding).
// sm_fix / mem_fix > 0: that clock column has this one value in every
// candidate of the call, and its tests are folded into unconditional nodes.
// fold (device, nullable): the state written by launch_fold_check; the build
// then runs only if that state changed.
int launch_build_walk_nodes(const PNode* grid, int64_t n, const int32_t* roots, int32_t n_trees,
                            const int32_t* wroots, const double* thr, const int32_t* thr_off, int32_t sm_fix,
                            int32_t mem_fix, const int32_t* fold, WNode* dst, void* stream);
// The catalog's folded clocks on the device (one block): fold[0..1] = sm /
// mem value or 0, fold[2] = whether that changed, for up to two models.
int launch_fold_check(const int32_t* sm, const int32_t* mem, int32_t C, int32_t enable, int32_t* fold_a,
                      int32_t* fold_b, void* stream);

// Largest clock catalog the fused kernels take (32 lanes x 16 clocks).
constexpr int kMaxClocks = 512;
constexpr int kMaxCols = 1024;

}  // namespace gd
