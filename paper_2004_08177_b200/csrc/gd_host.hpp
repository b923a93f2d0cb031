// gd_host.hpp -- host-side runtime objects behind the C ABI (include/gdvfs.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "gd_device.cuh"
#include "gdvfs.h"

// A device buffer kept across calls (grow-only): the latency path pays no
// cudaMallocAsync / cudaFreeAsync per call.  `ev` marks the last use, so a
// call on a different stream first waits for it.
struct gd_pbuf {
    char* base = nullptr;
    size_t cap = 0;
    uint64_t generation = 0;  // bumped when the buffer moves (captured graphs hold its address)
    cudaEvent_t ev = nullptr;
    cudaStream_t stream = nullptr;
};

// A captured small-call pipeline (staged H2D -> rank -> walk -> accumulate
// -> D2H into pinned staging), replayed with one cudaGraphLaunch.
struct gd_graph_entry {
    uint64_t me = 0, mt = 0;  // model uids
    int64_t n_apps = 0;
    int64_t n_records = 0;  // staged piece offsets (cat_t .. budgets) depend on it
    int32_t n_clocks = 0, n_cols = 0, n_cat = 0, sm_col = 0, mem_col = 0;
    int32_t mode = 0, objective = 0, best_effort = 0;
    cudaStream_t stream = nullptr;
    uint64_t gen0 = 0, gen1 = 0;  // pbuf generations at capture
    cudaGraphExec_t exec = nullptr;
};

struct gd_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    // Measurement hook (gd_ctx_set_timing): events around each grid kernel.
    bool timing = false;
    std::vector<cudaEvent_t> events;  // pool, grown on demand
    std::vector<const char*> marks;   // kernel name per interval of the last call
    // Pinned staging for small host-buffer calls (one H2D copy instead of
    // one per input array); stage_ev guards reuse.
    char* stage = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev = nullptr;
    gd_pbuf pbuf[2];  // 0: grid kernel scratch, 1: host-buffer call inputs / outputs
    char* out_stage = nullptr;  // pinned, kStageLimit bytes: decisions of graph replays
    std::vector<gd_graph_entry> graphs;  // most recent last
    // Large host-buffer calls: batch inputs streamed on copy_stream, one
    // event per batch (grow-only pool).
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> batch_events;
};

struct gd_model {
    // Device the model lives on (-1: host-only, parsed / packed but never
    // uploaded).  Models do not hold their creating gd_ctx: a context may be
    // destroyed while its models live on, and a model serves any context of
    // its device.
    int device = -1;
    uint64_t uid = 0;  // process-unique (graph cache keys survive address reuse)
    int32_t kind = GD_KIND_GBT;
    int32_t target = GD_TARGET_ENERGY;
    int32_t n_cols = 0;
    int32_t max_depth = 0;
    double base = 0.0;  // GBT base_prediction or linear intercept
    double lr = 0.0;
    // Host copy in the caller's node numbering (export / leaf-id meaning).
    std::vector<int64_t> offsets;
    std::vector<int32_t> feature, left, right;
    std::vector<double> threshold, leaf;
    std::vector<double> coef;
    std::vector<std::string> columns;  // from a model file; empty when uploaded
    // Device copy.
    gd::PNode* d_nodes = nullptr;
    int32_t* d_roots = nullptr;
    double* d_coef = nullptr;
    int64_t packed_nodes = 0;
    int32_t max_pair_nodes = 0;
    int32_t max_tree_nodes = 0;  // largest packed size of two consecutive trees (2q, 2q+1)
    // Grid variant of d_nodes: the sm / mem clock columns recoded as
    // feat = kFeatSm / kFeatMem (built on first use per column pair).
    mutable gd::PNode* d_grid_nodes = nullptr;
    // Rank form for the walk kernel: sorted distinct thresholds per feature,
    // walk-node tree offsets (trees padded to an even count) and the walk
    // nodes themselves (built with the grid nodes).
    double* d_thr = nullptr;
    int32_t* d_thr_off = nullptr;
    int32_t* d_wroots = nullptr;
    int64_t n_wnodes = 0;
    // Per tree: walk nodes a walk can load -- the breadth-first prefix up to
    // the last internal node (leaves are never loaded: parents flag them),
    // rounded up to an even count.
    int32_t* d_wint = nullptr;
    int32_t max_wint = 0;
    int32_t max_thr_per_feature = 0;
    mutable gd::WNode* d_wnodes = nullptr;
    mutable int32_t grid_sm_col = -1, grid_mem_col = -1;
    // Folded constant clocks of the walk nodes (0: none; -2: set on the device
    // by a device-buffer call, d_fold holds them).
    mutable int32_t grid_sm_fix = 0, grid_mem_fix = 0;
    mutable int32_t* d_fold = nullptr;  // device {sm_fix, mem_fix, changed}

    int32_t n_trees() const { return offsets.empty() ? 0 : static_cast<int32_t>(offsets.size() - 1); }
};

namespace gdh {

int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* where);

// Packer: validate the trees and lay them out breadth-first with adjacent
// children (gd_pack.cpp).
int pack_forest(const gd_forest_view& f, int32_t n_cols, std::vector<gd::PNode>& nodes,
                std::vector<int32_t>& roots, int32_t& max_depth);

// "gpudvfs-model 1" parser (gd_model_io.cpp); fills the host fields of `m`.
int parse_model_file(const char* path, gd_model& m);

// gd_grid_select over host buffers; with keep_dev_out the decisions stay on
// the device (*keep_dev_out, the context's persistent buffer) instead of
// being copied to `out` (gd_capi.cpp).
int grid_select_host(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid* g, const gd_select_opts* o,
                     gd_decision* out, double* e_out, double* t_out, gd_decision** keep_dev_out);

// fit_gbt's booster on the device (gd_train.cu): fills the forest arrays in
// fit_gbt's node order and the base prediction.
int fit_gbt_device(gd_ctx* ctx, const double* rows, int64_t n, int32_t p, const double* targets,
                   const gd_gbt_config& cfg, std::vector<int64_t>& offsets, std::vector<int32_t>& feature,
                   std::vector<double>& threshold, std::vector<int32_t>& left, std::vector<int32_t>& right,
                   std::vector<double>& leaf, double& base);

// A device copy of `src` (any model holding its host arrays) on ctx's device
// (gd_capi.cpp; used by gd_multi_model_replicate).
int clone_model(gd_ctx* ctx, const gd_model* src, gd_model** out);

// Host selection for one job at a dynamic budget (gd_edf.cpp); the same
// rules as the device epilogue.
void select_one(const double* E, const double* T, const int32_t* sm, int32_t n, double budget,
                const gd_select_opts& o, gd_decision& out);

}  // namespace gdh
