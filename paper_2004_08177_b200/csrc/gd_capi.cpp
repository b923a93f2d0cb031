// gd_capi.cpp -- the thin C ABI over the sm_100a kernels (include/gdvfs.h).
//
// Host-buffer entry points stage inputs with stream-ordered allocations
// (cudaMallocAsync from a pool that keeps its memory), enqueue the kernel
// and copy results back before returning.  *_device entry points take
// device pointers and only enqueue.  There is no CPU compute fallback: a
// missing/failed device is an error (GD_ERR_CUDA).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gd_device.cuh"
#include "gd_host.hpp"

namespace gdh {

thread_local std::string g_error;

int set_error(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

int cuda_error(cudaError_t e, const char* where) {
    return set_error(GD_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace gdh

using gdh::cuda_error;
using gdh::set_error;

#define GD_CUDA(call, where)                                   \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return cuda_error(_e, where);   \
    } while (0)

namespace {

constexpr size_t kStageLimit = 256 << 10;  // host-buffer calls whose inputs fit are staged

uint64_t next_model_uid() {
    static std::atomic<uint64_t> n{0};
    return ++n;
}

// One stream-ordered scratch allocation carved into aligned pieces; with a
// gd_pbuf it is that persistent buffer (grown when too small) instead.
struct Scratch {
    cudaStream_t stream;
    gd_pbuf* keep = nullptr;
    char* base = nullptr;
    size_t size = 0;
    std::vector<std::pair<size_t, size_t>> pieces;  // offset, bytes

    size_t add(size_t bytes) {
        size = (size + 255) & ~static_cast<size_t>(255);
        pieces.push_back({size, bytes});
        size += bytes;
        return pieces.size() - 1;
    }
    void* ptr(size_t i) const { return pieces[i].second ? base + pieces[i].first : nullptr; }
    cudaError_t alloc() {
        if (!size) return cudaSuccess;
        if (!keep) return cudaMallocAsync(reinterpret_cast<void**>(&base), size, stream);
        cudaError_t e = cudaSuccess;
        if (!keep->ev && (e = cudaEventCreateWithFlags(&keep->ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        if (keep->stream && keep->stream != stream && (e = cudaStreamWaitEvent(stream, keep->ev, 0)) != cudaSuccess) {
            return e;
        }
        if (size > keep->cap) {
            if (keep->base) cudaFreeAsync(keep->base, stream);
            keep->base = nullptr;
            keep->cap = 0;
            const size_t cap = size + size / 4;
            if ((e = cudaMallocAsync(reinterpret_cast<void**>(&keep->base), cap, stream)) != cudaSuccess) return e;
            keep->cap = cap;
            ++keep->generation;
        }
        base = keep->base;
        return cudaSuccess;
    }
    ~Scratch() {
        if (keep) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(stream, &cs);
            if (base && cs == cudaStreamCaptureStatusNone) {  // (a captured replay reuses the same stream)
                cudaEventRecord(keep->ev, stream);
                keep->stream = stream;
            }
        } else if (base) {
            cudaFreeAsync(base, stream);
        }
    }
};

int activate(gd_ctx* ctx) {
    if (!ctx) return set_error(GD_ERR_INVALID_ARGUMENT, "null gd_ctx");
    GD_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    return GD_OK;
}

int check_model(const gd_ctx* ctx, const gd_model* m, const char* who) {
    if (!m) return set_error(GD_ERR_INVALID_ARGUMENT, std::string(who) + ": null model");
    if (m->device < 0) return set_error(GD_ERR_INVALID_ARGUMENT, std::string(who) + ": host-only model (no gd_ctx)");
    if (m->device != ctx->device) {
        return set_error(GD_ERR_INVALID_ARGUMENT, std::string(who) + ": model lives on device " +
                                                      std::to_string(m->device) + ", context on device " +
                                                      std::to_string(ctx->device));
    }
    return GD_OK;
}

// Model creation accepts ctx == NULL: the model is parsed / packed /
// validated on the host only (used by CPU-side tooling and tests).
int activate_opt(gd_ctx* ctx) { return ctx ? activate(ctx) : GD_OK; }

int upload_model(gd_model* m) {
    if (m->kind == GD_KIND_GBT) {
        gd_forest_view v{m->n_trees(), m->offsets.data(), m->feature.data(), m->threshold.data(),
                         m->left.data(),  m->right.data(),   m->leaf.data()};
        std::vector<gd::PNode> nodes;
        std::vector<int32_t> roots;
        int rc = gdh::pack_forest(v, m->n_cols, nodes, roots, m->max_depth);
        if (rc) return rc;
        m->packed_nodes = static_cast<int64_t>(nodes.size());
        // Sentinel: tree t occupies packed nodes [roots[t], roots[t + 1]).
        roots.push_back(static_cast<int32_t>(nodes.size()));
        m->max_pair_nodes = 0;
        m->max_tree_nodes = 0;
        for (size_t t = 0; t + 1 < roots.size(); ++t) {
            if (roots[t + 1] - roots[t] > m->max_tree_nodes) m->max_tree_nodes = roots[t + 1] - roots[t];
        }
        for (size_t t = 0; t + 1 < roots.size(); t += 2) {
            const int32_t end = roots[t + 2 < roots.size() ? t + 2 : roots.size() - 1];
            if (end - roots[t] > m->max_pair_nodes) m->max_pair_nodes = end - roots[t];
        }
        // Rank form (gd_device.cuh WNode): sorted distinct thresholds per
        // feature and the walk-node tree offsets.
        std::vector<std::vector<double>> per(static_cast<size_t>(m->n_cols));
        for (const gd::PNode& x : nodes) {
            if (x.feat >= 0 && x.v == x.v) per[static_cast<size_t>(x.feat)].push_back(x.v);
        }
        std::vector<double> thr;
        std::vector<int32_t> thr_off(1, 0), wroots(1, 0);
        m->max_thr_per_feature = 0;
        for (auto& v : per) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end(), [](double a, double b) { return a == b; }), v.end());
            thr.insert(thr.end(), v.begin(), v.end());
            thr_off.push_back(static_cast<int32_t>(thr.size()));
            if (static_cast<int32_t>(v.size()) > m->max_thr_per_feature) m->max_thr_per_feature = static_cast<int32_t>(v.size());
        }
        for (size_t t = 0; t + 1 < roots.size(); ++t) wroots.push_back(wroots.back() + ((roots[t + 1] - roots[t] + 1) & ~1));
        m->n_wnodes = wroots.back();
        std::vector<int32_t> wint;
        m->max_wint = 0;
        for (size_t t = 0; t + 1 < roots.size(); ++t) {
            int32_t last = -1;
            for (int32_t i = roots[t]; i < roots[t + 1]; ++i) {
                if (nodes[static_cast<size_t>(i)].feat >= 0) last = i - roots[t];
            }
            const int32_t w = ((last + 1) + 1) & ~1;
            wint.push_back(w < 2 ? 2 : w);
            if (wint.back() > m->max_wint) m->max_wint = wint.back();
        }
        if (m->device < 0) return GD_OK;  // host-only model: validated, never uploaded
        if (!thr.empty()) {
            GD_CUDA(cudaMalloc(&m->d_thr, thr.size() * sizeof(double)), "cudaMalloc(thresholds)");
            GD_CUDA(cudaMemcpy(m->d_thr, thr.data(), thr.size() * sizeof(double), cudaMemcpyHostToDevice),
                    "cudaMemcpy(thresholds)");
        }
        GD_CUDA(cudaMalloc(&m->d_thr_off, thr_off.size() * sizeof(int32_t)), "cudaMalloc(threshold offsets)");
        GD_CUDA(cudaMemcpy(m->d_thr_off, thr_off.data(), thr_off.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
                "cudaMemcpy(threshold offsets)");
        if (!wint.empty()) {
            GD_CUDA(cudaMalloc(&m->d_wint, wint.size() * sizeof(int32_t)), "cudaMalloc(walk prefixes)");
            GD_CUDA(cudaMemcpy(m->d_wint, wint.data(), wint.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
                    "cudaMemcpy(walk prefixes)");
        }
        GD_CUDA(cudaMalloc(&m->d_wroots, wroots.size() * sizeof(int32_t)), "cudaMalloc(walk roots)");
        GD_CUDA(cudaMemcpy(m->d_wroots, wroots.data(), wroots.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
                "cudaMemcpy(walk roots)");
        if (!nodes.empty()) {
            GD_CUDA(cudaMalloc(&m->d_nodes, nodes.size() * sizeof(gd::PNode)), "cudaMalloc(nodes)");
            GD_CUDA(cudaMemcpy(m->d_nodes, nodes.data(), nodes.size() * sizeof(gd::PNode), cudaMemcpyHostToDevice),
                    "cudaMemcpy(nodes)");
        }
        if (!roots.empty()) {
            GD_CUDA(cudaMalloc(&m->d_roots, roots.size() * sizeof(int32_t)), "cudaMalloc(roots)");
            GD_CUDA(cudaMemcpy(m->d_roots, roots.data(), roots.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
                    "cudaMemcpy(roots)");
        }
    } else {
        if (m->device >= 0 && !m->coef.empty()) {
            GD_CUDA(cudaMalloc(&m->d_coef, m->coef.size() * sizeof(double)), "cudaMalloc(coef)");
            GD_CUDA(cudaMemcpy(m->d_coef, m->coef.data(), m->coef.size() * sizeof(double), cudaMemcpyHostToDevice),
                    "cudaMemcpy(coef)");
        }
    }
    return GD_OK;
}

void release_model(gd_model* m) {
    if (m->d_grid_nodes) cudaFree(m->d_grid_nodes);
    m->d_grid_nodes = nullptr;
    if (m->d_wnodes) cudaFree(m->d_wnodes);
    m->d_wnodes = nullptr;
    if (m->d_thr) cudaFree(m->d_thr);
    if (m->d_thr_off) cudaFree(m->d_thr_off);
    if (m->d_wroots) cudaFree(m->d_wroots);
    if (m->d_fold) cudaFree(m->d_fold);
    m->d_fold = nullptr;
    if (m->d_wint) cudaFree(m->d_wint);
    m->d_wint = nullptr;
    m->d_thr = nullptr;
    m->d_thr_off = nullptr;
    m->d_wroots = nullptr;
    if (m->d_nodes) cudaFree(m->d_nodes);
    if (m->d_roots) cudaFree(m->d_roots);
    if (m->d_coef) cudaFree(m->d_coef);
    m->d_nodes = nullptr;
    m->d_roots = nullptr;
    m->d_coef = nullptr;
}

int predict_rows_impl(gd_ctx* ctx, const gd_model* m, const double* d_rows, int64_t n_rows, int32_t n_cols,
                      double* d_out, int32_t* d_leaf) {
    if (n_cols != m->n_cols) {
        char buf[128];
        std::snprintf(buf, sizeof(buf), "predict: column mismatch (model expects %d columns, rows have %d)", m->n_cols,
                      n_cols);
        return set_error(GD_ERR_INVALID_ARGUMENT, buf);
    }
    if (n_rows == 0) return GD_OK;
    const int clamp = m->target == GD_TARGET_ENERGY ? 1 : 0;
    int e;
    if (m->kind == GD_KIND_GBT) {
        if (n_cols > gd::kMaxCols) return set_error(GD_ERR_UNSUPPORTED, "predict: more than 1024 columns");
        e = gd::launch_predict_gbt(m->d_nodes, m->d_roots, m->n_trees(), m->base, m->lr, clamp, d_rows, n_rows, n_cols,
                                   d_out, d_leaf, ctx->sm_count, ctx->stream);
    } else {
        e = gd::launch_predict_linear(m->d_coef, m->base, clamp, d_rows, n_rows, n_cols, d_out, ctx->sm_count,
                                      ctx->stream);
    }
    ++ctx->launches;
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "predict kernel launch");
    return GD_OK;
}

int validate_grid(const gd_model* me, const gd_model* mt, const gd_grid* g, const gd_select_opts* o) {
    if (!g || !o) return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: null grid/options");
    if (me->kind != GD_KIND_GBT || mt->kind != GD_KIND_GBT) {
        return set_error(GD_ERR_UNSUPPORTED, "grid_select: energy and time models must be GBT ensembles");
    }
    if (me->target != GD_TARGET_ENERGY || mt->target != GD_TARGET_TIME) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: expected an energy model and a time model");
    }
    if (g->n_cols != me->n_cols || g->n_cols != mt->n_cols) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "predict: column mismatch between grid rows and models");
    }
    if (g->n_cols <= 0 || g->n_cols > gd::kMaxCols) return set_error(GD_ERR_UNSUPPORTED, "grid_select: bad column count");
    if (g->n_clocks <= 0) return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: empty clock catalog");
    if (g->n_apps < 0 || g->n_records < 0 || g->n_cat < 0 || g->n_cat > g->n_cols) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: negative sizes");
    }
    if (!g->rec_of_clock && g->n_records < g->n_apps) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: one record per app required without rec_of_clock");
    }
    if (g->sm_col >= g->n_cols || g->mem_col >= g->n_cols || g->sm_col < -1 || g->mem_col < -1) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: clock column out of range");
    }
    if (o->mode != GD_MODE_TEXT && o->mode != GD_MODE_LITERAL) return set_error(GD_ERR_INVALID_ARGUMENT, "bad mode");
    if (o->objective != GD_OBJECTIVE_ENERGY && o->objective != GD_OBJECTIVE_POWER) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "bad objective");
    }
    return GD_OK;
}

// The partial-evaluation kernel walks a copy of the packed nodes whose clock
// columns are recoded (gd_device.cuh kFeatSm / kFeatMem); built once per
// (model, sm_col, mem_col) on the context stream.
int ensure_fold_state(gd_ctx* ctx, const gd_model* m) {
    if (m->d_fold) return GD_OK;
    GD_CUDA(cudaMalloc(&m->d_fold, 4 * sizeof(int32_t)), "cudaMalloc(fold state)");
    const int32_t none[4] = {-1, -1, 1, 0};  // no state yet: the first check reports a change
    GD_CUDA(cudaMemcpyAsync(m->d_fold, none, sizeof(none), cudaMemcpyHostToDevice, ctx->stream), "fold state");
    return cudaStreamSynchronize(ctx->stream) == cudaSuccess ? GD_OK : set_error(GD_ERR_CUDA, "fold state sync");
}

int ensure_grid_nodes(gd_ctx* ctx, const gd_model* m, int32_t sm_col, int32_t mem_col, int32_t sm_fix, int32_t mem_fix) {
    if (m->d_grid_nodes && m->grid_sm_col == sm_col && m->grid_mem_col == mem_col && m->grid_sm_fix == sm_fix &&
        m->grid_mem_fix == mem_fix)
        return GD_OK;
    if (m->packed_nodes == 0) return GD_OK;
    if (int rc = ensure_fold_state(ctx, m)) return rc;
    if (!m->d_grid_nodes) {
        GD_CUDA(cudaMalloc(&m->d_grid_nodes, static_cast<size_t>(m->packed_nodes) * sizeof(gd::PNode)),
                "cudaMalloc(grid nodes)");
    }
    if (!m->d_wnodes) {
        GD_CUDA(cudaMalloc(&m->d_wnodes, static_cast<size_t>(m->n_wnodes) * sizeof(gd::WNode)),
                "cudaMalloc(walk nodes)");
    }
    int e = gd::launch_recode_clock_nodes(m->d_nodes, m->d_grid_nodes, m->packed_nodes, sm_col, mem_col, ctx->stream);
    ++ctx->launches;
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "recode kernel");
    GD_CUDA(cudaMemsetAsync(m->d_wnodes, 0, static_cast<size_t>(m->n_wnodes) * sizeof(gd::WNode), ctx->stream),
            "memset(walk nodes)");
    e = gd::launch_build_walk_nodes(m->d_grid_nodes, m->packed_nodes, m->d_roots, m->n_trees(), m->d_wroots,
                                    m->d_thr, m->d_thr_off, sm_fix, mem_fix, nullptr, m->d_wnodes, ctx->stream);
    ++ctx->launches;
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "walk-node kernel");
    {  // the device mirror of the state (device-buffer calls check against it)
        static thread_local int32_t st[4];
        st[0] = sm_fix;
        st[1] = mem_fix;
        st[2] = 0;
        st[3] = 0;
        GD_CUDA(cudaMemcpyAsync(m->d_fold, st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream), "fold state");
        GD_CUDA(cudaStreamSynchronize(ctx->stream), "fold state sync");
    }
    m->grid_sm_col = sm_col;
    m->grid_mem_col = mem_col;
    m->grid_sm_fix = sm_fix;
    m->grid_mem_fix = mem_fix;
    return GD_OK;
}

// Timing hook: an event after each launch (the first event precedes them).
cudaEvent_t timing_event(gd_ctx* ctx, size_t i) {
    while (ctx->events.size() <= i) {
        cudaEvent_t ev = nullptr;
        if (cudaEventCreate(&ev) != cudaSuccess) return nullptr;
        ctx->events.push_back(ev);
    }
    return ctx->events[i];
}

void timing_begin(gd_ctx* ctx) {
    ctx->marks.clear();
    cudaEvent_t ev = timing_event(ctx, 0);
    if (ev) cudaEventRecord(ev, ctx->stream);
}

void timing_mark(void* user, const char* name) {
    gd_ctx* ctx = static_cast<gd_ctx*>(user);
    cudaEvent_t ev = timing_event(ctx, ctx->marks.size() + 1);
    if (ev) cudaEventRecord(ev, ctx->stream);
    ctx->marks.push_back(name);
}

gd::GridParams grid_params(const gd_model* me, const gd_model* mt, const gd_grid& g, const gd_select_opts& o,
                           bool general) {
    gd::GridParams p{};
    p.e_nodes = general ? me->d_nodes : me->d_grid_nodes;
    p.e_roots = me->d_roots;
    p.e_trees = me->n_trees();
    p.e_max_pair_nodes = me->max_pair_nodes;
    p.t_max_pair_nodes = mt->max_pair_nodes;
    p.max_tree_nodes = me->max_tree_nodes > mt->max_tree_nodes ? me->max_tree_nodes : mt->max_tree_nodes;
    p.e_base = me->base;
    p.e_lr = me->lr;
    p.t_nodes = general ? mt->d_nodes : mt->d_grid_nodes;
    p.e_wnodes = me->d_wnodes;
    p.t_wnodes = mt->d_wnodes;
    p.e_wroots = me->d_wroots;
    p.t_wroots = mt->d_wroots;
    p.e_wint = me->d_wint;
    p.t_wint = mt->d_wint;
    p.max_wint = me->max_wint > mt->max_wint ? me->max_wint : mt->max_wint;
    p.e_thr = me->d_thr;
    p.t_thr = mt->d_thr;
    p.e_thr_off = me->d_thr_off;
    p.t_thr_off = mt->d_thr_off;
    p.rank16 = me->max_thr_per_feature <= 65535 && mt->max_thr_per_feature <= 65535;
    p.rank8 = me->max_thr_per_feature <= 255 && mt->max_thr_per_feature <= 255;
    p.t_roots = mt->d_roots;
    p.t_trees = mt->n_trees();
    p.t_base = mt->base;
    p.t_lr = mt->lr;
    p.rows = g.rows;
    p.cat_t = g.cat_t;
    p.cat_cols = g.cat_cols;
    p.rec_of_clock = g.rec_of_clock;
    p.sm = g.sm_clock;
    p.mem = g.mem_clock;
    p.budgets = g.budgets;
    p.n_apps = g.n_apps;
    p.n_cols = g.n_cols;
    p.n_cat = g.n_cat;
    p.n_clocks = g.n_clocks;
    p.sm_col = g.sm_col;
    p.mem_col = g.mem_col;
    p.mode = o.mode;
    p.objective = o.objective;
    p.best_effort = o.best_effort;
    p.out_stride = g.n_clocks;
    return p;
}

// Whether a call takes the partial-evaluation pipeline: no per-clock records
// (rec_of_clock), catalog clocks that pack into 16 bits (force_general
// otherwise), and models the walk handles (gd::grid_fast_path_ok).  Every
// other shape runs the general per-candidate kernel -- on the GPU, never an
// error.
bool takes_fast_path(const gd_model* me, const gd_model* mt, const gd_grid& g, const gd_select_opts& o,
                     bool force_general) {
    if (g.rec_of_clock || force_general) return false;
    return gd::grid_fast_path_ok(grid_params(me, mt, g, o, true));
}

// begin_timing: false when the caller already opened the timing interval list
// (the host-buffer path marks its copies around the kernels).  Catalogs wider
// than gd::kMaxClocks run in 512-clock chunks that write the E/T tables
// (row stride = the full catalog), then one wide selection.
// Clock columns with ONE value across a call's catalog (a single memory
// clock, as on the B200 / P100 grids): their tests are folded into the walk
// nodes (launch_build_walk_nodes), so no residue carries them.  0 = varies.
// GDVFS_FOLD=0 disables.
void clock_fix(const int32_t* sm, const int32_t* mem, int64_t C, int32_t& sm_fix, int32_t& mem_fix) {
    sm_fix = mem_fix = 0;
    const char* env = std::getenv("GDVFS_FOLD");
    if ((env && env[0] == '0') || C <= 0) return;
    sm_fix = sm[0];
    mem_fix = mem[0];
    for (int64_t c = 1; c < C; ++c) {
        if (sm[c] != sm_fix) sm_fix = 0;
        if (mem[c] != mem_fix) mem_fix = 0;
    }
}

// Host-side inputs of a large host-buffer call, streamed batch by batch
// (grid_select_host).
struct StreamedInputs {
    const double* rows;
    const double* cat_t;
    const double* budgets;
};

// Device-buffer calls: the catalog stays on the device, so the fold check runs
// there too (launch_fold_check) and each model's walk nodes are rebuilt by a
// kernel that exits at once unless the folded state changed -- no read-back,
// no host sync between the caller's work and the kernels.
int ensure_grid_nodes_device(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid& g) {
    const gd_model* ms[2] = {me, mt != me ? mt : nullptr};
    for (const gd_model* m : ms) {
        if (!m || m->packed_nodes == 0) continue;
        if (int rc = ensure_fold_state(ctx, m)) return rc;
        if (!m->d_grid_nodes || m->grid_sm_col != g.sm_col || m->grid_mem_col != g.mem_col) {
            // new clock columns: recode the grid nodes, then force a walk-node build
            if (int rc = ensure_grid_nodes(ctx, m, g.sm_col, g.mem_col, m->grid_sm_fix, m->grid_mem_fix)) return rc;
            const int32_t none[4] = {-1, -1, 1, 0};
            GD_CUDA(cudaMemcpyAsync(m->d_fold, none, sizeof(none), cudaMemcpyHostToDevice, ctx->stream), "fold state");
            GD_CUDA(cudaStreamSynchronize(ctx->stream), "fold state sync");
        }
    }
    const char* env = std::getenv("GDVFS_FOLD");
    const int enable = !(env && env[0] == '0');
    int e = gd::launch_fold_check(g.sm_clock, g.mem_clock, g.n_clocks, enable, ms[0] ? ms[0]->d_fold : nullptr,
                                  ms[1] ? ms[1]->d_fold : nullptr, ctx->stream);
    ++ctx->launches;
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "fold check kernel");
    for (const gd_model* m : ms) {
        if (!m || m->packed_nodes == 0) continue;
        e = gd::launch_build_walk_nodes(m->d_grid_nodes, m->packed_nodes, m->d_roots, m->n_trees(), m->d_wroots,
                                        m->d_thr, m->d_thr_off, 0, 0, m->d_fold, m->d_wnodes, ctx->stream);
        ++ctx->launches;
        if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "walk-node kernel");
        m->grid_sm_fix = m->grid_mem_fix = -2;  // known on the device only
    }
    return GD_OK;
}

// h_fix: the catalog's folded clocks (clock_fix) when the caller has the
// catalog on the host; null: a device-buffer call (ensure_grid_nodes_device).
int grid_impl(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid& g, const gd_select_opts& o,
              gd_decision* d_out, double* d_e, double* d_t, bool begin_timing = true, bool force_general = false,
              const StreamedInputs* sin = nullptr, const int32_t* h_fix = nullptr) {
    if (g.n_apps == 0) return GD_OK;
    const bool general = !takes_fast_path(me, mt, g, o, force_general);
    if (!general) {
        int rc;
        if (h_fix) {
            rc = ensure_grid_nodes(ctx, me, g.sm_col, g.mem_col, h_fix[0], h_fix[1]);
            if (!rc) rc = ensure_grid_nodes(ctx, mt, g.sm_col, g.mem_col, h_fix[0], h_fix[1]);
        } else {
            rc = ensure_grid_nodes_device(ctx, me, mt, g);
        }
        if (rc) return rc;
    }
    gd::GridParams p = grid_params(me, mt, g, o, general);
    p.out = d_out;
    p.e_out = d_e;
    p.t_out = d_t;
    const int64_t A = g.n_apps, C = g.n_clocks;
    const bool wide = C > gd::kMaxClocks;
    if (sin) {  // the caller left rows / cat_t / budgets on the host for this path
        if (general || wide) return set_error(GD_ERR_UNSUPPORTED, "grid_impl: streamed inputs on a chunked path");
        const int64_t B = gd::grid_batch_apps(p), nb = (A + B - 1) / B;
        if (!ctx->copy_stream) GD_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
        while (static_cast<int64_t>(ctx->batch_events.size()) < nb + 1) {
            cudaEvent_t ev;
            GD_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "batch event");
            ctx->batch_events.push_back(ev);
        }
        // The copy stream starts after everything already on the call's stream
        // (the scratch allocation and the other inputs).
        cudaEvent_t start = ctx->batch_events[nb];
        GD_CUDA(cudaEventRecord(start, ctx->stream), "copy start event");
        GD_CUDA(cudaStreamWaitEvent(ctx->copy_stream, start, 0), "copy stream wait");
        p.h_rows = sin->rows;
        p.h_cat_t = sin->cat_t;
        p.h_budgets = sin->budgets;
        p.copy_stream = ctx->copy_stream;
        p.batch_ready = reinterpret_cast<void* const*>(ctx->batch_events.data());
    }
    // General mode reads per-record time rows (the categorical columns
    // replaced by their time encoding); wide mode needs the full tables.
    Scratch side{ctx->stream};
    const size_t i_rt = side.add(general && g.n_records > 0 ? static_cast<size_t>(g.n_records) * g.n_cols * sizeof(double) : 0);
    const size_t i_we = side.add(wide && !d_e ? static_cast<size_t>(A) * C * sizeof(double) : 0);
    const size_t i_wt = side.add(wide && !d_t ? static_cast<size_t>(A) * C * sizeof(double) : 0);
    const size_t i_wd = side.add(wide ? static_cast<size_t>(A) * sizeof(gd_decision) : 0);
    GD_CUDA(side.alloc(), "cudaMallocAsync(grid side buffers)");
    if (general && g.n_records > 0) {
        p.rows_t = static_cast<double*>(side.ptr(i_rt));
        int e = gd::launch_build_rows_t(g.rows, g.cat_t, g.cat_cols, g.n_cat, g.n_records, g.n_cols,
                                        const_cast<double*>(p.rows_t), ctx->stream);
        ++ctx->launches;
        if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "rows_t kernel");
    }
    gd::LaunchMark mark = nullptr;
    if (ctx->timing) {
        if (begin_timing) timing_begin(ctx);
        mark = timing_mark;
    }
    auto run = [&](const gd::GridParams& q) -> int {
        Scratch s{ctx->stream, &ctx->pbuf[0]};
        const size_t bytes = gd::grid_scratch_bytes(q, general);
        const size_t i_scr = s.add(bytes);
        GD_CUDA(s.alloc(), "cudaMallocAsync(grid scratch)");
        int e = gd::launch_grid_select(q, general, ctx->sm_count, ctx->stream, s.ptr(i_scr), bytes, &ctx->launches,
                                       mark, ctx);
        if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "grid kernel launch");
        return GD_OK;
    };
    if (!wide) return run(p);
    double* E = d_e ? d_e : static_cast<double*>(side.ptr(i_we));
    double* T = d_t ? d_t : static_cast<double*>(side.ptr(i_wt));
    for (int64_t c0 = 0; c0 < C; c0 += gd::kMaxClocks) {
        gd::GridParams q = p;
        q.n_clocks = static_cast<int32_t>(C - c0 < gd::kMaxClocks ? C - c0 : gd::kMaxClocks);
        q.sm = g.sm_clock + c0;
        q.mem = g.mem_clock + c0;
        if (g.rec_of_clock) q.rec_of_clock = g.rec_of_clock + c0;
        q.e_out = E + c0;
        q.t_out = T + c0;
        q.out = static_cast<gd_decision*>(side.ptr(i_wd));  // per-chunk choices are discarded
        q.out_stride = C;
        int rc = run(q);
        if (rc) return rc;
    }
    gd::SelectParams sp{};
    sp.energy = E;
    sp.time = T;
    sp.sm = g.sm_clock;
    sp.budgets = g.budgets;
    sp.out = d_out;
    sp.n_apps = A;
    sp.n_clocks = static_cast<int32_t>(C);
    sp.mode = o.mode;
    sp.objective = o.objective;
    sp.best_effort = o.best_effort;
    int e = gd::launch_select_wide(sp, ctx->sm_count, ctx->stream);
    ++ctx->launches;
    if (mark) mark(ctx, "select");
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "select kernel launch");
    return GD_OK;
}

}  // namespace

extern "C" {

const char* gd_last_error(void) { return gdh::g_error.c_str(); }

const char* gd_version(void) { return "gdvfs-b200 0.1 (sm_100a)"; }

int gd_ctx_create(int32_t device, gd_ctx** out) {
    if (!out) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_ctx_create: null out");
    *out = nullptr;
    int n = 0;
    GD_CUDA(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_ctx_create: no such device");
    GD_CUDA(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    GD_CUDA(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) {
        return set_error(GD_ERR_CUDA, std::string("gd_ctx_create: sm_100a kernels need a Blackwell GPU, found ") +
                                          prop.name);
    }
    auto* c = new gd_ctx;
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_error(e, "cudaStreamCreate");
    }
    c->stream = c->own;
    // Keep stream-ordered scratch in the pool between calls.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = c;
    return GD_OK;
}

int gd_ctx_destroy(gd_ctx* ctx) {
    if (!ctx) return GD_OK;
    cudaSetDevice(ctx->device);
    if (ctx->own) {
        cudaStreamSynchronize(ctx->own);
        cudaStreamDestroy(ctx->own);
    }
    for (cudaEvent_t ev : ctx->events) cudaEventDestroy(ev);
    if (ctx->stage_ev) {
        cudaEventSynchronize(ctx->stage_ev);
        cudaEventDestroy(ctx->stage_ev);
    }
    if (ctx->stage) cudaFreeHost(ctx->stage);
    for (gd_graph_entry& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
    if (ctx->out_stage) cudaFreeHost(ctx->out_stage);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    for (cudaEvent_t ev : ctx->batch_events) cudaEventDestroy(ev);
    for (gd_pbuf& b : ctx->pbuf) {
        if (b.ev) cudaEventDestroy(b.ev);
        if (b.base) cudaFree(b.base);
    }
    delete ctx;
    return GD_OK;
}

int gd_ctx_set_stream(gd_ctx* ctx, void* stream) {
    if (!ctx) return set_error(GD_ERR_INVALID_ARGUMENT, "null gd_ctx");
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    return GD_OK;
}

int gd_ctx_synchronize(gd_ctx* ctx) {
    int rc = activate(ctx);
    if (rc) return rc;
    GD_CUDA(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    return GD_OK;
}

int64_t gd_ctx_launch_count(const gd_ctx* ctx) { return ctx ? ctx->launches : -1; }

int gd_ctx_set_timing(gd_ctx* ctx, int on) {
    if (!ctx) return set_error(GD_ERR_INVALID_ARGUMENT, "null gd_ctx");
    ctx->timing = on != 0;
    ctx->marks.clear();
    return GD_OK;
}

int gd_ctx_kernel_times(gd_ctx* ctx, float* ms, const char** names, int32_t max, int32_t* n) {
    int rc = activate(ctx);
    if (rc) return rc;
    if (!n) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_ctx_kernel_times: null n");
    const int32_t k = static_cast<int32_t>(ctx->marks.size());
    *n = k;
    for (int32_t i = 0; i < k && i < max; ++i) {
        GD_CUDA(cudaEventSynchronize(ctx->events[static_cast<size_t>(i) + 1]), "cudaEventSynchronize");
        float t = 0.0f;
        GD_CUDA(cudaEventElapsedTime(&t, ctx->events[static_cast<size_t>(i)], ctx->events[static_cast<size_t>(i) + 1]),
                "cudaEventElapsedTime");
        if (ms) ms[i] = t;
        if (names) names[i] = ctx->marks[static_cast<size_t>(i)];
    }
    return GD_OK;
}

int gd_model_upload_gbt(gd_ctx* ctx, const gd_forest_view* f, double base, double lr, int32_t n_cols, int32_t target,
                        gd_model** out) {
    if (!out || !f) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_upload_gbt: null argument");
    *out = nullptr;
    int rc = activate_opt(ctx);
    if (rc) return rc;
    if (n_cols < 0) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_upload_gbt: negative column count");
    if (target != GD_TARGET_ENERGY && target != GD_TARGET_TIME) return set_error(GD_ERR_INVALID_ARGUMENT, "bad target");
    if (f->n_trees < 0 || (f->n_trees > 0 && !f->tree_offsets)) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_upload_gbt: bad tree offsets");
    }
    auto* m = new gd_model;
    m->uid = next_model_uid();
    m->device = ctx ? ctx->device : -1;
    m->kind = GD_KIND_GBT;
    m->target = target;
    m->n_cols = n_cols;
    m->base = base;
    m->lr = lr;
    const int64_t n_nodes = f->n_trees > 0 ? f->tree_offsets[f->n_trees] - f->tree_offsets[0] : 0;
    m->offsets.assign(f->tree_offsets, f->tree_offsets + f->n_trees + 1);
    if (f->n_trees == 0) m->offsets.assign(1, 0);
    const int64_t o0 = m->offsets.front();
    for (auto& o : m->offsets) o -= o0;
    if (n_nodes > 0) {
        m->feature.assign(f->feature + o0, f->feature + o0 + n_nodes);
        m->threshold.assign(f->threshold + o0, f->threshold + o0 + n_nodes);
        m->left.assign(f->left + o0, f->left + o0 + n_nodes);
        m->right.assign(f->right + o0, f->right + o0 + n_nodes);
        m->leaf.assign(f->leaf_value + o0, f->leaf_value + o0 + n_nodes);
    }
    rc = upload_model(m);
    if (rc) {
        release_model(m);
        delete m;
        return rc;
    }
    *out = m;
    return GD_OK;
}

int gd_model_upload_linear(gd_ctx* ctx, const double* coef, int32_t n_cols, double intercept, int32_t kind,
                           int32_t target, gd_model** out) {
    if (!out || (n_cols > 0 && !coef) || n_cols < 0) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_upload_linear: bad argument");
    }
    *out = nullptr;
    int rc = activate_opt(ctx);
    if (rc) return rc;
    if (kind != GD_KIND_OLS && kind != GD_KIND_LASSO) return set_error(GD_ERR_INVALID_ARGUMENT, "bad linear kind");
    auto* m = new gd_model;
    m->uid = next_model_uid();
    m->device = ctx ? ctx->device : -1;
    m->kind = kind;
    m->target = target;
    m->n_cols = n_cols;
    m->base = intercept;
    m->coef.assign(coef, coef + n_cols);
    m->offsets.assign(1, 0);
    rc = upload_model(m);
    if (rc) {
        release_model(m);
        delete m;
        return rc;
    }
    *out = m;
    return GD_OK;
}

int gd_model_load_file(gd_ctx* ctx, const char* path, gd_model** out) {
    if (!out) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_load_file: null out");
    *out = nullptr;
    int rc = activate_opt(ctx);
    if (rc) return rc;
    auto* m = new gd_model;
    m->uid = next_model_uid();
    m->device = ctx ? ctx->device : -1;
    rc = gdh::parse_model_file(path, *m);
    if (!rc) rc = upload_model(m);
    if (rc) {
        release_model(m);
        delete m;
        return rc;
    }
    *out = m;
    return GD_OK;
}

}  // extern "C"

namespace gdh {

int clone_model(gd_ctx* ctx, const gd_model* src, gd_model** out) {
    if (!src || !out) return set_error(GD_ERR_INVALID_ARGUMENT, "clone_model: null argument");
    *out = nullptr;
    int rc = activate(ctx);
    if (rc) return rc;
    auto* m = new gd_model;
    m->uid = next_model_uid();
    m->device = ctx->device;
    m->kind = src->kind;
    m->target = src->target;
    m->n_cols = src->n_cols;
    m->base = src->base;
    m->lr = src->lr;
    m->offsets = src->offsets;
    m->feature = src->feature;
    m->left = src->left;
    m->right = src->right;
    m->threshold = src->threshold;
    m->leaf = src->leaf;
    m->coef = src->coef;
    m->columns = src->columns;
    rc = upload_model(m);
    if (rc) {
        release_model(m);
        delete m;
        return rc;
    }
    *out = m;
    return GD_OK;
}

}  // namespace gdh

extern "C" {

int gd_fit_gbt(gd_ctx* ctx, const double* rows, int64_t n_rows, int32_t n_cols, const double* targets,
               const gd_gbt_config* cfg, int32_t target, gd_model** out) {
    if (!out || !cfg) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_fit_gbt: null argument");
    *out = nullptr;
    int rc = activate(ctx);
    if (rc) return rc;
    // models.cpp:37-42 (require_rows) and :46-53 (validate_config), same messages.
    if (n_rows <= 0 || !rows) return set_error(GD_ERR_INVALID_ARGUMENT, "fit_gbt: empty training matrix");
    if (!targets) return set_error(GD_ERR_INVALID_ARGUMENT, "fit_gbt: row/target count mismatch");
    if (cfg->iterations < 0) return set_error(GD_ERR_INVALID_ARGUMENT, "gbt config: iterations must be >= 0");
    if (cfg->depth < 1) return set_error(GD_ERR_INVALID_ARGUMENT, "gbt config: depth must be >= 1");
    if (!(cfg->learning_rate > 0.0) || cfg->learning_rate > 1.0) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "gbt config: learning_rate must lie in (0, 1]");
    }
    if (cfg->l2_leaf_reg < 0.0) return set_error(GD_ERR_INVALID_ARGUMENT, "gbt config: l2_leaf_reg must be >= 0");
    if (n_cols < 0 || n_rows > INT32_MAX) return set_error(GD_ERR_INVALID_ARGUMENT, "fit_gbt: bad shape");
    if (target != GD_TARGET_ENERGY && target != GD_TARGET_TIME) return set_error(GD_ERR_INVALID_ARGUMENT, "bad target");
    auto* m = new gd_model;
    m->uid = next_model_uid();
    m->device = ctx->device;
    m->kind = GD_KIND_GBT;
    m->target = target;
    m->n_cols = n_cols;
    m->lr = cfg->learning_rate;
    rc = gdh::fit_gbt_device(ctx, rows, n_rows, n_cols, targets, *cfg, m->offsets, m->feature, m->threshold, m->left,
                             m->right, m->leaf, m->base);
    if (!rc) rc = upload_model(m);
    if (rc) {
        release_model(m);
        delete m;
        return rc;
    }
    *out = m;
    return GD_OK;
}

int gd_model_info_get(const gd_model* m, gd_model_info* out) {
    if (!m || !out) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_info_get: null argument");
    out->kind = m->kind;
    out->target = m->target;
    out->n_cols = m->n_cols;
    out->n_trees = m->n_trees();
    out->n_nodes = static_cast<int64_t>(m->feature.size());
    out->max_depth = m->max_depth;
    out->pad = 0;
    out->base_prediction = m->base;
    out->learning_rate = m->lr;
    return GD_OK;
}

const char* gd_model_column(const gd_model* m, int32_t j) {
    if (!m || j < 0 || static_cast<size_t>(j) >= m->columns.size()) return nullptr;
    return m->columns[static_cast<size_t>(j)].c_str();
}

int gd_model_export(const gd_model* m, int64_t* tree_offsets, int32_t* feature, double* threshold, int32_t* left,
                    int32_t* right, double* leaf_value) {
    if (!m) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_model_export: null model");
    if (tree_offsets) std::memcpy(tree_offsets, m->offsets.data(), m->offsets.size() * sizeof(int64_t));
    if (feature) std::memcpy(feature, m->feature.data(), m->feature.size() * sizeof(int32_t));
    if (threshold) std::memcpy(threshold, m->threshold.data(), m->threshold.size() * sizeof(double));
    if (left) std::memcpy(left, m->left.data(), m->left.size() * sizeof(int32_t));
    if (right) std::memcpy(right, m->right.data(), m->right.size() * sizeof(int32_t));
    if (leaf_value) std::memcpy(leaf_value, m->leaf.data(), m->leaf.size() * sizeof(double));
    return GD_OK;
}

int gd_model_free(gd_model* m) {
    if (!m) return GD_OK;
    if (m->device >= 0) cudaSetDevice(m->device);
    release_model(m);
    delete m;
    return GD_OK;
}

int gd_predict_rows_device(gd_ctx* ctx, const gd_model* m, const double* d_rows, int64_t n_rows, int32_t n_cols,
                           double* d_out, int32_t* d_leaf) {
    int rc = activate(ctx);
    if (rc) return rc;
    if ((rc = check_model(ctx, m, "predict"))) return rc;
    if (n_rows < 0 || (n_rows > 0 && (!d_rows || !d_out))) return set_error(GD_ERR_INVALID_ARGUMENT, "predict: bad rows");
    return predict_rows_impl(ctx, m, d_rows, n_rows, n_cols, d_out, d_leaf);
}

int gd_predict_rows(gd_ctx* ctx, const gd_model* m, const double* rows, int64_t n_rows, int32_t n_cols, double* out,
                    int32_t* leaf_ids) {
    int rc = activate(ctx);
    if (rc) return rc;
    if ((rc = check_model(ctx, m, "predict"))) return rc;
    if (n_rows < 0 || (n_rows > 0 && (!rows || !out))) return set_error(GD_ERR_INVALID_ARGUMENT, "predict: bad rows");
    if (n_cols != m->n_cols) return predict_rows_impl(ctx, m, nullptr, 0, n_cols, nullptr, nullptr);
    if (n_rows == 0) return GD_OK;
    Scratch s{ctx->stream};
    const size_t i_rows = s.add(static_cast<size_t>(n_rows) * n_cols * sizeof(double));
    const size_t i_out = s.add(static_cast<size_t>(n_rows) * sizeof(double));
    const size_t i_leaf = s.add(leaf_ids ? static_cast<size_t>(n_rows) * m->n_trees() * sizeof(int32_t) : 0);
    GD_CUDA(s.alloc(), "cudaMallocAsync");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_rows), rows, static_cast<size_t>(n_rows) * n_cols * sizeof(double),
                            cudaMemcpyHostToDevice, ctx->stream),
            "H2D rows");
    rc = predict_rows_impl(ctx, m, static_cast<double*>(s.ptr(i_rows)), n_rows, n_cols,
                           static_cast<double*>(s.ptr(i_out)), static_cast<int32_t*>(s.ptr(i_leaf)));
    if (rc) return rc;
    GD_CUDA(cudaMemcpyAsync(out, s.ptr(i_out), static_cast<size_t>(n_rows) * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream),
            "D2H out");
    if (leaf_ids && m->n_trees() > 0) {
        GD_CUDA(cudaMemcpyAsync(leaf_ids, s.ptr(i_leaf), static_cast<size_t>(n_rows) * m->n_trees() * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream),
                "D2H leaf ids");
    }
    GD_CUDA(cudaStreamSynchronize(ctx->stream), "predict sync");
    return GD_OK;
}

int gd_grid_select_device(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid* g,
                          const gd_select_opts* o, gd_decision* d_out, double* d_e, double* d_t) {
    int rc = activate(ctx);
    if (rc) return rc;
    if ((rc = check_model(ctx, me, "grid_select")) || (rc = check_model(ctx, mt, "grid_select"))) return rc;
    if ((rc = validate_grid(me, mt, g, o))) return rc;
    if (!d_out) return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: null decisions");
    return grid_impl(ctx, me, mt, *g, *o, d_out, d_e, d_t);
}

}  // extern "C"

namespace {

// Small host-buffer calls (the configs[4] stream) replay a captured graph:
// one cudaGraphLaunch instead of a staged copy, three kernel launches and a
// result copy issued one by one (GDVFS_GRAPHS=0 disables).
bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("GDVFS_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool same_key(const gd_graph_entry& a, const gd_graph_entry& b) {
    return a.me == b.me && a.mt == b.mt && a.n_apps == b.n_apps && a.n_records == b.n_records && a.n_clocks == b.n_clocks && a.n_cols == b.n_cols &&
           a.n_cat == b.n_cat && a.sm_col == b.sm_col && a.mem_col == b.mem_col && a.mode == b.mode &&
           a.objective == b.objective && a.best_effort == b.best_effort && a.stream == b.stream;
}

gd_graph_entry* find_graph(gd_ctx* ctx, const gd_graph_entry& key) {
    for (size_t i = 0; i < ctx->graphs.size(); ++i) {
        gd_graph_entry& e = ctx->graphs[i];
        if (!same_key(e, key)) continue;
        if (e.gen0 != ctx->pbuf[0].generation || e.gen1 != ctx->pbuf[1].generation) {  // buffers moved
            cudaGraphExecDestroy(e.exec);
            ctx->graphs.erase(ctx->graphs.begin() + static_cast<std::ptrdiff_t>(i));
            return nullptr;
        }
        return &e;
    }
    return nullptr;
}

// Capture the pipeline of a call that just ran (so every buffer is sized and
// every model structure built): staged inputs -> kernels -> decisions into
// ctx->out_stage.  Failures leave no entry (the normal path keeps working).
void capture_graph(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid& dg, const gd_select_opts& o,
                   gd_graph_entry key, void* dev_in, size_t in_end, gd_decision* dev_out, const int32_t* fix) {
    const size_t out_bytes = static_cast<size_t>(dg.n_apps) * sizeof(gd_decision);
    if (!ctx->out_stage && cudaHostAlloc(reinterpret_cast<void**>(&ctx->out_stage), kStageLimit, cudaHostAllocMapped) !=
                               cudaSuccess) {
        ctx->out_stage = nullptr;
        cudaGetLastError();
        return;
    }
    // Decisions go straight from the selection epilogue into the mapped
    // pinned staging (24 B per app over the bus) instead of a device buffer
    // plus a copy node (GDVFS_GRAPH_D2H=1 keeps the copy).
    gd_decision* host_out = nullptr;
    const char* d2h = std::getenv("GDVFS_GRAPH_D2H");
    if (!(d2h && d2h[0] == '1') &&
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&host_out), ctx->out_stage, 0) != cudaSuccess) {
        host_out = nullptr;
        cudaGetLastError();
    }
    const int64_t launches = ctx->launches;
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
        ok = cudaMemcpyAsync(dev_in, ctx->stage, in_end, cudaMemcpyHostToDevice, ctx->stream) == cudaSuccess;
        ok = ok && grid_impl(ctx, me, mt, dg, o, host_out ? host_out : dev_out, nullptr, nullptr, false, false, nullptr,
                             fix) == GD_OK;
        if (!host_out) {
            ok = ok &&
                 cudaMemcpyAsync(ctx->out_stage, dev_out, out_bytes, cudaMemcpyDeviceToHost, ctx->stream) == cudaSuccess;
        }
        ok = (cudaStreamEndCapture(ctx->stream, &graph) == cudaSuccess) && ok;
    }
    ctx->launches = launches;
    cudaGraphExec_t exec = nullptr;
    if (ok && graph) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (!ok || !exec) return;
    key.gen0 = ctx->pbuf[0].generation;
    key.gen1 = ctx->pbuf[1].generation;
    key.exec = exec;
    if (ctx->graphs.size() >= 8) {
        cudaGraphExecDestroy(ctx->graphs.front().exec);
        ctx->graphs.erase(ctx->graphs.begin());
    }
    ctx->graphs.push_back(key);
}

}  // namespace

namespace gdh {

// gd_grid_select's body.  With keep_dev_out set, the decisions are left in
// the context's persistent device buffer (*keep_dev_out, valid until the
// next call on ctx) instead of being copied to `out`: the multi-device path
// gathers them with NCCL (gd_multi.cpp).
int grid_select_host(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid* g, const gd_select_opts* o,
                     gd_decision* out, double* e_out, double* t_out, gd_decision** keep_dev_out) {
    int rc = activate(ctx);
    if (rc) return rc;
    if ((rc = check_model(ctx, me, "grid_select")) || (rc = check_model(ctx, mt, "grid_select"))) return rc;
    if ((rc = validate_grid(me, mt, g, o))) return rc;
    if (g->n_apps > 0 && ((!out && !keep_dev_out) || !g->rows || !g->budgets || !g->sm_clock || !g->mem_clock ||
                          (g->n_cat > 0 && (!g->cat_t || !g->cat_cols)))) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: null input array");
    }
    if (g->n_apps == 0) return GD_OK;
    const int64_t A = g->n_apps, R = g->n_records, C = g->n_clocks;
    bool force_general = false;
    for (int64_t c = 0; c < C; ++c) {
        if (g->sm_clock[c] <= 0 || g->mem_clock[c] <= 0) {
            return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: clock frequencies must be positive");
        }
        if (g->sm_clock[c] > 65535 || g->mem_clock[c] > 65535) force_general = true;  // no 16-bit clock keys
    }
    for (int32_t k = 0; k < g->n_cat; ++k) {
        if (g->cat_cols[k] < 0 || g->cat_cols[k] >= g->n_cols) {
            return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: categorical column out of range");
        }
    }
    if (g->rec_of_clock) {
        for (int64_t i = 0; i < A * C; ++i) {
            if (g->rec_of_clock[i] < 0 || g->rec_of_clock[i] >= R) {
                return set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: record index out of range");
            }
        }
    }
    int32_t fix[2];
    clock_fix(g->sm_clock, g->mem_clock, C, fix[0], fix[1]);
    Scratch s{ctx->stream, &ctx->pbuf[1]};
    const size_t i_rows = s.add(static_cast<size_t>(R) * g->n_cols * sizeof(double));
    const size_t i_cat = s.add(static_cast<size_t>(R) * g->n_cat * sizeof(double));
    const size_t i_catc = s.add(static_cast<size_t>(g->n_cat) * sizeof(int32_t));
    const size_t i_rec = s.add(g->rec_of_clock ? static_cast<size_t>(A) * C * sizeof(int32_t) : 0);
    const size_t i_sm = s.add(static_cast<size_t>(C) * sizeof(int32_t));
    const size_t i_mem = s.add(static_cast<size_t>(C) * sizeof(int32_t));
    const size_t i_bud = s.add(static_cast<size_t>(A) * sizeof(double));
    const size_t i_out = s.add(static_cast<size_t>(A) * sizeof(gd_decision));
    const size_t i_e = s.add(e_out ? static_cast<size_t>(A) * C * sizeof(double) : 0);
    const size_t i_t = s.add(t_out ? static_cast<size_t>(A) * C * sizeof(double) : 0);
    const size_t in_end0 = s.pieces[i_bud].first + s.pieces[i_bud].second;
    const bool graphable = graphs_enabled() && !keep_dev_out && !ctx->timing && !e_out && !t_out &&
                           takes_fast_path(me, mt, *g, *o, force_general) && C <= gd::kMaxClocks &&
                           in_end0 <= kStageLimit && static_cast<size_t>(A) * sizeof(gd_decision) <= kStageLimit;
    gd_graph_entry key;
    key.me = me->uid;
    key.mt = mt->uid;
    key.n_apps = A;
    key.n_records = R;
    key.n_clocks = static_cast<int32_t>(C);
    key.n_cols = g->n_cols;
    key.n_cat = g->n_cat;
    key.sm_col = g->sm_col;
    key.mem_col = g->mem_col;
    key.mode = o->mode;
    key.objective = o->objective;
    key.best_effort = o->best_effort;
    key.stream = ctx->stream;
    const std::pair<size_t, const void*> inputs[] = {{i_rows, g->rows},        {i_cat, g->cat_t},
                                                     {i_catc, g->cat_cols},    {i_rec, g->rec_of_clock},
                                                     {i_sm, g->sm_clock},      {i_mem, g->mem_clock},
                                                     {i_bud, g->budgets}};
    if (graphable && ctx->stage) {
        gd_graph_entry* hit = find_graph(ctx, key);
        // The graph holds the models' grid nodes as recoded for its clock
        // columns; a call with other columns in between rebuilt them in place.
        if (hit && (me->grid_sm_col != g->sm_col || me->grid_mem_col != g->mem_col || mt->grid_sm_col != g->sm_col ||
                    mt->grid_mem_col != g->mem_col || me->grid_sm_fix != fix[0] || me->grid_mem_fix != fix[1] ||
                    mt->grid_sm_fix != fix[0] || mt->grid_mem_fix != fix[1])) {
            cudaGraphExecDestroy(hit->exec);
            ctx->graphs.erase(ctx->graphs.begin() + (hit - ctx->graphs.data()));
            hit = nullptr;
        }
        if (hit) {
            GD_CUDA(cudaEventSynchronize(ctx->stage_ev), "stage reuse");
            for (const auto& in : inputs) {
                if (s.pieces[in.first].second) std::memcpy(ctx->stage + s.pieces[in.first].first, in.second, s.pieces[in.first].second);
            }
            GD_CUDA(cudaGraphLaunch(hit->exec, ctx->stream), "cudaGraphLaunch");
            ctx->launches += 3;
            GD_CUDA(cudaEventRecord(ctx->stage_ev, ctx->stream), "stage event record");
            GD_CUDA(cudaStreamSynchronize(ctx->stream), "grid sync");
            std::memcpy(out, ctx->out_stage, static_cast<size_t>(A) * sizeof(gd_decision));
            return GD_OK;
        }
    }
    GD_CUDA(s.alloc(), "cudaMallocAsync");
    if (ctx->timing) timing_begin(ctx);
    // A large call of several app batches on the fast path streams its rows
    // in batch by batch, overlapping the upload with the kernels
    // (GDVFS_STREAM_INPUTS=0 disables).
    bool stream_in = false;
    if (in_end0 > kStageLimit && !g->rec_of_clock && C <= gd::kMaxClocks && !force_general &&
        takes_fast_path(me, mt, *g, *o, force_general)) {
        const char* env = std::getenv("GDVFS_STREAM_INPUTS");
        if (!env || env[0] != '0') stream_in = gd::grid_batch_apps(grid_params(me, mt, *g, *o, false)) < A;
    }
    // Inputs occupy the scratch prefix [0, in_end).  Small calls (the online
    // stream's 64-job batches) pack them into pinned staging with the same
    // offsets and move them in ONE copy: per-copy latency, not bandwidth,
    // bounds them.  Large calls copy each array straight from the caller.
    const size_t in_end = in_end0;
    if (in_end <= kStageLimit) {
        if (!ctx->stage_ev) GD_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev, cudaEventDisableTiming), "stage event");
        GD_CUDA(cudaEventSynchronize(ctx->stage_ev), "stage reuse");
        if (!ctx->stage) {
            GD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->stage), kStageLimit, cudaHostAllocDefault),
                    "cudaHostAlloc(stage)");
            ctx->stage_bytes = kStageLimit;
        }
        for (const auto& in : inputs) {
            if (s.pieces[in.first].second) std::memcpy(ctx->stage + s.pieces[in.first].first, in.second, s.pieces[in.first].second);
        }
        GD_CUDA(cudaMemcpyAsync(s.base, ctx->stage, in_end, cudaMemcpyHostToDevice, ctx->stream), "H2D staged inputs");
        GD_CUDA(cudaEventRecord(ctx->stage_ev, ctx->stream), "stage event record");
    } else if (stream_in) {
        // Several app batches on the fast path: the small inputs now, rows /
        // cat_t / budgets batch by batch on the copy stream (grid_impl).
        for (size_t i : {i_catc, i_sm, i_mem}) {
            const void* src = i == i_catc ? static_cast<const void*>(g->cat_cols)
                                          : (i == i_sm ? static_cast<const void*>(g->sm_clock) : g->mem_clock);
            if (s.pieces[i].second) {
                GD_CUDA(cudaMemcpyAsync(s.ptr(i), src, s.pieces[i].second, cudaMemcpyHostToDevice, ctx->stream),
                        "H2D grid input");
            }
        }
    } else {
        // The rows go straight from the caller's buffer; the rest (scratch
        // range [cat_t, budgets]) is packed into the pinned staging while
        // that copy runs and follows in one more copy, when it fits.
        const size_t rest0 = s.pieces[i_cat].first, rest = in_end - rest0;
        if (s.pieces[i_rows].second) {
            GD_CUDA(cudaMemcpyAsync(s.ptr(i_rows), g->rows, s.pieces[i_rows].second, cudaMemcpyHostToDevice,
                                    ctx->stream),
                    "H2D rows");
        }
        if (rest <= kStageLimit) {
            if (!ctx->stage_ev) GD_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev, cudaEventDisableTiming), "stage event");
            GD_CUDA(cudaEventSynchronize(ctx->stage_ev), "stage reuse");
            if (!ctx->stage) {
                GD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->stage), kStageLimit, cudaHostAllocDefault),
                        "cudaHostAlloc(stage)");
                ctx->stage_bytes = kStageLimit;
            }
            for (const auto& in : inputs) {
                if (in.first == i_rows || !s.pieces[in.first].second) continue;
                std::memcpy(ctx->stage + (s.pieces[in.first].first - rest0), in.second, s.pieces[in.first].second);
            }
            GD_CUDA(cudaMemcpyAsync(s.base + rest0, ctx->stage, rest, cudaMemcpyHostToDevice, ctx->stream),
                    "H2D staged inputs");
            GD_CUDA(cudaEventRecord(ctx->stage_ev, ctx->stream), "stage event record");
        } else {
            for (const auto& in : inputs) {
                if (in.first == i_rows || !s.pieces[in.first].second) continue;
                GD_CUDA(cudaMemcpyAsync(s.ptr(in.first), in.second, s.pieces[in.first].second, cudaMemcpyHostToDevice,
                                        ctx->stream),
                        "H2D grid input");
            }
        }
    }
    gd_grid dg = *g;
    dg.rows = static_cast<double*>(s.ptr(i_rows));
    dg.cat_t = static_cast<double*>(s.ptr(i_cat));
    dg.cat_cols = static_cast<int32_t*>(s.ptr(i_catc));
    dg.rec_of_clock = static_cast<int32_t*>(s.ptr(i_rec));
    dg.sm_clock = static_cast<int32_t*>(s.ptr(i_sm));
    dg.mem_clock = static_cast<int32_t*>(s.ptr(i_mem));
    dg.budgets = static_cast<double*>(s.ptr(i_bud));
    if (ctx->timing) timing_mark(ctx, "h2d");
    const StreamedInputs sin{g->rows, g->cat_t, g->budgets};
    rc = grid_impl(ctx, me, mt, dg, *o, static_cast<gd_decision*>(s.ptr(i_out)), static_cast<double*>(s.ptr(i_e)),
                   static_cast<double*>(s.ptr(i_t)), false, force_general, stream_in ? &sin : nullptr, fix);
    if (rc) return rc;
    if (keep_dev_out) {
        *keep_dev_out = static_cast<gd_decision*>(s.ptr(i_out));
    } else {
        GD_CUDA(cudaMemcpyAsync(out, s.ptr(i_out), static_cast<size_t>(A) * sizeof(gd_decision), cudaMemcpyDeviceToHost,
                                ctx->stream),
                "D2H decisions");
    }
    if (e_out) {
        GD_CUDA(cudaMemcpyAsync(e_out, s.ptr(i_e), static_cast<size_t>(A) * C * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream),
                "D2H energy");
    }
    if (t_out) {
        GD_CUDA(cudaMemcpyAsync(t_out, s.ptr(i_t), static_cast<size_t>(A) * C * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream),
                "D2H time");
    }
    if (ctx->timing) timing_mark(ctx, "d2h");
    GD_CUDA(cudaStreamSynchronize(ctx->stream), "grid sync");
    if (graphable && ctx->stage) capture_graph(ctx, me, mt, dg, *o, key, s.base, in_end, static_cast<gd_decision*>(s.ptr(i_out)), fix);
    return GD_OK;
}

}  // namespace gdh

extern "C" {

int gd_grid_select(gd_ctx* ctx, const gd_model* me, const gd_model* mt, const gd_grid* g, const gd_select_opts* o,
                   gd_decision* out, double* e_out, double* t_out) {
    return gdh::grid_select_host(ctx, me, mt, g, o, out, e_out, t_out, nullptr);
}

int gd_select(gd_ctx* ctx, const double* energy, const double* time, int64_t n_apps, const int32_t* sm_clock,
              int32_t n_clocks, const double* budgets, const gd_select_opts* o, gd_decision* out) {
    int rc = activate(ctx);
    if (rc) return rc;
    if (!o || n_apps < 0 || n_clocks <= 0 ||
        (n_apps > 0 && (!energy || !time || !sm_clock || !budgets || !out))) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "gd_select: bad arguments");
    }
    if (n_apps == 0) return GD_OK;
    const int64_t A = n_apps, C = n_clocks;
    Scratch s{ctx->stream};
    const size_t i_e = s.add(static_cast<size_t>(A) * C * sizeof(double));
    const size_t i_t = s.add(static_cast<size_t>(A) * C * sizeof(double));
    const size_t i_sm = s.add(static_cast<size_t>(C) * sizeof(int32_t));
    const size_t i_b = s.add(static_cast<size_t>(A) * sizeof(double));
    const size_t i_o = s.add(static_cast<size_t>(A) * sizeof(gd_decision));
    GD_CUDA(s.alloc(), "cudaMallocAsync");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_e), energy, s.pieces[i_e].second, cudaMemcpyHostToDevice, ctx->stream), "H2D E");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_t), time, s.pieces[i_t].second, cudaMemcpyHostToDevice, ctx->stream), "H2D T");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_sm), sm_clock, s.pieces[i_sm].second, cudaMemcpyHostToDevice, ctx->stream), "H2D sm");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_b), budgets, s.pieces[i_b].second, cudaMemcpyHostToDevice, ctx->stream), "H2D b");
    gd::SelectParams p{};
    p.energy = static_cast<double*>(s.ptr(i_e));
    p.time = static_cast<double*>(s.ptr(i_t));
    p.sm = static_cast<int32_t*>(s.ptr(i_sm));
    p.budgets = static_cast<double*>(s.ptr(i_b));
    p.out = static_cast<gd_decision*>(s.ptr(i_o));
    p.n_apps = A;
    p.n_clocks = n_clocks;
    p.mode = o->mode;
    p.objective = o->objective;
    p.best_effort = o->best_effort;
    int e = gd::launch_select(p, ctx->sm_count, ctx->stream);
    ++ctx->launches;
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "select kernel launch");
    GD_CUDA(cudaMemcpyAsync(out, s.ptr(i_o), s.pieces[i_o].second, cudaMemcpyDeviceToHost, ctx->stream), "D2H out");
    GD_CUDA(cudaStreamSynchronize(ctx->stream), "select sync");
    return GD_OK;
}

int gd_frontier(gd_ctx* ctx, const double* energy, const double* time, int64_t n_apps, const int32_t* sm_clock,
                int32_t n_clocks, int32_t objective, double* t_sorted, int32_t* best, int32_t* first) {
    int rc = activate(ctx);
    if (rc) return rc;
    if (n_apps < 0 || n_clocks <= 0 || n_clocks > gd::kMaxClocks ||
        (objective != GD_OBJECTIVE_ENERGY && objective != GD_OBJECTIVE_POWER) ||
        (n_apps > 0 && (!energy || !time || !sm_clock || !t_sorted || !best || !first))) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "gd_frontier: bad arguments");
    }
    if (n_apps == 0) return GD_OK;
    const int64_t A = n_apps, C = n_clocks;
    Scratch s{ctx->stream};
    const size_t i_e = s.add(static_cast<size_t>(A) * C * sizeof(double));
    const size_t i_t = s.add(static_cast<size_t>(A) * C * sizeof(double));
    const size_t i_sm = s.add(static_cast<size_t>(C) * sizeof(int32_t));
    const size_t i_ts = s.add(static_cast<size_t>(A) * C * sizeof(double));
    const size_t i_b = s.add(static_cast<size_t>(A) * C * sizeof(int32_t));
    const size_t i_f = s.add(static_cast<size_t>(A) * sizeof(int32_t));
    GD_CUDA(s.alloc(), "cudaMallocAsync");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_e), energy, s.pieces[i_e].second, cudaMemcpyHostToDevice, ctx->stream), "H2D E");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_t), time, s.pieces[i_t].second, cudaMemcpyHostToDevice, ctx->stream), "H2D T");
    GD_CUDA(cudaMemcpyAsync(s.ptr(i_sm), sm_clock, s.pieces[i_sm].second, cudaMemcpyHostToDevice, ctx->stream),
            "H2D sm");
    int e = gd::launch_frontier(static_cast<double*>(s.ptr(i_e)), static_cast<double*>(s.ptr(i_t)),
                                static_cast<int32_t*>(s.ptr(i_sm)), A, n_clocks, objective,
                                static_cast<double*>(s.ptr(i_ts)), static_cast<int32_t*>(s.ptr(i_b)),
                                static_cast<int32_t*>(s.ptr(i_f)), ctx->sm_count, ctx->stream);
    ++ctx->launches;
    if (e != cudaSuccess) return cuda_error(static_cast<cudaError_t>(e), "frontier kernel launch");
    GD_CUDA(cudaMemcpyAsync(t_sorted, s.ptr(i_ts), s.pieces[i_ts].second, cudaMemcpyDeviceToHost, ctx->stream),
            "D2H t_sorted");
    GD_CUDA(cudaMemcpyAsync(best, s.ptr(i_b), s.pieces[i_b].second, cudaMemcpyDeviceToHost, ctx->stream), "D2H best");
    GD_CUDA(cudaMemcpyAsync(first, s.ptr(i_f), s.pieces[i_f].second, cudaMemcpyDeviceToHost, ctx->stream),
            "D2H first");
    GD_CUDA(cudaStreamSynchronize(ctx->stream), "frontier sync");
    return GD_OK;
}

int gd_microbench_dadd(gd_ctx* ctx, double* adds_per_second) {
    int rc = activate(ctx);
    if (rc) return rc;
    if (!adds_per_second) return set_error(GD_ERR_INVALID_ARGUMENT, "gd_microbench_dadd: null out");
    const int blocks = ctx->sm_count * 8, iters = 1 << 14;
    double* scratch = nullptr;
    GD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), blocks * sizeof(double), ctx->stream), "malloc");
    cudaEvent_t a, b;
    GD_CUDA(cudaEventCreate(&a), "event");
    GD_CUDA(cudaEventCreate(&b), "event");
    gd::launch_dadd_probe(scratch, blocks, iters, ctx->stream);  // warm-up
    GD_CUDA(cudaEventRecord(a, ctx->stream), "record");
    const int reps = 5;
    for (int r = 0; r < reps; ++r) gd::launch_dadd_probe(scratch, blocks, iters, ctx->stream);
    GD_CUDA(cudaEventRecord(b, ctx->stream), "record");
    ctx->launches += reps + 1;
    GD_CUDA(cudaEventSynchronize(b), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFreeAsync(scratch, ctx->stream);
    GD_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    const double adds = static_cast<double>(blocks) * 256.0 * 8.0 * iters * reps;
    *adds_per_second = adds / (ms * 1e-3);
    return GD_OK;
}

}  // extern "C"
