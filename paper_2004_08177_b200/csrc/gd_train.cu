// gd_train.cu -- fit_gbt on the GPU: the level-wise
// exact-greedy booster of models.cpp:161-393 (GbtCore), node for node.
//
// Bit-exactness pins the order of every floating-point reduction, so the
// parallelism is across (feature, frontier node) segments, never inside one:
//
//   scan     one thread per (feature, node): walks the feature's presorted
//            rows, keeps the node's rows, accumulates left_sum in that order
//            (models.cpp:263-283) and evaluates the gain
//            left + right - parent at every value change (strict >: the
//            first best position wins);
//   pick     one thread per node: the best feature in the tree's shuffled
//            feature order (strict >, models.cpp:249-252 outer loop), or a
//            leaf value sum / (count + l2) (models.cpp:306-307);
//   route    one thread per row: the row's child (col <= threshold goes
//            left) or its settled leaf value (models.cpp:310-320);
//   stats    one thread per child: sum / count / min / max of its rows'
//            residuals in row order (models.cpp:321-331);
//   update   one thread per row: predictions += lr * settled, residual =
//            target - base - prediction (models.cpp:343-347).
//
// The host keeps only the tree's node list (the order children are appended
// in, models.cpp:294-304) and the per-tree feature shuffle
// (SplitMix64(hash_mix(seed, t + 1)), rng.hpp), which are sequential by
// definition and tiny.  Doubles are combined with __dadd_rn / __dmul_rn /
// __ddiv_rn only (no FMA contraction, like the reference's Release build).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "gd_host.hpp"

namespace gd {
namespace {

constexpr double kMinSplitGain = 1e-12;  // models.cpp:21

struct Frontier {
    double sum, min_r, max_r;
    int32_t count;
    int32_t tree_node;
};

struct Best {
    double gain;
    double threshold;
    int32_t found;
    int32_t pad;
};

__device__ __forceinline__ double leaf_score(double sum, int32_t count, double l2) {
    return __ddiv_rn(__dmul_rn(sum, sum), __dadd_rn(static_cast<double>(count), l2));
}

__device__ __forceinline__ bool pure(const Frontier& f) { return __dadd_rn(f.max_r, -f.min_r) <= kMinSplitGain; }

// scan: thread (f, nd) over feature f's presorted rows (models.cpp:252-283).
__global__ void scan_kernel(const double* __restrict__ cols, const uint32_t* __restrict__ sorted,
                            const int32_t* __restrict__ node_of, const double* __restrict__ residual,
                            const Frontier* __restrict__ frontier, int32_t n_front, int64_t n, int32_t p, double l2,
                            Best* __restrict__ best) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= static_cast<int64_t>(p) * n_front) return;
    const int32_t f = static_cast<int32_t>(tid / n_front);
    const int32_t nd = static_cast<int32_t>(tid - static_cast<int64_t>(f) * n_front);
    Best b{-INFINITY, 0.0, 0, 0};
    const Frontier node = frontier[nd];
    if (!pure(node)) {
        const double parent = leaf_score(node.sum, node.count, l2);
        const double* col = cols + static_cast<int64_t>(f) * n;
        const uint32_t* ids = sorted + static_cast<int64_t>(f) * n;
        double left_sum = 0.0, last = 0.0;
        int32_t left_count = 0;
        bool has_last = false;
        for (int64_t k = 0; k < n; ++k) {
            const uint32_t idx = __ldg(ids + k);
            if (__ldg(node_of + idx) != nd) continue;
            const double value = __ldg(col + idx);
            if (has_last && value > last && left_count > 0) {
                const double right_sum = __dadd_rn(node.sum, -left_sum);
                const int32_t right_count = node.count - left_count;
                const double gain = __dadd_rn(__dadd_rn(leaf_score(left_sum, left_count, l2),
                                                        leaf_score(right_sum, right_count, l2)),
                                              -parent);
                if (gain > b.gain) {
                    b.gain = gain;
                    b.threshold = __dmul_rn(0.5, __dadd_rn(last, value));
                    b.found = 1;
                }
            }
            left_sum = __dadd_rn(left_sum, __ldg(residual + idx));
            ++left_count;
            last = value;
            has_last = true;
        }
    }
    best[tid] = b;
}

// pick: thread nd; features in the tree's shuffled order (models.cpp:249).
__global__ void pick_kernel(const Best* __restrict__ best, const int32_t* __restrict__ order, int32_t p,
                            const Frontier* __restrict__ frontier, int32_t n_front, double l2, int32_t* best_feature,
                            double* best_threshold, double* leaf_value) {
    const int32_t nd = blockIdx.x * blockDim.x + threadIdx.x;
    if (nd >= n_front) return;
    double g = -INFINITY, thr = 0.0;
    int32_t bf = -1;
    for (int32_t k = 0; k < p; ++k) {
        const int32_t f = __ldg(order + k);
        const Best b = best[static_cast<int64_t>(f) * n_front + nd];
        if (b.found && b.gain > g) {
            g = b.gain;
            bf = f;
            thr = b.threshold;
        }
    }
    best_feature[nd] = bf;
    best_threshold[nd] = thr;
    const Frontier node = frontier[nd];
    leaf_value[nd] = __ddiv_rn(node.sum, __dadd_rn(static_cast<double>(node.count), l2));
}

// route: thread i (models.cpp:310-320).  child_of[2 nd + side] = next frontier index.
__global__ void route_kernel(const double* __restrict__ cols, int64_t n, int32_t* node_of,
                             const int32_t* __restrict__ best_feature, const double* __restrict__ best_threshold,
                             const double* __restrict__ leaf_value, const int32_t* __restrict__ child_of,
                             double* settled) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t nd = node_of[i];
    if (nd < 0) return;
    const int32_t bf = __ldg(best_feature + nd);
    if (bf < 0) {
        settled[i] = __ldg(leaf_value + nd);
        node_of[i] = -1;
        return;
    }
    const bool left = __ldg(cols + static_cast<int64_t>(bf) * n + i) <= __ldg(best_threshold + nd);
    node_of[i] = __ldg(child_of + 2 * nd + (left ? 0 : 1));
}

// stats: thread c over rows in index order (models.cpp:321-331).
__global__ void stats_kernel(const int32_t* __restrict__ node_of, const double* __restrict__ residual, int64_t n,
                             Frontier* next, int32_t n_next) {
    const int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_next) return;
    double sum = 0.0, mn = 0.0, mx = 0.0;
    int32_t count = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (__ldg(node_of + i) != c) continue;
        const double r = __ldg(residual + i);
        if (count == 0) {
            mn = r;
            mx = r;
        } else {
            mn = r < mn ? r : mn;  // std::min(mn, r)
            mx = mx < r ? r : mx;  // std::max(mx, r)
        }
        sum = __dadd_rn(sum, r);
        ++count;
    }
    next[c].sum = sum;
    next[c].min_r = mn;
    next[c].max_r = mx;
    next[c].count = count;
}

// Root frontier: all rows, sums in row order (models.cpp:236-245).
__global__ void root_kernel(const double* __restrict__ residual, int64_t n, Frontier* f, int32_t* node_of) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double sum = 0.0, mn = residual[0], mx = residual[0];
        for (int64_t i = 0; i < n; ++i) {
            const double r = residual[i];
            sum = __dadd_rn(sum, r);
            mn = r < mn ? r : mn;  // std::min(a, b): b < a ? b : a
            mx = mx < r ? r : mx;  // std::max(a, b): a < b ? b : a
        }
        f[0].sum = sum;
        f[0].min_r = mn;
        f[0].max_r = mx;
        f[0].count = static_cast<int32_t>(n);
    }
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        node_of[i] = 0;
}

// update: thread i (models.cpp:336-347); final frontier leaves settle first.
__global__ void update_kernel(int64_t n, const int32_t* __restrict__ node_of, const double* __restrict__ leaf_value,
                              double* settled, double* predictions, double* residual, const double* __restrict__ targets,
                              double base, double lr) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t nd = node_of[i];
    const double s = nd >= 0 ? __ldg(leaf_value + nd) : settled[i];
    const double pr = __dadd_rn(predictions[i], __dmul_rn(lr, s));
    predictions[i] = pr;
    residual[i] = __dadd_rn(__dadd_rn(__ldg(targets + i), -base), -pr);
}

__global__ void init_residual_kernel(const double* __restrict__ targets, int64_t n, double base, double* residual,
                                     double* predictions) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    residual[i] = __dadd_rn(targets[i], -base);
    predictions[i] = 0.0;
}

// rng.hpp: SplitMix64, hash_mix, deterministic_shuffle (same constants).
struct SplitMix64 {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    size_t bounded(size_t n) { return n == 0 ? 0 : static_cast<size_t>(next() % n); }
};

uint64_t hash_mix(uint64_t a, uint64_t b) {
    SplitMix64 g{a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2))};
    return g.next();
}

}  // namespace
}  // namespace gd

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

#define TRY(call, where)                                             \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return gdh::cuda_error(_e, where);    \
    } while (0)

int grid_of(int64_t n, int threads) { return static_cast<int>((n + threads - 1) / threads); }

}  // namespace

namespace gdh {

// fit_gbt (models.cpp:381-393) through GbtCore (models.cpp:161-368).  The
// trees land in `out`'s host arrays in fit_gbt's node order.
int fit_gbt_device(gd_ctx* ctx, const double* rows, int64_t n, int32_t p, const double* targets,
                   const gd_gbt_config& cfg, std::vector<int64_t>& offsets, std::vector<int32_t>& feature,
                   std::vector<double>& threshold, std::vector<int32_t>& left, std::vector<int32_t>& right,
                   std::vector<double>& leaf, double& base) {
    using namespace gd;
    cudaStream_t st = ctx->stream;
    // Columns and presorted ids (models.cpp:167-181): value ascending, ties by row index.
    std::vector<double> cols(static_cast<size_t>(p) * n);
    std::vector<uint32_t> sorted(static_cast<size_t>(p) * n);
    for (int32_t j = 0; j < p; ++j) {
        double* c = cols.data() + static_cast<size_t>(j) * n;
        for (int64_t i = 0; i < n; ++i) c[i] = rows[i * p + j];
        uint32_t* ids = sorted.data() + static_cast<size_t>(j) * n;
        std::iota(ids, ids + n, 0u);
        std::sort(ids, ids + n, [&](uint32_t a, uint32_t b) {
            if (c[a] != c[b]) return c[a] < c[b];
            return a < b;
        });
    }
    double mean = 0.0;
    for (int64_t i = 0; i < n; ++i) mean += targets[i];
    mean /= static_cast<double>(n);
    base = mean;

    const int64_t cap = std::min<int64_t>(int64_t(1) << std::min(cfg.depth, 24), 2 * n + 2);
    const int32_t max_front = static_cast<int32_t>(cap);
    DevBuf d_cols, d_sorted, d_targets, d_res, d_pred, d_settled, d_node, d_front, d_next, d_best, d_order, d_bf,
        d_thr, d_leaf, d_child;
    TRY(cudaMalloc(&d_cols.p, cols.size() * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_sorted.p, sorted.size() * sizeof(uint32_t)), "cudaMalloc");
    TRY(cudaMalloc(&d_targets.p, n * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_res.p, n * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_pred.p, n * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_settled.p, n * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_node.p, n * sizeof(int32_t)), "cudaMalloc");
    TRY(cudaMalloc(&d_front.p, static_cast<size_t>(max_front) * sizeof(Frontier)), "cudaMalloc");
    TRY(cudaMalloc(&d_next.p, static_cast<size_t>(max_front) * sizeof(Frontier)), "cudaMalloc");
    TRY(cudaMalloc(&d_best.p, static_cast<size_t>(p) * (max_front / 2 + 1) * sizeof(Best)), "cudaMalloc");
    TRY(cudaMalloc(&d_order.p, std::max<size_t>(1, p) * sizeof(int32_t)), "cudaMalloc");
    TRY(cudaMalloc(&d_bf.p, static_cast<size_t>(max_front) * sizeof(int32_t)), "cudaMalloc");
    TRY(cudaMalloc(&d_thr.p, static_cast<size_t>(max_front) * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_leaf.p, static_cast<size_t>(max_front) * sizeof(double)), "cudaMalloc");
    TRY(cudaMalloc(&d_child.p, static_cast<size_t>(max_front) * 2 * sizeof(int32_t)), "cudaMalloc");
    TRY(cudaMemcpyAsync(d_cols.p, cols.data(), cols.size() * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    TRY(cudaMemcpyAsync(d_sorted.p, sorted.data(), sorted.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st), "H2D");
    TRY(cudaMemcpyAsync(d_targets.p, targets, n * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    init_residual_kernel<<<grid_of(n, 256), 256, 0, st>>>(d_targets.as<double>(), n, mean, d_res.as<double>(),
                                                          d_pred.as<double>());
    ctx->launches += 1;

    offsets.assign(1, 0);
    feature.clear();
    threshold.clear();
    left.clear();
    right.clear();
    leaf.clear();
    std::vector<int32_t> order(static_cast<size_t>(p)), h_bf, child_of;
    std::vector<double> h_thr, h_leaf;
    std::vector<int32_t> front_node;  // tree node of each frontier entry
    for (int t = 0; t < cfg.iterations; ++t) {
        // Node list of this tree (models.cpp:232-233, GbtNode defaults).
        std::vector<int32_t> tf(1, -1), tl(1, -1), tr(1, -1);
        std::vector<double> tt(1, 0.0), tv(1, 0.0);
        std::iota(order.begin(), order.end(), 0);
        SplitMix64 rng{hash_mix(cfg.seed, static_cast<uint64_t>(t) + 1)};  // trees_built() + 1
        for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[rng.bounded(i)]);
        TRY(cudaMemcpyAsync(d_order.p, order.data(), order.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
        root_kernel<<<std::max(1, std::min(grid_of(n, 256), 4 * ctx->sm_count)), 256, 0, st>>>(
            d_res.as<double>(), n, d_front.as<Frontier>(), d_node.as<int32_t>());
        ctx->launches += 1;
        front_node.assign(1, 0);
        int32_t n_front = 1;
        for (int depth = 0; depth < cfg.depth && n_front > 0; ++depth) {
            const int64_t segs = static_cast<int64_t>(p) * n_front;
            if (segs > 0) {
                scan_kernel<<<grid_of(segs, 128), 128, 0, st>>>(d_cols.as<double>(), d_sorted.as<uint32_t>(),
                                                                d_node.as<int32_t>(), d_res.as<double>(),
                                                                d_front.as<Frontier>(), n_front, n, p, cfg.l2_leaf_reg,
                                                                d_best.as<Best>());
                ctx->launches += 1;
            }
            pick_kernel<<<grid_of(n_front, 128), 128, 0, st>>>(d_best.as<Best>(), d_order.as<int32_t>(), p,
                                                              d_front.as<Frontier>(), n_front, cfg.l2_leaf_reg,
                                                              d_bf.as<int32_t>(), d_thr.as<double>(),
                                                              d_leaf.as<double>());
            ctx->launches += 1;
            h_bf.resize(static_cast<size_t>(n_front));
            h_thr.resize(static_cast<size_t>(n_front));
            h_leaf.resize(static_cast<size_t>(n_front));
            TRY(cudaMemcpyAsync(h_bf.data(), d_bf.p, n_front * sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
            TRY(cudaMemcpyAsync(h_thr.data(), d_thr.p, n_front * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
            TRY(cudaMemcpyAsync(h_leaf.data(), d_leaf.p, n_front * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
            TRY(cudaStreamSynchronize(st), "train sync");
            // Materialise splits (models.cpp:286-308).
            child_of.assign(static_cast<size_t>(n_front) * 2, -1);
            std::vector<int32_t> next_node;
            for (int32_t nd = 0; nd < n_front; ++nd) {
                const int32_t tn = front_node[static_cast<size_t>(nd)];
                if (h_bf[static_cast<size_t>(nd)] >= 0) {
                    tf[static_cast<size_t>(tn)] = h_bf[static_cast<size_t>(nd)];
                    tt[static_cast<size_t>(tn)] = h_thr[static_cast<size_t>(nd)];
                    const int32_t l = static_cast<int32_t>(tf.size());
                    tl[static_cast<size_t>(tn)] = l;
                    tr[static_cast<size_t>(tn)] = l + 1;
                    for (int k = 0; k < 2; ++k) {
                        tf.push_back(-1);
                        tl.push_back(-1);
                        tr.push_back(-1);
                        tt.push_back(0.0);
                        tv.push_back(0.0);
                    }
                    child_of[2 * static_cast<size_t>(nd)] = static_cast<int32_t>(next_node.size());
                    child_of[2 * static_cast<size_t>(nd) + 1] = static_cast<int32_t>(next_node.size() + 1);
                    next_node.push_back(l);
                    next_node.push_back(l + 1);
                } else {
                    tv[static_cast<size_t>(tn)] = h_leaf[static_cast<size_t>(nd)];
                }
            }
            TRY(cudaMemcpyAsync(d_child.p, child_of.data(), child_of.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st),
                "H2D");
            route_kernel<<<grid_of(n, 256), 256, 0, st>>>(d_cols.as<double>(), n, d_node.as<int32_t>(),
                                                         d_bf.as<int32_t>(), d_thr.as<double>(), d_leaf.as<double>(),
                                                         d_child.as<int32_t>(), d_settled.as<double>());
            const int32_t n_next = static_cast<int32_t>(next_node.size());
            if (n_next > 0) {
                stats_kernel<<<grid_of(n_next, 64), 64, 0, st>>>(d_node.as<int32_t>(), d_res.as<double>(), n,
                                                               d_next.as<Frontier>(), n_next);
                ctx->launches += 1;
            }
            ctx->launches += 1;
            std::swap(d_front.p, d_next.p);
            front_node = std::move(next_node);
            n_front = n_next;
        }
        // Depth limit: the remaining frontier leafs out (models.cpp:335-341).
        if (n_front > 0) {
            pick_kernel<<<grid_of(n_front, 128), 128, 0, st>>>(d_best.as<Best>(), d_order.as<int32_t>(), 0,
                                                              d_front.as<Frontier>(), n_front, cfg.l2_leaf_reg,
                                                              d_bf.as<int32_t>(), d_thr.as<double>(),
                                                              d_leaf.as<double>());
            ctx->launches += 1;
            h_leaf.resize(static_cast<size_t>(n_front));
            TRY(cudaMemcpyAsync(h_leaf.data(), d_leaf.p, n_front * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        }
        update_kernel<<<grid_of(n, 256), 256, 0, st>>>(n, d_node.as<int32_t>(), d_leaf.as<double>(),
                                                       d_settled.as<double>(), d_pred.as<double>(), d_res.as<double>(),
                                                       d_targets.as<double>(), mean, cfg.learning_rate);
        ctx->launches += 1;
        TRY(cudaStreamSynchronize(st), "train sync");
        for (int32_t nd = 0; nd < n_front; ++nd) tv[static_cast<size_t>(front_node[static_cast<size_t>(nd)])] = h_leaf[static_cast<size_t>(nd)];
        feature.insert(feature.end(), tf.begin(), tf.end());
        threshold.insert(threshold.end(), tt.begin(), tt.end());
        left.insert(left.end(), tl.begin(), tl.end());
        right.insert(right.end(), tr.begin(), tr.end());
        leaf.insert(leaf.end(), tv.begin(), tv.end());
        offsets.push_back(static_cast<int64_t>(feature.size()));
    }
    TRY(cudaGetLastError(), "train kernels");
    return GD_OK;
}

}  // namespace gdh
