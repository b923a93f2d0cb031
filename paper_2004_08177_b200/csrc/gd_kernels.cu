// gd_kernels.cu -- sm_100a kernels other than the fused grid (gd_grid.cu).
//
//   K1  predict_gbt / predict_linear   models::predict over materialised rows
//                                      (models.cpp:395-428, :370-377, :71-78)
//   K3  select                         selection over given E/T tables
//                                      (scheduler.cpp:54-100, 212-223)
//   build_rows_t                       time-encoded rows for the general grid
//   dadd_probe                         FP64 add-pipe peak for the roofline
//
// No tensor cores: tree traversal is not a contraction.
#include <cstdlib>
#include <math_constants.h>

#include "gd_common.cuh"

namespace gd {
namespace {

using namespace dev;

// ---------------------------------------------------------------------------
// K1: warp per row, lane per tree (32 trees in flight), then the 32 leaf
// values are folded into the row's accumulator in tree order by shuffles.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) predict_gbt_kernel(const PNode* __restrict__ nodes,
                                                          const int32_t* __restrict__ roots, int32_t n_trees,
                                                          double base, double lr, int clamp,
                                                          const double* __restrict__ rows, int64_t n_rows,
                                                          int32_t n_cols, double* __restrict__ out,
                                                          int32_t* __restrict__ leaf_ids) {
    extern __shared__ double smem_rows[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    double* row = smem_rows + static_cast<int64_t>(warp) * n_cols;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * wpb + warp; r < n_rows;
         r += static_cast<int64_t>(gridDim.x) * wpb) {
        __syncwarp();
        for (int j = lane; j < n_cols; j += 32) row[j] = __ldg(rows + r * n_cols + j);
        __syncwarp();
        double acc = 0.0;
        for (int32_t t0 = 0; t0 < n_trees; t0 += 32) {
            const int32_t t = t0 + lane;
            double v = 0.0;
            int32_t leaf = 0;
            if (t < n_trees) {
                int32_t n = __ldg(roots + t);
                int32_t feat, aux;
                while (true) {
                    load_node(nodes, n, v, feat, aux);
                    if (feat < 0) break;
                    n = (row[feat] <= v) ? aux : aux + 1;
                }
                leaf = aux;
                if (leaf_ids) leaf_ids[r * n_trees + t] = leaf;
            }
            const int nt = min(32, n_trees - t0);
            for (int j = 0; j < nt; ++j) acc = __dadd_rn(acc, __shfl_sync(kFull, v, j));
        }
        if (lane == 0) {
            double y = finish(base, lr, acc);
            out[r] = clamp ? clamp_energy(y) : y;
        }
    }
}

// K1, rows on lanes: a warp takes 32 rows and every lane walks the SAME tree
// for its own row, trees in model order (the in-order sum stays per lane).
// Top levels are one broadcast load for the whole warp and only the deep
// levels diverge, so each tree costs ~1/2 the L1 wavefronts of the
// lanes-on-trees form above; rows sit transposed in shared memory
// ([feature][lane]: conflict-free whatever feature each lane tests).  Two
// trees per lane advance in lockstep for ILP.
constexpr int kK1Warps = 4;
#ifndef GD_K1_WALKS
#define GD_K1_WALKS 2
#endif
constexpr int kK1Walks = GD_K1_WALKS;  // trees per lane in lockstep
__global__ void __launch_bounds__(kK1Warps * 32) predict_gbt_rows_kernel(
    const PNode* __restrict__ nodes, const int32_t* __restrict__ roots, int32_t n_trees, double base, double lr,
    int clamp, const double* __restrict__ rows, int64_t n_rows, int32_t n_cols, double* __restrict__ out,
    int32_t* __restrict__ leaf_ids) {
    extern __shared__ double smem_rows[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* rt = smem_rows + static_cast<int64_t>(warp) * n_cols * 32;  // [feature][lane]
    const int64_t n_blocks = (n_rows + 31) / 32;
    for (int64_t rb = static_cast<int64_t>(blockIdx.x) * kK1Warps + warp; rb < n_blocks;
         rb += static_cast<int64_t>(gridDim.x) * kK1Warps) {
        const int64_t r0 = rb * 32;
        const int nr = static_cast<int>(min(static_cast<int64_t>(32), n_rows - r0));
        __syncwarp();
        for (int i = lane; i < nr * n_cols; i += 32) {  // coalesced global, transposed shared
            const int r = i / n_cols, f = i - r * n_cols;
            rt[f * 32 + r] = __ldg(rows + r0 * n_cols + i);
        }
        __syncwarp();
        const bool valid = lane < nr;
        const double* myrow = rt + lane;  // feature f at myrow[32 f]
        double acc = 0.0;
        int32_t t = 0;
        for (; t + kK1Walks <= n_trees; t += kK1Walks) {
            int32_t n[kK1Walks], f[kK1Walks], aux[kK1Walks];
            double v[kK1Walks];
#pragma unroll
            for (int h = 0; h < kK1Walks; ++h) {
                n[h] = __ldg(roots + t + h);
                load_node(nodes, n[h], v[h], f[h], aux[h]);
            }
            bool any = true;
            while (any) {
                any = false;
#pragma unroll
                for (int h = 0; h < kK1Walks; ++h) {
                    if (f[h] >= 0) {
                        n[h] = (myrow[32 * f[h]] <= v[h]) ? aux[h] : aux[h] + 1;
                        load_node(nodes, n[h], v[h], f[h], aux[h]);
                        any = true;
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < kK1Walks; ++h) {
                acc = __dadd_rn(acc, v[h]);
                if (leaf_ids && valid) leaf_ids[(r0 + lane) * n_trees + t + h] = aux[h];
            }
        }
        for (; t < n_trees; ++t) {
            int32_t n = __ldg(roots + t);
            double v;
            int32_t f, aux;
            load_node(nodes, n, v, f, aux);
            while (f >= 0) {
                n = (myrow[32 * f] <= v) ? aux : aux + 1;
                load_node(nodes, n, v, f, aux);
            }
            acc = __dadd_rn(acc, v);
            if (leaf_ids && valid) leaf_ids[(r0 + lane) * n_trees + t] = aux;
        }
        if (valid) {
            const double y = finish(base, lr, acc);
            out[r0 + lane] = clamp ? clamp_energy(y) : y;
        }
    }
}

// models.cpp:421-422: v = intercept; v += coef_j * row_j (no FMA).
__global__ void __launch_bounds__(256) predict_linear_kernel(const double* __restrict__ coef, double intercept,
                                                             int clamp, const double* __restrict__ rows,
                                                             int64_t n_rows, int32_t n_cols,
                                                             double* __restrict__ out) {
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = intercept;
        for (int j = 0; j < n_cols; ++j) v = __dadd_rn(v, __dmul_rn(__ldg(coef + j), __ldg(rows + r * n_cols + j)));
        out[r] = clamp ? clamp_energy(v) : v;
    }
}

__global__ void build_rows_t_kernel(const double* __restrict__ rows, const double* __restrict__ cat_t,
                                    const int32_t* __restrict__ cat_cols, int32_t n_cat, int64_t n_records,
                                    int32_t n_cols, double* __restrict__ rows_t) {
    const int64_t total = n_records * n_cols;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / n_cols;
        const int32_t c = static_cast<int32_t>(i - r * n_cols);
        double v = rows[i];
        for (int k = 0; k < n_cat; ++k) {
            if (cat_cols[k] == c) v = cat_t[r * n_cat + k];
        }
        rows_t[i] = v;
    }
}

// K3 alone: warp per app over given candidate tables.
template <int CPL>
__global__ void __launch_bounds__(256) select_kernel(const __grid_constant__ SelectParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    int smv[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
        const int c = lane * CPL + i;
        smv[i] = c < p.n_clocks ? __ldg(p.sm + c) : 0;
    }
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * wpb + warp; a < p.n_apps;
         a += static_cast<int64_t>(gridDim.x) * wpb) {
        double E[CPL], T[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int c = lane * CPL + i;
            E[i] = c < p.n_clocks ? __ldg(p.energy + a * p.n_clocks + c) : 0.0;
            T[i] = c < p.n_clocks ? __ldg(p.time + a * p.n_clocks + c) : 0.0;
        }
        int cidx[CPL];
        contiguous_cidx<CPL>(lane, p.n_clocks, cidx);
        select_epilogue<CPL>(E, T, smv, cidx, lane, __ldg(p.budgets + a), p.mode, p.objective, p.best_effort,
                             p.out + a);
    }
}

// K3 for catalogs wider than a warp's CPL <= 16 register layout (> 512
// clocks): a warp per app, lane l takes clocks l, l + 32, ...  Text mode and
// the best-effort fallback are argmins of a total key (same rules as
// select_epilogue); literal mode is select_literal's order-dependent scan,
// run by lane 0 over the whole row.
__global__ void __launch_bounds__(256) select_wide_kernel(const __grid_constant__ SelectParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int64_t C = p.n_clocks;
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * wpb + warp; a < p.n_apps;
         a += static_cast<int64_t>(gridDim.x) * wpb) {
        const double* E = p.energy + a * C;
        const double* T = p.time + a * C;
        const double budget = __ldg(p.budgets + a);
        Cand best;
        best.idx = -1;
        best.obj = best.t = best.e = 0.0;
        best.sm = 0;
        if (p.mode == GD_MODE_TEXT) {
            for (int64_t c = lane; c < C; c += 32) {
                const double t = __ldg(T + c), e = __ldg(E + c);
                if (t > budget) continue;
                Cand k{objective_value(e, t, p.objective), t, e, __ldg(p.sm + c), static_cast<int>(c)};
                if (text_less(k, best)) best = k;
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) {
                Cand o = shfl_cand(best, m);
                if (text_less(o, best)) best = o;
            }
        } else {
            if (lane == 0) {  // scheduler.cpp:86-100
                double min_objective = DBL_MAX, max_time = budget;
                for (int64_t c = 0; c < C; ++c) {
                    const double e = __ldg(E + c), t = __ldg(T + c);
                    const double value = objective_value(e, t, p.objective);
                    if (value < min_objective && t <= max_time) {
                        min_objective = value;
                        max_time = t;
                        best.idx = static_cast<int>(c);
                        best.e = e;
                        best.t = t;
                    }
                }
            }
            best.idx = __shfl_sync(kFull, best.idx, 0);
            best.e = __shfl_sync(kFull, best.e, 0);
            best.t = __shfl_sync(kFull, best.t, 0);
        }
        int note = GD_NOTE_NONE;
        if (best.idx < 0 && p.best_effort) {
            for (int64_t c = lane; c < C; c += 32) {
                Cand k{0.0, __ldg(T + c), __ldg(E + c), __ldg(p.sm + c), static_cast<int>(c)};
                if (fast_less(k, best)) best = k;
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) {
                Cand o = shfl_cand(best, m);
                if (fast_less(o, best)) best = o;
            }
            note = GD_NOTE_BEST_EFFORT;
        }
        if (lane == 0) {
            gd_decision d;
            d.clock_index = best.idx;
            d.status = best.idx >= 0 ? GD_SCHEDULED : GD_REJECTED;
            d.note = best.idx >= 0 ? note : GD_NOTE_NONE;
            d.energy_ws = best.idx >= 0 ? best.e : 0.0;
            d.time_s = best.idx >= 0 ? best.t : 0.0;
            p.out[a] = d;
        }
    }
}

// ---------------------------------------------------------------------------
// Selection frontier (the remaining_time EDF loop's per-job query, SURVEY
// §8f #2): per app, the candidates sorted by (T, E, catalog index) and the
// prefix argmin of select_text's key (objective, T, sm, index).  For a budget
// b the feasible set {T <= b} is a prefix of that order, so the text-mode
// choice is best[k-1] with k = #{T <= b} (one binary search), and the
// best-effort choice (argmin (T, E, index), scheduler.cpp:215-220) is the
// first element.  Apps with a non-finite E or T (outside the contract, where
// the sequential scan is not a total order) get first = -2: the host scans
// them instead.  One CTA of kFrontThreads per app, bitonic sort in shared
// memory, Hillis-Steele scan for the prefix argmin.
// ---------------------------------------------------------------------------
constexpr int kFrontThreads = 256;

__device__ __forceinline__ bool sort_less(double ta, double ea, int ia, double tb, double eb, int ib) {
    if (ta != tb) return ta < tb;
    if (ea != eb) return ea < eb;
    return ia < ib;
}

__global__ void __launch_bounds__(kFrontThreads) frontier_kernel(const double* __restrict__ E,
                                                                 const double* __restrict__ T,
                                                                 const int32_t* __restrict__ sm, int64_t n_apps,
                                                                 int32_t C, int32_t objective, double* t_sorted,
                                                                 int32_t* best, int32_t* first) {
    __shared__ double st[kMaxClocks], se[kMaxClocks];
    __shared__ int si[kMaxClocks], sb[kMaxClocks];
    __shared__ int bad;
    int P = 1;
    while (P < C) P <<= 1;
    for (int64_t a = blockIdx.x; a < n_apps; a += gridDim.x) {
        if (threadIdx.x == 0) bad = 0;
        __syncthreads();
        for (int k = threadIdx.x; k < P; k += blockDim.x) {
            if (k < C) {
                st[k] = __ldg(T + a * C + k);
                se[k] = __ldg(E + a * C + k);
                si[k] = k;
                if (!isfinite(st[k]) || !isfinite(se[k])) bad = 1;
            } else {
                st[k] = CUDART_INF;
                se[k] = CUDART_INF;
                si[k] = INT_MAX;
            }
        }
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int k = threadIdx.x; k < P; k += blockDim.x) {
                    const int l = k ^ stride;
                    if (l > k) {
                        const bool up = (k & size) == 0;
                        const bool lt = sort_less(st[l], se[l], si[l], st[k], se[k], si[k]);
                        if (lt == up) {
                            const double t = st[k], e = se[k];
                            const int i = si[k];
                            st[k] = st[l];
                            se[k] = se[l];
                            si[k] = si[l];
                            st[l] = t;
                            se[l] = e;
                            si[l] = i;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // Prefix argmin of (objective, T, sm, index) over the sorted order.
        for (int k = threadIdx.x; k < C; k += blockDim.x) sb[k] = k;
        __syncthreads();
        for (int d = 1; d < C; d <<= 1) {
            int nb[2] = {0, 0};
            int m = 0;
            for (int k = threadIdx.x; k < C; k += blockDim.x, ++m) {
                int cur = sb[k];
                if (k >= d) {
                    const int o = sb[k - d];
                    Cand x{objective_value(se[o], st[o], objective), st[o], se[o], __ldg(sm + si[o]), si[o]};
                    Cand y{objective_value(se[cur], st[cur], objective), st[cur], se[cur], __ldg(sm + si[cur]), si[cur]};
                    if (text_less(x, y)) cur = o;
                }
                if (m < 2) nb[m] = cur;
            }
            __syncthreads();
            m = 0;
            for (int k = threadIdx.x; k < C; k += blockDim.x, ++m)
                if (m < 2) sb[k] = nb[m];
            __syncthreads();
        }
        for (int k = threadIdx.x; k < C; k += blockDim.x) {
            t_sorted[a * C + k] = st[k];
            best[a * C + k] = si[sb[k]];
        }
        if (threadIdx.x == 0) first[a] = bad ? -2 : si[0];
        __syncthreads();
    }
}

// FP64 add-pipe throughput probe: 8 independent __dadd_rn chains per thread,
// enough warps to saturate every SM.  Used to measure the binding roofline's
// peak (in-order FP64 adds) on the box the bench runs on.
__global__ void __launch_bounds__(256) dadd_probe_kernel(double* out, int iters, double step) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
        a0 = __dadd_rn(a0, step);
        a1 = __dadd_rn(a1, step);
        a2 = __dadd_rn(a2, step);
        a3 = __dadd_rn(a3, step);
        a4 = __dadd_rn(a4, step);
        a5 = __dadd_rn(a5, step);
        a6 = __dadd_rn(a6, step);
        a7 = __dadd_rn(a7, step);
    }
    const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 1.2345) out[blockIdx.x] = r;  // keep the chains live
}

__global__ void recode_clock_nodes_kernel(const PNode* __restrict__ src, PNode* __restrict__ dst, int64_t n,
                                          int32_t sm_col, int32_t mem_col) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        PNode x = src[i];
        if (x.feat >= 0) {
            if (x.feat == sm_col) x.feat = kFeatSm;
            else if (x.feat == mem_col) x.feat = kFeatMem;
        }
        dst[i] = x;
    }
}

// Walk nodes (gd_device.cuh WNode) from grid nodes: tree t's grid nodes
// [roots[t], roots[t+1]) map to walk nodes [wroots[t], ...) in the same order.
// Which clock columns are one value across the catalog (fold[0] = sm value
// or 0, fold[1] = mem value or 0) and whether that differs from the state the
// models' walk nodes were last built for (fold[2]); one block.
__global__ void fold_check_kernel(const int32_t* __restrict__ sm, const int32_t* __restrict__ mem, int32_t C,
                                  int32_t enable, int32_t* fold_a, int32_t* fold_b) {
    __shared__ int ok_sm, ok_mem;
    if (threadIdx.x == 0) {
        ok_sm = 1;
        ok_mem = 1;
    }
    __syncthreads();
    const int32_t s0 = sm[0], m0 = mem[0];
    for (int32_t c = threadIdx.x; c < C; c += blockDim.x) {
        if (sm[c] != s0) ok_sm = 0;
        if (mem[c] != m0) ok_mem = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int32_t smf = enable && ok_sm ? s0 : 0, memf = enable && ok_mem ? m0 : 0;
        int32_t* folds[2] = {fold_a, fold_b};
        for (int32_t* f : folds) {
            if (!f) continue;
            f[2] = f[0] != smf || f[1] != memf;
            f[0] = smf;
            f[1] = memf;
        }
    }
}

// fold (device, nullable): take sm_fix / mem_fix from fold[0..1] and build
// only if fold[2] says the state changed (the device-buffer call path, which
// never reads the catalog back to the host).
__global__ void build_walk_nodes_kernel(const PNode* __restrict__ grid, int64_t n, const int32_t* __restrict__ roots,
                                        int32_t n_trees, const int32_t* __restrict__ wroots,
                                        const double* __restrict__ thr, const int32_t* __restrict__ thr_off,
                                        int32_t sm_fix, int32_t mem_fix, const int32_t* __restrict__ fold,
                                        WNode* __restrict__ dst) {
    if (fold) {
        if (!fold[2]) return;
        sm_fix = fold[0];
        mem_fix = fold[1];
    }
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int32_t lo = 0, hi = n_trees - 1;  // last tree with roots[t] <= i
        while (lo < hi) {
            const int32_t mid = (lo + hi + 1) >> 1;
            if (__ldg(roots + mid) <= i) lo = mid;
            else hi = mid - 1;
        }
        const int32_t root = __ldg(roots + lo);
        const PNode x = grid[i];
        WNode w;
        if (x.feat == kFeatLeaf) {
            w.key = static_cast<int32_t>(i);
            w.fc = static_cast<int32_t>(0xfff80000u);  // feat = kFeatLeaf
        } else {
            const int32_t child = x.aux - root;
            int32_t feat = x.feat;
            const int32_t fix = x.feat == kFeatSm ? sm_fix : (x.feat == kFeatMem ? mem_fix : 0);
            if (fix > 0) {
                // A clock column every candidate of the call shares: the test
                // (double)fix <= thr has one outcome, so the node becomes an
                // unconditional row node (feature 0; rank <= INT_MAX always
                // goes left, rank <= -1 never) and no residue carries it.
                feat = 0;
                w.key = static_cast<double>(fix) <= x.v ? 0x7fffffff : -1;
            } else if (x.feat < 0) {
                w.key = static_cast<int32_t>(t16_of(x.v));
            } else {
                const int32_t o = __ldg(thr_off + x.feat), c = __ldg(thr_off + x.feat + 1) - o;
                const int32_t r = rank_of(thr + o, c, x.v);
                w.key = (x.v == x.v && r < c) ? r : -1;  // exact match; NaN thresholds never pass
            }
            // Leaf flags in the free low bits of the child offset: bit 0 the
            // left child is a leaf, bit 1 the right one -- a walk stops at
            // the parent and never loads a leaf node.
            const uint32_t lf = (grid[x.aux].feat == kFeatLeaf ? 1u : 0u) | (grid[x.aux + 1].feat == kFeatLeaf ? 2u : 0u);
            w.fc = static_cast<int32_t>((static_cast<uint32_t>(feat) << 19) | (static_cast<uint32_t>(child) * 8u) | lf);
        }
        dst[__ldg(wroots + lo) + (i - root)] = w;
    }
}

template <int CPL>
int launch_select_cpl(const SelectParams& p, int sm_count, cudaStream_t stream) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<CPL>, 256, 0);
    const int blocks = grid_blocks(8, p.n_apps, sm_count, per_sm);
    select_kernel<CPL><<<blocks, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace

int launch_predict_gbt(const PNode* nodes, const int32_t* roots, int32_t n_trees, double base, double lr, int clamp,
                       const double* rows, int64_t n_rows, int32_t n_cols, double* out, int32_t* leaf_ids,
                       int sm_count, void* stream) {
    const char* env = std::getenv("GDVFS_K1_TREES_ON_LANES");
    const size_t rows_smem = static_cast<size_t>(kK1Warps) * n_cols * 32 * sizeof(double);
    // The lanes-on-trees form: for comparison, and for very wide rows whose
    // 32-row transposed tile would not fit shared memory.
    const bool few_rows = (n_rows + 31) / 32 < 4LL * sm_count * kK1Warps;  // too few 32-row tiles to fill the GPU
    if ((env && env[0] == '1') || rows_smem > 200 * 1024 || (few_rows && !(env && env[0] == '0'))) {
        const int threads = 256;
        const size_t smem = static_cast<size_t>(threads / 32) * n_cols * sizeof(double);
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(predict_gbt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_gbt_kernel, threads, smem);
        const int blocks = grid_blocks(threads / 32, n_rows, sm_count, per_sm);
        predict_gbt_kernel<<<blocks, threads, smem, static_cast<cudaStream_t>(stream)>>>(
            nodes, roots, n_trees, base, lr, clamp, rows, n_rows, n_cols, out, leaf_ids);
        return cudaGetLastError();
    }
    const size_t smem = rows_smem;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(predict_gbt_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, predict_gbt_rows_kernel, kK1Warps * 32, smem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t n_blocks = (n_rows + 31) / 32;
    const int blocks = grid_blocks(kK1Warps, n_blocks, sm_count, per_sm);
    predict_gbt_rows_kernel<<<blocks, kK1Warps * 32, smem, static_cast<cudaStream_t>(stream)>>>(
        nodes, roots, n_trees, base, lr, clamp, rows, n_rows, n_cols, out, leaf_ids);
    return cudaGetLastError();
}

int launch_predict_linear(const double* coef, double intercept, int clamp, const double* rows, int64_t n_rows,
                          int32_t n_cols, double* out, int sm_count, void* stream) {
    const int threads = 256;
    const int blocks = grid_blocks(threads, n_rows, sm_count, 8);
    predict_linear_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(coef, intercept, clamp, rows,
                                                                                     n_rows, n_cols, out);
    return cudaGetLastError();
}

int launch_build_rows_t(const double* rows, const double* cat_t, const int32_t* cat_cols, int32_t n_cat,
                        int64_t n_records, int32_t n_cols, double* rows_t, void* stream) {
    const int64_t total = n_records * n_cols;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    build_rows_t_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, cat_t, cat_cols, n_cat,
                                                                              n_records, n_cols, rows_t);
    return cudaGetLastError();
}

int launch_recode_clock_nodes(const PNode* src, PNode* dst, int64_t n, int32_t sm_col, int32_t mem_col, void* stream) {
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 8192) blocks = 8192;
    if (blocks < 1) blocks = 1;
    recode_clock_nodes_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n, sm_col, mem_col);
    return cudaGetLastError();
}

int launch_fold_check(const int32_t* sm, const int32_t* mem, int32_t C, int32_t enable, int32_t* fold_a,
                      int32_t* fold_b, void* stream) {
    fold_check_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(sm, mem, C, enable, fold_a, fold_b);
    return cudaGetLastError();
}

int launch_build_walk_nodes(const PNode* grid, int64_t n, const int32_t* roots, int32_t n_trees,
                            const int32_t* wroots, const double* thr, const int32_t* thr_off, int32_t sm_fix,
                            int32_t mem_fix, const int32_t* fold, WNode* dst, void* stream) {
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 8192) blocks = 8192;
    if (blocks < 1) blocks = 1;
    build_walk_nodes_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(grid, n, roots, n_trees, wroots,
                                                                                  thr, thr_off, sm_fix, mem_fix, fold,
                                                                                  dst);
    return cudaGetLastError();
}

int launch_frontier(const double* E, const double* T, const int32_t* sm, int64_t n_apps, int32_t n_clocks,
                    int32_t objective, double* t_sorted, int32_t* best, int32_t* first, int sm_count, void* stream) {
    if (n_clocks > 2 * kFrontThreads) return cudaErrorInvalidValue;  // two slots per thread in the scan
    const int64_t blocks = n_apps < 8LL * sm_count ? n_apps : 8LL * sm_count;
    frontier_kernel<<<static_cast<int>(blocks > 0 ? blocks : 1), kFrontThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        E, T, sm, n_apps, n_clocks, objective, t_sorted, best, first);
    return cudaGetLastError();
}

int launch_dadd_probe(double* scratch, int blocks, int iters, void* stream) {
    dadd_probe_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(scratch, iters, 1.0e-9);
    return cudaGetLastError();
}

int launch_select_wide(const SelectParams& p, int sm_count, void* stream) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_wide_kernel, 256, 0);
    const int blocks = grid_blocks(8, p.n_apps, sm_count, per_sm);
    select_wide_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
    return cudaGetLastError();
}

int launch_select(const SelectParams& p, int sm_count, void* stream) {
    if (p.n_clocks > kMaxClocks) return launch_select_wide(p, sm_count, stream);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int cpl = (p.n_clocks + 31) / 32;
    if (cpl <= 1) return launch_select_cpl<1>(p, sm_count, s);
    if (cpl <= 2) return launch_select_cpl<2>(p, sm_count, s);
    if (cpl <= 4) return launch_select_cpl<4>(p, sm_count, s);
    if (cpl <= 7) return launch_select_cpl<7>(p, sm_count, s);
    if (cpl <= 9) return launch_select_cpl<9>(p, sm_count, s);
    if (cpl <= 12) return launch_select_cpl<12>(p, sm_count, s);
    return launch_select_cpl<16>(p, sm_count, s);
}

}  // namespace gd
