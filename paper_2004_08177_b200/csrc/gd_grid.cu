// gd_grid.cu -- K2+K3: the fused (app x clock) grid kernel.
//
// Replaces ModelPredictorState::build + 2x models::predict
// (scheduler.cpp:329-370) and decide()'s selection (scheduler.cpp:54-100,
// 187-234): candidate rows are never materialised, both ensembles are
// evaluated for every catalog clock of an app, and the deadline-masked
// selection runs in the same CTA.
//
// Work split.  A warp PAIR owns one app at a time: the even warp evaluates
// the energy ensemble, the odd warp the time ensemble, each lane owning the
// contiguous catalog clocks l*CPL .. l*CPL+CPL-1 (one in-order accumulator
// per clock).  The time warp hands its CPL times per lane to the energy warp
// through shared memory (two named barriers per app); the energy warp runs
// the selection epilogue.
//
// Partial evaluation.  For one app every candidate row is identical except
// the sm_clock / mem_clock columns, so every non-clock node test has the same
// outcome for all C clocks.  Per chunk of 32 trees a warp
//   phase 1 (lane per work item): walks each tree's row-only path from the
//     root; a path ending on a leaf is a constant for all C clocks.  A path
//     ending on a clock node becomes a residue node and queues its two
//     children, walked the same way in later rounds -- a warp-wide
//     breadth-first expansion with ballot-prefix allocation (no atomics, no
//     per-lane stacks);
//   phase 2 (lane per clock range): adds, in tree order, the constant or the
//     residue's leaf to each owned accumulator with __dadd_rn.  A residue
//     that is one test between two leaves (the common case) is evaluated
//     branch-free with one compare + select per clock.
// The leaf each candidate reaches is exactly predict_row's leaf
// (models.cpp:71-78), so the ordered sums are bit-identical.
//
// Clock packing.  Each owned clock is one register ck = sm << 16 | mem
// (1 <= sm, mem <= 65535, validated on the host).  A test `(double)sm <= thr`
// is `ck <= ((clamp(floor(thr), 0, 65535) << 16) | 0xffff)` (unsigned); a test
// `(double)mem <= thr` is `(ck & 0xffff) <= clamp(floor(thr), 0, 65535)`.
#include "gd_common.cuh"

namespace gd {
namespace {

using namespace dev;

// Resident CTAs per SM the partial kernel is compiled for (register cap
// 65536 / (128 * N)); 6 -> 80 registers, 24 warps per SM.
#ifndef GD_GRID_MIN_BLOCKS
#define GD_GRID_MIN_BLOCKS 6
#endif

constexpr int kWarps = 4;  // 2 warp pairs = 2 apps in flight per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kRnCap = 96;         // residue clock nodes per warp per chunk
constexpr int kRlCap = 192;        // residue leaves per warp per chunk
constexpr int kQCap = 2 * kRnCap;  // queued walks (two per residue node)

// Per warp: row[F] | cval[32] | root[32], first[32] | rn[kRnCap] | rl[kRlCap] | q[kQCap]
__host__ __device__ constexpr size_t smem_per_warp(int n_cols) {
    return static_cast<size_t>(n_cols) * 8 + 32 * 8 + 64 * 4 + kRnCap * 16 + kRlCap * 8 + kQCap * 8;
}
// Per pair: the time warp's T values, 32 lanes x CPL.
__host__ __device__ constexpr size_t smem_per_pair(int cpl) { return 32 * static_cast<size_t>(cpl) * 8; }

struct Scratch {
    double* row;
    double* cval;  // constant leaf per tree of the chunk
    int* root;     // residue root (rn index) per tree
    int* first;    // first clock node per tree (fallback start)
    int4* rn;      // {0 = sm | 1 = mem, packed key, lo code, hi code}; code < 0: ~leaf slot
    double* rl;    // residue leaves
    int2* q;       // {node, dest (rn*2 + side) | tree << 16}
};

struct ModelRef {
    const PNode* nodes;
    const int32_t* roots;
    int32_t n_trees;
};

__device__ __forceinline__ int clamp16(int t) { return min(max(t, 0), 65535); }

// Packed comparison key of a clock test (see the header comment).
__device__ __forceinline__ int clock_key(bool on_mem, double thr) {
    const int t = clamp16(thr_to_int(thr));
    return on_mem ? t : static_cast<int>((static_cast<unsigned>(t) << 16) | 0xffffu);
}

__device__ __forceinline__ bool goes_left(int kind, int key, unsigned ck) {
    return kind ? ((ck & 0xffffu) <= static_cast<unsigned>(key)) : (ck <= static_cast<unsigned>(key));
}

__device__ __forceinline__ void walk_row(const PNode* __restrict__ nodes, int32_t n, const double* row, int sm_col,
                                         int mem_col, double& v, int32_t& feat, int32_t& aux) {
    while (true) {
        load_node(nodes, n, v, feat, aux);
        if (feat < 0 || feat == sm_col || feat == mem_col) return;
        n = (row[feat] <= v) ? aux : aux + 1;
    }
}

// Phase 1 for the chunk [t0, t0 + nt): fills cval / root / first / rn / rl.
// Returns the masks of non-constant trees and of trees whose residue did not
// fit the pool (those fall back to per-clock traversal from `first`).
__device__ __forceinline__ void expand_chunk(const ModelRef& m, int32_t t0, int nt, const double* row, int sm_col,
                                             int mem_col, const Scratch& s, int lane, unsigned& nonconst,
                                             unsigned& fallback) {
    const unsigned lt = (1u << lane) - 1u;
    double v = 0.0;
    int32_t feat = -1, aux = 0, first = 0;
    bool clk = false;
    if (lane < nt) {
        first = __ldg(m.roots + t0 + lane);
        while (true) {
            load_node(m.nodes, first, v, feat, aux);
            if (feat < 0 || feat == sm_col || feat == mem_col) break;
            first = (row[feat] <= v) ? aux : aux + 1;
        }
        if (feat < 0) s.cval[lane] = v;
        clk = feat >= 0;
    }
    const unsigned mclk = __ballot_sync(kFull, clk);
    nonconst = mclk;
    fallback = 0u;
    if (mclk == 0u) return;
    unsigned fb = 0u;
    int n_rn = __popc(mclk);  // <= 32 <= kRnCap
    int tail = 2 * n_rn;      // <= 64 <= kQCap
    int n_rl = 0;
    if (clk) {
        const int idx = __popc(mclk & lt);
        const bool on_mem = feat == mem_col;
        s.rn[idx] = make_int4(on_mem ? 1 : 0, clock_key(on_mem, v), 0, 0);
        s.root[lane] = idx;
        s.first[lane] = first;
        s.q[2 * idx] = make_int2(aux, (idx * 2) | (lane << 16));
        s.q[2 * idx + 1] = make_int2(aux + 1, (idx * 2 + 1) | (lane << 16));
    }
    __syncwarp();
    int head = 0;
    while (head < tail) {
        const int qi = head + lane;
        const bool have = qi < tail;
        int2 item = make_int2(0, 0);
        bool leaf = false, node = false;
        if (have) {
            item = s.q[qi];
            walk_row(m.nodes, item.x, row, sm_col, mem_col, v, feat, aux);
            leaf = feat < 0;
            node = !leaf;
        }
        const unsigned mleaf = __ballot_sync(kFull, leaf);
        const unsigned mnode = __ballot_sync(kFull, node);
        const int tree = item.y >> 16, dest = item.y & 0xffff;
        const int node_room = min(kRnCap - n_rn, (kQCap - tail) / 2);  // tail, kQCap even
        bool over = false;
        int child = 0;
        if (leaf) {
            const int li = n_rl + __popc(mleaf & lt);
            if (li < kRlCap) {
                s.rl[li] = v;
                child = ~li;
            } else {
                over = true;
            }
        }
        if (node) {
            const int p = __popc(mnode & lt);
            const int ri = n_rn + p, q2 = tail + 2 * p;
            if (p < node_room) {
                const bool on_mem = feat == mem_col;
                s.rn[ri] = make_int4(on_mem ? 1 : 0, clock_key(on_mem, v), 0, 0);
                s.q[q2] = make_int2(aux, (ri * 2) | (tree << 16));
                s.q[q2 + 1] = make_int2(aux + 1, (ri * 2 + 1) | (tree << 16));
                child = ri;
            } else {
                over = true;
            }
        }
        if (have && !over) reinterpret_cast<int*>(s.rn)[(dest >> 1) * 4 + 2 + (dest & 1)] = child;
        fb |= __reduce_or_sync(kFull, over ? (1u << tree) : 0u);
        // Allocations that fitted are a prefix of each lane-ordered group.
        n_rl += max(0, min(__popc(mleaf), kRlCap - n_rl));
        const int nodes_fit = max(0, min(__popc(mnode), node_room));
        n_rn += nodes_fit;
        head = min(head + 32, tail);
        tail += 2 * nodes_fit;
        __syncwarp();
    }
    fallback = fb;
}

// Full per-candidate traversal from node n with a packed clock.
__device__ __forceinline__ double eval_full_packed(const PNode* __restrict__ nodes, int32_t n, const double* row,
                                                   int sm_col, int mem_col, unsigned ck) {
    return eval_full(nodes, n, row, sm_col, mem_col, static_cast<int>(ck >> 16), static_cast<int>(ck & 0xffffu));
}

template <int CPL>
__device__ __forceinline__ void accumulate_model(const ModelRef& m, const double* row, int sm_col, int mem_col,
                                                 const Scratch& s, const unsigned (&ck)[CPL], int lane,
                                                 double (&acc)[CPL]) {
    for (int32_t t0 = 0; t0 < m.n_trees; t0 += 32) {
        const int nt = min(32, m.n_trees - t0);
        unsigned nonconst, fallback;
        expand_chunk(m, t0, nt, row, sm_col, mem_col, s, lane, nonconst, fallback);
        __syncwarp();
        int j = 0;
        while (j < nt) {
            // Two constant trees at once (one LDS.128), in tree order.
            if (!(j & 1) && j + 1 < nt && !((nonconst >> j) & 3u)) {
                const double2 vv = *reinterpret_cast<const double2*>(s.cval + j);
#pragma unroll
                for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], vv.x);
#pragma unroll
                for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], vv.y);
                j += 2;
                continue;
            }
            const unsigned bit = 1u << j;
            if (!(nonconst & bit)) {
                const double vv = s.cval[j];
#pragma unroll
                for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], vv);
            } else if (fallback & bit) {
                const int32_t n = s.first[j];
#pragma unroll
                for (int i = 0; i < CPL; ++i)
                    acc[i] = __dadd_rn(acc[i], eval_full_packed(m.nodes, n, row, sm_col, mem_col, ck[i]));
            } else {
                const int4 r = s.rn[s.root[j]];
                if (r.z < 0 && r.w < 0) {
                    // One clock test between two leaves: compare + select.
                    const double lv = s.rl[~r.z], rv = s.rl[~r.w];
                    const unsigned key = static_cast<unsigned>(r.y);
                    if (r.x) {
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], (ck[i] & 0xffffu) <= key ? lv : rv);
                    } else {
#pragma unroll
                        for (int i = 0; i < CPL; ++i) acc[i] = __dadd_rn(acc[i], ck[i] <= key ? lv : rv);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < CPL; ++i) {
                        int code = goes_left(r.x, r.y, ck[i]) ? r.z : r.w;
                        while (code >= 0) {
                            const int4 q = s.rn[code];
                            code = goes_left(q.x, q.y, ck[i]) ? q.z : q.w;
                        }
                        acc[i] = __dadd_rn(acc[i], s.rl[~code]);
                    }
                }
            }
            ++j;
        }
        __syncwarp();
    }
}

// Named barrier for one warp pair.  The warp reconverges first (independent
// thread scheduling does not guarantee it after the data-dependent loops),
// and the non-.aligned form is used.
__device__ __forceinline__ void named_sync(int id, int threads) {
    __syncwarp();
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int CPL>
__global__ void __launch_bounds__(kThreads, GD_GRID_MIN_BLOCKS) grid_partial_kernel(const __grid_constant__ GridParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp >> 1;
    const bool is_time = warp & 1;
    const int F = p.n_cols;
    unsigned char* base = smem + smem_per_warp(F) * warp;
    Scratch s;
    s.row = reinterpret_cast<double*>(base);
    s.cval = s.row + F;
    s.root = reinterpret_cast<int*>(s.cval + 32);
    s.first = s.root + 32;
    s.rn = reinterpret_cast<int4*>(s.first + 32);
    s.rl = reinterpret_cast<double*>(s.rn + kRnCap);
    s.q = reinterpret_cast<int2*>(s.rl + kRlCap);
    double* tbuf = reinterpret_cast<double*>(smem + smem_per_warp(F) * kWarps + smem_per_pair(CPL) * pair);

    unsigned ck[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
        const int c = lane * CPL + i;  // lane l owns clocks l*CPL .. l*CPL+CPL-1
        ck[i] = c < p.n_clocks ? ((static_cast<unsigned>(__ldg(p.sm + c)) << 16) | static_cast<unsigned>(__ldg(p.mem + c)))
                               : 0u;
    }
    // Field-wise selects (a ternary over two ModelRef aggregates built from
    // __grid_constant__ fields picked the energy model for both roles).
    ModelRef m;
    m.nodes = is_time ? p.t_nodes : p.e_nodes;
    m.roots = is_time ? p.t_roots : p.e_roots;
    m.n_trees = is_time ? p.t_trees : p.e_trees;
    const int sm_col = p.sm_col, mem_col = p.mem_col;
    const int bar_a = 1 + 2 * pair, bar_b = 2 + 2 * pair;

    for (int64_t a = static_cast<int64_t>(blockIdx.x) * (kWarps / 2) + pair; a < p.n_apps;
         a += static_cast<int64_t>(gridDim.x) * (kWarps / 2)) {
        double acc[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) acc[i] = 0.0;
        __syncwarp();
        const double* src = p.rows + a * F;
        for (int j = lane; j < F; j += 32) s.row[j] = __ldg(src + j);
        __syncwarp();
        if (is_time) {
            // the time model sees the time-encoded categorical columns
            for (int k = lane; k < p.n_cat; k += 32) s.row[__ldg(p.cat_cols + k)] = __ldg(p.cat_t + a * p.n_cat + k);
            __syncwarp();
        }
        accumulate_model<CPL>(m, s.row, sm_col, mem_col, s, ck, lane, acc);
        if (is_time) {
            named_sync(bar_a, 64);  // the energy warp is done reading the previous app's times
#pragma unroll
            for (int i = 0; i < CPL; ++i) tbuf[lane * CPL + i] = finish(p.t_base, p.t_lr, acc[i]);
            named_sync(bar_b, 64);
        } else {
            double E[CPL], T[CPL];
            int smv[CPL];
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                E[i] = clamp_energy(finish(p.e_base, p.e_lr, acc[i]));
                smv[i] = static_cast<int>(ck[i] >> 16);
            }
            named_sync(bar_a, 64);
            named_sync(bar_b, 64);
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                T[i] = tbuf[lane * CPL + i];
                const int c = lane * CPL + i;
                if (c < p.n_clocks) {
                    if (p.e_out) p.e_out[a * p.n_clocks + c] = E[i];
                    if (p.t_out) p.t_out[a * p.n_clocks + c] = T[i];
                }
            }
            select_epilogue<CPL>(E, T, smv, lane, p.n_clocks, __ldg(p.budgets + a), p.mode, p.objective,
                                 p.best_effort, p.out + a);
        }
    }
}

// Rows genuinely differ per clock (nearest-record substitution from several
// profiled records, scheduler.cpp:341-359): full traversal per candidate.
template <int CPL>
__global__ void __launch_bounds__(256) grid_general_kernel(const __grid_constant__ GridParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    int smv[CPL], memv[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
        const int c = lane * CPL + i;
        smv[i] = c < p.n_clocks ? __ldg(p.sm + c) : 0;
        memv[i] = c < p.n_clocks ? __ldg(p.mem + c) : 0;
    }
    const int F = p.n_cols;
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * wpb + warp; a < p.n_apps;
         a += static_cast<int64_t>(gridDim.x) * wpb) {
        double accE[CPL], accT[CPL];
        const double* rE[CPL];
        const double* rT[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            accE[i] = accT[i] = 0.0;
            const int c = lane * CPL + i;
            const int64_t rec = c < p.n_clocks ? (p.rec_of_clock ? __ldg(p.rec_of_clock + a * p.n_clocks + c) : a) : 0;
            rE[i] = p.rows + rec * F;
            rT[i] = p.rows_t + rec * F;
        }
        for (int32_t t = 0; t < p.e_trees; ++t) {
            const int32_t root = __ldg(p.e_roots + t);
#pragma unroll
            for (int i = 0; i < CPL; ++i)
                accE[i] = __dadd_rn(accE[i], eval_full(p.e_nodes, root, rE[i], p.sm_col, p.mem_col, smv[i], memv[i]));
        }
        for (int32_t t = 0; t < p.t_trees; ++t) {
            const int32_t root = __ldg(p.t_roots + t);
#pragma unroll
            for (int i = 0; i < CPL; ++i)
                accT[i] = __dadd_rn(accT[i], eval_full(p.t_nodes, root, rT[i], p.sm_col, p.mem_col, smv[i], memv[i]));
        }
        double E[CPL], T[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            E[i] = clamp_energy(finish(p.e_base, p.e_lr, accE[i]));
            T[i] = finish(p.t_base, p.t_lr, accT[i]);
            const int c = lane * CPL + i;
            if (c < p.n_clocks) {
                if (p.e_out) p.e_out[a * p.n_clocks + c] = E[i];
                if (p.t_out) p.t_out[a * p.n_clocks + c] = T[i];
            }
        }
        select_epilogue<CPL>(E, T, smv, lane, p.n_clocks, __ldg(p.budgets + a), p.mode, p.objective,
                             p.best_effort, p.out + a);
    }
}

template <int CPL>
int launch_cpl(const GridParams& p, bool general, int sm_count, cudaStream_t stream) {
    if (general) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grid_general_kernel<CPL>, 256, 0);
        const int blocks = grid_blocks(8, p.n_apps, sm_count, per_sm);
        grid_general_kernel<CPL><<<blocks, 256, 0, stream>>>(p);
        return cudaGetLastError();
    }
    const size_t smem = smem_per_warp(p.n_cols) * kWarps + smem_per_pair(CPL) * (kWarps / 2);
    auto kern = grid_partial_kernel<CPL>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    const int blocks = grid_blocks(kWarps / 2, p.n_apps, sm_count, per_sm);
    kern<<<blocks, kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace

int launch_grid_select(const GridParams& p, bool general, int sm_count, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int cpl = (p.n_clocks + 31) / 32;
    if (cpl <= 1) return launch_cpl<1>(p, general, sm_count, s);
    if (cpl <= 2) return launch_cpl<2>(p, general, sm_count, s);
    if (cpl <= 4) return launch_cpl<4>(p, general, sm_count, s);
    if (cpl <= 7) return launch_cpl<7>(p, general, sm_count, s);
    if (cpl <= 9) return launch_cpl<9>(p, general, sm_count, s);
    if (cpl <= 12) return launch_cpl<12>(p, general, sm_count, s);
    return launch_cpl<16>(p, general, sm_count, s);
}

}  // namespace gd
