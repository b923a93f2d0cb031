// gd_common.cuh -- device helpers shared by the sm_100a kernels.
//
// Bit-exactness rules: node test `x <= thr` in IEEE
// double; leaves summed in tree order into a double accumulator with
// __dadd_rn; `base + lr*acc` as __dmul_rn then __dadd_rn (never an FMA);
// energy clamp `(0.0 < v) ? v : 0.0`; power objective `E / max(T, 1e-12)`
// with __ddiv_rn.
#pragma once

#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>

#include "gd_device.cuh"

namespace gd {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void load_node(const PNode* __restrict__ nodes, int32_t n, double& v, int32_t& feat,
                                          int32_t& aux) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(nodes) + n);
    v = __hiloint2double(q.y, q.x);
    feat = q.z;
    aux = q.w;
}

// models.cpp:424  std::max(0.0, v)
__device__ __forceinline__ double clamp_energy(double v) { return (0.0 < v) ? v : 0.0; }

// models.cpp:419 + 376: base + (lr * acc), two roundings, no contraction.
__device__ __forceinline__ double finish(double base, double lr, double acc) {
    return __dadd_rn(base, __dmul_rn(lr, acc));
}

// scheduler.cpp:54-57
__device__ __forceinline__ double objective_value(double e, double t, int objective) {
    if (objective == GD_OBJECTIVE_POWER) return __ddiv_rn(e, (t < 1e-12) ? 1e-12 : t);
    return e;
}

// (double)clk <= thr  <=>  clk <= thr_to_int(thr)  for integer clk > INT_MIN.
__device__ __forceinline__ int thr_to_int(double thr) {
    if (!(thr >= -2147483648.0)) return INT_MIN;  // NaN or below int range: never <=
    if (thr >= 2147483647.0) return INT_MAX;
    return static_cast<int>(floor(thr));
}

__device__ __forceinline__ int clamp16(int t) { return min(max(t, 0), 65535); }

// Key of a clock test: (double)clk <= thr  <=>  clk <= t16  for 1 <= clk <= 65535.
__device__ __forceinline__ uint32_t t16_of(double thr) { return static_cast<uint32_t>(clamp16(thr_to_int(thr))); }

// Number of sorted thresholds t[0..n) with t < x (NaN x: n).
__device__ __forceinline__ int rank_of(const double* __restrict__ t, int n, double x) {
    if (x != x) return n;
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(t + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// Selection epilogue (K3).  Lane l owns the contiguous catalog clocks
// l*CPL .. l*CPL+CPL-1, so lane-major order is catalog order.
// ---------------------------------------------------------------------------
struct Cand {
    double obj, t, e;
    int sm, idx;  // idx < 0: none
};

// select_text's replacement rule (scheduler.cpp:73-75) closed over catalog
// order: for finite values the scan returns the argmin of (obj, T, sm, idx).
__device__ __forceinline__ bool text_less(const Cand& a, const Cand& b) {
    if (a.idx < 0) return false;
    if (b.idx < 0) return true;
    if (a.obj < b.obj) return true;
    if (a.obj != b.obj) return false;
    if (a.t < b.t) return true;
    if (a.t != b.t) return false;
    if (a.sm < b.sm) return true;
    if (a.sm != b.sm) return false;
    return a.idx < b.idx;
}

// best-effort fastest clock (scheduler.cpp:215-220): argmin (T, E, idx).
__device__ __forceinline__ bool fast_less(const Cand& a, const Cand& b) {
    if (a.idx < 0) return false;
    if (b.idx < 0) return true;
    if (a.t < b.t) return true;
    if (a.t != b.t) return false;
    if (a.e < b.e) return true;
    if (a.e != b.e) return false;
    return a.idx < b.idx;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int mask) {
    Cand o;
    o.obj = __shfl_xor_sync(kFull, c.obj, mask);
    o.t = __shfl_xor_sync(kFull, c.t, mask);
    o.e = __shfl_xor_sync(kFull, c.e, mask);
    o.sm = __shfl_xor_sync(kFull, c.sm, mask);
    o.idx = __shfl_xor_sync(kFull, c.idx, mask);
    return o;
}

// cidx[i] = catalog index of this lane's slot i (-1 = empty).  Lane-major
// slot order must be catalog order (literal mode scans it).
template <int CPL>
__device__ __forceinline__ void select_epilogue(const double (&E)[CPL], const double (&T)[CPL], const int (&smv)[CPL],
                                                const int (&cidx)[CPL], int lane, double budget, int mode,
                                                int objective, int best_effort, gd_decision* out) {
    Cand best;
    best.idx = -1;
    best.obj = best.t = best.e = 0.0;
    best.sm = 0;
    if (mode == GD_MODE_TEXT) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int c = cidx[i];
            if (c >= 0 && !(T[i] > budget)) {
                Cand k{objective_value(E[i], T[i], objective), T[i], E[i], smv[i], c};
                if (text_less(k, best)) best = k;
            }
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            Cand o = shfl_cand(best, m);
            if (text_less(o, best)) best = o;
        }
    } else {
        // scheduler.cpp:86-100: sequential scan in catalog order, DBL_MAX
        // init, bound tightened to each accepted candidate's time.  Every lane
        // runs the same scan on broadcast values.
        double min_objective = DBL_MAX, max_time = budget;
        for (int l = 0; l < 32; ++l) {
#pragma unroll
            for (int i = 0; i < CPL; ++i) {
                const int c = __shfl_sync(kFull, cidx[i], l);
                const double e = __shfl_sync(kFull, E[i], l);
                const double t = __shfl_sync(kFull, T[i], l);
                if (c < 0) continue;
                const double value = objective_value(e, t, objective);
                if (value < min_objective && t <= max_time) {
                    min_objective = value;
                    max_time = t;
                    best.idx = c;
                    best.e = e;
                    best.t = t;
                }
            }
        }
    }
    int note = GD_NOTE_NONE;
    if (best.idx < 0 && best_effort) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int c = cidx[i];
            if (c >= 0) {
                Cand k{0.0, T[i], E[i], smv[i], c};
                if (fast_less(k, best)) best = k;
            }
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
        *out = d;
    }
}

// Contiguous slot map: lane l owns catalog clocks l*CPL .. l*CPL+CPL-1.
template <int CPL>
__device__ __forceinline__ void contiguous_cidx(int lane, int n_clocks, int (&cidx)[CPL]) {
#pragma unroll
    for (int i = 0; i < CPL; ++i) cidx[i] = lane * CPL + i < n_clocks ? lane * CPL + i : -1;
}

// Full per-candidate traversal from node n (row + clock override): the
// reference's predict_row on the substituted row (models.cpp:71-78,
// scheduler.cpp:352-357).
__device__ __forceinline__ double eval_full(const PNode* __restrict__ nodes, int32_t n, const double* row,
                                            int sm_col, int mem_col, int sm, int mem) {
    double v;
    int32_t feat, aux;
    while (true) {
        load_node(nodes, n, v, feat, aux);
        if (feat < 0) return v;
        const double x = (feat == sm_col) ? static_cast<double>(sm)
                                          : (feat == mem_col) ? static_cast<double>(mem) : row[feat];
        n = (x <= v) ? aux : aux + 1;
    }
}

inline int grid_blocks(int64_t units_per_block, int64_t n, int sm_count, int blocks_per_sm) {
    int64_t want = (n + units_per_block - 1) / units_per_block;
    int64_t cap = static_cast<int64_t>(sm_count) * (blocks_per_sm > 0 ? blocks_per_sm : 1);
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return static_cast<int>(want);
}

}  // namespace dev
}  // namespace gd
