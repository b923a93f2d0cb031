// gd_edf.cpp -- the sequential half of schedule_d_dvfs: the EDF event loop.
//
// run_edf_loop (scheduler.cpp:105-147) is inherently sequential under the
// default remaining_time budget: a job's budget is arrival + deadline - now
// and `now` advances by the execution time of every scheduled job.  The GPU
// computes every job's per-clock E/T (gd_grid_select); this loop walks the
// jobs in EDF order and answers each job at its budget.
//
// Same order as the reference, in O(n log n) instead of the reference's
// O(n^2) std::min_element scan: arrivals sorted by (arrival, app_id), the
// available set a binary heap on (arrival + deadline, arrival, app_id,
// insertion order) -- the last key reproduces min_element's
// first-in-vector tie rule.
#include <algorithm>
#include <cfloat>
#include <cstring>
#include <queue>
#include <vector>

#include "gd_host.hpp"

namespace gdh {
namespace {

// scheduler.cpp:54-57
inline double objective_value(double e, double t, int32_t objective) {
    if (objective == GD_OBJECTIVE_POWER) return e / ((t < 1e-12) ? 1e-12 : t);
    return e;
}

}  // namespace

// scheduler.cpp:62-100 (select_text / select_literal) + :212-223 (best effort).
void select_one(const double* E, const double* T, const int32_t* sm, int32_t n, double budget,
                const gd_select_opts& o, gd_decision& out) {
    std::memset(&out, 0, sizeof(out));
    int32_t chosen = -1;
    if (o.mode == GD_MODE_TEXT) {
        for (int32_t c = 0; c < n; ++c) {
            if (T[c] > budget) continue;
            if (chosen < 0) {
                chosen = c;
                continue;
            }
            const double cv = objective_value(E[c], T[c], o.objective);
            const double bv = objective_value(E[chosen], T[chosen], o.objective);
            if (cv < bv || (cv == bv && (T[c] < T[chosen] || (T[c] == T[chosen] && sm[c] < sm[chosen])))) chosen = c;
        }
    } else {
        double min_objective = DBL_MAX, max_time = budget;
        for (int32_t c = 0; c < n; ++c) {
            const double v = objective_value(E[c], T[c], o.objective);
            if (v < min_objective && T[c] <= max_time) {
                min_objective = v;
                max_time = T[c];
                chosen = c;
            }
        }
    }
    if (chosen < 0 && o.best_effort && n > 0) {
        chosen = 0;
        for (int32_t c = 1; c < n; ++c) {
            if (T[c] < T[chosen] || (T[c] == T[chosen] && E[c] < E[chosen])) chosen = c;
        }
        out.note = GD_NOTE_BEST_EFFORT;
    }
    if (chosen >= 0) {
        out.status = GD_SCHEDULED;
        out.clock_index = chosen;
        out.energy_ws = E[chosen];
        out.time_s = T[chosen];
    } else {
        out.status = GD_REJECTED;
        out.clock_index = -1;
    }
}

}  // namespace gdh

namespace {

// Text-mode selection answered from a frontier (gd_frontier): k = #{T <= b}
// by binary search over the app's sorted times; the prefix argmin at k-1 is
// select_text's choice, first[] the best-effort one.
void select_frontier(const double* E, const double* T, const double* ts, const int32_t* best, int32_t first,
                     const int32_t* sm, int32_t n, double budget, const gd_select_opts& o, gd_decision& out) {
    if (o.mode != GD_MODE_TEXT || first < 0) {
        gdh::select_one(E, T, sm, n, budget, o, out);
        return;
    }
    std::memset(&out, 0, sizeof(out));
    const int32_t k = static_cast<int32_t>(std::upper_bound(ts, ts + n, budget) - ts);
    int32_t chosen = k > 0 ? best[k - 1] : -1;
    if (chosen < 0 && o.best_effort) {
        chosen = first;
        out.note = GD_NOTE_BEST_EFFORT;
    }
    if (chosen >= 0) {
        out.status = GD_SCHEDULED;
        out.clock_index = chosen;
        out.energy_ws = E[chosen];
        out.time_s = T[chosen];
    } else {
        out.status = GD_REJECTED;
        out.clock_index = -1;
    }
}

}  // namespace

extern "C" int gd_schedule_edf(const gd_job* jobs, int64_t n_jobs, const double* energy, const double* time,
                               const int32_t* sm_clock, int32_t n_clocks, int32_t budget_kind,
                               const gd_select_opts* opts, const double* exec_time, gd_exec_fn exec_fn,
                               void* exec_user, gd_decision* out, int64_t* order) {
    return gd_schedule_edf_frontier(jobs, n_jobs, energy, time, nullptr, nullptr, nullptr, sm_clock, n_clocks,
                                    budget_kind, opts, exec_time, exec_fn, exec_user, out, order);
}

extern "C" int gd_schedule_edf_frontier(const gd_job* jobs, int64_t n_jobs, const double* energy, const double* time,
                                        const double* t_sorted, const int32_t* best, const int32_t* first,
                                        const int32_t* sm_clock, int32_t n_clocks, int32_t budget_kind,
                                        const gd_select_opts* opts, const double* exec_time, gd_exec_fn exec_fn,
                                        void* exec_user, gd_decision* out, int64_t* order) {
    const bool frontier = t_sorted && best && first;
    if (n_jobs < 0 || n_clocks <= 0 || !opts || !out || !order || (n_jobs > 0 && !jobs)) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_schedule_edf: invalid arguments");
    }
    if (!exec_time && !exec_fn) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_schedule_edf: no execution-time source");
    }
    if (n_jobs > 0 && (!energy || !time || !sm_clock)) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_schedule_edf: null prediction tables");
    }
    std::vector<int64_t> pending(static_cast<size_t>(n_jobs));
    for (int64_t i = 0; i < n_jobs; ++i) pending[i] = i;
    // scheduler.cpp:109-112
    std::stable_sort(pending.begin(), pending.end(), [&](int64_t a, int64_t b) {
        if (jobs[a].arrival_s != jobs[b].arrival_s) return jobs[a].arrival_s < jobs[b].arrival_s;
        return jobs[a].app_rank < jobs[b].app_rank;
    });
    struct Entry {
        double abs_deadline, arrival;
        int64_t rank, seq, job;
    };
    // scheduler.cpp:130-136 comparator, plus insertion order for exact ties.
    auto later = [](const Entry& a, const Entry& b) {
        if (a.abs_deadline != b.abs_deadline) return a.abs_deadline > b.abs_deadline;
        if (a.arrival != b.arrival) return a.arrival > b.arrival;
        if (a.rank != b.rank) return a.rank > b.rank;
        return a.seq > b.seq;
    };
    std::priority_queue<Entry, std::vector<Entry>, decltype(later)> available(later);
    int64_t next_pending = 0, n_out = 0;
    double now = 0.0;
    while (next_pending < n_jobs || !available.empty()) {
        while (next_pending < n_jobs && jobs[pending[next_pending]].arrival_s <= now) {
            const gd_job& j = jobs[pending[next_pending]];
            available.push(Entry{j.arrival_s + j.deadline_s, j.arrival_s, j.app_rank, next_pending,
                                 pending[next_pending]});
            ++next_pending;
        }
        if (available.empty()) {
            now = jobs[pending[next_pending]].arrival_s;
            continue;
        }
        const Entry e = available.top();
        available.pop();
        const gd_job& job = jobs[e.job];
        gd_decision d;
        std::memset(&d, 0, sizeof(d));
        if (job.app_index < 0) {
            // scheduler.cpp:194-198: predictor returned nullopt
            d.clock_index = -1;
            d.status = GD_REJECTED;
            d.note = GD_NOTE_MISSING_DATA;
        } else {
            // scheduler.cpp:203-205
            const double budget =
                budget_kind == GD_BUDGET_FULL ? job.deadline_s : (job.arrival_s + job.deadline_s) - now;
            const int64_t off = static_cast<int64_t>(job.app_index) * n_clocks;
            if (frontier) {
                select_frontier(energy + off, time + off, t_sorted + off, best + off, first[job.app_index], sm_clock,
                                n_clocks, budget, *opts, d);
            } else {
                gdh::select_one(energy + off, time + off, sm_clock, n_clocks, budget, *opts, d);
            }
            if (d.status == GD_SCHEDULED) {
                now += exec_time ? exec_time[off + d.clock_index] : exec_fn(exec_user, e.job, d.clock_index);
            }
        }
        out[n_out] = d;
        order[n_out] = e.job;
        ++n_out;
    }
    return GD_OK;
}
