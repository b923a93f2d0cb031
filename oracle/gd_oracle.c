/*
 * oracle/gd_oracle.c -- TEST INFRASTRUCTURE ONLY (see gd_oracle.h).
 *
 * Scalar CPU restatement of the reference hot path.  Built with
 * -O2 -ffp-contract=off so that `base + lr*acc` and the linear dot product
 * are separate IEEE multiply/add steps, as in the reference's Release build
 * (-O3 -DNDEBUG, no -march: x86-64 baseline has no FMA).
 */
#include "gd_oracle.h"

#include <float.h>
#include <stdlib.h>
#include <string.h>

/* models.cpp:71-78  GbtTree::predict_row, returning the leaf's node index
 * instead of its value (the reference only exposes the value). */
int32_t gdo_leaf_index(const gdo_forest* f, int32_t tree, const double* row) {
    const int64_t base = f->tree_offsets[tree];
    int32_t idx = 0;
    while (f->feature[base + idx] >= 0) {
        const int64_t n = base + idx;
        idx = (row[f->feature[n]] <= f->threshold[n]) ? f->left[n] : f->right[n];
    }
    return idx;
}

/* models.cpp:370-377  gbt_raw_prediction: ordered double sum, then * lr. */
static double gbt_raw_prediction(const gdo_forest* f, double learning_rate, const double* row,
                                 int32_t* leaf_ids) {
    double acc = 0.0;
    for (int32_t t = 0; t < f->n_trees; ++t) {
        const int32_t idx = gdo_leaf_index(f, t, row);
        if (leaf_ids) leaf_ids[t] = idx;
        acc += f->leaf_value[f->tree_offsets[t] + idx];
    }
    return learning_rate * acc;
}

/* models.cpp:424  std::max(0.0, v) == (0.0 < v) ? v : 0.0 */
static double clamp_energy(double v) { return (0.0 < v) ? v : 0.0; }

/* models.cpp:395-428, gbt branch (:418-419) and energy clamp (:424). */
void gdo_predict_gbt(const gdo_forest* f, double base, double learning_rate, int32_t clamp_nonneg,
                     const double* rows, int64_t n_rows, int32_t n_cols, double* out,
                     int32_t* leaf_ids) {
    for (int64_t r = 0; r < n_rows; ++r) {
        const double* row = rows + r * (int64_t)n_cols;
        double v = base + gbt_raw_prediction(f, learning_rate, row,
                                             leaf_ids ? leaf_ids + r * (int64_t)f->n_trees : NULL);
        if (clamp_nonneg) v = clamp_energy(v);
        out[r] = v;
    }
}

/* models.cpp:421-422 linear branch (ols / lasso), then the clamp. */
void gdo_predict_linear(const double* coef, double intercept, int32_t clamp_nonneg, const double* rows,
                        int64_t n_rows, int32_t n_cols, double* out) {
    for (int64_t r = 0; r < n_rows; ++r) {
        const double* row = rows + r * (int64_t)n_cols;
        double v = intercept;
        for (int32_t j = 0; j < n_cols; ++j) v += coef[j] * row[j];
        if (clamp_nonneg) v = clamp_energy(v);
        out[r] = v;
    }
}

/* scheduler.cpp:54-57  objective_value; std::max(t, 1e-12) == (t < 1e-12) ? 1e-12 : t */
static double objective_value(double e, double t, int32_t objective) {
    if (objective == 1) return e / ((t < 1e-12) ? 1e-12 : t);
    return e;
}

/* scheduler.cpp:62-81  select_text */
static int32_t select_text(const double* E, const double* T, const int32_t* sm, int32_t n, double budget,
                           int32_t objective) {
    int32_t best = -1;
    for (int32_t c = 0; c < n; ++c) {
        if (T[c] > budget) continue;
        if (best < 0) {
            best = c;
            continue;
        }
        const double cv = objective_value(E[c], T[c], objective);
        const double bv = objective_value(E[best], T[best], objective);
        if (cv < bv || (cv == bv && (T[c] < T[best] || (T[c] == T[best] && sm[c] < sm[best])))) best = c;
    }
    return best;
}

/* scheduler.cpp:86-100  select_literal */
static int32_t select_literal(const double* E, const double* T, int32_t n, double budget, int32_t objective) {
    double min_objective = DBL_MAX;
    double max_time = budget;
    int32_t chosen = -1;
    for (int32_t c = 0; c < n; ++c) {
        const double value = objective_value(E[c], T[c], objective);
        if (value < min_objective && T[c] <= max_time) {
            min_objective = value;
            max_time = T[c];
            chosen = c;
        }
    }
    return chosen;
}

/* scheduler.cpp:203-234  budget already applied; selection + best-effort. */
void gdo_select(const double* E, const double* T, const int32_t* sm, int32_t n, double budget, int32_t mode,
                int32_t objective, int32_t best_effort, gdo_decision* out) {
    memset(out, 0, sizeof(*out));
    int32_t chosen = (mode == 0) ? select_text(E, T, sm, n, budget, objective)
                                 : select_literal(E, T, n, budget, objective);
    if (chosen < 0 && best_effort && n > 0) {
        /* scheduler.cpp:215-222 fastest predicted clock, ties by energy */
        int32_t fastest = -1;
        for (int32_t c = 0; c < n; ++c) {
            if (fastest < 0 || T[c] < T[fastest] || (T[c] == T[fastest] && E[c] < E[fastest])) fastest = c;
        }
        chosen = fastest;
        out->note = 1;
    }
    if (chosen >= 0) {
        out->status = 0;
        out->clock_index = chosen;
        out->energy_ws = E[chosen];
        out->time_s = T[chosen];
    } else {
        out->status = 1;
        out->clock_index = -1;
    }
}

/* scheduler.cpp:329-370 (ModelPredictorState::build, the row copy + clock
 * override of :341-359 and the two apply_encoding/predict calls of :361-364)
 * and scheduler.cpp:187-234 (decide) for every app of the batch. */
void gdo_grid_select(const gdo_forest* fe, double base_e, double lr_e, const gdo_forest* ft, double base_t,
                     double lr_t, const double* rows, int64_t n_records, int32_t n_cols,
                     const double* cat_t, const int32_t* cat_cols, int32_t n_cat,
                     const int32_t* rec_of_clock, int64_t n_apps, const int32_t* sm_clock,
                     const int32_t* mem_clock, int32_t n_clocks, int32_t sm_col, int32_t mem_col,
                     const double* budgets, int32_t mode, int32_t objective, int32_t best_effort,
                     gdo_decision* out, double* e_out, double* t_out) {
    (void)n_records;
    double* row_e = (double*)malloc(sizeof(double) * (size_t)n_cols);
    double* row_t = (double*)malloc(sizeof(double) * (size_t)n_cols);
    double* E = (double*)malloc(sizeof(double) * (size_t)n_clocks);
    double* T = (double*)malloc(sizeof(double) * (size_t)n_clocks);
    for (int64_t a = 0; a < n_apps; ++a) {
        for (int32_t c = 0; c < n_clocks; ++c) {
            const int64_t rec = rec_of_clock ? (int64_t)rec_of_clock[a * n_clocks + c] : a;
            memcpy(row_e, rows + rec * n_cols, sizeof(double) * (size_t)n_cols);
            if (sm_col >= 0) row_e[sm_col] = (double)sm_clock[c];
            if (mem_col >= 0) row_e[mem_col] = (double)mem_clock[c];
            memcpy(row_t, row_e, sizeof(double) * (size_t)n_cols);
            for (int32_t k = 0; k < n_cat; ++k) row_t[cat_cols[k]] = cat_t[rec * n_cat + k];
            gdo_predict_gbt(fe, base_e, lr_e, 1, row_e, 1, n_cols, &E[c], NULL);
            gdo_predict_gbt(ft, base_t, lr_t, 0, row_t, 1, n_cols, &T[c], NULL);
        }
        gdo_select(E, T, sm_clock, n_clocks, budgets[a], mode, objective, best_effort, &out[a]);
        if (e_out) memcpy(e_out + a * n_clocks, E, sizeof(double) * (size_t)n_clocks);
        if (t_out) memcpy(t_out + a * n_clocks, T, sizeof(double) * (size_t)n_clocks);
    }
    free(row_e);
    free(row_t);
    free(E);
    free(T);
}

/* scheduler.cpp:109-112  pending order: (arrival, app_id) */
static const gdo_job* g_jobs;
static int cmp_pending(const void* pa, const void* pb) {
    const gdo_job* a = &g_jobs[*(const int64_t*)pa];
    const gdo_job* b = &g_jobs[*(const int64_t*)pb];
    if (a->arrival_s != b->arrival_s) return a->arrival_s < b->arrival_s ? -1 : 1;
    if (a->app_rank != b->app_rank) return a->app_rank < b->app_rank ? -1 : 1;
    /* std::sort leaves equal keys unordered; fall back to input order */
    return *(const int64_t*)pa < *(const int64_t*)pb ? -1 : (*(const int64_t*)pa > *(const int64_t*)pb);
}

/* core.hpp:95  Job::absolute_deadline_s */
static double abs_deadline(const gdo_job* j) { return j->arrival_s + j->deadline_s; }

/* scheduler.cpp:105-147 run_edf_loop (O(n^2) min_element kept verbatim) with
 * scheduler.cpp:187-234 decide. */
void gdo_schedule_edf(const gdo_job* jobs, int64_t n_jobs, const double* energy, const double* time,
                      const double* exec_time, const int32_t* sm_clock, int32_t n_clocks, int32_t mode,
                      int32_t budget_kind, int32_t objective, int32_t best_effort, gdo_decision* out,
                      int64_t* order) {
    int64_t* pending = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_jobs + 1));
    int64_t* available = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_jobs + 1));
    for (int64_t i = 0; i < n_jobs; ++i) pending[i] = i;
    g_jobs = jobs;
    qsort(pending, (size_t)n_jobs, sizeof(int64_t), cmp_pending);
    int64_t n_avail = 0, next_pending = 0, n_out = 0;
    double now = 0.0;
    while (next_pending < n_jobs || n_avail > 0) {
        while (next_pending < n_jobs && jobs[pending[next_pending]].arrival_s <= now) {
            available[n_avail++] = pending[next_pending++];
        }
        if (n_avail == 0) {
            now = jobs[pending[next_pending]].arrival_s;
            continue;
        }
        int64_t best = 0;
        for (int64_t k = 1; k < n_avail; ++k) {
            const gdo_job* a = &jobs[available[k]];
            const gdo_job* b = &jobs[available[best]];
            int less;
            if (abs_deadline(a) != abs_deadline(b)) less = abs_deadline(a) < abs_deadline(b);
            else if (a->arrival_s != b->arrival_s) less = a->arrival_s < b->arrival_s;
            else less = a->app_rank < b->app_rank;
            if (less) best = k;
        }
        const int64_t j = available[best];
        memmove(available + best, available + best + 1, sizeof(int64_t) * (size_t)(n_avail - best - 1));
        --n_avail;

        gdo_decision d;
        memset(&d, 0, sizeof(d));
        const gdo_job* job = &jobs[j];
        if (job->app_index < 0) {
            /* scheduler.cpp:194-198 predictor returned nullopt */
            d.status = 1;
            d.clock_index = -1;
            d.note = 2;
        } else {
            const double budget = budget_kind == 1 ? job->deadline_s : abs_deadline(job) - now;
            const int64_t off = (int64_t)job->app_index * n_clocks;
            gdo_select(energy + off, time + off, sm_clock, n_clocks, budget, mode, objective, best_effort, &d);
            if (d.status == 0) now += exec_time[off + d.clock_index];
        }
        out[n_out] = d;
        order[n_out] = j;
        ++n_out;
    }
    free(pending);
    free(available);
}
