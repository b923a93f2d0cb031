/*
 * oracle/gd_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C restatement of the reference's hot path (batched GBT evaluation of
 * the energy and time ensembles over every (app x clock) candidate, then the
 * deadline-aware selection and the EDF loop that calls it).  Every function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.  The product path (paper_2004_08177_b200/) never links
 * or calls anything under oracle/.
 *
 * Parity pinning: this restatement is checked against (a) golden vectors
 * produced by the reference itself (tests/golden/, generated through
 * oracle/_ref, the reference's own sources compiled by oracle/Makefile) and
 * (b) live calls into oracle/_ref where that library has been built.
 */
#ifndef GD_ORACLE_H
#define GD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One tree ensemble as flat SoA arrays over all trees; node fields mirror
 * models::GbtNode (include/gpudvfs/models.hpp:35-43).  left/right are
 * tree-local node indices, feature < 0 marks a leaf. */
typedef struct gdo_forest {
    int32_t n_trees;
    const int64_t* tree_offsets; /* n_trees + 1 */
    const int32_t* feature;
    const double* threshold;
    const int32_t* left;
    const int32_t* right;
    const double* leaf_value;
} gdo_forest;

typedef struct gdo_decision {
    int32_t clock_index; /* catalog index, -1 when rejected */
    int16_t status;      /* 0 scheduled, 1 rejected_infeasible */
    int16_t note;        /* 0 none, 1 "best_effort", 2 "missing correlated data" */
    double energy_ws;
    double time_s;
} gdo_decision;

typedef struct gdo_job {
    double arrival_s;
    double deadline_s;
    int64_t app_rank;  /* rank of the job's app_id under std::string '<' */
    int32_t app_index; /* row of the per-app E/T/exec tables; -1 = missing data */
    int32_t pad;
} gdo_job;

/* mode: 0 text_semantics, 1 literal_pseudocode; objective: 0 energy, 1 power;
 * budget: 0 remaining_time, 1 full_deadline. */

int32_t gdo_leaf_index(const gdo_forest* f, int32_t tree, const double* row);

void gdo_predict_gbt(const gdo_forest* f, double base, double learning_rate, int32_t clamp_nonneg,
                     const double* rows, int64_t n_rows, int32_t n_cols, double* out,
                     int32_t* leaf_ids /* nullable, n_rows x n_trees */);

void gdo_predict_linear(const double* coef, double intercept, int32_t clamp_nonneg, const double* rows,
                        int64_t n_rows, int32_t n_cols, double* out);

void gdo_select(const double* energy, const double* time, const int32_t* sm_clock, int32_t n_clocks,
                double budget, int32_t mode, int32_t objective, int32_t best_effort, gdo_decision* out);

/* The (app x clock) grid: rows are materialised exactly as
 * ModelPredictorState::build does (nearest-record copy + clock override +
 * per-target categorical values), both ensembles evaluated, then selected. */
void gdo_grid_select(const gdo_forest* fe, double base_e, double lr_e, const gdo_forest* ft, double base_t,
                     double lr_t, const double* rows, int64_t n_records, int32_t n_cols,
                     const double* cat_t, const int32_t* cat_cols, int32_t n_cat,
                     const int32_t* rec_of_clock, int64_t n_apps, const int32_t* sm_clock,
                     const int32_t* mem_clock, int32_t n_clocks, int32_t sm_col, int32_t mem_col,
                     const double* budgets, int32_t mode, int32_t objective, int32_t best_effort,
                     gdo_decision* out, double* e_out, double* t_out);

/* run_edf_loop + schedule_d_dvfs::decide over precomputed per-app E/T. */
void gdo_schedule_edf(const gdo_job* jobs, int64_t n_jobs, const double* energy, const double* time,
                      const double* exec_time, const int32_t* sm_clock, int32_t n_clocks, int32_t mode,
                      int32_t budget_kind, int32_t objective, int32_t best_effort, gdo_decision* out,
                      int64_t* order);

#ifdef __cplusplus
}
#endif

#endif
