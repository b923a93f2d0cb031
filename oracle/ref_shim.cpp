// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the reference's OWN compiled sources
// (oracle/_ref/libgpudvfs_ref.so, built by oracle/Makefile from
// /root/reference/proj/src/*.cpp).  Tests use it to pin the C restatement
// (gd_oracle.c) and the CUDA path against the real reference, to generate the
// golden fixtures under tests/golden/, and bench.py --impl reference uses it
// to time the reference's CPU predict/select on the box's host cores.
// Nothing here is part of the product path.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "gpudvfs/clustering.hpp"
#include "gpudvfs/core.hpp"
#include "gpudvfs/ingest.hpp"
#include "gpudvfs/models.hpp"
#include "gpudvfs/rng.hpp"
#include "gpudvfs/scheduler.hpp"
#include "gpudvfs/synthdata.hpp"

using namespace gpudvfs;

namespace {

thread_local std::string g_err;

struct ForestView {
    int32_t n_trees;
    const int64_t* tree_offsets;
    const int32_t* feature;
    const double* threshold;
    const int32_t* left;
    const int32_t* right;
    const double* leaf_value;
};

struct Decision {
    int32_t clock_index;
    int16_t status;
    int16_t note;
    double energy_ws;
    double time_s;
};

struct JobIn {
    double arrival_s;
    double deadline_s;
    int64_t app_rank;
    int32_t app_index;
    int32_t pad;
};

std::vector<std::string> column_names(int n) {
    std::vector<std::string> c;
    for (int j = 0; j < n; ++j) {
        char buf[32];
        std::snprintf(buf, sizeof(buf), "c%03d", j);
        c.push_back(buf);
    }
    return c;
}

models::FittedModel forest_model(const ForestView* f, double base, double lr, int target, int n_cols) {
    models::FittedModel m;
    m.kind = models::ModelKind::gbt;
    m.target = target == 0 ? TargetKind::energy : TargetKind::time;
    m.columns = column_names(n_cols);
    m.gbt.base_prediction = base;
    m.gbt.learning_rate = lr;
    for (int t = 0; t < f->n_trees; ++t) {
        models::GbtTree tree;
        for (int64_t k = f->tree_offsets[t]; k < f->tree_offsets[t + 1]; ++k) {
            models::GbtNode n;
            n.feature = f->feature[k];
            n.threshold = f->threshold[k];
            n.left = f->left[k];
            n.right = f->right[k];
            n.leaf_value = f->leaf_value[k];
            tree.nodes.push_back(n);
        }
        m.gbt.trees.push_back(std::move(tree));
    }
    return m;
}

ingest::EncodedMatrix matrix_of(const double* rows, int64_t n_rows, int n_cols, const std::vector<std::string>& cols) {
    ingest::EncodedMatrix m;
    m.columns = cols;
    m.rows.resize(static_cast<std::size_t>(n_rows));
    for (int64_t r = 0; r < n_rows; ++r) m.rows[r].assign(rows + r * n_cols, rows + (r + 1) * n_cols);
    m.targets.assign(static_cast<std::size_t>(n_rows), 0.0);
    return m;
}

Decision to_decision(const sched::ScheduleDecision& d, const std::vector<ClockSet>& catalog) {
    Decision o{};
    o.clock_index = -1;
    o.status = d.status == sched::DecisionStatus::scheduled ? 0 : 1;
    o.note = d.note == "best_effort" ? 1 : (d.note == "missing correlated data" ? 2 : 0);
    if (d.chosen_clock) {
        for (std::size_t i = 0; i < catalog.size(); ++i) {
            if (catalog[i] == *d.chosen_clock) o.clock_index = static_cast<int32_t>(i);
        }
    }
    if (d.predicted_energy_ws) o.energy_ws = *d.predicted_energy_ws;
    if (d.predicted_time_s) o.time_s = *d.predicted_time_s;
    return o;
}

template <typename T>
void write_bin(const std::string& path, const std::vector<T>& v) {
    std::ofstream out(path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

std::string app_name(int64_t rank) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "app%010lld", static_cast<long long>(rank));
    return buf;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// models::predict over a synthetic forest (models.cpp:395-428).
int ref_predict_forest(const ForestView* f, double base, double lr, int target, const double* rows,
                       int64_t n_rows, int n_cols, double* out) {
    try {
        models::FittedModel m = forest_model(f, base, lr, target, n_cols);
        std::vector<double> p = models::predict(m, matrix_of(rows, n_rows, n_cols, m.columns));
        std::memcpy(out, p.data(), p.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Write a forest as a "gpudvfs-model 1" file through the reference's save_model.
int ref_save_forest(const ForestView* f, double base, double lr, int target, int n_cols, const char* path) {
    try {
        models::save_model_file(forest_model(f, base, lr, target, n_cols), path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// load_model_file + predict on raw rows (the production CLI path, cli.cpp:457-458).
int ref_predict_model_file(const char* path, const double* rows, int64_t n_rows, int n_cols, double* out) {
    try {
        models::FittedModel m = models::load_model_file(path);
        if (static_cast<int>(m.columns.size()) != n_cols) {
            g_err = "column count mismatch";
            return 1;
        }
        std::vector<double> p = models::predict(m, matrix_of(rows, n_rows, n_cols, m.columns));
        std::memcpy(out, p.data(), p.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Exercise the reference's column check (models.cpp:396-412); returns the message.
int ref_predict_column_mismatch(const char* model_path, const char* const* cols, int n_cols, char* msg, int cap) {
    try {
        models::FittedModel m = models::load_model_file(model_path);
        ingest::EncodedMatrix rows;
        for (int j = 0; j < n_cols; ++j) rows.columns.push_back(cols[j]);
        rows.rows.push_back(std::vector<double>(static_cast<std::size_t>(n_cols), 0.0));
        rows.targets.push_back(0.0);
        models::predict(m, rows);
        return 0;
    } catch (const std::invalid_argument& e) {
        std::snprintf(msg, static_cast<std::size_t>(cap), "%s", e.what());
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// schedule_d_dvfs (scheduler.cpp:182-237) with a ClockPredictor over E/T
// tables and an ExecutionTimeSource over an exec table.  Job app_ids are
// synthesised so that std::string order equals app_rank order.
int ref_schedule_tables(const JobIn* jobs, int64_t n_jobs, const double* energy, const double* time,
                        const double* exec_time, const int32_t* sm, const int32_t* mem, int32_t n_clocks,
                        int mode, int budget, int objective, int best_effort, Decision* out, int64_t* order) {
    try {
        DeviceSpec dev;
        dev.name = "tables";
        ClockSet top{0, 0};
        for (int c = 0; c < n_clocks; ++c) {
            ClockSet cs{sm[c], mem[c]};
            dev.supported_clocks.push_back(cs);
            if (cs.sm_clock_mhz > top.sm_clock_mhz ||
                (cs.sm_clock_mhz == top.sm_clock_mhz && cs.mem_clock_mhz > top.mem_clock_mhz)) {
                top = cs;
            }
        }
        dev.default_clock = dev.supported_clocks.front();
        dev.max_clock = top;
        std::vector<ClockSet> catalog = clock_catalog(dev);
        std::map<ClockSet, int> clock_index;
        for (int c = 0; c < n_clocks; ++c) clock_index[catalog[c]] = c;

        Workload w;
        w.device = dev;
        std::map<std::string, int32_t> app_index;
        std::map<std::string, std::vector<int64_t>> job_of_key;
        for (int64_t i = 0; i < n_jobs; ++i) {
            Job j;
            j.app_id = app_name(jobs[i].app_rank);
            j.arrival_s = jobs[i].arrival_s;
            j.deadline_s = jobs[i].deadline_s;
            j.default_profile.clock = dev.default_clock;
            app_index[j.app_id] = jobs[i].app_index;
            w.jobs.push_back(j);
        }
        sched::ClockPredictor pred = [&](const Job& job, const ClockSet& clock) -> std::optional<sched::ClockPrediction> {
            int32_t a = app_index.at(job.app_id);
            if (a < 0) return std::nullopt;
            int c = clock_index.at(clock);
            return sched::ClockPrediction{energy[static_cast<int64_t>(a) * n_clocks + c],
                                          time[static_cast<int64_t>(a) * n_clocks + c]};
        };
        sched::ExecutionTimeSource exec = [&](const Job& job, const ClockSet& clock) {
            int32_t a = app_index.at(job.app_id);
            return exec_time[static_cast<int64_t>(a) * n_clocks + clock_index.at(clock)];
        };
        sched::SchedulerOptions opt;
        opt.mode = mode == 0 ? sched::SelectionMode::text_semantics : sched::SelectionMode::literal_pseudocode;
        opt.budget = budget == 0 ? sched::DeadlineBudget::remaining_time : sched::DeadlineBudget::full_deadline;
        opt.objective = objective == 0 ? sched::Objective::energy : sched::Objective::power;
        opt.best_effort_fallback = best_effort != 0;
        std::vector<sched::ScheduleDecision> ds = sched::schedule_d_dvfs(w, pred, exec, opt);
        // Map decisions back to input job indices (jobs are distinct by
        // (app_rank, arrival, deadline) in the tests that use this).
        std::vector<bool> used(static_cast<std::size_t>(n_jobs), false);
        for (std::size_t k = 0; k < ds.size(); ++k) {
            out[k] = to_decision(ds[k], catalog);
            order[k] = -1;
            for (int64_t i = 0; i < n_jobs; ++i) {
                if (!used[i] && w.jobs[i].app_id == ds[k].job.app_id && w.jobs[i].arrival_s == ds[k].job.arrival_s &&
                    w.jobs[i].deadline_s == ds[k].job.deadline_s) {
                    used[i] = true;
                    order[k] = i;
                    break;
                }
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// The paper-scale C1 scenario through the reference's production path
// (cli.cpp:400-481): P100 device, 12-app suite catalog at `stride`, GBT
// energy/time models {iters, depth, 0.1, 3.0, seed} saved + reloaded as
// "gpudvfs-model 1" files, k-means clusters (select_k, cli.cpp:470-472),
// `n_jobs` seeded query apps, make_model_predictor + schedule_d_dvfs.
// Everything the GPU path needs (and every reference output) goes to out_dir.
int ref_c1_scenario(const char* out_dir, uint64_t seed, int stride, int iters, int depth, int n_jobs, int mode,
                    int budget, int objective, int best_effort) {
    try {
        const std::string dir(out_dir);
        synth::SyntheticGpu p100 = synth::builtin_p100_gpu();
        synth::ArchetypeSuite suite = synth::builtin_default_suite();
        Dataset catalog = p100.generate_dataset(suite, stride);

        ingest::EncodeResult enc_e = ingest::encode(catalog, catalog, TargetKind::energy, 1.0, seed);
        ingest::EncodeResult enc_t = ingest::encode(catalog, catalog, TargetKind::time, 1.0, seed);
        models::GBTConfig cfg{iters, depth, 0.1, 3.0, seed};
        models::FittedModel me = models::fit_gbt(enc_e.train, cfg);
        models::FittedModel mt = models::fit_gbt(enc_t.train, cfg);
        me.encoding_ref = "encoding_energy.txt";
        mt.encoding_ref = "encoding_time.txt";
        models::save_model_file(me, dir + "/model_energy_gbt.txt");
        models::save_model_file(mt, dir + "/model_time_gbt.txt");
        ingest::save_encoding_file(enc_e.metadata, dir + "/encoding_energy.txt");
        ingest::save_encoding_file(enc_t.metadata, dir + "/encoding_time.txt");
        // Production numbering: reload (preorder ids, models.cpp:581-607).
        me = models::load_model_file(dir + "/model_energy_gbt.txt");
        mt = models::load_model_file(dir + "/model_time_gbt.txt");
        ingest::EncodingMetadata ee = ingest::load_encoding_file(dir + "/encoding_energy.txt");
        ingest::EncodingMetadata te = ingest::load_encoding_file(dir + "/encoding_time.txt");

        cluster::PointMatrix points = cluster::default_clock_points(catalog);
        int k_max = std::min<int>(9, static_cast<int>(points.rows.size()));
        cluster::KMeansModel clusters = cluster::select_k(points, 1, k_max, seed).best_model;

        // Seeded query apps inside the suite's parameter ranges (synthdata.cpp:304-315).
        synth::ArchetypeSuite queries;
        for (int i = 0; i < n_jobs; ++i) {
            SplitMix64 r(seed ^ (0x5151ULL + static_cast<uint64_t>(i) * 0x9e3779b97f4a7c15ULL));
            synth::AppArchetype a;
            a.app_id = app_name(i);
            a.compute_work = r.uniform(420.0, 5300.0);
            a.memory_work = r.uniform(70.0, 1950.0);
            a.stall_s = r.uniform(0.10, 1.40);
            a.power_coeff_core = r.uniform(0.034, 0.105);
            a.power_coeff_mem = r.uniform(0.007, 0.058);
            a.noise_seed = static_cast<uint64_t>(i) + 1;
            queries.apps.push_back(a);
        }
        std::vector<ProfileRecord> default_profiles;
        for (const auto& a : queries.apps) default_profiles.push_back(p100.profile(a, p100.device().default_clock));
        sched::WorkloadGenConfig gen;
        gen.seed = seed;
        Workload workload = sched::generate_workload(default_profiles, p100.device(), gen);
        sched::ExecutionTimeSource exec = sched::make_truth_exec(queries, p100);

        std::vector<ClockSet> cat = clock_catalog(catalog.device);
        const int C = static_cast<int>(cat.size());
        const int F = static_cast<int>(ee.columns.size());

        // Row material for the GPU path: every catalog record encoded once per
        // target (ingest.cpp:401-439); the kernel overrides the clock columns.
        ingest::EncodedMatrix rows_e = ingest::apply_encoding(ee, catalog.records);
        ingest::EncodedMatrix rows_t = ingest::apply_encoding(te, catalog.records);
        std::vector<double> rows_flat, cat_t;
        std::vector<int32_t> cat_cols;
        for (const auto& name : ee.categorical_columns) cat_cols.push_back(static_cast<int32_t>(*rows_e.column_index(name)));
        for (std::size_t r = 0; r < rows_e.rows.size(); ++r) {
            rows_flat.insert(rows_flat.end(), rows_e.rows[r].begin(), rows_e.rows[r].end());
            for (int32_t c : cat_cols) cat_t.push_back(rows_t.rows[r][static_cast<std::size_t>(c)]);
        }

        // Per job: matched app (clustering.cpp:346-411) and the nearest-record
        // map (scheduler.cpp:341-359), jobs in workload order.
        std::vector<int32_t> rec_of_clock;
        std::vector<double> arrival, deadline, exec_tab;
        for (const Job& job : workload.jobs) {
            cluster::CorrelationResult match = cluster::correlate(clusters, catalog, job.default_profile);
            std::vector<int32_t> recs;
            for (std::size_t r = 0; r < catalog.records.size(); ++r) {
                if (catalog.records[r].app_id == match.matched_app) recs.push_back(static_cast<int32_t>(r));
            }
            for (const ClockSet& clock : cat) {
                int32_t nearest = recs.front();
                auto dist = [&](int32_t r) {
                    const ClockSet& rc = catalog.records[static_cast<std::size_t>(r)].clock;
                    return std::make_pair(std::abs(rc.mem_clock_mhz - clock.mem_clock_mhz),
                                          std::abs(rc.sm_clock_mhz - clock.sm_clock_mhz));
                };
                for (int32_t r : recs) {
                    if (dist(r) < dist(nearest)) nearest = r;
                }
                rec_of_clock.push_back(nearest);
                exec_tab.push_back(exec(job, clock));
            }
            arrival.push_back(job.arrival_s);
            deadline.push_back(job.deadline_s);
        }

        // The reference's own predictor outputs and decisions.
        sched::ClockPredictor predictor =
            sched::make_model_predictor(me, ee, mt, te, catalog, clusters);
        std::vector<double> pe, pt;
        for (const Job& job : workload.jobs) {
            for (const ClockSet& clock : cat) {
                auto p = predictor(job, clock);
                pe.push_back(p ? p->energy_ws : -1.0);
                pt.push_back(p ? p->time_s : -1.0);
            }
        }
        sched::SchedulerOptions opt;
        opt.mode = mode == 0 ? sched::SelectionMode::text_semantics : sched::SelectionMode::literal_pseudocode;
        opt.budget = budget == 0 ? sched::DeadlineBudget::remaining_time : sched::DeadlineBudget::full_deadline;
        opt.objective = objective == 0 ? sched::Objective::energy : sched::Objective::power;
        opt.best_effort_fallback = best_effort != 0;
        std::vector<sched::ScheduleDecision> ds = sched::schedule_d_dvfs(workload, predictor, exec, opt);
        std::vector<Decision> dout;
        std::vector<int64_t> order;
        for (const auto& d : ds) {
            dout.push_back(to_decision(d, cat));
            for (std::size_t i = 0; i < workload.jobs.size(); ++i) {
                if (workload.jobs[i].app_id == d.job.app_id) order.push_back(static_cast<int64_t>(i));
            }
        }
        std::vector<int32_t> sm, mem;
        for (const auto& c : cat) {
            sm.push_back(c.sm_clock_mhz);
            mem.push_back(c.mem_clock_mhz);
        }
        std::vector<int32_t> meta = {static_cast<int32_t>(workload.jobs.size()), C, F,
                                     static_cast<int32_t>(catalog.records.size()),
                                     static_cast<int32_t>(cat_cols.size()),
                                     static_cast<int32_t>(*rows_e.column_index("sm_clock")),
                                     static_cast<int32_t>(*rows_e.column_index("mem_clock"))};
        write_bin(dir + "/meta.i32", meta);
        write_bin(dir + "/rows.f64", rows_flat);
        write_bin(dir + "/cat_t.f64", cat_t);
        write_bin(dir + "/cat_cols.i32", cat_cols);
        write_bin(dir + "/rec_of_clock.i32", rec_of_clock);
        write_bin(dir + "/sm.i32", sm);
        write_bin(dir + "/mem.i32", mem);
        write_bin(dir + "/arrival.f64", arrival);
        write_bin(dir + "/deadline.f64", deadline);
        write_bin(dir + "/exec.f64", exec_tab);
        write_bin(dir + "/pred_energy.f64", pe);
        write_bin(dir + "/pred_time.f64", pt);
        write_bin(dir + "/decisions.bin", dout);
        write_bin(dir + "/order.i64", order);
        std::ofstream cols(dir + "/columns.txt");
        for (const auto& c : ee.columns) cols << c << "\n";
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// The encoded training matrix of the paper-scale C1 catalog (P100 suite at
// `stride`, ingest::encode for `target`): rows == NULL returns the shape only.
int ref_c1_train(uint64_t seed, int stride, int target, double* rows, double* targets, int64_t* n_rows,
                 int32_t* n_cols) {
    try {
        synth::SyntheticGpu p100 = synth::builtin_p100_gpu();
        Dataset catalog = p100.generate_dataset(synth::builtin_default_suite(), stride);
        ingest::EncodeResult enc = ingest::encode(catalog, catalog, target == 0 ? TargetKind::energy : TargetKind::time,
                                                  1.0, seed);
        *n_rows = static_cast<int64_t>(enc.train.rows.size());
        *n_cols = static_cast<int32_t>(enc.train.columns.size());
        if (rows) {
            for (std::size_t r = 0; r < enc.train.rows.size(); ++r) {
                std::memcpy(rows + r * enc.train.columns.size(), enc.train.rows[r].data(),
                            enc.train.columns.size() * sizeof(double));
                targets[r] = enc.train.targets[r];
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// models::fit_gbt on a given matrix; the trees stay in fit_gbt's node order
// (NOT reloaded).  ref_fit_gbt fits and keeps the model; ref_fit_gbt_export
// copies it out (arrays sized by the n_trees / n_nodes ref_fit_gbt returned).
thread_local models::FittedModel g_fit;
int ref_fit_gbt(const double* rows, int64_t n_rows, int n_cols, const double* targets, int iterations, int depth,
                double lr, double l2, uint64_t seed, int target, int32_t* n_trees, int64_t* n_nodes, double* base) {
    try {
        ingest::EncodedMatrix m = matrix_of(rows, n_rows, n_cols, column_names(n_cols));
        m.targets.assign(targets, targets + n_rows);
        m.target = target == 0 ? TargetKind::energy : TargetKind::time;
        models::GBTConfig cfg{iterations, depth, lr, l2, seed};
        g_fit = models::fit_gbt(m, cfg);
        *n_trees = static_cast<int32_t>(g_fit.gbt.trees.size());
        int64_t nn = 0;
        for (const auto& t : g_fit.gbt.trees) nn += static_cast<int64_t>(t.nodes.size());
        *n_nodes = nn;
        *base = g_fit.gbt.base_prediction;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_fit_gbt_export(int64_t* offsets, int32_t* feature, double* threshold, int32_t* left, int32_t* right,
                       double* leaf_value) {
    int64_t k = 0;
    offsets[0] = 0;
    for (std::size_t t = 0; t < g_fit.gbt.trees.size(); ++t) {
        for (const auto& n : g_fit.gbt.trees[t].nodes) {
            feature[k] = n.feature;
            threshold[k] = n.threshold;
            left[k] = n.left;
            right[k] = n.right;
            leaf_value[k] = n.leaf_value;
            ++k;
        }
        offsets[t + 1] = k;
    }
    return 0;
}

// Acceptance #1 material: truth E/T over the P100 catalog for
// the 12 suite apps with noise offset `seed_offset`, and oracle_per_job's
// decision for each app at the given relative deadlines (scheduler.cpp:257-281).
int ref_truth_oracle(uint64_t seed_offset, const double* deadlines, double* energy, double* time, Decision* out,
                     int32_t* sm_out) {
    try {
        synth::SyntheticGpu p100 = synth::builtin_p100_gpu();
        synth::ArchetypeSuite suite = synth::builtin_default_suite(seed_offset);
        std::vector<ClockSet> cat = clock_catalog(p100.device());
        const int C = static_cast<int>(cat.size());
        for (int c = 0; c < C; ++c) sm_out[c] = cat[c].sm_clock_mhz;
        for (std::size_t a = 0; a < suite.apps.size(); ++a) {
            for (int c = 0; c < C; ++c) {
                energy[a * C + c] = p100.true_energy_ws(suite.apps[a], cat[c]);
                time[a * C + c] = p100.true_time_s(suite.apps[a], cat[c]);
            }
            Job job;
            job.app_id = suite.apps[a].app_id;
            job.deadline_s = deadlines[a];
            out[a] = to_decision(sched::oracle_per_job(job, suite.apps[a], p100), cat);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// CPU baseline for bench.py: the reference's models::predict (E and T) over
// materialised (app x clock) rows of a bounded app sample, then the
// reference's schedule_d_dvfs (full_deadline, energy, text) over the
// predictions; `threads` independent contiguous app partitions.  Returns
// elapsed seconds (or < 0 on error); decisions are written for checking.
double ref_bench_grid(const ForestView* fe, double base_e, double lr_e, const ForestView* ft, double base_t,
                      double lr_t, const double* rows, int n_cols, const double* cat_t, const int32_t* cat_cols,
                      int n_cat, int64_t n_apps, const int32_t* sm, const int32_t* mem, int32_t n_clocks, int sm_col,
                      int mem_col, const double* budgets, int threads, Decision* out, double* e_out,
                      double* t_out) {
    try {
        models::FittedModel me = forest_model(fe, base_e, lr_e, 0, n_cols);
        models::FittedModel mt = forest_model(ft, base_t, lr_t, 1, n_cols);
        if (threads < 1) threads = 1;
        std::vector<std::thread> pool;
        std::atomic<int> failed{0};
        auto t0 = std::chrono::steady_clock::now();
        for (int w = 0; w < threads; ++w) {
            int64_t a0 = n_apps * w / threads, a1 = n_apps * (w + 1) / threads;
            pool.emplace_back([&, a0, a1]() {
                try {
                    for (int64_t a = a0; a < a1; ++a) {
                        ingest::EncodedMatrix xe, xt;
                        xe.columns = me.columns;
                        xt.columns = mt.columns;
                        for (int c = 0; c < n_clocks; ++c) {
                            std::vector<double> r(rows + a * n_cols, rows + (a + 1) * n_cols);
                            if (sm_col >= 0) r[sm_col] = sm[c];
                            if (mem_col >= 0) r[mem_col] = mem[c];
                            std::vector<double> rt = r;
                            for (int k = 0; k < n_cat; ++k) rt[cat_cols[k]] = cat_t[a * n_cat + k];
                            xe.rows.push_back(std::move(r));
                            xt.rows.push_back(std::move(rt));
                        }
                        std::vector<double> e = models::predict(me, xe);
                        std::vector<double> t = models::predict(mt, xt);
                        if (e_out) std::copy(e.begin(), e.end(), e_out + a * n_clocks);
                        if (t_out) std::copy(t.begin(), t.end(), t_out + a * n_clocks);
                        DeviceSpec dev;
                        dev.name = "bench";
                        for (int c = 0; c < n_clocks; ++c) dev.supported_clocks.push_back({sm[c], mem[c]});
                        dev.default_clock = dev.supported_clocks.front();
                        dev.max_clock = dev.supported_clocks.front();
                        Workload wl;
                        wl.device = dev;
                        Job job;
                        job.app_id = "a";
                        job.deadline_s = budgets[a];
                        wl.jobs.push_back(job);
                        std::map<ClockSet, int> idx;
                        for (int c = 0; c < n_clocks; ++c) idx[{sm[c], mem[c]}] = c;
                        sched::ClockPredictor pred = [&](const Job&, const ClockSet& cs) {
                            int c = idx.at(cs);
                            return std::optional<sched::ClockPrediction>(sched::ClockPrediction{e[c], t[c]});
                        };
                        sched::ExecutionTimeSource ex = [](const Job&, const ClockSet&) { return 0.0; };
                        sched::SchedulerOptions opt;
                        opt.budget = sched::DeadlineBudget::full_deadline;
                        auto ds = sched::schedule_d_dvfs(wl, pred, ex, opt);
                        std::vector<ClockSet> cat = clock_catalog(dev);
                        out[a] = to_decision(ds.front(), cat);
                    }
                } catch (...) {
                    failed = 1;
                }
            });
        }
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        if (failed) {
            g_err = "worker failed";
            return -1.0;
        }
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

}  // extern "C"
