// integration/gpudvfs_gpu.cpp -- implementation of include/gpudvfs_b200/gpu_api.hpp.
//
// This is the reference-side binding: it is compiled against the reference's
// own headers and links into the reference's library, and it reaches the
// GPU only through the C ABI (gdvfs.h).  Everything per (app x clock) runs on
// the device.  The per-job host steps are restructured around
// what they depend on: correlation (clustering.cpp:346-411) recomputes the
// catalog's default-clock points, their cluster labels and default times on
// every call -- here they are computed once per predictor (CatalogIndex) and
// a query costs one k-means assignment plus a scan of the catalog apps; and a
// job's candidate rows (scheduler.cpp:330-359) depend only on the catalog app
// it correlates to, so the nearest-record substitution, the categorical
// encoding (the reference's apply_encoding, ingest.cpp:401-439) and the GPU
// evaluation run once per distinct matched app, not once per job.
#include "gpudvfs_b200/gpu_api.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace gpudvfs::gpu {
namespace {

thread_local int t_device = 0;

[[noreturn]] void throw_gd(int rc) {
    const std::string m = gd_last_error();
    switch (rc) {
        case GD_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case GD_ERR_DATA: throw data_error(m);
        case GD_ERR_MISSING_ARTIFACT: throw missing_artifact_error(m);
        case GD_ERR_IO: throw io_error(m);
        default: throw std::runtime_error("gdvfs: " + m);
    }
}

void check(int rc) {
    if (rc != GD_OK) throw_gd(rc);
}

struct CtxHolder {
    gd_ctx* ctx = nullptr;
    int device = -1;
    ~CtxHolder() {
        if (ctx) gd_ctx_destroy(ctx);
    }
};

gd_ctx* context() {
    thread_local CtxHolder h;
    if (!h.ctx || h.device != t_device) {
        if (h.ctx) gd_ctx_destroy(h.ctx);
        h.ctx = nullptr;
        check(gd_ctx_create(t_device, &h.ctx));
        h.device = t_device;
    }
    return h.ctx;
}

struct ModelHandle {
    gd_model* m = nullptr;
    ModelHandle() = default;
    ModelHandle(const ModelHandle&) = delete;
    ModelHandle& operator=(const ModelHandle&) = delete;
    ~ModelHandle() {
        if (m) gd_model_free(m);
    }
};

std::unique_ptr<ModelHandle> upload(const models::FittedModel& fm) {
    auto h = std::make_unique<ModelHandle>();
    const int32_t n_cols = static_cast<int32_t>(fm.columns.size());
    const int32_t target = fm.target == TargetKind::energy ? GD_TARGET_ENERGY : GD_TARGET_TIME;
    if (fm.kind == models::ModelKind::gbt) {
        std::vector<int64_t> off{0};
        std::vector<int32_t> feat, left, right;
        std::vector<double> thr, leaf;
        for (const auto& tree : fm.gbt.trees) {
            for (const auto& n : tree.nodes) {
                feat.push_back(n.feature);
                thr.push_back(n.threshold);
                left.push_back(n.left);
                right.push_back(n.right);
                leaf.push_back(n.leaf_value);
            }
            off.push_back(static_cast<int64_t>(feat.size()));
        }
        gd_forest_view v{static_cast<int32_t>(fm.gbt.trees.size()), off.data(), feat.data(), thr.data(),
                         left.data(), right.data(), leaf.data()};
        check(gd_model_upload_gbt(context(), &v, fm.gbt.base_prediction, fm.gbt.learning_rate, n_cols, target, &h->m));
    } else {
        const int32_t kind = fm.kind == models::ModelKind::ols ? GD_KIND_OLS : GD_KIND_LASSO;
        check(gd_model_upload_linear(context(), fm.linear.coefficients.data(), n_cols, fm.linear.intercept, kind,
                                     target, &h->m));
    }
    return h;
}

// models.cpp:396-412 -- the reference's column check, same messages.
void check_columns(const std::vector<std::string>& model, const std::vector<std::string>& rows) {
    if (model.size() != rows.size()) {
        const std::size_t limit = std::min(model.size(), rows.size());
        for (std::size_t j = 0; j < limit; ++j) {
            if (model[j] != rows[j]) {
                throw std::invalid_argument("predict: column mismatch at '" + rows[j] + "' (model expects '" +
                                            model[j] + "')");
            }
        }
        const auto& longer = model.size() > rows.size() ? model : rows;
        throw std::invalid_argument("predict: column mismatch at '" + longer[limit] + "'");
    }
    for (std::size_t j = 0; j < model.size(); ++j) {
        if (model[j] != rows[j]) {
            throw std::invalid_argument("predict: column mismatch at '" + rows[j] + "' (model expects '" + model[j] +
                                        "')");
        }
    }
}

int column_of(const std::vector<std::string>& cols, const std::string& name) {
    auto it = std::find(cols.begin(), cols.end(), name);
    return it == cols.end() ? -1 : static_cast<int>(it - cols.begin());
}

// The catalog side of cluster::correlate (clustering.cpp:346-411), computed
// once: default-clock points, each catalog app's cluster label and
// default-clock time, and each app's records in catalog order.
struct CatalogIndex {
    struct Candidate {
        std::string app_id;
        double time_s = 0.0;
        int label = -1;
    };
    bool ok = false;  // false: correlate would throw for every query
    cluster::PointMatrix points;
    std::vector<Candidate> candidates;
    std::map<std::string, std::vector<std::size_t>> records_of;

    void build(const Dataset& catalog, const cluster::KMeansModel& clusters) {
        for (std::size_t i = 0; i < catalog.records.size(); ++i) records_of[catalog.records[i].app_id].push_back(i);
        if (catalog.records.empty()) return;
        try {
            points = cluster::default_clock_points(catalog);
            for (std::size_t i = 0; i < points.rows.size(); ++i) {
                Candidate c;
                c.app_id = points.ids[i];
                c.label = clusters.assign(points.rows[i], points.columns);
                for (std::size_t r : records_of[c.app_id]) {  // first default-clock record, catalog order
                    if (catalog.records[r].clock == catalog.device.default_clock) {
                        c.time_s = catalog.records[r].time_s;
                        break;
                    }
                }
                candidates.push_back(std::move(c));
            }
            ok = true;
        } catch (const std::exception&) {
            ok = false;
        }
    }

    // correlate(...).matched_app for `query`; throws where correlate throws.
    const std::string& matched_app(const cluster::KMeansModel& clusters, const Dataset& catalog,
                                   const ProfileRecord& query) const {
        if (catalog.records.empty()) throw std::invalid_argument("correlate: catalog is empty");
        if (query.clock != catalog.device.default_clock) {
            throw std::invalid_argument("correlate: query record must be at the device default clock");
        }
        if (!ok) throw std::invalid_argument("correlate: catalog points unavailable");
        std::vector<double> row;
        row.reserve(points.columns.size());
        for (const auto& name : points.columns) {
            auto it = query.features.numeric.find(name);
            if (it == query.features.numeric.end()) {
                throw std::invalid_argument("correlate: query lacks numeric feature '" + name + "'");
            }
            row.push_back(it->second);
        }
        const int label = clusters.assign(row, points.columns);
        auto better = [&](const Candidate& a, const Candidate& b) {  // clustering.cpp:384-389
            const double da = std::abs(query.time_s - a.time_s), db = std::abs(query.time_s - b.time_s);
            if (da != db) return da < db;
            return a.app_id < b.app_id;
        };
        const Candidate* best = nullptr;
        for (const auto& c : candidates) {
            if (c.label != label || c.app_id == query.app_id) continue;
            if (best == nullptr || better(c, *best)) best = &c;
        }
        if (best == nullptr) {  // singleton cluster fallback (clustering.cpp:396-403)
            for (const auto& c : candidates) {
                if (best == nullptr || better(c, *best)) best = &c;
            }
        }
        if (best == nullptr) throw std::invalid_argument("correlate: no candidates");
        return best->app_id;
    }
};

using ClockTable = std::map<ClockSet, sched::ClockPrediction>;

// ---------------------------------------------------------------------------
// The GPU-backed ClockPredictor (replaces ModelPredictorState,
// scheduler.cpp:304-371).
// ---------------------------------------------------------------------------
struct GpuPredictorState {
    models::FittedModel energy_model, time_model;
    ingest::EncodingMetadata energy_encoding, time_encoding;
    Dataset catalog;
    cluster::KMeansModel clusters;
    CatalogIndex index;
    std::unique_ptr<ModelHandle> ge, gt;
    std::vector<ClockSet> clocks;
    std::vector<int32_t> sm, mem;
    std::map<std::string, std::shared_ptr<const ClockTable>> cache;  // per job app
    std::set<std::string> failed;                                     // per job app
    std::map<std::string, std::shared_ptr<const ClockTable>> by_match;  // per matched catalog app
    std::set<std::string> match_failed;
    bool columns_ok = true;

    // One batched launch for every not-yet-seen matched app among `jobs`.
    void prime(const std::vector<const Job*>& jobs) {
        struct Pending {
            std::string app_id;  // the matched catalog app
            std::vector<ProfileRecord> records;
            std::vector<int32_t> rec_local;  // per catalog clock
        };
        std::vector<std::pair<std::string, std::string>> resolved;  // (job app, matched app)
        std::vector<Pending> todo;
        std::set<std::string> queued;
        for (const Job* job : jobs) {
            if (cache.count(job->app_id) || failed.count(job->app_id)) continue;
            std::string m;
            try {
                m = index.matched_app(clusters, catalog, job->default_profile);
            } catch (const std::exception&) {
                failed.insert(job->app_id);
                continue;
            }
            resolved.emplace_back(job->app_id, m);
            if (by_match.count(m) || match_failed.count(m) || queued.count(m)) continue;
            queued.insert(m);
            // scheduler.cpp:330-359: the matched app's records and the nearest
            // profiled record per catalog clock.
            Pending p;
            p.app_id = m;
            for (std::size_t r : index.records_of[m]) p.records.push_back(catalog.records[r]);
            if (p.records.empty()) {
                match_failed.insert(m);
                continue;
            }
            for (const ClockSet& clock : clocks) {
                std::size_t nearest = 0;
                auto dist = [&](std::size_t i) {
                    return std::make_pair(std::abs(p.records[i].clock.mem_clock_mhz - clock.mem_clock_mhz),
                                          std::abs(p.records[i].clock.sm_clock_mhz - clock.sm_clock_mhz));
                };
                for (std::size_t i = 0; i < p.records.size(); ++i) {
                    if (dist(i) < dist(nearest)) nearest = i;
                }
                p.rec_local.push_back(static_cast<int32_t>(nearest));
            }
            todo.push_back(std::move(p));
        }
        if (!columns_ok) {
            for (const auto& p : todo) match_failed.insert(p.app_id);
            todo.clear();
        }
        if (!todo.empty()) evaluate(todo);
        for (const auto& [job_app, m] : resolved) {
            auto it = by_match.find(m);
            if (it == by_match.end()) failed.insert(job_app);
            else cache[job_app] = it->second;
        }
    }

    template <class P>
    void evaluate(std::vector<P>& todo) {
        const auto& cols = energy_encoding.columns;
        const int F = static_cast<int>(cols.size());
        std::vector<int32_t> cat_cols;
        for (const auto& name : energy_encoding.categorical_columns) cat_cols.push_back(column_of(cols, name));
        const int K = static_cast<int>(cat_cols.size());
        std::vector<double> rows, cat_t, budgets;
        std::vector<int32_t> rec_of_clock;
        std::vector<P*> batch;
        for (auto& p : todo) {
            try {
                ingest::EncodedMatrix xe = ingest::apply_encoding(energy_encoding, p.records);
                ingest::EncodedMatrix xt = ingest::apply_encoding(time_encoding, p.records);
                const int32_t base = static_cast<int32_t>(rows.size() / static_cast<std::size_t>(F));
                for (std::size_t r = 0; r < xe.rows.size(); ++r) {
                    rows.insert(rows.end(), xe.rows[r].begin(), xe.rows[r].end());
                    for (int32_t c : cat_cols) cat_t.push_back(xt.rows[r][static_cast<std::size_t>(c)]);
                }
                for (int32_t rl : p.rec_local) rec_of_clock.push_back(base + rl);
                budgets.push_back(0.0);
                batch.push_back(&p);
            } catch (const std::exception&) {
                match_failed.insert(p.app_id);
            }
        }
        if (batch.empty()) return;
        const int64_t A = static_cast<int64_t>(batch.size());
        const int32_t C = static_cast<int32_t>(clocks.size());
        std::vector<gd_decision> dec(static_cast<std::size_t>(A));
        std::vector<double> e(static_cast<std::size_t>(A) * C), t(static_cast<std::size_t>(A) * C);
        gd_grid g{};
        g.rows = rows.data();
        g.n_records = static_cast<int64_t>(rows.size() / static_cast<std::size_t>(F));
        g.n_cols = F;
        g.n_cat = K;
        g.cat_t = cat_t.data();
        g.cat_cols = cat_cols.data();
        g.rec_of_clock = rec_of_clock.data();
        g.n_apps = A;
        g.sm_clock = sm.data();
        g.mem_clock = mem.data();
        g.n_clocks = C;
        g.sm_col = column_of(cols, "sm_clock");
        g.mem_col = column_of(cols, "mem_clock");
        g.budgets = budgets.data();
        gd_select_opts o{GD_MODE_TEXT, GD_OBJECTIVE_ENERGY, 0, 0};
        check(gd_grid_select(context(), ge->m, gt->m, &g, &o, dec.data(), e.data(), t.data()));
        for (int64_t a = 0; a < A; ++a) {
            auto table = std::make_shared<ClockTable>();
            for (int32_t c = 0; c < C; ++c) {
                (*table)[clocks[static_cast<std::size_t>(c)]] =
                    sched::ClockPrediction{e[static_cast<std::size_t>(a * C + c)], t[static_cast<std::size_t>(a * C + c)]};
            }
            by_match[batch[static_cast<std::size_t>(a)]->app_id] = std::move(table);
        }
    }
};

struct GpuPredictorFn {
    std::shared_ptr<GpuPredictorState> state;
    std::optional<sched::ClockPrediction> operator()(const Job& job, const ClockSet& clock) const {
        if (state->failed.count(job.app_id)) return std::nullopt;
        auto hit = state->cache.find(job.app_id);
        if (hit == state->cache.end()) {
            state->prime({&job});
            hit = state->cache.find(job.app_id);
            if (hit == state->cache.end()) return std::nullopt;
        }
        auto it = hit->second->find(clock);
        if (it == hit->second->end()) return std::nullopt;
        return it->second;
    }
};

thread_local const sched::ExecutionTimeSource* t_exec = nullptr;
thread_local const std::vector<Job>* t_jobs = nullptr;
thread_local const std::vector<ClockSet>* t_catalog = nullptr;

double exec_trampoline(void*, int64_t job, int32_t clock_index) {
    return (*t_exec)((*t_jobs)[static_cast<std::size_t>(job)], (*t_catalog)[static_cast<std::size_t>(clock_index)]);
}

}  // namespace

void select_device(int device) { t_device = device; }

std::vector<double> predict(const models::FittedModel& model, const ingest::EncodedMatrix& rows) {
    check_columns(model.columns, rows.columns);
    const int32_t F = static_cast<int32_t>(model.columns.size());
    std::vector<double> flat;
    flat.reserve(rows.rows.size() * static_cast<std::size_t>(F));
    for (const auto& r : rows.rows) {
        if (r.size() != static_cast<std::size_t>(F)) throw std::invalid_argument("predict: ragged row");
        flat.insert(flat.end(), r.begin(), r.end());
    }
    std::vector<double> out(rows.rows.size());
    if (rows.rows.empty()) return out;
    auto h = upload(model);
    check(gd_predict_rows(context(), h->m, flat.data(), static_cast<int64_t>(rows.rows.size()), F, out.data(), nullptr));
    return out;
}

sched::ClockPredictor make_model_predictor(models::FittedModel energy_model, ingest::EncodingMetadata energy_encoding,
                                           models::FittedModel time_model, ingest::EncodingMetadata time_encoding,
                                           Dataset catalog, cluster::KMeansModel clusters) {
    auto s = std::make_shared<GpuPredictorState>();
    s->energy_model = std::move(energy_model);
    s->energy_encoding = std::move(energy_encoding);
    s->time_model = std::move(time_model);
    s->time_encoding = std::move(time_encoding);
    s->catalog = std::move(catalog);
    s->clusters = std::move(clusters);
    if (s->energy_encoding.columns != s->time_encoding.columns) {
        throw std::invalid_argument("make_model_predictor: energy and time encodings disagree on columns");
    }
    // models::predict's column check (models.cpp:396-412).  The reference
    // throws it inside build(), which predictions_for turns into a per-job
    // "missing correlated data" rejection (scheduler.cpp:316-324); same here.
    try {
        check_columns(s->energy_model.columns, s->energy_encoding.columns);
        check_columns(s->time_model.columns, s->time_encoding.columns);
    } catch (const std::invalid_argument&) {
        s->columns_ok = false;
    }
    s->index.build(s->catalog, s->clusters);
    s->ge = upload(s->energy_model);
    s->gt = upload(s->time_model);
    s->clocks = clock_catalog(s->catalog.device);
    for (const auto& c : s->clocks) {
        s->sm.push_back(c.sm_clock_mhz);
        s->mem.push_back(c.mem_clock_mhz);
    }
    return GpuPredictorFn{s};
}

std::vector<sched::ScheduleDecision> schedule_d_dvfs(const Workload& workload, const sched::ClockPredictor& predictor,
                                                     const sched::ExecutionTimeSource& exec,
                                                     const sched::SchedulerOptions& options) {
    const std::vector<ClockSet> catalog = clock_catalog(workload.device);
    const int32_t C = static_cast<int32_t>(catalog.size());
    const int64_t n = static_cast<int64_t>(workload.jobs.size());
    if (const GpuPredictorFn* fn = predictor.target<GpuPredictorFn>()) {
        std::vector<const Job*> all;
        for (const auto& j : workload.jobs) all.push_back(&j);
        fn->state->prime(all);  // one launch for the whole batch
    }
    // Per-job candidate tables in catalog order (scheduler.cpp:193-201).
    std::vector<double> E(static_cast<std::size_t>(n) * C), T(static_cast<std::size_t>(n) * C);
    std::vector<std::string> ids;
    for (const auto& j : workload.jobs) ids.push_back(j.app_id);
    std::vector<std::string> sorted_ids = ids;
    std::sort(sorted_ids.begin(), sorted_ids.end());
    std::vector<gd_job> jobs(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const Job& job = workload.jobs[static_cast<std::size_t>(i)];
        gd_job& gj = jobs[static_cast<std::size_t>(i)];
        gj.arrival_s = job.arrival_s;
        gj.deadline_s = job.deadline_s;
        gj.app_rank = std::lower_bound(sorted_ids.begin(), sorted_ids.end(), job.app_id) - sorted_ids.begin();
        gj.app_index = static_cast<int32_t>(i);
        gj.pad = 0;
        for (int32_t c = 0; c < C; ++c) {
            auto p = predictor(job, catalog[static_cast<std::size_t>(c)]);
            if (!p) {
                gj.app_index = -1;
                break;
            }
            E[static_cast<std::size_t>(i * C + c)] = p->energy_ws;
            T[static_cast<std::size_t>(i * C + c)] = p->time_s;
        }
    }
    std::vector<int32_t> sm;
    for (const auto& c : catalog) sm.push_back(c.sm_clock_mhz);
    gd_select_opts o{};
    o.mode = options.mode == sched::SelectionMode::text_semantics ? GD_MODE_TEXT : GD_MODE_LITERAL;
    o.objective = options.objective == sched::Objective::energy ? GD_OBJECTIVE_ENERGY : GD_OBJECTIVE_POWER;
    o.best_effort = options.best_effort_fallback ? 1 : 0;
    const int32_t budget =
        options.budget == sched::DeadlineBudget::full_deadline ? GD_BUDGET_FULL : GD_BUDGET_REMAINING;
    std::vector<gd_decision> dec(static_cast<std::size_t>(n));
    std::vector<int64_t> order(static_cast<std::size_t>(n));
    t_exec = &exec;
    t_jobs = &workload.jobs;
    t_catalog = &catalog;
    // The per-job tables live on the host here, so the O(C) scan beats
    // shipping them to the GPU for a frontier (gd_frontier pays off when the
    // tables are device-resident; scripts/edf_scale.py).
    check(gd_schedule_edf(jobs.data(), n, E.data(), T.data(), sm.data(), C, budget, &o, nullptr, exec_trampoline,
                          nullptr, dec.data(), order.data()));
    std::vector<sched::ScheduleDecision> out;
    out.reserve(static_cast<std::size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        const gd_decision& d = dec[static_cast<std::size_t>(k)];
        sched::ScheduleDecision sd;
        sd.job = workload.jobs[static_cast<std::size_t>(order[static_cast<std::size_t>(k)])];
        if (d.status == GD_SCHEDULED) {
            sd.status = sched::DecisionStatus::scheduled;
            sd.chosen_clock = catalog[static_cast<std::size_t>(d.clock_index)];
            sd.predicted_energy_ws = d.energy_ws;
            sd.predicted_time_s = d.time_s;
        } else {
            sd.status = sched::DecisionStatus::rejected_infeasible;
        }
        if (d.note == GD_NOTE_BEST_EFFORT) sd.note = "best_effort";
        if (d.note == GD_NOTE_MISSING_DATA) sd.note = "missing correlated data";
        out.push_back(std::move(sd));
    }
    return out;
}

}  // namespace gpudvfs::gpu
