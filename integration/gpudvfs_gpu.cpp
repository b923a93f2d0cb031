// integration/gpudvfs_gpu.cpp -- implementation of include/gpudvfs_b200/gpu_api.hpp.
//
// This is the reference-side binding: it is compiled against the reference's
// own headers and links into the reference's library, and it reaches the
// GPU only through the C ABI (gdvfs.h).  Everything per (app x clock) runs on
// the device.  The per-job host steps are restructured around
// what they depend on:
//   * correlation (clustering.cpp:346-411) recomputes the catalog's
//     default-clock points, their cluster labels and default times on every
//     call -- here they are computed once per predictor (CatalogIndex) and a
//     query costs one k-means assignment plus a scan of the catalog apps;
//   * a job's candidate rows (scheduler.cpp:330-359) depend only on the
//     catalog app it correlates to, so the nearest-record substitution, the
//     encoding and the GPU evaluation run once per distinct MATCHED app;
//   * the encoding (apply_encoding, ingest.cpp:401-439: per record and
//     column, a name lookup plus a std::map lookup and a division per
//     categorical level) becomes an EncodingPlan built once per predictor:
//     per column either "numeric" or a per-level value table for BOTH
//     targets, applied once per distinct matched record.
// The grid call takes the fast partial-evaluation path whenever a matched
// app's candidates use few distinct records (each (app, record) group is a
// virtual app whose clock columns the kernel overrides), and the general
// per-candidate kernel otherwise (every clock its own profiled record, as in
// the paper-scale catalog).
#include "gpudvfs_b200/gpu_api.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace gpudvfs::gpu {
namespace {

thread_local std::vector<int> t_devices{0};
thread_local bool t_group = false;  // select_devices: predictors run through a gd_multi group

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

// One gd_ctx per (host thread, device), alive for the thread: switching
// devices never destroys a context, and models (which carry only their
// device) stay valid for every context of their device.
gd_ctx* context_for(int device) {
    struct Holder {
        gd_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx) gd_ctx_destroy(ctx);
        }
    };
    thread_local std::map<int, Holder> ctxs;
    Holder& h = ctxs[device];
    if (!h.ctx) check(gd_ctx_create(device, &h.ctx));
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

// A FittedModel flattened to the packer's arrays (also the predict cache's
// identity: two models with equal flat forms predict identically).
struct FlatModel {
    int32_t kind = 0, target = 0, n_cols = 0;
    double base = 0.0, lr = 0.0;
    std::vector<int64_t> off;
    std::vector<int32_t> feat, left, right;
    std::vector<double> thr, leaf;

    static FlatModel of(const models::FittedModel& fm) {
        FlatModel f;
        f.n_cols = static_cast<int32_t>(fm.columns.size());
        f.target = fm.target == TargetKind::energy ? GD_TARGET_ENERGY : GD_TARGET_TIME;
        if (fm.kind == models::ModelKind::gbt) {
            f.kind = GD_KIND_GBT;
            f.base = fm.gbt.base_prediction;
            f.lr = fm.gbt.learning_rate;
            f.off.push_back(0);
            for (const auto& tree : fm.gbt.trees) {
                for (const auto& n : tree.nodes) {
                    f.feat.push_back(n.feature);
                    f.thr.push_back(n.threshold);
                    f.left.push_back(n.left);
                    f.right.push_back(n.right);
                    f.leaf.push_back(n.leaf_value);
                }
                f.off.push_back(static_cast<int64_t>(f.feat.size()));
            }
        } else {
            f.kind = fm.kind == models::ModelKind::ols ? GD_KIND_OLS : GD_KIND_LASSO;
            f.base = fm.linear.intercept;
            f.thr = fm.linear.coefficients;
        }
        return f;
    }

    template <class T>
    static bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
        return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
    }
    bool operator==(const FlatModel& o) const {
        return kind == o.kind && target == o.target && n_cols == o.n_cols &&
               std::memcmp(&base, &o.base, sizeof base) == 0 && std::memcmp(&lr, &o.lr, sizeof lr) == 0 &&
               same_bits(off, o.off) && same_bits(feat, o.feat) && same_bits(left, o.left) &&
               same_bits(right, o.right) && same_bits(thr, o.thr) && same_bits(leaf, o.leaf);
    }

    std::unique_ptr<ModelHandle> upload(gd_ctx* ctx) const {
        auto h = std::make_unique<ModelHandle>();
        if (kind == GD_KIND_GBT) {
            gd_forest_view v{static_cast<int32_t>(off.size() - 1), off.data(), feat.data(), thr.data(),
                             left.data(), right.data(), leaf.data()};
            check(gd_model_upload_gbt(ctx, &v, base, lr, n_cols, target, &h->m));
        } else {
            check(gd_model_upload_linear(ctx, thr.data(), n_cols, base, kind, target, &h->m));
        }
        return h;
    }
};

std::unique_ptr<ModelHandle> upload(const models::FittedModel& fm, gd_ctx* ctx) {
    return FlatModel::of(fm).upload(ctx);
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

// apply_encoding (ingest.cpp:401-439) precomputed: per encoded column,
// numeric (copied from the record) or categorical with the encoded value of
// every known level, computed with the reference's expression
// (sum + w * mean) / (count + w); unseen levels encode as the global mean.
struct EncodingPlan {
    struct Col {
        std::string name;
        bool categorical = false;  // decided per record: numeric features win (ingest.cpp:418-422)
        std::map<std::string, double> level_value;
        double unseen = 0.0;
    };
    std::vector<Col> cols;

    static EncodingPlan of(const ingest::EncodingMetadata& md) {
        EncodingPlan p;
        for (const auto& name : md.columns) {
            Col c;
            c.name = name;
            auto st = md.level_stats.find(name);
            if (st != md.level_stats.end()) {
                c.categorical = true;
                for (const auto& [level, s] : st->second) {
                    c.level_value[level] = (s.target_sum + md.prior_weight * md.global_target_mean) /
                                           (static_cast<double>(s.count) + md.prior_weight);
                }
            }
            c.unseen = md.global_target_mean;
            p.cols.push_back(std::move(c));
        }
        return p;
    }

    // One encoded row; throws apply_encoding's invalid_argument for a missing
    // feature (and std::out_of_range, like level_stats.at, for a categorical
    // value in a column the metadata never encoded).
    void row(const ProfileRecord& r, double* out) const {
        for (std::size_t c = 0; c < cols.size(); ++c) {
            const Col& col = cols[c];
            auto num = r.features.numeric.find(col.name);
            if (num != r.features.numeric.end()) {
                out[c] = num->second;
                continue;
            }
            auto cat = r.features.categorical.find(col.name);
            if (cat == r.features.categorical.end()) {
                throw std::invalid_argument("apply_encoding: record lacks feature '" + col.name + "'");
            }
            if (!col.categorical) throw std::out_of_range("apply_encoding: no level statistics for '" + col.name + "'");
            auto it = col.level_value.find(to_string(cat->second));
            out[c] = it == col.level_value.end() ? col.unseen : it->second;
        }
    }
};

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

// Per matched catalog app: E and T of every catalog clock, catalog order.
struct AppTable {
    std::vector<double> e, t;
};
using TablePtr = std::shared_ptr<const AppTable>;

struct MultiHolder {
    gd_multi* m = nullptr;
    ~MultiHolder() {
        if (m) gd_multi_destroy(m);
    }
};

// Matched apps whose candidates use at most this many distinct records run
// as (app, record) virtual apps on the partial-evaluation path; more (e.g.
// every clock profiled) go to the general per-candidate kernel.
constexpr std::size_t kMaxFastRecords = 4;

// ---------------------------------------------------------------------------
// The GPU-backed ClockPredictor (replaces ModelPredictorState,
// scheduler.cpp:304-371).
// ---------------------------------------------------------------------------
struct GpuPredictorState {
    models::FittedModel energy_model, time_model;
    ingest::EncodingMetadata energy_encoding, time_encoding;
    EncodingPlan plan_e, plan_t;
    Dataset catalog;
    cluster::KMeansModel clusters;
    CatalogIndex index;
    std::vector<int> devices;
    std::unique_ptr<MultiHolder> multi;                       // devices.size() > 1
    std::vector<std::unique_ptr<ModelHandle>> ge, gt;         // one per device
    std::vector<ClockSet> clocks;
    std::map<ClockSet, int32_t> clock_index;
    std::vector<int32_t> sm, mem;
    std::map<std::string, TablePtr> cache;  // per job app_id (the reference's cache)
    std::set<std::string> failed;           // per job app_id
    std::map<std::string, TablePtr> by_match;  // per matched catalog app
    std::set<std::string> match_failed;
    bool columns_ok = true;
    bool shared_rows = true;  // both encodings have the same columns: one row set + time categoricals

    // The matched app of `job`'s own default profile, or "" when correlate throws.
    std::string match_of(const Job& job) const {
        try {
            return index.matched_app(clusters, catalog, job.default_profile);
        } catch (const std::exception&) {
            return std::string();
        }
    }

    // Evaluate every not-yet-seen matched app in `matched` with batched launches.
    void ensure(const std::vector<std::string>& matched) {
        std::vector<std::string> todo;
        std::set<std::string> queued;
        for (const auto& m : matched) {
            if (m.empty() || by_match.count(m) || match_failed.count(m) || queued.count(m)) continue;
            queued.insert(m);
            auto it = index.records_of.find(m);
            if (it == index.records_of.end() || it->second.empty()) {
                match_failed.insert(m);  // "correlated app has no records" (scheduler.cpp:336)
                continue;
            }
            todo.push_back(m);
        }
        if (!columns_ok) {
            for (const auto& m : todo) match_failed.insert(m);
            return;
        }
        if (todo.empty()) return;
        try {
            if (shared_rows) evaluate(todo);
            else evaluate_separate(todo);
        } catch (const std::exception&) {
            // build() failures reject the job (scheduler.cpp:318-323): every
            // app of the failed batch answers nullopt, as the reference would.
            for (const auto& m : todo) {
                if (!by_match.count(m)) match_failed.insert(m);
            }
        }
    }

    // The table a job gets when its own profile decides (nullptr: rejected).
    TablePtr table_for_match(const std::string& m) const {
        if (m.empty()) return nullptr;
        auto it = by_match.find(m);
        return it == by_match.end() ? nullptr : it->second;
    }

    // Lazy path of the ClockPredictor: first query of an app_id decides.
    TablePtr lookup(const Job& job) {
        if (failed.count(job.app_id)) return nullptr;
        auto hit = cache.find(job.app_id);
        if (hit != cache.end()) return hit->second;
        const std::string m = match_of(job);
        ensure({m});
        TablePtr t = table_for_match(m);
        if (t) cache[job.app_id] = t;
        else failed.insert(job.app_id);
        return t;
    }

    // scheduler.cpp:338-359: the nearest profiled record of app `recs` for each catalog clock.
    std::vector<std::size_t> nearest_records(const std::vector<std::size_t>& recs) const {
        std::vector<std::size_t> out;
        out.reserve(clocks.size());
        for (const ClockSet& clock : clocks) {
            std::size_t nearest = recs.front();
            auto dist = [&](std::size_t i) {
                const ClockSet& c = catalog.records[i].clock;
                return std::make_pair(std::abs(c.mem_clock_mhz - clock.mem_clock_mhz),
                                      std::abs(c.sm_clock_mhz - clock.sm_clock_mhz));
            };
            for (std::size_t i : recs) {
                if (dist(i) < dist(nearest)) nearest = i;
            }
            out.push_back(nearest);
        }
        return out;
    }

    // One (virtual) app batch through the grid call: per-device sharded when
    // several devices are selected.  rows / cat_t hold one row per record.
    void grid_call(std::vector<double>& rows, std::vector<double>& cat_t, std::vector<int32_t>& cat_cols,
                   const std::vector<int32_t>* rec_of_clock, int64_t n_apps, int F, std::vector<double>& e,
                   std::vector<double>& t) {
        const int32_t C = static_cast<int32_t>(clocks.size());
        std::vector<double> budgets(static_cast<std::size_t>(n_apps), 0.0);
        std::vector<gd_decision> dec(static_cast<std::size_t>(n_apps));
        e.assign(static_cast<std::size_t>(n_apps) * C, 0.0);
        t.assign(static_cast<std::size_t>(n_apps) * C, 0.0);
        gd_grid g{};
        g.rows = rows.data();
        g.n_records = static_cast<int64_t>(rows.size() / static_cast<std::size_t>(F));
        g.n_cols = F;
        g.n_cat = static_cast<int32_t>(cat_cols.size());
        g.cat_t = cat_t.data();
        g.cat_cols = cat_cols.data();
        g.rec_of_clock = rec_of_clock ? rec_of_clock->data() : nullptr;
        g.n_apps = n_apps;
        g.sm_clock = sm.data();
        g.mem_clock = mem.data();
        g.n_clocks = C;
        g.sm_col = column_of(energy_encoding.columns, "sm_clock");
        g.mem_col = column_of(energy_encoding.columns, "mem_clock");
        g.budgets = budgets.data();
        gd_select_opts o{GD_MODE_TEXT, GD_OBJECTIVE_ENERGY, 0, 0};
        if (multi) {
            std::vector<gd_model*> me, mt;
            for (auto& h : ge) me.push_back(h->m);
            for (auto& h : gt) mt.push_back(h->m);
            check(gd_multi_grid_select(multi->m, me.data(), mt.data(), &g, &o, dec.data(), e.data(), t.data()));
        } else {
            check(gd_grid_select(context_for(devices[0]), ge[0]->m, gt[0]->m, &g, &o, dec.data(), e.data(), t.data()));
        }
    }

    void evaluate(const std::vector<std::string>& todo) {
        const int F = static_cast<int>(energy_encoding.columns.size());
        const int32_t C = static_cast<int32_t>(clocks.size());
        std::vector<int32_t> cat_cols;
        for (const auto& name : energy_encoding.categorical_columns) cat_cols.push_back(column_of(energy_encoding.columns, name));
        // Encoded rows of each distinct matched record, shared by both
        // batches (energy encoding + the time encoding's categorical values).
        struct App {
            std::string id;
            std::vector<std::size_t> rec_of_clock;  // catalog record per clock
            std::vector<std::size_t> distinct;      // its distinct records, first-use order
        };
        std::vector<App> apps;
        std::vector<double> erow(static_cast<std::size_t>(F)), trow(static_cast<std::size_t>(F));
        std::map<std::size_t, std::pair<std::vector<double>, std::vector<double>>> enc;  // record -> (row, cat_t)
        for (const auto& m : todo) {
            App a;
            a.id = m;
            a.rec_of_clock = nearest_records(index.records_of.at(m));
            try {
                for (std::size_t r : a.rec_of_clock) {
                    if (std::find(a.distinct.begin(), a.distinct.end(), r) == a.distinct.end()) a.distinct.push_back(r);
                    if (enc.count(r)) continue;
                    // The clock columns are overridden per candidate by the kernel.
                    plan_e.row(catalog.records[r], erow.data());
                    plan_t.row(catalog.records[r], trow.data());
                    std::vector<double> ct;
                    for (int32_t c : cat_cols) ct.push_back(trow[static_cast<std::size_t>(c)]);
                    enc[r] = {erow, std::move(ct)};
                }
                apps.push_back(std::move(a));
            } catch (const std::exception&) {
                match_failed.insert(m);  // build() threw: every job of this match is rejected
            }
        }
        // Fast batch: one virtual app per (app, distinct record); general
        // batch: the app's C candidates each read their own record.
        std::vector<double> f_rows, f_cat, g_rows, g_cat;
        std::vector<int32_t> g_rec;
        std::vector<std::pair<std::size_t, std::size_t>> f_of;  // virtual app -> (app, record)
        std::vector<std::size_t> g_apps;
        std::map<std::size_t, int32_t> g_local;  // record -> row in g_rows
        for (std::size_t i = 0; i < apps.size(); ++i) {
            const App& a = apps[i];
            if (a.distinct.size() <= kMaxFastRecords) {
                for (std::size_t r : a.distinct) {
                    const auto& rc = enc.at(r);
                    f_rows.insert(f_rows.end(), rc.first.begin(), rc.first.end());
                    f_cat.insert(f_cat.end(), rc.second.begin(), rc.second.end());
                    f_of.emplace_back(i, r);
                }
            } else {
                for (std::size_t r : a.rec_of_clock) {
                    auto it = g_local.find(r);
                    if (it == g_local.end()) {
                        const auto& rc = enc.at(r);
                        it = g_local.emplace(r, static_cast<int32_t>(g_rows.size() / static_cast<std::size_t>(F))).first;
                        g_rows.insert(g_rows.end(), rc.first.begin(), rc.first.end());
                        g_cat.insert(g_cat.end(), rc.second.begin(), rc.second.end());
                    }
                    g_rec.push_back(it->second);
                }
                g_apps.push_back(i);
            }
        }
        std::vector<AppTable> tables(apps.size());
        for (auto& tb : tables) {
            tb.e.assign(static_cast<std::size_t>(C), 0.0);
            tb.t.assign(static_cast<std::size_t>(C), 0.0);
        }
        std::vector<double> e, t;
        if (!f_of.empty()) {
            grid_call(f_rows, f_cat, cat_cols, nullptr, static_cast<int64_t>(f_of.size()), F, e, t);
            for (std::size_t v = 0; v < f_of.size(); ++v) {
                const auto [i, r] = f_of[v];
                for (int32_t c = 0; c < C; ++c) {
                    if (apps[i].rec_of_clock[static_cast<std::size_t>(c)] != r) continue;
                    tables[i].e[static_cast<std::size_t>(c)] = e[v * C + static_cast<std::size_t>(c)];
                    tables[i].t[static_cast<std::size_t>(c)] = t[v * C + static_cast<std::size_t>(c)];
                }
            }
        }
        if (!g_apps.empty()) {
            grid_call(g_rows, g_cat, cat_cols, &g_rec, static_cast<int64_t>(g_apps.size()), F, e, t);
            for (std::size_t k = 0; k < g_apps.size(); ++k) {
                AppTable& tb = tables[g_apps[k]];
                std::copy(e.begin() + static_cast<std::ptrdiff_t>(k * C), e.begin() + static_cast<std::ptrdiff_t>((k + 1) * C),
                          tb.e.begin());
                std::copy(t.begin() + static_cast<std::ptrdiff_t>(k * C), t.begin() + static_cast<std::ptrdiff_t>((k + 1) * C),
                          tb.t.begin());
            }
        }
        for (std::size_t i = 0; i < apps.size(); ++i) by_match[apps[i].id] = std::make_shared<AppTable>(std::move(tables[i]));
    }

    // Encodings with different column sets (allowed by the reference): no
    // shared row layout, so each model predicts over its own materialised
    // candidate rows with K1 (gd_predict_rows) -- still one batched launch
    // per model.
    void evaluate_separate(const std::vector<std::string>& todo) {
        const int32_t C = static_cast<int32_t>(clocks.size());
        std::vector<std::string> ok;
        std::vector<double> er, tr;
        for (const auto& m : todo) {
            const std::vector<std::size_t> rec = nearest_records(index.records_of.at(m));
            std::vector<ProfileRecord> rows;
            for (std::size_t c = 0; c < clocks.size(); ++c) {  // scheduler.cpp:351-357
                ProfileRecord row = catalog.records[rec[c]];
                row.clock = clocks[c];
                if (row.features.numeric.count("sm_clock")) row.features.numeric["sm_clock"] = clocks[c].sm_clock_mhz;
                if (row.features.numeric.count("mem_clock")) row.features.numeric["mem_clock"] = clocks[c].mem_clock_mhz;
                rows.push_back(std::move(row));
            }
            try {
                std::vector<double> e1(plan_e.cols.size()), t1(plan_t.cols.size()), es, ts;
                for (const auto& r : rows) {
                    plan_e.row(r, e1.data());
                    plan_t.row(r, t1.data());
                    es.insert(es.end(), e1.begin(), e1.end());
                    ts.insert(ts.end(), t1.begin(), t1.end());
                }
                er.insert(er.end(), es.begin(), es.end());
                tr.insert(tr.end(), ts.begin(), ts.end());
                ok.push_back(m);
            } catch (const std::exception&) {
                match_failed.insert(m);
            }
        }
        if (ok.empty()) return;
        const int64_t n = static_cast<int64_t>(ok.size()) * C;
        std::vector<double> e(static_cast<std::size_t>(n)), t(static_cast<std::size_t>(n));
        gd_ctx* ctx = context_for(devices[0]);
        check(gd_predict_rows(ctx, ge[0]->m, er.data(), n, static_cast<int32_t>(plan_e.cols.size()), e.data(), nullptr));
        check(gd_predict_rows(ctx, gt[0]->m, tr.data(), n, static_cast<int32_t>(plan_t.cols.size()), t.data(), nullptr));
        for (std::size_t i = 0; i < ok.size(); ++i) {
            auto tb = std::make_shared<AppTable>();
            tb->e.assign(e.begin() + static_cast<std::ptrdiff_t>(i * C), e.begin() + static_cast<std::ptrdiff_t>((i + 1) * C));
            tb->t.assign(t.begin() + static_cast<std::ptrdiff_t>(i * C), t.begin() + static_cast<std::ptrdiff_t>((i + 1) * C));
            by_match[ok[i]] = std::move(tb);
        }
    }
};

struct GpuPredictorFn {
    std::shared_ptr<GpuPredictorState> state;
    std::optional<sched::ClockPrediction> operator()(const Job& job, const ClockSet& clock) const {
        TablePtr t = state->lookup(job);
        if (!t) return std::nullopt;
        auto it = state->clock_index.find(clock);
        if (it == state->clock_index.end()) return std::nullopt;
        const auto c = static_cast<std::size_t>(it->second);
        return sched::ClockPrediction{t->e[c], t->t[c]};
    }
};

thread_local const sched::ExecutionTimeSource* t_exec = nullptr;
thread_local const std::vector<Job>* t_jobs = nullptr;
thread_local const std::vector<ClockSet>* t_catalog = nullptr;

// The last (clock, execution time) the source returned per job: the
// decider fixpoint below re-runs the EDF loop, and a job keeping its clock
// does not query the source again (the reference queries it once per
// scheduled job; a pure ExecutionTimeSource gives identical values).
thread_local std::vector<std::pair<int32_t, double>> t_exec_memo;

double exec_trampoline(void*, int64_t job, int32_t clock_index) {
    auto& m = t_exec_memo[static_cast<std::size_t>(job)];
    if (m.first == clock_index) return m.second;
    const double v =
        (*t_exec)((*t_jobs)[static_cast<std::size_t>(job)], (*t_catalog)[static_cast<std::size_t>(clock_index)]);
    m = {clock_index, v};
    return v;
}

}  // namespace

void select_device(int device) {
    t_devices.assign(1, device);
    t_group = false;
}

void select_devices(const std::vector<int>& devices) {
    if (devices.empty()) throw std::invalid_argument("select_devices: empty device list");
    t_devices = devices;
    t_group = true;
}

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
    // Packed device models are cached per (thread, device): a repeated
    // predict with an equal model skips the pack + upload.
    struct Cached {
        int device;
        FlatModel flat;
        std::shared_ptr<ModelHandle> h;
    };
    thread_local std::vector<Cached> cache;
    const int device = t_devices[0];
    FlatModel fm = FlatModel::of(model);
    std::shared_ptr<ModelHandle> h;
    for (std::size_t i = 0; i < cache.size(); ++i) {
        if (cache[i].device == device && cache[i].flat == fm) {
            h = cache[i].h;
            std::rotate(cache.begin(), cache.begin() + static_cast<std::ptrdiff_t>(i),
                        cache.begin() + static_cast<std::ptrdiff_t>(i) + 1);  // most recent first
            break;
        }
    }
    gd_ctx* ctx = context_for(device);
    if (!h) {
        h = fm.upload(ctx);
        cache.insert(cache.begin(), Cached{device, std::move(fm), h});
        if (cache.size() > 4) cache.pop_back();
    }
    check(gd_predict_rows(ctx, h->m, flat.data(), static_cast<int64_t>(rows.rows.size()), F, out.data(), nullptr));
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
    s->plan_e = EncodingPlan::of(s->energy_encoding);
    s->plan_t = EncodingPlan::of(s->time_encoding);
    s->shared_rows = s->energy_encoding.columns == s->time_encoding.columns;
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
    s->devices = t_devices;
    if (t_group) {
        s->multi = std::make_unique<MultiHolder>();
        check(gd_multi_create(s->devices.data(), static_cast<int32_t>(s->devices.size()), &s->multi->m));
        for (const auto* fm : {&s->energy_model, &s->time_model}) {
            auto host = FlatModel::of(*fm).upload(nullptr);  // packed + validated once, replicated per device
            std::vector<gd_model*> rep(s->devices.size(), nullptr);
            check(gd_multi_model_replicate(s->multi->m, host->m, rep.data()));
            auto& dst = fm == &s->energy_model ? s->ge : s->gt;
            for (gd_model* r : rep) {
                auto h = std::make_unique<ModelHandle>();
                h->m = r;
                dst.push_back(std::move(h));
            }
        }
    } else {
        gd_ctx* ctx = context_for(s->devices[0]);
        s->ge.push_back(upload(s->energy_model, ctx));
        s->gt.push_back(upload(s->time_model, ctx));
    }
    s->clocks = clock_catalog(s->catalog.device);
    for (std::size_t c = 0; c < s->clocks.size(); ++c) {
        s->sm.push_back(s->clocks[c].sm_clock_mhz);
        s->mem.push_back(s->clocks[c].mem_clock_mhz);
        s->clock_index.emplace(s->clocks[c], static_cast<int32_t>(c));
    }
    return GpuPredictorFn{s};
}

std::vector<sched::ScheduleDecision> schedule_d_dvfs(const Workload& workload, const sched::ClockPredictor& predictor,
                                                     const sched::ExecutionTimeSource& exec,
                                                     const sched::SchedulerOptions& options) {
    const std::vector<ClockSet> catalog = clock_catalog(workload.device);
    const int32_t C = static_cast<int32_t>(catalog.size());
    const int64_t n = static_cast<int64_t>(workload.jobs.size());
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
    std::vector<double> E(static_cast<std::size_t>(n) * C), T(static_cast<std::size_t>(n) * C);
    t_exec = &exec;
    t_jobs = &workload.jobs;
    t_catalog = &catalog;
    t_exec_memo.assign(static_cast<std::size_t>(n), {-1, 0.0});
    // The per-job tables live on the host here, so the O(C) scan beats
    // shipping them to the GPU for a frontier (gd_frontier pays off when the
    // tables are device-resident; scripts/edf_scale.py).
    auto run_edf = [&] {
        check(gd_schedule_edf(jobs.data(), n, E.data(), T.data(), sm.data(), C, budget, &o, nullptr, exec_trampoline,
                              nullptr, dec.data(), order.data()));
    };

    const GpuPredictorFn* fn = predictor.target<GpuPredictorFn>();
    if (fn && catalog == fn->state->clocks) {
        GpuPredictorState& st = *fn->state;
        // The reference fills its per-app_id cache lazily in EDF processing
        // order, from the FIRST processed job of each app_id
        // (scheduler.cpp:316-327 called from decide, :188-195).  Jobs of one
        // app_id usually correlate identically; where their profiles match
        // different catalog apps, the deciding job is found by fixpoint:
        // guess the first in arrival order, run the loop, re-run with the
        // first processed job until they agree.
        std::vector<std::string> match(static_cast<std::size_t>(n));
        std::map<std::string, std::vector<int64_t>> jobs_of;
        for (int64_t i = 0; i < n; ++i) {
            const Job& job = workload.jobs[static_cast<std::size_t>(i)];
            jobs_of[job.app_id].push_back(i);
            if (!st.cache.count(job.app_id) && !st.failed.count(job.app_id)) match[static_cast<std::size_t>(i)] = st.match_of(job);
        }
        st.ensure(match);  // one batched evaluation for every distinct match
        std::vector<int64_t> pend(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) pend[static_cast<std::size_t>(i)] = i;
        std::stable_sort(pend.begin(), pend.end(), [&](int64_t a, int64_t b) {  // run_edf_loop's pending order
            const Job& x = workload.jobs[static_cast<std::size_t>(a)];
            const Job& y = workload.jobs[static_cast<std::size_t>(b)];
            if (x.arrival_s != y.arrival_s) return x.arrival_s < y.arrival_s;
            return x.app_id < y.app_id;
        });
        std::map<std::string, int64_t> decider;  // app_id -> job whose profile decides (uncached apps)
        std::set<std::string> ambiguous;
        for (const auto& [app, js] : jobs_of) {
            if (st.cache.count(app) || st.failed.count(app)) continue;
            for (int64_t j : js) {
                if (match[static_cast<std::size_t>(j)] != match[static_cast<std::size_t>(js[0])]) ambiguous.insert(app);
            }
        }
        for (int64_t i : pend) decider.emplace(workload.jobs[static_cast<std::size_t>(i)].app_id, i);
        auto table_of = [&](const std::string& app) -> TablePtr {
            if (st.failed.count(app)) return nullptr;
            auto hit = st.cache.find(app);
            if (hit != st.cache.end()) return hit->second;
            return st.table_for_match(match[static_cast<std::size_t>(decider.at(app))]);
        };
        for (int pass = 0; pass < 16; ++pass) {
            for (int64_t i = 0; i < n; ++i) {
                const Job& job = workload.jobs[static_cast<std::size_t>(i)];
                TablePtr t = table_of(job.app_id);
                jobs[static_cast<std::size_t>(i)].app_index = t ? static_cast<int32_t>(i) : -1;
                if (t) {
                    std::memcpy(&E[static_cast<std::size_t>(i) * C], t->e.data(), sizeof(double) * C);
                    std::memcpy(&T[static_cast<std::size_t>(i) * C], t->t.data(), sizeof(double) * C);
                }
            }
            run_edf();
            bool stable = true;
            std::set<std::string> seen;
            for (int64_t k = 0; k < n; ++k) {
                const int64_t j = order[static_cast<std::size_t>(k)];
                const std::string& app = workload.jobs[static_cast<std::size_t>(j)].app_id;
                if (!seen.insert(app).second || !ambiguous.count(app)) continue;
                if (decider[app] != j) {
                    decider[app] = j;
                    stable = false;
                }
            }
            if (stable) break;
        }
        // Leave the predictor in the state the reference's would be in.
        for (const auto& [app, j] : decider) {
            if (st.cache.count(app) || st.failed.count(app)) continue;  // decided by an earlier query
            TablePtr t = st.table_for_match(match[static_cast<std::size_t>(j)]);
            if (t) st.cache[app] = t;
            else st.failed.insert(app);
        }
    } else {
        // Any other ClockPredictor: per-job candidate tables through the
        // callback (scheduler.cpp:193-201).
        for (int64_t i = 0; i < n; ++i) {
            const Job& job = workload.jobs[static_cast<std::size_t>(i)];
            for (int32_t c = 0; c < C; ++c) {
                auto p = predictor(job, catalog[static_cast<std::size_t>(c)]);
                if (!p) {
                    jobs[static_cast<std::size_t>(i)].app_index = -1;
                    break;
                }
                E[static_cast<std::size_t>(i * C + c)] = p->energy_ws;
                T[static_cast<std::size_t>(i * C + c)] = p->time_s;
            }
        }
        run_edf();
    }
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
