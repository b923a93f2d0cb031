// integration/facade_test.cpp -- drop-in check of include/gpudvfs_b200/gpu_api.hpp.
//
// Runs the reference's production path (cli.cpp:400-481 shape: fit_gbt ->
// save/load model files -> select_k clusters -> make_model_predictor ->
// schedule_d_dvfs) twice on identical inputs -- once with the reference's own
// functions, once with the gpu:: drop-ins -- and requires identical
// decisions (job order, clock, predicted E/T bits, status, note) for every
// SchedulerOptions combination; then models::predict vs gpu::predict and the
// column-mismatch exception message.  Exit 0 = identical.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <string>

#include "gpudvfs/rng.hpp"
#include "gpudvfs/synthdata.hpp"
#include "gpudvfs_b200/gpu_api.hpp"

using namespace gpudvfs;

namespace {

int failures = 0;

void expect(bool ok, const std::string& what) {
    if (!ok) {
        ++failures;
        std::printf("MISMATCH: %s\n", what.c_str());
    }
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

bool same(const sched::ScheduleDecision& a, const sched::ScheduleDecision& b) {
    if (a.job.app_id != b.job.app_id || a.job.arrival_s != b.job.arrival_s) return false;
    if (a.status != b.status || a.note != b.note || a.chosen_clock != b.chosen_clock) return false;
    if (a.predicted_energy_ws.has_value() != b.predicted_energy_ws.has_value()) return false;
    if (a.predicted_energy_ws && !same_bits(*a.predicted_energy_ws, *b.predicted_energy_ws)) return false;
    if (a.predicted_time_s.has_value() != b.predicted_time_s.has_value()) return false;
    if (a.predicted_time_s && !same_bits(*a.predicted_time_s, *b.predicted_time_s)) return false;
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    // --bench [reps]: time the paper-scale production path (cold predictor +
    // schedule_d_dvfs, full_deadline) through the reference and through the
    // drop-in, `reps` times each, and print one JSON line (bench.py --config c1).
    int bench_reps = 0;
    if (argc > 1 && std::string(argv[1]) == "--bench") {
        bench_reps = argc > 2 ? std::atoi(argv[2]) : 5;
        argv += 2;
        argc -= 2;
    }
    const int iters = argc > 1 ? std::atoi(argv[1]) : 100;
    const int depth = argc > 2 ? std::atoi(argv[2]) : 10;
    const int n_jobs = argc > 3 ? std::atoi(argv[3]) : 100;
    // catalog profiling stride: 2 = every other clock (each candidate its own
    // nearest record -> general kernel); 25 = three records per app (clocks
    // share records -> (app, record) virtual apps on the fast path)
    const int stride = argc > 4 ? std::atoi(argv[4]) : 2;
    // 1: the drop-in runs through a gd_multi device group (select_devices)
    const bool multi = argc > 5 && std::atoi(argv[5]) != 0;
    if (multi) gpu::select_devices({0});
    const std::uint64_t seed = 7;
    const std::string dir = std::filesystem::temp_directory_path() / "gd_facade_test";
    std::filesystem::create_directories(dir);

    synth::SyntheticGpu p100 = synth::builtin_p100_gpu();
    Dataset catalog = p100.generate_dataset(synth::builtin_default_suite(), stride);
    ingest::EncodeResult enc_e = ingest::encode(catalog, catalog, TargetKind::energy, 1.0, seed);
    ingest::EncodeResult enc_t = ingest::encode(catalog, catalog, TargetKind::time, 1.0, seed);
    models::GBTConfig cfg{iters, depth, 0.1, 3.0, seed};
    models::FittedModel me = models::fit_gbt(enc_e.train, cfg);
    models::FittedModel mt = models::fit_gbt(enc_t.train, cfg);
    models::save_model_file(me, dir + "/e.txt");
    models::save_model_file(mt, dir + "/t.txt");
    me = models::load_model_file(dir + "/e.txt");
    mt = models::load_model_file(dir + "/t.txt");
    cluster::PointMatrix points = cluster::default_clock_points(catalog);
    cluster::KMeansModel clusters = cluster::select_k(points, 1, 9, seed).best_model;

    synth::ArchetypeSuite queries;
    for (int i = 0; i < n_jobs; ++i) {
        SplitMix64 r(seed * 31 + static_cast<std::uint64_t>(i));
        synth::AppArchetype a;
        a.app_id = "q" + std::to_string(1000 + i);
        a.compute_work = r.uniform(420.0, 5300.0);
        a.memory_work = r.uniform(70.0, 1950.0);
        a.stall_s = r.uniform(0.10, 1.40);
        a.power_coeff_core = r.uniform(0.034, 0.105);
        a.power_coeff_mem = r.uniform(0.007, 0.058);
        a.noise_seed = static_cast<std::uint64_t>(i) + 1;
        queries.apps.push_back(a);
    }
    std::vector<ProfileRecord> defaults;
    for (const auto& a : queries.apps) defaults.push_back(p100.profile(a, p100.device().default_clock));
    sched::WorkloadGenConfig gen;
    gen.seed = seed;
    Workload workload = sched::generate_workload(defaults, p100.device(), gen);
    // Duplicate app_ids whose default profiles differ: the reference's
    // predictor caches the FIRST PROCESSED job's correlation per app_id
    // (scheduler.cpp:316-327), which the drop-in must reproduce.
    {
        std::vector<Job> jobs = workload.jobs;
        const std::size_t n0 = jobs.size();
        for (std::size_t i = 0; i + n0 / 2 < n0 && i < n0 / 4; ++i) {
            Job d = jobs[i + n0 / 2];
            d.app_id = jobs[i].app_id;
            d.arrival_s = jobs[i].arrival_s + 0.25 * static_cast<double>(i % 3);
            jobs.push_back(d);
        }
        workload = make_workload(std::move(jobs), p100.device());
    }
    sched::ExecutionTimeSource exec = sched::make_truth_exec(queries, p100);

    if (bench_reps > 0) {
        sched::SchedulerOptions o;
        o.budget = sched::DeadlineBudget::full_deadline;
        std::vector<double> ref_ms, gpu_ms;
        bool identical = true;
        int scheduled = 0;
        for (int r = 0; r < bench_reps + 1; ++r) {  // the first repetition warms up
            auto t0 = std::chrono::steady_clock::now();
            sched::ClockPredictor rp =
                sched::make_model_predictor(me, enc_e.metadata, mt, enc_t.metadata, catalog, clusters);
            auto want = sched::schedule_d_dvfs(workload, rp, exec, o);
            auto t1 = std::chrono::steady_clock::now();
            sched::ClockPredictor gp =
                gpu::make_model_predictor(me, enc_e.metadata, mt, enc_t.metadata, catalog, clusters);
            auto got = gpu::schedule_d_dvfs(workload, gp, exec, o);
            auto t2 = std::chrono::steady_clock::now();
            identical = identical && want.size() == got.size();
            scheduled = 0;
            for (std::size_t k = 0; k < want.size() && k < got.size(); ++k) {
                identical = identical && same(want[k], got[k]);
                scheduled += got[k].status == sched::DecisionStatus::scheduled;
            }
            if (r == 0) continue;
            ref_ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
            gpu_ms.push_back(std::chrono::duration<double, std::milli>(t2 - t1).count());
        }
        std::sort(ref_ms.begin(), ref_ms.end());
        std::sort(gpu_ms.begin(), gpu_ms.end());
        std::printf("{\"jobs\": %zu, \"clocks\": %zu, \"catalog_records\": %zu, \"trees\": %d, \"depth\": %d, "
                    "\"reps\": %d, \"reference_ms_median\": %.4f, \"dropin_ms_median\": %.4f, "
                    "\"reference_ms_min\": %.4f, \"dropin_ms_min\": %.4f, \"scheduled\": %d, "
                    "\"decisions_identical\": %s}\n",
                    workload.jobs.size(), clock_catalog(catalog.device).size(), catalog.records.size(), iters, depth,
                    bench_reps, ref_ms[ref_ms.size() / 2], gpu_ms[gpu_ms.size() / 2], ref_ms.front(), gpu_ms.front(),
                    scheduled, identical ? "true" : "false");
        return identical ? 0 : 1;
    }

    sched::ClockPredictor ref_pred = sched::make_model_predictor(me, enc_e.metadata, mt, enc_t.metadata, catalog,
                                                                 clusters);
    sched::ClockPredictor gpu_pred = gpu::make_model_predictor(me, enc_e.metadata, mt, enc_t.metadata, catalog,
                                                               clusters);
    int combos = 0, scheduled = 0;
    for (int mode = 0; mode < 2; ++mode) {
        for (int budget = 0; budget < 2; ++budget) {
            for (int obj = 0; obj < 2; ++obj) {
                for (int be = 0; be < 2; ++be) {
                    sched::SchedulerOptions o;
                    o.mode = mode ? sched::SelectionMode::literal_pseudocode : sched::SelectionMode::text_semantics;
                    o.budget = budget ? sched::DeadlineBudget::full_deadline : sched::DeadlineBudget::remaining_time;
                    o.objective = obj ? sched::Objective::power : sched::Objective::energy;
                    o.best_effort_fallback = be != 0;
                    auto want = sched::schedule_d_dvfs(workload, ref_pred, exec, o);
                    auto got = gpu::schedule_d_dvfs(workload, gpu_pred, exec, o);
                    expect(want.size() == got.size(), "decision count");
                    for (std::size_t k = 0; k < want.size() && k < got.size(); ++k) {
                        expect(same(want[k], got[k]), "combo " + std::to_string(combos) + " decision " +
                                                          std::to_string(k) + " (" + want[k].job.app_id + ")");
                        scheduled += want[k].status == sched::DecisionStatus::scheduled;
                    }
                    // also the GPU path with the reference's own predictor (generic seam)
                    auto mixed = gpu::schedule_d_dvfs(workload, ref_pred, exec, o);
                    for (std::size_t k = 0; k < want.size() && k < mixed.size(); ++k) {
                        expect(same(want[k], mixed[k]), "mixed combo " + std::to_string(combos));
                    }
                    ++combos;
                }
            }
        }
    }
    // Perfect predictor (acceptance #1 seam, scheduler.cpp:283-291).
    synth::ArchetypeSuite suite = synth::builtin_default_suite();
    sched::ClockPredictor truth = sched::make_truth_predictor(queries, p100);
    sched::SchedulerOptions full;
    full.budget = sched::DeadlineBudget::full_deadline;
    auto tw = sched::schedule_d_dvfs(workload, truth, exec, full);
    auto tg = gpu::schedule_d_dvfs(workload, truth, exec, full);
    for (std::size_t k = 0; k < tw.size(); ++k) expect(same(tw[k], tg[k]), "truth decision " + std::to_string(k));

    // models::predict drop-in on the encoded catalog (K1).
    for (const auto* pair : {&enc_e, &enc_t}) {
        const models::FittedModel& m = pair == &enc_e ? me : mt;
        auto want = models::predict(m, pair->train);
        auto got = gpu::predict(m, pair->train);
        expect(want.size() == got.size(), "predict size");
        for (std::size_t i = 0; i < want.size(); ++i) {
            if (!same_bits(want[i], got[i])) {
                expect(false, "predict row " + std::to_string(i));
                break;
            }
        }
    }
    ingest::EncodedMatrix wrong = enc_e.train;
    wrong.columns[3] = "bogus";
    std::string want_msg, got_msg;
    try {
        models::predict(me, wrong);
    } catch (const std::invalid_argument& e) {
        want_msg = e.what();
    }
    try {
        gpu::predict(me, wrong);
    } catch (const std::invalid_argument& e) {
        got_msg = e.what();
    }
    expect(!want_msg.empty() && want_msg == got_msg, "column-mismatch message: '" + got_msg + "'");

    // Wall time of one cold batch (fresh predictors: correlation, row
    // construction, encoding, prediction, EDF) -- reference vs drop-in.
    {
        sched::SchedulerOptions o;
        o.budget = sched::DeadlineBudget::full_deadline;
        auto t0 = std::chrono::steady_clock::now();
        sched::ClockPredictor rp =
            sched::make_model_predictor(me, enc_e.metadata, mt, enc_t.metadata, catalog, clusters);
        auto want = sched::schedule_d_dvfs(workload, rp, exec, o);
        auto t1 = std::chrono::steady_clock::now();
        sched::ClockPredictor gp = gpu::make_model_predictor(me, enc_e.metadata, mt, enc_t.metadata, catalog, clusters);
        auto got = gpu::schedule_d_dvfs(workload, gp, exec, o);
        auto t2 = std::chrono::steady_clock::now();
        for (std::size_t k = 0; k < want.size() && k < got.size(); ++k) expect(same(want[k], got[k]), "timed batch");
        std::printf("cold batch of %zu jobs: reference %.2f ms, drop-in %.2f ms (incl. model upload)\n",
                    workload.jobs.size(), std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count());
    }

    std::printf("%s: %d option combos x %zu jobs, %d scheduled decisions compared; %d mismatches\n",
                failures ? "FACADE FAIL" : "FACADE OK", combos, workload.jobs.size(), scheduled, failures);
    return failures ? 1 : 0;
}
