// gpudvfs_b200/gpu_api.hpp -- C++ drop-in for the reference's hot-path API.
//
// Same signatures and semantics as the reference (paths relative to
// /root/reference/proj), backed by the sm_100a kernels through the C ABI in
// gdvfs.h.  Compile it INTO the reference's library (it includes the
// reference's own headers, include/gpudvfs/*.hpp) and swap the calls:
//
//   models::predict(model, rows)                 (models.hpp:94)
//     -> gpu::predict(model, rows)
//   sched::make_model_predictor(e, ee, t, te, catalog, clusters)
//                                                (scheduler.hpp:112-115)
//     -> gpu::make_model_predictor(...)
//   sched::schedule_d_dvfs(workload, predictor, exec, options)
//                                                (scheduler.hpp:83-85)
//     -> gpu::schedule_d_dvfs(...)
//
// Exceptions are the reference's: std::invalid_argument for column
// mismatches (models.cpp:396-412), data_error / missing_artifact_error /
// io_error from core.hpp; device failures raise std::runtime_error (there is
// no CPU fallback).  Decisions are bit-identical to the reference's.
#ifndef GPUDVFS_B200_GPU_API_HPP
#define GPUDVFS_B200_GPU_API_HPP

#include <memory>
#include <vector>

#include "gdvfs.h"
#include "gpudvfs/clustering.hpp"
#include "gpudvfs/core.hpp"
#include "gpudvfs/ingest.hpp"
#include "gpudvfs/models.hpp"
#include "gpudvfs/scheduler.hpp"

namespace gpudvfs::gpu {

/// The device the drop-in API runs on (one gd_ctx per (host thread, device),
/// kept for the thread's lifetime; device 0 unless select_device() is called
/// first on that thread).  A predictor keeps the device(s) selected when it
/// was made.
void select_device(int device);

/// Row-shard the predictors made after this call on this thread over several
/// devices: one replica of each model per device, contiguous
/// matched-app ranges per device, one NCCL gather of the decisions
/// (gd_multi_grid_select).  Results are identical to one device.
void select_devices(const std::vector<int>& devices);

/// models::predict on the GPU (kernel K1): one value per row, energy clamped
/// at 0, identical bits.  Throws std::invalid_argument naming the first
/// mismatched column, like the reference.
std::vector<double> predict(const models::FittedModel& model, const ingest::EncodedMatrix& rows);

/// make_model_predictor on the GPU: the same correlation and nearest-record
/// substitution, but the candidate rows are generated inside the fused
/// kernel (K2) instead of being materialised.  The returned ClockPredictor
/// answers exactly what the reference's would.
sched::ClockPredictor make_model_predictor(models::FittedModel energy_model, ingest::EncodingMetadata energy_encoding,
                                           models::FittedModel time_model, ingest::EncodingMetadata time_encoding,
                                           Dataset catalog, cluster::KMeansModel clusters);

/// schedule_d_dvfs: every job's per-clock predictions in one batched launch
/// when `predictor` came from gpu::make_model_predictor (else via the
/// predictor callback), then the EDF loop of scheduler.cpp:105-147 in
/// O(n log n) (gd_schedule_edf).
std::vector<sched::ScheduleDecision> schedule_d_dvfs(const Workload& workload, const sched::ClockPredictor& predictor,
                                                     const sched::ExecutionTimeSource& exec,
                                                     const sched::SchedulerOptions& options = {});

}  // namespace gpudvfs::gpu

#endif
