// The reference-side binding of the B200 path: what a
// maintainer adds to /root/reference/proj/core to route the hot path through
// libloratwin_gpu.so. Same signatures and exceptions as the reference
// functions it stands in for; compiled against the reference's own headers.
#pragma once

#include <cstdint>
#include <vector>

#include "loratwin/engine.hpp"
#include "loratwin/metrics.hpp"
#include "loratwin/placement.hpp"

namespace loratwin::gpu {

// run_simulation (engine.hpp:70-71) + compute_metrics (metrics.hpp:49-50):
// the full SimulationResult (requests with their emit times, load events,
// the iteration trace when options.record_iteration_trace) and its metrics.
SimulationResult run_simulation(const WorkloadSpec& workload, const ServerConfig& config, LengthMode mode,
                                const SimOptions& options, MetricsSummary* metrics);

// run_scripted (engine.hpp:76-78) + compute_metrics.
SimulationResult run_scripted(const std::vector<Request>& requests, const std::vector<AdapterSpec>& adapters,
                              double duration_s, const ServerConfig& config, const SimOptions& options,
                              MetricsSummary* metrics);

// sweep_optimal (placement.hpp:100-102) for many conditions in one device
// call; throws the lowest-index failing condition's exception, as
// run_parallel does (placement.cpp:93-95).
std::vector<PlacementResult> sweep_optimal_batch(const std::vector<Condition>& conditions,
                                                 const ServerConfig& config, const SweepGrid& grid,
                                                 double duration_s, std::uint64_t seed, const SweepOptions& options);

// The device set a host thread's context uses: CUDA devices of the mask
// (bit d = device d), default device 0. Call before the first GPU call.
void set_device_mask(std::uint64_t mask);

}  // namespace loratwin::gpu
