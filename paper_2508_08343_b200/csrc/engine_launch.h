// The engine kernel's compiled builds (k_engine.cuh), each in its own
// translation unit (engine_*.cu, compiled in parallel); the host code
// (capi.cu) sizes, queries and launches them through these entry points.
#pragma once

#include <cuda_runtime.h>

#include "lt_device.cuh"

namespace lt {

// 1: latency (8 warps/SM, engine_kernel<256,1>), 2: occupancy (16 warps/SM,
// <256,2>), 3: throughput (12 warps/SM, <384,1>), 4: report / checked build
// (<256,1,true>), 5: recording build of the percentile path (<256,1,false,true>).
enum EngineBuild { kEngineLatency = 1, kEngineOcc16 = 2, kEngineOcc12 = 3, kEngineChecked = 4, kEngineRecord = 5 };

const void* engine_kernel_fn(int build);
void launch_engine_build(int build, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                         const EngineParams& E);

// fresh-queue chain links of the linked builds (link_kernel, engine_latency.cu)
void link_launch(unsigned grid, size_t smem, cudaStream_t st, const DScen* scen, int n_scen, int max_adapters,
                 const int32_t* r_in, const int32_t* r_adp, int32_t* r_link);

// per-build entry points (one translation unit each)
const void* engine_fn_latency();
const void* engine_fn_occ16();
const void* engine_fn_occ12();
const void* engine_fn_checked();
const void* engine_fn_record();
void engine_launch_latency(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E);
void engine_launch_occ16(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E);
void engine_launch_occ12(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E);
void engine_launch_checked(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E);
void engine_launch_record(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E);

inline const void* engine_kernel_fn(int build) {
  switch (build) {
    case kEngineOcc16: return engine_fn_occ16();
    case kEngineOcc12: return engine_fn_occ12();
    case kEngineChecked: return engine_fn_checked();
    case kEngineRecord: return engine_fn_record();
    default: return engine_fn_latency();
  }
}

inline void launch_engine_build(int build, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                                const EngineParams& E) {
  switch (build) {
    case kEngineOcc16: engine_launch_occ16(grid, block, smem, st, E); break;
    case kEngineOcc12: engine_launch_occ12(grid, block, smem, st, E); break;
    case kEngineChecked: engine_launch_checked(grid, block, smem, st, E); break;
    case kEngineRecord: engine_launch_record(grid, block, smem, st, E); break;
    default: engine_launch_latency(grid, block, smem, st, E); break;
  }
}

}  // namespace lt
