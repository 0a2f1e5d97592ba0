// engine_kernel<256, 1, false, true> in its own translation unit
// (engine_launch.h): the latency build plus the single-pass ITL recording of
// the percentile path, without the report / invariant-check code.
#include "engine_launch.h"
#include "k_engine.cuh"

namespace lt {

const void* engine_fn_record() { return reinterpret_cast<const void*>(engine_kernel<256, 1, false, true>); }

void engine_launch_record(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E) {
  engine_kernel<256, 1, false, true><<<grid, block, smem, st>>>(E);
}

}  // namespace lt
