// engine_kernel<256, 1, true> in its own translation unit (engine_launch.h).
#include "engine_launch.h"
#include "k_engine.cuh"

namespace lt {

const void* engine_fn_checked() { return reinterpret_cast<const void*>(engine_kernel<256, 1, true>); }

void engine_launch_checked(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E) {
  engine_kernel<256, 1, true><<<grid, block, smem, st>>>(E);
}

}  // namespace lt
