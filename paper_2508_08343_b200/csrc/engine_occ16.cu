// engine_kernel<256, 2, false> in its own translation unit (engine_launch.h).
#include "engine_launch.h"
#include "k_engine.cuh"

namespace lt {

const void* engine_fn_occ16() { return reinterpret_cast<const void*>(engine_kernel<256, 2, false>); }

void engine_launch_occ16(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E) {
  engine_kernel<256, 2, false><<<grid, block, smem, st>>>(E);
}

}  // namespace lt
