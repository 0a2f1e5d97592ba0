// engine_kernel<384, 1, false> in its own translation unit (engine_launch.h).
#include "engine_launch.h"
#include "k_engine.cuh"

namespace lt {

const void* engine_fn_occ12() { return reinterpret_cast<const void*>(engine_kernel<384, 1, false>); }

void engine_launch_occ12(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E) {
  engine_kernel<384, 1, false><<<grid, block, smem, st>>>(E);
}

}  // namespace lt
