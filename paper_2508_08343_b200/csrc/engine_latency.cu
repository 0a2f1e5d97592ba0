// engine_kernel<256, 1, false> in its own translation unit (engine_launch.h),
// with link_kernel, which computes the chain links the linked builds' ingest
// reads (k_engine.cuh, kLinks).
#include "engine_launch.h"
#include "k_engine.cuh"

namespace lt {

const void* engine_fn_latency() { return reinterpret_cast<const void*>(engine_kernel<256, 1, false>); }

// Fresh-queue chain links of every request, built before each engine pass
// from the request arrays (generated or scripted): r_link[i] = the same
// adapter's next request in index order that is not oversized (kLinkNone at
// the end) | kLinkFirst on an adapter's first one. Oversized requests (in + 1 >
// capacity) go to the engine's oversized FIFO instead and are rejected when a
// scan passes them. The engine's ingest (engine.cpp:88-92; per-adapter FIFO
// order of kv_scheduler.cpp:109-166) then writes whole nodes in one store and
// only notes which chains turned non-empty. One warp per scenario, 32
// requests per step: __match_any_sync finds each request's in-step neighbours
// of its adapter, last[] the previous step's tail.
__global__ void __launch_bounds__(256) link_kernel(const DScen* scen, int n_scen, int max_adapters,
                                                  const int32_t* r_in, const int32_t* r_adp,
                                                  int32_t* r_link) {
  extern __shared__ int32_t link_last[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
  int32_t* last = link_last + warp * max_adapters;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (int s = blockIdx.x * warps + warp; s < n_scen; s += gridDim.x * warps) {
    const int n = scen[s].n_req;
    if (scen[s].status != LT_OK || n <= 0) continue;
    const int na = scen[s].n_adapters;
    const int64_t rb = scen[s].req_begin, cap = scen[s].capacity;
    for (int a = lane; a < na; a += 32) last[a] = -1;
    __syncwarp();
    // Four steps (128 requests) at a time, the next four steps' loads issued
    // before this group's links: the steps are a serial chain through last[],
    // the loads are not (one step at a time waited on each load: 0.45 ms for
    // C2's 15 k-request engines; one step ahead: 0.24 ms).
    constexpr int kAhead = 4;
    int a_n[kAhead], in_n[kAhead];
#pragma unroll
    for (int u = 0; u < kAhead; ++u) {
      const int j = u * 32 + lane;
      a_n[u] = j < n ? r_adp[rb + j] : 0;
      in_n[u] = j < n ? r_in[rb + j] : 0;
    }
    for (int base0 = 0; base0 < n; base0 += 32 * kAhead) {
      int a_c[kAhead], in_c[kAhead];
#pragma unroll
      for (int u = 0; u < kAhead; ++u) {
        a_c[u] = a_n[u];
        in_c[u] = in_n[u];
        const int j = base0 + 32 * kAhead + u * 32 + lane;
        a_n[u] = j < n ? r_adp[rb + j] : 0;
        in_n[u] = j < n ? r_in[rb + j] : 0;
      }
#pragma unroll
      for (int u = 0; u < kAhead; ++u) {
        const int base = base0 + u * 32;
        if (base >= n) break;
        const int i = base + lane;
        const bool v = i < n;
        const int a = a_c[u], in = in_c[u];
        const bool over = v && static_cast<int64_t>(in) + 1 > cap;
        const bool chained = v && !over;
        const unsigned mm = __match_any_sync(0xffffffffu, chained ? a : -1 - lane);
        const unsigned later = mm & ~lt & ~(1u << lane);
        int flags = 0;
        if (chained) {
          if (!(mm & lt)) {  // first of its adapter in this step: link from the previous tail
            const int p = last[a];  // index | its kLinkFirst flag, or -1
            if (p < 0)
              flags = kLinkFirst;
            else
              r_link[rb + (p & kLinkNone)] = i | (p & kLinkFirst);
          }
          r_link[rb + i] = (later ? base + __ffs(later) - 1 : kLinkNone) | flags;
        } else if (v) {
          r_link[rb + i] = kLinkNone;
        }
        __syncwarp();
        if (chained && !later) last[a] = i | flags;
        __syncwarp();
      }
    }
  }
}

void link_launch(unsigned grid, size_t smem, cudaStream_t st, const DScen* scen, int n_scen, int max_adapters,
                 const int32_t* r_in, const int32_t* r_adp, int32_t* r_link) {
  link_kernel<<<grid, 256, smem, st>>>(scen, n_scen, max_adapters, r_in, r_adp, r_link);
}

void engine_launch_latency(unsigned grid, unsigned block, size_t smem, cudaStream_t st, const EngineParams& E) {
  engine_kernel<256, 1, false><<<grid, block, smem, st>>>(E);
}

}  // namespace lt
