// Device-side differential check of the lt_libm.h ports (the code the K0
// kernels run: nvcc, sm_100a, --fmad=false) against the host's glibc libm.
//   libm_device <fma|generic|auto> <samples per function> <seed>
// Inputs cover the reference's RNG domains (rng.hpp:54, :65-70): -u for
// log1p, u for log, 2*pi*u for sin/cos with u = (x >> 11) * 2^-53 (3 of 4
// samples), plus wider random ranges (1 of 4). Prints one line per function
// "<name> <samples> <mismatches>"; exit 0 when every result is bit-identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "lt_libm.h"

template <bool F>
__global__ void eval_kernel(int which, const double* x, double* y, long n) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double v = x[i];
    double r;
    switch (which) {
      case 0: r = lt::glibc_log1p<F>(v); break;
      case 1: r = lt::glibc_log<F>(v); break;
      case 2: r = lt::glibc_sin<F>(v); break;
      default: r = lt::glibc_cos<F>(v); break;
    }
    y[i] = r;
  }
}

static void gen_inputs(int which, uint64_t seed, long n, double* x) {
  const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    pool.emplace_back([=] {
      const long b = n * t / threads, e = n * (t + 1) / threads;
      std::mt19937_64 g(seed * 1000003ULL + which * 7919ULL + t);
      for (long i = b; i < e; ++i) {
        const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
        const bool wide = (i & 3) == 0;
        const double w = static_cast<double>(g() >> 11) * 0x1.0p-53;
        switch (which) {
          case 0: x[i] = wide ? w * 8.0 - 0.999 : -u; break;
          case 1: x[i] = wide ? std::ldexp(1.0 + u, static_cast<int>(g() % 200) - 100) : u; break;
          default: x[i] = wide ? w * 40.0 - 20.0 : (2.0 * M_PI) * u; break;
        }
        if (which == 1 && x[i] == 0.0) x[i] = 0x1.0p-53;  // log's domain: u1 > 0 (rng.hpp:65-66 resamples)
      }
    });
  }
  for (auto& th : pool) th.join();
}

static long compare(int which, const double* x, const double* y, long n, long* first_bad) {
  const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  std::atomic<long> bad{0};
  std::atomic<long> first{-1};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const long b = n * t / threads, e = n * (t + 1) / threads;
      long local = 0;
      for (long i = b; i < e; ++i) {
        double want;
        switch (which) {
          case 0: want = std::log1p(x[i]); break;
          case 1: want = std::log(x[i]); break;
          case 2: want = std::sin(x[i]); break;
          default: want = std::cos(x[i]); break;
        }
        if (lt::as_u64(want) != lt::as_u64(y[i])) {
          ++local;
          long exp = -1;
          first.compare_exchange_strong(exp, i);
        }
      }
      bad += local;
    });
  }
  for (auto& th : pool) th.join();
  *first_bad = first.load();
  return bad.load();
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "auto";
  const long samples = argc > 2 ? std::atol(argv[2]) : 100000000L;
  const uint64_t seed = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1;
  bool fma = mode == "fma";
  if (mode == "auto") {  // which glibc build does this host run? (the device follows it, as lt_sim_options does)
    std::mt19937_64 g(5);
    long diff = 0;
    for (int i = 0; i < 200000; ++i) {
      const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
      diff += lt::as_u64(std::log1p(-u)) != lt::as_u64(lt::glibc_log1p<true>(-u));
    }
    fma = diff == 0;
  }
  std::printf("variant %s\n", fma ? "fma" : "generic");
  const long chunk = 1L << 24;
  double *dx = nullptr, *dy = nullptr;
  if (cudaMalloc(&dx, chunk * 8) != cudaSuccess || cudaMalloc(&dy, chunk * 8) != cudaSuccess) {
    std::printf("no device\n");
    return 3;
  }
  std::vector<double> x(chunk), y(chunk);
  const char* names[4] = {"log1p", "log", "sin", "cos"};
  long total_bad = 0;
  for (int which = 0; which < 4; ++which) {
    long bad = 0;
    for (long done = 0; done < samples; done += chunk) {
      const long n = std::min(chunk, samples - done);
      gen_inputs(which, seed + static_cast<uint64_t>(done / chunk), n, x.data());
      cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
      if (fma)
        eval_kernel<true><<<148 * 8, 256>>>(which, dx, dy, n);
      else
        eval_kernel<false><<<148 * 8, 256>>>(which, dx, dy, n);
      if (cudaMemcpy(y.data(), dy, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        std::printf("cuda error: %s\n", cudaGetErrorString(cudaGetLastError()));
        return 2;
      }
      long first = -1;
      const long b = compare(which, x.data(), y.data(), n, &first);
      if (b && bad == 0) std::printf("  %s mismatch x=%a device=%a\n", names[which], x[first], y[first]);
      bad += b;
    }
    std::printf("%s %ld %ld\n", names[which], samples, bad);
    total_bad += bad;
  }
  cudaFree(dx);
  cudaFree(dy);
  return total_bad ? 1 : 0;
}
