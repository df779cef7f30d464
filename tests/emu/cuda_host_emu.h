// cuda_host_emu.h — lets the product's kernel headers (paper_1610_08035_b200/csrc/
// engine.cuh, model_dev.cuh, devmat.cuh) compile as plain host C++ so the exact
// device code paths can be executed on the CPU, one emulated thread at a time.
// TEST INFRASTRUCTURE ONLY (used by tests/emu/emu.cpp).  Cooperative kernels
// (the shared-memory reductions) are not emulated; the emulator sums on the host.
#pragma once
#define SPINGP_HOST_EMU 1
#include <algorithm>
#include <cmath>
#include <cstdint>

#define __device__
#define __host__
#define __forceinline__ inline
#define __global__
#define __launch_bounds__(...)
#define __shared__ static
#define __restrict__ __restrict

struct dim3 {
    unsigned x = 1, y = 1, z = 1;
    dim3() = default;
    dim3(unsigned a, unsigned b = 1, unsigned c = 1) : x(a), y(b), z(c) {}
};
inline thread_local dim3 threadIdx, blockIdx, blockDim, gridDim;
inline void __syncthreads() {}
inline unsigned long long atomicMin(unsigned long long* p, unsigned long long v) {
    const unsigned long long o = *p;
    if (v < o) *p = v;
    return o;
}
using std::isfinite;
inline double rsqrt(double x) { return 1.0 / std::sqrt(x); }
using std::max;
using std::min;

// Run `body` for every (block, thread) of a 1-D grid, in order.
template <class F>
void emu_launch(unsigned grid, unsigned block, F&& body) {
    gridDim = dim3(grid);
    blockDim = dim3(block);
    for (unsigned b = 0; b < grid; ++b)
        for (unsigned t = 0; t < block; ++t) {
            blockIdx = dim3(b);
            threadIdx = dim3(t);
            body();
        }
}
