// Box probe: device properties, FP64 DFMA peak, HBM copy cross-check.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dchain(double* out, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = 1.0 + threadIdx.x;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) y = sqrt(y + 1.0);
  long long t3 = clock64();
  double z = 2.0 + threadIdx.x;
  for (int i = 0; i < iters; ++i) z = 1.0 / (z + 1.0);
  long long t4 = clock64();
  double w = 0.5;
  for (int i = 0; i < iters; ++i) w = exp(-w);
  long long t5 = clock64();
  if (threadIdx.x == 0) printf("latency cycles: dfma %.2f  sqrt+add %.2f  rcp+add %.2f  exp %.2f\n",
     (double)(t1-t0)/iters, (double)(t3-t2)/iters, (double)(t4-t3)/iters, (double)(t5-t4)/iters);
  out[threadIdx.x] = x + y + z + w;
}
__global__ void copyk(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("name %s sms %d smemPerSM %zu smemPerBlockOptin %zu regsPerSM %d L2 %d MB HBM %.1f GB clock %d kHz memclk %d kHz busw %d\n",
    p.name, p.multiProcessorCount, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor,
    p.l2CacheSize >> 20, p.totalGlobalMem / 1e9, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int tpb : {128, 256, 512}) for (int bps : {4, 8, 16}) {
    int blocks = p.multiProcessorCount * bps * 512 / tpb / 4;
    dfma_peak<<<blocks, tpb>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_peak<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * tpb;
    printf("dfma tpb %d blocks %d : %.2f TFLOP/s fp64\n", tpb, blocks, flops / ms / 1e9);
  }
  dchain<<<1, 32>>>(out, 1000, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
  size_t n = (size_t)1 << 28; double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  float best = 1e9;
  for (int r = 0; r < 6; ++r) { cudaEventRecord(e0); copyk<<<p.multiProcessorCount * 8, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("copy kernel %.1f GB/s (read+write, 8 GiB)\n", 2.0 * n * 16 / best / 1e6);
  return 0;
}
