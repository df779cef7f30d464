// Cost of one cooperative grid.sync() on this GPU (diagnostics for the fused upper levels).
#include <cooperative_groups.h>
#include <cstdio>
__global__ void k(int n, int* sink) {
    auto g = cooperative_groups::this_grid();
    for (int i = 0; i < n; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = n;
}
__global__ void kb(int n, int* sink) {
    for (int i = 0; i < n; ++i) __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = n;
}
int main() {
    int* sink; cudaMalloc(&sink, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int per : {1, 2}) {
        int grid = sms * per, n = 1000;
        void* args[] = {&n, &sink};
        cudaLaunchCooperativeKernel((void*)k, grid, 128, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k, grid, 128, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("grid %d x 128: %.3f us per grid.sync (%s)\n", grid, 1e3 * ms / n, cudaGetErrorString(cudaGetLastError()));
    }
    int n = 1000;
    kb<<<1, 128>>>(n, sink);
    cudaEventRecord(a); kb<<<1, 128>>>(n, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("__syncthreads: %.4f us\n", 1e3 * ms / n);
    cudaEventRecord(a); for (int i = 0; i < 100; ++i) kb<<<1, 128>>>(0, sink); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("empty launch: %.2f us\n", 1e3 * ms / 100);
    return 0;
}
