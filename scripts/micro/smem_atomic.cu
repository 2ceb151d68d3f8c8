// Microbenchmark: shared-memory fp32 atomicAdd vs plain RMW throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atomic(float *out, int iters, int range, int mode) {
    extern __shared__ float h[];
    for (int i = threadIdx.x; i < range; i += blockDim.x) h[i] = 0.f;
    __syncthreads();
    unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    for (int i = 0; i < iters; i++) {
        x = x * 1664525u + 1013904223u;
        int idx;
        if (mode == 0) idx = (warp * 32 + lane * 37 + (x >> 20)) % range;      // random-ish spread
        else if (mode == 1) idx = ((x >> 16) % (range / 32)) * 32 + lane;      // distinct banks
        else idx = (x >> 16) % 64;                                               // heavy collisions
        atomicAdd(&h[idx], 1.0f);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < range; i += blockDim.x) out[blockIdx.x * range + i] = h[i];
}
template <class T>
__global__ void k_atomic_int(float *out, int iters, int range, int mode) {
    extern __shared__ float hf[];
    T *h = (T *)hf;
    int r = range / (sizeof(T) / 4);
    for (int i = threadIdx.x; i < r; i += blockDim.x) h[i] = 0;
    __syncthreads();
    unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    for (int i = 0; i < iters; i++) {
        x = x * 1664525u + 1013904223u;
        int idx = mode == 0 ? (warp * 32 + lane * 37 + (x >> 20)) % r : ((x >> 16) % (r / 32)) * 32 + lane;
        atomicAdd(&h[idx], (T)(x & 0xffff));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < r; i += blockDim.x) out[blockIdx.x * range + i] = (float)h[i];
}
__global__ void k_rmw(float *out, int iters, int range) {
    extern __shared__ float h[];
    for (int i = threadIdx.x; i < range; i += blockDim.x) h[i] = 0.f;
    __syncthreads();
    unsigned lane = threadIdx.x & 31;
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    for (int i = 0; i < iters; i++) {
        x = x * 1664525u + 1013904223u;
        int idx = ((x >> 16) % (range / 32 / (blockDim.x / 32))) * blockDim.x + threadIdx.x;  // private column
        h[idx] += 1.0f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < range; i += blockDim.x) out[blockIdx.x * range + i] = h[i];
}
int main() {
    int range = 8192, iters = 4096, blocks = 148 * 4, threads = 256;
    float *out;
    cudaMalloc(&out, (size_t)blocks * range * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 8; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (mode < 3) k_atomic<<<blocks, threads, range * 4>>>(out, iters, range, mode);
            else if (mode == 3) k_rmw<<<blocks, threads, range * 4>>>(out, iters, range);
            else if (mode < 6) k_atomic_int<unsigned><<<blocks, threads, range * 4>>>(out, iters, range, mode - 4);
            else k_atomic_int<unsigned long long><<<blocks, threads, range * 4>>>(out, iters, range, mode - 6);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters;
            if (rep) printf("mode %d: %.3f ms  %.3e lane-ops/s  %.2f lane-ops/clk/SM @1.9GHz\n", mode, ms, ops / ms * 1e3,
                            ops / ms * 1e3 / 148 / 1.9e9);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
