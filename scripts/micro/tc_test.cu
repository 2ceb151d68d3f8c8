// Standalone check of k_tc_gemm (tcgen05 3xTF32, pre-split B tiles) against an
// fp64 CPU reference, plus timing at the ESAI shapes.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_1603_06400_b200/csrc/tcgemm.cuh"

using namespace cacsi;

static double run(int M, int N, int K, int S, bool positive, bool timeit, int reps = 3) {
    const int lda = (K + 31) / 32 * 32, nkc = lda / 32;
    std::vector<float> A((size_t)M * lda, 0.f), B((size_t)N * K);
    srand(M + N + K);
    for (int i = 0; i < M; i++)
        for (int k = 0; k < K; k++) A[(size_t)i * lda + k] = (float)rand() / RAND_MAX;
    for (auto &x : B) x = (float)rand() / RAND_MAX - (positive ? 0.f : 0.3f);
    const int ntiles = (N + 127) / 128;
    std::vector<float> Bt((size_t)ntiles * nkc * 8192);
    tc_pack_b(B.data(), N, K, K, nkc, Bt.data());
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, Bt.size() * 4);
    const int ldc = (N + 3) / 4 * 4;
    cudaMalloc(&dC, (size_t)S * M * ldc * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    const int cps = (nkc + S - 1) / S;
    dim3 grid(ntiles, (M + 127) / 128, S);
    cudaFuncSetAttribute(k_tc_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    k_tc_gemm<<<grid, TC_T, TC_SMEM>>>(M, N, K, lda, nkc, cps, dA, dB, dC, ldc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("launch error %s\n", cudaGetErrorString(e));
        exit(1);
    }
    double rl2 = -1;
    if (!timeit) {
        std::vector<float> C((size_t)S * M * ldc);
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0, num = 0, den = 0;
        for (int i = 0; i < M; i++)
            for (int j = 0; j < N; j++) {
                double ref = 0;
                for (int k = 0; k < K; k++) ref += (double)A[(size_t)i * lda + k] * B[(size_t)j * K + k];
                double got = 0;
                for (int z = 0; z < S; z++) got += C[(size_t)z * M * ldc + (size_t)i * ldc + j];
                num += (got - ref) * (got - ref);
                den += ref * ref;
                maxrel = fmax(maxrel, fabs(got - ref) / (fabs(ref) + 1e-30));
            }
        rl2 = sqrt(num / den);
        printf("M=%d N=%d K=%d S=%d %s: rel_l2=%.3e max_rel=%.3e\n", M, N, K, S, positive ? "pos" : "mixed", rl2,
               maxrel);
    } else {
        cudaEvent_t t0, t1;
        cudaEventCreate(&t0);
        cudaEventCreate(&t1);
        for (int r = 0; r < reps; r++) {
            cudaEventRecord(t0);
            k_tc_gemm<<<grid, TC_T, TC_SMEM>>>(M, N, K, lda, nkc, cps, dA, dB, dC, ldc);
            cudaEventRecord(t1);
            cudaEventSynchronize(t1);
            float ms;
            cudaEventElapsedTime(&ms, t0, t1);
            printf("time M=%d N=%d K=%d S=%d: %.3f ms (%.1f TFLOP/s fp32-equivalent)\n", M, N, K, S, ms,
                   2.0 * M * N * K / ms / 1e9);
        }
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    return rl2;
}

int main() {
    run(300, 260, 200, 1, false, false);
    run(130, 7, 64, 1, true, false);
    run(257, 128, 7424, 1, true, false);
    run(257, 128, 7424, 8, true, false);
    run(257, 128, 7424, 16, true, false);
    run(257, 128, 7424, 32, true, false);
    run(257, 128, 7424, 1, false, false);
    run(257, 128, 7424, 16, false, false);
    run(257, 13, 37, 1, true, false);
    run(16384, 7424, 128, 1, true, true);
    run(16384, 128, 7424, 8, true, true);
    run(16384, 128, 7424, 16, true, true);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
