// sgemm.cuh -- fp32 SIMT GEMM used by the ESAI contraction over q
// (W = F S~^T and b2 = A S~).  128x128 CTA tile, 8x8 register micro-tile per
// thread, K step 8, register-staged double buffering, arbitrary M/N/K (zero
// fill at the edges).  Optional split-K over gridDim.z writes partial tiles.
#pragma once
#include <cuda_runtime.h>

namespace cacsi {

constexpr int GM_BM = 128, GM_BN = 128, GM_BK = 8, GM_T = 256;

// C[z][M][N] = sum_{k in slice z} A[M][K] * B(k, n)
//   B_NK: B stored [N][K] (C = A B^T);  else B stored [K][N] (C = A B).
template <bool B_NK>
__global__ void __launch_bounds__(GM_T) k_sgemm(int M, int N, int K, int k_per_split, const float *__restrict__ A,
                                                 const float *__restrict__ B, float *__restrict__ C) {
    __shared__ __align__(16) float As[2][GM_BK][GM_BM + 4];
    __shared__ __align__(16) float Bs[2][GM_BK][GM_BN + 4];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.y * GM_BM, n0 = blockIdx.x * GM_BN;
    const int kb = blockIdx.z * k_per_split;
    const int ke = min(K, kb + k_per_split);
    C += (size_t)blockIdx.z * M * N;

    // loader mapping: A tile 128 x 8 -> thread loads rows (tid >> 1), k (tid & 1) * 4 .. +4
    const int a_row = tid >> 1, a_k = (tid & 1) * 4;
    // B tile: B_NK like A; else 8 x 128 -> row k = tid >> 5, cols (tid & 31) * 4 .. +4
    const int b_row = B_NK ? (tid >> 1) : (tid >> 5);
    const int b_col = B_NK ? (tid & 1) * 4 : (tid & 31) * 4;
    float ra[4], rb[4];

    auto load = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int m = m0 + a_row, k = k0 + a_k + i;
            ra[i] = (m < M && k < ke) ? A[(size_t)m * K + k] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
            if (B_NK) {
                const int n = n0 + b_row, k = k0 + b_col + i;
                rb[i] = (n < N && k < ke) ? B[(size_t)n * K + k] : 0.0f;
            } else {
                const int k = k0 + b_row, n = n0 + b_col + i;
                rb[i] = (k < ke && n < N) ? B[(size_t)k * N + n] : 0.0f;
            }
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 4; i++) As[buf][a_k + i][a_row] = ra[i];
        if (B_NK) {
#pragma unroll
            for (int i = 0; i < 4; i++) Bs[buf][b_col + i][b_row] = rb[i];
        } else {
            *(float4 *)&Bs[buf][b_row][b_col] = make_float4(rb[0], rb[1], rb[2], rb[3]);
        }
    };

    // compute mapping: thread (tx, ty) owns rows ty*4 + {0..3} and 64 + ty*4 + {0..3},
    // cols tx*4 + {0..3} and 64 + tx*4 + {0..3}
    const int tx = tid & 15, ty = tid >> 4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.0f;

    int buf = 0;
    load(kb);
    store(0);
    __syncthreads();
    for (int k0 = kb; k0 < ke; k0 += GM_BK) {
        const bool more = k0 + GM_BK < ke;
        if (more) load(k0 + GM_BK);
#pragma unroll
        for (int kk = 0; kk < GM_BK; kk++) {
            const float4 a0 = *(const float4 *)&As[buf][kk][ty * 4];
            const float4 a1 = *(const float4 *)&As[buf][kk][64 + ty * 4];
            const float4 b0 = *(const float4 *)&Bs[buf][kk][tx * 4];
            const float4 b1 = *(const float4 *)&Bs[buf][kk][64 + tx * 4];
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
            if (n < N) C[(size_t)m * N + n] = acc[i][j];
        }
    }
}

}  // namespace cacsi
