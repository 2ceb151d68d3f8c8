// tcgemm16.cuh -- the ESAI contractions (W = F S~^T, b2 = A S~) on the tensor cores
// at the fp16 rate with an fp32-level result: a two-term fp16 split of both operands
// (option gemm16=1).
//
//   x' = s x  (s a power of two: |x'| < 2^14),  hi = fp16_rn(x'),  lo = fp16_rn(x' - hi)
//   C  = (A_hi B_hi + (A_hi B_lo + A_lo B_hi)) / (s_A s_B)
//
// Error per product: |x' - hi - lo| <= 2^-11 |x' - hi| <= 2^-22 |x'| for each operand
// (round to nearest twice; x' - hi is exact in fp32) and the dropped A_lo B_lo term is
// <= 2^-22 |ab|, so ~3 2^-22 = 7e-7 relative per product -- below the 3xTF32 split of
// tcgemm.cuh (truncated hi, 2^-20) -- as long as x' stays in fp16's normal range
// (|x'| >= 2^-14, i.e. down to 2^-28 of the scaled maximum; below that the split keeps
// an absolute error of 2^-25, ~2^-39 of the maximum).  fp16 x fp16 products are exact
// in the fp32 accumulator; kind::f16 has K = 16 per instruction, so a contraction
// takes half the accumulate steps of kind::tf32 (K = 8).
// Scales: A = f (W GEMM) per ROW, from the row's max |f| (the panel holds the whole K
// = nq); A = the backward's histogram matrix (b2 GEMM) one global power of two from
// its fixed-point bound |A[v][b]| <= vbound[v] max|w| (esai.cu: every bin sum stays
// below 2^30 units of vbound[v] max|w| / 2^30); B = S~ one global power of two
// (Esai.s16_exp, from max |S~| at create).  Scaling by powers of two is exact.
//
// Operand layout: K-major SWIZZLE_128B as in tcgemm.cuh, one 128-byte row = 64 fp16, so
// a K chunk is 64 wide; the descriptors and the 32-byte k-step advance are the same
// bytes as the TF32 kernels' (K = 16 fp16 = 32 B).  A arrives as raw fp32 by TMA
// tensor loads (two 128 x 32 boxes per chunk, 32 KB) and is split IN PLACE: row r's
// 64 fp32 occupy bytes [r 128, r 128 + 128) of the two 16 KB halves, exactly where
// its 64 fp16 hi and 64 fp16 lo go, so each thread converts its own row with no
// cross-thread hazard.
#pragma once
#include <cuda_fp16.h>

#include "tcgemm.cuh"

namespace cacsi {

constexpr int TC16_KC = 64;                // K chunk (64 fp16 = one 128-byte swizzle row)
constexpr int TC16_OPB = TC_M * TC16_KC * 2;  // one operand half (hi or lo): 16 KB
constexpr int TC16_CH = 2 * TC16_OPB;         // hi + lo chunk: 32 KB

// instruction descriptor: D fp32, A/B fp16, both K-major, N = 128, M = 128
__host__ __device__ constexpr uint32_t tc_idesc_f16() {
    return (1u << 4)                        // c_format F32 (a_format = b_format = 0: F16)
           | ((uint32_t)(TC_N >> 3) << 17)  // n_dim
           | ((uint32_t)(TC_M >> 4) << 24); // m_dim
}

__device__ __forceinline__ void tc_mma16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// byte offset of fp16 element (row, k), k in [0, 64), inside a 128 x 64 tile
__host__ __device__ __forceinline__ uint32_t tc_swz16(int row, int k) {
    return (uint32_t)(row * 128 + ((((k >> 3) ^ (row & 7)) << 4) | ((k & 7) << 1)));
}

// the power-of-two exponent e with |x| 2^e < 2^14 for every |x| <= amax (amax >= 0),
// clamped so that 2^e and 2^-e are normal fp32
__host__ __device__ __forceinline__ int f16_scale_exp(float amax) {
    if (!(amax > 0.0f) || !(amax < 3.0e38f)) return 0;
    int ex;
    frexpf(amax, &ex);  // amax = m 2^ex, m in [0.5, 1): amax < 2^ex
    return max(-126, min(126, 14 - ex));
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }

// Raw fp32 row r of a 32 KB chunk region (two 128 x 32 SWIZZLE_128B boxes) -> registers
__device__ __forceinline__ void f16_load_row(const unsigned char *cb, int r, float (&v)[64]) {
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
        for (int cc = 0; cc < 8; cc++) {
            const float4 t = *(const float4 *)(cb + h * TC16_OPB + r * 128 + ((cc ^ (r & 7)) << 4));
            v[32 * h + 4 * cc] = t.x, v[32 * h + 4 * cc + 1] = t.y, v[32 * h + 4 * cc + 2] = t.z,
                          v[32 * h + 4 * cc + 3] = t.w;
        }
}

// ... and the split of those registers (scaled by sc) written back as row r of the
// fp16 hi tile (first 16 KB) and lo tile (second 16 KB)
__device__ __forceinline__ void f16_store_row(unsigned char *cb, int r, const float (&v)[64], float sc) {
#pragma unroll
    for (int c16 = 0; c16 < 8; c16++) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float x0 = v[8 * c16 + 2 * i] * sc, x1 = v[8 * c16 + 2 * i + 1] * sc;
            const __half2 h = __floats2half2_rn(x0, x1);
            const float2 hf = __half22float2(h);
            hw[i] = h2_bits(h);
            lw[i] = h2_bits(__floats2half2_rn(x0 - hf.x, x1 - hf.y));
        }
        const uint32_t off = (uint32_t)(r * 128 + ((c16 ^ (r & 7)) << 4));
        *(uint4 *)(cb + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *(uint4 *)(cb + TC16_OPB + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// ---- W = F S~^T: A-resident, persistent, warp-specialized (k_tc_gemm_ar's structure) --
// Warp 4 lane 0: producer (the f panel of each M tile by 2 nkc TMA boxes, B chunks into
// an NSB-stage ring); warp 5 lane 0: MMAs (12 per 64-wide chunk: 4 k-steps x 3 products)
// into one of two TMEM accumulator pairs; warps 0-3 and 6-9: at each new panel, split
// it in place -- warp w converts rows 32 (w % 4) .. + 31 of K chunk (w < 4 ? 0 : 1), the
// row maxima meet in shared memory -- then drain tiles (they own the same rows in TMEM,
// so each thread keeps its row's output scale in a register).
// TMAST: the epilogue stores each 32 x 32 block by a TMA tensor store (tmC: box 32 x 32,
// SWIZZLE_128B -- the layout the transpose already writes) from one of two staging
// buffers per warp, instead of 8 STG.128 per lane; rows past M / columns past N are
// clipped by the tensor map (its rows are C's: mrow0 + tile row).
constexpr int TCA16_T = 320;
constexpr int tca16_smem(int nkc, int nsb, bool tmast = false) {
    return nkc * TC16_CH + nsb * TC16_CH + (tmast ? 2 : 1) * 8 * 32 * 32 * 4 + 128 * 2 * 4 + 1024 + 256;
}
template <int NSB, bool TMAST = false>
__global__ void __launch_bounds__(TCA16_T, 1)
    k_tc_gemm_ar16(int M, int N, int nkc, int mtiles, int ntiles, const __half *__restrict__ Bt, float *__restrict__ C,
                   int ldc, const int *__restrict__ tpre, const int2 *__restrict__ tntr,
                   const __grid_constant__ CUtensorMap tmA, int mrow0, int bexp, const __grid_constant__ CUtensorMap tmC) {
    extern __shared__ __align__(1024) unsigned char t16_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)t16_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;                          // [nkc][hi, lo] 32 KB each (raw fp32 on arrival)
    unsigned char *sB = sA + nkc * TC16_CH;            // [NSB][hi, lo]
    float *ebuf = (float *)(sB + NSB * TC16_CH);       // [8][TMAST ? 2 : 1][32][32]
    float *rmax = ebuf + (TMAST ? 2 : 1) * 8 * 32 * 32;  // [2][128]: per K half, per panel row
    uint64_t *bars = (uint64_t *)(rmax + 2 * 128);
    uint64_t *a_full = bars, *a_empty = bars + 1, *b_full = bars + 2, *b_empty = bars + 2 + NSB,
             *t_full = bars + 2 + 2 * NSB, *t_empty = bars + 4 + 2 * NSB, *a_conv = bars + 6 + 2 * NSB;
    uint32_t *tmem_slot = (uint32_t *)(bars + 7 + 2 * NSB);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    TileWalk tw{tpre, tntr, mtiles, ntiles, 0, 0};
    const long long T = tw.count();
    const int t0 = (int)(T * blockIdx.x / gridDim.x), t1 = (int)(T * (blockIdx.x + 1) / gridDim.x);
    tw.start(t0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        // a_conv: one arrival per converter warp (8); t_empty: one per epilogue warp (8)
        for (int i = 0; i < 7 + 2 * NSB; i++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bars + i)),
                         "r"((i >= 4 + 2 * NSB && i < 6 + 2 * NSB) || i == 6 + 2 * NSB ? 8 : 1));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (tid == 160) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        if (lane == 0) {
            int cur_m = -1;
            uint32_t loads = 0, bc = 0;
            TileWalk w = tw;
            for (int t = t0; t < t1; t++, w.next()) {
                const int m = w.m, n = w.n;
                if (m != cur_m) {
                    if (loads > 0) mbar_wait(smem_u32(a_empty), (loads - 1) & 1);
                    const uint32_t mb = smem_u32(a_full);
                    // the converters' generic writes of the previous panel were ordered before
                    // the MMAs that released it; the proxy fence orders them before these
                    // async-proxy writes
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                                 "r"(nkc * (uint32_t)TC16_CH)
                                 : "memory");
                    for (int c = 0; c < 2 * nkc; c++)  // boxes past K land as zeros
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
                            "{%2, %3}], [%4];\n" ::"r"(smem_u32(sA + c * TC16_OPB)),
                            "l"(&tmA), "r"(c * 32), "r"(mrow0 + m * TC_M), "r"(mb)
                            : "memory");
                    cur_m = m;
                    loads++;
                }
                for (int c = 0; c < nkc; c++, bc++) {
                    const int st = bc % NSB;
                    if (bc >= NSB) mbar_wait(smem_u32(b_empty + st), ((bc / NSB) - 1) & 1);
                    const uint32_t mb = smem_u32(b_full + st);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(TC16_CH)
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(sB + st * TC16_CH)),
                        "l"(Bt + ((size_t)n * nkc + c) * (2 * TC_N * TC16_KC)), "r"(TC16_CH), "r"(mb)
                        : "memory");
                }
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            const uint32_t idesc = tc_idesc_f16();
            int cur_m = -1;
            uint32_t loads = 0, bc = 0, tc = 0;
            TileWalk w = tw;
            for (int t = t0; t < t1; t++, tc++) {
                const int m = w.m;
                w.next();
                if (m != cur_m) {
                    mbar_wait(smem_u32(a_conv), loads & 1);
                    loads++;
                    cur_m = m;
                }
                const int ab = tc & 1;
                if (tc >= 2) mbar_wait(smem_u32(t_empty + ab), ((tc >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t dmain = tmem + ab * 2 * TC_N, dcross = dmain + TC_N;
                for (int c = 0; c < nkc; c++, bc++) {
                    const int st = bc % NSB;
                    mbar_wait(smem_u32(b_full + st), (bc / NSB) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    const uint32_t ah0 = smem_u32(sA + c * TC16_CH), al0 = ah0 + TC16_OPB;
                    const uint32_t bh0 = smem_u32(sB + st * TC16_CH), bl0 = bh0 + TC16_OPB;
#pragma unroll
                    for (int ks = 0; ks < TC16_KC / 16; ks++) {
                        const uint32_t off = ks * 32;
                        tc_mma16(dmain, tc_desc(ah0 + off), tc_desc(bh0 + off), idesc, (c | ks) != 0);
                        tc_mma16(dcross, tc_desc(ah0 + off), tc_desc(bl0 + off), idesc, (c | ks) != 0);
                        tc_mma16(dcross, tc_desc(al0 + off), tc_desc(bh0 + off), idesc, 1);
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(b_empty + st)));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(t_full + ab)));
                if (t + 1 == t1 || w.m != m)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(a_empty)));
            }
        }
    } else {
        // warps 0-3 and 6-9: TMEM lanes 32 (warp % 4) .. + 31 = tile rows; warps 0-3 drain
        // columns 0-63 and convert K chunk 0, warps 6-9 columns 64-127 and K chunk 1
        const int ew = warp < 4 ? warp : warp - 2, lq = warp & 3, ch = warp < 4 ? 0 : TC_N / 2, kh = warp < 4 ? 0 : 1;
        const int row = lq * 32 + lane;
        float *buf = ebuf + ew * (TMAST ? 2 : 1) * (32 * 32);
        uint32_t bsel = 0;  // TMAST: staging buffer of the next block
        const int cq = 4 * (lane & 7);
        uint32_t tc = 0, loads = 0;
        int cur_m = -1;
        float osc = 0.0f;  // this thread's row: output scale 2^-(e_row + bexp)
        TileWalk w = tw;
        for (int t = t0; t < t1; t++, tc++, w.next()) {
            const int m = w.m, n = w.n;
            if (m != cur_m) {
                // split the new panel: row max over both K halves, then this thread's half
                cur_m = m;
                mbar_wait(smem_u32(a_full), loads & 1);
                loads++;
                float v[64];
                float mx = 0.0f;
                if (kh < nkc) {
                    f16_load_row(sA + kh * TC16_CH, row, v);
#pragma unroll
                    for (int i = 0; i < 64; i++) mx = fmaxf(mx, fabsf(v[i]));
                }
                rmax[kh * 128 + row] = mx;
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
                const int ea = f16_scale_exp(fmaxf(rmax[row], rmax[128 + row]));
                osc = ldexpf(1.0f, -(ea + bexp));
                if (kh < nkc) f16_store_row(sA + kh * TC16_CH, row, v, ldexpf(1.0f, ea));
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(a_conv)) : "memory");
            }
            const int ab = tc & 1;
            mbar_wait(smem_u32(t_full + ab), (tc >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const int m0 = m * TC_M, n0 = n * TC_N;
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * 2 * TC_N);
            uint32_t r[32], x[32];
            tmem_ld32(tbase + ch, r);
            tmem_ld32(tbase + TC_N + ch, x);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll 1
            for (int c0 = ch; c0 < ch + TC_N / 2; c0 += 32) {
                float *bb = buf;
                if (TMAST) {
                    // the store issued from this buffer two blocks ago has finished reading it
                    bb = buf + bsel * (32 * 32);
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; j++)
                    *(float4 *)(bb + lane * 32 + 4 * (j ^ (lane & 7))) =
                        make_float4((__uint_as_float(r[4 * j]) + __uint_as_float(x[4 * j])) * osc,
                                    (__uint_as_float(r[4 * j + 1]) + __uint_as_float(x[4 * j + 1])) * osc,
                                    (__uint_as_float(r[4 * j + 2]) + __uint_as_float(x[4 * j + 2])) * osc,
                                    (__uint_as_float(r[4 * j + 3]) + __uint_as_float(x[4 * j + 3])) * osc);
                if (c0 + 32 < ch + TC_N / 2) {
                    tmem_ld32(tbase + c0 + 32, r);
                    tmem_ld32(tbase + TC_N + c0 + 32, x);
                }
                if (TMAST) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(&tmC),
                            "r"(n0 + c0), "r"(mrow0 + m0 + lq * 32), "r"(smem_u32(bb))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                    }
                    bsel ^= 1u;
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
                    continue;
                }
                __syncwarp();
                const int nn = n0 + c0 + cq;
#pragma unroll 4
                for (int i = 0; i < 8; i++) {
                    const int rr = 4 * i + (lane >> 3);
                    const int grow = m0 + lq * 32 + rr;
                    if (grow < M && nn < N) {
                        const float4 v4 = *(const float4 *)(buf + rr * 32 + 4 * ((lane & 7) ^ (rr & 7)));
                        float *dst = C + (size_t)grow * ldc + nn;
                        if (nn + 4 <= N && (ldc & 3) == 0)
                            *(float4 *)dst = v4;
                        else {
                            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
                            for (int j = 0; j < 4 && nn + j < N; j++) dst[j] = vv[j];
                        }
                    }
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(t_empty + ab)) : "memory");
        }
        if (TMAST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- b2 = A S~: split-K, streamed A (k_tc_gemm_splitk's structure) ------------------
// A ring of NA stages (two TMA boxes of raw fp32 A each, split in place by warps 4-7, one
// row per thread, with the global scale 2^ea) and a separate ring of NB B chunks (pre-
// split fp16, one bulk copy each): A streams from HBM and wants the deeper ring, B comes
// from L2.  Warp 8 lane 0 produces A, warp 10 lane 0 produces B, warp 9 lane 0 issues 12
// MMAs per 64-wide chunk, warps 0-3 drain with the output scale 2^-(ea + bexp).  ea comes
// from the fixed-point bound vbmax max|w| (the device scalar *wmax the backward used).
// TMAST: the partials are stored by TMA tensor stores (tmC: a 3-D map over C as
// [nsplit][M][ldc], box 32 x 32 x 1, SWIZZLE_128B, so rows past M are clipped inside their
// split) from two 4 KB staging buffers per epilogue warp.
constexpr int TCS16_T = 352;
constexpr int tcs16_smem(bool tmast, int na, int nb) {
    return (na + nb) * TC16_CH + (tmast ? 4 * 2 * 32 * 32 * 4 : 4 * 32 * 33 * 4) + 1024 + 256;
}
template <bool TMAST, int NA, int NB>
__global__ void __launch_bounds__(TCS16_T, 1)
    k_tc_gemm_splitk16(const __grid_constant__ CUtensorMap tmA, int M, int N, int nkc, int cps, int nsplit, int mtiles,
                       const __half *__restrict__ Bt, float *__restrict__ C, int ldc, const int2 *__restrict__ trng,
                       int mreal, const float *__restrict__ wmax, float vbmax, int bexp,
                       const __grid_constant__ CUtensorMap tmC) {
    auto krange = [&](int z, int m, int &c0, int &c1) {
        c0 = z * cps;
        c1 = min(nkc, (z + 1) * cps);
        if (m >= mreal) {
            c1 = c0;
        } else if (trng) {
            const int2 r = trng[m];
            c0 = max(c0, r.x / TC16_KC);
            c1 = min(c1, (r.y + TC16_KC - 1) / TC16_KC);
        }
    };
    extern __shared__ __align__(1024) unsigned char s16_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)s16_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base, *sB = base + NA * TC16_CH;
    float *ebuf = (float *)(sB + NB * TC16_CH);
    uint64_t *bars = (uint64_t *)(ebuf + (TMAST ? 4 * 2 * 32 * 32 : 4 * 32 * 33));
    uint64_t *a_full = bars, *conv_full = bars + NA, *a_empty = bars + 2 * NA, *b_full = bars + 3 * NA,
             *b_empty = b_full + NB, *t_full = b_empty + NB, *t_empty = t_full + 2;
    uint32_t *tmem_slot = (uint32_t *)(t_empty + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nunits = nsplit * mtiles;
    const int u0 = (int)blockIdx.x, ustep = gridDim.x;
    // |A| <= vbmax max|w| (1 + 1e-2 for the bin rounding): the A scale
    const int ea = f16_scale_exp((float)((double)vbmax * (double)*wmax * 1.01));

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        for (int i = 0; i < NA; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(a_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;\n" ::"r"(smem_u32(conv_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(a_empty + i)));
        }
        for (int i = 0; i < NB; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b_empty + i)));
        }
        for (int i = 0; i < 2; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(t_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;\n" ::"r"(smem_u32(t_empty + i)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    if (tid == 256) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp == 8 || warp == 10) {
        // producers: warp 8 the A ring, warp 10 the B ring (the same chunk sequence)
        if (lane == 0) {
            const bool pa = warp == 8;
            const int ns = pa ? NA : NB;
            uint32_t cnt = 0;
            for (int u = u0; u < nunits; u += ustep) {
                const int z = u / mtiles, m = u % mtiles;
                int cA, c1;
                krange(z, m, cA, c1);
                for (int c = cA; c < c1; c++, cnt++) {
                    const int st = cnt % ns;
                    if (cnt >= (uint32_t)ns) {
                        mbar_wait(smem_u32((pa ? a_empty : b_empty) + st), ((cnt / ns) - 1) & 1);
                        // (A: the converters' generic writes into this stage precede the MMAs
                        // that released it; order them before the async-proxy refill)
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    }
                    const uint32_t mb = smem_u32((pa ? a_full : b_full) + st);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                                 "r"((uint32_t)TC16_CH)
                                 : "memory");
                    if (pa) {
                        unsigned char *sa = sA + st * TC16_CH;
                        for (int hb = 0; hb < 2; hb++)
                            asm volatile(
                                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
                                "{%2, %3}], [%4];\n" ::"r"(smem_u32(sa + hb * TC16_OPB)),
                                "l"(&tmA), "r"(c * TC16_KC + 32 * hb), "r"(m * TC_M), "r"(mb)
                                : "memory");
                    } else {
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                smem_u32(sB + st * TC16_CH)),
                            "l"(Bt + (size_t)c * (2 * TC_N * TC16_KC)), "r"((uint32_t)TC16_CH), "r"(mb)
                            : "memory");
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        const int row = tid - 128;
        const float sc = ldexpf(1.0f, ea);
        uint32_t cnt = 0;
        for (int u = u0; u < nunits; u += ustep) {
            const int z = u / mtiles, m = u % mtiles;
            int cA, c1;
            krange(z, m, cA, c1);
            for (int c = cA; c < c1; c++, cnt++) {
                const int st = cnt % NA;
                mbar_wait(smem_u32(a_full + st), (cnt / NA) & 1);
                unsigned char *sa = sA + st * TC16_CH;
                float v[64];
                f16_load_row(sa, row, v);
#if CACSI_CHECKS
                for (int i = 0; i < 64; i++) CACSI_CHECK(!(fabsf(v[i] * sc) >= 32768.0f));
#endif
                f16_store_row(sa, row, v, sc);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(conv_full + st)) : "memory");
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {
            const uint32_t idesc = tc_idesc_f16();
            uint32_t cnt = 0, uc = 0;
            for (int u = u0; u < nunits; u += ustep, uc++) {
                const int z = u / mtiles, m = u % mtiles;
                int c0, c1;
                krange(z, m, c0, c1);
                const int ab = uc & 1;
                if (uc >= 2) mbar_wait(smem_u32(t_empty + ab), ((uc >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t dmain = tmem + ab * 2 * TC_N, dcross = dmain + TC_N;
                for (int c = c0; c < c1; c++, cnt++) {
                    const int sa = cnt % NA, sb = cnt % NB;
                    mbar_wait(smem_u32(conv_full + sa), (cnt / NA) & 1);
                    mbar_wait(smem_u32(b_full + sb), (cnt / NB) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    const uint32_t ah0 = smem_u32(sA + sa * TC16_CH), al0 = ah0 + TC16_OPB;
                    const uint32_t bh0 = smem_u32(sB + sb * TC16_CH), bl0 = bh0 + TC16_OPB;
#pragma unroll
                    for (int ks = 0; ks < TC16_KC / 16; ks++) {
                        const uint32_t off = ks * 32;
                        const uint32_t accf = (c != c0 || ks != 0) ? 1u : 0u;
                        tc_mma16(dmain, tc_desc(ah0 + off), tc_desc(bh0 + off), idesc, accf);
                        tc_mma16(dcross, tc_desc(ah0 + off), tc_desc(bl0 + off), idesc, accf);
                        tc_mma16(dcross, tc_desc(al0 + off), tc_desc(bh0 + off), idesc, 1);
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                            smem_u32(a_empty + sa)));
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                            smem_u32(b_empty + sb)));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(t_full + ab)));
            }
        }
    } else if (warp < 4) {
        const float osc = ldexpf(1.0f, -(ea + bexp));
        float *buf = ebuf + warp * (TMAST ? 2 * 32 * 32 : 32 * 33);
        const int cq = 4 * (lane & 7);
        uint32_t uc = 0, bsel = 0;
        for (int u = u0; u < nunits; u += ustep, uc++) {
            const int z = u / mtiles, m = u % mtiles;
            int cA, cB;
            krange(z, m, cA, cB);
            const bool empty_unit = cB <= cA;
            const int ab = uc & 1;
            mbar_wait(smem_u32(t_full + ab), (uc >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            float *Cz = C + (size_t)z * M * ldc;
            const int m0 = m * TC_M;
#pragma unroll 1
            for (int c0 = 0; c0 < TC_N && c0 < N; c0 += 32) {
                uint32_t r[32], x[32];
                const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ab * 2 * TC_N + c0);
                tmem_ld32(taddr, r);
                tmem_ld32(taddr + TC_N, x);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n");
                if (TMAST) {
                    float *bb = buf + bsel * (32 * 32);
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (!empty_unit)
                            v4 = make_float4((__uint_as_float(r[4 * j]) + __uint_as_float(x[4 * j])) * osc,
                                             (__uint_as_float(r[4 * j + 1]) + __uint_as_float(x[4 * j + 1])) * osc,
                                             (__uint_as_float(r[4 * j + 2]) + __uint_as_float(x[4 * j + 2])) * osc,
                                             (__uint_as_float(r[4 * j + 3]) + __uint_as_float(x[4 * j + 3])) * osc);
                        *(float4 *)(bb + lane * 32 + 4 * (j ^ (lane & 7))) = v4;
                    }
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(&tmC),
                            "r"(c0), "r"(m0 + warp * 32), "r"(z), "r"(smem_u32(bb))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                    }
                    bsel ^= 1u;
                    continue;
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 32; j++)
                    buf[lane * 33 + j] = empty_unit ? 0.0f : (__uint_as_float(r[j]) + __uint_as_float(x[j])) * osc;
                __syncwarp();
                const int nn = c0 + cq;
#pragma unroll 4
                for (int i = 0; i < 8; i++) {
                    const int rr = 4 * i + (lane >> 3);
                    const int grow = m0 + warp * 32 + rr;
                    if (grow < M && nn < N) {
                        const float *br = buf + rr * 33 + cq;
                        float *dst = Cz + (size_t)grow * ldc + nn;
                        if (nn + 4 <= N && (ldc & 3) == 0)
                            *(float4 *)dst = make_float4(br[0], br[1], br[2], br[3]);
                        else
                            for (int j = 0; j < 4 && nn + j < N; j++) dst[j] = br[j];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(t_empty + ab)) : "memory");
        }
        if (TMAST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// Packing of B (N x K; element (n, kk) at B[n sn + kk sk]) into pre-split fp16 tiles
// [ceil(N / 128)][nkc][hi, lo][128 x 64] (tc_swz16 layout), scaled by 2^bexp.
__global__ void __launch_bounds__(256) k_tc_pack_b16(const float *__restrict__ B, int N, int K, int sn, int sk, int nkc,
                                                     __half *__restrict__ out, int bexp) {
    const int ntiles = (N + TC_N - 1) / TC_N;
    const size_t total = (size_t)ntiles * nkc * TC_N * TC16_KC;
    const float sc = ldexpf(1.0f, bexp);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % TC16_KC), r = (int)((i / TC16_KC) % TC_N);
        const size_t tc = i / (TC16_KC * TC_N);  // tile * nkc + chunk
        const int c = (int)(tc % nkc), nt = (int)(tc / nkc);
        const int n = nt * TC_N + r, kk = c * TC16_KC + k;
        const float x = ((n < N && kk < K) ? B[(size_t)n * sn + (size_t)kk * sk] : 0.0f) * sc;
        const __half h = __float2half_rn(x);
        unsigned char *tile = (unsigned char *)(out + tc * (2 * TC_N * TC16_KC));
        *(__half *)(tile + tc_swz16(r, k)) = h;
        *(__half *)(tile + TC16_OPB + tc_swz16(r, k)) = __float2half_rn(x - __half2float(h));
    }
}

}  // namespace cacsi
