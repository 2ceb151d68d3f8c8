// tcgemm.cuh -- fp32-accurate GEMM on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM) for the ESAI contractions
// over q (W = F S~^T, b2 = A S~).
//
//   C[z][M][ldc] = sum_{k in split z} A[M][lda] B[N][K]^T     (both operands K-major)
//
// 3xTF32: x = hi + lo with hi = x truncated to TF32 and lo = x - hi (exact in
// fp32); C = A_hi B_hi + (A_hi B_lo + A_lo B_hi) (relative error ~2^-21 per
// product).  The main and the cross terms accumulate in two separate TMEM
// accumulators (columns [0,128) and [128,256)), so the small cross terms do
// not add to the main accumulator's rounding count; the TMEM accumulation
// error still grows with the number of k-steps (measured ~6e-8 per
// accumulate), so long-K contractions are split (split-K partials are summed
// in fp64 by the caller).
//
// B is a CONSTANT of the geometry (S~ or S~^T): it is split into hi / lo once
// at create time and stored pre-swizzled as tiles [n_tile][k_chunk] of
// {hi 128x32, lo 128x32} fp32 (32 KB), so one cp.async.bulk per chunk lands it
// in shared memory.  A is split on the fly by the 128 threads (one row each).
//
// Shared-memory operand layout = canonical K-major SWIZZLE_128B: 8-row x
// 128-byte atoms (1 KB, 1024-aligned), 16-byte chunk index XOR (row % 8).
// Pipeline: 2 stages; chunk c+1's A loads and B bulk copy overlap chunk c's
// 12 MMAs (4 k-steps x 3 products, M = N = 128, K = 8), which one elected
// thread issues and commits to an mbarrier.  Epilogue: tcgen05.ld, warp w
// owns TMEM lanes (tile rows) 32w..32w+31.
#pragma once
#include <cuda.h>  // CUtensorMap (the encoder is fetched through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <stdint.h>

namespace cacsi {

constexpr int TC_M = 128, TC_N = 128, TC_KC = 32;   // tile and K chunk (32 fp32 = one 128-byte swizzle row)
constexpr int TC_T = 128;                            // threads
constexpr int TC_PSTRIDE = TC_N - 2;                 // column stride of the overlapping PAIRS tiles
constexpr int TC_OPB = TC_M * TC_KC * 4;             // bytes of one operand half-tile (16 KB)
constexpr int TC_STAGE = 4 * TC_OPB;                 // A_hi, A_lo, B_hi, B_lo
constexpr int TC_SMEM = 2 * TC_STAGE + 1024 + 128;   // 2 stages + alignment + barriers
constexpr int tc_smem(int stages) { return stages * TC_STAGE + 1024 + 128; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 "version 1"):
// start >> 4 in [0,14), LBO = 1 (16 B, unused for swizzled K-major), SBO = 1024 B
// between 8-row atoms, version 1 at bit 46, layout type 2 (SWIZZLE_128B) at bit 61.
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// instruction descriptor: D fp32, A/B TF32, both K-major, N = 128, M = 128
__host__ __device__ constexpr uint32_t tc_idesc_tf32() {
    return (1u << 4)                        // c_format F32
           | (2u << 7)                      // a_format TF32
           | (2u << 10)                     // b_format TF32
           | ((uint32_t)(TC_N >> 3) << 17)  // n_dim
           | ((uint32_t)(TC_M >> 4) << 24); // m_dim
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// byte offset of element (row, k) (k in [0, 32)) inside a 128 x 32 fp32 tile
__host__ __device__ __forceinline__ uint32_t tc_swz(int row, int k) {
    const int chunk = k >> 2;  // 16-byte chunk within the 128-byte row
    return (uint32_t)(row * 128 + (((chunk ^ (row & 7)) << 4) | ((k & 3) << 2)));
}

__host__ __device__ __forceinline__ float tf32_hi(float x) {
#ifdef __CUDA_ARCH__
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
#else
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
#endif
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
        "r"(phase)
        : "memory");  // no shared-memory access may move above the wait
}

// C[z] (rows < M, columns < N) = A * B^T over k-chunks [z * cps, min(nkc, (z+1) * cps)).
//   A: [M][lda] fp32, lda % 4 == 0, columns >= nkc * 32 read as zero beyond K
//   Bt: pre-split tiles [ntiles][nkc][2][128 x 32] (see tc_pack_b)
// PAIRS: tiles overlap by two columns (tile nt covers B rows 126 nt .. 126 nt + 127,
// tc_pack_b with stride TC_PSTRIDE = 126) and the epilogue writes C as float2
// pairs (C[m][n], C[m][n + 1]) for n < N - 1, 126 per tile (an even stride keeps
// every 2-pair store 16-byte aligned), so a consumer interpolating between
// neighbouring columns gathers one 8-byte entry (ldc in float2 units).
// STAGES = 2: chunk c+1's loads overlap chunk c's MMAs (long K); STAGES = 1:
// half the shared memory, so two CTAs share an SM and one CTA's epilogue
// overlaps the other's loads and MMAs (short K, store-heavy epilogue).
// A_PACKED: A is given as pre-split, pre-swizzled tiles [ceil(M/128)][nkc][hi, lo]
// (the layout of tc_pack_b, built on the device by k_tc_pack_a) and lands in
// shared memory by one cp.async.bulk per chunk like B -- the threads only run
// the epilogue.
template <bool PAIRS, int STAGES = 2, bool A_PACKED = false>
__global__ void __launch_bounds__(TC_T) k_tc_gemm(int M, int N, int K, int lda, int nkc, int cps,
                                                  const float *__restrict__ A, const float *__restrict__ Bt,
                                                  float *__restrict__ C, int ldc) {
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *bars = (uint64_t *)(base + STAGES * TC_STAGE);  // [0, S) B landed, [S, 2S) MMAs of stage done
    uint32_t *tmem_slot = (uint32_t *)(bars + 4);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int m0 = blockIdx.y * TC_M, nt = blockIdx.x, n0 = nt * (PAIRS ? TC_PSTRIDE : TC_N);
    const int kc0 = blockIdx.z * cps, kc1 = min(nkc, kc0 + cps);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        for (int i = 0; i < 2 * STAGES; i++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bars + i)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = tc_idesc_tf32();
    const int row = tid, gm = m0 + row;
    const float *arow = A + (size_t)(gm < M ? gm : 0) * (A_PACKED ? 0 : lda);

    for (int c = kc0; c < kc1; c++) {
        const int it = c - kc0, st = it % STAGES, use = it / STAGES;
        unsigned char *sA_hi = base + st * TC_STAGE, *sA_lo = sA_hi + TC_OPB, *sB = sA_hi + 2 * TC_OPB;
        // the MMAs that last read this stage (iteration it - STAGES) must be done
        if (it >= STAGES) mbar_wait(smem_u32(bars + STAGES + st), (use - 1) & 1);
        if (tid == 0) {
            const uint32_t mb = smem_u32(bars + st);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                         "r"((A_PACKED ? 4 : 2) * TC_OPB));
            const float *src = Bt + ((size_t)nt * nkc + c) * (2 * TC_M * TC_KC);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    smem_u32(sB)),
                "l"(src), "r"(2 * TC_OPB), "r"(mb)
                : "memory");
            if (A_PACKED) {
                const float *asrc = A + ((size_t)blockIdx.y * nkc + c) * (2 * TC_M * TC_KC);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        smem_u32(sA_hi)),
                    "l"(asrc), "r"(2 * TC_OPB), "r"(mb)
                    : "memory");
            }
        }
        if (!A_PACKED) {
            // A: this thread's row, 32 columns of chunk c, split into hi / lo
            const int k0 = c * TC_KC;
#pragma unroll
            for (int k4 = 0; k4 < TC_KC; k4 += 4) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (gm < M && k0 + k4 < K) v = __ldg((const float4 *)(arow + k0 + k4));
                const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                const uint32_t off = tc_swz(row, k4);
                *(float4 *)(sA_hi + off) = h;
                *(float4 *)(sA_lo + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
            }
            asm volatile("fence.proxy.async.shared::cta;\n");
        }
        __syncthreads();
        if (tid == 0) {
            mbar_wait(smem_u32(bars + st), use & 1);  // B tile landed
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t ah0 = smem_u32(sA_hi), al0 = smem_u32(sA_lo);
            const uint32_t bh0 = smem_u32(sB), bl0 = smem_u32(sB + TC_OPB);
#pragma unroll
            for (int ks = 0; ks < TC_KC / 8; ks++) {
                const uint32_t off = ks * 32;  // 8 tf32 = 32 bytes along K inside the swizzle row
                tc_mma(tmem, tc_desc(ah0 + off), tc_desc(bh0 + off), idesc, (it | ks) != 0);
                tc_mma(tmem + TC_N, tc_desc(ah0 + off), tc_desc(bl0 + off), idesc, (it | ks) != 0);
                tc_mma(tmem + TC_N, tc_desc(al0 + off), tc_desc(bh0 + off), idesc, 1);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(bars + STAGES + st)));
        }
    }
    // all MMAs done (the last commit covers every earlier MMA of this thread)
    const int nit = kc1 - kc0;
    if (nit > 0) mbar_wait(smem_u32(bars + STAGES + (nit - 1) % STAGES), ((nit - 1) / STAGES) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n");

    // ---- epilogue: TMEM -> registers -> global (warp w reads lanes 32w..32w+31)
    if (!PAIRS) {
        // each warp transposes its 32 rows x 32 columns through a [32][33] shared
        // buffer (conflict-free both ways) so that every store instruction writes
        // four 128-byte row segments (coalesced) instead of 32 scattered 16-byte
        // pieces.  The operand stages are free: every MMA has completed.
        float *Cz = C + (size_t)blockIdx.z * M * ldc;
        float *buf = (float *)base + warp * (32 * 33);
        const int lane = tid & 31;
        const int cq = 4 * (lane & 7);
#pragma unroll 1
        for (int c0 = 0; c0 < TC_N; c0 += 32) {
            uint32_t r[32], x[32];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
            tmem_ld32(taddr, r);
            tmem_ld32(taddr + TC_N, x);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; j++) buf[lane * 33 + j] = nit > 0 ? __uint_as_float(r[j]) + __uint_as_float(x[j]) : 0.0f;
            __syncwarp();
            const int n = n0 + c0 + cq;
#pragma unroll 4
            for (int i = 0; i < 8; i++) {
                const int rr = 4 * i + (lane >> 3);
                const int grow = m0 + warp * 32 + rr;
                if (grow < M && n < N) {
                    const float *br = buf + rr * 33 + cq;
                    float *dst = Cz + (size_t)grow * ldc + n;
                    if (n + 4 <= N && (ldc & 3) == 0) {
                        *(float4 *)dst = make_float4(br[0], br[1], br[2], br[3]);
                    } else {
                        for (int j = 0; j < 4 && n + j < N; j++) dst[j] = br[j];
                    }
                }
            }
        }
    } else {
        // pairs (v[c], v[c + 1]) for tile columns c = 0 .. 126.  Each warp
        // transposes its 32 rows x 32 columns through a [32][33] shared buffer
        // (conflict-free both ways; column 32 = the next chunk's first column)
        // so every store writes 32 consecutive pairs of ONE row (coalesced).
        // The operand stages are free: every MMA has completed (waited above).
        float2 *Cz = (float2 *)C + (size_t)blockIdx.z * M * ldc;
        float *buf = (float *)base + warp * (32 * 33);
        const int lane = tid & 31;
        float cur[32], nxt[32];
        auto load = [&](int c0, float (&v)[32]) {
            uint32_t r[32], x[32];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
            tmem_ld32(taddr, r);
            tmem_ld32(taddr + TC_N, x);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int j = 0; j < 32; j++) v[j] = nit > 0 ? __uint_as_float(r[j]) + __uint_as_float(x[j]) : 0.0f;
        };
        load(0, cur);
#pragma unroll 1
        for (int c0 = 0; c0 < TC_N; c0 += 32) {
            if (c0 + 32 < TC_N) load(c0 + 32, nxt);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; j++) buf[lane * 33 + j] = cur[j];
            buf[lane * 33 + 32] = c0 + 32 < TC_N ? nxt[0] : 0.0f;
            __syncwarp();
            // lane l: row 2 i + (l >> 4) of the pass, pairs jp, jp + 1 (jp = 2 (l & 15)):
            // one 16-byte store per lane, two 256-byte row segments per warp store
            const int jp = 2 * (lane & 15);
            const int n = n0 + c0 + jp;
            const bool ok0 = c0 + jp < TC_PSTRIDE && n + 1 < N;
            const bool ok1 = c0 + jp + 1 < TC_PSTRIDE && n + 2 < N;
#pragma unroll 4
            for (int i = 0; i < 16; i++) {
                const int rr = 2 * i + (lane >> 4);
                const int grow = m0 + warp * 32 + rr;
                if (grow < M && ok0) {
                    const float *br = buf + rr * 33 + jp;
                    float2 *dst = Cz + (size_t)grow * ldc + n;
                    if (ok1)
                        *(float4 *)dst = make_float4(br[0], br[1], br[1], br[2]);
                    else
                        *dst = make_float2(br[0], br[1]);
                }
            }
#pragma unroll
            for (int j = 0; j < 32; j++) cur[j] = nxt[j];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(2 * TC_N));
}

// ---- A-resident persistent GEMM (short K): C = A B^T with K <= 128 -------------
// The whole A panel of an M tile (nkc <= 4 chunks, hi + lo: <= 128 KB) stays in
// shared memory while the CTA walks its contiguous range of output tiles (M-major
// order: at most a few panel loads per CTA), so each output tile costs only its
// B panel in L2 -> SM traffic (the A + B reload of k_tc_gemm halved).  Warp
// roles: warp 4 lane 0 issues the bulk copies (A panels, B chunks into a 2-stage
// ring), warp 5 lane 0 issues the MMAs into one of two TMEM accumulator pairs
// (512 columns), warps 0-3 drain the other pair (tcgen05.ld -> transposed
// shared buffer -> coalesced row stores), so loads, MMAs and stores of
// consecutive tiles overlap.  Barriers: a_full / a_empty (panel), b_full /
// b_empty (ring), t_full / t_empty (accumulators).
constexpr int TCA_T1 = 320;  // k_tc_gemm_ar / _ar2: 8 epilogue warps
constexpr int TCA_T1R = 352; // k_tc_gemm_ar<NSB, true>: + warp 10, the A-panel converter
constexpr int tca_smem(int nkc, int nsb = 2) { return nkc * TC_STAGE / 2 + nsb * TC_STAGE / 2 + 8 * 32 * 33 * 4 + 1024 + 256; }
// Output tiles of k_tc_gemm_ar in M-major order, either all mtiles x ntiles or -- with
// a tile list (pre, ntr) -- only N tiles ntr[m].x .. ntr[m].y of each M tile (pre: the
// exclusive prefix count of listed tiles, pre[0] the base; the CTAs split the LISTED
// tiles evenly).  start(t) positions on the t-th tile of the walk, next() steps.
struct TileWalk {
    const int *pre;
    const int2 *ntr;
    int mtiles, ntiles, m, n;
    __device__ long long count() const { return pre ? (long long)(pre[mtiles] - pre[0]) : (long long)mtiles * ntiles; }
    __device__ void start(int t) {
        if (!pre) {
            m = t / ntiles;
            n = t % ntiles;
            return;
        }
        const int g = pre[0] + t;
        int lo = 0, hi = mtiles;  // the last m with pre[m] <= g (empty M tiles share their successor's prefix)
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= g) lo = mid; else hi = mid;
        }
        m = lo;
        n = ntr[m].x + (g - pre[m]);
    }
    __device__ void next() {
        if (!pre) {
            if (++n == ntiles) n = 0, m++;
            return;
        }
        if (++n > ntr[m].y) {
            do m++; while (m < mtiles && pre[m + 1] == pre[m]);
            if (m < mtiles) n = ntr[m].x;
        }
    }
};

// RAW: the A panel is loaded from the raw fp32 matrix by TMA tensor loads (tmA: rows
// x K, box 128 x 32, SWIZZLE_128B -- the operand layout; out-of-range rows and K
// columns land as zeros) into the hi slots, and warp 10 splits it in place (hi =
// TF32 truncation, lo = rest, the split k_tc_pack_a does), proxy-fences and arrives
// a_conv -- no separate pack pass.  mrow0: the first M tile's row in tmA.
template <int NSB, bool RAW = false>
__global__ void __launch_bounds__(RAW ? TCA_T1R : TCA_T1, 1)
    k_tc_gemm_ar(int M, int N, int nkc, int mtiles, int ntiles, const float *__restrict__ Ap,
                 const float *__restrict__ Bt, float *__restrict__ C, int ldc, const int *__restrict__ tpre,
                 const int2 *__restrict__ tntr, const __grid_constant__ CUtensorMap tmA, int mrow0) {
    extern __shared__ __align__(1024) unsigned char tca_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)tca_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;                              // [nkc][hi, lo] 32 KB each
    unsigned char *sB = sA + nkc * (TC_STAGE / 2);         // [NSB][hi, lo]
    float *ebuf = (float *)(sB + NSB * (TC_STAGE / 2));    // [8][32][33]
    uint64_t *bars = (uint64_t *)(ebuf + 8 * 32 * 33);
    uint64_t *a_full = bars, *a_empty = bars + 1, *b_full = bars + 2, *b_empty = bars + 2 + NSB,
             *t_full = bars + 2 + 2 * NSB, *t_empty = bars + 4 + 2 * NSB;
    uint64_t *a_conv = bars + 6 + 2 * NSB;  // RAW: the A panel split
    uint32_t *tmem_slot = (uint32_t *)(bars + 7 + 2 * NSB);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    TileWalk tw{tpre, tntr, mtiles, ntiles, 0, 0};
    const long long T = tw.count();
    const int t0 = (int)(T * blockIdx.x / gridDim.x), t1 = (int)(T * (blockIdx.x + 1) / gridDim.x);
    tw.start(t0);
    constexpr uint32_t CHB = TC_STAGE / 2;  // bytes of one hi + lo chunk (32 KB)

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        for (int i = 0; i < 7 + 2 * NSB; i++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bars + i)),
                         "r"(i >= 4 + 2 * NSB && i < 6 + 2 * NSB ? 8 : 1));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
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
                    if (RAW) {
                        // (the converter's generic writes of the previous panel were ordered
                        // before the MMAs that released it; the proxy fence orders them
                        // before these async-proxy writes)
                        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                                     "r"(nkc * (uint32_t)TC_OPB)
                                     : "memory");
                        for (int c = 0; c < nkc; c++)
                            asm volatile(
                                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
                                "{%2, %3}], [%4];\n" ::"r"(smem_u32(sA + c * CHB)),
                                "l"(&tmA), "r"(c * TC_KC), "r"(mrow0 + m * TC_M), "r"(mb)
                                : "memory");
                    } else {
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(nkc * CHB)
                                     : "memory");
                        for (int c = 0; c < nkc; c++)
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                    smem_u32(sA + c * CHB)),
                                "l"(Ap + ((size_t)m * nkc + c) * (2 * TC_M * TC_KC)), "r"(CHB), "r"(mb)
                                : "memory");
                    }
                    cur_m = m;
                    loads++;
                }
                for (int c = 0; c < nkc; c++, bc++) {
                    const int st = bc % NSB;
                    if (bc >= NSB) mbar_wait(smem_u32(b_empty + st), ((bc / NSB) - 1) & 1);
                    const uint32_t mb = smem_u32(b_full + st);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(CHB)
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(sB + st * CHB)),
                        "l"(Bt + ((size_t)n * nkc + c) * (2 * TC_N * TC_KC)), "r"(CHB), "r"(mb)
                        : "memory");
                }
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            const uint32_t idesc = tc_idesc_tf32();
            int cur_m = -1;
            uint32_t loads = 0, bc = 0, tc = 0;
            TileWalk w = tw;
            for (int t = t0; t < t1; t++, tc++) {
                const int m = w.m;
                w.next();  // w: the next tile (its M tile decides whether the A panel is released)
                if (m != cur_m) {
                    mbar_wait(smem_u32(RAW ? a_conv : a_full), loads & 1);
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
                    const uint32_t ah0 = smem_u32(sA + c * CHB), al0 = ah0 + TC_OPB;
                    const uint32_t bh0 = smem_u32(sB + st * CHB), bl0 = bh0 + TC_OPB;
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 8; ks++) {
                        const uint32_t off = ks * 32;
                        tc_mma(dmain, tc_desc(ah0 + off), tc_desc(bh0 + off), idesc, (c | ks) != 0);
                        tc_mma(dcross, tc_desc(ah0 + off), tc_desc(bl0 + off), idesc, (c | ks) != 0);
                        tc_mma(dcross, tc_desc(al0 + off), tc_desc(bh0 + off), idesc, 1);
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
    } else if (warp == 10) {
        // RAW only: split each landed A panel in place (position-independent: the hi and
        // lo slots share the swizzled layout), then release it to the MMA thread
        int cur_m = -1;
        uint32_t loads = 0;
        TileWalk w = tw;
        for (int t = t0; t < t1; t++, w.next()) {
            if (w.m == cur_m) continue;
            cur_m = w.m;
            mbar_wait(smem_u32(a_full), loads & 1);
            loads++;
            for (int c = 0; c < nkc; c++) {
                float4 *hi = (float4 *)(sA + c * CHB), *lo = (float4 *)(sA + c * CHB + TC_OPB);
                for (int i4 = lane; i4 < TC_OPB / 16; i4 += 32) {
                    const float4 v = hi[i4];
                    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                    hi[i4] = h;
                    lo[i4] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(a_conv)) : "memory");
        }
    } else {
        // epilogue warps 0-3 and 6-9: TMEM lanes 32 (warp % 4) .. + 31 = tile rows; warps
        // 0-3 drain columns 0-63, warps 6-9 columns 64-127
        const int ew = warp < 4 ? warp : warp - 2, lq = warp & 3, ch = warp < 4 ? 0 : TC_N / 2;
        float *buf = ebuf + ew * (32 * 33);
        const int cq = 4 * (lane & 7);
        uint32_t tc = 0;
        TileWalk w = tw;
        for (int t = t0; t < t1; t++, tc++, w.next()) {
            const int m = w.m, n = w.n;
            const int ab = tc & 1;
            mbar_wait(smem_u32(t_full + ab), (tc >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const int m0 = m * TC_M, n0 = n * TC_N;
            // software-pipelined drain: chunk c0 + 32's TMEM loads are in flight while
            // chunk c0 is transposed and stored
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * 2 * TC_N);
            uint32_t r[32], x[32];
            tmem_ld32(tbase + ch, r);
            tmem_ld32(tbase + TC_N + ch, x);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll 1
            for (int c0 = ch; c0 < ch + TC_N / 2; c0 += 32) {
                __syncwarp();
                // row `lane` of the 32 x 32 block as 8 float4, 16-byte chunk j at j ^ (lane & 7):
                // the stores (8 lanes span all 32 banks) and the row reads below are conflict-free
#pragma unroll
                for (int j = 0; j < 8; j++)
                    *(float4 *)(buf + lane * 32 + 4 * (j ^ (lane & 7))) =
                        make_float4(__uint_as_float(r[4 * j]) + __uint_as_float(x[4 * j]),
                                    __uint_as_float(r[4 * j + 1]) + __uint_as_float(x[4 * j + 1]),
                                    __uint_as_float(r[4 * j + 2]) + __uint_as_float(x[4 * j + 2]),
                                    __uint_as_float(r[4 * j + 3]) + __uint_as_float(x[4 * j + 3]));
                if (c0 + 32 < ch + TC_N / 2) {
                    tmem_ld32(tbase + c0 + 32, r);
                    tmem_ld32(tbase + TC_N + c0 + 32, x);
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
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- the same on CTA pairs (tcgen05 cta_group::2, M = 256 per pair) ----------
// A cluster of two CTAs on one TPC computes 256 x 128 output tiles: each CTA
// keeps ITS 128-row A panel resident and loads only HALF of each B chunk (64
// rows, 16 KB hi + lo), the leader's single thread issues the pair MMA
// (A rows from both CTAs' shared memory, B halves from both, each CTA's TMEM
// holding its 128 rows), so every SM moves half the B bytes of k_tc_gemm_ar
// and the B ring gets four stages.  Synchronisation across the pair: the
// follower's copies land on its own barriers and a forwarding thread re-arrives
// them on the leader's (pa_full, pb_full); MMA completion is committed to both
// CTAs' barriers by multicast; both epilogues arrive on the leader's t_empty.
constexpr int TCA2_NS = 4;
constexpr int TCA2_HB = TC_OPB / 2;  // one 64-row half of a 128 x 32 operand tile (8 KB)
constexpr int tca2_smem(int nkc) { return nkc * TC_STAGE / 2 + TCA2_NS * 2 * TCA2_HB + 8 * 32 * 33 * 4 + 1024 + 256; }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void remote_arrive(uint32_t local_bar, uint32_t rank) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}\n" ::"r"(local_bar),
        "r"(rank)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit2_mc(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
}
__host__ __device__ constexpr uint32_t tc_idesc_tf32_m256() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TCA_T1, 1)
    k_tc_gemm_ar2(int M, int N, int nkc, int mpairs, int ntiles, const float *__restrict__ Ap,
                  const float *__restrict__ Bt, float *__restrict__ C, int ldc) {
    extern __shared__ __align__(1024) unsigned char tca_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)tca_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;                                  // [nkc][hi, lo] 32 KB each
    unsigned char *sB = sA + nkc * (TC_STAGE / 2);             // [NS][hi, lo] 8 KB each
    float *ebuf = (float *)(sB + TCA2_NS * 2 * TCA2_HB);       // [8][32][33]
    uint64_t *bars = (uint64_t *)(ebuf + 8 * 32 * 33);
    uint64_t *a_full = bars, *a_empty = bars + 1, *pa_full = bars + 2, *t_full = bars + 3, *t_empty = bars + 5,
             *b_full = bars + 7, *b_empty = b_full + TCA2_NS, *pb_full = b_empty + TCA2_NS;
    uint32_t *tmem_slot = (uint32_t *)(pb_full + TCA2_NS);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const long long T = (long long)mpairs * ntiles;
    const int t0 = (int)(T * pair / npairs), t1 = (int)(T * (pair + 1) / npairs);
    constexpr uint32_t CHB = TC_STAGE / 2;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(a_full)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(a_empty)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(pa_full)));
        for (int i = 0; i < 2; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(t_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;\n" ::"r"(smem_u32(t_empty + i)));
        }
        for (int i = 0; i < TCA2_NS; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b_empty + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(pb_full + i)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        if (lane == 0) {
            int cur_mp = -1;
            uint32_t loads = 0, bc = 0;
            for (int t = t0; t < t1; t++) {
                const int mp = t / ntiles, n = t % ntiles;
                const int m = 2 * mp + (int)rank;
                if (mp != cur_mp) {
                    if (loads > 0) mbar_wait(smem_u32(a_empty), (loads - 1) & 1);
                    const uint32_t mb = smem_u32(a_full);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(nkc * CHB)
                                 : "memory");
                    for (int c = 0; c < nkc; c++)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                smem_u32(sA + c * CHB)),
                            "l"(Ap + ((size_t)m * nkc + c) * (2 * TC_M * TC_KC)), "r"(CHB), "r"(mb)
                            : "memory");
                    cur_mp = mp;
                    loads++;
                }
                for (int c = 0; c < nkc; c++, bc++) {
                    const int st = bc % TCA2_NS;
                    if (bc >= TCA2_NS) mbar_wait(smem_u32(b_empty + st), ((bc / TCA2_NS) - 1) & 1);
                    const uint32_t mb = smem_u32(b_full + st);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                                 "r"((uint32_t)(2 * TCA2_HB))
                                 : "memory");
                    const float *src = Bt + ((size_t)n * nkc + c) * (2 * TC_N * TC_KC) + rank * (TC_N / 2) * TC_KC;
                    unsigned char *dst = sB + st * 2 * TCA2_HB;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(dst)),
                        "l"(src), "r"((uint32_t)TCA2_HB), "r"(mb)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(dst + TCA2_HB)),
                        "l"(src + TC_N * TC_KC), "r"((uint32_t)TCA2_HB), "r"(mb)
                        : "memory");
                }
            }
        }
    } else if (warp == 5) {
        if (lane == 0 && rank == 1) {
            // forwarder: this CTA's panel / chunk landed -> the leader's pa_full / pb_full
            int cur_mp = -1;
            uint32_t loads = 0, bc = 0;
            for (int t = t0; t < t1; t++) {
                const int mp = t / ntiles;
                if (mp != cur_mp) {
                    mbar_wait(smem_u32(a_full), loads & 1);
                    remote_arrive(smem_u32(pa_full), 0);
                    loads++;
                    cur_mp = mp;
                }
                for (int c = 0; c < nkc; c++, bc++) {
                    const int st = bc % TCA2_NS;
                    mbar_wait(smem_u32(b_full + st), (bc / TCA2_NS) & 1);
                    remote_arrive(smem_u32(pb_full + st), 0);
                }
            }
        } else if (lane == 0 && rank == 0) {
            const uint32_t idesc = tc_idesc_tf32_m256();
            int cur_mp = -1;
            uint32_t loads = 0, bc = 0, tc = 0;
            for (int t = t0; t < t1; t++, tc++) {
                const int mp = t / ntiles;
                if (mp != cur_mp) {
                    mbar_wait(smem_u32(a_full), loads & 1);
                    mbar_wait_cl(smem_u32(pa_full), loads & 1);
                    loads++;
                    cur_mp = mp;
                }
                const int ab = tc & 1;
                if (tc >= 2) mbar_wait_cl(smem_u32(t_empty + ab), ((tc >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t dmain = tmem + ab * 2 * TC_N, dcross = dmain + TC_N;
                for (int c = 0; c < nkc; c++, bc++) {
                    const int st = bc % TCA2_NS;
                    mbar_wait(smem_u32(b_full + st), (bc / TCA2_NS) & 1);
                    mbar_wait_cl(smem_u32(pb_full + st), (bc / TCA2_NS) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    const uint32_t ah0 = smem_u32(sA + c * CHB), al0 = ah0 + TC_OPB;
                    const uint32_t bh0 = smem_u32(sB + st * 2 * TCA2_HB), bl0 = bh0 + TCA2_HB;
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 8; ks++) {
                        const uint32_t off = ks * 32;
                        tc_mma2(dmain, tc_desc(ah0 + off), tc_desc(bh0 + off), idesc, (c | ks) != 0);
                        tc_mma2(dcross, tc_desc(ah0 + off), tc_desc(bl0 + off), idesc, (c | ks) != 0);
                        tc_mma2(dcross, tc_desc(al0 + off), tc_desc(bh0 + off), idesc, 1);
                    }
                    tc_commit2_mc(smem_u32(b_empty + st));
                }
                tc_commit2_mc(smem_u32(t_full + ab));
                if (t + 1 == t1 || (t + 1) / ntiles != mp) tc_commit2_mc(smem_u32(a_empty));
            }
        }
    } else {
        // epilogue warps 0-3 and 6-9 (as in k_tc_gemm_ar): TMEM lanes 32 (warp % 4) ..,
        // warps 0-3 drain columns 0-63, warps 6-9 columns 64-127
        const int ew = warp < 4 ? warp : warp - 2, lq = warp & 3, ch = warp < 4 ? 0 : TC_N / 2;
        float *buf = ebuf + ew * (32 * 33);
        const int cq = 4 * (lane & 7);
        uint32_t tc = 0;
        for (int t = t0; t < t1; t++, tc++) {
            const int mp = t / ntiles, n = t % ntiles;
            const int ab = tc & 1;
            mbar_wait(smem_u32(t_full + ab), (tc >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const int m0 = (2 * mp + (int)rank) * TC_M, n0 = n * TC_N;
            const uint32_t tbase = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(ab * 2 * TC_N);
            uint32_t r[32], x[32];
            tmem_ld32(tbase + ch, r);
            tmem_ld32(tbase + TC_N + ch, x);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll 1
            for (int c0 = ch; c0 < ch + TC_N / 2; c0 += 32) {
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; j++)
                    *(float4 *)(buf + lane * 32 + 4 * (j ^ (lane & 7))) =
                        make_float4(__uint_as_float(r[4 * j]) + __uint_as_float(x[4 * j]),
                                    __uint_as_float(r[4 * j + 1]) + __uint_as_float(x[4 * j + 1]),
                                    __uint_as_float(r[4 * j + 2]) + __uint_as_float(x[4 * j + 2]),
                                    __uint_as_float(r[4 * j + 3]) + __uint_as_float(x[4 * j + 3]));
                if (c0 + 32 < ch + TC_N / 2) {
                    tmem_ld32(tbase + c0 + 32, r);
                    tmem_ld32(tbase + TC_N + c0 + 32, x);
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
            if (lane == 0) remote_arrive(smem_u32(t_empty + ab), 0);  // the leader's (rank 0: its own)
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- split-K GEMM with a streamed fp32 A (long K): C[z] = A B^T over split z --
// For b2 = A S~ (A: n_vox x ldw fp32, written by the backward; B = S~^T packed).
// Persistent CTAs walk units (split z, M tile) -- consecutive units share z, so
// concurrently running CTAs read the same B chunks from L2.  Warp roles:
//   warp 8 lane 0: producer -- per K chunk, a TMA tensor load of the raw fp32 A
//     tile (128 rows x 32, SWIZZLE_128B: the MMA operand layout) into the stage's
//     A_hi slot and one cp.async.bulk of the pre-split B chunk (load_full);
//   warps 4-7: split the A tile in place (hi = TF32 truncation, lo = rest into
//     A_lo; one row per thread), proxy fence, arrive conv_full;
//   warp 9 lane 0: 12 MMAs per chunk into one of two TMEM accumulator pairs,
//     commit -> empty (stage free) and, after a unit's last chunk, -> t_full;
//   warps 0-3: drain the accumulator pair (transposed, coalesced stores of the
//     fp32 partial), arrive t_empty.
constexpr int TCS_T = 320, TCS_NS = 3;
constexpr int tcs_smem() { return TCS_NS * TC_STAGE + 4 * 32 * 33 * 4 + 1024 + 256; }
__global__ void __launch_bounds__(TCS_T, 1) k_tc_gemm_splitk(const __grid_constant__ CUtensorMap tmA, int M, int N,
                                                             int nkc, int cps, int nsplit, int mtiles,
                                                             const float *__restrict__ Bt, float *__restrict__ C,
                                                             int ldc, const int2 *__restrict__ trng, int mreal) {
    // the K chunks of unit (z, m): the split's range cut to the tile's column range
    // (trng, optional: A is written only there); tiles m >= mreal are empty
    auto krange = [&](int z, int m, int &c0, int &c1) {
        c0 = z * cps;
        c1 = min(nkc, (z + 1) * cps);
        if (m >= mreal) {
            c1 = c0;
        } else if (trng) {
            const int2 r = trng[m];
            c0 = max(c0, r.x / TC_KC);
            c1 = min(c1, (r.y + TC_KC - 1) / TC_KC);
        }
    };
    extern __shared__ __align__(1024) unsigned char tcs_raw[];
    unsigned char *base = (unsigned char *)(((uintptr_t)tcs_raw + 1023) & ~(uintptr_t)1023);
    float *ebuf = (float *)(base + TCS_NS * TC_STAGE);
    uint64_t *bars = (uint64_t *)(ebuf + 4 * 32 * 33);
    uint64_t *load_full = bars, *conv_full = bars + TCS_NS, *empty = bars + 2 * TCS_NS, *t_full = bars + 3 * TCS_NS,
             *t_empty = t_full + 2;
    uint32_t *tmem_slot = (uint32_t *)(t_empty + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nunits = nsplit * mtiles;
    const int u0 = (int)blockIdx.x, ustep = gridDim.x;  // this CTA's units: u0, u0 + ustep, ...

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) {
        for (int i = 0; i < TCS_NS; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(load_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;\n" ::"r"(smem_u32(conv_full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(empty + i)));
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

    if (warp == 8) {
        if (lane == 0) {
            uint32_t cnt = 0;
            for (int u = u0; u < nunits; u += ustep) {
                const int z = u / mtiles, m = u % mtiles;
                int cA, c1;
                krange(z, m, cA, c1);
                for (int c = cA; c < c1; c++, cnt++) {
                    const int st = cnt % TCS_NS;
                    if (cnt >= TCS_NS) mbar_wait(smem_u32(empty + st), ((cnt / TCS_NS) - 1) & 1);
                    unsigned char *sa = base + st * TC_STAGE;
                    const uint32_t mb = smem_u32(load_full + st);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                                 "r"((uint32_t)(3 * TC_OPB))
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                        "[%4];\n" ::"r"(smem_u32(sa)),
                        "l"(&tmA), "r"(c * TC_KC), "r"(m * TC_M), "r"(mb)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                            smem_u32(sa + 2 * TC_OPB)),
                        "l"(Bt + (size_t)c * (2 * TC_N * TC_KC)), "r"((uint32_t)(2 * TC_OPB)), "r"(mb)
                        : "memory");
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        const int row = tid - 128;
        uint32_t cnt = 0;
        for (int u = u0; u < nunits; u += ustep) {
            const int z = u / mtiles, m = u % mtiles;
            int cA, c1;
            krange(z, m, cA, c1);
            for (int c = cA; c < c1; c++, cnt++) {
                const int st = cnt % TCS_NS;
                mbar_wait(smem_u32(load_full + st), (cnt / TCS_NS) & 1);
                unsigned char *sa = base + st * TC_STAGE;
#pragma unroll
                for (int k4 = 0; k4 < TC_KC; k4 += 4) {
                    const uint32_t off = tc_swz(row, k4);
                    const float4 v = *(const float4 *)(sa + off);
                    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                    *(float4 *)(sa + off) = h;
                    *(float4 *)(sa + TC_OPB + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(conv_full + st)) : "memory");
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {
            const uint32_t idesc = tc_idesc_tf32();
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
                    const int st = cnt % TCS_NS;
                    mbar_wait(smem_u32(conv_full + st), (cnt / TCS_NS) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    const uint32_t ah0 = smem_u32(base + st * TC_STAGE), al0 = ah0 + TC_OPB;
                    const uint32_t bh0 = ah0 + 2 * TC_OPB, bl0 = ah0 + 3 * TC_OPB;
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 8; ks++) {
                        const uint32_t off = ks * 32;
                        const uint32_t accf = (c != c0 || ks != 0) ? 1u : 0u;
                        tc_mma(dmain, tc_desc(ah0 + off), tc_desc(bh0 + off), idesc, accf);
                        tc_mma(dcross, tc_desc(ah0 + off), tc_desc(bl0 + off), idesc, accf);
                        tc_mma(dcross, tc_desc(al0 + off), tc_desc(bh0 + off), idesc, 1);
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                            smem_u32(empty + st)));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(t_full + ab)));
            }
        }
    } else {
        // warps 0-3: TMEM lanes 32 warp .. 32 warp + 31 = tile rows
        float *buf = ebuf + warp * (32 * 33);
        const int cq = 4 * (lane & 7);
        uint32_t uc = 0;
        for (int u = u0; u < nunits; u += ustep, uc++) {
            const int z = u / mtiles, m = u % mtiles;
            int cA, cB;
            krange(z, m, cA, cB);
            const bool empty_unit = cB <= cA;  // no MMA wrote the accumulator: store zeros
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
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 32; j++)
                    buf[lane * 33 + j] = empty_unit ? 0.0f : __uint_as_float(r[j]) + __uint_as_float(x[j]);
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
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// Device: pack A (M x K, row-major, lda) into the tile layout of tc_pack_b
// (rows zero-padded to a multiple of 128, K to nkc * 32): one thread per element.
__global__ void k_tc_pack_a(const float *__restrict__ A, int M, int K, int lda, int nkc, float *__restrict__ out) {
    const size_t n = (size_t)((M + TC_M - 1) / TC_M) * nkc * TC_M * TC_KC;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % TC_KC);
        const int r = (int)((i / TC_KC) % TC_M);
        const size_t tile = i / ((size_t)TC_M * TC_KC);  // mt * nkc + c
        const int c = (int)(tile % nkc);
        const int m = (int)(tile / nkc) * TC_M + r, kk = c * TC_KC + k;
        const float x = (m < M && kk < K) ? A[(size_t)m * lda + kk] : 0.0f;
        const float h = tf32_hi(x);
        unsigned char *t = (unsigned char *)(out + tile * (2 * TC_M * TC_KC));
        *(float *)(t + tc_swz(r, k)) = h;
        *(float *)(t + TC_OPB + tc_swz(r, k)) = x - h;
    }
}

// Packing of B (N x K) into pre-split swizzled tiles [ntiles][nkc][hi, lo][128 x 32] (k_tc_pack_b
// above, on the device at create): stride = TC_N (disjoint tiles) or TC_PSTRIDE (overlapping
// tiles of k_tc_gemm<true>); ntiles = ceil(N / 128) resp. ceil((N - 1) / TC_PSTRIDE).
inline int tc_ntiles(int N, int stride) { return stride == TC_N ? (N + TC_N - 1) / TC_N : (N - 1 + stride - 1) / stride; }
// (PAIRS tiles: pairs n = 0 .. N - 2, stride TC_PSTRIDE per tile)

// Device version of tc_pack_b: element (n, kk) of B read at B[n * sn + kk * sk] (sn = ldb,
// sk = 1 for row-major B; sn = 1, sk = ld for B given transposed), one thread per packed
// element pair (hi, lo); the same tf32 truncation and exact subtraction as the host's.
__global__ void __launch_bounds__(256) k_tc_pack_b(const float *__restrict__ B, int N, int K, int sn, int sk,
                                                   int nkc, float *__restrict__ out, int stride) {
    const int ntiles = stride == TC_N ? (N + TC_N - 1) / TC_N : (N - 1 + stride - 1) / stride;
    const size_t total = (size_t)ntiles * nkc * TC_N * TC_KC;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % TC_KC), r = (int)((i / TC_KC) % TC_N);
        const size_t tc = i / (TC_KC * TC_N);  // tile * nkc + chunk
        const int c = (int)(tc % nkc), nt = (int)(tc / nkc);
        const int n = nt * stride + r, kk = c * TC_KC + k;
        const float x = (n < N && kk < K) ? B[(size_t)n * sn + (size_t)kk * sk] : 0.0f;
        const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        unsigned char *tile = (unsigned char *)(out + tc * (2 * TC_N * TC_KC));
        *(float *)(tile + tc_swz(r, k)) = h;
        *(float *)(tile + TC_OPB + tc_swz(r, k)) = x - h;
    }
}

}  // namespace cacsi
