// operators.cu -- forward g = A f and backward b = A^T w (SURVEY.md §8 rows
// a3, a4), direct per-term SIMT path for both detector modes.
//
// Forward (PAPER.md:129-153 computes the same sum): output-stationary, one
// thread per detector pixel, voxels streamed in chunks whose q-profiles are
// staged in shared memory as a zero-padded hat table (value at the midpoint,
// slope) so each energy term is one LDS.64 + two FMAs; no atomics.  Voxels
// are split across CTAs (split-K) and the partial images are summed in fp64
// in a fixed order by a second kernel (deterministic).
//
// Backward: voxel-stationary, one CTA per voxel gathering
// over its whole detector footprint; each thread owns a private column of a
// [nq+4][threads] shared-memory histogram (bank = lane, conflict-free, no
// atomics); the columns are summed in fp64 at the end.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "pair.cuh"

namespace cacsi {

static inline float __uint_as_float_host(unsigned u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

namespace {

constexpr int FWD_T = 128;  // pixels per CTA
constexpr int FWD_VC = 16;  // voxels per shared-memory chunk
constexpr int FWD_KU = 8;   // energies per iteration of the resolving forward (ILP)
constexpr int BWD_T = 128;  // threads per voxel CTA
constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- forward --
template <bool RES>
__global__ void __launch_bounds__(FWD_T) k_forward(const Params p, const float *__restrict__ f, int vox_per_split,
                                                   void *__restrict__ partial) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne, Q3 = Q + 3;
    // energy rows padded so that every unrolled batch stays inside: a batch starts at most
    // at whi <= K - 1 and reads FWD_KU (+ 1 for the even start of the pair layout) rows
    const int K4 = (K + 2 * FWD_KU) / FWD_KU * FWD_KU;
    float2 *en = (float2 *)smem4;          // [K4] (alpha_k, c_k), padded with copies of the last energy
    float2 *tab = en + K4;                 // [VC][Q + 3] (mid, slope), entry n at index n + 2
    // RES: accumulators as energy pairs [K4 / 2][FWD_T] float2 (one 8-byte read-modify-write per two
    // terms), alpha_k [K4] padded with 1e30 (a padding energy's u clamps onto the zero entry)
    float2 *acc2 = (float2 *)(tab + FWD_VC * Q3 + (FWD_VC * Q3 & 1));
    float *alpha = (float *)(acc2 + (RES ? (K4 / 2) * FWD_T : 0));
    const int tid = threadIdx.x;
    const int pix = blockIdx.x * FWD_T + tid;
    const bool valid = pix < p.n_det;
    const float2 d = p.det[valid ? pix : 0];
    const int v0 = blockIdx.y * vox_per_split;
    const int v1 = min(p.n_vox, v0 + vox_per_split);
    for (int k = tid; k < K4; k += FWD_T) en[k] = p.energy[min(k, K - 1)];
    if (RES) {
        for (int k = tid; k < K4; k += FWD_T) alpha[k] = k < K ? p.energy[k].x : 1e30f;
        for (int k = 0; k < K4 / 2; k++) acc2[k * FWD_T + tid] = make_float2(0.0f, 0.0f);
    }
    double tot = 0.0;
    for (int c0 = v0; c0 < v1; c0 += FWD_VC) {
        const int nc = min(FWD_VC, v1 - c0);
        __syncthreads();
        for (int i = tid; i < nc * Q3; i += FWD_T) {
            const int vv = i / Q3, n = i - vv * Q3 - 2;
            const float *fr = f + (size_t)(c0 + vv) * Q;
            const float a = (n >= 0 && n < Q) ? fr[n] : 0.0f;
            const float b = (n + 1 >= 0 && n + 1 < Q) ? fr[n + 1] : 0.0f;
            tab[i] = make_float2(0.5f * (a + b), b - a);
        }
        __syncthreads();
        float csum = 0.0f;
        for (int vv = 0; vv < nc; vv++) {
            const int v = c0 + vv;
            const VoxelRec vr = p.vox[v];
            const bool open = valid && mask_open(p, v, pix, vr, d);
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if (open) {
                pair_geom(p, vr, d, P, sh);
                k_range(p, sh, klo, khi);
            }
            const int wlo = __reduce_min_sync(FULL, klo);
            const int whi = __reduce_max_sync(FULL, khi);
            const float2 *tv = tab + vv * Q3 + 2;
            if (!RES) {
                float ap = 0.0f;  // sum_k c_k f~(u_k) of this pair
                for (int k = wlo; k <= whi; k++) {
                    const float2 e = en[k];
                    float tt;
                    const int n = hat_coord(p, e.x, sh, tt);
                    CACSI_CHECK(n >= -2 && n <= Q);
                    const float2 t = tv[n];
                    ap = fmaf(e.y, fmaf(tt, t.y, t.x), ap);
                }
                csum = fmaf(P, ap, csum);
            } else {
                // FWD_KU energies per iteration: their accumulator and table loads
                // are independent (no read-after-write through shared memory
                // between them), so their latencies overlap; the accumulator
                // rows are padded to a multiple of FWD_KU (acc_s has K4 rows)
                for (int k = wlo & ~1; k <= whi; k += FWD_KU) {
                    // energies past the lanes' windows (and the padding) land on the zero
                    // entries of the clamped hat table: no predicate needed
                    float tt[FWD_KU];
                    float2 t[FWD_KU], a[FWD_KU / 2];
#pragma unroll
                    for (int j = 0; j < FWD_KU; j++) {
                        const int n = hat_coord(p, alpha[k + j], sh, tt[j]);
                        CACSI_CHECK(n >= -2 && n <= Q && k + j < K4);
                        t[j] = tv[n];
                    }
#pragma unroll
                    for (int j = 0; j < FWD_KU / 2; j++) a[j] = acc2[((k >> 1) + j) * FWD_T + tid];
#pragma unroll
                    for (int j = 0; j < FWD_KU / 2; j++) {
                        a[j].x = fmaf(P, fmaf(tt[2 * j], t[2 * j].y, t[2 * j].x), a[j].x);
                        a[j].y = fmaf(P, fmaf(tt[2 * j + 1], t[2 * j + 1].y, t[2 * j + 1].x), a[j].y);
                        acc2[((k >> 1) + j) * FWD_T + tid] = a[j];
                    }
                }
            }
        }
        tot += (double)csum;
    }
    if (!RES) {
        if (valid) ((double *)partial)[(size_t)blockIdx.y * p.n_det + pix] = tot;
    } else {
        __syncthreads();
        // coalesced store of this CTA's [pixels][K] block, scaled by c_k
        float *out = (float *)partial + ((size_t)blockIdx.y * p.n_det + (size_t)blockIdx.x * FWD_T) * K;
        const int npx = min(FWD_T, p.n_det - (int)blockIdx.x * FWD_T);
        for (int i = tid; i < npx * K; i += FWD_T) {
            const int px = i / K, k = i - px * K;
            const float2 a2 = acc2[(k >> 1) * FWD_T + px];
            out[i] = en[k].y * ((k & 1) ? a2.y : a2.x);
        }
    }
}

// Energy-resolving forward with the per-pixel energy sums in REGISTERS: acc[KR] (KR >= ne, a
// multiple of 8, fully unrolled), alpha_k as compile-time-indexed kernel parameters
// (constant-bank operands), energy blocks of 8 outside the warp's window union skipped by a
// warp-uniform branch.  The same arithmetic in the same order per (pixel, energy) as
// k_forward<true> (acc = fmaf(P, hat, acc) voxel by voxel), without its shared-memory
// read-modify-write per two terms, and with the hat interpolant tabulated as (c0, slope)
// (f~ = c0_n + u' slope_n: one FFMA, no fraction; not bit-identical to the (mid, slope)
// form, within ~1e-6 per term); the final [pixels][ne] block is staged through shared
// memory for coalesced stores.  Option er_fwd_reg.
constexpr int KR_MAX = 128;
__device__ __forceinline__ float2 lds2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}
struct AlphaTab {
    float a[KR_MAX];  // alpha_k for k < ne, 1e30 (clamps onto the zero table entry) beyond
};
template <int KR>
__global__ void __launch_bounds__(FWD_T, 3) k_forward_reg(const Params p, const float *__restrict__ f,
                                                          int vox_per_split, float *__restrict__ partial,
                                                          const AlphaTab at, int nlo, int QR) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne;
    // [VC][QR] (mid, slope), entry n at index n + nlo (n = -nlo .. Q): nlo covers u' down to
    // -q_min/dq - 1/2 (sin(theta/2) >= 0), so only the upper clamp is needed; reused to stage the output
    float2 *tab = (float2 *)smem4;
    const int tid = threadIdx.x;
    const int pix = blockIdx.x * FWD_T + tid;
    const bool valid = pix < p.n_det;
    const float2 d = p.det[valid ? pix : 0];
    const int v0 = blockIdx.y * vox_per_split;
    const int v1 = min(p.n_vox, v0 + vox_per_split);
    float acc[KR];
#pragma unroll
    for (int k = 0; k < KR; k++) acc[k] = 0.0f;
    for (int c0 = v0; c0 < v1; c0 += FWD_VC) {
        const int nc = min(FWD_VC, v1 - c0);
        __syncthreads();
        for (int i = tid; i < nc * QR; i += FWD_T) {
            const int vv = i / QR, n = i - vv * QR - nlo;
            const float *fr = f + (size_t)(c0 + vv) * Q;
            const float a = (n >= 0 && n < Q) ? fr[n] : 0.0f;
            const float b = (n + 1 >= 0 && n + 1 < Q) ? fr[n + 1] : 0.0f;
            // (c0, slope): f~(u) = c0_n + u' slope_n on [n - 1/2, n + 1/2) of u' = u - 1/2, with
            // c0_n = mid_n - n slope_n (one rounding, in fp64): one FFMA per term, no fraction
            tab[i] = make_float2((float)(0.5 * ((double)a + (double)b) - (double)n * ((double)b - (double)a)), b - a);
        }
        __syncthreads();
        for (int vv = 0; vv < nc; vv++) {
            const int v = c0 + vv;
            const VoxelRec vr = p.vox[v];
            const bool open = valid && mask_open(p, v, pix, vr, d);
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if (open) {
                pair_geom(p, vr, d, P, sh);
                k_range(p, sh, klo, khi);
            }
            const int wlo = __reduce_min_sync(FULL, klo);
            const int whi = __reduce_max_sync(FULL, khi);
            // byte address of entry n of this voxel's row, folded with the magic constant's bits:
            // entry(n) = tb + 8 * bits(n + 1.5 * 2^23)  (one LEA per term)
            uint32_t tb = (uint32_t)__cvta_generic_to_shared(tab + vv * QR + nlo) - (uint32_t)kMagicBits * 8u;
            tb = __shfl_sync(FULL, tb, 0);  // a per-lane register for ptxas: keeps the folded base (LEA per term)
#pragma unroll
            for (int kb = 0; kb < KR; kb += 8) {
                if (kb + 8 <= wlo || kb > whi) continue;  // warp-uniform
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    // u' = u - 1/2 >= -q_min/dq - 1/2 needs no lower clamp (entries down to -nlo are zero)
                    const float u = fminf(fmaf(at.a[kb + j], sh, p.nb), p.qm);
                    const float vm = u + kMagic;
                    CACSI_CHECK(__float_as_int(vm) - kMagicBits >= -nlo && __float_as_int(vm) - kMagicBits <= Q);
                    const float2 t = lds2(tb + ((uint32_t)__float_as_int(vm) << 3));
                    acc[kb + j] = fmaf(P, fmaf(u, t.y, t.x), acc[kb + j]);
                }
            }
        }
    }
    // [pixels][K] block of this CTA through shared memory (coalesced stores), scaled by c_k
    float *stage = (float *)smem4;
    const int npx = min(FWD_T, p.n_det - (int)blockIdx.x * FWD_T);
    float *out = partial + ((size_t)blockIdx.y * p.n_det + (size_t)blockIdx.x * FWD_T) * K;
    for (int kb = 0; kb < KR; kb += 32) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; j++)
            if (kb + j < KR) stage[j * (FWD_T + 1) + tid] = acc[kb + j];
        __syncthreads();
        const int kn = min(32, K - kb);
        for (int i = tid; i < npx * kn; i += FWD_T) {
            const int px = i / kn, k = i - px * kn;
            out[(size_t)px * K + kb + k] = p.energy[kb + k].y * stage[k * (FWD_T + 1) + px];
        }
    }
}

constexpr int FWL_VC = 32;  // voxels per staged chunk of k_forward_lane (a 32-bit open mask per lane)
// The register forward with PER-LANE voxel streams (option er_fwd_lane, default): lanes stay
// pixels with their KR energy sums in registers, but within each staged chunk of FWD_VC voxels a
// lane walks only ITS open voxels (a 16-bit mask of mask tests), so a step costs one open pair
// per busy lane instead of one voxel for all 32 lanes with about half of them closed (config 4:
// ~0.6 instead of ~0.45 useful lane-slots, and the pair geometry only for open pairs).  Each lane
// reads its own voxel's row of the (c0, slope) table (row stride QR odd: rows start on different
// banks); the warp's energy blocks span the union of its lanes' windows.  Same per-term arithmetic
// as k_forward_reg; the order of the voxels in each pixel's sum is unchanged (increasing v).
template <int KR>
__global__ void __launch_bounds__(FWD_T, 3) k_forward_lane(const Params p, const float *__restrict__ f,
                                                           int vox_per_split, float *__restrict__ partial,
                                                           const AlphaTab at, int nlo, int QR) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne;
    float2 *tab = (float2 *)smem4;                          // [VC][QR] (c0, slope); reused to stage the output
    VoxelRec *svox = (VoxelRec *)(tab + ((FWL_VC * QR + 1) & ~1));  // [VC]
    const int tid = threadIdx.x;
    const int pix = blockIdx.x * FWD_T + tid;
    const bool valid = pix < p.n_det;
    const float2 d = p.det[valid ? pix : 0];
    const int v0 = blockIdx.y * vox_per_split;
    const int v1 = min(p.n_vox, v0 + vox_per_split);
    const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(tab + nlo) - (uint32_t)kMagicBits * 8u;
    float acc[KR];
#pragma unroll
    for (int k = 0; k < KR; k++) acc[k] = 0.0f;
    for (int c0 = v0; c0 < v1; c0 += FWL_VC) {
        const int nc = min(FWL_VC, v1 - c0);
        __syncthreads();
        for (int i = tid; i < nc * QR; i += FWD_T) {
            const int vv = i / QR, n = i - vv * QR - nlo;
            const float *fr = f + (size_t)(c0 + vv) * Q;
            const float a = (n >= 0 && n < Q) ? fr[n] : 0.0f;
            const float b = (n + 1 >= 0 && n + 1 < Q) ? fr[n + 1] : 0.0f;
            tab[i] = make_float2((float)(0.5 * ((double)a + (double)b) - (double)n * ((double)b - (double)a)), b - a);
        }
        if (tid < nc) svox[tid] = p.vox[c0 + tid];
        __syncthreads();
        // this lane's open voxels of the chunk
        uint32_t m = 0u;
        if (valid)
            for (int vv = 0; vv < nc; vv++) m |= (uint32_t)mask_open(p, c0 + vv, pix, svox[vv], d) << vv;
        while (__any_sync(FULL, m != 0u)) {
            const int vv = m ? __ffs(m) - 1 : -1;
            m &= m - 1u;
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if (vv >= 0) {
                pair_geom(p, svox[vv], d, P, sh);
                k_range(p, sh, klo, khi);
            }
            const int wlo = __reduce_min_sync(FULL, klo);
            const int whi = __reduce_max_sync(FULL, khi);
            const uint32_t tb = tab0 + (uint32_t)(max(vv, 0) * QR) * 8u;  // this lane's row, folded with the magic bits
#pragma unroll
            for (int kb = 0; kb < KR; kb += 8) {
                if (kb + 8 <= wlo || kb > whi) continue;  // warp-uniform
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const float u = fminf(fmaf(at.a[kb + j], sh, p.nb), p.qm);
                    const float vm = u + kMagic;
                    CACSI_CHECK(__float_as_int(vm) - kMagicBits >= -nlo && __float_as_int(vm) - kMagicBits <= Q);
                    const float2 t = lds2(tb + ((uint32_t)__float_as_int(vm) << 3));
                    acc[kb + j] = fmaf(P, fmaf(u, t.y, t.x), acc[kb + j]);
                }
            }
        }
    }
    // [pixels][K] block of this CTA through shared memory (coalesced stores), scaled by c_k
    float *stage = (float *)smem4;
    const int npx = min(FWD_T, p.n_det - (int)blockIdx.x * FWD_T);
    float *out = partial + ((size_t)blockIdx.y * p.n_det + (size_t)blockIdx.x * FWD_T) * K;
    for (int kb = 0; kb < KR; kb += 32) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; j++)
            if (kb + j < KR) stage[j * (FWD_T + 1) + tid] = acc[kb + j];
        __syncthreads();
        const int kn = min(32, K - kb);
        for (int i = tid; i < npx * kn; i += FWD_T) {
            const int px = i / kn, k = i - px * kn;
            out[(size_t)px * K + kb + k] = p.energy[kb + k].y * stage[k * (FWD_T + 1) + px];
        }
    }
}

// (c0, slope) table of every voxel for k_forward_rec: row v = entries n = -nlo .. QR - nlo - 1 of
// f[v], exactly k_forward_lane's staging arithmetic (so the two forwards are bit-identical); one
// zero row of padding past the last voxel (the bulk copies round their byte counts up to 16)
__global__ void k_fl_tab(const Params p, const float *__restrict__ f, int nlo, int QR, float2 *__restrict__ tab) {
    const size_t n = (size_t)(p.n_vox + 1) * QR;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int v = (int)(i / QR), n0 = (int)(i % QR) - nlo;
        float a = 0.0f, b = 0.0f;
        if (v < p.n_vox) {
            const float *fr = f + (size_t)v * p.nq;
            a = (n0 >= 0 && n0 < p.nq) ? fr[n0] : 0.0f;
            b = (n0 + 1 >= 0 && n0 + 1 < p.nq) ? fr[n0 + 1] : 0.0f;
        }
        tab[i] = make_float2((float)(0.5 * ((double)a + (double)b) - (double)n0 * ((double)b - (double)a)), b - a);
    }
}

__device__ __forceinline__ void fr_mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
        "r"(phase)
        : "memory");
}

// The register forward fed by the pixel-major open-pair records (option er_fwd_rec, default when
// the records exist): the same lanes = pixels, KR energy sums in registers, per-lane
// voxel streams and per-term arithmetic as k_forward_lane, but
//  * no mask tests and no pair geometry per call: each lane walks its pixel's records (voxel,
//    energy window, P, sin(theta/2) as one 16-byte word; er_fcache_build) in increasing voxel
//    order through a 3-slot per-lane ring in shared memory filled by cp.async (three records
//    in flight);
//  * the (c0, slope) rows come from one table per call (k_fl_tab) by cp.async.bulk, two chunks of
//    FWL_VC voxels in flight: while chunk c is worked on, a lane that has finished its chunk-c
//    records goes on with chunk c + 1 once its rows have landed, so the warp's steps are bounded
//    by the lane with the most records over two chunks rather than one;
//  * no CTA barrier per chunk: each warp counts itself done with a buffer, and the last one
//    refills it, so warps drift apart by up to a chunk instead of waiting for the slowest;
//  * lanes more than `win` voxels past the warp's lowest wait (fewer distinct table rows per
//    step: fewer bank conflicts), and lanes whose window misses an energy block skip its table
//    reads, adding earlier (finite) table values with weight 0.
// The voxels of each pixel's sum are added in the same order, so the result is bit-identical to
// k_forward_lane with the same splits.
template <int KR>
__global__ void __launch_bounds__(FWD_T, 3) k_forward_rec(const Params p, const ErCache c,
                                                          const float2 *__restrict__ gtab, int vox_per_split,
                                                          float *__restrict__ partial, const AlphaTab at, int nlo,
                                                          int QR, int win) {
    extern __shared__ float4 smem4[];
    const int K = p.ne;
    float2 *tab = (float2 *)smem4;  // [2][VC][QR] (c0, slope); reused to stage the output
    uint64_t *full = (uint64_t *)(tab + 2 * FWL_VC * QR);  // [2] (2 * VC * QR * 8 is a multiple of 16)
    int *cnt = (int *)(full + 2);                          // [2] warps done with each buffer (monotone); [4]: pad
    const int tid = threadIdx.x;
    const int pix = blockIdx.x * FWD_T + tid;
    const bool valid = pix < p.n_det;
    const int v0 = blockIdx.y * vox_per_split;
    const int v1 = min(p.n_vox, v0 + vox_per_split);
    const int nch = (v1 - v0 + FWL_VC - 1) / FWL_VC;
    const uint32_t rowb = (uint32_t)QR * 8u;
    const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(tab + nlo) - (uint32_t)kMagicBits * 8u;
    auto issue = [&](int ci) {  // chunk ci -> buffer ci & 1
        const int cb = v0 + ci * FWL_VC, nc = min(FWL_VC, v1 - cb);
        const uint32_t bytes = ((uint32_t)nc * rowb + 15u) & ~15u;
        const uint32_t mb = (uint32_t)__cvta_generic_to_shared(full + (ci & 1));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(tab + (size_t)(ci & 1) * FWL_VC * QR)),
                     "l"(gtab + (size_t)cb * QR), "r"(bytes), "r"(mb)
                     : "memory");
    };
    if (tid == 0) {
        cnt[0] = cnt[1] = 0;
        for (int i = 0; i < 2; i++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(full + i)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
        issue(0);
        if (nch > 1) issue(1);
    }
    // this lane's records of the split (v0 and v1 are multiples of kErVB or v1 = n_vox)
    long long r = 0, rend = 0;
    if (valid) {
        const long long o = c.off[pix];
        r = o + c.boff[(size_t)(v0 / kErVB) * p.n_det + pix];
        rend = o + c.boff[(size_t)(v1 == p.n_vox ? c.nvb : v1 / kErVB) * p.n_det + pix];
    }
    // records r, r + 1, r + 2 in a per-lane ring of three shared-memory slots filled by cp.async
    // (16-byte words vw, P, s); the slot of the record in use is refilled with record r + 3, so
    // each load has three steps to land.  One commit group per step (empty past the end), so
    // wait_group 2 leaves only records r + 1, r + 2 in flight.
    const uint4 *rec = (const uint4 *)c.vw;
    uint4 *ring = (uint4 *)(cnt + 4) + tid;  // slot i at ring[i * FWD_T]
    auto fetch = [&](long long i, int slot) {
        if (i < rend)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(ring + slot * FWD_T)),
                         "l"(rec + i)
                         : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    fetch(r, 0);
    fetch(r + 1, 1);
    fetch(r + 2, 2);
    int ph = 0;  // slot of record r
    asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    uint4 cr = r < rend ? ring[0] : make_uint4(0u, 0u, 0x3f800000u, 0u);
    int curv = r < rend ? (int)(cr.x & 0xFFFFu) : 0x7FFFFFFF;
    float acc[KR];
#pragma unroll
    for (int k = 0; k < KR; k++) acc[k] = 0.0f;
    float2 tv[8];  // the block's table values (finite: zero, or an earlier read)
#pragma unroll
    for (int j = 0; j < 8; j++) tv[j] = make_float2(0.0f, 0.0f);
    const int lane = tid & 31;
    __syncthreads();  // mbarrier init visible
    for (int ci = 0; ci < nch; ci++) {
        const int cb = v0 + ci * FWL_VC;
        const int endc = min(v1, cb + FWL_VC);
        fr_mbar_wait((uint32_t)__cvta_generic_to_shared(full + (ci & 1)), (uint32_t)(ci >> 1) & 1u);
        // a lane may run ahead into chunk ci + 1 once its rows have landed (they land when every
        // warp has finished chunk ci - 1; tested without blocking)
        const uint32_t mbn = (uint32_t)__cvta_generic_to_shared(full + ((ci + 1) & 1));
        const uint32_t phn = (uint32_t)((ci + 1) >> 1) & 1u;
        int endn = endc;
        while (__any_sync(FULL, curv < endc)) {
            if (endn == endc && ci + 1 < nch) {
                uint32_t ok = 0u;
                if (lane == 0)
                    asm volatile(
                        "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                        "selp.u32 %0, 1, 0, P1;\n\t}\n"
                        : "=r"(ok)
                        : "r"(mbn), "r"(phn)
                        : "memory");
                if (__shfl_sync(FULL, ok, 0)) endn = min(v1, cb + 2 * FWL_VC);
            }
            // lanes more than `win` voxels past the warp's lowest wait: fewer distinct table rows per
            // step, so fewer shared-memory bank conflicts, at the price of a few more steps
            const int vmin = __reduce_min_sync(FULL, curv);
            const bool act = curv < endn && curv <= vmin + win;
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1, vv = 0;
            if (act) {
                P = __uint_as_float(cr.y), sh = __uint_as_float(cr.z);
                klo = (int)((cr.x >> 16) & 0xFFu), khi = (int)(cr.x >> 24);
                vv = curv - cb;
            }
            const int wlo = __reduce_min_sync(FULL, klo);
            const int whi = __reduce_max_sync(FULL, khi);
            // this lane's row: chunk ci + (vv >= VC) sits in buffer (ci + (vv >> 5)) & 1
            const uint32_t tb = tab0 + (uint32_t)((((ci + (vv >> 5)) & 1) << 5) + (vv & 31)) * rowb;
            static_assert(FWL_VC == 32, "row index split");
            // energy blocks in PAIRS (16 independent terms per basic block): a pair is worked when
            // either of its blocks meets the warp's window union; a block outside the union has no
            // lane whose window meets it, so its terms are exact zeros with no table reads
            auto block = [&](const int kb) {
                // lanes whose own window misses the block (or idle lanes) do not read the table:
                // their terms are exact zeros, and their reads would only add bank conflicts
                // (such a lane keeps the finite table values of an earlier read in tv[] and adds
                // them with weight 0: no zeroing per term)
                const bool mine = kb + 8 > klo && kb <= khi;
                const float Pm = mine ? P : 0.0f;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const float u = fminf(fmaf(at.a[kb + j], sh, p.nb), p.qm);
                    const float vm = u + kMagic;
                    CACSI_CHECK(__float_as_int(vm) - kMagicBits >= -nlo && __float_as_int(vm) - kMagicBits < QR - nlo);
                    if (mine) tv[j] = lds2(tb + ((uint32_t)__float_as_int(vm) << 3));
                    acc[kb + j] = fmaf(Pm, fmaf(u, tv[j].y, tv[j].x), acc[kb + j]);
                }
            };
#pragma unroll
            for (int kb = 0; kb < KR; kb += 16) {
                if (kb + 16 <= wlo || kb > whi) continue;  // warp-uniform
                block(kb);
                if (kb + 8 < KR) block(kb + 8);
            }
            if (act) {
                // refill the slot just used with record r + 3, then step to record r + 1
                fetch(r + 3, ph);
                r++;
                ph = ph == 2 ? 0 : ph + 1;
                asm volatile("cp.async.wait_group 2;\n" ::: "memory");
                if (r < rend) cr = ring[ph * FWD_T];
                curv = r < rend ? (int)(cr.x & 0xFFFFu) : 0x7FFFFFFF;
            }
        }
        // this warp is done with chunk ci; the last of the CTA's warps to get here refills its
        // buffer with chunk ci + 2 (arrival counts only grow: round ci's last arrival is number
        // NW (ci / 2 + 1) on counter ci & 1)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            const int old = atomicAdd(cnt + (ci & 1), 1);
            if (old == (FWD_T / 32) * ((ci >> 1) + 1) - 1 && ci + 2 < nch) {
                __threadfence_block();  // the other warps' reads of the buffer before the async-proxy write
                issue(ci + 2);
            }
        }
    }
    __syncthreads();  // every warp past its last chunk before the tables are reused for the output
    // [pixels][K] block of this CTA through shared memory (coalesced stores), scaled by c_k
    float *stage = (float *)smem4;
    const int npx = min(FWD_T, p.n_det - (int)blockIdx.x * FWD_T);
    float *out = partial + ((size_t)blockIdx.y * p.n_det + (size_t)blockIdx.x * FWD_T) * K;
    for (int kb = 0; kb < KR; kb += 32) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; j++)
            if (kb + j < KR) stage[j * (FWD_T + 1) + tid] = acc[kb + j];
        __syncthreads();
        const int kn = min(32, K - kb);
        for (int i = tid; i < npx * kn; i += FWD_T) {
            const int px = i / kn, k = i - px * kn;
            out[(size_t)px * K + kb + k] = p.energy[kb + k].y * stage[k * (FWD_T + 1) + px];
        }
    }
}

// [rows][cols] -> [cols][rows] (32 x 32 shared-memory tiles)
__global__ void k_transpose(const float *__restrict__ in, int rows, int cols, float *__restrict__ out) {
    __shared__ float t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[i][threadIdx.x] = in[(size_t)r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[(size_t)c * rows + r] = t[threadIdx.x][i];
    }
}

__global__ void k_sum_f64(const double *__restrict__ part, int S, size_t n, float *__restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < S; j++) s += part[j * n + i];
        out[i] = (float)s;
    }
}

__global__ void k_sum_f32(const float *__restrict__ part, int S, size_t n, float *__restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < S; j++) s += (double)part[j * n + i];
        out[i] = (float)s;
    }
}

// --------------------------------------------------------------- backward --
template <bool RES>
__global__ void __launch_bounds__(BWD_T) k_backward(const Params p, const float *__restrict__ w,
                                                    float *__restrict__ b) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne;
    float2 *en = (float2 *)smem4;                  // [K]
    float *hist = (float *)(en + ((K + 1) & ~1));  // [Q + 4][BWD_T]; bin = node + 2
    const int tid = threadIdx.x;
    const int v = blockIdx.x;
    for (int k = tid; k < K; k += BWD_T) en[k] = p.energy[k];
    for (int i = tid; i < (Q + 4) * BWD_T; i += BWD_T) hist[i] = 0.0f;
    __syncthreads();
    const VoxelRec vr = p.vox[v];
    float *hb = hist + tid;
    const int nd_round = (p.n_det + BWD_T - 1) / BWD_T * BWD_T;
    for (int q = tid; q < nd_round; q += BWD_T) {
        const bool valid = q < p.n_det;
        const float2 d = p.det[valid ? q : 0];
        const bool open = valid && mask_open(p, v, q, vr, d);
        float P = 0.0f, sh = 1.0f;
        int klo = K, khi = -1;
        if (open) {
            pair_geom(p, vr, d, P, sh);
            k_range(p, sh, klo, khi);
        }
        const int wlo = __reduce_min_sync(FULL, klo);
        const int whi = __reduce_max_sync(FULL, khi);
        if (!RES) {
            const float a = open ? P * w[q] : 0.0f;
            for (int k = wlo; k <= whi; k++) {
                const float2 e = en[k];
                float tt;
                const int n = hat_coord(p, e.x, sh, tt);
                const float ca = e.y * a;
                const float hi = fmaf(tt, ca, 0.5f * ca);
                float *h0 = hb + (n + 2) * BWD_T;
                h0[0] += ca - hi;
                h0[BWD_T] += hi;
            }
        } else {
            // w is passed TRANSPOSED here ([ne][n_det], launch_backward): lanes = consecutive
            // pixels read consecutive addresses for the same energy (coalesced)
            const float *wq = w + (valid ? q : 0);
            for (int k = wlo; k <= whi; k++) {
                const float2 e = en[k];
                float tt;
                const int n = hat_coord(p, e.x, sh, tt);
                const float ca = (open && k >= klo && k <= khi) ? P * e.y * __ldg(wq + (size_t)k * p.n_det) : 0.0f;
                const float hi = fmaf(tt, ca, 0.5f * ca);
                float *h0 = hb + (n + 2) * BWD_T;
                h0[0] += ca - hi;
                h0[BWD_T] += hi;
            }
        }
    }
    __syncthreads();
    for (int j = tid; j < Q; j += BWD_T) {
        const float *row = hist + (j + 2) * BWD_T;
        double s = 0.0;
        for (int t = 0; t < BWD_T; t++) s += (double)row[(t + j) % BWD_T];  // rotate: bank spread
        b[(size_t)v * Q + j] = (float)s;
    }
}

// Energy-resolving backward with compacted open pairs: as k_backward<true>
// (one CTA per voxel, lane-private histogram columns), but each warp first
// evaluates the mask and geometry of 64 pixels, appends the OPEN ones to a
// per-warp queue (P, sin(theta/2), pixel, energy window) and processes full
// batches of 32 queued pairs -- lanes never idle on closed pairs (about half of
// all pairs), and each batch's energy loop spans its lanes' windows only.
struct ErQ {
    float P, sh;
    int q, kw;  // kw = klo | khi << 16
};
constexpr int ERQ_CAP = 96;
__global__ void __launch_bounds__(BWD_T) k_backward_er_c(const Params p, const float *__restrict__ w,
                                                         float *__restrict__ b) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne;
    float2 *en = (float2 *)smem4;                  // [K]
    float *hist = (float *)(en + ((K + 1) & ~1));  // [Q + 4][BWD_T]; bin = node + 2
    ErQ *queue = (ErQ *)(hist + (Q + 4) * BWD_T);  // [BWD_T / 32][ERQ_CAP]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int v = blockIdx.x;
    for (int k = tid; k < K; k += BWD_T) en[k] = p.energy[k];
    for (int i = tid; i < (Q + 4) * BWD_T; i += BWD_T) hist[i] = 0.0f;
    __syncthreads();
    const VoxelRec vr = p.vox[v];
    float *hb = hist + tid;
    ErQ *wq = queue + warp * ERQ_CAP;
    int qn = 0;  // queued pairs (warp-uniform)
    auto batch = [&](int cnt) {
        // lanes < cnt take queue entries 0 .. cnt - 1
        ErQ e = {0.0f, 1.0f, 0, K};
        if (lane < cnt) e = wq[lane];
        const int klo = e.kw & 0xFFFF, khi = (e.kw >> 16) - 1;  // stored as khi + 1 (empty: klo = K, khi = -1)
        const int wlo = __reduce_min_sync(FULL, klo);
        const int whi = __reduce_max_sync(FULL, khi);
        const float *wp = w + e.q;
        // w of the next two energies in flight while this one deposits (the gathers'
        // L2 latency was the kernel's main stall: profiles/r2l_er_direct_ncu.json)
        float w0 = wlo <= whi ? __ldg(wp + (size_t)wlo * p.n_det) : 0.0f;
        float w1 = wlo + 1 <= whi ? __ldg(wp + (size_t)(wlo + 1) * p.n_det) : 0.0f;
        for (int k = wlo; k <= whi; k++) {
            const float wk = w0;
            w0 = w1;
            w1 = k + 2 <= whi ? __ldg(wp + (size_t)(k + 2) * p.n_det) : 0.0f;
            const float2 en_k = en[k];
            float tt;
            const int n = hat_coord(p, en_k.x, e.sh, tt);
            // no window test: a term outside this lane's [klo, khi] has its hat coordinate
            // clamped onto the padding rows (node -2 / nq), which the readout skips
            const float ca = e.P * en_k.y * wk;
            const float hi = fmaf(tt, ca, 0.5f * ca);
            float *h0 = hb + (n + 2) * BWD_T;
            h0[0] += ca - hi;
            h0[BWD_T] += hi;
        }
    };
    for (int base = warp * 64; base < p.n_det; base += (BWD_T / 32) * 64) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = base + 32 * h + lane;
            const bool valid = q < p.n_det;
            const float2 d = p.det[valid ? q : 0];
            bool open = valid && mask_open(p, v, q, vr, d);
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if (open) {
                pair_geom(p, vr, d, P, sh);
                k_range(p, sh, klo, khi);
                open = klo <= khi;
            }
            const unsigned m = __ballot_sync(FULL, open);
            if (open) wq[qn + __popc(m & ((1u << lane) - 1u))] = ErQ{P, sh, q, klo | ((khi + 1) << 16)};
            qn += __popc(m);
        }
        __syncwarp();
        while (qn >= 32) {
            batch(32);
            __syncwarp();
            // move the remainder (< 64 entries) to the front
            const int rem = qn - 32;
            ErQ t0, t1;
            if (lane < rem) t0 = wq[32 + lane];
            if (lane + 32 < rem) t1 = wq[64 + lane];
            __syncwarp();
            if (lane < rem) wq[lane] = t0;
            if (lane + 32 < rem) wq[lane + 32] = t1;
            __syncwarp();
            qn = rem;
        }
    }
    if (qn > 0) batch(qn);
    __syncthreads();
    for (int j = tid; j < Q; j += BWD_T) {
        const float *row = hist + (j + 2) * BWD_T;
        double s = 0.0;
        for (int t = 0; t < BWD_T; t++) s += (double)row[(t + j) % BWD_T];  // rotate: bank spread
        b[(size_t)v * Q + j] = (float)s;
    }
}

// ------------------------------------------- fixed-point energy-resolving backward --
// k_backward_er_x (option er_bwd_fx, default): the compacted open pairs of
// k_backward_er_c, with each lane's histogram column kept in FIXED POINT and
// updated by native shared-memory integer reductions (red.shared.add.s32):
// no read-modify-write through shared memory, so consecutive deposits of a
// lane no longer serialise on their load -> add -> store chains; the column
// is private to the lane (bank = lane, no conflicts), and integer sums are
// order-free.  Per term (u' = alpha_k sigma - q_min/dq - 1/2, n = round(u'),
// tt = u' - n): a = P s_v c_k w[q][k] is rounded to an integer by the
// 1.5 * 2^23 addition, hi = round((tt + 1/2) a) goes to node n + 1 and
// lo = round(a) - hi to node n (exactly the hat split of PAPER.md:248-270 in
// the energy-resolved form).  The per-voxel scale s_v keeps
// every bin's total below 2^31 units (a bound on sum P c_k hat measured at
// create, times max |w|) and every single deposit below 2^22 units (max P
// times max |c_k w|: the range of the rounding addition); columns wrap
// modulo 2^32, their int32 sum is exact because the true total fits.  w
// arrives pre-scaled by c_k in energy blocks of 4 ([ne4 / 4][n_det] float4,
// k_erx_wprep): lanes on nearby pixels read nearby 16-byte words, one load
// per lane per 4 energies.
__device__ __forceinline__ void red_s32(uint32_t addr, uint32_t v) {
    // no memory clobber: the histogram is read only after a CTA barrier, and table loads may
    // move across the reductions
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v));
}

// per pixel: union of the energy windows of its open pairs ([klo, khi], or (1, 0) if none)
__global__ void __launch_bounds__(256) k_erx_pix(const Params p, int2 *__restrict__ pwin, unsigned *__restrict__ smin) {
    const int lane = threadIdx.x & 31;
    float sm = 1e30f;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < p.n_det; q += (gridDim.x * blockDim.x) >> 5) {
        const float2 d = p.det[q];
        int lo = p.ne, hi = -1;
        for (int v = lane; v < p.n_vox; v += 32) {
            const VoxelRec vr = p.vox[v];
            if (!mask_open(p, v, q, vr, d)) continue;
            float P, sh;
            pair_geom(p, vr, d, P, sh);
            int klo, khi;
            k_range(p, sh, klo, khi);
            if (klo <= khi && P > 0.0f) lo = min(lo, klo), hi = max(hi, khi), sm = fminf(sm, sh);
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        if (lane == 0) pwin[q] = lo <= hi ? make_int2(lo, hi) : make_int2(1, 0);
    }
    atomicMin(smin, __float_as_uint(sm));  // positive floats order as their bit patterns
}

// per voxel: sum_q P and max_q P over its open pairs with a non-empty window
__global__ void __launch_bounds__(256) k_erx_vox(const Params p, float csum, float *__restrict__ vb,
                                                 float *__restrict__ pm) {
    __shared__ double ss[8];
    __shared__ float sm[8];
    const int v = blockIdx.x, tid = threadIdx.x;
    const VoxelRec vr = p.vox[v];
    double s = 0.0;
    float m = 0.0f;
    for (int q = tid; q < p.n_det; q += 256) {
        const float2 d = p.det[q];
        if (!mask_open(p, v, q, vr, d)) continue;
        float P, sh;
        pair_geom(p, vr, d, P, sh);
        int klo, khi;
        k_range(p, sh, klo, khi);
        if (klo <= khi && P > 0.0f) s += (double)P, m = fmaxf(m, P);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o), m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    if ((tid & 31) == 0) ss[tid >> 5] = s, sm[tid >> 5] = m;
    __syncthreads();
    if (tid == 0) {
        for (int i = 1; i < 8; i++) s += ss[i], m = fmaxf(m, sm[i]);
        vb[v] = (float)(s * (double)csum * (1.0 + 1e-5));  // loose bin bound: sum_k c_k hat <= sum_k c_k
        pm[v] = m * (1.0f + 1e-6f);
    }
}

// wt[kb][q] = (c_k w[q][k], k = 4 kb .. 4 kb + 3) as float4 (energy blocks of 4, zero-padded past ne;
// ONES: w = 1): lanes holding nearby pixels read nearby 16-byte words, 4 energies per load.
// mx[0] = max |w|, mx[1] = max |c_k w| over the entries inside each pixel's window union
// (the only ones that can reach a real histogram bin)
template <bool ONES>
__global__ void __launch_bounds__(256) k_erx_wprep(const Params p, const float *__restrict__ w, int ne4,
                                                   const int2 *__restrict__ pwin, float4 *__restrict__ wt,
                                                   unsigned *__restrict__ mx) {
    float m0 = 0.0f, m1 = 0.0f;
    const int nkb = ne4 >> 2;
    const size_t n = (size_t)p.n_det * nkb;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int kb = (int)(i / p.n_det), q = (int)(i - (size_t)kb * p.n_det);
        const int2 win = __ldg(pwin + q);
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int k = 4 * kb + j;
            o[j] = 0.0f;
            if (k < p.ne) {
                const float wv = ONES ? 1.0f : __ldg(w + (size_t)q * p.ne + k);
                o[j] = __ldg(&p.energy[k].y) * wv;
                if (k >= win.x && k <= win.y) m0 = fmaxf(m0, fabsf(wv)), m1 = fmaxf(m1, fabsf(o[j]));
            }
        }
        wt[i] = make_float4(o[0], o[1], o[2], o[3]);
    }
    for (int o = 16; o; o >>= 1) m0 = fmaxf(m0, __shfl_xor_sync(FULL, m0, o)), m1 = fmaxf(m1, __shfl_xor_sync(FULL, m1, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMax(mx, __float_as_uint(m0));  // nonnegative floats order as their bit patterns
        atomicMax(mx + 1, __float_as_uint(m1));
    }
}

struct ErxQ {
    float cs, sh;  // P s_v, sin(theta/2)
    int q, kw;     // pixel, klo | (khi + 1) << 16
};
constexpr int ERX_CAP = 96;
#ifndef CACSI_ERX_PF
#define CACSI_ERX_PF 8
#endif
#ifndef CACSI_ERX_F
#define CACSI_ERX_F 2
#endif
#ifndef CACSI_ERX_NRL
#define CACSI_ERX_NRL 4
#endif
#ifndef CACSI_ERX_PFR
#define CACSI_ERX_PFR 2
#endif
constexpr int ERX_PF = CACSI_ERX_PF;  // w~ blocks of look-ahead (Little's law: ~20 sectors per request from L2)
constexpr int ERX_NRL = CACSI_ERX_NRL;  // open-pair records per lane per unit (cached path)
constexpr int ERX_PFR = CACSI_ERX_PFR;  // w~ ring depth per record (cached path)
constexpr int ERX_F = CACSI_ERX_F;    // first w~ blocks of the next batch loaded during the current one (cached path)
// Open-pair cache of the energy-resolving backward (option er_vcache): per voxel, its
// open pairs with a non-empty energy window in pixel order, SoA: word = q | klo << 17 | (khi + 1) << 24,
// P, sin(theta/2) (12 B per open pair; 39 GB on config 4); vc_off[v] = first record of voxel v.
struct ErxCache {
    const long long *off;
    const uint32_t *w;
    const float *P, *s;
};
template <bool CACHE>
__global__ void __launch_bounds__(BWD_T) k_backward_er_x(const Params p, const float4 *__restrict__ wt, int ne4,
                                                         int nlo, const float *__restrict__ vb,
                                                         const float *__restrict__ pm, const unsigned *__restrict__ mx,
                                                         const ErxCache vc, float *__restrict__ b) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne, NR = Q + 2 + nlo;      // rows: nodes -nlo .. nq + 1
    float *alpha = (float *)smem4;                       // [ne4] (alpha_k; 1e30 beyond ne)
    uint32_t *hist = (uint32_t *)(alpha + ne4);           // [NR][BWD_T]; row = node + nlo
    ErxQ *queue = (ErxQ *)(hist + NR * BWD_T);           // [BWD_T / 32][ERX_CAP]
    __shared__ float s_scale;
    __shared__ int s_next;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int v = blockIdx.x;
    for (int k = tid; k < ne4; k += BWD_T) alpha[k] = k < K ? p.energy[k].x : 1e30f;
    for (int i = tid; i < NR * BWD_T; i += BWD_T) hist[i] = 0u;
    if (tid == 0) {
        const double m0 = (double)__uint_as_float(mx[0]), m1 = (double)__uint_as_float(mx[1]);
        const double bv = (double)vb[v], pv = (double)pm[v];
        double s = 0.0;
        if (m0 > 0.0 && bv > 0.0) {
            s = 2.1e9 / (bv * m0);                                    // bin totals < 2^31 (int32 sum of the columns)
            if (pv * m1 > 0.0) s = fmin(s, 4.19e6 / (pv * m1));       // single deposits < 2^22 (rounding by 1.5 * 2^23)
        }
        s_scale = (float)s;
        s_next = BWD_T / 32;  // groups 0 .. BWD_T/32 - 1 go to the warps in order, the rest on demand
    }
    __syncthreads();
    const float sv = s_scale;
    const VoxelRec vr = p.vox[v];
    const float nb = p.nb, qm = p.qm;
    const size_t wstride = (size_t)p.n_det * sizeof(float4);  // bytes between energy blocks of one pixel
    // byte address of row (n + nlo) of this thread's column, folded with the magic constant's
    // bits: row(n) = hb0 + bits(n + 1.5 * 2^23) * 4 * BWD_T
    const uint32_t hb0 = (uint32_t)__cvta_generic_to_shared(hist + tid) + (uint32_t)(nlo - kMagicBits) * (uint32_t)(4 * BWD_T);
    ErxQ *wq = queue + warp * ERX_CAP;
    int qn = 0;
    // u = alpha sigma - q_min/dq (true coordinates: nb + 1/2, clamp qm + 1/2) rounded DOWN to its
    // node n (FADD.RM against 1.5 * 2^23), fraction u - n exact: lower node (1 - frac) a, upper frac a
    const float nb1 = nb + 0.5f, qm1 = qm + 0.5f;
    const uint32_t hbl = __shfl_sync(FULL, hb0, lane);  // opaque to ptxas: one LEA per row address
    auto term = [&](float al, float wk, float sh, float cs) {
        // u >= -nlo + 1 (no lower clamp); a term outside this lane's window lands on the padding
        // rows (nodes < 0 or >= nq; at the clamp u = nq the whole deposit goes to node nq)
        const float u = fminf(fmaf(al, sh, nb1), qm1);
        const float vm = __fadd_rd(u, kMagic);
        const float fr = u - (vm - kMagic);
        const float a = cs * wk;
        const uint32_t ab = __float_as_uint(a + kMagic);
        const uint32_t hb = __float_as_uint(fmaf(fr, a, kMagic));
        const uint32_t addr = hbl + (__float_as_uint(vm) << 9);
        static_assert(4 * BWD_T == 512, "row stride");
        CACSI_CHECK(__float_as_int(vm) - kMagicBits >= -nlo && __float_as_int(vm) - kMagicBits <= Q);
        red_s32(addr, ab - hb);
        red_s32(addr + 4 * BWD_T, hb - (uint32_t)kMagicBits);
    };
    auto batch = [&](int cnt) {
        ErxQ e = {0.0f, 1.0f, 0, K};
        if (lane < cnt) e = wq[lane];
        const int klo = e.kw & 0xFFFF, khi = (e.kw >> 16) - 1;
        const int wlo = __reduce_min_sync(FULL, klo);
        const int whi = __reduce_max_sync(FULL, khi);
        if (wlo > whi) return;
        // energy block kb of this lane's pixel at wr + kb * wstride; the next ERX_PF blocks in
        // flight in a register ring (static indices: the block loop is unrolled by ERX_PF)
        const char *wr = (const char *)(wt + e.q);
        const int kb0 = wlo >> 2, kb1 = whi >> 2;
        float4 wn[ERX_PF];
        const char *pf = wr + (size_t)kb0 * wstride;
#pragma unroll
        for (int i = 0; i < ERX_PF; i++) {
            wn[i] = kb0 + i <= kb1 ? __ldg((const float4 *)pf) : make_float4(0.f, 0.f, 0.f, 0.f);
            pf += wstride;
        }
        for (int kb = kb0; kb <= kb1; kb += ERX_PF) {
#pragma unroll
            for (int i = 0; i < ERX_PF; i++) {
                if (kb + i > kb1) break;  // warp-uniform
                const float4 wc = wn[i];
                if (kb + i + ERX_PF <= kb1) wn[i] = __ldg((const float4 *)pf);
                pf += wstride;
                const float4 a4 = *(const float4 *)(alpha + ((kb + i) << 2));
                term(a4.x, wc.x, e.sh, e.cs);
                term(a4.y, wc.y, e.sh, e.cs);
                term(a4.z, wc.z, e.sh, e.cs);
                term(a4.w, wc.w, e.sh, e.cs);
            }
        }
    };
    if constexpr (CACHE) {
        // the voxel's open pairs straight from the cache, NRL records per lane per unit (record j =
        // unit base + 32 j + lane), their deposits side by side so every energy block gives 4 NRL
        // independent dependency chains; units on demand.  Records are loaded two units ahead; the
        // first ERX_F energy blocks of w of the NEXT unit are loaded while the current one
        // deposits; each lane loads only the blocks of its own windows (the union's other blocks
        // deposit on the padding rows whatever w they use)
        constexpr int NRL = ERX_NRL, UNIT = 32 * NRL;
        const long long r0 = vc.off[v], r1 = vc.off[v + 1];
        struct Rec {
            uint32_t w;
            float P, s;
        };
        struct RecN {
            Rec x[NRL];
        };
        auto load = [&](long long bi) {
            RecN z;
#pragma unroll
            for (int j = 0; j < NRL; j++) {
                const long long r = r0 + bi * UNIT + 32 * j + lane;
                z.x[j] = Rec{0u, 0.0f, 1.0f};
                if (r < r1) z.x[j].w = __ldg(vc.w + r), z.x[j].P = __ldg(vc.P + r), z.x[j].s = __ldg(vc.s + r);
            }
            return z;
        };
        struct Dec {
            uint32_t q;              // pixel
            float cs, sh;
            int lo4, span4;          // own window in energy blocks of 4: lo4 .. lo4 + span4 (none: lo4 huge)
        };
        struct DecN {
            Dec x[NRL];
            int kb0, kb1;            // the warp's union over the unit, in energy blocks of 4
        };
        auto decode = [&](const RecN &z, long long bi) {
            DecN d;
            int lo = K, hi = -1;
#pragma unroll
            for (int j = 0; j < NRL; j++) {
                const bool valid = r0 + bi * UNIT + 32 * j + lane < r1;
                const int klo = valid ? (int)((z.x[j].w >> 17) & 127u) : K;
                const int khi = valid ? (int)(z.x[j].w >> 24) - 1 : -1;
                d.x[j].q = valid ? (z.x[j].w & 0x1FFFFu) : 0u;
                d.x[j].cs = z.x[j].P * sv, d.x[j].sh = z.x[j].s;
                d.x[j].lo4 = klo <= khi ? klo >> 2 : 0x40000000;
                d.x[j].span4 = klo <= khi ? (khi >> 2) - (klo >> 2) : 0;
                lo = min(lo, klo), hi = max(hi, khi);
            }
            d.kb0 = __reduce_min_sync(FULL, lo) >> 2;
            hi = __reduce_max_sync(FULL, hi);
            d.kb1 = hi < 0 ? -1 : hi >> 2;
            return d;
        };
        // block kb of this lane's pixel into x if it is in the lane's own window; otherwise x keeps
        // the stale (finite) w of an earlier block: those terms land on the padding rows, or on
        // node 0 with a weight of exactly 0 (u = -1)
        const uint32_t ndet = (uint32_t)p.n_det;
        auto wload = [&](float4 &x, const Dec &d, int kb) {
            if ((uint32_t)(kb - d.lo4) <= (uint32_t)d.span4) x = __ldg(wt + ((uint32_t)kb * ndet + d.q));
        };
        auto deposit4a = [&](const Dec &d, const float4 &a4, const float4 &wc) {
            term(a4.x, wc.x, d.sh, d.cs);
            term(a4.y, wc.y, d.sh, d.cs);
            term(a4.z, wc.z, d.sh, d.cs);
            term(a4.w, wc.w, d.sh, d.cs);
        };
        auto next_unit = [&]() {
            int g = 0;
            if (lane == 0) g = atomicAdd(&s_next, 1);
            return (long long)__shfl_sync(FULL, g, 0);
        };
        constexpr int PF2 = ERX_PFR;  // ring depth per record
        static_assert(PF2 % 2 == 0, "alpha double buffer");
        long long ba = warp, bb = next_unit();
        RecN A = load(ba), B = load(bb);
        DecN dA = decode(A, ba);
        float4 fw[NRL][ERX_F], rw[NRL][PF2];  // zeroed once; afterwards stale blocks stay finite
#pragma unroll
        for (int j = 0; j < NRL; j++) {
#pragma unroll
            for (int i = 0; i < ERX_F; i++) fw[j][i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int i = 0; i < PF2; i++) rw[j][i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int i = 0; i < ERX_F; i++) wload(fw[j][i], dA.x[j], dA.kb0 + i);
        }
        while (r0 + ba * UNIT < r1) {
            const long long bc = next_unit();
            const RecN C = load(bc);
            // the rest of this unit's blocks: the next PF2 per record in flight in register rings
            const int kr0 = dA.kb0 + ERX_F;
#pragma unroll
            for (int i = 0; i < PF2; i++)
#pragma unroll
                for (int j = 0; j < NRL; j++) wload(rw[j][i], dA.x[j], kr0 + i);
#pragma unroll
            for (int i = 0; i < ERX_F; i++)
                if (dA.kb0 + i <= dA.kb1) {  // warp-uniform
                    const float4 a4 = *(const float4 *)(alpha + ((dA.kb0 + i) << 2));
#pragma unroll
                    for (int j = 0; j < NRL; j++) deposit4a(dA.x[j], a4, fw[j][i]);
                }
            // the next unit: window union and its first blocks, landing while this one deposits
            const DecN dB = decode(B, bb);
#pragma unroll
            for (int j = 0; j < NRL; j++)
#pragma unroll
                for (int i = 0; i < ERX_F; i++) wload(fw[j][i], dB.x[j], dB.kb0 + i);
            // alpha of the next block read one block ahead (past the last block it reads a harmless
            // word of the histogram)
            float4 an[2];
            an[0] = *(const float4 *)(alpha + (kr0 << 2));
            for (int kb = kr0; kb <= dA.kb1; kb += PF2) {
#pragma unroll
                for (int i = 0; i < PF2; i++) {
                    if (kb + i > dA.kb1) break;  // warp-uniform
                    an[(i + 1) & 1] = *(const float4 *)(alpha + ((kb + i + 1) << 2));
#pragma unroll
                    for (int j = 0; j < NRL; j++) deposit4a(dA.x[j], an[i & 1], rw[j][i]);
#pragma unroll
                    for (int j = 0; j < NRL; j++) wload(rw[j][i], dA.x[j], kb + i + PF2);
                }
            }
            ba = bb, bb = bc;
            dA = dB;
            B = C;
        }
    } else {
    // 64-pixel groups: the first one per warp fixed, the rest taken on demand (balances the
    // warps' open-pair counts, which the final CTA barrier would otherwise wait for)
    for (int grp = warp;;) {
        const int base = grp * 64;
        if (base >= p.n_det) break;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = base + 32 * h + lane;
            const bool valid = q < p.n_det;
            const float2 d = p.det[valid ? q : 0];
            bool open = valid && mask_open(p, v, q, vr, d);
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if (open) {
                pair_geom(p, vr, d, P, sh);
                k_range(p, sh, klo, khi);
                open = klo <= khi;
            }
            const unsigned m = __ballot_sync(FULL, open);
            if (open) wq[qn + __popc(m & ((1u << lane) - 1u))] = ErxQ{P * sv, sh, q, klo | ((khi + 1) << 16)};
            qn += __popc(m);
        }
        __syncwarp();
        while (qn >= 32) {
            batch(32);
            __syncwarp();
            const int rem = qn - 32;
            ErxQ t0, t1;
            if (lane < rem) t0 = wq[32 + lane];
            if (lane + 32 < rem) t1 = wq[64 + lane];
            __syncwarp();
            if (lane < rem) wq[lane] = t0;
            if (lane + 32 < rem) wq[lane + 32] = t1;
            __syncwarp();
            qn = rem;
        }
        int g = 0;
        if (lane == 0) g = atomicAdd(&s_next, 1);
        grp = __shfl_sync(FULL, g, 0);
    }
    if (qn > 0) batch(qn);
    }
    __syncthreads();
    const double inv = sv > 0.0f ? 1.0 / (double)sv : 0.0;
    for (int j = tid; j < Q; j += BWD_T) {
        const uint32_t *row = hist + (j + nlo) * BWD_T;
        uint32_t s = 0u;
        for (int t = 0; t < BWD_T; t++) s += row[(t + j) % BWD_T];  // modulo 2^32; rotate: bank spread
        b[(size_t)v * Q + j] = (float)((double)(int32_t)s * inv);
    }
}

// open pairs with a non-empty window (the backward's queue criterion), per voxel in pixel order
__device__ __forceinline__ bool erx_pair(const Params &p, int v, const VoxelRec &vr, int q, float &P, float &sh,
                                        int &klo, int &khi) {
    if (!mask_open(p, v, q, vr, p.det[q])) return false;
    pair_geom(p, vr, p.det[q], P, sh);
    k_range(p, sh, klo, khi);
    return klo <= khi;
}
__global__ void __launch_bounds__(256) k_erx_vcount(const Params p, long long *__restrict__ cnt) {
    __shared__ int sc[8];
    const int v = blockIdx.x, tid = threadIdx.x;
    const VoxelRec vr = p.vox[v];
    int c = 0;
    for (int q = tid; q < p.n_det; q += 256) {
        float P, sh;
        int klo, khi;
        c += erx_pair(p, v, vr, q, P, sh, klo, khi);
    }
    c = __reduce_add_sync(FULL, c);
    if ((tid & 31) == 0) sc[tid >> 5] = c;
    __syncthreads();
    if (tid == 0) {
        long long t = 0;
        for (int i = 0; i < 8; i++) t += sc[i];
        cnt[v] = t;
    }
}
__global__ void __launch_bounds__(256) k_erx_vfill(const Params p, const long long *__restrict__ off,
                                                   uint32_t *__restrict__ vw, float *__restrict__ vP,
                                                   float *__restrict__ vs) {
    __shared__ int sc[8];
    const int v = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const VoxelRec vr = p.vox[v];
    long long o = off[v];
    for (int q0 = 0; q0 < p.n_det; q0 += 256) {
        const int q = q0 + tid;
        float P = 0.0f, sh = 0.0f;
        int klo = 0, khi = -1;
        const bool op = q < p.n_det && erx_pair(p, v, vr, q, P, sh, klo, khi);
        const unsigned m = __ballot_sync(FULL, op);
        if (lane == 0) sc[warp] = __popc(m);
        __syncthreads();
        int before = 0, tot = 0;
        for (int i = 0; i < 8; i++) before += i < warp ? sc[i] : 0, tot += sc[i];
        if (op) {
            const long long i = o + before + __popc(m & ((1u << lane) - 1u));
            vw[i] = (uint32_t)q | ((uint32_t)klo << 17) | ((uint32_t)(khi + 1) << 24);
            vP[i] = P;
            vs[i] = sh;
        }
        o += tot;
        __syncthreads();
    }
}

// vb[v] = 1.02 max_j b1[v][j] (+ a floor): the measured bin bound of the fixed-point backward
__global__ void k_erx_vmax(const float *__restrict__ b1, int nq, int n_vox, float *__restrict__ vb) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n_vox; v += gridDim.x * blockDim.x) {
        float m = 0.0f;
        for (int j = 0; j < nq; j++) m = fmaxf(m, fabsf(b1[(size_t)v * nq + j]));
        vb[v] = m > 0.0f ? 1.02f * m : vb[v];
    }
}

int num_sms(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    if (device >= 0 && device < 64) cached[device] = n;
    return n;
}

}  // namespace

cudaError_t launch_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches) {
    if (g->esai.enabled) return esai_forward(g, f, out, s, launches);
    if (g->er.enabled) return er_forward(g, f, out, s, launches);
    const Params &p = g->p;
    const bool res = p.energy_resolving != 0;
    const int tiles = (p.n_det + FWD_T - 1) / FWD_T;
    const int target = 8 * num_sms(g->device);
    int S = (target + tiles - 1) / tiles;
    const int max_s = (p.n_vox + FWD_VC - 1) / FWD_VC;
    if (res) S = max(S, (p.n_vox + 1023) / 1024);  // fp32 partial sums over <= 1024 voxels
    S = max(1, min(S, max_s));
    int vps = (p.n_vox + S - 1) / S;
    // energy-resolving register forwards: splits on record-block boundaries (k_forward_rec reads
    // its records' offsets per kErVB voxels; k_forward_lane uses the same splits, same bits)
    const int vround = res && g->opt.er_fwd_reg ? kErVB : FWD_VC;
    vps = (vps + vround - 1) / vround * vround;
    S = (p.n_vox + vps - 1) / vps;
    const size_t n_out = (size_t)p.n_det * (res ? p.ne : 1);
    const size_t part_bytes = (size_t)S * n_out * (res ? sizeof(float) : sizeof(double));
    const size_t K4 = (size_t)(p.ne + 2 * FWD_KU) / FWD_KU * FWD_KU;  // as in k_forward
    size_t smem = K4 * sizeof(float2) + (size_t)(FWD_VC * (p.nq + 3) + 1) * sizeof(float2);
    if (res) smem += K4 * FWD_T * sizeof(float) + K4 * sizeof(float);
    void *part = nullptr;
    cudaError_t e = cudaMallocAsync(&part, part_bytes, s);
    if (e != cudaSuccess) return e;
    dim3 grid(tiles, S);
    if (res && g->opt.er_fwd_reg && p.ne <= KR_MAX &&
        (g->opt.er_fwd_lane ? FWL_VC : FWD_VC) * ((p.nq + 4 + (int)std::ceil(-(double)p.nb)) | 1) * 8 <= 72 * 1024) {
        // register accumulators: the smallest instantiated KR >= ne
        AlphaTab at;
        std::vector<float2> en(p.ne);
        e = cudaMemcpy(en.data(), p.energy, p.ne * sizeof(float2), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            cudaFreeAsync(part, s);
            return e;
        }
        for (int k = 0; k < KR_MAX; k++) at.a[k] = k < p.ne ? en[k].x : 1e30f;
        auto kf = p.ne <= 16 ? k_forward_reg<16> : p.ne <= 32 ? k_forward_reg<32> : p.ne <= 64 ? k_forward_reg<64>
                : p.ne <= 104 ? k_forward_reg<104> : k_forward_reg<128>;
        if (g->opt.er_fwd_lane)
            kf = p.ne <= 16 ? k_forward_lane<16> : p.ne <= 32 ? k_forward_lane<32> : p.ne <= 64 ? k_forward_lane<64>
               : p.ne <= 104 ? k_forward_lane<104> : k_forward_lane<128>;
        // table entries below node 0: u' >= nb = -q_min/dq - 1/2 rounds to n >= -(ceil(-nb) + 1)
        const int nlo = std::max(2, (int)std::ceil(-(double)p.nb) + 2);
        const int QR = (p.nq + 1 + nlo) | 1;  // odd row stride (float2): rows start on different banks
        const int vc = g->opt.er_fwd_lane ? FWL_VC : FWD_VC;
        const size_t sm2 = std::max((size_t)((vc * QR + 1) & ~1) * sizeof(float2) + vc * sizeof(VoxelRec),
                                    (size_t)32 * (FWD_T + 1) * sizeof(float));
        if (g->erf.enabled && g->opt.er_fwd_rec && g->opt.er_fwd_lane && vps % kErVB == 0) {
            // the record-fed forward: one (c0, slope) table per call, chunks landed by cp.async.bulk
            auto kr = p.ne <= 16 ? k_forward_rec<16> : p.ne <= 32 ? k_forward_rec<32> : p.ne <= 64 ? k_forward_rec<64>
                    : p.ne <= 104 ? k_forward_rec<104> : k_forward_rec<128>;
            float2 *gt = nullptr;
            e = cudaMallocAsync(&gt, (size_t)(p.n_vox + 1) * QR * sizeof(float2), s);
            if (e == cudaSuccess) {
                {
                    KScope kt_(g, s, "k_fl_tab");
                    k_fl_tab<<<4 * num_sms(g->device), 256, 0, s>>>(p, f, nlo, QR, gt);
                }
                const size_t sm3 = std::max((size_t)2 * FWL_VC * QR * sizeof(float2) + 32 + 3 * FWD_T * 16,
                                            (size_t)32 * (FWD_T + 1) * sizeof(float));
                cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
                {
                    KScope kt_(g, s, "k_forward_er");
                    kr<<<grid, FWD_T, sm3, s>>>(p, g->erf, gt, vps, (float *)part, at, nlo, QR, g->opt.er_fwd_win);
                }
                cudaFreeAsync(gt, s);
                *launches += 1;
            }
            if (e != cudaSuccess) {
                cudaFreeAsync(part, s);
                return e;
            }
        } else {
            cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
            KScope kt_(g, s, "k_forward_er");
            kf<<<grid, FWD_T, sm2, s>>>(p, f, vps, (float *)part, at, nlo, QR);
        }
    } else if (res) {
        cudaFuncSetAttribute(k_forward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        {
            KScope kt_(g, s, "k_forward_er");
            k_forward<true><<<grid, FWD_T, smem, s>>>(p, f, vps, part);
        }
    } else {
        cudaFuncSetAttribute(k_forward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        {
            KScope kt_(g, s, "k_forward");
            k_forward<false><<<grid, FWD_T, smem, s>>>(p, f, vps, part);
        }
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        const int nb = (int)min((n_out + 255) / 256, (size_t)(16 * num_sms(g->device)));
        if (res)
            {
                KScope kt_(g, s, "k_sum_f32");
                k_sum_f32<<<nb, 256, 0, s>>>((const float *)part, S, n_out, out);
            }
        else
            {
                KScope kt_(g, s, "k_sum_f64");
                k_sum_f64<<<nb, 256, 0, s>>>((const double *)part, S, n_out, out);
            }
        e = cudaGetLastError();
    }
    cudaFreeAsync(part, s);
    *launches += 2;
    return e;
}

namespace {
// the fixed-point energy-resolving backward: w pre-scaled into padded rows, then one CTA per voxel
cudaError_t erx_backward(const cacsi_geometry *g, const float *w, bool ones, float *b, cudaStream_t s, int *launches) {
    const Params &p = g->p;
    const int ne4 = (p.ne + 3) & ~3;
    float4 *wt = nullptr;
    cudaError_t e = cudaMallocAsync(&wt, (size_t)p.n_det * ne4 * sizeof(float) + 16, s);
    if (e != cudaSuccess) return e;
    unsigned *mx = (unsigned *)(wt + (size_t)p.n_det * (ne4 / 4));
    cudaMemsetAsync(mx, 0, 8, s);
    const int nb = 4 * num_sms(g->device);
    {
        KScope kt_(g, s, "k_erx_wprep");
        if (ones) k_erx_wprep<true><<<nb, 256, 0, s>>>(p, w, ne4, (const int2 *)g->d_erx_pw, wt, mx);
        else k_erx_wprep<false><<<nb, 256, 0, s>>>(p, w, ne4, (const int2 *)g->d_erx_pw, wt, mx);
    }
    const int nlo = g->erx_nlo;  // rows below node 0 (no lower clamp)
    const size_t smem = (size_t)ne4 * sizeof(float) + (size_t)(p.nq + 2 + nlo) * BWD_T * sizeof(uint32_t) +
                        (size_t)(BWD_T / 32) * ERX_CAP * sizeof(ErxQ);
    const bool cache = g->d_erx_voff && g->opt.er_vcache_use;
    auto kb = cache ? k_backward_er_x<true> : k_backward_er_x<false>;
    const ErxCache vc{(const long long *)g->d_erx_voff, (const uint32_t *)g->d_erx_vw, (const float *)g->d_erx_vP,
                      (const float *)g->d_erx_vs};
    cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    {
        KScope kt_(g, s, "k_backward_er");
        kb<<<p.n_vox, BWD_T, smem, s>>>(p, wt, ne4, nlo, (const float *)g->d_erx_vb, (const float *)g->d_erx_pm, mx,
                                        vc, b);
    }
    e = cudaGetLastError();
    cudaFreeAsync(wt, s);
    *launches += 2;
    return e;
}
}  // namespace

// tables of the fixed-point backward (create time): per-pixel window unions, per-voxel max P and a
// loose bin bound (sum P times sum_k c_k), then the bound measured by one backward of w = 1 with
// the loose bound's scale (accurate to ~1e-5, so 1.02x of it is safe)
cudaError_t erx_build(cacsi_geometry *g) {
    const Params &p = g->p;
    if (p.nq + 2 + std::max(2, (int)std::ceil(-(double)p.nb) + 2) > 400) return cudaSuccess;  // fp32-histogram kernel
    g->erx_nlo = std::max(2, (int)std::ceil(-(double)p.nb) + 2);  // refined below
    cudaError_t e = cudaMalloc(&g->d_erx_vb, (size_t)p.n_vox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_erx_pm, (size_t)p.n_vox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_erx_pw, (size_t)p.n_det * sizeof(int2));
    if (e != cudaSuccess) return e;
    std::vector<float2> en(p.ne);
    e = cudaMemcpy(en.data(), p.energy, p.ne * sizeof(float2), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return e;
    double csum = 0.0;
    for (int k = 0; k < p.ne; k++) csum += std::fabs((double)en[k].y);
    cudaStream_t s = 0;
    unsigned *smin = nullptr;
    e = cudaMalloc(&smin, sizeof(unsigned));
    if (e != cudaSuccess) return e;
    cudaMemset(smin, 0x7f, sizeof(unsigned));
    k_erx_pix<<<(p.n_det + 7) / 8, 256, 0, s>>>(p, (int2 *)g->d_erx_pw, smin);
    unsigned smin_bits = 0;
    e = cudaMemcpy(&smin_bits, smin, sizeof(unsigned), cudaMemcpyDeviceToHost);
    cudaFree(smin);
    if (e != cudaSuccess) return e;
    {
        // lowest u' = alpha sigma + nb of any term (alpha >= alpha_0, sigma >= the smallest open-pair
        // sigma; inactive lanes carry sigma = 1): rows down to its rounding, with fp32 margins
        float amin = 1e30f;
        for (int k = 0; k < p.ne; k++) amin = std::min(amin, en[k].x);
        const double sgm = std::min(1.0, (double)__uint_as_float_host(smin_bits));
        const double ulo = (double)amin * sgm * (1.0 - 1e-5) + (double)p.nb - 1e-4 * (1.0 + std::fabs((double)p.nb));
        g->erx_nlo = std::max(2, (int)std::ceil(-ulo) + 2);
    }
    k_erx_vox<<<p.n_vox, 256, 0, s>>>(p, (float)(csum * (1.0 + 1e-6)), (float *)g->d_erx_vb, (float *)g->d_erx_pm);
    // the voxel-major open-pair cache (option er_vcache): counts, exclusive scan, fill; skipped
    // when it would not leave 8 GB of device memory free or the pixel index needs > 17 bits
    if (g->opt.er_vcache && p.n_det <= (1 << 17) && p.ne <= 127) {
        long long *cnt = nullptr;
        e = cudaMalloc(&g->d_erx_voff, (size_t)(p.n_vox + 1) * sizeof(long long));
        if (e != cudaSuccess) return e;
        cnt = (long long *)g->d_erx_voff;
        k_erx_vcount<<<p.n_vox, 256, 0, s>>>(p, cnt);
        std::vector<long long> h(p.n_vox + 1);
        e = cudaMemcpy(h.data(), cnt, (size_t)p.n_vox * sizeof(long long), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return e;
        long long tot = 0;
        for (int v = 0; v < p.n_vox; v++) {
            const long long c = h[v];
            h[v] = tot;
            tot += c;
        }
        h[p.n_vox] = tot;
        size_t fr = 0, totmem = 0;
        cudaMemGetInfo(&fr, &totmem);
        const size_t need = (size_t)tot * 12 + 64;
        if (need + ((size_t)8 << 30) <= fr) {
            e = cudaMemcpy(cnt, h.data(), (size_t)(p.n_vox + 1) * sizeof(long long), cudaMemcpyHostToDevice);
            if (e == cudaSuccess) e = cudaMalloc(&g->d_erx_vw, (size_t)tot * 4 + 16);
            if (e == cudaSuccess) e = cudaMalloc(&g->d_erx_vP, (size_t)tot * 4 + 16);
            if (e == cudaSuccess) e = cudaMalloc(&g->d_erx_vs, (size_t)tot * 4 + 16);
            if (e != cudaSuccess) return e;
            k_erx_vfill<<<p.n_vox, 256, 0, s>>>(p, cnt, (uint32_t *)g->d_erx_vw, (float *)g->d_erx_vP,
                                                 (float *)g->d_erx_vs);
            e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            g->erx_vc_n = tot;
        } else {
            cudaFree(g->d_erx_voff);
            g->d_erx_voff = nullptr;
        }
    }
    // the pixel-major records of the forward (option er_fcache; k_forward_rec), same 8 GB margin
    if (g->opt.er_fcache) {
        e = er_fcache_build(g, (size_t)8 << 30);
        if (e != cudaSuccess) return e;
    }
    float *b1 = nullptr;
    e = cudaMalloc(&b1, (size_t)p.n_vox * p.nq * sizeof(float));
    if (e != cudaSuccess) return e;
    int n = 0;
    e = erx_backward(g, nullptr, true, b1, s, &n);
    if (e == cudaSuccess) {
        k_erx_vmax<<<(p.n_vox + 255) / 256, 256, 0, s>>>(b1, p.nq, p.n_vox, (float *)g->d_erx_vb);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(b1);
    return e;
}

cudaError_t launch_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches) {
    if (g->esai.enabled) return esai_backward(g, w, b, s, launches);
    if (g->er.enabled) return er_backward(g, w, b, s, launches);
    const Params &p = g->p;
    const size_t smem =
        (size_t)((p.ne + 1) & ~1) * sizeof(float2) + (size_t)(p.nq + 4) * BWD_T * sizeof(float);
    // the fixed-point kernel's histogram rows (nq + 2 + nlo) x 512 B must fit next to two more CTAs
    if (p.energy_resolving && g->opt.er_bwd_fx && g->d_erx_vb)
        return erx_backward(g, w, false, b, s, launches);
    if (p.energy_resolving) {
        float *wT = nullptr;
        cudaError_t e = cudaMallocAsync(&wT, (size_t)p.n_det * p.ne * sizeof(float), s);
        if (e != cudaSuccess) return e;
        {
            KScope kt_(g, s, "k_transpose");
            k_transpose<<<dim3((p.ne + 31) / 32, (p.n_det + 31) / 32), dim3(32, 8), 0, s>>>(w, p.n_det, p.ne, wT);
        }
        if (!g->opt.er_bwd_dense) {  // er_bwd_dense: lanes on all pixels (A/B reference)
            const size_t smc = smem + (size_t)(BWD_T / 32) * ERQ_CAP * sizeof(ErQ);
            cudaFuncSetAttribute(k_backward_er_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
            KScope kt_(g, s, "k_backward_er");
            k_backward_er_c<<<p.n_vox, BWD_T, smc, s>>>(p, wT, b);
        } else {
            cudaFuncSetAttribute(k_backward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            KScope kt_(g, s, "k_backward_er");
            k_backward<true><<<p.n_vox, BWD_T, smem, s>>>(p, wT, b);
        }
        cudaFreeAsync(wT, s);
        *launches += 1;
    } else {
        cudaFuncSetAttribute(k_backward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        {
            KScope kt_(g, s, "k_backward");
            k_backward<false><<<p.n_vox, BWD_T, smem, s>>>(p, w, b);
        }
    }
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace cacsi
