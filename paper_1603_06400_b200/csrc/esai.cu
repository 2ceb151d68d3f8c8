// esai.cu -- Exact Scatter-Angle Interpolation (ESAI): the energy-integrating
// forward and backward operators as (per-pair gather) x (dense contraction
// over q).  DESIGN.md "ESAI".
//
// The paper accelerates the forward model by tabulating the spectral factor
// on a uniform grid of scatter angles and interpolating the effective
// spectral factor W(r, theta) = int S(theta, q) f(r, q) dq (scatter-angle
// interpolation; Alg. 2, 176) -- an approximation
// (NRMSE 6.2 %).  In the discrete energy form the spectral
// factor of one pair is, with sigma = sin(theta/2),
//     S~(sigma)[j] = sum_k c_k Lambda(alpha_k sigma - beta0 - j),
// which is EXACTLY piecewise linear in sigma with kinks only where
// alpha_k sigma - beta0 is an integer m in [-1, nq].  Tabulating S~ at those
// kinks ("breakpoints" s_b) makes linear interpolation in sigma exact:
//     S~(sigma) = (1 - tau) S~_b + tau S~_{b+1},  s_b <= sigma <= s_{b+1}.
// Hence
//     forward : g[r'] = sum_r P [(1 - tau) W[r, b] + tau W[r, b+1]],  W = F S~^T
//     backward: A[r, b] = sum_{r'} P w[r'] hat_b(sigma),  b2 = A S~
// The per-term energy loop disappears from the pair loop; the q contraction
// becomes a dense GEMM.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cudaTypedefs.h>

#include "pair.cuh"
#include "tcgemm.cuh"
#include "tcgemm16.cuh"

namespace cacsi {

namespace {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- create --
// Per voxel: min / max sigma over ALL pixels (superset of the open pairs, same
// fp32 arithmetic as the operators) and sum_pixels P (fixed-point bound).
__global__ void __launch_bounds__(256) k_pair_stats(const Params p, float *shmin, float *shmax, float *ptot) {
    __shared__ float smin[8], smax[8];
    __shared__ double ssum[8];
    const int v = blockIdx.x, tid = threadIdx.x;
    const VoxelRec vr = p.vox[v];
    float lo = 3.0f, hi = -1.0f;
    double sum = 0.0;
    for (int q = tid; q < p.n_det; q += 256) {
        float P, sh;
        pair_geom(p, vr, p.det[q], P, sh);
        lo = fminf(lo, sh);
        hi = fmaxf(hi, sh);
        sum += (double)fabsf(P);
    }
    for (int o = 16; o; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
        sum += __shfl_xor_sync(FULL, sum, o);
    }
    if ((tid & 31) == 0) {
        smin[tid >> 5] = lo;
        smax[tid >> 5] = hi;
        ssum[tid >> 5] = sum;
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 1; i < 8; i++) {
            lo = fminf(lo, smin[i]);
            hi = fmaxf(hi, smax[i]);
        }
        double s = 0.0;
        for (int i = 0; i < 8; i++) s += ssum[i];
        shmin[v] = smin[0] < lo ? smin[0] : lo;
        shmax[v] = smax[0] > hi ? smax[0] : hi;
        ptot[v] = (float)(s * (1.0 + 1e-5));  // round up: an upper bound
    }
}

int host_locate(const std::vector<float> &sb, float s) {
    const int nb = (int)sb.size();
    int b = (int)(std::upper_bound(sb.begin(), sb.end(), s) - sb.begin()) - 1;
    return std::max(0, std::min(nb - 2, b));
}


// ---- transmission bitmaps (built once at create) ---------------------------
// One thread per 32-bit word: 32 mask tests by the exact rule (fp32 fast path,
// fp64 re-test near cell edges), packed in the order the pair kernels visit.
__global__ void k_tbits_fwd_tiled(const Params p, uint32_t *tb) {
    // word (c, pix): bit i = T(voxel 32c + i, pix)
    const size_t n = (size_t)((p.n_vox + 31) / 32) * p.n_det;
    for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < n; w += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(w / p.n_det), pix = (int)(w % p.n_det);
        const float2 d = p.det[pix];
        uint32_t bits = 0;
        for (int i = 0; i < 32; i++) {
            const int v = c * 32 + i;
            if (v < p.n_vox && mask_open(p, v, pix, p.vox[v], d)) bits |= 1u << i;
        }
        tb[w] = bits;
    }
}

__global__ void k_tbits_fwd_ts(const Params p, uint32_t *tb) {
    // word ((iz * det_nx + ix) * nyb + c) * det_ny + jy: bit k = T(voxel (32c + k, iz), pixel (ix, jy))
    const int nyb = (p.ny + 31) / 32;
    const size_t n = (size_t)p.nz * p.det_nx * nyb * p.det_ny;
    for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < n; w += (size_t)gridDim.x * blockDim.x) {
        const int jy = (int)(w % p.det_ny);
        size_t r = w / p.det_ny;
        const int c = (int)(r % nyb);
        r /= nyb;
        const int ix = (int)(r % p.det_nx), iz = (int)(r / p.det_nx);
        const int pix = ix * p.det_ny + jy;
        const float2 d = p.det[pix];
        uint32_t bits = 0;
        for (int k = 0; k < 32; k++) {
            const int iy = c * 32 + k;
            if (iy < p.ny && mask_open(p, iy * p.nz + iz, pix, p.vox[iy * p.nz + iz], d)) bits |= 1u << k;
        }
        tb[w] = bits;
    }
}

// seen[j] = OR over voxels of tb_bwd[v][j]: the pixels at least one open pair reaches
// (grid.y splits the voxels; seen is zeroed first, the chunks OR in)
__global__ void k_seen(const Params p, const uint32_t *__restrict__ tb, uint32_t *__restrict__ seen) {
    const int nw = (p.n_det + 31) / 32;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nw) return;
    const int per = (p.n_vox + gridDim.y - 1) / gridDim.y;
    const int v0 = blockIdx.y * per, v1 = min(p.n_vox, v0 + per);
    uint32_t m = 0u;
    for (int v = v0; v < v1; v++) m |= __ldg(tb + (size_t)v * nw + j);
    if (m) atomicOr(seen + j, m);
}

__global__ void k_tbits_bwd(const Params p, uint32_t *tb) {
    // word v * nw + j (nw = ceil(n_det / 32)): bit i = T(v, pixel 32 j + i)
    const int nw = (p.n_det + 31) / 32;
    const size_t n = (size_t)p.n_vox * nw;
    for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < n; w += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(w % nw), v = (int)(w / nw);
        const VoxelRec vr = p.vox[v];
        uint32_t bits = 0;
        for (int i = 0; i < 32; i++) {
            const int q = 32 * j + i;
            if (q < p.n_det && mask_open(p, v, q, vr, p.det[q])) bits |= 1u << i;
        }
        tb[w] = bits;
    }
}

// ------------------------------------------------------------ device side --
// Breakpoint location in SHARED memory, branch-free in the common case.  The
// sorted fp32 breakpoints s_b (+ kLocD +inf pads) and a LUT over the fp32 BIT
// PATTERN of sigma are staged once per persistent CTA.  For positive floats
// the bit pattern is monotone and piecewise linear in log2 (exponent,
// mantissa), so equal-width cells in bit space track the breakpoint density
// (~7x variation in log sigma) without a MUFU.LG2, and the cell index is
// exact integer arithmetic:
//   c = (bits(sigma) - lut_b0) >> lut_sh,  b = lut[c] + #{i = 1..kLocD : s_{lut[c]+i} <= sigma}
// lut[c] = the last breakpoint <= the cell's first float; a cell holding more
// than kLocD breakpoints is flagged (kLutSlow, ~0.1 % of cells) and walked.
// Returns b with s_b <= sigma < s_{b+1} (clamped to [0, nb-2]) and tau in [0,1].
constexpr int kLocD = 3;
constexpr unsigned kLutSlow = 0x8000u;

// (float)i for |i| < 2^22 without I2F (an XU instruction): integer add + FADD
__device__ __forceinline__ float exact_float(int i) {
    return __int_as_float(i + 0x4B400000) - 12582912.0f;
}

// Pop one set bit (the highest of the low word, else of the high word) of a
// 64-voxel transmission batch: 32-bit FLO + SEL instead of 64-bit ffs.
__device__ __forceinline__ int pop_bit(uint32_t &lo, uint32_t &hi) {
    const bool l = lo != 0u;
    const uint32_t w = l ? lo : hi;
    const int i = 31 - __clz(w);
    const uint32_t m = 1u << i;
    lo = l ? lo ^ m : lo;
    hi = l ? hi : hi ^ m;
    return l ? i : i + 32;
}

__device__ __forceinline__ void load_bp(const Esai &e, float *sb, uint16_t *lut) {
    for (int i = threadIdx.x; i < e.nb + kLocD; i += blockDim.x) sb[i] = __ldg(e.sb + i);
    for (int i = threadIdx.x; i < e.nl; i += blockDim.x) lut[i] = __ldg(e.lut16 + i);
}

__device__ __forceinline__ int locate(const Esai &e, const float *sb, const uint16_t *lut, float s, float &tau) {
    int c = (__float_as_int(s) - e.lut_b0) >> e.lut_sh;
    c = min(max(c, 0), e.nl - 1);
    const unsigned ent = lut[c];
    int b = (int)(ent & (kLutSlow - 1u));
    if (ent & kLutSlow) {
        while (b < e.nb - 2 && sb[b + 1] <= s) b++;
    } else {
        b += (int)(sb[b + 1] <= s) + (int)(sb[b + 2] <= s) + (int)(sb[b + 3] <= s);
        b = min(b, e.nb - 2);
    }
    const float s0 = sb[b], s1 = sb[b + 1];
    tau = fminf(fmaxf(__fdividef(s - s0, s1 - s0), 0.0f), 1.0f);
    return b;
}

// Scatter-angle interpolation (p.sai_n > 0): the nodes are the boundaries
// between tabulated angles, the pair takes its cell's row (tau = 0, nearest
// neighbour).  Within kSaiGuard (relative) of a boundary the
// fp32 sigma cannot decide the nearest angle; the cell is then re-derived from
// the fp64 angle by the rounding rule of reading R22 (same decision as the
// oracle).
constexpr float kSaiGuard = 4e-6f;

__device__ __forceinline__ int sai_cell(const Params &p, const Esai &e, const float *sb, float s, int b, int v, int q) {
    const bool near_lo = b > 0 && (s - sb[b]) < kSaiGuard * s;
    const bool near_hi = b + 2 < e.nb && (sb[b + 1] - s) < kSaiGuard * s;
    if (near_lo || near_hi) {
        const double th = theta64(p, v, q);
        double i = floor((th - p.sai_tmin) / p.sai_h + 0.5);
        i = fmin(fmax(i, 0.0), (double)(p.sai_n - 1));
        b = min(max((int)i - e.sai_i0, 0), e.nb - 2);
    }
    return b;
}

// locate for a pair (v, q): exact ESAI (tau = position in the breakpoint
// interval) or SAI (tau = 0 in the nearest-angle cell)
template <bool SAI>
__device__ __forceinline__ int locate_pair(const Params &p, const Esai &e, const float *sb, const uint16_t *lut,
                                           float s, int v, int q, float &tau) {
    int b = locate(e, sb, lut, s, tau);
    if (SAI) {
        b = sai_cell(p, e, sb, s, b, v, q);
        tau = 0.0f;
    }
    return b;
}

__device__ __forceinline__ size_t bp_smem_bytes(const Esai &e) {
    return ((size_t)(e.nb + kLocD) * sizeof(float) + (size_t)e.nl * sizeof(uint16_t) + 15) & ~(size_t)15;
}


constexpr int PF_TX = 16, PF_TY = 16, PF_T = PF_TX * PF_TY;  // 2D pixel tile
constexpr int PF_CH = 32;                                     // voxels per transmission word

// Forward pair stage (persistent): items (tile, voxel split);
// g_partial[split][pix] = sum_{v in split} P [(1-tau) W[v,b] + tau W[v,b+1]].
// The transmission bits of 32 voxels come in one word; lanes iterate only
// over their open voxels, two pairs per iteration.
template <bool SAI>
__global__ void __launch_bounds__(PF_T) k_esai_fwd(const Params p, const Esai e, const float2 *__restrict__ W,
                                                   int vox_per_split, int n_tiles, int n_items,
                                                   double *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem[];
    float *sb = (float *)smem;
    uint16_t *lut = (uint16_t *)(sb + e.nb + kLocD);
    load_bp(e, sb, lut);
    __syncthreads();
    const int tiles_y = (p.det_ny + PF_TY - 1) / PF_TY;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int tile = item % n_tiles, split = item / n_tiles;
        const int tx = tile / tiles_y, ty = tile % tiles_y;
        const int ix = tx * PF_TX + threadIdx.x / PF_TY;
        const int jy = ty * PF_TY + threadIdx.x % PF_TY;
        const bool valid = ix < p.det_nx && jy < p.det_ny;
        const int pix = valid ? ix * p.det_ny + jy : 0;
        const float2 d = p.det[pix];
        const int v0 = split * vox_per_split;
        const int v1 = min(p.n_vox, v0 + vox_per_split);
        double tot = 0.0;
        for (int c0 = v0; c0 < v1; c0 += PF_CH) {
            __syncwarp();  // reconverge after the previous batch's divergent pair loop
            uint32_t bits = valid ? __ldg(e.tb_fwd + (size_t)(c0 / PF_CH) * p.n_det + pix) : 0u;
            float acc = 0.0f;
            float qP1 = 0.0f, qP2 = 0.0f, qt1 = 0.0f, qt2 = 0.0f, qa1 = 0.0f, qb1 = 0.0f, qa2 = 0.0f, qb2 = 0.0f;
            while (bits) {
                const int i1 = __ffs(bits) - 1;
                bits &= bits - 1;
                const bool two = bits != 0;
                const int i2 = two ? __ffs(bits) - 1 : i1;
                bits &= bits - 1;
                float P1, s1, P2, s2, t1, t2;
                pair_geom(p, p.vox[c0 + i1], d, P1, s1, !SAI);
                pair_geom(p, p.vox[c0 + i2], d, P2, s2, !SAI);
                const int b1 = locate_pair<SAI>(p, e, sb, lut, s1, c0 + i1, pix, t1);
                const int b2 = locate_pair<SAI>(p, e, sb, lut, s2, c0 + i2, pix, t2);
                // consume the previous couple first, then load into the same registers
                acc = fmaf(qP1, fmaf(qt1, qb1 - qa1, qa1), acc);
                acc = fmaf(qP2, fmaf(qt2, qb2 - qa2, qa2), acc);
                const float2 w1 = __ldg(W + (size_t)(c0 + i1) * e.ldw + b1);  // (W_b, W_{b+1})
                const float2 w2 = __ldg(W + (size_t)(c0 + i2) * e.ldw + b2);
                qa1 = w1.x;
                qb1 = w1.y;
                qa2 = w2.x;
                qb2 = w2.y;
                qP1 = P1;
                qP2 = two ? P2 : 0.0f;
                qt1 = t1;
                qt2 = t2;
            }
            acc = fmaf(qP1, fmaf(qt1, qb1 - qa1, qa1), acc);
            acc = fmaf(qP2, fmaf(qt2, qb2 - qa2, qa2), acc);
            tot += (double)acc;
        }
        if (valid) partial[(size_t)split * p.n_det + pix] = tot;
    }
}

// ---- translation-symmetric forward (Alg. 2) --
// When the voxel y pitch is rho detector pitches, s = r' - r depends only on
// (iz, ix, d = jy - rho iy): |s|, G_od and dtheta of every pair of a detector
// row and a voxel row z are one "footprint" of n_jy + rho (ny - 1) entries.  A
// CTA owns TS_R 128-pixel row segments, builds the footprint of each voxel row
// z in shared memory (the paper's "compute once, shift by rho columns"), and
// reuses it for all ny voxels of that row as integer shifts.  Only the
// source-side quantities (r^, G_so) stay per pair.  Persistent CTAs over items
// (row group, z chunk).
constexpr int TS_T = 128, TS_R = 4;

__global__ void __launch_bounds__(TS_T * TS_R, 2) k_esai_fwd_ts(const Params p, const Esai e,
                                                             const float2 *__restrict__ W, int iz_per_chunk,
                                                             int n_groups, int n_items, double *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int rho = p.ts_rho, ny = p.ny, nz = p.nz;
    const int nfoot = TS_T + rho * (ny - 1);
    float *sb = (float *)smem;
    uint16_t *lut = (uint16_t *)(sb + e.nb + kLocD);
    float2 *foot_all = (float2 *)(smem + bp_smem_bytes(e));  // [TS_R][nfoot] (1/|s|, G_od dtheta)
    load_bp(e, sb, lut);
    const int r = threadIdx.x / TS_T, tid = threadIdx.x % TS_T;
    float2 *foot = foot_all + r * nfoot;
    const int segs = (p.det_ny + TS_T - 1) / TS_T;
    const int nyb = (ny + 31) / 32;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int grp = item % n_groups, chunk = item / n_groups;
        const int ix = (grp / segs) * TS_R + r, jy0 = (grp % segs) * TS_T;
        const int jy = jy0 + tid;
        const bool valid = ix < p.det_nx && jy < p.det_ny;
        // lanes past the row end still build footprint entries: they need the row's x
        const int pix = min(ix, p.det_nx - 1) * p.det_ny + min(jy, p.det_ny - 1);
        const float2 dd = p.det[pix];
        const float sx = dd.x;
        const int dmin = jy0 - rho * (ny - 1);
        const int iz0 = chunk * iz_per_chunk, iz1 = min(nz, iz0 + iz_per_chunk);
        double tot = 0.0;
        for (int iz = iz0; iz < iz1; iz++) {
            const float sz = p.vox[iz].sz;  // iy = 0 record: z-row quantity
            __syncthreads();
            if (ix < p.det_nx)
                for (int i = tid; i < nfoot; i += TS_T) {
                    const float sy = fmaf(p.pitch_d, (float)(dmin + i), p.ts_c0);
                    const float syz2 = fmaf(sy, sy, sz * sz);
                    const float rs = rsqrtf(fmaf(sx, sx, syz2));
                    const float rs2 = rs * rs;
                    const float x = p.pitch_d * fast_sqrt(syz2) * rs2 * fmaf(p.quarter_p2, rs2, 1.0f);
                    const float dth = x * fmaf(-0.33333334f * x, x, 1.0f);
                    foot[i] = make_float2(rs, sz * rs * rs2 * dth);
                }
            __syncthreads();
            // source-side quantities of voxel (iy, iz) are evaluated per pair
            // (y = y_0 + iy dy, r^ = r / |r|, G_so = z / |r|^3) and s_y from the
            // integer offset jy - rho iy (the footprint's own expression): the
            // pair reads only an 8-byte footprint entry from shared memory
            // (the L1/LSU data pipe is these kernels' bound)
            const float zr = p.vox[iz].z, z2 = zr * zr;
            // W row of voxel (iy, iz) = Wz + iy * wstride (32-bit offsets: n_vox * ldw < 2^32, esai_build)
            const float2 *Wz = W + (size_t)iz * e.ldw;
            const unsigned wstride = (unsigned)nz * (unsigned)e.ldw;
            const uint32_t *tbrow = e.tb_fwd + ((size_t)(iz * p.det_nx + (valid ? ix : 0)) * nyb) * p.det_ny +
                                    (valid ? jy : 0);
            float acc = 0.0f;
            // software pipeline: the W gathers of one pair couple are consumed one
            // iteration later, so their L2 latency overlaps the next couple's
            // geometry and locate (pending P = 0 contributes nothing)
            float qP1 = 0.0f, qP2 = 0.0f, qt1 = 0.0f, qt2 = 0.0f, qa1 = 0.0f, qb1 = 0.0f, qa2 = 0.0f, qb2 = 0.0f;
            // 64 voxels per batch (two transmission words): less lane imbalance
            for (int iyb = 0; iyb < ny; iyb += 64) {
                __syncwarp();  // reconverge after the previous batch's divergent pair loop
                uint32_t blo = 0u, bhi = 0u;
                if (valid) {
                    blo = __ldg(tbrow + (size_t)(iyb / 32) * p.det_ny);
                    if (iyb + 32 < ny) bhi = __ldg(tbrow + (size_t)(iyb / 32 + 1) * p.det_ny);
                }
                while (blo | bhi) {
                    const int k1 = pop_bit(blo, bhi);
                    const bool two = (blo | bhi) != 0u;
                    const int k2 = two ? pop_bit(blo, bhi) : k1;
                    float Pp[2], sh[2];
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        const int iy = iyb + (u ? k2 : k1);
                        CACSI_CHECK(tid + rho * (ny - 1 - iy) >= 0 && tid + rho * (ny - 1 - iy) < nfoot);
                        const float2 f = foot[tid + rho * (ny - 1 - iy)];
                        const float fiy = exact_float(iy);
                        const float sy = fmaf(p.pitch_d, exact_float(jy - rho * iy), p.ts_c0);
                        const float yr = fmaf(fiy, p.vy_step, p.vy0);
                        const float ir = rsqrtf(fmaf(yr, yr, z2));
                        const float ry = yr * ir, rz = zr * ir;
                        const float cos_t = fmaf(ry, sy, rz * sz) * f.x;
                        const float e1 = fmaf(ry, p.det_z, -rz * dd.y);
                        const float sin_t = fast_sqrt(fmaf(e1, e1, sx * sx)) * f.x;
                        const float h = fmaf(0.5f, cos_t, 0.5f);
                        const float rh = rsqrtf(h);
                        Pp[u] = rz * ir * ir * f.y * fmaf(cos_t, cos_t, 1.0f) * (h * rh);  // G_so = z/|r|^3
                        sh[u] = 0.5f * sin_t * rh;
                    }
                    float t1, t2;
                    const int b1 = locate(e, sb, lut, sh[0], t1);
                    const int b2 = locate(e, sb, lut, sh[1], t2);
                    // consume the previous couple first, then load into the same registers
                    acc = fmaf(qP1, fmaf(qt1, qb1 - qa1, qa1), acc);
                    acc = fmaf(qP2, fmaf(qt2, qb2 - qa2, qa2), acc);
                    // one 8-byte gather per pair: (W_b, W_{b+1}) (k_tc_gemm<true> pairs)
                    const float2 w1 = __ldg(Wz + ((unsigned)(iyb + k1) * wstride + (unsigned)b1));
                    const float2 w2 = __ldg(Wz + ((unsigned)(iyb + k2) * wstride + (unsigned)b2));
                    qa1 = w1.x;
                    qb1 = w1.y;
                    qa2 = w2.x;
                    qb2 = w2.y;
                    qP1 = Pp[0];
                    qP2 = two ? Pp[1] : 0.0f;
                    qt1 = t1;
                    qt2 = t2;
                }
            }
            acc = fmaf(qP1, fmaf(qt1, qb1 - qa1, qa1), acc);
            acc = fmaf(qP2, fmaf(qt2, qb2 - qa2, qa2), acc);
            tot += (double)acc;
        }
        if (valid) partial[(size_t)chunk * p.n_det + pix] = tot;
    }
}

// Subset forward (ordered subsets, Alg. 6): lanes = LISTED pixels, items =
// (256-pixel chunk of the list, voxel split).  T is evaluated per pair by the
// exact rule (mask_open; the transmission bitmaps are laid out for the full
// detector), 32 voxels per bit batch as in k_esai_fwd.
constexpr int PL_T = 256;

template <bool SAI>
__global__ void __launch_bounds__(PL_T) k_esai_fwd_list(const Params p, const Esai e, const float *__restrict__ W,
                                                        const int32_t *__restrict__ list, int n, int vox_per_split,
                                                        int n_items, double *__restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smem[];
    float *sb = (float *)smem;
    uint16_t *lut = (uint16_t *)(sb + e.nb + kLocD);
    load_bp(e, sb, lut);
    __syncthreads();
    const int n_chunks = (n + PL_T - 1) / PL_T;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int chunk = item % n_chunks, split = item / n_chunks;
        const int i = chunk * PL_T + threadIdx.x;
        const bool valid = i < n;
        const int pix = valid ? list[i] : list[0];
        const float2 d = p.det[pix];
        const int v0 = split * vox_per_split;
        const int v1 = min(p.n_vox, v0 + vox_per_split);
        double tot = 0.0;
        for (int c0 = v0; c0 < v1; c0 += 32) {
            __syncwarp();
            uint32_t bits = 0u;
            if (valid)
                for (int k = 0; k < 32 && c0 + k < v1; k++)
                    if (mask_open(p, c0 + k, pix, p.vox[c0 + k], d)) bits |= 1u << k;
            float acc = 0.0f;
            while (bits) {
                const int k = 31 - __clz(bits);
                bits ^= 1u << k;
                float P, sh, t;
                pair_geom(p, p.vox[c0 + k], d, P, sh, !SAI);
                const int b = locate_pair<SAI>(p, e, sb, lut, sh, c0 + k, pix, t);
                // plain W rows (the A-resident GEMM's output): W_b and W_{b+1}
                const float *wp = W + (size_t)(c0 + k) * e.ldw + b;
                const float wa = __ldg(wp), wb = __ldg(wp + 1);
                acc = fmaf(P, fmaf(t, wb - wa, wa), acc);
            }
            tot += (double)acc;
        }
        if (valid) partial[(size_t)split * n + i] = tot;
    }
}

// out[list[i]] = sum_s partial[s][i] in fp64: one warp per listed pixel, lane l
// sums splits l, l + 32, ... and a fixed shuffle tree combines the lanes
// (deterministic; a subset has few pixels and up to ~n_vox / 32 splits, so one
// thread per pixel would be a long chain of dependent loads)
__global__ void k_sum_list(const double *__restrict__ part, int S, const int32_t *__restrict__ list, int n,
                           float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int j = lane; j < S; j += 32) s += part[(size_t)j * n + i];
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if (lane == 0) out[list[i]] = (float)s;
    }
}

// pixel list -> detector bitmap (bit i of word j = pixel 32 j + i)
__global__ void k_list_to_mask(const int32_t *__restrict__ list, int n, uint32_t *__restrict__ mask) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicOr(mask + (list[i] >> 5), 1u << (list[i] & 31));
}

// max |w| over the detector (fixed-point scale of the backward histogram)
// (pmask != nullptr: only the subset's pixels count -- the fixed-point unit of a
// subset backward must not be set by weights it never deposits)
// (seen: only pixels with at least one open pair count -- the others never deposit)
__global__ void __launch_bounds__(1024) k_absmax(const float *__restrict__ w, size_t n, const uint32_t *pmask,
                                                 const uint32_t *seen, float *out) {
    __shared__ float s[32];
    float m = 0.0f;
    for (size_t i = threadIdx.x; i < n; i += 1024)
        if ((pmask == nullptr || ((pmask[i >> 5] >> (i & 31)) & 1u)) &&
            (seen == nullptr || ((seen[i >> 5] >> (i & 31)) & 1u)))
            m = fmaxf(m, fabsf(w[i]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 32; i++) m = fmaxf(m, s[i]);
        *out = fmaxf(m, s[0]);
    }
}

constexpr int PB_T = 1024, PB_WARPS = PB_T / 32;
constexpr int PB_QW = 32;  // transmission words (1024 pixels) per warp chunk

// Backward pair stage (persistent over voxels): A[v, b] = sum_pixels P w hat_b(sigma).
// Deposits go to a shared-memory histogram over the voxel's breakpoint window
// in FIXED POINT with native 32-bit integer shared atomics (fp32 atomicAdd on
// shared memory is a CAS loop on sm_100).  The per-voxel scale
//     2^30 / (vbound[v] max|w|),   vbound[v] >= max_b sum_pixels P hat_b(sigma)
// (a bound measured once at create with w = 1, esai_build) keeps every partial
// bin sum below 2^30 (|sum P w hat| <= max|w| sum P hat); the deposit
// x = P w scale is split exactly into the integers rint(x tau) -> b + 1 and
// rint(x) - rint(x tau) -> b.  One unit is 2^-30 of the voxel's largest bin
// (~2^-40 of its total response); integer adds are exact and
// order-independent, so the backward is deterministic.
// Pairs are interchangeable between lanes here (no per-lane accumulator), so
// each warp first COMPACTS the open pixels of a 1024-pixel chunk (transmission
// words, warp prefix sum of popcounts) into a pixel-sorted shared queue and
// then sweeps it with all 32 lanes: converged lanes, coalesced pixel / w loads.
// BOUND = true: w = 1, scale from the conservative bound sum_pixels |P| (used
// once to measure vbound).
template <bool BOUND, bool SAI>
__global__ void __launch_bounds__(PB_T) k_esai_bwd(const Params p, const Esai e, const float *__restrict__ w,
                                                   const float *__restrict__ wmax, const float *__restrict__ vbound,
                                                   const uint32_t *__restrict__ pmask, float *__restrict__ A) {
    extern __shared__ __align__(16) unsigned char smem[];
    float *sb = (float *)smem;
    uint16_t *lut = (uint16_t *)(sb + e.nb + kLocD);
    int *hist = (int *)(smem + bp_smem_bytes(e));  // [max_win]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint16_t *queue = (uint16_t *)(hist + ((e.max_win + 3) & ~3)) + warp * (PB_QW * 32);
    load_bp(e, sb, lut);
    const float wm = BOUND ? 1.0f : *wmax;
    const int nw = (p.n_det + 31) / 32;
    const int nchunk = (nw + PB_QW - 1) / PB_QW;
    for (int v = blockIdx.x; v < p.n_vox; v += gridDim.x) {
        const int2 win = e.vwin[v];
        const int nwin = win.y - win.x + 1;
        __syncthreads();  // previous voxel's histogram has been written out
        for (int i = tid; i < nwin; i += PB_T) hist[i] = 0;
        __syncthreads();
        const double bound = (double)vbound[v] * (double)wm;
        const float scale = bound > 0.0 ? (float)(1073741824.0 / bound) : 0.0f;
        const VoxelRec vr = p.vox[v];
        int *hv = hist - win.x;
        const uint32_t *tbv = e.tb_bwd + (size_t)v * nw;
        for (int ch = warp; scale > 0.0f && ch < nchunk; ch += PB_WARPS) {
            // compaction: lane l owns word ch * PB_QW + l (pixels 32 j .. 32 j + 31)
            const int j = ch * PB_QW + lane;
            uint32_t m = j < nw ? __ldg(tbv + j) : 0u;
            if (pmask != nullptr && j < nw) m &= __ldg(pmask + j);  // subset-restricted (Alg. 6)
            const int cnt = __popc(m);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = __shfl_sync(FULL, incl, 31);
            int off = incl - cnt;
            while (m) {
                const int i = 31 - __clz(m);
                queue[off++] = (uint16_t)(lane * 32 + i);
                m ^= 1u << i;
            }
            __syncwarp();
            const int qbase = ch * PB_QW * 32;
            for (int k = lane; k < total; k += 64) {
                const bool two = k + 32 < total;
                const int q1 = qbase + queue[k], q2 = two ? qbase + queue[k + 32] : q1;
                float P1, s1, P2, s2, t1, t2;
                pair_geom(p, vr, p.det[q1], P1, s1, !SAI);
                pair_geom(p, vr, p.det[q2], P2, s2, !SAI);
                const int b1 = locate_pair<SAI>(p, e, sb, lut, s1, v, q1, t1);
                const int b2 = locate_pair<SAI>(p, e, sb, lut, s2, v, q2, t2);
                const float a1 = BOUND ? P1 * scale : P1 * __ldg(w + q1) * scale;
                const float a2 = two ? (BOUND ? P2 * scale : P2 * __ldg(w + q2) * scale) : 0.0f;
                const int x1 = __float2int_rn(a1 * t1), x2 = __float2int_rn(a2 * t2);
                CACSI_CHECK(b1 >= win.x && b1 + 1 <= win.y && b2 >= win.x && b2 + 1 <= win.y);
                atomicAdd(hv + b1, __float2int_rn(a1) - x1);
                atomicAdd(hv + b1 + 1, x1);
                atomicAdd(hv + b2, __float2int_rn(a2) - x2);
                atomicAdd(hv + b2 + 1, x2);
            }
            __syncwarp();  // queue reuse
        }
        __syncthreads();
        const float unit = scale > 0.0f ? (float)(bound / 1073741824.0) : 0.0f;
        float *Ar = A + (size_t)v * e.ldw;
        for (int b = tid; b < e.ldw; b += PB_T) {
            const int i = b - win.x;
            Ar[b] = (i >= 0 && i < nwin) ? (float)hist[i] * unit : 0.0f;
        }
    }
}

// Subset backward (Alg. 6) over a pixel LIST: one warp per voxel with its own
// fixed-point histogram in shared memory (no CTA-wide barriers: the voxels of a
// CTA proceed independently), lanes take the listed pixels, test the pair's
// transmission bit and deposit as k_esai_bwd (same scale rule, so the same
// integers).  A subset has few pixels, so k_esai_bwd's per-voxel scan of the
// whole detector bitmap and its CTA-wide phases dominated there.
template <bool SAI>
__global__ void __launch_bounds__(256) k_esai_bwd_list(const Params p, const Esai e, const float *__restrict__ w,
                                                       const float *__restrict__ wmax, const int32_t *__restrict__ list,
                                                       int n, float *__restrict__ A) {
    extern __shared__ __align__(16) unsigned char smem[];
    float *sb = (float *)smem;
    uint16_t *lut = (uint16_t *)(sb + e.nb + kLocD);
    const int hstride = (e.max_win + 3) & ~3;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int *hist = (int *)(smem + bp_smem_bytes(e)) + warp * hstride;
    load_bp(e, sb, lut);
    __syncthreads();
    const float wm = *wmax;
    const int nw = (p.n_det + 31) / 32;
    for (int v = blockIdx.x * nwarps + warp; v < p.n_vox; v += gridDim.x * nwarps) {
        const int2 win = e.vwin[v];
        const int nwin = win.y - win.x + 1;
        for (int i = lane; i < nwin; i += 32) hist[i] = 0;
        __syncwarp();
        const double bound = (double)e.vbound[v] * (double)wm;
        const float scale = bound > 0.0 ? (float)(1073741824.0 / bound) : 0.0f;
        const VoxelRec vr = p.vox[v];
        int *hv = hist - win.x;
        const uint32_t *tbv = e.tb_bwd + (size_t)v * nw;
        // two listed pixels per lane per iteration: independent chains (bit test, geometry,
        // locate, deposit) whose latencies overlap
        for (int k = lane; scale > 0.0f && k < n; k += 64) {
            const bool two = k + 32 < n;
            const int q1 = __ldg(list + k), q2 = two ? __ldg(list + k + 32) : q1;
            const bool o1 = (__ldg(tbv + (q1 >> 5)) >> (q1 & 31)) & 1u;
            const bool o2 = two && ((__ldg(tbv + (q2 >> 5)) >> (q2 & 31)) & 1u);
            if (o1 || o2) {
                float P1, s1, P2, s2, t1, t2;
                pair_geom(p, vr, p.det[q1], P1, s1, !SAI);
                pair_geom(p, vr, p.det[q2], P2, s2, !SAI);
                const int b1 = locate_pair<SAI>(p, e, sb, lut, s1, v, q1, t1);
                const int b2 = locate_pair<SAI>(p, e, sb, lut, s2, v, q2, t2);
                const float a1 = o1 ? P1 * __ldg(w + q1) * scale : 0.0f;
                const float a2 = o2 ? P2 * __ldg(w + q2) * scale : 0.0f;
                const int x1 = __float2int_rn(a1 * t1), x2 = __float2int_rn(a2 * t2);
                CACSI_CHECK(!o1 || (b1 >= win.x && b1 + 1 <= win.y));
                CACSI_CHECK(!o2 || (b2 >= win.x && b2 + 1 <= win.y));
                if (o1) {
                    atomicAdd(hv + b1, __float2int_rn(a1) - x1);
                    atomicAdd(hv + b1 + 1, x1);
                }
                if (o2) {
                    atomicAdd(hv + b2, __float2int_rn(a2) - x2);
                    atomicAdd(hv + b2 + 1, x2);
                }
            }
        }
        __syncwarp();
        const float unit = scale > 0.0f ? (float)(bound / 1073741824.0) : 0.0f;
        float *Ar = A + (size_t)v * e.ldw;
        for (int b = lane; b < e.ldw; b += 32) {
            const int i = b - win.x;
            Ar[b] = (i >= 0 && i < nwin) ? (float)hist[i] * unit : 0.0f;
        }
        __syncwarp();
    }
}

#include "pair_cache.cuh"

static size_t bwd_smem_bytes(size_t bpb, int max_win) {
    return bpb + (size_t)((max_win + 3) & ~3) * sizeof(int) + (size_t)PB_WARPS * PB_QW * 32 * sizeof(uint16_t);
}

// vbound[v] = (max_b A1[v, b] + n_det units) (1 + 1e-3): a bound on every bin of
// the voxel with w = 1, A1 measured by k_esai_bwd<true> (units of its
// conservative scale; each of <= n_det deposits per bin rounds by <= 1/2 unit).
__global__ void __launch_bounds__(256) k_vbound(const float *__restrict__ A1, int ldw, const float *__restrict__ ptot,
                                                int n_det, float *__restrict__ vbound) {
    __shared__ float sm[8];
    const int v = blockIdx.x;
    float m = 0.0f;
    for (int b = threadIdx.x; b < ldw; b += 256) m = fmaxf(m, A1[(size_t)v * ldw + b]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 8; i++) m = fmaxf(m, sm[i]);
        m = fmaxf(m, sm[0]);
        const double unit = (double)ptot[v] / 1073741824.0;
        vbound[v] = (float)(((double)m + n_det * unit) * (1.0 + 1e-3));
    }
}

#include "elementwise.cuh"

// What the final partial sum t_i = sum_j part[j][i] writes: the operator output
// (EpiStore), or -- inside cacsi_iterate -- the ratio w_i = y_i / (t_i + r_i) and
// max |w| (EpiRatio, for the backward's fixed-point scale), or the f update with
// b2_i = t_i (EpiUpdate).  The stand-alone kernels (k_ratio, k_absmax, k_update)
// compute the same bits from the stored t_i (elementwise.cuh).
struct EpiStore {
    float *out;
    static constexpr bool kMax = false;
    __device__ float operator()(size_t i, double t) const {
        out[i] = (float)t;
        return 0.0f;
    }
};
struct EpiRatio {
    const float *y, *r;
    float *out;
    unsigned *wmax;  // bits of max |w| (non-negative floats order as unsigned); zeroed by the caller
    const uint32_t *seen;  // the max runs over the pixels some open pair sees (k_absmax's rule)
    static constexpr bool kMax = true;
    __device__ float operator()(size_t i, double t) const {
        const float v = guarded_ratio(y[i], (float)t + r[i]);
        out[i] = v;
        return (seen == nullptr || ((__ldg(seen + (i >> 5)) >> (i & 31)) & 1u)) ? fabsf(v) : 0.0f;
    }
};
struct EpiUpdate {
    Params p;
    const float *f_hat, *b1;
    float beta;
    double delta;
    float *f_new;
    static constexpr bool kMax = false;
    __device__ float operator()(size_t i, double t) const {
        f_new[i] = update_at(p, f_hat, b1, (float)t, beta, delta, (unsigned)i);
        return 0.0f;
    }
    // four consecutive elements of one voxel (k_sum_parts_v4 when nq % 4 == 0): the same bits
    __device__ bool quad(size_t i0, double t0, double t1, double t2, double t3) const {
        if (p.nq % 4 != 0) return false;
        *(float4 *)(f_new + i0) = update_at4(p, f_hat, b1, make_float4((float)t0, (float)t1, (float)t2, (float)t3), beta,
                                             delta, (unsigned)i0);
        return true;
    }
};
template <class Epi>
__device__ __forceinline__ bool epi_quad(const Epi &epi, size_t i0, double t0, double t1, double t2, double t3) {
    if constexpr (std::is_same<Epi, EpiUpdate>::value)
        return epi.quad(i0, t0, t1, t2, t3);
    else
        return false;
}
template <class Epi>
__device__ __forceinline__ void epi_max(const Epi &epi, float m) {
    if constexpr (Epi::kMax) {
        // fmaxf drops NaN (as k_absmax does); one atomic per warp
        const unsigned bits = __reduce_max_sync(0xFFFFFFFFu, __float_as_uint(m));
        if ((threadIdx.x & 31) == 0 && bits != 0u) atomicMax(epi.wmax, bits);
    }
}

// out[i] = sum_j part[j][i] (j < S), in double, in a fixed order: warp w of the block
// sums the slices j = w, w + 8, ... in increasing j for SP_U x 32 outputs (coalesced
// loads, SP_U x 2 in flight per thread), then one thread per output adds the 8
// warp sums in warp order -- deterministic, and the S-long loop is split 8 ways
// (a thread per output walking all S slices was latency-bound: 0.033 ms for
// S = 296 on config 1)
constexpr int SP_U = 2;
template <typename T, class Epi>
__global__ void __launch_bounds__(256) k_sum_parts(const T *__restrict__ part, int S, size_t n, Epi epi) {
    __shared__ double red[8][32 * SP_U];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t i0 = (size_t)blockIdx.x * (32 * SP_U);
    double acc[SP_U];
#pragma unroll
    for (int u = 0; u < SP_U; u++) acc[u] = 0.0;
    int j = warp;
    for (; j + 8 < S; j += 16) {
        T x[SP_U], y[SP_U];
#pragma unroll
        for (int u = 0; u < SP_U; u++) {
            const size_t i = i0 + lane + 32 * u;
            x[u] = i < n ? part[(size_t)j * n + i] : (T)0;
            y[u] = i < n ? part[(size_t)(j + 8) * n + i] : (T)0;
        }
#pragma unroll
        for (int u = 0; u < SP_U; u++) acc[u] = (acc[u] + (double)x[u]) + (double)y[u];
    }
    if (j < S) {
#pragma unroll
        for (int u = 0; u < SP_U; u++) {
            const size_t i = i0 + lane + 32 * u;
            acc[u] += i < n ? (double)part[(size_t)j * n + i] : 0.0;
        }
    }
#pragma unroll
    for (int u = 0; u < SP_U; u++) red[warp][lane + 32 * u] = acc[u];
    __syncthreads();
    float m = 0.0f;
    if (threadIdx.x < 32 * SP_U && i0 + threadIdx.x < n) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; w++) t += red[w][threadIdx.x];
        m = epi(i0 + threadIdx.x, t);
    }
    epi_max(epi, m);
}
// few slices or many outputs (the b2 split-K partials: 2M outputs on config 2, where
// the thread-per-output loop already streams at ~4.6 TB/s): one thread per output
// walks the slices in order
template <typename T, class Epi>
__global__ void k_sum_parts_seq(const T *__restrict__ part, int S, size_t n, Epi epi) {
    float m = 0.0f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < S; j++) s += (double)part[j * n + i];
        m = fmaxf(m, epi(i, s));
    }
    epi_max(epi, m);
}
// the same per-output order (j = 0, 1, ... from 0.0, so the same bits as k_sum_parts_seq)
// for fp32 partials with n % 4 == 0: four consecutive outputs per thread (16-byte loads),
// the slices loaded 8 at a time before they are added, so 8 x 16 B are in flight per
// thread instead of one dependent load per slice (config 2's b2 partials: 16 x 8 MB)
template <class Epi>
__global__ void __launch_bounds__(256) k_sum_parts_v4(const float *__restrict__ part, int S, size_t n, Epi epi) {
    float m = 0.0f;
    const size_t n4 = n / 4;
    for (size_t i4 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i4 < n4; i4 += (size_t)gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        const float4 *p4 = (const float4 *)part + i4;
        int j = 0;
        for (; j + 8 <= S; j += 8) {
            float4 x[8];
#pragma unroll
            for (int u = 0; u < 8; u++) x[u] = __ldcs(p4 + (size_t)(j + u) * n4);
#pragma unroll
            for (int u = 0; u < 8; u++) s0 += (double)x[u].x, s1 += (double)x[u].y, s2 += (double)x[u].z, s3 += (double)x[u].w;
        }
        for (; j < S; j++) {
            const float4 x = __ldcs(p4 + (size_t)j * n4);
            s0 += (double)x.x, s1 += (double)x.y, s2 += (double)x.z, s3 += (double)x.w;
        }
        if (epi_quad(epi, 4 * i4, s0, s1, s2, s3)) continue;
        m = fmaxf(m, epi(4 * i4, s0));
        m = fmaxf(m, epi(4 * i4 + 1, s1));
        m = fmaxf(m, epi(4 * i4 + 2, s2));
        m = fmaxf(m, epi(4 * i4 + 3, s3));
    }
    epi_max(epi, m);
}
template <typename T, class Epi>
void sum_parts(const T *part, int S, size_t n, Epi epi, cudaStream_t s) {
    if (S >= 16 && n < 200000)
        k_sum_parts<T, Epi><<<(unsigned)((n + 32 * SP_U - 1) / (32 * SP_U)), 256, 0, s>>>(part, S, n, epi);
    else if (std::is_same<T, float>::value && n % 4 == 0 && (uintptr_t)part % 16 == 0)
        k_sum_parts_v4<Epi><<<(unsigned)std::min((n / 4 + 255) / 256, (size_t)8 * 148), 256, 0, s>>>(
            (const float *)part, S, n, epi);
    else
        k_sum_parts_seq<T, Epi><<<(unsigned)std::min((n + 255) / 256, (size_t)4096), 256, 0, s>>>(part, S, n, epi);
}

int sm_count(int dev) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

}  // namespace

int fbits(float x) {
    int i;
    std::memcpy(&i, &x, 4);
    return i;
}
float ffrom(int i) {
    float x;
    std::memcpy(&x, &i, 4);
    return x;
}

static size_t host_bp_bytes(const Esai &E) {
    return ((size_t)(E.nb + kLocD) * sizeof(float) + (size_t)E.nl * sizeof(uint16_t) + 15) & ~(size_t)15;
}

// persistent grid: CTAs per SM limited by shared memory and threads
static int persistent_grid(const cacsi_geometry *g, size_t smem, int threads) {
    int per_sm = std::max(1, std::min((int)(227 * 1024 / (smem + 1024)), 2048 / threads));
    return per_sm * sm_count(g->device);
}

// Build the ESAI tables (energy-integrating handles).  Host fp64 arithmetic
// for the breakpoints and S~; DESIGN.md "ESAI tables".
// setup stage clock: stage i's wall time since the previous mark (setup_us[i])
struct SetupClock {
    cacsi_geometry *g;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(int i) {
        const auto n = std::chrono::steady_clock::now();
        g->setup_us[i] += std::chrono::duration_cast<std::chrono::microseconds>(n - t).count();
        t = n;
    }
};

cudaError_t esai_build(cacsi_geometry *g, const cacsi_geometry_desc *d) {
    const Params &p = g->p;
    SetupClock clk{g};
    const int nv = p.n_vox, Q = p.nq, K = p.ne;
    float *dmin = nullptr, *dmax = nullptr, *dpt = nullptr;
    cudaError_t e = cudaMalloc(&dmin, nv * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&dmax, nv * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&dpt, nv * sizeof(float));
    if (e == cudaSuccess) {
        k_pair_stats<<<nv, 256>>>(p, dmin, dmax, dpt);
        e = cudaGetLastError();
    }
    std::vector<float> shmin(nv), shmax(nv), ptot(nv);
    if (e == cudaSuccess) e = cudaMemcpy(shmin.data(), dmin, nv * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(shmax.data(), dmax, nv * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(ptot.data(), dpt, nv * 4, cudaMemcpyDeviceToHost);
    cudaFree(dmin);
    cudaFree(dmax);
    if (e != cudaSuccess) {
        cudaFree(dpt);
        return e;
    }
    g->d_esai_ptot = dpt;
    const float smin = *std::min_element(shmin.begin(), shmin.end());
    const float smax = *std::max_element(shmax.begin(), shmax.end());
    const double lo = (double)smin * (1.0 - 1e-6), hi = (double)smax * (1.0 + 1e-6);

    // breakpoints s_{k,m} = (m + beta0) / alpha_k, m in [-1, nq]   (fp64)
    const double dq = (d->q_max - d->q_min) / (d->nq - 1);
    const double beta0 = d->q_min / dq;
    std::vector<double> alpha(K), ck(K);
    for (int k = 0; k < K; k++) {
        alpha[k] = d->energy_kev[k] / (kHc * dq);
        ck[k] = d->scale * d->phi[k] * d->energy_kev[k];
    }
    // (fp32 node, exact fp64 kink) pairs; S~ is evaluated at the exact kink so
    // that nodes which are exactly unreachable stay exactly zero
    std::vector<std::pair<float, double>> nodes;
    nodes.push_back({(float)lo, (double)(float)lo});
    nodes.push_back({(float)hi, (double)(float)hi});
    const bool sai = p.sai_n > 0;
    if (!sai) {
        for (int k = 0; k < K; k++)
            for (int m = -1; m <= Q; m++) {
                const double s = (m + beta0) / alpha[k];
                if (s > lo && s < hi) nodes.push_back({(float)s, s});
            }
    } else {
        // SAI: nodes = sigma at the boundaries between tabulated angles,
        // t_{i+1/2} = t_min + (i + 1/2) h (nearest-angle cells, reading R22)
        for (int i = 0; i + 1 < p.sai_n; i++) {
            const double s = std::sin(0.5 * (p.sai_tmin + (i + 0.5) * p.sai_h));
            if (s > lo && s < hi) nodes.push_back({(float)s, s});
        }
    }
    std::sort(nodes.begin(), nodes.end());
    std::vector<float> sb;
    std::vector<double> sx;
    for (auto &n : nodes)
        if (sb.empty() || n.first != sb.back()) {
            sb.push_back(n.first);
            sx.push_back(n.second);
        }
    const int nb = (int)sb.size();
    // (s_b, 1 / (s_{b+1} - s_b)) and S~ at the kinks
    std::vector<float2> bp(nb);
    std::vector<float> stab((size_t)nb * Q, 0.0f);
    std::vector<double> row(Q);
    // SAI: angle index of the first cell = number of boundaries <= lo
    int sai_i0 = 0;
    if (sai)
        while (sai_i0 + 1 < p.sai_n && std::sin(0.5 * (p.sai_tmin + (sai_i0 + 0.5) * p.sai_h)) <= lo) sai_i0++;
    for (int b = 0; b < nb; b++) {
        double s = sx[b], ang = 1.0;
        if (sai) {  // row of cell b: the spectral-angular factor at its tabulated angle
            const double t = p.sai_tmin + std::min(sai_i0 + std::min(b, nb - 2), p.sai_n - 1) * p.sai_h;
            s = std::sin(0.5 * t);
            ang = (1.0 + std::cos(t) * std::cos(t)) * std::cos(0.5 * t);
        }
        bp[b] = make_float2(sb[b], b + 1 < nb ? (float)(1.0 / ((double)sb[b + 1] - (double)sb[b])) : 0.0f);
        std::fill(row.begin(), row.end(), 0.0);
        for (int k = 0; k < K; k++) {
            const double u = alpha[k] * s - beta0;
            const double j0 = std::floor(u), t = u - j0;
            const long j = (long)j0;
            if (j >= 0 && j < Q) row[j] += ck[k] * (1.0 - t);
            if (j + 1 >= 0 && j + 1 < Q) row[j + 1] += ck[k] * t;
        }
        for (int j = 0; j < Q; j++) stab[(size_t)b * Q + j] = (float)(row[j] * ang);
    }
    // LUT over the fp32 bit patterns of [s_0, s_{nb-1}]: nl = (span >> sh) + 1
    // <= ~4 nb cells (device locate above); 15-bit entries + the slow flag
    if (nb > (int)kLutSlow - 1) {  // outside the LUT's index range: per-term kernels
        g->esai.enabled = 0;
        return cudaSuccess;
    }
    const int b0 = fbits(sb[0]);
    const long long span = (long long)fbits(sb[nb - 1]) - b0;
    const long long target = std::min<long long>(32768, std::max(64, 4 * nb));
    int sh = 0;
    while ((span >> sh) + 1 > target) sh++;
    const int nl = (int)(span >> sh) + 1;
    std::vector<uint16_t> lut(nl);
    int n_slow = 0;
    for (int c = 0; c < nl; c++) {
        const int c0 = b0 + (int)((long long)c << sh);
        const long long c1 = (long long)b0 + ((long long)(c + 1) << sh) - 1;  // last float of the cell
        int b = host_locate(sb, ffrom(c0));
        int inside = 0;
        for (int i = b + 1; i < nb && fbits(sb[i]) <= c1; i++)
            if (fbits(sb[i]) > c0) inside++;
        lut[c] = (uint16_t)b;
        if (inside > kLocD) {
            lut[c] |= (uint16_t)kLutSlow;
            n_slow++;
        }
    }
    // per-voxel breakpoint windows (deposits land in [locate(min), locate(max) + 1])
    std::vector<int2> vwin(nv);
    int max_win = 1;
    long long win_sum = 0;
    for (int v = 0; v < nv; v++) {
        vwin[v] = make_int2(host_locate(sb, shmin[v]), host_locate(sb, shmax[v]) + 1);
        max_win = std::max(max_win, vwin[v].y - vwin[v].x + 1);
        win_sum += vwin[v].y - vwin[v].x + 1;
    }
    // per 128-voxel GEMM tile: the union of its voxels' windows.  Neither contraction
    // needs W or A outside it (the forward reads W only inside each voxel's window,
    // the backward deposits only there), so the W GEMM skips N tiles and the b2 GEMM
    // K chunks outside it, and the backward writes A rows only inside it.
    std::vector<int2> trng((nv + 127) / 128);
    {
        long long tile_span = 0;
        for (int m0 = 0; m0 < nv; m0 += 128) {
            int lo = 1 << 30, hi = 0;
            for (int v = m0; v < std::min(nv, m0 + 128); v++) {
                lo = std::min(lo, vwin[v].x);
                hi = std::max(hi, vwin[v].y + 1);
            }
            trng[m0 / 128] = make_int2(lo, hi);
            tile_span += (long long)(((hi + 31) / 32) - lo / 32) * 32;
        }
        g->esai.stat_win_permille = (int)(1000 * win_sum / ((long long)nv * nb));
        g->esai.stat_tile_permille = (int)(1000 * tile_span / ((long long)((nv + 127) / 128) * nb));
    }
    e = cudaMalloc(&g->d_esai_bp, nb * sizeof(float2));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_esai_bp, bp.data(), nb * sizeof(float2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_esai_lut, nl * sizeof(uint16_t));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_esai_lut, lut.data(), nl * sizeof(uint16_t), cudaMemcpyHostToDevice);
    std::vector<float> sbp(sb);
    for (int i = 0; i < kLocD; i++) sbp.push_back(INFINITY);  // pads: the branch-free count never passes them
    if (e == cudaSuccess) e = cudaMalloc(&g->d_esai_sb, sbp.size() * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_esai_sb, sbp.data(), sbp.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_esai_stab, stab.size() * sizeof(float));
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_esai_stab, stab.data(), stab.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_esai_vwin, nv * sizeof(int2));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_esai_vwin, vwin.data(), nv * sizeof(int2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_esai_trng, trng.size() * sizeof(int2));
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_esai_trng, trng.data(), trng.size() * sizeof(int2), cudaMemcpyHostToDevice);
    // the W GEMM's tile list: per M tile the N tiles (128 bins) covering [lo & ~3, hi) -- the
    // forward stages each voxel's W window from win.x & ~3 -- and their prefix count
    const int mtl = (int)trng.size();
    std::vector<int> wtl(2 * mtl + mtl + 1);  // [mtl] int2 ranges, then [mtl + 1] prefix
    {
        int2 *ntr = (int2 *)wtl.data();
        int *pre = wtl.data() + 2 * mtl;
        pre[0] = 0;
        for (int m = 0; m < mtl; m++) {
            const int lo = trng[m].x & ~3, hi = trng[m].y;
            ntr[m] = hi > lo ? make_int2(lo / 128, (hi - 1) / 128) : make_int2(0, -1);
            pre[m + 1] = pre[m] + (ntr[m].y - ntr[m].x + 1);
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&g->d_w_tiles, wtl.size() * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_w_tiles, wtl.data(), wtl.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    Esai &E = g->esai;
    E.nb = nb;
    E.nl = nl;
    E.lut_b0 = b0;
    E.lut_sh = sh;
    E.n_slow = n_slow;
    E.sai_i0 = sai_i0;
    E.lut16 = (const uint16_t *)g->d_esai_lut;
    E.sb = (const float *)g->d_esai_sb;
    E.stab = (const float *)g->d_esai_stab;
    E.vwin = (const int2 *)g->d_esai_vwin;
    E.trng = (const int2 *)g->d_esai_trng;
    E.w_ntr = (const int2 *)g->d_w_tiles;
    E.w_pre = (const int *)g->d_w_tiles + 2 * mtl;
    E.ptot = (const float *)g->d_esai_ptot;
    E.max_win = max_win;
    // tensor-core operands: S~ (N = nb, K = nq) for W = F S~^T and S~^T (N = nq, K = nb) for b2 = A S~,
    // pre-split into TF32 hi / lo and pre-swizzled (tcgemm.cuh)
    E.ldw = (nb + 31) / 32 * 32;
    {
        // packed on the device from S~ (already uploaded): the same arithmetic as the host
        // tc_pack_b (tf32 truncation and an exact subtraction), so the same bits
        const int nkcW = (Q + TC_KC - 1) / TC_KC, nkcB = E.ldw / TC_KC;
        const size_t nW = (size_t)tc_ntiles(nb, TC_PSTRIDE) * nkcW * 2 * TC_N * TC_KC;  // W2 pairs (stride 126)
        const size_t nB = (size_t)((Q + TC_N - 1) / TC_N) * nkcB * 2 * TC_N * TC_KC;    // S~^T for b2 = A S~
        const size_t nW1 = (size_t)tc_ntiles(nb, TC_N) * nkcW * 2 * TC_N * TC_KC;      // plain W tiles
        e = cudaMalloc(&g->d_tc_w, nW * sizeof(float));
        if (e == cudaSuccess) e = cudaMalloc(&g->d_tc_b, nB * sizeof(float));
        if (e == cudaSuccess) e = cudaMalloc(&g->d_tc_w1, nW1 * sizeof(float));
        if (e != cudaSuccess) return e;
        const float *st = (const float *)g->d_esai_stab;
        const int gp = 8 * sm_count(g->device);
        k_tc_pack_b<<<gp, 256>>>(st, nb, Q, Q, 1, nkcW, (float *)g->d_tc_w, TC_PSTRIDE);
        k_tc_pack_b<<<gp, 256>>>(st, Q, nb, 1, Q, nkcB, (float *)g->d_tc_b, TC_N);   // B = S~^T (transposed read)
        k_tc_pack_b<<<gp, 256>>>(st, nb, Q, Q, 1, nkcW, (float *)g->d_tc_w1, TC_N);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        E.tc_w = (const float *)g->d_tc_w;
        E.tc_w1 = (const float *)g->d_tc_w1;
        E.tc_b = (const float *)g->d_tc_b;
        // fp16 two-term split of the same operands (tcgemm16.cuh, option gemm16), one global
        // power-of-two scale from max |S~|
        float smax = 0.0f;
        for (float x : stab) smax = std::max(smax, std::fabs(x));
        E.s16_exp = f16_scale_exp(smax);
        const int nk16W = (Q + TC16_KC - 1) / TC16_KC, nk16B = (E.ldw + TC16_KC - 1) / TC16_KC;
        const size_t n16W = (size_t)tc_ntiles(nb, TC_N) * nk16W * 2 * TC_N * TC16_KC;
        const size_t n16B = (size_t)((Q + TC_N - 1) / TC_N) * nk16B * 2 * TC_N * TC16_KC;
        e = cudaMalloc(&g->d_tc16_w1, n16W * sizeof(__half));
        if (e == cudaSuccess) e = cudaMalloc(&g->d_tc16_b, n16B * sizeof(__half));
        if (e != cudaSuccess) return e;
        k_tc_pack_b16<<<gp, 256>>>(st, nb, Q, Q, 1, nk16W, (__half *)g->d_tc16_w1, E.s16_exp);
        k_tc_pack_b16<<<gp, 256>>>(st, Q, nb, 1, Q, nk16B, (__half *)g->d_tc16_b, E.s16_exp);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        E.tc16_w1 = g->d_tc16_w1;
        E.tc16_b = g->d_tc16_b;
    }
    clk.mark(0);  // pair stats, breakpoints, S~, LUT, windows, tensor-core operand tiles
    // transmission bitmaps
    {
        const size_t nfw = p.ts_rho > 0 ? (size_t)p.nz * p.det_nx * ((p.ny + 31) / 32) * p.det_ny
                                        : (size_t)((p.n_vox + 31) / 32) * p.n_det;
        const size_t nbw = (size_t)p.n_vox * ((p.n_det + 31) / 32);
        e = cudaMalloc(&g->d_tb_fwd, nfw * sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMalloc(&g->d_tb_bwd, nbw * sizeof(uint32_t));
        if (e != cudaSuccess) return e;
        const int blocks = 8 * sm_count(g->device);
        if (p.ts_rho > 0)
            k_tbits_fwd_ts<<<blocks, 256>>>(p, (uint32_t *)g->d_tb_fwd);
        else
            k_tbits_fwd_tiled<<<blocks, 256>>>(p, (uint32_t *)g->d_tb_fwd);
        k_tbits_bwd<<<blocks, 256>>>(p, (uint32_t *)g->d_tb_bwd);
        const int nwd = (p.n_det + 31) / 32;
        e = cudaMalloc(&g->d_seen, nwd * sizeof(uint32_t));
        if (e == cudaSuccess) {
            e = cudaMemset(g->d_seen, 0, nwd * sizeof(uint32_t));
            k_seen<<<dim3((nwd + 127) / 128, std::min(p.n_vox, 256)), 128>>>(p, (const uint32_t *)g->d_tb_bwd,
                                                                              (uint32_t *)g->d_seen);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
        }
        if (e != cudaSuccess) return e;
        E.seen = (const uint32_t *)g->d_seen;
        clk.mark(1);  // transmission bitmaps
        E.tb_fwd = (const uint32_t *)g->d_tb_fwd;
        E.tb_bwd = (const uint32_t *)g->d_tb_bwd;
    }
    if ((double)nv * E.ldw >= 4294967296.0) {  // W / A offsets are 32-bit in the pair kernels
        E.enabled = 0;
        return cudaSuccess;
    }
    // shared-memory budgets of the pair kernels (227 KB per CTA); beyond them the
    // per-term kernels serve the handle
    {
        const size_t fwd = p.ts_rho > 0 ? host_bp_bytes(E) + (size_t)TS_R * (TS_T + p.ts_rho * (p.ny - 1)) * 8
                                        : host_bp_bytes(E);
        const size_t bwd = bwd_smem_bytes(host_bp_bytes(E), E.max_win);
        if (fwd > 227 * 1024 || bwd > 227 * 1024) {
            E.enabled = 0;
            return cudaSuccess;
        }
    }
    // backward fixed-point bound: vbound[v] >= max_b sum_pixels P hat_b, measured
    // with w = 1 under the conservative scale sum_pixels |P| (k_esai_bwd)
    {
        float *A1 = nullptr;
        e = cudaMalloc(&g->d_esai_vbound, nv * sizeof(float));
        if (e == cudaSuccess) e = cudaMalloc(&A1, (size_t)nv * E.ldw * sizeof(float));
        if (e == cudaSuccess) {
            const size_t smem = bwd_smem_bytes(host_bp_bytes(E), E.max_win);
            auto kb = sai ? k_esai_bwd<true, true> : k_esai_bwd<true, false>;
            cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kb<<<persistent_grid(g, smem, PB_T), PB_T, smem>>>(p, E, nullptr, nullptr, E.ptot, nullptr, A1);
            k_vbound<<<nv, 256>>>(A1, E.ldw, E.ptot, p.n_det, (float *)g->d_esai_vbound);
            e = cudaDeviceSynchronize();
        }
        cudaFree(A1);
        if (e != cudaSuccess) return e;
        E.vbound = (const float *)g->d_esai_vbound;
        {
            std::vector<float> vb(nv);
            e = cudaMemcpy(vb.data(), g->d_esai_vbound, nv * sizeof(float), cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return e;
            E.vbmax = 0.0f;
            for (float x : vb) E.vbmax = std::max(E.vbmax, x);
        }
        clk.mark(2);  // fixed-point bound pass
    }
    // pair cache (above): counts -> device scan -> fill, if it fits in half the free memory
    E.pc = 0;
    E.pc_segwin = nullptr;
    if (g->opt.pair_cache && (size_t)p.det_ny <= 65535) {
        const size_t nl = (size_t)nv * p.det_nx;
        // segments (voxel, block of R rows) of the voxel-major forward, padded to
        // multiples of 128 records (the padding belongs to the segment's last list)
        const int n_rb = pcv_row_blocks(g);
        const int R = n_rb > 0 ? (p.det_nx + n_rb - 1) / n_rb : 0;
        const int segR = (R > 0 && !g->opt.pc_plain) ? R : 0;  // pc_plain: no padding / bank-aware order
        long long *cnt = nullptr, *tot = nullptr;
        void *tmp = nullptr;
        size_t tmp_b = 0;
        e = cudaMalloc(&g->d_pc_off, (nl + 1) * sizeof(long long));
        if (e == cudaSuccess) e = cudaMalloc(&cnt, (nl + 1) * sizeof(long long));
        if (e == cudaSuccess) e = cudaMalloc(&tot, 2 * sizeof(long long));
        if (e == cudaSuccess)
            e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_b, cnt, (long long *)g->d_pc_off, (int)(nl + 1));
        if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_b);
        long long ht[2] = {0, 0};
        if (e == cudaSuccess) {
            e = cudaMemset(tot, 0, 2 * sizeof(long long));
            k_pc_count<<<8 * sm_count(g->device), 256>>>(p, E, cnt, nl);
            k_pc_pad<<<8 * sm_count(g->device), 256>>>(p, segR, g->opt.pc_win, cnt, tot);
            if (e == cudaSuccess)
                e = cub::DeviceScan::ExclusiveSum(tmp, tmp_b, cnt, (long long *)g->d_pc_off, (int)(nl + 1));
            if (e == cudaSuccess) e = cudaMemcpy(ht, tot, sizeof(ht), cudaMemcpyDeviceToHost);  // syncs
        }
        cudaFree(cnt);
        cudaFree(tot);
        cudaFree(tmp);
        if (e != cudaSuccess) return e;
        const long long nopen = ht[0], nrec = ht[1];
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        const size_t jyb = p.n_det <= 65536 ? 2 : 4;
        // + 8 records of padding: bulk copies read whole 8-record groups (16-byte aligned)
        const size_t rec = (size_t)std::max(nrec, 1ll) + 8;
        const size_t need = rec * (sizeof(uint32_t) + sizeof(float) + jyb);
        int bbits = 1;
        while ((1 << bbits) < E.nb) bbits++;
        // the cache may take half of the free memory (the permutation runs in place)
        if (!(need <= free_b / 2 && bbits <= 16)) {
            cudaFree(g->d_pc_off);
            g->d_pc_off = nullptr;
        } else {
            if (e == cudaSuccess) e = cudaMalloc(&g->d_pc_bt, rec * sizeof(uint32_t));
            if (e == cudaSuccess) e = cudaMalloc(&g->d_pc_P, rec * sizeof(float));
            if (e == cudaSuccess) e = cudaMalloc(&g->d_pc_q, rec * jyb);
            if (e != cudaSuccess) return e;
            E.pc_off = (const long long *)g->d_pc_off;
            E.pc_bt = (const uint32_t *)g->d_pc_bt;
            E.pc_P = (const float *)g->d_pc_P;
            E.pc_q = g->d_pc_q;
            E.pc_tbits = std::min(32 - bbits, 24);  // tau's fp32 mantissa carries 24 bits
            E.pc_qb = (int)jyb;
            E.pc_n = nrec;
            E.pc_nopen = nopen;
            E.pc_R = segR;
            const size_t smem = host_bp_bytes(E);
            const int gr = persistent_grid(g, smem, 256);
            int *unsafe = nullptr;
            e = cudaMalloc(&unsafe, sizeof(int));
            if (e == cudaSuccess) e = cudaMemset(unsafe, 0, sizeof(int));
            if (e != cudaSuccess) return e;
            if (jyb == 2) {
                auto kf = sai ? k_pc_fill<true, uint16_t> : k_pc_fill<false, uint16_t>;
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                kf<<<gr, 256, smem>>>(p, E, (uint32_t *)g->d_pc_bt, (float *)g->d_pc_P, (uint16_t *)g->d_pc_q, unsafe);
            } else {
                auto kf = sai ? k_pc_fill<true, uint32_t> : k_pc_fill<false, uint32_t>;
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                kf<<<gr, 256, smem>>>(p, E, (uint32_t *)g->d_pc_bt, (float *)g->d_pc_P, (uint32_t *)g->d_pc_q, unsafe);
            }
            e = cudaDeviceSynchronize();
            int hu = 1;
            if (e == cudaSuccess) e = cudaMemcpy(&hu, unsafe, sizeof(int), cudaMemcpyDeviceToHost);
            cudaFree(unsafe);
            if (e != cudaSuccess) return e;
            E.pc_padq = (segR > 0 && hu == 0) ? 1 : 0;
            clk.mark(3);  // pair cache: count, scan, allocation, fill
            E.pcb_bt = E.pc_bt;
            E.pcb_P = E.pc_P;
            E.pcb_q = E.pc_q;
            if (segR > 0) {
                // bank-aware order, permuted in place (one copy serves both operators: a
                // separate cells-only copy for the backward measured no faster)
                {
                    const int gr2 = 8 * sm_count(g->device);
                    uint32_t *kb = (uint32_t *)g->d_pc_bt;
                    float *Pb = (float *)g->d_pc_P;
                    const int wn = g->opt.pc_win;
                    if (wn == 128 && g->opt.pc_perm_lane && E.pc_n % 128 == 0) {
                        // one window per lane (bit-identical to k_pc_perm<., 128>)
                        const size_t sm = (size_t)PERM2_W * 5 * 4096;
                        const long long nwin = E.pc_n / 128;
                        const int gr3 = 2 * sm_count(g->device);
                        if (jyb == 2) {
                            cudaFuncSetAttribute(k_pc_perm128<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                            k_pc_perm128<uint16_t><<<gr3, PERM2_W * 32, sm>>>(nwin, E.pc_tbits, kb, Pb, (uint16_t *)g->d_pc_q);
                        } else {
                            cudaFuncSetAttribute(k_pc_perm128<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                            k_pc_perm128<uint32_t><<<gr3, PERM2_W * 32, sm>>>(nwin, E.pc_tbits, kb, Pb, (uint32_t *)g->d_pc_q);
                        }
                    } else if (jyb == 2) {
                        uint16_t *qb = (uint16_t *)g->d_pc_q;
                        if (wn == 512) k_pc_perm<uint16_t, 512><<<gr2, PERM_W * 32>>>(p, E, segR, kb, Pb, qb);
                        else if (wn == 256) k_pc_perm<uint16_t, 256><<<gr2, PERM_W * 32>>>(p, E, segR, kb, Pb, qb);
                        else k_pc_perm<uint16_t, 128><<<gr2, PERM_W * 32>>>(p, E, segR, kb, Pb, qb);
                    } else {
                        uint32_t *qb = (uint32_t *)g->d_pc_q;
                        if (wn == 512) k_pc_perm<uint32_t, 512><<<gr2, PERM_W * 32>>>(p, E, segR, kb, Pb, qb);
                        else if (wn == 256) k_pc_perm<uint32_t, 256><<<gr2, PERM_W * 32>>>(p, E, segR, kb, Pb, qb);
                        else k_pc_perm<uint32_t, 128><<<gr2, PERM_W * 32>>>(p, E, segR, kb, Pb, qb);
                    }
                    e = cudaDeviceSynchronize();
                }
                if (e != cudaSuccess) return e;
                clk.mark(4);  // bank-aware permutation
                E.pcb_bt = E.pc_bt;
                E.pcb_P = E.pc_P;
                E.pcb_q = E.pc_q;
                // per-segment W windows for the voxel-major forward (and the padding re-binned
                // inside them)
                const size_t nseg = (size_t)nv * ((p.det_nx + segR - 1) / segR);
                e = cudaMalloc(&g->d_pc_segwin, nseg * sizeof(int2));
                if (e == cudaSuccess) {
                    k_pc_segwin<<<8 * sm_count(g->device), 256>>>(p, E, segR, (uint32_t *)g->d_pc_bt,
                                                                 (const float *)g->d_pc_P, (int2 *)g->d_pc_segwin);
                    e = cudaDeviceSynchronize();
                }
                if (e != cudaSuccess) return e;
                if (g->opt.pc_segwin) E.pc_segwin = (const int2 *)g->d_pc_segwin;
                // 8-byte records: a 9-bit pixel offset per record and a base per 128-record
                // window, if every window's pixel span fits and tau keeps >= 9 bits
                E.pc_q8 = 0;
                const int q8mode = g->opt.pc_q8;
                E.pc_tb8 = q8mode == 2 ? E.pc_tbits - 5 : E.pc_tbits - 9;
                if (q8mode && jyb == 2 && E.pc_tb8 >= 9 && (nrec % 128) == 0) {
                    const long long nwin = nrec / 128;
                    unsigned *span = nullptr;
                    unsigned hs = 0;
                    e = cudaMalloc(&span, sizeof(unsigned));
                    if (e == cudaSuccess) e = cudaMemset(span, 0, sizeof(unsigned));
                    if (e == cudaSuccess) {
                        k_pc_qspan<<<8 * sm_count(g->device), 256>>>(nwin, (const uint16_t *)g->d_pc_q, span);
                        e = cudaMemcpy(&hs, span, sizeof(unsigned), cudaMemcpyDeviceToHost);
                    }
                    cudaFree(span);
                    if (e == cudaSuccess && hs <= 511) {
                        // + 32 bases of slack: the backward's bulk copy of a chunk's bases reads whole 16-byte groups
                        e = cudaMalloc(&g->d_pc_qbase, (size_t)(nwin + 32) * sizeof(uint16_t));
                        if (e == cudaSuccess) e = cudaMemset(g->d_pc_qbase, 0, (size_t)(nwin + 32) * sizeof(uint16_t));
                        if (e == cudaSuccess) {
                            k_pc_pack8<<<8 * sm_count(g->device), 256>>>(nwin, E.pc_tbits, E.pc_tb8, q8mode,
                                                                          (const uint16_t *)g->d_pc_q, (uint32_t *)g->d_pc_bt,
                                                                          (float *)g->d_pc_P, (uint16_t *)g->d_pc_qbase);
                            e = cudaDeviceSynchronize();
                        }
                        if (e == cudaSuccess) {
                            cudaFree(g->d_pc_q);
                            g->d_pc_q = nullptr;
                            E.pc_q = E.pcb_q = nullptr;
                            E.pc_qbase = (const uint16_t *)g->d_pc_qbase;
                            E.pc_q8 = q8mode;
                        }
                    }
                    if (e != cudaSuccess) return e;
                }
                clk.mark(5);  // per-segment windows, 8-byte packing
            }
            E.pc = 1;
        }
    }
    E.enabled = 1;
    return cudaSuccess;
}

static cudaError_t esai_forward_impl(const cacsi_geometry *g, const float *f, const int32_t *pixels, int n_pix,
                                     float *out, cudaStream_t s, int *launches, const FwdRatioEpi *epi = nullptr);
static bool tmap_rows_f32(CUtensorMap *tm, const float *base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t box_rows = TC_M);

// Row blocks of the voxel-major pair-cache forward (0: the W windows do not fit
// shared memory, the per-list kernel runs).  One 1024-thread CTA per SM with a
// large row block (fewer W window re-stagings, longer per-voxel record runs)
// measured faster than two 512-thread CTAs.
int pcv_row_blocks(const cacsi_geometry *g) {
    const Esai &E = g->esai;
    const Params &p = g->p;
    // a bank-ordered cache fixes the segments (records are permuted across the
    // lists of a segment): the forward must use exactly those row blocks
    if (E.pc && E.pc_R > 0) return (p.det_nx + E.pc_R - 1) / E.pc_R;
    const int wcap = (E.max_win + 3 + 3) & ~3;
    const size_t budget = (size_t)g->opt.pcv_budget_kb * 1024;  // KB of shared memory per CTA
    const long long acc_max = (long long)budget - 2ll * wcap * (long long)sizeof(float) - 32 - 128;
    const int r_max = acc_max > 0 ? (int)(acc_max / ((long long)p.det_ny * sizeof(float))) : 0;
    return r_max >= 1 ? (p.det_nx + r_max - 1) / r_max : 0;
}

cudaError_t esai_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches) {
    return esai_forward_impl(g, f, nullptr, 0, out, s, launches);
}

cudaError_t esai_forward_list(const cacsi_geometry *g, const float *f, const int32_t *pixels, int n, float *out,
                              cudaStream_t s, int *launches) {
    return esai_forward_impl(g, f, pixels, n, out, s, launches);
}

cudaError_t esai_forward_ratio(const cacsi_geometry *g, const float *f, const FwdRatioEpi &epi, float *w,
                               cudaStream_t s, int *launches) {
    return esai_forward_impl(g, f, nullptr, 0, w, s, launches, &epi);
}

static cudaError_t esai_forward_impl(const cacsi_geometry *g, const float *f, const int32_t *pixels, int n_pix,
                                     float *out, cudaStream_t s, int *launches, const FwdRatioEpi *epi) {
    const Params &p = g->p;
    const Esai &E = g->esai;
    float *W = nullptr;
    double *part = nullptr;
    const size_t bpb = host_bp_bytes(E);
    int S;  // number of partial images
    float *fp = nullptr;
    const int ldf = (p.nq + TC_KC - 1) / TC_KC * TC_KC;
    cudaError_t e = cudaMallocAsync(&W, (size_t)p.n_vox * E.ldw * sizeof(float2), s);  // W2 pairs
    // packed A tiles: [ceil(n_vox / 128)][ldf / 32][hi, lo][128 x 32]
    // (an even tile count: the CTA-pair W GEMM takes M tiles two at a time; the spare tile is zero)
    const size_t mt_even = ((size_t)(p.n_vox + TC_M - 1) / TC_M + 1) & ~(size_t)1;
    if (e == cudaSuccess) e = cudaMallocAsync(&fp, mt_even * TC_M * ldf * 2 * sizeof(float), s);
    if (e == cudaSuccess && mt_even * TC_M > (size_t)(p.n_vox + TC_M - 1) / TC_M * TC_M) {
        const size_t tile = (size_t)TC_M * ldf * 2;
        e = cudaMemsetAsync(fp + (mt_even - 1) * tile, 0, tile * sizeof(float), s);
    }
    if (e != cudaSuccess) {
        if (W) cudaFreeAsync(W, s);
        return e;
    }
    const int nkcA = ldf / TC_KC;
    const Opts &o = g->opt;
    const bool ar_path = ((E.pc && pixels == nullptr) || pixels != nullptr) && nkcA <= 4 && o.wgemm == 0;
    const int nfc = (epi && epi->f_chunks > 0) ? epi->f_chunks : 0;
    // the A-resident W GEMM reads f itself (TMA tensor loads + in-kernel TF32 split) when
    // f's rows are 16-byte multiples; otherwise k_tc_pack_a pre-splits it
    CUtensorMap tmF;
    memset(&tmF, 0, sizeof(tmF));
    const bool raw = ar_path && (p.nq % 4) == 0 && !o.wgemm_pack &&
                     tmap_rows_f32(&tmF, f, (uint64_t)p.n_vox, (uint64_t)p.nq, (uint64_t)p.nq);
    // option gemm16: the same A-resident GEMM on a two-term fp16 split (tcgemm16.cuh)
    // (option w_tmast: the epilogue stores W by TMA tensor stores, tmW: box 32 x 32)
    CUtensorMap tmW;
    memset(&tmW, 0, sizeof(tmW));
    const bool f16 = raw && o.gemm16;
    const bool tmast = f16 && o.w_tmast && tmap_rows_f32(&tmW, W, (uint64_t)p.n_vox, (uint64_t)E.nb, (uint64_t)E.ldw, 32);
    const int nk16 = (p.nq + TC16_KC - 1) / TC16_KC;
    const int nsb16 = tca16_smem(nk16, 4, tmast) <= 227 * 1024 ? 4 : 3;
    auto kar16 = tmast ? (nsb16 == 4 ? k_tc_gemm_ar16<4, true> : k_tc_gemm_ar16<3, true>)
                       : (nsb16 == 4 ? k_tc_gemm_ar16<4> : k_tc_gemm_ar16<3>);
    if (f16) cudaFuncSetAttribute(kar16, cudaFuncAttributeMaxDynamicSharedMemorySize, tca16_smem(nk16, nsb16, tmast));
    if (nfc > 0 && !ar_path)
        for (int c = 0; c < nfc && e == cudaSuccess; c++) e = cudaStreamWaitEvent(s, epi->f_ready[c], 0);
    if (nfc > 0 && ar_path) {
        // f staged from the host in row chunks: pack + W GEMM per chunk as it lands, so the
        // upload of chunk c + 1 overlaps the contraction of chunk c (cacsi_iterate_host)
        const int rows = fchunk_rows(p.n_vox, nfc), nt = tc_ntiles(E.nb, TC_N);
        const int nsb = tca_smem(nkcA, 3) <= 227 * 1024 ? 3 : 2;
        auto kar = raw ? (nsb == 3 ? k_tc_gemm_ar<3, true> : k_tc_gemm_ar<2, true>)
                       : (nsb == 3 ? k_tc_gemm_ar<3> : k_tc_gemm_ar<2>);
        cudaFuncSetAttribute(kar, cudaFuncAttributeMaxDynamicSharedMemorySize, tca_smem(nkcA, nsb));
        for (int c = 0; c < nfc && e == cudaSuccess; c++) {
            const int r0 = c * rows;
            e = cudaStreamWaitEvent(s, epi->f_ready[c], 0);
            if (r0 >= p.n_vox || e != cudaSuccess) continue;
            const int nr = std::min(rows, p.n_vox - r0), mtc = (nr + TC_M - 1) / TC_M;
            float *fpc = fp + (size_t)(r0 / TC_M) * nkcA * (2 * TC_M * TC_KC);
            if (!raw) {
                KScope kt_(g, s, "k_tc_pack_a");
                k_tc_pack_a<<<4 * sm_count(g->device), 256, 0, s>>>(f + (size_t)r0 * p.nq, nr, p.nq, p.nq, nkcA, fpc);
                *launches += 1;
            }
            {
                KScope kt_(g, s, "k_tc_gemm_W");
                if (f16)
                    kar16<<<std::min(mtc * nt, sm_count(g->device)), TCA16_T, tca16_smem(nk16, nsb16, tmast), s>>>(
                        nr, E.nb, nk16, mtc, nt, (const __half *)E.tc16_w1, W + (size_t)r0 * E.ldw, E.ldw,
                        E.w_pre + r0 / TC_M, E.w_ntr + r0 / TC_M, tmF, r0, E.s16_exp, tmW);
                else
                    kar<<<std::min(mtc * nt, sm_count(g->device)), raw ? TCA_T1R : TCA_T1, tca_smem(nkcA, nsb), s>>>(
                        nr, E.nb, nkcA, mtc, nt, fpc, E.tc_w1, W + (size_t)r0 * E.ldw, E.ldw, E.w_pre + r0 / TC_M,
                        E.w_ntr + r0 / TC_M, tmF, r0);
            }
            *launches += 1;
        }
        *launches -= 2;  // counted again below (pack + GEMM)
    } else if (raw) {
        *launches -= 1;  // no pack pass: the W GEMM loads and splits f itself
    } else {
        // f -> pre-split (TF32 hi / lo), pre-swizzled A tiles: the GEMM lands them by bulk copy
        KScope kt_(g, s, "k_tc_pack_a");
        k_tc_pack_a<<<4 * sm_count(g->device), 256, 0, s>>>(f, p.n_vox, p.nq, p.nq, nkcA, fp);
    }
    if (!(nfc > 0 && ar_path)) {
        // W[v][b] = sum_j f[v][j] S~[b][j] on the tensor cores (3xTF32)
        KScope kt_(g, s, "k_tc_gemm_W");
        if ((E.pc && pixels == nullptr) || pixels != nullptr) {
            // plain W rows (n_vox x ldw fp32): the pair-cache and the subset forwards gather W_b
            // and W_{b+1}; the pair layout below serves the full on-the-fly kernels
            const int nt = tc_ntiles(E.nb, TC_N), mt = (p.n_vox + TC_M - 1) / TC_M;
            if (nkcA <= 4 && o.wgemm == 1) {
                // the CTA-pair (cta_group::2) variant: bit-identical, measured slower
                const int mp = (int)(mt_even / 2);
                cudaFuncSetAttribute(k_tc_gemm_ar2, cudaFuncAttributeMaxDynamicSharedMemorySize, tca2_smem(nkcA));
                const int npairs = std::max(1, std::min(mp * nt, sm_count(g->device) / 2));
                k_tc_gemm_ar2<<<2 * npairs, TCA_T1, tca2_smem(nkcA), s>>>(p.n_vox, E.nb, nkcA, mp, nt, fp, E.tc_w1, W,
                                                                        E.ldw);
            } else if (f16) {
                kar16<<<std::min(mt * nt, sm_count(g->device)), TCA16_T, tca16_smem(nk16, nsb16, tmast), s>>>(
                    p.n_vox, E.nb, nk16, mt, nt, (const __half *)E.tc16_w1, W, E.ldw, E.w_pre, E.w_ntr, tmF, 0,
                    E.s16_exp, tmW);
            } else if (nkcA <= 4 && o.wgemm == 0) {
                // B ring depth: 3 stages where they fit beside the resident A panel (nkc <= 2), else 2
                // (config 2, nq = 128: nkc = 4, the 128 KB panel leaves room for 2)
                const int nsb = tca_smem(nkcA, 3) <= 227 * 1024 ? 3 : 2;
                auto kar = raw ? (nsb == 3 ? k_tc_gemm_ar<3, true> : k_tc_gemm_ar<2, true>)
                               : (nsb == 3 ? k_tc_gemm_ar<3> : k_tc_gemm_ar<2>);
                cudaFuncSetAttribute(kar, cudaFuncAttributeMaxDynamicSharedMemorySize, tca_smem(nkcA, nsb));
                // only the N tiles inside each M tile's window union (E.w_pre / w_ntr; ~84 % on
                // config 2), split evenly over the CTAs; W outside them is never read
                kar<<<std::min(mt * nt, sm_count(g->device)), raw ? TCA_T1R : TCA_T1, tca_smem(nkcA, nsb), s>>>(
                    p.n_vox, E.nb, nkcA, mt, nt, fp, E.tc_w1, W, E.ldw, E.w_pre, E.w_ntr, tmF, 0);
            } else {
                dim3 gg(nt, mt, 1);
                cudaFuncSetAttribute(k_tc_gemm<false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(1));
                k_tc_gemm<false, 1, true><<<gg, TC_T, tc_smem(1), s>>>(p.n_vox, E.nb, p.nq, ldf, nkcA, nkcA, fp,
                                                                      E.tc_w1, W, E.ldw);
            }
        } else {
            dim3 gg(tc_ntiles(E.nb, TC_PSTRIDE), (p.n_vox + TC_M - 1) / TC_M, 1);
            cudaFuncSetAttribute(k_tc_gemm<true, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(1));
            k_tc_gemm<true, 1, true><<<gg, TC_T, tc_smem(1), s>>>(p.n_vox, E.nb, p.nq, ldf, nkcA, nkcA, fp, E.tc_w, W,
                                                                 E.ldw);
        }
    }
    if (pixels != nullptr) {
        // subset: g = 0 outside the list, listed pixels by k_esai_fwd_list
        e = cudaMemsetAsync(out, 0, (size_t)p.n_det * sizeof(float), s);
        const int n_chunks = (n_pix + PL_T - 1) / PL_T;
        const int grid = persistent_grid(g, bpb, PL_T);
        // voxel splits of 16 (half a bit batch): twice the threads of 32-voxel splits and
        // half the dependent pair chain per thread (a subset has few pixels)
        S = std::max(1, std::min((8 * grid + n_chunks - 1) / n_chunks, (p.n_vox + 15) / 16));
        int vps = (p.n_vox + S - 1) / S;
        vps = (vps + 15) / 16 * 16;
        S = (p.n_vox + vps - 1) / vps;
        if (e == cudaSuccess) e = cudaMallocAsync(&part, (size_t)S * n_pix * sizeof(double), s);
        if (e == cudaSuccess) {
            {
                KScope kt_(g, s, "k_esai_fwd_list");
                auto kl = p.sai_n > 0 ? k_esai_fwd_list<true> : k_esai_fwd_list<false>;
                cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bpb);
                kl<<<grid, PL_T, bpb, s>>>(p, E, W, pixels, n_pix, vps, n_chunks * S, part);
            }
            {
                KScope kt_(g, s, "k_sum_list");
                k_sum_list<<<std::min((n_pix + 7) / 8, 8 * sm_count(g->device)), 256, 0, s>>>(part, S, pixels, n_pix,
                                                                                               out);
            }
        }
        if (e == cudaSuccess) e = cudaGetLastError();
        *launches += 4;
        if (part) cudaFreeAsync(part, s);
        cudaFreeAsync(fp, s);
        cudaFreeAsync(W, s);
        return e;
    } else if (E.pc) {
        const int wcap = (E.max_win + 3 + 3) & ~3;
        const int n_rb = pcv_row_blocks(g);
        if (n_rb > 0 && (E.pc_R > 0 || !o.pc_fwd_list)) {  // pc_fwd_list: per-list kernel (plain layout only)
            // voxel-major: items (voxel chunk, row block), fp64 partials per voxel chunk
            const int R = (p.det_nx + n_rb - 1) / n_rb;
            const int ipsm = o.pcv_items;  // voxel chunks per SM
            int Sv = std::max(1, std::min(p.n_vox, (ipsm * sm_count(g->device) + n_rb - 1) / n_rb));
            const int vchunk = (p.n_vox + Sv - 1) / Sv;
            const int n_chunks = (p.n_vox + vchunk - 1) / vchunk;
            const size_t smem = ((size_t)((R * p.det_ny + 32 + 3) & ~3) + 2 * (size_t)wcap) * sizeof(float) + 16;
            const int cps = std::max(1, std::min(2, (int)((227 * 1024) / (smem + 1024))));
            // G CTAs per row block, each owning n_chunks / G voxel chunks: G partials
            const int G = std::max(1, std::min(n_chunks, cps * sm_count(g->device) / n_rb));
            S = G;
            e = cudaMallocAsync(&part, (size_t)S * p.n_det * sizeof(double), s);
            if (e == cudaSuccess) {
                KScope kt_(g, s, "k_pc_fwd");
                const int pf = o.pcv_pf;  // L2 prefetch distance (voxels ahead)
                const int n_items = n_chunks * n_rb;
                const int U = o.pcv_u;  // records per thread per step
                // (768 threads x 8 records per thread measured slower: 1.23 vs 1.13 ms)
                const int T = cps == 1 ? 1024 : 512;
                const bool geom = o.pc_fwd_geom && E.pc_qb == 2 && p.n_det <= 65536 && !E.pc_q8;
                const bool padq = E.pc_padq && o.pcv_padq && !geom && E.pc_qb == 2 && T == 1024 && o.pcv_pipe;
                auto kf = padq ? (E.pc_q8 == 2 ? k_pc_fwd_v<uint16_t, 4, 1024, false, true, 2, true>
                                  : E.pc_q8 == 1 ? k_pc_fwd_v<uint16_t, 4, 1024, false, true, 1, true>
                                                 : k_pc_fwd_v<uint16_t, 4, 1024, false, true, 0, true>)
                        : E.pc_q8 == 2 ? (T == 1024 ? k_pc_fwd_v<uint16_t, 4, 1024, false, true, 2>
                                                    : k_pc_fwd_v<uint16_t, 4, 512, false, true, 2>)
                        : E.pc_q8 ? (T == 1024 ? k_pc_fwd_v<uint16_t, 4, 1024, false, true, 1>
                                               : k_pc_fwd_v<uint16_t, 4, 512, false, true, 1>)
                        : E.pc_qb == 2 ? (T == 1024 ? (geom ? k_pc_fwd_v<uint16_t, 4, 1024, true>
                                                            : o.pcv_pipe ? k_pc_fwd_v<uint16_t, 4, 1024, false, true>
                                                                         : k_pc_fwd_v<uint16_t, 4, 1024>)
                                                    : U == 8 ? k_pc_fwd_v<uint16_t, 8, 512>
                                                             : (geom ? k_pc_fwd_v<uint16_t, 4, 512, true> : k_pc_fwd_v<uint16_t, 4, 512>))
                                       : (T == 1024 ? k_pc_fwd_v<uint32_t, 4, 1024> : k_pc_fwd_v<uint32_t, 4, 512>);
                cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                kf<<<G * n_rb, T, smem, s>>>(p, E, W, R, vchunk, n_rb, n_items, pf, part);
            }
        } else {
        // pair cache, per list: items (z chunk, detector row), fp64 partials per z chunk
        int izc = std::max(1, (p.nz * p.det_nx) / (8 * sm_count(g->device) * 4));  // >= ~4 items per resident CTA
        izc = std::min(izc, p.nz);
        S = (p.nz + izc - 1) / izc;
        e = cudaMallocAsync(&part, (size_t)S * p.n_det * sizeof(double), s);
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_pc_fwd");
            const size_t smem = (size_t)PCF_W * p.det_ny * sizeof(float);
            const int n_items = S * p.det_nx;
            auto kf = E.pc_qb == 2 ? k_pc_fwd<uint16_t> : k_pc_fwd<uint32_t>;
            cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kf<<<std::min(n_items, 16 * sm_count(g->device)), PCF_W * 32, smem, s>>>(p, E, W, izc, n_items, part);
        }
        }
    } else if (p.ts_rho > 0) {
        const int segs = (p.det_ny + TS_T - 1) / TS_T;
        const int n_groups = ((p.det_nx + TS_R - 1) / TS_R) * segs;
        const size_t smem = bpb + (size_t)TS_R * (TS_T + p.ts_rho * (p.ny - 1)) * sizeof(float2);
        const int grid = persistent_grid(g, smem, TS_T * TS_R);
        int izc = std::max(1, (p.nz * n_groups) / (4 * grid));  // >= ~4 items per CTA
        izc = std::min(izc, p.nz);
        S = (p.nz + izc - 1) / izc;
        e = cudaMallocAsync(&part, (size_t)S * p.n_det * sizeof(double), s);
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_esai_fwd_ts");
            cudaFuncSetAttribute(k_esai_fwd_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_esai_fwd_ts<<<grid, TS_T * TS_R, smem, s>>>(p, E, (const float2 *)W, izc, n_groups, n_groups * S, part);
        }
    } else {
        const int n_tiles = ((p.det_nx + PF_TX - 1) / PF_TX) * ((p.det_ny + PF_TY - 1) / PF_TY);
        const size_t smem = bpb;
        const int grid = persistent_grid(g, smem, PF_T);
        S = std::max(1, std::min((4 * grid + n_tiles - 1) / n_tiles, (p.n_vox + PF_CH - 1) / PF_CH));
        int vps = (p.n_vox + S - 1) / S;
        vps = (vps + PF_CH - 1) / PF_CH * PF_CH;
        S = (p.n_vox + vps - 1) / vps;
        e = cudaMallocAsync(&part, (size_t)S * p.n_det * sizeof(double), s);
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_esai_fwd");
            auto kf = p.sai_n > 0 ? k_esai_fwd<true> : k_esai_fwd<false>;
            cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kf<<<grid, PF_T, smem, s>>>(p, E, (const float2 *)W, vps, n_tiles, n_tiles * S, part);
        }
    }
    if (e == cudaSuccess) {
        KScope kt_(g, s, "k_sum_parts_f64");
        if (epi && epi->yr_ready) e = cudaStreamWaitEvent(s, epi->yr_ready, 0);
        if (epi)
            sum_parts(part, S, (size_t)p.n_det, EpiRatio{epi->y, epi->r, out, (unsigned *)epi->wmax, E.seen}, s);
        else
            sum_parts(part, S, (size_t)p.n_det, EpiStore{out}, s);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    *launches += 4;  // pack, W GEMM, pair kernel, partial sum (adjusted above for the raw / chunked GEMM)
    if (part) cudaFreeAsync(part, s);
    cudaFreeAsync(fp, s);
    cudaFreeAsync(W, s);
    return e;
}

cudaError_t esai_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches) {
    return esai_backward_masked(g, w, nullptr, b, s, launches, nullptr, 0);
}

// TMA tensor map of a row-major fp32 matrix (rows x cols, row stride ld floats),
// box 128 rows x 32 columns, 128-byte swizzle (the tcgen05 K-major operand layout)
static bool tmap_rows_f32(CUtensorMap *tm, const float *base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            enc = nullptr;
        if (!enc) return false;
    }
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {ld * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)TC_KC, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D map over the split-K partials C[S][rows][cols] (box 32 x 32 x 1, SWIZZLE_128B): a
// store of tile rows past `rows` is clipped inside its own split instead of landing in the
// next split's first rows
static bool tmap_parts_f32(CUtensorMap *tm, const float *base, uint64_t S, uint64_t rows, uint64_t cols) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            enc = nullptr;
        if (!enc) return false;
    }
    const cuuint64_t dims[3] = {cols, rows, S};
    const cuuint64_t strides[2] = {cols * sizeof(float), rows * cols * sizeof(float)};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t esai_backward_masked(const cacsi_geometry *g, const float *w, const uint32_t *pmask, float *b,
                                 cudaStream_t s, int *launches, const int32_t *list, int n_list,
                                 const BwdUpdateEpi *epi) {
    const Params &p = g->p;
    const Esai &E = g->esai;
    float *A = nullptr, *part = nullptr, *wmax = nullptr;
    // split-K of the A S~ contraction: fp32 partials, fp64 sum.  16 splits keep the TMEM
    // accumulation error ~3e-6 (tcgemm.cuh); the fp16 GEMM (default) keeps 16 (option
    // b2_splits): 8 would halve the partials (-0.016 ms) but doubled the measured backward
    // error on configs 1-2
    const Opts &o = g->opt;
    const bool f16 = o.gemm16 && p.nq <= TC_N && !o.b2gemm_tiles;
    const int nkc = f16 ? (E.ldw + TC16_KC - 1) / TC16_KC : E.ldw / TC_KC;
    const int nsp = f16 ? o.b2_splits : 16;
    const int cps = (nkc + nsp - 1) / nsp;
    const int S_eff = (nkc + cps - 1) / cps;
    cudaError_t e = cudaMallocAsync(&A, (size_t)p.n_vox * E.ldw * sizeof(float), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&part, (size_t)S_eff * p.n_vox * p.nq * sizeof(float), s);
    if (e == cudaSuccess && !epi) e = cudaMallocAsync(&wmax, sizeof(float), s);
    // the contraction: the persistent split-K GEMM skips each tile's chunks outside the
    // union of its voxels' windows (A is zero there); the per-tile GEMM reads whole rows
    const int mt = (p.n_vox + TC_M - 1) / TC_M;
    CUtensorMap tm;
    const bool splitk = p.nq <= TC_N && !o.b2gemm_tiles &&
                        tmap_rows_f32(&tm, A, (uint64_t)p.n_vox, (uint64_t)E.ldw, (uint64_t)E.ldw);
    if (e == cudaSuccess) {
        if (epi) {
            wmax = (float *)epi->wmax;  // computed by the fused forward (not freed here)
        } else {
            KScope kt_(g, s, "k_absmax");
            k_absmax<<<1, 1024, 0, s>>>(w, (size_t)p.n_det, pmask, E.seen, wmax);
        }
        if (E.pc && pmask == nullptr) {
            KScope kt_(g, s, "k_pc_bwd");
            const size_t hs = (size_t)E.max_win * sizeof(int);
            if (!o.pc_bwd_flat || E.pc_q8) {  // pc_bwd_flat: the register-fed kernel (A/B reference, 10-byte records)
                // 512 threads x 4 records, two stages (measured best of 128/256/512/1024 threads
                // and 2/3 stages with the vector mapping): ~69 KB with the histogram, 3 CTAs/SM
                constexpr int U = 4, T = 512, NS = 2;
                auto kb = E.pc_q8 == 2 ? (o.pcb_pfl1 ? k_pc_bwd_tma<uint16_t, T, U, NS, 2, true> : k_pc_bwd_tma<uint16_t, T, U, NS, 2>)
                        : E.pc_q8 ? (o.pcb_pfl1 ? k_pc_bwd_tma<uint16_t, T, U, NS, 1, true> : k_pc_bwd_tma<uint16_t, T, U, NS, 1>)
                        : E.pc_qb == 2 ? (o.pcb_pfl1 ? k_pc_bwd_tma<uint16_t, T, U, NS, 0, true> : k_pc_bwd_tma<uint16_t, T, U, NS>)
                                       : k_pc_bwd_tma<uint32_t, T, U, NS>;
                const size_t sm = (size_t)NS * (T * U * (8 + (E.pc_q8 ? 0 : E.pc_qb)) + (E.pc_q8 ? ((T * U / 128 + 14) & ~7) * 2 : 0)) +
                                  2 * NS * sizeof(uint64_t) + hs;
                cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                // (options pcb_ctas / pcb_carve: CTAs per SM and the shared-memory carveout
                // preference -- fewer CTAs leave more of the SM's 256 KB to L1 for the w gathers)
                if (o.pcb_carve > 0) cudaFuncSetAttribute(kb, cudaFuncAttributePreferredSharedMemoryCarveout, o.pcb_carve);
                int nb = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kb, T, sm);
                if (o.pcb_ctas > 0) nb = std::min(nb, o.pcb_ctas);
                kb<<<std::min(p.n_vox, std::max(1, nb) * sm_count(g->device)), T, sm, s>>>(p, E, w, wmax, A);
            } else {
            const int pf = o.pcb_pf;  // rolling L2 prefetch (steps ahead)
            auto kb = E.pc_qb == 2 ? k_pc_bwd<uint16_t> : k_pc_bwd<uint32_t>;
            cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs);
            kb<<<std::min(p.n_vox, 8 * sm_count(g->device)), PCB_T, hs, s>>>(p, E, w, wmax, pf, A);
            }
        } else if (list != nullptr && !o.subset_bwd_mask) {
            // warps per CTA: as many voxel histograms as fit next to the breakpoint tables
            const size_t bpb = host_bp_bytes(E), hb = (size_t)((E.max_win + 3) & ~3) * sizeof(int);
            const int nwarps = (int)std::max((size_t)1, std::min((size_t)8, ((size_t)200 * 1024 - bpb) / hb));
            const size_t smem = bpb + nwarps * hb;
            KScope kt_(g, s, "k_esai_bwd");
            auto kb = p.sai_n > 0 ? k_esai_bwd_list<true> : k_esai_bwd_list<false>;
            cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kb, nwarps * 32, smem);
            kb<<<std::max(1, nb) * sm_count(g->device), nwarps * 32, smem, s>>>(p, E, w, wmax, list, n_list, A);
        } else {
        const size_t smem = bwd_smem_bytes(host_bp_bytes(E), E.max_win);
        {
            KScope kt_(g, s, "k_esai_bwd");
            auto kb = p.sai_n > 0 ? k_esai_bwd<false, true> : k_esai_bwd<false, false>;
            cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kb<<<persistent_grid(g, smem, PB_T), PB_T, smem, s>>>(p, E, w, wmax, E.vbound, pmask, A);
        }
        }
        {
            KScope kt_(g, s, "k_tc_gemm_b2");
            if (splitk && f16) {
                // (option b2_tmast: the partials leave by TMA tensor stores, tmP: box 32 x 32)
                CUtensorMap tmP;
                memset(&tmP, 0, sizeof(tmP));
                const bool tmast = o.b2_tmast && (p.nq % 4) == 0 &&
                                   tmap_parts_f32(&tmP, part, (uint64_t)S_eff, (uint64_t)p.n_vox, (uint64_t)p.nq);
                // A / B ring depths (option b2_rings: 0 = 3 / 3, 1 = 4 / 2, 2 = 2 / 4)
                const int na = o.b2_rings == 1 ? 4 : o.b2_rings == 2 ? 2 : 3, nbr = 6 - na;
                auto ks = tmast ? (na == 4 ? k_tc_gemm_splitk16<true, 4, 2> : na == 2 ? k_tc_gemm_splitk16<true, 2, 4>
                                                                                      : k_tc_gemm_splitk16<true, 3, 3>)
                                : (na == 4 ? k_tc_gemm_splitk16<false, 4, 2> : na == 2 ? k_tc_gemm_splitk16<false, 2, 4>
                                                                                       : k_tc_gemm_splitk16<false, 3, 3>);
                const int sm16 = tcs16_smem(tmast, na, nbr);
                cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, sm16);
                ks<<<std::min(S_eff * mt, sm_count(g->device)), TCS16_T, sm16, s>>>(
                    tm, p.n_vox, p.nq, nkc, cps, S_eff, mt, (const __half *)E.tc16_b, part, p.nq, E.trng, mt, wmax,
                    E.vbmax, E.s16_exp, tmP);
            } else if (splitk) {
                {
                    cudaFuncSetAttribute(k_tc_gemm_splitk, cudaFuncAttributeMaxDynamicSharedMemorySize, tcs_smem());
                    k_tc_gemm_splitk<<<std::min(S_eff * mt, sm_count(g->device)), TCS_T, tcs_smem(), s>>>(
                        tm, p.n_vox, p.nq, nkc, cps, S_eff, mt, E.tc_b, part, p.nq, E.trng, mt);
                }
            } else if (f16) {
                e = cudaErrorInvalidValue;  // (the fp16 GEMM needs the TMA tensor map of A)
            } else {
                dim3 gg((p.nq + TC_N - 1) / TC_N, mt, S_eff);
                cudaFuncSetAttribute(k_tc_gemm<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(1));
                k_tc_gemm<false, 1><<<gg, TC_T, tc_smem(1), s>>>(p.n_vox, p.nq, E.nb, E.ldw, nkc, cps, A, E.tc_b, part,
                                                               p.nq);
            }
        }
        const size_t n = (size_t)p.n_vox * p.nq;
        {
            KScope kt_(g, s, "k_sum_parts_f32");
            if (epi)
                sum_parts(part, S_eff, n, EpiUpdate{p, epi->f_hat, epi->b1, epi->beta, epi->delta, epi->f_new}, s);
            else
                sum_parts(part, S_eff, n, EpiStore{b}, s);
        }
        if (e == cudaSuccess) e = cudaGetLastError();
        *launches += epi ? 3 : 4;
    }
    if (wmax && !epi) cudaFreeAsync(wmax, s);
    if (part) cudaFreeAsync(part, s);
    if (A) cudaFreeAsync(A, s);
    return e;
}


// Subset-restricted operators of Alg. 6.  ESAI handles run
// only the listed pixels' pairs; other handles run the full operator on the
// GPU and restrict its input / output (the plain definitions A_p f = (A f)|_p,
// A_p^T w = A^T (w 1_p)).
__global__ void k_restrict(float *__restrict__ x, int per_pixel, const uint32_t *__restrict__ mask, size_t n_det) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_det * per_pixel;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t q = i / per_pixel;
        if (!((mask[q >> 5] >> (q & 31)) & 1u)) x[i] = 0.0f;
    }
}

static cudaError_t make_mask(const cacsi_geometry *g, const int32_t *pixels, int n, uint32_t **mask, cudaStream_t s) {
    const size_t nw = (size_t)(g->p.n_det + 31) / 32;
    cudaError_t e = cudaMallocAsync((void **)mask, nw * sizeof(uint32_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(*mask, 0, nw * sizeof(uint32_t), s);
    if (e == cudaSuccess && n > 0) {
        KScope kt_(g, s, "k_list_to_mask");
        k_list_to_mask<<<(n + 255) / 256, 256, 0, s>>>(pixels, n, *mask);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_forward_subset(const cacsi_geometry *g, const float *f, const int32_t *pixels, int n, float *out,
                                  cudaStream_t s, int *launches) {
    if (n <= 0) return cudaMemsetAsync(out, 0, g->n_detout * sizeof(float), s);
    if (g->esai.enabled) return esai_forward_list(g, f, pixels, n, out, s, launches);
    uint32_t *mask = nullptr;
    cudaError_t e = make_mask(g, pixels, n, &mask, s);
    if (e == cudaSuccess) e = launch_forward(g, f, out, s, launches);
    if (e == cudaSuccess) {
        KScope kt_(g, s, "k_restrict");
        k_restrict<<<4 * sm_count(g->device), 256, 0, s>>>(out, g->energy_resolving ? g->ne : 1, mask, g->p.n_det);
        e = cudaGetLastError();
        *launches += 2;
    }
    if (mask) cudaFreeAsync(mask, s);
    return e;
}

cudaError_t launch_backward_subset(const cacsi_geometry *g, const float *w, const int32_t *pixels, int n, float *b,
                                   cudaStream_t s, int *launches) {
    if (n <= 0) return cudaMemsetAsync(b, 0, g->n_obj * sizeof(float), s);
    uint32_t *mask = nullptr;
    cudaError_t e = make_mask(g, pixels, n, &mask, s);
    *launches += 1;
    if (e == cudaSuccess && g->esai.enabled) {
        e = esai_backward_masked(g, w, mask, b, s, launches, pixels, n);
    } else if (e == cudaSuccess) {
        float *wr = nullptr;
        e = cudaMallocAsync(&wr, g->n_detout * sizeof(float), s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(wr, w, g->n_detout * sizeof(float), cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_restrict");
            k_restrict<<<4 * sm_count(g->device), 256, 0, s>>>(wr, g->energy_resolving ? g->ne : 1, mask, g->p.n_det);
            e = cudaGetLastError();
            *launches += 1;
        }
        if (e == cudaSuccess) e = launch_backward(g, wr, b, s, launches);
        if (wr) cudaFreeAsync(wr, s);
    }
    if (mask) cudaFreeAsync(mask, s);
    return e;
}

}  // namespace cacsi
