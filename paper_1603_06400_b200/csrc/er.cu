// er.cu -- energy-resolving operators (rows a3/a4 with output g[dx][dy][ne],
// DESIGN.md reading R12): g[r', k] = sum_r P c_k f~_r(u_k),
// b[r, j] = sum_{r', k} P c_k w[r', k] Lambda(u_k - j).
//
// Every (pair, energy) term is an output (forward) or an input (backward), so
// there is no q-contraction to factor out (ESAI does not apply); the kernels
// evaluate the terms directly, organised so that LANES = the in-range
// energies of ONE pair: u_k = alpha_k sigma - beta0 increases with k, so a
// pair's in-range energies are one contiguous window [klo, khi]
// (~43 % of K on config 4) and 32 lanes cover it in one or two rounds with no
// dead slots; accumulators indexed by k are then touched by consecutive lanes
// (conflict-free shared memory, coalesced output).  The pair geometry is
// computed lane-parallel (lane = voxel or pixel) and broadcast with shuffles;
// closed pairs are skipped with the precomputed transmission bitmap.
#include <algorithm>

#include "pair.cuh"

namespace cacsi {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int ER_T = 256, ER_W = ER_T / 32;  // 8 warps
constexpr int ER_PPW = 8;                    // forward: pixels per warp per voxel batch
constexpr int ER_VPW = 8;                    // backward: voxels per warp

// ------------------------------------------------------------------ forward --
// CTA: 64 consecutive pixels (8 warps x 8) x one voxel split [v0, v1) (<= 1024
// voxels, multiple of 32: fp32 accumulation stays short, partials summed in
// fp64 in a fixed order by k_sum_f32).  Per batch of 32 voxels the CTA stages
// their zero-padded hat tables (midpoint value, slope); each warp then, for
// each of its pixels, computes the 32 pair geometries lane-parallel and loops
// over the open ones with lanes = energies.
__global__ void __launch_bounds__(ER_T) k_er_fwd(const Params p, const float *__restrict__ f,
                                                 const uint32_t *__restrict__ tb, int vox_per_split,
                                                 float *__restrict__ partial) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne, Q3 = Q + 3;
    float *alpha = (float *)smem4;                         // [K]
    float2 *tab = (float2 *)(alpha + ((K + 3) & ~3));      // [32][Q + 3], entry n at index n + 2
    float *acc = (float *)(tab + 32 * Q3 + (32 * Q3 & 1));  // [ER_W * ER_PPW][K]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pix0 = blockIdx.x * (ER_W * ER_PPW);
    const int v0 = blockIdx.y * vox_per_split, v1 = min(p.n_vox, v0 + vox_per_split);
    for (int k = tid; k < K; k += ER_T) alpha[k] = p.energy[k].x;
    for (int i = tid; i < ER_W * ER_PPW * K; i += ER_T) acc[i] = 0.0f;
    for (int c0 = v0; c0 < v1; c0 += 32) {
        const int nc = min(32, v1 - c0);
        __syncthreads();
        for (int i = tid; i < nc * Q3; i += ER_T) {
            const int vv = i / Q3, n = i - vv * Q3 - 2;
            const float *fr = f + (size_t)(c0 + vv) * Q;
            const float a = (n >= 0 && n < Q) ? fr[n] : 0.0f;
            const float b = (n + 1 >= 0 && n + 1 < Q) ? fr[n + 1] : 0.0f;
            tab[i] = make_float2(0.5f * (a + b), b - a);
        }
        __syncthreads();
        for (int pp = 0; pp < ER_PPW; pp++) {
            const int pix = pix0 + warp * ER_PPW + pp;
            if (pix >= p.n_det) break;  // warp-uniform
            uint32_t bits = __ldg(tb + (size_t)(c0 / 32) * p.n_det + pix);
            if (nc < 32) bits &= (1u << nc) - 1u;
            // lane-parallel geometry of the pair (voxel c0 + lane, pix)
            const float2 d = p.det[pix];
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if ((bits >> lane) & 1u) {
                pair_geom(p, p.vox[c0 + lane], d, P, sh);
                k_range(p, sh, klo, khi);
            }
            float *accp = acc + (warp * ER_PPW + pp) * K;
            while (bits) {
                const int i = __ffs(bits) - 1;
                bits &= bits - 1;
                const float Pi = __shfl_sync(FULL, P, i), si = __shfl_sync(FULL, sh, i);
                const int lo = __shfl_sync(FULL, klo, i), hi = __shfl_sync(FULL, khi, i);
                const float2 *tv = tab + i * Q3 + 2;
                for (int kb = lo; kb <= hi; kb += 32) {
                    const int k = kb + lane;
                    if (k <= hi) {
                        float tt;
                        const int n = hat_coord(p, alpha[k], si, tt);
                        const float2 t = tv[n];
                        accp[k] = fmaf(Pi, fmaf(tt, t.y, t.x), accp[k]);
                    }
                }
            }
        }
    }
    __syncthreads();
    // coalesced store of this CTA's [pixels][K] block, scaled by c_k
    const int npx = min(ER_W * ER_PPW, p.n_det - pix0);
    float *out = partial + ((size_t)blockIdx.y * p.n_det + pix0) * K;
    for (int i = tid; i < npx * K; i += ER_T) out[i] = p.energy[i % K].y * acc[i];
}

// ----------------------------------------------------------------- backward --
// CTA: 64 consecutive voxels (8 warps x 8) sweeping all pixels in tiles of 32.
// Per tile the CTA stages w (already scaled by c_k) for the 32 pixels and the
// transmission words; each warp, for each of its voxels, computes the 32 pair
// geometries lane-parallel and loops over the open ones with lanes = energies,
// depositing a (1 - t) and a t into the voxel's q-histogram.  Lanes of one pair
// can hit the same node (when the energy step in u is < 1), so the deposits
// are integer shared atomics in two-word fixed point (exact, deterministic;
// scale 2^(30+lb) / (sum_pixels |P| * max|c w|), esai.cu for the scheme).
__global__ void __launch_bounds__(ER_T) k_er_bwd(const Params p, const float *__restrict__ w,
                                                 const uint32_t *__restrict__ tb, const float *__restrict__ ptot,
                                                 const float *__restrict__ wmax, float cmax, int lo_bits,
                                                 float *__restrict__ b) {
    extern __shared__ float4 smem4[];
    const int Q = p.nq, K = p.ne, QB = Q + 4;
    float *alpha = (float *)smem4;                    // [K]
    float *ws = alpha + ((K + 3) & ~3);               // [32][K] staged w * c_k
    uint32_t *tbs = (uint32_t *)(ws + 32 * K);        // [2][32] transmission words of the tile (64 voxels)
    float *sscale = (float *)(tbs + 64);              // [64] fixed-point scale per voxel
    int *hist = (int *)(sscale + 64);                 // [ER_W * ER_VPW][2][Q + 4]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int vb0 = blockIdx.x * (ER_W * ER_VPW);
    for (int k = tid; k < K; k += ER_T) alpha[k] = p.energy[k].x;
    for (int i = tid; i < ER_W * ER_VPW * 2 * QB; i += ER_T) hist[i] = 0;
    const double full = ldexp(1.0, 30 + lo_bits);
    const float inv_lo = ldexpf(1.0f, -lo_bits), lo_unit = ldexpf(1.0f, lo_bits);
    // |a| <= P c_k |w|; a bin gets at most n_det * K deposits: bound = sum_pixels P * cmax * max|w| * K
    const float wm = *wmax * cmax * (float)K;
    if (tid < ER_W * ER_VPW) {
        const int v = vb0 + tid;
        const double bound = v < p.n_vox ? (double)ptot[v] * (double)wm : 0.0;
        sscale[tid] = bound > 0.0 ? (float)(full / bound) : 0.0f;
    }
    for (int q0 = 0; q0 < p.n_det; q0 += 32) {
        const int nq = min(32, p.n_det - q0);
        __syncthreads();
        for (int i = tid; i < nq * K; i += ER_T) ws[i] = w[(size_t)q0 * K + i] * p.energy[i % K].y;
        if (tid < 64) {
            const int cw = vb0 / 32 + tid / 32, qq = q0 + (tid & 31);
            tbs[tid] = ((tid & 31) < nq && cw * 32 < p.n_vox) ? __ldg(tb + (size_t)cw * p.n_det + qq) : 0u;
        }
        __syncthreads();
        const int q = q0 + lane;
        const float2 d = p.det[min(q, p.n_det - 1)];
#pragma unroll 1
        for (int j = 0; j < ER_VPW; j++) {
            const int vl = warp * ER_VPW + j, v = vb0 + vl;
            const float sc = sscale[vl];
            if (v >= p.n_vox || sc == 0.0f) continue;  // warp-uniform
            // transmission words hold 32 voxels; a 64-voxel CTA spans two words
            const uint32_t word = tbs[(vl / 32) * 32 + lane];
            uint32_t bits = __ballot_sync(FULL, lane < nq && ((word >> (v & 31)) & 1u));
            float P = 0.0f, sh = 1.0f;
            int klo = K, khi = -1;
            if ((bits >> lane) & 1u) {
                pair_geom(p, p.vox[v], d, P, sh);
                k_range(p, sh, klo, khi);
            }
            int *hh = hist + vl * 2 * QB + 2;  // bin index = node + 2
            unsigned *hl = (unsigned *)(hh + QB);
            while (bits) {
                const int i = __ffs(bits) - 1;
                bits &= bits - 1;
                const float Pi = __shfl_sync(FULL, P, i) * sc, si = __shfl_sync(FULL, sh, i);
                const int lo = __shfl_sync(FULL, klo, i), hi = __shfl_sync(FULL, khi, i);
                const float *wr = ws + i * K;
                for (int kb = lo; kb <= hi; kb += 32) {
                    const int k = kb + lane;
                    if (k <= hi) {
                        float tt;
                        const int n = hat_coord(p, alpha[k], si, tt);  // n in [-2, nq]
                        const float a = Pi * wr[k];
                        const float x1 = rintf(a * (0.5f + tt));
                        const float x0 = rintf(a) - x1;
                        const float h0 = floorf(x0 * inv_lo), h1 = floorf(x1 * inv_lo);
                        atomicAdd(hh + n, (int)h0);
                        atomicAdd(hl + n, (unsigned)(x0 - h0 * lo_unit));
                        atomicAdd(hh + n + 1, (int)h1);
                        atomicAdd(hl + n + 1, (unsigned)(x1 - h1 * lo_unit));
                    }
                }
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < ER_W * ER_VPW * Q; i += ER_T) {
        const int vl = i / Q, jq = i - vl * Q, v = vb0 + vl;
        if (v >= p.n_vox) continue;
        const int *hh = hist + vl * 2 * QB + 2;
        const long long t = (long long)hh[jq] * (1ll << lo_bits) + (long long)(unsigned)hh[QB + jq];
        const double bound = (double)ptot[v] * (double)wm;
        b[(size_t)v * Q + jq] = bound > 0.0 ? (float)((double)t * (bound / full)) : 0.0f;
    }
}

__global__ void k_er_absmax(const float *__restrict__ w, size_t n, float *out) {
    __shared__ float s[32];
    float m = 0.0f;
    for (size_t i = threadIdx.x; i < n; i += 1024) m = fmaxf(m, fabsf(w[i]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < 32; i++) m = fmaxf(m, s[i]);
        *out = fmaxf(m, s[0]);
    }
}

__global__ void k_er_sum(const float *__restrict__ part, int S, size_t n, float *__restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < S; j++) s += (double)part[j * n + i];
        out[i] = (float)s;
    }
}

int er_sms(int device) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

}  // namespace

cudaError_t er_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches) {
    const Params &p = g->p;
    const int groups = (p.n_det + ER_W * ER_PPW - 1) / (ER_W * ER_PPW);
    int S = std::max(1, (p.n_vox + 1023) / 1024);  // fp32 partial sums over <= 1024 voxels
    int vps = (p.n_vox + S - 1) / S;
    vps = (vps + 31) / 32 * 32;
    S = (p.n_vox + vps - 1) / vps;
    const size_t n_out = (size_t)p.n_det * p.ne;
    const size_t smem = (size_t)((p.ne + 3) & ~3) * 4 + (size_t)(32 * (p.nq + 3) + 1) * 8 +
                        (size_t)ER_W * ER_PPW * p.ne * 4;
    float *part = nullptr;
    cudaError_t e = cudaMallocAsync(&part, (size_t)S * n_out * sizeof(float), s);
    if (e != cudaSuccess) return e;
    {
        KScope kt_(g, s, "k_er_fwd");
        cudaFuncSetAttribute(k_er_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_er_fwd<<<dim3(groups, S), ER_T, smem, s>>>(p, f, g->er.tb, vps, part);
    }
    {
        KScope kt_(g, s, "k_er_sum");
        k_er_sum<<<(int)std::min((n_out + 255) / 256, (size_t)16 * er_sms(g->device)), 256, 0, s>>>(part, S, n_out,
                                                                                                  out);
    }
    e = cudaGetLastError();
    cudaFreeAsync(part, s);
    *launches += 2;
    return e;
}

cudaError_t er_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches) {
    const Params &p = g->p;
    float *wmax = nullptr;
    cudaError_t e = cudaMallocAsync(&wmax, sizeof(float), s);
    if (e != cudaSuccess) return e;
    {
        KScope kt_(g, s, "k_er_absmax");
        k_er_absmax<<<1, 1024, 0, s>>>(w, (size_t)p.n_det * p.ne, wmax);
    }
    const size_t smem = (size_t)((p.ne + 3) & ~3) * 4 + (size_t)32 * p.ne * 4 + 64 * 4 + 64 * 4 +
                        (size_t)ER_W * ER_VPW * 2 * (p.nq + 4) * 4;
    {
        KScope kt_(g, s, "k_er_bwd");
        cudaFuncSetAttribute(k_er_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_er_bwd<<<(p.n_vox + ER_W * ER_VPW - 1) / (ER_W * ER_VPW), ER_T, smem, s>>>(
            p, w, g->er.tb, g->er.ptot, wmax, g->er.cmax, g->er.lo_bits, b);
    }
    e = cudaGetLastError();
    cudaFreeAsync(wmax, s);
    *launches += 2;
    return e;
}

}  // namespace cacsi
