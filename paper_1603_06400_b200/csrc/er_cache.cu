// er_cache.cu -- the energy-resolving operators (detector records g[r', k], BASELINE
// configs[4]) from a pair cache.
//
//   g[r', k] = sum_r P(r, r') c_k f~_r(u_k),   u_k = alpha_k sin(theta/2) - q_min/dq
//   b[r, j]  = sum_{r', k} P(r, r') c_k w[r', k] Lambda(u_k - j)
// (PAPER.md:94-124, 248-270 in the energy-resolved form of PAPER.md:559-575; c_k =
// C_E phi_k E_k, f~ the hat interpolant in q, reading R5).  Every (pair, energy) term
// is an output or an input here -- there is no contraction over q to factor out as in
// the energy-integrating ESAI path -- so the operators are bound by the per-term work.
//
// Pair cache (the paper's online/offline trade-off, taken to HBM):
// the open pairs' P, sin(theta/2) and energy window are computed once at create, per
// detector pixel in increasing voxel order (12 B per open pair; 39 GB on config 4 of
// 180 GB).  Closed pairs and the pair geometry vanish from the operators.
//
// Forward k_er_fwd: one warp per detector pixel (7 pixels in turn), LANES = ENERGIES:
// the two half-warps take two pairs of the pixel at a time, lane i of a half owns the
// energies k = 16 r + i (r = 0 .. nr-1) and keeps their sums in REGISTERS.  A pair
// touches only the rounds r of its energy window (a ~43-energy window of 100 on config
// 4: ~3.6 rounds of 16).  The hat tables of 32 voxels at a time are staged in shared
// memory by cp.async.bulk (3-buffer ring, mbarriers), shared by the CTA's 16 warps;
// per term: one FFMA for u, a clamp, the rounding, one 8-byte table read, two FFMA.
// The fp32 register sums are flushed into fp64 every 4 chunks (128 voxels).
//
// Backward k_er_bwd: items (block of 128 voxels, quarter of the detector); one warp per
// pixel, lanes = energies again (w[r', k] c_k of the pixel in registers); each term
// deposits into the voxel block's shared-memory histogram in FIXED POINT with native
// integer shared atomics, split exactly between the two hat nodes as the ESAI backward
// does.  The per-voxel scale keeps every deposit below 2^21 units (so the
// rounding is an FADD against 1.5 * 2^23, no F2I) and every bin below 2^30; integer sums
// are order-free, so the backward is deterministic.  The quarters' integer partials
// are summed exactly (int64) by k_er_bsum.
#include <algorithm>
#include <vector>

#include "pair.cuh"

namespace cacsi {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int ER_VC = 32;     // voxels per forward table chunk (= one 32-record batch per pixel)
constexpr int ER_NBUF = 3;    // forward table ring depth
constexpr int ER_FW = 16;     // forward warps per CTA
constexpr int ER_PW = 6;      // forward pixels per warp
constexpr int ER_FL = 4;      // forward chunks between fp64 flushes
constexpr int ER_BT = 512;    // backward threads
constexpr int ER_SPLIT = 4;   // backward detector splits (integer partials)

// ---------------------------------------------------------------- build ----
// per voxel, over ALL pixels (a superset of the open pairs): max P and sum P
__global__ void __launch_bounds__(256) k_er_vstats(const Params p, float *pmax, float *psum) {
    __shared__ float smax[8];
    __shared__ double ssum[8];
    const int v = blockIdx.x, tid = threadIdx.x;
    const VoxelRec vr = p.vox[v];
    float m = 0.0f;
    double sum = 0.0;
    for (int q = tid; q < p.n_det; q += 256) {
        float P, sh;
        pair_geom(p, vr, p.det[q], P, sh);
        m = fmaxf(m, P);
        sum += (double)P;
    }
    for (int o = 16; o; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
        sum += __shfl_xor_sync(FULL, sum, o);
    }
    if ((tid & 31) == 0) smax[tid >> 5] = m, ssum[tid >> 5] = sum;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < 8; i++) m = fmaxf(m, smax[i]), s += ssum[i];
        pmax[v] = m * (1.0f + 1e-6f);
        psum[v] = (float)(s * (1.0 + 1e-5));
    }
}

// records per pixel: open pairs whose energy window is not empty (one warp per pixel)
__device__ __forceinline__ bool er_pair(const Params &p, int v, int q, float2 d, float &P, float &sh, int &klo,
                                        int &khi) {
    if (!mask_open(p, v, q, p.vox[v], d)) return false;
    pair_geom(p, p.vox[v], d, P, sh);
    k_range(p, sh, klo, khi);
    return klo <= khi && P > 0.0f;
}

__global__ void __launch_bounds__(256) k_er_count(const Params p, long long *cnt) {
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < p.n_det; q += (gridDim.x * blockDim.x) >> 5) {
        const float2 d = p.det[q];
        int c = 0;
        for (int v0 = 0; v0 < p.n_vox; v0 += 32) {
            const int v = v0 + lane;
            float P = 0.0f, sh = 0.0f;
            int klo = 0, khi = -1;
            const bool o = v < p.n_vox && er_pair(p, v, q, d, P, sh, klo, khi);
            c += __popc(__ballot_sync(FULL, o));
        }
        if (lane == 0) cnt[q] = c;
    }
}

__global__ void __launch_bounds__(256) k_er_fill(const Params p, const long long *__restrict__ off, uint32_t *vw,
                                                 float *Pout, float *sout, uint32_t *boff, int nvb) {
    const int lane = threadIdx.x & 31;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < p.n_det; q += (gridDim.x * blockDim.x) >> 5) {
        const float2 d = p.det[q];
        const long long base = off[q];
        int c = 0;
        for (int v0 = 0; v0 < p.n_vox; v0 += 32) {
            if (v0 % kErVB == 0 && lane == 0) boff[(size_t)(v0 / kErVB) * p.n_det + q] = (uint32_t)c;
            const int v = v0 + lane;
            float P = 0.0f, sh = 0.0f;
            int klo = 0, khi = -1;
            const bool o = v < p.n_vox && er_pair(p, v, q, d, P, sh, klo, khi);
            const unsigned m = __ballot_sync(FULL, o);
            if (o) {
                const long long i = base + c + __popc(m & ((1u << lane) - 1u));
                vw[i] = (uint32_t)v | ((uint32_t)klo << 16) | ((uint32_t)khi << 24);
                Pout[i] = P;
                sout[i] = sh;
            }
            c += __popc(m);
        }
        if (lane == 0) boff[(size_t)nvb * p.n_det + q] = (uint32_t)c;
    }
}

// ------------------------------------------------------------- helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
        "r"(phase)
        : "memory");  // no shared-memory access may move above the wait
}
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

// alpha_k of lane i's energies k = 16 r + i; padding energies (k >= ne) get 1e30
// (their u clamps onto the table's zero top entry / the histogram's pad rows)
template <int NR>
__device__ __forceinline__ void er_alphas(const Params &p, int i, float (&al)[NR]) {
#pragma unroll
    for (int r = 0; r < NR; r++) {
        const int k = 16 * r + i;
        al[r] = k < p.ne ? __ldg(&p.energy[k].x) : 1e30f;
    }
}

// --------------------------------------------------------------- forward ----
// table of voxel v: entry e = n + nlo (n = -nlo .. nq) holds the hat interpolant of
// f[v] on [n + 1/2, n + 3/2) in the (mid, slope) form of k_forward (operators.cu):
// f~(u) = mid_n + tt slope_n, u' = u - 1/2, n = round(u'), tt = u' - n
__global__ void k_er_tab(const Params p, int nlo, int nt, const float *__restrict__ f, float2 *__restrict__ tab) {
    const size_t n = (size_t)p.n_vox * nt;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int v = (int)(i / nt), e = (int)(i % nt), j = e - nlo;
        const float *fr = f + (size_t)v * p.nq;
        const float a = (j >= 0 && j < p.nq) ? fr[j] : 0.0f;
        const float b = (j + 1 >= 0 && j + 1 < p.nq) ? fr[j + 1] : 0.0f;
        tab[i] = make_float2(0.5f * (a + b), b - a);
    }
}

template <int NR>
__global__ void __launch_bounds__(ER_FW * 32, 1) k_er_fwd(const Params p, const ErCache c, const float2 *__restrict__ tab,
                                                          int gsize, int n_groups, float *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int NT = c.nt;
    const int tabw = ER_VC * NT;  // float2 per buffer
    float2 *tabs = (float2 *)sm;
    double *acc64 = (double *)(tabs + ER_NBUF * tabw);                     // [warps][ER_PW][NR * 16]
    uint64_t *full = (uint64_t *)(acc64 + ER_FW * ER_PW * NR * 16);
    uint64_t *empty = full + ER_NBUF;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, li = lane & 15;
    const int nch = (p.n_vox + ER_VC - 1) / ER_VC;
    const int my_groups = blockIdx.x < n_groups ? (n_groups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const long long total = (long long)my_groups * nch;  // chunks this CTA consumes
    if (tid == 0) {
        for (int i = 0; i < ER_NBUF; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(empty + i)), "r"(ER_FW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    double *myacc = acc64 + (size_t)warp * ER_PW * NR * 16;
    for (int i = lane; i < ER_PW * NR * 16; i += 32) myacc[i] = 0.0;
    __syncthreads();
    // producer (thread 0): chunk gc of the CTA's sequence -> buffer gc % ER_NBUF
    auto issue = [&](long long gc) {
        const int ch = (int)(gc % nch);
        const int v0 = ch * ER_VC, nv = min(ER_VC, p.n_vox - v0);
        const uint32_t bytes = (uint32_t)nv * NT * 8u;
        const int b = (int)(gc % ER_NBUF);
        const uint32_t mb = smem_u32(full + b);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(tabs + (size_t)b * tabw)),
                     "l"(tab + (size_t)v0 * NT), "r"(bytes), "r"(mb)
                     : "memory");
    };
    if (tid == 0)
        for (long long gc = 0; gc < min((long long)ER_NBUF, total); gc++) issue(gc);
    float al[NR];
    er_alphas<NR>(p, li, al);
    const float nb = p.nb, qm = p.qm;
    long long gc = 0;
    for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
        // this warp's pixels: q0 + s, s < npx
        const int q0 = g * gsize + warp * ER_PW;
        const int npx = max(0, min(ER_PW, min(p.n_det, (g + 1) * gsize) - q0));
        int cur[ER_PW];
#pragma unroll
        for (int s = 0; s < ER_PW; s++) cur[s] = 0;
        float acc[ER_PW][NR];
#pragma unroll
        for (int s = 0; s < ER_PW; s++)
#pragma unroll
            for (int r = 0; r < NR; r++) acc[s][r] = 0.0f;
        // this chunk's records of pixel slot s: at most ER_VC = 32, so one 32-record batch
        // (records in voxel order: the chunk's are a prefix of the batch)
        auto load = [&](int s, uint32_t &rv, float &rP, float &rs) {
            rv = 0xFFFFFFFFu, rP = 0.0f, rs = 0.0f;
            if (s < npx) {
                const long long b0 = __ldg(c.off + q0 + s), b1 = __ldg(c.off + q0 + s + 1);
                const long long idx = b0 + cur[s] + lane;
                if (idx < b1) rv = __ldg(c.vw + idx), rP = __ldg(c.P + idx), rs = __ldg(c.s + idx);
            }
        };
        for (int ch = 0; ch < nch; ch++, gc++) {
            const int buf = (int)(gc % ER_NBUF);
            const int v0 = ch * ER_VC, v_end = v0 + ER_VC;
            uint32_t rv;
            float rP, rs;
            load(0, rv, rP, rs);  // issued before the table wait: its latency overlaps it
            mbar_wait(smem_u32(full + buf), (uint32_t)((gc / ER_NBUF) & 1));
            const uint32_t tb0 = smem_u32(tabs + (size_t)buf * tabw);
#pragma unroll
            for (int s = 0; s < ER_PW; s++) {
                const unsigned m = __ballot_sync(FULL, rv != 0xFFFFFFFFu && (int)(rv & 0xFFFFu) < v_end);
                const int n = __popc(m);
                cur[s] += n;
                const uint32_t cv = rv;
                const float cP = rP, cs = rs;
                if (s + 1 < ER_PW) load(s + 1, rv, rP, rs);  // next slot's batch in flight
                for (int t = 0; t < n; t += 2) {
                    const int src = t + half;
                    const uint32_t w = __shfl_sync(FULL, cv, src & 31);
                    float P = __shfl_sync(FULL, cP, src & 31);
                    const float sg = __shfl_sync(FULL, cs, src & 31);
                    const bool act = src < n;
                    if (!act) P = 0.0f;
                    int rlo = act ? (int)((w >> 16) & 0xFFu) >> 4 : 1 << 20;
                    int rhi = act ? (int)(w >> 24) >> 4 : -1;
                    rlo = min(rlo, __shfl_xor_sync(FULL, rlo, 16));
                    rhi = max(rhi, __shfl_xor_sync(FULL, rhi, 16));
                    // byte address of table entry n = round(u') of voxel (w & 0xFFFF), folded with
                    // the magic constant's bits: addr = base + 8 * bits(u' + 1.5 * 2^23)
                    const int vl = act ? (int)(w & 0xFFFFu) - v0 : 0;
                    const uint32_t tb = tb0 + (uint32_t)(vl * NT + c.nlo) * 8u - (uint32_t)kMagicBits * 8u;
#pragma unroll
                    for (int r = 0; r < NR; r++)
                        if (r >= rlo && r <= rhi) {
                            const float u = fminf(fmaf(al[r], sg, nb), qm);
                            const float vm = u + kMagic;
                            const float tt = u - (vm - kMagic);
                            const float2 e = lds_f2(tb + (uint32_t)__float_as_int(vm) * 8u);
                            acc[s][r] = fmaf(P, fmaf(tt, e.y, e.x), acc[s][r]);
                        }
                }
            }
            // release the buffer: one arrival per warp after all its reads
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(empty + buf)) : "memory");
            if (tid == 0 && gc + ER_NBUF < total) {
                mbar_wait(smem_u32(empty + buf), (uint32_t)((gc / ER_NBUF) & 1));
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                issue(gc + ER_NBUF);
            }
            // fp64 flush of the fp32 sums (both halves' sums of the same pixel and energy
            // added first), every ER_FL chunks and at the end
            if ((ch + 1) % ER_FL == 0 || ch + 1 == nch) {
#pragma unroll
                for (int s = 0; s < ER_PW; s++)
#pragma unroll
                    for (int r = 0; r < NR; r++) {
                        const float o = __shfl_xor_sync(FULL, acc[s][r], 16);
                        if (half == 0) myacc[(s * NR + r) * 16 + li] += (double)(acc[s][r] + o);
                        acc[s][r] = 0.0f;
                    }
            }
        }
        // g[q][k] = c_k sum (c_k applied once per output)
        __syncwarp();
        for (int s = 0; s < npx; s++) {
            float *o = out + (size_t)(q0 + s) * p.ne;
            for (int k = lane; k < p.ne; k += 32) {
                const int r = k >> 4, i = k & 15;
                o[k] = (float)((double)__ldg(&p.energy[k].y) * myacc[(s * NR + r) * 16 + i]);
            }
        }
        __syncwarp();
        for (int i = lane; i < ER_PW * NR * 16; i += 32) myacc[i] = 0.0;
        __syncwarp();
    }
}

// -------------------------------------------------------------- backward ----
// max |w| over the pixels with at least one record (only their weights deposit)
__global__ void __launch_bounds__(1024) k_er_absmax(const Params p, const long long *__restrict__ off,
                                                    const float *__restrict__ w, float *out) {
    __shared__ float sm[32];
    float m = 0.0f;
    for (int q = threadIdx.x; q < p.n_det; q += 1024)
        if (off[q + 1] > off[q])
            for (int k = 0; k < p.ne; k++) m = fmaxf(m, fabsf(w[(size_t)q * p.ne + k]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 32; i++) m = fmaxf(m, sm[i]);
        *out = m;
    }
}

// ONES: w = 1 everywhere and scale = sv (the create-time bound measurement);
// else scale = sv / max|w|
template <int NR, bool ONES>
__global__ void __launch_bounds__(ER_BT) k_er_bwd(const Params p, const ErCache c, const float *__restrict__ w,
                                                  const float *__restrict__ wmax, const float *__restrict__ sv,
                                                  int *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int HB = p.nq + 4;                        // rows -2 .. nq + 1 (pads)
    int *hist = (int *)sm;                          // [kErVB][HB]
    float *scl = (float *)(hist + kErVB * HB);      // [kErVB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, li = lane & 15;
    const int nwarps = ER_BT / 32;
    const float wm = ONES ? 1.0f : *wmax;
    float al[NR], ck[NR];
    er_alphas<NR>(p, li, al);
#pragma unroll
    for (int r = 0; r < NR; r++) {
        const int k = 16 * r + li;
        ck[r] = k < p.ne ? __ldg(&p.energy[k].y) : 0.0f;
    }
    const float nbb = p.nb + 0.5f;  // -q_min / dq: u = alpha sigma + nbb
    const float qf = (float)p.nq;
    const int n_items = c.nvb * ER_SPLIT;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int vb = it / ER_SPLIT, sp = it % ER_SPLIT;
        const int V0 = vb * kErVB;
        __syncthreads();  // the previous item's histogram has been written out
        for (int i = tid; i < kErVB * HB; i += ER_BT) hist[i] = 0;
        for (int i = tid; i < kErVB; i += ER_BT) {
            const float s = V0 + i < p.n_vox ? sv[V0 + i] : 0.0f;
            scl[i] = (wm > 0.0f) ? s / wm : 0.0f;
        }
        __syncthreads();
        const int qa = (int)((long long)p.n_det * sp / ER_SPLIT), qb = (int)((long long)p.n_det * (sp + 1) / ER_SPLIT);
        for (int q = qa + warp; q < qb; q += nwarps) {
            const long long b0 = __ldg(c.off + q);
            const int a0 = (int)__ldg(c.boff + (size_t)vb * p.n_det + q);
            const int a1 = (int)__ldg(c.boff + (size_t)(vb + 1) * p.n_det + q);
            if (a0 >= a1) continue;
            float wc[NR];
#pragma unroll
            for (int r = 0; r < NR; r++) {
                const int k = 16 * r + li;
                wc[r] = ONES ? ck[r] : (k < p.ne ? ck[r] * __ldg(w + (size_t)q * p.ne + k) : 0.0f);
            }
            for (int a = a0; a < a1; a += 32) {
                const int n = min(32, a1 - a);
                const bool in = lane < n;
                const uint32_t rv = in ? __ldg(c.vw + b0 + a + lane) : 0u;
                const float rP = in ? __ldg(c.P + b0 + a + lane) : 0.0f;
                const float rs = in ? __ldg(c.s + b0 + a + lane) : 0.0f;
                for (int t = 0; t < n; t += 2) {
                    const int src = t + half;
                    const uint32_t wv = __shfl_sync(FULL, rv, src & 31);
                    const float P = __shfl_sync(FULL, rP, src & 31);
                    const float sg = __shfl_sync(FULL, rs, src & 31);
                    const bool act = src < n;
                    const int vl = act ? (int)(wv & 0xFFFFu) - V0 : 0;
                    const float Ps = act ? P * scl[vl] : 0.0f;
                    int rlo = act ? (int)((wv >> 16) & 0xFFu) >> 4 : 1 << 20;
                    int rhi = act ? (int)(wv >> 24) >> 4 : -1;
                    rlo = min(rlo, __shfl_xor_sync(FULL, rlo, 16));
                    rhi = max(rhi, __shfl_xor_sync(FULL, rhi, 16));
                    int *hrow = hist + vl * HB + 2;
#pragma unroll
                    for (int r = 0; r < NR; r++)
                        if (r >= rlo && r <= rhi) {
                            const float u = fminf(fmaxf(fmaf(al[r], sg, nbb), -1.0f), qf);
                            const float vm = (u - 0.5f) + kMagic;  // round(u - 1/2) = floor(u) up to ties
                            const int j0 = __float_as_int(vm) - kMagicBits;
                            const float t1 = u - (vm - kMagic);    // in [0, 1]
                            const float av = wc[r] * Ps;           // |av| <= 2^21 (scale rule)
                            const int xa = __float_as_int(av + kMagic);
                            const int x1 = __float_as_int(fmaf(av, t1, kMagic));
                            atomicAdd(hrow + j0, xa - x1);
                            atomicAdd(hrow + j0 + 1, x1 - kMagicBits);
                        }
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < kErVB * p.nq; i += ER_BT) {
            const int vl = i / p.nq, j = i - vl * p.nq;
            if (V0 + vl < p.n_vox) part[((size_t)sp * p.n_vox + V0 + vl) * p.nq + j] = hist[vl * HB + j + 2];
        }
    }
}

// b[v][j] = (sum of the splits' integers) / scale_v   (exact integer sum: deterministic)
__global__ void k_er_bsum(const Params p, const int *__restrict__ part, const float *__restrict__ sv,
                          const float *__restrict__ wmax, float *__restrict__ b) {
    const float wm = wmax ? *wmax : 1.0f;
    const size_t n = (size_t)p.n_vox * p.nq;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        long long s = 0;
        for (int k = 0; k < ER_SPLIT; k++) s += part[(size_t)k * n + i];
        const float scale = wm > 0.0f ? sv[i / p.nq] / wm : 0.0f;
        b[i] = scale > 0.0f ? (float)((double)s / (double)scale) : 0.0f;
    }
}

// vbound[v] (as the scale factor sv) from the w = 1 measurement: A1 = max_j bin in
// real units, plus the deposits' rounding (<= 1 unit each, <= n_det ne of them)
__global__ void k_er_scale(const Params p, const float *__restrict__ A1, const float *__restrict__ sv0,
                           const float *__restrict__ pmax, float cmax, float *__restrict__ sv) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < p.n_vox; v += gridDim.x * blockDim.x) {
        float m = 0.0f;
        for (int j = 0; j < p.nq; j++) m = fmaxf(m, A1[(size_t)v * p.nq + j]);
        const double unit0 = sv0[v] > 0.0f ? 1.0 / (double)sv0[v] : 0.0;
        const double bound = ((double)m + (double)p.n_det * p.ne * unit0) * (1.0 + 1e-3);
        double s = bound > 0.0 ? 1073741824.0 / bound : 0.0;
        if (pmax[v] > 0.0f) s = fmin(s, 2097152.0 / ((double)pmax[v] * cmax));
        sv[v] = (float)s;
    }
}

int sms(int dev) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

template <int NR>
cudaError_t er_fwd_launch(const cacsi_geometry *g, const float2 *tab, float *out, cudaStream_t s) {
    const Params &p = g->p;
    const ErCache &c = g->er;
    const size_t smem = (size_t)ER_NBUF * ER_VC * c.nt * 8 + (size_t)ER_FW * ER_PW * NR * 16 * 8 + 2 * ER_NBUF * 8;
    const int nsm = sms(g->device);
    int ng = (p.n_det + ER_FW * ER_PW - 1) / (ER_FW * ER_PW);
    ng = (ng + nsm - 1) / nsm * nsm;                      // a whole number of groups per SM
    const int gsize = (p.n_det + ng - 1) / ng;            // <= ER_FW * ER_PW
    ng = (p.n_det + gsize - 1) / gsize;
    cudaFuncSetAttribute(k_er_fwd<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_er_fwd<NR><<<std::min(ng, nsm), ER_FW * 32, smem, s>>>(p, c, tab, gsize, ng, out);
    return cudaGetLastError();
}

template <int NR, bool ONES>
cudaError_t er_bwd_launch(const cacsi_geometry *g, const float *w, const float *wmax, const float *sv, int *part,
                          cudaStream_t s) {
    const Params &p = g->p;
    const size_t smem = (size_t)kErVB * (p.nq + 4) * 4 + kErVB * 4;
    auto kb = k_er_bwd<NR, ONES>;
    cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kb, ER_BT, smem);
    kb<<<std::min(g->er.nvb * ER_SPLIT, std::max(1, nb) * sms(g->device)), ER_BT, smem, s>>>(p, g->er, w, wmax, sv,
                                                                                              part);
    return cudaGetLastError();
}

#define ER_DISPATCH(NRV, CALL)            \
    switch (NRV) {                        \
        case 1: return CALL(1);           \
        case 2: return CALL(2);           \
        case 3: return CALL(3);           \
        case 4: return CALL(4);           \
        case 5: return CALL(5);           \
        case 6: return CALL(6);           \
        case 7: return CALL(7);           \
        default: return CALL(8);          \
    }

cudaError_t er_fwd_any(const cacsi_geometry *g, const float2 *tab, float *out, cudaStream_t s) {
#define C_(N) er_fwd_launch<N>(g, tab, out, s)
    ER_DISPATCH(g->er.nr, C_)
#undef C_
}
template <bool ONES>
cudaError_t er_bwd_any(const cacsi_geometry *g, const float *w, const float *wmax, const float *sv, int *part,
                       cudaStream_t s) {
#define C_(N) er_bwd_launch<N, ONES>(g, w, wmax, sv, part, s)
    ER_DISPATCH(g->er.nr, C_)
#undef C_
}

}  // namespace

// Build the energy-resolving pair cache (create time).  Leaves
// g->er.enabled = 0 (the direct per-term kernels then serve the handle) when the
// geometry is outside the cache's limits or the cache does not fit.
cudaError_t er_build(cacsi_geometry *g, const cacsi_geometry_desc *d) {
    Params &p = g->p;
    ErCache &E = g->er;
    E.enabled = 0;
    E.nr = (p.ne + 15) / 16;
    const double dq = (d->q_max - d->q_min) / (d->nq - 1), beta0 = d->q_min / dq;
    E.nlo = (int)std::ceil(std::max(0.0, beta0)) + 2;
    if (p.n_vox > 65535 || p.ne > 128 || E.nlo > 64) return cudaSuccess;
    E.nt = (E.nlo + p.nq + 1 + 1) & ~1;
    E.nvb = (p.n_vox + kErVB - 1) / kErVB;
    E.cmax = 0.0f;
    for (int k = 0; k < p.ne; k++) E.cmax = std::max(E.cmax, (float)(d->scale * d->phi[k] * d->energy_kev[k]));
    // forward shared memory (3 table buffers + fp64 sums) must fit
    const size_t fsm = (size_t)ER_NBUF * ER_VC * E.nt * 8 + (size_t)ER_FW * ER_PW * E.nr * 16 * 8 + 64;
    const size_t bsm = (size_t)kErVB * (p.nq + 4) * 4 + kErVB * 4;
    if (fsm > 227 * 1024 || bsm > 227 * 1024) return cudaSuccess;
    const int nsm = sms(g->device);
    long long *cnt = nullptr;
    cudaError_t e = cudaMalloc(&cnt, (size_t)p.n_det * sizeof(long long));
    if (e != cudaSuccess) return e;
    k_er_count<<<8 * nsm, 256>>>(p, cnt);
    std::vector<long long> hc(p.n_det), off(p.n_det + 1, 0);
    e = cudaMemcpy(hc.data(), cnt, p.n_det * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(cnt);
    if (e != cudaSuccess) return e;
    for (int q = 0; q < p.n_det; q++) off[q + 1] = off[q] + hc[q];
    const long long nrec = off[p.n_det];
    const size_t need = (size_t)std::max(nrec, 1ll) * 12 + (size_t)(p.n_det + 1) * 8 +
                        (size_t)(E.nvb + 1) * p.n_det * 4;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (need > free_b / 2) return cudaSuccess;  // leave room for the operators' scratch and other handles
    e = cudaMalloc(&g->d_er_off, (p.n_det + 1) * sizeof(long long));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_er_off, off.data(), (p.n_det + 1) * sizeof(long long), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_er_vw, std::max(nrec, 1ll) * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_er_P, std::max(nrec, 1ll) * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_er_s, std::max(nrec, 1ll) * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_er_boff, (size_t)(E.nvb + 1) * p.n_det * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_er_sv, p.n_vox * sizeof(float));
    if (e != cudaSuccess) return e;
    E.n = nrec;
    E.off = (const long long *)g->d_er_off;
    E.vw = (const uint32_t *)g->d_er_vw;
    E.P = (const float *)g->d_er_P;
    E.s = (const float *)g->d_er_s;
    E.boff = (const uint32_t *)g->d_er_boff;
    E.sv = (const float *)g->d_er_sv;
    k_er_fill<<<8 * nsm, 256>>>(p, E.off, (uint32_t *)g->d_er_vw, (float *)g->d_er_P, (float *)g->d_er_s,
                                (uint32_t *)g->d_er_boff, E.nvb);
    e = cudaGetLastError();
    // backward fixed-point scale: the largest bin with w = 1, measured once under the
    // conservative scale min(2^30 / (sum P sum c), 2^21 / (max P max c)) (k_er_scale)
    float *pmax = nullptr, *psum = nullptr, *sv0 = nullptr, *A1 = nullptr;
    int *part = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&pmax, p.n_vox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&psum, p.n_vox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&sv0, p.n_vox * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&A1, (size_t)p.n_vox * p.nq * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&part, (size_t)ER_SPLIT * p.n_vox * p.nq * sizeof(int));
    if (e == cudaSuccess) {
        k_er_vstats<<<p.n_vox, 256>>>(p, pmax, psum);
        std::vector<float> hm(p.n_vox), hs(p.n_vox), h0(p.n_vox);
        e = cudaMemcpy(hm.data(), pmax, p.n_vox * 4, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(hs.data(), psum, p.n_vox * 4, cudaMemcpyDeviceToHost);
        double csum = 0.0;
        for (int k = 0; k < p.ne; k++) csum += d->scale * d->phi[k] * d->energy_kev[k];
        for (int v = 0; v < p.n_vox; v++) {
            double s = hs[v] > 0.0f ? 1073741824.0 / ((double)hs[v] * csum) : 0.0;
            if (hm[v] > 0.0f) s = std::min(s, 2097152.0 / ((double)hm[v] * E.cmax));
            h0[v] = (float)s;
        }
        if (e == cudaSuccess) e = cudaMemcpy(sv0, h0.data(), p.n_vox * 4, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = er_bwd_any<true>(g, nullptr, nullptr, sv0, part, 0);
    if (e == cudaSuccess) {
        k_er_bsum<<<4 * nsm, 256>>>(p, part, sv0, nullptr, A1);
        k_er_scale<<<(p.n_vox + 255) / 256, 256>>>(p, A1, sv0, pmax, E.cmax, (float *)g->d_er_sv);
        e = cudaDeviceSynchronize();
    }
    cudaFree(pmax);
    cudaFree(psum);
    cudaFree(sv0);
    cudaFree(A1);
    cudaFree(part);
    if (e != cudaSuccess) return e;
    E.enabled = 1;
    return cudaSuccess;
}

cudaError_t er_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches) {
    const Params &p = g->p;
    const ErCache &c = g->er;
    float2 *tab = nullptr;
    cudaError_t e = cudaMallocAsync(&tab, (size_t)p.n_vox * c.nt * sizeof(float2), s);
    if (e != cudaSuccess) return e;
    {
        KScope kt_(g, s, "k_er_tab");
        k_er_tab<<<4 * sms(g->device), 256, 0, s>>>(p, c.nlo, c.nt, f, tab);
    }
    {
        KScope kt_(g, s, "k_er_fwd");
        e = er_fwd_any(g, tab, out, s);
    }
    *launches += 2;
    cudaFreeAsync(tab, s);
    return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t er_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches) {
    const Params &p = g->p;
    int *part = nullptr;
    float *wmax = nullptr;
    cudaError_t e = cudaMallocAsync(&part, (size_t)ER_SPLIT * p.n_vox * p.nq * sizeof(int), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&wmax, sizeof(float), s);
    if (e == cudaSuccess) {
        {
            KScope kt_(g, s, "k_er_absmax");
            k_er_absmax<<<1, 1024, 0, s>>>(p, g->er.off, w, wmax);
        }
        {
            KScope kt_(g, s, "k_er_bwd");
            e = er_bwd_any<false>(g, w, wmax, g->er.sv, part, s);
        }
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_er_bsum");
            k_er_bsum<<<4 * sms(g->device), 256, 0, s>>>(p, part, g->er.sv, wmax, b);
            e = cudaGetLastError();
        }
        *launches += 3;
    }
    if (wmax) cudaFreeAsync(wmax, s);
    if (part) cudaFreeAsync(part, s);
    return e;
}

}  // namespace cacsi
