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

// the same records as one 16-byte word each (vw, P, s, 0): one 128-bit load per record
__global__ void __launch_bounds__(256) k_er_fill16(const Params p, const long long *__restrict__ off, uint4 *rec,
                                                   uint32_t *boff, int nvb) {
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
            if (o)
                rec[base + c + __popc(m & ((1u << lane) - 1u))] =
                    make_uint4((uint32_t)v | ((uint32_t)klo << 16) | ((uint32_t)khi << 24), __float_as_uint(P),
                               __float_as_uint(sh), 0u);
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

// One CTA per item (a block of <= 32 PG consecutive pixels), NR x PG warps: warp (pg, r)
// owns pixels 32 pg + lane and the energies k = 16 r + j (j < 16) -- 16 fp32 sums in
// REGISTERS -- and walks the voxels in chunks of ER_VC with the whole CTA:
//   fill:    the chunk's records of every pixel of the item (one 32-record batch per
//            pixel) are scattered into a dense shared tile pt[voxel][pixel] = (P, sigma),
//            closed pairs written as (0, 0);
//   compute: per voxel, skip the round if no lane's energies reach the q grid (exact
//            test, the u' bounds of the round's first / last energy), else 16
//            independent terms per lane -- FFMA, clamp, round, one 8-byte table read
//            (adjacent pixels of one voxel read nearby entries: few bank wavefronts),
//            two FFMA.
// The hat tables of the chunk are landed by cp.async.bulk one chunk ahead (2 buffers;
// the CTA barrier that ends a chunk releases its buffer).  Every ER_FL chunks the fp32
// register sums are added into fp64 sums in shared memory; the item's outputs are
// written coalesced from there (c_k applied once).
template <int NR>
__global__ void __launch_bounds__(896, 1) k_er_fwd(const Params p, const ErCache c, const float2 *__restrict__ tab,
                                                   int isize, int n_items, float *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int NT = c.nt, tabw = ER_VC * NT;
    const int nwarps = blockDim.x >> 5, PG = nwarps / NR, NPX = 32 * PG;
    float2 *tabs = (float2 *)sm;                                   // [2][ER_VC * NT]
    double *acc64 = (double *)(tabs + 2 * tabw);                   // [NPX][NR * 16]
    float2 *pt = (float2 *)(acc64 + (size_t)NPX * NR * 16);        // [ER_VC][NPX]
    int *cur = (int *)(pt + ER_VC * NPX);                          // [NPX]
    uint64_t *full = (uint64_t *)(((uintptr_t)(cur + NPX) + 7) & ~(uintptr_t)7);  // [2]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int pg = warp / NR, r = warp % NR;
    const int nch = (p.n_vox + ER_VC - 1) / ER_VC;
    const int my_items = (int)blockIdx.x < n_items ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const long long total = (long long)my_items * nch;
    if (tid == 0) {
        for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(full + i)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    auto issue = [&](long long gc) {  // chunk gc of this CTA's sequence -> buffer gc & 1
        const int ch = (int)(gc % nch);
        const int v0 = ch * ER_VC, nv = min(ER_VC, p.n_vox - v0);
        const uint32_t bytes = (uint32_t)nv * NT * 8u;
        const uint32_t mb = smem_u32(full + (gc & 1));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(tabs + (size_t)(gc & 1) * tabw)),
                     "l"(tab + (size_t)v0 * NT), "r"(bytes), "r"(mb)
                     : "memory");
    };
    // this warp's energies: alpha of k = 16 r + j (padding energies: 1e30, their u clamps
    // onto the table's zero top entry)
    float al[16];
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const int k = 16 * r + j;
        al[j] = k < p.ne ? __ldg(&p.energy[k].x) : 1e30f;
    }
    const float a_lo = al[0], a_hi = __ldg(&p.energy[min(p.ne - 1, 16 * r + 15)].x);
    const float nb = p.nb, qm = p.qm;
    const int px = pg * 32 + lane;  // this thread's pixel within the item
    double *my64 = acc64 + (size_t)px * NR * 16 + 16 * r;
    __syncthreads();
    if (tid == 0 && total > 0) issue(0);
    long long gc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int P0 = it * isize, npx = min(isize, p.n_det - P0);
        __syncthreads();  // the previous item's output pass (reads every thread's fp64 sums) is done
        for (int i = tid; i < NPX; i += blockDim.x) cur[i] = 0;
#pragma unroll
        for (int j = 0; j < 16; j++) my64[j] = 0.0;
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0.0f;
        for (int ch = 0; ch < nch; ch++, gc++) {
            const int v0 = ch * ER_VC, v_end = v0 + ER_VC;
            __syncthreads();  // the previous chunk's tile reads and this item's cursor resets are done
            if (tid == 0 && gc + 1 < total) issue(gc + 1);  // its buffer's last reader was chunk gc - 1
            // fill: warp w takes pixels w, w + nwarps, ...; lanes = the pixel's next 32 records
            for (int q = warp; q < NPX; q += nwarps) {
                uint32_t vw = 0xFFFFFFFFu;
                float P = 0.0f, sg = 0.0f;
                int n = 0;
                if (q < npx) {
                    const long long b0 = __ldg(c.off + P0 + q), b1 = __ldg(c.off + P0 + q + 1);
                    const long long idx = b0 + cur[q] + lane;
                    if (idx < b1) {
                        vw = __ldg(c.vw + idx);
                        if ((int)(vw & 0xFFFFu) < v_end) P = __ldg(c.P + idx), sg = __ldg(c.s + idx);
                    }
                }
                const bool rec = vw != 0xFFFFFFFFu && (int)(vw & 0xFFFFu) < v_end;
                n = __popc(__ballot_sync(FULL, rec));  // voxel order: the chunk's records are a prefix
                const unsigned have = __reduce_or_sync(FULL, rec ? 1u << ((vw & 0xFFFFu) - v0) : 0u);
                if (rec) pt[((vw & 0xFFFFu) - v0) * NPX + q] = make_float2(P, sg);
                if (!((have >> lane) & 1u)) pt[lane * NPX + q] = make_float2(0.0f, 0.0f);
                if (lane == 0) cur[q] += n;
            }
            __syncthreads();
            mbar_wait(smem_u32(full + (gc & 1)), (uint32_t)((gc >> 1) & 1));
            const uint32_t tb0 = smem_u32(tabs + (size_t)(gc & 1) * tabw) + (uint32_t)c.nlo * 8u -
                                 (uint32_t)kMagicBits * 8u;
            const int nv = min(ER_VC, p.n_vox - v0);
            for (int vl = 0; vl < nv; vl++) {
                const float2 ps = pt[vl * NPX + px];
                // exact skip test: u' of the round's first / last energy against (-3/2, qm)
                const bool act = ps.x > 0.0f && fmaf(a_hi, ps.y, nb) > -1.5f && fmaf(a_lo, ps.y, nb) < qm;
                if (!__any_sync(FULL, act)) continue;
                const uint32_t tb = tb0 + (uint32_t)(vl * NT) * 8u;
                const float P = act ? ps.x : 0.0f;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const float u = fminf(fmaf(al[j], ps.y, nb), qm);
                    const float vm = u + kMagic;
                    const float tt = u - (vm - kMagic);
                    CACSI_CHECK(__float_as_int(vm) - kMagicBits + c.nlo >= 0 && __float_as_int(vm) - kMagicBits + c.nlo < NT);
                    const float2 e = lds_f2(tb + (uint32_t)__float_as_int(vm) * 8u);
                    acc[j] = fmaf(P, fmaf(tt, e.y, e.x), acc[j]);
                }
            }
            if ((ch + 1) % ER_FL == 0 || ch + 1 == nch) {
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    my64[j] += (double)acc[j];
                    acc[j] = 0.0f;
                }
            }
        }
        __syncthreads();
        // g[q][k] = c_k sum, coalesced over the item's [npx][ne] block
        for (int i = tid; i < npx * p.ne; i += blockDim.x) {
            const int q = i / p.ne, k = i - q * p.ne;
            out[(size_t)P0 * p.ne + i] = (float)((double)__ldg(&p.energy[k].y) * acc64[(size_t)q * NR * 16 + k]);
        }
    }
}

// Compacted forward (option er_fwd=1): items (block of F2_R pixels, segment of F2_VS * 128
// voxels); per chunk of 32 voxels the CTA scatters the chunk's records of its pixels into a
// shared (voxel x pixel) tile and appends each record's pixel to its voxel's list (shared
// atomic slot -- the order within a voxel's list does not matter: its pixels are distinct,
// and voxels are taken in order, so every sum is accumulated in voxel order); then every
// warp walks every voxel's list with LANES = the voxel's OPEN pairs (no closed-pair slots)
// and adds its energy blocks (4 energies each, blocks w, w + 8, ...) into the item's shared
// accumulators acc[k][pixel] (warps own disjoint energies: no races).  fp32 partial images
// per segment, summed in fp64 in a fixed order by k_er_fsum.
constexpr int F2_R = 128, F2_RS = F2_R + 1;  // pixels per item; accumulator row stride (bank spread, pad column)
constexpr int F2_VS = 16;                    // voxel blocks of kErVB per segment (2048 voxels)
constexpr int F2_W = 8;                      // warps
template <int NB>
__global__ void __launch_bounds__(F2_W * 32, 1) k_er_fwd2(const Params p, const ErCache c, const float2 *__restrict__ tab,
                                                          int n_pb, int n_items, float *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int NT = c.nt, tabw = ER_VC * NT, KP = 4 * ((p.ne + 3) / 4);
    float2 *tabs = (float2 *)sm;                                 // [2][ER_VC * NT]
    float *acc = (float *)(tabs + 2 * tabw);                     // [KP][F2_RS]
    float2 *pt = (float2 *)(acc + (size_t)KP * F2_RS + (KP * F2_RS & 1));  // [ER_VC][F2_R]
    uint8_t *lst = (uint8_t *)(pt + ER_VC * F2_R);               // [ER_VC][F2_R]
    int *cnt = (int *)(lst + ER_VC * F2_R);                      // [2][ER_VC]
    int *rs = cnt + 2 * ER_VC;                                   // [F2_R] record start (relative to off[q])
    int *rn = rs + F2_R;                                         // [F2_R] record end
    int *cur = rn + F2_R;                                        // [F2_R] cursor
    uint64_t *full = (uint64_t *)(((uintptr_t)(cur + F2_R) + 7) & ~(uintptr_t)7);  // [2]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nbk = KP / 4;
    const int segv = F2_VS * kErVB;
    // this warp's energy blocks b = warp + F2_W i: alpha per energy (padding: 1e30) and the
    // first / last real alpha per block (the exact skip test)
    float al[NB][4], alo[NB], ahi[NB];
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = warp + F2_W * i;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int k = 4 * b + j;
            al[i][j] = (b < nbk && k < p.ne) ? __ldg(&p.energy[k].x) : 1e30f;
        }
        alo[i] = al[i][0];
        ahi[i] = (b < nbk) ? __ldg(&p.energy[min(p.ne - 1, 4 * b + 3)].x) : 1e30f;
    }
    const float nb = p.nb, qm = p.qm;
    if (tid == 0) {
        for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(full + i)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    // chunks of this CTA in sequence (gc): item it, chunk ch
    const int nsegs = (p.n_vox + segv - 1) / segv;
    auto seg_chunks = [&](int it) {
        const int sg = it / n_pb;
        const int V0 = sg * segv, V1 = min(p.n_vox, V0 + segv);
        return (V1 - V0 + ER_VC - 1) / ER_VC;
    };
    // issue chunk ch of item it into buffer (gc & 1)
    auto issue = [&](int it, int ch, long long gc) {
        const int V0 = (it / n_pb) * segv;
        const int v0 = V0 + ch * ER_VC, nv = min(ER_VC, min(p.n_vox, V0 + segv) - v0);
        const uint32_t bytes = (uint32_t)nv * NT * 8u;
        const uint32_t mb = smem_u32(full + (gc & 1));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         smem_u32(tabs + (size_t)(gc & 1) * tabw)),
                     "l"(tab + (size_t)v0 * NT), "r"(bytes), "r"(mb)
                     : "memory");
    };
    (void)nsegs;
    __syncthreads();
    if (tid == 0 && (int)blockIdx.x < n_items) issue(blockIdx.x, 0, 0);
    long long gc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int sg = it / n_pb, pb = it % n_pb;
        const int P0 = pb * F2_R, npx = min(F2_R, p.n_det - P0);
        const int V0 = sg * segv, vb0 = V0 / kErVB, vb1 = min(c.nvb, vb0 + F2_VS);
        const int nch = seg_chunks(it);
        __syncthreads();  // the previous item's output pass is done
        for (int i = tid; i < KP * F2_RS; i += blockDim.x) acc[i] = 0.0f;
        for (int i = tid; i < F2_R; i += blockDim.x) {
            int a = 0, z = 0;
            if (i < npx) {
                a = (int)__ldg(c.boff + (size_t)vb0 * p.n_det + P0 + i);
                z = (int)__ldg(c.boff + (size_t)vb1 * p.n_det + P0 + i);
            }
            rs[i] = a, rn[i] = z, cur[i] = a;
        }
        for (int i = tid; i < 2 * ER_VC; i += blockDim.x) cnt[i] = 0;
        for (int ch = 0; ch < nch; ch++, gc++) {
            const int v0 = V0 + ch * ER_VC, v_end = v0 + ER_VC;
            const int par = ch & 1;
            __syncthreads();  // previous chunk's lists / tile / table buffer reads are done
            if (tid == 0) {
                // next chunk of this CTA's sequence (this item's next, or the next item's first)
                if (ch + 1 < nch) issue(it, ch + 1, gc + 1);
                else if (it + (int)gridDim.x < n_items) issue(it + gridDim.x, 0, gc + 1);
            }
            if (tid < ER_VC) cnt[(par ^ 1) * ER_VC + tid] = 0;  // the next chunk's list counts
            // fill: warp w takes pixels w, w + 8, ...; lanes = the pixel's next 32 records
            for (int px = warp; px < npx; px += F2_W) {
                const long long b0 = __ldg(c.off + P0 + px);
                const int idx = cur[px] + lane;
                uint32_t vw = 0xFFFFFFFFu;
                if (idx < rn[px]) vw = __ldg(c.vw + b0 + idx);
                const bool rec = vw != 0xFFFFFFFFu && (int)(vw & 0xFFFFu) < v_end;
                const int n = __popc(__ballot_sync(FULL, rec));
                if (rec) {
                    const int vl = (int)(vw & 0xFFFFu) - v0;
                    pt[vl * F2_R + px] = make_float2(__ldg(c.P + b0 + idx), __ldg(c.s + b0 + idx));
                    lst[vl * F2_R + atomicAdd(cnt + par * ER_VC + vl, 1)] = (uint8_t)px;
                }
                __syncwarp();
                if (lane == 0) cur[px] += n;
            }
            __syncthreads();
            mbar_wait(smem_u32(full + (gc & 1)), (uint32_t)((gc >> 1) & 1));
            const uint32_t tb0 = smem_u32(tabs + (size_t)(gc & 1) * tabw) + (uint32_t)c.nlo * 8u -
                                 (uint32_t)kMagicBits * 8u;
            const int nv = min(ER_VC, p.n_vox - v0);
            for (int vl = 0; vl < nv; vl++) {
                const int n = cnt[par * ER_VC + vl];
                const uint32_t tb = tb0 + (uint32_t)(vl * NT) * 8u;
                for (int r = 0; r < n; r += 32) {
                    const bool act = r + lane < n;
                    const int px = act ? lst[vl * F2_R + r + lane] : F2_R;  // inactive lanes: the pad column
                    const float2 ps = act ? pt[vl * F2_R + px] : make_float2(0.0f, 0.0f);
                    float *ap = acc + px;
#pragma unroll
                    for (int i = 0; i < NB; i++) {
                        const bool in = act && fmaf(ahi[i], ps.y, nb) > -1.5f && fmaf(alo[i], ps.y, nb) < qm;
                        if (!__any_sync(FULL, in)) continue;
                        const int k0 = 4 * (warp + F2_W * i);
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const float u = fminf(fmaf(al[i][j], ps.y, nb), qm);
                            const float vm = u + kMagic;
                            const float tt = u - (vm - kMagic);
                            const float2 e = lds_f2(tb + (uint32_t)__float_as_int(vm) * 8u);
                            float *a = ap + (k0 + j) * F2_RS;
                            *a = fmaf(ps.x, fmaf(tt, e.y, e.x), *a);
                        }
                    }
                }
            }
        }
        __syncthreads();
        // the segment's fp32 partial image of this pixel block, [q][k] (coalesced)
        float *o = part + ((size_t)sg * p.n_det + P0) * p.ne;
        for (int i = tid; i < npx * p.ne; i += blockDim.x) {
            const int q = i / p.ne, k = i - q * p.ne;
            o[i] = acc[k * F2_RS + q];
        }
    }
}

// g[q][k] = c_k sum_seg part[seg][q][k] (fp64, segments in order)
__global__ void k_er_fsum(const Params p, const float *__restrict__ part, int nseg, float *__restrict__ g) {
    const size_t n = (size_t)p.n_det * p.ne;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nseg; k++) s += (double)part[(size_t)k * n + i];
        g[i] = (float)((double)__ldg(&p.energy[i % p.ne].y) * s);
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

__device__ __forceinline__ void red_s32(uint32_t addr, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Items (block of kErVB voxels, quarter of the detector); one warp per pixel of the
// quarter, lanes = energies: lane i of half h owns k = 16 r + i and holds w[q, k] c_k in
// registers.  The pixel's records in the voxel block go through a per-warp stage, 32 at a
// time; for each round r in the union of the batch's energy windows (one uniform branch
// per batch and round) the two halves sweep the staged pairs two by two (two pairs per
// half per step: independent chains), each term depositing exactly-rounded fixed-point
// integers into the voxel's histogram row with red.shared.add (no return value).
// ONES: w = 1 everywhere and scale = sv (the create-time bound measurement);
// else scale = sv / max|w|
template <int NR, bool ONES>
__global__ void __launch_bounds__(ER_BT) k_er_bwd(const Params p, const ErCache c, const float *__restrict__ w,
                                                  const float *__restrict__ wmax, const float *__restrict__ sv,
                                                  int *__restrict__ part) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int HB = p.nq + 4;                             // rows -2 .. nq + 1 (pads)
    float4 *stage_all = (float4 *)sm;                    // [warps][36]
    int *hist = (int *)(stage_all + (ER_BT / 32) * 36);  // [kErVB][HB]
    float *scl = (float *)(hist + kErVB * HB);           // [kErVB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, li = lane & 15;
    const int nwarps = ER_BT / 32;
    float4 *stage = stage_all + warp * 36;
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
    const uint32_t hbase = smem_u32(hist) + 8u - (uint32_t)kMagicBits * 4u;  // row offset + j0 bits folded in
    if (lane < 4) stage[32 + lane] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);    // pads: Ps = 0
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
                int rlo = 1 << 20, rhi = -1;
                {
                    float4 st = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    if (lane < n) {
                        const uint32_t rv = __ldg(c.vw + b0 + a + lane);
                        const int vl = (int)(rv & 0xFFFFu) - V0;
                        // (row byte offset, sigma, P scale)
                        st = make_float4(__int_as_float(vl * HB * 4), __ldg(c.s + b0 + a + lane),
                                         __ldg(c.P + b0 + a + lane) * scl[vl], 0.0f);
                        rlo = (int)((rv >> 16) & 0xFFu) >> 4;
                        rhi = (int)(rv >> 24) >> 4;
                    }
                    __syncwarp();
                    stage[lane] = st;
                    rlo = __reduce_min_sync(FULL, rlo);
                    rhi = __reduce_max_sync(FULL, rhi);
                    __syncwarp();
                }
#pragma unroll
                for (int r = 0; r < NR; r++) {
                    if (r < rlo || r > rhi) continue;
                    const float a_r = al[r], w_r = wc[r];
                    for (int t = 0; t < n; t += 4) {
                        const float4 d0 = stage[t + half], d1 = stage[t + 2 + half];
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const float4 d = h ? d1 : d0;
                            const float u = fminf(fmaxf(fmaf(a_r, d.y, nbb), -1.0f), qf);
                            const float vm = (u - 0.5f) + kMagic;  // round(u - 1/2) = floor(u) up to ties
                            const float t1 = u - (vm - kMagic);    // in [0, 1]
                            const float av = w_r * d.z;            // |av| <= 2^21 (scale rule)
                            const int xa = __float_as_int(av + kMagic);
                            const int x1 = __float_as_int(fmaf(av, t1, kMagic));
                            CACSI_CHECK(__float_as_int(vm) - kMagicBits >= -2 && __float_as_int(vm) - kMagicBits + 1 <= p.nq + 1 &&
                                        __float_as_int(d.x) >= 0 && __float_as_int(d.x) < kErVB * HB * 4);
                            const uint32_t ad = hbase + (uint32_t)__float_as_int(d.x) + (uint32_t)__float_as_int(vm) * 4u;
                            red_s32(ad, xa - x1);
                            red_s32(ad + 4u, x1 - kMagicBits);
                        }
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

size_t er_fwd2_smem(const Params &p, const ErCache &c) {
    const int KP = 4 * ((p.ne + 3) / 4);
    return (size_t)2 * ER_VC * c.nt * 8 + ((size_t)KP * F2_RS + 1) * 4 + (size_t)ER_VC * F2_R * 8 + ER_VC * F2_R +
           2 * ER_VC * 4 + 3 * F2_R * 4 + 64;
}
template <int NB>
cudaError_t er_fwd2_launch(const cacsi_geometry *g, const float2 *tab, float *part, int n_pb, int n_items,
                           cudaStream_t s) {
    const size_t smem = er_fwd2_smem(g->p, g->er);
    cudaFuncSetAttribute(k_er_fwd2<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device);
    k_er_fwd2<NB><<<std::min(n_items, nsm), F2_W * 32, smem, s>>>(g->p, g->er, tab, n_pb, n_items, part);
    return cudaGetLastError();
}
size_t er_bwd_smem(const Params &p) { return (size_t)(ER_BT / 32) * 36 * 16 + (size_t)kErVB * (p.nq + 4) * 4 + kErVB * 4; }
int er_fwd_pg(int nr) { return std::max(1, std::min(8, 28 / nr)); }
size_t er_fwd_smem(const ErCache &c, int nr) {
    const int npx = 32 * er_fwd_pg(nr);
    return (size_t)2 * ER_VC * c.nt * 8 + (size_t)npx * nr * 16 * 8 + (size_t)ER_VC * npx * 8 + npx * 4 + 64;
}

template <int NR>
cudaError_t er_fwd_launch(const cacsi_geometry *g, const float2 *tab, float *out, cudaStream_t s) {
    const Params &p = g->p;
    const ErCache &c = g->er;
    const int PG = er_fwd_pg(NR), threads = 32 * PG * NR;
    const size_t smem = er_fwd_smem(c, NR);
    const int nsm = sms(g->device);
    // items: a whole number per SM (the persistent CTAs finish together), <= 32 PG pixels each
    int ni = (p.n_det + 32 * PG - 1) / (32 * PG);
    ni = (ni + nsm - 1) / nsm * nsm;
    const int isize = (p.n_det + ni - 1) / ni;
    ni = (p.n_det + isize - 1) / isize;
    cudaFuncSetAttribute(k_er_fwd<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_er_fwd<NR><<<std::min(ni, nsm), threads, smem, s>>>(p, c, tab, isize, ni, out);
    return cudaGetLastError();
}

template <int NR, bool ONES>
cudaError_t er_bwd_launch(const cacsi_geometry *g, const float *w, const float *wmax, const float *sv, int *part,
                          cudaStream_t s) {
    const Params &p = g->p;
    const size_t smem = er_bwd_smem(p);
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
    const size_t fsm = er_fwd_smem(E, E.nr);
    const size_t bsm = er_bwd_smem(p);
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

// The pixel-major records alone (no backward scales), for the default energy-resolving
// forward k_forward_rec (operators.cu, option er_fcache): the records and per-block offsets of
// er_build, each record one 16-byte word (vw, P, s, 0) read by a single 128-bit load; built only
// when they leave `reserve` bytes of device memory free.
// Leaves g->erf.enabled = 0 when skipped.
cudaError_t er_fcache_build(cacsi_geometry *g, size_t reserve) {
    const Params &p = g->p;
    ErCache &E = g->erf;
    E.enabled = 0;
    if (p.n_vox > 65535 || p.ne > 128) return cudaSuccess;
    E.nvb = (p.n_vox + kErVB - 1) / kErVB;
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
    const size_t need = (size_t)(std::max(nrec, 1ll) + 2) * 16 + (size_t)(p.n_det + 1) * 8 +
                        (size_t)(E.nvb + 1) * p.n_det * 4 + 64;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (need + reserve > free_b) return cudaSuccess;
    e = cudaMalloc(&g->d_erf_off, (p.n_det + 1) * sizeof(long long));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_erf_off, off.data(), (p.n_det + 1) * sizeof(long long), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_erf_vw, (std::max(nrec, 1ll) + 2) * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_erf_boff, (size_t)(E.nvb + 1) * p.n_det * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    E.n = nrec;
    E.off = (const long long *)g->d_erf_off;
    E.vw = (const uint32_t *)g->d_erf_vw;  // uint4 records (vw, P, s, 0)
    E.P = nullptr;
    E.s = nullptr;
    E.boff = (const uint32_t *)g->d_erf_boff;
    E.sv = nullptr;
    k_er_fill16<<<8 * nsm, 256>>>(p, E.off, (uint4 *)g->d_erf_vw, (uint32_t *)g->d_erf_boff, E.nvb);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
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
    if (g->opt.er_fwd == 1 && er_fwd2_smem(p, c) <= 227 * 1024) {
        const int segv = F2_VS * kErVB, nseg = (p.n_vox + segv - 1) / segv;
        const int n_pb = (p.n_det + F2_R - 1) / F2_R;
        float *part = nullptr;
        e = cudaMallocAsync(&part, (size_t)nseg * p.n_det * p.ne * sizeof(float), s);
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_er_fwd");
            const int nbk = (p.ne + 3) / 4, NB = (nbk + F2_W - 1) / F2_W;
            e = NB <= 1 ? er_fwd2_launch<1>(g, tab, part, n_pb, n_pb * nseg, s)
                : NB == 2 ? er_fwd2_launch<2>(g, tab, part, n_pb, n_pb * nseg, s)
                : NB == 3 ? er_fwd2_launch<3>(g, tab, part, n_pb, n_pb * nseg, s)
                          : er_fwd2_launch<4>(g, tab, part, n_pb, n_pb * nseg, s);
        }
        if (e == cudaSuccess) {
            KScope kt_(g, s, "k_er_fsum");
            k_er_fsum<<<8 * sms(g->device), 256, 0, s>>>(p, part, nseg, out);
            e = cudaGetLastError();
        }
        if (part) cudaFreeAsync(part, s);
        *launches += 3;
    } else {
        KScope kt_(g, s, "k_er_fwd");
        e = er_fwd_any(g, tab, out, s);
        *launches += 2;
    }
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
