// pair_cache.cuh -- the pair-cache kernels: records built once at
// create (k_pc_count, k_pc_fill, k_pc_perm) and streamed by the operators (the
// voxel-major forward k_pc_fwd_v, its per-list fallback k_pc_fwd, the bulk-copy-ring
// backward k_pc_bwd_tma and its register-fed reference k_pc_bwd).
//
// Not a self-contained header: esai.cu includes it inside namespace cacsi::{anonymous},
// after the breakpoint-location helpers (locate_pair, load_bp, ...) it uses.
#pragma once

// bulk prefetch of [ptr, ptr + bytes) into L2 by the TMA unit (one thread issues
// it; no registers, no completion to wait for): the next voxel's record ranges
// are in L2 by the time the CTA's loads reach them
__device__ __forceinline__ void l2_prefetch(const void *ptr, size_t bytes) {
    uintptr_t a = (uintptr_t)ptr & ~(uintptr_t)15;
    const uintptr_t end = ((uintptr_t)ptr + bytes + 15) & ~(uintptr_t)15;
    while (a < end) {
        const uint32_t n = (uint32_t)min((uintptr_t)65536, end - a);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
        a += n;
    }
}

// ---- pair cache: the online/offline trade-off taken to HBM --
// Every open pair's interpolation weights into the breakpoint basis depend on
// the geometry only, so they can be computed ONCE at create and streamed by
// every later operator call: per list (voxel v, detector row ix), the open
// pixels in increasing jy, each a record of P (fp32), (b, tau) packed in 32 bits
// (b in the high bits, tau in the remaining >= 16 fraction bits: |tau error| <=
// 2^-(tbits+1), i.e. a weight error P |dtau| |W_{b+1} - W_b|, below fp32
// rounding for tbits = 20) and the pixel q (2 bytes for n_det <= 65536, else
// 4): 10 bytes per open pair on config 2 (5.8e8 pairs, 5.8 GB of 180 GB).  A
// voxel's records are contiguous (lists v * det_nx + ix), so both operators
// stream them flat.
// The paper precomputes what is cheaper to load than to recompute ("if the cost
// of computing the factor is equivalent to the speed of loading the factor from
// main memory, then the computations should be performed online"); on a B200,
// streaming 10 bytes is cheaper than the ~100 instructions of pair geometry and
// breakpoint location.  Both operators read the same records: the forward by
// (z, row, y) with the W gathers of one list on one W row, the backward by
// voxel.  Built only if it fits (cacsi_query "pair_cache_records" > 0).

// records per list (v, ix) = open pixels of row ix (transmission bitmap tb_bwd); cnt[n] = 0
// (the exclusive scan over n + 1 entries then ends with the total)
__global__ void k_pc_count(const Params p, const Esai e, long long *__restrict__ cnt, size_t n_lists) {
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[n_lists] = 0;
    const int nw = (p.n_det + 31) / 32;
    const size_t n = (size_t)p.n_vox * p.det_nx;
    for (size_t l = blockIdx.x * (size_t)blockDim.x + threadIdx.x; l < n; l += (size_t)gridDim.x * blockDim.x) {
        const int v = (int)(l / p.det_nx), ix = (int)(l % p.det_nx);
        const uint32_t *tb = e.tb_bwd + (size_t)v * nw;
        const int q0 = ix * p.det_ny, q1 = q0 + p.det_ny;  // [q0, q1)
        int c = 0;
        for (int wd = q0 >> 5; wd <= (q1 - 1) >> 5; wd++) {
            uint32_t m = __ldg(tb + wd);
            const int lo = max(q0 - 32 * wd, 0), hi = min(q1 - 32 * wd, 32);  // bits [lo, hi)
            m &= (hi == 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & (0xFFFFFFFFu << lo);
            c += __popc(m);
        }
        cnt[l] = c;
    }
}

// segment padding: the last list of each (voxel, block of R rows) segment gets the records
// that round the segment up to a multiple of win (R = 0: no padding); tot[0] += open pairs,
// tot[1] += records incl. padding (one warp per segment)
__global__ void k_pc_pad(const Params p, int R, int win, long long *__restrict__ cnt, long long *tot) {
    const int Rs = R > 0 ? R : p.det_nx;
    const int nseg_v = (p.det_nx + Rs - 1) / Rs;
    const size_t nseg = (size_t)p.n_vox * nseg_v;
    const int lane = threadIdx.x & 31;
    const size_t warp0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (size_t)blockDim.x) >> 5;
    for (size_t sg = warp0; sg < nseg; sg += nwarps) {
        const int v = (int)(sg / nseg_v), s = (int)(sg % nseg_v);
        const size_t l0 = (size_t)v * p.det_nx + (size_t)s * Rs;
        const int nlst = min(Rs, p.det_nx - s * Rs);
        long long c = 0;
        for (int i = lane; i < nlst; i += 32) c += cnt[l0 + i];
        c = __reduce_add_sync(0xFFFFFFFFu, (unsigned)c);  // a segment holds < 2^32 records
        if (lane == 0) {
            const long long pad = R > 0 ? ((c + win - 1) / win) * win - c : 0;
            cnt[l0 + nlst - 1] += pad;
            atomicAdd((unsigned long long *)tot, (unsigned long long)c);
            atomicAdd((unsigned long long *)(tot + 1), (unsigned long long)(c + pad));
        }
    }
}

// fill: one warp per list, 32 pixels per step, ballot-compacted records
// Padding pixel (bank-ordered layout): a pixel of the segment's rows that is CLOSED for the
// voxel -- no real record of the segment touches it, so the forward may add the padding's
// zero there without a select (k_pc_fwd_v<..., PADQ>); the last list's row is searched
// first, then the rows above it.  A segment with every pixel open keeps the list's first
// pixel and raises *unsafe (the forward then keeps its dummy-slot select).
template <bool SAI, typename QT>
__global__ void __launch_bounds__(256) k_pc_fill(const Params p, const Esai e, uint32_t *__restrict__ bt,
                                                 float *__restrict__ Pout, QT *__restrict__ qout,
                                                 int *__restrict__ unsafe) {
    const float tone = (float)(1u << e.pc_tbits);
    const uint32_t tmax = (1u << e.pc_tbits) - 1u;
    extern __shared__ __align__(16) unsigned char smem[];
    float *sb = (float *)smem;
    uint16_t *lut = (uint16_t *)(sb + e.nb + kLocD);
    load_bp(e, sb, lut);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (p.n_det + 31) / 32;
    const size_t n = (size_t)p.n_vox * p.det_nx;
    for (size_t l = (size_t)blockIdx.x * 8 + warp; l < n; l += (size_t)gridDim.x * 8) {
        const int v = (int)(l / p.det_nx), ix = (int)(l % p.det_nx);
        const VoxelRec vr = p.vox[v];
        long long base = e.pc_off[l];
        for (int jy0 = 0; jy0 < p.det_ny; jy0 += 32) {
            const int jy = jy0 + lane, q = ix * p.det_ny + jy;
            const bool open = jy < p.det_ny && ((__ldg(e.tb_bwd + (size_t)v * nw + (q >> 5)) >> (q & 31)) & 1u);
            float P = 0.0f, sh = 0.0f, t = 0.0f;
            int b = 0;
            if (open) {
                pair_geom(p, vr, p.det[q], P, sh, !SAI);
                b = locate_pair<SAI>(p, e, sb, lut, sh, v, q, t);
            }
            const uint32_t m = __ballot_sync(FULL, open);
            if (open) {
                const long long o = base + __popc(m & ((1u << lane) - 1u));
                // tau fraction all-ones is reserved for padding records (k_pc_fwd_v<..., GEOM>)
                bt[o] = ((uint32_t)b << e.pc_tbits) | min(__float2uint_rn(t * tone), tmax - 1u);
                Pout[o] = P;
                qout[o] = (QT)q;
            }
            base += __popc(m);
        }
        // segment padding (last list of a segment): P = 0 records, bins spread over
        // the voxel's window (their zero deposits must not pile onto one bank)
        const long long end = e.pc_off[l + 1];
        if (base < end) {
            const int2 win = e.vwin[v];
            const int span = max(1, win.y - win.x);
            int padq = -1;
            const int rs0 = e.pc_R > 0 ? (ix / e.pc_R) * e.pc_R : ix;
            for (int r = ix; r >= rs0 && padq < 0; r--)
                for (int jy0 = 0; jy0 < p.det_ny && padq < 0; jy0 += 32) {
                    const int jy = jy0 + lane, q = r * p.det_ny + jy;
                    const bool closed = jy < p.det_ny && !((__ldg(e.tb_bwd + (size_t)v * nw + (q >> 5)) >> (q & 31)) & 1u);
                    const uint32_t m = __ballot_sync(FULL, closed);
                    if (m) padq = r * p.det_ny + jy0 + __ffs(m) - 1;
                }
            if (padq < 0) {
                padq = ix * p.det_ny;
                if (lane == 0) atomicOr(unsafe, 1);
            }
            for (long long o = base + lane; o < end; o += 32) {
                bt[o] = ((uint32_t)(win.x + (int)((o - base) % span)) << e.pc_tbits) | tmax;
                Pout[o] = 0.0f;
                qout[o] = (QT)padq;
            }
        }
    }
}

// Bank-aware order (build time): within each 128-record window of a padded
// segment, assign the records greedily to the window's 32-record groups (one
// warp access each) so that within a group the breakpoint cells b (histogram /
// W-window bank = b mod 32 up to a per-voxel shift) and the pixels q (forward
// accumulator bank) repeat as little as possible: record i (in list order) goes to
// the non-full group g minimising 2 cb[g][b mod 32] + cq[g][q mod 32] (lowest g on
// ties).  One WARP per window: the window is loaded coalesced, the greedy's state
// (counts per group and colour) lives in the warp's shared memory, lanes 0..3
// score the four groups of each record in parallel and a shuffle reduction picks
// the winner; the permuted window is written back coalesced.  (The greedy is
// sequential in the records; the previous one-thread-per-window kernel kept its
// state in local memory and read the window uncoalesced: ~108 ms per geometry on
// config 2.)
constexpr int PERM_W = 8;  // warps per CTA
// WIN (128, 256 or 512) records per window = WIN / 32 groups: group g = (warp g / 4 of the
// WIN / 128 warps that stream the window, record slot g % 4 of every lane's four); a wider
// window gives the greedy more records to spread over the banks (option pc_win).
// In place: a warp reads its whole window into registers before it writes any record back.
// The same greedy assignment for 128-record windows, one window per LANE: the greedy is
// sequential within a window, so k_pc_perm's warp-per-window form spends each record on a
// warp reduction with 4 of 32 lanes scoring; here 32 windows run side by side, each lane
// scoring its window's four groups from lane-private counters in shared memory ([..][lane]
// bytes: conflict-free).  Every segment is padded to whole windows, so window w is records
// 128 w .. 128 w + 127.  Same scores, same tie rule (lowest group), same positions
// (4 * fill + group): the cache comes out bit-identical to k_pc_perm<QT, 128>.
constexpr int PERM2_W = 4;  // warps per CTA (80 KB of shared memory)
template <typename QT>
__global__ void __launch_bounds__(PERM2_W * 32) k_pc_perm128(long long nwin, int tbits, uint32_t *bt, float *Pr,
                                                             QT *qr) {
    extern __shared__ __align__(16) uint8_t sm8[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    uint8_t *s_b = sm8 + wl * 5 * 4096;   // [128 records][32 windows]
    uint8_t *s_q = s_b + 4096;            // [128][32]
    uint8_t *s_pos = s_q + 4096;          // [128][32]
    uint8_t *s_cb = s_pos + 4096;         // [4 groups][32 colours][32 windows] -- cell colours
    uint8_t *s_cq = s_cb + 4096;          // [4][32][32] -- pixel colours
    for (long long wb = (long long)blockIdx.x * PERM2_W + wl; wb * 32 < nwin; wb += (long long)gridDim.x * PERM2_W) {
        const long long w0 = wb * 32;                      // first window of this warp
        const int nw = (int)min(32LL, nwin - w0);          // windows (lanes) with work
        const size_t r0 = (size_t)w0 * 128;                // first record
        // counters to zero (32-bit stores) and the windows' colours, record-major per lane
        for (int i = lane; i < 2048; i += 32) ((uint32_t *)s_cb)[i] = 0u;  // s_cb and s_cq (8 KB)
        for (int i = lane; i < nw * 128; i += 32) {
            const int ww = i >> 7, r = i & 127;
            s_b[r * 32 + ww] = (uint8_t)((bt[r0 + i] >> tbits) & 31u);
            s_q[r * 32 + ww] = (uint8_t)((uint32_t)qr[r0 + i] & 31u);
        }
        __syncwarp();
        if (lane < nw) {
            int f0 = 0, f1 = 0, f2 = 0, f3 = 0;
            for (int r = 0; r < 128; r++) {
                const int b = s_b[r * 32 + lane], qq = s_q[r * 32 + lane];
                uint8_t *cb = s_cb + b * 32 + lane, *cq = s_cq + qq * 32 + lane;
                const int b0 = cb[0], b1 = cb[1024], b2 = cb[2048], b3 = cb[3072];
                const int q0 = cq[0], q1 = cq[1024], q2 = cq[2048], q3 = cq[3072];
                const int s0 = f0 < 32 ? 2 * b0 + q0 : 1 << 24, s1 = f1 < 32 ? 2 * b1 + q1 : 1 << 24;
                const int s2 = f2 < 32 ? 2 * b2 + q2 : 1 << 24, s3 = f3 < 32 ? 2 * b3 + q3 : 1 << 24;
                // argmin, lowest group on ties
                int g = 0, sc = s0, fb = f0, bb = b0, qb = q0;
                if (s1 < sc) g = 1, sc = s1, fb = f1, bb = b1, qb = q1;
                if (s2 < sc) g = 2, sc = s2, fb = f2, bb = b2, qb = q2;
                if (s3 < sc) g = 3, sc = s3, fb = f3, bb = b3, qb = q3;
                s_pos[r * 32 + lane] = (uint8_t)(4 * fb + g);
                cb[g * 1024] = (uint8_t)(bb + 1);
                cq[g * 1024] = (uint8_t)(qb + 1);
                f0 += g == 0, f1 += g == 1, f2 += g == 2, f3 += g == 3;
            }
        }
        __syncwarp();
        // apply: window by window, each lane moves records 4 lane .. 4 lane + 3 of it
        for (int ww = 0; ww < nw; ww++) {
            const size_t base = r0 + (size_t)ww * 128;
            uint32_t k[4];
            float P[4];
            QT q[4];
            int pos[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int r = 4 * lane + j;
                k[j] = bt[base + r];
                P[j] = Pr[base + r];
                q[j] = qr[base + r];
                pos[j] = s_pos[r * 32 + ww];
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; j++) {
                bt[base + pos[j]] = k[j];
                Pr[base + pos[j]] = P[j];
                qr[base + pos[j]] = q[j];
            }
            __syncwarp();
        }
    }
}

template <typename QT, int WIN>
__global__ void __launch_bounds__(PERM_W * 32) k_pc_perm(const Params p, const Esai e, int R, uint32_t *bt, float *Pr,
                                                         QT *qr) {
    constexpr int G = WIN / 32, PL = WIN / 32;  // groups; records per lane
    __shared__ uint8_t s_cb[PERM_W][G][32], s_cq[PERM_W][G][32];
    __shared__ uint8_t s_b[PERM_W][WIN], s_q[PERM_W][WIN];
    __shared__ uint16_t s_pos[PERM_W][WIN];  // output slot of record i (within the window)
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int nseg_v = (p.det_nx + R - 1) / R;
    const size_t nseg = (size_t)p.n_vox * nseg_v;
    // windows: (segment, WIN-record window of it); segments are whole windows (padded)
    for (size_t sg = blockIdx.x * (size_t)PERM_W + wl; sg < nseg; sg += (size_t)gridDim.x * PERM_W) {
        const int v = (int)(sg / nseg_v), sgi = (int)(sg % nseg_v);
        const size_t l0 = (size_t)v * p.det_nx;
        const long long a = e.pc_off[l0 + sgi * R], z = e.pc_off[l0 + min(p.det_nx, (sgi + 1) * R)];
        for (long long w0 = a; w0 < z; w0 += WIN) {
            const int n = (int)min((long long)WIN, z - w0), cap = n / G;
            uint32_t k[PL];
            float P[PL];
            QT q[PL];
#pragma unroll
            for (int u = 0; u < PL; u++) {
                const int i = lane + 32 * u;
                if (i < n) {
                    k[u] = bt[w0 + i];
                    P[u] = Pr[w0 + i];
                    q[u] = qr[w0 + i];
                    s_b[wl][i] = (uint8_t)((k[u] >> e.pc_tbits) & 31u);
                    s_q[wl][i] = (uint8_t)((uint32_t)q[u] & 31u);
                }
            }
#pragma unroll
            for (int g = 0; g < G; g++) s_cb[wl][g][lane] = 0, s_cq[wl][g][lane] = 0;
            __syncwarp();
            int fill = 0;  // lane g < G: records placed in group g
            for (int i = 0; i < n; i++) {
                const int b = s_b[wl][i], qq = s_q[wl][i];
                int sc = 1 << 24;
                if (lane < G && fill < cap) sc = 2 * s_cb[wl][lane][b] + s_cq[wl][lane][qq];
                // argmin over lanes 0..G-1, lowest lane on ties: key = score * 32 + lane
                const int key = __reduce_min_sync(0xFFFFFFFFu, lane < G ? sc * 32 + lane : 0x7FFFFFFF);
                const int best = key & 31;
                if (lane == best) {
                    s_pos[wl][i] = (uint16_t)(128 * (best >> 2) + 4 * fill + (best & 3));
                    fill++;
                    s_cb[wl][best][b]++;
                    s_cq[wl][best][qq]++;
                }
                __syncwarp();
            }
#pragma unroll
            for (int u = 0; u < PL; u++) {
                const int i = lane + 32 * u;
                if (i < n) {
                    const long long o = w0 + s_pos[wl][i];
                    bt[o] = k[u];
                    Pr[o] = P[u];
                    qr[o] = q[u];
                }
            }
            __syncwarp();
        }
    }
}

// forward from the cache: items (z chunk, detector row); warps take voxel rows
// y, lanes the list's records; per-warp row accumulators in shared memory (the
// jy of one list are distinct: conflict-free, no atomics), fp64 partials per z chunk
constexpr int PCF_W = 8;
template <typename QT>
__global__ void __launch_bounds__(PCF_W * 32) k_pc_fwd(const Params p, const Esai e, const float *__restrict__ W,
                                                     int iz_per_chunk, int n_items, double *__restrict__ partial) {
    extern __shared__ float acc_s[];  // [PCF_W][det_ny]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tb = e.pc_tbits;
    const uint32_t tmask = (1u << tb) - 1u;
    const float tunit = 1.0f / (float)(1u << tb);
    const QT *pq = (const QT *)e.pc_q;
    float *acc = acc_s + warp * p.det_ny;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int chunk = item / p.det_nx, ix = item % p.det_nx;
        for (int i = lane; i < p.det_ny; i += 32) acc[i] = 0.0f;
        __syncwarp();
        const int iz0 = chunk * iz_per_chunk, iz1 = min(p.nz, iz0 + iz_per_chunk);
        for (int iz = iz0; iz < iz1; iz++)
            for (int iy = warp; iy < p.ny; iy += PCF_W) {
                const int v = iy * p.nz + iz;
                const size_t list = (size_t)v * p.det_nx + ix;
                const long long o0 = e.pc_off[list], o1 = e.pc_off[list + 1];
                const float *Wv = W + (size_t)v * e.ldw;
                // four records per lane per step: their loads are issued together
                // (memory-level parallelism); the jy of one list are distinct, so
                // the four accumulator updates never alias
                for (long long o = o0 + lane; o < o1; o += 128) {
                    uint32_t k[4], jy[4];
                    float P[4], wa[4], wb[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const bool in = o + 32 * u < o1;
                        k[u] = in ? __ldg(e.pc_bt + o + 32 * u) : 0u;
                        P[u] = in ? __ldg(e.pc_P + o + 32 * u) : 0.0f;
                        jy[u] = in ? (uint32_t)__ldg(pq + o + 32 * u) - (uint32_t)(ix * p.det_ny) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const float *wp = Wv + (k[u] >> tb);
                        wa[u] = __ldg(wp);
                        wb[u] = __ldg(wp + 1);
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (o + 32 * u < o1) {
                            const float t = (float)(k[u] & tmask) * tunit;
                            CACSI_CHECK(jy[u] < (uint32_t)p.det_ny && (k[u] >> tb) + 1 < (uint32_t)e.ldw);
                            float *ap = acc + jy[u];
                            *ap = fmaf(P[u], fmaf(t, wb[u] - wa[u], wa[u]), *ap);
                        }
                }
            }
        __syncthreads();
        for (int jy = threadIdx.x; jy < p.det_ny; jy += PCF_W * 32) {
            double t = 0.0;
            for (int ww = 0; ww < PCF_W; ww++) t += (double)acc_s[ww * p.det_ny + jy];
            partial[(size_t)chunk * p.n_det + (size_t)ix * p.det_ny + jy] = t;
        }
        __syncthreads();
    }
}

// forward from the cache, voxel-major: items (voxel chunk, block of R detector
// rows), chunks of consecutive voxels; per voxel the CTA holds the voxel's W
// window in shared memory (one cp.async.bulk per voxel, issued a voxel ahead
// into the other of two buffers, completion on an mbarrier) and streams the
// voxel's records of those rows -- one contiguous range -- 4 per thread per
// step; the W reads are shared-memory gathers and each record adds into the
// CTA's row-block accumulator acc[q - q0].  The pixels of one voxel's records
// are distinct (no two updates of one voxel alias); voxels are separated by a
// barrier, so the sums are plain fp32 in a fixed order (deterministic).
// Per (voxel, row block) segment of the bank-ordered cache: the W columns its real
// records read, [min b, max b + 1] (one warp per segment), then the segment's
// padding records (P = 0) re-binned inside that window (spread over it, as k_pc_fill
// spreads them over the voxel's) -- so the voxel-major forward stages only the
// segment's part of the voxel's W window (with two row blocks, each reads roughly
// half of it instead of all of it).  Empty segments get [win.x, win.x + 1].
__global__ void k_pc_segwin(const Params p, const Esai e, int R, uint32_t *__restrict__ bt,
                            const float *__restrict__ P, int2 *__restrict__ segwin) {
    const int nseg_v = (p.det_nx + R - 1) / R;
    const size_t nseg = (size_t)p.n_vox * nseg_v;
    const int lane = threadIdx.x & 31;
    const size_t warp0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * (size_t)blockDim.x) >> 5;
    for (size_t sg = warp0; sg < nseg; sg += nwarps) {
        const int v = (int)(sg / nseg_v), s = (int)(sg % nseg_v);
        const size_t l0 = (size_t)v * p.det_nx;
        const long long a = e.pc_off[l0 + s * R], z = e.pc_off[l0 + min(p.det_nx, (s + 1) * R)];
        int lo = 1 << 30, hi = -1;
        for (long long o = a + lane; o < z; o += 32)
            if (P[o] != 0.0f) {
                const int b = (int)(bt[o] >> e.pc_tbits);
                lo = min(lo, b);
                hi = max(hi, b + 1);
            }
        lo = __reduce_min_sync(0xFFFFFFFFu, lo);
        hi = __reduce_max_sync(0xFFFFFFFFu, hi);
        if (hi < 0) lo = e.vwin[v].x, hi = lo + 1;
        if (lane == 0) segwin[sg] = make_int2(lo, hi);
        const int span = hi - lo;  // padding bins b in [lo, hi - 1]: b + 1 <= hi stays inside
        const uint32_t tmax = (1u << e.pc_tbits) - 1u;  // padding marker (k_pc_fill)
        for (long long o = a + lane; o < z; o += 32)
            if (P[o] == 0.0f) bt[o] = ((uint32_t)(lo + (int)((o - a) % span)) << e.pc_tbits) | tmax;
    }
}

// 8-byte records (build time, after the permutation and the segment windows): one warp per
// 128-record window.  Pass 1 measures the largest pixel span of a window; if it fits 9 bits,
// pass 2 rewrites every record word in place as (b << tbits) | (tau8 << 9) | (q - qbase)
// with tau rounded to tau8 = tbits - 9 bits, and stores the window's base pixel.
__global__ void k_pc_qspan(long long nwin, const uint16_t *__restrict__ q, unsigned *maxspan) {
    const int lane = threadIdx.x & 31;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nwin;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const uint2 v = *(const uint2 *)(q + w * 128 + 4 * lane);
        const unsigned a = v.x & 0xFFFFu, b = v.x >> 16, c = v.y & 0xFFFFu, d = v.y >> 16;
        const unsigned lo = __reduce_min_sync(0xFFFFFFFFu, min(min(a, b), min(c, d)));
        const unsigned hi = __reduce_max_sync(0xFFFFFFFFu, max(max(a, b), max(c, d)));
        if (lane == 0) atomicMax(maxspan, hi - lo);
    }
}
// MODE 1: (b | tau in tb8 = tbits - 9 bits at bit 9 | 9-bit pixel offset), P unchanged.
// MODE 2 ("P-packed"): P rounded to 28 bits (19 explicit mantissa bits, relative error
// <= 2^-20) carries the offset's low 4 bits in its low nibble; the b word keeps tau with
// tb8 = tbits - 5 bits at bit 5 and the offset's high 5 bits in bits 0-4 (reading R23).
__global__ void k_pc_pack8(long long nwin, int tbits, int tb8, int mode, const uint16_t *__restrict__ q, uint32_t *bt,
                           float *Pr, uint16_t *__restrict__ qbase) {
    const int lane = threadIdx.x & 31, sh = tbits - tb8;
    const uint32_t tmax8 = (1u << tb8) - 1u, tmask = (1u << tbits) - 1u;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nwin;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const uint2 v = *(const uint2 *)(q + w * 128 + 4 * lane);
        const unsigned qq[4] = {v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16};
        const unsigned lo = __reduce_min_sync(0xFFFFFFFFu, min(min(qq[0], qq[1]), min(qq[2], qq[3])));
        uint4 k = *(const uint4 *)(bt + w * 128 + 4 * lane);
        uint32_t kk[4] = {k.x, k.y, k.z, k.w};
        if (mode == 2) {
            float4 pv = *(const float4 *)(Pr + w * 128 + 4 * lane);
            float pp[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t off = qq[u] - lo;
                const uint32_t t8 = min(((kk[u] & tmask) + (1u << (sh - 1))) >> sh, tmax8);
                kk[u] = (kk[u] & ~tmask) | (t8 << 5) | (off >> 4);
                const uint32_t pb = (__float_as_uint(pp[u]) + 0x8u) & 0xFFFFFFF0u;  // P >= 0: round to 28 bits
                pp[u] = __uint_as_float(pb | (off & 0xFu));
            }
            *(float4 *)(Pr + w * 128 + 4 * lane) = make_float4(pp[0], pp[1], pp[2], pp[3]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t t8 = min(((kk[u] & tmask) + (1u << (sh - 1))) >> sh, tmax8);
                kk[u] = (kk[u] & ~tmask) | (t8 << 9) | (qq[u] - lo);
            }
        }
        *(uint4 *)(bt + w * 128 + 4 * lane) = make_uint4(kk[0], kk[1], kk[2], kk[3]);
        if (lane == 0) qbase[w] = (uint16_t)lo;
    }
}
// 8-byte record decode: the pixel offset from the window base and P (MODE from Esai.pc_q8)
__device__ __forceinline__ uint32_t q8_off(int mode, uint32_t k, float P) {
    return mode == 2 ? ((__float_as_uint(P) & 0xFu) | ((k & 0x1Fu) << 4)) : (k & 511u);
}
__device__ __forceinline__ float q8_P(int mode, float P) {
    return mode == 2 ? __uint_as_float(__float_as_uint(P) & 0xFFFFFFF0u) : P;
}

// the W columns a (voxel, row block) segment reads: its own window when the cache
// recorded one (k_pc_segwin), else the voxel's
__device__ __forceinline__ int2 seg_window(const Esai &e, int v, int n_rb, int rb) {
    return e.pc_segwin ? e.pc_segwin[(size_t)v * n_rb + rb] : e.vwin[v];
}
__device__ __forceinline__ void pcv_stage(const Esai &e, const float *W, int v, int2 win, float *dst, uint64_t *mbar) {
    const int a = win.x & ~3;
    const uint32_t bytes = (uint32_t)(((win.y + 1 - a) + 3) & ~3) * 4u;
    const uint32_t mb = smem_u32(mbar);
    // the threads' earlier reads of dst (generic proxy, ordered before this thread by
    // the CTA barrier) before the bulk copy (async proxy) that overwrites it
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(W + (size_t)v * e.ldw + a), "r"(bytes), "r"(mb)
                 : "memory");
}
// GEOM: the records' P is not read -- the pair's geometric factor is recomputed from the
// pixel index and the voxel (translation-symmetric s_y = c0 + p (jy - rho iy) when
// ts_rho > 0), 6 instead of 10 bytes per record (padding records carry the all-ones tau
// marker and contribute 0).  An A/B variant (option pc_fwd_geom): DESIGN.md 4.2b.
// PIPE: the vector record loop is software-pipelined -- each thread's next 4 records are
// loaded before the current 4 are deposited (two steps of loads in flight per thread).
// Q8: 8-byte records (pixel = window base + 9-bit offset, tau with pc_tb8 bits at bit
// pc_tsh8; MODE 2 keeps 8 offset bits in P's low byte -- k_pc_pack8)
// PADQ: every padding record's pixel is closed for its voxel (k_pc_fill, Esai.pc_padq):
// its zero is added in place, without the select into the dummy slot.
template <typename QT, int U, int PCV_T, bool GEOM = false, bool PIPE = false, int Q8 = 0, bool PADQ = false>
__global__ void __launch_bounds__(PCV_T, 1024 / PCV_T) k_pc_fwd_v(const Params p, const Esai e, const float *__restrict__ W,
                                                     int R, int vchunk, int n_rb, int n_items, int pf,
                                                     double *__restrict__ partial) {
    extern __shared__ __align__(16) float smv[];
    const int wcap = (e.max_win + 3 + 3) & ~3;
    float *acc = smv;                                   // [R * det_ny] + 32 dummy slots
    float *dummy = acc + R * p.det_ny + (threadIdx.x & 31);
    float *ws = smv + ((R * p.det_ny + 32 + 3) & ~3);   // [2][wcap]
    uint64_t *mbar = (uint64_t *)(ws + 2 * wcap);       // [2]
    const int tid = threadIdx.x;
    const int tb = e.pc_tbits;
    const uint32_t tmask = (1u << tb) - 1u;
    const float tunit = 1.0f / (float)(1u << tb);
    const uint32_t tmask8 = (1u << e.pc_tb8) - 1u;
    const float tunit8 = 1.0f / (float)(1u << e.pc_tb8);
    const QT *pq = (const QT *)e.pc_q;
    const bool vec = e.pc_R > 0;  // bank-ordered layout: segments 128-record aligned (vector loads)
    if (tid == 0) {
        for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(mbar + i)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    __syncthreads();
    uint32_t uses = 0;  // bit i: parity of buffer i's next completion
    // gridDim.x = G n_rb: the CTA keeps ONE row block (blockIdx.x % n_rb) for all its
    // voxel chunks, accumulates them in shared memory and writes one fp64 partial
    // (index blockIdx.x / n_rb) at the end -- G partials, not one per chunk
    const int rb = blockIdx.x % n_rb;
    const int r0 = rb * R, r1 = min(p.det_nx, r0 + R);
    const int q0 = r0 * p.det_ny, nacc = (r1 - r0) * p.det_ny;
    for (int i = tid; i < nacc; i += PCV_T) acc[i] = 0.0f;
    // every thread's zeroing before any thread's first deposit (the mbarrier wait below
    // orders only the bulk copy, not the other warps' stores)
    __syncthreads();
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int c = item / n_rb;
        const int v0 = c * vchunk, v1 = min(p.n_vox, v0 + vchunk);
        if (tid == 0) pcv_stage(e, W, v0, seg_window(e, v0, n_rb, rb), ws, mbar);
        for (int v = v0; v < v1; v++) {
            const int buf = (v - v0) & 1;
            if (tid == 0 && v + 1 < v1)
                pcv_stage(e, W, v + 1, seg_window(e, v + 1, n_rb, rb), ws + (buf ^ 1) * wcap, mbar + (buf ^ 1));
            const size_t l0 = (size_t)v * p.det_nx;
            const long long o0 = __ldg(e.pc_off + l0 + r0), o1 = __ldg(e.pc_off + l0 + r1);
            if (tid == 0 && pf > 0 && v + pf < v1) {
                const size_t l2 = (size_t)(v + pf) * p.det_nx;
                const long long a0 = __ldg(e.pc_off + l2 + r0), a1 = __ldg(e.pc_off + l2 + r1);
                l2_prefetch(e.pc_bt + a0, (size_t)(a1 - a0) * sizeof(uint32_t));
                l2_prefetch(e.pc_P + a0, (size_t)(a1 - a0) * sizeof(float));
                if (!Q8) l2_prefetch(pq + a0, (size_t)(a1 - a0) * sizeof(QT));  // (Q8: no pixel array)
            }
            mbar_wait(smem_u32(mbar + buf), (uses >> buf) & 1u);
            uses ^= 1u << buf;
            const int2 swin = seg_window(e, v, n_rb, rb);
            const float *wv = ws + buf * wcap - (swin.x & ~3);
            float *accq = acc - q0;
            // 32-bit indices from the voxel's first record; full steps unchecked, then the tail
            const uint32_t *kb = e.pc_bt + o0;
            const float *Pb = e.pc_P + o0;
            const QT *qb = pq + o0;
            const int n = (int)(o1 - o0);
            // each thread takes U CONSECUTIVE records (16-byte vector loads, U / 4 quads); the
            // bank-aware order puts record j of every lane's quad in one conflict-light group,
            // so the warp's j-th shared-memory access touches distinct banks
            const uint32_t kpad = ((uint32_t)swin.x << tb) | tmask;  // padding marker
            // P = 0: segment padding, whose pixel may repeat a real record's -- it
            // adds into the lane's dummy slot past the row block (branch-free)
            const VoxelRec vr = GEOM ? p.vox[v] : VoxelRec{};
            const int iyr = GEOM ? p.ts_rho * (v / p.nz) : 0;
            auto geom_P = [&](uint32_t k, uint32_t q) {
                const uint32_t ix = __umulhi(q, p.det_div), jy = q - ix * (uint32_t)p.det_ny;
                const float sx = fmaf(exact_float((int)ix), p.pitch_d, p.det_x0);
                const float sy = p.ts_rho > 0 ? fmaf(p.pitch_d, exact_float((int)jy - iyr), p.ts_c0)
                                              : fmaf(exact_float((int)jy), p.pitch_d, p.det_y0) - vr.y;
                const float sz = vr.sz;
                const float syz2 = fmaf(sy, sy, sz * sz);
                const float rs = rsqrtf(fmaf(sx, sx, syz2));
                const float rs2 = rs * rs;
                const float cos_t = fmaf(vr.ry, sy, vr.rz * sz) * rs;
                const float h = fmaf(0.5f, cos_t, 0.5f);
                const float x = p.pitch_d * fast_sqrt(syz2) * rs2 * fmaf(p.quarter_p2, rs2, 1.0f);
                const float dth = x * fmaf(-0.33333334f * x, x, 1.0f);
                const float P = vr.gso * (sz * rs * rs2) * dth * fmaf(cos_t, cos_t, 1.0f) * (h * rsqrtf(h));
                return (k & tmask) == tmask ? 0.0f : P;
            };
            auto deposit = [&](const uint32_t (&k)[U], const float (&P0)[U], const uint32_t (&q)[U]) {
                float P[U];
#pragma unroll
                for (int u = 0; u < U; u++) P[u] = GEOM ? geom_P(k[u], q[u]) : P0[u];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int b = (int)(k[u] >> tb);
                    CACSI_CHECK(b >= (swin.x & ~3) && b + 1 < (swin.x & ~3) + wcap);
                    CACSI_CHECK((P[u] == 0.0f && !PADQ) || (q[u] >= (uint32_t)q0 && q[u] < (uint32_t)(q0 + nacc)));
                    const float wa = wv[b], wb = wv[b + 1];
                    const float t = Q8 ? (float)((k[u] >> (Q8 == 2 ? 5 : 9)) & tmask8) * tunit8 : (float)(k[u] & tmask) * tunit;
                    float *ap = PADQ ? accq + q[u] : P[u] != 0.0f ? accq + q[u] : dummy;
                    *ap = fmaf(P[u], fmaf(t, wb - wa, wa), *ap);
                }
            };
            if (vec && PIPE && U == 4 && sizeof(QT) == 2) {
                // two register sets (A, B) in ping-pong: the next step's loads land in the
                // set not being deposited, with no register copies between steps
                struct Rec4 {
                    uint4 k;
                    float4 P;
                    uint2 q;
                };
                auto ld = [&](Rec4 &r, int j) {
                    r.k = __ldg((const uint4 *)(kb + j));
                    if (!GEOM) r.P = __ldg((const float4 *)(Pb + j));
                    if (Q8)  // the warp's 128 records are one window: one base per warp step
                        r.q.x = __ldg(e.pc_qbase + ((o0 + j) >> 7));
                    else
                        r.q = __ldg((const uint2 *)(qb + j));
                };
                auto dep = [&](const Rec4 &r) {
                    uint32_t k[U], q[U];
                    float P[U];
                    k[0] = r.k.x, k[1] = r.k.y, k[2] = r.k.z, k[3] = r.k.w;
                    P[0] = r.P.x, P[1] = r.P.y, P[2] = r.P.z, P[3] = r.P.w;
                    if (Q8) {
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            q[u] = r.q.x + q8_off(Q8, k[u], P[u]);
                            P[u] = q8_P(Q8, P[u]);
                        }
                    } else {
                        q[0] = r.q.x & 0xFFFFu, q[1] = r.q.x >> 16, q[2] = r.q.y & 0xFFFFu, q[3] = r.q.y >> 16;
                    }
                    deposit(k, P, q);
                };
                constexpr int ST = 4 * PCV_T;
                Rec4 ra, rb;
                ra.P = rb.P = make_float4(0.f, 0.f, 0.f, 0.f);
                ra.q = rb.q = make_uint2(0u, 0u);
                int i = 4 * tid;
                if (i < n) ld(ra, i);
                for (; i < n; i += 2 * ST) {
                    if (i + ST < n) ld(rb, i + ST);
                    dep(ra);
                    if (i + ST >= n) break;
                    if (i + 2 * ST < n) ld(ra, i + 2 * ST);
                    dep(rb);
                }
            } else if (vec) {
                // bank-ordered layout: the voxel's range is whole 128-record windows (n % 128 == 0),
                // so every thread's U records are in range -- no bounds test in the loop
                for (int i = U * tid; i < n; i += U * PCV_T) {
                    uint32_t k[U], q[U];
                    float P[U];
#pragma unroll
                    for (int h = 0; h < U; h += 4) {
                        const uint4 kv = __ldg((const uint4 *)(kb + i + h));
                        const float4 pv = GEOM ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg((const float4 *)(Pb + i + h));
                        k[h] = kv.x, k[h + 1] = kv.y, k[h + 2] = kv.z, k[h + 3] = kv.w;
                        P[h] = pv.x, P[h + 1] = pv.y, P[h + 2] = pv.z, P[h + 3] = pv.w;
                        if (sizeof(QT) == 2) {
                            const uint2 qv = __ldg((const uint2 *)(qb + i + h));
                            q[h] = qv.x & 0xFFFFu, q[h + 1] = qv.x >> 16, q[h + 2] = qv.y & 0xFFFFu, q[h + 3] = qv.y >> 16;
                        } else {
                            const uint4 qv = __ldg((const uint4 *)(qb + i + h));
                            q[h] = qv.x, q[h + 1] = qv.y, q[h + 2] = qv.z, q[h + 3] = qv.w;
                        }
                    }
                    deposit(k, P, q);
                }
            } else {
                for (int i = U * tid; i < n; i += U * PCV_T) {
                    uint32_t k[U], q[U];
                    float P[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const bool in = i + u < n;
                        k[u] = in ? __ldg(kb + i + u) : kpad;
                        P[u] = in ? __ldg(Pb + i + u) : 0.0f;
                        q[u] = in ? (uint32_t)__ldg(qb + i + u) : 0u;
                    }
                    deposit(k, P, q);
                }
            }
            // the barrier orders every thread's reads of this W buffer before thread 0's
            // next bulk copy into it (pcv_stage fences the proxies first)
            __syncthreads();
        }
    }
    for (int i = tid; i < nacc; i += PCV_T) partial[(size_t)(blockIdx.x / n_rb) * p.n_det + q0 + i] = (double)acc[i];
}

// backward from the cache: one CTA per voxel (grid-stride), warps take detector
// rows, lanes the records; fixed-point deposits as k_esai_bwd (same scale rule)
constexpr int PCB_T = 256;
template <typename QT>
__global__ void __launch_bounds__(PCB_T) k_pc_bwd(const Params p, const Esai e, const float *__restrict__ w,
                                                  const float *__restrict__ wmax, int pf, float *__restrict__ A) {
    extern __shared__ int hist_s[];  // [max_win]
    const int tid = threadIdx.x;
    const int tb = e.pc_tbits;
    const uint32_t tmask = (1u << tb) - 1u;
    const float tunit = 1.0f / (float)(1u << tb);
    const QT *pq = (const QT *)e.pcb_q;
    const float wm = *wmax;
    for (int v = blockIdx.x; v < p.n_vox; v += gridDim.x) {
        const int2 win = e.vwin[v];
        const int nwin = win.y - win.x + 1;
        __syncthreads();
        for (int i = tid; i < nwin; i += PCB_T) hist_s[i] = 0;
        __syncthreads();
        const double bound = (double)e.vbound[v] * (double)wm;
        const float scale = bound > 0.0 ? (float)(1073741824.0 / bound) : 0.0f;
        int *hv = hist_s - win.x;
        // the voxel's records (all its lists) are one contiguous range, streamed flat
        const long long o0 = __ldg(e.pc_off + (size_t)v * p.det_nx);
        const long long o1 = scale > 0.0f ? __ldg(e.pc_off + (size_t)(v + 1) * p.det_nx) : o0;
        for (long long o = o0 + tid; o < o1; o += 4 * PCB_T) {
            if (tid == 0 && pf > 0) {
                // rolling L2 prefetch of the records pf steps ahead
                const long long a0 = o + (long long)pf * 4 * PCB_T, a1 = min(o1, a0 + 4 * PCB_T);
                if (a0 < a1) {
                    l2_prefetch(e.pcb_bt + a0, (size_t)(a1 - a0) * sizeof(uint32_t));
                    l2_prefetch(e.pcb_P + a0, (size_t)(a1 - a0) * sizeof(float));
                    l2_prefetch(pq + a0, (size_t)(a1 - a0) * sizeof(QT));
                }
            }
            uint32_t k[4], q[4];
            float P[4], wq[4];
            // branch-free: slots past the end deposit zero into the window's first bin
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const bool in = o + u * PCB_T < o1;
                k[u] = in ? __ldg(e.pcb_bt + o + u * PCB_T) : ((uint32_t)win.x << tb);
                P[u] = in ? __ldg(e.pcb_P + o + u * PCB_T) : 0.0f;
                q[u] = in ? (uint32_t)__ldg(pq + o + u * PCB_T) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) wq[u] = __ldg(w + q[u]) * scale;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                // the pair's P w scale split exactly between bins b and b + 1
                const int b = (int)(k[u] >> tb);
                const float a = P[u] * wq[u];
                const int x1 = __float2int_rn(a * ((float)(k[u] & tmask) * tunit));
                CACSI_CHECK(b >= win.x && b + 1 <= win.y);
                atomicAdd(hv + b, __float2int_rn(a) - x1);
                atomicAdd(hv + b + 1, x1);
            }
        }
        __syncthreads();
        const float unit = scale > 0.0f ? (float)(bound / 1073741824.0) : 0.0f;
        float *Ar = A + (size_t)v * e.ldw;
        for (int b = tid; b < e.ldw; b += PCB_T) {
            const int i = b - win.x;
            Ar[b] = (i >= 0 && i < nwin) ? (float)hist_s[i] * unit : 0.0f;
        }
    }
}

// backward from the cache with the records fed through shared memory: thread 0
// streams the CTA's chunks (PBT_CH records, 16-byte-aligned groups of 8) with
// cp.async.bulk into a PBT_NS-stage ring ("full" mbarrier: bytes landed;
// "empty" mbarrier: every warp has read the stage), PBT_NS - 1 chunks ahead of
// the consumers and across voxel boundaries; the threads only gather w and
// deposit.  Same deposits and order-free integer sums as k_pc_bwd.
// Q8: 8-byte records -- the stage holds (b, tau, pixel offset) and P only; each warp's 128
// records are one window, whose pixel base it reads once per chunk
// PFL1: warp 1 peeks at the NEXT ring stage (non-blocking); if it has landed, its lanes
// sample 32 of its records' pixels and prefetch the w lines between their min and max into
// L1 (prefetch.global.L1), so the next chunk's gathers can hit L1 (option pcb_pfl1).
template <typename QT, int PBT_T, int PBT_U, int PBT_NS, int Q8 = 0, bool PFL1 = false>
__global__ void __launch_bounds__(PBT_T) k_pc_bwd_tma(const Params p, const Esai e, const float *__restrict__ w,
                                                      const float *__restrict__ wmax, float *__restrict__ A) {
    extern __shared__ __align__(16) unsigned char smb[];
    constexpr int PBT_CH = PBT_T * PBT_U;
    // Q8: + the chunk's window bases, copied from a 16-byte-aligned start (up to 7 extra)
    constexpr int QBN = (PBT_CH / 128 + 7 + 7) & ~7;
    constexpr int SB = PBT_CH * (8 + (Q8 ? 0 : (int)sizeof(QT))) + (Q8 ? QBN * 2 : 0);
    uint64_t *full = (uint64_t *)(smb + PBT_NS * SB);
    uint64_t *empty = full + PBT_NS;
    int *hist_s = (int *)(empty + PBT_NS);
    const int tid = threadIdx.x;
    const int tb = e.pc_tbits;
    const uint32_t tmask = Q8 ? (1u << e.pc_tb8) - 1u : (1u << tb) - 1u;
    const float tunit = Q8 ? 1.0f / (float)(1u << e.pc_tb8) : 1.0f / (float)(1u << tb);
    const int tsh = Q8 == 2 ? 5 : Q8 == 1 ? 9 : 0;  // tau's position in the record word
    const QT *pq = (const QT *)e.pcb_q;
    const bool vec = e.pc_R > 0;  // bank-ordered layout (segments 128-record aligned)
    const float wm = *wmax;
    if (tid == 0) {
        for (int i = 0; i < PBT_NS; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(full + i)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(empty + i)), "r"(PBT_T / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    __syncthreads();
    // producer state (thread 0): voxel pv, next chunk start pa, range end pe, chunks issued
    int pv = blockIdx.x;
    long long pa = 0, pe = 0;
    uint32_t issued = 0;
    if (tid == 0 && pv < p.n_vox) {
        pa = __ldg(e.pc_off + (size_t)pv * p.det_nx) & ~7ll;
        pe = __ldg(e.pc_off + (size_t)(pv + 1) * p.det_nx);
    }
    auto produce = [&](uint32_t limit) {
        while (issued < limit) {
            while (pv < p.n_vox && pa >= pe) {
                pv += gridDim.x;
                if (pv < p.n_vox) {
                    pa = __ldg(e.pc_off + (size_t)pv * p.det_nx) & ~7ll;
                    pe = __ldg(e.pc_off + (size_t)(pv + 1) * p.det_nx);
                }
            }
            if (pv >= p.n_vox) return;
            const int st = issued % PBT_NS;
            const uint32_t use = issued / PBT_NS;
            if (use > 0) {
                // every warp's reads of the stage (generic proxy) were released by its arrival
                // on "empty" and acquired by this wait: one proxy fence here orders them
                // before the bulk copy (async proxy) that overwrites the stage
                mbar_wait(smem_u32(empty + st), (use - 1) & 1);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            }
            const uint32_t n = (uint32_t)((min((long long)PBT_CH, pe - pa) + 7) & ~7ll);
            const uint32_t mb = smem_u32(full + st);
            unsigned char *dst = smb + st * SB;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                         "r"(n * (8u + (Q8 ? 0u : (uint32_t)sizeof(QT))) + (Q8 ? QBN * 2u : 0u)));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(dst)), "l"(e.pcb_bt + pa), "r"(n * 4u), "r"(mb) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             smem_u32(dst + PBT_CH * 4)), "l"(e.pcb_P + pa), "r"(n * 4u), "r"(mb) : "memory");
            if (!Q8)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                 smem_u32(dst + PBT_CH * 8)), "l"(pq + pa), "r"(n * (uint32_t)sizeof(QT)), "r"(mb) : "memory");
            else
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                 smem_u32(dst + PBT_CH * 8)), "l"(e.pc_qbase + ((pa >> 7) & ~7ll)), "r"(QBN * 2u),
                             "r"(mb) : "memory");
            pa += PBT_CH;
            issued++;
        }
    };
    if (tid == 0) produce(PBT_NS - 1);
    uint32_t consumed = 0;
    for (int v = blockIdx.x; v < p.n_vox; v += gridDim.x) {
        const int2 win = e.vwin[v];
        const int nwin = win.y - win.x + 1;
        for (int i = tid; i < nwin; i += PBT_T) hist_s[i] = 0;
        __syncthreads();
        const double bound = (double)e.vbound[v] * (double)wm;
        const float scale = bound > 0.0 ? (float)(1073741824.0 / bound) : 0.0f;
        int *hv = hist_s - win.x;
        const long long o0 = __ldg(e.pc_off + (size_t)v * p.det_nx), o1 = __ldg(e.pc_off + (size_t)(v + 1) * p.det_nx);
        // slots outside the voxel's range deposit zero (branch-free) into lane-spread bins,
        // not all into one address
        const uint32_t kinv = (uint32_t)(win.x + (tid & 31) % max(1, nwin - 1)) << tb;
        for (long long a = o0 & ~7ll; a < o1; a += PBT_CH) {
            if (tid == 0) produce(consumed + PBT_NS);
            const int st = consumed % PBT_NS;
            mbar_wait(smem_u32(full + st), (consumed / PBT_NS) & 1);
            const unsigned char *src = smb + st * SB;
            // this chunk's valid slots [lo, hi) (32-bit)
            const int lo = (int)max(o0 - a, 0ll), hi = (int)min(o1 - a, (long long)PBT_CH);
            // each thread takes 4 CONSECUTIVE records (vector reads of the stage): record u of
            // every lane's four forms one bank-aware group (k_pc_perm)
            static_assert(PBT_U == 4, "4 consecutive records per thread");
            uint32_t k[PBT_U], q[PBT_U];
            float P[PBT_U];
            {
                const uint4 kv = ((const uint4 *)src)[tid];
                const float4 pv = ((const float4 *)(src + PBT_CH * 4))[tid];
                k[0] = kv.x, k[1] = kv.y, k[2] = kv.z, k[3] = kv.w;
                P[0] = pv.x, P[1] = pv.y, P[2] = pv.z, P[3] = pv.w;
                if (Q8) {
                    // chunks start on window boundaries in the bank-ordered layout: warp w's 128
                    // records are window (a >> 7) + w (a read past the table's end only for
                    // slots outside the voxel, which are masked below)
                    const uint16_t *qbs = (const uint16_t *)(src + PBT_CH * 8) + ((a >> 7) & 7);
                    const uint32_t qb = 4 * tid < hi ? qbs[tid >> 5] : 0u;
#pragma unroll
                    for (int u = 0; u < PBT_U; u++) {
                        q[u] = qb + q8_off(Q8, k[u], P[u]);
                        P[u] = q8_P(Q8, P[u]);
                    }
                } else if (sizeof(QT) == 2) {
                    const uint2 qv = ((const uint2 *)(src + PBT_CH * 8))[tid];
                    q[0] = qv.x & 0xFFFFu, q[1] = qv.x >> 16, q[2] = qv.y & 0xFFFFu, q[3] = qv.y >> 16;
                } else {
                    const uint4 qv = ((const uint4 *)(src + PBT_CH * 8))[tid];
                    q[0] = qv.x, q[1] = qv.y, q[2] = qv.z, q[3] = qv.w;
                }
                if (vec) {
                    // bank-ordered layout: voxel ranges are whole 128-record windows (lo = 0,
                    // hi % 128 == 0), so a thread's four records are all in range or all out
                    if (4 * tid >= hi) {
#pragma unroll
                        for (int u = 0; u < PBT_U; u++) k[u] = kinv, P[u] = 0.0f, q[u] = 0u;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < PBT_U; u++) {
                        const int i = 4 * tid + u;
                        if (!(i >= lo && i < hi)) {
                            k[u] = kinv;
                            P[u] = 0.0f;
                            q[u] = 0u;
                        }
                    }
                }
            }
            if (PFL1 && (tid >> 5) == 1 && PBT_NS >= 2) {
                const int st2 = (consumed + 1) % PBT_NS;
                uint32_t landed;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(landed)
                    : "r"(smem_u32(full + st2)), "r"(((consumed + 1) / PBT_NS) & 1)
                    : "memory");
                if (landed) {
                    // (Q8: the stage's window bases, up to 8 + 7 of them from a 16-byte-aligned
                    // start; a base plus the 9-bit offsets spans <= 512 pixels)
                    uint32_t qs;
                    if (Q8) {
                        const uint16_t *qbn = (const uint16_t *)(smb + st2 * SB + PBT_CH * 8);
                        qs = (uint32_t)qbn[(tid & 31) % QBN] + ((tid & 1) ? 511u : 0u);
                    } else {
                        const QT *qn = (const QT *)(smb + st2 * SB + PBT_CH * 8);
                        qs = (uint32_t)qn[(tid & 31) * (PBT_CH / 32)];
                    }
                    const uint32_t qlo = __reduce_min_sync(0xFFFFFFFFu, qs), qhi = __reduce_max_sync(0xFFFFFFFFu, qs);
                    if (qhi >= qlo && qhi < (uint32_t)p.n_det && qhi - qlo < 16384u) {
                        const uintptr_t l0 = (uintptr_t)(w + qlo) & ~(uintptr_t)127, l1 = (uintptr_t)(w + qhi);
                        for (uintptr_t ad = l0 + 128 * (tid & 31); ad <= l1; ad += 128 * 32)
                            asm volatile("prefetch.global.L1 [%0];\n" ::"l"(ad));
                    }
                }
            }
            // one arrival per warp (release: this warp's stage reads happen before it)
            __syncwarp();
            if ((tid & 31) == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(empty + st)) : "memory");
            consumed++;
            float wq[PBT_U];
#pragma unroll
            for (int u = 0; u < PBT_U; u++) wq[u] = __ldg(w + q[u]) * scale;
#pragma unroll
            for (int u = 0; u < PBT_U; u++) {
                const int b = (int)(k[u] >> tb);
                const float av = P[u] * wq[u];
                const int x1 = __float2int_rn(av * ((float)((k[u] >> tsh) & tmask) * tunit));
                CACSI_CHECK(b >= win.x && b + 1 <= win.y);
                atomicAdd(hv + b, __float2int_rn(av) - x1);
                atomicAdd(hv + b + 1, x1);
            }
        }
        __syncthreads();
        const float unit = scale > 0.0f ? (float)(bound / 1073741824.0) : 0.0f;
        // whole rows (zeros outside the window): writing only the tile's chunk range that
        // the b2 GEMM reads measured slower (gaps between the rows of neighbouring voxels)
        float *Ar = A + (size_t)v * e.ldw;
        for (int b = tid; b < e.ldw; b += PBT_T) {
            const int i = b - win.x;
            Ar[b] = (i >= 0 && i < nwin) ? (float)hist_s[i] * unit : 0.0f;
        }
        __syncthreads();
    }
}

