// internal.h -- library-private types of libcacsi (not shared with oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <vector>

#include "cacsi.h"

// Device-side bounds checks of the hot kernels' shared-memory and table indices,
// compiled in only for the checked build (python -m paper_1603_06400_b200.build --checked
// -> libcacsi_checked.so, loaded by the binding when CACSI_CHECKED=1): the stand-in for
// compute-sanitizer, which this pool does not run.  A failed check prints and traps.
#ifdef CACSI_CHECKS
#define CACSI_CHECK(c)                                                                          \
    do {                                                                                        \
        if (!(c)) {                                                                             \
            printf("CACSI_CHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define CACSI_CHECK(c) \
    do {               \
    } while (0)
#endif

namespace cacsi {

constexpr double kHc = 12.3984193;          // keV Angstrom
constexpr float kMagic = 12582912.0f;        // 1.5 * 2^23: x + kMagic rounds x to an integer
constexpr int kMagicBits = 0x4B400000;       // __float_as_int(kMagic)
constexpr float kMaskGuard = 5e-4f;          // minimum mask-cell guard band, cells
constexpr double kAtanXMax = 0.0149;         // dtheta's atan(x) = x (1 - x^2/3) is used for x <= this (x^4/5 < 1e-8)

// fp32 per-voxel record (32 B, two float4 loads).  All derived in fp64 on the
// host from the descriptor ("precompute G_so").
struct alignas(16) VoxelRec {
    float y, z;    // centre (config frame)
    float ry, rz;  // r^ = r / |r|
    float sz;      // det_z - z  (> 0 by validation)
    float gso;     // G_so = z / |r|^3
    float tq;      // t / mask_pitch,  t = (mask_z - z) / (det_z - z)
    float ay;      // (y (1 - t) - m0y) / mask_pitch: u_y = tq * y_d + ay
};

// Everything a kernel needs, passed by value (lives in the constant bank).
struct Params {
    int ny, nz, nq, ne;
    int det_nx, det_ny;
    int n_vox, n_det;
    int mask_nx, mask_ny, mask_words;  // mask_words = 32-bit words per mask row (x)
    int energy_resolving;
    int uniform_e;                     // energies uniformly spaced -> closed-form k range
    float det_z;
    float pitch_d;                     // detector pitch p
    float quarter_p2;                  // p^2 / 4
    float ax;                          // -m0x / mask_pitch: u_x = tq * x_d + ax
    float mask_guard;                  // fp32 cell coordinates within this of an edge take the fp64 rule
    float nb;                          // -(q_min / dq) - 1/2   (u' = alpha_k sh + nb = u - 1/2)
    float qm;                          // nq - 1/2               (clamp bound of u')
    float klo_num, khi_num;            // (q_min/dq - 1), (q_min/dq + nq): alpha range numerators
    float a0, inv_da;                  // alpha_k = a0 + k / inv_da when uniform_e
    // translation symmetry: voxel y pitch = ts_rho * detector pitch
    // => y_d(jy) - y_r(iy) = ts_c0 + pitch_d * (jy - ts_rho * iy); 0 = not applicable
    int ts_rho;
    float ts_c0;
    float vy0, vy_step;                // voxel centre y = vy0 + iy * vy_step (fp32, the TS forward's r^)
    float det_x0, det_y0;              // pixel (0, 0) centre (fp32): x = det_x0 + ix p, y = det_y0 + jy p
    uint32_t det_div;                  // ix = umulhi(q, det_div) for q < 2^16 (floor(2^32 / det_ny) + 1)
    // fp64 guard path (exact oracle op order, reading R8)
    double m0x, m0y, mask_pitch64;
    double det_z64;
    // scatter-angle interpolation (reading R22): sai_n > 0
    int sai_n;
    double sai_tmin, sai_h;
    // device tables
    const VoxelRec *vox;
    const double *vy64, *vz64, *vt64;  // voxel y, z, t in fp64
    const float2 *det;                 // pixel (x, y) fp32
    const double *dx64, *dy64;         // pixel x, y fp64
    const uint32_t *maskbits;          // [mask_nx][mask_words], bit j of word w = cell (i, 32w + j)
    const float2 *energy;              // (alpha_k, c_k): alpha_k = E_k/(hc dq), c_k = scale phi_k E_k
};

// ESAI tables (energy-integrating handles; esai.cu).
struct Esai {
    int enabled;
    int nb;             // breakpoints s_0 < ... < s_{nb-1} (fp32, strictly increasing)
    int nl;             // lookup cells over the fp32 bit patterns of [s_0, s_{nb-1}]
    int max_win;        // max per-voxel breakpoint window (backward histogram size)
    int n_slow;         // LUT cells flagged kLutSlow (diagnostic)
    int sai_i0;         // SAI: tabulated-angle index of the first cell (cell b <-> angle sai_i0 + b)
    int lut_b0, lut_sh; // cell c = (float_as_int(sigma) - lut_b0) >> lut_sh
    const float *sb;    // breakpoints s_b (fp32, strictly increasing), kLocD +inf pads
    const uint16_t *lut16;  // per cell: b at the cell start | kLutSlow if > kLocD breakpoints inside
    const float *vbound;    // per voxel max_b sum_pixels P hat_b (backward fixed-point bound)
    const float *stab;  // S~ [nb][nq] (scale, phi_k, E_k folded in)
    const int2 *vwin;   // per voxel [b_lo, b_hi] reachable by any of its pairs
    const int2 *trng;   // per 128-voxel GEMM tile: the union of its voxels' windows, [lo, hi) in bins
    const int2 *pc_segwin;  // bank-ordered cache: per (voxel, row block) segment, the W columns it reads (or null)
    const int *w_pre;   // W GEMM tile list: exclusive prefix count of the N tiles inside trng, per M tile [+1]
    const int2 *w_ntr;  // W GEMM tile list: first / last N tile inside trng, per M tile
    const float *ptot;  // per voxel sum_pixels |P| (fixed-point bound)
    // pixels seen by at least one open pair ([ceil(n_det / 32)] bits): only their
    // weights can reach a backward histogram, so max |w| (the fixed-point scale) is
    // taken over them -- a huge w on a pixel no voxel sees (e.g. the ratio guard
    // y / 1e-12 where A f + r = 0) cannot wipe out every other deposit
    const uint32_t *seen;
    // precomputed transmission bits T(r, r') (mask factors computed
    // offline), one bit per pair in the order each pair kernel visits them
    const uint32_t *tb_fwd;  // forward (TS or tiled layout, esai.cu)
    int ldw;                 // row stride of W / A (nb rounded up to 32, zero padded)
    const float *tc_w;       // S~ as pre-split, pre-swizzled tensor-core B tiles (W = F S~^T), pair tiles
    const float *tc_w1;      // the same in disjoint tiles (plain W rows)
    const float *tc_b;       // S~^T likewise (b2 = A S~)
    // the same operands split into fp16 hi / lo (scaled by 2^s16_exp) for the fp16-rate
    // GEMMs of tcgemm16.cuh (option gemm16): S~ in disjoint 128 x 64 tiles, S~^T
    const void *tc16_w1, *tc16_b;
    int s16_exp;             // 2^s16_exp max|S~| < 2^14
    float vbmax;             // max_v vbound[v] (the b2 GEMM's A scale: |A| <= vbmax max|w|)
    const uint32_t *tb_bwd;  // backward: [voxel][ceil(n_det/32)], bit i of word j = pixel 32 j + i
    // pair cache (esai.cu "pair cache"): per open pair of list (voxel v, detector row ix),
    // pixels; with pc_R > 0 each (voxel, block of pc_R rows) segment
    // is padded to a multiple of 32 records (P = 0) and permuted in 128-record
    // windows so that the 32 records of each warp access hit distinct banks
    int pc;                   // built
    long long pc_n;           // records incl. padding
    long long pc_nopen;       // open pairs
    int pc_R;                 // rows per segment (0: plain per-list layout)
    const long long *pc_off;  // [n_vox * det_nx + 1] first record of list (v, ix)
    const uint32_t *pc_bt;    // (b << pc_tbits) | round(tau 2^pc_tbits)
    const float *pc_P;        // P (the pair's geometric-spectral factor, transmission included)
    const void *pc_q;         // pixel q, uint16 (n_det <= 65536) or uint32
    // the records the backward reads (= pc_*; kept separate for layout experiments)
    const uint32_t *pcb_bt;
    const float *pcb_P;
    const void *pcb_q;
    int pc_tbits;             // fraction bits of tau (>= 16); also b's shift in the packed word
    // 8-byte records (pc_q8): the pixel is stored as a 9-bit offset (bits 0-8) from a per-window
    // base (pc_qbase, one uint16 per 128-record window) and tau keeps pc_tb8 bits (bits 9 ..),
    // b stays at bit pc_tbits; the pixel array pc_q is then not kept
    int pc_q8;                // 0: 10-byte records; 1, 2: 8-byte (k_pc_pack8 MODE)
    int pc_tb8;               // tau bits of the 8-byte records (at bit 9 in mode 1, bit 5 in mode 2)
    const uint16_t *pc_qbase;
    int pc_qb;                // bytes per q (2 or 4)
    int pc_padq;              // every padding record's pixel is closed for its voxel (k_pc_fill)
    int stat_win_permille, stat_tile_permille;  // mean voxel window / 128-voxel tile K span, per mille of nb
};

// Energy-resolving pair cache (er_cache.cu): every open pair with an
// in-range energy, per detector pixel q in increasing voxel order, as SoA records
//   vw = v | klo << 16 | khi << 24   (voxel, first / last energy whose u_k can lie in (-1, nq))
//   P  = the pair's geometric-spectral factor (transmission included), s = sin(theta/2)
// plus per (voxel block of kErVB voxels, pixel) the record offset relative to off[q].
constexpr int kErVB = 128;
struct ErCache {
    int enabled;
    long long n;              // records
    int nvb;                  // voxel blocks
    int nr;                   // energy rounds of 16
    int nlo;                  // lower table pad (entries below q node 0)
    int nt;                   // forward table entries per voxel (nlo + nq + 1, even)
    float cmax;               // max_k c_k
    const long long *off;     // [n_det + 1]
    const uint32_t *vw;
    const float *P, *s;
    const uint32_t *boff;     // [nvb + 1][n_det], relative to off[q]
    const float *sv;          // per voxel fixed-point scale factor of the backward (times 1 / max|w|)
};

// Kernel-variant options of a handle (cacsi_geometry_create_ex "key=value,..." and
// cacsi_set_option).  The defaults are the measured-best settings;
// every other value selects a kernel that computes the same operator (an A/B
// measurement or an independent cross-check in the tests).  Nothing in the
// library reads the process environment.
struct Opts {
    // create-time (fixed for the life of the handle)
    int pair_cache = 1;       // "pair_cache": 0 = recompute the pair geometry per call
    int ts = 1;               // "ts": 0 = no translation-symmetric on-the-fly forward
    int direct = 0;           // "direct": 1 = per-term kernels instead of ESAI
    int pc_plain = 0;         // "pc_plain": 1 = pair cache in list order, unpadded
    int pc_segwin = 1;        // "pc_segwin": 0 = stage whole voxel windows in the forward
    int pc_win = 128;         // "pc_win": records per bank-aware permutation window (128, 256, 512)
    int pc_q8 = 2;            // "pc_q8": 8-byte records (pixel offset from a per-window base): 1 = 10-bit tau; 2 = P rounded to 28 bits carrying 4 offset bits, tau with tbits - 5 bits
    int pcv_budget_kb = 200;  // "pcv_budget_kb": shared memory of the voxel-major forward
    int er_cache = 0;         // "er_cache": 1 = energy-resolving operators from the pair cache (er_cache.cu)
    int pc_perm_lane = 1;     // "pc_perm_lane": 0 = the bank-aware permutation one window per warp (k_pc_perm)
    int er_vcache = 1;        // "er_vcache": 0 = no voxel-major open-pair cache for the energy-resolving backward
    int er_fcache = 1;        // "er_fcache": 0 = no pixel-major open-pair records for the energy-resolving forward (k_forward_rec)
    // per call (cacsi_set_option may change them between calls)
    int wgemm = 0;            // "wgemm": 0 A-resident, 1 CTA-pair (cta_group::2), 2 per-tile
    int wgemm_pack = 0;       // "wgemm_pack": 1 = pre-split f (k_tc_pack_a) instead of TMA + in-kernel split
    int b2gemm_tiles = 0;     // "b2gemm_tiles": 1 = per-tile b2 GEMM instead of the persistent split-K one
    int gemm16 = 1;           // "gemm16": 0 = W and b2 GEMMs on 3xTF32 (tcgemm.cuh) instead of the fp16 split (tcgemm16.cuh)
    int w_tmast = 1;          // "w_tmast": 0 = the fp16 W GEMM stores W per lane (STG) instead of by TMA tensor stores
    int b2_tmast = 1;         // "b2_tmast": 0 = the fp16 b2 GEMM stores its partials per lane (STG) instead of by TMA tensor stores
    int b2_rings = 1;         // "b2_rings": A / B ring depths of the fp16 b2 GEMM (0: 3 / 3, 1: 4 / 2, 2: 2 / 4)
    int b2_splits = 16;       // "b2_splits": split-K count of the fp16 b2 GEMM (16: accuracy)
    int pc_fwd_list = 0;      // "pc_fwd_list": 1 = per-list pair-cache forward (plain layout only)
    int pc_fwd_geom = 0;      // "pc_fwd_geom": 1 = the voxel-major forward recomputes P (6-byte records)
    int pcv_items = 2;        // "pcv_items": voxel chunks per SM of the voxel-major forward
    int pcv_pf = 1;           // "pcv_pf": L2 prefetch distance (voxels) of the voxel-major forward
    int pcv_u = 4;            // "pcv_u": records per thread per step (4 or 8)
    int pcv_padq = 1;         // "pcv_padq": 0 = the voxel-major forward redirects padding to dummy slots
    int pcv_pipe = 1;         // "pcv_pipe": 0 = the voxel-major forward without software-pipelined record loads
    int pc_bwd_flat = 0;      // "pc_bwd_flat": 1 = register-fed pair-cache backward
    int pcb_pf = 2;           // "pcb_pf": its rolling L2 prefetch distance
    int pcb_ctas = 0;         // "pcb_ctas": ring-backward CTAs per SM (0: as many as fit)
    int pcb_carve = 0;        // "pcb_carve": its shared-memory carveout preference in percent (0: the driver's)
    int pcb_pfl1 = 1;         // "pcb_pfl1": 0 = the ring backward does not prefetch the next chunk's w lines into L1
    int subset_bwd_mask = 0;  // "subset_bwd_mask": 1 = bitmap-masked subset backward
    int er_bwd_dense = 0;     // "er_bwd_dense": 1 = energy-resolving backward without compaction
    int er_fwd_reg = 1;       // "er_fwd_reg": 0 = the direct energy-resolving forward with shared-memory accumulators
    int er_fwd = 0;           // "er_fwd" (er_cache=1 only): 1 = the compacted pair-cache forward k_er_fwd2
    int er_fwd_lane = 1;      // "er_fwd_lane": 0 = the register forward with warp-uniform voxels (k_forward_reg)
    int er_bwd_fx = 1;        // "er_bwd_fx": 0 = the direct energy-resolving backward with fp32 shared-memory histograms
    int er_vcache_use = 1;    // "er_vcache_use": 0 = its pair geometry recomputed per call even when the cache exists
    int er_fwd_win = 6;       // "er_fwd_win": k_forward_rec lanes wait while more than this many voxels past the warp's lowest
    int er_fwd_rec = 1;       // "er_fwd_rec": 0 = k_forward_lane (mask tests and pair geometry per call) even when the forward records exist
    int graphs = 1;           // "graphs": 0 = cacsi_osem by stream launches
};

}  // namespace cacsi

struct cacsi_geometry {
    int device;
    cacsi::Opts opt;
    cacsi::Params p;
    // copies of the descriptor scalars we need later
    int32_t ny, nz, nq, ne, det_nx, det_ny, energy_resolving;
    size_t n_obj, n_detout;
    // device allocations (owned)
    void *d_vox, *d_vy64, *d_vz64, *d_vt64, *d_det, *d_dx64, *d_dy64, *d_mask, *d_energy;
    // ESAI (energy-integrating only)
    cacsi::Esai esai;
    void *d_esai_bp, *d_esai_lut, *d_esai_sb, *d_esai_stab, *d_esai_vwin, *d_esai_ptot, *d_tb_fwd, *d_tb_bwd, *d_tc_w, *d_tc_b,
        *d_esai_vbound, *d_pc_off, *d_pc_bt, *d_pc_P, *d_pc_q, *d_tc_w1, *d_esai_trng, *d_w_tiles, *d_pc_segwin, *d_seen, *d_pc_qbase,
        *d_tc16_w1, *d_tc16_b;
    // energy-resolving pair cache (er_cache.cu)
    cacsi::ErCache er;
    void *d_er_off, *d_er_vw, *d_er_P, *d_er_s, *d_er_boff, *d_er_sv;
    // the same pixel-major records alone, for the default energy-resolving forward (option er_fcache)
    cacsi::ErCache erf;
    void *d_erf_off, *d_erf_vw, *d_erf_P, *d_erf_s, *d_erf_boff;
    // fixed-point energy-resolving backward (operators.cu): per voxel bin bound
    // and max P, per pixel energy-window union over its open pairs (built at create)
    void *d_erx_vb, *d_erx_pm, *d_erx_pw;
    void *d_erx_voff, *d_erx_vw, *d_erx_vP, *d_erx_vs;  // its voxel-major open-pair cache (option er_vcache)
    long long erx_vc_n;
    int erx_nlo;  // its histogram rows below node 0: u' >= alpha_0 min(sin(theta/2)) - q_min/dq - 1/2
    // host staging for the *_host entry points (device scratch)
    float *d_stage_a, *d_stage_b, *d_stage_c, *d_stage_d, *d_stage_ws;
    // side stream + events of cacsi_iterate_host: y, r, b1 upload while the forward runs
    cudaStream_t stage_stream;
    cudaEvent_t stage_ev[3];
    cudaEvent_t stage_fev[4];  // f row chunks landed (cacsi_iterate_host, ESAI handles)
    mutable int32_t last_launches;
    // geometry_create stage times (host wall clock, microseconds; cacsi_query "setup_us_<stage>")
    long long setup_us[8];
    // per-kernel CUDA-event timing (cacsi_set_timing / cacsi_kernel_times)
    mutable int32_t timing;
    void *timers;  // cacsi::Timers*
    void *osem_graph;  // cacsi::OsemGraph*: the captured outer iteration of cacsi_osem (api.cu)
};

namespace cacsi {

// sets the handle's device for the scope of an entry point, restores the caller's after
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

struct TimerRec {
    const char *name;
    cudaEvent_t a, b;
};
struct Timers {
    std::vector<TimerRec> recs;
};

// Records a CUDA event pair around one kernel launch when timing is enabled
// on the handle (the bench's "kernel duration measured live with events").
struct KScope {
    const cacsi_geometry *g;
    cudaStream_t s;
    const char *name;
    cudaEvent_t a = nullptr, b = nullptr;
    KScope(const cacsi_geometry *g_, cudaStream_t s_, const char *name_);
    ~KScope();
};

// launchers (operators.cu / recon.cu).  Each returns a cudaError_t of the
// first failing launch and adds the number of kernels enqueued to *launches.
cudaError_t launch_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches);
cudaError_t launch_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches);
cudaError_t launch_ratio(const cacsi_geometry *g, const float *l, const float *y, const float *r, float *ratio,
                         double *partials, int nblocks, cudaStream_t s, int *launches);
// delta <= 0: quadratic potential; delta > 0: Huber psi_delta (recon.cu)
cudaError_t launch_update(const cacsi_geometry *g, const float *f_hat, const float *b1, const float *b2,
                          float beta, double delta, float *f_new, cudaStream_t s, int *launches);
cudaError_t launch_loglik(const cacsi_geometry *g, const float *l, const float *y, const float *r, const float *f,
                          float beta, double delta, double *partials, double *out, cudaStream_t s, int *launches);
// subset-restricted operators (Alg. 6): `pixels` = device list of n distinct detector pixels
cudaError_t launch_forward_subset(const cacsi_geometry *g, const float *f, const int32_t *pixels, int n, float *out,
                                  cudaStream_t s, int *launches);
cudaError_t launch_backward_subset(const cacsi_geometry *g, const float *w, const int32_t *pixels, int n, float *b,
                                   cudaStream_t s, int *launches);
cudaError_t esai_forward_list(const cacsi_geometry *g, const float *f, const int32_t *pixels, int n, float *out,
                              cudaStream_t s, int *launches);
// Fused epilogues of cacsi_iterate on ESAI handles: the forward's final partial sum
// writes w = y ./ (A f + r) and max |w| (as unsigned bits; *wmax zeroed by the
// caller) instead of A f; the backward takes that max (no k_absmax) and its final
// partial sum writes the f update (Eq. f_update) instead of b2.  Same bits as the
// unfused forward -> k_ratio -> backward -> k_update sequence (elementwise.cuh).
struct FwdRatioEpi {
    const float *y, *r;
    float *wmax;
    // optional: f arrives in f_chunks row chunks of fchunk_rows() rows (f_ready[c] recorded
    // when chunk c is on the device); the W GEMM starts on each chunk as it lands
    const cudaEvent_t *f_ready = nullptr;
    int f_chunks = 0;
    cudaEvent_t yr_ready = nullptr;  // optional: waited before the final sum (y, r staged)
};
inline int fchunk_rows(int n_vox, int n_chunks) {
    const int mt = (n_vox + 127) / 128;
    return (mt + n_chunks - 1) / n_chunks * 128;
}
struct BwdUpdateEpi {
    const float *wmax;
    const float *f_hat, *b1;
    float beta;
    double delta;
    float *f_new;
};
cudaError_t esai_backward_masked(const cacsi_geometry *g, const float *w, const uint32_t *pmask, float *b,
                                 cudaStream_t s, int *launches, const int32_t *list = nullptr, int n_list = 0,
                                 const BwdUpdateEpi *epi = nullptr);
cudaError_t esai_forward_ratio(const cacsi_geometry *g, const float *f, const FwdRatioEpi &epi, float *w,
                               cudaStream_t s, int *launches);
size_t recon_workspace_bytes(const cacsi_geometry *g);
cudaError_t esai_build(cacsi_geometry *g, const cacsi_geometry_desc *d);
cudaError_t er_build(cacsi_geometry *g, const cacsi_geometry_desc *d);
cudaError_t er_fcache_build(cacsi_geometry *g, size_t reserve);
cudaError_t er_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches);
cudaError_t er_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches);
cudaError_t erx_build(cacsi_geometry *g);
int pcv_row_blocks(const cacsi_geometry *g);
void osem_graph_free(cacsi_geometry *g);
cudaError_t esai_forward(const cacsi_geometry *g, const float *f, float *out, cudaStream_t s, int *launches);
cudaError_t esai_backward(const cacsi_geometry *g, const float *w, float *b, cudaStream_t s, int *launches);

}  // namespace cacsi
