// api.cu -- C ABI entry points and host setup.
//
// Host setup = the offline half of the paper's online/offline trade-off
// (PAPER.md:236-241): per-voxel G_so, r^ and mask-plane parameters, per-pixel
// centres, per-energy constants and the bit-packed mask are computed ONCE in
// fp64 and uploaded; esai_build (esai.cu) then builds the ESAI tables, the
// transmission bitmaps and the pair cache (each open pair's P and breakpoint
// cell, computed once on the device and streamed by every operator call).
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

using cacsi::Params;
using cacsi::VoxelRec;

namespace {

// Voxel / pixel centres, exactly the op order of DESIGN.md reading R9 (the
// fp64 guard path of the mask rule depends on bit-identical coordinates).
double centre(double lo, double hi, int n, int i) {
    double pitch = (hi - lo) / n;
    return lo + (i + 0.5) * pitch;
}
static uint32_t __float_as_uint_host(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
}
double det_centre(double c, int n, double p, int i) { return c + ((i + 0.5) - 0.5 * n) * p; }

// Fast-path preconditions, from the descriptor alone.
// (1) dtheta's series: x = p |s_yz| / (|s|^2 - p^2/4) <= p / (s - p^2 / (4 s)) with
//     s = det_z - z_max <= |s_yz|; atan(x) = x (1 - x^2/3) is used up to kAtanXMax.
double atan_xmax_of(const cacsi_geometry_desc *d) {
    const double sz = d->det_z - d->z_max, pp = d->det_pitch;
    return sz > pp ? pp / (sz - pp * pp / (4.0 * sz)) : INFINITY;
}
// (2) the fp32 mask-cell coordinate u = fma(tq, x, a) (pair.cuh mask_fast) has error
//     <= 1/2 ulp(|u|max) + 2^-23 |tq x|max + 1/2 ulp(|a|max) per axis (tq, x, a rounded
//     to fp32 once, as create rounds them); the guard band is 4x that, at least kMaskGuard.
double mask_guard_of(const cacsi_geometry_desc *d) {
    auto ulp = [](double v) { return v > 0.0 ? std::ldexp(1.0, std::ilogb(v) - 23) : 0.0; };
    const double mp = d->mask_pitch;
    const double m0x = d->mask_cx - (0.5 * d->mask_nx) * mp, m0y = d->mask_cy - (0.5 * d->mask_ny) * mp;
    double tqm = 0.0, aym = 0.0, xdm = 0.0, ydm = 0.0;
    for (int iy = 0; iy < d->ny; iy += std::max(1, d->ny - 1))  // t and |y| are extreme at the ends
        for (int iz = 0; iz < d->nz; iz++) {
            const double y = centre(d->y_min, d->y_max, d->ny, iy), z = centre(d->z_min, d->z_max, d->nz, iz);
            const double t = (d->mask_z - z) / (d->det_z - z);
            tqm = std::fmax(tqm, std::fabs((double)(float)(t / mp)));
            aym = std::fmax(aym, std::fabs((double)(float)((y * (1.0 - t) - m0y) / mp)));
        }
    for (int i = 0; i < d->det_nx; i += std::max(1, d->det_nx - 1))
        xdm = std::fmax(xdm, std::fabs((double)(float)det_centre(d->det_cx, d->det_nx, d->det_pitch, i)));
    for (int j = 0; j < d->det_ny; j += std::max(1, d->det_ny - 1))
        ydm = std::fmax(ydm, std::fabs((double)(float)det_centre(d->det_cy, d->det_ny, d->det_pitch, j)));
    const double axm = std::fabs((double)(float)(-m0x / mp));
    const double bx = 0.5 * ulp(tqm * xdm + axm) + std::ldexp(tqm * xdm, -23) + 0.5 * ulp(axm);
    const double by = 0.5 * ulp(tqm * ydm + aym) + std::ldexp(tqm * ydm, -23) + 0.5 * ulp(aym);
    return std::fmax((double)cacsi::kMaskGuard, 4.0 * std::fmax(bx, by));
}

cacsi_status validate(const cacsi_geometry_desc *d) {
    if (!d->energy_kev || !d->phi || !d->mask) return CACSI_ERR_NULL;
    if (d->ny < 1 || d->nz < 1 || d->nq < 2 || d->ne < 1 || d->mask_nx < 1 || d->mask_ny < 1 || d->det_nx < 1 ||
        d->det_ny < 1)
        return CACSI_ERR_INVALID;
    if (d->ne > 256 || d->nq > 400) return CACSI_ERR_INVALID;  // shared-memory tables
    // 32-bit element indexing of the object and the detector in the elementwise kernels
    if ((long long)d->ny * d->nz * d->nq >= (1ll << 31) || (long long)d->det_nx * d->det_ny * d->ne >= (1ll << 31))
        return CACSI_ERR_INVALID;
    if (!(d->y_min < d->y_max) || !(0.0 < d->z_min) || !(d->z_min < d->z_max) || !(d->z_max < d->mask_z) ||
        !(d->mask_z < d->det_z))
        return CACSI_ERR_INVALID;
    if (!(d->q_min < d->q_max) || !(d->mask_pitch > 0.0) || !(d->det_pitch > 0.0)) return CACSI_ERR_INVALID;
    if (!(d->scale > 0.0) || !std::isfinite(d->scale)) return CACSI_ERR_INVALID;
    if (d->energy_resolving != 0 && d->energy_resolving != 1) return CACSI_ERR_INVALID;
    if (d->sai_n_theta < 0) return CACSI_ERR_INVALID;
    if (d->sai_n_theta > 0) {
        if (d->energy_resolving) return CACSI_ERR_INVALID;  // SAI is the energy-integrating model's (Alg. 2)
        if (!std::isfinite(d->sai_theta_min) || !std::isfinite(d->sai_theta_max) || !(d->sai_theta_min >= 0.0))
            return CACSI_ERR_INVALID;
        if (d->sai_n_theta > 1 && !(d->sai_theta_min < d->sai_theta_max && d->sai_theta_max <= M_PI))
            return CACSI_ERR_INVALID;
    }
    for (int k = 0; k < d->ne; k++) {
        if (!(d->energy_kev[k] > 0.0) || !std::isfinite(d->energy_kev[k])) return CACSI_ERR_INVALID;
        if (k > 0 && !(d->energy_kev[k] > d->energy_kev[k - 1])) return CACSI_ERR_INVALID;
        if (!(d->phi[k] >= 0.0) || !std::isfinite(d->phi[k])) return CACSI_ERR_INVALID;
    }
    size_t nm = (size_t)d->mask_nx * d->mask_ny;
    for (size_t i = 0; i < nm; i++)
        if (d->mask[i] > 1) return CACSI_ERR_INVALID;
    const double v[] = {d->y_min, d->y_max, d->z_min, d->z_max, d->q_min, d->q_max, d->mask_z, d->mask_pitch,
                        d->mask_cx, d->mask_cy, d->det_z, d->det_pitch, d->det_cx, d->det_cy};
    for (double x : v)
        if (!std::isfinite(x)) return CACSI_ERR_INVALID;
    if (!(atan_xmax_of(d) <= cacsi::kAtanXMax)) return CACSI_ERR_INVALID;  // pixel too wide for the dtheta series
    if (!(mask_guard_of(d) < 0.25)) return CACSI_ERR_INVALID;              // fp32 mask coordinates too coarse
    return CACSI_OK;
}

template <class T>
cudaError_t upload(void **dst, const std::vector<T> &src) {
    cudaError_t e = cudaMalloc(dst, src.size() * sizeof(T));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
}

cacsi_status map_err(cudaError_t e) {
    if (e == cudaSuccess) return CACSI_OK;
    if (e == cudaErrorMemoryAllocation) return CACSI_ERR_NOMEM;
    return CACSI_ERR_CUDA;
}

void free_all(cacsi_geometry *g) {
    void *ptrs[] = {g->d_vox,  g->d_vy64, g->d_vz64,      g->d_vt64,      g->d_det,       g->d_dx64,
                    g->d_dy64, g->d_mask, g->d_energy,    g->d_stage_a,   g->d_stage_b,   g->d_stage_c,
                    g->d_stage_d, g->d_stage_ws, g->d_esai_bp, g->d_esai_lut, g->d_esai_sb, g->d_esai_stab,
                    g->d_esai_vwin, g->d_esai_ptot, g->d_esai_vbound, g->d_pc_off, g->d_pc_bt, g->d_pc_P, g->d_pc_q, g->d_tc_w1, g->d_esai_trng, g->d_w_tiles, g->d_pc_segwin, g->d_seen, g->d_tb_fwd, g->d_tb_bwd, g->d_tc_w, g->d_tc_b, g->d_er_off, g->d_er_vw, g->d_er_P, g->d_er_s, g->d_er_boff, g->d_er_sv, g->d_erx_vb, g->d_erx_pm, g->d_erx_pw, g->d_erx_voff, g->d_erx_vw, g->d_erx_vP, g->d_erx_vs, g->d_erf_off, g->d_erf_vw, g->d_erf_P, g->d_erf_s, g->d_erf_boff, g->d_pc_qbase, g->d_tc16_w1, g->d_tc16_b};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}

// ---- kernel-variant options (internal.h Opts) ----------------
struct OptKey {
    const char *name;
    int cacsi::Opts::*field;
    bool create_only;
    int lo, hi;
};
const OptKey kOptKeys[] = {
    {"pair_cache", &cacsi::Opts::pair_cache, true, 0, 1},
    {"ts", &cacsi::Opts::ts, true, 0, 1},
    {"direct", &cacsi::Opts::direct, true, 0, 1},
    {"pc_plain", &cacsi::Opts::pc_plain, true, 0, 1},
    {"pc_segwin", &cacsi::Opts::pc_segwin, true, 0, 1},
    {"pc_win", &cacsi::Opts::pc_win, true, 128, 512},
    {"pc_q8", &cacsi::Opts::pc_q8, true, 0, 2},
    {"pcv_budget_kb", &cacsi::Opts::pcv_budget_kb, true, 16, 227},
    {"er_cache", &cacsi::Opts::er_cache, true, 0, 1},
    {"pc_perm_lane", &cacsi::Opts::pc_perm_lane, true, 0, 1},
    {"er_vcache", &cacsi::Opts::er_vcache, true, 0, 1},
    {"er_fcache", &cacsi::Opts::er_fcache, true, 0, 1},
    {"wgemm", &cacsi::Opts::wgemm, false, 0, 2},
    {"wgemm_pack", &cacsi::Opts::wgemm_pack, false, 0, 1},
    {"b2gemm_tiles", &cacsi::Opts::b2gemm_tiles, false, 0, 1},
    {"gemm16", &cacsi::Opts::gemm16, false, 0, 1},
    {"b2_splits", &cacsi::Opts::b2_splits, false, 1, 64},
    {"w_tmast", &cacsi::Opts::w_tmast, false, 0, 1},
    {"b2_tmast", &cacsi::Opts::b2_tmast, false, 0, 1},
    {"b2_rings", &cacsi::Opts::b2_rings, false, 0, 2},
    {"pc_fwd_list", &cacsi::Opts::pc_fwd_list, false, 0, 1},
    {"pc_fwd_geom", &cacsi::Opts::pc_fwd_geom, false, 0, 1},
    {"pcv_items", &cacsi::Opts::pcv_items, false, 1, 64},
    {"pcv_pf", &cacsi::Opts::pcv_pf, false, 0, 16},
    {"pcv_u", &cacsi::Opts::pcv_u, false, 4, 8},
    {"pcv_pipe", &cacsi::Opts::pcv_pipe, false, 0, 1},
    {"pcv_padq", &cacsi::Opts::pcv_padq, false, 0, 1},
    {"pc_bwd_flat", &cacsi::Opts::pc_bwd_flat, false, 0, 1},
    {"pcb_pf", &cacsi::Opts::pcb_pf, false, 0, 64},
    {"pcb_pfl1", &cacsi::Opts::pcb_pfl1, false, 0, 1},
    {"pcb_ctas", &cacsi::Opts::pcb_ctas, false, 0, 8},
    {"pcb_carve", &cacsi::Opts::pcb_carve, false, 0, 100},
    {"subset_bwd_mask", &cacsi::Opts::subset_bwd_mask, false, 0, 1},
    {"er_bwd_dense", &cacsi::Opts::er_bwd_dense, false, 0, 1},
    {"er_fwd", &cacsi::Opts::er_fwd, false, 0, 1},
    {"er_fwd_reg", &cacsi::Opts::er_fwd_reg, false, 0, 1},
    {"er_fwd_lane", &cacsi::Opts::er_fwd_lane, false, 0, 1},
    {"er_bwd_fx", &cacsi::Opts::er_bwd_fx, false, 0, 1},
    {"er_vcache_use", &cacsi::Opts::er_vcache_use, false, 0, 1},
    {"er_fwd_rec", &cacsi::Opts::er_fwd_rec, false, 0, 1},
    {"er_fwd_win", &cacsi::Opts::er_fwd_win, false, 0, 1 << 20},
    {"graphs", &cacsi::Opts::graphs, false, 0, 1},
};

cacsi_status set_opt(cacsi::Opts &o, const char *key, size_t klen, long long v, bool at_create) {
    for (const OptKey &k : kOptKeys)
        if (strlen(k.name) == klen && strncmp(k.name, key, klen) == 0) {
            if ((k.create_only && !at_create) || v < k.lo || v > k.hi) return CACSI_ERR_INVALID;
            o.*(k.field) = (int)v;
            return CACSI_OK;
        }
    return CACSI_ERR_INVALID;
}

// "key=value,key=value" (integers; spaces not allowed); NULL or "" = defaults
cacsi_status parse_opts(const char *s, cacsi::Opts &o) {
    o = cacsi::Opts();
    if (!s) return CACSI_OK;
    while (*s) {
        const char *eq = strchr(s, '=');
        if (!eq || eq == s) return CACSI_ERR_INVALID;
        if (!((eq[1] >= '0' && eq[1] <= '9') || eq[1] == '-')) return CACSI_ERR_INVALID;
        char *end = nullptr;
        const long long v = strtoll(eq + 1, &end, 10);
        if (end == eq + 1 || (*end != ',' && *end != '\0') || (*end == ',' && end[1] == '\0'))
            return CACSI_ERR_INVALID;
        const cacsi_status st = set_opt(o, s, (size_t)(eq - s), v, true);
        if (st != CACSI_OK) return st;
        s = *end == ',' ? end + 1 : end;
    }
    return CACSI_OK;
}

}  // namespace

namespace cacsi {
// NVTX range per entry point (visible in Nsight Systems / ncu --nvtx; no cost without a tool)
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};
// Every entry point that touches a handle's device memory runs on the handle's
// device and restores the caller's current device on return.
DeviceGuard::DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
    else prev = -1;
}
DeviceGuard::~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
}
}  // namespace cacsi

extern "C" {

const char *cacsi_status_string(cacsi_status s) {
    switch (s) {
        case CACSI_OK: return "ok";
        case CACSI_ERR_NULL: return "null pointer";
        case CACSI_ERR_INVALID: return "invalid argument";
        case CACSI_ERR_CUDA: return "CUDA error";
        case CACSI_ERR_NOMEM: return "out of memory";
    }
    return "unknown status";
}

cacsi_status cacsi_geometry_create(const cacsi_geometry_desc *d, int device, cacsi_geometry **out) {
    return cacsi_geometry_create_ex(d, device, nullptr, out);
}

cacsi_status cacsi_geometry_create_ex(const cacsi_geometry_desc *d, int device, const char *options,
                                      cacsi_geometry **out) {
    const auto t_start = std::chrono::steady_clock::now();
    if (!d || !out) return CACSI_ERR_NULL;
    *out = nullptr;
    cacsi_status st = validate(d);
    if (st != CACSI_OK) return st;
    cacsi::Opts opt;
    st = parse_opts(options, opt);
    if (st != CACSI_OK) return st;
    if (opt.pc_win != 128 && opt.pc_win != 256 && opt.pc_win != 512) return CACSI_ERR_INVALID;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return CACSI_ERR_CUDA;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return CACSI_ERR_CUDA;
    cacsi::DeviceGuard dg(device);
    cacsi::Nvtx nv_("cacsi_geometry_create");
    // keep stream-ordered scratch (W / A, split partials) cached across calls
    // instead of returning it to the OS at every synchronisation
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }

    cacsi_geometry *g = (cacsi_geometry *)calloc(1, sizeof(cacsi_geometry));
    if (!g) return CACSI_ERR_NOMEM;
    g->device = device;
    g->opt = opt;
    g->ny = d->ny;
    g->nz = d->nz;
    g->nq = d->nq;
    g->ne = d->ne;
    g->det_nx = d->det_nx;
    g->det_ny = d->det_ny;
    g->energy_resolving = d->energy_resolving;
    const int nvox = d->ny * d->nz, ndet = d->det_nx * d->det_ny;
    g->n_obj = (size_t)nvox * d->nq;
    g->n_detout = (size_t)ndet * (d->energy_resolving ? d->ne : 1);

    Params &p = g->p;
    p.ny = d->ny;
    p.nz = d->nz;
    p.nq = d->nq;
    p.ne = d->ne;
    p.det_nx = d->det_nx;
    p.det_ny = d->det_ny;
    p.n_vox = nvox;
    p.n_det = ndet;
    p.mask_nx = d->mask_nx;
    p.mask_ny = d->mask_ny;
    p.mask_words = (d->mask_ny + 31) / 32;
    p.energy_resolving = d->energy_resolving;

    const double mp = d->mask_pitch;
    const double m0x = d->mask_cx - (0.5 * d->mask_nx) * mp;  // reading R8 op order
    const double m0y = d->mask_cy - (0.5 * d->mask_ny) * mp;
    const double dq = (d->q_max - d->q_min) / (d->nq - 1);
    p.m0x = m0x;
    p.m0y = m0y;
    p.mask_pitch64 = mp;
    p.det_z = (float)d->det_z;
    p.det_z64 = d->det_z;
    p.sai_n = d->sai_n_theta;
    p.sai_tmin = d->sai_theta_min;
    p.sai_h = d->sai_n_theta > 1 ? (d->sai_theta_max - d->sai_theta_min) / (d->sai_n_theta - 1) : 1.0;
    p.pitch_d = (float)d->det_pitch;
    p.det_x0 = (float)det_centre(d->det_cx, d->det_nx, d->det_pitch, 0);
    p.det_y0 = (float)det_centre(d->det_cy, d->det_ny, d->det_pitch, 0);
    p.det_div = (uint32_t)(4294967296.0 / d->det_ny) + 1u;
    p.quarter_p2 = (float)(0.25 * d->det_pitch * d->det_pitch);
    p.ax = (float)(-m0x / mp);
    const double beta0 = d->q_min / dq;
    p.nb = (float)(-beta0 - 0.5);
    p.qm = (float)(d->nq - 0.5);
    p.klo_num = (float)(beta0 - 1.0);
    p.khi_num = (float)(beta0 + d->nq);

    // per-voxel tables
    std::vector<VoxelRec> vox(nvox);
    std::vector<double> vy(nvox), vz(nvox), vt(nvox);
    for (int iy = 0; iy < d->ny; iy++)
        for (int iz = 0; iz < d->nz; iz++) {
            const int v = iy * d->nz + iz;
            const double y = centre(d->y_min, d->y_max, d->ny, iy);
            const double z = centre(d->z_min, d->z_max, d->nz, iz);
            const double rn = std::sqrt(y * y + z * z);
            const double t = (d->mask_z - z) / (d->det_z - z);  // reading R8 op order
            VoxelRec &r = vox[v];
            r.y = (float)y;
            r.z = (float)z;
            r.ry = (float)(y / rn);
            r.rz = (float)(z / rn);
            r.sz = (float)(d->det_z - z);
            r.gso = (float)(z / (rn * rn * rn));  // G_so, PAPER.md:633 (config frame)
            r.tq = (float)(t / mp);
            r.ay = (float)((y * (1.0 - t) - m0y) / mp);
            vy[v] = y;
            vz[v] = z;
            vt[v] = t;
        }
    // per-pixel tables
    std::vector<float2> det(ndet);
    std::vector<double> dx(ndet), dy(ndet);
    for (int ix = 0; ix < d->det_nx; ix++)
        for (int jy = 0; jy < d->det_ny; jy++) {
            const int q = ix * d->det_ny + jy;
            dx[q] = det_centre(d->det_cx, d->det_nx, d->det_pitch, ix);
            dy[q] = det_centre(d->det_cy, d->det_ny, d->det_pitch, jy);
            det[q] = make_float2((float)dx[q], (float)dy[q]);
        }
    // per-energy constants; uniform spacing enables the closed-form k range
    std::vector<float2> en(d->ne);
    for (int k = 0; k < d->ne; k++)
        en[k] = make_float2((float)(d->energy_kev[k] / (cacsi::kHc * dq)),
                            (float)(d->scale * d->phi[k] * d->energy_kev[k]));
    p.uniform_e = 0;
    if (d->ne >= 2) {
        const double e0 = d->energy_kev[0], de = (d->energy_kev[d->ne - 1] - e0) / (d->ne - 1);
        bool uni = de > 0;
        for (int k = 0; k < d->ne && uni; k++)
            if (std::fabs(d->energy_kev[k] - (e0 + k * de)) > 1e-9 * d->energy_kev[d->ne - 1]) uni = false;
        if (uni) {
            p.uniform_e = 1;
            p.a0 = (float)(e0 / (cacsi::kHc * dq));
            p.inv_da = (float)((cacsi::kHc * dq) / de);
        }
    }
    p.mask_guard = (float)mask_guard_of(d);  // fast-path guard band (validated above)
    // bit-packed mask: word w of row i holds cells (i, 32w .. 32w+31)
    std::vector<uint32_t> bits((size_t)d->mask_nx * p.mask_words, 0u);
    for (int i = 0; i < d->mask_nx; i++)
        for (int j = 0; j < d->mask_ny; j++)
            if (d->mask[(size_t)i * d->mask_ny + j]) bits[(size_t)i * p.mask_words + j / 32] |= 1u << (j % 32);

    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = upload(&g->d_vox, vox);
    if (e == cudaSuccess) e = upload(&g->d_vy64, vy);
    if (e == cudaSuccess) e = upload(&g->d_vz64, vz);
    if (e == cudaSuccess) e = upload(&g->d_vt64, vt);
    if (e == cudaSuccess) e = upload(&g->d_det, det);
    if (e == cudaSuccess) e = upload(&g->d_dx64, dx);
    if (e == cudaSuccess) e = upload(&g->d_dy64, dy);
    if (e == cudaSuccess) e = upload(&g->d_mask, bits);
    if (e == cudaSuccess) e = upload(&g->d_energy, en);
    if (e != cudaSuccess) {
        free_all(g);
        free(g);
        cudaGetLastError();
        return map_err(e);
    }
    p.vox = (const VoxelRec *)g->d_vox;
    p.vy64 = (const double *)g->d_vy64;
    p.vz64 = (const double *)g->d_vz64;
    p.vt64 = (const double *)g->d_vt64;
    p.det = (const float2 *)g->d_det;
    p.dx64 = (const double *)g->d_dx64;
    p.dy64 = (const double *)g->d_dy64;
    p.maskbits = (const uint32_t *)g->d_mask;
    p.energy = (const float2 *)g->d_energy;
    // translation symmetry: voxel y pitch an integer multiple rho of the detector pitch
    {
        const double dyv = (d->y_max - d->y_min) / d->ny;
        const double rho = std::floor(dyv / d->det_pitch + 0.5);
        p.ts_rho = 0;
        if (rho >= 1.0 && rho <= 64.0 && std::fabs(dyv - rho * d->det_pitch) <= 1e-9 * d->det_pitch &&
            g->opt.ts && d->sai_n_theta == 0) {  // SAI runs the tiled forward
            p.ts_rho = (int)rho;
            p.ts_c0 = (float)(det_centre(d->det_cy, d->det_ny, d->det_pitch, 0) - centre(d->y_min, d->y_max, d->ny, 0));
            p.vy0 = (float)centre(d->y_min, d->y_max, d->ny, 0);
            p.vy_step = (float)dyv;
        }
    }
    // ESAI tables for the energy-integrating operators (option direct=1 keeps
    // the per-term kernels, used as a cross-check in the tests)
    if (d->sai_n_theta > 0 && g->opt.direct) {  // SAI lives in the ESAI tables
        free_all(g);
        free(g);
        return CACSI_ERR_INVALID;
    }
    if (!d->energy_resolving && !g->opt.direct) {
        e = cacsi::esai_build(g, d);
        if (e == cudaSuccess && d->sai_n_theta > 0 && !g->esai.enabled) {  // beyond the table limits
            free_all(g);
            free(g);
            return CACSI_ERR_INVALID;
        }
        if (e != cudaSuccess) {
            free_all(g);
            free(g);
            cudaGetLastError();
            return map_err(e);
        }
    }
    g->setup_us[6] = std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t_start)
                         .count();
    for (int i = 0; i < 6; i++) g->setup_us[6] -= g->setup_us[i];  // host tables, uploads, validation
    if (d->energy_resolving && !g->opt.direct && g->opt.er_cache) {
        e = cacsi::er_build(g, d);
        if (e != cudaSuccess) {
            free_all(g);
            free(g);
            cudaGetLastError();
            return map_err(e);
        }
    }
    if (d->energy_resolving && !g->er.enabled) {  // tables of the fixed-point direct backward
        e = cacsi::erx_build(g);
        if (e != cudaSuccess) {
            free_all(g);
            free(g);
            cudaGetLastError();
            return map_err(e);
        }
    }
    g->setup_us[7] = std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t_start)
                         .count();
    *out = g;
    return CACSI_OK;
}

cacsi_status cacsi_set_option(cacsi_geometry *g, const char *key, int64_t value) {
    if (!g || !key) return CACSI_ERR_NULL;
    return set_opt(g->opt, key, strlen(key), (long long)value, false);
}

void cacsi_geometry_destroy(cacsi_geometry *g) {
    if (!g) return;
    cacsi::DeviceGuard dg(g->device);
    cudaDeviceSynchronize();
    if (g->timers) {
        const char *names[64];
        double ms[64];
        int32_t n[64];
        cacsi_kernel_times(g, 64, names, ms, n);  // releases the recorded events
        delete (cacsi::Timers *)g->timers;
    }
    cacsi::osem_graph_free(g);
    if (g->stage_stream) cudaStreamDestroy(g->stage_stream);
    for (int i = 0; i < 3; i++)
        if (g->stage_ev[i]) cudaEventDestroy(g->stage_ev[i]);
    for (int i = 0; i < 4; i++)
        if (g->stage_fev[i]) cudaEventDestroy(g->stage_fev[i]);
    free_all(g);
    free(g);
}

size_t cacsi_workspace_bytes(const cacsi_geometry *g) { return g ? cacsi::recon_workspace_bytes(g) : 0; }
size_t cacsi_object_size(const cacsi_geometry *g) { return g ? g->n_obj : 0; }
size_t cacsi_detector_size(const cacsi_geometry *g) { return g ? g->n_detout : 0; }
int32_t cacsi_last_launch_count(const cacsi_geometry *g) { return g ? g->last_launches : 0; }

cacsi_status cacsi_forward(const cacsi_geometry *g, const float *f, float *out, void *stream) {
    if (!g || !f || !out) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_forward");
    int n = 0;
    cudaError_t e = cacsi::launch_forward(g, f, out, (cudaStream_t)stream, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_backward(const cacsi_geometry *g, const float *w, float *b, void *stream) {
    if (!g || !w || !b) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_backward");
    int n = 0;
    cudaError_t e = cacsi::launch_backward(g, w, b, (cudaStream_t)stream, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

// workspace layout (recon.cu: recon_workspace_bytes)
static void ws_split(const cacsi_geometry *g, void *ws, float **l, float **b2, float **fnew, double **part) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char *p = (char *)ws;
    *l = (float *)p;
    p += al(g->n_detout * sizeof(float));
    *b2 = (float *)p;
    p += al(g->n_obj * sizeof(float));
    *fnew = (float *)p;
    p += al(g->n_obj * sizeof(float));
    *part = (double *)p;
}

// penalty descriptor -> delta (<= 0: quadratic), or -1 on an invalid descriptor
static double pen_delta(const cacsi_penalty *pen) {
    if (!pen || pen->kind == CACSI_PENALTY_QUADRATIC) return 0.0;
    if (pen->kind == CACSI_PENALTY_HUBER && pen->delta > 0.0 && std::isfinite(pen->delta)) return pen->delta;
    return -1.0;
}

cacsi_status cacsi_neg_loglik_ex(const cacsi_geometry *g, const float *f, const float *y, const float *r, float beta,
                                 const cacsi_penalty *pen, double *out_dev, void *ws, void *stream) {
    if (!g || !f || !y || !r || !out_dev || !ws) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_neg_loglik_ex");
    const double delta = pen_delta(pen);
    if (delta < 0.0) return CACSI_ERR_INVALID;
    float *l, *b2, *fnew;
    double *part;
    ws_split(g, ws, &l, &b2, &fnew, &part);
    cudaStream_t s = (cudaStream_t)stream;
    int n = 0;
    cudaError_t e = cacsi::launch_forward(g, f, l, s, &n);
    if (e == cudaSuccess) e = cacsi::launch_loglik(g, l, y, r, f, beta, delta, part, out_dev, s, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_neg_loglik(const cacsi_geometry *g, const float *f, const float *y, const float *r, float beta,
                              double *out_dev, void *ws, void *stream) {
    return cacsi_neg_loglik_ex(g, f, y, r, beta, nullptr, out_dev, ws, stream);
}

// One Alg. 5 iteration f -> f_new.  ESAI handles run it fused: the
// forward's final partial sum writes w = y ./ (A f + r) and max |w| into *wmax_scratch,
// the backward's final sum the update (Eq. f_update) -- the same bits as the unfused
// forward -> ratio -> backward -> update sequence the other handles run.  wait_yr /
// wait_b1 (optional): events the ratio / the update must wait for (staged inputs).
static cudaError_t iterate_once(const cacsi_geometry *g, const float *fc, const float *y, const float *r,
                                const float *b1, float beta, double delta, float *fn, float *l, float *b2,
                                float *wmax_scratch, cudaStream_t s, int *n, cudaEvent_t wait_yr, cudaEvent_t wait_b1,
                                const cudaEvent_t *f_ready = nullptr, int f_chunks = 0) {
    cudaError_t e = cudaSuccess;
    if (g->esai.enabled) {
        e = cudaMemsetAsync(wmax_scratch, 0, sizeof(float), s);
        cacsi::FwdRatioEpi fe{y, r, wmax_scratch};
        fe.f_ready = f_ready;
        fe.f_chunks = f_chunks;
        fe.yr_ready = wait_yr;  // y, r are read only by the forward's final sum
        if (e == cudaSuccess) e = cacsi::esai_forward_ratio(g, fc, fe, l, s, n);
        if (e == cudaSuccess && wait_b1) e = cudaStreamWaitEvent(s, wait_b1, 0);
        const cacsi::BwdUpdateEpi up{wmax_scratch, fc, b1, beta, delta, fn};
        if (e == cudaSuccess) e = cacsi::esai_backward_masked(g, l, nullptr, b2, s, n, nullptr, 0, &up);
        return e;
    }
    e = cacsi::launch_forward(g, fc, l, s, n);                                     // z = A f (+ r below)
    if (e == cudaSuccess && wait_yr) e = cudaStreamWaitEvent(s, wait_yr, 0);
    if (e == cudaSuccess) e = cacsi::launch_ratio(g, l, y, r, l, nullptr, 0, s, n);  // y ./ z
    if (e == cudaSuccess) e = cacsi::launch_backward(g, l, b2, s, n);             // b2 = A^T (y ./ z)
    if (e == cudaSuccess && wait_b1) e = cudaStreamWaitEvent(s, wait_b1, 0);
    if (e == cudaSuccess) e = cacsi::launch_update(g, fc, b1, b2, beta, delta, fn, s, n);  // Eq. f_update
    return e;
}

cacsi_status cacsi_iterate_ex(const cacsi_geometry *g, float *f, const float *y, const float *r, const float *b1,
                              float beta, const cacsi_penalty *pen, int32_t n_iter, void *ws, void *stream) {
    if (!g || !f || !y || !r || !b1 || !ws) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_iterate_ex");
    const double delta = pen_delta(pen);
    if (n_iter < 0 || !(beta >= 0.0f) || !std::isfinite(beta) || delta < 0.0) return CACSI_ERR_INVALID;
    float *l, *b2, *fnew;
    double *part;
    ws_split(g, ws, &l, &b2, &fnew, &part);
    cudaStream_t s = (cudaStream_t)stream;
    int n = 0;
    cudaError_t e = cudaSuccess;
    // ping-pong between f and fnew; an odd iteration count ends with one copy back into f
    float *fc = f, *fn = fnew;
    for (int t = 0; t < n_iter && e == cudaSuccess; t++) {
        e = iterate_once(g, fc, y, r, b1, beta, delta, fn, l, b2, (float *)part, s, &n, nullptr, nullptr);
        std::swap(fc, fn);
    }
    if (e == cudaSuccess && fc != f) e = cudaMemcpyAsync(f, fc, g->n_obj * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_iterate(const cacsi_geometry *g, float *f, const float *y, const float *r, const float *b1,
                           float beta, int32_t n_iter, void *ws, void *stream) {
    return cacsi_iterate_ex(g, f, y, r, b1, beta, nullptr, n_iter, ws, stream);
}

cacsi_status cacsi_ratio(const cacsi_geometry *g, const float *l, const float *y, const float *r, float *ratio,
                         void *stream) {
    if (!g || !l || !y || !r || !ratio) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_ratio");
    int n = 0;
    cudaError_t e = cacsi::launch_ratio(g, l, y, r, ratio, nullptr, 0, (cudaStream_t)stream, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_update_ex(const cacsi_geometry *g, const float *f_hat, const float *b1, const float *b2, float beta,
                             const cacsi_penalty *pen, float *f_new, void *stream) {
    if (!g || !f_hat || !b1 || !b2 || !f_new) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_update_ex");
    const double delta = pen_delta(pen);
    if (!(beta >= 0.0f) || !std::isfinite(beta) || delta < 0.0) return CACSI_ERR_INVALID;
    int n = 0;
    cudaError_t e = cacsi::launch_update(g, f_hat, b1, b2, beta, delta, f_new, (cudaStream_t)stream, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_update(const cacsi_geometry *g, const float *f_hat, const float *b1, const float *b2, float beta,
                          float *f_new, void *stream) {
    return cacsi_update_ex(g, f_hat, b1, b2, beta, nullptr, f_new, stream);
}

// ---- ordered subsets (Alg. 6) ----------------------------
cacsi_status cacsi_symmetric_subsets(int32_t det_nx, int32_t det_ny, int32_t rho_x, int32_t rho_y,
                                     int32_t *subset_of_pixel, int32_t *n_subsets) {
    if (!subset_of_pixel || !n_subsets) return CACSI_ERR_NULL;
    if (det_nx < 2 || det_ny < 2 || det_nx % 2 || rho_x < 1 || (det_nx / 2) % rho_x || rho_y < 2 || rho_y % 2 ||
        det_ny % rho_y)
        return CACSI_ERR_INVALID;
    const int M = det_nx, N = det_ny, half = rho_y / 2;
    for (int i = 0; i < M; i++) {
        // vertical group: row i and its up-down mirror M-1-i share m = (min(i, M-1-i) mod rho_x)
        const int iu = i < M / 2 ? i : M - 1 - i;
        const int m = iu % rho_x;
        for (int j = 0; j < N; j++) {
            // horizontal group: columns n + k rho_y (r = j mod rho_y < rho_y/2) and their
            // left-right mirrors N-1-(n + k rho_y) (r >= rho_y/2 -> n = (N-1-j) mod rho_y)
            const int rj = j % rho_y;
            const int n = rj < half ? rj : (N - 1 - j) % rho_y;
            subset_of_pixel[(size_t)i * N + j] = m * half + n;
        }
    }
    *n_subsets = rho_x * half;
    return CACSI_OK;
}

cacsi_status cacsi_forward_subset(const cacsi_geometry *g, const float *f, const int32_t *pixels, int32_t n_pixels,
                                  float *out, void *stream) {
    if (!g || !f || !out || (n_pixels > 0 && !pixels)) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_forward_subset");
    if (n_pixels < 0 || n_pixels > g->p.n_det) return CACSI_ERR_INVALID;
    int n = 0;
    cudaError_t e = cacsi::launch_forward_subset(g, f, pixels, n_pixels, out, (cudaStream_t)stream, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_backward_subset(const cacsi_geometry *g, const float *w, const int32_t *pixels, int32_t n_pixels,
                                   float *b, void *stream) {
    if (!g || !w || !b || (n_pixels > 0 && !pixels)) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_backward_subset");
    if (n_pixels < 0 || n_pixels > g->p.n_det) return CACSI_ERR_INVALID;
    int n = 0;
    cudaError_t e = cacsi::launch_backward_subset(g, w, pixels, n_pixels, b, (cudaStream_t)stream, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

}  // extern "C"

// ---- cacsi_osem: one outer iteration (P subset sub-iterations, ~11 launches each)
// is captured once into a CUDA graph and replayed; the capture is cached per handle
// and reused while the call's arguments (pointers, subset offsets, beta, penalty)
// are the same -- the launch-bound loop then costs one graph launch per outer
// iteration instead of ~700 stream launches.
namespace cacsi {
struct OsemGraph {
    std::mutex mu;
    cudaStream_t cap = nullptr;  // capture stream (the caller's may be the legacy stream)
    cudaGraphExec_t exec = nullptr;
    std::vector<uint64_t> key;
    int launches = 0;
};
void osem_graph_free(cacsi_geometry *g) {
    OsemGraph *og = (OsemGraph *)g->osem_graph;
    if (!og) return;
    if (og->exec) cudaGraphExecDestroy(og->exec);
    if (og->cap) cudaStreamDestroy(og->cap);
    delete og;
    g->osem_graph = nullptr;
}
static cudaError_t osem_outer(const cacsi_geometry *g, float *f, const float *y, const float *r, const float *b1_subsets,
                              const int32_t *pixels, const int32_t *offsets, int32_t n_subsets, float beta_p,
                              double delta, float *l, float *b2, float *fnew, cudaStream_t s, int *n) {
    // ping-pong between f and fnew; an odd subset count ends with one copy back into f
    float *fc = f, *fn = fnew;
    cudaError_t e = cudaSuccess;
    for (int p = 0; p < n_subsets && e == cudaSuccess; p++) {
        const int32_t *px = pixels + offsets[p];
        const int np = offsets[p + 1] - offsets[p];
        e = launch_forward_subset(g, fc, px, np, l, s, n);                    // z_p = A_p f (+ r_p)
        if (e == cudaSuccess) e = launch_ratio(g, l, y, r, l, nullptr, 0, s, n);  // y_p ./ z_p
        if (e == cudaSuccess) e = launch_backward_subset(g, l, px, np, b2, s, n);  // b2_p
        if (e == cudaSuccess)
            e = launch_update(g, fc, b1_subsets + (size_t)p * g->n_obj, b2, beta_p, delta, fn, s, n);
        std::swap(fc, fn);
    }
    if (e == cudaSuccess && fc != f) e = cudaMemcpyAsync(f, fc, g->n_obj * sizeof(float), cudaMemcpyDeviceToDevice, s);
    return e;
}
}  // namespace cacsi

extern "C" {

cacsi_status cacsi_osem(const cacsi_geometry *g, float *f, const float *y, const float *r, const float *b1_subsets,
                        const int32_t *pixels, const int32_t *offsets, int32_t n_subsets, float beta,
                        const cacsi_penalty *pen, int32_t n_outer, void *ws, void *stream) {
    if (!g || !f || !y || !r || !b1_subsets || !pixels || !offsets || !ws) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_osem");
    const double delta = pen_delta(pen);
    if (n_subsets < 1 || n_outer < 0 || !(beta >= 0.0f) || !std::isfinite(beta) || delta < 0.0)
        return CACSI_ERR_INVALID;
    if (offsets[0] != 0) return CACSI_ERR_INVALID;
    for (int p = 0; p < n_subsets; p++)
        if (offsets[p + 1] < offsets[p] || offsets[p + 1] > g->p.n_det) return CACSI_ERR_INVALID;
    float *l, *b2, *fnew;
    double *part;
    ws_split(g, ws, &l, &b2, &fnew, &part);
    cudaStream_t s = (cudaStream_t)stream;
    const float beta_p = beta / (float)n_subsets;  // reading R20: the subset term stands for 1/P of L
    int n = 0;
    cudaError_t e = cudaSuccess;
    const bool use_graph = n_outer > 0 && !g->timing && g->opt.graphs;
    if (use_graph) {
        cacsi_geometry *gm = const_cast<cacsi_geometry *>(g);
        if (!gm->osem_graph) gm->osem_graph = new cacsi::OsemGraph();
        cacsi::OsemGraph *og = (cacsi::OsemGraph *)gm->osem_graph;
        std::lock_guard<std::mutex> lock(og->mu);
        std::vector<uint64_t> key = {(uint64_t)f, (uint64_t)y, (uint64_t)r, (uint64_t)b1_subsets, (uint64_t)pixels,
                                     (uint64_t)ws, (uint64_t)n_subsets, (uint64_t)__float_as_uint_host(beta_p),
                                     (uint64_t)(delta * 1e12)};
        for (int p = 0; p <= n_subsets; p++) key.push_back((uint64_t)offsets[p]);
        if (!og->exec || og->key != key) {
            if (og->exec) cudaGraphExecDestroy(og->exec);
            og->exec = nullptr;
            if (!og->cap) e = cudaStreamCreateWithFlags(&og->cap, cudaStreamNonBlocking);
            cudaGraph_t graph = nullptr;
            if (e == cudaSuccess) e = cudaStreamBeginCapture(og->cap, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
                int nl = 0;
                cudaError_t ec = cacsi::osem_outer(g, f, y, r, b1_subsets, pixels, offsets, n_subsets, beta_p, delta, l,
                                                   b2, fnew, og->cap, &nl);
                e = cudaStreamEndCapture(og->cap, &graph);
                if (ec != cudaSuccess) e = ec;
                og->launches = nl;
            }
            if (e == cudaSuccess) e = cudaGraphInstantiate(&og->exec, graph, 0);
            if (graph) cudaGraphDestroy(graph);
            if (e == cudaSuccess) og->key = key;
        }
        for (int t = 0; t < n_outer && e == cudaSuccess; t++) {
            e = cudaGraphLaunch(og->exec, s);
            n += og->launches;
        }
        if (e != cudaSuccess) {
            (void)cudaGetLastError();  // capture unsupported here: fall back to stream launches
            if (og->exec) cudaGraphExecDestroy(og->exec);
            og->exec = nullptr;
            og->key.clear();
            e = cudaSuccess;
            n = 0;
        } else {
            g->last_launches = n;
            return CACSI_OK;
        }
    }
    for (int t = 0; t < n_outer && e == cudaSuccess; t++)
        e = cacsi::osem_outer(g, f, y, r, b1_subsets, pixels, offsets, n_subsets, beta_p, delta, l, b2, fnew, s, &n);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

// ---- host-buffer variants (end-to-end timing path) -------------------------
static cudaError_t ensure_stage(const cacsi_geometry *gc) {
    cacsi_geometry *g = const_cast<cacsi_geometry *>(gc);
    cudaError_t e = cudaSuccess;
    if (!g->d_stage_a) e = cudaMalloc((void **)&g->d_stage_a, g->n_obj * sizeof(float));
    if (e == cudaSuccess && !g->d_stage_b) e = cudaMalloc((void **)&g->d_stage_b, g->n_detout * sizeof(float));
    if (e == cudaSuccess && !g->d_stage_c) e = cudaMalloc((void **)&g->d_stage_c, g->n_detout * sizeof(float));
    if (e == cudaSuccess && !g->d_stage_d) e = cudaMalloc((void **)&g->d_stage_d, g->n_obj * sizeof(float));
    if (e == cudaSuccess && !g->d_stage_ws) e = cudaMalloc((void **)&g->d_stage_ws, cacsi::recon_workspace_bytes(g));
    return e;
}

cacsi_status cacsi_forward_host(const cacsi_geometry *g, const float *fh, float *gh, void *stream) {
    if (!g || !fh || !gh) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_forward_host");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = ensure_stage(g);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->d_stage_a, fh, g->n_obj * 4, cudaMemcpyHostToDevice, s);
    int n = 0;
    if (e == cudaSuccess) e = cacsi::launch_forward(g, g->d_stage_a, g->d_stage_b, s, &n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(gh, g->d_stage_b, g->n_detout * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_backward_host(const cacsi_geometry *g, const float *wh, float *bh, void *stream) {
    if (!g || !wh || !bh) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_backward_host");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = ensure_stage(g);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->d_stage_b, wh, g->n_detout * 4, cudaMemcpyHostToDevice, s);
    int n = 0;
    if (e == cudaSuccess) e = cacsi::launch_backward(g, g->d_stage_b, g->d_stage_a, s, &n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bh, g->d_stage_a, g->n_obj * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

cacsi_status cacsi_iterate_host(const cacsi_geometry *g, float *fh, const float *yh, const float *rh,
                                const float *b1h, float beta, int32_t n_iter, void *stream) {
    if (!g || !fh || !yh || !rh || !b1h) return CACSI_ERR_NULL;
    cacsi::DeviceGuard dg_(g->device);
    cacsi::Nvtx nv_("cacsi_iterate_host");
    if (n_iter < 0 || !(beta >= 0.0f) || !std::isfinite(beta)) return CACSI_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    cacsi_geometry *gm = const_cast<cacsi_geometry *>(g);
    cudaError_t e = ensure_stage(g);
    if (e == cudaSuccess && !gm->stage_stream) {
        e = cudaStreamCreateWithFlags(&gm->stage_stream, cudaStreamNonBlocking);
        for (int i = 0; i < 3 && e == cudaSuccess; i++)
            e = cudaEventCreateWithFlags(&gm->stage_ev[i], cudaEventDisableTiming);
        for (int i = 0; i < 4 && e == cudaSuccess; i++)
            e = cudaEventCreateWithFlags(&gm->stage_fev[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return map_err(e);
    cudaStream_t s2 = g->stage_stream;
    // the side stream first waits for the caller's earlier work (it may still read the
    // staging buffers), then uploads f, y, r, b1 in that order.  ESAI handles: f in four
    // row chunks, the forward's W GEMM starting on each as it lands; others: f whole
    // before the forward.  The ratio waits for y, r, the update for b1.
    const bool fchunks = g->esai.enabled && n_iter > 0;
    const int nfc = fchunks ? 4 : 0;
    e = cudaEventRecord(g->stage_ev[0], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s2, g->stage_ev[0], 0);
    if (fchunks) {
        const size_t rows = (size_t)cacsi::fchunk_rows(g->p.n_vox, nfc), row_b = (size_t)g->p.nq * 4;
        for (int c = 0; c < nfc && e == cudaSuccess; c++) {
            const size_t r0 = std::min((size_t)g->p.n_vox, c * rows), r1 = std::min((size_t)g->p.n_vox, r0 + rows);
            if (r1 > r0)
                e = cudaMemcpyAsync((char *)g->d_stage_a + r0 * row_b, (const char *)fh + r0 * row_b, (r1 - r0) * row_b,
                                    cudaMemcpyHostToDevice, s2);
            if (e == cudaSuccess) e = cudaEventRecord(g->stage_fev[c], s2);
        }
    } else {
        e = cudaMemcpyAsync(g->d_stage_a, fh, g->n_obj * 4, cudaMemcpyHostToDevice, s);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->d_stage_b, yh, g->n_detout * 4, cudaMemcpyHostToDevice, s2);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->d_stage_c, rh, g->n_detout * 4, cudaMemcpyHostToDevice, s2);
    if (e == cudaSuccess) e = cudaEventRecord(g->stage_ev[1], s2);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->d_stage_d, b1h, g->n_obj * 4, cudaMemcpyHostToDevice, s2);
    if (e == cudaSuccess) e = cudaEventRecord(g->stage_ev[2], s2);
    if (e != cudaSuccess) return map_err(e);
    float *l, *b2, *fnew;
    double *part;
    ws_split(g, g->d_stage_ws, &l, &b2, &fnew, &part);
    float *fc = g->d_stage_a, *fn = fnew;  // ping-pong: no device copy between iterations
    int n = 0;
    for (int t = 0; t < n_iter && e == cudaSuccess; t++) {
        e = iterate_once(g, fc, g->d_stage_b, g->d_stage_c, g->d_stage_d, beta, 0.0, fn, l, b2, (float *)part, s, &n,
                         t == 0 ? g->stage_ev[1] : nullptr, t == 0 ? g->stage_ev[2] : nullptr,
                         t == 0 ? g->stage_fev : nullptr, t == 0 ? nfc : 0);
        std::swap(fc, fn);
    }
    if (e == cudaSuccess && n_iter == 0) e = cudaStreamWaitEvent(s, g->stage_ev[2], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(fh, fc, g->n_obj * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) g->last_launches = n;
    return map_err(e);
}

}  // extern "C"

// ---- per-kernel CUDA-event timing ------------------------------------------
namespace cacsi {
KScope::KScope(const cacsi_geometry *g_, cudaStream_t s_, const char *name_) : g(g_), s(s_), name(name_) {
    if (g && g->timing && g->timers) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
    }
}
KScope::~KScope() {
    if (a) {
        cudaEventRecord(b, s);
        ((Timers *)g->timers)->recs.push_back({name, a, b});
    }
}
}  // namespace cacsi

extern "C" {

cacsi_status cacsi_set_timing(const cacsi_geometry *g, int32_t enable) {
    if (!g) return CACSI_ERR_NULL;
    if (!g->timers) const_cast<cacsi_geometry *>(g)->timers = new cacsi::Timers();
    g->timing = enable ? 1 : 0;
    return CACSI_OK;
}

int32_t cacsi_kernel_times(const cacsi_geometry *g, int32_t max, const char **names, double *total_ms,
                           int32_t *launches) {
    if (!g || !g->timers) return 0;
    auto &recs = ((cacsi::Timers *)g->timers)->recs;
    int32_t n = 0;
    for (auto &r : recs) {
        float ms = 0.0f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&ms, r.a, r.b);
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
        int i = 0;
        while (i < n && strcmp(names[i], r.name) != 0) i++;
        if (i == n) {
            if (n >= max) continue;
            names[n] = r.name;
            total_ms[n] = 0.0;
            launches[n] = 0;
            n++;
        }
        total_ms[i] += ms;
        launches[i] += 1;
    }
    recs.clear();
    return n;
}

int64_t cacsi_query(const cacsi_geometry *g, const char *key) {
    if (!g || !key) return -1;
    if (!strcmp(key, "esai_breakpoints")) return g->esai.enabled ? g->esai.nb : 0;
    if (!strcmp(key, "ts_rho")) return g->p.ts_rho;
    if (!strcmp(key, "esai_max_window")) return g->esai.enabled ? g->esai.max_win : 0;
    if (!strcmp(key, "esai_lut_cells")) return g->esai.enabled ? g->esai.nl : 0;
    if (!strcmp(key, "esai_lut_slow_cells")) return g->esai.enabled ? g->esai.n_slow : 0;
    if (!strcmp(key, "esai_window_permille")) return g->esai.enabled ? g->esai.stat_win_permille : 0;
    if (!strcmp(key, "esai_tile_span_permille")) return g->esai.enabled ? g->esai.stat_tile_permille : 0;
    if (!strcmp(key, "pair_cache_records")) return g->esai.enabled && g->esai.pc ? g->esai.pc_nopen : 0;
    if (!strcmp(key, "pair_cache_padded_records")) return g->esai.enabled && g->esai.pc ? g->esai.pc_n : 0;
    if (!strcmp(key, "pair_cache_record_bytes"))
        return g->esai.enabled && g->esai.pc ? 2 * (long long)sizeof(float) + (g->esai.pc_q8 ? 0 : g->esai.pc_qb) : 0;
    if (!strcmp(key, "pair_cache_window_base_bytes"))  // the 8-byte format's per-window pixel bases
        return g->esai.enabled && g->esai.pc && g->esai.pc_q8 ? 2 * (g->esai.pc_n / 128) : 0;
    if (!strcmp(key, "pair_cache_tau_bits")) return g->esai.enabled && g->esai.pc ? g->esai.pc_tbits : 0;
    if (!strcmp(key, "pair_cache_padding_closed")) return g->esai.enabled && g->esai.pc ? g->esai.pc_padq : 0;
    if (!strcmp(key, "pair_cache_fwd_row_blocks"))
        return g->esai.enabled && g->esai.pc ? cacsi::pcv_row_blocks(g) : 0;
    if (!strcmp(key, "esai_ldw")) return g->esai.enabled ? g->esai.ldw : 0;
    if (!strcmp(key, "energy_resolving")) return g->p.energy_resolving;
    if (!strcmp(key, "er_cache_records")) return g->er.enabled ? g->er.n : 0;
    if (!strcmp(key, "er_vcache_records")) return g->d_erx_voff ? g->erx_vc_n : 0;
    if (!strcmp(key, "er_fcache_records")) return g->erf.enabled ? g->erf.n : 0;
    if (!strcmp(key, "mask_guard_ppm")) return (int64_t)std::llround(g->p.mask_guard * 1e6);
    static const char *stages[8] = {"setup_us_tables", "setup_us_bitmaps", "setup_us_bound", "setup_us_pc_fill",
                                    "setup_us_pc_perm", "setup_us_pc_segwin", "setup_us_host", "setup_us_total"};
    for (int i = 0; i < 8; i++)
        if (!strcmp(key, stages[i])) return g->setup_us[i];
    return -1;
}

}  // extern "C"
