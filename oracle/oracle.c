/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of the forward
 * model g = A f and its adjoint b = A^T w of arXiv 1603.06400.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1603_06400_b200/); neither includes the other.
 *
 * Built with: gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction, so the
 * mask-cell rule of DESIGN.md reading R8 is reproducible bit for bit).
 *
 * Every quantity is the plain definition written out:
 *
 *   config frame (BASELINE.json configs[0]): source at origin, beam +z,
 *   fan plane x = 0, voxel r = (0, y_r, z_r), pixel r' = (x_d, y_d, z_d).
 *   The paper's frame maps x->z, y->y, z->x.
 *
 *   G_so  = |n_o . r^| / r^2 = z_r / (y_r^2 + z_r^2)^{3/2}
 *   G_od  = |n_d . s^| / s^2 = |s_z| / |s|^3
 *   theta = angle(r^, s^)
 *   dtheta= angle between s + (p/2) x^ and s - (p/2) x^
 *   T     = mask bit where the ray r -> r' crosses z = z_m
 *   P     = C_E G_so G_od T dtheta (1 + cos^2 theta) cos(theta/2)
 *   u_k   = (E_k sin(theta/2) / hc - q_0) / dq   (Bragg)
 *   A[r' ; (r, j)] = P sum_k phi_k E_k Lambda(u_k - j)         energy-integrating
 *   A[(r', k) ; (r, j)] = P phi_k E_k Lambda(u_k - j)           energy-resolving
 *
 * The energy form is the paper's energy-integrated model (PAPER.md:585-590,
 * 599-618) integrated over q instead of E (reading R2).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HC_KEV_ANGSTROM 12.3984193

typedef struct {
    int32_t ny, nz;
    double y_min, y_max, z_min, z_max;
    int32_t nq;
    double q_min, q_max;
    int32_t ne;
    const double *energy_kev, *phi;
    int32_t mask_nx, mask_ny;
    double mask_z, mask_pitch, mask_cx, mask_cy;
    const uint8_t *mask; /* [mask_nx][mask_ny], 1 = open */
    int32_t det_nx, det_ny;
    double det_z, det_pitch, det_cx, det_cy;
    int32_t energy_resolving;
    double scale; /* C_E */
    /* scatter-angle interpolation:
     * sai_n_theta > 0 replaces the spectral-angular factor of every pair by its
     * value at the nearest of sai_n_theta uniform angles on
     * [sai_theta_min, sai_theta_max] (reading R22); 0 = the exact operator. */
    int32_t sai_n_theta;
    double sai_theta_min, sai_theta_max;
} oracle_desc;

/* ---- discretisation (readings R4, R9) ------------------------- */

/* voxel centre: min + (i + 1/2) * ((max - min) / n) */
static double voxel_y(const oracle_desc *d, int iy) {
    double pitch = (d->y_max - d->y_min) / d->ny;
    return d->y_min + (iy + 0.5) * pitch;
}
static double voxel_z(const oracle_desc *d, int iz) {
    double pitch = (d->z_max - d->z_min) / d->nz;
    return d->z_min + (iz + 0.5) * pitch;
}
/* detector centre: c + ((i + 1/2) - n/2) * pitch */
static double det_x(const oracle_desc *d, int ix) {
    return d->det_cx + ((ix + 0.5) - 0.5 * d->det_nx) * d->det_pitch;
}
static double det_y(const oracle_desc *d, int jy) {
    return d->det_cy + ((jy + 0.5) - 0.5 * d->det_ny) * d->det_pitch;
}
static double q_step(const oracle_desc *d) { return (d->q_max - d->q_min) / (d->nq - 1); }

/* the centre conventions above, exported for the tests' hand-value pins */
void oracle_voxel_centre(const oracle_desc *d, int iy, int iz, double out[2]) {
    out[0] = voxel_y(d, iy);
    out[1] = voxel_z(d, iz);
}
void oracle_det_centre(const oracle_desc *d, int ix, int jy, double out[2]) {
    out[0] = det_x(d, ix);
    out[1] = det_y(d, jy);
}

/* ---- vector helpers ------------------------------------------------------ */
static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double norm3(const double a[3]) { return sqrt(dot3(a, a)); }
static void cross3(const double a[3], const double b[3], double c[3]) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

/* ---- the factors of H, for arbitrary points (config frame) -------------- */

/* G_so(r) = |n_o . r^| / |r|^2, n_o = beam axis z^ */
double oracle_G_so(const double r[3]) {
    double rn = norm3(r);
    return fabs(r[2] / rn) / (rn * rn);
}
/* G_od(s) = |n_d . s^| / |s|^2, n_d = z^ */
double oracle_G_od(const double s[3]) {
    double sn = norm3(s);
    return fabs(s[2] / sn) / (sn * sn);
}
/* theta = angle between r^ and s^: atan2(|r x s|, r . s) */
double oracle_theta(const double r[3], const double rp[3]) {
    double s[3] = {rp[0] - r[0], rp[1] - r[1], rp[2] - r[2]};
    double c[3];
    cross3(r, s, c);
    return atan2(norm3(c), dot3(r, s));
}
/* dtheta: angle between the vectors from r to the midpoints of the pixel's
 * two edges along the out-of-fan axis x (reading R6):
 * a = s + (p/2) x^, b = s - (p/2) x^, angle = atan2(|a x b|, a . b). */
double oracle_dtheta(const double r[3], const double rp[3], double pitch) {
    double a[3] = {rp[0] + 0.5 * pitch - r[0], rp[1] - r[1], rp[2] - r[2]};
    double b[3] = {rp[0] - 0.5 * pitch - r[0], rp[1] - r[1], rp[2] - r[2]};
    double c[3];
    cross3(a, b, c);
    return atan2(norm3(c), dot3(a, b));
}

/* T(r, r'): the mask bit at the crossing of the ray with z = mask_z
 * (reading R8).  Exactly this op order, no FMA:
 *   t  = (z_m - z_r) / (z_d - z_r)
 *   px = t * x_d,  py = y_r + t * (y_d - y_r)
 *   m0 = c - (0.5 * n) * pitch
 *   u  = (p - m0) / pitch,  cell = floor(u),  outside the raster -> 0      */
int oracle_mask_cell(const oracle_desc *d, double y_r, double z_r, double x_d, double y_d,
                     int *cx, int *cy) {
    double t = (d->mask_z - z_r) / (d->det_z - z_r);
    double px = t * x_d;
    double py = y_r + t * (y_d - y_r);
    double m0x = d->mask_cx - (0.5 * d->mask_nx) * d->mask_pitch;
    double m0y = d->mask_cy - (0.5 * d->mask_ny) * d->mask_pitch;
    double ux = (px - m0x) / d->mask_pitch;
    double uy = (py - m0y) / d->mask_pitch;
    double fx = floor(ux), fy = floor(uy);
    *cx = -1;
    *cy = -1;
    if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)d->mask_nx && fy < (double)d->mask_ny)) return 0;
    *cx = (int)fx;
    *cy = (int)fy;
    return 1;
}
static double mask_T(const oracle_desc *d, double y_r, double z_r, double x_d, double y_d) {
    int cx, cy;
    if (!oracle_mask_cell(d, y_r, z_r, x_d, y_d, &cx, &cy)) return 0.0;
    return d->mask[(size_t)cx * d->mask_ny + cy] ? 1.0 : 0.0;
}

/* Scatter-angle interpolation: the nearest of the N
 * uniformly spaced angles theta_i = theta_min + i h, h = (theta_max -
 * theta_min) / (N - 1), i = 0 .. N-1 (reading R22).  Written as the plain
 * rounding rule i = floor((theta - theta_min) / h + 1/2), clamped. */
double oracle_sai_angle(const oracle_desc *d, double theta) {
    int N = d->sai_n_theta;
    if (N <= 1) return d->sai_theta_min;
    double h = (d->sai_theta_max - d->sai_theta_min) / (N - 1);
    double i = floor((theta - d->sai_theta_min) / h + 0.5);
    if (i < 0.0) i = 0.0;
    if (i > (double)(N - 1)) i = (double)(N - 1);
    return d->sai_theta_min + i * h;
}

/* Per-pair factors.  out[0..7] = P, sin(theta/2), cos(theta/2), theta,
 * dtheta, T, G_so, G_od.  P = C_E G_so G_od T dtheta (1+cos^2 theta) cos(theta/2) */
void oracle_pair(const oracle_desc *d, int iy, int iz, int ix, int jy, double out[8]) {
    double r[3] = {0.0, voxel_y(d, iy), voxel_z(d, iz)};
    double rp[3] = {det_x(d, ix), det_y(d, jy), d->det_z};
    double s[3] = {rp[0] - r[0], rp[1] - r[1], rp[2] - r[2]};
    double gso = oracle_G_so(r);
    double god = oracle_G_od(s);
    double th = oracle_theta(r, rp);
    double dth = oracle_dtheta(r, rp, d->det_pitch);
    double T = mask_T(d, r[1], r[2], rp[0], rp[1]);
    /* the angle at which the spectral factor S(theta, q) -- here its energy
     * form (1 + cos^2 th) cos(th/2) sum_k phi_k E_k Lambda(u_k - j) -- is
     * evaluated: theta itself, or under scatter-angle interpolation the
     * nearest tabulated angle (nearest neighbour) */
    double ts = th;
    if (d->sai_n_theta > 0) ts = oracle_sai_angle(d, th);
    double c = cos(ts);
    out[0] = d->scale * gso * god * T * dth * (1.0 + c * c) * cos(0.5 * ts);
    out[1] = sin(0.5 * ts);
    out[2] = cos(0.5 * ts);
    out[3] = th;
    out[4] = dth;
    out[5] = T;
    out[6] = gso;
    out[7] = god;
}

/* Lambda(x) = max(0, 1 - |x|): the linear-interpolation (hat) basis in q
 * (reading R5: f is zero outside the Q nodes).  f~(u) = sum_j f_j Lambda(u-j)
 * has at most two non-zero terms, j = floor(u) and floor(u) + 1. */
static double hat(double x) {
    double a = 1.0 - fabs(x);
    return a > 0.0 ? a : 0.0;
}

/* u_k for one pair: Bragg q = E sin(theta/2)/hc on the node scale */
static double node_coord(const oracle_desc *d, double E, double sh) {
    return (E * sh / HC_KEV_ANGSTROM - d->q_min) / q_step(d);
}

/* ---- forward: g = A f  (Alg. 1 structure) -------------
 * One output pixel at a time, summed over voxels r in a fixed order, then
 * over energies k; f is [ny][nz][nq]; out is 1 value (integrating) or ne. */
static void forward_pixel(const oracle_desc *d, const double *f, int ix, int jy, double *out) {
    int K = d->ne, Q = d->nq;
    int nout = d->energy_resolving ? K : 1;
    for (int k = 0; k < nout; k++) out[k] = 0.0;
    for (int iy = 0; iy < d->ny; iy++) {
        for (int iz = 0; iz < d->nz; iz++) {
            double fac[8];
            oracle_pair(d, iy, iz, ix, jy, fac);
            double P = fac[0], sh = fac[1];
            if (P == 0.0) continue; /* T = 0: the whole row of H is zero */
            const double *fr = f + ((size_t)iy * d->nz + iz) * Q;
            double W = 0.0; /* effective spectral factor */
            for (int k = 0; k < K; k++) {
                double u = node_coord(d, d->energy_kev[k], sh);
                double j0 = floor(u);
                double ft = 0.0;
                for (int jj = 0; jj < 2; jj++) {
                    double j = j0 + jj;
                    if (j >= 0.0 && j <= (double)(Q - 1)) ft += fr[(int)j] * hat(u - j);
                }
                double term = d->phi[k] * d->energy_kev[k] * ft;
                if (d->energy_resolving)
                    out[k] += P * term;
                else
                    W += term;
            }
            if (!d->energy_resolving) out[0] += P * W;
        }
    }
}

void oracle_forward(const oracle_desc *d, const double *f, double *g) {
    int nout = d->energy_resolving ? d->ne : 1;
    long npix = (long)d->det_nx * d->det_ny;
#pragma omp parallel for schedule(dynamic, 4)
    for (long p = 0; p < npix; p++)
        forward_pixel(d, f, (int)(p / d->det_ny), (int)(p % d->det_ny), g + p * nout);
}

/* forward restricted to a list of pixel indices (p = ix * det_ny + jy) */
void oracle_forward_pixels(const oracle_desc *d, const double *f, long n, const int64_t *pix,
                           double *out) {
    int nout = d->energy_resolving ? d->ne : 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (long i = 0; i < n; i++)
        forward_pixel(d, f, (int)(pix[i] / d->det_ny), (int)(pix[i] % d->det_ny), out + i * nout);
}

/* ---- backward: b = A^T w  (Alg. 3 structure) ----------
 * One voxel at a time; b[r, j] = sum_{r'} sum_k P phi_k E_k w Lambda(u_k - j) */
static void backward_voxel(const oracle_desc *d, const double *w, int iy, int iz, double *b) {
    int K = d->ne, Q = d->nq;
    for (int j = 0; j < Q; j++) b[j] = 0.0;
    for (int ix = 0; ix < d->det_nx; ix++) {
        for (int jy = 0; jy < d->det_ny; jy++) {
            double fac[8];
            oracle_pair(d, iy, iz, ix, jy, fac);
            double P = fac[0], sh = fac[1];
            if (P == 0.0) continue;
            long p = (long)ix * d->det_ny + jy;
            for (int k = 0; k < K; k++) {
                double wk = d->energy_resolving ? w[p * K + k] : w[p];
                double u = node_coord(d, d->energy_kev[k], sh);
                double j0 = floor(u);
                for (int jj = 0; jj < 2; jj++) {
                    double j = j0 + jj;
                    if (j >= 0.0 && j <= (double)(Q - 1))
                        b[(int)j] += P * d->phi[k] * d->energy_kev[k] * wk * hat(u - j);
                }
            }
        }
    }
}

void oracle_backward(const oracle_desc *d, const double *w, double *b) {
    long nvox = (long)d->ny * d->nz;
#pragma omp parallel for schedule(dynamic, 1)
    for (long v = 0; v < nvox; v++)
        backward_voxel(d, w, (int)(v / d->nz), (int)(v % d->nz), b + v * d->nq);
}

/* backward restricted to a list of voxel indices (v = iy * nz + iz) */
void oracle_backward_voxels(const oracle_desc *d, const double *w, long n, const int64_t *vox,
                            double *out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (long i = 0; i < n; i++)
        backward_voxel(d, w, (int)(vox[i] / d->nz), (int)(vox[i] % d->nz), out + i * d->nq);
}

/* backward restricted to a list of detector pixels (A_p^T w of Alg. 6,
 * PAPER.md:393-412): b[r, j] = sum_{r' in list} sum_k P phi_k E_k w Lambda(u_k - j) */
void oracle_backward_pixels(const oracle_desc *d, const double *w, long npix, const int64_t *pix, double *b) {
    long nvox = (long)d->ny * d->nz;
    int K = d->ne, Q = d->nq;
#pragma omp parallel for schedule(dynamic, 1)
    for (long v = 0; v < nvox; v++) {
        int iy = (int)(v / d->nz), iz = (int)(v % d->nz);
        double *bv = b + v * Q;
        for (int j = 0; j < Q; j++) bv[j] = 0.0;
        for (long i = 0; i < npix; i++) {
            int ix = (int)(pix[i] / d->det_ny), jy = (int)(pix[i] % d->det_ny);
            double fac[8];
            oracle_pair(d, iy, iz, ix, jy, fac);
            double P = fac[0], sh = fac[1];
            if (P == 0.0) continue;
            long p = pix[i];
            for (int k = 0; k < K; k++) {
                double wk = d->energy_resolving ? w[p * K + k] : w[p];
                double u = node_coord(d, d->energy_kev[k], sh);
                double j0 = floor(u);
                for (int jj = 0; jj < 2; jj++) {
                    double j = j0 + jj;
                    if (j >= 0.0 && j <= (double)(Q - 1))
                        bv[(int)j] += P * d->phi[k] * d->energy_kev[k] * wk * hat(u - j);
                }
            }
        }
    }
}

/* ---- work accounting ---------------------------
 * counts[0] = pairs, counts[1] = open pairs (T = 1),
 * counts[2] = effective terms: open pairs x energies with -1 < u_k < Q.     */
void oracle_count_terms(const oracle_desc *d, long n, const int64_t *pix, int64_t counts[3]) {
    int64_t c0 = 0, c1 = 0, c2 = 0;
#pragma omp parallel for reduction(+ : c0, c1, c2) schedule(dynamic, 1)
    for (long i = 0; i < n; i++) {
        int ix = (int)(pix[i] / d->det_ny), jy = (int)(pix[i] % d->det_ny);
        for (int iy = 0; iy < d->ny; iy++)
            for (int iz = 0; iz < d->nz; iz++) {
                double fac[8];
                oracle_pair(d, iy, iz, ix, jy, fac);
                c0++;
                if (fac[5] == 0.0) continue;
                c1++;
                for (int k = 0; k < d->ne; k++) {
                    double u = node_coord(d, d->energy_kev[k], fac[1]);
                    if (u > -1.0 && u < (double)d->nq) c2++;
                }
            }
    }
    counts[0] = c0;
    counts[1] = c1;
    counts[2] = c2;
}
