/*
 * cacsi.h -- C ABI of the B200-native forward/backward operators of fan-beam
 * coded-aperture X-ray coherent-scatter imaging (arXiv 1603.06400,
 * "Joint System and Algorithm Design for Computationally Efficient Fan Beam
 * Coded Aperture X-ray Coherent Scatter Imaging").
 *
 * The problem: an unknown object scatter density
 * f(r, q) >= 0 over B fan-slice pixels r = (y, z) and Q momentum-transfer
 * nodes q (J = B x Q unknowns), detector counts y with a known
 * background r (Eq. poisson_model), the system matrix
 * H = A of Eq. (1), and the penalized Poisson objective
 * J = L + beta R minimised over f >= 0 by the EM-type iteration of Alg. 5
 * (PAPER.md:363-377).
 *
 * Frame (config frame): source at the origin, beam along +z, fan
 * in the x = 0 plane.  Voxel r = (0, y, z); detector pixel r' = (x, y, det_z)
 * with rows along x (out of fan) and columns along y; the secondary mask lies
 * in the plane z = mask_z.  Lengths in mm, q in 1/Angstrom, E in keV.
 *
 * Operator:
 *   A[r'; (r, j)]      = P(r, r') sum_k phi_k E_k Lambda(u_k - j)   (energy-integrating)
 *   A[(r', k); (r, j)] = P(r, r') phi_k E_k Lambda(u_k - j)         (energy-resolving)
 *   P = scale * G_so(r) G_od(s) T(r, r') dtheta (1 + cos^2 theta) cos(theta / 2)
 *   u_k = (E_k sin(theta/2) / hc - q_min) / dq,  hc = 12.3984193 keV A,
 *   Lambda(x) = max(0, 1 - |x|)  (linear interpolation in q, zero outside).
 *
 * Memory layouts (all row-major, fp32, caller-owned DEVICE buffers unless a
 * function name ends in _host):
 *   f, b  : [ny][nz][nq]                 (object / backprojection)
 *   g, w  : [det_nx][det_ny]             (energy_resolving = 0)
 *           [det_nx][det_ny][ne]         (energy_resolving = 1)
 *   y, r  : same shape as g              (counts, background)
 *
 * Conventions:
 *   - Every call is asynchronous and ordered on `stream` (a cudaStream_t
 *     passed as void*, NULL = legacy default stream) unless stated otherwise.
 *   - Outputs are OVERWRITTEN, never accumulated into.
 *   - A handle is immutable after create.  Calls on one handle may run
 *     concurrently on different streams only if each uses its own workspace;
 *     the operators' internal scratch comes from the stream-ordered allocator
 *     (cudaMallocAsync) on the caller's stream.
 *   - Run-time NaN / negative inputs are not checked (documented).
 *   - There is no CPU fallback: without a usable sm_100 device every call
 *     that launches work returns CACSI_ERR_CUDA.
 */
#ifndef CACSI_H
#define CACSI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CACSI_API __attribute__((visibility("default")))
#else
#define CACSI_API
#endif

typedef enum {
    CACSI_OK = 0,
    CACSI_ERR_NULL = 1,    /* a required pointer was NULL                       */
    CACSI_ERR_INVALID = 2, /* descriptor / argument violates a documented rule  */
    CACSI_ERR_CUDA = 3,    /* CUDA launch / runtime failure, or no sm_100 device */
    CACSI_ERR_NOMEM = 4    /* device or host allocation failed                  */
} cacsi_status;

typedef struct cacsi_geometry cacsi_geometry; /* opaque, immutable after create */

/* Geometry descriptor.  Read only during cacsi_geometry_create (all arrays are
 * copied).  Validation (-> CACSI_ERR_INVALID):
 *   ny, nz, ne, mask_nx, mask_ny, det_nx, det_ny >= 1; 2 <= nq <= 400; ne <= 256
 *       (shared-memory table limits);
 *   y_min < y_max, 0 < z_min < z_max < mask_z < det_z   (plane order, so that
 *       every scatter vector has s_z > 0 and crosses the mask plane);
 *   q_min < q_max; mask_pitch > 0; det_pitch > 0; scale > 0 and finite;
 *   energy_kev strictly increasing and > 0; phi >= 0; mask bytes in {0, 1};
 *   energy_resolving in {0, 1}; sai_n_theta >= 0 (see below).                */
typedef struct {
    /* object slice: voxel centres y_i = y_min + (i + 1/2) (y_max - y_min)/ny,
     * likewise z ("B spatial bins")                            */
    int32_t ny, nz;
    double y_min, y_max, z_min, z_max;
    /* momentum-transfer nodes q_j = q_min + j (q_max - q_min)/(nq - 1)
     * ("evenly spaced momentum transfer bins")                */
    int32_t nq;
    double q_min, q_max;
    /* source spectrum sampled at ne energies E_k (keV, increasing) with
     * weights phi_k >= 0 (the bin integral of Phi(E))        */
    int32_t ne;
    const double *energy_kev; /* host, [ne], copied */
    const double *phi;        /* host, [ne], copied */
    /* secondary mask: binary image [mask_nx][mask_ny] (1 = open) in the plane
     * z = mask_z; cell (i, j) covers x in [m0x + i p, m0x + (i+1) p) with
     * m0x = mask_cx - (0.5 mask_nx) p, likewise y            */
    int32_t mask_nx, mask_ny;
    double mask_z, mask_pitch, mask_cx, mask_cy;
    const uint8_t *mask; /* host, [mask_nx][mask_ny], copied */
    /* detector: pixel centres x_i = det_cx + ((i + 1/2) - det_nx/2) det_pitch,
     * likewise y; plane z = det_z                            */
    int32_t det_nx, det_ny;
    double det_z, det_pitch, det_cx, det_cy;
    int32_t energy_resolving; /* 0: g[dx][dy]; 1: g[dx][dy][ne]             */
    double scale;             /* C_E, the calibration constant */
    /* Scatter-angle interpolation,
     * the paper's approximate operator: sai_n_theta > 0 evaluates each pair's
     * spectral-angular factor (1 + cos^2 t) cos(t/2) sum_k phi_k E_k
     * Lambda(E_k sin(t/2)/hc - q) at the NEAREST of sai_n_theta angles
     * t_i = sai_theta_min + i h, h = (max - min)/(n - 1) (reading R22;
     * G_so, G_od, T, dtheta stay exact per pair).  0 = the exact operator.
     * Energy-integrating handles only; requires 0 <= min < max <= pi when
     * n >= 2 (else CACSI_ERR_INVALID).                                      */
    int32_t sai_n_theta;
    double sai_theta_min, sai_theta_max;
} cacsi_geometry_desc;

/* Validate `desc`, precompute the per-voxel / per-pixel / per-energy tables
 * in fp64 (the offline part of the online/offline
 * trade-off), bit-pack the mask and upload everything to `device`.
 * Synchronous.  On success *out owns the device tables.  Every call on the
 * handle runs on `device` and restores the caller's current device on return.
 * Errors: CACSI_ERR_NULL (desc, out or a desc array NULL), CACSI_ERR_INVALID
 * (including ny nz nq >= 2^31 or det_nx det_ny ne >= 2^31: 32-bit element
 * indexing), CACSI_ERR_CUDA (no such device / not sm_100), CACSI_ERR_NOMEM. */
CACSI_API cacsi_status cacsi_geometry_create(const cacsi_geometry_desc *desc, int device, cacsi_geometry **out);

/* As cacsi_geometry_create, with kernel-variant options: NULL / "" = the
 * defaults, else "key=value[,key=value...]" (integer values, no spaces).
 * Every option selects among kernels that compute the same operator (A/B
 * measurements and independent cross-checks; DESIGN.md 4.5 lists them).
 * Create-time keys: pair_cache (1; 0 = recompute the pair geometry per call),
 * ts (1; 0 = no translation-symmetric on-the-fly forward), direct (0; 1 = the
 * per-term kernels instead of ESAI), pc_plain (0; 1 = list-ordered unpadded
 * pair cache), pc_segwin (1), pc_q8 (2: 8-byte records, P rounded to 28 bits
 * carrying 4 pixel-offset bits; 1: 10-bit tau; 0: 10-byte records), pc_win
 * (128), pcv_budget_kb (200), er_cache (0; 1 = the
 * energy-resolving operators from a pair cache), er_vcache (1:
 * the energy-resolving backward's voxel-major open-pair records, 12 B each),
 * er_fcache (1: the energy-resolving forward's pixel-major open-pair records,
 * 16 B each; both built only with 8 GB of device memory to spare, DESIGN.md
 * 4.3).  Per-call keys (also
 * settable with cacsi_set_option): wgemm (0 A-resident, 1 CTA-pair, 2 per-tile),
 * wgemm_pack, b2gemm_tiles, pc_fwd_list, pcv_items, pcv_pf, pcv_u, pc_bwd_flat,
 * pcb_pf, subset_bwd_mask, er_bwd_dense, graphs (1; 0 = cacsi_osem by stream
 * launches), gemm16 (1: the ESAI contractions on a two-term fp16 split at the
 * fp16 tensor-core rate; 0 = 3xTF32), b2_splits (16: split-K count of the fp16
 * b2 GEMM), w_tmast / b2_tmast (1: the fp16 GEMMs' epilogues store by TMA
 * tensor stores; 0 = per-lane stores), b2_rings (1: A / B ring depths of
 * the fp16 b2 GEMM, 0 = 3 / 3, 1 = 4 / 2, 2 = 2 / 4), er_fwd_rec (1: the
 * record-fed energy-resolving forward; 0 = mask tests and pair geometry per
 * call), er_fwd_win (6: its lanes' voxel window), er_fwd_lane, er_fwd_reg,
 * er_bwd_fx, er_vcache_use (1).  An unknown key or out-of-range value
 * -> CACSI_ERR_INVALID.
 * The library never reads the process environment.                          */
CACSI_API cacsi_status cacsi_geometry_create_ex(const cacsi_geometry_desc *desc, int device, const char *options,
                                                cacsi_geometry **out);

/* Change a per-call option of a handle (the keys above): later calls launch the
 * selected kernel variant.  Not synchronised with calls running concurrently on
 * the handle.  Errors: CACSI_ERR_NULL; CACSI_ERR_INVALID (unknown key, a
 * create-time key, or a value out of range).                                */
CACSI_API cacsi_status cacsi_set_option(cacsi_geometry *geom, const char *key, int64_t value);

/* Free the handle and its device tables (synchronises the device).  NULL ok. */
CACSI_API void cacsi_geometry_destroy(cacsi_geometry *geom);

/* Bytes of device workspace cacsi_iterate / cacsi_neg_loglik need (the caller
 * allocates it; 256-byte aligned).  0 for a NULL handle.                    */
CACSI_API size_t cacsi_workspace_bytes(const cacsi_geometry *geom);

/* Sizes implied by the handle (elements, not bytes).  0 for NULL.           */
CACSI_API size_t cacsi_object_size(const cacsi_geometry *geom);   /* ny*nz*nq            */
CACSI_API size_t cacsi_detector_size(const cacsi_geometry *geom); /* det_nx*det_ny[*ne]  */

/* Forward model g = A f  (Eq. 1; Alg. 1 computes the same sum,
 * PAPER.md:129-153).  f: device [ny][nz][nq]; g: device, detector shape.
 * Errors: CACSI_ERR_NULL, CACSI_ERR_CUDA, CACSI_ERR_NOMEM.                   */
CACSI_API cacsi_status cacsi_forward(const cacsi_geometry *geom, const float *f, float *g, void *stream);

/* Backward (adjoint) model b = A^T w  (Alg. 3).
 * w: device, detector shape; b: device [ny][nz][nq].                        */
CACSI_API cacsi_status cacsi_backward(const cacsi_geometry *geom, const float *w, float *b, void *stream);

/* Penalized negative log-likelihood J(f) = L(f) + beta R(f)
 * with L = sum_i (l_i + r_i) - y_i ln(l_i + r_i),
 * l = A f (the constant sum ln y_i! is omitted), and
 * R = sum_j sum_{k in N_j} (f_j - f_k)^2 / 2 over the 4-connected (y, z)
 * neighbours within one q node (each unordered pair counted twice, as in
 * Eq. 7).  Writes ONE double to DEVICE memory *out_dev (stream-ordered,
 * deterministic).  ws: device workspace of cacsi_workspace_bytes() bytes.   */
CACSI_API cacsi_status cacsi_neg_loglik(const cacsi_geometry *geom, const float *f, const float *y, const float *r,
                              float beta, double *out_dev, void *ws, void *stream);

/* n_iter iterations of the EM-type algorithm (Alg. 5),
 * updating f IN PLACE:
 *   z = A f + r;  b2 = A^T (y ./ z);  f <- Eq. f_update
 * with the quadratic potential psi(x) = x^2/2, 4-connected (y, z) neighbours,
 * unit weights.  b1 = A^T 1 is supplied by the caller (computed once,
 * PAPER.md:370).  Ratio guard: y/z = 0 where y = 0 and z = 0, y / 1e-12
 * where z = 0 < y.  f must be >= 0 on entry and stays >= 0.
 * ws: device workspace of cacsi_workspace_bytes() bytes.
 * On ESAI handles the iteration runs as two operator calls whose final
 * partial sums carry the elementwise steps (the forward's writes y ./ z and
 * max |y ./ z|, the backward's writes the update) -- the same bits as
 * cacsi_forward, cacsi_ratio, cacsi_backward, cacsi_update in turn.  The
 * iterates alternate between f and the workspace; an odd n_iter ends with one
 * device copy into f.                                                       */
CACSI_API cacsi_status cacsi_iterate(const cacsi_geometry *geom, float *f, const float *y, const float *r,
                           const float *b1, float beta, int32_t n_iter, void *ws, void *stream);

/* The two fused elementwise steps of Alg. 5, exposed for stage timing (the
 * same kernels cacsi_iterate runs):
 *   cacsi_ratio : ratio = y ./ (l + r) with the guard above (K4); detector
 *                 shape; ratio may alias l.
 *   cacsi_update: f_new = Eq. f_update(f_hat, b1, b2, beta) (K5); object
 *                 shape; f_new must not alias f_hat.                        */
CACSI_API cacsi_status cacsi_ratio(const cacsi_geometry *geom, const float *l, const float *y, const float *r,
                                   float *ratio, void *stream);
CACSI_API cacsi_status cacsi_update(const cacsi_geometry *geom, const float *f_hat, const float *b1, const float *b2,
                                    float beta, float *f_new, void *stream);

/* End-to-end variants on HOST buffers (pageable or pinned): copy the inputs
 * to device scratch owned by the handle, run the device call, copy the output
 * back, and synchronise `stream` before returning.  Same shapes as above.
 * Not re-entrant on one handle (they share the handle's staging buffers).
 * cacsi_iterate_host uploads f, y, r, b1 (in that order) on a side stream the
 * handle owns (created on first use, after waiting for earlier work on
 * `stream`): on ESAI handles f goes in four row chunks and the forward's
 * tensor-core contraction starts on each chunk as it lands; y, r are waited
 * for only before the ratio, b1 only before the update (other handles: f is
 * uploaded whole on `stream` first).                                        */
CACSI_API cacsi_status cacsi_forward_host(const cacsi_geometry *geom, const float *f_host, float *g_host, void *stream);
CACSI_API cacsi_status cacsi_backward_host(const cacsi_geometry *geom, const float *w_host, float *b_host, void *stream);
CACSI_API cacsi_status cacsi_iterate_host(const cacsi_geometry *geom, float *f_host, const float *y_host,
                                const float *r_host, const float *b1_host, float beta, int32_t n_iter,
                                void *stream);

/* ---- Edge-preserving penalty ---------------------
 * psi_delta of Eq. 7 with the separable quadratic
 * surrogate of PAPER.md:686-698 (curvature omega = psi_dot / x).
 *   CACSI_PENALTY_QUADRATIC: psi(x) = x^2 / 2 (delta ignored) -- the default
 *                            of the non-_ex calls (reading R13);
 *   CACSI_PENALTY_HUBER:     psi(x) = x^2/2 for |x| <= delta,
 *                            delta |x| - delta^2/2 otherwise; delta > 0 finite
 *                            (reading R21).
 * A NULL descriptor means quadratic; an invalid one -> CACSI_ERR_INVALID.  */
typedef enum { CACSI_PENALTY_QUADRATIC = 0, CACSI_PENALTY_HUBER = 1 } cacsi_penalty_kind;
typedef struct {
    int32_t kind;  /* cacsi_penalty_kind */
    double delta;  /* Huber scale (> 0), same units as f */
} cacsi_penalty;

/* As cacsi_update / cacsi_iterate / cacsi_neg_loglik with the potential `pen`
 * (R = sum_j sum_{k in N_j} psi(f_j - f_k), each unordered pair twice).     */
CACSI_API cacsi_status cacsi_update_ex(const cacsi_geometry *geom, const float *f_hat, const float *b1,
                                       const float *b2, float beta, const cacsi_penalty *pen, float *f_new,
                                       void *stream);
CACSI_API cacsi_status cacsi_iterate_ex(const cacsi_geometry *geom, float *f, const float *y, const float *r,
                                        const float *b1, float beta, const cacsi_penalty *pen, int32_t n_iter,
                                        void *ws, void *stream);
CACSI_API cacsi_status cacsi_neg_loglik_ex(const cacsi_geometry *geom, const float *f, const float *y,
                                           const float *r, float beta, const cacsi_penalty *pen, double *out_dev,
                                           void *ws, void *stream);

/* ---- Ordered subsets (Alg. 6) ----
 * cacsi_symmetric_subsets: the symmetry-preserving partition of the detector
 * (Fig. 6): rows i (the paper's vertical index, config x)
 * grouped as m:rho_x:M/2 with their up-down mirrors, columns j (y) as
 * n:rho_y:N with their left-right mirrors; subset id = m (rho_y/2) + n
 * (0-based, row-group-major), P = rho_x rho_y / 2 equal subsets.  HOST only
 * (no device work): subset_of_pixel is a caller-owned host array
 * [det_nx * det_ny].  Errors: CACSI_ERR_NULL; CACSI_ERR_INVALID unless
 * det_nx is even, rho_x >= 1 divides det_nx/2, rho_y >= 2 is even and
 * divides det_ny.                                                           */
CACSI_API cacsi_status cacsi_symmetric_subsets(int32_t det_nx, int32_t det_ny, int32_t rho_x, int32_t rho_y,
                                               int32_t *subset_of_pixel, int32_t *n_subsets);

/* Subset-restricted operators of Alg. 6: `pixels` is a DEVICE list of
 * n_pixels distinct detector pixel indices (ix * det_ny + jy).
 *   cacsi_forward_subset : g = A_p f on the listed pixels, 0 elsewhere
 *                          (detector shape, overwritten);
 *   cacsi_backward_subset: b = A_p^T w = A^T (w restricted to the list).
 * Energy-integrating (ESAI) handles run only the listed pixels' pairs; other
 * handles run the full operator and restrict it.  Errors: CACSI_ERR_NULL,
 * CACSI_ERR_INVALID (n_pixels < 0 or > det_nx * det_ny), CACSI_ERR_CUDA.  */
CACSI_API cacsi_status cacsi_forward_subset(const cacsi_geometry *geom, const float *f, const int32_t *pixels,
                                            int32_t n_pixels, float *g, void *stream);
CACSI_API cacsi_status cacsi_backward_subset(const cacsi_geometry *geom, const float *w, const int32_t *pixels,
                                             int32_t n_pixels, float *b, void *stream);

/* n_outer outer iterations of Alg. 6, updating f in place.  Subset p owns the
 * device pixels[offsets[p] .. offsets[p+1]) (offsets: HOST [n_subsets + 1],
 * offsets[0] = 0); b1_subsets: DEVICE [n_subsets][ny][nz][nq] with
 * b1_p = A_p^T 1 (cacsi_backward_subset of ones, computed once by the
 * caller).  Each sub-iteration: z_p = A_p f + r, b2_p = A_p^T (y ./ z_p),
 * f <- Eq. f_update(f, b1_p, b2_p) with penalty weight beta / n_subsets
 * (reading R20: the subset data term stands for 1/P of L).  Subsets are swept
 * in index order.  ws: cacsi_workspace_bytes() bytes.
 * One outer iteration is captured into a CUDA graph on first use and replayed;
 * the graph is cached in the handle (one per handle, guarded by a mutex) and
 * re-captured when any argument (pointers, offsets, beta, penalty) changes.
 * Option graphs=0 or cacsi_set_timing(1) selects plain stream launches.    */
CACSI_API cacsi_status cacsi_osem(const cacsi_geometry *geom, float *f, const float *y, const float *r,
                                  const float *b1_subsets, const int32_t *pixels, const int32_t *offsets,
                                  int32_t n_subsets, float beta, const cacsi_penalty *pen, int32_t n_outer,
                                  void *ws, void *stream);

/* Number of kernels the last successful device call on this handle enqueued
 * (for the bench's gpu_launches count).                                     */
CACSI_API int32_t cacsi_last_launch_count(const cacsi_geometry *geom);

/* Per-kernel timing: when enabled, every kernel the handle launches is
 * bracketed by a CUDA event pair on the launching stream.
 * cacsi_kernel_times synchronises those events, returns the number of distinct
 * kernel names (<= max) and fills names[i] (static strings), total_ms[i] and
 * launches[i] accumulated since the previous query, then resets.            */
CACSI_API cacsi_status cacsi_set_timing(const cacsi_geometry *geom, int32_t enable);
CACSI_API int32_t cacsi_kernel_times(const cacsi_geometry *geom, int32_t max, const char **names, double *total_ms,
                                     int32_t *launches);

/* Integer facts about a handle: "esai_breakpoints" (0 if the per-term
 * kernels are used), "esai_max_window", "esai_lut_cells",
 * "esai_lut_slow_cells", "esai_ldw" (row stride of the breakpoint tables),
 * "pair_cache_records" (open pairs held in the pair cache, 0 if not built),
 * "pair_cache_record_bytes" (bytes per record: P, packed (b, tau), pixel q),
 * "pair_cache_tau_bits" (fraction bits of the stored tau),
 * "pair_cache_padding_closed" (1: every padding record's pixel is closed for
 * its voxel, so the forward adds its zero in place),
 * "pair_cache_fwd_row_blocks" (detector row blocks of the voxel-major
 * forward; 0 = the per-list forward runs),
 * "ts_rho" (0 = no translation symmetry), "energy_resolving".  -1 for an
 * unknown key or NULL.
 * The pair cache is built at create when it fits in half of the
 * free device memory; the option pair_cache=0 disables it (the operators then
 * recompute the pair geometry per call).                                    */
CACSI_API int64_t cacsi_query(const cacsi_geometry *geom, const char *key);

/* Static description of a status code (never NULL). */
CACSI_API const char *cacsi_status_string(cacsi_status status);

#ifdef __cplusplus
}
#endif
#endif /* CACSI_H */
