// elementwise.cuh -- the per-element arithmetic of the iteration, shared by the
// stand-alone kernels (recon.cu: k_ratio, k_update) and the fused epilogues of the
// operators' final partial sums (esai.cu: cacsi_iterate's forward -> ratio and
// backward -> update), so the fused and unfused paths compute the same bits.
// Included inside namespace cacsi::{anonymous}.
#pragma once

__device__ __forceinline__ float guarded_ratio(float y, float z) {
    // y/z; 0 where y = 0 and z = 0; y / 1e-12 where z = 0 < y (reading R14/SPEC.md:452)
    if (z > 0.0f) return y / z;
    return y > 0.0f ? y * 1e12f : 0.0f;
}

// Edge-preserving potential (Eq. 7): psi, psi_dot and the
// surrogate curvature omega = psi_dot / x.  delta <= 0
// selects the quadratic psi(x) = x^2/2 (reading R13), else Huber (R21).
__device__ __forceinline__ double pen_psi(double x, double delta) {
    const double ax = fabs(x);
    return (delta <= 0.0 || ax <= delta) ? 0.5 * x * x : delta * ax - 0.5 * delta * delta;
}
__device__ __forceinline__ void pen_dot_omega(double x, double delta, double &pd, double &om) {
    const double ax = fabs(x);
    if (delta <= 0.0 || ax <= delta) {
        pd = x;
        om = 1.0;
    } else {
        pd = x > 0.0 ? delta : -delta;
        om = delta / ax;
    }
}

// Eq. f_update, 4-connected (y, z) neighbours, w = 1,
// symmetric (N^b = N, so b4 = b3 and b6 = b5):
//   b3 = 2 sum_k omega(f^_j - f^_k),  b5 = sum_k psi_dot(f^_j - f^_k)
//   chi1 = beta (b3 + b4),  chi2 = b1 + beta (-f^ (b3 + b4) + b5 + b6),  chi3 = f^ b2
// (quadratic psi: chi1 = 4 beta |N_j|, chi2 = b1 - 2 beta (|N_j| f^ + sum_k f^_k)).
// root = 2 chi3 / (chi2 + sqrt(D)) if chi2 > 0 (same number as the paper's
// (-chi2 + sqrt D)/(2 chi1), no cancellation), else (-chi2 + sqrt D)/(2 chi1);
// chi1 = 0 and chi2 <= 0 (voxel never seen): keep f^ (reading R14).
// The root of one element from its loaded neighbourhood (f^_j, its <= 4 neighbours with
// validity flags, b1_j, b2_j): the arithmetic of update_at, shared with update_at4.
__device__ __forceinline__ float update_core(double fj, const float (&nb)[4], const bool (&ok)[4], float b1i,
                                            float b2i, float beta, double delta) {
    double som = 0.0, spd = 0.0, pd, om;
#pragma unroll
    for (int t = 0; t < 4; t++)
        if (ok[t]) { pen_dot_omega(fj - nb[t], delta, pd, om); som += om; spd += pd; }
    const double bt = beta;
    const double b34 = 4.0 * som, b56 = 2.0 * spd;
    const double chi1 = bt * b34;
    const double chi2 = (double)b1i + bt * (-fj * b34 + b56);
    const double chi3 = fj * (double)b2i;
    const double sq = sqrt(fmax(chi2 * chi2 + 4.0 * chi1 * chi3, 0.0));
    double x;
    if (chi2 > 0.0)
        x = 2.0 * chi3 / (chi2 + sq);
    else if (chi1 > 0.0)
        x = (-chi2 + sq) / (2.0 * chi1);
    else
        x = fj;
    return (float)x;
}

// Four consecutive elements i0 .. i0 + 3 of one voxel (nq % 4 == 0, i0 % 4 == 0): the
// neighbourhood by 16-byte loads, then update_core per element -- the same bits as four
// update_at calls (the sum over neighbours runs in the same order).
__device__ __forceinline__ float4 update_at4(const Params &p, const float *__restrict__ f_hat,
                                            const float *__restrict__ b1, float4 b2, float beta, double delta,
                                            unsigned i0) {
    const unsigned sz = (unsigned)p.nq, sy = (unsigned)p.nz * (unsigned)p.nq;
    const unsigned vq = i0 / sz;
    const int iy = (int)(vq / (unsigned)p.nz), iz = (int)(vq - (unsigned)iy * (unsigned)p.nz);
    const bool ok[4] = {iy > 0, iy + 1 < p.ny, iz > 0, iz + 1 < p.nz};
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 c = *(const float4 *)(f_hat + i0);
    const float4 n0 = ok[0] ? *(const float4 *)(f_hat + i0 - sy) : z4;
    const float4 n1 = ok[1] ? *(const float4 *)(f_hat + i0 + sy) : z4;
    const float4 n2 = ok[2] ? *(const float4 *)(f_hat + i0 - sz) : z4;
    const float4 n3 = ok[3] ? *(const float4 *)(f_hat + i0 + sz) : z4;
    const float4 bb = *(const float4 *)(b1 + i0);
    const float cc[4] = {c.x, c.y, c.z, c.w}, q0[4] = {n0.x, n0.y, n0.z, n0.w}, q1[4] = {n1.x, n1.y, n1.z, n1.w},
                q2[4] = {n2.x, n2.y, n2.z, n2.w}, q3[4] = {n3.x, n3.y, n3.z, n3.w}, b1v[4] = {bb.x, bb.y, bb.z, bb.w},
                b2v[4] = {b2.x, b2.y, b2.z, b2.w};
    float r[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const float nb[4] = {q0[e], q1[e], q2[e], q3[e]};
        r[e] = update_core((double)cc[e], nb, ok, b1v[e], b2v[e], beta, delta);
    }
    return make_float4(r[0], r[1], r[2], r[3]);
}

__device__ __forceinline__ float update_at(const Params &p, const float *__restrict__ f_hat,
                                          const float *__restrict__ b1, float b2i, float beta, double delta,
                                          unsigned i) {
    // 32-bit index arithmetic (n_vox * nq < 2^31, checked at create): the 64-bit
    // divisions of the neighbour indexing dominated this kernel
    const unsigned sz = (unsigned)p.nq, sy = (unsigned)p.nz * (unsigned)p.nq;
    const unsigned vq = i / sz;  // voxel index iy * nz + iz
    const int iy = (int)(vq / (unsigned)p.nz), iz = (int)(vq - (unsigned)iy * (unsigned)p.nz);
    const bool ok[4] = {iy > 0, iy + 1 < p.ny, iz > 0, iz + 1 < p.nz};
    const float nb[4] = {ok[0] ? f_hat[i - sy] : 0.0f, ok[1] ? f_hat[i + sy] : 0.0f, ok[2] ? f_hat[i - sz] : 0.0f,
                         ok[3] ? f_hat[i + sz] : 0.0f};
    return update_core((double)f_hat[i], nb, ok, b1[i], b2i, beta, delta);
}
