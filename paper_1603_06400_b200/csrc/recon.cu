// recon.cu -- the fused elementwise kernels around the operators
// and the objective.
//
//   K4 ratio:   y_i / (l_i + r_i)                            Alg. 5
//   K5 update:  4-neighbour stencil -> chi1, chi2, chi3 -> positive root of
//               chi1 x^2 + chi2 x - chi3 = 0                Eq. f_update
//   loglik:     J = sum (z - y ln z) + beta R
// Reductions are two-level with a fixed block count and fixed order, in fp64,
// so cacsi_neg_loglik is deterministic.
#include "internal.h"

namespace cacsi {

namespace {

constexpr int RT = 256;          // threads per reduction / elementwise block
constexpr int RED_BLOCKS = 592;  // fixed partial count (4 x 148)

__device__ __forceinline__ float guarded_ratio(float y, float z) {
    // y/z; 0 where y = 0 and z = 0; y / 1e-12 where z = 0 < y (reading R14/SPEC.md:452)
    if (z > 0.0f) return y / z;
    return y > 0.0f ? y * 1e12f : 0.0f;
}

__global__ void k_ratio(const float *__restrict__ l, const float *__restrict__ y, const float *__restrict__ r,
                        float *__restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = guarded_ratio(y[i], l[i] + r[i]);
}

__device__ double block_sum(double v, double *sh) {
    const int tid = threadIdx.x;
    sh[tid] = v;
    __syncthreads();
    for (int s = RT / 2; s > 0; s >>= 1) {
        if (tid < s) sh[tid] += sh[tid + s];
        __syncthreads();
    }
    return sh[0];
}

// partial[blockIdx] = sum over this block's grid-stride share of L_i
__global__ void __launch_bounds__(RT) k_loglik_part(const float *__restrict__ l, const float *__restrict__ y,
                                                    const float *__restrict__ r, size_t n, double *partial) {
    __shared__ double sh[RT];
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)RT + threadIdx.x; i < n; i += (size_t)gridDim.x * RT) {
        const double z = (double)l[i] + (double)r[i];
        const double yy = y[i];
        acc += yy > 0.0 ? z - yy * log(z) : z;
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
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

// partial[blockIdx] = sum over elements j of sum_{k in N_j} psi(f_j - f_k)
__global__ void __launch_bounds__(RT) k_penalty_part(const Params p, const float *__restrict__ f, double delta,
                                                     double *partial) {
    __shared__ double sh[RT];
    const size_t n = (size_t)p.n_vox * p.nq;
    const size_t sz = p.nq, sy = (size_t)p.nz * p.nq;
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)RT + threadIdx.x; i < n; i += (size_t)gridDim.x * RT) {
        const int iy = (int)(i / sy), iz = (int)((i / sz) % p.nz);
        const double fj = f[i];
        double s = 0.0;
        if (iy > 0) s += pen_psi(fj - f[i - sy], delta);
        if (iy + 1 < p.ny) s += pen_psi(fj - f[i + sy], delta);
        if (iz > 0) s += pen_psi(fj - f[i - sz], delta);
        if (iz + 1 < p.nz) s += pen_psi(fj - f[i + sz], delta);
        acc += s;
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_loglik_final(const double *lpart, const double *rpart, int nb, float beta, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double L = 0.0, R = 0.0;
        for (int i = 0; i < nb; i++) L += lpart[i];
        for (int i = 0; i < nb; i++) R += rpart[i];
        *out = L + (double)beta * R;
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
__global__ void k_update(const Params p, const float *__restrict__ f_hat, const float *__restrict__ b1,
                         const float *__restrict__ b2, float beta, double delta, float *__restrict__ f_new) {
    // 32-bit index arithmetic (n_vox * nq < 2^31, checked at create): the 64-bit
    // divisions of the neighbour indexing dominated this kernel
    const unsigned n = (unsigned)p.n_vox * (unsigned)p.nq;
    const unsigned sz = (unsigned)p.nq, sy = (unsigned)p.nz * (unsigned)p.nq;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned vq = i / sz;  // voxel index iy * nz + iz
        const int iy = (int)(vq / (unsigned)p.nz), iz = (int)(vq - (unsigned)iy * (unsigned)p.nz);
        const double fj = f_hat[i];
        double som = 0.0, spd = 0.0, pd, om;
        if (iy > 0) { pen_dot_omega(fj - f_hat[i - sy], delta, pd, om); som += om; spd += pd; }
        if (iy + 1 < p.ny) { pen_dot_omega(fj - f_hat[i + sy], delta, pd, om); som += om; spd += pd; }
        if (iz > 0) { pen_dot_omega(fj - f_hat[i - sz], delta, pd, om); som += om; spd += pd; }
        if (iz + 1 < p.nz) { pen_dot_omega(fj - f_hat[i + sz], delta, pd, om); som += om; spd += pd; }
        const double bt = beta;
        const double b34 = 4.0 * som, b56 = 2.0 * spd;
        const double chi1 = bt * b34;
        const double chi2 = (double)b1[i] + bt * (-fj * b34 + b56);
        const double chi3 = fj * (double)b2[i];
        const double sq = sqrt(fmax(chi2 * chi2 + 4.0 * chi1 * chi3, 0.0));
        double x;
        if (chi2 > 0.0)
            x = 2.0 * chi3 / (chi2 + sq);
        else if (chi1 > 0.0)
            x = (-chi2 + sq) / (2.0 * chi1);
        else
            x = fj;
        f_new[i] = (float)x;
    }
}

int grid_for(size_t n) { return (int)min((n + RT - 1) / RT, (size_t)RED_BLOCKS * 4); }

}  // namespace

size_t recon_workspace_bytes(const cacsi_geometry *g) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return al(g->n_detout * sizeof(float)) + 2 * al(g->n_obj * sizeof(float)) + al(2 * RED_BLOCKS * sizeof(double));
}

cudaError_t launch_ratio(const cacsi_geometry *g, const float *l, const float *y, const float *r, float *ratio,
                         double *, int, cudaStream_t s, int *launches) {
    {
        KScope kt_(g, s, "k_ratio");
        k_ratio<<<grid_for(g->n_detout), RT, 0, s>>>(l, y, r, ratio, g->n_detout);
    }
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_update(const cacsi_geometry *g, const float *f_hat, const float *b1, const float *b2, float beta,
                          double delta, float *f_new, cudaStream_t s, int *launches) {
    {
        KScope kt_(g, s, "k_update");
        k_update<<<grid_for(g->n_obj), RT, 0, s>>>(g->p, f_hat, b1, b2, beta, delta, f_new);
    }
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_loglik(const cacsi_geometry *g, const float *l, const float *y, const float *r, const float *f,
                          float beta, double delta, double *partials, double *out, cudaStream_t s, int *launches) {
    k_loglik_part<<<RED_BLOCKS, RT, 0, s>>>(l, y, r, g->n_detout, partials);
    k_penalty_part<<<RED_BLOCKS, RT, 0, s>>>(g->p, f, delta, partials + RED_BLOCKS);
    k_loglik_final<<<1, 32, 0, s>>>(partials, partials + RED_BLOCKS, RED_BLOCKS, beta, out);
    *launches += 3;
    return cudaGetLastError();
}

}  // namespace cacsi
