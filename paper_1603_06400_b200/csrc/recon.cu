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

#include "elementwise.cuh"

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

__global__ void k_update(const Params p, const float *__restrict__ f_hat, const float *__restrict__ b1,
                         const float *__restrict__ b2, float beta, double delta, float *__restrict__ f_new) {
    const unsigned n = (unsigned)p.n_vox * (unsigned)p.nq;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        f_new[i] = update_at(p, f_hat, b1, b2[i], beta, delta, i);
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
