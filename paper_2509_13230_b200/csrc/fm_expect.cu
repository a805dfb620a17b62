// fm_expect.cu -- closed-form expectations under the model: per node i, over
// j != i, the exact fp64 sums
//     k_i  = sum_j p_ij,                 kvar_i = sum_j p_ij (1 - p_ij)           (Eq. 4)
//     s_i  = sum_j p_ij / (1 - t_ij),    svar_i = sum_j Var[w_ij]                 (Eq. 3-5)
// with p_ij = X/(1+X), X = x_i x_j (UBCM) or p_ij = z/((1-t)+z), z = (x_i y_i)(x_j y_j),
// t = y_i y_j (ECM), and, for an ECM edge, w ~ Geometric on {1, 2, ...} with ratio t: E[w] =
// p/(1-t), E[w^2] = p(1+t)/(1-t)^2.  These are what the statistical gates on the sampler's output
// compare against (per-node mean degree / strength within 5 sigma, Bonferroni over all nodes).
//
// O(N * n_nodes) pair evaluations: one thread per listed node, the j loop over shared-memory tiles
// of (x_j, y_j) (every thread of a block reads the same j: broadcast), compensated (Kahan-Babuska)
// summation per accumulator, so the sums are exact to a few ulp regardless of N.
#include "fm_internal.cuh"

namespace fm {
namespace {

constexpr int kExpThreads = 256;
constexpr int kExpTile = 2048;

struct Kahan {
    double s = 0.0, c = 0.0;
    __device__ __forceinline__ void add(double v)
    {
        const double t = __dadd_rn(s, v);
        // Neumaier: the rounding error of s + v, whichever operand is larger
        c = __dadd_rn(c, fabs(s) >= fabs(v) ? __dadd_rn(__dsub_rn(s, t), v) : __dadd_rn(__dsub_rn(v, t), s));
        s = t;
    }
    __device__ __forceinline__ double get() const { return __dadd_rn(s, c); }
};

template <bool kEcm>
__global__ void __launch_bounds__(kExpThreads) k_expected(int64_t n, const double *__restrict__ x,
                                                          const double *__restrict__ y,
                                                          const int32_t *__restrict__ nodes, int64_t n_nodes,
                                                          double *__restrict__ k, double *__restrict__ kvar,
                                                          double *__restrict__ s, double *__restrict__ svar)
{
    __shared__ double sx[kExpTile], sy[kEcm ? kExpTile : 1];
    const int64_t c = (int64_t)blockIdx.x * kExpThreads + threadIdx.x;
    const bool ok = c < n_nodes;
    const int64_t i = ok ? (nodes ? (int64_t)nodes[c] : c) : -1;
    const double xi = ok ? x[i] : 0.0;
    const double yi = (kEcm && ok) ? y[i] : 0.0;
    const double ki = __dmul_rn(xi, yi);
    Kahan K, KV, S, SV;
    for (int64_t j0 = 0; j0 < n; j0 += kExpTile) {
        const int m = (int)min((int64_t)kExpTile, n - j0);
        __syncthreads();
        for (int t = threadIdx.x; t < m; t += kExpThreads) {
            if (kEcm) {
                const double yj = y[j0 + t];
                sx[t] = __dmul_rn(x[j0 + t], yj);  // kappa_j = x_j y_j
                sy[t] = yj;
            } else {
                sx[t] = x[j0 + t];
            }
        }
        __syncthreads();
        if (!ok) continue;
        for (int t = 0; t < m; t++) {
            if (j0 + t == i) continue;
            if (kEcm) {
                const double z = __dmul_rn(ki, sx[t]);
                const double tij = __dmul_rn(yi, sy[t]);
                const double omt = __dsub_rn(1.0, tij);
                const double p = __ddiv_rn(z, __dadd_rn(omt, z));
                K.add(p);
                KV.add(__dmul_rn(p, __dsub_rn(1.0, p)));
                const double ew = __ddiv_rn(p, omt);
                const double ew2 = __ddiv_rn(__dmul_rn(p, __dadd_rn(1.0, tij)), __dmul_rn(omt, omt));
                S.add(ew);
                SV.add(__dsub_rn(ew2, __dmul_rn(ew, ew)));
            } else {
                const double X = __dmul_rn(xi, sx[t]);
                const double p = __ddiv_rn(X, __dadd_rn(1.0, X));
                K.add(p);
                KV.add(__dmul_rn(p, __dsub_rn(1.0, p)));
            }
        }
    }
    if (!ok) return;
    if (k) k[c] = K.get();
    if (kvar) kvar[c] = KV.get();
    if (kEcm) {
        if (s) s[c] = S.get();
        if (svar) svar[c] = SV.get();
    }
}

}  // namespace

cudaError_t launch_expected(int model, int64_t n, const double *x, const double *y, const int32_t *nodes,
                            int64_t n_nodes, double *k, double *kvar, double *s, double *svar, cudaStream_t st)
{
    if (n_nodes <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((n_nodes + kExpThreads - 1) / kExpThreads);
    count_launch();
    if (model == FM_ECM)
        k_expected<true><<<grid, kExpThreads, 0, st>>>(n, x, y, nodes, n_nodes, k, kvar, s, svar);
    else
        k_expected<false><<<grid, kExpThreads, 0, st>>>(n, x, y, nodes, n_nodes, k, kvar, s, svar);
    return cudaGetLastError();
}

}  // namespace fm
