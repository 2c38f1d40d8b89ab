// psd.cuh -- Newton-PCG with the per-particle tangent blocks projected to positive semidefinite
// ("per-particle tangent blocks are eigen-projected to positive semidefinite before assembly";
// DESIGN.md R23).  A robustness variant, not the timed path: per Newton iteration
// every particle's block T = d^2 Psi / dF dF (D^2 x D^2 in vec(dF), row-major; symmetric) at F(u) is
// eigen-decomposed by cyclic Jacobi rotations, negative eigenvalues are clamped to 0, and the projected
// block T+ (packed upper triangle) is kept per particle; the HVP and the Jacobi diagonal then use
//   dF_p = (sum_j d_j grad N_jp^T) F_p^n,  y_i += V0_p (T+_p vec dF_p) F_p^nT grad N_ip,
// as plain per-particle scatters (fp64 atomics; this path is not bitwise reproducible).
#pragma once
#include "kernels.cuh"

namespace osmpm {

template <int D> struct PSD {
    static constexpr int N = D * D;              // block size
    static constexpr int NP = N * (N + 1) / 2;   // packed upper triangle
    static __host__ __device__ constexpr int at(int i, int j)
    {
        return i <= j ? i * N - i * (i - 1) / 2 + (j - i) : j * N - j * (j - 1) / 2 + (i - j);
    }
};

// dP = mu dF + (mu - lam ln J) A dF^T A + lam (A : dF) A,  A = F^{-T}  (R2)
template <int D>
__device__ __forceinline__ void dP_apply(const double* A, double c, double mu, double lam, const double* dF, double* dP)
{
    double AdF = 0.0;
#pragma unroll
    for (int k = 0; k < D * D; ++k) AdF += A[k] * dF[k];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
            double t = 0.0;  // (A dF^T A)_ab = sum_kl A_ak dF_lk A_lb
#pragma unroll
            for (int k = 0; k < D; ++k)
#pragma unroll
                for (int l = 0; l < D; ++l) t += A[a * D + k] * dF[l * D + k] * A[l * D + b];
            dP[a * D + b] = mu * dF[a * D + b] + c * t + lam * AdF * A[a * D + b];
        }
}

template <int D>
__device__ void psd_block(const double* F, double mu, double lam, double* Tp)
{
    constexpr int N = D * D;
    double C[D * D], A[D * D];
    cofactor<D, double>(F, C);
    const double J = det<D, double>(F);
#pragma unroll
    for (int k = 0; k < N; ++k) A[k] = C[k] / J;
    const double c = mu - lam * log(J);
    double T[N * N], Q[N * N];
    for (int k = 0; k < N; ++k) {
        double E[N], col[N];
        for (int q = 0; q < N; ++q) E[q] = (q == k) ? 1.0 : 0.0;
        dP_apply<D>(A, c, mu, lam, E, col);
        for (int i = 0; i < N; ++i) T[i * N + k] = col[i];
    }
    for (int i = 0; i < N; ++i) {
        for (int j = i + 1; j < N; ++j) {
            const double s = 0.5 * (T[i * N + j] + T[j * N + i]);
            T[i * N + j] = T[j * N + i] = s;
        }
        for (int j = 0; j < N; ++j) Q[i * N + j] = (i == j) ? 1.0 : 0.0;
    }
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                if (i == j) dia += T[i * N + i] * T[i * N + i];
                else off += T[i * N + j] * T[i * N + j];
            }
        if (off <= 1e-32 * dia) break;
        for (int p = 0; p < N - 1; ++p)
            for (int q = p + 1; q < N; ++q) {
                const double apq = T[p * N + q];
                if (apq == 0.0) continue;
                const double theta = (T[q * N + q] - T[p * N + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < N; ++k) {
                    const double akp = T[k * N + p], akq = T[k * N + q];
                    T[k * N + p] = cs * akp - sn * akq;
                    T[k * N + q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < N; ++k) {
                    const double apk = T[p * N + k], aqk = T[q * N + k];
                    T[p * N + k] = cs * apk - sn * aqk;
                    T[q * N + k] = sn * apk + cs * aqk;
                }
                for (int k = 0; k < N; ++k) {
                    const double qkp = Q[k * N + p], qkq = Q[k * N + q];
                    Q[k * N + p] = cs * qkp - sn * qkq;
                    Q[k * N + q] = sn * qkp + cs * qkq;
                }
            }
    }
    for (int i = 0; i < N; ++i)
        for (int j = i; j < N; ++j) {
            double s = 0.0;
            for (int k = 0; k < N; ++k) {
                const double l = T[k * N + k];
                if (l > 0.0) s += Q[i * N + k] * l * Q[j * N + k];
            }
            Tp[PSD<D>::at(i, j)] = s;
        }
}

// the particle's stencil (box-local base cell c, weights) and grad u gathered from the node vector uu
template <int D, typename R>
__device__ __forceinline__ void psd_stencil(const R* __restrict__ P, int64_t cap, int64_t p, const BoxDev& b, int* c,
                                            double (*w)[3], double (*dw)[3])
{
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double f;
        c[a] = base_of<double>((double)P[(PL<D>::X + a) * cap + p], b.o[a], b.inv_dx, &f) - b.lo[a];
        bspline<double>(f, b.inv_dx, w[a], dw[a]);
    }
}
template <int D>
__device__ __forceinline__ void gradN(const double (*w)[3], const double (*dw)[3], int i, int j, int k, double* gN)
{
    if (D == 3) {
        gN[0] = dw[0][i] * w[1][j] * w[2][k];
        gN[1] = w[0][i] * dw[1][j] * w[2][k];
        gN[2] = w[0][i] * w[1][j] * dw[2][k];
    } else {
        gN[0] = dw[0][i] * w[1][j];
        gN[1] = w[0][i] * dw[1][j];
    }
}
// sum_j v_j grad N_j^T over the 3^D stencil of node vector v (box layout, components innermost)
template <int D>
__device__ __forceinline__ void gather_grad_global(const BoxDev& b, const int* c, const double (*w)[3],
                                                   const double (*dw)[3], const double* __restrict__ v, double* G)
{
#pragma unroll
    for (int k = 0; k < D * D; ++k) G[k] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < Tile<D>::K3; ++k) {
                double gN[3];
                gradN<D>(w, dw, i, j, k, gN);
                const int64_t n = box_node<D>(b, c[0] + i, c[1] + j, c[2] + k);
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) G[a * D + bb] += v[n * D + a] * gN[bb];
            }
}

// T+ of every particle at F(u) = (I + grad u) F^n  ->  T[k * cap + p], k < PSD<D>::NP
template <int D, typename R>
__global__ void k_psd_tangent(const R* __restrict__ P, int64_t cap, int64_t n, const int* __restrict__ mat, BoxDev b,
                              MatTable mt, const double* __restrict__ u, double* __restrict__ T)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int c[3] = {0, 0, 0};
    double w[3][3], dw[3][3], G[D * D], Fn[D * D], Fu[D * D];
    psd_stencil<D, R>(P, cap, p, b, c, w, dw);
    gather_grad_global<D>(b, c, w, dw, u, G);
#pragma unroll
    for (int k = 0; k < D * D; ++k) Fn[k] = (double)P[(PL<D>::F + k) * cap + p];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int bb = 0; bb < D; ++bb) {
            double s = Fn[a * D + bb];
#pragma unroll
            for (int k = 0; k < D; ++k) s += G[a * D + k] * Fn[k * D + bb];
            Fu[a * D + bb] = s;
        }
    double Tp[PSD<D>::NP];
    const int m = mat[p];
    psd_block<D>(Fu, mt.mu[m], mt.lam[m], Tp);
    for (int k = 0; k < PSD<D>::NP; ++k) T[(int64_t)k * cap + p] = Tp[k];
}

// y += sum_p V0 (T+ vec dF) F^nT grad N,  dF = (sum_j d_j grad N_j^T) F^n
template <int D, typename R>
__global__ void k_hvp_psd(const R* __restrict__ P, int64_t cap, int64_t n, BoxDev b, const double* __restrict__ T,
                          const double* __restrict__ din, double* __restrict__ yout)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int c[3] = {0, 0, 0};
    double w[3][3], dw[3][3], G[D * D], Fn[D * D], dF[D * D], dP[D * D], Q[D * D];
    psd_stencil<D, R>(P, cap, p, b, c, w, dw);
    gather_grad_global<D>(b, c, w, dw, din, G);
#pragma unroll
    for (int k = 0; k < D * D; ++k) Fn[k] = (double)P[(PL<D>::F + k) * cap + p];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int bb = 0; bb < D; ++bb) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s += G[a * D + k] * Fn[k * D + bb];
            dF[a * D + bb] = s;
        }
    for (int i = 0; i < D * D; ++i) {
        double s = 0.0;
        for (int k = 0; k < D * D; ++k) s += T[(int64_t)PSD<D>::at(i, k) * cap + p] * dF[k];
        dP[i] = s;
    }
    const double V0 = (double)P[PL<D>::VOL * cap + p];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int bb = 0; bb < D; ++bb) {
            double s = 0.0;  // (dP F^nT)_ab
#pragma unroll
            for (int k = 0; k < D; ++k) s += dP[a * D + k] * Fn[bb * D + k];
            Q[a * D + bb] = V0 * s;
        }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < Tile<D>::K3; ++k) {
                double gN[3];
                gradN<D>(w, dw, i, j, k, gN);
                const int64_t nd = box_node<D>(b, c[0] + i, c[1] + j, c[2] + k);
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    double s = 0.0;
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) s += Q[a * D + bb] * gN[bb];
                    atomicAdd(&yout[nd * D + a], s);
                }
            }
}

// diag_{i,a} += V0 sum_{b,c} h_b h_c T+[(a,b),(a,c)],  h = F^nT grad N_i
template <int D, typename R>
__global__ void k_diag_psd(const R* __restrict__ P, int64_t cap, int64_t n, BoxDev b, const double* __restrict__ T,
                           double* __restrict__ dg)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int c[3] = {0, 0, 0};
    double w[3][3], dw[3][3], Fn[D * D];
    psd_stencil<D, R>(P, cap, p, b, c, w, dw);
#pragma unroll
    for (int k = 0; k < D * D; ++k) Fn[k] = (double)P[(PL<D>::F + k) * cap + p];
    const double V0 = (double)P[PL<D>::VOL * cap + p];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < Tile<D>::K3; ++k) {
                double gN[3], h[3];
                gradN<D>(w, dw, i, j, k, gN);
#pragma unroll
                for (int bb = 0; bb < D; ++bb) {
                    double s = 0.0;
#pragma unroll
                    for (int e = 0; e < D; ++e) s += Fn[e * D + bb] * gN[e];
                    h[bb] = s;
                }
                const int64_t nd = box_node<D>(b, c[0] + i, c[1] + j, c[2] + k);
                for (int a = 0; a < D; ++a) {
                    double s = 0.0;
                    for (int bb = 0; bb < D; ++bb)
                        for (int cc = 0; cc < D; ++cc)
                            s += h[bb] * h[cc] * T[(int64_t)PSD<D>::at(a * D + bb, a * D + cc) * cap + p];
                    atomicAdd(&dg[nd * D + a], V0 * s);
                }
            }
}

__global__ void k_add_mass_diag(int64_t nn, int d, const double* __restrict__ m, double idt2, double* __restrict__ dg)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    for (int a = 0; a < d; ++a) dg[i * d + a] += m[i] * idt2;
}

}  // namespace osmpm
