// kernels.cuh -- the sm_100a kernels of one implicit MPM sub-step (§2.2, Alg. 1).
//
// Data layout:
//   particles  field-major SoA of R (fp64 or fp32), capacity `cap`, sorted tile-major by cell:
//              x[D] v[D] F[D*D] B[D*D] m V0   (+ int32 mat, uint8 bnd, int32 pid)
//   cache      per-particle Newton linearisation, field-major R:
//              S' = V0 mu F^n F^nT (sym), Ah = (I + grad u)^{-T}, c' = V0 (mu - lam ln J), l' = V0 lam
//   node box   dense fp64 arrays over the step's tight box (BoxDev), components innermost.
#pragma once
#include "device.cuh"

namespace osmpm {

template <int D> struct PL {
    static constexpr int X = 0, V = D, F = 2 * D, B = 2 * D + D * D, M = 2 * D + 2 * D * D, VOL = M + 1,
                         NF = VOL + 1;
};
template <int D> struct CL {
    static constexpr int S = 0, A = Sym<D>::N, C = A + D * D, L = C + 1, NF = L + 1;
};

constexpr int MAX_MATS = 16;
struct MatTable {
    int n;
    double mu[MAX_MATS], lam[MAX_MATS];
};

// =============================================================================================
// a1: binning + sort support
// =============================================================================================

// lowest / highest base node per axis, and the safe-interior check
template <int D, typename R>
__global__ void k_bounds(const R* __restrict__ P, int64_t cap, int64_t n, BoxDev g, int* bounds,
                         const int* __restrict__ pid, ErrLatch* err)
{
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            R f;
            int b = base_of<R>(P[(PL<D>::X + a) * cap + p], g.o[a], g.inv_dx, &f);
            if (b < 0 || b + 2 > g.gdims[a] - 1) latch_error(err, 2 /*OUT_OF_DOMAIN*/, pid[p]);
            lo[a] = min(lo[a], b);
            hi[a] = max(hi[a], b);
        }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
        for (int off = 16; off > 0; off >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], off));
            hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], off));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&bounds[a], lo[a]);
            atomicMax(&bounds[3 + a], hi[a]);
        }
    }
}

template <int D, typename R>
__global__ void k_keys(const R* __restrict__ P, int64_t cap, int64_t n, BoxDev b, uint32_t* keys, int* vals,
                       const int* __restrict__ pid, ErrLatch* err)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int c[3] = {0, 0, 0};
    bool in = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        R f;
        c[a] = base_of<R>(P[(PL<D>::X + a) * cap + p], b.o[a], b.inv_dx, &f) - b.lo[a];
        in = in && c[a] >= 0 && c[a] < b.nc[a];
    }
    if (!in) {  // outside this (slab's) box: a missed migration; never silently corrupt the sort
        latch_error(err, 2 /*OUT_OF_DOMAIN*/, pid[p]);
        c[0] = c[1] = c[2] = 0;
    }
    keys[p] = cell_key<D>(b, c[0], c[1], c[2]);
    vals[p] = (int)p;
}

// gather-permute all real fields (field-major) and the integer fields
template <typename R>
__global__ void k_permute(const R* __restrict__ src, R* __restrict__ dst, int nf, int64_t cap, int64_t n,
                          const int* __restrict__ perm, const int* __restrict__ mat_s, int* __restrict__ mat_d,
                          const uint8_t* __restrict__ bnd_s, uint8_t* __restrict__ bnd_d,
                          const int* __restrict__ pid_s, int* __restrict__ pid_d)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int j = perm[i];
    for (int f = 0; f < nf; ++f) dst[f * cap + i] = src[f * cap + j];
    mat_d[i] = mat_s[j];
    bnd_d[i] = bnd_s[j];
    pid_d[i] = pid_s[j];
}

// cell_start[k] = first sorted particle with key >= k, for k in [0, ncells]
__global__ void k_cell_start(const uint32_t* __restrict__ keys, int64_t n, int64_t ncells, int* cell_start)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t lo = (i == 0) ? 0 : (int64_t)keys[i - 1] + 1;
    int64_t hi = (i == n) ? ncells : (int64_t)keys[i];
    for (int64_t k = lo; k <= hi; ++k) cell_start[k] = (int)i;
}

// node pass: active <=> m > thr (R4), v^n = (mv) / m
template <int D>
__global__ void k_p2g_nodes(int64_t nn, const double* __restrict__ m, const double* __restrict__ mom,
                            double* __restrict__ vn, uint8_t* __restrict__ act, double thr)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const bool a = m[i] > thr;
    act[i] = a;
#pragma unroll
    for (int k = 0; k < D; ++k) vn[i * D + k] = a ? mom[i * D + k] / m[i] : 0.0;
}

// boundary-particle mass m^b_i = sum_{p in P^∂} m_p N_ip
template <int D, typename R>
__global__ void k_bmass(const R* __restrict__ P, int64_t cap, int64_t n, const uint8_t* __restrict__ bnd, BoxDev b,
                        double* __restrict__ mb)
{
    using L = PL<D>;
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n || !bnd[p]) return;
    R w[3][3], dw[3][3], f[3];
    int c[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = base_of<R>(P[(L::X + a) * cap + p], b.o[a], b.inv_dx, &f[a]) - b.lo[a];
        bspline<R>(f[a], (R)b.inv_dx, w[a], dw[a]);
    }
    const R mp = P[L::M * cap + p];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < Tile<D>::K3; ++k) {
                R N = (D == 3) ? w[0][i] * w[1][j] * w[2][k] : w[0][i] * w[1][j];
                atomicAdd(&mb[box_node<D>(b, c[0] + i, c[1] + j, c[2] + k)], (double)(mp * N));
            }
}

}  // namespace osmpm
#include "tiled.cuh"
#include "hvp_sw.cuh"
#include "p2g_tiled.cuh"
#include "grad_sw.cuh"
namespace osmpm {

// node terms of the gradient / diagonal / energy:
//   g += m/dt^2 (u - dt v^n) - m grav ;  diag += m/dt^2 ;
//   E_node = m/(2dt^2)|u - dt v^n|^2 - u . m grav ;  |g_free|^2
//   noise scale m/(2dt^2)(|u|^2 + |dt v^n|^2) + |u . m grav|  (R8)
//   force scale |m (|v^n|/dt + |grav|)|^2 over free DOFs      (R6)
// partials per block: {E_node, E_abs node terms, |g_free|^2, force scale^2}
template <int D>
__global__ void k_grad_nodes(int64_t nn, int64_t nown, const double* __restrict__ m, const double* __restrict__ vn,
                             const double* __restrict__ u, const uint8_t* __restrict__ fmask, double dt,
                             double g0, double g1, double g2, double* __restrict__ g, double* __restrict__ dg,
                             double* __restrict__ partials)
{
    double red[4] = {0.0, 0.0, 0.0, 0.0};
    const double grav[3] = {g0, g1, g2};
    const double idt2 = 1.0 / (dt * dt);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
        const double mi = m[i];
        double q = 0.0, wf = 0.0, qa = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const double ua = u[i * D + a], va = vn[i * D + a];
            const double r = ua - dt * va;
            const double fe = mi * grav[a];
            q += r * r;
            wf += ua * fe;
            qa += ua * ua + dt * dt * va * va;
            const double gv = g[i * D + a] + mi * idt2 * r - fe;
            g[i * D + a] = gv;
            dg[i * D + a] += mi * idt2;
            if (fmask[i * D + a] && i < nown) {
                red[2] += gv * gv;
                const double fs = mi * fabs(va) / dt + fabs(fe);
                red[3] += fs * fs;
            }
        }
        if (i < nown) {
            red[0] += 0.5 * mi * idt2 * q - wf;
            red[1] += 0.5 * mi * idt2 * qa + fabs(wf);
        }
    }
    block_reduce_store<4>(red, partials);
}

// =============================================================================================
// a8: G2P + F update + advection, per particle
// =============================================================================================
#ifndef OSMPM_G2P_MINB
#define OSMPM_G2P_MINB 4
#endif
template <int D, typename R>
__global__ void __launch_bounds__(128, OSMPM_G2P_MINB) k_g2p(R* __restrict__ P, int64_t cap, int64_t n, const int* __restrict__ pid, BoxDev b,
                      const double* __restrict__ vg, double dt, ErrLatch* err)
{
    using L = PL<D>;
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    R w[3][3], dw[3][3], f[3];
    int c[3] = {0, 0, 0};
    const R inv_dx = (R)b.inv_dx, dx = (R)b.dx;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = base_of<R>(P[(L::X + a) * cap + p], b.o[a], b.inv_dx, &f[a]) - b.lo[a];
        bspline<R>(f[a], inv_dx, w[a], dw[a]);
    }
    // tensor-product gather (contract the last axis first): per component a the seven sums
    //   N v, dN/dx_b v (b < D), N v (l_b - f_b) (b < D)
    // with per-axis weight sets w, dw and wo = w (l - f) (the node offset taken per node, so
    // B_p = dx sum N v (l - f)^T carries no cancellation), 147 FMA per component in 3D instead of the
    // per-node products of N, grad N and the offsets
    R wo[3][3];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int l = 0; l < 3; ++l) wo[a][l] = w[a][l] * (R(l) - f[a]);
    R vp[D], Bp[D * D], gv[D * D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        vp[a] = 0;
#pragma unroll
        for (int bb = 0; bb < D; ++bb) Bp[a * D + bb] = gv[a * D + bb] = 0;
    }
    if (D == 3) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            R Yww[3] = {0, 0, 0}, Ydw[3] = {0, 0, 0}, Yow[3] = {0, 0, 0}, Ywd[3] = {0, 0, 0}, Ywo[3] = {0, 0, 0};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double* vv = vg + box_node<D>(b, c[0] + i, c[1] + j, c[2]) * D;
                R Zw[3] = {0, 0, 0}, Zd[3] = {0, 0, 0}, Zo[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < 3; ++k)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const R va = (R)vv[k * 3 + a];
                        Zw[a] = fma(w[2][k], va, Zw[a]);
                        Zd[a] = fma(dw[2][k], va, Zd[a]);
                        Zo[a] = fma(wo[2][k], va, Zo[a]);
                    }
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    Yww[a] = fma(w[1][j], Zw[a], Yww[a]);
                    Ydw[a] = fma(dw[1][j], Zw[a], Ydw[a]);
                    Yow[a] = fma(wo[1][j], Zw[a], Yow[a]);
                    Ywd[a] = fma(w[1][j], Zd[a], Ywd[a]);
                    Ywo[a] = fma(w[1][j], Zo[a], Ywo[a]);
                }
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                vp[a] = fma(w[0][i], Yww[a], vp[a]);
                gv[a * 3 + 0] = fma(dw[0][i], Yww[a], gv[a * 3 + 0]);
                gv[a * 3 + 1] = fma(w[0][i], Ydw[a], gv[a * 3 + 1]);
                gv[a * 3 + 2] = fma(w[0][i], Ywd[a], gv[a * 3 + 2]);
                Bp[a * 3 + 0] = fma(wo[0][i], Yww[a], Bp[a * 3 + 0]);
                Bp[a * 3 + 1] = fma(w[0][i], Yow[a], Bp[a * 3 + 1]);
                Bp[a * 3 + 2] = fma(w[0][i], Ywo[a], Bp[a * 3 + 2]);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double* vv = vg + box_node<D>(b, c[0] + i, c[1], 0) * D;
            R Yw[2] = {0, 0}, Yd[2] = {0, 0}, Yo[2] = {0, 0};
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const R va = (R)vv[j * 2 + a];
                    Yw[a] = fma(w[1][j], va, Yw[a]);
                    Yd[a] = fma(dw[1][j], va, Yd[a]);
                    Yo[a] = fma(wo[1][j], va, Yo[a]);
                }
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                vp[a] = fma(w[0][i], Yw[a], vp[a]);
                gv[a * 2 + 0] = fma(dw[0][i], Yw[a], gv[a * 2 + 0]);
                gv[a * 2 + 1] = fma(w[0][i], Yd[a], gv[a * 2 + 1]);
                Bp[a * 2 + 0] = fma(wo[0][i], Yw[a], Bp[a * 2 + 0]);
                Bp[a * 2 + 1] = fma(w[0][i], Yo[a], Bp[a * 2 + 1]);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < D * D; ++k) Bp[k] *= dx;
    R F[D * D], Fn[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] = P[(L::F + k) * cap + p];
    const R rdt = (R)dt;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int bb = 0; bb < D; ++bb) {
            R s = F[a * D + bb];
#pragma unroll
            for (int k = 0; k < D; ++k) s += rdt * gv[a * D + k] * F[k * D + bb];
            Fn[a * D + bb] = s;
        }
    if (!(det<D, R>(Fn) > R(0))) latch_error(err, 3 /*INVERTED_F*/, pid[p]);
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
        P[(L::F + k) * cap + p] = Fn[k];
        P[(L::B + k) * cap + p] = Bp[k];
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const R xn = P[(L::X + a) * cap + p] + rdt * vp[a];
        P[(L::X + a) * cap + p] = xn;
        P[(L::V + a) * cap + p] = vp[a];
        R ff;
        const int bn = base_of<R>(xn, b.o[a], b.inv_dx, &ff);
        if (bn < 0 || bn + 2 > b.gdims[a] - 1) latch_error(err, 2 /*OUT_OF_DOMAIN*/, pid[p]);
    }
}

// =============================================================================================
// node-level kernels: masks, Newton / PCG vector operations (a3, a6)
// =============================================================================================
// fmask = active & !dirichlet ; Newton initial guess (R5)
template <int D>
__global__ void k_newton_init(int64_t nn, const uint8_t* __restrict__ act, const uint8_t* __restrict__ dmask,
                              const double* __restrict__ dval, const double* __restrict__ vn, double dt, int guess,
                              uint8_t* __restrict__ fmask, double* __restrict__ u)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const bool dir = (dmask[i] >> a) & 1;
        const bool fr = act[i] && !dir;
        fmask[i * D + a] = fr;
        u[i * D + a] = fr ? (guess == 1 ? 0.0 : dt * vn[i * D + a]) : ((act[i] && dir) ? dt * dval[i * D + a] : 0.0);
    }
}

struct CGScalars {
    double rz, pq, alpha, beta, rr, gn, tol2, E0, Eabs0;
    int done, it, negcurv_first, fixed;
};

// r = -g (free), z = r/diag, p = z, x = 0, y = 0 ; partials {rz, rr}
template <int D>
__global__ void k_cg_init(int64_t ndof, int64_t nown_dof, const uint8_t* __restrict__ fm, const double* __restrict__ g,
                          double* __restrict__ dg, double* __restrict__ r, double* __restrict__ z,
                          double* __restrict__ p, double* __restrict__ x, double* __restrict__ y,
                          double* __restrict__ partials)
{
    double red[2] = {0.0, 0.0};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndof; k += (int64_t)gridDim.x * blockDim.x) {
        const bool f = fm[k];
        if (!f) dg[k] = 1.0;
        const double rk = f ? -g[k] : 0.0;
        const double zk = rk / dg[k];
        r[k] = rk;
        z[k] = zk;
        p[k] = zk;
        x[k] = 0.0;
        y[k] = 0.0;
        if (f && k < nown_dof) {
            red[0] += rk * zk;
            red[1] += rk * rk;
        }
    }
    block_reduce_store<2>(red, partials);
}

__device__ __forceinline__ void cg_init_fin(const double* v, CGScalars* s, double gn, double cg_rtol, int fixed)
{
    {
        s->rz = v[0];
        s->rr = v[1];
        s->gn = gn;
        s->tol2 = cg_rtol * cg_rtol * gn * gn;
        s->it = 0;
        s->negcurv_first = 0;
        s->fixed = fixed;
        s->done = (!fixed && v[1] <= s->tol2) ? 1 : 0;
        s->alpha = s->beta = 0.0;
    }
}
__global__ void k_cg_init_fin(const double* partials, int nb, CGScalars* s, double gn, double cg_rtol, int fixed)
{
    double v[2];
    final_sum<2>(partials, nb, v);
    if (threadIdx.x == 0) cg_init_fin(v, s, gn, cg_rtol, fixed);
}
// group-reduced variant: v = {r.z, r.r} already summed over slabs and ranks
__global__ void k_cg_init_fin_sum(const double* v, CGScalars* s, double gn, double cg_rtol, int fixed)
{
    cg_init_fin(v, s, gn, cg_rtol, fixed);
}

// q = y + m/dt^2 p on free DOFs, 0 elsewhere (in place in y) ; partial p.q
template <int D>
__global__ void k_cg_q(int64_t nn, int64_t nown, const uint8_t* __restrict__ fm, const double* __restrict__ m, double idt2,
                       const double* __restrict__ p, double* __restrict__ y, const CGScalars* s,
                       double* __restrict__ partials)
{
    double red[1] = {0.0};
    if (!s->done) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int64_t k = i * D + a;
                // non-free DOFs (inactive, Dirichlet) are skipped without touching memory: their p is
                // 0 and y there is never read (k_cg_update skips them too; k_cg_p re-zeroes y)
                if (!fm[k]) continue;
                const double q = y[k] + m[i] * idt2 * p[k];
                y[k] = q;
                if (i < nown) red[0] += p[k] * q;
            }
        }
    }
    block_reduce_store<1>(red, partials);
}

__device__ __forceinline__ void cg_alpha(const double* v, CGScalars* s)
{
    {
        s->pq = v[0];
        if (!(v[0] > 0.0)) {
            // non-positive curvature: stop, in fixed-iteration mode too (the remaining launches of a
            // fixed solve then leave x unchanged; R7)
            s->alpha = 0.0;
            if (s->it == 0) s->negcurv_first = 1;
            s->done = 2;
        } else {
            s->alpha = s->rz / v[0];
        }
    }
}
__global__ void k_cg_alpha(const double* partials, int nb, CGScalars* s)
{
    if (s->done) return;
    double v[1];
    final_sum<1>(partials, nb, v);
    if (threadIdx.x == 0) cg_alpha(v, s);
}
__global__ void k_cg_alpha_sum(const double* v, CGScalars* s)
{
    if (!s->done) cg_alpha(v, s);
}

// x += alpha p ; r -= alpha q ; z = r/diag ; partials {r.z, r.r}
__global__ void k_cg_update(int64_t ndof, int64_t nown_dof, const uint8_t* __restrict__ fm, const double* __restrict__ p,
                            const double* __restrict__ q, const double* __restrict__ dg, double* __restrict__ x,
                            double* __restrict__ r, double* __restrict__ z, const CGScalars* s,
                            double* __restrict__ partials)
{
    double red[2] = {0.0, 0.0};
    if (!s->done) {
        const double al = s->alpha;
        for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndof; k += (int64_t)gridDim.x * blockDim.x) {
            if (!fm[k]) continue;  // x, r, z stay 0 on non-free DOFs (k_cg_init)
            const double xk = x[k] + al * p[k];
            const double rk = r[k] - al * q[k];
            const double zk = rk / dg[k];
            x[k] = xk;
            r[k] = rk;
            z[k] = zk;
            if (k < nown_dof) {
                red[0] += rk * zk;
                red[1] += rk * rk;
            }
        }
    }
    block_reduce_store<2>(red, partials);
}

__device__ __forceinline__ void cg_beta(const double* v, CGScalars* s)
{
    {
        s->beta = (s->rz > 0.0) ? v[0] / s->rz : 0.0;
        s->rz = v[0];
        s->rr = v[1];
        s->it += 1;
        if (!s->fixed && v[1] <= s->tol2) s->done = 1;
    }
}
__global__ void k_cg_beta(const double* partials, int nb, CGScalars* s)
{
    if (s->done) return;
    double v[2];
    final_sum<2>(partials, nb, v);
    if (threadIdx.x == 0) cg_beta(v, s);
}
__global__ void k_cg_beta_sum(const double* v, CGScalars* s)
{
    if (!s->done) cg_beta(v, s);
}
// single-block final sum that skips the work once CG is done (group reductions of the CG loop)
template <int NV>
__global__ void k_final_sum_cg(const double* partials, int nb, const CGScalars* s, double* out)
{
    if (s->done) return;
    final_sum<NV>(partials, nb, out);
}

// p = z + beta p ; y = 0
// L2 reuse between the PCG's vector passes: the grid-stride sweeps of k_cg_q_alpha and
// k_cg_p run from the last DOF down, k_cg_update_beta from the first up, so that each pass starts where
// the previous one ended -- on the lines still in the 126 MB L2 (a vector is 59 MB at C5).
// (measured on C5: PCG vector kernels 77.3 vs 77.6 ms per sub-step, HVP 650.4 vs 650.8 ms -- the HVP's
// first tiles find k_cg_p's last p lines; the opposite assignment, 77.8 ms)
__device__ __forceinline__ int64_t rev_index(int64_t t, int64_t n) { return n - 1 - t; }
__device__ __forceinline__ int64_t fwd_index(int64_t t, int64_t) { return t; }

__global__ void k_cg_p(int64_t ndof, const uint8_t* __restrict__ fm, const double* __restrict__ z,
                       double* __restrict__ p, double* __restrict__ y, const CGScalars* s)
{
    if (s->done) return;
    const double be = s->beta;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ndof; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = rev_index(t, ndof);
        if (fm[k]) p[k] = z[k] + be * p[k];  // p stays 0 on non-free DOFs
        y[k] = 0.0;
    }
}

// ---------------------------------------------------------------------------------------------
// Standard PCG of one slab (no exchange between the partial sums and the scalars): 3 vector kernels
// per iteration instead of 3 + 2 single-block ones.  The last block of k_cg_q_alpha / k_cg_update_beta
// to finish (an atomic ticket after each block's partial is fenced) reduces all block partials in the
// fixed order of final_sum and sets alpha / beta itself.  k_cg_q_alpha only reduces p.q; the update
// recomputes q = y + m/dt^2 p with the same expression instead of reading it back (one vector write
// less per iteration).  Same scalars and vectors as k_cg_q / k_cg_alpha / k_cg_update / k_cg_beta.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ bool last_block_ticket(unsigned* counter)
{
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    return last;
}

template <int D>
__global__ void k_cg_q_alpha(int64_t nn, int64_t nown, const uint8_t* __restrict__ fm, const double* __restrict__ m,
                             double idt2, const double* __restrict__ p, const double* __restrict__ y, CGScalars* s,
                             double* __restrict__ partials, unsigned* counter)
{
    if (s->done) return;
    double red[1] = {0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nn; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = rev_index(t, nn);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int64_t k = i * D + a;
            if (!fm[k]) continue;
            const double q = y[k] + m[i] * idt2 * p[k];
            if (i < nown) red[0] += p[k] * q;
        }
    }
    block_reduce_store<1>(red, partials);
    if (last_block_ticket(counter)) {
        double v[1];
        final_sum<1>(partials, gridDim.x, v);
        if (threadIdx.x == 0) {
            cg_alpha(v, s);
            *counter = 0u;
        }
    }
}

template <int D>
__global__ void k_cg_update_beta(int64_t ndof, int64_t nown_dof, const uint8_t* __restrict__ fm,
                                 const double* __restrict__ m, double idt2, const double* __restrict__ p,
                                 const double* __restrict__ y, const double* __restrict__ dg, double* __restrict__ x,
                                 double* __restrict__ r, double* __restrict__ z, CGScalars* s,
                                 double* __restrict__ partials, unsigned* counter)
{
    if (s->done) return;
    const double al = s->alpha;
    double red[2] = {0.0, 0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ndof; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = fwd_index(t, ndof);
        if (!fm[k]) continue;
        const double q = y[k] + m[k / D] * idt2 * p[k];
        const double xk = x[k] + al * p[k];
        const double rk = r[k] - al * q;
        const double zk = rk / dg[k];
        x[k] = xk;
        r[k] = rk;
        z[k] = zk;
        if (k < nown_dof) {
            red[0] += rk * zk;
            red[1] += rk * rk;
        }
    }
    block_reduce_store<2>(red, partials);
    if (last_block_ticket(counter)) {
        double v[2];
        final_sum<2>(partials, gridDim.x, v);
        if (threadIdx.x == 0) {
            cg_beta(v, s);
            *counter = 0u;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Single-reduction Jacobi PCG (Chronopoulos & Gear; R22), one reduction per iteration:
//   init      r = -g, u = diag^-1 r, x = p = s = 0, y = 0;  partials {r.u, r.r, u^T M u / dt^2}
//   HVP(u)    y = K u; per-CTA partials u^T K u
//   scalar    gamma = r.u, delta = u^T (K + M/dt^2) u, beta = gamma / gamma_old (0 first),
//             c = delta - beta gamma / alpha_old (= p^T H p; delta first), c <= 0 -> stop, alpha = gamma / c
//   update    p = u + beta p, s = (y + M u / dt^2) + beta s, x += alpha p, r -= alpha s, u = diag^-1 r,
//             y = 0;  partials for the next iteration
// (the oracle's pcg_single_reduction, same recurrences)
// ---------------------------------------------------------------------------------------------
template <int D>
__global__ void k_cgs_init(int64_t ndof, int64_t nown_dof, const uint8_t* __restrict__ fm, const double* __restrict__ g,
                           double* __restrict__ dg, double* __restrict__ r, double* __restrict__ u,
                           double* __restrict__ p, double* __restrict__ sv, double* __restrict__ x,
                           double* __restrict__ y, const double* __restrict__ m, double idt2,
                           double* __restrict__ partials)
{
    double red[3] = {0.0, 0.0, 0.0};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndof; k += (int64_t)gridDim.x * blockDim.x) {
        const bool f = fm[k];
        if (!f) dg[k] = 1.0;
        const double rk = f ? -g[k] : 0.0;
        const double uk = rk / dg[k];
        r[k] = rk;
        u[k] = uk;
        p[k] = 0.0;
        sv[k] = 0.0;
        x[k] = 0.0;
        y[k] = 0.0;
        if (f && k < nown_dof) {
            red[0] += rk * uk;
            red[1] += rk * rk;
            red[2] += m[k / D] * idt2 * uk * uk;
        }
    }
    block_reduce_store<3>(red, partials);
}

__global__ void k_cgs_start(CGScalars* s, double gn, double cg_rtol, int fixed)
{
    s->rz = s->rr = s->alpha = s->beta = s->pq = 0.0;
    s->gn = gn;
    s->tol2 = cg_rtol * cg_rtol * gn * gn;
    s->it = 0;
    s->negcurv_first = 0;
    s->fixed = fixed;
    s->done = 0;
}
__device__ __forceinline__ void cgs_scalar(double gamma, double rr, double delta, CGScalars* s)
{
    if (!s->fixed && rr <= s->tol2) {
        s->done = 1;
        return;
    }
    const double beta = (s->it == 0 || !(s->rz > 0.0)) ? 0.0 : gamma / s->rz;
    const double c = (s->it == 0) ? delta : delta - beta * gamma / s->alpha;
    s->pq = c;
    if (!(c > 0.0)) {
        if (s->it == 0) s->negcurv_first = 1;
        s->done = 2;
        return;
    }
    s->beta = beta;
    s->alpha = gamma / c;
    s->rz = gamma;
    s->rr = rr;
    s->it += 1;
}
// partB: 3 per block {r.u, r.r, u^T M u}; partH: u^T K u per HVP tile
__global__ void k_cgs_scalar(const double* partB, int nb, const double* partH, int nh, CGScalars* s)
{
    if (s->done) return;
    double v[3], w[1];
    final_sum<3>(partB, nb, v);
    __syncthreads();
    final_sum<1>(partH, nh, w);
    if (threadIdx.x == 0) cgs_scalar(v[0], v[1], v[2] + w[0], s);
}
// remote: sum this rank's partials -> out[0..2] = {r.u, r.r, u^T (K + M/dt^2) u} for the all-reduce
__global__ void k_cgs_local_sum(const double* partB, int nb, const double* partH, int nh, const CGScalars* s,
                                double* out)
{
    if (s->done) return;
    double v[3], w[1];
    final_sum<3>(partB, nb, v);
    __syncthreads();
    final_sum<1>(partH, nh, w);
    if (threadIdx.x == 0) {
        out[0] = v[0];
        out[1] = v[1];
        out[2] = v[2] + w[0];
    }
}
__global__ void k_cgs_scalar_sum(const double* v, CGScalars* s)
{
    if (!s->done) cgs_scalar(v[0], v[1], v[2], s);
}

template <int D>
__global__ void k_cgs_update(int64_t ndof, int64_t nown_dof, const uint8_t* __restrict__ fm, const double* __restrict__ dg,
                             const double* __restrict__ m, double idt2, double* __restrict__ u, double* __restrict__ y,
                             double* __restrict__ p, double* __restrict__ sv, double* __restrict__ x,
                             double* __restrict__ r, const CGScalars* s, double* __restrict__ partials)
{
    if (s->done) return;
    const double al = s->alpha, be = s->beta;
    double red[3] = {0.0, 0.0, 0.0};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndof; k += (int64_t)gridDim.x * blockDim.x) {
        if (fm[k]) {
            const double mk = m[k / D] * idt2;
            const double uk = u[k];
            const double pk = uk + be * p[k];
            const double sk = (y[k] + mk * uk) + be * sv[k];
            const double rk = r[k] - al * sk;
            const double un = rk / dg[k];
            p[k] = pk;
            sv[k] = sk;
            x[k] += al * pk;
            r[k] = rk;
            u[k] = un;
            if (k < nown_dof) {
                red[0] += rk * un;
                red[1] += rk * rk;
                red[2] += mk * un * un;
            }
        }
        y[k] = 0.0;
    }
    block_reduce_store<3>(red, partials);
}

// partials of a . b over the free owned DOFs
__global__ void k_dot_free(int64_t ndof, int64_t nown_dof, const uint8_t* __restrict__ fm, const double* __restrict__ a,
                           const double* __restrict__ b, double* __restrict__ partials)
{
    double red[1] = {0.0};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndof; k += (int64_t)gridDim.x * blockDim.x)
        if (fm[k] && k < nown_dof) red[0] += a[k] * b[k];
    block_reduce_store<1>(red, partials);
}

// ut = u + alpha x on free DOFs
__global__ void k_axpy_free(int64_t ndof, const uint8_t* __restrict__ fm, const double* __restrict__ u, double alpha,
                            const double* __restrict__ x, double* __restrict__ ut)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ndof; k += (int64_t)gridDim.x * blockDim.x)
        ut[k] = fm[k] ? u[k] + alpha * x[k] : u[k];
}

template <int NV>
__global__ void k_final_sum(const double* partials, int nb, double* out)
{
    final_sum<NV>(partials, nb, out);
}

// v^{n+1} = u / dt on active nodes ("v = (x - x^n)/dT")
template <int D>
__global__ void k_vnew(int64_t nn, const uint8_t* __restrict__ act, const double* __restrict__ u, double inv_dt,
                       double* __restrict__ v)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
#pragma unroll
    for (int a = 0; a < D; ++a) v[i * D + a] = act[i] ? u[i * D + a] * inv_dt : 0.0;
}

// =============================================================================================
// dense <-> box node vectors
// =============================================================================================
template <int D, typename T>
__global__ void k_box_to_dense(BoxDev b, int64_t nown, int ncomp, const T* __restrict__ src, T* __restrict__ dst)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nown) return;  // ghost planes are exported by their owner
    int i2 = (D == 3) ? (int)(i % b.nn[2]) : 0;
    int i1 = (D == 3) ? (int)((i / b.nn[2]) % b.nn[1]) : (int)(i % b.nn[1]);
    int i0 = (D == 3) ? (int)(i / ((int64_t)b.nn[2] * b.nn[1])) : (int)(i / b.nn[1]);
    int g0 = b.lo[0] + i0, g1 = b.lo[1] + i1, g2 = (D == 3) ? b.lo[2] + i2 : 0;
    if (g0 >= b.gdims[0] || g1 >= b.gdims[1] || (D == 3 && g2 >= b.gdims[2])) return;
    int64_t g = (D == 3) ? ((int64_t)g0 * b.gdims[1] + g1) * b.gdims[2] + g2 : (int64_t)g0 * b.gdims[1] + g1;
    for (int a = 0; a < ncomp; ++a) dst[g * ncomp + a] = src[i * ncomp + a];
}

template <int D, typename T>
__global__ void k_dense_to_box(BoxDev b, int ncomp, const T* __restrict__ src, T* __restrict__ dst)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= b.nnodes) return;
    int i2 = (D == 3) ? (int)(i % b.nn[2]) : 0;
    int i1 = (D == 3) ? (int)((i / b.nn[2]) % b.nn[1]) : (int)(i % b.nn[1]);
    int i0 = (D == 3) ? (int)(i / ((int64_t)b.nn[2] * b.nn[1])) : (int)(i / b.nn[1]);
    int g0 = b.lo[0] + i0, g1 = b.lo[1] + i1, g2 = (D == 3) ? b.lo[2] + i2 : 0;
    bool in = !(g0 >= b.gdims[0] || g1 >= b.gdims[1] || (D == 3 && g2 >= b.gdims[2]));
    int64_t g = (D == 3) ? ((int64_t)g0 * b.gdims[1] + g1) * b.gdims[2] + g2 : (int64_t)g0 * b.gdims[1] + g1;
    for (int a = 0; a < ncomp; ++a) dst[i * ncomp + a] = in ? src[g * ncomp + a] : T(0);
}

// Dirichlet list (global node index, mask, values) -> box arrays
template <int D>
__global__ void k_scatter_dirichlet(BoxDev b, int64_t n, const int64_t* __restrict__ gidx,
                                    const uint8_t* __restrict__ mask, const double* __restrict__ val,
                                    uint8_t* __restrict__ dmask, double* __restrict__ dval)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int64_t g = gidx[k];
    int g2 = (D == 3) ? (int)(g % b.gdims[2]) : 0;
    int g1 = (D == 3) ? (int)((g / b.gdims[2]) % b.gdims[1]) : (int)(g % b.gdims[1]);
    int g0 = (D == 3) ? (int)(g / ((int64_t)b.gdims[2] * b.gdims[1])) : (int)(g / b.gdims[1]);
    int i0 = g0 - b.lo[0], i1 = g1 - b.lo[1], i2 = (D == 3) ? g2 - b.lo[2] : 0;
    if (i0 < 0 || i1 < 0 || i2 < 0 || i0 >= b.nn[0] || i1 >= b.nn[1] || (D == 3 && i2 >= b.nn[2])) return;
    int64_t i = box_node<D>(b, i0, i1, i2);
    dmask[i] |= mask[k];
#pragma unroll
    for (int a = 0; a < D; ++a)
        if ((mask[k] >> a) & 1) dval[i * D + a] = val[k * D + a];
}

// unsort: dst[pid[i]] = src[i] for every real field
template <typename R>
__global__ void k_unsort_field(const R* __restrict__ src, int64_t n, const int* __restrict__ pid, int ncomp_stride,
                               int comp, double* __restrict__ dst)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    dst[(int64_t)pid[i] * ncomp_stride + comp] = (double)src[i];
}

template <typename R>
__global__ void k_sort_field(const double* __restrict__ src, int64_t n, const int* __restrict__ pid, int ncomp_stride,
                             int comp, R* __restrict__ dst)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    dst[i] = (R)src[(int64_t)pid[i] * ncomp_stride + comp];
}


template <int D>
__global__ void k_fext(int64_t nn, const double* m, double g0, double g1, double g2, double* out)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const double gg[3] = {g0, g1, g2};
    for (int a = 0; a < D; ++a) out[i * D + a] = m[i] * gg[a];
}

// halo reverse-add: dst[i] += src[i]
__global__ void k_add_vec(int64_t n, const double* __restrict__ src, double* __restrict__ dst)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

template <int D>
__global__ void k_add_mass(int64_t nn, const double* m, double idt2, const double* d, double* y)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    for (int a = 0; a < D; ++a) y[i * D + a] += m[i] * idt2 * d[i * D + a];
}

// node part of E_h for the line search: {E_node, |E_node terms|}
template <int D>
__global__ void k_energy_nodes(int64_t nn, int64_t nown, const double* __restrict__ m, const double* __restrict__ vn,
                               const double* __restrict__ uu, double dt, double g0, double g1, double g2,
                               double* __restrict__ partials)
{
    double red[2] = {0.0, 0.0};
    const double grav[3] = {g0, g1, g2};
    const double idt2 = 1.0 / (dt * dt);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nown; i += (int64_t)gridDim.x * blockDim.x) {
        double q = 0.0, wf = 0.0, qa = 0.0;
        for (int a = 0; a < D; ++a) {
            const double ua = uu[i * D + a], va = vn[i * D + a];
            const double rr = ua - dt * va;
            q += rr * rr;
            wf += ua * m[i] * grav[a];
            qa += ua * ua + dt * dt * va * va;
        }
        red[0] += 0.5 * m[i] * idt2 * q - wf;
        red[1] += 0.5 * m[i] * idt2 * qa + fabs(wf);
    }
    block_reduce_store<2>(red, partials);
}

}  // namespace osmpm
