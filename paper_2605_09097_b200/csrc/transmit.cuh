// transmit.cuh -- coarse<->fine transmission operators (§3.2.2-3.2.3):
//   Pi_{S->B}  mass-weighted projection, Eq. spatial_projection
//   I_{B->S}   shape-function interpolation, Eq. interp_BtoS
//   T_m        linear temporal interpolation, Eq. temporal_interp
#pragma once
#include "group.cuh"

namespace osmpm {

// coarse quadratic stencil of a point: 3^D (global coarse node index or -1 outside the dense box, N)
template <int D>
__device__ __forceinline__ void coarse_stencil(const double* xp, const double* o, double inv_dx, const int* gd,
                                               int64_t* idx, double* N)
{
    int base[3] = {0, 0, 0};
    double w[3][3], dw[3][3];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double X = (xp[a] - o[a]) * inv_dx;
        double b = floor(X - 0.5);
        base[a] = (int)b;
        bspline<double>(X - b, inv_dx, w[a], dw[a]);
    }
    int c = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < Tile<D>::K3; ++k) {
                int k0 = base[0] + i, k1 = base[1] + j, k2 = (D == 3) ? base[2] + k : 0;
                bool in = k0 >= 0 && k0 < gd[0] && k1 >= 0 && k1 < gd[1] && (D == 2 || (k2 >= 0 && k2 < gd[2]));
                idx[c] = in ? ((D == 3) ? ((int64_t)k0 * gd[1] + k1) * gd[2] + k2 : (int64_t)k0 * gd[1] + k1) : -1;
                N[c] = (D == 3) ? w[0][i] * w[1][j] * w[2][k] : w[0][i] * w[1][j];
                ++c;
            }
}

struct GridGeo {
    double o[3];
    double dx, inv_dx;
    int gd[3];
};

// Pi numerator / denominator: every ACTIVE fine box node scatters m_j [v_j, 1] N_B,I(x_j)
template <int D>
__global__ void k_project(BoxDev fb, int64_t nown, const uint8_t* __restrict__ act, const double* __restrict__ m,
                          const double* __restrict__ v, GridGeo cg, double* __restrict__ num, double* __restrict__ den)
{
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nown || !act[j]) return;  // ghost planes are projected by their owner
    int i2 = (D == 3) ? (int)(j % fb.nn[2]) : 0;
    int i1 = (D == 3) ? (int)((j / fb.nn[2]) % fb.nn[1]) : (int)(j % fb.nn[1]);
    int i0 = (D == 3) ? (int)(j / ((int64_t)fb.nn[2] * fb.nn[1])) : (int)(j / fb.nn[1]);
    const int gi[3] = {fb.lo[0] + i0, fb.lo[1] + i1, fb.lo[2] + i2};
    double xj[3];
#pragma unroll
    for (int a = 0; a < D; ++a) xj[a] = fb.o[a] + fb.dx * (double)gi[a];
    int64_t idx[27];
    double N[27];
    coarse_stencil<D>(xj, cg.o, cg.inv_dx, cg.gd, idx, N);
    const double mj = m[j];
#pragma unroll
    for (int s = 0; s < Tile<D>::NS; ++s) {
        if (idx[s] < 0) continue;
        const double wgt = mj * N[s];
        atomicAdd(&den[idx[s]], wgt);
#pragma unroll
        for (int a = 0; a < D; ++a) atomicAdd(&num[idx[s] * D + a], wgt * v[j * D + a]);
    }
}

template <int D>
__global__ void k_project_out(int64_t nt, const int64_t* __restrict__ targets, const double* __restrict__ num,
                              const double* __restrict__ den, double eps, double* __restrict__ out)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int64_t I = targets ? targets[t] : t;
#pragma unroll
    for (int a = 0; a < D; ++a) out[t * D + a] = num[I * D + a] / (den[I] + eps);
}

// ---------------------------------------------------------------------------------------------
// Affine variant of Pi (OSMPM_PI=affine; R21, NOT the paper's operator): the same weights
// w_j = m_j N_B,I(x_j) feed the normal equations of the weighted least-squares affine fit
// v ~ a + B xi, xi = (x_j - x_I)/dx_B, and the coarse value is a -- exact for affine fields under any
// fine masses (the paper's support-wide mean is exact only for uniform masses, which biases the
// rotation a bending section transmits).  Moments per coarse node: the symmetric (1+D)^2 matrix
// (upper triangle, AF<D>::NA) and the (1+D) x D right-hand sides.
template <int D> struct AF {
    static constexpr int K = 1 + D, NA = K * (K + 1) / 2, NM = NA + K * D;
    static __host__ __device__ constexpr int ai(int r, int q) { return r * K - r * (r - 1) / 2 + (q - r); }  // r <= q
};
static inline bool pi_affine()
{
    const char* e = getenv("OSMPM_PI");
    return e && std::string(e) == "affine";
}
template <int D>
__global__ void k_project_affine(BoxDev fb, int64_t nown, const uint8_t* __restrict__ act, const double* __restrict__ m,
                                 const double* __restrict__ v, GridGeo cg, double* __restrict__ mom)
{
    using A = AF<D>;
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nown || !act[j]) return;
    int i2 = (D == 3) ? (int)(j % fb.nn[2]) : 0;
    int i1 = (D == 3) ? (int)((j / fb.nn[2]) % fb.nn[1]) : (int)(j % fb.nn[1]);
    int i0 = (D == 3) ? (int)(j / ((int64_t)fb.nn[2] * fb.nn[1])) : (int)(j / fb.nn[1]);
    const int gi[3] = {fb.lo[0] + i0, fb.lo[1] + i1, fb.lo[2] + i2};
    double xj[3];
#pragma unroll
    for (int a = 0; a < D; ++a) xj[a] = fb.o[a] + fb.dx * (double)gi[a];
    int64_t idx[27];
    double N[27];
    coarse_stencil<D>(xj, cg.o, cg.inv_dx, cg.gd, idx, N);
    const double mj = m[j];
    for (int s = 0; s < Tile<D>::NS; ++s) {
        const int64_t I = idx[s];
        if (I < 0) continue;
        int kI[3] = {0, 0, 0};
        if (D == 3) {
            kI[2] = (int)(I % cg.gd[2]);
            kI[1] = (int)((I / cg.gd[2]) % cg.gd[1]);
            kI[0] = (int)(I / ((int64_t)cg.gd[2] * cg.gd[1]));
        } else {
            kI[1] = (int)(I % cg.gd[1]);
            kI[0] = (int)(I / cg.gd[1]);
        }
        double phi[A::K];
        phi[0] = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) phi[1 + a] = (xj[a] - (cg.o[a] + cg.dx * (double)kI[a])) * cg.inv_dx;
        const double w = mj * N[s];
        double* mo = mom + I * A::NM;
#pragma unroll
        for (int r = 0; r < A::K; ++r) {
#pragma unroll
            for (int q = r; q < A::K; ++q) atomicAdd(&mo[A::ai(r, q)], w * phi[r] * phi[q]);
#pragma unroll
            for (int a = 0; a < D; ++a) atomicAdd(&mo[A::NA + r * D + a], w * phi[r] * v[j * D + a]);
        }
    }
}

// solve the normal equations of each target coarse node (Gaussian elimination with partial pivoting);
// a node whose fine support does not span D dimensions keeps the mass-weighted mean num / (den + eps)
template <int D>
__global__ void k_project_out_affine(int64_t nt, const int64_t* __restrict__ targets, const double* __restrict__ num,
                                     const double* __restrict__ den, const double* __restrict__ mom, double eps,
                                     double* __restrict__ out)
{
    using A = AF<D>;
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int64_t I = targets ? targets[t] : t;
    const double* mo = mom + I * A::NM;
    double M[A::K][A::K], rhs[A::K][D];
#pragma unroll
    for (int r = 0; r < A::K; ++r) {
#pragma unroll
        for (int q = 0; q < A::K; ++q) M[r][q] = mo[A::ai(r < q ? r : q, r < q ? q : r)];
#pragma unroll
        for (int a = 0; a < D; ++a) rhs[r][a] = mo[A::NA + r * D + a];
    }
#pragma unroll
    for (int a = 0; a < D; ++a) out[t * D + a] = num[I * D + a] / (den[I] + eps);
    const double s0 = M[0][0];
    if (!(s0 > 0.0)) return;
    M[0][0] += eps;
    for (int col = 0; col < A::K; ++col) {
        int piv = col;
        for (int r = col + 1; r < A::K; ++r)
            if (fabs(M[r][col]) > fabs(M[piv][col])) piv = r;
        if (!(fabs(M[piv][col]) > 1e-4 * s0)) return;  // the fit would amplify rounding: keep the mean
        if (piv != col) {
            for (int q = 0; q < A::K; ++q) {
                const double tq = M[col][q];
                M[col][q] = M[piv][q];
                M[piv][q] = tq;
            }
            for (int a = 0; a < D; ++a) {
                const double ta = rhs[col][a];
                rhs[col][a] = rhs[piv][a];
                rhs[piv][a] = ta;
            }
        }
        for (int r = col + 1; r < A::K; ++r) {
            const double f = M[r][col] / M[col][col];
            for (int q = col; q < A::K; ++q) M[r][q] -= f * M[col][q];
            for (int a = 0; a < D; ++a) rhs[r][a] -= f * rhs[col][a];
        }
    }
    double sol[A::K][D];
    for (int r = A::K - 1; r >= 0; --r)
        for (int a = 0; a < D; ++a) {
            double tv = rhs[r][a];
            for (int q = r + 1; q < A::K; ++q) tv -= M[r][q] * sol[q][a];
            sol[r][a] = tv / M[r][r];
        }
#pragma unroll
    for (int a = 0; a < D; ++a) out[t * D + a] = sol[0][a];
}

// I + T: v_j = (1 - alpha) sum_I v0_I N_I(x_j) + alpha sum_I v1_I N_I(x_j); the coarse fields live
// on the coarse subdomain's box (nodes outside the box carry zero velocity)
template <int D>
__global__ void k_interp(int64_t nt, const int64_t* __restrict__ targets, GridGeo fg, BoxDev cb,
                         const double* __restrict__ v0, const double* __restrict__ v1, double alpha,
                         double* __restrict__ out)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int64_t j = targets ? targets[t] : t;
    int g2 = (D == 3) ? (int)(j % fg.gd[2]) : 0;
    int g1 = (D == 3) ? (int)((j / fg.gd[2]) % fg.gd[1]) : (int)(j % fg.gd[1]);
    int g0 = (D == 3) ? (int)(j / ((int64_t)fg.gd[2] * fg.gd[1])) : (int)(j / fg.gd[1]);
    const int gi[3] = {g0, g1, g2};
    double xj[3];
#pragma unroll
    for (int a = 0; a < D; ++a) xj[a] = fg.o[a] + fg.dx * (double)gi[a];
    int64_t idx[27];
    double N[27];
    coarse_stencil<D>(xj, cb.o, cb.inv_dx, cb.gdims, idx, N);
    double I0[3] = {0, 0, 0}, I1[3] = {0, 0, 0};
#pragma unroll
    for (int s = 0; s < Tile<D>::NS; ++s) {
        if (idx[s] < 0) continue;
        const int64_t I = idx[s];
        int k2 = (D == 3) ? (int)(I % cb.gdims[2]) : 0;
        int k1 = (D == 3) ? (int)((I / cb.gdims[2]) % cb.gdims[1]) : (int)(I % cb.gdims[1]);
        int k0 = (D == 3) ? (int)(I / ((int64_t)cb.gdims[2] * cb.gdims[1])) : (int)(I / cb.gdims[1]);
        int l0 = k0 - cb.lo[0], l1 = k1 - cb.lo[1], l2 = (D == 3) ? k2 - cb.lo[2] : 0;
        if (l0 < 0 || l1 < 0 || l2 < 0 || l0 >= cb.nn[0] || l1 >= cb.nn[1] || (D == 3 && l2 >= cb.nn[2])) continue;
        const int64_t bi = box_node<D>(cb, l0, l1, l2);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            I0[a] += v0[bi * D + a] * N[s];
            if (v1) I1[a] += v1[bi * D + a] * N[s];
        }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) out[t * D + a] = (1.0 - alpha) * I0[a] + alpha * I1[a];
}

template <typename S>
static GridGeo geo_of(const S* s)
{
    GridGeo g{};
    for (int a = 0; a < 3; ++a) {
        g.o[a] = s->origin[a];
        g.gd[a] = (int)s->gdims[a];
    }
    g.dx = s->dx;
    g.inv_dx = 1.0 / s->dx;
    return g;
}

// Pi over ALL coarse dense nodes: num (nnB*D), den (nnB) device buffers of the coarse side.  The
// fine side may be a group of slabs (each projects its owned nodes; sums all-reduced over ranks).
template <int D, typename R>
osmpm_status project_accumulate_group(SlabGroup<D, R> F, Sub<D, R>* coarse, bool use_solved, double* num)
{
    cudaStream_t st = F.st;
    const int64_t nnb = coarse->dense_nodes();
    OSMPM_CU(cudaMemsetAsync(num, 0, nnb * (D + 1) * sizeof(double), st));
    double* denp = num + nnb * D;  // num and den contiguous: one all-reduce
    auto& pf = F.ctx->prof;
    if (pf.on) pf.begin("transmit", st);
    for (int i = 0; i < F.ns; ++i) {
        Sub<D, R>* fine = F.s[i];
        const double* v = use_solved ? fine->vnew.p : fine->vn.p;
        fine->KC();
        k_project<D><<<nblk_all(fine->box.nnodes, 256), 256, 0, st>>>(fine->box, fine->nown, fine->act.p, fine->m.p, v,
                                                                      geo_of(coarse), num, denp);
        OSMPM_LAUNCH_CHECK();
    }
    OSMPM_TRY(group_allreduce<D, R>(F, num, (int)(nnb * (D + 1))));
    if (pi_affine()) {
        OSMPM_TRY(coarse->pi_mom.need((size_t)nnb * AF<D>::NM));
        OSMPM_CU(cudaMemsetAsync(coarse->pi_mom.p, 0, nnb * AF<D>::NM * sizeof(double), st));
        for (int i = 0; i < F.ns; ++i) {
            Sub<D, R>* fine = F.s[i];
            const double* v = use_solved ? fine->vnew.p : fine->vn.p;
            fine->KC();
            k_project_affine<D><<<nblk_all(fine->box.nnodes, 256), 256, 0, st>>>(
                fine->box, fine->nown, fine->act.p, fine->m.p, v, geo_of(coarse), coarse->pi_mom.p);
            OSMPM_LAUNCH_CHECK();
        }
        OSMPM_TRY(group_allreduce<D, R>(F, coarse->pi_mom.p, (int)(nnb * AF<D>::NM)));
    }
    if (pf.on) pf.end("transmit", st);
    return OSMPM_OK;
}

// the projected coarse values of nt target nodes (Pi, or its affine variant under OSMPM_PI=affine)
template <int D, typename R>
osmpm_status project_out(cudaStream_t st, Sub<D, R>* coarse, int64_t nt, const int64_t* targets, const double* num,
                         const double* den, double eps, double* out)
{
    if (nt <= 0) return OSMPM_OK;
    coarse->KC();
    if (pi_affine())
        k_project_out_affine<D><<<nblk_all(nt, 256), 256, 0, st>>>(nt, targets, num, den, coarse->pi_mom.p, eps, out);
    else
        k_project_out<D><<<nblk_all(nt, 256), 256, 0, st>>>(nt, targets, num, den, eps, out);
    OSMPM_LAUNCH_CHECK();
    return OSMPM_OK;
}
template <int D, typename R>
osmpm_status project_accumulate(Sub<D, R>* fine, Sub<D, R>* coarse, bool use_solved, DBuf<double>& num,
                                DBuf<double>& den)
{
    const int64_t nnb = coarse->dense_nodes();
    OSMPM_TRY(num.need(nnb * (D + 1)));
    OSMPM_TRY(project_accumulate_group<D, R>(fine->self_group(), coarse, use_solved, num.p));
    // den as its own buffer for the coupler's host reads
    OSMPM_TRY(den.need(nnb));
    OSMPM_CU(cudaMemcpyAsync(den.p, num.p + nnb * D, nnb * sizeof(double), cudaMemcpyDeviceToDevice, fine->st()));
    return OSMPM_OK;
}

// src / dst: a standalone subdomain (Sub) or, on the fine side, a slab group.  FINE_TO_COARSE reads
// the source's (group's) grid and writes coarse values; COARSE_TO_FINE reads the coarse source's grid
// and only the destination's geometry.
template <int D, typename R>
osmpm_status transmit_impl(SlabGroup<D, R> SG, Sub<D, R>* src, Sub<D, R>* dstc, GridGeo dst_geo, int64_t dst_nodes,
                           osmpm_direction dir, double alpha, double eps, int64_t nt, const int64_t* targets,
                           double* out, osmpm_memspace sp)
{
    cudaStream_t st = SG.st;
    for (int i = 0; i < SG.ns; ++i)
        if (!SG.s[i]->have_grid) {
            set_error("transmit: source subdomain has no grid (call osmpm_p2g)");
            return OSMPM_E_STATE;
        }
    if (alpha < 0.0 || alpha > 1.0) {
        set_error("transmit: alpha = %g outside [0, 1] (m > M, SPEC.md:330)", alpha);
        return OSMPM_E_INVALID_ARG;
    }
    const bool need_solved = alpha > 0.0;
    for (int i = 0; i < SG.ns; ++i)
        if (need_solved && !SG.s[i]->have_vnew) {
            set_error("transmit: alpha > 0 needs the source's solved grid velocity");
            return OSMPM_E_STATE;
        }
    if (!targets && nt != dst_nodes) {
        set_error("transmit: targets == NULL requires n_targets == dst node count (%lld)", (long long)dst_nodes);
        return OSMPM_E_INVALID_ARG;
    }
    osmpm_ctx* cx = SG.ctx;
    const int64_t* tptr = targets;
    if (targets && sp == OSMPM_HOST) {
        int64_t* tg = (int64_t*)cx->get_scratch(0, nt * sizeof(int64_t));
        if (!tg) return OSMPM_E_OOM;
        OSMPM_CU(cudaMemcpyAsync(tg, targets, nt * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        tptr = tg;
    }
    double* optr = out;
    if (sp == OSMPM_HOST) {
        optr = (double*)cx->get_scratch(1, nt * D * sizeof(double));
        if (!optr) return OSMPM_E_OOM;
    }
    if (dir == OSMPM_FINE_TO_COARSE) {
        if (alpha != 0.0 && alpha != 1.0) {
            set_error("transmit FINE_TO_COARSE: alpha selects v^n (0) or v^{n+1} (1)");
            return OSMPM_E_INVALID_ARG;
        }
        if (!dstc) {
            set_error("transmit FINE_TO_COARSE: the coarse subdomain must not be decomposed");
            return OSMPM_E_INVALID_ARG;
        }
        double* num = (double*)cx->get_scratch(2, dstc->dense_nodes() * (D + 1) * sizeof(double));
        if (!num) return OSMPM_E_OOM;
        OSMPM_TRY(project_accumulate_group<D, R>(SG, dstc, alpha == 1.0, num));
        OSMPM_TRY(project_out<D, R>(st, dstc, nt, tptr, num, num + dstc->dense_nodes() * D, eps, optr));
    } else {
        if (!src) {
            set_error("transmit COARSE_TO_FINE: the coarse subdomain must not be decomposed");
            return OSMPM_E_INVALID_ARG;
        }
        if (nt > 0) {
            if (src->ctx->prof.on) src->ctx->prof.begin("transmit", st);
            src->KC();
            k_interp<D><<<nblk_all(nt, 256), 256, 0, st>>>(nt, tptr, dst_geo, src->box, src->vn.p,
                                                           need_solved ? src->vnew.p : nullptr, alpha, optr);
            OSMPM_LAUNCH_CHECK();
            if (src->ctx->prof.on) src->ctx->prof.end("transmit", st);
        }
    }
    if (sp == OSMPM_HOST) {
        OSMPM_CU(cudaMemcpyAsync(out, optr, nt * D * sizeof(double), cudaMemcpyDeviceToHost, st));
        OSMPM_CU(cudaStreamSynchronize(st));
    }
    return OSMPM_OK;
}

}  // namespace osmpm
