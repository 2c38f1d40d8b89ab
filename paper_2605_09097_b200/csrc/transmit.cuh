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

// ---------------------------------------------------------------------------------------------
// Pi numerator / denominator (Eq. spatial_projection) as a GATHER:
//   num_I = sum_j m_j v_j N_B,I(x_j),  den_I = sum_j m_j N_B,I(x_j)   over the active fine nodes j.
// The coarse shape function is a tensor product, N_B,I(x_j) = prod_a N1((x_j,a - x_I,a)/dx_B), and the
// fine nodes form a lattice, so the sum factorises into one 1-D pass per axis (last axis first):
//   pass A  T1[i0][i1][c2] = sum_{i2} N1(.) f(i0,i1,i2),   f = act ? m [v, 1] : 0
//   pass B  T2[i0][c1][c2] = sum_{i1} N1(.) T1[i0][i1][c2]                           (3D only)
//   pass C  num/den[I0,I1,I2] += sum_{i0 owned} N1(.) T2[i0][c1][c2]
// Every output is a fixed-order sum (no atomics: deterministic, and the fine box is read once);
// c_a ranges over the coarse nodes whose support meets the fine box, clipped to the coarse dense box
// (coarse nodes outside it receive nothing, R9).  Ghost planes (i0 >= n0own) belong to
// the neighbour slab and are skipped in pass C.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double bspline_kernel(double t)
{
    const double a = fabs(t);
    if (a < 0.5) return 0.75 - a * a;
    if (a < 1.5) return 0.5 * (1.5 - a) * (1.5 - a);
    return 0.0;
}

// one axis of the factorised sum: coarse node I (global index along the axis) against fine box nodes
// l in [0, n): x_f(l) = xf0 + df l, x_I = oc + dc I
struct PiAxis {
    double xf0, df, oc, dc, inv_dc;
    int n;       // fine box nodes along the axis
    int clo, nc; // coarse range [clo, clo + nc)
};
__device__ __forceinline__ void pi_support(const PiAxis& ax, int I, int& l0, int& l1)
{
    const double xI = ax.oc + ax.dc * (double)I;
    l0 = max(0, (int)ceil((xI - 1.5 * ax.dc - ax.xf0) / ax.df) - 1);
    l1 = min(ax.n - 1, (int)floor((xI + 1.5 * ax.dc - ax.xf0) / ax.df) + 1);
}
__device__ __forceinline__ double pi_weight(const PiAxis& ax, int I, int l)
{
    return bspline_kernel((ax.xf0 + ax.df * (double)l - (ax.oc + ax.dc * (double)I)) * ax.inv_dc);
}

template <int D>
struct PiGeo {
    PiAxis ax[3];
};

// pass A: the last axis, from the fine node fields
template <int D>
__global__ void k_pi_pass_a(PiGeo<D> G, int64_t nout, const uint8_t* __restrict__ act, const double* __restrict__ m,
                            const double* __restrict__ v, double* __restrict__ T1)
{
    constexpr int F = D + 1;
    const PiAxis& A = G.ax[D - 1];
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < nout; o += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(o % A.nc);
        const int64_t row = o / A.nc;  // (i0, i1) in 3D, i0 in 2D
        const int I = A.clo + c;
        int l0, l1;
        pi_support(A, I, l0, l1);
        double acc[F];
#pragma unroll
        for (int k = 0; k < F; ++k) acc[k] = 0.0;
        for (int l = l0; l <= l1; ++l) {
            const int64_t j = row * A.n + l;
            if (!act[j]) continue;
            const double w = pi_weight(A, I, l);
            if (w == 0.0) continue;
            const double mw = m[j] * w;
#pragma unroll
            for (int a = 0; a < D; ++a) acc[a] += mw * v[j * D + a];
            acc[D] += mw;
        }
#pragma unroll
        for (int k = 0; k < F; ++k) T1[o * F + k] = acc[k];
    }
}

// pass B (3D): axis 1.  T1[i0][i1][c2][F] -> T2[i0][c1][c2][F]
__global__ void k_pi_pass_b(PiGeo<3> G, int64_t nout, const double* __restrict__ T1, double* __restrict__ T2)
{
    constexpr int F = 4;
    const PiAxis& A = G.ax[1];
    const int nc2 = G.ax[2].nc;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < nout; o += (int64_t)gridDim.x * blockDim.x) {
        const int c2 = (int)(o % nc2);
        const int c1 = (int)((o / nc2) % A.nc);
        const int64_t i0 = o / ((int64_t)nc2 * A.nc);
        const int I = A.clo + c1;
        int l0, l1;
        pi_support(A, I, l0, l1);
        double acc[F] = {0.0, 0.0, 0.0, 0.0};
        for (int l = l0; l <= l1; ++l) {
            const double w = pi_weight(A, I, l);
            if (w == 0.0) continue;
            const double* t = T1 + ((i0 * A.n + l) * nc2 + c2) * F;
#pragma unroll
            for (int k = 0; k < F; ++k) acc[k] += w * t[k];
        }
#pragma unroll
        for (int k = 0; k < F; ++k) T2[o * F + k] = acc[k];
    }
}

// pass C: axis 0 over the owned planes, added into the coarse dense num (nnb*D) / den (nnb)
template <int D>
__global__ void k_pi_pass_c(PiGeo<D> G, int n0own, const int* __restrict__ gdc, const double* __restrict__ T,
                            double* __restrict__ num, double* __restrict__ den)
{
    constexpr int F = D + 1;
    const PiAxis& A = G.ax[0];
    const int nc1 = G.ax[1].nc, nc2 = (D == 3) ? G.ax[2].nc : 1;
    const int64_t nout = (int64_t)A.nc * nc1 * nc2;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < nout; o += (int64_t)gridDim.x * blockDim.x) {
        const int c2 = (int)(o % nc2);
        const int c1 = (int)((o / nc2) % nc1);
        const int c0 = (int)(o / ((int64_t)nc2 * nc1));
        const int I0 = A.clo + c0;
        int l0, l1;
        pi_support(A, I0, l0, l1);
        l1 = min(l1, n0own - 1);
        double acc[F];
#pragma unroll
        for (int k = 0; k < F; ++k) acc[k] = 0.0;
        for (int l = l0; l <= l1; ++l) {
            const double w = pi_weight(A, I0, l);
            if (w == 0.0) continue;
            const double* t = T + (((int64_t)l * nc1 + c1) * nc2 + c2) * F;
#pragma unroll
            for (int k = 0; k < F; ++k) acc[k] += w * t[k];
        }
        const int I1 = G.ax[1].clo + c1;
        const int64_t I = (D == 3) ? ((int64_t)I0 * gdc[1] + I1) * gdc[2] + (G.ax[2].clo + c2) : (int64_t)I0 * gdc[1] + I1;
#pragma unroll
        for (int a = 0; a < D; ++a) num[I * D + a] += acc[a];
        den[I] += acc[D];
    }
}

// targets of a transmit call must lie in the destination's dense node box; an index outside it is
// skipped (output 0) and latched as INVALID_ARG with its position in the target list
__device__ __forceinline__ bool target_ok(int64_t I, int64_t nmax, ErrLatch* err, int64_t t)
{
    if (I >= 0 && I < nmax) return true;
    latch_error(err, OSMPM_E_INVALID_ARG, t);
    return false;
}

template <int D>
__global__ void k_project_out(int64_t nt, const int64_t* __restrict__ targets, int64_t nnb, const double* __restrict__ num,
                              const double* __restrict__ den, double eps, double* __restrict__ out, ErrLatch* err)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int64_t I = targets ? targets[t] : t;
    if (!target_ok(I, nnb, err, t)) {
#pragma unroll
        for (int a = 0; a < D; ++a) out[t * D + a] = 0.0;
        return;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) out[t * D + a] = num[I * D + a] / (den[I] + eps);
}

// I + T: v_j = (1 - alpha) sum_I v0_I N_I(x_j) + alpha sum_I v1_I N_I(x_j); the coarse fields live
// on the coarse subdomain's box (nodes outside the box carry zero velocity)
template <int D>
__global__ void k_interp(int64_t nt, const int64_t* __restrict__ targets, GridGeo fg, BoxDev cb,
                         const double* __restrict__ v0, const double* __restrict__ v1, double alpha,
                         double* __restrict__ out, ErrLatch* err)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int64_t j = targets ? targets[t] : t;
    const int64_t nfine = (int64_t)fg.gd[0] * fg.gd[1] * (D == 3 ? fg.gd[2] : 1);
    if (!target_ok(j, nfine, err, t)) {
#pragma unroll
        for (int a = 0; a < D; ++a) out[t * D + a] = 0.0;
        return;
    }
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
// fine side may be a group of slabs (each projects its owned nodes, in slab order; sums all-reduced
// over ranks).
template <int D, typename R>
osmpm_status project_accumulate_group(SlabGroup<D, R> F, Sub<D, R>* coarse, bool use_solved, double* num)
{
    cudaStream_t st = F.st;
    const int64_t nnb = coarse->dense_nodes();
    OSMPM_CU(cudaMemsetAsync(num, 0, nnb * (D + 1) * sizeof(double), st));
    double* denp = num + nnb * D;  // num and den contiguous: one all-reduce
    auto& pf = F.ctx->prof;
    if (pf.on) pf.begin("pi", st);
    int* gdc = coarse->pi_gd.p;
    if (!gdc) {
        OSMPM_TRY(coarse->pi_gd.need(3));
        int h[3] = {(int)coarse->gdims[0], (int)coarse->gdims[1], (int)coarse->gdims[2]};
        OSMPM_CU(cudaMemcpy(coarse->pi_gd.p, h, sizeof(h), cudaMemcpyHostToDevice));
        gdc = coarse->pi_gd.p;
    }
    for (int i = 0; i < F.ns; ++i) {
        Sub<D, R>* fine = F.s[i];
        if (fine->box.nnodes == 0 || fine->nown == 0) continue;
        const double* v = use_solved ? fine->vnew.p : fine->vn.p;
        PiGeo<D> G{};
        bool empty = false;
        for (int a = 0; a < D; ++a) {
            PiAxis& A = G.ax[a];
            A.df = fine->box.dx;
            A.xf0 = fine->box.o[a] + fine->box.dx * (double)fine->box.lo[a];
            A.n = fine->box.nn[a];
            A.oc = coarse->origin[a];
            A.dc = coarse->dx;
            A.inv_dc = 1.0 / coarse->dx;
            const double xlo = A.xf0, xhi = A.xf0 + A.df * (A.n - 1);
            const int lo = std::max<int>(0, (int)std::floor((xlo - 1.5 * A.dc - A.oc) / A.dc) - 1);
            const int hi = std::min<int>((int)coarse->gdims[a] - 1, (int)std::ceil((xhi + 1.5 * A.dc - A.oc) / A.dc) + 1);
            A.clo = lo;
            A.nc = hi - lo + 1;
            if (A.nc <= 0) empty = true;
        }
        if (empty) continue;
        const int64_t plane = (D == 3) ? (int64_t)fine->box.nn[1] * fine->box.nn[2] : fine->box.nn[1];
        const int n0own = (int)(fine->nown / plane);
        const int64_t n_a = (D == 3) ? (int64_t)G.ax[0].n * G.ax[1].n * G.ax[2].nc : (int64_t)G.ax[0].n * G.ax[1].nc;
        double* T1 = (double*)F.ctx->get_scratch(4, (size_t)n_a * (D + 1) * sizeof(double));
        if (!T1) return OSMPM_E_OOM;
        fine->KC();
        k_pi_pass_a<D><<<nblk_all(n_a, 256), 256, 0, st>>>(G, n_a, fine->act.p, fine->m.p, v, T1);
        OSMPM_LAUNCH_CHECK();
        const double* Tc = T1;
        if constexpr (D == 3) {
            const int64_t n_b = (int64_t)G.ax[0].n * G.ax[1].nc * G.ax[2].nc;
            double* T2 = (double*)F.ctx->get_scratch(5, (size_t)n_b * 4 * sizeof(double));
            if (!T2) return OSMPM_E_OOM;
            fine->KC();
            k_pi_pass_b<<<nblk_all(n_b, 256), 256, 0, st>>>(G, n_b, T1, T2);
            OSMPM_LAUNCH_CHECK();
            Tc = T2;
        }
        const int64_t n_c = (int64_t)G.ax[0].nc * G.ax[1].nc * (D == 3 ? G.ax[2].nc : 1);
        fine->KC();
        k_pi_pass_c<D><<<nblk_all(n_c, 256), 256, 0, st>>>(G, n0own, gdc, Tc, num, denp);
        OSMPM_LAUNCH_CHECK();
    }
    OSMPM_TRY(group_allreduce<D, R>(F, num, (int)(nnb * (D + 1))));
    if (pf.on) pf.end("pi", st);
    return OSMPM_OK;
}

// the projected coarse values of nt target nodes
template <int D, typename R>
osmpm_status project_out(cudaStream_t st, Sub<D, R>* coarse, int64_t nt, const int64_t* targets, const double* num,
                         const double* den, double eps, double* out)
{
    if (nt <= 0) return OSMPM_OK;
    coarse->KC();
    k_project_out<D><<<nblk_all(nt, 256), 256, 0, st>>>(nt, targets, coarse->dense_nodes(), num, den, eps, out,
                                                        coarse->err.p);
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
        // host targets are checked here; device targets in the kernels (latched, surfaced at the next
        // synchronising call)
        const int64_t nmax = (dir == OSMPM_FINE_TO_COARSE) ? (dstc ? dstc->dense_nodes() : 0) : dst_nodes;
        for (int64_t t = 0; t < nt; ++t)
            if (targets[t] < 0 || targets[t] >= nmax) {
                set_error("transmit: target %lld = node %lld outside the destination node box (%lld nodes)",
                          (long long)t, (long long)targets[t], (long long)nmax);
                return OSMPM_E_INVALID_ARG;
            }
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
            if (src->ctx->prof.on) src->ctx->prof.begin("interp", st);
            src->KC();
            k_interp<D><<<nblk_all(nt, 256), 256, 0, st>>>(nt, tptr, dst_geo, src->box, src->vn.p,
                                                           need_solved ? src->vnew.p : nullptr, alpha, optr,
                                                           src->err.p);
            OSMPM_LAUNCH_CHECK();
            if (src->ctx->prof.on) src->ctx->prof.end("interp", st);
        }
    }
    if (sp == OSMPM_HOST) {
        OSMPM_CU(cudaMemcpyAsync(out, optr, nt * D * sizeof(double), cudaMemcpyDeviceToHost, st));
        OSMPM_CU(cudaStreamSynchronize(st));
    }
    return OSMPM_OK;
}

}  // namespace osmpm
