/*
 * osmpm_oracle.c -- plain, slow, fp64 CPU oracle of the OS-MPM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2605_09097_b200/) never links, imports or executes it, and shares no
 * source, header, table or helper with it.
 *
 * Source of truth: /root/reference/PAPER.md (arXiv 2605.09097).  Where the paper is
 * silent we take the readings listed in SURVEY.md §8(c).2 (Z1-Z35) and DESIGN.md §2.
 * Each function cites the passage it follows.  Everything is written as the plain
 * definition: loops over particles in creation order and nodes in lexicographic
 * order, no blocking, no fusion, no reordering.  Compile with -O2 -ffp-contract=off.
 *
 * Conventions
 *   dim d in {2,3}; node box n[0..2] (n[2]=1 in 2D); node (k0,k1,k2) has linear index
 *   (k0*n1 + k1)*n2 + k2 and position x_i = o + dx*k (Eq. interpolation).
 *   Particle p: x[p*d+a], v[p*d+a], F[p*d*d + a*d + b] (row-major), B likewise, m[p], V0[p],
 *   mat[p] (material id), bnd[p] (boundary flag P^∂).
 *   Node vectors: [node*d + a].  Materials: E[k], nu[k].
 *
 * Parity-pin status of every exported function: see oracle/README in DESIGN.md §4;
 * every function below is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t d;
    double o[3];
    double dx;
    int64_t n[3];
} orc_grid;

typedef struct {
    int32_t max_newton, max_cg, fixed_iters, guess;
    double newton_rtol, newton_atol, cg_rtol, ls_min_alpha, energy_noise_rtol;
    int32_t cg_variant; /* 0: standard Jacobi PCG; 1: single-reduction (Chronopoulos-Gear) */
    int32_t psd;        /* PSD projection of the per-particle tangent blocks (R23):
                           0 never, 1 when the Newton direction fails the descent check, 2 always */
} orc_newton_settings;

typedef struct {
    int32_t newton_iters, cg_iters, ls_halvings, status;
    double grad_norm0, grad_norm, energy;
    /* events that change what a solve returns (R7, R8): PCG solves cut short by
     * non-positive curvature; fixed-iteration Newton steps whose line search found no decrease
     * (alpha = 0 taken); converged solves accepted at the energy round-off floor */
    int32_t negcurv, ls_failures, floor_accept, psd_solves; /* psd_solves: PCG solves run with the
                                                             projected tangent (R23) */
} orc_solve_stats;

enum { ORC_OK = 0, ORC_OUT_OF_DOMAIN = 1, ORC_INVERTED = 2, ORC_NEWTON_NC = 3, ORC_LS_STAGNATION = 4 };

/* ------------------------------------------------------------------------------------------ */
/* O1: quadratic B-spline (App. B.1).  f = X - base in [1/2, 3/2).               */
/* ------------------------------------------------------------------------------------------ */
void orc_bspline1(double f, double dx, double* w, double* dw)
{
    w[0] = 0.5 * (1.5 - f) * (1.5 - f);
    w[1] = 0.75 - (f - 1.0) * (f - 1.0);
    w[2] = 0.5 * (f - 0.5) * (f - 0.5);
    dw[0] = (f - 1.5) / dx;
    dw[1] = -2.0 * (f - 1.0) / dx;
    dw[2] = (f - 0.5) / dx;
}

static int64_t nidx(const orc_grid* g, const int64_t* k)
{
    if (g->d == 3) return (k[0] * g->n[1] + k[1]) * g->n[2] + k[2];
    return k[0] * g->n[1] + k[1];
}

static int64_t n_nodes(const orc_grid* g)
{
    return g->d == 3 ? g->n[0] * g->n[1] * g->n[2] : g->n[0] * g->n[1];
}

/* Stencil of a point x: node indices, N_i(x), grad N_i(x), x_i - x.  Returns the number of
 * stencil nodes (3^d), or -1 if x is outside the safe interior (base >= 0 and
 * base + 2 <= n - 1).  PAPER.md:128 (Eq. interpolation). */
int orc_stencil(const orc_grid* g, const double* x, int64_t* idx, double* N, double* gN, double* xip)
{
    int d = g->d;
    int64_t base[3] = {0, 0, 0};
    double w[3][3], dw[3][3];
    for (int a = 0; a < d; ++a) {
        double X = (x[a] - g->o[a]) / g->dx;
        base[a] = (int64_t)floor(X - 0.5);
        double f = X - (double)base[a];
        if (base[a] < 0 || base[a] + 2 > g->n[a] - 1) return -1;
        orc_bspline1(f, g->dx, w[a], dw[a]);
    }
    int c = 0;
    int n2 = (d == 3) ? 3 : 1;
    for (int i0 = 0; i0 < 3; ++i0)
        for (int i1 = 0; i1 < 3; ++i1)
            for (int i2 = 0; i2 < n2; ++i2) {
                int64_t k[3] = {base[0] + i0, base[1] + i1, base[2] + i2};
                idx[c] = nidx(g, k);
                if (d == 3) {
                    N[c] = w[0][i0] * w[1][i1] * w[2][i2];
                    gN[c * 3 + 0] = dw[0][i0] * w[1][i1] * w[2][i2];
                    gN[c * 3 + 1] = w[0][i0] * dw[1][i1] * w[2][i2];
                    gN[c * 3 + 2] = w[0][i0] * w[1][i1] * dw[2][i2];
                } else {
                    N[c] = w[0][i0] * w[1][i1];
                    gN[c * 2 + 0] = dw[0][i0] * w[1][i1];
                    gN[c * 2 + 1] = w[0][i0] * dw[1][i1];
                }
                for (int a = 0; a < d; ++a) xip[c * d + a] = (g->o[a] + g->dx * (double)k[a]) - x[a];
                ++c;
            }
    return c;
}

/* Same stencil, but nodes outside the box are reported with idx = -1 instead of failing
 * (used by the coarse<->fine transmission, where a fine node may sit near the coarse box edge). */
static int stencil_partial(const orc_grid* g, const double* x, int64_t* idx, double* N)
{
    int d = g->d;
    int64_t base[3] = {0, 0, 0};
    double w[3][3], dw[3][3];
    for (int a = 0; a < d; ++a) {
        double X = (x[a] - g->o[a]) / g->dx;
        base[a] = (int64_t)floor(X - 0.5);
        orc_bspline1(X - (double)base[a], g->dx, w[a], dw[a]);
    }
    int c = 0;
    int n2 = (d == 3) ? 3 : 1;
    for (int i0 = 0; i0 < 3; ++i0)
        for (int i1 = 0; i1 < 3; ++i1)
            for (int i2 = 0; i2 < n2; ++i2) {
                int64_t k[3] = {base[0] + i0, base[1] + i1, base[2] + i2};
                int inside = 1;
                for (int a = 0; a < d; ++a)
                    if (k[a] < 0 || k[a] > g->n[a] - 1) inside = 0;
                idx[c] = inside ? nidx(g, k) : -1;
                N[c] = (d == 3) ? w[0][i0] * w[1][i1] * w[2][i2] : w[0][i0] * w[1][i1];
                ++c;
            }
    return c;
}

/* ------------------------------------------------------------------------------------------ */
/* small dense linear algebra (d x d, row-major)                                              */
/* ------------------------------------------------------------------------------------------ */
static double det_d(int d, const double* A)
{
    if (d == 2) return A[0] * A[3] - A[1] * A[2];
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}

/* inverse transpose A^{-T} by the adjugate */
static void inv_T(int d, const double* A, double* R)
{
    double J = det_d(d, A);
    if (d == 2) {
        /* A^{-1} = [[a3, -a1], [-a2, a0]] / J ; transpose */
        R[0] = A[3] / J;
        R[1] = -A[2] / J;
        R[2] = -A[1] / J;
        R[3] = A[0] / J;
        return;
    }
    /* cofactor matrix C_ab = (-1)^{a+b} M_ab ; A^{-T} = C / J */
    R[0] = (A[4] * A[8] - A[5] * A[7]) / J;
    R[1] = -(A[3] * A[8] - A[5] * A[6]) / J;
    R[2] = (A[3] * A[7] - A[4] * A[6]) / J;
    R[3] = -(A[1] * A[8] - A[2] * A[7]) / J;
    R[4] = (A[0] * A[8] - A[2] * A[6]) / J;
    R[5] = -(A[0] * A[7] - A[1] * A[6]) / J;
    R[6] = (A[1] * A[5] - A[2] * A[4]) / J;
    R[7] = -(A[0] * A[5] - A[2] * A[3]) / J;
    R[8] = (A[0] * A[4] - A[1] * A[3]) / J;
}

static void matmul(int d, const double* A, const double* B, double* C)
{
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            double s = 0.0;
            for (int c = 0; c < d; ++c) s += A[a * d + c] * B[c * d + b];
            C[a * d + b] = s;
        }
}

static void transpose(int d, const double* A, double* T)
{
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) T[a * d + b] = A[b * d + a];
}

/* ------------------------------------------------------------------------------------------ */
/* O3: Neo-Hookean ("Neo-Hookean"; form per SPEC.md:160 / SURVEY.md Z4)           */
/*   Psi = mu/2 (F:F - d) - mu ln J + lam/2 (ln J)^2                                           */
/*   P   = mu F + (lam ln J - mu) F^{-T}                                                        */
/*   dP  = mu dF + (mu - lam ln J) F^{-T} dF^T F^{-T} + lam (F^{-T}:dF) F^{-T}                  */
/* ------------------------------------------------------------------------------------------ */
void orc_lame(double E, double nu, double* mu, double* lam)
{
    *mu = E / (2.0 * (1.0 + nu));
    *lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
}

double orc_psi(int d, const double* F, double mu, double lam)
{
    double J = det_d(d, F);
    if (!(J > 0.0)) return INFINITY;
    double FF = 0.0;
    for (int i = 0; i < d * d; ++i) FF += F[i] * F[i];
    double lnJ = log(J);
    return 0.5 * mu * (FF - (double)d) - mu * lnJ + 0.5 * lam * lnJ * lnJ;
}

void orc_P(int d, const double* F, double mu, double lam, double* P)
{
    double FiT[9];
    inv_T(d, F, FiT);
    double lnJ = log(det_d(d, F));
    for (int i = 0; i < d * d; ++i) P[i] = mu * F[i] + (lam * lnJ - mu) * FiT[i];
}

void orc_dP(int d, const double* F, const double* dF, double mu, double lam, double* dP)
{
    double A[9], dFT[9], T1[9], T2[9];
    inv_T(d, F, A);
    double lnJ = log(det_d(d, F));
    transpose(d, dF, dFT);
    matmul(d, A, dFT, T1);
    matmul(d, T1, A, T2);
    double AdF = 0.0;
    for (int i = 0; i < d * d; ++i) AdF += A[i] * dF[i];
    for (int i = 0; i < d * d; ++i) dP[i] = mu * dF[i] + (mu - lam * lnJ) * T2[i] + lam * AdF * A[i];
}

/* PSD projection of the per-particle tangent block ("per-particle tangent blocks are
 * eigen-projected to positive semidefinite"; R23).  The block is the d^2 x d^2 matrix
 * T = d^2 Psi / dF dF (symmetric: a Hessian) acting on vec(dF), row-major vec; its columns are orc_dP
 * of the unit directions.  T = Q diag(l) Q^T by cyclic Jacobi rotations (plain, to convergence), then
 * T+ = Q diag(max(l, 0)) Q^T, and dP = T+ vec(dF). */
static void sym_eig_jacobi(int n, double* A, double* Q)
{
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) Q[i * n + j] = (i == j) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                if (i == j) diag += A[i * n + i] * A[i * n + i];
                else off += A[i * n + j] * A[i * n + j];
            }
        if (off <= 1e-32 * diag) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double apq = A[p * n + q];
                if (apq == 0.0) continue;
                double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
                double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int k = 0; k < n; ++k) { /* A <- J^T A J, columns p, q then rows p, q */
                    double akp = A[k * n + p], akq = A[k * n + q];
                    A[k * n + p] = c * akp - sn * akq;
                    A[k * n + q] = sn * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    double apk = A[p * n + k], aqk = A[q * n + k];
                    A[p * n + k] = c * apk - sn * aqk;
                    A[q * n + k] = sn * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    double qkp = Q[k * n + p], qkq = Q[k * n + q];
                    Q[k * n + p] = c * qkp - sn * qkq;
                    Q[k * n + q] = sn * qkp + c * qkq;
                }
            }
    }
}

void orc_tangent_psd(int d, const double* F, double mu, double lam, double* Tp)
{
    int n = d * d;
    double T[81], Q[81], E[9] = {0}, col[9];
    for (int k = 0; k < n; ++k) {
        memset(E, 0, sizeof(E));
        E[k] = 1.0;
        orc_dP(d, F, E, mu, lam, col);
        for (int i = 0; i < n; ++i) T[i * n + k] = col[i];
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double a = 0.5 * (T[i * n + j] + T[j * n + i]);
            T[i * n + j] = T[j * n + i] = a;
        }
    sym_eig_jacobi(n, T, Q);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) {
                double l = T[k * n + k];
                if (l > 0.0) s += Q[i * n + k] * l * Q[j * n + k];
            }
            Tp[i * n + j] = s;
        }
}

void orc_dP_psd(int d, const double* F, const double* dF, double mu, double lam, double* dP)
{
    int n = d * d;
    double Tp[81];
    orc_tangent_psd(d, F, mu, lam, Tp);
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = 0; k < n; ++k) s += Tp[i * n + k] * dF[k];
        dP[i] = s;
    }
}

static void tangent_apply(int psd, int d, const double* F, const double* dF, double mu, double lam, double* dP)
{
    if (psd) orc_dP_psd(d, F, dF, mu, lam, dP);
    else orc_dP(d, F, dF, mu, lam, dP);
}

static int cmp_double(const void* a, const void* b)
{
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

double orc_median(int64_t n, const double* v)
{
    if (n <= 0) return 0.0;
    double* c = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(c, v, sizeof(double) * (size_t)n);
    qsort(c, (size_t)n, sizeof(double), cmp_double);
    double r = (n % 2) ? c[n / 2] : 0.5 * (c[n / 2 - 1] + c[n / 2]);
    free(c);
    return r;
}

/* ------------------------------------------------------------------------------------------ */
/* O2: APIC P2G of mass, momentum, body force and stress.                                      */
/*   m_i = sum_p m_p N_ip ;  (mv)_i = sum_p m_p N_ip (v_p + B_p D_p^{-1} (x_i - x_p)),          */
/*   D_p = (dx^2/4) I  (Eq. p2g_transfer)                           */
/*   f_ext,i = sum_p m_p g N_ip                                                 */
/*   f^sigma_i = - sum_p V0_p (P_p F_p^T) grad N_ip                             */
/*   active_i <=> m_i > 1e-12 * median_p m_p; v_i = (mv)_i / m_i               */
/* Outputs are dense over the node box and overwritten.  Returns ORC_OK or ORC_OUT_OF_DOMAIN   */
/* (then *bad = offending particle).                                                          */
/* ------------------------------------------------------------------------------------------ */
int orc_p2g(const orc_grid* g, int64_t np, const double* x, const double* v, const double* F,
            const double* B, const double* m, const double* V0, const int32_t* mat,
            const double* E, const double* nu, const double* grav,
            double* mi, double* pi, double* vi, double* fext, double* fsig, uint8_t* active,
            int64_t* bad)
{
    int d = g->d;
    int64_t nn = n_nodes(g);
    memset(mi, 0, sizeof(double) * (size_t)nn);
    memset(pi, 0, sizeof(double) * (size_t)(nn * d));
    memset(fsig, 0, sizeof(double) * (size_t)(nn * d));
    int64_t idx[27];
    double N[27], gN[81], xip[81];
    double Dinv = 4.0 / (g->dx * g->dx);
    for (int64_t p = 0; p < np; ++p) {
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) {
            if (bad) *bad = p;
            return ORC_OUT_OF_DOMAIN;
        }
        double mu, lam, P[9], FT[9], tau[9];
        orc_lame(E[mat[p]], nu[mat[p]], &mu, &lam);
        orc_P(d, F + p * d * d, mu, lam, P);
        transpose(d, F + p * d * d, FT);
        matmul(d, P, FT, tau);
        const double* Bp = B + p * d * d;
        for (int s = 0; s < c; ++s) {
            int64_t i = idx[s];
            mi[i] += m[p] * N[s];
            for (int a = 0; a < d; ++a) {
                double aff = 0.0;
                for (int b = 0; b < d; ++b) aff += Bp[a * d + b] * Dinv * xip[s * d + b];
                pi[i * d + a] += m[p] * N[s] * (v[p * d + a] + aff);
                double t = 0.0;
                for (int b = 0; b < d; ++b) t += tau[a * d + b] * gN[s * d + b];
                fsig[i * d + a] -= V0[p] * t;
            }
        }
    }
    double thr = 1e-12 * orc_median(np, m);
    for (int64_t i = 0; i < nn; ++i) {
        active[i] = mi[i] > thr;
        for (int a = 0; a < d; ++a) {
            vi[i * d + a] = active[i] ? pi[i * d + a] / mi[i] : 0.0;
            fext[i * d + a] = mi[i] * grav[a];
        }
    }
    return ORC_OK;
}

/* Boundary-particle mass m^∂_i = sum_{p in P^∂} m_p N_ip (Eq. boundary_grid_set) */
int orc_boundary_mass(const orc_grid* g, int64_t np, const double* x, const double* m,
                      const uint8_t* bnd, double* mb)
{
    int d = g->d;
    int64_t nn = n_nodes(g);
    memset(mb, 0, sizeof(double) * (size_t)nn);
    int64_t idx[27];
    double N[27], gN[81], xip[81];
    for (int64_t p = 0; p < np; ++p) {
        if (!bnd[p]) continue;
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) return ORC_OUT_OF_DOMAIN;
        for (int s = 0; s < c; ++s) mb[idx[s]] += m[p] * N[s];
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* F_p(u) = (I + sum_i u_i grad N_ip^T) F_p^n   (Eq. F_update; u = xhat - x^n)  */
/* ------------------------------------------------------------------------------------------ */
static void F_of_u(int d, int c, const int64_t* idx, const double* gN, const double* u,
                   const double* Fn, double* Fu)
{
    double G[9];
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            double s = (a == b) ? 1.0 : 0.0;
            for (int t = 0; t < c; ++t) s += u[idx[t] * d + a] * gN[t * d + b];
            G[a * d + b] = s;
        }
    matmul(d, G, Fn, Fu);
}

/* ------------------------------------------------------------------------------------------ */
/* O4: incremental potential (Eq. discrete_energy) in u = xhat - x^n:            */
/*   E(u) = sum_i m_i/(2dt^2) |u_i - dt v_i^n|^2 + sum_p V0 Psi(F_p(u)) - sum_i u_i . f_ext,i  */
/* (xhat - xtilde = u - dt v^n; the constant -sum_i x_i^n . f_ext,i is dropped: DESIGN.md R3).  */
/* E_abs is the same sum of absolute term values (noise scale of the line search, Z10).        */
/* ------------------------------------------------------------------------------------------ */
int orc_energy(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
               const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
               const double* vn, const double* fext, const double* u, double* Eout, double* Eabs)
{
    int d = g->d;
    int64_t nn = n_nodes(g);
    double e = 0.0, ea = 0.0;
    for (int64_t i = 0; i < nn; ++i) {
        double q = 0.0, w = 0.0, qa = 0.0;
        for (int a = 0; a < d; ++a) {
            double r = u[i * d + a] - dt * vn[i * d + a];
            q += r * r;
            w += u[i * d + a] * fext[i * d + a];
            qa += u[i * d + a] * u[i * d + a] + dt * dt * vn[i * d + a] * vn[i * d + a];
        }
        e += mi[i] / (2.0 * dt * dt) * q - w;
        /* round-off scale of the inertia term |u - dt v|^2 is |u|^2 + |dt v|^2 (R8) */
        ea += mi[i] / (2.0 * dt * dt) * qa + fabs(w);
    }
    int64_t idx[27];
    double N[27], gN[81], xip[81], Fu[9];
    int inverted = 0;
    for (int64_t p = 0; p < np; ++p) {
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) return ORC_OUT_OF_DOMAIN;
        double mu, lam;
        orc_lame(E[mat[p]], nu[mat[p]], &mu, &lam);
        F_of_u(d, c, idx, gN, u, F + p * d * d, Fu);
        double psi = orc_psi(d, Fu, mu, lam);
        if (isinf(psi)) inverted = 1;
        e += V0[p] * psi;
        ea += V0[p] * fabs(psi);
    }
    *Eout = inverted ? INFINITY : e;
    if (Eabs) *Eabs = ea;
    return ORC_OK;
}

/* gradient g_i = m_i/dt^2 (u_i - dt v_i^n) - f_ext,i + sum_p V0 P(F_p(u)) F_p^{nT} grad N_ip
 * (derivative of orc_energy; f_int = -dPhi/dxhat). Dense over all node DOFs. */
int orc_gradient(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
                 const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
                 const double* vn, const double* fext, const double* u, double* gout)
{
    int d = g->d;
    int64_t nn = n_nodes(g);
    for (int64_t i = 0; i < nn; ++i)
        for (int a = 0; a < d; ++a)
            gout[i * d + a] = mi[i] / (dt * dt) * (u[i * d + a] - dt * vn[i * d + a]) - fext[i * d + a];
    int64_t idx[27];
    double N[27], gN[81], xip[81], Fu[9], P[9], FnT[9], PFnT[9];
    for (int64_t p = 0; p < np; ++p) {
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) return ORC_OUT_OF_DOMAIN;
        double mu, lam;
        orc_lame(E[mat[p]], nu[mat[p]], &mu, &lam);
        F_of_u(d, c, idx, gN, u, F + p * d * d, Fu);
        if (!(det_d(d, Fu) > 0.0)) return ORC_INVERTED;
        orc_P(d, Fu, mu, lam, P);
        transpose(d, F + p * d * d, FnT);
        matmul(d, P, FnT, PFnT);
        for (int s = 0; s < c; ++s)
            for (int a = 0; a < d; ++a) {
                double t = 0.0;
                for (int b = 0; b < d; ++b) t += PFnT[a * d + b] * gN[s * d + b];
                gout[idx[s] * d + a] += V0[p] * t;
            }
    }
    return ORC_OK;
}

/* O5: Hessian-vector product of E at u along dvec ((M/dt^2 + K) with
 * K = Hessian of Phi; K via Eq. F_update):
 *   y_i = m_i/dt^2 d_i + sum_p V0 dP(F_p(u); dF_p) F_p^{nT} grad N_ip,
 *   dF_p = (sum_j d_j grad N_jp^T) F_p^n.
 * `node_mask` (may be NULL) restricts the output to masked nodes (sampled full-size parity):
 * only particles whose stencil touches a masked node are visited; the rest of y is zero. */
int orc_hvp_ex(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
               const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
               const double* u, const double* dvec, const uint8_t* node_mask, double* y, int psd)
{
    int d = g->d;
    int64_t nn = n_nodes(g);
    for (int64_t i = 0; i < nn; ++i)
        for (int a = 0; a < d; ++a)
            y[i * d + a] = (node_mask == NULL || node_mask[i]) ? mi[i] / (dt * dt) * dvec[i * d + a] : 0.0;
    int64_t idx[27];
    double N[27], gN[81], xip[81], Fu[9], G[9], dF[9], dP[9], FnT[9], dPFnT[9];
    for (int64_t p = 0; p < np; ++p) {
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) return ORC_OUT_OF_DOMAIN;
        if (node_mask) {
            int touch = 0;
            for (int s = 0; s < c; ++s) touch |= node_mask[idx[s]];
            if (!touch) continue;
        }
        double mu, lam;
        orc_lame(E[mat[p]], nu[mat[p]], &mu, &lam);
        const double* Fn = F + p * d * d;
        F_of_u(d, c, idx, gN, u, Fn, Fu);
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                double s = 0.0;
                for (int t = 0; t < c; ++t) s += dvec[idx[t] * d + a] * gN[t * d + b];
                G[a * d + b] = s;
            }
        matmul(d, G, Fn, dF);
        tangent_apply(psd, d, Fu, dF, mu, lam, dP);
        transpose(d, Fn, FnT);
        matmul(d, dP, FnT, dPFnT);
        for (int s = 0; s < c; ++s) {
            if (node_mask && !node_mask[idx[s]]) continue;
            for (int a = 0; a < d; ++a) {
                double t = 0.0;
                for (int b = 0; b < d; ++b) t += dPFnT[a * d + b] * gN[s * d + b];
                y[idx[s] * d + a] += V0[p] * t;
            }
        }
    }
    return ORC_OK;
}

int orc_hvp(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
            const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
            const double* u, const double* dvec, const uint8_t* node_mask, double* y)
{
    return orc_hvp_ex(g, np, x, F, V0, mat, E, nu, dt, mi, u, dvec, node_mask, y, 0);
}

/* O6: Jacobi diagonal, by definition diag_{i,a} = e_{i,a}^T H e_{i,a}:
 *   m_i/dt^2 + sum_p V0 (e_a h^T) : dP(F_p(u); e_a h^T),  h = F_p^{nT} grad N_ip.            */
int orc_diag_ex(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
                const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
                const double* u, double* diag, int psd)
{
    int d = g->d;
    int64_t nn = n_nodes(g);
    for (int64_t i = 0; i < nn; ++i)
        for (int a = 0; a < d; ++a) diag[i * d + a] = mi[i] / (dt * dt);
    int64_t idx[27];
    double N[27], gN[81], xip[81], Fu[9], dF[9], dP[9];
    for (int64_t p = 0; p < np; ++p) {
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) return ORC_OUT_OF_DOMAIN;
        double mu, lam;
        orc_lame(E[mat[p]], nu[mat[p]], &mu, &lam);
        const double* Fn = F + p * d * d;
        F_of_u(d, c, idx, gN, u, Fn, Fu);
        for (int s = 0; s < c; ++s) {
            double h[3];
            for (int b = 0; b < d; ++b) {
                double t = 0.0;
                for (int e = 0; e < d; ++e) t += Fn[e * d + b] * gN[s * d + e]; /* (F^{nT} gradN)_b */
                h[b] = t;
            }
            for (int a = 0; a < d; ++a) {
                memset(dF, 0, sizeof(dF));
                for (int b = 0; b < d; ++b) dF[a * d + b] = h[b];
                tangent_apply(psd, d, Fu, dF, mu, lam, dP);
                double q = 0.0;
                for (int k = 0; k < d * d; ++k) q += dF[k] * dP[k];
                diag[idx[s] * d + a] += V0[p] * q;
            }
        }
    }
    return ORC_OK;
}

int orc_diag(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
             const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
             const double* u, double* diag)
{
    return orc_diag_ex(g, np, x, F, V0, mat, E, nu, dt, mi, u, diag, 0);
}

/* ------------------------------------------------------------------------------------------ */
/* O7: backward-Euler Newton with Jacobi-PCG and backtracking line search                      */
/* (§2.2.5; linear solver / tolerances / guess per SURVEY.md Z6-Z11).        */
/* free_mask[DOF] = 1 for unknown DOFs (active and not Dirichlet).  u holds on entry the        */
/* prescribed values of the non-free DOFs (dt * v_D on Dirichlet DOFs, 0 on inactive ones) and */
/* on exit the solution; free DOFs are initialised here (guess 0: dt v^n = xtilde; 1: 0).       */
/* ------------------------------------------------------------------------------------------ */
static double dot_free(int64_t n, const uint8_t* fm, const double* a, const double* b)
{
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k)
        if (fm[k]) s += a[k] * b[k];
    return s;
}

/* Single-reduction Jacobi PCG (Chronopoulos & Gear 1989; R22): the same Krylov iterates as
 * the standard PCG in exact arithmetic, with the two inner products of an iteration taken together
 * after the one Hessian-vector product, so a distributed solve needs one reduction per iteration.
 * Iteration k (one HVP each, max_cg in all):
 *   [tolerance mode: stop if |r_k| <= cg_rtol |g|]
 *   u_k = diag^-1 r_k,  w_k = H u_k,  gamma_k = (r_k, u_k),  delta_k = (w_k, u_k)
 *   k = 0: beta = 0, c = delta_0;  k > 0: beta = gamma_k / gamma_{k-1}, c = delta_k - beta gamma_k / alpha_{k-1}
 *   (c = p_k^T H p_k); c <= 0: non-positive curvature -> stop (k = 0: x = u_0)  [R7]
 *   alpha_k = gamma_k / c,  p_k = u_k + beta p_{k-1},  s_k = w_k + beta s_{k-1}  (= H p_k)
 *   x_{k+1} = x_k + alpha_k p_k,  r_{k+1} = r_k - alpha_k s_k
 * Arrays: xs (x), r, z (u), pv (p), q (w), ut (s), all over nd DOFs. */
static int pcg_single_reduction(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
                                const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
                                const double* u, const double* gr, const double* dg, const uint8_t* free_mask,
                                const orc_newton_settings* st, double gn, int64_t nd, double* xs, double* r, double* z,
                                double* pv, double* q, double* sv, orc_solve_stats* stats, int psd)
{
    for (int64_t k = 0; k < nd; ++k) {
        xs[k] = 0.0;
        r[k] = free_mask[k] ? -gr[k] : 0.0;
        pv[k] = 0.0;
        sv[k] = 0.0;
    }
    double gamma_old = 0.0, alpha_old = 0.0;
    for (int cg = 0; cg < st->max_cg; ++cg) {
        double rn = sqrt(dot_free(nd, free_mask, r, r));
        if (!st->fixed_iters && rn <= st->cg_rtol * gn) break;
        for (int64_t k = 0; k < nd; ++k) z[k] = free_mask[k] ? r[k] / dg[k] : 0.0;
        int rc = orc_hvp_ex(g, np, x, F, V0, mat, E, nu, dt, mi, u, z, NULL, q, psd);
        if (rc) return rc;
        for (int64_t k = 0; k < nd; ++k)
            if (!free_mask[k]) q[k] = 0.0;
        stats->cg_iters++;
        double gamma = dot_free(nd, free_mask, r, z);
        double delta = dot_free(nd, free_mask, q, z);
        double beta = (cg == 0 || !(gamma_old > 0.0)) ? 0.0 : gamma / gamma_old;
        double c = (cg == 0) ? delta : delta - beta * gamma / alpha_old;
        if (!(c > 0.0)) {
            if (cg == 0)
                for (int64_t k = 0; k < nd; ++k) xs[k] = z[k];
            stats->negcurv++;
            break;
        }
        double alpha = gamma / c;
        for (int64_t k = 0; k < nd; ++k) {
            pv[k] = z[k] + beta * pv[k];
            sv[k] = q[k] + beta * sv[k];
            xs[k] += alpha * pv[k];
            r[k] -= alpha * sv[k];
        }
        gamma_old = gamma;
        alpha_old = alpha;
    }
    return ORC_OK;
}

/* Standard Jacobi PCG on H dx = -g over the free DOFs (stops per DESIGN.md R6, R7). */
static int pcg_standard(const orc_grid* g, int64_t np, const double* x, const double* F, const double* V0,
                        const int32_t* mat, const double* E, const double* nu, double dt, const double* mi,
                        const double* u, const double* gr, const double* dg, const uint8_t* free_mask,
                        const orc_newton_settings* st, double gn, int64_t nd, double* xs, double* r, double* z,
                        double* pv, double* q, orc_solve_stats* stats, int psd)
{
    int rc;
    for (int64_t k = 0; k < nd; ++k) {
        xs[k] = 0.0;
        r[k] = free_mask[k] ? -gr[k] : 0.0;
        z[k] = r[k] / dg[k];
        pv[k] = z[k];
    }
    double rz = dot_free(nd, free_mask, r, z);
    for (int cg = 0; cg < st->max_cg; ++cg) {
        double rn = sqrt(dot_free(nd, free_mask, r, r));
        if (!st->fixed_iters && rn <= st->cg_rtol * gn) break;
        rc = orc_hvp_ex(g, np, x, F, V0, mat, E, nu, dt, mi, u, pv, NULL, q, psd);
        if (rc) return rc;
        for (int64_t k = 0; k < nd; ++k)
            if (!free_mask[k]) q[k] = 0.0;
        stats->cg_iters++;
        double pq = dot_free(nd, free_mask, pv, q);
        if (!(pq > 0.0)) {
            /* non-positive curvature: stop with the current iterate, or the preconditioned
             * steepest-descent direction -diag^-1 g if it is the first (R7; the same in
             * fixed-iteration mode, whose remaining iterations then leave xs unchanged) */
            if (cg == 0)
                for (int64_t k = 0; k < nd; ++k) xs[k] = z[k];
            stats->negcurv++;
            break;
        }
        double alpha = rz / pq;
        for (int64_t k = 0; k < nd; ++k) {
            xs[k] += alpha * pv[k];
            r[k] -= alpha * q[k];
            z[k] = free_mask[k] ? r[k] / dg[k] : 0.0;
        }
        double rz_new = dot_free(nd, free_mask, r, z);
        double beta = (rz > 0.0) ? rz_new / rz : 0.0;
        rz = rz_new;
        for (int64_t k = 0; k < nd; ++k) pv[k] = z[k] + beta * pv[k];
    }
    return ORC_OK;
}

int orc_implicit_solve(const orc_grid* g, int64_t np, const double* x, const double* F,
                       const double* V0, const int32_t* mat, const double* E, const double* nu,
                       double dt, const double* mi, const double* vn, const double* fext,
                       const uint8_t* free_mask, const orc_newton_settings* st, double* u,
                       orc_solve_stats* stats)
{
    int d = g->d;
    int64_t nd = n_nodes(g) * d;
    double* gr = (double*)calloc((size_t)nd, sizeof(double));
    double* dg = (double*)calloc((size_t)nd, sizeof(double));
    double* xs = (double*)calloc((size_t)nd, sizeof(double));
    double* r = (double*)calloc((size_t)nd, sizeof(double));
    double* z = (double*)calloc((size_t)nd, sizeof(double));
    double* pv = (double*)calloc((size_t)nd, sizeof(double));
    double* q = (double*)calloc((size_t)nd, sizeof(double));
    double* ut = (double*)calloc((size_t)nd, sizeof(double));
    int rc = ORC_OK;
    memset(stats, 0, sizeof(*stats));
    for (int64_t k = 0; k < nd; ++k)
        if (free_mask[k]) u[k] = (st->guess == 1) ? 0.0 : dt * vn[k];
    double g0 = 0.0;
    int converged = 0;
    /* natural force scale f_s = || m_i (|v_i^n| / dt + |g|) || over the free DOFs: the Newton test is
     * relative to max(|g^(0)|, f_s) so that a state already at equilibrium counts as converged
     * (R6) */
    double fs = 0.0;
    for (int64_t k = 0; k < nd; ++k)
        if (free_mask[k]) {
            double t = mi[k / d] * fabs(vn[k]) / dt + fabs(fext[k]);
            fs += t * t;
        }
    fs = sqrt(fs);
    double gref = 0.0;
    for (int it = 0; it < st->max_newton; ++it) {
        rc = orc_gradient(g, np, x, F, V0, mat, E, nu, dt, mi, vn, fext, u, gr);
        if (rc) goto done;
        for (int64_t k = 0; k < nd; ++k)
            if (!free_mask[k]) gr[k] = 0.0;
        double gn = sqrt(dot_free(nd, free_mask, gr, gr));
        if (it == 0) {
            g0 = gn;
            gref = g0 > fs ? g0 : fs;
        }
        stats->grad_norm = gn;
        if (!st->fixed_iters && (gn <= st->newton_rtol * gref || gn <= st->newton_atol)) {
            converged = 1;
            break;
        }
        /* the Newton direction: Jacobi PCG (standard or single-reduction, R22), with the per-particle
         * tangent blocks projected to PSD always (psd = 2) or, psd = 1, in a second solve when the first
         * direction fails the descent check g . dx < 0 (R23) */
        for (int psd_now = (st->psd == 2);;) {
            rc = orc_diag_ex(g, np, x, F, V0, mat, E, nu, dt, mi, u, dg, psd_now);
            if (rc) goto done;
            for (int64_t k = 0; k < nd; ++k)
                if (!free_mask[k]) dg[k] = 1.0;
            /* projected solves use the standard PCG (as the GPU path, whose projected HVP yields no
             * single-reduction curvature partials) */
            if (st->cg_variant == 1 && !psd_now)
                rc = pcg_single_reduction(g, np, x, F, V0, mat, E, nu, dt, mi, u, gr, dg, free_mask, st, gn, nd, xs,
                                          r, z, pv, q, ut, stats, psd_now);
            else
                rc = pcg_standard(g, np, x, F, V0, mat, E, nu, dt, mi, u, gr, dg, free_mask, st, gn, nd, xs, r, z,
                                  pv, q, stats, psd_now);
            if (rc) goto done;
            if (psd_now) stats->psd_solves++;
            if (st->psd == 1 && !psd_now && !(dot_free(nd, free_mask, gr, xs) < 0.0)) {
                psd_now = 1;
                continue;
            }
            break;
        }
        /* backtracking line search: halve alpha from 1 until E decreases (Z10) */
        double E0, Ea0, Et, Eat;
        rc = orc_energy(g, np, x, F, V0, mat, E, nu, dt, mi, vn, fext, u, &E0, &Ea0);
        if (rc) goto done;
        double alpha = 1.0;
        int at_floor = 0;
        for (;;) {
            for (int64_t k = 0; k < nd; ++k) ut[k] = free_mask[k] ? u[k] + alpha * xs[k] : u[k];
            rc = orc_energy(g, np, x, F, V0, mat, E, nu, dt, mi, vn, fext, ut, &Et, &Eat);
            if (rc) goto done;
            if (Et < E0 || (isfinite(Et) && fabs(Et - E0) <= st->energy_noise_rtol * Ea0)) break;
            alpha *= 0.5;
            stats->ls_halvings++;
            if (alpha < st->ls_min_alpha) {
                /* fixed-iteration mode (timing): no decrease found -> take alpha = 0 (u unchanged),
                 * count it and go on, so the work per solve stays fixed (R8) */
                if (st->fixed_iters) {
                    at_floor = 2;
                    break;
                }
                /* no decrease of E_h is resolvable any more: once |g| has dropped below
                 * sqrt(rtol) * gref the iterate is accepted as converged at the roundoff floor of
                 * E_h (R8), otherwise the stagnation is an error */
                if (gn <= sqrt(st->newton_rtol) * gref) {
                    at_floor = 1;
                    break;
                }
                rc = ORC_LS_STAGNATION;
                goto done;
            }
        }
        if (at_floor == 1) {
            stats->floor_accept = 1;
            converged = 1;
            break;
        }
        if (at_floor == 2) {
            stats->ls_failures++;
        } else {
            memcpy(u, ut, sizeof(double) * (size_t)nd);
            stats->energy = Et;
        }
        stats->newton_iters = it + 1;
    }
    if (!st->fixed_iters && !converged) {
        /* final check after the last update */
        rc = orc_gradient(g, np, x, F, V0, mat, E, nu, dt, mi, vn, fext, u, gr);
        if (rc) goto done;
        for (int64_t k = 0; k < nd; ++k)
            if (!free_mask[k]) gr[k] = 0.0;
        double gn = sqrt(dot_free(nd, free_mask, gr, gr));
        stats->grad_norm = gn;
        if (!(gn <= st->newton_rtol * gref || gn <= st->newton_atol)) rc = ORC_NEWTON_NC;
    }
done:
    stats->grad_norm0 = g0;
    stats->status = rc;
    free(gr); free(dg); free(xs); free(r); free(z); free(pv); free(q); free(ut);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* O8: APIC G2P + F update + advection (Eqs. g2p_v, g2p_B, F_update,         */
/* advection; substep forms PAPER.md:416-423).  vg: grid velocity v^{n+1} (dense).             */
/* ------------------------------------------------------------------------------------------ */
int orc_g2p(const orc_grid* g, int64_t np, double* x, double* v, double* F, double* B,
            const double* vg, double dt, int64_t* bad)
{
    int d = g->d;
    int64_t idx[27];
    double N[27], gN[81], xip[81];
    for (int64_t p = 0; p < np; ++p) {
        int c = orc_stencil(g, x + p * d, idx, N, gN, xip);
        if (c < 0) {
            if (bad) *bad = p;
            return ORC_OUT_OF_DOMAIN;
        }
        double vp[3] = {0, 0, 0}, Bp[9] = {0}, gv[9] = {0};
        for (int s = 0; s < c; ++s)
            for (int a = 0; a < d; ++a) {
                double va = vg[idx[s] * d + a];
                vp[a] += N[s] * va;
                for (int b = 0; b < d; ++b) {
                    Bp[a * d + b] += N[s] * va * xip[s * d + b];
                    gv[a * d + b] += va * gN[s * d + b];
                }
            }
        double Lm[9], Fn[9];
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) Lm[a * d + b] = (a == b ? 1.0 : 0.0) + dt * gv[a * d + b];
        matmul(d, Lm, F + p * d * d, Fn);
        if (!(det_d(d, Fn) > 0.0)) {
            if (bad) *bad = p;
            return ORC_INVERTED;
        }
        memcpy(F + p * d * d, Fn, sizeof(double) * (size_t)(d * d));
        memcpy(B + p * d * d, Bp, sizeof(double) * (size_t)(d * d));
        for (int a = 0; a < d; ++a) {
            v[p * d + a] = vp[a];
            x[p * d + a] += dt * vp[a];
        }
        /* the advected position must stay in the safe interior (SPEC.md:123 advect "errors") */
        if (orc_stencil(g, x + p * d, idx, N, gN, xip) < 0) {
            if (bad) *bad = p;
            return ORC_OUT_OF_DOMAIN;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* O9: Pi_{S->B} (Eq. spatial_projection): for every coarse node I,              */
/*   num_I = sum_{j in N_S active} m_S,j v_S,j N_B,I(x_S,j),  den_I = sum_j m_S,j N_B,I(x_S,j) */
/*   v_B,I = num_I / (den_I + eps_tol).                                                         */
/* Coarse stencil nodes outside the coarse box receive nothing (R9).                 */
/* ------------------------------------------------------------------------------------------ */
int orc_project(const orc_grid* gs, const double* ms, const double* vs, const uint8_t* act_s,
                const orc_grid* gb, double eps_tol, double* num, double* den, double* vb)
{
    int d = gs->d;
    int64_t nns = n_nodes(gs), nnb = n_nodes(gb);
    memset(num, 0, sizeof(double) * (size_t)(nnb * d));
    memset(den, 0, sizeof(double) * (size_t)nnb);
    int64_t idx[27];
    double N[27];
    for (int64_t j = 0; j < nns; ++j) {
        if (!act_s[j]) continue;
        int64_t k[3];
        if (d == 3) {
            k[0] = j / (gs->n[1] * gs->n[2]);
            k[1] = (j / gs->n[2]) % gs->n[1];
            k[2] = j % gs->n[2];
        } else {
            k[0] = j / gs->n[1];
            k[1] = j % gs->n[1];
            k[2] = 0;
        }
        double xj[3];
        for (int a = 0; a < d; ++a) xj[a] = gs->o[a] + gs->dx * (double)k[a];
        int c = stencil_partial(gb, xj, idx, N);
        for (int s = 0; s < c; ++s) {
            if (idx[s] < 0) continue;
            den[idx[s]] += ms[j] * N[s];
            for (int a = 0; a < d; ++a) num[idx[s] * d + a] += ms[j] * vs[j * d + a] * N[s];
        }
    }
    for (int64_t i = 0; i < nnb; ++i)
        for (int a = 0; a < d; ++a) vb[i * d + a] = num[i * d + a] / (den[i] + eps_tol);
    return ORC_OK;
}

/* O10: I_{B->S} (Eq. interp_BtoS) at the fine node positions `targets`, applied
 * to both endpoint fields (Eq. spatial_interp_n), then T_m with weight alpha
 * (Eq. temporal_interp): v = (1 - alpha) I(v_B^n) + alpha I(v_B^{n+1}). */
int orc_interp(const orc_grid* gb, const double* vb0, const double* vb1, double alpha,
               const orc_grid* gs, int64_t nt, const int64_t* targets, double* vout)
{
    int d = gb->d;
    int64_t idx[27];
    double N[27];
    for (int64_t t = 0; t < nt; ++t) {
        int64_t j = targets[t], k[3];
        if (d == 3) {
            k[0] = j / (gs->n[1] * gs->n[2]);
            k[1] = (j / gs->n[2]) % gs->n[1];
            k[2] = j % gs->n[2];
        } else {
            k[0] = j / gs->n[1];
            k[1] = j % gs->n[1];
            k[2] = 0;
        }
        double xj[3];
        for (int a = 0; a < d; ++a) xj[a] = gs->o[a] + gs->dx * (double)k[a];
        int c = stencil_partial(gb, xj, idx, N);
        double I0[3] = {0, 0, 0}, I1[3] = {0, 0, 0};
        for (int s = 0; s < c; ++s) {
            if (idx[s] < 0) continue;
            for (int a = 0; a < d; ++a) {
                I0[a] += vb0[idx[s] * d + a] * N[s];
                I1[a] += vb1[idx[s] * d + a] * N[s];
            }
        }
        for (int a = 0; a < d; ++a) vout[t * d + a] = (1.0 - alpha) * I0[a] + alpha * I1[a];
    }
    return ORC_OK;
}
