// grad_sw.cuh -- sliding-window tiled Newton gradient + energy + Jacobi diagonal + linearisation
// cache (a4), the default gradient kernel; same arithmetic as k_grad (tiled.cuh):
//   M = I + grad u, F(u) = M F^n, J = det M det F^n,  Ah = M^{-T},  S' = V0 mu F^n F^nT
//   G_grad = V0 P(F(u)) F^nT = M S' - c' Ah ;  diag_a += gradN^T (S' + (c' + l') Ah_a Ah_a^T) gradN
//   V0 Psi = 1/2 (tr(M S' M^T) - V0 mu d) - V0 mu ln J + V0 lam/2 ln^2 J
// (PAPER.md:151-164 Eq. discrete_energy, 186-191 Eq. F_update, 205-210 Newton).
// Structure of k_hvp_sw (hvp_sw.cuh): per layer, phase 1 (thread per particle) with the particle
// inputs x, F^n, V0 read from the sorted SoA, phase 2 (thread per (cell, a, i)) accumulating the
// gradient and the diagonal in two 3-plane register windows, plane-wise staged fixed-order sums and
// one fp64 RED per node; fp64 arithmetic for every particle precision (R14).
#pragma once
#include "hvp_sw.cuh"

namespace osmpm {

// particle inputs of phase 1: x, F^n, V0 (13 fields in 3D), read straight from the sorted SoA (coalesced)
template <int D> struct GradIn {
    static constexpr int NF = D + D * D + 1;
    __device__ static int field(int f) { return f < D ? PL<D>::X + f : (f < D + D * D ? PL<D>::F + f - D : PL<D>::VOL); }
};

// [16 B][node tile][gradient and diagonal staging][records, per-cell skew].  75 KB in 3D with 8-layer
// tiles: three 144-thread CTAs per SM.  (Streaming the 13 input fields by TMA needs 15 KB more per CTA,
// i.e. two CTAs per SM: measured 34.1 ms per C5 sub-step against 33.0 ms for three CTAs with direct
// loads.)  When deeper tiles would push it past the three-CTA budget, the gradient and the diagonal
// share one staging buffer (flushed one after the other, two more barriers per layer).
template <int D> struct GradLay {
    using T = Tile<D>;
    static constexpr size_t BODY = (size_t)SW<D>::NNP * SVS<D, double>::S + (size_t)GradRec<D>::RS * T::NT +
                                   (size_t)T::LC * 2 /* per-cell record skew, hvp_sw.cuh SWRec::SK */;
    static constexpr bool ONE_STG = 16 + (BODY + 2 * (size_t)SW<D>::STG) * sizeof(double) > 76000;
    static constexpr int NSTG = ONE_STG ? 1 : 2;
};
template <int D, typename R>
constexpr size_t grad_sw_smem_bytes()
{
    return 16 + (GradLay<D>::BODY + (size_t)GradLay<D>::NSTG * SW<D>::STG) * sizeof(double);
}

template <int D, typename R>
__global__ void __launch_bounds__(Tile<D>::NT, 3)
k_grad_sw(const R* __restrict__ P, R* __restrict__ cache, int64_t cap, const int* __restrict__ mat,
          const int* __restrict__ cell_start, BoxDev b, MatTable mt, const double* __restrict__ uin,
          double* __restrict__ gout, double* __restrict__ dout, double* __restrict__ partials,
          double* __restrict__ tbg, double* __restrict__ tbd)
{
    using T = Tile<D>;
    using GR = GradRec<D>;
    using C = CL<D>;
    using In = GradIn<D>;
    using S = SW<D>;
    using Rd = double;
    constexpr int RS = GR::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Rd* sv = reinterpret_cast<Rd*>(smem_raw + 16);
    Rd* stg = sv + S::NNP * SVS<D, Rd>::S;
    constexpr bool ONE = GradLay<D>::ONE_STG;
    Rd* stgd = ONE ? stg : stg + S::STG;
    Rd* rec = stg + GradLay<D>::NSTG * S::STG;
    const int tile = blockIdx.x;
    const int64_t kt = (int64_t)tile * T::NC;
    double red[3] = {0.0, 0.0, 0.0};
    __shared__ int scs[T::NC + 1];
    for (int i = threadIdx.x; i <= T::NC; i += T::NT) scs[i] = cell_start[kt + i];
    __syncthreads();
    if (scs[0] == scs[T::NC]) {
        if (threadIdx.x == 0) partials[blockIdx.x * 3 + 0] = partials[blockIdx.x * 3 + 1] = partials[blockIdx.x * 3 + 2] = 0.0;
        return;
    }
    auto layer_empty = [&](int l) { return scs[l * T::LC] == scs[(l + 1) * T::LC]; };
    int t[3];
    tile_coords<D>(b, tile, t);
    const FlushItem<D, Rd> fli(b, t, nullptr);
    sw_stage_tile<D, Rd, T::NT>(b, t, uin, sv);
    for (int k = threadIdx.x; k < GradLay<D>::NSTG * S::STG; k += T::NT) stg[k] = 0.0;
    __syncthreads();
    const int it = threadIdx.x;
    int icell, icomp, ii;
    item_of<D>(it, icell, icomp, ii);
    Rd acc[S::NACC], accd[S::NACC];
#pragma unroll
    for (int k = 0; k < S::NACC; ++k) acc[k] = accd[k] = 0.0;
    for (int layer = 0; layer < T::NL + 2; ++layer) {
        if (layer < T::NL && !layer_empty(layer)) {
            const int lb = scs[layer * T::LC], le = scs[(layer + 1) * T::LC];
            const int ks = scs[layer * T::LC + icell];
            const int ke = scs[layer * T::LC + icell + 1];
            for (int sb = lb; sb < le; sb += T::NT) {
                const int se = min(sb + T::NT, le);
                const int q = threadIdx.x, p = sb + q;
                if (sb != lb) __syncthreads();
                if (p < se) {
                    auto in = [&](int f) -> Rd { return (Rd)P[(int64_t)In::field(f) * cap + p]; };
                    Rd x[3], w[3][3], dw[3][3];
                    int lc[3] = {0, 0, 0};
#pragma unroll
                    for (int a = 0; a < D; ++a) x[a] = in(a);
                    weights_at<D, Rd>(x, b, t, lc, w, dw);
                    const RecPtr<Rd> r(rec + (D == 3 ? lc[0] * T::T1 + lc[1] : lc[0]) * 2, q, RS);
                    store_weights<D, Rd>(r, w, dw);
                    Rd Mx[D * D];
                    sw_gather<D, Rd>(sv, lc, w, dw, Mx);
#pragma unroll
                    for (int a = 0; a < D; ++a) Mx[a * D + a] += 1.0;
                    Rd Fn[D * D];
#pragma unroll
                    for (int k = 0; k < D * D; ++k) Fn[k] = in(D + k);
                    const Rd V0 = in(D + D * D);
                    const int mid = mat[p];
                    const Rd mu = mt.mu[mid], lam = mt.lam[mid];
                    Rd Sm[Sym<D>::N];
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int bb = a; bb < D; ++bb) {
                            Rd sm = 0;
#pragma unroll
                            for (int k = 0; k < D; ++k) sm = fma(Fn[a * D + k], Fn[bb * D + k], sm);
                            Sm[sym_idx<D>(a, bb)] = V0 * mu * sm;
                        }
                    const Rd detM = det<D, Rd>(Mx), detFn = det<D, Rd>(Fn);
                    Rd Ah[D * D];
                    cofactor<D, Rd>(Mx, Ah);
                    const Rd invdet = 1.0 / detM;
#pragma unroll
                    for (int k = 0; k < D * D; ++k) Ah[k] *= invdet;
                    const bool ok = detM > 0.0 && detFn > 0.0;
                    const Rd lnJ = ok ? log(detM) + log(detFn) : 0.0;
                    const Rd cc = V0 * (mu - lam * lnJ), ll = V0 * lam;
                    Rd trMSM = 0;
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) {
                            Rd sm = 0;
#pragma unroll
                            for (int k = 0; k < D; ++k) sm = fma(Mx[a * D + k], Sm[sym_idx<D>(k, bb)], sm);
                            trMSM = fma(sm, Mx[a * D + bb], trMSM);
                            *r.at(Rec<D>::G + a * D + bb) = fma(-cc, Ah[a * D + bb], sm);
                        }
                    const Rd psiV = 0.5 * (trMSM - V0 * mu * D) - V0 * mu * lnJ + 0.5 * V0 * lam * lnJ * lnJ;
                    red[0] += psiV;
                    red[1] += fabs(psiV);
                    if (!ok) red[2] += 1.0;
#pragma unroll
                    for (int k = 0; k < Sym<D>::N; ++k) {
                        *r.at(GR::S + k) = Sm[k];
                        cache[(C::S + k) * cap + p] = (R)Sm[k];
                    }
#pragma unroll
                    for (int k = 0; k < D * D; ++k) {
                        *r.at(GR::A + k) = Ah[k];
                        cache[(C::A + k) * cap + p] = (R)Ah[k];
                    }
                    cache[C::C * cap + p] = (R)cc;
                    cache[C::L * cap + p] = (R)ll;
                    *r.at(GR::CL) = cc + ll;
                }
                __syncthreads();  // records ready
                if (it < T::ITEMS) {
                    const int p0 = max(ks, sb), p1 = min(ke, se);
                    const int len = p1 - p0;
                    Rd* const cbase = rec + icell * 2 + (p0 - sb) * RS;  // per-cell skew (hvp_sw.cuh SWRec)
                    for (int k = 0; k < len; ++k) {
                        const RecPtr<Rd> r(cbase, k, RS);
                        ItemW<D, Rd> W;
                        W.load(r, ii);
                        Rd sg[D], Ar[D], Q[Sym<D>::N];
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) {
                            sg[bb] = *r.at(Rec<D>::G + icomp * D + bb);
                            Ar[bb] = *r.at(GR::A + icomp * D + bb);
                        }
                        const Rd clv = *r.at(GR::CL);
#pragma unroll
                        for (int a = 0; a < D; ++a)
#pragma unroll
                            for (int bb = a; bb < D; ++bb)
                                Q[sym_idx<D>(a, bb)] = fma(clv * Ar[a], Ar[bb], *r.at(GR::S + sym_idx<D>(a, bb)));
                        item_linear<D, Rd>(sg, W, acc);
                        item_quadratic<D, Rd>(Q, W, accd);
                    }
                }
            }
        }
        double nodot = 0.0;
        double* const tbgl = tbg ? tbg + (int64_t)tile * T::NN * D : nullptr;
        double* const tbdl = tbd ? tbd + (int64_t)tile * T::NN * D : nullptr;
        if constexpr (ONE) {
            if (it < T::ITEMS) sw_emit<D, Rd>(icell, icomp, ii, acc, stg);
            __syncthreads();
            fli.template flush<false>(layer, stg, gout, tbgl, nullptr, nullptr, nodot, nullptr);
            __syncthreads();
            if (it < T::ITEMS) sw_emit<D, Rd>(icell, icomp, ii, accd, stgd);
            __syncthreads();
            fli.template flush<false>(layer, stgd, dout, tbdl, nullptr, nullptr, nodot, nullptr);
        } else {
            if (it < T::ITEMS) {
                sw_emit<D, Rd>(icell, icomp, ii, acc, stg);
                sw_emit<D, Rd>(icell, icomp, ii, accd, stgd);
            }
            __syncthreads();
            fli.template flush<false>(layer, stg, gout, tbgl, nullptr, nullptr, nodot, nullptr);
            fli.template flush<false>(layer, stgd, dout, tbdl, nullptr, nullptr, nodot, nullptr);
        }
        if (layer + 1 >= T::NL || layer_empty(layer + 1)) __syncthreads();
    }
    block_reduce_store<3>(red, partials);
}

}  // namespace osmpm

namespace osmpm {

// a7: line-search energy sum_p V0 Psi(F_p(u)), tiled: one CTA per tile stages u on the
// tile's nodes in shared memory and evaluates Psi for the tile's (contiguous) particles; per-CTA
// partials {sum V0 Psi, sum V0 |Psi|, inverted}.  Same formula as k_energy.
template <int D, typename R>
__global__ void __launch_bounds__(Tile<D>::NT)
k_energy_tiled(const R* __restrict__ P, int64_t cap, const int* __restrict__ mat, const int* __restrict__ cell_start,
               BoxDev b, MatTable mt, const double* __restrict__ u, double* __restrict__ partials)
{
    using T = Tile<D>;
    using L = PL<D>;
    __shared__ double sv[SW<D>::NNP * SVS<D, double>::S];
    const int tile = blockIdx.x;
    const int64_t kt = (int64_t)tile * T::NC;
    const int p_lo = cell_start[kt], p_hi = cell_start[kt + T::NC];
    double red[3] = {0.0, 0.0, 0.0};
    if (p_lo == p_hi) {
        if (threadIdx.x == 0) partials[blockIdx.x * 3 + 0] = partials[blockIdx.x * 3 + 1] = partials[blockIdx.x * 3 + 2] = 0.0;
        return;
    }
    int t[3];
    tile_coords<D>(b, tile, t);
    sw_stage_tile<D, double, T::NT>(b, t, u, sv);
    __syncthreads();
    for (int p = p_lo + threadIdx.x; p < p_hi; p += T::NT) {
        double x[3], w[3][3], dw[3][3], Mx[D * D];
        int lc[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = (double)P[(L::X + a) * cap + p];
        weights_at<D, double>(x, b, t, lc, w, dw);
        sw_gather<D, double>(sv, lc, w, dw, Mx);
#pragma unroll
        for (int a = 0; a < D; ++a) Mx[a * D + a] += 1.0;
        double Fn[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) Fn[k] = (double)P[(L::F + k) * cap + p];
        const double V0 = (double)P[L::VOL * cap + p];
        const int mid = mat[p];
        const double mu = mt.mu[mid], lam = mt.lam[mid];
        const double detM = det<D, double>(Mx), detFn = det<D, double>(Fn);
        if (!(detM > 0.0 && detFn > 0.0)) {
            red[2] += 1.0;
            continue;
        }
        const double lnJ = log(detM) + log(detFn);
        double tr = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int bb = 0; bb < D; ++bb) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) s += Mx[a * D + k] * Fn[k * D + bb];
                tr += s * s;  // |M F^n|_F^2 = tr(M S M^T)
            }
        const double psiV = V0 * (0.5 * mu * (tr - D) - mu * lnJ + 0.5 * lam * lnJ * lnJ);
        red[0] += psiV;
        red[1] += fabs(psiV);
    }
    block_reduce_store<3>(red, partials);
}

}  // namespace osmpm
