// p2g_tiled.cuh -- tiled APIC P2G (a2) of mass, momentum and the stress force
// (PAPER.md:171 Eq. p2g_transfer, 178 f_ext, 183 f_int; APIC D_p = dx^2/4 I, R1).
//
//   m_i     = sum_p m_p N_ip
//   (mv)_i  = sum_p m_p N_ip (v_p + (4/dx^2) B_p (x_i - x_p))
//   f^sig_i = -sum_p V0_p P(F_p) F_p^T grad N_ip
//
// Per axis x_i - x_p = dx (l - f) with l the node offset in the stencil and f the particle's
// fractional position, so (mv)_i = sum_p N_ip (c_p + E_p l), c_p = m_p (v_p - (4/dx) B_p f),
// E_p = (4/dx) m_p B_p, and f^sig_i = sum_p G_p grad N_ip with G_p = -V0_p tau_p, tau = P F^T.
// One CTA per tile, layers along the last axis (the tile geometry of the HVP, tiled.cuh):
// phase 1 (thread per particle) writes weights, m, c, E, G to a record; phase 2 (thread per
// (cell, component a, x-offset i)) accumulates the cell's particles in registers; the partials are
// staged per contributing cell (no atomics), summed in a fixed order into shared node tiles, and each
// tile node is written with one fp64 RED per field component at the end.  Replaces 27 x (1 + 2D)
// global REDs per particle of the per-particle scatter (k_p2g).
#pragma once
#include "tiled.cuh"

namespace osmpm {

template <int D> struct P2GRec {
    static constexpr int W = 0, M = 6 * D, CV = M + 1, E = CV + D, G = E + D * D, USED = G + D * D;
    static constexpr int RS = (D == 3) ? 42 : 26;  // odd number of 16-B units
    static_assert(USED <= RS, "record");
};

// staging of one NC-component field: (lateral node, last-axis offset, comp) x NSLOT
template <int D, int NC> struct P2GStage {
    using T = Tile<D>;
    static constexpr int NXY = (D == 3) ? T::N0 * T::N1 : T::N0;
    static constexpr int NSLOT = (D == 3) ? 9 : 3;
    static constexpr int NITEM = NXY * 3 * NC;
    static constexpr int SIZE = NITEM * NSLOT;
};

template <int D, typename R, int NC>
__device__ __forceinline__ void p2g_stage(int cellL, int a, int i, const R* acc, R* stg)
{
    using T = Tile<D>;
    if (D == 3) {
        const int cx = cellL / T::T1, cy = cellL % T::T1;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                const int nxy = (cx + i) * T::N1 + (cy + j);
                stg[((nxy * 3 + kk) * NC + a) * 9 + i * 3 + j] = acc[j * 3 + kk];
            }
    } else {
#pragma unroll
        for (int j = 0; j < 3; ++j) stg[(((cellL + i) * 3 + j) * NC + a) * 3 + i] = acc[j];
    }
}

template <int D, typename R, int NC>
__device__ __forceinline__ void p2g_layer_flush(int layer, const R* stg, R* sy)
{
    using T = Tile<D>;
    using S = P2GStage<D, NC>;
    for (int it = threadIdx.x; it < S::NITEM; it += T::NT) {
        const R* p = stg + it * S::NSLOT;
        R s = p[0];
#pragma unroll
        for (int k = 1; k < S::NSLOT; ++k) s += p[k];
        const int a = it % NC, kk = (it / NC) % 3, nxy = it / (3 * NC);
        sy[((D == 3) ? (nxy * T::N2 + layer + kk) : (nxy * T::N1 + layer + kk)) * NC + a] += s;
    }
}

// tb != nullptr: deterministic mode (hvp_sw.cuh sw_flush): the tile's node block is stored whole
// (tile-local node order, zeros included) for k_det_gather instead of RED-ed
template <int D, typename R, int NC>
__device__ __forceinline__ void p2g_tile_flush(const BoxDev& b, const int* t, const R* sy, double* __restrict__ out,
                                               double* __restrict__ tb = nullptr)
{
    using T = Tile<D>;
    for (int idx = threadIdx.x; idx < T::NN * NC; idx += T::NT) {
        const R s = sy[idx];
        if (tb) {
            tb[idx] = (double)s;
        } else if (s != R(0)) {
            const int a = idx % NC, l = idx / NC;
            int c[3];
            tnode_coords<D>(l, c);
            const int64_t g = box_node<D>(b, t[0] * T::T0 + c[0], t[1] * T::T1 + c[1], t[2] * T::T2 + c[2]);
            atomicAdd(&out[g * NC + a], (double)s);
        }
    }
}

// the three fields (momentum, stress force, mass) are staged together, one zero / stage / flush
// sequence (three barriers) per layer instead of one per field (nine)
template <int D> struct P2GStageAll {
    static constexpr int SP = P2GStage<D, D>::SIZE, SM1 = P2GStage<D, 1>::SIZE;
    static constexpr int SIZE = 2 * SP + SM1;
};

template <int D, typename R>
constexpr size_t p2g_tiled_smem_bytes()
{
    using T = Tile<D>;
    constexpr size_t rec = (size_t)P2GRec<D>::RS * T::NT;
    constexpr size_t stg = ((size_t)P2GStageAll<D>::SIZE + 1) / 2 * 2;  // 16-B multiple for the zeroing
    return ((size_t)T::NN * (1 + 2 * D) + (rec > stg ? rec : stg)) * sizeof(R);
}

#ifndef OSMPM_P2G_MINB
#define OSMPM_P2G_MINB 2
#endif
template <int D, typename R>
__global__ void __launch_bounds__(Tile<D>::NT, OSMPM_P2G_MINB)
k_p2g_tiled(const R* __restrict__ P, int64_t cap, const int* __restrict__ mat, const int* __restrict__ cell_start,
            BoxDev b, MatTable mt, double* __restrict__ m, double* __restrict__ mom, double* __restrict__ fsig,
            double* __restrict__ tbm, double* __restrict__ tbp, double* __restrict__ tbf)
{
    using T = Tile<D>;
    using L = PL<D>;
    using RC = P2GRec<D>;
    constexpr int RS = RC::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* sm = reinterpret_cast<R*>(smem_raw);  // node tiles: m (NN), p (NN*D), f (NN*D)
    R* sp = sm + T::NN;
    R* sf = sp + T::NN * D;
    R* rec = sf + T::NN * D;
    R* stg = rec;  // the staging array reuses the records once phase 2 is done
    const int tile = blockIdx.x;
    const int64_t kt = (int64_t)tile * T::NC;
    __shared__ int scs[T::NC + 1];
    for (int i = threadIdx.x; i <= T::NC; i += T::NT) scs[i] = cell_start[kt + i];
    for (int i = threadIdx.x; i < T::NN * (1 + 2 * D); i += T::NT) sm[i] = R(0);
    __syncthreads();
    if (scs[0] == scs[T::NC]) return;
    int t[3];
    tile_coords<D>(b, tile, t);
    const int it = threadIdx.x;
    const int icell = it / (D * 3), icomp = (it / 3) % D, ii = it % 3;
    const R inv_dx = (R)b.inv_dx;
    for (int layer = 0; layer < T::NL; ++layer) {
        const int lb = scs[layer * T::LC], le = scs[(layer + 1) * T::LC];
        if (lb == le) continue;
        const int ks = scs[layer * T::LC + icell];
        const int ke = scs[layer * T::LC + icell + 1];
        R accp[T::NACC], accf[T::NACC], accm[T::NACC];
#pragma unroll
        for (int k = 0; k < T::NACC; ++k) accp[k] = accf[k] = accm[k] = R(0);
        for (int sb = lb; sb < le; sb += T::NT) {
            const int se = min(sb + T::NT, le);
            const int q = threadIdx.x, p = sb + q;
            if (p < se) {
                R x[3], w[3][3], dw[3][3];
                int lc[3] = {0, 0, 0};
#pragma unroll
                for (int a = 0; a < D; ++a) x[a] = P[(L::X + a) * cap + p];
                weights_at<D, R>(x, b, t, lc, w, dw);
                R f[3];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    R ff;
                    base_of<R>(x[a], b.o[a], b.inv_dx, &ff);
                    f[a] = ff;
                }
                const RecPtr<R> r(rec, q, RS);
                store_weights<D, R>(r, w, dw);
                R F[D * D], B[D * D], v[D];
#pragma unroll
                for (int k = 0; k < D * D; ++k) {
                    F[k] = P[(L::F + k) * cap + p];
                    B[k] = P[(L::B + k) * cap + p];
                }
#pragma unroll
                for (int a = 0; a < D; ++a) v[a] = P[(L::V + a) * cap + p];
                const R mp = P[L::M * cap + p], V0 = P[L::VOL * cap + p];
                const int mid = mat[p];
                const R mu = (R)mt.mu[mid], lam = (R)mt.lam[mid];
                const R lnJ = log(det<D, R>(F));
                const R fourdx = R(4) * inv_dx;
                *r.at(RC::M) = mp;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    R Bf = 0;
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) {
                        Bf = fma(B[a * D + bb], f[bb], Bf);
                        *r.at(RC::E + a * D + bb) = fourdx * mp * B[a * D + bb];
                        // G = -V0 tau, tau = mu F F^T + (lam ln J - mu) I
                        R s = 0;
#pragma unroll
                        for (int k = 0; k < D; ++k) s = fma(F[a * D + k], F[bb * D + k], s);
                        const R tau = mu * s + (a == bb ? lam * lnJ - mu : R(0));
                        *r.at(RC::G + a * D + bb) = -V0 * tau;
                    }
                    *r.at(RC::CV + a) = mp * (v[a] - fourdx * Bf);
                }
            }
            __syncthreads();  // records ready
            if (it < T::ITEMS) {
                const int p0 = max(ks, sb), p1 = min(ke, se);
                const int len = p1 - p0, r7 = icell & 7;
                const int rot = r7 < len ? r7 : (len > 0 ? r7 % len : 0);
                for (int k = 0; k < len; ++k) {
                    const RecPtr<R> r(rec, rotated(p0, len, k, rot) - sb, RS);
                    ItemW<D, R> W;
                    W.load(r, ii);
                    R g[D];
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) g[bb] = *r.at(RC::G + icomp * D + bb);
                    item_linear<D, R>(g, W, accf);
                    const R mp = *r.at(RC::M);
                    const R s0 = fma(*r.at(RC::E + icomp * D + 0), R(ii), *r.at(RC::CV + icomp));
                    if (D == 3) {
                        const R e1 = *r.at(RC::E + icomp * D + 1), e2 = *r.at(RC::E + icomp * D + 2);
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const R wxy = W.wx * W.wy[j];
                            const R tj = fma(e1, R(j), s0);
#pragma unroll
                            for (int kk = 0; kk < 3; ++kk) {
                                const R Nw = wxy * W.wz[kk];
                                accp[j * 3 + kk] = fma(Nw, fma(e2, R(kk), tj), accp[j * 3 + kk]);
                                if (icomp == 0) accm[j * 3 + kk] = fma(Nw, mp, accm[j * 3 + kk]);
                            }
                        }
                    } else {
                        const R e1 = *r.at(RC::E + icomp * D + 1);
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const R Nw = W.wx * W.wy[j];
                            accp[j] = fma(Nw, fma(e1, R(j), s0), accp[j]);
                            if (icomp == 0) accm[j] = fma(Nw, mp, accm[j]);
                        }
                    }
                }
            }
            __syncthreads();  // records consumed
        }
        // momentum, stress force, mass: stage -> fixed-order slot sums -> node tiles
        {
            using SA = P2GStageAll<D>;
            R* stgp = stg;
            R* stgf = stg + SA::SP;
            R* stgm = stg + 2 * SA::SP;
            {
                constexpr int UE = 16 / sizeof(R);
                const int4 z = make_int4(0, 0, 0, 0);
                for (int u = threadIdx.x; u < (SA::SIZE + UE - 1) / UE; u += T::NT) reinterpret_cast<int4*>(stg)[u] = z;
            }
            __syncthreads();
            if (it < T::ITEMS) {
                p2g_stage<D, R, D>(icell, icomp, ii, accp, stgp);
                p2g_stage<D, R, D>(icell, icomp, ii, accf, stgf);
                if (icomp == 0) p2g_stage<D, R, 1>(icell, 0, ii, accm, stgm);
            }
            __syncthreads();
            p2g_layer_flush<D, R, D>(layer, stgp, sp);
            p2g_layer_flush<D, R, D>(layer, stgf, sf);
            p2g_layer_flush<D, R, 1>(layer, stgm, sm);
            __syncthreads();
        }
    }
    const int64_t tn = (int64_t)tile * T::NN;
    p2g_tile_flush<D, R, 1>(b, t, sm, m, tbm ? tbm + tn : nullptr);
    p2g_tile_flush<D, R, D>(b, t, sp, mom, tbp ? tbp + tn * D : nullptr);
    p2g_tile_flush<D, R, D>(b, t, sf, fsig, tbf ? tbf + tn * D : nullptr);
}

}  // namespace osmpm
