// hvp_ws.cuh -- warp-specialised, persistent Hessian-vector product (a5).
//
// Same arithmetic as k_hvp (tiled.cuh): y += sum_p G_p grad N, G_p = gd S' + c' Ah gd^T Ah + l' (Ah:gd) Ah.
// Work unit = (tile, layer, sub-chunk of <= CAP particles).  One persistent CTA per SM walks its tiles;
// three warp roles are connected by mbarrier rings instead of CTA-wide barriers:
//   loader warp   TMA bulk copies (cp.async.bulk) of each unit's particle inputs (x + Newton cache)
//                 into an NIN-slot input ring; the tile's node values (d) into a 2-slot node ring
//   gather warps  NG warps, one particle per lane: weights, tensor-product gather, G_p -> record ring
//   scatter warps one (cell, component, x-offset) item per lane: register accumulation over the
//                 cell's particles; per layer the partials are staged node-major and summed into the
//                 scatter warps' node tile (named barrier among the scatter warps only); per tile one
//                 fp64 RED per node and component.
#pragma once
#include "tiled.cuh"

namespace osmpm {

template <int D> struct WS {
    using T = Tile<D>;
    static constexpr int NG = 4;                       // gather warps
    static constexpr int CAP = NG * 32;                // particles per unit
    static constexpr int NS = (T::ITEMS + 31) / 32;    // scatter warps
    static constexpr int NWARP = 1 + NG + NS;
    static constexpr int NTHR = 32 * NWARP;
    static constexpr int NIN = 4;                      // input ring slots
    static constexpr int NREC = 2;                     // record ring slots
    static constexpr int NVS = 4;                      // node-tile ring slots
};

template <int D, typename R> struct WSLayout {
    using T = Tile<D>;
    using W = WS<D>;
    static constexpr int NF = D + CL<D>::NF;
    static constexpr int UE = 16 / sizeof(R);
    static constexpr int PFS = W::CAP + 2 * UE;
    static constexpr int RS = HvpRec<D, R>::RS;
    // mbarriers: in_full[NIN], in_empty[NIN], rec_full[NREC], rec_empty[NREC], sv_full[NVS], sv_empty[NVS]
    static constexpr int NBAR = 2 * W::NIN + 2 * W::NREC + 2 * W::NVS;
    static constexpr size_t BAR_BYTES = ((NBAR * 8 + 15) / 16) * 16;
    static constexpr size_t SVN = (size_t)T::NN * osmpm::SV<D>::S;
    static constexpr size_t SY = (size_t)T::NN * D;
    static constexpr size_t STG = Stage<D>::SIZE;
    static constexpr size_t IN = (size_t)NF * PFS;
    static constexpr size_t REC = (size_t)RS * W::CAP;
    static constexpr int INFO = ((T::NC + 2 + 3) / 4) * 4;  // ints: tile id, NC + 1 cell starts (16-B padded)
    static constexpr size_t INFO_BYTES = (size_t)W::NVS * INFO * sizeof(int);
    static constexpr size_t BYTES =
        BAR_BYTES + INFO_BYTES + (W::NVS * SVN + SY + STG + W::NIN * IN + W::NREC * REC) * sizeof(R);
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// deterministic unit enumeration shared by every role; the current tile's layer bounds are held
// in registers (one batch of loads per tile)
template <int NL>
struct UnitIter {
    const int* cs;       // cell_start
    int ntiles, stride;
    int tile, layer, sb, lb, le;  // current unit
    int64_t kt;
    int LC, NC, CAP;
    int lbnd[NL + 1];             // layer boundaries of the current tile
    int loaded_tile;
    __device__ __forceinline__ void load_tile()
    {
        kt = (int64_t)tile * NC;
#pragma unroll
        for (int l = 0; l <= NL; ++l) lbnd[l] = __ldg(cs + kt + l * LC);
        loaded_tile = tile;
    }
    __device__ __forceinline__ bool layer_range(int l)
    {
        int b0 = lbnd[0], b1 = lbnd[1];
#pragma unroll
        for (int k = 1; k < NL; ++k)
            if (l == k) {
                b0 = lbnd[k];
                b1 = lbnd[k + 1];
            }
        lb = b0;
        le = b1;
        return lb < le;
    }
    // advance to the first unit at or after (tile, layer); returns false when done
    __device__ __forceinline__ bool seek()
    {
        while (tile < ntiles) {
            if (loaded_tile != tile) load_tile();
            if (lbnd[0] < lbnd[NL]) {
                while (layer < NL) {
                    if (layer_range(layer)) {
                        if (sb < lb) sb = lb;
                        if (sb < le) return true;
                    }
                    ++layer;
                    sb = -1;
                }
            }
            tile += stride;
            layer = 0;
            sb = -1;
        }
        return false;
    }
    __device__ __forceinline__ void init(const int* c, int nt, int first, int st, int lc, int nc, int cap)
    {
        cs = c;
        ntiles = nt;
        tile = first;
        stride = st;
        layer = 0;
        sb = -1;
        LC = lc;
        NC = nc;
        CAP = cap;
        loaded_tile = -1;
    }
    __device__ __forceinline__ int se() const { return min(sb + CAP, le); }
    __device__ __forceinline__ bool last_of_layer() const { return sb + CAP >= le; }
    // the tile's particles end with this unit / start with it (layers are contiguous in memory)
    __device__ __forceinline__ bool last_of_tile() const { return sb + CAP >= le && le == lbnd[NL]; }
    __device__ __forceinline__ bool first_of_tile() const { return sb == lbnd[0]; }
    __device__ __forceinline__ void next()
    {
        sb += CAP;
        if (sb >= le) {
            ++layer;
            sb = -1;
        }
    }
};

template <int D, typename R>
__global__ void __launch_bounds__(WS<D>::NTHR, 1)
k_hvp_ws(const R* __restrict__ P, const R* __restrict__ cache, int64_t cap, const int* __restrict__ cell_start,
         BoxDev b, const double* __restrict__ din, double* __restrict__ yout)
{
    using T = Tile<D>;
    using W = WS<D>;
    using Lay = WSLayout<D, R>;
    using C = CL<D>;
    constexpr int RS = Lay::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* in_full = bars;
    uint64_t* in_empty = in_full + W::NIN;
    uint64_t* rec_full = in_empty + W::NIN;
    uint64_t* rec_empty = rec_full + W::NREC;
    uint64_t* sv_full = rec_empty + W::NREC;
    uint64_t* sv_empty = sv_full + W::NVS;
    int* info_ring = reinterpret_cast<int*>(smem_raw + Lay::BAR_BYTES);
    R* sv_ring = reinterpret_cast<R*>(smem_raw + Lay::BAR_BYTES + Lay::INFO_BYTES);
    R* sy = sv_ring + W::NVS * Lay::SVN;
    R* stg = sy + Lay::SY;
    R* in_ring = stg + Lay::STG;
    R* rec_ring = in_ring + W::NIN * Lay::IN;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < W::NIN; ++s) {
            mbar_init(in_full + s, 1);
            mbar_init(in_empty + s, W::NG * 32);
        }
        for (int s = 0; s < W::NREC; ++s) {
            mbar_init(rec_full + s, W::NG * 32);
            mbar_init(rec_empty + s, W::NS * 32);
        }
        for (int s = 0; s < W::NVS; ++s) {
            mbar_init(sv_full + s, 32);
            mbar_init(sv_empty + s, (W::NG + W::NS) * 32);
        }
        fence_async_smem();
    }
    __syncthreads();

    if (warp == 0) {
        // ================================ loader ================================
        // walks this CTA's tiles, publishes each non-empty tile (id, cell ranges, node values) in the
        // tile ring, then streams its units' particle inputs with TMA; a tile id of -1 ends the work
        UnitIter<T::NL> U;
        U.init(cell_start, b.ntiles, blockIdx.x, gridDim.x, T::LC, T::NC, W::CAP);
        int u = 0, ntile = 0;
        int published = -1;
        for (;;) {
            const bool more = U.seek();
            if (!more || U.tile != published) {
                const int vs = ntile % W::NVS;
                if (ntile >= W::NVS) mbar_wait(sv_empty + vs, ((ntile / W::NVS) - 1) & 1);
                int* info = info_ring + vs * Lay::INFO;
                if (!more) {
                    if (lane == 0) info[0] = -1;
                    __syncwarp();
                    mbar_arrive(sv_full + vs);
                    break;
                }
                for (int i = lane; i <= T::NC; i += 32) info[1 + i] = __ldg(cell_start + U.kt + i);
                if (lane == 0) info[0] = U.tile;
                int t[3];
                tile_coords<D>(b, U.tile, t);
                R* sv = sv_ring + vs * Lay::SVN;
                for (int idx = lane; idx < T::NN * D; idx += 32) {
                    const int a = idx % D, l = idx / D;
                    int c[3];
                    tnode_coords<D>(l, c);
                    const int64_t g = box_node<D>(b, t[0] * T::T0 + c[0], t[1] * T::T1 + c[1], t[2] * T::T2 + c[2]);
                    sv[l * SV<D>::S + a] = (R)__ldg(din + g * D + a);
                }
                mbar_arrive(sv_full + vs);
                published = U.tile;
                ++ntile;
            }
            const int s = u % W::NIN;
            if (u >= W::NIN) mbar_wait(in_empty + s, ((u / W::NIN) - 1) & 1);
            if (lane == 0) {
                const int sb0 = U.sb & ~(Lay::UE - 1);
                const int cnt = U.se() - sb0;
                const int cnt_al = (cnt + Lay::UE - 1) & ~(Lay::UE - 1);
                const uint32_t bytes = (uint32_t)cnt_al * sizeof(R);
                R* dst = in_ring + s * Lay::IN;
                fence_async_smem();
                mbar_expect_tx(in_full + s, bytes * Lay::NF);
                for (int f = 0; f < Lay::NF; ++f) {
                    const R* src = (f < D) ? P + (int64_t)(PL<D>::X + f) * cap + sb0 : cache + (int64_t)(f - D) * cap + sb0;
                    bulk_g2s(dst + f * Lay::PFS, src, bytes, in_full + s);
                }
            }
            __syncwarp();
            ++u;
            U.next();
        }
        return;
    }

    // consumers: tiles in the loader's order, units in (layer, sub-chunk) order from the smem info
    const bool gatherer = warp <= W::NG;
    const int gw = warp - 1;
    const int it = threadIdx.x - 32 * (1 + W::NG);
    constexpr int NSTHR = 32 * W::NS;
    const bool item = !gatherer && it < T::ITEMS;
    const int icell = it / (D * 3), icomp = (it / 3) % D, ii = it % 3;
    int u = 0;
    for (int ntile = 0;; ++ntile) {
        const int vs = ntile % W::NVS;
        mbar_wait(sv_full + vs, (ntile / W::NVS) & 1);
        const int* info = info_ring + vs * Lay::INFO;
        const int tile = info[0];
        if (tile < 0) break;
        const int* cs = info + 1;
        const R* sv = sv_ring + vs * Lay::SVN;
        int t[3];
        tile_coords<D>(b, tile, t);
        if (!gatherer) {
            for (int idx = it; idx < T::NN * D; idx += NSTHR) sy[idx] = R(0);
        }
        for (int layer = 0; layer < T::NL; ++layer) {
            const int lb = cs[layer * T::LC], le = cs[(layer + 1) * T::LC];
            if (lb == le) continue;
            int ks = 0, ke = 0;
            R acc[T::NACC];
            if (item) {
                ks = cs[layer * T::LC + icell];
                ke = cs[layer * T::LC + icell + 1];
#pragma unroll
                for (int k = 0; k < T::NACC; ++k) acc[k] = R(0);
            }
            for (int sb = lb; sb < le; sb += W::CAP, ++u) {
                const int se = min(sb + W::CAP, le);
                const int rs = u % W::NREC;
                if (gatherer) {
                    // ------------------------------ gather ------------------------------
                    const int s = u % W::NIN;
                    mbar_wait(in_full + s, (u / W::NIN) & 1);
                    if (u >= W::NREC) mbar_wait(rec_empty + rs, ((u / W::NREC) - 1) & 1);
                    const int q = gw * 32 + lane;
                    const int p = sb + q;
                    if (p < se) {
                        const R* src = in_ring + s * Lay::IN + (p - (sb & ~(Lay::UE - 1)));
                        R x[3], S[Sym<D>::N], A[D * D];
#pragma unroll
                        for (int a = 0; a < D; ++a) x[a] = src[a * Lay::PFS];
#pragma unroll
                        for (int k = 0; k < Sym<D>::N; ++k) S[k] = src[(D + C::S + k) * Lay::PFS];
#pragma unroll
                        for (int k = 0; k < D * D; ++k) A[k] = src[(D + C::A + k) * Lay::PFS];
                        const R cc = src[(D + C::C) * Lay::PFS], ll = src[(D + C::L) * Lay::PFS];
                        R w[3][3], dw[3][3];
                        int lc[3] = {0, 0, 0};
                        weights_at<D, R>(x, b, t, lc, w, dw);
                        R gd[D * D];
                        gather_grad<D, R>(sv, lc, w, dw, gd);
                        const RecPtr<R> r(rec_ring + rs * Lay::REC, q, RS);
                        store_weights<D, R>(r, w, dw);
                        R M2[D * D], tr = R(0);
#pragma unroll
                        for (int a = 0; a < D; ++a)
#pragma unroll
                            for (int bb = 0; bb < D; ++bb) {
                                R sacc = R(0);
#pragma unroll
                                for (int k = 0; k < D; ++k) sacc = fma(A[a * D + k], gd[bb * D + k], sacc);
                                M2[a * D + bb] = sacc;
                                tr = fma(A[a * D + bb], gd[a * D + bb], tr);
                            }
                        const R ltr = ll * tr;
#pragma unroll
                        for (int a = 0; a < D; ++a)
#pragma unroll
                            for (int bb = 0; bb < D; ++bb) {
                                R s1 = R(0), s2 = R(0);
#pragma unroll
                                for (int k = 0; k < D; ++k) {
                                    s1 = fma(gd[a * D + k], S[sym_idx<D>(k, bb)], s1);
                                    s2 = fma(M2[a * D + k], A[k * D + bb], s2);
                                }
                                *r.at(Rec<D>::G + a * D + bb) = fma(cc, s2, fma(ltr, A[a * D + bb], s1));
                            }
                    }
                    // every lane arrives (release of its own smem reads / writes)
                    mbar_arrive(in_empty + s);
                    mbar_arrive(rec_full + rs);
                } else {
                    // ------------------------------ scatter -----------------------------
                    mbar_wait(rec_full + rs, (u / W::NREC) & 1);
                    if (item) {
                        const int p0 = max(ks, sb), p1 = min(ke, se);
                        const int len = p1 - p0, rot = len > 0 ? (icell & 7) % len : 0;
                        R* rr = rec_ring + rs * Lay::REC;
                        for (int k = 0; k < len; ++k) {
                            const RecPtr<R> r(rr, rotated(p0, len, k, rot) - sb, RS);
                            ItemW<D, R> Wt;
                            Wt.load(r, ii);
                            R sg[D];
#pragma unroll
                            for (int bb = 0; bb < D; ++bb) sg[bb] = *r.at(Rec<D>::G + icomp * D + bb);
                            item_linear<D, R>(sg, Wt, acc);
                        }
                    }
                    mbar_arrive(rec_empty + rs);
                }
            }
            if (!gatherer) {
                // stage + flush of the layer among the scatter warps (named barrier 1)
                for (int idx = it; idx < Stage<D>::SIZE / Lay::UE; idx += NSTHR)
                    reinterpret_cast<int4*>(stg)[idx] = make_int4(0, 0, 0, 0);
                named_sync(1, NSTHR);
                if (item) stage_item<D, R>(icell, icomp, ii, acc, stg);
                named_sync(1, NSTHR);
                using S = Stage<D>;
                for (int j = it; j < S::NITEM; j += NSTHR) {
                    const R* pp = stg + j * S::NSLOT;
                    R sum = pp[0];
#pragma unroll
                    for (int k = 1; k < S::NSLOT; ++k) sum += pp[k];
                    const int a = j % D, kk = (j / D) % 3, nxy = j / (3 * D);
                    sy[((D == 3) ? (nxy * T::N2 + layer + kk) : (nxy * T::N1 + layer + kk)) * D + a] += sum;
                }
                named_sync(1, NSTHR);
            }
        }
        if (!gatherer) {
            for (int idx = it; idx < T::NN * D; idx += NSTHR) {
                const R sval = sy[idx];
                if (sval != R(0)) {
                    const int a = idx % D, l = idx / D;
                    int c[3];
                    tnode_coords<D>(l, c);
                    const int64_t g = box_node<D>(b, t[0] * T::T0 + c[0], t[1] * T::T1 + c[1], t[2] * T::T2 + c[2]);
                    atomicAdd(&yout[g * D + a], (double)sval);
                }
            }
            named_sync(1, NSTHR);
        }
        mbar_arrive(sv_empty + vs);  // every consumer lane releases the tile slot
    }
}

}  // namespace osmpm
