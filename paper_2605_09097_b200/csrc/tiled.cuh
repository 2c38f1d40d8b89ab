// tiled.cuh -- tiled particle-loop scatter kernels: the Hessian-vector product (a5) and the
// Newton gradient / energy / Jacobi diagonal / linearisation cache (a4).
//
// One CTA per tile of T0 x T1 x T2 cells (a "cell" = the particles sharing a base node).  The tile's
// (T+2)^D nodes of the input vector are staged in shared memory once.  The tile is then walked
// layer by layer along its last axis; per layer (sub-chunked if it holds more than NT particles):
//   phase 1  thread per particle: weights, tensor-product gather from smem, per-particle source
//            G_p (a D x D matrix) -> a per-particle smem record (XOR-swizzled 16-B units)
//   phase 2  thread per (cell, component a, x-offset i): register accumulation, over the cell's
//            particles, of G_p[a] . grad N for the 3^(D-1) stencil nodes with x-offset i
//   phase 3  the partials go to a node-major staging array (one slot per contributing cell, no
//            conflicts, slots of cells outside the tile zero) and each (node, component) sums its
//            3^(D-1) slots into a shared-memory node accumulator
// and after the last layer one fp64 RED per tile node and component writes the result.
// The HVP streams its per-particle inputs (x and the Newton cache) with TMA bulk copies
// (cp.async.bulk + mbarrier): the next layer is in flight while the current one is computed.
#pragma once
#include "device.cuh"

namespace osmpm {

template <int D>
__device__ __forceinline__ void tile_coords(const BoxDev& b, int tile, int* t)
{
    if (D == 3) {
        t[2] = tile % b.nt[2];
        t[1] = (tile / b.nt[2]) % b.nt[1];
        t[0] = tile / (b.nt[2] * b.nt[1]);
    } else {
        t[2] = 0;
        t[1] = tile % b.nt[1];
        t[0] = tile / b.nt[1];
    }
}

template <int D>
__device__ __forceinline__ int tnode(int l0, int l1, int l2)
{
    using T = Tile<D>;
    return (D == 3) ? (l0 * T::N1 + l1) * T::N2 + l2 : l0 * T::N1 + l1;
}

template <int D>
__device__ __forceinline__ void tnode_coords(int l, int* c)
{
    using T = Tile<D>;
    if (D == 3) {
        c[2] = l % T::N2;
        c[1] = (l / T::N2) % T::N1;
        c[0] = l / (T::N2 * T::N1);
    } else {
        c[2] = 0;
        c[1] = l % T::N1;
        c[0] = l / T::N1;
    }
}

// ---------------------------------------------------------------------------------------------
// TMA bulk copy + mbarrier (sm_90+ PTX; SASS UBLKCP / SYNCS)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------------------------------------
// shared-memory layouts
// ---------------------------------------------------------------------------------------------
// node tile: SV reals per node (3D: 4 = 3 components + pad, for 16-B loads)
template <int D> struct SV { static constexpr int S = (D == 3) ? 4 : 2; };

// node-major staging array of one layer
template <int D> struct Stage {
    using T = Tile<D>;
    static constexpr int NXY = (D == 3) ? T::N0 * T::N1 : T::N0;   // lateral node positions
    static constexpr int NSLOT = (D == 3) ? 9 : 3;                  // contributing cells per node
    static constexpr int NITEM = NXY * 3 * D;                       // (lateral node, last-axis offset, comp)
    static constexpr int SIZE = NITEM * NSLOT;
};

// Per-particle record: RS reals = an ODD number of 16-byte units, so the 16-B accesses of 8
// consecutive particles (phase-1 stores) hit distinct bank groups; phase 2 walks each cell's
// particles starting at a per-cell rotation so that lanes of neighbouring cells read records
// 8k+k apart (regular 8-per-cell lattices would otherwise map them to one bank group).
// Elements: [axis a: (w0,dw0,w1,dw1,w2,dw2)] x D | G (D*D) | extra (gradient kernel)
template <int D> struct Rec {
    static constexpr int WP = 0, G = 6 * D, X = 6 * D + D * D;
};
template <int D, typename R> struct HvpRec {
    static constexpr int RS = (sizeof(R) == 8) ? ((D == 3) ? 30 : 18) : ((D == 3) ? 28 : 20);
};
template <int D> struct GradRec {
    static constexpr int S = Rec<D>::X, A = S + Sym<D>::N, CL = A + D * D;
    static constexpr int RS = (D == 3) ? 44 : 26;  // 43 used; even for the 16-B weight pairs
};

template <typename R>
struct RecPtr {
    R* base;
    __device__ __forceinline__ RecPtr(R* rec, int q, int RS) : base(rec + q * RS) {}
    __device__ __forceinline__ R* at(int e) const { return base + e; }
};

// Phase-2 item (cell, component a, x-offset i) of thread `it`.  3D: the 9 items of a cell do not fit
// an 8-lane quarter-warp, and shared-memory broadcast loads cost twice as many wavefronts when a
// broadcast group straddles quarters (scripts/smem_probe.cu: LDS.128 2 vs 4, LDS.64 1 vs 2).  So
// threads 0-127 hold the first 8 items of cells 0-15 (one cell per quarter) and threads 128-143 the
// ninth item (a = 2, i = 2) of each cell.  2D: consecutive (cell, a, i).
template <int D>
__device__ __forceinline__ void item_of(int it, int& icell, int& icomp, int& ii)
{
    using T = Tile<D>;
    if (D == 3 && T::LC == 16) {
        const int pair = it < 128 ? (it & 7) : 8;
        icell = it < 128 ? (it >> 3) : it - 128;
        icomp = pair / 3;
        ii = pair % 3;
    } else {
        icell = it / (D * 3);
        icomp = (it / 3) % D;
        ii = it % 3;
    }
}

// k-th particle of [p0, p1) in the rotated order starting at offset rot
__device__ __forceinline__ int rotated(int p0, int len, int k, int rot)
{
    int o = k + rot;
    o = (o >= len) ? o - len : o;
    return p0 + o;
}

template <typename R> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

// gather gd[a][b] = sum_i v_i,a dN_i/dx_b (tensor-product order, explicit FMA)
template <int D, typename R>
__device__ __forceinline__ void gather_grad(const R* sv, const int* lc, const R (*w)[3], const R (*dw)[3], R* gd)
{
    using V2 = typename Vec2<R>::type;
#pragma unroll
    for (int k = 0; k < D * D; ++k) gd[k] = R(0);
    if (D == 3) {
        const R* base = sv + tnode<D>(lc[0], lc[1], lc[2]) * 4;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            R U0[3] = {0, 0, 0}, U1[3] = {0, 0, 0}, U2[3] = {0, 0, 0};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                R T0[3] = {0, 0, 0}, T1[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const R* sp = base + ((i * Tile<3>::N1 + j) * Tile<3>::N2 + k) * 4;
                    const V2 v01 = *reinterpret_cast<const V2*>(sp);
                    const R s[3] = {v01.x, v01.y, sp[2]};
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        T0[a] = fma(s[a], w[2][k], T0[a]);
                        T1[a] = fma(s[a], dw[2][k], T1[a]);
                    }
                }
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    U0[a] = fma(T0[a], w[1][j], U0[a]);
                    U1[a] = fma(T0[a], dw[1][j], U1[a]);
                    U2[a] = fma(T1[a], w[1][j], U2[a]);
                }
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                gd[a * 3 + 0] = fma(U0[a], dw[0][i], gd[a * 3 + 0]);
                gd[a * 3 + 1] = fma(U1[a], w[0][i], gd[a * 3 + 1]);
                gd[a * 3 + 2] = fma(U2[a], w[0][i], gd[a * 3 + 2]);
            }
        }
    } else {
        const R* base = sv + tnode<D>(lc[0], lc[1], 0) * 2;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            R U0[2] = {0, 0}, U1[2] = {0, 0};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const V2 v = *reinterpret_cast<const V2*>(base + (i * Tile<2>::N1 + j) * 2);
                const R s[2] = {v.x, v.y};
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    U0[a] = fma(s[a], w[1][j], U0[a]);
                    U1[a] = fma(s[a], dw[1][j], U1[a]);
                }
            }
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                gd[a * 2 + 0] = fma(U0[a], dw[0][i], gd[a * 2 + 0]);
                gd[a * 2 + 1] = fma(U1[a], w[0][i], gd[a * 2 + 1]);
            }
        }
    }
}

template <int D, typename R>
__device__ __forceinline__ void store_weights(const RecPtr<R>& r, const R (*w)[3], const R (*dw)[3])
{
    using V2 = typename Vec2<R>::type;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            V2 v;
            v.x = w[a][k];
            v.y = dw[a][k];
            *reinterpret_cast<V2*>(r.at(Rec<D>::WP + a * 6 + 2 * k)) = v;
        }
}

// weights of one particle as seen by item (i): x pair at offset i, full y / z pairs
template <int D, typename R>
struct ItemW {
    R wx, dwx, wy[3], dwy[3], wz[3], dwz[3];
    __device__ __forceinline__ void load(const RecPtr<R>& r, int i)
    {
        using V2 = typename Vec2<R>::type;
        const V2 x = *reinterpret_cast<const V2*>(r.at(2 * i));
        wx = x.x;
        dwx = x.y;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const V2 y = *reinterpret_cast<const V2*>(r.at(6 + 2 * k));
            wy[k] = y.x;
            dwy[k] = y.y;
            if (D == 3) {
                const V2 z = *reinterpret_cast<const V2*>(r.at(12 + 2 * k));
                wz[k] = z.x;
                dwz[k] = z.y;
            }
        }
    }
};

// acc[(j,k)] += sum_b s_b dN_{(i,j,k)}/dx_b
template <int D, typename R>
__device__ __forceinline__ void item_linear(const R* s, const ItemW<D, R>& W, R* acc)
{
    if (D == 3) {
        const R ax = s[0] * W.dwx, bx = s[1] * W.wx, cx = s[2] * W.wx;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const R A = fma(ax, W.wy[j], bx * W.dwy[j]);
            const R B = cx * W.wy[j];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                acc[j * 3 + k] = fma(A, W.wz[k], acc[j * 3 + k]);
                acc[j * 3 + k] = fma(B, W.dwz[k], acc[j * 3 + k]);
            }
        }
    } else {
        const R ax = s[0] * W.dwx, bx = s[1] * W.wx;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            acc[j] = fma(ax, W.wy[j], acc[j]);
            acc[j] = fma(bx, W.dwy[j], acc[j]);
        }
    }
}

// acc[(j,k)] += gradN^T Q gradN, Q symmetric (Sym<D> storage)
template <int D, typename R>
__device__ __forceinline__ void item_quadratic(const R* Q, const ItemW<D, R>& W, R* acc)
{
    const R pxx = W.dwx * W.dwx, pxw = W.dwx * W.wx, pww = W.wx * W.wx;
    if (D == 3) {
        const R a00 = Q[0] * pxx, a11 = Q[1] * pww, a22 = Q[2] * pww, a01 = R(2) * Q[3] * pxw,
                a02 = R(2) * Q[4] * pxw, a12 = R(2) * Q[5] * pww;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const R y2 = W.wy[j] * W.wy[j], yy = W.wy[j] * W.dwy[j], dy2 = W.dwy[j] * W.dwy[j];
            const R C2 = fma(a00, y2, fma(a11, dy2, a01 * yy));
            const R C1 = fma(a02, y2, a12 * yy);
            const R C0 = a22 * y2;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const R z2 = W.wz[k] * W.wz[k], zz = W.wz[k] * W.dwz[k], dz2 = W.dwz[k] * W.dwz[k];
                acc[j * 3 + k] = fma(C2, z2, acc[j * 3 + k]);
                acc[j * 3 + k] = fma(C1, zz, acc[j * 3 + k]);
                acc[j * 3 + k] = fma(C0, dz2, acc[j * 3 + k]);
            }
        }
    } else {
        const R a00 = Q[0] * pxx, a11 = Q[1] * pww, a01 = R(2) * Q[2] * pxw;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            acc[j] = fma(a00, W.wy[j] * W.wy[j], acc[j]);
            acc[j] = fma(a11, W.dwy[j] * W.dwy[j], acc[j]);
            acc[j] = fma(a01, W.wy[j] * W.dwy[j], acc[j]);
        }
    }
}

// fixed NSLOT-term sums -> node accumulator tile sy
template <int D, typename R>
__device__ __forceinline__ void layer_flush(int layer, const R* stg, R* sy)
{
    using T = Tile<D>;
    using S = Stage<D>;
    for (int it = threadIdx.x; it < S::NITEM; it += T::NT) {
        const R* p = stg + it * S::NSLOT;
        R s = p[0];
#pragma unroll
        for (int k = 1; k < S::NSLOT; ++k) s += p[k];
        const int a = it % D, kk = (it / D) % 3, nxy = it / (3 * D);
        sy[((D == 3) ? (nxy * T::N2 + layer + kk) : (nxy * T::N1 + layer + kk)) * D + a] += s;
    }
}

// final: one RED per tile node and component
template <int D, typename R>
__device__ __forceinline__ void tile_flush(const BoxDev& b, const int* t, const R* sy, double* __restrict__ out)
{
    using T = Tile<D>;
    for (int idx = threadIdx.x; idx < T::NN * D; idx += T::NT) {
        const R s = sy[idx];
        if (s != R(0)) {
            const int a = idx % D, l = idx / D;
            int c[3];
            tnode_coords<D>(l, c);
            const int64_t g = box_node<D>(b, t[0] * T::T0 + c[0], t[1] * T::T1 + c[1], t[2] * T::T2 + c[2]);
            atomicAdd(&out[g * D + a], (double)s);
        }
    }
}

// local cell + weights of a particle from its position
template <int D, typename Rw>
__device__ __forceinline__ void weights_at(const Rw* x, const BoxDev& b, const int* t, int* lc, Rw (*w)[3],
                                           Rw (*dw)[3])
{
    using T = Tile<D>;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int tt = a == 0 ? T::T0 : (a == 1 ? T::T1 : T::T2);
        Rw f;
        lc[a] = base_of<Rw>(x[a], b.o[a], b.inv_dx, &f) - b.lo[a] - t[a] * tt;
        bspline<Rw>(f, (Rw)b.inv_dx, w[a], dw[a]);
    }
}

// =============================================================================================
// a5: HVP  y += sum_p V0 dP(F_p(u); gd F^n) F^nT grad N  =  sum_p G_p grad N with
//     G = gd S' + c' Ah gd^T Ah + l' (Ah : gd) Ah   (derivation from PAPER.md:188, 208)
// =============================================================================================
template <int D, typename R> struct HvpIn {
    static constexpr int NF = D + CL<D>::NF;
    static constexpr int UE = 16 / sizeof(R);
    static constexpr int PFS = Tile<D>::NT + 2 * UE;  // per-field capacity (alignment slack)
};

}  // namespace osmpm
