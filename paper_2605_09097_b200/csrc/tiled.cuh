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
    static constexpr int RS = (D == 3) ? 46 : 26;
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

// phase 0: sv = input vector on the tile nodes, sy (NOUT tiles) = 0
template <int D, typename R, int NOUT>
__device__ __forceinline__ void stage_nodes(const BoxDev& b, const int* t, const double* __restrict__ vec, R* sv,
                                            R* sy)
{
    using T = Tile<D>;
    for (int idx = threadIdx.x; idx < T::NN * D; idx += T::NT) {
        const int a = idx % D, l = idx / D;
        int c[3];
        tnode_coords<D>(l, c);
        const int64_t g = box_node<D>(b, t[0] * T::T0 + c[0], t[1] * T::T1 + c[1], t[2] * T::T2 + c[2]);
        sv[l * SV<D>::S + a] = (R)vec[g * D + a];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) sy[o * T::NN * D + idx] = R(0);
    }
}

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

// zero the staging array (16-B stores)
template <int D, typename R>
__device__ __forceinline__ void stage_zero(R* stg)
{
    using T = Tile<D>;
    constexpr int UE = 16 / sizeof(R);
    static_assert(Stage<D>::SIZE % UE == 0, "stage size");
    int4 z = make_int4(0, 0, 0, 0);
    for (int u = threadIdx.x; u < Stage<D>::SIZE / UE; u += T::NT) reinterpret_cast<int4*>(stg)[u] = z;
}

// phase-2 partials -> staging: item (cell (cx,cy), comp a, x-offset i) owns slot (i, j) of the nodes
// (cx+i, cy+j, layer+kk); acc index (j*3 + kk) in 3D, (j) in 2D (j = last-axis offset there)
template <int D, typename R>
__device__ __forceinline__ void stage_item(int cellL, int a, int i, const R* acc, R* stg)
{
    using T = Tile<D>;
    if (D == 3) {
        const int cx = cellL / T::T1, cy = cellL % T::T1;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                const int nxy = (cx + i) * T::N1 + (cy + j);
                stg[((nxy * 3 + kk) * 3 + a) * 9 + i * 3 + j] = acc[j * 3 + kk];
            }
    } else {
#pragma unroll
        for (int j = 0; j < 3; ++j) stg[(((cellL + i) * 3 + j) * 2 + a) * 3 + i] = acc[j];
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
template <int D, bool PF> struct HvpOcc { static constexpr int MIN_BLOCKS = (D == 3) ? (PF ? 3 : 4) : 4; };

// per-particle streamed inputs: x (D) and the Newton cache (CL<D>::NF fields)
template <int D, typename R> struct HvpIn {
    static constexpr int NF = D + CL<D>::NF;
    static constexpr int UE = 16 / sizeof(R);
    static constexpr int PFS = Tile<D>::NT + 2 * UE;  // per-field capacity (alignment slack)
};

template <int D, typename R, bool PF = true>
constexpr size_t hvp_smem_bytes()
{
    using T = Tile<D>;
    constexpr size_t rec = (size_t)HvpRec<D, R>::RS * T::NT;
    constexpr size_t recstg = rec > (size_t)Stage<D>::SIZE ? rec : (size_t)Stage<D>::SIZE;
    return 16 + ((size_t)T::NN * SV<D>::S + T::NN * D + recstg +
                 (PF ? (size_t)HvpIn<D, R>::NF * HvpIn<D, R>::PFS : 0)) * sizeof(R);
}

// issue the TMA bulk copies of the first min(NT, le - lb) particles of a layer
template <int D, typename R>
__device__ __forceinline__ int hvp_prefetch(const R* __restrict__ P, const R* __restrict__ cache, int64_t cap, int lb,
                                            int le, R* pf, uint64_t* bar)
{
    using In = HvpIn<D, R>;
    const int lb0 = lb & ~(In::UE - 1);                       // 16-B aligned start
    const int cnt = min(le, lb + Tile<D>::NT) - lb0;
    const int cnt_al = (cnt + In::UE - 1) & ~(In::UE - 1);    // 16-B multiple
    const uint32_t bytes = (uint32_t)cnt_al * sizeof(R);
    fence_async_smem();
    mbar_expect_tx(bar, bytes * In::NF);
#pragma unroll 1
    for (int f = 0; f < In::NF; ++f) {
        const R* src = (f < D) ? P + (int64_t)(PL<D>::X + f) * cap + lb0 : cache + (int64_t)(f - D) * cap + lb0;
        bulk_g2s(pf + f * In::PFS, src, bytes, bar);
    }
    return lb0;
}

template <int D, typename R, bool PF = true>
__global__ void __launch_bounds__(Tile<D>::NT, HvpOcc<D, PF>::MIN_BLOCKS)
k_hvp(const R* __restrict__ P, const R* __restrict__ cache, int64_t cap, const int* __restrict__ cell_start,
      BoxDev b, const double* __restrict__ din, double* __restrict__ yout)
{
    using T = Tile<D>;
    using C = CL<D>;
    using In = HvpIn<D, R>;
    constexpr int RS = HvpRec<D, R>::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    R* sv = reinterpret_cast<R*>(smem_raw + 16);
    R* sy = sv + T::NN * SV<D>::S;
    R* pf = sy + T::NN * D;                 // streamed particle inputs (NF fields x PFS)
    R* rec = pf + (PF ? In::NF * In::PFS : 0);  // per-particle records, aliased by the staging array
    R* stg = rec;
    const int tile = blockIdx.x;
    const int64_t kt = (int64_t)tile * T::NC;
    __shared__ int scs[T::NC + 1];  // the tile's cell ranges
    for (int i = threadIdx.x; i <= T::NC; i += T::NT) scs[i] = cell_start[kt + i];
    __syncthreads();
    if (scs[0] == scs[T::NC]) return;
    // first non-empty layer and its prefetch
    int layer = 0;
    while (scs[layer * T::LC] == scs[(layer + 1) * T::LC]) ++layer;
    int lb0 = 0;
    if (PF && threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_async_smem();
        lb0 = hvp_prefetch<D, R>(P, cache, cap, scs[layer * T::LC], scs[(layer + 1) * T::LC], pf, bar);
    }
    int t[3];
    tile_coords<D>(b, tile, t);
    stage_nodes<D, R, 1>(b, t, din, sv, sy);
    __syncthreads();
    const int it = threadIdx.x;
    const int icell = it / (D * 3), icomp = (it / 3) % D, ii = it % 3;
    uint32_t parity = 0;
    while (layer < T::NL) {
        const int lb = scs[layer * T::LC], le = scs[(layer + 1) * T::LC];
        int next = layer + 1;
        while (next < T::NL && scs[next * T::LC] == scs[(next + 1) * T::LC]) ++next;
        const int pf_base = lb & ~(In::UE - 1);
        const int ks = scs[layer * T::LC + icell];
        const int ke = scs[layer * T::LC + icell + 1];
        R acc[T::NACC];
#pragma unroll
        for (int k = 0; k < T::NACC; ++k) acc[k] = R(0);
        for (int sb = lb; sb < le; sb += T::NT) {
            const int se = min(sb + T::NT, le);
            const int q = threadIdx.x, p = sb + q;
            const bool from_pf = PF && (sb == lb);
            if (from_pf) mbar_wait(bar, parity);
            if (p < se) {
                // streamed inputs: smem copy of the first NT particles, global beyond
                R x[3], S[Sym<D>::N], A[D * D], cc, ll;
                if (from_pf) {
                    const R* s = pf + (p - pf_base);
#pragma unroll
                    for (int a = 0; a < D; ++a) x[a] = s[a * In::PFS];
#pragma unroll
                    for (int k = 0; k < Sym<D>::N; ++k) S[k] = s[(D + C::S + k) * In::PFS];
#pragma unroll
                    for (int k = 0; k < D * D; ++k) A[k] = s[(D + C::A + k) * In::PFS];
                    cc = s[(D + C::C) * In::PFS];
                    ll = s[(D + C::L) * In::PFS];
                } else {
#pragma unroll
                    for (int a = 0; a < D; ++a) x[a] = P[(PL<D>::X + a) * cap + p];
#pragma unroll
                    for (int k = 0; k < Sym<D>::N; ++k) S[k] = cache[(C::S + k) * cap + p];
#pragma unroll
                    for (int k = 0; k < D * D; ++k) A[k] = cache[(C::A + k) * cap + p];
                    cc = cache[C::C * cap + p];
                    ll = cache[C::L * cap + p];
                }
                R w[3][3], dw[3][3];
                int lc[3] = {0, 0, 0};
                weights_at<D, R>(x, b, t, lc, w, dw);
                R gd[D * D];
                gather_grad<D, R>(sv, lc, w, dw, gd);
                const RecPtr<R> r(rec, q, RS);
                store_weights<D, R>(r, w, dw);
                // M2 = A gd^T ; tr = A : gd
                R M2[D * D], tr = R(0);
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) {
                        R s = R(0);
#pragma unroll
                        for (int k = 0; k < D; ++k) s = fma(A[a * D + k], gd[bb * D + k], s);
                        M2[a * D + bb] = s;
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
            __syncthreads();
            if (from_pf) {
                parity ^= 1u;
                // the streamed buffer is free: start the next layer's copies now
                if (threadIdx.x == 0 && next < T::NL)
                    hvp_prefetch<D, R>(P, cache, cap, scs[next * T::LC], scs[(next + 1) * T::LC], pf, bar);
            }
            if (it < T::ITEMS) {
                const int p0 = max(ks, sb), p1 = min(ke, se);
                const int len = p1 - p0, rot = len > 0 ? (icell & 7) % len : 0;
                for (int k = 0; k < len; ++k) {
                    const RecPtr<R> r(rec, rotated(p0, len, k, rot) - sb, RS);
                    ItemW<D, R> W;
                    W.load(r, ii);
                    R s[D];
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) s[bb] = *r.at(Rec<D>::G + icomp * D + bb);
                    item_linear<D, R>(s, W, acc);
                }
            }
            __syncthreads();
        }
        stage_zero<D, R>(stg);
        __syncthreads();
        if (it < T::ITEMS) stage_item<D, R>(icell, icomp, ii, acc, stg);
        __syncthreads();
        layer_flush<D, R>(layer, stg, sy);
        __syncthreads();
        layer = next;
    }
    (void)lb0;
    tile_flush<D, R>(b, t, sy, yout);
}

// =============================================================================================
// a4: gradient + energy + Newton cache + Jacobi diagonal (tiled, fp64 arithmetic: DESIGN.md R14)
//   M = I + grad u, F(u) = M F^n, J = det M det F^n,  Ah = M^{-T},  S' = V0 mu F^n F^nT
//   G_grad = V0 P(F(u)) F^nT = M S' - c' Ah ;  diag_a += gradN^T (S' + (c' + l') Ah_a Ah_a^T) gradN
//   V0 Psi = 1/2 (tr(M S' M^T) - V0 mu d) - V0 mu ln J + V0 lam/2 ln^2 J
// partials per CTA: {sum V0 Psi, sum V0 |Psi|, inverted}
// =============================================================================================
template <int D>
constexpr size_t grad_smem_bytes()
{
    using T = Tile<D>;
    constexpr size_t rec = (size_t)GradRec<D>::RS * T::NT;
    constexpr size_t recstg = rec > (size_t)Stage<D>::SIZE ? rec : (size_t)Stage<D>::SIZE;
    return ((size_t)T::NN * SV<D>::S + 2 * T::NN * D + recstg) * sizeof(double);
}

template <int D, typename R>
__global__ void __launch_bounds__(Tile<D>::NT)
k_grad(const R* __restrict__ P, R* __restrict__ cache, int64_t cap, const int* __restrict__ mat,
       const int* __restrict__ cell_start, BoxDev b, MatTable mt, const double* __restrict__ uin,
       double* __restrict__ gout, double* __restrict__ dout, double* __restrict__ partials)
{
    using T = Tile<D>;
    using GR = GradRec<D>;
    using L = PL<D>;
    using C = CL<D>;
    using Rd = double;
    constexpr int RS = GR::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Rd* sv = reinterpret_cast<Rd*>(smem_raw);
    Rd* sy = sv + T::NN * SV<D>::S;  // [0]: gradient tile, [NN*D]: diagonal tile
    Rd* rec = sy + 2 * T::NN * D;
    Rd* stg = rec;
    const int tile = blockIdx.x;
    const int64_t kt = (int64_t)tile * T::NC;
    double red[3] = {0.0, 0.0, 0.0};
    __shared__ int scs[T::NC + 1];  // the tile's cell ranges
    for (int i = threadIdx.x; i <= T::NC; i += T::NT) scs[i] = cell_start[kt + i];
    __syncthreads();
    if (scs[0] == scs[T::NC]) {
        if (threadIdx.x == 0) {
            partials[blockIdx.x * 3 + 0] = 0.0;
            partials[blockIdx.x * 3 + 1] = 0.0;
            partials[blockIdx.x * 3 + 2] = 0.0;
        }
        return;
    }
    int t[3];
    tile_coords<D>(b, tile, t);
    stage_nodes<D, Rd, 2>(b, t, uin, sv, sy);
    __syncthreads();
    const int it = threadIdx.x;
    const int icell = it / (D * 3), icomp = (it / 3) % D, ii = it % 3;
    for (int layer = 0; layer < T::NL; ++layer) {
        const int lb = scs[layer * T::LC], le = scs[(layer + 1) * T::LC];
        if (lb == le) continue;
        const int ks = scs[layer * T::LC + icell];
        const int ke = scs[layer * T::LC + icell + 1];
        Rd acc[T::NACC], accd[T::NACC];
#pragma unroll
        for (int k = 0; k < T::NACC; ++k) acc[k] = accd[k] = 0.0;
        for (int sb = lb; sb < le; sb += T::NT) {
            const int se = min(sb + T::NT, le);
            const int q = threadIdx.x, p = sb + q;
            if (p < se) {
                Rd x[3], w[3][3], dw[3][3];
                int lc[3] = {0, 0, 0};
#pragma unroll
                for (int a = 0; a < D; ++a) x[a] = (Rd)P[(L::X + a) * cap + p];
                weights_at<D, Rd>(x, b, t, lc, w, dw);
                Rd Mx[D * D];
                gather_grad<D, Rd>(sv, lc, w, dw, Mx);
                const RecPtr<Rd> r(rec, q, RS);
                store_weights<D, Rd>(r, w, dw);
#pragma unroll
                for (int a = 0; a < D; ++a) Mx[a * D + a] += 1.0;
                Rd Fn[D * D];
#pragma unroll
                for (int k = 0; k < D * D; ++k) Fn[k] = (Rd)P[(L::F + k) * cap + p];
                const Rd V0 = (Rd)P[L::VOL * cap + p];
                const int mid = mat[p];
                const Rd mu = mt.mu[mid], lam = mt.lam[mid];
                Rd S[Sym<D>::N];
#pragma unroll
                for (int a = 0; a < D; ++a)
#pragma unroll
                    for (int bb = a; bb < D; ++bb) {
                        Rd s = 0;
#pragma unroll
                        for (int k = 0; k < D; ++k) s = fma(Fn[a * D + k], Fn[bb * D + k], s);
                        S[sym_idx<D>(a, bb)] = V0 * mu * s;
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
                        Rd s = 0;
#pragma unroll
                        for (int k = 0; k < D; ++k) s = fma(Mx[a * D + k], S[sym_idx<D>(k, bb)], s);
                        trMSM = fma(s, Mx[a * D + bb], trMSM);
                        *r.at(Rec<D>::G + a * D + bb) = fma(-cc, Ah[a * D + bb], s);
                    }
                const Rd psiV = 0.5 * (trMSM - V0 * mu * D) - V0 * mu * lnJ + 0.5 * V0 * lam * lnJ * lnJ;
                red[0] += psiV;
                red[1] += fabs(psiV);
                if (!ok) red[2] += 1.0;
#pragma unroll
                for (int k = 0; k < Sym<D>::N; ++k) {
                    *r.at(GR::S + k) = S[k];
                    cache[(C::S + k) * cap + p] = (R)S[k];
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
            __syncthreads();
            if (it < T::ITEMS) {
                const int p0 = max(ks, sb), p1 = min(ke, se);
                const int len = p1 - p0, rot = len > 0 ? (icell & 7) % len : 0;
                for (int k = 0; k < len; ++k) {
                    const RecPtr<Rd> r(rec, rotated(p0, len, k, rot) - sb, RS);
                    ItemW<D, Rd> W;
                    W.load(r, ii);
                    Rd s[D], Ar[D], Q[Sym<D>::N];
#pragma unroll
                    for (int bb = 0; bb < D; ++bb) {
                        s[bb] = *r.at(Rec<D>::G + icomp * D + bb);
                        Ar[bb] = *r.at(GR::A + icomp * D + bb);
                    }
                    const Rd clv = *r.at(GR::CL);
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int bb = a; bb < D; ++bb)
                            Q[sym_idx<D>(a, bb)] = fma(clv * Ar[a], Ar[bb], *r.at(GR::S + sym_idx<D>(a, bb)));
                    item_linear<D, Rd>(s, W, acc);
                    item_quadratic<D, Rd>(Q, W, accd);
                }
            }
            __syncthreads();
        }
        stage_zero<D, Rd>(stg);
        __syncthreads();
        if (it < T::ITEMS) stage_item<D, Rd>(icell, icomp, ii, acc, stg);
        __syncthreads();
        layer_flush<D, Rd>(layer, stg, sy);
        __syncthreads();
        stage_zero<D, Rd>(stg);
        __syncthreads();
        if (it < T::ITEMS) stage_item<D, Rd>(icell, icomp, ii, accd, stg);
        __syncthreads();
        layer_flush<D, Rd>(layer, stg, sy + T::NN * D);
        __syncthreads();
    }
    tile_flush<D, Rd>(b, t, sy, gout);
    tile_flush<D, Rd>(b, t, sy + T::NN * D, dout);
    block_reduce_store<3>(red, partials);
}

}  // namespace osmpm
