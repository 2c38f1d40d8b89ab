// device.cuh -- sm_100a device helpers of the OS-MPM hot path: tile geometry, the quadratic
// B-spline (kernel choice DESIGN.md R1), small-matrix algebra, reductions.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace osmpm {

// ---------------------------------------------------------------------------------------------
// Tile geometry.  Particles are binned by the base node b = floor((x - o)/dx - 1/2) of their
// quadratic stencil ("cell" b covers nodes b..b+2).  Cells are grouped into tiles of T0 x T1 x T2
// cells; a tile owns the (T0+2)(T1+2)(T2+2) nodes its particles touch.  One CTA per tile.
// ---------------------------------------------------------------------------------------------
// Inside a tile, cells are ordered LAYER-MAJOR along the last axis (z in 3D, y in 2D): a layer
// is the LC = T0 (x T1) cells with one last-axis index; the tiled kernels walk the layers in order.
#ifndef OSMPM_T2
// layers per 3D tile (cells along z).  C5 step, ms (HVP per step): 8 -> 748.1 (624.3), 10 -> 734.1 (612.8),
// 12 -> 734.5 (612.1), 14 -> 798.4 (672.4); deeper tiles amortise the two tail planes and the tile
// prologue over more layers until the node tile no longer leaves room for three HVP CTAs per SM
#define OSMPM_T2 12
#endif
template <int D> struct Tile;
template <> struct Tile<3> {
    static constexpr int T0 = 4, T1 = 4, T2 = OSMPM_T2;
    static constexpr int NC = T0 * T1 * T2;                   // cells per tile
    static constexpr int LC = T0 * T1;                        // cells per layer
    static constexpr int NL = T2;                             // layers per tile
    static constexpr int N0 = T0 + 2, N1 = T1 + 2, N2 = T2 + 2;
    static constexpr int NN = N0 * N1 * N2;                   // nodes per tile
    static constexpr int NS = 27;                             // stencil nodes
    static constexpr int K3 = 3;
    static constexpr int ITEMS = LC * 3 * 3;                  // scatter items (cell, comp, i)
    static constexpr int NACC = 9;                            // accumulators per item (j, k)
    static constexpr int NT = 144;                            // threads per CTA (= ITEMS)
};
template <> struct Tile<2> {
    static constexpr int T0 = 16, T1 = 4, T2 = 1;
    static constexpr int NC = T0 * T1;
    static constexpr int LC = T0;
    static constexpr int NL = T1;
    static constexpr int N0 = T0 + 2, N1 = T1 + 2, N2 = 1;
    static constexpr int NN = N0 * N1;
    static constexpr int NS = 9;
    static constexpr int K3 = 1;
    static constexpr int ITEMS = LC * 2 * 3;
    static constexpr int NACC = 3;                            // accumulators per item (j)
    static constexpr int NT = 96;                             // threads per CTA (= ITEMS)
};

// Node box of the current step (all integers are global node / cell indices).
struct BoxDev {
    int lo[3];      // global node index of box node 0 (= lowest base node of any particle)
    int nc[3];      // cells per axis, padded to a tile multiple (1 on unused axes)
    int nn[3];      // nodes per axis = nc + 2 (1 on unused axes)
    int nt[3];      // tiles per axis
    int gdims[3];   // dims of the global (dense) node box
    double o[3];    // global origin
    double dx, inv_dx;
    int64_t nnodes, ncells;
    int ntiles;
};

template <int D>
__device__ __forceinline__ int64_t box_node(const BoxDev& b, int i0, int i1, int i2)
{
    if (D == 3) return ((int64_t)i0 * b.nn[1] + i1) * b.nn[2] + i2;
    return (int64_t)i0 * b.nn[1] + i1;
}

// tile-major cell key of box-local cell c
template <int D>
__device__ __forceinline__ uint32_t cell_key(const BoxDev& b, int c0, int c1, int c2)
{
    using T = Tile<D>;
    int t0 = c0 / T::T0, t1 = c1 / T::T1, t2 = (D == 3) ? c2 / T::T2 : 0;
    int l0 = c0 - t0 * T::T0, l1 = c1 - t1 * T::T1, l2 = (D == 3) ? c2 - t2 * T::T2 : 0;
    uint32_t tile = (D == 3) ? ((uint32_t)t0 * b.nt[1] + t1) * b.nt[2] + t2 : (uint32_t)t0 * b.nt[1] + t1;
    // layer-major: the last axis is slowest inside the tile
    uint32_t loc = (D == 3) ? (l2 * T::T0 + l0) * T::T1 + l1 : l1 * T::T0 + l0;
    return tile * T::NC + loc;
}

// ---------------------------------------------------------------------------------------------
// quadratic B-spline, per axis: f = X - base in [1/2, 3/2) (R1)
// ---------------------------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ void bspline(R f, R inv_dx, R* w, R* dw)
{
    R a = R(1.5) - f, b = f - R(1), c = f - R(0.5);
    w[0] = R(0.5) * a * a;
    w[1] = R(0.75) - b * b;
    w[2] = R(0.5) * c * c;
    dw[0] = -a * inv_dx;
    dw[1] = R(-2) * b * inv_dx;
    dw[2] = c * inv_dx;
}

// base node (global) and fractional offset of a particle along one axis
template <typename R>
__device__ __forceinline__ int base_of(R x, double o, double inv_dx, R* f)
{
    double X = ((double)x - o) * inv_dx;
    double b = floor(X - 0.5);
    *f = (R)(X - b);
    return (int)b;
}

// ---------------------------------------------------------------------------------------------
// small matrices (row-major)
// ---------------------------------------------------------------------------------------------
template <int D, typename T>
__device__ __forceinline__ T det(const T* A)
{
    if (D == 2) return A[0] * A[3] - A[1] * A[2];
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}

// cofactor matrix (= det(A) * A^{-T})
template <int D, typename T>
__device__ __forceinline__ void cofactor(const T* A, T* C)
{
    if (D == 2) {
        C[0] = A[3]; C[1] = -A[2]; C[2] = -A[1]; C[3] = A[0];
        return;
    }
    C[0] = A[4] * A[8] - A[5] * A[7];
    C[1] = A[5] * A[6] - A[3] * A[8];
    C[2] = A[3] * A[7] - A[4] * A[6];
    C[3] = A[2] * A[7] - A[1] * A[8];
    C[4] = A[0] * A[8] - A[2] * A[6];
    C[5] = A[1] * A[6] - A[0] * A[7];
    C[6] = A[1] * A[5] - A[2] * A[4];
    C[7] = A[2] * A[3] - A[0] * A[5];
    C[8] = A[0] * A[4] - A[1] * A[3];
}

// symmetric D x D stored as D(D+1)/2: 3D (00,11,22,01,02,12), 2D (00,11,01)
template <int D> struct Sym { static constexpr int N = D * (D + 1) / 2; };
template <int D>
__device__ __forceinline__ int sym_idx(int a, int b)
{
    if (a == b) return a;
    if (D == 2) return 2;
    int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo == 0 ? (hi == 1 ? 3 : 4) : 5;
}

// ---------------------------------------------------------------------------------------------
// block reduction of NV doubles -> partials[blockIdx.x * NV + k]  (deterministic order)
// ---------------------------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_reduce_store(double* v, double* partials)
{
    __shared__ double red[32][NV];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = v[k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        v[k] = s;
    }
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) red[wid][k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[w][k];
            partials[(int64_t)blockIdx.x * NV + k] = s;
        }
    }
}

// single-block final sum of nb partial vectors (fixed order -> bitwise reproducible)
template <int NV>
__device__ __forceinline__ void final_sum(const double* partials, int nb, double* out)
{
    __shared__ double red[32][NV];
    double v[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = 0.0;
#pragma unroll 4
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] += partials[(int64_t)i * NV + k];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = v[k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        v[k] = s;
    }
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) red[wid][k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[w][k];
            out[k] = s;
        }
    }
}

// device-side error latch: first error wins
struct ErrLatch {
    int code;       // osmpm_status
    int pad;
    long long index; // creation index of the offending particle
};
__device__ __forceinline__ void latch_error(ErrLatch* e, int code, long long index)
{
    if (atomicCAS(&e->code, 0, code) == 0) e->index = index;
}

}  // namespace osmpm
