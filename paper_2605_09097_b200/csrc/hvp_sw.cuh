// hvp_sw.cuh -- sliding-window tiled Hessian-vector product (a5), the default HVP.
//
// Same arithmetic as k_hvp (tiled.cuh):  y += sum_p G_p grad N_p,
//   G_p = gd S' + c' Ah gd^T Ah + l' (Ah : gd) Ah,   gd = sum_j d_j grad N_j^T
// (derived from PAPER.md:188 Eq. F_update and PAPER.md:208, K = d^2 Phi).
//
// One CTA per tile of cells, layers walked in order along the last axis.  Differences from k_hvp:
//  * sliding window: a scatter item (cell, component a, x-offset i) keeps 3 node planes of
//    accumulators (last-axis offsets kk = 0, 1, 2 relative to the current layer).  After layer L the
//    kk = 0 plane (node plane L) has received every contribution it will ever get from this tile
//    (layers L-2, L-1, L), so the item emits it and shifts the window.  There is no shared-memory
//    node accumulator tile, no per-layer zeroing, and 3x fewer staged partials.
//  * per emitted plane, the staged partials (one slot per contributing cell; slots of cells outside
//    the tile are zeroed once and never written) are summed in a fixed order and written with one
//    fp64 RED per node and component straight to global memory.
//  * two CTA barriers per layer (records ready / plane staged) instead of six.
//  * the node tile is stored with a padded row stride so that the four cells of a warp's lanes hit
//    distinct bank groups in the tensor-product gather.
// Particle inputs (x + Newton cache) are streamed with TMA bulk copies (cp.async.bulk + mbarrier),
// the next non-empty layer in flight while the current one computes.
#pragma once
#include <cuda.h>  // CUtensorMap (the encoder is fetched at run time: cudaGetDriverEntryPoint)

#include "osmpm.h"

#include "tiled.cuh"

namespace osmpm {

// threads of an HVP CTA.  3D: 128 = 16 cells x 8 (component, x-offset) items, four full warps; the
// ninth item (component 2, x-offset 2) of each cell is split over the cell's eight lanes, one particle
// each (SPLIT9), and its emitted plane is summed over them with shuffles -- instead of a fifth,
// half-populated warp that idles through phase 1 and runs its FP64 work at half width.  2D: 96.
template <int D> struct HvpT {
    static constexpr int NT = (D == 3) ? 128 : Tile<D>::NT;
    static constexpr bool SPLIT9 = D == 3;
};
// warps per HVP CTA (the per-warp curvature partials of k_hvp_sw)
template <int D> constexpr int HVP_NW = (HvpT<D>::NT + 31) / 32;

template <int D, typename R> struct SWRec {
    // G row a starts at GROW(a): 3D fp64 rows padded to 4 reals (16-B aligned: one 16-B + one 8-B load
    // per row; the 30-real record has exactly the room), otherwise packed
    static constexpr int GP = (D == 3 && sizeof(R) == 8) ? 4 : D;
    static constexpr int RS = HvpRec<D, R>::RS;
    // Records of the particles of layer cell c start SK reals (16 B) per cell further on: the quarter
    // warps of phase 2 (one cell each) read their cells' k-th records at bank-group offsets 15k + 121c
    // (mod 8, fp64, 8 particles per cell) -- distinct without rotating each cell's particle order, so
    // the record addresses are per-thread bases plus compile-time offsets (no per-particle index math)
    static constexpr int SK = 16 / sizeof(R);
};

template <int D> struct SW {
    using T = Tile<D>;
    static constexpr int NZP = (D == 3) ? T::N2 : T::N1;  // last-axis stride of the node tile
    static constexpr int NNP = (D == 3) ? T::N0 * T::N1 * NZP : T::N0 * T::N1;
    static constexpr int NLAT = (D == 3) ? T::N0 * T::N1 : T::N0;   // lateral nodes of a plane
    static constexpr int NSLOT = (D == 3) ? 9 : 3;                  // contributing cells per node
    static constexpr int NITEM = NLAT * D;                          // (lateral node, comp)
    static constexpr int STG = NITEM * NSLOT;
    static constexpr int NACC = T::NACC;                            // 3D: (j, kk); 2D: kk
};

// reals per node of the node tile: 3D fp64 3 (24-B nodes; with 4x4xT2 tiles the rows of the four
// cells of a warp's lanes start 4 banks apart: conflict-free 8-B loads), 3D fp32 4 (16-B nodes), 2D 2
template <int D, typename R> struct SVS {
    static constexpr int S = (D == 3) ? (sizeof(R) == 8 ? 3 : 4) : 2;
    // 3D fp64 split layout: components 0,1 as 16-B pairs [NNP][2], component 2 as a
    // separate [NNP] plane -- one 16-B and one 8-B load per node instead of three 8-B loads, same
    // footprint; rows of 10 nodes put the four cells of a warp at bank offsets 0/8/16/24 (pairs) and
    // 0/20/8/28 (plane): conflict-free
    static constexpr bool SPLIT = D == 3 && sizeof(R) == 8;
};
// shared-memory element of (node, component) in the node tile
template <int D, typename R>
__device__ __forceinline__ int sv_elem(int node, int a, int nnp)
{
    if constexpr (SVS<D, R>::SPLIT) return a < 2 ? node * 2 + a : 2 * nnp + node;
    return node * SVS<D, R>::S + a;
}

template <int D>
__device__ __forceinline__ int sw_node(int l0, int l1, int l2)
{
    using T = Tile<D>;
    return (D == 3) ? (l0 * T::N1 + l1) * SW<D>::NZP + l2 : l0 * T::N1 + l1;
}

// node values of a node vector (fp64, components innermost) on the tile's nodes -> the node tile.
// fp64 tiles: cp.async (LDGSTS) so every thread's loads are in flight at once instead of one
// load-store round trip each (the tile prologue is latency-bound); the caller's barrier follows
// cp.async.wait_all.  fp32 tiles convert through registers.
__device__ __forceinline__ void cp_async_8(void* sdst, const void* gsrc)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
template <int D, typename R, int NTHR, bool WAIT = true>
__device__ __forceinline__ void sw_stage_tile(const BoxDev& b, const int* t, const double* __restrict__ src, R* sv)
{
    using T = Tile<D>;
    constexpr int ROWS = T::N0 * T::N1, RL = T::N2 * D;  // 3D: rows along z are contiguous in global memory
    if constexpr (D == 3 && NTHR >= ROWS) {
        // thread -> (row, part): one row base address per thread, then every TPR-th element of the row
        // with its (node, component) advanced incrementally (no per-element index divisions); threads
        // beyond TPR * ROWS stay idle
        constexpr int TPR = NTHR / ROWS;
        const int row = threadIdx.x / TPR, part = threadIdx.x % TPR;
        if (row < ROWS) {
            const int c0 = row / T::N1, c1 = row % T::N1;
            const double* gs = src + box_node<D>(b, t[0] * T::T0 + c0, t[1] * T::T1 + c1, t[2] * T::T2) * D;
            const int n0 = sw_node<D>(c0, c1, 0);
            int z = part / D, a = part % D;
#pragma unroll
            for (int e = part; e < RL; e += TPR) {
                R* dst = sv + sv_elem<D, R>(n0 + z, a, SW<D>::NNP);
                if constexpr (sizeof(R) == 8)
                    cp_async_8(dst, gs + e);
                else
                    *dst = (R)gs[e];
                a += TPR % D;
                z += TPR / D;
                if (a >= D) {
                    a -= D;
                    z += 1;
                }
            }
        }
    } else {
        for (int idx = threadIdx.x; idx < T::NN * D; idx += NTHR) {
            const int a = idx % D, l = idx / D;
            int c[3];
            tnode_coords<D>(l, c);
            const int64_t g = box_node<D>(b, t[0] * T::T0 + c[0], t[1] * T::T1 + c[1], t[2] * T::T2 + c[2]);
            R* dst = sv + sv_elem<D, R>(sw_node<D>(c[0], c[1], c[2]), a, SW<D>::NNP);
            if constexpr (sizeof(R) == 8)
                cp_async_8(dst, src + g * D + a);
            else
                *dst = (R)src[g * D + a];
        }
    }
    if constexpr (sizeof(R) == 8)
        if (WAIT) asm volatile("cp.async.wait_all;" ::: "memory");
}

// host: tensor maps of the streamed HVP inputs (x of the particle SoA, the Newton cache) as 2-D
// tensors [fields][cap] with one box of {PFS particles, all fields}
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static inline PFN_encodeTiled encode_tiled_fn()
{
    static PFN_encodeTiled fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}
// Shared-memory block of one layer's streamed inputs: x (D fields) then the Newton cache (CL::NF
// fields), PFS particles per field starting at the 16-B aligned particle lb0 = lb & ~(UE - 1) (<= UE - 1
// slack + NT particles, rounded to 16 B).  The x block is padded to 128 B so that both blocks are
// destinations of 2-D tensor copies (128-B aligned shared memory; the tensor start coordinate must
// be 16-B aligned too: measured, scripts/tma_probe.cu).
template <int D, typename R> struct SWIn {
    static constexpr int NF = D + CL<D>::NF;
    static constexpr int UE = 16 / sizeof(R);
    static constexpr int PFS = HvpT<D>::NT + UE;
    static constexpr int XB = (int)(((D * PFS * sizeof(R) + 127) / 128 * 128) / sizeof(R));
    static constexpr int TOT = XB + CL<D>::NF * PFS;
    static __host__ __device__ constexpr int off(int f) { return f < D ? f * PFS : XB + (f - D) * PFS; }
};
static_assert(HvpT<3>::NT % 4 == 0 && HvpT<2>::NT % 4 == 0, "NT a multiple of the 16-B unit");

template <typename R>
static inline bool encode_fields_map(CUtensorMap* m, const R* base, int nfields, int64_t cap, int box_particles)
{
    PFN_encodeTiled fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cap, (cuuint64_t)nfields};
    const cuuint64_t strides[1] = {(cuuint64_t)cap * sizeof(R)};
    const cuuint32_t box[2] = {(cuuint32_t)box_particles, (cuuint32_t)nfields};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
              const_cast<R*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, typename R>
constexpr size_t hvp_sw_smem_bytes()
{
    using T = Tile<D>;
    return 16 + 128 /* alignment of the streamed-input block */ + ((size_t)SW<D>::NNP * SVS<D, R>::S + SW<D>::STG +
                 (size_t)SWIn<D, R>::TOT +
                 (size_t)SWRec<D, R>::RS * HvpT<D>::NT + (size_t)T::LC * SWRec<D, R>::SK) *
                    sizeof(R);
}

// gd[a][b] = sum_i d_i,a dN_i/dx_b from the padded node tile (tensor-product order, explicit FMA)
template <int D, typename R>
__device__ __forceinline__ void sw_gather(const R* sv, const int* lc, const R (*w)[3], const R (*dw)[3], R* gd)
{
    using V2 = typename Vec2<R>::type;
    using T = Tile<D>;
#pragma unroll
    for (int k = 0; k < D * D; ++k) gd[k] = R(0);
    if constexpr (D == 3 && sizeof(R) == 4) {
        // fp32 tiles: the same FMAs in the same order, paired into FFMA2 (fma.rn.f32x2: two lanes per
        // issue; the FMA pipe takes a scalar FFMA only every second cycle per SMSP) -- (T0, T1) against
        // (w_k, dw_k), (U0, U1) against (w_j, dw_j), (gd_1, gd_2) against w_i; bitwise the scalar result
        const int n0 = sw_node<D>(lc[0], lc[1], lc[2]);
        const float* base = reinterpret_cast<const float*>(sv) + n0 * 4;
        float2 wz[3], wy[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            wz[k] = make_float2((float)w[2][k], (float)dw[2][k]);
            wy[k] = make_float2((float)w[1][k], (float)dw[1][k]);
        }
        float g0[3] = {0.f, 0.f, 0.f};
        float2 g12[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            float2 U01[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float U2[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                float2 Tp[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const float4 v = *reinterpret_cast<const float4*>(base + ((i * T::N1 + j) * SW<D>::NZP + k) * 4);
                    Tp[0] = __ffma2_rn(make_float2(v.x, v.x), wz[k], Tp[0]);
                    Tp[1] = __ffma2_rn(make_float2(v.y, v.y), wz[k], Tp[1]);
                    Tp[2] = __ffma2_rn(make_float2(v.z, v.z), wz[k], Tp[2]);
                }
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    U01[a] = __ffma2_rn(make_float2(Tp[a].x, Tp[a].x), wy[j], U01[a]);
                    U2[a] = fmaf(Tp[a].y, wy[j].x, U2[a]);
                }
            }
            const float w0 = (float)w[0][i], dw0 = (float)dw[0][i];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                g0[a] = fmaf(U01[a].x, dw0, g0[a]);
                g12[a] = __ffma2_rn(make_float2(U01[a].y, U2[a]), make_float2(w0, w0), g12[a]);
            }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            gd[a * 3 + 0] = (R)g0[a];
            gd[a * 3 + 1] = (R)g12[a].x;
            gd[a * 3 + 2] = (R)g12[a].y;
        }
    } else if (D == 3) {
        constexpr int NS = SVS<D, R>::S;
        const int n0 = sw_node<D>(lc[0], lc[1], lc[2]);
        const R* base = sv + n0 * NS;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            R U0[3] = {0, 0, 0}, U1[3] = {0, 0, 0}, U2[3] = {0, 0, 0};
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                R T0[3] = {0, 0, 0}, T1[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const int off = (i * T::N1 + j) * SW<D>::NZP + k;
                    const R* sp = base + off * NS;
                    R s[3];
                    if constexpr (SVS<D, R>::SPLIT) {
                        const V2 v01 = *reinterpret_cast<const V2*>(sv + (n0 + off) * 2);
                        s[0] = v01.x;
                        s[1] = v01.y;
                    } else if constexpr (NS == 4) {
                        const V2 v01 = *reinterpret_cast<const V2*>(sp);
                        s[0] = v01.x;
                        s[1] = v01.y;
                    } else {
                        s[0] = sp[0];
                        s[1] = sp[1];
                    }
                    s[2] = SVS<D, R>::SPLIT ? sv[2 * SW<D>::NNP + n0 + off] : sp[2];
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
        gather_grad<D, R>(sv, lc, w, dw, gd);
    }
}

// item (cell, a, i): emit the completed kk = 0 plane into the staging slots, shift the window
template <int V> struct ICst { static constexpr int value = V; };

template <int D, typename R>
__device__ __forceinline__ void sw_emit(int cellL, int a, int i, R* acc, R* stg)
{
    using T = Tile<D>;
    if (D == 3) {
        const int cx = cellL / T::T1, cy = cellL % T::T1;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int nxy = (cx + i) * T::N1 + (cy + j);
            stg[(i * 3 + j) * SW<D>::NITEM + nxy * 3 + a] = acc[j * 3 + 0];  // slot-major
            acc[j * 3 + 0] = acc[j * 3 + 1];
            acc[j * 3 + 1] = acc[j * 3 + 2];
            acc[j * 3 + 2] = R(0);
        }
    } else {
        stg[i * SW<D>::NITEM + (cellL + i) * 2 + a] = acc[0];
        acc[0] = acc[1];
        acc[1] = acc[2];
        acc[2] = R(0);
    }
}

// Fused halo of the HVP over x-slabs (R24).  The last two x node planes
// of a slab with a right neighbour are that neighbour's first two planes.  Instead of a halo pass after
// the HVP (reverse-add of the ghost planes, copy back), every flushed partial sum of a node on those
// planes is also RED-ed into the neighbour's copy of y -- a slab on the same device, or the neighbouring
// rank's buffer mapped over NVLink (CUDA IPC) -- so that both copies hold the complete sum when the
// kernels of both slabs have finished.  Between ranks, the last CTA of the kernel bumps the neighbours'
// inbox words after a system-scope fence; the consumer waits for them (k_halo_wait).
struct HaloDev {
    double* yL = nullptr;       // left neighbour's y: its last two planes are this slab's planes 0, 1
    double* yR = nullptr;       // right neighbour's y: its planes 0, 1 are this slab's last two
    int64_t offL = 0, offR = 0;  // node-index offsets of this box's nodes in yL / yR
    int ixR = 0x7fffffff;        // first box x-plane shared with the right neighbour
    unsigned* done = nullptr;    // CTA completion counter of the launch (own memory; the last CTA resets it)
    unsigned* sigL = nullptr;    // inbox words of remote neighbours, bumped once per launch
    unsigned* sigR = nullptr;
};

// fire-and-forget fp64 reduction (RED, no return value).  Spelled out: with the system-scope fence of
// halo_signal in the same kernel, nvcc emits atomicAdd as ATOM with a return (measured 6 % slower HVP)
__device__ __forceinline__ void red_add(double* p, double v)
{
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// the CTA's REDs into peer memory are complete before the launch's last CTA signals the remote
// neighbours (release: system-scope fence of every thread, then one atomic per neighbour)
__device__ __forceinline__ void halo_signal(const HaloDev& h)
{
    if (!h.sigL && !h.sigR) return;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(h.done, 1u);
        if (prev == gridDim.x - 1) {
            *h.done = 0u;
            __threadfence_system();
            if (h.sigL) atomicAdd_system(h.sigL, 1u);
            if (h.sigR) atomicAdd_system(h.sigR, 1u);
        }
    }
}

// the consumer side: wait until the inbox words reach the expected launch counts (acquire, system
// scope); a neighbour that does not arrive within ~10 s latches OSMPM_E_CUDA instead of hanging
__global__ void k_halo_wait(const unsigned* inbox, unsigned expL, unsigned expR, ErrLatch* err)
{
    if (threadIdx.x != 0) return;
    const long long t0 = clock64();
    for (;;) {
        unsigned l, r;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(l) : "l"(inbox) : "memory");
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(r) : "l"(inbox + 1) : "memory");
        if ((int)(l - expL) >= 0 && (int)(r - expR) >= 0) return;
        if (clock64() - t0 > 20000000000LL) {
            latch_error(err, OSMPM_E_CUDA, -1);
            return;
        }
        __nanosleep(200);
    }
}

// Plane flush: fixed-order NSLOT-term sums of plane `plane` (tile-local last-axis node index) -> one RED each
//
// Deterministic mode (tb != nullptr, OSMPM_DETERMINISTIC=1): instead of the RED, every sum (zeros
// included) is stored to the tile's own block of node values tb[tile-local node][component]; the node
// pass k_det_gather then adds the <= 2^D tile blocks covering each node in a fixed tile order, so the
// result does not depend on the order in which tiles finish (bitwise reproducible).
// With DOT, the flushing thread also accumulates d_node . (this tile's partial y_node) into dot: summed
// over all tiles that is d^T K d, the PCG curvature (no separate pass over y), from d as staged in the
// node tile (fp64) or re-read from global memory (fp32 tiles hold d rounded).
// With a HaloDev (fused halo, R24), sums of nodes on planes shared with a neighbouring slab also go to
// the neighbour's copy.
// The thread's flush item is fixed for the whole tile (NITEM <= threads): its node / component,
// global node index, node-tile element, tile-block index and halo targets are computed once per tile and
// advance by one node per plane (x slowest, the last axis fastest in both the box and the node tile), so
// a plane's flush is the fixed-order slot sum, the RED and nothing else.  Same sums, same order.
template <int D, typename R>
struct FlushItem {
    bool valid = false, toR = false, toL = false;
    int a = 0, it = 0, ln0 = 0, tb0 = 0;
    int64_t g0 = 0;
    __device__ __forceinline__ FlushItem(const BoxDev& b, const int* t, const HaloDev* hl)
    {
        using T = Tile<D>;
        static_assert(SW<D>::NITEM <= Tile<D>::NT && SW<D>::NITEM <= HvpT<D>::NT, "one flush item per thread");
        it = threadIdx.x;
        valid = it < SW<D>::NITEM;
        a = it % D;
        const int nxy = it / D;
        const int l0 = (D == 3) ? nxy / T::N1 : nxy, l1 = (D == 3) ? nxy % T::N1 : 0;
        if (D == 3) {
            g0 = box_node<D>(b, t[0] * T::T0 + l0, t[1] * T::T1 + l1, t[2] * T::T2);
            ln0 = sw_node<D>(l0, l1, 0);
            tb0 = nxy * T::N2;
        } else {
            g0 = box_node<D>(b, t[0] * T::T0 + l0, t[1] * T::T1, 0);
            ln0 = sw_node<D>(l0, 0, 0);
            tb0 = nxy * T::N1;
        }
        if (hl) {
            const int ix = t[0] * T::T0 + l0;
            toR = hl->yR && ix >= hl->ixR;
            toL = hl->yL && ix < 2;
        }
    }
    template <bool DOT>
    __device__ __forceinline__ void flush(int plane, const R* stg, double* __restrict__ out, double* __restrict__ tb,
                                          const R* sv, const double* __restrict__ din, double& dot,
                                          const HaloDev* hl) const
    {
        if (!valid) return;
        R s = stg[it];
#pragma unroll
        for (int k = 1; k < SW<D>::NSLOT; ++k) s += stg[k * SW<D>::NITEM + it];
        if (tb) tb[(tb0 + plane) * D + a] = (double)s;
        if (s != R(0) && (tb == nullptr || DOT)) {
            const int64_t g = g0 + plane;
            if (!tb) {
                red_add(&out[g * D + a], (double)s);
                if (hl) {
                    if (toR) red_add(&hl->yR[(g + hl->offR) * D + a], (double)s);
                    if (toL) red_add(&hl->yL[(g + hl->offL) * D + a], (double)s);
                }
            }
            if constexpr (DOT) {
                double dv;
                if constexpr (sizeof(R) == 8)
                    dv = (double)sv[sv_elem<D, R>(ln0 + plane, a, SW<D>::NNP)];
                else
                    dv = din[g * D + a];
                dot = fma(dv, (double)s, dot);
            }
        }
    }
};

// out[node] = sum over the non-empty tiles covering the node, in increasing tile order per axis, of
// the tile blocks written by sw_flush in deterministic mode (all nodes of the box, plain stores)
template <int D, int NC = D>
__global__ void k_det_gather(BoxDev b, const int* __restrict__ cell_start, const double* __restrict__ tb,
                             double* __restrict__ out)
{
    using T = Tile<D>;
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= b.nnodes) return;
    const int tt[3] = {T::T0, T::T1, T::T2};
    int ix[3] = {0, 0, 0};
    if (D == 3) {
        ix[2] = (int)(n % b.nn[2]);
        ix[1] = (int)((n / b.nn[2]) % b.nn[1]);
        ix[0] = (int)(n / ((int64_t)b.nn[2] * b.nn[1]));
    } else {
        ix[1] = (int)(n % b.nn[1]);
        ix[0] = (int)(n / b.nn[1]);
    }
    // per axis: the tiles t with t T <= i <= t T + T + 1 (one or two), lowest first
    int tl[3][2], nt[3] = {1, 1, 1};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (a >= D) {
            tl[a][0] = 0;
            continue;
        }
        const int t1 = min(ix[a] / tt[a], b.nt[a] - 1);
        if (t1 > 0 && ix[a] - t1 * tt[a] <= 1) {
            tl[a][0] = t1 - 1;
            tl[a][1] = t1;
            nt[a] = 2;
        } else {
            tl[a][0] = t1;
        }
    }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int u = 0; u < nt[0]; ++u)
        for (int v = 0; v < nt[1]; ++v)
            for (int w = 0; w < nt[2]; ++w) {
                const int tx = tl[0][u], ty = tl[1][v], tz = tl[2][w];
                const int tile = (D == 3) ? (tx * b.nt[1] + ty) * b.nt[2] + tz : tx * b.nt[1] + ty;
                const int64_t kt = (int64_t)tile * T::NC;
                if (cell_start[kt] == cell_start[kt + T::NC]) continue;  // empty tile: block not written
                const int lx = ix[0] - tx * T::T0, ly = ix[1] - ty * T::T1, lz = ix[2] - tz * T::T2;
                const int ln = (D == 3) ? (lx * T::N1 + ly) * T::N2 + lz : lx * T::N1 + ly;
                const double* p = tb + ((int64_t)tile * T::NN + ln) * NC;
#pragma unroll
                for (int a = 0; a < NC; ++a) acc[a] += p[a];
            }
#pragma unroll
    for (int a = 0; a < NC; ++a) out[n * NC + a] = acc[a];
}

// TMA bulk copies of the first min(NT, le - lb) particles of a layer, one field per lane of warp 0
// (NF <= 32 copies issued in parallel instead of a serial loop on one thread)
template <int D, typename R>
__device__ __forceinline__ void sw_prefetch(const R* __restrict__ P, const R* __restrict__ cache, int64_t cap, int lb,
                                            int le, R* pf, uint64_t* bar, int lane)
{
    using In = SWIn<D, R>;
    static_assert(In::NF <= 32, "one field per lane");
    const int lb0 = lb & ~(In::UE - 1);                       // 16-B aligned start
    const int cnt = min(le, lb + HvpT<D>::NT) - lb0;
    const uint32_t bytes = (uint32_t)((cnt + In::UE - 1) & ~(In::UE - 1)) * sizeof(R);
    fence_async_smem();
    if (lane == 0) mbar_expect_tx(bar, bytes * In::NF);
    __syncwarp();
    if (lane < In::NF) {
        const R* src = (lane < D) ? P + (int64_t)(PL<D>::X + lane) * cap + lb0 : cache + (int64_t)(lane - D) * cap + lb0;
        bulk_g2s(pf + In::off(lane), src, bytes, bar);
    }
}

// Two 2-D TMA tensor copies per layer instead of one bulk copy per field: the streamed inputs are the
// field-major SoA arrays seen as 2-D tensors [fields][particles] (x: 3 fields of the particle SoA,
// the Newton cache: 17 fields), and one box of {PFS particles, fields} lands exactly in the pf
// layout (field f at pf + f * PFS).  When the host cannot encode the tensor maps (use_tmap = 0) the
// per-field bulk copies of sw_prefetch are used instead.
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// boxes of {PFS particles, fields} at the 16-B aligned particle lb0 into the SWIn layout (the tail
// beyond the particle count reads zeros)
template <int D, typename R>
__device__ __forceinline__ void sw_prefetch_tmap(const CUtensorMap* mx, const CUtensorMap* mc, int lb, R* pf,
                                                 uint64_t* bar, int lane)
{
    using In = SWIn<D, R>;
    if (lane == 0) {
        const int lb0 = lb & ~(In::UE - 1);
        fence_async_smem();
        mbar_expect_tx(bar, (uint32_t)(In::PFS * In::NF * sizeof(R)));
        tma_2d(pf, mx, lb0, 0, bar);
        tma_2d(pf + In::XB, mc, lb0, 0, bar);
    }
}

// 3 CTAs per SM in fp64 (shared memory ~71 KB); the fp32 variant has half the shared memory (records,
// streamed inputs, node tile and staging in fp32): 4
template <int D, typename R>
__global__ void __launch_bounds__(HvpT<D>::NT, sizeof(R) == 8 ? 3 : 4)
k_hvp_sw(const R* __restrict__ P, const R* __restrict__ cache, int64_t cap, const int* __restrict__ cell_start,
         BoxDev b, const double* __restrict__ din, double* __restrict__ yout, const __grid_constant__ CUtensorMap tmx,
         const __grid_constant__ CUtensorMap tmc, int use_tmap, double* __restrict__ tbuf,
         double* __restrict__ pkp, const __grid_constant__ HaloDev halo)
{
    // pkp (optional): per-CTA partials of d^T K d = sum over tiles of d . (the tile's partial y), the
    // curvature the PCG step length needs, accumulated by the plane flushes (FlushItem)
    using T = Tile<D>;
    using C = CL<D>;
    using In = HvpIn<D, R>;
    using S = SW<D>;
    using SR = SWRec<D, R>;
    constexpr int RS = SR::RS;
    constexpr int NTH = HvpT<D>::NT;
    constexpr bool SPLIT9 = HvpT<D>::SPLIT9;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    R* sv = reinterpret_cast<R*>(smem_raw + 16);
    R* stg = sv + S::NNP * SVS<D, R>::S;
    // streamed-input block, 128-B aligned for the tensor copies
    R* pf;
    {
        const uint32_t base = smem_u32(smem_raw);
        const uint32_t off = 16 + (uint32_t)((S::NNP * SVS<D, R>::S + S::STG) * sizeof(R));
        pf = reinterpret_cast<R*>(smem_raw + (((base + off + 127u) & ~127u) - base));
    }
    const bool tmap = use_tmap != 0;
    R* rec = pf + SWIn<D, R>::TOT;
    const int tile = blockIdx.x;
    const int64_t kt = (int64_t)tile * T::NC;
    __shared__ int scs[T::NC + 1];  // the tile's cell ranges
    __shared__ double wdot[HVP_NW<D>];
    int t[3];
    tile_coords<D>(b, tile, t);
    // the node tile of d (fp64: asynchronous, in flight while the cell ranges load) and the staging
    // slots (zeroed once: slots of cells outside the tile are never written)
    constexpr bool ASYNC = sizeof(R) == 8;
    // warp 0 starts the first non-empty layer's input copies straight from the layer boundaries in
    // global memory, before the cell ranges reach shared memory
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int v = lane <= T::NL ? cell_start[kt + lane * T::LC] : 0;
        const int vn = __shfl_down_sync(0xffffffffu, v, 1);
        const unsigned ne = __ballot_sync(0xffffffffu, lane < T::NL && vn > v);
        if (lane == 0) mbar_init(bar, 1);
        __syncwarp();
        if (ne) {
            const int f = __ffs(ne) - 1;
            const int lb0 = __shfl_sync(0xffffffffu, v, f), le0 = __shfl_sync(0xffffffffu, v, f + 1);
            if (tmap)
                sw_prefetch_tmap<D, R>(&tmx, &tmc, lb0, pf, bar, lane);
            else
                sw_prefetch<D, R>(P, cache, cap, lb0, le0, pf, bar, lane);
        }
    }
    if constexpr (ASYNC) sw_stage_tile<D, R, NTH, false>(b, t, din, sv);
    for (int i = threadIdx.x; i <= T::NC; i += NTH) scs[i] = cell_start[kt + i];
    for (int k = threadIdx.x; k < S::STG; k += NTH) stg[k] = R(0);
    __syncthreads();
    if (scs[0] == scs[T::NC]) {
        if constexpr (ASYNC) asm volatile("cp.async.wait_all;" ::: "memory");
        if (pkp && threadIdx.x == 0) pkp[tile] = 0.0;
        halo_signal(halo);
        return;
    }
    const bool fused = halo.yL || halo.yR;
    double dkd = 0.0;  // this thread's flushed nodes' d . y_tile
    double* const tbl = tbuf ? tbuf + (int64_t)tile * T::NN * D : nullptr;
    const HaloDev* const hl = fused ? &halo : nullptr;
    const FlushItem<D, R> fli(b, t, hl);
    // non-empty layers as a bit mask (one shared-memory pass instead of re-reading the cell ranges)
    unsigned nem = 0;
#pragma unroll
    for (int l = 0; l < T::NL; ++l)
        if (scs[l * T::LC] != scs[(l + 1) * T::LC]) nem |= 1u << l;
    auto layer_empty = [&](int l) { return ((nem >> l) & 1u) == 0u; };
    if constexpr (ASYNC)
        asm volatile("cp.async.wait_all;" ::: "memory");
    else
        sw_stage_tile<D, R, NTH>(b, t, din, sv);
    __syncthreads();
    const int it = threadIdx.x;
    int icell, icomp, ii;
    item_of<D>(it, icell, icomp, ii);
    uint32_t parity = 0;
    R acc[S::NACC], acc9[S::NACC];  // acc9: this lane's share of its cell's ninth item (SPLIT9)
#pragma unroll
    for (int k = 0; k < S::NACC; ++k) acc[k] = acc9[k] = R(0);
    for (int layer = 0; layer < T::NL + 2; ++layer) {
        if (layer < T::NL && !layer_empty(layer)) {
            const int lb = scs[layer * T::LC], le = scs[(layer + 1) * T::LC];
            int next = layer + 1;
            {
                const unsigned later = nem >> (layer + 1);
                next = later ? layer + __ffs(later) : T::NL;
            }
            const int pf_base = lb & ~(In::UE - 1);
            const int ks = scs[layer * T::LC + icell];
            const int ke = scs[layer * T::LC + icell + 1];
            for (int sb = lb; sb < le; sb += NTH) {
                const int se = min(sb + NTH, le);
                const int q = threadIdx.x, p = sb + q;
                const bool from_pf = sb == lb;
                if (sb != lb) __syncthreads();  // previous chunk's records consumed
                if (from_pf) mbar_wait(bar, parity);
                // phase 1, instantiated for the two sources of the streamed fields (the shared-memory copy
                // of the first chunk; global memory for the rare further chunks of a layer holding more
                // than NT particles) so that the common path carries no predicated global loads
                auto phase1 = [&](auto fromc) {
                    constexpr int FROM = decltype(fromc)::value;  // 1 smem, 0 global, 2 either (runtime)
                    // streamed field f of particle p.  The Newton cache is read only after the gather
                    // (register pressure: the weights and gather temporaries are dead by then).
                    const R* s = pf + (p - pf_base);
                    auto in = [&](int f) -> R {
                        if constexpr (FROM == 1)
                            return s[SWIn<D, R>::off(f)];
                        else if constexpr (FROM == 0)
                            return f < D ? P[(int64_t)(PL<D>::X + f) * cap + p] : cache[(int64_t)(f - D) * cap + p];
                        else
                            return from_pf ? s[SWIn<D, R>::off(f)]
                                           : (f < D ? P[(int64_t)(PL<D>::X + f) * cap + p]
                                                    : cache[(int64_t)(f - D) * cap + p]);
                    };
                    R x[3];
#pragma unroll
                    for (int a = 0; a < D; ++a) x[a] = in(a);
                    R w[3][3], dw[3][3];
                    int lc[3] = {0, 0, 0};
                    weights_at<D, R>(x, b, t, lc, w, dw);
                    const RecPtr<R> r(rec + (D == 3 ? lc[0] * T::T1 + lc[1] : lc[0]) * SR::SK, q, RS);
                    store_weights<D, R>(r, w, dw);
                    R gd[D * D];
                    sw_gather<D, R>(sv, lc, w, dw, gd);
                    R Sv[Sym<D>::N], A[D * D];
#pragma unroll
                    for (int k = 0; k < Sym<D>::N; ++k) Sv[k] = in(D + C::S + k);
#pragma unroll
                    for (int k = 0; k < D * D; ++k) A[k] = in(D + C::A + k);
                    const R cc = in(D + C::C), ll = in(D + C::L);
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
                    for (int a = 0; a < D; ++a) {
                        R Ga[D];
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) {
                            R s1 = R(0), s2 = R(0);
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                s1 = fma(gd[a * D + k], Sv[sym_idx<D>(k, bb)], s1);
                                s2 = fma(M2[a * D + k], A[k * D + bb], s2);
                            }
                            Ga[bb] = fma(cc, s2, fma(ltr, A[a * D + bb], s1));
                        }

                        if constexpr (SR::GP == 4) {
                            using V2 = typename Vec2<R>::type;
                            V2 g01;
                            g01.x = Ga[0];
                            g01.y = Ga[1];
                            *reinterpret_cast<V2*>(r.at(Rec<D>::G + 4 * a)) = g01;
                            *r.at(Rec<D>::G + 4 * a + 2) = Ga[D - 1];
                        } else {
#pragma unroll
                            for (int bb = 0; bb < D; ++bb) *r.at(Rec<D>::G + a * D + bb) = Ga[bb];
                        }
                    }
                };
                if (p < se) {
                    if (from_pf)
                        phase1(ICst<1>{});
                    else
                        phase1(ICst<0>{});
                }
                __syncthreads();  // records ready; the streamed buffer is free
                if (sb == lb) {
                    if (from_pf) parity ^= 1u;
                    if (threadIdx.x < 32 && next < T::NL) {
                        if (tmap)
                            sw_prefetch_tmap<D, R>(&tmx, &tmc, scs[next * T::LC], pf, bar, threadIdx.x);
                        else
                            sw_prefetch<D, R>(P, cache, cap, scs[next * T::LC], scs[(next + 1) * T::LC], pf, bar,
                                              threadIdx.x);
                    }
                }
                if (it < T::ITEMS) {
                    const int p0 = max(ks, sb), p1 = min(ke, se);
                    const int len = p1 - p0;
                    R* const cbase = rec + icell * SR::SK + (p0 - sb) * RS;  // this cell's first record
#ifndef OSMPM_P2_UNROLL
#define OSMPM_P2_UNROLL 4
#endif
                    // with the skewed records (constant offsets): 4 (C5 fp64 1.249 ms vs 1.256 at 8, 1.262 at
                    // 2, 1.269 at 1; fp32 unchanged); with the earlier rotated order 8 was best
                    constexpr int kUnroll = OSMPM_P2_UNROLL;
#pragma unroll kUnroll
                    for (int k = 0; k < len; ++k) {
                        const RecPtr<R> r(cbase, k, RS);
                        ItemW<D, R> W;
                        R s[D];
                        W.load(r, ii);
#pragma unroll
                        for (int bb = 0; bb < D; ++bb) s[bb] = *r.at(Rec<D>::G + icomp * SR::GP + bb);
                        item_linear<D, R>(s, W, acc);
                    }
                    if constexpr (SPLIT9) {
                        // the cell's ninth item: particles pr, pr + 8, ... of the cell in this chunk
#pragma unroll 1
                        for (int k = it & 7; k < len; k += 8) {
                            const RecPtr<R> r(cbase, k, RS);
                            ItemW<D, R> W;
                            R s[D];
                            W.load(r, 2);
#pragma unroll
                            for (int bb = 0; bb < D; ++bb) s[bb] = *r.at(Rec<D>::G + 2 * SR::GP + bb);
                            item_linear<D, R>(s, W, acc9);
                        }
                    }
                }
            }
        }
        // node plane `layer` is complete: stage it, then sum the slots and RED
        if (it < T::ITEMS) sw_emit<D, R>(icell, icomp, ii, acc, stg);
        if constexpr (SPLIT9) {
            // the ninth item's plane: the eight lanes' shares summed over the quarter warp (fixed
            // butterfly order), staged by its first lane; every lane shifts its own window
            R e9[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                e9[j] = acc9[j * 3 + 0];
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) e9[j] += __shfl_xor_sync(0xffffffffu, e9[j], o);
            }
            if ((it & 7) == 0) {
#pragma unroll
                for (int j = 0; j < 3; ++j) acc9[j * 3 + 0] = e9[j];
                sw_emit<D, R>(icell, 2, 2, acc9, stg);
            } else {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    acc9[j * 3 + 0] = acc9[j * 3 + 1];
                    acc9[j * 3 + 1] = acc9[j * 3 + 2];
                    acc9[j * 3 + 2] = R(0);
                }
            }
        }
        __syncthreads();
        if (pkp)
            fli.template flush<true>(layer, stg, yout, tbl, sv, din, dkd, hl);
        else
            fli.template flush<false>(layer, stg, yout, tbl, sv, din, dkd, hl);
        // the next emit must not overwrite slots still being summed: a non-empty next layer has its
        // records barrier in between; otherwise synchronise here
        if (pkp && layer == T::NL + 1) {
            // warp partials of the curvature into shared memory before the closing barrier
            const unsigned mask = __activemask();
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dkd += __shfl_xor_sync(mask, dkd, o);
            if ((threadIdx.x & 31) == 0) wdot[threadIdx.x >> 5] = dkd;
        }
        if (layer + 1 >= T::NL || layer_empty(layer + 1)) __syncthreads();
    }
    // the last layer's closing barrier above has made every warp's partial visible: one per CTA, in a
    // fixed order
    if (pkp && threadIdx.x == 0) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < HVP_NW<D>; ++w) v += wdot[w];
        pkp[tile] = v;
    }
    halo_signal(halo);
}

}  // namespace osmpm
