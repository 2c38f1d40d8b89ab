// radix_sort.cuh -- hand-written stable LSD radix sort of (uint32 key, int32 value) pairs (a1).
//
// The particles are binned every step by the tile-major key of their base cell (north_star: "particles
// sorted into grid blocks each step with a block-level radix sort"; needed by the tiled P2G / HVP /
// gradient kernels).  Keys need ceil(log2(#cells)) bits (C5: 22), sorted 8 bits per
// pass, least-significant digit first; every pass is stable, so the whole sort is (equal keys keep
// their input order: the result is deterministic).
//
// One pass = three kernels over tiles of TILE = 256 threads x 16 keys:
//   upsweep    per-tile digit histogram (shared-memory counters) -> hist[digit][tile]
//   scan       exclusive scan of hist in digit-major order (one CTA per digit row, then the 256 row
//              totals) -> the first output slot of every (digit, tile)
//   downsweep  per-tile stable ranks: each warp walks its 16 keys in input order, peers with the same
//              digit found with __match_any_sync, per-warp digit counters in shared memory, then an
//              exclusive scan of the counters across the 8 warps; the pairs are staged in shared memory
//              in their sorted order within the tile and stored from there, so that the consecutive
//              slots slot(digit, tile) + rank of one digit are written by consecutive threads.
// Keys of a tile are read warp-striped (item i of lane l of warp w = tile base + 512 w + 32 i + l),
// which is also the ranking order, so stability needs no extra bookkeeping.
#pragma once
#include <cstdint>

#include "device.cuh"

namespace osmpm {

struct RS {
    static constexpr int BITS = 8, RADIX = 1 << BITS, THREADS = 256, WARPS = THREADS / 32, IPT = 16;
    static constexpr int TILE = THREADS * IPT;
    static_assert(THREADS == RADIX, "the downsweep scans one digit per thread");
};

__global__ void __launch_bounds__(RS::THREADS) k_rs_upsweep(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                            uint32_t mask, uint32_t* __restrict__ hist, int nblk)
{
    __shared__ uint32_t cnt[RS::RADIX];
    for (int d = threadIdx.x; d < RS::RADIX; d += RS::THREADS) cnt[d] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS::TILE;
#pragma unroll 4
    for (int i = 0; i < RS::IPT; ++i) {
        const int64_t k = base + (int64_t)i * RS::THREADS + threadIdx.x;
        if (k < n) atomicAdd(&cnt[(keys[k] >> shift) & mask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RS::RADIX; d += RS::THREADS) hist[(int64_t)d * nblk + blockIdx.x] = cnt[d];
}

// exclusive scan of one digit's row hist[d][0..nblk) in place; row total -> tot[d]
__global__ void __launch_bounds__(1024) k_rs_scan_rows(uint32_t* __restrict__ hist, int nblk, uint32_t* __restrict__ tot)
{
    __shared__ uint32_t ws[32];
    uint32_t* row = hist + (int64_t)blockIdx.x * nblk;
    uint32_t carry = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c0 = 0; c0 < nblk; c0 += 1024) {
        const int i = c0 + threadIdx.x;
        const uint32_t v = i < nblk ? row[i] : 0u;
        uint32_t s = v;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += t;
        }
        if (lane == 31) ws[w] = s;
        __syncthreads();
        if (w == 0) {
            uint32_t x = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += t;
            }
            ws[lane] = x;  // inclusive prefix of the warp totals
        }
        __syncthreads();
        const uint32_t excl = carry + (w ? ws[w - 1] : 0u) + s - v;
        if (i < nblk) row[i] = excl;
        carry += ws[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// exclusive scan of the RADIX digit totals (one CTA of RADIX threads)
__global__ void __launch_bounds__(RS::RADIX) k_rs_scan_totals(uint32_t* __restrict__ tot)
{
    __shared__ uint32_t s[RS::RADIX];
    s[threadIdx.x] = tot[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int d = 0; d < RS::RADIX; ++d) {
            const uint32_t t = s[d];
            s[d] = run;
            run += t;
        }
    }
    __syncthreads();
    tot[threadIdx.x] = s[threadIdx.x];
}

__global__ void __launch_bounds__(RS::THREADS) k_rs_downsweep(const uint32_t* __restrict__ kin, const int* __restrict__ vin,
                                                              uint32_t* __restrict__ kout, int* __restrict__ vout,
                                                              int64_t n, int shift, uint32_t mask,
                                                              const uint32_t* __restrict__ hist,
                                                              const uint32_t* __restrict__ tot, int nblk)
{
    __shared__ uint32_t cnt[RS::WARPS][RS::RADIX];
    __shared__ uint32_t doff[RS::RADIX];           // the tile's exclusive digit offsets
    __shared__ uint32_t sk[RS::TILE];              // the tile's pairs in sorted order, for coalesced stores
    __shared__ int svv[RS::TILE];
    for (int e = threadIdx.x; e < RS::WARPS * RS::RADIX; e += RS::THREADS) (&cnt[0][0])[e] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t tbase = (int64_t)blockIdx.x * RS::TILE;
    const int64_t base = tbase + (int64_t)w * (32 * RS::IPT) + lane;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t key[RS::IPT], rank[RS::IPT];
    int val[RS::IPT];
#pragma unroll
    for (int i = 0; i < RS::IPT; ++i) {
        const int64_t k = base + 32 * i;
        const bool ok = k < n;
        key[i] = ok ? kin[k] : 0xffffffffu;  // the tail ranks last (digit RADIX - 1) and is not stored
        val[i] = ok ? vin[k] : 0;
    }
#pragma unroll
    for (int i = 0; i < RS::IPT; ++i) {
        const uint32_t d = (key[i] >> shift) & mask;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = cnt[w][d];
        rank[i] = before + __popc(peers & lt);
        __syncwarp();
        if ((peers & lt) == 0) cnt[w][d] = before + __popc(peers);  // the lowest lane of the group
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive scan of the per-warp counts across the warps; digit totals of the tile
    uint32_t dtot = 0;
    const int d0 = threadIdx.x;  // RS::THREADS == RS::RADIX: one digit per thread
    {
        uint32_t run = 0;
#pragma unroll
        for (int q = 0; q < RS::WARPS; ++q) {
            const uint32_t t = cnt[q][d0];
            cnt[q][d0] = run;
            run += t;
        }
        dtot = run;
    }
    // exclusive scan of the digit totals over the block (warp scans + warp totals)
    {
        __shared__ uint32_t wsum[RS::WARPS];
        uint32_t x = dtot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        uint32_t pre = 0;
        for (int q = 0; q < w; ++q) pre += wsum[q];
        doff[d0] = pre + x - dtot;
    }
    __syncthreads();
    // stage the pairs at their sorted position inside the tile
#pragma unroll
    for (int i = 0; i < RS::IPT; ++i) {
        if (base + 32 * i >= n) continue;
        const uint32_t d = (key[i] >> shift) & mask;
        const uint32_t pos = doff[d] + cnt[w][d] + rank[i];
        sk[pos] = key[i];
        svv[pos] = val[i];
    }
    __syncthreads();
    // consecutive tile positions of one digit go to consecutive global slots: coalesced stores
    const int64_t nvalid = min((int64_t)RS::TILE, n - tbase);
    for (int pos = threadIdx.x; pos < nvalid; pos += RS::THREADS) {
        const uint32_t kk = sk[pos];
        const uint32_t d = (kk >> shift) & mask;
        const int64_t g = (int64_t)tot[d] + hist[(int64_t)d * nblk + blockIdx.x] + (pos - doff[d]);
        kout[g] = kk;
        vout[g] = svv[pos];
    }
}

// Sorts n (key, value) pairs on the low `nbits` bits of the keys.  (k0, v0) hold the input; (k1, v1) are
// scratch of the same size; the result lands in (k1, v1) if the function returns true, else in (k0, v0).
// hist: >= RADIX * ceil(n / TILE) + RADIX words.  launches: incremented per kernel.
inline bool radix_sort_pairs(uint32_t* k0, int* v0, uint32_t* k1, int* v1, int64_t n, int nbits, uint32_t* hist,
                             cudaStream_t st, int64_t& launches)
{
    if (n <= 0 || nbits <= 0) return false;
    const int nblk = (int)((n + RS::TILE - 1) / RS::TILE);
    uint32_t* tot = hist + (int64_t)RS::RADIX * nblk;
    bool second = false;
    for (int shift = 0; shift < nbits; shift += RS::BITS) {
        const int b = nbits - shift < RS::BITS ? nbits - shift : RS::BITS;
        const uint32_t mask = (1u << b) - 1u;
        uint32_t* ki = second ? k1 : k0;
        int* vi = second ? v1 : v0;
        uint32_t* ko = second ? k0 : k1;
        int* vo = second ? v0 : v1;
        k_rs_upsweep<<<nblk, RS::THREADS, 0, st>>>(ki, n, shift, mask, hist, nblk);
        k_rs_scan_rows<<<RS::RADIX, 1024, 0, st>>>(hist, nblk, tot);
        k_rs_scan_totals<<<1, RS::RADIX, 0, st>>>(tot);
        k_rs_downsweep<<<nblk, RS::THREADS, 0, st>>>(ki, vi, ko, vo, n, shift, mask, hist, tot, nblk);
        launches += 4;
        second = !second;
    }
    return second;
}
inline size_t radix_hist_words(int64_t n) { return (size_t)RS::RADIX * ((n + RS::TILE - 1) / RS::TILE) + RS::RADIX; }

}  // namespace osmpm
