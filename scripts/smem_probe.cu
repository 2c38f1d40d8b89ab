// Microbenchmark of shared-memory load cost (wavefronts per warp instruction) for the lane -> address
// patterns of the HVP's phases on sm_100a.  Each kernel launch uses one pattern; run under
// ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_probe scripts/smem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

// pattern: address (in 16-B units) read by lane l
__device__ __forceinline__ int addr16(int pat, int lane, int it)
{
    switch (pat) {
    case 0: return 0;                                   // all lanes one address
    case 1: return (lane / 8) * 15;                     // 8-lane groups, 4 addresses (odd stride)
    case 2: return (lane / 9) * 15;                     // 9-lane groups (HVP phase 2: 9 items / cell)
    case 3: return (lane / 16) * 15;                    // half-warps, 2 addresses
    case 4: return lane;                                // 32 distinct consecutive
    case 5: return (lane / 8) * 15 + (lane % 3);        // 8-lane groups, 3 chunks of one record each
    case 6: return (lane / 9) * 15 + (lane % 3);        // 9-lane groups, 3 chunks (wx pair by item i)
    case 7: return lane * 15;                           // 32 distinct records (phase-1 record store)
    }
    return 0;
}

template <int WIDTH>  // bytes per lane: 8 or 16
__global__ void probe(int pat, int iters, double* out)
{
    __shared__ __align__(16) double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int a = addr16(pat, lane, 0) * 2;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int off = (it & 7) * 512;  // move around to defeat hoisting
        if (WIDTH == 16) {
            const double2 v = *reinterpret_cast<const double2*>(&buf[(a + off) & 4095]);
            acc += v.x + v.y;
        } else {
            acc += buf[(a + off) & 4095];
        }
    }
    if (acc == -1.0) out[0] = acc;
}

int main()
{
    double* out;
    cudaMalloc(&out, 8);
    for (int pat = 0; pat < 8; ++pat) {
        probe<16><<<148, 128>>>(pat, 4096, out);
        probe<8><<<148, 128>>>(pat, 4096, out);
    }
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
