// Standalone check of the HVP's 2-D tensor-map copy pattern on sm_100a: a [nf][cap] fp64 field array,
// boxes of {nt particles, nf fields} at particle lb into 128-B aligned shared memory, one mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe scripts/tma_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, int nt, int nf, int lb, double* out,
                  int mode)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    double* buf = reinterpret_cast<double*>(sm + 128 + (mode & 1) * 0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(nt * nf * 8)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                s32(buf)),
            "l"(reinterpret_cast<uint64_t>((mode & 2) ? gm : &m)), "r"(lb), "r"(0), "r"(s32(bar))
            : "memory");
    }
    __syncthreads();
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(s32(bar))
        : "memory");
    for (int i = threadIdx.x; i < nt * nf; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv)
{
    // argv: mode (bit 1: tensor map in global memory), lb, nt, dtype (0 f64, 1 u64, 2 f32-pairs)
    const int mode = argc > 1 ? atoi(argv[1]) : 0, lb = argc > 2 ? atoi(argv[2]) : 37;
    const int cap = 4100, nt = argc > 3 ? atoi(argv[3]) : 144, dt = argc > 4 ? atoi(argv[4]) : 0;
    for (int nf : {2, 17}) {
        std::vector<double> h((size_t)nf * cap);
        for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
        double *d, *o;
        cudaMalloc(&d, h.size() * 8);
        cudaMalloc(&o, nt * nf * 8);
        cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)cap, (cuuint64_t)nf}, str[1] = {(cuuint64_t)cap * 8};
        cuuint32_t box[2] = {(cuuint32_t)nt, (cuuint32_t)nf}, es[2] = {1, 1};
        CUresult r = cuTensorMapEncodeTiled(&m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, dims, str, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        CUtensorMap* gm;
        cudaMalloc(&gm, sizeof(CUtensorMap));
        cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
        k<<<1, 128, 128 + nt * nf * 8>>>(m, gm, nt, nf, lb, o, mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> ho(nt * nf);
        cudaMemcpy(ho.data(), o, nt * nf * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int f = 0; f < nf; ++f)
            for (int p = 0; p < nt; ++p) bad += ho[f * nt + p] != (double)(f * cap + lb + p);
        printf("mode=%d lb=%d nt=%d dt=%d nf=%d encode=%d run=%s bad=%d\n", mode, lb, nt, dt, nf, (int)r, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
        cudaFree(d);
        cudaFree(o);
    }
    return 0;
}
