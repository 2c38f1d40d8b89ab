// CTA dispatch-order probe (B200): a grid shaped like the C5 HVP (18513 CTAs x 144 threads, 76 KB
// dynamic shared memory -> 3 CTAs/SM) records each CTA's start time, SM and the start of the CTA
// with blockIdx - 1, - 17, - 561 (the fused PCG's lower neighbours).  Prints how often a CTA starts
// before a lower-indexed one and the distribution of start-time differences.
#include <cstdio>
#include <vector>
#include <algorithm>
__global__ void k(unsigned long long* t0, int* sm, int spin_ns)
{
    extern __shared__ char smem[];
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) {
        t0[blockIdx.x] = t;
        int s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        sm[blockIdx.x] = s;
    }
    smem[threadIdx.x] = 0;
    unsigned long long e = t;
    while (e - t < (unsigned long long)spin_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(e));
}
int main()
{
    const int n = 18513, smem = 76 * 1024;
    unsigned long long* d;
    int* s;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&s, n * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) k<<<n, 144, smem>>>(d, s, 30000);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> t(n);
    std::vector<int> sm(n);
    cudaMemcpy(t.data(), d, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(sm.data(), s, n * 4, cudaMemcpyDeviceToHost);
    unsigned long long tmin = *std::min_element(t.begin(), t.end());
    int offs[3] = {1, 17, 561};
    for (int o : offs) {
        int before = 0;
        std::vector<long long> dd;
        for (int i = o; i < n; ++i) {
            long long df = (long long)t[i] - (long long)t[i - o];
            if (df < 0) ++before;
            dd.push_back(df);
        }
        std::sort(dd.begin(), dd.end());
        printf("offset %d: started before the lower CTA %d of %d; dt(ns) p1 %lld p50 %lld p99 %lld min %lld\n", o, before,
               n - o, dd[dd.size() / 100], dd[dd.size() / 2], dd[dd.size() * 99 / 100], dd[0]);
    }
    printf("first 12 CTAs: ");
    for (int i = 0; i < 12; ++i) printf("(%d sm%d +%lluns) ", i, sm[i], t[i] - tmin);
    printf("\nCTAs 444-455: ");
    for (int i = 444; i < 456; ++i) printf("(%d sm%d +%lluns) ", i, sm[i], t[i] - tmin);
    printf("\n");
    return 0;
}
