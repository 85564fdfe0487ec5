// Dev probe: shared-memory limits and real CTA co-residency on this GPU (which smem sizes let
// two 256-thread CTAs share an SM). nvcc -gencode arch=compute_100a,code=sm_100a occ_probe.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) probe(unsigned* smid, unsigned long long* t) {
    extern __shared__ unsigned char s[];
    if (threadIdx.x == 0) {
        unsigned id;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
        unsigned long long a, b;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
        do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b)); } while (b - a < 200000);
        s[0] = 1;
        smid[blockIdx.x] = id;
        t[2 * blockIdx.x] = a;
        t[2 * blockIdx.x + 1] = b;
    }
}

__global__ void __launch_bounds__(256, 1) probe_tmem(unsigned* smid, unsigned long long* t) {
    extern __shared__ unsigned char s[];
    __shared__ unsigned slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a, b;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
        do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b)); } while (b - a < 200000);
        s[0] = 1;
        t[2 * blockIdx.x] = a;
        t[2 * blockIdx.x + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(64));
}

int main() {
    int v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0); printf("smem/SM %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); printf("smem/block optin %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, 0); printf("reserved/block %d\n", v);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(probe, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    unsigned* smid; unsigned long long* t;
    cudaMalloc(&smid, 4 * 2 * sms); cudaMalloc(&t, 16 * 2 * sms);
    for (int kb : {64, 80, 88, 90, 92, 94, 96, 100, 104, 108, 110, 112}) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe, 256, kb * 1024);
        probe<<<2 * sms, 256, kb * 1024>>>(smid, t);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<unsigned> h(2 * sms); std::vector<unsigned long long> ht(4 * sms);
        cudaMemcpy(h.data(), smid, 8 * sms, cudaMemcpyDeviceToHost);
        cudaMemcpy(ht.data(), t, 32 * sms, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, t1 = 0;
        for (int i = 0; i < 2 * sms; ++i) { t0 = ht[2*i] < t0 ? ht[2*i] : t0; t1 = ht[2*i+1] > t1 ? ht[2*i+1] : t1; }
        printf("dyn smem %3d KB: occupancy API %d, 2x%d CTAs took %.0f us (%s)\n", kb, occ, sms, (t1 - t0) / 1e3,
               cudaGetErrorString(e));
    }
    cudaFuncSetAttribute(probe_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int kb : {64, 94}) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe_tmem, 256, kb * 1024);
        probe_tmem<<<2 * sms, 256, kb * 1024>>>(smid, t);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<unsigned long long> ht(4 * sms);
        cudaMemcpy(ht.data(), t, 32 * sms, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull, t1 = 0;
        for (int i = 0; i < 2 * sms; ++i) { t0 = ht[2*i] < t0 ? ht[2*i] : t0; t1 = ht[2*i+1] > t1 ? ht[2*i+1] : t1; }
        printf("tmem kernel, dyn smem %3d KB: occupancy API %d, took %.0f us (%s)\n", kb, occ, (t1 - t0) / 1e3, cudaGetErrorString(e));
    }
    return 0;
}
