// Occupancy probe: does a kernel that allocates TMEM get more than one CTA
// per SM from the occupancy calculator / the hardware?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/occ_probe tools/occ_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 2) plain_kernel(int* out) {
    if (threadIdx.x == 0) out[blockIdx.x] = 1;
}

__global__ void __launch_bounds__(256, 2) tmem_kernel(int* out, unsigned long long* t) {
    __shared__ uint32_t taddr;
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const long long t0 = clock64();
    while (clock64() - t0 < 20000000) { }
    if (threadIdx.x == 0) { out[blockIdx.x] = smid; t[blockIdx.x] = clock64(); }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" :: "r"(taddr));
}

int main() {
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, plain_kernel, 256, 40000);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tmem_kernel, 256, 40000);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, tmem_kernel);
    printf("occupancy plain %d, tmem %d (regs %d)\n", a, b, fa.numRegs);
    // launch 2 CTAs per SM of the TMEM kernel and see whether they co-run
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* out; unsigned long long* t;
    cudaMalloc(&out, 4 * 2 * sms); cudaMalloc(&t, 8 * 2 * sms);
    cudaFuncSetAttribute(tmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int g = 1; g <= 2; ++g) {
        cudaEventRecord(e0);
        tmem_kernel<<<g * sms, 256, 40000>>>(out, t);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d x %d CTAs: %.2f ms (%s)\n", g, sms, ms, cudaGetErrorString(err));
    }
    return 0;
}
