// Microbenchmark: tcgen05.ld / tcgen05.st throughput between TMEM and
// registers (is TMEM usable as extra per-SM storage for Nordsieck rows?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NT>
__global__ void __launch_bounds__(NT, 1) tmem_kernel(int iters, int mode, unsigned long long* cyc,
                                                    unsigned* sink) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = taddr_s;
    // warp w: lane quarter w % 4, column block (w / 4) * 128
    const uint32_t ta = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
    unsigned acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t a = ta + (uint32_t)((it & (mode == 3 ? 1 : 7)) * 16);
        if (mode == 0) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                           "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                           "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(a));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int i = 0; i < 16; ++i) acc += r[i];
        } else if (mode == 2) {
            // read-modify-write of 16 words (4 complex doubles): the Nordsieck
            // row update pattern (ld, wait, add, st)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                           "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                           "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(a));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] += 3u;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                         :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                            "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]),
                            "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
        } else if (mode == 3) {
            // 4 independent x16 loads, one wait (the batched row read pattern)
            uint32_t q[48];
#pragma unroll
            for (int j = 0; j < 3; ++j)
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                             : "=r"(q[16*j+0]), "=r"(q[16*j+1]), "=r"(q[16*j+2]), "=r"(q[16*j+3]), "=r"(q[16*j+4]), "=r"(q[16*j+5]),
                               "=r"(q[16*j+6]), "=r"(q[16*j+7]), "=r"(q[16*j+8]), "=r"(q[16*j+9]), "=r"(q[16*j+10]), "=r"(q[16*j+11]),
                               "=r"(q[16*j+12]), "=r"(q[16*j+13]), "=r"(q[16*j+14]), "=r"(q[16*j+15])
                             : "r"(a + 16u * j));
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                           "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                           "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(a + 48u));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int i = 0; i < 48; ++i) acc += q[i];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc += r[i];
        } else {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                         :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                            "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]),
                            "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
            asm volatile("tcgen05.wait::st.sync.aligned;\n");
            r[it & 15] += 1;
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    sink[blockIdx.x * NT + threadIdx.x] = acc + r[3];
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(base));
}

template <int NT>
void run(int mode) {
    const int grid = 148, iters = 4096;
    unsigned long long* cyc;
    unsigned* sink;
    cudaMalloc(&cyc, grid * 8);
    cudaMalloc(&sink, grid * NT * 4);
    tmem_kernel<NT><<<grid, NT>>>(16, mode, cyc, sink);
    tmem_kernel<NT><<<grid, NT>>>(iters, mode, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += h[i];
    avg /= grid;
    const double bytes = (double)iters * NT * 16 * 4 * (mode == 3 ? 4 : 1);  // per CTA
    static const char* names[] = {"ld", "st", "rmw", "ld4"};
    printf("%s NT=%d: %s  %.0f cycles, %.1f B/cycle/SM (%.1f cycles per warp-instruction)\n",
           names[mode], NT, cudaGetErrorString(e), avg, bytes / avg,
           avg / iters);
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    for (int m = 0; m < 4; ++m) { run<32>(m); run<128>(m); run<256>(m); run<512>(m); }
    return 0;
}
