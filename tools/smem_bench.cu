// smem_bench.cu -- shared-memory / texture data-path throughput on B200 for the
// access shapes of the staged-operator SpMV:
//   1. LDS.128, 32 distinct conflict-free addresses (the gathered x)
//   2. LDS.128, every lane the same address
//   3. LDS.128, 8 distinct addresses per warp (a small value dictionary)
//   4. LDS.64 / LDS.32, distinct addresses
//   5. tex1Dfetch<int4> from a 1 KB table, 8 distinct addresses per warp
//   6. 1 + 5 interleaved: do the texture fetches ride on top of the LDS traffic?
// Prints cycles per warp instruction per SM at 16 resident warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_bench tools/smem_bench.cu && ./smem_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int UNR = 8;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(cudaTextureObject_t tex, long long* out, int4* sink) {
    __shared__ int4 buf[2048];  // 32 KB
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 2048; i += blockDim.x) buf[i] = make_int4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    int4 acc = make_int4(0, 0, 0, 0);
    int idx;
    if (MODE == 1 || MODE == 4 || MODE == 6 || MODE == 7 || MODE == 8 || MODE >= 9) idx = lane;
    else if (MODE == 2) idx = 5;
    else idx = (lane * 7) & 7;  // 8 distinct
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        // the addresses depend on the running xor once per outer iteration only,
        // so the UNR loads of an iteration are independent (throughput, not latency)
        const int o1 = acc.x & 1024, o2 = acc.y & 32;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (MODE == 1 || MODE == 2 || MODE == 3) {
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            } else if (MODE == 7) {
                const int2 v = reinterpret_cast<const int2*>(buf)[(idx + 32 * u + o1) & 4095];
                acc.x ^= v.x; acc.y ^= v.y;
            } else if (MODE == 8) {
                const int v = reinterpret_cast<const int*>(buf)[(idx + 32 * u + o1) & 8191];
                acc.x ^= v;
            } else if (MODE == 5) {
                const int4 v = tex1Dfetch<int4>(tex, (idx + 8 * u + o2) & 63);
                acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
            } else if (MODE == 6) {
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int4 w = tex1Dfetch<int4>(tex, (((lane * 7) & 7) + 8 * u + o2) & 63);
                acc.x ^= v.x ^ w.w; acc.y ^= v.y ^ w.z; acc.z ^= v.z ^ w.y; acc.w ^= v.w ^ w.x;
            } else if (MODE == 9) {
                // two conflict-free LDS.128 with distinct addresses
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int4 w = buf[(lane + 32 * u + 1024 + o2) & 2047];
                acc.x ^= v.x ^ w.w; acc.y ^= v.y ^ w.z; acc.z ^= v.z ^ w.y; acc.w ^= v.w ^ w.x;
            } else if (MODE == 10) {
                // gather + the value as two LDS.64 halves from an 8-entry table
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int2* const h = reinterpret_cast<const int2*>(buf);
                const int2 a = h[(((lane * 7) & 7) + 8 * u + o2) & 63];
                const int2 b = h[((((lane * 7) & 7) + 8 * u + o2) & 63) + 2048];
                acc.x ^= v.x ^ a.x; acc.y ^= v.y ^ a.y; acc.z ^= v.z ^ b.x; acc.w ^= v.w ^ b.y;
            } else if (MODE == 11) {
                // gather + one-address LDS.128 (a warp-uniform value)
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int4 w = buf[(5 + 8 * u + o2) & 63];
                acc.x ^= v.x ^ w.w; acc.y ^= v.y ^ w.z; acc.z ^= v.z ^ w.y; acc.w ^= v.w ^ w.x;
            } else if (MODE == 4) {
                // two LDS.128 per step (x + value, both through shared memory)
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int4 w = buf[(((lane * 7) & 7) + 8 * u + o2) & 63];
                acc.x ^= v.x ^ w.w; acc.y ^= v.y ^ w.z; acc.z ^= v.z ^ w.y; acc.w ^= v.w ^ w.x;
            }
        }
    }
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    if (acc.x == 0x7fffffff) sink[0] = acc;
}

template <int MODE>
static void run(const char* name, cudaTextureObject_t tex, long long* d_out, int4* d_sink, int sms) {
    k<MODE><<<sms, 512>>>(tex, d_out, d_sink);
    cudaDeviceSynchronize();
    k<MODE><<<sms, 512>>>(tex, d_out, d_sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    long long h[256];
    cudaMemcpy(h, d_out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i];
    avg /= sms;
    const double per_warp_inst = avg / ((double)ITERS * UNR * 16);  // 16 warps per SM
    printf("%-58s %8.2f SM-cycles per warp step (16 warps/SM)\n", name, per_warp_inst);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int4 host[64];
    for (int i = 0; i < 64; ++i) host[i] = make_int4(i, 2 * i, 3 * i, 4 * i);
    int4* d_tab = nullptr;
    cudaMalloc(&d_tab, sizeof(host));
    cudaMemcpy(d_tab, host, sizeof(host), cudaMemcpyHostToDevice);
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = d_tab;
    rd.res.linear.desc = cudaCreateChannelDesc<int4>();
    rd.res.linear.sizeInBytes = sizeof(host);
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    long long* d_out = nullptr;
    int4* d_sink = nullptr;
    cudaMalloc(&d_out, sizeof(long long) * 256);
    cudaMalloc(&d_sink, sizeof(int4));
    run<1>("LDS.128, 32 distinct addresses", tex, d_out, d_sink, sms);
    run<2>("LDS.128, one address for the warp", tex, d_out, d_sink, sms);
    run<3>("LDS.128, 8 distinct addresses", tex, d_out, d_sink, sms);
    run<7>("LDS.64, 32 distinct addresses", tex, d_out, d_sink, sms);
    run<8>("LDS.32, 32 distinct addresses", tex, d_out, d_sink, sms);
    run<4>("LDS.128 distinct + LDS.128 8-address (x + value)", tex, d_out, d_sink, sms);
    run<9>("LDS.128 distinct + LDS.128 distinct", tex, d_out, d_sink, sms);
    run<10>("LDS.128 distinct + 2 x LDS.64 8-address (split value)", tex, d_out, d_sink, sms);
    run<11>("LDS.128 distinct + LDS.128 one address", tex, d_out, d_sink, sms);
    run<5>("tex1Dfetch<int4>, 8 distinct addresses", tex, d_out, d_sink, sms);
    run<6>("LDS.128 distinct + tex1Dfetch<int4> (x + value via TEX)", tex, d_out, d_sink, sms);
    return 0;
}
