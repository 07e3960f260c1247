// smem_bench.cu -- shared-memory / texture data-path throughput on B200 for the
// access shapes of the staged-operator SpMV:
//   1. LDS.128, 32 distinct conflict-free addresses (the gathered x)
//   2. LDS.128, every lane the same address
//   3. LDS.128, 8 distinct addresses per warp (a small value dictionary)
//   4. LDS.64 / LDS.32, distinct addresses
//   5. tex1Dfetch<int4> from a 1 KB table, 8 distinct addresses per warp
//   6. 1 + 5 interleaved: do the texture fetches ride on top of the LDS traffic?
//   7. LDS.64 values (purely imaginary entries), alone and beside the gather; per-lane
//      mixes of predicated LDS.128 / LDS.64 values; a dominant value held in registers
// Prints cycles per warp instruction per SM at 16 resident warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_bench tools/smem_bench.cu && ./smem_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int UNR = 8;

// predicated shared loads (the predicate is per lane; inactive lanes keep the default)
__device__ __forceinline__ int4 lds128_if(const void* p, int on, int4 d) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("{ .reg .pred q; setp.ne.s32 q, %5, 0; @q ld.shared.v4.s32 {%0,%1,%2,%3}, [%4]; }"
                 : "+r"(d.x), "+r"(d.y), "+r"(d.z), "+r"(d.w) : "r"(a), "r"(on));
    return d;
}
__device__ __forceinline__ int2 lds64_if(const void* p, int on, int2 d) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("{ .reg .pred q; setp.ne.s32 q, %3, 0; @q ld.shared.v2.s32 {%0,%1}, [%2]; }"
                 : "+r"(d.x), "+r"(d.y) : "r"(a), "r"(on));
    return d;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(cudaTextureObject_t tex, long long* out, int4* sink) {
    __shared__ int4 buf[2048];  // 32 KB
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 2048; i += blockDim.x) buf[i] = make_int4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    int4 acc = make_int4(0, 0, 0, 0);
    int idx;
    if (MODE == 1 || MODE == 4 || MODE == 6 || MODE == 7 || MODE == 8 || MODE >= 9) idx = lane;  // (modes >= 12 use idx only for the gather)
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
            } else if (MODE == 12 || MODE == 13) {
                // LDS.64: one address / 8 distinct addresses
                const int2* const h = reinterpret_cast<const int2*>(buf);
                const int2 a = h[((MODE == 12 ? 5 : ((lane * 7) & 7)) + 8 * u + o2) & 63];
                acc.x ^= a.x; acc.y ^= a.y;
            } else if (MODE == 18 || MODE == 19) {
                // gather + LDS.64 value (one address / 8 distinct)
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int2* const h = reinterpret_cast<const int2*>(buf);
                const int2 a = h[((MODE == 18 ? 5 : ((lane * 7) & 7)) + 8 * u + o2) & 63];
                acc.x ^= v.x ^ a.x; acc.y ^= v.y ^ a.y; acc.z ^= v.z; acc.w ^= v.w;
            } else if (MODE == 20 || MODE == 21 || MODE == 22) {
                // gather + per-lane choice: complex value (LDS.128) on the lanes with
                // popcount(lane) == 2 [20] / lanes 0..7 [21] / none [22], imaginary-only
                // value (LDS.64) on the others; both from 8-entry dictionaries
                const int on = MODE == 20 ? (__popc(lane) == 2) : MODE == 21 ? (lane < 8) : (acc.w == 0x7ffffff1);
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int2* const h = reinterpret_cast<const int2*>(buf);
                const int j = (((lane * 7) & 7) + 8 * u + o2) & 63;
                const int4 w = lds128_if(&buf[j], on, make_int4(0, 0, 0, 0));
                const int2 a = lds64_if(&h[j + 2048], !on, make_int2(w.z, w.w));
                acc.x ^= v.x ^ w.x; acc.y ^= v.y ^ w.y; acc.z ^= v.z ^ a.x; acc.w ^= v.w ^ a.y;
            } else if (MODE == 23) {
                // gather + dominant value in registers, dictionary LDS.128 only on the
                // lanes with popcount(lane) == 2
                const int4 v = buf[(idx + 32 * u + o1) & 2047];
                const int4 w = lds128_if(&buf[(((lane * 7) & 7) + 8 * u + o2) & 63], __popc(lane) == 2, make_int4(o2, 2, 3, 4));
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
    run<12>("LDS.64, one address for the warp", tex, d_out, d_sink, sms);
    run<13>("LDS.64, 8 distinct addresses", tex, d_out, d_sink, sms);
    run<18>("LDS.128 distinct + LDS.64 one address", tex, d_out, d_sink, sms);
    run<19>("LDS.128 distinct + LDS.64 8-address", tex, d_out, d_sink, sms);
    run<20>("LDS.128 distinct + @p LDS.128 / @!p LDS.64, 10 lanes complex", tex, d_out, d_sink, sms);
    run<21>("LDS.128 distinct + @p LDS.128 / @!p LDS.64, lanes 0..7 complex", tex, d_out, d_sink, sms);
    run<22>("LDS.128 distinct + @p LDS.128 / @!p LDS.64, no lane complex", tex, d_out, d_sink, sms);
    run<23>("LDS.128 distinct + @p LDS.128 10 lanes (dominant value in registers)", tex, d_out, d_sink, sms);
    run<5>("tex1Dfetch<int4>, 8 distinct addresses", tex, d_out, d_sink, sms);
    run<6>("LDS.128 distinct + tex1Dfetch<int4> (x + value via TEX)", tex, d_out, d_sink, sms);
    return 0;
}
