// qtm_rng.cuh -- per-trajectory random streams on the device.
//
// Every thread of a trajectory's CTA evaluates the same stream redundantly
// (a few integer ops per draw, 1 + 2*jumps draws per trajectory), so draws
// never need to be broadcast.  Streams are keyed by the GLOBAL trajectory
// index k, which makes results independent of sharding and scheduling.
//
//   philox   : draw n = word (n & 3) of Philox4x32-10(ctr = (n >> 2, k_lo, k_hi, 0),
//              key = (seed_lo, seed_hi)) * 2^-32   (Salmon et al., SC'11)
//   lfsr113  : the reference's combined Tausworthe generator, one stream per
//              trajectory seeded with derive_stream(seed, k)
//              (/root/reference/pkg/src/mcwf/rng.py:37-90)
//   scripted : replay of a host-supplied list, then a fallback value
//              (reference tests/oracles.py:60-72)
#pragma once
#include <cstdint>

namespace qtm {

enum StreamKind : int { kPhilox = 0, kLfsr113 = 1, kScripted = 2 };

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

__device__ __forceinline__ uint32_t lfsr113_step(uint32_t z[4]) {
    uint32_t b;
    b = ((z[0] << 6) ^ z[0]) >> 13;  z[0] = ((z[0] & 4294967294u) << 18) ^ b;
    b = ((z[1] << 2) ^ z[1]) >> 27;  z[1] = ((z[1] & 4294967288u) << 2) ^ b;
    b = ((z[2] << 13) ^ z[2]) >> 21; z[2] = ((z[2] & 4294967280u) << 7) ^ b;
    b = ((z[3] << 3) ^ z[3]) >> 12;  z[3] = ((z[3] & 4294967168u) << 13) ^ b;
    return z[0] ^ z[1] ^ z[2] ^ z[3];
}

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct Stream {
    int kind;
    uint64_t seed, k, n;
    uint32_t z[4];           // lfsr113 state
    const double* script;    // scripted row
    int64_t script_len;
    double fallback;

    __device__ void init(int kind_, uint64_t seed_, uint64_t k_, const double* script_row,
                         int64_t len, double fb) {
        kind = kind_; seed = seed_; k = k_; n = 0;
        script = script_row; script_len = len; fallback = fb;
        z[0] = z[1] = z[2] = z[3] = 0;
        if (kind == kLfsr113) {
            const uint64_t golden = 0x9E3779B97F4A7C15ull;
            uint64_t x = seed ^ ((k + 1) * golden);
            uint32_t w[4];
            x = splitmix_mix(x + golden); w[0] = (uint32_t)x; w[1] = (uint32_t)(x >> 32);
            x = splitmix_mix(x + golden); w[2] = (uint32_t)x; w[3] = (uint32_t)(x >> 32);
            const uint32_t lo[4] = {1u, 7u, 15u, 127u};
#pragma unroll
            for (int i = 0; i < 4; ++i) z[i] = w[i] <= lo[i] ? (w[i] | (lo[i] + 1u)) : w[i];
            for (int i = 0; i < 16; ++i) lfsr113_step(z);
        }
    }

    __device__ __noinline__ double next() {
        const uint64_t i = n++;
        if (kind == kPhilox) {
            uint32_t c[4] = {(uint32_t)(i >> 2), (uint32_t)k, (uint32_t)(k >> 32), 0u};
            philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
            const uint32_t w = (i & 3) == 0 ? c[0] : (i & 3) == 1 ? c[1] : (i & 3) == 2 ? c[2] : c[3];
            return (double)w * 2.3283064365386963e-10;
        }
        if (kind == kLfsr113) return (double)lfsr113_step(z) * 2.3283064365386963e-10;
        return (int64_t)i < script_len ? script[i] : fallback;
    }
};

}  // namespace qtm
