// qtm_tmem.cuh -- Tensor Memory (TMEM) as per-thread storage for the
// Nordsieck history (sm_100a).
//
// Each SM has 256 KB of TMEM (128 lanes x 512 columns x 32 bit) next to its
// 256 KB register file.  The tensor cores have no FP64 kind, but TMEM is
// also plain addressable storage: with the 32x32b access shape a warp reads
// or writes 32 lanes (one per thread) x N consecutive columns, so every
// thread owns a private row of columns in its warp's lane quarter.  Holding
// Nordsieck rows >= 2 and the corrector terms e / e_prev there frees the
// registers and shared memory that otherwise limit a d = 1024 trajectory to
// one per SM: two trajectory CTAs then share an SM (128 registers/thread).
//
// Measured on the pool's B200 (tools/tmem_bench.cu): a 2 KB
// warp load (x16) + wait is ~125 cycles, a store ~120 cycles without a
// wait; 16 warps sustain > 400 B/cycle/SM of reads.
//
// Ordering: tcgen05.ld/st are asynchronous.  Registers written by a load are
// valid only after tcgen05.wait::ld; the wait below takes the destination
// registers as read-write operands so the compiler cannot move their uses
// above it.  A load of columns stored earlier by the same thread is preceded
// by tcgen05.wait::st (tm_wait_st), placed at the start of every load phase.
#pragma once
#include <cstdint>

namespace qtm {
namespace tm {

// ---- allocation (one warp of the CTA; the address goes through smem)
__device__ __forceinline__ void alloc(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(smem_dst)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// address of this thread's column block: lane quarter of the warp (warp % 4)
// in bits 16+, columns (warp / 4) * ncols_per_thread
__device__ __forceinline__ uint32_t thread_base(uint32_t taddr, int cols_per_thread) {
    const int warp = threadIdx.x >> 5;
    return taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * cols_per_thread);
}

// ---- raw 32-bit transfers: issue (no wait) / wait with the registers tied
#define QTM_R4(r, o) "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3])
#define QTM_R4IN(r, o) "r"(r[o + 0]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3])
#define QTM_R4T(r, o) "+r"(r[o + 0]), "+r"(r[o + 1]), "+r"(r[o + 2]), "+r"(r[o + 3])

__device__ __forceinline__ void issue_ld16(uint32_t a, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : QTM_R4(r, 0), QTM_R4(r, 4), QTM_R4(r, 8), QTM_R4(r, 12) : "r"(a));
}
__device__ __forceinline__ void wait_ld16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : QTM_R4T(r, 0), QTM_R4T(r, 4), QTM_R4T(r, 8), QTM_R4T(r, 12) :: "memory");
}
__device__ __forceinline__ void st16(uint32_t a, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 "
                 "[%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                 :: "r"(a), QTM_R4IN(r, 0), QTM_R4IN(r, 4), QTM_R4IN(r, 8), QTM_R4IN(r, 12) : "memory");
}
// 24 columns (6 complex doubles): x16 + x8
__device__ __forceinline__ void issue_ld24(uint32_t a, uint32_t (&r)[24]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%24];\n\t"
                 "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%25];\n"
                 : QTM_R4(r, 0), QTM_R4(r, 4), QTM_R4(r, 8), QTM_R4(r, 12), QTM_R4(r, 16), QTM_R4(r, 20)
                 : "r"(a), "r"(a + 16u));
}
__device__ __forceinline__ void wait_ld24(uint32_t (&r)[24]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : QTM_R4T(r, 0), QTM_R4T(r, 4), QTM_R4T(r, 8), QTM_R4T(r, 12), QTM_R4T(r, 16),
                   QTM_R4T(r, 20) :: "memory");
}
__device__ __forceinline__ void st24(uint32_t a, const uint32_t (&r)[24]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 "
                 "[%0], {%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17};\n\t"
                 "tcgen05.st.sync.aligned.32x32b.x8.b32 [%1], {%18,%19,%20,%21,%22,%23,%24,%25};\n"
                 :: "r"(a), "r"(a + 16u), QTM_R4IN(r, 0), QTM_R4IN(r, 4), QTM_R4IN(r, 8), QTM_R4IN(r, 12),
                    QTM_R4IN(r, 16), QTM_R4IN(r, 20) : "memory");
}
__device__ __forceinline__ void issue_ld4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void st4(uint32_t a, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" :: "r"(a), QTM_R4IN(r, 0) : "memory");
}
// W columns (W in 4..24, a multiple of 4) in x16 / x8 / x4 pieces
template <int W>
__device__ __forceinline__ void issue_ld(uint32_t a, uint32_t (&r)[W]) {
    static_assert(W % 4 == 0 && W >= 4 && W <= 28, "4..28 columns");
    if constexpr (W >= 16) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                     "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                     : QTM_R4(r, 0), QTM_R4(r, 4), QTM_R4(r, 8), QTM_R4(r, 12) : "r"(a));
    }
    constexpr int B = W >= 16 ? 16 : 0;
    if constexpr (W - B >= 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : QTM_R4(r, B), QTM_R4(r, B + 4) : "r"(a + B));
    }
    constexpr int C = B + ((W - B) >= 8 ? 8 : 0);
    if constexpr (W - C >= 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                     : QTM_R4(r, C) : "r"(a + C));
    }
}
// wait for every outstanding load; the registers are re-defined after the
// wait (empty asm, tied), so their uses cannot move above it
template <int W>
__device__ __forceinline__ void wait_ld(uint32_t (&r)[W]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < W; ++i) asm volatile("" : "+r"(r[i]));
}
template <int W>
__device__ __forceinline__ void st(uint32_t a, const uint32_t (&r)[W]) {
    static_assert(W % 4 == 0 && W >= 4 && W <= 28, "4..28 columns");
    if constexpr (W >= 16) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 "
                     "[%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                     :: "r"(a), QTM_R4IN(r, 0), QTM_R4IN(r, 4), QTM_R4IN(r, 8), QTM_R4IN(r, 12) : "memory");
    }
    constexpr int B = W >= 16 ? 16 : 0;
    if constexpr (W - B >= 8) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                     :: "r"(a + B), QTM_R4IN(r, B), QTM_R4IN(r, B + 4) : "memory");
    }
    constexpr int C = B + ((W - B) >= 8 ? 8 : 0);
    if constexpr (W - C >= 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n"
                     :: "r"(a + C), QTM_R4IN(r, C) : "memory");
    }
}
#undef QTM_R4
#undef QTM_R4IN
#undef QTM_R4T

// ---- complex doubles <-> 32-bit column words (lo, hi of x, then of y)
template <int N, int W>
__device__ __forceinline__ void unpack(const uint32_t (&r)[W], double2 (&v)[N]) {
    static_assert(W == 4 * N, "4 columns per complex double");
#pragma unroll
    for (int k = 0; k < N; ++k)
        v[k] = make_double2(__hiloint2double((int)r[4 * k + 1], (int)r[4 * k]),
                            __hiloint2double((int)r[4 * k + 3], (int)r[4 * k + 2]));
}
template <int N, int W>
__device__ __forceinline__ void pack(const double2 (&v)[N], uint32_t (&r)[W]) {
    static_assert(W == 4 * N, "4 columns per complex double");
#pragma unroll
    for (int k = 0; k < N; ++k) {
        r[4 * k + 0] = (uint32_t)__double2loint(v[k].x);
        r[4 * k + 1] = (uint32_t)__double2hiint(v[k].x);
        r[4 * k + 2] = (uint32_t)__double2loint(v[k].y);
        r[4 * k + 3] = (uint32_t)__double2hiint(v[k].y);
    }
}

}  // namespace tm
}  // namespace qtm
