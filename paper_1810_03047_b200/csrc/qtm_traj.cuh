// qtm_traj.cuh -- persistent sm_100a kernel that integrates whole quantum
// trajectories on chip.
//
// Mapping.  One CTA owns one trajectory at a time; NT threads each own E
// state components (component i = tid + NT*e, so shared-memory traffic is
// conflict-free).  The Nordsieck history z[0..q] lives in REGISTERS for rows
// j < RREG (rows >= RREG, reached only when the order climbs past the
// variant's budget, spill to a per-CTA global scratch).  Every thread
// evaluates the scalar controller (t, h, q, crate, ialth, nef, ncf, r, ...)
// redundantly from bitwise-identical block reductions, so control flow is
// CTA-uniform with no broadcasts.  The CTA pulls the next trajectory index
// from a global atomic counter when it finishes one (dynamic load balance
// for the heavy-tailed step counts); outputs land in per-trajectory slots,
// so results do not depend on scheduling.
//
// Reference behaviour reproduced per attempt:
//   predict / corrector / error test / commit ..... _kernels.py:117-192
//   retry loop, rejects, restarts ................. ode.py:261-329
//   order & step control .......................... ode.py:441-466
//   jump test, bisection, collapse, cold restart .. trajectory.py:133-182, 216-246
//   expectation recording ......................... trajectory.py:122-130, 206-214
// Differences from the reference are rounding-level only: block reductions
// are tree sums (the reference sums sequentially), the predicted history is
// undone in place on a rejected attempt instead of kept in a second copy,
// WRMS norms multiply by host-computed reciprocals of d and tau instead of
// dividing (FP64 division sits on the per-attempt critical path),
// hypot comes from CUDA's libdevice and the controller's fractional
// powers are exp2(y log2 x) (the reference: glibc hypot/pow).
#pragma once
#include <cstdint>
#include <type_traits>

#include <math_constants.h>

#include "qtm_rng.cuh"
#include "qtm_tmem.cuh"

namespace qtm {

constexpr int LROWS = 13;
constexpr int MAXOPS = 32;
constexpr int MAXTD = 8;    // time-dependent generator terms (QTM_MAX_TD_TERMS)
constexpr int KRED = 4;  // values carried by one block reduction
constexpr int NSTATS = 16;

enum Status : int {
    kOk = 0, kErrMaxSteps = -1, kErrRepeatedErrTest = -4, kErrStepCollapse = -5,
    kErrCorrector = -6, kErrBracket = -10, kErrNoSupport = -11, kErrZeroVector = -12,
};

enum Stat : int {
    sAttempts = 0, sSteps, sCorrFail, sErrReject, sNfe, sCorrIters, sJumps, sBisect, sSumQ,
    sOrderUp, sOrderDown, sDraws, sSumQQ1, sOverflow, sLuFactor,
};

// one compiled kernel configuration (see build.py VARIANTS)
struct VariantDesc {
    int threads, comps, reg_rows, min_blocks, auto_upto, td;
    size_t smem;
    const void* fn;
    int tm;     // Nordsieck rows 2..7 and e / e_prev in TMEM (HistT)
    int small;  // one thread per trajectory for d <= small (traj1_kernel, qtm_small.cuh); 0: no
    int lanes;  // small: trajectories per warp
};

struct DevCsr {
    const int* rp;
    const int* ci;
    const double2* v;
};

struct DevProblem {
    int d, nc, ne, n_pts, max_order;
    long long max_steps;
    double t_from, t_to, rtol, atol, h0_first;
    DevCsr g;
    DevCsr c[MAXOPS];
    DevCsr e[MAXOPS];
    const double2* psi0;
    const double* times;
    // G in sliced-ELL form for shared-memory staging (built per kernel
    // variant on the host): slice = 32 consecutive rows, the E slices of a
    // warp interleaved per column (SellSlots), entries uint32
    // (16*value-index | 16*col << 16), widths padded to be uniform per warp;
    // the value index points into a dictionary of the distinct entries of G
    // (index 0 = 0.0, used for padding).
    // sell_mode 0 = plain CSR through L1/L2 (d > 4096 or > 4095 distinct values).
    int sell_mode;
    int sell_entries, sell_dict_n;
    const uint32_t* sell_ent;
    const double2* sell_dict;
    // variants with sell_uses_tex(): the dictionary as a linear texture over
    // sell_dict; the entries' low half is then the value INDEX instead of its
    // byte offset
    unsigned long long sell_tex;
    // variants with sell_uses_dom(): when one purely imaginary value (0, b)
    // makes up most of G's stored entries (every off-diagonal of c4's Ising
    // chain is i h), its entries carry bit 0 instead of a dictionary offset
    // and take the value from this field: no dictionary load for them
    // (sell_dom_on bit 0).  Other purely imaginary values are stored as one
    // double behind the complex dictionary; their entries carry bit 1 and the
    // double's byte offset (sell_dom_on bit 1): an 8-byte load.
    int sell_dom_on;
    double sell_dom;
    const int* sell_off;    // [NT/32] first entry slot of each warp (SellSlots)
    const int* sell_w;      // [DP/32] width of each slice (uniform over a warp's E slices)
    // TD variants: the SELL above is built on the union pattern of G0 and
    // the sell_td staged time-dependent terms, and sell_td_ent ([sell_td]
    // arrays of uint16 per slot, same slot layout) holds the byte offset of
    // G_k's value in sell_td_dict (offset 0 = 0.0); staged after the G0 entries
    // sell_td == -1: a single staged term whose stored entries all hold ONE
    // value (c4td: the modulated transverse field) needs no per-slot table at
    // all -- bit 2 of the G0 entry says "G_1 has an entry here", its value is
    // sell_td_dom (which shares the storage of the two unused table
    // pointers), and G0's dominant value rides on bit 0 as in the
    // time-independent kernels.  (No new fields: growing this struct moves
    // the offsets of the kernel's second parameter, and with that alone the
    // register allocation of the time-independent TMEM variant gained 112
    // spill instructions and c4 ran 1.3 % slower.)
    int sell_td, sell_td_dict_n;
    union {
        struct {
            const double2* sell_td_dict;
            const uint16_t* sell_td_ent;
        };
        double sell_td_dom[2];
    };
    // observables that are diagonal in the basis (number operators, sigma_z):
    // bit k of e_diag_mask set => dense values at e_diag[k * DP + i]
    unsigned e_diag_mask;
    const double2* e_diag;
    int e_need_gather;      // some observable is not diagonal (needs all of psi)
    // diagonal observables with real entries and <= 256 distinct values are
    // staged in shared memory (bit k of e_stage_mask): a byte index per state
    // component, idx[k * DP + i], into a per-observable value dictionary
    // starting at entry e_dict_off[k]; the tables sit at byte offset
    // e_stage_off of the dynamic shared memory (copied from e_idx_g/e_dict_g)
    unsigned e_stage_mask;
    int e_stage_off, e_stage_idx_bytes, e_dict_n;
    int e_dict_off[MAXOPS];
    const uint8_t* e_idx_g;
    const double* e_dict_g;
    // e_fast: every observable is staged (recording takes the transposed
    // warp reduction); e_stage_dense: the staged table is the dense real
    // diagonal [ne][DP] (doubles, copied from e_dense_g) instead of bytes
    int e_fast, e_stage_dense;
    const double* e_dense_g;
    // small-state kernel (traj1_kernel): G, C_k, E_k as dense [d_max][d_max]
    // blocks, [1 + nc + ne][d_max][d_max]
    const double2* small_ops;
    double l[LROWS][LROWS];
    double tau1[LROWS], tau2[LROWS], tau3[LROWS];
    // per-order constants the reference evaluates inline, tabulated on the
    // host with the same IEEE operations: 0.5/(q+2), 1/(q+1), 1/q, 1/(q+2)
    double conit[LROWS], rq1[LROWS], rq0[LROWS], rq2[LROWS];
    // reciprocals for the WRMS norms: sqrt(acc / d) / tau becomes
    // sqrt(acc * inv_d) * inv_tau (last-bit differences only)
    double inv_d;
    double inv_tau1[LROWS], inv_tau2[LROWS], inv_tau3[LROWS];
    // order control keeps q and h (every ratio < 1.1) iff est > keep_same[q],
    // est_down > keep_down[q] (when q > 1) and est_up > keep_up[q] (when
    // raising is possible): ((1/1.1 - 1e-6) / bias)^k, k = q+1, q, q+2
    double keep_same[LROWS], keep_down[LROWS], keep_up[LROWS];
    // time-dependent right side G(t) = G + sum_k c_k(t) G_k (timedep.py):
    // c_k(t) = td_c[k][3] + td_c[k][0] cos(td_c[k][1] t + td_c[k][2])
    int n_td;
    DevCsr td[MAXTD];
    double td_c[MAXTD][4];
};

struct RunParams {
    uint64_t seed;
    long long traj_begin, n_traj;
    int stream_kind;
    const double* script;
    const long long* script_len;
    long long script_stride;
    double script_fallback;
    double* values;          // [n_traj][ne][n_pts] (written by finalize_records)
    double* rec_partial;     // [n_traj][n_pts][ne+1][NT/32] per-warp partial sums
    long long* stats;        // [n_traj][NSTATS]
    int* status;             // [n_traj]
    double* err;             // [n_traj][4]: t, h, aux0, aux1   (aux2 = r in err_r)
    double* err_r;           // [n_traj]
    long long* jump_count;   // [n_traj]
    double* jump_t;          // [n_traj][max_jumps]
    int* jump_idx;           // [n_traj][max_jumps]
    long long max_jumps;
    double2* zovf;           // [gridDim.x][LROWS-RREG][NT*E]
    unsigned long long* counter;
    unsigned long long* first_fail;  // atomicMin over failing rows
    unsigned long long* phase_cycles;  // [16] (QTM_PHASES builds only)
    int lanes;               // traj1_kernel: trajectories per warp
    // processing order of the launch's trajectories (nullptr: by index): the
    // j-th pull of the work counter integrates row order[j].  Outputs are
    // keyed by row, so the order changes when a trajectory runs, never what
    // it computes (qtm_capi.cu sorts by the first jump threshold, longest
    // expected trajectory first, to shorten the tail of the last wave)
    const int* order;
    // psi snapshots (diagnostics / parity): slot of each grid index (-1 =
    // none; nullptr = no snapshots) and the output [n_traj][n_psi][d]
    const int* psi_slot;
    double2* psi_out;
    int n_psi;
};

// next trajectory row of this launch from the global work counter (>= n_traj:
// none left), through the launch's processing order when it has one
__device__ __forceinline__ long long next_row(const RunParams& R) {
    const long long j = (long long)atomicAdd(R.counter, 1ull);
    return (R.order && j < R.n_traj) ? (long long)R.order[j] : j;
}

// ---------------------------------------------------------------- helpers
// The reference's numba kernels are compiled without fast-math, so no a*b+c
// is fused there.  The throughput build (build.py) lets nvcc contract into
// DFMA -- a ~1-ulp rounding difference per operation, the same order as the
// tree reductions, inside every parity tolerance; QTM_FMAD=0 builds the
// unfused parity library with the reference's rounding per operation.
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// |a| for the error weights 1/(atol + rtol |y_i|) (ode.py: np.abs, i.e.
// hypot).  QTM_FAST_ABS (default): sqrt(re^2 + im^2) -- within an ulp or two
// of hypot for the |y_i| <= 1 of a normalised state (an underflowing square
// only where atol dominates the weight anyway), at a fraction of hypot's
// instructions (c4 +1.3 %); QTM_FAST_ABS=0 restores hypot.
#ifndef QTM_FAST_ABS
#define QTM_FAST_ABS 1
#endif
__device__ __forceinline__ double cmod(double2 a) {
#if QTM_FAST_ABS
    return sqrt(a.x * a.x + a.y * a.y);
#else
    return hypot(a.x, a.y);
#endif
}

// The error weight 1/(atol + rtol |y|) (ode.py: the WRMS weights), with the
// correctly rounded reciprocal.  (Hardware rsqrt/rcp approximations with two
// Newton steps each: c4 +0.7 %, c5 +1.2 %, but the c5 sample mean moved from
// 1e-7 to 2e-6 against the reference: measured, not kept.)
__device__ __forceinline__ double err_weight(double atol, double rtol, double2 y) {
    return __drcp_rn(atol + rtol * cmod(y));
}

// est ** (1/(q+1)) etc. in the step-size controller (ode.py:302, 445-453):
// x > 0 and a small exponent, evaluated as exp2(y * log2(x)); within a few
// ulp of the correctly rounded power, at a fraction of pow()'s latency.
static __device__ __noinline__ double ctl_pow(double x, double y) {
    return x > 0.0 ? exp2(y * log2(x)) : (x == 0.0 ? 0.0 : pow(x, y));
}

// acc += v * x: the product (ac - bd, ad + bc), then the sum, as the
// reference's complex_mul + add (_kernels.py:18-26).  The rounding sequence
// is pinned with intrinsics, so it does not depend on which of the legal
// contractions the compiler would pick in a given loop shape (two forms of
// the imaginary part differ in the last bit, and did between variants):
//   throughput build:  re = fma(a, c, -rn(b d)),  im = fma(b, c, rn(a d))
//   QTM_FMAD=0:        every product and sum rounded, as numba computes it
// (Accumulating the four real products straight into the sums with FMAs
// saves two FP64 instructions per entry but moved c4 jump times by 9e-6
// against the reference, and was no faster: measured, not kept.)
#ifndef QTM_FMAD
#define QTM_FMAD 1
#endif
__device__ __forceinline__ void cmac(double& sr, double& si, double2 v, double2 x) {
#if QTM_FMAD
    sr = __dadd_rn(sr, __fma_rn(v.x, x.x, -__dmul_rn(v.y, x.y)));
    si = __dadd_rn(si, __fma_rn(v.y, x.x, __dmul_rn(v.x, x.y)));
#else
    sr = __dadd_rn(sr, __dsub_rn(__dmul_rn(v.x, x.x), __dmul_rn(v.y, x.y)));
    si = __dadd_rn(si, __dadd_rn(__dmul_rn(v.x, x.y), __dmul_rn(v.y, x.x)));
#endif
}

// y_i = sum_j M_ij x_j, left to right, each product (ac - bd, ad + bc) then
// accumulated (reference _kernels.py:150-154, numba complex_mul).
// not inlined: it serves the cold paths (recording of off-diagonal
// observables, collapse channels, the non-staged fallback) and keeping a
// single copy keeps the kernel's instruction footprint small
static __device__ __noinline__ double2 row_dot(const DevCsr& m, int i, const double2* __restrict__ x) {
    double sr = 0.0, si = 0.0;
    const int b = __ldg(m.rp + i), en = __ldg(m.rp + i + 1);
    for (int j = b; j < en; ++j) {
        cmac(sr, si, __ldg(m.v + j), x[__ldg(m.ci + j)]);
    }
    return make_double2(sr, si);
}

// Time-dependent right side: f_i + sum_k c_k(t) (G_k x)_i, the terms added
// one by one in order (TimeDependentGenerator.__call__, timedep.py), with
// c_k(t) = offset + amp cos(omega t + phase) evaluated once per product.
// Only the TD kernel variants carry these calls.
static __device__ __noinline__ double td_coef(const DevProblem& P, int k, double t) {
    return P.td_c[k][3] + P.td_c[k][0] * cos(P.td_c[k][1] * t + P.td_c[k][2]);
}
__device__ __forceinline__ double2 td_term(const DevCsr& m, double c, int i, const double2* __restrict__ x,
                                           double2 f) {
    const double2 g = row_dot(m, i, x);
    return make_double2(f.x + c * g.x, f.y + c * g.y);
}

// Entry slots of a warp in the staged sliced-ELL copy.  The E slices a warp
// walks together (rows tid + NT*e) are interleaved per ELL column k, in
// groups of V = 4 / 2 / 1 components (E % 4 == 0 / E even / E odd):
//   slot(k, e, lane) = k*32*E + (e/V)*32*V + lane*V + (e%V)      (+ warp base)
// so one 128-bit (64-bit) shared load fetches the entries of 4 (2) of the
// thread's rows, every load of column k is an immediate offset from one
// pointer that advances by 32*E per column, and the accesses are
// conflict-free (lane stride V words with V-word loads).
template <int E>
struct SellSlots {
    static constexpr int V = E % 4 == 0 ? 4 : (E % 2 == 0 ? 2 : 1);
    // slot of (e, lane) inside column 0 (add k*32*E for column k)
    __host__ __device__ static constexpr int in_col(int e, int lane) {
        return (e / V) * 32 * V + lane * V + (e % V);
    }
    // the E entries of this lane for one column; p = column base + lane*V
    __device__ __forceinline__ static void load(const uint32_t* __restrict__ p, uint32_t (&u)[E]) {
        if constexpr (V == 4) {
#pragma unroll
            for (int g = 0; g < E / 4; ++g) {
                const uint4 w = *reinterpret_cast<const uint4*>(p + g * 128);
                u[4 * g] = w.x; u[4 * g + 1] = w.y; u[4 * g + 2] = w.z; u[4 * g + 3] = w.w;
            }
        } else if constexpr (V == 2) {
#pragma unroll
            for (int g = 0; g < E / 2; ++g) {
                const uint2 w = *reinterpret_cast<const uint2*>(p + g * 64);
                u[2 * g] = w.x; u[2 * g + 1] = w.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) u[e] = p[e * 32];
        }
    }
    // the same for a uint16 array in the slot layout (TD term offsets)
    __device__ __forceinline__ static void load16(const uint16_t* __restrict__ p, uint32_t (&t)[E]) {
        if constexpr (V == 4) {
#pragma unroll
            for (int g = 0; g < E / 4; ++g) {
                const uint2 w = *reinterpret_cast<const uint2*>(p + g * 128);
                t[4 * g] = w.x & 0xFFFFu; t[4 * g + 1] = w.x >> 16;
                t[4 * g + 2] = w.y & 0xFFFFu; t[4 * g + 3] = w.y >> 16;
            }
        } else if constexpr (V == 2) {
#pragma unroll
            for (int g = 0; g < E / 2; ++g) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(p + g * 64);
                t[2 * g] = w & 0xFFFFu; t[2 * g + 1] = w >> 16;
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) t[e] = p[e * 32];
        }
    }
};

// f = G x for this thread's E rows from the staged sliced-ELL copy: the E
// rows' chains are interleaved for ILP; each row is still summed in column
// order (entries k ascending), so the rounding matches row_dot exactly.
// Entry = dictionary byte offset (low half) | x byte offset (col*16, high
// half): each entry costs two 16-byte shared loads and two address
// instructions (mask + uniform dictionary base; shift-add onto the gather
// buffer).
// Software-pipelined (PF = 1): the entries of column k+1 are loaded while
// column k is multiplied, the last column peeled so the loop carries no
// clamp.  The compact shared-history variants (RREG = 0) keep the plain loop
// (their code size matters more than the load latency).  (A distance-2
// pipeline that also prefetched the operands cost 4E registers more and lost
// wherever registers are tight: measured, dropped.)
#ifndef QTM_SPMV_PF
#define QTM_SPMV_PF(RREG) ((RREG) == 0 ? 0 : 1)
#endif
// unroll factor of the pipelined column loop: 1 (measured on c4 under the
// TMEM variant's 128-register cap: the compiler's own choice of 2 spilled more
// and ran 1.5 % slower; c5 / c2 / c4td within 1 % either way)
#ifndef QTM_SPMV_UNROLL
#define QTM_SPMV_UNROLL 1
#endif
#define QTM_PRAGMA_(x) _Pragma(#x)
#define QTM_PRAGMA(x) QTM_PRAGMA_(x)
#define QTM_SPMV_UNROLL_PRAGMA QTM_PRAGMA(unroll QTM_SPMV_UNROLL)
__device__ __forceinline__ double2 sell_val(const char* db, uint32_t u) {
    return *reinterpret_cast<const double2*>(db + (u & 0xFFFFu));
}
__device__ __forceinline__ double2 sell_x(const char* xb, uint32_t u) {
    return *reinterpret_cast<const double2*>(xb + (u >> 16));
}
// QTM_SELL_TEX: the dictionary values come through the TEXTURE pipe
// (tex1Dfetch over the dictionary in HBM, L1/TEX-cached) instead of shared
// memory.  The shared-memory (LSU) data pipe is this kernel's binding
// resource and the texture pipe runs beside it: measured with
// tools/smem_bench.cu, a 16-byte gather plus a 16-byte dictionary load from
// shared memory cost 4 + 4 SM-cycles per warp on the LSU pipe; with the value
// as a tex1Dfetch<int4> the pair still takes 8 (the fetch alone: 8), but only
// 4 of them on the LSU pipe -- the fetch overlaps the shared-memory load
// completely.
// Where it pays (measured A/B, bitwise the same results): the three-warp
// one-row-per-thread variants at 8 CTAs per SM (c3, (96, 1, 9): 486 -> 452 ms
// per step) -- enough warps to hide the texture latency, and a SpMV short
// enough that the fetches of one column cover most of it.  Elsewhere it does
// not: the wide variants lose (c4 109 -> 127 ms, c5 2 810 -> 3 123 ms per
// 4 096 trajectories even with the values prefetched a column ahead: 16 warps
// per SM do not cover ~500 cycles per column), and the other small shapes are
// mixed on 512-trajectory samples ((64, 1, 13) on c2 13.1 -> 15.2 ms,
// (32, 1, 13) 13.1 -> 11.5, (128, 1, 13) on c3 30.4 -> 30.9), so they keep the
// dictionary in shared memory.
#ifndef QTM_SELL_TEX
#define QTM_SELL_TEX 1
#endif
// the variants whose dictionary goes through the texture pipe
__host__ __device__ constexpr bool sell_uses_tex(int threads, int comps, int reg_rows, bool td) {
    return QTM_SELL_TEX && comps == 1 && reg_rows > 0 && threads == 96 && !td;
}
__device__ __forceinline__ double2 tex_val(unsigned long long tex, uint32_t u) {
    const int4 t = tex1Dfetch<int4>((cudaTextureObject_t)tex, (int)(u & 0xFFFFu));
    return make_double2(__hiloint2double(t.y, t.x), __hiloint2double(t.w, t.z));
}
// QTM_SELL_DOM: the dominant purely imaginary value of G comes from the kernel
// parameters instead of the dictionary (DevProblem::sell_dom).  The load is
// predicated per lane on bit 0 of the entry; the product is formed by the same
// cmac from the same bits (re = +0.0), so the results are bitwise unchanged.
#ifndef QTM_SELL_DOM
#define QTM_SELL_DOM 1
#endif
// the variants that take it: the wide register / TMEM variants (several rows
// per thread, pipelined SpMV), whose bound is the shared-memory data pipe
__host__ __device__ constexpr bool sell_uses_dom(int threads, int comps, int reg_rows, bool td) {
    return QTM_SELL_DOM && comps > 1 && reg_rows > 0 && !td && !sell_uses_tex(threads, comps, reg_rows, td);
}
// the TD variants that take the single-valued-term form (sell_spmv_tdd)
__host__ __device__ constexpr bool sell_uses_tdd(int comps, int reg_rows, bool td) {
    return QTM_SELL_DOM && td && comps > 1 && reg_rows > 0;
}
// MODE bit 0: entries with bit 0 take the dominant value; MODE bit 1: entries
// with bit 1 are purely imaginary and load 8 bytes (the imaginary part) from
// the offset in bits 3..15.  The loads are predicated per lane; lanes whose
// predicate is off move nothing through the shared-memory pipe.
template <int MODE>
__device__ __forceinline__ double2 sell_val_flag(uint32_t dbs, uint32_t u, double dom) {
    double2 v = make_double2(0.0, (MODE & 1) ? dom : 0.0);
    const uint32_t a = dbs + (u & 0xFFF8u);
    if constexpr (MODE == 1) {
        asm("{\n\t.reg .pred q;\n\t.reg .b32 t;\n\tand.b32 t, %3, 1;\n\tsetp.eq.u32 q, t, 0;\n\t"
            "@q ld.shared.v2.f64 {%0, %1}, [%2];\n\t}"
            : "+d"(v.x), "+d"(v.y) : "r"(a), "r"(u));
    } else if constexpr (MODE == 2) {
        asm("{\n\t.reg .pred q;\n\t.reg .b32 t;\n\tand.b32 t, %3, 2;\n\tsetp.eq.u32 q, t, 0;\n\t"
            "@q ld.shared.v2.f64 {%0, %1}, [%2];\n\t@!q ld.shared.f64 %1, [%2];\n\t}"
            : "+d"(v.x), "+d"(v.y) : "r"(a), "r"(u));
    } else {
        asm("{\n\t.reg .pred q, r;\n\t.reg .b32 t;\n\tand.b32 t, %3, 3;\n\tsetp.eq.u32 q, t, 0;\n\t"
            "and.b32 t, %3, 2;\n\tsetp.ne.u32 r, t, 0;\n\t"
            "@q ld.shared.v2.f64 {%0, %1}, [%2];\n\t@r ld.shared.f64 %1, [%2];\n\t}"
            : "+d"(v.x), "+d"(v.y) : "r"(a), "r"(u));
    }
    return v;
}
// the pipelined column loop of the wide variants with flagged entries (one
// copy per MODE, chosen per problem: problems without such entries keep the
// plain loop below and pay nothing)
template <int E, int MODE>
__device__ __forceinline__ void sell_cols_flag(const uint32_t* __restrict__ p, const char* db, const char* xb,
                                               int width, double dom, double (&sr)[E], double (&si)[E]) {
    using S = SellSlots<E>;
    if (width <= 0) return;
    const uint32_t dbs = (uint32_t)__cvta_generic_to_shared(db);
    uint32_t u[E];
    S::load(p, u);
    QTM_SPMV_UNROLL_PRAGMA
    for (int k = 1; k < width; ++k) {
        double2 v[E], xv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            v[e] = sell_val_flag<MODE>(dbs, u[e], dom);
            xv[e] = sell_x(xb, u[e]);
        }
        p += 32 * E;
        S::load(p, u);
#pragma unroll
        for (int e = 0; e < E; ++e) cmac(sr[e], si[e], v[e], xv[e]);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) cmac(sr[e], si[e], sell_val_flag<MODE>(dbs, u[e], dom), sell_x(xb, u[e]));
}
template <int NT, int E, int PF, bool TEX = false, bool DOM = false>
__device__ __forceinline__ void sell_spmv(const uint32_t* __restrict__ ent,
                                          const double2* __restrict__ dict, int woff,
                                          int width, const double2* __restrict__ x,
                                          double2 (&out)[E], unsigned long long tex = 0,
                                          int dom_on = 0, double dom = 0.0) {
    using S = SellSlots<E>;
    const int lane = threadIdx.x & 31;
    const char* const xb = reinterpret_cast<const char*>(x);
    const char* const db = reinterpret_cast<const char*>(dict);
    const uint32_t* p = ent + woff + lane * S::V;
    double sr[E], si[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { sr[e] = 0.0; si[e] = 0.0; }
    if constexpr (TEX) {
        // values one column ahead through the texture pipe (long latency), the
        // gathered x just in time from shared memory
        if (width > 0) {
            uint32_t u[E];
            double2 v[E];
            S::load(p, u);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = tex_val(tex, u[e]);
            QTM_SPMV_UNROLL_PRAGMA
            for (int k = 1; k < width; ++k) {
                double2 xv[E], vn[E];
#pragma unroll
                for (int e = 0; e < E; ++e) xv[e] = sell_x(xb, u[e]);
                p += 32 * E;
                S::load(p, u);
#pragma unroll
                for (int e = 0; e < E; ++e) vn[e] = tex_val(tex, u[e]);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    cmac(sr[e], si[e], v[e], xv[e]);
                    v[e] = vn[e];
                }
            }
#pragma unroll
            for (int e = 0; e < E; ++e) cmac(sr[e], si[e], v[e], sell_x(xb, u[e]));
        }
    } else if constexpr (PF == 0) {
#pragma unroll (E >= 4 ? 1 : 2)
        for (int k = 0; k < width; ++k) {
            uint32_t u[E];
            S::load(p, u);
            p += 32 * E;
#pragma unroll
            for (int e = 0; e < E; ++e) cmac(sr[e], si[e], sell_val(db, u[e]), sell_x(xb, u[e]));
        }
    } else if constexpr (E == 1) {
        // one row per thread (a few entries per row): the clamped prefetch
        // keeps a single copy of the loop body
        uint32_t u = width > 0 ? p[0] : 0u;
        for (int k = 0; k < width; ++k) {
            const int kn = k + 1 < width ? k + 1 : k;
            const double2 v = sell_val(db, u), xv = sell_x(xb, u);
            u = p[kn * 32];
            cmac(sr[0], si[0], v, xv);
        }
    } else if (DOM && dom_on) {
        if (dom_on == 1) sell_cols_flag<E, 1>(p, db, xb, width, dom, sr, si);
        else if (dom_on == 2) sell_cols_flag<E, 2>(p, db, xb, width, dom, sr, si);
        else sell_cols_flag<E, 3>(p, db, xb, width, dom, sr, si);
    } else if (width > 0) {
        uint32_t u[E];
        S::load(p, u);
        QTM_SPMV_UNROLL_PRAGMA
        for (int k = 1; k < width; ++k) {
            double2 v[E], xv[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                v[e] = sell_val(db, u[e]);
                xv[e] = sell_x(xb, u[e]);
            }
            p += 32 * E;
            S::load(p, u);
#pragma unroll
            for (int e = 0; e < E; ++e) cmac(sr[e], si[e], v[e], xv[e]);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) cmac(sr[e], si[e], sell_val(db, u[e]), sell_x(xb, u[e]));
    }
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] = make_double2(sr[e], si[e]);
}

// G0 x and G1 x in one pass over the union-pattern SELL (TD variants with a
// single time-dependent term): each row of each product is summed in column
// order, as csr_matvec sums the row (zero-valued slots add exact zeros).
template <int NT, int E>
__device__ __forceinline__ void sell_spmv_td(const uint32_t* __restrict__ ent, const double2* __restrict__ dict,
                                             const uint16_t* __restrict__ tent, const double2* __restrict__ tdict,
                                             int woff, int width, const double2* __restrict__ x,
                                             double2 (&out0)[E], double2 (&out1)[E]) {
    using S = SellSlots<E>;
    const int lane = threadIdx.x & 31;
    const char* const xb = reinterpret_cast<const char*>(x);
    const char* const db = reinterpret_cast<const char*>(dict);
    const char* const tb = reinterpret_cast<const char*>(tdict);
    double sr[E], si[E], tr[E], ti[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { sr[e] = 0.0; si[e] = 0.0; tr[e] = 0.0; ti[e] = 0.0; }
    const uint32_t* p = ent + woff + lane * S::V;
    const uint16_t* pt = tent + woff + lane * S::V;
    for (int k = 0; k < width; ++k) {
        uint32_t u[E], tu[E];
        S::load(p, u);
        S::load16(pt, tu);
        p += 32 * E;
        pt += 32 * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double2 v = sell_val(db, u[e]);
            const double2 w = *reinterpret_cast<const double2*>(tb + tu[e]);
            const double2 xv = sell_x(xb, u[e]);
            cmac(sr[e], si[e], v, xv);
            cmac(tr[e], ti[e], w, xv);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        out0[e] = make_double2(sr[e], si[e]);
        out1[e] = make_double2(tr[e], ti[e]);
    }
}

#ifndef QTM_TDD_PF
#define QTM_TDD_PF 0
#endif
// The same two products when G_1's stored entries all hold one value
// (DevProblem::sell_td == -1): G_1's value per slot is `tdom` where bit 2 of
// the entry is set and an exact zero elsewhere -- the bits sell_spmv_td reads
// from its tables -- and G0's dominant value comes from `dom` (bit 0).  Two
// shared-memory loads per slot (entry, gathered x) plus the diagonal's value
// instead of five.
template <int NT, int E>
__device__ __forceinline__ void sell_spmv_tdd(const uint32_t* __restrict__ ent, const double2* __restrict__ dict,
                                              int woff, int width, const double2* __restrict__ x,
                                              double2 (&out0)[E], double2 (&out1)[E], double dom, double2 tdom) {
    using S = SellSlots<E>;
    const int lane = threadIdx.x & 31;
    const char* const xb = reinterpret_cast<const char*>(x);
    const uint32_t dbs = (uint32_t)__cvta_generic_to_shared(dict);
    double sr[E], si[E], tr[E], ti[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { sr[e] = 0.0; si[e] = 0.0; tr[e] = 0.0; ti[e] = 0.0; }
    const uint32_t* p = ent + woff + lane * S::V;
#if QTM_TDD_PF
    // the entries of column k+1 loaded while column k is multiplied (as the
    // time-independent wide loop does)
    if (width > 0) {
        uint32_t u[E];
        S::load(p, u);
        for (int k = 1; k <= width; ++k) {
            double2 v[E], xv[E];
            uint32_t f[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                v[e] = sell_val_flag<1>(dbs, u[e], dom);
                xv[e] = sell_x(xb, u[e]);
                f[e] = u[e] & 4u;
            }
            if (k < width) {
                p += 32 * E;
                S::load(p, u);
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const double2 w = f[e] ? tdom : make_double2(0.0, 0.0);
                cmac(sr[e], si[e], v[e], xv[e]);
                cmac(tr[e], ti[e], w, xv[e]);
            }
        }
    }
#else
    for (int k = 0; k < width; ++k) {
        uint32_t u[E];
        S::load(p, u);
        p += 32 * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double2 v = sell_val_flag<1>(dbs, u[e], dom);
            const double2 w = (u[e] & 4u) ? tdom : make_double2(0.0, 0.0);
            const double2 xv = sell_x(xb, u[e]);
            cmac(sr[e], si[e], v, xv);
            cmac(tr[e], ti[e], w, xv);
        }
    }
#endif
#pragma unroll
    for (int e = 0; e < E; ++e) {
        out0[e] = make_double2(sr[e], si[e]);
        out1[e] = make_double2(tr[e], ti[e]);
    }
}

// G_k x alone over the union-pattern SELL (TD variants with several staged
// terms): G_k's value per slot from its uint16 offsets, rows in column order.
template <int NT, int E>
__device__ __forceinline__ void sell_spmv_term(const uint32_t* __restrict__ ent, const uint16_t* __restrict__ tent,
                                               const double2* __restrict__ tdict, int woff, int width,
                                               const double2* __restrict__ x, double2 (&out)[E]) {
    using S = SellSlots<E>;
    const int lane = threadIdx.x & 31;
    const char* const xb = reinterpret_cast<const char*>(x);
    const char* const tb = reinterpret_cast<const char*>(tdict);
    double tr[E], ti[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { tr[e] = 0.0; ti[e] = 0.0; }
    const uint32_t* p = ent + woff + lane * S::V;
    const uint16_t* pt = tent + woff + lane * S::V;
    for (int k = 0; k < width; ++k) {
        uint32_t u[E], tu[E];
        S::load(p, u);
        S::load16(pt, tu);
        p += 32 * E;
        pt += 32 * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double2 w = *reinterpret_cast<const double2*>(tb + tu[e]);
            const double2 xv = sell_x(xb, u[e]);
            cmac(tr[e], ti[e], w, xv);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] = make_double2(tr[e], ti[e]);
}

// One lane-halving level of a multi-value warp reduction: lanes with bit m
// clear keep the first half of a[0..N), the others the second half, and
// each adds its partner's copy of the half it keeps (a fixed order, so the
// result is deterministic).  After log2(N) levels lane l holds value slot
// (bits of l selected by the masks) summed over the lanes that agree with
// it in those bits.
template <int N, int S>
__device__ __forceinline__ void warp_halve(double (&a)[S], int m) {
    const bool upper = (threadIdx.x & m) != 0;
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
        const double send = upper ? a[j] : a[j + N / 2];
        const double keep = upper ? a[j + N / 2] : a[j];
        a[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
}

// Bitwise-identical sums on every thread of the CTA.  Inside each warp the K
// values are reduced by halving levels (each lane keeps half of the slots it
// still holds) and then butterflies, so K = 3 costs 12 shuffles instead of
// 30; the lanes holding a finished slot publish it; after ONE barrier every
// thread adds the NW warp partials of each slot in warp order -- the same
// data in the same order everywhere.  Double-buffered scratch => one
// barrier per reduction.  (One warp: plain xor-butterfly, all lanes agree.)
template <int NT, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red, int& phase) {
    static_assert(K >= 1 && K <= KRED, "block_sum carries at most KRED values");
    if constexpr (NT == 32) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], m);
        }
    } else {
        constexpr int NW = NT / 32;
        double* buf = red + phase * (KRED * NW);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if constexpr (K == 1) {
            double s = v[0];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
            if (lane == 0) buf[warp] = s;
        } else if constexpr (K == 2) {
            double a[2] = {v[0], v[1]};
            warp_halve<2>(a, 16);
#pragma unroll
            for (int m = 8; m >= 1; m >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], m);
            if ((lane & 15) == 0) buf[(lane >> 4) * NW + warp] = a[0];
        } else {
            double a[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) a[k] = k < K ? v[k] : 0.0;
            warp_halve<4>(a, 16);
            warp_halve<2>(a, 8);
#pragma unroll
            for (int m = 4; m >= 1; m >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], m);
            const int slot = ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
            if ((lane & 7) == 0 && slot < K) buf[slot * NW + warp] = a[0];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = buf[k * NW];
#pragma unroll
            for (int w = 1; w < NW; ++w) s += buf[k * NW + w];
            v[k] = s;
        }
        phase ^= 1;
    }
}


// Sum over the 32 lanes of a warp; the result is valid in lane 0 (the
// tree order is fixed, so it is deterministic).
template <int K>
__device__ __forceinline__ void warp_sum_lane0(double (&v)[K]) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] += __shfl_down_sync(0xffffffffu, v[k], m);
    }
}

// Recording when every observable is a staged real diagonal: per warp the
// partial <psi|E_k|psi> = sum_i E_k(i) |psi_i|^2 for k < ne and <psi|psi>
// (slot ne), in groups of 8 slots.  The 8 per-lane values of a group are
// reduced by three halving levels (16, 8, 4) and two butterflies (2, 1):
// 18 shuffles for 8 values instead of 80; lanes 4j' store the slots.
template <int NT, int E, bool DENSE>
__device__ __forceinline__ void record_staged(const DevProblem& P, const double2* smem,
                                              const double (&pw)[E], double* rp) {
    constexpr int DP = NT * E;
    const int lane = threadIdx.x & 31;
    const char* const base = reinterpret_cast<const char*>(smem) + P.e_stage_off;
    const double* const dense = reinterpret_cast<const double*>(base) + threadIdx.x;
    const uint8_t* const idx = reinterpret_cast<const uint8_t*>(base) + threadIdx.x;
    const double* const dict = reinterpret_cast<const double*>(base + P.e_stage_idx_bytes);
    for (int g = 0; g <= P.ne; g += 8) {
        double a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = g + j;
            double acc = 0.0;
            if (k < P.ne) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const double v = DENSE ? dense[k * DP + NT * e]
                                           : dict[P.e_dict_off[k] + idx[k * DP + NT * e]];
                    acc += v * pw[e];
                }
            } else if (k == P.ne) {
#pragma unroll
                for (int e = 0; e < E; ++e) acc += pw[e];
            }
            a[j] = acc;
        }
        warp_halve<8>(a, 16);
        warp_halve<4>(a, 8);
        warp_halve<2>(a, 4);
        a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
        a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
        const int slot = g + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        if ((lane & 3) == 0 && slot <= P.ne) rp[(size_t)slot * (NT / 32)] = a[0];
    }
}

// ------------------------------------------------ Nordsieck history helpers
// Rows j < RREG are a register array (static indices after unrolling, with
// uniform runtime predicates on q); rows j >= RREG live in the thread's
// overflow column ovf[e][(j - RREG) * DP] and are walked by plain runtime
// loops, so the register path carries no overflow code.
template <int RREG, int E, int DP>
struct Hist {
    using Z = double2[RREG][E];
    // this thread's overflow column: row j >= RREG of component e
    struct O {
        double2* p;
        __device__ __forceinline__ double2& at(int j, int e) const { return p[(j - RREG) * DP + e * (DP / E)]; }
    };

    __device__ __forceinline__ static double2& at(Z& z, int j, int e) { return z[j][e]; }
    __device__ __forceinline__ static const double2& at(const Z& z, int j, int e) { return z[j][e]; }

    // ---- order-specialised register paths (q + 1 <= RREG): straight-line
    // code, no per-row guards.  Dispatch by switch on the uniform order.
    template <int Q>
    __device__ __forceinline__ static void predict_q(Z& z) {
#pragma unroll
        for (int r = 0; r < Q; ++r)
#pragma unroll
            for (int j = Q - 1; j >= r; --j)
#pragma unroll
                for (int e = 0; e < E; ++e) z[j][e] = cadd(z[j][e], z[j + 1][e]);
    }
    template <int Q>
    __device__ __forceinline__ static void undo_q(Z& z) {
#pragma unroll
        for (int r = Q - 1; r >= 0; --r)
#pragma unroll
            for (int j = r; j < Q; ++j)
#pragma unroll
                for (int e = 0; e < E; ++e) z[j][e] = csub(z[j][e], z[j + 1][e]);
    }
    template <int Q>
    __device__ __forceinline__ static void rescale_q(Z& z, double ratio) {
        double f = 1.0;
#pragma unroll
        for (int j = 1; j <= Q; ++j) {
            f *= ratio;
#pragma unroll
            for (int e = 0; e < E; ++e) z[j][e] = cscale(f, z[j][e]);
        }
    }
    template <int Q>
    __device__ __forceinline__ static void commit_q(Z& z, const double* l, const double2 (&ev)[E]) {
#pragma unroll
        for (int j = 0; j <= Q; ++j) {
            const double lj = l[j];
#pragma unroll
            for (int e = 0; e < E; ++e) z[j][e] = cadd(z[j][e], cscale(lj, ev[e]));
        }
    }
    template <int Q>
    __device__ __forceinline__ static void horner_q(const Z& z, double s, double2 (&out)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = z[Q][e];
#pragma unroll
        for (int j = Q - 1; j >= 0; --j)
#pragma unroll
            for (int e = 0; e < E; ++e) out[e] = cadd(cscale(s, out[e]), z[j][e]);
    }

#define QTM_QSWITCH(CALL)                                                    \
    switch (q) {                                                             \
        case 1: if constexpr (2 <= RREG) { CALL(1); return; } break;         \
        case 2: if constexpr (3 <= RREG) { CALL(2); return; } break;         \
        case 3: if constexpr (4 <= RREG) { CALL(3); return; } break;         \
        case 4: if constexpr (5 <= RREG) { CALL(4); return; } break;         \
        case 5: if constexpr (6 <= RREG) { CALL(5); return; } break;         \
        case 6: if constexpr (7 <= RREG) { CALL(6); return; } break;         \
        case 7: if constexpr (8 <= RREG) { CALL(7); return; } break;         \
        case 8: if constexpr (9 <= RREG) { CALL(8); return; } break;         \
        case 9: if constexpr (10 <= RREG) { CALL(9); return; } break;        \
        case 10: if constexpr (11 <= RREG) { CALL(10); return; } break;      \
        case 11: if constexpr (12 <= RREG) { CALL(11); return; } break;      \
        case 12: if constexpr (13 <= RREG) { CALL(12); return; } break;      \
        default: break;                                                      \
    }

    // ---- general paths (any q; rows >= RREG in the overflow column)
    // zp = Pascal(z) in place, passes r = 0..q-1, j = q-1 down to r
    // (_kernels.py:133-137)
    __device__ __forceinline__ static void predict(Z& z, const O& ovf, int q) {
#define CALL_(Q) predict_q<Q>(z)
        QTM_QSWITCH(CALL_)
#undef CALL_
        for (int r = 0; r < q; ++r) {
            for (int j = q - 1; j >= (r > RREG ? r : RREG); --j) {
#pragma unroll
                for (int e = 0; e < E; ++e)
                    ovf.at(j, e) = cadd(ovf.at(j, e), ovf.at(j + 1, e));
            }
            if (RREG - 1 >= r && RREG - 1 < q) {
#pragma unroll
                for (int e = 0; e < E; ++e) z[RREG - 1][e] = cadd(z[RREG - 1][e], ovf.at(RREG, e));
            }
#pragma unroll
            for (int j = RREG - 2; j >= 0; --j) {
                if (j >= r && j < q) {
#pragma unroll
                    for (int e = 0; e < E; ++e) z[j][e] = cadd(z[j][e], z[j + 1][e]);
                }
            }
        }
    }

    // inverse of predict (rejected attempt): passes r = q-1..0, j = r..q-1
    __device__ __forceinline__ static void undo(Z& z, const O& ovf, int q) {
        for (int r = q - 1; r >= 0; --r) {
#pragma unroll
            for (int j = 0; j < RREG - 1; ++j) {
                if (j >= r && j < q) {
#pragma unroll
                    for (int e = 0; e < E; ++e) z[j][e] = csub(z[j][e], z[j + 1][e]);
                }
            }
            if (RREG - 1 >= r && RREG - 1 < q) {
#pragma unroll
                for (int e = 0; e < E; ++e) z[RREG - 1][e] = csub(z[RREG - 1][e], ovf.at(RREG, e));
            }
            for (int j = (r > RREG ? r : RREG); j < q; ++j) {
#pragma unroll
                for (int e = 0; e < E; ++e)
                    ovf.at(j, e) = csub(ovf.at(j, e), ovf.at(j + 1, e));
            }
        }
    }

    // z[j] *= ratio^j, j = 1..q, ratio^j by repeated multiplication
    // (nordsieck_rescale, _kernels.py:107-114)
    __device__ __forceinline__ static void rescale(Z& z, const O& ovf, int q, double ratio) {
        double f = 1.0;
#pragma unroll
        for (int j = 1; j < RREG; ++j) {
            if (j <= q) {
                f *= ratio;
#pragma unroll
                for (int e = 0; e < E; ++e) z[j][e] = cscale(f, z[j][e]);
            }
        }
        for (int j = RREG; j <= q; ++j) {
            f *= ratio;
#pragma unroll
            for (int e = 0; e < E; ++e) ovf.at(j, e) = cscale(f, ovf.at(j, e));
        }
    }

    // z[j] += l_j e, j = 0..q (_kernels.py:187-191)
    __device__ __forceinline__ static void commit(Z& z, const O& ovf, int q, const double* l,
                                                  const double2 (&ev)[E]) {
#define CALL_(Q) commit_q<Q>(z, l, ev)
        QTM_QSWITCH(CALL_)
#undef CALL_
#pragma unroll
        for (int j = 0; j < RREG; ++j) {
            if (j <= q) {
                const double lj = l[j];
#pragma unroll
                for (int e = 0; e < E; ++e) z[j][e] = cadd(z[j][e], cscale(lj, ev[e]));
            }
        }
        for (int j = RREG; j <= q; ++j) {
            const double lj = l[j];
#pragma unroll
            for (int e = 0; e < E; ++e) ovf.at(j, e) = cadd(ovf.at(j, e), cscale(lj, ev[e]));
        }
    }

    __device__ __forceinline__ static void row_all(const Z& z, const O& ovf, int j, double2 (&out)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = row(z, ovf, j, e);
    }
    __device__ __forceinline__ static void set_row_all(Z& z, const O& ovf, int j, const double2 (&v)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) set_row(z, ovf, j, e, v[e]);
    }
    __device__ __forceinline__ static double2 row(const Z& z, const O& ovf, int j, int e) {
        if (j >= RREG) return ovf.at(j, e);
        double2 out = z[0][e];
#pragma unroll
        for (int jj = 1; jj < RREG; ++jj) if (jj == j) out = z[jj][e];
        return out;
    }

    __device__ __forceinline__ static void set_row(Z& z, const O& ovf, int j, int e, double2 v) {
        if (j >= RREG) { ovf.at(j, e) = v; return; }
#pragma unroll
        for (int jj = 0; jj < RREG; ++jj) if (jj == j) z[jj][e] = v;
    }

    __device__ __forceinline__ static void horner_fast(const Z& z, const O& ovf, int q, double s, double2 (&out)[E]) {
        horner(z, ovf, q, s, out);
    }
    // psi(s) = Horner over rows q..0 (nordsieck_eval, _kernels.py:61-69)
    __device__ __forceinline__ static void horner(const Z& z, const O& ovf, int q, double s, double2 (&out)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = row(z, ovf, q, e);
        for (int j = q - 1; j >= RREG; --j) {
#pragma unroll
            for (int e = 0; e < E; ++e) out[e] = cadd(cscale(s, out[e]), ovf.at(j, e));
        }
#pragma unroll
        for (int j = RREG - 1; j >= 0; --j) {
            if (j < q) {
#pragma unroll
                for (int e = 0; e < E; ++e) out[e] = cadd(cscale(s, out[e]), z[j][e]);
            }
        }
    }
#undef QTM_QSWITCH
};

// ---------------------------------------- history in shared memory (RREG = 0)
// Small-state variants keep all Nordsieck rows in shared memory: row j of
// component e of thread t at p[j*DP + t + (DP/E)*e] (conflict-free, each
// thread touches only its own column).  The operations become short runtime
// loops, so the kernel's code stays small and its registers few -- this
// regime (d <= ~100, one or a few warps per trajectory) is bound by
// instruction fetch and latency, not by the row arithmetic.
template <int E, int DP>
struct HistS {
    struct Z {
        double2* p;
    };
    struct O {
        double2* p;
    };
    __device__ __forceinline__ static double2& at(const Z& z, int j, int e) {
        return z.p[j * DP + threadIdx.x + (DP / E) * e];
    }
    __device__ __forceinline__ static void predict(Z& z, const O&, int q) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            for (int r = 0; r < q; ++r) {
                double2 carry = at(z, q, e);
                for (int j = q - 1; j >= r; --j) {
                    const double2 v = cadd(at(z, j, e), carry);
                    at(z, j, e) = v;
                    carry = v;
                }
            }
        }
    }
    __device__ __forceinline__ static void undo(Z& z, const O&, int q) {
#pragma unroll
        for (int e = 0; e < E; ++e)
            for (int r = q - 1; r >= 0; --r)
                for (int j = r; j < q; ++j) at(z, j, e) = csub(at(z, j, e), at(z, j + 1, e));
    }
    __device__ __forceinline__ static void rescale(Z& z, const O&, int q, double ratio) {
        double f = 1.0;
        for (int j = 1; j <= q; ++j) {
            f *= ratio;
#pragma unroll
            for (int e = 0; e < E; ++e) at(z, j, e) = cscale(f, at(z, j, e));
        }
    }
    __device__ __forceinline__ static void commit(Z& z, const O&, int q, const double* l,
                                                  const double2 (&ev)[E]) {
        for (int j = 0; j <= q; ++j) {
            const double lj = l[j];
#pragma unroll
            for (int e = 0; e < E; ++e) at(z, j, e) = cadd(at(z, j, e), cscale(lj, ev[e]));
        }
    }
    __device__ __forceinline__ static double2 row(const Z& z, const O&, int j, int e) { return at(z, j, e); }
    __device__ __forceinline__ static void set_row(Z& z, const O&, int j, int e, double2 v) { at(z, j, e) = v; }
    __device__ __forceinline__ static void row_all(const Z& z, const O& o, int j, double2 (&out)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = at(z, j, e);
    }
    __device__ __forceinline__ static void set_row_all(Z& z, const O& o, int j, const double2 (&v)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) at(z, j, e) = v[e];
    }
    __device__ __forceinline__ static void horner_fast(const Z& z, const O& o, int q, double s, double2 (&out)[E]) {
        horner(z, o, q, s, out);
    }
    __device__ __forceinline__ static void horner(const Z& z, const O&, int q, double s, double2 (&out)[E]) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            double2 acc = at(z, q, e);
            for (int j = q - 1; j >= 0; --j) acc = cadd(cscale(s, acc), at(z, j, e));
            out[e] = acc;
        }
    }
};


// ------------------------------------------ history in TMEM (HistT, sm_100a)
// Row 1 (read by every corrector iteration) stays in registers, row 0 in the
// thread's private shared-memory slots (also read by every iteration, and
// the register file is what limits two CTAs per SM), rows 2..7 and the
// corrector terms e / e_prev live in the thread's private TMEM columns
// (qtm_tmem.cuh), rows >= 8 in the overflow column as in Hist<8>.
// Column layout of a thread's 32E columns (E = 4: 128):
//   [0, 4E)        e buffer slot 0, component e at 4e (lo x, hi x, lo y, hi y)
//   [4E, 8E)       e buffer slot 1
//   [8E + 24e, +24) rows 2..7 of component e
// Every history operation runs per component: the 6 TMEM rows of component
// e+1 are loaded while component e is processed with the register code of
// Hist<8, 1> (so the arithmetic, and its rounding, is exactly Hist<8>'s),
// then stored back.
template <int E, int DP>
struct HistT {
    static_assert(E == 4, "e-buffer slots are one x16 TMEM access (E = 4)");
    static constexpr int ROWS = 8;
    static constexpr int COLS = 32 * E;  // TMEM columns per thread
    using H1 = Hist<ROWS, 1, DP>;
    using O = typename Hist<ROWS, E, DP>::O;
    struct Z {
        double2 r1[E];  // row 1
        double2* z0;    // row 0: z0[(DP / E) * e] (this thread's shared-memory slots)
        uint32_t ta;    // this thread's column block (tm::thread_base)
    };
    __device__ __forceinline__ static double2& at(Z& z, int j, int e) {
        return j == 0 ? z.z0[(DP / E) * e] : z.r1[e];
    }
    __device__ __forceinline__ static const double2& at(const Z& z, int j, int e) {
        return j == 0 ? z.z0[(DP / E) * e] : z.r1[e];
    }
    __device__ __forceinline__ static uint32_t rows_col(const Z& z, int e) { return z.ta + 8u * E + 24u * e; }

    // Single-buffered: one component's 24 columns in flight at a time keeps
    // the register footprint small (the TMEM latency is hidden by the second
    // CTA on the SM, not by prefetching).
    // runtime-indexed access to a small register array without local memory
    __device__ __forceinline__ static double2 sel(const double2 (&a)[E], int e) {
        double2 v = a[0];
#pragma unroll
        for (int k = 1; k < E; ++k) if (e == k) v = a[k];
        return v;
    }
    __device__ __forceinline__ static void put(double2 (&a)[E], int e, double2 v) {
#pragma unroll
        for (int k = 0; k < E; ++k) if (e == k) a[k] = v;
    }
    // QTM_TM_UNROLL=0: the component loop is not unrolled, so its body (an
    // order switch over the register code of Hist<8, 1>) exists once -- a
    // smaller instruction footprint for more local-memory traffic (r1).
#ifndef QTM_TM_UNROLL
#define QTM_TM_UNROLL 1
#endif
    template <bool STORE, class F>
    __device__ __forceinline__ static void per_comp(Z& z, const O& ovf, F&& f) {
        tm::wait_st();
#if QTM_TM_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int e = 0; e < E; ++e) {
            uint32_t raw[24];
            tm::issue_ld24(rows_col(z, e), raw);
            tm::wait_ld24(raw);
            double2 t[6];
            tm::unpack<6>(raw, t);
            double2 zc[ROWS][1];
            zc[0][0] = z.z0[(DP / E) * e];
            zc[1][0] = sel(z.r1, e);
#pragma unroll
            for (int k = 0; k < 6; ++k) zc[2 + k][0] = t[k];
            const typename H1::O o1{ovf.p + e * (DP / E)};
            f(zc, o1, e);
            if constexpr (STORE) {
                z.z0[(DP / E) * e] = zc[0][0];
                put(z.r1, e, zc[1][0]);
#pragma unroll
                for (int k = 0; k < 6; ++k) t[k] = zc[2 + k][0];
                tm::pack<6>(t, raw);
                tm::st24(rows_col(z, e), raw);
            }
        }
    }
    // Order-specialised form for Q <= 7 (every row on chip): only the TMEM
    // rows 2..Q move, in one load of 4(Q-1) columns per component, and the
    // arithmetic is Hist<8, 1>'s straight-line code for order Q.
    // QTM_TM_DB=1: the rows of component e+1 are loaded while
    // component e is processed (two raw buffers, 4(Q-1) registers more), so
    // only the first component's TMEM latency is exposed.  Measured on c4:
    // 111.9 vs 109.2 ms per step -- the second CTA on the SM already hides
    // that latency, and the extra registers cost more: off by default.
#ifndef QTM_TM_DB
#define QTM_TM_DB 0
#endif
    template <int Q, bool STORE = true, class F>
    __device__ __forceinline__ static void per_comp_q(Z& z, F&& f) {
        constexpr int N = Q - 1;  // TMEM rows 2..Q
        constexpr int W = 4 * (N > 0 ? N : 1);
        if constexpr (N > 0) tm::wait_st();
#if QTM_TM_DB
        uint32_t rawa[W], rawb[W];
        if constexpr (N > 0) tm::issue_ld(rows_col(z, 0), rawa);
#endif
#pragma unroll
        for (int e = 0; e < E; ++e) {
            double2 zc[ROWS][1];
#if QTM_TM_DB
            uint32_t (&raw)[W] = (e & 1) ? rawb : rawa;
            uint32_t (&nxt)[W] = (e & 1) ? rawa : rawb;
#else
            uint32_t raw[W];
#endif
            if constexpr (N > 0) {
#if QTM_TM_DB
                tm::wait_ld(raw);
                if (e + 1 < E) tm::issue_ld(rows_col(z, e + 1), nxt);
#else
                tm::issue_ld(rows_col(z, e), raw);
                tm::wait_ld(raw);
#endif
                double2 t[N > 0 ? N : 1];
                tm::unpack<(N > 0 ? N : 1)>(raw, t);
#pragma unroll
                for (int k = 0; k < N; ++k) zc[2 + k][0] = t[k];
            }
            zc[0][0] = z.z0[(DP / E) * e];
            zc[1][0] = z.r1[e];
            f(zc, e);
            if constexpr (!STORE) continue;
            z.z0[(DP / E) * e] = zc[0][0];
            z.r1[e] = zc[1][0];
            if constexpr (N > 0) {
                double2 t[N];
#pragma unroll
                for (int k = 0; k < N; ++k) t[k] = zc[2 + k][0];
                tm::pack<N>(t, raw);
                tm::st(rows_col(z, e), raw);
            }
        }
    }
#define QTM_TM_QSWITCH(CALL)                                                 \
    switch (q) {                                                             \
        case 1: CALL(1); return;                                             \
        case 2: CALL(2); return;                                             \
        case 3: CALL(3); return;                                             \
        case 4: CALL(4); return;                                             \
        case 5: CALL(5); return;                                             \
        case 6: CALL(6); return;                                             \
        case 7: CALL(7); return;                                             \
        default: break;                                                      \
    }
    __device__ __forceinline__ static void predict(Z& z, const O& ovf, int q) {
#define CALL_(Q) per_comp_q<Q>(z, [&](double2 (&zc)[ROWS][1], int) { H1::template predict_q<Q>(zc); })
        QTM_TM_QSWITCH(CALL_)
#undef CALL_
        per_comp<true>(z, ovf, [&](double2 (&zc)[ROWS][1], const typename H1::O& o, int) {
            H1::predict(zc, o, q);
        });
    }
    __device__ __forceinline__ static void undo(Z& z, const O& ovf, int q) {
#define CALL_(Q) per_comp_q<Q>(z, [&](double2 (&zc)[ROWS][1], int) { H1::template undo_q<Q>(zc); })
        QTM_TM_QSWITCH(CALL_)
#undef CALL_
        per_comp<true>(z, ovf, [&](double2 (&zc)[ROWS][1], const typename H1::O& o, int) {
            H1::undo(zc, o, q);
        });
    }
    __device__ __forceinline__ static void rescale(Z& z, const O& ovf, int q, double ratio) {
        per_comp<true>(z, ovf, [&](double2 (&zc)[ROWS][1], const typename H1::O& o, int) {
            H1::rescale(zc, o, q, ratio);
        });
    }
    // commit, then post(e, z0) with component e's committed row 0 (the error
    // weights are computed there, while the component is in registers)
    template <class Post>
    __device__ __forceinline__ static void commit(Z& z, const O& ovf, int q, const double* l,
                                                  const double2 (&ev)[E], Post&& post) {
#define CALL_(Q)                                                                        \
        per_comp_q<Q>(z, [&](double2 (&zc)[ROWS][1], int e) {                           \
            const double2 ev1[1] = {sel(ev, e)};                                        \
            H1::template commit_q<Q>(zc, l, ev1);                                       \
            post(e, zc[0][0]);                                                          \
        })
        QTM_TM_QSWITCH(CALL_)
#undef CALL_
        per_comp<true>(z, ovf, [&](double2 (&zc)[ROWS][1], const typename H1::O& o, int e) {
            const double2 ev1[1] = {sel(ev, e)};
            H1::commit(zc, o, q, l, ev1);
            post(e, zc[0][0]);
        });
    }
    __device__ __forceinline__ static void commit(Z& z, const O& ovf, int q, const double* l,
                                                  const double2 (&ev)[E]) {
#define CALL_(Q)                                                                        \
        per_comp_q<Q>(z, [&](double2 (&zc)[ROWS][1], int e) {                           \
            const double2 ev1[1] = {sel(ev, e)};                                        \
            H1::template commit_q<Q>(zc, l, ev1);                                       \
        })
        QTM_TM_QSWITCH(CALL_)
#undef CALL_
        per_comp<true>(z, ovf, [&](double2 (&zc)[ROWS][1], const typename H1::O& o, int e) {
            const double2 ev1[1] = {sel(ev, e)};
            H1::commit(zc, o, q, l, ev1);
        });
    }
    // the per-step grid recording's Horner (the one hot call site): with every
    // row on chip (q <= 7) only rows 2..q are loaded, straight-line code
    __device__ __forceinline__ static void horner_fast(Z& z, const O& ovf, int q, double s, double2 (&out)[E]) {
#define CALL_(Q)                                                                        \
        per_comp_q<Q, false>(z, [&](double2 (&zc)[ROWS][1], int e) {                    \
            double2 o1[1];                                                              \
            H1::template horner_q<Q>(zc, s, o1);                                        \
            out[e] = o1[0];                                                             \
        })
        QTM_TM_QSWITCH(CALL_)
#undef CALL_
        horner(z, ovf, q, s, out);
    }
    __device__ __forceinline__ static void horner(Z& z, const O& ovf, int q, double s, double2 (&out)[E]) {
        per_comp<false>(z, ovf, [&](double2 (&zc)[ROWS][1], const typename H1::O& o, int e) {
            double2 o1[1];
            H1::horner(zc, o, q, s, o1);
            put(out, e, o1[0]);
        });
    }
    __device__ __forceinline__ static void row_all(const Z& z, const O& ovf, int j, double2 (&out)[E]) {
        if (j < 2) {
#pragma unroll
            for (int e = 0; e < E; ++e) out[e] = at(z, j, e);
        } else if (j < ROWS) {
            tm::wait_st();
            uint32_t r[4 * E];
#pragma unroll
            for (int e = 0; e < E; ++e)
                tm::issue_ld4(rows_col(z, e) + 4u * (j - 2), r[4 * e], r[4 * e + 1], r[4 * e + 2], r[4 * e + 3]);
            tm::wait_ld16(r);
            tm::unpack<E>(r, out);
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) out[e] = ovf.at(j, e);
        }
    }
    __device__ __forceinline__ static void set_row_all(Z& z, const O& ovf, int j, const double2 (&v)[E]) {
        if (j < 2) {
#pragma unroll
            for (int e = 0; e < E; ++e) at(z, j, e) = v[e];
        } else if (j < ROWS) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                uint32_t r[4];
                const double2 one[1] = {v[e]};
                tm::pack<1>(one, r);
                tm::st4(rows_col(z, e) + 4u * (j - 2), r);
            }
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) ovf.at(j, e) = v[e];
        }
    }
    // e / e_prev buffer slots
    __device__ __forceinline__ static void eb_store(const Z& z, int slot, const double2 (&v)[E]) {
        uint32_t r[16];
        tm::pack<E>(v, r);
        tm::st16(z.ta + 4u * E * slot, r);
    }
    __device__ __forceinline__ static void eb_load(const Z& z, int slot, double2 (&v)[E]) {
        tm::wait_st();
        uint32_t r[16];
        tm::issue_ld16(z.ta + 4u * E * slot, r);
        tm::wait_ld16(r);
        tm::unpack<E>(r, v);
    }
    __device__ __forceinline__ static void eb_load2(const Z& z, int slot, double2 (&a)[E], double2 (&b)[E]) {
        tm::wait_st();
        uint32_t ra[16], rb[16];
        tm::issue_ld16(z.ta + 4u * E * slot, ra);
        tm::issue_ld16(z.ta + 4u * E * (slot ^ 1), rb);
        tm::wait_ld16(ra);
        tm::wait_ld16(rb);
        tm::unpack<E>(ra, a);
        tm::unpack<E>(rb, b);
    }
};

// ------------------------------------------------------------- the kernel
template <int NT, int E, int RREG, bool TM = false>
struct TrajKernel {
    static constexpr int DP = NT * E;  // padded state length
    static constexpr int NW = NT / 32;
    // gather buffers [2][DP] and (not with TM: those live in TMEM) the e
    // buffers [2][DP], plus RREG == 0's Nordsieck rows
    static constexpr int VEC_BUFS = (TM ? 3 : 4) + (RREG == 0 ? LROWS : 0);  // TM: + row 0

    // fixed part of the dynamic shared memory; the staged operator follows
    __host__ __device__ static constexpr size_t smem_bytes() {
        return sizeof(double2) * (size_t)DP * VEC_BUFS +
               sizeof(double) * 2 * KRED * (NW > 1 ? NW : 1) + sizeof(double) * (size_t)DP;
    }
    // TMEM columns one CTA allocates (a power of two >= 32)
    __host__ __device__ static constexpr uint32_t tmem_cols() { return TM ? (uint32_t)(NW / 4) * 32u * E : 0u; }
};

// Row access: rows < RREG are register arrays indexed by compile-time j
// (every loop over j is fully unrolled), rows >= RREG live in the CTA's
// overflow scratch.
#define STAT(which, amount) do { if (tid == 0) s_stats[which] += (amount); } while (0)
// Phase timing (profiling builds with -DQTM_PHASES): thread 0 attributes
// clock64() deltas to the phases of the attempt loop.
#ifdef QTM_PHASES
#define PH_MARK(k)                                                           \
    do {                                                                     \
        if (tid == 0) {                                                      \
            const long long now__ = clock64();                               \
            ph_acc[k] += now__ - ph_last;                                    \
            ph_last = now__;                                                 \
        }                                                                    \
    } while (0)
#else
#define PH_MARK(k) do { } while (0)
#endif

// TD: variant compiled with the time-dependent generator terms (td_apply
// calls cost registers even when not taken, so constant-generator variants
// are built without them)
// Register cap of the TMEM variants: 128 (what __launch_bounds__(256, 2)
// allows; two CTAs per SM do co-reside -- the runtime's occupancy calculator
// claims otherwise for tcgen05 kernels, see variant_occupancy in
// qtm_capi.cu).  Measured on c4: 112 -> 29.2k, 120 -> 33.0k, 128 -> 35.4k
// trajectories/s.
#ifndef QTM_TM_MAXNREG
#define QTM_TM_MAXNREG 128
#endif
#define QTM_MAXNREG(NT, MINB, TM) __maxnreg__((TM) ? QTM_TM_MAXNREG : 65536 / ((NT) * (MINB)) > 255 ? 255 : 65536 / ((NT) * (MINB)))
// TM: Nordsieck rows 2..7 and the e buffers in TMEM (HistT; RREG must be 8,
// the rows held on chip)
template <int NT, int E, int RREG, int MINB, bool TD, bool TM = false>
__global__ void __launch_bounds__(NT, MINB) QTM_MAXNREG(NT, MINB, TM)
traj_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ RunParams R) {
    constexpr int DP = NT * E;
    static_assert(!TM || (RREG == 8 && NT % 128 == 0), "TMEM history: 8 rows on chip, whole lane quarters");
    using H = std::conditional_t<TM, HistT<E, DP>,
                                 std::conditional_t<RREG == 0, HistS<E, DP>, Hist<(RREG > 0 ? RREG : 2), E, DP>>>;
    extern __shared__ double2 smem[];
    // gath[2][DP]: double-buffered gather buffers; gath[gbuf] is the most
    //              recently published vector (the corrector iterate lives here)
    // ebuf[2][DP]: corrector term e of the current attempt / of the previous
    //              accepted step (e_prev); "e_prev = e.copy()" is a flip
    //              (TM: in TMEM, HistT::eb_*)
    double2* const gath = smem;
    double2* const ebuf = smem + 2 * DP;
    // TM: row 0 of the Nordsieck history at smem + 2 DP (HistT)
    double* const red = reinterpret_cast<double*>(smem + (TM ? 3 : 4) * DP);
    // wsm[DP]: error weights 1/(atol + rtol |z0_i|), thread-private slots
    // (read once per corrector iteration; kept out of the register file)
    double* const wsm = red + 2 * KRED * (NT / 32 > 1 ? NT / 32 : 1);
    // RREG == 0: the Nordsieck rows follow the weights
    double2* const zrows = reinterpret_cast<double2*>(wsm + DP);
    __shared__ long long s_row;
    __shared__ long long s_stats[NSTATS];
    __shared__ Stream s_stream;
    __shared__ double s_draw;
    // Per-warp copies of the controller state that is not needed inside the
    // corrector iteration (every lane holds the same value; a warp only ever
    // touches its own copy, so no barrier is involved).  Keeping them out of
    // the register file leaves the registers to the Nordsieck history.
    struct WarpCold {
        double t_lo, r_thr, crate;
        double t_next;  // P.times[gi] (+inf once every grid point is recorded)
        long long row, steps_in_segment, njumps;
        int gi, nef, ncf;
        unsigned c_att, c_q, c_qq, c_it, c_steps;
    };
    __shared__ WarpCold s_cold[NT / 32];
    WarpCold& ws = s_cold[threadIdx.x >> 5];

    const int tid = threadIdx.x;
    const int d = P.d;
    const int npts = P.n_pts;
    // component e of this thread is state index II(e); ACT(e): inside the state
#define II(e) (tid + NT * (e))
#define ACT(e) (II(e) < d)
    // overflow column of this thread (rows >= RREG), rebuilt where used so it
    // holds no register across the hot loop
#define OVF() (typename H::O{R.zovf + (size_t)blockIdx.x * (RREG > 0 ? LROWS - RREG : 0) * DP + tid})

    // ---- stage G (sliced ELL + value dictionary) in shared memory once
    double2* const s_dict = reinterpret_cast<double2*>(reinterpret_cast<char*>(smem) +
                                                       TrajKernel<NT, E, RREG, TM>::smem_bytes());
    // ---- TMEM for the history (TM): allocated once per persistent CTA
    __shared__ uint32_t s_taddr;
    if constexpr (TM) {
        if ((threadIdx.x >> 5) == 0) tm::alloc(&s_taddr, TrajKernel<NT, E, RREG, TM>::tmem_cols());
        tm::fence_before_sync();
        __syncthreads();
        tm::fence_after_sync();
    }
    uint32_t* const s_ent = reinterpret_cast<uint32_t*>(s_dict + P.sell_dict_n);
    double2* const s_tdict = reinterpret_cast<double2*>(s_ent + P.sell_entries);
    uint16_t* const s_tent = reinterpret_cast<uint16_t*>(s_tdict + P.sell_td_dict_n);
    // ---- stage the diagonal observables' index + dictionary tables
    const uint8_t* const s_eidx = reinterpret_cast<const uint8_t*>(smem) + P.e_stage_off;
    const double* const s_edict = reinterpret_cast<const double*>(s_eidx + P.e_stage_idx_bytes);
    if (P.e_stage_dense) {
        double* const dd = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + P.e_stage_off);
        for (int i = tid; i < P.ne * DP; i += NT) dd[i] = P.e_dense_g[i];
    } else if (P.e_stage_mask) {
        uint8_t* const di = reinterpret_cast<uint8_t*>(smem) + P.e_stage_off;
        double* const dd = reinterpret_cast<double*>(di + P.e_stage_idx_bytes);
        const uint32_t* const si = reinterpret_cast<const uint32_t*>(P.e_idx_g);
        for (int i = tid; i < P.e_stage_idx_bytes / 4; i += NT) reinterpret_cast<uint32_t*>(di)[i] = si[i];
        for (int i = tid; i < P.e_dict_n; i += NT) dd[i] = P.e_dict_g[i];
    }
    int goff = 0, gwidth = 0;
    if (P.sell_mode) {
        for (int i = tid; i < P.sell_dict_n; i += NT) s_dict[i] = P.sell_dict[i];
        for (int i = tid; i < P.sell_entries; i += NT) s_ent[i] = P.sell_ent[i];
        if (TD && P.sell_td > 0) {
            for (int i = tid; i < P.sell_td_dict_n; i += NT) s_tdict[i] = P.sell_td_dict[i];
            for (int i = tid; i < P.sell_td * P.sell_entries; i += NT) s_tent[i] = P.sell_td_ent[i];
        }
        const int warp = tid >> 5;
        goff = P.sell_off[warp];
        gwidth = P.sell_w[warp];
        __syncthreads();
    }
// f[E] = G(t) x (x gathered in shared memory): constant part, then the
// time-dependent terms at time tt (ode.py: rhs(t_new, y) in the corrector,
// rhs(t, y) at cold start / restart)
#define GSPMV_T(xs, f, tt)                                                   \
    do {                                                                     \
        if constexpr (TD) {                                                  \
            if (P.sell_td == 1 || P.sell_td == -1) {                         \
                double2 g__[E];                                              \
                if (P.sell_td < 0)                                           \
                    sell_spmv_tdd<NT, E>(s_ent, s_dict, goff, gwidth, (xs), f, g__, P.sell_dom, \
                                         make_double2(P.sell_td_dom[0], P.sell_td_dom[1])); \
                else                                                         \
                    sell_spmv_td<NT, E>(s_ent, s_dict, s_tent, s_tdict, goff, gwidth, (xs), f, g__); \
                const double c__ = td_coef(P, 0, (tt));                      \
                _Pragma("unroll") for (int e = 0; e < E; ++e)                \
                    f[e] = make_double2(f[e].x + c__ * g__[e].x, f[e].y + c__ * g__[e].y); \
                break;                                                       \
            }                                                                \
            if (P.sell_td > 1) {                                             \
                GSPMV(xs, f);                                                \
                for (int k__ = 0; k__ < P.sell_td; ++k__) {                  \
                    double2 g__[E];                                          \
                    sell_spmv_term<NT, E>(s_ent, s_tent + k__ * P.sell_entries, s_tdict, goff, \
                                          gwidth, (xs), g__);                \
                    const double c__ = td_coef(P, k__, (tt));                \
                    _Pragma("unroll") for (int e = 0; e < E; ++e)            \
                        f[e] = make_double2(f[e].x + c__ * g__[e].x, f[e].y + c__ * g__[e].y); \
                }                                                            \
                break;                                                       \
            }                                                                \
        }                                                                    \
        GSPMV(xs, f);                                                        \
        if constexpr (TD) {                                                  \
            for (int k__ = 0; k__ < P.n_td; ++k__) {                         \
                const double c__ = td_coef(P, k__, (tt));                    \
                _Pragma("unroll") for (int e = 0; e < E; ++e)                \
                    if (ACT(e)) f[e] = td_term(P.td[k__], c__, II(e), (xs), f[e]); \
            }                                                                \
        }                                                                    \
    } while (0)
// f[E] = G x (x gathered in shared memory)
#define GSPMV(xs, f)                                                         \
    do {                                                                     \
        if (P.sell_mode) {                                                   \
            sell_spmv<NT, E, QTM_SPMV_PF(RREG), sell_uses_tex(NT, E, RREG, TD), sell_uses_dom(NT, E, RREG, TD)>( \
                s_ent, s_dict, goff, gwidth, (xs), f, P.sell_tex, P.sell_dom_on, P.sell_dom); \
        } else {                                                             \
            _Pragma("unroll") for (int e = 0; e < E; ++e)                    \
                f[e] = ACT(e) ? row_dot(P.g, II(e), (xs)) : make_double2(0.0, 0.0); \
        }                                                                    \
    } while (0)

    int gbuf = 0, rphase = 0, ecur = 0;

    for (;;) {
        if (tid == 0) s_row = next_row(R);
        __syncthreads();
        ws.row = s_row;
        if (ws.row >= R.n_traj) break;
        if (tid < NSTATS) s_stats[tid] = 0;
        if (tid == 0)
            s_stream.init(R.stream_kind, R.seed, (uint64_t)(R.traj_begin + ws.row),
                          R.script ? R.script + ws.row * R.script_stride : nullptr,
                          R.script_len ? R.script_len[ws.row] : 0, R.script_fallback);
        __syncthreads();

        ws.njumps = 0;
        int rc = kOk;
        // hot per-attempt counters live in registers (folded into s_stats at
        // the end of the trajectory); rare events go straight to s_stats
        ws.c_att = 0; ws.c_q = 0; ws.c_qq = 0; ws.c_it = 0; ws.c_steps = 0;
#ifdef QTM_PHASES
        long long ph_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        long long ph_last = clock64();
#endif

        typename H::Z z;  // Nordsieck history: registers (rows < RREG), shared memory (RREG == 0) or TMEM (TM)
        if constexpr (TM) {
            z.ta = tm::thread_base(s_taddr, H::COLS);
            z.z0 = smem + 2 * DP + tid;
        }
        else if constexpr (RREG == 0) z.p = zrows;
#define W(e) wsm[II(e)]
        double t, h;
        int q, ialth;
        bool has_eprev;

// publish x[E] as the next gather buffer (write, barrier); yields `xs`
#define GATHER(xsrc, xs)                                                     \
    double2* const xs = gath + (gbuf ^ 1) * DP;                              \
    _Pragma("unroll") for (int e = 0; e < E; ++e) if (ACT(e)) xs[II(e)] = (xsrc)[e]; \
    __syncthreads();                                                         \
    gbuf ^= 1;

// Horner evaluation of the history polynomial at s into out[E]
#define HORNER(s_, out) H::horner(z, OVF(), q, (s_), out)

// z[j] *= ratio^j for j = 1..q, h *= ratio (nordsieck_rescale + _rescale)
#define RESCALE(ratio_)                                                      \
    do {                                                                     \
        const double rr__ = (ratio_);                                        \
        H::rescale(z, OVF(), q, rr__);                                         \
        h *= rr__;                                                           \
        has_eprev = false;                                                   \
        ialth = q + 1;                                                       \
    } while (0)

#define FAIL4(code_, a_, b_, c_, d_)                                         \
    do {                                                                     \
        rc = (code_);                                                        \
        if (tid == 0) {                                                      \
            double* eo__ = R.err + (size_t)ws.row * 4;                          \
            eo__[0] = (a_); eo__[1] = (b_); eo__[2] = (c_); eo__[3] = (d_);  \
        }                                                                    \
        goto traj_done;                                                      \
    } while (0)
#define FAIL(code_) FAIL4(code_, t, h, 0.0, 0.0)

// one uniform draw, evaluated by thread 0 and broadcast
#define DRAW(var)                                                            \
    do {                                                                     \
        __syncthreads();                                                     \
        if (tid == 0) s_draw = s_stream.next();                              \
        __syncthreads();                                                     \
        var = s_draw;                                                        \
    } while (0)

        // ---- record(ws.gi) of the state in `psi` (trajectory.py:122-130, 206-214).
        // The reduction over the state is deferred: every warp stores its
        // partial <psi|E_k|psi> and <psi|psi> sums, and finalize_records
        // (qtm_capi.cu) adds the warps in a fixed order and divides.  No
        // barrier here unless an observable is off-diagonal (then psi is
        // gathered for the ws.row products).
#define RECORD(psi, gi_)                                                     \
    do {                                                                     \
        if (R.psi_slot) {                                                    \
            const int sl__ = R.psi_slot[(gi_)];                              \
            if (sl__ >= 0) {                                                 \
                double2* const po__ = R.psi_out + ((size_t)ws.row * R.n_psi + sl__) * d; \
                _Pragma("unroll") for (int e = 0; e < E; ++e) if (ACT(e)) po__[II(e)] = (psi)[e]; \
            }                                                                \
        }                                                                    \
        const double2* xs__ = gath;                                          \
        if (P.e_need_gather) {                                               \
            GATHER(psi, xg__);                                               \
            xs__ = xg__;                                                     \
        }                                                                    \
        double* const rp__ = R.rec_partial +                                 \
            ((size_t)ws.row * npts + (gi_)) * (size_t)(P.ne + 1) * (NT / 32) + (tid >> 5); \
        if (RREG > 0 && P.e_fast) { /* (RREG = 0: compact code wins) */     \
            double pw__[E];                                                  \
            _Pragma("unroll") for (int e = 0; e < E; ++e) pw__[e] = ACT(e) ? cabs2(psi[e]) : 0.0; \
            if (P.e_stage_dense)                                             \
                record_staged<NT, E, true>(P, smem, pw__, rp__);             \
            else                                                             \
                record_staged<NT, E, false>(P, smem, pw__, rp__);            \
            break;                                                           \
        }                                                                    \
        double nrm__ = 0.0;                                                  \
        _Pragma("unroll") for (int e = 0; e < E; ++e) if (ACT(e)) nrm__ += cabs2(psi[e]); \
        for (int k0 = 0; k0 <= P.ne; k0 += KRED) {                           \
            double v__[KRED];                                                \
            _Pragma("unroll") for (int kk = 0; kk < KRED; ++kk) {            \
                const int k = k0 + kk;                                       \
                double acc__ = 0.0;                                          \
                if (k < P.ne && ((P.e_stage_mask >> k) & 1u)) {             \
                    /* staged real diagonal: sum_i E_ii |psi_i|^2 */         \
                    const double* const dk__ = s_edict + P.e_dict_off[k];    \
                    const double* const dd__ = reinterpret_cast<const double*>(s_eidx); \
                    _Pragma("unroll") for (int e = 0; e < E; ++e) if (ACT(e)) \
                        acc__ += (P.e_stage_dense ? dd__[k * DP + II(e)]        \
                                                  : dk__[s_eidx[k * DP + II(e)]]) * cabs2(psi[e]); \
                } else if (k < P.ne) {                                       \
                    const bool dg__ = (P.e_diag_mask >> k) & 1u;             \
                    _Pragma("unroll") for (int e = 0; e < E; ++e) if (ACT(e)) { \
                        double2 s;                                           \
                        if (dg__) {                                          \
                            const double2 ev__ = P.e_diag[(size_t)k * DP + II(e)]; \
                            s = make_double2(0.0 + (ev__.x * psi[e].x - ev__.y * psi[e].y), \
                                             0.0 + (ev__.x * psi[e].y + ev__.y * psi[e].x)); \
                        } else {                                             \
                            s = row_dot(P.e[k], II(e), xs__);                \
                        }                                                    \
                        acc__ += psi[e].x * s.x - (-psi[e].y) * s.y;         \
                    }                                                        \
                } else if (k == P.ne) {                                      \
                    acc__ = nrm__;                                           \
                }                                                            \
                v__[kk] = acc__;                                             \
            }                                                                \
            warp_sum_lane0<KRED>(v__);                                       \
            if ((tid & 31) == 0) {                                           \
                _Pragma("unroll") for (int kk = 0; kk < KRED; ++kk)          \
                    if (k0 + kk <= P.ne) rp__[(size_t)(k0 + kk) * (NT / 32)] = v__[kk]; \
            }                                                                \
        }                                                                    \
    } while (0)

        // ---- cold start of the solver at (t0, y0[E]) with step h0 (ode.py:164-217)
#define COLD_START(t0_, y0, h0_)                                             \
    do {                                                                     \
        t = (t0_); ws.t_lo = t; q = 1; h = (h0_);                               \
        GATHER(y0, xs__);                                                    \
        STAT(sNfe, 1);                                                       \
        double2 f__[E];                                                      \
        GSPMV_T(xs__, f__, t);                                               \
        _Pragma("unroll") for (int e = 0; e < E; ++e) {                      \
            H::at(z, 0, e) = (y0)[e];                                        \
            H::at(z, 1, e) = cscale(h, f__[e]);                              \
            W(e) = ACT(e) ? err_weight(P.atol, P.rtol, (y0)[e]) : 0.0; \
        }                                                                    \
        ws.crate = 0.7; ialth = 2; has_eprev = false;                        \
    } while (0)

        t = P.t_from;
        h = P.h0_first;
        {
            double2 psi[E];
#pragma unroll
            for (int e = 0; e < E; ++e) psi[e] = ACT(e) ? P.psi0[II(e)] : make_double2(0.0, 0.0);
            RECORD(psi, 0);  // record(0) from psi0
            DRAW(ws.r_thr);
            COLD_START(P.t_from, psi, P.h0_first);
            ws.gi = 1;
            ws.t_next = npts > 1 ? P.times[1] : CUDART_INF;
            ws.steps_in_segment = 0;

            while (ws.gi < npts) {
                // ================= OdeSolver.step() (ode.py:261-312) =================
                ws.nef = 0; ws.ncf = 0;
                double est = 0.0, nrm2 = 0.0;
                for (;;) {
                    PH_MARK(0);  // [0] step-level work since the last mark
                    if (t + h == t) FAIL(kErrStepCollapse);
                    ws.c_att++;
                    ws.c_q += q;
                    ws.c_qq += q * (q + 1);
                    if (q + 1 > RREG) STAT(sOverflow, 1);
                    // predict: in-place Pascal triangle (_kernels.py:133-137)
                    H::predict(z, OVF(), q);
                    // functional corrector (_kernels.py:139-174).  The iterate
                    // lives in the gather buffers: iteration m reads gath[gbuf]
                    // and writes its update into gath[gbuf^1], which the
                    // reduction barrier then publishes for iteration m+1.
                    const double l0 = P.l[q][0];
                    const double conit = P.conit[q];
                    bool converged = false;
                    double delp = 0.0, del = 0.0, acc_e = 0.0;
                    {
                        double2 y0p[E];
#pragma unroll
                        for (int e = 0; e < E; ++e) y0p[e] = H::at(z, 0, e);
                        PH_MARK(1);  // [1] predict
                        GATHER(y0p, xs0);
                        PH_MARK(2);  // [2] gather z0 + barrier
                    }
                    double2* const ecurp = ebuf + ecur * DP;

                    for (int m = 0; m < 3; ++m) {
                        const double2* const cur = gath + gbuf * DP;
                        double2* const nxt = gath + (gbuf ^ 1) * DP;
                        ws.c_it++;
                        double v[3] = {0.0, 0.0, 0.0};
                        double2 fg[E];
                        double2 etm[E];  // TM: this iteration's e, stored to TMEM below
                        GSPMV_T(cur, fg, t + h);
                        PH_MARK(3);  // [3] SpMV
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            if (ACT(e)) {
                                const double2 f = fg[e];
                                const double2 z1 = H::at(z, 1, e), z0 = H::at(z, 0, e);
                                const double2 ei = csub(cscale(h, f), z1);
                                const double2 yn = cadd(z0, cscale(l0, ei));
                                const double2 dd = csub(yn, cur[II(e)]);
                                const double we = W(e);
                                v[0] += cabs2(dd) * we * we;
                                v[1] += cabs2(ei) * we * we;
                                v[2] += cabs2(yn);
                                nxt[II(e)] = yn;
                                if constexpr (TM) etm[e] = ei;
                                else ecurp[II(e)] = ei;
                            } else if constexpr (TM) {
                                etm[e] = make_double2(0.0, 0.0);
                            }
                        }
                        // TM: e goes to TMEM right away (an asynchronous store),
                        // so it holds no registers across the next SpMV
                        if constexpr (TM) H::eb_store(z, ecur, etm);
                        PH_MARK(4);  // [4] corrector update
                        block_sum<NT, 3>(v, red, rphase);
                        if constexpr (NT == 32) __syncwarp();
                        PH_MARK(5);  // [5] reduction
                        gbuf ^= 1;
                        del = sqrt(v[0] * P.inv_d);
                        acc_e = v[1];
                        nrm2 = v[2];
                        if (m > 0) {
                            const double a = 0.2 * ws.crate, b = del / delp;
                            ws.crate = b > a ? b : a;
                        }
                        const double c15 = 1.5 * ws.crate;
                        if (del * (c15 < 1.0 ? c15 : 1.0) <= conit) { converged = true; break; }
                        if (m > 0 && del > 2.0 * delp) break;
                        delp = del;
                        PH_MARK(6);  // [6] convergence control
                    }
                    PH_MARK(6);
                    if (converged) {
                        est = sqrt(acc_e * P.inv_d) * P.inv_tau2[q];
                        if (!(est > 1.0)) {
                            // commit zp[j] += l_j e (_kernels.py:187-191)
                            double2 evr[E];
                            if constexpr (TM) {
                                H::eb_load(z, ecur, evr);
                            } else {
#pragma unroll
                                for (int e = 0; e < E; ++e) evr[e] = ACT(e) ? ecurp[II(e)] : make_double2(0.0, 0.0);
                            }
                            if constexpr (TM) {
                                // the error weights of the accepted state from each
                                // committed z0 component inside the TMEM pass
                                H::commit(z, OVF(), q, P.l[q], evr, [&](int e, double2 z0n) {
                                    W(e) = ACT(e) ? err_weight(P.atol, P.rtol, z0n) : 0.0;
                                });
                            } else {
                                H::commit(z, OVF(), q, P.l[q], evr);
                            }
                            break;  // accepted
                        }
                    }
                    // rejected attempt: restore the un-predicted history
                    H::undo(z, OVF(), q);
                    if (!converged) {
                        STAT(sCorrFail, 1);
                        if (++ws.ncf >= 10) FAIL(kErrCorrector);
                        RESCALE(0.25);
                        continue;
                    }
                    STAT(sErrReject, 1);
                    if (++ws.nef >= 10) FAIL(kErrRepeatedErrTest);
                    if (ws.nef >= 3) {
                        // _restart_order_one(0.1), ode.py:314-323
                        q = 1;
                        h *= 0.1;
                        double2 y0c[E];
#pragma unroll
                        for (int e = 0; e < E; ++e) y0c[e] = H::at(z, 0, e);
                        GATHER(y0c, xs);
                        STAT(sNfe, 1);
                        double2 fr[E];
                        GSPMV_T(xs, fr, t);
#pragma unroll
                        for (int e = 0; e < E; ++e) H::at(z, 1, e) = cscale(h, fr[e]);
                        has_eprev = false;
                        ialth = q + 1;
                    } else {
                        const double rr = __drcp_rn(1.2 * ctl_pow(est, P.rq1[q]) + 1e-6);
                        const double m1 = 0.9 < rr ? 0.9 : rr;
                        RESCALE(m1 > 0.1 ? m1 : 0.1);
                    }
                }
                PH_MARK(7);  // [7] error test + commit / undo + reject handling
                // accepted step bookkeeping (ode.py:281-292)
                ws.t_lo = t;
                t += h;
                ws.c_steps++;
                if constexpr (!TM) {  // (TM: computed in the commit pass)
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const double2 z0 = H::at(z, 0, e);
                        W(e) = ACT(e) ? err_weight(P.atol, P.rtol, z0) : 0.0;
                    }
                }
                PH_MARK(11);  // [11] accepted-step bookkeeping + error weights
                ialth -= 1;
                if (ialth == 0) {
                    // _order_step_control (ode.py:441-466)
                    const bool need_d = q > 1;
                    const bool need_u = q < P.max_order && has_eprev;
                    double v[2] = {0.0, 0.0};
                    {
                        double2 zq[E], ec[E], ep[E];
                        H::row_all(z, OVF(), q, zq);
                        if constexpr (TM) {
                            H::eb_load2(z, ecur, ec, ep);
                        } else {
#pragma unroll
                            for (int e = 0; e < E; ++e) {
                                ec[e] = ACT(e) ? ebuf[ecur * DP + II(e)] : make_double2(0.0, 0.0);
                                ep[e] = ACT(e) ? ebuf[(ecur ^ 1) * DP + II(e)] : make_double2(0.0, 0.0);
                            }
                        }
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            if (ACT(e)) {
                                const double2 de = csub(ec[e], ep[e]);
                                const double we = W(e);
                                v[0] += cabs2(zq[e]) * we * we;
                                v[1] += cabs2(de) * we * we;
                            }
                        }
                    }
                    block_sum<NT, 2>(v, red, rphase);
                    const double est_d = sqrt(v[0] * P.inv_d) * P.inv_tau1[q];
                    const double est_u = sqrt(v[1] * P.inv_d) * P.inv_tau3[q];
                    // every candidate ratio below 1.1 <=> every estimate above
                    // its host-tabulated threshold (r = 1/(c est^(1/k) + 1e-6)
                    // is decreasing in est): keep order and step without
                    // evaluating the three powers -- the common outcome
                    if (est > P.keep_same[q] && (!need_d || est_d > P.keep_down[q]) &&
                        (!need_u || est_u > P.keep_up[q])) {
                        ialth = 3;
                        ecur ^= 1;  // e_prev = e
                        has_eprev = true;
                        goto order_done;
                    }
                    {
                    const double r_same = __drcp_rn(1.2 * ctl_pow(est, P.rq1[q]) + 1e-6);
                    const double pd = __drcp_rn(1.3 * ctl_pow(est_d, P.rq0[q]) + 1e-6);
                    const double pu = __drcp_rn(1.4 * ctl_pow(est_u, P.rq2[q]) + 1e-6);
                    const double r_down = need_d ? pd : 0.0;
                    const double r_up = need_u ? pu : 0.0;
                    double best = r_same;
                    if (r_down > best) best = r_down;
                    if (r_up > best) best = r_up;
                    if (best < 1.1) {
                        ialth = 3;
                        ecur ^= 1;  // e_prev = e
                        has_eprev = true;
                    } else {
                        if (best == r_up) {
                            const double cu = P.l[q][q] / (q + 1);
                            double2 ec[E];
                            if constexpr (TM) {
                                H::eb_load(z, ecur, ec);
                            } else {
#pragma unroll
                                for (int e = 0; e < E; ++e) ec[e] = ACT(e) ? ebuf[ecur * DP + II(e)] : make_double2(0.0, 0.0);
                            }
#pragma unroll
                            for (int e = 0; e < E; ++e) ec[e] = ACT(e) ? cscale(cu, ec[e]) : make_double2(0.0, 0.0);
                            H::set_row_all(z, OVF(), q + 1, ec);
                            q = q + 1;
                            STAT(sOrderUp, 1);
                        } else if (best == r_down) {
                            q = q - 1;
                            STAT(sOrderDown, 1);
                        }
                        const double m1 = 10.0 < best ? 10.0 : best;
                        RESCALE(m1 > 0.1 ? m1 : 0.1);
                    }
                    }
                order_done:;
                } else {
                    ecur ^= 1;  // e_prev = e
                    has_eprev = true;
                }
                PH_MARK(8);  // [8] weights + order/step control
                // ================= trajectory loop body (trajectory.py:225-246) =======
                ws.steps_in_segment += 1;
                if (ws.steps_in_segment > P.max_steps) FAIL(kErrMaxSteps);
                if (P.nc > 0 && nrm2 < ws.r_thr) {
                    // locate_jump_time (trajectory.py:157-182)
                    double v2[2] = {0.0, 0.0};
                    {
                        double2 a1[E], a2[E];
                        HORNER((ws.t_lo - t) / h, a1);
                        HORNER((t - t) / h, a2);
#pragma unroll
                        for (int e = 0; e < E; ++e) if (ACT(e)) { v2[0] += cabs2(a1[e]); v2[1] += cabs2(a2[e]); }
                    }
                    block_sum<NT, 2>(v2, red, rphase);
                    const double f_lo = v2[0], f_hi = v2[1];
                    const double tol = 1e-9 * ws.r_thr;
                    if (f_lo < ws.r_thr - tol || f_hi > ws.r_thr + tol) {
                        if (tid == 0) R.err_r[ws.row] = ws.r_thr;
                        FAIL4(kErrBracket, ws.t_lo, t, f_lo, f_hi);
                    }
                    double ts;
                    if (f_lo <= ws.r_thr + tol) {
                        ts = ws.t_lo;
                    } else {
                        double a = ws.t_lo, b = t;
                        bool found = false;
                        ts = 0.0;
                        for (int it = 0; it < 60; ++it) {
                            const double mid = 0.5 * (a + b);
                            double v1[1] = {0.0};
                            {
                                double2 am[E];
                                HORNER((mid - t) / h, am);
#pragma unroll
                                for (int e = 0; e < E; ++e) if (ACT(e)) v1[0] += cabs2(am[e]);
                            }
                            block_sum<NT, 1>(v1, red, rphase);
                            STAT(sBisect, 1);
                            if (fabs(v1[0] - ws.r_thr) <= tol) { ts = mid; found = true; break; }
                            if (v1[0] > ws.r_thr) a = mid; else b = mid;
                        }
                        if (!found) ts = 0.5 * (a + b);
                    }
                    if (ts <= P.t_to) {
                        while (ws.t_next <= ts) {
                            double2 pg[E];
                            HORNER((ws.t_next - t) / h, pg);
                            RECORD(pg, ws.gi);
                            ws.gi++;
                            ws.t_next = ws.gi < npts ? P.times[ws.gi] : CUDART_INF;
                        }
                        // psi(t*) and the collapse (trajectory.py:235-241, 133-154)
                        double2 pst[E];
                        HORNER((ts - t) / h, pst);
                        double u;
                        DRAW(u);
                        GATHER(pst, xs);
                        double wts[MAXOPS];
                        for (int c0 = 0; c0 < P.nc; c0 += KRED) {
                            double v4[KRED] = {0.0, 0.0, 0.0, 0.0};
                            for (int kk = 0; kk < KRED; ++kk) {
                                if (c0 + kk < P.nc) {
#pragma unroll
                                    for (int e = 0; e < E; ++e)
                                        if (ACT(e)) v4[kk] += cabs2(row_dot(P.c[c0 + kk], II(e), xs));
                                }
                            }
                            block_sum<NT, KRED>(v4, red, rphase);
                            for (int kk = 0; kk < KRED; ++kk) if (c0 + kk < P.nc) wts[c0 + kk] = v4[kk];
                        }
                        double dp = 0.0;
                        for (int c = 0; c < P.nc; ++c) dp += wts[c];
                        if (dp <= 0.0) FAIL(kErrNoSupport);
                        int idx = 0;
                        for (int c = 0; c < P.nc; ++c) if (wts[c] > 0.0) idx = c;
                        double cum = 0.0;
                        for (int c = 0; c < P.nc; ++c) {
                            cum += wts[c] / dp;
                            if (wts[c] > 0.0 && cum >= u) { idx = c; break; }
                        }
                        const double scl = 1.0 / sqrt(wts[idx]);
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            pst[e] = ACT(e) ? cscale(scl, row_dot(P.c[idx], II(e), xs)) : make_double2(0.0, 0.0);
                        if (tid == 0 && ws.njumps < R.max_jumps) {
                            R.jump_t[(size_t)ws.row * R.max_jumps + ws.njumps] = ts;
                            R.jump_idx[(size_t)ws.row * R.max_jumps + ws.njumps] = idx;
                        }
                        ws.njumps++;
                        STAT(sJumps, 1);
                        DRAW(ws.r_thr);
                        COLD_START(ts, pst, h);
                        ws.steps_in_segment = 0;
                        continue;
                    }
                }
                PH_MARK(9);  // [9] jump test (+ jumps)
                while (ws.t_next <= t) {
                    double2 pg[E];
                    H::horner_fast(z, OVF(), q, (ws.t_next - t) / h, pg);
                    RECORD(pg, ws.gi);
                    ws.gi++;
                    ws.t_next = ws.gi < npts ? P.times[ws.gi] : CUDART_INF;
                }
                PH_MARK(10);  // [10] grid recording
            }
        }
    traj_done:
#ifdef QTM_PHASES
        if (tid == 0)
            for (int k = 0; k < 12; ++k) atomicAdd(R.phase_cycles + k, (unsigned long long)ph_acc[k]);
#endif
        if (tid == 0) {
            s_stats[sDraws] = (long long)s_stream.n;
            s_stats[sAttempts] += ws.c_att;
            s_stats[sSumQ] += ws.c_q;
            s_stats[sSumQQ1] += ws.c_qq;
            s_stats[sCorrIters] += ws.c_it;
            s_stats[sNfe] += ws.c_it;
            s_stats[sSteps] += ws.c_steps;
            long long* so = R.stats + (size_t)ws.row * NSTATS;
#pragma unroll
            for (int s = 0; s < NSTATS; ++s) so[s] = s_stats[s];
            R.status[ws.row] = rc;
            R.jump_count[ws.row] = ws.njumps;
            if (rc != kOk) atomicMin(R.first_fail, (unsigned long long)ws.row);
        }
        __syncthreads();
    }
    if constexpr (TM) {
        tm::fence_before_sync();
        __syncthreads();
        tm::fence_after_sync();
        if ((threadIdx.x >> 5) == 0) tm::dealloc(s_taddr, TrajKernel<NT, E, RREG, TM>::tmem_cols());
    }
#undef OVF
#undef W
#undef II
#undef ACT
#undef GATHER
#undef GSPMV
#undef GSPMV_T
#undef HORNER
#undef RESCALE
#undef FAIL
#undef FAIL4
#undef DRAW
#undef RECORD
#undef COLD_START
}

#undef STAT
#undef PH_MARK

}  // namespace qtm
