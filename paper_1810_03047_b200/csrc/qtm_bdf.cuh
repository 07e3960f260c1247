// qtm_bdf.cuh -- persistent sm_100a kernel for the BDF method family:
// quantum trajectories integrated with the reference's general engine,
// BDF orders 1-6 with the modified-Newton corrector on the iteration matrix
// M = I - h l0 G (G = the constant CSR generator, i.e. the Jacobian).
//
// Reference behaviour reproduced (see oracle/mcwf_oracle.c for the CPU
// restatement this kernel is checked against):
//   _attempt_general: weights, save, predict, Newton, error test,
//     commit or restore .................................... ode.py:334-356
//   _newton_correct: <= 3 iterations, resid = y - l0 (h G y - z1) - ypred,
//     dy = -M^{-1} resid, one retry with a fresh matrix ..... ode.py:379-407
//   _ensure_iteration_matrix: refactor when there is no LU, the Jacobian is
//     stale, or |h l0 / h l0_fact - 1| > 0.3; crate = 0.7 .. ode.py:409-423
//   scipy lu_factor / lu_solve (LAPACK zgetrf / zgetrs): unblocked
//     right-looking LU with partial pivoting (izamax: first row of maximal
//     |re| + |im|), reciprocal scaling of the sub-column, rank-1 update;
//     row interchanges, unit-lower and upper column-oriented solves
//   step retry loop, order/step control, jumps, recording: as the Adams
//     kernel (ode.py:261-329, 441-466; trajectory.py:133-250)
//
// Mapping.  One CTA per trajectory at a time (persistent, atomic work
// counter; 32 threads for d <= 64, else 256), NT threads own components
// i = tid + NT*k.  Every vector of the
// trajectory -- 7 Nordsieck rows, their saved copy, the Newton vectors --
// and the LU of M live in one per-CTA workspace: dynamic shared memory when
// it fits (d <= ~100), otherwise a per-CTA slice of HBM (L2-resident for
// moderate d).  The LU factorisation and the triangular solves are
// sequential in the pivot index, so they run as CTA-wide sweeps with one
// barrier per pivot; the trailing update walks columns by warp and rows by
// lane (column-major storage: coalesced, conflict-free).  There are no
// reductions inside the LU or the substitution solves, so in the unfused
// parity build (QTM_FMAD=0) they are bit-identical to the oracle's
// restatement.  From d = 48 up the
// Newton solve applies the explicit inverse instead (bdf_invert, LAPACK
// zgetri order after the same pivoted LU): one parallel matrix-vector
// product per iteration instead of 2d barrier-separated substitution
// steps; the result differs from the substitution at the rounding level,
// as LAPACK's blocked zgetrs does.
#pragma once
#include "qtm_traj.cuh"

#ifndef QTM_BDF128_MINB
#define QTM_BDF128_MINB 4  // 128-thread BDF CTAs per SM (the HBM-workspace range 64 < d <= 256)
#endif

namespace qtm {

constexpr int BDF_ROWS = 7;  // BDF order <= 6 (ode.py:46): rows 0..6

struct BdfParams {
    double2* ws;             // per-CTA workspaces in HBM (when not in shared memory)
    long long ws_stride;     // double2 elements per CTA workspace
    int in_smem;             // 1: the workspace is the kernel's dynamic shared memory
    int inverse;             // 1: Newton solves apply M^{-1} (zgetri after zgetrf), 0: substitution
};

// workspace layout in double2 units (d = state dimension)
struct BdfLayout {
    long long z, save, ypred, z1p, ycur, dy, x, e0, e1, psi, w2, ipiv, rowat, pos, dflag, dk, lu, total;
    __host__ __device__ static BdfLayout make(long long d) {
        BdfLayout L{};
        long long o = 0;
        L.z = o;     o += BDF_ROWS * d;
        L.save = o;  o += BDF_ROWS * d;
        L.ypred = o; o += d;
        L.z1p = o;   o += d;
        L.ycur = o;  o += d;
        L.dy = o;    o += d;
        L.x = o;     o += d;
        L.e0 = o;    o += d;
        L.e1 = o;    o += d;
        L.psi = o;   o += d;
        L.w2 = o;    o += (d + 1) / 2;   // doubles
        L.ipiv = o;  o += (d + 3) / 4;   // ints: pivot row of step k (zgetrf ipiv)
        L.rowat = o; o += (d + 3) / 4;   // ints: original row at position k after the interchanges
        L.pos = o;   o += (d + 3) / 4;   // ints: position of row i after the interchanges
        L.dflag = o; o += (d + 3) / 4;   // ints: branch of the division by U(k, k)
        L.dk = o;    o += d;             // (rat, scl) of the division by U(k, k)
        L.lu = o;    o += d * d;         // column-major: A(i, j) at lu[j*d + i]
        L.total = o;
        return L;
    }
};

// a / b in numpy's order (Smith's algorithm, npymath complex divide)
__device__ __forceinline__ double2 cdiv_np(double2 a, double2 b) {
    const double abr = fabs(b.x), abi = fabs(b.y);
    if (abr >= abi) {
        if (abr == 0.0 && abi == 0.0) return make_double2(a.x / abr, a.y / abr);
        const double rat = b.y / b.x, scl = 1.0 / (b.x + b.y * rat);
        return make_double2((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
    }
    const double rat = b.x / b.y, scl = 1.0 / (b.y + b.x * rat);
    return make_double2((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// cj[i] -= ck[i] * ukj for rows i = lo + lane, lo + lane + 32, ... < d: four
// rows in flight per lane (the loads of an HBM/L2-resident workspace would
// otherwise serialise on their latency for large d); same per-element
// arithmetic as the plain loop
__device__ __forceinline__ void col_axpy(double2* __restrict__ cj, const double2* __restrict__ ck,
                                         double2 ukj, int lo, int d, int lane) {
    int i = lo + lane;
    for (; i + 96 < d; i += 128) {
        double2 l[4], a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) { l[r] = ck[i + 32 * r]; a[r] = cj[i + 32 * r]; }
#pragma unroll
        for (int r = 0; r < 4; ++r)
            cj[i + 32 * r] = make_double2(a[r].x - (l[r].x * ukj.x - l[r].y * ukj.y),
                                          a[r].y - (l[r].x * ukj.y + l[r].y * ukj.x));
    }
    for (; i < d; i += 32) {
        const double2 l = ck[i], a = cj[i];
        cj[i] = make_double2(a.x - (l.x * ukj.x - l.y * ukj.y), a.y - (l.x * ukj.y + l.y * ukj.x));
    }
}

// M = I - hl0 G from the CSR generator, factored in place (zgetf2 order)
// izamax over rows k..d-1 of column ck: the first row of maximal |re| + |im|
// (every thread gets the same answer)
template <int NT>
__device__ __forceinline__ int pivot_row(const double2* __restrict__ ck, int k, int d, double* s_pv, int* s_pi) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double bv = -1.0;
    int bi = d;
    for (int i = k + tid; i < d; i += NT) {
        const double2 a = ck[i];
        const double v = fabs(a.x) + fabs(a.y);
        if (v > bv) { bv = v; bi = i; }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, m);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if constexpr (NW > 1) {
        if (lane == 0) { s_pv[warp] = bv; s_pi[warp] = bi; }
        __syncthreads();
        bv = s_pv[0];
        bi = s_pi[0];
        for (int w = 1; w < NW; ++w)
            if (s_pv[w] > bv || (s_pv[w] == bv && s_pi[w] < bi)) { bv = s_pv[w]; bi = s_pi[w]; }
    }
    return bi < d ? bi : k;
}

constexpr int LU_NB = 32;        // panel width of the blocked LU
constexpr int LU_MB = 64;        // rows of a trailing-update tile
// shared memory of the blocked LU's trailing-update tiles (double2 units)
constexpr int LU_TILE_ELEMS = LU_NB * LU_MB + LU_NB * 32;

// Blocked right-looking LU (LAPACK zgetrf structure) for a matrix that lives
// in HBM: per panel of LU_NB columns the unblocked factorisation restricted
// to the panel, the panel's row interchanges on the other columns, the
// triangular solve for the panel rows of the trailing columns, and the
// trailing update in LU_MB x 32 tiles staged through shared memory (each
// entry read and written once per panel instead of once per pivot).  Every
// entry still receives its updates one product at a time in pivot order,
// and the interchanges commute with the row-wise updates, so the result is
// bit-identical to the unblocked sweep.  Requires NT = 256.
template <int NT>
__device__ __forceinline__ void lu_blocked(double2* __restrict__ A, int* __restrict__ ipiv, int d, double2* tiles,
                           double* s_pv, int* s_pi) {
    static_assert(NT == 256, "tile mapping assumes 8 warps");
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double2* const sL = tiles;                   // [LU_NB][LU_MB]
    double2* const sU = tiles + LU_NB * LU_MB;   // [LU_NB][32]
    for (int k0 = 0; k0 < d; k0 += LU_NB) {
        const int kend = min(k0 + LU_NB, d), kb = kend - k0;
        // ---- panel: unblocked steps on columns k0..kend-1
        for (int k = k0; k < kend; ++k) {
            double2* const ck = A + (long long)k * d;
            const int p = pivot_row<NT>(ck, k, d, s_pv, s_pi);
            if (tid == 0) ipiv[k] = p;
            const double2 piv = ck[p];
            __syncthreads();
            if (piv.x != 0.0 || piv.y != 0.0) {
                if (p != k && tid < kb) {
                    double2* const cj = A + (long long)(k0 + tid) * d;
                    const double2 t = cj[k];
                    cj[k] = cj[p];
                    cj[p] = t;
                }
                const double2 rcp = cdiv_np(make_double2(1.0, 0.0), piv);
                __syncthreads();
                for (int i = k + 1 + tid; i < d; i += NT) ck[i] = cmul2(ck[i], rcp);
            }
            __syncthreads();
            for (int j = k + 1 + warp; j < kend; j += NW) {
                double2* const cj = A + (long long)j * d;
                col_axpy(cj, ck, cj[k], k + 1, d, lane);
            }
            __syncthreads();
        }
        // ---- the panel's interchanges on every other column (zlaswp)
        for (int j = tid; j < d; j += NT) {
            if (j >= k0 && j < kend) continue;
            double2* const cj = A + (long long)j * d;
            for (int k = k0; k < kend; ++k) {
                const int p = ipiv[k];
                if (p != k) { const double2 t = cj[k]; cj[k] = cj[p]; cj[p] = t; }
            }
        }
        __syncthreads();
        if (kend >= d) break;
        // ---- U12: panel rows of the trailing columns (unit-lower solve, ztrsm)
        for (int j = kend + tid; j < d; j += NT) {
            double2* const cj = A + (long long)j * d;
            for (int k = k0 + 1; k < kend; ++k) {
                double2 s = cj[k];
                for (int kp = k0; kp < k; ++kp) {
                    const double2 l = A[(long long)kp * d + k], u = cj[kp];
                    s = make_double2(s.x - (l.x * u.x - l.y * u.y), s.y - (l.x * u.y + l.y * u.x));
                }
                cj[k] = s;
            }
        }
        __syncthreads();
        // ---- A22 -= L21 U12, tile by tile, products subtracted in pivot order
        for (int rb = kend; rb < d; rb += LU_MB) {
            for (int idx = tid; idx < kb * LU_MB; idx += NT) {
                const int k = idx / LU_MB, r = idx - k * LU_MB;
                sL[k * LU_MB + r] = rb + r < d ? A[(long long)(k0 + k) * d + rb + r] : make_double2(0.0, 0.0);
            }
            for (int cb = kend; cb < d; cb += 32) {
                for (int idx = tid; idx < kb * 32; idx += NT) {
                    const int c = idx / kb, k = idx - c * kb;
                    sU[k * 32 + c] = cb + c < d ? A[(long long)(cb + c) * d + k0 + k] : make_double2(0.0, 0.0);
                }
                __syncthreads();
                double2 acc[2][4];
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int i = rb + lane + 32 * a, j = cb + 4 * warp + c;
                        acc[a][c] = (i < d && j < d) ? A[(long long)j * d + i] : make_double2(0.0, 0.0);
                    }
                for (int k = 0; k < kb; ++k) {
                    const double2 l0 = sL[k * LU_MB + lane], l1 = sL[k * LU_MB + lane + 32];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const double2 u = sU[k * 32 + 4 * warp + c];
                        acc[0][c] = make_double2(acc[0][c].x - (l0.x * u.x - l0.y * u.y),
                                                 acc[0][c].y - (l0.x * u.y + l0.y * u.x));
                        acc[1][c] = make_double2(acc[1][c].x - (l1.x * u.x - l1.y * u.y),
                                                 acc[1][c].y - (l1.x * u.y + l1.y * u.x));
                    }
                }
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int i = rb + lane + 32 * a, j = cb + 4 * warp + c;
                        if (i < d && j < d) A[(long long)j * d + i] = acc[a][c];
                    }
                __syncthreads();
            }
        }
    }
}

template <int NT>
__device__ __forceinline__ void bdf_factor(const DevProblem& P, double2* __restrict__ A, int* __restrict__ ipiv,
                           int* __restrict__ rowat, int* __restrict__ pos, int* __restrict__ dflag,
                           double2* __restrict__ dk, double hl0, double* s_pv, int* s_pi,
                           double2* tiles) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = P.d;
    const long long dd = (long long)d * d;
    for (long long k = tid; k < dd; k += NT) A[k] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int i = tid; i < d; i += NT) {
        const int b = __ldg(P.g.rp + i), en = __ldg(P.g.rp + i + 1);
        for (int j = b; j < en; ++j) {
            const double2 v = __ldg(P.g.v + j);
            A[(long long)__ldg(P.g.ci + j) * d + i] = make_double2(-hl0 * v.x, -hl0 * v.y);
        }
        A[(long long)i * d + i].x += 1.0;
    }
    __syncthreads();
    bool blocked = false;
    if constexpr (NT == 256) {
        if (tiles) {
            lu_blocked<NT>(A, ipiv, d, tiles, s_pv, s_pi);
            blocked = true;
        }
    }
    for (int k = 0; k < d && !blocked; ++k) {
        double2* const ck = A + (long long)k * d;
        const int p = pivot_row<NT>(ck, k, d, s_pv, s_pi);
        if (tid == 0) ipiv[k] = p;
        const double2 piv = ck[p];
        __syncthreads();  // every thread holds the pivot before the rows move
        if (piv.x != 0.0 || piv.y != 0.0) {
            if (p != k) {
                for (int j = tid; j < d; j += NT) {
                    double2* const cj = A + (long long)j * d;
                    const double2 t = cj[k];
                    cj[k] = cj[p];
                    cj[p] = t;
                }
            }
            const double2 rcp = cdiv_np(make_double2(1.0, 0.0), piv);
            __syncthreads();
            for (int i = k + 1 + tid; i < d; i += NT) ck[i] = cmul2(ck[i], rcp);
        }
        __syncthreads();
        // trailing update: A(i, j) -= L(i, k) U(k, j), columns by warp, rows by lane
        for (int j = k + 1 + warp; j < d; j += NW) {
            double2* const cj = A + (long long)j * d;
            col_axpy(cj, ck, cj[k], k + 1, d, lane);
        }
        __syncthreads();
    }
    // Solve-side constants, computed once per factorisation: pos[i] = where
    // b[i] lands after zlaswp's sequential interchanges (the caller writes the
    // residual pre-permuted), and the divisor-only part of cdiv_np(x, U(k,k))
    // -- rat and scl depend on U(k, k) alone, so the back substitution needs
    // no division and stays bit-identical to cdiv_np.
    if (tid == 0) {
        for (int k = 0; k < d; ++k) rowat[k] = k;
        for (int k = 0; k < d; ++k) {
            const int p = ipiv[k];
            if (p != k) { const int t = rowat[k]; rowat[k] = rowat[p]; rowat[p] = t; }
        }
    }
    for (int k = tid; k < d; k += NT) {
        const double2 b = A[(long long)k * d + k];
        const double abr = fabs(b.x), abi = fabs(b.y);
        if (abr >= abi) {
            if (abr == 0.0 && abi == 0.0) {
                dflag[k] = 2;
                dk[k] = make_double2(0.0, 0.0);
            } else {
                const double rat = b.y / b.x;
                dflag[k] = 0;
                dk[k] = make_double2(rat, 1.0 / (b.x + b.y * rat));
            }
        } else {
            const double rat = b.x / b.y;
            dflag[k] = 1;
            dk[k] = make_double2(rat, 1.0 / (b.y + b.x * rat));
        }
    }
    __syncthreads();
    for (int k = tid; k < d; k += NT) pos[rowat[k]] = k;
    __syncthreads();
}

// xk = cdiv_np(b, U(k, k)) with the divisor part precomputed (see bdf_factor)
__device__ __forceinline__ double2 udiv(double2 b, double2 rs, int fl) {
    if (fl == 0) return make_double2((b.x + b.y * rs.x) * rs.y, (b.y - b.x * rs.x) * rs.y);
    if (fl == 1) return make_double2((b.x * rs.x + b.y) * rs.y, (b.y * rs.x - b.x) * rs.y);
    return make_double2(b.x / rs.y, b.y / rs.y);  // U(k, k) = 0: rs = (0, 0), numpy's b / 0
}

// b_i -= sum_j y_j A(i, k0 + j) over the block's pivots j (ascending for
// the forward sweep, descending for the backward one, skipping pivots whose
// value was exactly zero, as the column sweep does) for rows i in
// [lo, hi).  Each thread carries up to 4 rows (d <= 4 NT) as independent
// chains; the A loads do not depend on the sums, so they run ahead.
template <int NT, bool FWD>
__device__ __forceinline__ void block_rows_update(const double2* __restrict__ A, int d, int k0, int kb,
                                                  int lo, int hi, const double2* sY, const int* sF,
                                                  double2* __restrict__ b) {
    for (int base = lo; base < hi; base += 4 * NT) {
        double2 s[4];
        int iv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            iv[r] = base + threadIdx.x + r * NT;
            s[r] = iv[r] < hi ? b[iv[r]] : make_double2(0.0, 0.0);
        }
#pragma unroll 2
        for (int jj = 0; jj < kb; ++jj) {
            const int j = FWD ? jj : kb - 1 - jj;
            const double2* const cj = A + (long long)(k0 + j) * d;
            double2 a[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = iv[r] < hi ? cj[iv[r]] : make_double2(0.0, 0.0);
            if (sF[j]) {
                const double2 y = sY[j];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    s[r] = make_double2(s[r].x - (y.x * a[r].x - y.y * a[r].y),
                                        s[r].y - (y.x * a[r].y + y.y * a[r].x));
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (iv[r] < hi) b[iv[r]] = s[r];
    }
}

// Blocked substitution for an HBM-resident LU (NT = 256): per block of 32
// pivots, warp 0 solves the diagonal block from shared memory with shuffles
// (no CTA barrier per pivot) and all threads then apply the block's 32
// updates to the remaining rows, row by row in pivot order.  Each row sees
// the same update sequence as the column sweep of bdf_solve, so the result
// is bit-identical; the L/U columns stream through once, coalesced, with 3
// barriers per block instead of one per pivot.  b arrives interchanged.
template <int NT>
__device__ __forceinline__ void bdf_solve_blocked(int d, const double2* __restrict__ A, const int* __restrict__ dflag,
                                  const double2* __restrict__ dk, double2* __restrict__ b,
                                  double2* __restrict__ x, double2* tiles) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double2* const sD = tiles;             // [32][32] diagonal block, column-major
    double2* const sY = tiles + 32 * 32;   // [32] solved values of the block
    int* const sF = reinterpret_cast<int*>(sY + 32);  // [32] 1 = the pivot's update applies
    __syncthreads();
    for (int k0 = 0; k0 < d; k0 += 32) {
        const int kb = min(32, d - k0);
        for (int idx = tid; idx < kb * 32; idx += NT) {
            const int j = idx >> 5, i = idx & 31;
            sD[idx] = i < kb ? A[(long long)(k0 + j) * d + k0 + i] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        if (warp == 0) {
            double2 bl = lane < kb ? b[k0 + lane] : make_double2(0.0, 0.0);
            for (int j = 0; j < kb; ++j) {
                const double2 yj = make_double2(__shfl_sync(0xffffffffu, bl.x, j),
                                                __shfl_sync(0xffffffffu, bl.y, j));
                const bool nz = yj.x != 0.0 || yj.y != 0.0;
                if (lane == 0) { sY[j] = yj; sF[j] = nz; }
                if (nz && lane > j && lane < kb) {
                    const double2 a = sD[j * 32 + lane];
                    bl = make_double2(bl.x - (yj.x * a.x - yj.y * a.y), bl.y - (yj.x * a.y + yj.y * a.x));
                }
            }
            if (lane < kb) b[k0 + lane] = bl;
        }
        __syncthreads();
        block_rows_update<NT, true>(A, d, k0, kb, k0 + kb, d, sY, sF, b);
        __syncthreads();
    }
    for (int k0 = ((d - 1) / 32) * 32; k0 >= 0; k0 -= 32) {
        const int kb = min(32, d - k0);
        for (int idx = tid; idx < kb * 32; idx += NT) {
            const int j = idx >> 5, i = idx & 31;
            sD[idx] = i < kb ? A[(long long)(k0 + j) * d + k0 + i] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        if (warp == 0) {
            double2 bl = lane < kb ? b[k0 + lane] : make_double2(0.0, 0.0);
            for (int j = kb - 1; j >= 0; --j) {
                const double2 bj = make_double2(__shfl_sync(0xffffffffu, bl.x, j),
                                                __shfl_sync(0xffffffffu, bl.y, j));
                const bool nz = bj.x != 0.0 || bj.y != 0.0;
                const double2 xj = nz ? udiv(bj, dk[k0 + j], dflag[k0 + j]) : bj;
                if (lane == 0) { sY[j] = xj; sF[j] = nz; x[k0 + j] = xj; }
                if (nz && lane < j) {
                    const double2 a = sD[j * 32 + lane];
                    bl = make_double2(bl.x - (xj.x * a.x - xj.y * a.y), bl.y - (xj.x * a.y + xj.y * a.x));
                }
            }
        }
        __syncthreads();
        block_rows_update<NT, false>(A, d, k0, kb, 0, k0, sY, sF, b);
        __syncthreads();
    }
}

// M^{-1} in place from its LU (LAPACK zgetri, unblocked): inv(U) column by
// column (ztrti2), then inv(M) L = inv(U) from the last column back
// (zgemv per column), then the column interchanges in reverse pivot order.
// Every entry is a sequential dot product owned by one thread (rows by
// thread, column-major storage: conflict-free), two barriers per column.
// The Newton solve then is one parallel matrix-vector product instead of
// 2d barrier-separated substitution steps.  t: d-vector scratch.
template <int NT>
__device__ __forceinline__ void bdf_invert(int d, double2* __restrict__ A, const int* __restrict__ ipiv,
                           double2* __restrict__ t) {
    const int tid = threadIdx.x;
    for (int j = 0; j < d; ++j) {
        double2* const cj = A + (long long)j * d;
        for (int i = tid; i < j; i += NT) t[i] = cj[i];
        const double2 ujj = cdiv_np(make_double2(1.0, 0.0), cj[j]);  // read before thread 0 overwrites it
        __syncthreads();
        const double2 ajj = make_double2(-ujj.x, -ujj.y);
        for (int i = tid; i < j; i += NT) {
            double sr = 0.0, si = 0.0;
#pragma unroll 4
            for (int k = i; k < j; ++k) {
                const double2 u = A[(long long)k * d + i], v = t[k];
                sr = sr + (u.x * v.x - u.y * v.y);
                si = si + (u.x * v.y + u.y * v.x);
            }
            cj[i] = make_double2(ajj.x * sr - ajj.y * si, ajj.x * si + ajj.y * sr);
        }
        if (tid == 0) cj[j] = ujj;
        __syncthreads();
    }
    for (int j = d - 1; j >= 0; --j) {
        double2* const cj = A + (long long)j * d;
        for (int i = j + 1 + tid; i < d; i += NT) {
            t[i] = cj[i];
            cj[i] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        if (j < d - 1) {
            for (int i = tid; i < d; i += NT) {
                double2 s = cj[i];
#pragma unroll 4
                for (int k = j + 1; k < d; ++k) {
                    const double2 a = A[(long long)k * d + i], w = t[k];
                    s = make_double2(s.x - (a.x * w.x - a.y * w.y), s.y - (a.x * w.y + a.y * w.x));
                }
                cj[i] = s;
            }
        }
        __syncthreads();
    }
    for (int j = d - 2; j >= 0; --j) {
        const int jp = ipiv[j];
        if (jp != j) {
            double2* const cj = A + (long long)j * d;
            double2* const cp = A + (long long)jp * d;
            for (int i = tid; i < d; i += NT) {
                const double2 a = cj[i];
                cj[i] = cp[i];
                cp[i] = a;
            }
            __syncthreads();
        }
    }
}

// x = M^{-1} b with the explicit inverse: row i summed over j in order
template <int NT>
__device__ __forceinline__ void bdf_apply_inverse(int d, const double2* __restrict__ A, const double2* __restrict__ b,
                                  double2* __restrict__ x) {
    const int tid = threadIdx.x;
    __syncthreads();
    for (int i = tid; i < d; i += NT) {
        double sr = 0.0, si = 0.0;
#pragma unroll 4
        for (int j = 0; j < d; ++j) {
            const double2 a = A[(long long)j * d + i], v = b[j];
            sr = sr + (a.x * v.x - a.y * v.y);
            si = si + (a.x * v.y + a.y * v.x);
        }
        x[i] = make_double2(sr, si);
    }
    __syncthreads();
}

// x = M^{-1} b (zgetrs).  b arrives already interchanged (the caller writes
// row i of the residual at pos[i]) and is overwritten by the forward sweep.
template <int NT>
__device__ __forceinline__ void bdf_solve(int d, const double2* __restrict__ A, const int* __restrict__ dflag,
                          const double2* __restrict__ dk, double2* __restrict__ b,
                          double2* __restrict__ x) {
    const int tid = threadIdx.x;
    __syncthreads();
    for (int k = 0; k < d; ++k) {
        const double2 bk = b[k];
        if (bk.x == 0.0 && bk.y == 0.0) continue;
        const double2* const ck = A + (long long)k * d;
        for (int i = k + 1 + tid; i < d; i += NT) {
            const double2 a = ck[i], bi = b[i];
            b[i] = make_double2(bi.x - (bk.x * a.x - bk.y * a.y), bi.y - (bk.x * a.y + bk.y * a.x));
        }
        __syncthreads();
    }
    for (int k = d - 1; k >= 0; --k) {
        double2 xk = b[k];
        if (xk.x != 0.0 || xk.y != 0.0) {
            // xk = cdiv_np(b[k], U(k, k)) with the divisor part precomputed
            const double2 rs = dk[k];
            const int fl = dflag[k];
            xk = udiv(xk, rs, fl);
            const double2* const ck = A + (long long)k * d;
            for (int i = tid; i < k; i += NT) {
                const double2 a = ck[i], bi = b[i];
                b[i] = make_double2(bi.x - (xk.x * a.x - xk.y * a.y), bi.y - (xk.x * a.y + xk.y * a.x));
            }
        }
        if (tid == 0) x[k] = xk;
        __syncthreads();
    }
}

template <int NT>
__device__ __forceinline__ double bsum1(double v, double* red, int& phase) {
    double a[1] = {v};
    block_sum<NT, 1>(a, red, phase);
    return a[0];
}

// Horner of the history polynomial at s for component i (nordsieck_eval)
__device__ __forceinline__ double2 bdf_horner(const double2* Z, int d, int q, double s, int i) {
    double2 acc = Z[(long long)q * d + i];
    for (int j = q - 1; j >= 0; --j) acc = cadd(cscale(s, acc), Z[(long long)j * d + i]);
    return acc;
}

// SMEM: the workspace is the dynamic shared memory (known at compile time,
// so every workspace access compiles to LDS/STS instead of generic
// loads/stores that resolve the address space at run time)
// (one-warp CTAs: capped at 128 registers so ~16 trajectories share an SM)
template <int NT, bool SMEM>
__global__ void __launch_bounds__(NT, NT == 32 ? 16 : (NT == 64 ? 8 : (NT == 128 ? QTM_BDF128_MINB : 1)))
bdf_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ RunParams R,
           const __grid_constant__ BdfParams B) {
    constexpr int NW = NT / 32;
    extern __shared__ double2 smem[];
    __shared__ double red[2 * KRED * (NW > 1 ? NW : 1)];
    __shared__ double s_pv[NW];
    __shared__ int s_pi[NW];
    __shared__ long long s_row;
    __shared__ Stream s_stream;
    __shared__ double s_draw;

    const int tid = threadIdx.x, lane = tid & 31;
    const int d = P.d, npts = P.n_pts;
    const BdfLayout L = BdfLayout::make(d);
    double2* const ws = SMEM ? smem : B.ws + (long long)blockIdx.x * B.ws_stride;
    double2* const Z = ws + L.z;
    double2* const SV = ws + L.save;
    double2* const YP = ws + L.ypred;
    double2* const Z1 = ws + L.z1p;
    double2* const YC = ws + L.ycur;
    double2* const DY = ws + L.dy;
    double2* const X = ws + L.x;
    double2* const PS = ws + L.psi;
    double* const W2 = reinterpret_cast<double*>(ws + L.w2);
    int* const IPIV = reinterpret_cast<int*>(ws + L.ipiv);
    int* const ROWAT = reinterpret_cast<int*>(ws + L.rowat);
    int* const POS = reinterpret_cast<int*>(ws + L.pos);
    int* const DFLAG = reinterpret_cast<int*>(ws + L.dflag);
    double2* const DK = ws + L.dk;
    double2* const A = ws + L.lu;
    int rphase = 0;

    for (;;) {
        if (tid == 0) s_row = next_row(R);
        __syncthreads();
        const long long row = s_row;
        if (row >= R.n_traj) break;
        if (tid == 0)
            s_stream.init(R.stream_kind, R.seed, (uint64_t)(R.traj_begin + row),
                          R.script ? R.script + row * R.script_stride : nullptr,
                          R.script_len ? R.script_len[row] : 0, R.script_fallback);
        __syncthreads();

        long long st[NSTATS];
#pragma unroll
        for (int s = 0; s < NSTATS; ++s) st[s] = 0;
        int rc = kOk;
        double err0 = 0.0, err1 = 0.0, err2 = 0.0, err3 = 0.0;
        long long njumps = 0, steps_in_segment = 0;
        double t = P.t_from, h = P.h0_first, t_lo = P.t_from, crate = 0.7, hl0_fact = 1.0, r_thr = 0.0;
        int q = 1, ialth = 2, gi = 1, ecur = 0;
        bool has_eprev = false, has_lu = false, jac_stale = true;

        // one uniform draw (thread 0 evaluates, broadcast)
        auto draw = [&]() -> double {
            __syncthreads();
            if (tid == 0) s_draw = s_stream.next();
            __syncthreads();
            return s_draw;
        };
        // per-warp partial sums of <psi|E_k|psi> and <psi|psi> (PS complete)
        auto record = [&](int g) {
            __syncthreads();
            if (R.psi_slot && R.psi_slot[g] >= 0) {
                double2* const po = R.psi_out + ((size_t)row * R.n_psi + R.psi_slot[g]) * d;
                for (int i = tid; i < d; i += NT) po[i] = PS[i];
            }
            double* const rp = R.rec_partial + ((size_t)row * npts + g) * (size_t)(P.ne + 1) * NW + (tid >> 5);
            for (int k = 0; k <= P.ne; ++k) {
                double acc[1] = {0.0};
                for (int i = tid; i < d; i += NT) {
                    const double2 p = PS[i];
                    if (k < P.ne) {
                        const double2 s = row_dot(P.e[k], i, PS);
                        acc[0] += p.x * s.x - (-p.y) * s.y;
                    } else {
                        acc[0] += cabs2(p);
                    }
                }
                warp_sum_lane0<1>(acc);
                if (lane == 0) rp[(size_t)k * NW] = acc[0];
            }
        };
        // psi at grid point g (Horner at the current step), then record
        auto record_grid = [&](int g) {
            const double s = (P.times[g] - t) / h;
            __syncthreads();
            for (int i = tid; i < d; i += NT) PS[i] = bdf_horner(Z, d, q, s, i);
            record(g);
        };
        // new solver at (t0, y0 in vector Y) with step h0 (ode.py:164-217)
        auto cold_start = [&](double t0, const double2* Y, double h0) {
            t = t0; t_lo = t0; q = 1; h = h0;
            __syncthreads();
            for (int i = tid; i < d; i += NT) {
                const double2 f = row_dot(P.g, i, Y);
                Z[i] = Y[i];
                Z[(long long)d + i] = cscale(h, f);
            }
            st[sNfe]++;
            crate = 0.7; ialth = 2; has_eprev = false; has_lu = false; jac_stale = true;
            __syncthreads();
        };
        auto rescale = [&](double r) {
            double f = 1.0;
            for (int j = 1; j <= q; ++j) {
                f *= r;
                for (int i = tid; i < d; i += NT) Z[(long long)j * d + i] = cscale(f, Z[(long long)j * d + i]);
            }
            h *= r;
            has_eprev = false;
            ialth = q + 1;
        };

        for (int i = tid; i < d; i += NT) PS[i] = P.psi0[i];
        record(0);
        r_thr = draw();
        for (int i = tid; i < d; i += NT) YC[i] = P.psi0[i];
        cold_start(P.t_from, YC, P.h0_first);

        while (gi < npts) {
            // ================= OdeSolver.step() (ode.py:261-312) =================
            int nef = 0, ncf = 0;
            double est = 0.0;
            for (;;) {
                if (t + h == t) { rc = kErrStepCollapse; err0 = t; err1 = h; goto traj_done; }
                st[sAttempts]++;
                st[sSumQ] += q;
                st[sSumQQ1] += q * (q + 1);
                const double* const lv = P.l[q];
                const double l0 = lv[0], conit = P.conit[q];
                // weights, save, predict (ode.py:336-342)
                for (int i = tid; i < d; i += NT) {
                    const double2 z0 = Z[i];
                    const double w = 1.0 / (P.atol + P.rtol * hypot(z0.x, z0.y));
                    W2[i] = w * w;
                    for (int j = 0; j <= q; ++j) SV[(long long)j * d + i] = Z[(long long)j * d + i];
                    for (int r = 0; r < q; ++r)
                        for (int j = q - 1; j >= r; --j)
                            Z[(long long)j * d + i] = cadd(Z[(long long)j * d + i], Z[(long long)(j + 1) * d + i]);
                    YP[i] = Z[i];
                    Z1[i] = Z[(long long)d + i];
                }
                bool converged = false;
                for (int attempt = 0; attempt < 2 && !converged; ++attempt) {
                    // _ensure_iteration_matrix (ode.py:409-423)
                    const double hl0 = h * l0;
                    if (!(has_lu && !jac_stale && fabs(hl0 / hl0_fact - 1.0) <= 0.3)) {
                        jac_stale = false;
                        bdf_factor<NT>(P, A, IPIV, ROWAT, POS, DFLAG, DK, hl0, s_pv, s_pi,
                                       SMEM ? nullptr : smem);
                        if (B.inverse) bdf_invert<NT>(d, A, IPIV, X);
                        st[sLuFactor]++;
                        has_lu = true;
                        hl0_fact = hl0;
                        crate = 0.7;
                    }
                    for (int i = tid; i < d; i += NT) YC[i] = YP[i];
                    __syncthreads();
                    double delp = 0.0;
                    for (int m = 0; m < 3; ++m) {
                        // resid = ycur - l0 * (h G ycur - z1pred) - ypred (left to right)
                        for (int i = tid; i < d; i += NT) {
                            const double2 f = row_dot(P.g, i, YC);
                            DY[B.inverse ? i : POS[i]] =
                                csub(csub(YC[i], cscale(l0, csub(cscale(h, f), Z1[i]))), YP[i]);
                        }
                        st[sNfe]++;
                        if (B.inverse)
                            bdf_apply_inverse<NT>(d, A, DY, X);
                        else if (NT == 256 && !SMEM)
                            bdf_solve_blocked<NT>(d, A, DFLAG, DK, DY, X, smem);
                        else
                            bdf_solve<NT>(d, A, DFLAG, DK, DY, X);
                        double acc = 0.0;
                        for (int i = tid; i < d; i += NT) {
                            const double2 xi = X[i];
                            const double2 dy = make_double2(-xi.x, -xi.y);
                            YC[i] = cadd(YC[i], dy);
                            acc += cabs2(dy) * W2[i];
                        }
                        st[sCorrIters]++;
                        const double del = sqrt(bsum1<NT>(acc, red, rphase) / (double)d);
                        if (m > 0) {
                            const double a = 0.2 * crate, b = del / delp;
                            crate = b > a ? b : a;  // Python max(a, b)
                        }
                        const double c15 = 1.5 * crate;
                        if (del * (c15 < 1.0 ? c15 : 1.0) <= conit) { converged = true; break; }
                        if (m > 0 && del > 2.0 * delp) break;
                        delp = del;
                    }
                    if (converged) break;
                    if (!jac_stale && attempt == 0) {  // retry once with a fresh matrix
                        jac_stale = true;
                        has_lu = false;
                        continue;
                    }
                    break;
                }
                if (converged) {
                    // e = (ycur - ypred) / l0: numpy divides by (l0 + 0j) = times 1/l0
                    const double rl0 = 1.0 / l0;
                    double2* const ec = ws + (ecur ? L.e1 : L.e0);
                    double acc = 0.0;
                    for (int i = tid; i < d; i += NT) {
                        const double2 e = cscale(rl0, csub(YC[i], YP[i]));
                        ec[i] = e;
                        acc += cabs2(e) * W2[i];
                    }
                    est = sqrt(bsum1<NT>(acc, red, rphase) / (double)d) / P.tau2[q];
                    if (!(est > 1.0)) {
                        for (int i = tid; i < d; i += NT) {
                            const double2 e = ec[i];
                            for (int j = 0; j <= q; ++j)
                                Z[(long long)j * d + i] = cadd(Z[(long long)j * d + i], cscale(lv[j], e));
                        }
                        break;  // accepted
                    }
                }
                // rejected: restore the saved history (ode.py:346, 350)
                for (int i = tid; i < d; i += NT)
                    for (int j = 0; j <= q; ++j) Z[(long long)j * d + i] = SV[(long long)j * d + i];
                if (!converged) {
                    st[sCorrFail]++;
                    ncf++;
                    jac_stale = true;  // ode.py:308-309
                    has_lu = false;
                    if (ncf >= 10) { rc = kErrCorrector; err0 = t; err1 = h; goto traj_done; }
                    rescale(0.25);
                    continue;
                }
                st[sErrReject]++;
                if (++nef >= 10) { rc = kErrRepeatedErrTest; err0 = t; err1 = h; goto traj_done; }
                if (nef >= 3) {
                    // _restart_order_one(0.1), ode.py:314-323
                    q = 1;
                    h *= 0.1;
                    __syncthreads();
                    for (int i = tid; i < d; i += NT) X[i] = Z[i];
                    __syncthreads();
                    for (int i = tid; i < d; i += NT) Z[(long long)d + i] = cscale(h, row_dot(P.g, i, X));
                    st[sNfe]++;
                    has_eprev = false;
                    ialth = q + 1;
                    has_lu = false;
                } else {
                    const double rr = 1.0 / (1.2 * pow(est, P.rq1[q]) + 1e-6);
                    const double m1 = 0.9 < rr ? 0.9 : rr;
                    rescale(m1 > 0.1 ? m1 : 0.1);
                }
            }
            // accepted step bookkeeping (ode.py:281-292)
            t_lo = t;
            t += h;
            st[sSteps]++;
            if (--ialth == 0) {
                // _order_step_control (ode.py:441-466); weights from the new z0
                const bool need_d = q > 1, need_u = q < P.max_order && has_eprev;
                double v[2] = {0.0, 0.0};
                const double2* const ecp = ws + (ecur ? L.e1 : L.e0);
                const double2* const epp = ws + (ecur ? L.e0 : L.e1);
                for (int i = tid; i < d; i += NT) {
                    const double2 z0 = Z[i];
                    const double w = 1.0 / (P.atol + P.rtol * hypot(z0.x, z0.y));
                    const double2 zq = Z[(long long)q * d + i];
                    const double2 de = csub(ecp[i], epp[i]);
                    v[0] += cabs2(zq) * w * w;
                    v[1] += cabs2(de) * w * w;
                }
                block_sum<NT, 2>(v, red, rphase);
                const double r_same = 1.0 / (1.2 * pow(est, P.rq1[q]) + 1e-6);
                double r_down = 0.0, r_up = 0.0;
                if (need_d) r_down = 1.0 / (1.3 * pow(sqrt(v[0] / (double)d) / P.tau1[q], P.rq0[q]) + 1e-6);
                if (need_u) r_up = 1.0 / (1.4 * pow(sqrt(v[1] / (double)d) / P.tau3[q], P.rq2[q]) + 1e-6);
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
                        for (int i = tid; i < d; i += NT) Z[(long long)(q + 1) * d + i] = cscale(cu, ecp[i]);
                        q = q + 1;
                        st[sOrderUp]++;
                    } else if (best == r_down) {
                        q = q - 1;
                        st[sOrderDown]++;
                    }
                    const double m1 = 10.0 < best ? 10.0 : best;
                    rescale(m1 > 0.1 ? m1 : 0.1);
                }
            } else {
                ecur ^= 1;  // e_prev = e
                has_eprev = true;
            }
            // ================= trajectory loop body (trajectory.py:225-246) =======
            if (++steps_in_segment > P.max_steps) { rc = kErrMaxSteps; err0 = t; err1 = h; goto traj_done; }
            if (P.nc > 0) {
                double nrm = 0.0;
                for (int i = tid; i < d; i += NT) nrm += cabs2(Z[i]);
                nrm = bsum1<NT>(nrm, red, rphase);
                if (nrm < r_thr) {
                    // locate_jump_time (trajectory.py:157-182)
                    double v2[2] = {0.0, 0.0};
                    const double s_lo = (t_lo - t) / h, s_hi = (t - t) / h;
                    for (int i = tid; i < d; i += NT) {
                        v2[0] += cabs2(bdf_horner(Z, d, q, s_lo, i));
                        v2[1] += cabs2(bdf_horner(Z, d, q, s_hi, i));
                    }
                    block_sum<NT, 2>(v2, red, rphase);
                    const double f_lo = v2[0], f_hi = v2[1];
                    const double tol = 1e-9 * r_thr;
                    if (f_lo < r_thr - tol || f_hi > r_thr + tol) {
                        rc = kErrBracket; err0 = t_lo; err1 = t; err2 = f_lo; err3 = f_hi;
                        goto traj_done;
                    }
                    double ts;
                    if (f_lo <= r_thr + tol) {
                        ts = t_lo;
                    } else {
                        double a = t_lo, b = t;
                        bool found = false;
                        ts = 0.0;
                        for (int it = 0; it < 60; ++it) {
                            const double mid = 0.5 * (a + b);
                            const double sm = (mid - t) / h;
                            double acc = 0.0;
                            for (int i = tid; i < d; i += NT) acc += cabs2(bdf_horner(Z, d, q, sm, i));
                            const double fm = bsum1<NT>(acc, red, rphase);
                            st[sBisect]++;
                            if (fabs(fm - r_thr) <= tol) { ts = mid; found = true; break; }
                            if (fm > r_thr) a = mid; else b = mid;
                        }
                        if (!found) ts = 0.5 * (a + b);
                    }
                    if (ts <= P.t_to) {
                        while (gi < npts && P.times[gi] <= ts) { record_grid(gi); gi++; }
                        // psi(t*) and the collapse (trajectory.py:235-241, 133-154)
                        const double sst = (ts - t) / h;
                        __syncthreads();
                        for (int i = tid; i < d; i += NT) PS[i] = bdf_horner(Z, d, q, sst, i);
                        const double u = draw();  // (draw() synchronises: PS complete)
                        double wts[MAXOPS];
                        for (int c0 = 0; c0 < P.nc; c0 += KRED) {
                            double v4[KRED] = {0.0, 0.0, 0.0, 0.0};
                            for (int kk = 0; kk < KRED; ++kk)
                                if (c0 + kk < P.nc)
                                    for (int i = tid; i < d; i += NT) v4[kk] += cabs2(row_dot(P.c[c0 + kk], i, PS));
                            block_sum<NT, KRED>(v4, red, rphase);
                            for (int kk = 0; kk < KRED; ++kk) if (c0 + kk < P.nc) wts[c0 + kk] = v4[kk];
                        }
                        double dp = 0.0;
                        for (int c = 0; c < P.nc; ++c) dp += wts[c];
                        if (dp <= 0.0) { rc = kErrNoSupport; err0 = t; err1 = h; goto traj_done; }
                        int idx = 0;
                        for (int c = 0; c < P.nc; ++c) if (wts[c] > 0.0) idx = c;
                        double cum = 0.0;
                        for (int c = 0; c < P.nc; ++c) {
                            cum += wts[c] / dp;
                            if (wts[c] > 0.0 && cum >= u) { idx = c; break; }
                        }
                        const double scl = 1.0 / sqrt(wts[idx]);
                        for (int i = tid; i < d; i += NT) YC[i] = cscale(scl, row_dot(P.c[idx], i, PS));
                        if (tid == 0 && njumps < R.max_jumps) {
                            R.jump_t[(size_t)row * R.max_jumps + njumps] = ts;
                            R.jump_idx[(size_t)row * R.max_jumps + njumps] = idx;
                        }
                        njumps++;
                        st[sJumps]++;
                        r_thr = draw();
                        cold_start(ts, YC, h);
                        steps_in_segment = 0;
                        continue;
                    }
                }
            }
            while (gi < npts && P.times[gi] <= t) { record_grid(gi); gi++; }
        }
    traj_done:
        if (tid == 0) {
            st[sDraws] = (long long)s_stream.n;
            long long* so = R.stats + (size_t)row * NSTATS;
            for (int s = 0; s < NSTATS; ++s) so[s] = st[s];
            R.status[row] = rc;
            R.jump_count[row] = njumps;
            if (rc != kOk) {
                double* eo = R.err + (size_t)row * 4;
                eo[0] = err0; eo[1] = err1; eo[2] = err2; eo[3] = err3;
                if (rc == kErrBracket) R.err_r[row] = r_thr;
                atomicMin(R.first_fail, (unsigned long long)row);
            }
        }
        __syncthreads();
    }
}

}  // namespace qtm
