/*
 * mcwf_oracle.c -- CPU restatement of the reference quantum-trajectory hot
 * path.  TEST INFRASTRUCTURE / CPU BASELINE ONLY: the product path
 * (paper_1810_03047_b200/csrc) never links or calls this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's CPU leg may load it.
 *
 * It follows, statement by statement, the reference package `mcwf`
 * (/root/reference/pkg/src/mcwf, Python + numba):
 *   - csr_matvec / csr_quadform / vec_norm_sq ......... _kernels.py:19-49
 *   - nordsieck_eval / nordsieck_eval_norm_sq ......... _kernels.py:61-81
 *   - wrms_weighted / wrms_diff_weighted ............... _kernels.py:84-104
 *   - nordsieck_rescale ................................ _kernels.py:107-114
 *   - adams_csr_step (predict, functional corrector,
 *     error test, commit) .............................. _kernels.py:117-192
 *   - OdeSolver.__init__ cold start .................... ode.py:164-217
 *   - OdeSolver.step retry loop ........................ ode.py:261-312
 *   - _restart_order_one / _rescale .................... ode.py:314-329
 *   - _order_step_control .............................. ode.py:441-466
 *   - interpolate_at ................................... ode.py:470-479
 *   - locate_jump_time ................................. trajectory.py:157-182
 *   - apply_collapse ................................... trajectory.py:133-154
 *   - record / record_expectation ...................... trajectory.py:122-130, 206-214
 *   - run_single_trajectory ............................ trajectory.py:190-250
 *   Time-dependent right side (rhs_fn = a TimeDependentGenerator, run by the
 *   reference's general engine with the Adams functional corrector,
 *   ode.py:227-230, 334-377): every G y becomes G0 y + sum_k c_k(t) G_k y,
 *   evaluated at t (cold start, restart) or t + h (corrector), in the
 *   callable's order (timedep.py: G0 row sums, then + c_k * (G_k row) per k).
 *   BDF (method = MO_METHOD_BDF, the general engine with a CSR generator):
 *   - _attempt_general (save, predict, Newton, error test,
 *     commit / restore) ................................. ode.py:334-356
 *   - _newton_correct (modified Newton, <= 3 iterations,
 *     one retry with a fresh iteration matrix) ......... ode.py:379-407
 *   - _ensure_iteration_matrix (refactor when |h l0 / h l0_fact - 1| > 0.3,
 *     stale, or no LU; M = I - h l0 J, J = G) ........... ode.py:409-423
 *   - scipy lu_factor / lu_solve = LAPACK zgetrf / zgetrs, restated as the
 *     unblocked right-looking LU with partial pivoting (pivot = first row of
 *     maximal |re| + |im|, izamax), row swaps, reciprocal scaling of the
 *     sub-column and the rank-1 update; then the row interchanges and the
 *     unit-lower / upper triangular solves (column-oriented, ztrsm order).
 *     OpenBLAS blocks the trailing update differently, so agreement with
 *     the reference is at the rounding level here, not bitwise.
 * with the same summation orders (rows left to right, components in index
 * order) and no FMA contraction (build with -ffp-contract=off, as numba's
 * default non-fastmath LLVM lowering).  Two places use numpy/BLAS in the
 * reference and are restated with a sequential order here: the weights
 * np.vdot(c psi, c psi) in apply_collapse (OpenBLAS zdotc, blocked) and the
 * normalisation `out /= sqrt(w)` which numpy performs as complex division
 * by (s + 0j), i.e. Smith's algorithm = multiply by 1/s.  The automatic
 * first step (ode.py:247-252, a BLAS dot) is computed by the host and
 * passed in as h0_first.
 *
 * Random streams (per trajectory, keyed by the global index k): Philox4x32-10,
 * the reference LFSR113 with derive_stream(seed, k) (rng.py:37-90), or a
 * scripted list with fallback (tests/oracles.py:60-72).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mcwf_oracle.h"

typedef struct { double re, im; } cplx;

/* ---- complex helpers in numba's operation order (numbers.py complex_mul) */
static inline cplx cmul(cplx a, cplx b) {
    cplx r;
    double ac = a.re * b.re, bd = a.im * b.im, ad = a.re * b.im, bc = a.im * b.re;
    r.re = ac - bd;
    r.im = ad + bc;
    return r;
}
static inline cplx cadd(cplx a, cplx b) { cplx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cplx csub(cplx a, cplx b) { cplx r = {a.re - b.re, a.im - b.im}; return r; }
/* real scalar times complex: numba/numpy promote the scalar to (s + 0j); the
 * zero cross terms only affect signs of zeros, so scale componentwise. */
static inline cplx cscale(double s, cplx a) { cplx r = {s * a.re, s * a.im}; return r; }
static inline double cabs2(cplx a) { return a.re * a.re + a.im * a.im; }
static inline double cabs_(cplx a) { return hypot(a.re, a.im); }
static inline double cabs1(cplx a) { return fabs(a.re) + fabs(a.im); }
/* a / b in numpy's order (Smith's algorithm, npymath complex divide) */
static inline cplx cdiv(cplx a, cplx b) {
    double abr = fabs(b.re), abi = fabs(b.im);
    cplx r;
    if (abr >= abi) {
        if (abr == 0.0 && abi == 0.0) { r.re = a.re / abr; r.im = a.im / abr; return r; }
        double rat = b.im / b.re, scl = 1.0 / (b.re + b.im * rat);
        r.re = (a.re + a.im * rat) * scl;
        r.im = (a.im - a.re * rat) * scl;
    } else {
        double rat = b.re / b.im, scl = 1.0 / (b.im + b.re * rat);
        r.re = (a.re * rat + a.im) * scl;
        r.im = (a.im * rat - a.re) * scl;
    }
    return r;
}

/* ---------------------------------------------------------------- streams */
#define M32 0xFFFFFFFFu

static void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint32_t lfsr113_next(uint32_t z[4]) {
    uint32_t b;
    b = ((z[0] << 6) ^ z[0]) >> 13;  z[0] = ((z[0] & 4294967294u) << 18) ^ b;
    b = ((z[1] << 2) ^ z[1]) >> 27;  z[1] = ((z[1] & 4294967288u) << 2) ^ b;
    b = ((z[2] << 13) ^ z[2]) >> 21; z[2] = ((z[2] & 4294967280u) << 7) ^ b;
    b = ((z[3] << 3) ^ z[3]) >> 12;  z[3] = ((z[3] & 4294967168u) << 13) ^ b;
    return z[0] ^ z[1] ^ z[2] ^ z[3];
}

static uint64_t splitmix_mix(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void mo_lfsr113_derive(uint64_t seed, uint64_t index, uint32_t z[4]) {
    const uint64_t golden = 0x9E3779B97F4A7C15ull;
    uint64_t x = seed ^ ((index + 1) * golden);
    static const uint32_t lo[4] = {1, 7, 15, 127};
    uint32_t w[4];
    for (int i = 0; i < 2; ++i) {
        x = splitmix_mix(x + golden);
        w[2 * i] = (uint32_t)x;
        w[2 * i + 1] = (uint32_t)(x >> 32);
    }
    for (int i = 0; i < 4; ++i) z[i] = w[i] <= lo[i] ? (w[i] | (lo[i] + 1)) : w[i];
    for (int i = 0; i < 16; ++i) lfsr113_next(z);
}

typedef struct {
    int kind;
    uint64_t seed, k, n;
    uint32_t lz[4];
    uint32_t block[4];
    const double* script;
    int64_t script_len;
    double fallback;
} stream_t;

static const double INV_2_32 = 2.3283064365386963e-10;

static void stream_init(stream_t* s, const mo_run_args* a, uint64_t k) {
    memset(s, 0, sizeof(*s));
    s->kind = a->stream_kind;
    s->seed = a->seed;
    s->k = k;
    if (s->kind == MO_STREAM_LFSR113) mo_lfsr113_derive(a->seed, k, s->lz);
    if (s->kind == MO_STREAM_SCRIPTED) {
        int64_t row = (int64_t)(k - (uint64_t)a->traj_begin);
        s->script = a->script + row * a->script_stride;
        s->script_len = a->script_len ? a->script_len[row] : 0;
        s->fallback = a->script_fallback;
    }
}

static double stream_next(stream_t* s) {
    uint64_t n = s->n++;
    if (s->kind == MO_STREAM_PHILOX) {
        if ((n & 3) == 0 || n == 0) {
            uint32_t ctr[4] = {(uint32_t)(n >> 2), (uint32_t)s->k, (uint32_t)(s->k >> 32), 0};
            uint32_t key[2] = {(uint32_t)s->seed, (uint32_t)(s->seed >> 32)};
            philox4x32_10(ctr, key, s->block);
        }
        return s->block[n & 3] * INV_2_32;
    }
    if (s->kind == MO_STREAM_LFSR113) return lfsr113_next(s->lz) * INV_2_32;
    return (int64_t)n < s->script_len ? s->script[n] : s->fallback;
}

double mo_philox_u01(uint64_t seed, uint64_t k, uint64_t n) {
    uint32_t ctr[4] = {(uint32_t)(n >> 2), (uint32_t)k, (uint32_t)(k >> 32), 0};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    philox4x32_10(ctr, key, out);
    return out[n & 3] * INV_2_32;
}

/* ----------------------------------------------------------- linear algebra */
static void csr_matvec(const mo_csr* m, const cplx* x, cplx* out, int64_t n) {
    const cplx* v = (const cplx*)m->values;
    for (int64_t i = 0; i < n; ++i) {
        cplx s = {0.0, 0.0};
        for (int64_t j = m->row_ptr[i]; j < m->row_ptr[i + 1]; ++j) s = cadd(s, cmul(v[j], x[m->col_ind[j]]));
        out[i] = s;
    }
}

/* out = G(t) x: the constant generator, then the time-dependent terms */
static double td_coef(const mo_problem* P, int k, double t) {
    const double* c = P->td_coef + 4 * k;
    return c[3] + c[0] * cos(c[1] * t + c[2]);
}

static void g_apply(const mo_problem* P, double t, const cplx* x, cplx* out, int64_t n) {
    csr_matvec(&P->g, x, out, n);
    for (int k = 0; k < P->n_td; ++k) {
        const double c = td_coef(P, k, t);
        const mo_csr* m = &P->td[k];
        const cplx* v = (const cplx*)m->values;
        for (int64_t i = 0; i < n; ++i) {
            cplx s = {0.0, 0.0};
            for (int64_t j = m->row_ptr[i]; j < m->row_ptr[i + 1]; ++j) s = cadd(s, cmul(v[j], x[m->col_ind[j]]));
            out[i] = cadd(out[i], cscale(c, s));
        }
    }
}

/* (<psi|M|psi>, <psi|psi>) -- _kernels.py:30-41 */
static void csr_quadform(const mo_csr* m, const cplx* psi, int64_t n, cplx* acc_out, double* nrm_out) {
    const cplx* v = (const cplx*)m->values;
    cplx acc = {0.0, 0.0};
    double nrm = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        cplx s = {0.0, 0.0};
        for (int64_t j = m->row_ptr[i]; j < m->row_ptr[i + 1]; ++j) s = cadd(s, cmul(v[j], psi[m->col_ind[j]]));
        cplx cj = {psi[i].re, -psi[i].im};
        acc = cadd(acc, cmul(cj, s));
        nrm += psi[i].re * psi[i].re + psi[i].im * psi[i].im;
    }
    *acc_out = acc;
    *nrm_out = nrm;
}

static double vec_norm_sq(const cplx* v, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i].re * v[i].re + v[i].im * v[i].im;
    return s;
}

static void nordsieck_eval(const cplx* z, int64_t n, int nord, double s, cplx* out) {
    for (int64_t i = 0; i < n; ++i) {
        cplx acc = z[nord * n + i];
        for (int j = nord - 1; j >= 0; --j) acc = cadd(cscale(s, acc), z[j * n + i]);
        out[i] = acc;
    }
}

static double nordsieck_eval_norm_sq(const cplx* z, int64_t n, int nord, double s) {
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        cplx acc = z[nord * n + i];
        for (int j = nord - 1; j >= 0; --j) acc = cadd(cscale(s, acc), z[j * n + i]);
        total += acc.re * acc.re + acc.im * acc.im;
    }
    return total;
}

static double wrms_weighted(const cplx* v, const cplx* yref, int64_t n, double atol, double rtol) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double w = 1.0 / (atol + rtol * cabs_(yref[i]));
        acc += (v[i].re * v[i].re + v[i].im * v[i].im) * w * w;
    }
    return sqrt(acc / (double)n);
}

static double wrms_diff_weighted(const cplx* a, const cplx* b, const cplx* yref, int64_t n, double atol,
                                 double rtol) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        cplx d = csub(a[i], b[i]);
        double w = 1.0 / (atol + rtol * cabs_(yref[i]));
        acc += (d.re * d.re + d.im * d.im) * w * w;
    }
    return sqrt(acc / (double)n);
}

static void nordsieck_rescale(cplx* z, int64_t n, int nord, double ratio) {
    double f = 1.0;
    for (int j = 1; j <= nord; ++j) {
        f *= ratio;
        for (int64_t i = 0; i < n; ++i) z[j * n + i] = cscale(f, z[j * n + i]);
    }
}

/* ------------------------------------------------------------------ solver */
enum { STEP_OK = 0, STEP_CORRECTOR_FAIL = 1, STEP_ERROR_REJECT = 2 };
#define MAXCOR 3
#define BIAS_SAME 1.2
#define BIAS_DOWN 1.3
#define BIAS_UP 1.4

typedef struct {
    const mo_problem* P;
    int64_t n;
    double t, t_lo, h;
    int q;
    double crate;
    int ialth;
    int has_eprev;
    cplx *z, *zp, *e, *eprev, *ycur, *f, *psi, *work;
    /* BDF: saved history rows, predicted y and z1, Newton step, iteration
     * matrix LU (column-major n x n) with its pivots, squared weights */
    cplx *save, *ypred, *z1pred, *dy, *lu;
    int64_t* ipiv;
    double* w2;
    int has_lu, jac_stale;
    double hl0_fact;
    /* psi snapshots: slot per grid index (-1 = none) and this trajectory's output */
    const int32_t* psi_slot;
    cplx* psi_out;
    /* stats */
    int64_t* st;
} solver_t;

static const double* L(const mo_problem* P, int q) { return P->l_table + (int64_t)q * MO_LROWS; }

static double step_kernel(solver_t* S, int* status) {
    /* adams_csr_step, _kernels.py:117-192 */
    const mo_problem* P = S->P;
    int64_t n = S->n;
    int nord = S->q, Lr = nord + 1;
    cplx *z = S->z, *zp = S->zp, *e = S->e, *ycur = S->ycur, *f = S->f;
    const double* lvec = L(P, S->q);
    double tau2 = P->tau2[S->q];
    double conit = 0.5 / (S->q + 2);
    double h = S->h;
    const cplx* gv = (const cplx*)P->g.values;

    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < Lr; ++j) zp[j * n + i] = z[j * n + i];
    for (int r = 0; r < nord; ++r)
        for (int j = nord - 1; j >= r; --j)
            for (int64_t i = 0; i < n; ++i) zp[j * n + i] = cadd(zp[j * n + i], zp[(j + 1) * n + i]);

    double l0 = lvec[0];
    int converged = 0;
    double delp = 0.0, del = 0.0;
    for (int64_t i = 0; i < n; ++i) ycur[i] = zp[i];
    for (int m = 0; m < MAXCOR; ++m) {
        for (int64_t i = 0; i < n; ++i) {
            cplx s = {0.0, 0.0};
            for (int64_t j = P->g.row_ptr[i]; j < P->g.row_ptr[i + 1]; ++j)
                s = cadd(s, cmul(gv[j], ycur[P->g.col_ind[j]]));
            f[i] = s;
        }
        if (P->n_td) g_apply(P, S->t + S->h, ycur, f, n);  /* G(t_new) ycur */
        S->st[MO_STAT_NFE]++;
        S->st[MO_STAT_CORR_ITERS]++;
        del = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            cplx ei = csub(cscale(h, f[i]), zp[n + i]);
            cplx ynew = cadd(zp[i], cscale(l0, ei));
            cplx d = csub(ynew, ycur[i]);
            double wi = 1.0 / (P->atol + P->rtol * cabs_(z[i]));
            del += (d.re * d.re + d.im * d.im) * wi * wi;
            e[i] = ei;
            ycur[i] = ynew;
        }
        del = sqrt(del / (double)n);
        if (m > 0) {
            double a = 0.2 * S->crate, b = del / delp;
            S->crate = a > b ? a : b;  /* max(0.2*crate, del/delp) */
        }
        double mn = 1.5 * S->crate < 1.0 ? 1.5 * S->crate : 1.0;
        if (del * mn <= conit) { converged = 1; break; }
        if (m > 0 && del > 2.0 * delp) break;
        delp = del;
    }
    if (!converged) { *status = STEP_CORRECTOR_FAIL; return 0.0; }
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double wi = 1.0 / (P->atol + P->rtol * cabs_(z[i]));
        acc += (e[i].re * e[i].re + e[i].im * e[i].im) * wi * wi;
    }
    double est = sqrt(acc / (double)n) / tau2;
    if (est > 1.0) { *status = STEP_ERROR_REJECT; return est; }
    for (int j = 0; j < Lr; ++j) {
        double lj = lvec[j];
        for (int64_t i = 0; i < n; ++i) zp[j * n + i] = cadd(zp[j * n + i], cscale(lj, e[i]));
    }
    *status = STEP_OK;
    return est;
}

/* ------------------------------------------------------------ BDF engine */
/* M = I - hl0 G built from the CSR generator (ode.py:418-420: -hl0 * jac,
 * then += 1 on the diagonal), factored in place: column-major LU with
 * partial pivoting (zgetf2 order). */
static void bdf_factor(solver_t* S, double hl0) {
    const mo_problem* P = S->P;
    int64_t n = S->n;
    cplx* a = S->lu;
    const cplx* gv = (const cplx*)P->g.values;
    memset(a, 0, sizeof(cplx) * n * n);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = P->g.row_ptr[i]; j < P->g.row_ptr[i + 1]; ++j)
            a[P->g.col_ind[j] * n + i] = cscale(-hl0, gv[j]);
    for (int64_t i = 0; i < n; ++i) a[i * n + i].re += 1.0;
    for (int64_t k = 0; k < n; ++k) {
        cplx* ck = a + k * n;
        int64_t p = k;
        double best = cabs1(ck[k]);
        for (int64_t i = k + 1; i < n; ++i) {
            double v = cabs1(ck[i]);
            if (v > best) { best = v; p = i; }
        }
        S->ipiv[k] = p;
        if (ck[p].re != 0.0 || ck[p].im != 0.0) {
            if (p != k)
                for (int64_t j = 0; j < n; ++j) {
                    cplx t = a[j * n + k]; a[j * n + k] = a[j * n + p]; a[j * n + p] = t;
                }
            cplx one = {1.0, 0.0};
            cplx rcp = cdiv(one, ck[k]);
            for (int64_t i = k + 1; i < n; ++i) ck[i] = cmul(ck[i], rcp);
        }
        for (int64_t j = k + 1; j < n; ++j) {
            cplx* cj = a + j * n;
            cplx ukj = cj[k];
            for (int64_t i = k + 1; i < n; ++i) cj[i] = csub(cj[i], cmul(ck[i], ukj));
        }
    }
}

/* b <- M^{-1} b (zgetrs: row interchanges, unit-lower then upper solve) */
static void bdf_solve(solver_t* S, cplx* b) {
    int64_t n = S->n;
    const cplx* a = S->lu;
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = S->ipiv[k];
        if (p != k) { cplx t = b[k]; b[k] = b[p]; b[p] = t; }
    }
    for (int64_t k = 0; k < n; ++k) {
        cplx bk = b[k];
        if (bk.re == 0.0 && bk.im == 0.0) continue;
        for (int64_t i = k + 1; i < n; ++i) b[i] = csub(b[i], cmul(bk, a[k * n + i]));
    }
    for (int64_t k = n - 1; k >= 0; --k) {
        if (b[k].re == 0.0 && b[k].im == 0.0) continue;
        b[k] = cdiv(b[k], a[k * n + k]);
        cplx bk = b[k];
        for (int64_t i = 0; i < k; ++i) b[i] = csub(b[i], cmul(bk, a[k * n + i]));
    }
}

static double wrms_w2(const cplx* v, const double* w2, int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += (v[i].re * v[i].re + v[i].im * v[i].im) * w2[i];
    return sqrt(acc / (double)n);
}

/* _attempt_general with the BDF corrector, ode.py:334-356, 379-423 */
static double step_bdf(solver_t* S, int* status) {
    const mo_problem* P = S->P;
    int64_t n = S->n;
    int q = S->q;
    cplx* z = S->z;
    const double* lvec = L(P, q);
    const double l0 = lvec[0], conit = 0.5 / (q + 2), h = S->h;
    const cplx* gv = (const cplx*)P->g.values;
    for (int64_t i = 0; i < n; ++i) {
        double w = 1.0 / (P->atol + P->rtol * cabs_(z[i]));
        S->w2[i] = w * w;
    }
    memcpy(S->save, z, sizeof(cplx) * n * (q + 1));
    for (int r = 0; r < q; ++r)
        for (int j = q - 1; j >= r; --j)
            for (int64_t i = 0; i < n; ++i) z[j * n + i] = cadd(z[j * n + i], z[(j + 1) * n + i]);
    memcpy(S->ypred, z, sizeof(cplx) * n);
    memcpy(S->z1pred, z + n, sizeof(cplx) * n);
    int converged = 0;
    for (int attempt = 0; attempt < 2 && !converged; ++attempt) {
        /* _ensure_iteration_matrix */
        const double hl0 = h * l0;
        if (!(S->has_lu && !S->jac_stale && fabs(hl0 / S->hl0_fact - 1.0) <= 0.3)) {
            S->jac_stale = 0;
            bdf_factor(S, hl0);
            S->st[MO_STAT_LU_FACTOR]++;
            S->has_lu = 1;
            S->hl0_fact = hl0;
            S->crate = 0.7;
        }
        memcpy(S->ycur, S->ypred, sizeof(cplx) * n);
        double delp = 0.0;
        for (int m = 0; m < MAXCOR; ++m) {
            cplx* f = S->f;
            for (int64_t i = 0; i < n; ++i) {
                cplx s = {0.0, 0.0};
                for (int64_t j = P->g.row_ptr[i]; j < P->g.row_ptr[i + 1]; ++j)
                    s = cadd(s, cmul(gv[j], S->ycur[P->g.col_ind[j]]));
                f[i] = s;
            }
            S->st[MO_STAT_NFE]++;
            /* resid = ycur - l0 * (h f - z1pred) - ypred, left to right */
            for (int64_t i = 0; i < n; ++i)
                S->dy[i] = csub(csub(S->ycur[i], cscale(l0, csub(cscale(h, f[i]), S->z1pred[i]))), S->ypred[i]);
            bdf_solve(S, S->dy);
            for (int64_t i = 0; i < n; ++i) {
                S->dy[i].re = -S->dy[i].re;
                S->dy[i].im = -S->dy[i].im;
                S->ycur[i] = cadd(S->ycur[i], S->dy[i]);
            }
            S->st[MO_STAT_CORR_ITERS]++;
            double del = wrms_w2(S->dy, S->w2, n);
            if (m > 0) {
                double a = 0.2 * S->crate, b = del / delp;
                S->crate = b > a ? b : a;  /* Python max(a, b) */
            }
            double c15 = 1.5 * S->crate;
            if (del * (c15 < 1.0 ? c15 : 1.0) <= conit) { converged = 1; break; }
            if (m > 0 && del > 2.0 * delp) break;
            delp = del;
        }
        if (converged) break;
        if (!S->jac_stale && attempt == 0) {
            /* retry once with a fresh iteration matrix */
            S->jac_stale = 1;
            S->has_lu = 0;
            continue;
        }
        break;
    }
    if (!converged) {
        memcpy(z, S->save, sizeof(cplx) * n * (q + 1));
        *status = STEP_CORRECTOR_FAIL;
        return 0.0;
    }
    /* e = (ycur - ypred) / l0: numpy divides by (l0 + 0j), i.e. times 1/l0 */
    const double rl0 = 1.0 / l0;
    for (int64_t i = 0; i < n; ++i) S->e[i] = cscale(rl0, csub(S->ycur[i], S->ypred[i]));
    double est = wrms_w2(S->e, S->w2, n) / P->tau2[q];
    if (est > 1.0) {
        memcpy(z, S->save, sizeof(cplx) * n * (q + 1));
        *status = STEP_ERROR_REJECT;
        return est;
    }
    for (int j = 0; j <= q; ++j) {
        double lj = lvec[j];
        for (int64_t i = 0; i < n; ++i) z[j * n + i] = cadd(z[j * n + i], cscale(lj, S->e[i]));
    }
    *status = STEP_OK;
    return est;
}

static void solver_rescale(solver_t* S, double r) {
    nordsieck_rescale(S->z, S->n, S->q, r);
    S->h *= r;
    S->has_eprev = 0;
    S->ialth = S->q + 1;
}

static void solver_restart_order_one(solver_t* S, double r) {
    S->q = 1;
    S->h *= r;
    S->has_lu = 0;
    g_apply(S->P, S->t, S->z, S->f, S->n);
    S->st[MO_STAT_NFE]++;
    for (int64_t i = 0; i < S->n; ++i) S->z[S->n + i] = cscale(S->h, S->f[i]);
    S->has_eprev = 0;
    S->ialth = S->q + 1;
}

static void solver_cold_start(solver_t* S, double t0, const cplx* y0, double h0) {
    /* OdeSolver.__init__, ode.py:164-217 (h0 is the hint or the host auto step) */
    int64_t n = S->n;
    S->t = t0;
    S->t_lo = t0;
    S->q = 1;
    memset(S->z, 0, sizeof(cplx) * n * MO_LROWS);
    for (int64_t i = 0; i < n; ++i) S->z[i] = y0[i];
    g_apply(S->P, t0, y0, S->f, n);
    S->st[MO_STAT_NFE]++;
    S->h = h0;
    for (int64_t i = 0; i < n; ++i) S->z[n + i] = cscale(S->h, S->f[i]);
    S->crate = 0.7;
    S->ialth = S->q + 1;
    S->has_eprev = 0;
    S->has_lu = 0;
    S->jac_stale = 1;
}

static void order_step_control(solver_t* S, double est) {
    /* ode.py:441-466 */
    const mo_problem* P = S->P;
    int q = S->q;
    int64_t n = S->n;
    const cplx* yref = S->z;
    double r_same = 1.0 / (BIAS_SAME * pow(est, 1.0 / (q + 1)) + 1e-6);
    double r_down = 0.0, r_up = 0.0;
    if (q > 1) {
        double est_d = wrms_weighted(S->z + (int64_t)q * n, yref, n, P->atol, P->rtol) / P->tau1[q];
        r_down = 1.0 / (BIAS_DOWN * pow(est_d, 1.0 / q) + 1e-6);
    }
    if (q < P->max_order && S->has_eprev) {
        double est_u = wrms_diff_weighted(S->e, S->eprev, yref, n, P->atol, P->rtol) / P->tau3[q];
        r_up = 1.0 / (BIAS_UP * pow(est_u, 1.0 / (q + 2)) + 1e-6);
    }
    double best = r_same;  /* Python max(): first maximal argument */
    if (r_down > best) best = r_down;
    if (r_up > best) best = r_up;
    if (best < 1.1) {
        S->ialth = 3;
        memcpy(S->eprev, S->e, sizeof(cplx) * n);
        S->has_eprev = 1;
        return;
    }
    if (best == r_up) {
        double c = L(P, q)[q] / (q + 1);
        for (int64_t i = 0; i < n; ++i) S->z[(int64_t)(q + 1) * n + i] = cscale(c, S->e[i]);
        S->q = q + 1;
        S->st[MO_STAT_ORDER_UP]++;
    } else if (best == r_down) {
        S->q = q - 1;
        S->st[MO_STAT_ORDER_DOWN]++;
    }
    double r = best < 10.0 ? best : 10.0;
    solver_rescale(S, r > 0.1 ? r : 0.1);
}

/* OdeSolver.step, ode.py:261-312.  Returns 0 or a negative istate. */
static int solver_step(solver_t* S) {
    int nef = 0, ncf = 0;
    for (;;) {
        if (S->t + S->h == S->t) return MO_ERR_STEP_COLLAPSE;
        int status;
        S->st[MO_STAT_ATTEMPTS]++;
        S->st[MO_STAT_SUM_Q] += S->q;
        const int bdf = S->P->method == MO_METHOD_BDF;
        double est = bdf ? step_bdf(S, &status) : step_kernel(S, &status);
        if (status == STEP_OK) {
            if (!bdf) { cplx* tmp = S->z; S->z = S->zp; S->zp = tmp; }
            S->t_lo = S->t;
            S->t += S->h;
            S->st[MO_STAT_STEPS]++;
            S->ialth -= 1;
            if (S->ialth == 0) order_step_control(S, est);
            else { memcpy(S->eprev, S->e, sizeof(cplx) * S->n); S->has_eprev = 1; }
            return 0;
        }
        if (status == STEP_ERROR_REJECT) {
            S->st[MO_STAT_ERR_REJECT]++;
            nef += 1;
            if (nef >= 10) return MO_ERR_REPEATED_ERRTEST;
            if (nef >= 3) solver_restart_order_one(S, 0.1);
            else {
                double r = 1.0 / (BIAS_SAME * pow(est, 1.0 / (S->q + 1)) + 1e-6);
                r = r < 0.9 ? r : 0.9;
                solver_rescale(S, r > 0.1 ? r : 0.1);
            }
            continue;
        }
        S->st[MO_STAT_CORR_FAIL]++;
        ncf += 1;
        S->jac_stale = 1;  /* ode.py:308-309 */
        S->has_lu = 0;
        if (ncf >= 10) return MO_ERR_CORRECTOR;
        solver_rescale(S, 0.25);
    }
}

/* ------------------------------------------------------------- trajectory */
static int record(solver_t* S, const cplx* psi, int64_t gi, double* values) {
    const mo_problem* P = S->P;
    if (S->psi_slot && S->psi_slot[gi] >= 0)  /* the state record_expectation receives */
        memcpy(S->psi_out + (int64_t)S->psi_slot[gi] * S->n, psi, sizeof(cplx) * S->n);
    for (int k = 0; k < P->n_expect; ++k) {
        cplx num;
        double nrm;
        csr_quadform(&P->expect[k], psi, S->n, &num, &nrm);
        if (nrm == 0.0) return MO_ERR_ZERO_VECTOR;
        values[(int64_t)k * (P->n_steps + 1) + gi] = num.re / nrm;
    }
    return 0;
}

static int record_grid(solver_t* S, int64_t gi, double* values) {
    nordsieck_eval(S->z, S->n, S->q, (S->P->times[gi] - S->t) / S->h, S->psi);
    return record(S, S->psi, gi, values);
}

#define JUMP_REL_TOL 1e-9
#define JUMP_MAX_ITER 60

static int locate_jump_time(solver_t* S, double r, double t_lo, double t_hi, double* t_star, mo_error* err) {
    const cplx* z = S->z;
    int nord = S->q;
    double t_cur = S->t, h = S->h;
    double f_lo = nordsieck_eval_norm_sq(z, S->n, nord, (t_lo - t_cur) / h);
    double f_hi = nordsieck_eval_norm_sq(z, S->n, nord, (t_hi - t_cur) / h);
    double tol = JUMP_REL_TOL * r;
    if (f_lo < r - tol || f_hi > r + tol) {
        err->t = t_lo; err->h = t_hi; err->aux0 = f_lo; err->aux1 = f_hi; err->aux2 = r;
        return MO_ERR_BRACKET;
    }
    if (f_lo <= r + tol) { *t_star = t_lo; return 0; }
    double a = t_lo, b = t_hi;
    for (int it = 0; it < JUMP_MAX_ITER; ++it) {
        double mid = 0.5 * (a + b);
        double f_mid = nordsieck_eval_norm_sq(z, S->n, nord, (mid - t_cur) / h);
        S->st[MO_STAT_BISECT]++;
        if (fabs(f_mid - r) <= tol) { *t_star = mid; return 0; }
        if (f_mid > r) a = mid; else b = mid;
    }
    *t_star = 0.5 * (a + b);
    return 0;
}

static int apply_collapse(solver_t* S, const cplx* psi, double u, cplx* out, int* idx_out) {
    const mo_problem* P = S->P;
    int64_t n = S->n;
    double wts[MO_MAX_OPS];
    double dp = 0.0;
    for (int c = 0; c < P->n_collapse; ++c) {
        csr_matvec(&P->collapse[c], psi, S->work, n);
        double rr = 0.0, ii = 0.0;
        for (int64_t i = 0; i < n; ++i) { rr += S->work[i].re * S->work[i].re; ii += S->work[i].im * S->work[i].im; }
        wts[c] = rr + ii;
        dp += wts[c];  /* Python sum(): left to right from 0 */
    }
    if (dp <= 0.0) return MO_ERR_NO_SUPPORT;
    int idx = -1;
    for (int c = 0; c < P->n_collapse; ++c) if (wts[c] > 0.0) idx = c;
    double cum = 0.0;
    for (int c = 0; c < P->n_collapse; ++c) {
        cum += wts[c] / dp;
        if (wts[c] > 0.0 && cum >= u) { idx = c; break; }
    }
    csr_matvec(&P->collapse[idx], psi, out, n);
    double rr = 0.0, ii = 0.0;
    for (int64_t i = 0; i < n; ++i) { rr += out[i].re * out[i].re; ii += out[i].im * out[i].im; }
    double scl = 1.0 / sqrt(rr + ii);
    for (int64_t i = 0; i < n; ++i) out[i] = cscale(scl, out[i]);
    *idx_out = idx;
    return 0;
}

static int run_trajectory(solver_t* S, stream_t* rs, double* values, double* jt, int32_t* jidx,
                          int64_t max_jumps, int64_t* n_jumps, mo_error* err) {
    const mo_problem* P = S->P;
    int64_t n = S->n, n_pts = P->n_steps + 1;
    const cplx* psi0 = (const cplx*)P->psi0;
    int rc = record(S, psi0, 0, values);
    if (rc) return rc;
    double r = stream_next(rs);
    solver_cold_start(S, P->t_from, psi0, P->h0_first);
    int64_t gi = 1, steps_in_segment = 0;
    *n_jumps = 0;
    while (gi < n_pts) {
        rc = solver_step(S);
        if (rc) { err->t = S->t; err->h = S->h; return rc; }
        steps_in_segment += 1;
        if (steps_in_segment > P->max_steps) { err->t = S->t; err->h = S->h; return MO_ERR_MAX_STEPS; }
        if (P->n_collapse > 0 && vec_norm_sq(S->z, n) < r) {
            double t_star;
            rc = locate_jump_time(S, r, S->t_lo, S->t, &t_star, err);
            if (rc) return rc;
            if (t_star <= P->t_to) {
                while (gi < n_pts && P->times[gi] <= t_star) {
                    rc = record_grid(S, gi, values);
                    if (rc) return rc;
                    gi++;
                }
                /* interpolate_at(t_star), ode.py:470-479 (bracket holds by construction) */
                nordsieck_eval(S->z, n, S->q, (t_star - S->t) / S->h, S->psi);
                double u = stream_next(rs);
                int idx;
                rc = apply_collapse(S, S->psi, u, S->ycur, &idx);
                if (rc) return rc;
                if (*n_jumps < max_jumps) { jt[*n_jumps] = t_star; jidx[*n_jumps] = idx; }
                (*n_jumps)++;
                S->st[MO_STAT_JUMPS]++;
                r = stream_next(rs);
                memcpy(S->psi, S->ycur, sizeof(cplx) * n);
                solver_cold_start(S, t_star, S->psi, S->h);
                steps_in_segment = 0;
                continue;
            }
        }
        while (gi < n_pts && P->times[gi] <= S->t) {
            rc = record_grid(S, gi, values);
            if (rc) return rc;
            gi++;
        }
    }
    S->st[MO_STAT_DRAWS] += (int64_t)rs->n;
    return 0;
}

/* ------------------------------------------------------------------ driver */
typedef struct {
    const mo_problem* P;
    const mo_run_args* A;
    mo_run_out* O;
    const int32_t* psi_slot;
    int64_t next;
    int64_t first_fail;
    pthread_mutex_t mu;
} shared_t;

static void* worker(void* arg) {
    shared_t* sh = (shared_t*)arg;
    const mo_problem* P = sh->P;
    const mo_run_args* A = sh->A;
    mo_run_out* O = sh->O;
    int64_t n = P->dim, n_pts = P->n_steps + 1;
    solver_t S;
    memset(&S, 0, sizeof(S));
    S.P = P;
    S.n = n;
    const int bdf = P->method == MO_METHOD_BDF;
    cplx* mem = (cplx*)calloc((size_t)n * (3 * MO_LROWS + 11) + (bdf ? (size_t)n * n : 0), sizeof(cplx));
    S.z = mem; S.zp = S.z + n * MO_LROWS; S.e = S.zp + n * MO_LROWS; S.eprev = S.e + n;
    S.ycur = S.eprev + n; S.f = S.ycur + n; S.psi = S.f + n; S.work = S.psi + n;
    S.save = S.work + n; S.ypred = S.save + n * MO_LROWS; S.z1pred = S.ypred + n; S.dy = S.z1pred + n;
    S.lu = S.dy + n;
    S.ipiv = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    S.w2 = (double*)calloc((size_t)n, sizeof(double));
    for (;;) {
        pthread_mutex_lock(&sh->mu);
        int64_t row = sh->next++;
        pthread_mutex_unlock(&sh->mu);
        int64_t count = A->traj_end - A->traj_begin;
        if (row >= count) break;
        uint64_t k = (uint64_t)(A->traj_begin + row);
        stream_t rs;
        stream_init(&rs, A, k);
        int64_t* st = O->stats + row * MO_NSTATS;
        memset(st, 0, sizeof(int64_t) * MO_NSTATS);
        S.st = st;
        S.psi_slot = sh->psi_slot;
        S.psi_out = sh->psi_slot ? (cplx*)O->psi + row * (int64_t)A->n_psi_points * n : NULL;
        double* vals = O->values + row * (int64_t)P->n_expect * n_pts;
        int64_t nj = 0;
        mo_error err;
        memset(&err, 0, sizeof(err));
        int rc = run_trajectory(&S, &rs, vals, O->jump_t ? O->jump_t + row * A->max_jumps : NULL,
                                O->jump_idx ? O->jump_idx + row * A->max_jumps : NULL,
                                O->jump_t ? A->max_jumps : 0, &nj, &err);
        if (O->jump_count) O->jump_count[row] = nj;
        if (O->status) O->status[row] = rc;
        if (rc) {
            pthread_mutex_lock(&sh->mu);
            if (sh->first_fail < 0 || row < sh->first_fail) {
                sh->first_fail = row;
                err.code = rc;
                err.traj = (int64_t)k;
                err.max_steps = P->max_steps;
                O->error = err;
            }
            pthread_mutex_unlock(&sh->mu);
        }
    }
    free(mem);
    free(S.ipiv);
    free(S.w2);
    return NULL;
}

int mo_run(const mo_problem* P, const mo_run_args* A, mo_run_out* O) {
    if (P->dim < 1 || A->traj_end < A->traj_begin) return MO_ERR_ARGS;
    if (P->n_collapse > MO_MAX_OPS || P->n_expect > MO_MAX_OPS) return MO_ERR_ARGS;
    if (P->method != MO_METHOD_ADAMS && P->method != MO_METHOD_BDF) return MO_ERR_ARGS;
    if (P->method == MO_METHOD_BDF && P->max_order > MO_BDF_MAX_ORDER) return MO_ERR_ARGS;
    if (P->n_td < 0 || (P->n_td > 0 && (P->method != MO_METHOD_ADAMS || !P->td || !P->td_coef))) return MO_ERR_ARGS;
    shared_t sh;
    sh.P = P; sh.A = A; sh.O = O; sh.next = 0; sh.first_fail = -1;
    int32_t* slot = NULL;
    if (A->n_psi_points > 0 && A->psi_points && O->psi) {
        slot = (int32_t*)malloc(sizeof(int32_t) * (P->n_steps + 1));
        for (int64_t g = 0; g <= P->n_steps; ++g) slot[g] = -1;
        for (int32_t k = 0; k < A->n_psi_points; ++k)
            if (A->psi_points[k] >= 0 && A->psi_points[k] <= P->n_steps) slot[A->psi_points[k]] = k;
    }
    sh.psi_slot = slot;
    pthread_mutex_init(&sh.mu, NULL);
    memset(&O->error, 0, sizeof(O->error));
    int nt = A->n_threads > 0 ? A->n_threads : 1;
    if (nt == 1) worker(&sh);
    else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
        for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, worker, &sh);
        for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&sh.mu);
    free(slot);
    return sh.first_fail >= 0 ? O->error.code : 0;
}

/* single-step probes used by the oracle's unit tests ---------------------- */
void mo_csr_matvec(const mo_csr* m, int64_t n, const double* x, double* out) {
    csr_matvec(m, (const cplx*)x, (cplx*)out, n);
}
