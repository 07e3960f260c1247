/* mcwf_oracle.h -- CPU restatement of the reference trajectory path
 * (TEST INFRASTRUCTURE / CPU BASELINE; see mcwf_oracle.c).  The structs
 * deliberately mirror include/qtm.h so the same host packing feeds both. */
#ifndef MCWF_ORACLE_H
#define MCWF_ORACLE_H
#include <stdint.h>

#define MO_LROWS 13     /* Adams max order 12 + 1 (ode.py:46, 189-190) */
#define MO_MAX_OPS 64
#define MO_BDF_MAX_ORDER 6 /* ode.py:46 */

enum {
    MO_STREAM_PHILOX = 0,
    MO_STREAM_LFSR113 = 1,
    MO_STREAM_SCRIPTED = 2,
};

/* error codes; the host maps them onto the reference exception types */
enum {
    MO_OK = 0,
    MO_ERR_MAX_STEPS = -1,        /* OdeFailure(-1), trajectory.py:226-228 */
    MO_ERR_REPEATED_ERRTEST = -4, /* OdeFailure(-4), ode.py:297-298 */
    MO_ERR_STEP_COLLAPSE = -5,    /* OdeFailure(-5), ode.py:266-267 */
    MO_ERR_CORRECTOR = -6,        /* OdeFailure(-5), ode.py:310-311 */
    MO_ERR_BRACKET = -10,         /* RuntimeError, trajectory.py:166-169 */
    MO_ERR_NO_SUPPORT = -11,      /* ValueError, trajectory.py:143-144 */
    MO_ERR_ZERO_VECTOR = -12,     /* ValueError, trajectory.py:126-127 */
    MO_ERR_ARGS = -20,
};

enum {
    MO_STAT_ATTEMPTS = 0, MO_STAT_STEPS, MO_STAT_CORR_FAIL, MO_STAT_ERR_REJECT, MO_STAT_NFE,
    MO_STAT_CORR_ITERS, MO_STAT_JUMPS, MO_STAT_BISECT, MO_STAT_SUM_Q, MO_STAT_ORDER_UP,
    MO_STAT_ORDER_DOWN, MO_STAT_DRAWS, MO_STAT_LU_FACTOR = 14, MO_NSTATS = 16
};

typedef struct {
    const int64_t* row_ptr;
    const int64_t* col_ind;
    const double* values; /* interleaved (re, im) */
    int64_t nnz;
} mo_csr;

typedef struct {
    int64_t dim;
    mo_csr g;
    int32_t n_collapse;
    const mo_csr* collapse;
    int32_t n_expect;
    const mo_csr* expect;
    const double* psi0; /* interleaved */
    double t_from, t_to;
    int64_t n_steps;
    const double* times; /* n_steps + 1, np.linspace */
    double rtol, atol;
    int32_t max_order;
    int64_t max_steps;
    double h0_first;        /* first-segment step: initial_step or the host auto step */
    const double* l_table;  /* [MO_LROWS][MO_LROWS], row q = Adams l-vector (ode.py:90-121) */
    const double* tau1;     /* [MO_LROWS] */
    const double* tau2;
    const double* tau3;
    int32_t method;         /* 0 = ADAMS (numba kernel path), 1 = BDF (modified Newton, dense LU) */
    /* time-dependent right side G(t) = G + sum_k c_k(t) G_k with
     * c_k(t) = offset + amp cos(omega t + phase)  (paper_1810_03047_b200/timedep.py) */
    int32_t n_td;
    const mo_csr* td;
    const double* td_coef;  /* [n_td][4]: amp, omega, phase, offset */
} mo_problem;

enum { MO_METHOD_ADAMS = 0, MO_METHOD_BDF = 1 };

typedef struct {
    uint64_t seed;
    int64_t traj_begin, traj_end; /* global trajectory indices [begin, end) */
    int32_t stream_kind;
    const double* script;         /* scripted: [count][script_stride] */
    const int64_t* script_len;
    int64_t script_stride;
    double script_fallback;
    int64_t max_jumps;            /* jump-log capacity per trajectory */
    int32_t n_threads;
    int32_t n_psi_points;         /* psi snapshots at these grid indices (0 = none) */
    const int64_t* psi_points;
} mo_run_args;

typedef struct {
    int32_t code;
    int64_t traj;
    double t, h;
    int64_t max_steps;
    double aux0, aux1, aux2;
} mo_error;

typedef struct {
    double* values;      /* [count][n_expect][n_steps+1] */
    int64_t* stats;      /* [count][MO_NSTATS] */
    int32_t* status;     /* [count] or NULL */
    int64_t* jump_count; /* [count] or NULL */
    double* jump_t;      /* [count][max_jumps] or NULL */
    int32_t* jump_idx;   /* [count][max_jumps] or NULL */
    mo_error error;      /* first failing trajectory (lowest index) */
    double* psi;         /* [count][n_psi_points][2*dim] or NULL */
} mo_run_out;

int mo_run(const mo_problem* P, const mo_run_args* A, mo_run_out* O);
void mo_lfsr113_derive(uint64_t seed, uint64_t index, uint32_t z[4]);
double mo_philox_u01(uint64_t seed, uint64_t k, uint64_t n);
void mo_csr_matvec(const mo_csr* m, int64_t n, const double* x, double* out);

#endif
