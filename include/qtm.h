/*
 * qtm.h -- C ABI of the B200 quantum-trajectory engine (libqtm.so).
 *
 * Drop-in boundary for the reference's data-parallel trajectory loop.  The
 * reference (Python package `mcwf`, /root/reference/pkg/src/mcwf) has no
 * FFI; its seams are Python calls, and each entry point below replaces one:
 *
 *   qtm_problem_create   <- QuantumProblem / OdeSolver set-up: the CSR
 *                           generator G = -i H_eff (operators.py:116-126,
 *                           trajectory.py:46-103), collapse/expectation
 *                           operators, psi0, grid (trajectory.py:89-90) and
 *                           OdeConfig (ode.py:124-151) copied to HBM once.
 *   qtm_run              <- run_inline / run_worker's trajectory loop
 *                           (cluster.py:472-482, 395-427) over
 *                           run_single_trajectory (trajectory.py:190-250),
 *                           including the count-weighted reduction
 *                           average_trajectories (trajectory.py:253-273) in
 *                           the form of per-point sums and sums of squares.
 *   qtm_problem_destroy  <- end of the problem's lifetime.
 *
 * Both method families of OdeConfig run on the device: ADAMS (the numba
 * kernel path, _kernels.py:117-192) and BDF (the general engine's modified
 * Newton with a dense LU, ode.py:334-423).  A time-dependent right side
 * (QuantumProblem.rhs_fn, trajectory.py:61, 186) is accepted in the form
 * H(t) = H0 + sum_k c_k(t) H_k through the n_td/td/td_coef fields (ADAMS).
 *
 * Plain pointers and sizes only.  The caller owns every host buffer; the
 * problem handle owns the device copies.  A call blocks until its device
 * work is finished; calls on different handles/devices may run concurrently
 * from different host threads.  No callbacks.
 *
 * Error codes mirror the reference's failure modes (ode.py:53-62,
 * trajectory.py:126-169); the failing trajectory and its (t, h) come back in
 * qtm_error so the host can re-raise the same exception text.
 */
#ifndef QTM_H
#define QTM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QTM_ABI_VERSION 3   /* 2: BDF method, time-dependent terms; 3: per-block partial sums */
#define QTM_BLOCK 256     /* trajectories per fixed-order reduction block */
#define QTM_LROWS 13      /* Nordsieck rows: Adams order <= 12 (ode.py:46) */
#define QTM_MAX_OPS 32    /* collapse / expectation operators per problem */
#define QTM_NSTATS 16
#define QTM_MAX_TD_TERMS 8 /* time-dependent generator terms */

enum qtm_stream_kind { QTM_STREAM_PHILOX = 0, QTM_STREAM_LFSR113 = 1, QTM_STREAM_SCRIPTED = 2 };

enum qtm_status {
    QTM_OK = 0,
    QTM_ERR_MAX_STEPS = -1,         /* OdeFailure(-1)  trajectory.py:226-228 */
    QTM_ERR_REPEATED_ERRTEST = -4,  /* OdeFailure(-4)  ode.py:297-298 */
    QTM_ERR_STEP_COLLAPSE = -5,     /* OdeFailure(-5)  ode.py:266-267 */
    QTM_ERR_CORRECTOR = -6,         /* OdeFailure(-5)  ode.py:310-311 */
    QTM_ERR_BRACKET = -10,          /* RuntimeError    trajectory.py:166-169 */
    QTM_ERR_NO_SUPPORT = -11,       /* ValueError      trajectory.py:143-144 */
    QTM_ERR_ZERO_VECTOR = -12,      /* ValueError      trajectory.py:126-127 */
    QTM_ERR_ARGS = -20,             /* invalid arguments (see qtm_last_error) */
    QTM_ERR_CUDA = -21,             /* CUDA runtime failure (see qtm_last_error) */
    QTM_ERR_UNSUPPORTED = -22,      /* problem outside the device path */
};

/* per-trajectory counters (qtm_run_out.stats rows) */
enum qtm_stat {
    QTM_STAT_ATTEMPTS = 0, QTM_STAT_STEPS, QTM_STAT_CORR_FAIL, QTM_STAT_ERR_REJECT,
    QTM_STAT_NFE, QTM_STAT_CORR_ITERS, QTM_STAT_JUMPS, QTM_STAT_BISECT, QTM_STAT_SUM_Q,
    QTM_STAT_ORDER_UP, QTM_STAT_ORDER_DOWN, QTM_STAT_DRAWS, QTM_STAT_SUM_QQ1,
    QTM_STAT_OVERFLOW_ATTEMPTS, QTM_STAT_LU_FACTOR  /* BDF: factorisations of I - h l0 G */
};

/* Square complex CSR operator in the reference layout (linalg.py:43-60):
 * int64 row_ptr[n+1], int64 col_ind[nnz] strictly increasing per row,
 * values[2*nnz] = interleaved (re, im) float64. */
typedef struct {
    const int64_t* row_ptr;
    const int64_t* col_ind;
    const double* values;
    int64_t nnz;
} qtm_csr;

typedef struct {
    int32_t abi_version;       /* QTM_ABI_VERSION */
    int64_t dim;
    qtm_csr generator;         /* G = -i H_eff */
    int32_t n_collapse;
    const qtm_csr* collapse;   /* [n_collapse] */
    int32_t n_expect;
    const qtm_csr* expect;     /* [n_expect] */
    const double* psi0;        /* [2*dim] interleaved, unit norm */
    double t_from, t_to;
    int64_t n_steps;           /* grid has n_steps + 1 points */
    const double* times;       /* [n_steps+1]  np.linspace(t_from, t_to, n_steps+1) */
    int32_t method;            /* 0 = ADAMS (numba kernel path), 1 = BDF (modified Newton, ode.py:334-423) */
    double rtol, atol;
    int32_t max_order;         /* 1..12 (ADAMS), 1..6 (BDF) */
    int64_t max_steps;
    double h0_first;           /* first-segment step: initial_step or auto step (ode.py:199-203) */
    const double* l_table;     /* [13*13] l-vectors of the method, row q (ode.py:90-121) */
    const double* tau1;        /* [13] */
    const double* tau2;        /* [13] */
    const double* tau3;        /* [13] */
    int32_t device;            /* CUDA device ordinal */
    int32_t variant;           /* -1 = automatic kernel selection, else a qtm_variant index */
    /* Time-dependent right side (replaces QuantumProblem.rhs_fn for
     * H(t) = H0 + sum_k c_k(t) H_k, trajectory.py:61, 186; ADAMS only):
     * psi' = (G + sum_k c_k(t) G_k) psi with `generator` = G0 and
     * c_k(t) = offset + amp cos(omega t + phase).  n_td = 0: constant G. */
    int32_t n_td;              /* 0..QTM_MAX_TD_TERMS */
    const qtm_csr* td;         /* [n_td] G_k = -i H_k */
    const double* td_coef;     /* [n_td][4] amp, omega, phase, offset */
} qtm_problem_desc;

typedef struct qtm_problem qtm_problem;

typedef struct {
    uint64_t seed;
    int64_t traj_begin, traj_end;   /* GLOBAL trajectory indices [begin, end) */
    int32_t stream_kind;            /* enum qtm_stream_kind */
    const double* script;           /* scripted: [count][script_stride] host array */
    const int64_t* script_len;      /* scripted: [count] */
    int64_t script_stride;
    double script_fallback;
    int64_t max_jumps;              /* jump-log capacity per trajectory (0 = no log) */
    void* cuda_stream;              /* cudaStream_t or NULL for the handle's stream */
    /* psi snapshots: the (unnormalised, interpolated) state each trajectory
     * records at these grid indices -- the argument the reference passes to
     * record_expectation (trajectory.py:206-214) -- into qtm_run_out.psi */
    int32_t n_psi_points;           /* 0 = none */
    const int64_t* psi_points;      /* [n_psi_points] distinct grid indices */
} qtm_run_args;

typedef struct {
    int32_t code;
    int64_t traj;                   /* global index of the first failing trajectory */
    double t, h;
    int64_t max_steps;
    double aux0, aux1, aux2;        /* bracket: f_lo, f_hi, r */
} qtm_error;

/* Sums run over the trajectories that completed; a failing trajectory is
 * excluded and counted in n_failed, and the call returns the failure code of
 * the lowest failing index (details in `error`), like the reference's first
 * error.  The caller chooses whether to raise (reference behaviour) or keep
 * the average over the completed trajectories. */
typedef struct {
    double* sum;          /* [n_expect*(n_steps+1)]  sum over completed trajectories (required) */
    double* sumsq;        /* [n_expect*(n_steps+1)]  sum of squares (or NULL) */
    double* values;       /* [count][n_expect][n_steps+1] per trajectory (or NULL) */
    int64_t* stats;       /* [count][QTM_NSTATS] (or NULL) */
    int64_t* stats_total; /* [QTM_NSTATS] summed over trajectories (or NULL) */
    int32_t* status;      /* [count] (or NULL) */
    int64_t* jump_count;  /* [count] (or NULL) */
    double* jump_t;       /* [count][max_jumps] (or NULL) */
    int32_t* jump_idx;    /* [count][max_jumps] (or NULL) */
    qtm_error error;      /* filled when the call returns a trajectory failure */
    float kernel_ms;      /* device time of the trajectory kernel (CUDA events) */
    float total_ms;       /* device time of the whole call's device work */
    int32_t variant;      /* kernel variant that ran */
    int32_t grid;         /* CTAs launched */
    int64_t launches;     /* kernels launched by this call */
    int64_t n_failed;     /* trajectories that failed (excluded from the sums) */
    double* psi;          /* [count][n_psi_points][2*dim] interleaved (or NULL) */
    /* The ensemble sums are reduced in two fixed stages: per block of
     * QTM_BLOCK consecutive trajectories (in trajectory order), then over the
     * blocks in block order, sum = ((0 + b_0) + b_1) + ...  These are the
     * stage-1 block partials (block i = trajectories traj_begin + 256 i ...),
     * so shards that start on a block boundary can be combined by another
     * process into exactly the single-run sums (multi-GPU, run_sharded). */
    double* block_sum;    /* [ceil(count/QTM_BLOCK)][n_expect*(n_steps+1)] (or NULL) */
    double* block_sumsq;  /* same shape (or NULL) */
} qtm_run_out;

int qtm_problem_create(const qtm_problem_desc* desc, qtm_problem** out);
int qtm_run(qtm_problem* problem, const qtm_run_args* args, qtm_run_out* out);
void qtm_problem_destroy(qtm_problem* problem);
/* trajectories the problem's kernel variant keeps in flight on its device
 * (SMs x resident CTAs per SM): the persistent grid of a large run */
int qtm_max_resident(qtm_problem* problem, int32_t* ctas);
/* where the Nordsieck history lives for this problem's kernel variant: rows
 * held in registers, rows in shared memory (the rest spill to global
 * scratch), and the dynamic shared memory of one CTA */
int qtm_problem_layout(qtm_problem* problem, int32_t* reg_rows, int32_t* smem_rows,
                       int64_t* smem_bytes);

/* Device-resident variant for benchmarking: results stay on the device;
 * only the per-point sums are copied out.  Same semantics as qtm_run. */
int qtm_run_resident(qtm_problem* problem, const qtm_run_args* args, qtm_run_out* out);

const char* qtm_last_error(void);
int qtm_abi_version(void);
int qtm_num_variants(void);
/* describe kernel variant i: threads per trajectory CTA, components per
 * thread, register-resident Nordsieck rows */
int qtm_variant_info(int i, int32_t* threads, int32_t* comps, int32_t* reg_rows);
/* 1 if variant i was compiled with the time-dependent generator terms
 * (required when n_td > 0), 0 if not, < 0 on a bad index */
int qtm_variant_time_dependent(int i);
/* Nordsieck rows variant i keeps in Tensor Memory (rows 2..7 with the e
 * buffers: 6), 0 for register / shared-memory histories, < 0 on a bad index */
int qtm_variant_tmem_rows(int i);
/* one-thread-per-trajectory variants (csrc/qtm_small.cuh): the largest
 * state dimension (0 for the CTA-per-trajectory variants) and the
 * trajectories sharing a warp */
int qtm_variant_small(int i, int32_t* d_max, int32_t* lanes);
/* kernel variant a problem runs (-1: the BDF kernel) */
int qtm_problem_variant(qtm_problem* problem);
int qtm_device_count(void);
/* measured FP64 FMA throughput of `device` in TFLOP/s (2 flops per DFMA):
 * the denominator of the FP64 roofline fraction bench.py reports */
int qtm_measure_fp64_peak(int device, double* tflops);
/* measured FP64 tensor-core (DMMA m8n8k4) throughput of `device` in TFLOP/s:
 * the ceiling a dense H_eff path on the FP64 tensor pipe would have */
int qtm_measure_dmma_peak(int device, double* tflops);
/* per-phase clock64() totals of thread 0 of every CTA for the last qtm_run
 * (profiling builds compiled with -DQTM_PHASES; zeros otherwise) */
int qtm_phase_cycles(uint64_t* out16);

#ifdef __cplusplus
}
#endif
#endif
