"""Insert the QTM_PHASES instrumentation into qtm_traj.cuh (idempotent helper
used while the kernel was being restructured)."""
import sys
path = sys.argv[1]
s = open(path).read()
if "PH_MARK" in s:
    sys.exit(0)
def rep(a, b):
    global s
    assert a in s, a[:80]
    s = s.replace(a, b)
rep("""    unsigned long long* counter;
    unsigned long long* first_fail;  // atomicMin over failing rows
};""", """    unsigned long long* counter;
    unsigned long long* first_fail;  // atomicMin over failing rows
    unsigned long long* phase_cycles;  // [16] (QTM_PHASES builds only)
};""")
rep("#define STAT(which, amount) do { if (tid == 0) s_stats[which] += (amount); } while (0)",
"""#define STAT(which, amount) do { if (tid == 0) s_stats[which] += (amount); } while (0)
// Phase timing (profiling builds with -DQTM_PHASES): thread 0 attributes
// clock64() deltas to the phases of the attempt loop.
#ifdef QTM_PHASES
#define PH_MARK(k)                                                           \\
    do {                                                                     \\
        if (tid == 0) {                                                      \\
            const long long now__ = clock64();                               \\
            ph_acc[k] += now__ - ph_last;                                    \\
            ph_last = now__;                                                 \\
        }                                                                    \\
    } while (0)
#else
#define PH_MARK(k) do { } while (0)
#endif""")
rep("""        unsigned c_att = 0, c_q = 0, c_qq = 0, c_it = 0, c_steps = 0;
""", """        unsigned c_att = 0, c_q = 0, c_qq = 0, c_it = 0, c_steps = 0;
#ifdef QTM_PHASES
        long long ph_acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        long long ph_last = clock64();
#endif
""")
rep("""                for (;;) {
                    if (t + h == t) FAIL(kErrStepCollapse);
                    c_att++;""", """                for (;;) {
                    PH_MARK(0);  // [0] step-level work since the last mark
                    if (t + h == t) FAIL(kErrStepCollapse);
                    c_att++;""")
rep("""                        GATHER(y0p, xs0);
                    }""", """                        PH_MARK(1);  // [1] predict
                        GATHER(y0p, xs0);
                        PH_MARK(2);  // [2] gather z0 + barrier
                    }""")
rep("""                        double2 fg[E];
                        GSPMV(cur, fg);""", """                        double2 fg[E];
                        GSPMV(cur, fg);
                        PH_MARK(3);  // [3] SpMV""")
rep("""                        block_sum<NT, 3>(v, red, rphase);
                        if constexpr (NT == 32) __syncwarp();
                        gbuf ^= 1;""", """                        PH_MARK(4);  // [4] corrector update
                        block_sum<NT, 3>(v, red, rphase);
                        if constexpr (NT == 32) __syncwarp();
                        PH_MARK(5);  // [5] reduction
                        gbuf ^= 1;""")
rep("""                        delp = del;
                    }
                    if (converged) {""", """                        delp = del;
                        PH_MARK(6);  // [6] convergence control
                    }
                    PH_MARK(6);
                    if (converged) {""")
rep("""                // accepted step bookkeeping (ode.py:281-292)
                t_lo = t;""", """                PH_MARK(7);  // [7] error test + commit / undo + reject handling
                // accepted step bookkeeping (ode.py:281-292)
                t_lo = t;""")
rep("""                // ================= trajectory loop body (trajectory.py:225-246) =======
                steps_in_segment += 1;""", """                PH_MARK(8);  // [8] weights + order/step control
                // ================= trajectory loop body (trajectory.py:225-246) =======
                steps_in_segment += 1;""")
rep("""                while (gi < npts && P.times[gi] <= t) {
                    double2 pg[E];
                    HORNER((P.times[gi] - t) / h, pg);
                    RECORD(pg, gi);
                    gi++;
                }
            }
        }
    traj_done:""", """                PH_MARK(9);  // [9] jump test (+ jumps)
                while (gi < npts && P.times[gi] <= t) {
                    double2 pg[E];
                    HORNER((P.times[gi] - t) / h, pg);
                    RECORD(pg, gi);
                    gi++;
                }
                PH_MARK(10);  // [10] grid recording
            }
        }
    traj_done:
#ifdef QTM_PHASES
        if (tid == 0)
            for (int k = 0; k < 12; ++k) atomicAdd(R.phase_cycles + k, (unsigned long long)ph_acc[k]);
#endif""")
s = s.replace("#undef STAT\n", "#undef STAT\n#undef PH_MARK\n")
open(path, "w").write(s)
