// qtm_small.cuh -- one THREAD per trajectory for tiny states (d <= DMAX).
//
// For d = 2 (c1) the per-trajectory CTA of traj_kernel wastes 30 of its 32
// lanes and spends its attempts in warp butterflies and shuffles; the run is
// a latency chain of ~220 attempts per trajectory.  Here a thread owns a
// whole trajectory: the Nordsieck history z[0..12][0..DMAX) in registers
// (Hist<13, DMAX>: the same order-specialised code as traj_kernel), the
// operators staged densely in shared memory ([op][i][j], padded to DMAX;
// zero entries add exact zeros, so every row still sums in CSR column order,
// csr_matvec, _kernels.py:18-26), and every norm a sequential sum over the
// components in index order -- the reference's own order (_kernels.py,
// wrms_weighted / vec_norm_sq), not a tree.  No shuffles, no barriers, no
// shared controller state.
//
// `lanes` trajectories share a warp (RunParams.lanes, 1..32): fewer lanes
// per warp means less divergence between trajectories that take different
// branches (reject / accept / jump / record), more means fewer warps.
//
// Reference behaviour per attempt is traj_kernel's (qtm_traj.cuh), itself
// following _kernels.py:117-192, ode.py:261-329, 441-466 and
// trajectory.py:122-250; outputs use the same RunParams layout with one
// "warp" partial per recorded point, so finalize_records / the ensemble
// reductions are shared.
#pragma once
#include "qtm_traj.cuh"

namespace qtm {

template <int DMAX>
struct SmallKernel {
    // dense operators G, C_0.., E_0.. in shared memory
    __host__ __device__ static constexpr size_t op_bytes(int nc, int ne) {
        return sizeof(double2) * (size_t)(1 + nc + ne) * DMAX * DMAX;
    }
};

// y = M x for a dense DMAX x DMAX block (rows in column order)
template <int DMAX>
__device__ __forceinline__ void dense_mv(const double2* __restrict__ m, const double2 (&x)[DMAX],
                                         double2 (&y)[DMAX]) {
#pragma unroll
    for (int i = 0; i < DMAX; ++i) {
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
            const double2 v = m[i * DMAX + j];
            sr = sr + (v.x * x[j].x - v.y * x[j].y);
            si = si + (v.x * x[j].y + v.y * x[j].x);
        }
        y[i] = make_double2(sr, si);
    }
}

template <int DMAX>
__global__ void __launch_bounds__(128)
traj1_kernel(const __grid_constant__ DevProblem P, const __grid_constant__ RunParams R) {
    using H = Hist<LROWS, DMAX, DMAX>;
    extern __shared__ double2 smem[];
    const int nops = 1 + P.nc + P.ne;
    for (int i = threadIdx.x; i < nops * DMAX * DMAX; i += blockDim.x) smem[i] = P.small_ops[i];
    __syncthreads();
    const double2* const Gm = smem;
    const double2* const Cm = smem + DMAX * DMAX;
    const double2* const Em = smem + (1 + P.nc) * DMAX * DMAX;

    const int lane = threadIdx.x & 31;
    const int lanes = R.lanes;
    if (lane >= lanes) return;
    const long long row = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * lanes + lane;
    if (row >= R.n_traj) return;

    const int d = P.d;
    const int npts = P.n_pts;
    Stream st;
    st.init(R.stream_kind, R.seed, (uint64_t)(R.traj_begin + row),
            R.script ? R.script + row * R.script_stride : nullptr, R.script_len ? R.script_len[row] : 0,
            R.script_fallback);
    long long stats[NSTATS];
#pragma unroll
    for (int k = 0; k < NSTATS; ++k) stats[k] = 0;
    long long njumps = 0, steps_in_segment = 0;
    int rc = kOk;
    const typename H::O ovf{nullptr};  // 13 register rows: no overflow

    typename H::Z z;
    double2 eb[2][DMAX];  // e of this attempt / of the previous accepted step
    double w[DMAX];       // error weights 1/(atol + rtol |z0_i|)
    double t, h, t_lo, r_thr, crate;
    int q, ialth, ecur = 0, gi;
    bool has_eprev;
#define ACT1(e) ((e) < d)

    auto record = [&](const double2 (&psi)[DMAX], int g) {
        if (R.psi_slot) {
            const int sl = R.psi_slot[g];
            if (sl >= 0) {
                double2* const po = R.psi_out + ((size_t)row * R.n_psi + sl) * d;
#pragma unroll
                for (int e = 0; e < DMAX; ++e) if (ACT1(e)) po[e] = psi[e];
            }
        }
        double* const rp = R.rec_partial + ((size_t)row * npts + g) * (size_t)(P.ne + 1);
        double nrm = 0.0;
#pragma unroll
        for (int e = 0; e < DMAX; ++e) if (ACT1(e)) nrm += cabs2(psi[e]);
        for (int k = 0; k < P.ne; ++k) {
            double2 s[DMAX];
            dense_mv<DMAX>(Em + k * DMAX * DMAX, psi, s);
            double acc = 0.0;
#pragma unroll
            for (int e = 0; e < DMAX; ++e) if (ACT1(e)) acc += psi[e].x * s[e].x - (-psi[e].y) * s[e].y;
            rp[k] = acc;
        }
        rp[P.ne] = nrm;
    };
    auto weights = [&](const double2 (&y)[DMAX]) {
#pragma unroll
        for (int e = 0; e < DMAX; ++e) w[e] = ACT1(e) ? err_weight(P.atol, P.rtol, y[e]) : 0.0;
    };
    auto cold_start = [&](double t0, const double2 (&y0)[DMAX], double h0) {
        t = t0; t_lo = t; q = 1; h = h0;
        stats[sNfe] += 1;
        double2 f[DMAX];
        dense_mv<DMAX>(Gm, y0, f);
#pragma unroll
        for (int e = 0; e < DMAX; ++e) {
            z[0][e] = y0[e];
            z[1][e] = cscale(h, f[e]);
        }
        weights(y0);
        crate = 0.7; ialth = 2; has_eprev = false;
    };
    auto rescale = [&](double ratio) {
        H::rescale(z, ovf, q, ratio);
        h *= ratio;
        has_eprev = false;
        ialth = q + 1;
    };
    auto wrms = [&](const double2 (&v)[DMAX]) {
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < DMAX; ++e) if (ACT1(e)) s += cabs2(v[e]) * w[e] * w[e];
        return s;
    };
    auto norm_sq = [&](const double2 (&v)[DMAX]) {
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < DMAX; ++e) if (ACT1(e)) s += cabs2(v[e]);
        return s;
    };
    auto fail = [&](int code, double a, double b, double c, double dd) {
        rc = code;
        double* const eo = R.err + (size_t)row * 4;
        eo[0] = a; eo[1] = b; eo[2] = c; eo[3] = dd;
    };

    {
        double2 psi[DMAX];
#pragma unroll
        for (int e = 0; e < DMAX; ++e) psi[e] = ACT1(e) ? P.psi0[e] : make_double2(0.0, 0.0);
        record(psi, 0);
        r_thr = st.next();
        cold_start(P.t_from, psi, P.h0_first);
    }
    gi = 1;
    double t_next = npts > 1 ? P.times[1] : CUDART_INF;

    while (gi < npts) {
        // ================= OdeSolver.step() (ode.py:261-312) =================
        int nef = 0, ncf = 0;
        double est = 0.0, nrm2 = 0.0;
        for (;;) {
            if (t + h == t) { fail(kErrStepCollapse, t, h, 0.0, 0.0); goto done; }
            stats[sAttempts] += 1;
            stats[sSumQ] += q;
            stats[sSumQQ1] += q * (q + 1);
            H::predict(z, ovf, q);
            const double l0 = P.l[q][0];
            const double conit = P.conit[q];
            bool converged = false;
            double delp = 0.0, del = 0.0, acc_e = 0.0;
            double2 y[DMAX];
#pragma unroll
            for (int e = 0; e < DMAX; ++e) y[e] = z[0][e];
            for (int m = 0; m < 3; ++m) {
                stats[sCorrIters] += 1;
                double2 f[DMAX], yn[DMAX], dd[DMAX];
                dense_mv<DMAX>(Gm, y, f);
#pragma unroll
                for (int e = 0; e < DMAX; ++e) {
                    const double2 ei = csub(cscale(h, f[e]), z[1][e]);
                    eb[ecur][e] = ACT1(e) ? ei : make_double2(0.0, 0.0);
                    yn[e] = cadd(z[0][e], cscale(l0, ei));
                    dd[e] = csub(yn[e], y[e]);
                }
                del = sqrt(wrms(dd) * P.inv_d);
                acc_e = wrms(eb[ecur]);
                nrm2 = norm_sq(yn);
#pragma unroll
                for (int e = 0; e < DMAX; ++e) y[e] = yn[e];
                if (m > 0) {
                    const double a = 0.2 * crate, b = del / delp;
                    crate = b > a ? b : a;
                }
                const double c15 = 1.5 * crate;
                if (del * (c15 < 1.0 ? c15 : 1.0) <= conit) { converged = true; break; }
                if (m > 0 && del > 2.0 * delp) break;
                delp = del;
            }
            if (converged) {
                est = sqrt(acc_e * P.inv_d) * P.inv_tau2[q];
                if (!(est > 1.0)) {
                    H::commit(z, ovf, q, P.l[q], eb[ecur]);  // _kernels.py:187-191
                    break;
                }
            }
            H::undo(z, ovf, q);
            if (!converged) {
                stats[sCorrFail] += 1;
                if (++ncf >= 10) { fail(kErrCorrector, t, h, 0.0, 0.0); goto done; }
                rescale(0.25);
                continue;
            }
            stats[sErrReject] += 1;
            if (++nef >= 10) { fail(kErrRepeatedErrTest, t, h, 0.0, 0.0); goto done; }
            if (nef >= 3) {
                // _restart_order_one(0.1), ode.py:314-323
                q = 1;
                h *= 0.1;
                stats[sNfe] += 1;
                double2 y0c[DMAX], fr[DMAX];
#pragma unroll
                for (int e = 0; e < DMAX; ++e) y0c[e] = z[0][e];
                dense_mv<DMAX>(Gm, y0c, fr);
#pragma unroll
                for (int e = 0; e < DMAX; ++e) z[1][e] = cscale(h, fr[e]);
                has_eprev = false;
                ialth = q + 1;
            } else {
                const double rr = __drcp_rn(1.2 * ctl_pow(est, P.rq1[q]) + 1e-6);
                const double m1 = 0.9 < rr ? 0.9 : rr;
                rescale(m1 > 0.1 ? m1 : 0.1);
            }
        }
        // accepted step bookkeeping (ode.py:281-292)
        t_lo = t;
        t += h;
        stats[sSteps] += 1;
        {
            double2 z0[DMAX];
#pragma unroll
            for (int e = 0; e < DMAX; ++e) z0[e] = z[0][e];
            weights(z0);
        }
        ialth -= 1;
        if (ialth == 0) {
            // _order_step_control (ode.py:441-466)
            const bool need_d = q > 1;
            const bool need_u = q < P.max_order && has_eprev;
            double2 zq[DMAX], de[DMAX];
            H::row_all(z, ovf, q, zq);
#pragma unroll
            for (int e = 0; e < DMAX; ++e) de[e] = csub(eb[ecur][e], eb[ecur ^ 1][e]);
            const double est_d = sqrt(wrms(zq) * P.inv_d) * P.inv_tau1[q];
            const double est_u = sqrt(wrms(de) * P.inv_d) * P.inv_tau3[q];
            if (est > P.keep_same[q] && (!need_d || est_d > P.keep_down[q]) &&
                (!need_u || est_u > P.keep_up[q])) {
                ialth = 3;
                ecur ^= 1;  // e_prev = e
                has_eprev = true;
            } else {
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
                    ecur ^= 1;
                    has_eprev = true;
                } else {
                    if (best == r_up) {
                        const double cu = P.l[q][q] / (q + 1);
                        double2 nz[DMAX];
#pragma unroll
                        for (int e = 0; e < DMAX; ++e) nz[e] = ACT1(e) ? cscale(cu, eb[ecur][e]) : make_double2(0.0, 0.0);
                        H::set_row_all(z, ovf, q + 1, nz);
                        q = q + 1;
                        stats[sOrderUp] += 1;
                    } else if (best == r_down) {
                        q = q - 1;
                        stats[sOrderDown] += 1;
                    }
                    const double m1 = 10.0 < best ? 10.0 : best;
                    rescale(m1 > 0.1 ? m1 : 0.1);
                }
            }
        } else {
            ecur ^= 1;  // e_prev = e
            has_eprev = true;
        }
        // ================= trajectory loop body (trajectory.py:225-246) =======
        steps_in_segment += 1;
        if (steps_in_segment > P.max_steps) { fail(kErrMaxSteps, t, h, 0.0, 0.0); goto done; }
        if (P.nc > 0 && nrm2 < r_thr) {
            // locate_jump_time (trajectory.py:157-182)
            double2 a1[DMAX], a2[DMAX];
            H::horner(z, ovf, q, (t_lo - t) / h, a1);
            H::horner(z, ovf, q, (t - t) / h, a2);
            const double f_lo = norm_sq(a1), f_hi = norm_sq(a2);
            const double tol = 1e-9 * r_thr;
            if (f_lo < r_thr - tol || f_hi > r_thr + tol) {
                R.err_r[row] = r_thr;
                fail(kErrBracket, t_lo, t, f_lo, f_hi);
                goto done;
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
                    double2 am[DMAX];
                    H::horner(z, ovf, q, (mid - t) / h, am);
                    const double v = norm_sq(am);
                    stats[sBisect] += 1;
                    if (fabs(v - r_thr) <= tol) { ts = mid; found = true; break; }
                    if (v > r_thr) a = mid; else b = mid;
                }
                if (!found) ts = 0.5 * (a + b);
            }
            if (ts <= P.t_to) {
                while (t_next <= ts) {
                    double2 pg[DMAX];
                    H::horner(z, ovf, q, (t_next - t) / h, pg);
                    record(pg, gi);
                    gi++;
                    t_next = gi < npts ? P.times[gi] : CUDART_INF;
                }
                // psi(t*) and the collapse (trajectory.py:235-241, 133-154)
                double2 pst[DMAX];
                H::horner(z, ovf, q, (ts - t) / h, pst);
                const double u = st.next();
                double wts[MAXOPS];
                double dp = 0.0;
                for (int c = 0; c < P.nc; ++c) {
                    double2 cv[DMAX];
                    dense_mv<DMAX>(Cm + c * DMAX * DMAX, pst, cv);
                    wts[c] = norm_sq(cv);
                }
                for (int c = 0; c < P.nc; ++c) dp += wts[c];
                if (dp <= 0.0) { fail(kErrNoSupport, t, h, 0.0, 0.0); goto done; }
                int idx = 0;
                for (int c = 0; c < P.nc; ++c) if (wts[c] > 0.0) idx = c;
                double cum = 0.0;
                for (int c = 0; c < P.nc; ++c) {
                    cum += wts[c] / dp;
                    if (wts[c] > 0.0 && cum >= u) { idx = c; break; }
                }
                const double scl = 1.0 / sqrt(wts[idx]);
                double2 cv[DMAX];
                dense_mv<DMAX>(Cm + idx * DMAX * DMAX, pst, cv);
#pragma unroll
                for (int e = 0; e < DMAX; ++e) pst[e] = ACT1(e) ? cscale(scl, cv[e]) : make_double2(0.0, 0.0);
                if (njumps < R.max_jumps) {
                    R.jump_t[(size_t)row * R.max_jumps + njumps] = ts;
                    R.jump_idx[(size_t)row * R.max_jumps + njumps] = idx;
                }
                njumps++;
                stats[sJumps] += 1;
                r_thr = st.next();
                cold_start(ts, pst, h);
                steps_in_segment = 0;
                continue;
            }
        }
        while (t_next <= t) {
            double2 pg[DMAX];
            H::horner(z, ovf, q, (t_next - t) / h, pg);
            record(pg, gi);
            gi++;
            t_next = gi < npts ? P.times[gi] : CUDART_INF;
        }
    }
done:
    stats[sDraws] = (long long)st.n;
    stats[sNfe] += stats[sCorrIters];
    {
        long long* so = R.stats + (size_t)row * NSTATS;
#pragma unroll
        for (int s = 0; s < NSTATS; ++s) so[s] = stats[s];
    }
    R.status[row] = rc;
    R.jump_count[row] = njumps;
    if (rc != kOk) atomicMin(R.first_fail, (unsigned long long)row);
#undef ACT1
}

}  // namespace qtm
