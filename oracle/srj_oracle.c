/*
 * srj_oracle.c -- CPU restatement of the reference's weighted-Jacobi hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker ("oracle") for the
 * CUDA path in paper_1511_04292_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never calls it and has no CPU fallback.
 *
 * What it restates (reference = /root/reference/pkg/src/srj/grids.py):
 *   oracle_wj1/2/3   <- _wj1 (grids.py:331-348), _wj2 (:351-376), _wj3 (:379-408)
 *   oracle_solve     <- _iterate (:602-629) driven as srj_solve (:642-687)
 *   oracle_gs        <- _gs1 (grids.py:410-424), _gs2 (:426-448), _gs3 (:450-474): in-place
 *                       lexicographic Gauss-Seidel / SOR sweeps
 *   oracle_residual  <- GridProblem.residual_field (:249-266), reduced to
 *                       (sum r^2, max |r|) -- the L2 norm is this project's
 *                       addition (BASELINE north_star), not in the reference.
 *   nonlinear source -- NOT in the reference (claimed only in PAPER.md:31-32);
 *                       semantics defined in DESIGN.md section "Nonlinear source".
 *
 * Arithmetic contract (must stay bit-identical to numba's output for _wj*):
 *   r  = s - ((((c*uc + am0*u[i-1]) + ap0*u[i+1]) + am1*u[j-1]) + ap1*u[j+1])
 *        (3D appends  + am2*u[k-1]  then  + ap2*u[k+1]  inside the bracket)
 *   d  = (omega*r)/c ;  un = uc + d
 *   dmax/rmax use "if (|x| > m) m = |x|" so NaNs never enter the max.
 * Compile with -ffp-contract=off (no FMA contraction) -- see oracle/Makefile.
 *
 * Layout: the reference's own dense C-order arrays.  u/un carry one ghost layer
 * per face (shape n+2 per axis); s, c, lower[], upper[], act, kappa are
 * interior-shaped.  act may be NULL (all cells active).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OVERFLOW_LIMIT 1e300 /* grids.py:53 */

/* Nonlinear source s(psi) = kappa * psi^5 with a fixed multiplication order:
 * p2 = psi*psi ; p4 = p2*p2 ; s = kappa * (p4*psi).  kappa = 2*pi*rho is
 * precomputed by the caller. */
static inline double nl_source(double kappa, double psi) {
    double p2 = psi * psi;
    double p4 = p2 * p2;
    return kappa * (p4 * psi);
}

static inline void upd_max(double *m, double x) {
    double a = fabs(x);
    if (a > *m) *m = a;
}

/* ---------------------------------------------------------------- 1D */
static void wj1_rows(int64_t n0, const double *u, double *un, const double *s,
                     const double *kap, const double *c, const double *am0,
                     const double *ap0, const uint8_t *act, double omega,
                     double *dmax, double *rmax) {
    double dm = 0.0, rm = 0.0;
    for (int64_t i = 0; i < n0; ++i) {
        if (!act || act[i]) {
            double uc = u[i + 1];
            double si = kap ? nl_source(kap[i], uc) : s[i];
            double r = si - ((c[i] * uc + am0[i] * u[i]) + ap0[i] * u[i + 2]);
            double d = (omega * r) / c[i];
            un[i + 1] = uc + d;
            upd_max(&dm, d);
            upd_max(&rm, r);
        } else {
            un[i + 1] = u[i + 1];
        }
    }
    *dmax = dm;
    *rmax = rm;
}

/* ---------------------------------------------------------------- 2D */
static void wj2_row(int64_t i, int64_t n1, const double *u, double *un,
                    const double *s, const double *kap, const double *c,
                    const double *am0, const double *ap0, const double *am1,
                    const double *ap1, const uint8_t *act, double omega,
                    double *dm, double *rm) {
    const int64_t P = n1 + 2;
    const double *um = u + i * P;       /* row i-1 (ghost-indexed i)   */
    const double *uc_ = u + (i + 1) * P; /* row i                       */
    const double *up = u + (i + 2) * P;  /* row i+1                     */
    double *out = un + (i + 1) * P;
    for (int64_t j = 0; j < n1; ++j) {
        int64_t q = i * n1 + j;
        if (!act || act[q]) {
            double uc = uc_[j + 1];
            double si = kap ? nl_source(kap[q], uc) : s[q];
            double acc = c[q] * uc;
            acc = acc + am0[q] * um[j + 1];
            acc = acc + ap0[q] * up[j + 1];
            acc = acc + am1[q] * uc_[j];
            acc = acc + ap1[q] * uc_[j + 2];
            double r = si - acc;
            double d = (omega * r) / c[q];
            out[j + 1] = uc + d;
            upd_max(dm, d);
            upd_max(rm, r);
        } else {
            out[j + 1] = uc_[j + 1];
        }
    }
}

/* ---------------------------------------------------------------- 3D */
static void wj3_plane(int64_t i, int64_t n1, int64_t n2, const double *u,
                      double *un, const double *s, const double *kap,
                      const double *c, const double *const *lo,
                      const double *const *hi, const uint8_t *act, double omega,
                      double *dm, double *rm) {
    const int64_t P2 = n2 + 2;
    const int64_t PL = (n1 + 2) * P2;
    for (int64_t j = 0; j < n1; ++j) {
        const double *base = u + (i + 1) * PL + (j + 1) * P2;
        double *out = un + (i + 1) * PL + (j + 1) * P2;
        for (int64_t k = 0; k < n2; ++k) {
            int64_t q = (i * n1 + j) * n2 + k;
            if (!act || act[q]) {
                double uc = base[k + 1];
                double si = kap ? nl_source(kap[q], uc) : s[q];
                double acc = c[q] * uc;
                acc = acc + lo[0][q] * base[k + 1 - PL];
                acc = acc + hi[0][q] * base[k + 1 + PL];
                acc = acc + lo[1][q] * base[k + 1 - P2];
                acc = acc + hi[1][q] * base[k + 1 + P2];
                acc = acc + lo[2][q] * base[k];
                acc = acc + hi[2][q] * base[k + 2];
                double r = si - acc;
                double d = (omega * r) / c[q];
                out[k + 1] = uc + d;
                upd_max(dm, d);
                upd_max(rm, r);
            } else {
                out[k + 1] = base[k + 1];
            }
        }
    }
}

/* One weighted-Jacobi step; returns 0 or -1 on bad ndim.
 * lower/upper: arrays of ndim interior-shaped coefficient pointers.
 * s may be NULL when kappa (nonlinear) is given, and vice versa. */
int oracle_wj(int ndim, const int64_t *n, const double *u, double *un,
              const double *s, const double *kappa, const double *c,
              const double *const *lower, const double *const *upper,
              const uint8_t *act, double omega, double *dmax, double *rmax,
              int nthreads) {
    double dm = 0.0, rm = 0.0;
    if (ndim == 1) {
        wj1_rows(n[0], u, un, s, kappa, c, lower[0], upper[0], act, omega, &dm,
                 &rm);
    } else if (ndim == 2 || ndim == 3) {
#ifdef _OPENMP
        if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
#endif
        {
            double ldm = 0.0, lrm = 0.0;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
            for (int64_t i = 0; i < n[0]; ++i) {
                if (ndim == 2)
                    wj2_row(i, n[1], u, un, s, kappa, c, lower[0], upper[0],
                            lower[1], upper[1], act, omega, &ldm, &lrm);
                else
                    wj3_plane(i, n[1], n[2], u, un, s, kappa, c, lower, upper,
                              act, omega, &ldm, &lrm);
            }
#ifdef _OPENMP
#pragma omp critical
#endif
            {
                /* max is exact and order-free; NaN never enters (upd_max) */
                if (ldm > dm) dm = ldm;
                if (lrm > rm) rm = lrm;
            }
        }
    } else {
        return -1;
    }
    *dmax = dm;
    *rmax = rm;
    return 0;
}

/* One in-place lexicographic Gauss-Seidel/SOR sweep (_gs2 / _gs3): each cell
 * uses the already-updated values of its lower neighbours along every axis
 * and the old values of its upper neighbours.  Sequential by definition. */
int oracle_gs(int ndim, const int64_t *n, double *u, const double *s,
              const double *c, const double *const *lower,
              const double *const *upper, const uint8_t *act, double omega,
              double *dmax, double *rmax) {
    double dm = 0.0, rm = 0.0;
    if (ndim == 1) { /* _gs1, grids.py:410-424 */
        for (int64_t i = 0; i < n[0]; ++i) {
            if (act && !act[i]) continue;
            const double uc = u[i + 1];
            const double acc = c[i] * uc + lower[0][i] * u[i] + upper[0][i] * u[i + 2];
            const double r = s[i] - acc;
            const double d = omega * r / c[i];
            u[i + 1] = uc + d;
            upd_max(&dm, d);
            upd_max(&rm, r);
        }
    } else if (ndim == 2) {
        const int64_t n0 = n[0], n1 = n[1], w = n1 + 2;
        for (int64_t i = 0; i < n0; ++i)
            for (int64_t j = 0; j < n1; ++j) {
                const int64_t q = i * n1 + j;
                if (act && !act[q]) continue;
                const int64_t g = (i + 1) * w + (j + 1);
                const double uc = u[g];
                const double acc = c[q] * uc + lower[0][q] * u[g - w] +
                                   upper[0][q] * u[g + w] + lower[1][q] * u[g - 1] +
                                   upper[1][q] * u[g + 1];
                const double r = s[q] - acc;
                const double d = omega * r / c[q];
                u[g] = uc + d;
                upd_max(&dm, d);
                upd_max(&rm, r);
            }
    } else if (ndim == 3) {
        const int64_t n0 = n[0], n1 = n[1], n2 = n[2];
        const int64_t w = n2 + 2, pl = (n1 + 2) * w;
        for (int64_t i = 0; i < n0; ++i)
            for (int64_t j = 0; j < n1; ++j)
                for (int64_t k = 0; k < n2; ++k) {
                    const int64_t q = (i * n1 + j) * n2 + k;
                    if (act && !act[q]) continue;
                    const int64_t g = (i + 1) * pl + (j + 1) * w + (k + 1);
                    const double uc = u[g];
                    const double acc = c[q] * uc + lower[0][q] * u[g - pl] +
                                       upper[0][q] * u[g + pl] + lower[1][q] * u[g - w] +
                                       upper[1][q] * u[g + w] + lower[2][q] * u[g - 1] +
                                       upper[2][q] * u[g + 1];
                    const double r = s[q] - acc;
                    const double d = omega * r / c[q];
                    u[g] = uc + d;
                    upd_max(&dm, d);
                    upd_max(&rm, r);
                }
    } else {
        return -1;
    }
    *dmax = dm;
    *rmax = rm;
    return 0;
}

static int64_t field_len(int ndim, const int64_t *n) {
    int64_t t = 1;
    for (int a = 0; a < ndim; ++a) t *= (n[a] + 2);
    return t;
}

/* Run nsteps elementary steps of the schedule starting at step index `first`
 * (omega_k = weights[k mod m]).  u (ghosted) is updated in place (the final
 * iterate is copied back), norms[2*t] = dmax, norms[2*t+1] = rmax of step t
 * (un-normalised, as returned by _wj*).  If tol > 0 the loop applies the
 * reference stopping rule of _iterate (grids.py:613-628) to dmax/|omega| and
 * stops early; tol < 0 keeps only the overflow guard; tol == 0 runs all steps.  Returns the number of steps performed; *status = 0 exhausted,
 * 1 converged, 2 diverged (overflow guard), <0 error. */
int64_t oracle_run(int ndim, const int64_t *n, double *u, const double *s,
                   const double *kappa, const double *c,
                   const double *const *lower, const double *const *upper,
                   const uint8_t *act, const double *weights, int64_t m,
                   int64_t first, int64_t nsteps, double tol, double *norms,
                   int *status, int nthreads) {
    int64_t len = field_len(ndim, n);
    double *scratch = (double *)malloc(sizeof(double) * (size_t)len);
    if (!scratch) {
        *status = -2;
        return 0;
    }
    /* the copy seeds the scratch ghost frame, as _Sweeper does (grids.py:542) */
    memcpy(scratch, u, sizeof(double) * (size_t)len);
    double *a = u, *b = scratch;
    int64_t done = 0;
    *status = 0;
    for (int64_t t = 0; t < nsteps; ++t) {
        double omega = weights[(first + t) % m];
        double dm, rm;
        if (oracle_wj(ndim, n, a, b, s, kappa, c, lower, upper, act, omega, &dm,
                      &rm, nthreads) != 0) {
            *status = -1;
            break;
        }
        double *tmp = a;
        a = b;
        b = tmp;
        norms[2 * t] = dm;
        norms[2 * t + 1] = rm;
        done = t + 1;
        if (tol != 0.0) { /* tol < 0: divergence guard only */
            double metric = dm / fabs(omega); /* grids.py:684 */
            if (!isfinite(metric) || metric > ORACLE_OVERFLOW_LIMIT) {
                *status = 2;
                break;
            }
            if (tol > 0.0 && metric < tol) {
                *status = 1;
                break;
            }
        }
    }
    if (a != u) memcpy(u, a, sizeof(double) * (size_t)len);
    free(scratch);
    return done;
}

/* (sum r^2, max |r|) of r = s - A u over active cells, row-major order.
 * Order of the operator terms matches the sweep (grids.py:249-266 applies the
 * same association: center, then lower/upper per axis). */
int oracle_residual(int ndim, const int64_t *n, const double *u,
                    const double *s, const double *kappa, const double *c,
                    const double *const *lower, const double *const *upper,
                    const uint8_t *act, double *out) {
    double ss = 0.0, rm = 0.0;
    if (ndim == 2) {
        const int64_t n0 = n[0], n1 = n[1], P = n1 + 2;
        for (int64_t i = 0; i < n0; ++i)
            for (int64_t j = 0; j < n1; ++j) {
                int64_t q = i * n1 + j;
                if (act && !act[q]) continue;
                const double *b = u + (i + 1) * P + (j + 1);
                double uc = *b;
                double si = kappa ? nl_source(kappa[q], uc) : s[q];
                double acc = c[q] * uc;
                acc = acc + lower[0][q] * b[-P];
                acc = acc + upper[0][q] * b[P];
                acc = acc + lower[1][q] * b[-1];
                acc = acc + upper[1][q] * b[1];
                double r = si - acc;
                ss += r * r;
                upd_max(&rm, r);
            }
    } else if (ndim == 3) {
        const int64_t n0 = n[0], n1 = n[1], n2 = n[2];
        const int64_t P2 = n2 + 2, PL = (n1 + 2) * P2;
        for (int64_t i = 0; i < n0; ++i)
            for (int64_t j = 0; j < n1; ++j)
                for (int64_t k = 0; k < n2; ++k) {
                    int64_t q = (i * n1 + j) * n2 + k;
                    if (act && !act[q]) continue;
                    const double *b = u + (i + 1) * PL + (j + 1) * P2 + (k + 1);
                    double uc = *b;
                    double si = kappa ? nl_source(kappa[q], uc) : s[q];
                    double acc = c[q] * uc;
                    acc = acc + lower[0][q] * b[-PL];
                    acc = acc + upper[0][q] * b[PL];
                    acc = acc + lower[1][q] * b[-P2];
                    acc = acc + upper[1][q] * b[P2];
                    acc = acc + lower[2][q] * b[-1];
                    acc = acc + upper[2][q] * b[1];
                    double r = si - acc;
                    ss += r * r;
                    upd_max(&rm, r);
                }
    } else {
        return -1;
    }
    out[0] = ss;
    out[1] = rm;
    return 0;
}

int oracle_abi_version(void) { return 1; }
