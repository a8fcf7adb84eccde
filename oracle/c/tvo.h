/*
 * tvo.h -- plain C11 fp64 CPU ORACLE of the TV-Stokes overlapping-Schwarz dual iteration
 * (arXiv 2602.17494).  TEST INFRASTRUCTURE ONLY: nothing in the product path may link or call it
 * (see oracle/__init__.py).  It shares no code, table or constant with the CUDA library; the
 * calls mirror the library's boundary (SURVEY 8(b) "Oracle": tvo_step1 / tvo_step2 / tvo_denoise
 * with double and host pointers).  Citations P:<line> are PAPER.md lines; readings A1..A21 are
 * SURVEY 8(c) / DESIGN.md section 2.
 *
 * Conventions: row-major double arrays, row i (y) of n1 values, 0-based; vector fields as
 * contiguous planes (x-component first); step-1 duals as 4 planes p11 p12 p21 p22 on Omega~ =
 * (n2+1) x (n1+1); step-2 duals as 2 planes on Omega = n2 x n1.  layout = {m2, m1, overlap_y,
 * overlap_x} (readings A6-A8).  Fixed schedules (reading A10), warm start from the previous sweep's
 * local solution (A9), alpha = 1/lambda (A4).  `threads` > 1 runs the local solves of a sweep on
 * that many POSIX threads, one task per subdomain (the paper's threading); results do not
 * depend on it (the solutions are combined in subdomain order).
 * Return codes: 0 ok, 1 invalid argument, 2 layout error, 7 out of memory (as tvs_status).
 * stats = {primal energy, dual energy D(p), duality gap} of the returned solution (SURVEY C-13,
 * C-15).
 */
#ifndef TVO_H
#define TVO_H

#ifdef __cplusplus
extern "C" {
#endif

int tvo_step1(const double *d0, int n2, int n1, double delta, const int layout[4], int sweeps,
              int inner, double t, int threads, double *tau, double *p, double stats[3]);
int tvo_step2(const double *tau, const double *d0, int n2, int n1, double lambda,
              const int layout[4], int sweeps, int inner, double t, int threads, double *d,
              double *p, double stats[3]);
int tvo_denoise(const double *d0, int n2, int n1, double delta, double lambda, const int layout[4],
                const int it1[2], const int it2[2], double t, int threads, double *d, double *tau,
                double stats1[3], double stats2[3]);

/* operators and pieces, for the pins (tests/test_oracle_c.py) */
void tvo_grad(const double *u, int n2, int n1, double *out /* 2 planes */);
void tvo_div(const double *p /* 2 planes */, int n2, int n1, double *out);
int tvo_lap_pinv(const double *q, int n2, int n1, double *out);
int tvo_project(const double *w /* 2 planes */, int n2, int n1, double *out /* 2 planes */);
void tvo_tau0(const double *d0, int n2, int n1, double *tau /* 2 planes on Omega~ */);
int tvo_layout_range(int n, int m, int s, int k, int *lo, int *hi);
double tvo_layout_theta(int n, int m, int s, int k, int x);

#ifdef __cplusplus
}
#endif
#endif
