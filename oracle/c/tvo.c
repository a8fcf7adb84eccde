/*
 * tvo.c -- plain C11 fp64 CPU ORACLE (test infrastructure only; see tvo.h).  Written from
 * PAPER.md (P:<line>), step by step in the paper's order and notation, with no blocking, fusion
 * or reordering beyond the formulas: finite differences (section 4.1), the DCT-II
 * matrix and Delta^dagger, the projection P_K (Eq. formula:PKh), the overlapping
 * layout / partition of unity / coloring weight (section 6.1), Alg. 2 with the
 * localized inner loops Alg. 3 (step 2) and Alg. 5 (step 1) whose local
 * projection is the literal block-DCT sum of Eq. invLaplLowCapLong.
 * Dense products are plain triple loops (O(N^3)): slow on purpose, obviously correct.
 */
#define _DEFAULT_SOURCE   /* M_PI */
#include "tvo.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define IDX(i, j, n1) ((size_t)(i) * (size_t)(n1) + (size_t)(j))

/* ------------------------------------------------------------------ finite differences */

/* (D+_x u)_{i,j} = u_{i,j+1} - u_{i,j} for j < N1-1, 0 at the last column */
static void dplus_x(const double *u, int n2, int n1, double *o) {
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n1; ++j)
      o[IDX(i, j, n1)] = j < n1 - 1 ? u[IDX(i, j + 1, n1)] - u[IDX(i, j, n1)] : 0.0;
}
/* (D+_y u)_{i,j} = u_{i+1,j} - u_{i,j} for i < N2-1, 0 at the last row */
static void dplus_y(const double *u, int n2, int n1, double *o) {
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n1; ++j)
      o[IDX(i, j, n1)] = i < n2 - 1 ? u[IDX(i + 1, j, n1)] - u[IDX(i, j, n1)] : 0.0;
}
/* three-case backward difference: u_1 | u_j - u_{j-1} | -u_{N-1} */
static void dminus_x(const double *u, int n2, int n1, double *o) {
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n1; ++j) {
      double v;
      if (j == 0) v = u[IDX(i, 0, n1)];
      else if (j < n1 - 1) v = u[IDX(i, j, n1)] - u[IDX(i, j - 1, n1)];
      else v = -u[IDX(i, n1 - 2, n1)];
      o[IDX(i, j, n1)] = v;
    }
}
static void dminus_y(const double *u, int n2, int n1, double *o) {
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n1; ++j) {
      double v;
      if (i == 0) v = u[IDX(0, j, n1)];
      else if (i < n2 - 1) v = u[IDX(i, j, n1)] - u[IDX(i - 1, j, n1)];
      else v = -u[IDX(n2 - 2, j, n1)];
      o[IDX(i, j, n1)] = v;
    }
}

/* grad u = (D+_x u, D+_y u) (Eq. defGradDis) */
void tvo_grad(const double *u, int n2, int n1, double *out) {
  dplus_x(u, n2, n1, out);
  dplus_y(u, n2, n1, out + (size_t)n2 * n1);
}
/* div p = D-_x p_1 + D-_y p_2 (Eq. defDivDis) */
void tvo_div(const double *p, int n2, int n1, double *out) {
  const size_t pl = (size_t)n2 * n1;
  double *t = malloc(pl * sizeof(double));
  dminus_x(p, n2, n1, out);
  dminus_y(p + pl, n2, n1, t);
  for (size_t e = 0; e < pl; ++e) out[e] += t[e];
  free(t);
}
/* multigrad / multidiv act row-wise on 2x2 fields: planes p11 p12 p21 p22 */
static void multigrad(const double *u, int n2, int n1, double *out) {
  const size_t pl = (size_t)n2 * n1;
  tvo_grad(u, n2, n1, out);
  tvo_grad(u + pl, n2, n1, out + 2 * pl);
}
static void multidiv(const double *p, int n2, int n1, double *out) {
  const size_t pl = (size_t)n2 * n1;
  tvo_div(p, n2, n1, out);
  tvo_div(p + 2 * pl, n2, n1, out + pl);
}

/* tau_0 = (-D_y^{neum-} d_0, D_x^{neum-} d_0) on Omega~ (Eq. def:backdiffNeumann P:576-590):
 * D_x^{neum-}: 0 on the first / last column, d_{i,j} - d_{i,j-1} inside, extra row N2 mirrors row
 * N2-1; D_y^{neum-}: 0 on the first / last row, extra column N1 mirrors column N1-1. */
void tvo_tau0(const double *d0, int n2, int n1, double *tau) {
  const int g2 = n2 + 1, g1 = n1 + 1;
  double *t1 = tau, *t2 = tau + (size_t)g2 * g1;
  memset(tau, 0, 2 * (size_t)g2 * g1 * sizeof(double));
  for (int i = 0; i < g2; ++i)
    for (int j = 1; j < n1; ++j) {   /* D_x^{neum-} */
      const int r = i < n2 ? i : n2 - 1;
      t2[IDX(i, j, g1)] = d0[IDX(r, j, n1)] - d0[IDX(r, j - 1, n1)];
    }
  for (int i = 1; i < n2; ++i)
    for (int j = 0; j < g1; ++j) {   /* D_y^{neum-}, negated */
      const int c = j < n1 ? j : n1 - 1;
      t1[IDX(i, j, g1)] = -(d0[IDX(i, c, n1)] - d0[IDX(i - 1, c, n1)]);
    }
}

/* ------------------------------------------------------------------ spectral */

/* C_N of Eq. form:DCTmat: row k = sqrt(2/N) w_k cos(k (2j+1) pi / (2N)), w_0 = 1/sqrt 2 */
static double *dct_matrix(int n) {
  double *c = malloc((size_t)n * n * sizeof(double));
  if (!c) return NULL;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) {
      double v = sqrt(2.0 / n) * cos((double)k * (2.0 * j + 1.0) * M_PI / (2.0 * n));
      c[IDX(k, j, n)] = k == 0 ? v / sqrt(2.0) : v;
    }
  return c;
}
/* sigma_{N,k} = 2 sin(k pi / (2N)) (h = 1) */
static double sigma_nk(int n, int k) { return 2.0 * sin((double)k * M_PI / (2.0 * n)); }
/* (Delta~)^dagger_{ij} = -1/(sigma_{N2,i}^2 + sigma_{N1,j}^2), (0,0) -> 0; row i pairs with N2 and
 * column j with N1 (reading A2; the printed pairing fails the Penrose identities off-square) */
static double lam_ij(int n2, int n1, int i, int j) {
  const double d = sigma_nk(n2, i) * sigma_nk(n2, i) + sigma_nk(n1, j) * sigma_nk(n1, j);
  return (i == 0 && j == 0) || d == 0.0 ? 0.0 : -1.0 / d;
}

/* C[m x n] = A[m x k] B[k x n], plain loops */
static void matmul(const double *A, const double *B, double *C, int m, int n, int k) {
  for (int i = 0; i < m; ++i) {
    double *ci = C + (size_t)i * n;
    for (int j = 0; j < n; ++j) ci[j] = 0.0;
    for (int l = 0; l < k; ++l) {
      const double a = A[(size_t)i * k + l];
      const double *bl = B + (size_t)l * n;
      for (int j = 0; j < n; ++j) ci[j] += a * bl[j];
    }
  }
}
static double *transpose(const double *A, int m, int n) {
  double *T = malloc((size_t)m * n * sizeof(double));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) T[(size_t)j * m + i] = A[(size_t)i * n + j];
  return T;
}

/* (Delta)^dagger q = C^{-1} (Delta~)^dagger C q with C q = C_{N2} q C_{N1}^T (Eqs. form:DiscInvLapl
 * P:611-612, eq:DCT2D P:627-629, eq:DCT2Dinv P:649-651) */
int tvo_lap_pinv(const double *q, int n2, int n1, double *out) {
  double *c2 = dct_matrix(n2), *c1 = dct_matrix(n1);
  double *c1t = c1 ? transpose(c1, n1, n1) : NULL, *c2t = c2 ? transpose(c2, n2, n2) : NULL;
  double *a = malloc((size_t)n2 * n1 * sizeof(double)), *x = malloc((size_t)n2 * n1 * sizeof(double));
  if (!c2 || !c1 || !c1t || !c2t || !a || !x) return 7;
  matmul(c2, q, a, n2, n1, n2);       /* C_{N2} q */
  matmul(a, c1t, x, n2, n1, n1);      /* (C_{N2} q) C_{N1}^T */
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n1; ++j) x[IDX(i, j, n1)] *= lam_ij(n2, n1, i, j);
  matmul(c2t, x, a, n2, n1, n2);      /* C_{N2}^T Y */
  matmul(a, c1, out, n2, n1, n1);     /* (C_{N2}^T Y) C_{N1} */
  free(c2), free(c1), free(c1t), free(c2t), free(a), free(x);
  return 0;
}

/* P_{K^h} w = w - grad (Delta)^dagger div w (Eq. formula:PKh) */
int tvo_project(const double *w, int n2, int n1, double *out) {
  const size_t pl = (size_t)n2 * n1;
  double *q = malloc(pl * sizeof(double)), *phi = malloc(pl * sizeof(double));
  double *g = malloc(2 * pl * sizeof(double));
  if (!q || !phi || !g) return 7;
  tvo_div(w, n2, n1, q);
  int st = tvo_lap_pinv(q, n2, n1, phi);
  if (st) return st;
  tvo_grad(phi, n2, n1, g);
  for (size_t e = 0; e < 2 * pl; ++e) out[e] = w[e] - g[e];
  free(q), free(phi), free(g);
  return 0;
}

/* R_B (Delta)^dagger E_A q_A by the literal block-DCT sum of Eq. invLaplLowCapLong (
 * Lemma lmChainOp, Eq. locglobprojpart3): sum over frequency blocks
 * (lambda2, lambda1) of the core partitions cuts_y x cuts_x of
 *   ([C_{N2}]^{lambda2}_{B})^T ( (Delta~)^dagger on the block ) ([C_{N2}]^{A}_{lambda2} q
 *   ([C_{N1}]^{A}_{lambda1})^T ) [C_{N1}]^{lambda1}_{B}.
 * A = rows [ay0, ay1] x cols [ax0, ax1], B likewise (inclusive, on the n2 x n1 grid). */
static int lap_pinv_block(const double *qa, int ay0, int ay1, int ax0, int ax1, int by0, int by1,
                          int bx0, int bx1, int n2, int n1, const int *cy, int my, const int *cx,
                          int mx, const double *c2, const double *c1, double *out) {
  const int ar = ay1 - ay0 + 1, ac = ax1 - ax0 + 1, br = by1 - by0 + 1, bc = bx1 - bx0 + 1;
  memset(out, 0, (size_t)br * bc * sizeof(double));
  int fymax = 0, fxmax = 0;
  for (int l = 0; l < my; ++l) fymax = cy[l + 1] - cy[l] > fymax ? cy[l + 1] - cy[l] : fymax;
  for (int l = 0; l < mx; ++l) fxmax = cx[l + 1] - cx[l] > fxmax ? cx[l + 1] - cx[l] : fxmax;
  const int big = ar > br ? ar : br, bigc = ac > bc ? ac : bc;
  double *c2k = malloc((size_t)fymax * big * sizeof(double));    /* [C_{N2}]^{A}_{lambda2} */
  double *c2m = malloc((size_t)fymax * big * sizeof(double));    /* [C_{N2}]^{lambda2}_{B} */
  double *c1kt = malloc((size_t)bigc * fxmax * sizeof(double));  /* ([C_{N1}]^{A}_{lambda1})^T */
  double *c1m = malloc((size_t)fxmax * bigc * sizeof(double));   /* [C_{N1}]^{lambda1}_{B} */
  double *t1 = malloc((size_t)fymax * bigc * sizeof(double));
  double *blk = malloc((size_t)fymax * fxmax * sizeof(double));
  double *c2mt = malloc((size_t)big * fymax * sizeof(double));
  double *t2 = malloc((size_t)big * fxmax * sizeof(double));
  double *o = malloc((size_t)br * bc * sizeof(double));
  if (!c2k || !c2m || !c1kt || !c1m || !t1 || !blk || !c2mt || !t2 || !o) return 7;
  for (int l2 = 0; l2 < my; ++l2) {
    const int f0 = cy[l2], fy = cy[l2 + 1] - cy[l2];
    for (int r = 0; r < fy; ++r) {
      for (int c = 0; c < ar; ++c) c2k[(size_t)r * ar + c] = c2[IDX(f0 + r, ay0 + c, n2)];
      for (int c = 0; c < br; ++c) c2m[(size_t)r * br + c] = c2[IDX(f0 + r, by0 + c, n2)];
    }
    for (int l1 = 0; l1 < mx; ++l1) {
      const int g0 = cx[l1], fx = cx[l1 + 1] - cx[l1];
      for (int c = 0; c < ac; ++c)
        for (int r = 0; r < fx; ++r) c1kt[(size_t)c * fx + r] = c1[IDX(g0 + r, ax0 + c, n1)];
      for (int r = 0; r < fx; ++r)
        for (int c = 0; c < bc; ++c) c1m[(size_t)r * bc + c] = c1[IDX(g0 + r, bx0 + c, n1)];
      matmul(c2k, qa, t1, fy, ac, ar);     /* [C2]^A_l2 q_A */
      matmul(t1, c1kt, blk, fy, fx, ac);   /* ... ([C1]^A_l1)^T */
      for (int r = 0; r < fy; ++r)
        for (int c = 0; c < fx; ++c) blk[(size_t)r * fx + c] *= lam_ij(n2, n1, f0 + r, g0 + c);
      for (int r = 0; r < fy; ++r)
        for (int c = 0; c < br; ++c) c2mt[(size_t)c * fy + r] = c2m[(size_t)r * br + c];
      matmul(c2mt, blk, t2, br, fx, fy);   /* ([C2]^l2_B)^T blk */
      matmul(t2, c1m, o, br, bc, fx);      /* ... [C1]^l1_B */
      for (size_t e = 0; e < (size_t)br * bc; ++e) out[e] += o[e];
    }
  }
  free(c2k), free(c2m), free(c1kt), free(c1m), free(t1), free(blk), free(c2mt), free(t2), free(o);
  return 0;
}

/* ------------------------------------------------------------------ layout */

/* subdomain k of an axis of length n with m subdomains and overlap s: [c_k - floor(s/2),
 * c_{k+1} - 1 + ceil(s/2)] clipped, c_k = floor(k n / m) (readings A6, A8); -1 if invalid */
int tvo_layout_range(int n, int m, int s, int k, int *lo, int *hi) {
  if (m < 1 || n < 2 || m > n || k < 0 || k >= m) return 1;
  if (m > 1) {
    if (s < 1) return 2;
    for (int q = 0; q < m; ++q)
      if ((long long)(q + 1) * n / m - (long long)q * n / m <= s) return 2;   /* reading A17 */
  }
  long long a = (long long)k * n / m - (k > 0 ? s / 2 : 0);
  long long b = (long long)(k + 1) * n / m - 1 + (k < m - 1 ? (s + 1) / 2 : 0);
  *lo = a < 0 ? 0 : (int)a;
  *hi = b > n - 1 ? n - 1 : (int)b;
  return 0;
}
/* partition of unity (reading A7 of P:1303-1308): linear ramps over each shared band [L, R] */
double tvo_layout_theta(int n, int m, int s, int k, int x) {
  int lo, hi;
  if (tvo_layout_range(n, m, s, k, &lo, &hi)) return 0.0;
  if (x < lo || x > hi) return 0.0;
  if (k + 1 < m) {
    int l2, h2;
    tvo_layout_range(n, m, s, k + 1, &l2, &h2);
    if (x >= l2) return (double)(hi - x + 1) / (s + 1.0);
  }
  if (k > 0) {
    int l0, h0;
    tvo_layout_range(n, m, s, k - 1, &l0, &h0);
    if (x <= h0) return (double)(x - lo + 1) / (s + 1.0);
  }
  return 1.0;
}
static double alpha_hat(int m2, int m1) {   /* coloring relaxation */
  if (m1 == 1 && m2 == 1) return 1.0;
  if (m1 == 1 || m2 == 1) return 0.5;
  return 0.25;
}

/* one rectangle: rows [y0, y1] x cols [x0, x1] (inclusive) */
typedef struct {
  int y0, y1, x0, x1;
} rect;
static int rh(rect r) { return r.y1 - r.y0 + 1; }
static int rw(rect r) { return r.x1 - r.x0 + 1; }
/* A_+ (reading A12): one more row below and one more column right, clipped */
static rect rect_plus(rect r, int n2, int n1) {
  rect o = r;
  o.y1 = r.y1 + 1 < n2 - 1 ? r.y1 + 1 : n2 - 1;
  o.x1 = r.x1 + 1 < n1 - 1 ? r.x1 + 1 : n1 - 1;
  return o;
}
/* E_inner into outer (zero outside), `planes` planes */
static void extend(const double *a, rect in, rect out, int planes, double *o) {
  const int oh = rh(out), ow = rw(out), ih = rh(in), iw = rw(in);
  memset(o, 0, (size_t)planes * oh * ow * sizeof(double));
  for (int c = 0; c < planes; ++c)
    for (int i = 0; i < ih; ++i)
      for (int j = 0; j < iw; ++j)
        o[(size_t)c * oh * ow + IDX(in.y0 - out.y0 + i, in.x0 - out.x0 + j, ow)] =
            a[(size_t)c * ih * iw + IDX(i, j, iw)];
}
/* R_inner of arrays living on outer */
static void restrict_(const double *a, rect out, rect in, int planes, double *o) {
  const int oh = rh(out), ow = rw(out), ih = rh(in), iw = rw(in);
  for (int c = 0; c < planes; ++c)
    for (int i = 0; i < ih; ++i)
      for (int j = 0; j < iw; ++j)
        o[(size_t)c * ih * iw + IDX(i, j, iw)] =
            a[(size_t)c * oh * ow + IDX(in.y0 - out.y0 + i, in.x0 - out.x0 + j, ow)];
}

/* the layout on Omega~ and its subdomains (row-major over (m2, m1)) */
typedef struct {
  int n2, n1, m2, m1, sy, sx;
  int *ylo, *yhi, *xlo, *xhi;
  double ahat;
} layout_t;
static int layout_make(layout_t *L, int n2, int n1, const int lay[4]) {
  L->n2 = n2, L->n1 = n1, L->m2 = lay[0], L->m1 = lay[1], L->sy = lay[2], L->sx = lay[3];
  L->ylo = malloc(L->m2 * sizeof(int)), L->yhi = malloc(L->m2 * sizeof(int));
  L->xlo = malloc(L->m1 * sizeof(int)), L->xhi = malloc(L->m1 * sizeof(int));
  for (int a = 0; a < L->m2; ++a)
    if (tvo_layout_range(n2 + 1, L->m2, L->sy, a, &L->ylo[a], &L->yhi[a])) return 2;
  for (int b = 0; b < L->m1; ++b)
    if (tvo_layout_range(n1 + 1, L->m1, L->sx, b, &L->xlo[b], &L->xhi[b])) return 2;
  L->ahat = alpha_hat(L->m2, L->m1);
  return 0;
}
static void layout_free(layout_t *L) { free(L->ylo), free(L->yhi), free(L->xlo), free(L->xhi); }
/* Gamma_m on Omega~ (extended) or Omega~_m cap Omega */
static rect sub_rect(const layout_t *L, int a, int b, int extended) {
  rect r = {L->ylo[a], L->yhi[a], L->xlo[b], L->xhi[b]};
  if (!extended) {
    if (r.y1 > L->n2 - 1) r.y1 = L->n2 - 1;
    if (r.x1 > L->n1 - 1) r.x1 = L->n1 - 1;
  }
  return r;
}
/* theta_m on its own rectangle: theta_y(a) * theta_x(b) (separable, reading A7) */
static void sub_theta(const layout_t *L, int a, int b, rect r, double *th) {
  for (int i = 0; i < rh(r); ++i)
    for (int j = 0; j < rw(r); ++j)
      th[IDX(i, j, rw(r))] = tvo_layout_theta(L->n2 + 1, L->m2, L->sy, a, r.y0 + i) *
                             tvo_layout_theta(L->n1 + 1, L->m1, L->sx, b, r.x0 + j);
}

/* v_k <- (theta v_k + t theta psi_k) / (theta + t |psi_k|) per dual row k (Alg. 3/5, P:1349-1352,
 * P:1746-1749); theta = 0 gives v = 0 (reading A13).  rows = 1 (2-vector) or 2 (2x2). */
static void rowwise_update(double *v, const double *psi, const double *th, int rows, size_t pl,
                           double t) {
  for (int k = 0; k < rows; ++k)
    for (size_t e = 0; e < pl; ++e) {
      double *vx = v + (2 * k) * pl + e, *vy = v + (2 * k + 1) * pl + e;
      const double px = psi[(2 * k) * pl + e], py = psi[(2 * k + 1) * pl + e];
      if (th[e] > 0.0) {
        const double den = th[e] + t * sqrt(px * px + py * py);
        *vx = (th[e] * *vx + t * th[e] * px) / den;
        *vy = (th[e] * *vy + t * th[e] * py) / den;
      } else {
        *vx = 0.0, *vy = 0.0;
      }
    }
}

/* ------------------------------------------------------------------ energies (SURVEY C-13/C-15) */

/* TV(u) channel-wise (reading A15) and the gap sum (|grad u| + q . grad u) of one scalar field */
static void tv_gap(const double *u, const double *qx, const double *qy, int n2, int n1, double *tv,
                   double *gap) {
  const size_t pl = (size_t)n2 * n1;
  double *g = malloc(2 * pl * sizeof(double));
  tvo_grad(u, n2, n1, g);
  for (size_t e = 0; e < pl; ++e) {
    const double nrm = sqrt(g[e] * g[e] + g[pl + e] * g[pl + e]);
    *tv += nrm;
    if (qx) *gap += nrm + qx[e] * g[e] + qy[e] * g[pl + e];
  }
  free(g);
}

/* ------------------------------------------------------------------ Alg. 2 + Alg. 5 (step 1) */

typedef struct {
  const layout_t *L;
  const double *p, *r;       /* p^n (4 planes) and r^n = f - P multidiv p^n (2 planes), Omega~ */
  double **qhat;             /* per subdomain: 4 planes on Gamma_m (warm start in, solution out) */
  int inner;
  double t;
  const int *cy, *cx;
  const double *c2, *c1;     /* DCT matrices of Omega~ */
  int next, err;
  pthread_mutex_t mu;
} tfs_job;

/* R_{S+} P E_{S+} w (Eq. locglobprojpart1) for w (2 planes on S+): q = div_T E w on
 * T = (S+)_+ (resDiv), phi = R_T Delta^dagger E_T q by the block-DCT sum, w - R_{S+} grad_T
 * phi (resGrad) */
static int local_projection(const tfs_job *J, const double *w, rect sp, double *out) {
  const int n2t = J->L->n2 + 1, n1t = J->L->n1 + 1;
  const rect T = rect_plus(sp, n2t, n1t);
  const size_t tp = (size_t)rh(T) * rw(T), spp = (size_t)rh(sp) * rw(sp);
  double *we = malloc(2 * tp * sizeof(double)), *q = malloc(tp * sizeof(double));
  double *phi = malloc(tp * sizeof(double)), *g = malloc(2 * tp * sizeof(double));
  double *gr = malloc(2 * spp * sizeof(double));
  if (!we || !q || !phi || !g || !gr) return 7;
  extend(w, sp, T, 2, we);
  tvo_div(we, rh(T), rw(T), q);
  int st = lap_pinv_block(q, T.y0, T.y1, T.x0, T.x1, T.y0, T.y1, T.x0, T.x1, n2t, n1t, J->cy,
                          J->L->m2, J->cx, J->L->m1, J->c2, J->c1, phi);
  if (st) return st;
  tvo_grad(phi, rh(T), rw(T), g);
  restrict_(g, T, sp, 2, gr);
  for (size_t e = 0; e < 2 * spp; ++e) out[e] = w[e] - gr[e];
  free(we), free(q), free(phi), free(g), free(gr);
  return 0;
}

/* Alg. 5 for subdomain (a, b):
 *   omega0 = R_{S+} r + R_{S+} P E_{S+} multidiv_{S+} E_S (theta_m p)   (reading A11);
 *   inner times: w = multidiv_{S+} E_S v; psi = R_S multigrad_{S+}(P_loc w - omega0);
 *   v_k <- (theta v_k + t theta psi_k)/(theta + t |psi_k|). */
static int tfs_local(const tfs_job *J, int a, int b) {
  const layout_t *L = J->L;
  const int n2t = L->n2 + 1, n1t = L->n1 + 1;
  const rect s = sub_rect(L, a, b, 1), sp = rect_plus(s, n2t, n1t);
  const rect whole = {0, n2t - 1, 0, n1t - 1};
  const size_t sps = (size_t)rh(s) * rw(s), spp = (size_t)rh(sp) * rw(sp);
  double *th = malloc(sps * sizeof(double)), *tp = malloc(4 * sps * sizeof(double));
  double *ext = malloc(4 * spp * sizeof(double)), *w = malloc(2 * spp * sizeof(double));
  double *pw = malloc(2 * spp * sizeof(double)), *om = malloc(2 * spp * sizeof(double));
  double *mg = malloc(4 * spp * sizeof(double)), *psi = malloc(4 * sps * sizeof(double));
  if (!th || !tp || !ext || !w || !pw || !om || !mg || !psi) return 7;
  sub_theta(L, a, b, s, th);
  restrict_(J->p, whole, s, 4, tp);
  for (int c = 0; c < 4; ++c)
    for (size_t e = 0; e < sps; ++e) tp[c * sps + e] *= th[e];
  extend(tp, s, sp, 4, ext);
  multidiv(ext, rh(sp), rw(sp), w);
  int st = local_projection(J, w, sp, pw);
  if (st) return st;
  restrict_(J->r, whole, sp, 2, om);
  for (size_t e = 0; e < 2 * spp; ++e) om[e] += pw[e];
  double *v = J->qhat[a * L->m1 + b];
  for (int it = 0; it < J->inner; ++it) {
    extend(v, s, sp, 4, ext);
    multidiv(ext, rh(sp), rw(sp), w);
    st = local_projection(J, w, sp, pw);
    if (st) return st;
    for (size_t e = 0; e < 2 * spp; ++e) pw[e] -= om[e];
    multigrad(pw, rh(sp), rw(sp), mg);
    restrict_(mg, sp, s, 4, psi);
    rowwise_update(v, psi, th, 2, sps, J->t);
  }
  free(th), free(tp), free(ext), free(w), free(pw), free(om), free(mg), free(psi);
  return 0;
}
static void *tfs_worker(void *arg) {
  tfs_job *J = arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int m = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (m >= J->L->m2 * J->L->m1) break;
    const int st = tfs_local(J, m / J->L->m1, m % J->L->m1);
    if (st) {
      pthread_mutex_lock(&J->mu);
      J->err = st;
      pthread_mutex_unlock(&J->mu);
    }
  }
  return NULL;
}

/* run the local solves of one sweep on `threads` threads (one task per subdomain) */
static int run_sweep(void *(*worker)(void *), void *job, int *next, int *err, int threads, int M) {
  *next = 0, *err = 0;
  if (threads <= 1 || M <= 1) {
    worker(job);
    return *err;
  }
  const int nt = threads < M ? threads : M;
  pthread_t *th = malloc(nt * sizeof(pthread_t));
  for (int k = 0; k < nt; ++k) pthread_create(&th[k], NULL, worker, job);
  for (int k = 0; k < nt; ++k) pthread_join(th[k], NULL);
  free(th);
  return *err;
}

/* Alg. 2 for TFS on Omega~ with the localized Alg. 5; f = delta^{-1} P tau_0 (P:675,
 * reading A1), r^n once per sweep (A11); tau = P tau_0 - delta P multidiv p^S */
int tvo_step1(const double *d0, int n2, int n1, double delta, const int lay[4], int sweeps,
              int inner, double t, int threads, double *tau, double *p_out, double stats[3]) {
  if (!d0 || !tau || n2 < 2 || n1 < 2 || !(delta > 0) || !(t > 0 && t <= 0.125) || sweeps < 0 ||
      inner < 0)
    return 1;
  layout_t L;
  int st = layout_make(&L, n2, n1, lay);
  if (st) return st;
  const int g2 = n2 + 1, g1 = n1 + 1, M = L.m2 * L.m1;
  const size_t pl = (size_t)g2 * g1;
  double *t0 = malloc(2 * pl * sizeof(double)), *f = malloc(2 * pl * sizeof(double));
  double *p = calloc(4 * pl, sizeof(double)), *md = malloc(2 * pl * sizeof(double));
  double *pmd = malloc(2 * pl * sizeof(double)), *r = malloc(2 * pl * sizeof(double));
  double *acc = malloc(4 * pl * sizeof(double));
  double **qhat = calloc(M, sizeof(double *));
  int *cy = malloc((L.m2 + 1) * sizeof(int)), *cx = malloc((L.m1 + 1) * sizeof(int));
  double *c2 = dct_matrix(g2), *c1 = dct_matrix(g1);
  if (!t0 || !f || !p || !md || !pmd || !r || !acc || !qhat || !cy || !cx || !c2 || !c1) return 7;
  for (int k = 0; k <= L.m2; ++k) cy[k] = (int)((long long)k * g2 / L.m2);   /* reading A8 */
  for (int k = 0; k <= L.m1; ++k) cx[k] = (int)((long long)k * g1 / L.m1);
  for (int a = 0; a < L.m2; ++a)
    for (int b = 0; b < L.m1; ++b) {
      const rect s = sub_rect(&L, a, b, 1);
      qhat[a * L.m1 + b] = calloc(4 * (size_t)rh(s) * rw(s), sizeof(double));
    }
  tvo_tau0(d0, n2, n1, t0);
  if ((st = tvo_project(t0, g2, g1, f))) return st;
  for (size_t e = 0; e < 2 * pl; ++e) f[e] /= delta;
  tfs_job J = {&L, p, r, qhat, inner, t, cy, cx, c2, c1, 0, 0, PTHREAD_MUTEX_INITIALIZER};
  for (int n = 0; n < sweeps; ++n) {
    multidiv(p, g2, g1, md);
    if ((st = tvo_project(md, g2, g1, pmd))) return st;
    for (size_t e = 0; e < 2 * pl; ++e) r[e] = f[e] - pmd[e];
    if ((st = run_sweep(tfs_worker, &J, &J.next, &J.err, threads, M))) return st;
    memset(acc, 0, 4 * pl * sizeof(double));
    for (int a = 0; a < L.m2; ++a)   /* combine in subdomain order */
      for (int b = 0; b < L.m1; ++b) {
        const rect s = sub_rect(&L, a, b, 1);
        const double *q = qhat[a * L.m1 + b];
        const size_t sps = (size_t)rh(s) * rw(s);
        for (int c = 0; c < 4; ++c)
          for (int i = 0; i < rh(s); ++i)
            for (int j = 0; j < rw(s); ++j)
              acc[c * pl + IDX(s.y0 + i, s.x0 + j, g1)] += q[c * sps + IDX(i, j, rw(s))];
      }
    for (size_t e = 0; e < 4 * pl; ++e) p[e] = (1.0 - L.ahat) * p[e] + L.ahat * acc[e];
  }
  multidiv(p, g2, g1, md);
  if ((st = tvo_project(md, g2, g1, pmd))) return st;
  for (size_t e = 0; e < 2 * pl; ++e) tau[e] = delta * (f[e] - pmd[e]);
  if (stats) {   /* E_1 = TV(tau) + ||tau - P tau_0||^2/(2 delta), D = ||tau/delta||^2, gap */
    double tv = 0, gap = 0, fit = 0, dd = 0;
    for (int k = 0; k < 2; ++k)
      tv_gap(tau + k * pl, p + 2 * k * pl, p + (2 * k + 1) * pl, g2, g1, &tv, &gap);
    for (size_t e = 0; e < 2 * pl; ++e) {
      const double x = tau[e] - delta * f[e];
      fit += x * x;
      dd += (tau[e] / delta) * (tau[e] / delta);
    }
    stats[0] = tv + fit / (2.0 * delta), stats[1] = dd, stats[2] = gap;
  }
  if (p_out) memcpy(p_out, p, 4 * pl * sizeof(double));
  for (int m = 0; m < M; ++m) free(qhat[m]);
  free(qhat), free(t0), free(f), free(p), free(md), free(pmd), free(r), free(acc), free(cy), free(cx);
  free(c2), free(c1);
  layout_free(&L);
  return 0;
}

/* ------------------------------------------------------------------ Alg. 2 + Alg. 3 (step 2) */

typedef struct {
  const layout_t *L;
  const double *p, *res;   /* p^n (2 planes) and f - div p^n (1 plane), Omega */
  double **qhat;
  int inner;
  double t;
  int next, err;
  pthread_mutex_t mu;
} irv_job;

/* Alg. 3 for Lambda = div on Omega, localized (resDiv / resGrad P:1417-1426):
 * omega0 = R_{S+}(f - div p) + div_{S+} E_S (theta_m p); inner times u = div_{S+} E v - omega0,
 * psi = R_S grad_{S+} u, v <- (theta v + t theta psi)/(theta + t |psi|). */
static int irv_local(const irv_job *J, int a, int b) {
  const layout_t *L = J->L;
  const int n2 = L->n2, n1 = L->n1;
  const rect s = sub_rect(L, a, b, 0), sp = rect_plus(s, n2, n1);
  const rect whole = {0, n2 - 1, 0, n1 - 1};
  const size_t sps = (size_t)rh(s) * rw(s), spp = (size_t)rh(sp) * rw(sp);
  double *th = malloc(sps * sizeof(double)), *tp = malloc(2 * sps * sizeof(double));
  double *ext = malloc(2 * spp * sizeof(double)), *dv = malloc(spp * sizeof(double));
  double *om = malloc(spp * sizeof(double)), *g = malloc(2 * spp * sizeof(double));
  double *psi = malloc(2 * sps * sizeof(double));
  if (!th || !tp || !ext || !dv || !om || !g || !psi) return 7;
  sub_theta(L, a, b, s, th);
  restrict_(J->p, whole, s, 2, tp);
  for (int c = 0; c < 2; ++c)
    for (size_t e = 0; e < sps; ++e) tp[c * sps + e] *= th[e];
  extend(tp, s, sp, 2, ext);
  tvo_div(ext, rh(sp), rw(sp), dv);
  restrict_(J->res, whole, sp, 1, om);
  for (size_t e = 0; e < spp; ++e) om[e] += dv[e];
  double *v = J->qhat[a * L->m1 + b];
  for (int it = 0; it < J->inner; ++it) {
    extend(v, s, sp, 2, ext);
    tvo_div(ext, rh(sp), rw(sp), dv);
    for (size_t e = 0; e < spp; ++e) dv[e] -= om[e];
    tvo_grad(dv, rh(sp), rw(sp), g);
    restrict_(g, sp, s, 2, psi);
    rowwise_update(v, psi, th, 1, sps, J->t);
  }
  free(th), free(tp), free(ext), free(dv), free(om), free(g), free(psi);
  return 0;
}
static void *irv_worker(void *arg) {
  irv_job *J = arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int m = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (m >= J->L->m2 * J->L->m1) break;
    const int st = irv_local(J, m / J->L->m1, m % J->L->m1);
    if (st) {
      pthread_mutex_lock(&J->mu);
      J->err = st;
      pthread_mutex_unlock(&J->mu);
    }
  }
  return NULL;
}

/* Step 2, IRV2 (Eq. ir2dualdis): alpha = 1/lambda (reading A4); g by backward
 * differences of tau^perp integrated along row 0 then down each column, zero mean (reading A3);
 * f = alpha (d_0 - g); Alg. 2 + Alg. 3; d = d_0 - div p / alpha */
int tvo_step2(const double *tau, const double *d0, int n2, int n1, double lambda,
              const int lay[4], int sweeps, int inner, double t, int threads, double *d,
              double *p_out, double stats[3]) {
  if (!tau || !d0 || !d || n2 < 2 || n1 < 2 || !(lambda > 0) || !(t > 0 && t <= 0.125) ||
      sweeps < 0 || inner < 0)
    return 1;
  layout_t L;
  int st = layout_make(&L, n2, n1, lay);
  if (st) return st;
  const int M = L.m2 * L.m1, g1 = n1 + 1;
  const size_t pl = (size_t)n2 * n1;
  const double alpha = 1.0 / lambda;
  const double *t1 = tau, *t2 = tau + (size_t)(n2 + 1) * g1;
  double *g = malloc(pl * sizeof(double)), *f = malloc(pl * sizeof(double));
  double *p = calloc(2 * pl, sizeof(double)), *dv = malloc(pl * sizeof(double));
  double *res = malloc(pl * sizeof(double)), *acc = malloc(2 * pl * sizeof(double));
  double **qhat = calloc(M, sizeof(double *));
  if (!g || !f || !p || !dv || !res || !acc || !qhat) return 7;
  for (int a = 0; a < L.m2; ++a)
    for (int b = 0; b < L.m1; ++b) {
      const rect s = sub_rect(&L, a, b, 0);
      qhat[a * L.m1 + b] = calloc(2 * (size_t)rh(s) * rw(s), sizeof(double));
    }
  g[0] = 0.0;   /* g_{i,j} - g_{i,j-1} = tau_2[i,j], g_{i,j} - g_{i-1,j} = -tau_1[i,j] */
  for (int j = 1; j < n1; ++j) g[j] = g[j - 1] + t2[IDX(0, j, g1)];
  for (int i = 1; i < n2; ++i)
    for (int j = 0; j < n1; ++j) g[IDX(i, j, n1)] = g[IDX(i - 1, j, n1)] - t1[IDX(i, j, g1)];
  double mean = 0.0;
  for (size_t e = 0; e < pl; ++e) mean += g[e];
  mean /= (double)pl;
  for (size_t e = 0; e < pl; ++e) g[e] -= mean, f[e] = alpha * (d0[e] - g[e]);
  irv_job J = {&L, p, res, qhat, inner, t, 0, 0, PTHREAD_MUTEX_INITIALIZER};
  for (int n = 0; n < sweeps; ++n) {
    tvo_div(p, n2, n1, dv);
    for (size_t e = 0; e < pl; ++e) res[e] = f[e] - dv[e];
    if ((st = run_sweep(irv_worker, &J, &J.next, &J.err, threads, M))) return st;
    memset(acc, 0, 2 * pl * sizeof(double));
    for (int a = 0; a < L.m2; ++a)
      for (int b = 0; b < L.m1; ++b) {
        const rect s = sub_rect(&L, a, b, 0);
        const double *q = qhat[a * L.m1 + b];
        const size_t sps = (size_t)rh(s) * rw(s);
        for (int c = 0; c < 2; ++c)
          for (int i = 0; i < rh(s); ++i)
            for (int j = 0; j < rw(s); ++j)
              acc[c * pl + IDX(s.y0 + i, s.x0 + j, n1)] += q[c * sps + IDX(i, j, rw(s))];
      }
    for (size_t e = 0; e < 2 * pl; ++e) p[e] = (1.0 - L.ahat) * p[e] + L.ahat * acc[e];
  }
  tvo_div(p, n2, n1, dv);
  for (size_t e = 0; e < pl; ++e) d[e] = d0[e] - dv[e] / alpha;
  if (stats) {   /* E_2 = TV(d - g) + alpha/2 ||d - d_0||^2, D = ||div p - f||^2, gap */
    double tv = 0, gap = 0, fit = 0, dd = 0;
    for (size_t e = 0; e < pl; ++e) res[e] = d[e] - g[e];
    tv_gap(res, p, p + pl, n2, n1, &tv, &gap);
    for (size_t e = 0; e < pl; ++e) {
      fit += (d[e] - d0[e]) * (d[e] - d0[e]);
      dd += (dv[e] - f[e]) * (dv[e] - f[e]);
    }
    stats[0] = tv + 0.5 * alpha * fit, stats[1] = dd, stats[2] = gap;
  }
  if (p_out) memcpy(p_out, p, 2 * pl * sizeof(double));
  for (int m = 0; m < M; ++m) free(qhat[m]);
  free(qhat), free(g), free(f), free(p), free(dv), free(res), free(acc);
  layout_free(&L);
  return 0;
}

/* step 1 then step 2 on the same splitting */
int tvo_denoise(const double *d0, int n2, int n1, double delta, double lambda, const int lay[4],
                const int it1[2], const int it2[2], double t, int threads, double *d, double *tau,
                double stats1[3], double stats2[3]) {
  const size_t tp = 2 * (size_t)(n2 + 1) * (n1 + 1);
  double *tb = tau ? tau : malloc(tp * sizeof(double));
  if (!tb) return 7;
  int st = tvo_step1(d0, n2, n1, delta, lay, it1[0], it1[1], t, threads, tb, NULL, stats1);
  if (!st) st = tvo_step2(tb, d0, n2, n1, lambda, lay, it2[0], it2[1], t, threads, d, NULL, stats2);
  if (!tau) free(tb);
  return st;
}
