// Hand-written sm_100a kernels of the TV-Stokes Schwarz dual iteration (arXiv 2602.17494).
// Citations P:<line> refer to PAPER.md.  Index conventions: row i (y), column j (x), 0-based.
// Global fields are planes of n2 rows with row pitch `ld` floats; batched per-subdomain buffers
// use the uniform geometry of tvs::Geo (see tvs_internal.h).
#include "tvs_internal.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <math.h>
#include <stdlib.h>
#include <string.h>

namespace tvs {

// ----------------------------------------------------------------------------- helpers

// round-to-nearest tf32 (low 13 mantissa bits zero): the "hi" half of a 3xTF32 operand split
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}
// store v either as full fp32 (lo == nullptr) or as the exact split hi = tf32(v), lo = v - hi
__device__ __forceinline__ void store_split(float *hi, float *lo, size_t idx, double v) {
  if (lo) {
    float h = tf32_rna((float)v);
    hi[idx] = h;
    lo[idx] = (float)(v - (double)h);
  } else {
    hi[idx] = (float)v;
  }
}

__device__ __forceinline__ float theta_at(const float *thy, const float *thx, const SubDesc &sd,
                                          const Geo &g, int li, int lj) {
  return thy[sd.iy * g.A + li] * thx[sd.ix * g.B + lj];
}

// Value of a per-subdomain plane on S at local (li, lj), zero outside S (extension E_S).
__device__ __forceinline__ float vS(const float *__restrict__ plane, int li, int lj, int a, int b,
                                    int ld) {
  return (li >= 0 && li < a && lj >= 0 && lj < b) ? __ldg(plane + (size_t)li * ld + lj) : 0.f;
}

// Global discrete divergence (Eq. defDivDis P:594 with the three-case D-) of a
// 2-vector field that vanishes outside S, evaluated at local (li, lj) = global (gi, gj).
// (x-part: [gj < n1-1] u(gj) - [gj > 0] u(gj-1); the u outside S are zero.)
__device__ __forceinline__ float div_S(const float *vx, const float *vy, int li, int lj, int gi,
                                       int gj, int a, int b, int ld, int n2, int n1) {
  float dx = (gj < n1 - 1 ? vS(vx, li, lj, a, b, ld) : 0.f) - vS(vx, li, lj - 1, a, b, ld);
  float dy = (gi < n2 - 1 ? vS(vy, li, lj, a, b, ld) : 0.f) - vS(vy, li - 1, lj, a, b, ld);
  return dx + dy;
}

// ball update with fast MUFU square root and reciprocal (each within ~2 ulp; no slow-path
// branches): v <- (th v + t th psi) / (th + t|psi|).  __fdividef(a, b) returns 0 for b in
// (2^126, 2^128); with th <= 1 and t <= 1/8 that range needs |psi| > 2^129, i.e. only |psi| = inf
// (overflow of psx^2 + psy^2) reaches it -- where IEEE division gives 0 as well.  A dual that has
// blown up that far is written as NaN instead, so the combine's non-finite flag reports
// TVS_ENUMERIC rather than silently resetting v to 0.
__device__ __forceinline__ void ball_update_fast(float th, float t, float psx, float psy,
                                                 float &vx, float &vy) {
  float nrm;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(nrm) : "f"(psx * psx + psy * psy));
  const float inv = __fdividef(th, th + t * nrm);
  const bool finite = nrm <= 3.402823466e38f;   // false for inf and NaN
  const float bad = __int_as_float(0x7fc00000);
  const float nx = (vx + t * psx) * inv, ny = (vy + t * psy) * inv;
  vx = th > 0.f ? (finite ? nx : bad) : 0.f;
  vy = th > 0.f ? (finite ? ny : bad) : 0.f;
}

// ----------------------------------------------------------------------------- step data

// tau_0 = (-D_y^{neum-} d0, D_x^{neum-} d0) on Omega~ (Eq. def:backdiffNeumann P:576-591).
__global__ void k_tau0(const float *__restrict__ d0, int n2, int n1, float *__restrict__ tau,
                       int ldt) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i > n2 || j > n1) return;
  float dxv = 0.f, dyv = 0.f;
  if (j != 0 && j != n1) {
    int r = i < n2 ? i : n2 - 1;                    // mirrored extra row
    dxv = d0[(size_t)r * n1 + j] - d0[(size_t)r * n1 + j - 1];
  }
  if (i != 0 && i != n2) {
    int c = j < n1 ? j : n1 - 1;                    // mirrored extra column
    dyv = d0[(size_t)i * n1 + c] - d0[(size_t)(i - 1) * n1 + c];
  }
  size_t plane = (size_t)(n2 + 1) * ldt;
  tau[(size_t)i * ldt + j] = -dyv;
  tau[plane + (size_t)i * ldt + j] = dxv;
}

// g on row 0 by backward-difference integration along x (reading A3): g[0][j] = sum tau_2[0][1..j].
__global__ void k_g_row0(const float *__restrict__ tau2, int n1, double *__restrict__ g0) {
  __shared__ double part[1024];
  int tid = threadIdx.x, nt = blockDim.x;
  int chunk = (n1 + nt - 1) / nt;
  int a = tid * chunk, b = min(n1, a + chunk);
  double s = 0.0;
  for (int j = a; j < b; ++j) s += (j >= 1) ? (double)tau2[j] : 0.0;
  part[tid] = s;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {          // inclusive Hillis-Steele scan
    double add = tid >= off ? part[tid - off] : 0.0;
    __syncthreads();
    part[tid] += add;
    __syncthreads();
  }
  double acc = tid > 0 ? part[tid - 1] : 0.0;
  for (int j = a; j < b; ++j) {
    acc += (j >= 1) ? (double)tau2[j] : 0.0;
    g0[j] = acc;
  }
}

// f = alpha (d0 - g) (Eq. ir2dualdis), g integrated down each column with
// g[i][j] = g[i-1][j] - tau_1[i][j] (reading A3), accumulated in fp64.
__global__ void k_irv2_f(const float *__restrict__ tau1, int ldt, const double *__restrict__ g0,
                         const float *__restrict__ d0, int n2, int n1, float alpha,
                         float *__restrict__ f, int ldf) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n1) return;
  double acc = g0[j];
  f[j] = alpha * (float)((double)d0[j] - acc);
#pragma unroll 8
  for (int i = 1; i < n2; ++i) {
    acc -= (double)tau1[(size_t)i * ldt + j];
    f[(size_t)i * ldf + j] = (float)((double)alpha * ((double)d0[(size_t)i * n1 + j] - acc));
  }
}

// Column-parallel form of k_irv2_f: the column integration runs in chunks of IRV2_ROWS rows (one
// thread per (chunk, column)); chunk sums of tau_1 first, then each chunk starts from g0 minus the
// sums of the chunks above (fp64 throughout; the same integral in a chunked summation order).
constexpr int IRV2_ROWS = 64;
__global__ void k_irv2_chunk_sums(const float *__restrict__ tau1, int ldt, int n2, int n1,
                                  double *__restrict__ csum) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (j >= n1) return;
  const int i0 = max(1, c * IRV2_ROWS), i1 = min(n2, (c + 1) * IRV2_ROWS);
  double acc = 0.0;
  for (int i = i0; i < i1; ++i) acc += (double)tau1[(size_t)i * ldt + j];
  csum[(size_t)c * n1 + j] = acc;
}
__global__ void k_irv2_f_chunked(const float *__restrict__ tau1, int ldt,
                                 const double *__restrict__ g0, const float *__restrict__ d0, int n2,
                                 int n1, float alpha, float *__restrict__ f, int ldf,
                                 const double *__restrict__ csum) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (j >= n1) return;
  double acc = g0[j];
  for (int k = 0; k < c; ++k) acc -= csum[(size_t)k * n1 + j];
  const int i0 = c * IRV2_ROWS, i1 = min(n2, (c + 1) * IRV2_ROWS);
  for (int i = i0; i < i1; ++i) {
    if (i >= 1) acc -= (double)tau1[(size_t)i * ldt + j];
    f[(size_t)i * ldf + j] = (float)((double)alpha * ((double)d0[(size_t)i * n1 + j] - acc));
  }
}

// IRV1 data (Eq. ir1dualdis): f = alpha d0 - div xi, xi = tau_perp / sqrt(|tau_perp|^2 + eps)
// with tau_perp = R_Omega(tau_2, -tau_1) (Eq. defXi2:discrete); div with the three-case
// D- (P:560-571).  Also stores div xi for the recovery d = d0 - (div p + div xi)/alpha.
__global__ void k_irv1_f(const float *__restrict__ tau1, const float *__restrict__ tau2, int ldt,
                         const float *__restrict__ d0, int n2, int n1, float alpha, float eps,
                         float *__restrict__ f, float *__restrict__ dxi, int ldf) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= n2 || j >= n1) return;
  auto xi1 = [&](int a, int b) {   // x-component tau_2 / |tau|_eps
    const float t1 = tau1[(size_t)a * ldt + b], t2 = tau2[(size_t)a * ldt + b];
    return t2 * rsqrtf(t1 * t1 + t2 * t2 + eps);
  };
  auto xi2 = [&](int a, int b) {   // y-component -tau_1 / |tau|_eps
    const float t1 = tau1[(size_t)a * ldt + b], t2 = tau2[(size_t)a * ldt + b];
    return -t1 * rsqrtf(t1 * t1 + t2 * t2 + eps);
  };
  const float dv = (j < n1 - 1 ? xi1(i, j) : 0.f) - (j > 0 ? xi1(i, j - 1) : 0.f) +
                   (i < n2 - 1 ? xi2(i, j) : 0.f) - (i > 0 ? xi2(i - 1, j) : 0.f);
  f[(size_t)i * ldf + j] = alpha * d0[(size_t)i * n1 + j] - dv;
  dxi[(size_t)i * ldf + j] = dv;
}

// ----------------------------------------------------------------------------- step 2 (IRV2)

// omega0_m = R_{S+}(f - div p^n + div(theta_m p^n)) (Alg. 3 with Lambda = div, P:1348,
// localized by resDiv P:1417).  One plane per subdomain on S+.
__global__ void k_omega0_2(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ thy,
                           const float *__restrict__ thx, const float *__restrict__ f,
                           const float *__restrict__ p1, const float *__restrict__ p2, int ld,
                           int n2, int n1, float *__restrict__ om) {
  const SubDesc sd = subs[blockIdx.z];
  int lj = blockIdx.x * blockDim.x + threadIdx.x;
  int li = blockIdx.y * blockDim.y + threadIdx.y;
  int gi = sd.y0 + li, gj = sd.x0 + lj;
  if (gi > sd.py1 || gj > sd.px1) return;
  int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  auto P1 = [&](int i, int j) { return p1[(size_t)i * ld + j]; };
  auto P2 = [&](int i, int j) { return p2[(size_t)i * ld + j]; };
  float divp = (gj < n1 - 1 ? P1(gi, gj) : 0.f) - (gj > 0 ? P1(gi, gj - 1) : 0.f) +
               (gi < n2 - 1 ? P2(gi, gj) : 0.f) - (gi > 0 ? P2(gi - 1, gj) : 0.f);
  auto U1 = [&](int i, int j) {   // theta_m p_1 extended by zero outside S (local coords)
    return (i >= 0 && i < a && j >= 0 && j < b)
               ? theta_at(thy, thx, sd, g, i, j) * P1(sd.y0 + i, sd.x0 + j) : 0.f;
  };
  auto U2 = [&](int i, int j) {
    return (i >= 0 && i < a && j >= 0 && j < b)
               ? theta_at(thy, thx, sd, g, i, j) * P2(sd.y0 + i, sd.x0 + j) : 0.f;
  };
  float divu = (gj < n1 - 1 ? U1(li, lj) : 0.f) - U1(li, lj - 1) +
               (gi < n2 - 1 ? U2(li, lj) : 0.f) - U2(li - 1, lj);
  om[((size_t)blockIdx.z * g.AP + li) * g.ldP + lj] = f[(size_t)gi * ld + gj] - divp + divu;
}



// Kernel (a), vectorised streaming form (default): lane l owns the column pair
// (c0 - 2 + 2l, c0 - 1 + 2l) -> 8-byte loads/stores; a warp produces 60 output columns
// (lanes 1..30), lane 0 supplies the left halo column and lane 31 the right one.  Two rows of
// loads are kept in flight ahead of the arithmetic (bytes in flight per SM ~ 3x the scalar form).
constexpr int SV_OUT = 60, SV_WARPS = 4;
__global__ void __launch_bounds__(32 * SV_WARPS)
k_sweep2v(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ thy,
          const float *__restrict__ thx, const float *__restrict__ vin,
          const float *__restrict__ om, float *__restrict__ vout, int n2, int n1, float t, int rb) {
  const SubDesc sd = subs[blockIdx.z];
  const int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  const int ap = sd.py1 - sd.y0 + 1, bp = sd.px1 - sd.x0 + 1;
  const int lane = threadIdx.x, strip = blockIdx.x * SV_WARPS + threadIdx.y;
  const int c0 = strip * SV_OUT;
  if (c0 >= b) return;
  const int r0 = blockIdx.y * rb;
  if (r0 >= a) return;
  const int r1 = min(a, r0 + rb);
  const int jA = c0 - 2 + 2 * lane, jB = jA + 1;          // local columns of this lane
  // a column pair is loaded as one float2 when both columns lie inside the plane's extent
  const bool SA = jA >= 0 && jA < b, SB = jB >= 0 && jB < b;
  const bool PA = jA >= 0 && jA < bp, PB = jB >= 0 && jB < bp;
  const bool outA = lane >= 1 && lane <= 30 && jA < b;
  const bool outB = lane >= 1 && lane <= 30 && jB < b;
  const float xkA = (sd.x0 + jA < n1 - 1) ? 1.f : 0.f, xkB = (sd.x0 + jB < n1 - 1) ? 1.f : 0.f;
  const float *v1 = vin + (size_t)blockIdx.z * 2 * g.A * g.ldS;
  const float *v2 = v1 + (size_t)g.A * g.ldS;
  const float *omm = om + (size_t)blockIdx.z * g.AP * g.ldP;
  float *o1 = vout + (size_t)blockIdx.z * 2 * g.A * g.ldS;
  float *o2 = o1 + (size_t)g.A * g.ldS;
  const float thA = SA ? thx[sd.ix * g.B + jA] : 0.f, thB = SB ? thx[sd.ix * g.B + jB] : 0.f;
  auto ldpair = [&](const float *base, int ld, int li, int rows, bool okA, bool okB) {
    float2 r = make_float2(0.f, 0.f);
    if (li < 0 || li >= rows) return r;
    const float *p = base + (size_t)li * ld + jA;
    if (okA && okB) return __ldg(reinterpret_cast<const float2 *>(p));
    if (okA) r.x = __ldg(p);
    if (okB) r.y = __ldg(p + 1);
    return r;
  };
  struct Row { float2 w1, w2, o; };
  auto ldrow = [&](int li) {
    Row r;
    r.w1 = ldpair(v1, g.ldS, li, a, SA, SB);
    r.w2 = ldpair(v2, g.ldS, li, a, SA, SB);
    r.o = ldpair(omm, g.ldP, li, ap, PA, PB);
    return r;
  };
  // u for the lane's pair at row li, given that row and v_2 of the row above
  auto ucalc = [&](int li, const Row &r, float2 w2m) {
    const float leftA = __shfl_up_sync(0xffffffffu, r.w1.y, 1);    // v_1 at column jA - 1
    const bool gy = (sd.y0 + li < n2 - 1);
    float2 u;
    u.x = (PA && li < ap) ? (xkA * r.w1.x - leftA + (gy ? r.w2.x : 0.f) - w2m.x - r.o.x) : 0.f;
    u.y = (PB && li < ap) ? (xkB * r.w1.y - r.w1.x + (gy ? r.w2.y : 0.f) - w2m.y - r.o.y) : 0.f;
    return u;
  };
  Row c = ldrow(r0), n = ldrow(r0 + 1);
  const Row pr = ldrow(r0 - 1);
  float2 u_c = ucalc(r0, c, pr.w2);
  for (int li = r0; li < r1; ++li) {
    const Row m = ldrow(li + 2);                     // two rows in flight
    const float2 u_n = ucalc(li + 1, n, c.w2);
    const float urA = __shfl_down_sync(0xffffffffu, u_c.x, 1);   // u at column jB + 1
    const float psxA = (jA + 1 < bp) ? u_c.y - u_c.x : 0.f;
    const float psxB = (jB + 1 < bp) ? urA - u_c.y : 0.f;
    const float psyA = (li + 1 < ap) ? u_n.x - u_c.x : 0.f;
    const float psyB = (li + 1 < ap) ? u_n.y - u_c.y : 0.f;
    const float ty = thy[sd.iy * g.A + li];
    float2 nv1 = c.w1, nv2 = c.w2;
    ball_update_fast(ty * thA, t, psxA, psyA, nv1.x, nv2.x);
    ball_update_fast(ty * thB, t, psxB, psyB, nv1.y, nv2.y);
    float *q1 = o1 + (size_t)li * g.ldS + jA, *q2 = o2 + (size_t)li * g.ldS + jA;
    if (outA && outB) {
      *reinterpret_cast<float2 *>(q1) = nv1;
      *reinterpret_cast<float2 *>(q2) = nv2;
    } else {
      if (outA) { q1[0] = nv1.x; q2[0] = nv2.x; }
      if (outB) { q1[1] = nv1.y; q2[1] = nv2.y; }
    }
    c = n;
    n = m;
    u_c = u_n;
  }
}


// Kernel (a), 4 columns per lane (default): lane l owns columns c0-4+4l .. c0-1+4l (16-byte loads
// and stores); lanes 1..30 produce 120 output columns, lane 0 / lane 31 are the halo columns.
// Two rows of loads in flight ahead of the arithmetic; registers capped for 50 % occupancy.
constexpr int SQ_OUT = 120, SQ_RB = 64, SQ_WARPS = 4;
__global__ void __launch_bounds__(32 * SQ_WARPS, 8)
k_sweep2q(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ thy,
          const float *__restrict__ thx, const float *__restrict__ vin,
          const float *__restrict__ om, float *__restrict__ vout, int n2, int n1, float t) {
  const SubDesc sd = subs[blockIdx.z];
  const int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  const int ap = sd.py1 - sd.y0 + 1, bp = sd.px1 - sd.x0 + 1;
  const int lane = threadIdx.x, strip = blockIdx.x * SQ_WARPS + threadIdx.y;
  const int c0 = strip * SQ_OUT;
  if (c0 >= b) return;
  const int r0 = blockIdx.y * SQ_RB;
  if (r0 >= a) return;
  const int r1 = min(a, r0 + SQ_RB);
  const int j0 = c0 - 4 + 4 * lane;                   // first local column of this lane
  // per-column masks (S for v, S+ for u / omega0), output lanes, global D-_x rule at n1 - 1
  float mS[4], mP[4], xk[4], thc[4];
  bool fullS = true, fullP = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + q;
    const bool s_ = j >= 0 && j < b, p_ = j >= 0 && j < bp;
    mS[q] = s_ ? 1.f : 0.f;
    mP[q] = p_ ? 1.f : 0.f;
    fullS &= s_;
    fullP &= p_;
    xk[q] = (sd.x0 + j < n1 - 1) ? 1.f : 0.f;
    thc[q] = s_ ? thx[sd.ix * g.B + j] : 0.f;
  }
  const bool out_lane = lane >= 1 && lane <= 30;
  const float *v1 = vin + (size_t)blockIdx.z * 2 * g.A * g.ldS;
  const float *v2 = v1 + (size_t)g.A * g.ldS;
  const float *omm = om + (size_t)blockIdx.z * g.AP * g.ldP;
  float *o1 = vout + (size_t)blockIdx.z * 2 * g.A * g.ldS;
  float *o2 = o1 + (size_t)g.A * g.ldS;
  auto ld4 = [&](const float *base, int ld, int li, int rows, bool full, const float *m) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (li < 0 || li >= rows) return r;
    const float *p = base + (size_t)li * ld + j0;
    if (full) return __ldg(reinterpret_cast<const float4 *>(p));
    if (m[0] != 0.f) r.x = __ldg(p);
    if (m[1] != 0.f) r.y = __ldg(p + 1);
    if (m[2] != 0.f) r.z = __ldg(p + 2);
    if (m[3] != 0.f) r.w = __ldg(p + 3);
    return r;
  };
  struct Row { float4 w1, w2, o; };
  auto ldrow = [&](int li) {
    Row r;
    r.w1 = ld4(v1, g.ldS, li, a, fullS, mS);
    r.w2 = ld4(v2, g.ldS, li, a, fullS, mS);
    r.o = ld4(omm, g.ldP, li, ap, fullP, mP);
    return r;
  };
  auto ucalc = [&](int li, const Row &r, float4 w2m) {
    const float left = __shfl_up_sync(0xffffffffu, r.w1.w, 1);   // v_1 at column j0 - 1
    const float gy = (sd.y0 + li < n2 - 1) ? 1.f : 0.f;
    const float rowok = (li < ap) ? 1.f : 0.f;
    float4 u;
    u.x = rowok * mP[0] * (xk[0] * r.w1.x - left + gy * r.w2.x - w2m.x - r.o.x);
    u.y = rowok * mP[1] * (xk[1] * r.w1.y - r.w1.x + gy * r.w2.y - w2m.y - r.o.y);
    u.z = rowok * mP[2] * (xk[2] * r.w1.z - r.w1.y + gy * r.w2.z - w2m.z - r.o.z);
    u.w = rowok * mP[3] * (xk[3] * r.w1.w - r.w1.z + gy * r.w2.w - w2m.w - r.o.w);
    return u;
  };
  Row c = ldrow(r0), n = ldrow(r0 + 1);
  const float4 pw2 = ld4(v2, g.ldS, r0 - 1, a, fullS, mS);
  float4 u_c = ucalc(r0, c, pw2);
  const bool lastx[4] = {j0 + 1 >= bp, j0 + 2 >= bp, j0 + 3 >= bp, j0 + 4 >= bp};
  for (int li = r0; li < r1; ++li) {
    const Row m = ldrow(li + 2);
    const float4 u_n = ucalc(li + 1, n, c.w2);
    const float ur = __shfl_down_sync(0xffffffffu, u_c.x, 1);      // u at column j0 + 4
    const float ydiff = (li + 1 < ap) ? 1.f : 0.f;
    const float psx0 = lastx[0] ? 0.f : u_c.y - u_c.x, psy0 = ydiff * (u_n.x - u_c.x);
    const float psx1 = lastx[1] ? 0.f : u_c.z - u_c.y, psy1 = ydiff * (u_n.y - u_c.y);
    const float psx2 = lastx[2] ? 0.f : u_c.w - u_c.z, psy2 = ydiff * (u_n.z - u_c.z);
    const float psx3 = lastx[3] ? 0.f : ur - u_c.w, psy3 = ydiff * (u_n.w - u_c.w);
    const float ty = thy[sd.iy * g.A + li];
    float4 a1 = c.w1, a2 = c.w2;
    ball_update_fast(ty * thc[0], t, psx0, psy0, a1.x, a2.x);
    ball_update_fast(ty * thc[1], t, psx1, psy1, a1.y, a2.y);
    ball_update_fast(ty * thc[2], t, psx2, psy2, a1.z, a2.z);
    ball_update_fast(ty * thc[3], t, psx3, psy3, a1.w, a2.w);
    if (out_lane) {
      float *q1 = o1 + (size_t)li * g.ldS + j0, *q2 = o2 + (size_t)li * g.ldS + j0;
      if (fullS) {
        *reinterpret_cast<float4 *>(q1) = a1;
        *reinterpret_cast<float4 *>(q2) = a2;
      } else {
        if (mS[0] != 0.f) { q1[0] = a1.x; q2[0] = a2.x; }
        if (mS[1] != 0.f) { q1[1] = a1.y; q2[1] = a2.y; }
        if (mS[2] != 0.f) { q1[2] = a1.z; q2[2] = a2.z; }
        if (mS[3] != 0.f) { q1[3] = a1.w; q2[3] = a2.w; }
      }
    }
    c = n;
    n = m;
    u_c = u_n;
  }
}

// Kernel (a) with two inner iterations per pass (temporal blocking of Alg. 3's inner loop,
// P:1346-1352; omega0 is fixed within a sweep): the same 4-columns-per-lane streaming layout as
// k_sweep2q; the column halo of lanes 0 / 31 is 4 wide and a level-k result is wrong only k columns
// from a halo edge, so lanes 1..30 stay exact for two levels.  Rows: level 1 is computed on rows
// r0-1 .. r1 and level 2 on r0 .. r1-1 from a register ring (raw rows up to r1+2 in flight).  Each
// element goes through exactly the operations of two k_sweep2q launches (bitwise identical);
// HBM traffic per update is about half.
template <int MINB>
__global__ void __launch_bounds__(32 * SQ_WARPS, MINB)
k_sweep2q2(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ thy,
           const float *__restrict__ thx, const float *__restrict__ vin,
           const float *__restrict__ om, float *__restrict__ vout, int n2, int n1, float t) {
  const SubDesc sd = subs[blockIdx.z];
  const int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  const int ap = sd.py1 - sd.y0 + 1, bp = sd.px1 - sd.x0 + 1;
  const int lane = threadIdx.x, strip = blockIdx.x * SQ_WARPS + threadIdx.y;
  const int c0 = strip * SQ_OUT;
  if (c0 >= b) return;
  const int r0 = blockIdx.y * SQ_RB;
  if (r0 >= a) return;
  const int r1 = min(a, r0 + SQ_RB);
  const int j0 = c0 - 4 + 4 * lane;
  float mS[4], mP[4], xk[4], thc[4];
  bool fullS = true, fullP = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + q;
    const bool s_ = j >= 0 && j < b, p_ = j >= 0 && j < bp;
    mS[q] = s_ ? 1.f : 0.f;
    mP[q] = p_ ? 1.f : 0.f;
    fullS &= s_;
    fullP &= p_;
    xk[q] = (sd.x0 + j < n1 - 1) ? 1.f : 0.f;
    thc[q] = s_ ? thx[sd.ix * g.B + j] : 0.f;
  }
  const bool out_lane = lane >= 1 && lane <= 30;
  const float *v1 = vin + (size_t)blockIdx.z * 2 * g.A * g.ldS;
  const float *v2 = v1 + (size_t)g.A * g.ldS;
  const float *omm = om + (size_t)blockIdx.z * g.AP * g.ldP;
  float *o1 = vout + (size_t)blockIdx.z * 2 * g.A * g.ldS;
  float *o2 = o1 + (size_t)g.A * g.ldS;
  auto ld4 = [&](const float *base, int ld, int li, int rows, bool full, const float *m) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (li < 0 || li >= rows) return r;
    const float *p = base + (size_t)li * ld + j0;
    if (full) return __ldg(reinterpret_cast<const float4 *>(p));
    if (m[0] != 0.f) r.x = __ldg(p);
    if (m[1] != 0.f) r.y = __ldg(p + 1);
    if (m[2] != 0.f) r.z = __ldg(p + 2);
    if (m[3] != 0.f) r.w = __ldg(p + 3);
    return r;
  };
  struct Raw { float4 w1, w2, o; };
  struct V2 { float4 w1, w2; };
  auto ldraw = [&](int li) {
    Raw r;
    r.w1 = ld4(v1, g.ldS, li, a, fullS, mS);
    r.w2 = ld4(v2, g.ldS, li, a, fullS, mS);
    r.o = ld4(omm, g.ldP, li, ap, fullP, mP);
    return r;
  };
  // u = div_{S+} E v - omega0 at row li (global D- rules), given v at li and v_2 at li - 1
  auto ucalc = [&](int li, float4 w1, float4 w2, float4 w2m, float4 o) {
    const float left = __shfl_up_sync(0xffffffffu, w1.w, 1);
    const float gy = (sd.y0 + li < n2 - 1) ? 1.f : 0.f;
    const float rowok = (li >= 0 && li < ap) ? 1.f : 0.f;
    float4 u;
    u.x = rowok * mP[0] * (xk[0] * w1.x - left + gy * w2.x - w2m.x - o.x);
    u.y = rowok * mP[1] * (xk[1] * w1.y - w1.x + gy * w2.y - w2m.y - o.y);
    u.z = rowok * mP[2] * (xk[2] * w1.z - w1.y + gy * w2.z - w2m.z - o.z);
    u.w = rowok * mP[3] * (xk[3] * w1.w - w1.z + gy * w2.w - w2m.w - o.w);
    return u;
  };
  const bool lastx[4] = {j0 + 1 >= bp, j0 + 2 >= bp, j0 + 3 >= bp, j0 + 4 >= bp};
  // one Chambolle update of row li from u at li and li + 1 (theta = 0 outside S)
  auto upd = [&](int li, V2 w, float4 u_c, float4 u_n) {
    const float ur = __shfl_down_sync(0xffffffffu, u_c.x, 1);
    const float ydiff = (li + 1 < ap) ? 1.f : 0.f;
    const float psx0 = lastx[0] ? 0.f : u_c.y - u_c.x, psy0 = ydiff * (u_n.x - u_c.x);
    const float psx1 = lastx[1] ? 0.f : u_c.z - u_c.y, psy1 = ydiff * (u_n.y - u_c.y);
    const float psx2 = lastx[2] ? 0.f : u_c.w - u_c.z, psy2 = ydiff * (u_n.z - u_c.z);
    const float psx3 = lastx[3] ? 0.f : ur - u_c.w, psy3 = ydiff * (u_n.w - u_c.w);
    const float ty = (li >= 0 && li < a) ? thy[sd.iy * g.A + li] : 0.f;
    ball_update_fast(ty * thc[0], t, psx0, psy0, w.w1.x, w.w2.x);
    ball_update_fast(ty * thc[1], t, psx1, psy1, w.w1.y, w.w2.y);
    ball_update_fast(ty * thc[2], t, psx2, psy2, w.w1.z, w.w2.z);
    ball_update_fast(ty * thc[3], t, psx3, psy3, w.w1.w, w.w2.w);
    return w;
  };
  // ---- warm-up: raw rows r0-2 .. r0+2, level 1 on r0-1 and r0, level-2 u' on r0
  const Raw Rm2 = ldraw(r0 - 2), Rm1 = ldraw(r0 - 1), R0 = ldraw(r0);
  Raw Rn = ldraw(r0 + 1), Rm = ldraw(r0 + 2);
  const float4 u_m1 = ucalc(r0 - 1, Rm1.w1, Rm1.w2, Rm2.w2, Rm1.o);
  const float4 u_0 = ucalc(r0, R0.w1, R0.w2, Rm1.w2, R0.o);
  float4 u_n = ucalc(r0 + 1, Rn.w1, Rn.w2, R0.w2, Rn.o);
  const V2 vp_m1 = upd(r0 - 1, V2{Rm1.w1, Rm1.w2}, u_m1, u_0);
  V2 vp_c = upd(r0, V2{R0.w1, R0.w2}, u_0, u_n);
  float4 up_c = ucalc(r0, vp_c.w1, vp_c.w2, vp_m1.w2, R0.o);
  for (int li = r0; li < r1; ++li) {
    const Raw Rq = ldraw(li + 3);
    const float4 u_m = ucalc(li + 2, Rm.w1, Rm.w2, Rn.w2, Rm.o);           // level 1, row li+2
    const V2 vp_n = upd(li + 1, V2{Rn.w1, Rn.w2}, u_n, u_m);               // level 1, row li+1
    const float4 up_n = ucalc(li + 1, vp_n.w1, vp_n.w2, vp_c.w2, Rn.o);    // level 2 u, row li+1
    const V2 vo = upd(li, vp_c, up_c, up_n);                               // level 2, row li
    if (out_lane) {
      float *q1 = o1 + (size_t)li * g.ldS + j0, *q2 = o2 + (size_t)li * g.ldS + j0;
      if (fullS) {
        *reinterpret_cast<float4 *>(q1) = vo.w1;
        *reinterpret_cast<float4 *>(q2) = vo.w2;
      } else {
        if (mS[0] != 0.f) { q1[0] = vo.w1.x; q2[0] = vo.w2.x; }
        if (mS[1] != 0.f) { q1[1] = vo.w1.y; q2[1] = vo.w2.y; }
        if (mS[2] != 0.f) { q1[2] = vo.w1.z; q2[2] = vo.w2.z; }
        if (mS[3] != 0.f) { q1[3] = vo.w1.w; q2[3] = vo.w2.w; }
      }
    }
    Rn = Rm;
    Rm = Rq;
    u_n = u_m;
    vp_c = vp_n;
    up_c = up_n;
  }
}


// Sum over the local layout-row ky of sum_kx qhat (subdomains stored column-major per rank:
// m = kx * m2loc + (ky - k0)).
__device__ __forceinline__ float ky_part(const float *__restrict__ q, const Geo &g, int planes,
                                         int c, int ky, int k0, int m2loc, int i, int j,
                                         int2 cx, const int *__restrict__ loy,
                                         const int *__restrict__ lox) {
  float part = 0.f;
  for (int kx = cx.x; kx < cx.x + cx.y; ++kx) {
    const int m = kx * m2loc + (ky - k0);
    const int li = i - loy[ky], lj = j - lox[kx];
    part += q[(((size_t)m * planes + c) * g.A + li) * g.ldS + lj];
  }
  return part;
}

// p^{n+1} = (1 - ahat) p^n + ahat sum_m E qhat_m (Alg. 2) on rows [row0, row1).  The sum
// is grouped as sum_ky (sum_kx qhat) in ascending ky, where the parts of layout rows owned by the
// slab neighbours (ky < k0: `up`, ky >= k1: `dn`, rows [*_r0, *_r1)) arrive as partial sums over
// NCCL -- so overlaps are bitwise identical for every GPU count.  Flags non-finite values.
// Four consecutive columns per thread: float4 loads and stores whenever the quad has one x-cover
// and its subdomain rows are 16-byte aligned (every interior quad of a strip layout), else the
// columns one by one.  Per element the same operations in the same order either way.
template <int C>
__global__ void k_combine(const SubDesc *__restrict__ subs, Geo g,
                          const int2 *__restrict__ covy, const int2 *__restrict__ covx,
                          const int *__restrict__ loy, const int *__restrict__ lox, int m2loc,
                          int k0, int k1, const float *__restrict__ q, float *__restrict__ p,
                          int ld, int n2, int row0, int row1, int n1, float ahat, int *bad,
                          const float *__restrict__ up, int up_r0, int up_r1,
                          const float *__restrict__ dn, int dn_r0, int dn_r1) {
  const int jq = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int i = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= row1 || jq >= n1) return;
  const int2 cy = covy[i];
  const size_t qpl = (size_t)g.A * g.ldS;   // plane stride inside one subdomain's block
  const int2 cx = covx[jq];
  bool quad = jq + 3 < n1;
  if (quad) {
    const int2 cx3 = covx[jq + 3];
    quad = cx3.x == cx.x && cx3.y == cx.y && ((jq - lox[cx.x]) & 3) == 0 &&
           (cx.y < 2 || ((jq - lox[cx.x + 1]) & 3) == 0);
  }
  bool finite = true;
  if (quad) {
    // every load is issued before the sums: p first, then the (at most 2 x 2, layout check)
    // covering subdomains' values
    float4 pv[C];
#pragma unroll
    for (int c = 0; c < C; ++c)
      pv[c] = *reinterpret_cast<const float4 *>(p + (size_t)c * n2 * ld + (size_t)i * ld + jq);
    float4 acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (t >= cy.y) break;
      const int ky = cy.x + t;
      float4 part[C];
#pragma unroll
      for (int c = 0; c < C; ++c) part[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ky < k0) {
        if (i >= up_r0 && i < up_r1)
#pragma unroll
          for (int c = 0; c < C; ++c)
            part[c] = *reinterpret_cast<const float4 *>(up + ((size_t)c * (up_r1 - up_r0) + (i - up_r0)) * ld + jq);
      } else if (ky >= k1) {
        if (i >= dn_r0 && i < dn_r1)
#pragma unroll
          for (int c = 0; c < C; ++c)
            part[c] = *reinterpret_cast<const float4 *>(dn + ((size_t)c * (dn_r1 - dn_r0) + (i - dn_r0)) * ld + jq);
      } else {   // sum over kx of this layout row (same grouping as k_partial)
        const int li = i - loy[ky];
        const float *qa = q + ((size_t)(cx.x * m2loc + (ky - k0)) * C * g.A + li) * g.ldS + (jq - lox[cx.x]);
        float4 av[C], bv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) av[c] = __ldg(reinterpret_cast<const float4 *>(qa + c * qpl));
        if (cx.y > 1) {
          const int kx = cx.x + 1;
          const float *qb = q + ((size_t)(kx * m2loc + (ky - k0)) * C * g.A + li) * g.ldS + (jq - lox[kx]);
#pragma unroll
          for (int c = 0; c < C; ++c) bv[c] = __ldg(reinterpret_cast<const float4 *>(qb + c * qpl));
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          part[c].x += av[c].x; part[c].y += av[c].y; part[c].z += av[c].z; part[c].w += av[c].w;
          if (cx.y > 1) {
            part[c].x += bv[c].x; part[c].y += bv[c].y; part[c].z += bv[c].z; part[c].w += bv[c].w;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        acc[c].x += part[c].x; acc[c].y += part[c].y; acc[c].z += part[c].z; acc[c].w += part[c].w;
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float4 v;
      v.x = (1.f - ahat) * pv[c].x + ahat * acc[c].x;
      v.y = (1.f - ahat) * pv[c].y + ahat * acc[c].y;
      v.z = (1.f - ahat) * pv[c].z + ahat * acc[c].z;
      v.w = (1.f - ahat) * pv[c].w + ahat * acc[c].w;
      finite = finite && isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
      *reinterpret_cast<float4 *>(p + (size_t)c * n2 * ld + (size_t)i * ld + jq) = v;
    }
  } else {
    for (int j = jq; j < min(jq + 4, n1); ++j) {
      const int2 cxj = covx[j];
      float pv[C];
#pragma unroll
      for (int c = 0; c < C; ++c) pv[c] = p[(size_t)c * n2 * ld + (size_t)i * ld + j];
      float acc[C];
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0.f;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (t >= cy.y) break;
        const int ky = cy.x + t;
        float part[C];
#pragma unroll
        for (int c = 0; c < C; ++c) part[c] = 0.f;
        if (ky < k0) {
          if (i >= up_r0 && i < up_r1)
#pragma unroll
            for (int c = 0; c < C; ++c) part[c] = up[((size_t)c * (up_r1 - up_r0) + (i - up_r0)) * ld + j];
        } else if (ky >= k1) {
          if (i >= dn_r0 && i < dn_r1)
#pragma unroll
            for (int c = 0; c < C; ++c) part[c] = dn[((size_t)c * (dn_r1 - dn_r0) + (i - dn_r0)) * ld + j];
        } else {
          const int li = i - loy[ky];
          const float *qa = q + ((size_t)(cxj.x * m2loc + (ky - k0)) * C * g.A + li) * g.ldS + (j - lox[cxj.x]);
          float av[C], bv[C];
#pragma unroll
          for (int c = 0; c < C; ++c) av[c] = __ldg(qa + c * qpl);
          if (cxj.y > 1) {
            const int kx = cxj.x + 1;
            const float *qb = q + ((size_t)(kx * m2loc + (ky - k0)) * C * g.A + li) * g.ldS + (j - lox[kx]);
#pragma unroll
            for (int c = 0; c < C; ++c) bv[c] = __ldg(qb + c * qpl);
          }
#pragma unroll
          for (int c = 0; c < C; ++c) {
            part[c] += av[c];
            if (cxj.y > 1) part[c] += bv[c];
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] += part[c];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const size_t idx = (size_t)c * n2 * ld + (size_t)i * ld + j;
        const float v = (1.f - ahat) * pv[c] + ahat * acc[c];
        finite = finite && isfinite(v);
        p[idx] = v;
      }
    }
  }
  if (!finite) atomicOr(bad, 1);
}

// Partial sums of the local subdomains on rows [ra, rb) for a slab neighbour:
// out[c][i - ra][j] = sum_{local ky covering i} sum_kx qhat (same grouping as k_combine).
__global__ void k_partial(const SubDesc *__restrict__ subs, Geo g, int planes,
                          const int2 *__restrict__ covy, const int2 *__restrict__ covx,
                          const int *__restrict__ loy, const int *__restrict__ lox, int m2loc,
                          int k0, int k1, const float *__restrict__ q, int ra, int rb, int n1,
                          int ld, float *__restrict__ out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = ra + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= rb || j >= n1) return;
  int2 cy = covy[i], cx = covx[j];
  for (int c = 0; c < planes; ++c) {
    float acc = 0.f;
    for (int ky = cy.x; ky < cy.x + cy.y; ++ky)
      if (ky >= k0 && ky < k1) acc += ky_part(q, g, planes, c, ky, k0, m2loc, i, j, cx, loy, lox);
    out[((size_t)c * (rb - ra) + (i - ra)) * ld + j] = acc;
  }
}

// d = d0 - div p / alpha.
// d = d0 - (div p + shift) / alpha (IRV1: shift = div xi, Eq. tau_hat)
__global__ void k_recover2(const float *__restrict__ d0, const float *__restrict__ p1,
                           const float *__restrict__ p2, int ld, int n2, int n1, float inv_alpha,
                           const float *__restrict__ shift, float *__restrict__ d, int row0,
                           int row1) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= row1 || j >= n1) return;
  auto P1 = [&](int a, int b) { return p1[(size_t)a * ld + b]; };
  auto P2 = [&](int a, int b) { return p2[(size_t)a * ld + b]; };
  float dv = (j < n1 - 1 ? P1(i, j) : 0.f) - (j > 0 ? P1(i, j - 1) : 0.f) +
             (i < n2 - 1 ? P2(i, j) : 0.f) - (i > 0 ? P2(i - 1, j) : 0.f);
  const float sh = shift ? shift[(size_t)i * ld + j] : 0.f;
  d[(size_t)i * n1 + j] = d0[(size_t)i * n1 + j] - (dv + sh) * inv_alpha;
}

// ----------------------------------------------------------------------------- dual energies

// Deterministic fp64 reductions for the dual energies D(p) of Eq. opt_dual_discrete:
// per-block partial sums in a fixed grid order, then one block sums the partials in order.
constexpr int RED_T = 256;
__device__ __forceinline__ void block_sum_store(double v, double *out) {
  __shared__ double sh[RED_T / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RED_T / 32; ++w) t += sh[w];
    *out = t;
  }
}
// Step 2: sum over rows [row0, row1) of (div p - f)^2 (three-case D-).
__global__ void __launch_bounds__(RED_T)
k_dual2_partial(const float *__restrict__ p1, const float *__restrict__ p2, const float *__restrict__ f,
                int ld, int n2, int n1, int row0, int row1, double *__restrict__ part) {
  double acc = 0.0;
  const long long total = (long long)(row1 - row0) * n1;
  for (long long e = (long long)blockIdx.x * RED_T + threadIdx.x; e < total;
       e += (long long)gridDim.x * RED_T) {
    const int i = row0 + (int)(e / n1), j = (int)(e % n1);
    const size_t o = (size_t)i * ld + j;
    const float dv = (j < n1 - 1 ? p1[o] : 0.f) - (j > 0 ? p1[o - 1] : 0.f) +
                     (i < n2 - 1 ? p2[o] : 0.f) - (i > 0 ? p2[o - ld] : 0.f);
    const double r = (double)dv - (double)f[o];
    acc += r * r;
  }
  block_sum_store(acc, part + blockIdx.x);
}
// Step 1: D_TFS(p^n) = ||r^n||^2 with r^n = f - P multidiv p^n (two planes, rows [row0, row1)).
__global__ void __launch_bounds__(RED_T)
k_sumsq2_partial(const float *__restrict__ r, size_t plane, int ld, int n1, int row0, int row1,
                 double *__restrict__ part) {
  double acc = 0.0;
  const long long total = (long long)(row1 - row0) * n1;
  for (long long e = (long long)blockIdx.x * RED_T + threadIdx.x; e < total;
       e += (long long)gridDim.x * RED_T) {
    const size_t o = (size_t)(row0 + (int)(e / n1)) * ld + (int)(e % n1);
    const double a = r[o], b = r[o + plane];
    acc += a * a + b * b;
  }
  block_sum_store(acc, part + blockIdx.x);
}
// Zero-mean convention of g (reading A3): the integrated g of k_irv2_f has
// g[0][0] = 0; with f = alpha (d0 - g), mean(g) = mean(d0) - mean(f)/alpha, so f + alpha mean(g)
// is alpha (d0 - (g - mean g)).  Partials of (sum f, sum d0) per block.
__global__ void __launch_bounds__(RED_T)
k_sum_fd_partial(const float *__restrict__ f, int ldf, const float *__restrict__ d0, int n2, int n1,
                 double *__restrict__ part) {
  double sf = 0.0, sd = 0.0;
  const long long total = (long long)n2 * n1;
  for (long long e = (long long)blockIdx.x * RED_T + threadIdx.x; e < total;
       e += (long long)gridDim.x * RED_T) {
    const int i = (int)(e / n1), j = (int)(e % n1);
    sf += f[(size_t)i * ldf + j];
    sd += d0[e];
  }
  block_sum_store(sf, part + 2 * blockIdx.x);
  __syncthreads();
  block_sum_store(sd, part + 2 * blockIdx.x + 1);
}
__global__ void k_fd_shift(const double *__restrict__ part, int nb, double alpha, double npix,
                           double *__restrict__ shift) {
  if (threadIdx.x != 0) return;
  double sf = 0.0, sd = 0.0;
  for (int b = 0; b < nb; ++b) {
    sf += part[2 * b];
    sd += part[2 * b + 1];
  }
  *shift = alpha * (sd / npix) - sf / npix;   // alpha mean(g)
}
__global__ void k_add_shift(float *__restrict__ f, int ldf, int n2, int n1,
                            const double *__restrict__ shift) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= n2 || j >= n1) return;
  f[(size_t)i * ldf + j] = (float)((double)f[(size_t)i * ldf + j] + *shift);
}
__global__ void __launch_bounds__(RED_T) k_sum_partials(const double *__restrict__ part, int n,
                                                        double *__restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += RED_T) acc += part[i];   // fixed assignment per thread
  block_sum_store(acc, out);
}

// Primal energies and duality gaps (SURVEY C-13, C-15), fp64 terms per pixel, fixed-order block
// partials.  For a scalar field u with dual row q = (q_x, q_y) at pixel (i, j): grad u = (D+_x u,
// D+_y u) with the forward difference zero at the last index (Eq. defGradDis),
// TV term |grad u| (channel-wise TV, reading A15) and gap term |grad u| + q . grad u >= 0
// (TV(u) = sup_{|q| <= 1} -<grad u, q>, so the gap vanishes iff q attains the sup).
__device__ __forceinline__ void tv_gap_terms(double u, double ur, double ud, double qx, double qy,
                                             double &tv, double &gap) {
  const double gx = ur - u, gy = ud - u;
  const double nrm = sqrt(gx * gx + gy * gy);
  tv += nrm;
  gap += nrm + qx * gx + qy * gy;
}
__device__ __forceinline__ void block_sum_store3(double a, double b, double c, double *out,
                                                 int stride) {
  block_sum_store(a, out);
  __syncthreads();
  block_sum_store(b, out + stride);
  __syncthreads();
  block_sum_store(c, out + 2 * stride);
}
// Step 1 (Cor. tfsdual P:245-249): over rows [row0, row1) of Omega~, per block
//   part[0][b] = sum_k TV-terms of tau_k,  part[1][b] = sum (tau - P tau_0)^2 with P tau_0 = delta f,
//   part[2][b] = sum_k gap-terms of (tau_k, p_k);
// E_1 = part0 + part1 / (2 delta) is formed by the host after the sums (and the ranks' all-reduce).
__global__ void __launch_bounds__(RED_T)
k_primal1_partial(const float *__restrict__ tau, size_t plane, int ld, const float *__restrict__ f,
                  const float *__restrict__ p, int n2, int n1, int row0, int row1, float delta,
                  float scale, double *__restrict__ part) {
  double tv = 0.0, fit = 0.0, gap = 0.0;
  const long long total = (long long)(row1 - row0) * n1;
  for (long long e = (long long)blockIdx.x * RED_T + threadIdx.x; e < total;
       e += (long long)gridDim.x * RED_T) {
    const int i = row0 + (int)(e / n1), j = (int)(e % n1);
    const size_t o = (size_t)i * ld + j;
    for (int k = 0; k < 2; ++k) {
      const float *t = tau + k * plane;
      const double u = (double)scale * t[o];   // tau = scale * the plane (1 or delta)
      const double ur = j < n1 - 1 ? (double)scale * t[o + 1] : u;
      const double ud = i < n2 - 1 ? (double)scale * t[o + ld] : u;
      tv_gap_terms(u, ur, ud, p[2 * k * plane + o], p[(2 * k + 1) * plane + o], tv, gap);
      const double r = u - (double)delta * (double)f[k * plane + o];
      fit += r * r;
    }
  }
  block_sum_store3(tv, fit, gap, part + blockIdx.x, gridDim.x);
}
// Step 2 over rows [row0, row1) of Omega: u = d - g (IRV2, Eq. modifiedStep2; with
// f = alpha (d_0 - g): g = d_0 - f / alpha) or u = d (IRV1, Eq. IRPXi, dxi != null);
//   part[0][b] = TV-terms of u, part[1][b] = sum (d - d_0)^2, part[2][b] = gap-terms of (u, p),
//   part[3][b] = sum d * div xi (IRV1; 0 for IRV2).
// E_2 = part0 + alpha/2 part1 (+ part3 for IRV1), formed by the host.
__global__ void __launch_bounds__(RED_T)
k_primal2_partial(const float *__restrict__ d, const float *__restrict__ d0,
                  const float *__restrict__ f, const float *__restrict__ dxi,
                  const float *__restrict__ p1, const float *__restrict__ p2, int ldf, int n2,
                  int n1, int row0, int row1, float inv_alpha, double *__restrict__ part) {
  double tv = 0.0, fit = 0.0, gap = 0.0, cross = 0.0;
  const long long total = (long long)(row1 - row0) * n1;
  auto U = [&](int i, int j) -> double {
    const size_t e = (size_t)i * n1 + j;
    if (dxi) return (double)d[e];
    return (double)d[e] - (double)d0[e] + (double)f[(size_t)i * ldf + j] * (double)inv_alpha;
  };
  for (long long e = (long long)blockIdx.x * RED_T + threadIdx.x; e < total;
       e += (long long)gridDim.x * RED_T) {
    const int i = row0 + (int)(e / n1), j = (int)(e % n1);
    const size_t o = (size_t)i * ldf + j, od = (size_t)i * n1 + j;
    const double u = U(i, j);
    const double ur = j < n1 - 1 ? U(i, j + 1) : u;
    const double ud = i < n2 - 1 ? U(i + 1, j) : u;
    tv_gap_terms(u, ur, ud, p1[o], p2[o], tv, gap);
    const double r = (double)d[od] - (double)d0[od];
    fit += r * r;
    if (dxi) cross += (double)d[od] * (double)dxi[o];
  }
  block_sum_store3(tv, fit, gap, part + blockIdx.x, gridDim.x);
  __syncthreads();
  block_sum_store(cross, part + 3 * gridDim.x + blockIdx.x);
}
// out[q] = sum of part[q][0..n) in a fixed order, one block per quantity q.
__global__ void __launch_bounds__(RED_T) k_sum_partials_multi(const double *__restrict__ part, int n,
                                                              double *__restrict__ out) {
  const double *pq = part + (size_t)blockIdx.x * n;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += RED_T) acc += pq[i];
  block_sum_store(acc, out + blockIdx.x);
}

// out[i] = sum over ranks q = 0..world-1, in that order, of vals[q * stride + i] (the virtual
// group's all-reduce; every rank forms the same fixed-order sum).
__global__ void k_sum_ranks(const double *__restrict__ vals, int world, int stride, int n,
                            double *__restrict__ out) {
  const int i = threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int q = 0; q < world; ++q) acc += vals[(size_t)q * stride + i];
  out[i] = acc;
}

// ----------------------------------------------------------------------------- step 1 (TFS)

// w = multidiv p: w_k = div(p_k1, p_k2); p has 4 planes [p11 p12 p21 p22].
__global__ void k_multidiv(const float *__restrict__ p, int ld, int n2, int n1,
                           float *__restrict__ w, int row0, int row1) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= row1 || j >= n1) return;
  size_t pl = (size_t)n2 * ld;
  for (int k = 0; k < 2; ++k) {
    const float *px = p + (2 * k) * pl, *py = p + (2 * k + 1) * pl;
    float dv = (j < n1 - 1 ? px[(size_t)i * ld + j] : 0.f) - (j > 0 ? px[(size_t)i * ld + j - 1] : 0.f) +
               (i < n2 - 1 ? py[(size_t)i * ld + j] : 0.f) - (i > 0 ? py[(size_t)(i - 1) * ld + j] : 0.f);
    w[k * pl + (size_t)i * ld + j] = dv;
  }
}

// q = div w.
__global__ void k_div(const float *__restrict__ w1, const float *__restrict__ w2, int ld, int n2,
                      int n1, float *__restrict__ q, float *__restrict__ qlo, int row0, int row1) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= row1 || j >= n1) return;
  float dv = (j < n1 - 1 ? w1[(size_t)i * ld + j] : 0.f) - (j > 0 ? w1[(size_t)i * ld + j - 1] : 0.f) +
             (i < n2 - 1 ? w2[(size_t)i * ld + j] : 0.f) - (i > 0 ? w2[(size_t)(i - 1) * ld + j] : 0.f);
  store_split(q, qlo, (size_t)i * ld + j, dv);
}

// out = sa a + sb b (+ sc c), two planes.
__global__ void k_axpby2(const float *__restrict__ a, const float *__restrict__ b,
                         const float *__restrict__ c, int ld, int n2, int n1, float sa, float sb,
                         float sc, float *__restrict__ out, int row0, int row1) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= row1 || j >= n1) return;
  size_t pl = (size_t)n2 * ld;
  for (int k = 0; k < 2; ++k) {
    size_t idx = k * pl + (size_t)i * ld + j;
    float v = sa * a[idx] + sb * b[idx];
    if (c) v += sc * c[idx];
    out[idx] = v;
  }
}

// v_m = R_S (theta_m p^n) (4 planes) -- the argument of the omega0 projection (Alg. 5).
__global__ void k_load_tp(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ thy,
                          const float *__restrict__ thx, const float *__restrict__ p, int ld,
                          int n2, float *__restrict__ v) {
  const SubDesc sd = subs[blockIdx.z];
  int lj = blockIdx.x * blockDim.x + threadIdx.x;
  int li = blockIdx.y * blockDim.y + threadIdx.y;
  int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  if (li >= a || lj >= b) return;
  float th = theta_at(thy, thx, sd, g, li, lj);
  size_t pl = (size_t)n2 * ld;
  for (int c = 0; c < 4; ++c)
    v[(((size_t)blockIdx.z * 4 + c) * g.A + li) * g.ldS + lj] =
        th * p[c * pl + (size_t)(sd.y0 + li) * ld + sd.x0 + lj];
}

// Pre-div of Alg. 5: q = div_T E_{S+} multidiv_{S+} E_S v on T.  Both divergences use
// the global rules (resDiv), so the result equals the global div of the
// zero-extended field restricted to T.
__device__ __forceinline__ float w_S(const float *vb, int k, int li, int lj, int gi, int gj,
                                     int a, int b, const Geo &g, int n2, int n1) {
  const float *vx = vb + (size_t)(2 * k) * g.A * g.ldS;
  const float *vy = vx + (size_t)g.A * g.ldS;
  return div_S(vx, vy, li, lj, gi, gj, a, b, g.ldS, n2, n1);
}


// omega0_loc = R_{S+} r^n + (R_{S+} P E_{S+}) multidiv_{S+} E_S (theta_m p^n)  (Alg. 5, P:1740;
// r^n = f - P multidiv p^n is the global part, reading A11), with P w = w - grad phi.  The inner
// loop only ever needs grad phi(v) + omega0, and the local projection is linear, so this kernel
// stores the projection-free part c = R r^n + multidiv(theta p) and every inner update projects
// q(v) - q(theta p) (k_prediv1s with qsub) and adds c: the same sum, one projection per sweep and
// subdomain group fewer than projecting theta p on its own.
__global__ void k_omega0_1(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ r,
                           int ld, const float *__restrict__ v, int n2, int n1,
                           float *__restrict__ om) {
  const SubDesc sd = subs[blockIdx.z];
  int lj = blockIdx.x * blockDim.x + threadIdx.x;
  int li = blockIdx.y * blockDim.y + threadIdx.y;
  int gi = sd.y0 + li, gj = sd.x0 + lj;
  if (gi > sd.py1 || gj > sd.px1) return;
  int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  const float *vb = v + (size_t)blockIdx.z * 4 * g.A * g.ldS;
  size_t pl = (size_t)n2 * ld;
  for (int k = 0; k < 2; ++k) {
    const float w = w_S(vb, k, li, lj, gi, gj, a, b, g, n2, n1);
    om[(((size_t)blockIdx.z * 2 + k) * g.AP + li) * g.ldP + lj] = r[k * pl + (size_t)gi * ld + gj] + w;
  }
}


// Streaming forms of the step-1 stencils (default): lane l owns the column pair
// (c0 - 2 + 2l, c0 - 1 + 2l) of the subdomain-local grid, lanes 1..30 produce 60 output
// columns, lane 0 / lane 31 are halo columns, and each warp walks RB rows with the next rows'
// loads in flight (same scheme as k_sweep2v).
constexpr int S1_OUT = 60, S1_WARPS = 4;
// kernel (a') is capped at 64 registers (eight CTAs per SM, 32 warps): 510 -> 486 us per config-4
// update, bitwise the same (78 registers and six CTAs otherwise; 7 CTAs: 495 us)
constexpr int S1_MINB = 8;

struct PairCtx {
  int jA, jB;
  bool SA, SB, PA, PB;
  float xkA, xkB;
};

// Branch-free variant: one 8-byte load from a clamped address (inside the row pitch: jA is even and
// ld a multiple of 4, so an in-range pair is never moved), then the masks.  Faster in the pre-div
// (-7 %), slower in kernel (a') (+14 % at config 4), so only the pre-div uses it.
__device__ __forceinline__ float2 ld_pair_nb(const float *__restrict__ base, int ld, int li,
                                             int rows, const PairCtx &pc, bool okA, bool okB) {
  const bool rok = li >= 0 && li < rows;
  const int lc = min(max(li, 0), rows - 1), jc = min(max(pc.jA, 0), ld - 2);
  const float2 x = __ldg(reinterpret_cast<const float2 *>(base + (size_t)lc * ld + jc));
  return make_float2(rok && okA ? x.x : 0.f, rok && okB ? x.y : 0.f);
}

__device__ __forceinline__ float2 ld_pair(const float *__restrict__ base, int ld, int li, int rows,
                                          const PairCtx &pc, bool okA, bool okB) {
  float2 r = make_float2(0.f, 0.f);
  if (li < 0 || li >= rows) return r;
  const float *p = base + (size_t)li * ld + pc.jA;
  if (okA && okB) return __ldg(reinterpret_cast<const float2 *>(p));
  if (okA) r.x = __ldg(p);
  if (okB) r.y = __ldg(p + 1);
  return r;
}

// global-rule divergence of (vx, vy) for the lane's pair at row li, given vy of row li - 1
__device__ __forceinline__ float2 div_pair(const PairCtx &pc, int gi, int n2, float2 vx, float2 vy,
                                           float2 vym) {
  const float leftA = __shfl_up_sync(0xffffffffu, vx.y, 1);
  const float gy = (gi < n2 - 1) ? 1.f : 0.f;
  return make_float2(pc.xkA * vx.x - leftA + gy * vy.x - vym.x,
                     pc.xkB * vx.y - vx.x + gy * vy.y - vym.y);
}

// q = div_T E_{S+} multidiv E_S v on T (Alg. 5 pre-div), minus qsub when given (the
// inner loop passes the pre-div of theta_m p^n: the projection is linear, so one projection of
// q(v) - q(theta p) gives grad phi(v) - grad phi(theta p), see step1_impl)
__global__ void __launch_bounds__(32 * S1_WARPS)
k_prediv1s(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ v, int n2, int n1,
           float *__restrict__ q, const float *__restrict__ qsub, int rb) {
  const SubDesc sd = subs[blockIdx.z];
  const int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  const int at = sd.ty1 - sd.y0 + 1, bt = sd.tx1 - sd.x0 + 1;
  const int lane = threadIdx.x, strip = blockIdx.x * S1_WARPS + threadIdx.y;
  const int c0 = strip * S1_OUT;
  if (c0 >= bt) return;
  const int r0 = blockIdx.y * rb;
  if (r0 >= at) return;
  const int r1 = min(at, r0 + rb);
  PairCtx pc;
  pc.jA = c0 - 2 + 2 * lane;
  pc.jB = pc.jA + 1;
  pc.SA = pc.jA >= 0 && pc.jA < b;
  pc.SB = pc.jB >= 0 && pc.jB < b;
  pc.xkA = (sd.x0 + pc.jA < n1 - 1) ? 1.f : 0.f;
  pc.xkB = (sd.x0 + pc.jB < n1 - 1) ? 1.f : 0.f;
  const bool outA = lane >= 1 && lane <= 30 && pc.jA < bt;
  const bool outB = lane >= 1 && lane <= 30 && pc.jB < bt;
  const float *vb = v + (size_t)blockIdx.z * 4 * g.A * g.ldS;
  const size_t pl = (size_t)g.A * g.ldS;
  struct Row { float2 a11, a12, a21, a22; };
  auto ldrow = [&](int li) {
    Row r;
    r.a11 = ld_pair_nb(vb, g.ldS, li, a, pc, pc.SA, pc.SB);
    r.a12 = ld_pair_nb(vb + pl, g.ldS, li, a, pc, pc.SA, pc.SB);
    r.a21 = ld_pair_nb(vb + 2 * pl, g.ldS, li, a, pc, pc.SA, pc.SB);
    r.a22 = ld_pair_nb(vb + 3 * pl, g.ldS, li, a, pc, pc.SA, pc.SB);
    return r;
  };
  // w_k = div(v_k1, v_k2) at row li needs v_k2 at li - 1
  Row pm = ldrow(r0 - 2), c = ldrow(r0 - 1);
  float2 w2p = div_pair(pc, sd.y0 + r0 - 1, n2, c.a21, c.a22, pm.a22);   // w_2 at row r0 - 1
  Row n = ldrow(r0);
  const int qo = sd.x0 & 3;
  float *qb = q + (size_t)blockIdx.z * g.AT * g.ldT + qo;
  const float *qsb = qsub ? qsub + (size_t)blockIdx.z * g.AT * g.ldT + qo : nullptr;
  for (int li = r0; li < r1; ++li) {
    const Row m = ldrow(li + 1);
    const int gi = sd.y0 + li;
    const float2 w1 = div_pair(pc, gi, n2, n.a11, n.a12, c.a12);
    const float2 w2 = div_pair(pc, gi, n2, n.a21, n.a22, c.a22);
    const float w1left = __shfl_up_sync(0xffffffffu, w1.y, 1);
    const float gxA = (sd.x0 + pc.jA > 0) ? 1.f : 0.f;
    const float gyk = (gi < n2 - 1) ? 1.f : 0.f, gyp = (gi > 0) ? 1.f : 0.f;
    const float qA = pc.xkA * w1.x - gxA * w1left + gyk * w2.x - gyp * w2p.x;
    const float qB = pc.xkB * w1.y - w1.x + gyk * w2.y - gyp * w2p.y;
    const size_t o = (size_t)li * g.ldT + pc.jA;
    if (outA) qb[o] = qsb ? qA - __ldg(qsb + o) : qA;
    if (outB) qb[o + 1] = qsb ? qB - __ldg(qsb + o + 1) : qB;
    w2p = w2;
    c = n;
    n = m;
  }
}

// Kernel (a') streaming form: rho_k = w_k - grad phi_k - omega0_k on S+, psi_k = grad rho_k,
// row-wise ball update of (v_k1, v_k2) (Alg. 5)
template <bool OM>
__global__ void __launch_bounds__(32 * S1_WARPS, S1_MINB)
k_sweep1s(const SubDesc *__restrict__ subs, Geo g, const float *__restrict__ thy,
          const float *__restrict__ thx, const float *__restrict__ vin,
          const float *__restrict__ gphi, int ldg, const float *__restrict__ om,
          float *__restrict__ vout, int n2, int n1, float t, int rb) {
  const SubDesc sd = subs[blockIdx.z];
  const int a = sd.y1 - sd.y0 + 1, b = sd.x1 - sd.x0 + 1;
  const int ap = sd.py1 - sd.y0 + 1, bp = sd.px1 - sd.x0 + 1;
  const int lane = threadIdx.x, strip = blockIdx.x * S1_WARPS + threadIdx.y;
  const int c0 = strip * S1_OUT;
  if (c0 >= b) return;
  const int r0 = blockIdx.y * rb;
  if (r0 >= a) return;
  const int r1 = min(a, r0 + rb);
  PairCtx pc;
  pc.jA = c0 - 2 + 2 * lane;
  pc.jB = pc.jA + 1;
  pc.SA = pc.jA >= 0 && pc.jA < b;
  pc.SB = pc.jB >= 0 && pc.jB < b;
  pc.PA = pc.jA >= 0 && pc.jA < bp;
  pc.PB = pc.jB >= 0 && pc.jB < bp;
  pc.xkA = (sd.x0 + pc.jA < n1 - 1) ? 1.f : 0.f;
  pc.xkB = (sd.x0 + pc.jB < n1 - 1) ? 1.f : 0.f;
  const bool outA = lane >= 1 && lane <= 30 && pc.jA < b;
  const bool outB = lane >= 1 && lane <= 30 && pc.jB < b;
  const float *vb = vin + (size_t)blockIdx.z * 4 * g.A * g.ldS;
  float *ob = vout + (size_t)blockIdx.z * 4 * g.A * g.ldS;
  const size_t pl = (size_t)g.A * g.ldS;
  const float *g1 = gphi + ((size_t)0 * g.MG + blockIdx.z) * g.AP * ldg;
  const float *g2 = gphi + ((size_t)1 * g.MG + blockIdx.z) * g.AP * ldg;
  const float *o1 = OM ? om + ((size_t)blockIdx.z * 2 + 0) * g.AP * g.ldP : nullptr;
  const float *o2 = OM ? om + ((size_t)blockIdx.z * 2 + 1) * g.AP * g.ldP : nullptr;
  const float thA = pc.SA ? thx[sd.ix * g.B + pc.jA] : 0.f;
  const float thB = pc.SB ? thx[sd.ix * g.B + pc.jB] : 0.f;
  struct Row { float2 a11, a12, a21, a22, h1, h2; };   // h_k = grad phi_k + omega0_k
  auto ldrow = [&](int li) {
    Row r;
    r.a11 = ld_pair(vb, g.ldS, li, a, pc, pc.SA, pc.SB);
    r.a12 = ld_pair(vb + pl, g.ldS, li, a, pc, pc.SA, pc.SB);
    r.a21 = ld_pair(vb + 2 * pl, g.ldS, li, a, pc, pc.SA, pc.SB);
    r.a22 = ld_pair(vb + 3 * pl, g.ldS, li, a, pc, pc.SA, pc.SB);
    const float2 ga = ld_pair(g1, ldg, li, ap, pc, pc.PA, pc.PB);
    const float2 gb = ld_pair(g2, ldg, li, ap, pc, pc.PA, pc.PB);
    if constexpr (OM) {   // h = grad phi + omega0; OM = false: gphi already holds the sum
      const float2 oa = ld_pair(o1, g.ldP, li, ap, pc, pc.PA, pc.PB);
      const float2 obb = ld_pair(o2, g.ldP, li, ap, pc, pc.PA, pc.PB);
      r.h1 = make_float2(ga.x + oa.x, ga.y + oa.y);
      r.h2 = make_float2(gb.x + obb.x, gb.y + obb.y);
    } else {
      r.h1 = ga;
      r.h2 = gb;
    }
    return r;
  };
  auto rho = [&](int li, const Row &r, float2 v12m, float2 v22m, float2 &r1o, float2 &r2o) {
    const int gi = sd.y0 + li;
    const float2 w1 = div_pair(pc, gi, n2, r.a11, r.a12, v12m);
    const float2 w2 = div_pair(pc, gi, n2, r.a21, r.a22, v22m);
    const bool row_ok = li < ap;
    r1o = make_float2((row_ok && pc.PA) ? w1.x - r.h1.x : 0.f, (row_ok && pc.PB) ? w1.y - r.h1.y : 0.f);
    r2o = make_float2((row_ok && pc.PA) ? w2.x - r.h2.x : 0.f, (row_ok && pc.PB) ? w2.y - r.h2.y : 0.f);
  };
  Row c = ldrow(r0), n = ldrow(r0 + 1);
  const Row pr = ldrow(r0 - 1);
  float2 rc1, rc2;
  rho(r0, c, pr.a12, pr.a22, rc1, rc2);
  for (int li = r0; li < r1; ++li) {
    const Row m = ldrow(li + 2);
    float2 rn1, rn2;
    rho(li + 1, n, c.a12, c.a22, rn1, rn2);
    const float rr1 = __shfl_down_sync(0xffffffffu, rc1.x, 1);
    const float rr2 = __shfl_down_sync(0xffffffffu, rc2.x, 1);
    const bool xa = pc.jA + 1 < bp, xb = pc.jB + 1 < bp, yd = li + 1 < ap;
    const float ty = thy[sd.iy * g.A + li];
    // channel 1: (v11, v12); channel 2: (v21, v22)
    float2 a11 = c.a11, a12 = c.a12, a21 = c.a21, a22 = c.a22;
    ball_update_fast(ty * thA, t, xa ? rc1.y - rc1.x : 0.f, yd ? rn1.x - rc1.x : 0.f, a11.x, a12.x);
    ball_update_fast(ty * thB, t, xb ? rr1 - rc1.y : 0.f, yd ? rn1.y - rc1.y : 0.f, a11.y, a12.y);
    ball_update_fast(ty * thA, t, xa ? rc2.y - rc2.x : 0.f, yd ? rn2.x - rc2.x : 0.f, a21.x, a22.x);
    ball_update_fast(ty * thB, t, xb ? rr2 - rc2.y : 0.f, yd ? rn2.y - rc2.y : 0.f, a21.y, a22.y);
    const size_t o = (size_t)li * g.ldS + pc.jA;
    if (outA && outB) {
      *reinterpret_cast<float2 *>(ob + o) = a11;
      *reinterpret_cast<float2 *>(ob + pl + o) = a12;
      *reinterpret_cast<float2 *>(ob + 2 * pl + o) = a21;
      *reinterpret_cast<float2 *>(ob + 3 * pl + o) = a22;
    } else {
      if (outA) { ob[o] = a11.x; ob[pl + o] = a12.x; ob[2 * pl + o] = a21.x; ob[3 * pl + o] = a22.x; }
      if (outB) { ob[o + 1] = a11.y; ob[pl + o + 1] = a12.y; ob[2 * pl + o + 1] = a21.y; ob[3 * pl + o + 1] = a22.y; }
    }
    c = n;
    n = m;
    rc1 = rn1;
    rc2 = rn2;
  }
}

// ----------------------------------------------------------------------------- projection (b)
//
// phi = R_T Delta^dagger E_T q (Eq. locglobprojpart3/invLaplLowCapLong),
// refactored exactly: Delta = L_y (+) L_x is separable and C_{N1} diagonalises L_x, so
//   R_T Delta^dagger E_T = sum_j [R_Ty (L_y - s_j)^{-1} E_Ty] (x) [R_Tx c_j c_j^T E_Tx],
// s_j = sigma_{N1,j}^2 (j = 0: the Neumann pseudo-inverse L_y^dagger).  The restricted y-inverse
// is a tridiagonal solve on T's rows whose end diagonals carry the exact Schur complement of the
// rows outside T.  Only grad phi is ever formed (precision rule C-10): the x-derivative
// spectrally (c_j(x+1) - c_j(x) = -s_j sigma_j sin(pi j (x+1)/N)), the y-derivative by fp64
// differencing of the solved column.

// Tables: cf[x][j] = cos(pi j (2x+1) / (2n)) (forward), cn[j][x] (same, transposed),
// sn[j][x] = sin(pi j (x+1) / n) and snT[x][j] (transposed), evaluated in fp64 with exact
// integer argument reduction.
__global__ void k_dct_tables(int n, float *__restrict__ cf, float *__restrict__ cn,
                             float *__restrict__ sn, float *__restrict__ snT,
                             float *__restrict__ split6, int ld) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= n || j >= n) return;
  long long mc = ((long long)j * (2LL * x + 1)) % (4LL * n);
  long long ms = ((long long)j * (x + 1LL)) % (2LL * n);
  double c = cospi((double)mc / (2.0 * n));
  double s = sinpi((double)ms / (double)n);
  cf[(size_t)x * ld + j] = (float)c;
  cn[(size_t)j * ld + x] = (float)c;
  sn[(size_t)j * ld + x] = (float)s;
  snT[(size_t)x * ld + j] = (float)s;
  // 3xTF32 splits: [cf_hi, cf_lo, cn_hi, cn_lo, snT_hi, snT_lo], each n x ld
  const size_t pl = (size_t)n * ld;
  store_split(split6 + 0 * pl, split6 + 1 * pl, (size_t)x * ld + j, c);
  store_split(split6 + 2 * pl, split6 + 3 * pl, (size_t)j * ld + x, c);
  store_split(split6 + 4 * pl, split6 + 5 * pl, (size_t)x * ld + j, s);
}

// Thomas pivots of the Schur-corrected tridiagonal M_T(s_j) on rows [ty0, ty1] of an axis of
// length n2 (Neumann Laplacian L_y), one thread per (chain, j >= 1):
//   exterior chain of length L (far end Neumann): e_1 = -1 - s, e_k = -2 - s - 1/e_{k-1};
//   the Schur complement adds -1/e_L to T's end diagonal; rinv_k = 1 / (Thomas pivot k).
// Pivots r_k = 1/e_k of the Schur-corrected tridiagonal y-systems (one chain per distinct row
// range).  Tail compression: the interior recurrence e_k = -2 - s - 1/e_{k-1} reaches an exact
// fp64 fixed point after ~18 / sqrt(s) rows (every frequency but the lowest ~N/250), from which
// all interior pivots are bitwise equal; pcut[c][j] = first row of that constant run (nt - 1 if
// none), pinf = its value, plast = the last row's pivot (bottom Schur correction).  The solve reads
// the table only above pcut (the table below it is still written, and identical).
__global__ void k_pivots(const ProjTile *__restrict__ tiles, const int *__restrict__ first,
                         int nchains, int n2, int n1, double *__restrict__ rinv, int ldn, int AT,
                         int *__restrict__ pcut, double *__restrict__ pinf,
                         double *__restrict__ plast) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int c = blockIdx.y;
  if (j >= n1 || c >= nchains) return;
  const ProjTile tl = tiles[first[c]];
  double *out = rinv + (size_t)c * AT * ldn;
  int nt = tl.ty1 - tl.ty0 + 1;
  const size_t pj = (size_t)c * ldn + j;
  if (j == 0) {
    for (int k = 0; k < nt; ++k) out[(size_t)k * ldn] = 0.0;
    pcut[pj] = 0;
    pinf[pj] = 0.0;
    plast[pj] = 0.0;
    return;
  }
  double sg = 2.0 * sinpi((double)j / (2.0 * n1));
  double s = sg * sg;
  auto chain_corr = [&](int L) {
    double e = -1.0 - s;
    for (int k = 2; k <= L; ++k) e = -2.0 - s - 1.0 / e;
    return -1.0 / e;
  };
  double dtop = tl.ty0 > 0 ? (-2.0 - s + chain_corr(tl.ty0)) : (-1.0 - s);
  double dbot = tl.ty1 < n2 - 1 ? (-2.0 - s + chain_corr(n2 - 1 - tl.ty1)) : (-1.0 - s);
  double e = dtop;
  out[j] = 1.0 / e;
  int cut = nt - 1;
  for (int k = 1; k < nt; ++k) {
    double dk = (k == nt - 1) ? dbot : (-2.0 - s);
    const double prev = e;
    e = dk - 1.0 / e;
    out[(size_t)k * ldn + j] = 1.0 / e;
    if (cut == nt - 1 && k < nt - 1 && e == prev) cut = k - 1;   // r_{k-1} = r_k = ... = r_{nt-2}
  }
  pcut[pj] = cut;
  pinf[pj] = out[(size_t)min(cut, nt - 1) * ldn + j];
  plast[pj] = out[(size_t)(nt - 1) * ldn + j];
}


// Segmented form of the per-frequency y-solve (default).  Both Thomas sweeps are first-order
// linear recurrences in the precomputed pivots r_k = 1/e_k:
//   forward   z_k = b_k - r_{k-1} z_{k-1}         (z_0 = b_0)
//   backward  u_k = r_k (z_k - u_{k+1})           (u_nt = 0)
// so the rows of T are cut into nseg segments per frequency (one warp per segment, 32 frequencies
// per CTA): every segment runs its recurrence from a zero carry and records (end value, product of
// coefficients); one fp64 scan over the segments in shared memory gives every segment its exact
// carry; the segment then re-runs with it.  Same operator as one serial sweep, different rounding
// order.  z is kept in an fp32 scratch: its rounding moves grad phi by < 1e-7 of max|grad phi|
// (flat in N).  j = 0 (singular Neumann L_y^dagger) uses the same skeleton for
// its prefix sums: D+_y u = prefix(b) - mu (y + 1), mu = sum(b) / n2.
constexpr int SJB = 32, SSEG_MAX = 16, SU = 8;
// solve3 (tall tiles: config-4 strips, the global projections, config 5) takes up to 32 segments
// per column (1024 threads): its fp64 recurrences are latency-bound chains, and with one CTA per SM
// (the staged column block fills shared memory) shorter chains and twice the warps hide them
constexpr int S3SEG_MAX = 32;
// Pivots r_kk of one batch of SU rows, kk = kb + D u (D = +1 ascending, -1 descending), handed to
// f as a functor R(u).  pcb is the CTA's largest pcut (warp-uniform: a CTA's warps share its 32
// columns): the table is exact at every row (k_pivots writes all of them) and bitwise the tail
// value from pcut on, so reading it above pcb and the tail values from pcb on gives every column
// its own pivots -- with one uniform branch per batch instead of a per-row select, no loads at all
// in the (common) all-tail batch, and a pointer walk instead of per-row 64-bit indexing.
template <int D, class F>
__device__ __forceinline__ void with_piv(int kb, int pcb, int nt, const double *__restrict__ ri,
                                         size_t st, double rinf, double rlast, F &&f) {
  const int lo = D > 0 ? kb : kb - (SU - 1), hi = D > 0 ? kb + SU - 1 : kb;
  if (lo >= pcb && hi < nt - 1) {
    f([&](int) { return rinf; });
    return;
  }
  double rv[SU];
  if (hi < pcb) {
    const double *p = ri + (size_t)kb * st;
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      rv[u] = __ldg(p);
      if (D > 0) p += st; else p -= st;
    }
  } else {
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int kk = kb + D * u;
      rv[u] = kk < pcb ? __ldg(ri + (size_t)kk * st) : (kk == nt - 1 ? rlast : rinf);
    }
  }
  f([&](int u) { return rv[u]; });
}

// store v (fp32), or its tf32 head and fp32 tail at p + dl when the split planes are requested
__device__ __forceinline__ void put_split(float *p, ptrdiff_t dl, bool split, double v) {
  if (split) {
    const float h = tf32_rna((float)v);
    p[0] = h;
    p[dl] = (float)(v - (double)h);
  } else {
    p[0] = (float)v;
  }
}

// SMEM = true: the CTA's column block of qhat (JB columns) is staged in shared memory by the
// first pass and overwritten in place by z (fp32), so qhat is read from HBM once and z never
// leaves the SM (AT x 4 JB B of dynamic shared memory; JB = 16: two CTAs per SM).  SMEM = false:
// z in a global scratch (JB = 32).
template <bool SMEM, int JB>
__global__ void __launch_bounds__(JB *S3SEG_MAX, 1024 / (JB * S3SEG_MAX))
k_proj_solve3(const ProjTile *__restrict__ tiles, int n2, int n1, const float *__restrict__ qhat,
              int AT, int ldn, const double *__restrict__ rinv, float *__restrict__ zs,
              float *__restrict__ phx, float *__restrict__ phy, float *__restrict__ phx_lo,
              float *__restrict__ phy_lo, int AP, const int *__restrict__ pcut,
              const double *__restrict__ pinf, const double *__restrict__ plast) {
  __shared__ double sh_a[S3SEG_MAX][JB], sh_c[S3SEG_MAX][JB];
  __shared__ double sh_tot[JB];
  extern __shared__ __align__(16) float sbuf[];   // SMEM: [AT][JB]
  const int tx = threadIdx.x, sg = threadIdx.y, nseg = blockDim.y;
  const int j = blockIdx.x * JB + tx;
  const int tix = blockIdx.y;
  const bool valid = j < n1;
  const ProjTile tl = tiles[tix];
  const int nt = tl.ty1 - tl.ty0 + 1, nout = tl.py1 - tl.ty0 + 1, po = tl.po;
  const int LS = (nt + nseg - 1) / nseg;
  const int k0 = min(nt, sg * LS), k1 = min(nt, k0 + LS);
  const int jj = valid ? j : 0;
  const size_t st = (size_t)ldn;   // row stride of every global plane
  const float *__restrict__ b = qhat + (size_t)tix * AT * st + jj;
  const double *__restrict__ ri = rinv + (size_t)tl.chain * AT * st + jj;
  // pivot r_k: the table above the constant tail (see k_pivots), the tail value below it
  const int pc = pcut[(size_t)tl.chain * st + jj];
  const int pcb = __reduce_max_sync(0xffffffffu, pc);
  const double rinf = pinf[(size_t)tl.chain * st + jj], rlast = plast[(size_t)tl.chain * st + jj];
  auto piv = [&](int kk) -> double {
    return kk < pcb ? __ldg(ri + (size_t)kk * st) : (kk == nt - 1 ? rlast : rinf);
  };
  // z (and, in SMEM mode, the staged b) live at zb with row stride zst
  float *zb = SMEM ? sbuf + tx : zs + (size_t)tix * AT * st + jj;
  const size_t zst = SMEM ? (size_t)JB : st;
  const float *bb = SMEM ? zb : b;   // second read of b
  const double s2 = (j == 0 ? 1.0 : 2.0) / (double)n1;   // s_j^2 (Eq. form:DCTmat normalisation)

  if constexpr (SMEM) {
    // stage the CTA's [nt x 32] column block of qhat in shared memory with asynchronous 16-byte
    // copies issued by every thread (all rows in flight at once), then every pass reads it there
    const float *blk = qhat + (size_t)tix * AT * st + (size_t)blockIdx.x * JB;
    const int nthr = JB * nseg, lt = sg * JB + tx;
    for (int e = lt; e < nt * (JB / 4); e += nthr) {
      const int k = e / (JB / 4), c = e % (JB / 4);
      float *dst = sbuf + k * JB + 4 * c;
      if (blockIdx.x * JB + 4 * c < ldn) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                     "l"(blk + (size_t)k * st + 4 * c) : "memory");
      } else {
        dst[0] = dst[1] = dst[2] = dst[3] = 0.f;
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  const float *b1 = SMEM ? zb : b;   // first read of b
  const size_t b1st = SMEM ? zst : st;

  // ---- forward, local pass from a zero carry: end value a and coefficient product g
  double a = 0.0, g = 1.0;
  if (valid) {
    if (j == 0) {
      const float *bp = b1 + (size_t)k0 * b1st;
      for (int k = k0; k < k1; ++k, bp += b1st) a += (double)*bp;
    } else {
      int k = k0;
      if (k == 0 && k < k1) {   // z_0 = b_0 (no coupling above row 0 of T)
        a = (double)b1[0];
        g = 0.0;
        k = 1;
      }
      const float *bp = b1 + (size_t)k * b1st;
      for (; k + SU <= k1; k += SU, bp += SU * b1st) {
        float bv[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) bv[u] = bp[u * b1st];   // the whole batch of loads first
        with_piv<1>(k - 1, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
          for (int u = 0; u < SU; ++u) {
            a = fma(-R(u), a, (double)bv[u]);
            g *= -R(u);
          }
        });
      }
      for (; k < k1; ++k, bp += b1st) {
        const double r = piv(k - 1);
        a = fma(-r, a, (double)*bp);
        g *= -r;
      }
    }
  }
  sh_a[sg][tx] = a;
  sh_c[sg][tx] = g;
  __syncthreads();
  if (sg == 0) {   // carry into segment s: Z_{s-1};  Z_s = a_s + g_s Z_{s-1}
    double Z = 0.0;
    for (int s = 0; s < nseg; ++s) {
      const double as = sh_a[s][tx], gs = sh_c[s][tx];
      sh_c[s][tx] = Z;
      Z = fma(gs, Z, as);
    }
    sh_tot[tx] = Z;
  }
  __syncthreads();
  const double fcarry = sh_c[sg][tx];

  // ---- forward, final pass with the exact carry: z (fp32)
  if (valid && j > 0 && k0 < k1) {
    double zc = fcarry;
    int k = k0;
    if (k == 0) {
      zc = (double)bb[0];
      zb[0] = (float)zc;
      k = 1;
    }
    const float *bp = bb + (size_t)k * zst;
    float *zp = zb + (size_t)k * zst;
    for (; k + SU <= k1; k += SU, bp += SU * zst, zp += SU * zst) {
      float bv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) bv[u] = bp[u * zst];
      with_piv<1>(k - 1, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          zc = fma(-R(u), zc, (double)bv[u]);
          zp[u * zst] = (float)zc;
        }
      });
    }
    for (; k < k1; ++k, bp += zst, zp += zst) {
      zc = fma(-piv(k - 1), zc, (double)*bp);
      *zp = (float)zc;
    }
  }
  // ---- backward, local pass from a zero carry (u_{k1} = 0)
  a = 0.0;
  g = 1.0;
  if (valid && j > 0 && k0 < k1) {
    int k = k1 - 1;
    const float *zp = zb + (size_t)k * zst;
    for (; k - SU + 1 >= k0; k -= SU, zp -= SU * zst) {
      float zv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) zv[u] = zp[-(ptrdiff_t)(u * zst)];
      with_piv<-1>(k, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          a = R(u) * ((double)zv[u] - a);
          g *= -R(u);
        }
      });
    }
    for (; k >= k0; --k, zp -= zst) {
      const double r = piv(k);
      a = r * ((double)*zp - a);
      g *= -r;
    }
  }
  __syncthreads();   // every thread has read its forward carry
  sh_a[sg][tx] = a;
  sh_c[sg][tx] = g;
  __syncthreads();
  if (sg == 0) {   // carry into segment s from below: U_{s+1};  U_s = a_s + g_s U_{s+1}
    double U = 0.0;
    for (int s = nseg - 1; s >= 0; --s) {
      const double as = sh_a[s][tx], gs = sh_c[s][tx];
      sh_c[s][tx] = U;
      U = fma(gs, U, as);
    }
  }
  __syncthreads();
  if (!valid || k0 >= k1) return;
  const size_t obase = (size_t)tix * AP * st + jj - (size_t)po * st;
  float *__restrict__ ox = phx + obase;
  float *__restrict__ oy = phy + obase;
  float *__restrict__ oxl = phx_lo ? phx_lo + obase : nullptr;
  float *__restrict__ oyl = phy_lo ? phy_lo + obase : nullptr;
  if (j == 0) {   // L_y^dagger: D+_y u = prefix(b) - mu (y + 1), mu = sum(b) / n2
    const double mu = sh_tot[tx] / (double)n2;
    double pre = fcarry;
    for (int k = k0; k < min(k1, nout); ++k) {
      pre += (double)bb[(size_t)k * zst];
      const int y = tl.ty0 + k;
      const double w = (y == n2 - 1) ? 0.0 : pre - mu * (double)(y + 1);
      if (k >= po) {
        store_split(ox, oxl, (size_t)k * st, 0.0);
        store_split(oy, oyl, (size_t)k * st, s2 * w);
      }
    }
    return;
  }
  const double sg_j = 2.0 * sinpi((double)j / (2.0 * n1));
  const double cx = -s2 * sg_j;
  const bool split = oxl != nullptr;
  const ptrdiff_t dlx = split ? oxl - ox : 0, dly = split ? oyl - oy : 0;
  // ---- backward, final pass with the exact carry; outputs on rows [po, nout)
  double un = sh_c[sg][tx];
  int k = k1 - 1;
  const float *zp = zb + (size_t)k * zst;
  auto emit = [&](int kk, double uk) {
    if (kk >= po && kk < nout) {
      store_split(ox, oxl, (size_t)kk * st, cx * uk);
      // D+_y u = u_{k+1} - u_k; 0 on the global last row (T = S+ in y there)
      store_split(oy, oyl, (size_t)kk * st, (kk == nt - 1) ? 0.0 : s2 * (un - uk));
    }
    un = uk;
  };
  for (; k - SU + 1 >= k0; k -= SU, zp -= SU * zst) {
    float zv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) zv[u] = zp[-(ptrdiff_t)(u * zst)];
    const bool inner = k - SU + 1 >= po && k < nout && k < nt - 1;   // all rows are output rows
    with_piv<-1>(k, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
      if (inner) {
        float *px = ox + (size_t)k * st, *py = oy + (size_t)k * st;
#pragma unroll
        for (int u = 0; u < SU; ++u, px -= st, py -= st) {
          const double uk = R(u) * ((double)zv[u] - un);
          put_split(px, dlx, split, cx * uk);
          put_split(py, dly, split, s2 * (un - uk));
          un = uk;
        }
      } else {
#pragma unroll
        for (int u = 0; u < SU; ++u) emit(k - u, R(u) * ((double)zv[u] - un));
      }
    });
  }
  for (; k >= k0; --k, zp -= zst) emit(k, piv(k) * ((double)*zp - un));
}

// ---------------------------------------------------------------------------------------------
// Global y-solve in fixed segments (the global projection r^n = f - P multidiv p^n):
// the rows of the whole-grid tile are cut into segments at the layout's core cuts (one "virtual
// slab" per layout row, each split into equal sub-segments of ~256 rows) -- the same segments at
// every GPU count.  A rank solves only the segments of its own slabs:
//   A  forward pass of each owned segment from a zero carry -> (a_s, g_s) per frequency;
//      all-gather of the (a, g) of every segment (2 doubles per segment and frequency);
//   B  every rank scans ALL segments in the same order (identical carries on every rank), runs
//      the owned segments' forward pass with the exact carry (z, fp32 scratch) and their backward
//      pass from a zero carry -> (a'_s, g'_s); all-gather;
//   C  reverse scan, backward pass with the exact carry, outputs grad phi's spectral planes on the
//      owned rows (the rows of the valid band beyond them arrive from the slab neighbours).
// Only the (a, g) pairs travel (not the partial x-DCT of every row), no rank solves the whole
// grid, and tau is bitwise the same for every GPU count.  Same recurrences and fma orders as
// k_proj_solve3; j = 0 (the singular Neumann column) is the prefix sum D+_y u = prefix(b) - mu (y+1).
// agg layout: [segment][2][ldn] doubles.  One thread per (frequency, owned segment).
// The pivots come through with_piv with the warp's largest pcut (the frequencies of a warp are 32
// consecutive j), the rows in batches of SU loads -- the per-row latency chain otherwise bounds
// these one-thread-per-(frequency, segment) loops.
__device__ __forceinline__ double gs_piv(const double *ri, int k, size_t st, int pc, int nt,
                                         double rinf, double rlast) {
  return k < pc ? __ldg(ri + (size_t)k * st) : (k == nt - 1 ? rlast : rinf);
}
__global__ void __launch_bounds__(128)
k_gsolve_a(const int *__restrict__ seglo, int s0, int s1, int n1, const float *__restrict__ qhat,
           int ldn, const double *__restrict__ rinv, const int *__restrict__ pcut,
           const double *__restrict__ pinf, const double *__restrict__ plast, int nt,
           double *__restrict__ agg) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, s = s0 + blockIdx.y;
  const bool ok = j < n1 && s < s1;
  const int pcb = __reduce_max_sync(0xffffffffu, ok ? pcut[j] : 0);
  if (!ok) return;
  const size_t st = ldn;
  const int k0 = seglo[s], k1 = seglo[s + 1];
  const float *b = qhat + j;
  double a = 0.0, g = 1.0;
  if (j == 0) {
    for (int k = k0; k < k1; ++k) a += (double)b[(size_t)k * st];
  } else {
    const double *ri = rinv + j;
    const double rinf = pinf[j], rlast = plast[j];
    int k = k0;
    if (k == 0) {   // z_0 = b_0 (no coupling above row 0)
      a = (double)b[0];
      g = 0.0;
      k = 1;
    }
    const float *bp = b + (size_t)k * st;
    for (; k + SU <= k1; k += SU, bp += SU * st) {
      float bv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) bv[u] = __ldg(bp + u * st);
      with_piv<1>(k - 1, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          a = fma(-R(u), a, (double)bv[u]);
          g *= -R(u);
        }
      });
    }
    for (; k < k1; ++k, bp += st) {
      const double r = gs_piv(ri, k - 1, st, pcb, nt, rinf, rlast);
      a = fma(-r, a, (double)*bp);
      g *= -r;
    }
  }
  agg[((size_t)s * 2 + 0) * st + j] = a;
  agg[((size_t)s * 2 + 1) * st + j] = g;
}
__global__ void __launch_bounds__(128)
k_gsolve_b(const int *__restrict__ seglo, int nseg, int s0, int s1, int n1,
           const float *__restrict__ qhat, int ldn, const double *__restrict__ rinv,
           const int *__restrict__ pcut, const double *__restrict__ pinf,
           const double *__restrict__ plast, int nt, const double *__restrict__ agg,
           float *__restrict__ zs, double *__restrict__ aggb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, s = s0 + blockIdx.y;
  const bool ok = j < n1 && s < s1;
  const int pcb = __reduce_max_sync(0xffffffffu, ok ? pcut[j] : 0);
  if (!ok || j == 0) return;   // j = 0 needs no z / backward pass
  const size_t st = ldn;
  const int k0 = seglo[s], k1 = seglo[s + 1];
  double Z = 0.0;   // forward carry into segment s: Z_t = a_t + g_t Z_{t-1}, all ranks alike
  for (int t = 0; t < s; ++t)
    Z = fma(agg[((size_t)t * 2 + 1) * st + j], Z, agg[((size_t)t * 2 + 0) * st + j]);
  const double *ri = rinv + j;
  const double rinf = pinf[j], rlast = plast[j];
  const float *b = qhat + j;
  float *z = zs + j;
  double zc = Z;
  int k = k0;
  if (k == 0) {
    zc = (double)b[0];
    z[0] = (float)zc;
    k = 1;
  }
  {
    const float *bp = b + (size_t)k * st;
    float *zp = z + (size_t)k * st;
    for (; k + SU <= k1; k += SU, bp += SU * st, zp += SU * st) {
      float bv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) bv[u] = __ldg(bp + u * st);
      with_piv<1>(k - 1, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          zc = fma(-R(u), zc, (double)bv[u]);
          zp[u * st] = (float)zc;
        }
      });
    }
    for (; k < k1; ++k, bp += st, zp += st) {
      zc = fma(-gs_piv(ri, k - 1, st, pcb, nt, rinf, rlast), zc, (double)*bp);
      *zp = (float)zc;
    }
  }
  double a = 0.0, g = 1.0;   // backward, zero carry: u_k = r_k (z_k - u_{k+1})
  k = k1 - 1;
  {
    const float *zp = z + (size_t)k * st;
    for (; k - SU + 1 >= k0; k -= SU, zp -= SU * st) {
      float zv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) zv[u] = zp[-(ptrdiff_t)(u * st)];
      with_piv<-1>(k, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          a = R(u) * ((double)zv[u] - a);
          g *= -R(u);
        }
      });
    }
    for (; k >= k0; --k, zp -= st) {
      const double r = gs_piv(ri, k, st, pcb, nt, rinf, rlast);
      a = r * ((double)*zp - a);
      g *= -r;
    }
  }
  aggb[((size_t)s * 2 + 0) * st + j] = a;
  aggb[((size_t)s * 2 + 1) * st + j] = g;
}
__global__ void __launch_bounds__(128)
k_gsolve_c(const int *__restrict__ seglo, int nseg, int s0, int s1, int n1, int n2,
           const float *__restrict__ qhat, int ldn, const double *__restrict__ rinv,
           const int *__restrict__ pcut, const double *__restrict__ pinf,
           const double *__restrict__ plast, int nt, const double *__restrict__ agg,
           const double *__restrict__ aggb, const float *__restrict__ zs, float *__restrict__ phx,
           float *__restrict__ phy, int po) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, s = s0 + blockIdx.y;
  const bool ok = j < n1 && s < s1;
  const int pcb = __reduce_max_sync(0xffffffffu, ok ? pcut[j] : 0);
  if (!ok) return;
  const size_t st = ldn;
  const int k0 = seglo[s], k1 = seglo[s + 1];
  float *ox = phx + j - (size_t)po * st, *oy = phy + j - (size_t)po * st;
  const double s2 = (j == 0 ? 1.0 : 2.0) / (double)n1;   // s_j^2 (Eq. form:DCTmat normalisation)
  if (j == 0) {   // L_y^dagger: D+_y u = prefix(b) - mu (y + 1), mu = sum(b) / n2
    double pre = 0.0, tot = 0.0;
    for (int t = 0; t < nseg; ++t) {
      const double at = agg[((size_t)t * 2 + 0) * st];
      if (t < s) pre += at;
      tot += at;
    }
    const double mu = tot / (double)n2;
    for (int k = k0; k < k1; ++k) {
      pre += (double)qhat[(size_t)k * st];
      const double w = (k == n2 - 1) ? 0.0 : pre - mu * (double)(k + 1);
      ox[(size_t)k * st] = 0.f;
      oy[(size_t)k * st] = (float)(s2 * w);
    }
    return;
  }
  double U = 0.0;   // backward carry into segment s from below: U_t = a'_t + g'_t U_{t+1}
  for (int t = nseg - 1; t > s; --t)
    U = fma(aggb[((size_t)t * 2 + 1) * st + j], U, aggb[((size_t)t * 2 + 0) * st + j]);
  const double *ri = rinv + j;
  const double rinf = pinf[j], rlast = plast[j];
  const double cx = -s2 * (2.0 * sinpi((double)j / (2.0 * n1)));
  double un = U;
  int k = k1 - 1;
  const float *zp = zs + (size_t)k * st + j;
  auto emit = [&](int kk, double uk) {
    ox[(size_t)kk * st] = (float)(cx * uk);
    // D+_y u = u_{k+1} - u_k; 0 on the global last row
    oy[(size_t)kk * st] = (kk == nt - 1) ? 0.f : (float)(s2 * (un - uk));
    un = uk;
  };
  for (; k - SU + 1 >= k0; k -= SU, zp -= SU * st) {
    float zv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) zv[u] = zp[-(ptrdiff_t)(u * st)];
    with_piv<-1>(k, pcb, nt, ri, st, rinf, rlast, [&](auto R) {
#pragma unroll
      for (int u = 0; u < SU; ++u) emit(k - u, R(u) * ((double)zv[u] - un));
    });
  }
  for (; k >= k0; --k, zp -= st) emit(k, gs_piv(ri, k, st, pcb, nt, rinf, rlast) * ((double)*zp - un));
}

// Products of the recurrence coefficients over each solve segment (data-independent, computed
// once per plan): forward GF_s = prod_{k in seg} (-r_{k-1}) (r_{-1} = 0), backward GB_s =
// prod_{k in seg} (-r_k); segments of LS = ceil(nt / nseg) rows as in k_proj_solve4.
// segprod layout: [chain][2][nseg][ldn].
__global__ void k_segprod(const ProjTile *__restrict__ tiles, const int *__restrict__ first,
                          int nchains, const double *__restrict__ rinv, int ldn, int AT, int n1,
                          int nseg, double *__restrict__ segprod) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (j >= n1 || c >= nchains) return;
  const ProjTile tl = tiles[first[c]];
  const int nt = tl.ty1 - tl.ty0 + 1, LS = (nt + nseg - 1) / nseg;
  const double *r = rinv + (size_t)c * AT * ldn + j;
  double *gf = segprod + (size_t)c * 2 * nseg * ldn + j, *gb = gf + (size_t)nseg * ldn;
  for (int sg = 0; sg < nseg; ++sg) {
    const int k0 = min(nt, sg * LS), k1 = min(nt, k0 + LS);
    double pf = 1.0, pb = 1.0;
    for (int k = k0; k < k1; ++k) {
      pf *= k > 0 ? -r[(size_t)(k - 1) * ldn] : 0.0;
      pb *= -r[(size_t)k * ldn];
    }
    gf[(size_t)sg * ldn] = pf;
    gb[(size_t)sg * ldn] = pb;
  }
}

// Segmented y-solve, shared-memory form (default when a tile's column block fits): the same four
// passes as k_proj_solve3<true> with 32-bit shared indices and precomputed segment products.  The
// CTA's [nt x 32] blocks of Q-hat (fp32) and of the pivots (fp64) are staged in shared memory with
// cp.async, so the pivots are read from L2 once instead of four times and every pass runs on
// shared-memory data.  Outputs are plain fp32.
template <int J>
__global__ void __launch_bounds__(J *SSEG_MAX)
k_proj_solve4(const ProjTile *__restrict__ tiles, int n2, int n1, const float *__restrict__ qhat,
              int AT, int ldn, const double *__restrict__ rinv, const double *__restrict__ segprod,
              float *__restrict__ phx, float *__restrict__ phy, int AP,
              const SolveMaps *__restrict__ maps, int srows, const int *__restrict__ order,
              int per_chain) {
  __shared__ double sh_a[SSEG_MAX][J], sh_c[SSEG_MAX][J];
  __shared__ double sh_tot[J];
  __shared__ uint64_t sbar;
  extern __shared__ __align__(128) double sr4[];   // [srows][J] pivots, then [srows][J] floats
  float *sb4 = reinterpret_cast<float *>(sr4 + (size_t)srows * J);   // Q-hat, overwritten by z
  const int tx = threadIdx.x, sg = threadIdx.y, nseg = blockDim.y;
  // grid (frequency block, tile within its chain, chain): adjacent CTAs stage adjacent 128-byte
  // row segments (DRAM locality: -4 % against tile-fastest), and the tiles sharing a pivot block
  // (one layout row) still run within one wave, so their pivot reads hit L2
  const int jb = blockIdx.x;
  const int tix = order[blockIdx.z * per_chain + blockIdx.y];
  if (tix < 0) return;
  const int j = jb * J + tx;
  const bool valid = j < n1;
  const ProjTile tl = tiles[tix];
  const int nt = tl.ty1 - tl.ty0 + 1, nout = tl.py1 - tl.ty0 + 1, po = tl.po;
  const int LS = (nt + nseg - 1) / nseg;
  const int k0 = min(nt, sg * LS), k1 = min(nt, k0 + LS);
  const int jj = valid ? j : 0;
  // segment products of the two carry scans: loaded now so their latency overlaps the staging
  const double *__restrict__ gp = segprod + (size_t)tl.chain * 2 * nseg * ldn + jj;
  const double gpf = (valid && j > 0) ? __ldg(gp + (size_t)sg * ldn) : 1.0;
  const double gpb = (valid && j > 0) ? __ldg(gp + (size_t)(nseg + sg) * ldn) : 1.0;
  {   // stage both column blocks with TMA (nbox boxes of {J columns, box_rows rows})
    const int lt = sg * J + tx;
    if (lt == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&sbar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sbar);
    if (lt == 0) {
      const int br = maps->box_rows, nb = maps->nbox;
      const uint32_t bytes = (uint32_t)(nb * br * J * (sizeof(float) + sizeof(double)));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      const int col = jb * J;
      // Q-hat: row-major (column jb J, row tix AT) or column-block-major (block jb, same rows)
      const int qcol = maps->q_blk_rows > 0 ? 0 : col;
      const int qrow0 = (maps->q_blk_rows > 0 ? jb * maps->q_blk_rows : 0) + tix * AT;
      for (int bi = 0; bi < nb; ++bi) {
        const uint32_t dq = (uint32_t)__cvta_generic_to_shared(sb4 + (size_t)bi * br * J);
        const uint32_t dr = (uint32_t)__cvta_generic_to_shared(sr4 + (size_t)bi * br * J);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dq),
            "l"(reinterpret_cast<uint64_t>(&maps->q)), "r"(qcol), "r"(qrow0 + bi * br), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dr),
            "l"(reinterpret_cast<uint64_t>(&maps->r)), "r"(col), "r"(tl.chain * AT + bi * br), "r"(bar)
            : "memory");
      }
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(bar) : "memory");
  }
  const double *ri = sr4 + tx;   // pivot of row k at ri[k * J]
  float *sbt = sb4 + tx;                                                     // row k at sbt[k*J]
  const double s2 = (j == 0 ? 1.0 : 2.0) / (double)n1;

  // ---- forward, local pass (zero carry): end value
  double a = 0.0;
  if (valid) {
    if (j == 0) {
      for (int k = k0; k < k1; ++k) a += (double)sbt[k * J];
    } else {
      int k = k0;
      if (k == 0 && k < k1) {
        a = (double)sbt[0];
        k = 1;
      }
      for (; k + SU <= k1; k += SU) {
        float bv[SU];
        double rv[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          bv[u] = sbt[(k + u) * J];
          rv[u] = ri[(k + u - 1) * J];
        }
#pragma unroll
        for (int u = 0; u < SU; ++u) a = fma(-rv[u], a, (double)bv[u]);
      }
      for (; k < k1; ++k) a = fma(-ri[(k - 1) * J], a, (double)sbt[k * J]);
    }
  }
  sh_a[sg][tx] = a;
  sh_c[sg][tx] = gpf;
  __syncthreads();
  if (sg == 0) {
    double Z = 0.0;
    for (int s = 0; s < nseg; ++s) {
      const double as = sh_a[s][tx], gs = sh_c[s][tx];
      sh_c[s][tx] = Z;
      Z = fma(gs, Z, as);
    }
    sh_tot[tx] = Z;
  }
  __syncthreads();
  const double fcarry = sh_c[sg][tx];

  // ---- forward, final pass: z overwrites b in shared memory
  if (valid && j > 0 && k0 < k1) {
    double zc = fcarry;
    int k = k0;
    if (k == 0) {
      zc = (double)sbt[0];
      k = 1;
    }
    for (; k + SU <= k1; k += SU) {
      float bv[SU];
      double rv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        bv[u] = sbt[(k + u) * J];
        rv[u] = ri[(k + u - 1) * J];
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        zc = fma(-rv[u], zc, (double)bv[u]);
        sbt[(k + u) * J] = (float)zc;
      }
    }
    for (; k < k1; ++k) {
      zc = fma(-ri[(k - 1) * J], zc, (double)sbt[k * J]);
      sbt[k * J] = (float)zc;
    }
  }
  // ---- backward, local pass (u_{k1} = 0)
  a = 0.0;
  if (valid && j > 0 && k0 < k1) {
    int k = k1 - 1;
    for (; k - SU + 1 >= k0; k -= SU) {
      float zv[SU];
      double rv[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        zv[u] = sbt[(k - u) * J];
        rv[u] = ri[(k - u) * J];
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) a = rv[u] * ((double)zv[u] - a);
    }
    for (; k >= k0; --k) a = ri[k * J] * ((double)sbt[k * J] - a);
  }
  __syncthreads();
  sh_a[sg][tx] = a;
  sh_c[sg][tx] = gpb;
  __syncthreads();
  if (sg == 0) {
    double U = 0.0;
    for (int s = nseg - 1; s >= 0; --s) {
      const double as = sh_a[s][tx], gs = sh_c[s][tx];
      sh_c[s][tx] = U;
      U = fma(gs, U, as);
    }
  }
  __syncthreads();
  if (!valid || k0 >= k1) return;
  float *__restrict__ ox = phx + (size_t)tix * AP * ldn + jj - (size_t)po * ldn;
  float *__restrict__ oy = phy + (size_t)tix * AP * ldn + jj - (size_t)po * ldn;
  if (j == 0) {
    const double mu = sh_tot[tx] / (double)n2;
    double pre = fcarry;
    for (int k = k0; k < min(k1, nout); ++k) {
      pre += (double)sbt[k * J];
      const int y = tl.ty0 + k;
      const double w = (y == n2 - 1) ? 0.0 : pre - mu * (double)(y + 1);
      if (k >= po) {
        ox[(size_t)k * ldn] = 0.f;
        oy[(size_t)k * ldn] = (float)(s2 * w);
      }
    }
    return;
  }
  const double sg_j = 2.0 * sinpi((double)j / (2.0 * n1));
  const double cx = -s2 * sg_j;
  double un = sh_c[sg][tx];
  const int klo = max(k0, po), khi = min(k1, nout);   // output rows of this segment
  int k = k1 - 1;
  // rows above nout (T rows below S+) only carry the recurrence
  for (; k >= khi && k >= k0; --k) un = ri[k * J] * ((double)sbt[k * J] - un);
  for (; k - SU + 1 >= klo; k -= SU) {
    float zv[SU];
    double rv[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      zv[u] = sbt[(k - u) * J];
      rv[u] = ri[(k - u) * J];
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const double uk = rv[u] * ((double)zv[u] - un);
      ox[(size_t)(k - u) * ldn] = (float)(cx * uk);
      // D+_y u = u_{k+1} - u_k; 0 on the global last row (T = S+ in y there)
      oy[(size_t)(k - u) * ldn] = (k - u == nt - 1) ? 0.f : (float)(s2 * (un - uk));
      un = uk;
    }
  }
  for (; k >= klo; --k) {
    const double uk = ri[k * J] * ((double)sbt[k * J] - un);
    ox[(size_t)k * ldn] = (float)(cx * uk);
    oy[(size_t)k * ldn] = (k == nt - 1) ? 0.f : (float)(s2 * (un - uk));
    un = uk;
  }
}

// Batched fp32 SIMT GEMM, C = A * B (row-major), 128 x 128 x 8 CTA tile, 256 threads, 8 x 8
// register micro-tile, double-buffered shared memory.  blockIdx.z selects the batch entry.
constexpr int GBM = 128, GBN = 128, GBK = 8;
__global__ void __launch_bounds__(256) k_gemm(const GemmDesc *__restrict__ descs) {
  const GemmDesc d = descs[blockIdx.z];
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  if (m0 >= d.M || n0 >= d.N) return;
  __shared__ __align__(16) float As[2][GBK][GBM];
  __shared__ __align__(16) float Bs[2][GBK][GBN];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float ra[4], rb[4];
  auto load_global = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int idx = tid + e * 256;
      int r = idx / GBK, kk = idx % GBK;
      int gm = m0 + r, gk = k0 + kk;
      ra[e] = (gm < d.M && gk < d.K) ? __ldg(d.A + (size_t)gm * d.lda + gk) : 0.f;
      int kb = idx / GBN, cb = idx % GBN;
      int gkb = k0 + kb, gn = n0 + cb;
      rb[e] = (gkb < d.K && gn < d.N) ? __ldg(d.B + (size_t)gkb * d.ldb + gn) : 0.f;
    }
  };
  auto store_shared = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int idx = tid + e * 256;
      As[buf][idx % GBK][idx / GBK] = ra[e];
      Bs[buf][idx / GBN][idx % GBN] = rb[e];
    }
  };
  int nk = (d.K + GBK - 1) / GBK;
  load_global(0);
  store_shared(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    int buf = kt & 1;
    if (kt + 1 < nk) load_global((kt + 1) * GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
      float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4 + 64]);
      float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4 + 64]);
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store_shared(buf ^ 1);
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (gm >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (gn < d.N) d.C[(size_t)gm * d.ldc + gn] = acc[i][j];
    }
  }
}

// ----------------------------------------------------------------------------- launchers

thread_local int g_extra_launches = 0;

cudaError_t smem_optin(const void *func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> done;   // (device, kernel) -> bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t &have = done[std::make_pair(dev, func)];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

int sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  cache[dev] = n;
  return n;
}

static inline dim3 grid2(int nx, int ny, int bx, int by, int z = 1) {
  return dim3((nx + bx - 1) / bx, (ny + by - 1) / by, z);
}

cudaError_t launch_tau0(const float *d0, int n2, int n1, float *tau, int ldt, cudaStream_t s) {
  k_tau0<<<grid2(n1 + 1, n2 + 1, 32, 8), dim3(32, 8), 0, s>>>(d0, n2, n1, tau, ldt);
  return cudaGetLastError();
}
cudaError_t launch_g_row0(const float *tau2, int ldt, int n1, double *g_row0, cudaStream_t s) {
  (void)ldt;
  k_g_row0<<<1, 1024, 0, s>>>(tau2, n1, g_row0);
  return cudaGetLastError();
}
cudaError_t launch_irv2_f(const float *tau1, int ldt, const double *g_row0, const float *d0,
                          int n2, int n1, float alpha, float *f, int ldf, double *csum,
                          cudaStream_t s) {
  if (!csum) {   // one thread per column, sequential down the column
    k_irv2_f<<<(n1 + 127) / 128, 128, 0, s>>>(tau1, ldt, g_row0, d0, n2, n1, alpha, f, ldf);
    return cudaGetLastError();
  }
  const int nch = (n2 + IRV2_ROWS - 1) / IRV2_ROWS;
  const dim3 grid((n1 + 127) / 128, nch);
  g_extra_launches += 1;
  k_irv2_chunk_sums<<<grid, 128, 0, s>>>(tau1, ldt, n2, n1, csum);
  k_irv2_f_chunked<<<grid, 128, 0, s>>>(tau1, ldt, g_row0, d0, n2, n1, alpha, f, ldf, csum);
  return cudaGetLastError();
}
cudaError_t launch_irv1_f(const float *tau1, const float *tau2, int ldt, const float *d0, int n2,
                          int n1, float alpha, float eps, float *f, float *dxi, int ldf,
                          cudaStream_t s) {
  k_irv1_f<<<grid2(n1, n2, 32, 8), dim3(32, 8), 0, s>>>(tau1, tau2, ldt, d0, n2, n1, alpha, eps, f,
                                                        dxi, ldf);
  return cudaGetLastError();
}
cudaError_t launch_omega0_2(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                            const float *f, const float *p1, const float *p2, int ld, int n2,
                            int n1, float *om, cudaStream_t s) {
  k_omega0_2<<<grid2(g.BP, g.AP, 32, 8, g.M), dim3(32, 8), 0, s>>>(subs, g, thy, thx, f, p1, p2,
                                                                   ld, n2, n1, om);
  return cudaGetLastError();
}
// Rows per warp of the streaming stencil kernels: the longest of 32 / 16 / 8 that still gives
// >= 8192 warps (~55 per SM) -- short row blocks cost 2-3 halo rows each, but small subdomains
// (config 3: 64 x 274 x 274) need the extra warps to keep loads in flight (measured: kernel (a)
// 46 -> 34 us, (a') 95 -> 76 us from 32 to 8 rows).
static int stencil_rb(int rows, int nsub, int strips) {
  for (int rb : {32, 16})
    if ((long long)strips * nsub * ((rows + rb - 1) / rb) >= 8192) return rb;
  return 8;
}
cudaError_t launch_sweep2x2(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                            const float *vin, const float *om, float *vout, int n2, int n1,
                            float t, cudaStream_t s) {
  const int strips = (g.B + SQ_OUT - 1) / SQ_OUT;
  dim3 grid((strips + SQ_WARPS - 1) / SQ_WARPS, (g.A + SQ_RB - 1) / SQ_RB, g.M);
  k_sweep2q2<4><<<grid, dim3(32, SQ_WARPS), 0, s>>>(subs, g, thy, thx, vin, om, vout, n2, n1, t);
  return cudaGetLastError();
}
cudaError_t launch_sweep2(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                          const float *vin, const float *om, float *vout, int n2, int n1, float t,
                          cudaStream_t s) {
  if (g.B < 512) {
    // narrow subdomains (L2-resident regime): the 2-column form keeps more warps in flight
    const int strips = (g.B + SV_OUT - 1) / SV_OUT, rb = stencil_rb(g.A, g.M, strips);
    dim3 grid((strips + SV_WARPS - 1) / SV_WARPS, (g.A + rb - 1) / rb, g.M);
    k_sweep2v<<<grid, dim3(32, SV_WARPS), 0, s>>>(subs, g, thy, thx, vin, om, vout, n2, n1, t, rb);
  } else {
    const int strips = (g.B + SQ_OUT - 1) / SQ_OUT;
    dim3 grid((strips + SQ_WARPS - 1) / SQ_WARPS, (g.A + SQ_RB - 1) / SQ_RB, g.M);
    k_sweep2q<<<grid, dim3(32, SQ_WARPS), 0, s>>>(subs, g, thy, thx, vin, om, vout, n2, n1, t);
  }
  return cudaGetLastError();
}
cudaError_t launch_combine(const SubDesc *subs, Geo g, int planes, const int2 *covy,
                           const int2 *covx, const int *loy, const int *lox, int m2loc, int k0,
                           int k1, const float *q, float *p, int ld, int n2, int row0, int row1,
                           int n1, float ahat, int *bad, const float *up, int up_r0, int up_r1,
                           const float *dn, int dn_r0, int dn_r1, cudaStream_t s) {
  if (row1 <= row0) return cudaSuccess;
  if (planes == 4)
    k_combine<4><<<grid2((n1 + 3) / 4, row1 - row0, 32, 8), dim3(32, 8), 0, s>>>(
        subs, g, covy, covx, loy, lox, m2loc, k0, k1, q, p, ld, n2, row0, row1, n1, ahat, bad, up,
        up_r0, up_r1, dn, dn_r0, dn_r1);
  else
    k_combine<2><<<grid2((n1 + 3) / 4, row1 - row0, 32, 8), dim3(32, 8), 0, s>>>(
        subs, g, covy, covx, loy, lox, m2loc, k0, k1, q, p, ld, n2, row0, row1, n1, ahat, bad, up,
        up_r0, up_r1, dn, dn_r0, dn_r1);
  return cudaGetLastError();
}
cudaError_t launch_partial(const SubDesc *subs, Geo g, int planes, const int2 *covy,
                           const int2 *covx, const int *loy, const int *lox, int m2loc, int k0,
                           int k1, const float *q, int ra, int rb, int n1, int ld, float *out,
                           cudaStream_t s) {
  if (rb <= ra) return cudaSuccess;
  k_partial<<<grid2(n1, rb - ra, 32, 8), dim3(32, 8), 0, s>>>(subs, g, planes, covy, covx, loy,
                                                              lox, m2loc, k0, k1, q, ra, rb, n1,
                                                              ld, out);
  return cudaGetLastError();
}
cudaError_t launch_recover2(const float *d0, const float *p1, const float *p2, int ld, int n2,
                            int n1, float inv_alpha, const float *shift, float *d, int row0,
                            int row1, cudaStream_t s) {
  if (row1 <= row0) return cudaSuccess;
  k_recover2<<<grid2(n1, row1 - row0, 32, 8), dim3(32, 8), 0, s>>>(d0, p1, p2, ld, n2, n1,
                                                                   inv_alpha, shift, d, row0, row1);
  return cudaGetLastError();
}
constexpr int RED_BLOCKS = 592;   // 4 x 148 SMs
cudaError_t launch_dual_energy2(const float *p1, const float *p2, const float *f, int ld, int n2,
                                int n1, int row0, int row1, double *part, double *out,
                                cudaStream_t s) {
  g_extra_launches += 1;
  k_dual2_partial<<<RED_BLOCKS, RED_T, 0, s>>>(p1, p2, f, ld, n2, n1, row0, row1, part);
  k_sum_partials<<<1, RED_T, 0, s>>>(part, RED_BLOCKS, out);
  return cudaGetLastError();
}
cudaError_t launch_irv2_zero_mean_g(float *f, int ldf, const float *d0, int n2, int n1,
                                    float alpha, double *part, double *shift, cudaStream_t s) {
  g_extra_launches += 2;
  k_sum_fd_partial<<<RED_BLOCKS / 2, RED_T, 0, s>>>(f, ldf, d0, n2, n1, part);
  k_fd_shift<<<1, 32, 0, s>>>(part, RED_BLOCKS / 2, (double)alpha, (double)n2 * n1, shift);
  k_add_shift<<<grid2(n1, n2, 32, 8), dim3(32, 8), 0, s>>>(f, ldf, n2, n1, shift);
  return cudaGetLastError();
}
cudaError_t launch_sumsq2(const float *r, size_t plane, int ld, int n1, int row0, int row1,
                          double *part, double *out, cudaStream_t s) {
  g_extra_launches += 1;
  k_sumsq2_partial<<<RED_BLOCKS, RED_T, 0, s>>>(r, plane, ld, n1, row0, row1, part);
  k_sum_partials<<<1, RED_T, 0, s>>>(part, RED_BLOCKS, out);
  return cudaGetLastError();
}
cudaError_t launch_primal1(const float *tau, size_t plane, int ld, const float *f, const float *p,
                           int n2, int n1, int row0, int row1, float delta, float scale,
                           double *part, double *out, cudaStream_t s) {
  g_extra_launches += 1;
  k_primal1_partial<<<RED_BLOCKS, RED_T, 0, s>>>(tau, plane, ld, f, p, n2, n1, row0, row1, delta,
                                                 scale, part);
  k_sum_partials_multi<<<3, RED_T, 0, s>>>(part, RED_BLOCKS, out);
  return cudaGetLastError();
}
cudaError_t launch_primal2(const float *d, const float *d0, const float *f, const float *dxi,
                           const float *p1, const float *p2, int ldf, int n2, int n1, int row0,
                           int row1, float inv_alpha, double *part, double *out, cudaStream_t s) {
  g_extra_launches += 1;
  k_primal2_partial<<<RED_BLOCKS, RED_T, 0, s>>>(d, d0, f, dxi, p1, p2, ldf, n2, n1, row0, row1,
                                                 inv_alpha, part);
  k_sum_partials_multi<<<4, RED_T, 0, s>>>(part, RED_BLOCKS, out);
  return cudaGetLastError();
}
cudaError_t launch_sum_ranks(const double *vals, int world, int stride, int n, double *out,
                             cudaStream_t s) {
  k_sum_ranks<<<1, 32, 0, s>>>(vals, world, stride, n, out);
  return cudaGetLastError();
}
cudaError_t launch_multidiv(const float *p, int ld, int n2, int n1, float *w, int row0, int row1,
                            cudaStream_t s) {
  if (row1 <= row0) return cudaSuccess;
  k_multidiv<<<grid2(n1, row1 - row0, 32, 8), dim3(32, 8), 0, s>>>(p, ld, n2, n1, w, row0, row1);
  return cudaGetLastError();
}
cudaError_t launch_div(const float *w1, const float *w2, int ld, int n2, int n1, float *q,
                       float *qlo, int row0, int row1, cudaStream_t s) {
  if (row1 <= row0) return cudaSuccess;
  k_div<<<grid2(n1, row1 - row0, 32, 8), dim3(32, 8), 0, s>>>(w1, w2, ld, n2, n1, q, qlo, row0,
                                                              row1);
  return cudaGetLastError();
}
cudaError_t launch_axpby2(const float *a, const float *b, const float *c, int ld, int n2, int n1,
                          float sa, float sb, float sc, float *out, int row0, int row1,
                          cudaStream_t s) {
  if (row1 <= row0) return cudaSuccess;
  k_axpby2<<<grid2(n1, row1 - row0, 32, 8), dim3(32, 8), 0, s>>>(a, b, c, ld, n2, n1, sa, sb, sc,
                                                                 out, row0, row1);
  return cudaGetLastError();
}
cudaError_t launch_load_tp(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                           const float *p, int ld, int n2, int n1, float *v, cudaStream_t s) {
  (void)n1;
  k_load_tp<<<grid2(g.B, g.A, 32, 8, g.M), dim3(32, 8), 0, s>>>(subs, g, thy, thx, p, ld, n2, v);
  return cudaGetLastError();
}
cudaError_t launch_prediv1(const SubDesc *subs, Geo g, const float *v, int n2, int n1, float *q,
                           const float *qsub, cudaStream_t s) {
  const int strips = (g.BT + S1_OUT - 1) / S1_OUT, rb = stencil_rb(g.AT, g.M, strips);
  dim3 grid((strips + S1_WARPS - 1) / S1_WARPS, (g.AT + rb - 1) / rb, g.M);
  k_prediv1s<<<grid, dim3(32, S1_WARPS), 0, s>>>(subs, g, v, n2, n1, q, qsub, rb);
  return cudaGetLastError();
}
cudaError_t launch_omega0_1(const SubDesc *subs, Geo g, const float *r, int ld, const float *v,
                            int n2, int n1, float *om, cudaStream_t s) {
  k_omega0_1<<<grid2(g.BP, g.AP, 32, 8, g.M), dim3(32, 8), 0, s>>>(subs, g, r, ld, v, n2, n1, om);
  return cudaGetLastError();
}
cudaError_t launch_sweep1(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                          const float *vin, const float *gphi, int ldg, const float *om,
                          float *vout, int n2, int n1, float t, cudaStream_t s) {
  const int strips = (g.B + S1_OUT - 1) / S1_OUT, rb = stencil_rb(g.A, g.M, strips);
  dim3 grid((strips + S1_WARPS - 1) / S1_WARPS, (g.A + rb - 1) / rb, g.M);
  if (om)
    k_sweep1s<true><<<grid, dim3(32, S1_WARPS), 0, s>>>(subs, g, thy, thx, vin, gphi, ldg, om, vout,
                                                        n2, n1, t, rb);
  else
    k_sweep1s<false><<<grid, dim3(32, S1_WARPS), 0, s>>>(subs, g, thy, thx, vin, gphi, ldg, om, vout,
                                                         n2, n1, t, rb);
  return cudaGetLastError();
}
cudaError_t launch_dct_tables(int n, float *cf, float *cn, float *sn, float *snT, float *split6,
                              int ld, cudaStream_t s) {
  k_dct_tables<<<grid2(n, n, 32, 8), dim3(32, 8), 0, s>>>(n, cf, cn, sn, snT, split6, ld);
  return cudaGetLastError();
}
cudaError_t launch_pivots(const ProjTile *tiles, const int *first, int nchains, int n2, int n1,
                          double *rinv, int ldn, int AT, int *pcut, double *pinf, double *plast,
                          cudaStream_t s) {
  k_pivots<<<dim3((n1 + 127) / 128, nchains), 128, 0, s>>>(tiles, first, nchains, n2, n1, rinv,
                                                           ldn, AT, pcut, pinf, plast);
  return cudaGetLastError();
}
cudaError_t launch_gemm(const GemmDesc *descs, int batch, int maxM, int maxN, cudaStream_t s) {
  k_gemm<<<dim3((maxN + GBN - 1) / GBN, (maxM + GBM - 1) / GBM, batch), 256, 0, s>>>(descs);
  return cudaGetLastError();
}
int solve_nseg(int AT) {
  constexpr int ls = 32;   // target rows per segment
  return std::min(SSEG_MAX, std::max(1, (AT + ls - 1) / ls));
}
// column block width of solve4: 16 for tiles up to 512 rows (four CTAs per SM instead of two:
// config 3 -3 %), else 32
static int solve_j(int AT) {
  return AT <= 512 ? 16 : 32;
}
int solve4_width(int AT) { return solve_j(AT); }
bool solve4_fits(int AT) { return (size_t)(AT + 1) * solve_j(AT) * (sizeof(float) + sizeof(double)) <= 200 * 1024; }
cudaError_t launch_segprod(const ProjTile *tiles, const int *first, int nchains, const double *rinv,
                           int ldn, int AT, int n1, double *segprod, cudaStream_t s) {
  k_segprod<<<dim3((n1 + 127) / 128, nchains), 128, 0, s>>>(tiles, first, nchains, rinv, ldn, AT,
                                                            n1, solve_nseg(AT), segprod);
  return cudaGetLastError();
}
cudaError_t launch_proj_solve4(const ProjTile *tiles, int ntiles, int n2, int n1,
                               const float *qhat, int AT, int ldn, const double *rinv,
                               const double *segprod, float *phx, float *phy, int AP,
                               const SolveMaps *maps, int smem_rows, const int *order,
                               int nchains, int per_chain, cudaStream_t s) {
  const int nseg = solve_nseg(AT), J = solve_j(AT);
  const int srows = maps ? smem_rows : AT;
  const size_t smem = (size_t)srows * J * (sizeof(float) + sizeof(double));
  // (the kernel also has up to ~8.5 KB of static shared memory: opt in whenever the sum passes 48 KB)
  if (smem + 9 * 1024 > 48 * 1024) {
    cudaError_t e = smem_optin(J == 16 ? (const void *)k_proj_solve4<16> : (const void *)k_proj_solve4<32>, smem);
    if (e != cudaSuccess) return e;
  }
  (void)ntiles;
  if (J == 16)
    k_proj_solve4<16><<<dim3((n1 + 15) / 16, per_chain, nchains), dim3(16, nseg), smem, s>>>(
        tiles, n2, n1, qhat, AT, ldn, rinv, segprod, phx, phy, AP, maps, srows, order, per_chain);
  else
    k_proj_solve4<32><<<dim3((n1 + 31) / 32, per_chain, nchains), dim3(32, nseg), smem, s>>>(
        tiles, n2, n1, qhat, AT, ldn, rinv, segprod, phx, phy, AP, maps, srows, order, per_chain);
  return cudaGetLastError();
}
cudaError_t launch_gsolve(int phase, const int *seglo, int nseg, int s0, int s1, int n1, int n2,
                          const float *qhat, int ldn, const double *rinv, const int *pcut,
                          const double *pinf, const double *plast, int nt, const double *agg,
                          double *aggb_or_out, float *zs, float *phx, float *phy, int po,
                          cudaStream_t s) {
  if (s1 <= s0) return cudaSuccess;
  const dim3 grid((n1 + 127) / 128, s1 - s0);
  if (phase == 0)
    k_gsolve_a<<<grid, 128, 0, s>>>(seglo, s0, s1, n1, qhat, ldn, rinv, pcut, pinf, plast, nt,
                                    aggb_or_out);
  else if (phase == 1)
    k_gsolve_b<<<grid, 128, 0, s>>>(seglo, nseg, s0, s1, n1, qhat, ldn, rinv, pcut, pinf, plast,
                                    nt, agg, zs, aggb_or_out);
  else
    k_gsolve_c<<<grid, 128, 0, s>>>(seglo, nseg, s0, s1, n1, n2, qhat, ldn, rinv, pcut, pinf,
                                    plast, nt, agg, aggb_or_out, zs, phx, phy, po);
  return cudaGetLastError();
}
cudaError_t launch_proj_solve3(const ProjTile *tiles, int ntiles, int n2, int n1,
                               const float *qhat, int AT, int ldn, const double *rinv, float *z,
                               float *phx, float *phy, float *phx_lo, float *phy_lo, int AP,
                               const int *pcut, const double *pinf, const double *plast,
                               cudaStream_t s) {
  // one warp per segment of >= 32 rows, at most S3SEG_MAX segments (the max tile height decides);
  // the staged form whenever a 32-column block would fit 160 KB (the plan sizes the global z
  // scratch with the same rule, proj_tile_bytes)
  const int nseg = std::min(S3SEG_MAX, std::max(1, AT / 32));
  if ((size_t)AT * SJB * sizeof(float) <= 160 * 1024) {
    // staged form in 16-column blocks (512 threads, <= 64 registers): two CTAs per SM, so one
    // CTA's staging overlaps the other's passes (config-4 local solve 286 -> 273 us against
    // 32-column blocks, bitwise the same)
    const dim3 grid16((n1 + 15) / 16, ntiles), block16(16, nseg);
    const size_t smem16 = (size_t)AT * 16 * sizeof(float);
    cudaError_t e = smem_optin((const void *)k_proj_solve3<true, 16>, smem16);
    if (e != cudaSuccess) return e;
    k_proj_solve3<true, 16><<<grid16, block16, smem16, s>>>(tiles, n2, n1, qhat, AT, ldn, rinv, z,
                                                             phx, phy, phx_lo, phy_lo, AP, pcut,
                                                             pinf, plast);
    return cudaGetLastError();
  }
  const dim3 grid((n1 + SJB - 1) / SJB, ntiles), block(SJB, nseg);   // z in the global scratch
  k_proj_solve3<false, SJB><<<grid, block, 0, s>>>(tiles, n2, n1, qhat, AT, ldn, rinv, z, phx, phy,
                                               phx_lo, phy_lo, AP, pcut, pinf, plast);
  return cudaGetLastError();
}
}  // namespace tvs
