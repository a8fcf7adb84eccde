// Fast partial x-DCTs of the projection kernel (b) by the chirp-z transform (
// "Fast DCT could help").  Same operators as the dense contractions of tvs_gemm_tc.cu:
//   forward  Qhat[j]  = sum_{x in tile} q[x] cos(theta j (2x+1))              j = 0 .. N-1
//   inverse  out_y[x] = sum_j Phi_y[j] cos(theta j (2x+1))                    x in the tile
//            out_x[x] = sum_j Phi_x[j] sin(theta j (2x+2))
// with theta = pi / (2N) (Eq. form:DCTmat, and the spectral x-derivative of
// DESIGN.md section 5).  With x = tx0 + u (u tile-relative) and 2jv = j^2 + v^2 - (j - v)^2 every
// sum is  out[v] = Op( post[v] sum_u in[u] pre[u] h[v - u] ),  h[m] = e^{-i theta m^2} (even in m),
// a linear convolution with a chirp, evaluated by an in-place radix-4 FFT of size M (power of 4)
// in shared memory: DIF (natural -> digit-reversed), multiply by the precomputed digit-reversed
// FFT of the circular kernel window, DIT (digit-reversed -> natural).  Inputs are cut into chunks
// of Uc and outputs into passes of Vp with Uc + Vp - 1 <= M; chunk c / pass p uses the kernel
// window g[n] = h[(v0 - u0) + n] for n in [-(M - Vp), Vp - 1].  When the tile spans the whole axis
// and M = 2N - 2 one pass suffices (h even: the one colliding index holds the same value).
// Cost per row O(M log M) instead of O(width * N): the dense GEMM stays faster for narrow tiles
// (config 3), the chirp-z for full-width strips and large N (configs 4, 5).  fp32 FFT arithmetic;
// pre/post chirps from per-job tables built on the host (phases reduced exactly mod 4N in
// integers, angles in fp64, one rounding), kernel FFTs in fp64 on the host.
//
// Makhoul form (CztGeom::mk; whenever M = 2N - 2 is a power of 4, e.g. N = 2049, 8193): every
// transform is a DFT_N of a COMPLEX sequence that packs two real ones, evaluated by Bluestein
// (X_k = conj(c_k) sum_n z_n conj(c_n) c_{k-n}, c_m = e^{i pi m^2 / N}, even, so the one aliased
// lag of the cyclic length 2N - 2 holds the same value):
//   kind 3, forward, rows r and r+1 at once: Makhoul's DCT-II, v_n = q_{2n} (n < (N+1)/2),
//     v_{N-1-n} = q_{2n+1}; Z = DFT_N(v_a + i v_b); A_k = (Z_k + conj Z_{N-k}) / 2,
//     B_k = (Z_k - conj Z_{N-k}) / (2i); Qhat_a[k] = Re(e^{-i pi k/(2N)} A_k), same for b;
//   kind 4, inverse y, rows r and r+1: the DCT-III T(a)[x] = sum_j a_j cos(theta j (2x+1)) by the
//     inverse Makhoul map V_k = e^{i pi k/(2N)} (a''_k - i a''_{N-k}) (a''_0 = 2 a_0, a''_N = 0),
//     v = (N/2) IDFT_N(V_a + i V_b) (both real parts), T(a)[2n] = v_n, T(a)[2n+1] = v_{N-1-n};
//   kind 5, inverse x, one row: sum_j b_j sin(theta j (2x+2)) = (-1)^x T(c)[x] + T(d)[x] with
//     c_k = b_{N-k} cos(delta_{N-k}) (c_0 = 0), d_k = b_k sin(delta_k), delta_k = pi k/(2N)
//     (sin(theta j (2x+2)) = sin(A_j + delta_j) and sin A_j = (-1)^x cos A_{N-j}), both DCT-IIIs
//     packed in one DFT -- the global projection's form (its error enters tau directly);
//   kind 6, inverse x, rows r and r+1 -- the local projections of the inner loop: sum_j b_j sin(theta j (2x+2)) = phi(x+1) - phi(x) with
//     phi = T(a), a_j = b_j xs_j, xs_j = -1 / (2 sin(pi j/(2N))) (xs_0 = 0: the constant mode has
//     no x-derivative) -- b_j sin(theta j (2x+2)) = a_j (cos(theta j (2x+3)) - cos(theta j (2x+1)));
//     the DCT-III by the kind-4 map, phi(x+1) from the neighbouring lane.  phi is formed in fp32
//     shared memory and differenced (never stored): on the config-3 P tau_0 field the error is
//     ~2x that of the direct sine form (4e-7 vs 2e-7 of max |D+_x phi|),
//     for one DFT per row pair instead of one per row.
// Per pair of rows: 1 transform forward (general form: 2); inverse 2 (local, kind 6) or 3 (global,
// kind 5; general form: 4).
#include "tvs_internal.h"

#include <cmath>
#include <complex>
#include <map>
#include <vector>

namespace tvs {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {   // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
#ifndef TVS_CZT_THREADS
#define TVS_CZT_THREADS 512
#endif
constexpr int CZT_THREADS = TVS_CZT_THREADS;   // threads per chirp-z CTA (build-time A/B: 512 / 1024)

// Row pointers of one chunk for the pruned first / last FFT passes.
struct CztIo {
  const float *in;
  const float2 *pre;
  int ucnt;
  float *out;
  const float *add;   // nullable: out = transform + add (same row layout as out)
  const float2 *post;
  int vcnt, kind;
  bool pin, pout;
  bool half = false;   // Makhoul form: nonzero inputs / needed outputs only at indices 0 .. M/2
};

// Shared-memory FFT layout: element i lives at i + i/16 (one float2 of padding per 16), which
// makes every access pattern below at most 2-way bank-conflicted.
__device__ __forceinline__ int pz(int i) { return i + (i >> 4); }
// pz(base + m S) - pz(base) for the 16-element groups of the fused passes: exact whenever S is a
// multiple of 16, or S = 4 with base % 16 < 4 (every call below); with S and m compile-time
// constants the group's 16 accesses become immediate offsets from one address.
__device__ __forceinline__ int pzo(int m, int S) { return m * S + ((m * S) >> 4); }

// Twiddle w^n = e^{-2 pi i n / M}.  TVS_CZT_TWG (default): one read of the full M-entry table in
// global memory (L1 / L2-resident, off the shared-memory pipe the FFT passes saturate);
// otherwise a two-level table in shared memory, fine[n & 255] * coarse[n >> 8].
#ifndef TVS_CZT_TWG
#define TVS_CZT_TWG 1
#endif
// (Measured and rejected: all 15 twiddles of a fused pair read from the table instead of 2 reads
// and 13 complex products -- forward +43 %, inverse +41 % at config 4: L2 latency.)
struct Tw {
  const float2 *fine, *coarse, *full;
  __device__ __forceinline__ float2 operator()(int n) const {
#if TVS_CZT_TWG
    return __ldg(full + n);
#else
    const float2 f = fine[n & 255];
    return (n >> 8) ? cmul(f, coarse[n >> 8]) : f;
#endif
  }
};

__device__ __forceinline__ void bfly4_dif(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
  const float2 a0 = make_float2(x0.x + x2.x, x0.y + x2.y), a1 = make_float2(x0.x - x2.x, x0.y - x2.y);
  const float2 a2 = make_float2(x1.x + x3.x, x1.y + x3.y), a3 = make_float2(x1.x - x3.x, x1.y - x3.y);
  x0 = make_float2(a0.x + a2.x, a0.y + a2.y);
  x1 = make_float2(a1.x + a3.y, a1.y - a3.x);   // a1 - i a3
  x2 = make_float2(a0.x - a2.x, a0.y - a2.y);
  x3 = make_float2(a1.x - a3.y, a1.y + a3.x);   // a1 + i a3
}
__device__ __forceinline__ void bfly4_dit(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
  const float2 a0 = make_float2(x0.x + x2.x, x0.y + x2.y), a1 = make_float2(x0.x - x2.x, x0.y - x2.y);
  const float2 a2 = make_float2(x1.x + x3.x, x1.y + x3.y), a3 = make_float2(x1.x - x3.x, x1.y - x3.y);
  x0 = make_float2(a0.x + a2.x, a0.y + a2.y);
  x1 = make_float2(a1.x - a3.y, a1.y + a3.x);   // a1 + i a3
  x2 = make_float2(a0.x - a2.x, a0.y - a2.y);
  x3 = make_float2(a1.x + a3.y, a1.y - a3.x);   // a1 - i a3
}

// In-place radix-4 DIF on z (natural order in, base-4 digit-reversed out).  Consecutive stage
// pairs (spans L and L/4) are fused: a thread loads the 16 elements {base + m L/4} that the two
// stages mix, runs both in registers and stores them back (one shared-memory round trip per
// pair); an odd number of stages ends with one plain radix-4 stage (span 1).
// e^{-2 pi i e / 16} for compile-time e (the fixed part of a fused pair's twiddles)
__device__ __forceinline__ float2 w16(int e) {
  constexpr float C[16] = {1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                           0.f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                           -1.f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                           0.f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
  return make_float2(C[e & 15], -C[(e + 12) & 15]);   // sin(x) = cos(x - pi/2)
}

// The last DIF pass (span 1, or the pair of spans 4 and 1) is left to czt_middle, which fuses it
// with the pointwise kernel multiply and the first DIT pass: both touch the same 4 (or 16)
// consecutive elements, so the three run in registers.
// PIN (narrow input, ucnt <= M/16): the first pair (spans M/4, M/16) sees one nonzero element per
// group, element kp = in[kp] pre[kp] (kp < M/16), so its 16 outputs are that value times W^t V^c;
// it reads the input row straight from global memory (no staging pass) and performs exactly the
// products of the full pass (the butterflies only add zeros), so the result is bitwise the same.
// HALF (Makhoul form, inputs zero at and beyond index M/2 + 1): the first pair (spans M/4, M/16,
// base = kp) reads only its elements m < 8 and, for kp = 0, m = 8 (index M/2); the rest are zero.
template <int logM4, bool PIN, bool HALF = false>
__device__ __forceinline__ void fft_dif(float2 *z, const Tw &tw, const float *__restrict__ in,
                                        const float2 *__restrict__ pre, int ucnt) {
  constexpr int M = 1 << (2 * logM4), nth = CZT_THREADS;
  const int tid = threadIdx.x;
  if constexpr (PIN) {
    constexpr int Q = M >> 4;   // s1 = 1 on the first pair
    for (int kp = tid; kp < Q; kp += nth) {
      float2 a = make_float2(0.f, 0.f);
      if (kp < ucnt) {
        const float x = __ldg(in + kp);
        const float2 c = __ldg(pre + kp);
        a = make_float2(x * c.x, x * c.y);
      }
      const float2 W1 = tw(kp), W2 = cmul(W1, W1), W3 = cmul(W1, W2);
      const float2 V1 = tw(4 * kp), V2 = cmul(V1, V1), V3 = cmul(V1, V2);
      const float2 aw[4] = {a, cmul(a, W1), cmul(a, W2), cmul(a, W3)};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        z[pz(kp + (4 * t) * Q)] = aw[t];
        z[pz(kp + (4 * t + 1) * Q)] = cmul(aw[t], V1);
        z[pz(kp + (4 * t + 2) * Q)] = cmul(aw[t], V2);
        z[pz(kp + (4 * t + 3) * Q)] = cmul(aw[t], V3);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int lg = PIN ? logM4 - 3 : logM4 - 1; lg >= 2; lg -= 2) {
    const int L = 1 << (2 * lg), Q = L >> 2, s1 = M >> (2 * lg + 2);
#pragma unroll
    for (int it = 0; it < ((M >> 4) + nth - 1) / nth; ++it) {   // compile-time trip count
      const int gidx = tid + it * nth;
      if (((M >> 4) % nth) && gidx >= (M >> 4)) break;
      const int blk = gidx >> (2 * lg - 2), kp = gidx & (Q - 1);
      const int base = blk * 4 * L + kp;
      float2 x[16];
      float2 *zb = z + pz(base);   // base % 16 = kp < Q when Q = 4
      if (HALF && lg == logM4 - 1) {
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = zb[pzo(m, Q)];
        x[8] = kp == 0 ? zb[pzo(8, Q)] : make_float2(0.f, 0.f);
#pragma unroll
        for (int m = 9; m < 16; ++m) x[m] = make_float2(0.f, 0.f);
      } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) x[m] = zb[pzo(m, Q)];
      }
      // twiddles of the pair from two lookups: stage 1 (span L, k = kp + r Q) uses
      // w^{c k s1} = W^c * e^{-2 pi i c r / 16} with W = w^{kp s1}; stage 2 (span Q, k = kp,
      // stride 4 s1) uses V^c with V = w^{4 kp s1} (looked up, not W^4: keeps the error flat).
      const float2 W1 = tw(kp * s1), W2 = cmul(W1, W1), W3 = cmul(W1, W2);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        bfly4_dif(x[r], x[r + 4], x[r + 8], x[r + 12]);
        x[r + 4] = cmul(x[r + 4], r ? cmul(W1, w16(r)) : W1);
        x[r + 8] = cmul(x[r + 8], r ? cmul(W2, w16(2 * r)) : W2);
        x[r + 12] = cmul(x[r + 12], r ? cmul(W3, w16(3 * r)) : W3);
      }
      const float2 V1 = tw(4 * kp * s1), V2 = cmul(V1, V1), V3 = cmul(V1, V2);   // direct lookup
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        bfly4_dif(x[4 * t], x[4 * t + 1], x[4 * t + 2], x[4 * t + 3]);
        x[4 * t + 1] = cmul(x[4 * t + 1], V1);
        x[4 * t + 2] = cmul(x[4 * t + 2], V2);
        x[4 * t + 3] = cmul(x[4 * t + 3], V3);
      }
#pragma unroll
      for (int m = 0; m < 16; ++m) zb[pzo(m, Q)] = x[m];
    }
    __syncthreads();
  }
}

// Last DIF pass, pointwise multiply by the transformed kernel gk (digit-reversed order, as the
// DIF output), first DIT pass.  logM4 odd: span-1 stages on 4 consecutive elements (no twiddles);
// even: the span-4/span-1 pairs on 16 consecutive elements (kp = 0: twiddles e^{-2 pi i c r/16}).
template <int logM4>
__device__ __forceinline__ void czt_middle(float2 *z, const float2 *__restrict__ gk) {
  constexpr int M = 1 << (2 * logM4), nth = CZT_THREADS;
  const int tid = threadIdx.x;
  if constexpr (logM4 & 1) {
    for (int b = tid; b < (M >> 2); b += nth) {
      const float4 g01 = __ldg(reinterpret_cast<const float4 *>(gk + 4 * b));
      const float4 g23 = __ldg(reinterpret_cast<const float4 *>(gk + 4 * b + 2));
      float2 x0 = z[pz(4 * b)], x1 = z[pz(4 * b + 1)], x2 = z[pz(4 * b + 2)], x3 = z[pz(4 * b + 3)];
      bfly4_dif(x0, x1, x2, x3);
      x0 = cmul(x0, make_float2(g01.x, g01.y));
      x1 = cmul(x1, make_float2(g01.z, g01.w));
      x2 = cmul(x2, make_float2(g23.x, g23.y));
      x3 = cmul(x3, make_float2(g23.z, g23.w));
      bfly4_dit(x0, x1, x2, x3);
      z[pz(4 * b)] = x0;
      z[pz(4 * b + 1)] = x1;
      z[pz(4 * b + 2)] = x2;
      z[pz(4 * b + 3)] = x3;
    }
  } else {
#pragma unroll
    for (int it = 0; it < ((M >> 4) + nth - 1) / nth; ++it) {   // compile-time trip count
      const int gidx = tid + it * nth;
      if (((M >> 4) % nth) && gidx >= (M >> 4)) break;
      const int base = gidx * 16;
      float4 g[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) g[m] = __ldg(reinterpret_cast<const float4 *>(gk + base) + m);
      float2 x[16];
      float2 *zb = z + 17 * gidx;   // pz(16 gidx + m) = 17 gidx + m
#pragma unroll
      for (int m = 0; m < 16; ++m) x[m] = zb[m];
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // DIF span 4, k = r
        bfly4_dif(x[r], x[r + 4], x[r + 8], x[r + 12]);
        if (r) {
          x[r + 4] = cmul(x[r + 4], w16(r));
          x[r + 8] = cmul(x[r + 8], w16(2 * r));
          x[r + 12] = cmul(x[r + 12], w16(3 * r));
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) bfly4_dif(x[4 * t], x[4 * t + 1], x[4 * t + 2], x[4 * t + 3]);
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        x[2 * m] = cmul(x[2 * m], make_float2(g[m].x, g[m].y));
        x[2 * m + 1] = cmul(x[2 * m + 1], make_float2(g[m].z, g[m].w));
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) bfly4_dit(x[4 * t], x[4 * t + 1], x[4 * t + 2], x[4 * t + 3]);
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // DIT span 4, k = r
        if (r) {
          x[r + 4] = cmulc(x[r + 4], w16(r));
          x[r + 8] = cmulc(x[r + 8], w16(2 * r));
          x[r + 12] = cmulc(x[r + 12], w16(3 * r));
        }
        bfly4_dit(x[r], x[r + 4], x[r + 8], x[r + 12]);
      }
#pragma unroll
      for (int m = 0; m < 16; ++m) zb[m] = x[m];
    }
  }
  __syncthreads();
}

// In-place radix-4 DIT with conjugate twiddles (digit-reversed in, natural out): the inverse
// transform times M.  Mirror image of fft_dif: after czt_middle's first pass, fused pairs of
// spans L and 4L.
// POUT (narrow output, vcnt <= M/16): the last pair (spans M/16, M/4) is evaluated only for its
// output element 0 of each group, kp < vcnt, in the full pass's operation order, and the result
// goes through the post-chirp straight to global memory (kind 2: imaginary part).
// HALF (Makhoul form, only outputs 0 .. M/2 are read): the last pair (spans M/16, M/4, base = kp)
// stores only its elements m < 8 and, for kp = 0, m = 8.
template <int logM4, bool POUT, bool HALF = false>
__device__ __forceinline__ void fft_dit_inv(float2 *z, const Tw &tw, float *__restrict__ out,
                                            const float2 *__restrict__ post, int vcnt, int kind,
                                            const float *__restrict__ add) {
  constexpr int M = 1 << (2 * logM4), nth = CZT_THREADS;
  const int tid = threadIdx.x;
#pragma unroll
  for (int lg = (logM4 & 1) ? 1 : 2; lg < (POUT ? logM4 - 2 : logM4); lg += 2) {   // first pass: czt_middle
    const int L = 1 << (2 * lg), s2 = M >> (2 * lg + 4);
#pragma unroll
    for (int it = 0; it < ((M >> 4) + nth - 1) / nth; ++it) {   // compile-time trip count
      const int gidx = tid + it * nth;
      if (((M >> 4) % nth) && gidx >= (M >> 4)) break;
      const int blk = gidx >> (2 * lg), kp = gidx & (L - 1);
      const int base = blk * 16 * L + kp;
      float2 x[16];
      float2 *zb = z + pz(base);   // base % 16 = kp < L when L = 4
#pragma unroll
      for (int m = 0; m < 16; ++m) x[m] = zb[pzo(m, L)];
      // stage 2 (span 4L, k = kp + r L, stride s2) uses U^c e^{-2 pi i c r/16}, U = w^{kp s2};
      // stage 1 (span L, k = kp, stride 4 s2) uses U^{4c}
      const float2 U1 = tw(kp * s2), U2 = cmul(U1, U1), U3 = cmul(U1, U2);
      const float2 V1 = tw(4 * kp * s2), V2 = cmul(V1, V1), V3 = cmul(V1, V2);   // direct lookup
#pragma unroll
      for (int t = 0; t < 4; ++t) {   // span L, k = kp
        x[4 * t + 1] = cmulc(x[4 * t + 1], V1);
        x[4 * t + 2] = cmulc(x[4 * t + 2], V2);
        x[4 * t + 3] = cmulc(x[4 * t + 3], V3);
        bfly4_dit(x[4 * t], x[4 * t + 1], x[4 * t + 2], x[4 * t + 3]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // span 4L, k = kp + r L
        x[r + 4] = cmulc(x[r + 4], r ? cmul(U1, w16(r)) : U1);
        x[r + 8] = cmulc(x[r + 8], r ? cmul(U2, w16(2 * r)) : U2);
        x[r + 12] = cmulc(x[r + 12], r ? cmul(U3, w16(3 * r)) : U3);
        bfly4_dit(x[r], x[r + 4], x[r + 8], x[r + 12]);
      }
      if (HALF && lg == logM4 - 2) {
#pragma unroll
        for (int m = 0; m < 8; ++m) zb[pzo(m, L)] = x[m];
        if (kp == 0) zb[pzo(8, L)] = x[8];
      } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) zb[pzo(m, L)] = x[m];
      }
    }
    __syncthreads();
  }
  if constexpr (POUT) {
    constexpr int L = M >> 4;   // s2 = 1 on the last pair
    for (int kp = tid; kp < vcnt; kp += nth) {
      float2 x[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) x[m] = z[pz(kp + m * L)];
      const float2 U1 = tw(kp), U2 = cmul(U1, U1), U3 = cmul(U1, U2);
      const float2 V1 = tw(4 * kp), V2 = cmul(V1, V1), V3 = cmul(V1, V2);
      float2 y[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {   // span L, k = kp: first butterfly output = plain sum
        const float2 b1 = cmulc(x[4 * t + 1], V1), b2 = cmulc(x[4 * t + 2], V2),
                     b3 = cmulc(x[4 * t + 3], V3);
        const float2 a0 = make_float2(x[4 * t].x + b2.x, x[4 * t].y + b2.y);
        const float2 a2 = make_float2(b1.x + b3.x, b1.y + b3.y);
        y[t] = make_float2(a0.x + a2.x, a0.y + a2.y);
      }
      // span 4L, r = 0: twiddles U^c, first output
      const float2 c1 = cmulc(y[1], U1), c2 = cmulc(y[2], U2), c3 = cmulc(y[3], U3);
      const float2 a0 = make_float2(y[0].x + c2.x, y[0].y + c2.y);
      const float2 a2 = make_float2(c1.x + c3.x, c1.y + c3.y);
      const float2 o = cmul(__ldg(post + kp), make_float2(a0.x + a2.x, a0.y + a2.y));
      const float v = kind == 2 ? o.y : o.x;
      out[kp] = add ? v + add[kp] : v;
    }
  }
}


// FFT -> kernel multiply -> inverse FFT of one chunk, with the size a compile-time constant so
// every shared-memory offset inside a pass folds to an immediate.
template <int logM4, bool PIN, bool POUT, bool HALF = false>
__device__ __forceinline__ void czt_fft_pair_t(float2 *z, const Tw &tw, const float2 *__restrict__ gk,
                                               const CztIo &io) {
  fft_dif<logM4, PIN, HALF>(z, tw, io.in, io.pre, io.ucnt);
  czt_middle<logM4>(z, gk);
  fft_dit_inv<logM4, POUT, HALF>(z, tw, io.out, io.post, io.vcnt, io.kind, io.add);
}
template <int logM4>
__device__ __forceinline__ void czt_fft_pair_p(float2 *z, const Tw &tw, const float2 *__restrict__ gk,
                                               const CztIo &io) {
  if constexpr (logM4 >= 3) {
    if (io.half) return czt_fft_pair_t<logM4, false, false, true>(z, tw, gk, io);
    if (io.pin && io.pout) return czt_fft_pair_t<logM4, true, true>(z, tw, gk, io);
    if (io.pin) return czt_fft_pair_t<logM4, true, false>(z, tw, gk, io);
    if (io.pout) return czt_fft_pair_t<logM4, false, true>(z, tw, gk, io);
  }
  czt_fft_pair_t<logM4, false, false>(z, tw, gk, io);
}
__device__ __forceinline__ void czt_fft_pair(float2 *z, int logM4, const Tw &tw,
                                             const float2 *__restrict__ gk, const CztIo &io) {
  switch (logM4) {
    case 1: czt_fft_pair_p<1>(z, tw, gk, io); break;
    case 2: czt_fft_pair_p<2>(z, tw, gk, io); break;
    case 3: czt_fft_pair_p<3>(z, tw, gk, io); break;
    case 4: czt_fft_pair_p<4>(z, tw, gk, io); break;
    case 5: czt_fft_pair_p<5>(z, tw, gk, io); break;
    case 6: czt_fft_pair_p<6>(z, tw, gk, io); break;
    default: czt_fft_pair_p<7>(z, tw, gk, io); break;
  }
}

// Makhoul form (see the file header): one CTA per (row pair or row, job).  pre = c table,
// post = e table (n, k < N).
// L2 prefetch (TVS_CZT_L2PF): one CTA per SM and nothing to overlap its load / output phases with,
// so while the FFT pair runs, four threads ask L2 for (a) this item's omega0 rows (read by the
// output phase, TVS ncu: the output phase's first uses are long-scoreboard stalls) and (b) the
// input rows of the item one wave ahead (linear CTA id + G.ahead): its load phase then waits on
// L2 instead of DRAM.  No shared memory or registers held (the staged variant's carve-out cost the
// tables their L1); results bitwise the same.
#ifndef TVS_CZT_L2PF
#define TVS_CZT_L2PF 1
#endif
__device__ __forceinline__ void l2_prefetch(const float *p, int n) {
  if (!p || n <= 0) return;
  const unsigned long long a = reinterpret_cast<unsigned long long>(p), lo = a & ~15ull;
  const unsigned long long hi = (a + 4ull * (unsigned long long)n + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(lo), "r"((unsigned)(hi - lo))
               : "memory");
}

template <int KSET>   // 1: forward (kind 3 only), 2: inverse (kinds 4, 5, 6)
__device__ __forceinline__ void czt_makhoul(const CztJob &jb, const CztJob *__restrict__ jobs,
                                            const CztGeom &G, const float2 *__restrict__ gtab,
                                            const float2 *__restrict__ tw, float2 *zsm, int MP) {
  const int N = G.N, M = G.M, tid = threadIdx.x, nth = blockDim.x;
  const int kind = KSET == 1 ? 3 : jb.kind;
  const int r0 = kind == 5 ? blockIdx.x : 2 * blockIdx.x;   // kind 5: one row, else a row pair
  if (r0 >= jb.rows) return;
  const bool two = kind != 5 && r0 + 1 < jb.rows;
  float2 *tfine = zsm + MP, *tcoarse = tfine + 256;
  for (int i = tid; i < 256; i += nth) tfine[i] = i < M ? __ldg(tw + i) : make_float2(1.f, 0.f);
  for (int i = tid; i <= (M >> 8); i += nth) tcoarse[i] = (i << 8) < M ? __ldg(tw + (i << 8)) : make_float2(1.f, 0.f);
  const Tw twd{tfine, tcoarse, tw};
  const float2 *__restrict__ cc = jb.pre;    // c_n = e^{i pi n^2 / N}
  const float2 *__restrict__ ee = jb.post;   // e_k = e^{i pi k / (2N)}
  const float *__restrict__ ia = jb.in + (size_t)r0 * jb.ldin;
  const float *__restrict__ ib = two ? ia + jb.ldin : nullptr;
  const int h = (N + 1) >> 1;
  // loads are issued in batches of B per thread (all loads of a batch before any use: the
  // kernel is latency-bound on them otherwise)
  // B = 9: 9 x 512 x 2 >= N = 8193 -- two batches per thread; with 8 a third batch leaves one thread
  // waiting out a load latency alone before the barrier (config 4: forward 630 -> 603 us, inverse
  // 1838 -> 1792 us)
  constexpr int B = 9;
  // only indices 0 .. N - 1 = M/2 are written when the HALF first FFT pair runs (M >= 64); the
  // smaller transforms read every index, so the tail is zero-filled for them
  const int nw = G.logM4 >= 3 ? N : M;
  if (kind == 3) {   // forward: z_n = (v_a[n] + i v_b[n]) conj(c_n), v = Makhoul permutation of q
    for (int n0 = tid; n0 < nw; n0 += B * nth) {
      float a[B], b[B];
      float2 c[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int n = n0 + r * nth;
        const int x = n < N ? (n < h ? 2 * n : 2 * (N - 1 - n) + 1) - jb.tx0 : -1;
        const bool ok = x >= 0 && x < jb.ulen;
        a[r] = ok ? __ldg(ia + x) : 0.f;
        b[r] = ok && ib ? __ldg(ib + x) : 0.f;
        c[r] = n < N ? __ldg(cc + n) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int n = n0 + r * nth;
        if (n < nw) zsm[pz(n)] = make_float2(a[r] * c[r].x + b[r] * c[r].y, b[r] * c[r].x - a[r] * c[r].y);
      }
    }
  } else {           // inverse: u_k = conj(V_a + i V_b)_k conj(c_k)
    for (int k0 = tid; k0 < nw; k0 += B * nth) {
      float p[B], q[B], r_[B], s[B];
      float2 e[B], c[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int k = k0 + r * nth;
        const bool in = k < N, nz = in && k > 0;
        const int km = nz ? N - k : 0;   // N - k in [1, N - 1] (index N reads as 0)
        e[r] = in ? __ldg(ee + k) : make_float2(0.f, 0.f);
        c[r] = in ? __ldg(cc + k) : make_float2(0.f, 0.f);
        if (kind != 5) {   // V_a = e (a''_k - i a''_{N-k}), V_b likewise; kind 6: a = Phi_x xs
          p[r] = in ? __ldg(ia + k) : 0.f;
          q[r] = nz ? __ldg(ia + km) : 0.f;
          r_[r] = in && ib ? __ldg(ib + k) : 0.f;
          s[r] = nz && ib ? __ldg(ib + km) : 0.f;
          if (kind == 6) {
            const float xk = in ? __ldg(jb.xs + k) : 0.f, xm = nz ? __ldg(jb.xs + km) : 0.f;
            p[r] *= xk;
            r_[r] *= xk;
            q[r] *= xm;
            s[r] *= xm;
          }
        } else {           // b_k, b_{N-k} and e_{N-k} of one Phi_x row (cos / sin of delta)
          p[r] = in ? __ldg(ia + k) : 0.f;
          q[r] = nz ? __ldg(ia + km) : 0.f;
          const float2 em = nz ? __ldg(ee + km) : make_float2(0.f, 0.f);
          r_[r] = em.x;
          s[r] = em.y;
        }
      }
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int k = k0 + r * nth;
        if (k >= nw) break;
        float pp, qq, rr, ss;
        if (kind != 5) {
          pp = k == 0 ? 2.f * p[r] : p[r];   // a''_0 = 2 a_0
          qq = q[r];
          rr = k == 0 ? 2.f * r_[r] : r_[r];
          ss = s[r];
        } else {   // c_k = b_{N-k} cos(delta_{N-k}), c_{N-k} = b_k cos(delta_k), d_k, d_{N-k}
          pp = q[r] * r_[r];
          qq = k ? p[r] * e[r].x : 0.f;
          rr = p[r] * e[r].y;
          ss = q[r] * s[r];
        }
        const float2 ek = e[r];
        const float2 va = make_float2(ek.x * pp + ek.y * qq, ek.y * pp - ek.x * qq);
        const float2 vb = make_float2(ek.x * rr + ek.y * ss, ek.y * rr - ek.x * ss);
        const float2 w = make_float2(va.x - vb.y, va.y + vb.x);   // W = V_a + i V_b
        zsm[pz(k)] = make_float2(w.x * c[r].x - w.y * c[r].y, -(w.x * c[r].y + w.y * c[r].x));
      }
    }
  }
  __syncthreads();
  const CztIo io{nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, 0, false, false, true};
#if TVS_CZT_L2PF
  if (tid < 4 && G.ahead > 0) {
    if (tid < 2) {   // this item's omega0 rows (output phase)
      if (jb.add && (tid == 0 || two)) l2_prefetch(jb.add + (size_t)(r0 + tid) * jb.ldadd, jb.vlen);
    } else {         // the input rows of the item one wave ahead
      const long long ln = (long long)blockIdx.y * gridDim.x + blockIdx.x + G.ahead;
      if (ln < (long long)gridDim.x * gridDim.y) {
        const CztJob &jn = jobs[ln / gridDim.x];
        const int bxn = (int)(ln % gridDim.x), kn = KSET == 1 ? 3 : jn.kind;
        const int rn = (kn == 5 ? bxn : 2 * bxn) + (tid - 2);
        if ((tid == 2 || kn != 5) && rn < jn.rows)
          l2_prefetch(jn.in + (size_t)rn * jn.ldin, kn == 3 ? jn.ulen : N);
      }
    }
  }
#endif
  czt_fft_pair(zsm, G.logM4, twd, gtab, io);
  float *__restrict__ oa = jb.out + (size_t)r0 * jb.ldout;
  float *__restrict__ ob = two ? oa + jb.ldout : nullptr;
  // inverse jobs of the inner loop: out = grad phi + omega0 (added here, see CztJob::add)
  const float *__restrict__ aa = jb.add ? jb.add + (size_t)r0 * jb.ldadd : nullptr;
  const float *__restrict__ ab = (jb.add && two) ? aa + jb.ldadd : nullptr;
  if (kind == 3) {   // Qhat_a[k] = Re(conj(e_k) A_k), Qhat_b[k] = Re(conj(e_k) B_k)
    for (int k0 = tid; k0 < jb.vlen; k0 += B * nth) {
      float2 ck[B], cm[B], e[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int k = min(k0 + r * nth, jb.vlen - 1);
        ck[r] = __ldg(cc + k);   // c_{N-k} = (-1)^N c_k = -c_k (N = M/2 + 1 odd), c_0 for k = 0
        e[r] = __ldg(ee + k);
        cm[r] = k ? make_float2(-ck[r].x, -ck[r].y) : ck[r];
      }
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int k = k0 + r * nth;
        if (k >= jb.vlen) break;
        const int m = k ? N - k : 0;
        const float2 zk = cmulc(zsm[pz(k)], ck[r]), zm = cmulc(zsm[pz(m)], cm[r]);
        // A = (zk + conj zm)/2, B = (zk - conj zm)/(2i); Re(conj(e) A) = e.x A.x + e.y A.y
        const float ax = 0.5f * (zk.x + zm.x), ay = 0.5f * (zk.y - zm.y);
        const float bx = 0.5f * (zk.y + zm.y), by = -0.5f * (zk.x - zm.x);
        oa[k] = e[r].x * ax + e[r].y * ay;
        if (ob) ob[k] = e[r].x * bx + e[r].y * by;
      }
    }
  } else if (kind == 6) {   // phi(x) = conj(conj(c_n) z_n) / 2; out = phi(x + 1) - phi(x)
    // the lanes hold consecutive columns: phi(x + 1) comes from the next lane (lane 31 forms it)
    const int lane = tid & 31;
    auto col_n = [&](int x) { return (x & 1) ? N - 1 - (x >> 1) : (x >> 1); };
    for (int i0 = tid - lane; i0 < jb.vlen; i0 += B * nth) {   // warp-uniform trip count
      float2 cn[B], cn1[B];
      float av[B], bv[B];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int i = i0 + lane + r * nth, x = jb.tx0 + i;
        const bool ok = i < jb.vlen;
        cn[r] = x < N ? __ldg(cc + col_n(x)) : make_float2(0.f, 0.f);
        cn1[r] = (lane == 31 && x + 1 < N) ? __ldg(cc + col_n(x + 1)) : make_float2(0.f, 0.f);
        av[r] = ok && aa ? __ldg(aa + i) : 0.f;
        bv[r] = ok && ab ? __ldg(ab + i) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int i = i0 + lane + r * nth, x = jb.tx0 + i;
        const float2 y = x < N ? cmulc(zsm[pz(col_n(x))], cn[r]) : make_float2(0.f, 0.f);
        float fa = 0.5f * y.x, fb = -0.5f * y.y;   // phi_a(x), phi_b(x)
        float na = __shfl_down_sync(0xffffffffu, fa, 1), nb = __shfl_down_sync(0xffffffffu, fb, 1);
        if (lane == 31) {
          const float2 y1 = x + 1 < N ? cmulc(zsm[pz(col_n(x + 1))], cn1[r]) : make_float2(0.f, 0.f);
          na = 0.5f * y1.x;
          nb = -0.5f * y1.y;
        }
        if (i >= jb.vlen) continue;
        // D+_x phi = 0 on the last column (sin(pi j) = 0 in the spectral form)
        const float da = x < N - 1 ? na - fa : 0.f, db = x < N - 1 ? nb - fb : 0.f;
        oa[i] = aa ? da + av[r] : da;
        if (ob) ob[i] = ab ? db + bv[r] : db;
      }
    }
  } else {           // v = conj(conj(c_n) z_n) / 2 at the Makhoul position of column x
    for (int i0 = tid; i0 < jb.vlen; i0 += B * nth) {
      float2 cn[B];
      float av[B], bv[B];   // omega0 of the inner loop's jobs, loaded with the chirp values
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int ic = min(i0 + r * nth, jb.vlen - 1), x = jb.tx0 + ic;
        cn[r] = __ldg(cc + ((x & 1) ? N - 1 - (x >> 1) : (x >> 1)));
        av[r] = aa ? __ldg(aa + ic) : 0.f;
        bv[r] = ab ? __ldg(ab + ic) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < B; ++r) {
        const int i = i0 + r * nth;
        if (i >= jb.vlen) break;
        const int x = jb.tx0 + i;
        const int n = (x & 1) ? N - 1 - (x >> 1) : (x >> 1);
        const float2 y = cmulc(zsm[pz(n)], cn[r]);   // Y_n; v = conj(Y) / 2
        // (no "+ 0" when there is nothing to add: the plain outputs keep their signed zeros)
        if (kind == 4) {
          oa[i] = aa ? 0.5f * y.x + av[r] : 0.5f * y.x;
          if (ob) ob[i] = ab ? -0.5f * y.y + bv[r] : -0.5f * y.y;
        } else {
          const float v = 0.5f * ((x & 1) ? -y.x : y.x) - 0.5f * y.y;
          oa[i] = aa ? v + av[r] : v;
        }
      }
    }
  }
}

// One CTA per (row, job, output pass).  kind 0: forward cos (pre u^2, post v^2 + v(2tx0+1), Re);
// kind 1: inverse cos (pre u^2 + u(2tx0+1), post v^2, Re); kind 2: inverse sin (pre u^2 +
// u(2tx0+2), post v^2, Im).
// KSET (compile time): 0 general form, 1 Makhoul forward, 2 Makhoul inverse -- separate
// instantiations, so the forward's register allocation does not carry the inverse's paths.
template <int KSET>
__global__ void __launch_bounds__(CZT_THREADS)
k_czt(const CztJob *__restrict__ jobs, CztGeom G, const float2 *__restrict__ gtab,
      const float2 *__restrict__ tw) {
  extern __shared__ float2 zsm[];
  const int MP = G.M + (G.M >> 4);                     // padded FFT buffer
  float2 *tfine = zsm + MP, *tcoarse = tfine + 256;      // twiddle tables
  float *acc = reinterpret_cast<float *>(tcoarse + (G.M >> 8) + 1);
  const CztJob jb = jobs[blockIdx.y];
  if (G.mk) {
    if constexpr (KSET != 0) czt_makhoul<KSET>(jb, jobs, G, gtab, tw, zsm, MP);
    return;
  }
  const int row = blockIdx.x;
  if (row >= jb.rows) return;
  const int v0 = blockIdx.z * G.Vp;
  if (v0 >= jb.vlen) return;
  const int vcnt = min(G.Vp, jb.vlen - v0);
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int i = tid; i < vcnt; i += nth) acc[i] = 0.f;
  for (int i = tid; i < 256; i += nth) tfine[i] = i < G.M ? __ldg(tw + i) : make_float2(1.f, 0.f);
  for (int i = tid; i <= (G.M >> 8); i += nth) tcoarse[i] = (i << 8) < G.M ? __ldg(tw + (i << 8)) : make_float2(1.f, 0.f);
  const Tw twd{tfine, tcoarse, tw};
  const float *__restrict__ in = jb.in + (size_t)row * jb.ldin;
  const int nuc = (jb.ulen + G.Uc - 1) / G.Uc;
  float *__restrict__ out = jb.out + (size_t)row * jb.ldout + v0;
  const float *__restrict__ addr = jb.add ? jb.add + (size_t)row * jb.ldadd + v0 : nullptr;
  // pruned first / last passes for narrow inputs / outputs (tiles of a wide layout)
  const bool pin = G.prune && G.logM4 >= 3 && jb.ulen <= (G.M >> 4);
  const bool pout = G.prune && G.logM4 >= 3 && nuc == 1 && vcnt <= (G.M >> 4);
  for (int uc = 0; uc < nuc; ++uc) {
    const int u0 = uc * G.Uc, ucnt = min(G.Uc, jb.ulen - u0);
    // input row chunk times the pre-chirp: the row values and chirps of eight elements are in
    // flight per thread before any use
    for (int i0 = tid; i0 < (pin ? 0 : G.M); i0 += 8 * nth) {
      float xv[8];
      float2 cv[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r * nth;
        xv[r] = i < ucnt ? __ldg(in + u0 + i) : 0.f;
        cv[r] = i < ucnt ? __ldg(jb.pre + u0 + i) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r * nth;
        if (i >= G.M) break;
        zsm[pz(i)] = make_float2(xv[r] * cv[r].x, xv[r] * cv[r].y);
      }
    }
    __syncthreads();
    const CztIo io{in + u0, jb.pre + u0, ucnt, out, addr, jb.post + v0, vcnt, jb.kind, pin, pout};
    czt_fft_pair(zsm, G.logM4, twd, gtab + (size_t)(blockIdx.z * G.nuc + uc) * G.M, io);
    for (int i0 = tid; i0 < (pout ? 0 : vcnt); i0 += 4 * nth) {
      float2 pv[4];
      float av[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = i0 + r * nth;
        pv[r] = i < vcnt ? __ldg(jb.post + v0 + i) : make_float2(0.f, 0.f);
        av[r] = (addr && nuc == 1 && i < vcnt) ? __ldg(addr + i) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = i0 + r * nth;
        if (i >= vcnt) break;
        const float2 c = cmul(pv[r], zsm[pz(i)]);
        const float val = jb.kind == 2 ? c.y : c.x;
        if (nuc == 1) out[i] = addr ? val + av[r] : val;   // one input chunk: straight out
        else acc[i] += val;
      }
    }
    __syncthreads();
  }
  if (nuc > 1)
    for (int i = tid; i < vcnt; i += nth) out[i] = addr ? acc[i] + addr[i] : acc[i];
}

// ------------------------------------------------------------------------------------ host side

namespace {
void fft64(std::vector<std::complex<double>> &a) {   // iterative radix-2, e^{-2 pi i / n}
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = -2.0 * M_PI / (double)len;
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < len / 2; ++k) {
        const std::complex<double> w(std::cos(ang * k), std::sin(ang * k));
        const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}
int digitrev4(int n, int logM4) {
  int r = 0;
  for (int d = 0; d < logM4; ++d) {
    r = r * 4 + (n & 3);
    n >>= 2;
  }
  return r;
}
}  // namespace

// Geometry for inputs of length <= ulen_max and outputs of length <= vlen_max on an axis of N.
bool czt_geometry(int N, int ulen_max, int vlen_max, int max_m, CztGeom *g) {
  g->N = N;
  auto pow4 = [](long long x) {
    long long m = 4;
    while (m < x) m <<= 2;
    return m;
  };
  const long long trick = 2LL * N - 2;
  if (ulen_max == N && vlen_max == N && trick <= max_m && pow4(trick) == trick) {
    g->M = (int)trick;
    g->Uc = g->Vp = N;
  } else {
    long long m = pow4((long long)ulen_max + vlen_max - 1);
    if (m <= max_m) {
      g->M = (int)m;
      g->Uc = ulen_max;
      g->Vp = (int)(m - ulen_max + 1);
    } else {
      g->M = max_m;
      if (ulen_max <= max_m / 4) {          // narrow input (forward of a tile): output passes
        g->Uc = ulen_max;
        g->Vp = max_m - ulen_max + 1;
      } else if (vlen_max <= max_m / 4) {   // narrow output (inverse to a tile): input chunks
        g->Vp = vlen_max;
        g->Uc = max_m - vlen_max + 1;
      } else {
        g->Uc = max_m / 2;
        g->Vp = max_m / 2;
      }
    }
  }
  g->logM4 = 0;
  while ((1 << (2 * g->logM4)) < g->M) ++g->logM4;
  g->nuc = (ulen_max + g->Uc - 1) / g->Uc;
  g->nvp = (vlen_max + g->Vp - 1) / g->Vp;
  return (1 << (2 * g->logM4)) == g->M && g->logM4 >= 1 && g->logM4 <= 7;   // k_czt instantiates M = 4 .. 16384
}

bool czt_makhoul_geometry(int N, int max_m, CztGeom *g) {
  const long long M = 2LL * N - 2;
  long long p4 = 4;
  int lg = 1;
  while (p4 < M) {
    p4 <<= 2;
    ++lg;
  }
  if (N < 3 || p4 != M || M > max_m || lg < 2 || lg > 7) return false;   // g untouched
  g->N = N;
  g->M = (int)M;
  g->Uc = g->Vp = N;
  g->nuc = g->nvp = 1;
  g->logM4 = lg;
  g->mk = 1;
  g->prune = 0;
  return true;
}

void czt_makhoul_tables(int N, std::vector<float2> &ctab, std::vector<float2> &etab,
                        std::vector<float> &xtab) {
  ctab.resize(N);
  etab.resize(N);
  xtab.assign(N, 0.f);   // kind 6: xs_k = -1 / (2 sin(pi k/(2N))), xs_0 = 0
  for (int k = 1; k < N; ++k) xtab[k] = (float)(-0.5 / std::sin(M_PI * (double)k / (2.0 * N)));
  const long long n2 = 2LL * N;
  for (long long n = 0; n < N; ++n) {
    const long long r = (n * n) % n2;   // e^{i pi n^2 / N}: n^2 mod 2N exactly
    const double a = M_PI * (double)r / (double)N;
    ctab[n] = make_float2((float)std::cos(a), (float)std::sin(a));
    const double d = M_PI * (double)n / (2.0 * N);
    etab[n] = make_float2((float)std::cos(d), (float)std::sin(d));
  }
}

// Kernel tables: for output pass p and input chunk c the digit-reversed FFT of the circular window
// g[n] = h[(p Vp - c Uc) + n], n in [-(M - Vp), Vp - 1], scaled by 1/M (fp64 on the host).
// Chirp tables of the jobs: pre-chirp offset c = 0 (forward) or 2 tx0 + kind (inverse cos / sin),
// post-chirp offset 2 tx0 + 1 (forward) or 0 (inverse); phases m = v^2 + c v reduced exactly mod 4N
// in integers, angles in fp64, one rounding to fp32.  Tables shared by equal (c, length).
std::vector<float2> czt_chirp_tables(int N, std::vector<CztJob> &jobs, std::vector<size_t> &pre_off,
                                     std::vector<size_t> &post_off) {
  std::map<std::pair<long long, int>, size_t> at;
  std::vector<float2> tab;
  const long long n4 = 4LL * N;
  auto get = [&](long long c, int len) {
    const auto key = std::make_pair(c, len);
    const auto it = at.find(key);
    if (it != at.end()) return it->second;
    const size_t off = tab.size();
    at[key] = off;
    for (long long v = 0; v < len; ++v) {
      long long m = (v * v + c * v) % n4;
      if (m < 0) m += n4;
      const double ang = M_PI * (double)m / (2.0 * (double)N);
      tab.push_back(make_float2((float)std::cos(ang), (float)std::sin(ang)));
    }
    return off;
  };
  pre_off.assign(jobs.size(), 0);
  post_off.assign(jobs.size(), 0);
  for (size_t i = 0; i < jobs.size(); ++i) {
    const CztJob &j = jobs[i];
    const long long cpre = j.kind == 0 ? 0 : 2LL * j.tx0 + j.kind;
    const long long cpost = j.kind == 0 ? 2LL * j.tx0 + 1 : 0;
    pre_off[i] = get(cpre, j.ulen);
    post_off[i] = get(cpost, j.vlen);
  }
  return tab;
}

void czt_tables(const CztGeom &g, std::vector<float2> &gtab, std::vector<float2> &tw) {
  const int M = g.M;
  gtab.assign((size_t)g.nvp * g.nuc * M, make_float2(0.f, 0.f));
  const long long n4 = 4LL * g.N;
  std::vector<std::complex<double>> a(M);
  for (int p = 0; p < g.nvp; ++p)
    for (int c = 0; c < g.nuc; ++c) {
      const long long d = (long long)p * g.Vp - (long long)c * g.Uc;
      for (int i = 0; i < M; ++i) {
        const long long n = i < g.Vp ? i : (long long)i - M;
        const long long m = d + n;
        if (g.mk) {   // Makhoul form: h_m = c_m = e^{i pi m^2 / N}, m^2 mod 2N exactly
          const long long n2 = 2LL * g.N;
          const long long r = ((m % n2) * (m % n2)) % n2;
          const double ph = M_PI * (double)r / (double)g.N;
          a[i] = std::complex<double>(std::cos(ph), std::sin(ph));
          continue;
        }
        long long r = ((m % n4) * (m % n4)) % n4;   // m^2 mod 4N exactly
        if (r < 0) r += n4;
        const double ph = -M_PI * (double)r / (2.0 * g.N);
        a[i] = std::complex<double>(std::cos(ph), std::sin(ph));
      }
      fft64(a);
      float2 *dst = gtab.data() + (size_t)(p * g.nuc + c) * M;
      for (int k = 0; k < M; ++k) {
        const std::complex<double> v = a[k] / (double)M;
        dst[digitrev4(k, g.logM4)] = make_float2((float)v.real(), (float)v.imag());
      }
    }
  tw.resize((size_t)M);
  for (int n = 0; n < M; ++n) {
    const double ph = -2.0 * M_PI * (double)n / (double)M;
    tw[n] = make_float2((float)std::cos(ph), (float)std::sin(ph));
  }
}

cudaError_t launch_czt(const CztJob *jobs, int njobs, int max_rows, const CztGeom &g,
                       const float2 *gtab, const float2 *tw, cudaStream_t s, bool fwd) {
  const size_t smem = (size_t)(g.M + (g.M >> 4) + 256 + (g.M >> 8) + 1) * sizeof(float2) +
                      (size_t)g.Vp * sizeof(float);
  const void *fn = !g.mk ? (const void *)k_czt<0> : fwd ? (const void *)k_czt<1> : (const void *)k_czt<2>;
  if (smem > 48 * 1024) {
    cudaError_t e = smem_optin(fn, smem);
    if (e != cudaSuccess) return e;
  }
  if (max_rows <= 0 || njobs <= 0) return cudaSuccess;
  CztGeom gg = g;
  gg.prune = g.mk ? 0 : 1;
  gg.ahead = sm_count();   // one CTA per SM: the next wave starts ~one SM count later
  const dim3 grid(max_rows, njobs, g.nvp);
  if (!g.mk) k_czt<0><<<grid, CZT_THREADS, smem, s>>>(jobs, gg, gtab, tw);
  else if (fwd) k_czt<1><<<grid, CZT_THREADS, smem, s>>>(jobs, gg, gtab, tw);
  else k_czt<2><<<grid, CZT_THREADS, smem, s>>>(jobs, gg, gtab, tw);
  return cudaGetLastError();
}

}  // namespace tvs
