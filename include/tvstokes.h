/*
 * tvstokes.h -- C-ABI of the B200-native TV-Stokes overlapping-Schwarz dual iteration
 * (arXiv 2602.17494, "Functional Analysis and Parallel Domain Decomposition for the TV-Stokes
 * Model").  Citations "P:<line>" refer to PAPER.md lines.
 *
 * What the library computes (all on the GPU, hand-written sm_100a kernels):
 *   step 1 (TFS, P:675 Eq. tfsdualdis): the dual of tangent-field smoothing on the extended grid
 *     Omega~ = (n2+1) x (n1+1), solved by the discrete parallel domain decomposition Alg. 2
 *      whose local solves are the localized TFS inner loop Alg. 5 with
 *     the divergence-free projection evaluated in its local form (Eqs. locglobprojpart1 P:1481,
 *     invLaplLowCapLong P:1669).  Output tau = P tau_0 - delta P multidiv p.
 *   step 2 (IRV2, P:679 Eq. ir2dualdis): the ROF-type dual on Omega = n2 x n1 with
 *     g from tau (grad g = tau^perp, backward differences), solved by Alg. 2 with the
 *     inner loop Alg. 3.  Output d = d_0 - div p / alpha, alpha = 1/lambda.
 *   denoise: step 1 then step 2 on the same splitting.
 *
 * Conventions (all entry points):
 *   - Images are row-major float32, row i (y) of n1 pixels, 0-based; h = 1.
 *   - Vector / 2x2 dual fields are stored as contiguous planes: tau = [tau_1 | tau_2] each
 *     (n2+1)*(n1+1); step-1 p = [p_11 | p_12 | p_21 | p_22] (p_k = (p_k1 x-comp, p_k2 y-comp));
 *     step-2 p = [p_1 | p_2] each n2*n1.
 *   - Device-pointer entry points take pointers on the ctx's GPU and enqueue on `cuda_stream`
 *     (a cudaStream_t; NULL = legacy default stream).  They return after enqueueing and a final
 *     stream synchronisation (results are complete on return).
 *   - `_host` entry points take host pointers and do the host<->device copies themselves.
 *   - The caller owns every input/output buffer; the library owns its scratch (cached per
 *     (n2, n1, layout) plan in the ctx, freed by tvs_destroy).
 *   - Fixed schedule: exactly it.sweeps outer sweeps of it.inner local dual updates, no stopping
 *     test (reading A10).  Warm start v^0 = R_S qhat_m of the previous sweep (reading A9).
 *   - Layout and schedule structs are passed by const pointer (never by value: struct-by-value
 *     with mixed int/float members is mis-marshalled by some FFIs, e.g. libffi/ctypes).
 *   - Errors: every call returns a tvs_status; no exception crosses the ABI.  The message of the
 *     last failure is available from tvs_last_error(ctx).
 */
#ifndef TVSTOKES_H
#define TVSTOKES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TVS_OK = 0,
  TVS_EINVAL = 1,   /* bad argument: t not in (0, 1/8], delta <= 0, lambda <= 0, n < 2  */
  TVS_ELAYOUT = 2,  /* a core width <= overlap (reading A17) or m > n                          */
  TVS_ENUMERIC = 4, /* non-finite value in the dual after a sweep                               */
  TVS_ECUDA = 5,    /* CUDA runtime failure (message has the CUDA error string)                 */
  TVS_ENCCL = 6,    /* NCCL failure                                                             */
  TVS_ENOMEM = 7    /* device allocation failed                                                 */
} tvs_status;

/* Overlapping layout: m2 x m1 subdomains of Omega~ (rows x cols), adjacent
 * subdomains share a band of exactly `overlap_*` grid points (reading A6); core cuts at
 * floor(k N~ / M) (reading A8); Omega_m = Omega~_m cap Omega. */
typedef struct {
  int32_t m2, m1;
  int32_t overlap_y, overlap_x;
} tvs_layout;

/* Schedule: `sweeps` outer iterations of Alg. 2, `inner` updates of Alg. 3/5 per sweep,
 * dual step t in (0, 1/8]. */
typedef struct {
  int32_t sweeps, inner;
  float t;
} tvs_iters;

/* Per-call statistics. pixel_updates = sum_m |Gamma_m| * sweeps * inner (overlap pixels counted
 * per subdomain, reading A21); launches = kernels this call launched. */
typedef struct {
  double seconds;           /* device time of the call (CUDA events on cuda_stream)          */
  int64_t pixel_updates;
  int64_t launches;
  double flops_proj;        /* algorithmic fp32 MACs*2 of the projection contractions (step 1) */
  double bytes_sweep;       /* algorithmic HBM bytes of the fused dual-sweep kernels            */
  double dual_energy;       /* D(p) of the returned dual (Eq. opt_dual_discrete),
                               fp64 reduction over the whole grid (all ranks)                   */
  int64_t sweeps_run;       /* outer sweeps performed (< sweeps when a stopping rule fired)     */
  double primal_energy;     /* primal energy of the returned solution, fp64 reduction over the
                               whole grid (all ranks): step 1 E_1 = TV(tau) + ||tau - P tau_0||^2
                               / (2 delta) (Cor. tfsdual; channel-wise TV, reading
                               A15); step 2 E_2 = TV(d - g) + alpha/2 ||d - d_0||^2 (Eq.
                               modifiedStep2), IRV1 E = TV(d) + <d, div xi> + alpha/2
                               ||d - d_0||^2 (Eq. IRPXi)                            */
  double gap;               /* duality gap sum_k sum_px (|grad u_k| + p_k . grad u_k) >= 0 with
                               u = tau (step 1), d - g (IRV2) or d (IRV1): equals E(u(p)) - G(p),
                               G the dual objective; 0 iff p is optimal      */
} tvs_stats;

typedef struct tvs_ctx tvs_ctx;   /* opaque: device, plans, scratch, profiling, communicator */

/* Create a context on CUDA device `device` (argument order of SURVEY 8(b)).  Single process /
 * single GPU: rank = 0, world = 1, nccl_id = NULL.  Multi-GPU (one process per GPU): every rank
 * passes the same 128-byte ncclUniqueId obtained from tvs_nccl_unique_id on rank 0; the context
 * owns its NCCL communicator (band send/recv per sweep, all-gathers, all-reduces).
 * Errors: TVS_EINVAL (ctx NULL, rank/world out of range, world > 1 without an id), TVS_ECUDA
 * (bad device), TVS_ENCCL (communicator init).  *ctx is NULL on failure. */
tvs_status tvs_create(tvs_ctx **ctx, int rank, int world, const uint8_t *nccl_id, int device);
tvs_status tvs_destroy(tvs_ctx *ctx);

/* Virtual slab group on ONE GPU: creates `world` contexts ctxs[0..world-1] on `device`, ranks of a
 * slab decomposition exactly as with one process per GPU, except that their
 * exchanges -- the per-sweep band send/recv, the row all-gathers (partial x-DCT rows, outputs) and
 * the energy all-reduces -- are device-to-device copies on that GPU instead of NCCL calls.  Each
 * context must be driven from its own host thread (SPMD: every rank calls the same entry points
 * with the same arguments) and should get its own CUDA stream; the threads rendezvous inside the
 * calls.  Results are bitwise those of world = 1 (tests/test_gpu_virtual.py).  Purpose: run the
 * multi-GPU data path under a single-GPU test (SURVEY 4 "virtual slab mode").  A rank that fails
 * aborts the group (the others return TVS_ENCCL).  Free each context with tvs_destroy.
 * Errors: TVS_EINVAL (world < 1 or > 64), TVS_ECUDA, TVS_ENOMEM. */
tvs_status tvs_create_virtual_group(tvs_ctx **ctxs, int world, int device);
const char *tvs_last_error(const tvs_ctx *ctx);
tvs_status tvs_nccl_unique_id(uint8_t id_out[128]);

/* Rows [row_begin, row_end) of Omega~ whose final values this rank owns for a given layout
 * (slab of whole subdomain rows).  Pure host computation; valid without a GPU. */
tvs_status tvs_owned_rows(int32_t n2, int32_t n1, const tvs_layout *L, int rank, int world,
                          int32_t *row_begin, int32_t *row_end);

/* Slab decomposition of the step grid for `rank` of `world` (host only, no GPU; step 1 = Omega~,
 * step 2 = Omega).  out = {k0, k1, R0, R1, E0, E1, V0, V1, us0, us1, ur0, ur1, ds0, ds1, dr0, dr1}:
 * layout rows [k0,k1) of this rank, core (output) rows [R0,R1), rows covered by its subdomains
 * [E0,E1), rows where it keeps p valid [V0,V1) = E +- 1, and the band rows whose partial sums it
 * sends to / receives from rank-1 (us/ur) and rank+1 (ds/dr) every sweep.
 * TVS_ELAYOUT if the layout cannot be split over `world` ranks (m2 < world, overlap < 2, ...). */
tvs_status tvs_dist_rows(int32_t n2, int32_t n1, const tvs_layout *L, int32_t step, int rank,
                         int world, int32_t out[16]);

/* Layout query (host only): inclusive ranges of subdomain k along an axis of length n with
 * m subdomains and overlap s (reading A8), and the partition-of-unity weight theta_k(x)
 * (reading A7).  Used by tests to check the ABI agrees with the paper's layout rules. */
tvs_status tvs_layout_range(int32_t n, int32_t m, int32_t s, int32_t k, int32_t *lo, int32_t *hi);
tvs_status tvs_layout_theta(int32_t n, int32_t m, int32_t s, int32_t k, int32_t x, double *theta);

/* Outer-loop stopping rule of this context (default 0: fixed schedule, reading A10).
 * criterion 1: |D(p^n)^{1/2} - D(p^{n+1})^{1/2}| < c tol with c = (2|Omega~|)^{1/2} for step 1 and
 *              |Omega|^{1/2} for step 2 (the criteria of section 5.2);
 * criterion 2: |D(p^n)^2 - D(p^{n+1})^2| / |Gamma| < tol (section 6.3, printed squares,
 *              reading A19).
 * D is evaluated on the device after every sweep (one fp64 reduction; step 1 reuses the residual
 * r^n = f - P multidiv p^n of the next sweep) and read back by the host, so an active rule adds one
 * stream synchronisation per sweep.  TVS_EINVAL for an unknown criterion or tol < 0. */
tvs_status tvs_set_stopping(tvs_ctx *ctx, int32_t criterion, double tol);

/* Per-sweep energy trace (the energy-convergence protocol of section 6.3 / Fig. 7, P:1769-1782;
 * SURVEY 8(f) NEXT 3).  With cap > 0 every following tv_stokes_step1 / step2 / step2_irv1 call of
 * this context writes, for the Schwarz iterates n = 0 .. sweeps_run (at most cap), the primal energy
 * E(u(p^n)), the dual energy D(p^n) (Eq. opt_dual_discrete) and the duality gap
 * (SURVEY C-15) to out[3 n + {0, 1, 2}] (host memory owned by the caller, valid until the call
 * returns) and the number of entries to *count (nullable).  Step 1: tau^n = delta r^n, r^n the
 * sweep's global residual; step 2: d^n = d0 - div p^n / alpha.  fp64
 * device reductions summed over ranks; one extra reduction pass per sweep (and the step-1 side
 * stream overlap is off while tracing).  cap = 0 turns it off.  TVS_EINVAL for cap < 0 or a null
 * buffer with cap > 0. */
tvs_status tvs_set_trace(tvs_ctx *ctx, double *out, int32_t cap, int32_t *count);

/* Step 1 (TFS).  d0: device [n2*n1]; tau: device out [2][(n2+1)*(n1+1)];
 * p: device out (nullable) [4][(n2+1)*(n1+1)]. */
tvs_status tv_stokes_step1(tvs_ctx *ctx, const float *d0, int32_t n2, int32_t n1, float delta,
                           const tvs_layout *L, const tvs_iters *it, float *tau, float *p, tvs_stats *st,
                           void *cuda_stream);

/* Step 2 (IRV2).  tau: device [2][(n2+1)*(n1+1)] (e.g. step 1's output); d0: device [n2*n1];
 * lambda = 1/alpha (reading A4); d: device out [n2*n1]; p: device out (nullable) [2][n2*n1]. */
tvs_status tv_stokes_step2(tvs_ctx *ctx, const float *tau, const float *d0, int32_t n2,
                           int32_t n1, float lambda, const tvs_layout *L, const tvs_iters *it,
                           float *d,
                           float *p, tvs_stats *st, void *cuda_stream);

/* Step 2, variant IRV1 (Eq. ir1dualdis; Cor. irdual P:403-417): same dual iteration with
 * f = alpha d0 - div xi, xi = tau_perp / sqrt(|tau_perp|^2 + epsilon), tau_perp = R_Omega(tau_2,
 * -tau_1) (Eq. defXi2:discrete P:683-686), and d = d0 - (div p + div xi)/alpha.  mu = 1/alpha
 * (P:930); epsilon > 0 (the paper's DD run uses 1e-3).  Arguments, layouts,
 * ownership and errors as tv_stokes_step2 (TVS_EINVAL also for epsilon <= 0). */
tvs_status tv_stokes_step2_irv1(tvs_ctx *ctx, const float *tau, const float *d0, int32_t n2,
                                int32_t n1, float mu, float epsilon, const tvs_layout *L,
                                const tvs_iters *it, float *d, float *p, tvs_stats *st,
                                void *cuda_stream);

/* Step 1 then step 2 on the same splitting.  tau (nullable) receives step 1's field. */
tvs_status tv_stokes_denoise(tvs_ctx *ctx, const float *d0, int32_t n2, int32_t n1, float delta,
                             float lambda, const tvs_layout *L, const tvs_iters *it1,
                             const tvs_iters *it2, float *d,
                             float *tau, tvs_stats *st1, tvs_stats *st2, void *cuda_stream);

/* Host-buffer variant of tv_stokes_denoise: d0, d, tau are host pointers (pinned or pageable);
 * the host->device copy of d0 and the device->host copies of d (and tau) are part of the call. */
tvs_status tv_stokes_denoise_host(tvs_ctx *ctx, const float *d0, int32_t n2, int32_t n1,
                                  float delta, float lambda, const tvs_layout *L,
                                  const tvs_iters *it1, const tvs_iters *it2, float *d, float *tau, tvs_stats *st1,
                                  tvs_stats *st2, void *cuda_stream);

/* Per-kernel profiling with CUDA events on the launching stream.  When enabled, every launch of
 * the library's kernels is bracketed by events; tvs_kernel_times reports, per kernel family,
 * the number of launches and the summed device milliseconds since the last reset.
 * Families: 0 sweep2 (kernel a), 1 sweep1 (kernel a'), 2 prediv, 3 proj_fwd_gemm, 4 proj_solve,
 * 5 proj_inv_gemm, 6 omega0/combine/other stencils, 7 proj_fwd_czt, 8 proj_inv_czt (the chirp-z
 * form of the two partial x-DCTs; flops are the dense-equivalent 2MNK of the contraction). */
#define TVS_NUM_KERNEL_FAMILIES 9
tvs_status tvs_set_profiling(tvs_ctx *ctx, int enable);
tvs_status tvs_kernel_times(tvs_ctx *ctx, int64_t counts[TVS_NUM_KERNEL_FAMILIES],
                            double ms[TVS_NUM_KERNEL_FAMILIES],
                            double bytes[TVS_NUM_KERNEL_FAMILIES],
                            double flops[TVS_NUM_KERNEL_FAMILIES]);
tvs_status tvs_reset_kernel_times(tvs_ctx *ctx);

/* Diagnostics: run the projection GEMM (impl 0 = SIMT fp32, 1 = tcgen05 3xTF32 with 128-wide
 * tiles, 2 = tcgen05 3xTF32 with 144-wide tiles, 3 = tcgen05 3xTF32 on pre-split hi/lo operands
 * with the cp.async pipeline, 4 = the same through TMA tensor maps, 5 = the persistent
 * warp-specialised TMA kernel that splits A in shared memory -- the production path, 6 = the
 * same with A split into tensor memory and read by the MMA from there) on seeded
 * random A[M x K], B[K x N] and return
 * max_ij |C - C_fp64| / sum_k |A_ik B_kj| (host reference).  Test-only; allocates its own memory. */
tvs_status tvs_selftest_gemm(tvs_ctx *ctx, int32_t M, int32_t N, int32_t K, int32_t impl,
                             uint64_t seed, double *max_rel_err);

#ifdef __cplusplus
}
#endif
#endif /* TVSTOKES_H */
