// Internal declarations shared by the kernels (tvs_kernels.cu) and the host driver (tvs_api.cu).
// Nothing here is part of the ABI (see include/tvstokes.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace tvs {

// Dynamic shared-memory opt-in of kernel `func` for `bytes` on the CURRENT device.  The attribute
// belongs to a device context, so the (device, func) pairs already opted in are kept in a
// mutex-guarded table: thread-safe, and a context on a second device opts in again.
cudaError_t smem_optin(const void *func, size_t bytes);
// Multiprocessor count of the current device (cached per device).
int sm_count();
// Kernels a launcher started beyond its first (launchers that start several add k - 1 here; the
// host driver resets it before and reads it after every launcher call to count launches exactly).
extern thread_local int g_extra_launches;

// One overlapping subdomain Gamma_m of the step grid (Omega~ for step 1, Omega for step 2).
// S = [y0, y1] x [x0, x1]; S+ = [y0, py1] x [x0, px1] (one more row/col, clipped, reading A12);
// T = [y0, ty1] x [x0, tx1] (S+ plus one more row/col, clipped: support of div E_{S+}).
struct SubDesc {
  int y0, y1, x0, x1;
  int py1, px1;
  int ty1, tx1;
  int iy, ix;   // subdomain indices (m2, m1)
};

// One tile of the batched projection phi = R_T Delta^dagger E_T q, grad phi on [ty0..py1]x[tx0..px1].
struct ProjTile {
  int ty0, ty1, tx0, tx1;
  int py1, px1;
  int chain;    // index of the precomputed Thomas pivots (distinct row range [ty0, ty1])
  int po;       // first output row relative to ty0 (output rows [ty0 + po, py1], stored from 0)
};

// Batched fp32 GEMM descriptor: C[M x N] = A[M x K] * B[K x N], all row-major.
struct GemmDesc {
  const float *A;
  const float *B;
  float *C;
  int M, N, K;
  int lda, ldb, ldc;
};

// Pre-split (3xTF32) GEMM descriptor: C = (A_hi + A_lo) (B_hi + B_lo)^T, all K-contiguous,
// every row start 16-byte aligned; hi planes hold values exactly representable in tf32.
struct GemmDesc2 {
  const float *Ahi, *Alo, *Bhi, *Blo;
  float *C;
  int M, N, K;
  int lda, ldb, ldc;
};

// TMA form of a pre-split GEMM: one 2D tensor map per operand plane (fp32 elements, 128-byte
// swizzle, box {32, rows}, out-of-bounds elements read as zero).  Lives in device memory.
struct alignas(64) TmaGemmDesc {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
  float *C;
  int M, N, K, ldc;
  // > 0: A is stored column-block-major, [K/32][a_blk_rows][32] (k-step kt of rows m0.. is the
  // contiguous box at row kt * a_blk_rows + m0 of a 32-wide map); 0: row-major [M][lda]
  int a_blk_rows = 0;
  // > 0: C is stored column-block-major, element (row, col) at
  // C + (col / c_blk) * c_plane + row * c_blk + col % c_blk (ldc unused); 0: row-major, pitch ldc
  int c_blk = 0;
  long long c_plane = 0;
};
// Tensor maps of the y-solve's staged column blocks (Q-hat fp32 and pivots fp64), boxes of
// {32 columns, box_rows rows}, nbox boxes per CTA.
struct alignas(64) SolveMaps {
  CUtensorMap q, r;
  int box_rows, nbox;
  // > 0: Q-hat is column-block-major ([J-column block][q_blk_rows rows][J]); the map is J wide
  int q_blk_rows = 0;
};
cudaError_t encode_plain_2d(CUtensorMap *map, const void *base, bool fp64, int cols, int rows,
                            int ld_elems, int box_cols, int box_rows);
// host: encode the four tensor maps of d for a tile of width bn
cudaError_t make_tma_desc(TmaGemmDesc *out, const GemmDesc2 &d, int bn);

// Chirp-z evaluation of the partial x-DCTs (tvs_czt.cu).  One job = `rows` rows of one tile:
// out[row][v] = Op(post[v] sum_u in[row][u] pre[u] h[v-u]) for u < ulen, v < vlen (see the file
// header); kind 0 forward cos, 1 inverse cos, 2 inverse sin; tx0 = first global column of the tile.
struct CztJob {
  const float *in;
  float *out;
  int rows, ldin, ldout;
  int tx0, ulen, vlen, kind;
  // chirp tables (fp64-accurate, rounded once): pre[u] = e^{i theta (u^2 + cpre u)} for
  // u in [0, ulen), post[v] = e^{i theta (v^2 + cpost v)} for v in [0, vlen)
  const float2 *pre = nullptr, *post = nullptr;
  // nullable: out = transform + add (rows of ldadd floats) -- the inner loop's inverse jobs write
  // grad phi + omega0 so kernel (a') reads one field instead of two (bitwise the same sum)
  const float *add = nullptr;
  int ldadd = 0;
  // kind 6 (Makhoul inverse x): per-frequency scale Phi_x -> the cosine coefficients of phi
  const float *xs = nullptr;
};
// host: fill the chirp tables of every job (deduplicated by (c, length)); returns the table
std::vector<float2> czt_chirp_tables(int N, std::vector<CztJob> &jobs, std::vector<size_t> &pre_off,
                                     std::vector<size_t> &post_off);
struct CztGeom {
  int N;          // axis length (theta = pi / (2N))
  int M, logM4;   // FFT size (power of 4) and log4 M
  int Uc, Vp;     // input chunk and output pass lengths (Uc + Vp - 1 <= M, or the M = 2N-2 case)
  int nuc, nvp;   // numbers of chunks / passes for the largest job
  int prune = 1;  // pruned first / last FFT passes for narrow jobs (general form)
  int mk = 0;     // 1: Makhoul form -- the partial x-DCTs as DFT_N's of packed real sequences by
                  // Bluestein with M = 2N - 2 (job kinds 3, 4, 6; see tvs_czt.cu)
  int ahead = 0;  // Makhoul form: L2 prefetch of the item this many CTAs ahead (set by launch_czt)
};
bool czt_geometry(int N, int ulen_max, int vlen_max, int max_m, CztGeom *g);
// Makhoul form on an axis of N (any tile): M = 2N - 2 must be a power of 4 <= max_m.
bool czt_makhoul_geometry(int N, int max_m, CztGeom *g);
// its per-axis tables: c[n] = e^{i pi n^2 / N} and e[k] = e^{i pi k / (2N)}, n, k < N
// and xs[k] = -1 / (2 sin(pi k/(2N))) (xs[0] = 0), the kind-6 scale
void czt_makhoul_tables(int N, std::vector<float2> &ctab, std::vector<float2> &etab,
                        std::vector<float> &xtab);
void czt_tables(const CztGeom &g, std::vector<float2> &gtab, std::vector<float2> &tw);
cudaError_t launch_czt(const CztJob *jobs, int njobs, int max_rows, const CztGeom &g,
                       const float2 *gtab, const float2 *tw, cudaStream_t s, bool fwd);   // fwd: Makhoul forward jobs (kind 3)

// Uniform per-subdomain buffer geometry (every subdomain uses the max dims, row pitch `ld`).
struct Geo {
  int M;          // number of subdomains in the batch (grid z of the launches)
  int MG;         // plane stride of the grad-phi planes, in subdomains (>= M; the capacity of a
                  // subdomain group, see Plan::sg in tvs_api.cu)
  int A, B;       // rows/cols of S (max)
  int AP, BP;     // rows/cols of S+ (max)
  int AT, BT;     // rows/cols of T (max)
  int ldS, ldP, ldT;  // pitches (floats) of S, S+, T planes
};

// ---------------------------------------------------------------- launchers (tvs_kernels.cu)
// all return cudaGetLastError() of the launch; `s` is the stream.
cudaError_t launch_tau0(const float *d0, int n2, int n1, float *tau, int ldt, cudaStream_t s);
cudaError_t launch_g_row0(const float *tau2, int ldt, int n1, double *g_row0, cudaStream_t s);
cudaError_t launch_irv2_f(const float *tau1, int ldt, const double *g_row0, const float *d0,
                          int n2, int n1, float alpha, float *f, int ldf, double *csum,
                          cudaStream_t s);

cudaError_t launch_omega0_2(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                            const float *f, const float *p1, const float *p2, int ld, int n2,
                            int n1, float *om, cudaStream_t s);
// two inner iterations of kernel (a) in one pass (temporal blocking; bitwise = two launch_sweep2)
cudaError_t launch_sweep2x2(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                            const float *vin, const float *om, float *vout, int n2, int n1,
                            float t, cudaStream_t s);
cudaError_t launch_sweep2(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                          const float *vin, const float *om, float *vout, int n2, int n1, float t,
                          cudaStream_t s);
cudaError_t launch_combine(const SubDesc *subs, Geo g, int planes, const int2 *covy,
                           const int2 *covx, const int *loy, const int *lox, int m2loc, int k0,
                           int k1, const float *q, float *p, int ld, int n2, int row0, int row1,
                           int n1, float ahat, int *bad, const float *up, int up_r0, int up_r1,
                           const float *dn, int dn_r0, int dn_r1, cudaStream_t s);
cudaError_t launch_partial(const SubDesc *subs, Geo g, int planes, const int2 *covy,
                           const int2 *covx, const int *loy, const int *lox, int m2loc, int k0,
                           int k1, const float *q, int ra, int rb, int n1, int ld, float *out,
                           cudaStream_t s);
cudaError_t launch_recover2(const float *d0, const float *p1, const float *p2, int ld, int n2,
                            int n1, float inv_alpha, const float *shift, float *d, int row0,
                            int row1, cudaStream_t s);
// IRV1 data: f = alpha d0 - div xi and div xi (pitch ldf)
cudaError_t launch_irv1_f(const float *tau1, const float *tau2, int ldt, const float *d0, int n2,
                          int n1, float alpha, float eps, float *f, float *dxi, int ldf,
                          cudaStream_t s);

// dual energies (deterministic fp64 reductions; part has >= 592 doubles, out one double)
cudaError_t launch_dual_energy2(const float *p1, const float *p2, const float *f, int ld, int n2,
                                int n1, int row0, int row1, double *part, double *out,
                                cudaStream_t s);
// IRV2 f with the zero-mean g of the oracle (reading A3): f += alpha mean(g)  (part >= 592 doubles)
cudaError_t launch_irv2_zero_mean_g(float *f, int ldf, const float *d0, int n2, int n1,
                                    float alpha, double *part, double *shift, cudaStream_t s);
// Primal-energy / duality-gap raw sums (see k_primal1_partial / k_primal2_partial): part needs
// 3 (step 1) or 4 (step 2) x 592 doubles; out receives 3 or 4 doubles.
cudaError_t launch_primal1(const float *tau, size_t plane, int ld, const float *f, const float *p,
                           int n2, int n1, int row0, int row1, float delta, float scale,
                           double *part, double *out, cudaStream_t s);
cudaError_t launch_primal2(const float *d, const float *d0, const float *f, const float *dxi,
                           const float *p1, const float *p2, int ldf, int n2, int n1, int row0,
                           int row1, float inv_alpha, double *part, double *out, cudaStream_t s);
cudaError_t launch_sum_ranks(const double *vals, int world, int stride, int n, double *out,
                             cudaStream_t s);
cudaError_t launch_sumsq2(const float *r, size_t plane, int ld, int n1, int row0, int row1,
                          double *part, double *out, cudaStream_t s);

// step 1
cudaError_t launch_multidiv(const float *p, int ld, int n2, int n1, float *w, int row0, int row1,
                            cudaStream_t s);
cudaError_t launch_div(const float *w1, const float *w2, int ld, int n2, int n1, float *q,
                       float *qlo, int row0, int row1, cudaStream_t s);
cudaError_t launch_axpby2(const float *a, const float *b, const float *c, int ld, int n2, int n1,
                          float sa, float sb, float sc, float *out, int row0, int row1,
                          cudaStream_t s);
cudaError_t launch_load_tp(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                           const float *p, int ld, int n2, int n1, float *v, cudaStream_t s);
cudaError_t launch_prediv1(const SubDesc *subs, Geo g, const float *v, int n2, int n1, float *q,
                           const float *qsub, cudaStream_t s);
cudaError_t launch_omega0_1(const SubDesc *subs, Geo g, const float *r, int ld, const float *v,
                            int n2, int n1, float *om, cudaStream_t s);
cudaError_t launch_sweep1(const SubDesc *subs, Geo g, const float *thy, const float *thx,
                          const float *vin, const float *gphi, int ldg, const float *om,
                          float *vout, int n2, int n1, float t, cudaStream_t s);

// projection (kernel b)
cudaError_t launch_dct_tables(int n, float *cf, float *cn, float *sn, float *snT, float *split6,
                              int ld, cudaStream_t s);
// pivots r_k of every chain, plus the constant-tail compression (pcut, pinf, plast: [chain][ldn])
cudaError_t launch_pivots(const ProjTile *chains_tiles, const int *chain_first_tile, int nchains,
                          int n2, int n1, double *rinv, int ldn, int AT, int *pcut, double *pinf,
                          double *plast, cudaStream_t s);
cudaError_t launch_gemm(const GemmDesc *descs, int batch, int maxM, int maxN, cudaStream_t s);
// tcgen05 3xTF32 GEMM: C = A * Bt^T, Bt given as [N][K] row-major (tvs_gemm_tc.cu)
cudaError_t launch_gemm_tc(const GemmDesc *descs, int batch, int maxM, int maxN, int bn,
                           bool b_aligned, cudaStream_t s);
cudaError_t launch_gemm_tc2(const GemmDesc2 *descs, int batch, int maxM, int maxN, int bn,
                            cudaStream_t s);
// persistent warp-specialised form: A given as ONE fp32 plane (a_hi map), split in shared memory
cudaError_t launch_gemm_tma_p(const TmaGemmDesc *descs, int batch, int maxM, int maxN, int bn,
                              cudaStream_t s);
// TS form: A split into tensor memory (tcgen05.st), MMA with [a-tmem]; same descriptors as _p
cudaError_t launch_gemm_tma_ts(const TmaGemmDesc *descs, int batch, int maxM, int maxN, int bn,
                               cudaStream_t s);
// CTA-pair TS form (cta_group::2, 256 x 144 tiles); descriptors whose B maps have 72-row boxes
cudaError_t launch_gemm_tma_ts2(const TmaGemmDesc *descs, int batch, int maxM, int maxN,
                                cudaStream_t s);
cudaError_t launch_gemm_tma(const TmaGemmDesc *descs, int batch, int maxM, int maxN, int bn,
                            cudaStream_t s);
// segmented y-solve, shared-memory form (default when solve4_fits(AT)); segprod from
// launch_segprod ([chain][2][solve_nseg(AT)][ldn] doubles), outputs plain fp32
int solve_nseg(int AT);
bool solve4_fits(int AT);
int solve4_width(int AT);   // column block width of k_proj_solve4 (16 or 32)
cudaError_t launch_segprod(const ProjTile *tiles, const int *first, int nchains, const double *rinv,
                           int ldn, int AT, int n1, double *segprod, cudaStream_t s);
cudaError_t launch_proj_solve4(const ProjTile *tiles, int ntiles, int n2, int n1,
                               const float *qhat, int AT, int ldn, const double *rinv,
                               const double *segprod, float *phx, float *phy, int AP,
                               const SolveMaps *maps, int smem_rows, const int *order,
                               int nchains, int per_chain, cudaStream_t s);
// chain-shared y-solve (one pivot block per CTA for the tiles of a layout row); needs the TMA maps
// global y-solve in fixed segments (see k_gsolve_* in tvs_kernels.cu): phase 0 writes the forward
// aggregates of segments [s0, s1) into aggb_or_out; phase 1 reads the all-gathered forward
// aggregates `agg`, writes z and the backward aggregates into aggb_or_out; phase 2 reads both
// (agg forward, aggb_or_out backward) and writes the spectral gradient planes of the owned rows
cudaError_t launch_gsolve(int phase, const int *seglo, int nseg, int s0, int s1, int n1, int n2,
                          const float *qhat, int ldn, const double *rinv, const int *pcut,
                          const double *pinf, const double *plast, int nt, const double *agg,
                          double *aggb_or_out, float *zs, float *phx, float *phy, int po,
                          cudaStream_t s);
// segmented y-solve: fp32 z scratch [tile][AT][ldn]
cudaError_t launch_proj_solve3(const ProjTile *tiles, int ntiles, int n2, int n1,
                               const float *qhat, int AT, int ldn, const double *rinv, float *z,
                               float *phx, float *phy, float *phx_lo, float *phy_lo, int AP,
                               const int *pcut, const double *pinf, const double *plast,
                               cudaStream_t s);

}  // namespace tvs
