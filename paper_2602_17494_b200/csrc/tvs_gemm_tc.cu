// Batched fp32-accurate GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32), used by
// the projection kernel (b) for the partial x-DCT contractions of Eq. invLaplLowCapLong
// (P:1669-1677).  C[M x N] = A[M x K] * Bt[N x K]^T with A and Bt row-major, K contiguous.
//
// Accuracy: 3xTF32 error compensation.  Each operand x is split as hi = tf32(x) rounded to
// nearest (low 13 mantissa bits zero, so the tensor core reads it exactly) and lo = x - hi
// (exact in fp32);
// C = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in fp32 in TMEM.  The dropped lo*lo term and
// the tf32 rounding of lo are O(2^-21) relative -- fp32-level, which is what the projection needs
// (precision rule C-10: the DCT contractions are fp32, the y-solves fp64).
//
// Structure (one CTA = 128 threads = 4 warps, tile 128 x BN, K step 16, 3-stage smem ring):
//   all threads load the next K slice from global into registers, split hi/lo and store it into
//   shared memory in the canonical K-major SWIZZLE_NONE core-matrix layout (8 rows x 16 B core
//   matrices); fence.proxy.async makes the generic-proxy stores visible to the tensor core;
//   thread 0 issues 2 k-steps x 3 tcgen05.mma (M=128, N=BN, K=8) and tcgen05.commit's them to the
//   stage's mbarrier; a stage is refilled only after its mbarrier phase completes.  The fp32
//   accumulator lives in TMEM (lane = row, column = n); the epilogue reads it with tcgen05.ld.
#include "tvs_internal.h"

#include <stdint.h>

namespace tvs {
namespace tc {

constexpr int BM = 128, BK = 16, STAGES = 3, NT = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset 0, lbo mode 0, layout SWIZZLE_NONE (0) [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  return d;
}

// Instruction descriptor (cute::UMMA::InstrDescriptor): C f32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// byte offset of element (r, k) of an R x 16 K-major block in core-matrix layout
__device__ __forceinline__ uint32_t core_off(int r, int k, int R) {
  return (uint32_t)((((k >> 2) * (R >> 3) + (r >> 3)) << 7) + ((r & 7) << 4) + ((k & 3) << 2));
}

__device__ __forceinline__ void split(float x, float &hi, float &lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));   // round to nearest, low 13 bits zero
  hi = __uint_as_float(h);
  lo = x - hi;                                            // exact in fp32, |lo| <= 2^-12 |x|
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(z), "r"(z), "r"(z), "r"(z)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

template <int BN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;   // A_hi A_lo B_hi B_lo
  static constexpr int TOTAL = STAGES * STAGE + 128;         // + mbarriers + tmem slot
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

template <int BN, bool B_ALIGNED>
__global__ void __launch_bounds__(NT) k_gemm_tc(const GemmDesc *__restrict__ descs) {
  using SM = Smem<BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const GemmDesc d = descs[blockIdx.z];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= d.M || n0 >= d.N) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * SM::STAGE);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + STAGES * SM::STAGE + 64);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(SM::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  // register staging of one K slice: A row `tid`, B rows `tid` (+128)
  constexpr int BROWS = (BN + NT - 1) / NT;
  float ra[BK], rb[BROWS][BK];
  const int nk = (d.K + BK - 1) / BK;

  auto load = [&](int kt) {
    const int k0 = kt * BK;
    const int gm = m0 + tid;
    const bool full_k = (k0 + BK <= d.K);
    if (gm < d.M && full_k) {
      const float4 *p = reinterpret_cast<const float4 *>(d.A + (size_t)gm * d.lda + k0);
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        float4 v = __ldg(p + q);
        ra[4 * q] = v.x; ra[4 * q + 1] = v.y; ra[4 * q + 2] = v.z; ra[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < BK; ++k)
        ra[k] = (gm < d.M && k0 + k < d.K) ? __ldg(d.A + (size_t)gm * d.lda + k0 + k) : 0.f;
    }
#pragma unroll
    for (int rr = 0; rr < BROWS; ++rr) {
      const int r = tid + rr * NT;
      const int gn = n0 + r;
      const bool ok = (r < BN) && (gn < d.N);
      if (B_ALIGNED && ok && full_k) {
        const float4 *p = reinterpret_cast<const float4 *>(d.B + (size_t)gn * d.ldb + k0);
#pragma unroll
        for (int q = 0; q < BK / 4; ++q) {
          float4 v = __ldg(p + q);
          rb[rr][4 * q] = v.x; rb[rr][4 * q + 1] = v.y; rb[rr][4 * q + 2] = v.z; rb[rr][4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < BK; ++k)
          rb[rr][k] = (ok && k0 + k < d.K) ? __ldg(d.B + (size_t)gn * d.ldb + k0 + k) : 0.f;
      }
    }
  };

  auto store = [&](int s) {
    uint8_t *base = smem + s * SM::STAGE;
    uint8_t *ahi = base, *alo = base + SM::A_BYTES;
    uint8_t *bhi = base + 2 * SM::A_BYTES, *blo = bhi + SM::B_BYTES;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      float4 h, l;
      split(ra[4 * q], h.x, l.x);
      split(ra[4 * q + 1], h.y, l.y);
      split(ra[4 * q + 2], h.z, l.z);
      split(ra[4 * q + 3], h.w, l.w);
      uint32_t off = core_off(tid, 4 * q, BM);
      *reinterpret_cast<float4 *>(ahi + off) = h;
      *reinterpret_cast<float4 *>(alo + off) = l;
    }
#pragma unroll
    for (int rr = 0; rr < BROWS; ++rr) {
      const int r = tid + rr * NT;
      if (r >= BN) continue;
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        float4 h, l;
        split(rb[rr][4 * q], h.x, l.x);
        split(rb[rr][4 * q + 1], h.y, l.y);
        split(rb[rr][4 * q + 2], h.z, l.z);
        split(rb[rr][4 * q + 3], h.w, l.w);
        uint32_t off = core_off(r, 4 * q, BN);
        *reinterpret_cast<float4 *>(bhi + off) = h;
        *reinterpret_cast<float4 *>(blo + off) = l;
      }
    }
  };

  constexpr uint32_t IDESC = make_idesc(BM, BN);
  constexpr uint32_t LBO_A = (BM / 8) * 128, LBO_B = (BN / 8) * 128, SBO = 128;

  load(0);
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    if (kt >= STAGES) mbar_wait(&bars[s], ((kt / STAGES) - 1) & 1);
    store(s);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (kt + 1 < nk) load(kt + 1);
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = smem_u32(smem + s * SM::STAGE);
      const uint32_t ahi = base, alo = base + SM::A_BYTES;
      const uint32_t bhi = base + 2 * SM::A_BYTES, blo = bhi + SM::B_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint64_t dah = make_desc(ahi + ks * 2 * LBO_A, LBO_A, SBO);
        const uint64_t dal = make_desc(alo + ks * 2 * LBO_A, LBO_A, SBO);
        const uint64_t dbh = make_desc(bhi + ks * 2 * LBO_B, LBO_B, SBO);
        const uint64_t dbl = make_desc(blo + ks * 2 * LBO_B, LBO_B, SBO);
        const uint32_t acc0 = (kt > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, dal, dbh, IDESC, acc0);   // small terms first
        mma_tf32(tmem, dah, dbl, IDESC, 1u);
        mma_tf32(tmem, dah, dbh, IDESC, 1u);
      }
      mma_commit(&bars[s]);
    }
    __syncwarp();
  }
  // wait for the last commit (tracks completion of every earlier tcgen05.mma of this thread)
  {
    const int last = nk - 1;
    mbar_wait(&bars[last % STAGES], (last / STAGES) & 1);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");

  // epilogue: TMEM lane (32*warp + lane) = tile row, 16 columns per tcgen05.ld
  const int row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < d.M) {
      float *out = d.C + (size_t)row * d.ldc + n0 + c0;
      const int nvalid = d.N - (n0 + c0);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nvalid) out[j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(SM::TMEM_COLS));
}

// ---------------------------------------------------------------------------------------------
// v2: operands arrive pre-split (A_hi/A_lo, B_hi/B_lo planes written by their producers, hi
// exactly representable in tf32).  The mainloop is pure data movement: 16-byte zero-filling
// cp.async copies straight into the core-matrix layout, a STAGES-deep cp.async group ring, and
// the same single-thread tcgen05.mma issue + mbarrier commit per stage.

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int BN>
__global__ void __launch_bounds__(NT) k_gemm_tc2(const GemmDesc2 *__restrict__ descs) {
  using SM = Smem<BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const GemmDesc2 d = descs[blockIdx.z];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= d.M || n0 >= d.N) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * SM::STAGE);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + STAGES * SM::STAGE + 64);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(SM::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int nk = (d.K + BK - 1) / BK;
  const uint32_t sbase = smem_u32(smem);

  // one K slice = (A_hi, A_lo: 128 rows x 4 chunks) + (B_hi, B_lo: BN rows x 4 chunks) of 16 B
  constexpr int A_CH = BM * (BK / 4), B_CH = BN * (BK / 4);
  constexpr int TOT = 2 * A_CH + 2 * B_CH;
  auto issue = [&](int s, int kt) {
    const int k0 = kt * BK;
    const uint32_t st = sbase + s * SM::STAGE;
#pragma unroll 1
    for (int c = tid; c < TOT; c += NT) {
      int part, rem;
      if (c < 2 * A_CH) { part = c / A_CH; rem = c - part * A_CH; }
      else { part = 2 + (c - 2 * A_CH) / B_CH; rem = (c - 2 * A_CH) - (part - 2) * B_CH; }
      const int row = rem >> 2, kc = rem & 3;
      const int k = k0 + 4 * kc;
      const bool isA = part < 2;
      const int R = isA ? BM : BN;
      const int grow = (isA ? m0 : n0) + row;
      const int lim = isA ? d.M : d.N;
      const float *src = isA ? (part == 0 ? d.Ahi : d.Alo) : (part == 2 ? d.Bhi : d.Blo);
      const int ld = isA ? d.lda : d.ldb;
      int valid = d.K - k;
      valid = valid < 0 ? 0 : (valid > 4 ? 4 : valid);
      if (grow >= lim) valid = 0;
      const float *g = valid ? src + (size_t)grow * ld + k : src;
      const uint32_t off = isA ? (part == 0 ? 0 : SM::A_BYTES) : (2 * SM::A_BYTES + (part == 2 ? 0 : SM::B_BYTES));
      const uint32_t dst = st + off + core_off(row, 4 * kc, R);
      cp_async16(dst, g, (uint32_t)(valid * 4));
    }
  };

  constexpr uint32_t IDESC = make_idesc(BM, BN);
  constexpr uint32_t LBO_A = (BM / 8) * 128, LBO_B = (BN / 8) * 128, SBO = 128;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    cp_async_wait<STAGES - 2>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t base = sbase + s * SM::STAGE;
      const uint32_t ahi = base, alo = base + SM::A_BYTES;
      const uint32_t bhi = base + 2 * SM::A_BYTES, blo = bhi + SM::B_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint64_t dah = make_desc(ahi + ks * 2 * LBO_A, LBO_A, SBO);
        const uint64_t dal = make_desc(alo + ks * 2 * LBO_A, LBO_A, SBO);
        const uint64_t dbh = make_desc(bhi + ks * 2 * LBO_B, LBO_B, SBO);
        const uint64_t dbl = make_desc(blo + ks * 2 * LBO_B, LBO_B, SBO);
        const uint32_t acc0 = (kt > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, dal, dbh, IDESC, acc0);
        mma_tf32(tmem, dah, dbl, IDESC, 1u);
        mma_tf32(tmem, dah, dbh, IDESC, 1u);
      }
      mma_commit(&bars[s]);
    }
    __syncwarp();
    const int kn = kt + STAGES - 1;
    if (kn < nk) {
      if (kt >= 1) mbar_wait(&bars[(kt - 1) % STAGES], ((kt - 1) / STAGES) & 1);
      issue(kn % STAGES, kn);
    }
    cp_async_commit();
  }
  {
    const int last = nk - 1;
    mbar_wait(&bars[last % STAGES], (last / STAGES) & 1);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < d.M) {
      float *out = d.C + (size_t)row * d.ldc + n0 + c0;
      const int nvalid = d.N - (n0 + c0);
      if (nvalid >= 16 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          reinterpret_cast<float4 *>(out)[q] =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                          __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < nvalid) out[j] = __uint_as_float(v[j]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(SM::TMEM_COLS));
}

template <int BN>
static cudaError_t launch_two(const GemmDesc2 *descs, int batch, int maxM, int maxN,
                              cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc2<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Smem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((maxN + BN - 1) / BN, (maxM + BM - 1) / BM, batch);
  k_gemm_tc2<BN><<<grid, NT, Smem<BN>::TOTAL, s>>>(descs);
  return cudaGetLastError();
}

template <int BN, bool AL>
static cudaError_t launch_one(const GemmDesc *descs, int batch, int maxM, int maxN,
                              cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<BN, AL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Smem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((maxN + BN - 1) / BN, (maxM + BM - 1) / BM, batch);
  k_gemm_tc<BN, AL><<<grid, NT, Smem<BN>::TOTAL, s>>>(descs);
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t launch_gemm_tc2(const GemmDesc2 *descs, int batch, int maxM, int maxN, int bn,
                            cudaStream_t s) {
  return bn == 144 ? tc::launch_two<144>(descs, batch, maxM, maxN, s)
                   : tc::launch_two<128>(descs, batch, maxM, maxN, s);
}

// bn: 128 or 144 (tile width); b_aligned: every Bt row start is 16-byte aligned and ldb % 4 == 0.
cudaError_t launch_gemm_tc(const GemmDesc *descs, int batch, int maxM, int maxN, int bn,
                           bool b_aligned, cudaStream_t s) {
  if (bn == 144) {
    return b_aligned ? tc::launch_one<144, true>(descs, batch, maxM, maxN, s)
                     : tc::launch_one<144, false>(descs, batch, maxM, maxN, s);
  }
  return b_aligned ? tc::launch_one<128, true>(descs, batch, maxM, maxN, s)
                   : tc::launch_one<128, false>(descs, batch, maxM, maxN, s);
}

}  // namespace tvs
