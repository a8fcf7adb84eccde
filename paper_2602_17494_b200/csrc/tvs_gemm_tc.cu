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
#include <stdlib.h>
#include <string.h>

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

  // one K slice = (A_hi, A_lo: 128 rows x 4 chunks) + (B_hi, B_lo: BN rows x 4 chunks) of 16 B.
  // Chunk c = tid + NT*i: its 16-byte column kc = tid & 3 is the same for every i (A_CH, B_CH and
  // NT are multiples of 4), so each thread's source rows and smem slots are fixed across k-tiles
  // and precomputed here; per k-tile a copy costs one pointer add and one cp.async.
  constexpr int A_CH = BM * (BK / 4), B_CH = BN * (BK / 4);
  constexpr int TOT = 2 * A_CH + 2 * B_CH;
  constexpr int PER = (TOT + NT - 1) / NT;
  const int kc = tid & 3;
  const float *src[PER];
  uint32_t dst[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = tid + NT * i;
    src[i] = nullptr;
    dst[i] = 0xFFFFFFFFu;
    if (c >= TOT) continue;
    int part, rem;
    if (c < 2 * A_CH) { part = c / A_CH; rem = c - part * A_CH; }
    else { part = 2 + (c - 2 * A_CH) / B_CH; rem = (c - 2 * A_CH) - (part - 2) * B_CH; }
    const int row = rem >> 2;
    const bool isA = part < 2;
    const int grow = (isA ? m0 : n0) + row;
    const int lim = isA ? d.M : d.N;
    const float *base = isA ? (part == 0 ? d.Ahi : d.Alo) : (part == 2 ? d.Bhi : d.Blo);
    const int ld = isA ? d.lda : d.ldb;
    if (grow < lim) src[i] = base + (size_t)grow * ld + 4 * kc;
    const uint32_t off = isA ? (part == 0 ? 0 : SM::A_BYTES) : (2 * SM::A_BYTES + (part == 2 ? 0 : SM::B_BYTES));
    dst[i] = off + core_off(row, 4 * kc, isA ? BM : BN);
  }
  auto issue = [&](int s, int kt) {
    const int k0 = kt * BK;
    const uint32_t st = sbase + s * SM::STAGE;
    int valid = d.K - (k0 + 4 * kc);
    valid = valid < 0 ? 0 : (valid > 4 ? 4 : valid);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (dst[i] == 0xFFFFFFFFu) continue;
      const bool ok = src[i] != nullptr && valid > 0;
      cp_async16(st + dst[i], ok ? (const void *)(src[i] + k0) : (const void *)d.Ahi,
                 ok ? (uint32_t)(valid * 4) : 0u);
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
  {
    cudaError_t e = smem_optin((const void *)k_gemm_tc2<BN>, Smem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((maxN + BN - 1) / BN, (maxM + BM - 1) / BM, batch);
  k_gemm_tc2<BN><<<grid, NT, Smem<BN>::TOTAL, s>>>(descs);
  return cudaGetLastError();
}

template <int BN, bool AL>
static cudaError_t launch_one(const GemmDesc *descs, int batch, int maxM, int maxN,
                              cudaStream_t s) {
  {
    cudaError_t e = smem_optin((const void *)k_gemm_tc<BN, AL>, Smem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((maxN + BN - 1) / BN, (maxM + BM - 1) / BM, batch);
  k_gemm_tc<BN, AL><<<grid, NT, Smem<BN>::TOTAL, s>>>(descs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// v3 (default): TMA + tcgen05, warp-specialised.  Per stage one cp.async.bulk.tensor per operand
// plane (box = {32 fp32 = 128 B, rows}, SWIZZLE_128B, OOB zero-fill handles every M/N/K tail);
// warp 0 lane 0 produces (full[s] with expect_tx), warp 1 lane 0 issues 4 k-steps x 3 MMAs per
// stage and commits to empty[s]; after the last stage a commit to `accum` releases the epilogue.
// K-major SWIZZLE_128B smem descriptors: LBO field 1, SBO = 1024 B (8 rows x 128 B), start
// address advanced by 32 B per k-step inside the 128-B swizzle atom (tiles 1024-B aligned).
constexpr int TBK = 32, TSTAGES = 3;

template <int BN>
struct TSmem {
  static constexpr int A_BYTES = BM * TBK * 4;      // 16 KB
  static constexpr int B_BYTES = BN * TBK * 4;      // 18 KB for BN = 144
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int TOTAL = TSTAGES * STAGE + 256 + 1024;   // barriers + alignment slack
  static constexpr int TMEM_COLS = BN <= 128 ? 128 : 256;
};

__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;                 // LBO (unused for swizzled K-major) = 1
  d |= (uint64_t)(1024u >> 4) << 32;       // SBO = 1024 B between 8-row groups
  d |= (uint64_t)1u << 46;                 // version (Blackwell)
  d |= (uint64_t)2u << 61;                 // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <int BN>
__global__ void __launch_bounds__(NT, 1) k_gemm_tma(const TmaGemmDesc *__restrict__ descs) {
  using SM = TSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const TmaGemmDesc *dp = descs + blockIdx.z;
  const int M = dp->M, N = dp->N, K = dp->K, ldc = dp->ldc;
  float *C = dp->C;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M || n0 >= N) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + TSTAGES * SM::STAGE);
  uint64_t *empty = full + TSTAGES;
  uint64_t *accum = empty + TSTAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accum + 1);
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(SM::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dp->a_hi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dp->b_hi)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const int nk = (K + TBK - 1) / TBK;
  const uint32_t sbase = smem_u32(smem);

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------------ TMA producer
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TSTAGES;
      if (kt >= TSTAGES) mbar_wait(&empty[s], ((kt / TSTAGES) - 1) & 1);
      mbar_expect_tx(&full[s], SM::STAGE);
      const uint32_t st = sbase + s * SM::STAGE;
      tma_load_2d(st, &dp->a_hi, kt * TBK, m0, &full[s]);
      tma_load_2d(st + SM::A_BYTES, &dp->a_lo, kt * TBK, m0, &full[s]);
      tma_load_2d(st + 2 * SM::A_BYTES, &dp->b_hi, kt * TBK, n0, &full[s]);
      tma_load_2d(st + 2 * SM::A_BYTES + SM::B_BYTES, &dp->b_lo, kt * TBK, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = make_idesc(BM, BN);
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TSTAGES;
      mbar_wait(&full[s], (kt / TSTAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t st = sbase + s * SM::STAGE;
      const uint32_t ahi = st, alo = st + SM::A_BYTES;
      const uint32_t bhi = st + 2 * SM::A_BYTES, blo = bhi + SM::B_BYTES;
#pragma unroll
      for (int ks = 0; ks < TBK / 8; ++ks) {
        const uint64_t dah = make_desc_sw128(ahi + 32 * ks), dal = make_desc_sw128(alo + 32 * ks);
        const uint64_t dbh = make_desc_sw128(bhi + 32 * ks), dbl = make_desc_sw128(blo + 32 * ks);
        mma_tf32(tmem, dal, dbh, IDESC, (kt > 0 || ks > 0) ? 1u : 0u);
        mma_tf32(tmem, dah, dbl, IDESC, 1u);
        mma_tf32(tmem, dah, dbh, IDESC, 1u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(accum);
  }
  __syncwarp();
  // ------------------------------------------------------------------ epilogue (all 4 warps)
  mbar_wait(accum, 0);
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
    if (row < M) {
      float *out = C + (size_t)row * ldc + n0 + c0;
      const int nvalid = N - (n0 + c0);
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
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(SM::TMEM_COLS));
}

template <int BN>
static cudaError_t launch_tma(const TmaGemmDesc *descs, int batch, int maxM, int maxN,
                              cudaStream_t s) {
  {
    cudaError_t e = smem_optin((const void *)k_gemm_tma<BN>, TSmem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((maxN + BN - 1) / BN, (maxM + BM - 1) / BM, batch);
  k_gemm_tma<BN><<<grid, NT, TSmem<BN>::TOTAL, s>>>(descs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Persistent form (default): one CTA per SM loops over the (desc, m-block, n-block) tiles.
// Warp roles (10 warps):
//   warp 0      TMA producer: A (raw fp32, one plane) + B_hi + B_lo per K slice of 32
//   warps 6..9  split A in shared memory: hi = tf32_rna(a) in place, lo = a - hi (exact), then
//               fence.proxy.async so the tensor core sees the generic-proxy stores
//   warp 1      MMA issuer: 4 k-steps x 3 tcgen05.mma per stage into one of two TMEM accumulators
//   warps 2..5  epilogue: tcgen05.ld of the finished accumulator (warp w owns TMEM lanes
//               32 (w % 4) ..), float4 stores; it overlaps the next tile's main loop.
// The A operand therefore streams from HBM/L2 once, in fp32 (half the bytes of pre-split hi/lo
// planes); B (DCT tables, L2-resident) stays pre-split.  Same arithmetic as k_gemm_tma.
constexpr int PSTAGES = 3, PNT = 320;

template <int BN>
struct PSmem {
  static constexpr int A_BYTES = BM * TBK * 4;                 // 16 KB
  static constexpr int B_BYTES = BN * TBK * 4;                 // 18 KB for BN = 144
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;      // A (-> hi), A lo, B hi, B lo
  static constexpr int TX = A_BYTES + 2 * B_BYTES;             // bytes landed by TMA per stage
  static constexpr int TOTAL = PSTAGES * STAGE + 256 + 1024;
  static constexpr int ACC = BN <= 128 ? 128 : 256;            // TMEM columns per accumulator
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int BN>
__global__ void __launch_bounds__(PNT, 1)
k_gemm_tma_p(const TmaGemmDesc *__restrict__ descs, int batch, int mblocks, int nblocks) {
  using SM = PSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + PSTAGES * SM::STAGE);
  uint64_t *conv = full + PSTAGES;
  uint64_t *empty = conv + PSTAGES;
  uint64_t *accf = empty + PSTAGES;   // [2]
  uint64_t *acce = accf + 2;          // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(2 * SM::ACC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  const int per = mblocks * nblocks, ntiles = batch * per;
  // tile decode shared by every role (n fastest: neighbouring CTAs share the A rows)
  auto decode = [&](int t, const TmaGemmDesc *&dp, int &m0, int &n0) {
    const int z = t / per, r = t - z * per;
    dp = descs + z;
    m0 = (r / nblocks) * BM;
    n0 = (r % nblocks) * BN;
    return m0 < dp->M && n0 < dp->N;
  };

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TmaGemmDesc *dp;
        int m0, n0;
        if (!decode(t, dp, m0, n0)) continue;
        const int nk = (dp->K + TBK - 1) / TBK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % PSTAGES;
          if (it >= PSTAGES) mbar_wait(&empty[s], ((it / PSTAGES) - 1) & 1);
          mbar_expect_tx(&full[s], SM::TX);
          const uint32_t st = sbase + s * SM::STAGE;
          tma_load_2d(st, &dp->a_hi, kt * TBK, m0, &full[s]);
          tma_load_2d(st + 2 * SM::A_BYTES, &dp->b_hi, kt * TBK, n0, &full[s]);
          tma_load_2d(st + 2 * SM::A_BYTES + SM::B_BYTES, &dp->b_lo, kt * TBK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      constexpr uint32_t IDESC = make_idesc(BM, BN);
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TmaGemmDesc *dp;
        int m0, n0;
        if (!decode(t, dp, m0, n0)) continue;
        const int b = tc & 1;
        if (tc >= 2) mbar_wait(&acce[b], ((tc >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + (uint32_t)(b * SM::ACC);
        const int nk = (dp->K + TBK - 1) / TBK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int s = it % PSTAGES;
          mbar_wait(&conv[s], (it / PSTAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = sbase + s * SM::STAGE;
          const uint32_t ahi = st, alo = st + SM::A_BYTES;
          const uint32_t bhi = st + 2 * SM::A_BYTES, blo = bhi + SM::B_BYTES;
#pragma unroll
          for (int ks = 0; ks < TBK / 8; ++ks) {
            const uint64_t dah = make_desc_sw128(ahi + 32 * ks), dal = make_desc_sw128(alo + 32 * ks);
            const uint64_t dbh = make_desc_sw128(bhi + 32 * ks), dbl = make_desc_sw128(blo + 32 * ks);
            mma_tf32(acc, dal, dbh, IDESC, (kt > 0 || ks > 0) ? 1u : 0u);
            mma_tf32(acc, dah, dbl, IDESC, 1u);
            mma_tf32(acc, dah, dbh, IDESC, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accf[b]);
        ++tc;
      }
    }
  } else if (warp >= 6) {   // ----------------------------------------------- A split
    const int ct = tid - 6 * 32;   // 0..127
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TmaGemmDesc *dp;
      int m0, n0;
      if (!decode(t, dp, m0, n0)) continue;
      const int nk = (dp->K + TBK - 1) / TBK;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const int s = it % PSTAGES;
        mbar_wait(&full[s], (it / PSTAGES) & 1);
        float4 *a = reinterpret_cast<float4 *>(smem + s * SM::STAGE);
        float4 *lo = reinterpret_cast<float4 *>(smem + s * SM::STAGE + SM::A_BYTES);
#pragma unroll
        for (int q = 0; q < SM::A_BYTES / 16 / 128; ++q) {   // element-wise: layout agnostic
          const int i = ct + q * 128;
          float4 x = a[i], h, l;
          split(x.x, h.x, l.x);
          split(x.y, h.y, l.y);
          split(x.z, h.z, l.z);
          split(x.w, h.w, l.w);
          a[i] = h;
          lo[i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ct == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {   // warps 2..5 ------------------------------------------------------ epilogue
    const int q4 = warp & 3;   // TMEM lane quarter this warp may access
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TmaGemmDesc *dp;
      int m0, n0;
      if (!decode(t, dp, m0, n0)) continue;
      const int b = tc & 1;
      mbar_wait(&accf[b], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int M = dp->M, N = dp->N, ldc = dp->ldc;
      float *C = dp->C;
      const int row = m0 + q4 * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(b * SM::ACC + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
          float *out = C + (size_t)row * ldc + n0 + c0;
          const int nvalid = N - (n0 + c0);
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      ++tc;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * SM::ACC));
}

template <int BN>
static cudaError_t launch_tma_p(const TmaGemmDesc *descs, int batch, int maxM, int maxN,
                                cudaStream_t s) {
  {
    cudaError_t e = smem_optin((const void *)k_gemm_tma_p<BN>, PSmem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
  }
  const int nsm = sm_count();
  const int mb = (maxM + BM - 1) / BM, nb = (maxN + BN - 1) / BN;
  const int ntiles = batch * mb * nb;
  const int grid = ntiles < nsm ? ntiles : nsm;
  k_gemm_tma_p<BN><<<grid, PNT, PSmem<BN>::TOTAL, s>>>(descs, batch, mb, nb);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// TS form (A in tensor memory): same persistent roles as k_gemm_tma_p, but the split warps write
// A_hi / A_lo into TMEM with tcgen05.st and the MMAs read A from TMEM ([a-tmem] operand), so the
// tensor core reads only B from shared memory and a shared-memory stage holds A raw + B hi/lo
// (52 KB: four stages in flight instead of three).  TMEM: accumulators at columns 0 and 256
// (BN = 144 each), A slots (hi 32 + lo 32 columns) at 144 and 400.
constexpr int QSTAGES = 4;

template <int BN>
struct QSmem {
  static constexpr int A_BYTES = BM * TBK * 4;                 // 16 KB (raw fp32 A)
  static constexpr int B_BYTES = BN * TBK * 4;
  static constexpr int STAGE = A_BYTES + 2 * B_BYTES;          // A raw, B hi, B lo
  static constexpr int TX = STAGE;
  static constexpr int STG = QSTAGES * STAGE + 256;            // epilogue staging: 4 KB per warp
  static constexpr int TOTAL = STG + 4 * 4096 + 1024;
};

// Coalesced epilogue of one 32-row TMEM lane quarter: columns are read from TMEM 32 at a time,
// transposed through a 4 KB shared-memory block (16-byte chunk j of row r at chunk j ^ (r & 7):
// conflict-free both ways), and written as whole 128-byte row segments (8 lanes per row), so every
// global store instruction covers four full lines instead of 32 partial ones.
template <int BN>
__device__ __forceinline__ void epilogue_quarter(uint32_t tacc, float *stg, float *C, int ldc, int M,
                                                 int N, int row0, int n0, int lane, int c_blk = 0,
                                                 long long c_plane = 0) {
  // column-block-major C (c_blk = 16 or 32): a 4-column group never straddles a block
  const bool vec = (c_blk > 0 || (ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
  const int cj = lane & 7, rq = lane >> 3;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    const int w = BN - c0 < 32 ? BN - c0 : 32;   // 32, or 16 for the last chunk of BN = 144
    uint32_t v[32];
    if (w == 32) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
            "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
            "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(tacc + (uint32_t)c0));
    } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tacc + (uint32_t)c0));
#pragma unroll
      for (int j = 16; j < 32; ++j) v[j] = 0u;
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!vec) {   // unaligned output rows: per-thread row stores
      const int row = row0 + lane;
      if (row < M) {
        float *out = C + (size_t)row * ldc + n0 + c0;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < w && n0 + c0 + j < N) out[j] = __uint_as_float(v[j]);
      }
      continue;
    }
    __syncwarp();   // the previous chunk's reads of the staging block are done
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (4 * j < w)
        reinterpret_cast<float4 *>(stg + lane * 32)[j ^ (lane & 7)] =
            make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                        __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
    __syncwarp();
    const int col = n0 + c0 + 4 * cj;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 4 * i + rq, row = row0 + r;
      if (4 * cj < w && row < M && col < N) {
        const float4 x = reinterpret_cast<const float4 *>(stg + r * 32)[cj ^ (r & 7)];
        float *out = c_blk > 0 ? C + (size_t)(col / c_blk) * c_plane + (size_t)row * c_blk + col % c_blk
                               : C + (size_t)row * ldc + col;
        if (col + 3 < N) {
          *reinterpret_cast<float4 *>(out) = x;
        } else {
          out[0] = x.x;
          if (col + 1 < N) out[1] = x.y;
          if (col + 2 < N) out[2] = x.z;
        }
      }
    }
  }
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
  uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(
          tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate), "r"(z), "r"(z), "r"(z), "r"(z)
      : "memory");
}

#define TST32(addr, v)                                                                              \
  asm volatile(                                                                                     \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),               \
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),       \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), \
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),          \
      "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),          \
      "r"(v[30]), "r"(v[31])                                                                        \
      : "memory")

template <int BN, int NS>
__global__ void __launch_bounds__(PNT, 1)
k_gemm_tma_ts(const TmaGemmDesc *__restrict__ descs, int batch, int mblocks, int nblocks) {
  static_assert(BN <= 144, "TMEM column plan assumes BN <= 144");
  using SM = QSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + QSTAGES * SM::STAGE);
  uint64_t *empty = full + QSTAGES;       // smem stage free (MMA done)
  uint64_t *aful = empty + QSTAGES;       // [NS] TMEM A slot written
  uint64_t *aemp = aful + 3;              // [NS] TMEM A slot free (MMA done)
  uint64_t *accf = aemp + 3;              // [2]
  uint64_t *acce = accf + 2;              // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int q = 0; q < QSTAGES; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int b = 0; b < NS; ++b) {
      mbar_init(&aful[b], 1);
      mbar_init(&aemp[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  // TMEM columns: NS = 2: accumulators 0 / 256, A slots 144 / 400; NS = 3: accumulators 0 / 144,
  // A slots 288 / 352 / 416 (each slot: hi 32 + lo 32 columns)
  // (computed, not tables: an indexed array lands in local memory, an LDL on the MMA issue path)
  auto ACC = [](int b) { return (uint32_t)b * (NS == 2 ? 256u : 144u); };
  auto ASLOT = [](int a) { return NS == 2 ? 144u + 256u * (uint32_t)a : 288u + 64u * (uint32_t)a; };
  const int per = mblocks * nblocks, ntiles = batch * per;
  auto decode = [&](int t, const TmaGemmDesc *&dp, int &m0, int &n0) {
    const int z = t / per, r = t - z * per;
    dp = descs + z;
    m0 = (r / nblocks) * BM;
    n0 = (r % nblocks) * BN;
    return m0 < dp->M && n0 < dp->N;
  };

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TmaGemmDesc *dp;
        int m0, n0;
        if (!decode(t, dp, m0, n0)) continue;
        const int nk = (dp->K + TBK - 1) / TBK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int q = it % QSTAGES;
          if (it >= QSTAGES) mbar_wait(&empty[q], ((it / QSTAGES) - 1) & 1);
          mbar_expect_tx(&full[q], SM::TX);
          const uint32_t st = sbase + q * SM::STAGE;
          if (dp->a_blk_rows > 0)
            tma_load_2d(st, &dp->a_hi, 0, kt * dp->a_blk_rows + m0, &full[q]);
          else
            tma_load_2d(st, &dp->a_hi, kt * TBK, m0, &full[q]);
          tma_load_2d(st + SM::A_BYTES, &dp->b_hi, kt * TBK, n0, &full[q]);
          tma_load_2d(st + SM::A_BYTES + SM::B_BYTES, &dp->b_lo, kt * TBK, n0, &full[q]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      constexpr uint32_t IDESC = make_idesc(BM, BN);
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TmaGemmDesc *dp;
        int m0, n0;
        if (!decode(t, dp, m0, n0)) continue;
        const int b = tc & 1;
        if (tc >= 2) mbar_wait(&acce[b], ((tc >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + ACC(b);
        const int nk = (dp->K + TBK - 1) / TBK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int q = it % QSTAGES, a = it % NS;
          mbar_wait(&full[q], (it / QSTAGES) & 1);   // B landed (TMA, async proxy)
          mbar_wait(&aful[a], (it / NS) & 1);        // A slot written to TMEM
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = sbase + q * SM::STAGE;
          const uint32_t bhi = st + SM::A_BYTES, blo = bhi + SM::B_BYTES;
          const uint32_t ahi = tmem + ASLOT(a), alo = ahi + 32;
#pragma unroll
          for (int ks = 0; ks < TBK / 8; ++ks) {
            const uint64_t dbh = make_desc_sw128(bhi + 32 * ks), dbl = make_desc_sw128(blo + 32 * ks);
            mma_tf32_ts(acc, alo + 8 * ks, dbh, IDESC, (kt > 0 || ks > 0) ? 1u : 0u);
            mma_tf32_ts(acc, ahi + 8 * ks, dbl, IDESC, 1u);
            mma_tf32_ts(acc, ahi + 8 * ks, dbh, IDESC, 1u);
          }
          mma_commit(&empty[q]);
          mma_commit(&aemp[a]);
        }
        mma_commit(&accf[b]);
        ++tc;
      }
    }
  } else if (warp >= 6) {   // ----------------------------------------------- A split -> TMEM
    const int q4 = warp & 3, row = q4 * 32 + lane;   // this thread's A row (TMEM lane)
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TmaGemmDesc *dp;
      int m0, n0;
      if (!decode(t, dp, m0, n0)) continue;
      const int nk = (dp->K + TBK - 1) / TBK;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const int q = it % QSTAGES, a = it % NS;
        mbar_wait(&full[q], (it / QSTAGES) & 1);
        if (it >= NS) mbar_wait(&aemp[a], ((it / NS) - 1) & 1);
        // row `row` of the 128-B swizzled A tile: 16-B chunk c sits at chunk c ^ (row & 7)
        const uint32_t ar = sbase + (uint32_t)(q * SM::STAGE + row * 128);   // shared window
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                       : "r"(ar + 16u * (uint32_t)(c ^ (row & 7)))
                       : "memory");
          float h, l;
          split(x.x, h, l); hi[4 * c] = __float_as_uint(h); lo[4 * c] = __float_as_uint(l);
          split(x.y, h, l); hi[4 * c + 1] = __float_as_uint(h); lo[4 * c + 1] = __float_as_uint(l);
          split(x.z, h, l); hi[4 * c + 2] = __float_as_uint(h); lo[4 * c + 2] = __float_as_uint(l);
          split(x.w, h, l); hi[4 * c + 3] = __float_as_uint(h); lo[4 * c + 3] = __float_as_uint(l);
        }
        const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + ASLOT(a);
        TST32(ta, hi);
        TST32(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 6 * 32) mbar_arrive(&aful[a]);
      }
    }
  } else {   // warps 2..5 ------------------------------------------------------ epilogue
    const int q4 = warp & 3;
    int tc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TmaGemmDesc *dp;
      int m0, n0;
      if (!decode(t, dp, m0, n0)) continue;
      const int b = tc & 1;
      mbar_wait(&accf[b], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      epilogue_quarter<BN>(tmem + ((uint32_t)(q4 * 32) << 16) + ACC(b),
                           reinterpret_cast<float *>(smem + SM::STG) + q4 * 1024, dp->C, dp->ldc,
                           dp->M, dp->N, m0 + q4 * 32, n0, lane, dp->c_blk, dp->c_plane);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      ++tc;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int BN>
static cudaError_t launch_tma_ts(const TmaGemmDesc *descs, int batch, int maxM, int maxN,
                                 cudaStream_t s) {
  {
    cudaError_t e = smem_optin((const void *)k_gemm_tma_ts<BN, 2>, QSmem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
  }
  const int nsm = sm_count();
  const int mb = (maxM + BM - 1) / BM, nb = (maxN + BN - 1) / BN;
  const int ntiles = batch * mb * nb;
  const int grid = ntiles < nsm ? ntiles : nsm;
  k_gemm_tma_ts<BN, 2><<<grid, PNT, QSmem<BN>::TOTAL, s>>>(descs, batch, mb, nb);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// CTA-pair form of the TS kernel (cta_group::2, M = 256 per MMA): a cluster of two CTAs on one
// TPC computes a 256 x 144 tile.  Each CTA stages its own 128 A rows (raw fp32 -> split into its
// TMEM) and HALF of the pre-split B tile (72 of the 144 rows, hi + lo); the leader CTA issues the
// MMAs, which read A from both CTAs' TMEM and B from both CTAs' shared memory.  Per SM this halves
// the B bytes from L2 and the B reads from shared memory, and a stage shrinks to 34 KB (6 stages).
// Barriers: A landed -> local fullA; B halves of both CTAs -> the leader's fullB (2-SM TMA);
// A split written -> the leader's aful (remote arrive, count 2); MMA commits multicast to both
// CTAs (empty, aemp, accf); epilogue done -> the leader's acce (remote arrive, count 8).
constexpr int RSTAGES = 6;

template <int BN>
struct RSmem {
  static constexpr int A_BYTES = BM * TBK * 4;                 // 16 KB
  static constexpr int BH_BYTES = (BN / 2) * TBK * 4;          // 9 KB (72 rows)
  static constexpr int STAGE = A_BYTES + 2 * BH_BYTES;         // 34 KB
  static constexpr int TOTAL = RSTAGES * STAGE + 512 + 1024;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_remote(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                                uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                                 uint32_t idesc, uint32_t accumulate) {
  uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8, %9, %10, %11, %12}, p;\n\t}" ::"r"(
          tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate), "r"(z), "r"(z), "r"(z), "r"(z), "r"(z),
      "r"(z), "r"(z), "r"(z)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PNT, 1)
k_gemm_tma_ts2(const TmaGemmDesc *__restrict__ descs, int batch, int mpairs, int nblocks) {
  using SM = RSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  uint64_t *fullA = reinterpret_cast<uint64_t *>(smem + RSTAGES * SM::STAGE);
  uint64_t *fullB = fullA + RSTAGES;     // leader only
  uint64_t *empty = fullB + RSTAGES;
  uint64_t *aful = empty + RSTAGES;      // [2] leader only
  uint64_t *aemp = aful + 2;             // [2]
  uint64_t *accf = aemp + 2;             // [2]
  uint64_t *acce = accf + 2;             // [2] leader only
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acce + 2);
  if (tid == 0) {
    for (int q = 0; q < RSTAGES; ++q) {
      mbar_init(&fullA[q], 1);
      mbar_init(&fullB[q], 1);
      mbar_init(&empty[q], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&aful[b], 2);
      mbar_init(&aemp[b], 1);
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);
  auto ACC = [](int b) { return 256u * (uint32_t)b; };
  auto ASLOT = [](int a) { return 144u + 256u * (uint32_t)a; };
  const int per = mpairs * nblocks, ntiles = batch * per;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  auto decode = [&](int t, const TmaGemmDesc *&dp, int &mp0, int &n0) {
    const int z = t / per, r = t - z * per;
    dp = descs + z;
    mp0 = (r / nblocks) * (2 * BM);
    n0 = (r % nblocks) * BN;
    return mp0 < dp->M && n0 < dp->N;
  };

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ TMA producer (both)
      int it = 0;
      const uint32_t fullB0 = map_to_rank0(smem_u32(fullB));
      for (int t = cid; t < ntiles; t += ncl) {
        const TmaGemmDesc *dp;
        int mp0, n0;
        if (!decode(t, dp, mp0, n0)) continue;
        const int nk = (dp->K + TBK - 1) / TBK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int q = it % RSTAGES;
          if (it >= RSTAGES) mbar_wait(&empty[q], ((it / RSTAGES) - 1) & 1);
          const uint32_t st = sbase + q * SM::STAGE;
          mbar_expect_tx(&fullA[q], SM::A_BYTES);
          tma_load_2d(st, &dp->a_hi, kt * TBK, mp0 + (int)rank * BM, &fullA[q]);
          if (leader) mbar_expect_tx(&fullB[q], 4 * SM::BH_BYTES);   // both CTAs' hi + lo halves
          const uint32_t fb = fullB0 + q * 8;
          tma_load_2d_2sm(st + SM::A_BYTES, &dp->b_hi, kt * TBK, n0 + (int)rank * (BN / 2), fb);
          tma_load_2d_2sm(st + SM::A_BYTES + SM::BH_BYTES, &dp->b_lo, kt * TBK,
                          n0 + (int)rank * (BN / 2), fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {   // ---------------------------------- MMA issuer (leader only)
      constexpr uint32_t IDESC = make_idesc(2 * BM, BN);
      int it = 0, tc = 0;
      for (int t = cid; t < ntiles; t += ncl) {
        const TmaGemmDesc *dp;
        int mp0, n0;
        if (!decode(t, dp, mp0, n0)) continue;
        const int b = tc & 1;
        if (tc >= 2) mbar_wait(&acce[b], ((tc >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + ACC(b);
        const int nk = (dp->K + TBK - 1) / TBK;
        for (int kt = 0; kt < nk; ++kt, ++it) {
          const int q = it % RSTAGES, a = it & 1;
          mbar_wait(&fullB[q], (it / RSTAGES) & 1);
          mbar_wait(&aful[a], (it >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = sbase + q * SM::STAGE;
          const uint32_t bhi = st + SM::A_BYTES, blo = bhi + SM::BH_BYTES;
          const uint32_t ahi = tmem + ASLOT(a), alo = ahi + 32;
#pragma unroll
          for (int ks = 0; ks < TBK / 8; ++ks) {
            const uint64_t dbh = make_desc_sw128(bhi + 32 * ks), dbl = make_desc_sw128(blo + 32 * ks);
            mma_tf32_ts_pair(acc, alo + 8 * ks, dbh, IDESC, (kt > 0 || ks > 0) ? 1u : 0u);
            mma_tf32_ts_pair(acc, ahi + 8 * ks, dbl, IDESC, 1u);
            mma_tf32_ts_pair(acc, ahi + 8 * ks, dbh, IDESC, 1u);
          }
          mma_commit_pair(&empty[q]);
          mma_commit_pair(&aemp[a]);
        }
        mma_commit_pair(&accf[b]);
        ++tc;
      }
    }
  } else if (warp >= 6) {   // ----------------------------------------------- A split -> TMEM
    const int q4 = warp & 3, row = q4 * 32 + lane;
    const uint32_t aful0 = map_to_rank0(smem_u32(aful));
    int it = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      const TmaGemmDesc *dp;
      int mp0, n0;
      if (!decode(t, dp, mp0, n0)) continue;
      const int nk = (dp->K + TBK - 1) / TBK;
      for (int kt = 0; kt < nk; ++kt, ++it) {
        const int q = it % RSTAGES, a = it & 1;
        mbar_wait(&fullA[q], (it / RSTAGES) & 1);
        if (it >= 2) mbar_wait(&aemp[a], ((it >> 1) - 1) & 1);
        const uint32_t ar = sbase + (uint32_t)(q * SM::STAGE + row * 128);   // shared window
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                       : "r"(ar + 16u * (uint32_t)(c ^ (row & 7)))
                       : "memory");
          float h, l;
          split(x.x, h, l); hi[4 * c] = __float_as_uint(h); lo[4 * c] = __float_as_uint(l);
          split(x.y, h, l); hi[4 * c + 1] = __float_as_uint(h); lo[4 * c + 1] = __float_as_uint(l);
          split(x.z, h, l); hi[4 * c + 2] = __float_as_uint(h); lo[4 * c + 2] = __float_as_uint(l);
          split(x.w, h, l); hi[4 * c + 3] = __float_as_uint(h); lo[4 * c + 3] = __float_as_uint(l);
        }
        const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + ASLOT(a);
        TST32(ta, hi);
        TST32(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 6 * 32) mbar_arrive_remote(aful0 + a * 8);
      }
    }
  } else {   // warps 2..5 ------------------------------------------------------ epilogue
    const int q4 = warp & 3;
    const uint32_t acce0 = map_to_rank0(smem_u32(acce));
    int tc = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      const TmaGemmDesc *dp;
      int mp0, n0;
      if (!decode(t, dp, mp0, n0)) continue;
      const int b = tc & 1;
      mbar_wait(&accf[b], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int M = dp->M, N = dp->N, ldc = dp->ldc;
      float *C = dp->C;
      const int row = mp0 + (int)rank * BM + q4 * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + ACC(b) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
          float *out = C + (size_t)row * ldc + n0 + c0;
          const int nvalid = N - (n0 + c0);
          if (nvalid >= 16 && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq)
              reinterpret_cast<float4 *>(out)[qq] =
                  make_float4(__uint_as_float(v[4 * qq]), __uint_as_float(v[4 * qq + 1]),
                              __uint_as_float(v[4 * qq + 2]), __uint_as_float(v[4 * qq + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < nvalid) out[j] = __uint_as_float(v[j]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acce0 + b * 8);
      ++tc;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int BN>
static cudaError_t launch_tma_ts2(const TmaGemmDesc *descs, int batch, int maxM, int maxN,
                                  cudaStream_t s) {
  {
    cudaError_t e = smem_optin((const void *)k_gemm_tma_ts2<BN>, RSmem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
  }
  const int nsm = sm_count();
  const int mp = (maxM + 2 * BM - 1) / (2 * BM), nb = (maxN + BN - 1) / BN;
  const int ntiles = batch * mp * nb;
  const int clusters = ntiles < nsm / 2 ? ntiles : nsm / 2;
  k_gemm_tma_ts2<BN><<<2 * clusters, PNT, RSmem<BN>::TOTAL, s>>>(descs, batch, mp, nb);
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t launch_gemm_tma_ts2(const TmaGemmDesc *descs, int batch, int maxM, int maxN,
                                cudaStream_t s) {
  return tc::launch_tma_ts2<144>(descs, batch, maxM, maxN, s);
}

cudaError_t launch_gemm_tma_ts(const TmaGemmDesc *descs, int batch, int maxM, int maxN, int bn,
                               cudaStream_t s) {
  return bn == 144 ? tc::launch_tma_ts<144>(descs, batch, maxM, maxN, s)
                   : tc::launch_tma_ts<128>(descs, batch, maxM, maxN, s);
}

cudaError_t launch_gemm_tma_p(const TmaGemmDesc *descs, int batch, int maxM, int maxN, int bn,
                              cudaStream_t s) {
  return bn == 144 ? tc::launch_tma_p<144>(descs, batch, maxM, maxN, s)
                   : tc::launch_tma_p<128>(descs, batch, maxM, maxN, s);
}

cudaError_t launch_gemm_tma(const TmaGemmDesc *descs, int batch, int maxM, int maxN, int bn,
                            cudaStream_t s) {
  return bn == 144 ? tc::launch_tma<144>(descs, batch, maxM, maxN, s)
                   : tc::launch_tma<128>(descs, batch, maxM, maxN, s);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static cudaError_t encode_2d(CUtensorMap *map, const float *base, int cols, int rows, int ld,
                             int box_rows) {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || !p) return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)(cols > 0 ? cols : 1), (cuuint64_t)(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)tc::TBK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Plain (unswizzled) 2D tensor map for the y-solve's staged blocks: fp32 or fp64 elements.
cudaError_t encode_plain_2d(CUtensorMap *map, const void *base, bool fp64, int cols, int rows,
                            int ld_elems, int box_cols, int box_rows) {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || !p) return e != cudaSuccess ? e : cudaErrorSymbolNotFound;
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  const size_t es = fp64 ? 8 : 4;
  const cuuint64_t dims[2] = {(cuuint64_t)(cols > 0 ? cols : 1), (cuuint64_t)(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld_elems * es};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, fp64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_tma_desc(TmaGemmDesc *out, const GemmDesc2 &d, int bn) {
  memset(out, 0, sizeof *out);
  cudaError_t e;
  if ((e = encode_2d(&out->a_hi, d.Ahi, d.K, d.M, d.lda, tc::BM)) != cudaSuccess) return e;
  if (d.Alo && (e = encode_2d(&out->a_lo, d.Alo, d.K, d.M, d.lda, tc::BM)) != cudaSuccess) return e;
  if ((e = encode_2d(&out->b_hi, d.Bhi, d.K, d.N, d.ldb, bn)) != cudaSuccess) return e;
  if ((e = encode_2d(&out->b_lo, d.Blo, d.K, d.N, d.ldb, bn)) != cudaSuccess) return e;
  out->C = d.C;
  out->M = d.M;
  out->N = d.N;
  out->K = d.K;
  out->ldc = d.ldc;
  return cudaSuccess;
}

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
