// Microbenchmark: tcgen05.mma issue rate per SM (one CTA per SM, one issuing thread).
#include "../paper_2602_17494_b200/csrc/tvs_gemm_tc.cu"  // build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/mma_bench profiles/mma_bench.cu -lcuda
#include <cstdio>
namespace tvs { namespace tc {
__device__ __forceinline__ void mma_bf16_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc) {
  uint32_t z = 0;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(1u) : "memory");
  (void)z;
}
__global__ void k_mma_bench(int iters, int mode, int n, long long *cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int nfl = (mode >= 3 ? 4 * 53248 : 65536) / 4;
  for (int i = tid; i < nfl; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u; h ^= h >> 13; h *= 0x85ebca6bu; h ^= h >> 16;
    reinterpret_cast<float *>(smem)[i] = mode >= 3 || mode < 0 ? ((float)(h & 0xffff) / 65536.f - 0.5f) : 0.f;
  }
  if (tid == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot, sb = smem_u32(smem);
  if (tid == 0) {
    const uint32_t id_tf32 = make_idesc(128, n);
    const uint32_t id_bf16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = make_desc_sw128(sb), db = make_desc_sw128(sb + 32768);
    long long t0 = clock64();
    if (mode >= 3) {
      for (int it = 0; it < iters / 12; ++it) {
        const uint32_t st = sb + (it % 4) * 53248;
        const uint32_t bhi = st + 16384, blo = bhi + 18432;
        const uint32_t ahi = tmem + 256 + 64 * (it & 1), alo = ahi + 32;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t dbh = make_desc_sw128(bhi + 32 * ks), dbl = make_desc_sw128(blo + 32 * ks);
          mma_tf32_ts(tmem, alo + 8 * ks, dbh, id_tf32, (it > 0 || ks > 0) ? 1u : 0u);
          mma_tf32_ts(tmem, ahi + 8 * ks, dbl, id_tf32, 1u);
          mma_tf32_ts(tmem, ahi + 8 * ks, dbh, id_tf32, 1u);
        }
        if (mode == 4) { mma_commit(&bar2); mma_commit(&bar2); }
      }
    } else
    for (int i = 0; i < iters; ++i) {
      if (mode == 0) mma_tf32_ts(tmem, tmem + 256, db, id_tf32, 1u);
      else if (mode == 1) mma_tf32(tmem, da, db, id_tf32, 1u);
      else mma_bf16_ss(tmem, da, db, id_bf16);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}
}}
int main() {
  long long *d; cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(tvs::tc::k_mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 53248 + 1024);
  const char *names[5] = {"tf32 TS", "tf32 SS", "bf16 SS", "tf32 TS ring", "tf32 TS ring+commit"};
  for (int mode = 0; mode < 5; ++mode)
    for (int n : {144}) {
      const int iters = 4096;
      tvs::tc::k_mma_bench<<<148, 128, 4 * 53248 + 1024>>>(iters, mode, n, d);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      tvs::tc::k_mma_bench<<<148, 128, 4 * 53248 + 1024>>>(iters, mode, n, d);
      cudaEventRecord(b); cudaError_t e = cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      const int K = mode == 2 ? 16 : 8;
      const double flops = 2.0 * 128 * n * K * iters * 148;
      printf("%s N=%3d: %.1f cycles/MMA, kernel %.3f ms -> %.0f TFLOP/s (%s)\n", names[mode], n, avg / iters, ms, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
    }
  return 0;
}
