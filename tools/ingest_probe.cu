// Per-SM global->shared ingest probe (dev tool): bulk-copy (TMA engine) vs
// cp.async (LSU) vs both at once, L2-resident source, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ingest tools/ingest_probe.cu && /tmp/ingest
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t m, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(m), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t m, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t m, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(m), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(m) : "memory");
}

// mode bit 0: bulk copies by thread 0 (ring of NB x CH bytes)
// mode bit 1: cp.async 16 B by warps 1..7 into a separate region
template <int CH, int NB>
__global__ void __launch_bounds__(256, 1) probe(const uint8_t *src, size_t span, int iters, int mode, int *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NB * CH + 64 * 1024);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(su32(&bar[i]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t base = ((size_t)blockIdx.x * 7919 * CH) % (span - (size_t)iters * CH - CH);
  if ((mode & 1) && tid == 0) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % NB;
      if (it >= NB) mbar_wait(su32(&bar[st]), ((it / NB) - 1) & 1);
      mbar_expect(su32(&bar[st]), CH);
      bulk(su32(sm + st * CH), src + (base + (size_t)it * CH) % (span - CH), CH, su32(&bar[st]));
    }
    for (int it = iters > NB ? iters - NB : 0; it < iters; ++it) mbar_wait(su32(&bar[it % NB]), (it / NB) & 1);
  }
  if ((mode & 2) && tid >= 32) {
    // 7 warps, 16 B per thread per step, 64 KB region, 4 groups in flight
    const int t = tid - 32;
    uint8_t *dst = sm + NB * CH;
    const int steps = (int)(((size_t)iters * CH) / (224 * 16));
    for (int k = 0; k < steps; ++k) {
      const size_t off = (base + (size_t)k * 224 * 16 + t * 16) % (span - 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + ((k * 224 + t) * 16) % (64 * 1024))),
                   "l"(src + off));
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 6;");
    }
    asm volatile("cp.async.wait_group 0;");
  }
  __syncthreads();
  if (tid == 0 && iters < 0) sink[0] = sm[0];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t span = 48u << 20;  // L2 resident
  uint8_t *src;
  int *sink;
  cudaMalloc(&src, span);
  cudaMemset(src, 1, span);
  cudaMalloc(&sink, 4);
  constexpr int CH = 16384, NB = 8;
  const size_t smem = NB * CH + 64 * 1024 + 1024;
  cudaFuncSetAttribute(probe<CH, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 4000;
  for (int grid : {sms, sms / 2, 16}) {
    for (int mode : {1, 2, 3}) {
      probe<CH, NB><<<grid, 256, smem>>>(src, span, 200, mode, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      probe<CH, NB><<<grid, 256, smem>>>(src, span, iters, mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      double bytes = 0;
      if (mode & 1) bytes += (double)iters * CH;
      if (mode & 2) bytes += (double)((size_t)iters * CH / (224 * 16)) * 224 * 16;
      const double per_sm = bytes / (ms * 1e-3);
      printf("grid %3d mode %d (%s): %.1f GB/s per SM, %.1f B/clk/SM at %d MHz nominal, aggregate %.2f TB/s  (%s)\n",
             grid, mode, mode == 1 ? "bulk" : mode == 2 ? "cp.async" : "both", per_sm / 1e9,
             per_sm / (clk * 1e3), clk / 1000, per_sm * grid / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
