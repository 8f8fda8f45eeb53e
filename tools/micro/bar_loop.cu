// Microbenchmark: cost per iteration of a level-sweep-like loop on one CTA
// (named barrier of n threads, a shared-memory load + atomic per thread).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int iters, int nact, int mode, unsigned long long* out, uint32_t* g) {
  __shared__ uint32_t sm[2][4096];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ __align__(16) uint32_t dst[1024];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(g), "r"(4096), "r"(su32(&bar)) : "memory");
    uint32_t done = 0;
    while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(su32(&bar)), "r"(0) : "memory");
  }
  const uint32_t tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) (&sm[0][0])[i] = i;
  __syncthreads();
  if (tid >= (uint32_t)nact) return;
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t* r = sm[it & 1];
    uint32_t* w = sm[(it + 1) & 1];
    if (mode >= 1) {
      uint32_t v = r[(tid * 7 + it) & 4095];
      acc += v;
      if (mode >= 2) atomicAdd(&w[(tid * 13 + it) & 4095], v);
      if (mode >= 3) g[it * 64 + tid] = v;
    }
    if (mode == 4 && tid == (uint32_t)nact - 1) {
      for (int j = 0; j < 2; ++j) {
        uint32_t done = 0;
        while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(su32(&bar)), "r"(0) : "memory");
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nact) : "memory");
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (unsigned long long)(t1 - t0);
  if (acc == 12345) g[0] = acc;
}
int main() {
  unsigned long long* d; uint32_t* g;
  cudaMalloc(&d, 8); cudaMalloc(&g, 64 * 100000 * 4);
  for (int nact : {64, 256, 1024})
    for (int mode = 0; mode < 5; ++mode) {
      k<<<1, 1024>>>(20000, nact, mode, d, g);
      unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("nact %4d mode %d: %.1f cycles/iter\n", nact, mode, c / 20000.0);
    }
}
