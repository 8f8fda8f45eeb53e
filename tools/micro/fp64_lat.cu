// Dependent-chain latency of FP64 ops on this GPU (one warp, clock64): DADD, DMUL, DFMA, and the
// IEEE division __ddiv_rn.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, double y) {
  double x = x0;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, y);
  long long t1 = clock64();
  for (int i = 0; i < 1024; ++i) x = __dmul_rn(x, y);
  long long t2 = clock64();
  for (int i = 0; i < 1024; ++i) x = __fma_rn(x, y, y);
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) x = __ddiv_rn(y, x);
  long long t4 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, 1.0, 1.0000001); cudaDeviceSynchronize(); }
  printf("DADD %.1f  DMUL %.1f  DFMA %.1f  DDIV %.1f cycles per dependent op\n", c[0] / 1024.0, c[1] / 1024.0,
         c[2] / 1024.0, c[3] / 256.0);
}
