// Dependent-chain latency of the arithmetic the ICP and raycast chains are
// made of (SM cycles per operation, one warp, clock64 around 1024 ops).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp_latency.cu -o fp_latency
#include <cstdio>
#include <cuda_runtime.h>

template <int kOp>
__global__ void chain(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-9;
  float xf = (float)x;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (kOp == 0) x = fma(x, 1.0000001, 1e-9);             // DFMA
      if (kOp == 1) x = x + 1e-9;                              // DADD
      if (kOp == 2) x = 1.0 / (x + 1.0);                       // DDIV (IEEE)
      if (kOp == 3) x = sqrt(x + 1.0);                         // DSQRT (IEEE)
      if (kOp == 4) xf = fmaf(xf, 1.0000001f, 1e-9f);          // FFMA
      if (kOp == 5) x = (double)(float)(x * 1.0000001);       // DMUL + F2F round trip
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    out[0] = x + xf;
  }
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  const char* names[] = {"DFMA", "DADD", "DDIV (IEEE, 1/(x+1))", "DSQRT (IEEE)", "FFMA", "DMUL + F2F.F32 + F2F.F64"};
  void (*ks[])(double*, long long*, double) = {chain<0>, chain<1>, chain<2>, chain<3>, chain<4>, chain<5>};
  for (int k = 0; k < 6; ++k) {
    long long best = 1LL << 62;
    for (int r = 0; r < 5; ++r) {
      ks[k]<<<1, 32>>>(d, c, 0.5);
      long long h = 0;
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      if (h < best) best = h;
    }
    std::printf("%-28s %7.1f cycles per dependent op\n", names[k], best / 1024.0);
  }
  return 0;
}
