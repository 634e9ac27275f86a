// Microbenchmark: DMMA m8n8k4 latency (dependent chain) and throughput vs independent
// accumulator chains per warp and warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void kern(double* out, long long* cyc, int iters, double a, double b) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x] = s;
}
template <int CH>
void run(double* out, long long* cyc, int warps) {
  const int iters = 512;
  long long c = 0;
  for (int r = 0; r < 2; ++r) {
    kern<CH><<<1, 32 * warps>>>(out, cyc, iters, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  }
  const double per = (double)c / iters / CH;
  printf("chains %2d warps %2d: %6.2f clk per DMMA per warp  -> SM rate %.1f FMA/clk\n", CH, warps, per,
         256.0 * warps / per);
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16}) {
    run<1>(out, cyc, w);
    run<2>(out, cyc, w);
    run<4>(out, cyc, w);
    run<8>(out, cyc, w);
  }
  return 0;
}
