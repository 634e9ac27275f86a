// Microbenchmark: the 4 x 7 complex rank-1 register update of the Gauss-Jordan panel step
// (a[q][c] -= g[q] * p[c]) at 1..8 warps: V0 p from shared memory (broadcast LDS.128), V1 p in
// registers.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o upd_bench upd_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef double2 zt;
template <int V>
__global__ void __launch_bounds__(256, 1) kern(const zt* in, zt* out, long long* cyc, int iters) {
  __shared__ zt pr[2][28];
  const int tid = threadIdx.x;
  if (tid < 56) pr[tid / 28][tid % 28] = in[tid];
  __syncthreads();
  zt a[4][7], g[4], p[7];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    g[q] = in[q + (tid & 7)];
#pragma unroll
    for (int c = 0; c < 7; ++c) a[q][c] = in[(q * 7 + c + tid) & 63];
  }
#pragma unroll
  for (int c = 0; c < 7; ++c) p[c] = in[c + 40];
  const int cg = tid & 3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const zt pc = V == 0 ? pr[it & 1][cg * 7 + c] : p[c];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q][c].x = fma(-g[q].x, pc.x, a[q][c].x);
        a[q][c].y = fma(-g[q].x, pc.y, a[q][c].y);
        a[q][c].x = fma(g[q].y, pc.y, a[q][c].x);
        a[q][c].y = fma(-g[q].y, pc.x, a[q][c].y);
      }
    }
    if (V == 1) {
#pragma unroll
      for (int c = 0; c < 7; ++c) p[c].x += 1e-300;
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  zt s = make_double2(0, 0);
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < 7; ++c) s.x += a[q][c].x + a[q][c].y;
  out[tid] = s;
}
int main() {
  zt *in, *out;
  long long* cyc;
  cudaMalloc(&in, 128 * sizeof(zt));
  cudaMalloc(&out, 256 * sizeof(zt));
  cudaMalloc(&cyc, 8);
  zt h[128];
  for (int i = 0; i < 128; ++i) h[i] = make_double2(1e-3 * i, -1e-3 * i);
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 1000;
  for (int v = 0; v < 2; ++v)
    for (int w : {1, 2, 4, 8}) {
      long long c = 0;
      for (int r = 0; r < 2; ++r) {
        if (v == 0) kern<0><<<1, 32 * w>>>(in, out, cyc, iters);
        else kern<1><<<1, 32 * w>>>(in, out, cyc, iters);
        cudaDeviceSynchronize();
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      }
      printf("V%d (%s) warps %d: %7.1f clk/step (112 DFMA/thread)\n", v, v ? "p in regs" : "p from smem", w, (double)c / iters);
    }
  return 0;
}
