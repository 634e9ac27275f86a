// Microbenchmark: latencies of the operations on the Gauss-Jordan pivot-step critical path
// (dependent chains, one warp unless noted).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bar_sync_n(int id, int cnt) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(cnt) : "memory"); }

template <int V>
__global__ void kern(double* out, long long* cyc, int iters, double a, double b) {
  __shared__ double sh[1024];
  __shared__ double2 srow[32];
  const int tid = threadIdx.x;
  sh[tid] = tid * 1e-3;
  __syncthreads();
  double x = a + tid * 1e-9, y = b;
  unsigned u = tid;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (V == 0) {  // DFMA chain
      x = fma(x, y, b);
    } else if (V == 1) {  // DMUL chain
      x = x * y;
    } else if (V == 2) {  // MUFU.RCP64H chain
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(x));
    } else if (V == 3) {  // REDUX chain
      u = __reduce_max_sync(0xffffffffu, u) + 1;
    } else if (V == 4) {  // LDS chain (address from data)
      x = sh[((int)x) & 1023] + 1.0;
    } else if (V == 5) {  // bar.sync 256 threads
      bar_sync_n(1, 256);
    } else if (V == 6) {  // one lane stores 28 x 16 B, bar.sync 256, everyone loads 1
      if (tid == (i & 255)) {
#pragma unroll
        for (int j = 0; j < 28; ++j) srow[j] = make_double2(x + j, y);
      }
      bar_sync_n(1, 256);
      x += srow[i & 15].x * 1e-30;
    } else if (V == 7) {  // DFMA throughput: 8 independent chains (per-warp)
      double z0 = x, z1 = x + 1, z2 = x + 2, z3 = x + 3, z4 = x + 4, z5 = x + 5, z6 = x + 6, z7 = x + 7;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        z0 = fma(z0, y, b); z1 = fma(z1, y, b); z2 = fma(z2, y, b); z3 = fma(z3, y, b);
        z4 = fma(z4, y, b); z5 = fma(z5, y, b); z6 = fma(z6, y, b); z7 = fma(z7, y, b);
      }
      x = z0 + z1 + z2 + z3 + z4 + z5 + z6 + z7;
    } else if (V == 8) {  // DFMA throughput: 32 independent chains
      double z[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) z[c] = x + c;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 32; ++c) z[c] = fma(z[c], y, b);
      double s = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) s += z[c];
      x = s;
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  out[tid] = x + u;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 8);
  cudaMalloc(&cyc, 8);
  const char* nm[] = {"DFMA lat", "DMUL lat", "RCP64H lat", "REDUX lat", "LDS lat", "bar.sync(256)",
                      "28xSTS.128+bar+LDS", "DFMA 8ch x128 (per iter)", "DFMA 32ch x128 (per iter)"};
  const int iters = 2048;
  for (int v = 0; v < 9; ++v) {
    for (int thr : {32, 64, 128, 256}) {
      if ((v == 5 || v == 6) && thr != 256) continue;
      if (v < 5 && thr != 32) continue;
      long long c = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (v) {
          case 0: kern<0><<<1, thr>>>(out, cyc, iters, 1.0000001, 0.999999); break;
          case 1: kern<1><<<1, thr>>>(out, cyc, iters, 1.0000001, 0.999999); break;
          case 2: kern<2><<<1, thr>>>(out, cyc, iters, 1.0000001, 0.999999); break;
          case 3: kern<3><<<1, thr>>>(out, cyc, iters, 1.0000001, 0.999999); break;
          case 4: kern<4><<<1, thr>>>(out, cyc, iters, 0.0, 0.999999); break;
          case 5: kern<5><<<1, thr>>>(out, cyc, iters, 1.0000001, 0.999999); break;
          case 6: kern<6><<<1, thr>>>(out, cyc, iters, 1.0000001, 0.999999); break;
          case 7: kern<7><<<1, thr>>>(out, cyc, iters / 16, 1.0000001, 0.999999); break;
          case 8: kern<8><<<1, thr>>>(out, cyc, iters / 16, 1.0000001, 0.999999); break;
        }
        cudaDeviceSynchronize();
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      }
      const double per = v >= 7 ? (double)c / (iters / 16) / 128.0 : (double)c / iters;
      printf("%-30s threads %4d: %8.2f clk %s\n", nm[v], thr, per, v >= 7 ? "per DFMA per warp-instr-slot" : "per op");
      fflush(stdout);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
