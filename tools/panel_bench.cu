// Microbenchmark: cost of one Gauss-Jordan panel step (register-resident rows, 256 threads),
// split into its parts.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o panel_bench panel_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef double2 zt;
constexpr int NB = 28;

__device__ __forceinline__ zt zmul(zt a, zt b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ zt zinv_fast(zt a) {
  const double d = fma(a.x, a.x, a.y * a.y);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return make_double2(a.x * r, -a.y * r);
}
template <int N>
__device__ __forceinline__ void row_rotate(zt (&row)[N]) {
  const zt t = row[0];
#pragma unroll
  for (int j = 0; j < N - 1; ++j) row[j] = row[j + 1];
  row[N - 1] = t;
}
template <int N>
__device__ __forceinline__ void row_step(zt (&row)[N], const zt* pr, zt inv) {
  const zt g = zmul(row[0], inv);
  const double ngx = -g.x, ngy = -g.y;
#pragma unroll
  for (int j = 1; j < N; ++j) {
    const zt pj = pr[j];
    row[j].x = fma(ngx, pj.x, row[j].x);
    row[j].y = fma(ngx, pj.y, row[j].y);
    row[j].x = fma(g.y, pj.y, row[j].x);
    row[j].y = fma(ngy, pj.x, row[j].y);
  }
  row[0] = make_double2(ngx, ngy);
}
__device__ __forceinline__ unsigned pivot_key(zt f, int local) {
  const double m = f.x * f.x + f.y * f.y;
  const unsigned hi = (unsigned)(__double_as_longlong(m) >> 32);
  return (hi & ~511u) | (unsigned)(511 - local);
}
__device__ __forceinline__ void bar_sync_n(int id, int cnt) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(cnt) : "memory"); }

// V: 0 full step, 1 no row update, 2 row update only (fixed pivot row), 3 full, 512 threads
// (256 idle at another barrier), 4 full without rotation (fixed slot, unrolled by 4 steps)
template <int V>
__global__ void __launch_bounds__(512, 1) kern(const zt* in, zt* outp, long long* cyc, int steps) {
  __shared__ zt wrow[2][8][NB];
  __shared__ unsigned wkey[2][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __syncthreads();
  if (tid >= 256) {
    bar_sync_n(5, 512);
    return;
  }
  zt row[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) row[j] = in[tid * NB + j];
  if (V == 2) {
    for (int j = 0; j < NB; ++j) wrow[0][0][j] = in[j];
  }
  bool pivoted = false;
  bar_sync_n(1, 256);
  long long t0 = clock64();
  long long st[4] = {0, 0, 0, 0};
  for (int k = 0; k < steps; ++k) {
    const int par = k & 1;
    long long c0 = clock64();
    if (V != 2) {
      const unsigned key = !pivoted ? pivot_key(row[0], tid) : 0u;
      const unsigned wk = __reduce_max_sync(0xffffffffu, key);
      if (wk != 0u && key == wk) {
#pragma unroll
        for (int j = 0; j < NB; ++j) wrow[par][warp][j] = row[j];
        wkey[par][warp] = wk;
      } else if (wk == 0u && lane == 0) {
        wkey[par][warp] = 0u;
      }
      long long c1 = clock64();
      st[0] += c1 - c0;
      bar_sync_n(1, 256);
      unsigned best = wkey[par][0];
      int bw = 0;
#pragma unroll
      for (int w2 = 1; w2 < 8; ++w2) {
        const unsigned kv = wkey[par][w2];
        if (kv > best) {
          best = kv;
          bw = w2;
        }
      }
      const int r = 511 - (int)(best & 511u);
      const zt* pr = wrow[par][bw];
      const zt inv = zinv_fast(pr[0]);
      long long c2 = clock64();
      st[1] += c2 - c1;
      if (tid == r) pivoted = true;
      if (V != 1) row_step<NB>(row, pr, inv);
      else row[0] = zmul(row[0], inv);
      long long c3 = clock64();
      st[2] += c3 - c2;
    } else {
      const zt* pr = wrow[0][0];
      const zt inv = zinv_fast(pr[0]);
      row_step<NB>(row, pr, inv);
    }
    row_rotate<NB>(row);
    if ((k & 255) == 255) pivoted = false;
  }
  long long t1 = clock64();
  if (tid == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = st[0];
    cyc[2] = st[1];
    cyc[3] = st[2];
  }
  zt acc = make_double2(0, 0);
#pragma unroll
  for (int j = 0; j < NB; ++j) acc.x += row[j].x + row[j].y;
  outp[tid] = acc;
  if (V == 3) bar_sync_n(5, 512);
}

int main() {
  const int steps = 1024;
  zt *in, *out;
  long long* cyc;
  cudaMalloc(&in, 256 * NB * sizeof(zt));
  cudaMalloc(&out, 512 * sizeof(zt));
  cudaMalloc(&cyc, 64);
  cudaMemset(cyc, 0, 64);
  zt h[256 * NB];
  unsigned s = 1;
  for (int i = 0; i < 256 * NB; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = make_double2((s >> 8) * 1e-7 + 0.5, ((s >> 4) & 0xffff) * 1e-5 - 0.3);
  }
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* names[] = {"full step", "no row update", "row update only", "full, +256 idle threads", ""};
  printf("start\n"); fflush(stdout);
  for (int v = 0; v < 4; ++v) {
    long long c = 0;
    for (int rep = 0; rep < 3; ++rep) {
      const int thr = v == 3 ? 512 : 256;
      if (v == 0) kern<0><<<1, thr>>>(in, out, cyc, steps);
      if (v == 1) kern<1><<<1, thr>>>(in, out, cyc, steps);
      if (v == 2) kern<2><<<1, thr>>>(in, out, cyc, steps);
      if (v == 3) kern<3><<<1, thr>>>(in, out, cyc, steps);
      cudaDeviceSynchronize();
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
    long long cs[4];
    cudaMemcpy(cs, cyc, 32, cudaMemcpyDeviceToHost);
    printf("%-28s %8.1f clk/step  [key+publish %.0f | bar+select+inv %.0f | row update %.0f] (%s)\n", names[v],
           (double)c / steps, (double)cs[1] / steps, (double)cs[2] / steps, (double)cs[3] / steps,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  return 0;
}
