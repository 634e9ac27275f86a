// Microbenchmark: the 4-rows x 7-columns register-blocked Gauss-Jordan panel step (as in
// zgj_ws_kernel's panel warps), 256 threads = 256 rows x 28 columns, in isolation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o panel47_bench panel47_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef double2 zt;
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
__device__ __forceinline__ unsigned pivot_key(zt f, int local) {
  const double m = f.x * f.x + f.y * f.y;
  const unsigned hi = (unsigned)(__double_as_longlong(m) >> 32);
  return (hi & ~511u) | (unsigned)(511 - local);
}
__device__ __forceinline__ void bar_sync_n(int id, int cnt) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(cnt) : "memory"); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ volatile int g_stop;
__device__ long long g_bg_iters;
// background update warps (threads 256..511): 3 DMMA only, 4 DMMA + LDS.128 fragments (3 per 8
// DMMA, as zgj_ws_kernel), 5 as 4 plus LDG/STG of the accumulators every 56 DMMAs
template <int BG>
__device__ void background(const zt* in, zt* outp, const zt* sm) {
  const int lane = threadIdx.x & 31;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  zt a = make_double2(1e-3, 2e-3), b0 = a, b1 = a;
  int it = 0;
  for (; !g_stop; ++it) {
#pragma unroll
    for (int k4 = 0; k4 < 7; ++k4) {
      if (BG >= 4) {
        a = sm[(lane & 7) * 28 + k4 * 4 + (lane >> 3)];
        b0 = sm[224 + (lane & 3) * 34 + (lane >> 2) + k4];
        b1 = sm[224 + (lane & 3) * 34 + 8 + (lane >> 2) + k4];
      }
      dmma(c[0][0], c[0][1], a.x, b0.x); dmma(c[1][0], c[1][1], a.x, b1.x);
      dmma(c[2][0], c[2][1], a.x, b0.y); dmma(c[3][0], c[3][1], a.x, b1.y);
      dmma(c[0][0], c[0][1], -a.y, b0.y); dmma(c[1][0], c[1][1], -a.y, b1.y);
      dmma(c[2][0], c[2][1], a.y, b0.x); dmma(c[3][0], c[3][1], a.y, b1.x);
      if (BG == 6) __nanosleep(32);
      if (BG == 7) __nanosleep(0);
    }
    if (BG >= 5) {
      const int idx = (threadIdx.x * 4 + it * 1024) & 8191;
      zt v = in[idx];
      c[0][0] += v.x;
      outp[256 * 64 + (idx & 4095)] = make_double2(c[0][0], c[1][1]);
    }
  }
  outp[256 * 64 + 4096 + (threadIdx.x & 255)] = make_double2(c[0][0] + c[1][0] + c[2][0] + c[3][0], c[0][1]);
  if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&g_bg_iters, (unsigned long long)it);

}

template <int MODE>  // 0 full; 1 no row update; 2 no publish (fixed pivot row); 3-5 full + background warps
__global__ void __launch_bounds__(512, 1) kern(const zt* in, zt* outp, long long* cyc, int npanels, int n) {
  __shared__ zt prow4[2][28];
  __shared__ __align__(16) unsigned wkey4[2][8];
  __shared__ zt bgsm[224 + 4 * 34 + 64];
  if (threadIdx.x < 256) {  // background = warps 0-7; panel = warps 8-15 (arbiter favours high ids)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
    if (MODE >= 3) {
      for (int i = threadIdx.x; i < 224 + 4 * 34 + 64; i += 256) bgsm[i] = in[i];
      asm volatile("bar.sync 2, 256;\n" ::: "memory");
      if (MODE == 3) background<3>(in, outp, bgsm);
      if (MODE == 4) background<4>(in, outp, bgsm);
      if (MODE == 5) background<5>(in, outp, bgsm);
      if (MODE == 6) background<6>(in, outp, bgsm);
      if (MODE == 7) background<7>(in, outp, bgsm);
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
  const int tid = threadIdx.x - 256, lane = tid & 31, wp = tid >> 5, cg = lane & 3, rg = lane >> 2;
  int rq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) rq[q] = wp * 32 + q * 8 + rg;
  const bool warp_live = wp * 32 < n;
  long long tot = 0;
  for (int pn = 0; pn < npanels; ++pn) {
    bool piv[4] = {false, false, false, false};
    zt a[4][7];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 7; ++c) a[q][c] = in[((rq[q] * 28 + cg * 7 + c) * 7 + pn) & 8191];
    bar_sync_n(1, 256);
    long long t0 = clock64();
    for (int cga = 0; cga < 4; ++cga) {
      const bool act = cg == cga;
      const int src = (lane & ~3) | cga;
#pragma unroll
      for (int s = 0; s < 7; ++s) {
        const int kk = cga * 7 + s, par = kk & 1;
        int r;
        if (MODE != 2) {
          unsigned key = 0u;
          if (act) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (!piv[q] && rq[q] < n) key = max(key, pivot_key(a[q][s], rq[q]));
          }
          key = __reduce_max_sync(0xffffffffu, key);
          if (lane == 0) wkey4[par][wp] = key;
          bar_sync_n(1, 256);
          const uint4 k03 = *reinterpret_cast<const uint4*>(&wkey4[par][0]);
          const uint4 k47 = *reinterpret_cast<const uint4*>(&wkey4[par][4]);
          const unsigned best = max(max(max(k03.x, k03.y), max(k03.z, k03.w)), max(max(k47.x, k47.y), max(k47.z, k47.w)));
          r = 511 - (int)(best & 511u);
          if (wp == (r >> 5) && rg == (r & 7)) {
            const int qq = (r >> 3) & 3;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q == qq) {
#pragma unroll
                for (int c = 0; c < 7; ++c) prow4[par][cg * 7 + c] = a[q][c];
              }
          }
          bar_sync_n(1, 256);
        } else {
          r = kk;
          if (tid < 28 && pn == 0 && kk == 0) prow4[0][tid] = in[tid], prow4[1][tid] = in[tid + 1];
          bar_sync_n(1, 256);
        }
        if (warp_live && MODE != 1) {
          const zt inv = zinv_fast(prow4[par][kk]);
          zt g[4];
          bool isp[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const zt v = a[q][s];
            g[q] = zmul(make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)), inv);
            isp[q] = rq[q] == r;
          }
          if (wp == (r >> 5)) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (isp[q]) {
                piv[q] = true;
                g[q] = make_double2(-inv.x, -inv.y);
#pragma unroll
                for (int c = 0; c < 7; ++c) a[q][c] = make_double2(0.0, 0.0);
              }
          }
#pragma unroll
          for (int c = 0; c < 7; ++c) {
            const zt pc = prow4[par][cg * 7 + c];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              a[q][c].x = fma(-g[q].x, pc.x, a[q][c].x);
              a[q][c].y = fma(-g[q].x, pc.y, a[q][c].y);
              a[q][c].x = fma(g[q].y, pc.y, a[q][c].x);
              a[q][c].y = fma(-g[q].y, pc.x, a[q][c].y);
            }
          }
          if (act) {
#pragma unroll
            for (int q = 0; q < 4; ++q) a[q][s] = make_double2(-g[q].x, -g[q].y);
          }
        } else if (MODE == 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (rq[q] == r) piv[q] = true;
        }
      }
    }
    tot += clock64() - t0;
    zt acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 7; ++c) acc.x += a[q][c].x + a[q][c].y;
    outp[tid + pn * 256] = acc;
  }
  if (tid == 0) {
    cyc[0] = tot;
    g_stop = 1;
  }
}
int main() {
  zt *in, *out;
  long long* cyc;
  cudaMalloc(&in, 8192 * sizeof(zt));
  cudaMalloc(&out, 256 * 64 * sizeof(zt));
  cudaMalloc(&cyc, 8);
  static zt h[8192];
  unsigned s = 1;
  for (int i = 0; i < 8192; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = make_double2((s >> 8) * 1e-7 - 0.8, ((s >> 4) & 0xffff) * 1e-5 - 0.3);
  }
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int np = 16;
  const char* nm[] = {"full", "no row update", "no pivot search/publish", "full + DMMA warps",
                      "full + DMMA/LDS warps", "full + DMMA/LDS/LDG warps", "  ... + nanosleep(32) per 8 DMMA",
                      "  ... + nanosleep(0) per 8 DMMA"};
  cudaMalloc(&out, (256 * 64 + 8192) * sizeof(zt));
  for (int mode = 0; mode < 8; ++mode)
    for (int n : {128, 224}) {
      long long c = 0;
      for (int r = 0; r < 2; ++r) {
        int zero = 0;
        long long z64 = 0;
        cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
        cudaMemcpyToSymbol(g_bg_iters, &z64, 8);
        if (mode == 0) kern<0><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 1) kern<1><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 2) kern<2><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 3) kern<3><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 4) kern<4><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 5) kern<5><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 6) kern<6><<<1, 512>>>(in, out, cyc, np, n);
        if (mode == 7) kern<7><<<1, 512>>>(in, out, cyc, np, n);
        cudaDeviceSynchronize();
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      }
      long long bi = 0;
      cudaMemcpyFromSymbol(&bi, g_bg_iters, 8);
      const double steps = np * 28.0;
      printf("%-34s n=%3d: %9.1f clk/step; background DMMA per step per SM %.0f (%.0f%% of pipe)\n", nm[mode], n,
             (double)c / steps, bi * 56.0 / 2 / steps, 100.0 * bi * 56.0 / 2 * 16.0 / 4 / c);
      fflush(stdout);
    }
  return 0;
}
