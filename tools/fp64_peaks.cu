// Microbenchmark: FP64 DFMA (SIMT) and DMMA (mma.sync f64) peak throughput
// and a plain HBM read/write copy on one B200. Output: one JSON object.
// These numbers are the roofline denominators for the FP64-bound kernels
// (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma884_loop(double* out, int iters, double a0, double b0) {
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = 0; d[c][1] = threadIdx.x; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma16816_loop(double* out, int iters, double a0, double b0) {
  double d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = 0; d[c][1] = threadIdx.x; d[c][2] = 0; d[c][3] = 1; }
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = a0 + k * 1e-9;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = b0 + k * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main() {
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  printf("{\"n_sm\": %d", nsm);
  // DFMA: 8 warps/block x 4 blocks/SM, 8 independent chains
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1 << 16, threads = 256, blocks = nsm * 8;
    dfma_loop<8><<<blocks, threads>>>(out, 1000, 1.0000001, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * (double)iters * threads * blocks;
    if (rep) printf(", \"dfma_tflops\": %.3f", fl / ms / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1 << 14, threads = 256, blocks = nsm * 8;
    dmma884_loop<8><<<blocks, threads>>>(out, 100, 1.0, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma884_loop<8><<<blocks, threads>>>(out, iters, 1.0, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (threads / 32) * blocks;
    if (rep) printf(", \"dmma_m8n8k4_tflops\": %.3f", fl / ms / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 1 << 12, threads = 256, blocks = nsm * 8;
    dmma16816_loop<4><<<blocks, threads>>>(out, 100, 1.0, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma16816_loop<4><<<blocks, threads>>>(out, iters, 1.0, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 16 * 4 * (double)iters * (threads / 32) * blocks;
    if (rep) printf(", \"dmma_m16n8k16_tflops\": %.3f", fl / ms / 1e9);
  }
  {
    size_t n = (size_t)1 << 27;  // 4 GiB per buffer in double4? 2^27 * 32B = 4 GiB
    double4 *a, *b; CK(cudaMalloc(&a, n * 32)); CK(cudaMalloc(&b, n * 32));
    CK(cudaMemset(a, 0, n * 32));
    float best = 1e30;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      copy_k<<<nsm * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * n * 32 / best / 1e6);
    cudaFree(a); cudaFree(b);
  }
  printf("}\n");
  return 0;
}
