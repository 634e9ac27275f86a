// Integer-slice form of the big complex products (knob `gemm_slices` = s, default 0 = off; DESIGN.md 11,
// "beyond the FP64 tensor roof").  The merge products of Algorithm 1 are
// FP64 products; this file forms the same product from s signed 7-bit slices per real operand:
//
//   3M form (DESIGN 3.14):  T1 = A_r B_r,  T2 = A_i B_i,  T3 = (A_r + A_i)(B_r + B_i)
//   each real product X Y:  X = 2^ex(row) * sum_i X_i 128^-(i+1),  Y = 2^ey(col) * sum_j Y_j 128^-(j+1),
//                           X_i, Y_j integer in [-64, 64] (exact remainders), and
//                           X Y ~= 2^(ex+ey) * sum_{w<s} 128^-(w+2) * sum_{i+j=w} X_i Y_j^T
//
// The slice products X_i Y_j^T are exact in int32 (4096 K s < 2^31) and run on the INT8 tensor path
// through the cuBLASLt library GEMM (s8 x s8 -> s32, a plain library GEMM; loaded with dlopen on
// first use, so libhps has no link-time dependency and falls back to its own DMMA kernels when the
// library is not there).  The slicing kernel (operands read through the ZOp maps) and the folding
// kernel (weights summed in FP64 from the smallest up, alpha / beta Cin / diag, ZOut maps) are ours.
// Dropped terms (i + j >= s) bound the error at ~s 2^(-7 s + 2) relative to |X||Y| per row / column
// scale: 3e-13 at s = 7, 3e-15 at s = 8 (tools/ozaki_probe.py, profiles/r02_ozaki_probe.txt).
// Off by default: the default path runs only this repo's kernels.
#include <cublasLt.h>
#include <dlfcn.h>

#include <cstdio>
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "hps_internal.cuh"

namespace {

__device__ __forceinline__ zt zmul(zt a, zt b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }

struct Lt {
  void* so = nullptr;
  cublasLtHandle_t h = nullptr;
  bool ok = false;
  decltype(&cublasLtCreate) create = nullptr;
  decltype(&cublasLtMatmulDescCreate) desc_create = nullptr;
  decltype(&cublasLtMatmulDescSetAttribute) desc_set = nullptr;
  decltype(&cublasLtMatmulDescDestroy) desc_destroy = nullptr;
  decltype(&cublasLtMatrixLayoutCreate) lay_create = nullptr;
  decltype(&cublasLtMatrixLayoutDestroy) lay_destroy = nullptr;
  decltype(&cublasLtMatmulPreferenceCreate) pref_create = nullptr;
  decltype(&cublasLtMatmulPreferenceSetAttribute) pref_set = nullptr;
  decltype(&cublasLtMatmulPreferenceDestroy) pref_destroy = nullptr;
  decltype(&cublasLtMatmulAlgoGetHeuristic) heur = nullptr;
  decltype(&cublasLtMatmul) matmul = nullptr;
};

std::mutex g_lt_mu;
Lt g_lt;
bool g_lt_tried = false;

template <class F>
bool sym(void* so, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(so, name));
  return f != nullptr;
}

Lt* lt() {
  std::lock_guard<std::mutex> lk(g_lt_mu);
  if (g_lt_tried) return g_lt.ok ? &g_lt : nullptr;
  g_lt_tried = true;
  for (const char* n : {"libcublasLt.so.12", "/usr/local/cuda/lib64/libcublasLt.so.12", "libcublasLt.so"}) {
    g_lt.so = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    if (g_lt.so) break;
  }
  if (!g_lt.so) {
    fprintf(stderr, "[hps] gemm_slices: cuBLASLt not found (%s); DMMA products used\n", dlerror());
    return nullptr;
  }
  Lt& L = g_lt;
  bool ok = sym(L.so, "cublasLtCreate", L.create) && sym(L.so, "cublasLtMatmulDescCreate", L.desc_create) &&
            sym(L.so, "cublasLtMatmulDescSetAttribute", L.desc_set) &&
            sym(L.so, "cublasLtMatmulDescDestroy", L.desc_destroy) &&
            sym(L.so, "cublasLtMatrixLayoutCreate", L.lay_create) &&
            sym(L.so, "cublasLtMatrixLayoutDestroy", L.lay_destroy) &&
            sym(L.so, "cublasLtMatmulPreferenceCreate", L.pref_create) &&
            sym(L.so, "cublasLtMatmulPreferenceSetAttribute", L.pref_set) &&
            sym(L.so, "cublasLtMatmulPreferenceDestroy", L.pref_destroy) &&
            sym(L.so, "cublasLtMatmulAlgoGetHeuristic", L.heur) && sym(L.so, "cublasLtMatmul", L.matmul);
  if (ok) ok = L.create(&L.h) == CUBLAS_STATUS_SUCCESS;
  if (!ok) fprintf(stderr, "[hps] gemm_slices: cuBLASLt symbols / handle unavailable; DMMA products used\n");
  L.ok = ok;
  return ok ? &L : nullptr;
}

// One s8 x s8 -> s32 product shape: D^T (N x M, column-major, ld N) = Y8 (Kk x N, ld)^T X8 (Kk x M, ld)
struct LtPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo;
  size_t ws = 0;
  bool ok = false;
};
constexpr size_t kLtWs = 64u << 20;
std::map<std::tuple<int, int, int, int, int>, LtPlan> g_plans;

LtPlan* lt_plan(Lt& L, int M, int N, int Kp, int ld) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_lt_mu);
  auto key = std::make_tuple(dev, M, N, Kp, ld);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return it->second.ok ? &it->second : nullptr;
  LtPlan& P = g_plans[key];
  const cublasOperation_t tr = CUBLAS_OP_T, nt = CUBLAS_OP_N;
  bool ok = L.desc_create(&P.op, CUBLAS_COMPUTE_32I, CUDA_R_32I) == CUBLAS_STATUS_SUCCESS &&
            L.desc_set(P.op, CUBLASLT_MATMUL_DESC_TRANSA, &tr, sizeof(tr)) == CUBLAS_STATUS_SUCCESS &&
            L.desc_set(P.op, CUBLASLT_MATMUL_DESC_TRANSB, &nt, sizeof(nt)) == CUBLAS_STATUS_SUCCESS &&
            L.lay_create(&P.a, CUDA_R_8I, Kp, N, ld) == CUBLAS_STATUS_SUCCESS &&
            L.lay_create(&P.b, CUDA_R_8I, Kp, M, ld) == CUBLAS_STATUS_SUCCESS &&
            L.lay_create(&P.c, CUDA_R_32I, N, M, N) == CUBLAS_STATUS_SUCCESS;
  if (ok) {
    cublasLtMatmulPreference_t pref = nullptr;
    ok = L.pref_create(&pref) == CUBLAS_STATUS_SUCCESS;
    if (ok) {
      size_t ws = kLtWs;
      L.pref_set(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof(ws));
      cublasLtMatmulHeuristicResult_t res;
      int found = 0;
      ok = L.heur(L.h, P.op, P.a, P.b, P.c, P.c, pref, 1, &res, &found) == CUBLAS_STATUS_SUCCESS && found > 0;
      if (ok) {
        P.algo = res.algo;
        P.ws = res.workspaceSize;
      }
      L.pref_destroy(pref);
    }
  }
  if (!ok) fprintf(stderr, "[hps] gemm_slices: no s8 algorithm for %d x %d x %d; DMMA product used\n", M, N, Kp);
  P.ok = ok;
  return ok ? &P : nullptr;
}

// ---------------------------------------------------------------------------------------------
// Slicing: one CTA per kept index r (row i of A, or column j of B); the reduced index is k.
//   planes [3][R][s][Kp] int8 (k fastest: the "TN" operand layout of the s8 GEMM), exps [3][R].  Row r
//   holds its slices side by side -- A: X_0 .. X_{s-1}, B: Y_{s-1} .. Y_0 -- so that the equal-weight
//   sum  sum_{i+j=w} X_i Y_j^T  is ONE product over the concatenated index: the first (w + 1) Kp entries
//   of an A row against the last (w + 1) Kp entries of a B row (s products per real product, each
//   written once, instead of s (s + 1) / 2 accumulated ones).
// ---------------------------------------------------------------------------------------------
template <bool IS_B>
__device__ __forceinline__ zt slice_elem(const ZGemm& g, const zt* base, const int* rm, int r, int k) {
  int ri, cj;
  if (IS_B) {
    ri = rm ? rm[k] : k;  // B rows follow the row map only (as in the tiled kernel)
    cj = zcol(g.B.cmap, r, g.B.cskip_at, g.B.cskip_len);
    if (ri < 0 || cj < 0) return make_double2(0.0, 0.0);
    return base[(int64_t)ri * g.B.rs + (int64_t)cj * g.B.cs];
  }
  ri = zrow(g.A, rm, r);
  cj = zcol(g.A.cmap, k, g.A.cskip_at, g.A.cskip_len);
  if (ri < 0 || cj < 0) return make_double2(0.0, 0.0);
  return base[(int64_t)ri * g.A.rs + (int64_t)cj * g.A.cs];
}

__device__ __forceinline__ int slice_exp(double m) {  // |x| <= m  =>  |x / 2^e| < 1/2
  if (!(m > 0.0)) return 0;
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return e + 1;
}

template <bool IS_B>
__global__ void __launch_bounds__(256) zslice_kernel(const ZGemm g, int b, int R, int Kp, int s, int8_t* planes, int* exps) {
  __shared__ double red[3][8];
  __shared__ int se[3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const zt* base = IS_B ? g.B.ptr + zboff(g.B, b) : g.A.ptr + zboff(g.A, b);
  const ZOp& op = IS_B ? g.B : g.A;
  const int* rm = op.rmap ? op.rmap + (int64_t)b * op.rmap_bs : nullptr;
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    double m0 = 0.0, m1 = 0.0, m2 = 0.0;
    for (int k = tid; k < g.K; k += 256) {
      const zt v = slice_elem<IS_B>(g, base, rm, r, k);
      m0 = fmax(m0, fabs(v.x));
      m1 = fmax(m1, fabs(v.y));
      m2 = fmax(m2, fabs(v.x + v.y));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
      m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
      m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    }
    if (lane == 0) {
      red[0][warp] = m0;
      red[1][warp] = m1;
      red[2][warp] = m2;
    }
    __syncthreads();
    if (tid < 3) {
      double m = 0.0;
      for (int w = 0; w < 8; ++w) m = fmax(m, red[tid][w]);
      const int e = slice_exp(m);
      se[tid] = e;
      exps[(int64_t)tid * R + r] = e;
    }
    __syncthreads();
    const int e0 = se[0], e1 = se[1], e2 = se[2];
    // four consecutive k per thread: one 4-byte store per plane
    for (int k4 = tid * 4; k4 < Kp; k4 += 256 * 4) {
      double y[3][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k4 + q;
        zt v = make_double2(0.0, 0.0);
        if (k < g.K) v = slice_elem<IS_B>(g, base, rm, r, k);
        y[0][q] = ldexp(v.x, -e0);
        y[1][q] = ldexp(v.y, -e1);
        y[2][q] = ldexp(v.x + v.y, -e2);
      }
      for (int i = 0; i < s; ++i) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          char4 c;
          signed char* cp = reinterpret_cast<signed char*>(&c);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double z = y[t][q] * 128.0;
            const double rq = rint(z);
            cp[q] = (signed char)(int)rq;
            y[t][q] = z - rq;  // exact: |z| <= 64, the remainder keeps every remaining bit
          }
          const int slot = IS_B ? s - 1 - i : i;
          *reinterpret_cast<char4*>(planes + (((int64_t)t * R + r) * s + slot) * Kp + k4) = c;
        }
      }
    }
    __syncthreads();
  }
}

// Folding: C(i, j) = alpha * (T1 - T2, T3 - T1 - T2) + beta * Cin(i, j) + diag [i == j],
//   T_t = 2^(eA[t][i] + eB[t][j]) * sum_{w = s-1 .. 0} 128^-(w + 2) * acc[t][w](i, j)
__global__ void __launch_bounds__(256) zfold_kernel(const ZGemm g, int b, int s, const int* acc, const int* eA, const int* eB) {
  const int64_t mn = (int64_t)g.M * g.N;
  const int* Crm = g.C.rmap ? g.C.rmap + (int64_t)b * g.C.rmap_bs : nullptr;
  const int* Irm = g.Cin.rmap ? g.Cin.rmap + (int64_t)b * g.Cin.rmap_bs : nullptr;
  zt* Cb = g.C.ptr + zboff(g.C, b);
  const zt* Ib = g.Cin.ptr ? g.Cin.ptr + zboff(g.Cin, b) : nullptr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / g.N), j = (int)(e - (int64_t)i * g.N);
    const int ro = zrow(g.C, Crm, i), co = zcol(g.C.cmap, j, g.C.cskip_at, g.C.cskip_len);
    if (ro < 0 || co < 0) continue;
    double T[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      double a = 0.0;
      for (int w = s - 1; w >= 0; --w) a += ldexp((double)acc[((int64_t)t * s + w) * mn + e], -7 * (w + 2));
      T[t] = ldexp(a, eA[(int64_t)t * g.M + i] + eB[(int64_t)t * g.N + j]);
    }
    zt v = zmul(g.alpha, make_double2(T[0] - T[1], (T[2] - T[0]) - T[1]));
    if (Ib) {
      const int ri = zrow(g.Cin, Irm, i), ci = zcol(g.Cin.cmap, j, g.Cin.cskip_at, g.Cin.cskip_len);
      if (ri >= 0 && ci >= 0) {
        const zt w = zmul(g.beta, Ib[(int64_t)ri * g.Cin.rs + (int64_t)ci * g.Cin.cs]);
        v.x += w.x;
        v.y += w.y;
      }
    }
    if (i == j) {
      v.x += g.diag.x;
      v.y += g.diag.y;
    }
    Cb[(int64_t)ro * g.C.rs + (int64_t)co * g.C.cs] = v;
  }
}

}  // namespace

// Returns false when the shape is not eligible or the library is unavailable (the caller then runs
// the DMMA product).  Everything is enqueued on st; the workspaces are stream-ordered allocations.
bool zgemm_slices(const ZGemm& g, cudaStream_t st) {
  const int s = knob(KN_GEMM_SLICES), mn_min = knob(KN_GEMM_SLICES_MIN);
  if (s < 2 || s > 9) return false;
  if (g.M < mn_min || g.N < mn_min || g.K < mn_min || (g.N & 3) || g.batch > 64 || g.ksplit > 1) return false;
  const int Kp = (g.K + 15) / 16 * 16;
  if (4096.0 * Kp * s >= 2147483648.0) return false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return false;
  Lt* L = lt();
  if (!L) return false;
  LtPlan* P[9];
  size_t lws = 1;
  for (int w = 0; w < s; ++w) {
    P[w] = lt_plan(*L, g.M, g.N, (w + 1) * Kp, s * Kp);
    if (!P[w]) return false;
    lws = std::max(lws, P[w]->ws);
  }

  const size_t a8 = (size_t)3 * s * g.M * Kp, b8 = (size_t)3 * s * g.N * Kp;
  const size_t accb = sizeof(int) * (size_t)3 * s * g.M * g.N;
  const size_t eb = sizeof(int) * (size_t)3 * (g.M + g.N);
  auto up = [](size_t v) { return (v + 255) / 256 * 256; };
  char* ws = nullptr;
  const size_t total = up(a8) + up(b8) + up(accb) + up(eb) + up(lws);
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), total, st) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int8_t* A8 = reinterpret_cast<int8_t*>(ws);
  int8_t* B8 = reinterpret_cast<int8_t*>(ws + up(a8));
  int* acc = reinterpret_cast<int*>(ws + up(a8) + up(b8));
  int* eA = reinterpret_cast<int*>(ws + up(a8) + up(b8) + up(accb));
  int* eB = eA + (size_t)3 * g.M;
  void* ltws = ws + up(a8) + up(b8) + up(accb) + up(eb);
  const int one = 1, zero = 0;
  const int fold_grid = (int)std::min<int64_t>(((int64_t)g.M * g.N + 255) / 256, (int64_t)hps_num_sms() * 16);
  bool ok = true;
  int folded = 0;
  for (int b = 0; b < g.batch && ok; ++b) {
    zslice_kernel<false><<<g.M, 256, 0, st>>>(g, b, g.M, Kp, s, A8, eA);
    zslice_kernel<true><<<g.N, 256, 0, st>>>(g, b, g.N, Kp, s, B8, eB);
    for (int t = 0; t < 3 && ok; ++t)
      for (int w = 0; w < s && ok; ++w) {
        const int8_t* X = A8 + (size_t)t * g.M * s * Kp;                           // rows [X_0 .. X_w | ...]
        const int8_t* Y = B8 + (size_t)t * g.N * s * Kp + (size_t)(s - 1 - w) * Kp;  // rows [... | Y_w .. Y_0]
        int* D = acc + ((size_t)t * s + w) * g.M * g.N;                            // [M][N] = column-major N x M
        ok = L->matmul(L->h, P[w]->op, &one, Y, P[w]->a, X, P[w]->b, &zero, D, P[w]->c, D, P[w]->c, &P[w]->algo, ltws,
                       P[w]->ws, st) == CUBLAS_STATUS_SUCCESS;
      }
    if (ok) {
      zfold_kernel<<<fold_grid, 256, 0, st>>>(g, b, s, acc, eA, eB);
      ++folded;
    }
  }
  cudaFreeAsync(ws, st);
  if (!ok) {
    // before the first fold C is untouched and the caller's DMMA product takes over; after it C may
    // already hold results that alias Cin (in-place updates), so a redo would be wrong: fail loudly
    if (folded) throw HpsError{-4, "gemm_slices: cublasLtMatmul failed after part of the batch was written"};
    fprintf(stderr, "[hps] gemm_slices: cublasLtMatmul failed (%d x %d x %d); DMMA product used\n", g.M, g.N, g.K);
    return false;
  }
  HPS_CUDA_CHECK(cudaGetLastError());
  return true;
}
