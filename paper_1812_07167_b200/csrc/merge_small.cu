// merge_small.cu — one CTA per merge for the lowest merge levels (Algorithm 1 lines 5-13,
// PAPER.md:640-666): gathers, W = I - R33b R33a, W^{-1}, Phi^a, Phi^b and R^tau of a level with
// n3 <= 28 and child boundaries nbc <= 112 in ONE launch.  On the GEMM path such a level is ~10
// launches of products with K = n3 <= 28 (14 at the level above the leaves), latency- and
// prologue-bound at 7-19 TFLOP/s; here every product is formed in shared memory by the CTA that
// needs it and the operators are written once.
//
// Same outputs, layouts and algebra as build_merge (hps_api.cu): the retained blocks R33a, R33b,
// R13a, R23b, W^{-1} (partial pivoting), Phi^a = W^{-1} [R33b R31a | -R32b],
// Phi^b = -[R31a | 0] - R33a Phi^a (the equivalent short form), and
// R^tau = diag(R11a, R22b) + [R13a Phi^a ; R23b Phi^b] scattered to canonical order through pp.
#include <algorithm>

#include "hps_internal.cuh"

namespace {

__device__ __forceinline__ zt zmul(zt a, zt b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ void zmac(zt& acc, zt a, zt b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ zt zinv(zt a) {
  const double d = 1.0 / fma(a.x, a.x, a.y * a.y);
  return make_double2(a.x * d, -a.y * d);
}

constexpr int MS_T = 256;   // threads per CTA
constexpr int MS_TW = 16;   // column tile of Phi / R^tau

__global__ void __launch_bounds__(MS_T) merge_small_kernel(const MergeSmallArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n3 = a.n3, n1 = a.n1, n2 = a.n2, nt = a.ntau, nbc = a.nbc, tid = threadIdx.x, b = blockIdx.x;
  zt* sR33a = reinterpret_cast<zt*>(smem_raw);  // [n3][n3]
  zt* sR33b = sR33a + n3 * n3;                  // [n3][n3]
  zt* sW = sR33b + n3 * n3;                     // [n3][2 n3]: [W | I] -> [I | W^{-1}]
  zt* sR13a = sW + 2 * n3 * n3;                 // [n1][n3]
  zt* sR23b = sR13a + n1 * n3;                  // [n2][n3]
  zt* sG = sR23b + n2 * n3;                     // [n3][TW]  gathered R31a columns
  zt* sX = sG + n3 * MS_TW;                     // [n3][TW]
  zt* sPA = sX + n3 * MS_TW;                    // [n3][TW]
  zt* sPB = sPA + n3 * MS_TW;                   // [n3][TW]
  __shared__ int s_piv;
  __shared__ double s_pmax[1];
  const zt* Ra = a.R + (int64_t)(2 * b) * nbc * nbc;
  const zt* Rb = Ra + (int64_t)nbc * nbc;
  // ---- (a) retained child blocks, also written out ----
  for (int e = tid; e < n3 * n3; e += MS_T) {
    const int i = e / n3, j = e - i * n3;
    const zt va = Ra[(int64_t)a.I3a[i] * nbc + a.I3a[j]], vb = Rb[(int64_t)a.I3b[i] * nbc + a.I3b[j]];
    sR33a[e] = va;
    sR33b[e] = vb;
    a.R33a[(int64_t)b * n3 * n3 + e] = va;
    a.R33b[(int64_t)b * n3 * n3 + e] = vb;
  }
  for (int e = tid; e < n1 * n3; e += MS_T) {
    const int i = e / n3, j = e - i * n3;
    const zt v = Ra[(int64_t)a.I1a[i] * nbc + a.I3a[j]];
    sR13a[e] = v;
    a.R13a[(int64_t)b * n1 * n3 + e] = v;
  }
  for (int e = tid; e < n2 * n3; e += MS_T) {
    const int i = e / n3, j = e - i * n3;
    const zt v = Rb[(int64_t)a.I2b[i] * nbc + a.I3b[j]];
    sR23b[e] = v;
    a.R23b[(int64_t)b * n2 * n3 + e] = v;
  }
  __syncthreads();
  // ---- (b) W = I - R33b R33a, as [W | I] (line 7) ----
  for (int e = tid; e < n3 * n3; e += MS_T) {
    const int i = e / n3, j = e - i * n3;
    zt acc = make_double2(0.0, 0.0);
    for (int k = 0; k < n3; ++k) zmac(acc, sR33b[i * n3 + k], sR33a[k * n3 + j]);
    sW[i * 2 * n3 + j] = make_double2((i == j ? 1.0 : 0.0) - acc.x, -acc.y);
    sW[i * 2 * n3 + n3 + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  // ---- (c) W^{-1} by Gauss-Jordan with partial pivoting on [W | I] (reading Q10) ----
  const int w2 = 2 * n3;
  bool singular = false;
  for (int k = 0; k < n3; ++k) {
    if (tid < 32) {  // pivot search over rows k .. n3-1 by warp 0
      double best = -1.0;
      int bi = k;
      for (int r = k + tid; r < n3; r += 32) {
        const zt v = sW[r * w2 + k];
        const double m = fma(v.x, v.x, v.y * v.y);
        if (m > best) {
          best = m;
          bi = r;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (tid == 0) {
        s_piv = bi;
        s_pmax[0] = best;
      }
    }
    __syncthreads();
    const int r = s_piv;
    if (!(s_pmax[0] > 0.0)) singular = true;
    if (r != k)  // swap rows k and r
      for (int j = tid; j < w2; j += MS_T) {
        const zt t = sW[k * w2 + j];
        sW[k * w2 + j] = sW[r * w2 + j];
        sW[r * w2 + j] = t;
      }
    __syncthreads();
    const zt inv = zinv(sW[k * w2 + k]);
    // row k scaled (after every thread has read the pivot); every other row i: row_i -= W[i][k] row_k
    zt* rk = sW + k * w2;
    __syncthreads();
    for (int j = tid; j < w2; j += MS_T) rk[j] = zmul(rk[j], inv);
    __syncthreads();
    for (int e = tid; e < n3 * w2; e += MS_T) {
      const int i = e / w2, j = e - i * w2;
      if (i == k || j == k) continue;
      const zt f = sW[i * w2 + k];
      zt v = sW[e];
      const zt p = rk[j];
      v.x = fma(-f.x, p.x, fma(f.y, p.y, v.x));
      v.y = fma(-f.x, p.y, fma(-f.y, p.x, v.y));
      sW[e] = v;
    }
    __syncthreads();
    for (int i = tid; i < n3; i += MS_T)
      if (i != k) sW[i * w2 + k] = make_double2(0.0, 0.0);
    __syncthreads();
  }
  if (singular && tid == 0) atomicCAS(a.info, 0, 1);
  // W^{-1} = right half; written out (the solve applies it)
  for (int e = tid; e < n3 * n3; e += MS_T) {
    const int i = e / n3, j = e - i * n3;
    a.Winv[(int64_t)b * n3 * n3 + e] = sW[i * w2 + n3 + j];
  }
  // ---- (d)-(f) per column tile J of [I1, I2] order ----
  const zt* Wi = sW + n3;  // row stride w2
  zt* PhiA = a.PhiA + (int64_t)b * n3 * nt;
  zt* PhiB = a.PhiB + (int64_t)b * n3 * nt;
  zt* Rt = a.Rtau ? a.Rtau + (int64_t)b * nt * nt : nullptr;
  for (int j0 = 0; j0 < nt; j0 += MS_TW) {
    const int tw = min(MS_TW, nt - j0);
    __syncthreads();  // the previous tile's buffers are consumed
    // G = R31a(:, J) for J in I1 (zero in I2)
    for (int e = tid; e < n3 * MS_TW; e += MS_T) {
      const int i = e / MS_TW, jj = e - i * MS_TW, j = j0 + jj;
      sG[e] = (jj < tw && j < n1) ? Ra[(int64_t)a.I3a[i] * nbc + a.I1a[j]] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    // X = [R33b R31a | -R32b]  (line 8)
    for (int e = tid; e < n3 * MS_TW; e += MS_T) {
      const int i = e / MS_TW, jj = e - i * MS_TW, j = j0 + jj;
      zt v = make_double2(0.0, 0.0);
      if (jj < tw) {
        if (j < n1) {
          for (int k = 0; k < n3; ++k) zmac(v, sR33b[i * n3 + k], sG[k * MS_TW + jj]);
        } else {
          const zt r = Rb[(int64_t)a.I3b[i] * nbc + a.I2b[j - n1]];
          v = make_double2(-r.x, -r.y);
        }
      }
      sX[e] = v;
    }
    __syncthreads();
    // Phi^a = W^{-1} X
    for (int e = tid; e < n3 * MS_TW; e += MS_T) {
      const int i = e / MS_TW, jj = e - i * MS_TW;
      zt v = make_double2(0.0, 0.0);
      for (int k = 0; k < n3; ++k) zmac(v, Wi[i * w2 + k], sX[k * MS_TW + jj]);
      sPA[e] = v;
      if (jj < tw) PhiA[(int64_t)i * nt + j0 + jj] = v;
    }
    __syncthreads();
    // Phi^b = -[R31a | 0] - R33a Phi^a  (line 10, short form)
    for (int e = tid; e < n3 * MS_TW; e += MS_T) {
      const int i = e / MS_TW, jj = e - i * MS_TW;
      zt v = make_double2(0.0, 0.0);
      for (int k = 0; k < n3; ++k) zmac(v, sR33a[i * n3 + k], sPA[k * MS_TW + jj]);
      v = make_double2(-v.x - sG[e].x, -v.y - sG[e].y);
      sPB[e] = v;
      if (jj < tw) PhiB[(int64_t)i * nt + j0 + jj] = v;
    }
    __syncthreads();
    if (!Rt) continue;
    // R^tau(:, J) = diag(R11a, R22b)(:, J) + [R13a Phi^a ; R23b Phi^b](:, J), canonical order (line 12)
    for (int e = tid; e < (n1 + n2) * MS_TW; e += MS_T) {
      const int i = e / MS_TW, jj = e - i * MS_TW, j = j0 + jj;
      if (jj >= tw) continue;
      zt v = make_double2(0.0, 0.0), v1 = v;
      if (i < n1) {
        const zt* ar = sR13a + i * n3;
        int k = 0;
        for (; k + 1 < n3; k += 2) {
          zmac(v, ar[k], sPA[k * MS_TW + jj]);
          zmac(v1, ar[k + 1], sPA[(k + 1) * MS_TW + jj]);
        }
        if (k < n3) zmac(v, ar[k], sPA[k * MS_TW + jj]);
        if (j < n1) {
          const zt r = Ra[(int64_t)a.I1a[i] * nbc + a.I1a[j]];
          v.x += r.x;
          v.y += r.y;
        }
      } else {
        const zt* br = sR23b + (i - n1) * n3;
        int k = 0;
        for (; k + 1 < n3; k += 2) {
          zmac(v, br[k], sPB[k * MS_TW + jj]);
          zmac(v1, br[k + 1], sPB[(k + 1) * MS_TW + jj]);
        }
        if (k < n3) zmac(v, br[k], sPB[k * MS_TW + jj]);
        if (j >= n1) {
          const zt r = Rb[(int64_t)a.I2b[i - n1] * nbc + a.I2b[j - n1]];
          v.x += r.x;
          v.y += r.y;
        }
      }
      v.x += v1.x;
      v.y += v1.y;
      Rt[(int64_t)a.pp[i] * nt + a.pp[j]] = v;
    }
  }
}

}  // namespace

size_t merge_small_smem(int n3, int n1, int n2) {
  return sizeof(zt) * ((size_t)4 * n3 * n3 + (size_t)(n1 + n2) * n3 + (size_t)4 * n3 * MS_TW);
}

bool merge_small_applies(int n3, int n1, int n2) { return n3 <= 28 && merge_small_smem(n3, n1, n2) <= 160 * 1024; }

void launch_merge_small(const MergeSmallArgs& a, int np, cudaStream_t st) {
  const size_t smem = merge_small_smem(a.n3, a.n1, a.n2);
  static bool attr = false;
  if (!attr) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(merge_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  const double n3 = a.n3, n1 = a.n1, nt = a.ntau;
  ProfScope ps(K_GJ_FUSED,
               8.0 * np * (2.0 * n3 * n3 * n3 + n3 * n3 * n1 + 2.0 * n3 * n3 * nt + (a.Rtau ? nt * nt * n3 : 0.0)),
               16.0 * np * (2.0 * a.nbc * a.nbc + 2.0 * n3 * nt + 3.0 * n3 * n3 + 2.0 * n1 * n3 + (a.Rtau ? nt * nt : 0.0)),
               st);
  for (int b0 = 0; b0 < np; b0 += 65535) {
    MergeSmallArgs c = a;
    const int nb = std::min(65535, np - b0);
    c.R = a.R + (int64_t)2 * b0 * a.nbc * a.nbc;
    c.R33a = a.R33a + (int64_t)b0 * a.n3 * a.n3;
    c.R33b = a.R33b + (int64_t)b0 * a.n3 * a.n3;
    c.R13a = a.R13a + (int64_t)b0 * a.n1 * a.n3;
    c.R23b = a.R23b + (int64_t)b0 * a.n2 * a.n3;
    c.Winv = a.Winv + (int64_t)b0 * a.n3 * a.n3;
    c.PhiA = a.PhiA + (int64_t)b0 * a.n3 * a.ntau;
    c.PhiB = a.PhiB + (int64_t)b0 * a.n3 * a.ntau;
    c.Rtau = a.Rtau ? a.Rtau + (int64_t)b0 * a.ntau * a.ntau : nullptr;
    merge_small_kernel<<<nb, MS_T, smem, st>>>(c);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
}
