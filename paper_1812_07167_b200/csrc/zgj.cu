// zgj.cu — batched explicit inverse by Gauss-Jordan elimination with partial pivoting.
//
// Used for the leaf matrix B (Psi and Y are the column blocks of B^{-1},
// reading Q11) and for W = I - R33b R33a of every merge (the paper stores
// W^{-1} explicitly, computed there by zgetrf + zgetri).
// Gauss-Jordan costs the same n^3 complex multiply-adds as LU + triangular inverse and has a
// full-height trailing update, which maps onto the DMMA GEMM (zgemm.cu).
//
// In-place GJ step k (row pivoting):  r = argmax_{i>=k} |A(i,k)|; swap rows k, r;
//   row k <- row k / A(k,k) with A(k,k) <- 1/A(k,k);  for i != k: A(i,:) -= A(i,k) * row k
//   (with A(i,k) reset to 0 first, so it ends as -A(i,k)/pivot).  After the last step the
//   column swaps are undone in reverse order: out(:, j) = A(:, pi(j)).
// Blocked form (n > kSmallMax): panel of nb columns factored by one thread-block cluster
// (rows of the panel distributed over the cluster's shared memory, pivot search and pivot row
// exchanged through distributed shared memory), then for every other column j:
//   apply the panel's row swaps, Z = A(panel rows, j), A(panel rows, j) = 0,
//   A(:, j) += T Z   with T = the panel's stored transform columns   (DMMA GEMM).
#include <cooperative_groups.h>

#include <algorithm>

#include "hps_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kSmallMax = 112;  // whole matrix in shared memory: 112*113*16 B = 202 KB
constexpr int kThreads = 256;

__device__ __forceinline__ double zabs2(zt a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ zt zmul(zt a, zt b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ zt zinv(zt a) {
  const double d = a.x * a.x + a.y * a.y;
  return make_double2(a.x / d, -a.y / d);
}

// argmax reduction helper: larger value wins, ties -> smaller index
__device__ __forceinline__ void amax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

// ---------------------------------------------------------------------------
// Small: one CTA per matrix, whole matrix in shared memory.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) zgj_small_kernel(const zt* __restrict__ A, int64_t lda, int64_t bs,
                                                             zt* __restrict__ out, int64_t ldo, int64_t obs, int n,
                                                             int* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = n + 1;
  zt* M = reinterpret_cast<zt*>(smem_raw);  // n x ld
  zt* col = M + n * ld;                       // n
  zt* prow = col + n;                         // n (scaled pivot row)
  int* piv = reinterpret_cast<int*>(prow + n);  // n
  __shared__ int s_r;
  __shared__ zt s_inv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const zt* Ab = A + (int64_t)b * bs;
  for (int e = tid; e < n * n; e += kThreads) {
    const int i = e / n, j = e % n;
    M[i * ld + j] = Ab[(int64_t)i * lda + j];
  }
  __syncthreads();
  bool singular = false;
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double bv = -1.0;
      int bi = k;
      for (int i = k + lane; i < n; i += 32) amax_merge(bv, bi, zabs2(M[i * ld + k]), i);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        amax_merge(bv, bi, v2, i2);
      }
      if (lane == 0) {
        s_r = bi;
        piv[k] = bi;
        if (bv == 0.0) singular = true;
        s_inv = zinv(M[bi * ld + k]);
      }
    }
    __syncthreads();
    const int r = s_r;
    const zt inv = s_inv;
    // swap rows k and r; scaled pivot row into prow; save column k
    for (int j = tid; j < n; j += kThreads) {
      const zt vr = M[r * ld + j];
      if (r != k) M[r * ld + j] = M[k * ld + j];
      prow[j] = (j == k) ? inv : zmul(vr, inv);
    }
    __syncthreads();
    for (int i = tid; i < n; i += kThreads) {
      col[i] = (i == k) ? make_double2(0.0, 0.0) : M[i * ld + k];
      if (i != k) M[i * ld + k] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    // rank-1 update of all rows but k; row k <- prow
    for (int i = warp; i < n; i += kThreads / 32) {
      if (i == k) {
        for (int j = lane; j < n; j += 32) M[k * ld + j] = prow[j];
      } else {
        const zt f = col[i];
        for (int j = lane; j < n; j += 32) {
          zt a = M[i * ld + j];
          const zt pj = prow[j];
          a.x -= f.x * pj.x - f.y * pj.y;
          a.y -= f.x * pj.y + f.y * pj.x;
          M[i * ld + j] = a;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (singular) atomicCAS(info, 0, b + 1);
    // pi = S_{n-1} o ... o S_0 as an array: right-compose swaps for k = n-1 .. 0
    int* pi = reinterpret_cast<int*>(col);  // reuse
    for (int j = 0; j < n; ++j) pi[j] = j;
    for (int k = n - 1; k >= 0; --k) {
      const int t = pi[k];
      pi[k] = pi[piv[k]];
      pi[piv[k]] = t;
    }
  }
  __syncthreads();
  const int* pi = reinterpret_cast<const int*>(col);
  zt* ob = out + (int64_t)b * obs;
  for (int e = tid; e < n * n; e += kThreads) {
    const int i = e / n, j = e % n;
    ob[(int64_t)i * ldo + j] = M[i * ld + pi[j]];
  }
}

// ---------------------------------------------------------------------------
// Blocked: cluster panel factorisation.  Cluster = CS CTAs per matrix; CTA c owns panel rows
// [c*RP, min(n, (c+1)*RP)).  Shared: P[RP][nb], prow[nb], tmp[nb], slot (val, idx).
// ---------------------------------------------------------------------------
struct Slot {
  double v;
  int i;
  int pad;
};

__global__ void __launch_bounds__(kThreads) zgj_panel_kernel(zt* A, int64_t lda, int64_t bs, int n, int k0, int nb,
                                                             int RP, int* piv_all, int* info) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int b = blockIdx.x / CS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zt* P = reinterpret_cast<zt*>(smem_raw);  // RP x nb
  zt* prow = P + RP * nb;                   // nb
  zt* tmp = prow + nb;                      // nb
  Slot* slot = reinterpret_cast<Slot*>(tmp + nb);
  __shared__ double red_v[kThreads / 32];
  __shared__ int red_i[kThreads / 32];
  __shared__ int s_r;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = c * RP, r1 = min(n, r0 + RP), nr = max(0, r1 - r0);
  zt* Ab = A + (int64_t)b * bs;
  int* piv = piv_all + (int64_t)b * n;
  for (int e = tid; e < nr * nb; e += kThreads) {
    const int i = e / nb, j = e % nb;
    P[i * nb + j] = Ab[(int64_t)(r0 + i) * lda + k0 + j];
  }
  __syncthreads();
  bool singular = false;
  for (int kk = 0; kk < nb; ++kk) {
    const int k = k0 + kk;
    // local argmax over owned rows i >= k
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = max(k, r0) + tid; i < r1; i += kThreads) amax_merge(bv, bi, zabs2(P[(i - r0) * nb + kk]), i);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      amax_merge(bv, bi, v2, i2);
    }
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kThreads / 32; ++w) amax_merge(bv, bi, red_v[w], red_i[w]);
      slot->v = bv;
      slot->i = bi;
    }
    cluster.sync();  // (1) slots visible
    if (tid == 0) {
      double gv = -1.0;
      int gi = 0x7fffffff;
      for (int q = 0; q < CS; ++q) {
        const Slot* rs = cluster.map_shared_rank(slot, q);
        amax_merge(gv, gi, rs->v, rs->i);
      }
      if (gv <= 0.0) {
        singular = true;
        if (gi == 0x7fffffff) gi = k;
      }
      s_r = gi;
    }
    __syncthreads();
    const int r = s_r;
    const int own_r = r / RP, own_k = k / RP;
    {  // pivot row (remote read) -> prow ; if I own r: old row k -> tmp
      const zt* src = cluster.map_shared_rank(P, own_r) + (r - own_r * RP) * nb;
      for (int j = tid; j < nb; j += kThreads) prow[j] = src[j];
      if (c == own_r && r != k) {
        const zt* srck = cluster.map_shared_rank(P, own_k) + (k - own_k * RP) * nb;
        for (int j = tid; j < nb; j += kThreads) tmp[j] = srck[j];
      }
    }
    cluster.sync();  // (2) all remote reads done
    const zt inv = zinv(prow[kk]);
    __syncthreads();
    for (int j = tid; j < nb; j += kThreads) prow[j] = (j == kk) ? inv : zmul(prow[j], inv);
    if (c == own_r && r != k)
      for (int j = tid; j < nb; j += kThreads) P[(r - r0) * nb + j] = tmp[j];
    __syncthreads();
    // update owned rows
    for (int i = r0 + warp; i < r1; i += kThreads / 32) {
      zt* row = P + (i - r0) * nb;
      if (i == k) {
        for (int j = lane; j < nb; j += 32) row[j] = prow[j];
      } else {
        const zt f = row[kk];
        __syncwarp();
        for (int j = lane; j < nb; j += 32) {
          zt a = (j == kk) ? make_double2(0.0, 0.0) : row[j];
          const zt pj = prow[j];
          a.x -= f.x * pj.x - f.y * pj.y;
          a.y -= f.x * pj.y + f.y * pj.x;
          row[j] = a;
        }
      }
    }
    if (c == 0 && tid == 0) piv[k] = r;
    __syncthreads();
  }
  for (int e = tid; e < nr * nb; e += kThreads) {
    const int i = e / nb, j = e % nb;
    Ab[(int64_t)(r0 + i) * lda + k0 + j] = P[i * nb + j];
  }
  if (singular && c == 0 && tid == 0) atomicCAS(info, 0, b + 1);
  cluster.sync();  // keep shared memory alive until every remote reader is done
}

// Row swaps of the panel applied to every non-panel column; Z = panel rows (compact
// columns), panel rows zeroed.  grid: (ceil((n - w)/256), batch)
__global__ void zgj_swapz_kernel(zt* A, int64_t lda, int64_t bs, int n, int k0, int w, const int* piv_all, zt* Z) {
  const int b = blockIdx.y;
  const int jj = blockIdx.x * blockDim.x + threadIdx.x;
  const int nc = n - w;
  if (jj >= nc) return;
  const int j = jj < k0 ? jj : jj + w;
  zt* Ab = A + (int64_t)b * bs;
  const int* piv = piv_all + (int64_t)b * n;
  for (int k = k0; k < k0 + w; ++k) {
    const int r = piv[k];
    if (r != k) {
      const zt t = Ab[(int64_t)k * lda + j];
      Ab[(int64_t)k * lda + j] = Ab[(int64_t)r * lda + j];
      Ab[(int64_t)r * lda + j] = t;
    }
  }
  zt* Zb = Z + (int64_t)b * w * nc;
  for (int kk = 0; kk < w; ++kk) {
    Zb[(int64_t)kk * nc + jj] = Ab[(int64_t)(k0 + kk) * lda + j];
    Ab[(int64_t)(k0 + kk) * lda + j] = make_double2(0.0, 0.0);
  }
}

// pi = S_{n-1} o ... o S_0 (one thread per matrix)
__global__ void zgj_pi_kernel(const int* piv_all, int* pi_all, int n, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int* piv = piv_all + (int64_t)b * n;
  int* pi = pi_all + (int64_t)b * n;
  for (int j = 0; j < n; ++j) pi[j] = j;
  for (int k = n - 1; k >= 0; --k) {
    const int r = piv[k];
    const int t = pi[k];
    pi[k] = pi[r];
    pi[r] = t;
  }
}

// out(i, j) = A(i, pi(j))
__global__ void zgj_colperm_kernel(const zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs,
                                   const int* pi_all, int n, int batch) {
  const int64_t total = (int64_t)batch * n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % n);
    const int64_t t = e / n;
    const int i = (int)(t % n);
    const int b = (int)(t / n);
    out[(int64_t)b * obs + (int64_t)i * ldo + j] = A[(int64_t)b * bs + (int64_t)i * lda + pi_all[(int64_t)b * n + j]];
  }
}

struct PanelPlan {
  int nb, cs, rp;
  size_t smem;
};

PanelPlan panel_plan(int n) {
  const size_t budget = 150 * 1024;
  for (int nb : {32, 16}) {
    for (int cs = 1; cs <= 16; cs *= 2) {
      const int rp = (n + cs - 1) / cs;
      const size_t smem = sizeof(zt) * ((size_t)rp * nb + 2 * nb) + 64;
      if (smem <= budget) return PanelPlan{nb, cs, rp, smem};
    }
  }
  return PanelPlan{16, 16, (n + 15) / 16, sizeof(zt) * ((size_t)((n + 15) / 16) * 16 + 32) + 64};
}

}  // namespace

size_t zgj_workspace_bytes(int n, int batch) {
  if (n <= kSmallMax) return 0;
  const PanelPlan pp = panel_plan(n);
  size_t z = sizeof(zt) * (size_t)batch * pp.nb * n;
  size_t piv = sizeof(int) * (size_t)batch * n * 2;
  return ((z + 255) / 256) * 256 + piv + 256;
}

void zgj_invert(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch, void* ws,
                int* info, cudaStream_t st, int64_t* launches) {
  (void)launches;
  if (n <= 0 || batch <= 0) return;
  if (n <= kSmallMax) {
    const size_t smem = sizeof(zt) * ((size_t)n * (n + 1) + 2 * n) + sizeof(int) * n + 16;
    static bool attr = false;
    if (!attr) {
      HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(zt) * ((size_t)kSmallMax * (kSmallMax + 1) + 2 * kSmallMax) +
                                                sizeof(int) * kSmallMax + 16)));
      attr = true;
    }
    ProfScope ps(K_GJ_SMALL, 8.0 * n * n * (double)n * batch, 32.0 * n * (double)n * batch, st);
    for (int b0 = 0; b0 < batch; b0 += 65535) {
      const int nbatch = std::min(65535, batch - b0);
      zgj_small_kernel<<<nbatch, kThreads, smem, st>>>(A + (int64_t)b0 * bs, lda, bs, out + (int64_t)b0 * obs, ldo,
                                                       obs, n, info);
      HPS_CUDA_CHECK(cudaGetLastError());
      count_launch();
    }
    return;
  }
  const PanelPlan pp = panel_plan(n);
  char* w = static_cast<char*>(ws);
  zt* Z = reinterpret_cast<zt*>(w);
  size_t zbytes = ((sizeof(zt) * (size_t)batch * pp.nb * n + 255) / 256) * 256;
  int* piv = reinterpret_cast<int*>(w + zbytes);
  int* pi = piv + (size_t)batch * n;
  static bool attr = false;
  if (!attr) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  for (int k0 = 0; k0 < n; k0 += pp.nb) {
    const int wdt = std::min(pp.nb, n - k0);
    {
      ProfScope ps(K_GJ_PANEL, 8.0 * n * (double)wdt * wdt * batch, 32.0 * n * (double)wdt * batch, st);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(batch * pp.cs);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = pp.smem;
      cfg.stream = st;
      cudaLaunchAttribute attr_[1];
      attr_[0].id = cudaLaunchAttributeClusterDimension;
      attr_[0].val.clusterDim.x = pp.cs;
      attr_[0].val.clusterDim.y = 1;
      attr_[0].val.clusterDim.z = 1;
      cfg.attrs = attr_;
      cfg.numAttrs = 1;
      HPS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zgj_panel_kernel, A, lda, bs, n, k0, wdt, pp.rp, piv, info));
      count_launch();
    }
    const int nc = n - wdt;
    if (nc > 0) {
      {
        dim3 g((nc + 255) / 256, batch);
        ProfScope ps(K_GJ_AUX, 0.0, 16.0 * 4.0 * wdt * (double)nc * batch, st);
        zgj_swapz_kernel<<<g, 256, 0, st>>>(A, lda, bs, n, k0, wdt, piv, Z);
        HPS_CUDA_CHECK(cudaGetLastError());
        count_launch();
      }
      ZGemm gm;
      gm.M = n;
      gm.N = nc;
      gm.K = wdt;
      gm.batch = batch;
      gm.A.ptr = A + k0;
      gm.A.rs = lda;
      gm.A.bs = bs;
      gm.B.ptr = Z;
      gm.B.rs = nc;
      gm.B.bs = (int64_t)wdt * nc;
      gm.Cin.ptr = A;
      gm.Cin.rs = lda;
      gm.Cin.bs = bs;
      gm.Cin.cskip_at = k0;
      gm.Cin.cskip_len = wdt;
      gm.C.ptr = A;
      gm.C.rs = lda;
      gm.C.bs = bs;
      gm.C.cskip_at = k0;
      gm.C.cskip_len = wdt;
      gm.beta = make_double2(1.0, 0.0);
      zgemm(gm, st);
    }
  }
  {
    ProfScope ps(K_GJ_AUX, 0.0, 8.0 * n * (double)batch, st);
    zgj_pi_kernel<<<(batch + 127) / 128, 128, 0, st>>>(piv, pi, n, batch);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
  const int64_t total = (int64_t)batch * n * n;
  ProfScope ps(K_GJ_AUX, 0.0, 32.0 * (double)total, st);
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  zgj_colperm_kernel<<<blocks, 256, 0, st>>>(A, lda, bs, out, ldo, obs, pi, n, batch);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}
