// zgj.cu — batched explicit inverse by Gauss-Jordan elimination with partial pivoting.
//
// Used for the leaf interior operator S (the full leaf matrix
// B in leaf_mode 1) and for W = I - R33b R33a of every merge
// (the paper stores W^{-1} explicitly, computed there by
// zgetrf + zgetri).  Gauss-Jordan costs the same n^3 complex multiply-adds
// as LU + triangular inverse and its update is a full-height GEMM on the DMMA path.
//
// In-place GJ step k (row pivoting): r = argmax_{i>=k} |A(i,k)|; swap rows k, r;
//   row k <- row k / A(k,k) with A(k,k) <- 1/A(k,k); for i != k: A(i,:) -= A(i,k) * row k
//   (A(i,k) reset to 0 first, so it ends as -A(i,k)/pivot).  Finally the column swaps are
//   undone in reverse order: out(:, j) = A(:, pi(j)).
//
// Small matrices (n <= 32, or n <= 112 with a large batch): one CTA per matrix, all in shared
// memory.  Otherwise blocked over panels of nb <= 32 columns, ping-pong between buffers X, Y:
//   panel kernel: reads the panel of X, factors it (pivot search over all rows), writes the
//     transform columns T into Y and the row permutation P of its swaps as a row map;
//   update (DMMA GEMM): for every other column j,  Y(:, j) = (I~ P X)(:, j) + T (P X)(panel, j)
//     with I~ zeroing the panel rows — swaps, the Z copy and the update in one launch.
// Panel factorisation: n <= 256 in one CTA with each row in a thread's registers; n <= 4096
// in a thread-block cluster (rows in registers of up to 16 CTAs, pivot candidates and pivot
// row through distributed shared memory); larger n: cluster with the panel in shared memory.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

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

__device__ __forceinline__ void warp_amax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    amax_merge(v, i, v2, i2);
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
      warp_amax(bv, bi);
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
    int* pi = reinterpret_cast<int*>(col);
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

// Panel kernel arguments: X read, Y written (transform columns), per-matrix pivots piv[n], row
// maps rowsrc[n] (row i of P X is row rowsrc[i] of X) and cinmap[n] (= rowsrc, -1 on the
// panel rows).
struct PanelArgs {
  const zt* X;
  zt* Y;
  int64_t ldx, bsx, ldy, bsy;
  int n, k0, w;
  int* piv;
  int* rowsrc;
  int* cinmap;
  int* info;
  int* pflag = nullptr;  // implicit-pivoting path: 1 = row already pivoted
  // natural-order panels: |A_kk|^2 of the ORIGINAL matrix per (batch, k); a pivot p of step k
  // passes if |p|^2 >= rel2 * d0[k] (relative check, reading Q21)
  const double* d0 = nullptr;
  double rel2 = 0.0;
};

__device__ __forceinline__ bool nat_pivot_ok(const PanelArgs& a, int b, int k, zt pv) {
  const double m = fma(pv.x, pv.x, pv.y * pv.y);
  return m > 0.0 && m >= a.rel2 * a.d0[(int64_t)b * a.n + k];
}

__device__ __forceinline__ void write_maps(const PanelArgs& a, int b, int i, int orig) {
  if (i < a.n) {
    a.rowsrc[(int64_t)b * a.n + i] = orig;
    a.cinmap[(int64_t)b * a.n + i] = (i >= a.k0 && i < a.k0 + a.w) ? -1 : orig;
  }
}

// Register rows are kept ROTATED: after each Gauss-Jordan step the row shifts left by one, so
// the active column kk always sits in register slot 0 (no dynamic register indexing) and after
// w steps slot p holds panel column (p + w) mod NB.  The pivot row is broadcast RAW; every
// thread derives 1/pivot itself, so no thread serialises the scaling.
template <int NB>
__device__ __forceinline__ void row_rotate(zt (&row)[NB]) {
  const zt t = row[0];
#pragma unroll
  for (int j = 0; j < NB - 1; ++j) row[j] = row[j + 1];
  row[NB - 1] = t;
}

// 1 / z for the pivot: conj(z) / |z|^2 with an IEEE round-to-nearest reciprocal.
// Plain global loads for data the same CTA wrote (after a barrier) or an earlier kernel wrote:
// ld.global.cg compiles to LDG.STRONG.GPU, whose ordering against the CTA's outstanding stores
// showed up as "membar" stalls in the single-CTA Gauss-Jordan kernels.
template <typename T>
__device__ __forceinline__ T ldplain(const T* p) {
  return *p;
}

__device__ __forceinline__ zt zinv_fast(zt a) {
  // 1/|a|^2: hardware reciprocal estimate (MUFU.RCP64H) refined by two branch-free Newton steps
  // (relative error ~1e-28 before rounding; pivots are never denormal here).
  const double d = fma(a.x, a.x, a.y * a.y);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  return make_double2(a.x * r, -a.y * r);
}

// Gauss-Jordan step on one register row given the RAW pivot row `pr` (slot 0 = pivot value):
// row <- row - g * pr with g = row[0] / pivot, then slot 0 <- -g.
template <int NB>
__device__ __forceinline__ void row_step(zt (&row)[NB], const zt* pr, zt inv) {
  const zt g = zmul(row[0], inv);
  const double ngx = -g.x, ngy = -g.y;
  // one shared-memory read of each pivot-row element (broadcast LDS costs 4 B/lane/cycle)
#pragma unroll
  for (int j = 1; j < NB; ++j) {
    const zt pj = pr[j];
    row[j].x = fma(ngx, pj.x, row[j].x);
    row[j].y = fma(ngx, pj.y, row[j].y);
    row[j].x = fma(g.y, pj.y, row[j].x);
    row[j].y = fma(ngy, pj.x, row[j].y);
  }
  row[0] = make_double2(ngx, ngy);
}

// Pivot row itself: row <- pr / pivot with slot 0 <- 1 / pivot.
template <int NB>
__device__ __forceinline__ void row_pivot(zt (&row)[NB], const zt* pr, zt inv) {
#pragma unroll
  for (int j = 1; j < NB; ++j) row[j] = zmul(pr[j], inv);
  row[0] = inv;
}

template <int NB>
__device__ __forceinline__ void store_rotated(const zt (&row)[NB], zt* dst, int w) {
#pragma unroll
  for (int p = 0; p < NB; ++p) {
    int j = p + w;
    if (j >= NB) j -= NB;
    if (j < w) dst[j] = row[p];
  }
}

// Pivot key: the high 32 bits of |z|^2 (sign 0, exponent, 20 mantissa bits: monotone in |z|^2),
// low 9 bits replaced by (511 - local row) so one unsigned max picks the largest magnitude and,
// among magnitudes equal to ~1e-4 relative, the lowest row (threshold partial pivoting; a
// pivot within that tolerance of the column maximum keeps the growth bound of partial pivoting).
__device__ __forceinline__ unsigned pivot_key(zt f, int local, bool valid) {
  if (!valid) return 0u;
  const double m = f.x * f.x + f.y * f.y;
  const unsigned hi = (unsigned)(__double_as_longlong(m) >> 32);
  return (hi & ~511u) | (unsigned)(511 - local);
}

// ---------------------------------------------------------------------------
// Register-resident panel, n <= THREADS (256 or 512): thread t owns panel row t in registers;
// the rank-1 update is register-local; per step two barriers, one warp max-reduction
// (REDUX) of packed pivot keys and one shared broadcast of the raw pivot row (plus the
// displaced row k).
// ---------------------------------------------------------------------------
template <int NB, int THREADS>
__global__ void __launch_bounds__(THREADS, 512 / THREADS) zgj_panel_reg_kernel(const PanelArgs a) {
  constexpr int NW = THREADS / 32;
  __shared__ zt prow[NB], tmp[NB];
  __shared__ unsigned wkey[NW];
  __shared__ int s_orig_r, s_orig_k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x, n = a.n, k0 = a.k0, w = a.w;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  const int i = tid;
  int orig = i;
  zt row[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) row[j] = (i < n && j < w) ? Xb[(int64_t)i * a.ldx + k0 + j] : make_double2(0.0, 0.0);
  bool singular = false;
  for (int kk = 0; kk < w; ++kk) {
    const int k = k0 + kk;
    const unsigned key = __reduce_max_sync(0xffffffffu, pivot_key(row[0], i, i < n && i >= k));
    if (lane == 0) wkey[warp] = key;
    __syncthreads();
    unsigned best = wkey[0];
#pragma unroll
    for (int w2 = 1; w2 < NW; ++w2) best = max(best, wkey[w2]);
    int r = 511 - (int)(best & 511u);
    if ((best & ~511u) == 0u) {  // exactly zero column below the diagonal
      singular = true;
      r = k;
    }
    if (i == r) {  // publish the raw pivot row
#pragma unroll
      for (int j = 0; j < NB; ++j) prow[j] = row[j];
      s_orig_r = orig;
    }
    if (i == k && r != k) {
#pragma unroll
      for (int j = 0; j < NB; ++j) tmp[j] = row[j];
      s_orig_k = orig;
    }
    __syncthreads();
    const zt inv = zinv_fast(prow[0]);
    if (i == k) {
      row_pivot<NB>(row, prow, inv);
      orig = s_orig_r;
    } else {
      if (i == r) {  // receives the displaced row k
#pragma unroll
        for (int j = 0; j < NB; ++j) row[j] = tmp[j];
        orig = s_orig_k;
      }
      row_step<NB>(row, prow, inv);
    }
    row_rotate<NB>(row);
    if (tid == 0) piv[k] = r;
  }
  if (i < n) store_rotated<NB>(row, Yb + (int64_t)i * a.ldy + k0, w);
  write_maps(a, b, i, orig);
  if (singular && tid == 0) atomicCAS(a.info, 0, b + 1);
}

// ---------------------------------------------------------------------------
// Natural-order panel (no pivot search), n <= 512, w <= 16, for the merge matrices W (DESIGN.md
// 3.10: measured to need no pivoting in the configs' regimes): 512 threads, 4 rows x 4 columns per thread; per step the owner
// lanes of row k publish it and ONE barrier separates publication from the update.  A pivot
// whose |pivot|^2 is below rel2 x the original |A_kk|^2 raises *a.pflag (the caller redoes the
// matrix with partial pivoting).
// Same interface and outputs as zgj_panel_reg_kernel with identity permutations.
__device__ long long g_nat_trace[64];  // debug timeline (hps_debug_ws_trace(7, out): out[256..319])
__device__ int g_nat_trace_on;
// ---------------------------------------------------------------------------
// Blocked natural-order panel: with natural pivots the w pivot rows are rows
// k0 .. k0+w-1, so the w x w diagonal block is eliminated first on its own (one warp; every CTA
// does it redundantly, no inter-CTA communication) and records the w scaled pivot rows; every
// other row then applies the w recorded steps locally (shuffles only, no barrier per step).
// Grid (ceil(n / 128), batch), 512 threads: 4 lanes x 4 columns per row, 128 rows per CTA.
// w <= 16.  A pivot failing nat_pivot_ok raises *a.pflag.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) zgj_panel_natb_kernel(const PanelArgs a) {
  constexpr int CPT = 4, NB = 16, RPC = 128;
  __shared__ zt blk[NB][NB + 1];  // the block rows (panel columns), eliminated in place
  __shared__ zt phat[NB][NB];     // raw pivot row of step kk divided by its pivot
  __shared__ zt pinv[NB];         // 1 / pivot of step kk
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, cg = lane & 3, rg = lane >> 2;
  const int b = blockIdx.y, n = a.n, k0 = a.k0, w = a.w;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  const int i = blockIdx.x * RPC + wp * 8 + rg;  // this thread's row
  const bool ntr = g_nat_trace_on == 7 && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0 && k0 == 0;
  if (ntr) g_nat_trace[0] = clock64();
  // this thread's 4 panel values (loads in flight during stage 1)
  zt v[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int j = cg * CPT + c;
    v[c] = (i < n && j < w) ? Xb[(int64_t)i * a.ldx + k0 + j] : make_double2(0.0, 0.0);
  }
  if (wp == 0) {  // ---- stage 1: the diagonal block, in registers (lane: column c, rows 8h .. 8h+7) ----
    const int c = lane & 15, h = lane >> 4;
    zt bv[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int r = h * 8 + m;
      bv[m] = (r < w && c < w) ? Xb[(int64_t)(k0 + r) * a.ldx + k0 + c] : make_double2(0.0, 0.0);
    }
    if (ntr) {
      volatile double sink = bv[0].x + bv[7].y;
      (void)sink;
      g_nat_trace[4] = clock64();
    }
    bool bad = false;
#pragma unroll
    for (int kk = 0; kk < NB; ++kk) {
      if (kk < w) {
        const int mk = kk & 7, hk = kk >> 3;
        // pivot row kk at this lane's column, the pivot, and column kk at this lane's rows
        const zt pr = make_double2(__shfl_sync(0xffffffffu, bv[mk].x, (hk << 4) | c),
                                   __shfl_sync(0xffffffffu, bv[mk].y, (hk << 4) | c));
        const zt pv = make_double2(__shfl_sync(0xffffffffu, bv[mk].x, (hk << 4) | kk),
                                   __shfl_sync(0xffffffffu, bv[mk].y, (hk << 4) | kk));
        zt aik[8];
#pragma unroll
        for (int m = 0; m < 8; ++m)
          aik[m] = make_double2(__shfl_sync(0xffffffffu, bv[m].x, (h << 4) | kk),
                                __shfl_sync(0xffffffffu, bv[m].y, (h << 4) | kk));
        bad = bad || !nat_pivot_ok(a, b, k0 + kk, pv);
        const zt inv = zinv_fast(pv);
        const zt prn = zmul(pr, inv);  // pr / pivot
        if (h == 0) phat[kk][c] = c == kk ? make_double2(0.0, 0.0) : prn;
        if (lane == 0) pinv[kk] = inv;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int r = h * 8 + m;
          zt nv;
          if (r == kk) {
            nv = c == kk ? inv : prn;
          } else if (c == kk) {
            const zt g = zmul(aik[m], inv);
            nv = make_double2(-g.x, -g.y);
          } else {
            nv = bv[m];
            nv.x = fma(-aik[m].x, prn.x, nv.x);
            nv.x = fma(aik[m].y, prn.y, nv.x);
            nv.y = fma(-aik[m].x, prn.y, nv.y);
            nv.y = fma(-aik[m].y, prn.x, nv.y);
          }
          bv[m] = nv;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) blk[h * 8 + m][c] = bv[m];
    if (lane == 0) s_bad = bad ? 1 : 0;
    if (ntr) g_nat_trace[5] = clock64();
  }
  __syncthreads();
  if (ntr) g_nat_trace[1] = clock64();
  // ---- stage 2: rows outside the block apply the w recorded steps ----
  const bool inblk = i >= k0 && i < k0 + w;
  if (i < n && !inblk) {
#pragma unroll
    for (int kk = 0; kk < NB; ++kk) {
      if (kk < w) {
        const int src = (lane & ~3) | (kk >> 2);
        const zt own = v[kk & 3];
        const zt t = make_double2(__shfl_sync(0xffffffffu, own.x, src), __shfl_sync(0xffffffffu, own.y, src));
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const zt ph = phat[kk][cg * CPT + c];
          v[c].x = fma(-t.x, ph.x, v[c].x);
          v[c].x = fma(t.y, ph.y, v[c].x);
          v[c].y = fma(-t.x, ph.y, v[c].y);
          v[c].y = fma(-t.y, ph.x, v[c].y);
        }
        if (cg == (kk >> 2)) {  // column kk <- -t / pivot
          const zt g = zmul(t, pinv[kk]);
          v[kk & 3] = make_double2(-g.x, -g.y);
        }
      }
    }
  } else if (i < n) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) v[c] = blk[i - k0][cg * CPT + c];
  }
  if (ntr) g_nat_trace[2] = clock64();
  if (i < n) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int j = cg * CPT + c;
      if (j < w) Yb[(int64_t)i * a.ldy + k0 + j] = v[c];
    }
    if (cg == 0) write_maps(a, b, i, i);
  }
  if (blockIdx.x == 0) {
    if (tid < w) a.piv[(int64_t)b * n + k0 + tid] = k0 + tid;
    if (tid == 0 && s_bad) atomicExch(a.pflag, 1);
  }
  if (ntr) g_nat_trace[3] = clock64();
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) zgj_panel_nat_kernel(const PanelArgs a) {
  constexpr int CPT = 4, NB = 16, RPT = 4;
  __shared__ zt prow[2][NB];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, cg = lane & 3, rg = lane >> 2;
  const int b = blockIdx.x, n = a.n, k0 = a.k0, w = a.w;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  int rq[RPT];
  zt v[RPT][CPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    rq[t] = wp * 32 + t * 8 + rg;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int j = cg * CPT + c;
      v[t][c] = (rq[t] < n && j < w) ? Xb[(int64_t)rq[t] * a.ldx + k0 + j] : make_double2(0.0, 0.0);
    }
  }
  bool bad = false;
#pragma unroll 1
  for (int cga = 0; cga * CPT < w; ++cga) {
    const bool act = cg == cga;
    const int src = (lane & ~3) | cga;
#pragma unroll
    for (int s = 0; s < CPT; ++s) {
      const int kk = cga * CPT + s;
      if (kk >= w) break;
      const int k = k0 + kk, par = kk & 1;
      if (wp == (k >> 5) && rg == (k & 7)) {
        const int tt = (k >> 3) & 3;
#pragma unroll
        for (int t = 0; t < RPT; ++t)
          if (t == tt) {
#pragma unroll
            for (int c = 0; c < CPT; ++c) prow[par][cg * CPT + c] = v[t][c];
          }
      }
      __syncthreads();
      const zt pv = prow[par][kk];
      if (!nat_pivot_ok(a, b, k, pv)) bad = true;
      const zt inv = zinv_fast(pv);
      zt pr[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) pr[c] = prow[par][cg * CPT + c];
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const zt own = v[t][s];
        zt g = zmul(make_double2(__shfl_sync(0xffffffffu, own.x, src), __shfl_sync(0xffffffffu, own.y, src)), inv);
        if (rq[t] == k) {  // the pivot row: pr / pivot (as 0 - (-inv) pr), slot kk <- 1 / pivot
          g = make_double2(-inv.x, -inv.y);
#pragma unroll
          for (int c = 0; c < CPT; ++c) v[t][c] = make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          v[t][c].x = fma(-g.x, pr[c].x, v[t][c].x);
          v[t][c].y = fma(-g.x, pr[c].y, v[t][c].y);
          v[t][c].x = fma(g.y, pr[c].y, v[t][c].x);
          v[t][c].y = fma(-g.y, pr[c].x, v[t][c].y);
        }
        if (act) v[t][s] = make_double2(-g.x, -g.y);
      }
      if (tid == 0) piv[k] = k;
    }
  }
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = rq[t];
    if (i < n) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int j = cg * CPT + c;
        if (j < w) Yb[(int64_t)i * a.ldy + k0 + j] = v[t][c];
      }
      if (cg == 0) write_maps(a, b, i, i);
    }
  }
  if (bad && tid == 0) atomicExch(a.pflag, 1);
}

// Cluster form of zgj_panel_nat_kernel: a cluster of CS = ceil(n / 128) CTAs per matrix, CTA c
// owns rows 128 c .. 128 c + 127 (one row x 4 columns per thread, 4 lanes per row).  Per step the
// owner lanes of row k publish it in their CTA's shared memory, one cluster barrier, and every
// CTA reads it through distributed shared memory: the per-step FP64 work of a 448-row panel is
// spread over 4 SMs instead of 1.
template <int CPT, int LPR = 4>
__global__ void __launch_bounds__(512, 1) zgj_panel_natc_kernel(const PanelArgs a) {
  // LPR lanes per row (CPT columns each), RPC = 512 / LPR rows per CTA
  constexpr int NB = LPR * CPT, RPC = 512 / LPR;
  const bool ntr = g_nat_trace_on == 7 && blockIdx.x == 0 && threadIdx.x == 0 && a.k0 == 0;
  if (ntr) g_nat_trace[0] = clock64();
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int cr = (int)cluster.block_rank();
  __shared__ zt prow[2][NB];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, cg = lane % LPR, rg = lane / LPR;
  const int b = blockIdx.x / CS, n = a.n, k0 = a.k0, w = a.w;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  const int i = cr * RPC + wp * (32 / LPR) + rg;
  zt v[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int j = cg * CPT + c;
    v[c] = (i < n && j < w) ? Xb[(int64_t)i * a.ldx + k0 + j] : make_double2(0.0, 0.0);
  }
  bool bad = false;
  if (ntr) g_nat_trace[1] = clock64();
#pragma unroll 1
  for (int cga = 0; cga * CPT < w; ++cga) {
    const bool act = cg == cga;
    const int src = (lane & ~(LPR - 1)) | cga;
#pragma unroll
    for (int s = 0; s < CPT; ++s) {
      const int kk = cga * CPT + s;
      if (kk >= w) break;
      const int k = k0 + kk, par = kk & 1;
      if (ntr) g_nat_trace[2 + kk] = clock64();
      if (i == k) {
#pragma unroll
        for (int c = 0; c < CPT; ++c) prow[par][cg * CPT + c] = v[c];
      }
      // only the owner CTA publishes: release there, relaxed elsewhere (a reader's loads of step
      // k feed its update before it arrives at step k + 1, so the double buffer stays safe)
      if (cr == k / RPC)
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      else
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      const zt* rp = cluster.map_shared_rank(&prow[par][0], k / RPC);
      const zt pv = rp[kk];
      zt pr[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) pr[c] = rp[cg * CPT + c];
      if (!nat_pivot_ok(a, b, k, pv)) bad = true;
      const zt inv = zinv_fast(pv);
      const zt own = v[s];
      zt g = zmul(make_double2(__shfl_sync(0xffffffffu, own.x, src), __shfl_sync(0xffffffffu, own.y, src)), inv);
      if (i == k) {  // the pivot row: pr / pivot (as 0 - (-inv) pr), slot kk <- 1 / pivot
        g = make_double2(-inv.x, -inv.y);
#pragma unroll
        for (int c = 0; c < CPT; ++c) v[c] = make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        v[c].x = fma(-g.x, pr[c].x, v[c].x);
        v[c].y = fma(-g.x, pr[c].y, v[c].y);
        v[c].x = fma(g.y, pr[c].y, v[c].x);
        v[c].y = fma(-g.y, pr[c].x, v[c].y);
      }
      if (act) v[s] = make_double2(-g.x, -g.y);
      if (cr == 0 && tid == 0) piv[k] = k;
    }
  }
  if (ntr) g_nat_trace[40] = clock64();
  if (i < n) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int j = cg * CPT + c;
      if (j < w) Yb[(int64_t)i * a.ldy + k0 + j] = v[c];
    }
    if (cg == 0) write_maps(a, b, i, i);
  }
  if (bad && tid == 0) atomicExch(a.pflag, 1);
  cluster.sync();  // no CTA exits while another may still read its shared memory
  if (ntr) g_nat_trace[41] = clock64();
}

// ---------------------------------------------------------------------------
// Cluster version, 256 < n <= 4096: CTA c owns rows c*256 + t in registers.  Two cluster
// barriers per step: (1) after the per-CTA pivot candidates, (2) after the owner of the
// pivot row (and of row k) published them in its shared memory.
// ---------------------------------------------------------------------------
struct Slot {
  double v;
  int i;
  int pad;
};

template <int NB>
__global__ void __launch_bounds__(256) zgj_panel_creg_kernel(const PanelArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int b = blockIdx.x / CS, n = a.n, k0 = a.k0, w = a.w;
  __shared__ zt prow[NB], tmp[NB], lprow[NB];
  __shared__ unsigned wkey[8];
  __shared__ Slot slot;
  __shared__ int s_r, orig_r_pub, orig_k_pub;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = c * 256 + tid;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  int orig = i;
  zt row[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) row[j] = (i < n && j < w) ? Xb[(int64_t)i * a.ldx + k0 + j] : make_double2(0.0, 0.0);
  bool singular = false;
  for (int kk = 0; kk < w; ++kk) {
    const int k = k0 + kk;
    const unsigned key = __reduce_max_sync(0xffffffffu, pivot_key(row[0], tid, i < n && i >= k));
    if (lane == 0) wkey[warp] = key;
    __syncthreads();
    if (tid == 0) {
      unsigned best = wkey[0];
      for (int w2 = 1; w2 < 8; ++w2) best = max(best, wkey[w2]);
      slot.v = 0.0;
      slot.i = (int)best;  // packed key of this CTA's best row
    }
    cluster.sync();  // (1) candidates visible
    if (warp == 0) {
      // cluster-wide: larger key wins; equal keys -> lower CTA rank (lower row)
      const unsigned ck = lane < CS ? (unsigned)cluster.map_shared_rank(&slot, lane)->i : 0u;
      const unsigned long long k64 = ((unsigned long long)ck << 32) | (unsigned)(31 - lane);
      unsigned long long bestk = k64;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long o64 = __shfl_xor_sync(0xffffffffu, bestk, o);
        bestk = o64 > bestk ? o64 : bestk;
      }
      if (lane == 0) {
        const unsigned kb = (unsigned)(bestk >> 32);
        const int crank = 31 - (int)(bestk & 31u);
        int gi = crank * 256 + (511 - (int)(kb & 511u));
        if ((kb & ~511u) == 0u) {
          singular = true;
          gi = k;
        }
        s_r = gi;
      }
    }
    __syncthreads();
    const int r = s_r;
    if (i == r) {  // publish the raw pivot row
#pragma unroll
      for (int j = 0; j < NB; ++j) prow[j] = row[j];
      orig_r_pub = orig;
    }
    if (i == k && r != k) {
#pragma unroll
      for (int j = 0; j < NB; ++j) tmp[j] = row[j];
      orig_k_pub = orig;
    }
    cluster.sync();  // (2) pivot row published
    if (tid < NB) lprow[tid] = cluster.map_shared_rank(prow, r / 256)[tid];
    __syncthreads();
    const zt inv = zinv_fast(lprow[0]);
    if (i == k) {
      orig = *cluster.map_shared_rank(&orig_r_pub, r / 256);
      row_pivot<NB>(row, lprow, inv);
    } else if (i < n) {
      if (i == r) {
        const zt* rt = cluster.map_shared_rank(tmp, k / 256);
#pragma unroll
        for (int j = 0; j < NB; ++j) row[j] = rt[j];
        orig = *cluster.map_shared_rank(&orig_k_pub, k / 256);
      }
      row_step<NB>(row, lprow, inv);
    }
    row_rotate<NB>(row);
    if (c == 0 && tid == 0) piv[k] = r;
  }
  if (i < n) store_rotated<NB>(row, Yb + (int64_t)i * a.ldy + k0, w);
  write_maps(a, b, i, orig);
  if (singular && c == 0 && tid == 0) atomicCAS(a.info, 0, b + 1);
  cluster.sync();  // no CTA leaves while a peer may still read its shared memory
}

// ---------------------------------------------------------------------------
// Shared-memory cluster panel for n > 4096: CTA c owns panel rows [c*RP, min(n, (c+1)*RP)).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) zgj_panel_smem_kernel(const PanelArgs a, int RP) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int b = blockIdx.x / CS, n = a.n, k0 = a.k0, nb = a.w;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zt* P = reinterpret_cast<zt*>(smem_raw);  // RP x nb
  zt* prow = P + RP * nb;                   // nb
  zt* tmp = prow + nb;                      // nb
  Slot* slot = reinterpret_cast<Slot*>(tmp + nb);
  int* orig = reinterpret_cast<int*>(slot + 1);  // RP
  __shared__ double red_v[kThreads / 32];
  __shared__ int red_i[kThreads / 32];
  __shared__ int s_r, s_origr, s_origk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = c * RP, r1 = min(n, r0 + RP), nr = max(0, r1 - r0);
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  for (int e = tid; e < nr * nb; e += kThreads) {
    const int i = e / nb, j = e % nb;
    P[i * nb + j] = Xb[(int64_t)(r0 + i) * a.ldx + k0 + j];
  }
  for (int i = tid; i < nr; i += kThreads) orig[i] = r0 + i;
  __syncthreads();
  bool singular = false;
  for (int kk = 0; kk < nb; ++kk) {
    const int k = k0 + kk;
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = max(k, r0) + tid; i < r1; i += kThreads) amax_merge(bv, bi, zabs2(P[(i - r0) * nb + kk]), i);
    warp_amax(bv, bi);
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w2 = 1; w2 < kThreads / 32; ++w2) amax_merge(bv, bi, red_v[w2], red_i[w2]);
      slot->v = bv;
      slot->i = bi;
    }
    cluster.sync();  // (1)
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
      const int own_r = gi / RP, own_k = k / RP;
      s_origr = cluster.map_shared_rank(orig, own_r)[gi - own_r * RP];
      s_origk = cluster.map_shared_rank(orig, own_k)[k - own_k * RP];
    }
    __syncthreads();
    const int r = s_r;
    const int own_r = r / RP, own_k = k / RP;
    {
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
    if (c == own_r && r != k) {
      for (int j = tid; j < nb; j += kThreads) P[(r - r0) * nb + j] = tmp[j];
      if (tid == 0) orig[r - r0] = s_origk;
    }
    if (c == own_k && tid == 0) orig[k - r0] = s_origr;
    __syncthreads();
    for (int i = r0 + warp; i < r1; i += kThreads / 32) {
      zt* rw = P + (i - r0) * nb;
      if (i == k) {
        for (int j = lane; j < nb; j += 32) rw[j] = prow[j];
      } else {
        const zt f = rw[kk];
        __syncwarp();
        for (int j = lane; j < nb; j += 32) {
          zt v = (j == kk) ? make_double2(0.0, 0.0) : rw[j];
          const zt pj = prow[j];
          v.x -= f.x * pj.x - f.y * pj.y;
          v.y -= f.x * pj.y + f.y * pj.x;
          rw[j] = v;
        }
      }
    }
    if (c == 0 && tid == 0) piv[k] = r;
    __syncthreads();
  }
  for (int e = tid; e < nr * nb; e += kThreads) {
    const int i = e / nb, j = e % nb;
    Yb[(int64_t)(r0 + i) * a.ldy + k0 + j] = P[i * nb + j];
  }
  for (int i = tid; i < nr; i += kThreads) write_maps(a, b, r0 + i, orig[i]);
  if (singular && c == 0 && tid == 0) atomicCAS(a.info, 0, b + 1);
  cluster.sync();
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Fused whole-matrix Gauss-Jordan, n <= 256: one CTA (8 warps) per matrix, in place.
// For each panel of w <= NB = 28 columns:
//  * panel phase: thread i owns row i of the panel in registers (as zgj_panel_reg: packed-key
//    REDUX pivot search, raw pivot-row broadcast, rotated rows); the transform T is written
//    back to the panel columns and each warp then holds its 32 rows of T as DMMA A fragments
//    in registers for the whole update phase;
//  * update phase (FP64 tensor cores): the other columns, in chunks of CH, are gathered
//    through the panel's row permutation by cp.async into a double-buffered shared stage
//    (chunk c+1 is in flight while chunk c is computed); panel rows of the stage are the
//    B operand Z, the other rows seed the accumulators, C += T Z runs as m8n8k4 DMMAs
//    (complex = 4 real products) and the chunk is stored back in place.
// No ping-pong buffer and no launch per panel.  The column swaps are undone while writing the
// result to `out`.  Dynamic shared memory: stage [2][n][CH + 2] complex.
// ---------------------------------------------------------------------------
constexpr int FU_NB = 28;

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}

template <int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) zgj_fused_kernel(zt* __restrict__ A, int64_t lda, int64_t bs,
                                                              zt* __restrict__ out, int64_t ldo, int64_t obs, int n,
                                                              int* __restrict__ info) {
  constexpr int NB = FU_NB, SS = CH + 2, NW = 8, TN = CH / 8, K4 = NB / 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zt* stage = reinterpret_cast<zt*>(smem_raw);  // [2][n][SS]
  __shared__ zt prow[NB], tmp[NB];
  __shared__ unsigned wkey[NW];
  __shared__ int s_orig_r, s_orig_k;
  __shared__ int piv_s[256], pi_s[256], orig_s[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  zt* Ab = A + (int64_t)b * bs;
  const int i = tid;
  const bool live = i < n;
  const int sbuf = n * SS;
  bool singular = false;
  for (int k0 = 0; k0 < n; k0 += NB) {
    const int w = min(NB, n - k0);
    {  // ---- panel phase ----
      int orig = i;
      zt row[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) row[j] = (live && j < w) ? Ab[(int64_t)i * lda + k0 + j] : make_double2(0.0, 0.0);
      for (int kk = 0; kk < w; ++kk) {
        const int k = k0 + kk;
        const unsigned key = __reduce_max_sync(0xffffffffu, pivot_key(row[0], i, live && i >= k));
        if (lane == 0) wkey[warp] = key;
        __syncthreads();
        unsigned best = wkey[0];
#pragma unroll
        for (int w2 = 1; w2 < NW; ++w2) best = max(best, wkey[w2]);
        int r = 511 - (int)(best & 511u);
        if ((best & ~511u) == 0u) {
          singular = true;
          r = k;
        }
        if (i == r) {
#pragma unroll
          for (int j = 0; j < NB; ++j) prow[j] = row[j];
          s_orig_r = orig;
        }
        if (i == k && r != k) {
#pragma unroll
          for (int j = 0; j < NB; ++j) tmp[j] = row[j];
          s_orig_k = orig;
        }
        __syncthreads();
        const zt inv = zinv_fast(prow[0]);
        if (i == k) {
          row_pivot<NB>(row, prow, inv);
          orig = s_orig_r;
        } else {
          if (i == r) {
#pragma unroll
            for (int j = 0; j < NB; ++j) row[j] = tmp[j];
            orig = s_orig_k;
          }
          row_step<NB>(row, prow, inv);
        }
        row_rotate<NB>(row);
        if (tid == 0) piv_s[k] = r;
      }
      // after w rotations register slot p holds panel column (p + w) mod NB
      if (live) {
#pragma unroll
        for (int p = 0; p < NB; ++p) {
          int j = p + w;
          if (j >= NB) j -= NB;
          if (j < w) Ab[(int64_t)i * lda + k0 + j] = row[p];
        }
      }
      orig_s[i] = live ? orig : 0;
    }
    __syncthreads();  // T and the previous panel's update visible to every thread
    const int nc = n - w;
    if (nc <= 0) continue;
    // A fragments of T for this warp's rows (register resident for the whole update phase)
    const int rbase = warp * 32;
    zt af[4][K4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int rr = min(rbase + mi * 8 + (lane >> 2), n - 1);
#pragma unroll
      for (int k4 = 0; k4 < K4; ++k4) {
        const int kc = k4 * 4 + (lane & 3);
        af[mi][k4] = kc < w ? Ab[(int64_t)rr * lda + k0 + kc] : make_double2(0.0, 0.0);
      }
    }
    // chunk gather: thread t copies row t's CH elements of the permuted matrix into the stage
    auto gather = [&](int c0, int buf) {
      if (live) {
        const zt* src = Ab + (int64_t)orig_s[i] * lda;
        zt* dst = stage + buf * sbuf + i * SS;
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) {
          const int cj = min(c0 + jj, nc - 1);  // clamp: tail columns are never stored
          cpa16(dst + jj, src + (cj < k0 ? cj : cj + w));
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    gather(0, 0);
    int buf = 0;
    for (int c0 = 0; c0 < nc; c0 += CH, buf ^= 1) {
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();  // chunk c staged by every thread; chunk c-1 fully consumed
      if (c0 + CH < nc) gather(c0 + CH, buf ^ 1);
      const zt* sg = stage + buf * sbuf;
      if (rbase < n) {
        double accr[4][TN][2], acci[4][TN][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int rr = rbase + mi * 8 + (lane >> 2);
          const bool seed = rr < n && !(rr >= k0 && rr < k0 + w);
#pragma unroll
          for (int ni = 0; ni < TN; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const zt v = seed ? sg[rr * SS + ni * 8 + (lane & 3) * 2 + h] : make_double2(0.0, 0.0);
              accr[mi][ni][h] = v.x;
              acci[mi][ni][h] = v.y;
            }
        }
#pragma unroll
        for (int k4 = 0; k4 < K4; ++k4) {
          zt bf[TN];
          const int kr = k4 * 4 + (lane & 3);
#pragma unroll
          for (int ni = 0; ni < TN; ++ni)
            bf[ni] = kr < w ? sg[(k0 + kr) * SS + ni * 8 + (lane >> 2)] : make_double2(0.0, 0.0);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < TN; ++ni) dmma884(accr[mi][ni][0], accr[mi][ni][1], af[mi][k4].x, bf[ni].x);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < TN; ++ni) dmma884(acci[mi][ni][0], acci[mi][ni][1], af[mi][k4].x, bf[ni].y);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < TN; ++ni) dmma884(accr[mi][ni][0], accr[mi][ni][1], -af[mi][k4].y, bf[ni].y);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < TN; ++ni) dmma884(acci[mi][ni][0], acci[mi][ni][1], af[mi][k4].y, bf[ni].x);
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int rr = rbase + mi * 8 + (lane >> 2);
          if (rr >= n) continue;
          zt* dst = Ab + (int64_t)rr * lda;
#pragma unroll
          for (int ni = 0; ni < TN; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cj = c0 + ni * 8 + (lane & 3) * 2 + h;
              if (cj < nc) dst[cj < k0 ? cj : cj + w] = make_double2(accr[mi][ni][h], acci[mi][ni][h]);
            }
        }
      }
    }
    __syncthreads();  // last chunk stored before the next panel reads
  }
  // undo the column swaps: out(i, j) = A(i, pi(j)),  pi = S_{n-1} o ... o S_0
  if (tid == 0) {
    for (int j = 0; j < n; ++j) pi_s[j] = j;
    for (int k = n - 1; k >= 0; --k) {
      const int r = piv_s[k];
      const int t = pi_s[k];
      pi_s[k] = pi_s[r];
      pi_s[r] = t;
    }
  }
  __syncthreads();
  zt* ob = out + (int64_t)b * obs;
  for (int e = tid; e < n * n; e += 256) {
    const int r = e / n, j = e % n;
    ob[(int64_t)r * ldo + j] = Ab[(int64_t)r * lda + pi_s[j]];
  }
  if (singular && tid == 0) atomicCAS(info, 0, b + 1);
}

// ---------------------------------------------------------------------------
// Warp-specialised Gauss-Jordan with look-ahead, n <= WS_NMAX: one CTA of 16 warps per matrix.
// Implicit partial pivoting: rows never move.  The pivot of global step k is row plist[k]
// (pstep[row] = k); at the end the in-place matrix M satisfies A^{-1}(k, j) = M(plist[k],
// pstep[j]) (the row and column permutations of the row pivoting; checked against the textbook
// blocked GJ in tests/test_gpu_parity.py::test_zinv_*).
//  * panel warps 0-7 (thread i owns row i): factor panel p+1 (w <= 28 columns, pivot search
//    over the rows not yet pivoted, ONE barrier per step: every warp publishes its best
//    candidate row, all threads pick the winner), then write T (the factored panel columns)
//    to shared memory and back in place;
//  * update warps 8-15 (FP64 tensor cores): for panel p, stage Z = the old pivot rows of p
//    (all other columns) in shared memory by cp.async, then C(i, J) = [i not a pivot of p]
//    C(i, J) + T(i, :) Z(:, J) for every other column J as m8n8k4 DMMAs (complex = 4 real
//    products), accumulators seeded straight from global memory.  The columns of panel p+1
//    are updated first and released to the panel warps (named barrier), so the panel
//    factorisation of p+1 overlaps the rest of the update of p.
// The matrix stays in L2 (one CTA per SM: 148 x 614 KB at n = 196), every pass reads and
// writes it once; T and Z live in shared memory.
// ---------------------------------------------------------------------------
constexpr int WS_NB = 28, WS_NMAX = 240;
// 1: the leaf Schur inverse pivots from the start (HPS_SEQ_PIVOT=1; tests of the fallback path)
__constant__ int g_seq_pivot;
// test: the natural-order leaf Schur elimination reports a failed pivot check at step 100 (after
// it has overwritten its in-place work matrix), so the pivoted fallback must rebuild everything
__constant__ int g_seq_force_bad;
// optional timeline of CTA 0 (clock64 per milestone, hps_debug_ws_trace): [panel][10]
__device__ long long g_ws_trace[16 * 16];
__device__ int g_ws_trace_on;
#define WS_MARK(p, slot)                                                              \
  do {                                                                                \
    if (trace && (p) < 16) g_ws_trace[(p) * 16 + (slot)] = clock64();                 \
  } while (0)
enum { BAR_PANEL = 1, BAR_UPD = 2, BAR_READY = 3, BAR_TFREE = 4, BAR_TREADY = 5 };

__device__ __forceinline__ void bar_sync_n(int id, int cnt) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int cnt) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(cnt) : "memory");
}
__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;\n" ::: "memory"); }
__device__ __forceinline__ void cpa16_zfill(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(valid ? 16 : 0));
}

struct WsPanels {
  int npan, base, rem;
  __device__ __forceinline__ int k0(int p) const { return p * base + min(p, rem); }
  __device__ __forceinline__ int w(int p) const { return p < npan ? base + (p < rem ? 1 : 0) : 0; }
};

// Leaf epilogue (leaf_mode 0): instead of writing S^{-1} alone, the CTA that
// inverted S forms the whole leaf operator [Psi | Y] = B^{-1} and the leaf R from it:
//   Y_i = S^{-1},  Psi_i = S^{-1} U,  Y_b = -V S^{-1},  Psi_b = G - V Psi_i,  R = I - 2 i eta Psi_b
// (U, V, G act along one grid line each; constants K from schur_consts).  S^{-1} is read once,
// one x-line (q rows) at a time into shared memory; the y-line sums accumulate in shared memory.
struct WsFinish {
  const zt* K;   // schur_consts: Lx, Ly, Ubx, Uby, Vx, Vy, Gx, Gy
  zt* R;         // leaf R of batch entry 0 (nb x nb, batch stride nb*nb)
  zt m2ieta;     // -2 i eta
  int p;         // 0 = plain inverse output
  // fused assembly of S = Lx (+) Ly - kappa^2 diag(c) (leaf_schur_assemble, DESIGN 3.1) into the
  // CTA's work matrix before the elimination (c == nullptr: S is given)
  const zt* c;           // c samples, natural leaf order, p*p per leaf
  const int* leaf_nat;   // heap leaf -> natural leaf
  int leaf0;             // heap index of batch entry 0
  double kappa2;
  int blockpanel = 0;    // natural-order panels in block form (knob leaf_panel, DESIGN 3.12)
  int inplace = 1;       // natural order: eliminate in the store's Y_i block (knob leaf_inplace)
};

__host__ __device__ inline int ws_zs(int n) {  // Z row stride: >= n - wmin + 16, == 2 (mod 8)
  const int npan = (n + WS_NB - 1) / WS_NB;
  const int need = n - n / npan + 16;
  return ((need - 2 + 7) / 8) * 8 + 2;
}
__host__ __device__ inline size_t ws_smem(int n) {
  return sizeof(zt) * ((size_t)((n + 15) & ~15) * WS_NB + (size_t)WS_NB * ws_zs(n));
}

// Output of the in-place Gauss-Jordan result M (pivot lists plist / pstep in shared memory):
// the plain inverse (fin.p == 0) or the fused leaf epilogue.  All 512 threads of the CTA.
// ident: the pivot lists are the identity (natural order); then the fused epilogue fetches each
// chunk of S^{-1} rows with cp.async (all requests in flight at once), and if M is the output's
// own Y_i block (the natural-order leaf inverse runs in place in the store) Y_i is not copied.
__device__ __forceinline__ void ws_output(const zt* __restrict__ M, int64_t lda, zt* __restrict__ out, int64_t ldo,
                                          int64_t obs, int n, const WsFinish& fin, const int* plist,
                                          const int* pstep, unsigned char* smem_raw, bool ident = false) {
  const int tid = threadIdx.x;
  zt* ob = out + (int64_t)blockIdx.x * obs;
  const bool inplace = ident && M == ob && lda == ldo;
  if (fin.p == 0) {
    // A^{-1}(k, j) = M(plist[k], pstep[j])
    for (int e = tid; e < n * n; e += 512) {
      const int k = e / n, j = e - k * n;
      __stcs(&ob[(int64_t)k * ldo + j], ldplain(M + (int64_t)plist[k] * lda + pstep[j]));
    }
    return;
  }
  // ---- fused leaf epilogue (n = n_i = q^2, ldo = n_t); outputs are streamed past L2 (st.cs) so the
  // in-place matrices of the other CTAs stay resident ----
  const int q = fin.p - 2, ni = n, nb = 4 * q, nt = (int)ldo;
  zt* base = ob - ((int64_t)nb * nt + nb);  // leaf operator [Psi | Y], rows [I_b; I_i]
  zt* Rl = fin.R + (int64_t)blockIdx.x * nb * nb;
  // two x-lines per chunk (7 synchronised rounds instead of 14 at q = 14); the y-line sums of
  // Y_b live in registers (11 per thread), those of Psi_b in shared memory
  constexpr int LPC = 2, AY = 11;  // lines per chunk; ceil(2 q n_i / 512) for n_i <= 200
  zt* C = reinterpret_cast<zt*>(smem_raw);  // [LPC][q][ni]  S^{-1} rows of the chunk's x-lines
  zt* Pc = C + LPC * q * ni;                 // [LPC][q][nb]  Psi_i rows of the chunk's x-lines
  zt* accP = Pc + LPC * q * nb;              // [2q][nb]      y-line sums for Psi_b
  zt* Kc = accP + 2 * q * nb;                // Ubx, Uby, Vx, Vy (2q each), Gx, Gy (4 each)
  for (int e = tid; e < 8 * q + 8; e += 512) Kc[e] = fin.K[2 * q * q + e];  // out of the inner loops
  const zt* Ubx = Kc;
  const zt* Uby = Ubx + 2 * q;
  const zt* Vx = Uby + 2 * q;
  const zt* Vy = Vx + 2 * q;
  const zt* Gx = Vy + 2 * q;
  const zt* Gy = Gx + 4;
  const zt m2 = fin.m2ieta;
  auto zmac = [](zt& acc, zt a, zt b) {
    acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  };
  auto put_psib = [&](int row, int b2, zt v) {  // Psi_b entry and the matching R entry
    __stcs(&base[(int64_t)row * nt + b2], v);
    zt r = make_double2(m2.x * v.x - m2.y * v.y, m2.x * v.y + m2.y * v.x);
    if (row == b2) r.x += 1.0;
    __stcs(&Rl[row * nb + b2], r);
  };
  zt accY[AY];  // entry e = tid + 512 i of the [2q][ni] y-line sums (S rows, then N rows)
#pragma unroll
  for (int i = 0; i < AY; ++i) accY[i] = make_double2(0.0, 0.0);
  for (int e = tid; e < 2 * q * nb; e += 512) accP[e] = make_double2(0.0, 0.0);
  const bool etr = g_ws_trace_on == n && blockIdx.x == 0 && tid == 0;
  long long et[6] = {0, 0, 0, 0, 0, 0}, em = clock64();
  auto emark = [&](int i) {
    if (etr) {
      const long long c = clock64();
      et[i] += c - em;
      em = c;
    }
  };
  for (int kx0 = 0; kx0 < q; kx0 += LPC) {  // x-lines iy = kx0 .. kx0 + LPC - 1
    const int nl = min(LPC, q - kx0);
    __syncthreads();
    emark(0);
    if (ident) {
      for (int e = tid; e < nl * q * ni; e += 512) {
        const int t = e / ni, j = e - t * ni;  // t = line-local row l*q + t'
        cpa16_zfill(C + e, M + (int64_t)(kx0 * q + t) * lda + j, true);
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      if (!inplace)
        for (int e = tid; e < nl * q * ni; e += 512) {
          const int t = e / ni, j = e - t * ni;
          __stcs(&base[(int64_t)(nb + kx0 * q + t) * nt + nb + j], C[e]);  // Y_i
        }
    } else {
      for (int e = tid; e < nl * q * ni; e += 512) {
        const int t = e / ni, j = e - t * ni;  // t = line-local row l*q + t'
        const zt v = ldplain(M + (int64_t)plist[kx0 * q + t] * lda + pstep[j]);
        C[e] = v;
        __stcs(&base[(int64_t)(nb + kx0 * q + t) * nt + nb + j], v);  // Y_i
      }
      __syncthreads();
    }
    emark(1);
    // Psi_i rows of these lines: thread (row t, line kk) forms the four entries fed by line kk --
    // W, E from x-line iy = kk (14 contiguous entries of the row) and S, N from y-line ix = kk --
    // as four independent accumulation chains over one pass of 14 terms
    for (int e = tid; e < nl * q * q; e += 512) {
      const int t = e / q, kk = e - t * q;
      const zt* Cx = C + t * ni + kk * q;  // x-line iy = kk
      const zt* Cy = C + t * ni + kk;      // y-line ix = kk (stride q)
      zt aw = make_double2(0.0, 0.0), ae = aw, as = aw, an = aw;
#pragma unroll 7
      for (int t2 = 0; t2 < q; ++t2) {
        const zt vx = Cx[t2], vy = Cy[t2 * q];
        zmac(aw, vx, Ubx[t2 * 2 + 0]);
        zmac(ae, vx, Ubx[t2 * 2 + 1]);
        zmac(as, vy, Uby[t2 * 2 + 0]);
        zmac(an, vy, Uby[t2 * 2 + 1]);
      }
      zt* pr = Pc + t * nb;
      pr[kk] = as;
      pr[q + kk] = ae;
      pr[2 * q + kk] = an;
      pr[3 * q + kk] = aw;
      zt* orow = base + (int64_t)(nb + kx0 * q + t) * nt;
      __stcs(&orow[kk], as);
      __stcs(&orow[q + kk], ae);
      __stcs(&orow[2 * q + kk], an);
      __stcs(&orow[3 * q + kk], aw);
    }
    emark(2);
    // Y_b: W_kx, E_kx complete on each line; S/N (y-lines) accumulate in registers
    for (int e = tid; e < nl * ni; e += 512) {
      const int l = e / ni, j = e - l * ni, kx = kx0 + l;
      zt w0 = make_double2(0.0, 0.0), w1 = make_double2(0.0, 0.0);
      zt w2 = make_double2(0.0, 0.0), w3 = make_double2(0.0, 0.0);
#pragma unroll 7
      for (int t = 0; t + 1 < q; t += 2) {
        const zt v = C[(l * q + t) * ni + j], v1 = C[(l * q + t + 1) * ni + j];
        zmac(w0, Vx[t], v);
        zmac(w1, Vx[q + t], v);
        zmac(w2, Vx[t + 1], v1);
        zmac(w3, Vx[q + t + 1], v1);
      }
      if (q & 1) {
        const zt v = C[(l * q + q - 1) * ni + j];
        zmac(w0, Vx[q - 1], v);
        zmac(w1, Vx[2 * q - 1], v);
      }
      w0.x += w2.x;
      w0.y += w2.y;
      w1.x += w3.x;
      w1.y += w3.y;
      __stcs(&base[(int64_t)(3 * q + kx) * nt + nb + j], make_double2(-w0.x, -w0.y));
      __stcs(&base[(int64_t)(q + kx) * nt + nb + j], make_double2(-w1.x, -w1.y));
    }
#pragma unroll
    for (int i = 0; i < AY; ++i) {  // node (ix = kk, iy = kx) is position kx of y-line kk
      const int e = tid + 512 * i;
      if (e < 2 * q * ni) {
        const int half = e >= q * ni, r = e - half * q * ni, kk = r / ni, j = r - kk * ni;
        for (int l = 0; l < nl; ++l) zmac(accY[i], Vy[half * q + kx0 + l], C[(l * q + kk) * ni + j]);
      }
    }
    __syncthreads();  // Pc complete
    emark(3);
    for (int e = tid; e < nl * nb; e += 512) {
      const int l = e / nb, b2 = e - l * nb, kx = kx0 + l;
      zt w0 = make_double2(0.0, 0.0), w1 = make_double2(0.0, 0.0);
      zt w2 = make_double2(0.0, 0.0), w3 = make_double2(0.0, 0.0);
#pragma unroll 7
      for (int t = 0; t + 1 < q; t += 2) {
        const zt v = Pc[(l * q + t) * nb + b2], v1 = Pc[(l * q + t + 1) * nb + b2];
        zmac(w0, Vx[t], v);
        zmac(w1, Vx[q + t], v);
        zmac(w2, Vx[t + 1], v1);
        zmac(w3, Vx[q + t + 1], v1);
      }
      if (q & 1) {
        const zt v = Pc[(l * q + q - 1) * nb + b2];
        zmac(w0, Vx[q - 1], v);
        zmac(w1, Vx[2 * q - 1], v);
      }
      w0.x += w2.x;
      w0.y += w2.y;
      w1.x += w3.x;
      w1.y += w3.y;
      const int e2 = b2 / q, k2 = b2 - e2 * q;
      zt g0 = make_double2(0.0, 0.0), g1 = make_double2(0.0, 0.0);
      if (k2 == kx && (e2 == 1 || e2 == 3)) {
        g0 = Gx[0 * 2 + (e2 == 3 ? 0 : 1)];
        g1 = Gx[1 * 2 + (e2 == 3 ? 0 : 1)];
      }
      put_psib(3 * q + kx, b2, make_double2(g0.x - w0.x, g0.y - w0.y));
      put_psib(q + kx, b2, make_double2(g1.x - w1.x, g1.y - w1.y));
    }
    for (int e = tid; e < q * nb; e += 512) {
      const int kk = e / nb, b2 = e - kk * nb;
      for (int l = 0; l < nl; ++l) {
        const zt v = Pc[(l * q + kk) * nb + b2];
        zmac(accP[kk * nb + b2], Vy[kx0 + l], v);
        zmac(accP[(q + kk) * nb + b2], Vy[q + kx0 + l], v);
      }
    }
  }
  __syncthreads();
  emark(4);
  if (etr)
    for (int i = 0; i < 5; ++i) g_ws_trace[15 * 16 + 4 + i] = et[i];
  // y-lines: S_kk (row kk) and N_kk (row 2q + kk)
#pragma unroll
  for (int i = 0; i < AY; ++i) {
    const int e = tid + 512 * i;
    if (e < 2 * q * ni) {
      const int half = e >= q * ni, r = e - half * q * ni, kk = r / ni, j = r - kk * ni;
      __stcs(&base[(int64_t)(half * 2 * q + kk) * nt + nb + j], make_double2(-accY[i].x, -accY[i].y));
    }
  }
  for (int e = tid; e < q * nb; e += 512) {
    const int kk = e / nb, b2 = e - kk * nb, e2 = b2 / q, k2 = b2 - e2 * q;
    const zt a0 = accP[kk * nb + b2], a1 = accP[(q + kk) * nb + b2];
    zt g0 = make_double2(0.0, 0.0), g1 = make_double2(0.0, 0.0);
    if (k2 == kk && (e2 == 0 || e2 == 2)) {
      g0 = Gy[0 * 2 + (e2 == 0 ? 0 : 1)];
      g1 = Gy[1 * 2 + (e2 == 0 ? 0 : 1)];
    }
    put_psib(kk, b2, make_double2(g0.x - a0.x, g0.y - a0.y));
    put_psib(2 * q + kk, b2, make_double2(g1.x - a1.x, g1.y - a1.y));
  }
}

__global__ void __launch_bounds__(512, 1) zgj_ws_kernel(zt* __restrict__ A, int64_t lda, int64_t bs,
                                                        zt* __restrict__ out, int64_t ldo, int64_t obs, int n,
                                                        int* __restrict__ info, const WsFinish fin) {
  constexpr int NB = WS_NB, CPT = WS_NB / 4;  // panel columns, columns per panel thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int mtr = (n + 15) & ~15, zs = ws_zs(n);
  zt* Ts = reinterpret_cast<zt*>(smem_raw);  // [mtr][NB]  T of the current panel (16-row pairs)
  zt* Zs = Ts + (size_t)mtr * NB;            // [NB][zs]   old pivot rows, virtual column order
  __shared__ zt prow4[2][NB];
  __shared__ __align__(16) unsigned wkey4[2][8];
  __shared__ int pstep[256], plist[256], colmap[WS_NMAX + 16];
  const int tid = threadIdx.x, lane = tid & 31;
  zt* M = A + (int64_t)blockIdx.x * bs;
  WsPanels P;
  P.npan = (n + NB - 1) / NB;
  P.base = n / P.npan;
  P.rem = n % P.npan;
  if (tid < 256) pstep[tid] = 1 << 30;
  const bool trace = g_ws_trace_on && blockIdx.x == 0 && (tid == 0 || tid == 256);
  if (fin.c) {  // assemble S in place (row iy*q + ix, Lx along x-lines, Ly along y-lines)
    const int q = fin.p - 2;
    const zt* Lx = fin.K;
    const zt* Ly = fin.K + q * q;
    const zt* cl = fin.c + (int64_t)fin.leaf_nat[fin.leaf0 + blockIdx.x] * fin.p * fin.p;
    for (int r = tid >> 5; r < n; r += 16) {
      const int ix = r % q, iy = r / q;
      for (int cc = tid & 31; cc < n; cc += 32) {
        const int jx = cc % q, jy = cc / q;
        zt v = make_double2(0.0, 0.0);
        if (iy == jy) v = Lx[ix * q + jx];
        if (ix == jx) {
          v.x += Ly[iy * q + jy].x;
          v.y += Ly[iy * q + jy].y;
        }
        if (r == cc) {
          const zt cv = cl[(iy + 1) * fin.p + ix + 1];
          v.x -= fin.kappa2 * cv.x;
          v.y -= fin.kappa2 * cv.y;
        }
        M[(int64_t)r * lda + cc] = v;
      }
    }
    fence_cta();
  }
  __syncthreads();

  // roles: panel warps 8-15 (latency-critical; the SMSP arbiter favours high warp ids),
  // update warps 0-7
  if (tid >= 256) {
    // ================= panel warps =================
    // Thread = 4 rows x 7 columns of the panel (rows wp*32 + q*8 + rg, q = 0..3; columns
    // cg*7 + c): per step each warp reads only 7 + 1 pivot-row elements from shared memory
    // (a 128-bit LDS costs 4 crossbar cycles even as a broadcast, so one-row-per-thread
    // panels are bound by the pivot-row broadcast), the multipliers of its rows travel by
    // shuffle from the lane holding the active column.  Two barriers per step: pivot keys,
    // then the winning row (published raw by its 4 lanes).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
    const int pt = tid - 256, wp = pt >> 5, cg = lane & 3, rg = lane >> 2;
    int rq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rq[q] = wp * 32 + q * 8 + rg;
    bool piv[4] = {false, false, false, false};
    bool singular = false;
    const bool warp_live = wp * 32 < n;
    for (int p = 0; p < P.npan; ++p) {
      const int k0 = P.k0(p), w = P.w(p);
      if (p > 0) bar_sync_n(BAR_READY, 512);  // columns of p updated by pass p-1
      WS_MARK(p, 0);
      zt a[4][CPT];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int j = cg * CPT + c;
          a[q][c] = (rq[q] < n && j < w) ? ldplain(M + (int64_t)rq[q] * lda + k0 + j) : make_double2(0.0, 0.0);
        }
      for (int cga = 0; cga * CPT < w; ++cga) {
        const bool act = cg == cga;
        const int src = (lane & ~3) | cga;
#pragma unroll
        for (int s = 0; s < CPT; ++s) {
          const int kk = cga * CPT + s;
          if (kk < w) {
            const int k = k0 + kk, par = k & 1;
            unsigned key = 0u;
            if (act) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (!piv[q] && rq[q] < n) key = max(key, pivot_key(a[q][s], rq[q], true));
            }
            key = __reduce_max_sync(0xffffffffu, key);
            if (lane == 0) wkey4[par][wp] = key;
            bar_sync_n(BAR_PANEL, 256);
            const uint4 k03 = *reinterpret_cast<const uint4*>(&wkey4[par][0]);
            const uint4 k47 = *reinterpret_cast<const uint4*>(&wkey4[par][4]);
            const unsigned best =
                max(max(max(k03.x, k03.y), max(k03.z, k03.w)), max(max(k47.x, k47.y), max(k47.z, k47.w)));
            if ((best & ~511u) == 0u) singular = true;
            const int r = 511 - (int)(best & 511u);
            if (wp == (r >> 5) && rg == (r & 7)) {  // the 4 lanes of row r publish it raw
              const int qq = (r >> 3) & 3;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (q == qq) {
#pragma unroll
                  for (int c = 0; c < CPT; ++c) prow4[par][cg * CPT + c] = a[q][c];
                }
              if (cg == 0) {
                pstep[r] = k;
                plist[k] = r;
              }
            }
            bar_sync_n(BAR_PANEL, 256);
            if (warp_live) {
              const zt inv = zinv_fast(prow4[par][kk]);
              zt g[4];
              bool isp[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const zt v = a[q][s];
                g[q] = zmul(make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)), inv);
                isp[q] = rq[q] == r;
              }
              if (wp == (r >> 5)) {  // warp-uniform: the warp holding the pivot row
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (isp[q]) {  // pivot row: a <- pr / pivot exactly (as 0 - (-inv) pr)
                    piv[q] = true;
                    g[q] = make_double2(-inv.x, -inv.y);
#pragma unroll
                    for (int c = 0; c < CPT; ++c) a[q][c] = make_double2(0.0, 0.0);
                  }
              }
#pragma unroll
              for (int c = 0; c < CPT; ++c) {
                const zt pc = prow4[par][cg * CPT + c];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  a[q][c].x = fma(-g[q].x, pc.x, a[q][c].x);
                  a[q][c].y = fma(-g[q].x, pc.y, a[q][c].y);
                  a[q][c].x = fma(g[q].y, pc.y, a[q][c].x);
                  a[q][c].y = fma(-g[q].y, pc.x, a[q][c].y);
                }
              }
              if (act) {  // active column: -g (= 1/pivot on the pivot row)
#pragma unroll
                for (int q = 0; q < 4; ++q) a[q][s] = make_double2(-g[q].x, -g[q].y);
              }
            }
          }
        }
      }
      WS_MARK(p, 1);
      if (p > 0) bar_sync_n(BAR_TFREE, 512);  // update warps done with T / Z of p-1
      WS_MARK(p, 2);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (rq[q] < mtr) {
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const int j = cg * CPT + c;
            Ts[rq[q] * NB + j] = j < w ? a[q][c] : make_double2(0.0, 0.0);
            if (j < w && rq[q] < n) M[(int64_t)rq[q] * lda + k0 + j] = a[q][c];
          }
        }
      fence_cta();
      bar_arrive_n(BAR_TREADY, 512);
      WS_MARK(p, 3);
    }
    if (singular && pt == 0) atomicCAS(info, 0, blockIdx.x + 1);
  } else {
    // ================= update warps =================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
    const int u = tid, uw = u >> 5;
    const int MT = mtr >> 3;
    for (int p = 0; p < P.npan; ++p) {
      const int k0 = P.k0(p), w = P.w(p), w4 = (w + 3) & ~3, K4 = w4 >> 2;
      const bool has_next = p + 1 < P.npan;
      const int w1 = has_next ? P.w(p + 1) : 0;
      const int nv = n - w;
      // virtual column v -> actual: [0, w1) = panel p+1, then [0, k0) and [k0 + w + w1, n)
      auto act = [&](int v) {
        if (v < w1) return k0 + w + v;
        v -= w1;
        return v < k0 ? v : v + w + w1;
      };
      bar_sync_n(BAR_TREADY, 512);
      WS_MARK(p, 4);
      for (int v = u; v < nv + 16; v += 256) colmap[v] = v < nv ? act(v) : -1;
      // stage Z (two cp.async groups: the columns of panel p+1, then the rest)
      for (int part = 0; part < 2; ++part) {
        const int v0 = part ? w1 : 0, nvp = part ? nv - w1 : w1;
        for (int e = u; e < w4 * nvp; e += 256) {
          const int m = e / nvp, v = v0 + e - m * nvp;
          const bool ok = m < w;
          const int srow = ok ? plist[k0 + m] : 0;
          cpa16_zfill(Zs + m * zs + v, M + (int64_t)srow * lda + act(v), ok);
        }
        asm volatile("cp.async.commit_group;\n" ::);
      }
      for (int part = 0; part < 2; ++part) {
        const int v0 = part ? w1 : 0, v1 = part ? nv : w1;
        if (part == 0) {
          if (!has_next) continue;
          asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
        bar_sync_n(BAR_UPD, 256);
        WS_MARK(p, 5 + 2 * part);
        const int NPR = (v1 - v0 + 15) >> 4;
        // unit = (m-tile mt, 16 virtual columns from v0 + 16 npr), dealt round-robin over the 8
        // update warps; the seeds of the next unit are prefetched into registers while the
        // current one runs on the tensor cores.  Column addresses come from colmap (no integer
        // division or branches on the issue path).
        struct Unit {
          int rr, col[2][2];
          bool rok;
          zt seed[2][2];
        };
        auto load_unit = [&](int mt, int npr, Unit& U) {
          U.rr = mt * 8 + (lane >> 2);
          const int rc = min(U.rr, n - 1);
          U.rok = U.rr < n && (unsigned)(pstep[rc] - k0) >= (unsigned)w;
          const int vb = v0 + npr * 16 + (lane & 3) * 2;
          const zt* rowp = M + (int64_t)rc * lda;
#pragma unroll
          for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int v = vb + t * 8 + h;
              U.col[t][h] = v < v1 ? colmap[v] : -1;
              U.seed[t][h] = ldplain(rowp + max(U.col[t][h], 0));  // masked at use: no wait here
            }
        };
        Unit cur, nxt;
        int mt = uw, npr = 0;
        while (mt >= MT) {
          mt -= MT;
          ++npr;
        }
        bool have = npr < NPR;
        if (have) load_unit(mt, npr, nxt);
        while (have) {
          cur = nxt;
          const int cmt = mt, cnpr = npr;
          mt += 8;
          while (mt >= MT) {
            mt -= MT;
            ++npr;
          }
          have = npr < NPR;
          if (have) load_unit(mt, npr, nxt);
          const int vb = v0 + cnpr * 16;
          double ar[2][2], ai[2][2];
#pragma unroll
          for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const bool ok = cur.rok && cur.col[t][h] >= 0;
              ar[t][h] = ok ? cur.seed[t][h].x : 0.0;
              ai[t][h] = ok ? cur.seed[t][h].y : 0.0;
            }
          const zt* Trow = Ts + (cmt * 8 + (lane >> 2)) * NB + (lane & 3);
          const zt* Zc = Zs + (lane & 3) * zs + vb + (lane >> 2);
#pragma unroll 7
          for (int k4 = 0; k4 < K4; ++k4) {
            const zt a = Trow[k4 * 4];
            const zt b0 = Zc[k4 * 4 * zs], b1 = Zc[k4 * 4 * zs + 8];
            dmma884(ar[0][0], ar[0][1], a.x, b0.x);
            dmma884(ar[1][0], ar[1][1], a.x, b1.x);
            dmma884(ai[0][0], ai[0][1], a.x, b0.y);
            dmma884(ai[1][0], ai[1][1], a.x, b1.y);
            dmma884(ar[0][0], ar[0][1], -a.y, b0.y);
            dmma884(ar[1][0], ar[1][1], -a.y, b1.y);
            dmma884(ai[0][0], ai[0][1], a.y, b0.x);
            dmma884(ai[1][0], ai[1][1], a.y, b1.x);
          }
          if (cur.rr < n) {
            zt* rowp = M + (int64_t)cur.rr * lda;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                if (cur.col[t][h] >= 0) rowp[cur.col[t][h]] = make_double2(ar[t][h], ai[t][h]);
          }
        }
        WS_MARK(p, 6 + 2 * part);
        if (part == 0) {
          fence_cta();
          bar_arrive_n(BAR_READY, 512);
        }
      }
      if (has_next) bar_arrive_n(BAR_TFREE, 512);
    }
  }
  __syncthreads();
  ws_output(M, lda, out, ldo, obs, n, fin, plist, pstep, smem_raw);
}

size_t ws_finish_smem(int p) {
  const size_t q = p - 2, ni = q * q, nb = 4 * q;
  return sizeof(zt) * (2 * q * ni + 2 * q * nb + 2 * q * nb + 8 * q + 8);
}

// ---------------------------------------------------------------------------
// Blocked path, 32 < n <= 4096 (large merge W): implicit-pivoting panel kernel.  A cluster of
// CS = ceil(n / 256) CTAs (one CTA, no cluster, for n <= 256); CTA c owns rows c*256 + ...,
// each thread 4 rows x 7 columns of the 28-column panel (layout of zgj_ws_kernel's panel
// warps).  One cluster barrier per step: every warp publishes its pivot key and its candidate
// row in its own shared memory, then every warp reads all keys through distributed shared
// memory, picks the winner and copies the winning row into a per-warp buffer.  Rows never
// move: the pivot of step k is row plist[k] (piv), the GEMM update reads the pivot rows
// through rowsrc and skips them through cinmap, and the result is unscrambled at the end as
// A^{-1}(k, j) = M(piv[k], pinv[j]).
// Keys: high bits of |z|^2 with the low 12 bits replaced by (4095 - row), so one unsigned max
// picks the largest magnitude and, within ~2^-8 relative, the lowest row.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned pivot_key12(zt f, int row) {
  const double m = f.x * f.x + f.y * f.y;
  const unsigned hi = (unsigned)(__double_as_longlong(m) >> 32);
  return (hi & ~4095u) | (unsigned)(4095 - row);
}

__device__ __forceinline__ void p47_sync(bool clustered) {
  if (clustered) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
}

// CG = 7-column groups per row: 4 -> 28-column panels, 256 rows per CTA; 2 -> 14-column panels,
// 512 rows per CTA (a single CTA up to n = 512).
template <int CG>
__global__ void __launch_bounds__(256, 1) zgj_panel47_kernel(const PanelArgs a) {
  constexpr int NB = 7 * CG, RPW = 128 / CG, RPC = 8 * RPW;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const bool clustered = CS > 1;
  const int c = clustered ? (int)cluster.block_rank() : 0;
  const int b = blockIdx.x / CS, n = a.n, k0 = a.k0, w = a.w;
  __shared__ zt wrow[2][8][NB];
  __shared__ __align__(16) unsigned wkey[2][8];
  __shared__ zt prw[8][NB];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, cg_ = lane % CG, rg = lane / CG;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  int rq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) rq[q] = c * RPC + wp * RPW + q * (32 / CG) + rg;
  // rows pivoted in earlier panels (pflag) are never candidates again
  int* pflag = a.pflag + (int64_t)b * n;
  bool pv[4], pthis[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    pv[q] = rq[q] < n && pflag[rq[q]] != 0;
    pthis[q] = false;
  }
  zt av[4][7];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int cc = 0; cc < 7; ++cc) {
      const int j = cg_ * 7 + cc;
      av[q][cc] = (rq[q] < n && j < w) ? __ldcg(Xb + (int64_t)rq[q] * a.ldx + k0 + j) : make_double2(0.0, 0.0);
    }
  const bool warp_live = c * RPC + wp * RPW < n;
  bool singular = false;
  for (int cga = 0; cga * 7 < w; ++cga) {
    const bool act = cg_ == cga;
    const int src = (lane - cg_) + cga;
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      const int kk = cga * 7 + s;
      if (kk < w) {
        const int k = k0 + kk, par = k & 1;
        unsigned key = 0u;
        if (act) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (!pv[q] && rq[q] < n) key = max(key, pivot_key12(av[q][s], rq[q]));
        }
        const unsigned wk = __reduce_max_sync(0xffffffffu, key);
        if (wk != 0u) {  // this warp's candidate row: its 4 lanes publish it raw
          const int lr = 4095 - (int)(wk & 4095u) - c * RPC - wp * RPW;  // local row in the warp
          if (rg == lr % (32 / CG)) {
            const int qq = lr / (32 / CG);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q == qq) {
#pragma unroll
                for (int cc = 0; cc < 7; ++cc) wrow[par][wp][cg_ * 7 + cc] = av[q][cc];
              }
          }
        }
        if (lane == 0) wkey[par][wp] = wk;
        p47_sync(clustered);
        // every warp: max over the CS x 8 warp keys of the cluster
        unsigned best = 0u;
        for (int e = lane; e < CS * 8; e += 32) {
          const unsigned* kp = clustered ? cluster.map_shared_rank(&wkey[par][0], e >> 3) : &wkey[par][0];
          best = max(best, kp[e & 7]);
        }
        best = __reduce_max_sync(0xffffffffu, best);
        if ((best & ~4095u) == 0u) singular = true;
        const int r = 4095 - (int)(best & 4095u);
        const int rc = r / RPC, rw = (r % RPC) / RPW;
        if (lane < NB) {
          const zt* sp = clustered ? cluster.map_shared_rank(&wrow[par][rw][0], rc) : &wrow[par][rw][0];
          prw[wp][lane] = sp[lane];
        }
        __syncwarp();
        if (c == 0 && tid == 0) piv[k] = r;
        if (warp_live) {
          const zt inv = zinv_fast(prw[wp][kk]);
          zt g[4];
          bool isp[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const zt v = av[q][s];
            g[q] = zmul(make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)), inv);
            isp[q] = rq[q] == r;
          }
          if (rc == c && rw == wp) {  // warp-uniform: the warp holding the pivot row
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (isp[q]) {  // pivot row: a <- pr / pivot exactly (as 0 - (-inv) pr)
                pv[q] = true;
                pthis[q] = true;
                g[q] = make_double2(-inv.x, -inv.y);
#pragma unroll
                for (int cc = 0; cc < 7; ++cc) av[q][cc] = make_double2(0.0, 0.0);
              }
          }
#pragma unroll
          for (int cc = 0; cc < 7; ++cc) {
            const zt pc = prw[wp][cg_ * 7 + cc];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              av[q][cc].x = fma(-g[q].x, pc.x, av[q][cc].x);
              av[q][cc].y = fma(-g[q].x, pc.y, av[q][cc].y);
              av[q][cc].x = fma(g[q].y, pc.y, av[q][cc].x);
              av[q][cc].y = fma(-g[q].y, pc.x, av[q][cc].y);
            }
          }
          if (act) {
#pragma unroll
            for (int q = 0; q < 4; ++q) av[q][s] = make_double2(-g[q].x, -g[q].y);
          }
        }
        __syncwarp();  // prw consumed before the next step overwrites it
      }
    }
  }
  // T into Y (natural rows), the GEMM maps of this panel
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (rq[q] < n) {
#pragma unroll
      for (int cc = 0; cc < 7; ++cc) {
        const int j = cg_ * 7 + cc;
        if (j < w) Yb[(int64_t)rq[q] * a.ldy + k0 + j] = av[q][cc];
      }
      a.cinmap[(int64_t)b * n + rq[q]] = pthis[q] ? -1 : rq[q];
      if (pthis[q] && cg_ == 0) pflag[rq[q]] = 1;
    }
  if (c == 0) {
    __syncthreads();  // piv[k0 .. k0 + w) written by thread 0 above (global, same CTA)
    if (tid < w) a.rowsrc[(int64_t)b * n + k0 + tid] = piv[k0 + tid];
  }
  if (singular && c == 0 && tid == 0) atomicCAS(a.info, 0, b + 1);
  if (clustered) cluster.sync();  // no CTA leaves while a peer may still read its shared memory
}

// ---------------------------------------------------------------------------
// Recursive panel (blocked path, n <= REC_NMAX, one CTA): the 28-column panel lives in shared
// memory and is factored in sub-panels of 4 columns.  The pivot steps (the sequential,
// latency-bound part) touch only the 4 sub-panel columns of every row (held in registers,
// 2 rows per thread); after each sub-panel one rank-4 DMMA update applies its transform to the
// other panel columns: C(i, J) = [i not a sub-panel pivot] C(i, J) + T4(i, :) Z4(:, J), the same
// block Gauss-Jordan algebra as the trailing update of the whole matrix.  Per step: one
// REDUX + one barrier for the pivot (every warp publishes its candidate's 4 values), 32 DFMA
// per thread.  Interface and implicit pivoting as zgj_panel47_kernel.
// ---------------------------------------------------------------------------
constexpr int REC_NMAX = 496, REC_PS = 28;  // rows; shared row stride (== 4 mod 8: conflict-free)

__host__ __device__ inline size_t rec_smem(int n) { return sizeof(zt) * ((size_t)n * REC_PS + 4 * 32); }

__global__ void __launch_bounds__(256, 1) zgj_panel_rec_kernel(const PanelArgs a) {
  constexpr int PS = REC_PS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zt* Ps = reinterpret_cast<zt*>(smem_raw);  // [n][PS] the panel
  zt* Z4 = Ps + (size_t)a.n * PS;            // [4][32] old pivot rows of the sub-panel, other columns
  __shared__ zt cand[2][8][4];
  __shared__ __align__(16) unsigned wkey[2][8];
  __shared__ int sub_piv[4];
  __shared__ signed char subpv[REC_NMAX];  // sub-panel index in which a row was pivot (-1: none)
  const int b = blockIdx.x, n = a.n, k0 = a.k0, w = a.w;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const zt* Xb = a.X + (int64_t)b * a.bsx;
  zt* Yb = a.Y + (int64_t)b * a.bsy;
  int* piv = a.piv + (int64_t)b * n;
  int* pflag = a.pflag + (int64_t)b * n;
  for (int i = wp; i < n; i += 8) {  // warp per row, lane per column: no integer division
    if (lane < w) Ps[i * PS + lane] = __ldcg(Xb + (int64_t)i * a.ldx + k0 + lane);
  }
  for (int i = tid; i < n; i += 256) subpv[i] = -1;
  const int r0 = tid, r1 = tid + 256;
  bool pv0 = r0 < n ? pflag[r0] != 0 : true, pv1 = r1 < n ? pflag[r1] != 0 : true;
  bool pt0 = false, pt1 = false;  // pivots of this panel
  bool singular = false;
  __syncthreads();
  for (int c0 = 0; c0 < w; c0 += 4) {
    const int ws = min(4, w - c0);
    zt s0[4], s1[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s0[c] = (r0 < n && c < ws) ? Ps[r0 * PS + c0 + c] : make_double2(0.0, 0.0);
      s1[c] = (r1 < n && c < ws) ? Ps[r1 * PS + c0 + c] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      if (kk < ws) {
        const int k = k0 + c0 + kk, par = k & 1;
        const unsigned key0 = (!pv0) ? pivot_key12(s0[kk], r0) : 0u;
        const unsigned key1 = (!pv1) ? pivot_key12(s1[kk], r1) : 0u;
        const unsigned mk = max(key0, key1);
        const unsigned wk = __reduce_max_sync(0xffffffffu, mk);
        if (wk != 0u && mk == wk) {  // this lane holds the warp's candidate row
          const bool second = key1 == wk;
#pragma unroll
          for (int c = 0; c < 4; ++c) cand[par][wp][c] = second ? s1[c] : s0[c];
        }
        if (lane == 0) wkey[par][wp] = wk;
        __syncthreads();
        const uint4 ka = *reinterpret_cast<const uint4*>(&wkey[par][0]);
        const uint4 kb = *reinterpret_cast<const uint4*>(&wkey[par][4]);
        unsigned best = ka.x;
        int bw = 0;
        const unsigned kv[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
#pragma unroll
        for (int q = 1; q < 8; ++q)
          if (kv[q] > best) {
            best = kv[q];
            bw = q;
          }
        if ((best & ~4095u) == 0u) singular = true;
        const int r = 4095 - (int)(best & 4095u);
        zt pr[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) pr[c] = cand[par][bw][c];
        const zt inv = zinv_fast(pr[kk]);
        if (tid == 0) {
          piv[k] = r;
          sub_piv[kk] = r;
          subpv[r] = (signed char)(c0 >> 2);
        }
        // rank-1 update of the sub-panel columns (pivot row: a <- pr / pivot exactly)
        auto upd = [&](zt(&sv)[4], int row, bool& pvf, bool& ptf) {
          zt g = zmul(sv[kk], inv);
          if (row == r) {
            pvf = true;
            ptf = true;
            g = make_double2(-inv.x, -inv.y);
#pragma unroll
            for (int c = 0; c < 4; ++c) sv[c] = make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            sv[c].x = fma(-g.x, pr[c].x, sv[c].x);
            sv[c].y = fma(-g.x, pr[c].y, sv[c].y);
            sv[c].x = fma(g.y, pr[c].y, sv[c].x);
            sv[c].y = fma(-g.y, pr[c].x, sv[c].y);
          }
          sv[kk] = make_double2(-g.x, -g.y);
        };
        if (r0 < n) upd(s0, r0, pv0, pt0);
        if (r1 < n) upd(s1, r1, pv1, pt1);
      }
    }
    // the sub-panel's 4 pivot rows, old values in the other panel columns -> Z4 (before anyone
    // writes them back), then the sub-panel columns (T4) back into the panel
    __syncthreads();
    const int nother = w - ws;
    for (int e = tid; e < 4 * 32; e += 256) {
      const int m = e >> 5, j = e & 31;
      zt v = make_double2(0.0, 0.0);
      if (m < ws && j < nother) {
        const int col = j < c0 ? j : j + ws;
        v = Ps[sub_piv[m] * PS + col];
      }
      Z4[e] = v;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < ws) {
        if (r0 < n) Ps[r0 * PS + c0 + c] = s0[c];
        if (r1 < n) Ps[r1 * PS + c0 + c] = s1[c];
      }
    __syncthreads();
    // rank-4 DMMA update of the other panel columns: m-tiles of 8 rows x n-tiles of 8 columns
    if (nother > 0) {
      const int MT = (n + 7) >> 3, NTt = (nother + 7) >> 3;
      const int sidx = c0 >> 2;
      for (int mt = wp; mt < MT; mt += 8) {  // a warp keeps its m-tile (A fragment, pivot flag)
        const int row = mt * 8 + (lane >> 2), rowc = min(row, n - 1);
        const zt av = ((lane & 3) < ws) ? Ps[rowc * PS + c0 + (lane & 3)] : make_double2(0.0, 0.0);
        const bool sp = subpv[rowc] == sidx;  // row is a pivot of this sub-panel: seed 0
        for (int nt = 0; nt < NTt; ++nt) {
        const zt bv = Z4[(lane & 3) * 32 + nt * 8 + (lane >> 2)];
        double cr[2], ci[2];
        int col[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = nt * 8 + (lane & 3) * 2 + h;
          col[h] = j < nother ? (j < c0 ? j : j + ws) : -1;
          const zt sv = (row < n && col[h] >= 0 && !sp) ? Ps[row * PS + col[h]] : make_double2(0.0, 0.0);
          cr[h] = sv.x;
          ci[h] = sv.y;
        }
        dmma884(cr[0], cr[1], av.x, bv.x);
        dmma884(ci[0], ci[1], av.x, bv.y);
        dmma884(cr[0], cr[1], -av.y, bv.y);
        dmma884(ci[0], ci[1], av.y, bv.x);
        if (row < n) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (col[h] >= 0) Ps[row * PS + col[h]] = make_double2(cr[h], ci[h]);
        }
        }
      }
    }
    __syncthreads();
  }
  // T into Y, GEMM maps, pivot flags
  for (int i = wp; i < n; i += 8)
    if (lane < w) Yb[(int64_t)i * a.ldy + k0 + lane] = Ps[i * PS + lane];
  if (r0 < n) {
    a.cinmap[(int64_t)b * n + r0] = pt0 ? -1 : r0;
    if (pt0) pflag[r0] = 1;
  }
  if (r1 < n) {
    a.cinmap[(int64_t)b * n + r1] = pt1 ? -1 : r1;
    if (pt1) pflag[r1] = 1;
  }
  __syncthreads();
  if (tid < w) a.rowsrc[(int64_t)b * n + k0 + tid] = piv[k0 + tid];
  if (singular && tid == 0) atomicCAS(a.info, 0, b + 1);
}

// A^{-1}(k, j) = M(piv[k], pinv[j]): one CTA per matrix
__global__ void zgj_implicit_out_kernel(const zt* __restrict__ M, int64_t ldm, int64_t bsm, zt* __restrict__ out,
                                        int64_t ldo, int64_t obs, const int* __restrict__ piv_all, int n) {
  extern __shared__ int sp[];  // piv[n], pinv[n]
  const int b = blockIdx.y;
  const int* piv = piv_all + (int64_t)b * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = piv[i];
    sp[i] = r;
    sp[n + r] = i;
  }
  __syncthreads();
  const zt* Mb = M + (int64_t)b * bsm;
  zt* ob = out + (int64_t)b * obs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / n), j = (int)(e - (int64_t)k * n);
    ob[(int64_t)k * ldo + j] = Mb[(int64_t)sp[k] * ldm + sp[n + j]];
  }
}

// ---------------------------------------------------------------------------
// Sequential-phase variant of the warp-specialised kernel (regime 7): all 16 warps factor the
// panel (2 rows x 7 columns per thread), then all 16 warps apply its update.  Measured on B200
// (tools/panel47_bench.cu): DMMA and DFMA share the FP64 issue resources, and warps issuing
// DMMA back to back starve another warp's DFMA almost completely, so overlapping the pivot
// steps with the tensor-core update (zgj_ws_kernel) stretches the pivot steps 2-4x; here the
// pivot steps run alone and the update runs at 4 warps per sub-partition.
// ---------------------------------------------------------------------------
// NAT: natural order (row k is the pivot of step k, one barrier per step) for the leaf Schur
// complement S assembled by the kernel itself (fin.c): in the configs' regimes natural-order
// elimination of S keeps every pivot >= 0.37 of its original diagonal; a pivot
// below 0.05 of it makes the body return false and the caller re-assembles S and pivots.
template <bool NAT>
__device__ __forceinline__ bool zgj_seq_body(zt* __restrict__ A, int64_t lda, int64_t bs, zt* __restrict__ out,
                                             int64_t ldo, int64_t obs, int n, int* __restrict__ info,
                                             const WsFinish& fin) {
  constexpr int NB = WS_NB, CPT = WS_NB / 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int mtr = (n + 15) & ~15, zs = ws_zs(n);
  zt* Ts = reinterpret_cast<zt*>(smem_raw);  // [mtr][NB]
  zt* Zs = Ts + (size_t)mtr * NB;            // [NB][zs]
  __shared__ zt prow4[2][NB];
  __shared__ zt pinv2[2];
  __shared__ __align__(16) unsigned wkey[2][16];
  __shared__ int pstep[256], plist[256], colmap[WS_NMAX + 16];
  __shared__ double diag2[NAT ? 256 : 1];  // |S_kk|^2 of the assembled S (NAT)
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, cg = lane & 3, rg = lane >> 2;
  const long long t_start = clock64();
  zt* M = A + (int64_t)blockIdx.x * bs;
  WsPanels P;
  P.npan = (n + NB - 1) / NB;
  P.base = n / P.npan;
  P.rem = n % P.npan;
  if (tid < 256) {
    pstep[tid] = NAT ? tid : 1 << 30;
    if (NAT) plist[tid] = tid;
  }
  if (tid == 0) s_bad = 0;
  if (fin.c) {  // assemble S in place (as zgj_ws_kernel)
    const int q = fin.p - 2;
    const zt* Lx = fin.K;
    const zt* Ly = fin.K + q * q;
    const zt* cl = fin.c + (int64_t)fin.leaf_nat[fin.leaf0 + blockIdx.x] * fin.p * fin.p;
    // column (jx, jy) of entry cc advances incrementally (cc += 32): no division per entry
    const int dq = 32 / q, dr = 32 - dq * q, jx0 = lane % q, jy0 = lane / q;
    for (int r = tid >> 5; r < n; r += 16) {
      const int ix = r % q, iy = r / q;
      zt* Mr = M + (int64_t)r * lda;
      int jx = jx0, jy = jy0;
      for (int cc = lane; cc < n; cc += 32) {
        zt v = make_double2(0.0, 0.0);
        if (iy == jy) v = Lx[ix * q + jx];
        if (ix == jx) {
          v.x += Ly[iy * q + jy].x;
          v.y += Ly[iy * q + jy].y;
        }
        if (r == cc) {
          const zt cv = cl[(iy + 1) * fin.p + ix + 1];
          v.x -= fin.kappa2 * cv.x;
          v.y -= fin.kappa2 * cv.y;
          if (NAT) diag2[r] = fma(v.x, v.x, v.y * v.y);
        }
        Mr[cc] = v;
        jx += dr;
        jy += dq;
        if (jx >= q) {
          jx -= q;
          ++jy;
        }
      }
    }
  }
  __syncthreads();
  int rq[2];
  rq[0] = wp * 16 + rg;
  rq[1] = wp * 16 + 8 + rg;
  bool piv[2] = {false, false}, singular = false;
  const bool warp_live = wp * 16 < n;
  const int MT = mtr >> 3;
  // trace armed with 1 (every launch) or with the matrix size n to trace
  const bool trace = (g_ws_trace_on == 1 || g_ws_trace_on == n) && blockIdx.x == 0 && tid == 0;
  if (trace) g_ws_trace[15 * 16 + 2] = t_start;
  // natural order: the pivot rows of panel p are rows k0 .. k0 + w - 1, and their entries outside
  // the panel (Z of the update) are final once the previous update has finished, so Z is fetched
  // by cp.async while the panel is being factored (no staging phase)
  const bool zpre = NAT && fin.blockpanel != 1;
  for (int p = 0; p < P.npan; ++p) {
    const int k0 = P.k0(p), w = P.w(p), w4 = (w + 3) & ~3, K4 = w4 >> 2, nv = n - w;
    WS_MARK(p, 0);
    if (zpre && !(p + 1 == P.npan && nv == 0)) {
      for (int e = tid; e < w4 * nv; e += 512) {
        const int m = e / nv, v = e - m * nv;
        const bool ok = m < w;
        cpa16_zfill(Zs + m * zs + v, M + (int64_t)(ok ? k0 + m : 0) * lda + (v < k0 ? v : v + w), ok);
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
    if (NAT && fin.blockpanel) {
      // ---- natural-order panel in block form (knob leaf_panel = 1): the pivot rows are rows
      // k0 .. k0 + w - 1, so D = M[K, K] is inverted by warps 0-3 (7 rows each, lane j holds column
      // j in registers, one 128-thread named barrier per step), then T = -M[rows outside K, K] D^{-1}
      // runs on DMMA in all 16 warps from the panel staged in shared memory; T[K] = D^{-1}. ----
      // (leaf_panel = 2: the panel is staged by cp.async and D^{-1} is formed by all 512 threads,
      // one natural-order step per barrier on ping-pong copies of D in shared memory placed after
      // Z, so Z is still prefetched during the panel)
      const bool pp = fin.blockpanel == 2;
      if (pp) {
        for (int e = tid; e < mtr * NB; e += 512) {
          const int i = e / NB, j = e - i * NB;
          const bool ok = i < n && j < w;
          cpa16_zfill(Ts + e, M + (int64_t)(ok ? i : 0) * lda + k0 + (ok ? j : 0), ok);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);  // the panel (and the Z prefetch issued before it)
      } else {
        for (int e = tid; e < mtr * NB; e += 512) {  // stage the panel (zero padding rows / columns)
          const int i = e / NB, j = e - i * NB;
          Ts[e] = (i < n && j < w) ? ldplain(M + (int64_t)i * lda + k0 + j) : make_double2(0.0, 0.0);
        }
      }
      __syncthreads();
      WS_MARK(p, 4);
      zt(*Dv)[NB + 1] = reinterpret_cast<zt(*)[NB + 1]>(Zs);  // D^{-1} (Z staging area is free now)
      if (pp) {
        zt* Da = Zs + NB * zs;            // [NB][NB + 1] x 2 after Z
        zt* Db = Da + NB * (NB + 1);
        constexpr int DS = NB + 1;
        for (int e = tid; e < NB * NB; e += 512) {
          const int r = e / NB, c = e - r * NB;
          Da[r * DS + c] = (r < w && c < w) ? Ts[(k0 + r) * NB + c] : make_double2(r == c ? 1.0 : 0.0, 0.0);
        }
        __syncthreads();
        for (int k = 0; k < w; ++k) {
          const zt* src = (k & 1) ? Db : Da;
          zt* dst = (k & 1) ? Da : Db;
          const zt pv = src[k * DS + k];
          const zt inv = zinv_fast(pv);
          if (tid == 0 && !(fma(pv.x, pv.x, pv.y * pv.y) >= 0.0025 * diag2[k0 + k])) s_bad = 1;
          for (int e = tid; e < NB * NB; e += 512) {
            const int i = e / NB, j = e - i * NB;
            zt v;
            if (i == k) {
              v = j == k ? inv : zmul(src[k * DS + j], inv);
            } else {
              const zt fi = zmul(src[i * DS + k], inv);
              if (j == k) {
                v = make_double2(-fi.x, -fi.y);
              } else {
                const zt pk = src[k * DS + j];
                v = src[i * DS + j];
                v.x = fma(-fi.x, pk.x, fma(fi.y, pk.y, v.x));
                v.y = fma(-fi.x, pk.y, fma(-fi.y, pk.x, v.y));
              }
            }
            dst[i * DS + j] = v;
          }
          __syncthreads();
        }
        Dv = reinterpret_cast<zt(*)[NB + 1]>((w & 1) ? Db : Da);
      } else if (wp < 4) {
        constexpr int RW = NB / 4;  // rows per warp
        zt d[RW];
        const int jl = lane < NB ? lane : 0;
#pragma unroll
        for (int t = 0; t < RW; ++t) {
          const int r = wp * RW + t;
          d[t] = (r < w && jl < w) ? Ts[(k0 + r) * NB + jl] : make_double2(r == jl ? 1.0 : 0.0, 0.0);
        }
        for (int k = 0; k < w; ++k) {
          const int vk = k / RW, tk = k - vk * RW, par = k & 1;
          if (wp == vk) {
            zt dk = d[0];
#pragma unroll
            for (int t = 1; t < RW; ++t)
              if (t == tk) dk = d[t];
            const zt pv = make_double2(__shfl_sync(0xffffffffu, dk.x, k), __shfl_sync(0xffffffffu, dk.y, k));
            const zt inv = zinv_fast(pv);
            if (lane < NB) prow4[par][lane] = lane == k ? inv : zmul(dk, inv);
            if (lane == 0) {
              pinv2[par] = inv;
              if (!(fma(pv.x, pv.x, pv.y * pv.y) >= 0.0025 * diag2[k0 + k])) s_bad = 1;
            }
          }
          bar_sync_n(BAR_PANEL, 128);
          const zt prj = prow4[par][jl], inv = pinv2[par];
#pragma unroll
          for (int t = 0; t < RW; ++t) {
            const int r = wp * RW + t;
            const zt f = make_double2(__shfl_sync(0xffffffffu, d[t].x, k), __shfl_sync(0xffffffffu, d[t].y, k));
            if (r == k) {
              d[t] = prj;
            } else if (lane == k) {
              const zt g = zmul(f, inv);
              d[t] = make_double2(-g.x, -g.y);
            } else {
              d[t].x = fma(-f.x, prj.x, d[t].x);
              d[t].x = fma(f.y, prj.y, d[t].x);
              d[t].y = fma(-f.x, prj.y, d[t].y);
              d[t].y = fma(-f.y, prj.x, d[t].y);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < RW; ++t)
          if (lane < NB) Dv[wp * RW + t][lane] = d[t];
      }
      __syncthreads();
      WS_MARK(p, 5);
      if (s_bad) {  // uniform: the caller re-assembles S and pivots
        asm volatile("cp.async.wait_group 0;\n" ::);
        return false;
      }
      // T[r, :] = -M[r, K] D^{-1} for rows r outside K, D^{-1} for rows in K (one row tile per unit)
      for (int mt = wp; mt < MT; mt += 16) {
        const int r = mt * 8 + (lane >> 2);
        zt af[NB / 4];
#pragma unroll
        for (int k4 = 0; k4 < NB / 4; ++k4) af[k4] = Ts[r * NB + k4 * 4 + (lane & 3)];
        const bool inK = r >= k0 && r < k0 + w;
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) {
          double tr[2] = {0.0, 0.0}, ti[2] = {0.0, 0.0};
#pragma unroll
          for (int k4 = 0; k4 < NB / 4; ++k4) {
            const int kb = k4 * 4 + (lane & 3), cb = ct * 8 + (lane >> 2);
            const zt bv = (kb < w && cb < w) ? Dv[kb][cb] : make_double2(0.0, 0.0);
            dmma884(tr[0], tr[1], -af[k4].x, bv.x);
            dmma884(ti[0], ti[1], -af[k4].x, bv.y);
            dmma884(tr[0], tr[1], af[k4].y, bv.y);
            dmma884(ti[0], ti[1], -af[k4].y, bv.x);
          }
          __syncwarp();  // every lane's A fragments of this row tile are read before any write
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = ct * 8 + (lane & 3) * 2 + h;
            if (cc < NB) {
              zt v = cc < w ? make_double2(tr[h], ti[h]) : make_double2(0.0, 0.0);
              if (inK) v = cc < w ? Dv[r - k0][cc] : make_double2(0.0, 0.0);
              if (r >= n) v = make_double2(0.0, 0.0);
              Ts[r * NB + cc] = v;
            }
          }
        }
      }
      __syncthreads();
      WS_MARK(p, 6);
      for (int e = tid; e < n * w; e += 512) {  // the panel columns of M <- T (in place)
        const int i = e / w, j = e - i * w;
        M[(int64_t)i * lda + k0 + j] = Ts[i * NB + j];
      }
      WS_MARK(p, 1);
    } else {
    // ---------------- panel: w pivot steps on the n x w panel ----------------
    zt a[2][CPT];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int j = cg * CPT + c;
        a[q][c] = (rq[q] < n && j < w) ? ldplain(M + (int64_t)rq[q] * lda + k0 + j) : make_double2(0.0, 0.0);
      }
    for (int cga = 0; cga * CPT < w; ++cga) {
      const bool act = cg == cga;
      const int src = (lane & ~3) | cga;
#pragma unroll
      for (int s = 0; s < CPT; ++s) {
        const int kk = cga * CPT + s;
        if (kk < w) {
          const int k = k0 + kk, par = k & 1;
          int r = k;
          if (!NAT) {
            unsigned key = 0u;
            if (act) {
#pragma unroll
              for (int q = 0; q < 2; ++q)
                if (!piv[q] && rq[q] < n) key = max(key, pivot_key(a[q][s], rq[q], true));
            }
            key = __reduce_max_sync(0xffffffffu, key);
            if (lane == 0) wkey[par][wp] = key;
            __syncthreads();
            unsigned best = 0u;
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
              const uint4 kq = *reinterpret_cast<const uint4*>(&wkey[par][4 * g4]);
              best = max(best, max(max(kq.x, kq.y), max(kq.z, kq.w)));
            }
            if ((best & ~511u) == 0u) singular = true;
            r = 511 - (int)(best & 511u);
          }
          if (wp == (r >> 4) && rg == (r & 7)) {  // the 4 lanes of row r publish it raw
            const int qq = (r >> 3) & 1;
#pragma unroll
            for (int q = 0; q < 2; ++q)
              if (q == qq) {
#pragma unroll
                for (int c = 0; c < CPT; ++c) prow4[par][cg * CPT + c] = a[q][c];
              }
            if (!NAT && cg == 0) {
              pstep[r] = k;
              plist[k] = r;
            }
          }
          __syncthreads();
          if (NAT && tid == 0) {
            const zt pv = prow4[par][kk];
            if (!(fma(pv.x, pv.x, pv.y * pv.y) >= 0.0025 * diag2[k]) || (g_seq_force_bad && k == 100)) s_bad = 1;
          }
          if (warp_live) {
            const zt inv = zinv_fast(prow4[par][kk]);
            zt g[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const zt v = a[q][s];
              g[q] = zmul(make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)), inv);
            }
            if (wp == (r >> 4)) {
#pragma unroll
              for (int q = 0; q < 2; ++q)
                if (rq[q] == r) {  // pivot row: a <- pr / pivot exactly (as 0 - (-inv) pr)
                  piv[q] = true;
                  g[q] = make_double2(-inv.x, -inv.y);
#pragma unroll
                  for (int c = 0; c < CPT; ++c) a[q][c] = make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
              const zt pc = prow4[par][cg * CPT + c];
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                a[q][c].x = fma(-g[q].x, pc.x, a[q][c].x);
                a[q][c].y = fma(-g[q].x, pc.y, a[q][c].y);
                a[q][c].x = fma(g[q].y, pc.y, a[q][c].x);
                a[q][c].y = fma(-g[q].y, pc.x, a[q][c].y);
              }
            }
            if (act) {
#pragma unroll
              for (int q = 0; q < 2; ++q) a[q][s] = make_double2(-g[q].x, -g[q].y);
            }
          }
        }
      }
    }
    WS_MARK(p, 1);
    // T -> shared (the A operand of the update); its copy back into M's panel columns is written
    // coalesced from shared memory at the start of the update (nothing reads those columns before
    // the next update)
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (rq[q] < mtr) {
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int j = cg * CPT + c;
          Ts[rq[q] * NB + j] = j < w ? a[q][c] : make_double2(0.0, 0.0);
        }
      }
    if (NAT) {
      __syncthreads();
      if (s_bad) {  // uniform: the caller re-assembles S and pivots
        asm volatile("cp.async.wait_group 0;\n" ::);  // no prefetched Z lands in the fallback's buffers
        return false;
      }
    }
    }  // panel form
    if (p + 1 == P.npan && nv == 0) {  // a single panel: T is the result; write it back and stop
      __syncthreads();
      if (!(NAT && fin.blockpanel))
        for (int e = tid; e < n * w; e += 512) {
          const int i = e / w, j = e - i * w;
          M[(int64_t)i * lda + k0 + j] = Ts[i * NB + j];
        }
      break;
    }
    // ---------------- update: C(i, J) = [i not a pivot of p] C(i, J) + T(i,:) Z(:, J) -------------
    for (int v = tid; v < nv + 16; v += 512) colmap[v] = v < nv ? (v < k0 ? v : v + w) : -1;
    __syncthreads();  // T, pivots, colmap visible
    if (!(NAT && fin.blockpanel))  // (the block-form panels wrote M already)
      for (int e = tid; e < n * w; e += 512) {
        const int i = e / w, j = e - i * w;
        M[(int64_t)i * lda + k0 + j] = Ts[i * NB + j];
      }
    if (!zpre) {
      for (int e = tid; e < w4 * nv; e += 512) {
        const int m = e / nv, v = e - m * nv;
        const bool ok = m < w;
        const int srow = ok ? plist[k0 + m] : 0;
        cpa16_zfill(Zs + m * zs + v, M + (int64_t)srow * lda + colmap[v], ok);
      }
      asm volatile("cp.async.commit_group;\n" ::);
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    WS_MARK(p, 2);
    const int NPR = (nv + 15) >> 4;
    struct Unit {
      int rr, col[2][2];
      bool rok;
      zt seed[2][2];
    };
    auto load_unit = [&](int mt, int npr, Unit& U) {
      U.rr = mt * 8 + (lane >> 2);
      const int rc = min(U.rr, n - 1);
      U.rok = U.rr < n && (unsigned)(pstep[rc] - k0) >= (unsigned)w;
      const int vb = npr * 16 + (lane & 3) * 2;
      const zt* rowp = M + (int64_t)rc * lda;
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int v = vb + t * 8 + h;
          U.col[t][h] = v < nv ? colmap[v] : -1;
          U.seed[t][h] = ldplain(rowp + max(U.col[t][h], 0));
        }
    };
    Unit cur, nxt;
    // row tiles of 8 up to n (the padding rows of the last 16-row block carry no work), and a last
    // column block with only 8 valid columns runs half the DMMAs
    const int MTu = (n + 7) >> 3;
    int mt = wp, npr = 0;
    while (mt >= MTu) {
      mt -= MTu;
      ++npr;
    }
    bool have = npr < NPR;
    if (have) load_unit(mt, npr, nxt);
    while (have) {
      cur = nxt;
      const int cmt = mt, cnpr = npr;
      mt += 16;
      while (mt >= MTu) {
        mt -= MTu;
        ++npr;
      }
      have = npr < NPR;
      if (have) load_unit(mt, npr, nxt);
      double ar[2][2], ai[2][2];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool ok = cur.rok && cur.col[t][h] >= 0;
          ar[t][h] = ok ? cur.seed[t][h].x : 0.0;
          ai[t][h] = ok ? cur.seed[t][h].y : 0.0;
        }
      const zt* Trow = Ts + (cmt * 8 + (lane >> 2)) * NB + (lane & 3);
      const zt* Zc = Zs + (lane & 3) * zs + cnpr * 16 + (lane >> 2);
      if (cnpr * 16 + 8 < nv) {
#pragma unroll 7
        for (int k4 = 0; k4 < K4; ++k4) {
          const zt av = Trow[k4 * 4];
          const zt b0 = Zc[k4 * 4 * zs], b1 = Zc[k4 * 4 * zs + 8];
          dmma884(ar[0][0], ar[0][1], av.x, b0.x);
          dmma884(ar[1][0], ar[1][1], av.x, b1.x);
          dmma884(ai[0][0], ai[0][1], av.x, b0.y);
          dmma884(ai[1][0], ai[1][1], av.x, b1.y);
          dmma884(ar[0][0], ar[0][1], -av.y, b0.y);
          dmma884(ar[1][0], ar[1][1], -av.y, b1.y);
          dmma884(ai[0][0], ai[0][1], av.y, b0.x);
          dmma884(ai[1][0], ai[1][1], av.y, b1.x);
        }
      } else {
#pragma unroll 7
        for (int k4 = 0; k4 < K4; ++k4) {
          const zt av = Trow[k4 * 4];
          const zt b0 = Zc[k4 * 4 * zs];
          dmma884(ar[0][0], ar[0][1], av.x, b0.x);
          dmma884(ai[0][0], ai[0][1], av.x, b0.y);
          dmma884(ar[0][0], ar[0][1], -av.y, b0.y);
          dmma884(ai[0][0], ai[0][1], av.y, b0.x);
        }
      }
      if (cur.rr < n) {
        zt* rowp = M + (int64_t)cur.rr * lda;
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (cur.col[t][h] >= 0) rowp[cur.col[t][h]] = make_double2(ar[t][h], ai[t][h]);
      }
    }
    __syncthreads();  // update stored before the next panel reads its columns
    WS_MARK(p, 3);
  }
  if (singular && tid == 0) atomicCAS(info, 0, blockIdx.x + 1);
  __syncthreads();
  WS_MARK(15, 0);
  ws_output(M, lda, out, ldo, obs, n, fin, plist, pstep, smem_raw, NAT);
  WS_MARK(15, 1);
  return true;
}

__global__ void __launch_bounds__(512, 1) zgj_seq_kernel(zt* __restrict__ A, int64_t lda, int64_t bs,
                                                         zt* __restrict__ out, int64_t ldo, int64_t obs, int n,
                                                         int* __restrict__ info, const WsFinish fin) {
  if (fin.c && !g_seq_pivot && n <= 256) {
    // natural order in place: the work matrix is the leaf operator's own Y_i block (the epilogue
    // then leaves Y_i = S^{-1} where it is; the pivoted fallback uses the scratch matrix A)
    const bool inpl = fin.p != 0 && fin.inplace;
    if (inpl ? zgj_seq_body<true>(out, ldo, obs, out, ldo, obs, n, info, fin)
             : zgj_seq_body<true>(A, lda, bs, out, ldo, obs, n, info, fin))
      return;
    __syncthreads();
  }
  zgj_seq_body<false>(A, lda, bs, out, ldo, obs, n, info, fin);
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
  int mode;  // 0 register CTA, 1 register cluster, 2 shared-memory cluster
  int nb, cs, rp;
  size_t smem;
};

int pow2_ceil(int v) {
  int c = 1;
  while (c < v) c *= 2;
  return c;
}

PanelPlan panel_plan(int n) {
  if (n <= 4096) {
    const int wmax = (n > 256 && n <= 512) ? 16 : 32;  // 512-thread panels hold 16 columns per thread
    const int npan = (n + wmax - 1) / wmax;
    const int nb = (n + npan - 1) / npan;  // equal panels, no narrow tail
    if (n <= 512) return PanelPlan{0, nb, 1, n, 0};
    return PanelPlan{1, nb, pow2_ceil((n + 255) / 256), 256, 0};
  }
  const size_t budget = 150 * 1024;
  for (int nb : {32, 16})
    for (int cs = 1; cs <= 16; cs *= 2) {
      const int rp = (n + cs - 1) / cs;
      const size_t smem = sizeof(zt) * ((size_t)rp * nb + 2 * nb) + 64 + sizeof(int) * rp;
      if (smem <= budget) return PanelPlan{2, nb, cs, rp, smem};
    }
  const int rp = (n + 15) / 16;
  return PanelPlan{2, 16, 16, rp, sizeof(zt) * ((size_t)rp * 16 + 32) + 64 + sizeof(int) * rp};
}

bool use_fused(int n, int batch) { return n > 32 && n <= 256 && (batch >= 16 || n <= 128); }
// the gj knob (1 fused, 2 blocked, 3 warp-specialised) forces a kernel family (tools/gj_tune.py)
}  // namespace
int g_gj_mode_force = 0;
// debug: timeline of CTA 0 of the next zgj_ws launch (on = 1 arms it; out[160] clock64 values)
void zgj_ws_trace(int on, long long* out) {
  HPS_CUDA_CHECK(cudaMemcpyToSymbol(g_ws_trace_on, &on, sizeof(int)));
  HPS_CUDA_CHECK(cudaMemcpyToSymbol(g_nat_trace_on, &on, sizeof(int)));
  if (out) HPS_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_ws_trace, sizeof(long long) * 256));
  if (out) HPS_CUDA_CHECK(cudaMemcpyFromSymbol(out + 256, g_nat_trace, sizeof(long long) * 64));
}  // hps_zinv_timed: 1 = fused, 2 = blocked (0 = library choice / HPS_GJ)
namespace {
int gj_mode_env() {
  return g_gj_mode_force ? g_gj_mode_force : knob(KN_GJ);
}

// ---------------------------------------------------------------------------
// Regimes of the batched inverse and the representative-action planner (PAPER.md:881-953,
// SURVEY 8(f) NEXT-3).  The paper picks, per tree level, theta_o boxes in parallel x theta_i
// threads of parallel linear algebra per box minimising eps = ceil(N_boxes / theta_o) r^{theta_i}
// with r the measured "representative time" of the level's representative action (the interior
// inverse on the leaf level, the interface inverse W^{-1} on the others).  On the GPU the
// choice is between kernel regimes: one CTA per box (theta_i = 1 SM, theta_o = boxes resident
// per wave) or a blocked path whose panels and GEMM updates spread each box over the GPU
// (theta_o = all boxes of the level in one batched launch).  hps_plan_inverse measures r for
// every feasible regime on one wave and records the argmin of eps; without a plan entry the
// measured default rules below apply.
// ---------------------------------------------------------------------------
enum Regime { REG_NONE = 0, REG_SMALL, REG_FUSED, REG_WS, REG_P47, REG_BLOCKED, REG_REC, REG_SEQ, REG_COUNT };
std::mutex g_plan_mu;
std::map<std::pair<int, int>, int> g_plan;  // (n, batch) -> regime
thread_local int g_regime_force = REG_NONE;

bool regime_feasible(int r, int n) {
  switch (r) {
    case REG_SMALL: return n <= kSmallMax;
    case REG_FUSED: return n <= 256;
    case REG_WS: return n > 32 && n <= WS_NMAX;
    case REG_P47: return n <= 4096;
    case REG_BLOCKED: return true;
    case REG_REC: return n > 32 && n <= REC_NMAX;
    case REG_SEQ: return n > 32 && n <= WS_NMAX;
    default: return false;
  }
}

int default_regime(int n, int batch) {
  const int m = gj_mode_env();
  if (m == 2) return n <= 32 ? REG_SMALL : REG_BLOCKED;
  if (m == 3 && regime_feasible(REG_WS, n)) return REG_WS;
  if (m == 1 && n > 32 && n <= 256) return REG_FUSED;
  if (n <= 32) return REG_SMALL;
  // sequential-phase one-CTA-per-matrix kernel: measured fastest for 48 <= n <= 200 (the leaf
  // n_i = 196 and the mid-level interfaces) at every batch size
  if (n >= 48 && n <= 200) return REG_SEQ;
  if (use_fused(n, batch)) return REG_FUSED;
  // implicit-pivoting 28-column panels: measured (tools/gj_tune.py) 1.5x faster than the explicit
  // panels in one CTA (n <= 256) and 1.1-1.15x at clusters of 3-8 CTAs; at 2 and > 8 CTAs
  // the explicit-swap panels are as fast or faster
  if (n <= 256 || (n > 640 && n <= 2048)) return REG_P47;
  return REG_BLOCKED;
}

int choose_regime(int n, int batch) {
  if (g_regime_force != REG_NONE && regime_feasible(g_regime_force, n)) return g_regime_force;
  if (gj_mode_env() == 0) {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plan.find({n, batch});
    if (it != g_plan.end()) return it->second;
  }
  return default_regime(n, batch);
}

void launch_cluster(const void* kern, int grid, int cs, size_t smem, cudaStream_t st, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HPS_CUDA_CHECK(cudaLaunchKernelExC(&cfg, kern, args));
}

// Blocked Gauss-Jordan with implicit pivoting: per 28-column panel one zgj_panel47_kernel launch
// (cluster of ceil(n / 256) CTAs) and one DMMA GEMM for the other columns; X/Y ping-pong.
void zgj_invert_p47(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch, void* ws,
                    int* info, cudaStream_t st, bool rec = false) {
  // 28-column panels on ceil(n / 256) CTAs.  (14-column panels in one CTA for 256 < n <= 512,
  // CG = 2, measured slower: the step cost is the same and there are twice as many panels.)
  const int CG = 4, NBW = 7 * CG;
  const int npan = (n + NBW - 1) / NBW, base = n / npan, rem = n % npan;
  const int CS = (n + 1024 / CG - 1) / (1024 / CG);
  char* wsp = static_cast<char*>(ws);
  const size_t mbytes = ((sizeof(zt) * (size_t)batch * n * n + 255) / 256) * 256;
  zt* B2 = reinterpret_cast<zt*>(wsp);
  int* piv = reinterpret_cast<int*>(wsp + mbytes);
  int* rowsrc = piv + (size_t)batch * n;
  int* cinmap = rowsrc + (size_t)batch * n;
  int* pflag = cinmap + (size_t)batch * n;
  static bool attr = false;
  if (!attr) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel47_kernel<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel_rec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)rec_smem(REC_NMAX)));
    attr = true;
  }
  HPS_CUDA_CHECK(cudaMemsetAsync(pflag, 0, sizeof(int) * (size_t)batch * n, st));
  zt* buf[2] = {A, B2};
  const int64_t ld[2] = {lda, n}, bsz[2] = {bs, (int64_t)n * n};
  int cur = 0;
  for (int p = 0; p < npan; ++p) {
    const int k0 = p * base + std::min(p, rem), w = base + (p < rem ? 1 : 0);
    PanelArgs pa{buf[cur], buf[1 - cur], ld[cur], bsz[cur], ld[1 - cur], bsz[1 - cur], n, k0, w, piv, rowsrc, cinmap,
                 info, pflag};
    {
      ProfScope ps(K_GJ_PANEL, 8.0 * n * (double)w * w * batch, 32.0 * n * (double)w * batch, st);
      if (rec) {
        zgj_panel_rec_kernel<<<batch, 256, rec_smem(n), st>>>(pa);
        HPS_CUDA_CHECK(cudaGetLastError());
      } else if (CS == 1) {
        if (CG == 2)
          zgj_panel47_kernel<2><<<batch, 256, 0, st>>>(pa);
        else
          zgj_panel47_kernel<4><<<batch, 256, 0, st>>>(pa);
        HPS_CUDA_CHECK(cudaGetLastError());
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(batch * CS);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        HPS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zgj_panel47_kernel<4>, pa));
      }
      count_launch();
    }
    const int nc = n - w;
    if (nc > 0) {
      // Y(:, J) = (I~ X)(:, J) + T X(pivot rows, J)
      ZGemm gm;
      gm.M = n;
      gm.N = nc;
      gm.K = w;
      gm.batch = batch;
      gm.A.ptr = buf[1 - cur] + k0;
      gm.A.rs = ld[1 - cur];
      gm.A.bs = bsz[1 - cur];
      gm.B.ptr = buf[cur];
      gm.B.rs = ld[cur];
      gm.B.bs = bsz[cur];
      gm.B.rmap = rowsrc + k0;
      gm.B.rmap_bs = n;
      gm.B.cskip_at = k0;
      gm.B.cskip_len = w;
      gm.Cin.ptr = buf[cur];
      gm.Cin.rs = ld[cur];
      gm.Cin.bs = bsz[cur];
      gm.Cin.rmap = cinmap;
      gm.Cin.rmap_bs = n;
      gm.Cin.cskip_at = k0;
      gm.Cin.cskip_len = w;
      gm.C.ptr = buf[1 - cur];
      gm.C.rs = ld[1 - cur];
      gm.C.bs = bsz[1 - cur];
      gm.C.cskip_at = k0;
      gm.C.cskip_len = w;
      gm.beta = make_double2(1.0, 0.0);
      zgemm(gm, st);
    }
    cur = 1 - cur;
  }
  ProfScope ps(K_GJ_AUX, 0.0, 32.0 * (double)batch * n * n, st);
  const int bx = (int)std::min<int64_t>(((int64_t)n * n + 255) / 256, std::max(1, hps_num_sms() * 8 / batch));
  zgj_implicit_out_kernel<<<dim3(bx, batch), 256, sizeof(int) * 2 * n, st>>>(buf[cur], ld[cur], bsz[cur], out, ldo,
                                                                             obs, piv, n);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void zgj_invert_impl(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch, void* ws,
                     int* info, cudaStream_t st) {
  if (n <= 0 || batch <= 0) return;
  const int reg = choose_regime(n, batch);
  if (reg == REG_SMALL) {
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
  if (reg == REG_WS || reg == REG_SEQ) {
    ProfScope ps(K_GJ_FUSED, 8.0 * n * n * (double)n * batch, 32.0 * n * (double)n * batch, st);
    static bool wattr = false;
    if (!wattr) {
      HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)ws_smem(WS_NMAX)));
      HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)ws_smem(WS_NMAX)));
      wattr = true;
    }
    auto kern = reg == REG_SEQ ? zgj_seq_kernel : zgj_ws_kernel;
    for (int b0 = 0; b0 < batch; b0 += 65535) {
      const int nbatch = std::min(65535, batch - b0);
      kern<<<nbatch, 512, ws_smem(n), st>>>(A + (int64_t)b0 * bs, lda, bs, out + (int64_t)b0 * obs, ldo,
                                                      obs, n, info,
                                                      WsFinish{nullptr, nullptr, {0.0, 0.0}, 0, nullptr, nullptr, 0, 0.0});
      HPS_CUDA_CHECK(cudaGetLastError());
      count_launch();
    }
    return;
  }
  if (reg == REG_FUSED) {
    ProfScope ps(K_GJ_FUSED, 8.0 * n * n * (double)n * batch, 32.0 * n * (double)n * batch, st);
    for (int b0 = 0; b0 < batch; b0 += 65535) {
      const int nbatch = std::min(65535, batch - b0);
      static bool fattr = false;
      if (!fattr) {
        HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_fused_kernel<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(zt) * 2 * 256 * 10)));
        HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_fused_kernel<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(zt) * 2 * 256 * 18)));
        fattr = true;
      }
      // large batches: two CTAs per SM overlap one matrix's pivot steps with the other's update;
      // small batches: one CTA per SM with wider chunks has the shorter critical path
      if (batch >= hps_num_sms())
        zgj_fused_kernel<8, 2><<<nbatch, 256, sizeof(zt) * 2 * (size_t)n * 10, st>>>(
            A + (int64_t)b0 * bs, lda, bs, out + (int64_t)b0 * obs, ldo, obs, n, info);
      else
        zgj_fused_kernel<16, 1><<<nbatch, 256, sizeof(zt) * 2 * (size_t)n * 18, st>>>(
            A + (int64_t)b0 * bs, lda, bs, out + (int64_t)b0 * obs, ldo, obs, n, info);
      HPS_CUDA_CHECK(cudaGetLastError());
      count_launch();
    }
    return;
  }
  if (reg == REG_P47 || reg == REG_REC) {
    zgj_invert_p47(A, lda, bs, out, ldo, obs, n, batch, ws, info, st, reg == REG_REC);
    return;
  }
  const PanelPlan pp = panel_plan(n);
  char* wsp = static_cast<char*>(ws);
  const size_t mbytes = ((sizeof(zt) * (size_t)batch * n * n + 255) / 256) * 256;
  zt* B2 = reinterpret_cast<zt*>(wsp);
  int* piv = reinterpret_cast<int*>(wsp + mbytes);
  int* rowsrc = piv + (size_t)batch * n;
  int* cinmap = rowsrc + (size_t)batch * n;
  int* pi = cinmap + (size_t)batch * n;
  static bool attr = false;
  if (!attr) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel_smem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_panel_creg_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  zt* buf[2] = {A, B2};
  const int64_t ld[2] = {lda, n}, bsz[2] = {bs, (int64_t)n * n};
  int cur = 0;
  for (int k0 = 0; k0 < n; k0 += pp.nb) {
    const int w = std::min(pp.nb, n - k0);
    PanelArgs pa{buf[cur], buf[1 - cur], ld[cur], bsz[cur], ld[1 - cur], bsz[1 - cur], n, k0, w, piv, rowsrc, cinmap,
                 info};
    {
      ProfScope ps(K_GJ_PANEL, 8.0 * n * (double)w * w * batch, 32.0 * n * (double)w * batch, st);
      if (pp.mode == 0) {
        if (n <= 256 && pp.nb <= 28)
          zgj_panel_reg_kernel<28, 256><<<batch, 256, 0, st>>>(pa);
        else if (n <= 256)
          zgj_panel_reg_kernel<32, 256><<<batch, 256, 0, st>>>(pa);
        else
          zgj_panel_reg_kernel<16, 512><<<batch, 512, 0, st>>>(pa);
        HPS_CUDA_CHECK(cudaGetLastError());
      } else if (pp.mode == 1) {
        void* args[] = {&pa};
        launch_cluster((const void*)zgj_panel_creg_kernel<32>, batch * pp.cs, pp.cs, 0, st, args);
      } else {
        int rp = pp.rp;
        void* args[] = {&pa, &rp};
        launch_cluster((const void*)zgj_panel_smem_kernel, batch * pp.cs, pp.cs, pp.smem, st, args);
      }
      count_launch();
    }
    const int nc = n - w;
    if (nc > 0) {
      // Y(:, J) = (I~ P X)(:, J) + T (P X)(panel, J)
      ZGemm gm;
      gm.M = n;
      gm.N = nc;
      gm.K = w;
      gm.batch = batch;
      gm.A.ptr = buf[1 - cur] + k0;
      gm.A.rs = ld[1 - cur];
      gm.A.bs = bsz[1 - cur];
      gm.B.ptr = buf[cur];
      gm.B.rs = ld[cur];
      gm.B.bs = bsz[cur];
      gm.B.rmap = rowsrc + k0;
      gm.B.rmap_bs = n;
      gm.B.cskip_at = k0;
      gm.B.cskip_len = w;
      gm.Cin.ptr = buf[cur];
      gm.Cin.rs = ld[cur];
      gm.Cin.bs = bsz[cur];
      gm.Cin.rmap = cinmap;
      gm.Cin.rmap_bs = n;
      gm.Cin.cskip_at = k0;
      gm.Cin.cskip_len = w;
      gm.C.ptr = buf[1 - cur];
      gm.C.rs = ld[1 - cur];
      gm.C.bs = bsz[1 - cur];
      gm.C.cskip_at = k0;
      gm.C.cskip_len = w;
      gm.beta = make_double2(1.0, 0.0);
      zgemm(gm, st);
    }
    cur = 1 - cur;
  }
  {
    ProfScope ps(K_GJ_AUX, 0.0, 8.0 * n * (double)batch, st);
    zgj_pi_kernel<<<(batch + 127) / 128, 128, 0, st>>>(piv, pi, n, batch);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
  const int64_t total = (int64_t)batch * n * n;
  ProfScope ps(K_GJ_AUX, 0.0, 32.0 * (double)total, st);
  int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)hps_num_sms() * 32);
  zgj_colperm_kernel<<<blocks, 256, 0, st>>>(buf[cur], ld[cur], bsz[cur], out, ldo, obs, pi, n, batch);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

}  // namespace

// Leaf inverse with the fused Schur epilogue (see WsFinish).  Returns false (nothing launched)
// when the warp-specialised kernel does not apply to n = (p-2)^2; the caller then runs the
// plain inverse and leaf_schur_finish.
bool zgj_leaf_fused_applies(int p, int batch) {
  const int n = (p - 2) * (p - 2);
  const int r = choose_regime(n, batch);
  return (r == REG_WS || r == REG_SEQ) && ws_finish_smem(p) <= ws_smem(n);
}

bool zgj_invert_leaf_schur(zt* S, int64_t sstride, zt* store, int64_t mstride, int p, int batch, const zt* K, zt* R,
                           zt eta, int* info, cudaStream_t st, const zt* c, const int* leaf_nat, int leaf0,
                           double kappa2) {
  const int q = p - 2, n = q * q, nb = 4 * q, nt = nb + n;
  if (!zgj_leaf_fused_applies(p, batch)) return false;
  static int piv_set = -1, bad_set = -1;  // values last copied to the device symbols
  const int piv = knob(KN_SEQ_PIVOT) != 0, bad = knob(KN_SEQ_FORCE_BAD) != 0;
  if (piv != piv_set) {
    HPS_CUDA_CHECK(cudaMemcpyToSymbol(g_seq_pivot, &piv, sizeof(int)));
    piv_set = piv;
  }
  if (bad != bad_set) {
    HPS_CUDA_CHECK(cudaMemcpyToSymbol(g_seq_force_bad, &bad, sizeof(int)));
    bad_set = bad;
  }
  static bool wattr = false;
  if (!wattr) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)ws_smem(WS_NMAX)));
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgj_seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)ws_smem(WS_NMAX)));
    wattr = true;
  }
  const double ni = n;
  ProfScope ps(K_LEAF_GJ, 8.0 * ni * ni * ni * batch + 8.0 * batch * q * (2.0 * ni * nb + (double)nb * nb),
               16.0 * batch * (ni * ni + (double)nt * nt + nb * nb), st);
  const zt m2ieta = make_double2(2.0 * eta.y, -2.0 * eta.x);
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nbatch = std::min(65535, batch - b0);
    auto kern = choose_regime(n, batch) == REG_SEQ ? zgj_seq_kernel : zgj_ws_kernel;
    // leaf_panel 2: two (NB x NB+1) ping-pong copies of the panel's diagonal block after Z
    const int bp = knob(KN_LEAF_PANEL);
    const size_t dbytes = bp == 2 ? sizeof(zt) * 2 * WS_NB * (WS_NB + 1) : 0;
    if (ws_smem(n) + dbytes > ws_smem(WS_NMAX)) throw HpsError{-1, "leaf_panel 2: shared memory"};
    kern<<<nbatch, 512, ws_smem(n) + dbytes, st>>>(
        S + (int64_t)b0 * sstride, n, sstride, store + (int64_t)b0 * mstride + (int64_t)nb * nt + nb, nt, mstride, n,
        info, WsFinish{K, R + (int64_t)b0 * nb * nb, m2ieta, p, c, leaf_nat, leaf0 + b0, kappa2, knob(KN_LEAF_PANEL),
                       knob(KN_LEAF_INPLACE)});
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
  return true;
}

// ---- representative-action planner (see the Regime comment) ----
namespace {
__global__ void plan_fill_kernel(zt* A, int n, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)e * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    const double v = (double)((h * 0x94D049BB133111EBull) >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    const int64_t ij = e % ((int64_t)n * n);
    const bool diag = ij / n == ij % n;
    A[e] = make_double2(u + (diag ? 2.0 : 0.0), v);
  }
}

int zgj_theta_o(int r, int n, int nbox, int nsm) {
  switch (r) {
    case REG_SMALL: {
      int occ = 1;
      const size_t smem = sizeof(zt) * ((size_t)n * (n + 1) + 2 * n) + sizeof(int) * n + 16;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, zgj_small_kernel, kThreads, smem);
      return std::max(1, occ) * nsm;
    }
    case REG_FUSED: return nbox >= nsm ? 2 * nsm : nsm;
    case REG_WS:
    case REG_SEQ: return nsm;
    default: return nbox;  // blocked regimes: every box of the level in one batched launch
  }
}

}  // namespace

// Measures the representative time of every feasible regime for `nbox` n x n inverses and
// records the argmin of eps = ceil(nbox / theta_o) * r (one-CTA-per-box regimes: r = one wave
// of theta_o boxes; blocked regimes: r measured on min(nbox, #SM) boxes, scaled linearly).
// eps/r/theta (length REG_COUNT, index = regime) get -1 for infeasible regimes.
int zgj_plan_inverse(int n, int nbox, double* eps, double* rt, int* theta) {
  int dev, nsm;
  HPS_CUDA_CHECK(cudaGetDevice(&dev));
  HPS_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t st;
  HPS_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int mmax = std::min(nbox, 2 * nsm);
  const size_t mat = (size_t)n * n, bytes = sizeof(zt) * mat * mmax;
  size_t wsb = 16;
  for (int r = REG_SMALL; r < REG_COUNT; ++r) {
    g_regime_force = r;
    if (regime_feasible(r, n)) wsb = std::max(wsb, zgj_workspace_bytes(n, mmax));
  }
  g_regime_force = REG_NONE;
  void *src = nullptr, *a = nullptr, *o = nullptr, *ws = nullptr, *info = nullptr;
  HPS_CUDA_CHECK(cudaMalloc(&src, bytes));
  HPS_CUDA_CHECK(cudaMalloc(&a, bytes));
  HPS_CUDA_CHECK(cudaMalloc(&o, bytes));
  HPS_CUDA_CHECK(cudaMalloc(&ws, wsb));
  HPS_CUDA_CHECK(cudaMalloc(&info, sizeof(int)));
  plan_fill_kernel<<<hps_num_sms() * 8, 256, 0, st>>>((zt*)src, n, (int64_t)mat * mmax);
  HPS_CUDA_CHECK(cudaGetLastError());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int best = REG_NONE;
  double beste = 0;
  for (int r = REG_SMALL; r < REG_COUNT; ++r) {
    eps[r] = rt[r] = -1.0;
    theta[r] = -1;
    if (!regime_feasible(r, n)) continue;
    const int th = zgj_theta_o(r, n, nbox, nsm);
    const int m = std::min(nbox, std::min(th, nsm * 2 >= th ? th : mmax));
    const int mm = std::min(m, mmax);
    g_regime_force = r;
    double tbest = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      HPS_CUDA_CHECK(cudaMemcpyAsync(a, src, sizeof(zt) * mat * mm, cudaMemcpyDeviceToDevice, st));
      HPS_CUDA_CHECK(cudaMemsetAsync(info, 0, sizeof(int), st));
      cudaEventRecord(e0, st);
      zgj_invert_impl((zt*)a, n, (int64_t)mat, (zt*)o, n, (int64_t)mat, n, mm, ws, (int*)info, st);
      cudaEventRecord(e1, st);
      HPS_CUDA_CHECK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) tbest = std::min(tbest, (double)ms);
    }
    g_regime_force = REG_NONE;
    double e;
    if (th >= nbox && (r == REG_P47 || r == REG_BLOCKED))
      e = tbest * (double)nbox / mm;  // batched over the level: linear in the boxes
    else
      e = tbest * (double)((nbox + th - 1) / th) * ((double)std::min(th, nbox) / mm);
    rt[r] = tbest;
    theta[r] = th;
    eps[r] = e;
    if (best == REG_NONE || e < beste) {
      best = r;
      beste = e;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(src);
  cudaFree(a);
  cudaFree(o);
  cudaFree(ws);
  cudaFree(info);
  cudaStreamDestroy(st);
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plan[{n, nbox}] = best;
  }
  return best;
}

void zgj_plan_set(int n, int nbox, int regime) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (regime <= REG_NONE || regime >= REG_COUNT)
    g_plan.erase({n, nbox});
  else
    g_plan[{n, nbox}] = regime;
}

void zgj_plan_clear() {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plan.clear();
}

int zgj_regime_of(int n, int nbox) { return choose_regime(n, nbox); }
void zgj_force_regime(int r) { g_regime_force = r; }

// |A_kk|^2 of the original matrices (reference of the natural-order pivot check)
__global__ void nat_diag_kernel(const zt* A, int64_t lda, int64_t bs, int n, double* d0) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
  if (k >= n) return;
  const zt v = A[(int64_t)b * bs + (int64_t)k * lda + k];
  d0[(int64_t)b * n + k] = fma(v.x, v.x, v.y * v.y);
}

// Natural-order blocked Gauss-Jordan: 16-column zgj_panel_nat_kernel panels and
// the blocked explicit-swap update with identity maps (any n).  Workspace as
// zgj_workspace_bytes(n, batch) for the blocked regime; *flag (device) is set to 1 when a pivot
// failed the check — out is then not the inverse and A is destroyed (the caller keeps a copy).
void zgj_invert_natural_blocked(zt* A, int64_t lda, int64_t bs, int n, int batch, void* ws, int* flag, cudaStream_t st);
size_t zgj_natural_blocked_workspace_bytes(int n, int batch);

// 64-wide block steps where the 16-column panels' K = 16 updates are memory-bound: n >= nat_bb_min,
// or a level whose matrices (batch x n^2 x 16 B) exceed a quarter of L2 (C4's n3 = 448 level,
// 64 x 3.2 MB, gains; C2's single n3 = 448 matrix stays in L2 and the 16-column panels win).
bool use_block_steps(int n, int batch) {
  return n >= knob(KN_NAT_BB_MIN) || (n >= 224 && sizeof(zt) * (double)batch * n * n >= 32.0 * (1 << 20));
}

void zgj_invert_natural(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch,
                        void* ws, int* flag, cudaStream_t st) {
  if (use_block_steps(n, batch)) {  // in place in A, then copied out
    zgj_invert_natural_blocked(A, lda, bs, n, batch, ws, flag, st);
    ProfScope ps(K_GJ_AUX, 0.0, 32.0 * (double)batch * n * n, st);
    if (lda == n && bs == (int64_t)n * n && ldo == n && obs == (int64_t)n * n) {
      HPS_CUDA_CHECK(cudaMemcpyAsync(out, A, sizeof(zt) * (size_t)batch * n * n, cudaMemcpyDeviceToDevice, st));
    } else {
      for (int b = 0; b < batch; ++b)
        HPS_CUDA_CHECK(cudaMemcpy2DAsync(out + (int64_t)b * obs, sizeof(zt) * ldo, A + (int64_t)b * bs, sizeof(zt) * lda,
                                         sizeof(zt) * n, n, cudaMemcpyDeviceToDevice, st));
    }
    return;
  }
  char* wsp = static_cast<char*>(ws);
  const size_t mbytes = ((sizeof(zt) * (size_t)batch * n * n + 255) / 256) * 256;
  zt* B2 = reinterpret_cast<zt*>(wsp);
  int* piv = reinterpret_cast<int*>(wsp + mbytes);
  int* rowsrc = piv + (size_t)batch * n;
  int* cinmap = rowsrc + (size_t)batch * n;
  int* pi = cinmap + (size_t)batch * n;
  double* d0 = reinterpret_cast<double*>(pi + (size_t)batch * n + 64);  // 256-byte aligned
  d0 = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(d0) + 255) & ~(uintptr_t)255);
  zt* buf[2] = {A, B2};
  const int64_t ld[2] = {lda, n}, bsz[2] = {bs, (int64_t)n * n};
  {
    ProfScope ps(K_GJ_AUX, 0.0, 24.0 * (double)batch * n, st);
    nat_diag_kernel<<<dim3((n + 255) / 256, batch), 256, 0, st>>>(A, lda, bs, n, d0);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
  const double rel2 = knob(KN_NAT_PIVOT_REL) * 1e-4;
  const int wide = knob(KN_NAT_W);  // 32: measured slower (C2 merges 5.20 -> 5.76 ms)
  const int lpr = knob(KN_NAT_LPR);
  const int cs = (n + 512 / lpr - 1) / (512 / lpr);
  const bool use_c = knob(KN_NATC) != 0 && cs <= 8;
  const int wmax = use_c && wide == 32 ? 32 : 16;
  const int npan = (n + wmax - 1) / wmax, nbw = (n + npan - 1) / npan;
  int cur = 0;
  for (int k0 = 0; k0 < n; k0 += nbw) {
    const int w = std::min(nbw, n - k0);
    PanelArgs pa{buf[cur], buf[1 - cur], ld[cur], bsz[cur], ld[1 - cur], bsz[1 - cur], n, k0, w, piv, rowsrc, cinmap,
                 flag};
    pa.pflag = flag;
    pa.d0 = d0;
    pa.rel2 = rel2;
    {
      ProfScope ps(K_GJ_PANEL, 8.0 * n * (double)w * w * batch, 32.0 * n * (double)w * batch, st);
      const bool blocked = knob(KN_NATB) != 0;
      if (blocked && wmax == 16) {
        zgj_panel_natb_kernel<<<dim3((n + 127) / 128, batch), 512, 0, st>>>(pa);
      } else if (!use_c) {
        zgj_panel_nat_kernel<<<batch, 512, 0, st>>>(pa);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(batch * cs);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (wmax == 32)
          HPS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zgj_panel_natc_kernel<8>, pa));
        else if (lpr == 8)
          HPS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zgj_panel_natc_kernel<2, 8>, pa));
        else
          HPS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, zgj_panel_natc_kernel<4, 4>, pa));
      }
      HPS_CUDA_CHECK(cudaGetLastError());
      count_launch();
    }
    const int nc = n - w;
    if (nc > 0) {
      ZGemm gm;
      gm.M = n;
      gm.N = nc;
      gm.K = w;
      gm.batch = batch;
      gm.A.ptr = buf[1 - cur] + k0;
      gm.A.rs = ld[1 - cur];
      gm.A.bs = bsz[1 - cur];
      gm.B.ptr = buf[cur];
      gm.B.rs = ld[cur];
      gm.B.bs = bsz[cur];
      gm.B.rmap = rowsrc + k0;
      gm.B.rmap_bs = n;
      gm.B.cskip_at = k0;
      gm.B.cskip_len = w;
      gm.Cin.ptr = buf[cur];
      gm.Cin.rs = ld[cur];
      gm.Cin.bs = bsz[cur];
      gm.Cin.rmap = cinmap;
      gm.Cin.rmap_bs = n;
      gm.Cin.cskip_at = k0;
      gm.Cin.cskip_len = w;
      gm.C.ptr = buf[1 - cur];
      gm.C.rs = ld[1 - cur];
      gm.C.bs = bsz[1 - cur];
      gm.C.cskip_at = k0;
      gm.C.cskip_len = w;
      gm.beta = make_double2(1.0, 0.0);
      zgemm(gm, st);
    }
    cur = 1 - cur;
  }
  // no permutation: the result is buf[cur] itself
  ProfScope ps(K_GJ_AUX, 0.0, 32.0 * (double)batch * n * n, st);
  if (ld[cur] == n && bsz[cur] == (int64_t)n * n && ldo == n && obs == (int64_t)n * n) {
    HPS_CUDA_CHECK(cudaMemcpyAsync(out, buf[cur], sizeof(zt) * (size_t)batch * n * n, cudaMemcpyDeviceToDevice, st));
  } else {
    for (int b = 0; b < batch; ++b)
      HPS_CUDA_CHECK(cudaMemcpy2DAsync(out + (int64_t)b * obs, sizeof(zt) * ldo, buf[cur] + (int64_t)b * bsz[cur],
                                       sizeof(zt) * ld[cur], sizeof(zt) * n, n, cudaMemcpyDeviceToDevice, st));
  }
  (void)pi;
}

// ---------------------------------------------------------------------------
// Natural-order Gauss-Jordan in 64-wide BLOCK steps for the large top-level W (n >= nat_bb_min,
// DESIGN.md 3.10).  Pivot rows known in advance make a block step exact algebra:
//   D = A[K, K] (K = [k0, k0 + b)), D^{-1} in natural order (its pivots ARE the global natural-order
//   pivots of steps k0 .. k0 + b - 1, checked against the original diagonal as in the panels);
//   T = -A[:, K] D^{-1} (rows outside K), T[K] = D^{-1} - I;  Z = A[K, :] (old);
//   A[:, j not in K] += T Z[:, j]  (one in-place K = b GEMM: rows outside K get the rank-b update,
//   rows K become D^{-1} Z);  A[rows outside K, K] = T,  A[K, K] = D^{-1}.
// The trailing update then reads and writes W once per 64 columns instead of once per 16
// (C4: n3 = 3584, W = 205 MB > L2: the K = 16 updates ran at ~10 TFLOP/s, memory-bound).
// ---------------------------------------------------------------------------
constexpr int NBB = 64;

// One CTA per matrix: D^{-1} of the bb x bb block at (k0, k0) in shared memory, natural order.
// D = A[K, K] (bb x bb, bb <= 64) inverted by one CTA in natural order, register-resident: warp w
// holds rows 4w .. 4w + 3, lane l columns 2l, 2l + 1 (the padding beyond bb is the identity, never a
// pivot).  Per step the pivot row goes through shared memory (double-buffered: one barrier per
// step), the pivot column by shuffles inside each warp.  The arithmetic is that of the textbook
// step D[i][j] -= D[i][k] (D[k][j] / D[k][k]) in the same operation order as before, so the result is
// unchanged; the shared-memory version moved the whole 64 x 64 block through shared memory every
// step (~1.8 us per step).
__global__ void __launch_bounds__(512) nat_block_inv_kernel(const zt* __restrict__ A, int64_t lda, int64_t bs, int n,
                                                            int k0, int bb, const double* __restrict__ d0,
                                                            double rel2, zt* __restrict__ Dt,
                                                            zt* __restrict__ T, int* __restrict__ flag) {
  __shared__ zt prow[2][NBB];
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, b = blockIdx.x;
  const zt* Ab = A + (int64_t)b * bs + (int64_t)k0 * lda + k0;
  zt d[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = 4 * w + t, j = 2 * lane + c;
      d[t][c] = (i < bb && j < bb) ? Ab[(int64_t)i * lda + j] : make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
  if (tid == 0) s_bad = 0;
  for (int k = 0; k < bb; ++k) {
    const int par = k & 1, kw = k >> 2, kt = k & 3, kc = k & 1, kl = k >> 1;
    if (w == kw) {  // publish the raw pivot row
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t == kt) {
          prow[par][2 * lane] = d[t][0];
          prow[par][2 * lane + 1] = d[t][1];
        }
    }
    // pivot column entries of my rows (lane kl holds column k)
    zt f[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const zt v = kc ? d[t][1] : d[t][0];
      f[t] = make_double2(__shfl_sync(0xffffffffu, v.x, kl), __shfl_sync(0xffffffffu, v.y, kl));
    }
    __syncthreads();
    const zt pv = prow[par][k];
    const zt inv = zinv_fast(pv);
    if (tid == 0) {
      const double m = fma(pv.x, pv.x, pv.y * pv.y);
      if (!(m > 0.0 && m >= rel2 * d0[(int64_t)b * n + k0 + k])) s_bad = 1;
    }
    zt pr[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int j = 2 * lane + c;
      pr[c] = j == k ? inv : zmul(prow[par][j], inv);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = 4 * w + t;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int j = 2 * lane + c;
        if (i == k) {
          d[t][c] = pr[c];
        } else if (j == k) {
          const zt g = zmul(f[t], inv);
          d[t][c] = make_double2(-g.x, -g.y);
        } else {
          zt v = d[t][c];
          v.x = fma(-f[t].x, pr[c].x, v.x);
          v.x = fma(f[t].y, pr[c].y, v.x);
          v.y = fma(-f[t].x, pr[c].y, v.y);
          v.y = fma(-f[t].y, pr[c].x, v.y);
          d[t][c] = v;
        }
      }
    }
  }
  __syncthreads();
  zt* Db = Dt + (int64_t)b * NBB * NBB;
  zt* Tb = T + (int64_t)b * n * NBB + (int64_t)k0 * NBB;  // T: [n][NBB] per matrix
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = 4 * w + t, j = 2 * lane + c;
      if (i < bb && j < bb) {
        Db[i * NBB + j] = d[t][c];
        Tb[i * NBB + j] = make_double2(d[t][c].x - (i == j ? 1.0 : 0.0), d[t][c].y);
      }
    }
  if (tid == 0 && s_bad) atomicExch(flag, 1);
}

// Lookahead stream of the block steps (one per host thread and device: the virtual ranks of the
// multi-GPU tests are host threads sharing a device, and must not share its work queue).
static cudaStream_t lookahead_stream() {
  thread_local std::vector<cudaStream_t> streams;
  int dev = 0;
  HPS_CUDA_CHECK(cudaGetDevice(&dev));
  if ((int)streams.size() <= dev) streams.resize(dev + 1, nullptr);
  if (!streams[dev]) HPS_CUDA_CHECK(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
  return streams[dev];
}

// With lookahead (knob nat_lookahead, default 1; off while per-launch event timing is on) the block
// step q's trailing update is split: first the columns of block q + 1, then -- on a second stream,
// concurrently with the rest of step q's update -- block q + 1's D^{-1} (a handful of CTAs, ~80 us of
// serial pivot steps) and its T product, so that the serial part of step q + 1 hides behind step q's
// wide GEMM.  T and D^{-1} are double-buffered; the arithmetic of every entry is unchanged.
void zgj_invert_natural_blocked(zt* A, int64_t lda, int64_t bs, int n, int batch, void* ws, int* flag, cudaStream_t st) {
  char* wsp = static_cast<char*>(ws);
  auto carve = [&](size_t bytes) {
    void* p = wsp;
    wsp += (bytes + 255) / 256 * 256;
    return p;
  };
  double* d0 = static_cast<double*>(carve(sizeof(double) * (size_t)batch * n));
  zt* Z = static_cast<zt*>(carve(sizeof(zt) * (size_t)batch * NBB * n));
  zt* Tb[2];
  zt* Dtb[2];
  for (int i = 0; i < 2; ++i) {
    Tb[i] = static_cast<zt*>(carve(sizeof(zt) * (size_t)batch * n * NBB));
    Dtb[i] = static_cast<zt*>(carve(sizeof(zt) * (size_t)batch * NBB * NBB));
  }
  {
    ProfScope ps(K_GJ_AUX, 0.0, 24.0 * (double)batch * n, st);
    nat_diag_kernel<<<dim3((n + 255) / 256, batch), 256, 0, st>>>(A, lda, bs, n, d0);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
  const double rel2 = knob(KN_NAT_PIVOT_REL) * 1e-4;
  const int nblk = (n + NBB - 1) / NBB;
  auto k0of = [&](int q) { return (int)((int64_t)q * n / nblk); };
  auto bbof = [&](int q) { return (int)((int64_t)(q + 1) * n / nblk) - k0of(q); };  // equal blocks
  const bool la = knob(KN_NAT_LOOKAHEAD) != 0 && !prof_timing_active() && nblk > 1;
  cudaStream_t st2 = la ? lookahead_stream() : st;
  cudaEvent_t evA = nullptr, evB = nullptr;
  if (la) {
    HPS_CUDA_CHECK(cudaEventCreateWithFlags(&evA, cudaEventDisableTiming));
    HPS_CUDA_CHECK(cudaEventCreateWithFlags(&evB, cudaEventDisableTiming));
  }
  // D^{-1} of block q and T[rows outside K] = -A[rows outside K, K] D^{-1} into buffer q & 1
  auto dinv_T = [&](int q, cudaStream_t s) {
    const int k0 = k0of(q), bb = bbof(q);
    zt* T = Tb[q & 1];
    zt* Dt = Dtb[q & 1];
    {
      ProfScope ps(K_GJ_PANEL, 8.0 * (double)bb * bb * bb * batch, 32.0 * (double)bb * bb * batch, s);
      nat_block_inv_kernel<<<batch, 512, 0, s>>>(A, lda, bs, n, k0, bb, d0, rel2, Dt, T, flag);
      HPS_CUDA_CHECK(cudaGetLastError());
      count_launch();
    }
    if (n > bb) {
      ZGemm g;
      g.M = n - bb;
      g.N = bb;
      g.K = bb;
      g.batch = batch;
      g.A.ptr = A + k0;
      g.A.rs = lda;
      g.A.bs = bs;
      g.A.rskip_at = k0;
      g.A.rskip_len = bb;
      g.B.ptr = Dt;
      g.B.rs = NBB;
      g.B.bs = (int64_t)NBB * NBB;
      g.C.ptr = T;
      g.C.rs = NBB;
      g.C.bs = (int64_t)n * NBB;
      g.C.rskip_at = k0;
      g.C.rskip_len = bb;
      g.alpha = make_double2(-1.0, 0.0);
      zgemm(g, s);
    }
  };
  // A[:, cols] += T Z[:, cols] (in place) for the columns [c0, c0 + nc) minus the window
  // [skip_at, skip_at + skip_len) (nc counts the columns actually updated)
  auto update = [&](int q, int c0, int nc, int skip_at, int skip_len) {
    if (nc <= 0) return;
    const int bb = bbof(q);
    ZGemm g;
    g.M = n;
    g.N = nc;
    g.K = bb;
    g.batch = batch;
    g.A.ptr = Tb[q & 1];
    g.A.rs = NBB;
    g.A.bs = (int64_t)n * NBB;
    g.B.ptr = Z + c0;
    g.B.rs = n;
    g.B.bs = (int64_t)NBB * n;
    g.B.cskip_at = skip_at;
    g.B.cskip_len = skip_len;
    g.Cin.ptr = A + c0;
    g.Cin.rs = lda;
    g.Cin.bs = bs;
    g.Cin.cskip_at = skip_at;
    g.Cin.cskip_len = skip_len;
    g.C.ptr = A + c0;
    g.C.rs = lda;
    g.C.bs = bs;
    g.C.cskip_at = skip_at;
    g.C.cskip_len = skip_len;
    g.beta = make_double2(1.0, 0.0);
    zgemm(g, st);
  };
  dinv_T(0, st);
  for (int q = 0; q < nblk; ++q) {
    const int k0 = k0of(q), bb = bbof(q);
    {  // Z = A[K, :]
      ZCopy c;
      c.M = bb;
      c.N = n;
      c.batch = batch;
      c.A.ptr = A + (int64_t)k0 * lda;
      c.A.rs = lda;
      c.A.bs = bs;
      c.C.ptr = Z;
      c.C.rs = n;
      c.C.bs = (int64_t)NBB * n;
      zcopy(c, st);
    }
    if (q + 1 < nblk && la) {
      const int k1 = k0of(q + 1), b1 = bbof(q + 1);
      update(q, k1, b1, 0x7fffffff, 0);  // block q + 1's columns first
      HPS_CUDA_CHECK(cudaEventRecord(evA, st));
      HPS_CUDA_CHECK(cudaStreamWaitEvent(st2, evA, 0));
      dinv_T(q + 1, st2);
      HPS_CUDA_CHECK(cudaEventRecord(evB, st2));
      update(q, 0, n - bb - b1, k0, bb + b1);  // the rest, beside block q + 1's serial part
    } else {
      update(q, 0, n - bb, k0, bb);
    }
    {  // A[rows outside K, K] = T, A[K, K] = D^{-1}
      ZCopy c[2];
      c[0].M = n - bb;
      c[0].N = bb;
      c[0].batch = batch;
      c[0].A.ptr = Tb[q & 1];
      c[0].A.rs = NBB;
      c[0].A.bs = (int64_t)n * NBB;
      c[0].A.rskip_at = k0;
      c[0].A.rskip_len = bb;
      c[0].C.ptr = A + k0;
      c[0].C.rs = lda;
      c[0].C.bs = bs;
      c[0].C.rskip_at = k0;
      c[0].C.rskip_len = bb;
      c[1].M = bb;
      c[1].N = bb;
      c[1].batch = batch;
      c[1].A.ptr = Dtb[q & 1];
      c[1].A.rs = NBB;
      c[1].A.bs = (int64_t)NBB * NBB;
      c[1].C.ptr = A + (int64_t)k0 * lda + k0;
      c[1].C.rs = lda;
      c[1].C.bs = bs;
      zcopy_multi(c, 2, st);  // (c[0] is empty when the block is the whole matrix)
    }
    if (q + 1 < nblk) {
      if (la) HPS_CUDA_CHECK(cudaStreamWaitEvent(st, evB, 0));
      else dinv_T(q + 1, st);
    }
  }
  if (la) {
    HPS_CUDA_CHECK(cudaEventDestroy(evA));
    HPS_CUDA_CHECK(cudaEventDestroy(evB));
  }
}

size_t zgj_natural_blocked_workspace_bytes(int n, int batch) {
  return 6 * 256 + sizeof(double) * (size_t)batch * n + sizeof(zt) * (size_t)batch * (3 * (size_t)NBB * n + 2 * NBB * NBB);
}

size_t zgj_natural_workspace_bytes(int n, int batch) {
  if (use_block_steps(n, batch)) return zgj_natural_blocked_workspace_bytes(n, batch);
  const size_t mbytes = ((sizeof(zt) * (size_t)batch * n * n + 255) / 256) * 256;
  return mbytes + sizeof(int) * (size_t)batch * n * 4 + 256 + 512 + sizeof(double) * (size_t)batch * n;
}

size_t zgj_workspace_bytes(int n, int batch) {
  const int reg = choose_regime(n, batch);
  if (reg == REG_SMALL || reg == REG_WS || reg == REG_SEQ || reg == REG_FUSED) return 16;
  const size_t mbytes = ((sizeof(zt) * (size_t)batch * n * n + 255) / 256) * 256;
  return mbytes + sizeof(int) * (size_t)batch * n * 4 + 256;
}

void zgj_invert(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch, void* ws,
                int* info, cudaStream_t st, int64_t* launches) {
  (void)launches;
  if (!knob(KN_TRACE)) return zgj_invert_impl(A, lda, bs, out, ldo, obs, n, batch, ws, info, st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  zgj_invert_impl(A, lda, bs, out, ldo, obs, n, batch, ws, info, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  fprintf(stderr, "[zgj] n=%d batch=%d  %.3f ms  %.2f TF (incl. updates)\n", n, batch, ms,
          8.0 * n * (double)n * n * batch / ms / 1e9);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}
