// zgemm.cu — batched complex128 GEMM on the FP64 tensor cores of sm_100a.
//
// Every dense product of the HPS merge (Algorithm 1 lines 7-13), of the
// blocked Gauss-Jordan update (zgj.cu) and of the solve sweeps (Algorithm 2) is one call of
// this kernel.  sm_100a has no tcgen05 / TMEM path for f64 (ptxas rejects .kind::f64), so the
// FP64 tensor path is warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4).  A complex product is four
// real DMMAs, Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br, or (M3, knob gemm_3m) three:
// T1 += Ar Br, T2 += Ai Bi, T3 += (Ar + Ai)(Br + Bi), then Cr = T1 - T2, Ci = T3 - T1 - T2 -- the
// 3M form of ZGEMM3M, all in FP64 (normwise error bound a small constant times the 4M one).
// Operands are staged global -> shared with cp.async (16 B = one complex element, zero-fill
// for ragged edges and for "zero" map entries), double-buffered.  Shared-memory strides are
// chosen so that the 8x4 / 4x8 DMMA fragments load as conflict-free 16-byte LDS.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "hps_internal.cuh"

namespace {

constexpr int BK = 16;  // K depth of one pipeline stage (complex elements)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ zt zmul(zt a, zt b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }

template <int BM, int BN, int WM, int WN>
struct Cfg {
  static constexpr int NWM = BM / WM, NWN = BN / WN, NT = NWM * NWN * 32;
  static constexpr int TM = WM / 8, TN = WN / 8;
  static constexpr int AS = BK + 4;  // A tile row stride (complex)
  static constexpr int BS = BN + 2;  // B tile row stride (complex)
  static constexpr int ITA = BM * BK / NT, ITB = BK * BN / NT;
  static constexpr size_t SMEM = sizeof(zt) * 2 * (BM * AS + BK * BS);
  static_assert(NT % BK == 0 && ITA >= 1 && ITB >= 1 && (BM * BK) % NT == 0 && (BK * BN) % NT == 0, "cfg");
  static_assert(NT % BN == 0 || BN % NT == 0, "cfg");
};

// BCOL: B is column-major (rs == 1, no maps: the solve reads s in the ABI layout [RHS][leaf][n_i],
// columns 0.2-3 GB apart): the B tile is loaded k-fastest, so that a warp's cp.async requests cover
// runs of BK consecutive elements of a column instead of one 16-byte piece per column.
template <int BM, int BN, int WM, int WN, bool BCOL = false, bool M3 = false>
__global__ void __launch_bounds__(Cfg<BM, BN, WM, WN>::NT, (BM == 64 && BN == 32) ? 3 : 0) zgemm_kernel(const ZGemm g) {
  using C = Cfg<BM, BN, WM, WN>;
  constexpr int NT = C::NT, TM = C::TM, TN = C::TN, AS = C::AS, BS = C::BS, ITA = C::ITA, ITB = C::ITB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  zt* As = reinterpret_cast<zt*>(smem_raw);  // [2][BM][AS]
  zt* Bs = As + 2 * BM * AS;                 // [2][BK][BS]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::NWN, wn = warp % C::NWN;
  // Tile order: row-major (group_m = 1), or grouped -- consecutive CTAs sweep a group of group_m
  // row blocks column by column, so the CTAs in flight share a few A row blocks and B column
  // blocks instead of streaming all of B once per row block (L2 reuse: the C4 root product read
  // 96 GB of DRAM for 4.5 GB of operands).  The 64 x 32 kernel is held to 3 CTAs per SM by its
  // launch bounds (round 2's first grouped order raised it to 180 registers, 2 CTAs per SM).
  const int tilesN = (g.N + BN - 1) / BN;
  int m0, n0;
  constexpr bool kGroup = BM == 64 && (BN == 32 || (BN == 64 && WN == 32));  // the long-K merge tiles (registers elsewhere)
  if (!kGroup || g.group_m <= 1) {
    m0 = (blockIdx.x / tilesN) * BM;
    n0 = (blockIdx.x % tilesN) * BN;
  } else {
    const int tilesM = (g.M + BM - 1) / BM, per_group = g.group_m * tilesN, grp = blockIdx.x / per_group;
    const int first_m = grp * g.group_m, gm = min(tilesM - first_m, g.group_m), local = blockIdx.x - grp * per_group;
    m0 = (first_m + local % gm) * BM;
    n0 = (local / gm) * BN;
  }

  // Fixed per-thread load coordinates: A column (k) and B column (n) are fixed across the
  // unrolled iterations; A rows / B rows step by NT/BK and NT/BN.
  const int a_c = tid % BK, a_r0 = tid / BK;
  const int b_c = tid % BN, b_r0 = tid / BN;
  constexpr int A_RSTEP = NT / BK;
  constexpr int B_RSTEP = (NT >= BN) ? NT / BN : 1;

  // split-K: this CTA's slice [kbeg, kend) of K (whole BK stages; slice 0 carries Cin)
  const int ksl = blockIdx.z;
  const int kchunk = ((g.K + (int)gridDim.z - 1) / (int)gridDim.z + BK - 1) / BK * BK;
  const int kbeg = ksl * kchunk, kend = min(g.K, kbeg + kchunk);
  for (int b = blockIdx.y; b < g.batch; b += gridDim.y) {
    const zt* Ab = g.A.ptr + zboff(g.A, b);
    const zt* Bb = g.B.ptr + zboff(g.B, b);
    const int* Arm = g.A.rmap ? g.A.rmap + (int64_t)b * g.A.rmap_bs : nullptr;
    const int* Brm = g.B.rmap ? g.B.rmap + (int64_t)b * g.B.rmap_bs : nullptr;
    const int* Crm = g.C.rmap ? g.C.rmap + (int64_t)b * g.C.rmap_bs : nullptr;
    const int* Irm = g.Cin.rmap ? g.Cin.rmap + (int64_t)b * g.Cin.rmap_bs : nullptr;
    // A row offsets (fixed over k)
    int64_t a_roff[ITA];
    bool a_rok[ITA];
#pragma unroll
    for (int it = 0; it < ITA; ++it) {
      const int gi = m0 + a_r0 + it * A_RSTEP;
      int ri = gi < g.M ? zrow(g.A, Arm, gi) : -1;
      a_rok[it] = ri >= 0;
      a_roff[it] = (int64_t)(ri < 0 ? 0 : ri) * g.A.rs;
    }
    // B column offset (fixed over k)
    int64_t b_coff;
    bool b_cok;
    {
      const int gj = n0 + b_c;
      int cj = gj < g.N ? zcol(g.B.cmap, gj, g.B.cskip_at, g.B.cskip_len) : -1;
      b_cok = cj >= 0;
      b_coff = (int64_t)(cj < 0 ? 0 : cj) * g.B.cs;
    }
    // BCOL: thread (k = tid % BK, columns tid / BK + it * NT / BK)
    constexpr int BC_JSTEP = NT / BK;
    int64_t bc_off[BCOL ? ITB : 1];
    bool bc_ok[BCOL ? ITB : 1];
    if constexpr (BCOL) {
#pragma unroll
      for (int it = 0; it < ITB; ++it) {
        const int gj = n0 + tid / BK + it * BC_JSTEP;
        bc_ok[it] = gj < g.N;
        bc_off[it] = (int64_t)(gj < g.N ? gj : 0) * g.B.cs;
      }
    }

    auto load_stage = [&](int stage, int k0) {
      {
        const int gk = k0 + a_c;
        int ck = gk < kend ? zcol(g.A.cmap, gk, g.A.cskip_at, g.A.cskip_len) : -1;
        const int64_t coff = (int64_t)(ck < 0 ? 0 : ck) * g.A.cs;
#pragma unroll
        for (int it = 0; it < ITA; ++it) {
          const bool ok = a_rok[it] && ck >= 0;
          cp_async16(&As[(stage * BM + a_r0 + it * A_RSTEP) * AS + a_c], ok ? Ab + a_roff[it] + coff : g.A.ptr, ok);
        }
      }
      if constexpr (BCOL) {
        const int kk = tid % BK, gk = k0 + kk;
#pragma unroll
        for (int it = 0; it < ITB; ++it) {
          const int jj = tid / BK + it * BC_JSTEP;
          const bool ok = bc_ok[it] && gk < kend;
          cp_async16(&Bs[(stage * BK + kk) * BS + jj], ok ? Bb + gk + bc_off[it] : g.B.ptr, ok);
        }
      } else {
#pragma unroll
        for (int it = 0; it < ITB; ++it) {
          const int r = b_r0 + it * B_RSTEP;
          const int gk = k0 + r;
          int rk = gk < kend ? (Brm ? Brm[gk] : gk) : -1;
          const bool ok = b_cok && rk >= 0;
          cp_async16(&Bs[(stage * BK + r) * BS + b_c], ok ? Bb + (int64_t)rk * g.B.rs + b_coff : g.B.ptr, ok);
        }
      }
      cp_async_commit();
    };

    const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
    if (nk > 0) load_stage(0, kbeg);

    // Accumulators start at (beta / alpha) Cin, so the Cin loads overlap the first stage.  When
    // beta == alpha (every use but one) the raw values are loaded with no arithmetic, so all
    // loads are in flight together and the first DMMA is the first consumer.
    // M3: accr = T1, acci = T3, acc2 = T2 (started at Cr, Cr + Ci and 0; converted before the epilogue)
    double accr[TM][TN][2], acci[TM][TN][2], acc2[TM][TN][2];
    const zt* Cinb = (g.Cin.ptr && ksl == 0) ? g.Cin.ptr + zboff(g.Cin, b) : nullptr;
    const bool raw = g.beta.x == g.alpha.x && g.beta.y == g.alpha.y;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int gi = m0 + wm * C::TM * 8 + i * 8 + (lane >> 2);
      const int ri = (Cinb && gi < g.M) ? zrow(g.Cin, Irm, gi) : -1;
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gj = n0 + wn * C::TN * 8 + j * 8 + (lane & 3) * 2 + h;
          zt v = make_double2(0.0, 0.0);
          if (ri >= 0 && gj < g.N) {
            const int cj = zcol(g.Cin.cmap, gj, g.Cin.cskip_at, g.Cin.cskip_len);
            if (cj >= 0) v = Cinb[(int64_t)ri * g.Cin.rs + (int64_t)cj * g.Cin.cs];
          }
          accr[i][j][h] = v.x;
          acci[i][j][h] = v.y;
        }
    }
    if (Cinb && !raw) {
      const double d = g.alpha.x * g.alpha.x + g.alpha.y * g.alpha.y;
      const zt ba = zmul(g.beta, make_double2(g.alpha.x / d, -g.alpha.y / d));
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const zt v = zmul(ba, make_double2(accr[i][j][h], acci[i][j][h]));
            accr[i][j][h] = v.x;
            acci[i][j][h] = v.y;
          }
    }
    if constexpr (M3) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            acci[i][j][h] += accr[i][j][h];
            acc2[i][j][h] = 0.0;
          }
    }

    for (int kt = 0; kt < nk; ++kt) {
      if (kt + 1 < nk) {
        load_stage((kt + 1) & 1, kbeg + (kt + 1) * BK);
        cp_async_wait1();
      } else {
        cp_async_wait0();
      }
      __syncthreads();
      const zt* Ast = As + (kt & 1) * BM * AS + (wm * C::TM * 8) * AS;
      const zt* Bst = Bs + (kt & 1) * BK * BS + wn * C::TN * 8;
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        zt af[TM], bf[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) af[i] = Ast[(i * 8 + (lane >> 2)) * AS + kk * 4 + (lane & 3)];
#pragma unroll
        for (int j = 0; j < TN; ++j) bf[j] = Bst[(kk * 4 + (lane & 3)) * BS + j * 8 + (lane >> 2)];
        if constexpr (M3) {
          double as[TM], bs[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i) as[i] = af[i].x + af[i].y;
#pragma unroll
          for (int j = 0; j < TN; ++j) bs[j] = bf[j].x + bf[j].y;
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(accr[i][j][0], accr[i][j][1], af[i].x, bf[j].x);
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(acc2[i][j][0], acc2[i][j][1], af[i].y, bf[j].y);
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(acci[i][j][0], acci[i][j][1], as[i], bs[j]);
        } else {
        // four real sub-products, ordered so that consecutive DMMAs on one accumulator are
        // 2*TM*TN instructions apart (no back-to-back accumulator dependency)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(accr[i][j][0], accr[i][j][1], af[i].x, bf[j].x);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(acci[i][j][0], acci[i][j][1], af[i].x, bf[j].y);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(accr[i][j][0], accr[i][j][1], -af[i].y, bf[j].y);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(acci[i][j][0], acci[i][j][1], af[i].y, bf[j].x);
        }
      }
      __syncthreads();
    }

    if constexpr (M3) {  // (T1, T3, T2) -> (Cr, Ci)
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double t1 = accr[i][j][h], t2 = acc2[i][j][h];
            accr[i][j][h] = t1 - t2;
            acci[i][j][h] = (acci[i][j][h] - t1) - t2;
          }
    }
    if (g.ws) {  // split-K: the raw partial tile of this slice (alpha, diag and C's maps in the reduction)
      zt* Wb = g.ws + ((int64_t)ksl * g.batch + b) * g.M * g.N;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int gi = m0 + wm * C::TM * 8 + i * 8 + (lane >> 2);
        if (gi >= g.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gj = n0 + wn * C::TN * 8 + j * 8 + (lane & 3) * 2 + h;
            if (gj < g.N) Wb[(int64_t)gi * g.N + gj] = make_double2(accr[i][j][h], acci[i][j][h]);
          }
      }
      continue;
    }
    // Epilogue: C = alpha * acc + diag * [i == j]
    zt* Cb = g.C.ptr + zboff(g.C, b);
    // Column-contiguous output (rs == 1: the solve writes u straight into the ABI layout, RHS
    // outermost): the tile goes through shared memory so that each column is stored as BM
    // consecutive elements instead of 16-byte pieces 0.26 GB apart.
    constexpr bool kTr = BN * (BM + 1) <= 2 * (BM * AS + BK * BS);
    if (kTr && g.C.rs == 1 && !Crm && !g.C.cmap && g.C.rskip_len == 0) {
      zt* Ct = As;  // [BN][BM + 1]; the operand tiles are free (the K loop ended with a barrier)
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int lr = wm * C::TM * 8 + i * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int lc = wn * C::TN * 8 + j * 8 + (lane & 3) * 2 + h;
            zt v = zmul(g.alpha, make_double2(accr[i][j][h], acci[i][j][h]));
            if (m0 + lr == n0 + lc) {
              v.x += g.diag.x;
              v.y += g.diag.y;
            }
            Ct[lc * (BM + 1) + lr] = v;
          }
      }
      __syncthreads();
      for (int e = tid; e < BM * BN; e += NT) {
        const int lc = e / BM, lr = e - lc * BM, gi = m0 + lr, gj = n0 + lc;
        if (gi < g.M && gj < g.N) Cb[(int64_t)gi + (int64_t)gj * g.C.cs] = Ct[lc * (BM + 1) + lr];
      }
      __syncthreads();  // Ct is the next batch entry's operand buffer
      continue;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int gi = m0 + wm * C::TM * 8 + i * 8 + (lane >> 2);
      if (gi >= g.M) continue;
      const int ro = zrow(g.C, Crm, gi);
      if (ro < 0) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gj = n0 + wn * C::TN * 8 + j * 8 + (lane & 3) * 2 + h;
          if (gj >= g.N) continue;
          zt v = zmul(g.alpha, make_double2(accr[i][j][h], acci[i][j][h]));
          if (gi == gj) {
            v.x += g.diag.x;
            v.y += g.diag.y;
          }
          const int co = zcol(g.C.cmap, gj, g.C.cskip_at, g.C.cskip_len);
          if (co >= 0) Cb[(int64_t)ro * g.C.rs + (int64_t)co * g.C.cs] = v;
        }
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, bool BCOL = false>
void launch(const ZGemm& g, cudaStream_t st) {
  using C = Cfg<BM, BN, WM, WN>;
  static bool attr_set = false;
  const bool m3 = knob(KN_GEMM_3M) != 0;
  auto kern = m3 ? zgemm_kernel<BM, BN, WM, WN, BCOL, true> : zgemm_kernel<BM, BN, WM, WN, BCOL, false>;
  if (!attr_set) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgemm_kernel<BM, BN, WM, WN, BCOL, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    HPS_CUDA_CHECK(cudaFuncSetAttribute(zgemm_kernel<BM, BN, WM, WN, BCOL, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr_set = true;
  }
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  dim3 grid(tiles, g.batch < 65535 ? g.batch : 65535, g.ws ? g.ksplit : 1);
  kern<<<grid, C::NT, C::SMEM, st>>>(g);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

// Skinny products (N <= 4, the solve sweeps at few right-hand sides): one warp per output
// row, lanes stride over K with coalesced 16-byte loads of the A row, warp-shuffle reduction.
// Bandwidth-bound (A is read once); parallel over M x batch warps, so the long-K / single-merge
// matvecs at the top of the tree do not serialise on a handful of CTAs.
template <int NMAX, int KS>
__global__ void __launch_bounds__(256) zgemv_kernel(const ZGemm g) {
  // KS warps share one output row (K split KS ways, partial sums reduced through shared
  // memory), so the long-K matvecs at the top of the tree (few rows) still fill the GPU; the
  // K loop keeps 4 independent A/B loads in flight per lane.
  constexpr int RPB = 8 / KS;
  __shared__ double part[8][NMAX][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, kw = warp % KS;
  const int row = blockIdx.x * RPB + warp / KS;
  const bool live = row < g.M;
  for (int b = blockIdx.y; b < g.batch; b += gridDim.y) {
    const int* Arm = g.A.rmap ? g.A.rmap + (int64_t)b * g.A.rmap_bs : nullptr;
    const int* Brm = g.B.rmap ? g.B.rmap + (int64_t)b * g.B.rmap_bs : nullptr;
    const int* Crm = g.C.rmap ? g.C.rmap + (int64_t)b * g.C.rmap_bs : nullptr;
    const int* Irm = g.Cin.rmap ? g.Cin.rmap + (int64_t)b * g.Cin.rmap_bs : nullptr;
    const int ra = live ? (Arm ? Arm[row] : row) : -1;
    double accr[NMAX], acci[NMAX];
#pragma unroll
    for (int r = 0; r < NMAX; ++r) accr[r] = acci[r] = 0.0;
    if (ra >= 0) {
      const zt* Ab = g.A.ptr + zboff(g.A, b) + (int64_t)ra * g.A.rs;
      const zt* Bb = g.B.ptr + zboff(g.B, b);
      int64_t bco[NMAX];
      bool bok[NMAX];
#pragma unroll
      for (int r = 0; r < NMAX; ++r) {
        const int cj = r < g.N ? zcol(g.B.cmap, r, g.B.cskip_at, g.B.cskip_len) : -1;
        bok[r] = cj >= 0;
        bco[r] = (int64_t)(cj < 0 ? 0 : cj) * g.B.cs;
      }
      constexpr int U = 4;
      for (int k0 = kw * 32 + lane; k0 < g.K; k0 += 32 * KS * U) {
        zt av[U], bv[U][NMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u * 32 * KS;
          const int ck = k < g.K ? zcol(g.A.cmap, k, g.A.cskip_at, g.A.cskip_len) : -1;
          const int rk = k < g.K ? (Brm ? Brm[k] : k) : -1;
          const bool ok = ck >= 0 && rk >= 0;
          av[u] = ok ? Ab[(int64_t)ck * g.A.cs] : make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 0; r < NMAX; ++r)
            bv[u][r] = (ok && bok[r]) ? Bb[(int64_t)rk * g.B.rs + bco[r]] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < NMAX; ++r) {
            accr[r] = fma(av[u].x, bv[u][r].x, accr[r]);
            accr[r] = fma(-av[u].y, bv[u][r].y, accr[r]);
            acci[r] = fma(av[u].x, bv[u][r].y, acci[r]);
            acci[r] = fma(av[u].y, bv[u][r].x, acci[r]);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < NMAX; ++r)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        accr[r] += __shfl_xor_sync(0xffffffffu, accr[r], o);
        acci[r] += __shfl_xor_sync(0xffffffffu, acci[r], o);
      }
    if (KS > 1) {
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < NMAX; ++r) {
          part[warp][r][0] = accr[r];
          part[warp][r][1] = acci[r];
        }
      }
      __syncthreads();
      if (kw == 0) {
#pragma unroll
        for (int r = 0; r < NMAX; ++r)
#pragma unroll
          for (int j = 1; j < KS; ++j) {
            accr[r] += part[warp + j][r][0];
            acci[r] += part[warp + j][r][1];
          }
      }
      __syncthreads();
    }
    if (!live || kw != 0) continue;
    const int ro = Crm ? Crm[row] : row;
    if (ro < 0) continue;
#pragma unroll
    for (int r = 0; r < NMAX; ++r) {
      if (lane != r || r >= g.N) continue;
      zt v = zmul(g.alpha, make_double2(accr[r], acci[r]));
      if (g.Cin.ptr) {
        const int ri = Irm ? Irm[row] : row;
        const int cj = zcol(g.Cin.cmap, r, g.Cin.cskip_at, g.Cin.cskip_len);
        if (ri >= 0 && cj >= 0) {
          const zt cv = zmul(g.beta, g.Cin.ptr[zboff(g.Cin, b) + (int64_t)ri * g.Cin.rs + (int64_t)cj * g.Cin.cs]);
          v.x += cv.x;
          v.y += cv.y;
        }
      }
      if (row == r) {
        v.x += g.diag.x;
        v.y += g.diag.y;
      }
      const int co = zcol(g.C.cmap, r, g.C.cskip_at, g.C.cskip_len);
      if (co >= 0) g.C.ptr[zboff(g.C, b) + (int64_t)ro * g.C.rs + (int64_t)co * g.C.cs] = v;
    }
  }
}

// Short-K variant (K <= 128): LPR lanes per output row (32 / LPR rows per warp), no shared-memory
// reduction; the 32-lane form leaves most lanes idle when K is a few dozen (the solve's Psi t,
// K = n_b = 56).
template <int NMAX, int LPR>
__global__ void __launch_bounds__(256) zgemv_short_kernel(const ZGemm g) {
  constexpr int RW = 32 / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, li = lane % LPR;
  const int row = (blockIdx.x * 8 + warp) * RW + lane / LPR;
  const bool live = row < g.M;
  for (int b = blockIdx.y; b < g.batch; b += gridDim.y) {
    const int* Arm = g.A.rmap ? g.A.rmap + (int64_t)b * g.A.rmap_bs : nullptr;
    const int* Brm = g.B.rmap ? g.B.rmap + (int64_t)b * g.B.rmap_bs : nullptr;
    const int* Crm = g.C.rmap ? g.C.rmap + (int64_t)b * g.C.rmap_bs : nullptr;
    const int* Irm = g.Cin.rmap ? g.Cin.rmap + (int64_t)b * g.Cin.rmap_bs : nullptr;
    const int ra = live ? (Arm ? Arm[row] : row) : -1;
    double accr[NMAX], acci[NMAX];
#pragma unroll
    for (int r = 0; r < NMAX; ++r) accr[r] = acci[r] = 0.0;
    if (ra >= 0) {
      const zt* Ab = g.A.ptr + zboff(g.A, b) + (int64_t)ra * g.A.rs;
      const zt* Bb = g.B.ptr + zboff(g.B, b);
      int64_t bco[NMAX];
      bool bok[NMAX];
#pragma unroll
      for (int r = 0; r < NMAX; ++r) {
        const int cj = r < g.N ? zcol(g.B.cmap, r, g.B.cskip_at, g.B.cskip_len) : -1;
        bok[r] = cj >= 0;
        bco[r] = (int64_t)(cj < 0 ? 0 : cj) * g.B.cs;
      }
      constexpr int U = 4;
      for (int k0 = li; k0 < g.K; k0 += LPR * U) {
        zt av[U], bv[U][NMAX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u * LPR;
          const int ck = k < g.K ? zcol(g.A.cmap, k, g.A.cskip_at, g.A.cskip_len) : -1;
          const int rk = k < g.K ? (Brm ? Brm[k] : k) : -1;
          const bool ok = ck >= 0 && rk >= 0;
          av[u] = ok ? Ab[(int64_t)ck * g.A.cs] : make_double2(0.0, 0.0);
#pragma unroll
          for (int r = 0; r < NMAX; ++r)
            bv[u][r] = (ok && bok[r]) ? Bb[(int64_t)rk * g.B.rs + bco[r]] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < NMAX; ++r) {
            accr[r] = fma(av[u].x, bv[u][r].x, accr[r]);
            accr[r] = fma(-av[u].y, bv[u][r].y, accr[r]);
            acci[r] = fma(av[u].x, bv[u][r].y, acci[r]);
            acci[r] = fma(av[u].y, bv[u][r].x, acci[r]);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < NMAX; ++r)
#pragma unroll
      for (int o = LPR / 2; o; o >>= 1) {
        accr[r] += __shfl_xor_sync(0xffffffffu, accr[r], o);
        acci[r] += __shfl_xor_sync(0xffffffffu, acci[r], o);
      }
    if (!live) continue;
    const int ro = Crm ? Crm[row] : row;
    if (ro < 0) continue;
#pragma unroll
    for (int r = 0; r < NMAX; ++r) {
      if (li != r || r >= g.N) continue;
      zt v = zmul(g.alpha, make_double2(accr[r], acci[r]));
      if (g.Cin.ptr) {
        const int ri = Irm ? Irm[row] : row;
        const int cj = zcol(g.Cin.cmap, r, g.Cin.cskip_at, g.Cin.cskip_len);
        if (ri >= 0 && cj >= 0) {
          const zt cv = zmul(g.beta, g.Cin.ptr[zboff(g.Cin, b) + (int64_t)ri * g.Cin.rs + (int64_t)cj * g.Cin.cs]);
          v.x += cv.x;
          v.y += cv.y;
        }
      }
      if (row == r) {
        v.x += g.diag.x;
        v.y += g.diag.y;
      }
      const int co = zcol(g.C.cmap, r, g.C.cskip_at, g.C.cskip_len);
      if (co >= 0) g.C.ptr[zboff(g.C, b) + (int64_t)ro * g.C.rs + (int64_t)co * g.C.cs] = v;
    }
  }
}

// Skinny-product launcher: KS from the work size (enough warps to fill the GPU, K >= 64 per warp)
template <int NMAX>
void launch_gemv(const ZGemm& g, cudaStream_t st) {
  const int64_t rows = (int64_t)g.M * g.batch;
  const bool short_off = knob(KN_GEMV_SHORT) == 0;
  const int short16 = knob(KN_GEMV_K16);
  const int nsm = hps_num_sms();
  if (g.K <= 128 && !short_off) {  // 8 lanes per row: 32 rows per 256-thread block
    dim3 grid((g.M + 31) / 32, g.batch < 65535 ? g.batch : 65535);
    zgemv_short_kernel<NMAX, 8><<<grid, 256, 0, st>>>(g);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
    return;
  }
  if (g.K <= short16 && !short_off && rows >= nsm * 64) {  // 16 lanes per row (the leaf Y s, K = n_i)
    dim3 grid((g.M + 15) / 16, g.batch < 65535 ? g.batch : 65535);
    zgemv_short_kernel<NMAX, 16><<<grid, 256, 0, st>>>(g);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
    return;
  }
  int ks = 1;
  while (ks < 8 && rows * ks < nsm * 48 && g.K / (2 * ks) >= 64) ks *= 2;
  const int rpb = 8 / ks;
  dim3 grid((g.M + rpb - 1) / rpb, g.batch < 65535 ? g.batch : 65535);
  switch (ks) {
    case 1: zgemv_kernel<NMAX, 1><<<grid, 256, 0, st>>>(g); break;
    case 2: zgemv_kernel<NMAX, 2><<<grid, 256, 0, st>>>(g); break;
    case 4: zgemv_kernel<NMAX, 4><<<grid, 256, 0, st>>>(g); break;
    default: zgemv_kernel<NMAX, 8><<<grid, 256, 0, st>>>(g); break;
  }
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

template <typename IT>
__global__ void zcopy_kernel(const ZCopy c) {
  // IT = unsigned for totals below 2^32 (32-bit index arithmetic: a 64-bit division per element
  // costs more than the copy itself)
  const IT total = (IT)c.batch * c.M * c.N;
  for (IT e = blockIdx.x * (IT)blockDim.x + threadIdx.x; e < total; e += (IT)gridDim.x * blockDim.x) {
    const IT t = e / (IT)c.N;
    const int j = (int)(e - t * (IT)c.N);
    const IT bq = t / (IT)c.M;
    const int i = (int)(t - bq * (IT)c.M);
    const int b = (int)bq;
    const int ro = zrow(c.C, c.C.rmap ? c.C.rmap + (int64_t)b * c.C.rmap_bs : nullptr, i);
    const int co = zcol(c.C.cmap, j, c.C.cskip_at, c.C.cskip_len);
    if (ro < 0 || co < 0) continue;
    const int ri = zrow(c.A, c.A.rmap ? c.A.rmap + (int64_t)b * c.A.rmap_bs : nullptr, i);
    const int ci = zcol(c.A.cmap, j, c.A.cskip_at, c.A.cskip_len);
    zt v = make_double2(0.0, 0.0);
    if (ri >= 0 && ci >= 0) v = zmul(c.alpha, c.A.ptr[zboff(c.A, b) + (int64_t)ri * c.A.rs + (int64_t)ci * c.A.cs]);
    c.C.ptr[zboff(c.C, b) + (int64_t)ro * c.C.rs + (int64_t)co * c.C.cs] = v;
  }
}

}  // namespace

// HPS_TRACE=1: time every ZGEMM with events (synchronous) and print its shape to stderr.
static bool trace_on() {
  return knob(KN_TRACE) != 0;
}

void zgemm_impl(const ZGemm& g, cudaStream_t st);

void zgemm(const ZGemm& g, cudaStream_t st) {
  if (!trace_on()) return zgemm_impl(g, st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  zgemm_impl(g, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double fl = 8.0 * g.M * (double)g.N * g.K * g.batch;
  fprintf(stderr, "[zgemm] M=%d N=%d K=%d batch=%d cin=%d maps=%d%d%d%d  %.3f ms  %.2f TF\n", g.M, g.N, g.K, g.batch,
          g.Cin.ptr != nullptr, g.A.rmap != nullptr, g.B.rmap != nullptr, g.B.cmap != nullptr, g.C.rmap != nullptr,
          ms, fl / ms / 1e9);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

// split-K reduction: C(i, j) = alpha * sum_s ws[s](i, j) + diag [i == j], slices summed in order
__global__ void zsplit_reduce_kernel(const ZGemm g) {
  const int64_t mn = (int64_t)g.M * g.N, total = mn * g.batch;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / mn);
    const int64_t r = e - (int64_t)b * mn;
    const int i = (int)(r / g.N), j = (int)(r - (int64_t)i * g.N);
    const int* Crm = g.C.rmap ? g.C.rmap + (int64_t)b * g.C.rmap_bs : nullptr;
    const int ro = zrow(g.C, Crm, i), co = zcol(g.C.cmap, j, g.C.cskip_at, g.C.cskip_len);
    if (ro < 0 || co < 0) continue;
    zt acc = g.ws[e];
    for (int s = 1; s < g.ksplit; ++s) {
      const zt v = g.ws[(int64_t)s * total + e];
      acc.x += v.x;
      acc.y += v.y;
    }
    zt v = zmul(g.alpha, acc);
    if (i == j) {
      v.x += g.diag.x;
      v.y += g.diag.y;
    }
    g.C.ptr[zboff(g.C, b) + (int64_t)ro * g.C.rs + (int64_t)co * g.C.cs] = v;
  }
}

thread_local int g_zgemm_force = -1;  // tile configuration override (tests / tuning)

static bool bcol_applies(const ZGemm& g) {
  return g.B.rs == 1 && g.B.cs > 1 && !g.B.rmap && !g.B.cmap && g.B.cskip_len == 0 && knob(KN_GEMM_BCOL);
}

bool launch_cfg_tile(int cfg, const ZGemm& g, cudaStream_t st);

// A configuration is tile | (split << 8): split-K with `split` slices (2, 4, 8) of the tiled
// kernels (not the GEMV), partial tiles in a stream-ordered workspace and one reduction launch.
bool launch_cfg(int cfg, const ZGemm& g0, cudaStream_t st) {
  const int split = cfg >> 8, tile = cfg & 255;
  if (split <= 1 || tile == 9) return launch_cfg_tile(tile, g0, st);
  ZGemm g = g0;
  g.ksplit = split;
  const size_t bytes = sizeof(zt) * (size_t)split * g.batch * g.M * g.N;
  HPS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&g.ws), bytes, st));
  const bool ok = launch_cfg_tile(tile, g, st);
  if (ok) {
    const int64_t total = (int64_t)g.batch * g.M * g.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * hps_num_sms());
    zsplit_reduce_kernel<<<blocks, 256, 0, st>>>(g);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
  HPS_CUDA_CHECK(cudaFreeAsync(g.ws, st));
  return ok;
}

bool launch_cfg_tile(int cfg, const ZGemm& g, cudaStream_t st) {
  switch (cfg) {
    case 0: launch<64, 8, 16, 8>(g, st); return true;
    case 1: bcol_applies(g) ? launch<16, 16, 8, 8, true>(g, st) : launch<16, 16, 8, 8>(g, st); return true;
    case 2: bcol_applies(g) ? launch<32, 32, 16, 16, true>(g, st) : launch<32, 32, 16, 16>(g, st); return true;
    case 3: launch<64, 64, 32, 32>(g, st); return true;
    case 4: launch<64, 64, 32, 16>(g, st); return true;
    case 5: launch<64, 32, 32, 16>(g, st); return true;
    case 6: launch<32, 64, 16, 32>(g, st); return true;
    case 7: launch<128, 64, 32, 32>(g, st); return true;
    case 8: launch<64, 64, 16, 32>(g, st); return true;
    case 10: bcol_applies(g) ? launch<64, 16, 16, 16, true>(g, st) : launch<64, 16, 16, 16>(g, st); return true;
    case 11: bcol_applies(g) ? launch<128, 16, 32, 16, true>(g, st) : launch<128, 16, 32, 16>(g, st); return true;
    case 12: bcol_applies(g) ? launch<64, 16, 32, 8, true>(g, st) : launch<64, 16, 32, 8>(g, st); return true;
    case 13: bcol_applies(g) ? launch<32, 16, 16, 16, true>(g, st) : launch<32, 16, 16, 16>(g, st); return true;
    case 9: {
      if (g.N == 1) launch_gemv<1>(g, st);
      else if (g.N <= 4) launch_gemv<4>(g, st);
      else return false;
      return true;
    }
    default: return false;
  }
}

void zgemm_impl(const ZGemm& g0, cudaStream_t st) {
  if (g0.M <= 0 || g0.N <= 0 || g0.batch <= 0) return;
  ZGemm g = g0;
  g.group_m = std::max(1, knob(KN_GEMM_GROUP));
  const double mn = (double)g.M * g.N, bt = (double)g.batch;
  // a forced configuration (tests / tuning), else the planned one of this shape (zgemm_plan_shape)
  int force = g_zgemm_force;
  if (force == -1) {
    const int lay = (g.B.rs == 1 && g.B.cs > 1 && !g.B.rmap && !g.B.cmap ? 1 : 0) | (g.C.rs == 1 && g.C.cs > 1 ? 2 : 0);
    const int pc = zgemm_plan_lookup(g.M, g.N, g.K, g.batch, g.Cin.ptr != nullptr, lay);
    if (pc >= 0) force = pc;
  }
  // N <= 4 runs the GEMV kernel: bound by HBM (the A operand is read once), its own class
  const bool gemv = (force < 0 && g.N <= 4) || force == 9;
  ProfScope ps(gemv ? K_ZGEMV : K_ZGEMM, 8.0 * mn * g.K * bt,
               16.0 * bt * ((double)g.M * g.K + (double)g.K * g.N + mn * (g.Cin.ptr ? 2.0 : 1.0)), st);
  // opt-in: the big products as integer-slice products on the INT8 tensor path (off by default)
  if (!gemv && g_zgemm_force == -1 && knob(KN_GEMM_SLICES) > 0 && zgemm_slices(g, st)) return;
  if (force >= 0 && launch_cfg(force, g, st)) return;
  if (g.N <= 4 && force != -2) {
    if (g.N == 1)
      launch_gemv<1>(g, st);
    else
      launch_gemv<4>(g, st);
    return;
  }
  // Tile choice from the sweep in profiles/r01_gemm_tune.txt: 32x32 tiles (5 CTAs / SM) win
  // for the short-K and Cin-heavy shapes of the merges and the Gauss-Jordan updates; 64x32 tiles
  // win once K is long enough to amortise the tile loads.
  const int64_t tiles32 = (int64_t)((g.M + 31) / 32) * ((g.N + 31) / 32) * g.batch;
  const bool small_k16 = knob(KN_GEMM_SMALLK) != 0;
  const int nsm = hps_num_sms();
  // column-major B without maps (s in the ABI layout): the k-fastest B loader
  const bool bcol = bcol_applies(g);
  if (g.N <= 8)
    launch<64, 8, 16, 8>(g, st);
  else if (g.N <= 16 && g.M > 16 && g.K >= 1024 && (int64_t)((g.M + 63) / 64) * g.batch < nsm)
    launch<16, 16, 8, 8>(g, st);    // long-K products of the top levels' solve: more, smaller CTAs
  else if (g.N <= 16 && g.M > 16 && g.M <= 48)
    launch<32, 16, 16, 16>(g, st);  // the low levels' solve products (n3 = 28, 42): less padding
  else if (g.N <= 16 && g.M > 16)
    bcol ? launch<64, 16, 16, 16, true>(g, st) : launch<64, 16, 16, 16>(g, st);  // 16 RHS: no half-empty tiles
  else if (g.M <= 16 || (small_k16 && g.K <= 32 && tiles32 < 2 * nsm))
    launch<16, 16, 8, 8>(g, st);  // short K on a grid of few 32x32 tiles: more, smaller CTAs
  else if (g.K >= 1024 && tiles32 < nsm)
    launch<16, 16, 8, 8>(g, st);  // long K on less than one wave of 32x32 tiles (the top levels' solve
                                  // at 64 RHS: 1.8x faster, profiles/r02 plan tables)
  else if (g.K >= 512)
    launch<64, 32, 32, 16>(g, st);
  else
    bcol ? launch<32, 32, 16, 16, true>(g, st) : launch<32, 32, 16, 16>(g, st);
}

// Several independent copies in one launch (blockIdx.y selects the copy): the merge gathers are a
// few microseconds each and launch-latency bound.
struct ZCopyList {
  ZCopy c[6];
};
template <typename IT>
__global__ void zcopy_multi_kernel(const ZCopyList L) {
  const ZCopy& c = L.c[blockIdx.y];
  const IT total = (IT)c.batch * c.M * c.N;
  for (IT e = blockIdx.x * (IT)blockDim.x + threadIdx.x; e < total; e += (IT)gridDim.x * blockDim.x) {
    const IT t = e / (IT)c.N;
    const int j = (int)(e - t * (IT)c.N);
    const IT bq = t / (IT)c.M;
    const int i = (int)(t - bq * (IT)c.M);
    const int b = (int)bq;
    const int ro = zrow(c.C, c.C.rmap ? c.C.rmap + (int64_t)b * c.C.rmap_bs : nullptr, i);
    const int co = zcol(c.C.cmap, j, c.C.cskip_at, c.C.cskip_len);
    if (ro < 0 || co < 0) continue;
    const int ri = zrow(c.A, c.A.rmap ? c.A.rmap + (int64_t)b * c.A.rmap_bs : nullptr, i);
    const int ci = zcol(c.A.cmap, j, c.A.cskip_at, c.A.cskip_len);
    zt v = make_double2(0.0, 0.0);
    if (ri >= 0 && ci >= 0) v = zmul(c.alpha, c.A.ptr[zboff(c.A, b) + (int64_t)ri * c.A.rs + (int64_t)ci * c.A.cs]);
    c.C.ptr[zboff(c.C, b) + (int64_t)ro * c.C.rs + (int64_t)co * c.C.cs] = v;
  }
}

void zcopy_multi(const ZCopy* cs, int n, cudaStream_t st) {
  std::vector<const ZCopy*> live;
  for (int k = 0; k < n; ++k)
    if ((int64_t)cs[k].batch * cs[k].M * cs[k].N > 0) live.push_back(&cs[k]);
  for (size_t g0 = 0; g0 < live.size(); g0 += 6) {
    const int m = (int)std::min<size_t>(6, live.size() - g0);
    ZCopyList L;
    int64_t maxt = 0, bytes = 0;
    for (int u = 0; u < m; ++u) {
      L.c[u] = *live[g0 + u];
      const int64_t total = (int64_t)L.c[u].batch * L.c[u].M * L.c[u].N;
      maxt = std::max(maxt, total);
      bytes += 32 * total;
    }
    ProfScope ps(K_LAYOUT, 0.0, (double)bytes, st);
    const int blocks = (int)std::min<int64_t>((maxt + 255) / 256, hps_num_sms() * 32 / m + 1);
    if (maxt < ((int64_t)1 << 32))
      zcopy_multi_kernel<unsigned><<<dim3(blocks, m), 256, 0, st>>>(L);
    else
      zcopy_multi_kernel<uint64_t><<<dim3(blocks, m), 256, 0, st>>>(L);
    HPS_CUDA_CHECK(cudaGetLastError());
    count_launch();
  }
}

void zcopy(const ZCopy& c, cudaStream_t st) {
  const int64_t total = (int64_t)c.batch * c.M * c.N;
  if (total <= 0) return;
  ProfScope ps(K_LAYOUT, 0.0, 32.0 * total, st);
  int blocks = (int)((total + 255) / 256);
  if (blocks > hps_num_sms() * 32) blocks = hps_num_sms() * 32;
  if (total < ((int64_t)1 << 32))
    zcopy_kernel<unsigned><<<blocks, 256, 0, st>>>(c);
  else
    zcopy_kernel<uint64_t><<<blocks, 256, 0, st>>>(c);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

// ---------------------------------------------------------------------------
// Representative-action plan of the GEMM tile configuration (Table 1's
// upward / downward matvec rows): the paper times each level's representative action for every
// thread split once per machine and keeps the fastest; here the "split" of a batched product is
// its tile configuration (CTA granularity), timed on synthetic operands of the same shape (a
// sample of the batch covering several waves) and recorded per (M, N, K, batch, Cin) for the
// rest of the process.  Shapes without an entry use the fixed rules of zgemm_impl.
// ---------------------------------------------------------------------------
namespace {
std::mutex g_plan_mu;
std::map<std::tuple<int, int, int, int, int, int>, int> g_plan;
std::atomic<int> g_plan_n{0};

__global__ void zfill_kernel(zt* p, int64_t n, uint64_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = ((uint64_t)e + seed) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    p[e] = make_double2((double)(h >> 11) * 1.1102230246251565e-16 - 0.5,
                        (double)((h * 0x94D049BB133111EBull) >> 11) * 1.1102230246251565e-16 - 0.5);
  }
}
}  // namespace

int zgemm_plan_lookup(int M, int N, int K, int batch, bool cin, int lay) {
  if (g_plan_n.load(std::memory_order_relaxed) == 0) return -1;
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plan.find(std::make_tuple(M, N, K, batch, (int)cin, lay));
  return it == g_plan.end() ? -1 : it->second;
}

void zgemm_plan_set(int M, int N, int K, int batch, bool cin, int lay, int cfg) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  const auto key = std::make_tuple(M, N, K, batch, (int)cin, lay);
  if (cfg < 0) g_plan.erase(key);
  else g_plan[key] = cfg;
  g_plan_n.store((int)g_plan.size());
}

void zgemm_plan_clear() {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plan.clear();
  g_plan_n.store(0);
}

int zgemm_candidates(int N, int* out) {
  // cfg 3 (64 x 64, 32 x 32 warps) only in the 3M form: its 96 accumulators spill a little, yet
  // it beats the 64 x 32 tile there on the top-level products (41.8 vs 40.2 TFLOP/s, DESIGN 3.14)
  static const int c4[] = {9, 0, 1}, c16[] = {0, 1, 10, 11, 12, 13}, cbig[] = {2, 5, 4, 6, 1, 13, 3};
  const int* c = N <= 4 ? c4 : N <= 16 ? c16 : cbig;
  const int n = N <= 4 ? 3 : N <= 16 ? 6 : (knob(KN_GEMM_3M) ? 7 : 6);
  for (int i = 0; i < n; ++i) out[i] = c[i];
  return n;
}

// Times every candidate configuration (and the fixed rule, cfg -1) of one shape on a sample of
// the batch; records the fastest in the plan if it beats the rule by more than 3 %.  Writes the
// per-candidate times extrapolated to the full batch (ms, -1 where infeasible) to t_out[0..ncand)
// and the rule's to *t_rule; returns the chosen configuration (-1: the rule).
int zgemm_plan_shape(int M, int N, int K, int batch, bool cin, int lay, double* t_out, double* t_rule, int* cands,
                     int* ncand, cudaStream_t st) {
  int nc = zgemm_candidates(N, cands);
  // split-K candidates (deterministic, launch_cfg) for long-K shapes whose tiles do not fill the GPU:
  // the top levels' merge products at C2 and the top levels' solve products
  {
    const int64_t t16 = (int64_t)((M + 15) / 16) * ((N + 15) / 16) * batch;
    if (K >= 256 && t16 < 4LL * hps_num_sms()) {
      const int tiles[2] = {1, N <= 16 ? 13 : 2};
      for (int sp = 2; sp <= 8; sp *= 2)
        if (K / sp >= 64)
          for (int t : tiles) cands[nc++] = t | (sp << 8);
    }
  }
  *ncand = nc;
  // sample: enough 16 x 16 tiles for ~8 waves of 8 resident CTAs on every SM
  const int64_t t16 = (int64_t)((M + 15) / 16) * ((N + 15) / 16);
  const int64_t want = std::max<int64_t>(1, (8LL * 8 * hps_num_sms() + t16 - 1) / t16);
  const int bs = (int)std::min<int64_t>(batch, want);
  const double scale = (double)batch / bs;
  zt *A, *B, *C, *Ci = nullptr;
  // column-major B / C keep the FULL batch's column stride (s and u in the ABI layout have columns
  // K * batch / M * batch elements apart: 50-270 MB at C3/C4, a different TLB regime from the
  // sample's); only the sampled entries are touched
  const size_t na = (size_t)M * K * bs;
  const size_t nb = (lay & 1) ? (size_t)K * batch * (N - 1) + (size_t)K * bs : (size_t)K * N * bs;
  const size_t nm = (lay & 2) ? (size_t)M * batch * (N - 1) + (size_t)M * bs : (size_t)M * N * bs;
  const size_t ni = (size_t)M * N * bs;
  HPS_CUDA_CHECK(cudaMallocAsync(&A, sizeof(zt) * std::max<size_t>(na, 1), st));
  HPS_CUDA_CHECK(cudaMallocAsync(&B, sizeof(zt) * std::max<size_t>(nb, 1), st));
  HPS_CUDA_CHECK(cudaMallocAsync(&C, sizeof(zt) * nm, st));
  if (cin) HPS_CUDA_CHECK(cudaMallocAsync(&Ci, sizeof(zt) * ni, st));
  zfill_kernel<<<592, 256, 0, st>>>(A, (int64_t)na, 1);
  zfill_kernel<<<592, 256, 0, st>>>(B, (int64_t)nb, 2);
  if (cin) zfill_kernel<<<592, 256, 0, st>>>(Ci, (int64_t)ni, 3);
  ZGemm g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = bs;
  g.A.ptr = A;
  g.A.rs = K;
  g.A.bs = (int64_t)M * K;
  g.B.ptr = B;
  g.B.rs = N;
  g.B.bs = (int64_t)K * N;
  if (lay & 1) {  // column-major B as s in the ABI layout [RHS][box][K]
    g.B.rs = 1;
    g.B.cs = (int64_t)K * batch;
    g.B.bs = K;
  }
  if (cin) {
    g.Cin.ptr = Ci;
    g.Cin.rs = N;
    g.Cin.bs = (int64_t)M * N;
    g.beta = make_double2(1.0, 0.0);
  }
  g.C.ptr = C;
  g.C.rs = N;
  g.C.bs = (int64_t)M * N;
  if (lay & 2) {  // column-major C as u in the ABI layout [RHS][box][M]
    g.C.rs = 1;
    g.C.cs = (int64_t)M * batch;
    g.C.bs = M;
  }
  cudaEvent_t e0, e1;
  HPS_CUDA_CHECK(cudaEventCreate(&e0));
  HPS_CUDA_CHECK(cudaEventCreate(&e1));
  auto time_cfg = [&](int cfg) {
    g_zgemm_force = cfg < 0 ? -3 : cfg;  // -3: the fixed rule, ignoring the plan
    double best = 1e30;
    int reps = 4;
    for (int r = 0; r < reps; ++r) {  // first run warms up; products above 30 ms are timed once
      HPS_CUDA_CHECK(cudaEventRecord(e0, st));
      zgemm_impl(g, st);
      HPS_CUDA_CHECK(cudaEventRecord(e1, st));
      HPS_CUDA_CHECK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) best = std::min(best, (double)ms);
      else if (ms > 30.0f) reps = 2;
    }
    g_zgemm_force = -1;
    return best * scale;
  };
  *t_rule = time_cfg(-1);
  int bi = -1;
  double bt = *t_rule;
  for (int i = 0; i < nc; ++i) {
    if (cands[i] == 9 && N > 4) {
      t_out[i] = -1;
      continue;
    }
    t_out[i] = time_cfg(cands[i]);
    if (t_out[i] < bt) {
      bt = t_out[i];
      bi = i;
    }
  }
  const int chosen = (bi >= 0 && bt < 0.97 * *t_rule) ? cands[bi] : -1;
  zgemm_plan_set(M, N, K, batch, cin, lay, chosen);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(A, st);
  cudaFreeAsync(B, st);
  cudaFreeAsync(C, st);
  if (Ci) cudaFreeAsync(Ci, st);
  HPS_CUDA_CHECK(cudaStreamSynchronize(st));
  return chosen;
}

// ---------------------------------------------------------------------------
// Live FP64 tensor peak (hps_fp64_peak): every warp of 8 per CTA, 8 CTAs per SM runs 8
// independent m8n8k4 DMMA chains -- the roofline denominator measured in the same process and
// at the same clocks as the kernels it is compared with (tools/fp64_peaks.cu is the standalone form).
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters, double a0, double b0) {
  double d[8][2];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    d[c][0] = 0;
    d[c][1] = threadIdx.x;
  }
  const double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}
}  // namespace

double fp64_dmma_peak_tflops(cudaStream_t st) {
  const int nsm = hps_num_sms(), blocks = nsm * 8, threads = 256, iters = 1 << 14;
  double* out;
  HPS_CUDA_CHECK(cudaMallocAsync(&out, sizeof(double) * threads, st));
  cudaEvent_t e0, e1;
  HPS_CUDA_CHECK(cudaEventCreate(&e0));
  HPS_CUDA_CHECK(cudaEventCreate(&e1));
  dmma_peak_kernel<<<blocks, threads, 0, st>>>(out, 256, 1.0, 1e-7);  // warm-up (clocks up)
  double best = 0;
  for (int r = 0; r < 3; ++r) {
    HPS_CUDA_CHECK(cudaEventRecord(e0, st));
    dmma_peak_kernel<<<blocks, threads, 0, st>>>(out, iters, 1.0, 1e-7);
    HPS_CUDA_CHECK(cudaEventRecord(e1, st));
    HPS_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (threads / 32) * blocks;
    best = std::max(best, fl / ms / 1e9);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  HPS_CUDA_CHECK(cudaStreamSynchronize(st));
  return best;
}
