// hps_internal.cuh — shared declarations of libhps.so (product path; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges are no-ops unless a tool (nsys, ncu) injects

typedef double2 zt;  // complex128, interleaved (re, im)

// ---------------------------------------------------------------------------
// Errors
// ---------------------------------------------------------------------------
struct HpsError {
  int code;
  std::string msg;
};
void hps_set_error(const std::string& msg);

// ---------------------------------------------------------------------------
// Debug / tuning knobs (hps_debug_set in hps.h).  Process-wide, set only through the explicit
// debug ABI — the library reads no environment variables.  Fault-injection knobs (*_FORCE_*,
// *_PIVOT) exist for the tests of the fallback paths; their defaults are the product behaviour.
// ---------------------------------------------------------------------------
enum HpsKnob {
  KN_DEBUG_ALLOC = 0,  // print large-allocation timings to stderr
  KN_BIG_CACHE,        // 1: cache large blocks across handles (hps_release_cache)
  KN_SIDE,             // 1: side stream for the build's independent products (DESIGN 3.11)
  KN_SIDE_SOLVE,       // 1: side stream in the solve
  KN_NAT_MIN,          // natural-order W^{-1} for NAT_MIN <= n3 <= NAT_MAX (DESIGN 3.10)
  KN_NAT_MAX,
  KN_NAT_FORCE_FAIL,   // test: every natural-order W^{-1} reports a failed pivot check
  KN_DGJ_PIVOT,        // test: real leaf eliminations pivot from the start
  KN_DGJ_FORCE_BAD,    // test: the natural-order real leaf elimination fails its first check
  KN_DGJ_RPT,          // rows per thread of the real leaf Gauss-Jordan (2 or 4)
  KN_LR_TRACE,         // print the real-leaf CTA-0 timeline
  KN_GEMV_SHORT,       // 1: 8/16-lane GEMV rows for short K
  KN_GEMV_K16,         // largest K of the 16-lane GEMV
  KN_TRACE,            // time and print every ZGEMM / inverse (synchronous)
  KN_GEMM_SMALLK,      // 1: 16x16 tiles for short-K GEMMs on small grids
  KN_GJ,               // kernel family of the batched inverse: 0 library, 1 fused, 2 blocked, 3 ws
  KN_SEQ_PIVOT,        // test: the complex leaf Schur inverse pivots from the start
  KN_NAT_W,            // natural-order panel width (16 or 32)
  KN_NAT_LPR,          // natural-order update lanes per row
  KN_NATC,             // 1: cluster panel for the natural-order inverse
  KN_NATB,             // 1: blocked natural-order panel (DESIGN 3.10)
  KN_NAT_PIVOT_REL,    // natural-order W^{-1}: pivot accepted if |p|^2 >= REL/1e4 * |W_kk|^2
  KN_NAT_BB_MIN,       // natural-order W^{-1} with 64-wide block steps (D^{-1} kernel + GEMMs) for n >= this
  KN_LEAF_PANEL,       // complex leaf Schur inverse, natural order: 0 step-by-step panels, 1 block form
  KN_GEMM_BCOL,        // 1: k-fastest B loader for column-major B (s in the ABI layout)
  KN_GEMM_GROUP,       // GEMM tile order: 1 row-major, G > 1 grouped by G row blocks (L2 reuse)
  KN_LEAF_INPLACE,     // 1: natural-order complex leaf inverse in the store's Y_i block (no Y_i copy)
  KN_SEQ_FORCE_BAD,    // test: the natural-order complex leaf inverse fails its check at step 100
  KN_RHS_CHUNK,        // right-hand sides per solve chunk (0: as many as fit in 40 % of free memory)
  KN_DGJ_NT,           // threads per CTA of the real leaf Gauss-Jordan: 512 (one leaf per SM) or 256 (two)
  KN_MERGE_SMALL,      // 1: levels with n3 <= 28 merged by one CTA per merge (merge_small.cu)
  KN_GEMM_3M,          // 1: tiled ZGEMM by three real products per complex MAC (3M form, DESIGN 3.14)
  KN_NAT_LOOKAHEAD,    // 1: block-step W^{-1} with lookahead (next block's D^{-1} beside the update)
  KN_SOLVE_GRAPH,      // 1: repeated identical solves replay a CUDA graph (hps_solve)
  KN_GEMM_SLICES,      // s > 0: big products as s 7-bit integer slices on the INT8 tensor path (zgemm_slices.cu)
  KN_GEMM_SLICES_MIN,  // smallest M, N and K of a product that takes the integer-slice form
  KN_COUNT
};
int knob(HpsKnob k);
int hps_num_sms();  // multiprocessors of the current device (cached per device)

#define HPS_CUDA_CHECK(x)                                                                     \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      throw HpsError{-4, std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +      \
                             __FILE__ + ":" + std::to_string(__LINE__)};                       \
  } while (0)

// ---------------------------------------------------------------------------
// Batched complex GEMM on FP64 tensor cores (DMMA m8n8k4), zgemm.cu
//   C[b](i, j) = alpha * sum_k A[b](i, k) B[b](k, j) + beta * Cin[b](i, j) + (i == j) * diag
// Operand element (i, k) of batch b lives at ptr + b*bs + R(i)*rs + Cc(k)*cs where R / Cc are
// the optional int maps (identity when NULL).  A negative map entry means "zero" for loads and
// "skip" for stores.  Complex products are four real DMMAs (re/im sub-GEMMs).
// ---------------------------------------------------------------------------
// Without a column map, column j may skip a window: j -> j + (j >= cskip_at ? cskip_len : 0)
// (used by the blocked Gauss-Jordan update, which touches every column but the panel).
// rmap_bs: batch stride of the row map (0 = one map shared by the whole batch).
// bmap: batch map -- batch entry b lives at ptr + bmap[b]*bs (the solve reads s and writes u in
// the ABI's natural leaf order while the leaves are stored in heap order).
struct ZOp {
  const zt* ptr = nullptr;
  int64_t rs = 0, cs = 1, bs = 0;
  const int* rmap = nullptr;
  const int* cmap = nullptr;
  int cskip_at = 0x7fffffff, cskip_len = 0;
  int64_t rmap_bs = 0;
  const int* bmap = nullptr;
  int rskip_at = 0x7fffffff, rskip_len = 0;  // row window skipped like cskip (no row map)
};

struct ZOut {
  zt* ptr = nullptr;
  int64_t rs = 0, cs = 1, bs = 0;
  const int* rmap = nullptr;
  const int* cmap = nullptr;
  int cskip_at = 0x7fffffff, cskip_len = 0;
  int64_t rmap_bs = 0;
  const int* bmap = nullptr;
  int rskip_at = 0x7fffffff, rskip_len = 0;
};

template <class T>
__device__ __forceinline__ int64_t zboff(const T& o, int b) {
  return (int64_t)(o.bmap ? o.bmap[b] : b) * o.bs;
}

__device__ __forceinline__ int zcol(const int* cmap, int j, int skip_at, int skip_len) {
  return cmap ? cmap[j] : j + (j >= skip_at ? skip_len : 0);
}
// row i of an operand: its row map, else i with the row window [rskip_at, rskip_at + rskip_len) skipped
template <class T>
__device__ __forceinline__ int zrow(const T& o, const int* rm, int i) {
  return rm ? rm[i] : i + (i >= o.rskip_at ? o.rskip_len : 0);
}

struct ZGemm {
  int M = 0, N = 0, K = 0, batch = 1;
  int group_m = 1;  // tile order: 1 row-major, > 1 grouped by group_m row blocks (set by zgemm from the knob)
  ZOp A, B, Cin;  // Cin.ptr == nullptr => beta term omitted
  ZOut C;
  zt alpha = {1.0, 0.0};
  zt beta = {0.0, 0.0};
  zt diag = {0.0, 0.0};
  // split-K (set by zgemm from the plan): ksplit slices of K, each CTA slice writes its raw partial
  // tile to ws[slice][batch][M][N]; a second kernel sums the slices in slice order (deterministic)
  int ksplit = 1;
  zt* ws = nullptr;
};

void zgemm(const ZGemm& g, cudaStream_t st);
// integer-slice form of one product (zgemm_slices.cu); false: not eligible / unavailable, nothing written
bool zgemm_slices(const ZGemm& g, cudaStream_t st);

// Planned tile configurations of batched products (zgemm.cu, representative-action planner of the
// solve's matrix products): lookup (-1: none), set (cfg -1 removes), clear, candidates for N,
// and timing of one shape (records the fastest configuration if it beats the fixed rule by 3 %).
// lay: operand layouts of the shape (bit 0: column-major B, s in the ABI layout; bit 1: column-major C, u)
int zgemm_plan_lookup(int M, int N, int K, int batch, bool cin, int lay);
void zgemm_plan_set(int M, int N, int K, int batch, bool cin, int lay, int cfg);
void zgemm_plan_clear();
int zgemm_candidates(int N, int* out);
int zgemm_plan_shape(int M, int N, int K, int batch, bool cin, int lay, double* t_out, double* t_rule, int* cands,
                     int* ncand, cudaStream_t st);
double fp64_dmma_peak_tflops(cudaStream_t st);  // live DMMA m8n8k4 throughput of this device

// Batched 2-D gather/scale copy: C[b](i, j) = alpha * A[b](i, j) (+ beta * Cin), maps as above.
struct ZCopy {
  int M = 0, N = 0, batch = 1;
  ZOp A;
  ZOut C;
  zt alpha = {1.0, 0.0};
};
void zcopy(const ZCopy& c, cudaStream_t st);
void zcopy_multi(const ZCopy* cs, int n, cudaStream_t st);  // independent copies, one launch per 6

// ---------------------------------------------------------------------------
// Batched explicit inverse by Gauss-Jordan with partial pivoting, zgj.cu
//   A: batch of n x n row-major matrices (lda, stride bs) — destroyed.
//   out: batch of n x n row-major (ldo, stride obs) receives A^{-1}.
//   ws: workspace from zgj_workspace_bytes.  info: device int, set to 1 + batch index of the
//   first matrix with an exactly zero pivot (0 = success).
// ---------------------------------------------------------------------------
size_t zgj_workspace_bytes(int n, int batch);
void zgj_invert(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch,
                void* ws, int* info, cudaStream_t st, int64_t* launches);

// Natural-order blocked inverse of the merge matrices W (n <= 512); *flag (device
// int) is set to 1 if a pivot failed its check (A destroyed, out invalid: redo with zgj_invert).
void zgj_invert_natural(zt* A, int64_t lda, int64_t bs, zt* out, int64_t ldo, int64_t obs, int n, int batch,
                        void* ws, int* flag, cudaStream_t st);
size_t zgj_natural_workspace_bytes(int n, int batch);

// Leaf S^{-1} by the warp-specialised Gauss-Jordan kernel with the fused Schur epilogue: writes
// the whole leaf operator [Psi | Y] (n_t x n_t, stride mstride) and the leaf R (nb x nb, batch
// stride nb*nb) for `batch` leaves; S (n_i x n_i, stride sstride) is destroyed.  K =
// schur_consts.  Returns false without launching when the kernel does not apply.
// With c != nullptr the kernel also assembles S itself (c samples in natural leaf order, leaf_nat
// the heap -> natural map, leaf0 the heap index of batch entry 0); S is then only workspace.
bool zgj_leaf_fused_applies(int p, int batch);

// Leaf operators by real elimination of the interior block (leaf_real.cu): for
// kappa^2 c real, A_ii is real and B^{-1} follows from A_ii^{-1} and the complex n_b x n_b
// Schur complement Sigma = F_b - F_i A_ii^{-1} A_ib.  K = [D2x | D2y] interior blocks (q x q
// each), KR = A_ib / F_i line coefficients, fb = F_b line closures (layouts in leaf_real.cu).
bool leaf_real_fits(int p);
size_t leaf_real_scratch_bytes(int p, int batch);
void leaf_real_c_bounds(const zt* c, int64_t n, double& cmax, double& imax, cudaStream_t st);
void launch_leaf_real(int p, int leaf0, int batch, const int* leaf_nat, const zt* c, double kappa2, const double* K,
                      const double* KR, const zt (&fb)[2][2][2], zt eta, zt* store, int64_t mstride, zt* R,
                      void* work, int* info, cudaStream_t st, bool pivot);
bool zgj_invert_leaf_schur(zt* S, int64_t sstride, zt* store, int64_t mstride, int p, int batch, const zt* K, zt* R,
                           zt eta, int* info, cudaStream_t st, const zt* c = nullptr, const int* leaf_nat = nullptr,
                           int leaf0 = 0, double kappa2 = 0.0);

// Representative-action planner for the batched inverse (zgj.cu): regimes 1 small (shared
// memory), 2 fused (one CTA per matrix, explicit swaps), 3 warp-specialised, 4 blocked with
// implicit-pivoting panels, 5 blocked with explicit-swap panels.
int zgj_plan_inverse(int n, int nbox, double* eps, double* rt, int* theta);
void zgj_plan_set(int n, int nbox, int regime);
void zgj_plan_clear();
int zgj_regime_of(int n, int nbox);
void zgj_force_regime(int r);  // this thread; 0 = none

// Debug timeline of the warp-specialised Gauss-Jordan kernel (hps_debug_ws_trace).
void zgj_ws_trace(int on, long long* out);

// One CTA per merge for the lowest merge levels (merge_small.cu): gathers, W, W^{-1}, Phi^a,
// Phi^b and R^tau of a level in one launch, same outputs and layouts as build_merge.
struct MergeSmallArgs {
  const zt* R = nullptr;  // children's R: [2 np][nbc][nbc] (alpha = 2b, beta = 2b + 1)
  int nbc = 0, n1 = 0, n2 = 0, n3 = 0, ntau = 0;
  const int *I1a = nullptr, *I2b = nullptr, *I3a = nullptr, *I3b = nullptr, *pp = nullptr;
  zt *R33a = nullptr, *R33b = nullptr, *R13a = nullptr, *R23b = nullptr, *Winv = nullptr, *PhiA = nullptr,
     *PhiB = nullptr;
  zt* Rtau = nullptr;  // [np][ntau][ntau] canonical, or nullptr (root without keep_root_R)
  int* info = nullptr;  // set to 1 on an exactly singular W
};
bool merge_small_applies(int n3, int n1, int n2);
size_t merge_small_smem(int n3, int n1, int n2);
void launch_merge_small(const MergeSmallArgs& a, int np, cudaStream_t st);

// Launch counter used for the gpu_launches report.
extern thread_local int64_t* g_launch_counter;
inline void count_launch(int k = 1) {
  if (g_launch_counter) *g_launch_counter += k;
}

// ---------------------------------------------------------------------------
// Per-kernel-class accounting (hps_kernel_stats): launches, algorithmic FLOPs / bytes, and —
// when profiling is on — device time from CUDA events recorded on the launching stream.
// ---------------------------------------------------------------------------
enum KClass { K_ZGEMM = 0, K_GJ_PANEL, K_GJ_SMALL, K_GJ_AUX, K_LEAF_ASM, K_LAYOUT, K_GJ_FUSED, K_LEAF_GJ, K_ZGEMV, K_NCLASS };

struct KStats {
  int64_t launches[K_NCLASS] = {};
  double flops[K_NCLASS] = {};
  double bytes[K_NCLASS] = {};
  double ms[K_NCLASS] = {};
};

struct Prof;
extern thread_local Prof* g_prof;
void prof_begin(int cls, double flops, double bytes, cudaStream_t st);
bool prof_timing_active();  // per-launch event timing on for this thread (side streams stay off)
void prof_end(cudaStream_t st);

struct ProfScope {
  cudaStream_t st;
  ProfScope(int cls, double flops, double bytes, cudaStream_t s) : st(s) { prof_begin(cls, flops, bytes, s); }
  ~ProfScope() { prof_end(st); }
};

// NVTX range for the duration of a scope (build / solve phases and merge levels; visible in
// ncu --nvtx and nsys timelines, free when no tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  template <class... A>
  NvtxRange(const char* fmt, A... a) {
    char buf[96];
    snprintf(buf, sizeof(buf), fmt, a...);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
