/* hps.h — C-ABI of libhps.so: the B200-native HPS direct solver with
 * impedance-to-impedance (ItI) operators for the variable-coefficient
 * Helmholtz impedance problem (arXiv:1812.07167).
 *
 *   -Laplace(u) - kappa^2 c(x) u = s(x)  in the rectangle Omega
 *   du/dnu + i eta u             = t(x)  on its boundary            (eq. 1)
 *
 * hps_build is the precomputation stage (Algorithm 1): the
 * batched leaf build and the level-by-level merge tree
 * (PAPER.md:472-625).  hps_solve is the solve stage (Algorithm 2,
 * PAPER.md:670-710): upward body-load sweep, downward impedance sweep.
 * Every step runs in this library's own sm_100a CUDA kernels (no cuBLAS /
 * cuSOLVER), in complex128.
 *
 * Conventions:
 *  - Leaf discretisation: p x p Chebyshev-Lobatto tensor grid, corners dropped
 *    (PAPER.md:300-325).  q = p - 2 boundary nodes per leaf edge.
 *  - Node (ix, iy) of a leaf's tensor grid has index iy*p + ix (x fastest),
 *    x_k = x0 + (1 - cos(k pi/(p-1))) h/2.
 *  - Boundary order of every box: [S, E, N, W], each edge by increasing
 *    coordinate (PAPER.md:321 fixes [s, e, n, w]; within-edge order is ours).
 *  - Leaf natural order: leaf (ix, iy) has index iy*nx + ix.
 *  - Complex numbers are interleaved (re, im) doubles (== cuDoubleComplex ==
 *    std::complex<double> == numpy complex128).
 *  - Matrices returned by the export calls are row-major.
 *
 * Ownership: the handle owns all device memory for the stored operators.
 * Input pointers are borrowed for the duration of the call; they may be host
 * or device (CUDA-visible) memory — the library asks the driver which.
 * Output buffers are caller-allocated, host or device.
 * Ordering: without hps_opts.stream the library works on a non-blocking stream
 * of its own that waits for NO other stream: device inputs must be complete
 * when a call is made (the Python layer synchronises torch's current stream
 * first).  With hps_opts.stream, everything is ordered on the caller's stream.
 *
 * Errors: every int-returning call returns 0 or a negative HPS_E* code; the
 * message of the last failure on the calling thread is hps_last_error().  No
 * C++ exception crosses the ABI.  On a build error *out is set to NULL; on a
 * solve error the contents of u are unspecified and the handle stays valid.
 * Calls on one handle must not overlap (one call at a time per handle).
 */
#ifndef HPS_H_
#define HPS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_OK 0
#define HPS_EINVAL (-1)    /* invalid argument (message says which) */
#define HPS_ESINGULAR (-2) /* zero pivot while inverting B (leaf) or W (merge); message names the level */
#define HPS_ENOMEM (-3)    /* device allocation failed */
#define HPS_ECUDA (-4)     /* CUDA runtime / launch error */
#define HPS_ENOTKEPT (-5)  /* export of an operator the handle did not keep */
#define HPS_ENCCL (-6)     /* NCCL failure / NCCL not loadable (multi-GPU only) */

#define HPS_NCCL_ID_BYTES 128 /* == sizeof(ncclUniqueId) */

typedef struct {
  double x0, x1, y0, y1; /* the rectangle Omega, x1 > x0, y1 > y0 */
  int32_t nx, ny;        /* leaves per side, powers of two (1 allowed) */
} hps_grid;

typedef struct {
  double re, im;
} hps_c128;

typedef struct hps_handle hps_handle;
typedef struct hps_comm hps_comm; /* communicator of the subtree-sharded build / solve (below) */

typedef struct {
  int32_t keep_root_R;  /* 1: form the root ItI operator R^1 (Algorithm 1, tau = 1).  Algorithm 2
                           never uses it; 0 skips the two root GEMMs (default 1). */
  int32_t keep_all_R;   /* 1: keep every box's R for hps_export_R (debug / parity; default 0) */
  int32_t device;       /* CUDA device ordinal (default: current device) */
  int32_t leaf_chunk;   /* leaves factored per batch (0 = automatic) */
  int32_t profile;      /* bit mask of kernel classes (see hps_kernel_stats) to time with CUDA
                           events on the library stream; -1 = all; 0: counters only (default) */
  int32_t leaf_mode;    /* 0 (default): automatic -- mode 3 where it applies (real c samples,
                           p - 2 <= 14 and kappa^2 max Re c < 0.9 pi^2 (1/hx^2 + 1/hy^2), the
                           lowest Dirichlet eigenvalue of a leaf), else B^{-1} through the
                           interior Schur complement with [Psi | Y] and R formed
                           in the epilogue of the inverse kernel;
                           1: Gauss-Jordan on the full n^tau x n^tau matrix B;
                           2: complex interior Schur complement with the separate finish kernel;
                           3: real elimination of the interior block: one REAL
                           inverse of A_ii per leaf plus the complex n_b x n_b complement
                           Sigma = F_b - F_i A_ii^{-1} A_ib (eq. 7 rows reordered); needs real
                           c samples and p - 2 <= 14 (else HPS_EINVAL), no resonance check.
                           Other values: HPS_EINVAL */
  int32_t boundary_basis; /* root boundary data t of hps_solve / hps_solve_top sampled at
                           0 (default): the q = p - 2 corner-free Chebyshev-Lobatto nodes of each
                             leaf edge (hps_root_boundary_nodes; the paper's scheme);
                           1: the q = p - 2 Gauss-Legendre nodes of each leaf edge
                             (hps_boundary_nodes_gl, same segment order; SURVEY 8(f) NEXT-2,
                             DESIGN.md 3.9): the library interpolates each segment's degree-(q-1)
                             polynomial to its Chebyshev nodes.
                           2: the Gauss-Legendre EDGE representation (beyond the
                             paper, which only cites it): q GL nodes on EVERY
                             leaf edge, any 2 <= q <= p - 2 (the q argument of hps_build).  Leaf
                             incoming data are interpolated from the q GL nodes to the edge's p - 2
                             Chebyshev nodes (P), outgoing data from the Chebyshev nodes to the GL
                             nodes (Q): R_leaf = Qblk R Pblk, Psi = Psi Pblk, so every merge works
                             on q nodes per leaf edge; t is given at hps_boundary_nodes_glq(g, q),
                             hps_export_R returns the GL-based maps, hps_export_leaf Psi Pblk
                             ((p^2-4) x 4q).  Exact for solutions whose edge traces are polynomials
                             of degree < q.
                           u is always returned at the Chebyshev leaf nodes.  Other values: HPS_EINVAL */
  /* ---- multi-GPU and stream; zero-initialised = single GPU ---- */
  int32_t n_gpus;       /* 1, 2, 4, 8, ... (power of two): SPMD, one process (or virtual rank) per GPU;
                           0 = the communicator's size (1 without one) */
  void* nccl_comm;      /* an ncclComm_t of n_gpus ranks (hps_nccl_comm_init, or the caller's own);
                           the library wraps it (collective: every rank's hps_build must run) */
  void* stream;         /* cudaStream_t to order ALL of the handle's work on; NULL = a stream the
                           library creates.  Device inputs must be complete in this stream's order.
                           hps_build always returns synchronised (it reads pivot flags); with a
                           caller stream and device pointers hps_solve returns WITHOUT waiting
                           (hps_sync waits); host pointers make it synchronous */
  hps_comm* comm;       /* library communicator (hps_comm_wrap_nccl, hps_vcomm_rank); takes
                           precedence over nccl_comm */
} hps_opts;

/* Precomputation stage (Algorithm 1).
 *  Multi-GPU (n_gpus = G > 1, a communicator in opts): SPMD -- every rank calls hps_build with the
 *  SAME g, p, q, kappa, eta and its own c_samples.  The top log2(G) splits of the tree give G
 *  congruent rectangles (hps_subtree_grid(g, log2 G, rank)); rank r builds the leaves and every
 *  merge of its rectangle with no communication, then the top log2(G) levels run with the group
 *  split of SURVEY §8(e): at a level with 2^k merges, the G / 2^k ranks under a box all-gather
 *  the children's ItI maps, form W and W^{-1} (replicated in the group) and each computes a
 *  1 / (G / 2^k) column slice of Phi^alpha, Phi^beta and R^tau (R^tau stays column-distributed
 *  until the next level's all-gather).  With keep_root_R the root R is gathered at the end.
 *  g         : domain and leaf grid (nx, ny powers of two; leaves must be congruent rectangles).
 *  p         : Chebyshev points per leaf side, p >= 4.
 *  q         : boundary nodes per leaf edge; must equal p - 2 (corner-free scheme),
 *              except with opts.boundary_basis = 2 (Gauss-Legendre edges): 2 <= q <= p - 2.
 *  kappa     : wavenumber, kappa >= 0 (PAPER.md:227 has kappa > 0; 0 is allowed).
 *  eta       : impedance parameter, Re(eta) != 0.
 *  c_samples : c(x) at every leaf's p*p tensor nodes, [nx*ny leaves, natural order][p*p]; corner
 *              values are ignored.  Host or device memory; complex (the PDE allows complex c).
 *              Multi-GPU: this rank's rectangle only, [nx*ny/G][p*p] in the rectangle's own
 *              natural order.
 *  opt       : NULL for defaults.
 *  out       : receives the handle (NULL on error). */
int hps_build(const hps_grid* g, int p, int q, double kappa, hps_c128 eta, const hps_c128* c_samples,
              const hps_opts* opt, hps_handle** out);

/* Solve stage (Algorithm 2) for nrhs right-hand sides.
 *  s : body load at interior nodes, [nrhs][nx*ny leaves][q*q] (x fastest); NULL means s = 0 and
 *      the upward pass is skipped.
 *  t : incoming impedance data on the root boundary, [nrhs][2(nx+ny)q] in [S,E,N,W] order.
 *  u : output, [nrhs][nx*ny leaves][p*p-4]; each leaf in [I_b (S,E,N,W); I_i] order
 *      (PAPER.md:321-325).  Nodes on a shared edge appear once per leaf.
 *  Host or device pointers.  Right-hand sides are processed in chunks (each a full upward +
 *  downward sweep) of as many as fit in 40 % of the free device memory (knob rhs_chunk fixes it;
 *  SURVEY hard part 7); host buffers are staged chunk by chunk.  Several chunks make the call
 *  synchronous.  Multi-GPU (collective): s and u are this rank's rectangle
 *  ([nrhs][nx*ny/G][...], local natural order), t is the whole root boundary on every rank. */
int hps_solve(hps_handle* h, int nrhs, const hps_c128* s, const hps_c128* t, hps_c128* u);

/* Wait for the handle's enqueued work (a stream-ordered hps_solve) and finish its timings.
 * Returns 0 or HPS_ECUDA. */
int hps_sync(hps_handle* h);

/* ---- Communicators (multi-GPU) ----------------------------------------------------------
 * NCCL: rank 0 calls hps_nccl_unique_id and sends the HPS_NCCL_ID_BYTES bytes to every rank
 * (the Python layer uses torch.distributed); every rank then calls hps_nccl_comm_init on its own
 * device (ncclCommInitRank) and passes the result as opts.nccl_comm, or wraps it once with
 * hps_comm_wrap_nccl (collective; creates the group split communicators) and passes opts.comm.
 * NCCL is loaded at run time (libnccl.so.2 already in the process, else the loader's path):
 * HPS_ENCCL if it is missing.
 * Virtual ranks (tests, one GPU): hps_vcomm_create(G) makes a group, hps_vcomm_rank(group, r) the
 * communicator of rank r; rank r's calls must run on their own host thread, all on one device.
 * hps_comm_selftest: collective all-gather of rank-stamped data in groups of gs, checked. */
int hps_nccl_unique_id(char* id /* HPS_NCCL_ID_BYTES */);
int hps_nccl_comm_init(int nranks, int rank, const char* id, void** nccl_comm);
int hps_nccl_comm_destroy(void* nccl_comm);
int hps_comm_wrap_nccl(void* nccl_comm, hps_comm** out);
int hps_vcomm_create(int nranks, void** group);
int hps_vcomm_rank(void* group, int rank, hps_comm** out);
int hps_vcomm_destroy(void* group);
int hps_comm_info(const hps_comm* c, int* rank, int* size);
int hps_comm_selftest(hps_comm* c, int gs);
void hps_comm_free(hps_comm* c);

/* Host-only plan of the sharded top levels for rank `rank` of G: for each top depth d = 0 ..
 * log2(G) - 1 (root first) writes 8 ints to info[8 d ...]: group size gs, rank in the group,
 * side (0: under the alpha child, 1: beta), n3, n1, n_tau, first column j0 and width w of this
 * rank's column slice of Phi / R^tau (in [I1, I2] order).  Returns log2(G) or HPS_EINVAL. */
int hps_dist_plan(const hps_grid* g, int p, int G, int rank, int32_t* info, int maxlev);

/* ---- Subtree sharding (multi-GPU) ---------------------------------------
 * The tree's top `depth` levels are split off: rank r builds the subtree of the depth-`depth`
 * box with heap index r (hps_subtree_grid gives its rectangle) with hps_build, the subtree-root
 * ItI operators of all ranks are gathered, and hps_build_top merges them (Algorithm 1 for the
 * boxes above `depth`).  The solve splits the same way: hps_solve_up on every subtree, gather
 * of the subtree-root outgoing data h, hps_solve_top (upward merges above `depth`, then the
 * downward pass from the root data t to the depth-`depth` boxes), hps_solve_down on every
 * subtree.  Layouts: R_sub [2^depth][nb][nb] row-major (heap order), h_sub / t_sub
 * [2^depth][nrhs][nb] with nb = n_b of a depth-`depth` box. */

/* Rectangle and leaf offset (ix0, iy0 in leaves) of the depth-`depth` box with heap index
 * `index` (0 .. 2^depth - 1) of grid g.  Host-only geometry. */
int hps_subtree_grid(const hps_grid* g, int depth, int64_t index, hps_grid* sub, int32_t* leaf_i0,
                     int32_t* leaf_j0);

/* Merge tree above `depth` from the given subtree-root ItI operators (Algorithm 1
 * for the boxes tau < 2^depth).  The handle's R of box 1 is exported by hps_export_R when
 * keep_root_R = 1. */
int hps_build_top(const hps_grid* g, int p, int q, double kappa, hps_c128 eta, int depth, const hps_c128* R_sub,
                  const hps_opts* opt, hps_handle** out);

/* Upward pass of a (sub)tree handle: body load s as for hps_solve (NULL = 0); writes the root's
 * outgoing particular impedance data h_root [nrhs][n_b(root)] (eq. flux_part) and keeps the
 * leaf particular solutions and interface corrections for the matching hps_solve_down. */
int hps_solve_up(hps_handle* h, int nrhs, const hps_c128* s, hps_c128* h_root);

/* Downward pass of a (sub)tree handle from the root incoming data t [nrhs][n_b(root)]; u as in
 * hps_solve.  Uses the state of the preceding hps_solve_up with the same nrhs (else s = 0). */
int hps_solve_down(hps_handle* h, int nrhs, const hps_c128* t, hps_c128* u);

/* Top handle: upward merges from h_sub (NULL = 0), downward pass from the root data t_root
 * [nrhs][n_b(1)] to the depth boxes' incoming data t_sub. */
int hps_solve_top(hps_handle* h, int nrhs, const hps_c128* h_sub, const hps_c128* t_root, hps_c128* t_sub);

/* ItI operator of a box (heap numbering: root 1, children 2*tau (alpha: west / south) and
 * 2*tau + 1 (beta: east / north)).  out: n_b(box)^2, row-major, canonical
 * order.  The root is available when keep_root_R = 1; other boxes need keep_all_R = 1. */
int hps_export_R(const hps_handle* h, int64_t box, hps_c128* out);

/* Leaf operators Psi ((p^2-4) x (4p-8)) and Y ((p^2-4) x (p-2)^2), row-major, of the leaf with
 * natural index `leaf`.  Either output may be NULL.  With boundary_basis 2 Psi
 * is the Gauss-Legendre-edge operator Psi Pblk, (p^2-4) x 4q. */
int hps_export_leaf(const hps_handle* h, int64_t leaf, hps_c128* psi, hps_c128* y);

/* Sizes: n_b of a box (heap id), number of boxes, leaf depth. Returns -1 on a bad id. */
int64_t hps_box_nb(const hps_handle* h, int64_t box);
int64_t hps_num_boxes(const hps_handle* h);

/* Gauss-Legendre root boundary nodes (boundary_basis 1): the q = p - 2 Gauss-Legendre nodes of
 * every leaf-edge segment, canonical order [S, E, N, W], increasing coordinate within an edge;
 * x, y, nx, ny as for hps_root_boundary_nodes (2 (nx + ny) q entries each, host memory). */
int hps_boundary_nodes_gl(const hps_grid* g, int p, double* x, double* y, double* nx, double* ny);
/* The same with q Gauss-Legendre nodes per segment (boundary_basis 2): 2 (nx + ny) q entries each. */
int hps_boundary_nodes_glq(const hps_grid* g, int q, double* x, double* y, double* nx, double* ny);

/* Tensor-node coordinates of every leaf, [nx*ny][p*p] (x fastest), and the root boundary
 * nodes with their outward unit normals, [2(nx+ny)(p-2)] in [S,E,N,W] order.  Host pointers.
 * Pure geometry (no device work); lets callers sample c, s, t. */
int hps_leaf_nodes(const hps_grid* g, int p, double* x, double* y);
int hps_root_boundary_nodes(const hps_grid* g, int p, double* x, double* y, double* nx, double* ny);

/* Device time (ms, CUDA events on the library stream) of the last build / solve, split by phase:
 * which = 0 build total, 1 leaf factor, 2 merges, 3 solve total, 4 upward, 5 downward. */
double hps_last_time_ms(const hps_handle* h, int which);

/* Statistics of the last build/solve for the roofline report: number of kernel launches and
 * algorithmic FLOPs (8 real flops per complex multiply-add). which: 0 build, 1 solve. */
int64_t hps_last_launches(const hps_handle* h, int which);
double hps_last_flops(const hps_handle* h, int which);

/* Per-kernel-class statistics accumulated since the handle was built (or hps_reset_stats):
 * class 0 ZGEMM (DMMA), 1 Gauss-Jordan panel, 2 Gauss-Jordan small (in shared memory),
 * 3 Gauss-Jordan swaps/permutation, 4 leaf assembly, 5 gathers / layout, 6 fused whole-matrix
 * Gauss-Jordan (one CTA per matrix), 7 leaf operators (one CTA per leaf: the complex Schur
 * inverse with the fused epilogue, or the real interior elimination), 8 ZGEMV (products with
 * N <= 4 right-hand sides: HBM-bound, flops and bytes as for class 0).  ms is the sum of
 * CUDA-event durations around each launch (only while profiling is on); flops and bytes are
 * ALGORITHMIC (8 flops per complex multiply-add; operand bytes read + written once). */
int hps_set_profiling(hps_handle* h, int mask);

/* The leaf path hps_build took (leaf_mode numbering: 0 complex Schur fused, 1 full B, 2 complex
 * Schur unfused, 3 real interior elimination); -1 for a top handle; HPS_EINVAL for NULL. */
int hps_leaf_path(const hps_handle* h);
int hps_kernel_stats(const hps_handle* h, int cls, int64_t* launches, double* ms, double* flops, double* bytes);
int hps_reset_stats(hps_handle* h);

/* Batched explicit inverse (the library's Gauss-Jordan kernels with partial pivoting, the same
 * code path that inverts the leaf matrices and W).  A: batch x n x n row-major, out: same
 * shape; host or device pointers; A is not modified.  Returns HPS_ESINGULAR on an exactly
 * zero pivot.  Exposed for kernel-level tests. */
int hps_zinv_batched(int n, int batch, const hps_c128* A, hps_c128* out);

/* As hps_zinv_batched, but runs the inversion `reps` times (each on a fresh device copy of A)
 * and returns the mean device time of the inversion alone (CUDA events) in *ms.  `mode`
 * selects the kernel family (0 = library choice, 1 = whole-matrix fused, 2 = blocked
 * panel + GEMM, 3 = warp-specialised look-ahead, n <= 240; 4-7 = planner regimes 4-7, see
 * hps_plan_inverse) for kernel comparisons.  Exposed for kernel tests and tuning. */
int hps_zinv_timed(int mode, int n, int batch, const hps_c128* A, hps_c128* out, int reps, double* ms);

/* Representative-action planner.
 * hps_rep_actions: host-only.  For the tree of grid g at order p, writes the size n and the box
 * count of every level's representative action (Table 1): entry 0 the leaf
 * interior x interior inverse (n_i, #leaves), entries 1..L the interface inverse W of the merge
 * levels bottom-up (n3, 2^d).  Returns the number of entries (L + 1) or HPS_EINVAL (also when
 * maxlev is too small).
 * hps_plan_inverse: measures on the current device the representative time r of every regime
 * of the batched inverse for `nbox` n x n matrices and records, for later builds in this
 * process, the regime minimising eps = ceil(nbox / theta_o) * r.  Regimes (array index):
 * 1 shared-memory matrix per CTA, 2 one CTA per matrix with explicit swaps, 3 warp-specialised
 * look-ahead CTA per matrix, 4 blocked with implicit-pivoting panels + DMMA GEMM, 5 blocked with
 * explicit-swap panels + DMMA GEMM, 6 blocked with recursive 4-column sub-panels in shared memory
 * (n <= 496), 7 sequential-phase CTA per matrix (n <= 240).  eps, rep_ms (ms), theta_o: caller
 * arrays of length 8;
 * infeasible regimes get -1.  Returns the chosen regime (> 0) or a negative error code.
 * hps_plan_set / hps_plan_clear: set (regime 0 = remove) / forget plan entries (hps_plan_clear also
 * forgets the GEMM tile plan of hps_plan_solve).
 * hps_plan_regime: the regime the library will use for (n, nbox). */
int hps_rep_actions(const hps_grid* g, int p, int maxlev, int* n_out, int* nbox_out);

/* Solve-stage representative actions (Table 1's upward and downward matvec rows, the
 * solve half of the planner).  hps_solve_actions: host-only; writes for
 * every batched matrix product of Algorithm 2 on the tree of g at order p with nrhs right-hand
 * sides 7 ints to out[7 i ...]: level (-1 = leaf level, d = merge depth of the parent boxes),
 * kind (0 leaf u~ = Y s, 1 leaf u = Psi t (+ u~), 2 Upsilon action R33b h3a - h3b and R33a t~a +
 * h3a, 3 W^{-1} (.), 4 Gamma^tau action R13a t~a + h1a (and R23b t~b + h2b), 5 Phi t (+ t~)), M, N
 * (= nrhs), K, batch (boxes of the level), cin (1: the product adds a vector).  Returns the
 * number of actions, or HPS_EINVAL (also when maxn > 0 is too small; maxn = 0 only counts).
 * hps_plan_solve: times every distinct shape on the current device with each candidate tile
 * configuration of the library's GEMM (synthetic operands, a sample of the batch covering several
 * waves, extrapolated to the full batch) and records, for later calls in this process, the
 * fastest one where it beats the fixed rule by more than 3 %.  actions: [maxn][7] as above;
 * chosen[i]: the configuration recorded for action i (-1: the fixed rule stays); t_rule / t_best
 * (ms): the rule's and the chosen configuration's extrapolated times.  Returns the number of
 * actions or a negative error code.  hps_plan_clear forgets these entries too. */
int hps_solve_actions(const hps_grid* g, int p, int nrhs, int maxn, int32_t* out);
/* The build's batched products (Algorithm 1 lines 7-12 per merge level, and
 * the trailing updates of the natural-order W^{-1}), same 7-int layout; kinds
 * 6 R33b R31a, 7 W = I - R33b R33a, 8 Phi^a = W^{-1} X, 9 R^tau rows of I1 (and I2; absent at the
 * root with keep_root_R = 0), 10 Phi^b, 11 W^{-1} block-step update.  hps_plan_build plans them
 * like hps_plan_solve. */
int hps_build_actions(const hps_grid* g, int p, int keep_root_R, int maxn, int32_t* out);
int hps_plan_build(const hps_grid* g, int p, int keep_root_R, int maxn, int32_t* actions, int32_t* chosen,
                   double* t_rule, double* t_best);
int hps_plan_solve(const hps_grid* g, int p, int nrhs, int maxn, int32_t* actions, int32_t* chosen, double* t_rule,
                   double* t_best);
int hps_plan_inverse(int n, int nbox, double* eps, double* rep_ms, int* theta_o);
int hps_plan_set(int n, int nbox, int regime);
int hps_plan_clear(void);
int hps_plan_regime(int n, int nbox);

/* Debug: arm (on = 1) / disarm the clock64 timeline of CTA 0 of the warp-specialised
 * Gauss-Jordan kernel and copy the last one (320 values: the [16][16] clock64 timeline, then 64 of the natural-order panel) to host `out` (may be
 * NULL).  Used by tools/gj_tune.py only. */
int hps_debug_ws_trace(int on, int64_t* out);

/* Batched complex GEMM through the library's DMMA kernel: C = alpha A B + beta Cin for
 * contiguous row-major A [batch][M][K], B [batch][K][N], Cin / C [batch][M][N] (Cin may be
 * NULL).  cfg selects a tile configuration (-1 = the library's choice; tile | (slices << 8) with
 * slices 2, 4 or 8 is the deterministic split-K form of a tiled configuration: per-slice partial
 * tiles in a stream-ordered workspace summed in slice order); the call runs `reps` times after one
 * warm-up and returns the mean device time in *ms.  Exposed for kernel tests and tuning.  An unknown
 * cfg falls back to the library's choice. */
int hps_zgemm_batched(int cfg, int M, int N, int K, int batch, const hps_c128* A, const hps_c128* B,
                      const hps_c128* Cin, hps_c128* C, hps_c128 alpha, hps_c128 beta, int reps, double* ms);

/* Live FP64 tensor-core peak of the current device: 8 independent m8n8k4 DMMA chains per warp, 8
 * CTAs of 8 warps per SM, best of 3 timed launches (~0.1 s).  The roofline denominator of the
 * FP64-bound kernels measured in the same process and at the same clocks (MEASURED_PEAKS.json has no
 * FP64 entry).  Returns 0 or HPS_ECUDA. */
int hps_fp64_peak(double* tflops);

void hps_free(hps_handle* h);

/* Memory policy.  Device memory comes from the device's stream-ordered pool (cudaMallocAsync on
 * the handle's stream).  When the last live handle is freed the pool is trimmed, so the memory is
 * available to other allocators in the process (torch, NCCL) again.
 * hps_set_cache_limit(bytes > 0) OPTS IN to a process-wide cache of blocks >= 256 MB freed by
 * hps_free (leaf and merge operator stores, solve vectors), handed to later handles of the same
 * shapes: a fresh mapping of tens of GB costs ~0.25 s.  At most `bytes` are parked;
 * the cache is emptied before any library allocation is allowed to fail; 0 (default) disables it
 * and frees what it holds.  hps_release_cache returns every cached block to the driver and trims
 * the pool now (synchronises the devices concerned).  hps_cache_bytes: bytes parked now.
 * Return 0 / HPS_EINVAL (negative limit). */
int hps_set_cache_limit(int64_t bytes);
int64_t hps_cache_bytes(void);
int hps_release_cache(void);

/* Debug and tuning knobs (process-wide; the library reads no environment variables).  `name` is
 * one of: debug_alloc, big_cache, side, side_solve, nat_min, nat_max, nat_force_fail, dgj_pivot,
 * dgj_force_bad, dgj_rpt, lr_trace, gemv_short, gemv_k16, trace, gemm_smallk, gj, seq_pivot,
 * nat_w, nat_lpr, natc, natb, nat_pivot_rel, nat_bb_min, leaf_panel, gemm_bcol, gemm_group, leaf_inplace, seq_force_bad, rhs_chunk, dgj_nt, merge_small, gemm_3m, nat_lookahead, solve_graph, gemm_slices, gemm_slices_min (meanings in csrc/hps_internal.cuh).  The *_force_*
 * and *_pivot knobs are FAULT INJECTION for the tests of the pivoted fallback paths: never set
 * them in production.  value -1 restores the default.  Returns 0 or HPS_EINVAL (unknown name). */
int hps_debug_set(const char* name, int value);
int hps_debug_get(const char* name, int* value);
const char* hps_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HPS_H_ */
