// hps_oracle.cpp — CPU ORACLE for the HPS / ItI method of arXiv:1812.07167.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.  The
// product path (paper_1812_07167_b200/, libhps.so) never links, imports or
// calls anything here, and nothing here is shared with it (no headers, no
// helpers, no tables).
//
// What it is: a plain, slow, literal rendering of the paper, in complex128:
//   * Chebyshev grid + spectral differentiation (Trefethen)
//   * corner-free leaf discretisation A, N, F, G, B
//   * leaf operators Psi, Y, R = G Psi, Gamma = G Y        (eqs 7-10)
//     -- B^{-1} by a naive LU with partial pivoting, R and Gamma by EXPLICIT
//        products with G (not the I - 2i eta Psi_b shortcut the GPU uses)
//   * merge, Algorithm 1 lines 5-14 with EXPLICIT Upsilon^a, Upsilon^b and
//     Gamma^tau, Phi^b in the paper's long form
//   * solve, Algorithm 2 with the explicit Upsilon / Gamma^tau
//   * a brute-force global collocation solve (all leaves at once, interface
//     coupling t3^a = -g3^b, g3^a = -t3^b of PAPER.md:538, dense LU) used as
//     an independent check of the merge algebra.
// Index sets are built from GEOMETRIC node keys (which grid line, which leaf
// edge segment, which Chebyshev node) and I1/I2/I3 are found by set
// intersection, literally as PAPER.md:500-510 defines them.
//
// Readings of garbled / silent passages:
//   Q1  N uses geometric outward normals: S -d/dy, E +d/dx, N +d/dy, W -d/dx.
//   Q2  the particular-problem matrix is the same B as eq. (7).
//   Q3  R^tau uses the block-diagonal [R13a 0; 0 R23b], not the
//       dimensionally impossible stacked form of Algorithm 1 line 12.
//   Q4  Lobatto nodes x_k = -cos(k pi/(p-1)) ascending; D closed form; D2 = D*D.
//   Q5  every box's boundary is ordered [S, E, N, W], each edge by increasing
//       coordinate; R^tau is permuted from [I1, I2] into that order.
//   Q6  split rule: split the longer side (in leaves), ties vertical; children
//       alpha = west/south = 2*tau, beta = east/north = 2*tau+1 (root = 1).
//
// Parallelism: OpenMP over independent boxes of one tree level only (the
// paper's theta_i = 1 regime); no BLAS.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

typedef std::complex<double> cplx;
static const cplx I_UNIT(0.0, 1.0);

// ----------------------------------------------------------------------------
// Dense matrices (row-major) and naive linear algebra
// ----------------------------------------------------------------------------
struct Mat {
  int m = 0, n = 0;
  std::vector<cplx> a;
  Mat() {}
  Mat(int m_, int n_) : m(m_), n(n_), a((size_t)m_ * n_, cplx(0, 0)) {}
  cplx& operator()(int i, int j) { return a[(size_t)i * n + j]; }
  const cplx& operator()(int i, int j) const { return a[(size_t)i * n + j]; }
};

static Mat identity(int n) {
  Mat I(n, n);
  for (int i = 0; i < n; ++i) I(i, i) = 1.0;
  return I;
}

// C = A * B, triple loop.  Rows of C are independent: for big products they are spread over
// OpenMP threads (each element still accumulates over k in increasing order, so the result is
// bitwise the same for any thread count; nested inside the per-box loops it runs serially).
static Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.m, B.n);
#pragma omp parallel for schedule(static) if ((double)A.m * A.n * B.n > 4e6)
  for (int i = 0; i < A.m; ++i)
    for (int k = 0; k < A.n; ++k) {
      const cplx aik = A(i, k);
      if (aik == cplx(0, 0)) continue;
      for (int j = 0; j < B.n; ++j) C(i, j) += aik * B(k, j);
    }
  return C;
}

static Mat add(const Mat& A, const Mat& B, double sb = 1.0) {
  Mat C = A;
  for (size_t i = 0; i < C.a.size(); ++i) C.a[i] += sb * B.a[i];
  return C;
}

static Mat neg(const Mat& A) {
  Mat C = A;
  for (auto& v : C.a) v = -v;
  return C;
}

static Mat sub(const Mat& A, const std::vector<int>& rows, const std::vector<int>& cols) {
  Mat S((int)rows.size(), (int)cols.size());
  for (size_t i = 0; i < rows.size(); ++i)
    for (size_t j = 0; j < cols.size(); ++j) S((int)i, (int)j) = A(rows[i], cols[j]);
  return S;
}

// [A | B] side by side
static Mat hcat(const Mat& A, const Mat& B) {
  Mat C(A.m, A.n + B.n);
  for (int i = 0; i < A.m; ++i) {
    for (int j = 0; j < A.n; ++j) C(i, j) = A(i, j);
    for (int j = 0; j < B.n; ++j) C(i, A.n + j) = B(i, j);
  }
  return C;
}

// [A ; B] stacked
static Mat vcat(const Mat& A, const Mat& B) {
  Mat C(A.m + B.m, A.n);
  for (int i = 0; i < A.m; ++i)
    for (int j = 0; j < A.n; ++j) C(i, j) = A(i, j);
  for (int i = 0; i < B.m; ++i)
    for (int j = 0; j < B.n; ++j) C(A.m + i, j) = B(i, j);
  return C;
}

// Textbook LU with partial pivoting, PA = LU (Doolittle, in place).
// Returns 0, or -(k+1) if column k has no nonzero pivot.
static int lu_factor(Mat& A, std::vector<int>& perm) {
  const int n = A.n;
  perm.resize(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int r = k;
    double best = std::abs(A(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > best) { best = std::abs(A(i, k)); r = i; }
    if (best == 0.0) return -(k + 1);
    if (r != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(r, j));
      std::swap(perm[k], perm[r]);
    }
    // rows below the pivot are independent (same per-element operations for any thread count)
#pragma omp parallel for schedule(static) if ((double)(n - k) * (n - k) > 1e5)
    for (int i = k + 1; i < n; ++i) {
      A(i, k) /= A(k, k);
      const cplx l = A(i, k);
      for (int j = k + 1; j < n; ++j) A(i, j) -= l * A(k, j);
    }
  }
  return 0;
}

// Solve A X = Bm given the LU factors of A (forward then back substitution).
// Columns of X are independent: big solves split the columns over OpenMP threads (every element
// sees the same operations in the same order for any thread count).
static Mat lu_solve(const Mat& LU, const std::vector<int>& perm, const Mat& Bm) {
  const int n = LU.n, nr = Bm.n;
  Mat X(n, nr);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < nr; ++j) X(i, j) = Bm(perm[i], j);
  const int cw = 32;  // column block
#pragma omp parallel for schedule(dynamic, 1) if ((double)n * n * nr > 4e6)
  for (int j0 = 0; j0 < nr; j0 += cw) {
    const int j1 = std::min(nr, j0 + cw);
    for (int i = 0; i < n; ++i)          // L y = P b (unit lower)
      for (int k = 0; k < i; ++k) {
        const cplx l = LU(i, k);
        if (l == cplx(0, 0)) continue;
        for (int j = j0; j < j1; ++j) X(i, j) -= l * X(k, j);
      }
    for (int i = n - 1; i >= 0; --i) {   // U x = y
      for (int k = i + 1; k < n; ++k) {
        const cplx u = LU(i, k);
        if (u == cplx(0, 0)) continue;
        for (int j = j0; j < j1; ++j) X(i, j) -= u * X(k, j);
      }
      const cplx d = LU(i, i);
      for (int j = j0; j < j1; ++j) X(i, j) /= d;
    }
  }
  return X;
}

// Explicit inverse: LU with partial pivoting, then solve against the identity
// (the zgetrf + zgetri pair of PAPER.md:724-725, written out naively).
static int inverse(const Mat& A, Mat& Ainv) {
  Mat LU = A;
  std::vector<int> perm;
  int rc = lu_factor(LU, perm);
  if (rc) return rc;
  Ainv = lu_solve(LU, perm, identity(A.n));
  return 0;
}

// ----------------------------------------------------------------------------
// Chebyshev grid and differentiation matrix (reading Q4)
// ----------------------------------------------------------------------------
// Lobatto points on [-1, 1] in ascending order, x_k = -cos(k pi / (p-1)).
static std::vector<double> cheb_nodes(int p) {
  std::vector<double> x(p);
  const int N = p - 1;
  for (int k = 0; k < p; ++k) x[k] = -std::cos(M_PI * k / N);
  // exact symmetry / endpoints
  x[0] = -1.0;
  x[N] = 1.0;
  if (p % 2 == 1) x[N / 2] = 0.0;
  return x;
}

// Trefethen's closed form: D_ij = (c_i/c_j) (-1)^{i+j} / (x_i - x_j), i != j,
// c_0 = c_N = 2, else 1; D_ii = -sum_{j != i} D_ij.  (Spectral Methods in
// MATLAB, cheb.m; the formula is ordering-independent.)
static std::vector<double> cheb_diff(const std::vector<double>& x) {
  const int p = (int)x.size(), N = p - 1;
  std::vector<double> D((size_t)p * p, 0.0);
  for (int i = 0; i < p; ++i) {
    double rowsum = 0.0;
    for (int j = 0; j < p; ++j) {
      if (i == j) continue;
      const double ci = (i == 0 || i == N) ? 2.0 : 1.0;
      const double cj = (j == 0 || j == N) ? 2.0 : 1.0;
      const double sgn = ((i + j) % 2 == 0) ? 1.0 : -1.0;
      D[(size_t)i * p + j] = (ci / cj) * sgn / (x[i] - x[j]);
      rowsum += D[(size_t)i * p + j];
    }
    D[(size_t)i * p + i] = -rowsum;
  }
  return D;
}

// ----------------------------------------------------------------------------
// Leaf index sets (Fig. 2)
// Tensor node (ix, iy) has natural index iy*p + ix (x fastest).
// ----------------------------------------------------------------------------
struct LeafIndex {
  std::vector<int> Is, Ie, In, Iw, Ib, Ii, It;  // It = [Ib, Ii]
};

static LeafIndex leaf_index(int p) {
  LeafIndex L;
  for (int ix = 1; ix <= p - 2; ++ix) L.Is.push_back(0 * p + ix);          // south, increasing x
  for (int iy = 1; iy <= p - 2; ++iy) L.Ie.push_back(iy * p + (p - 1));    // east, increasing y
  for (int ix = 1; ix <= p - 2; ++ix) L.In.push_back((p - 1) * p + ix);    // north, increasing x
  for (int iy = 1; iy <= p - 2; ++iy) L.Iw.push_back(iy * p + 0);          // west, increasing y
  for (auto v : {&L.Is, &L.Ie, &L.In, &L.Iw}) L.Ib.insert(L.Ib.end(), v->begin(), v->end());
  for (int iy = 1; iy <= p - 2; ++iy)
    for (int ix = 1; ix <= p - 2; ++ix) L.Ii.push_back(iy * p + ix);
  L.It = L.Ib;
  L.It.insert(L.It.end(), L.Ii.begin(), L.Ii.end());
  return L;
}

// ----------------------------------------------------------------------------
// Leaf operators
// ----------------------------------------------------------------------------
struct LeafOps {
  Mat Psi, Y, R, Gamma;
};

struct LeafDisc {
  Mat Ahat;  // p^2 x p^2
  Mat N, F, G, B;
};

// Assemble A-hat = -Dx^2 - Dy^2 - C, N, F, G and B (eq. 7) for a leaf of
// width hx, height hy.  c holds kappa-independent c(x_k) at the p*p tensor
// nodes (x fastest); corner values are never used.
static LeafDisc leaf_disc(int p, double hx, double hy, double kappa, cplx eta, const cplx* c) {
  const int P2 = p * p;
  std::vector<double> xi = cheb_nodes(p);
  std::vector<double> D = cheb_diff(xi);
  // Full p^2 x p^2 tensor-product differentiation matrices.
  Mat Dx(P2, P2), Dy(P2, P2);
  for (int iy = 0; iy < p; ++iy)
    for (int ix = 0; ix < p; ++ix) {
      const int r = iy * p + ix;
      for (int k = 0; k < p; ++k) {
        Dx(r, iy * p + k) = D[(size_t)ix * p + k] * (2.0 / hx);
        Dy(r, k * p + ix) = D[(size_t)iy * p + k] * (2.0 / hy);
      }
    }
  Mat Dxx = matmul(Dx, Dx), Dyy = matmul(Dy, Dy);
  LeafDisc L;
  L.Ahat = Mat(P2, P2);
  for (int i = 0; i < P2; ++i)
    for (int j = 0; j < P2; ++j) L.Ahat(i, j) = -Dxx(i, j) - Dyy(i, j);
  for (int k = 0; k < P2; ++k) L.Ahat(k, k) -= kappa * kappa * c[k];

  LeafIndex ix = leaf_index(p);
  const int nb = (int)ix.Ib.size(), nt = (int)ix.It.size();
  // N: outward normal derivatives (reading Q1).
  Mat Ns = neg(sub(Dy, ix.Is, ix.It));
  Mat Ne = sub(Dx, ix.Ie, ix.It);
  Mat Nn = sub(Dy, ix.In, ix.It);
  Mat Nw = neg(sub(Dx, ix.Iw, ix.It));
  L.N = vcat(vcat(Ns, Ne), vcat(Nn, Nw));
  // F = N + i eta I(Ib, It), G = N - i eta I(Ib, It)
  Mat E = sub(identity(P2), ix.Ib, ix.It);
  L.F = L.N; L.G = L.N;
  for (int i = 0; i < nb; ++i)
    for (int j = 0; j < nt; ++j) {
      L.F(i, j) += I_UNIT * eta * E(i, j);
      L.G(i, j) -= I_UNIT * eta * E(i, j);
    }
  // B = [F ; Ahat(Ii, Ib) Ahat(Ii, Ii)] = [F ; Ahat(Ii, It)]  (eq. 7, reading Q2)
  L.B = vcat(L.F, sub(L.Ahat, ix.Ii, ix.It));
  return L;
}

static int leaf_ops(int p, double hx, double hy, double kappa, cplx eta, const cplx* c, LeafOps& out,
                    Mat* Bout = nullptr) {
  LeafDisc L = leaf_disc(p, hx, hy, kappa, eta, c);
  const int nb = 4 * p - 8, nt = p * p - 4;
  Mat Binv;
  int rc = inverse(L.B, Binv);
  if (rc) return rc;
  std::vector<int> cb, ci;
  for (int j = 0; j < nb; ++j) cb.push_back(j);
  for (int j = nb; j < nt; ++j) ci.push_back(j);
  std::vector<int> all;
  for (int j = 0; j < nt; ++j) all.push_back(j);
  out.Psi = sub(Binv, all, cb);      // B Psi = [I; 0]   (eq. 8)
  out.Y = sub(Binv, all, ci);        // B Y   = [0; I]   (eq. 10)
  out.R = matmul(L.G, out.Psi);      // R = G Psi
  out.Gamma = matmul(L.G, out.Y);    // Gamma = G Y
  if (Bout) *Bout = L.B;
  return 0;
}

// ----------------------------------------------------------------------------
// Boxes, geometric node keys and the tree (Fig. 1)
// ----------------------------------------------------------------------------
// A boundary node of any box lies on a leaf edge.  Key = (orientation,
// grid line, leaf segment along the line, Chebyshev node 1..p-2).
typedef int64_t Key;
static Key make_key(int vertical, int line, int seg, int k) {
  return ((Key)vertical << 60) | ((Key)line << 36) | ((Key)seg << 12) | (Key)k;
}

struct Box {
  int i0, i1, j0, j1;  // leaf-index ranges [i0,i1) x [j0,j1)
  int level = 0;       // depth from the root (root = 0)
  bool leaf = false;
  int vertical = 0;    // split orientation for non-leaves (1 = alpha west | beta east)
};

// Canonical boundary key list: [S, E, N, W], each edge increasing coordinate; ne nodes per
// leaf-edge segment (p - 2 Chebyshev nodes, or the q Gauss-Legendre nodes of the GL edge
// representation, oracle_build_gl).
static std::vector<Key> box_keys(const Box& b, int ne) {
  std::vector<Key> K;
  for (int i = b.i0; i < b.i1; ++i)
    for (int k = 1; k <= ne; ++k) K.push_back(make_key(0, b.j0, i, k));  // S
  for (int j = b.j0; j < b.j1; ++j)
    for (int k = 1; k <= ne; ++k) K.push_back(make_key(1, b.i1, j, k));  // E
  for (int i = b.i0; i < b.i1; ++i)
    for (int k = 1; k <= ne; ++k) K.push_back(make_key(0, b.j1, i, k));  // N
  for (int j = b.j0; j < b.j1; ++j)
    for (int k = 1; k <= ne; ++k) K.push_back(make_key(1, b.i0, j, k));  // W
  return K;
}

struct Tree {
  int nx, ny, L;  // leaves nx x ny; L = depth of the leaf level
  std::vector<Box> box;  // 1-based; box[0] unused
};

// Split the longer side (in leaves), ties vertical (reading Q6).
static Tree make_tree(int nx, int ny) {
  Tree T;
  T.nx = nx; T.ny = ny;
  T.box.resize(2);
  T.box[1] = Box{0, nx, 0, ny, 0, false, 0};
  // breadth-first; children of tau are 2 tau (alpha) and 2 tau + 1 (beta)
  for (size_t tau = 1; tau < T.box.size(); ++tau) {
    Box& b = T.box[tau];
    const int w = b.i1 - b.i0, h = b.j1 - b.j0;
    if (w == 1 && h == 1) { b.leaf = true; continue; }
    Box a = b, c = b;
    a.level = c.level = b.level + 1;
    if (w >= h) {  // vertical interface
      b.vertical = 1;
      a.i1 = b.i0 + w / 2; c.i0 = a.i1;
    } else {
      b.vertical = 0;
      a.j1 = b.j0 + h / 2; c.j0 = a.j1;
    }
    if (T.box.size() < 2 * tau + 2) T.box.resize(2 * tau + 2);
    T.box[2 * tau] = a;
    T.box[2 * tau + 1] = c;
  }
  T.L = T.box.back().level;
  return T;
}

// ----------------------------------------------------------------------------
// Merge (Algorithm 1 lines 5-14)
// ----------------------------------------------------------------------------
struct MergeOps {
  std::vector<Key> keys;       // parent canonical boundary
  std::vector<int> I1, I2, I3a, I3b;  // positions in alpha / beta key lists
  std::vector<int> perm;       // perm[c] = position in [I1, I2] of canonical entry c
  Mat Winv, PhiA, PhiB, UpsA, UpsB, GammaT;  // Phi, Upsilon, Gamma^tau in [I1, I2] order
  Mat Rtau;                    // canonical order
};

static int merge_boxes(const std::vector<Key>& ka, const Mat& Ra, const std::vector<Key>& kb, const Mat& Rb,
                       const std::vector<Key>& kparent, MergeOps& M) {
  // Index sets by geometric intersection.
  std::map<Key, int> pos_b;
  for (size_t j = 0; j < kb.size(); ++j) pos_b[kb[j]] = (int)j;
  std::map<Key, int> pos_a;
  for (size_t j = 0; j < ka.size(); ++j) pos_a[ka[j]] = (int)j;
  M.I1.clear(); M.I2.clear(); M.I3a.clear(); M.I3b.clear();
  for (size_t j = 0; j < ka.size(); ++j) {
    auto it = pos_b.find(ka[j]);
    if (it == pos_b.end()) M.I1.push_back((int)j);
    else { M.I3a.push_back((int)j); M.I3b.push_back(it->second); }
  }
  for (size_t j = 0; j < kb.size(); ++j)
    if (!pos_a.count(kb[j])) M.I2.push_back((int)j);
  const int n1 = (int)M.I1.size(), n2 = (int)M.I2.size(), n3 = (int)M.I3a.size();
  // Blocks (eqs. 11, 12)
  Mat R11a = sub(Ra, M.I1, M.I1), R13a = sub(Ra, M.I1, M.I3a);
  Mat R31a = sub(Ra, M.I3a, M.I1), R33a = sub(Ra, M.I3a, M.I3a);
  Mat R22b = sub(Rb, M.I2, M.I2), R23b = sub(Rb, M.I2, M.I3b);
  Mat R32b = sub(Rb, M.I3b, M.I2), R33b = sub(Rb, M.I3b, M.I3b);
  // (7)  W = I - R33b R33a
  Mat W = add(identity(n3), matmul(R33b, R33a), -1.0);
  int rc = inverse(W, M.Winv);
  if (rc) return rc;
  // (8)  Phi^a = W^{-1} [R33b R31a | -R32b]
  M.PhiA = matmul(M.Winv, hcat(matmul(R33b, R31a), neg(R32b)));
  // (9)  Upsilon^a = [W^{-1} R33b | -W^{-1}]
  M.UpsA = hcat(matmul(M.Winv, R33b), neg(M.Winv));
  // (10) Phi^b = [-R31a - R33a W^{-1} R33b R31a | R33a W^{-1} R32b]
  Mat R33aWi = matmul(R33a, M.Winv);
  M.PhiB = hcat(add(neg(R31a), matmul(matmul(R33aWi, R33b), R31a), -1.0), matmul(R33aWi, R32b));
  // (11) Upsilon^b = [-(I + R33a W^{-1} R33b) | R33a W^{-1}]
  M.UpsB = hcat(neg(add(identity(n3), matmul(R33aWi, R33b))), R33aWi);
  // (12) R^tau = diag(R11a, R22b) + diag(R13a, R23b) [Phi^a; Phi^b]   (reading Q3)
  Mat top = matmul(R13a, M.PhiA), bot = matmul(R23b, M.PhiB);
  Mat R12(n1 + n2, n1 + n2);
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n1 + n2; ++j) R12(i, j) = top(i, j) + (j < n1 ? R11a(i, j) : cplx(0, 0));
  for (int i = 0; i < n2; ++i)
    for (int j = 0; j < n1 + n2; ++j) R12(n1 + i, j) = bot(i, j) + (j >= n1 ? R22b(i, j - n1) : cplx(0, 0));
  // (13) Gamma^tau = diag(R13a, R23b) [Upsilon^a; Upsilon^b]
  M.GammaT = vcat(matmul(R13a, M.UpsA), matmul(R23b, M.UpsB));
  // Permute [I1, I2] -> parent canonical order (reading Q5).
  std::map<Key, int> pos12;
  for (int j = 0; j < n1; ++j) pos12[ka[M.I1[j]]] = j;
  for (int j = 0; j < n2; ++j) pos12[kb[M.I2[j]]] = n1 + j;
  if ((int)kparent.size() != n1 + n2) return -1000;
  M.perm.resize(n1 + n2);
  for (int c = 0; c < n1 + n2; ++c) {
    auto it = pos12.find(kparent[c]);
    if (it == pos12.end()) return -1001;
    M.perm[c] = it->second;
  }
  M.Rtau = Mat(n1 + n2, n1 + n2);
  for (int i = 0; i < n1 + n2; ++i)
    for (int j = 0; j < n1 + n2; ++j) M.Rtau(i, j) = R12(M.perm[i], M.perm[j]);
  M.keys = kparent;
  return 0;
}

// ----------------------------------------------------------------------------
// The whole tree: Algorithm 1 (build) and Algorithm 2 (solve)
// ----------------------------------------------------------------------------
struct Oracle {
  double x0, x1, y0, y1;
  int nx, ny, p;
  double kappa;
  cplx eta;
  int keep_all_R;
  Tree T;
  std::vector<LeafOps> leaf;         // indexed by box id (only leaves filled)
  std::vector<MergeOps> merge;       // indexed by box id (only non-leaves filled)
  std::vector<Mat> R;                // kept R (all if keep_all_R, else root only)
  std::vector<std::vector<Key>> keys;
  std::string err;
  double build_seconds = 0, solve_seconds = 0;
};

static thread_local std::string g_err;

// leaf natural index (iy, ix) of a leaf box
static int leaf_nat(const Oracle& O, const Box& b) { return b.j0 * O.nx + b.i0; }

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_cheb(int p, double* x, double* D) {
  if (p < 2) return -1;
  std::vector<double> xs = cheb_nodes(p), Ds = cheb_diff(xs);
  if (x) std::memcpy(x, xs.data(), sizeof(double) * p);
  if (D) std::memcpy(D, Ds.data(), sizeof(double) * p * p);
  return 0;
}

// Coordinates of every tensor node of every leaf: [nleaf natural (iy,ix)][p*p] (x fastest).
int oracle_leaf_nodes(double x0, double x1, double y0, double y1, int nx, int ny, int p, double* X, double* Y) {
  if (p < 2 || nx < 1 || ny < 1) return -1;
  std::vector<double> xi = cheb_nodes(p);
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  for (int ly = 0; ly < ny; ++ly)
    for (int lx = 0; lx < nx; ++lx) {
      const size_t base = ((size_t)ly * nx + lx) * p * p;
      const double ax = x0 + lx * hx, ay = y0 + ly * hy;
      for (int iy = 0; iy < p; ++iy)
        for (int ix = 0; ix < p; ++ix) {
          X[base + iy * p + ix] = ax + (1.0 + xi[ix]) * 0.5 * hx;
          Y[base + iy * p + ix] = ay + (1.0 + xi[iy]) * 0.5 * hy;
        }
    }
  return 0;
}

// Coordinates and outward normals of the root boundary nodes, canonical
// [S, E, N, W] order (each edge increasing coordinate).
int oracle_root_boundary(double x0, double x1, double y0, double y1, int nx, int ny, int p, double* X, double* Y,
                         double* NX, double* NY) {
  if (p < 4 || nx < 1 || ny < 1) return -1;
  std::vector<double> xi = cheb_nodes(p);
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  Box root{0, nx, 0, ny, 0, false, 0};
  std::vector<Key> K = box_keys(root, p - 2);
  for (size_t j = 0; j < K.size(); ++j) {
    const int vertical = (int)(K[j] >> 60), line = (int)((K[j] >> 36) & 0xFFFFFF);
    const int seg = (int)((K[j] >> 12) & 0xFFFFFF), k = (int)(K[j] & 0xFFF);
    if (!vertical) {
      X[j] = x0 + seg * hx + (1.0 + xi[k]) * 0.5 * hx;
      Y[j] = y0 + line * hy;
      NX[j] = 0.0;
      NY[j] = (line == 0) ? -1.0 : 1.0;
    } else {
      X[j] = x0 + line * hx;
      Y[j] = y0 + seg * hy + (1.0 + xi[k]) * 0.5 * hy;
      NX[j] = (line == 0) ? -1.0 : 1.0;
      NY[j] = 0.0;
    }
  }
  return 0;
}

// One leaf: any output pointer may be NULL.  Row-major outputs.
// Psi (nt x nb), Y (nt x ni), R (nb x nb), Gamma (nb x ni), B (nt x nt).
int oracle_leaf(int p, double hx, double hy, double kappa, double eta_re, double eta_im, const cplx* c,
                cplx* Psi, cplx* Y, cplx* R, cplx* Gamma, cplx* B) {
  if (p < 4) { g_err = "p < 4"; return -1; }
  LeafOps L;
  Mat Bm;
  int rc = leaf_ops(p, hx, hy, kappa, cplx(eta_re, eta_im), c, L, &Bm);
  if (rc) { g_err = "singular leaf matrix B"; return -2; }
  if (Psi) std::copy(L.Psi.a.begin(), L.Psi.a.end(), Psi);
  if (Y) std::copy(L.Y.a.begin(), L.Y.a.end(), Y);
  if (R) std::copy(L.R.a.begin(), L.R.a.end(), R);
  if (Gamma) std::copy(L.Gamma.a.begin(), L.Gamma.a.end(), Gamma);
  if (B) std::copy(Bm.a.begin(), Bm.a.end(), B);
  return 0;
}

// Leaf discretisation pieces for tests: Ahat (p2 x p2), N, F, G (nb x nt).
int oracle_leaf_disc(int p, double hx, double hy, double kappa, double eta_re, double eta_im, const cplx* c,
                     cplx* Ahat, cplx* N, cplx* F, cplx* G) {
  if (p < 4) return -1;
  LeafDisc L = leaf_disc(p, hx, hy, kappa, cplx(eta_re, eta_im), c);
  if (Ahat) std::copy(L.Ahat.a.begin(), L.Ahat.a.end(), Ahat);
  if (N) std::copy(L.N.a.begin(), L.N.a.end(), N);
  if (F) std::copy(L.F.a.begin(), L.F.a.end(), F);
  if (G) std::copy(L.G.a.begin(), L.G.a.end(), G);
  return 0;
}

// Standalone merge of two congruent children of cnx x cny leaves each;
// vertical = 1: alpha west of beta, 0: alpha south of beta.  Ra, Rb are the
// children's R in canonical order (row-major).  Outputs (any may be NULL):
// Rtau canonical (nb_tau^2), PhiA / PhiB (n3 x (n1+n2), [I1, I2] columns),
// Winv (n3^2), UpsA / UpsB (n3 x 2 n3), GammaT ((n1+n2) x 2 n3, [I1, I2] rows).
int oracle_merge(int p, int cnx, int cny, int vertical, const cplx* Ra, const cplx* Rb, cplx* Rtau,
                 cplx* PhiA, cplx* PhiB, cplx* Winv, cplx* UpsA, cplx* UpsB, cplx* GammaT) {
  Box a{0, cnx, 0, cny, 1, false, 0}, b = a, t{0, cnx, 0, cny, 0, false, vertical};
  if (vertical) { b.i0 = cnx; b.i1 = 2 * cnx; t.i1 = 2 * cnx; }
  else { b.j0 = cny; b.j1 = 2 * cny; t.j1 = 2 * cny; }
  std::vector<Key> ka = box_keys(a, p - 2), kb = box_keys(b, p - 2), kt = box_keys(t, p - 2);
  Mat RA((int)ka.size(), (int)ka.size()), RB((int)kb.size(), (int)kb.size());
  std::copy(Ra, Ra + RA.a.size(), RA.a.begin());
  std::copy(Rb, Rb + RB.a.size(), RB.a.begin());
  MergeOps M;
  int rc = merge_boxes(ka, RA, kb, RB, kt, M);
  if (rc) { g_err = "merge failed (singular W or index mismatch)"; return -2; }
  if (Rtau) std::copy(M.Rtau.a.begin(), M.Rtau.a.end(), Rtau);
  if (PhiA) std::copy(M.PhiA.a.begin(), M.PhiA.a.end(), PhiA);
  if (PhiB) std::copy(M.PhiB.a.begin(), M.PhiB.a.end(), PhiB);
  if (Winv) std::copy(M.Winv.a.begin(), M.Winv.a.end(), Winv);
  if (UpsA) std::copy(M.UpsA.a.begin(), M.UpsA.a.end(), UpsA);
  if (UpsB) std::copy(M.UpsB.a.begin(), M.UpsB.a.end(), UpsB);
  if (GammaT) std::copy(M.GammaT.a.begin(), M.GammaT.a.end(), GammaT);
  return 0;
}

// Leaf-index rectangle [i0, i1) x [j0, j1) and split orientation of box `box` (heap id).
int oracle_box_rect(int nx, int ny, int64_t box, int* i0, int* i1, int* j0, int* j1, int* vertical) {
  Tree T = make_tree(nx, ny);
  if (box < 1 || box >= (int64_t)T.box.size()) return -1;
  const Box& b = T.box[box];
  *i0 = b.i0;
  *i1 = b.i1;
  *j0 = b.j0;
  *j1 = b.j1;
  *vertical = b.leaf ? -1 : b.vertical;
  return 0;
}

// Tree facts for tests: number of boxes, leaf depth, per-box n_b.
int oracle_tree_info(int nx, int ny, int p, int64_t* nboxes, int* depth) {
  Tree T = make_tree(nx, ny);
  if (nboxes) *nboxes = (int64_t)T.box.size() - 1;
  if (depth) *depth = T.L;
  return 0;
}

}  // extern "C"

// Gauss-Legendre edge representation (beyond the paper, which samples every
// leaf edge at its p - 2 corner-free Chebyshev nodes; the ItI representation it
// cites, uses q Gauss-Legendre nodes per edge).  Incoming data f on an edge
// is given at the q GL nodes; the Chebyshev leaf sees P f (P: (p-2) x q, the degree-(q-1)
// Lagrange interpolant through the GL nodes evaluated at the edge's Chebyshev nodes) and its
// outgoing data g at the Chebyshev nodes is returned as Q g (Q: q x (p-2), the degree-(p-3)
// interpolant through the Chebyshev nodes evaluated at the GL nodes).  With the edge maps
// block-diagonal over [S, E, N, W]:  Psi <- Psi Pblk,  R <- Qblk R Pblk,  Gamma <- Qblk Gamma.
static Mat edge_blocks(const double* A, int m, int n) {  // 4 copies of the m x n edge map
  Mat B(4 * m, 4 * n);
  for (int e = 0; e < 4; ++e)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) B(e * m + i, e * n + j) = cplx(A[(size_t)i * n + j], 0.0);
  return B;
}

static void leaf_to_gl(LeafOps& L, const Mat& Pblk, const Mat& Qblk) {
  L.Psi = matmul(L.Psi, Pblk);
  L.R = matmul(matmul(Qblk, L.R), Pblk);
  L.Gamma = matmul(Qblk, L.Gamma);
}

// Algorithm 1 (precomputation).  c: [nleaf natural (iy, ix)][p*p].  qe = 0: the paper's
// Chebyshev edges; qe > 0: the GL edge representation with the maps P ((p-2) x qe) and
// Qm (qe x (p-2)), row-major.
static void* build_impl(double x0, double x1, double y0, double y1, int nx, int ny, int p, int qe,
                        const double* P, const double* Qm, double kappa, double eta_re, double eta_im,
                        const cplx* c, int keep_all_R) {
  if (p < 4 || nx < 1 || ny < 1 || !(x1 > x0) || !(y1 > y0)) { g_err = "invalid arguments"; return nullptr; }
  if (qe < 0 || (qe > 0 && (!P || !Qm))) { g_err = "invalid GL edge maps"; return nullptr; }
  const int ne = qe > 0 ? qe : p - 2;
  Mat Pblk, Qblk;
  if (qe > 0) {
    Pblk = edge_blocks(P, p - 2, qe);
    Qblk = edge_blocks(Qm, qe, p - 2);
  }
  auto t0 = std::chrono::steady_clock::now();
  Oracle* O = new Oracle();
  O->x0 = x0; O->x1 = x1; O->y0 = y0; O->y1 = y1;
  O->nx = nx; O->ny = ny; O->p = p; O->kappa = kappa; O->eta = cplx(eta_re, eta_im);
  O->keep_all_R = keep_all_R;
  O->T = make_tree(nx, ny);
  const int nbox = (int)O->T.box.size();
  O->leaf.resize(nbox);
  O->merge.resize(nbox);
  O->R.resize(nbox);
  O->keys.resize(nbox);
  for (int tau = 1; tau < nbox; ++tau) O->keys[tau] = box_keys(O->T.box[tau], ne);
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  int fail = 0;
  // Algorithm 1 loops tau = N_boxes ... 1; boxes of one level are independent
  // (Algorithm 3), so each level is an OpenMP parallel loop.
  for (int lev = O->T.L; lev >= 0; --lev) {
    std::vector<int> ids;
    for (int tau = nbox - 1; tau >= 1; --tau)
      if (O->T.box[tau].level == lev) ids.push_back(tau);
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t q = 0; q < ids.size(); ++q) {
      const int tau = ids[q];
      const Box& b = O->T.box[tau];
      if (b.leaf) {
        const cplx* cl = c + (size_t)leaf_nat(*O, b) * p * p;
        if (leaf_ops(p, hx, hy, kappa, O->eta, cl, O->leaf[tau])) {
#pragma omp atomic write
          fail = tau;
          continue;
        }
        if (qe > 0) leaf_to_gl(O->leaf[tau], Pblk, Qblk);
        O->R[tau] = O->leaf[tau].R;
      } else {
        const int a = 2 * tau, bb = 2 * tau + 1;
        if (merge_boxes(O->keys[a], O->R[a], O->keys[bb], O->R[bb], O->keys[tau], O->merge[tau])) {
#pragma omp atomic write
          fail = tau;
          continue;
        }
        O->R[tau] = O->merge[tau].Rtau;
      }
    }
    if (fail) break;
    // Algorithm 1 line 14: delete the children's R (unless kept for parity).
    if (!keep_all_R)
      for (int tau = 1; tau < nbox; ++tau)
        if (O->T.box[tau].level == lev + 1) O->R[tau] = Mat();
  }
  if (fail) {
    g_err = "singular matrix at box " + std::to_string(fail);
    delete O;
    return nullptr;
  }
  O->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return O;
}

extern "C" {

void* oracle_build(double x0, double x1, double y0, double y1, int nx, int ny, int p, double kappa,
                   double eta_re, double eta_im, const cplx* c, int keep_all_R) {
  return build_impl(x0, x1, y0, y1, nx, ny, p, 0, nullptr, nullptr, kappa, eta_re, eta_im, c, keep_all_R);
}

// The same tree with the Gauss-Legendre edge representation: qe nodes per leaf edge, P and Qm
// the edge maps above (the caller computes them; tests/ pins them).  t of oracle_solve is then
// given at the root's GL nodes, [nrhs][2 (nx + ny) qe].
void* oracle_build_gl(double x0, double x1, double y0, double y1, int nx, int ny, int p, int qe, const double* P,
                      const double* Qm, double kappa, double eta_re, double eta_im, const cplx* c, int keep_all_R) {
  if (qe < 1) { g_err = "qe < 1"; return nullptr; }
  return build_impl(x0, x1, y0, y1, nx, ny, p, qe, P, Qm, kappa, eta_re, eta_im, c, keep_all_R);
}

double oracle_build_seconds(void* h) { return h ? ((Oracle*)h)->build_seconds : -1; }
double oracle_solve_seconds(void* h) { return h ? ((Oracle*)h)->solve_seconds : -1; }

// Algorithm 2 (solve).  s: [nrhs][nleaf][(p-2)^2]; t: [nrhs][nb_root];
// u: [nrhs][nleaf][p*p-4] in [Ib; Ii] order per leaf, natural leaf order.
int oracle_solve(void* h, int nrhs, const cplx* s, const cplx* t, cplx* u) {
  if (!h) return -1;
  Oracle& O = *(Oracle*)h;
  auto t0 = std::chrono::steady_clock::now();
  const int p = O.p, ni = (p - 2) * (p - 2), nt = p * p - 4;
  const int nbox = (int)O.T.box.size(), nleaf = O.nx * O.ny;
  const int nbr = (int)O.keys[1].size();
  for (int r = 0; r < nrhs; ++r) {
    std::vector<Mat> hv(nbox), ut(nbox), tt_a(nbox), tt_b(nbox), tv(nbox);
    // Upward pass (lines 1-9)
    for (int lev = O.T.L; lev >= 0; --lev) {
      std::vector<int> ids;
      for (int tau = nbox - 1; tau >= 1; --tau)
        if (O.T.box[tau].level == lev) ids.push_back(tau);
#pragma omp parallel for schedule(dynamic, 1)
      for (size_t q = 0; q < ids.size(); ++q) {
        const int tau = ids[q];
        const Box& b = O.T.box[tau];
        if (b.leaf) {
          Mat sv(ni, 1);
          const cplx* sl = s + ((size_t)r * nleaf + leaf_nat(O, b)) * ni;
          for (int k = 0; k < ni; ++k) sv(k, 0) = sl[k];
          ut[tau] = matmul(O.leaf[tau].Y, sv);       // u~ = Y s
          hv[tau] = matmul(O.leaf[tau].Gamma, sv);   // h  = Gamma s
        } else {
          const MergeOps& M = O.merge[tau];
          const int a = 2 * tau, bb = 2 * tau + 1;
          const int n1 = (int)M.I1.size(), n2 = (int)M.I2.size(), n3 = (int)M.I3a.size();
          Mat h3(2 * n3, 1);
          for (int k = 0; k < n3; ++k) { h3(k, 0) = hv[a](M.I3a[k], 0); h3(n3 + k, 0) = hv[bb](M.I3b[k], 0); }
          tt_a[tau] = matmul(M.UpsA, h3);   // t~a = Upsilon^a [h3a; h3b]
          tt_b[tau] = matmul(M.UpsB, h3);   // t~b = Upsilon^b [h3a; h3b]
          Mat g = matmul(M.GammaT, h3);     // eq. (flux_part), [I1, I2] order
          Mat h12(n1 + n2, 1);
          for (int k = 0; k < n1; ++k) h12(k, 0) = hv[a](M.I1[k], 0) + g(k, 0);
          for (int k = 0; k < n2; ++k) h12(n1 + k, 0) = hv[bb](M.I2[k], 0) + g(n1 + k, 0);
          hv[tau] = Mat(n1 + n2, 1);
          for (int cidx = 0; cidx < n1 + n2; ++cidx) hv[tau](cidx, 0) = h12(M.perm[cidx], 0);
        }
      }
    }
    // Downward pass (lines 10-18).  Root incoming data is the given t.
    tv[1] = Mat(nbr, 1);
    for (int k = 0; k < nbr; ++k) tv[1](k, 0) = t[(size_t)r * nbr + k];
    for (int lev = 0; lev <= O.T.L; ++lev) {
      std::vector<int> ids;
      for (int tau = 1; tau < nbox; ++tau)
        if (O.T.box[tau].level == lev) ids.push_back(tau);
#pragma omp parallel for schedule(dynamic, 1)
      for (size_t q = 0; q < ids.size(); ++q) {
        const int tau = ids[q];
        const Box& b = O.T.box[tau];
        if (b.leaf) {
          Mat uv = add(matmul(O.leaf[tau].Psi, tv[tau]), ut[tau]);  // u = Psi t + u~
          cplx* ul = u + ((size_t)r * nleaf + leaf_nat(O, b)) * nt;
          for (int k = 0; k < nt; ++k) ul[k] = uv(k, 0);
        } else {
          const MergeOps& M = O.merge[tau];
          const int a = 2 * tau, bb = 2 * tau + 1;
          const int n1 = (int)M.I1.size(), n2 = (int)M.I2.size(), n3 = (int)M.I3a.size();
          Mat t12(n1 + n2, 1);
          for (int cidx = 0; cidx < n1 + n2; ++cidx) t12(M.perm[cidx], 0) = tv[tau](cidx, 0);
          Mat t3a = add(matmul(M.PhiA, t12), tt_a[tau]);  // t3a = Phi^a t + t~a
          Mat t3b = add(matmul(M.PhiB, t12), tt_b[tau]);  // t3b = Phi^b t + t~b
          tv[a] = Mat((int)O.keys[a].size(), 1);
          tv[bb] = Mat((int)O.keys[bb].size(), 1);
          for (int k = 0; k < n1; ++k) tv[a](M.I1[k], 0) = t12(k, 0);
          for (int k = 0; k < n2; ++k) tv[bb](M.I2[k], 0) = t12(n1 + k, 0);
          for (int k = 0; k < n3; ++k) { tv[a](M.I3a[k], 0) = t3a(k, 0); tv[bb](M.I3b[k], 0) = t3b(k, 0); }
        }
      }
    }
  }
  O.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return 0;
}

int64_t oracle_box_nb(void* h, int64_t box) {
  if (!h) return -1;
  Oracle& O = *(Oracle*)h;
  if (box < 1 || box >= (int64_t)O.keys.size()) return -1;
  return (int64_t)O.keys[box].size();
}

// R of one box (row-major, canonical order).  Needs keep_all_R for non-root boxes.
int oracle_export_R(void* h, int64_t box, cplx* out) {
  if (!h) return -1;
  Oracle& O = *(Oracle*)h;
  if (box < 1 || box >= (int64_t)O.R.size() || O.R[box].a.empty()) { g_err = "R not kept"; return -2; }
  std::copy(O.R[box].a.begin(), O.R[box].a.end(), out);
  return 0;
}

// Leaf operators of leaf box `box` (heap id).
int oracle_export_leaf(void* h, int64_t box, cplx* Psi, cplx* Y) {
  if (!h) return -1;
  Oracle& O = *(Oracle*)h;
  if (box < 1 || box >= (int64_t)O.leaf.size() || !O.T.box[box].leaf) return -2;
  if (Psi) std::copy(O.leaf[box].Psi.a.begin(), O.leaf[box].Psi.a.end(), Psi);
  if (Y) std::copy(O.leaf[box].Y.a.begin(), O.leaf[box].Y.a.end(), Y);
  return 0;
}

// Heap id of the leaf with natural index (iy, ix).
int64_t oracle_leaf_box(void* h, int ix, int iy) {
  if (!h) return -1;
  Oracle& O = *(Oracle*)h;
  for (size_t tau = 1; tau < O.T.box.size(); ++tau) {
    const Box& b = O.T.box[tau];
    if (b.leaf && b.i0 == ix && b.j0 == iy) return (int64_t)tau;
  }
  return -1;
}

void oracle_free(void* h) { delete (Oracle*)h; }

// ----------------------------------------------------------------------------
// Brute-force global collocation (all leaves, dense LU).  Unknowns: every
// leaf's [Ib; Ii] values.  Rows per leaf: interior collocation Ahat(Ii, It) u
// = s; per boundary node: F u = t on the outer boundary, and on an interface
// F^a_j u^a + G^b_j' u^b = 0 (t3^a = -g3^b).  Returns u for each
// RHS, and (if Rroot != NULL) the root ItI operator, column by column
// (t = e_j, s = 0, R e_j = G u on the outer boundary).
// ----------------------------------------------------------------------------
int oracle_global_dense(double x0, double x1, double y0, double y1, int nx, int ny, int p, double kappa,
                        double eta_re, double eta_im, const cplx* c, int nrhs, const cplx* s, const cplx* t,
                        cplx* u, cplx* Rroot) {
  const cplx eta(eta_re, eta_im);
  const int nb = 4 * p - 8, ni = (p - 2) * (p - 2), nt = p * p - 4, nleaf = nx * ny;
  const int Ntot = nleaf * nt;
  const double hx = (x1 - x0) / nx, hy = (y1 - y0) / ny;
  std::vector<LeafDisc> D(nleaf);
  std::vector<std::vector<Key>> K(nleaf);
  std::map<Key, std::vector<std::pair<int, int>>> owners;  // key -> (leaf, local boundary pos)
  for (int ly = 0; ly < ny; ++ly)
    for (int lx = 0; lx < nx; ++lx) {
      const int l = ly * nx + lx;
      D[l] = leaf_disc(p, hx, hy, kappa, eta, c + (size_t)l * p * p);
      Box b{lx, lx + 1, ly, ly + 1, 0, true, 0};
      K[l] = box_keys(b, p - 2);
      for (int j = 0; j < nb; ++j) owners[K[l][j]].push_back({l, j});
    }
  Box root{0, nx, 0, ny, 0, false, 0};
  std::vector<Key> kr = box_keys(root, p - 2);
  std::map<Key, int> rootpos;
  for (size_t j = 0; j < kr.size(); ++j) rootpos[kr[j]] = (int)j;
  const int nbr = (int)kr.size();
  Mat A(Ntot, Ntot);
  // which RHS entries: boundary rows on the outer boundary take t(rootpos)
  std::vector<int> row_root(Ntot, -1);
  for (int l = 0; l < nleaf; ++l) {
    const int off = l * nt;
    for (int j = 0; j < nb; ++j) {
      const int row = off + j;
      auto& own = owners[K[l][j]];
      for (int k = 0; k < nt; ++k) A(row, off + k) = D[l].F(j, k);
      if (own.size() == 1) {
        row_root[row] = rootpos.at(K[l][j]);
      } else {
        const auto other = (own[0].first == l) ? own[1] : own[0];
        const int ooff = other.first * nt;
        for (int k = 0; k < nt; ++k) A(row, ooff + k) += D[other.first].G(other.second, k);
      }
    }
    LeafIndex ix = leaf_index(p);
    for (int i = 0; i < ni; ++i)
      for (int k = 0; k < nt; ++k) A(off + nb + i, off + k) = D[l].Ahat(ix.Ii[i], ix.It[k]);
  }
  Mat LU = A;
  std::vector<int> perm;
  if (lu_factor(LU, perm)) { g_err = "singular global system"; return -2; }
  if (u && nrhs > 0) {
    Mat rhs(Ntot, nrhs);
    for (int r = 0; r < nrhs; ++r)
      for (int l = 0; l < nleaf; ++l) {
        for (int j = 0; j < nb; ++j) {
          const int row = l * nt + j;
          if (row_root[row] >= 0) rhs(row, r) = t[(size_t)r * nbr + row_root[row]];
        }
        for (int i = 0; i < ni; ++i) rhs(l * nt + nb + i, r) = s[((size_t)r * nleaf + l) * ni + i];
      }
    Mat X = lu_solve(LU, perm, rhs);
    for (int r = 0; r < nrhs; ++r)
      for (int i = 0; i < Ntot; ++i) u[(size_t)r * Ntot + i] = X(i, r);
  }
  if (Rroot) {
    Mat rhs(Ntot, nbr);
    for (int row = 0; row < Ntot; ++row)
      if (row_root[row] >= 0) rhs(row, row_root[row]) = 1.0;
    Mat X = lu_solve(LU, perm, rhs);
    // outgoing data on the outer boundary: g = G u (row of the owning leaf)
    for (int l = 0; l < nleaf; ++l)
      for (int j = 0; j < nb; ++j) {
        const int row = l * nt + j;
        if (row_root[row] < 0) continue;
        const int rr = row_root[row];
        for (int col = 0; col < nbr; ++col) {
          cplx g = 0;
          for (int k = 0; k < nt; ++k) g += D[l].G(j, k) * X(l * nt + k, col);
          Rroot[(size_t)rr * nbr + col] = g;
        }
      }
  }
  return 0;
}

// Naive LU inverse exported for its own residual test.
int oracle_invert(int n, const cplx* A, cplx* Ainv) {
  Mat M(n, n);
  std::copy(A, A + (size_t)n * n, M.a.begin());
  Mat Mi;
  if (inverse(M, Mi)) return -2;
  std::copy(Mi.a.begin(), Mi.a.end(), Ainv);
  return 0;
}

// Thread count of the oracle's OpenMP loops (tests pin that results do not depend on it).
int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

int oracle_matmul(int m, int k, int n, const cplx* A, const cplx* B, cplx* C) {
  Mat a(m, k), b(k, n);
  std::copy(A, A + (size_t)m * k, a.a.begin());
  std::copy(B, B + (size_t)k * n, b.a.begin());
  Mat cm = matmul(a, b);
  std::copy(cm.a.begin(), cm.a.end(), C);
  return 0;
}

}  // extern "C"
