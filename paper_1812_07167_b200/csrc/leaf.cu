// leaf.cu — batched leaf assembly and small layout kernels.
//
// B = [F ; Ahat(I_i, I^tau)]  (eq. 7; reading Q2), n^tau x n^tau row-major, columns in
// I^tau = [I_b (S, E, N, W); I_i] order.  F = N + i eta I(I_b, I^tau) with N the outward
// normal derivative (reading Q1: S -d/dy, E +d/dx, N +d/dy, W -d/dx).
// Ahat = -Dx^2 - Dy^2 - diag(kappa^2 c) on the p x p tensor grid.
// One CTA per leaf; one thread per row (each row has at most 2p nonzeros).
#include "hps_internal.cuh"
#include "hps_kernels.cuh"

namespace {

__global__ void leaf_assemble_kernel(zt* __restrict__ B, int64_t bstride, int leaf0, int nleaf_chunk,
                                     const int* __restrict__ leaf_nat, const zt* __restrict__ c, int p,
                                     const double* __restrict__ dmat,  // [4][p][p]: Dx, Dy, Dxx, Dyy
                                     const int* __restrict__ pos,      // [p*p] -> I^tau position or -1
                                     const int* __restrict__ node,     // [n^tau] -> tensor node
                                     double kappa2, zt eta) {
  const int lc = blockIdx.x;
  if (lc >= nleaf_chunk) return;
  const int q = p - 2, nb = 4 * q, nt = p * p - 4;
  zt* Bl = B + (int64_t)lc * bstride;
  const zt* cl = c + (int64_t)leaf_nat[leaf0 + lc] * p * p;
  const int64_t n2 = (int64_t)nt * nt;
  for (int64_t e = threadIdx.x; e < n2; e += blockDim.x) Bl[e] = make_double2(0.0, 0.0);
  __syncthreads();
  const double* Dx = dmat;
  const double* Dy = dmat + p * p;
  const double* Dxx = dmat + 2 * p * p;
  const double* Dyy = dmat + 3 * p * p;
  for (int rho = threadIdx.x; rho < nt; rho += blockDim.x) {
    const int tn = node[rho];
    const int ix = tn % p, iy = tn / p;
    zt* row = Bl + (int64_t)rho * nt;
    if (rho < nb) {
      const int edge = rho / q;  // 0 S, 1 E, 2 N, 3 W
      for (int k = 0; k < p; ++k) {
        if (edge == 0 || edge == 2) {  // -+ d/dy along the column (ix, k)
          const int col = pos[k * p + ix];
          const double v = (edge == 0 ? -1.0 : 1.0) * Dy[iy * p + k];
          if (col >= 0) row[col].x += v;
        } else {                       // +- d/dx along the row (k, iy)
          const int col = pos[iy * p + k];
          const double v = (edge == 1 ? 1.0 : -1.0) * Dx[ix * p + k];
          if (col >= 0) row[col].x += v;
        }
      }
      // + i eta on the diagonal
      row[rho].x += -eta.y;
      row[rho].y += eta.x;
    } else {
      for (int k = 0; k < p; ++k) {
        row[pos[iy * p + k]].x -= Dxx[ix * p + k];
        row[pos[k * p + ix]].x -= Dyy[iy * p + k];
      }
      const zt cv = cl[tn];
      row[rho].x -= kappa2 * cv.x;
      row[rho].y -= kappa2 * cv.y;
    }
  }
}

// R = I - 2 i eta Psi(I_b, :)  (from G = F - 2 i eta I(I_b, .) and F Psi = I)
__global__ void leaf_R_kernel(const zt* __restrict__ store, int64_t sstride, zt* __restrict__ R, int nleaf, int nt,
                              int nb, zt m2ieta) {
  const int64_t total = (int64_t)nleaf * nb * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % nb);
    const int64_t t = e / nb;
    const int i = (int)(t % nb);
    const int l = (int)(t / nb);
    const zt psi = store[(int64_t)l * sstride + (int64_t)i * nt + j];
    zt v = make_double2(m2ieta.x * psi.x - m2ieta.y * psi.y, m2ieta.x * psi.y + m2ieta.y * psi.x);
    if (i == j) v.x += 1.0;
    R[e] = v;
  }
}

__global__ void zsum_slots_kernel(zt* out, const zt* base, const zt* slots, int nslot, int64_t slot_stride,
                                  int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    zt a = base ? base[i] : make_double2(0.0, 0.0);
    for (int k = 0; k < nslot; ++k) {
      const zt v = slots[k * slot_stride + i];
      a.x += v.x;
      a.y += v.y;
    }
    out[i] = a;
  }
}

// external [r * sr + map[l] * sb + i] -> internal [l][n][nrhs]   (ABI: sr = nleaf n, sb = n)
__global__ void rhs_in_kernel(const zt* __restrict__ src, zt* __restrict__ dst, const int* __restrict__ map,
                              int nbox, int n, int nrhs, int64_t sr, int64_t sb) {
  const int64_t total = (int64_t)nbox * n * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % nrhs);
    const int64_t t = e / nrhs;
    const int i = (int)(t % n);
    const int l = (int)(t / n);
    dst[e] = src[(int64_t)r * sr + (int64_t)map[l] * sb + i];
  }
}

// internal [map[ln]][n][nrhs] -> external [r * sr + ln * sb + i]
__global__ void rhs_out_kernel(const zt* __restrict__ src, zt* __restrict__ dst, const int* __restrict__ map,
                               int nbox, int n, int nrhs, int64_t sr, int64_t sb) {
  const int64_t total = (int64_t)nbox * n * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n);
    const int64_t t = e / n;
    const int ln = (int)(t % nbox);
    const int r = (int)(t / nbox);
    dst[(int64_t)r * sr + (int64_t)ln * sb + i] = src[((int64_t)map[ln] * n + i) * nrhs + r];
  }
}

// Tiled versions for nrhs >= 8: each 256-thread block moves 32 x 32 (node, rhs) tiles through
// shared memory so both the node-contiguous ABI side and the rhs-contiguous internal side are
// read and written in 512-byte rows (the element-wise kernels above read one of the two sides
// with a stride of nrhs or of a whole RHS slice).
__global__ void __launch_bounds__(256) rhs_in_tiled_kernel(const zt* __restrict__ src, zt* __restrict__ dst,
                                                           const int* __restrict__ map, int nbox, int n, int nrhs,
                                                           int64_t sr, int64_t sb) {
  __shared__ zt tile[32][33];
  const int ti = (n + 31) / 32, tr = (nrhs + 31) / 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t blk = blockIdx.x; blk < (int64_t)nbox * ti * tr; blk += gridDim.x) {
    const int l = (int)(blk / (ti * tr)), rem = (int)(blk % (ti * tr)), i0 = (rem / tr) * 32, r0 = (rem % tr) * 32;
    const zt* sp = src + (int64_t)map[l] * sb;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // read: i contiguous
      const int r = r0 + ty + 8 * k, i = i0 + tx;
      if (r < nrhs && i < n) tile[ty + 8 * k][tx] = sp[(int64_t)r * sr + i];
    }
    __syncthreads();
    zt* dp = dst + (int64_t)l * n * nrhs;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // write: r contiguous
      const int i = i0 + ty + 8 * k, r = r0 + tx;
      if (r < nrhs && i < n) dp[(int64_t)i * nrhs + r] = tile[tx][ty + 8 * k];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) rhs_out_tiled_kernel(const zt* __restrict__ src, zt* __restrict__ dst,
                                                            const int* __restrict__ map, int nbox, int n, int nrhs,
                                                            int64_t sr, int64_t sb) {
  __shared__ zt tile[32][33];
  const int ti = (n + 31) / 32, tr = (nrhs + 31) / 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t blk = blockIdx.x; blk < (int64_t)nbox * ti * tr; blk += gridDim.x) {
    const int ln = (int)(blk / (ti * tr)), rem = (int)(blk % (ti * tr)), i0 = (rem / tr) * 32, r0 = (rem % tr) * 32;
    const zt* sp = src + (int64_t)map[ln] * n * nrhs;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // read: r contiguous
      const int i = i0 + ty + 8 * k, r = r0 + tx;
      if (r < nrhs && i < n) tile[ty + 8 * k][tx] = sp[(int64_t)i * nrhs + r];
    }
    __syncthreads();
    zt* dp = dst + (int64_t)ln * sb;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // write: i contiguous
      const int r = r0 + ty + 8 * k, i = i0 + tx;
      if (r < nrhs && i < n) dp[(int64_t)r * sr + i] = tile[tx][ty + 8 * k];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Schur-complement leaf: the boundary block F_b of B couples
// each boundary node only with the opposite node of the same grid line (S_ix <-> N_ix,
// W_iy <-> E_iy), so F_b^{-1} = G is a set of 2x2 blocks and eliminating u_b first leaves the
// interior operator  S = A_ii - A_ib G F_i = Lx (+) Ly - kappa^2 diag(c)  (line operators Lx,
// Ly shared by every leaf).  Then  Y_i = S^{-1}, Psi_i = S^{-1} Ub, Y_b = -V S^{-1},
// Psi_b = G - V Psi_i  with Ub = -A_ib G and V = G F_i (both one-line sparse).
// consts layout (complex): Lx[q*q] Ly[q*q] Ubx[q][2] Uby[q][2] Vx[2][q] Vy[2][q] Gx[2][2] Gy[2][2]
// ---------------------------------------------------------------------------
__global__ void leaf_schur_assemble_kernel(zt* __restrict__ S, int64_t sstride, int leaf0, int nchunk,
                                           const int* __restrict__ leaf_nat, const zt* __restrict__ c, int p,
                                           const zt* __restrict__ K, double kappa2) {
  const int lc = blockIdx.x;
  if (lc >= nchunk) return;
  const int q = p - 2, ni = q * q;
  const zt* Lx = K;
  const zt* Ly = K + q * q;
  const zt* cl = c + (int64_t)leaf_nat[leaf0 + lc] * p * p;
  zt* Sl = S + (int64_t)lc * sstride;
  for (int e = threadIdx.x; e < ni * ni; e += blockDim.x) {
    const int r = e / ni, cc = e % ni;
    const int ix = r % q, iy = r / q, jx = cc % q, jy = cc / q;
    zt v = make_double2(0.0, 0.0);
    if (iy == jy) {
      v.x += Lx[ix * q + jx].x;
      v.y += Lx[ix * q + jx].y;
    }
    if (ix == jx) {
      v.x += Ly[iy * q + jy].x;
      v.y += Ly[iy * q + jy].y;
    }
    if (r == cc) {
      const zt cv = cl[(iy + 1) * p + ix + 1];
      v.x -= kappa2 * cv.x;
      v.y -= kappa2 * cv.y;
    }
    Sl[e] = v;
  }
}

__device__ __forceinline__ void zfma(zt& acc, zt a, zt b) {
  acc.x += a.x * b.x - a.y * b.y;
  acc.y += a.x * b.y + a.y * b.x;
}

// store[l] = [Psi | Y] (nt x nt, row-major); on entry its (I_i, I_i) block holds S^{-1}.
// Psi_i: each warp stages one row of S^{-1} in shared memory (one coalesced read) and its lanes
// form the 4q outputs of that row.  Y_b and Psi_b: the two boundary nodes of a grid line read
// the same rows, so each thread forms both (S_k with N_k, W_k with E_k): S^{-1} is read twice.
// Dynamic shared memory: 8 warps x n_i complex.
__global__ void __launch_bounds__(256) leaf_schur_finish_kernel(zt* __restrict__ store, int64_t sstride, int leaf0,
                                                                int nchunk, int p, const zt* __restrict__ K) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lc = blockIdx.x;
  if (lc >= nchunk) return;
  const int q = p - 2, ni = q * q, nb = 4 * q, nt = nb + ni;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const zt* Ubx = K + 2 * q * q;
  const zt* Uby = Ubx + 2 * q;
  const zt* Vx = Uby + 2 * q;
  const zt* Vy = Vx + 2 * q;
  const zt* Gx = Vy + 2 * q;
  const zt* Gy = Gx + 4;
  zt* base = store + (int64_t)(leaf0 + lc) * sstride;
  const zt* Si = base + (int64_t)nb * nt + nb;  // S^{-1}, ld nt
  zt* rowbuf = reinterpret_cast<zt*>(smem_raw) + warp * ni;
  // Psi_i = S^{-1} Ub
  for (int r = warp; r < ni; r += 8) {
    for (int c = lane; c < ni; c += 32) rowbuf[c] = Si[(int64_t)r * nt + c];
    __syncwarp();
    for (int b = lane; b < nb; b += 32) {
      const int edge = b / q, k = b % q;
      zt acc = make_double2(0.0, 0.0);
      if (edge == 0 || edge == 2) {  // S_k / N_k: y-line ix = k
        const int side = edge == 0 ? 0 : 1;
        for (int t = 0; t < q; ++t) zfma(acc, rowbuf[t * q + k], Uby[t * 2 + side]);
      } else {                       // E_k / W_k: x-line iy = k
        const int side = edge == 3 ? 0 : 1;
        for (int t = 0; t < q; ++t) zfma(acc, rowbuf[k * q + t], Ubx[t * 2 + side]);
      }
      base[(int64_t)(nb + r) * nt + b] = acc;
    }
    __syncwarp();
  }
  // Y_b = -V S^{-1}: thread (line type, k, cc) forms both nodes of the line
  for (int e = threadIdx.x; e < 2 * q * ni; e += blockDim.x) {
    const int ltype = e / (q * ni), rem = e % (q * ni), k = rem / ni, cc = rem % ni;
    zt a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    if (ltype == 0) {  // y-line ix = k: S_k (side 0), N_k (side 1)
      for (int t = 0; t < q; ++t) {
        const zt v = Si[(int64_t)(t * q + k) * nt + cc];
        zfma(a0, Vy[t], v);
        zfma(a1, Vy[q + t], v);
      }
      base[(int64_t)k * nt + nb + cc] = make_double2(-a0.x, -a0.y);
      base[(int64_t)(2 * q + k) * nt + nb + cc] = make_double2(-a1.x, -a1.y);
    } else {           // x-line iy = k: W_k (side 0), E_k (side 1)
      for (int t = 0; t < q; ++t) {
        const zt v = Si[(int64_t)(k * q + t) * nt + cc];
        zfma(a0, Vx[t], v);
        zfma(a1, Vx[q + t], v);
      }
      base[(int64_t)(3 * q + k) * nt + nb + cc] = make_double2(-a0.x, -a0.y);
      base[(int64_t)(q + k) * nt + nb + cc] = make_double2(-a1.x, -a1.y);
    }
  }
  __syncthreads();
  // Psi_b = G - V Psi_i
  const zt* Pi = base + (int64_t)nb * nt;  // Psi_i rows
  for (int e = threadIdx.x; e < 2 * q * nb; e += blockDim.x) {
    const int ltype = e / (q * nb), rem = e % (q * nb), k = rem / nb, b2 = rem % nb;
    const int e2 = b2 / q, k2 = b2 % q;
    zt a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    zt g0 = make_double2(0.0, 0.0), g1 = make_double2(0.0, 0.0);
    if (ltype == 0) {
      for (int t = 0; t < q; ++t) {
        const zt v = Pi[(int64_t)(t * q + k) * nt + b2];
        zfma(a0, Vy[t], v);
        zfma(a1, Vy[q + t], v);
      }
      if (k2 == k && (e2 == 0 || e2 == 2)) {
        g0 = Gy[0 * 2 + (e2 == 0 ? 0 : 1)];
        g1 = Gy[1 * 2 + (e2 == 0 ? 0 : 1)];
      }
      base[(int64_t)k * nt + b2] = make_double2(g0.x - a0.x, g0.y - a0.y);
      base[(int64_t)(2 * q + k) * nt + b2] = make_double2(g1.x - a1.x, g1.y - a1.y);
    } else {
      for (int t = 0; t < q; ++t) {
        const zt v = Pi[(int64_t)(k * q + t) * nt + b2];
        zfma(a0, Vx[t], v);
        zfma(a1, Vx[q + t], v);
      }
      if (k2 == k && (e2 == 1 || e2 == 3)) {
        g0 = Gx[0 * 2 + (e2 == 3 ? 0 : 1)];
        g1 = Gx[1 * 2 + (e2 == 3 ? 0 : 1)];
      }
      base[(int64_t)(3 * q + k) * nt + b2] = make_double2(g0.x - a0.x, g0.y - a0.y);
      base[(int64_t)(q + k) * nt + b2] = make_double2(g1.x - a1.x, g1.y - a1.y);
    }
  }
}

inline int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > hps_num_sms() * 32) b = hps_num_sms() * 32;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

void launch_leaf_assemble(zt* B, int64_t bstride, int leaf0, int nchunk, const int* leaf_nat, const zt* c, int p,
                          const double* dmat, const int* pos, const int* node, double kappa2, zt eta,
                          cudaStream_t st) {
  const double nt = p * p - 4;
  ProfScope ps(K_LEAF_ASM, 0.0, 16.0 * nt * nt * nchunk, st);
  leaf_assemble_kernel<<<nchunk, 256, 0, st>>>(B, bstride, leaf0, nchunk, leaf_nat, c, p, dmat, pos, node, kappa2,
                                                eta);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_leaf_R(const zt* store, int64_t sstride, zt* R, int nleaf, int nt, int nb, zt eta, cudaStream_t st) {
  const zt m2ieta = make_double2(2.0 * eta.y, -2.0 * eta.x);  // -2 i eta
  ProfScope ps(K_LAYOUT, 0.0, 32.0 * (double)nleaf * nb * nb, st);
  leaf_R_kernel<<<grid_for((int64_t)nleaf * nb * nb), 256, 0, st>>>(store, sstride, R, nleaf, nt, nb, m2ieta);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_rhs_in(const zt* src, zt* dst, const int* map, int nbox, int n, int nrhs, int64_t sr, int64_t sb,
                   cudaStream_t st) {
  ProfScope ps(K_LAYOUT, 0.0, 32.0 * (double)nbox * n * nrhs, st);
  if (nrhs >= 8)
    rhs_in_tiled_kernel<<<grid_for((int64_t)nbox * ((n + 31) / 32) * ((nrhs + 31) / 32) * 256), 256, 0, st>>>(
        src, dst, map, nbox, n, nrhs, sr, sb);
  else
    rhs_in_kernel<<<grid_for((int64_t)nbox * n * nrhs), 256, 0, st>>>(src, dst, map, nbox, n, nrhs, sr, sb);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_zsum_slots(zt* out, const zt* base, const zt* slots, int nslot, int64_t slot_stride, int64_t n,
                       cudaStream_t st) {
  if (n <= 0) return;
  ProfScope ps(K_LAYOUT, 0.0, 16.0 * (double)n * (nslot + 1 + (base ? 1 : 0)), st);
  zsum_slots_kernel<<<grid_for(n), 256, 0, st>>>(out, base, slots, nslot, slot_stride, n);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_rhs_out(const zt* src, zt* dst, const int* map, int nbox, int n, int nrhs, int64_t sr, int64_t sb,
                    cudaStream_t st) {
  ProfScope ps(K_LAYOUT, 0.0, 32.0 * (double)nbox * n * nrhs, st);
  if (nrhs >= 8)
    rhs_out_tiled_kernel<<<grid_for((int64_t)nbox * ((n + 31) / 32) * ((nrhs + 31) / 32) * 256), 256, 0, st>>>(
        src, dst, map, nbox, n, nrhs, sr, sb);
  else
    rhs_out_kernel<<<grid_for((int64_t)nbox * n * nrhs), 256, 0, st>>>(src, dst, map, nbox, n, nrhs, sr, sb);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_leaf_schur_assemble(zt* S, int64_t sstride, int leaf0, int nchunk, const int* leaf_nat, const zt* c, int p,
                                const zt* consts, double kappa2, cudaStream_t st) {
  const double ni = (p - 2) * (p - 2);
  ProfScope ps(K_LEAF_ASM, 0.0, 16.0 * ni * ni * nchunk, st);
  leaf_schur_assemble_kernel<<<nchunk, 256, 0, st>>>(S, sstride, leaf0, nchunk, leaf_nat, c, p, consts, kappa2);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}

void launch_leaf_schur_finish(zt* store, int64_t sstride, int leaf0, int nchunk, int p, const zt* consts,
                              cudaStream_t st) {
  const double q = p - 2, ni = q * q, nb = 4 * q;
  ProfScope ps(K_LEAF_ASM, 8.0 * nchunk * q * (2.0 * ni * nb + nb * nb),
               16.0 * nchunk * (2.0 * ni * ni + 2.0 * ni * nb + nb * nb + ni * nb), st);
  const size_t smem = sizeof(zt) * 8 * (size_t)(p - 2) * (p - 2);
  if (smem > 48 * 1024)
    HPS_CUDA_CHECK(cudaFuncSetAttribute(leaf_schur_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  leaf_schur_finish_kernel<<<nchunk, 256, smem, st>>>(store, sstride, leaf0, nchunk, p, consts);
  HPS_CUDA_CHECK(cudaGetLastError());
  count_launch();
}
