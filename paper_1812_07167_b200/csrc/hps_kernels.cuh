// hps_kernels.cuh — launchers of the leaf / layout kernels (leaf.cu).
#pragma once
#include "hps_internal.cuh"

void launch_leaf_assemble(zt* B, int64_t bstride, int leaf0, int nchunk, const int* leaf_nat, const zt* c, int p,
                          const double* dmat, const int* pos, const int* node, double kappa2, zt eta,
                          cudaStream_t st);
void launch_leaf_R(const zt* store, int64_t sstride, zt* R, int nleaf, int nt, int nb, zt eta, cudaStream_t st);
void launch_rhs_in(const zt* src, zt* dst, const int* map, int nbox, int n, int nrhs, int64_t sr, int64_t sb,
                   cudaStream_t st);
void launch_rhs_out(const zt* src, zt* dst, const int* map, int nbox, int n, int nrhs, int64_t sr, int64_t sb,
                    cudaStream_t st);
void launch_leaf_schur_assemble(zt* S, int64_t sstride, int leaf0, int nchunk, const int* leaf_nat, const zt* c, int p,
                                const zt* consts, double kappa2, cudaStream_t st);
void launch_leaf_schur_finish(zt* store, int64_t sstride, int leaf0, int nchunk, int p, const zt* consts,
                              cudaStream_t st);
// out[i] = (base ? base[i] : 0) + sum_{k < nslot} slots[k * slot_stride + i], k in increasing order
// (the deterministic reduction of the sharded solve), i < n.
void launch_zsum_slots(zt* out, const zt* base, const zt* slots, int nslot, int64_t slot_stride, int64_t n,
                       cudaStream_t st);
