#!/usr/bin/env python
"""Feasibility probe for the step AFTER the DMMA roof (DESIGN 11, "beyond the FP64 tensor roof"):
the merge products as error-free integer-slice products (Ozaki scheme) on the B200 INT8 tensor
path (tcgen05 kind::i8, 4.5 POP/s nominal against 37 TF/s of DMMA).

Not part of the product path, the tests or the bench; nothing here is called by the library.

CPU part (always): a complex product C = A B of merge-like operands (A = W^-1,
B = R33^beta R31^alpha, entries O(1) with a wide row range) is formed from s signed 7-bit slices per
real operand (rows of A and columns of B scaled by powers of two, slice products exact in int64,
the s(s+1)/2 products with i + j < s kept, summed in fp64 from the smallest weight up), in the 3M
complex form the library uses (DESIGN 3.14), and compared with the fp64 product and a
longdouble product.  Prints the relative error per slice count: what s the 1e-9 parity bar and the
library's own 1e-13 level need.

GPU part (only with CUDA): times torch._int_mm (cuBLASLt s8 x s8 -> s32; a LIBRARY call, here only
to measure what the INT8 tensor path delivers on this box) at merge-like shapes and prints the
FP64-equivalent rate for each s: 2 M N K / (3 real products x s(s+1)/2 slice products x time).
"""
import sys
import time

import numpy as np


def split(X, s, axis, bits=7):
    """X (real, fp64) -> scale (power of two per row/column), s integer slices of `bits` bits."""
    m = np.max(np.abs(X), axis=axis, keepdims=True)
    m[m == 0] = 1.0
    e = np.ceil(np.log2(m)) + 1            # |X / 2^e| < 1/2
    Y = X / np.exp2(e)
    sl = []
    for _ in range(s):
        Y = Y * (1 << bits)
        q = np.rint(Y)                       # |q| <= 2^(bits-1) = 64: fits s8
        sl.append(q.astype(np.int64))
        Y = Y - q
    return np.exp2(e), sl


def sliced_real(A, B, s, bits=7):
    ea, sa = split(A, s, 1, bits)
    eb, sb = split(B, s, 0, bits)
    acc = np.zeros((A.shape[0], B.shape[1]))
    for w in range(s - 1, -1, -1):           # weight 2^-(bits (i + j + 2)), smallest first
        P = np.zeros(acc.shape, dtype=np.int64)
        for i in range(w + 1):
            P += sa[i] @ sb[w - i]
        acc += P.astype(np.float64) * 2.0 ** (-bits * (w + 2))
    return acc * ea * eb


def sliced_complex_3m(A, B, s):
    ar, ai, br, bi = A.real, A.imag, B.real, B.imag
    t1 = sliced_real(ar, br, s)
    t2 = sliced_real(ai, bi, s)
    t3 = sliced_real(ar + ai, br + bi, s)
    return (t1 - t2) + 1j * (t3 - t1 - t2)


def operands(n, k, m, seed):
    rng = np.random.default_rng(seed)
    # W = I - (contraction-like product), A = W^-1; B with rows spanning six decades
    Q1 = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))[0]
    Q2 = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))[0]
    W = np.eye(n) - 0.9 * Q1 @ Q2
    A = np.linalg.inv(W)[:, :k]
    B = (rng.standard_normal((k, m)) + 1j * rng.standard_normal((k, m))) * 10.0 ** rng.uniform(-6, 0, (k, 1))
    return A, B


def cpu_part():
    n, k, m = 224, 224, 336
    A, B = operands(n, k, m, 1)
    ref = (A.astype(np.clongdouble) @ B.astype(np.clongdouble)).astype(np.complex128)
    d = A @ B
    nrm = np.max(np.abs(ref))
    print(f"operands {n}x{k} @ {k}x{m}: fp64 product vs longdouble {np.max(np.abs(d - ref)) / nrm:.2e}")
    for s in range(3, 10):
        C = sliced_complex_3m(A, B, s)
        print(f"  s = {s}: {s * (s + 1) // 2:3d} slice products per real product, "
              f"rel err vs longdouble {np.max(np.abs(C - ref)) / nrm:.2e}")


def gpu_part():
    import torch
    if not torch.cuda.is_available():
        print("no CUDA device: GPU part skipped")
        return
    dev = "cuda:0"
    shapes = [(8192, 8192, 8192), (3584, 3584, 10752), (1792, 1792, 5376), (448, 448, 1344)]
    for (M, K, N) in shapes:
        a = torch.randint(-64, 65, (M, K), dtype=torch.int8, device=dev)
        b = torch.randint(-64, 65, (N, K), dtype=torch.int8, device=dev).t()   # K-contiguous (TN)
        try:
            torch._int_mm(a, b)
        except Exception as e:                     # noqa: BLE001
            print(f"torch._int_mm unavailable on this box: {e}")
            return
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps * 1e-3
        tops = 2.0 * M * N * K / t / 1e12
        eq = {s: 8.0 * M * N * K / (3 * (s * (s + 1) // 2) * t) / 1e12 for s in (5, 6, 7, 8)}
        print(f"s8 GEMM {M}x{K}x{N}: {t * 1e3:.3f} ms, {tops:.0f} TOP/s; complex-FP64-equivalent "
              f"(8 flop per complex MAC, 3M x s(s+1)/2 slice products, slicing and fp64 accumulation "
              f"not counted): " + ", ".join(f"s={s}: {v:.0f} TF/s" for s, v in eq.items()))


def gpu_full(M=3584, K=3584, N=10752, s=7, bits=7):
    """The whole sliced complex product on the GPU with torch ops around torch._int_mm (an upper
    bound on the time: every slice, partial sum and weight is its own torch kernel), against
    torch's complex128 matmul (cuBLAS ZGEMM) for value and time."""
    import torch
    if not torch.cuda.is_available():
        return
    dev = "cuda:0"
    g = torch.Generator(device=dev).manual_seed(3)
    A = torch.randn(M, K, 2, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn(K, N, 2, dtype=torch.float64, device=dev, generator=g)
    B = B * 10.0 ** (-6 * torch.rand(K, 1, 1, dtype=torch.float64, device=dev, generator=g))
    Ac, Bc = torch.view_as_complex(A), torch.view_as_complex(B)

    def tsplit(X, dim):
        m = X.abs().amax(dim=dim, keepdim=True).clamp_min(1e-300)
        e = torch.ceil(torch.log2(m)) + 1
        Y = X * torch.exp2(-e)
        out = []
        for _ in range(s):
            Y = Y * (1 << bits)
            q = torch.round(Y)
            q8 = q.to(torch.int8)
            out.append(q8.t().contiguous().t() if dim == 0 else q8)   # B slices K-contiguous (TN)
            Y = Y - q
        return torch.exp2(e), out

    def real_prod(X, Y):
        ex, sx = tsplit(X, 1)
        ey, sy = tsplit(Y, 0)
        acc = torch.zeros(M, N, dtype=torch.float64, device=dev)
        for w in range(s - 1, -1, -1):
            P = torch._int_mm(sx[0], sy[w])
            for i in range(1, w + 1):
                P += torch._int_mm(sx[i], sy[w - i])
            acc += P.to(torch.float64) * 2.0 ** (-bits * (w + 2))
        return acc * ex * ey

    def prod():
        ar, ai, br, bi = A[..., 0], A[..., 1], B[..., 0], B[..., 1]
        t1, t2, t3 = real_prod(ar, br), real_prod(ai, bi), real_prod(ar + ai, br + bi)
        return torch.complex(t1 - t2, t3 - t1 - t2)

    def timed(f, reps=3):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            r = f()
        e1.record()
        torch.cuda.synchronize()
        return r, e0.elapsed_time(e1) / reps

    try:
        C, t_s = timed(prod)
    except Exception as e:                         # noqa: BLE001
        print(f"sliced product failed: {e}")
        return
    D, t_z = timed(lambda: Ac @ Bc)
    err = ((C - D).abs().max() / D.abs().max()).item()
    fl = 8.0 * M * N * K
    print(f"complex {M}x{K}x{N}, s = {s}: sliced (torch ops + _int_mm) {t_s:.2f} ms = {fl / t_s / 1e9:.1f} TF/s-equivalent, "
          f"cuBLAS ZGEMM {t_z:.2f} ms = {fl / t_z / 1e9:.1f} TF/s, max rel diff {err:.2e}")


if __name__ == "__main__":
    t0 = time.time()
    cpu_part()
    print(f"cpu part {time.time() - t0:.1f} s")
    if "--cpu" not in sys.argv:
        gpu_part()
        for sh in ((3584, 3584, 10752), (1792, 1792, 5376), (896, 896, 2688)):
            for ns in (6, 7, 8):
                gpu_full(*sh, s=ns)
