// calib.cuh — calibration for the rotation (§4.2):
//   covariance  C = scale * X^T X (+ C)   over a batch of calibration activations X [n][d] bf16
//               (eq. 1: Cov = (1/M) sum_i X_i^T X_i, uncentered; the caller passes
//               scale = 1/M and accumulates batches / sequences);
//   rotation    Q = eigenvectors of C, eigenvalues descending, each eigenvector's largest-|entry|
//               component made positive (lowest row on ties).
// The covariance runs on the tcgen05 path of the fold (fold_tc.cuh, fp32 epilogue) when d % 128
// == 0 and n % 64 == 0, else on the CUDA-core kernel below; the eigensolver is our parallel
// cyclic two-sided Jacobi in fp64 (below), followed by the ordering / sign kernel.
#pragma once
#include "common.cuh"
#include "gemv.cuh"

namespace larosa {

// C[i][j] = scale * sum_t X[t][i] X[t][j] (+ C[i][j]); 32 x 32 output tile per CTA, 32-token
// chunks staged in shared memory, fp32 accumulation in token order.
__global__ void __launch_bounds__(256) covariance_simt_kernel(const uint16_t* __restrict__ X, int n, int d, float scale,
                                                              int accumulate, float* __restrict__ C) {
    __shared__ float xi[32][33], xj[32][33];
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t0 = 0; t0 < n; t0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            const int t = t0 + r;
            xi[r][tx] = (t < n && i0 + tx < d) ? bf16f(X[(size_t)t * d + i0 + tx]) : 0.f;
            xj[r][tx] = (t < n && j0 + tx < d) ? bf16f(X[(size_t)t * d + j0 + tx]) : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            const float b = xj[r][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fmaf(xi[r][ty + 8 * u], b, acc[u]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty + 8 * u, j = j0 + tx;
        if (i < d && j < d) {
            const float v = scale * acc[u];
            C[(size_t)i * d + j] = accumulate ? C[(size_t)i * d + j] + v : v;
        }
    }
}

// ---- the eigensolver: cyclic two-sided Jacobi in fp64 (the oracle's
// solver, parallelised) ----------------------------------------------------------------------------
// A sweep visits every pair (p, q) once, as n - 1 rounds of n/2 DISJOINT pairs (the round-robin
// "circle" tournament, n = d rounded up to even; a phantom index pairs with nobody): round r pairs
// (r, n - 1) and ((r + i) mod (n - 1), (r - i) mod (n - 1)) for i = 1 .. n/2 - 1.  Within a round the
// rotations commute, so A <- J^T A J and V <- V J are applied to all pairs at once: every 2 x 2 block
// (rows of pair k, columns of pair l) becomes R_k^T B R_l.  Rotation (the oracle's jacobi_eigh):
// theta = (a_qq - a_pp) / (2 a_pq), t = sgn(theta) / (|theta| + sqrt(1 + theta^2)), c = 1/sqrt(1+t^2),
// s = t c; new col p = c col_p - s col_q, new col q = s col_p + c col_q; a_pq <- 0.  Sweeps repeat
// until off(A) <= 1e-12 ||A||_F (at most 100), like the oracle.  A and V are fp64 row-major [d][d].
// A, V are n x n (n = d rounded up to even): an odd d gets one zero row / column, an exact zero
// "phantom" eigenvalue whose rotations are all the identity (a_pq = 0 -> c = 1, s = 0); it is
// dropped when the eigenvalues are ordered.
__global__ void jacobi_init_kernel(const float* __restrict__ C, double* __restrict__ A, double* __restrict__ V, int d,
                                   int n) {
    const size_t nn = (size_t)n * n;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nn; e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / n), j = (int)(e % n);
        A[e] = (i < d && j < d) ? 0.5 * ((double)C[(size_t)i * d + j] + (double)C[(size_t)j * d + i]) : 0.0;
        V[e] = i == j ? 1.0 : 0.0;
    }
}

__device__ __forceinline__ void jacobi_pair(int r, int i, int n, int& p, int& q) {
    const int m = n - 1;
    int a, b;
    if (i == 0) {
        a = r;
        b = m;
    } else {
        a = (r + i) % m;
        b = (r - i + m) % m;
    }
    p = min(a, b);
    q = max(a, b);
}

// round r: every pair's (c, s)
__global__ void jacobi_angles_kernel(const double* __restrict__ A, int n, int r, int* __restrict__ pq,
                                     double2* __restrict__ cs) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n / 2) return;
    int p, q;
    jacobi_pair(r, i, n, p, q);
    double c = 1.0, s = 0.0;
    {
        const double apq = A[(size_t)p * n + q];
        if (apq != 0.0) {
            const double theta = (A[(size_t)q * n + q] - A[(size_t)p * n + p]) / (2.0 * apq);
            double t;
            if (fabs(theta) > 1e150) {
                t = 0.5 / theta;
            } else {
                t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
            }
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
        }
    }
    pq[2 * i] = p;
    pq[2 * i + 1] = q;
    cs[i] = make_double2(c, s);
}

// A <- J^T A J: thread (k, l), k <= l, owns the 2 x 2 blocks (k, l) and (l, k)
__global__ void __launch_bounds__(256) jacobi_rotate_a_kernel(double* __restrict__ A, int d, int npairs,
                                                              const int* __restrict__ pq, const double2* __restrict__ cs) {
    const int l = blockIdx.x * 16 + (threadIdx.x & 15), k = blockIdx.y * 16 + (threadIdx.x >> 4);
    if (k >= npairs || l >= npairs || k > l) return;
    const int pk = pq[2 * k], qk = pq[2 * k + 1], pl = pq[2 * l], ql = pq[2 * l + 1];
    const double2 rk = cs[k], rl = cs[l];
    const double ck = rk.x, sk = rk.y, cl = rl.x, sl = rl.y;
    double* r0 = A + (size_t)pk * d;
    double* r1 = A + (size_t)qk * d;
    const double b00 = r0[pl], b01 = r0[ql], b10 = r1[pl], b11 = r1[ql];
    // B R_l (columns), then R_k^T (rows)
    const double c00 = cl * b00 - sl * b01, c01 = sl * b00 + cl * b01;
    const double c10 = cl * b10 - sl * b11, c11 = sl * b10 + cl * b11;
    double n00 = ck * c00 - sk * c10, n01 = ck * c01 - sk * c11;
    double n10 = sk * c00 + ck * c10, n11 = sk * c01 + ck * c11;
    if (k == l) {   // the pair's own block: the rotation annihilates a_pq
        n01 = 0.0;
        n10 = 0.0;
        r0[pl] = n00;
        r0[ql] = n01;
        r1[pl] = n10;
        r1[ql] = n11;
        return;
    }
    r0[pl] = n00;
    r0[ql] = n01;
    r1[pl] = n10;
    r1[ql] = n11;
    double* s0 = A + (size_t)pl * d;   // the mirrored block (l, k) = transpose
    double* s1 = A + (size_t)ql * d;
    s0[pk] = n00;
    s0[qk] = n10;
    s1[pk] = n01;
    s1[qk] = n11;
}

// V <- V J: thread (row i, pair k)
__global__ void __launch_bounds__(256) jacobi_rotate_v_kernel(double* __restrict__ V, int d, int npairs,
                                                              const int* __restrict__ pq, const double2* __restrict__ cs) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (e >= (size_t)d * npairs) return;
    const int k = (int)(e % npairs), i = (int)(e / npairs);
    const int p = pq[2 * k], q = pq[2 * k + 1];
    const double2 r = cs[k];
    double* row = V + (size_t)i * d;
    const double vp = row[p], vq = row[q];
    row[p] = r.x * vp - r.y * vq;
    row[q] = r.y * vp + r.x * vq;
}

// off(A)^2 and ||A||_F^2, fixed-order two-level reduction (part[2 * gridDim.x], then CTA 0 of the
// second launch sums them)
__global__ void __launch_bounds__(256) jacobi_norms_kernel(const double* __restrict__ A, int d, double* __restrict__ part) {
    __shared__ double so[8], sf[8];
    double off = 0.0, fro = 0.0;
    const size_t n = (size_t)d * d;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const double a = A[e];
        fro += a * a;
        if (e / d != e % d) off += a * a;
    }
    for (int o = 16; o > 0; o >>= 1) {
        off += __shfl_xor_sync(0xffffffffu, off, o);
        fro += __shfl_xor_sync(0xffffffffu, fro, o);
    }
    if ((threadIdx.x & 31) == 0) {
        so[threadIdx.x >> 5] = off;
        sf[threadIdx.x >> 5] = fro;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += so[w];
            b += sf[w];
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}
__global__ void jacobi_norms_final_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < nparts; ++i) {
            a += part[2 * i];
            b += part[2 * i + 1];
        }
        out[0] = a;
        out[1] = b;
    }
}

// rank of eigenvalue j in descending order, stable (lower index first on exact ties; Z7)
__global__ void eig_rank_kernel(const double* __restrict__ A, int d, int ld, int* __restrict__ src_of_rank) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d) return;
    const double wj = A[(size_t)j * ld + j];
    int rank = 0;
    for (int i = 0; i < d; ++i) {
        const double wi = A[(size_t)i * ld + i];
        rank += wi > wj || (wi == wj && i < j);
    }
    src_of_rank[rank] = j;
}

// One CTA per output direction c (eigenvalue rank c, descending): V's column src_of_rank[c], sign so
// that the largest-|entry| component (lowest row on ties) is positive; Q[r][c] fp32 row-major;
// lam[c] = max(lambda, 0) (the oracle clamps round-off negatives, Z7).
__global__ void __launch_bounds__(256) pca_order_sign_kernel(const double* __restrict__ V, const double* __restrict__ A,
                                                             const int* __restrict__ src_of_rank, int d, int ld,
                                                             float* __restrict__ Q, float* __restrict__ lam) {
    __shared__ double sbest[8];
    __shared__ int sidx[8];
    const int c = blockIdx.x, src = src_of_rank[c];
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = threadIdx.x; r < d; r += blockDim.x) {
        const double a = fabs(V[(size_t)r * ld + src]);
        if (a > best || (a == best && r < bi)) {
            best = a;
            bi = r;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sbest[threadIdx.x >> 5] = best;
        sidx[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
            if (sbest[k] > sbest[0] || (sbest[k] == sbest[0] && sidx[k] < sidx[0])) {
                sbest[0] = sbest[k];
                sidx[0] = sidx[k];
            }
        lam[c] = (float)fmax(A[(size_t)src * ld + src], 0.0);
    }
    __syncthreads();
    const double sgn = V[(size_t)sidx[0] * ld + src] < 0.0 ? -1.0 : 1.0;
    for (int r = threadIdx.x; r < d; r += blockDim.x) Q[(size_t)r * d + c] = (float)(sgn * V[(size_t)r * ld + src]);
}

}  // namespace larosa

namespace larosa {
// Prefill: every token keeps its own Top-K (full sparsification of
// prompt tokens P:77).  X_hi / X_lo [n][d] bf16 = split(x_t[i] * s_t) where token t keeps i (its
// rule: key > Tk or key == Tk and i <= Ti), else 0; the GEMM Y = X_hi W + X_lo W then runs on the
// tensor cores (cuBLAS, fp32 accumulation; the hi/lo split keeps ~16 mantissa bits of the fp32
// activations, like the batched tcgen05 GEMV).
__global__ void prefill_mask_split_kernel(const float* __restrict__ X, int n, int d, const ThreshOut* __restrict__ rules,
                                          uint16_t* __restrict__ Xhi, uint16_t* __restrict__ Xlo) {
    const size_t total = (size_t)n * d;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int t = (int)(e / d), i = (int)(e % d);
        const ThreshOut r = rules[t];
        const float x = X[e];
        const uint32_t key = __float_as_uint(x) & 0x7fffffffu;
        const bool keep = key > r.tk || (key == r.tk && i <= r.ti);
        const float v = keep ? x * r.scale : 0.f;
        const uint16_t h = f2bf16_rne(v);
        Xhi[e] = h;
        Xlo[e] = f2bf16_rne(v - bf16f(h));
    }
}
}  // namespace larosa
