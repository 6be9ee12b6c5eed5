// calib.cuh — calibration for the rotation (§4.2):
//   covariance  C = scale * X^T X (+ C)   over a batch of calibration activations X [n][d] bf16
//               (eq. 1: Cov = (1/M) sum_i X_i^T X_i, uncentered; the caller passes
//               scale = 1/M and accumulates batches / sequences);
//   rotation    Q = eigenvectors of C, eigenvalues descending, each eigenvector's largest-|entry|
//               component made positive (lowest row on ties).
// The covariance runs on the tcgen05 path of the fold (fold_tc.cuh, fp32 epilogue) when d % 128
// == 0 and n % 64 == 0, else on the CUDA-core kernel below; the eigensolver is cuSOLVER's
// symmetric divide-and-conquer in fp64 (a library primitive), followed by the ordering / sign
// kernel here.
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

__global__ void f32_to_f64_sym_kernel(const float* __restrict__ C, double* __restrict__ A, int d) {
    // A (column-major for cuSOLVER) = symmetrised C: A[i + j d] = (C[i][j] + C[j][i]) / 2
    const size_t n = (size_t)d * d;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % d), j = (int)(e / d);
        A[e] = 0.5 * ((double)C[(size_t)i * d + j] + (double)C[(size_t)j * d + i]);
    }
}

// One CTA per output direction c (eigenvalue rank c, descending): cuSOLVER's column
// d - 1 - c (ascending order), sign so that the largest-|entry| component (lowest row on ties)
// is positive; Q[r][c] fp32 row-major; lam[c] clamped at 0.
__global__ void __launch_bounds__(256) pca_order_sign_kernel(const double* __restrict__ V, const double* __restrict__ w,
                                                             int d, float* __restrict__ Q, float* __restrict__ lam) {
    __shared__ double sbest[8];
    __shared__ int sidx[8];
    const int c = blockIdx.x, src = d - 1 - c;
    const double* col = V + (size_t)src * d;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = threadIdx.x; r < d; r += blockDim.x) {
        const double a = fabs(col[r]);
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
        lam[c] = (float)fmax(w[src], 0.0);
    }
    __syncthreads();
    const double sgn = col[sidx[0]] < 0.0 ? -1.0 : 1.0;
    for (int r = threadIdx.x; r < d; r += blockDim.x) Q[(size_t)r * d + c] = (float)(sgn * col[r]);
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
