// aux.cuh — batch>1 column union, weight packing, and the CUDA-core fold
// baseline.
#pragma once
#include "common.cuh"
#include "gemv.cuh"

namespace larosa {

// ------------------------------------------------------------------------------------------
// idx lists -> bitmasks (standalone batched GEMV only; the layer gets masks from Top-K).
// mask must be zeroed first.  One thread per (token, list entry).
// ------------------------------------------------------------------------------------------
__global__ void idx_to_mask_kernel(const int32_t* __restrict__ idx, int64_t k, int batch, int nwords,
                                   uint32_t* __restrict__ mask) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = (int64_t)batch * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(t / k);
        const int i = idx[t];
        atomicOr(&mask[(size_t)b * nwords + (i >> 5)], 1u << (i & 31));
    }
}

// ------------------------------------------------------------------------------------------
// Union of the tokens' kept rows.  rows[] = ascending union U, V[r][b] = token b's value at
// row U[r] (its entry in the ascending list vals[b][*], found by rank = popcount of the
// token's mask below the row) or 0 when token b did not keep that row.  *nrows = |U|.
// grid = ceil(nwords / 32) CTAs x 1024 threads; CTA handles words [32*cta, 32*cta + 32).
// ------------------------------------------------------------------------------------------
constexpr int kUnionThreads = 1024;

__global__ void __launch_bounds__(kUnionThreads) union_kernel(const uint32_t* __restrict__ mask, int nwords, int batch,
                                                              int bp, const float* __restrict__ vals, int64_t k,
                                                              int d, int32_t* __restrict__ rows,
                                                              float* __restrict__ V, int* __restrict__ nrows) {
    __shared__ int s_base[17];        // [0..batch) rank bases, [16] union base
    __shared__ int s_wpre[17][33];    // per-word exclusive prefix inside the CTA (per token, union)
    __shared__ uint32_t s_w[17][32];  // the CTA's words (per token, union)
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w0 = blockIdx.x * 32;

    // bases: popcount of all words before w0 (warp b for token b, warp 16 for the union)
    if (warp <= 16 && (warp < batch || warp == 16)) {
        int acc = 0;
        for (int w = lane; w < w0; w += 32) {
            uint32_t m;
            if (warp == 16) {
                m = 0u;
                for (int b = 0; b < batch; ++b) m |= mask[(size_t)b * nwords + w];
            } else {
                m = mask[(size_t)warp * nwords + w];
            }
            acc += __popc(m);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        // this CTA's 32 words and their exclusive prefix
        uint32_t m = 0u;
        const int w = w0 + lane;
        if (w < nwords) {
            if (warp == 16) {
                for (int b = 0; b < batch; ++b) m |= mask[(size_t)b * nwords + w];
            } else {
                m = mask[(size_t)warp * nwords + w];
            }
        }
        const int pc = __popc(m);
        const int inc = warp_incl_scan(pc);
        s_w[warp][lane] = m;
        s_wpre[warp][lane] = inc - pc;
        if (lane == 0) s_base[warp] = acc;
    }
    __syncthreads();

    const int i = w0 * 32 + tid;   // the row this thread owns
    if (i < d) {
        const int wl = tid >> 5, bit = tid & 31;
        const uint32_t um = s_w[16][wl];
        if ((um >> bit) & 1u) {
            const uint32_t lt = (1u << bit) - 1u;
            const int pos = s_base[16] + s_wpre[16][wl] + __popc(um & lt);
            rows[pos] = i;
            for (int b = 0; b < bp; ++b) {
                float v = 0.f;
                if (b < batch) {
                    const uint32_t mb = s_w[b][wl];
                    if ((mb >> bit) & 1u) {
                        const int rank = s_base[b] + s_wpre[b][wl] + __popc(mb & lt);
                        v = vals[(size_t)b * k + rank];
                    }
                }
                V[(size_t)pos * bp + b] = v;
            }
        }
    }
    // CTA 0 publishes |U| (union popcount of all words)
    if (blockIdx.x == 0 && warp == 0) {
        int acc = 0;
        for (int w = lane; w < nwords; w += 32) {
            uint32_t m = 0u;
            for (int b = 0; b < batch; ++b) m |= mask[(size_t)b * nwords + w];
            acc += __popc(m);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) *nrows = acc;
    }
}

// ------------------------------------------------------------------------------------------
// Decode-step glue.
// resid[b][i] = E'[tokens[b]][i]  (the folded embedding E' = E Q_0, bf16 -> fp32)
// ------------------------------------------------------------------------------------------
__global__ void embed_kernel(const uint16_t* __restrict__ E, const int32_t* __restrict__ tokens, int d,
                             float* __restrict__ resid) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const uint16_t* row = E + (size_t)tokens[b] * d;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x)
        resid[(size_t)b * d + i] = bf16f(row[i]);
}

// xs[b][i] = x[b][i] * s_b,  s_b = 1 / sqrt(mean_i x[b][i]^2 + eps)   (one CTA per token,
// fixed-order reduction; the final RMSNorm whose gain is folded into the head)
constexpr int kRowThreads = 1024;
__global__ void __launch_bounds__(kRowThreads) rms_rows_kernel(const float* __restrict__ x, int d, float eps,
                                                               float* __restrict__ xs) {
    __shared__ float sw[32];
    pdl_wait();
    pdl_trigger();
    const float* xr = x + (size_t)blockIdx.x * d;
    float ssq = 0.f;
    for (int i = threadIdx.x; i < d; i += kRowThreads) ssq = fmaf(xr[i], xr[i], ssq);
    const float tot = block_sum<kRowThreads>(ssq, sw);
    const float s = 1.0f / sqrtf(tot / (float)d + eps);
    for (int i = threadIdx.x; i < d; i += kRowThreads) xs[(size_t)blockIdx.x * d + i] = xr[i] * s;
}

// out[b] = argmax_i logits[b][i], the lowest index on exact ties (greedy decoding)
__device__ __forceinline__ void argmax_merge(float& v, int& i, float v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
    }
}
__global__ void __launch_bounds__(kRowThreads) argmax_kernel(const float* __restrict__ logits, int64_t ld, int n,
                                                             int32_t* __restrict__ out) {
    __shared__ float sv[32];
    __shared__ int si[32];
    pdl_wait();
    pdl_trigger();
    const float* row = logits + (size_t)blockIdx.x * ld;
    float v = -INFINITY;
    int idx = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += kRowThreads) argmax_merge(v, idx, row[i], i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
        argmax_merge(v, idx, v2, i2);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sv[wid] = v;
        si[wid] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kRowThreads / 32; ++w) argmax_merge(v, idx, sv[w], si[w]);
        out[blockIdx.x] = idx;
    }
}

// gathered [world][batch][dl] (an NCCL rank-major all-gather of per-rank [batch][dl] blocks)
// -> out [batch][world * dl] (column order of the full vector)
__global__ void gather_permute_kernel(const float* __restrict__ gathered, int world, int batch, int64_t dl,
                                      float* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = (int64_t)world * batch * dl;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % dl, t = i / dl;
        const int64_t b = t % batch, r = t / batch;
        out[(size_t)b * world * dl + (size_t)r * dl + c] = gathered[i];
    }
}

// ------------------------------------------------------------------------------------------
// Wgu[r][t*2B + j] = j < B ? Wg[r][t*B + j] : Wu[r][t*B + j - B]   (B = kGuBlock)
// ------------------------------------------------------------------------------------------
__global__ void pack_gate_up_kernel(const uint16_t* __restrict__ wg, const uint16_t* __restrict__ wu,
                                    uint16_t* __restrict__ wgu, int64_t d, int64_t inter) {
    constexpr int B = 64;
    const int64_t n = d * 2 * inter;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / (2 * inter), cc = t % (2 * inter);
        const int64_t blk = cc / (2 * B), j = cc % (2 * B);
        wgu[t] = j < B ? wg[r * inter + blk * B + j] : wu[r * inter + blk * B + j - B];
    }
}

}  // namespace larosa

namespace larosa {
// ------------------------------------------------------------------------------------------
// CUDA-core fp32 fold (baseline / fallback for shapes the tensor-core fold does not take):
//   LEFT  : C[i][o] = sum_m Q[m][i] * gamma[m] * W[m][o]     (M = K = d, N = cols)
//   RIGHT : C[r][j] = sum_m W[r][m] * Q[m][j]                (M = rows, N = K = d)
// 64x64 output tile per CTA, K step 16, 256 threads x (4x4) outputs, bf16 RNE store.
// ------------------------------------------------------------------------------------------
// Wf (LEFT only, may be NULL): an fp32 right factor used instead of the bf16 W (the residual
// adapter Q_l^T Q_{l+1} with both factors in fp32).
template <bool LEFT>
__global__ void __launch_bounds__(256) fold_simt_kernel(const float* __restrict__ Q, const float* __restrict__ gamma,
                                                        const uint16_t* __restrict__ W, uint16_t* __restrict__ out,
                                                        int M, int N, int K, const float* __restrict__ Wf) {
    __shared__ float As[16][64 + 4];
    __shared__ float Bs[16][64 + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 64; t += 256) {
            const int kk = t / 64, mm = t % 64;
            const int m = m0 + mm, kg = k0 + kk;
            float av = 0.f, bv = 0.f;
            if (LEFT) {
                // A[m][kg] = Q[kg][m] * gamma[kg]
                if (m < M && kg < K) av = Q[(size_t)kg * M + m] * (gamma ? gamma[kg] : 1.f);
                const int n = n0 + mm;
                if (n < N && kg < K) bv = Wf ? Wf[(size_t)kg * N + n] : bf16f(W[(size_t)kg * N + n]);
            } else {
                if (m < M && kg < K) av = bf16f(W[(size_t)m * K + kg]);
                const int n = n0 + mm;
                if (n < N && kg < K) bv = Q[(size_t)kg * N + n];
            }
            As[kk][mm] = av;
            Bs[kk][mm] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a4[4], b4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a4[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b4[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a4[i], b4[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
            if (m < M && n < N) out[(size_t)m * N + n] = f2bf16_rne(acc[i][j]);
        }
}
// ---- P2P push / wait of the sharded decode step (larosa_peer_push / _shard_wait)
__global__ void peer_push_kernel(const float* __restrict__ src, int batch, int d_local, int64_t src_ld, PeerOut peer) {
    pdl_wait();
    pdl_trigger();
    const int64_t n = (int64_t)batch * d_local;
    unsigned cnt = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(i / d_local), c = (int)(i % d_local);
        peer_put(peer, b, c, src[(size_t)b * src_ld + c]);
    }
    // values stored by this CTA (the grid-stride ranges are disjoint and cover [0, n))
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x)
        cnt += (unsigned)(n - i0 < (int64_t)blockDim.x ? n - i0 : (int64_t)blockDim.x);
    peer_signal(peer, cnt);
}

#ifndef LAROSA_PEER_SLEEP
#define LAROSA_PEER_SLEEP 0
#endif
__global__ void peer_wait_kernel(const uint32_t* flag, uint32_t* expected, uint32_t count) {
    pdl_wait();   // the stream's previous kernel (this rank's own producer) is complete
    if (threadIdx.x == 0) {
        const uint32_t t = *expected + count;
        *expected = t;
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if ((int32_t)(v - t) >= 0) break;
#if LAROSA_PEER_SLEEP
            __nanosleep(LAROSA_PEER_SLEEP);
#endif
        }
    }
    __syncthreads();
    pdl_trigger();
}

}  // namespace larosa
