// img_layout.cuh — the batch 8-16 token operand ("image") of gemv_img.cuh: per 64-row chunk of a
// site vector, the 16 tokens' values as bf16 hi (MMA rows 0-15) and lo (rows 16-31), K-major with
// the 128-byte swizzle the tcgen05 MMA reads.  Shared by its writers (the Top-K rule kernels, the
// image kernels) and the GEMV.
#pragma once

namespace larosa {

constexpr int kImgChunkBytes = 4096;   // 32 MMA rows (16 hi, 16 lo) x 64 K x bf16
constexpr int kImgChunkK = 64;

// byte offset of value (MMA row n in 0..31, K index k in 0..63) inside a chunk's 4 KB image
__host__ __device__ constexpr int img_off(int n, int k) {
    return (n >> 3) * 1024 + (n & 7) * 128 + ((((k >> 3) ^ (n & 7))) << 4) + (k & 7) * 2;
}
}  // namespace larosa
