// Probe: achieved DRAM read bandwidth of a gathered-row stream on B200 as a function of the
// contiguous segment each warp reads per row (512 B .. 8 KB) and of the in-flight depth.
// Models the sparse GEMV: k kept rows (random, ascending) of a [d_in][ld] bf16 matrix,
// columns split into slices of SEG bytes; grid = slices x splits, one wave.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
template <int N> __device__ __forceinline__ void cpwait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cpcommit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// CH = 16-byte chunks per lane per row (segment = CH * 512 bytes per warp), STAGES rows in flight per warp
template <int CH, int STAGES>
__global__ void __launch_bounds__(256) gather(const char* W, long ld_bytes, const int* rows, int k, int n_splits,
                                              float* out) {
    extern __shared__ __align__(16) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slice = blockIdx.x, split = blockIdx.y;
    const int rps = (k + n_splits - 1) / n_splits;
    const int r0 = split * rps, r1 = min(k, r0 + rps);
    char* ring = sm + warp * (STAGES * CH * 512) + lane * 16;
    const char* base = W + (long)slice * CH * 512 + lane * 16;
    float acc = 0.f;
    // my rows: r0 + warp + 8 m
    const int nm = r1 > r0 + warp ? (r1 - r0 - warp + 7) / 8 : 0;
    for (int s = 0; s < STAGES; ++s) {
        if (s < nm) {
            const char* src = base + (long)rows[r0 + warp + 8 * s] * ld_bytes;
#pragma unroll
            for (int c = 0; c < CH; ++c) cp16(ring + (s * CH + c) * 512, src + c * 512);
        }
        cpcommit();
    }
    for (int m = 0; m < nm; ++m) {
        cpwait<STAGES - 1>();
        const int s = m % STAGES;
#pragma unroll
        for (int c = 0; c < CH; ++c) acc += *reinterpret_cast<const float*>(ring + (s * CH + c) * 512);
        const int mn = m + STAGES;
        if (mn < nm) {
            const char* src = base + (long)rows[r0 + warp + 8 * mn] * ld_bytes;
#pragma unroll
            for (int c = 0; c < CH; ++c) cp16(ring + (s * CH + c) * 512, src + c * 512);
        }
        cpcommit();
    }
    if (acc == 123.456f) out[0] = acc;
}

__global__ void stream_read(const float4* p, long n, float* out) {
    float4 a = make_float4(0, 0, 0, 0);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        float4 v = __ldcs(p + i);
        a.x += v.x;
    }
    if (a.x == 123.456f) out[0] = a.x;
}

template <int CH, int STAGES>
void run(const char* W, long ld_bytes, const int* rows, int k, int d_out_bytes, float* out, int ncopies, long copy_bytes,
         const char* tag) {
    const int slices = d_out_bytes / (CH * 512);
    const size_t smem = 8 * STAGES * CH * 512;
    cudaFuncSetAttribute(gather<CH, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather<CH, STAGES>, 256, smem);
    const int splits = std::max(1, 148 * per_sm / slices);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i)
        gather<CH, STAGES><<<dim3(slices, splits), 256, smem>>>(W + (i % ncopies) * copy_bytes, ld_bytes, rows, k, splits, out);
    cudaEventRecord(e0);
    const int reps = 40;
    for (int i = 0; i < reps; ++i)
        gather<CH, STAGES><<<dim3(slices, splits), 256, smem>>>(W + (i % ncopies) * copy_bytes, ld_bytes, rows, k, splits, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)k * d_out_bytes;
    printf("%-10s seg %5d B  stages %d  ctas/sm %d  grid %3dx%-3d  %.2f us  %.0f GB/s\n", tag, CH * 512, STAGES, per_sm,
           slices, splits, ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9);
}

int main() {
    const int d_in = 11008, d_out = 8192;
    const long ld_bytes = (long)d_out * 2, copy_bytes = (long)d_in * ld_bytes;   // 180 MB per copy
    const int ncopies = 4;
    char* W;
    cudaMalloc(&W, copy_bytes * ncopies);
    cudaMemset(W, 0, copy_bytes * ncopies);
    float* out;
    cudaMalloc(&out, 64);
    for (int kk : {2048, 5504}) {
        std::vector<int> idx(d_in);
        for (int i = 0; i < d_in; ++i) idx[i] = i;
        std::mt19937 g(1);
        std::shuffle(idx.begin(), idx.end(), g);
        idx.resize(kk);
        std::sort(idx.begin(), idx.end());
        int* rows;
        cudaMalloc(&rows, kk * 4);
        cudaMemcpy(rows, idx.data(), kk * 4, cudaMemcpyHostToDevice);
        printf("k = %d rows x %d bytes = %.1f MB\n", kk, d_out * 2, kk * (double)d_out * 2 / 1e6);
        run<1, 4>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        run<1, 8>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        run<2, 4>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        run<4, 2>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        run<4, 4>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        run<8, 2>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        run<16, 1>(W, ld_bytes, rows, kk, d_out * 2, out, ncopies, copy_bytes, "gather");
        cudaFree(rows);
    }
    // plain contiguous read
    for (long mb : {16L, 48L, 96L, 512L}) {
        const long n = mb * 1000000 / 16;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int i = 0; i < 3; ++i) stream_read<<<148 * 8, 256>>>((const float4*)(W + (i % ncopies) * copy_bytes), n, out);
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) stream_read<<<148 * 8, 256>>>((const float4*)(W + (i % ncopies) * copy_bytes), n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("stream read %4ld MB: %.2f us  %.0f GB/s\n", mb, ms * 1e3 / 20, n * 16.0 / (ms * 1e-3 / 20) / 1e9);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
