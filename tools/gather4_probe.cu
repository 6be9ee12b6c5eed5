// Probe: streaming gathered weight rows (512-byte segments of 256 bf16 columns) into shared
// memory on B200 -- TMA tile::gather4 (4 rows per instruction, one issuing thread, mbarrier
// ring) vs per-warp LDGSTS rings (the current GEMV stream).  Grid = 16 slices x 18 splits
// (2 CTAs / SM), W = [16384][4096] bf16 (128 MB >> L2), k kept rows (random, ascending) per
// call.  Reports GB/s of row bytes.   nvcc -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, int bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, int ph) {
    asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}

constexpr int NT = 256, STAGES = 32, ROWS_PER_STAGE = 4, COLS = 256;
constexpr int STAGE_BYTES = ROWS_PER_STAGE * COLS * 2;

__global__ void __launch_bounds__(NT) k_gather4(const __grid_constant__ CUtensorMap tm, const int* rows, int nrows,
                                                int n_splits, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    const int slice = blockIdx.x, split = blockIdx.y;
    const int per = (nrows + n_splits - 1) / n_splits;
    const int r0 = min(nrows, split * per), r1 = min(nrows, r0 + per);
    const int nst = (r1 - r0 + ROWS_PER_STAGE - 1) / ROWS_PER_STAGE;
    int* srows = reinterpret_cast<int*>(empty + STAGES);
    for (int i = threadIdx.x; i < r1 - r0; i += NT) srows[i] = rows[r0 + i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], NT / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    if (threadIdx.x == 0) {   // producer (also consumes as part of warp 0 below? keep it simple: issue ahead)
        for (int st = 0; st < min(nst, STAGES); ++st) {
            int rr[4];
            for (int g = 0; g < 4; ++g) rr[g] = srows[min(r1 - r0 - 1, 4 * st + g)];
            mb_expect(&full[st], STAGE_BYTES);
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                ::"r"(su32(sm + st * STAGE_BYTES)), "l"(&tm), "r"(slice * COLS), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]), "r"(su32(&full[st])) : "memory");
        }
    }
    for (int st = 0; st < nst; ++st) {
        const int s = st % STAGES, ph = (st / STAGES) & 1;
        mb_wait(&full[s], ph);
        const uint4 v = *reinterpret_cast<const uint4*>(sm + s * STAGE_BYTES + threadIdx.x * 8);
        acc += __uint_as_float(v.x << 16) + __uint_as_float(v.w & 0xffff0000u);
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mb_arrive(&empty[s]);
        if (threadIdx.x == 0 && st + STAGES < nst) {
            const int nx = st + STAGES;
            mb_wait(&empty[s], ph);
            int rr[4];
            for (int g = 0; g < 4; ++g) rr[g] = srows[min(r1 - r0 - 1, 4 * nx + g)];
            mb_expect(&full[s], STAGE_BYTES);
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                ::"r"(su32(sm + s * STAGE_BYTES)), "l"(&tm), "r"(slice * COLS), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]), "r"(su32(&full[s])) : "memory");
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

// the current design: per-warp rings of LDGSTS (warp w takes rows w, w+8, ...), 4 stages x 4 rows
__global__ void __launch_bounds__(NT) k_ldgsts(const uint16_t* W, int ld, const int* rows, int nrows, int n_splits,
                                               float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int slice = blockIdx.x, split = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per = (nrows + n_splits - 1) / n_splits;
    const int r0 = min(nrows, split * per), r1 = min(nrows, r0 + per);
    const int n = r1 - r0;
    const int n_my = n > warp ? (n - warp + 7) / 8 : 0;
    const int n_st = (n_my + 3) / 4;
    unsigned char* ring = sm + warp * 8192 + lane * 16;
    int* srows = reinterpret_cast<int*>(sm + 65536);
    for (int i = threadIdx.x; i < n; i += NT) srows[i] = rows[r0 + i];
    __syncthreads();
    const uint16_t* wc = W + slice * COLS + lane * 8;
    auto issue = [&](int st) {
        if (st < n_st)
            for (int g = 0; g < 4; ++g) {
                const int m = 4 * st + g;
                const int row = m < n_my ? srows[warp + 8 * m] : 0;
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}"
                    ::"r"(su32(ring + (st & 3) * 2048 + g * 512)), "l"(wc + (size_t)row * ld), "r"((int)(m < n_my)) : "memory");
            }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int st = 0; st < 4; ++st) issue(st);
    float acc = 0.f;
    for (int st = 0; st < n_st; ++st) {
        asm volatile("cp.async.wait_group 3;" ::: "memory");
        for (int g = 0; g < 4; ++g) {
            if (4 * st + g >= n_my) break;
            const uint4 v = *reinterpret_cast<const uint4*>(ring + (st & 3) * 2048 + g * 512);
            acc += __uint_as_float(v.x << 16) + __uint_as_float(v.w & 0xffff0000u);
        }
        issue(st + 4);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (acc == 12345.f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int D_IN = 16384, LD = 4096, NSL = 16;
    uint16_t* W;
    cudaMalloc(&W, (size_t)D_IN * LD * 2);
    cudaMemset(W, 0x3c, (size_t)D_IN * LD * 2);
    float* out;
    cudaMalloc(&out, 64);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)LD, (cuuint64_t)D_IN};
    cuuint64_t strides[1] = {(cuuint64_t)LD * 2};
    cuuint32_t box[2] = {COLS, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    std::mt19937 rng(1);
    const int reps = 20;
    for (int k : {2048, 4096, 8192}) {
        std::vector<int*> drows(reps);
        for (int t = 0; t < reps; ++t) {
            std::vector<int> all(D_IN);
            for (int i = 0; i < D_IN; ++i) all[i] = i;
            std::shuffle(all.begin(), all.end(), rng);
            std::vector<int> sel(all.begin(), all.begin() + k);
            std::sort(sel.begin(), sel.end());
            cudaMalloc(&drows[t], k * 4);
            cudaMemcpy(drows[t], sel.data(), k * 4, cudaMemcpyHostToDevice);
        }
        for (int splits : {9, 18}) {
            const size_t smg = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 4096 * 4;
            cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, 110000);
            cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int variant = 0; variant < 2; ++variant) {
                for (int w = 0; w < 2; ++w) {   // warm + timed
                    cudaEventRecord(e0);
                    for (int t = 0; t < reps; ++t) {
                        if (variant == 0) k_gather4<<<dim3(NSL, splits), NT, smg>>>(tm, drows[t], k, splits, out);
                        else k_ldgsts<<<dim3(NSL, splits), NT, 65536 + 4096 * 4>>>(W, LD, drows[t], k, splits, out);
                    }
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)k * LD * 2 * reps;
                printf("k=%5d splits=%2d %-8s: %.2f us/call, %.0f GB/s  (err %s)\n", k, splits,
                       variant == 0 ? "gather4" : "ldgsts", ms * 1e3 / reps, bytes / (ms * 1e-3) / 1e9,
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
