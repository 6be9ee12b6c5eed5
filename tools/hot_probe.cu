// Probe: latency of the first dependent loads of a freshly released CTA when 288 CTAs (2 per SM)
// read the SAME small region (the consumer's histogram lookup) vs a private replica per CTA or per
// 8 CTAs.  Each CTA: spin until a start flag (set by a host-side memset after all CTAs are resident
// is not possible -- instead CTA 0 thread 0 sets it after a delay), then warp 0 loads 4 KB (256
// words per lane group, as load256 x 4) and records %globaltimer before / after.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long clk() { unsigned long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) :: "memory"); return t; }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void probe(const uint32_t* __restrict__ buf, int replicas, int bytes, volatile int* flag, unsigned long long* out, int mode) {
    __shared__ uint32_t sink[32];
    (void)sink;
    const int cta = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (cta == 0 && threadIdx.x == 0) {
        unsigned long long t0 = gt();
        while (gt() - t0 < 20000) {}
        __threadfence();
        *flag = 1;
    }
    if (threadIdx.x == 0) while (*flag == 0) {}
    __syncthreads();
    unsigned long long t1 = clk();
    const int rep = replicas > 0 ? cta % replicas : 0;
    const uint32_t* b = buf + (size_t)rep * (bytes / 4);
    uint32_t acc = 0;
    if (warp == 0) {
        const int words = bytes / 4;
        for (int i = lane * 4; i < words; i += 128) {
            uint4 v;
            if (mode == 0) v = __ldca(reinterpret_cast<const uint4*>(b + i));
            else v = __ldcg(reinterpret_cast<const uint4*>(b + i));
            acc += v.x + v.y + v.z + v.w;
        }
        acc = __reduce_add_sync(0xffffffffu, acc);
    }
    asm volatile("" ::"r"(acc) : "memory");
    unsigned long long t2 = clk();
    if (warp == 0 && lane == 0) { out[cta * 2] = t1; out[cta * 2 + 1] = t2; out[2 * gridDim.x + cta] = acc; }
}
int main() {
    const int ctas = 288;
    uint32_t* buf; cudaMalloc(&buf, 64 << 20); cudaMemset(buf, 1, 64 << 20);
    int* flag; cudaMalloc(&flag, 4);
    unsigned long long* out; cudaMalloc(&out, ctas * 24);
    std::vector<unsigned long long> h(ctas * 2);
    for (int bytes : {1024, 4096, 16384}) for (int mode : {0, 1}) for (int rep : {0, 2, 8, 36, 288}) {
        std::vector<double> meds, maxs;
        for (int it = 0; it < 20; ++it) {
            cudaMemset(flag, 0, 4);
            probe<<<ctas, 256>>>(buf, rep, bytes, flag, out, mode);
            cudaDeviceSynchronize();
            cudaMemcpy(h.data(), out, ctas * 16, cudaMemcpyDeviceToHost);
            std::vector<double> d;
            for (int c = 0; c < ctas; ++c) d.push_back((h[c * 2 + 1] - h[c * 2]) / 1965.0);
            std::sort(d.begin(), d.end());
            meds.push_back(d[ctas / 2]); maxs.push_back(d.back());
        }
        std::sort(meds.begin(), meds.end()); std::sort(maxs.begin(), maxs.end());
        printf("bytes %6d %s replicas %3d: median CTA %.3f us, max CTA %.3f us\n", bytes, mode ? "ldcg" : "ldca", rep, meds[10], maxs[10]);
    }
    return 0;
}
