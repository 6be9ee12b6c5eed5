// Probe: latency of a consumer CTA's first histogram read right after griddepcontrol.wait when the
// previous kernel (PDL-chained) has just written that histogram with atomics (the SELECT GEMV's
// coarse lookup), vs plain stores, vs an untouched region.  Per consumer CTA: %globaltimer after
// the wait and after 8 x 16-byte loads per lane of warp 0 (coarse bins + 3 fine bin ranges) are used.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/atomic_probe tools/atomic_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory"); return t; }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
constexpr int kFine = 65536, kCoarse = 256;
// mode 0: atomics (red coarse + returning atomicAdd fine), 1: plain stores, 2: untouched
__global__ void producer(uint32_t* hist, int mode, int writers, unsigned long long* tend) {
    pdl_wait();
    pdl_trigger();
    // some work so the consumer CTAs are resident and waiting
    unsigned long long t0 = gt();
    while (gt() - t0 < 3000) {}
    if ((int)blockIdx.x < writers && mode != 2) {
        const uint32_t h = (blockIdx.x * 256 + threadIdx.x) * 2654435761u;
        const uint32_t k16 = 0x3e00 + (h >> 24);          // fine bins near one coarse bucket
        if (mode == 0) {
            atomicAdd(hist + kFine + (k16 >> 8), 1u);
            atomicAdd(hist + k16, 1u);
        } else {
            hist[kFine + (k16 >> 8)] = 1u;
            hist[k16] = 1u;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) tend[blockIdx.x] = gt();
}
__global__ void consumer(const uint32_t* hist, unsigned long long* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long t0 = gt();
    pdl_wait();
    unsigned long long t1 = gt();
    uint32_t acc = 0;
    if (warp == 0) {
        const uint4* c = reinterpret_cast<const uint4*>(hist + kFine);
        const uint4* f = reinterpret_cast<const uint4*>(hist + 256 * 0x3e);
        uint4 v[8];
        v[0] = c[lane]; v[1] = c[lane + 32];
        v[2] = f[lane]; v[3] = f[lane + 32]; v[4] = f[lane + 64]; v[5] = f[lane + 96];
        v[6] = f[lane + 128]; v[7] = f[lane + 160];
        for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
        acc = __reduce_add_sync(0xffffffffu, acc);
    }
    unsigned long long t2 = gt();
    if (threadIdx.x == 0) { out[blockIdx.x * 4] = t0; out[blockIdx.x * 4 + 1] = t1; out[blockIdx.x * 4 + 2] = t2; out[blockIdx.x * 4 + 3] = acc; }
}
int main() {
    const int ctas = 288, writers = 16;
    uint32_t* hist; cudaMalloc(&hist, (kFine + kCoarse) * 4 + 4096);
    unsigned long long *out, *tend; cudaMalloc(&out, ctas * 32); cudaMalloc(&tend, ctas * 8);
    cudaStream_t st; cudaStreamCreate(&st);
    std::vector<unsigned long long> h(ctas * 4), he(ctas);
    const char* names[3] = {"atomics", "stores", "untouched"};
    for (int mode = 0; mode < 3; ++mode) {
        std::vector<double> wmed, rmed, rmax, gapmed;
        for (int it = 0; it < 30; ++it) {
            cudaMemsetAsync(hist, 0, (kFine + kCoarse) * 4, st);
            producer<<<ctas, 256, 0, st>>>(hist, mode, writers, tend);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(256); cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, consumer, (const uint32_t*)hist, out);
            cudaStreamSynchronize(st);
            cudaMemcpy(h.data(), out, ctas * 32, cudaMemcpyDeviceToHost);
            cudaMemcpy(he.data(), tend, ctas * 8, cudaMemcpyDeviceToHost);
            unsigned long long pend = *std::max_element(he.begin(), he.end());
            std::vector<double> r, g;
            for (int c = 0; c < ctas; ++c) { r.push_back((double)(h[c * 4 + 2] - h[c * 4 + 1])); g.push_back((double)((long long)h[c * 4 + 1] - (long long)pend)); }
            std::sort(r.begin(), r.end()); std::sort(g.begin(), g.end());
            rmed.push_back(r[ctas / 2]); rmax.push_back(r.back()); gapmed.push_back(g[ctas / 2]);
        }
        std::sort(rmed.begin(), rmed.end()); std::sort(rmax.begin(), rmax.end()); std::sort(gapmed.begin(), gapmed.end());
        printf("%-10s first lookup after the wait: median %.0f ns (max over CTAs %.0f ns); wait release after producer end: %.0f ns\n",
               names[mode], rmed[15], rmax[15], gapmed[15]);
    }
    return 0;
}
