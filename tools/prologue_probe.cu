// Probe: latency of the GEMV select prologue's first step on B200 -- 288 CTAs x 256 threads
// each reading the SAME 16 KB histogram (4 x 16 B per thread) and 16 KB vector (cp.async),
// right after a producer kernel wrote them (atomics / stores).  Per-CTA %globaltimer deltas.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void producer(unsigned* hist, float* x, int mode) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 4096) {
        if (mode == 0) atomicAdd(hist + (i * 7) % 4096, 1u);
        else hist[i] = i;
        x[i] = (float)i;
    }
}

template <int VAR>
__global__ void __launch_bounds__(256) consumer(const unsigned* hist, const float* x, unsigned long long* out) {
    __shared__ __align__(16) float xs[4096];
    const int tid = threadIdx.x;
    unsigned long long t0 = gt();
    if (VAR == 1 || VAR == 3)
        for (int c = tid; c < 1024; c += 256)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(xs + 4 * c)), "l"(x + 4 * c) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    unsigned s = 0;
    const uint4* hp = reinterpret_cast<const uint4*>(hist + 4096 - 16 * (tid + 1));
    if (VAR <= 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) { uint4 v = __ldcg(hp + q); s += v.x + v.y + v.z + v.w; }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) { uint4 v = __ldcg(reinterpret_cast<const uint4*>(hist) + q * 256 + tid); s += v.x + v.y + v.z + v.w; }
    }
    unsigned long long t1 = gt();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    unsigned long long t2 = gt();
    if (tid == 0) {
        const int c = blockIdx.y * gridDim.x + blockIdx.x;
        out[c * 4 + 0] = t0;
        out[c * 4 + 1] = t1;
        out[c * 4 + 2] = t2;
        out[c * 4 + 3] = s + (unsigned)xs[5];
    }
}

int main() {
    unsigned* hist;
    float* x;
    unsigned long long* out;
    cudaMalloc(&hist, 4096 * 4);
    cudaMalloc(&x, 4096 * 4);
    cudaMalloc(&out, 1024 * 32);
    std::vector<unsigned long long> h(1024 * 4);
    for (int mode = 0; mode < 2; ++mode)
        for (int var = 0; var < 4; ++var) {
            std::vector<double> tl, tw;
            for (int rep = 0; rep < 20; ++rep) {
                producer<<<16, 256>>>(hist, x, mode);
                if (var == 0) consumer<0><<<dim3(48, 6), 256>>>(hist, x, out);
                if (var == 1) consumer<1><<<dim3(48, 6), 256>>>(hist, x, out);
                if (var == 2) consumer<2><<<dim3(48, 6), 256>>>(hist, x, out);
                if (var == 3) consumer<3><<<dim3(48, 6), 256>>>(hist, x, out);
                cudaDeviceSynchronize();
                cudaMemcpy(h.data(), out, 288 * 32, cudaMemcpyDeviceToHost);
                if (rep < 3) continue;
                for (int c = 0; c < 288; ++c) {
                    tl.push_back((h[c * 4 + 1] - h[c * 4 + 0]) / 1e3);
                    tw.push_back((h[c * 4 + 2] - h[c * 4 + 0]) / 1e3);
                }
            }
            std::sort(tl.begin(), tl.end());
            std::sort(tw.begin(), tw.end());
            printf("producer %s  var %d (%s%s): hist loads med %.2f us max %.2f | +x wait med %.2f max %.2f\n",
                   mode ? "stores " : "atomics", var, var & 1 ? "cp.async x + " : "", var < 2 ? "thread-contiguous hist" : "coalesced hist",
                   tl[tl.size() / 2], tl.back(), tw[tw.size() / 2], tw.back());
        }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
