// Probe: latency of 3 dependent 1 KB warp reads (like the SELECT rule's coarse -> fine -> pool
// lookups) when N CTAs read the SAME lines at the same time, vs private lines per CTA.
// Per-CTA %globaltimer deltas (ns), median / max over CTAs.   nvcc -arch=sm_100a -O3
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void producer(unsigned* buf, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(buf + i, 1u);
}

// mode 0: all CTAs read the same 3 KB; mode 1: CTA c reads its own copy (stride 64 KB)
__global__ void __launch_bounds__(256) consumer(const unsigned* buf, unsigned long long* out, int mode, int active) {
    if ((int)blockIdx.x >= active) return;
    __shared__ unsigned sink;
    const int lane = threadIdx.x & 31;
    const unsigned* base = buf + (mode ? (size_t)blockIdx.x * 16384 : 0);
    unsigned long long t0 = gt();
    unsigned long long t[4];
    t[0] = t0;
    if (threadIdx.x < 32) {
        int off = 0;
        for (int r = 0; r < 3; ++r) {
            const uint4* p = reinterpret_cast<const uint4*>(base + 256 * r + off + 8 * lane);
            uint4 a = __ldca(p), b = __ldca(p + 1);
            unsigned s = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
            #pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            off = (s & 1) * 0;   // dependent address (always 0) so the reads serialise
            off += (int)(s >> 31);
            t[r + 1] = gt();
        }
        if (lane == 0) sink = off;
    }
    __syncthreads();
    if (threadIdx.x == 0) for (int r = 0; r < 4; ++r) out[blockIdx.x * 4 + r] = t[r] - (r ? 0 : 0);
}

int main() {
    unsigned* buf; unsigned long long* out;
    const int ncta = 296;
    cudaMalloc(&buf, sizeof(unsigned) * 16384 * ncta);
    cudaMemset(buf, 0, sizeof(unsigned) * 16384 * ncta);
    cudaMalloc(&out, sizeof(unsigned long long) * 4 * ncta);
    std::vector<unsigned long long> h(4 * ncta);
    for (int mode = 0; mode < 2; ++mode) {
        for (int active : {1, 16, 74, 148, 296}) {
            std::vector<double> d1, d2, d3;
            for (int rep = 0; rep < 20; ++rep) {
                producer<<<148, 256>>>(buf, mode ? 16384 * ncta : 4096);
                consumer<<<ncta, 256>>>(buf, out, mode, active);
                cudaDeviceSynchronize();
                cudaMemcpy(h.data(), out, sizeof(unsigned long long) * 4 * ncta, cudaMemcpyDeviceToHost);
                for (int c = 0; c < active; ++c) {
                    d1.push_back((double)(h[4 * c + 1] - h[4 * c]));
                    d2.push_back((double)(h[4 * c + 2] - h[4 * c + 1]));
                    d3.push_back((double)(h[4 * c + 3] - h[4 * c + 2]));
                }
            }
            auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
            auto mx = [](std::vector<double> v) { return *std::max_element(v.begin(), v.end()); };
            printf("mode %s active %3d: rt1 %6.0f/%6.0f  rt2 %6.0f/%6.0f  rt3 %6.0f/%6.0f ns (med/max)\n",
                   mode ? "private" : "shared ", active, med(d1), mx(d1), med(d2), mx(d2), med(d3), mx(d3));
        }
    }
    return 0;
}
