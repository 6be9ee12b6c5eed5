// Probe: cost of a loop of dependent shared-memory accesses whose address is recomputed from
// SR_CgaCtaId each iteration (generic -> shared conversion) vs a hoisted 32-bit shared address.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k_generic(int n, long long* out, int* sink) {
    extern __shared__ unsigned char sm[];
    unsigned short* xs = reinterpret_cast<unsigned short*>(sm);
    unsigned* wm = reinterpret_cast<unsigned*>(sm + 4096);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) xs[i] = i * 7;
    __syncthreads();
    long long t0 = clock64();
    unsigned acc = 0;
    for (int j = threadIdx.x >> 5; j < n; j += 8) {
        unsigned k = xs[(32 * j + (threadIdx.x & 31)) & 2047] + acc;
        unsigned m = __ballot_sync(0xffffffffu, k & 1);
        if ((threadIdx.x & 31) == 0) wm[j & 255] = m;
        acc += m & 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345) sink[0] = acc;
}
__global__ void k_hoisted(int n, long long* out, int* sink) {
    extern __shared__ unsigned char sm[];
    unsigned base;
    asm volatile("mov.u32 %0, %1;" : "=r"(base) : "r"(su32(sm)));
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) reinterpret_cast<unsigned short*>(sm)[i] = i * 7;
    __syncthreads();
    long long t0 = clock64();
    unsigned acc = 0;
    for (int j = threadIdx.x >> 5; j < n; j += 8) {
        unsigned k;
        unsigned a = base + 2u * ((32 * j + (threadIdx.x & 31)) & 2047);
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(k) : "r"(a));
        k += acc;
        unsigned m = __ballot_sync(0xffffffffu, k & 1);
        if ((threadIdx.x & 31) == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(base + 4096u + 4u * (j & 255)), "r"(m));
        acc += m & 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345) sink[0] = acc;
}
int main() {
    long long* out; int* sink; long long h[4];
    cudaMalloc(&out, 64); cudaMalloc(&sink, 64);
    for (int n : {8, 48, 400}) {
        k_generic<<<1, 256, 8192>>>(n, out, sink); cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        long long g = h[0];
        k_hoisted<<<1, 256, 8192>>>(n, out, sink); cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("n=%d words: generic %lld cyc, hoisted %lld cyc\n", n, g, h[0]);
    }
    return 0;
}
