// Probe: latency of loads issued by the LAST CTA of a kernel (ticket pattern) on lines that
// other CTAs of the same kernel just updated with atomics / stores.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned atom_acq_rel(unsigned* p) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}

template <int MODE>
__global__ void k(unsigned* hist, unsigned* ticket, unsigned* other, long long* out) {
    __shared__ int last;
    const int tid = threadIdx.x;
    // every CTA: 256 updates into a 64K-word array (random-ish bins)
    const unsigned bin = (blockIdx.x * 2654435761u + tid * 40503u) & 0xffffu;
    if (MODE == 0) atomicAdd(hist + bin, 1u);
    else if (MODE == 1) hist[bin] = tid;
    else if (MODE == 2) atomicAdd(other + bin, 1u);      // unrelated lines
    __syncthreads();
    if (tid == 0) last = atom_acq_rel(ticket) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    if (tid == 0) *ticket = 0;
    if (tid < 32) {
        long long t0 = clock64();
        unsigned p = tid;
        for (int s = 0; s < 16; ++s) {   // dependent loads over the updated array
            unsigned v;
            asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(hist + ((p * 977u + s * 131u) & 0xffffu)));
            p += v & 1;
        }
        long long t1 = clock64();
        if (tid == 0) { out[0] = (t1 - t0) / 16; out[1] = p; }
    }
}

int main() {
    unsigned *hist, *ticket, *other;
    long long* out;
    cudaMalloc(&hist, 65536 * 4);
    cudaMalloc(&other, 65536 * 4);
    cudaMalloc(&ticket, 4);
    cudaMalloc(&out, 16);
    cudaMemset(hist, 0, 65536 * 4);
    cudaMemset(ticket, 0, 4);
    long long h[2];
    const char* names[3] = {"atomics on the same lines", "stores on the same lines", "atomics on other lines"};
    for (int m = 0; m < 3; ++m) {
        for (int rep = 0; rep < 3; ++rep) {
            if (m == 0) k<0><<<288, 256>>>(hist, ticket, other, out);
            if (m == 1) k<1><<<288, 256>>>(hist, ticket, other, out);
            if (m == 2) k<2><<<288, 256>>>(hist, ticket, other, out);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("%s: %lld cycles per dependent load in the last CTA\n", names[m], h[0]);
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
