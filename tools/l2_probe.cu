// Probe: latency of the "ticket + last CTA reads the global histogram" pattern on B200.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long clk() { return clock64(); }

__global__ void k_ticket(unsigned* gh, unsigned* ticket, unsigned long long* out, int mode) {
    __shared__ int last;
    const int tid = threadIdx.x;
    // each CTA adds into ~150 bins
    if (mode >= 1)
        for (int i = tid; i < 4096; i += 256)
            if ((i % 27) == 0) atomicAdd(&gh[i], 1u);
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    unsigned long long t0 = clk();
    unsigned v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __ldcg(gh + tid * 16 + q);
    unsigned s = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += v[q];
    unsigned long long t1 = clk();
    __syncthreads();
    unsigned long long t2 = clk();
    unsigned v2[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v2[q] = __ldcg(gh + q * 256 + tid);
    for (int q = 0; q < 16; ++q) s += v2[q];
    unsigned long long t3 = clk();
    unsigned long long t4 = clk();
    __threadfence();
    unsigned long long t5 = clk();
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    unsigned long long t6 = clk();
    if (tid == 0) {
        out[3] = t5 - t4;
        out[4] = t6 - t5;
        out[0] = t1 - t0;
        out[1] = t3 - t2;
        out[2] = s;
        *ticket = 0;
    }
    for (int i = tid; i < 4096; i += 256) gh[i] = 0;
}

int main() {
    unsigned *gh, *tk;
    unsigned long long* out;
    cudaMalloc(&gh, 4096 * 4);
    cudaMalloc(&tk, 4);
    cudaMalloc(&out, 64);
    cudaMemset(gh, 0, 4096 * 4);
    cudaMemset(tk, 0, 4);
    unsigned long long h[5];
    for (int mode = 0; mode < 2; ++mode)
        for (int grid : {1, 4, 16}) {
            for (int r = 0; r < 3; ++r) k_ticket<<<grid, 256>>>(gh, tk, out, mode);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost);
            printf("mode %d grid %2d: 16 x strided ldcg+sum %llu cyc, 16 x coalesced ldcg+sum %llu cyc, threadfence %llu, fence.acq_rel %llu\n", mode, grid, h[0], h[1], h[3], h[4]);
        }
    return 0;
}
