// Probe: latency of a chain of DEPENDENT global loads (pointer chase) by one thread, on lines
// written by the previous kernel with (a) atomics from many SMs, (b) plain stores from many
// SMs, (c) untouched since a long time; ld.global.cg vs ld.global (default) vs ld.relaxed.gpu.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void writer(unsigned* buf, int n, int mode) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned next = (unsigned)((i * 97 + 13) % n);   // a permutation cycle-ish chain
        if (mode == 0) { atomicExch(buf + i, next); }
        else if (mode == 1) { buf[i] = next; }
    }
}

template <int LD>
__global__ void chaser(const unsigned* buf, int steps, unsigned long long* out) {
    unsigned p = 0;
    const long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        unsigned v;
        if (LD == 0) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(buf + p));
        else if (LD == 1) asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(buf + p));
        else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(buf + p));
        p = v;
    }
    const long long t1 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = p;
}

int main() {
    const int n = 1 << 16;   // 256 KB
    unsigned* buf;
    unsigned long long* out;
    cudaMalloc(&buf, n * 4);
    cudaMalloc(&out, 16);
    unsigned long long h[2];
    const char* wname[3] = {"atomics", "stores ", "stale  "};
    const char* lname[3] = {"ld.cg", "ld   ", "ld.relaxed.gpu"};
    for (int wm = 0; wm < 3; ++wm)
        for (int ld = 0; ld < 3; ++ld) {
            if (wm < 2) writer<<<296, 256>>>(buf, n, wm);
            else { writer<<<296, 256>>>(buf, n, 1); cudaDeviceSynchronize(); }
            if (ld == 0) chaser<0><<<1, 1>>>(buf, 64, out);
            if (ld == 1) chaser<1><<<1, 1>>>(buf, 64, out);
            if (ld == 2) chaser<2><<<1, 1>>>(buf, 64, out);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
            printf("written by %s, %s: %.0f cycles per dependent load (%.2f us at 1.965 GHz)\n", wname[wm], lname[ld],
                   h[0] / 64.0, h[0] / 64.0 / 1965.0);
        }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
