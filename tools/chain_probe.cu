// Chain-latency probe: back-to-back dependent launches (PDL on/off, CUDA graph) of
// tiny kernels with various CTA shapes.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) p[0] += 1;
}

__global__ void k_sync(int* p, int nsync) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ int s[1024];
    int v = threadIdx.x;
    for (int i = 0; i < nsync; ++i) {
        s[threadIdx.x] = v;
        __syncthreads();
        v += s[(threadIdx.x + 1) % blockDim.x];
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) p[0] += v;
}

__global__ void k_load(const float* x, float* y, int n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    float a = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a += __ldcg(x + i);
    if (a == 12345.f) y[0] = a;
}

__global__ void k_csync(int* p, int n) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int i = 0; i < n; ++i)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) p[0] += 1;
}

template <typename F>
float time_chain(F launch, int n, bool graph) {
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int i = 0; i < 10; ++i) launch(st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    if (graph) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < n; ++i) launch(st);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
    } else {
        cudaEventRecord(a, st);
        for (int i = 0; i < n; ++i) launch(st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    return ms * 1000.f / n;
}

template <typename... KA, typename... A>
void launch_ex(void (*k)(KA...), dim3 g, dim3 b, cudaStream_t st, bool pdl, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, args...);
}
template <typename... KA, typename... A>
void launch_cl(void (*k)(KA...), int cs, dim3 b, cudaStream_t st, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = b;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cs;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, k, args...);
}

int main() {
    int* p;
    cudaMalloc(&p, 4096);
    float *x, *y;
    cudaMalloc(&x, 1 << 20);
    cudaMalloc(&y, 4096);
    cudaMemset(x, 0, 1 << 20);
    const int N = 200;
    for (int cs : {1, 2, 4, 8}) {
        for (int nt : {128, 512, 1024}) {
            for (int ns : {0, 10, 40}) {
                float us = time_chain([&](cudaStream_t st) { launch_cl(k_csync, cs, dim3(nt), st, p, ns); }, N, true);
                printf("cluster %d x %4d thr, %2d cluster syncs: %6.2f us\n", cs, nt, ns, us);
            }
        }
    }
    for (int pdl = 0; pdl < 2; ++pdl) {
        for (int graph = 0; graph < 2; ++graph) {
            printf("pdl=%d graph=%d\n", pdl, graph);
            int shapes[][2] = {{1, 32}, {1, 128}, {1, 1024}, {148, 256}, {296, 256}, {16, 1024}};
            for (auto& sh : shapes) {
                float us = time_chain([&](cudaStream_t st) { launch_ex(k_empty, dim3(sh[0]), dim3(sh[1]), st, pdl, p); },
                                      N, graph);
                printf("  empty  grid %4d x %4d : %6.2f us/launch\n", sh[0], sh[1], us);
            }
            for (int ns : {4, 16}) {
                float us = time_chain([&](cudaStream_t st) { launch_ex(k_sync, dim3(1), dim3(1024), st, pdl, p, ns); },
                                      N, graph);
                printf("  1x1024 with %2d x 2 syncthreads: %6.2f us\n", ns, us);
            }
            for (int n : {4096, 11008, 44032}) {
                float us = time_chain(
                    [&](cudaStream_t st) { launch_ex(k_load, dim3(1), dim3(1024), st, pdl, (const float*)x, y, n); }, N,
                    graph);
                printf("  1x1024 load %6d floats: %6.2f us\n", n, us);
            }
        }
    }
    return 0;
}
