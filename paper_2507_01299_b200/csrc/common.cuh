// common.cuh — device helpers shared by the LaRoSA sm_100a kernels (inline PTX wrappers
// for mbarrier / bulk async copies / programmatic dependent launch, bf16 unpacking,
// deterministic block reductions and scans).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef __CUDACC__
#error "compile with nvcc"
#endif

namespace larosa {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- bf16 <-> fp32 (bf16 is the high half of an IEEE float) ---------------------------
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ float bf16f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t f2bf16_rne(float f) {
    // round-to-nearest-even; inputs are finite on this path
    uint32_t u = __float_as_uint(f);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// ---- programmatic dependent launch (PDL) ------------------------------------------------
// wait: block until the preceding kernel in the stream has completed and flushed memory
// (no-op when the kernel was launched without the PDL attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// trigger: allow the next kernel in the stream to start its prologue early.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- peer push of a sharded phase's output ----------------------------------
// The producing kernel stores every output value straight into every rank's gathered buffer (peer
// device memory over NVLink, e.g. torch symmetric memory) and then adds the number of values it
// wrote to every rank's arrival counter (release, system scope); the consumer waits until its
// counter reaches batch x the full width (larosa_shard_wait).  n = 0: off.
struct PeerOut {
    const unsigned long long* dst;    // [n] device addresses: rank p's buffer, at this rank's column 0
    const unsigned long long* flag;   // [n] device addresses: rank p's uint32 arrival counter
    int n;
    int ld;                           // token stride of the gathered buffers (floats): the full width
};
__device__ __forceinline__ void peer_put(const PeerOut& P, int b, int col, float v) {
    for (int q = 0; q < P.n; ++q) reinterpret_cast<float*>(P.dst[q])[(size_t)b * P.ld + col] = v;
}
// called by EVERY thread of the CTA after all of its peer_put calls; cnt = values the CTA wrote
#ifndef LAROSA_PEER_FENCE
#define LAROSA_PEER_FENCE 0   // 1: every thread also fences its own stores (fence.acq_rel.sys)
#endif
__device__ __forceinline__ void peer_signal(const PeerOut& P, unsigned cnt) {
    if (P.n == 0) return;
    if (LAROSA_PEER_FENCE) asm volatile("fence.acq_rel.sys;" ::: "memory");
    // the CTA barrier puts every thread's stores before thread 0's release in causality order, and
    // a release is cumulative (the arrive pattern of a grid barrier: bar.sync, then one red.release)
    __syncthreads();
    if (threadIdx.x == 0 && cnt)
        for (int q = 0; q < P.n; ++q)
            asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(P.flag[q]), "r"(cnt) : "memory");
}

// the push of a finalised column block [col0, col0 + ncols) x batch of `out` (written by this
// CTA; thread t re-reads column col0 + t, t < ncols <= blockDim.x) + the signal; out of line so
// the hot kernels' register allocation does not see it.  Every thread of the CTA calls it.
__device__ __noinline__ void peer_push_cols(const PeerOut P, const float* out, int64_t out_ld, int batch, int col0,
                                            int ncols) {
    __syncthreads();   // the block's writes of `out` are visible to all of its threads
    const int t = threadIdx.x;
    if (t < ncols)
        for (int b = 0; b < batch; ++b) peer_put(P, b, col0 + t, out[(size_t)b * out_ld + col0 + t]);
    peer_signal(P, (unsigned)(batch * (ncols > 0 ? ncols : 0)));
}

// ---- debug timeline (profiling aid; null pointer = off) -----------------------------------
// Per CTA (linear id c < 1024): tl[c * 16 + i] = %globaltimer (ns) at point i: 0 entry, 1 after
// griddepcontrol.wait, 2 after the prologue, 3 after the main loop, 4 exit.
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_stamp(unsigned long long* tl, int i) {
    if (tl && threadIdx.x == 0) {
        const int c = blockIdx.y * gridDim.x + blockIdx.x;
        if (c < 1024) tl[c * 16 + i] = gtime();
    }
}

// the same, from whichever single thread calls it
__device__ __forceinline__ void tl_stamp_any(unsigned long long* tl, int i) {
    if (tl) {
        const int c = blockIdx.y * gridDim.x + blockIdx.x;
        if (c < 1024) tl[c * 16 + i] = gtime();
    }
}

// ---- thread-block clusters / distributed shared memory -----------------------------------
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `local` (this CTA's shared memory) in cluster CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(const void* local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
    return r;
}
__device__ __forceinline__ float dsmem_ld_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// ---- fences ---------------------------------------------------------------------------------
// acquire-release fence at GPU scope (the ticket / last-CTA patterns need no more than
// this; __threadfence() is a sequentially consistent fence, ~3x slower on B200)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ---- mbarrier ----------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ---- bulk async copy global -> shared (TMA engine, non-tensor; SASS UBLKCP) -------------
// L2 evict-first policy for streamed weights so activations/partials stay L2-resident.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}

// ---- deterministic warp / block primitives ------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Exclusive block scan over one int per thread (NT threads, NT % 32 == 0).  `sw` must hold
// NT/32 + 1 ints.  Returns the exclusive prefix; *total gets the block total.  Contains two
// __syncthreads(); every thread of the block must call it.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* sw, int* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = warp_incl_scan(v);
    if (lane == 31) sw[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int t = lane < NW ? sw[lane] : 0;
        int ti = warp_incl_scan(t);
        if (lane < NW) sw[lane] = ti - t;
        if (lane == NW - 1) sw[NW] = ti;
    }
    __syncthreads();
    int r = sw[wid] + inc - v;
    *total = sw[NW];
    return r;
}

// Deterministic block sum of one float per thread (fixed tree order).  `sw` >= NT/32 floats.
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* sw) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sw[wid] = v;
    __syncthreads();
    float t = 0.f;
    if (wid == 0) {
        t = lane < NW ? sw[lane] : 0.f;
        t = warp_sum(t);
        if (lane == 0) sw[0] = t;
    }
    __syncthreads();
    return sw[0];
}

}  // namespace larosa
