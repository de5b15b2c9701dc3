// tma_stream.cu -- streaming throughput of a once-read HBM buffer into shared
// memory: cp.async.bulk (TMA) rings of S slots x B bytes per CTA, one CTA per
// SM, versus LDG.128 by all threads; optional per-lane L2 prefetch ahead.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_stream tma_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_tma(const char *src, size_t total, int slots, int chunk, int pf, unsigned *sink)
{
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[16];
    const size_t per = total / gridDim.x / 65536 * 65536;
    const char *base = src + per * blockIdx.x;
    const int n = (int)(per / chunk);
    if (threadIdx.x == 0) {
        for (int i = 0; i < slots; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned acc = 0;
    auto issue = [&](int k) {
        const int s = k % slots;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(sm + (size_t)s * chunk)), "l"(base + (size_t)k * chunk), "r"(chunk), "r"(sa(&bar[s])) : "memory");
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < slots - 1 && k < n; ++k) issue(k);
    for (int k = 0; k < n; ++k) {
        if (pf && threadIdx.x < 32 && k + pf < n) {
            const char *b = base + (size_t)(k + pf) * chunk;
            for (int o = threadIdx.x * 128; o < chunk; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(b + o));
        }
        if (threadIdx.x == 0 && k + slots - 1 < n) issue(k + slots - 1);
        const int s = k % slots;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(sa(&bar[s])), "r"((k / slots) & 1) : "memory");
        acc += ((const unsigned *)(sm + (size_t)s * chunk))[threadIdx.x];
        __syncthreads();  // slot s free before it is refilled
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_ldg(const uint4 *src, size_t n4, unsigned *sink)
{
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(src + i);
        acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main()
{
    const size_t total = 1ull << 30;
    char *buf;
    unsigned *sink;
    CK(cudaMalloc(&buf, total));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 1, total));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    struct { int slots, chunk, pf, threads; } cfgs[] = {
        {2, 16384, 0, 128}, {4, 16384, 0, 128}, {8, 16384, 0, 128}, {12, 16384, 0, 128},
        {4, 16384, 8, 128}, {4, 32768, 0, 128}, {6, 32768, 0, 128}, {3, 49152, 0, 128}, {8, 8192, 0, 128},
        {12, 8192, 0, 128}, {16, 8192, 0, 128}};
    for (auto c : cfgs) {
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            k_tma<<<sms, c.threads, (size_t)c.slots * c.chunk>>>(buf, total, c.slots, c.chunk, c.pf, sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("tma slots=%2d chunk=%6d pf=%d: %.3f ms  %.0f GB/s  (%d KB in flight per SM)\n", c.slots, c.chunk, c.pf,
               best, total / best / 1e6, (c.slots - 1) * c.chunk / 1024);
    }
    for (int bs : {256, 512, 1024}) {
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            k_ldg<<<sms * (2048 / bs), bs>>>((const uint4 *)buf, total / 16, sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("ldg.128 bs=%d: %.3f ms  %.0f GB/s\n", bs, best, total / best / 1e6);
    }
    return 0;
}
