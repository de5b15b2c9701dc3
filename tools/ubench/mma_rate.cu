// mma_rate.cu -- tcgen05.mma issue/execute rate on B200 for the binned
// products' shapes: kind::tf32 (K=8) vs kind::f16 (K=16), A from TMEM (TS)
// vs shared memory (SS), M=128, N in {64, 96}.  One CTA per SM, one issuing
// thread, groups of G MMAs per commit, double-buffered accumulators.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma_rate mma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
            return 1;                                                               \
        }                                                                           \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(bool f16, int m, int n)
{
    return (1u << 4) | ((f16 ? 0u : 2u) << 7) | ((f16 ? 0u : 2u) << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}

template <bool F16, bool TS>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a_tmem, uint64_t a_desc, uint64_t b, uint32_t id, uint32_t acc)
{
    if (F16) {
        if (TS)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                         "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
        else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                         "l"(a_desc), "l"(b), "r"(id), "r"(acc));
    } else {
        if (TS)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                         "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
        else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                         "l"(a_desc), "l"(b), "r"(id), "r"(acc));
    }
}

__device__ __forceinline__ void bar_init(uint64_t *b, unsigned c)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned par)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
}

template <bool F16, bool TS, int N, int ISSUERS = 1>
__global__ void __launch_bounds__(128, 1) k_rate(int groups, int G, unsigned long long *cyc)
{
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t done[2][2];
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        bar_init(&done[0][0], 1);
        bar_init(&done[0][1], 1);
        bar_init(&done[1][0], 1);
        bar_init(&done[1][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const int who = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && who < ISSUERS) {
        const uint32_t id = idesc(F16, 128, N);
        const uint64_t a = sdesc(sa(sm)), bb = sdesc(sa(sm + 32768));
        const int NB = TS ? 0 : 1;  // TS: accumulators at 256 (A at 0), SS: at 0
        const long long t0 = clock64();
        for (int g = 0; g < groups; ++g) {
            const int buf = g & 1;
            if (g >= 2) bar_wait(&done[who][buf], ((g >> 1) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t d = tm + (NB ? 0u : 256u) + (uint32_t)((ISSUERS * buf + who) * (ISSUERS == 1 ? N : N / 2));
            for (int i = 0; i < G / ISSUERS; ++i) {
                const uint64_t o = (uint64_t)(((i & 3) * 32) >> 4);
                mma<F16, TS>(d, tm + (uint32_t)(8 * (i & 15)), a + o, bb + o, id, i ? 1u : 0u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&done[who][buf]))
                         : "memory");
        }
        bar_wait(&done[who][(groups - 1) & 1], ((groups - 1) >> 1) & 1);
        const long long t1 = clock64();
        if (who == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <bool F16, bool TS, int N, int ISSUERS = 1>
int run(const char *name, int G)
{
    unsigned long long *d, h;
    CK(cudaMalloc(&d, 8));
    const int groups = 400;
    CK(cudaFuncSetAttribute(k_rate<F16, TS, N, ISSUERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024));
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(d, 0, 8));
        k_rate<F16, TS, N, ISSUERS><<<148, 128, 70 * 1024>>>(groups, G, d);
        CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    const double per = (double)h / 148.0 / groups / G;
    printf("%-22s N=%3d G=%2d issuers=%d: %6.1f cyc/mma  (floor %d)\n", name, N, G, ISSUERS, per, 128 * N / 256);
    CK(cudaFree(d));
    return 0;
}

int main()
{
    run<false, true, 96>("tf32 TS", 24);
    run<false, false, 96>("tf32 SS", 24);
    run<true, true, 96>("f16  TS", 12);
    run<false, true, 64>("tf32 TS", 36);
    run<true, true, 64>("f16  TS", 18);
    run<false, true, 128>("tf32 TS", 24);
    run<true, true, 128>("f16  TS", 12);
    run<false, false, 256>("tf32 SS", 24);
    run<true, false, 256>("f16  SS", 12);
    run<false, false, 192>("tf32 SS", 24);
    run<false, true, 96, 2>("tf32 TS 2 issuers", 24);
    run<false, true, 64, 2>("tf32 TS 2 issuers", 36);
    run<true, true, 96, 2>("f16 TS 2 issuers", 12);
    return 0;
}
