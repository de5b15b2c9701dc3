// f16_probe.cu -- validates kind::f16 tcgen05 operand layouts for the binned
// products: A (M=128 x K=64 f16) from TMEM (two f16 per 32-bit column) or from
// shared memory (K-major SWIZZLE_128B, 64 f16 per 128-byte row), B (N x K=64
// f16, K-major SWIZZLE_128B), fp32 accumulator; and the 2-term f16 split
// x = hi + lo (A_hi.B_hi + A_lo.B_hi + A_hi.B_lo) against an fp64 product.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o f16_probe f16_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
            return 1;                                                               \
        }                                                                           \
    } while (0)

constexpr int M = 128, K = 64;

__host__ __device__ inline uint32_t sw16(int row, int k)  // byte offset of f16 (row, k), K-major SW128
{
    return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + (((k >> 3) ^ (row & 7)) << 4) + (k & 7) * 2);
}
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n)
{
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// A: [2][M][K] f16 (hi, lo) row-major on input; B: [2][N][K] f16; out [M][N]
template <int N, bool TS>
__global__ void k_probe(const __half *A, const __half *B, float *out, int terms)
{
    extern __shared__ __align__(1024) unsigned char smr[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smr + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned char *sA = sm, *sB = sm + 2 * M * K * 2;  // A hi|lo, B hi|lo
    for (int i = threadIdx.x; i < 2 * M * K; i += blockDim.x) {
        const int h = i / (M * K), r = (i / K) % M, k = i % K;
        *reinterpret_cast<__half *>(sA + h * M * K * 2 + sw16(r, k)) = A[i];
    }
    for (int i = threadIdx.x; i < 2 * N * K; i += blockDim.x) {
        const int h = i / (N * K), r = (i / K) % N, k = i % K;
        *reinterpret_cast<__half *>(sB + h * N * K * 2 + sw16(r, k)) = B[i];
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    // A into TMEM: thread = row (4 warps), column c = f16 pair (2c, 2c+1), hi at 0, lo at K/2
    if (TS) {
        const int w = threadIdx.x >> 5, row = threadIdx.x;
        for (int h = 0; h < 2; ++h)
            for (int c = 0; c < K / 2; ++c) {
                const __half2 v = __halves2half2(A[h * M * K + row * K + 2 * c], A[h * M * K + row * K + 2 * c + 1]);
                const uint32_t u = *reinterpret_cast<const uint32_t *>(&v);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + ((uint32_t)(w * 32) << 16) +
                                                                                      (uint32_t)(h * K / 2 + c)),
                             "r"(u));
            }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_f16(M, N), d = tm + 128;
        const uint64_t ah = sdesc(sa(sA)), al = sdesc(sa(sA + M * K * 2));
        const uint64_t bh = sdesc(sa(sB)), bl = sdesc(sa(sB + N * K * 2));
        for (int kk = 0; kk < K / 16; ++kk) {
            const uint64_t o = (uint64_t)((kk * 32) >> 4);
            for (int t = 0; t < terms; ++t) {
                const uint32_t acc = (kk || t) ? 1u : 0u;
                const uint64_t b = (t == 2 ? bl : bh) + o;
                if (TS) {
                    const uint32_t a = tm + (uint32_t)((t == 1 ? K / 2 : 0) + 8 * kk);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                                 "r"(a), "l"(b), "r"(id), "r"(acc));
                } else {
                    const uint64_t a = (t == 1 ? al : ah) + o;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                 "l"(a), "l"(b), "r"(id), "r"(acc));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                     : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(sa(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {
        const int w = threadIdx.x >> 5, row = threadIdx.x;
        for (int c = 0; c < N; ++c) {
            uint32_t v;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v)
                         : "r"(tm + ((uint32_t)(w * 32) << 16) + 128u + (uint32_t)c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            out[row * N + c] = __uint_as_float(v);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

static void split(double x, double pre, __half &h, __half &l)
{
    const float xf = (float)(x * pre);
    h = __float2half_rn(xf);
    l = __float2half_rn(xf - __half2float(h));
}

template <int N, bool TS>
int run(double amag, double bmag)
{
    std::mt19937 g(7);
    std::normal_distribution<double> nd;
    std::vector<double> a(M * K), b(N * K);
    for (auto &x : a) x = nd(g) * amag;
    for (auto &x : b) x = nd(g) * bmag;
    // operand scaling into the f16 range: A by 2^sa, B by 2^sb (powers of two)
    double amax = 0, bmax = 0;
    for (double x : a) amax = std::max(amax, std::fabs(x));
    for (double x : b) bmax = std::max(bmax, std::fabs(x));
    int ea, eb;
    std::frexp(amax, &ea);
    std::frexp(bmax, &eb);
    const double pa = std::ldexp(1.0, 14 - ea), pb = std::ldexp(1.0, 8 - eb);
    std::vector<__half> A(2 * M * K), B(2 * N * K);
    for (int i = 0; i < M * K; ++i) split(a[i], pa, A[i], A[M * K + i]);
    for (int i = 0; i < N * K; ++i) split(b[i], pb, B[i], B[N * K + i]);
    __half *dA, *dB;
    float *dO;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dO, M * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    const int smem = 1024 + 2 * M * K * 2 + 2 * N * K * 2;
    CK(cudaFuncSetAttribute(k_probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int terms : {1, 3}) {
        k_probe<N, TS><<<1, 128, smem>>>(dA, dB, dO, terms);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(M * N);
        CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
        double num = 0, den = 0;
        for (int r = 0; r < M; ++r)
            for (int c = 0; c < N; ++c) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += a[r * K + k] * b[c * K + k];
                const double got = o[r * N + c] / (pa * pb);
                num += (got - ref) * (got - ref);
                den += ref * ref;
            }
        printf("%s N=%d |A|~%.0e |B|~%.0e terms=%d: rel_l2=%.3e\n", TS ? "TS" : "SS", N, amag, bmag, terms,
               std::sqrt(num / den));
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
    return 0;
}

int main()
{
    run<96, false>(1.0, 0.1);
    run<96, true>(1.0, 0.1);
    run<64, true>(1e-3, 0.1);
    run<64, false>(1e5, 1.0);
    return 0;
}
