// tc_probe.cu -- validates the hand-built tcgen05 descriptors used by the
// tensor-core SpMV kernels (kind::tf32, M=128, N=96 or 32, K-major
// SWIZZLE_128B operands in shared memory, fp32 accumulator in TMEM) and the
// 3xTF32 split (A_hi.B_hi + A_lo.B_hi + A_hi.B_lo), then times back-to-back
// MMAs.  One CTA; prints max relative error against an fp64 host product.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int M = 128, K = 32;

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, k) of a K-major SWIZZLE_128B tile of fp32 (32 per row)
__host__ __device__ __forceinline__ uint32_t sw128(int row, int k)
{
    return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + (k & 3) * 4);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8-row group stride
    d |= (uint64_t)1 << 46;                 // version (sm_100)
    d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
    return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int N>
__global__ void k_probe(const float *A, const float *B, float *out, int reps, long long *cyc)
{
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    unsigned char *Ahi = sm, *Alo = sm + M * 128, *Bhi = sm + 2 * M * 128, *Blo = Bhi + N * 128;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = A[i], h = tf32_hi(x);
        *(float *)(Ahi + sw128(r, k)) = h;
        *(float *)(Alo + sw128(r, k)) = x - h;
    }
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;  // B stored [n][k] (K-major)
        const float x = B[i], h = tf32_hi(x);
        *(float *)(Bhi + sw128(r, k)) = h;
        *(float *)(Blo + sw128(r, k)) = x - h;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        constexpr uint32_t id = idesc_tf32(M, N);
        const uint64_t ah = sdesc(sa(Ahi)), al = sdesc(sa(Alo)), bh = sdesc(sa(Bhi)), bl = sdesc(sa(Blo));
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int k = 0; k < K / 8; ++k) {
                const uint64_t o = (uint64_t)(k * 32 >> 4);  // +32 bytes per K step
                mma_tf32(tm, ah + o, bh + o, id, (r | k) != 0);
                mma_tf32(tm, al + o, bh + o, id, 1);
                mma_tf32(tm, ah + o, bl + o, id, 1);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(sa(&bar)) : "memory");
        *cyc = clock64() - t0;
    }
    __syncthreads();
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(sa(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32 && c0 + j < N; ++j) out[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

template <int N>
int run(int reps)
{
    std::mt19937 g(7);
    std::normal_distribution<float> nd;
    std::vector<float> A(M * K), B(N * K), out(M * N);
    for (auto &x : A) x = nd(g);
    for (auto &x : B) x = nd(g);
    float *dA, *dB, *dO;
    long long *dc, cyc;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dO, out.size() * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const int smem = 2 * M * 128 + 2 * N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_probe<N><<<1, 128, smem>>>(dA, dB, dO, reps, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    double num = 0, den = 0, maxe = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[n * K + k];
            r *= reps;
            const double e = out[m * N + n] - r;
            num += e * e;
            den += r * r;
            maxe = fmax(maxe, fabs(e));
        }
    const double mmas = 3.0 * (K / 8) * reps;
    printf("N=%d reps=%d rel_l2=%.3e max_abs=%.3e  cycles=%lld  cyc/mma=%.1f (floor %d)\n", N, reps,
           sqrt(num / den), maxe, cyc, cyc / mmas, M * N / 256);
    cudaFree(dA); cudaFree(dB); cudaFree(dO); cudaFree(dc);
    return 0;
}


// chained accumulation over nch chunks: D += s_c * A_{c%4} . B (s_c = +-1 via the
// a_negate bit), the DSC pattern of one voxel tile over all atom chunks
__global__ void k_chain(const float *A, const float *B, const int *sgn, int nch, float *out)
{
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    constexpr int N = 96;
    unsigned char *Bhi = sm + 8 * M * 128, *Blo = Bhi + N * 128;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = 0; t < 4; ++t)
        for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
            const int r = i / K, k = i % K;
            const float x = A[t * M * K + i], h = tf32_hi(x);
            *(float *)(sm + 2 * t * M * 128 + sw128(r, k)) = h;
            *(float *)(sm + (2 * t + 1) * M * 128 + sw128(r, k)) = x - h;
        }
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = B[i], h = tf32_hi(x);
        *(float *)(Bhi + sw128(r, k)) = h;
        *(float *)(Blo + sw128(r, k)) = x - h;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        const uint64_t bh = sdesc(sa(Bhi)), bl = sdesc(sa(Blo));
        for (int c = 0; c < nch; ++c) {
            const int t = c & 3;
            const uint64_t ah = sdesc(sa(sm + 2 * t * M * 128)), al = sdesc(sa(sm + (2 * t + 1) * M * 128));
            const uint32_t id = idesc_tf32(M, N) | (sgn[c] < 0 ? (1u << 13) : 0u);
#pragma unroll
            for (int k = 0; k < K / 8; ++k) {
                const uint64_t o = (uint64_t)(k * 32 >> 4);
                mma_tf32(tm, ah + o, bh + o, id, (c | k) != 0);
                mma_tf32(tm, al + o, bh + o, id, 1);
                mma_tf32(tm, ah + o, bl + o, id, 1);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    }
    __syncthreads();
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(sa(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) out[row * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int chain(int nch, bool sparse)
{
    constexpr int N = 96;
    std::mt19937 g(11);
    std::normal_distribution<float> nd;
    std::uniform_real_distribution<float> ud(0.f, 1.f);
    std::vector<float> A(4 * M * K), B(N * K), out(M * N);
    std::vector<int> s(nch);
    for (auto &x : A) x = (sparse && ud(g) < 0.6f) ? 0.f : ud(g);  // DSC-like: nonnegative, 40% dense
    for (auto &x : B) x = nd(g) * 0.1f;
    for (auto &x : s) x = ud(g) < 0.5f ? -1 : 1;
    float *dA, *dB, *dO;
    int *dS;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dO, out.size() * 4));
    CK(cudaMalloc(&dS, nch * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dS, s.data(), nch * 4, cudaMemcpyHostToDevice));
    const int smem = 8 * M * 128 + 2 * N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_chain<<<1, 128, smem>>>(dA, dB, dS, nch, dO);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out.data(), dO, out.size() * 4, cudaMemcpyDeviceToHost));
    double num = 0, den = 0, num32 = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0;
            float r32 = 0.f;  // sequential fp32 reference loop order (chunk by chunk, k ascending)
            for (int c = 0; c < nch; ++c)
                for (int k = 0; k < K; ++k) {
                    const double p = (double)s[c] * A[(c & 3) * M * K + m * K + k] * B[n * K + k];
                    r += p;
                    r32 = __builtin_fmaf((float)s[c] * A[(c & 3) * M * K + m * K + k], B[n * K + k], r32);
                }
            const double e = out[m * N + n] - r, e32 = r32 - r;
            num += e * e;
            num32 += e32 * e32;
            den += r * r;
        }
    printf("chain nch=%d sparse=%d: tcgen05 3xTF32 rel_l2=%.3e   (sequential fp32 fma loop: %.3e)\n", nch, (int)sparse,
           sqrt(num / den), sqrt(num32 / den));
    cudaFree(dA); cudaFree(dB); cudaFree(dO); cudaFree(dS);
    return 0;
}

// A operand from TMEM ("ts" form): A (128 x 32 fp32) written to TMEM lanes
// (row m -> lane m, k -> column a0 + k) with tcgen05.st; B (N x 32) K-major in
// shared memory; D = A . B^T in TMEM; plain tf32 (1 term) and 3xTF32.
template <int N>
__global__ void k_ts(const float *A, const float *B, float *out, float *out3)
{
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    unsigned char *Bhi = sm, *Blo = sm + N * 128;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = B[i], h = tf32_hi(x);
        *(float *)(Bhi + sw128(r, k)) = h;
        *(float *)(Blo + sw128(r, k)) = x - h;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    // A hi at columns 128.., A lo at columns 160.. ; D1 at 0.., D3 at 64..
    {
        const int row = warp * 32 + lane;
        uint32_t hv[32], lv[32];
        for (int k = 0; k < 32; ++k) {
            const float x = A[row * K + k], h = tf32_hi(x);
            hv[k] = __float_as_uint(h);
            lv[k] = __float_as_uint(x - h);
        }
        const uint32_t ah = tm + ((uint32_t)(warp * 32) << 16) + 128u, al = ah + 32u;
#define ST32(addr, v) asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
        ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), \
          "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory")
        ST32(ah, hv);
        ST32(al, lv);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        constexpr uint32_t id = idesc_tf32(M, N);
        const uint64_t bh = sdesc(sa(Bhi)), bl = sdesc(sa(Blo));
        for (int k = 0; k < K / 8; ++k) {
            const uint64_t o = (uint64_t)(k * 32 >> 4);
            const uint32_t ah = tm + 128u + 8u * k, al = tm + 160u + 8u * k;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(ah), "l"(bh + o), "r"(id), "r"((uint32_t)(k != 0)));
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 64u), "r"(ah), "l"(bh + o), "r"(id), "r"((uint32_t)(k != 0)));
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 64u), "r"(al), "l"(bh + o), "r"(id), "r"(1u));
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 64u), "r"(ah), "l"(bl + o), "r"(id), "r"(1u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    }
    __syncthreads();
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(sa(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int pass = 0; pass < 2; ++pass) {
        uint32_t v[32];
        const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + (pass ? 64u : 0u);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float *o = pass ? out3 : out;
        for (int j = 0; j < N; ++j) o[row * N + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

int ts_test()
{
    constexpr int N = 32;
    std::mt19937 g(5);
    std::normal_distribution<float> nd;
    std::vector<float> A(M * K), B(N * K), o1(M * N), o3(M * N);
    for (auto &x : A) x = nd(g);
    for (auto &x : B) x = nd(g);
    float *dA, *dB, *d1, *d3;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&d1, o1.size() * 4));
    CK(cudaMalloc(&d3, o3.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const int smem = 2 * N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_ts<N><<<1, 128, smem>>>(dA, dB, d1, d3);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(o1.data(), d1, o1.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(o3.data(), d3, o3.size() * 4, cudaMemcpyDeviceToHost));
    double n1 = 0, n3 = 0, den = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[n * K + k];
            n1 += (o1[m * N + n] - r) * (o1[m * N + n] - r);
            n3 += (o3[m * N + n] - r) * (o3[m * N + n] - r);
            den += r * r;
        }
    printf("ts (A in TMEM) N=%d: 1xTF32 rel_l2=%.3e  3xTF32 rel_l2=%.3e\n", N, sqrt(n1 / den), sqrt(n3 / den));
    return 0;
}

int main()
{
    if (ts_test()) return 1;
    if (chain(34, true) || chain(34, false) || chain(136, true)) return 1;
    if (run<96>(1)) return 1;
    if (run<32>(1)) return 1;
    if (run<96>(200)) return 1;
    if (run<32>(200)) return 1;
    if (run<128>(200)) return 1;
    return 0;
}
