// scatter_probe.cu -- random reduction throughput on B200 for WC's fascicle
// sums (100M contributions into Nf = 500k sums):
//   red64  : red.global.add.u64 (LSU path), one per contribution
//   red32f : red.global.add.f32
//   tmar   : cp.reduce.async.bulk.tensor tile::scatter4 .add (TMA path),
//            rows of 2 x u64 (16 B) or 4 x f32 (16 B): one useful element
//            per row, the others zero
//   tmag   : cp.async.bulk.tensor tile::gather4 (TMA path), 16-byte rows,
//            issued by 1..8 warps per SM
//   lds    : random 4-byte shared-memory loads (32 distinct addresses)
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o scatter_probe scatter_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_red64(const uint4 *__restrict__ idx, size_t n4, unsigned long long *t)
{
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 a = __ldcs(idx + i);
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(t + a.x), "l"(1ull) : "memory");
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(t + a.y), "l"(1ull) : "memory");
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(t + a.z), "l"(1ull) : "memory");
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(t + a.w), "l"(1ull) : "memory");
    }
}
__global__ void k_red32f(const uint4 *__restrict__ idx, size_t n4, float *t)
{
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 a = __ldcs(idx + i);
        atomicAdd(t + a.x, 1.f);
        atomicAdd(t + a.y, 1.f);
        atomicAdd(t + a.z, 1.f);
        atomicAdd(t + a.w, 1.f);
    }
}

// random 4-byte shared loads: each lane a random word of a 32 KB table
__global__ void k_lds(int iters, float *out)
{
    __shared__ float tab[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) tab[i] = (float)i;
    __syncthreads();
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            x = x * 1664525u + 1013904223u;
            v[e] = tab[(x >> 10) & 8191u];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += v[e];
    }
    if (acc == 1234.5f) out[0] = acc;
}

// TMA: each issuing lane owns a 64-byte slot per stage (4 rows of 16 B);
// reduce mode pushes the slot (rows: first element 1, rest 0) with
// scatter4 .add; gather mode fetches 4 rows.  A warp-round's ops complete
// on a bulk group (reduce) or an mbarrier (gather).
template <int STAGES, bool GATHER>
__global__ void k_tma(const __grid_constant__ CUtensorMap map, const uint32_t *__restrict__ idx,
                      size_t rounds, unsigned long long *done)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[32][STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    unsigned char *base = sm + (size_t)warp * STAGES * 32 * 64;
    if (!GATHER) {
        for (int i = lane; i < STAGES * 32 * 16; i += 32) {
            uint32_t *p = reinterpret_cast<uint32_t *>(base) + i;
            *p = 0u;
        }
        __syncwarp();
        for (int i = lane; i < STAGES * 32 * 4; i += 32)   // first 8 bytes of each 16-byte row = 1
            reinterpret_cast<unsigned long long *>(base)[2 * i] = 1ull;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const size_t gw = (size_t)blockIdx.x * nw + warp;
    const uint32_t *my = idx + gw * rounds * 128;
    for (size_t r = 0; r < rounds; ++r) {
        const int s = (int)(r % STAGES);
        const uint4 rows = __ldcs(reinterpret_cast<const uint4 *>(my + r * 128) + lane);
        const uint32_t dst = sa(base + ((size_t)s * 32 + lane) * 64);
        if (GATHER) {
            if (r >= STAGES) {
                const unsigned par = (unsigned)((r / STAGES - 1) & 1);
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, p;\n}"
                                 : "=r"(ok) : "r"(sa(&bar[warp][s])), "r"(par) : "memory");
            }
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[warp][s])),
                             "r"(32u * 64u) : "memory");
            __syncwarp();
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
                "l"(&map), "r"(sa(&bar[warp][s])), "r"(0), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w)
                : "memory");
        } else {
            asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group"
                         " [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(&map), "r"(dst), "r"(0), "r"(rows.x),
                         "r"(rows.y), "r"(rows.z), "r"(rows.w) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
        }
    }
    if (GATHER) {
        for (int s = 0; s < STAGES; ++s) {
            const size_t r = rounds >= (size_t)STAGES ? rounds - STAGES + s : s;
            if (r >= rounds) continue;
            const int ss = (int)(r % STAGES);
            const unsigned par = (unsigned)((r / STAGES) & 1);
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n}"
                             : "=r"(ok) : "r"(sa(&bar[warp][ss])), "r"(par) : "memory");
        }
    } else {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    if (threadIdx.x == 0) atomicAdd(done, 1ull);
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float time_ms(cudaEvent_t a, cudaEvent_t b)
{
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

int main()
{
    const size_t n = 100000000;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double clk = 1.965e9;
    uint32_t *d_idx;
    CK(cudaMalloc(&d_idx, n * 4));
    std::vector<uint32_t> h(n);
    const uint32_t nf = 500000;
    std::mt19937 g(1);
    for (size_t i = 0; i < n; ++i) h[i] = g() % nf;
    CK(cudaMemcpy(d_idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    unsigned long long *t64;
    CK(cudaMalloc(&t64, (size_t)nf * 8 * 4));
    CK(cudaMemset(t64, 0, (size_t)nf * 8 * 4));
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        k_red64<<<sms * 4, 512>>>(reinterpret_cast<const uint4 *>(d_idx), n / 4, t64);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        if (rep) printf("red64  Nf %u: %.3f ms per 100M (%.1f G/s, %.2f /clk/SM)\n", nf, time_ms(e0, e1),
                        n / time_ms(e0, e1) / 1e6, n / (time_ms(e0, e1) * 1e-3) / sms / clk);
    }
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        k_red32f<<<sms * 4, 512>>>(reinterpret_cast<const uint4 *>(d_idx), n / 4, reinterpret_cast<float *>(t64));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        if (rep) printf("red32f Nf %u: %.3f ms per 100M (%.1f G/s, %.2f /clk/SM)\n", nf, time_ms(e0, e1),
                        n / time_ms(e0, e1) / 1e6, n / (time_ms(e0, e1) * 1e-3) / sms / clk);
    }
    {
        float *out;
        CK(cudaMalloc(&out, 4));
        const int iters = 4096;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(e0));
            k_lds<<<sms, 1024>>>(iters, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            const double loads = (double)sms * 1024 * iters * 8;
            if (rep) printf("lds    random 4B: %.2f loads/clk/SM\n", loads / (time_ms(e0, e1) * 1e-3) / sms / clk);
        }
    }
    EncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    unsigned long long *done;
    CK(cudaMalloc(&done, 8));
    // rows of 16 bytes over the Nf-element table: u64 pairs (row = f / 2) or f32 quads (row = f / 4)
    struct Cfg { const char *name; CUtensorMapDataType dt; int epr; };
    const Cfg cfgs[2] = {{"u64x2", CU_TENSOR_MAP_DATA_TYPE_UINT64, 2}, {"f32x4", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4}};
    for (const Cfg &c : cfgs) {
        const uint32_t nrows = nf / c.epr;
        std::vector<uint32_t> hr(n);
        for (size_t i = 0; i < n; ++i) hr[i] = h[i] / c.epr;
        CK(cudaMemcpy(d_idx, hr.data(), n * 4, cudaMemcpyHostToDevice));
        CUtensorMap map;
        cuuint64_t gdim[2] = {(cuuint64_t)c.epr, nrows};
        cuuint64_t gstr[1] = {16};
        cuuint32_t box[2] = {(cuuint32_t)c.epr, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult cr = enc(&map, c.dt, 2, t64, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) {
            printf("encode %s failed %d\n", c.name, (int)cr);
            continue;
        }
        for (int mode = 0; mode < 2; ++mode)
            for (int warps : {1, 2, 4, 8}) {
                constexpr int ST = 4;
                const size_t nwarps = (size_t)sms * warps;
                const size_t rounds = n / (nwarps * 128);
                const size_t smem = (size_t)warps * ST * 32 * 64;
                auto kern = mode ? k_tma<ST, true> : k_tma<ST, false>;
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                for (int rep = 0; rep < 2; ++rep) {
                    CK(cudaEventRecord(e0));
                    kern<<<sms, warps * 32, smem>>>(map, d_idx, rounds, done);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    CK(cudaGetLastError());
                    const double rows = (double)rounds * nwarps * 128;
                    if (rep)
                        printf("%s %s warps %d: %.3f ms per 100M rows (%.1f G rows/s, %.2f rows/clk/SM)\n",
                               mode ? "tmag" : "tmar", c.name, warps, time_ms(e0, e1) * 1e8 / rows,
                               rows / time_ms(e0, e1) / 1e6, rows / (time_ms(e0, e1) * 1e-3) / sms / clk);
                }
            }
    }
    return 0;
}
