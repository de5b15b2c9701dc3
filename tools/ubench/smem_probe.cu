// smem_probe.cu -- random shared-memory access rates on B200 (per SM per clock)
// for the binned SpMV design: where do 100M random per-coefficient updates
// cost least?
//   lds      : random 4-byte loads (baseline)
//   rmw      : LDS + FADD + STS to random words (non-atomic)
//   red.u32 / red.u64 / red.f32 : red.shared.add, random words
//   atom.u32 : atom.shared.add.u32 (returns the old value)
//   dsm.ld   : ld.shared::cluster from a random CTA of the cluster (random word)
//   dsm.red  : red.shared::cluster.add.f32 / .u64 to a random CTA of the cluster
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o smem_probe smem_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

constexpr int kWords = 8192;  // 32 KB table

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k_local(int iters, float *out)
{
    __shared__ __align__(16) uint32_t tab[kWords];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) tab[i] = 0;
    __syncthreads();
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            x = x * 1664525u + 1013904223u;
            const uint32_t i = (x >> 8) & (kWords - 1);
            if (MODE == 0) {
                acc += __uint_as_float(tab[i]);
            } else if (MODE == 1) {
                float *f = reinterpret_cast<float *>(tab) + i;
                *f = *f + 1.0f;
            } else if (MODE == 2) {
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sa(tab + i)), "r"(x | 1u) : "memory");
            } else if (MODE == 3) {
                asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(sa(tab + (i & ~1u))), "l"(1ull) : "memory");
            } else if (MODE == 4) {
                asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(sa(tab + i)), "f"(1.0f) : "memory");
            } else {
                uint32_t old;
                asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(sa(tab + i)), "r"(x | 1u) : "memory");
                acc += (float)old;
            }
        }
    }
    __syncthreads();
    if (acc == 1234.5f || tab[threadIdx.x] == 0xFFFFFFFFu) out[0] = acc;
}

template <int MODE>
__global__ void k_dsm(int iters, float *out)
{
    __shared__ __align__(16) uint32_t tab[kWords];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) tab[i] = 0;
    cl.sync();
    const uint32_t nb = cl.num_blocks();
    const uint32_t base = sa(tab);
    uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            x = x * 1664525u + 1013904223u;
            const uint32_t i = (x >> 8) & (kWords - 1);
            const uint32_t r = (x >> 24) % nb;
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + 4 * i), "r"(r));
            if (MODE == 0) {
                uint32_t v;
                asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
                acc += __uint_as_float(v);
            } else if (MODE == 1) {
                asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(ra), "f"(1.0f) : "memory");
            } else {
                asm volatile("red.shared::cluster.add.u64 [%0], %1;" ::"r"(ra & ~7u), "l"(1ull) : "memory");
            }
        }
    }
    cl.sync();
    if (acc == 1234.5f || tab[threadIdx.x] == 0xFFFFFFFFu) out[0] = acc;
}

static double time_ms(cudaEvent_t a, cudaEvent_t b)
{
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

int main()
{
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    const double clk = 1.965e9;
    float *out;
    CK(cudaMalloc(&out, 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const char *names[6] = {"lds", "rmw (lds+fadd+sts)", "red.shared.add.u32", "red.shared.add.u64",
                            "red.shared.add.f32", "atom.shared.add.u32"};
    void (*ks[6])(int, float *) = {k_local<0>, k_local<1>, k_local<2>, k_local<3>, k_local<4>, k_local<5>};
    for (int m = 0; m < 6; ++m)
        for (int threads : {256, 1024}) {
            const int iters = 2048;
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaEventRecord(e0));
                ks[m]<<<sms * (1024 / threads), threads>>>(iters, out);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
                const double ops = (double)sms * 1024 * iters * 8;
                if (rep)
                    printf("%-22s blk %4d: %6.2f ops/clk/SM  (100M ops: %.3f ms)\n", names[m], threads,
                           ops / (time_ms(e0, e1) * 1e-3) / sms / clk, time_ms(e0, e1) * 1e8 / ops);
            }
        }
    const char *dn[3] = {"dsm ld.shared::cluster", "dsm red.add.f32", "dsm red.add.u64"};
    void (*kd[3])(int, float *) = {k_dsm<0>, k_dsm<1>, k_dsm<2>};
    for (int m = 0; m < 3; ++m)
        for (int csz : {2, 8, 16}) {
            if (csz == 16) CK(cudaFuncSetAttribute(kd[m], cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg = {};
            const int blocks = (sms / csz) * csz;
            cfg.gridDim = dim3(blocks);
            cfg.blockDim = dim3(1024);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = csz;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            const int iters = 512;
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaEventRecord(e0));
                cudaError_t le = cudaLaunchKernelEx(&cfg, kd[m], iters, out);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                if (le != cudaSuccess) {
                    printf("%s cluster %d: launch %s\n", dn[m], csz, cudaGetErrorString(le));
                    break;
                }
                CK(cudaGetLastError());
                const double ops = (double)blocks * 1024 * iters * 8;
                if (rep)
                    printf("%-22s cl %2d: %6.2f ops/clk/SM  (100M ops: %.3f ms)\n", dn[m], csz,
                           ops / (time_ms(e0, e1) * 1e-3) / blocks / clk, time_ms(e0, e1) * 1e8 / ops);
            }
        }
    return 0;
}
