// Microbenchmarks: FFMA vs FFMA2 (fma.rn.f32x2) throughput, shared-memory
// LDS.32 / LDS.128 (distinct and broadcast) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float *out, int iters, float a, float b)
{
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, int iters, float a, float b)
{
    unsigned long long x[8];
    float2 av = make_float2(a, a), bv = make_float2(b, b);
    unsigned long long ap = *reinterpret_cast<unsigned long long *>(&av);
    unsigned long long bp = *reinterpret_cast<unsigned long long *>(&bv);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 t = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
        x[i] = *reinterpret_cast<unsigned long long *>(&t);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(ap), "l"(bp));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 t = *reinterpret_cast<float2 *>(&x[i]);
        s += t.x + t.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mode 0: LDS.32 distinct (lane-consecutive), 1: LDS.128 distinct, 2: LDS.128 broadcast (all lanes same), 3: LDS.32 broadcast
template <int MODE>
__global__ void k_lds(float *out, int iters)
{
    __shared__ __align__(16) float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
    __syncthreads();
    float acc = 0.f;
    const int lane = threadIdx.x & 31;
    int base = (threadIdx.x >> 5) * 64;
    for (int it = 0; it < iters; ++it) {
        const int off = (base + it * 4) & 4095;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0) acc += s[off + u * 256 + lane];
            if (MODE == 1) {
                float4 v = *reinterpret_cast<const float4 *>(&s[((off + u * 512) & 8191 & ~3) + lane * 4 - (lane*4 >= 128 ? 0:0)]);
                acc += (v.x + v.y) + (v.z + v.w);
            }
            if (MODE == 2) {
                float4 v = *reinterpret_cast<const float4 *>(&s[(off + u * 16) & 8188]);
                acc += (v.x + v.y) + (v.z + v.w);
            }
            if (MODE == 3) acc += s[(off + u * 16) & 8191];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sms * 8 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    auto run = [&](const char *name, auto launch, double ops_per_thread) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double threads = (double)sms * 4 * 256;
        double per_sm_per_s = ops_per_thread * threads / (ms * 1e-3) / sms;
        printf("%-28s %8.3f ms  %10.2f G/s/SM  err=%s\n", name, ms, per_sm_per_s * 1e-9,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("FFMA (fma/clk/SM @ /1.9GHz)", [&] { k_ffma<<<sms * 4, 256>>>(out, iters, 1.0001f, 0.5f); },
        (double)iters * 16);
    run("FFMA2 (fma)", [&] { k_ffma2<<<sms * 4, 256>>>(out, iters, 1.0001f, 0.5f); },
        (double)iters * 16);
    run("LDS.32 distinct (req)", [&] { k_lds<0><<<sms * 4, 256>>>(out, iters / 4); },
        (double)iters / 4 * 8 / 32);
    run("LDS.128 distinct (req)", [&] { k_lds<1><<<sms * 4, 256>>>(out, iters / 4); },
        (double)iters / 4 * 8 / 32);
    run("LDS.128 broadcast (req)", [&] { k_lds<2><<<sms * 4, 256>>>(out, iters / 4); },
        (double)iters / 4 * 8 / 32);
    run("LDS.32 broadcast (req)", [&] { k_lds<3><<<sms * 4, 256>>>(out, iters / 4); },
        (double)iters / 4 * 8 / 32);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock rate attr %d kHz\n", clk);
    return 0;
}
