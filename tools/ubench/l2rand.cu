// l2rand.cu -- random gather / scatter-reduce throughput into an Nf-sized
// vector (the w gather of DSC and the fascicle scatter of WC at C2).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2rand l2rand.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldst(const uint4 *p)
{
    uint4 r;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// mode 0: stream idx only; 1: gather w[idx] (f32); 2: red.add.u64 wfix[idx];
// 3: red.add.f32 w[idx]; 4: gather 2 (f32) per idx pair sorted?;
template <int MODE>
__global__ void k(const uint4 *__restrict__ idx, size_t n4, const float *__restrict__ w,
                  float *wf, unsigned long long *wfix, float *out)
{
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride * 2) {
        uint4 a = ldst(idx + i);
        uint4 b = (i + stride < n4) ? ldst(idx + i + stride) : make_uint4(0, 0, 0, 0);
        const uint32_t f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        if (MODE == 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc += __uint_as_float(f[e]);
        } else if (MODE == 1) {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc += __ldg(w + f[e]);
        } else if (MODE == 2) {
#pragma unroll
            for (int e = 0; e < 8; ++e) atomicAdd(wfix + f[e], (unsigned long long)(f[e] & 7));
        } else if (MODE == 3) {
#pragma unroll
            for (int e = 0; e < 8; ++e) atomicAdd(wf + f[e], 1.0f);
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char **argv)
{
    const size_t n = 100000000;  // 100M indices
    int nf = argc > 1 ? atoi(argv[1]) : 500000;
    std::vector<uint32_t> h(n);
    std::mt19937 g(1);
    for (size_t i = 0; i < n; ++i) h[i] = g() % nf;
    uint32_t *d_idx;
    float *w, *out;
    unsigned long long *wfix;
    CK(cudaMalloc(&d_idx, n * 4));
    CK(cudaMalloc(&w, (size_t)nf * 4));
    CK(cudaMalloc(&wfix, (size_t)nf * 8));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemcpy(d_idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(w, 0, (size_t)nf * 4));
    CK(cudaMemset(wfix, 0, (size_t)nf * 8));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"stream idx", "gather f32", "red.add u64", "red.add f32"};
    for (int bs : {256, 512, 1024}) {
        for (int mode = 0; mode < 4; ++mode) {
            const int blocks = sms * (2048 / bs);
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                switch (mode) {
                case 0: k<0><<<blocks, bs>>>((uint4 *)d_idx, n / 4, w, w, wfix, out); break;
                case 1: k<1><<<blocks, bs>>>((uint4 *)d_idx, n / 4, w, w, wfix, out); break;
                case 2: k<2><<<blocks, bs>>>((uint4 *)d_idx, n / 4, w, w, wfix, out); break;
                case 3: k<3><<<blocks, bs>>>((uint4 *)d_idx, n / 4, w, w, wfix, out); break;
                }
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("nf=%d bs=%d %-12s %.3f ms  %.2f Gop/s  idx %.0f GB/s\n", nf, bs, names[mode], best,
                   n / best / 1e6, n * 4 / best / 1e6);
        }
    }
    return 0;
}
