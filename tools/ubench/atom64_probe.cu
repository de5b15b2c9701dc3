// atom64_probe.cu -- shared-memory random atomic add throughput on B200:
// red.shared.add.u32 x2 (two limbs) vs red.shared.add.u64 x1 per term.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o atom64_probe atom64_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(int iters, unsigned long long *out, unsigned long long *cyc)
{
    extern __shared__ unsigned long long s64[];
    uint32_t *s32 = reinterpret_cast<uint32_t *>(s64);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) s64[i] = 0;
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t slot = x >> 18;  // 0..16383
        if (MODE == 0) {
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(s32 + slot)), "r"(x) : "memory");
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(s32 + 16384 + slot)), "r"(x) : "memory");
        } else {
            asm volatile("red.shared.add.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(s64 + slot)), "l"((unsigned long long)x) : "memory");
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        atomicAdd(cyc, (unsigned long long)(t1 - t0));
        atomicAdd(out, s64[blockIdx.x & 16383]);
    }
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 16);
    const int iters = 4096;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(d, 0, 16);
            if (mode == 0) k<0><<<148, 1024, 131072>>>(iters, d, d + 1);
            else k<1><<<148, 1024, 131072>>>(iters, d, d + 1);
            cudaDeviceSynchronize();
        }
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double cyc = (double)h[1] / 148.0;
        printf("%s: %.2f terms/clk/SM (%.0f cycles for %d terms per SM)\n", mode ? "u64 x1" : "u32 x2",
               1024.0 * iters / cyc, cyc, 1024 * iters);
    }
    return 0;
}
