// gather_probe.cu -- random-access throughput on B200 for the two LiFE
// indirections (DSC's w[f] gather, WC's fascicle reduction):
//   ldg   : random 4-byte LDG gathers (LSU path, L1 no_allocate)
//   st    : random 4-byte st.global scatters
//   tma4  : cp.async.bulk.tensor tile::gather4 (TMA path), rows of R bytes
// over tables of T bytes (2 MB = Nf*4 at C2; 50 MB = an L2-resident wave
// buffer; 400 MB = not L2-resident).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o gather_probe gather_probe.cu -lcuda
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

__global__ void k_ldg(const uint4 *__restrict__ idx, size_t n4, const float *__restrict__ t, float *out)
{
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 2 * stride) {
        const uint4 a = __ldcs(idx + i);
        const uint4 b = i + stride < n4 ? __ldcs(idx + i + stride) : make_uint4(0, 0, 0, 0);
        const uint32_t f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
            asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v[e]) : "l"(t + f[e]));
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += v[e];
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void k_st(const uint4 *__restrict__ idx, size_t n4, float *t)
{
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 a = __ldcs(idx + i);
        t[a.x] = 1.f;
        t[a.y] = 2.f;
        t[a.z] = 3.f;
        t[a.w] = 4.f;
    }
}

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// WARPS issuing warps per CTA; each lane issues one gather4 per round into
// its own 4*R-byte slot; a round of a warp completes on one mbarrier; STAGES
// rounds in flight per warp.
template <int STAGES>
__global__ void k_tma4(const __grid_constant__ CUtensorMap map, const uint32_t *__restrict__ idx,
                       size_t nrounds_per_warp, int rowbytes, unsigned long long *done)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[32][STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const unsigned slot_bytes = 4u * rowbytes < 128u ? 128u : 4u * rowbytes;
    unsigned char *base = sm + (size_t)warp * STAGES * 32 * slot_bytes;
    const size_t gw = (size_t)blockIdx.x * nw + warp;
    const uint32_t *my = idx + gw * nrounds_per_warp * 128;
    for (size_t r = 0; r < nrounds_per_warp; ++r) {
        const int s = (int)(r % STAGES);
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
                         "r"(32u * 4u * (unsigned)rowbytes) : "memory");
        __syncwarp();
        const uint4 rows = __ldcs(reinterpret_cast<const uint4 *>(my + r * 128) + lane);
        const uint32_t dst = sa(base + ((size_t)s * 32 + lane) * slot_bytes);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
            "l"(&map), "r"(sa(&bar[warp][s])), "r"(0), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w)
            : "memory");
    }
    // drain
    for (int s = 0; s < STAGES; ++s) {
        const size_t r = nrounds_per_warp >= (size_t)STAGES ? nrounds_per_warp - STAGES + s : s;
        if (r >= nrounds_per_warp) continue;
        const int ss = (int)(r % STAGES);
        const unsigned par = (unsigned)((r / STAGES) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok) : "r"(sa(&bar[warp][ss])), "r"(par) : "memory");
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

int main(int argc, char **argv)
{
    const size_t n = 100000000;  // 100M random accesses
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *out;
    CK(cudaMalloc(&out, 4));
    uint32_t *d_idx;
    CK(cudaMalloc(&d_idx, n * 4));
    std::vector<uint32_t> h(n);
    const size_t tables[3] = {2u << 20, 50u << 20, 400u << 20};
    for (size_t tb : tables) {
        const uint32_t nel = (uint32_t)(tb / 4);
        std::mt19937 g(1);
        for (size_t i = 0; i < n; ++i) h[i] = g() % nel;
        CK(cudaMemcpy(d_idx, h.data(), n * 4, cudaMemcpyHostToDevice));
        float *t;
        CK(cudaMalloc(&t, tb));
        CK(cudaMemset(t, 0, tb));
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(e0));
            k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const uint4 *>(d_idx), n / 4, t, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            if (rep) printf("ldg   table %4zu MB: %.3f ms per 100M  (%.1f G/s)\n", tb >> 20, time_ms(e0, e1),
                            n / time_ms(e0, e1) / 1e6);
        }
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(e0));
            k_st<<<sms * 4, 512>>>(reinterpret_cast<const uint4 *>(d_idx), n / 4, t);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            if (rep) printf("st    table %4zu MB: %.3f ms per 100M  (%.1f G/s)\n", tb >> 20, time_ms(e0, e1),
                            n / time_ms(e0, e1) / 1e6);
        }
        // TMA gather4: rows of R bytes; row index space = tb / R
        EncodeTiled enc = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
        for (int R : {16, 32}) {
            const uint32_t nrows = (uint32_t)(tb / R);
            for (size_t i = 0; i < n; ++i) h[i] = g() % nrows;
            CK(cudaMemcpy(d_idx, h.data(), n * 4, cudaMemcpyHostToDevice));
            CUtensorMap map;
            cuuint64_t gdim[2] = {(cuuint64_t)(R / 4), nrows};
            cuuint64_t gstr[1] = {(cuuint64_t)R};
            cuuint32_t box[2] = {(cuuint32_t)(R / 4), 1};
            cuuint32_t es[2] = {1, 1};
            CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, t, gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) {
                printf("encode failed %d\n", (int)cr);
                continue;
            }
            unsigned long long *done;
            CK(cudaMalloc(&done, 8));
            for (int warps : {1, 2, 4, 8}) {
                constexpr int ST = 4;
                const size_t rows_total = n;  // gather 100M rows (25M gather4 ops)
                const size_t nwarps = (size_t)sms * warps;
                const size_t rounds = rows_total / (nwarps * 128);
                const size_t smem = (size_t)warps * ST * 32 * (4 * R < 128 ? 128 : 4 * R);
                CK(cudaFuncSetAttribute(k_tma4<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                for (int rep = 0; rep < 2; ++rep) {
                    CK(cudaEventRecord(e0));
                    k_tma4<ST><<<sms, warps * 32, smem>>>(map, d_idx, rounds, R, done);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    CK(cudaGetLastError());
                    const double rows = (double)rounds * nwarps * 128;
                    if (rep)
                        printf("tma4  table %4zu MB row %2d B warps %d: %.3f ms per 100M rows (%.1f G rows/s, %.2f rows/clk/SM @1.965GHz)\n",
                               tb >> 20, R, warps, time_ms(e0, e1) * 1e8 / rows,
                               rows / time_ms(e0, e1) / 1e6, rows / (time_ms(e0, e1) * 1e-3) / sms / 1.965e9);
                }
            }
            CK(cudaFree(done));
        }
        CK(cudaFree(t));
    }
    return 0;
}
