// life_dense.cu -- register-tiled DSC / WC for coefficient-dense voxels.
//
// Why: a coefficient needs a whole N_theta-long
// dictionary row.  Streaming that row from shared memory per coefficient
// (the sparse kernels in life_spmv.cu) costs one shared-memory word per FMA,
// a quarter of the FP32 pipe.  When voxels carry a large fraction of all
// atoms (STN96-shaped problems: ~500 coefficients per voxel, 1057 atoms),
// the per-voxel coefficient rows C[v, a] = sum_k w[f_k] value_k are dense
// enough that the product is better done as a register-tiled dense
// contraction  Y(16 voxels x N_theta) += C(16 x 64 atoms) . D(64 x N_theta)
// per (voxel tile, atom chunk), with C built on the fly in shared memory
// from the sorted coefficient stream.  Each lane owns 2 voxels x DPL
// directions (DPL = N_theta_pad / 4) and issues one fma.rn.f32x2 (FFMA2)
// per two FMAs; dictionary chunks are staged by TMA bulk copies into a
// double buffer shared by the CTA.  No tensor cores: the arithmetic stays
// IEEE fp32 FMA on CUDA cores.
//
// WC is the transposed contraction: Z(16 x 64) = Y . D^T per chunk (lane
// partial dots over its DPL directions + a transposing butterfly over the 4
// direction lanes), then each coefficient adds value * Z[cell] to its
// fascicle in 64-bit fixed point (RED.ADD, order independent).
//
// Layout: coefficients sorted by (voxel tile of 16, atom chunk of 64,
// duplicate rank, cell) where cell = (atom%64)*16 + voxel%16 and rank is the
// occurrence index of a (voxel, atom) pair in storage order, so each pass
// over one rank writes distinct cells (no shared-memory atomics, fixed
// summation order: bitwise reproducible).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "life_common.cuh"

namespace life {

constexpr int kTV = 16;           // voxels per warp tile
constexpr int kCA = 64;           // atoms per chunk
constexpr int kCells = kTV * kCA; // 1024
constexpr int kDenseWarps = 8;
constexpr int kDenseThreads = kDenseWarps * 32;

struct DenseArgs {
    const uint32_t *cr;
    const uint32_t *fiber;
    const float *val;
    const uint32_t *tptr;
    const float *D;
    int nv, nt, nt_pad, nch, n_tiles, na;
};

// ---- small PTX helpers --------------------------------------------------------
__device__ __forceinline__ unsigned long long pk(float a, float b)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

__device__ __forceinline__ void upk(unsigned long long r, float &a, float &b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}

// d = a * b + d on two fp32 lanes (one FFMA2)
__device__ __forceinline__ void ffma2(unsigned long long &d, unsigned long long a,
                                      unsigned long long b)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

__device__ __forceinline__ void dmbar_init(uint64_t *bar)
{
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void dmbar_wait(uint64_t *bar, unsigned parity)
{
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "DW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra DW_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}

// TMA bulk copy of one dictionary chunk (bytes multiple of 16) into smem.
__device__ __forceinline__ void issue_chunk(float *dst, const float *src, unsigned bytes,
                                            uint64_t *bar)
{
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
    for (unsigned off = 0; off < bytes; off += 32768u) {
        const unsigned sz = min(32768u, bytes - off);
        const unsigned dd = static_cast<unsigned>(__cvta_generic_to_shared(d + off));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dd),
            "l"(s + off), "r"(sz), "r"(b)
            : "memory");
    }
}

template <int BT>
__device__ __forceinline__ bool dense_last_block(unsigned *counter)
{
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

template <int BT, typename T, typename Op>
__device__ T dense_reduce(const T *part, int n, T init, Op op)
{
    __shared__ T s[32];
    T acc = init;
    for (int i = threadIdx.x; i < n; i += BT) acc = op(acc, __ldcg(part + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = op(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    T r = init;
    if (threadIdx.x < 32) {
        r = threadIdx.x < BT / 32 ? s[threadIdx.x] : init;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = op(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (threadIdx.x == 0) s[0] = r;
    }
    __syncthreads();
    r = s[0];
    __syncthreads();
    return r;
}

struct DAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct DMax {
    __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};

// ---- C tile build: C[cell] = sum of w[f]*value over the cell's coefficients,
//      in rank (= storage) order; returns the number of exact-zero products.
__device__ __forceinline__ unsigned build_ctile(float *C, const DenseArgs &A,
                                                const float *__restrict__ w,
                                                uint32_t p0, uint32_t p1, int lane)
{
    float4 *C4 = reinterpret_cast<float4 *>(C);
#pragma unroll
    for (int i = 0; i < kCells / 4 / 32; ++i) C4[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    unsigned zeros = 0;
    for (uint32_t base = p0; base < p1; base += 64) {
        const uint32_t k0 = base + lane, k1 = base + 32 + lane;
        const bool v0 = k0 < p1, v1 = k1 < p1;
        uint32_t cr0 = 0, cr1 = 0, f0 = 0, f1 = 0;
        float a0 = 0.f, a1 = 0.f;
        if (v0) {
            cr0 = ld_stream(A.cr + k0);
            f0 = ld_stream(A.fiber + k0);
            a0 = ld_stream(A.val + k0);
        }
        if (v1) {
            cr1 = ld_stream(A.cr + k1);
            f1 = ld_stream(A.fiber + k1);
            a1 = ld_stream(A.val + k1);
        }
        const float s0 = v0 ? __fmul_rn(__ldg(w + f0), a0) : 0.f;
        const float s1 = v1 ? __fmul_rn(__ldg(w + f1), a1) : 0.f;
        zeros += __popc(__ballot_sync(0xffffffffu, v0 && s0 == 0.f)) +
                 __popc(__ballot_sync(0xffffffffu, v1 && s1 == 0.f));
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const bool v = half ? v1 : v0;
            const uint32_t cr = half ? cr1 : cr0;
            const float s = half ? s1 : s0;
            const uint32_t r = cr >> 10, cell = cr & 1023u;
            const uint32_t rmin = __reduce_min_sync(0xffffffffu, v ? r : 0xFFFFFFFFu);
            const uint32_t rmax = __reduce_max_sync(0xffffffffu, v ? r : 0u);
            for (uint32_t rr = rmin; rr <= rmax && rmin != 0xFFFFFFFFu; ++rr) {
                if (v && r == rr) {
                    if (rr == 0) C[cell] = s;
                    else C[cell] += s;
                }
                __syncwarp();
            }
        }
    }
    return zeros;
}

// ---------------------------------------------------------------------------
// DSC: Y_tile += C_tile . D_chunk over all chunks, epilogue per voxel row
// ---------------------------------------------------------------------------
template <int DPL>
__global__ void __launch_bounds__(kDenseThreads, 2)
    k_dsc_dense(const DenseArgs A, const float *__restrict__ w, float *__restrict__ y,
                const float *__restrict__ b, const uint32_t flags, const ReduceSlots red,
                const DscOut out, const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar[2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vg = lane >> 2, dg = lane & 3;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kCA * A.nt_pad;
    float *Dbuf = sm;
    float *C = sm + 2 * chunk_floats + warp * kCells;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    const int n_ct = (A.n_tiles + kDenseWarps - 1) / kDenseWarps;
    const int my_tiles = (int)blockIdx.x < n_ct ? (n_ct - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_tiles * A.nch;
    if (threadIdx.x == 0) {
        dmbar_init(&bar[0]);
        dmbar_init(&bar[1]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2 && q < total; ++q)
            issue_chunk(Dbuf + q * chunk_floats, A.D + (size_t)(q % A.nch) * chunk_floats,
                        chunk_bytes, &bar[q]);
    }
    const bool accumulate = flags & LIFE_ACCUMULATE;
    const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
    const bool skip_zero = flags & LIFE_SKIP_ZERO;
    (void)skip_zero;  // zero products add nothing to C; the count is exact either way
    unsigned long long skipped = 0;
    double sq = 0.0;
    float amax = 0.f;
    int step = 0;
    for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
        const int wt = ct * kDenseWarps + warp;
        const bool tile_ok = wt < A.n_tiles;
        unsigned long long acc[2][DPL / 2];
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
            for (int j = 0; j < DPL / 2; ++j) acc[v][j] = 0ull;
        for (int c = 0; c < A.nch; ++c, ++step) {
            const int buf = step & 1;
            if (tile_ok) {
                const uint32_t *tp = A.tptr + (size_t)wt * A.nch + c;
                skipped += build_ctile(C, A, w, tp[0], tp[1], lane);
            }
            __syncwarp();
            dmbar_wait(&bar[buf], (step >> 1) & 1);
            if (tile_ok) {
                const float *D = Dbuf + buf * chunk_floats + dg * DPL;
                const float *Cv = C + vg * 2;
                const int na_c = min(kCA, A.na - c * kCA);
#pragma unroll 2
                for (int a = 0; a < na_c; ++a) {
                    const float2 cc = *reinterpret_cast<const float2 *>(Cv + a * kTV);
                    const float4 *d4 = reinterpret_cast<const float4 *>(D + a * A.nt_pad);
                    unsigned long long dp[DPL / 2];
#pragma unroll
                    for (int i = 0; i < DPL / 4; ++i) {
                        const float4 t = d4[i];
                        dp[2 * i] = pk(t.x, t.y);
                        dp[2 * i + 1] = pk(t.z, t.w);
                    }
                    const unsigned long long c0 = pk(cc.x, cc.x), c1 = pk(cc.y, cc.y);
#pragma unroll
                    for (int j = 0; j < DPL / 2; ++j) {
                        ffma2(acc[0][j], dp[j], c0);
                        ffma2(acc[1][j], dp[j], c1);
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0 && step + 2 < total)
                issue_chunk(Dbuf + buf * chunk_floats,
                            A.D + (size_t)((step + 2) % A.nch) * chunk_floats, chunk_bytes,
                            &bar[buf]);
        }
        if (tile_ok) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int voxel = wt * kTV + vg * 2 + v;
                if (voxel >= A.nv) continue;
                const size_t yo = (size_t)voxel * A.nt;
#pragma unroll
                for (int j = 0; j < DPL / 2; ++j) {
                    float o[2];
                    upk(acc[v][j], o[0], o[1]);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int t = dg * DPL + 2 * j + e;
                        if (t < A.nt) {
                            float r = o[e];
                            if (accumulate) r += y[yo + t];
                            if (subtract) r -= b[yo + t];
                            y[yo + t] = r;
                            sq += (double)r * (double)r;
                            amax = fmaxf(amax, fabsf(r));
                        }
                    }
                }
            }
        }
    }
    // fixed-order completion
    const int gw = blockIdx.x * kDenseWarps + warp;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    if (lane == 0) {
        red.part_d[gw] = sq;
        red.part_u[gw] = skipped;
        red.part_f[gw] = amax;
    }
    if (dense_last_block<kDenseThreads>(red.counter)) {
        const int W = gridDim.x * kDenseWarps;
        const double tsq = dense_reduce<kDenseThreads, double>(red.part_d, W, 0.0, DAdd{});
        const unsigned long long tsk =
            dense_reduce<kDenseThreads, unsigned long long>(red.part_u, W, 0ull, DAdd{});
        const float tmax = dense_reduce<kDenseThreads, float>(red.part_f, W, 0.f, DMax{});
        if (threadIdx.x == 0) {
            if (out.sumsq) *out.sumsq = tsq;
            if (out.skipped) *out.skipped = tsk;
            if (out.skipped_d) *out.skipped_d = (double)tsk;
            if (out.absmax) *out.absmax = tmax;
            *red.counter = 0;
            if (hooks.t_accum && hooks.t_begin) *hooks.t_accum += globaltimer() - *hooks.t_begin;
        }
    }
}

// ---------------------------------------------------------------------------
// WC: Z_tile = Y_tile . D_chunk^T, then value*Z[cell] -> fixed-point fascicle sums
// ---------------------------------------------------------------------------
using DenseFix = FixParams;

template <int DPL>
__global__ void __launch_bounds__(kDenseThreads, 2)
    k_wc_dense(const DenseArgs A, const float *__restrict__ y, const DenseFix fx,
               const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar[2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vg = lane >> 2, dg = lane & 3;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kCA * A.nt_pad;
    float *Dbuf = sm;
    float *Z = sm + 2 * chunk_floats + warp * kCells;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    const int n_ct = (A.n_tiles + kDenseWarps - 1) / kDenseWarps;
    const int my_tiles = (int)blockIdx.x < n_ct ? (n_ct - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_tiles * A.nch;
    const int ex = fix_exponent(fx, A.nt);
    const double scale = ldexp(1.0, ex);
    if (threadIdx.x == 0) {
        dmbar_init(&bar[0]);
        dmbar_init(&bar[1]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2 && q < total; ++q)
            issue_chunk(Dbuf + q * chunk_floats, A.D + (size_t)(q % A.nch) * chunk_floats,
                        chunk_bytes, &bar[q]);
    }
    int step = 0;
    for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
        const int wt = ct * kDenseWarps + warp;
        const bool tile_ok = wt < A.n_tiles;
        // this lane's 2 voxel rows x DPL directions of y, as fp32 pairs
        unsigned long long yp[2][DPL / 2];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int voxel = wt * kTV + vg * 2 + v;
            const bool ok = tile_ok && voxel < A.nv;
            const size_t yo = (size_t)(ok ? voxel : 0) * A.nt;
#pragma unroll
            for (int j = 0; j < DPL / 2; ++j) {
                const int t = dg * DPL + 2 * j;
                const float e0 = (ok && t < A.nt) ? y[yo + t] : 0.f;
                const float e1 = (ok && t + 1 < A.nt) ? y[yo + t + 1] : 0.f;
                yp[v][j] = pk(e0, e1);
            }
        }
        for (int c = 0; c < A.nch; ++c, ++step) {
            const int buf = step & 1;
            dmbar_wait(&bar[buf], (step >> 1) & 1);
            if (tile_ok) {
                const float *D = Dbuf + buf * chunk_floats + dg * DPL;
                const int na_c = min(kCA, A.na - c * kCA);
                for (int a0 = 0; a0 < na_c; a0 += 4) {
                    unsigned long long p[4][2];
#pragma unroll
                    for (int aa = 0; aa < 4; ++aa) {
                        p[aa][0] = 0ull;
                        p[aa][1] = 0ull;
                        const float4 *d4 = reinterpret_cast<const float4 *>(D + (a0 + aa) * A.nt_pad);
#pragma unroll
                        for (int i = 0; i < DPL / 4; ++i) {
                            const float4 t = d4[i];
                            const unsigned long long da = pk(t.x, t.y), db = pk(t.z, t.w);
                            ffma2(p[aa][0], yp[0][2 * i], da);
                            ffma2(p[aa][0], yp[0][2 * i + 1], db);
                            ffma2(p[aa][1], yp[1][2 * i], da);
                            ffma2(p[aa][1], yp[1][2 * i + 1], db);
                        }
                    }
                    float q[8];
#pragma unroll
                    for (int aa = 0; aa < 4; ++aa)
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            float lo, hi;
                            upk(p[aa][v], lo, hi);
                            q[aa * 2 + v] = lo + hi;
                        }
                    // butterfly over the 4 direction lanes: lane dg ends with
                    // atom a0+dg, voxels vg*2 + {0, 1}
                    {
                        const bool up = (lane & 2) != 0;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float send = up ? q[i] : q[i + 4];
                            const float keep = up ? q[i + 4] : q[i];
                            q[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
                        }
                    }
                    {
                        const bool up = (lane & 1) != 0;
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const float send = up ? q[i] : q[i + 2];
                            const float keep = up ? q[i + 2] : q[i];
                            q[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
                        }
                    }
                    *reinterpret_cast<float2 *>(Z + (a0 + dg) * kTV + vg * 2) = make_float2(q[0], q[1]);
                }
                __syncwarp();
                const uint32_t *tp = A.tptr + (size_t)wt * A.nch + c;
                const uint32_t p0 = tp[0], p1 = tp[1];
                for (uint32_t base = p0; base < p1; base += 32) {
                    const uint32_t k = base + lane;
                    if (k < p1) {
                        const uint32_t cell = ld_stream(A.cr + k) & 1023u;
                        const uint32_t f = ld_stream(A.fiber + k);
                        const float vv = ld_stream(A.val + k);
                        const float z = Z[cell] * vv;
                        const long long qv = __double2ll_rn((double)z * scale);
                        atomicAdd(fx.wfix + f, static_cast<unsigned long long>(qv));
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0 && step + 2 < total)
                issue_chunk(Dbuf + buf * chunk_floats,
                            A.D + (size_t)((step + 2) % A.nch) * chunk_floats, chunk_bytes,
                            &bar[buf]);
        }
    }
}

// ---------------------------------------------------------------------------
// layout construction
// ---------------------------------------------------------------------------
__global__ void k_dense_key1(const uint32_t *a, const uint32_t *v, int64_t n, int nch, int tv,
                             int cell_bits, unsigned long long *key, uint32_t *iota)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t at = a[i], vx = v[i];
        const unsigned long long tc = (unsigned long long)(vx / tv) * nch + at / kCA;
        const uint32_t cell = (at % kCA) * tv + vx % tv;
        key[i] = (tc << cell_bits) | cell;
        iota[i] = (uint32_t)i;
    }
}

// warp-specialized layout: one segment per (CTA tile round ct, atom chunk,
// producer warp p) = a pair of adjacent tiles, so one producer warp's step is
// one segment; cell (11 bits) = tile-in-pair, atom in chunk, voxel slot
__global__ void k_voxel_hist(const uint32_t *v, int64_t n, unsigned *cnt)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + v[i], 1u);
}

__global__ void k_ws_key1(const uint32_t *a, const uint32_t *v, const uint32_t *vslot, int64_t n,
                          int nch, int ca, int nprod, unsigned long long *key, uint32_t *iota)
{
    const int tpp = 8 / nprod, cbits = tpp == 2 ? 11 : 10;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t at = a[i], slot = vslot[v[i]];
        const uint32_t tile = slot / 32u;
        const unsigned long long seg =
            ((unsigned long long)(tile / 8u) * nch + at / ca) * nprod + (tile % 8u) / tpp;
        const uint32_t cell = (tile % tpp) << 10 | (at % ca) * 32u + slot % 32u;
        key[i] = (seg << cbits) | cell;
        iota[i] = (uint32_t)i;
    }
}

// tensor-core layout (life_tc.cu): 16-voxel row blocks, 8 per CTA tile of 128
// voxels; segment = (CTA tile, atom chunk of 32, row block); cell = fp32 index
// of (row, atom) in the K-major SWIZZLE_128B A tile (8-row groups of 1024 B,
// 16-byte units XOR-swizzled by row % 8)
__host__ __device__ __forceinline__ uint32_t tc_cell(uint32_t row, uint32_t k)
{
    return (row >> 3) * 256u + (row & 7u) * 32u + ((((k >> 2) ^ row) & 7u) << 2) + (k & 3u);
}

__global__ void k_tc_key1(const uint32_t *a, const uint32_t *v, const uint32_t *vslot, int64_t n,
                          int nch, unsigned long long *key, uint32_t *iota)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t at = a[i], slot = vslot[v[i]];
        const uint32_t blk = slot / 16u;  // row block of 16 voxels
        const unsigned long long seg =
            ((unsigned long long)(blk / 8u) * nch + at / (uint32_t)kTcCA) * 8u + blk % 8u;
        const uint32_t cell = tc_cell(slot % (uint32_t)kTcTV, at % (uint32_t)kTcCA);
        key[i] = (seg << kTcCellBits) | cell;
        iota[i] = (uint32_t)i;
    }
}

// rank = position within the run of equal keys;
// key2 = tc<<32 | rank<<cell_bits | cell
__global__ void k_dense_key2(const unsigned long long *sk, int64_t n, int cell_bits,
                             unsigned long long *key2, unsigned *max_rank)
{
    unsigned mr = 0;
    const unsigned long long cmask = (1ull << cell_bits) - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = sk[i];
        int64_t lo = 0, hi = i;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sk[mid] < k) lo = mid + 1; else hi = mid;
        }
        const unsigned long long rank = (unsigned long long)(i - lo);
        mr = max(mr, rank > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)rank);
        key2[i] = ((k >> cell_bits) << 32) | (rank << cell_bits) | (k & cmask);
    }
    atomicMax(max_rank, mr);
}

// cr = (mixed << 31) | rank << cell_bits | cell.  "mixed" (warp-specialized
// layout only) marks entries of a 32-entry window, counted from the start of
// their (tile, chunk) segment, whose ranks differ: only those windows need
// the ordered per-rank pass when building the coefficient tile.
__global__ void k_dense_gather(const unsigned long long *sk2, const uint32_t *perm, int64_t n,
                               const uint32_t *f, const double *val, const uint32_t *tptr,
                               int cell_bits, int mark_mixed, uint32_t *cr_out,
                               uint32_t *f_out, float *val_out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[i];
        const unsigned long long k = sk2[i];
        uint32_t cr = (uint32_t)(k & 0xFFFFFFFFull);
        if (mark_mixed) {
            const uint32_t tc = (uint32_t)(k >> 32);
            const int64_t seg0 = tptr[tc], seg1 = tptr[tc + 1];
            const int64_t w0 = seg0 + ((i - seg0) / 32) * 32;
            const int64_t w1 = (w0 + 32 < seg1 ? w0 + 32 : seg1) - 1;
            const uint32_t r0 = (uint32_t)(sk2[w0] & 0xFFFFFFFFull) >> cell_bits;
            const uint32_t r1 = (uint32_t)(sk2[w1] & 0xFFFFFFFFull) >> cell_bits;
            if (r0 != r1) cr |= 0x80000000u;
        }
        cr_out[i] = cr;
        f_out[i] = f[p];
        val_out[i] = (float)val[p];
    }
}

__global__ void k_dense_tptr(const unsigned long long *sk2, int64_t n, int64_t ntc, uint32_t *tptr)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= ntc;
         s += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)(sk2[mid] >> 32) < s) lo = mid + 1; else hi = mid;
        }
        tptr[s] = (uint32_t)lo;
    }
}

// ---- warp-specialized layout: per (tile, chunk) segment a rank-0 region
// (distinct cells) and a rank>=1 region, each padded to a multiple of 4
// entries (fiber = kWsSentinel) so producer warps stream 16-byte vectors.
constexpr uint32_t kWsSentinel = 0xFFFFFFFFu;

__global__ void k_ws_bounds(const unsigned long long *sk2, int64_t n, int64_t ntc, int cell_bits,
                            uint32_t *s0, uint32_t *s1)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntc;
         t += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k0 = (unsigned long long)t << 32;
        const unsigned long long k1 = k0 | (1ull << cell_bits);
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sk2[mid] < k0) lo = mid + 1; else hi = mid;
        }
        s0[t] = (uint32_t)lo;
        hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sk2[mid] < k1) lo = mid + 1; else hi = mid;
        }
        s1[t] = (uint32_t)lo;
    }
}

__global__ void k_ws_scatter(const unsigned long long *sk2, const uint32_t *perm, int64_t n,
                             const uint32_t *f, const double *val, const uint32_t *s0,
                             const uint32_t *s1, const uint32_t *P, const uint32_t *T1,
                             int cell_bits, uint32_t *cr_out, uint32_t *f_out, float *val_out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = sk2[i];
        const uint32_t tc = (uint32_t)(k >> 32);
        uint32_t cr = (uint32_t)(k & 0xFFFFFFFFull);
        const uint32_t rank = cr >> cell_bits;
        int64_t dest;
        if (rank == 0) {
            dest = (int64_t)P[tc] + (i - (int64_t)s0[tc]);
        } else {
            const int64_t o = i - (int64_t)s1[tc];
            dest = (int64_t)T1[tc] + o;
            // windows of 32 counted from the start of the rank>=1 region
            const int64_t w0 = (int64_t)s1[tc] + (o / 32) * 32;
            const int64_t end = s0[tc + 1];
            const int64_t w1 = (w0 + 32 < end ? w0 + 32 : end) - 1;
            const uint32_t r0 = (uint32_t)(sk2[w0] & 0xFFFFFFFFull) >> cell_bits;
            const uint32_t r1 = (uint32_t)(sk2[w1] & 0xFFFFFFFFull) >> cell_bits;
            if (r0 != r1) cr |= 0x80000000u;
        }
        const uint32_t p = perm[i];
        cr_out[dest] = cr;
        f_out[dest] = f[p];
        val_out[dest] = (float)val[p];
    }
}

// tensor-core layout: entries packed as pk = fascicle << 12 | cell (fascicles
// < 2^20 - 1; all ones = pad) and stored as 32-byte quads {pk[4], value[4]} so
// one bulk copy stages a whole step (all 8 producer segments)
__global__ void k_tc_pad(uint32_t *q, int64_t nquads)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nquads;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint4 *o = reinterpret_cast<uint4 *>(q + i * 8);
        o[0] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        o[1] = make_uint4(0u, 0u, 0u, 0u);
    }
}

__global__ void k_tc_scatter(const unsigned long long *sk2, const uint32_t *perm, int64_t n,
                             const uint32_t *f, const double *val, const uint32_t *s0,
                             const uint32_t *s1, const uint32_t *P, const uint32_t *T1, uint32_t *q)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = sk2[i];
        const uint32_t tc = (uint32_t)(k >> 32);
        const uint32_t cr = (uint32_t)(k & 0xFFFFFFFFull);
        const uint32_t rank = cr >> kTcCellBits;
        const int64_t dest = rank == 0 ? (int64_t)P[tc] + (i - (int64_t)s0[tc])
                                       : (int64_t)T1[tc] + (i - (int64_t)s1[tc]);
        const uint32_t p = perm[i];
        uint32_t *o = q + (dest >> 2) * 8 + (dest & 3);
        o[0] = (f[p] << kTcCellBits) | (cr & ((1u << kTcCellBits) - 1));
        const float v = (float)val[p];
        o[4] = __float_as_uint(v);
    }
}

static int gridn(int64_t n)
{
    int64_t b = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 65535 * 8));
}

static int dense_supported_dpl(int nt_pad)
{
    const int dpl = nt_pad / 4;
    switch (dpl) {
    case 4: case 8: case 12: case 16: case 20: case 24: case 32: case 40: return dpl;
    default: return 0;
    }
}

static int pad_dirs(int nt)
{
    int p = (nt + 15) / 16 * 16;
    if (p > 96 && p <= 128) p = 128;
    else if (p > 128 && p <= 160) p = 160;
    return p;
}

size_t ws_smem_bytes(int nt_pad, bool staged);
int ws_warps();
int ws_chunk_atoms();
int ws_slot_entries();
int ws_producers();

int build_dense(life_phi *phi, const uint32_t *a, const uint32_t *v, const uint32_t *f,
                const double *val, const std::vector<double> &hdict, cudaStream_t st)
{
    const int64_t n = phi->nc;
    // warp-specialized kernels (life_ws.cu) for n_dirs <= 96, the v1
    // register-tiled kernels above for n_dirs <= 160, else sparse only
    int kind = 2, tv = 32, ca = ws_chunk_atoms();
    int cell_bits = ws_producers() == 4 ? 11 : 10;
    int nt_pad = (phi->nt + 31) / 32 * 32;
    if (nt_pad > 96) {
        kind = 1;
        tv = kTV;
        cell_bits = 10;
        ca = kCA;
        nt_pad = pad_dirs(phi->nt);
        if (!dense_supported_dpl(nt_pad)) return LIFE_OK;
    }
    if (n == 0) return LIFE_OK;
    phi->d_kind = kind;
    phi->d_tv = tv;
    phi->d_ca = ca;
    phi->nt_pad = nt_pad;
    phi->n_tiles = (phi->nv + tv - 1) / tv;
    phi->n_chunks = (phi->na + ca - 1) / ca;
    // ws: whole CTA rounds of 8 tiles (segments of missing tiles stay empty)
    const int64_t n_ct = ((int64_t)phi->n_tiles + 7) / 8;
    // ws: one segment per producer warp and step (its one or two tiles)
    const int64_t ntc = kind == 2 ? n_ct * phi->n_chunks * ws_producers()
                                  : (int64_t)phi->n_tiles * phi->n_chunks;
    if (ntc >= (1ll << 31)) return LIFE_OK;
    unsigned long long *k1 = nullptr, *sk1 = nullptr, *k2 = nullptr, *sk2 = nullptr;
    uint32_t *iota = nullptr, *perm1 = nullptr, *perm = nullptr;
    unsigned *mr = nullptr;
    LIFE_CUDA(cudaMallocAsync(&k1, n * 8, st));
    LIFE_CUDA(cudaMallocAsync(&sk1, n * 8, st));
    LIFE_CUDA(cudaMallocAsync(&iota, n * 4, st));
    LIFE_CUDA(cudaMallocAsync(&perm1, n * 4, st));
    LIFE_CUDA(cudaMallocAsync(&mr, 4, st));
    LIFE_CUDA(cudaMemsetAsync(mr, 0, 4, st));
    if (kind == 2) {
        // Load balance: voxels sorted by coefficient count are dealt to the
        // tiles in snake order (round r gives tile i, or T-1-i on odd rounds,
        // its r-th slot), so every 32-voxel tile -- and every CTA's step --
        // carries about the same number of coefficients.  y rows are read and
        // written through slot -> voxel; the arithmetic per voxel is unchanged.
        unsigned *cnt = nullptr;
        LIFE_CUDA(cudaMallocAsync(&cnt, (size_t)phi->nv * 4, st));
        LIFE_CUDA(cudaMemsetAsync(cnt, 0, (size_t)phi->nv * 4, st));
        k_voxel_hist<<<gridn(n), 256, 0, st>>>(v, n, cnt);
        LIFE_CHECK_LAUNCH();
        std::vector<unsigned> hc(phi->nv);
        LIFE_CUDA(cudaMemcpyAsync(hc.data(), cnt, (size_t)phi->nv * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        LIFE_CUDA(cudaFreeAsync(cnt, st));
        std::vector<uint32_t> order(phi->nv);
        for (int i = 0; i < phi->nv; ++i) order[i] = (uint32_t)i;
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t x, uint32_t y) { return hc[x] > hc[y]; });
        const int64_t T = phi->n_tiles, nslots = n_ct * 8 * 32;
        std::vector<uint32_t> vslot(phi->nv);
        std::vector<int> slotv(nslots, -1);
        for (int64_t i = 0; i < phi->nv; ++i) {
            const int64_t r = i / T, q = i % T, tile = (r & 1) ? T - 1 - q : q;
            const int64_t slot = tile * 32 + r;
            vslot[order[i]] = (uint32_t)slot;
            slotv[slot] = (int)order[i];
        }
        LIFE_TRY(dalloc(phi, &phi->d_vslot, (size_t)phi->nv));
        LIFE_TRY(dalloc(phi, &phi->d_slotv, (size_t)nslots));
        LIFE_CUDA(cudaMemcpyAsync(phi->d_vslot, vslot.data(), (size_t)phi->nv * 4,
                                  cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaMemcpyAsync(phi->d_slotv, slotv.data(), (size_t)nslots * 4,
                                  cudaMemcpyHostToDevice, st));
        k_ws_key1<<<gridn(n), 256, 0, st>>>(a, v, phi->d_vslot, n, phi->n_chunks, ca,
                                             ws_producers(), k1, iota);
        LIFE_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    }
    else
        k_dense_key1<<<gridn(n), 256, 0, st>>>(a, v, n, phi->n_chunks, tv, cell_bits, k1, iota);
    LIFE_CHECK_LAUNCH();
    int bits_tc = 1;
    while (bits_tc < 40 && (ntc >> bits_tc) != 0) ++bits_tc;
    size_t tb = 0;
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, sk1, iota, perm1, n, 0, cell_bits + bits_tc, st));
    void *temp = nullptr;
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, k1, sk1, iota, perm1, n, 0, cell_bits + bits_tc, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    LIFE_CUDA(cudaFreeAsync(k1, st));
    LIFE_CUDA(cudaFreeAsync(iota, st));
    LIFE_CUDA(cudaMallocAsync(&k2, n * 8, st));
    k_dense_key2<<<gridn(n), 256, 0, st>>>(sk1, n, cell_bits, k2, mr);
    LIFE_CHECK_LAUNCH();
    unsigned hmr = 0;
    LIFE_CUDA(cudaMemcpyAsync(&hmr, mr, 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    // rank field: ws bits cell_bits..29 (bit 30 = pad, 31 = mixed); v1 bits 10..31
    if (hmr >= (kind == 2 ? (1u << (30 - cell_bits)) : (1u << (31 - cell_bits)))) {
        cudaFreeAsync(sk1, st); cudaFreeAsync(perm1, st); cudaFreeAsync(k2, st); cudaFreeAsync(mr, st);
        return LIFE_OK;  // pathological duplicate counts: stay sparse
    }
    LIFE_CUDA(cudaFreeAsync(sk1, st));
    LIFE_CUDA(cudaMallocAsync(&sk2, n * 8, st));
    LIFE_CUDA(cudaMallocAsync(&perm, n * 4, st));
    tb = 0;
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k2, sk2, perm1, perm, n, 0, 32 + bits_tc, st));
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, k2, sk2, perm1, perm, n, 0, 32 + bits_tc, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    LIFE_CUDA(cudaFreeAsync(k2, st));
    LIFE_CUDA(cudaFreeAsync(perm1, st));
    if (kind == 2) {
        uint32_t *s0 = nullptr, *s1 = nullptr, *Pd = nullptr, *T1d = nullptr;
        LIFE_CUDA(cudaMallocAsync(&s0, (ntc + 1) * 4, st));
        LIFE_CUDA(cudaMallocAsync(&s1, (ntc + 1) * 4, st));
        k_ws_bounds<<<gridn(ntc + 1), 256, 0, st>>>(sk2, n, ntc, cell_bits, s0, s1);
        LIFE_CHECK_LAUNCH();
        std::vector<uint32_t> h0(ntc + 1), h1(ntc + 1), hP(ntc + 1), hT(ntc + 1);
        LIFE_CUDA(cudaMemcpyAsync(h0.data(), s0, (ntc + 1) * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaMemcpyAsync(h1.data(), s1, (ntc + 1) * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        int64_t pos = 0;
        for (int64_t t = 0; t < ntc; ++t) {
            const int64_t n0 = (int64_t)h1[t] - h0[t], n1 = (int64_t)h0[t + 1] - h1[t];
            hP[t] = (uint32_t)pos;
            hT[t] = (uint32_t)(pos + (n0 + 3) / 4 * 4);
            pos += (n0 + 3) / 4 * 4 + (n1 + 3) / 4 * 4;
        }
        hP[ntc] = hT[ntc] = (uint32_t)pos;
        if (pos >= 0xFFFFFFFFll) return fail(LIFE_ERR_CONFIG_INVALID, "padded layout exceeds u32");
        // staged producers copy one segment per step into a fixed slot
        int64_t maxpw = 0;
        for (int64_t t = 0; t < ntc; ++t) maxpw = std::max<int64_t>(maxpw, (int64_t)hP[t + 1] - hP[t]);
        const int64_t maxpair = maxpw;
        phi->d_maxpw = maxpw;
        const char *unstaged = getenv("LIFE_WS_UNSTAGED");  // A/B diagnostics
        phi->d_staged = maxpw <= ws_slot_entries() && !(unstaged && unstaged[0] == '1');
        if (getenv("LIFE_DEBUG"))
            fprintf(stderr, "[life] ws layout: ntc=%lld padded=%lld maxpw=%lld maxpair=%lld staged=%d\n",
                    (long long)ntc, (long long)pos, (long long)maxpw, (long long)maxpair,
                    (int)phi->d_staged);
        const int64_t npad = std::max<int64_t>(pos, 1);
        LIFE_TRY(dalloc(phi, &phi->d_cr, npad));
        LIFE_TRY(dalloc(phi, &phi->d_fiber, npad));
        LIFE_TRY(dalloc(phi, &phi->d_val, npad));
        LIFE_TRY(dalloc(phi, &phi->d_tptr, ntc + 1));
        LIFE_TRY(dalloc(phi, &phi->d_t1, ntc + 1));
        LIFE_CUDA(cudaMemsetAsync(phi->d_cr, 0x40, npad * 4, st));  // pad bit 30
        LIFE_CUDA(cudaMemsetAsync(phi->d_fiber, 0xFF, npad * 4, st));  // kWsSentinel
        LIFE_CUDA(cudaMemsetAsync(phi->d_val, 0, npad * 4, st));
        LIFE_CUDA(cudaMemcpyAsync(phi->d_tptr, hP.data(), (ntc + 1) * 4, cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaMemcpyAsync(phi->d_t1, hT.data(), (ntc + 1) * 4, cudaMemcpyHostToDevice, st));
        k_ws_scatter<<<gridn(n), 256, 0, st>>>(sk2, perm, n, f, val, s0, s1, phi->d_tptr,
                                               phi->d_t1, cell_bits, phi->d_cr, phi->d_fiber,
                                               phi->d_val);
        LIFE_CHECK_LAUNCH();
        phi->d_npad = pos;
        LIFE_CUDA(cudaStreamSynchronize(st));
        LIFE_CUDA(cudaFreeAsync(s0, st));
        LIFE_CUDA(cudaFreeAsync(s1, st));
        (void)Pd;
        (void)T1d;
    } else {
        LIFE_TRY(dalloc(phi, &phi->d_cr, n));
        LIFE_TRY(dalloc(phi, &phi->d_fiber, n));
        LIFE_TRY(dalloc(phi, &phi->d_val, n));
        LIFE_TRY(dalloc(phi, &phi->d_tptr, ntc + 1));
        k_dense_tptr<<<gridn(ntc + 1), 256, 0, st>>>(sk2, n, ntc, phi->d_tptr);
        LIFE_CHECK_LAUNCH();
        k_dense_gather<<<gridn(n), 256, 0, st>>>(sk2, perm, n, f, val, phi->d_tptr, cell_bits, 0,
                                                 phi->d_cr, phi->d_fiber, phi->d_val);
        LIFE_CHECK_LAUNCH();
    }
    LIFE_CUDA(cudaFreeAsync(sk2, st));
    LIFE_CUDA(cudaFreeAsync(perm, st));
    LIFE_CUDA(cudaFreeAsync(mr, st));
    // zero-padded dictionary chunks [n_chunks][ca][nt_pad]
    std::vector<float> hD((size_t)phi->n_chunks * ca * nt_pad, 0.f);
    for (int at = 0; at < phi->na; ++at)
        for (int t = 0; t < phi->nt; ++t)
            hD[(size_t)at * nt_pad + t] = (float)hdict[(size_t)at * phi->nt + t];
    LIFE_TRY(dalloc(phi, &phi->d_D, hD.size()));
    LIFE_CUDA(cudaMemcpyAsync(phi->d_D, hD.data(), hD.size() * 4, cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    if (kind == 2) {
        phi->d_smem = ws_smem_bytes(nt_pad, phi->d_staged);
        phi->d_blocks = phi->sms;
        phi->d_W = phi->d_blocks * ws_warps();
    } else {
        phi->d_smem = ((size_t)2 * kCA * nt_pad + (size_t)kDenseWarps * kCells) * sizeof(float);
        // residency: 2 CTAs per SM when shared memory allows
        const int bps = (2 * (phi->d_smem + 1024) <= 227 * 1024) ? 2 : 1;
        phi->d_blocks = phi->sms * bps;
        phi->d_W = phi->d_blocks * kDenseWarps;
    }
    phi->has_dense = true;
    return LIFE_OK;
}

// ---------------------------------------------------------------------------
// tensor-core layout (life_tc.cu)
// ---------------------------------------------------------------------------
static void tf32_split(float x, float &hi, float &lo)
{
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    std::memcpy(&hi, &u, 4);
    lo = x - hi;
}

// B operand of the tensor-core WC (k_wc_tc): per chunk the dictionary rows
// of its 32 atoms (N) over nt_pad directions (K), K-major SWIZZLE_128B in
// blocks of 32 directions (4 KB each), split into tf32 hi and lo
int build_wc_tc(life_phi *phi, const std::vector<double> &hdict, cudaStream_t st)
{
    if (phi->d_kind != 2 || phi->nt_pad % 32 != 0 || phi->d_ca != 32) return LIFE_OK;
    const int nkb = phi->nt_pad / 32, nch = phi->n_chunks;
    const size_t per = (size_t)2 * nkb * 32 * 32;
    std::vector<float> hB((size_t)nch * per, 0.f);
    for (int c = 0; c < nch; ++c)
        for (int n = 0; n < 32; ++n)
            for (int t = 0; t < phi->nt_pad; ++t) {
                const int at = c * 32 + n;
                const float x = (at < phi->na && t < phi->nt) ? (float)hdict[(size_t)at * phi->nt + t] : 0.f;
                float hi, lo;
                tf32_split(x, hi, lo);
                const size_t o = (size_t)c * per + (size_t)(t / 32) * 1024 + tc_cell(n, t % 32);
                hB[o] = hi;
                hB[o + (size_t)nkb * 1024] = lo;
            }
    LIFE_TRY(dalloc(phi, &phi->d_Bwc, hB.size()));
    LIFE_CUDA(cudaMemcpyAsync(phi->d_Bwc, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    return LIFE_OK;
}

int build_tc(life_phi *phi, const uint32_t *a, const uint32_t *v, const uint32_t *f,
             const double *val, const std::vector<double> &hdict, cudaStream_t st)
{
    const int64_t n = phi->nc;
    const int N = (phi->nt + 31) / 32 * 32;  // MMA N: directions padded to 32
    if (n == 0 || N > 128 || phi->nf >= (1 << 20) - 1) return LIFE_OK;
    const int nch = (phi->na + kTcCA - 1) / kTcCA;
    const int64_t nblk = ((int64_t)phi->nv + 15) / 16;   // 16-voxel row blocks
    const int64_t n_ct = (nblk + 7) / 8;                 // CTA tiles of 128 voxels
    const int64_t ntc = n_ct * nch * kTcProd;            // segments
    if (ntc >= (1ll << 31)) return LIFE_OK;
    // Load balance: voxels sorted by coefficient count are dealt to the row
    // blocks in snake order, so every producer warp's segment carries about
    // the same number of coefficients.
    std::vector<uint32_t> vslot(phi->nv);
    const int64_t nslots = n_ct * kTcTV;
    std::vector<int> slotv(nslots, -1);
    {
        unsigned *cnt = nullptr;
        LIFE_CUDA(cudaMallocAsync(&cnt, (size_t)phi->nv * 4, st));
        LIFE_CUDA(cudaMemsetAsync(cnt, 0, (size_t)phi->nv * 4, st));
        k_voxel_hist<<<gridn(n), 256, 0, st>>>(v, n, cnt);
        LIFE_CHECK_LAUNCH();
        std::vector<unsigned> hc(phi->nv);
        LIFE_CUDA(cudaMemcpyAsync(hc.data(), cnt, (size_t)phi->nv * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        LIFE_CUDA(cudaFreeAsync(cnt, st));
        std::vector<uint32_t> order(phi->nv);
        for (int i = 0; i < phi->nv; ++i) order[i] = (uint32_t)i;
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t x, uint32_t y) { return hc[x] > hc[y]; });
        for (int64_t i = 0; i < phi->nv; ++i) {
            const int64_t r = i / nblk, q = i % nblk, blk = (r & 1) ? nblk - 1 - q : q;
            const int64_t slot = blk * 16 + r;
            vslot[order[i]] = (uint32_t)slot;
            slotv[slot] = (int)order[i];
        }
    }
    LIFE_TRY(dalloc(phi, &phi->t_vslot, (size_t)phi->nv));
    LIFE_TRY(dalloc(phi, &phi->t_slotv, (size_t)nslots));
    LIFE_CUDA(cudaMemcpyAsync(phi->t_vslot, vslot.data(), (size_t)phi->nv * 4, cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaMemcpyAsync(phi->t_slotv, slotv.data(), (size_t)nslots * 4, cudaMemcpyHostToDevice, st));
    unsigned long long *k1 = nullptr, *sk1 = nullptr, *k2 = nullptr, *sk2 = nullptr;
    uint32_t *iota = nullptr, *perm1 = nullptr, *perm = nullptr;
    unsigned *mr = nullptr;
    LIFE_CUDA(cudaMallocAsync(&k1, n * 8, st));
    LIFE_CUDA(cudaMallocAsync(&sk1, n * 8, st));
    LIFE_CUDA(cudaMallocAsync(&iota, n * 4, st));
    LIFE_CUDA(cudaMallocAsync(&perm1, n * 4, st));
    LIFE_CUDA(cudaMallocAsync(&mr, 4, st));
    LIFE_CUDA(cudaMemsetAsync(mr, 0, 4, st));
    k_tc_key1<<<gridn(n), 256, 0, st>>>(a, v, phi->t_vslot, n, nch, k1, iota);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    int bits_tc = 1;
    while (bits_tc < 40 && (ntc >> bits_tc) != 0) ++bits_tc;
    size_t tb = 0;
    void *temp = nullptr;
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, sk1, iota, perm1, n, 0, kTcCellBits + bits_tc, st));
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, k1, sk1, iota, perm1, n, 0, kTcCellBits + bits_tc, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    LIFE_CUDA(cudaFreeAsync(k1, st));
    LIFE_CUDA(cudaFreeAsync(iota, st));
    LIFE_CUDA(cudaMallocAsync(&k2, n * 8, st));
    k_dense_key2<<<gridn(n), 256, 0, st>>>(sk1, n, kTcCellBits, k2, mr);
    LIFE_CHECK_LAUNCH();
    unsigned hmr = 0;
    LIFE_CUDA(cudaMemcpyAsync(&hmr, mr, 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    LIFE_CUDA(cudaFreeAsync(sk1, st));
    if (hmr >= (1u << (30 - kTcCellBits))) {  // pathological duplicate counts
        cudaFreeAsync(perm1, st); cudaFreeAsync(k2, st); cudaFreeAsync(mr, st);
        return LIFE_OK;
    }
    LIFE_CUDA(cudaMallocAsync(&sk2, n * 8, st));
    LIFE_CUDA(cudaMallocAsync(&perm, n * 4, st));
    tb = 0;
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k2, sk2, perm1, perm, n, 0, 32 + bits_tc, st));
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, k2, sk2, perm1, perm, n, 0, 32 + bits_tc, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    LIFE_CUDA(cudaFreeAsync(k2, st));
    LIFE_CUDA(cudaFreeAsync(perm1, st));
    uint32_t *s0 = nullptr, *s1 = nullptr;
    LIFE_CUDA(cudaMallocAsync(&s0, (ntc + 1) * 4, st));
    LIFE_CUDA(cudaMallocAsync(&s1, (ntc + 1) * 4, st));
    k_ws_bounds<<<gridn(ntc + 1), 256, 0, st>>>(sk2, n, ntc, kTcCellBits, s0, s1);
    LIFE_CHECK_LAUNCH();
    std::vector<uint32_t> h0(ntc + 1), h1(ntc + 1), hP(ntc + 1), hT(ntc + 1);
    LIFE_CUDA(cudaMemcpyAsync(h0.data(), s0, (ntc + 1) * 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaMemcpyAsync(h1.data(), s1, (ntc + 1) * 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    // rank-0 and rank>=1 regions each padded to 4 entries (16-byte vectors)
    int64_t pos = 0, maxseg = 0, maxstep = 0;
    for (int64_t t = 0; t < ntc; ++t) {
        if (t % kTcProd == 0 && t) maxstep = std::max<int64_t>(maxstep, pos - hP[t - kTcProd]);
        const int64_t n0 = (int64_t)h1[t] - h0[t], n1 = (int64_t)h0[t + 1] - h1[t];
        hP[t] = (uint32_t)pos;
        hT[t] = (uint32_t)(pos + (n0 + 3) / 4 * 4);
        const int64_t len = (n0 + 3) / 4 * 4 + (n1 + 3) / 4 * 4;
        maxseg = std::max(maxseg, len);
        pos += len;
    }
    hP[ntc] = hT[ntc] = (uint32_t)pos;
    if (ntc) maxstep = std::max<int64_t>(maxstep, pos - hP[ntc - kTcProd]);
    if (pos >= 0xFFFFFFFFll) return fail(LIFE_ERR_CONFIG_INVALID, "padded layout exceeds u32");
    const int64_t npad = std::max<int64_t>(pos, 4);
    LIFE_TRY(dalloc(phi, &phi->t_q, (size_t)(npad / 4 + 1) * 8));
    LIFE_TRY(dalloc(phi, &phi->t_tptr, ntc + 1));
    LIFE_TRY(dalloc(phi, &phi->t_t1, ntc + 1));
    k_tc_pad<<<gridn(npad / 4 + 1), 256, 0, st>>>(phi->t_q, npad / 4 + 1);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaMemcpyAsync(phi->t_tptr, hP.data(), (ntc + 1) * 4, cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaMemcpyAsync(phi->t_t1, hT.data(), (ntc + 1) * 4, cudaMemcpyHostToDevice, st));
    k_tc_scatter<<<gridn(n), 256, 0, st>>>(sk2, perm, n, f, val, s0, s1, phi->t_tptr, phi->t_t1,
                                           phi->t_q);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaStreamSynchronize(st));
    LIFE_CUDA(cudaFreeAsync(s0, st));
    LIFE_CUDA(cudaFreeAsync(s1, st));
    LIFE_CUDA(cudaFreeAsync(sk2, st));
    LIFE_CUDA(cudaFreeAsync(perm, st));
    LIFE_CUDA(cudaFreeAsync(mr, st));
    // B operand: per chunk, D^T (N directions x 32 atoms) as the K-major
    // SWIZZLE_128B tile the MMA reads, split hi = tf32(x), lo = x - hi
    std::vector<float> hD((size_t)nch * 2 * N * kTcCA, 0.f);
    for (int c = 0; c < nch; ++c)
        for (int t = 0; t < N; ++t)
            for (int k = 0; k < kTcCA; ++k) {
                const int at = c * kTcCA + k;
                const float x = (at < phi->na && t < phi->nt) ? (float)hdict[(size_t)at * phi->nt + t] : 0.f;
                float hi, lo;
                tf32_split(x, hi, lo);
                const size_t base = (size_t)c * 2 * N * kTcCA;
                hD[base + tc_cell(t, k)] = hi;
                hD[base + (size_t)N * kTcCA + tc_cell(t, k)] = lo;
            }
    LIFE_TRY(dalloc(phi, &phi->t_D, hD.size()));
    LIFE_CUDA(cudaMemcpyAsync(phi->t_D, hD.data(), hD.size() * 4, cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    phi->t_nct = (int)n_ct;
    phi->t_nch = nch;
    phi->t_n = N;
    phi->t_npad = pos;
    phi->t_maxseg = maxseg;
    phi->t_maxstep = maxstep;
    phi->t_blocks = phi->sms;
    if (prepare_tc(phi) != LIFE_OK) {  // sets t_smem, t_W; segments too long: stay on CUDA cores
        ok();
        return LIFE_OK;
    }
    phi->has_tc = true;
    if (getenv("LIFE_DEBUG"))
        fprintf(stderr, "[life] tc layout: n_ct=%lld nch=%d N=%d padded=%lld maxseg=%lld maxstep=%lld maxrank=%u\n",
                (long long)n_ct, nch, N, (long long)pos, (long long)maxseg, (long long)maxstep, hmr);
    return LIFE_OK;
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <int DPL>
static int dense_dsc_t(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                       const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_dsc_dense<DPL>, phi->d_smem));
    DenseArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_D,
                phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
    k_dsc_dense<DPL><<<phi->d_blocks, kDenseThreads, phi->d_smem, st>>>(A, w, y, b, flags,
                                                                         phi->red, o, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int DPL>
static int dense_wc_t(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                      cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_wc_dense<DPL>, phi->d_smem));
    DenseArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_D,
                phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
    k_wc_dense<DPL><<<phi->d_blocks, kDenseThreads, phi->d_smem, st>>>(A, y, fx, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int DPL>
static int dense_prepare_t(life_phi *phi)
{
    LIFE_TRY(ensure_smem(k_dsc_dense<DPL>, phi->d_smem));
    LIFE_TRY(ensure_smem(k_wc_dense<DPL>, phi->d_smem));
    return LIFE_OK;
}

#define LIFE_DPL_DISPATCH(FN, ...)                                             \
    switch (phi->nt_pad / 4) {                                                 \
    case 4: return FN<4>(__VA_ARGS__);                                         \
    case 8: return FN<8>(__VA_ARGS__);                                         \
    case 12: return FN<12>(__VA_ARGS__);                                       \
    case 16: return FN<16>(__VA_ARGS__);                                       \
    case 20: return FN<20>(__VA_ARGS__);                                       \
    case 24: return FN<24>(__VA_ARGS__);                                       \
    case 32: return FN<32>(__VA_ARGS__);                                       \
    case 40: return FN<40>(__VA_ARGS__);                                       \
    default: return fail(LIFE_ERR_CONFIG_INVALID, "dense layout: unsupported n_dirs"); \
    }

int launch_dsc_ws(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                  const DscOut &o, const CallHooks &h, cudaStream_t st);
int launch_wc_ws(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                 cudaStream_t st);
int prepare_ws(life_phi *phi);

static int dense_v1_dsc(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                        const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_DPL_DISPATCH(dense_dsc_t, phi, w, y, b, flags, o, h, st);
}

static int dense_v1_wc(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                       cudaStream_t st)
{
    LIFE_DPL_DISPATCH(dense_wc_t, phi, fx, y, h, st);
}

static int dense_v1_prepare(life_phi *phi) { LIFE_DPL_DISPATCH(dense_prepare_t, phi); }

int launch_dsc_dense(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                     const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    if (phi->d_kind == 2) return launch_dsc_ws(phi, w, y, b, flags, o, h, st);
    return dense_v1_dsc(phi, w, y, b, flags, o, h, st);
}

int launch_wc_dense(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                    cudaStream_t st)
{
    if (phi->d_kind == 2) return launch_wc_ws(phi, fx, y, h, st);
    return dense_v1_wc(phi, fx, y, h, st);
}

int prepare_dense(life_phi *phi)
{
    if (phi->d_kind == 2) return prepare_ws(phi);
    return dense_v1_prepare(phi);
}

}  // namespace life
