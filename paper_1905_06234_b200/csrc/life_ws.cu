// life_ws.cu -- warp-specialized dense DSC / WC (the C2 hot path).
//
// Same contraction as life_dense.cu (Y_tile += C_tile . D_chunk for DSC,
// Z_tile = Y_tile . D_chunk^T then value*Z[cell] -> fascicles for WC), but
// split between two roles inside one persistent CTA per SM:
//
//   4 producer warps  stream the sorted coefficient segment of the next
//                     (voxel tile, atom chunk) step, gather w[f], and build
//                     the 64 x 32 coefficient tile C in shared memory (DSC);
//                     or scatter value * Z[cell] into the fixed-point fascicle
//                     sums with RED.ADD (WC).  Producer warp 0 also issues
//                     the TMA bulk copy of the next dictionary chunk.
//   8 consumer warps  do only register-tiled FFMA2 work: each lane owns
//                     8 voxels x 12 directions (96 fp32 accumulators), so a
//                     dictionary value feeds 8 FMAs and a coefficient 12.
//
// Steps are double buffered (C/Z tiles and dictionary chunks) and handed
// over with mbarriers (full/empty), so coefficient latency hides behind the
// consumers' FMA stream.  Each LDS.128 costs four shared-memory wavefronts on
// sm_100 (measured, tools/ubench); the 8x12 lane tile needs 5 of them per 96
// FMAs per lane, keeping shared memory (80 wavefronts per 96-cycle FMA step
// per SM) below the FP32 pipe.
#include <algorithm>

#include "life_common.cuh"

namespace life {

constexpr int kWsCons = 8;
constexpr int kWsProd = 4;
constexpr int kTPP = kWsCons / kWsProd;   // consumer tiles per producer warp
constexpr int kWsWarps = kWsCons + kWsProd;
constexpr int kWsThreads = kWsWarps * 32;
constexpr int kWsTV = 32;                  // voxels per consumer tile
constexpr int kWsCA = 64;                  // atoms per chunk
constexpr int kWsCells = kWsTV * kWsCA;    // 2048
constexpr int kWsCellBits = 11;
// optional register split between the roles (setmaxnreg, warpgroup-aligned).
// 8 producer warps at 88 registers measured slower than 4 at 168 (C2: DSC
// 1.93 vs 1.72 ms), so the split is off by default.
constexpr bool kSplitRegs = false;
constexpr int kRegCons = 168;
constexpr int kRegProd = 88;
static_assert(kWsCons % 4 == 0 && kWsProd % 4 == 0, "roles must be whole warpgroups");
static_assert(!kSplitRegs || kWsCons * kRegCons + kWsProd * kRegProd <= 2048, "register file");

struct WsArgs {
    const uint32_t *cr;
    const uint32_t *fiber;
    const float *val;
    const uint32_t *tptr;   // padded segment starts, [n_tiles*nch + 1]
    const uint32_t *t1;     // start of each segment's rank>=1 region
    const float *D;
    int nv, nt, nt_pad, nch, n_tiles, na;
};
constexpr uint32_t kSent = 0xFFFFFFFFu;  // padding entry (fiber field)
// Diagnostic isolation, compiled in only with -DLIFE_WS_DIAG (tools/ws_isolate.py):
// c_ws_isolate 1 = producers only, 2 = consumers only (results are garbage);
// c_ws_flags 1 = no L2 prefetch, 2 = __ldg streams, 4 = no gather.
#ifdef LIFE_WS_DIAG
__constant__ int c_ws_isolate = 0;
__constant__ int c_ws_flags = 0;
#else
constexpr int c_ws_isolate = 0;
constexpr int c_ws_flags = 0;
#endif

template <typename T>
__device__ __forceinline__ T ld_s(const T *p)
{
    return (c_ws_flags & 2) ? __ldg(p) : ld_stream(p);
}

__device__ __forceinline__ unsigned long long wpk(float a, float b)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void wupk(unsigned long long r, float &a, float &b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ void wfma2(unsigned long long &d, unsigned long long a,
                                      unsigned long long b)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

__device__ __forceinline__ unsigned smaddr(const void *p)
{
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smaddr(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smaddr(b)) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smaddr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WSW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WSW_%=;\n}" ::"r"(smaddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_chunk(float *dst, const float *src, unsigned bytes, uint64_t *b)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bar_arrive_tx(b, bytes);
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
    for (unsigned off = 0; off < bytes; off += 32768u) {
        const unsigned sz = min(32768u, bytes - off);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smaddr(d + off)),
            "l"(s + off), "r"(sz), "r"(smaddr(b))
            : "memory");
    }
}

template <typename T, typename Op>
__device__ T ws_reduce(const T *part, int n, T init, Op op)
{
    __shared__ T s[32];
    T acc = init;
    for (int i = threadIdx.x; i < n; i += kWsThreads) acc = op(acc, __ldcg(part + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = op(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    T r = init;
    if (threadIdx.x < 32) {
        r = threadIdx.x < kWsWarps ? s[threadIdx.x] : init;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = op(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (threadIdx.x == 0) s[0] = r;
    }
    __syncthreads();
    r = s[0];
    __syncthreads();
    return r;
}
struct WAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct WMax {
    __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};

__device__ __forceinline__ bool ws_last_block(unsigned *counter)
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

// ---- producer: coefficient tile build (DSC) ---------------------------------
// Segment of one (voxel tile, atom chunk): [p0, q0) holds each cell's first
// coefficient (rank 0, distinct cells) and [q0, p1) the repeats (rank >= 1);
// both regions are padded to 4-entry multiples, so the rank-0 region (~75%
// of all coefficients at C2) streams as 16-byte vectors, 4 coefficients per
// lane, with one plain STS per coefficient.  Repeats are added afterwards in
// rank order (windows straddling two ranks, flagged at build time, are
// applied rank by rank).  The next step's segments are prefetched into L2.
struct Seg1 {
    uint32_t p0, q0, p1;
};

__device__ __forceinline__ Seg1 seg_of(const WsArgs &A, int wt, int c)
{
    Seg1 S{0u, 0u, 0u};
    if (wt < A.n_tiles) {
        const size_t tc = (size_t)wt * A.nch + c;
        S.p0 = A.tptr[tc];
        S.q0 = A.t1[tc];
        S.p1 = A.tptr[tc + 1];
    }
    return S;
}

__device__ __forceinline__ void prefetch_l2(const void *ptr, uint32_t bytes)
{
    if (bytes == 0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_seg(const WsArgs &A, const Seg1 &S)
{
    if (S.p1 <= S.p0 || (c_ws_flags & 1)) return;
    const uint32_t bytes = (S.p1 - S.p0) * 4u;  // padded segments are 16-byte aligned
    prefetch_l2(A.cr + S.p0, bytes);
    prefetch_l2(A.fiber + S.p0, bytes);
    prefetch_l2(A.val + S.p0, bytes);
}

// 4 consecutive coefficients per lane (a 128-coefficient block per warp)
struct VBlk {
    uint4 cr, f;
    float4 v;
    float w[4];
    bool ok;
};

__device__ __forceinline__ void vb_load(VBlk &B, const WsArgs &A, uint32_t base, uint32_t end,
                                        int lane)
{
    const uint32_t k = base + 4u * (uint32_t)lane;
    B.ok = k < end;
    if (B.ok) {
        B.cr = ld_s(reinterpret_cast<const uint4 *>(A.cr + k));
        B.f = ld_s(reinterpret_cast<const uint4 *>(A.fiber + k));
        B.v = ld_s(reinterpret_cast<const float4 *>(A.val + k));
    } else {
        B.cr = make_uint4(0u, 0u, 0u, 0u);
        B.f = make_uint4(kSent, kSent, kSent, kSent);
        B.v = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

__device__ __forceinline__ void vb_gather(VBlk &B, const float *__restrict__ w)
{
    const uint32_t f[4] = {B.f.x, B.f.y, B.f.z, B.f.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
        B.w[e] = f[e] != kSent ? ((c_ws_flags & 4) ? 1.f : __ldg(w + f[e])) : 0.f;
}

__device__ __forceinline__ void vb_assign(const VBlk &B, float *C, unsigned &zeros)
{
    const uint32_t f[4] = {B.f.x, B.f.y, B.f.z, B.f.w};
    const uint32_t cr[4] = {B.cr.x, B.cr.y, B.cr.z, B.cr.w};
    const float v[4] = {B.v.x, B.v.y, B.v.z, B.v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (f[e] != kSent) {
            const float s = __fmul_rn(B.w[e], v[e]);
            zeros += (s == 0.f) ? 1u : 0u;
            C[cr[e] & (kWsCells - 1)] = s;
        }
    }
}

// Rounds of the rank>=1 region: their loads are issued at the start of the
// tile build (hidden behind the rank-0 stream), gathered and applied after.
constexpr int kSlowRounds = 8;
struct SlowRounds {
    uint32_t cr[kSlowRounds], f[kSlowRounds];
    float v[kSlowRounds], w[kSlowRounds];
};

__device__ __forceinline__ void sr_load(SlowRounds &R, const WsArgs &A, uint32_t base,
                                        uint32_t p1, int lane)
{
#pragma unroll
    for (int r = 0; r < kSlowRounds; ++r) {
        const uint32_t k = base + 32u * r + (uint32_t)lane;
        const bool in = k < p1;
        R.cr[r] = in ? ld_s(A.cr + k) : 0u;
        R.f[r] = in ? ld_s(A.fiber + k) : kSent;
        R.v[r] = in ? ld_s(A.val + k) : 0.f;
    }
}

__device__ __forceinline__ void sr_gather(SlowRounds &R, const float *__restrict__ w)
{
#pragma unroll
    for (int r = 0; r < kSlowRounds; ++r) R.w[r] = R.f[r] != kSent ? __ldg(w + R.f[r]) : 0.f;
}

// apply rounds in order; a round whose 32 entries straddle two rank levels
// (flag bit 31, set at build time) is applied rank by rank
__device__ __forceinline__ void sr_apply(const SlowRounds &R, float *C, unsigned &zeros)
{
#pragma unroll
    for (int r = 0; r < kSlowRounds; ++r) {
        const bool ok = R.f[r] != kSent;
        if (!__any_sync(0xffffffffu, ok)) break;
        const float s = __fmul_rn(R.w[r], R.v[r]);
        zeros += (ok && s == 0.f) ? 1u : 0u;
        const uint32_t cr = R.cr[r];
        const uint32_t rank = (cr >> kWsCellBits) & 0xFFFFFu, cell = cr & (kWsCells - 1);
        if (!__any_sync(0xffffffffu, ok && (cr >> 31))) {
            if (ok) C[cell] += s;
        } else {
            const uint32_t rmin = __reduce_min_sync(0xffffffffu, ok ? rank : 0xFFFFFFFFu);
            const uint32_t rmax = __reduce_max_sync(0xffffffffu, ok ? rank : 0u);
            for (uint32_t rr = rmin; rr <= rmax; ++rr) {
                if (ok && rank == rr) C[cell] += s;
                __syncwarp();
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ unsigned build_tile(float *C, const WsArgs &A,
                                               const float *__restrict__ w, const Seg1 &S,
                                               int lane)
{
    SlowRounds R;
    sr_load(R, A, S.q0, S.p1, lane);  // in flight during the rank-0 stream
    float4 *Z = reinterpret_cast<float4 *>(C);
#pragma unroll 4
    for (int i = 0; i < kWsCells / 4 / 32; ++i) Z[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    unsigned zeros = 0;
    // rank-0 region in batches of kFastBlocks x 128 coefficients: all loads of
    // a batch in flight, then all w-gathers, then the stores (two latency
    // epochs per batch; at C2 a tile's rank-0 region is ~6 blocks)
    constexpr int kFastBlocks = 6;
    for (uint32_t b0 = S.p0; b0 < S.q0; b0 += 128u * kFastBlocks) {
        VBlk B[kFastBlocks];
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) vb_load(B[j], A, b0 + 128u * j, S.q0, lane);
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) vb_gather(B[j], w);
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) vb_assign(B[j], C, zeros);
    }
    __syncwarp();
    for (uint32_t base = S.q0; base < S.p1; base += 32u * kSlowRounds) {
        if (base != S.q0) sr_load(R, A, base, S.p1, lane);
        sr_gather(R, w);
        sr_apply(R, C, zeros);
    }
    return zeros;
}

// next (ct, c) step of this CTA, or ct >= n_ct when none
__device__ __forceinline__ void next_step(int &ct, int &c, int nch)
{
    if (++c == nch) {
        c = 0;
        ct += gridDim.x;
    }
}

// ---------------------------------------------------------------------------
// DSC
// ---------------------------------------------------------------------------
template <int DPL>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_dsc_ws(const WsArgs A, const float *__restrict__ w, float *__restrict__ y,
             const float *__restrict__ b, const uint32_t flags, const ReduceSlots red,
             const DscOut out, const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t full[2], empty[2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kWsCA * A.nt_pad;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    float *Dbuf = sm;
    float *Cbuf = sm + 2 * chunk_floats;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&full[s], kWsProd + 1);
            bar_init(&empty[s], kWsCons);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double sq = 0.0;
    float amax = 0.f;
    unsigned long long skipped = 0;

    if (warp < kWsCons) {
        // ===== consumers: register-tiled FFMA2 =====
        if constexpr (kSplitRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegCons));
        const int vg = lane >> 3, dg = lane & 7;
        const bool accumulate = flags & LIFE_ACCUMULATE;
        const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
        int k = 0;
        for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
            const int wt = ct * kWsCons + warp;
            const bool tile_ok = wt < A.n_tiles;
            // acc[vp][t] = (y[2vp][t], y[2vp+1][t]): pairs across voxels so
            // the coefficient pair is a native 64-bit operand and the
            // dictionary value a broadcast scalar (FFMA2 Rd, Rc.F32x2, Rd.F32)
            unsigned long long acc[4][DPL];
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
                for (int j = 0; j < DPL; ++j) acc[v][j] = 0ull;
            for (int c = 0; c < A.nch; ++c, ++k) {
                const int s = k & 1;
                bar_wait(&full[s], (k >> 1) & 1);
                if (tile_ok && c_ws_isolate != 1) {
                    const float *C = Cbuf + (s * kWsCons + warp) * kWsCells + vg * 8;
                    const float *D = Dbuf + s * chunk_floats + dg * DPL;
                    const int na_c = min(kWsCA, A.na - c * kWsCA);
#pragma unroll 32
                    for (int a = 0; a < kWsCA; ++a) {
                        const float4 c0 = *reinterpret_cast<const float4 *>(C + a * kWsTV);
                        const float4 c1 = *reinterpret_cast<const float4 *>(C + a * kWsTV + 4);
                        const unsigned long long cp[4] = {wpk(c0.x, c0.y), wpk(c0.z, c0.w),
                                                          wpk(c1.x, c1.y), wpk(c1.z, c1.w)};
                        const float4 *d4 = reinterpret_cast<const float4 *>(D + a * A.nt_pad);
#pragma unroll
                        for (int i = 0; i < DPL / 4; ++i) {
                            const float4 t = d4[i];
                            const float dv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const unsigned long long dd = wpk(dv[e], dv[e]);
#pragma unroll
                                for (int vp = 0; vp < 4; ++vp) wfma2(acc[vp][4 * i + e], cp[vp], dd);
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&empty[s]);
            }
            if (tile_ok) {
#pragma unroll
                for (int vp = 0; vp < 4; ++vp) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int voxel = wt * kWsTV + vg * 8 + 2 * vp + h;
                        if (voxel >= A.nv) continue;
                        const size_t yo = (size_t)voxel * A.nt;
#pragma unroll
                        for (int j = 0; j < DPL; ++j) {
                            float o[2];
                            wupk(acc[vp][j], o[0], o[1]);
                            const int t = dg * DPL + j;
                            if (t < A.nt) {
                                float r = o[h];
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
    } else {
        // ===== producers: TMA for D, coefficient tiles =====
        if constexpr (kSplitRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProd));
        const int p = warp - kWsCons;
        int k = 0;
        for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
            for (int c = 0; c < A.nch; ++c, ++k) {
                const int s = k & 1;
                {   // warm L2 with the next step's coefficient segments
                    int nct = ct, nc = c;
                    next_step(nct, nc, A.nch);
                    if (nct < n_ct && lane < kTPP)
                        prefetch_seg(A, seg_of(A, nct * kWsCons + p * kTPP + lane, nc));
                }
                if (k >= 2) bar_wait(&empty[s], ((k - 2) >> 1) & 1);
                if (p == 0 && lane == 0)
                    tma_chunk(Dbuf + s * chunk_floats, A.D + (size_t)c * chunk_floats,
                              chunk_bytes, &full[s]);
#pragma unroll 1
                for (int q = 0; q < kTPP; ++q) {
                    const int tw = kTPP * p + q;
                    if (c_ws_isolate != 2)
                        skipped += build_tile(Cbuf + (s * kWsCons + tw) * kWsCells, A, w,
                                              seg_of(A, ct * kWsCons + tw, c), lane);
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&full[s]);
            }
        }
    }

    // ---- fixed-order completion --------------------------------------------
    const int gw = blockIdx.x * kWsWarps + warp;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        skipped += __shfl_xor_sync(0xffffffffu, skipped, o);  // producers count per lane
    }
    if (lane == 0) {
        red.part_d[gw] = sq;
        red.part_u[gw] = skipped;
        red.part_f[gw] = amax;
    }
    if (ws_last_block(red.counter)) {
        const int W = gridDim.x * kWsWarps;
        const double tsq = ws_reduce<double>(red.part_d, W, 0.0, WAdd{});
        const unsigned long long tsk = ws_reduce<unsigned long long>(red.part_u, W, 0ull, WAdd{});
        const float tmax = ws_reduce<float>(red.part_f, W, 0.f, WMax{});
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
// WC
// ---------------------------------------------------------------------------
using WsFix = FixParams;

template <int DPL>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_wc_ws(const WsArgs A, const float *__restrict__ y, const WsFix fx, const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t dfull[2], dempty[2], zfull[2], zempty[2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kWsCA * A.nt_pad;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    float *Dbuf = sm;
    float *Zbuf = sm + 2 * chunk_floats;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    const int my_ct = (int)blockIdx.x < n_ct ? (n_ct - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_ct * A.nch;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&dfull[s], 1);
            bar_init(&dempty[s], kWsCons);
            bar_init(&zfull[s], kWsCons);
            bar_init(&zempty[s], kWsProd);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp < kWsCons) {
        // ===== consumers: Z = Y . D^T =====
        if constexpr (kSplitRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegCons));
        const int vg = lane >> 3, dg = lane & 7;
        const int b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1, b0 = lane & 1;
        int k = 0;
        for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
            const int wt = ct * kWsCons + warp;
            const bool tile_ok = wt < A.n_tiles;
            // yv[vp][t] = (y[2vp][t], y[2vp+1][t]) over this lane's DPL
            // directions: pairs across voxels, so each dictionary value is a
            // broadcast scalar operand and partial dots come out as voxel pairs
            unsigned long long yv[4][DPL];
#pragma unroll
            for (int vp = 0; vp < 4; ++vp) {
                float e[2][DPL];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int voxel = wt * kWsTV + vg * 8 + 2 * vp + h;
                    const bool ok = tile_ok && voxel < A.nv;
                    const size_t yo = (size_t)(ok ? voxel : 0) * A.nt;
#pragma unroll
                    for (int j = 0; j < DPL; ++j) {
                        const int t = dg * DPL + j;
                        e[h][j] = (ok && t < A.nt) ? y[yo + t] : 0.f;
                    }
                }
#pragma unroll
                for (int j = 0; j < DPL; ++j) yv[vp][j] = wpk(e[0][j], e[1][j]);
            }
            for (int c = 0; c < A.nch; ++c, ++k) {
                const int s = k & 1;
                bar_wait(&dfull[s], (k >> 1) & 1);
                if (k >= 2) bar_wait(&zempty[s], ((k - 2) >> 1) & 1);
                if (tile_ok) {
                    float *Z = Zbuf + (s * kWsCons + warp) * kWsCells;
                    const float *D = Dbuf + s * chunk_floats + dg * DPL;
                    const int na_c = min(kWsCA, A.na - c * kWsCA);
#pragma unroll 1
                    for (int a0 = 0; a0 < na_c; a0 += 2) {
                        unsigned long long pp[2][4];
#pragma unroll
                        for (int aa = 0; aa < 2; ++aa) {
                            const float4 *d4 = reinterpret_cast<const float4 *>(D + (a0 + aa) * A.nt_pad);
#pragma unroll
                            for (int vp = 0; vp < 4; ++vp) pp[aa][vp] = 0ull;
#pragma unroll
                            for (int i = 0; i < DPL / 4; ++i) {
                                const float4 t = d4[i];
                                const float dv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const unsigned long long dd = wpk(dv[e], dv[e]);
#pragma unroll
                                    for (int vp = 0; vp < 4; ++vp) wfma2(pp[aa][vp], yv[vp][4 * i + e], dd);
                                }
                            }
                        }
                        float q[16];
#pragma unroll
                        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
                            for (int vp = 0; vp < 4; ++vp)
                                wupk(pp[aa][vp], q[aa * 8 + 2 * vp], q[aa * 8 + 2 * vp + 1]);
                        // butterfly over the 8 direction lanes of this voxel group
#pragma unroll
                        for (int m = 4, h = 8; m >= 1; m >>= 1, h >>= 1) {
                            const bool up = (lane & m) != 0;
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                if (i < h) {
                                    const float send = up ? q[i] : q[i + h];
                                    const float keep = up ? q[i + h] : q[i];
                                    q[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                                }
                            }
                        }
                        *reinterpret_cast<float2 *>(Z + (a0 + b2) * kWsTV + vg * 8 + 4 * b1 + 2 * b0) =
                            make_float2(q[0], q[1]);
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    bar_arrive(&dempty[s]);
                    bar_arrive(&zfull[s]);
                }
            }
        }
    } else {
        // ===== producers: D chunks via TMA; scatter value * Z[cell] =====
        if constexpr (kSplitRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProd));
        const int p = warp - kWsCons;
        const int ex = fix_exponent(fx, A.nt);
        const double scale = ldexp(1.0, ex);
        // z * 2^ex is exact in fp32 (power-of-two scale) when the exponent
        // stays in range, so the fixed-point term needs no fp64 arithmetic
        const bool f32_scale = ex >= -120 && ex <= 120;
        const float scalef = f32_scale ? ldexpf(1.f, ex) : 1.f;
        if (p == 0 && lane == 0 && total > 0)
            tma_chunk(Dbuf, A.D, chunk_bytes, &dfull[0]);
        int k = 0;
        for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
            for (int c = 0; c < A.nch; ++c, ++k) {
                const int s = k & 1;
                if (p == 0 && lane == 0 && k + 1 < total) {
                    const int s1 = (k + 1) & 1;
                    if (k + 1 >= 2) bar_wait(&dempty[s1], ((k - 1) >> 1) & 1);
                    const int c1 = (c + 1) % A.nch;
                    tma_chunk(Dbuf + s1 * chunk_floats, A.D + (size_t)c1 * chunk_floats,
                              chunk_bytes, &dfull[s1]);
                }
                __syncwarp();
                {
                    int nct = ct, nc = c;
                    next_step(nct, nc, A.nch);
                    if (nct < n_ct && lane < kTPP)
                        prefetch_seg(A, seg_of(A, nct * kWsCons + p * kTPP + lane, nc));
                }
                const Seg1 S0 = seg_of(A, ct * kWsCons + kTPP * p, c);
                VBlk B0, B1;
                vb_load(B0, A, S0.p0, S0.p1, lane);
                bar_wait(&zfull[s], (k >> 1) & 1);
#pragma unroll 1
                for (int q = 0; q < kTPP; ++q) {
                    const Seg1 S = q ? seg_of(A, ct * kWsCons + kTPP * p + q, c) : S0;
                    const float *Z = Zbuf + (s * kWsCons + kTPP * p + q) * kWsCells;
                    if (q) vb_load(B0, A, S.p0, S.p1, lane);
                    for (uint32_t base = S.p0; base < S.p1; base += 128u) {
                        vb_load(B1, A, base + 128u, S.p1, lane);
                        const uint32_t f[4] = {B0.f.x, B0.f.y, B0.f.z, B0.f.w};
                        const uint32_t cr[4] = {B0.cr.x, B0.cr.y, B0.cr.z, B0.cr.w};
                        const float v[4] = {B0.v.x, B0.v.y, B0.v.z, B0.v.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if (f[e] != kSent) {
                                const float z = Z[cr[e] & (kWsCells - 1)] * v[e];
                                const long long qv = f32_scale ? __float2ll_rn(z * scalef)
                                                               : __double2ll_rn((double)z * scale);
                                atomicAdd(fx.wfix + f[e], static_cast<unsigned long long>(qv));
                            }
                        }
                        B0 = B1;
                    }
                }
                __syncwarp();
                if (lane == 0) bar_arrive(&zempty[s]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <int DPL>
static int ws_dsc_t(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                    const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_dsc_ws<DPL>, phi->d_smem));
    WsArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_t1, phi->d_D,
             phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
    k_dsc_ws<DPL><<<phi->d_blocks, kWsThreads, phi->d_smem, st>>>(A, w, y, b, flags, phi->red,
                                                                   o, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int DPL>
static int ws_wc_t(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                   cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_wc_ws<DPL>, phi->d_smem));
    WsArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_t1, phi->d_D,
             phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
    k_wc_ws<DPL><<<phi->d_blocks, kWsThreads, phi->d_smem, st>>>(A, y, fx, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int DPL>
static int ws_prepare_t(life_phi *phi)
{
    LIFE_TRY(ensure_smem(k_dsc_ws<DPL>, phi->d_smem));
    LIFE_TRY(ensure_smem(k_wc_ws<DPL>, phi->d_smem));
    return LIFE_OK;
}

#define LIFE_WS_DISPATCH(FN, ...)                                              \
    switch (phi->nt_pad / 8) {                                                 \
    case 4: return FN<4>(__VA_ARGS__);                                         \
    case 8: return FN<8>(__VA_ARGS__);                                         \
    case 12: return FN<12>(__VA_ARGS__);                                       \
    default: return fail(LIFE_ERR_CONFIG_INVALID, "ws layout: unsupported n_dirs"); \
    }

int launch_dsc_ws(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                  const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_WS_DISPATCH(ws_dsc_t, phi, w, y, b, flags, o, h, st);
}

int launch_wc_ws(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                 cudaStream_t st)
{
    LIFE_WS_DISPATCH(ws_wc_t, phi, fx, y, h, st);
}

int prepare_ws(life_phi *phi) { LIFE_WS_DISPATCH(ws_prepare_t, phi); }

}  // namespace life

#ifdef LIFE_WS_DIAG
extern "C" LIFE_API int life_debug_ws_isolate(int mode)
{
    const int iso = mode & 0xFF, fl = mode >> 8;
    if (cudaMemcpyToSymbol(life::c_ws_isolate, &iso, sizeof(int)) != cudaSuccess) return 20;
    return cudaMemcpyToSymbol(life::c_ws_flags, &fl, sizeof(int)) == cudaSuccess ? 0 : 20;
}
#endif

namespace life {

int ws_warps() { return kWsWarps; }

size_t ws_smem_bytes(int nt_pad)
{
    return ((size_t)2 * kWsCA * nt_pad + (size_t)2 * kWsCons * kWsCells) * sizeof(float);
}

}  // namespace life
