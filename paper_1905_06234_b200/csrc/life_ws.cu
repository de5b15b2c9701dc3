// life_ws.cu -- warp-specialized dense DSC / WC (the C2 hot path).
//
// Same contraction as life_dense.cu (Y_tile += C_tile . D_chunk for DSC,
// Z_tile = Y_tile . D_chunk^T then value*Z[cell] -> fascicles for WC), split
// between two roles inside one persistent CTA per SM:
//
//   4 producer warps  build the 32 x 32 coefficient tiles C of the next
//                     (voxel tile, atom chunk) step in shared memory from the
//                     sorted coefficient stream and the gathered w[f] (DSC),
//                     or scatter value * Z[cell] into the fixed-point fascicle
//                     sums with RED.ADD (WC).  Producer warp 0 also issues
//                     the TMA bulk copy of the next dictionary chunk.
//   8 consumer warps  do only register-tiled FFMA2 work: each lane owns
//                     8 voxels x 12 directions (96 fp32 accumulators), so a
//                     dictionary value feeds 8 FMAs and a coefficient 12.
//
// Coefficient staging (the "staged" producer): the layout orders segments by
// (CTA tile round, atom chunk, warp tile, rank, cell), so the two tiles a
// producer warp owns in one step are ONE contiguous range of the stream.
// Lane 0 of each producer warp copies the next step's range into its own
// double-buffered shared-memory slot with three cp.async.bulk copies
// (index / fascicle / value arrays, mbarrier complete_tx) and prefetches the
// step after that into L2, so the producers see shared-memory latency for
// the stream and only the w[f] gathers (DSC) or RED.ADDs (WC) go to L2.
// Operators whose per-warp step range exceeds a slot fall back to the
// register-streaming producer (same results, bit for bit).
//
// Steps are double buffered (C/Z tiles and dictionary chunks) and handed over
// with mbarriers (full/empty).  Each LDS.128 costs four shared-memory
// wavefronts on sm_100 (measured, tools/ubench); the 8x12 lane tile needs 5 of
// them per 96 FMAs per lane, keeping shared memory below the FP32 pipe.
#include <algorithm>

#include "life_common.cuh"

namespace life {

constexpr int kWsCons = 8;
constexpr int kWsProd = 4;
constexpr int kTPP = kWsCons / kWsProd;   // consumer tiles per producer warp
constexpr int kWsWarps = kWsCons + kWsProd;
constexpr int kWsThreads = kWsWarps * 32;
constexpr int kWsTV = 32;                  // voxels per consumer tile
constexpr int kWsCA = 32;                  // atoms per chunk
constexpr int kWsCells = kWsTV * kWsCA;    // 1024
constexpr int kWsCellBits = 10;
constexpr int kWsRing = 2880;              // staged entries per producer warp (ring)
// load and gather the first rank>=1 batch together with the first rank-0 batch
#ifndef LIFE_WS_EARLY_SLOW
#define LIFE_WS_EARLY_SLOW 0
#endif
constexpr bool kEarlySlow = LIFE_WS_EARLY_SLOW;
static_assert(kTPP == 2, "a producer warp owns two adjacent tiles");

struct WsArgs {
    const uint32_t *cr;
    const uint32_t *fiber;
    const float *val;
    const uint32_t *tptr;   // padded segment starts, [n_ct*nch*8 + 1]
    const uint32_t *t1;     // start of each segment's rank>=1 region
    const float *D;
    const int *slotv;       // voxel of each tile slot (tile*32 + i), -1 for padding
    int nv, nt, nt_pad, nch, n_tiles, na;
};
constexpr uint32_t kSent = 0xFFFFFFFFu;  // padding entry (fiber field)
// Diagnostic isolation, compiled in only with -DLIFE_WS_DIAG (tools/ws_isolate.py):
// c_ws_isolate 1 = producers only, 2 = consumers only (results are garbage);
// c_ws_flags 1 = no L2 prefetch, 4 = no gather.
#ifdef LIFE_WS_DIAG
__constant__ int c_ws_isolate = 0;
__constant__ int c_ws_flags = 0;
#else
constexpr int c_ws_isolate = 0;
constexpr int c_ws_flags = 0;
#endif

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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smaddr(dst)),
        "l"(src), "r"(bytes), "r"(smaddr(b))
        : "memory");
}
__device__ __forceinline__ void tma_chunk(float *dst, const float *src, unsigned bytes, uint64_t *b)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bar_arrive_tx(b, bytes);
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
    for (unsigned off = 0; off < bytes; off += 32768u)
        bulk_g2s(d + off, s + off, min(32768u, bytes - off), b);
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

__device__ __forceinline__ void prefetch_l2(const void *ptr, uint32_t bytes)
{
    if (bytes == 0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// ---- a producer warp's step: its two tiles (2p, 2p+1) of one (ct, chunk) --
// Segment of one (tile, chunk): [p0, q0) holds each cell's first coefficient
// (rank 0, distinct cells) and [q0, p1) the repeats (rank >= 1); both regions
// are padded to 4-entry multiples (fiber = kSent), so the rank-0 region
// streams as 16-byte vectors, 4 coefficients per lane, with one plain STS per
// coefficient.  Repeats are added afterwards in rank order (32-entry windows
// straddling two ranks, flagged at build time, are applied rank by rank).
struct Seg2 {
    uint32_t a, q0, b, q1, e;  // tile 0 [a, q0) [q0, b); tile 1 [b, q1) [q1, e)
};

__device__ __forceinline__ size_t tc_of(const WsArgs &A, int ct, int c, int q)
{
    return ((size_t)ct * A.nch + c) * kWsCons + q;
}

__device__ __forceinline__ Seg2 seg2_of(const WsArgs &A, int ct, int c, int p)
{
    const size_t tc = tc_of(A, ct, c, kTPP * p);
    Seg2 S;
    S.a = __ldg(A.tptr + tc);
    S.q0 = __ldg(A.t1 + tc);
    S.b = __ldg(A.tptr + tc + 1);
    S.q1 = __ldg(A.t1 + tc + 1);
    S.e = __ldg(A.tptr + tc + 2);
    return S;
}

// the CTA's j-th step: (ct, c)
__device__ __forceinline__ void step_of(int j, int nch, int &ct, int &c)
{
    ct = (int)blockIdx.x + (j / nch) * (int)gridDim.x;
    c = j % nch;
}

__device__ __forceinline__ void prefetch_range(const WsArgs &A, const Seg2 &S, int lane)
{
    if ((c_ws_flags & 1) || S.e <= S.a || lane >= 3) return;
    const uint32_t bytes = (S.e - S.a) * 4u;  // padded ranges are 16-byte aligned
    const void *base = lane == 0 ? (const void *)(A.cr + S.a)
                     : lane == 1 ? (const void *)(A.fiber + S.a)
                                 : (const void *)(A.val + S.a);
    prefetch_l2(base, bytes);
}

// staging ring of one producer warp: three arrays of kWsRing entries; a step's
// range occupies [off, off + n) modulo kWsRing (offsets and sizes are
// multiples of 4, so a 16-byte vector never wraps).  The host checks that two
// consecutive steps of a warp always fit (life_dense.cu: build_dense).
struct Slot {
    uint32_t *cr;
    uint32_t *f;
    float *v;
    uint32_t off;
    __device__ __forceinline__ uint32_t at(uint32_t i) const
    {
        const uint32_t x = off + i;
        return x >= (uint32_t)kWsRing ? x - (uint32_t)kWsRing : x;
    }
};

__device__ __forceinline__ uint32_t ring_wrap(uint32_t x)
{
    return x >= (uint32_t)kWsRing ? x - (uint32_t)kWsRing : x;
}

__device__ __forceinline__ Slot slot_at(float *slots, int p, uint32_t off)
{
    uint32_t *base = reinterpret_cast<uint32_t *>(slots) + (size_t)p * 3 * kWsRing;
    return Slot{base, base + kWsRing, reinterpret_cast<float *>(base + 2 * kWsRing), off};
}

// lane 0: copy the step's range [S.a, S.e) into the ring at D.off
// (three arrays, split in two where the range wraps)
__device__ __forceinline__ void stage_issue(const WsArgs &A, const Seg2 &S, const Slot &D,
                                            uint64_t *bar)
{
    const unsigned n = S.e - S.a;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bar_arrive_tx(bar, 12u * n);
    if (n == 0) return;
    const unsigned n1 = min(n, (unsigned)kWsRing - D.off), n2 = n - n1;
    bulk_g2s(D.cr + D.off, A.cr + S.a, 4u * n1, bar);
    bulk_g2s(D.f + D.off, A.fiber + S.a, 4u * n1, bar);
    bulk_g2s(D.v + D.off, A.val + S.a, 4u * n1, bar);
    if (n2) {
        bulk_g2s(D.cr, A.cr + S.a + n1, 4u * n2, bar);
        bulk_g2s(D.f, A.fiber + S.a + n1, 4u * n2, bar);
        bulk_g2s(D.v, A.val + S.a + n1, 4u * n2, bar);
    }
}

// 4 consecutive coefficients per lane (a 128-coefficient block per warp)
struct VBlk {
    uint4 cr, f;
    float4 v;
    float w[4];
};

__device__ __forceinline__ void vb_empty(VBlk &B)
{
    B.cr = make_uint4(0u, 0u, 0u, 0u);
    B.f = make_uint4(kSent, kSent, kSent, kSent);
    B.v = make_float4(0.f, 0.f, 0.f, 0.f);
}

// staged: from the slot (k relative to the slot start)
__device__ __forceinline__ void vb_lds(VBlk &B, const Slot &S, uint32_t k, bool ok)
{
    if (ok) {
        const uint32_t x = S.at(k);
        B.cr = *reinterpret_cast<const uint4 *>(S.cr + x);
        B.f = *reinterpret_cast<const uint4 *>(S.f + x);
        B.v = *reinterpret_cast<const float4 *>(S.v + x);
    } else {
        vb_empty(B);
    }
}

// streamed: straight from global memory (fallback producer)
__device__ __forceinline__ void vb_ldg(VBlk &B, const WsArgs &A, uint32_t k, bool ok)
{
    if (ok) {
        B.cr = ld_stream(reinterpret_cast<const uint4 *>(A.cr + k));
        B.f = ld_stream(reinterpret_cast<const uint4 *>(A.fiber + k));
        B.v = ld_stream(reinterpret_cast<const float4 *>(A.val + k));
    } else {
        vb_empty(B);
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

// one 32-entry window of a rank>=1 region per round
constexpr int kSlowRounds = 8;
struct SlowRounds {
    uint32_t cr[kSlowRounds], f[kSlowRounds];
    float v[kSlowRounds], w[kSlowRounds];
    bool t1[kSlowRounds];  // window belongs to tile 1
};

__device__ __forceinline__ void sr_gather(SlowRounds &R, const float *__restrict__ w)
{
#pragma unroll
    for (int r = 0; r < kSlowRounds; ++r)
        R.w[r] = R.f[r] != kSent ? ((c_ws_flags & 4) ? 1.f : __ldg(w + R.f[r])) : 0.f;
}

// apply rounds in order; a round whose 32 entries straddle two rank levels
// (flag bit 31, set at build time) is applied rank by rank
__device__ __forceinline__ void sr_apply(const SlowRounds &R, float *C0, float *C1, unsigned &zeros)
{
#pragma unroll
    for (int r = 0; r < kSlowRounds; ++r) {
        const bool ok = R.f[r] != kSent;
        if (!__any_sync(0xffffffffu, ok)) continue;
        float *C = R.t1[r] ? C1 : C0;
        const float s = __fmul_rn(R.w[r], R.v[r]);
        zeros += (ok && s == 0.f) ? 1u : 0u;
        const uint32_t cr = R.cr[r];
        const uint32_t rank = (cr >> kWsCellBits) & 0x1FFFFFu, cell = cr & (kWsCells - 1);
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

// Build the producer warp's two coefficient tiles of one step.  STAGED reads
// the range from the warp's shared-memory slot (entry k at slot[k - S.a]),
// otherwise straight from global memory.
template <bool STAGED>
__device__ __forceinline__ unsigned build_pair(float *C0, float *C1, const WsArgs &A,
                                               const float *__restrict__ w, const Seg2 &S,
                                               const Slot &sl, int lane)
{
    float4 *Z0 = reinterpret_cast<float4 *>(C0);
    float4 *Z1 = reinterpret_cast<float4 *>(C1);
#pragma unroll
    for (int i = 0; i < kWsCells / 4 / 32; ++i) {
        Z0[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
        Z1[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    unsigned zeros = 0;
    // rank-0 regions of both tiles in batches of kFastBlocks x 128 entries
    // (all loads of a batch, then all w gathers, then the stores); the first
    // batch of rank>=1 windows is loaded and gathered together with the first
    // rank-0 batch, so a typical step has one gather round trip
    constexpr int kFastBlocks = 6;
    const int n0 = (int)((S.q0 - S.a + 127u) / 128u), n1 = (int)((S.q1 - S.b + 127u) / 128u);
    const int m0 = (int)((S.b - S.q0 + 31u) / 32u), m1 = (int)((S.e - S.q1 + 31u) / 32u);
    SlowRounds R;
    auto load_slow = [&](int r0) {
#pragma unroll
        for (int r = 0; r < kSlowRounds; ++r) {
            const int g = r0 + r;
            R.t1[r] = g >= m0;
            const uint32_t base = R.t1[r] ? S.q1 + 32u * (uint32_t)(g - m0) : S.q0 + 32u * (uint32_t)g;
            const uint32_t end = R.t1[r] ? S.e : S.b;
            const uint32_t k = base + (uint32_t)lane;
            const bool in = g < m0 + m1 && k < end;
            if (STAGED) {
                const uint32_t x = sl.at(k - S.a);
                R.cr[r] = in ? sl.cr[x] : 0u;
                R.f[r] = in ? sl.f[x] : kSent;
                R.v[r] = in ? sl.v[x] : 0.f;
            } else {
                R.cr[r] = in ? ld_stream(A.cr + k) : 0u;
                R.f[r] = in ? ld_stream(A.fiber + k) : kSent;
                R.v[r] = in ? ld_stream(A.val + k) : 0.f;
            }
        }
    };
    if (kEarlySlow) load_slow(0);
    for (int g0 = 0; g0 < n0 + n1; g0 += kFastBlocks) {
        VBlk B[kFastBlocks];
        bool second[kFastBlocks];
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) {
            const int g = g0 + j;
            second[j] = g >= n0;
            const uint32_t base = second[j] ? S.b + 128u * (uint32_t)(g - n0) : S.a + 128u * (uint32_t)g;
            const uint32_t end = second[j] ? S.q1 : S.q0;
            const uint32_t k = base + 4u * (uint32_t)lane;
            const bool ok = g < n0 + n1 && k < end;
            if (STAGED) vb_lds(B[j], sl, k - S.a, ok);
            else vb_ldg(B[j], A, k, ok);
        }
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) vb_gather(B[j], w);
        if (kEarlySlow && g0 == 0) sr_gather(R, w);
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) vb_assign(B[j], second[j] ? C1 : C0, zeros);
    }
    __syncwarp();
    // rank>=1 windows, in order, after every rank-0 store
    for (int r0 = 0; r0 < m0 + m1; r0 += kSlowRounds) {
        if (r0 || !kEarlySlow || n0 + n1 == 0) {
            load_slow(r0);
            sr_gather(R, w);
        }
        sr_apply(R, C0, C1, zeros);
    }
    return zeros;
}

// ---------------------------------------------------------------------------
// DSC
// ---------------------------------------------------------------------------
template <int DPL, bool STAGED>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_dsc_ws(const WsArgs A, const float *__restrict__ w, float *__restrict__ y,
             const float *__restrict__ b, const uint32_t flags, const ReduceSlots red,
             const DscOut out, const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t full[2], empty[2], slotbar[kWsProd][2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kWsCA * A.nt_pad;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    float *Dbuf = sm;
    float *Cbuf = sm + 2 * chunk_floats;
    float *slots = Cbuf + 2 * kWsCons * kWsCells;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    const int my_ct = (int)blockIdx.x < n_ct ? (n_ct - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_ct * A.nch;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&full[s], kWsProd + 1);
            bar_init(&empty[s], kWsCons);
            for (int p = 0; p < kWsProd; ++p) bar_init(&slotbar[p][s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double sq = 0.0;
    float amax = 0.f;
    unsigned long long skipped = 0;

    if (warp < kWsCons) {
        // ===== consumers: register-tiled FFMA2 =====
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
#pragma unroll
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
                        const int voxel = __ldg(A.slotv + wt * kWsTV + vg * 8 + 2 * vp + h);
                        if (voxel < 0) continue;
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
        // ===== producers: TMA for D and the coefficient ranges, tile build =====
        const int p = warp - kWsCons;
        Seg2 cur{}, nxt{};
        uint32_t off_cur = 0u, off_nxt = 0u;
        if (total > 0) {
            int ct, c;
            step_of(0, A.nch, ct, c);
            cur = seg2_of(A, ct, c, p);
            if (STAGED && lane == 0) stage_issue(A, cur, slot_at(slots, p, 0u), &slotbar[p][0]);
            off_nxt = ring_wrap(cur.e - cur.a);
        }
        if (total > 1) {
            int ct, c;
            step_of(1, A.nch, ct, c);
            nxt = seg2_of(A, ct, c, p);
            prefetch_range(A, nxt, lane);
        }
        for (int k = 0; k < total; ++k) {
            const int s = k & 1;
            int ct, c;
            step_of(k, A.nch, ct, c);
            Seg2 nn{};
            if (k + 2 < total) {
                int ct2, c2;
                step_of(k + 2, A.nch, ct2, c2);
                nn = seg2_of(A, ct2, c2, p);
            }
            // slot s^1 was last read in step k-1, which this warp finished
            if (STAGED && k + 1 < total && lane == 0)
                stage_issue(A, nxt, slot_at(slots, p, off_nxt), &slotbar[p][s ^ 1]);
            if (k >= 2) bar_wait(&empty[s], ((k - 2) >> 1) & 1);
            if (p == 0 && lane == 0)
                tma_chunk(Dbuf + s * chunk_floats, A.D + (size_t)c * chunk_floats, chunk_bytes,
                          &full[s]);
            if (k + 2 < total) prefetch_range(A, nn, lane);
            if (STAGED) bar_wait(&slotbar[p][s], (k >> 1) & 1);
            if (c_ws_isolate != 2)
                skipped += build_pair<STAGED>(Cbuf + (s * kWsCons + kTPP * p) * kWsCells,
                                              Cbuf + (s * kWsCons + kTPP * p + 1) * kWsCells, A,
                                              w, cur, slot_at(slots, p, off_cur), lane);
            __syncwarp();
            if (lane == 0) bar_arrive(&full[s]);
            off_cur = off_nxt;
            off_nxt = ring_wrap(off_nxt + (nxt.e - nxt.a));
            cur = nxt;
            nxt = nn;
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

// value * Z[cell] of 4 consecutive entries -> fixed-point fascicle sums
__device__ __forceinline__ void wc_scatter4(const VBlk &B, const float *Z, const WsFix &fx,
                                            bool f32_scale, float scalef, double scale)
{
    const uint32_t f[4] = {B.f.x, B.f.y, B.f.z, B.f.w};
    const uint32_t cr[4] = {B.cr.x, B.cr.y, B.cr.z, B.cr.w};
    const float v[4] = {B.v.x, B.v.y, B.v.z, B.v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (f[e] != kSent) {
            const float z = Z[cr[e] & (kWsCells - 1)] * v[e];
            const long long qv = f32_scale ? __float2ll_rn(z * scalef)
                                           : __double2ll_rn((double)z * scale);
            atomicAdd(fx.wfix + f[e], static_cast<unsigned long long>(qv));
        }
    }
}

template <int DPL, bool STAGED>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_wc_ws(const WsArgs A, const float *__restrict__ y, const WsFix fx, const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t dfull[2], dempty[2], zfull[2], zempty[2], slotbar[kWsProd][2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kWsCA * A.nt_pad;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    float *Dbuf = sm;
    float *Zbuf = sm + 2 * chunk_floats;
    float *slots = Zbuf + 2 * kWsCons * kWsCells;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    const int my_ct = (int)blockIdx.x < n_ct ? (n_ct - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_ct * A.nch;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&dfull[s], 1);
            bar_init(&dempty[s], kWsCons);
            bar_init(&zfull[s], kWsCons);
            bar_init(&zempty[s], kWsProd);
            for (int p = 0; p < kWsProd; ++p) bar_init(&slotbar[p][s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp < kWsCons) {
        // ===== consumers: Z = Y . D^T =====
        // Lane (vg, dg) holds 12 directions of 8 voxels; partial dots are
        // summed over the 8 direction lanes of a voxel group by a butterfly.
        // Slot u of the lane's 8 voxels holds voxel vg*8 + (u ^ dg), so every
        // butterfly stage keeps the low half of its values and sends the high
        // half (no lane-dependent selects), and slot 0 ends up holding
        // voxel vg*8 + dg, summed over all 96 directions.
        const int vg = lane >> 3, dg = lane & 7;
        int k = 0;
        for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
            const int wt = ct * kWsCons + warp;
            const bool tile_ok = wt < A.n_tiles;
            unsigned long long yv[4][DPL];  // (slot 2vp, slot 2vp+1) per direction
#pragma unroll
            for (int vp = 0; vp < 4; ++vp) {
                float e[2][DPL];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int voxel = tile_ok ? __ldg(A.slotv + wt * kWsTV + vg * 8 + ((2 * vp + h) ^ dg)) : -1;
                    const bool ok = voxel >= 0;
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
                if (tile_ok && c_ws_isolate != 1) {
                    float *Z = Zbuf + (s * kWsCons + warp) * kWsCells + vg * 8 + dg;
                    const float *D = Dbuf + s * chunk_floats + dg * DPL;
#pragma unroll 2
                    for (int a0 = 0; a0 < kWsCA; a0 += 2) {
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
#pragma unroll
                        for (int aa = 0; aa < 2; ++aa) {
                            float q[8];
#pragma unroll
                            for (int vp = 0; vp < 4; ++vp) wupk(pp[aa][vp], q[2 * vp], q[2 * vp + 1]);
#pragma unroll
                            for (int m = 4; m >= 1; m >>= 1)
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    if (i < m) q[i] += __shfl_xor_sync(0xffffffffu, q[i + m], m);
                            Z[(a0 + aa) * kWsTV] = q[0];
                        }
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
        const int p = warp - kWsCons;
        const int ex = fix_exponent(fx, A.nt);
        const double scale = ldexp(1.0, ex);
        // z * 2^ex is exact in fp32 (power-of-two scale) when the exponent
        // stays in range, so the fixed-point term needs no fp64 arithmetic
        const bool f32_scale = ex >= -120 && ex <= 120;
        const float scalef = f32_scale ? ldexpf(1.f, ex) : 1.f;
        if (p == 0 && lane == 0 && total > 0) tma_chunk(Dbuf, A.D, chunk_bytes, &dfull[0]);
        Seg2 cur{}, nxt{};
        uint32_t off_cur = 0u, off_nxt = 0u;
        if (total > 0) {
            int ct, c;
            step_of(0, A.nch, ct, c);
            cur = seg2_of(A, ct, c, p);
            if (STAGED && lane == 0) stage_issue(A, cur, slot_at(slots, p, 0u), &slotbar[p][0]);
            off_nxt = ring_wrap(cur.e - cur.a);
        }
        if (total > 1) {
            int ct, c;
            step_of(1, A.nch, ct, c);
            nxt = seg2_of(A, ct, c, p);
            prefetch_range(A, nxt, lane);
        }
        for (int k = 0; k < total; ++k) {
            const int s = k & 1;
            int ct, c;
            step_of(k, A.nch, ct, c);
            if (p == 0 && lane == 0 && k + 1 < total) {
                const int s1 = (k + 1) & 1;
                if (k + 1 >= 2) bar_wait(&dempty[s1], ((k - 1) >> 1) & 1);
                const int c1 = (c + 1) % A.nch;
                tma_chunk(Dbuf + s1 * chunk_floats, A.D + (size_t)c1 * chunk_floats, chunk_bytes,
                          &dfull[s1]);
            }
            __syncwarp();
            Seg2 nn{};
            if (k + 2 < total) {
                int ct2, c2;
                step_of(k + 2, A.nch, ct2, c2);
                nn = seg2_of(A, ct2, c2, p);
            }
            if (STAGED && k + 1 < total && lane == 0)
                stage_issue(A, nxt, slot_at(slots, p, off_nxt), &slotbar[p][s ^ 1]);
            if (k + 2 < total) prefetch_range(A, nn, lane);
            const Slot sl = slot_at(slots, p, off_cur);
            if (STAGED) bar_wait(&slotbar[p][s], (k >> 1) & 1);
            bar_wait(&zfull[s], (k >> 1) & 1);
            const float *Z0 = Zbuf + (s * kWsCons + kTPP * p) * kWsCells;
            // the pair's range [a, e) in 128-entry blocks; tile 1 starts at b
            // (a 4-aligned boundary, so no 4-entry group straddles it)
            constexpr int kB = 4;
            for (uint32_t base = cur.a; base < (c_ws_isolate == 2 ? cur.a : cur.e); base += 128u * kB) {
                VBlk B[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint32_t kk = base + 128u * j + 4u * (uint32_t)lane;
                    if (STAGED) vb_lds(B[j], sl, kk - cur.a, kk < cur.e);
                    else vb_ldg(B[j], A, kk, kk < cur.e);
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint32_t kk = base + 128u * j + 4u * (uint32_t)lane;
                    wc_scatter4(B[j], kk < cur.b ? Z0 : Z0 + kWsCells, fx, f32_scale, scalef, scale);
                }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&zempty[s]);
            off_cur = off_nxt;
            off_nxt = ring_wrap(off_nxt + (nxt.e - nxt.a));
            cur = nxt;
            nxt = nn;
        }
    }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <int DPL, bool STAGED>
static int ws_dsc_t(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                    const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_dsc_ws<DPL, STAGED>, phi->d_smem));
    WsArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_t1, phi->d_D,
             phi->d_slotv, phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
    k_dsc_ws<DPL, STAGED><<<phi->d_blocks, kWsThreads, phi->d_smem, st>>>(A, w, y, b, flags,
                                                                           phi->red, o, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int DPL, bool STAGED>
static int ws_wc_t(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                   cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_wc_ws<DPL, STAGED>, phi->d_smem));
    WsArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_t1, phi->d_D,
             phi->d_slotv, phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
    k_wc_ws<DPL, STAGED><<<phi->d_blocks, kWsThreads, phi->d_smem, st>>>(A, y, fx, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int DPL, bool STAGED>
static int ws_prepare_t(life_phi *phi)
{
    LIFE_TRY(ensure_smem(k_dsc_ws<DPL, STAGED>, phi->d_smem));
    LIFE_TRY(ensure_smem(k_wc_ws<DPL, STAGED>, phi->d_smem));
    return LIFE_OK;
}

#define LIFE_WS_DISPATCH(FN, ...)                                              \
    do {                                                                       \
        const bool staged_ = phi->d_staged;                                    \
        switch (phi->nt_pad / 8) {                                             \
        case 4: return staged_ ? FN<4, true>(__VA_ARGS__) : FN<4, false>(__VA_ARGS__);    \
        case 8: return staged_ ? FN<8, true>(__VA_ARGS__) : FN<8, false>(__VA_ARGS__);    \
        case 12: return staged_ ? FN<12, true>(__VA_ARGS__) : FN<12, false>(__VA_ARGS__); \
        default: return fail(LIFE_ERR_CONFIG_INVALID, "ws layout: unsupported n_dirs"); \
        }                                                                      \
    } while (0)

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
int ws_chunk_atoms() { return kWsCA; }
int ws_ring_entries() { return kWsRing; }

size_t ws_smem_bytes(int nt_pad, bool staged)
{
    size_t b = ((size_t)2 * kWsCA * nt_pad + (size_t)2 * kWsCons * kWsCells) * sizeof(float);
    if (staged) b += (size_t)kWsProd * 3 * kWsRing * 4;
    return b;
}

}  // namespace life
