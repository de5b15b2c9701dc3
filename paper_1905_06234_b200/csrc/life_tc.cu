// life_tc.cu -- DSC on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// The product per CTA tile of 128 voxels is a dense contraction over atom
// chunks of 32:  Y(128 x N) += C(128 x 32) . D_c(32 x N), N = directions
// padded to 32, with C[v, a] = sum_k w[f_k] value_k built on the fly in
// shared memory from the sorted coefficient stream (life_dense.cu
// build_tc).  Roles inside one persistent CTA per SM (16 warps: 8 builders,
// 3 gatherers, producer, MMA issuer, 4 epilogue; see DscTc in the code):
//
//   warps 0-7   builders.  Warp p owns voxel rows 16p..16p+15 of the A tile:
//               it zeroes them, stores C[cell] = s from the staged step
//               (rank 0: distinct cells), adds the repeats with shared-memory
//               reductions in rank order, then splits the rows into tf32
//               hi = x & ~0x1FFF and lo = x - hi in place.  Builder 0 stages
//               each step (one bulk copy of its packed quads, 3 steps ahead)
//               and issues the bulk copy of the chunk's pre-split,
//               pre-swizzled dictionary tile (B operand, hi | lo).
//   warps 13-16 gatherers: for each staged step, s = w[f] * value written
//               over the value field, ahead of the builders.
//   warp 8      MMA issuer (one lane).  3xTF32 per K step of 8 atoms:
//               hi.hi + lo.hi + hi.lo into an fp32 TMEM accumulator; every
//               kTcGroup chunks the accumulator is handed to the epilogue and
//               the next group starts in the other TMEM buffer.
//   warps 9-12  epilogue.  Thread = voxel row (TMEM lane): folds each group's
//               partial into fp32 registers (round-to-nearest adds; the tensor
//               core's own accumulation truncates, so groups stay short: see
//               tools/ubench/tc_probe.cu), and at the end of the tile writes
//               y (accumulate / subtract b) with the sum of squares and max|r|.
//
// Pipelines: A/B stages (full: 8 producer arrivals + the B copy's bytes;
// empty: tcgen05.commit), TMEM buffers (accfull: commit; accempty: 4
// epilogue warps).  Every wait traps after 4 s instead of hanging.
#include <algorithm>

#include "life_common.cuh"

namespace life {

constexpr int kTcMma = 8;                 // MMA warp
constexpr int kTcEpi = 9;                 // first epilogue warp
constexpr int kTcGat0 = 13;               // first gatherer warp
#ifndef LIFE_TC_GATHERERS
#define LIFE_TC_GATHERERS 3
#endif
constexpr int kTcGat = LIFE_TC_GATHERERS;  // gatherer warps
constexpr int kTcWarps = kTcGat0 + kTcGat;
constexpr int kTcThreads = kTcWarps * 32;
#ifndef LIFE_TC_STAGES
#define LIFE_TC_STAGES 2
#endif
constexpr int kTcStages = LIFE_TC_STAGES;  // A/B stages
#ifndef LIFE_TC_GROUP
#define LIFE_TC_GROUP 4
#endif
constexpr int kTcGroup = LIFE_TC_GROUP;    // chunks per TMEM accumulation group
constexpr uint32_t kTcCellMask = (1u << kTcCellBits) - 1;
constexpr uint32_t kTcSent = 0xFFFFFu;     // fascicle field of pad entries
#ifndef LIFE_TC_SLOTS
#define LIFE_TC_SLOTS 4
#endif
constexpr int kTcSlots = LIFE_TC_SLOTS;    // staged steps (kTcSlots-1 ahead of the one being built)
constexpr int kTcABytes = kTcTV * kTcCA * 4;  // 16 KB per A half (hi or lo)

struct TcArgs {
    const uint32_t *q;   // quads {pk[4], value[4]}, pk = fascicle << 12 | cell
    const uint32_t *tptr;
    const uint32_t *t1;
    const float *D;      // [nch][2][N][32] swizzled
    const int *slotv;
    int nt, nch, n_ct;
    int slot;            // staged entries per step slot (multiple of 4)
};

// Diagnostics, compiled in only with -DLIFE_WS_DIAG (tools/tc_isolate.py):
// c_tc_flags 1 = producers skip the tile build, 2 = no MMAs (commits only),
// 4 = no w gathers (w = 1), 8 = epilogue skips the TMEM loads, 16 = no L2
// prefetch, 32 = no dictionary (B) copies; g_tc_cyc
// accumulates per-role clock64 spans.
#ifdef LIFE_WS_DIAG
__constant__ int c_tc_flags = 0;
__device__ unsigned long long g_tc_cyc[16];
#define TC_T0(v) const long long v = clock64()
#define TC_ACC(i, v) (tcc[i] += (unsigned long long)(clock64() - (v)))
#define TC_DECL unsigned long long tcc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define TC_FLUSH                                                               \
    if ((threadIdx.x & 31) == 0)                                               \
        for (int i_ = 0; i_ < 8; ++i_)                                         \
            if (tcc[i_]) atomicAdd(&g_tc_cyc[i_], tcc[i_])
#else
#define TC_DECL
#define TC_FLUSH
constexpr int c_tc_flags = 0;
#define TC_T0(v)
#define TC_ACC(i, v)
#endif

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t tc_sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tc_bar_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_sa(b)), "r"(count));
}
__device__ __forceinline__ void tc_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_sa(b)) : "memory");
}
__device__ __forceinline__ void tc_arrive_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool tc_try(uint64_t *b, unsigned parity)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(tc_sa(b)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool tc_test(uint64_t *b, unsigned parity)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(tc_sa(b)), "r"(parity) : "memory");
    return ok != 0;
}
#ifndef LIFE_TC_SPIN
#define LIFE_TC_SPIN 0
#endif
// waits spin on test_wait (a try_wait that suspends the warp was measured to
// add ~1-2k cycles per hand-over); trap after 4 s instead of hanging
__device__ __forceinline__ void tc_wait(uint64_t *b, unsigned parity)
{
    if (LIFE_TC_SPIN) {
        if (tc_test(b, parity)) return;
        const unsigned long long t0 = globaltimer();
        unsigned n = 0;
        while (!tc_test(b, parity))
            if ((++n & 1023u) == 0 && globaltimer() - t0 > 4000000000ull) __trap();
    } else {
        if (tc_try(b, parity)) return;
        const unsigned long long t0 = globaltimer();
        while (!tc_try(b, parity))
            if (globaltimer() - t0 > 4000000000ull) __trap();
    }
}
__device__ __forceinline__ void tc_bulk(void *dst, const void *src, unsigned bytes, uint64_t *b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(tc_sa(dst)), "l"(src), "r"(bytes), "r"(tc_sa(b)) : "memory");
}
__device__ __forceinline__ uint64_t tc_pol_stream()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t tc_pol_keep()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tc_prefetch(const void *ptr, uint32_t bytes, uint64_t pol)
{
    if (bytes)
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(ptr), "r"(bytes), "l"(pol)
                     : "memory");
}
__device__ __forceinline__ uint4 tc_ld4(const void *p, uint64_t pol)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t tc_ld1(const void *p, uint64_t pol)
{
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float tc_gather(const float *w, uint32_t f, uint64_t pol)
{
    if (f == kTcSent) return 0.f;
    if (c_tc_flags & 4) return 1.f;
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(w + f), "l"(pol));
    return r;
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 version 1):
// 8-row groups 1024 B apart (SBO), 128-byte rows, base 1024-byte aligned
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t addr)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::tf32 instruction descriptor: fp32 accumulator, tf32 A/B, both K-major
__host__ __device__ constexpr uint32_t tc_idesc(int m, int n)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t *b)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc_sa(b))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tc_ld16(uint32_t addr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <typename T, typename Op>
__device__ T tc_reduce(const T *part, int n, T init, Op op)
{
    __shared__ T s[32];
    T acc = init;
    for (int i = threadIdx.x; i < n; i += kTcThreads) acc = op(acc, __ldcg(part + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = op(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    T r = init;
    if (threadIdx.x < 32) {
        r = threadIdx.x < kTcWarps ? s[threadIdx.x] : init;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = op(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (threadIdx.x == 0) s[0] = r;
    }
    __syncthreads();
    r = s[0];
    __syncthreads();
    return r;
}
struct TcAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct TcMax {
    __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};

// ---- builder: one 16-row block of the A tile for one chunk ---------------------
// The layout stores entries as 32-byte quads {pk[4], value[4]}; a step's 8
// segments are contiguous, so builder 0 stages the whole step with one bulk
// copy into a shared-memory slot, 3 steps ahead (kTcSlots slots), after an
// L2 prefetch 6 steps ahead.  A warp's segment is (p0, q0, p1): rank-0
// entries [p0, q0) (distinct cells), repeats [q0, p1) sorted by rank, each
// region padded to 4.  The gatherer warps turn value into s = w[f] * value in
// the slot before the builders read it.

// explicit shared-memory accesses (32-bit shared-window addresses)
__device__ __forceinline__ uint4 lds4(uint32_t a)
{
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds1(uint32_t a)
{
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ float ldsf(uint32_t a)
{
    float r;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ void stsf(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory"); }
__device__ __forceinline__ void sts4(uint32_t a, float4 v)
{
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 lds4f(uint32_t a)
{
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
    return r;
}

// a warp's segment inside a staged step: entries at slot offset < cap are in
// shared memory (quads at sbase), the rest (steps longer than a slot, rare)
// in global memory
struct TcSeg {
    uint32_t sbase;       // shared address of the step's slot
    const uint32_t *gq;   // global quads of the step
    uint32_t off;         // segment start, entries from the step start
    uint32_t nf, n;       // rank-0 entries, all entries
    uint32_t cap;         // staged entries
    // field 0 = pk, 1 = value of the 4 entries starting at k (k % 4 == 0)
    __device__ __forceinline__ uint4 q4(uint32_t k, int field) const
    {
        const uint32_t o = off + k;
        if (o < cap) return lds4(sbase + (o >> 2) * 32u + 16u * field);
        return __ldg(reinterpret_cast<const uint4 *>(gq + (o >> 2) * 8u + 4u * field));
    }
    __device__ __forceinline__ uint32_t word(uint32_t k, int field) const
    {
        const uint32_t o = off + k;
        if (o < cap) return lds1(sbase + (o >> 2) * 32u + 16u * field + 4u * (o & 3u));
        return __ldg(gq + (o >> 2) * 8u + 4u * field + (o & 3u));
    }
};

__device__ __forceinline__ void reds(uint32_t a, float v)
{
    asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// build from a step whose gatherers already replaced value by s = w[f] * value
// (slot field 1); entries beyond the slot (global) are gathered here
__device__ __forceinline__ unsigned tc_build_s(uint32_t C, const TcSeg &S, const float *__restrict__ w,
                                               int lane, uint64_t pol, uint32_t junk)
{
    unsigned zeros = 0;
    for (uint32_t k = 4u * (uint32_t)lane; k < S.nf; k += 128u) {
        const uint4 c4 = S.q4(k, 0);
        const uint4 v4 = S.q4(k, 1);
        const uint32_t c[4] = {c4.x, c4.y, c4.z, c4.w};
        float sv[4] = {__uint_as_float(v4.x), __uint_as_float(v4.y), __uint_as_float(v4.z), __uint_as_float(v4.w)};
        if (S.off + k >= S.cap) {  // not staged: the gatherers did not see it
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                sv[e] = __fmul_rn(tc_gather(w, c[e] >> kTcCellBits, pol), sv[e]);
                zeros += ((c[e] >> kTcCellBits) != kTcSent && sv[e] == 0.f) ? 1u : 0u;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) stsf((c[e] >> kTcCellBits) != kTcSent ? C + 4u * (c[e] & kTcCellMask) : junk, sv[e]);
    }
    __syncwarp();
    for (uint32_t k = S.nf + (uint32_t)lane; k < S.n; k += 32u) {
        const uint32_t c = S.word(k, 0);
        if ((c >> kTcCellBits) == kTcSent) continue;
        float sv = __uint_as_float(S.word(k, 1));
        if (S.off + k >= S.cap) {
            sv = __fmul_rn(tc_gather(w, c >> kTcCellBits, pol), sv);
            zeros += sv == 0.f ? 1u : 0u;
        }
        reds(C + 4u * (c & kTcCellMask), sv);
    }
    return zeros;
}

// bulk copy / L2 prefetch of a byte range in pieces of at most 32 KB
__device__ __forceinline__ void tc_stage_step(void *dst, const void *src, unsigned bytes, uint64_t *bar,
                                              uint64_t pol)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_arrive_tx(bar, bytes);
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
    for (unsigned o = 0; o < bytes; o += 32768u)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(tc_sa(d + o)), "l"(s + o), "r"(min(32768u, bytes - o)), "r"(tc_sa(bar)), "l"(pol)
                     : "memory");
}
__device__ __forceinline__ void tc_prefetch_step(const void *src, unsigned bytes, uint64_t pol)
{
    const char *s = reinterpret_cast<const char *>(src);
    for (unsigned o = 0; o < bytes; o += 32768u) tc_prefetch(s + o, min(32768u, bytes - o), pol);
}

template <int NJ>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_dsc_tc(const TcArgs A, const float *__restrict__ w, float *__restrict__ y,
             const float *__restrict__ b, const uint32_t flags, const ReduceSlots red,
             const DscOut out, const CallHooks hooks)
{
    constexpr int N = 32 * NJ;
    constexpr int kBBytes = 2 * N * kTcCA * 4;        // hi | lo
    constexpr int kStageBytes = 2 * kTcABytes + kBBytes;
    extern __shared__ __align__(1024) unsigned char tc_smraw[];
    __shared__ __align__(8) uint64_t full[kTcStages], empty[kTcStages], accfull[2], accempty[2];
    __shared__ __align__(8) uint64_t slotfull[kTcSlots], slotfree[kTcSlots], slotready[kTcSlots];
    __shared__ uint32_t tmem_base;
    __shared__ float junkbuf[kTcProd * 32];
    if (hooks.done && *hooks.done) return;
    unsigned char *sm = (unsigned char *)(((uintptr_t)tc_smraw + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int my_ct = (int)blockIdx.x < A.n_ct ? (A.n_ct - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_ct * A.nch;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            tc_bar_init(&full[s], kTcProd + 1);
            tc_bar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc_bar_init(&accfull[s], 1);
            tc_bar_init(&accempty[s], 4);
        }
        for (int j = 0; j < kTcSlots; ++j) {
            tc_bar_init(&slotready[j], kTcGat);
            tc_bar_init(&slotfull[j], 1);
            tc_bar_init(&slotfree[j], kTcProd);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kTcMma) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tc_sa(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    double sq = 0.0;
    float amax = 0.f;
    unsigned long long skipped = 0;
    TC_DECL;

    if (warp < kTcProd) {
        // ===== producers =====
        const int p = warp;
        const uint64_t pol_s = tc_pol_stream(), pol_k = tc_pol_keep();
        const uint32_t junk = tc_sa(junkbuf + p * 32 + lane);
        uint32_t *slotbase = reinterpret_cast<uint32_t *>(sm + (size_t)kTcStages * kStageBytes);
        const uint32_t slot_sa = tc_sa(slotbase);
        const uint32_t cap = (uint32_t)A.slot;
        // segment bounds of 32 steps per window, lane l holding step base+l:
        // {p0, q0, p1, step start, step end}; the next window is loaded 32
        // steps before it is needed
        uint32_t cb[5], nb[5];
        auto loadw = [&](int base, uint32_t (&o)[5]) {
            const int kk = base + lane;
            if (kk < total) {
                const size_t T = ((size_t)(blockIdx.x + (kk / A.nch) * gridDim.x) * A.nch + kk % A.nch) * kTcProd;
                o[0] = __ldg(A.tptr + T + p);
                o[1] = __ldg(A.t1 + T + p);
                o[2] = __ldg(A.tptr + T + p + 1);
                o[3] = __ldg(A.tptr + T);
                o[4] = __ldg(A.tptr + T + kTcProd);
            } else {
                o[0] = o[1] = o[2] = o[3] = o[4] = 0u;
            }
        };
        loadw(0, cb);
        loadw(32, nb);
        int wbase = 0;
        auto bnd = [&](int kk, int i) {
            const int d = kk - wbase;
            return __shfl_sync(0xffffffffu, d < 32 ? cb[i] : nb[i], d & 31);
        };
        auto segv = [&](int kk) {
            const uint32_t b0 = bnd(kk, 0), b1 = bnd(kk, 1), b2 = bnd(kk, 2), s0 = bnd(kk, 3);
            return TcSeg{slot_sa + (uint32_t)(kk % kTcSlots) * 8u * cap, A.q + (size_t)s0 * 2u, b0 - s0, b1 - b0, b2 - b0, cap};
        };
        auto stage = [&](int kk) {  // producer 0, lane 0
            const uint32_t s0 = bnd(kk, 3), s1 = bnd(kk, 4);
            const uint32_t n = min(s1 - s0, cap);
            const int j = kk % kTcSlots;
            if (lane == 0) {
                if (kk >= kTcSlots && !(c_tc_flags & 1024)) tc_wait(&slotfree[j], ((kk / kTcSlots) - 1) & 1);
                if (c_tc_flags & 128) { tc_arrive(&slotfull[j]); return; }
                tc_stage_step(slotbase + (size_t)j * 2u * cap, A.q + (size_t)s0 * 2u, n * 8u, &slotfull[j], pol_s);
            }
        };
        // L2 prefetch of a step: one 128-byte line per lane and instruction
        // (LSU-issued, many lines in flight; the bulk copy engine alone keeps
        // too few HBM requests outstanding for a once-read stream)
        auto prefetch = [&](int kk) {
            const uint32_t s0 = bnd(kk, 3), s1 = bnd(kk, 4);
            if (c_tc_flags & 16) return;
            const char *b = reinterpret_cast<const char *>(A.q + (size_t)s0 * 2u);
            const uint32_t bytes = (s1 - s0) * 8u;
            for (uint32_t o = (uint32_t)lane * 128u; o < bytes; o += 32u * 128u)
                asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(b + o));
        };
        constexpr int kAhead = kTcSlots - 1, kPre = 2 * kAhead;
        if (p == 0) {
            for (int kk = 0; kk < kAhead && kk < total; ++kk) stage(kk);
            for (int kk = kAhead; kk < kPre && kk < total; ++kk) prefetch(kk);
        }
        int c0 = 0;
        for (int k = 0; k < total; ++k) {
            const int s = k % kTcStages;
            if (k > 0 && (k & 31) == 0) {
#pragma unroll
                for (int i = 0; i < 5; ++i) cb[i] = nb[i];
                wbase = k;
                loadw(k + 32, nb);
            }
            if (p == 0) {
                if (k + kAhead < total) stage(k + kAhead);
                if (k + kPre < total) prefetch(k + kPre);
            }
            TC_T0(t_slot);
            if (!(c_tc_flags & 1024)) tc_wait(&slotready[k % kTcSlots], (k / kTcSlots) & 1);
            if (lane == 0) TC_ACC(0, t_slot);
            TC_T0(t_empty);
            if (k >= kTcStages && !(c_tc_flags & 1024)) tc_wait(&empty[s], ((k / kTcStages) - 1) & 1);
            if (lane == 0) TC_ACC(1, t_empty);
            TC_T0(t_build);
            unsigned char *st = sm + (size_t)s * kStageBytes;
            float *Ahi = reinterpret_cast<float *>(st);
            float *Alo = reinterpret_cast<float *>(st + kTcABytes);
            if (p == 0 && lane == 0) {
                if (c_tc_flags & 32) {
                    tc_arrive(&full[s]);
                } else {
                    tc_arrive_tx(&full[s], kBBytes);
                    tc_bulk(st + 2 * kTcABytes, A.D + (size_t)c0 * (kBBytes / 4), kBBytes, &full[s]);
                }
            }
            // zero this warp's rows (2 KB)
            const uint32_t H = tc_sa(Ahi) + (uint32_t)p * 2048u, L = tc_sa(Alo) + (uint32_t)p * 2048u;
#pragma unroll
            for (int i = 0; i < 4; ++i) sts4(H + 16u * (lane + 32 * i), make_float4(0.f, 0.f, 0.f, 0.f));
            __syncwarp();
            if (!(c_tc_flags & 1)) skipped += tc_build_s(tc_sa(Ahi), segv(k), w, lane, pol_k, junk);
            __syncwarp();
            if (lane == 0) {
                tc_arrive(&slotfree[k % kTcSlots]);  // this warp is done with the step's slot
                TC_ACC(2, t_build);
            }
            TC_T0(t_split);
            // tf32 split of this warp's rows: hi in place, lo alongside
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float4 x = lds4f(H + 16u * (lane + 32 * i));
                float4 h, l;
                h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
                h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
                h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
                h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
                l.x = x.x - h.x;
                l.y = x.y - h.y;
                l.z = x.z - h.z;
                l.w = x.w - h.w;
                sts4(H + 16u * (lane + 32 * i), h);
                sts4(L + 16u * (lane + 32 * i), l);
            }
            // generic-proxy stores -> visible to the tensor core (async proxy)
            if (!(c_tc_flags & 256)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) TC_ACC(3, t_split);
            if (lane == 0) tc_arrive(&full[s]);
            if (++c0 == A.nch) c0 = 0;
        }
    } else if (warp >= kTcGat0) {
        // ===== gatherers: s = w[f] * value in place, one staged step at a time =====
        const int g = warp - kTcGat0;
        const uint64_t pol_k = tc_pol_keep();
        const uint32_t slot_sa = tc_sa(sm + (size_t)kTcStages * kStageBytes);
        const uint32_t cap = (uint32_t)A.slot;
        uint32_t c3 = 0, c4v = 0, n3 = 0, n4 = 0;  // step start / end, windows of 32 steps
        auto loadw = [&](int base, uint32_t &o3, uint32_t &o4) {
            const int kk = base + lane;
            if (kk < total) {
                const size_t T = ((size_t)(blockIdx.x + (kk / A.nch) * gridDim.x) * A.nch + kk % A.nch) * kTcProd;
                o3 = __ldg(A.tptr + T);
                o4 = __ldg(A.tptr + T + kTcProd);
            } else {
                o3 = o4 = 0u;
            }
        };
        loadw(0, c3, c4v);
        loadw(32, n3, n4);
#ifndef LIFE_TC_GATHER_U
#define LIFE_TC_GATHER_U 1
#endif
        constexpr int kU = LIFE_TC_GATHER_U;  // quads per thread and pass (all loads first)
        for (int kk = 0; kk < total; ++kk) {
            if (kk > 0 && (kk & 31) == 0) {
                c3 = n3;
                c4v = n4;
                loadw(kk + 32, n3, n4);
            }
            const uint32_t s0 = __shfl_sync(0xffffffffu, c3, kk & 31);
            const uint32_t s1 = __shfl_sync(0xffffffffu, c4v, kk & 31);
            const int j = kk % kTcSlots;
            tc_wait(&slotfull[j], (kk / kTcSlots) & 1);
            const uint32_t n = min(s1 - s0, cap), nq = (n + 3u) / 4u;
            const uint32_t base = slot_sa + (uint32_t)j * 8u * cap;
            for (uint32_t q0 = (uint32_t)(g * 32 + lane); q0 < nq; q0 += (uint32_t)(kTcGat * 32 * kU)) {
                uint4 pk[kU], v4[kU];
                float wv[kU][4];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const uint32_t q = q0 + (uint32_t)(u * kTcGat * 32);
                    pk[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
                    if (q < nq) {
                        pk[u] = lds4(base + q * 32u);
                        v4[u] = lds4(base + q * 32u + 16u);
                    }
                    wv[u][0] = tc_gather(w, pk[u].x >> kTcCellBits, pol_k);
                    wv[u][1] = tc_gather(w, pk[u].y >> kTcCellBits, pol_k);
                    wv[u][2] = tc_gather(w, pk[u].z >> kTcCellBits, pol_k);
                    wv[u][3] = tc_gather(w, pk[u].w >> kTcCellBits, pol_k);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const uint32_t q = q0 + (uint32_t)(u * kTcGat * 32);
                    if (q >= nq) continue;
                    const uint32_t c[4] = {pk[u].x, pk[u].y, pk[u].z, pk[u].w};
                    const float v[4] = {__uint_as_float(v4[u].x), __uint_as_float(v4[u].y),
                                        __uint_as_float(v4[u].z), __uint_as_float(v4[u].w)};
                    float sv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        sv[e] = __fmul_rn(wv[u][e], v[e]);
                        skipped += ((c[e] >> kTcCellBits) != kTcSent && sv[e] == 0.f) ? 1u : 0u;
                    }
                    sts4(base + q * 32u + 16u, make_float4(sv[0], sv[1], sv[2], sv[3]));
                }
            }
            __syncwarp();
            if (lane == 0) tc_arrive(&slotready[j]);
        }
    } else if (warp == kTcMma) {
        // ===== MMA issuer =====
        if (lane == 0) {
            constexpr uint32_t id = tc_idesc(kTcTV, N);
            int k = 0, grp = 0;
            for (int i = 0; i < my_ct; ++i) {
                for (int c = 0; c < A.nch; ++c, ++k) {
                    const int s = k % kTcStages;
                    const int buf = grp & 1;
                    if (c % kTcGroup == 0) {
                        TC_T0(t_ae);
                        if (grp >= 2) tc_wait(&accempty[buf], ((grp >> 1) - 1) & 1);
                        TC_ACC(6, t_ae);
                        tc_fence_after();
                    }
                    TC_T0(t_full);
                    tc_wait(&full[s], (k / kTcStages) & 1);
                    TC_ACC(5, t_full);
                    tc_fence_after();
                    const uint32_t st = tc_sa(sm + (size_t)s * kStageBytes);
                    const uint64_t ah = tc_sdesc(st), al = tc_sdesc(st + kTcABytes);
                    const uint64_t bh = tc_sdesc(st + 2 * kTcABytes), bl = tc_sdesc(st + 2 * kTcABytes + N * 128);
                    const uint32_t d = tmem + (uint32_t)(buf * N);
#pragma unroll
                    for (int kk = 0; kk < kTcCA / 8; ++kk) {
                        const uint64_t o = (uint64_t)((kk * 32) >> 4);  // 8 tf32 = 32 bytes per K step
                        if (c_tc_flags & 2) continue;
                        tc_mma(d, ah + o, bh + o, id, (c % kTcGroup) != 0 || kk != 0);
                        tc_mma(d, al + o, bh + o, id, 1u);
                        tc_mma(d, ah + o, bl + o, id, 1u);
                    }
                    if (c_tc_flags & 512) tc_arrive(&empty[s]);
                    else tc_commit(&empty[s]);
                    if (c % kTcGroup == kTcGroup - 1 || c == A.nch - 1) {
                        if (c_tc_flags & 512) tc_arrive(&accfull[buf]);
                        else tc_commit(&accfull[buf]);
                        ++grp;
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ===== epilogue: thread = voxel row (TMEM lane) =====
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const bool accumulate = flags & LIFE_ACCUMULATE;
        const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
        const int ngroups = (A.nch + kTcGroup - 1) / kTcGroup;
        int grp = 0;
        for (int i = 0; i < my_ct; ++i) {
            const int ct = blockIdx.x + i * gridDim.x;
            float acc[N];
#pragma unroll
            for (int t = 0; t < N; ++t) acc[t] = 0.f;
            for (int g = 0; g < ngroups; ++g, ++grp) {
                const int buf = grp & 1;
                TC_T0(t_af);
                tc_wait(&accfull[buf], (grp >> 1) & 1);
                if (lane == 0) TC_ACC(7, t_af);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < 2 * NJ; ++j) {
                    if (c_tc_flags & 8) break;
                    float v[16];
                    tc_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * N + 16 * j), v);
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[16 * j + e] += v[e];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) tc_arrive(&accempty[buf]);
            }
            const int voxel = (c_tc_flags & 64) ? -1 : __ldg(A.slotv + (size_t)ct * kTcTV + row);
            if (voxel >= 0 && (A.nt & 3) == 0) {
                // 16-byte row accesses (rows are 16-byte aligned when nt % 4 == 0)
                const size_t yo = (size_t)voxel * A.nt;
                float4 *y4 = reinterpret_cast<float4 *>(y + yo);
                const float4 *b4 = reinterpret_cast<const float4 *>(subtract ? b + yo : y + yo);
#pragma unroll
                for (int t4 = 0; t4 < N / 4; ++t4) {
                    if (4 * t4 < A.nt) {
                        float r[4] = {acc[4 * t4], acc[4 * t4 + 1], acc[4 * t4 + 2], acc[4 * t4 + 3]};
                        if (accumulate) {
                            const float4 o = y4[t4];
                            r[0] += o.x; r[1] += o.y; r[2] += o.z; r[3] += o.w;
                        }
                        if (subtract) {
                            const float4 o = __ldg(b4 + t4);
                            r[0] -= o.x; r[1] -= o.y; r[2] -= o.z; r[3] -= o.w;
                        }
                        y4[t4] = make_float4(r[0], r[1], r[2], r[3]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            sq += (double)r[e] * (double)r[e];
                            amax = fmaxf(amax, fabsf(r[e]));
                        }
                    }
                }
            } else if (voxel >= 0) {
                const size_t yo = (size_t)voxel * A.nt;
#pragma unroll
                for (int t = 0; t < N; ++t) {
                    if (t < A.nt) {
                        float r = acc[t];
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

    // ---- teardown and fixed-order completion ------------------------------------
    TC_FLUSH;
    tc_fence_before();
    __syncthreads();
    if (warp == kTcMma) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
    const int gw = blockIdx.x * kTcWarps + warp;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        skipped += __shfl_xor_sync(0xffffffffu, skipped, o);
    }
    if (lane == 0) {
        red.part_d[gw] = sq;
        red.part_u[gw] = skipped;
        red.part_f[gw] = amax;
    }
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(red.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        const int W = gridDim.x * kTcWarps;
        const double tsq = tc_reduce<double>(red.part_d, W, 0.0, TcAdd{});
        const unsigned long long tsk = tc_reduce<unsigned long long>(red.part_u, W, 0ull, TcAdd{});
        const float tmax = tc_reduce<float>(red.part_f, W, 0.f, TcMax{});
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
// dispatch
// ---------------------------------------------------------------------------
static size_t tc_stage_bytes(int N) { return (size_t)kTcStages * (2 * kTcABytes + 2 * N * kTcCA * 4); }

// staged entries per step slot: what fits next to the A/B stages (kTcSlots
// slots x 8 bytes per entry), a multiple of 32
static int tc_slot_entries(int N)
{
    const long avail = 232448L - 1024 - 4096 - (long)tc_stage_bytes(N);  // dyn limit - align - static
    return (int)std::max(0L, avail / ((long)kTcSlots * 8) / 32 * 32);
}

static size_t tc_smem_bytes(int N)
{
    return tc_stage_bytes(N) + (size_t)kTcSlots * 8 * tc_slot_entries(N) + 1024;  // + alignment slack
}

template <int NJ>
static int tc_dsc_t(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                    const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    TcArgs A{phi->t_q, phi->t_tptr, phi->t_t1, phi->t_D, phi->t_slotv,
             phi->nt, phi->t_nch, phi->t_nct, tc_slot_entries(phi->t_n)};
    k_dsc_tc<NJ><<<phi->t_blocks, kTcThreads, phi->t_smem, st>>>(A, w, y, b, flags, phi->red, o, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int NJ>
static int tc_prepare_t(life_phi *phi)
{
    if (tc_slot_entries(32 * NJ) < 512)
        return fail(LIFE_ERR_CONFIG_INVALID, "tc layout: staging slots do not fit");
    phi->t_smem = tc_smem_bytes(32 * NJ);
    phi->t_W = phi->t_blocks * kTcWarps;
    return ensure_smem(k_dsc_tc<NJ>, phi->t_smem);
}

#define LIFE_TC_DISPATCH(FN, ...)                                              \
    switch (phi->t_n / 32) {                                                   \
    case 1: return FN<1>(__VA_ARGS__);                                         \
    case 2: return FN<2>(__VA_ARGS__);                                         \
    case 3: return FN<3>(__VA_ARGS__);                                         \
    case 4: return FN<4>(__VA_ARGS__);                                         \
    default: return fail(LIFE_ERR_CONFIG_INVALID, "tc layout: unsupported n_dirs"); \
    }

int launch_dsc_tc(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                  const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_TC_DISPATCH(tc_dsc_t, phi, w, y, b, flags, o, h, st);
}

int prepare_tc(life_phi *phi) { LIFE_TC_DISPATCH(tc_prepare_t, phi); }

}  // namespace life

#ifdef LIFE_WS_DIAG
extern "C" LIFE_API int life_debug_tc(int flags, unsigned long long *cyc_out)
{
    if (cyc_out) {
        if (cudaDeviceSynchronize() != cudaSuccess) return 20;
        if (cudaMemcpyFromSymbol(cyc_out, life::g_tc_cyc, 16 * sizeof(unsigned long long)) != cudaSuccess) return 20;
        unsigned long long z[16] = {};
        if (cudaMemcpyToSymbol(life::g_tc_cyc, z, sizeof(z)) != cudaSuccess) return 20;
    }
    return cudaMemcpyToSymbol(life::c_tc_flags, &flags, sizeof(int)) == cudaSuccess ? 0 : 20;
}
#endif
