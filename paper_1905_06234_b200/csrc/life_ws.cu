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
// Layout: one segment per (CTA tile round ct, atom chunk c, producer warp
// p), i.e. per PAIR of consumer tiles (2p, 2p+1): a rank-0 region (each
// cell's first coefficient; cells are 11 bits = tile-in-pair, atom, voxel
// slot, all distinct) then a rank>=1 region (repeats, sorted by rank), each
// padded to a multiple of 4 entries with pad entries (cr bit 30).  The pair's
// two C tiles are adjacent in shared memory, so an entry's tile is just bit 10
// of its cell.  Voxels are dealt to tile slots by coefficient count
// (life_dense.cu), so every segment carries about the same work.
//
// Coefficient staging (the "staged" producer): lane 0 of each producer warp
// copies the next step's segment into one of the warp's two shared-memory
// slots with three cp.async.bulk copies (index / fascicle / value arrays,
// mbarrier complete_tx) and prefetches the step after that into L2, so the
// producers see shared-memory latency for the stream and only the w[f]
// gathers (DSC) or RED.ADDs (WC) go to L2.  Operators with a segment larger
// than a slot fall back to the register-streaming producer (same results,
// bit for bit).
//
// Steps are double buffered (C/Z tiles and dictionary chunks) and handed over
// with mbarriers (full/empty).  Each LDS.128 costs four shared-memory
// wavefronts on sm_100 (measured, tools/ubench); the 8x12 lane tile needs 5 of
// them per 96 FMAs per lane, keeping shared memory below the FP32 pipe.
#include <algorithm>

#include "life_common.cuh"
#include "life_tcgen05.cuh"

namespace life {

constexpr int kWsCons = 8;
#ifndef LIFE_WS_PROD
#define LIFE_WS_PROD 8
#endif
#if LIFE_WS_PROD != 8
#error "the WC kernel pairs up the per-tile segments of the 8-producer layout"
#endif
constexpr int kWsProd = LIFE_WS_PROD;      // producer warps (4 or 8)
constexpr int kTPP = kWsCons / kWsProd;   // consumer tiles per producer warp
constexpr int kWsWarps = kWsCons + kWsProd;
// 8 producer warps: registers are split between the roles with setmaxnreg
// (consumers 168 for their 96 accumulators, producers 88)
constexpr bool kSplitRegs = kWsProd == 8;
constexpr int kRegCons = 168;
constexpr int kRegProd = 88;
static_assert(!kSplitRegs || kWsCons * kRegCons + kWsProd * kRegProd <= 2048, "register file");
constexpr int kWsThreads = kWsWarps * 32;
constexpr int kWsTV = 32;                  // voxels per consumer tile
constexpr int kWsCA = 32;                  // atoms per chunk
constexpr int kWsCells = kWsTV * kWsCA;    // 1024 cells per tile
constexpr int kWsCellBits = kTPP == 2 ? 11 : 10;  // cell within a producer's tiles
constexpr uint32_t kCellMask = kTPP * kWsCells - 1;
constexpr uint32_t kPadBit = 0x40000000u;  // pad entry
constexpr uint32_t kMixedBit = 0x80000000u;  // 32-window straddles two ranks
constexpr uint32_t kRankMask = (1u << (30 - kWsCellBits)) - 1;  // rank: bits cellbits..29
#ifndef LIFE_WS_CPASYNC
#define LIFE_WS_CPASYNC 0
#endif
// staged producers: gather w with cp.async into the slot one step ahead (1)
// or into registers within the step (0)
constexpr bool kCpAsyncGather = LIFE_WS_CPASYNC;
constexpr int kWsSlot = 720 * kTPP;        // staged entries per (producer warp, slot)
static_assert(kTPP == 1 || kTPP == 2, "a producer warp owns one or two adjacent tiles");

struct WsArgs {
    const uint32_t *cr;
    const uint32_t *fiber;
    const float *val;
    const uint32_t *tptr;   // padded pair-segment starts, [n_ct*nch*4 + 1]
    const uint32_t *t1;     // start of each segment's rank>=1 region
    const float *D;
    const int *slotv;       // voxel of each tile slot (tile*32 + i), -1 for padding
    int nv, nt, nt_pad, nch, n_tiles, na;
};
// Diagnostic isolation, compiled in only with -DLIFE_WS_DIAG (tools/ws_isolate.py):
// c_ws_isolate 1 = producers only, 2 = consumers only (results are garbage);
// c_ws_flags 1 = no L2 prefetch, 4 = no gather.
#ifdef LIFE_WS_DIAG
__constant__ int c_ws_isolate = 0;
__constant__ int c_ws_flags = 0;
// producer-warp cycle counters: [0] slot wait, [1] empty wait, [2] build, [3] steps,
// [4] consumer full wait, [5] consumer compute
__device__ unsigned long long g_ws_cyc[8];
#define WS_T0(v) const long long v = clock64()
#define WS_ACC(i, v) atomicAdd(&g_ws_cyc[i], (unsigned long long)(clock64() - (v)))
#else
#define WS_T0(v)
#define WS_ACC(i, v)
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
__device__ __forceinline__ bool bar_try(uint64_t *b, unsigned parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smaddr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// A wait that has not completed after 4 s of device time is a protocol
// deadlock: trap (the launch fails with an error) instead of hanging the GPU.
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned parity)
{
    if (bar_try(b, parity)) return;
    const unsigned long long t0 = globaltimer();
    while (!bar_try(b, parity))
        if (globaltimer() - t0 > 4000000000ull) __trap();
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

// L2 policies: the coefficient stream (read once per SpMV, 1.2 GB at C2) is
// evict-first so it does not push the gathered / scattered Nf-vectors (w,
// the fixed-point sums) out of L2; those are evict-last.
// (A/B: LIFE_WS_POL_STREAM / LIFE_WS_POL_KEEP = 0 evict_normal, 1 evict_first,
// 2 evict_last, 3 evict_unchanged)
#ifndef LIFE_WS_POL_STREAM
#define LIFE_WS_POL_STREAM 1
#endif
#ifndef LIFE_WS_POL_KEEP
#define LIFE_WS_POL_KEEP 2
#endif
template <int K>
__device__ __forceinline__ uint64_t make_policy()
{
    uint64_t p;
    if (K == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (K == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else if (K == 3) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_stream() { return make_policy<LIFE_WS_POL_STREAM>(); }
__device__ __forceinline__ uint64_t policy_keep() { return make_policy<LIFE_WS_POL_KEEP>(); }

__device__ __forceinline__ void prefetch_l2(const void *ptr, uint32_t bytes)
{
    if (bytes == 0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(ptr), "r"(bytes),
                 "l"(policy_stream())
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s_stream(void *dst, const void *src, unsigned bytes,
                                                uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smaddr(dst)),
        "l"(src), "r"(bytes), "r"(smaddr(b)), "l"(policy_stream())
        : "memory");
}

// w[f] gathers: evict-last in L2, no L1 allocation (the gathered lines are
// never reused from L1; allocating them cost DSC 5.5% at C2, 1.438 -> 1.359 ms)
__device__ __forceinline__ float ld_keep(const float *p, uint64_t pol)
{
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ void red_keep(unsigned long long *p, unsigned long long v, uint64_t pol)
{
    asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// Repeats (rank >= 1, sorted by rank then cell), all in a fixed summation
// order (each cell's repeats added in rank order):
//   LIFE_WS_ORDERED=2 (default) batches of 8 windows, one round of
//     read-modify-writes per rank level (cells are distinct within a level);
//   LIFE_WS_ORDERED=1 window by window, per-rank rounds only in windows that
//     straddle two levels;
//   LIFE_WS_ORDERED=0 shared-memory reductions in rank order (not native for
//     f32 on sm_100: a CAS loop; same time as 1 at C2).
#ifndef LIFE_WS_ORDERED
#define LIFE_WS_ORDERED 2
#endif
__device__ __forceinline__ void ws_red_add(float *p, float v)
{
    asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(smaddr(p)), "f"(v) : "memory");
}

// ---- a producer warp's step: the pair segment of (ct, chunk, p) ------------
struct Seg {
    uint32_t p0, q0, p1;  // rank-0 region [p0, q0), rank>=1 region [q0, p1)
};

__device__ __forceinline__ Seg seg_of(const WsArgs &A, int ct, int c, int p)
{
    const size_t t = ((size_t)ct * A.nch + c) * kWsProd + p;
    Seg S;
    S.p0 = __ldg(A.tptr + t);
    S.q0 = __ldg(A.t1 + t);
    S.p1 = __ldg(A.tptr + t + 1);
    return S;
}

// WC's balanced schedule: the n_ct * nch steps (ct, c), c fastest, are cut
// into gridDim.x contiguous ranges of equal length, so every CTA does the
// same number of steps (a round robin of whole CTA tiles leaves the last of
// 5.28 rounds 72% idle at C2).  WC has no state across chunks (Z is per chunk
// and the fascicle sums are integer), so a CTA tile may be split anywhere.
__device__ __forceinline__ void step_range(int n_ct, int nch, int &s0, int &s1)
{
    const long long total = (long long)n_ct * nch;
    s0 = (int)(total * blockIdx.x / gridDim.x);
    s1 = (int)(total * (blockIdx.x + 1) / gridDim.x);
}

// DSC: whole CTA tiles round robin over the grid
__device__ __forceinline__ void step_next_rr(int &ct, int &c, int nch)
{
    if (++c == nch) {
        c = 0;
        ct += gridDim.x;
    }
}

__device__ __forceinline__ void step_next(int &ct, int &c, int nch)
{
    if (++c == nch) {
        c = 0;
        ++ct;
    }
}

// L2 prefetch of a segment one step ahead of its use.  Only the unstaged
// (register-streaming) producers use it: staged producers' bulk copies
// already fetch the segment a step ahead, and the extra prefetch measured
// 2.6% (DSC) / 4% (WC) slower at C2.
#ifndef LIFE_WS_L2PREFETCH
#define LIFE_WS_L2PREFETCH 0
#endif
template <bool STAGED>
__device__ __forceinline__ void prefetch_seg(const WsArgs &A, const Seg &S, int lane)
{
    if (STAGED && !LIFE_WS_L2PREFETCH) return;
    if ((c_ws_flags & 1) || S.p1 <= S.p0 || lane >= 3) return;
    const uint32_t bytes = (S.p1 - S.p0) * 4u;  // padded segments are 16-byte aligned
    const void *base = lane == 0 ? (const void *)(A.cr + S.p0)
                     : lane == 1 ? (const void *)(A.fiber + S.p0)
                                 : (const void *)(A.val + S.p0);
    prefetch_l2(base, bytes);
}

// A segment's entries, relative to its start: a shared-memory slot (staged)
// or the global arrays offset by p0 (fallback).
struct View {
    const uint32_t *cr;
    const uint32_t *f;
    const float *v;
};

__device__ __forceinline__ View slot_view(float *slots, int p, int s)
{
    uint32_t *base = reinterpret_cast<uint32_t *>(slots) + (size_t)(p * 2 + s) * 3 * kWsSlot;
    return View{base, base + kWsSlot, reinterpret_cast<const float *>(base + 2 * kWsSlot)};
}

__device__ __forceinline__ View global_view(const WsArgs &A, const Seg &S)
{
    return View{A.cr + S.p0, A.fiber + S.p0, A.val + S.p0};
}

template <bool STAGED, typename T>
__device__ __forceinline__ T ldv(const T *p)
{
    if constexpr (STAGED) return *p;
    else return ld_stream(p);
}

// lane 0: copy segment S into the warp's slot (three bulk copies)
__device__ __forceinline__ void stage_issue(const WsArgs &A, const Seg &S, float *slots, int p,
                                            int s, uint64_t *bar)
{
    const unsigned n = S.p1 - S.p0, bytes = n * 4u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bar_arrive_tx(bar, 3u * bytes);
    if (n) {
        const View D = slot_view(slots, p, s);
        bulk_g2s_stream((void *)D.cr, A.cr + S.p0, bytes, bar);
        bulk_g2s_stream((void *)D.f, A.fiber + S.p0, bytes, bar);
        bulk_g2s_stream((void *)D.v, A.val + S.p0, bytes, bar);
    }
}

constexpr uint32_t kSent = 0xFFFFFFFFu;  // fascicle field of pad entries

__device__ __forceinline__ float gather_w(const float *__restrict__ w, uint32_t f)
{
    return f == kSent ? 0.f : ((c_ws_flags & 4) ? 1.f : ld_keep(w + f, policy_keep()));
}

// Build the producer warp's two coefficient tiles (C: 2 x 1024 floats) from
// its segment.  Two phases per batch keep few registers live: first every
// lane issues the w[f] gathers of its entries (4 per 128-entry block, one
// per 32-entry window), then it reloads index and value and stores
// C[cell] = w * value.  The first batch of rank>=1 windows is gathered with
// the rank-0 batch, so a typical step has one gather round trip.  Repeats
// are added after every rank-0 store, window by window in rank order; a
// window straddling two rank levels (kMixedBit) is applied rank by rank.
// Gather batch sizes: one 128-entry block of the rank-0 region and 4 repeat
// windows per batch.  Smaller batches measured faster than larger ones
// (C2 DSC 1.30 ms with 4 blocks / 8 windows, 1.19 ms with 1 / 4): fewer
// gathers in flight per SM queue less in the LSU and L2 while the tile stores
// of the previous batch proceed.
#ifndef LIFE_WS_FAST_BLOCKS
#define LIFE_WS_FAST_BLOCKS 1
#endif
constexpr int kFastBlocks = LIFE_WS_FAST_BLOCKS;  // 128-entry blocks per gather batch
// WC producers: 128-entry blocks loaded per scatter batch (1: C2 WC 0.937 ->
// 0.890 ms vs 4; fewer reductions in flight queue less in L2)
#ifndef LIFE_WC_BATCH
#define LIFE_WC_BATCH 1
#endif
#ifndef LIFE_WC_ATOMS
#define LIFE_WC_ATOMS 4
#endif
constexpr int kWcAtoms = LIFE_WC_ATOMS;  // atoms per WC consumer iteration
#ifndef LIFE_WS_SLOW_ROUNDS
#define LIFE_WS_SLOW_ROUNDS 4
#endif
constexpr int kSlowRounds = LIFE_WS_SLOW_ROUNDS;  // repeat windows per gather batch

template <bool STAGED>
__device__ __forceinline__ unsigned build_pair(float *C, const float *__restrict__ w,
                                               const Seg &S, const View &V, int junk,
                                               int lane)
{
    WS_T0(t_fast);
    float4 *Z = reinterpret_cast<float4 *>(C);
#pragma unroll
    for (int i = 0; i < kTPP * kWsCells / 4 / 32; ++i) Z[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    unsigned zeros = 0;
    const uint32_t nf = S.q0 - S.p0, n = S.p1 - S.p0;
    const int nb = (int)((nf + 127u) / 128u), nw = (int)((n - nf + 31u) / 32u);
    float ws[kSlowRounds];
    auto gather_slow = [&](int r0) {
#pragma unroll
        for (int r = 0; r < kSlowRounds; ++r) {
            const uint32_t k = nf + 32u * (uint32_t)(r0 + r) + (uint32_t)lane;
            ws[r] = 0.f;
            if (r0 + r < nw && k < n) ws[r] = gather_w(w, ldv<STAGED>(V.f + k));
        }
    };
    for (int b0 = 0; b0 < nb || (b0 == 0 && nw > 0); b0 += kFastBlocks) {
        float wf[kFastBlocks][4];
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) {
            const uint32_t k = 128u * (uint32_t)(b0 + j) + 4u * (uint32_t)lane;
            if (b0 + j < nb && k < nf) {
                const uint4 f = ldv<STAGED>(reinterpret_cast<const uint4 *>(V.f + k));
                wf[j][0] = gather_w(w, f.x);
                wf[j][1] = gather_w(w, f.y);
                wf[j][2] = gather_w(w, f.z);
                wf[j][3] = gather_w(w, f.w);
            }
        }
        if (b0 == 0) gather_slow(0);
#pragma unroll
        for (int j = 0; j < kFastBlocks; ++j) {
            const uint32_t k = 128u * (uint32_t)(b0 + j) + 4u * (uint32_t)lane;
            if (b0 + j < nb && k < nf) {
                const uint4 c4 = ldv<STAGED>(reinterpret_cast<const uint4 *>(V.cr + k));
                const float4 v4 = ldv<STAGED>(reinterpret_cast<const float4 *>(V.v + k));
                const uint32_t cr[4] = {c4.x, c4.y, c4.z, c4.w};
                const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    // branch-free: pad entries store into the warp's junk word
                    const bool ok = !(cr[e] & kPadBit);
                    const float sv = __fmul_rn(wf[j][e], v[e]);
                    zeros += (ok && sv == 0.f) ? 1u : 0u;
                    C[ok ? (int)(cr[e] & kCellMask) : junk] = sv;
                }
            }
        }
    }
    __syncwarp();
    if (lane == 0) WS_ACC(6, t_fast);
    WS_T0(t_slow);
    for (int r0 = 0; r0 < nw; r0 += kSlowRounds) {
        if (r0) gather_slow(r0);
        if (LIFE_WS_ORDERED == 2) {
            // level-batched, kLevelBatch windows at a time: within one rank
            // level all cells are distinct, so each level's read-modify-
            // writes are issued together (loads, then stores) and levels
            // follow in rank order -- the same per-cell summation order as
            // the window-by-window pass, bitwise
            constexpr int kLevelBatch = 4;
#pragma unroll
            for (int b = 0; b < kSlowRounds; b += kLevelBatch) {
                if (r0 + b >= nw) break;  // warp-uniform
                uint32_t cell[kLevelBatch], rank[kLevelBatch];
                float sv[kLevelBatch];
                uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
                for (int r = 0; r < kLevelBatch; ++r) {
                    const uint32_t k = nf + 32u * (uint32_t)(r0 + b + r) + (uint32_t)lane;
                    const bool in = r0 + b + r < nw && k < n;
                    const uint32_t cr = in ? ldv<STAGED>(V.cr + k) : kPadBit;
                    const bool ok = !(cr & kPadBit);
                    sv[r] = ok ? __fmul_rn(ws[b + r], ldv<STAGED>(V.v + k)) : 0.f;
                    zeros += (ok && sv[r] == 0.f) ? 1u : 0u;
                    cell[r] = cr & kCellMask;
                    rank[r] = ok ? (cr >> kWsCellBits) & kRankMask : 0xFFFFFFFFu;
                    if (ok) {
                        lo = min(lo, rank[r]);
                        hi = max(hi, rank[r]);
                    }
                }
                lo = __reduce_min_sync(0xffffffffu, lo);
                hi = __reduce_max_sync(0xffffffffu, hi);
                for (uint32_t rr = lo; rr <= hi && lo != 0xFFFFFFFFu; ++rr) {
                    float cv[kLevelBatch];
#pragma unroll
                    for (int r = 0; r < kLevelBatch; ++r) cv[r] = rank[r] == rr ? C[cell[r]] : 0.f;
#pragma unroll
                    for (int r = 0; r < kLevelBatch; ++r)
                        if (rank[r] == rr) C[cell[r]] = cv[r] + sv[r];
                    __syncwarp();
                }
            }
            continue;
        }
#pragma unroll
        for (int r = 0; r < kSlowRounds; ++r) {
            if (r0 + r >= nw) break;  // warp-uniform
            const uint32_t k = nf + 32u * (uint32_t)(r0 + r) + (uint32_t)lane;
            const uint32_t cr = k < n ? ldv<STAGED>(V.cr + k) : kPadBit;
            const bool ok = !(cr & kPadBit);
            const float sv = ok ? __fmul_rn(ws[r], ldv<STAGED>(V.v + k)) : 0.f;
            zeros += (ok && sv == 0.f) ? 1u : 0u;
            const uint32_t cell = cr & kCellMask;
            if (!LIFE_WS_ORDERED) {
                if (ok) ws_red_add(C + cell, sv);
            } else if (!__any_sync(0xffffffffu, ok && (cr & kMixedBit))) {
                if (ok) C[cell] += sv;
            } else {
                const uint32_t rank = (cr >> kWsCellBits) & kRankMask;
                const uint32_t rmin = __reduce_min_sync(0xffffffffu, ok ? rank : 0xFFFFFFFFu);
                const uint32_t rmax = __reduce_max_sync(0xffffffffu, ok ? rank : 0u);
                for (uint32_t rr = rmin; rr <= rmax; ++rr) {
                    if (ok && rank == rr) C[cell] += sv;
                    __syncwarp();
                }
            }
            if (LIFE_WS_ORDERED) __syncwarp();
        }
    }
    __syncwarp();
    if (lane == 0) WS_ACC(7, t_slow);
    return zeros;
}

// ---- staged, pipelined producer ---------------------------------------------
// The w[f] gathers of step k+1 are issued during step k as 4-byte cp.async
// copies (LDGSTS) that overwrite the slot's fascicle array in place with the
// gathered weights, so the L2 round trips of the gathers (bounded by the L2's
// random-sector rate, ~1 per cycle per SM) overlap the tile build of step k
// instead of stalling it.  Each lane gathers exactly the entries it later
// reads (4 per 128-entry block in the rank-0 region, 1 per 32-entry window
// after it), so cp.async.wait_group alone makes its values visible.
__device__ __forceinline__ void cp_async4(void *dst, const void *src, uint64_t pol)
{
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smaddr(dst)),
                 "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void gather_to_slot(const Seg &S, const View &V,
                                               const float *__restrict__ w, int lane)
{
    const uint64_t pol = policy_keep();
    uint32_t *F = const_cast<uint32_t *>(V.f);
    const uint32_t nf = S.q0 - S.p0, n = S.p1 - S.p0;
    if (!(c_ws_flags & 4)) {
        for (uint32_t k = 4u * (uint32_t)lane; k < nf; k += 128u) {
            const uint4 f = *reinterpret_cast<const uint4 *>(F + k);
            if (f.x != kSent) cp_async4(F + k, w + f.x, pol);
            if (f.y != kSent) cp_async4(F + k + 1, w + f.y, pol);
            if (f.z != kSent) cp_async4(F + k + 2, w + f.z, pol);
            if (f.w != kSent) cp_async4(F + k + 3, w + f.w, pol);
        }
        for (uint32_t k = nf + (uint32_t)lane; k < n; k += 32u) {
            const uint32_t f = F[k];
            if (f != kSent) cp_async4(F + k, w + f, pol);
        }
    }
    cp_async_commit();
}

// zero + rank-0 stores, from a slot whose fascicle array holds the gathered w
__device__ __forceinline__ unsigned build_fast_staged(float *C, const Seg &S, const View &V,
                                                      int junk, int lane)
{
    float4 *Z = reinterpret_cast<float4 *>(C);
#pragma unroll
    for (int i = 0; i < kTPP * kWsCells / 4 / 32; ++i) Z[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    unsigned zeros = 0;
    const uint32_t nf = S.q0 - S.p0;
    const float *W = reinterpret_cast<const float *>(V.f);
#pragma unroll 2
    for (uint32_t k = 4u * (uint32_t)lane; k < nf; k += 128u) {
        const uint4 c4 = *reinterpret_cast<const uint4 *>(V.cr + k);
        const float4 w4 = *reinterpret_cast<const float4 *>(W + k);
        const float4 v4 = *reinterpret_cast<const float4 *>(V.v + k);
        const uint32_t cr[4] = {c4.x, c4.y, c4.z, c4.w};
        const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool ok = !(cr[e] & kPadBit);
            const float sv = __fmul_rn((c_ws_flags & 4) ? 1.f : wv[e], v[e]);
            zeros += (ok && sv == 0.f) ? 1u : 0u;
            C[ok ? (int)(cr[e] & kCellMask) : junk] = sv;
        }
    }
    __syncwarp();
    return zeros;
}

// rank>=1 windows in order (after every rank-0 store of the tile)
__device__ __forceinline__ unsigned build_slow_staged(float *C, const Seg &S, const View &V,
                                                      int lane)
{
    unsigned zeros = 0;
    const uint32_t nf = S.q0 - S.p0, n = S.p1 - S.p0;
    const float *W = reinterpret_cast<const float *>(V.f);
    for (uint32_t base = nf; base < n; base += 32u) {
        const uint32_t k = base + (uint32_t)lane;
        const uint32_t cr = k < n ? V.cr[k] : kPadBit;
        const bool ok = !(cr & kPadBit);
        const float sv = ok ? __fmul_rn((c_ws_flags & 4) ? 1.f : W[k], V.v[k]) : 0.f;
        zeros += (ok && sv == 0.f) ? 1u : 0u;
        const uint32_t cell = cr & kCellMask;
        if (!LIFE_WS_ORDERED) {
            if (ok) ws_red_add(C + cell, sv);
        } else if (!__any_sync(0xffffffffu, ok && (cr & kMixedBit))) {
            if (ok) C[cell] += sv;
        } else {
            const uint32_t rank = (cr >> kWsCellBits) & kRankMask;
            const uint32_t rmin = __reduce_min_sync(0xffffffffu, ok ? rank : 0xFFFFFFFFu);
            const uint32_t rmax = __reduce_max_sync(0xffffffffu, ok ? rank : 0u);
            for (uint32_t rr = rmin; rr <= rmax; ++rr) {
                if (ok && rank == rr) C[cell] += sv;
                __syncwarp();
            }
        }
        if (LIFE_WS_ORDERED) __syncwarp();
    }
    __syncwarp();
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
    __shared__ float junkbuf[kWsProd * 32];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kWsCA * 8 * DPL;  // nt_pad == 8 * DPL
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    float *Dbuf = sm;
    float *Cbuf = sm + 2 * chunk_floats;
    float *slots = Cbuf + 2 * kWsCons * kWsCells;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    // DSC keeps whole CTA tiles per CTA (round robin): a voxel's chunks are
    // then always summed in one FMA chain, so results do not depend on the
    // grid or on multi-GPU sharding (bitwise)
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
        if constexpr (kSplitRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegCons));
        const int vg = lane >> 3, dg = lane & 7;
        const bool accumulate = flags & LIFE_ACCUMULATE;
        const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
        int k = 0;
        for (int ct = blockIdx.x; ct < n_ct; ct += gridDim.x) {
            const int cb = 0, ce = A.nch;
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
            for (int c = cb; c < ce; ++c, ++k) {
                const int s = k & 1;
                WS_T0(t_f);
                bar_wait(&full[s], (k >> 1) & 1);
                if (lane == 0) WS_ACC(4, t_f);
                WS_T0(t_c);
                if (tile_ok && c_ws_isolate != 1) {
                    const float *C = Cbuf + (s * kWsCons + warp) * kWsCells + vg * 8;
                    const float *D = Dbuf + s * chunk_floats + dg * DPL;
#pragma unroll
                    for (int a = 0; a < kWsCA; ++a) {
                        const float4 c0 = *reinterpret_cast<const float4 *>(C + a * kWsTV);
                        const float4 c1 = *reinterpret_cast<const float4 *>(C + a * kWsTV + 4);
                        const unsigned long long cp[4] = {wpk(c0.x, c0.y), wpk(c0.z, c0.w),
                                                          wpk(c1.x, c1.y), wpk(c1.z, c1.w)};
                        // nt_pad == 8 * DPL (dispatch): a compile-time stride folds into LDS offsets
                        const float4 *d4 = reinterpret_cast<const float4 *>(D + a * (8 * DPL));
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
                if (lane == 0) WS_ACC(5, t_c);
                if (lane == 0) bar_arrive(&empty[s]);
            }
            // y epilogue over a value source get(vp, j) -> (voxel 2vp, 2vp+1) pair
            auto epilogue = [&](auto get) {
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
                            wupk(get(vp, j), o[0], o[1]);
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
            };
            if (tile_ok) epilogue([&](int vp, int j) { return acc[vp][j]; });
        }
    } else {
        // ===== producers: TMA for D and the coefficient segments, tile build =====
        if constexpr (kSplitRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProd));
        const int p = warp - kWsCons;
        // steps k (current), k+1, k+2, k+3 -- c fastest
        int ct0 = blockIdx.x, c0 = 0, ct1 = ct0, c1 = c0, ct2, c2, ct3, c3;
        step_next_rr(ct1, c1, A.nch);
        ct2 = ct1; c2 = c1;
        step_next_rr(ct2, c2, A.nch);
        ct3 = ct2; c3 = c2;
        step_next_rr(ct3, c3, A.nch);
        float *Cp = nullptr;
        auto tiles = [&](int s) { return Cbuf + (s * kWsCons + kTPP * p) * kWsCells; };
        auto junk_of = [&](int s) { return (int)(junkbuf + p * 32 + lane - tiles(s)); };
        (void)Cp;
        if constexpr (STAGED && !kCpAsyncGather) {
            // segment k+1 is staged while step k builds; w gathered in registers
            Seg cur{}, nxt{};
            if (total > 0) {
                cur = seg_of(A, ct0, c0, p);
                if (lane == 0) stage_issue(A, cur, slots, p, 0, &slotbar[p][0]);
            }
            if (total > 1) {
                nxt = seg_of(A, ct1, c1, p);
                prefetch_seg<STAGED>(A, nxt, lane);
            }
            for (int k = 0; k < total; ++k) {
                const int s = k & 1;
                Seg nn{};
                if (k + 2 < total) nn = seg_of(A, ct2, c2, p);
                if (k + 1 < total && lane == 0) stage_issue(A, nxt, slots, p, s ^ 1, &slotbar[p][s ^ 1]);
                WS_T0(t_e);
                if (k >= 2) bar_wait(&empty[s], ((k - 2) >> 1) & 1);
                if (lane == 0) WS_ACC(1, t_e);
                if (p == 0 && lane == 0)
                    tma_chunk(Dbuf + s * chunk_floats, A.D + (size_t)c0 * chunk_floats,
                              chunk_bytes, &full[s]);
                if (k + 2 < total) prefetch_seg<STAGED>(A, nn, lane);
                WS_T0(t_s);
                bar_wait(&slotbar[p][s], (k >> 1) & 1);
                if (lane == 0) WS_ACC(0, t_s);
                WS_T0(t_b);
                if (c_ws_isolate != 2)
                    skipped += build_pair<true>(tiles(s), w, cur, slot_view(slots, p, s), junk_of(s),
                                                lane);
                __syncwarp();
                if (lane == 0) WS_ACC(2, t_b);
                if (lane == 0) bar_arrive(&full[s]);
                cur = nxt;
                nxt = nn;
                ct0 = ct1; c0 = c1;
                ct1 = ct2; c1 = c2;
                ct2 = ct3; c2 = c3;
                step_next_rr(ct3, c3, A.nch);
            }
        } else if constexpr (STAGED) {
            // segment k+1 is staged and its w gathered while step k builds;
            // segment k+2 is copied into slot k%2 once step k is done with it
            Seg cur{}, nxt{}, nn{};
            if (total > 0) {
                cur = seg_of(A, ct0, c0, p);
                if (lane == 0) stage_issue(A, cur, slots, p, 0, &slotbar[p][0]);
            }
            if (total > 1) {
                nxt = seg_of(A, ct1, c1, p);
                if (lane == 0) stage_issue(A, nxt, slots, p, 1, &slotbar[p][1]);
            }
            if (total > 2) {
                nn = seg_of(A, ct2, c2, p);
                prefetch_seg<STAGED>(A, nn, lane);
            }
            if (total > 0) {
                bar_wait(&slotbar[p][0], 0);
                gather_to_slot(cur, slot_view(slots, p, 0), w, lane);
            }
            for (int k = 0; k < total; ++k) {
                const int s = k & 1;
                Seg n3{};
                if (k + 3 < total) n3 = seg_of(A, ct3, c3, p);
                WS_T0(t_e);
                if (k >= 2) bar_wait(&empty[s], ((k - 2) >> 1) & 1);
                if (lane == 0) WS_ACC(1, t_e);
                if (p == 0 && lane == 0)
                    tma_chunk(Dbuf + s * chunk_floats, A.D + (size_t)c0 * chunk_floats,
                              chunk_bytes, &full[s]);
                WS_T0(t_s);
                cp_async_wait_all();
                __syncwarp();
                if (lane == 0) WS_ACC(0, t_s);
                WS_T0(t_b);
                const View V = slot_view(slots, p, s);
                if (c_ws_isolate != 2) skipped += build_fast_staged(tiles(s), cur, V, junk_of(s), lane);
                if (k + 1 < total) {
                    bar_wait(&slotbar[p][s ^ 1], ((k + 1) >> 1) & 1);
                    gather_to_slot(nxt, slot_view(slots, p, s ^ 1), w, lane);
                }
                if (c_ws_isolate != 2) skipped += build_slow_staged(tiles(s), cur, V, lane);
                __syncwarp();
                if (lane == 0) WS_ACC(2, t_b);
                if (lane == 0) bar_arrive(&full[s]);
                // slot s is free: stage segment k+2 into it
                if (k + 2 < total && lane == 0) stage_issue(A, nn, slots, p, s, &slotbar[p][s]);
                if (k + 3 < total) prefetch_seg<STAGED>(A, n3, lane);
                cur = nxt;
                nxt = nn;
                nn = n3;
                ct0 = ct1; c0 = c1;
                ct1 = ct2; c1 = c2;
                ct2 = ct3; c2 = c3;
                step_next_rr(ct3, c3, A.nch);
            }
        } else {
            // fallback: segments straight from global memory, gathers in registers
            Seg cur{}, nxt{};
            if (total > 0) cur = seg_of(A, ct0, c0, p);
            if (total > 1) {
                nxt = seg_of(A, ct1, c1, p);
                prefetch_seg<STAGED>(A, nxt, lane);
            }
            for (int k = 0; k < total; ++k) {
                const int s = k & 1;
                Seg nn{};
                if (k + 2 < total) nn = seg_of(A, ct2, c2, p);
                if (k >= 2) bar_wait(&empty[s], ((k - 2) >> 1) & 1);
                if (p == 0 && lane == 0)
                    tma_chunk(Dbuf + s * chunk_floats, A.D + (size_t)c0 * chunk_floats,
                              chunk_bytes, &full[s]);
                if (k + 2 < total) prefetch_seg<STAGED>(A, nn, lane);
                if (c_ws_isolate != 2)
                    skipped += build_pair<false>(tiles(s), w, cur, global_view(A, cur), junk_of(s),
                                                 lane);
                __syncwarp();
                if (lane == 0) bar_arrive(&full[s]);
                cur = nxt;
                nxt = nn;
                ct0 = ct1; c0 = c1;
                ct1 = ct2; c1 = c2;
                ct2 = ct3; c2 = c3;
                step_next_rr(ct3, c3, A.nch);
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

// value * Z[cell] -> fixed-point fascicle sum (pad entries skipped)
__device__ __forceinline__ void wc_scatter1(uint32_t cr, uint32_t f, float v, const float *Z,
                                            const WsFix &fx, bool f32_scale, float scalef,
                                            double scale)
{
    if (cr & kPadBit) return;
    const float z = Z[cr & kCellMask] * v;
    const long long qv = f32_scale ? __float2ll_rn(z * scalef) : __double2ll_rn((double)z * scale);
    red_keep(fx.wfix + f, static_cast<unsigned long long>(qv), policy_keep());
}

// ---- WC producers: 4 warps, each scattering two adjacent tiles per step ----
// The per-tile segments of tiles 2p and 2p+1 are adjacent in the layout, so a
// WC producer warp stages one contiguous range [p0, p1) with the boundary
// between its tiles at q0 (reusing Seg; the rank split is irrelevant to WC).
constexpr int kWcProd = 4;
constexpr int kWcWarps = kWsCons + kWcProd;
constexpr int kWcThreads = kWcWarps * 32;
constexpr int kWcSlot = 2 * kWsSlot;
static_assert(kWsProd == 8, "WC pairs up the per-tile segments of the 8-producer layout");

__device__ __forceinline__ Seg wc_seg_of(const WsArgs &A, int ct, int c, int p)
{
    const size_t t = ((size_t)ct * A.nch + c) * kWsProd + 2 * p;
    Seg S;
    S.p0 = __ldg(A.tptr + t);
    S.q0 = __ldg(A.tptr + t + 1);
    S.p1 = __ldg(A.tptr + t + 2);
    return S;
}

__device__ __forceinline__ View wc_slot_view(float *slots, int p, int s)
{
    uint32_t *base = reinterpret_cast<uint32_t *>(slots) + (size_t)(p * 2 + s) * 3 * kWcSlot;
    return View{base, base + kWcSlot, reinterpret_cast<const float *>(base + 2 * kWcSlot)};
}

__device__ __forceinline__ void wc_stage_issue(const WsArgs &A, const Seg &S, float *slots, int p,
                                               int s, uint64_t *bar)
{
    const unsigned n = S.p1 - S.p0, bytes = n * 4u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bar_arrive_tx(bar, 3u * bytes);
    if (n) {
        const View D = wc_slot_view(slots, p, s);
        bulk_g2s_stream((void *)D.cr, A.cr + S.p0, bytes, bar);
        bulk_g2s_stream((void *)D.f, A.fiber + S.p0, bytes, bar);
        bulk_g2s_stream((void *)D.v, A.val + S.p0, bytes, bar);
    }
}

template <int DPL, bool STAGED>
__global__ void __launch_bounds__(kWcThreads, 1)
    k_wc_ws(const WsArgs A, const float *__restrict__ y, const WsFix fx, const CallHooks hooks)
{
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t dfull[2], dempty[2], zfull[2], zempty[2], slotbar[kWcProd][2];
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    const int chunk_floats = kWsCA * A.nt_pad;
    const unsigned chunk_bytes = (unsigned)chunk_floats * 4u;
    float *Dbuf = sm;
    float *Zbuf = sm + 2 * chunk_floats;
    float *slots = Zbuf + 2 * kWsCons * kWsCells;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    int s_begin, s_end;
    step_range(n_ct, A.nch, s_begin, s_end);
    const int total = s_end - s_begin;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&dfull[s], 1);
            bar_init(&dempty[s], kWsCons);
            bar_init(&zfull[s], kWsCons);
            bar_init(&zempty[s], kWcProd);
            for (int p = 0; p < kWcProd; ++p) bar_init(&slotbar[p][s], 1);
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
        for (int st = s_begin; st < s_end;) {
            const int ct = st / A.nch, cb = st % A.nch;
            const int ce = min(A.nch, cb + (s_end - st));
            st += ce - cb;
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
            for (int c = cb; c < ce; ++c, ++k) {
                const int s = k & 1;
                bar_wait(&dfull[s], (k >> 1) & 1);
                if (k >= 2) bar_wait(&zempty[s], ((k - 2) >> 1) & 1);
                if (tile_ok && c_ws_isolate != 1) {
                    float *Z = Zbuf + (s * kWsCons + warp) * kWsCells + vg * 8 + dg;
                    const float *D = Dbuf + s * chunk_floats + dg * DPL;
#pragma unroll 1
                    for (int a0 = 0; a0 < kWsCA; a0 += kWcAtoms) {
                        // kWcAtoms independent accumulator sets keep the FMA
                        // pipe fed while earlier butterflies are in flight
                        unsigned long long pp[kWcAtoms][4];
#pragma unroll
                        for (int aa = 0; aa < kWcAtoms; ++aa)
#pragma unroll
                            for (int vp = 0; vp < 4; ++vp) pp[aa][vp] = 0ull;
#pragma unroll
                        for (int i = 0; i < DPL / 4; ++i) {
#pragma unroll
                            for (int aa = 0; aa < kWcAtoms; ++aa) {
                                const float4 t = reinterpret_cast<const float4 *>(D + (a0 + aa) * (8 * DPL))[i];
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
                        for (int aa = 0; aa < kWcAtoms; ++aa) {
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
        int ct0 = s_begin / A.nch, c0 = s_begin % A.nch, ct1 = ct0, c1 = c0, ct2, c2;
        if (p == 0 && lane == 0 && total > 0)
            tma_chunk(Dbuf, A.D + (size_t)c0 * chunk_floats, chunk_bytes, &dfull[0]);
        step_next(ct1, c1, A.nch);
        ct2 = ct1; c2 = c1;
        step_next(ct2, c2, A.nch);
        Seg cur{}, nxt{};
        if (total > 0) {
            cur = wc_seg_of(A, ct0, c0, p);
            if (STAGED && lane == 0) wc_stage_issue(A, cur, slots, p, 0, &slotbar[p][0]);
        }
        if (total > 1) {
            nxt = wc_seg_of(A, ct1, c1, p);
            prefetch_seg<STAGED>(A, nxt, lane);
        }
        for (int k = 0; k < total; ++k) {
            const int s = k & 1;
            if (p == 0 && lane == 0 && k + 1 < total) {
                const int s1 = (k + 1) & 1;
                if (k + 1 >= 2) bar_wait(&dempty[s1], ((k - 1) >> 1) & 1);
                tma_chunk(Dbuf + s1 * chunk_floats, A.D + (size_t)c1 * chunk_floats, chunk_bytes,
                          &dfull[s1]);
            }
            __syncwarp();
            Seg nn{};
            if (k + 2 < total) nn = wc_seg_of(A, ct2, c2, p);
            if (STAGED && k + 1 < total && lane == 0)
                wc_stage_issue(A, nxt, slots, p, s ^ 1, &slotbar[p][s ^ 1]);
            if (k + 2 < total) prefetch_seg<STAGED>(A, nn, lane);
            if (STAGED) bar_wait(&slotbar[p][s], (k >> 1) & 1);
            bar_wait(&zfull[s], (k >> 1) & 1);
            const float *Z = Zbuf + (s * kWsCons + 2 * p) * kWsCells;
            const View V = STAGED ? wc_slot_view(slots, p, s) : global_view(A, cur);
            const uint32_t mid = cur.q0 - cur.p0;  // tile 2p+1 starts here
            const uint32_t n = (c_ws_isolate == 2) ? 0u : cur.p1 - cur.p0;
            // 4 entries per lane, 4 blocks of 128 per round: loads first
            constexpr int kB = LIFE_WC_BATCH;
            for (uint32_t base = 0; base < n; base += 128u * kB) {
                uint4 cr[kB], f[kB];
                float4 v[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint32_t kk = base + 128u * j + 4u * (uint32_t)lane;
                    if (kk < n) {
                        cr[j] = ldv<STAGED>(reinterpret_cast<const uint4 *>(V.cr + kk));
                        f[j] = ldv<STAGED>(reinterpret_cast<const uint4 *>(V.f + kk));
                        v[j] = ldv<STAGED>(reinterpret_cast<const float4 *>(V.v + kk));
                    } else {
                        cr[j] = make_uint4(kPadBit, kPadBit, kPadBit, kPadBit);
                        f[j] = make_uint4(0u, 0u, 0u, 0u);
                        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    // a 4-entry group never straddles the 4-aligned tile boundary
                    const uint32_t kk = base + 128u * j + 4u * (uint32_t)lane;
                    const float *Zt = Z + (kk >= mid ? kWsCells : 0);
                    wc_scatter1(cr[j].x, f[j].x, v[j].x, Zt, fx, f32_scale, scalef, scale);
                    wc_scatter1(cr[j].y, f[j].y, v[j].y, Zt, fx, f32_scale, scalef, scale);
                    wc_scatter1(cr[j].z, f[j].z, v[j].z, Zt, fx, f32_scale, scalef, scale);
                    wc_scatter1(cr[j].w, f[j].w, v[j].w, Zt, fx, f32_scale, scalef, scale);
                }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&zempty[s]);
            cur = nxt;
            nxt = nn;
            ct0 = ct1; c0 = c1;
            ct1 = ct2; c1 = c2;
            step_next(ct2, c2, A.nch);
        }
    }
}

// ---------------------------------------------------------------------------
// WC with Z = Y . D^T on the tensor cores (k_wc_tc)
// ---------------------------------------------------------------------------
// Same layout, schedule and RED-scatter producers as k_wc_ws; the 8 FFMA
// consumer warps are replaced by tcgen05:
//   warps 0-3  RED producers (unchanged code path, segments read from global
//              memory with an L2 prefetch one step ahead).
//   warps 4-7  "YZ": at each CTA tile, y rows (thread = voxel = TMEM lane,
//              two 128-voxel halves) are split into tf32 hi/lo and stored in
//              TMEM (A operand); per step the Z accumulators are read back
//              from TMEM and stored to shared memory as the 32 x 32 tiles the
//              producers expect (cell = atom * 32 + voxel slot).
//   warp 8     MMA issuer: per half, 3xTF32 over K = directions (M = 128
//              voxels, N = 32 atoms), A from TMEM, B = the pre-split,
//              pre-swizzled dictionary chunk (K-major, 3 blocks of 32
//              directions) staged by producer 0's bulk copy.
// TMEM (512 columns): Y half h at h*2*ntp (hi) and h*2*ntp + ntp (lo), Z
// buffers at 4*ntp + s*64 + h*32.  Z accumulates 3*ntp/8 MMAs (36 at 96
// directions: ~2e-6 relative, tools/ubench/tc_probe.cu).
constexpr int kWtYZ = 4;
constexpr int kWtMma = kWcProd + kWtYZ;     // warp 8
constexpr int kWtWarps = kWtMma + 1;
constexpr int kWtThreads = kWtWarps * 32;

struct WtArgs {
    const float *B;   // [nch][hi|lo][nkb][32 atoms][32 dirs] swizzled
    int nkb;          // direction blocks of 32 (ntp = 32 * nkb <= 96)
};

// Z is single-buffered in shared memory (the TMEM accumulators are double
// buffered) so the producers' TMA-staged segment slots still fit.
template <bool STAGED>
__global__ void __launch_bounds__(kWtThreads, 1)
    k_wc_tc(const WsArgs A, const WtArgs T, const float *__restrict__ y, const WsFix fx, const CallHooks hooks)
{
    extern __shared__ __align__(1024) unsigned char wt_raw[];
    __shared__ __align__(8) uint64_t bfull[2], bempty[2], zfull[2], zempty[2], accfull[2], accempty[2];
    __shared__ __align__(8) uint64_t yready, yfree, slotbar[kWcProd][2];
    __shared__ uint32_t tmem_base;
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    unsigned char *sm = (unsigned char *)(((uintptr_t)wt_raw + 1023) & ~(uintptr_t)1023);
    const int ntp = 32 * T.nkb;
    const unsigned bbytes = 2u * (unsigned)T.nkb * 4096u;  // hi | lo
    unsigned char *Bbuf = sm;                               // 2 stages
    float *Zbuf = reinterpret_cast<float *>(sm + 2 * bbytes);  // 1 stage
    float *slots = Zbuf + kWsCons * kWsCells;
    const int n_ct = (A.n_tiles + kWsCons - 1) / kWsCons;
    int s_begin, s_end;
    step_range(n_ct, A.nch, s_begin, s_end);
    const int total = s_end - s_begin;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&bfull[s], 1);
            bar_init(&bempty[s], 1);
            bar_init(&zfull[s], kWtYZ);
            bar_init(&zempty[s], kWcProd);
            bar_init(&accfull[s], 1);
            bar_init(&accempty[s], kWtYZ);
        }
        bar_init(&yready, kWtYZ);
        bar_init(&yfree, 1);
        for (int p = 0; p < kWcProd; ++p)
            for (int s = 0; s < 2; ++s) bar_init(&slotbar[p][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kWtMma) tcg::alloc(&tmem_base, 512);
    tcg::fence_before();
    __syncthreads();
    tcg::fence_after();
    const uint32_t tmem = tmem_base;

    if (warp < kWcProd) {
        // ===== producers: dictionary chunks (bulk copy), RED scatter =====
        const int p = warp;
        const int ex = fix_exponent(fx, A.nt);
        const double scale = ldexp(1.0, ex);
        const bool f32_scale = ex >= -120 && ex <= 120;
        const float scalef = f32_scale ? ldexpf(1.f, ex) : 1.f;
        int ct0 = s_begin / A.nch, c0 = s_begin % A.nch, ct1 = ct0, c1 = c0, ct2, c2;
        if (p == 0 && lane == 0 && total > 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_arrive_tx(&bfull[0], bbytes);
            bulk_g2s(Bbuf, T.B + (size_t)c0 * (bbytes / 4), bbytes, &bfull[0]);
        }
        step_next(ct1, c1, A.nch);
        ct2 = ct1; c2 = c1;
        step_next(ct2, c2, A.nch);
        Seg cur{}, nxt{};
        if (total > 0) {
            cur = wc_seg_of(A, ct0, c0, p);
            if (STAGED && lane == 0) wc_stage_issue(A, cur, slots, p, 0, &slotbar[p][0]);
        }
        if (total > 1) {
            nxt = wc_seg_of(A, ct1, c1, p);
            prefetch_seg<STAGED>(A, nxt, lane);
        }
        for (int k = 0; k < total; ++k) {
            const int s = k & 1;
            if (p == 0 && lane == 0 && k + 1 < total) {
                const int s1 = (k + 1) & 1;
                if (k + 1 >= 2) bar_wait(&bempty[s1], ((k - 1) >> 1) & 1);
                bar_arrive_tx(&bfull[s1], bbytes);
                bulk_g2s(Bbuf + (size_t)s1 * bbytes, T.B + (size_t)c1 * (bbytes / 4), bbytes, &bfull[s1]);
            }
            __syncwarp();
            Seg nn{};
            if (k + 2 < total) nn = wc_seg_of(A, ct2, c2, p);
            if (STAGED && k + 1 < total && lane == 0)
                wc_stage_issue(A, nxt, slots, p, s ^ 1, &slotbar[p][s ^ 1]);
            if (k + 2 < total) prefetch_seg<STAGED>(A, nn, lane);
            if (STAGED) bar_wait(&slotbar[p][s], (k >> 1) & 1);
            bar_wait(&zfull[0], k & 1);
            const float *Z = Zbuf + (2 * p) * kWsCells;
            const View V = STAGED ? wc_slot_view(slots, p, s) : global_view(A, cur);
            const uint32_t mid = cur.q0 - cur.p0;
            const uint32_t n = cur.p1 - cur.p0;
            constexpr int kB = LIFE_WC_BATCH;
            for (uint32_t base = 0; base < n; base += 128u * kB) {
                uint4 cr[kB], f[kB];
                float4 v[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint32_t kk = base + 128u * j + 4u * (uint32_t)lane;
                    if (kk < n) {
                        cr[j] = ldv<STAGED>(reinterpret_cast<const uint4 *>(V.cr + kk));
                        f[j] = ldv<STAGED>(reinterpret_cast<const uint4 *>(V.f + kk));
                        v[j] = ldv<STAGED>(reinterpret_cast<const float4 *>(V.v + kk));
                    } else {
                        cr[j] = make_uint4(kPadBit, kPadBit, kPadBit, kPadBit);
                        f[j] = make_uint4(0u, 0u, 0u, 0u);
                        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    const uint32_t kk = base + 128u * j + 4u * (uint32_t)lane;
                    const float *Zt = Z + (kk >= mid ? kWsCells : 0);
                    wc_scatter1(cr[j].x, f[j].x, v[j].x, Zt, fx, f32_scale, scalef, scale);
                    wc_scatter1(cr[j].y, f[j].y, v[j].y, Zt, fx, f32_scale, scalef, scale);
                    wc_scatter1(cr[j].z, f[j].z, v[j].z, Zt, fx, f32_scale, scalef, scale);
                    wc_scatter1(cr[j].w, f[j].w, v[j].w, Zt, fx, f32_scale, scalef, scale);
                }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&zempty[0]);
            cur = nxt;
            nxt = nn;
            ct0 = ct1; c0 = c1;
            ct1 = ct2; c1 = c2;
            step_next(ct2, c2, A.nch);
        }
    } else if (warp < kWtMma) {
        // ===== YZ warps: y -> TMEM (A operand), Z TMEM -> shared =====
        const int q = warp & 3;  // TMEM lane quarter
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        int k = 0, tiles = 0;
        for (int st = s_begin; st < s_end;) {
            const int ct = st / A.nch, cb = st % A.nch;
            const int ce = min(A.nch, cb + (s_end - st));
            st += ce - cb;
            if (tiles > 0) bar_wait(&yfree, (tiles - 1) & 1);
            tcg::fence_after();
            // this thread's two voxel rows (one per 128-voxel half)
            const float *yr[2];
            bool yok[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int row = h * 128 + q * 32 + lane;
                const int tile = ct * kWsCons + row / kWsTV;
                const int voxel = tile < A.n_tiles ? __ldg(A.slotv + (size_t)ct * (kWsCons * kWsTV) + row) : -1;
                yok[h] = voxel >= 0;
                yr[h] = y + (size_t)(voxel < 0 ? 0 : voxel) * A.nt;
            }
            const bool vec = (A.nt & 3) == 0;  // rows 16-byte aligned
#pragma unroll 1
            for (int kb = 0; kb < T.nkb; ++kb) {
                // both halves' 32 directions in flight together
                float x[2][32];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (vec) {
#pragma unroll
                        for (int i4 = 0; i4 < 8; ++i4) {
                            const int t = kb * 32 + 4 * i4;
                            const float4 v = (yok[h] && t < A.nt) ? __ldg(reinterpret_cast<const float4 *>(yr[h] + t))
                                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
                            x[h][4 * i4] = v.x;
                            x[h][4 * i4 + 1] = v.y;
                            x[h][4 * i4 + 2] = v.z;
                            x[h][4 * i4 + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int t = kb * 32 + i;
                            x[h][i] = (yok[h] && t < A.nt) ? __ldg(yr[h] + t) : 0.f;
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t hv[32], lv[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const uint32_t hb = tcg::hi_bits(__float_as_uint(x[h][i]));
                        hv[i] = hb;
                        lv[i] = __float_as_uint(x[h][i] - __uint_as_float(hb));
                    }
                    tcg::st32(tmem + lane_base + (uint32_t)(h * 2 * ntp + kb * 32), hv);
                    tcg::st32(tmem + lane_base + (uint32_t)(h * 2 * ntp + ntp + kb * 32), lv);
                }
            }
            tcg::wait_st();
            tcg::fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&yready);
            ++tiles;
            for (int c = cb; c < ce; ++c, ++k) {
                const int s = k & 1;
                bar_wait(&accfull[s], (k >> 1) & 1);
                if (k >= 1) bar_wait(&zempty[0], (k - 1) & 1);
                tcg::fence_after();
                float *Zs = Zbuf;
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    uint32_t zr[32];
                    tcg::ld32(tmem + lane_base + (uint32_t)(4 * ntp + s * 64 + h * 32), zr);
                    // tile h*4 + q, cell = atom * 32 + voxel slot (= lane)
                    float *Zt = Zs + (h * 4 + q) * kWsCells + lane;
#pragma unroll
                    for (int a = 0; a < 32; ++a) Zt[a * kWsTV] = __uint_as_float(zr[a]);
                }
                tcg::fence_before();
                __syncwarp();
                if (lane == 0) {
                    bar_arrive(&accempty[s]);
                    bar_arrive(&zfull[0]);
                }
            }
        }
    } else {
        // ===== MMA issuer =====
        if (lane == 0) {
            const uint32_t id = tcg::idesc_tf32(128, 32);
            int k = 0, tiles = 0;
            for (int st = s_begin; st < s_end;) {
                const int cb = st % A.nch;
                const int ce = min(A.nch, cb + (s_end - st));
                st += ce - cb;
                bar_wait(&yready, tiles & 1);
                ++tiles;
                for (int c = cb; c < ce; ++c, ++k) {
                    const int s = k & 1;
                    bar_wait(&bfull[s], (k >> 1) & 1);
                    if (k >= 2) bar_wait(&accempty[s], ((k - 2) >> 1) & 1);
                    tcg::fence_after();
                    const uint32_t bs = tcg::sa(Bbuf + (size_t)s * bbytes);
                    const uint64_t bh = tcg::sdesc(bs), bl = tcg::sdesc(bs + (uint32_t)T.nkb * 4096u);
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t d = tmem + (uint32_t)(4 * ntp + s * 64 + h * 32);
                        const uint32_t ay = tmem + (uint32_t)(h * 2 * ntp);
#pragma unroll 1
                        for (int kk = 0; kk < ntp / 8; ++kk) {
                            const uint64_t o = (uint64_t)((((kk >> 2) * 4096) + (kk & 3) * 32) >> 4);
                            tcg::mma_ts(d, ay + 8u * kk, bh + o, id, kk != 0);
                            tcg::mma_ts(d, ay + (uint32_t)ntp + 8u * kk, bh + o, id, 1u);
                            tcg::mma_ts(d, ay + 8u * kk, bl + o, id, 1u);
                        }
                    }
                    tcg::commit(&bempty[s]);
                    tcg::commit(&accfull[s]);
                    if (c == ce - 1) tcg::commit(&yfree);
                }
            }
        }
        __syncwarp();
    }
    tcg::fence_before();
    __syncthreads();
    if (warp == kWtMma) {
        tcg::fence_after();
        tcg::dealloc(tmem, 512);
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
    k_wc_ws<DPL, STAGED><<<phi->d_blocks, kWcThreads, phi->d_smem, st>>>(A, y, fx, h);
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

size_t wc_tc_smem_bytes(int nkb, bool staged)
{
    return 1024 + 2 * (size_t)2 * nkb * 4096 + (size_t)kWsCons * kWsCells * 4 +
           (staged ? (size_t)kWcProd * 2 * 3 * kWcSlot * 4 : 0);
}

int launch_wc_ws(life_phi *phi, const FixParams &fx, const float *y, const CallHooks &h,
                 cudaStream_t st)
{
    if (phi->d_Bwc) {
        const bool staged = phi->d_staged && wc_tc_smem_bytes(phi->nt_pad / 32, true) <= 232448 - 2048;
        const size_t smem = wc_tc_smem_bytes(phi->nt_pad / 32, staged);
        WsArgs A{phi->d_cr, phi->d_fiber, phi->d_val, phi->d_tptr, phi->d_t1, phi->d_D,
                 phi->d_slotv, phi->nv, phi->nt, phi->nt_pad, phi->n_chunks, phi->n_tiles, phi->na};
        WtArgs T{phi->d_Bwc, phi->nt_pad / 32};
        if (staged) {
            LIFE_TRY(ensure_smem(k_wc_tc<true>, smem));
            k_wc_tc<true><<<phi->d_blocks, kWtThreads, smem, st>>>(A, T, y, fx, h);
        } else {
            LIFE_TRY(ensure_smem(k_wc_tc<false>, smem));
            k_wc_tc<false><<<phi->d_blocks, kWtThreads, smem, st>>>(A, T, y, fx, h);
        }
        LIFE_CHECK_LAUNCH();
        return LIFE_OK;
    }
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

// read and clear the cycle counters (8 x u64)
extern "C" LIFE_API int life_debug_ws_counters(unsigned long long *out)
{
    if (cudaDeviceSynchronize() != cudaSuccess) return 20;
    if (cudaMemcpyFromSymbol(out, life::g_ws_cyc, 8 * sizeof(unsigned long long)) != cudaSuccess) return 20;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(life::g_ws_cyc, z, sizeof(z)) == cudaSuccess ? 0 : 20;
}
#endif

namespace life {

int ws_warps() { return kWsWarps; }
int ws_chunk_atoms() { return kWsCA; }
int ws_slot_entries() { return kWsSlot; }
int ws_producers() { return kWsProd; }

size_t ws_smem_bytes(int nt_pad, bool staged)
{
    size_t b = ((size_t)2 * kWsCA * nt_pad + (size_t)2 * kWsCons * kWsCells) * sizeof(float);
    if (staged) b += (size_t)kWsProd * 2 * 3 * kWsSlot * 4;
    return b;
}

}  // namespace life
