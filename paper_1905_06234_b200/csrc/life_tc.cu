// life_tc.cu -- DSC on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// The product per CTA tile of 128 voxels is a dense contraction over atom
// chunks of 32:  Y(128 x N) += C(128 x 32) . D_c(32 x N), N = directions
// padded to 32, with C[v, a] = sum_k w[f_k] value_k built on the fly in
// shared memory from the sorted coefficient stream (life_dense.cu
// build_tc).  Roles inside one persistent CTA per SM (13 warps):
//
//   warps 0-7   producers.  Warp p owns voxel rows 16p..16p+15 of the A tile:
//               it zeroes them, streams its segment (index / fascicle / value,
//               16-byte loads, L2 prefetch one step ahead), gathers w[f],
//               stores C[cell] (rank 0: distinct cells) and adds the repeats
//               in rank order (deterministic), then splits the rows into
//               tf32 hi = x & ~0x1FFF and lo = x - hi in place.  Producer 0
//               also issues the bulk copy of the chunk's pre-split, pre-swizzled
//               dictionary tile (B operand, hi | lo).
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
#include "life_common.cuh"

namespace life {

constexpr int kTcMma = 8;                 // MMA warp
constexpr int kTcEpi = 9;                 // first epilogue warp
constexpr int kTcWarps = 13;
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTcStages = 3;
constexpr int kTcGroup = 4;               // chunks per TMEM accumulation group
constexpr uint32_t kTcPad = 0x40000000u;
constexpr uint32_t kTcMixed = 0x80000000u;
constexpr uint32_t kTcCellMask = (1u << kTcCellBits) - 1;
constexpr uint32_t kTcRankMask = (1u << (30 - kTcCellBits)) - 1;
constexpr uint32_t kTcSent = 0xFFFFFFFFu;
constexpr int kTcABytes = kTcTV * kTcCA * 4;  // 16 KB per A half (hi or lo)

struct TcArgs {
    const uint32_t *cr;
    const uint32_t *fiber;
    const float *val;
    const uint32_t *tptr;
    const uint32_t *t1;
    const float *D;      // [nch][2][N][32] swizzled
    const int *slotv;
    int nt, nch, n_ct;
};

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
__device__ __forceinline__ void tc_wait(uint64_t *b, unsigned parity)
{
    if (tc_try(b, parity)) return;
    const unsigned long long t0 = globaltimer();
    while (!tc_try(b, parity))
        if (globaltimer() - t0 > 4000000000ull) __trap();
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
    float r;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(w + f), "l"(pol));
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

// ---- producer: one 16-row block of the A tile for one chunk --------------------
// entries per lane and batch: kTcVec 16-byte vectors of the rank-0 region
// (128 entries per vector across the warp) and kTcWin windows of the rank>=1
// region (32 entries per window), gathered together so a step usually costs
// one load round trip and one gather round trip
constexpr int kTcVec = 3;
constexpr int kTcWin = 4;

__device__ __forceinline__ unsigned tc_build(float *C, const float *__restrict__ w, const TcArgs &A,
                                             uint32_t p0, uint32_t q0, uint32_t p1, int lane,
                                             uint64_t pol_s, uint64_t pol_k, float *junk)
{
    unsigned zeros = 0;
    const uint32_t nf = q0 - p0, n = p1 - p0;
    const int nb = (int)((nf + 127u) / 128u), nw = (int)((n - nf + 31u) / 32u);
    const uint32_t *cr = A.cr + p0;
    const uint32_t *fb = A.fiber + p0;
    const float *vl = A.val + p0;
    float wsl[kTcWin];
    uint32_t csl[kTcWin];
    float vsl[kTcWin];
    for (int b0 = 0; b0 < nb || b0 == 0; b0 += kTcVec) {
        uint4 c4[kTcVec], f4[kTcVec], v4[kTcVec];
#pragma unroll
        for (int j = 0; j < kTcVec; ++j) {
            const uint32_t k = 128u * (uint32_t)(b0 + j) + 4u * (uint32_t)lane;
            if (b0 + j < nb && k < nf) {
                c4[j] = tc_ld4(cr + k, pol_s);
                f4[j] = tc_ld4(fb + k, pol_s);
                v4[j] = tc_ld4(vl + k, pol_s);
            } else {
                c4[j] = make_uint4(kTcPad, kTcPad, kTcPad, kTcPad);
                f4[j] = make_uint4(kTcSent, kTcSent, kTcSent, kTcSent);
                v4[j] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
        if (b0 == 0) {
#pragma unroll
            for (int r = 0; r < kTcWin; ++r) {
                const uint32_t k = nf + 32u * (uint32_t)r + (uint32_t)lane;
                const bool in = r < nw && k < n;
                csl[r] = in ? tc_ld1(cr + k, pol_s) : kTcPad;
                const uint32_t f = in ? tc_ld1(fb + k, pol_s) : kTcSent;
                vsl[r] = in ? __uint_as_float(tc_ld1(vl + k, pol_s)) : 0.f;
                wsl[r] = tc_gather(w, f, pol_k);
            }
        }
        float wf[kTcVec][4];
#pragma unroll
        for (int j = 0; j < kTcVec; ++j) {
            wf[j][0] = tc_gather(w, f4[j].x, pol_k);
            wf[j][1] = tc_gather(w, f4[j].y, pol_k);
            wf[j][2] = tc_gather(w, f4[j].z, pol_k);
            wf[j][3] = tc_gather(w, f4[j].w, pol_k);
        }
#pragma unroll
        for (int j = 0; j < kTcVec; ++j) {
            const uint32_t c[4] = {c4[j].x, c4[j].y, c4[j].z, c4[j].w};
            const float v[4] = {__uint_as_float(v4[j].x), __uint_as_float(v4[j].y), __uint_as_float(v4[j].z),
                                __uint_as_float(v4[j].w)};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const bool ok = !(c[e] & kTcPad);
                const float sv = __fmul_rn(wf[j][e], v[e]);
                zeros += (ok && sv == 0.f) ? 1u : 0u;
                float *dst = ok ? C + (c[e] & kTcCellMask) : junk;
                *dst = sv;
            }
        }
    }
    __syncwarp();
    // repeats, window by window in rank order
    for (int r0 = 0; r0 < nw; r0 += kTcWin) {
        if (r0) {
#pragma unroll
            for (int r = 0; r < kTcWin; ++r) {
                const uint32_t k = nf + 32u * (uint32_t)(r0 + r) + (uint32_t)lane;
                const bool in = r0 + r < nw && k < n;
                csl[r] = in ? tc_ld1(cr + k, pol_s) : kTcPad;
                const uint32_t f = in ? tc_ld1(fb + k, pol_s) : kTcSent;
                vsl[r] = in ? __uint_as_float(tc_ld1(vl + k, pol_s)) : 0.f;
                wsl[r] = tc_gather(w, f, pol_k);
            }
        }
#pragma unroll
        for (int r = 0; r < kTcWin; ++r) {
            if (r0 + r >= nw) break;  // warp-uniform
            const uint32_t c = csl[r];
            const bool ok = !(c & kTcPad);
            const float sv = ok ? __fmul_rn(wsl[r], vsl[r]) : 0.f;
            zeros += (ok && sv == 0.f) ? 1u : 0u;
            const uint32_t cell = c & kTcCellMask;
            if (!__any_sync(0xffffffffu, ok && (c & kTcMixed))) {
                if (ok) C[cell] += sv;
            } else {
                const uint32_t rank = (c >> kTcCellBits) & kTcRankMask;
                const uint32_t rmin = __reduce_min_sync(0xffffffffu, ok ? rank : 0xFFFFFFFFu);
                const uint32_t rmax = __reduce_max_sync(0xffffffffu, ok ? rank : 0u);
                for (uint32_t rr = rmin; rr <= rmax; ++rr) {
                    if (ok && rank == rr) C[cell] += sv;
                    __syncwarp();
                }
            }
            __syncwarp();
        }
    }
    return zeros;
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

    if (warp < kTcProd) {
        // ===== producers =====
        const int p = warp;
        const uint64_t pol_s = tc_pol_stream(), pol_k = tc_pol_keep();
        float *junk = junkbuf + p * 32 + lane;
        int ct = blockIdx.x, c = 0;
        auto seg = [&](int ct_, int c_, uint32_t &s0, uint32_t &s1, uint32_t &s2) {
            const size_t t = ((size_t)ct_ * A.nch + c_) * kTcProd + p;
            s0 = __ldg(A.tptr + t);
            s1 = __ldg(A.t1 + t);
            s2 = __ldg(A.tptr + t + 1);
        };
        uint32_t p0 = 0, q0 = 0, p1 = 0, np0 = 0, nq0 = 0, np1 = 0;
        if (total > 0) seg(ct, c, p0, q0, p1);
        for (int k = 0; k < total; ++k) {
            const int s = k % kTcStages;
            // next step's segment: prefetch its three streams into L2
            int ctn = ct, cn = c + 1;
            if (cn == A.nch) { cn = 0; ctn += gridDim.x; }
            if (k + 1 < total) {
                seg(ctn, cn, np0, nq0, np1);
                if (lane < 3) {
                    const void *base = lane == 0 ? (const void *)(A.cr + np0)
                                     : lane == 1 ? (const void *)(A.fiber + np0) : (const void *)(A.val + np0);
                    tc_prefetch(base, (np1 - np0) * 4u, pol_s);
                }
            }
            if (k >= kTcStages) tc_wait(&empty[s], ((k / kTcStages) - 1) & 1);
            unsigned char *st = sm + (size_t)s * kStageBytes;
            float *Ahi = reinterpret_cast<float *>(st);
            float *Alo = reinterpret_cast<float *>(st + kTcABytes);
            if (p == 0 && lane == 0) {
                tc_arrive_tx(&full[s], kBBytes);
                tc_bulk(st + 2 * kTcABytes, A.D + (size_t)c * (kBBytes / 4), kBBytes, &full[s]);
            }
            // zero this warp's rows (2 KB)
            float4 *Z = reinterpret_cast<float4 *>(Ahi) + p * 128;
#pragma unroll
            for (int i = 0; i < 4; ++i) Z[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            skipped += tc_build(Ahi, w, A, p0, q0, p1, lane, pol_s, pol_k, junk);
            __syncwarp();
            // tf32 split of this warp's rows: hi in place, lo alongside
            float4 *H = reinterpret_cast<float4 *>(Ahi) + p * 128;
            float4 *L = reinterpret_cast<float4 *>(Alo) + p * 128;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float4 x = H[lane + 32 * i];
                float4 h, l;
                h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
                h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
                h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
                h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
                l.x = x.x - h.x;
                l.y = x.y - h.y;
                l.z = x.z - h.z;
                l.w = x.w - h.w;
                H[lane + 32 * i] = h;
                L[lane + 32 * i] = l;
            }
            // generic-proxy stores -> visible to the tensor core (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tc_arrive(&full[s]);
            ct = ctn;
            c = cn;
            p0 = np0; q0 = nq0; p1 = np1;
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
                        if (grp >= 2) tc_wait(&accempty[buf], ((grp >> 1) - 1) & 1);
                        tc_fence_after();
                    }
                    tc_wait(&full[s], (k / kTcStages) & 1);
                    tc_fence_after();
                    const uint32_t st = tc_sa(sm + (size_t)s * kStageBytes);
                    const uint64_t ah = tc_sdesc(st), al = tc_sdesc(st + kTcABytes);
                    const uint64_t bh = tc_sdesc(st + 2 * kTcABytes), bl = tc_sdesc(st + 2 * kTcABytes + N * 128);
                    const uint32_t d = tmem + (uint32_t)(buf * N);
#pragma unroll
                    for (int kk = 0; kk < kTcCA / 8; ++kk) {
                        const uint64_t o = (uint64_t)((kk * 32) >> 4);  // 8 tf32 = 32 bytes per K step
                        tc_mma(d, ah + o, bh + o, id, (c % kTcGroup) != 0 || kk != 0);
                        tc_mma(d, al + o, bh + o, id, 1u);
                        tc_mma(d, ah + o, bl + o, id, 1u);
                    }
                    tc_commit(&empty[s]);
                    if (c % kTcGroup == kTcGroup - 1 || c == A.nch - 1) {
                        tc_commit(&accfull[buf]);
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
                tc_wait(&accfull[buf], (grp >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int j = 0; j < 2 * NJ; ++j) {
                    float v[16];
                    tc_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * N + 16 * j), v);
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[16 * j + e] += v[e];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) tc_arrive(&accempty[buf]);
            }
            const int voxel = __ldg(A.slotv + (size_t)ct * kTcTV + row);
            if (voxel >= 0) {
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
static size_t tc_smem_bytes(int N)
{
    return (size_t)kTcStages * (2 * kTcABytes + 2 * N * kTcCA * 4) + 1024;  // + alignment slack
}

template <int NJ>
static int tc_dsc_t(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                    const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    TcArgs A{phi->t_cr, phi->t_fiber, phi->t_val, phi->t_tptr, phi->t_t1, phi->t_D, phi->t_slotv,
             phi->nt, phi->t_nch, phi->t_nct};
    k_dsc_tc<NJ><<<phi->t_blocks, kTcThreads, phi->t_smem, st>>>(A, w, y, b, flags, phi->red, o, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int NJ>
static int tc_prepare_t(life_phi *phi)
{
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
