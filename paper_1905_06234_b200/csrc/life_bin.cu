// life_bin.cu -- the binned two-phase DSC / WC products (default fp32 path).
//
// Every product of M = Phi x_1 D pairs two orders of the coefficients:
//
//   tile side  coefficients grouped by (tile of 128 voxel rows, chunk of KA
//              atoms): the dense contraction runs on tcgen05 (DSC:
//              Y += C . D_chunk with C[row, atom] = sum s; WC: Z = Y . D_chunk^T);
//   bin side   coefficients grouped by fascicle bin (a range of at most
//              kSB virtual fascicle slots): the per-coefficient random
//              access (DSC: w[f]; WC: the fascicle sum) hits a bin-sized
//              slice in shared memory instead of L2.
//
// The sides exchange one value per coefficient through a tile-major scratch
// vector: the DSC bin side writes s = w[f] * value there and the tile side
// reads it; the WC tile side writes z = Z[row, atom] there and the bin side
// reads it.  Both orders are stable sorts of the same coefficient list, so a
// segment (tile, chunk, bin) is contiguous in both: the bin side streams its
// bin-major arrays and reads/writes the scratch in runs.  Random accesses per
// coefficient are shared-memory only; global memory is streamed.
//
// Determinism without ordering constraints: the DSC C tile is int32 fixed
// point (per-call scale from max |s|, so the <= kRanks repeats of a (row,
// atom) cell add exactly with shared-memory atomics); WC fascicle sums are
// exact integers (64-bit fixed point, accumulated as two 32-bit limbs with
// native shared-memory atomics; a virtual fascicle slot holds at most
// kSlotCap coefficients so the limbs cannot overflow; flushed per fascicle
// run into int64 sums), so any summation order gives the same bits, across
// CTAs, slots, and ranks.
//
// Reference: _kernels.dsc_range / wc_range (/root/reference/pkg/src/
// lifespmv/_kernels.py:14-33, 57-68) under the owned regimes of
// engine.dsc_parallel / wc_parallel (engine.py:247-289, 372-413).
#include <cub/cub.cuh>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "life_common.cuh"
#include "life_tcgen05.cuh"

namespace life {
namespace bin {

constexpr int kTV = 128;            // tile rows (tcgen05 M)
constexpr int kRanks = 7;           // duplicate ranks per tile row (rank field value 7 = pad)
constexpr uint16_t kPad = 0xFFFFu;  // tile-major pad entry
constexpr int kFixRows = 32;        // partial rows per fixup piece (one warp)
constexpr int kSlotCap = 256;       // coefficients per virtual fascicle slot (2-limb fixed point)
constexpr int kSB = 16384;          // virtual slots per bin: 64 KB (DSC w) / 128 KB (WC limbs)
constexpr int kBuild = 8;           // builder / gatherer warps of the tile kernels
constexpr int kSideWarps = 32;      // bin-side CTA
constexpr int kSideU = 4;           // 32-entry chunks per warp batch on the bin side
constexpr int kSlots = 3;           // staged steps per tile kernel
#ifndef LIFE_KCH
#define LIFE_KCH 992
#endif
// 4-entry units per bin-side chunk: one per consumer thread (31 warps).  With
// 1024 the first consumer warp took two units per chunk and, holding every
// ring slot longest, paced the whole WC bin side (C2 WC 0.543 -> 0.501 ms)
constexpr int kCH = LIFE_KCH;

// Role timing, compiled in only with -DLIFE_BIN_DIAG (tools/bin_roles.py):
// clock64 spans per category summed over warps (lane 0) into g_bin_cyc.
#ifdef LIFE_BIN_DIAG
__device__ unsigned long long g_bin_cyc[32];
#define BD_T0(v) const long long v = clock64()
#define BD_ACC(i, v) (bdc[i] += (unsigned long long)(clock64() - (v)))
#define BD_DECL unsigned long long bdc[32] = {}
#define BD_FLUSH                                                               \
    if ((threadIdx.x & 31) == 0)                                               \
        for (int i_ = 0; i_ < 32; ++i_)                                        \
            if (bdc[i_]) atomicAdd(&g_bin_cyc[i_], bdc[i_])
#else
#define BD_T0(v)
#define BD_ACC(i, v)
#define BD_DECL
#define BD_FLUSH
#endif
#define BD_WAIT(i, expr) \
    do {                 \
        BD_T0(bt_);      \
        expr;            \
        BD_ACC(i, bt_);  \
    } while (0)

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool bar_try(uint64_t *b, unsigned parity)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(sa(b)), "r"(parity) : "memory");
    return ok != 0;
}
// host-mapped debug record of the first timed-out wait (life_debug_timeout)
__device__ unsigned *g_timeout_rec = nullptr;
// trap after 4 s instead of hanging the GPU
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned parity)
{
    if (bar_try(b, parity)) return;
    const unsigned long long t0 = globaltimer();
    while (!bar_try(b, parity))
        if (globaltimer() - t0 > 4000000000ull) {
            if (g_timeout_rec && atomicCAS(g_timeout_rec, 0u, 1u) == 0u) {
                g_timeout_rec[1] = blockIdx.x;
                g_timeout_rec[2] = threadIdx.x >> 5;
                g_timeout_rec[3] = sa(b);
                g_timeout_rec[4] = parity;
                __threadfence_system();
            }
            __trap();
        }
}
// bulk copy global -> shared in pieces of at most 32 KB, completing on bar
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *b, uint64_t pol)
{
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
    for (unsigned o = 0; o < bytes; o += 32768u)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(sa(d + o)), "l"(s + o), "r"(min(32768u, bytes - o)), "r"(sa(b)), "l"(pol)
                     : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *src, unsigned bytes)
{
    const char *s = reinterpret_cast<const char *>(src);
    for (unsigned o = 0; o < bytes; o += 32768u)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s + o), "r"(min(32768u, bytes - o)) : "memory");
}
__device__ __forceinline__ uint64_t pol_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void named_bar(int id, int threads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a)
{
    uint16_t r;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ float lds_f(uint32_t a)
{
    float r;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ void sts_f(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory"); }
__device__ __forceinline__ float4 lds_f4(uint32_t a)
{
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
    return r;
}
__device__ __forceinline__ void sts_f4(uint32_t a, float4 v)
{
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// TMEM stores / loads of 16 consecutive 32-bit columns of this thread's lane
__device__ __forceinline__ void tm_st16(uint32_t addr, const uint32_t (&v)[16])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t addr, uint32_t (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 64-bit fixed-point exponent of the WC bin side: every term |val * z| is at
// most vmax * dmax * ||y_v|| <= vmax * dmax * ynorm; scaled terms stay below
// 2^45 (two limbs: 24 low bits summed in u32 over <= 256 terms, the signed
// rest in i32), and a fascicle total (fmax_nnz terms, all ranks) below 2^62.
__host__ __device__ inline int bin_exponent(double vmax, double dmax, double ynorm, double fmax_nnz)
{
    const double bound = vmax * dmax * ynorm * (1.0 + 1.0 / 1024.0);
    if (!(bound > 0.0) || !(bound < 1e300)) return 0;
    int eb;
    frexp(bound, &eb);  // bound < 2^eb
    int ef;
    frexp(fmax_nnz > 1.0 ? fmax_nnz : 1.0, &ef);  // fmax_nnz < 2^ef
    int cap = 62 - ef;
    if (cap > 45) cap = 45;
    int ex = cap - eb;
    if (ex > 1000) ex = 1000;
    if (ex < -1000) ex = -1000;
    return ex;
}
__device__ inline int bin_exponent_dev(const FixParams &fx, int nt)
{
    const double yn = fx.yvbound ? (double)*fx.yvbound
                      : fx.ysumsq ? sqrt(*fx.ysumsq) : sqrt((double)nt) * (double)*fx.ymax;
    return bin_exponent(fx.vmax, fx.dmax, yn, fx.fmax_nnz);
}

// fixed-order reductions of per-warp partials (last CTA)
template <typename T, typename Op>
__device__ T block_finish(T acc, T init, Op op, int nthreads);
template <typename T, typename Op>
__device__ T block_reduce(const T *part, int n, T init, Op op, int nthreads)
{
    T acc = init;
    // loads batched 8 deep (one L2 round trip per batch instead of per
    // element), combined in the same ascending order: same bits as a plain loop
    for (int b = threadIdx.x; b < n; b += 8 * nthreads) {
        T v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = b + k * nthreads;
            v[k] = i < n ? __ldcg(part + i) : init;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (b + k * nthreads < n) acc = op(acc, v[k]);
    }
    return block_finish<T>(acc, init, op, nthreads);
}
// the block's per-thread values combined: warp shuffles, then warp 0 over
// the warps' results (fixed order)
template <typename T, typename Op>
__device__ T block_finish(T acc, T init, Op op, int nthreads)
{
    __shared__ T s[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = op(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    T r = init;
    if (threadIdx.x < 32) {
        r = threadIdx.x < (nthreads >> 5) ? s[threadIdx.x] : init;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = op(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (threadIdx.x == 0) s[0] = r;
    }
    __syncthreads();
    r = s[0];
    __syncthreads();
    return r;
}
struct OpSum {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct OpMaxF {
    __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};

__device__ __forceinline__ bool last_cta(unsigned *counter)
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

// DSC outputs from the tile/fixup partials and the bin side's skip partials
__device__ void dsc_finish(const ReduceSlots &red, int nparts, const unsigned long long *skip, int nskip,
                           const DscOut &out, unsigned *counter, const CallHooks &hooks, int nthreads,
                           unsigned *nonfinite)
{
    // the three reductions in one pass (each in block_reduce's order: the
    // same bits), so the last CTA waits on one round of loads, not three
    double a = 0.0;
    float m = 0.f;
    unsigned long long k = 0ull;
    const int nmax = max(nparts, nskip);
    for (int b = threadIdx.x; b < nmax; b += 8 * nthreads) {
        double va[8];
        float vm[8];
        unsigned long long vk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = b + j * nthreads;
            va[j] = i < nparts ? __ldcg(red.part_d + i) : 0.0;
            vm[j] = i < nparts ? __ldcg(red.part_f + i) : 0.f;
            vk[j] = i < nskip ? __ldcg(skip + i) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = b + j * nthreads;
            if (i < nparts) {
                a += va[j];
                m = fmaxf(m, vm[j]);
            }
            if (i < nskip) k += vk[j];
        }
    }
    const double tsq = block_finish<double>(a, 0.0, OpSum{}, nthreads);
    const float tmax = block_finish<float>(m, 0.f, OpMaxF{}, nthreads);
    const unsigned long long tsk = block_finish<unsigned long long>(k, 0ull, OpSum{}, nthreads);
    if (threadIdx.x == 0) {
        if (out.sumsq) *out.sumsq = tsq;
        if (out.absmax) *out.absmax = tmax;
        if (out.skipped) *out.skipped = tsk;
        if (out.skipped_d) *out.skipped_d = (double)tsk;
        *counter = 0;
        if (nonfinite) *nonfinite = 0u;
        if (hooks.t_accum && hooks.t_begin) *hooks.t_accum += globaltimer() - *hooks.t_begin;
    }
}

// ---------------------------------------------------------------------------
// construction kernels
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t gtid() { return blockIdx.x * (int64_t)blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

__global__ void k_iota(uint32_t *o, int64_t n)
{
    for (int64_t i = gtid(); i < n; i += gstride()) o[i] = (uint32_t)i;
}
template <typename K>
__global__ void k_key_va(const uint32_t *a, const uint32_t *v, int64_t n, uint32_t na, K *key)
{
    for (int64_t i = gtid(); i < n; i += gstride()) key[i] = (K)((unsigned long long)v[i] * na + a[i]);
}
// run heads of a sorted u64 key: head[p] = p at a run start, else 0
template <typename K>
__global__ void k_heads64(const K *k, int64_t n, uint32_t *head)
{
    for (int64_t p = gtid(); p < n; p += gstride()) head[p] = (p == 0 || k[p] != k[p - 1]) ? (uint32_t)p : 0u;
}
__global__ void k_heads32(const uint32_t *k, int64_t n, uint32_t *head)
{
    for (int64_t p = gtid(); p < n; p += gstride()) head[p] = (p == 0 || k[p] != k[p - 1]) ? (uint32_t)p : 0u;
}
// rank of each coefficient among the equal (voxel, atom) pairs in stable
// order, and the largest rank per voxel
template <typename K>
__global__ void k_rank_va(const K *sk, const uint32_t *perm, const uint32_t *rstart, int64_t n,
                          uint32_t na, uint32_t *rank_o, uint32_t *vmaxr)
{
    // p0 is warp-uniform (the grid stride is a multiple of 32); run ends of
    // one voxel are adjacent in key order, so their lanes combine before one
    // atomicMax per voxel per warp (was ~60M contended atomics at C2)
    for (int64_t p0 = gtid() - (threadIdx.x & 31); p0 < n; p0 += gstride()) {
        const int64_t p = p0 + (threadIdx.x & 31);
        const bool in = p < n;
        uint32_t r = 0, vox = 0xFFFFFFFFu;
        if (in) {
            r = (uint32_t)p - rstart[p];
            rank_o[perm[p]] = r;
            if (p == n - 1 || sk[p + 1] != sk[p]) vox = (uint32_t)(sk[p] / na);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, vox);
        const uint32_t m = __reduce_max_sync(peers, r);
        if (vox != 0xFFFFFFFFu && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicMax(&vmaxr[vox], m);
    }
}
__global__ void k_rows_per_voxel(const uint32_t *vmaxr, int nv, uint32_t *nr)
{
    for (int64_t v = gtid(); v < nv; v += gstride()) nr[v] = vmaxr[v] / kRanks + 1u;
}
__global__ void k_row_of(const uint32_t *v, const uint32_t *rank_o, const uint32_t *rowbase, int64_t n,
                         uint32_t *row_o, unsigned *rcnt)
{
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const uint32_t r = rowbase[v[i]] + rank_o[i] / kRanks;
        row_o[i] = r;
        atomicAdd(&rcnt[r], 1u);
    }
}
__global__ void k_hist(const uint32_t *x, int64_t n, unsigned *cnt)
{
    for (int64_t i = gtid(); i < n; i += gstride()) atomicAdd(&cnt[x[i]], 1u);
}
__global__ void k_slots_per_fiber(const unsigned *cnt, int nf, uint32_t *ns)
{
    for (int64_t f = gtid(); f < nf; f += gstride()) ns[f] = cnt[f] <= (unsigned)kSlotCap ? 1u : (cnt[f] + kSlotCap - 1) / kSlotCap;
}
__global__ void k_vf2f(const uint32_t *f2vf, int nf, uint32_t *vf2f)
{
    for (int64_t f = gtid(); f < nf; f += gstride())
        for (uint32_t s = f2vf[f]; s < f2vf[f + 1]; ++s) vf2f[s] = (uint32_t)f;
}
// virtual slot of each coefficient: the fascicle's occurrence index (stable
// order) in blocks of kSlotCap
__global__ void k_vf_split(const uint32_t *perm, const uint32_t *sf, const uint32_t *rstart, const uint32_t *f2vf,
                           int64_t n, uint32_t *vf_o)
{
    for (int64_t p = gtid(); p < n; p += gstride())
        vf_o[perm[p]] = f2vf[sf[p]] + ((uint32_t)p - rstart[p]) / kSlotCap;
}
__global__ void k_big_flags(const uint32_t *f, const unsigned *cnt, int64_t n, uint8_t *big)
{
    for (int64_t i = gtid(); i < n; i += gstride()) big[i] = cnt[f[i]] > (unsigned)kSlotCap ? 1 : 0;
}
__global__ void k_vf_identity(const uint32_t *f, const uint32_t *f2vf, int64_t n, uint32_t *vf_o)
{
    for (int64_t i = gtid(); i < n; i += gstride()) vf_o[i] = f2vf[f[i]];
}
// bin-major key (bin, tile, chunk) of each coefficient and the payload the
// placement needs, sorted along with it (no gathers afterwards): fp32 value
// bits << 32 | bin slot << 16 | tile cell
template <typename K>
__global__ void k_key_bm(const uint32_t *a, const uint32_t *row_o, const uint32_t *vf_o, const uint32_t *slot_of_row,
                         const double *val, int64_t n, int ka_shift, int ka, uint32_t nch, uint32_t ntiles,
                         K *kbm, unsigned long long *pay)
{
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const uint32_t sr = slot_of_row[row_o[i]], ai = a[i], vf = vf_o[i];
        const uint32_t t = sr / kTV, c = ai >> ka_shift, b = vf / kSB;
        kbm[i] = (K)(((unsigned long long)b * ntiles + t) * nch + c);
        const uint32_t cell = (sr % kTV) * (uint32_t)(ka + 4) + (ai & (uint32_t)(ka - 1));
        pay[i] = ((unsigned long long)__float_as_uint((float)val[i]) << 32) | ((vf % kSB) << 16) | cell;
    }
}
template <typename K>
__global__ void k_head_flags(const K *k, int64_t n, uint8_t *head, uint32_t *head32)
{
    for (int64_t p = gtid(); p < n; p += gstride()) {
        const bool h = p == 0 || k[p] != k[p - 1];
        head[p] = h ? 1 : 0;
        head32[p] = h ? 1u : 0u;
    }
}
// per segment (bin-major order): key, length in 4-entry units, and the
// tile-major sort key (tile, chunk, bin)
template <typename K>
__global__ void k_seg_info(const K *kbm_sorted, const uint32_t *first, int64_t nseg, int64_t n,
                           unsigned long long per_bin, uint32_t nbins, uint32_t *len4, unsigned long long *segkey,
                           unsigned long long *tmkey, uint32_t *step)
{
    for (int64_t s = gtid(); s < nseg; s += gstride()) {
        const uint32_t f0 = first[s], f1 = s + 1 < nseg ? first[s + 1] : (uint32_t)n;
        const unsigned long long k = (unsigned long long)kbm_sorted[f0];
        len4[s] = (f1 - f0 + 3u) / 4u;
        segkey[s] = k;
        const unsigned long long b = k / per_bin, tc = k % per_bin;
        tmkey[s] = tc * nbins + b;
        step[s] = (uint32_t)tc;
    }
}
__global__ void k_pad8(const unsigned *cnt, int64_t n, unsigned *pcnt)
{
    for (int64_t s = gtid(); s < n; s += gstride()) pcnt[s] = (cnt[s] + 7u) & ~7u;
}
__global__ void k_step_units(const uint32_t *step, const uint32_t *len4, int64_t nseg, unsigned *units)
{
    for (int64_t s = gtid(); s < nseg; s += gstride()) atomicAdd(&units[step[s]], len4[s]);
}
__global__ void k_step_pad(const unsigned *units, int64_t nsteps, unsigned *padded)
{
    for (int64_t s = gtid(); s < nsteps; s += gstride()) padded[s] = (4u * units[s] + 7u) & ~7u;
}
// tile-major exclusive unit prefix at the first segment of each step
__global__ void k_step_first(const uint32_t *perm_seg, const uint32_t *tm_excl, const uint32_t *step, int64_t nseg,
                             uint32_t *stepx)
{
    for (int64_t i = gtid(); i < nseg; i += gstride()) {
        const uint32_t st = step[perm_seg[i]];
        if (i == 0 || step[perm_seg[i - 1]] != st) stepx[st] = tm_excl[i];
    }
}
// tile-major start of each segment: its step's start + the 4-padded lengths
// of the step's earlier segments (lower rank, then lower bin)
__global__ void k_seg_tm(const uint32_t *perm_seg, const uint32_t *tm_excl, const uint32_t *step, int64_t nseg,
                         const uint32_t *step_ptr, const uint32_t *stepx, uint32_t *dst4)
{
    for (int64_t i = gtid(); i < nseg; i += gstride()) {
        const uint32_t s = perm_seg[i], st = step[s];
        dst4[s] = step_ptr[st] / 4u + (tm_excl[i] - stepx[st]);
    }
}
// place every coefficient in both orders
__global__ void k_place(const unsigned long long *pay, const uint32_t *segid, const uint32_t *first,
                        const uint32_t *src4, const uint32_t *dst4, int64_t n, uint16_t *vid, float *val32,
                        uint16_t *cellr)
{
    for (int64_t p = gtid(); p < n; p += gstride()) {
        const uint32_t s = segid[p] - 1u;
        const uint32_t idx = (uint32_t)p - first[s];
        const uint32_t bp = 4u * src4[s] + idx, tp = 4u * dst4[s] + idx;
        const unsigned long long q = pay[p];
        vid[bp] = (uint16_t)((uint32_t)q >> 16);
        val32[bp] = __uint_as_float((uint32_t)(q >> 32));
        cellr[tp] = (uint16_t)(q & 0xFFFFu);
    }
}
// lower bound of key b * per_bin over the bin-major segment keys
__global__ void k_bin_seg(const unsigned long long *segkey, int64_t nseg, int nbins, unsigned long long per_bin,
                          uint32_t *binseg)
{
    for (int64_t b = gtid(); b <= nbins; b += gstride()) {
        const unsigned long long key = (unsigned long long)b * per_bin;
        int64_t lo = 0, hi = nseg;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (segkey[mid] < key) lo = mid + 1; else hi = mid;
        }
        binseg[b] = (uint32_t)lo;
    }
}
// bin-side CTA c takes the segments whose start lies in units [c*U/g, (c+1)*U/g)
// bin-side CTA ranges balanced by cost = units + kSegCost per segment (a
// segment start is a scattered scratch access and a search; sparse bins of
// one-unit segments would otherwise make stragglers)
constexpr unsigned long long kSegCost = 4;
__global__ void k_cta_seg(const uint32_t *src4, int64_t nseg, int grid, uint32_t *ctaseg)
{
    for (int64_t c = gtid(); c <= grid; c += gstride()) {
        const unsigned long long total = (unsigned long long)src4[nseg] + kSegCost * (unsigned long long)nseg;
        const unsigned long long target = total * (unsigned long long)c / (unsigned long long)grid;
        int64_t lo = 0, hi = nseg;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((unsigned long long)src4[mid] + kSegCost * (unsigned long long)mid < target) lo = mid + 1; else hi = mid;
        }
        ctaseg[c] = (uint32_t)(c == grid ? nseg : lo);
    }
}
__global__ void k_gather_u32(const uint32_t *idx, const uint32_t *in, int64_t n, uint32_t *out)
{
    for (int64_t i = gtid(); i < n; i += gstride()) out[i] = in[idx[i]];
}
__global__ void k_fill_u16(uint16_t *x, int64_t n, uint16_t v)
{
    for (int64_t i = gtid(); i < n; i += gstride()) x[i] = v;
}

static int gridn(int64_t n)
{
    int64_t b = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 65535 * 8));
}
static int bits64(unsigned long long x)
{
    int b = 0;
    while (b < 64 && (x >> b) != 0) ++b;
    return std::max(b, 1);
}

template <typename K, typename V = uint32_t>
static int sort_pairs(const K *kin, K *kout, const V *vin, V *vout, int64_t n, int bits,
                      cudaStream_t st)
{
    size_t tb = 0;
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, bits, st));
    void *temp = nullptr;
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tb, kin, kout, vin, vout, n, 0, bits, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    return LIFE_OK;
}
static int scan_max(const uint32_t *in, uint32_t *out, int64_t n, cudaStream_t st)
{
    size_t tb = 0;
    LIFE_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, in, out, cub::Max(), n, st));
    void *temp = nullptr;
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceScan::InclusiveScan(temp, tb, in, out, cub::Max(), n, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return LIFE_OK;
}
// exclusive sum of n counts into out[0..n] (out[n] = total)
static int scan_excl(const uint32_t *in, uint32_t *out, int64_t n, cudaStream_t st)
{
    LIFE_CUDA(cudaMemsetAsync(out, 0, sizeof(uint32_t), st));
    if (n == 0) return LIFE_OK;
    size_t tb = 0;
    LIFE_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out + 1, n, st));
    void *temp = nullptr;
    LIFE_CUDA(cudaMallocAsync(&temp, tb, st));
    LIFE_CUDA(cub::DeviceScan::InclusiveSum(temp, tb, in, out + 1, n, st));
    LIFE_CUDA(cudaFreeAsync(temp, st));
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return LIFE_OK;
}

// tf32 split on the host (same bits as the device split)
static void tf32_split_h(float x, float &hi, float &lo)
{
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    std::memcpy(&hi, &u, 4);
    lo = x - hi;
}
// byte offset of f16 element (row, k) in a K-major SWIZZLE_128B tile (64 per row)
static inline size_t sw16(uint32_t row, uint32_t k)
{
    return (size_t)(row >> 3) * 1024u + (row & 7u) * 128u + ((((k >> 3) ^ row) & 7u) << 4) + (k & 7u) * 2u;
}

}  // namespace bin

// ---------------------------------------------------------------------------
// build
// ---------------------------------------------------------------------------
int prepare_bin(life_phi *phi);

int build_bin(life_phi *phi, const uint32_t *a, const uint32_t *v, const uint32_t *f, const double *val,
              const std::vector<double> &hdict, const std::function<int()> &ready_fv, cudaStream_t st)
{
    using namespace bin;
    const int64_t n = phi->nc;
    const int N = (phi->nt + 31) / 32 * 32;
    if (n == 0 || N > 192 || n >= 0xF0000000ll) return LIFE_OK;
    const int ka = 64, ka_shift = 6;
    const int nch = (phi->na + ka - 1) / ka;
    const uint32_t na = (uint32_t)phi->na;
    const int nv = phi->nv, nf = phi->nf;

    // temporaries (stream-ordered)
    std::vector<void *> tmp;
    auto talloc = [&](void **p, size_t bytes) -> int {
        LIFE_CUDA(cudaMallocAsync(p, std::max<size_t>(bytes, 16), st));
        tmp.push_back(*p);
        return LIFE_OK;
    };
    struct Free {
        std::vector<void *> &t;
        cudaStream_t s;
        ~Free()
        {
            for (void *p : t) cudaFreeAsync(p, s);
        }
    } freer{tmp, st};

    // 1. rank of each coefficient within its (voxel, atom) pair
    unsigned long long *kva, *skva;
    uint32_t *iota, *perm, *head, *rstart, *rank_o, *vmaxr;
    LIFE_TRY(talloc((void **)&kva, n * 8));
    LIFE_TRY(talloc((void **)&skva, n * 8));
    LIFE_TRY(talloc((void **)&iota, n * 4));
    LIFE_TRY(talloc((void **)&perm, n * 4));
    LIFE_TRY(talloc((void **)&head, n * 4));
    LIFE_TRY(talloc((void **)&rstart, n * 4));
    LIFE_TRY(talloc((void **)&rank_o, n * 4));
    LIFE_TRY(talloc((void **)&vmaxr, (size_t)nv * 4));
    k_iota<<<gridn(n), 256, 0, st>>>(iota, n);
    LIFE_CHECK_LAUNCH();
    const unsigned long long vamax = (unsigned long long)nv * na;
    LIFE_CUDA(cudaMemsetAsync(vmaxr, 0, (size_t)nv * 4, st));
    if (vamax <= 0xFFFFFFFFull) {  // 32-bit (voxel, atom) keys: a third less sort traffic
        uint32_t *k32 = reinterpret_cast<uint32_t *>(kva), *sk32 = reinterpret_cast<uint32_t *>(skva);
        k_key_va<uint32_t><<<gridn(n), 256, 0, st>>>(a, v, n, na, k32);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY(sort_pairs<uint32_t>(k32, sk32, iota, perm, n, bits64(vamax), st));
        k_heads64<uint32_t><<<gridn(n), 256, 0, st>>>(sk32, n, head);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY(scan_max(head, rstart, n, st));
        k_rank_va<uint32_t><<<gridn(n), 256, 0, st>>>(sk32, perm, rstart, n, na, rank_o, vmaxr);
        LIFE_CHECK_LAUNCH();
    } else {
        k_key_va<unsigned long long><<<gridn(n), 256, 0, st>>>(a, v, n, na, kva);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY(sort_pairs<unsigned long long>(kva, skva, iota, perm, n, bits64(vamax), st));
        k_heads64<unsigned long long><<<gridn(n), 256, 0, st>>>(skva, n, head);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY(scan_max(head, rstart, n, st));
        k_rank_va<unsigned long long><<<gridn(n), 256, 0, st>>>(skva, perm, rstart, n, na, rank_o, vmaxr);
        LIFE_CHECK_LAUNCH();
    }

    setup_mark(st, "bin phase 1");
    // 2. tile rows: a voxel gets one row per kRanks duplicate ranks
    uint32_t *nr, *rowbase, *row_o;
    unsigned *rcnt;
    LIFE_TRY(talloc((void **)&nr, (size_t)nv * 4));
    LIFE_TRY(talloc((void **)&rowbase, ((size_t)nv + 1) * 4));
    LIFE_TRY(talloc((void **)&row_o, n * 4));
    k_rows_per_voxel<<<gridn(nv), 256, 0, st>>>(vmaxr, nv, nr);
    LIFE_CHECK_LAUNCH();
    LIFE_TRY(scan_excl(nr, rowbase, nv, st));
    uint32_t R = 0;
    LIFE_CUDA(cudaMemcpyAsync(&R, rowbase + nv, 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    LIFE_TRY(talloc((void **)&rcnt, (size_t)R * 4));
    LIFE_CUDA(cudaMemsetAsync(rcnt, 0, (size_t)R * 4, st));
    k_row_of<<<gridn(n), 256, 0, st>>>(v, rank_o, rowbase, n, row_o, rcnt);
    LIFE_CHECK_LAUNCH();
    std::vector<uint32_t> hcnt(R), hbase(nv + 1);
    LIFE_CUDA(cudaMemcpyAsync(hcnt.data(), rcnt, (size_t)R * 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaMemcpyAsync(hbase.data(), rowbase, ((size_t)nv + 1) * 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));

    setup_mark(st, "bin phase 2");
    // 3. deal rows to tiles: counting sort by coefficient count (descending,
    // stable), snake order over the tiles so every tile carries about the
    // same number of coefficients
    // tile count rounded up to a multiple of the tile grid (one CTA per SM):
    // rows are dealt by coefficient count, so every CTA then gets the same
    // number of equally loaded tiles, instead of the last round leaving
    // CTAs idle (196 full tiles on 148 SMs: half the CTAs did 2 tiles).
    // Each row's products do not depend on its tile: results are unchanged.
    static const bool no_round = [] { const char *e = std::getenv("LIFE_B200_NO_TILE_ROUND"); return e && *e == '1'; }();
    const int64_t tiles_full = ((int64_t)R + kTV - 1) / kTV;
    const int64_t ntiles = no_round || tiles_full == 0 ? tiles_full
                                                       : (tiles_full + phi->sms - 1) / phi->sms * phi->sms;
    std::vector<uint32_t> slot_of_row(R);
    std::vector<int> rowvox((size_t)ntiles * kTV, -1), rowpart((size_t)ntiles * kTV, -1);
    {
        uint32_t cmax = 0;
        for (uint32_t c : hcnt) cmax = std::max(cmax, c);
        std::vector<uint32_t> start((size_t)cmax + 2, 0);
        for (uint32_t c : hcnt) ++start[cmax - c + 1];
        for (size_t i = 1; i < start.size(); ++i) start[i] += start[i - 1];
        std::vector<uint32_t> order(R);
        for (uint32_t r = 0; r < R; ++r) order[start[cmax - hcnt[r]]++] = r;
        for (int64_t i = 0; i < (int64_t)R; ++i) {
            const int64_t lane = i / ntiles, q = i % ntiles;
            const int64_t t = (lane & 1) ? ntiles - 1 - q : q;
            slot_of_row[order[i]] = (uint32_t)(t * kTV + lane);
        }
    }
    std::vector<uint32_t> fixptr(1, 0);
    std::vector<int> fixvox;
    int nprow = 0;
    for (int vx = 0; vx < nv; ++vx) {
        const uint32_t r0 = hbase[vx], r1 = hbase[vx + 1];
        for (uint32_t r = r0; r < r1; ++r) rowvox[slot_of_row[r]] = vx;
        if (r1 - r0 > 1) {
            for (uint32_t r = r0; r < r1; ++r) rowpart[slot_of_row[r]] = nprow++;
            fixptr.push_back((uint32_t)nprow);
            fixvox.push_back(vx);
        }
    }
    uint32_t *d_slot;
    LIFE_TRY(talloc((void **)&d_slot, (size_t)R * 4));
    LIFE_CUDA(cudaMemcpyAsync(d_slot, slot_of_row.data(), (size_t)R * 4, cudaMemcpyHostToDevice, st));
    LIFE_TRY(dalloc(phi, &phi->b_rowvox, rowvox.size()));
    LIFE_TRY(dalloc(phi, &phi->b_rowpart, rowpart.size()));
    LIFE_CUDA(cudaMemcpyAsync(phi->b_rowvox, rowvox.data(), rowvox.size() * 4, cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaMemcpyAsync(phi->b_rowpart, rowpart.data(), rowpart.size() * 4, cudaMemcpyHostToDevice, st));
    phi->b_nfix = (int)fixvox.size();
    phi->b_nprow = nprow;
    if (phi->b_nfix) {
        // fold work: pieces of at most kFixRows partial rows (one warp each);
        // a voxel of several pieces stores piece sums and is folded by a
        // whole CTA afterwards (fixed order: deterministic)
        std::vector<uint32_t> pcs, big, bpp(1, 0);
        uint32_t nsum = 0;
        for (int m = 0; m < phi->b_nfix; ++m) {
            const uint32_t r0 = fixptr[m], r1 = fixptr[m + 1];
            const bool multi = r1 - r0 > (uint32_t)kFixRows;
            for (uint32_t r = r0; r < r1; r += kFixRows) {
                pcs.push_back((uint32_t)fixvox[m]);
                pcs.push_back(r);
                pcs.push_back(std::min(r1, r + (uint32_t)kFixRows));
                pcs.push_back(multi ? nsum++ : 0xFFFFFFFFu);
            }
            if (multi) {
                big.push_back((uint32_t)fixvox[m]);
                bpp.push_back(nsum);
            }
        }
        phi->b_npc = (int)(pcs.size() / 4);
        phi->b_nbig = (int)big.size();
        LIFE_TRY(dalloc(phi, &phi->b_fixpc, pcs.size()));
        LIFE_TRY(dalloc(phi, &phi->b_ypart, (size_t)nprow * N));
        LIFE_CUDA(cudaMemcpyAsync(phi->b_fixpc, pcs.data(), pcs.size() * 4, cudaMemcpyHostToDevice, st));
        if (phi->b_nbig) {
            LIFE_TRY(dalloc(phi, &phi->b_fixbig, big.size()));
            LIFE_TRY(dalloc(phi, &phi->b_fixbpp, bpp.size()));
            LIFE_TRY(dalloc(phi, &phi->b_fixsum, (size_t)nsum * N));
            LIFE_CUDA(cudaMemcpyAsync(phi->b_fixbig, big.data(), big.size() * 4, cudaMemcpyHostToDevice, st));
            LIFE_CUDA(cudaMemcpyAsync(phi->b_fixbpp, bpp.data(), bpp.size() * 4, cudaMemcpyHostToDevice, st));
        }
        LIFE_CUDA(cudaStreamSynchronize(st));
    }

    setup_mark(st, "bin phase 3");
    LIFE_TRY(ready_fv());  // phases 1-3 read only atoms and voxels
    // 4. virtual fascicle slots (at most kSlotCap coefficients each) and bins
    unsigned *fcnt;
    uint32_t *nslot, *vf_o;
    LIFE_TRY(talloc((void **)&fcnt, (size_t)nf * 4));
    LIFE_TRY(talloc((void **)&nslot, (size_t)nf * 4));
    LIFE_TRY(talloc((void **)&vf_o, n * 4));
    LIFE_TRY(dalloc(phi, &phi->b_f2vf, (size_t)nf + 1));
    LIFE_CUDA(cudaMemsetAsync(fcnt, 0, (size_t)nf * 4, st));
    k_hist<<<gridn(n), 256, 0, st>>>(f, n, fcnt);
    LIFE_CHECK_LAUNCH();
    k_slots_per_fiber<<<gridn(nf), 256, 0, st>>>(fcnt, nf, nslot);
    LIFE_CHECK_LAUNCH();
    LIFE_TRY(scan_excl(nslot, phi->b_f2vf, nf, st));
    uint32_t nvf = 0;
    LIFE_CUDA(cudaMemcpyAsync(&nvf, phi->b_f2vf + nf, 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    LIFE_TRY(dalloc(phi, &phi->b_vf2f, (size_t)nvf));
    k_vf2f<<<gridn(nf), 256, 0, st>>>(phi->b_f2vf, nf, phi->b_vf2f);
    LIFE_CHECK_LAUNCH();
    if (nvf == (uint32_t)nf) {
        k_vf_identity<<<gridn(n), 256, 0, st>>>(f, phi->b_f2vf, n, vf_o);
        LIFE_CHECK_LAUNCH();
    } else {
        // one slot for fascicles of <= kSlotCap coefficients; the others
        // need each coefficient's occurrence index within its fascicle
        // (stable order): only their coefficients are selected and sorted
        // (at C2 a few percent of Phi instead of all 100M)
        k_vf_identity<<<gridn(n), 256, 0, st>>>(f, phi->b_f2vf, n, vf_o);
        LIFE_CHECK_LAUNCH();
        uint8_t *big;
        uint32_t *bidx, *bf, *sf, *bperm;
        int64_t *nbig;
        LIFE_TRY(talloc((void **)&big, n));
        LIFE_TRY(talloc((void **)&bidx, n * 4));
        LIFE_TRY(talloc((void **)&nbig, 8));
        k_big_flags<<<gridn(n), 256, 0, st>>>(f, fcnt, n, big);
        LIFE_CHECK_LAUNCH();
        {
            cub::CountingInputIterator<uint32_t> pos(0);
            size_t tb = 0;
            LIFE_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pos, big, bidx, nbig, n, st));
            void *temp = nullptr;
            LIFE_CUDA(cudaMallocAsync(&temp, std::max<size_t>(tb, 16), st));
            LIFE_CUDA(cub::DeviceSelect::Flagged(temp, tb, pos, big, bidx, nbig, n, st));
            LIFE_CUDA(cudaFreeAsync(temp, st));
        }
        int64_t m = 0;
        LIFE_CUDA(cudaMemcpyAsync(&m, nbig, 8, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        if (m > 0) {
            LIFE_TRY(talloc((void **)&bf, m * 4));
            LIFE_TRY(talloc((void **)&sf, m * 4));
            LIFE_TRY(talloc((void **)&bperm, m * 4));
            k_gather_u32<<<gridn(m), 256, 0, st>>>(bidx, f, m, bf);
            LIFE_CHECK_LAUNCH();
            LIFE_TRY(sort_pairs<uint32_t>(bf, sf, bidx, bperm, m, bits64((unsigned long long)nf), st));
            k_heads32<<<gridn(m), 256, 0, st>>>(sf, m, head);
            LIFE_CHECK_LAUNCH();
            LIFE_TRY(scan_max(head, rstart, m, st));
            k_vf_split<<<gridn(m), 256, 0, st>>>(bperm, sf, rstart, phi->b_f2vf, m, vf_o);
            LIFE_CHECK_LAUNCH();
        }
    }
    const int nbins = (int)((nvf + kSB - 1) / kSB);

    setup_mark(st, "bin phase 4");
    // 5. bin-major order (bin, tile, chunk), stable; its runs are the
    // segments, each padded to 4 entries in both orders
    unsigned long long *kbm = kva, *skbm = skva, *pay, *spay;
    LIFE_TRY(talloc((void **)&pay, n * 8));
    LIFE_TRY(talloc((void **)&spay, n * 8));
    const int64_t nsteps = ntiles * nch;
    const unsigned long long per_bin = (unsigned long long)ntiles * nch;
    // 32-bit (bin, tile, chunk) keys when they fit: a quarter less sort traffic
    const bool k32 = per_bin * (unsigned long long)nbins <= 0xFFFFFFFFull;
    uint32_t *kbm32 = reinterpret_cast<uint32_t *>(kbm), *skbm32 = reinterpret_cast<uint32_t *>(skbm);
    if (k32) {
        k_key_bm<uint32_t><<<gridn(n), 256, 0, st>>>(a, row_o, vf_o, d_slot, val, n, ka_shift, ka, (uint32_t)nch,
                                                     (uint32_t)ntiles, kbm32, pay);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY((sort_pairs<uint32_t, unsigned long long>(kbm32, skbm32, pay, spay, n, bits64(per_bin * nbins), st)));
    } else {
        k_key_bm<unsigned long long><<<gridn(n), 256, 0, st>>>(a, row_o, vf_o, d_slot, val, n, ka_shift, ka,
                                                               (uint32_t)nch, (uint32_t)ntiles, kbm, pay);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY((sort_pairs<unsigned long long, unsigned long long>(kbm, skbm, pay, spay, n, bits64(per_bin * nbins),
                                                                     st)));
    }
    uint8_t *seghead;
    uint32_t *head32 = head, *segid = rstart, *first;
    int64_t *nsel;
    LIFE_TRY(talloc((void **)&seghead, n));
    LIFE_TRY(talloc((void **)&nsel, 8));
    LIFE_TRY(talloc((void **)&first, n * 4));
    if (k32) k_head_flags<uint32_t><<<gridn(n), 256, 0, st>>>(skbm32, n, seghead, head32);
    else k_head_flags<unsigned long long><<<gridn(n), 256, 0, st>>>(skbm, n, seghead, head32);
    LIFE_CHECK_LAUNCH();
    {
        cub::CountingInputIterator<uint32_t> pos(0);
        size_t t1 = 0, t2 = 0;
        LIFE_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, pos, seghead, first, nsel, n, st));
        LIFE_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t2, head32, segid, n, st));
        void *temp = nullptr;
        LIFE_CUDA(cudaMallocAsync(&temp, std::max(t1, t2), st));
        LIFE_CUDA(cub::DeviceSelect::Flagged(temp, t1, pos, seghead, first, nsel, n, st));
        LIFE_CUDA(cub::DeviceScan::InclusiveSum(temp, t2, head32, segid, n, st));
        LIFE_CUDA(cudaFreeAsync(temp, st));
        g_launches.fetch_add(4, std::memory_order_relaxed);
    }
    int64_t nseg = 0;
    LIFE_CUDA(cudaMemcpyAsync(&nseg, nsel, 8, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    uint32_t *len4, *sstep, *seg_iota, *perm_seg, *tm_excl;
    unsigned long long *segkey, *tmkey, *stmkey;
    unsigned *units, *spad;
    LIFE_TRY(talloc((void **)&len4, (nseg + 1) * 4));
    LIFE_TRY(talloc((void **)&sstep, nseg * 4));
    LIFE_TRY(talloc((void **)&seg_iota, nseg * 4));
    LIFE_TRY(talloc((void **)&perm_seg, nseg * 4));
    LIFE_TRY(talloc((void **)&tm_excl, (nseg + 1) * 4));
    LIFE_TRY(talloc((void **)&segkey, nseg * 8));
    LIFE_TRY(talloc((void **)&tmkey, nseg * 8));
    LIFE_TRY(talloc((void **)&stmkey, nseg * 8));
    LIFE_TRY(talloc((void **)&units, nsteps * 4));
    LIFE_TRY(talloc((void **)&spad, nsteps * 4));
    if (k32)
        k_seg_info<uint32_t><<<gridn(nseg), 256, 0, st>>>(skbm32, first, nseg, n, per_bin, (uint32_t)nbins, len4, segkey,
                                                          tmkey, sstep);
    else
        k_seg_info<unsigned long long><<<gridn(nseg), 256, 0, st>>>(skbm, first, nseg, n, per_bin, (uint32_t)nbins, len4,
                                                                    segkey, tmkey, sstep);
    LIFE_CHECK_LAUNCH();
    // bin-major unit starts
    // +4: the bin side bulk-copies segment records rounded up to 16 bytes
    LIFE_TRY(dalloc(phi, &phi->b_segsrc, (size_t)nseg + 1 + 4));
    LIFE_TRY(scan_excl(len4, phi->b_segsrc, nseg, st));
    // tile-major: steps padded to 8 entries, segments in bin order inside
    LIFE_CUDA(cudaMemsetAsync(units, 0, nsteps * 4, st));
    k_step_units<<<gridn(nseg), 256, 0, st>>>(sstep, len4, nseg, units);
    LIFE_CHECK_LAUNCH();
    k_step_pad<<<gridn(nsteps), 256, 0, st>>>(units, nsteps, spad);
    LIFE_CHECK_LAUNCH();
    LIFE_TRY(dalloc(phi, &phi->b_step, (size_t)nsteps + 1));
    LIFE_TRY(scan_excl(spad, phi->b_step, nsteps, st));
    k_iota<<<gridn(nseg), 256, 0, st>>>(seg_iota, nseg);
    LIFE_CHECK_LAUNCH();
    LIFE_TRY(sort_pairs<unsigned long long>(tmkey, stmkey, seg_iota, perm_seg, nseg, bits64(per_bin * nbins), st));
    {   // tile-major exclusive scan of the segment lengths (in units)
        uint32_t *len_tm = seg_iota;  // reuse
        k_gather_u32<<<gridn(nseg), 256, 0, st>>>(perm_seg, len4, nseg, len_tm);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY(scan_excl(len_tm, tm_excl, nseg, st));
    }
    LIFE_TRY(dalloc(phi, &phi->b_segdst, (size_t)nseg + 1 + 4));
    uint32_t *stepx = (uint32_t *)spad;  // reuse: padded sizes are scanned already
    k_step_first<<<gridn(nseg), 256, 0, st>>>(perm_seg, tm_excl, sstep, nseg, stepx);
    LIFE_CHECK_LAUNCH();
    k_seg_tm<<<gridn(nseg), 256, 0, st>>>(perm_seg, tm_excl, sstep, nseg, phi->b_step, stepx, phi->b_segdst);
    LIFE_CHECK_LAUNCH();
    uint32_t npad = 0, nbm4 = 0;
    LIFE_CUDA(cudaMemcpyAsync(&npad, phi->b_step + nsteps, 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaMemcpyAsync(&nbm4, phi->b_segsrc + nseg, 4, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));

    setup_mark(st, "bin phase 5");
    // 6. placement (pads: cellr kPad, vid kPad, value 0)
    const int64_t nbm = (int64_t)nbm4 * 4;
    LIFE_TRY(dalloc(phi, &phi->b_cellr, (size_t)npad + 8));
    LIFE_TRY(dalloc(phi, &phi->b_scr, (size_t)npad + 8));
    LIFE_TRY(dalloc(phi, &phi->b_vid, (size_t)nbm + 8));
    LIFE_TRY(dalloc(phi, &phi->b_val, (size_t)nbm + 8));
    k_fill_u16<<<gridn(npad + 8), 256, 0, st>>>(phi->b_cellr, (int64_t)npad + 8, (uint16_t)ka);
    LIFE_CHECK_LAUNCH();
    k_fill_u16<<<gridn(nbm + 8), 256, 0, st>>>(phi->b_vid, nbm + 8, kPad);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaMemsetAsync(phi->b_val, 0, ((size_t)nbm + 8) * 4, st));
    LIFE_CUDA(cudaMemsetAsync(phi->b_scr, 0, ((size_t)npad + 8) * 4, st));
    k_place<<<gridn(n), 256, 0, st>>>(spay, segid, first, phi->b_segsrc, phi->b_segdst, n, phi->b_vid, phi->b_val,
                                      phi->b_cellr);
    LIFE_CHECK_LAUNCH();

    setup_mark(st, "bin phase 6");
    // 7. bin and CTA segment ranges of the bin side
    LIFE_TRY(dalloc(phi, &phi->b_binptr, (size_t)nbins + 1));
    k_bin_seg<<<gridn(nbins + 1), 256, 0, st>>>(segkey, nseg, nbins, per_bin, phi->b_binptr);
    LIFE_CHECK_LAUNCH();
    const int side_grid = phi->sms;
    {   // bin-side chunks: per CTA (balanced by units, cut at segment ends),
        // per bin piece, at most kCH units each
        uint32_t *dcs;
        LIFE_TRY(talloc((void **)&dcs, ((size_t)side_grid + 1) * 4));
        k_cta_seg<<<gridn(side_grid + 1), 256, 0, st>>>(phi->b_segsrc, nseg, side_grid, dcs);
        LIFE_CHECK_LAUNCH();
        std::vector<uint32_t> hsrc((size_t)nseg + 1), hbin((size_t)nbins + 1), hcta((size_t)side_grid + 1);
        LIFE_CUDA(cudaMemcpyAsync(hsrc.data(), phi->b_segsrc, hsrc.size() * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaMemcpyAsync(hbin.data(), phi->b_binptr, hbin.size() * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaMemcpyAsync(hcta.data(), dcs, hcta.size() * 4, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        // CTAs are independent: host threads build their chunk lists, which
        // are concatenated in CTA order
        const int nthr = std::max(1, std::min(8, side_grid));
        std::vector<std::vector<uint32_t>> tch(nthr);
        std::vector<std::vector<uint16_t>> tgr(nthr);
        std::vector<std::vector<uint32_t>> tcnt(nthr);  // chunks per CTA
        auto build = [&](int t) {
            const int c0 = side_grid * t / nthr, c1 = side_grid * (t + 1) / nthr;
            auto &chunks = tch[t];
            auto &cgrp = tgr[t];
            int b = (int)(std::upper_bound(hbin.begin(), hbin.end(), hcta[c0]) - hbin.begin()) - 1;
            b = std::max(0, std::min(b, nbins));
            for (int c = c0; c < c1; ++c) {
                const size_t before = chunks.size();
                const uint32_t S0 = hcta[c], S1 = hcta[c + 1];
                uint32_t s = S0;
                while (b < nbins && hbin[b + 1] <= S0) ++b;
                int bb = b;
                while (s < S1) {
                    while (bb < nbins && hbin[bb + 1] <= s) ++bb;
                    const uint32_t pe = std::min(S1, hbin[bb + 1]);
                    const uint32_t pu0 = hsrc[s], pu1 = hsrc[pe];
                    uint32_t sl = s;  // segment containing the chunk start
                    bool first = true;
                    for (uint32_t u0 = pu0; u0 < pu1; u0 += (uint32_t)kCH) {
                        const uint32_t u1 = std::min(pu1, u0 + (uint32_t)kCH);
                        while (hsrc[sl + 1] <= u0) ++sl;
                        uint32_t sh = sl;  // segment containing u1 - 1
                        while (hsrc[sh + 1] < u1) ++sh;
                        const uint32_t ns = sh - sl + 1;
                        // per 32-unit group of the chunk: its first segment
                        for (uint32_t g = 0, k = sl; g < 32; ++g) {
                            const uint32_t ug = u0 + 32u * g;
                            if (ug < u1)
                                while (hsrc[k + 1] <= ug) ++k;
                            cgrp.push_back((uint16_t)(ug < u1 ? k - sl : ns - 1));
                        }
                        chunks.push_back(u0);
                        chunks.push_back((u1 - u0) | (first ? 0x80000000u : 0u));
                        chunks.push_back(sl);
                        chunks.push_back(ns | ((uint32_t)bb << 16));
                        first = false;
                    }
                    s = pe;
                }
                tcnt[t].push_back((uint32_t)((chunks.size() - before) / 4));
            }
        };
        {
            std::vector<std::thread> pool;
            for (int t = 1; t < nthr; ++t) pool.emplace_back(build, t);
            build(0);
            for (auto &th : pool) th.join();
        }
        std::vector<uint32_t> chunks, ctachunk(1, 0);
        std::vector<uint16_t> cgrp;
        for (int t = 0; t < nthr; ++t) {
            chunks.insert(chunks.end(), tch[t].begin(), tch[t].end());
            cgrp.insert(cgrp.end(), tgr[t].begin(), tgr[t].end());
            for (uint32_t k : tcnt[t]) ctachunk.push_back(ctachunk.back() + k);
        }
        if (chunks.empty()) {
            chunks.assign(4, 0u);
            cgrp.assign(32, 0);
        }
        LIFE_TRY(dalloc(phi, &phi->b_chunks, chunks.size()));
        LIFE_TRY(dalloc(phi, &phi->b_cgrp, cgrp.size()));
        LIFE_CUDA(cudaMemcpyAsync(phi->b_cgrp, cgrp.data(), cgrp.size() * 2, cudaMemcpyHostToDevice, st));
        LIFE_TRY(dalloc(phi, &phi->b_ctachunk, ctachunk.size()));
        LIFE_CUDA(cudaMemcpyAsync(phi->b_chunks, chunks.data(), chunks.size() * 4, cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaMemcpyAsync(phi->b_ctachunk, ctachunk.data(), ctachunk.size() * 4, cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
    }

    setup_mark(st, "bin phase 7");
    // 8. dictionary chunks as the two B operands: f16 hi | lo of D * kDScale,
    // K-major SWIZZLE_128B (64 f16 per 128-byte row)
    {
        const int nkb = (N + 63) / 64;
        const size_t pd = (size_t)2 * N * ka, pw = (size_t)2 * nkb * ka * 64;  // halves per chunk
        std::vector<uint16_t> hd((size_t)nch * pd, 0), hw((size_t)nch * pw, 0);
        for (int c = 0; c < nch; ++c)
            for (int k = 0; k < ka; ++k) {
                const int at = c * ka + k;
                for (int t = 0; t < N; ++t) {
                    const float x = (at < phi->na && t < phi->nt) ? (float)hdict[(size_t)at * phi->nt + t] * 256.f : 0.f;
                    const __half h = __float2half_rn(x), l = __float2half_rn(x - __half2float(h));
                    const uint16_t hb = __half_as_ushort(h), lb = __half_as_ushort(l);
                    // DSC: rows = directions, K = the chunk's 64 atoms
                    const size_t od = (size_t)c * pd + sw16(t, k) / 2;
                    hd[od] = hb;
                    hd[od + (size_t)N * ka] = lb;
                    // WC: rows = atoms, K = directions in blocks of 64
                    const size_t ow = (size_t)c * pw + (size_t)(t / 64) * ka * 64 + sw16(k, t % 64) / 2;
                    hw[ow] = hb;
                    hw[ow + (size_t)nkb * ka * 64] = lb;
                }
            }
        LIFE_TRY(dalloc(phi, &phi->b_Ddsc, hd.size()));
        LIFE_TRY(dalloc(phi, &phi->b_Dwc, hw.size()));
        LIFE_CUDA(cudaMemcpyAsync(phi->b_Ddsc, hd.data(), hd.size() * 2, cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaMemcpyAsync(phi->b_Dwc, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
    }

    {   // per-fascicle int64 sums, then the non-finite flags (bytes) in the
        // same buffer so one all-reduce carries both
        const size_t words = (size_t)nf + ((size_t)nf + 7) / 8 + 3 * (size_t)kTailRanks;
        LIFE_TRY(dalloc(phi, &phi->b_wfix, words));
        phi->b_nanf = reinterpret_cast<unsigned char *>(phi->b_wfix + nf);
        LIFE_CUDA(cudaMemsetAsync(phi->b_wfix, 0, words * 8, st));
    }
    phi->b_ka = ka;
    phi->b_n = N;
    phi->b_nch = nch;
    phi->b_ntiles = (int)ntiles;
    phi->b_nbins = nbins;
    phi->b_sb = kSB;
    phi->b_nvf = nvf;
    phi->b_nsteps = nsteps;
    phi->b_nseg = nseg;
    phi->b_npad = npad;
    phi->b_tile_grid = (int)std::min<int64_t>(phi->sms, ntiles);
    phi->b_side_grid = side_grid;
    LIFE_TRY(dalloc(phi, &phi->b_skip, (size_t)phi->b_side_grid));
    LIFE_TRY(dalloc(phi, &phi->b_smax, (size_t)phi->b_side_grid));
    LIFE_TRY(dalloc(phi, &phi->b_nonfin, 1));
    LIFE_CUDA(cudaMemsetAsync(phi->b_nonfin, 0, 4, st));
    LIFE_CUDA(cudaMemsetAsync(phi->b_skip, 0, (size_t)phi->b_side_grid * 8, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    LIFE_TRY(prepare_bin(phi));
    phi->has_bin = true;
    if (getenv("LIFE_DEBUG"))
        fprintf(stderr, "[life] bin layout: N=%d KA=%d rows=%u tiles=%lld nch=%d nbins=%d nvf=%u steps=%lld "
                        "segs=%lld padded=%u/%lld split voxels=%d\n",
                N, ka, R, (long long)ntiles, nch, nbins, nvf, (long long)nsteps, (long long)nseg, npad,
                (long long)nbm, phi->b_nfix);
    return LIFE_OK;
}


// ===========================================================================
// bin side (streaming; per-coefficient random access in shared memory)
// ===========================================================================
namespace bin {

struct SideArgs {
    const uint16_t *vid;     // bin-major virtual slot within the bin (kPad = pad)
    const float *val;        // bin-major values (0 at pads)
    const uint32_t *src4;    // [nseg + 1] bin-major segment starts, 4-entry units
    const uint32_t *dst4;    // [nseg] tile-major segment starts, 4-entry units
    const uint32_t *binseg;  // [nbins + 1] first segment of each bin
    const uint32_t *vf2f;    // [nvf]
    int64_t nvf;
    int nbins;
};

constexpr int kSideUN = 4;   // 4-entry units per lane in flight

// Segment groups: a warp takes 32 consecutive segments of a bin piece (lane =
// segment record), an inclusive scan of their unit counts, and walks the
// group's units 32 * kSideUN at a time; each lane finds its unit's segment
// with a 5-step shuffle search, so no dependent global loads are on the path.
struct Group {
    uint32_t src, dst, P;  // this lane's segment: starts (units), inclusive prefix of unit counts
    uint32_t tot;          // units in the group
};
__device__ __forceinline__ Group load_group(const SideArgs &A, uint32_t gs, uint32_t pe, int lane)
{
    const uint32_t si = gs + (uint32_t)lane;
    Group g;
    g.src = si < pe ? __ldg(A.src4 + si) : 0u;
    const uint32_t n4 = si < pe ? __ldg(A.src4 + si + 1) - g.src : 0u;
    g.dst = si < pe ? __ldg(A.dst4 + si) : 0u;
    uint32_t P = n4;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, P, o);
        if (lane >= o) P += x;
    }
    g.P = P;
    g.tot = __shfl_sync(0xffffffffu, P, 31);
    return g;
}
// bin-major and tile-major unit of the group's unit u (all lanes call)
__device__ __forceinline__ void unit_of(const Group &g, uint32_t u, uint32_t &su, uint32_t &du)
{
    int sl = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t pv = __shfl_sync(0xffffffffu, g.P, sl + step - 1);
        if (pv <= u) sl += step;
    }
    sl = min(sl, 31);
    const uint32_t ex = __shfl_sync(0xffffffffu, g.P, max(sl - 1, 0));
    const uint32_t off = u - (sl ? ex : 0u);
    su = __shfl_sync(0xffffffffu, g.src, sl) + off;
    du = __shfl_sync(0xffffffffu, g.dst, sl) + off;
}
__device__ __forceinline__ int find_bin(const uint32_t *binseg, int nbins, uint32_t s)
{
    int lo = 0, hi = nbins;  // largest b with binseg[b] <= s
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(binseg + mid) <= s) lo = mid; else hi = mid;
    }
    return lo;
}

// Bin side, streamed: the CTA's bin-major range is cut (at build time) into
// chunks of at most kCH 4-entry units inside one bin; a producer warp stages
// each chunk's ids, values and segment records into a shared-memory ring with
// bulk copies (kNS in flight), so memory traffic is decoupled from the
// consumers' per-entry work.  Chunk descriptor (uint4): x = first unit, y =
// units | first-of-piece << 31, z = first segment, w = segments | bin << 16.
constexpr int kSideThreads = 1024;        // warp 0 produces, warps 1..31 consume
constexpr int kCons = kSideThreads - 32;
static_assert(kCH % 32 == 0 && kCH <= 1024, "a chunk's group table has 32 entries of 32 units");
// slot regions (16-byte aligned bulk-copy destinations; each holds its range
// plus the alignment slack of an unaligned global start)
constexpr uint32_t kSlotVid = 0, kSlotVal = (kCH * 8 + 16 + 15) / 16 * 16, kSlotSrc = kSlotVal + kCH * 16,
                   kSlotDst = kSlotSrc + ((kCH + 2) * 4 + 16 + 15) / 16 * 16,
                   kSlotGrp = kSlotDst + ((kCH + 1) * 4 + 16 + 15) / 16 * 16,
                   kSlotBytes = (kSlotGrp + 64 + 127) / 128 * 128;
#ifndef LIFE_NS_DSC
#define LIFE_NS_DSC 4  // 5 fits with kCH = 992 but measured no faster
#endif
constexpr int kNsDsc = LIFE_NS_DSC, kNsWc = 3;

struct ChunkArgs {
    const uint4 *chunks;      // chunk descriptors
    const uint32_t *ctachunk; // [grid + 1]
    const uint16_t *grp;      // [chunks][32] first segment (chunk-relative) of each 32-unit group
};

// producer: stage chunk j of the CTA into slot j % NS (header: byte offsets of
// the unaligned starts)
template <int NS, int CAT>
__device__ __forceinline__ void side_produce(const SideArgs &A, const uint4 *tab, const uint16_t *grp, int nch,
                                             unsigned char *ring, uint4 (*hdr)[2], uint64_t *full, uint64_t *empty)
{
    BD_DECL;
    const uint64_t pol = pol_first();
    uint4 cn = nch > 0 ? __ldg(tab) : make_uint4(0, 0, 0, 0), cnn = nch > 1 ? __ldg(tab + 1) : cn;
    for (int j = 0; j < nch; ++j) {
        const int sl = j % NS;
        const uint4 c = cn;  // descriptors prefetched two chunks ahead
        cn = cnn;
        if (j + 2 < nch) cnn = __ldg(tab + j + 2);
        if (j >= NS) BD_WAIT(CAT, bar_wait(&empty[sl], ((j / NS) - 1) & 1));
        const uint32_t u0 = c.x, nu = c.y & 0x7FFFFFFFu, s0 = c.z, ns = c.w & 0xFFFFu;
        unsigned char *slot = ring + (size_t)sl * kSlotBytes;
        const uint64_t vb0 = 8ull * u0, vb1 = 8ull * (u0 + nu);
        const uint64_t va = vb0 & ~15ull, vz = (vb1 + 15) & ~15ull;
        const uint64_t sb0 = 4ull * s0, sb1 = 4ull * (s0 + ns + 1);
        const uint64_t sa0 = sb0 & ~15ull, sz = (sb1 + 15) & ~15ull;
        const uint64_t db1 = 4ull * (s0 + ns);
        const uint64_t dz = (db1 + 15) & ~15ull;
        hdr[sl][0] = c;  // the descriptor and the byte offsets of the unaligned starts
        hdr[sl][1] = make_uint4((uint32_t)(vb0 - va), (uint32_t)(sb0 - sa0), 0u, 0u);
        const unsigned bytes = (unsigned)((vz - va) + 16ull * nu + (sz - sa0) + (dz - sa0) + 64ull);
        bar_arrive_tx(&full[sl], bytes);
        bulk_g2s(slot + kSlotVid, reinterpret_cast<const unsigned char *>(A.vid) + va, (unsigned)(vz - va), &full[sl], pol);
        bulk_g2s(slot + kSlotVal, reinterpret_cast<const unsigned char *>(A.val) + 16ull * u0, 16u * nu, &full[sl], pol);
        bulk_g2s(slot + kSlotSrc, reinterpret_cast<const unsigned char *>(A.src4) + sa0, (unsigned)(sz - sa0), &full[sl], pol);
        bulk_g2s(slot + kSlotDst, reinterpret_cast<const unsigned char *>(A.dst4) + sa0, (unsigned)(dz - sa0), &full[sl], pol);
        bulk_g2s(slot + kSlotGrp, reinterpret_cast<const unsigned char *>(grp + 32ull * j), 64u, &full[sl], pol);
    }
    BD_FLUSH;
}

// consumer: tile-major unit of chunk unit u (staged segment records): the
// segment lies between the first segments of u's 32-unit group and of the
// next group (build-time table); usually one or two candidates, at most 32
// when a sparse bin has one-unit segments (binary search)
__device__ __forceinline__ uint32_t side_dst(uint32_t slot_sa, uint32_t hs, uint32_t u0, uint32_t ns, uint32_t u)
{
    const uint32_t U = u0 + u;
    const uint32_t src = slot_sa + kSlotSrc + hs, dst = slot_sa + kSlotDst + hs;
    const uint32_t g = u >> 5;
    uint32_t lo, hi;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(lo) : "r"(slot_sa + kSlotGrp + 2u * g));
    if (g < 31) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(hi) : "r"(slot_sa + kSlotGrp + 2u * g + 2u));
    else hi = ns - 1;
    while (hi > lo) {  // largest k in [lo, hi] with src4[k] <= U
        const uint32_t mid = (lo + hi + 1) >> 1;
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(src + 4u * mid));
        if (v <= U) lo = mid; else hi = mid - 1;
    }
    uint32_t s0, d0;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(s0) : "r"(src + 4u * lo));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d0) : "r"(dst + 4u * lo));
    return d0 + (U - s0);
}

// DSC bin side: scr[tile-major] = s = w[f] * value, exact skip count (fp32
// s == 0, _kernels.py:24-28), max |s| and a non-finite flag
__global__ void __launch_bounds__(kSideThreads, 1)
    k_side_dsc(const SideArgs A, const ChunkArgs CA, const float *__restrict__ w, float *__restrict__ scr,
               int count_skips, unsigned long long *__restrict__ skip_part, float *__restrict__ smax_part,
               unsigned *__restrict__ nonfinite, const CallHooks hooks)
{
    extern __shared__ __align__(128) unsigned char side_sm[];
    __shared__ __align__(8) uint64_t full[kNsDsc], empty[kNsDsc];
    __shared__ uint4 hdr[kNsDsc][2];
    if (hooks.done && *hooks.done) return;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    float *ws = reinterpret_cast<float *>(side_sm);  // kSB
    unsigned char *ring = side_sm + kSB * 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = (int)__ldg(CA.ctachunk + blockIdx.x), nch = (int)__ldg(CA.ctachunk + blockIdx.x + 1) - c0;
    const uint4 *tab = CA.chunks + c0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kNsDsc; ++i) {
            bar_init(&full[i], 1);
            bar_init(&empty[i], kCons / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long zeros = 0;
    float smax = 0.f;
    bool nonfin = false;
    if (warp == 0) {
        if (lane == 0) side_produce<kNsDsc, 15>(A, tab, CA.grp + 32ull * c0, nch, ring, hdr, full, empty);
    } else {
        const uint32_t ct = threadIdx.x - 32;
        BD_DECL;
        for (int j = 0; j < nch; ++j) {
            const int sl = j % kNsDsc;
            BD_WAIT(13, bar_wait(&full[sl], (j / kNsDsc) & 1));
            BD_T0(t_p);
            const uint4 c = hdr[sl][0];
            const uint32_t u0 = c.x, nu = c.y & 0x7FFFFFFFu, ns = c.w & 0xFFFFu;
            if (c.y >> 31) {  // a new bin: its w slice into shared memory
                const int64_t s0 = (int64_t)(c.w >> 16) * kSB;
                const int nsl = (int)min((int64_t)kSB, A.nvf - s0);
                named_bar(1, kCons);
                // the bin's w slice: 8 independent gathers in flight per thread
                for (int i0 = ct; i0 < nsl; i0 += 8 * kCons) {
                    uint32_t fi[8];
                    float wv[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int i = i0 + k * kCons;
                        fi[k] = i < nsl ? __ldg(A.vf2f + s0 + i) : 0u;
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) wv[k] = i0 + k * kCons < nsl ? __ldg(w + fi[k]) : 0.f;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (i0 + k * kCons < nsl) ws[i0 + k * kCons] = wv[k];
                }
                named_bar(1, kCons);
            }
            const uint32_t slot_sa = sa(ring) + (uint32_t)sl * kSlotBytes;
            const uint32_t hv = hdr[sl][1].x, hs = hdr[sl][1].y;
            for (uint32_t u = ct; u < nu; u += kCons) {
                const uint32_t du = side_dst(slot_sa, hs, u0, ns, u);
                uint2 id;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(id.x), "=r"(id.y) : "r"(slot_sa + kSlotVid + hv + 8u * u));
                const float4 vv = lds_f4(slot_sa + kSlotVal + 16u * u);
                const uint32_t ids[4] = {id.x & 0xFFFFu, id.x >> 16, id.y & 0xFFFFu, id.y >> 16};
                const float vs[4] = {vv.x, vv.y, vv.z, vv.w};
                float o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool pad = ids[e] == kPad;
                    o[e] = pad ? 0.f : __fmul_rn(ws[pad ? 0 : ids[e]], vs[e]);
                    zeros += (!pad && o[e] == 0.f) ? 1ull : 0ull;
                    if (isfinite(o[e])) smax = fmaxf(smax, fabsf(o[e]));
                    else nonfin = true;
                }
                reinterpret_cast<float4 *>(scr)[du] = make_float4(o[0], o[1], o[2], o[3]);
            }
            BD_ACC(14, t_p);
            __syncwarp();
            if (lane == 0) bar_arrive(&empty[sl]);
        }
        BD_FLUSH;
    }
    // this call's non-finite flag (read by the tile kernel, cleared by the
    // CTA that finishes the call); per-CTA skip count and max |s|
    if (__any_sync(0xffffffffu, nonfin) && lane == 0) atomicAdd(nonfinite, 1u);
    __shared__ unsigned long long sz[32];
    __shared__ float smx[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
        smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    }
    if (lane == 0) {
        sz[warp] = zeros;
        smx[warp] = smax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        float m = 0.f;
        for (int i = 0; i < 32; ++i) {
            t += sz[i];
            m = fmaxf(m, smx[i]);
        }
        skip_part[blockIdx.x] = count_skips ? t : 0ull;
        smax_part[blockIdx.x] = m;
    }
}

// WC bin side: fascicle sums of value * z in 64-bit fixed point, two 32-bit
// limbs per virtual slot in shared memory (native u32 atomics: order
// independent, exact), flushed per bin piece into wfix (int64 atomics, also
// exact).  The consumers load the next chunk's z (tile-major scratch) while
// accumulating the current one.
__global__ void __launch_bounds__(kSideThreads, 1)
    k_side_wc(const SideArgs A, const ChunkArgs CA, const float *__restrict__ scr, const FixParams fx, int nt,
              unsigned long long *__restrict__ wfix, unsigned char *__restrict__ nanf, const CallHooks hooks)
{
    extern __shared__ __align__(128) unsigned char side_sm[];
    __shared__ __align__(8) uint64_t full[kNsWc], empty[kNsWc];
    __shared__ uint4 hdr[kNsWc][2];
    if (hooks.done && *hooks.done) return;
    uint32_t *lo = reinterpret_cast<uint32_t *>(side_sm), *hi = lo + kSB;
    unsigned char *ring = side_sm + kSB * 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = (int)__ldg(CA.ctachunk + blockIdx.x), nch = (int)__ldg(CA.ctachunk + blockIdx.x + 1) - c0;
    const uint4 *tab = CA.chunks + c0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kNsWc; ++i) {
            bar_init(&full[i], 1);
            bar_init(&empty[i], kCons / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) side_produce<kNsWc, 31>(A, tab, CA.grp + 32ull * c0, nch, ring, hdr, full, empty);
        return;
    }
    const uint32_t ct = threadIdx.x - 32;
    // fixed point in fp32 arithmetic (no 64-bit conversions): x = rint(t 2^e)
    // is exact (|x| < 2^45, power-of-two scaling split so neither factor
    // overflows), hi = floor(x / 2^24) and lo = x - hi 2^24 in [0, 2^24) are
    // exact integers in float; identical to __double2ll_rn((double)t * 2^e)
    // (ex > 252 only when every finite term is 0 in fp32: clamped, sc2 stays finite)
    const int ex = min(bin_exponent_dev(fx, nt), 252);
    const int ex1 = ex > 126 ? 126 : ex < -126 ? -126 : ex;
    const float sc1 = ldexpf(1.f, ex1), sc2 = ldexpf(1.f, ex - ex1);
    constexpr int UPT = (kCH + kCons - 1) / kCons;  // units per consumer thread per chunk
    float4 zc[UPT], zn[UPT];
    // z of chunk j (its records are staged) into z[]
    BD_DECL;
    auto load_z = [&](int j, float4 (&z)[UPT]) {
        const int sl = j % kNsWc;
        BD_WAIT(30, bar_wait(&full[sl], (j / kNsWc) & 1));
        const uint4 c = hdr[sl][0];
        const uint32_t u0 = c.x, nu = c.y & 0x7FFFFFFFu, ns = c.w & 0xFFFFu;
        const uint32_t slot_sa = sa(ring) + (uint32_t)sl * kSlotBytes, hs = hdr[sl][1].y;
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
            const uint32_t u = ct + (uint32_t)(kCons * i);
            if (u < nu) z[i] = __ldcs(reinterpret_cast<const float4 *>(scr) + side_dst(slot_sa, hs, u0, ns, u));
        }
    };
    int cur_bin = -1;
    // flush a bin piece into the per-fascicle sums: the virtual slots of a
    // fascicle are consecutive, so a warp first sums its runs (segmented
    // suffix scan) and only run heads issue the int64 atomic
    auto flush = [&]() {
        const int64_t s0 = (int64_t)cur_bin * kSB;
        const int nsl = (int)min((int64_t)kSB, A.nvf - s0);
        constexpr int kFU = 4;  // flush rounds with their fascicle ids loaded together
        for (int ib0 = (int)ct - lane; ib0 < nsl; ib0 += kFU * kCons) {
          uint32_t fids[kFU];
#pragma unroll
          for (int r = 0; r < kFU; ++r) {
              const int i = ib0 + r * kCons + lane;
              fids[r] = i < nsl ? __ldg(A.vf2f + s0 + i) : 0xFFFFFFFFu;
          }
#pragma unroll
          for (int r = 0; r < kFU; ++r) {
            const int ib = ib0 + r * kCons;
            if (ib >= nsl) break;  // warp-uniform
            const int i = ib + lane;
            long long v = 0;
            const uint32_t fid = fids[r];
            if (i < nsl) v = (long long)(int32_t)hi[i] * 16777216ll + (long long)lo[i];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long ov = __shfl_down_sync(0xffffffffu, v, o);
                const uint32_t of = __shfl_down_sync(0xffffffffu, fid, o);
                if (lane + o < 32 && of == fid) v += ov;
            }
            const uint32_t pf = __shfl_up_sync(0xffffffffu, fid, 1);
            if (i < nsl && (lane == 0 || pf != fid) && v) atomicAdd(wfix + fid, (unsigned long long)v);
          }
        }
    };
    if (nch > 0) load_z(0, zn);
    for (int j = 0; j < nch; ++j) {
        const int sl = j % kNsWc;
        const uint4 c = hdr[sl][0];  // chunk j is staged (load_z waited for it)
        const uint32_t nu = c.y & 0x7FFFFFFFu;
#pragma unroll
        for (int i = 0; i < UPT; ++i) zc[i] = zn[i];
        if (c.y >> 31) {  // a new bin: flush the previous one, clear the limbs
            named_bar(1, kCons);
            if (cur_bin >= 0) flush();
            named_bar(1, kCons);
            cur_bin = (int)(c.w >> 16);
            const int nsl = (int)min((int64_t)kSB, A.nvf - (int64_t)cur_bin * kSB);
            for (int i = ct; i < nsl; i += kCons) {
                lo[i] = 0u;
                hi[i] = 0u;
            }
            named_bar(1, kCons);
        }
        if (j + 1 < nch) load_z(j + 1, zn);  // next chunk's z, in flight meanwhile
        BD_T0(t_p);
        const uint32_t slot_sa = sa(ring) + (uint32_t)sl * kSlotBytes, hv = hdr[sl][1].x;
        const int64_t s0 = (int64_t)cur_bin * kSB;
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
            const uint32_t u = ct + (uint32_t)(kCons * i);
            if (u >= nu) continue;
            uint2 id;
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(id.x), "=r"(id.y) : "r"(slot_sa + kSlotVid + hv + 8u * u));
            const float4 vv = lds_f4(slot_sa + kSlotVal + 16u * u);
            const uint32_t ids[4] = {id.x & 0xFFFFu, id.x >> 16, id.y & 0xFFFFu, id.y >> 16};
            const float vs[4] = {vv.x, vv.y, vv.z, vv.w};
            const float zs[4] = {zc[i].x, zc[i].y, zc[i].z, zc[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (ids[e] == kPad) continue;
                const float t = __fmul_rn(zs[e], vs[e]);  // acc * value (_kernels.py:67)
                if (!isfinite(t)) {
                    nanf[__ldg(A.vf2f + s0 + ids[e])] = 1;
                    continue;
                }
                const float x = rintf(__fmul_rn(__fmul_rn(t, sc1), sc2));
                const float hf = floorf(__fmul_rn(x, 0x1p-24f));
                const float lf = __fsub_rn(x, __fmul_rn(hf, 0x1p24f));
                atomicAdd(lo + ids[e], (uint32_t)lf);
                atomicAdd(hi + ids[e], (uint32_t)(int32_t)hf);
            }
        }
        BD_ACC(9, t_p);
        __syncwarp();
        if (lane == 0) bar_arrive(&empty[sl]);
    }
    named_bar(1, kCons);
    if (cur_bin >= 0) flush();
    BD_FLUSH;
}

// WC finish: per-fascicle int64 sums (all-reduced first on multi-GPU runs)
// to fp32, the non-finite flags, accumulate / project, sum of squares; clears
// the sums and flags for the next call.
template <int BT>
__global__ void __launch_bounds__(BT)
    k_wc_fin(unsigned long long *__restrict__ wfix, unsigned char *__restrict__ nanf, int nf, float *__restrict__ w_out,
             const float *__restrict__ w_ref, uint32_t flags, const FixParams fx, int nt, double *part, unsigned *counter,
             double *sumsq_out, const CallHooks hooks)
{
    if (hooks.done && *hooks.done) return;
    const double inv = ldexp(1.0, -bin_exponent_dev(fx, nt));
    const bool accumulate = flags & LIFE_ACCUMULATE;
    const bool project = (flags & LIFE_PROJECT_GRAD) && w_ref != nullptr;
    double sq = 0.0;
    constexpr int U = 4;  // fascicles in flight per thread
    const int stride = gridDim.x * BT;
    for (int f0 = blockIdx.x * BT + threadIdx.x; f0 < nf; f0 += U * stride) {
        long long q[U];
        bool bad[U];
        float acc[U], ref[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int f = f0 + k * stride;
            q[k] = f < nf ? (long long)wfix[f] : 0ll;
            bad[k] = f < nf && nanf[f] != 0;
            acc[k] = (accumulate && f < nf) ? w_out[f] : 0.f;
            ref[k] = (project && f < nf) ? w_ref[f] : 1.f;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int f = f0 + k * stride;
            if (f >= nf) break;
            wfix[f] = 0ull;
            if (bad[k]) nanf[f] = 0;
            float o = bad[k] ? __int_as_float(0x7fc00000) : (float)((double)q[k] * inv);
            if (accumulate) o = acc[k] + o;
            if (project && ref[k] == 0.f && o > 0.f) o = 0.f;
            w_out[f] = o;
            sq += (double)o * (double)o;
        }
    }
    // block partial: warp shuffles, then the warps in order
    __shared__ double s[BT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < BT / 32; ++i) t += s[i];
        part[blockIdx.x] = t;
    }
    if (last_cta(counter)) {
        const double tot = block_reduce<double>(part, gridDim.x, 0.0, OpSum{}, BT);
        if (threadIdx.x == 0) {
            if (sumsq_out) *sumsq_out = tot;
            *counter = 0;
            if (hooks.t_accum && hooks.t_begin) *hooks.t_accum += globaltimer() - *hooks.t_begin;
        }
    }
}

// ===========================================================================
// tile side (tcgen05)
// ===========================================================================
struct TileArgs {
    const uint16_t *cellr;  // tile-major: C/Z tile word offset row * kCS + atom % kKA (pads: kKA)
    const uint32_t *step;   // [nsteps + 1]
    const uint16_t *D;      // dictionary chunks: product-specific B operand, f16 hi | lo, x kDScale
    const int *rowvox;      // [ntiles * 128]
    const int *rowpart;     // [ntiles * 128]
    float *ypart;           // [nprow * N]
    int ntiles, nch, nt;
};

constexpr int kKA = 64;            // atoms per step: one 128-byte row of f16
constexpr int kCS = kKA + 4;       // C / Z tile row stride (words): conflict-free row reads
constexpr int kUMax = 4;           // 4-entry units per thread prefetched one step ahead
constexpr float kDScale = 256.f;   // dictionary pre-scale (keeps the f16 lo parts normal)

__device__ __forceinline__ uint64_t idesc_f16(int m, int n)
{
    return (uint64_t)((1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24));
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tm_st8(uint32_t addr, const uint32_t (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
// x = hi + lo in f16 (2 x 11 significant bits); returns the packed pair words
__device__ __forceinline__ void split2(float x0, float x1, uint32_t &hi, uint32_t &lo)
{
    const __half2 h = __floats2half2_rn(x0, x1);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
    hi = *reinterpret_cast<const uint32_t *>(&h);
    lo = *reinterpret_cast<const uint32_t *>(&l);
}

#ifndef LIFE_DSC_FOLD1
#define LIFE_DSC_FOLD1 2
#endif
template <int N>
struct DscCfg {
    static constexpr int EQ = (N + 63) / 64;   // epilogue warps per TMEM lane quarter
    static constexpr int kNB = 16;             // builder warps: two groups of 8 on alternating steps
    static constexpr int kProdD = kNB;         // dictionary chunks
    static constexpr int kMma = kNB + 1;       // two issuers: even / odd steps (= builder groups)
    static constexpr int kProdS = kNB + 3;     // step entries into the groups' slots
    static constexpr int kEpi = kNB + 4;
    static constexpr int kWarps = kEpi + 4 * EQ;
    static constexpr int kThreads = kWarps * 32;
    static constexpr int DB = 2 * N * 128;     // one chunk: N rows x 64 f16, hi | lo
    static constexpr int CBytes = kTV * kCS * 4;
    static constexpr int NBLK = N / 16;
    static constexpr int MB = (NBLK + EQ - 1) / EQ;
    static constexpr int TACC = 128;           // TMEM: A stage e at 64 e (hi 32 cols | lo 32), accumulators from TACC
    static constexpr int NACC = TACC + 4 * N <= 512 ? 2 : 1;  // accumulator buffers per issuer
    // an issuer's own steps accumulated in TMEM per epilogue fold: 2 (128
    // atoms); with a single accumulator buffer (N > 128) the issuer waits
    // for every fold (LIFE_DSC_FOLD1)
    static constexpr int FOLD = NACC == 2 ? 2 : LIFE_DSC_FOLD1;
    static constexpr int kSlotsG = 2;          // staged steps per builder group
    static_assert(TACC + 2 * NACC * N <= 512, "TMEM budget");
};

// WC tile: Z tiles in a ring of 3 (2 when shared memory is short), and the
// accumulator released as soon as Z is in registers (C2 WC 0.499 -> 0.490 ms)
#ifndef LIFE_WC_NZ
#define LIFE_WC_NZ 3
#endif
#ifndef LIFE_WC_EARLY
#define LIFE_WC_EARLY 1
#endif
template <int N>
struct WcCfg {
    static constexpr int NKB = (N + 63) / 64;  // 64-direction K blocks of the B operand
    static constexpr int kProdD = kBuild;
    static constexpr int kMma = kBuild + 1;    // two issuers
    static constexpr int kYZ = kBuild + 3;     // 8 warps: two per TMEM lane quarter
    static constexpr int kWarps = kYZ + 8;
    static constexpr int kThreads = kWarps * 32;
    static constexpr int DB = 2 * NKB * kKA * 128;
    static constexpr int ZBytes = kTV * kCS * 4;
    // shared-memory Z tiles between the YZ warps and the gatherers (ring of NZ)
    static constexpr int NZ = 1024 + 2 * DB + LIFE_WC_NZ * ZBytes <= 232448 - 2048 ? LIFE_WC_NZ : 2;
    static constexpr int TZ = N;               // TMEM: Y hi at 0 (N/2 cols), lo at N/2, Z buffer e at TZ + e kKA
    static_assert(N + 2 * kKA <= 512, "TMEM budget");
};

__device__ __forceinline__ unsigned char *align1024(unsigned char *p)
{
    return (unsigned char *)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

// (tile, chunk) walk of a CTA's steps without divisions: step k is chunk
// k % nch of tile blockIdx.x + (k / nch) * gridDim.x
struct StepIter {
    int c, nch;
    size_t gs, tile_stride;
    __device__ StepIter(int k, int nch_) : c(k % nch_), nch(nch_)
    {
        gs = ((size_t)blockIdx.x + (size_t)(k / nch_) * gridDim.x) * nch_ + c;
        tile_stride = (size_t)gridDim.x * nch_;
    }
    __device__ __forceinline__ void next()
    {
        ++gs;
        if (++c == nch) {
            c = 0;
            gs += tile_stride - nch;
        }
    }
};

// One step's entries, prefetched into registers one step ahead (4 per unit)
constexpr int kUBld = 2;  // units per DSC builder thread prefetched (16 builder warps)
struct StepRegs {
    uint32_t p0, n;
    uint2 c[kUBld];
    float4 s[kUBld];
};

// voxels split over several tile rows: sum their partial rows in row order
// and apply the epilogue; then the DSC outputs over all partials
// final value of y[vx, col] from its folded sum
__device__ __forceinline__ void fix_store(float r, size_t o, float *__restrict__ y, const float *__restrict__ b,
                                          bool accumulate, bool subtract, double &sq, float &amax)
{
    if (accumulate) r += y[o];
    if (subtract) r -= b[o];
    y[o] = r;
    sq += (double)r * (double)r;
    amax = fmaxf(amax, fabsf(r));
}

// per-CTA (sum of squares, max) into the reduction slot part
__device__ __forceinline__ void fix_partial(double sq, float amax, const ReduceSlots &red, int part)
{
    __shared__ double s_sq[32];
    __shared__ float s_mx[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    if (lane == 0) {
        s_sq[warp] = sq;
        s_mx[warp] = amax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        float m = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            t += s_sq[i];
            m = fmaxf(m, s_mx[i]);
        }
        red.part_d[part] = t;
        red.part_f[part] = m;
    }
}

// pieces p0, p0 + pstride, ... of the split voxels (one warp each)
template <int N>
__device__ __forceinline__ void fix_pieces(const uint4 *__restrict__ pcs, int npc, const float *__restrict__ ypart,
                                           int nt, float *__restrict__ fixsum, float *__restrict__ y,
                                           const float *__restrict__ b, bool accumulate, bool subtract, int p0,
                                           int pstride, int lane, double &sq, float &amax)
{
    for (int p = p0; p < npc; p += pstride) {
        const uint4 d = __ldg(pcs + p);  // voxel, first row, end row, piece-sum slot (or ~0: final)
        // all of the lane's columns and 4 partial rows in flight per round
        // (the sums still run in row order: same bits as a plain loop)
        constexpr int CPL = (N + 31) / 32;
        float r[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) r[c] = 0.f;
        for (uint32_t q0 = d.y; q0 < d.z; q0 += 4) {
            float v[4][CPL];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const int col = lane + 32 * c;
                    v[k][c] = (q0 + k < d.z && col < nt) ? __ldcg(ypart + (size_t)(q0 + k) * N + col) : 0.f;
                }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (q0 + k < d.z)
#pragma unroll
                    for (int c = 0; c < CPL; ++c) r[c] += v[k][c];
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const int col = lane + 32 * c;
            if (col >= nt) continue;
            if (d.w != 0xFFFFFFFFu) fixsum[(size_t)d.w * N + col] = r[c];
            else fix_store(r[c], (size_t)d.x * nt + col, y, b, accumulate, subtract, sq, amax);
        }
    }
}

// DSC tile side.  Roles (warps):
//   0-7   builders: per step, C[row, atom] = sum of s as 32-bit fixed point
//         (red.shared.add.u32: order independent, deterministic) from entries
//         prefetched into registers one step ahead (L2-prefetched three
//         ahead); then each thread converts its (row, 32 atoms) to f16 hi/lo
//         into the step's TMEM A stage.  The C tile is never cleared: each
//         thread keeps its cells' previous totals and converts differences.
//   8     dictionary chunks (pre-split, pre-scaled f16 B operand), 2 stages
//   9-10  MMA issuers for even / odd steps (one issuing thread cannot keep
//         the tensor core busy at these shapes): Y_e = A_hi.D_hi + A_lo.D_hi +
//         A_hi.D_lo, kind::f16, A from TMEM, fp32 accumulator per step
//   11..  epilogue: fold every step's accumulator into fp32 registers (the
//         tensor core's accumulation truncates), write y (accumulate /
//         subtract b), sum of squares and max |r|
template <int N>
__global__ void __launch_bounds__(DscCfg<N>::kThreads, 1)
    k_tile_dsc(const TileArgs A, const float *__restrict__ scr, float *__restrict__ y, const float *__restrict__ b,
               const uint32_t flags, const ReduceSlots red, const DscOut out, const CallHooks hooks,
               const unsigned long long *__restrict__ skip_part, int nskip, const float *__restrict__ smax, int nsmax,
               unsigned *__restrict__ nonfinite, int finalize, int cap, const uint4 *__restrict__ fix_pcs, int fix_npc)
{
    using C = DscCfg<N>;
    extern __shared__ __align__(1024) unsigned char smraw[];
    __shared__ __align__(8) uint64_t d_full[2], d_empty[2], a_full[2], a_empty[2], acc_full[4], acc_empty[4],
        slot_full[4], slot_empty[4];
    __shared__ uint32_t s_hdr[4][2];  // staged step: tile-major start, entries
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t s_rowbad[2][4];  // rows with a non-finite s (slow path; per builder group)
    __shared__ float s_scale[2];
    if (hooks.done && *hooks.done) return;
    BD_DECL;
    unsigned char *sm = align1024(smraw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int my_tiles = (int)blockIdx.x < A.ntiles ? (A.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_tiles * A.nch;
    unsigned char *Dbuf = sm;
    const uint32_t Cs0 = sa(sm + 2 * C::DB);  // C tile of group g at Cs0 + g CBytes
    unsigned char *slots = sm + 2 * C::DB + 2 * C::CBytes;  // slot 2g + j: cap cellr, cap s
    if (threadIdx.x == 0) {
        for (int e = 0; e < 2; ++e) {
            bar_init(&d_full[e], 1);
            bar_init(&d_empty[e], 1);
            bar_init(&a_full[e], C::kNB / 2);
            bar_init(&a_empty[e], 1);
        }
        for (int b = 0; b < 4; ++b) {
            bar_init(&acc_full[b], 1);
            bar_init(&acc_empty[b], 4 * C::EQ);
        }
        for (int i = 0; i < 4; ++i) {
            bar_init(&slot_full[i], 1);
            bar_init(&slot_empty[i], C::kNB / 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == C::kMma) tcg::alloc(&tmem_base, 512);
    if (warp == 0) {
        // fixed-point scale: |s| * scale < 2^27, so a cell's kRanks terms stay below 2^30
        float m = 0.f;
        for (int i = lane; i < nsmax; i += 32) m = fmaxf(m, __ldcg(smax + i));
        m = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
        if (lane == 0) {
            int ex = 0;
            if (m > 0.f) {
                frexpf(m, &ex);  // m < 2^ex
                ex = 27 - ex;
            }
            s_scale[0] = ldexpf(1.f, ex);
            s_scale[1] = ldexpf(1.f, -ex) * (32768.f / kDScale);  // y = acc * inv_q * 2^15 / kDScale
        }
    }
    tcg::fence_before();
    __syncthreads();
    tcg::fence_after();
    const uint32_t tmem = tmem_base;
    double sq = 0.0;
    float amax = 0.f;
    auto step_of = [&](int k) -> size_t {
        return (size_t)((int)blockIdx.x + (k / A.nch) * (int)gridDim.x) * A.nch + (k % A.nch);
    };

    if (warp < C::kNB) {
        // ===== builders: group g (8 warps) takes the steps k = g (mod 2) =====
        const int g = warp >> 3, tid = threadIdx.x & 255;
        const int q = warp & 3, hh = (warp >> 2) & 1;  // lane quarter, 32-atom half
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t Cs = Cs0 + (uint32_t)(g * C::CBytes);
        const uint32_t rowaddr = Cs + 4u * (uint32_t)((q * 32 + lane) * kCS + hh * 32);
        const float scale = s_scale[0];
        const bool slow = *nonfinite != 0u;  // a non-finite s in this call: check every entry
        for (int i = tid; i < kTV * kCS / 4; i += 256) sts_f4(Cs + 16u * i, make_float4(0.f, 0.f, 0.f, 0.f));
        if (tid < 4) s_rowbad[g][tid] = 0u;
        named_bar(1 + g, 256);
        // fixed-point adds of 4 entries (pads hold s = 0 at a padding column)
        auto add4 = [&](uint2 c, float4 v) {
            const uint32_t o[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(Cs + 4u * o[e]),
                             "r"((uint32_t)__float2int_rn(x[e] * scale)) : "memory");
        };
        // slow path: rows that see a non-finite s become NaN
        auto add4_checked = [&](uint2 c, float4 v) {
            const uint32_t o[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (o[e] != (uint32_t)kKA && !isfinite(x[e])) {
                    const uint32_t row = o[e] / kCS;
                    atomicOr(&s_rowbad[g][row >> 5], 1u << (row & 31));
                    continue;
                }
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(Cs + 4u * o[e]),
                             "r"((uint32_t)__float2int_rn(x[e] * scale)) : "memory");
            }
        };
        for (int k = g, j = 0; k < total; k += 2, ++j) {
            const int sl = 2 * g + (j & 1);
            BD_WAIT(0, bar_wait(&slot_full[sl], (j >> 1) & 1));
            BD_T0(t_sc);
            const uint32_t p0 = s_hdr[sl][0], n = s_hdr[sl][1];
            const uint32_t nu = n / 4u, nst4 = min(n, (uint32_t)cap) / 4u;
            const uint32_t sc = sa(slots + (size_t)sl * cap * 6), ss = sc + (uint32_t)cap * 2u;
            auto unit = [&](uint32_t u, uint2 &c, float4 &v) {
                if (u < nst4) {
                    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(c.x), "=r"(c.y) : "r"(sc + 8u * u));
                    v = lds_f4(ss + 16u * u);
                } else {
                    c = __ldg(reinterpret_cast<const uint2 *>(A.cellr + p0) + u);
                    v = __ldcg(reinterpret_cast<const float4 *>(scr + p0) + u);
                }
            };
            if (!slow) {
                for (uint32_t u = tid; u < nu; u += 512u) {  // two units in flight per thread
                    uint2 c0, c1;
                    float4 v0, v1;
                    unit(u, c0, v0);
                    const bool two = u + 256u < nu;
                    if (two) unit(u + 256u, c1, v1);
                    add4(c0, v0);
                    if (two) add4(c1, v1);
                }
            } else {
                for (uint32_t u = tid; u < nu; u += 256u) {
                    uint2 c0;
                    float4 v0;
                    unit(u, c0, v0);
                    add4_checked(c0, v0);
                }
            }
            BD_ACC(1, t_sc);
            __syncwarp();
            if (lane == 0) bar_arrive(&slot_empty[sl]);
            BD_WAIT(2, named_bar(1 + g, 256));  // the step's sums are complete
            if (j >= 1) BD_WAIT(3, bar_wait(&a_empty[g], (j - 1) & 1));
            tcg::fence_after();
            BD_T0(t_cv);
            // this thread's row, 32 atoms: fixed point -> f16 hi/lo pairs into
            // TMEM A stage g, zeroing the cells behind
            uint32_t hv[16], lv[16];
            const float inv15 = 1.f / 32768.f;
            if (!slow) {
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                    const float4 x = lds_f4(rowaddr + 16u * i4);
                    sts_f4(rowaddr + 16u * i4, make_float4(0.f, 0.f, 0.f, 0.f));
                    split2((float)__float_as_int(x.x) * inv15, (float)__float_as_int(x.y) * inv15, hv[2 * i4], lv[2 * i4]);
                    split2((float)__float_as_int(x.z) * inv15, (float)__float_as_int(x.w) * inv15, hv[2 * i4 + 1],
                           lv[2 * i4 + 1]);
                }
            } else {
                const bool bad = (s_rowbad[g][q] >> lane) & 1u;
                const float nan = __int_as_float(0x7fc00000);
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                    const float4 x = lds_f4(rowaddr + 16u * i4);
                    sts_f4(rowaddr + 16u * i4, make_float4(0.f, 0.f, 0.f, 0.f));
                    split2(bad ? nan : (float)__float_as_int(x.x) * inv15, bad ? nan : (float)__float_as_int(x.y) * inv15,
                           hv[2 * i4], lv[2 * i4]);
                    split2(bad ? nan : (float)__float_as_int(x.z) * inv15, bad ? nan : (float)__float_as_int(x.w) * inv15,
                           hv[2 * i4 + 1], lv[2 * i4 + 1]);
                }
            }
            const uint32_t ta = tmem + lane_base + (uint32_t)(g * 64 + hh * 16);
            tm_st16(ta, hv);
            tm_st16(ta + 32u, lv);
            tcg::wait_st();
            tcg::fence_before();
            __syncwarp();
            BD_ACC(4, t_cv);
            if (lane == 0) bar_arrive(&a_full[g]);
            BD_WAIT(5, named_bar(1 + g, 256));  // C tile zeroed (and the row flags read) before the next step
            if (slow) {  // clear the row flags before the group's next adds
                if (tid < 4) s_rowbad[g][tid] = 0u;
                named_bar(1 + g, 256);
            }
        }
    } else if (warp < C::kEpi) {
      if (warp == C::kProdD) {
        // ===== dictionary chunks =====
        if (lane == 0) {
            const uint64_t pol = pol_last();
            StepIter it(0, A.nch), it3(3, A.nch);
            for (int k = 0; k < total; ++k, it.next(), it3.next()) {
                const int e = k & 1, c = it.c;
                if (k >= 2) BD_WAIT(10, bar_wait(&d_empty[e], ((k >> 1) - 1) & 1));
                bar_arrive_tx(&d_full[e], (unsigned)C::DB);
                bulk_g2s(Dbuf + (size_t)e * C::DB, reinterpret_cast<const unsigned char *>(A.D) + (size_t)c * C::DB,
                         (unsigned)C::DB, &d_full[e], pol);
            }
        }
      } else if (warp == C::kProdS) {
        // ===== step entries into the groups' slots (bulk copies), L2 prefetch
        // ahead; lane g serves builder group g (independent waits) =====
        if (lane < 2) {
            const int g = lane;
            const uint64_t pol = pol_first();
            constexpr int PF = 4;  // own steps: pointers loaded PF ahead, L2 prefetch PF - 1 ahead
            StepIter it(g, A.nch), itp(g + 2 * PF, A.nch);
            uint32_t pq[PF], nq[PF];
            {
                StepIter ip(g, A.nch);
#pragma unroll
                for (int i = 0; i < PF; ++i) {
                    const bool in = g + 2 * i < total;
                    pq[i] = in ? __ldg(A.step + ip.gs) : 0u;
                    nq[i] = in ? __ldg(A.step + ip.gs + 1) : 0u;
                    ip.next();
                    ip.next();
                }
            }
            for (int k = g, j = 0; k < total; k += 2, ++j) {
                const int sl = 2 * g + (j & 1);
                const uint32_t p0 = pq[0], n = nq[0] - pq[0];
                uint32_t pn = 0, en = 0;
                if (k + 2 * PF < total) {
                    pn = __ldg(A.step + itp.gs);
                    en = __ldg(A.step + itp.gs + 1);
                }
                itp.next();
                itp.next();
#pragma unroll
                for (int i = 0; i < PF - 1; ++i) {
                    pq[i] = pq[i + 1];
                    nq[i] = nq[i + 1];
                }
                pq[PF - 1] = pn;
                nq[PF - 1] = en;
                if (j >= 2) BD_WAIT(9, bar_wait(&slot_empty[sl], ((j >> 1) - 1) & 1));
                const uint32_t nst = min(n, (uint32_t)cap);
                s_hdr[sl][0] = p0;
                s_hdr[sl][1] = n;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bar_arrive_tx(&slot_full[sl], nst * 6u);
                unsigned char *dst = slots + (size_t)sl * cap * 6;
                if (nst) {
                    bulk_g2s(dst, A.cellr + p0, nst * 2u, &slot_full[sl], pol);
                    bulk_g2s(dst + (size_t)cap * 2, scr + p0, nst * 4u, &slot_full[sl], pol);
                }
                if (nq[PF - 2] > pq[PF - 2]) {
                    prefetch_l2(A.cellr + pq[PF - 2], (nq[PF - 2] - pq[PF - 2]) * 2u);
                    prefetch_l2(scr + pq[PF - 2], (nq[PF - 2] - pq[PF - 2]) * 4u);
                }
                it.next();
                it.next();
            }
        }
      } else if (warp < C::kMma + 2) {
        // ===== MMA issuers: warp kMma + e takes the steps k = e (mod 2) =====
        // Within a tile, an issuer accumulates pairs of its steps (128
        // atoms) in one TMEM buffer before the epilogue folds it.
        const int e = warp - C::kMma;
        if (lane == 0) {
            const uint32_t id = (uint32_t)idesc_f16(kTV, N);
            const uint32_t db = sa(Dbuf + (size_t)e * C::DB);
            const uint64_t bh = tcg::sdesc(db), bl = tcg::sdesc(db + (uint32_t)(N * 128));
            const uint32_t ah = tmem + (uint32_t)(e * 64), al = ah + 32u;
            int j = 0, f = 0;
            for (int i = 0; i < my_tiles; ++i) {
                const int c0 = (e + i * A.nch) & 1, nown = (A.nch - c0 + 1) >> 1;
                for (int oi = 0; oi < nown; ++oi, ++j) {
                    const int b = e * C::NACC + (C::NACC == 2 ? (f & 1) : 0);
                    const int fpar = C::NACC == 2 ? ((f >> 1) - 1) & 1 : (f - 1) & 1;
                    const bool start = (oi % C::FOLD) == 0, fold = (oi % C::FOLD) == C::FOLD - 1 || oi == nown - 1;
                    if (start && f >= C::NACC) BD_WAIT(6, bar_wait(&acc_empty[b], fpar));
                    BD_WAIT(7, bar_wait(&a_full[e], j & 1));
                    BD_WAIT(8, bar_wait(&d_full[e], j & 1));
                    tcg::fence_after();
                    const uint32_t d = tmem + (uint32_t)(C::TACC + b * N);
#pragma unroll
                    for (int kk = 0; kk < kKA / 16; ++kk) {
                        const uint64_t o = (uint64_t)((kk * 32) >> 4);
                        mma_f16(d, ah + 8u * kk, bh + o, id, (start && kk == 0) ? 0u : 1u);
                        mma_f16(d, al + 8u * kk, bh + o, id, 1u);
                        mma_f16(d, ah + 8u * kk, bl + o, id, 1u);
                    }
                    tcg::commit(&a_empty[e]);
                    tcg::commit(&d_empty[e]);
                    if (fold) {
                        tcg::commit(&acc_full[b]);
                        ++f;
                    }
                }
            }
        }
        __syncwarp();
      }
    } else {
        // ===== epilogue: thread = tile row (TMEM lane), a slice of columns =====
        const int ew = warp - C::kEpi, q = warp & 3, cs = ew >> 2;
        const int row = q * 32 + lane;
        const int b0 = cs * C::NBLK / C::EQ, b1 = (cs + 1) * C::NBLK / C::EQ;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const bool accumulate = flags & LIFE_ACCUMULATE;
        const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
        const float oscale = s_scale[1];
        int fcount[2] = {0, 0};  // folds seen per issuer
        for (int i = 0; i < my_tiles; ++i) {
            const int t = (int)blockIdx.x + i * (int)gridDim.x;
            float acc[C::MB * 16];
#pragma unroll
            for (int x = 0; x < C::MB * 16; ++x) acc[x] = 0.f;
            for (int c = 0; c < A.nch; ++c) {
                const int e = (i * A.nch + c) & 1, c0 = (e + i * A.nch) & 1;
                const int nown = (A.nch - c0 + 1) >> 1, oi = (c - c0) >> 1;
                if (!((oi % C::FOLD) == C::FOLD - 1 || oi == nown - 1)) continue;  // not a fold step
                const int f = fcount[e]++;
                const int b = e * C::NACC + (C::NACC == 2 ? (f & 1) : 0);
                const int par = C::NACC == 2 ? (f >> 1) & 1 : f & 1;
                BD_WAIT(11, bar_wait(&acc_full[b], par));
                tcg::fence_after();
                BD_T0(t_fd);
#pragma unroll
                for (int bb = 0; bb < C::MB; ++bb) {
                    if (b0 + bb < b1) {
                        uint32_t r[16];
                        tm_ld16(tmem + lane_base + (uint32_t)(C::TACC + b * N + 16 * (b0 + bb)), r);
                        tm_wait_ld();
#pragma unroll
                        for (int x = 0; x < 16; ++x) acc[16 * bb + x] += __uint_as_float(r[x]);
                    }
                }
                BD_ACC(12, t_fd);
                tcg::fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&acc_empty[b]);
            }
            const int rv = __ldg(A.rowvox + (size_t)t * kTV + row);
            const int rp = __ldg(A.rowpart + (size_t)t * kTV + row);
            if (rv < 0) continue;
            if (rp >= 0) {
                float *yp = A.ypart + (size_t)rp * N;
#pragma unroll
                for (int bb = 0; bb < C::MB; ++bb)
                    if (b0 + bb < b1)
#pragma unroll
                        for (int x = 0; x < 16; ++x) yp[16 * (b0 + bb) + x] = acc[16 * bb + x] * oscale;
                continue;
            }
            const size_t yo = (size_t)rv * A.nt;
            if ((A.nt & 3) == 0) {
#pragma unroll
                for (int bb = 0; bb < C::MB; ++bb) {
#pragma unroll
                    for (int e4 = 0; e4 < 4; ++e4) {
                        const int col = 16 * (b0 + bb) + 4 * e4;
                        if (b0 + bb < b1 && col < A.nt) {
                            float r[4] = {acc[16 * bb + 4 * e4] * oscale, acc[16 * bb + 4 * e4 + 1] * oscale,
                                          acc[16 * bb + 4 * e4 + 2] * oscale, acc[16 * bb + 4 * e4 + 3] * oscale};
                            float4 *y4 = reinterpret_cast<float4 *>(y + yo + col);
                            if (accumulate) {
                                const float4 o = *y4;
                                r[0] += o.x; r[1] += o.y; r[2] += o.z; r[3] += o.w;
                            }
                            if (subtract) {
                                const float4 o = __ldg(reinterpret_cast<const float4 *>(b + yo + col));
                                r[0] -= o.x; r[1] -= o.y; r[2] -= o.z; r[3] -= o.w;
                            }
                            *y4 = make_float4(r[0], r[1], r[2], r[3]);
#pragma unroll
                            for (int x = 0; x < 4; ++x) {
                                sq += (double)r[x] * (double)r[x];
                                amax = fmaxf(amax, fabsf(r[x]));
                            }
                        }
                    }
                }
            } else {
#pragma unroll
                for (int bb = 0; bb < C::MB; ++bb) {
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        const int col = 16 * (b0 + bb) + x;
                        if (b0 + bb < b1 && col < A.nt) {
                            float r = acc[16 * bb + x] * oscale;
                            if (accumulate) r += y[yo + col];
                            if (subtract) r -= b[yo + col];
                            y[yo + col] = r;
                            sq += (double)r * (double)r;
                            amax = fmaxf(amax, fabsf(r));
                        }
                    }
                }
            }
        }
    }

    // ---- teardown, fixed-order completion --------------------------------------
    BD_FLUSH;
    tcg::fence_before();
    __syncthreads();
    if (warp == C::kMma) {
        tcg::fence_after();
        tcg::dealloc(tmem, 512);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    const int gw = (int)blockIdx.x * C::kWarps + warp;
    if (lane == 0) {
        red.part_d[gw] = sq;
        red.part_f[gw] = amax;
    }
    if (finalize && last_cta(red.counter)) {
        int nparts = (int)gridDim.x * C::kWarps;
        if (fix_npc > 0) {
            // few voxels split over several rows (single pieces): every CTA
            // has written its partial rows, so the last CTA folds them here
            // instead of a fixup launch
            const bool accumulate = flags & LIFE_ACCUMULATE;
            const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
            double fsq = 0.0;
            float famax = 0.f;
            fix_pieces<N>(fix_pcs, fix_npc, A.ypart, A.nt, nullptr, y, b, accumulate, subtract, warp, C::kWarps, lane,
                          fsq, famax);
            fix_partial(fsq, famax, red, nparts);
            __syncthreads();
            nparts += 1;
        }
        dsc_finish(red, nparts, skip_part, nskip, out, red.counter, hooks, C::kThreads, nonfinite);
    }
}

// DSC fixup of split voxels, step 1: one warp per piece (at most kFixRows
// partial rows, lanes over directions); single-piece voxels are final here,
// the others store their piece sums for k_tile_dsc_fold
template <int N>
__global__ void __launch_bounds__(512)
    k_tile_dsc_fix(const uint4 *__restrict__ pcs, int npc, const float *__restrict__ ypart, int nt,
                   float *__restrict__ fixsum, float *__restrict__ y, const float *__restrict__ b, uint32_t flags,
                   const ReduceSlots red, int part0, int finish, const DscOut out, const CallHooks hooks,
                   const unsigned long long *__restrict__ skip_part, int nskip, unsigned *__restrict__ nonfinite)
{
    if (hooks.done && *hooks.done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool accumulate = flags & LIFE_ACCUMULATE;
    const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
    double sq = 0.0;
    float amax = 0.f;
    fix_pieces<N>(pcs, npc, ypart, nt, fixsum, y, b, accumulate, subtract, blockIdx.x * 16 + warp, gridDim.x * 16,
                  lane, sq, amax);
    fix_partial(sq, amax, red, part0 + blockIdx.x);
    if (finish && last_cta(red.counter))
        dsc_finish(red, part0 + (int)gridDim.x, skip_part, nskip, out, red.counter, hooks, 512, nonfinite);
}

// step 2: one CTA per voxel of several pieces; thread (group g, direction c)
// sums pieces g, g + G, ..., then the groups are added in order
template <int N>
__global__ void __launch_bounds__(1024)
    k_tile_dsc_fold(const uint32_t *__restrict__ big, const uint32_t *__restrict__ bpp, int nbig,
                    const float *__restrict__ fixsum, int nt, float *__restrict__ y, const float *__restrict__ b,
                    uint32_t flags, const ReduceSlots red, int part0, const DscOut out, const CallHooks hooks,
                    const unsigned long long *__restrict__ skip_part, int nskip, unsigned *__restrict__ nonfinite)
{
    if (hooks.done && *hooks.done) return;
    __shared__ float buf[1024];
    const bool accumulate = flags & LIFE_ACCUMULATE;
    const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
    const int G = 1024 / nt, t = threadIdx.x, c = t % nt, g = t / nt;
    double sq = 0.0;
    float amax = 0.f;
    for (int i = blockIdx.x; i < nbig; i += gridDim.x) {
        const uint32_t s0 = __ldg(bpp + i), s1 = __ldg(bpp + i + 1);
        float r = 0.f;
        if (g < G)
            for (uint32_t q = s0 + g; q < s1; q += G) r += fixsum[(size_t)q * N + c];
        buf[t] = r;
        __syncthreads();
        if (t < nt) {
            float tot = 0.f;
            for (int k = 0; k < G; ++k) tot += buf[k * nt + t];
            fix_store(tot, (size_t)__ldg(big + i) * nt + t, y, b, accumulate, subtract, sq, amax);
        }
        __syncthreads();
    }
    fix_partial(sq, amax, red, part0 + blockIdx.x);
    if (last_cta(red.counter))
        dsc_finish(red, part0 + (int)gridDim.x, skip_part, nskip, out, red.counter, hooks, 1024, nonfinite);
}

// WC tile side.  Roles (warps):
//   0-7   gatherers: per step, z = Z[row, atom] of every entry (cell offsets
//         prefetched into registers one step ahead) from the shared-memory Z
//         tile into the tile-major scratch (16-byte stores)
//   8     dictionary chunks (WC B operand: atoms x directions, f16 hi | lo)
//   9-10  MMA issuers for even / odd steps: Z_e = Y_hi.D_hi + Y_lo.D_hi +
//         Y_hi.D_lo (M = 128 rows, N = 64 atoms, K = directions), Y from TMEM
//   11-18 YZ: per tile, y rows (thread = row, scaled into the f16 range) split
//         into f16 hi/lo and stored to TMEM; per step, Z read back from TMEM,
//         rescaled, into a double-buffered shared-memory tile
template <int N>
__global__ void __launch_bounds__(WcCfg<N>::kThreads, 1)
    k_tile_wc(const TileArgs A, const float *__restrict__ y, float *__restrict__ scr, const float *__restrict__ ymax,
              const double *__restrict__ ysumsq, const CallHooks hooks)
{
    using C = WcCfg<N>;
    extern __shared__ __align__(1024) unsigned char smraw[];
    __shared__ __align__(8) uint64_t d_full[2], d_empty[2], acc_full[2], acc_empty[2], z_full[WcCfg<N>::NZ],
        z_empty[WcCfg<N>::NZ], y_ready, y_free;
    __shared__ uint32_t tmem_base;
    if (hooks.done && *hooks.done) return;
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    BD_DECL;
    unsigned char *sm = align1024(smraw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int my_tiles = (int)blockIdx.x < A.ntiles ? (A.ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_tiles * A.nch;
    unsigned char *Dbuf = sm;
    const uint32_t Zs = sa(sm + 2 * C::DB);
    if (threadIdx.x == 0) {
        for (int e = 0; e < 2; ++e) {
            bar_init(&d_full[e], 1);
            bar_init(&d_empty[e], 1);
            bar_init(&acc_full[e], 1);
            bar_init(&acc_empty[e], 8);
        }
        for (int e = 0; e < C::NZ; ++e) {
            bar_init(&z_full[e], 8);
            bar_init(&z_empty[e], kBuild);
        }
        bar_init(&y_ready, 8);
        bar_init(&y_free, 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == C::kMma) tcg::alloc(&tmem_base, 512);
    tcg::fence_before();
    __syncthreads();
    tcg::fence_after();
    const uint32_t tmem = tmem_base;
    auto step_of = [&](int k) -> size_t {
        return (size_t)((int)blockIdx.x + (k / A.nch) * (int)gridDim.x) * A.nch + (k % A.nch);
    };

    if (warp < kBuild) {
        // ===== gatherers =====
        const int tid = threadIdx.x;
        StepIter it2(0, A.nch);
        auto ptrs = [&](int k, uint32_t &p0, uint32_t &n) {
            if (k < total) {
                p0 = __ldg(A.step + it2.gs);
                n = __ldg(A.step + it2.gs + 1) - p0;
                it2.next();
            } else {
                p0 = n = 0;
            }
        };
        uint32_t cp0, cn, np0, nn;
        uint2 cc[kUMax], nc[kUMax];
        auto fetch = [&](uint32_t p0, uint32_t n, uint2 (&c)[kUMax]) {
#pragma unroll
            for (int i = 0; i < kUMax; ++i) {
                const uint32_t u = (uint32_t)tid + 256u * i;
                if (u < n / 4u) c[i] = __ldg(reinterpret_cast<const uint2 *>(A.cellr + p0) + u);
            }
        };
        ptrs(0, np0, nn);
        fetch(np0, nn, nc);
        uint32_t p2, n2;
        ptrs(1, p2, n2);
        for (int k = 0; k < total; ++k) {
            const int e = k & 1;
            cp0 = np0;  // this step: registers loaded during the previous one
            cn = nn;
#pragma unroll
            for (int i = 0; i < kUMax; ++i) cc[i] = nc[i];
            np0 = p2;
            nn = n2;
            fetch(np0, nn, nc);  // next step, in flight during this one
            ptrs(k + 2, p2, n2);
            const int zb = k % C::NZ;
            BD_WAIT(17, bar_wait(&z_full[zb], (k / C::NZ) & 1));
            BD_T0(t_g);
            const uint32_t Z = Zs + (uint32_t)(zb * C::ZBytes);
            float4 *dst = reinterpret_cast<float4 *>(scr + cp0);
            auto gat = [&](uint2 c, uint32_t u) {
                const uint32_t o[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
                dst[u] = make_float4(lds_f(Z + 4u * o[0]), lds_f(Z + 4u * o[1]), lds_f(Z + 4u * o[2]),
                                     lds_f(Z + 4u * o[3]));
            };
#pragma unroll
            for (int i = 0; i < kUMax; ++i) {
                const uint32_t u = (uint32_t)tid + 256u * i;
                if (u < cn / 4u) gat(cc[i], u);
            }
            for (uint32_t u = (uint32_t)tid + 256u * kUMax; u < cn / 4u; u += 256u)
                gat(__ldg(reinterpret_cast<const uint2 *>(A.cellr + cp0) + u), u);
            BD_ACC(18, t_g);
            __syncwarp();
            if (lane == 0) bar_arrive(&z_empty[zb]);
        }
    } else if (warp == C::kProdD) {
        if (lane == 0) {
            const uint64_t pol = pol_last();
            StepIter it(0, A.nch), it3(3, A.nch);
            for (int k = 0; k < total; ++k, it.next(), it3.next()) {
                const int e = k & 1, c = it.c;
                if (k >= 2) BD_WAIT(23, bar_wait(&d_empty[e], ((k >> 1) - 1) & 1));
                bar_arrive_tx(&d_full[e], (unsigned)C::DB);
                bulk_g2s(Dbuf + (size_t)e * C::DB, reinterpret_cast<const unsigned char *>(A.D) + (size_t)c * C::DB,
                         (unsigned)C::DB, &d_full[e], pol);
                if (k + 3 < total) {  // the gatherers' cell offsets, three steps ahead
                    const size_t g3 = it3.gs;
                    const uint32_t p3 = __ldg(A.step + g3), n3 = __ldg(A.step + g3 + 1) - p3;
                    if (n3) prefetch_l2(A.cellr + p3, n3 * 2u);
                }
            }
        }
    } else if (warp < C::kYZ) {
        // ===== MMA issuers =====
        const int e = warp - C::kMma;
        if (lane == 0) {
            const uint32_t id = (uint32_t)idesc_f16(kTV, kKA);
            const uint32_t db = sa(Dbuf + (size_t)e * C::DB);
            const uint64_t bh = tcg::sdesc(db), bl = tcg::sdesc(db + (uint32_t)(C::NKB * kKA * 128));
            const uint32_t d = tmem + (uint32_t)(C::TZ + e * kKA);
            int k = 0, j = 0;
            for (int i = 0; i < my_tiles; ++i) {
                BD_WAIT(19, bar_wait(&y_ready, i & 1));
                tcg::fence_after();
                for (int c = 0; c < A.nch; ++c, ++k) {
                    if ((k & 1) != e) continue;
                    if (j >= 1) BD_WAIT(21, bar_wait(&acc_empty[e], (j - 1) & 1));
                    BD_WAIT(20, bar_wait(&d_full[e], j & 1));
                    tcg::fence_after();
#pragma unroll
                    for (int kk = 0; kk < N / 16; ++kk) {
                        const uint64_t o = (uint64_t)((((kk >> 2) * kKA * 128) + (kk & 3) * 32) >> 4);
                        mma_f16(d, tmem + 8u * kk, bh + o, id, kk ? 1u : 0u);
                        mma_f16(d, tmem + (uint32_t)(N / 2) + 8u * kk, bh + o, id, 1u);
                        mma_f16(d, tmem + 8u * kk, bl + o, id, 1u);
                    }
                    tcg::commit(&d_empty[e]);
                    tcg::commit(&acc_full[e]);
                    ++j;
                }
                tcg::commit(&y_free);  // this issuer's MMAs of the tile (arrives at once if none)
            }
        }
        __syncwarp();
    } else {
        // ===== YZ =====
        const int ew = warp - C::kYZ, q = warp & 3, cs = ew >> 2;
        const int row = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        constexpr int NB8 = N / 16;                 // 16-direction blocks (8 TMEM columns of f16 pairs)
        constexpr int BPS = (NB8 + 1) / 2;          // blocks per slice (max)
        const int bb0 = cs * NB8 / 2, bb1 = (cs + 1) * NB8 / 2;
        const bool vec = (A.nt & 3) == 0;
        // y scale into the f16 range: |y| * ys < 2^14; z = Z / (ys * kDScale)
        const float yb = ysumsq ? (float)sqrt(*ysumsq) : *ymax;
        int ex = 0;
        if (yb > 0.f && isfinite(yb)) {
            frexpf(yb, &ex);
            ex = 14 - ex;
        }
        const float ys = ldexpf(1.f, ex), zinv = ldexpf(1.f, -ex) / kDScale;
        constexpr bool kPre = N <= 96;
        float yr[kPre ? BPS * 16 : 16];
        auto load_blk = [&](const float *src, bool ok, int blk, float *dstv) {
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
                const int col = 16 * blk + 4 * i4;
                if (ok && vec && col < A.nt) {
                    const float4 v = __ldg(reinterpret_cast<const float4 *>(src + col));
                    dstv[4 * i4] = v.x; dstv[4 * i4 + 1] = v.y; dstv[4 * i4 + 2] = v.z; dstv[4 * i4 + 3] = v.w;
                } else {
#pragma unroll
                    for (int x = 0; x < 4; ++x) dstv[4 * i4 + x] = (ok && col + x < A.nt) ? __ldg(src + col + x) : 0.f;
                }
            }
        };
        auto row_src = [&](int t, bool &ok) {
            const int rv = __ldg(A.rowvox + (size_t)t * kTV + row);
            ok = rv >= 0;
            return y + (size_t)(rv < 0 ? 0 : rv) * A.nt;
        };
        auto store_blk = [&](int blk, const float *v) {
            uint32_t hv[8], lv[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) split2(v[2 * x] * ys, v[2 * x + 1] * ys, hv[x], lv[x]);
            tm_st8(tmem + lane_base + (uint32_t)(8 * blk), hv);
            tm_st8(tmem + lane_base + (uint32_t)(N / 2 + 8 * blk), lv);
        };
        if (kPre && my_tiles > 0) {
            bool ok;
            const float *src = row_src((int)blockIdx.x, ok);
#pragma unroll
            for (int bb = 0; bb < BPS; ++bb)
                if (bb0 + bb < bb1) load_blk(src, ok, bb0 + bb, yr + 16 * bb);
        }
        int k = 0;
        for (int i = 0; i < my_tiles; ++i) {
            const int t = (int)blockIdx.x + i * (int)gridDim.x;
            if (i >= 1) BD_WAIT(24, bar_wait(&y_free, (i - 1) & 1));
            tcg::fence_after();
            BD_T0(t_y);
            if (kPre) {
#pragma unroll
                for (int bb = 0; bb < BPS; ++bb)
                    if (bb0 + bb < bb1) store_blk(bb0 + bb, yr + 16 * bb);
            } else {
                bool ok;
                const float *src = row_src(t, ok);
#pragma unroll 1
                for (int blk = bb0; blk < bb1; ++blk) {
                    load_blk(src, ok, blk, yr);
                    store_blk(blk, yr);
                }
            }
            tcg::wait_st();
            tcg::fence_before();
            __syncwarp();
            BD_ACC(25, t_y);
            if (lane == 0) bar_arrive(&y_ready);
            if (kPre && i + 1 < my_tiles) {  // next tile's rows, in flight meanwhile
                bool ok;
                const float *src = row_src(t + (int)gridDim.x, ok);
#pragma unroll
                for (int bb = 0; bb < BPS; ++bb)
                    if (bb0 + bb < bb1) load_blk(src, ok, bb0 + bb, yr + 16 * bb);
            }
            for (int c = 0; c < A.nch; ++c, ++k) {
                const int e = k & 1;
                BD_WAIT(26, bar_wait(&acc_full[e], (k >> 1) & 1));
                tcg::fence_after();
                BD_T0(t_z);
                uint32_t zr[32];
#pragma unroll
                for (int h16 = 0; h16 < 2; ++h16) {
                    uint32_t r[16];
                    tm_ld16(tmem + lane_base + (uint32_t)(C::TZ + e * kKA + cs * 32 + 16 * h16), r);
                    tm_wait_ld();
#pragma unroll
                    for (int x = 0; x < 16; ++x) zr[16 * h16 + x] = r[x];
                }
                BD_ACC(27, t_z);
                tcg::fence_before();
                if (LIFE_WC_EARLY) {  // Z is in registers: the accumulator is free for the MMA of step k + 2
                    __syncwarp();
                    if (lane == 0) bar_arrive(&acc_empty[e]);
                }
                const int zb = k % C::NZ;
                if (k >= C::NZ) BD_WAIT(28, bar_wait(&z_empty[zb], ((k / C::NZ) - 1) & 1));
                BD_T0(t_zs);
                const uint32_t za = Zs + (uint32_t)(zb * C::ZBytes) + 4u * (uint32_t)(row * kCS + cs * 32);
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4)
                    sts_f4(za + 16u * i4, make_float4(__uint_as_float(zr[4 * i4]) * zinv,
                                                      __uint_as_float(zr[4 * i4 + 1]) * zinv,
                                                      __uint_as_float(zr[4 * i4 + 2]) * zinv,
                                                      __uint_as_float(zr[4 * i4 + 3]) * zinv));
                BD_ACC(29, t_zs);
                __syncwarp();
                if (lane == 0) {
                    if (!LIFE_WC_EARLY) bar_arrive(&acc_empty[e]);
                    bar_arrive(&z_full[zb]);
                }
            }
        }
    }
    BD_FLUSH;
    tcg::fence_before();
    __syncthreads();
    if (warp == C::kMma) {
        tcg::fence_after();
        tcg::dealloc(tmem, 512);
    }
}

}  // namespace bin

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
namespace {
using namespace bin;

constexpr int kSmemMax = 232448 - 2048;  // opt-in dynamic limit minus static + alignment slack

SideArgs side_args(const life_phi *phi)
{
    return SideArgs{phi->b_vid, phi->b_val, phi->b_segsrc, phi->b_segdst, phi->b_binptr,
                    phi->b_vf2f, phi->b_nvf, phi->b_nbins};
}
ChunkArgs chunk_args(const life_phi *phi)
{
    return ChunkArgs{reinterpret_cast<const uint4 *>(phi->b_chunks), phi->b_ctachunk, phi->b_cgrp};
}

template <int N>
int prep_t(life_phi *phi)
{
    using CD = DscCfg<N>;
    using CW = WcCfg<N>;
    {
        const long avail = (long)kSmemMax - 1024L - 2L * CD::DB - 2L * CD::CBytes;
        phi->b_dsc_cap = (int)std::min(16384L, std::max(0L, avail / (4L * 6L) / 32 * 32));
    }
    phi->b_dsc_smem = 1024 + 2 * (size_t)CD::DB + 2 * (size_t)CD::CBytes + (size_t)4 * 6 * phi->b_dsc_cap;
    phi->b_wc_smem = 1024 + 2 * (size_t)CW::DB + (size_t)CW::NZ * CW::ZBytes;
    if (phi->b_dsc_smem > (size_t)kSmemMax || phi->b_wc_smem > (size_t)kSmemMax)
        return fail(LIFE_ERR_CONFIG_INVALID, "bin layout: shared memory does not fit");
    phi->b_side_smem = (size_t)kSB * 4 + (size_t)kNsDsc * kSlotBytes;
    phi->b_wcs_smem = (size_t)kSB * 8 + (size_t)kNsWc * kSlotBytes;
    LIFE_TRY(ensure_smem(k_tile_dsc<N>, phi->b_dsc_smem));
    LIFE_TRY(ensure_smem(k_tile_wc<N>, phi->b_wc_smem));
    LIFE_TRY(ensure_smem(k_side_dsc, phi->b_side_smem));
    LIFE_TRY(ensure_smem(k_side_wc, phi->b_wcs_smem));
    return LIFE_OK;
}

template <int N>
int dsc_t(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags, const DscOut &o,
          const CallHooks &h, cudaStream_t st)
{
    using CD = DscCfg<N>;
    k_side_dsc<<<phi->b_side_grid, kSideThreads, phi->b_side_smem, st>>>(
        side_args(phi), chunk_args(phi), w, phi->b_scr, (flags & LIFE_SKIP_ZERO) ? 1 : 0, phi->b_skip, phi->b_smax, phi->b_nonfin, h);
    LIFE_CHECK_LAUNCH();
    const TileArgs A{phi->b_cellr, phi->b_step, phi->b_Ddsc, phi->b_rowvox, phi->b_rowpart, phi->b_ypart,
                     phi->b_ntiles, phi->b_nch, phi->nt};
    // split voxels: a handful of single-piece ones are folded by the tile
    // kernel's last CTA; many, or multi-piece ones, by the fixup kernels
    const bool inline_fix = phi->b_nfix > 0 && phi->b_nbig == 0 && phi->b_npc <= 4 * CD::kWarps;
    const int fin = (phi->b_nfix == 0 || inline_fix) ? 1 : 0;
    k_tile_dsc<N><<<phi->b_tile_grid, CD::kThreads, phi->b_dsc_smem, st>>>(
        A, phi->b_scr, y, b, flags, phi->red, o, h, phi->b_skip, phi->b_side_grid, phi->b_smax, phi->b_side_grid,
        phi->b_nonfin, fin, phi->b_dsc_cap, inline_fix ? reinterpret_cast<const uint4 *>(phi->b_fixpc) : nullptr,
        inline_fix ? phi->b_npc : 0);
    LIFE_CHECK_LAUNCH();
    if (!fin) {
        const int part0 = phi->b_tile_grid * CD::kWarps;
        const int ga = std::max(1, std::min(phi->sms * 4, (phi->b_npc + 15) / 16));
        k_tile_dsc_fix<N><<<ga, 512, 0, st>>>(reinterpret_cast<const uint4 *>(phi->b_fixpc), phi->b_npc, phi->b_ypart,
                                              phi->nt, phi->b_fixsum, y, b, flags, phi->red, part0,
                                              phi->b_nbig == 0 ? 1 : 0, o, h, phi->b_skip, phi->b_side_grid,
                                              phi->b_nonfin);
        LIFE_CHECK_LAUNCH();
        if (phi->b_nbig) {
            const int gf = std::min(phi->sms, phi->b_nbig);
            k_tile_dsc_fold<N><<<gf, 1024, 0, st>>>(phi->b_fixbig, phi->b_fixbpp, phi->b_nbig, phi->b_fixsum, phi->nt,
                                                    y, b, flags, phi->red, part0 + ga, o, h, phi->b_skip,
                                                    phi->b_side_grid, phi->b_nonfin);
            LIFE_CHECK_LAUNCH();
        }
    }
    return LIFE_OK;
}

template <int N>
int wc_tile_t(life_phi *phi, const float *y, const FixParams &fx, const CallHooks &h, cudaStream_t st)
{
    using CW = WcCfg<N>;
    const TileArgs A{phi->b_cellr, phi->b_step, phi->b_Dwc, phi->b_rowvox, phi->b_rowpart, phi->b_ypart,
                     phi->b_ntiles, phi->b_nch, phi->nt};
    k_tile_wc<N><<<phi->b_tile_grid, CW::kThreads, phi->b_wc_smem, st>>>(A, y, phi->b_scr, fx.ymax, fx.ysumsq, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

#define LIFE_BIN_DISPATCH(FN, ...)                                             \
    switch (phi->b_n) {                                                        \
    case 32: return FN<32>(__VA_ARGS__);                                       \
    case 64: return FN<64>(__VA_ARGS__);                                       \
    case 96: return FN<96>(__VA_ARGS__);                                       \
    case 128: return FN<128>(__VA_ARGS__);                                     \
    case 160: return FN<160>(__VA_ARGS__);                                     \
    case 192: return FN<192>(__VA_ARGS__);                                     \
    default: return fail(LIFE_ERR_CONFIG_INVALID, "bin layout: unsupported n_dirs"); \
    }

}  // namespace

int prepare_bin(life_phi *phi) { LIFE_BIN_DISPATCH(prep_t, phi); }

int bin_tile_warps(const life_phi *phi)
{
    switch (phi->b_n) {
    case 32: case 64: return DscCfg<64>::kWarps;
    case 96: case 128: return DscCfg<128>::kWarps;
    default: return DscCfg<192>::kWarps;
    }
}

int launch_dsc_bin(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags, const DscOut &o,
                   const CallHooks &h, cudaStream_t st)
{
    LIFE_BIN_DISPATCH(dsc_t, phi, w, y, b, flags, o, h, st);
}

static int wc_tile(life_phi *phi, const float *y, const FixParams &fx, const CallHooks &h, cudaStream_t st)
{
    LIFE_BIN_DISPATCH(wc_tile_t, phi, y, fx, h, st);
}

// scalar tail of the WC buffer: value k of rank r at k * nranks + r, zeros
// elsewhere, so the integer SUM all-reduce delivers every rank's double
// untouched and all ranks add them in rank order (deterministic)
__global__ void k_tail_pack(const WcScalars sc, unsigned long long *tail, int rank, int nranks)
{
    for (int i = threadIdx.x; i < sc.n * nranks; i += blockDim.x) {
        const int k = i / nranks, r = i % nranks;
        tail[i] = r == rank ? (unsigned long long)__double_as_longlong(*sc.v[k]) : 0ull;
    }
}
__global__ void k_tail_unpack(const WcScalars sc, const unsigned long long *tail, int nranks)
{
    if (threadIdx.x < sc.n) {
        double t = 0.0;
        for (int r = 0; r < nranks; ++r) t += __longlong_as_double((long long)tail[threadIdx.x * nranks + r]);
        *sc.v[threadIdx.x] = t;
    }
}

int launch_wc_bin(life_phi *phi, const float *y, float *w, const float *w_ref, const FixParams &fx, uint32_t flags,
                  double *sumsq, const CallHooks &h, const life_comm *comm, cudaStream_t st, const WcScalars *sc)
{
    LIFE_TRY(wc_tile(phi, y, fx, h, st));
    k_side_wc<<<phi->b_side_grid, kSideThreads, phi->b_wcs_smem, st>>>(side_args(phi), chunk_args(phi), phi->b_scr, fx, phi->nt,
                                                                          phi->b_wfix, phi->b_nanf, h);
    LIFE_CHECK_LAUNCH();
    if (comm) {
        // one integer all-reduce: the fascicle sums, the non-finite flags as
        // 8-bit counters (8 fascicles per word, no carry below 256 ranks) and
        // the DSC scalars of this iteration (rank slots); sums are exact, so
        // every rank gets bit-identical totals whatever the reduction order
        const int64_t nflag = (phi->nf + 7) / 8;
        unsigned long long *tail = phi->b_wfix + phi->nf + nflag;
        const int ns = (sc && comm->nranks <= kTailRanks) ? sc->n : 0;
        if (sc && !ns)  // more ranks than tail slots: scalars on their own
            for (int k = 0; k < sc->n; ++k)
                if (comm->allreduce(sc->v[k], 1, LIFE_DT_F64, LIFE_OP_SUM, st, comm->ctx) != 0)
                    return fail(LIFE_ERR_NCCL, "allreduce(scalar) failed");
        if (ns) {
            k_tail_pack<<<1, 256, 0, st>>>(*sc, tail, comm->rank, comm->nranks);
            LIFE_CHECK_LAUNCH();
        }
        const int64_t cnt = (int64_t)phi->nf + nflag + (int64_t)ns * comm->nranks;
        if (comm->allreduce(phi->b_wfix, cnt, LIFE_DT_I64, LIFE_OP_SUM, st, comm->ctx) != 0)
            return fail(LIFE_ERR_NCCL, "allreduce(wfix) failed");
        if (ns) {
            k_tail_unpack<<<1, 32, 0, st>>>(*sc, tail, comm->nranks);
            LIFE_CHECK_LAUNCH();
        }
    }
    // enough CTAs for one round of 4 fascicles per thread (a latency-bound
    // pass: 3-4 dependent rounds with one CTA per SM cost ~9 us at C2)
    const int blocks = std::max(1, std::min(4 * phi->sms, (phi->nf + 1023) / 1024));
    k_wc_fin<256><<<blocks, 256, 0, st>>>(phi->b_wfix, phi->b_nanf, phi->nf, w, w_ref, flags, fx, phi->nt,
                                          phi->part_d2, phi->counter2, sumsq, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

}  // namespace life

#ifdef LIFE_BIN_DIAG
extern "C" LIFE_API int life_debug_bin(unsigned long long *cyc_out)
{
    if (cudaDeviceSynchronize() != cudaSuccess) return 20;
    if (cyc_out && cudaMemcpyFromSymbol(cyc_out, life::bin::g_bin_cyc, 32 * sizeof(unsigned long long)) != cudaSuccess)
        return 20;
    unsigned long long z[32] = {};
    return cudaMemcpyToSymbol(life::bin::g_bin_cyc, z, sizeof(z)) == cudaSuccess ? 0 : 20;
}
#endif

// Debugging aid: register a host-mapped u32[8] that receives (1, block, warp,
// shared address, parity) of the first mbarrier wait that times out.
extern "C" LIFE_API int life_debug_timeout(unsigned *host_mapped)
{
    unsigned *dptr = nullptr;
    if (host_mapped && cudaHostGetDevicePointer((void **)&dptr, host_mapped, 0) != cudaSuccess) return 20;
    return cudaMemcpyToSymbol(life::bin::g_timeout_rec, &dptr, sizeof(dptr)) == cudaSuccess ? 0 : 20;
}
