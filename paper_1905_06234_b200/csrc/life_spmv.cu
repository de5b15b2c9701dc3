// life_spmv.cu -- DSC (y = M w) and WC (w = M^T y) on sm_100a.
//
// Reference semantics: _kernels.dsc_range / wc_range
// (/root/reference/pkg/src/lifespmv/_kernels.py:14-68) driven by
// engine.dsc_* / wc_* (engine.py:218-413).
//
// fp32 fast path:
//   * coefficients sorted by (atom group, voxel); one persistent 512-thread
//     CTA per SM; the group's dictionary slice (<= ~220 KB) is staged in
//     shared memory by one TMA bulk copy (cp.async.bulk + mbarrier) per group;
//   * a warp owns a contiguous voxel range (no atomics on y); lane t holds
//     directions t, t+32, ... of the current voxel in registers;
//   * coefficient streams are read 32 at a time, coalesced, evict-first;
//   * DSC: zero-skip with an exact ballot count, fused residual / sum of
//     squares / abs-max epilogue, deterministic fixed-order reductions;
//   * WC: per-coefficient dots reduced 32-at-a-time by a transposing warp
//     butterfly, then accumulated per fascicle as 64-bit fixed point with
//     RED.ADD (integer adds commute: bitwise reproducible, no float atomics).
// fp64 exact path: same order and rounding as the reference loops
// (__dmul_rn/__dadd_rn, no contraction) on stable voxel / fascicle sorts.
#include <cmath>

#include "life_common.cuh"

namespace life {

struct FastArgs {
    const uint32_t *atom;
    const uint32_t *fiber;
    const float *val;
    const uint32_t *gptr;
    const int *wpart;
    const float *Dg;
    int nv, nt, G, ag, na, slice_floats;
};

// ---- TMA bulk staging of a dictionary slice --------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src,
                                             unsigned bytes, uint64_t *bar)
{
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}

// Stage slice g into smem; every thread returns after the bytes landed.
__device__ __forceinline__ void stage_slice(float *Ds, const FastArgs &A, int g,
                                            uint64_t *bar, unsigned &parity)
{
    __syncthreads();  // everyone finished reading the previous slice
    const int na_g = min(A.ag, A.na - g * A.ag);
    const unsigned bytes = (unsigned)(((na_g * A.nt + 3) / 4) * 16);
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, bytes);
        const char *src = reinterpret_cast<const char *>(A.Dg + (size_t)g * A.slice_floats);
        char *dst = reinterpret_cast<char *>(Ds);
        for (unsigned off = 0; off < bytes; off += 32768u) {
            const unsigned sz = min(32768u, bytes - off);
            tma_bulk_g2s(dst + off, src + off, sz, bar);
        }
    }
    mbar_wait(bar, parity);
    parity ^= 1u;
}

// ---- deterministic completion: per-warp partials, last CTA reduces ---------
template <int BT>
__device__ __forceinline__ bool last_block_arrive(unsigned *counter)
{
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned ticket = atomicAdd(counter, 1u);
        s_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// Fixed-order block reductions with 32-entry shared scratch (keeps static
// shared memory tiny next to the dictionary slice).
template <int BT, typename T, typename Op>
__device__ T block_reduce_fixed(const T *part, int n, T init, Op op)
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

struct OpAdd {
    template <typename T>
    __device__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
    __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};

template <int BT>
__device__ double block_sum_fixed(const double *part, int n)
{
    return block_reduce_fixed<BT, double>(part, n, 0.0, OpAdd{});
}

template <int BT>
__device__ unsigned long long block_sum_u64(const unsigned long long *part, int n)
{
    return block_reduce_fixed<BT, unsigned long long>(part, n, 0ull, OpAdd{});
}

template <int BT>
__device__ float block_max_f(const float *part, int n)
{
    return block_reduce_fixed<BT, float>(part, n, 0.f, OpMax{});
}

__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max_f(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Voxel boundary cursor: lane l caches gp[wbase + 1 + l] so that crossing a
// voxel boundary costs a shuffle instead of a dependent global load.
struct VoxelCursor {
    const uint32_t *gp;
    int ve;      // exclusive voxel end of this warp's range
    int wbase;   // window origin
    uint32_t win;
    __device__ __forceinline__ void load(int base, int lane)
    {
        wbase = base;
        const int idx = min(base + 1 + lane, ve);
        win = gp[idx];
    }
    // end offset of voxel cv's segment
    __device__ __forceinline__ uint32_t end_of(int cv, int lane)
    {
        if (cv - wbase >= 32) load(cv, lane);
        return __shfl_sync(0xffffffffu, win, cv - wbase);
    }
};

// ---------------------------------------------------------------------------
// DSC fp32
// ---------------------------------------------------------------------------

template <int NT, bool FULL>
__global__ void __launch_bounds__(kSpmvThreads, 1)
    k_dsc_f32(const FastArgs A, const float *__restrict__ w, float *__restrict__ y,
              const float *__restrict__ b, const uint32_t flags,
              const ReduceSlots red, const DscOut out, const CallHooks hooks)
{
    extern __shared__ __align__(128) float Ds[];
    __shared__ __align__(8) uint64_t bar;
    if (hooks.done && *hooks.done) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (kSpmvThreads / 32) + (threadIdx.x >> 5);
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned parity = 0;

    const int vb = A.wpart[gw], ve = A.wpart[gw + 1];
    const bool accumulate = flags & LIFE_ACCUMULATE;
    const bool skip_zero = flags & LIFE_SKIP_ZERO;
    const bool subtract = (flags & LIFE_SUBTRACT_B) && b != nullptr;
    const int nt = A.nt;
    unsigned long long skipped = 0;
    double sq = 0.0;
    float amax = 0.f;

    for (int g = 0; g < A.G; ++g) {
        stage_slice(Ds, A, g, &bar, parity);
        if (vb >= ve) continue;
        const bool first = g == 0, last = g == A.G - 1;
        const uint32_t *gp = A.gptr + (size_t)g * A.nv;
        VoxelCursor cur{gp, ve, 0, 0};
        cur.load(vb, lane);
        const uint32_t kb = gp[vb];
        const uint32_t kend = gp[ve];

        int cv = vb;
        uint32_t cs = kb;
        uint32_t ce = cur.end_of(cv, lane);
        float acc[NT];

        auto init = [&](int v, bool nonempty) {
            const size_t yo = (size_t)v * nt;
            const bool load = first ? accumulate : (last || nonempty);
#pragma unroll
            for (int q = 0; q < NT; ++q) {
                const int t = lane + 32 * q;
                acc[q] = (load && (FULL || t < nt)) ? y[yo + t] : 0.f;
            }
        };
        auto finish = [&](int v, bool nonempty) {
            const size_t yo = (size_t)v * nt;
            if (last) {
#pragma unroll
                for (int q = 0; q < NT; ++q) {
                    const int t = lane + 32 * q;
                    if (FULL || t < nt) {
                        float o = acc[q];
                        if (subtract) o -= b[yo + t];
                        y[yo + t] = o;
                        sq += (double)o * (double)o;
                        amax = fmaxf(amax, fabsf(o));
                    }
                }
            } else if (nonempty || (first && !accumulate)) {
#pragma unroll
                for (int q = 0; q < NT; ++q) {
                    const int t = lane + 32 * q;
                    if (FULL || t < nt) y[yo + t] = acc[q];
                }
            }
        };

        init(cv, cs < ce);
        for (uint32_t base = kb; base < kend; base += 32) {
            const uint32_t k = base + lane;
            const bool valid = k < kend;
            uint32_t a = 0;
            float sc = 0.f;
            if (valid) {
                a = ld_stream(A.atom + k);
                const uint32_t f = ld_stream(A.fiber + k);
                const float vv = ld_stream(A.val + k);
                sc = __fmul_rn(__ldg(w + f), vv);
            }
            const unsigned zm = __ballot_sync(0xffffffffu, valid && sc == 0.f);
            skipped += __popc(zm);
            unsigned m = __ballot_sync(0xffffffffu, valid);
            if (skip_zero) m &= ~zm;
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t kj = base + j;
                while (kj >= ce) {
                    finish(cv, cs < ce);
                    ++cv;
                    cs = ce;
                    ce = cur.end_of(cv, lane);
                    init(cv, cs < ce);
                }
                const uint32_t aj = __shfl_sync(0xffffffffu, a, j);
                const float sj = __shfl_sync(0xffffffffu, sc, j);
                const float *dr = Ds + aj * nt;
#pragma unroll
                for (int q = 0; q < NT; ++q) {
                    const int t = lane + 32 * q;
                    if (FULL || t < nt) acc[q] = fmaf(dr[t], sj, acc[q]);
                }
            }
        }
        // close the open voxel and any trailing (empty) voxels
        while (true) {
            finish(cv, cs < ce);
            ++cv;
            if (cv >= ve) break;
            cs = ce;
            ce = cur.end_of(cv, lane);
            init(cv, cs < ce);
        }
    }

    // per-warp partials (fixed slots) -> last CTA reduces in fixed order
    sq = warp_sum_d(sq);
    amax = warp_max_f(amax);
    if (lane == 0) {
        red.part_d[gw] = sq;
        red.part_u[gw] = skipped;
        red.part_f[gw] = amax;
    }
    if (last_block_arrive<kSpmvThreads>(red.counter)) {
        const int W = gridDim.x * (kSpmvThreads / 32);
        const double tsq = block_sum_fixed<kSpmvThreads>(red.part_d, W);
        const unsigned long long tsk = block_sum_u64<kSpmvThreads>(red.part_u, W);
        const float tmax = block_max_f<kSpmvThreads>(red.part_f, W);
        if (threadIdx.x == 0) {
            if (out.sumsq) *out.sumsq = tsq;
            if (out.skipped) *out.skipped = tsk;
            if (out.skipped_d) *out.skipped_d = (double)tsk;
            if (out.absmax) *out.absmax = tmax;
            *red.counter = 0;
            if (hooks.t_accum && hooks.t_begin)
                *hooks.t_accum += globaltimer() - *hooks.t_begin;
        }
    }
}

// ---------------------------------------------------------------------------
// WC fp32: per-coefficient dots + fixed-point fascicle accumulation
// ---------------------------------------------------------------------------
using WcFix = FixParams;

template <int NT, bool FULL>
__global__ void __launch_bounds__(kSpmvThreads, 1)
    k_wc_f32(const FastArgs A, const float *__restrict__ y, const WcFix fx,
             const CallHooks hooks)
{
    extern __shared__ __align__(128) float Ds[];
    __shared__ __align__(8) uint64_t bar;
    if (hooks.done && *hooks.done) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (kSpmvThreads / 32) + (threadIdx.x >> 5);
    if (hooks.t_begin && blockIdx.x == 0 && threadIdx.x == 0) *hooks.t_begin = globaltimer();
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned parity = 0;
    const int nt = A.nt;
    const int ex = fix_exponent(fx, nt);
    const double scale = ldexp(1.0, ex);
    const int vb = A.wpart[gw], ve = A.wpart[gw + 1];

    for (int g = 0; g < A.G; ++g) {
        stage_slice(Ds, A, g, &bar, parity);
        if (vb >= ve) continue;
        const uint32_t *gp = A.gptr + (size_t)g * A.nv;
        VoxelCursor cur{gp, ve, 0, 0};
        cur.load(vb, lane);
        const uint32_t kb = gp[vb];
        const uint32_t kend = gp[ve];
        int cv = vb;
        uint32_t ce = cur.end_of(cv, lane);
        float yv[NT];
        // skip leading empty voxels lazily: rows load when first used
        bool loaded = false;

        for (uint32_t base = kb; base < kend; base += 32) {
            const uint32_t k = base + lane;
            const bool valid = k < kend;
            uint32_t a = 0, f = 0;
            float vv = 0.f;
            if (valid) {
                a = ld_stream(A.atom + k);
                f = ld_stream(A.fiber + k);
                vv = ld_stream(A.val + k);
            }
            float p[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t kj = base + j;
                p[j] = 0.f;
                if (kj < kend) {
                    if (kj >= ce || !loaded) {
                        while (kj >= ce) {
                            ++cv;
                            ce = cur.end_of(cv, lane);
                        }
                        const size_t yo = (size_t)cv * nt;
#pragma unroll
                        for (int q = 0; q < NT; ++q) {
                            const int t = lane + 32 * q;
                            yv[q] = (FULL || t < nt) ? y[yo + t] : 0.f;
                        }
                        loaded = true;
                    }
                    const uint32_t aj = __shfl_sync(0xffffffffu, a, j);
                    const float *dr = Ds + aj * nt;
                    float d = 0.f;
#pragma unroll
                    for (int q = 0; q < NT; ++q) {
                        const int t = lane + 32 * q;
                        if (FULL || t < nt) d = fmaf(yv[q], dr[t], d);
                    }
                    p[j] = d;
                }
            }
            // transposing butterfly: lane L ends with sum over lanes of p[L]
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
                const bool up = (lane & s) != 0;
#pragma unroll
                for (int i = 0; i < s; ++i) {
                    const float send = up ? p[i] : p[i + s];
                    const float keep = up ? p[i + s] : p[i];
                    p[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
                }
            }
            if (valid) {
                const float z = p[0] * vv;
                const long long qv = __double2ll_rn((double)z * scale);
                atomicAdd(fx.wfix + f, static_cast<unsigned long long>(qv));
            }
        }
    }
    if (hooks.t_accum && hooks.t_begin) {
        // timing closes in the finalize kernel (stream order)
    }
}

// w_out = fixed-point sum (+ w_out if ACCUMULATE), optional projected-gradient
// epilogue (sbbnnls.project_gradient, sbbnnls.py:107-116); resets wfix.
template <int BT>
__global__ void __launch_bounds__(BT)
    k_wc_finalize(unsigned long long *__restrict__ wfix, float *__restrict__ w_out,
                  const float *__restrict__ w_ref, int nf, uint32_t flags,
                  const WcFix fx, int nt, double *part, unsigned *counter,
                  double *sumsq_out, const CallHooks hooks)
{
    if (hooks.done && *hooks.done) return;
    const int ex = fix_exponent(fx, nt);
    const double inv = ldexp(1.0, -ex);
    const bool accumulate = flags & LIFE_ACCUMULATE;
    const bool project = (flags & LIFE_PROJECT_GRAD) && w_ref != nullptr;
    double sq = 0.0;
    for (int f = blockIdx.x * BT + threadIdx.x; f < nf; f += gridDim.x * BT) {
        const long long q = static_cast<long long>(wfix[f]);
        wfix[f] = 0ull;
        float o = static_cast<float>((double)q * inv);
        if (accumulate) o = w_out[f] + o;
        if (project && w_ref[f] == 0.f && o > 0.f) o = 0.f;
        w_out[f] = o;
        sq += (double)o * (double)o;
    }
    __shared__ double s[BT];
    s[threadIdx.x] = sq;
    __syncthreads();
    for (int w = BT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
    if (last_block_arrive<BT>(counter)) {
        const double tot = block_sum_fixed<BT>(part, gridDim.x);
        if (threadIdx.x == 0) {
            if (sumsq_out) *sumsq_out = tot;
            *counter = 0;
            if (hooks.t_accum && hooks.t_begin)
                *hooks.t_accum += globaltimer() - *hooks.t_begin;
        }
    }
}

template <int BT>
__global__ void __launch_bounds__(BT)
    k_absmax_f32(const float *__restrict__ x, int64_t n, float *part,
                 unsigned *counter, float *out)
{
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)BT + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * BT)
        m = fmaxf(m, fabsf(x[i]));
    __shared__ float s[BT];
    s[threadIdx.x] = m;
    __syncthreads();
    for (int w = BT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] = fmaxf(s[threadIdx.x], s[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
    if (last_block_arrive<BT>(counter)) {
        const float r = block_max_f<BT>(part, gridDim.x);
        if (threadIdx.x == 0) {
            *out = r;
            *counter = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// fp64 exact kernels (bitwise equal to the reference sequential loops)
// ---------------------------------------------------------------------------
// DSC: per voxel, y[v*nt+t] accumulates in storage (stable-sort) order with
// s = w[f]*value hoisted (_kernels.py:23-32).  Lane = direction.
__global__ void __launch_bounds__(256)
    k_dsc_f64_exact(const uint32_t *__restrict__ atom, const uint32_t *__restrict__ fiber,
                    const double *__restrict__ val, const uint32_t *__restrict__ ptr,
                    const int *__restrict__ wpart, const double *__restrict__ D,
                    const double *__restrict__ w, double *__restrict__ y, int nt,
                    int skip_zero, unsigned long long *skipped_out, ReduceSlots red)
{
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int vb = wpart[gw], ve = wpart[gw + 1];
    unsigned long long skipped = 0;
    for (int v = vb; v < ve; ++v) {
        const uint32_t s = ptr[v], e = ptr[v + 1];
        if (s == e) continue;
        for (int t0 = 0; t0 < nt; t0 += 32) {
            const int t = t0 + lane;
            const bool tv = t < nt;
            double acc = tv ? y[(size_t)v * nt + t] : 0.0;
            for (uint32_t base = s; base < e; base += 32) {
                const uint32_t k = base + lane;
                const bool valid = k < e;
                uint32_t a = 0;
                double sc = 0.0;
                if (valid) {
                    a = atom[k];
                    sc = __dmul_rn(w[fiber[k]], val[k]);
                }
                const unsigned zm = __ballot_sync(0xffffffffu, valid && sc == 0.0);
                if (t0 == 0 && skip_zero) skipped += __popc(zm);  // counted only when skipping (_kernels.py:25-28)
                unsigned m = __ballot_sync(0xffffffffu, valid);
                if (skip_zero) m &= ~zm;
                while (m) {
                    const int j = __ffs(m) - 1;
                    m &= m - 1;
                    const uint32_t aj = __shfl_sync(0xffffffffu, a, j);
                    const double sj = __shfl_sync(0xffffffffu, sc, j);
                    if (tv) acc = __dadd_rn(acc, __dmul_rn(D[(size_t)aj * nt + t], sj));
                }
            }
            if (tv) y[(size_t)v * nt + t] = acc;
        }
    }
    if (lane == 0) red.part_u[gw] = skipped;
    if (last_block_arrive<256>(red.counter)) {
        const unsigned long long tot = block_sum_u64<256>(red.part_u, gridDim.x * 8);
        if (threadIdx.x == 0) {
            if (skipped_out) *skipped_out = tot;
            *red.counter = 0;
        }
    }
}

// WC: per coefficient acc = sum_t y*D strictly in t order, then
// w[f] += acc*value in storage order within each fascicle
// (_kernels.py:61-67).  Lane = coefficient, then an in-order fold.
__global__ void __launch_bounds__(256)
    k_wc_f64_exact(const uint32_t *__restrict__ atom, const uint32_t *__restrict__ voxel,
                   const uint32_t *__restrict__ fiber, const double *__restrict__ val,
                   const uint32_t *__restrict__ ptr, const int *__restrict__ wpart,
                   const double *__restrict__ D, const double *__restrict__ y,
                   double *__restrict__ w, int nt)
{
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int fb = wpart[gw], fe = wpart[gw + 1];
    if (fb >= fe) return;
    const uint32_t kb = ptr[fb], ke = ptr[fe];
    int curf = -1;
    double cur = 0.0;
    for (uint32_t base = kb; base < ke; base += 32) {
        const uint32_t k = base + lane;
        const bool valid = k < ke;
        double c = 0.0;
        int f = -1;
        if (valid) {
            const double *row = D + (size_t)atom[k] * nt;
            const double *sig = y + (size_t)voxel[k] * nt;
            double acc = 0.0;
            for (int t = 0; t < nt; ++t) acc = __dadd_rn(acc, __dmul_rn(sig[t], row[t]));
            c = __dmul_rn(acc, val[k]);
            f = (int)fiber[k];
        }
        const int cnt = min(32u, ke - base);
        for (int j = 0; j < cnt; ++j) {
            const int fj = __shfl_sync(0xffffffffu, f, j);
            const double cj = __shfl_sync(0xffffffffu, c, j);
            if (fj != curf) {
                if (curf >= 0 && lane == 0) w[curf] = cur;
                curf = fj;
                cur = w[fj];
            }
            cur = __dadd_rn(cur, cj);
        }
    }
    if (curf >= 0 && lane == 0) w[curf] = cur;
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <int NT, bool FULL>
static int launch_dsc_t(life_phi *phi, const float *w, float *y, const float *b,
                        uint32_t flags, const DscOut &o, const CallHooks &h,
                        cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_dsc_f32<NT, FULL>, phi->smem));
    FastArgs A{phi->atom, phi->fiber, phi->val, phi->gptr, phi->wpart, phi->Dg,
               phi->nv, phi->nt, phi->G, phi->ag, phi->na, phi->slice_floats};
    k_dsc_f32<NT, FULL><<<phi->nblocks, kSpmvThreads, phi->smem, st>>>(
        A, w, y, b, flags, phi->red, o, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int NT, bool FULL>
static int launch_wc_t(life_phi *phi, const float *y, const WcFix &fx,
                       const CallHooks &h, cudaStream_t st)
{
    LIFE_TRY(ensure_smem(k_wc_f32<NT, FULL>, phi->smem));
    FastArgs A{phi->atom, phi->fiber, phi->val, phi->gptr, phi->wpart, phi->Dg,
               phi->nv, phi->nt, phi->G, phi->ag, phi->na, phi->slice_floats};
    k_wc_f32<NT, FULL><<<phi->nblocks, kSpmvThreads, phi->smem, st>>>(A, y, fx, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

#define LIFE_NT_DISPATCH(FN, ...)                                              \
    switch ((phi->nt + 31) / 32) {                                             \
    case 1: return (phi->nt == 32) ? FN<1, true>(__VA_ARGS__) : FN<1, false>(__VA_ARGS__); \
    case 2: return (phi->nt == 64) ? FN<2, true>(__VA_ARGS__) : FN<2, false>(__VA_ARGS__); \
    case 3: return (phi->nt == 96) ? FN<3, true>(__VA_ARGS__) : FN<3, false>(__VA_ARGS__); \
    case 4: return (phi->nt == 128) ? FN<4, true>(__VA_ARGS__) : FN<4, false>(__VA_ARGS__); \
    case 5: return (phi->nt == 160) ? FN<5, true>(__VA_ARGS__) : FN<5, false>(__VA_ARGS__); \
    case 6: return (phi->nt == 192) ? FN<6, true>(__VA_ARGS__) : FN<6, false>(__VA_ARGS__); \
    case 7: return (phi->nt == 224) ? FN<7, true>(__VA_ARGS__) : FN<7, false>(__VA_ARGS__); \
    case 8: return (phi->nt == 256) ? FN<8, true>(__VA_ARGS__) : FN<8, false>(__VA_ARGS__); \
    case 9: return (phi->nt == 288) ? FN<9, true>(__VA_ARGS__) : FN<9, false>(__VA_ARGS__); \
    case 10: return (phi->nt == 320) ? FN<10, true>(__VA_ARGS__) : FN<10, false>(__VA_ARGS__); \
    default: return fail(LIFE_ERR_CONFIG_INVALID, "unsupported n_dirs");     \
    }

static int launch_dsc_sparse(life_phi *phi, const float *w, float *y, const float *b,
                             uint32_t flags, const DscOut &o, const CallHooks &h,
                             cudaStream_t st)
{
    LIFE_NT_DISPATCH(launch_dsc_t, phi, w, y, b, flags, o, h, st);
}

static int launch_dsc_kernel(life_phi *phi, const float *w, float *y, const float *b,
                             uint32_t flags, const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    if (phi->has_bin) return launch_dsc_bin(phi, w, y, b, flags, o, h, st);
    return launch_dsc_sparse(phi, w, y, b, flags, o, h, st);
}

__global__ void k_zero_skips(unsigned long long *sk, double *skd, const int *done)
{
    if (done && *done) return;
    if (sk) *sk = 0ull;
    if (skd) *skd = 0.0;
}

int launch_dsc(life_phi *phi, const float *w, float *y, const float *b,
               uint32_t flags, const DscOut &o, const CallHooks &h, cudaStream_t st)
{
    LIFE_TRY(launch_dsc_kernel(phi, w, y, b, flags, o, h, st));
    if (!(flags & LIFE_SKIP_ZERO) && (o.skipped || o.skipped_d)) {
        // KernelStats.skipped_coefficients is 0 when skip_zero is off
        // (_kernels.dsc_range counts only skipped products, _kernels.py:25-28)
        k_zero_skips<<<1, 1, 0, st>>>(o.skipped, o.skipped_d, h.done);
        LIFE_CHECK_LAUNCH();
    }
    return LIFE_OK;
}

static int launch_wc_sparse(life_phi *phi, const float *y, const WcFix &fx,
                            const CallHooks &h, cudaStream_t st)
{
    LIFE_NT_DISPATCH(launch_wc_t, phi, y, fx, h, st);
}

int launch_wc_main(life_phi *phi, const float *y, const WcFix &fx,
                   const CallHooks &h, cudaStream_t st)
{
    return launch_wc_sparse(phi, y, fx, h, st);
}

int launch_absmax(life_phi *phi, const float *x, int64_t n, float *out,
                  cudaStream_t st)
{
    const int blocks = std::max(1, std::min<int>(phi->sms * 4, (int)((n + 255) / 256)));
    k_absmax_f32<256><<<blocks, 256, 0, st>>>(x, n, phi->part_d2 ? reinterpret_cast<float *>(phi->part_d2) : nullptr,
                                             phi->counter2, out);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

template <int NT, bool FULL>
static int prepare_t(life_phi *phi)
{
    LIFE_TRY(ensure_smem(k_dsc_f32<NT, FULL>, phi->smem));
    LIFE_TRY(ensure_smem(k_wc_f32<NT, FULL>, phi->smem));
    return LIFE_OK;
}

static int prepare_sparse(life_phi *phi) { LIFE_NT_DISPATCH(prepare_t, phi); }

int prepare_spmv(life_phi *phi)
{
    if (phi->has_bin) return LIFE_OK;  // prepared at build (prepare_bin)
    return prepare_sparse(phi);
}

int launch_wc(life_phi *phi, const float *y, float *w, const float *w_ref,
              const float *ymax_dev, const double *ysumsq_dev, uint32_t flags, double *sumsq,
              const CallHooks &h, const life_comm *comm, cudaStream_t st,
              const float *yvbound_dev, const WcScalars *sc)
{
    if (phi->has_bin) {
        if (!ymax_dev && !ysumsq_dev && !yvbound_dev) {
            LIFE_TRY(launch_absmax(phi, y, (int64_t)phi->nv * phi->nt, phi->ybound, st));
            ymax_dev = phi->ybound;
        }
        FixParams fb{phi->wfix, ymax_dev, ysumsq_dev, phi->vmax, phi->dmax, (double)phi->fmax_nnz, yvbound_dev};
        return launch_wc_bin(phi, y, w, w_ref, fb, flags, sumsq, h, comm, st, sc);
    }
    if (comm && sc)  // other layouts: the scalars first (the scale needs the global sum of squares)
        for (int k = 0; k < sc->n; ++k)
            if (comm->allreduce(sc->v[k], 1, LIFE_DT_F64, LIFE_OP_SUM, st, comm->ctx) != 0)
                return fail(LIFE_ERR_NCCL, "allreduce(scalar) failed");
    if (!ymax_dev && !ysumsq_dev) {
        LIFE_TRY(launch_absmax(phi, y, (int64_t)phi->nv * phi->nt, phi->ybound, st));
        ymax_dev = phi->ybound;
    }
    WcFix fx{phi->wfix, ymax_dev, ysumsq_dev, phi->vmax, phi->dmax, (double)phi->fmax_nnz};
    LIFE_TRY(launch_wc_main(phi, y, fx, h, st));
    if (comm) {
        // fascicle partial sums of all voxel shards: integer sum, so every
        // rank gets bit-identical totals whatever the reduction order
        const int rc = comm->allreduce(phi->wfix, phi->nf, LIFE_DT_I64, LIFE_OP_SUM, st,
                                       comm->ctx);
        if (rc != 0) return fail(LIFE_ERR_NCCL, "allreduce(wfix) failed");
    }
    const int blocks = std::max(1, std::min(phi->sms * 4, (phi->nf + 255) / 256));
    k_wc_finalize<256><<<blocks, 256, 0, st>>>(phi->wfix, w, w_ref, phi->nf, flags, fx,
                                               phi->nt, phi->part_d2, phi->counter2,
                                               sumsq, h);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

}  // namespace life

using namespace life;

extern "C" {

int life_dsc_f32(life_phi *phi, const float *w, float *y, const float *b,
                 uint32_t flags, const life_spmv_out *out, void *stream)
{
    if (!phi || !w || !y) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (!phi->has_fast && !phi->has_bin)
        return fail(LIFE_ERR_CONFIG_INVALID, "operator has no fp32 layout");
    if ((flags & LIFE_SUBTRACT_B) && !b) return fail(LIFE_ERR_INVALID_ARGUMENT, "LIFE_SUBTRACT_B needs b");
    if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(y) |
         reinterpret_cast<uintptr_t>(b)) & 15u)
        return fail(LIFE_ERR_INVALID_ARGUMENT, "w, y and b must be 16-byte aligned");
    DscOut o{nullptr, nullptr, nullptr, nullptr};
    if (out) o = DscOut{out->skipped, out->sumsq, out->absmax, nullptr};
    CallHooks h{nullptr, nullptr, nullptr};
    LIFE_TRY(launch_dsc(phi, w, y, b, flags, o, h, static_cast<cudaStream_t>(stream)));
    return ok();
}

int life_wc_f32(life_phi *phi, const float *y, float *w, const float *w_ref,
                const float *y_absmax_dev, uint32_t flags,
                const life_spmv_out *out, void *stream)
{
    if (!phi || !w || !y) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (!phi->has_fast && !phi->has_bin)
        return fail(LIFE_ERR_CONFIG_INVALID, "operator has no fp32 layout");
    if ((flags & LIFE_PROJECT_GRAD) && !w_ref)
        return fail(LIFE_ERR_INVALID_ARGUMENT, "LIFE_PROJECT_GRAD needs w_ref");
    if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(y) |
         reinterpret_cast<uintptr_t>(w_ref)) & 15u)
        return fail(LIFE_ERR_INVALID_ARGUMENT, "y, w and w_ref must be 16-byte aligned");
    CallHooks h{nullptr, nullptr, nullptr};
    LIFE_TRY(launch_wc(phi, y, w, w_ref, y_absmax_dev, nullptr, flags,
                       out ? out->sumsq : nullptr, h, nullptr, static_cast<cudaStream_t>(stream)));
    return ok();
}

int life_dsc_f64(life_phi *phi, const double *w, double *y, uint32_t flags,
                 unsigned long long *skipped_dev, void *stream)
{
    if (!phi || !w || !y) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (!phi->has_exact) return fail(LIFE_ERR_CONFIG_INVALID, "operator built without LIFE_PHI_EXACT_F64");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_dsc_f64_exact<<<phi->xblocks, 256, 0, st>>>(
        phi->xv_atom, phi->xv_fiber, phi->xv_val, phi->xv_ptr, phi->xv_wpart, phi->D64, w,
        y, phi->nt, (flags & LIFE_SKIP_ZERO) ? 1 : 0, skipped_dev, phi->red);
    LIFE_CHECK_LAUNCH();
    return ok();
}

int life_wc_f64(life_phi *phi, const double *y, double *w, void *stream)
{
    if (!phi || !w || !y) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (!phi->has_exact) return fail(LIFE_ERR_CONFIG_INVALID, "operator built without LIFE_PHI_EXACT_F64");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_wc_f64_exact<<<phi->xblocks, 256, 0, st>>>(phi->xf_atom, phi->xf_voxel, phi->xf_fiber,
                                                 phi->xf_val, phi->xf_ptr, phi->xf_wpart,
                                                 phi->D64, y, w, phi->nt);
    LIFE_CHECK_LAUNCH();
    return ok();
}

}  // extern "C"
