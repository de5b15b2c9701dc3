// life_solver.cu -- SBBNNLS (Alg. 1 of arXiv:1905.06234) on the device.
//
// Reference: sbbnnls.solve (/root/reference/pkg/src/lifespmv/sbbnnls.py:223-291)
//   r  = M w - b                      (DSC, fused residual + <r,r>)
//   g~ = project_gradient(M^T r, w)   (WC, fused projection + <g~,g~>)
//   stop if ||g~|| < grad_tol
//   mg = M g~                         (DSC, fused <mg,mg>)
//   odd  i: alpha = <g~,g~> / <mg,mg>
//   even i: alpha = <mg,mg> / <M^T mg, M^T mg>   (one more WC)
//   stop if the denominator is 0 (DegenerateStep)
//   w  = max(w - alpha g~, 0)         (fused zero count, min, trace record)
// All scalars stay on the device; kernels no-op once a device `done` flag is
// set, so whole iteration pairs (odd+even) are replayed as one CUDA graph and
// the host only polls the flag every `poll_every` iterations.
#include <algorithm>
#include <cmath>
#include <vector>

#include "life_common.cuh"

namespace life {


struct Scal {
    // rr/skipped_d and mgmg/pad are adjacent: each pair is one all-reduce
    double rr, skipped_d, mgmg, mg_pad;
    double gg, mtmg2, alpha, obj, init_obj, final_obj;
    double bb, m1;            // ||b||^2, ||M 1||^2 for the default w0
    double vS, vB;            // voxel-sharded runs: max_v sum ||D_a|| |val| and max_v ||b_v|| (all ranks)
    float ybound, yb_pad;     // bound on max_v ||y_v|| of the next WC input
    unsigned vmax_bits, vcount;
    unsigned long long t_begin, dsc_ns, wc_ns;
    int done, term, iter, max_iters;
    double grad_tol;
};

// ---- tiny control kernels (single thread) ----------------------------------
__global__ void k_check_grad(Scal *s)
{
    if (s->done) return;
    s->obj = 0.5 * s->rr;
    if (s->iter == 1) s->init_obj = s->obj;
    const double gn = sqrt(s->gg);
    if (gn < s->grad_tol) {
        s->done = 1;
        s->term = LIFE_TERM_GRAD_TOL;
        s->final_obj = s->obj;
    }
}

__global__ void k_alpha(Scal *s, int even)
{
    if (s->done) return;
    const double num = even ? s->mgmg : s->gg;
    const double den = even ? s->mtmg2 : s->mgmg;
    if (den == 0.0) {
        s->done = 1;
        s->term = LIFE_TERM_DEGENERATE;
        s->final_obj = s->obj;
        return;
    }
    s->alpha = num / den;
}

template <typename T>
__global__ void k_w0_scale(const Scal *s, T *w, int nf)
{
    // w0 = ones * ||b|| / max(||M 1||, 1e-300)   (sbbnnls.py:237-240)
    const double scale = sqrt(s->bb) / fmax(sqrt(s->m1), 1e-300);
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x)
        w[f] = (T)(1.0 * scale);
}

template <typename T>
__global__ void k_fill(T *x, int64_t n, T v)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

template <typename T>
__global__ void k_project_nonneg(T *w, int n)
{
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x)
        w[f] = (w[f] >= T(0) || w[f] != w[f]) ? w[f] : T(0);  // np.maximum(v, 0): NaN propagates
}

// Bound on max_v ||y_v||_2 of the next WC input, identical on every rank
// before any collective (w and g~ are replicated):
//   y = M x - b:  ||y_v|| <= vS max|x| + vB;   y = M x:  ||y_v|| <= vS max|x|.
// Sets the WC fixed-point scale of voxel-sharded runs (FixParams::yvbound).
__global__ void __launch_bounds__(256) k_vbound(const float *__restrict__ x, int nf, Scal *s, int with_b)
{
    if (s->done) return;
    float m = 0.f;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(x[f]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s->vmax_bits, __float_as_uint(m));
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&s->vcount, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const double xm = (double)__uint_as_float(atomicAdd(&s->vmax_bits, 0u));
        const double b = s->vS * xm + (with_b ? s->vB : 0.0);
        s->ybound = (float)(b * (1.0 + 1e-5));
        s->vmax_bits = 0u;
        s->vcount = 0u;
    }
}

// max_v ||b_v||_2 into s->vB (before the MAX all-reduce of (vS, vB))
__global__ void __launch_bounds__(256) k_bnorm_max(const float *__restrict__ b, int nv, int nt, Scal *s)
{
    double m = 0.0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
        double q = 0.0;
        for (int t = 0; t < nt; ++t) q += (double)b[(size_t)v * nt + t] * (double)b[(size_t)v * nt + t];
        m = fmax(m, sqrt(q));
    }
    atomicMax(reinterpret_cast<unsigned long long *>(&s->vB), (unsigned long long)__double_as_longlong(m));
}

template <int BT>
__device__ __forceinline__ bool last_arrive(unsigned *counter)
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

// w = max(w - alpha g~, 0); zeros, min(w); writes the trace record and
// advances the iteration counter (sbbnnls.py:270-283).
template <typename T, int BT>
__global__ void __launch_bounds__(BT)
    k_update(T *__restrict__ w, const T *__restrict__ gt, int nf, Scal *s,
             life_trace_record *rec, double *part_min, unsigned long long *part_z,
             unsigned *counter, int even)
{
    if (s->done) return;
    const T alpha = (T)s->alpha;
    unsigned long long z = 0;
    T mn = T(INFINITY);
    for (int f = blockIdx.x * BT + threadIdx.x; f < nf; f += gridDim.x * BT) {
        T v = w[f] - alpha * gt[f];
        v = (v >= T(0) || v != v) ? v : T(0);  // np.maximum(v, 0.0): NaN propagates, -0 stays
        w[f] = v;
        z += (v == T(0)) ? 1ull : 0ull;
        mn = fmin(mn, v);
    }
    __shared__ double smn[BT];
    __shared__ unsigned long long sz[BT];
    smn[threadIdx.x] = (double)mn;
    sz[threadIdx.x] = z;
    __syncthreads();
    for (int o = BT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + o]);
            sz[threadIdx.x] += sz[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_min[blockIdx.x] = smn[0];
        part_z[blockIdx.x] = sz[0];
    }
    if (last_arrive<BT>(counter)) {
        // the block's threads fold the per-block partials (fixed order:
        // strided, then the shared-memory tree)
        double m = INFINITY;
        unsigned long long zz = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += BT) {
            m = fmin(m, __ldcg(part_min + b));
            zz += __ldcg(part_z + b);
        }
        smn[threadIdx.x] = m;
        sz[threadIdx.x] = zz;
        __syncthreads();
        for (int o = BT / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) {
                smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + o]);
                sz[threadIdx.x] += sz[threadIdx.x + o];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            m = smn[0];
            zz = sz[0];
            const int it = s->iter;
            life_trace_record r;
            r.iteration = it;
            r.zeros = (int)zz;
            r.dsc_skipped = (int64_t)s->skipped_d;
            r.objective = s->obj;
            r.alpha = s->alpha;
            r.grad_norm = sqrt(s->gg);
            r.w_min = nf ? m : 0.0;
            r.dsc_seconds = 1e-9 * (double)s->dsc_ns;
            r.wc_seconds = 1e-9 * (double)s->wc_ns;
            r.dsc_calls = 2;
            r.wc_calls = even ? 2 : 1;
            if (rec) rec[it - 1] = r;
            s->dsc_ns = 0;
            s->wc_ns = 0;
            s->iter = it + 1;
            if (it >= s->max_iters) {
                s->done = 1;
                s->term = LIFE_TERM_MAX_ITERS;
            }
            *counter = 0;
        }
    }
}

// ---- fp64 exact-mode vector kernels (deterministic reductions) -------------
// mode 0: out = x - b ; 1: out = project_gradient(x, w) ; 2: out = x
// accumulates sum(out^2) into *sum
template <int BT>
__global__ void __launch_bounds__(BT)
    k_vec64(double *__restrict__ x, const double *__restrict__ aux, int64_t n, int mode,
            double *part, unsigned *counter, double *sum, const int *done)
{
    if (done && *done) return;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)BT + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * BT) {
        double v = x[i];
        if (mode == 0) v = v - aux[i];
        if (mode == 1 && aux[i] == 0.0 && v > 0.0) v = 0.0;
        x[i] = v;
        sq += v * v;
    }
    __shared__ double s[BT];
    s[threadIdx.x] = sq;
    __syncthreads();
    for (int o = BT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
    if (last_arrive<BT>(counter)) {
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(part + b);
            *sum = t;
            *counter = 0;
        }
    }
}

template <typename T, int BT>
__global__ void __launch_bounds__(BT)
    k_sumsq(const T *__restrict__ x, int64_t n, double *part, unsigned *counter, double *sum)
{
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)BT + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * BT)
        sq += (double)x[i] * (double)x[i];
    __shared__ double s[BT];
    s[threadIdx.x] = sq;
    __syncthreads();
    for (int o = BT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
    if (last_arrive<BT>(counter)) {
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(part + b);
            *sum = t;
            *counter = 0;
        }
    }
}

__global__ void k_set_skipped(Scal *s, const unsigned long long *src)
{
    if (!s->done) s->skipped_d = (double)*src;
}

template <typename T>
static int blocks_for(const life_phi *phi, int64_t n)
{
    return (int)std::max<int64_t>(1, std::min<int64_t>(phi->sms * 4, (n + 255) / 256));
}

struct Solver {
    life_phi *phi;
    cudaStream_t st;
    bool exact;
    int skip;
    Scal *s = nullptr;
    life_trace_record *rec = nullptr;
    void *r = nullptr, *mg = nullptr, *gt = nullptr, *mtmg = nullptr;
    double *part = nullptr;
    unsigned long long *partz = nullptr;
    unsigned *counter = nullptr;
    unsigned long long *skipped_dev = nullptr;
    int nblk_f = 1;
    const life_comm *comm = nullptr;
};

// Enqueue an all-reduce through the caller's communicator (multi-GPU only).
static int comm_reduce(const Solver &S, void *buf, int64_t count, int dtype, int op)
{
    if (!S.comm) return LIFE_OK;
    if (S.comm->allreduce(buf, count, dtype, op, S.st, S.comm->ctx) != 0)
        return fail(LIFE_ERR_NCCL, "solver all-reduce failed");
    return LIFE_OK;
}

// One iteration, fp32 fast path.
static int iter_fast(Solver &S, const float *b, float *w, int even)
{
    life_phi *phi = S.phi;
    Scal *s = S.s;
    CallHooks hd{&s->done, &s->t_begin, &s->dsc_ns};
    CallHooks hw{&s->done, &s->t_begin, &s->wc_ns};
    float *r = (float *)S.r, *mg = (float *)S.mg, *gt = (float *)S.gt,
          *mtmg = (float *)S.mtmg;
    const uint32_t skip = S.skip ? LIFE_SKIP_ZERO : 0u;
    // r = M w - b; the WC fixed-point scale comes from sqrt(sum r^2), one
    // scalar that multi-GPU runs reduce together with the skip count
    LIFE_TRY(launch_dsc(phi, w, r, b, LIFE_SUBTRACT_B | skip,
                        DscOut{nullptr, &s->rr, nullptr, &s->skipped_d}, hd, S.st));
    // voxel-sharded runs: the WC scale comes from a bound every rank computes
    // alike, so this iteration's DSC scalars ride in the tail of the WC
    // all-reduce (one collective per WC)
    const float *yb = nullptr;
    if (S.comm) {
        k_vbound<<<S.nblk_f, 256, 0, S.st>>>(w, phi->nf, s, 1);
        LIFE_CHECK_LAUNCH();
        yb = &s->ybound;
    }
    const WcScalars sc_r{{&s->rr, &s->skipped_d, nullptr}, 2};
    LIFE_TRY(launch_wc(phi, r, gt, w, nullptr, &s->rr, LIFE_PROJECT_GRAD, &s->gg, hw, S.comm,
                       S.st, yb, S.comm ? &sc_r : nullptr));
    k_check_grad<<<1, 1, 0, S.st>>>(s);
    LIFE_CHECK_LAUNCH();
    LIFE_TRY(launch_dsc(phi, gt, mg, nullptr, skip, DscOut{nullptr, &s->mgmg, nullptr, nullptr},
                        hd, S.st));
    if (even) {
        if (S.comm) {
            k_vbound<<<S.nblk_f, 256, 0, S.st>>>(gt, phi->nf, s, 0);
            LIFE_CHECK_LAUNCH();
        }
        const WcScalars sc_m{{&s->mgmg, nullptr, nullptr}, 1};
        LIFE_TRY(launch_wc(phi, mg, mtmg, nullptr, nullptr, &s->mgmg, 0u, &s->mtmg2, hw, S.comm,
                           S.st, yb, S.comm ? &sc_m : nullptr));
    } else {
        LIFE_TRY(comm_reduce(S, &s->mgmg, 1, LIFE_DT_F64, LIFE_OP_SUM));  // ||M g~||^2 for alpha
    }
    k_alpha<<<1, 1, 0, S.st>>>(s, even);
    LIFE_CHECK_LAUNCH();
    k_update<float, 256><<<S.nblk_f, 256, 0, S.st>>>(w, gt, phi->nf, s, S.rec, S.part,
                                                     S.partz, S.counter, even);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

// One iteration, fp64 exact kernels.
static int iter_exact(Solver &S, const double *b, double *w, int even)
{
    life_phi *phi = S.phi;
    Scal *s = S.s;
    const int64_t ny = (int64_t)phi->nv * phi->nt;
    double *r = (double *)S.r, *mg = (double *)S.mg, *gt = (double *)S.gt,
           *mtmg = (double *)S.mtmg;
    const int by = blocks_for<double>(phi, ny), bf = blocks_for<double>(phi, phi->nf);
    // exact kernels have no done-gate: stop launching once done is visible
    LIFE_CUDA(cudaMemsetAsync(r, 0, ny * sizeof(double), S.st));
    LIFE_TRY(life_dsc_f64(phi, w, r, S.skip ? LIFE_SKIP_ZERO : 0u, S.skipped_dev, S.st));
    k_set_skipped<<<1, 1, 0, S.st>>>(s, S.skipped_dev);
    LIFE_CHECK_LAUNCH();
    k_vec64<256><<<by, 256, 0, S.st>>>(r, b, ny, 0, S.part, S.counter, &s->rr, &s->done);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaMemsetAsync(gt, 0, phi->nf * sizeof(double), S.st));
    LIFE_TRY(life_wc_f64(phi, r, gt, S.st));
    k_vec64<256><<<bf, 256, 0, S.st>>>(gt, w, phi->nf, 1, S.part, S.counter, &s->gg, &s->done);
    LIFE_CHECK_LAUNCH();
    k_check_grad<<<1, 1, 0, S.st>>>(s);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaMemsetAsync(mg, 0, ny * sizeof(double), S.st));
    LIFE_TRY(life_dsc_f64(phi, gt, mg, S.skip ? LIFE_SKIP_ZERO : 0u, S.skipped_dev + 1, S.st));
    k_vec64<256><<<by, 256, 0, S.st>>>(mg, nullptr, ny, 2, S.part, S.counter, &s->mgmg, &s->done);
    LIFE_CHECK_LAUNCH();
    if (even) {
        LIFE_CUDA(cudaMemsetAsync(mtmg, 0, phi->nf * sizeof(double), S.st));
        LIFE_TRY(life_wc_f64(phi, mg, mtmg, S.st));
        k_vec64<256><<<bf, 256, 0, S.st>>>(mtmg, nullptr, phi->nf, 2, S.part, S.counter,
                                           &s->mtmg2, &s->done);
        LIFE_CHECK_LAUNCH();
    }
    k_alpha<<<1, 1, 0, S.st>>>(s, even);
    LIFE_CHECK_LAUNCH();
    k_update<double, 256><<<bf, 256, 0, S.st>>>(w, gt, phi->nf, s, S.rec, S.part, S.partz,
                                                S.counter, even);
    LIFE_CHECK_LAUNCH();
    return LIFE_OK;
}

}  // namespace life

using namespace life;

// ---- solver session --------------------------------------------------------
struct life_sbb {
    Solver S;
    life_solver_config cfg;
    const void *b;
    void *w;
    int next_iter = 1;            // next iteration index to enqueue
    int64_t dsc_calls = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    size_t graph_kernels = 0;
    int *pinned = nullptr;
};

static void free_session(life_sbb *x)
{
    if (!x) return;
    Solver &S = x->S;
    cudaDeviceSynchronize();  // as cudaFree would: the blocks go back to the cache
    if (x->gexec) cudaGraphExecDestroy(x->gexec);
    if (x->graph) cudaGraphDestroy(x->graph);
    pinned_free(x->pinned);
    void *bufs[] = {S.s, S.rec, S.r, S.mg, S.gt, S.mtmg, S.part, S.partz, S.counter,
                    S.skipped_dev};
    for (void *p : bufs)
        dev_free(p);
    delete x;
}

extern "C" int life_sbb_create(life_phi *phi, const void *b_dev, void *w_dev,
                               const life_solver_config *cfg, void *stream, life_sbb **out)
{
    if (!phi || !b_dev || !w_dev || !cfg || !out)
        return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (cfg->max_iters < 1) return fail(LIFE_ERR_CONFIG_INVALID, "max_iters must be >= 1");
    if (cfg->grad_tol < 0) return fail(LIFE_ERR_CONFIG_INVALID, "grad_tol must be >= 0");
    const bool exact = cfg->exact_f64 != 0;
    if (exact && !phi->has_exact)
        return fail(LIFE_ERR_CONFIG_INVALID, "exact_f64 needs an operator built with LIFE_PHI_EXACT_F64");
    if (!exact && !phi->has_fast && !phi->has_bin)
        return fail(LIFE_ERR_CONFIG_INVALID, "operator has no fp32 layout");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t ny = (int64_t)phi->nv * phi->nt;
    const size_t es = exact ? sizeof(double) : sizeof(float);

    life_sbb *x = new life_sbb();
    struct Guard {
        life_sbb *p;
        ~Guard() { free_session(p); }
    } guard{x};
    x->cfg = *cfg;
    x->b = b_dev;
    x->w = w_dev;
    Solver &S = x->S;
    S.phi = phi;
    S.st = st;
    S.exact = exact;
    S.skip = cfg->skip_zero;
    S.nblk_f = blocks_for<float>(phi, phi->nf);
    S.comm = cfg->comm;
    if (S.comm && exact)
        return fail(LIFE_ERR_CONFIG_INVALID, "voxel-sharded runs use the fp32 path");
    LIFE_TRY(dev_alloc((void **)&S.s, sizeof(Scal)));
    LIFE_TRY(dev_alloc((void **)&S.rec, sizeof(life_trace_record) * cfg->max_iters));
    LIFE_TRY(dev_alloc((void **)&S.r, std::max<int64_t>(ny, 1) * es));
    LIFE_TRY(dev_alloc((void **)&S.mg, std::max<int64_t>(ny, 1) * es));
    LIFE_TRY(dev_alloc((void **)&S.gt, std::max(phi->nf, 1) * es));
    LIFE_TRY(dev_alloc((void **)&S.mtmg, std::max(phi->nf, 1) * es));
    LIFE_TRY(dev_alloc((void **)&S.part, phi->sms * 8 * sizeof(double)));
    LIFE_TRY(dev_alloc((void **)&S.partz, phi->sms * 8 * sizeof(unsigned long long)));
    LIFE_TRY(dev_alloc((void **)&S.counter, 16));
    LIFE_TRY(dev_alloc((void **)&S.skipped_dev, 16));
    LIFE_TRY(pinned_alloc((void **)&x->pinned, sizeof(int)));
    LIFE_CUDA(cudaMemsetAsync(S.counter, 0, 16, st));
    Scal h{};
    h.iter = 1;
    h.max_iters = cfg->max_iters;
    h.grad_tol = cfg->grad_tol;
    h.init_obj = NAN;
    h.final_obj = NAN;
    LIFE_CUDA(cudaMemcpyAsync(S.s, &h, sizeof(Scal), cudaMemcpyHostToDevice, st));

    // ---- w0 (sbbnnls.py:237-242) -------------------------------------------
    const int bf = blocks_for<float>(phi, phi->nf);
    const int by = blocks_for<float>(phi, ny);
    if (!cfg->has_w0) {
        const uint32_t skip = cfg->skip_zero ? LIFE_SKIP_ZERO : 0u;
        if (exact) {
            double *ones = (double *)S.gt, *tmp = (double *)S.r;
            k_fill<double><<<bf, 256, 0, st>>>(ones, phi->nf, 1.0);
            LIFE_CHECK_LAUNCH();
            LIFE_CUDA(cudaMemsetAsync(tmp, 0, ny * sizeof(double), st));
            LIFE_TRY(life_dsc_f64(phi, ones, tmp, skip, S.skipped_dev, st));
            k_sumsq<double, 256><<<by, 256, 0, st>>>(tmp, ny, S.part, S.counter, &S.s->m1);
            LIFE_CHECK_LAUNCH();
            k_sumsq<double, 256><<<by, 256, 0, st>>>((const double *)b_dev, ny, S.part,
                                                     S.counter, &S.s->bb);
            LIFE_CHECK_LAUNCH();
            k_w0_scale<double><<<bf, 256, 0, st>>>(S.s, (double *)w_dev, phi->nf);
        } else {
            float *ones = (float *)S.gt, *tmp = (float *)S.r;
            k_fill<float><<<bf, 256, 0, st>>>(ones, phi->nf, 1.0f);
            LIFE_CHECK_LAUNCH();
            CallHooks none{nullptr, nullptr, nullptr};
            LIFE_TRY(launch_dsc(phi, ones, tmp, nullptr, skip,
                                DscOut{nullptr, &S.s->m1, nullptr, nullptr}, none, st));
            k_sumsq<float, 256><<<by, 256, 0, st>>>((const float *)b_dev, ny, S.part,
                                                    S.counter, &S.s->bb);
            LIFE_CHECK_LAUNCH();
            LIFE_TRY(comm_reduce(S, &S.s->bb, 2, LIFE_DT_F64, LIFE_OP_SUM));  // bb, m1
            k_w0_scale<float><<<bf, 256, 0, st>>>(S.s, (float *)w_dev, phi->nf);
        }
        LIFE_CHECK_LAUNCH();
        x->dsc_calls += 1;
    } else {
        if (exact) k_project_nonneg<double><<<bf, 256, 0, st>>>((double *)w_dev, phi->nf);
        else k_project_nonneg<float><<<bf, 256, 0, st>>>((float *)w_dev, phi->nf);
        LIFE_CHECK_LAUNCH();
    }
    if (!exact && S.comm) {
        // WC scale bounds of voxel-sharded runs (k_vbound): local maxima, then
        // one MAX all-reduce at setup
        LIFE_CUDA(cudaMemcpyAsync(&S.s->vS, &phi->vsmax, sizeof(double), cudaMemcpyHostToDevice, st));
        LIFE_CUDA(cudaMemsetAsync(&S.s->vB, 0, sizeof(double), st));
        k_bnorm_max<<<blocks_for<float>(phi, phi->nv), 256, 0, st>>>((const float *)b_dev, phi->nv, phi->nt, S.s);
        LIFE_CHECK_LAUNCH();
        LIFE_TRY(comm_reduce(S, &S.s->vS, 2, LIFE_DT_F64, LIFE_OP_MAX));
    }
    if (!exact) {
        LIFE_TRY(prepare_spmv(phi));
        if (cfg->use_graph && !(S.comm && !S.comm->capturable)) {
            // capture one odd+even iteration pair; replays are parity-correct
            // because pairs always start at an odd iteration index
            // (captured on a private stream: the legacy default stream cannot
            // be captured; the graph is launched on the caller's stream)
            cudaStream_t cs = nullptr;
            LIFE_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            S.st = cs;
            LIFE_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            const uint64_t before = g_launches.load();
            int rc = iter_fast(S, (const float *)b_dev, (float *)w_dev, 0);
            if (rc == LIFE_OK) rc = iter_fast(S, (const float *)b_dev, (float *)w_dev, 1);
            cudaError_t ce = cudaStreamEndCapture(cs, &x->graph);
            cudaStreamDestroy(cs);
            S.st = st;
            x->graph_kernels = g_launches.load() - before;
            g_launches.fetch_sub(x->graph_kernels);  // counted when replayed
            if (rc != LIFE_OK) return rc;
            if (ce != cudaSuccess)
                return fail(LIFE_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
            LIFE_CUDA(cudaGraphInstantiate(&x->gexec, x->graph, 0));
        }
    }
    guard.p = nullptr;
    *out = x;
    return ok();
}

extern "C" int life_sbb_iterate(life_sbb *x, int n_iters, void *stream)
{
    if (!x) return fail(LIFE_ERR_INVALID_ARGUMENT, "null session");
    Solver &S = x->S;
    S.st = static_cast<cudaStream_t>(stream);
    while (n_iters > 0 && x->next_iter <= x->cfg.max_iters) {
        const int i = x->next_iter;
        if (S.exact) {
            LIFE_TRY(iter_exact(S, (const double *)x->b, (double *)x->w, (i % 2) == 0));
            x->next_iter += 1;
            n_iters -= 1;
        } else if (x->gexec && (i % 2) == 1 && n_iters >= 2) {
            LIFE_CUDA(cudaGraphLaunch(x->gexec, S.st));
            g_launches.fetch_add(x->graph_kernels, std::memory_order_relaxed);
            x->next_iter += 2;
            n_iters -= 2;
        } else {
            LIFE_TRY(iter_fast(S, (const float *)x->b, (float *)x->w, (i % 2) == 0));
            x->next_iter += 1;
            n_iters -= 1;
        }
    }
    return ok();
}

extern "C" int life_sbb_poll(life_sbb *x, int *done, void *stream)
{
    if (!x || !done) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    LIFE_CUDA(cudaMemcpyAsync(x->pinned, &x->S.s->done, sizeof(int), cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    *done = *x->pinned || x->next_iter > x->cfg.max_iters;
    return ok();
}

extern "C" int life_sbb_finish(life_sbb *x, life_trace_record *records,
                               life_solver_result *result, void *stream)
{
    if (!x || !result) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    Solver &S = x->S;
    life_phi *phi = S.phi;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    S.st = st;
    const int64_t ny = (int64_t)phi->nv * phi->nt;
    Scal hs{};
    LIFE_CUDA(cudaMemcpyAsync(&hs, S.s, sizeof(Scal), cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    const int iters = hs.iter - 1;  // completed (recorded) iterations
    int term = hs.term;
    double final_obj = hs.final_obj;
    int64_t dsc_calls = x->dsc_calls, wc_calls = 0;
    for (int i = 1; i <= iters; ++i) {
        dsc_calls += 2;
        wc_calls += (i % 2 == 0) ? 2 : 1;
    }
    if (term == LIFE_TERM_GRAD_TOL) {
        dsc_calls += 1;
        wc_calls += 1;
    } else if (term == LIFE_TERM_DEGENERATE) {
        const int i = iters + 1;
        dsc_calls += 2;
        wc_calls += (i % 2 == 0) ? 2 : 1;
    } else {
        // loop ended (max_iters, or the caller stopped early): final
        // objective via one more DSC (sbbnnls.py:284-287)
        term = LIFE_TERM_MAX_ITERS;
        const uint32_t skip = x->cfg.skip_zero ? LIFE_SKIP_ZERO : 0u;
        if (S.exact) {
            double *tmp = (double *)S.r;
            LIFE_CUDA(cudaMemsetAsync(tmp, 0, ny * sizeof(double), st));
            LIFE_TRY(life_dsc_f64(phi, (const double *)x->w, tmp, skip, S.skipped_dev, st));
            k_vec64<256><<<blocks_for<double>(phi, ny), 256, 0, st>>>(
                tmp, (const double *)x->b, ny, 0, S.part, S.counter, &S.s->rr, nullptr);
            LIFE_CHECK_LAUNCH();
        } else {
            CallHooks none{nullptr, nullptr, nullptr};
            LIFE_TRY(launch_dsc(phi, (const float *)x->w, (float *)S.r, (const float *)x->b,
                                LIFE_SUBTRACT_B | skip, DscOut{nullptr, &S.s->rr, nullptr, nullptr},
                                none, st));
            LIFE_TRY(comm_reduce(S, &S.s->rr, 1, LIFE_DT_F64, LIFE_OP_SUM));
        }
        double rr = 0;
        LIFE_CUDA(cudaMemcpyAsync(&rr, &S.s->rr, sizeof(double), cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        final_obj = 0.5 * rr;
        dsc_calls += 1;
    }
    if (records && iters > 0)
        LIFE_CUDA(cudaMemcpyAsync(records, S.rec, sizeof(life_trace_record) * iters,
                                  cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    result->termination = term;
    result->iterations = iters;
    result->initial_objective = hs.init_obj;
    result->final_objective = final_obj;
    result->total_dsc_calls = dsc_calls;
    result->total_wc_calls = wc_calls;
    result->loop_seconds = 0.0;
    return ok();
}

extern "C" int life_sbb_destroy(life_sbb *x)
{
    free_session(x);
    return ok();
}

extern "C" int life_solve(life_phi *phi, const void *b_dev, void *w_dev,
                          const life_solver_config *cfg, life_trace_record *records,
                          life_solver_result *result, void *stream)
{
    if (!result) return fail(LIFE_ERR_INVALID_ARGUMENT, "null result");
    life_sbb *x = nullptr;
    LIFE_TRY(life_sbb_create(phi, b_dev, w_dev, cfg, stream, &x));
    struct Guard {
        life_sbb *p;
        ~Guard() { free_session(p); }
    } guard{x};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaEvent_t e0, e1;
    LIFE_CUDA(cudaEventCreate(&e0));
    LIFE_CUDA(cudaEventCreate(&e1));
    LIFE_CUDA(cudaEventRecord(e0, st));
    const int poll = cfg->exact_f64 ? 1 : std::max(2, cfg->poll_every > 0 ? cfg->poll_every : 16);
    int done = 0;
    while (!done) {
        LIFE_TRY(life_sbb_iterate(x, poll, stream));
        LIFE_TRY(life_sbb_poll(x, &done, stream));
    }
    LIFE_CUDA(cudaEventRecord(e1, st));
    LIFE_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    LIFE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    LIFE_TRY(life_sbb_finish(x, records, result, stream));
    result->loop_seconds = ms * 1e-3;
    return ok();
}
