// life_common.cuh -- internal declarations shared by the liblife_b200 sources.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "life_b200.h"

namespace life {

// ---- errors ----------------------------------------------------------------
int fail(int status, const std::string &msg);  // records msg, returns status
int ok();                                      // clears msg, returns LIFE_OK
extern std::atomic<uint64_t> g_launches;

#define LIFE_CUDA(call)                                                        \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess)                                                 \
            return ::life::fail(e_ == cudaErrorMemoryAllocation                \
                                    ? LIFE_ERR_OUT_OF_MEMORY                   \
                                    : LIFE_ERR_CUDA,                           \
                                std::string(#call) + ": " +                    \
                                    cudaGetErrorString(e_));                   \
    } while (0)

#define LIFE_CHECK_LAUNCH()                                                    \
    do {                                                                       \
        ::life::g_launches.fetch_add(1, std::memory_order_relaxed);           \
        cudaError_t e_ = cudaGetLastError();                                   \
        if (e_ != cudaSuccess)                                                 \
            return ::life::fail(LIFE_ERR_CUDA, std::string("launch: ") +       \
                                                   cudaGetErrorString(e_));    \
    } while (0)

#define LIFE_TRY(expr)                                                         \
    do {                                                                       \
        int s_ = (expr);                                                       \
        if (s_ != LIFE_OK) return s_;                                          \
    } while (0)

constexpr int kMaxNT = 10;          // n_dirs <= 320 (SPEC: 10..300 directions)
constexpr int kSpmvThreads = 512;   // 16 warps per CTA, one CTA per SM

// ---- device helpers --------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename T>
__device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }

// Per-call reduction outputs, fixed-order (deterministic) completion.
struct ReduceSlots {
    double *part_d;               // [nwarps] sum of squares partials
    unsigned long long *part_u;   // [nwarps] counts
    float *part_f;                // [nwarps] abs-max partials
    unsigned *counter;            // blocks finished (reset by last block)
};

// Timing/termination hooks used by the on-device solver (all optional).
struct CallHooks {
    const int *done;                     // kernel no-ops when *done != 0
    unsigned long long *t_begin;         // globaltimer at entry (block 0)
    unsigned long long *t_accum;         // += (end - begin) ns by last block
};

}  // namespace life

// ---- the operator handle ---------------------------------------------------
struct life_phi {
    life_dims dims{};
    int na = 0, nv = 0, nf = 0, nt = 0;
    int64_t nc = 0;
    int sms = 0;
    int device = 0;

    // fp32 fast layout: coefficients sorted by (atom group, voxel), stable.
    bool has_fast = false;
    int G = 1;            // atom groups (D slices staged in shared memory)
    int ag = 0;           // atoms per group
    int slice_floats = 0; // floats per staged slice (16-byte padded)
    uint32_t *atom = nullptr;   // atom index local to its group
    uint32_t *fiber = nullptr;
    float *val = nullptr;
    uint32_t *gptr = nullptr;   // [G*nv + 1] segment starts
    int *wpart = nullptr;       // [W + 1] voxel range per persistent warp
    float *Dg = nullptr;        // [G*slice_floats] fp32 dictionary slices
    int nblocks = 0, W = 0;
    size_t smem = 0;

    // binned two-phase layout (life_bin.cu, the default fp32 products):
    // "tile side" = 128-row voxel tiles x atom chunks on tcgen05, "bin
    // side" = fascicle bins held in shared memory; the two meet in a
    // tile-major scratch vector (s = w[f]*value for DSC, z = (Y D^T)[cell]
    // for WC) through contiguous segments (tile, chunk, bin).
    bool has_bin = false;
    int b_ka = 0, b_n = 0, b_nch = 0, b_ntiles = 0, b_nbins = 0, b_sb = 0;
    int64_t b_nvf = 0, b_nsteps = 0, b_nseg = 0, b_npad = 0;
    uint16_t *b_cellr = nullptr;   // tile-major [npad]: rank << cellbits | row*KA + atom%KA
    uint16_t *b_vid = nullptr;     // bin-major [nc]: virtual fascicle slot within its bin
    float *b_val = nullptr;        // bin-major [nc]
    float *b_scr = nullptr;        // tile-major scratch [npad]
    uint32_t *b_step = nullptr;    // [nsteps + 1] tile-major start of each (tile, chunk)
    uint32_t *b_segsrc = nullptr;  // [nseg + 1] bin-major start of each (bin, tile, chunk), 4-entry units
    uint32_t *b_segdst = nullptr;  // [nseg] its tile-major start, 4-entry units
    uint32_t *b_binptr = nullptr;  // [nbins + 1] first segment of each bin
    uint32_t *b_chunks = nullptr;  // bin-side chunk descriptors (uint4: first unit, units | piece start, first segment, segments | bin)
    uint16_t *b_cgrp = nullptr;      // [chunks][32] first segment of each 32-unit group of a chunk
    uint32_t *b_ctachunk = nullptr;  // [side grid + 1] first chunk of each bin-side CTA
    uint32_t *b_vf2f = nullptr;    // [nvf] fascicle of each virtual slot
    uint32_t *b_f2vf = nullptr;    // [nf + 1] first virtual slot of each fascicle
    int *b_rowvox = nullptr;       // [ntiles*128] voxel of each tile row, -1 = empty
    int *b_rowpart = nullptr;      // [ntiles*128] partial-row index, -1 = the voxel's only row
    uint16_t *b_Ddsc = nullptr;    // per chunk: f16 [hi|lo][N][64 atoms] swizzled D^T * 256 (DSC B operand)
    uint16_t *b_Dwc = nullptr;     // per chunk: f16 [hi|lo][N/64][64 atoms][64] swizzled D * 256 (WC B operand)
    float *b_ypart = nullptr;      // [nprow * N] rows of voxels split over several rows
    uint32_t *b_fixpc = nullptr;   // [npc] uint4 fixup pieces: voxel, first row, end row, piece-sum slot (~0: final)
    uint32_t *b_fixbig = nullptr;  // [nbig] voxels folded from several pieces
    uint32_t *b_fixbpp = nullptr;  // [nbig + 1] their piece-sum slots
    float *b_fixsum = nullptr;     // [piece-sum slots][N]
    int b_nfix = 0, b_nprow = 0, b_npc = 0, b_nbig = 0;
    unsigned long long *b_wfix = nullptr;  // [nf + ceil(nf/8)] int64 fixed-point fascicle sums, then the flags (zero between calls)
    unsigned char *b_nanf = nullptr;       // [nf] non-finite term seen (bytes in the tail of b_wfix)
    unsigned long long *b_skip = nullptr;  // [side grid] skip-count partials of the bin side
    float *b_smax = nullptr;               // [side grid] max |s| partials (DSC fixed-point scale)
    unsigned *b_nonfin = nullptr;          // non-finite s seen by the DSC bin side (this call)
    int b_tile_grid = 0, b_side_grid = 0, b_dsc_cap = 0;
    size_t b_dsc_smem = 0, b_wc_smem = 0, b_side_smem = 0, b_wcs_smem = 0;

    // fixed-point WC accumulator and its scale inputs
    unsigned long long *wfix = nullptr;  // [nf] two's-complement int64
    double vmax = 0.0;                   // max |value|
    double dmax = 0.0;                   // max ||D_a||_2
    double vsmax = 0.0;                  // max_v sum_{c in v} ||D_a(c)||_2 |value_c| (||(M w)_v|| <= vsmax max|w|)
    int64_t fmax_nnz = 0;                // longest fascicle segment

    // fp64 bit-exact layouts (stable voxel sort, stable fiber sort)
    bool has_exact = false;
    uint32_t *xv_atom = nullptr, *xv_voxel = nullptr, *xv_fiber = nullptr;
    double *xv_val = nullptr;
    uint32_t *xv_ptr = nullptr;     // [nv + 1]
    int *xv_wpart = nullptr;        // [xW + 1] voxel ranges
    uint32_t *xf_atom = nullptr, *xf_voxel = nullptr, *xf_fiber = nullptr;
    double *xf_val = nullptr;
    uint32_t *xf_ptr = nullptr;     // [nf + 1]
    int *xf_wpart = nullptr;        // [xW + 1] fiber ranges
    double *D64 = nullptr;
    int xW = 0, xblocks = 0;

    // scratch
    life::ReduceSlots red{};
    double *part_d2 = nullptr;       // second slot set for finalize kernels
    unsigned long long *part_u2 = nullptr;
    unsigned *counter2 = nullptr;
    float *ybound = nullptr;         // device scalar for standalone WC
    int red_cap = 0;                 // capacity of partial arrays

    // statistics
    int64_t n_voxel_runs = 0, n_fiber_runs = 0, max_voxel_run = 0,
            max_fiber_run = 0;
    double sort_ms = 0.0;
    int64_t device_bytes = 0;
    std::vector<void *> allocs;
};

namespace life {
// pageable host -> device through pinned staging (life_phi.cu)
int h2d_staged(void *dst, const void *src, size_t bytes, cudaStream_t st);
int h2d_staged_cvt(void *dst, const void *src, size_t bytes, int mode, cudaStream_t st);  // 1: f64->f32, 2: u32->u16
int h2d_staged_pack_av(uint32_t *dst, const uint32_t *atoms, const uint32_t *voxels, int64_t n, int abits, int vbits,
                       cudaStream_t st);  // (voxel << abits) | atom, saturated fields
// LIFE_B200_SETUP_TRACE=1: synchronize and print the time since the last mark
// (operator construction phases, stderr)
void setup_mark(cudaStream_t st, const char *what);

// Device block cache (life_phi.cu).  Operators and solver sessions allocate
// GBs at C2; cudaMalloc / cudaFree of them costs 0.1-0.3 s per operator on
// some hosts (page mapping, implicit device syncs), so freed blocks are kept
// mapped per (device, size class) and handed to the next operator.
// dev_free's caller guarantees the device no longer uses the block.
int dev_alloc(void **p, size_t bytes);
void dev_free(void *p);
int pinned_alloc(void **p, size_t bytes);  // small page-locked host words (same idea)
void pinned_free(void *p);

template <typename T>
int dalloc(life_phi *phi, T **p, size_t n)
{
    *p = nullptr;
    if (n == 0) n = 1;
    const int rc = dev_alloc(reinterpret_cast<void **>(p), n * sizeof(T));
    if (rc != LIFE_OK) return rc;
    phi->allocs.push_back(*p);
    phi->device_bytes += static_cast<int64_t>(n * sizeof(T));
    return LIFE_OK;
}

// Fixed-point exponent for the WC accumulator: a coefficient term is at most
// vmax * dmax * ||y_v||_2; a fascicle sums at most fmax_nnz of them, and the
// total must stay below 2^62.  ||y_v||_2 is bounded either by sqrt(nt)*max|y|
// (standalone WC) or by sqrt(sum y^2) (solver: one scalar that multi-GPU
// runs all-reduce, so every rank derives the same exponent).
struct FixParams {
    unsigned long long *wfix;  // [nf] two's-complement int64 accumulators
    const float *ymax;         // device max|y|, or null
    const double *ysumsq;      // device sum of y^2, or null (takes precedence)
    double vmax, dmax, fmax_nnz;
    // bin layout, voxel-sharded runs: device bound on max_v ||y_v||_2 that
    // every rank computes identically before any collective (takes
    // precedence; life_solver.cu k_vbound)
    const float *yvbound = nullptr;
};

// DSC scalars (this rank's partial sums) carried in the tail of the WC
// all-reduce of a voxel-sharded run; replaced by the global sums
struct WcScalars {
    double *v[3];
    int n;
};
constexpr int kTailRanks = 64;  // scalar slots per value in the WC buffer tail (ranks)

__host__ __device__ inline int fix_exponent_from(double vmax, double dmax, double ynorm,
                                                 double fmax_nnz)
{
    const double bound = vmax * dmax * ynorm * fmax_nnz;
    if (!(bound > 0.0)) return 0;
    int e;
    frexp(bound, &e);  // bound < 2^e
    int ex = 62 - e;
    if (ex > 1000) ex = 1000;
    if (ex < -1000) ex = -1000;
    return ex;
}

__device__ inline int fix_exponent(const FixParams &fx, int nt)
{
    const double yn = fx.ysumsq ? sqrt(*fx.ysumsq) : sqrt((double)nt) * (double)*fx.ymax;
    return fix_exponent_from(fx.vmax, fx.dmax, yn, fx.fmax_nnz);
}

// Raise (never lower) a kernel's dynamic shared-memory limit.  The attribute
// caps every later launch of that function, so lowering it for a small
// operator would break a larger operator still in use.
int ensure_smem_ptr(const void *func, size_t bytes);
template <typename F>
int ensure_smem(F *func, size_t bytes)
{
    return ensure_smem_ptr(reinterpret_cast<const void *>(func), bytes);
}

// Internal launchers exposed across translation units.
struct DscOut {
    unsigned long long *skipped;
    double *sumsq;
    float *absmax;
    double *skipped_d;  // the skip count again as a double (packed solver scalars)
};
int launch_absmax(life_phi *phi, const float *x, int64_t n, float *out,
                  cudaStream_t st);
int launch_dsc(life_phi *phi, const float *w, float *y, const float *b,
               uint32_t flags, const DscOut &o, const CallHooks &h, cudaStream_t st);
int launch_wc(life_phi *phi, const float *y, float *w, const float *w_ref,
              const float *ymax_dev, const double *ysumsq_dev, uint32_t flags, double *sumsq,
              const CallHooks &h, const life_comm *comm, cudaStream_t st,
              const float *yvbound_dev = nullptr, const WcScalars *sc = nullptr);
int prepare_spmv(life_phi *phi);
// binned two-phase products (life_bin.cu)
int build_bin(life_phi *phi, const uint32_t *a, const uint32_t *v, const uint32_t *f,
              const double *val, const std::vector<double> &hdict, const std::function<int()> &ready_fv,
              cudaStream_t st);  // ready_fv(): fibers/values resident (called before they are read)
int launch_dsc_bin(life_phi *phi, const float *w, float *y, const float *b, uint32_t flags,
                   const DscOut &o, const CallHooks &h, cudaStream_t st);
int bin_tile_warps(const life_phi *phi);
int launch_wc_bin(life_phi *phi, const float *y, float *w, const float *w_ref, const FixParams &fx,
                  uint32_t flags, double *sumsq, const CallHooks &h, const life_comm *comm,
                  cudaStream_t st, const WcScalars *sc);
}  // namespace life
