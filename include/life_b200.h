/*
 * life_b200.h -- C ABI of the B200-native LiFE hot path (liblife_b200.so).
 *
 * The operator is M = Phi x_1 D of arXiv:1905.06234 (LiFE): Phi is a COO
 * sparse 3-tensor of (atom, voxel, fascicle, value) coefficients, D the dense
 * dictionary (atom-major, n_dirs values per atom).  Two products:
 *   DSC  y = M w     (diffusion signal computation)
 *   WC   w = M^T y   (weight computation)
 * and the SBBNNLS fit loop that calls both every iteration.
 *
 * The reference (lifespmv, /root/reference/pkg) has no FFI: its boundary is
 * the Python API plus the numba kernel ABI.  Each entry point below names the
 * reference interface it replaces (paths relative to
 * /root/reference/pkg/src/lifespmv/).
 *
 * Conventions
 *   - Plain C: pointers, sizes, status codes.  No torch or C++ types.
 *   - Every function returns a life_status; nothing throws.  The last error
 *     message of the calling thread is available from life_last_error().
 *   - "dev" pointers are CUDA device pointers; "stream" is a cudaStream_t
 *     passed as void* (NULL = legacy default stream).  All work is
 *     stream-ordered; nothing synchronizes the device unless documented.
 *   - Outputs are caller-allocated.  A life_phi handle owns its device copies
 *     of Phi and D; caller buffers are borrowed for the duration of a call.
 *   - A handle's scratch is shared by its calls: use one stream at a time
 *     per handle (the reference is single-caller per call as well).
 */
#ifndef LIFE_B200_H
#define LIFE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LIFE_API __attribute__((visibility("default")))
#else
#define LIFE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define LIFE_B200_ABI_VERSION 1

/* Status codes mirror the reference's LifeError family (errors.py:8-93). */
typedef enum life_status {
    LIFE_OK = 0,
    LIFE_ERR_CONFIG_INVALID = 1,          /* errors.ConfigInvalid          errors.py:76 */
    LIFE_ERR_DIMENSION_MISMATCH = 2,      /* errors.DimensionMismatch      errors.py:68 */
    LIFE_ERR_PLAN_TENSOR_MISMATCH = 3,    /* errors.PlanTensorMismatch     errors.py:64 */
    LIFE_ERR_STRATEGY_REQUIRES_SORTED = 4,/* errors.StrategyRequiresSorted errors.py:60 */
    LIFE_ERR_DEGENERATE_STEP = 5,         /* errors.DegenerateStep         errors.py:72 */
    LIFE_ERR_INDEX_OUT_OF_RANGE = 6,      /* errors.IndexOutOfRange        errors.py:12 */
    LIFE_ERR_ARITHMETIC_OVERFLOW = 7,     /* errors.ArithmeticOverflow     errors.py:48 */
    LIFE_ERR_NOT_SORTED = 8,              /* errors.NotSorted              errors.py:56 */
    LIFE_ERR_NON_FINITE = 9,              /* errors.NonFiniteValue         errors.py:39 */
    LIFE_ERR_CUDA = 20,                   /* CUDA runtime failure */
    LIFE_ERR_OUT_OF_MEMORY = 21,
    LIFE_ERR_INVALID_ARGUMENT = 22,       /* null handle / pointer */
    LIFE_ERR_NCCL = 23
} life_status;

/* Problem dimensions (tensor.Dims, tensor.py:44-73). */
typedef struct life_dims {
    int64_t n_atoms;
    int64_t n_voxels;
    int64_t n_fibers;
    int64_t n_dirs;
    int64_t n_coeffs;
} life_dims;

typedef struct life_phi life_phi; /* opaque device-resident operator */

/* ---- library --------------------------------------------------------- */
LIFE_API int life_abi_version(void);
LIFE_API const char *life_status_string(int status);
LIFE_API const char *life_last_error(void);
/* Number of kernel launches this process has issued through the library
 * (monotone counter; used by bench.py's gpu_launches claim). */
LIFE_API uint64_t life_launch_count(void);

/* ---- operator construction -------------------------------------------- */

/* flags for life_phi_create */
#define LIFE_PHI_HOST_INPUT   0x1u  /* input arrays are host pointers       */
#define LIFE_PHI_EXACT_F64    0x2u  /* also build the fp64 bit-exact layout */
#define LIFE_PHI_NO_FAST_F32  0x4u  /* skip the fp32 fast layout           */
#define LIFE_PHI_FORCE_SPARSE 0x8u  /* fp32: voxel-segment kernels only    */
#define LIFE_PHI_FORCE_DENSE  0x10u /* fp32: the tile layout (binned products) even for sparse operators */
#define LIFE_PHI_NO_TENSOR    0x20u /* fp32: no tcgen05 products (voxel-segment kernels) */
#define LIFE_PHI_TENSOR       0x40u /* retired in round 2 (the single-pass tcgen05 tile family); ignored */
#define LIFE_PHI_NO_BIN       0x80u /* fp32: not the binned products (voxel-segment kernels) */
#define LIFE_PHI_VALUES_F32   0x100u /* with HOST_INPUT: values may cross PCIe as f32 (fp32-only operator; ignored with EXACT_F64) */

/* Build the device operator from COO arrays (PhiTensor + Dictionary,
 * tensor.py:76-170).  atoms/voxels/fibers: u32[n_coeffs]; values:
 * f64[n_coeffs]; dict: f64[n_atoms*n_dirs] atom-major.  Indices are
 * range-checked on the device (LIFE_ERR_INDEX_OUT_OF_RANGE, the first bad
 * position in *bad_position when non-NULL).  The default fp32 layout is the
 * binned two-phase layout (tile-major and fascicle-bin-major orders, DESIGN.md
 * section 3) built from stable device sorts; the sparse layout refines
 * restructure.sort_by(tensor, "voxel") (restructure.py:54) by atom group; the
 * exact layout is the plain stable voxel sort plus the stable fiber sort.
 * With LIFE_PHI_HOST_INPUT the arrays are staged through pinned buffers:
 * atom and voxel packed into one u32 when both fit (saturated fields, so the
 * range check still sees out-of-range indices).  Synchronizes the stream. */
LIFE_API int life_phi_create(const life_dims *dims, const uint32_t *atoms,
                    const uint32_t *voxels, const uint32_t *fibers,
                    const double *values, const double *dict, uint32_t flags,
                    void *stream, life_phi **out, int64_t *bad_position);
LIFE_API int life_phi_destroy(life_phi *phi);

/* Device blocks of destroyed operators and solver sessions stay mapped in a
 * per-process cache (up to LIFE_B200_BLOCK_CACHE_MB, default 24 GiB) and are
 * reused by the next operator; cudaMalloc/cudaFree of the GBs an operator
 * holds cost 0.1-0.3 s on some hosts.  The reference has no counterpart (it
 * allocates numpy arrays per call, engine.py:218-244).  Release hands every
 * cached block back to the driver; bytes reports the cached total. */
LIFE_API int life_release_cached_memory(void);
LIFE_API int life_cached_memory_bytes(int64_t *bytes);

/* Copy bytes from pageable host memory to the device through pinned staging
 * buffers (host memcpy overlapped with the DMA); stream-ordered, returns when
 * the source may be reused.  Used for the LIFE_PHI_HOST_INPUT arrays and by
 * the Python layer for b / w0 (sbbnnls.solve's inputs, sbbnnls.py:223). */
LIFE_API int life_copy_h2d(void *dst_dev, const void *src_host, int64_t bytes, void *stream);
/* The same for an f64 host vector into an f32 device vector (rounded to
 * nearest on the host while staging: half the bytes cross PCIe); the fp32
 * solver's b (sbbnnls.py:223 problem.y). */
LIFE_API int life_copy_h2d_f32(float *dst_dev, const double *src_host, int64_t count, void *stream);

typedef struct life_phi_info {
    life_dims dims;
    int32_t atom_groups;        /* sparse kernels: passes over Phi (D slices); -2 = binned two-phase (tcgen05) */
    int32_t atoms_per_group;
    int32_t n_warps;            /* persistent warps of the SpMV kernels   */
    int32_t has_exact;          /* fp64 bit-exact layout present          */
    int64_t n_voxel_runs;       /* occupied voxels (RunTable.n_runs)      */
    int64_t n_fiber_runs;       /* occupied fascicles                     */
    int64_t max_fiber_run;      /* longest fascicle segment               */
    int64_t max_voxel_run;      /* longest voxel segment                  */
    int64_t device_bytes;       /* bytes owned by the handle              */
    double sort_ms;             /* restructuring time at create           */
    int32_t tensor_ops;         /* products on tcgen05: bit 0 DSC, bit 1 WC */
    int32_t reserved;
} life_phi_info;
LIFE_API int life_phi_get_info(const life_phi *phi, life_phi_info *info);

/* ---- restructuring (restructure.py:54-92) ------------------------------ */

/* Stable argsort of a u32 key (np.argsort(kind="stable"), restructure.py:64)
 * on the device: perm_dev[i] = original position of the i-th element in
 * sorted order.  keys_dev/perm_dev are device pointers; n may be 0. */
LIFE_API int life_stable_argsort_u32(const uint32_t *keys_dev, int64_t n,
                            int64_t *perm_dev, void *stream);

/* Maximal constant runs of a sorted key array (detect_runs,
 * restructure.py:76-92): boundaries_dev[0..n_runs] (int64, capacity n+1),
 * run_keys_dev[0..n_runs-1].  *n_runs_out is written on the host (the call
 * synchronizes the stream).  Returns LIFE_ERR_NOT_SORTED if keys decrease. */
LIFE_API int life_detect_runs_u32(const uint32_t *keys_dev, int64_t n,
                         int64_t *boundaries_dev, uint32_t *run_keys_dev,
                         int64_t *n_runs_out, void *stream);

/* Apply a permutation to the four coefficient arrays (the joint reorder of
 * sort_by, restructure.py:66-72), device to device. */
LIFE_API int life_gather_coo(const int64_t *perm_dev, int64_t n, const uint32_t *atoms,
                    const uint32_t *voxels, const uint32_t *fibers,
                    const double *values, uint32_t *atoms_out,
                    uint32_t *voxels_out, uint32_t *fibers_out,
                    double *values_out, void *stream);

/* ---- SpMV (engine.py:218-413 over _kernels.py:14-68) -------------------- */

/* flags for life_dsc / life_wc */
#define LIFE_ACCUMULATE   0x01u /* out += M x (reference accumulator contract) */
#define LIFE_SKIP_ZERO    0x02u /* skip coefficients with w[f]*value == 0      */
#define LIFE_SUBTRACT_B   0x04u /* DSC: out = M w - b  (residual epilogue)     */
#define LIFE_PROJECT_GRAD 0x08u /* WC:  out = project_gradient(M^T y, w_ref)   */

/* Per-call outputs written on the device (all optional, may be NULL). */
typedef struct life_spmv_out {
    unsigned long long *skipped; /* DSC: #coefficients with w[f]*value==0 (KernelStats) */
    double *sumsq;               /* sum of squares of the written output vector        */
    float *absmax;               /* max |output element| (WC fixed-point bound input)  */
} life_spmv_out;

/* The fp32 products stream vectors in 16-byte units: w, y, b and w_ref must
 * be 16-byte aligned (every cudaMalloc / torch allocation is); a misaligned
 * pointer returns LIFE_ERR_INVALID_ARGUMENT before any launch. */

/* y = M w (fp32, fast layout).  w: f32[Nf], y: f32[Nv*Nd], b: f32[Nv*Nd]
 * (LIFE_SUBTRACT_B only).  Replaces dsc_sequential / dsc_parallel
 * (engine.py:218,247) and the dsc_range kernel ABI (_kernels.py:14). */
LIFE_API int life_dsc_f32(life_phi *phi, const float *w, float *y, const float *b,
                 uint32_t flags, const life_spmv_out *out, void *stream);

/* w = M^T y (fp32 fast path).  y: f32[Nv*Nd]; w: f32[Nf]; w_ref: f32[Nf]
 * (LIFE_PROJECT_GRAD only).  y_absmax_dev: optional device scalar holding
 * max|y| (from a producing life_dsc_f32 call); NULL = computed here.
 * Accumulation over coefficients is exact fixed-point (order independent,
 * bitwise reproducible).  Replaces wc_sequential / wc_parallel
 * (engine.py:236,372) and the wc_range ABI (_kernels.py:57). */
LIFE_API int life_wc_f32(life_phi *phi, const float *y, float *w, const float *w_ref,
                const float *y_absmax_dev, uint32_t flags,
                const life_spmv_out *out, void *stream);

/* Bit-exact fp64 products (requires LIFE_PHI_EXACT_F64): same rounding and
 * per-output accumulation order as the reference's sequential kernels on the
 * tensor as given (_kernels.py:14-33, 57-68), so results equal
 * dsc_sequential / wc_sequential bit for bit.  Always accumulate semantics
 * (out += ...); clear the output first for a fresh product. */
LIFE_API int life_dsc_f64(life_phi *phi, const double *w, double *y, uint32_t flags,
                 unsigned long long *skipped_dev, void *stream);
LIFE_API int life_wc_f64(life_phi *phi, const double *y, double *w, void *stream);

/* ---- multi-GPU ------------------------------------------
 * Phi is sharded by contiguous voxel ranges, one process per GPU.  DSC is
 * local.  Each WC ends with ONE all-reduce: the length-Nf fixed-point
 * fascicle sums (int64, so every rank gets bit-identical totals), the
 * non-finite flags, and the DSC scalars of the same iteration (sum of
 * squares, skip count; rank slots, added in rank order).  The WC scale comes
 * from a bound every rank computes alike (max|w| times a per-voxel constant),
 * so no collective precedes the WC.  Odd iterations add one scalar all-reduce
 * (||M g||^2 for the step size).  The communicator is either the library's
 * own NCCL one (life_comm_init_nccl: ncclAllReduce on the solver stream,
 * capturable, so iterations run as CUDA graphs) or a caller-supplied
 * all-reduce that enqueues on `stream` (capturable = 0: no graphs). */
typedef enum life_dtype { LIFE_DT_F64 = 0, LIFE_DT_F32 = 1, LIFE_DT_I64 = 2 } life_dtype;
typedef enum life_redop { LIFE_OP_SUM = 0, LIFE_OP_MAX = 1 } life_redop;
typedef int (*life_allreduce_fn)(void *buf, int64_t count, int dtype, int op, void *stream,
                                 void *ctx);
typedef struct life_comm {
    life_allreduce_fn allreduce;
    void *ctx;
    int32_t rank;
    int32_t nranks;
    int32_t capturable;     /* allreduce may be captured in a CUDA graph   */
    int32_t reserved;
} life_comm;

/* NCCL communicator (libnccl.so.2 resolved at run time; the process's
 * already-loaded copy when there is one).  unique_id: 128 bytes
 * (ncclUniqueId) made by rank 0 with life_nccl_unique_id and shared by the
 * caller (e.g. torch.distributed broadcast).  life_comm_init_nccl fills
 * *comm (caller-owned struct); life_comm_destroy_nccl releases it. */
LIFE_API int life_nccl_unique_id(void *unique_id_out);
LIFE_API int life_comm_init_nccl(const void *unique_id, int rank, int nranks, life_comm *comm);
LIFE_API int life_comm_destroy_nccl(life_comm *comm);

/* Global bounds for the WC fixed-point scale (every rank must use the same
 * exponent): max |value| and the longest fascicle over the WHOLE problem,
 * and max ||D_a||_2.  Defaults are the handle's own (single-GPU) values. */
LIFE_API int life_phi_set_fix_bounds(life_phi *phi, double vmax, double dmax,
                                     int64_t fmax_nnz);
LIFE_API int life_phi_get_fix_bounds(const life_phi *phi, double *vmax, double *dmax,
                                     int64_t *fmax_nnz);

/* ---- SBBNNLS (sbbnnls.py:34-291) --------------------------------------- */

typedef struct life_solver_config {  /* sbbnnls.SolverConfig, sbbnnls.py:34-62 */
    int32_t max_iters;
    int32_t skip_zero;
    int32_t exact_f64;      /* 1: fp64 bit-exact kernels, 0: fp32 fast path */
    int32_t has_w0;         /* 0: w0 = 1*||b||/||M 1|| (sbbnnls.py:237-240)  */
    double grad_tol;
    int32_t poll_every;     /* iterations between host termination polls    */
    int32_t use_graph;      /* capture iterations in a CUDA graph           */
    const life_comm *comm;  /* NULL: single GPU; else voxel-sharded run     */
} life_solver_config;

typedef struct life_trace_record {   /* sbbnnls.TraceRecord, sbbnnls.py:65-85 */
    int32_t iteration;
    int32_t zeros;
    int64_t dsc_skipped;
    double objective;
    double alpha;
    double grad_norm;
    double w_min;
    double dsc_seconds;
    double wc_seconds;
    int32_t dsc_calls;
    int32_t wc_calls;
} life_trace_record;

#define LIFE_TERM_NONE 0
#define LIFE_TERM_MAX_ITERS 1
#define LIFE_TERM_GRAD_TOL 2
#define LIFE_TERM_DEGENERATE 3

typedef struct life_solver_result {  /* sbbnnls.SolverTrace, sbbnnls.py:88-99 */
    int32_t termination;
    int32_t iterations;
    double initial_objective;
    double final_objective;
    int64_t total_dsc_calls;
    int64_t total_wc_calls;
    double loop_seconds;    /* device time of the iteration loop (events)   */
} life_solver_result;

/* Run Alg. 1 (sbbnnls.solve, sbbnnls.py:223-291) on the device.
 * b_dev: signal (f64[Nv*Nd] when exact_f64 else f32); w_dev: in: w0 (if
 * has_w0) out: final weights, same dtype.  records: host array of capacity
 * max_iters (may be NULL).  Synchronizes the stream at the end. */
LIFE_API int life_solve(life_phi *phi, const void *b_dev, void *w_dev,
               const life_solver_config *cfg, life_trace_record *records,
               life_solver_result *result, void *stream);

/* Stepwise solver session (the same loop as life_solve, split so a caller
 * can time exactly N iterations or interleave its own work).
 *   create : buffers, w0 (one DSC when has_w0 == 0), CUDA-graph capture
 *   iterate: enqueue up to n more iterations (no host sync; kernels become
 *            no-ops once the device sets its termination flag)
 *   poll   : synchronize and report termination (or max_iters reached)
 *   finish : final objective DSC if needed, trace records, call counts */
typedef struct life_sbb life_sbb;
LIFE_API int life_sbb_create(life_phi *phi, const void *b_dev, void *w_dev,
                             const life_solver_config *cfg, void *stream,
                             life_sbb **out);
LIFE_API int life_sbb_iterate(life_sbb *sbb, int n_iters, void *stream);
LIFE_API int life_sbb_poll(life_sbb *sbb, int *done, void *stream);
LIFE_API int life_sbb_finish(life_sbb *sbb, life_trace_record *records,
                             life_solver_result *result, void *stream);
LIFE_API int life_sbb_destroy(life_sbb *sbb);

#ifdef __cplusplus
}
#endif
#endif /* LIFE_B200_H */
