/*
 * life_oracle.c -- CPU restatement of the lifespmv hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_1905_06234_b200/) may link, load or call this file.  It is the
 * checker: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg are its only users.
 *
 * Parity: PINNED.  Every routine below is checked bit-for-bit against golden
 * vectors produced by the reference package itself (tests/golden/, made by
 * tests/golden/make_golden.py importing /root/reference/pkg/src/lifespmv).
 *
 * Floating point: compiled with -ffp-contract=off and without -ffast-math so
 * that every multiply and add is rounded separately, in the same order as the
 * reference's numba loops (fastmath off, no contraction: _kernels.py:7-8).
 *
 * Reference map (paths relative to /root/reference/pkg/src/lifespmv/):
 *   lo_dsc_range          <- _kernels.dsc_range        _kernels.py:14-33
 *   lo_dsc_block          <- _kernels.dsc_block        _kernels.py:36-54
 *   lo_wc_range           <- _kernels.wc_range         _kernels.py:57-68
 *   lo_dsc_chunks_owned   <- engine._dsc_owned         engine.py:277-289
 *   lo_dsc_chunks_edge    <- engine._dsc_edge_private  engine.py:292-346
 *   lo_dsc_chunks_full    <- engine._dsc_full_private  engine.py:349-369
 *   lo_wc_chunks          <- engine.wc_parallel        engine.py:372-413
 *   lo_stable_argsort_u32 <- restructure.sort_by       restructure.py:54-73
 *                            (np.argsort(kind="stable") on a u32 key)
 *   lo_detect_runs        <- restructure.detect_runs   restructure.py:76-92
 *   lo_snap               <- engine.snap_to_run_boundaries engine.py:113-136
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* y[v*nd + t] += D[a*nd + t] * s over coefficients [start, end); s is the
 * hoisted w[f]*value product (_kernels.py:24), exact zeros are skipped and
 * counted when skip_zero is set (_kernels.py:25-28). */
int64_t lo_dsc_range(const uint32_t *atoms, const uint32_t *voxels,
                     const uint32_t *fibers, const double *values,
                     const double *dict, const double *w, double *y,
                     int64_t start, int64_t end, int64_t nd, int skip_zero)
{
    int64_t skipped = 0;
    for (int64_t k = start; k < end; ++k) {
        const double s = w[fibers[k]] * values[k];
        if (s == 0.0 && skip_zero) {
            ++skipped;
            continue;
        }
        const double *row = dict + (int64_t)atoms[k] * nd;
        double *out = y + (int64_t)voxels[k] * nd;
        for (int64_t t = 0; t < nd; ++t)
            out[t] += row[t] * s;
    }
    return skipped;
}

/* Same products, accumulated into a private nd-long buffer (one voxel run
 * split across workers, _kernels.py:36-54). */
int64_t lo_dsc_block(const uint32_t *atoms, const uint32_t *fibers,
                     const double *values, const double *dict,
                     const double *w, double *buf, int64_t start, int64_t end,
                     int64_t nd, int skip_zero)
{
    int64_t skipped = 0;
    for (int64_t k = start; k < end; ++k) {
        const double s = w[fibers[k]] * values[k];
        if (s == 0.0 && skip_zero) {
            ++skipped;
            continue;
        }
        const double *row = dict + (int64_t)atoms[k] * nd;
        for (int64_t t = 0; t < nd; ++t)
            buf[t] += row[t] * s;
    }
    return skipped;
}

/* w[f] += (sum_t y[v*nd+t]*D[a*nd+t]) * value, the dot strictly sequential
 * in t (_kernels.py:61-67). */
void lo_wc_range(const uint32_t *atoms, const uint32_t *voxels,
                 const uint32_t *fibers, const double *values,
                 const double *dict, const double *y, double *w_out,
                 int64_t start, int64_t end, int64_t nd)
{
    for (int64_t k = start; k < end; ++k) {
        const double *row = dict + (int64_t)atoms[k] * nd;
        const double *sig = y + (int64_t)voxels[k] * nd;
        double acc = 0.0;
        for (int64_t t = 0; t < nd; ++t)
            acc += sig[t] * row[t];
        w_out[fibers[k]] += acc * values[k];
    }
}

/* ---- parallel regimes (engine.py:247-413), OpenMP in place of the
 *      reference's ThreadPoolExecutor.  chunks is a flat [start0,end0,
 *      start1,end1,...] array, one pair per worker.  skips_out gets one
 *      count per chunk (the caller sums, as engine.py:289 does). */

/* Ownership regime: chunk boundaries sit on voxel-run boundaries, every y
 * block has one writer (engine.py:277-289). */
void lo_dsc_chunks_owned(const uint32_t *atoms, const uint32_t *voxels,
                         const uint32_t *fibers, const double *values,
                         const double *dict, const double *w, double *y,
                         const int64_t *chunks, int nchunks, int64_t nd,
                         int skip_zero, int64_t *skips_out)
{
#pragma omp parallel for schedule(static, 1)
    for (int i = 0; i < nchunks; ++i)
        skips_out[i] = lo_dsc_range(atoms, voxels, fibers, values, dict, w, y,
                                    chunks[2 * i], chunks[2 * i + 1], nd,
                                    skip_zero);
}

static int64_t lower_bound_u32(const uint32_t *keys, int64_t n, uint32_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (keys[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

static int64_t upper_bound_u32(const uint32_t *keys, int64_t n, uint32_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (keys[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Edge privatization on a voxel-sorted tensor (engine.py:292-346): the runs
 * cut by a chunk edge go to private nd-buffers merged in ascending chunk
 * order after all workers finish. */
void lo_dsc_chunks_edge(const uint32_t *atoms, const uint32_t *voxels,
                        const uint32_t *fibers, const double *values,
                        const double *dict, const double *w, double *y,
                        const int64_t *chunks, int nchunks, int64_t nc,
                        int64_t nd, int skip_zero, int64_t *skips_out)
{
    int64_t *mid = (int64_t *)calloc((size_t)nchunks * 2, sizeof(int64_t));
    double *left = (double *)calloc((size_t)nchunks * nd + 1, sizeof(double));
    double *right = (double *)calloc((size_t)nchunks * nd + 1, sizeof(double));
    for (int i = 0; i < nchunks; ++i) {
        int64_t s = chunks[2 * i], e = chunks[2 * i + 1];
        int64_t ms = s, me = e;
        if (e > s) {
            if (s > 0 && voxels[s - 1] == voxels[s]) {
                int64_t r = upper_bound_u32(voxels, nc, voxels[s]);
                ms = r < e ? r : e;
            }
            if (e < nc && voxels[e - 1] == voxels[e]) {
                int64_t l = lower_bound_u32(voxels, nc, voxels[e - 1]);
                me = l > ms ? l : ms;
            }
        }
        mid[2 * i] = ms;
        mid[2 * i + 1] = me;
    }
#pragma omp parallel for schedule(static, 1)
    for (int i = 0; i < nchunks; ++i) {
        int64_t s = chunks[2 * i], e = chunks[2 * i + 1];
        int64_t ms = mid[2 * i], me = mid[2 * i + 1];
        int64_t total = 0;
        if (e > s) {
            if (ms > s)
                total += lo_dsc_block(atoms, fibers, values, dict, w,
                                      left + (int64_t)i * nd, s, ms, nd,
                                      skip_zero);
            if (me > ms)
                total += lo_dsc_range(atoms, voxels, fibers, values, dict, w,
                                      y, ms, me, nd, skip_zero);
            if (me < e)
                total += lo_dsc_block(atoms, fibers, values, dict, w,
                                      right + (int64_t)i * nd, me, e, nd,
                                      skip_zero);
        }
        skips_out[i] = total;
    }
    for (int i = 0; i < nchunks; ++i) {
        int64_t s = chunks[2 * i], e = chunks[2 * i + 1];
        if (e <= s) continue;
        if (mid[2 * i] > s) {
            double *out = y + (int64_t)voxels[s] * nd;
            for (int64_t t = 0; t < nd; ++t) out[t] += left[(int64_t)i * nd + t];
        }
        if (mid[2 * i + 1] < e) {
            double *out = y + (int64_t)voxels[e - 1] * nd;
            for (int64_t t = 0; t < nd; ++t) out[t] += right[(int64_t)i * nd + t];
        }
    }
    free(mid);
    free(left);
    free(right);
}

/* Full privatization (engine.py:349-369): one private signal per non-empty
 * chunk, summed into y in ascending chunk order. */
void lo_dsc_chunks_full(const uint32_t *atoms, const uint32_t *voxels,
                        const uint32_t *fibers, const double *values,
                        const double *dict, const double *w, double *y,
                        const int64_t *chunks, int nchunks, int64_t ylen,
                        int64_t nd, int skip_zero, int64_t *skips_out)
{
    int nwork = 0;
    for (int i = 0; i < nchunks; ++i)
        if (chunks[2 * i + 1] > chunks[2 * i]) ++nwork;
    for (int i = 0; i < nchunks; ++i) skips_out[i] = 0;
    if (nwork <= 1) {
        for (int i = 0; i < nchunks; ++i)
            if (chunks[2 * i + 1] > chunks[2 * i])
                skips_out[i] = lo_dsc_range(atoms, voxels, fibers, values, dict,
                                            w, y, chunks[2 * i],
                                            chunks[2 * i + 1], nd, skip_zero);
        return;
    }
    double *priv = (double *)calloc((size_t)nchunks * ylen + 1, sizeof(double));
#pragma omp parallel for schedule(static, 1)
    for (int i = 0; i < nchunks; ++i) {
        if (chunks[2 * i + 1] > chunks[2 * i])
            skips_out[i] = lo_dsc_range(atoms, voxels, fibers, values, dict, w,
                                        priv + (int64_t)i * ylen, chunks[2 * i],
                                        chunks[2 * i + 1], nd, skip_zero);
    }
    for (int i = 0; i < nchunks; ++i) {
        if (chunks[2 * i + 1] <= chunks[2 * i]) continue;
        const double *p = priv + (int64_t)i * ylen;
        for (int64_t j = 0; j < ylen; ++j) y[j] += p[j];
    }
    free(priv);
}

/* WC (engine.py:372-413).  owned != 0: fiber-aligned chunks write w_out
 * directly; otherwise private weight buffers merged in ascending order. */
void lo_wc_chunks(const uint32_t *atoms, const uint32_t *voxels,
                  const uint32_t *fibers, const double *values,
                  const double *dict, const double *y, double *w_out,
                  const int64_t *chunks, int nchunks, int64_t nf, int64_t nd,
                  int owned)
{
    int nwork = 0;
    for (int i = 0; i < nchunks; ++i)
        if (chunks[2 * i + 1] > chunks[2 * i]) ++nwork;
    if (owned || nwork <= 1) {
#pragma omp parallel for schedule(static, 1)
        for (int i = 0; i < nchunks; ++i)
            if (chunks[2 * i + 1] > chunks[2 * i])
                lo_wc_range(atoms, voxels, fibers, values, dict, y, w_out,
                            chunks[2 * i], chunks[2 * i + 1], nd);
        return;
    }
    double *priv = (double *)calloc((size_t)nchunks * nf + 1, sizeof(double));
#pragma omp parallel for schedule(static, 1)
    for (int i = 0; i < nchunks; ++i)
        if (chunks[2 * i + 1] > chunks[2 * i])
            lo_wc_range(atoms, voxels, fibers, values, dict, y,
                        priv + (int64_t)i * nf, chunks[2 * i], chunks[2 * i + 1],
                        nd);
    for (int i = 0; i < nchunks; ++i) {
        if (chunks[2 * i + 1] <= chunks[2 * i]) continue;
        const double *p = priv + (int64_t)i * nf;
        for (int64_t j = 0; j < nf; ++j) w_out[j] += p[j];
    }
    free(priv);
}

/* Stable argsort of a u32 key by counting sort: equal keys keep their
 * original relative order, so the permutation equals
 * np.argsort(keys, kind="stable") (restructure.py:64).  perm[i] is the
 * original position of the i-th element in sorted order. */
int lo_stable_argsort_u32(const uint32_t *keys, int64_t n, int64_t *perm)
{
    if (n == 0) return 0;
    uint32_t kmax = 0;
    for (int64_t i = 0; i < n; ++i)
        if (keys[i] > kmax) kmax = keys[i];
    int64_t *count = (int64_t *)calloc((size_t)kmax + 2, sizeof(int64_t));
    if (!count) return -1;
    for (int64_t i = 0; i < n; ++i) ++count[(int64_t)keys[i] + 1];
    for (int64_t k = 1; k <= (int64_t)kmax + 1; ++k) count[k] += count[k - 1];
    for (int64_t i = 0; i < n; ++i) perm[count[keys[i]]++] = i;
    free(count);
    return 0;
}

/* Maximal constant runs of a sorted key array (restructure.py:76-92):
 * boundaries[0..n_runs] (boundaries[n_runs] == n), key of each run. */
int64_t lo_detect_runs(const uint32_t *keys, int64_t n, int64_t *boundaries,
                       uint32_t *run_keys)
{
    int64_t r = 0;
    boundaries[0] = 0;
    if (n == 0) return 0;
    for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || keys[i] != keys[i - 1]) {
            boundaries[r] = i;
            run_keys[r] = keys[i];
            ++r;
        }
    }
    boundaries[r] = n;
    return r;
}

/* snap_to_run_boundaries (engine.py:113-136): interior boundaries inside a
 * run move to the run end that adds fewer coefficients to the gaining
 * worker, ties to the later worker (run_start); then monotone repair. */
void lo_snap(const uint32_t *keys, int64_t n, int64_t *bounds, int nb)
{
    for (int i = 1; i < nb - 1; ++i) {
        int64_t b = bounds[i];
        if (b > 0 && b < n && keys[b - 1] == keys[b]) {
            int64_t rs = lower_bound_u32(keys, n, keys[b]);
            int64_t re = upper_bound_u32(keys, n, keys[b]);
            bounds[i] = (b - rs <= re - b) ? rs : re;
        }
    }
    for (int i = 1; i < nb; ++i)
        if (bounds[i] < bounds[i - 1]) bounds[i] = bounds[i - 1];
}

int lo_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void lo_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
