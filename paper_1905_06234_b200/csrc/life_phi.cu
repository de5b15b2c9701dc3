// life_phi.cu -- operator construction (restructuring), argsort, run
// detection, and the library's error plumbing.
//
// Restructuring follows restructure.sort_by / detect_runs
// (/root/reference/pkg/src/lifespmv/restructure.py:54-92): a STABLE sort of
// the coefficient list by a key, realised on the device with a LSD radix
// sort (stable by construction), so the permutation is bit-identical to
// np.argsort(kind="stable").
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <vector>
#include <unordered_map>

#include "life_common.cuh"

namespace life {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_last_error;

int fail(int status, const std::string &msg)
{
    t_last_error = msg;
    return status;
}

int ok()
{
    t_last_error.clear();
    return LIFE_OK;
}

int ensure_smem_ptr(const void *func, size_t bytes)
{
    static std::mutex mu;
    static std::unordered_map<const void *, size_t> have;
    std::lock_guard<std::mutex> lock(mu);
    size_t &cur = have[func];
    if (bytes <= cur || bytes <= 48 * 1024) return LIFE_OK;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess)
        return fail(LIFE_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    cur = bytes;
    return LIFE_OK;
}

// ---------------------------------------------------------------------------
// device block cache (see life_common.cuh)
// ---------------------------------------------------------------------------

namespace {
struct BlockCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void *> free_;      // (device, size class) -> block
    std::unordered_map<void *, std::pair<int, size_t>> owned;  // every block handed out
    size_t cached = 0, cap = 0;
};
BlockCache &bcache()
{
    static BlockCache *c = [] {
        auto *b = new BlockCache;  // process lifetime
        const char *e = std::getenv("LIFE_B200_BLOCK_CACHE_MB");
        b->cap = e ? (size_t)std::strtoull(e, nullptr, 10) << 20 : (size_t)24 << 30;
        return b;
    }();
    return *c;
}
size_t size_class(size_t b)
{
    if (b >= ((size_t)1 << 20)) return (b + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
    return (std::max<size_t>(b, 256) + 255) & ~(size_t)255;
}
// free cached blocks until `need` more bytes fit under the cap (largest first)
void trim_locked(BlockCache &c, size_t need)
{
    int cur = 0;
    cudaGetDevice(&cur);
    while (!c.free_.empty() && c.cached + need > c.cap) {
        auto it = std::prev(c.free_.end());
        c.cached -= it->first.second;
        c.owned.erase(it->second);
        if (it->first.first != cur) cudaSetDevice(it->first.first);  // the block's own device
        cudaFree(it->second);
        if (it->first.first != cur) cudaSetDevice(cur);
        c.free_.erase(it);
    }
}
}  // namespace

int dev_alloc(void **p, size_t bytes)
{
    *p = nullptr;
    const size_t r = size_class(bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    BlockCache &c = bcache();
    {
        std::lock_guard<std::mutex> lock(c.mu);
        // smallest cached block of this device that fits, at most 1/8 larger
        auto it = c.free_.lower_bound({dev, r});
        if (it != c.free_.end() && it->first.first == dev && it->first.second <= r + r / 8) {
            *p = it->second;
            c.cached -= it->first.second;
            c.free_.erase(it);
            return LIFE_OK;
        }
    }
    cudaError_t e = cudaMalloc(p, r);
    if (e == cudaErrorMemoryAllocation) {  // give the cache back and retry once
        cudaGetLastError();
        {
            std::lock_guard<std::mutex> lock(c.mu);
            cudaDeviceSynchronize();
            const size_t keep = c.cap;
            c.cap = 0;
            trim_locked(c, 0);
            c.cap = keep;
        }
        e = cudaMalloc(p, r);
    }
    if (e != cudaSuccess) {
        *p = nullptr;
        return fail(e == cudaErrorMemoryAllocation ? LIFE_ERR_OUT_OF_MEMORY : LIFE_ERR_CUDA,
                    std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lock(c.mu);
    c.owned[*p] = {dev, r};
    return LIFE_OK;
}

void dev_free(void *p)
{
    if (!p) return;
    BlockCache &c = bcache();
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.owned.find(p);
    if (it == c.owned.end()) {
        cudaFree(p);
        return;
    }
    const auto key = it->second;
    if (key.second > c.cap) {
        c.owned.erase(it);
        cudaFree(p);
        return;
    }
    trim_locked(c, key.second);
    c.free_.emplace(key, p);
    c.cached += key.second;
}

namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void *> g_pin_free;
std::unordered_map<void *, size_t> g_pin_size;
}  // namespace

int pinned_alloc(void **p, size_t bytes)
{
    const size_t r = size_class(bytes);
    {
        std::lock_guard<std::mutex> lock(g_pin_mu);
        auto it = g_pin_free.find(r);
        if (it != g_pin_free.end()) {
            *p = it->second;
            g_pin_free.erase(it);
            return LIFE_OK;
        }
    }
    cudaError_t e = cudaMallocHost(p, r);
    if (e != cudaSuccess) return fail(LIFE_ERR_CUDA, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
    std::lock_guard<std::mutex> lock(g_pin_mu);
    g_pin_size[*p] = r;
    return LIFE_OK;
}

void pinned_free(void *p)
{
    if (!p) return;
    std::lock_guard<std::mutex> lock(g_pin_mu);
    auto it = g_pin_size.find(p);
    if (it == g_pin_size.end()) {
        cudaFreeHost(p);
        return;
    }
    g_pin_free.emplace(it->second, p);
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------

__global__ void k_iota_u32(uint32_t *out, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = static_cast<uint32_t>(i);
}

__global__ void k_widen_u32_i64(const uint32_t *in, int64_t *out, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = static_cast<int64_t>(in[i]);
}

// first position k with idx[k] >= bound, per dimension (atomicMin)
__global__ void k_check_range(const uint32_t *a, const uint32_t *v,
                              const uint32_t *f, int64_t n, uint32_t na,
                              uint32_t nv, uint32_t nf,
                              unsigned long long *first_bad)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (a && a[i] >= na) atomicMin(&first_bad[0], (unsigned long long)i);
        if (v && v[i] >= nv) atomicMin(&first_bad[1], (unsigned long long)i);
        if (f && f[i] >= nf) atomicMin(&first_bad[2], (unsigned long long)i);
    }
}

__global__ void k_voxel_l1(const uint32_t *a, const uint32_t *v, const double *val, const double *dn, int64_t n,
                           double *acc)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&acc[v[i]], fabs(val[i]) * dn[a[i]]);
}
__global__ void k_unpack_av(const uint32_t *in, int64_t n, int abits, uint32_t vmax_field, uint32_t *a, uint32_t *v)
{
    const uint32_t am = (1u << abits) - 1u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t w = in[i], vv = w >> abits;
        a[i] = (w & am) == am ? 0xFFFFFFFFu : (w & am);   // saturated field: out of range
        v[i] = vv == vmax_field ? 0xFFFFFFFFu : vv;
    }
}
__global__ void k_widen_u16(const uint16_t *in, int64_t n, uint32_t *out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}
__global__ void k_widen_f32(const float *in, int64_t n, double *out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}

// composite key: (atom group) * nv + voxel
__global__ void k_group_voxel_key(const uint32_t *a, const uint32_t *v,
                                  int64_t n, uint32_t ag, uint32_t nv,
                                  uint32_t *key)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        key[i] = (a[i] / ag) * nv + v[i];
}

__global__ void k_gather_fast(const uint32_t *perm, int64_t n,
                              const uint32_t *a, const uint32_t *f,
                              const double *val, uint32_t ag, uint32_t *a_out,
                              uint32_t *f_out, float *val_out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[i];
        const uint32_t at = a[p];
        a_out[i] = at % ag;
        f_out[i] = f[p];
        val_out[i] = static_cast<float>(val[p]);
    }
}

__global__ void k_gather_exact(const uint32_t *perm, int64_t n,
                               const uint32_t *a, const uint32_t *v,
                               const uint32_t *f, const double *val,
                               uint32_t *a_out, uint32_t *v_out,
                               uint32_t *f_out, double *val_out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[i];
        a_out[i] = a[p];
        v_out[i] = v[p];
        f_out[i] = f[p];
        val_out[i] = val[p];
    }
}

__global__ void k_gather_coo(const int64_t *perm, int64_t n, const uint32_t *a,
                             const uint32_t *v, const uint32_t *f,
                             const double *val, uint32_t *a_out,
                             uint32_t *v_out, uint32_t *f_out, double *val_out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = perm[i];
        if (a_out) a_out[i] = a[p];
        if (v_out) v_out[i] = v[p];
        if (f_out) f_out[i] = f[p];
        if (val_out) val_out[i] = val[p];
    }
}

// ptr[s] = lower_bound(sorted_keys, s) for s in [0, nseg]
__global__ void k_segment_starts(const uint32_t *keys, int64_t n, int64_t nseg,
                                 uint32_t *ptr)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= nseg;
         s += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)keys[mid] < s) lo = mid + 1; else hi = mid;
        }
        ptr[s] = static_cast<uint32_t>(lo);
    }
}

__global__ void k_absmax_f64(const double *x, int64_t n, unsigned long long *out)
{
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(x[i]));
    // nonnegative doubles order like their bit patterns
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_run_flags(const uint32_t *keys, int64_t n, uint8_t *flags,
                            int *unsorted)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool head = (i == 0) || keys[i] != keys[i - 1];
        flags[i] = head ? 1 : 0;
        if (i > 0 && keys[i] < keys[i - 1]) *unsorted = 1;
    }
}

__global__ void k_set_i64(int64_t *p, int64_t v) { *p = v; }

static int grid_for(int64_t n, int threads = 256)
{
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 65535 * 8) b = 65535 * 8;
    return static_cast<int>(b);
}

// ---------------------------------------------------------------------------
// stable radix sort of (u32 key, u32 original index)
// ---------------------------------------------------------------------------
static int bits_for(uint64_t max_key)
{
    int b = 0;
    while (b < 32 && (max_key >> b) != 0) ++b;
    return b < 1 ? 1 : b;
}

// keys_in is not modified; perm_out[i] = original index of i-th sorted item;
// keys_out (optional) receives the sorted keys.
static int stable_sort_u32(const uint32_t *keys_in, int64_t n, uint64_t max_key,
                           uint32_t *perm_out, uint32_t *keys_out,
                           cudaStream_t st)
{
    if (n == 0) return LIFE_OK;
    uint32_t *iota = nullptr, *kout = keys_out;
    LIFE_CUDA(cudaMallocAsync(&iota, n * sizeof(uint32_t), st));
    bool own_kout = false;
    if (!kout) {
        LIFE_CUDA(cudaMallocAsync(&kout, n * sizeof(uint32_t), st));
        own_kout = true;
    }
    k_iota_u32<<<grid_for(n), 256, 0, st>>>(iota, n);
    LIFE_CHECK_LAUNCH();
    size_t temp = 0;
    const int end_bit = bits_for(max_key);
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys_in, kout, iota,
                                              perm_out, n, 0, end_bit, st));
    void *d_temp = nullptr;
    LIFE_CUDA(cudaMallocAsync(&d_temp, temp, st));
    LIFE_CUDA(cub::DeviceRadixSort::SortPairs(d_temp, temp, keys_in, kout, iota,
                                              perm_out, n, 0, end_bit, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    LIFE_CUDA(cudaFreeAsync(d_temp, st));
    LIFE_CUDA(cudaFreeAsync(iota, st));
    if (own_kout) LIFE_CUDA(cudaFreeAsync(kout, st));
    return LIFE_OK;
}

// Split [0, nseg) into `parts` contiguous ranges of near-equal cost where
// cost(s) = count(s) + lambda; counts given by a host prefix array
// `start[s]` (start[nseg] = total).  Mirrors the balancing intent of
// engine.build_plan's coefficient split snapped to run boundaries
// (engine.py:113-184): ranges never cut a segment.
static std::vector<int> balance_ranges(const std::vector<int64_t> &start,
                                       int64_t nseg, int parts, double lambda)
{
    std::vector<int> out(parts + 1, 0);
    const double total = (double)start[nseg] + lambda * (double)nseg;
    int64_t s = 0;
    for (int i = 1; i < parts; ++i) {
        const double target = total * (double)i / (double)parts;
        while (s < nseg && ((double)start[s] + lambda * (double)s) < target) ++s;
        out[i] = static_cast<int>(s);
    }
    out[parts] = static_cast<int>(nseg);
    for (int i = 1; i <= parts; ++i)
        if (out[i] < out[i - 1]) out[i] = out[i - 1];
    return out;
}

}  // namespace life

using namespace life;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Host -> device copies of pageable host arrays through a process-wide ring of
// pinned staging buffers: the host memcpy of chunk k+1 overlaps the DMA of
// chunk k (pageable cudaMemcpy runs at ~7 GB/s on the B200 hosts, pinned DMA
// at ~53 GB/s; tools/h2d_probe.py).
// ---------------------------------------------------------------------------
namespace {
constexpr int kMaxStageThreads = 32;
// chunk and thread count: LIFE_B200_STAGE_KB / LIFE_B200_STAGE_THREADS
size_t stage_chunk()
{
    static const size_t c = [] {
        const char *e = std::getenv("LIFE_B200_STAGE_KB");
        const size_t kb = e ? (size_t)std::strtoull(e, nullptr, 10) : 0;
        // 1 MiB: a thread's staged chunk can still be cache-resident when the DMA
        // reads it (C2 construction 79 -> 71 ms vs 16 MiB chunks; 256 KiB
        // chunks lose to per-copy overhead: tools/gpu_runs/stage_sweep.sh)
        return kb >= 64 ? kb << 10 : (size_t)1 << 20;
    }();
    return c;
}
int stage_threads()
{
    static const int t = [] {
        const char *e = std::getenv("LIFE_B200_STAGE_THREADS");
        const int n = e ? std::atoi(e) : 0;
        return n >= 1 ? std::min(n, kMaxStageThreads) : 12;  // one host memcpy stream reaches ~10 GB/s
    }();
    return t;
}
struct Staging {
    std::mutex mu;
    void *buf[kMaxStageThreads][2] = {};
    cudaEvent_t ev[kMaxStageThreads][2] = {};
    int dev = -1;
};
Staging &staging()
{
    static Staging *s = new Staging;  // process lifetime (pinned memory freed at exit)
    return *s;
}
}  // namespace

namespace life {
// Thread t copies chunks t, t + T, ... through its two pinned slots; the
// copies of all threads go to the caller's stream (distinct destinations, so
// their order does not matter); a slot is reused once its event completed.
void setup_mark(cudaStream_t st, const char *what)
{
    static const bool on = [] {
        const char *e = std::getenv("LIFE_B200_SETUP_TRACE");
        return e && *e && *e != '0';
    }();
    if (!on) return;
    static auto last = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[life setup] %-28s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

int h2d_staged(void *dst, const void *src, size_t bytes, cudaStream_t st) { return h2d_staged_cvt(dst, src, bytes, 0, st); }

// Staged copy of `bytes` destination bytes; stage(out, off, m) fills a
// pinned chunk with destination bytes [off, off + m)
static int h2d_staged_gen(void *dst, size_t bytes, const std::function<void(void *, size_t, size_t)> &stage,
                          cudaStream_t st);

// mode 0: copy; 1: f64 -> f32; 2: u32 -> u16, saturated (`bytes` counts the DESTINATION)
int h2d_staged_cvt(void *dst, const void *src, size_t bytes, int mode, cudaStream_t st)
{
    if (bytes == 0) return LIFE_OK;
    if (mode == 0 && bytes < (4u << 20)) {  // small: one direct copy
        LIFE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return LIFE_OK;
    }
    const size_t in_per_out = mode == 0 ? 1 : 2;  // source bytes per destination byte
    const char *in0 = static_cast<const char *>(src);
    return h2d_staged_gen(dst, bytes, [mode, in0, in_per_out](void *out, size_t off, size_t m) {
        const char *in = in0 + off * in_per_out;
        if (mode == 0) {
            std::memcpy(out, in, m);
        } else if (mode == 1) {
            const double *x = reinterpret_cast<const double *>(in);
            float *y = static_cast<float *>(out);
            for (size_t i = 0, k = m / 4; i < k; ++i) y[i] = (float)x[i];
        } else {  // an out-of-range atom stays out of range (0xFFFF >= n_atoms)
            const uint32_t *x = reinterpret_cast<const uint32_t *>(in);
            uint16_t *y = static_cast<uint16_t *>(out);
            for (size_t i = 0, k = m / 2; i < k; ++i) y[i] = (uint16_t)std::min<uint32_t>(x[i], 0xFFFFu);
        }
    }, st);
}

// atoms and voxels packed into one u32 per coefficient (atom in the low
// `abits` bits), fields saturated so an out-of-range index stays out of
// range for the device check: 4 bytes across PCIe instead of 2 + 4
int h2d_staged_pack_av(uint32_t *dst, const uint32_t *atoms, const uint32_t *voxels, int64_t n, int abits, int vbits,
                       cudaStream_t st)
{
    if (n <= 0) return LIFE_OK;
    const uint32_t am = (1u << abits) - 1u, vm = vbits >= 32 ? ~0u : (1u << vbits) - 1u;
    return h2d_staged_gen(dst, (size_t)n * 4, [=](void *out, size_t off, size_t m) {
        const size_t i0 = off / 4;
        uint32_t *y = static_cast<uint32_t *>(out);
        for (size_t i = 0, k = m / 4; i < k; ++i)
            y[i] = std::min(atoms[i0 + i], am) | (std::min(voxels[i0 + i], vm) << abits);
    }, st);
}

static int h2d_staged_gen(void *dst, size_t bytes, const std::function<void(void *, size_t, size_t)> &stage,
                          cudaStream_t st)
{
    Staging &S = staging();
    std::lock_guard<std::mutex> lk(S.mu);
    int dev = 0;
    LIFE_CUDA(cudaGetDevice(&dev));
    if (S.dev != dev) {  // (re)create on this device's context
        for (auto &row : S.ev)
            for (auto &e : row) {
                if (e) cudaEventDestroy(e);
                e = nullptr;
            }
        for (auto &row : S.buf)
            for (auto &p : row) {
                if (p) cudaFreeHost(p);
                p = nullptr;
            }
        for (int t = 0; t < stage_threads(); ++t)
            for (int j = 0; j < 2; ++j) {
                LIFE_CUDA(cudaHostAlloc(&S.buf[t][j], stage_chunk(), cudaHostAllocDefault));
                LIFE_CUDA(cudaEventCreateWithFlags(&S.ev[t][j], cudaEventDisableTiming));
            }
        S.dev = dev;
    }
    const size_t chunk = stage_chunk();
    const size_t nchunk = (bytes + chunk - 1) / chunk;
    const int T = (int)std::min<size_t>(stage_threads(), nchunk);
    std::vector<cudaError_t> err(T, cudaSuccess);
    auto work = [&](int t) {
        cudaError_t e = cudaSetDevice(dev);
        int n = 0;
        for (size_t k = t; k < nchunk && e == cudaSuccess; k += T, ++n) {
            const int j = n & 1;
            const size_t off = k * chunk, m = std::min(chunk, bytes - off);
            if ((e = cudaEventSynchronize(S.ev[t][j])) != cudaSuccess) break;  // slot's previous DMA done
            stage(S.buf[t][j], off, m);
            if ((e = cudaMemcpyAsync(static_cast<char *>(dst) + off, S.buf[t][j], m, cudaMemcpyHostToDevice, st)) !=
                cudaSuccess)
                break;
            e = cudaEventRecord(S.ev[t][j], st);
        }
        err[t] = e;
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    for (cudaError_t e : err)
        if (e != cudaSuccess) return fail(LIFE_ERR_CUDA, std::string("staged copy: ") + cudaGetErrorString(e));
    // the staging slots are reused by the next call: make its waits valid
    for (int t = 0; t < T; ++t)
        for (int j = 0; j < 2; ++j) LIFE_CUDA(cudaEventRecord(S.ev[t][j], st));
    return LIFE_OK;
}
}  // namespace life

extern "C" {

int life_abi_version(void) { return LIFE_B200_ABI_VERSION; }

const char *life_last_error(void) { return t_last_error.c_str(); }

uint64_t life_launch_count(void) { return g_launches.load(); }

const char *life_status_string(int status)
{
    switch (status) {
    case LIFE_OK: return "ok";
    case LIFE_ERR_CONFIG_INVALID: return "ConfigInvalid";
    case LIFE_ERR_DIMENSION_MISMATCH: return "DimensionMismatch";
    case LIFE_ERR_PLAN_TENSOR_MISMATCH: return "PlanTensorMismatch";
    case LIFE_ERR_STRATEGY_REQUIRES_SORTED: return "StrategyRequiresSorted";
    case LIFE_ERR_DEGENERATE_STEP: return "DegenerateStep";
    case LIFE_ERR_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
    case LIFE_ERR_ARITHMETIC_OVERFLOW: return "ArithmeticOverflow";
    case LIFE_ERR_NOT_SORTED: return "NotSorted";
    case LIFE_ERR_NON_FINITE: return "NonFiniteValue";
    case LIFE_ERR_CUDA: return "CudaError";
    case LIFE_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    case LIFE_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case LIFE_ERR_NCCL: return "NcclError";
    default: return "unknown";
    }
}

int life_stable_argsort_u32(const uint32_t *keys_dev, int64_t n,
                            int64_t *perm_dev, void *stream)
{
    if (n < 0 || (n > 0 && (!keys_dev || !perm_dev)))
        return fail(LIFE_ERR_INVALID_ARGUMENT, "null array");
    if (n > 0xFFFFFFFFll)
        return fail(LIFE_ERR_CONFIG_INVALID, "n exceeds 2^32-1");
    if (n == 0) return ok();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t *perm32 = nullptr;
    LIFE_CUDA(cudaMallocAsync(&perm32, n * sizeof(uint32_t), st));
    LIFE_TRY(stable_sort_u32(keys_dev, n, 0xFFFFFFFFull, perm32, nullptr, st));
    k_widen_u32_i64<<<grid_for(n), 256, 0, st>>>(perm32, perm_dev, n);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaFreeAsync(perm32, st));
    return ok();
}

int life_detect_runs_u32(const uint32_t *keys_dev, int64_t n,
                         int64_t *boundaries_dev, uint32_t *run_keys_dev,
                         int64_t *n_runs_out, void *stream)
{
    if (!boundaries_dev || !n_runs_out || (n > 0 && (!keys_dev || !run_keys_dev)))
        return fail(LIFE_ERR_INVALID_ARGUMENT, "null array");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        k_set_i64<<<1, 1, 0, st>>>(boundaries_dev, 0);
        LIFE_CHECK_LAUNCH();
        LIFE_CUDA(cudaStreamSynchronize(st));
        *n_runs_out = 0;
        return ok();
    }
    uint8_t *flags = nullptr;
    int *unsorted = nullptr;
    int64_t *nsel = nullptr;
    LIFE_CUDA(cudaMallocAsync(&flags, n, st));
    LIFE_CUDA(cudaMallocAsync(&unsorted, sizeof(int), st));
    LIFE_CUDA(cudaMallocAsync(&nsel, 2 * sizeof(int64_t), st));
    LIFE_CUDA(cudaMemsetAsync(unsorted, 0, sizeof(int), st));
    k_run_flags<<<grid_for(n), 256, 0, st>>>(keys_dev, n, flags, unsorted);
    LIFE_CHECK_LAUNCH();
    cub::CountingInputIterator<int64_t> pos(0);
    size_t t1 = 0, t2 = 0;
    LIFE_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, pos, flags, boundaries_dev,
                                         nsel, n, st));
    LIFE_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, keys_dev, flags,
                                         run_keys_dev, nsel + 1, n, st));
    void *temp = nullptr;
    LIFE_CUDA(cudaMallocAsync(&temp, std::max(t1, t2), st));
    LIFE_CUDA(cub::DeviceSelect::Flagged(temp, t1, pos, flags, boundaries_dev,
                                         nsel, n, st));
    LIFE_CUDA(cub::DeviceSelect::Flagged(temp, t2, keys_dev, flags,
                                         run_keys_dev, nsel + 1, n, st));
    g_launches.fetch_add(4, std::memory_order_relaxed);
    int64_t h_nsel[2] = {0, 0};
    int h_unsorted = 0;
    LIFE_CUDA(cudaMemcpyAsync(h_nsel, nsel, sizeof(h_nsel), cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaMemcpyAsync(&h_unsorted, unsorted, sizeof(int),
                              cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    k_set_i64<<<1, 1, 0, st>>>(boundaries_dev + h_nsel[0], n);
    LIFE_CHECK_LAUNCH();
    LIFE_CUDA(cudaFreeAsync(temp, st));
    LIFE_CUDA(cudaFreeAsync(flags, st));
    LIFE_CUDA(cudaFreeAsync(unsorted, st));
    LIFE_CUDA(cudaFreeAsync(nsel, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    if (h_unsorted) return fail(LIFE_ERR_NOT_SORTED, "key array is not sorted");
    *n_runs_out = h_nsel[0];
    return ok();
}

int life_gather_coo(const int64_t *perm_dev, int64_t n, const uint32_t *atoms,
                    const uint32_t *voxels, const uint32_t *fibers,
                    const double *values, uint32_t *atoms_out,
                    uint32_t *voxels_out, uint32_t *fibers_out,
                    double *values_out, void *stream)
{
    if (n == 0) return ok();
    if (!perm_dev) return fail(LIFE_ERR_INVALID_ARGUMENT, "null perm");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_gather_coo<<<grid_for(n), 256, 0, st>>>(perm_dev, n, atoms, voxels, fibers,
                                              values, atoms_out, voxels_out,
                                              fibers_out, values_out);
    LIFE_CHECK_LAUNCH();
    return ok();
}

// ---------------------------------------------------------------------------
// operator construction
// ---------------------------------------------------------------------------
static int build_exact(life_phi *phi, const uint32_t *a, const uint32_t *v,
                       const uint32_t *f, const double *val, const double *dict,
                       cudaStream_t st, std::vector<int64_t> &fiber_start)
{
    const int64_t n = phi->nc;
    uint32_t *perm = nullptr, *skeys = nullptr;
    LIFE_CUDA(cudaMallocAsync(&perm, std::max<int64_t>(n, 1) * sizeof(uint32_t), st));
    LIFE_CUDA(cudaMallocAsync(&skeys, std::max<int64_t>(n, 1) * sizeof(uint32_t), st));
    const int exact_threads = 256;
    phi->xblocks = phi->sms * 4;
    phi->xW = phi->xblocks * (exact_threads / 32);

    for (int pass = 0; pass < 2; ++pass) {
        const bool by_voxel = pass == 0;
        const uint32_t *key = by_voxel ? v : f;
        const int64_t nseg = by_voxel ? phi->nv : phi->nf;
        uint32_t **ao = by_voxel ? &phi->xv_atom : &phi->xf_atom;
        uint32_t **vo = by_voxel ? &phi->xv_voxel : &phi->xf_voxel;
        uint32_t **fo = by_voxel ? &phi->xv_fiber : &phi->xf_fiber;
        double **valo = by_voxel ? &phi->xv_val : &phi->xf_val;
        uint32_t **ptro = by_voxel ? &phi->xv_ptr : &phi->xf_ptr;
        int **wpo = by_voxel ? &phi->xv_wpart : &phi->xf_wpart;
        LIFE_TRY(dalloc(phi, ao, n));
        LIFE_TRY(dalloc(phi, vo, n));
        LIFE_TRY(dalloc(phi, fo, n));
        LIFE_TRY(dalloc(phi, valo, n));
        LIFE_TRY(dalloc(phi, ptro, nseg + 1));
        LIFE_TRY(stable_sort_u32(key, n, (uint64_t)nseg, perm, skeys, st));
        if (n > 0) {
            k_gather_exact<<<grid_for(n), 256, 0, st>>>(perm, n, a, v, f, val, *ao,
                                                        *vo, *fo, *valo);
            LIFE_CHECK_LAUNCH();
        }
        k_segment_starts<<<grid_for(nseg + 1), 256, 0, st>>>(skeys, n, nseg, *ptro);
        LIFE_CHECK_LAUNCH();
        std::vector<uint32_t> hptr(nseg + 1);
        LIFE_CUDA(cudaMemcpyAsync(hptr.data(), *ptro, (nseg + 1) * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> start(nseg + 1);
        for (int64_t s = 0; s <= nseg; ++s) start[s] = hptr[s];
        std::vector<int> parts = balance_ranges(start, nseg, phi->xW, 2.0);
        LIFE_TRY(dalloc(phi, wpo, phi->xW + 1));
        LIFE_CUDA(cudaMemcpyAsync(*wpo, parts.data(), (phi->xW + 1) * sizeof(int),
                                  cudaMemcpyHostToDevice, st));
        int64_t runs = 0, mx = 0;
        for (int64_t s = 0; s < nseg; ++s) {
            const int64_t len = start[s + 1] - start[s];
            if (len) ++runs;
            mx = std::max(mx, len);
        }
        if (by_voxel) {
            phi->n_voxel_runs = runs;
            phi->max_voxel_run = mx;
        } else {
            phi->n_fiber_runs = runs;
            phi->max_fiber_run = mx;
            fiber_start = start;
        }
        LIFE_CUDA(cudaStreamSynchronize(st));
    }
    LIFE_TRY(dalloc(phi, &phi->D64, (size_t)phi->na * phi->nt));
    LIFE_CUDA(cudaMemcpyAsync(phi->D64, dict, (size_t)phi->na * phi->nt * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
    LIFE_CUDA(cudaFreeAsync(perm, st));
    LIFE_CUDA(cudaFreeAsync(skeys, st));
    phi->has_exact = true;
    return LIFE_OK;
}

static int build_fast(life_phi *phi, const uint32_t *a, const uint32_t *v,
                      const uint32_t *f, const double *val,
                      const std::vector<double> &hdict, cudaStream_t st)
{
    const int64_t n = phi->nc;
    int optin = 0;
    LIFE_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                     phi->device));
    const int64_t budget = (int64_t)optin - 4096;  // static smem + slack
    const int64_t row_bytes = (int64_t)phi->nt * 4;
    int64_t ag = budget / row_bytes;
    if (ag < 1) return fail(LIFE_ERR_CONFIG_INVALID, "n_dirs too large for one shared-memory row");
    int G = 1;
    if (ag >= phi->na) {
        ag = phi->na;
    } else {
        G = (int)((phi->na + ag - 1) / ag);
        ag = (phi->na + G - 1) / G;  // equalize the groups
    }
    if ((int64_t)G * phi->nv >= 0xFFFFFFFFll)
        return fail(LIFE_ERR_CONFIG_INVALID, "atom groups x voxels exceed u32 keys");
    phi->G = G;
    phi->ag = (int)ag;
    phi->slice_floats = (int)(((ag * phi->nt) + 3) / 4 * 4);
    phi->smem = (size_t)phi->slice_floats * sizeof(float);

    // persistent grid: one 512-thread CTA per SM (the slice fills shared memory)
    int bps = 1;
    phi->nblocks = phi->sms * bps;
    phi->W = phi->nblocks * (kSpmvThreads / 32);

    // sort by (group, voxel), stable
    uint32_t *key = nullptr, *skeys = nullptr, *perm = nullptr;
    LIFE_CUDA(cudaMallocAsync(&key, std::max<int64_t>(n, 1) * sizeof(uint32_t), st));
    LIFE_CUDA(cudaMallocAsync(&skeys, std::max<int64_t>(n, 1) * sizeof(uint32_t), st));
    LIFE_CUDA(cudaMallocAsync(&perm, std::max<int64_t>(n, 1) * sizeof(uint32_t), st));
    const int64_t nseg = (int64_t)G * phi->nv;
    if (n > 0) {
        k_group_voxel_key<<<grid_for(n), 256, 0, st>>>(a, v, n, (uint32_t)ag,
                                                       (uint32_t)phi->nv, key);
        LIFE_CHECK_LAUNCH();
    }
    LIFE_TRY(stable_sort_u32(key, n, (uint64_t)nseg, perm, skeys, st));
    LIFE_TRY(dalloc(phi, &phi->atom, n));
    LIFE_TRY(dalloc(phi, &phi->fiber, n));
    LIFE_TRY(dalloc(phi, &phi->val, n));
    LIFE_TRY(dalloc(phi, &phi->gptr, nseg + 1));
    if (n > 0) {
        k_gather_fast<<<grid_for(n), 256, 0, st>>>(perm, n, a, f, val, (uint32_t)ag,
                                                   phi->atom, phi->fiber, phi->val);
        LIFE_CHECK_LAUNCH();
    }
    k_segment_starts<<<grid_for(nseg + 1), 256, 0, st>>>(skeys, n, nseg, phi->gptr);
    LIFE_CHECK_LAUNCH();
    std::vector<uint32_t> hptr(nseg + 1);
    LIFE_CUDA(cudaMemcpyAsync(hptr.data(), phi->gptr, (nseg + 1) * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    // per-voxel totals over groups -> warp partition
    std::vector<int64_t> start(phi->nv + 1, 0);
    int64_t runs = 0, mx = 0;
    for (int64_t vv = 0; vv < phi->nv; ++vv) {
        int64_t tot = 0;
        for (int g = 0; g < G; ++g)
            tot += (int64_t)hptr[(int64_t)g * phi->nv + vv + 1] - hptr[(int64_t)g * phi->nv + vv];
        start[vv + 1] = start[vv] + tot;
        if (tot) ++runs;
        mx = std::max(mx, tot);
    }
    phi->n_voxel_runs = runs;
    phi->max_voxel_run = mx;
    std::vector<int> parts = balance_ranges(start, phi->nv, phi->W, 2.0);
    LIFE_TRY(dalloc(phi, &phi->wpart, phi->W + 1));
    LIFE_CUDA(cudaMemcpyAsync(phi->wpart, parts.data(), (phi->W + 1) * sizeof(int),
                              cudaMemcpyHostToDevice, st));
    // fp32 dictionary slices, each 16-byte aligned
    std::vector<float> hD((size_t)G * phi->slice_floats, 0.f);
    for (int64_t at = 0; at < phi->na; ++at) {
        const int64_t g = at / ag, al = at % ag;
        for (int t = 0; t < phi->nt; ++t)
            hD[(size_t)g * phi->slice_floats + al * phi->nt + t] =
                static_cast<float>(hdict[(size_t)at * phi->nt + t]);
    }
    LIFE_TRY(dalloc(phi, &phi->Dg, hD.size()));
    LIFE_CUDA(cudaMemcpyAsync(phi->Dg, hD.data(), hD.size() * sizeof(float),
                              cudaMemcpyHostToDevice, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    LIFE_CUDA(cudaFreeAsync(key, st));
    LIFE_CUDA(cudaFreeAsync(skeys, st));
    LIFE_CUDA(cudaFreeAsync(perm, st));
    phi->has_fast = true;
    return LIFE_OK;
}

__global__ void k_fiber_hist(const uint32_t *f, int64_t n, unsigned *count)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&count[f[i]], 1u);
}

__global__ void k_max_u32(const unsigned *x, int64_t n, unsigned *mx, unsigned *nz)
{
    unsigned m = 0, c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        m = max(m, x[i]);
        c += x[i] ? 1u : 0u;
    }
    atomicMax(mx, m);
    atomicAdd(nz, c);
}

static void destroy_impl(life_phi *phi);

static int create_impl(const life_dims *dims, const uint32_t *atoms,
                       const uint32_t *voxels, const uint32_t *fibers,
                       const double *values, const double *dict, uint32_t flags,
                       cudaStream_t st, life_phi **out, int64_t *bad_position)
{
    if (!dims || !out) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (dims->n_atoms <= 0 || dims->n_voxels <= 0 || dims->n_fibers <= 0 ||
        dims->n_dirs <= 0 || dims->n_coeffs < 0)
        return fail(LIFE_ERR_CONFIG_INVALID, "dimensions must be positive");
    if (dims->n_atoms > 0x7FFFFFFF || dims->n_voxels > 0x7FFFFFFF ||
        dims->n_fibers > 0x7FFFFFFF || dims->n_coeffs > 0xFFFFFFFEll)
        return fail(LIFE_ERR_CONFIG_INVALID, "dimension exceeds the 32-bit index space");
    if (dims->n_dirs > 32 * kMaxNT)
        return fail(LIFE_ERR_CONFIG_INVALID, "n_dirs > 320 unsupported");
    if (dims->n_voxels * dims->n_dirs > 0xFFFFFFFFll * 4)
        return fail(LIFE_ERR_ARITHMETIC_OVERFLOW, "signal length too large");
    const int64_t n = dims->n_coeffs;
    if (n > 0 && (!atoms || !voxels || !fibers || !values))
        return fail(LIFE_ERR_INVALID_ARGUMENT, "null coefficient array");
    if (!dict) return fail(LIFE_ERR_INVALID_ARGUMENT, "null dictionary");

    auto t0 = std::chrono::steady_clock::now();
    setup_mark(st, "start");
    {   // keep freed stream-ordered allocations mapped for reuse (restructuring
        // temporaries are GBs at C2; re-mapping them each create costs seconds)
        static bool pool_set = false;
        if (!pool_set) {
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess &&
                cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            pool_set = true;
        }
    }
    life_phi *phi = new life_phi();
    phi->dims = *dims;
    phi->na = (int)dims->n_atoms;
    phi->nv = (int)dims->n_voxels;
    phi->nf = (int)dims->n_fibers;
    phi->nt = (int)dims->n_dirs;
    phi->nc = n;
    LIFE_CUDA(cudaGetDevice(&phi->device));
    LIFE_CUDA(cudaDeviceGetAttribute(&phi->sms, cudaDevAttrMultiProcessorCount, phi->device));

    struct Guard {
        life_phi **slot;
        life_phi *p;
        std::vector<void *> tmp;
        cudaStream_t st;
        ~Guard()
        {
            if (!tmp.empty()) cudaDeviceSynchronize();  // as cudaFree would
            for (void *q : tmp) dev_free(q);
            if (p) destroy_impl(p);  // keeps the error message of the failed build
        }
    } guard{out, phi, {}, st};

    const bool host = flags & LIFE_PHI_HOST_INPUT;
    const uint32_t *a = atoms, *v = voxels, *f = fibers;
    const double *val = values, *D = dict;
    const size_t dlen = (size_t)phi->na * phi->nt;
    // Host input: atoms, voxels and the dictionary are staged now; fibers and
    // values follow from a host thread on a side stream while the first
    // restructuring phases (which read only atoms and voxels) run.
    struct Deferred {
        std::thread th;
        cudaStream_t s2 = nullptr;
        cudaEvent_t ev = nullptr;
        int rc = LIFE_OK;
        std::string msg;
        ~Deferred()
        {
            if (th.joinable()) th.join();
            if (ev) cudaEventDestroy(ev);
            if (s2) cudaStreamDestroy(s2);
        }
    } dfr;
    if (host) {
        uint32_t *da, *dv, *df;
        double *dval, *dD;
        const size_t nn = std::max<int64_t>(n, 1);
        LIFE_TRY(dev_alloc((void **)&da, nn * 4)); guard.tmp.push_back(da);
        LIFE_TRY(dev_alloc((void **)&dv, nn * 4)); guard.tmp.push_back(dv);
        LIFE_TRY(dev_alloc((void **)&df, nn * 4)); guard.tmp.push_back(df);
        LIFE_TRY(dev_alloc((void **)&dval, nn * 8)); guard.tmp.push_back(dval);
        LIFE_TRY(dev_alloc((void **)&dD, dlen * 8)); guard.tmp.push_back(dD);
        // fewer bytes over PCIe: atoms as u16 when they fit (widened on the
        // device, lossless); values as f32 when the caller allows it
        // (LIFE_PHI_VALUES_F32: fp32-only operator, whose kernels round the
        // values to f32 anyway)
        // atoms and voxels packed into one u32 when both fields fit with an
        // all-ones value left over (>= the dimension: out of range)
        auto field_bits = [](int64_t dim) { int b = 1; while (b < 32 && ((1ll << b) - 1) < dim) ++b; return b; };
        const int abits = field_bits(phi->na), vbits = field_bits(phi->nv);
        static const bool no_pack = [] { const char *e = std::getenv("LIFE_B200_NO_PACK"); return e && *e == '1'; }();
        const bool pack = n > 0 && abits + vbits <= 32 && !no_pack;
        const bool a16 = !pack && phi->na < 65535 && n > 0;
        const bool v32 = (flags & LIFE_PHI_VALUES_F32) && !(flags & LIFE_PHI_EXACT_F64) && n > 0;
        void *narrow = nullptr;
        if (a16 || v32 || pack) {
            LIFE_TRY(dev_alloc((void **)&narrow, (size_t)n * 4));
            guard.tmp.push_back(narrow);
        }
        uint16_t *na16 = static_cast<uint16_t *>(narrow);
        float *nv32 = static_cast<float *>(narrow);  // reused after the atoms are widened
        if (pack) {
            uint32_t *pk = static_cast<uint32_t *>(narrow);
            LIFE_TRY(h2d_staged_pack_av(pk, atoms, voxels, n, abits, vbits, st));
            k_unpack_av<<<grid_for(n), 256, 0, st>>>(pk, n, abits, vbits >= 32 ? ~0u : (1u << vbits) - 1u, da, dv);
            LIFE_CHECK_LAUNCH();
        } else if (n > 0) {
            if (a16) {
                LIFE_TRY(h2d_staged_cvt(na16, atoms, (size_t)n * 2, 2, st));
                k_widen_u16<<<grid_for(n), 256, 0, st>>>(na16, n, da);
                LIFE_CHECK_LAUNCH();
            } else {
                LIFE_TRY(h2d_staged(da, atoms, (size_t)n * 4, st));
            }
            LIFE_TRY(h2d_staged(dv, voxels, (size_t)n * 4, st));
        }
        if (v32 && (a16 || pack)) {  // the side stream must not overwrite the narrow atoms before they are widened
            LIFE_CUDA(cudaStreamSynchronize(st));
        }
        LIFE_TRY(h2d_staged(dD, dict, dlen * 8, st));
        if (n > 0) {
            LIFE_CUDA(cudaStreamCreateWithFlags(&dfr.s2, cudaStreamNonBlocking));
            LIFE_CUDA(cudaEventCreateWithFlags(&dfr.ev, cudaEventDisableTiming));
            dfr.th = std::thread([&dfr, df, dval, fibers, values, n, v32, nv32, dev = phi->device] {
                cudaSetDevice(dev);
                int rc = h2d_staged(df, fibers, (size_t)n * 4, dfr.s2);
                if (rc == LIFE_OK) {
                    if (v32) {
                        rc = h2d_staged_cvt(nv32, values, (size_t)n * 4, 1, dfr.s2);
                        if (rc == LIFE_OK) {
                            k_widen_f32<<<grid_for(n), 256, 0, dfr.s2>>>(nv32, n, dval);
                            if (cudaGetLastError() != cudaSuccess) rc = fail(LIFE_ERR_CUDA, "widen launch");
                        }
                    } else {
                        rc = h2d_staged(dval, values, (size_t)n * 8, dfr.s2);
                    }
                }
                if (rc == LIFE_OK && cudaEventRecord(dfr.ev, dfr.s2) != cudaSuccess) rc = fail(LIFE_ERR_CUDA, "event record");
                if (rc != LIFE_OK) dfr.msg = life_last_error();
                dfr.rc = rc;
            });
        }
        a = da; v = dv; f = df; val = dval; D = dD;
    }
    setup_mark(st, "h2d (atoms, voxels)");

    // index range check (validate(), tensor.py:232-286; first bad position):
    // atoms and voxels now, fibers once they are on the device
    unsigned long long *bad = nullptr;
    LIFE_TRY(dev_alloc((void **)&bad, 3 * sizeof(unsigned long long)));
    guard.tmp.push_back(bad);
    auto range_check = [&](bool av, bool fib) -> int {
        LIFE_CUDA(cudaMemsetAsync(bad, 0xFF, 3 * sizeof(unsigned long long), st));
        if (n > 0) {
            k_check_range<<<grid_for(n), 256, 0, st>>>(av ? a : nullptr, av ? v : nullptr, fib ? f : nullptr, n,
                                                       phi->na, phi->nv, phi->nf, bad);
            LIFE_CHECK_LAUNCH();
        }
        unsigned long long hb[3];
        LIFE_CUDA(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        static const char *names[3] = {"atom", "voxel", "fiber"};
        for (int i = 0; i < 3; ++i)
            if (hb[i] != ~0ull) {
                if (bad_position) *bad_position = (int64_t)hb[i];
                return fail(LIFE_ERR_INDEX_OUT_OF_RANGE,
                            std::string(names[i]) + " index out of range at position " + std::to_string(hb[i]));
            }
        return LIFE_OK;
    };
    LIFE_TRY(range_check(true, !host));

    // host copy of the dictionary (small): fp32 slices and row norms
    std::vector<double> hdict(dlen);
    LIFE_CUDA(cudaMemcpyAsync(hdict.data(), D, dlen * 8, cudaMemcpyDeviceToHost, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    double dmax = 0.0;
    for (int64_t at = 0; at < phi->na; ++at) {
        double s = 0.0;
        for (int t = 0; t < phi->nt; ++t) s += hdict[at * phi->nt + t] * hdict[at * phi->nt + t];
        dmax = std::max(dmax, std::sqrt(s));
    }
    phi->dmax = dmax * (1.0 + 1e-6);

    // fibers and values resident (joins the staging thread), fiber range
    // check, value bound and fascicle sizes; idempotent
    bool fv_ready = false;
    auto ready_fv = [&]() -> int {
        if (fv_ready) return LIFE_OK;
        fv_ready = true;
        if (dfr.th.joinable()) {
            dfr.th.join();
            if (dfr.rc != LIFE_OK) return fail(dfr.rc, dfr.msg);
            LIFE_CUDA(cudaStreamWaitEvent(st, dfr.ev, 0));
            LIFE_TRY(range_check(false, true));
        }
        setup_mark(st, "h2d (fibers, values)");
        unsigned long long *vm = nullptr;
        unsigned *cnt = nullptr, *mx = nullptr;
        LIFE_TRY(dev_alloc((void **)&vm, 8)); guard.tmp.push_back(vm);
        LIFE_TRY(dev_alloc((void **)&cnt, (size_t)phi->nf * 4)); guard.tmp.push_back(cnt);
        LIFE_TRY(dev_alloc((void **)&mx, 8)); guard.tmp.push_back(mx);
        LIFE_CUDA(cudaMemsetAsync(vm, 0, 8, st));
        LIFE_CUDA(cudaMemsetAsync(cnt, 0, (size_t)phi->nf * 4, st));
        LIFE_CUDA(cudaMemsetAsync(mx, 0, 8, st));
        if (n > 0) {
            k_absmax_f64<<<std::min(grid_for(n), phi->sms * 8), 256, 0, st>>>(val, n, vm);
            LIFE_CHECK_LAUNCH();
            k_fiber_hist<<<grid_for(n), 256, 0, st>>>(f, n, cnt);
            LIFE_CHECK_LAUNCH();
        }
        k_max_u32<<<std::min(grid_for(phi->nf), phi->sms * 8), 256, 0, st>>>(cnt, phi->nf, mx, mx + 1);
        LIFE_CHECK_LAUNCH();
        unsigned long long hvm;
        unsigned hmx[2];
        LIFE_CUDA(cudaMemcpyAsync(&hvm, vm, 8, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaMemcpyAsync(hmx, mx, 8, cudaMemcpyDeviceToHost, st));
        LIFE_CUDA(cudaStreamSynchronize(st));
        double dv;
        std::memcpy(&dv, &hvm, 8);
        phi->vmax = dv * (1.0 + 1e-6);
        // max_v sum_{c in v} ||D_a||_2 |value|: bounds ||(M w)_v|| by max|w|
        // without a collective (voxel-sharded WC scale, life_solver.cu)
        if (n > 0) {
            double *dn = nullptr, *acc = nullptr;
            unsigned long long *mxv = nullptr;
            std::vector<double> hdn(phi->na);
            for (int64_t at = 0; at < phi->na; ++at) {
                double q = 0.0;
                for (int t = 0; t < phi->nt; ++t) q += hdict[at * phi->nt + t] * hdict[at * phi->nt + t];
                hdn[at] = std::sqrt(q);
            }
            LIFE_TRY(dev_alloc((void **)&dn, (size_t)phi->na * 8)); guard.tmp.push_back(dn);
            LIFE_TRY(dev_alloc((void **)&acc, (size_t)phi->nv * 8)); guard.tmp.push_back(acc);
            LIFE_TRY(dev_alloc((void **)&mxv, 8)); guard.tmp.push_back(mxv);
            LIFE_CUDA(cudaMemcpyAsync(dn, hdn.data(), (size_t)phi->na * 8, cudaMemcpyHostToDevice, st));
            LIFE_CUDA(cudaMemsetAsync(acc, 0, (size_t)phi->nv * 8, st));
            LIFE_CUDA(cudaMemsetAsync(mxv, 0, 8, st));
            k_voxel_l1<<<std::min(grid_for(n), phi->sms * 8), 256, 0, st>>>(a, v, val, dn, n, acc);
            LIFE_CHECK_LAUNCH();
            k_absmax_f64<<<std::min(grid_for(phi->nv), phi->sms * 8), 256, 0, st>>>(acc, phi->nv, mxv);
            LIFE_CHECK_LAUNCH();
            unsigned long long hm;
            LIFE_CUDA(cudaMemcpyAsync(&hm, mxv, 8, cudaMemcpyDeviceToHost, st));
            LIFE_CUDA(cudaStreamSynchronize(st));
            double vs;
            std::memcpy(&vs, &hm, 8);
            // rounded up to a power of two: the atomic sums' last bits vary
            // run to run, the bound (and so the WC scale) must not
            int e = 0;
            std::frexp(vs * (1.0 + 1e-6), &e);
            phi->vsmax = vs > 0.0 ? std::ldexp(1.0, e) : 0.0;
        }
        phi->fmax_nnz = std::max<int64_t>(hmx[0], 1);
        phi->max_fiber_run = hmx[0];
        phi->n_fiber_runs = hmx[1];
        return LIFE_OK;
    };

    if (!(flags & LIFE_PHI_NO_FAST_F32)) {
        // Layout choice: register-tiled dense kernels when voxels
        // carry >= 1/8 of all atoms on average, sparse segment kernels
        // otherwise; flags can force either.
        int64_t occupied = 0;
        {
            unsigned *cnt = nullptr, *mx = nullptr;
            LIFE_TRY(dev_alloc((void **)&cnt, (size_t)phi->nv * 4)); guard.tmp.push_back(cnt);
            LIFE_TRY(dev_alloc((void **)&mx, 8)); guard.tmp.push_back(mx);
            LIFE_CUDA(cudaMemsetAsync(cnt, 0, (size_t)phi->nv * 4, st));
            LIFE_CUDA(cudaMemsetAsync(mx, 0, 8, st));
            if (n > 0) {
                k_fiber_hist<<<grid_for(n), 256, 0, st>>>(v, n, cnt);
                LIFE_CHECK_LAUNCH();
            }
            k_max_u32<<<std::min(grid_for(phi->nv), phi->sms * 8), 256, 0, st>>>(cnt, phi->nv, mx, mx + 1);
            LIFE_CHECK_LAUNCH();
            unsigned hm[2];
            LIFE_CUDA(cudaMemcpyAsync(hm, mx, 8, cudaMemcpyDeviceToHost, st));
            LIFE_CUDA(cudaStreamSynchronize(st));
            occupied = hm[1];
            phi->n_voxel_runs = hm[1];
            phi->max_voxel_run = hm[0];
        }
        // Layout choice: the binned tile products when
        // voxels carry >= 1/8 of all atoms on average (and n_dirs <= 192),
        // the voxel-segment kernels otherwise; flags can force either.
        bool tile = (n * 8 >= occupied * (int64_t)phi->na) && n > 0;
        if (flags & LIFE_PHI_FORCE_SPARSE) tile = false;
        if (flags & LIFE_PHI_FORCE_DENSE) tile = n > 0;
        const char *bin_env = getenv("LIFE_BIN");
        const bool want_bin = tile && !(flags & (LIFE_PHI_NO_TENSOR | LIFE_PHI_NO_BIN)) &&
                              !(bin_env && bin_env[0] == '0');
        setup_mark(st, "checks + dictionary");
        if (want_bin) LIFE_TRY(build_bin(phi, a, v, f, val, hdict, ready_fv, st));
        setup_mark(st, "build_bin");
        LIFE_TRY(ready_fv());
        if (!phi->has_bin) LIFE_TRY(build_fast(phi, a, v, f, val, hdict, st));
    }
    LIFE_TRY(ready_fv());
    std::vector<int64_t> fiber_start;
    if (flags & LIFE_PHI_EXACT_F64)
        LIFE_TRY(build_exact(phi, a, v, f, val, D, st, fiber_start));

    // reduction scratch
    // fixed-point WC accumulator (both fp32 kernel families)
    LIFE_TRY(dalloc(phi, &phi->wfix, phi->nf));
    LIFE_CUDA(cudaMemsetAsync(phi->wfix, 0, (size_t)phi->nf * sizeof(unsigned long long), st));
    phi->red_cap = std::max(std::max(phi->W, phi->xW), phi->sms * 16) + 1;
    if (phi->has_bin)
        phi->red_cap = std::max(phi->red_cap, phi->b_tile_grid * bin_tile_warps(phi) + phi->sms * 8 + 1);
    LIFE_TRY(dalloc(phi, &phi->red.part_d, phi->red_cap));
    LIFE_TRY(dalloc(phi, &phi->red.part_u, phi->red_cap));
    LIFE_TRY(dalloc(phi, &phi->red.part_f, phi->red_cap));
    LIFE_TRY(dalloc(phi, &phi->red.counter, 4));
    LIFE_TRY(dalloc(phi, &phi->part_d2, phi->red_cap));
    LIFE_TRY(dalloc(phi, &phi->part_u2, phi->red_cap));
    LIFE_TRY(dalloc(phi, &phi->counter2, 4));
    LIFE_TRY(dalloc(phi, &phi->ybound, 4));
    LIFE_CUDA(cudaMemsetAsync(phi->red.counter, 0, 16, st));
    LIFE_CUDA(cudaMemsetAsync(phi->counter2, 0, 16, st));
    LIFE_CUDA(cudaStreamSynchronize(st));
    setup_mark(st, "finish");
    phi->sort_ms = std::chrono::duration<double, std::milli>(
                       std::chrono::steady_clock::now() - t0).count();
    guard.p = nullptr;
    *out = phi;
    return ok();
}

int life_phi_create(const life_dims *dims, const uint32_t *atoms,
                    const uint32_t *voxels, const uint32_t *fibers,
                    const double *values, const double *dict, uint32_t flags,
                    void *stream, life_phi **out, int64_t *bad_position)
{
    return create_impl(dims, atoms, voxels, fibers, values, dict, flags,
                       static_cast<cudaStream_t>(stream), out, bad_position);
}

static void destroy_impl(life_phi *phi)
{
    cudaDeviceSynchronize();
    for (void *p : phi->allocs) dev_free(p);
    delete phi;
}

int life_copy_h2d(void *dst_dev, const void *src_host, int64_t bytes, void *stream)
{
    if ((!dst_dev || !src_host) && bytes > 0) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (bytes < 0) return fail(LIFE_ERR_INVALID_ARGUMENT, "negative size");
    LIFE_TRY(h2d_staged(dst_dev, src_host, (size_t)bytes, static_cast<cudaStream_t>(stream)));
    return ok();
}

int life_copy_h2d_f32(float *dst_dev, const double *src_host, int64_t count, void *stream)
{
    if ((!dst_dev || !src_host) && count > 0) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    if (count < 0) return fail(LIFE_ERR_INVALID_ARGUMENT, "negative size");
    if (count > 0 && count * 4 < (4 << 20)) {  // small: round on the host, one copy
        std::vector<float> tmp((size_t)count);
        for (int64_t i = 0; i < count; ++i) tmp[i] = (float)src_host[i];
        LIFE_CUDA(cudaMemcpyAsync(dst_dev, tmp.data(), (size_t)count * 4, cudaMemcpyHostToDevice,
                                  static_cast<cudaStream_t>(stream)));
        LIFE_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        return ok();
    }
    LIFE_TRY(h2d_staged_cvt(dst_dev, src_host, (size_t)count * 4, 1, static_cast<cudaStream_t>(stream)));
    return ok();
}

int life_phi_destroy(life_phi *phi)
{
    if (phi) destroy_impl(phi);
    return ok();
}

int life_release_cached_memory(void)
{
    cudaDeviceSynchronize();
    BlockCache &c = bcache();
    std::lock_guard<std::mutex> lock(c.mu);
    const size_t keep = c.cap;
    c.cap = 0;
    trim_locked(c, 0);
    c.cap = keep;
    return ok();
}

int life_cached_memory_bytes(int64_t *bytes)
{
    if (!bytes) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    BlockCache &c = bcache();
    std::lock_guard<std::mutex> lock(c.mu);
    *bytes = (int64_t)c.cached;
    return ok();
}

int life_phi_set_fix_bounds(life_phi *phi, double vmax, double dmax, int64_t fmax_nnz)
{
    if (!phi) return fail(LIFE_ERR_INVALID_ARGUMENT, "null handle");
    if (!(vmax >= 0.0) || !(dmax >= 0.0) || fmax_nnz < 1)
        return fail(LIFE_ERR_CONFIG_INVALID, "fixed-point bounds must be positive");
    // never tighter than the handle's own data (the sum must not overflow)
    phi->vmax = std::max(phi->vmax, vmax);
    phi->dmax = std::max(phi->dmax, dmax);
    phi->fmax_nnz = std::max<int64_t>(phi->fmax_nnz, fmax_nnz);
    return ok();
}

int life_phi_get_fix_bounds(const life_phi *phi, double *vmax, double *dmax, int64_t *fmax_nnz)
{
    if (!phi || !vmax || !dmax || !fmax_nnz) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    *vmax = phi->vmax;
    *dmax = phi->dmax;
    *fmax_nnz = phi->fmax_nnz;
    return ok();
}

int life_phi_get_info(const life_phi *phi, life_phi_info *info)
{
    if (!phi || !info) return fail(LIFE_ERR_INVALID_ARGUMENT, "null argument");
    info->dims = phi->dims;
    info->atom_groups = phi->has_bin ? -2 : phi->G;
    info->atoms_per_group = phi->ag;
    info->n_warps = phi->W;
    info->has_exact = phi->has_exact ? 1 : 0;
    info->n_voxel_runs = phi->n_voxel_runs;
    info->n_fiber_runs = phi->n_fiber_runs;
    info->max_fiber_run = phi->max_fiber_run;
    info->max_voxel_run = phi->max_voxel_run;
    info->device_bytes = phi->device_bytes;
    info->sort_ms = phi->sort_ms;
    info->tensor_ops = phi->has_bin ? 3 : 0;
    info->reserved = 0;
    return ok();
}

}  // extern "C"
