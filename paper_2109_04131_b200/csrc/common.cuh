// common.cuh — ctx, error plumbing and deterministic block reductions shared by the usFFT
// kernels (sm_100a).  Nothing here is shared with oracle/ (see DESIGN.md §1).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "../../include/usfft.h"

// Bounds-checked build (tools/bounds_check.sh: -DUSFFT_BOUNDS): every computed shared-memory and
// DSMEM index of the on-chip kernels is asserted in range (compute-sanitizer is closed on this
// pool).  The product build compiles the checks out.
#ifdef USFFT_BOUNDS
#include <cassert>
#define UB_CHECK(cond) assert(cond)
#else
#define UB_CHECK(cond) ((void)0)
#endif

namespace usfft {
// Rader tables of one prime lattice size (fft.cu), owned by the ctx
struct RaderPlan {
    int64_t M = 0, N = 0;
    int nstage = 0;
    int radix[32] = {0};
    double2 *tw = nullptr;      // [N]  e^{-2 pi i k / N}
    int32_t *perm = nullptr;    // [N]  g^p mod M
    int32_t *outidx = nullptr;  // [N]  g^{-q} mod M
    double2 *bf = nullptr;      // [N]  FFT_N(b) / N
};
}  // namespace usfft

struct usfft_comm;                                           // comm.cu: NCCL communicator / loopback hub

struct usfft_ctx {
    int device = 0;
    usfft_comm *comm = nullptr;                              // nranks > 1 only
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    size_t smem_optin = 0;
    size_t l2_bytes = 0;                                     // L2 cache size of the device
    bool sticky = false;
    std::string err;
    int64_t launches = 0;
    // general device workspace — grows on demand
    void *ws = nullptr;
    size_t ws_size = 0;
    void *ws2 = nullptr;                                          // second workspace (eval phases)
    size_t ws2_size = 0;
    // small device scalar area (counters, maxima): 4 KB allocated at init
    void *dscal = nullptr;
    // cached tables
    std::map<int64_t, double2 *> twiddles;                  // M -> e^{-2 pi i m/M}, m < M
    std::map<std::tuple<int, int, int>, double *> sintab;    // (n, d, psi) -> psi factor tables
    std::map<std::pair<int, int>, double *> rhstab;          // (n, f_kind) -> centroid loads b
    std::map<int64_t, usfft::RaderPlan> rader;               // M -> Rader tables (M = 0: not Rader-able)
    // resident blocks per SM per (kernel, threads, smem): the query costs ~10 us per call
    std::map<std::pair<const void *, size_t>, int> occupancy;
};

namespace usfft {

// Small host arrays travel as kernel parameters (<= 32 KB parameter space on sm_70+, CUDA 12.1+),
// so no call needs a host sync to stage them.
constexpr int kMaxZ = 2048;      // L * t entries of z
constexpr int kMaxD = 64;        // parameter dimension d
constexpr int kMaxSlab = 64;     // exchange slabs (ranks)

struct LatParams {
    int32_t d, t, line_axis, L;
    int64_t M;
    int32_t z[kMaxZ];            // z < M <= 2^26: int32 halves the kernel-parameter copy per launch
    double shift[kMaxD];
};


inline usfft_status fail(usfft_ctx *c, usfft_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
    if (s == USFFT_ECUDA) c->sticky = true;
    return s;
}

#define USFFT_CUDA(c, expr)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return usfft::fail((c), USFFT_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,   \
                               cudaGetErrorString(e_));                                       \
    } while (0)

#define USFFT_CHECK_LAUNCH(c)                                                                 \
    do {                                                                                      \
        (c)->launches++;                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess)                                                                \
            return usfft::fail((c), USFFT_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__,      \
                               cudaGetErrorString(e_));                                       \
    } while (0)

#define USFFT_REQUIRE(c, cond, ...)                                                           \
    do {                                                                                      \
        if (!(cond)) return usfft::fail((c), USFFT_EINVAL, __VA_ARGS__);                      \
    } while (0)

// Every entry point: validate the ctx and make its device current for the call (restored on
// return), so contexts on different devices can be used from one thread.
struct DeviceGuard {
    int prev = -1, dev;
    explicit DeviceGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

// NVTX range per C-ABI call (header-only NVTX 3; a no-op unless a tool such as nsys / ncu
// --nvtx is attached): the range is named after the entry point and spans its host side
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

#define USFFT_ENTER(c)                                                                        \
    usfft::NvtxRange usfft_nvtx_range_(__func__);                                             \
    if (!(c)) return USFFT_EINVAL;                                                            \
    if ((c)->sticky) return USFFT_ECUDA;                                                      \
    (c)->err.clear();                                                                         \
    usfft::DeviceGuard usfft_device_guard_((c)->device)

// Grow-only device buffers.  Growth synchronises the stream first (buffers may be in use).
inline usfft_status ensure(usfft_ctx *c, void **buf, size_t *size, size_t need) {
    if (need <= *size) return USFFT_OK;
    size_t want = need + need / 4 + 4096;
    if (*buf) {
        USFFT_CUDA(c, cudaStreamSynchronize(c->stream));
        USFFT_CUDA(c, cudaFree(*buf));
        *buf = nullptr;
        *size = 0;
    }
    if (cudaMalloc(buf, want) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, USFFT_ENOMEM, "cudaMalloc(%zu) failed", want);
    }
    *size = want;
    return USFFT_OK;
}

// Raise the kernel's dynamic shared-memory limit to smem (once per value) and return its
// resident blocks per SM for (threads, smem), cached in the ctx.
// The attribute is a per-(device, function) setting shared by every ctx of the process, so its
// record is process-wide and only ever raised.
inline std::mutex &smem_attr_mutex() {
    static std::mutex m;
    return m;
}
inline std::map<std::pair<int, const void *>, size_t> &smem_attr_table() {
    static std::map<std::pair<int, const void *>, size_t> t;
    return t;
}

template <class K>
inline usfft_status kernel_fit(usfft_ctx *c, K kern, int threads, size_t smem, int *per_sm) {
    const void *f = reinterpret_cast<const void *>(kern);
    {
        std::lock_guard<std::mutex> lock(smem_attr_mutex());
        size_t &attr = smem_attr_table()[std::make_pair(c->device, f)];
        if (smem > attr) {
            USFFT_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr = smem;
        }
    }
    if (per_sm) {
        const auto key = std::make_pair(f, smem * 2048 + (size_t)threads);
        auto it = c->occupancy.find(key);
        if (it == c->occupancy.end()) {
            int ps = 0;
            USFFT_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, threads, smem));
            it = c->occupancy.emplace(key, ps).first;
        }
        *per_sm = it->second;
    }
    return USFFT_OK;
}

// the in-library collectives (comm.cu); every rank calls them in the same order
usfft_status comm_create(usfft_ctx *c, int rank, int nranks, const void *id, int loopback);
void comm_destroy(usfft_ctx *c);
int comm_size(const usfft_ctx *c);
usfft_status comm_alltoallv(usfft_ctx *c, const double *send, const int64_t *scount, const int64_t *sdispl,
                            double *recv, const int64_t *rcount, const int64_t *rdispl);
usfft_status comm_max_f64(usfft_ctx *c, double *buf, int64_t count);
usfft_status comm_sum_i32(usfft_ctx *c, int32_t *buf, int64_t count);

inline unsigned grid1d(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 0x7fffffff) g = 0x7fffffff;
    return static_cast<unsigned>(g);
}

}  // namespace usfft

// ---------------------------------------------------------------------------------------------
// Deterministic block reductions: each thread contributes one partial; the tree is fixed
// (xor-butterfly inside each warp, then warp partials summed in warp order), so the result
// depends only on blockDim and the partials, never on scheduling.
// ---------------------------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *scratch /* [32*NV] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) scratch[k * 32 + warp] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = 0.0;
        for (int w = 0; w < nwarp; ++w) s += scratch[k * 32 + w];
        v[k] = s;
    }
    __syncthreads();
}

// v_l = F[b]/M of a real-input spectrum stored for bins 0..M/2 (mirror bins conjugated, Z17/Z18)
__device__ __forceinline__ double2 spec_value(const double2 *__restrict__ row, int64_t M, int64_t b) {
    const int64_t Mh = M / 2 + 1;
    const double Md = (double)M;
    if (b < Mh) {
        const double2 v = row[b];
        return make_double2(v.x / Md, v.y / Md);
    }
    const double2 v = row[M - b];
    return make_double2(v.x / Md, -v.y / Md);
}

// Exclusive block scan of one int per thread (fixed order); *total receives the block sum.
__device__ __forceinline__ int block_exscan(int v, int *sh /* [33] */, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int w = 0; w < nwarp; ++w) {
            int t = sh[w];
            sh[w] = run;
            run += t;
        }
        sh[32] = run;
    }
    __syncthreads();
    const int ex = sh[warp] + x - v;
    *total = sh[32];
    __syncthreads();
    return ex;
}
