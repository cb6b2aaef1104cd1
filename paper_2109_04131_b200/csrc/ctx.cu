// ctx.cu — context lifetime and error reporting of the C-ABI (include/usfft.h).
#include <algorithm>

#include "common.cuh"

extern "C" usfft_status usfft_init(usfft_ctx **out, int device, void *stream, int rank, int nranks,
                                   const void *comm_id, int loopback) {
    if (!out) return USFFT_EINVAL;
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !comm_id)) return USFFT_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return USFFT_EINVAL;
    }
    usfft_ctx *c = new usfft_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return USFFT_ECUDA;
    }
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    c->sm_count = v > 0 ? v : 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    c->smem_optin = v > 0 ? (size_t)v : 48 * 1024;
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device);
    c->l2_bytes = v > 0 ? (size_t)v : (size_t)64 << 20;
    if (cudaMalloc(&c->dscal, 4096) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return USFFT_ENOMEM;
    }
    cudaMemset(c->dscal, 0, 4096);
    if (usfft_status s = usfft::comm_create(c, rank, nranks, comm_id, loopback)) {
        usfft::comm_destroy(c);
        cudaFree(c->dscal);
        delete c;
        return s;
    }
    *out = c;
    return USFFT_OK;
}

extern "C" usfft_status usfft_set_stream(usfft_ctx *c, void *stream) {
    if (!c) return USFFT_EINVAL;
    c->stream = static_cast<cudaStream_t>(stream);
    return USFFT_OK;
}

extern "C" usfft_status usfft_finalize(usfft_ctx *c) {
    if (!c) return USFFT_EINVAL;
    usfft::DeviceGuard guard(c->device);
    cudaStreamSynchronize(c->stream);
    usfft::comm_destroy(c);
    for (auto &kv : c->twiddles) cudaFree(kv.second);
    for (auto &kv : c->sintab) cudaFree(kv.second);
    for (auto &kv : c->rhstab) cudaFree(kv.second);
    for (auto &kv : c->rader) {
        cudaFree(kv.second.tw);
        cudaFree(kv.second.perm);
        cudaFree(kv.second.outidx);
        cudaFree(kv.second.bf);
    }
    if (c->ws) cudaFree(c->ws);
    if (c->ws2) cudaFree(c->ws2);
    if (c->dscal) cudaFree(c->dscal);
    delete c;
    return USFFT_OK;
}

extern "C" const char *usfft_last_error(const usfft_ctx *c) {
    if (!c) return "null ctx";
    return c->err.c_str();
}

extern "C" int64_t usfft_launch_count(const usfft_ctx *c) { return c ? c->launches : -1; }

// Device bytes the calls of one round allocate (caller-owned buffers not included): the ctx
// workspace they grow to, the per-M tables and, with nranks > 1, nothing more (usfft_transpose
// writes into the caller's slab buffer).  An upper bound from the sizes alone, no device work.
extern "C" usfft_status usfft_workspace_query(usfft_ctx *c, const usfft_round_desc *r, size_t *bytes) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, r && bytes, "NULL argument");
    USFFT_REQUIRE(c, r->n >= 2 && r->M >= 2 && r->L >= 1 && r->nJ >= 0 && r->s_tilde >= 1 && r->d >= 1, "bad round");
    const int P = usfft::comm_size(c);
    const int64_t G = (int64_t)(r->n - 1) * (r->n - 1), Gl = (G + P - 1) / P;
    size_t b = 0;
    b += 16 * (size_t)r->M;                                   // twiddles e^{-2 pi i m/M}
    b += (16 + 16 + 4 + 4) * (size_t)r->M;                    // Rader tables
    b += 8 * 2 * (size_t)r->d * (3 * (size_t)r->n + 1);       // psi factor tables
    b += 8 * (size_t)G;                                       // load table (f != x2)
    // PCG scratch of the scratch-slab kernel (n = 8 only; the others keep samples on chip)
    if (r->n == 8) b += 8 * (size_t)c->sm_count * 2 * 4096;
    // resolve / eval partials: bounded by the key chunk of the streamed selection
    b += 8 * (size_t)Gl * (size_t)std::min<int64_t>(r->nJ, 1 << 16);
    *bytes = b + 4096;
    return USFFT_OK;
}
