// ctx.cu — context lifetime and error reporting of the C-ABI (include/usfft.h).
#include "common.cuh"

extern "C" usfft_status usfft_init(usfft_ctx **out, int device, void *stream) {
    if (!out) return USFFT_EINVAL;
    *out = nullptr;
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
    if (cudaMalloc(&c->dscal, 4096) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return USFFT_ENOMEM;
    }
    cudaMemset(c->dscal, 0, 4096);
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
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
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
