// lattice.cu — K1 lattice nodes, K2 candidate index maps + injectivity, candidate row gather.
// usfft_lattice (header: include/usfft.h; a2 + a3 of SURVEY §8(a)).
#include "lattice.cuh"

namespace usfft {

// K1: nodes [d][nb] (sample fastest -> coalesced stores).
__global__ void k_nodes(const LatParams P, int64_t b0, int64_t nb, double *__restrict__ y) {
    const int64_t total = (int64_t)P.d * nb;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / nb);
        const int64_t bl = e - (int64_t)j * nb;
        y[e] = lattice_node(P, b0 + bl, j);
    }
}

// K2: b_l(k) = (k . z_l) mod M for k = (I_prev[a], kt[c]), j = a*n1 + c (Z10).
// Optional injectivity test: an M-bit occupancy bitset per lattice; a second hit of a bit
// marks the lattice as not reconstructing.
__global__ void k_bins(const LatParams P, const int16_t *__restrict__ I_prev, int64_t n_prev,
                       const int16_t *__restrict__ kt, int32_t n1, int32_t *__restrict__ bins,
                       unsigned int *__restrict__ bitset, int64_t words_per_lat,
                       int32_t *__restrict__ collide) {
    const int64_t nJ = n_prev * (int64_t)n1;
    const int64_t total = nJ * P.L;
    const int tp = P.t - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = e / nJ;
        const int64_t j = e - l * nJ;
        const int64_t a = j / n1;
        const int64_t cc = j - a * n1;
        const int32_t *z = P.z + l * P.t;
        int64_t s = (int64_t)kt[cc] * z[tp];
        for (int q = 0; q < tp; ++q) s += (int64_t)I_prev[a * tp + q] * z[q];
        int64_t b = s % P.M;
        if (b < 0) b += P.M;
        if (bins) bins[e] = (int32_t)b;
        if (bitset) {
            unsigned int bit = 1u << (b & 31);
            unsigned int old = atomicOr(bitset + l * words_per_lat + (b >> 5), bit);
            if (old & bit) collide[l] = 1;
        }
    }
}

__global__ void k_gather_rows(const int32_t *__restrict__ idx, int64_t n,
                              const int16_t *__restrict__ I_prev, int32_t t,
                              const int16_t *__restrict__ kt, int32_t n1,
                              int16_t *__restrict__ rows) {
    const int tp = t - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * t;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / t;
        const int c = (int)(e - q * t);
        const int64_t j = idx[q];
        const int64_t a = j / n1;
        rows[e] = (c < tp) ? I_prev[a * tp + c] : kt[j - a * n1];
    }
}

}  // namespace usfft

using namespace usfft;

extern "C" usfft_status usfft_lattice(usfft_ctx *c, const usfft_lattice_desc *lat, int64_t b0,
                                      int64_t nb, double *nodes, const int16_t *I_prev,
                                      int64_t n_prev, const int16_t *kt, int32_t n1,
                                      int32_t *bins, int32_t *injective) {
    USFFT_ENTER(c);
    static thread_local LatParams P;  // ~17 KB: filled on the host, passed as launch parameters
    usfft_status s = make_lat_params(c, lat, &P);
    if (s) return s;
    USFFT_REQUIRE(c, b0 >= 0 && nb >= 0 && b0 + nb <= (int64_t)P.L * P.M, "sample range out of [0, L*M)");
    const bool want_bins = bins != nullptr || injective != nullptr;
    if (want_bins) {
        USFFT_REQUIRE(c, kt != nullptr && n1 >= 1, "kt is NULL or n1 < 1");
        USFFT_REQUIRE(c, n_prev >= 1, "n_prev < 1");
        USFFT_REQUIRE(c, P.t == 1 || I_prev != nullptr, "I_prev is NULL with t > 1");
        USFFT_REQUIRE(c, n_prev * (int64_t)n1 <= 0x7fffffff, "|J| too large");
    }
    if (nodes && nb > 0) {
        k_nodes<<<grid1d((int64_t)P.d * nb, 256), 256, 0, c->stream>>>(P, b0, nb, nodes);
        USFFT_CHECK_LAUNCH(c);
    }
    if (!want_bins) return USFFT_OK;
    const int64_t nJ = n_prev * (int64_t)n1;
    unsigned int *bitset = nullptr;
    int32_t *collide = nullptr;
    const int64_t words = (P.M + 31) / 32;
    if (injective) {
        size_t need = (size_t)P.L * words * 4 + (size_t)P.L * 4 + 64;
        s = ensure(c, &c->ws, &c->ws_size, need);
        if (s) return s;
        bitset = static_cast<unsigned int *>(c->ws);
        collide = reinterpret_cast<int32_t *>(bitset + (size_t)P.L * words);
        USFFT_CUDA(c, cudaMemsetAsync(c->ws, 0, need, c->stream));
    }
    k_bins<<<grid1d(nJ * P.L, 256), 256, 0, c->stream>>>(P, I_prev, n_prev, kt, n1, bins, bitset,
                                                          words, collide);
    USFFT_CHECK_LAUNCH(c);
    if (injective) {
        USFFT_CUDA(c, cudaMemcpyAsync(injective, collide, sizeof(int32_t) * P.L,
                                      cudaMemcpyDeviceToHost, c->stream));
        USFFT_CUDA(c, cudaStreamSynchronize(c->stream));
        bool all = true;
        for (int l = 0; l < P.L; ++l) {
            injective[l] = injective[l] ? 0 : 1;
            all = all && injective[l];
        }
        if (!all) return fail(c, USFFT_ENOTRECON, "index map not injective on J_t");
    }
    return USFFT_OK;
}

extern "C" usfft_status usfft_gather_rows(usfft_ctx *c, const int32_t *idx, int64_t n,
                                          const int16_t *I_prev, int32_t t, const int16_t *kt,
                                          int32_t n1, int16_t *rows) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, n >= 0 && t >= 1 && n1 >= 1, "bad sizes");
    USFFT_REQUIRE(c, n == 0 || (idx && kt && rows && (t == 1 || I_prev)), "NULL pointer");
    if (n == 0) return USFFT_OK;
    k_gather_rows<<<grid1d(n * t, 256), 256, 0, c->stream>>>(idx, n, I_prev, t, kt, n1, rows);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}
