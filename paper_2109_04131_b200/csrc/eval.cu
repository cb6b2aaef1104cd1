// eval.cu — K11 evaluation of the approximant at test points (usfft_eval, include/usfft.h).
//
// U[g][q] = Re sum_k C[g][k] e^{2 pi i k.y_q} = sum_k Cre[g][k] cos(2 pi k.y_q) - Cim[g][k] sin(2 pi k.y_q)
// (eq. eval_formula P:468-470 with the identity periodization of the periodic model P:945-949).
// This is a real GEMM [G x 2|I|] . [2|I| x n] whose right operand comes from the sparse integer
// frequencies (k.y reduced mod 1, then sincospi): on the fp64 tensor pipe (DMMA m8n8k4) below.
#include <cstdlib>

#include "common.cuh"

namespace usfft {

constexpr int EV_TG = 64, EV_TQ = 64, EV_TK = 16;

// usfft_eval_err: per-tile partial sums (|.|, |.|^2, max) of |Uref - u| over the tile's 64 points,
// reduced in a fixed order; k_eval_err_reduce then adds the tiles of every node in tile order
// (P:885-891).
__global__ void k_eval_err_reduce(int64_t G, int64_t ntile, int64_t n, const double *__restrict__ part,
                                  double *__restrict__ err) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
        double s1 = 0.0, s2 = 0.0, mx = 0.0;
        for (int64_t t = 0; t < ntile; ++t) {
            const double *pp = part + (g * ntile + t) * 3;
            s1 += pp[0];
            s2 += pp[1];
            mx = fmax(mx, pp[2]);
        }
        err[g * 3 + 0] = s1 / (double)n;
        err[g * 3 + 1] = sqrt(s2 / (double)n);
        err[g * 3 + 2] = mx;
    }
}

// usfft_eval on the fp64 tensor pipe (DMMA, mma.sync m8n8k4 f64): the same product written as
// U = [Cre | -Cim] . [cos ; sin] with K = 2 x 12 per chunk.  8 warps per 128 x 64 tile (the
// phases of a chunk, d FMAs and a sincospi each, serve 128 nodes); warp (wg, wq) owns rows
// 64 wg .. +64 and columns 16 wq .. +16 as 8 x 2 tiles of 8 x 8.
// Fragments (PTX m8n8k4 .f64): A a0 = A[lane/4][lane%4], B b0 = B[lane%4][lane/4],
// C/D {d0, d1} = C[lane/4][2 (lane%4) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// The right operand once per call: E[0][k][q] = cos(2 pi k.y_q), E[1][k][q] = sin(2 pi k.y_q), with
// k.y_q reduced mod 1 before sincospi exactly as in the tile kernels (bit-identical values).  The
// DMMA kernels then stream E tiles instead of regenerating them for every row tile.
__global__ void k_phases(int32_t d, const int16_t *__restrict__ I, int64_t nI, const double *__restrict__ Y,
                         int64_t n, double *__restrict__ E) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t k = blockIdx.y;
    if (q >= n) return;
    double ph = 0.0;
    for (int j = 0; j < d; ++j) ph += (double)I[k * d + j] * Y[(int64_t)j * n + q];
    double c, sv;
    sincospi(2.0 * (ph - rint(ph)), &sv, &c);
    E[k * n + q] = c;
    E[(nI + k) * n + q] = sv;
}

__global__ void __launch_bounds__(256)
k_eval_mma(int32_t d, const int16_t *__restrict__ I, int64_t nI, const double2 *__restrict__ C,
           int64_t G, const double *__restrict__ Y, int64_t n, double *__restrict__ U,
           const double *__restrict__ E) {
    constexpr int TK = 12, K2 = 2 * TK, TG = 128, WT = TG / 16;      // WT row tiles per warp
    __shared__ double As[TG][K2 + 1];                     // [g][k]: Cre (k < TK), -Cim (k >= TK)
    __shared__ double Bs[K2][EV_TQ + 1];                  // [k][q]: cos (k < TK), sin (k >= TK)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wg = warp >> 2, wq = warp & 3;
    // with precomputed phases the row tiles of one column tile are neighbours in the grid (x), so
    // its E tile is read from L2 once for all of them
    const int64_t g0 = (int64_t)(E ? blockIdx.x : blockIdx.y) * TG, q0 = (int64_t)(E ? blockIdx.y : blockIdx.x) * EV_TQ;
    double acc[WT][2][2] = {};
    for (int64_t k0 = 0; k0 < nI; k0 += TK) {
        for (int e = threadIdx.x; e < TK * TG; e += blockDim.x) {
            const int kk = e / TG, gg = e % TG;
            double2 v = make_double2(0.0, 0.0);
            if (k0 + kk < nI && g0 + gg < G) v = C[(g0 + gg) * nI + k0 + kk];
            As[gg][kk] = v.x;
            As[gg][TK + kk] = -v.y;
        }
        for (int e = threadIdx.x; e < TK * EV_TQ; e += blockDim.x) {
            const int kk = e / EV_TQ, qq = e % EV_TQ;
            double c = 0.0, sv = 0.0;
            if (k0 + kk < nI && q0 + qq < n) {
                if (E) {
                    c = __ldg(E + (k0 + kk) * n + q0 + qq);
                    sv = __ldg(E + (nI + k0 + kk) * n + q0 + qq);
                } else {
                    double ph = 0.0;
                    for (int j = 0; j < d; ++j) ph += (double)I[(k0 + kk) * d + j] * Y[(int64_t)j * n + q0 + qq];
                    sincospi(2.0 * (ph - rint(ph)), &sv, &c);
                }
            }
            Bs[kk][qq] = c;
            Bs[TK + kk][qq] = sv;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < K2; k += 4) {
            double a[WT], b[2];
#pragma unroll
            for (int t = 0; t < WT; ++t) a[t] = As[8 * WT * wg + 8 * t + (lane >> 2)][k + (lane & 3)];
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) b[u2] = Bs[k + (lane & 3)][16 * wq + 8 * u2 + (lane >> 2)];
#pragma unroll
            for (int t = 0; t < WT; ++t)
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2) dmma_8x8x4(acc[t][u2][0], acc[t][u2][1], a[t], b[u2]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < WT; ++t) {
        const int64_t g = g0 + 8 * WT * wg + 8 * t + (lane >> 2);
        if (g >= G) continue;
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t q = q0 + 16 * wq + 8 * u2 + 2 * (lane & 3) + h;
                if (q < n) U[g * n + q] = acc[t][u2][h];
            }
    }
}

// The accuracy metric on the fp64 tensor pipe: the same DMMA product as k_eval_mma for the real
// part with A = [Cre | -Cim] and B = [cos; sin], and for the imaginary part with the same A and
// B' = [sin; -cos] (read from the same staged phases), then |Uref - (re + i im)| per element and
// per-row partial sums (mean, mean square, max) over the CTA's 64 columns in a fixed order, the
// layout k_eval_err_reduce reads.
__global__ void __launch_bounds__(256)
k_eval_err_mma(int32_t d, const int16_t *__restrict__ I, int64_t nI, const double2 *__restrict__ C,
               int64_t G, const double *__restrict__ Y, int64_t n, const double *__restrict__ Uref,
               double *__restrict__ part, const double *__restrict__ E) {
    constexpr int TK = 12, K2 = 2 * TK, TG = 64, WT = TG / 16;
    __shared__ double As[TG][K2 + 1];                     // [g][k]: Cre (k < TK), -Cim (k >= TK)
    __shared__ double Bs[K2][EV_TQ + 1];                  // [k][q]: cos (k < TK), sin (k >= TK)
    __shared__ double red[TG][4][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wg = warp >> 2, wq = warp & 3;
    const int64_t ti = E ? blockIdx.y : blockIdx.x, ntile = E ? gridDim.y : gridDim.x;   // column tile
    const int64_t g0 = (int64_t)(E ? blockIdx.x : blockIdx.y) * TG, q0 = ti * EV_TQ;
    double are[WT][2][2] = {}, aim[WT][2][2] = {};
    for (int64_t k0 = 0; k0 < nI; k0 += TK) {
        for (int e = threadIdx.x; e < TK * TG; e += blockDim.x) {
            const int kk = e / TG, gg = e % TG;
            double2 v = make_double2(0.0, 0.0);
            if (k0 + kk < nI && g0 + gg < G) v = C[(g0 + gg) * nI + k0 + kk];
            As[gg][kk] = v.x;
            As[gg][TK + kk] = -v.y;
        }
        for (int e = threadIdx.x; e < TK * EV_TQ; e += blockDim.x) {
            const int kk = e / EV_TQ, qq = e % EV_TQ;
            double c = 0.0, sv = 0.0;
            if (k0 + kk < nI && q0 + qq < n) {
                if (E) {
                    c = __ldg(E + (k0 + kk) * n + q0 + qq);
                    sv = __ldg(E + (nI + k0 + kk) * n + q0 + qq);
                } else {
                    double ph = 0.0;
                    for (int j = 0; j < d; ++j) ph += (double)I[(k0 + kk) * d + j] * Y[(int64_t)j * n + q0 + qq];
                    sincospi(2.0 * (ph - rint(ph)), &sv, &c);
                }
            }
            Bs[kk][qq] = c;
            Bs[TK + kk][qq] = sv;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < K2; k += 4) {
            double a[WT], b[2], bi[2];
#pragma unroll
            for (int t = 0; t < WT; ++t) a[t] = As[8 * WT * wg + 8 * t + (lane >> 2)][k + (lane & 3)];
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
                const int col = 16 * wq + 8 * u2 + (lane >> 2);
                b[u2] = Bs[k + (lane & 3)][col];
                bi[u2] = k < TK ? Bs[TK + k + (lane & 3)][col] : -Bs[k - TK + (lane & 3)][col];
            }
#pragma unroll
            for (int t = 0; t < WT; ++t)
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2) {
                    dmma_8x8x4(are[t][u2][0], are[t][u2][1], a[t], b[u2]);
                    dmma_8x8x4(aim[t][u2][0], aim[t][u2][1], a[t], bi[u2]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < WT; ++t) {
        const int r = 8 * WT * wg + 8 * t + (lane >> 2);
        const int64_t g = g0 + r;
        double s1 = 0.0, s2s = 0.0, mx = 0.0;
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t q = q0 + 16 * wq + 8 * u2 + 2 * (lane & 3) + h;
                if (g < G && q < n) {
                    const double m = hypot(Uref[g * n + q] - are[t][u2][h], -aim[t][u2][h]);
                    s1 += m;
                    s2s = fma(m, m, s2s);
                    mx = fmax(mx, m);
                }
            }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {           // the 4 lanes of one row
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2s += __shfl_xor_sync(0xffffffffu, s2s, o);
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((lane & 3) == 0) {
            red[r][wq][0] = s1;
            red[r][wq][1] = s2s;
            red[r][wq][2] = mx;
        }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < TG; r += blockDim.x) {             // the 4 column groups, in order
        const int64_t g = g0 + r;
        if (g >= G) continue;
        double *pp = part + (g * ntile + ti) * 3;
        pp[0] = ((red[r][0][0] + red[r][1][0]) + red[r][2][0]) + red[r][3][0];
        pp[1] = ((red[r][0][1] + red[r][1][1]) + red[r][2][1]) + red[r][3][1];
        pp[2] = fmax(fmax(red[r][0][2], red[r][1][2]), fmax(red[r][2][2], red[r][3][2]));
    }
}

}  // namespace usfft

using namespace usfft;

namespace {
// The phase matrix E [2][nI][n] in the second ctx workspace when it fits (<= 4 GiB) and the
// column tiles fit the grid's y dimension; NULL: the kernels generate phases per tile.
const double *phase_matrix(usfft_ctx *c, int32_t d, const int16_t *I, int64_t nI, const double *Y, int64_t n,
                           usfft_status *st) {
    *st = USFFT_OK;
    if (nI == 0) return nullptr;
    const size_t bytes = sizeof(double) * 2 * (size_t)nI * (size_t)n;
    if (bytes > (size_t(4) << 30) || (n + EV_TQ - 1) / EV_TQ > 65535 || nI > 65535) return nullptr;
    if ((*st = ensure(c, &c->ws2, &c->ws2_size, bytes))) return nullptr;
    double *E = static_cast<double *>(c->ws2);
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)nI);
    k_phases<<<grid, 256, 0, c->stream>>>(d, I, nI, Y, n, E);
    if (cudaPeekAtLastError() != cudaSuccess) {
        *st = fail(c, USFFT_ECUDA, "k_phases launch: %s", cudaGetErrorString(cudaGetLastError()));
        return nullptr;
    }
    return E;
}
}  // namespace

extern "C" usfft_status usfft_eval_err(usfft_ctx *c, int32_t d, const int16_t *I, int64_t nI,
                                       const double *C, int64_t G, const double *Y, int64_t n,
                                       const double *Uref, double *err) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, d >= 1 && d <= kMaxD && nI >= 0 && G >= 0 && n >= 1, "bad sizes");
    if (G == 0) return USFFT_OK;
    USFFT_REQUIRE(c, Y && Uref && err, "Y / Uref / err NULL");
    USFFT_REQUIRE(c, nI == 0 || (I && C), "I / C NULL");
    const int64_t ntile = (n + EV_TQ - 1) / EV_TQ;
    USFFT_REQUIRE(c, ntile <= 0x7fffffff && (G + EV_TG - 1) / EV_TG <= 65535, "grid too large");
    usfft_status s = ensure(c, &c->ws, &c->ws_size, sizeof(double) * 3 * (size_t)(G * ntile));
    if (s) return s;
    double *part = static_cast<double *>(c->ws);
    dim3 grid((unsigned)ntile, (unsigned)((G + EV_TG - 1) / EV_TG));
    {
        usfft_status st = USFFT_OK;
        const double *E = phase_matrix(c, d, I, nI, Y, n, &st);
        if (st) return st;
        const dim3 gr = E ? dim3((unsigned)((G + EV_TG - 1) / EV_TG), (unsigned)ntile) : grid;
        k_eval_err_mma<<<gr, 256, 0, c->stream>>>(d, I, nI, reinterpret_cast<const double2 *>(C), G, Y, n, Uref,
                                                   part, E);
    }
    USFFT_CHECK_LAUNCH(c);
    k_eval_err_reduce<<<grid1d(G, 128), 128, 0, c->stream>>>(G, ntile, n, part, err);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

extern "C" usfft_status usfft_eval(usfft_ctx *c, int32_t d, const int16_t *I, int64_t nI,
                                   const double *C, int64_t G, const double *Y, int64_t n,
                                   double *U) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, d >= 1 && d <= kMaxD && nI >= 0 && G >= 0 && n >= 0, "bad sizes");
    if (G == 0 || n == 0) return USFFT_OK;
    USFFT_REQUIRE(c, U != nullptr && Y != nullptr, "U / Y NULL");
    USFFT_REQUIRE(c, nI == 0 || (I && C), "I / C NULL");
    USFFT_REQUIRE(c, (n + EV_TQ - 1) / EV_TQ <= 0x7fffffff && (G + EV_TG - 1) / EV_TG <= 65535, "grid too large");
    dim3 grid((unsigned)((n + EV_TQ - 1) / EV_TQ), (unsigned)((G + EV_TG - 1) / EV_TG));
    {
        usfft_status st = USFFT_OK;
        const double *E = phase_matrix(c, d, I, nI, Y, n, &st);
        if (st) return st;
        const unsigned nq = (unsigned)((n + EV_TQ - 1) / EV_TQ), ng = (unsigned)((G + 127) / 128);
        const dim3 gm = E ? dim3(ng, nq) : dim3(nq, ng);
        k_eval_mma<<<gm, 256, 0, c->stream>>>(d, I, nI, reinterpret_cast<const double2 *>(C), G, Y, n, U, E);
    }
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}
