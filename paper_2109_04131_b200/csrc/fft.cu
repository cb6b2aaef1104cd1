// fft.cu — K6 lattice DFT along the sample axis + K7 candidate gather / detection key.
// usfft_lattice_fft (include/usfft.h; a7 + a8 of SURVEY §8(a)).
//
// K6 (this version): direct DFT per (node, lattice) row staged in shared memory, the phase index
// (i*m) mod M carried as an exact integer, twiddles e^{-2 pi i m/M} from a per-M table built with
// sincospi.  Real input, bins 0..M/2 (Z17).
// K7: v_l(j,g) = F[g][l][b]/M with b = bins[l][j] (conjugated mirror bin for b > M/2, Z17/Z18),
// kappa_l = fl(fl(re*re) + fl(im*im)) (no FMA contraction, Z5), kappa_min = min over l (Z1);
// the max over (g, j) of kappa_min is accumulated with an integer atomicMax on the bit pattern
// (non-negative doubles order like uint64), so it is exact and order-independent.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

#ifndef USFFT_KEYS_TILED_ALWAYS
#define USFFT_KEYS_TILED_ALWAYS 0                           // tools/keys_crossover.py builds with 1
#endif

namespace usfft {

struct SlabParams {
    int32_t nslab;
    int64_t b0[kMaxSlab + 1];
};

__global__ void k_twiddles(int64_t M, double2 *__restrict__ tw) {
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < M;
         m += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincospi((double)(2 * m) / (double)M, &s, &c);
        tw[m] = make_double2(c, -s);                              // e^{-2 pi i m / M}
    }
}

__device__ __forceinline__ double sample_at(const double *__restrict__ u, const SlabParams &S,
                                            int64_t G_loc, int64_t g, int64_t b) {
    int p = 0;
    while (p + 1 < S.nslab && b >= S.b0[p + 1]) ++p;
    const int64_t w = S.b0[p + 1] - S.b0[p];
    return u[G_loc * S.b0[p] + g * w + (b - S.b0[p])];
}

// one CTA per row (g, l): F[g][l][m] = sum_i u[g][l*M+i] e^{-2 pi i (i m mod M)/M}, m <= M/2
__global__ void k_dft_direct(const double *__restrict__ u, const SlabParams S, int64_t G_loc,
                             int64_t M, int32_t L, const double2 *__restrict__ tw,
                             double2 *__restrict__ F) {
    extern __shared__ double sm[];
    double *xs = sm;                                             // [M]
    double2 *ts = reinterpret_cast<double2 *>(sm + ((M + 1) & ~int64_t(1)));   // [M]
    const int64_t row = blockIdx.x;
    const int64_t g = row / L, l = row - g * L;
    const int64_t Mh = M / 2 + 1;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
        xs[i] = sample_at(u, S, G_loc, g, l * M + i);
        ts[i] = tw[i];
    }
    __syncthreads();
    for (int64_t m = threadIdx.x; m < Mh; m += blockDim.x) {
        double re = 0.0, im = 0.0;
        int64_t idx = 0;
        for (int64_t i = 0; i < M; ++i) {
            const double2 w = ts[idx];
            re += xs[i] * w.x;
            im += xs[i] * w.y;
            idx += m;
            if (idx >= M) idx -= M;
        }
        F[row * Mh + m] = make_double2(re, im);
    }
}

// Direct lattice DFT at the bins in use (Step 3 with cover lattices beyond the FFT kernels):
// coef[g][idx[a]] = (1/M) sum_i u[g][i] e^{-2 pi i (i b_a mod M)/M} -- a [G x M] . [M x n] complex
// product with the right operand generated from the exact phase index; 64 x 64 output tiles,
// 16-sample chunks staged in shared memory, 4 x 4 register tiles per thread.
constexpr int DB_TG = 64, DB_TA = 64, DB_TI = 16;

__global__ void __launch_bounds__(256)
k_dft_bins(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int64_t M,
           const double2 *__restrict__ tw, const int32_t *__restrict__ bins,
           const int32_t *__restrict__ idx, int64_t n, double2 *__restrict__ coef, int64_t nI) {
    __shared__ double us[DB_TI][DB_TG + 1];
    __shared__ double2 ws[DB_TI][DB_TA + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t g0 = (int64_t)blockIdx.y * DB_TG, a0 = (int64_t)blockIdx.x * DB_TA;
    double are[4][4] = {}, aim[4][4] = {};
    for (int64_t i0 = 0; i0 < M; i0 += DB_TI) {
        for (int e = threadIdx.x; e < DB_TI * DB_TG; e += blockDim.x) {
            const int ii = e % DB_TI, gg = e / DB_TI;
            us[ii][gg] = (i0 + ii < M && g0 + gg < G_loc) ? sample_at(u, S, G_loc, g0 + gg, i0 + ii) : 0.0;
        }
        for (int e = threadIdx.x; e < DB_TI * DB_TA; e += blockDim.x) {
            const int ii = e / DB_TA, aa = e % DB_TA;
            double2 w = make_double2(0.0, 0.0);
            if (i0 + ii < M && a0 + aa < n) w = tw[((i0 + ii) * (int64_t)bins[a0 + aa]) % M];
            ws[ii][aa] = w;
        }
        __syncthreads();
#pragma unroll 4
        for (int ii = 0; ii < DB_TI; ++ii) {
            double uv[4];
            double2 wv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                uv[r] = us[ii][ty * 4 + r];
                wv[r] = ws[ii][tx * 4 + r];
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    are[r][q] = fma(uv[r], wv[q].x, are[r][q]);
                    aim[r][q] = fma(uv[r], wv[q].y, aim[r][q]);
                }
        }
        __syncthreads();
    }
    const double Md = (double)M;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t g = g0 + ty * 4 + r;
        if (g >= G_loc) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t a = a0 + tx * 4 + q;
            if (a < n) coef[g * nI + idx[a]] = make_double2(are[r][q] / Md, aim[r][q] / Md);
        }
    }
}

// Keys with the bins tile shared by a group of nodes: CTA (candidate tile, node group) stages the
// tile's L bins rows once (coalesced) and then, node by node, gathers the node's L spectrum values
// per candidate straight from L1/L2 (L independent loads in flight per thread).  The bins are read
// G/KG_NODES times instead of G times, and no per-node spectrum staging sits on the critical path.
constexpr int KG_NODES = 8;

__global__ void __launch_bounds__(256)
k_kappa_grouped(const double2 *__restrict__ F, const int32_t *__restrict__ bins, int64_t ldb, int64_t nJ,
                int64_t M, int32_t L, int64_t G, double *__restrict__ kmin, int64_t ldk,
                unsigned long long *__restrict__ kmax, const double *__restrict__ tau) {
    extern __shared__ int32_t sbins[];                 // [L][256]
    __shared__ unsigned long long wmax[8];
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t g0 = (int64_t)blockIdx.y * KG_NODES;
    const int64_t Mh = M / 2 + 1;
    const double inv_m = 1.0 / (double)M;
#pragma unroll 4
    for (int l = 0; l < L; ++l) sbins[l * 256 + threadIdx.x] = j < nJ ? __ldg(bins + (int64_t)l * ldb + j) : 0;
    __syncthreads();
    unsigned long long best = 0ull;
    if (j < nJ) {
        for (int q = 0; q < KG_NODES && g0 + q < G; ++q) {
            const double2 *src = F + (g0 + q) * L * Mh;
            double km = 0.0;
#pragma unroll 8
            for (int l = 0; l < L; ++l) {
                const int b = sbins[l * 256 + threadIdx.x];
                const double2 f = __ldg(src + l * Mh + (b < (int)Mh ? b : (int)M - b));
                const double re = f.x * inv_m, im = f.y * inv_m;
                const double k = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
                km = (l == 0) ? k : fmin(km, k);
            }
            // streamed selection (Z29): a key <= the node's carry threshold can never enter
            kmin[(g0 + q) * ldk + j] = (tau && km <= tau[g0 + q]) ? 0.0 : km;
            const unsigned long long bits = (unsigned long long)__double_as_longlong(km);
            best = bits > best ? bits : best;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) best = wmax[w] > best ? wmax[w] : best;
        atomicMax(kmax, best);
    }
}

// K7 for |J| >> M (config 4's Step-2 rounds, |J| ~ 2e6 against M/2+1 ~ 1e3 bins): the candidates
// are the product set J = I_prev x kt (Z10, j = a n1 + c), so
//   bins[l][a n1 + c] = (bins[l][a n1] + bins[l][c] - bins[l][0]) mod M,
// and a (node, lattice) spectrum has only M/2+1 distinct values for ~|J| / (M/2) candidates each.
// One CTA per (node g, tile of KT = NT x KPT candidates): for every lattice the node's spectrum
// slice (M/2+1 complex) and the tile's bin terms are staged in shared memory (the next lattice's
// slice prefetched into registers meanwhile), each thread keeps the running min of its KPT
// candidates in registers.  The arithmetic per (g, j, l) and the min order over l are those of
// k_kappa_grouped, so the keys are bit-identical; the traffic is the spectra once per tile
// (G |J| L (M/2+1) 16 B / KT) instead of one 32-byte sector per (g, j, l) gather.
template <int NT, int KPT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
k_kappa_tiled(const double2 *__restrict__ F, const int32_t *__restrict__ bins, int64_t ldb, int64_t j0,
              int64_t nJ, int32_t n1, int32_t M, int32_t L, double *__restrict__ kmin, int64_t ldk,
              unsigned long long *__restrict__ kmax, const double *__restrict__ tau) {
    constexpr int KT = NT * KPT;
    const int Mh = M / 2 + 1;
    // [2][2M] keys |F/M|^2 of a slice: S[b] for every b = A + D in [0, 2M) (the bin b mod M,
    // folded to M - b above M/2: |F[M-m]| = |F[m]| for real samples), so a candidate's key is one load
    extern __shared__ double ssk[];
    const int AT = KT / n1 + 2;                          // a values a tile spans
    int32_t *sA = reinterpret_cast<int32_t *>(ssk + 4 * M);    // [2][AT]: bins[l][a n1]
    int32_t *sD = sA + 2 * AT;                                  // [2][n1]: bins[l][c] - bins[l][0] mod M
    __shared__ unsigned long long wmax[NT / 32];
    const int tid = threadIdx.x;
    const int64_t g = blockIdx.y;
    const int64_t t0 = j0 + (int64_t)blockIdx.x * KT, t1 = min(t0 + KT, j0 + nJ);
    const int64_t a_lo = t0 / n1;
    const int na = (int)((t1 - 1) / n1 - a_lo) + 1;
    const double2 *src = F + g * (int64_t)L * Mh;
    const double inv_m = 1.0 / (double)M;
    // the first candidate of this thread and the per-step increments (j += NT)
    const int64_t jt = t0 + tid;
    int a_first = (int)(jt / n1 - a_lo), c_first = (int)(jt % n1);
    const int qa = NT / n1, qc = NT % n1;
    constexpr int PF = 2;                                // prefetch registers per thread (double2)
    double2 pf[PF];
    auto fetch = [&](int l) {
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const int i = tid + k * NT;
            pf[k] = i < Mh ? __ldg(src + (int64_t)l * Mh + i) : make_double2(0.0, 0.0);
        }
    };
    // the key of a bin, by exactly the arithmetic of k_kappa_grouped (it depends on the bin only)
    auto key = [&](double2 f) -> double {
        const double re = f.x * inv_m, im = f.y * inv_m;
        return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
    };
    auto put = [&](double *S, int i, double kk) {        // key of bin i (< Mh) at i, M-i, M+i, 2M-i
        S[i] = kk;
        S[M + i] = kk;
        if (i > 0) {
            S[M - i] = kk;
            S[2 * M - i] = kk;
        }
    };
    auto stage = [&](int l, int buf) {                   // keys of lattice l's bins + bin terms -> buf
        double *S = ssk + buf * 2 * M;
#pragma unroll
        for (int k = 0; k < PF; ++k)
            if (tid + k * NT < Mh) put(S, tid + k * NT, key(pf[k]));
        for (int i = tid + PF * NT; i < Mh; i += NT) put(S, i, key(__ldg(src + (int64_t)l * Mh + i)));
        const int32_t *bl = bins + (int64_t)l * ldb;
        for (int i = tid; i < na; i += NT) sA[buf * AT + i] = __ldg(bl + (a_lo + i) * n1);
        const int32_t b00 = __ldg(bl);
        for (int i = tid; i < n1; i += NT) {
            const int32_t v = __ldg(bl + i) - b00;
            sD[buf * n1 + i] = v < 0 ? v + M : v;
        }
    };
    double km[KPT];
    fetch(0);
    stage(0, 0);
    __syncthreads();
    for (int l = 0; l < L; ++l) {
        const int buf = l & 1;
        if (l + 1 < L) fetch(l + 1);                      // in flight during the gathers below
        const double *S = ssk + buf * 2 * M;
        const int32_t *A = sA + buf * AT, *D = sD + buf * n1;
        int a = a_first, c = c_first;
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            if (t0 + tid + (int64_t)k * NT >= t1) break;     // ragged tile end (a, c past the staged range)
            UB_CHECK(a >= 0 && a < na && c >= 0 && c < n1);
            const int b = A[a] + D[c];
            UB_CHECK(b >= 0 && b < 2 * M);
            const double kk = S[b];
            km[k] = (l == 0) ? kk : fmin(km[k], kk);
            a += qa;
            c += qc;
            if (c >= n1) {
                c -= n1;
                ++a;
            }
        }
        if (l + 1 < L) {
            stage(l + 1, buf ^ 1);
            __syncthreads();
        }
    }
    unsigned long long best = 0ull;
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
        const int64_t j = t0 + tid + (int64_t)k * NT;
        if (j < t1) {
            kmin[g * ldk + (j - j0)] = (tau && km[k] <= tau[g]) ? 0.0 : km[k];
            const unsigned long long bits = (unsigned long long)__double_as_longlong(km[k]);
            best = bits > best ? bits : best;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other > best ? other : best;
    }
    if ((tid & 31) == 0) wmax[tid >> 5] = best;
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < NT / 32; ++w) best = wmax[w] > best ? wmax[w] : best;
        atomicMax(kmax, best);
    }
}

}  // namespace usfft

#include "rader.cuh"
#include "rader_t.cuh"
#include "fft400.cuh"
#include "fft_r.cuh"

using namespace usfft;

namespace {

template <int N, int WPR, int RPC>
usfft_status launch_rader_t(usfft_ctx *c, const double *u, const SlabParams &S, int64_t G_loc,
                            int32_t L, const RaderArgs &A, double2 *F) {
    const int64_t rows = G_loc * L;
    const size_t smem = sizeof(double2) * 2 * (size_t)N * RPC;
    auto kern = k_fft_rader_t<N, WPR, RPC>;
    int per_sm = 0;
    if (usfft_status s = kernel_fit(c, kern, WPR * 32 * RPC, smem, &per_sm)) return s;
    int64_t grid = (rows + RPC - 1) / RPC;
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * c->sm_count;
    if (grid > resident) grid = resident;                 // persistent: each group loops over rows
    kern<<<(unsigned)grid, WPR * 32 * RPC, smem, c->stream>>>(u, S, G_loc, L, A, F, rows);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

template <int N, int WPR, int RPC>
usfft_status launch_rader_tp(usfft_ctx *c, const double *u, const SlabParams &S, int64_t G_loc,
                             int32_t L, const RaderArgs &A, double2 *F) {
    const int64_t rows = G_loc * L, pairs = G_loc * ((L + 1) / 2);
    const size_t smem = sizeof(double2) * 2 * (size_t)(N + 2) * RPC;
    auto kern = k_fft_rader_tp<N, WPR, RPC>;
    int per_sm = 0;
    if (usfft_status s = kernel_fit(c, kern, WPR * 32 * RPC, smem, &per_sm)) return s;
    int64_t grid = (pairs + RPC - 1) / RPC;
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * c->sm_count;
    if (grid > resident) grid = resident;                 // persistent: each group loops over pairs
    kern<<<(unsigned)grid, WPR * 32 * RPC, smem, c->stream>>>(u, S, G_loc, L, A, F, rows);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

template <int N, int GROUP, int NPAIR, int MINB, int... Rs>
usfft_status launch_rader_r(usfft_ctx *c, const double *u, const SlabParams &S, int64_t G_loc,
                            int32_t L, const RaderArgs &A, double2 *F) {
    const int64_t rows = G_loc * L, pairs = G_loc * ((L + 1) / 2);
    constexpr int R0 = fr::First<Rs...>::value, MH = (N + 1) / 2 + 1, NB = 2 * MH > N + R0 ? 2 * MH : N + R0;
    const size_t smem = sizeof(double2) * (size_t)NB * NPAIR;
    auto kern = k_fft_rader_r<N, GROUP, NPAIR, MINB, Rs...>;
    int per_sm = 0;
    if (usfft_status s = kernel_fit(c, kern, GROUP * NPAIR, smem, &per_sm)) return s;
    int64_t grid = (pairs + NPAIR - 1) / NPAIR;
    const int64_t resident = (int64_t)(per_sm > 0 ? per_sm : 1) * c->sm_count;
    if (grid > resident) grid = resident;                 // persistent: each CTA loops over pairs
    kern<<<(unsigned)grid, GROUP * NPAIR, smem, c->stream>>>(u, S, G_loc, L, A, F, rows);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

bool is_prime64(int64_t n) {
    if (n < 2) return false;
    if (n % 2 == 0) return n == 2;
    for (int64_t f = 3; f * f <= n; f += 2)
        if (n % f == 0) return false;
    return true;
}

int64_t powmod(int64_t b, int64_t e, int64_t m) {
    int64_t r = 1 % m;
    b %= m;
    while (e > 0) {
        if (e & 1) r = (r * b) % m;
        b = (b * b) % m;
        e >>= 1;
    }
    return r;
}

// Rader plan for prime M with 7-smooth M-1 (nullptr-equivalent plan.M == 0 otherwise)
usfft_status get_rader(usfft_ctx *c, int64_t M, RaderPlan *out) {
    auto &cache = c->rader;                               // per ctx (device), freed by usfft_finalize
    const int64_t key = M;
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return USFFT_OK;
    }
    RaderPlan P;
    const int64_t N = M - 1;
    int64_t rem = N;
    int ns = 0;
    if (M >= 5 && is_prime64(M)) {
        for (int r : {4, 2, 3, 5, 7})
            while (rem % r == 0 && ns < 16) {
                P.radix[ns++] = r;
                rem /= r;
            }
    }
    if (rem != 1 || M < 5 || !is_prime64(M)) {          // not Rader-able: caller falls back
        cache[key] = P;
        *out = P;
        return USFFT_OK;
    }
    P.M = M;
    P.N = N;
    P.nstage = ns;
    // primitive root: g^(N/f) != 1 for every prime factor f of N
    int64_t gp = 2;
    for (;; ++gp) {
        bool ok = true;
        for (int64_t f : {2, 3, 5, 7})
            if (N % f == 0 && powmod(gp, N / f, M) == 1) ok = false;
        if (ok) break;
    }
    const int64_t ginv = powmod(gp, N - 1, M);
    std::vector<int32_t> perm(N), outidx(N);
    int64_t a = 1, bq = 1;
    for (int64_t k = 0; k < N; ++k) {
        perm[k] = (int32_t)a;
        outidx[k] = (int32_t)bq;
        a = (a * gp) % M;
        bq = (bq * ginv) % M;
    }
    const long double PI = 3.141592653589793238462643383279502884L;
    std::vector<long double> cN(N), sN(N);
    for (int64_t k = 0; k < N; ++k) {
        cN[k] = cosl(2.0L * PI * (long double)k / (long double)N);
        sN[k] = sinl(2.0L * PI * (long double)k / (long double)N);
    }
    std::vector<double2> tw(N), bf(N);
    for (int64_t k = 0; k < N; ++k) tw[k] = make_double2((double)cN[k], (double)-sN[k]);
    // b_n = e^{-2 pi i g^{-n}/M};  Bf[k] = (1/N) sum_n b_n e^{-2 pi i n k / N}  (long double)
    std::vector<long double> br(N), bi(N);
    for (int64_t n = 0; n < N; ++n) {
        const long double ang = 2.0L * PI * (long double)outidx[n] / (long double)M;
        br[n] = cosl(ang);
        bi[n] = -sinl(ang);
    }
    for (int64_t k = 0; k < N; ++k) {
        long double re = 0.0L, im = 0.0L;
        int64_t idx = 0;
        for (int64_t n = 0; n < N; ++n) {
            // (br + i bi) (cN[idx] - i sN[idx])
            re += br[n] * cN[idx] + bi[n] * sN[idx];
            im += bi[n] * cN[idx] - br[n] * sN[idx];
            idx += k;
            if (idx >= N) idx -= N;
        }
        bf[k] = make_double2((double)(re / (long double)N), (double)(im / (long double)N));
    }
    USFFT_CUDA(c, cudaMalloc(&P.tw, sizeof(double2) * N));
    USFFT_CUDA(c, cudaMalloc(&P.bf, sizeof(double2) * N));
    USFFT_CUDA(c, cudaMalloc(&P.perm, sizeof(int32_t) * N));
    USFFT_CUDA(c, cudaMalloc(&P.outidx, sizeof(int32_t) * N));
    USFFT_CUDA(c, cudaMemcpy(P.tw, tw.data(), sizeof(double2) * N, cudaMemcpyHostToDevice));
    USFFT_CUDA(c, cudaMemcpy(P.bf, bf.data(), sizeof(double2) * N, cudaMemcpyHostToDevice));
    USFFT_CUDA(c, cudaMemcpy(P.perm, perm.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice));
    USFFT_CUDA(c, cudaMemcpy(P.outidx, outidx.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice));
    cache[key] = P;
    *out = P;
    return USFFT_OK;
}

}  // namespace

static usfft_status get_twiddles(usfft_ctx *c, int64_t M, double2 **out) {
    auto it = c->twiddles.find(M);
    if (it != c->twiddles.end()) {
        *out = it->second;
        return USFFT_OK;
    }
    double2 *tw = nullptr;
    USFFT_CUDA(c, cudaMalloc(&tw, sizeof(double2) * M));
    k_twiddles<<<grid1d(M, 256), 256, 0, c->stream>>>(M, tw);
    USFFT_CHECK_LAUNCH(c);
    c->twiddles[M] = tw;
    *out = tw;
    return USFFT_OK;
}

namespace {
// K7: keys of nJ candidates (bins[l * ldb + j]) into kmin[g * ldk + j], max into kappa_max
// (NULL: a ctx scratch slot)
usfft_status launch_keys(usfft_ctx *c, int64_t M, int32_t L, int64_t G_loc, const double *spectra,
                         const int32_t *bins, int64_t ldb, int64_t nJ, double *kappa_min, int64_t ldk,
                         double *kappa_max, const double *tau = nullptr) {
    unsigned long long *km = reinterpret_cast<unsigned long long *>(kappa_max);
    if (!km) km = reinterpret_cast<unsigned long long *>(static_cast<char *>(c->dscal) + 8);
    const size_t tile_bytes = sizeof(int32_t) * 256 * (size_t)L;
    // the bins tile is shared by KG_NODES nodes whose spectra are gathered from L1/L2 (measured
    // on B200 against one CTA per node with its spectra staged in shared memory: 57 vs 64 us on
    // the config-2 round, 1.29 vs 1.99 s per streamed round of |J| = 8.2e6, L = 35)
    USFFT_REQUIRE(c, tile_bytes <= c->smem_optin, "L = %d lattices: bins tile too large", (int)L);
    USFFT_REQUIRE(c, (G_loc + KG_NODES - 1) / KG_NODES <= 65535, "too many nodes for the key grid");
    if (usfft_status s2 = kernel_fit(c, k_kappa_grouped, 0, tile_bytes, nullptr)) return s2;
    dim3 grid((unsigned)((nJ + 255) / 256), (unsigned)((G_loc + KG_NODES - 1) / KG_NODES));
    k_kappa_grouped<<<grid, 256, tile_bytes, c->stream>>>(reinterpret_cast<const double2 *>(spectra), bins, ldb,
                                                          nJ, M, L, G_loc, kappa_min, ldk, km, tau);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}
}  // namespace

extern "C" usfft_status usfft_lattice_fft(usfft_ctx *c, const usfft_lattice_desc *lat,
                                          int64_t G_loc, const double *u, int32_t nslab,
                                          const int64_t *slab_b0, const int32_t *bins, int64_t nJ,
                                          double *spectra, double *kappa_min, double *kappa_max) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, lat != nullptr, "lattice desc is NULL");
    const int64_t M = lat->M;
    const int32_t L = lat->L;
    USFFT_REQUIRE(c, M >= 2 && M <= (int64_t(1) << 26) && L >= 1, "bad M / L");
    USFFT_REQUIRE(c, G_loc >= 0 && nJ >= 0, "negative sizes");
    USFFT_REQUIRE(c, nslab >= 1 && nslab <= kMaxSlab && slab_b0 != nullptr, "nslab out of [1, %d]", kMaxSlab);
    USFFT_REQUIRE(c, slab_b0[0] == 0 && slab_b0[nslab] == (int64_t)L * M, "slab_b0 must span [0, L*M]");
    for (int p = 0; p < nslab; ++p)
        USFFT_REQUIRE(c, slab_b0[p + 1] >= slab_b0[p], "slab_b0 not monotone");
    USFFT_REQUIRE(c, G_loc == 0 || (u && spectra), "u / spectra NULL");
    USFFT_REQUIRE(c, nJ == 0 || G_loc == 0 || (bins && kappa_min), "bins / kappa_min NULL");
    const size_t smem = sizeof(double) * (size_t)((M + 1) & ~int64_t(1)) + sizeof(double2) * (size_t)M;
    SlabParams S;
    S.nslab = nslab;
    for (int p = 0; p <= nslab; ++p) S.b0[p] = slab_b0[p];

    if (kappa_max) USFFT_CUDA(c, cudaMemsetAsync(kappa_max, 0, sizeof(double), c->stream));
    if (G_loc == 0) return USFFT_OK;
    double2 *tw = nullptr;
    usfft_status s = get_twiddles(c, M, &tw);
    if (s) return s;
    const int64_t rows = G_loc * L;
    RaderPlan R;
    s = get_rader(c, M, &R);
    if (s) return s;
    const size_t smem_r = sizeof(double) * (size_t)((M + 1) & ~int64_t(1)) + 2 * sizeof(double2) * (size_t)(M - 1);
    if (R.M == M && smem_r <= c->smem_optin) {
        RaderArgs A;
        A.M = R.M;
        A.N = R.N;
        A.nstage = R.nstage;
        A.radix_code = 0;
        for (int k = 0; k < R.nstage && k < 16; ++k) A.radix_code |= (uint64_t)R.radix[k] << (4 * k);
        A.tw = R.tw;
        A.perm = R.perm;
        A.outidx = R.outidx;
        A.bf = R.bf;
        double2 *Fo = reinterpret_cast<double2 *>(spectra);
        // the lattice sizes of the BASELINE configs (Z2) have compile-time plans; other
        // Rader-able M take the runtime-plan kernel
        if (R.N == 96) s = launch_rader_t<96, 1, 4>(c, u, S, G_loc, L, A, Fo);
        else if (R.N == 400) s = launch_rader_r<400, 20, 8, 3, 20, 20>(c, u, S, G_loc, L, A, Fo);
        else if (R.N == 2016) s = launch_rader_tp<2016, 4, 1>(c, u, S, G_loc, L, A, Fo);
        else if (R.N == 4000) s = launch_rader_r<4000, 200, 1, 2, 20, 20, 10>(c, u, S, G_loc, L, A, Fo);
        else {
            if (usfft_status s2 = kernel_fit(c, k_fft_rader, 0, smem_r, nullptr)) return s2;
            const int threads = M <= 512 ? 128 : 256;
            k_fft_rader<<<(unsigned)rows, threads, smem_r, c->stream>>>(u, S, G_loc, L, A, Fo);
            USFFT_CHECK_LAUNCH(c);
        }
        if (s) return s;
    } else {
        USFFT_REQUIRE(c, smem <= c->smem_optin, "M = %lld too large for the direct DFT", (long long)M);
        if (usfft_status s2 = kernel_fit(c, k_dft_direct, 0, smem, nullptr)) return s2;
        k_dft_direct<<<(unsigned)rows, 256, smem, c->stream>>>(u, S, G_loc, M, L, tw,
                                                                reinterpret_cast<double2 *>(spectra));
        USFFT_CHECK_LAUNCH(c);
    }
    if (nJ > 0) return launch_keys(c, M, L, G_loc, spectra, bins, nJ, nJ, kappa_min, nJ, kappa_max);
    return USFFT_OK;
}

extern "C" usfft_status usfft_lattice_keys(usfft_ctx *c, const usfft_lattice_desc *lat, int64_t G_loc,
                                           const double *spectra, const int32_t *bins, int64_t ldb,
                                           int64_t nJ, double *kappa_min, int64_t ldk, double *kappa_max,
                                           const double *tau) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, lat != nullptr, "lattice desc is NULL");
    USFFT_REQUIRE(c, lat->M >= 2 && lat->M <= (int64_t(1) << 26) && lat->L >= 1, "bad M / L");
    USFFT_REQUIRE(c, G_loc >= 0 && nJ >= 0 && ldb >= nJ && ldk >= nJ, "bad sizes / leading dimensions");
    if (G_loc == 0 || nJ == 0) return USFFT_OK;
    USFFT_REQUIRE(c, spectra && bins && kappa_min && kappa_max, "NULL argument");
    return launch_keys(c, lat->M, lat->L, G_loc, spectra, bins, ldb, nJ, kappa_min, ldk, kappa_max, tau);
}

// a8 for the candidates j0 .. j0+nJ-1 of the product set J = I_prev x kt (j = a n1 + c, Z10):
// bins is the whole [L][ldb] map; keys into kappa_min[g * ldk + (j - j0)].  spectra larger than L2 and |J| >= 4 (M/2+1):
// k_kappa_tiled; otherwise the gather kernel on bins + j0 (both bit-identical).
extern "C" usfft_status usfft_lattice_keys_product(usfft_ctx *c, const usfft_lattice_desc *lat, int64_t G_loc,
                                                   const double *spectra, const int32_t *bins, int64_t ldb,
                                                   int64_t j0, int64_t nJ, int64_t n1, double *kappa_min,
                                                   int64_t ldk, double *kappa_max, const double *tau) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, lat != nullptr, "lattice desc is NULL");
    USFFT_REQUIRE(c, lat->M >= 2 && lat->M <= (int64_t(1) << 26) && lat->L >= 1, "bad M / L");
    USFFT_REQUIRE(c, G_loc >= 0 && nJ >= 0 && j0 >= 0 && n1 >= 1 && ldb >= j0 + nJ && ldk >= nJ,
                  "bad sizes / leading dimensions");
    USFFT_REQUIRE(c, ldb % n1 == 0 && ldb < (int64_t(1) << 31), "ldb must be |J| = n_prev * n1 (< 2^31)");
    if (G_loc == 0 || nJ == 0) return USFFT_OK;
    USFFT_REQUIRE(c, spectra && bins && kappa_min && kappa_max, "NULL argument");
    const int64_t M = lat->M, Mh = M / 2 + 1;
    constexpr int NT = 512, KPT = 24, MINB = 1, KT = NT * KPT;
    const size_t smem = sizeof(double) * 4 * (size_t)M + sizeof(int32_t) * 2 * (size_t)(KT / n1 + 2 + n1);
    // The gathers of k_kappa_grouped hit L2 while the spectra fit there (config 2: 52 MB): it is
    // then 1.1-3.6x faster than the tiled kernel for every |J|.  With spectra beyond L2 every
    // gather is a DRAM access and the tiled kernel, which streams each spectrum once per tile but
    // builds 2M keys per (node, lattice), wins from |J| ~ 2-4 (M/2+1) on: 1.8 vs 4.1 ms at
    // |J| = 4 (M/2+1) and 15.7 vs 50.1 ms at 64 (M/2+1) on config 4's shape, while at |J| <= 2
    // (M/2+1) the gathers are faster (configs 3, 5: 0.52 vs 0.78 ms, 3.5 vs 5.1 ms)
    // (tools/keys_crossover.py and bench.py, measured on the B200).
    const size_t spectra_bytes = sizeof(double2) * (size_t)G_loc * lat->L * Mh;
    const bool tiled = USFFT_KEYS_TILED_ALWAYS || (4 * spectra_bytes > 3 * c->l2_bytes && nJ >= 4 * Mh);
    if (!tiled || smem > c->smem_optin || G_loc > 65535)
        return launch_keys(c, M, lat->L, G_loc, spectra, bins + j0, ldb, nJ, kappa_min, ldk, kappa_max, tau);
    auto kern = k_kappa_tiled<NT, KPT, MINB>;
    if (usfft_status s = kernel_fit(c, kern, NT, smem, nullptr)) return s;
    dim3 grid((unsigned)((nJ + KT - 1) / KT), (unsigned)G_loc);
    kern<<<grid, NT, smem, c->stream>>>(reinterpret_cast<const double2 *>(spectra), bins, ldb, j0, nJ, (int32_t)n1,
                                        (int32_t)M, lat->L, kappa_min, ldk,
                                        reinterpret_cast<unsigned long long *>(kappa_max), tau);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

extern "C" usfft_status usfft_lattice_dft_bins(usfft_ctx *c, int64_t M, int64_t G_loc, const double *u,
                                               int32_t nslab, const int64_t *slab_b0,
                                               const int32_t *bins, const int32_t *idx, int64_t n,
                                               double *coef, int64_t nI) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, M >= 2 && M <= (int64_t(1) << 26) && G_loc >= 0 && n >= 0 && nI >= n, "bad sizes");
    USFFT_REQUIRE(c, nslab >= 1 && nslab <= kMaxSlab && slab_b0 != nullptr, "nslab out of [1, %d]", kMaxSlab);
    USFFT_REQUIRE(c, slab_b0[0] == 0 && slab_b0[nslab] == M, "slab_b0 must span [0, M]");
    if (G_loc == 0 || n == 0) return USFFT_OK;
    USFFT_REQUIRE(c, u && bins && idx && coef, "NULL argument");
    USFFT_REQUIRE(c, (n + DB_TA - 1) / DB_TA <= 0x7fffffff && (G_loc + DB_TG - 1) / DB_TG <= 65535, "grid too large");
    SlabParams S;
    S.nslab = nslab;
    for (int p = 0; p <= nslab; ++p) S.b0[p] = slab_b0[p];
    double2 *tw = nullptr;
    if (usfft_status s = get_twiddles(c, M, &tw)) return s;
    dim3 grid((unsigned)((n + DB_TA - 1) / DB_TA), (unsigned)((G_loc + DB_TG - 1) / DB_TG));
    k_dft_bins<<<grid, 256, 0, c->stream>>>(u, S, G_loc, M, tw, bins, idx, n, reinterpret_cast<double2 *>(coef), nI);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

