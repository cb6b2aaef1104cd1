// detect.cu — K8 threshold + per-node top-s~ selection + votes, K10 union/compaction, K7b resolve.
// usfft_detect_select / usfft_detect_union / usfft_resolve (include/usfft.h; a9-a12 of SURVEY §8(a)).
//
// Selection is a radix select on the 64-bit patterns of the keys (non-negative doubles order like
// uint64): 8 passes of 8 bits find the s~-th largest key T; then one ordered pass keeps every key
// > T and the first (by candidate index) keys == T up to s~ (Z6), and of those the ones with
// kappa >= theta^2 and kappa > 0 (Z5).  All decisions are integer/ordered comparisons of the same
// doubles, hence exact and independent of thread scheduling; votes are integer atomics.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace usfft {

__device__ __forceinline__ double theta2_of(double theta_rel, double theta_abs, const double *kmax) {
    if (theta_abs > 0.0) return __dmul_rn(theta_abs, theta_abs);
    return __dmul_rn(__dmul_rn(theta_rel, theta_rel), kmax[0]);
}

// one CTA per owned node g (128 threads: the radix passes are barrier-bound); the node's keys
// are staged in shared memory when |J| <= KSTAGE
constexpr int64_t KSTAGE = 6144;
// larger rows (the streamed chunks of Z29, mostly keys prefiltered to 0): the positive keys and
// their indices are compacted in order into shared memory when there are at most KCOMP of them
constexpr int KCOMP = 2048;

__global__ void __launch_bounds__(128)
k_select(const double *__restrict__ kmin, int64_t nJ, const double *__restrict__ kmax,
         int32_t s_tilde, double theta_rel, double theta_abs, int32_t *__restrict__ votes,
         int32_t *__restrict__ det_g, int32_t *__restrict__ n_det_g, double *__restrict__ th2_out) {
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_need;
    __shared__ bool s_exact;
    __shared__ unsigned int s_zero;
    __shared__ int scan_sh[33];
    extern __shared__ unsigned long long kst[];
    __shared__ int warp_cnt[4];
    const int64_t g = blockIdx.x;
    const unsigned long long *keys =
        reinterpret_cast<const unsigned long long *>(kmin + g * nJ);
    const int32_t *jmap = nullptr;                     // compacted row: entry q is candidate jmap[q]
    if (nJ <= KSTAGE) {
        for (int64_t j = threadIdx.x; j < nJ; j += blockDim.x) kst[j] = __ldg(keys + j);
        keys = kst;
        __syncthreads();
    } else {
        // order-preserving compaction of the positive keys: warp w owns the contiguous quarter
        // [w seg, (w+1) seg); pass 1 counts (ballots), pass 2 writes at the warp's offset.  Zero
        // keys are never taken, and with the zeros removed the radix select of the s~-th largest
        // and the index order of ties are those of the full row.
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const int64_t seg = (nJ + 3) / 4, lo = w * seg, hi = min(nJ, lo + seg);
        int cnt = 0;
        for (int64_t j0 = lo; j0 < hi; j0 += 32) {
            const int64_t j = j0 + lane;
            const unsigned long long key = j < hi ? __ldg(keys + j) : 0ull;
            cnt += __popc(__ballot_sync(0xffffffffu, key != 0ull));
        }
        if (lane == 0) warp_cnt[w] = cnt;
        __syncthreads();
        const int npos = warp_cnt[0] + warp_cnt[1] + warp_cnt[2] + warp_cnt[3];
        if (npos <= KCOMP) {
            unsigned long long *ck = kst;
            int32_t *cj = reinterpret_cast<int32_t *>(kst + KCOMP);
            int off = 0;
            for (int q = 0; q < w; ++q) off += warp_cnt[q];
            for (int64_t j0 = lo; j0 < hi; j0 += 32) {
                const int64_t j = j0 + lane;
                const unsigned long long key = j < hi ? __ldg(keys + j) : 0ull;
                const unsigned int b = __ballot_sync(0xffffffffu, key != 0ull);
                if (key != 0ull) {
                    const int pos = off + __popc(b & ((1u << lane) - 1u));
                    ck[pos] = key;
                    cj[pos] = (int32_t)j;
                }
                off += __popc(b);
            }
            __syncthreads();
            keys = ck;
            jmap = cj;
            nJ = npos;
        }
    }
    const double th2 = theta2_of(theta_rel, theta_abs, kmax);
    if (g == 0 && threadIdx.x == 0 && th2_out) th2_out[0] = th2;

    // Radix select of the s~-th largest key.  After a pass the bucket holding rank k is known;
    // if that bucket holds exactly k keys, every key >= its lower bound is a member and no tie
    // remains (early exit, typical for distinct doubles); otherwise keep refining.
    unsigned long long T = 0ull, Tmin = 0ull;
    long long need_eq = 0;
    bool by_min = false;                         // members = {key >= Tmin}
    if ((int64_t)s_tilde >= nJ) {
        by_min = true;                           // every candidate is within the top s~
        Tmin = 0ull;
    } else {
        unsigned long long prefix = 0ull, pmask = 0ull;
        long long k = s_tilde;                   // rank (1-based, from the top) still to find
        if (threadIdx.x == 0) s_zero = 0u;
        for (int pass = 0; pass < 8; ++pass) {
            const int shift = 56 - 8 * pass;
            for (int q = threadIdx.x; q < 256; q += blockDim.x) hist[q] = 0u;
            __syncthreads();
            unsigned int nzero = 0u;
#pragma unroll 8
            for (int64_t j = threadIdx.x; j < nJ; j += blockDim.x) {
                const unsigned long long key = keys[j];
                nzero += key == 0ull ? 1u : 0u;
                // zero keys are never members (take needs kv > 0) and, once there are more than
                // s~ positive keys, never hold rank s~: leaving them out of the histogram keeps
                // the threshold and avoids serialising on bucket 0 (the streamed chunks, Z29,
                // are mostly prefiltered zeros)
                if (key != 0ull && (key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255ull], 1u);
            }
            if (pass == 0) {                     // at most s~ positive keys: all of them are members
                if (nzero) atomicAdd(&s_zero, nzero);
                __syncthreads();
                if (nJ - (int64_t)s_zero <= (int64_t)s_tilde) {   // (zeros are never taken)
                    by_min = true;
                    Tmin = 1ull;
                    break;
                }
            }
            __syncthreads();
            if (threadIdx.x < 32) {              // warp-parallel search from the top bucket
                const int lane = threadIdx.x;
                unsigned int c8[8];
                unsigned int cl = 0;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    c8[b] = hist[8 * lane + b];
                    cl += c8[b];
                }
                long long suf = cl;              // sum over lanes >= lane
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long y = __shfl_down_sync(0xffffffffu, suf, o);
                    if (lane + o < 32) suf += y;
                }
                const unsigned int ball = __ballot_sync(0xffffffffu, suf >= k);
                const int Ls = __popc(ball) - 1;       // top-most lane whose suffix reaches k
                if (lane == Ls) {
                    long long cum = suf - cl;          // keys in buckets above this lane's
                    int digit = 8 * lane;
                    unsigned int cnt = 0;
                    for (int b = 7; b >= 0; --b) {
                        if (cum + (long long)c8[b] >= k) {
                            digit = 8 * lane + b;
                            cnt = c8[b];
                            break;
                        }
                        cum += c8[b];
                    }
                    s_prefix = prefix | ((unsigned long long)digit << shift);
                    s_need = k - cum;
                    s_exact = (long long)cnt == k - cum;
                }
            }
            __syncthreads();
            prefix = s_prefix;
            k = s_need;
            pmask |= 255ull << shift;
            if (s_exact) {                      // whole bucket selected: members are key >= prefix
                by_min = true;
                Tmin = prefix;
                break;
            }
        }
        T = prefix;
        need_eq = k;                             // how many keys == T are taken (by index)
    }
    // ordered pass: membership, threshold, output in ascending j, votes.  Keys are read OB blocks
    // at a time (OB loads in flight per thread) and a group of blocks without any key that could
    // be taken or counted (key >= the threshold) is skipped with one barrier
    int eq_run = 0, out_run = 0;
    int32_t *out = det_g + g * (int64_t)s_tilde;
    constexpr int OB = 8;
    for (int64_t base0 = 0; base0 < nJ; base0 += OB * (int64_t)blockDim.x) {
        unsigned long long kb[OB];
        bool any = false;
#pragma unroll
        for (int b = 0; b < OB; ++b) {
            const int64_t j = base0 + (int64_t)b * blockDim.x + threadIdx.x;
            kb[b] = j < nJ ? keys[j] : 0ull;
            any |= kb[b] != 0ull && (by_min ? kb[b] >= Tmin : kb[b] >= T);
        }
        if (!__syncthreads_or(any)) continue;
#pragma unroll 1
        for (int b = 0; b < OB; ++b) {
        const int64_t base = base0 + (int64_t)b * blockDim.x;
        if (base >= nJ) break;
        const int64_t j = base + threadIdx.x;
        const bool valid = j < nJ;
        const unsigned long long key = kb[b];
        const int is_eq = (!by_min && valid && key == T) ? 1 : 0;
        int eq_tot;
        const int eq_before = eq_run + block_exscan(is_eq, scan_sh, &eq_tot);
        const bool member = valid && (by_min ? key >= Tmin : (key > T || (is_eq && eq_before < need_eq)));
        const double kv = __longlong_as_double((long long)key);
        const int take = (member && kv >= th2 && kv > 0.0) ? 1 : 0;
        int tot;
        const int pos = out_run + block_exscan(take, scan_sh, &tot);
        if (take) {
            const int32_t jj = jmap ? jmap[j] : (int32_t)j;
            out[pos] = jj;
            atomicAdd(votes + jj, 1);
        }
        eq_run += eq_tot;
        out_run += tot;
        }
    }
    for (int q = out_run + threadIdx.x; q < s_tilde; q += blockDim.x) out[q] = -1;
    if (threadIdx.x == 0) n_det_g[g] = out_run;
}

// Small candidate sets (|J| <= 32 KPL): one warp per node with the node's keys in registers
// (candidate j = 32 k + lane in register k).  The s~-th largest key T is found by a bitwise binary
// search (largest T with #{key >= T} >= s~, 63 counting passes, warp reductions only), then one
// ordered pass takes every key > T and the first (by j) keys == T up to s~ - #{key > T}: the same
// members as the radix select of k_select, with no CTA barrier.
template <int KPL>
__global__ void __launch_bounds__(128)
k_select_warp(const double *__restrict__ kmin, int64_t nJ, int64_t G, const double *__restrict__ kmax,
              int32_t s_tilde, double theta_rel, double theta_abs, int32_t *__restrict__ votes,
              int32_t *__restrict__ det_g, int32_t *__restrict__ n_det_g, double *__restrict__ th2_out) {
    const int lane = threadIdx.x & 31;
    const int64_t g = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const double th2 = theta2_of(theta_rel, theta_abs, kmax);
    if (g == 0 && lane == 0 && th2_out) th2_out[0] = th2;
    if (g >= G) return;
    const unsigned long long *row = reinterpret_cast<const unsigned long long *>(kmin + g * nJ);
    unsigned long long key[KPL];
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
        const int64_t j = 32 * k + lane;
        key[k] = j < nJ ? __ldg(row + j) : 0ull;
    }
    auto count_ge = [&](unsigned long long t) -> int {
        unsigned c = 0;
#pragma unroll
        for (int k = 0; k < KPL; ++k) c += key[k] >= t ? 1u : 0u;
        return (int)__reduce_add_sync(0xffffffffu, c);   // one warp-reduce instruction (sm_80+)
    };
    unsigned long long T = 0ull;
    if ((int64_t)s_tilde < nJ) {
        for (int b = 62; b >= 0; --b) {                  // non-negative doubles: bit 63 is 0
            const unsigned long long cand = T | (1ull << b);
            if (count_ge(cand) >= s_tilde) T = cand;
        }
    }
    // members: key > T, and the first need_eq keys == T by index (T = 0: every key qualifies)
    unsigned gtl = 0;
#pragma unroll
    for (int k = 0; k < KPL; ++k) gtl += key[k] > T ? 1u : 0u;
    const int gt = (int)__reduce_add_sync(0xffffffffu, gtl);
    const int need_eq = (int64_t)s_tilde < nJ ? s_tilde - gt : KPL * 32;
    const unsigned lt = (1u << lane) - 1u;
    int eq_run = 0, out_run = 0;
    int32_t *out = det_g + g * (int64_t)s_tilde;
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
        const int64_t j = 32 * k + lane;
        const bool valid = j < nJ;
        const bool is_eq = valid && key[k] == T;
        const unsigned eqm = __ballot_sync(0xffffffffu, is_eq);
        const bool member = valid && (key[k] > T || (is_eq && eq_run + __popc(eqm & lt) < need_eq));
        const double kv = __longlong_as_double((long long)key[k]);
        const bool take = member && kv >= th2 && kv > 0.0;
        const unsigned tm = __ballot_sync(0xffffffffu, take);
        if (take) {
            out[out_run + __popc(tm & lt)] = (int32_t)j;
            atomicAdd(votes + j, 1);
        }
        eq_run += __popc(eqm);
        out_run += __popc(tm);
    }
    for (int q = out_run + lane; q < s_tilde; q += 32) out[q] = -1;
    if (lane == 0) n_det_g[g] = out_run;
}

// streamed selection (Z29): one CTA per owned node moves the selected (key, j) pairs of row g of
// merged to the carry (update mode), or emits det_g and votes from the final selection on the
// carry (emit mode, det_g != NULL).  The selection is read completely before anything is written,
// so merged may alias carry_k.
__global__ void __launch_bounds__(256)
k_carry(int32_t s, int64_t width, double *merged, double *carry_k, int32_t *__restrict__ carry_j,
        const int32_t *__restrict__ det_pos, const int32_t *__restrict__ n_det_g, int64_t j0,
        int32_t *__restrict__ det_g, int32_t *__restrict__ votes, double *__restrict__ tau) {
    __shared__ double wmin[8];
    extern __shared__ double ck[];                               // [s] keys, then [s] j
    int32_t *cj = reinterpret_cast<int32_t *>(ck + s);
    const int64_t g = blockIdx.x;
    const int n = n_det_g[g];
    const int32_t *pos = det_pos + g * (int64_t)s;
    double *row = merged + g * width;
    int32_t *jrow = carry_j + g * (int64_t)s;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const int p = pos[r];
        ck[r] = row[p];
        cj[r] = p < s ? jrow[p] : (int32_t)(j0 + p - s);
    }
    __syncthreads();
    if (det_g == nullptr) {
        double *krow = carry_k + g * (int64_t)s;
        double mn = 1.0 / 0.0;
        for (int r = threadIdx.x; r < s; r += blockDim.x) {
            const double k = r < n ? ck[r] : 0.0;
            row[r] = k;
            krow[r] = k;
            jrow[r] = r < n ? cj[r] : -1;
            mn = fmin(mn, k);
        }
        if (tau) {                               // the carry's s~-th key once it is full (else 0)
            for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = mn;
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mn = fmin(mn, wmin[w]);
                tau[g] = n == s ? mn : 0.0;
            }
        }
    } else {
        int32_t *out = det_g + g * (int64_t)s;
        for (int r = threadIdx.x; r < s; r += blockDim.x) {
            out[r] = r < n ? cj[r] : -1;
            if (r < n) atomicAdd(votes + cj[r], 1);
        }
    }
}

// single CTA: flags |= votes > 0; ordered compaction of this round's detections and of the union
__global__ void __launch_bounds__(1024)
k_union(const int32_t *__restrict__ votes, int64_t nJ, uint8_t *__restrict__ flags,
        int32_t *__restrict__ det_idx, int32_t *__restrict__ union_idx,
        long long *__restrict__ counts) {
    __shared__ int scan_sh[33];
    long long nd = 0, nu = 0;
    for (int64_t base = 0; base < nJ; base += blockDim.x) {
        const int64_t j = base + threadIdx.x;
        int v = 0, f = 0;
        if (j < nJ) {
            v = votes[j] > 0 ? 1 : 0;
            f = (flags[j] | v) ? 1 : 0;
            flags[j] = (uint8_t)f;
        }
        int tv, tf;
        const int pv = block_exscan(v, scan_sh, &tv);
        const int pf = block_exscan(f, scan_sh, &tf);
        if (v) det_idx[nd + pv] = (int32_t)j;
        if (f && union_idx) union_idx[nu + pf] = (int32_t)j;
        nd += tv;
        nu += tf;
    }
    if (threadIdx.x == 0) {
        counts[0] = nd;
        counts[1] = nu;
    }
}

__device__ __forceinline__ int member_sorted(const int32_t *__restrict__ a, int n, int32_t k) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && a[lo] == k) ? 1 : 0;
}

// one CTA per owned node g: l* = first lattice where k is alias-free w.r.t. D_g (Z1, a12).
// The occupancy tables of LC lattices at a time live in shared memory ([LC][M] counts of D_g's
// bins), so a chunk costs two barriers and every candidate walks its lattices in registers.
__global__ void __launch_bounds__(256)
k_resolve(const double2 *__restrict__ F, const int32_t *__restrict__ bins, int64_t nJ, int64_t M,
          int32_t L, const int32_t *__restrict__ det_g, const int32_t *__restrict__ n_det_g,
          int32_t s_tilde, const int32_t *__restrict__ det_idx, int64_t n_det,
          double2 *__restrict__ coef, int32_t *__restrict__ lstar, int32_t LC) {
    extern __shared__ int cnt[];                       // [LC][M], then D_g [s_tilde]
    int32_t *Ds = cnt + (int64_t)LC * M;
    const int64_t g = blockIdx.x;
    const int32_t *Dg = det_g + g * (int64_t)s_tilde;
    const int nD = n_det_g[g];
    const int64_t Mh = M / 2 + 1;
    int32_t *ls = lstar + g * n_det;
    for (int q = threadIdx.x; q < nD; q += blockDim.x) Ds[q] = Dg[q];
    for (int64_t q = threadIdx.x; q < n_det; q += blockDim.x) ls[q] = -1;
    for (int l0 = 0; l0 < L; l0 += LC) {
        const int lc = min(LC, L - l0);
        for (int64_t m = threadIdx.x; m < (int64_t)lc * M; m += blockDim.x) cnt[m] = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < nD * lc; e += blockDim.x) {
            const int q = e % nD, l = e / nD;
            atomicAdd(&cnt[(int64_t)l * M + bins[(int64_t)(l0 + l) * nJ + Ds[q]]], 1);
        }
        __syncthreads();
        for (int64_t q = threadIdx.x; q < n_det; q += blockDim.x) {
            if (ls[q] >= 0) continue;
            const int32_t k = det_idx[q];
            int mem = -1;                              // k in D_g (looked up once, lazily)
            for (int l = 0; l < lc; ++l) {
                const int64_t b = bins[(int64_t)(l0 + l) * nJ + k];
                const int c = cnt[(int64_t)l * M + b];
                if (c == 1 && mem < 0) mem = member_sorted(Ds, nD, k);
                // k's own entry (k in D_g) does not count as an alias
                if (c == 0 || (c == 1 && mem == 1)) {
                    ls[q] = l0 + l;
                    coef[g * n_det + q] = spec_value(F + (g * L + l0 + l) * Mh, M, b);
                    break;
                }
            }
        }
        __syncthreads();
    }
    // median fallback (componentwise, lower median for even L)
    for (int64_t q = threadIdx.x; q < n_det; q += blockDim.x) {
        if (ls[q] >= 0) continue;
        const int32_t k = det_idx[q];
        double re[64], im[64];
        for (int l = 0; l < L; ++l) {
            const double2 v = spec_value(F + (g * L + l) * Mh, M, bins[(int64_t)l * nJ + k]);
            re[l] = v.x;
            im[l] = v.y;
        }
        for (int a = 1; a < L; ++a) {              // insertion sort, L <= 64
            double x = re[a], y = im[a];
            int p = a - 1;
            while (p >= 0 && re[p] > x) { re[p + 1] = re[p]; --p; }
            re[p + 1] = x;
            p = a - 1;
            while (p >= 0 && im[p] > y) { im[p + 1] = im[p]; --p; }
            im[p + 1] = y;
        }
        coef[g * n_det + q] = make_double2(re[(L - 1) / 2], im[(L - 1) / 2]);
    }
}

}  // namespace usfft

using namespace usfft;

extern "C" usfft_status usfft_detect_select(usfft_ctx *c, int64_t G_loc, int64_t nJ,
                                            const double *kappa_min, double *kappa_max,
                                            int32_t s_tilde, double theta_rel, double theta_abs,
                                            int32_t *votes, int32_t *det_g, int32_t *n_det_g,
                                            double *theta2) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, G_loc >= 0 && nJ >= 0 && s_tilde >= 1, "bad sizes");
    USFFT_REQUIRE(c, nJ <= 0x7fffffff, "|J| too large");
    USFFT_REQUIRE(c, theta_rel >= 0.0 && theta_abs >= 0.0, "negative theta");
    USFFT_REQUIRE(c, nJ == 0 || votes != nullptr, "votes NULL");
    USFFT_REQUIRE(c, G_loc == 0 || nJ == 0 || (kappa_min && kappa_max && det_g && n_det_g), "NULL pointer");
    // C2: the relative threshold needs the max over ALL nodes (Z5): all-reduce MAX in place
    if (comm_size(c) > 1 && theta_abs <= 0.0 && theta_rel > 0.0) {
        USFFT_REQUIRE(c, kappa_max != nullptr, "kappa_max NULL");
        if (usfft_status s = comm_max_f64(c, kappa_max, 1)) return s;
    }
    if (nJ > 0) USFFT_CUDA(c, cudaMemsetAsync(votes, 0, sizeof(int32_t) * nJ, c->stream));
    if (G_loc == 0 || nJ == 0) {
        if (G_loc > 0 && n_det_g) USFFT_CUDA(c, cudaMemsetAsync(n_det_g, 0, sizeof(int32_t) * G_loc, c->stream));
        return USFFT_OK;
    }
    if (nJ <= 32 * 64) {                                  // one warp per node; else the CTA radix select
        const unsigned grid = (unsigned)((G_loc + 3) / 4);
        auto launch = [&](auto kern) {
            kern<<<grid, 128, 0, c->stream>>>(kappa_min, nJ, G_loc, kappa_max, s_tilde, theta_rel, theta_abs,
                                              votes, det_g, n_det_g, theta2);
        };
        if (nJ <= 32 * 8) launch(k_select_warp<8>);
        else if (nJ <= 32 * 16) launch(k_select_warp<16>);
        else if (nJ <= 32 * 32) launch(k_select_warp<32>);
        else launch(k_select_warp<64>);
        USFFT_CHECK_LAUNCH(c);
        return USFFT_OK;
    }
    const size_t kst = nJ <= KSTAGE ? sizeof(unsigned long long) * (size_t)nJ
                                    : (sizeof(unsigned long long) + sizeof(int32_t)) * (size_t)KCOMP;
    if (usfft_status s = kernel_fit(c, k_select, 0, kst, nullptr)) return s;
    k_select<<<(unsigned)G_loc, 128, kst, c->stream>>>(kappa_min, nJ, kappa_max, s_tilde, theta_rel,
                                                        theta_abs, votes, det_g, n_det_g, theta2);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

extern "C" usfft_status usfft_detect_carry(usfft_ctx *c, int64_t G_loc, int32_t s_tilde, int64_t width,
                                           double *merged, double *carry_k, int32_t *carry_j,
                                           const int32_t *det_pos, const int32_t *n_det_g, int64_t j0,
                                           int32_t *det_g, int32_t *votes, double *tau) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, G_loc >= 0 && s_tilde >= 1 && width >= s_tilde && j0 >= 0, "bad sizes");
    USFFT_REQUIRE(c, j0 + width - s_tilde <= 0x7fffffff, "candidate index beyond int32");
    if (G_loc == 0) return USFFT_OK;
    USFFT_REQUIRE(c, merged && carry_j && det_pos && n_det_g, "NULL argument");
    USFFT_REQUIRE(c, det_g != nullptr || carry_k != nullptr, "update mode needs carry_k");
    USFFT_REQUIRE(c, det_g == nullptr || (votes != nullptr && width == s_tilde), "emit mode: votes, width = s_tilde");
    const size_t dyn = (sizeof(double) + sizeof(int32_t)) * (size_t)s_tilde;
    if (usfft_status s = kernel_fit(c, k_carry, 0, dyn, nullptr)) return s;
    k_carry<<<(unsigned)G_loc, 256, dyn, c->stream>>>(s_tilde, width, merged, carry_k, carry_j, det_pos, n_det_g,
                                                       j0, det_g, votes, tau);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

extern "C" usfft_status usfft_detect_union(usfft_ctx *c, int64_t nJ, int32_t *votes,
                                           uint8_t *flags, int32_t *det_idx, int64_t *n_det,
                                           int32_t *union_idx, int64_t *n_union) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, nJ >= 0 && nJ <= 0x7fffffff, "bad |J|");
    USFFT_REQUIRE(c, nJ == 0 || (votes && flags && det_idx), "NULL pointer");
    USFFT_REQUIRE(c, n_det != nullptr || n_union == nullptr, "n_union without n_det");
    long long *counts = reinterpret_cast<long long *>(static_cast<char *>(c->dscal) + 64);
    // C3: union over the nodes of every rank (Step 2e P:318): all-reduce SUM of the votes
    if (comm_size(c) > 1 && nJ > 0)
        if (usfft_status s = comm_sum_i32(c, votes, nJ)) return s;
    if (nJ == 0) {
        if (n_det) *n_det = 0;
        if (n_union) *n_union = 0;
        return USFFT_OK;
    }
    k_union<<<1, 1024, 0, c->stream>>>(votes, nJ, flags, det_idx, union_idx, counts);
    USFFT_CHECK_LAUNCH(c);
    if (!n_det) return USFFT_OK;                          // asynchronous: the running flags are the output
    long long h[2];
    USFFT_CUDA(c, cudaMemcpyAsync(h, counts, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    USFFT_CUDA(c, cudaStreamSynchronize(c->stream));
    *n_det = h[0];
    if (n_union) *n_union = h[1];
    return USFFT_OK;
}

extern "C" usfft_status usfft_resolve(usfft_ctx *c, const usfft_lattice_desc *lat, int64_t G_loc,
                                      const double *spectra, const int32_t *bins, int64_t nJ,
                                      const int32_t *det_g, const int32_t *n_det_g, int32_t s_tilde,
                                      const int32_t *det_idx, int64_t n_det, double *coef,
                                      int32_t *lstar) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, lat != nullptr && lat->M >= 2 && lat->L >= 1 && lat->L <= 64, "bad lattice desc (L <= 64)");
    USFFT_REQUIRE(c, G_loc >= 0 && n_det >= 0 && s_tilde >= 1, "bad sizes");
    if (G_loc == 0 || n_det == 0) return USFFT_OK;
    USFFT_REQUIRE(c, spectra && bins && det_g && n_det_g && det_idx && coef, "NULL pointer");
    // as many lattices' occupancy tables as fit in ~96 KB (at least one)
    const int64_t per_l = (int64_t)sizeof(int) * lat->M;
    int32_t LC = (int32_t)std::max<int64_t>(1, std::min<int64_t>(lat->L, (96 * 1024 - 4 * (int64_t)s_tilde) / per_l));
    const size_t smem = (size_t)per_l * LC + sizeof(int) * (size_t)s_tilde;
    USFFT_REQUIRE(c, smem <= c->smem_optin, "M too large for the resolve occupancy table");
    int32_t *ls = lstar;
    if (!ls) {
        usfft_status s = ensure(c, &c->ws, &c->ws_size, sizeof(int32_t) * (size_t)G_loc * n_det);
        if (s) return s;
        ls = static_cast<int32_t *>(c->ws);
    }
    if (usfft_status s = kernel_fit(c, k_resolve, 0, smem, nullptr)) return s;
    k_resolve<<<(unsigned)G_loc, 256, smem, c->stream>>>(
        reinterpret_cast<const double2 *>(spectra), bins, nJ, lat->M, lat->L, det_g, n_det_g,
        s_tilde, det_idx, n_det, reinterpret_cast<double2 *>(coef), ls, LC);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

// Step 3 (Z26): coefficients of the frequencies assigned to one cover lattice
namespace usfft {
__global__ void k_cover_gather(int64_t M, int64_t G, const double2 *__restrict__ F,
                               const int32_t *__restrict__ idx, const int32_t *__restrict__ bin,
                               int64_t n, double2 *__restrict__ coef, int64_t nI) {
    const int64_t Mh = M / 2 + 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < G * n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = e / n, a = e - g * n;
        coef[g * nI + idx[a]] = spec_value(F + g * Mh, M, bin[a]);
    }
}
}  // namespace usfft

extern "C" usfft_status usfft_cover_gather(usfft_ctx *c, int64_t M, int64_t G, const double *spectra,
                                           const int32_t *idx, const int32_t *bin, int64_t n,
                                           double *coef, int64_t nI) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, M >= 2 && G >= 0 && n >= 0 && nI >= n, "bad sizes");
    if (G == 0 || n == 0) return USFFT_OK;
    USFFT_REQUIRE(c, spectra && idx && bin && coef, "NULL argument");
    k_cover_gather<<<grid1d(G * n, 256), 256, 0, c->stream>>>(
        M, G, reinterpret_cast<const double2 *>(spectra), idx, bin, n, reinterpret_cast<double2 *>(coef), nI);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

