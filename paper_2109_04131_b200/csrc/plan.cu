// plan.cu — the random round plan of Alg. 1 (usfft_plan_round, include/usfft.h).
//
// Step 1 & 2a: x'_j uniformly at random (j != t), line nodes l/K_t in slot t, K_t = 2N+1.
// Step 2: x'_{t+1..d} uniformly at random; sampling set for J_t from L rank-1 lattices
// (Algorithm A = random R1L).  The paper fixes neither the generator nor the sizes; the
// readings are DESIGN.md §3 Z2 (sizes), Z3 (z range), Z4 (counter-based SplitMix64 draws):
//   h = sm64(sm64(sm64(sm64(sm64(seed) ^ tag) ^ t) ^ i) ^ ((l << 20) ^ j))   (t, i, j 1-based)
//   x' = (h >> 11) * 2^-53,  z = 1 + h mod (M - 1);  tags 1/2 shifts, 3 z, 4|(M<<8) mode-R tries.
//   M = least prime >= max(4 s~, K+1) with M-1 7-smooth;  L = ceil(2 ln(2|J|)) rounded up to odd.
//   Mode R: such primes from max(2|J|, N+1) upward, 50 tries of z per prime, M <= 2^26; all 50
//   tries of one prime are tested in one launch (one bitset per try).
#include <algorithm>
#include <cmath>
#include <vector>

#include "lattice.cuh"

namespace usfft {

static inline uint64_t sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t seed, uint64_t tag, uint64_t t, uint64_t i, uint64_t l, uint64_t j) {
    uint64_t h = sm64(seed);
    h = sm64(h ^ tag);
    h = sm64(h ^ t);
    h = sm64(h ^ i);
    return sm64(h ^ ((l << 20) ^ j));
}

static inline double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

static bool prime(int64_t n) {
    if (n < 2) return false;
    if (n % 2 == 0) return n == 2;
    for (int64_t f = 3; f * f <= n; f += 2)
        if (n % f == 0) return false;
    return true;
}

static bool smooth7(int64_t n) {
    for (int64_t p : {2, 3, 5, 7})
        while (n > 1 && n % p == 0) n /= p;
    return n == 1;
}

static int64_t lattice_prime(int64_t lo) {
    int64_t p = lo < 3 ? 3 : lo;
    while (!(prime(p) && smooth7(p - 1))) ++p;
    return p;
}

}  // namespace usfft

using namespace usfft;

extern "C" usfft_status usfft_plan_round(usfft_ctx *c, const usfft_plan_in *in,
                                         const int16_t *I_prev, int64_t n_prev, const int16_t *kt,
                                         int32_t n1, usfft_plan_out *out) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, in && out, "NULL in/out");
    USFFT_REQUIRE(c, in->step == 1 || in->step == 2, "step must be 1 or 2");
    USFFT_REQUIRE(c, in->d >= 1 && in->d <= kMaxD, "d out of range");
    USFFT_REQUIRE(c, in->t >= 1 && in->t <= in->d, "t out of range");
    USFFT_REQUIRE(c, in->N >= 0 && in->s_tilde >= 1 && in->nJ >= 1, "N / s~ / |J|");
    const uint64_t seed = (uint64_t)in->seed, t = (uint64_t)in->t, i = (uint64_t)in->i;
    const int64_t K = 2 * (int64_t)in->N + 1;
    for (int j = 1; j <= in->d; ++j)
        out->shift[j - 1] = unit(draw(seed, in->step == 1 ? 1 : 2, t, i, 0, (uint64_t)j));
    if (in->step == 1) {                                    // line lattice z = 1, M = K_t
        out->M = K;
        out->L = 1;
        out->t_z = 1;
        out->line_axis = in->t - 1;
        out->z[0] = 1 % K;
        return USFFT_OK;
    }
    out->t_z = in->t;
    out->line_axis = -1;
    if (in->mode == 0) {                                    // mode A: L random R1Ls, shared M
        const int64_t M = lattice_prime(std::max<int64_t>(4 * (int64_t)in->s_tilde, K + 1));
        int64_t L = (int64_t)std::ceil(2.0 * std::log(2.0 * (double)in->nJ));
        if (L < 1) L = 1;
        if (L % 2 == 0) ++L;
        USFFT_REQUIRE(c, L * in->t <= kMaxZ, "L*t = %lld exceeds %d", (long long)(L * in->t), kMaxZ);
        out->M = M;
        out->L = (int32_t)L;
        for (int64_t l = 0; l < L; ++l)
            for (int j = 1; j <= in->t; ++j)
                out->z[l * in->t + (j - 1)] = 1 + (int64_t)(draw(seed, 3, t, i, (uint64_t)l, (uint64_t)j) % (uint64_t)(M - 1));
        return USFFT_OK;
    }
    // mode R: reconstructing single lattice for J_t, tries batched per prime
    USFFT_REQUIRE(c, in->mode == 1, "mode must be 0 (A) or 1 (R)");
    const int tries = 50;
    USFFT_REQUIRE(c, tries * in->t <= kMaxZ, "t too large for batched mode-R tries");
    usfft_lattice_desc desc;
    std::vector<int64_t> zt((size_t)tries * in->t);
    int64_t M = lattice_prime(std::max<int64_t>(2 * in->nJ, (int64_t)in->N + 1));
    std::vector<int32_t> inj(tries);
    while (M <= (int64_t(1) << 26)) {
        for (int r = 0; r < tries; ++r)
            for (int j = 1; j <= in->t; ++j)
                zt[(size_t)r * in->t + (j - 1)] =
                    1 + (int64_t)(draw(seed, 4ull | ((uint64_t)M << 8), t, i, (uint64_t)r, (uint64_t)j) % (uint64_t)(M - 1));
        desc.d = in->d;
        desc.t = in->t;
        desc.line_axis = -1;
        desc.L = tries;
        desc.M = M;
        desc.z = zt.data();
        desc.shift = out->shift;
        usfft_status s = usfft_lattice(c, &desc, 0, 0, nullptr, I_prev, n_prev, kt, n1, nullptr, inj.data());
        if (s != USFFT_OK && s != USFFT_ENOTRECON) return s;
        for (int r = 0; r < tries; ++r) {
            if (inj[r]) {
                out->M = M;
                out->L = 1;
                for (int j = 0; j < in->t; ++j) out->z[j] = zt[(size_t)r * in->t + j];
                c->err.clear();
                return USFFT_OK;
            }
        }
        M = lattice_prime(M + 1);
    }
    return fail(c, USFFT_ENOTRECON, "no reconstructing lattice with M <= 2^26");
}

// Step 3: multiple-R1L cover of I, reading Z26 (include/usfft.h).  Host only.
extern "C" usfft_status usfft_cover_plan(usfft_ctx *c, int64_t seed, int32_t d, int32_t N,
                                         const int16_t *I, int64_t nI, usfft_cover_desc *out,
                                         int32_t *assign, int32_t *bin) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, out && assign && bin && I, "NULL argument");
    USFFT_REQUIRE(c, d >= 1 && d <= 64 && N >= 0 && nI >= 1 && nI <= (int64_t(1) << 24), "bad sizes");
    const int64_t M = lattice_prime(std::max<int64_t>(4 * (nI - 1), (int64_t)N + 1));
    USFFT_REQUIRE(c, M < (int64_t(1) << 31), "cover lattice too large");
    out->nlat = 0;
    out->d = d;
    out->M = M;
    std::vector<int64_t> res((size_t)nI);
    std::vector<int32_t> cnt((size_t)M);
    for (int64_t a = 0; a < nI; ++a) assign[a] = -1;
    int64_t left = nI;
    int empty = 0;
    uint64_t attempt = 0;
    int64_t z[64];
    while (left > 0) {
        USFFT_REQUIRE(c, out->nlat < 64, "cover needs more than 64 lattices");
        const uint64_t q = (uint64_t)out->nlat + 1;
        for (int j = 1; j <= d; ++j)
            z[j - 1] = 1 + (int64_t)(draw((uint64_t)seed, 5, (uint64_t)d, q, attempt, (uint64_t)j) % (uint64_t)(M - 1));
        ++attempt;
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t a = 0; a < nI; ++a) {               // residues of the FULL set
            int64_t r = 0;
            for (int j = 0; j < d; ++j) r = (r + (int64_t)I[a * d + j] * z[j]) % M;
            if (r < 0) r += M;
            res[(size_t)a] = r;
            ++cnt[(size_t)r];
        }
        int64_t got = 0;
        for (int64_t a = 0; a < nI; ++a)
            if (assign[a] < 0 && cnt[(size_t)res[(size_t)a]] == 1) {
                assign[a] = out->nlat;
                bin[a] = (int32_t)res[(size_t)a];
                ++got;
            }
        if (got == 0) {
            if (++empty > 100) return fail(c, USFFT_ENOTRECON, "cover: 100 consecutive empty draws");
            continue;
        }
        empty = 0;
        attempt = 0;
        for (int j = 0; j < d; ++j) out->z[(int64_t)out->nlat * d + j] = z[j];
        ++out->nlat;
        left -= got;
    }
    return USFFT_OK;
}


// Z27: the global pole shift of the phi_Delta periodization, Delta = 1 / (4 M0) with M0 the
// Step-2 lattice size of the run (Lemma P:847-870, "Delta_opt = 1/(4M)"; every Step-2 round
// shares M0 = the Z2 lattice size for s_local).
extern "C" usfft_status usfft_plan_delta(usfft_ctx *c, int32_t N, int32_t s_local, int32_t lattice_factor,
                                         double *delta) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, N >= 0 && s_local >= 1 && lattice_factor >= 1 && delta, "bad arguments");
    const int64_t K = 2 * (int64_t)N + 1;
    const int64_t M0 = lattice_prime(std::max<int64_t>(4 * (int64_t)s_local * lattice_factor, K + 1));
    *delta = 1.0 / (4.0 * (double)M0);
    return USFFT_OK;
}
