// lattice.cuh — rank-1 lattice node rule (eq. lattice_nodes; Alg. 1 Step 2b P:309-311;
// Step 1 line nodes P:288-293) as a device function, plus the host-side descriptor check.
#pragma once
#include "common.cuh"

namespace usfft {

// y_{b,j} for sample b = l*M + i of the round:
//   Step 2 (line_axis < 0): ((i * z_{l,j}) mod M) / M for j < t, else shift_j
//   Step 1 (line_axis = a):  ((i * z_{l,0}) mod M) / M for j == a, else shift_j
// (i*z) < 2^52 is exact in int64; the quotient is one IEEE division (bit-exact with any
// correctly rounded implementation).
__device__ __forceinline__ double lattice_node(const LatParams &P, int64_t b, int j) {
    const int64_t l = b / P.M;
    const int64_t i = b - l * P.M;
    if (P.line_axis >= 0) {
        if (j == P.line_axis) return (double)((i * (int64_t)P.z[l * P.t]) % P.M) / (double)P.M;
        return P.shift[j];
    }
    if (j < P.t) return (double)((i * (int64_t)P.z[l * P.t + j]) % P.M) / (double)P.M;
    return P.shift[j];
}

inline usfft_status make_lat_params(usfft_ctx *c, const usfft_lattice_desc *L, LatParams *P) {
    USFFT_REQUIRE(c, L != nullptr, "lattice desc is NULL");
    USFFT_REQUIRE(c, L->d >= 1 && L->d <= kMaxD, "d = %d out of [1, %d]", L->d, kMaxD);
    USFFT_REQUIRE(c, L->t >= 1 && L->t <= L->d, "t = %d out of [1, d]", L->t);
    USFFT_REQUIRE(c, L->L >= 1 && (int64_t)L->L * L->t <= kMaxZ, "L*t = %lld exceeds %d",
                  (long long)L->L * L->t, kMaxZ);
    USFFT_REQUIRE(c, L->M >= 2 && L->M <= (int64_t(1) << 26), "M = %lld out of [2, 2^26]",
                  (long long)L->M);
    USFFT_REQUIRE(c, L->line_axis < L->d, "line_axis %d >= d", L->line_axis);
    USFFT_REQUIRE(c, L->line_axis < 0 || L->t == 1, "Step-1 line lattice needs t == 1");
    USFFT_REQUIRE(c, L->z != nullptr && L->shift != nullptr, "z / shift are NULL");
    P->d = L->d;
    P->t = L->t;
    P->line_axis = L->line_axis;
    P->L = L->L;
    P->M = L->M;
    for (int k = 0; k < L->L * L->t; ++k) {
        USFFT_REQUIRE(c, L->z[k] >= 0 && L->z[k] < L->M, "z[%d] = %lld not in [0, M)", k,
                      (long long)L->z[k]);
        P->z[k] = (int32_t)L->z[k];
    }
    for (int j = 0; j < L->d; ++j) {
        USFFT_REQUIRE(c, L->shift[j] >= 0.0 && L->shift[j] < 1.0, "shift[%d] not in [0,1)", j);
        P->shift[j] = L->shift[j];
    }
    return USFFT_OK;
}

}  // namespace usfft
