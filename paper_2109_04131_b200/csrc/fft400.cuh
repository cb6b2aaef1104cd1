// fft400.cuh — register DFT-20 codelet (20 = 4 x 5, constants folded) used by the register-radix
// lattice FFT (fft_r.cuh).  The earlier one-warp-per-row four-step kernels for M = 401 were
// replaced by k_fft_rader_r (0.088 -> 0.075 ms at config 2's shape, profiles/r2_fft_bench.txt).
// DFT-20 = 5 DFT-4 + 12 twiddles + 4 DFT-5 (radix split 20 = 4 x 5).
#pragma once

namespace usfft {
namespace f20 {
constexpr double C1 = 0.95105651629515357212, S1 = 0.30901699437494742410;   // cos / sin(2 pi / 20)
constexpr double C2 = 0.80901699437494742410, S2 = 0.58778525229247312917;   // cos / sin(4 pi / 20)
// W20^j = e^{-2 pi i j / 20} = wc[j] - i ws[j]
__device__ constexpr double wc[20] = {1, C1, C2, S2, S1, 0, -S1, -S2, -C2, -C1,
                                      -1, -C1, -C2, -S2, -S1, 0, S1, S2, C2, C1};
__device__ constexpr double ws[20] = {0, S1, S2, C2, C1, 1, C1, C2, S2, S1,
                                      0, -S1, -S2, -C2, -C1, -1, -C1, -C2, -S2, -S1};

__device__ __forceinline__ double2 mulw(double2 a, int j) {           // a * W20^j, j constant
    j %= 20;
    if (j == 0) return a;
    return make_double2(fma(a.x, wc[j], a.y * ws[j]), fma(a.y, wc[j], -a.x * ws[j]));
}

// out[k] = sum_n v[n] W20^{n k}:  n = 5 na + nb, k = ka + 4 kb
__device__ __forceinline__ void dft20(const double2 (&v)[20], double2 (&out)[20]) {
    double2 y[5][4];
#pragma unroll
    for (int nb = 0; nb < 5; ++nb) {                                     // DFT-4 over na
        const double2 a0 = v[nb], a1 = v[5 + nb], a2 = v[10 + nb], a3 = v[15 + nb];
        const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
        y[nb][0] = cadd(s02, s13);
        y[nb][2] = csub(s02, s13);
        y[nb][1] = make_double2(d02.x + d13.y, d02.y - d13.x);           // d02 - i d13
        y[nb][3] = make_double2(d02.x - d13.y, d02.y + d13.x);           // d02 + i d13
#pragma unroll
        for (int ka = 1; ka < 4; ++ka) y[nb][ka] = mulw(y[nb][ka], nb * ka);
    }
    constexpr double K1 = 0.30901699437494742410, K2 = -0.80901699437494742410;   // cos 2pi/5, 4pi/5
    constexpr double Q1 = 0.95105651629515357212, Q2 = 0.58778525229247312917;    // sin 2pi/5, 4pi/5
#pragma unroll
    for (int ka = 0; ka < 4; ++ka) {                                     // DFT-5 over nb
        const double2 x0 = y[0][ka], t1 = cadd(y[1][ka], y[4][ka]), t2 = cadd(y[2][ka], y[3][ka]);
        const double2 t3 = csub(y[1][ka], y[4][ka]), t4 = csub(y[2][ka], y[3][ka]);
        const double2 a1 = make_double2(fma(K2, t2.x, fma(K1, t1.x, x0.x)), fma(K2, t2.y, fma(K1, t1.y, x0.y)));
        const double2 a2 = make_double2(fma(K1, t2.x, fma(K2, t1.x, x0.x)), fma(K1, t2.y, fma(K2, t1.y, x0.y)));
        const double2 b1 = make_double2(fma(Q2, t4.x, Q1 * t3.x), fma(Q2, t4.y, Q1 * t3.y));
        const double2 b2 = make_double2(fma(-Q1, t4.x, Q2 * t3.x), fma(-Q1, t4.y, Q2 * t3.y));
        out[ka] = cadd(x0, cadd(t1, t2));
        out[ka + 4] = make_double2(a1.x + b1.y, a1.y - b1.x);            // a1 - i b1
        out[ka + 16] = make_double2(a1.x - b1.y, a1.y + b1.x);           // a1 + i b1
        out[ka + 8] = make_double2(a2.x + b2.y, a2.y - b2.x);            // a2 - i b2
        out[ka + 12] = make_double2(a2.x - b2.y, a2.y + b2.x);           // a2 + i b2
    }
}
}  // namespace f20
}  // namespace usfft
