// fft400.cuh — K6 for M = 401 (config 2's lattice size): Rader's algorithm (rader.cuh) with the
// two length-400 FFTs done as register-resident four-step transforms, 400 = 20 x 20.
//
// One warp per (node, lattice) row; lanes 0..19 carry the transform.  Forward FFT of a (lane n2
// holds a[20 n1 + n2], n1 = 0..19 in registers):
//   A[k1 + 20 k2] = sum_{n2} W20^{n2 k2} W400^{n2 k1} sum_{n1} a[20 n1 + n2] W20^{n1 k1}
// = a DFT-20 in registers, a twiddle, ONE shared-memory transpose, a DFT-20 in registers; the
// result sits in lane k1, register k2.  That is again the input layout of the second transform
// (lane = index mod 20, register = index div 20), so the pointwise product with FFT(b)/N and the
// second FFT (the inverse, done as conj(FFT(conj .))) need no exchange before their own single
// transpose.  Shared-memory traffic per row: the staged input, two transposes and the output
// scatter, instead of two reads and two writes per Stockham stage (8 stages) in rader_t.cuh.
// DFT-20 = 5 DFT-4 + 12 twiddles + 4 DFT-5 (radix split 20 = 4 x 5), constants folded.
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

// four-step FFT-400 core: v (lane n2 = index mod 20, register = index div 20) -> out (lane k1,
// register k2 holds X[k1 + 20 k2]).  T: the warp's [20][21] transpose buffer.
__device__ __forceinline__ void fft400_core(double2 (&v)[20], double2 (&out)[20], double2 *T,
                                            const double2 *__restrict__ tw400, int lane) {
    double2 y[20];
    if (lane < 20) {
        f20::dft20(v, y);
#pragma unroll
        for (int k1 = 1; k1 < 20; ++k1) y[k1] = cmul(y[k1], __ldg(tw400 + lane * k1));   // W400^{n2 k1}
#pragma unroll
        for (int k1 = 0; k1 < 20; ++k1) T[k1 * 21 + lane] = y[k1];
    }
    __syncwarp();
    if (lane < 20) {
#pragma unroll
        for (int n2 = 0; n2 < 20; ++n2) v[n2] = T[lane * 21 + n2];
        f20::dft20(v, out);
    }
    __syncwarp();
}

template <int RPC>
__global__ void __launch_bounds__(32 * RPC)
k_fft400(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int32_t L,
         const RaderArgs A, double2 *__restrict__ F, int64_t rows) {
    constexpr int M = 401, MH = 201, PER = (M + 31) / 32;
    constexpr int XS = 402;                               // staged real row (doubles, padded)
    constexpr int WB = XS / 2 + 20 * 21;                  // double2 per warp: row + transpose / output
    extern __shared__ double2 sm4[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *xs = reinterpret_cast<double *>(sm4 + (size_t)w * WB);
    double2 *T = sm4 + (size_t)w * WB + XS / 2;           // transpose buffer, then output staging
    const bool one_slab = S.nslab == 1;
    const int64_t stride = (int64_t)gridDim.x * RPC;
    int64_t row = (int64_t)blockIdx.x * RPC + w;
    double xv[PER];
    auto fetch = [&](int64_t rw) {
        const int64_t g = rw / L, l = rw - g * L;
        if (one_slab) {
            const double *src = u + g * (int64_t)L * M + l * M;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = lane + 32 * k;
                xv[k] = i < M ? __ldg(src + i) : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = lane + 32 * k;
                xv[k] = i < M ? sample_at(u, S, G_loc, g, l * M + i) : 0.0;
            }
        }
    };
    if (row < rows) fetch(row);
    for (; row < rows; row += stride) {
        double part = 0.0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = lane + 32 * k;
            if (i < M) xs[i] = xv[k];
            part += xv[k];
        }
        if (row + stride < rows) fetch(row + stride);     // overlaps the transforms below
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);   // X[0]
        __syncwarp();
        const double x0 = xs[0];
        double2 v[20], a[20];
        if (lane < 20) {
#pragma unroll
            for (int n1 = 0; n1 < 20; ++n1) v[n1] = make_double2(xs[__ldg(A.perm + 20 * n1 + lane)], 0.0);
        }
        fft400_core(v, a, T, A.tw, lane);                 // a: lane k1, register k2
        if (lane < 20) {
#pragma unroll
            for (int k2 = 0; k2 < 20; ++k2) {             // conj(A . FFT(b)/N)
                const double2 c = cmul(a[k2], __ldg(A.bf + lane + 20 * k2));
                v[k2] = make_double2(c.x, -c.y);
            }
        }
        fft400_core(v, a, T, A.tw, lane);                 // conj of N IFFT(A . bf)
        if (lane < 20) {
#pragma unroll
            for (int k2 = 0; k2 < 20; ++k2) {             // X[g^-q] = x0 + conv[q], bins <= M/2
                const int m = __ldg(A.outidx + lane + 20 * k2);
                if (m < MH) T[m] = make_double2(x0 + a[k2].x, -a[k2].y);
            }
        }
        __syncwarp();
        double2 *dst = F + row * MH;
        for (int m = lane; m < MH; m += 32) dst[m] = m == 0 ? make_double2(part, 0.0) : T[m];
        __syncwarp();                                     // buffers are reused by the next row
    }
}

// Two real rows per complex transform: z = a0 + i a1, the Rader sequences of the lattices
// 2j and 2j+1 of one node g (pairs never straddle nodes, so a row's result does not depend on
// how the nodes are split across ranks or launches; an odd L leaves its last lattice paired
// with a zero row).  By linearity FFT(z) . FFT(b)/N = C0 + i C1 (C_j = FFT(a_j) . FFT(b)/N), so
// the spectra need no separation; the second transform of conj(C0 + i C1) gives
// D = conj(conv0) - i conj(conv1), whose halves separate because each row's convolution
// satisfies conv[q + N/2] = conj(conv[q]) (k_fft_rader_tp in rader_t.cuh):
// conj(conv0[q]) = (D[q] + conj D[q+200]) / 2, conj(conv1[q]) = (conj D[q+200] - D[q]) / 2i.
template <int RPC>
__global__ void __launch_bounds__(32 * RPC)
k_fft400p(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int32_t L,
          const RaderArgs A, double2 *__restrict__ F, int64_t rows) {
    constexpr int M = 401, MH = 201, PER = (M + 31) / 32;
    constexpr int XS = 402;                               // one staged real row (doubles, padded)
    constexpr int WB = XS + 20 * 21;                      // double2 per warp: two rows + transpose
    extern __shared__ double2 sm4[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *xs0 = reinterpret_cast<double *>(sm4 + (size_t)w * WB), *xs1 = xs0 + XS;
    double2 *T = sm4 + (size_t)w * WB + XS;               // transpose buffer, then output staging
    const bool one_slab = S.nslab == 1;
    const int64_t LP = (L + 1) / 2, pairs = (rows / L) * LP;     // rows = G_loc * L
    const int64_t stride = (int64_t)gridDim.x * RPC;
    int64_t pr = (int64_t)blockIdx.x * RPC + w;
    double xv0[PER], xv1[PER];
    auto fetch1 = [&](int64_t rw, double (&xv)[PER]) {
        if (rw < 0) {
#pragma unroll
            for (int k = 0; k < PER; ++k) xv[k] = 0.0;
            return;
        }
        const int64_t g = rw / L, l = rw - g * L;
        if (one_slab) {
            const double *src = u + g * (int64_t)L * M + l * M;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = lane + 32 * k;
                xv[k] = i < M ? __ldg(src + i) : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = lane + 32 * k;
                xv[k] = i < M ? sample_at(u, S, G_loc, g, l * M + i) : 0.0;
            }
        }
    };
    // rows of pair q: (g, 2j) and (g, 2j+1) with g = q / LP, j = q % LP (-1: the zero row)
    auto row0 = [&](int64_t q) { return (q / LP) * L + 2 * (q % LP); };
    auto row1 = [&](int64_t q) { return 2 * (q % LP) + 1 < L ? row0(q) + 1 : int64_t(-1); };
    if (pr < pairs) {
        fetch1(row0(pr), xv0);
        fetch1(row1(pr), xv1);
    }
    for (; pr < pairs; pr += stride) {
        const int64_t r0 = row0(pr), r1 = row1(pr);
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = lane + 32 * k;
            if (i < M) {
                xs0[i] = xv0[k];
                xs1[i] = xv1[k];
            }
            p0 += xv0[k];
            p1 += xv1[k];
        }
        if (pr + stride < pairs) {                        // overlaps the transforms below
            fetch1(row0(pr + stride), xv0);
            fetch1(row1(pr + stride), xv1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {                // X[0] of both rows
            p0 += __shfl_xor_sync(0xffffffffu, p0, o);
            p1 += __shfl_xor_sync(0xffffffffu, p1, o);
        }
        __syncwarp();
        const double x00 = xs0[0], x01 = xs1[0];
        double2 v[20], a[20];
        if (lane < 20) {
#pragma unroll
            for (int n1 = 0; n1 < 20; ++n1) {
                const int pi = __ldg(A.perm + 20 * n1 + lane);
                v[n1] = make_double2(xs0[pi], xs1[pi]);
            }
        }
        fft400_core(v, a, T, A.tw, lane);                 // Z: lane k1, register k2
        if (lane < 20) {
#pragma unroll
            for (int k2 = 0; k2 < 20; ++k2) {             // conj(Z . FFT(b)/N)
                const double2 c = cmul(a[k2], __ldg(A.bf + lane + 20 * k2));
                v[k2] = make_double2(c.x, -c.y);
            }
        }
        fft400_core(v, a, T, A.tw, lane);                 // D = conj(conv0) - i conj(conv1)
        if (lane < 20) {
#pragma unroll
            for (int k2 = 0; k2 < 10; ++k2) {             // q = lane + 20 k2 < 200, q + 200 in register k2 + 10
                const double2 dq = a[k2], dh = a[k2 + 10];
                const double2 s = make_double2(0.5 * (dq.x + dh.x), 0.5 * (dq.y - dh.y));      // conj(conv0)
                const double2 tt = make_double2(0.5 * (dh.x - dq.x), 0.5 * (-dh.y - dq.y));    // conj(conv1) = -i tt
                const int m = __ldg(A.outidx + lane + 20 * k2);
                if (m < MH) {                             // X[g^-q] = x0 + conv[q]
                    T[m] = make_double2(x00 + s.x, -s.y);
                    T[MH + m] = make_double2(x01 + tt.y, tt.x);
                } else {                                  // q + 200 maps to M - m <= M/2
                    T[M - m] = make_double2(x00 + s.x, s.y);
                    T[MH + M - m] = make_double2(x01 + tt.y, -tt.x);
                }
            }
        }
        __syncwarp();
        double2 *dst0 = F + r0 * MH;
        for (int m = lane; m < MH; m += 32) dst0[m] = m == 0 ? make_double2(p0, 0.0) : T[m];
        if (r1 >= 0) {
            double2 *dst1 = F + r1 * MH;
            for (int m = lane; m < MH; m += 32) dst1[m] = m == 0 ? make_double2(p1, 0.0) : T[MH + m];
        }
        __syncwarp();                                     // buffers are reused by the next pair
    }
}

}  // namespace usfft
