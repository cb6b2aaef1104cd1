// fft_r.cuh — K6 for the Step-2 lattice sizes M = 401 and 4001 (configs 2 and 5; N = M-1 = 400,
// 4000): Rader's algorithm (rader.cuh) on row pairs, the two length-N FFTs as register-radix
// Stockham passes (N = 20 x 20 and 20 x 20 x 10), in place in ONE shared buffer per row pair.
//
// Two real rows share one complex transform by linearity (rader_t.cuh, k_fft_rader_tp): with
// z = a0 + i a1 the two Rader sequences, D = FFT(conj(FFT(z) . FFT(b)/N)) and
//   conj(conv0[q]) = (D[q] + conj D[q + N/2]) / 2,   conj(conv1[q]) = (conj D[q + N/2] - D[q]) / 2i,
// X_j[g^-q] = x0_j + conv_j[q] for q < N/2 covers every bin pair {m, M - m}.
//
// A pass of radix R loads the R inputs of each of its butterflies into registers (stride N/R),
// waits until every thread of the pair has loaded (the pass runs in place), applies the
// Stockham twiddles W_{Ns R}^{(j mod Ns) r} from the exact-index table, a register DFT-R
// (20 = 4 x 5, 10 = 2 x 5, constants folded), and stores the R outputs (stride Ns).  Fused into
// the passes: the Rader permutation a_p = z[g^p] (first pass of FFT 1 gathers through perm),
// the pointwise product with FFT(b)/N and the conjugation (last pass of FFT 1), and the split
// of the two rows with the output permutation g^-q (last pass of FFT 2: with Ns = N/R the
// outputs of a butterfly are D[jm + Ns s], s < R, so D[q] and D[q + N/2] sit in one thread).
// Shared-memory traffic per pair: the staged input, 2 x P passes (read + write) and the output
// staging, against 2 x (number of radix-2..7 stages) passes of the ping-pong Stockham kernels.
// NPAIR pairs per CTA, GROUP threads per pair (pairs may straddle warps; every barrier is
// CTA-wide and every pair takes the same path), persistent grid over the pairs.
#pragma once

namespace usfft {
namespace fr {

// out[k] = sum_n v[n] W5^{nk}
__device__ __forceinline__ void dft5(const double2 &x0, const double2 &x1, const double2 &x2, const double2 &x3,
                                     const double2 &x4, double2 &o0, double2 &o1, double2 &o2, double2 &o3,
                                     double2 &o4) {
    constexpr double K1 = 0.30901699437494742410, K2 = -0.80901699437494742410;   // cos 2pi/5, 4pi/5
    constexpr double Q1 = 0.95105651629515357212, Q2 = 0.58778525229247312917;    // sin 2pi/5, 4pi/5
    const double2 t1 = cadd(x1, x4), t2 = cadd(x2, x3), t3 = csub(x1, x4), t4 = csub(x2, x3);
    const double2 a1 = make_double2(fma(K2, t2.x, fma(K1, t1.x, x0.x)), fma(K2, t2.y, fma(K1, t1.y, x0.y)));
    const double2 a2 = make_double2(fma(K1, t2.x, fma(K2, t1.x, x0.x)), fma(K1, t2.y, fma(K2, t1.y, x0.y)));
    const double2 b1 = make_double2(fma(Q2, t4.x, Q1 * t3.x), fma(Q2, t4.y, Q1 * t3.y));
    const double2 b2 = make_double2(fma(-Q1, t4.x, Q2 * t3.x), fma(-Q1, t4.y, Q2 * t3.y));
    o0 = cadd(x0, cadd(t1, t2));
    o1 = make_double2(a1.x + b1.y, a1.y - b1.x);                        // a1 - i b1
    o4 = make_double2(a1.x - b1.y, a1.y + b1.x);                        // a1 + i b1
    o2 = make_double2(a2.x + b2.y, a2.y - b2.x);                        // a2 - i b2
    o3 = make_double2(a2.x - b2.y, a2.y + b2.x);                        // a2 + i b2
}

// out[k] = sum_n v[n] W10^{nk}:  n = 5 na + nb, k = ka + 2 kb
__device__ __forceinline__ void dft10(const double2 (&v)[10], double2 (&out)[10]) {
    double2 y0[5], y1[5];
#pragma unroll
    for (int nb = 0; nb < 5; ++nb) {
        y0[nb] = cadd(v[nb], v[5 + nb]);
        y1[nb] = f20::mulw(csub(v[nb], v[5 + nb]), 2 * nb);             // W10^{nb} = W20^{2 nb}
    }
    dft5(y0[0], y0[1], y0[2], y0[3], y0[4], out[0], out[2], out[4], out[6], out[8]);
    dft5(y1[0], y1[1], y1[2], y1[3], y1[4], out[1], out[3], out[5], out[7], out[9]);
}

__device__ __forceinline__ void dft4(const double2 &a0, const double2 &a1, const double2 &a2, const double2 &a3,
                                     double2 &o0, double2 &o1, double2 &o2, double2 &o3) {
    const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
    o0 = cadd(s02, s13);
    o2 = csub(s02, s13);
    o1 = make_double2(d02.x + d13.y, d02.y - d13.x);                    // d02 - i d13
    o3 = make_double2(d02.x - d13.y, d02.y + d13.x);                    // d02 + i d13
}

// out[k] = sum_n v[n] W8^{nk}: even / odd DFT-4, W8^k combine
__device__ __forceinline__ void dft8(const double2 (&v)[8], double2 (&out)[8]) {
    constexpr double H = 0.70710678118654752440;                      // cos(pi/4)
    double2 e0, e1, e2, e3, o0, o1, o2, o3;
    dft4(v[0], v[2], v[4], v[6], e0, e1, e2, e3);
    dft4(v[1], v[3], v[5], v[7], o0, o1, o2, o3);
    const double2 t1 = make_double2(H * (o1.x + o1.y), H * (o1.y - o1.x));      // W8^1 o1
    const double2 t2 = make_double2(o2.y, -o2.x);                              // W8^2 o2 = -i o2
    const double2 t3 = make_double2(H * (o3.y - o3.x), -H * (o3.x + o3.y));     // W8^3 o3
    out[0] = cadd(e0, o0);
    out[4] = csub(e0, o0);
    out[1] = cadd(e1, t1);
    out[5] = csub(e1, t1);
    out[2] = cadd(e2, t2);
    out[6] = csub(e2, t2);
    out[3] = cadd(e3, t3);
    out[7] = csub(e3, t3);
}

template <int R>
__device__ __forceinline__ void dft(const double2 (&v)[R], double2 (&out)[R]) {
    static_assert(R == 4 || R == 5 || R == 8 || R == 10 || R == 20, "register radix 4, 5, 8, 10, 20");
    if constexpr (R == 20) f20::dft20(v, out);
    else if constexpr (R == 10) dft10(v, out);
    else if constexpr (R == 8) dft8(v, out);
    else if constexpr (R == 5) dft5(v[0], v[1], v[2], v[3], v[4], out[0], out[1], out[2], out[3], out[4]);
    else dft4(v[0], v[1], v[2], v[3], out[0], out[1], out[2], out[3]);
}

enum { PLAIN = 0, GATHER = 1, MULBF = 2, SPLIT = 3 };

struct SplitOut {           // last pass of FFT 2: staged spectra of the two rows
    double2 *st;            // [2][MH]
    double x00, x01;        // x_0 of the two rows
    int MH, M;
    double2 *x0sum;         // (X0[0], X1[0]), written by the last pass of FFT 1
};

// physical slot of logical index k after the first pass: that pass stores its output s-major,
// T[s][j] with row stride N/R0 + 1 (its natural stores, stride R0 across lanes, would hit only
// 8 / gcd(R0, 8) of the 8 16-byte bank groups); the second pass reads through this map
template <int N, int R0>
__device__ __forceinline__ int tslot(int k) { return (k % R0) * (N / R0 + 1) + k / R0; }

// one in-place radix-R pass over a pair's buffer; t = thread index within the pair's group
template <int N, int R, int NS, int GROUP, int MODE, int R0>
__device__ __forceinline__ void pass(double2 *buf, const RaderArgs &A, int t, const SplitOut &so) {
    constexpr int NBF = N / R, BPT = (NBF + GROUP - 1) / GROUP, TSTEP = N / (NS * R);
    constexpr bool STORE_T = NS == 1, LOAD_T = NS == R0 && NS > 1;
    constexpr int M = N + 1;
    double2 v[BPT][R];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int j = t + b * GROUP;
        if (j < NBF) {
            // GATHER: a_{j + r NBF} = z[g^{j + r NBF}], g^{j + r NBF} = g^j (g^NBF)^r mod M
            int gp = MODE == GATHER ? A.perm[j] : 0;
            const int gstep = MODE == GATHER ? A.perm[NBF] : 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int idx = j + r * NBF;
                if (MODE == GATHER) {
                    UB_CHECK(gp >= 1 && gp < M);
                    v[b][r] = buf[gp];
                    gp = (gp * gstep) % M;
                } else {
                    UB_CHECK(idx < N && (!LOAD_T || tslot<N, R0>(idx) < N + R0));
                    v[b][r] = buf[LOAD_T ? tslot<N, R0>(idx) : idx];
                }
            }
        }
    }
    __syncthreads();                                      // in place: every input is in registers
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int j = t + b * GROUP;
        if (j >= NBF) continue;
        const int jm = j % NS;
        if (NS > 1) {   // W^r by recurrence from one table load (relative error <= R ulp)
            const double2 w1 = A.tw[jm * TSTEP];
            double2 wr = w1;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                v[b][r] = cmul(v[b][r], wr);
                if (r + 1 < R) wr = cmul(wr, w1);
            }
        }
        double2 y[R];
        dft<R>(v[b], y);
        const int base = (j / NS) * NS * R + jm;
        if (MODE == SPLIT) {
            static_assert(MODE != SPLIT || (NS * R == N && R % 2 == 0), "split needs the last pass");
            int m = A.outidx[jm];                                 // g^-(jm + NS s) = g^-jm (g^-NS)^s mod M
            const int mstep = A.outidx[NS];
#pragma unroll
            for (int s = 0; s < R / 2; ++s) {
                const int q = base + s * NS;                      // q < N/2; D[q + N/2] = y[s + R/2]
                const double2 dq = y[s], dh = y[s + R / 2];
                const double2 c0 = make_double2(0.5 * (dq.x + dh.x), 0.5 * (dq.y - dh.y));       // conj(conv0)
                const double2 c1 = make_double2(0.5 * (dh.x - dq.x), 0.5 * (-dh.y - dq.y));      // i conj(conv1)
                (void)q;
                UB_CHECK(m >= 1 && m < so.M && q < N / 2);
                if (m < so.MH) {
                    so.st[m] = make_double2(so.x00 + c0.x, -c0.y);
                    so.st[so.MH + m] = make_double2(so.x01 + c1.y, c1.x);
                } else {
                    so.st[so.M - m] = make_double2(so.x00 + c0.x, c0.y);
                    so.st[so.MH + so.M - m] = make_double2(so.x01 + c1.y, -c1.x);
                }
                m = (m * mstep) % M;
            }
        } else {
#pragma unroll
            for (int s = 0; s < R; ++s) {
                const int k = base + s * NS;
                double2 o = y[s];
                if (MODE == MULBF && k == 0) *so.x0sum = make_double2(so.x00 + o.x, so.x01 + o.y);
                if (MODE == MULBF) {                              // P = conj(Z . FFT(b)/N)
                    const double2 c = cmul(o, A.bf[k]);
                    o = make_double2(c.x, -c.y);
                }
                UB_CHECK(k < N && (!STORE_T || s * (NBF + 1) + j < N + R0));
                buf[STORE_T ? s * (NBF + 1) + j : k] = o;
            }
        }
    }
    __syncthreads();
}

// FFT_N over the radix list Rs (product N); the first pass in mode FIRST, the last in LAST
template <int N, int GROUP, int FIRST, int LAST, int R0, int NS, int R, int... Rest>
__device__ __forceinline__ void fft_passes(double2 *buf, const RaderArgs &A, int t, const SplitOut &so) {
    if constexpr (sizeof...(Rest) == 0) {
        static_assert(NS * R == N && NS > 1, "radix list must multiply to N (at least two passes)");
        pass<N, R, NS, GROUP, LAST, R0>(buf, A, t, so);
    } else {
        pass<N, R, NS, GROUP, (NS == 1 ? FIRST : PLAIN), R0>(buf, A, t, so);
        fft_passes<N, GROUP, FIRST, LAST, R0, NS * R, Rest...>(buf, A, t, so);
    }
}
template <int R0, int... Rs>
struct First { static constexpr int value = R0; };
}  // namespace fr

// streaming row loads that do not allocate in L1 (the FFT(b) and index tables should stay there)
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int N, int GROUP, int NPAIR, int MINB, int... Rs>
__global__ void __launch_bounds__(GROUP * NPAIR, MINB)
k_fft_rader_r(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int32_t L,
              const RaderArgs A, double2 *__restrict__ F, int64_t rows) {
    constexpr int M = N + 1, MH = M / 2 + 1, R0 = fr::First<Rs...>::value;
    constexpr int NB = 2 * MH > N + R0 ? 2 * MH : N + R0;  // staged pair (M), transposed pass (N + R0), output (2 MH)
    extern __shared__ double2 smf[];
    __shared__ double2 xz[NPAIR];                         // (X0[0], X1[0]) of each pair
    const int tid = threadIdx.x, pi = tid / GROUP, t = tid % GROUP;
    double2 *buf = smf + (size_t)pi * NB;
    const bool one_slab = S.nslab == 1;
    const int64_t LP = (L + 1) / 2, pairs = (rows / L) * LP;         // rows = G_loc * L
    auto row0 = [&](int64_t q) { return (q / LP) * L + 2 * (q % LP); };
    auto row1 = [&](int64_t q) { return 2 * (q % LP) + 1 < L ? row0(q) + 1 : int64_t(-1); };
    auto at = [&](int64_t rw, const double *src, int i) -> double {
        if (rw < 0) return 0.0;
        if (one_slab) return ld_stream(src + i);
        const int64_t g = rw / L, l = rw - g * L;
        return sample_at(u, S, G_loc, g, l * M + i);
    };
    // the FFT(b)/N table (16 N bytes, shared by every pair) into L1 once per CTA
    for (int k = tid * 8; k < N; k += GROUP * NPAIR * 8)
        asm volatile("prefetch.global.L1 [%0];" :: "l"(A.bf + k));
    // every pair of the CTA runs the same number of rounds (idle pairs transform zeros, not stored)
    const int64_t rounds = (pairs + (int64_t)gridDim.x * NPAIR - 1) / ((int64_t)gridDim.x * NPAIR);
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t pr = (rd * gridDim.x + blockIdx.x) * NPAIR + pi;
        const bool live = pr < pairs;
        const int64_t r0 = live ? row0(pr) : -1, r1 = live ? row1(pr) : -1;
        {   // z = x0 + i x1: every load of the pair issued before the first store (streaming, no L1 allocation)
            const double *src0 = u + (r0 < 0 ? 0 : r0 * (int64_t)M), *src1 = u + (r1 < 0 ? 0 : r1 * (int64_t)M);
            constexpr int PER = (M + GROUP - 1) / GROUP;
            double xa[PER], xb[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = t + k * GROUP;
                xa[k] = i < M ? at(r0, src0, i) : 0.0;
                xb[k] = i < M ? at(r1, src1, i) : 0.0;
            }
            // the next round's rows towards L2 while this pair is transformed (one 128-byte line per
            // thread and step; the rows of a pair are contiguous within a slab)
            const int64_t pn = ((rd + 1) * gridDim.x + blockIdx.x) * NPAIR + pi;
            if (one_slab && pn < pairs) {
                const int64_t rn = row0(pn);
                const char *nx = reinterpret_cast<const char *>(u + rn * (int64_t)M);
                const int nbytes = (row1(pn) >= 0 ? 2 : 1) * M * 8;
                for (int o = t * 128; o < nbytes; o += GROUP * 128)
                    asm volatile("prefetch.global.L2 [%0];" :: "l"(nx + o));
            }
#pragma unroll
            for (int k = 0; k < PER; ++k)
                if (t + k * GROUP < M) buf[t + k * GROUP] = make_double2(xa[k], xb[k]);
        }
        __syncthreads();
        const double2 z0 = buf[0];
        // X_j[0] = x0_j + sum_p a_p = x0_j + (FFT(z)[0]).{x, y}: taken in the last pass of FFT 1
        fr::SplitOut so{buf, z0.x, z0.y, MH, M, xz + pi};
        fr::fft_passes<N, GROUP, fr::GATHER, fr::MULBF, R0, 1, Rs...>(buf, A, t, so);
        fr::fft_passes<N, GROUP, fr::PLAIN, fr::SPLIT, R0, 1, Rs...>(buf, A, t, so);
        if (live) {                                       // bins 0 .. M/2 of both rows (Z17)
            double2 *d0 = F + r0 * MH;
            for (int m = t; m < MH; m += GROUP) d0[m] = m == 0 ? make_double2(xz[pi].x, 0.0) : buf[m];
            if (r1 >= 0) {
                double2 *d1 = F + r1 * MH;
                for (int m = t; m < MH; m += GROUP) d1[m] = m == 0 ? make_double2(xz[pi].y, 0.0) : buf[MH + m];
            }
        }
        __syncthreads();                                  // the buffer is reused by the next round
    }
}

}  // namespace usfft
