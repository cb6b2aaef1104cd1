// rader_t.cuh — compile-time specialisations of the Rader lattice FFT (rader.cuh) for the lattice
// sizes the size rule Z2 produces (M = 97, 401, 2017, 4001: N = M-1 = 96, 400, 2016, 4000).
// With N a template parameter every Stockham index (j / Ns, j % Ns, twiddle index) is a constant
// division and the stage list is unrolled.  A group of WPR warps transforms one row (WPR = 1:
// warp-synchronous, no CTA barrier); a CTA holds RPC rows.  Shared memory per row: two N-point
// complex ping-pong buffers; the real input row is staged in the second buffer.
#pragma once

namespace usfft {

template <int N>
struct RadixList {
    __host__ __device__ static constexpr int count() {
        int n = N, c = 0;
        for (int r : {4, 2, 3, 5, 7})
            while (n % r == 0) {
                n /= r;
                ++c;
            }
        return c;
    }
    __host__ __device__ static constexpr int radix(int st) {
        int n = N, c = 0;
        for (int r : {4, 2, 3, 5, 7})
            while (n % r == 0) {
                if (c == st) return r;
                n /= r;
                ++c;
            }
        return 1;
    }
    __host__ __device__ static constexpr int ns(int st) {            // product of the radices before stage st
        int p = 1;
        for (int k = 0; k < st; ++k) p *= radix(k);
        return p;
    }
};

template <int GROUP>
__device__ __forceinline__ void group_sync(int gid) {
    if (GROUP == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(GROUP) : "memory");
}

template <int N, int R, int NS, int GROUP>
__device__ __forceinline__ void stage_t(const double2 *__restrict__ in, double2 *__restrict__ out,
                                        const double2 *__restrict__ tw, int t) {
    constexpr int NBF = N / R, TSTEP = N / (NS * R), WR = N / R;
    for (int j = t; j < NBF; j += GROUP) {
        const int jm = j % NS;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double2 a = in[j + r * NBF];
            v[r] = (r == 0 || NS == 1) ? a : cmul(a, __ldg(tw + r * jm * TSTEP));
        }
        const int base = (j / NS) * NS * R + jm;
        dft_small<R>(v, out, base, NS, tw, WR);
    }
}

template <int N, int ST, int GROUP>
__device__ __forceinline__ double2 *fft_t(double2 *in, double2 *out, const double2 *__restrict__ tw,
                                          int t, int gid) {
    if constexpr (ST == RadixList<N>::count()) {
        return in;
    } else {
        constexpr int R = RadixList<N>::radix(ST);
        stage_t<N, R, RadixList<N>::ns(ST), GROUP>(in, out, tw, t);
        group_sync<GROUP>(gid);
        return fft_t<N, ST + 1, GROUP>(out, in, tw, t, gid);
    }
}

template <int N, int WPR, int RPC>
__global__ void __launch_bounds__(WPR * 32 * RPC)
k_fft_rader_t(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int32_t L,
              const RaderArgs A, double2 *__restrict__ F, int64_t rows) {
    constexpr int GROUP = WPR * 32;
    constexpr int M = N + 1, MH = M / 2 + 1;
    constexpr int PER = (M + GROUP - 1) / GROUP;          // samples per thread per row
    extern __shared__ double2 smt[];
    __shared__ double wsum[32];
    const int gid = threadIdx.x / GROUP, t = threadIdx.x % GROUP;
    double2 *b0 = smt + (size_t)gid * 2 * N;
    double2 *b1 = b0 + N;
    double *xs = reinterpret_cast<double *>(b1);           // real row staged in b1 (M <= 2N)
    const bool one_slab = S.nslab == 1;
    const int64_t stride = (int64_t)gridDim.x * RPC;
    int64_t row = (int64_t)blockIdx.x * RPC + gid;
    // register prefetch of the group's next row (one slab: the row is contiguous)
    double xv[PER];
    auto fetch = [&](int64_t rw) {
        const int64_t g = rw / L, l = rw - g * L;
        if (one_slab) {
            const double *src = u + g * (int64_t)L * M + l * M;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = t + k * GROUP;
                xv[k] = i < M ? __ldg(src + i) : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = t + k * GROUP;
                xv[k] = i < M ? sample_at(u, S, G_loc, g, l * M + i) : 0.0;
            }
        }
    };
    if (row < rows) fetch(row);
    for (; row < rows; row += stride) {
        double part = 0.0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = t + k * GROUP;
            if (i < M) xs[i] = xv[k];
            part += xv[k];
        }
        if (row + stride < rows) fetch(row + stride);       // overlaps the transforms below
        // X[0] = sum_i x_i: fixed tree over the group (shuffles, then warp partials in order)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (WPR > 1) {
            if ((t & 31) == 0) wsum[gid * WPR + (t >> 5)] = part;
        }
        group_sync<GROUP>(gid);
        if (WPR > 1) {
            double tot = 0.0;
#pragma unroll
            for (int w = 0; w < WPR; ++w) tot += wsum[gid * WPR + w];
            part = tot;
        }
        const double x0 = xs[0];
        for (int p = t; p < N; p += GROUP) b0[p] = make_double2(xs[__ldg(A.perm + p)], 0.0);
        group_sync<GROUP>(gid);
        double2 *Ahat = fft_t<N, 0, GROUP>(b0, b1, A.tw, t, gid);
        double2 *other = Ahat == b0 ? b1 : b0;
        for (int k = t; k < N; k += GROUP) {
            const double2 c = cmul(Ahat[k], __ldg(A.bf + k));
            Ahat[k] = make_double2(c.x, -c.y);
        }
        group_sync<GROUP>(gid);
        double2 *conv = fft_t<N, 0, GROUP>(Ahat, other, A.tw, t, gid);
        double2 *stage_out = conv == b0 ? b1 : b0;
        for (int q = t; q < N; q += GROUP) {
            const int32_t m = __ldg(A.outidx + q);
            if (m < MH) {
                const double2 c = conv[q];
                stage_out[m] = make_double2(x0 + c.x, -c.y);
            }
        }
        group_sync<GROUP>(gid);
        double2 *dst = F + row * MH;
        for (int m = t; m < MH; m += GROUP) dst[m] = m == 0 ? make_double2(part, 0.0) : stage_out[m];
        group_sync<GROUP>(gid);                               // buffers are reused by the next row
    }
}

}  // namespace usfft

namespace usfft {

// Two real rows per complex transform (lattices 2j and 2j+1 of one node g; an odd L pairs its
// last lattice with a zero row, so a row's result never depends on how nodes are split).
// With z = a0 + i a1 (the two Rader sequences) and C_j = FFT(a_j) . FFT(b)/N, linearity gives
// FFT(z) . FFT(b)/N = C0 + i C1 without separating the two spectra, and the second transform of
// P = conj(C0 + i C1) is D = conj(conv0) - i conj(conv1).  Each row's convolution satisfies
// conv[q + N/2] = conj(conv[q]) (real input: X[M - m] = conj X[m], g^{N/2} = -1 mod M), so
//   conj(conv0[q]) = (D[q] + conj D[q + N/2]) / 2,   conj(conv1[q]) = (conj D[q + N/2] - D[q]) / 2i,
// and q < N/2 covers every pair {m, M - m} once: X_j[m] = x0_j + conv_j[q] for m = g^-q <= M/2,
// else X_j[M - m] = conj(x0_j + conv_j[q]).  Half the transforms of k_fft_rader_t per row.
template <int N, int WPR, int RPC>
__global__ void __launch_bounds__(WPR * 32 * RPC)
k_fft_rader_tp(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int32_t L,
               const RaderArgs A, double2 *__restrict__ F, int64_t rows) {
    constexpr int GROUP = WPR * 32;
    constexpr int M = N + 1, MH = M / 2 + 1, NB = N + 2;  // buffer: N values (+2: staging room)
    constexpr int PER = (M + GROUP - 1) / GROUP;
    extern __shared__ double2 smt[];
    __shared__ double wsum[2][32];
    const int gid = threadIdx.x / GROUP, t = threadIdx.x % GROUP;
    double2 *b0 = smt + (size_t)gid * 2 * NB;
    double2 *b1 = b0 + NB;
    double *xs0 = reinterpret_cast<double *>(b1), *xs1 = xs0 + M;   // both real rows in b1 (2M <= 2 NB)
    const bool one_slab = S.nslab == 1;
    const int64_t LP = (L + 1) / 2, pairs = (rows / L) * LP;         // rows = G_loc * L
    const int64_t stride = (int64_t)gridDim.x * RPC;
    int64_t pr = (int64_t)blockIdx.x * RPC + gid;
    double xv0[PER], xv1[PER];
    auto fetch = [&](int64_t rw, double (&xv)[PER]) {
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
                const int i = t + k * GROUP;
                xv[k] = i < M ? __ldg(src + i) : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int i = t + k * GROUP;
                xv[k] = i < M ? sample_at(u, S, G_loc, g, l * M + i) : 0.0;
            }
        }
    };
    auto row0 = [&](int64_t q) { return (q / LP) * L + 2 * (q % LP); };
    auto row1 = [&](int64_t q) { return 2 * (q % LP) + 1 < L ? row0(q) + 1 : int64_t(-1); };
    if (pr < pairs) {
        fetch(row0(pr), xv0);
        fetch(row1(pr), xv1);
    }
    for (; pr < pairs; pr += stride) {
        const int64_t r0 = row0(pr), r1 = row1(pr);
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = t + k * GROUP;
            if (i < M) {
                xs0[i] = xv0[k];
                xs1[i] = xv1[k];
            }
            p0 += xv0[k];
            p1 += xv1[k];
        }
        if (pr + stride < pairs) {                          // overlaps the transforms below
            fetch(row0(pr + stride), xv0);
            fetch(row1(pr + stride), xv1);
        }
        // X[0] of both rows: fixed tree over the group (shuffles, then warp partials in order)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            p0 += __shfl_xor_sync(0xffffffffu, p0, o);
            p1 += __shfl_xor_sync(0xffffffffu, p1, o);
        }
        if (WPR > 1 && (t & 31) == 0) {
            wsum[0][gid * WPR + (t >> 5)] = p0;
            wsum[1][gid * WPR + (t >> 5)] = p1;
        }
        group_sync<GROUP>(gid);
        if (WPR > 1) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int w = 0; w < WPR; ++w) {
                s0 += wsum[0][gid * WPR + w];
                s1 += wsum[1][gid * WPR + w];
            }
            p0 = s0;
            p1 = s1;
        }
        const double x00 = xs0[0], x01 = xs1[0];
        for (int p = t; p < N; p += GROUP) {
            const int pi = __ldg(A.perm + p);
            b0[p] = make_double2(xs0[pi], xs1[pi]);
        }
        group_sync<GROUP>(gid);
        double2 *Z = fft_t<N, 0, GROUP>(b0, b1, A.tw, t, gid);
        double2 *other = Z == b0 ? b1 : b0;
        for (int k = t; k < N; k += GROUP) {                // P = conj(Z . FFT(b)/N)
            const double2 c = cmul(Z[k], __ldg(A.bf + k));
            Z[k] = make_double2(c.x, -c.y);
        }
        group_sync<GROUP>(gid);
        double2 *D = fft_t<N, 0, GROUP>(Z, other, A.tw, t, gid);
        double2 *st = D == b0 ? b1 : b0;                    // staging: row 0 at [0, MH), row 1 at [MH, 2 MH)
        for (int q = t; q < N / 2; q += GROUP) {
            const double2 dq = D[q], dh = D[q + N / 2];
            const double2 s = make_double2(0.5 * (dq.x + dh.x), 0.5 * (dq.y - dh.y));        // conj(conv0)
            const double2 tt = make_double2(0.5 * (dh.x - dq.x), 0.5 * (-dh.y - dq.y));      // 2i conj(conv1) / 2
            const int32_t m = __ldg(A.outidx + q);
            // conv0 = (s.x, -s.y); conv1 = (tt.y, tt.x)
            if (m < MH) {
                st[m] = make_double2(x00 + s.x, -s.y);
                st[MH + m] = make_double2(x01 + tt.y, tt.x);
            } else {
                st[M - m] = make_double2(x00 + s.x, s.y);
                st[MH + M - m] = make_double2(x01 + tt.y, -tt.x);
            }
        }
        group_sync<GROUP>(gid);
        double2 *d0 = F + r0 * MH;
        for (int m = t; m < MH; m += GROUP) d0[m] = m == 0 ? make_double2(p0, 0.0) : st[m];
        if (r1 >= 0) {
            double2 *d1 = F + r1 * MH;
            for (int m = t; m < MH; m += GROUP) d1[m] = m == 0 ? make_double2(p1, 0.0) : st[MH + m];
        }
        group_sync<GROUP>(gid);                             // buffers are reused by the next pair
    }
}

}  // namespace usfft
