// rader.cuh — K6 prime-length lattice FFT: Rader's algorithm over a mixed-radix Stockham FFT.
//
// For prime M with generator g of (Z/MZ)* and N = M-1 (7-smooth by the lattice-size rule Z2),
//   X[0] = sum_i x_i,   X[g^{-q}] = x_0 + (a * b)[q],  a_p = x_{g^p},  b_k = e^{-2 pi i g^{-k} / M},
// a length-N cyclic convolution evaluated as IFFT_N(FFT_N(a) . FFT_N(b)) with FFT_N(b)/N
// precomputed per M (host, long double) and the inverse done as conj(FFT(conj(.))).
// FFT_N: Stockham autosort, radices 4, 2, 3, 5, 7, ping-pong in shared memory, twiddles from an
// exact-index table e^{-2 pi i k/N}.  One CTA per (node, lattice) row; real input loaded
// coalesced, output staged in shared memory and written coalesced (bins 0..M/2, Z17).
#pragma once

namespace usfft {

struct RaderArgs {
    int64_t M, N;
    int nstage;
    uint64_t radix_code;        // radix of stage st in bits [4st, 4st+4)
    const double2 *tw;
    const int32_t *perm;
    const int32_t *outidx;
    const double2 *bf;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }


// y_s = sum_r v_r e^{-2 pi i r s / R}, written to out[base + s*stride].  Radix 2 and 4 by the
// textbook butterflies; 3 and 5 by the symmetric (real-coefficient) forms; 7 generic via twiddles.
template <int R>
__device__ __forceinline__ void dft_small(const double2 (&v)[R], double2 *__restrict__ out, int base,
                                          int stride, const double2 *__restrict__ tw, int wR) {
    if (R == 2) {
        out[base] = cadd(v[0], v[1]);
        out[base + stride] = csub(v[0], v[1]);
    } else if (R == 4) {
        const double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        const double2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
        out[base] = cadd(s02, s13);
        out[base + 2 * stride] = csub(s02, s13);
        out[base + stride] = make_double2(d02.x + d13.y, d02.y - d13.x);        // d02 - i d13
        out[base + 3 * stride] = make_double2(d02.x - d13.y, d02.y + d13.x);    // d02 + i d13
    } else if (R == 3) {
        const double S3 = 0.86602540378443864676;                              // sin(2 pi/3)
        const double2 t1 = cadd(v[1], v[2]), t2 = csub(v[1], v[2]);
        const double2 a = make_double2(fma(-0.5, t1.x, v[0].x), fma(-0.5, t1.y, v[0].y));
        const double2 b = make_double2(S3 * t2.x, S3 * t2.y);
        out[base] = cadd(v[0], t1);
        out[base + stride] = make_double2(a.x + b.y, a.y - b.x);                // a - i b
        out[base + 2 * stride] = make_double2(a.x - b.y, a.y + b.x);            // a + i b
    } else if (R == 5) {
        const double C1 = 0.30901699437494742410, C2 = -0.80901699437494742410;  // cos(2pi/5), cos(4pi/5)
        const double S1 = 0.95105651629515357212, S2 = 0.58778525229247312917;   // sin(2pi/5), sin(4pi/5)
        const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
        const double2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
        const double2 a1 = make_double2(fma(C2, t2.x, fma(C1, t1.x, v[0].x)), fma(C2, t2.y, fma(C1, t1.y, v[0].y)));
        const double2 a2 = make_double2(fma(C1, t2.x, fma(C2, t1.x, v[0].x)), fma(C1, t2.y, fma(C2, t1.y, v[0].y)));
        const double2 b1 = make_double2(fma(S2, t4.x, S1 * t3.x), fma(S2, t4.y, S1 * t3.y));
        const double2 b2 = make_double2(fma(-S1, t4.x, S2 * t3.x), fma(-S1, t4.y, S2 * t3.y));
        out[base] = cadd(v[0], cadd(t1, t2));
        out[base + stride] = make_double2(a1.x + b1.y, a1.y - b1.x);            // a1 - i b1
        out[base + 4 * stride] = make_double2(a1.x - b1.y, a1.y + b1.x);        // a1 + i b1
        out[base + 2 * stride] = make_double2(a2.x + b2.y, a2.y - b2.x);        // a2 - i b2
        out[base + 3 * stride] = make_double2(a2.x - b2.y, a2.y + b2.x);        // a2 + i b2
    } else {
#pragma unroll
        for (int s2 = 0; s2 < R; ++s2) {
            double2 acc = v[0];
#pragma unroll
            for (int r = 1; r < R; ++r) acc = cadd(acc, cmul(v[r], __ldg(tw + ((r * s2) % R) * wR)));
            out[base + s2 * stride] = acc;
        }
    }
}

// one Stockham stage of radix R: in -> out, Ns = product of earlier radices
template <int R>
__device__ __forceinline__ void stockham_stage(const double2 *__restrict__ in, double2 *__restrict__ out,
                                               int N, int Ns, const double2 *__restrict__ tw) {
    const int nbf = N / R;
    const int tstep = N / (Ns * R);
    for (int j = threadIdx.x; j < nbf; j += blockDim.x) {
        const int jm = j % Ns;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double2 a = in[j + r * nbf];
            v[r] = r == 0 ? a : cmul(a, __ldg(tw + (r * jm * tstep) % N));
        }
        const int base = (j / Ns) * Ns * R + jm;
        dft_small<R>(v, out, base, Ns, tw, N / R);
    }
}

// forward FFT_N of b0 over the stage list (ping-pong with b1); returns the buffer with the result
__device__ __forceinline__ double2 *fft_stockham(double2 *b0, double2 *b1, int N, int nstage,
                                                 uint64_t code, const double2 *__restrict__ tw) {
    int Ns = 1;
    double2 *in = b0, *out = b1;
    for (int st = 0; st < nstage; ++st) {
        const int R = (int)((code >> (4 * st)) & 15u);
        if (R == 4) stockham_stage<4>(in, out, N, Ns, tw);
        else if (R == 2) stockham_stage<2>(in, out, N, Ns, tw);
        else if (R == 3) stockham_stage<3>(in, out, N, Ns, tw);
        else if (R == 5) stockham_stage<5>(in, out, N, Ns, tw);
        else stockham_stage<7>(in, out, N, Ns, tw);
        __syncthreads();
        Ns *= R;
        double2 *t = in;
        in = out;
        out = t;
    }
    return in;
}

__global__ void __launch_bounds__(256)
k_fft_rader(const double *__restrict__ u, const SlabParams S, int64_t G_loc, int32_t L,
            const RaderArgs A, double2 *__restrict__ F) {
    extern __shared__ double smr[];
    __shared__ double red[32];
    const int64_t M = A.M, N = A.N, Mh = M / 2 + 1;
    double *xs = smr;                                                        // [M] (+pad)
    double2 *b0 = reinterpret_cast<double2 *>(smr + ((M + 1) & ~int64_t(1)));  // [N]
    double2 *b1 = b0 + N;                                                    // [N]
    const int64_t row = blockIdx.x;
    const int64_t g = row / L, l = row - g * L;
    // load the row: contiguous within each slab
    double part[1] = {0.0};
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
        const double v = sample_at(u, S, G_loc, g, l * M + i);
        xs[i] = v;
        part[0] += v;
    }
    block_sum<1>(part, red);                     // X[0] = sum_i x_i (fixed tree); also syncs xs
    const double x0 = xs[0];
    for (int64_t p = threadIdx.x; p < N; p += blockDim.x) b0[p] = make_double2(xs[__ldg(A.perm + p)], 0.0);
    __syncthreads();
    double2 *Ahat = fft_stockham(b0, b1, (int)N, A.nstage, A.radix_code, A.tw);
    double2 *other = Ahat == b0 ? b1 : b0;
    // pointwise product with FFT(b)/N, conjugated for the inverse transform
    for (int64_t k = threadIdx.x; k < N; k += blockDim.x) {
        const double2 c = cmul(Ahat[k], __ldg(A.bf + k));
        Ahat[k] = make_double2(c.x, -c.y);
    }
    __syncthreads();
    double2 *conv = fft_stockham(Ahat, other, (int)N, A.nstage, A.radix_code, A.tw);     // conj of the cyclic convolution
    double2 *stage_out = conv == b0 ? b1 : b0;
    // X[g^{-q}] = x0 + conv[q]; stage bins <= M/2 in natural order, then store coalesced
    for (int64_t q = threadIdx.x; q < N; q += blockDim.x) {
        const int32_t m = __ldg(A.outidx + q);
        if (m < Mh) {
            const double2 c = conv[q];
            stage_out[m] = make_double2(x0 + c.x, -c.y);
        }
    }
    __syncthreads();
    double2 *dst = F + row * Mh;
    for (int64_t m = threadIdx.x; m < Mh; m += blockDim.x)
        dst[m] = m == 0 ? make_double2(part[0], 0.0) : stage_out[m];
}

}  // namespace usfft
