// pcg_reg.cuh — register-resident batched PCG (K4c) for meshes with n-1 <= LX*BC interior
// columns: one CTA per sample, every node's PCG state in registers.
//
// Same discretisation as k_pcg (pde.cu header comment, Z11/Z12) and the same Jacobi PCG, written
// in the symmetrically scaled form: with D = diag(A), x^ = D^{1/2} x, r^ = D^{-1/2} r and
// A^ = D^{-1/2} A D^{-1/2} (unit diagonal), CG on A^ x^ = b^ produces the Jacobi-PCG iterates
// (z = D^-1 r <-> r^).  The loop is the Chronopoulos-Gear single-reduction variant:
//     w = A^ r^;  gamma = (r^,r^), delta = (w,r^), rho = sum d r^^2 (= ||r||_2^2)   [one reduction]
//     beta = gamma/gamma_old, alpha = gamma/(delta - beta*gamma/alpha_old)
//     p = r^ + beta p;  s = w + beta s;  x^ += alpha p;  r^ -= alpha s
// stopping on the true-residual recurrence ||r||_2 <= tol ||b||_2 (Z13).  Per iteration: one CTA
// barrier for the vertical halo, one fixed-tree reduction.  Mapping: a thread owns a BC x BR block
// of nodes (BC columns, BR rows); LX threads of a warp segment cover a row of blocks and exchange
// left/right neighbours by width-LX shuffles; row groups exchange their edge rows via shared
// memory.  All edge weights, the diagonal and the four CG vectors live in registers.
#pragma once

namespace usfft {

template <int BC, int BR, int LX, int NWARP>
__global__ void __launch_bounds__(NWARP * 32, 3)
k_pcg_reg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
          int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
          double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S) {
    constexpr int RGW = 32 / LX;                 // row groups per warp
    constexpr int NRG = NWARP * RGW;             // row groups per CTA
    constexpr int NCOL = LX * BC;                // covered columns
    extern __shared__ double sm[];
    __shared__ double red[3][NWARP];
    __shared__ double th_amp[kMaxD];
    __shared__ double topv[NRG][NCOL];           // each row group's top row of r^
    __shared__ double botv[NRG][NCOL];           // each row group's bottom row of r^

    const int n = Q.n, nx = n - 1, np = n + 1, W = 3 * n + 1;
    double *aT = sm;                             // [2 n^2] coefficient at triangle centroids
    double *dg = sm + 2 * n * n;                 // [(n+1)^2] diagonal of A (padded)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = lane / LX, lx = lane % LX;
    const int rg = warp * RGW + seg;
    const int col0 = lx * BC, row0 = rg * BR;    // 0-based interior column/row of the block
    const double inv_n3 = 1.0 / ((double)n * n * n);

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        // ---- K3: coefficient at the 2n^2 centroids, then the diagonal ----------------------
        if (tid < Q.d) {
            const double y = nodes ? nodes[(int64_t)tid * nb + bl] : lattice_node(P, b, tid);
            th_amp[tid] = Q.amp[tid] * theta_of(Q.theta, y);
        }
        __syncthreads();
        for (int e = tid; e < 2 * n * n; e += NWARP * 32) {
            const int cell = e >> 1, ci = cell % n, cj = cell / n;
            const int m1 = (e & 1) ? 3 * ci + 1 : 3 * ci + 2;     // T_up : T_lo
            const int m2 = (e & 1) ? 3 * cj + 2 : 3 * cj + 1;
            double s = 0.0;
            for (int j = 0; j < Q.d; ++j) s += th_amp[j] * S[j * W + m1] * S[j * W + m2];
            aT[e] = Q.form == 0 ? 1.0 + s : exp(s);
        }
        __syncthreads();
        // w_h(i,j) = (a_lo(i,j) + a_up(i,j-1))/2 ; w_v(i,j) = (a_up(i,j) + a_lo(i-1,j))/2
#define WH(i, j) (0.5 * (aT[2 * ((j) * n + (i))] + aT[2 * (((j) - 1) * n + (i)) + 1]))
#define WV(i, j) (0.5 * (aT[2 * ((j) * n + (i)) + 1] + aT[2 * ((j) * n + (i) - 1)]))
        for (int e = tid; e < nx * nx; e += NWARP * 32) {
            const int i = e % nx + 1, j = e / nx + 1;
            dg[j * np + i] = WH(i, j) + WH(i - 1, j) + WV(i, j) + WV(i, j - 1);
        }
        __syncthreads();
        // ---- per-thread state --------------------------------------------------------------
        double d[BR][BC], x[BR][BC], r[BR][BC], p[BR][BC], s[BR][BC];
        double wE[BR][BC + 1];                   // -w^ of the edge right of column c-1 (c=0: left edge)
        double wN[BR + 1][BC];                   // -w^ of the edge above row k-1 (k=0: bottom edge)
#pragma unroll
        for (int k = 0; k < BR; ++k)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = row0 + k + 1;
                const bool ok = i <= nx && j <= nx;
                d[k][c] = ok ? dg[j * np + i] : 1.0;
                x[k][c] = 0.0;
                p[k][c] = 0.0;
                s[k][c] = 0.0;
                r[k][c] = ok ? ((double)j * inv_n3) / sqrt(d[k][c]) : 0.0;      // b^ = D^-1/2 b
            }
#pragma unroll
        for (int k = 0; k < BR; ++k)
#pragma unroll
            for (int c = 0; c <= BC; ++c) {      // edge between columns i and i+1, i = col0 + c
                const int i = col0 + c, j = row0 + k + 1;
                double w = 0.0;
                if (i >= 1 && i + 1 <= nx && j <= nx)
                    w = -WH(i, j) / sqrt(dg[j * np + i] * dg[j * np + i + 1]);
                wE[k][c] = w;
            }
#pragma unroll
        for (int k = 0; k <= BR; ++k)
#pragma unroll
            for (int c = 0; c < BC; ++c) {       // edge between rows j and j+1, j = row0 + k
                const int i = col0 + c + 1, j = row0 + k;
                double w = 0.0;
                if (j >= 1 && j + 1 <= nx && i <= nx)
                    w = -WV(i, j) / sqrt(dg[j * np + i] * dg[(j + 1) * np + i]);
                wN[k][c] = w;
            }
#undef WH
#undef WV
        double bb = 0.0;                          // ||b||^2 = sum d r^^2 at start (reduced below)
        double gamma_old = 1.0, alpha_old = 1.0, rho = 0.0;
        int it = 0;
        bool first = true;
        while (true) {
            // ---- halo: own edge rows to shared memory, horizontal neighbours by shuffle -----
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                topv[rg][col0 + c] = r[BR - 1][c];
                botv[rg][col0 + c] = r[0][c];
            }
            double left[BR], right[BR];
#pragma unroll
            for (int k = 0; k < BR; ++k) {
                left[k] = __shfl_up_sync(0xffffffffu, r[k][BC - 1], 1, LX);
                right[k] = __shfl_down_sync(0xffffffffu, r[k][0], 1, LX);
            }
            __syncthreads();
            double below[BC], above[BC];
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                below[c] = rg > 0 ? topv[rg - 1][col0 + c] : 0.0;
                above[c] = rg + 1 < NRG ? botv[rg + 1][col0 + c] : 0.0;
            }
            // ---- w = A^ r^ and the three partial dots ---------------------------------------
            double acc[3] = {0.0, 0.0, 0.0};     // gamma, delta, rho
            double w[BR][BC];
#pragma unroll
            for (int k = 0; k < BR; ++k)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const double rl = c > 0 ? r[k][c - 1] : left[k];
                    const double rr = c + 1 < BC ? r[k][c + 1] : right[k];
                    const double rd = k > 0 ? r[k - 1][c] : below[c];
                    const double ru = k + 1 < BR ? r[k + 1][c] : above[c];
                    double v = fma(wE[k][c + 1], rr, r[k][c]);
                    v = fma(wE[k][c], rl, v);
                    v = fma(wN[k + 1][c], ru, v);
                    v = fma(wN[k][c], rd, v);
                    w[k][c] = v;
                    acc[0] = fma(r[k][c], r[k][c], acc[0]);
                    acc[1] = fma(v, r[k][c], acc[1]);
                    acc[2] = fma(d[k][c] * r[k][c], r[k][c], acc[2]);
                }
            // ---- one fixed-tree block reduction ----------------------------------------------
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                for (int q = 0; q < 3; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            }
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < 3; ++q) red[q][warp] = acc[q];
            }
            __syncthreads();
            double gamma = 0.0, delta = 0.0;
            rho = 0.0;
#pragma unroll
            for (int q = 0; q < NWARP; ++q) {
                gamma += red[0][q];
                delta += red[1][q];
                rho += red[2][q];
            }
            if (first) bb = rho;
            if (rho <= Q.tol2 * bb || it >= Q.maxit) break;
            double alpha, beta;
            if (first) {
                beta = 0.0;
                alpha = gamma / delta;
            } else {
                beta = gamma / gamma_old;
                alpha = gamma / (delta - beta * gamma / alpha_old);
            }
            first = false;
            gamma_old = gamma;
            alpha_old = alpha;
#pragma unroll
            for (int k = 0; k < BR; ++k)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    p[k][c] = fma(beta, p[k][c], r[k][c]);
                    s[k][c] = fma(beta, s[k][c], w[k][c]);
                    x[k][c] = fma(alpha, p[k][c], x[k][c]);
                    r[k][c] = fma(-alpha, s[k][c], r[k][c]);
                }
            ++it;
        }
        // ---- output: x = D^{-1/2} x^ ----------------------------------------------------------
#pragma unroll
        for (int k = 0; k < BR; ++k)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = row0 + k + 1;
                if (i <= nx && j <= nx) u[(int64_t)((j - 1) * nx + (i - 1)) * ldu + bl] = x[k][c] / sqrt(d[k][c]);
            }
        if (tid == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rho / bb);
            if (rho > Q.tol2 * bb) atomicAdd(noconv, 1);
        }
        __syncthreads();
    }
}

}  // namespace usfft
