// pcg_reg.cuh — register-resident batched PCG (K4c) for meshes with n-1 <= LX*BC interior
// columns: one CTA per sample, every node's PCG state in registers.
//
// Same discretisation as k_pcg (pde.cu header comment, Z11/Z12) and the same Jacobi PCG, written
// in the symmetrically scaled form: with D = diag(A), x^ = D^{1/2} x, r^ = D^{-1/2} r and
// A^ = D^{-1/2} A D^{-1/2} (unit diagonal), CG on A^ x^ = b^ produces the Jacobi-PCG iterates
// (z = D^-1 r <-> r^).  The loop is the Chronopoulos-Gear single-reduction variant:
//     w = A^ r^;  gamma = (r^,r^), delta = (w,r^) [+ rho = sum d r^^2 = ||r||_2^2]   [one reduction]
//     beta = gamma/gamma_old, alpha = gamma/(delta - beta*gamma/alpha_old)
//     p = r^ + beta p;  s = w + beta s;  x^ += alpha p;  r^ -= alpha s
// stopping on the true-residual recurrence ||r||_2 <= tol ||b||_2 (Z13).  Per iteration: one CTA
// barrier (shared by the reduction and the vertical halo, see the loop comment).  Mapping: a thread owns a BC x BR block
// of nodes (BC columns, BR rows); LX threads of a warp segment cover a row of blocks and exchange
// left/right neighbours by width-LX shuffles; row groups exchange their edge rows via shared
// memory.  All edge weights, the diagonal and the four CG vectors live in registers.
#pragma once

namespace usfft {

// 1/a for positive normal a: hardware seed (MUFU.RCP64H) refined by three Newton steps, no
// special-case branches (the CG scalars are positive and far from the fp64 range limits while
// the iteration runs; breakdown values stop the loop through the residual test first).
__device__ __forceinline__ double rcp_pos(double a) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    y = fma(y, e, y);
    e = fma(-a, y, 1.0);
    return fma(y, e, y);
}

template <int NC, int BC, int BR, int LX, int NWARP, int MINB>
__global__ void __launch_bounds__(NWARP * 32, MINB)
k_pcg_reg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
          int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
          double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S,
          const double *__restrict__ Bt) {
    constexpr int RGW = 32 / LX;                 // row groups per warp
    constexpr int NRG = NWARP * RGW;             // row groups per CTA
    constexpr int NCOL = LX * BC;                // covered columns
    extern __shared__ double sm[];
    __shared__ double red[2][4][NWARP];          // [parity][gamma, delta, rho, pad][warp]
    __shared__ unsigned long long dminmax[2];    // bit patterns of min / max diagonal (d > 0)
    __shared__ double th_amp[kMaxD];
    // edge-row halo buffers in dynamic shared memory after aT and dg:
    // [parity][top, bottom row][row group][col] of r_k, w_k, s_{k-1}
    typedef double HaloArr[2][2][NRG][NCOL];
    HaloArr &hr = *reinterpret_cast<HaloArr *>(sm + 2 * NC * NC + (NC + 1) * (NC + 1));
    HaloArr &hw = *reinterpret_cast<HaloArr *>(sm + 2 * NC * NC + (NC + 1) * (NC + 1) + 4 * NRG * NCOL);
    HaloArr &hs = *reinterpret_cast<HaloArr *>(sm + 2 * NC * NC + (NC + 1) * (NC + 1) + 8 * NRG * NCOL);

    constexpr int n = NC, nx = n - 1, np = n + 1, W = 3 * n + 1;   // NC = cells per side (== Q.n)
    double *aT = sm;                             // [2 n^2] coefficient at triangle centroids
    double *dg = sm + 2 * n * n;                 // [(n+1)^2] diagonal of A (padded)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = lane / LX, lx = lane % LX;
    const int rg = warp * RGW + seg;
    const int col0 = lx * BC, row0 = rg * BR;    // 0-based interior column/row of the block
    const double inv_n3 = 1.0 / ((double)n * n * n);
    // load of interior node (i, j): h^2 x2 = j / n^3 for f = x2, else the centroid-rule table
    auto bval = [&](int i, int j) -> double { return Bt ? __ldg(Bt + (j - 1) * nx + i - 1) : (double)j * inv_n3; };
    const double *Sy = S + (Q.psi ? Q.d * W : 0);

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        // ---- K3: coefficient at the 2n^2 centroids, then the diagonal ----------------------
        for (int j = tid; j < Q.d; j += blockDim.x) {      // d may exceed the CTA (n = 16: 32 threads)
            const double y = nodes ? nodes[(int64_t)j * nb + bl] : lattice_node(P, b, j);
            th_amp[j] = Q.amp[j] * theta_of(Q.theta, y, Q.delta);
        }
        __syncthreads();
        for (int e = tid; e < 2 * n * n; e += NWARP * 32) {
            const int cell = e >> 1, ci = cell % n, cj = cell / n;
            const int m1 = (e & 1) ? 3 * ci + 1 : 3 * ci + 2;     // T_up : T_lo
            const int m2 = (e & 1) ? 3 * cj + 2 : 3 * cj + 1;
            double s = 0.0;
            for (int j = 0; j < Q.d; ++j) s += th_amp[j] * S[j * W + m1] * Sy[j * W + m2];
            aT[e] = Q.form == 0 ? 1.0 + s : exp(s);
        }
        __syncthreads();
        // w_h(i,j) = (a_lo(i,j) + a_up(i,j-1))/2 ; w_v(i,j) = (a_up(i,j) + a_lo(i-1,j))/2
#define WH(i, j) (0.5 * (aT[2 * ((j) * n + (i))] + aT[2 * (((j) - 1) * n + (i)) + 1]))
#define WV(i, j) (0.5 * (aT[2 * ((j) * n + (i)) + 1] + aT[2 * ((j) * n + (i) - 1)]))
        if (tid == 0) {
            dminmax[0] = ~0ull;
            dminmax[1] = 0ull;
        }
        __syncthreads();
        for (int e = tid; e < np * np; e += NWARP * 32) {   // ring entries = 1 (padded nodes, r = 0)
            const int i = e % np, j = e / np;
            const bool in = i >= 1 && i <= nx && j >= 1 && j <= nx;
            const double v = in ? WH(i, j) + WH(i - 1, j) + WV(i, j) + WV(i, j - 1) : 1.0;
            dg[e] = v;
            if (in) {                                     // order-free min / max (positive doubles)
                atomicMin(&dminmax[0], (unsigned long long)__double_as_longlong(v));
                atomicMax(&dminmax[1], (unsigned long long)__double_as_longlong(v));
            }
        }
        __syncthreads();
        const double d_min = __longlong_as_double((long long)dminmax[0]);
        const double d_max = __longlong_as_double((long long)dminmax[1]);
        // ---- per-thread state --------------------------------------------------------------
        double x[BR][BC], r[BR][BC], p[BR][BC], s[BR][BC];
        const double *dgb = dg + (row0 + 1) * np + col0 + 1;   // diagonal of node (q, c): dgb[q*np + c]
        double wE[BR][BC + 1];                   // -w^ of the edge right of column c-1 (c=0: left edge)
        double wN[BR + 1][BC];                   // -w^ of the edge above row k-1 (k=0: bottom edge)
#pragma unroll
        for (int k = 0; k < BR; ++k)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = row0 + k + 1;
                const bool ok = i <= nx && j <= nx;
                x[k][c] = 0.0;
                p[k][c] = 0.0;
                s[k][c] = 0.0;
                r[k][c] = ok ? bval(i, j) / sqrt(dg[j * np + i]) : 0.0;               // b^ = D^-1/2 b
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
        // Iteration k (k = 0, 1, ...):  w_k = A^ r_k; one reduction -> gamma_k, delta_k, rho_k;
        // beta_k = gamma_k / gamma_{k-1}, alpha_k = gamma_k / (delta_k - gamma_k^2 / (gamma_{k-1}
        // alpha_{k-1})); then s_k = w_k + beta_k s_{k-1}, p_k = r_k + beta_k p_{k-1},
        // x += alpha_k p_k, r_{k+1} = r_k - alpha_k s_k.  The vertical halo needs r_{k+1} of the
        // neighbouring row groups: each thread publishes (r_k, w_k, s_{k-1}) of its edge rows
        // before the reduction barrier and every reader recomputes the neighbour's s_k and
        // r_{k+1} with the same fma sequence, so one barrier per iteration suffices (the halo
        // and partial-sum buffers alternate by iteration parity).
        // Stopping rule (Z13): ||r||_2^2 = rho = sum d r^^2 and d_min gamma <= rho <= d_max gamma
        // with gamma = (r^, r^).  rho is reduced only when gamma says the test may be close
        // (need_rho); otherwise d_max gamma <= tol^2 ||b||^2 (a sufficient condition) decides.  An
        // ambiguous iteration without rho continues, and the next one computes rho, so the loop
        // stops at most one iteration after the exact rule would.
        double rho = 0.0, bb = 0.0;
        bool need_rho = true, conv = false;
        double g_inv = 0.0, ga_inv = 0.0;        // 1/gamma_{k-1}, 1/(gamma_{k-1} alpha_{k-1})
        double below[BC], above[BC];             // neighbour r_k on the rows below/above
#pragma unroll
        for (int c = 0; c < BC; ++c) {           // r_0 of the neighbouring rows: b^ there
            const int i = col0 + c + 1;
            const int jb = row0, ja = row0 + BR + 1;
            below[c] = (jb >= 1 && i <= nx && rg > 0) ? bval(i, jb) / sqrt(dg[jb * np + i]) : 0.0;
            above[c] = (ja <= nx && i <= nx && rg + 1 < NRG) ? bval(i, ja) / sqrt(dg[ja * np + i]) : 0.0;
        }
        int it = 0;
        for (int k = 0;; ++k) {
            const int buf = k & 1;
            // ---- horizontal halo by shuffle, w = A^ r^ and the three partial dots ------------
            double left[BR], right[BR];
#pragma unroll
            for (int q = 0; q < BR; ++q) {
                left[q] = __shfl_up_sync(0xffffffffu, r[q][BC - 1], 1, LX);
                right[q] = __shfl_down_sync(0xffffffffu, r[q][0], 1, LX);
            }
            // partial dots in two interleaved chains per value (even / odd node) to halve the
            // dependent-FMA latency; combined in a fixed order below
            double acc2[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};   // [chain][gamma, delta, rho]
            double w[BR][BC];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const int ch = (q * BC + c) & 1;
                    const double rl = c > 0 ? r[q][c - 1] : left[q];
                    const double rr = c + 1 < BC ? r[q][c + 1] : right[q];
                    const double rd = q > 0 ? r[q - 1][c] : below[c];
                    const double ru = q + 1 < BR ? r[q + 1][c] : above[c];
                    double v = fma(wE[q][c + 1], rr, r[q][c]);
                    v = fma(wE[q][c], rl, v);
                    v = fma(wN[q + 1][c], ru, v);
                    v = fma(wN[q][c], rd, v);
                    w[q][c] = v;
                    acc2[ch][0] = fma(r[q][c], r[q][c], acc2[ch][0]);
                    acc2[ch][1] = fma(v, r[q][c], acc2[ch][1]);
                }
            if (need_rho) {                              // uniform branch (see the stopping rule)
#pragma unroll
                for (int q = 0; q < BR; ++q)
#pragma unroll
                    for (int c = 0; c < BC; ++c) {
                        const int ch = (q * BC + c) & 1;
                        acc2[ch][2] = fma(dgb[q * np + c] * r[q][c], r[q][c], acc2[ch][2]);   // padded: r = 0
                    }
            }
            double acc[4] = {acc2[0][0] + acc2[1][0], acc2[0][1] + acc2[1][1], acc2[0][2] + acc2[1][2], 0.0};
            // ---- publish the edge rows (r_k, w_k, s_{k-1}) for the neighbours ----------------
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                hr[buf][0][rg][col0 + c] = r[BR - 1][c];
                hw[buf][0][rg][col0 + c] = w[BR - 1][c];
                hs[buf][0][rg][col0 + c] = s[BR - 1][c];
                hr[buf][1][rg][col0 + c] = r[0][c];
                hw[buf][1][rg][col0 + c] = w[0][c];
                hs[buf][1][rg][col0 + c] = s[0][c];
            }
            // ---- warp reduction with value exchange: 6 double shuffles for 4 values ---------
            {
                const bool hi16 = lane & 16, hi8 = lane & 8;
                const double s0 = hi16 ? acc[0] : acc[2], s1 = hi16 ? acc[1] : acc[3];
                const double k0 = hi16 ? acc[2] : acc[0], k1 = hi16 ? acc[3] : acc[1];
                const double a0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
                const double a1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
                double v = (hi8 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                // lane 0: gamma, lane 8: delta, lane 16: rho, lane 24: pad
                if ((lane & 7) == 0) red[buf][lane >> 3][warp] = v;
            }
            __syncthreads();
            double gsum[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {            // fixed pairwise tree over the warps
                double t[NWARP];
#pragma unroll
                for (int ww = 0; ww < NWARP; ++ww) t[ww] = red[buf][q][ww];
#pragma unroll
                for (int h = 1; h < NWARP; h <<= 1)
#pragma unroll
                    for (int ww = 0; ww + h < NWARP; ww += 2 * h) t[ww] += t[ww + h];
                gsum[q] = t[0];
            }
            const double gamma = gsum[0], delta = gsum[1];
            rho = need_rho ? gsum[2] : d_max * gamma;    // exact, or an upper bound of ||r||^2
            if (k == 0) bb = rho;
            conv = rho <= Q.tol2 * bb;
            if (conv || it >= Q.maxit) break;
            need_rho = d_min * gamma <= 4.0 * Q.tol2 * bb;
            const double beta = k == 0 ? 0.0 : gamma * g_inv;
            const double alpha = gamma * rcp_pos(k == 0 ? delta : delta - gamma * gamma * ga_inv);
            g_inv = rcp_pos(gamma);                  // off the critical path of the next iteration
            ga_inv = rcp_pos(gamma * alpha);
            // the neighbours' edge rows (unconditional loads, clamped row groups); their latency overlaps
            // the vector updates below
            const int rgb = rg > 0 ? rg - 1 : rg, rga = rg + 1 < NRG ? rg + 1 : rg;
            double nb_r[BC], nb_w[BC], nb_s[BC], na_r[BC], na_w[BC], na_s[BC];
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                nb_r[c] = hr[buf][0][rgb][col0 + c];
                nb_w[c] = hw[buf][0][rgb][col0 + c];
                nb_s[c] = hs[buf][0][rgb][col0 + c];
                na_r[c] = hr[buf][1][rga][col0 + c];
                na_w[c] = hw[buf][1][rga][col0 + c];
                na_s[c] = hs[buf][1][rga][col0 + c];
            }
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    p[q][c] = fma(beta, p[q][c], r[q][c]);
                    s[q][c] = fma(beta, s[q][c], w[q][c]);
                    x[q][c] = fma(alpha, p[q][c], x[q][c]);
                    r[q][c] = fma(-alpha, s[q][c], r[q][c]);
                }
            // neighbours' r_{k+1} on the rows below / above, recomputed with the same fma chain
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const double vb = fma(-alpha, fma(beta, nb_s[c], nb_w[c]), nb_r[c]);
                const double va = fma(-alpha, fma(beta, na_s[c], na_w[c]), na_r[c]);
                below[c] = rg > 0 ? vb : 0.0;
                above[c] = rg + 1 < NRG ? va : 0.0;
            }
            ++it;
        }
        // ---- output: x = D^{-1/2} x^ ----------------------------------------------------------
#pragma unroll
        for (int k = 0; k < BR; ++k)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = row0 + k + 1;
                if (i <= nx && j <= nx) u[(int64_t)((j - 1) * nx + (i - 1)) * ldu + bl] = x[k][c] / sqrt(dg[j * np + i]);
            }
        if (tid == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rho / bb);       // exact or an upper bound
            if (noconv && !conv) atomicAdd(noconv, 1);
        }
        __syncthreads();
    }
}

}  // namespace usfft
