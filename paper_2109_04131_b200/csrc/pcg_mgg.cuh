// pcg_mgg.cuh — multigrid-preconditioned CG for the larger meshes (n = 64, 128: configs 3-5), one
// CTA per sample, grids in a per-CTA global scratch region (L1/L2 resident at n = 64).
//
// Same P1 discretisation (Z11/Z12) and the same preconditioner family as pcg_mg.cuh: a symmetric
// V(1,1) cycle with damped Jacobi smoothing (omega = 0.8 fine, 1 coarse), bilinear prolongation P, restriction
// R = P^T and rediscretised coarse operators whose coefficients are lookups into the fine
// per-triangle table (every coarse centroid is a fine centroid), down to the mesh of 4 cells per
// side whose 9 unknowns are solved exactly with a dense inverse (Gauss-Jordan once per sample).
// Levels: n = 64 -> 64, 32, 16, 8 smoothed + 4 exact; n = 128 -> one more.  CG in the
// Chronopoulos-Gear single-reduction form (x0 = 0) stopping on ||r||_2 <= tol ||b||_2 (Z13).  13-14 iterations at
// n = 64 and 128 against 280 and 560 with the Jacobi preconditioner (tools/mg_smoother_study.py).
//
// The n = 16, 32 kernel keeps the fine level in registers; at n = 64 (3969 unknowns) and 128
// (16129) a sample no longer fits one SM's registers + shared memory, so here every grid is a
// padded (m+1)^2 array with a zero Dirichlet ring in the CTA's scratch slab, every phase is a
// CTA-wide loop over grid points and a barrier separates phases (21 per CG iteration at n = 64).
// Reductions are fixed trees: a sample's result does not depend on the CTA or the launch split.
#pragma once

namespace usfft {

constexpr int kMggMaxLev = 7;

// Scratch layout per CTA (doubles), fixed at compile time for each mesh NN so every level offset
// and every per-level division below folds to a constant.  Level l has m_l = NN >> l cells and
// P_l = m_l + 1 points per row.  Level 0: WH, WV, DI, B (= CG residual r), Z, T, X, P, S, W (X, P, S
// contiguous: the per-triangle coefficient table of the setup aliases them).  Levels 1..L-1: WH,
// WV, DI, B, Z, T.  Level L (m_L = 4): WH, WV, B, Z, then the dense inverse AI [9][9].  The
// coarsest levels that fit BUDGET doubles live in shared memory; when the level-0 Z and T (read at
// 5-9 stencil neighbours in every V-cycle pass) fit too, they come first and the levels from 2 on
// follow.
template <int NN>
struct MggC {
    static constexpr int L = NN == 8 ? 1 : NN == 16 ? 2 : NN == 32 ? 3 : NN == 64 ? 4 : NN == 128 ? 5 : -1;
    static_assert(L >= 1, "mesh must be 8, 16, 32, 64 or 128 cells per side");
    static constexpr int64_t BUDGET = 12288;                  // 96 KB: two CTAs per SM
    __host__ __device__ static constexpr int64_t P(int l) { return (NN >> l) + 1; }
    __host__ __device__ static constexpr int arrays(int l) { return l == 0 ? 10 : (l < L ? 6 : 4); }
    __host__ __device__ static constexpr int64_t size(int l) { return arrays(l) * P(l) * P(l) + (l == L ? 81 : 0); }
    static constexpr int64_t FINE = 2 * P(0) * P(0);
    static constexpr bool FINE_SMEM = L >= 2 && FINE < BUDGET;
    __host__ __device__ static constexpr int smem_from() {
        int from = L + 1;
        int64_t tail = 0, room = BUDGET - (FINE_SMEM ? FINE : 0);
        for (int l = L; l >= (FINE_SMEM ? 2 : 1); --l) {
            tail += size(l);
            if (tail > room) break;
            from = l;
        }
        return from;
    }
    static constexpr int SMEM_FROM = smem_from();
    __host__ __device__ static constexpr int64_t off(int l) {   // in its space (global or shared)
        int64_t og = 0, os = FINE_SMEM ? FINE : 0;
        for (int q = 0; q < l; ++q) (q >= SMEM_FROM ? os : og) += size(q);
        return l >= SMEM_FROM ? os : og;
    }
    __host__ __device__ static constexpr int64_t region() {
        int64_t og = 0;
        for (int q = 0; q < SMEM_FROM && q <= L; ++q) og += size(q);
        return (og + 31) & ~int64_t(31);
    }
    __host__ __device__ static constexpr int64_t smem() {
        int64_t os = FINE_SMEM ? FINE : 0;
        for (int q = SMEM_FROM; q <= L; ++q) os += size(q);
        return os;
    }
};

template <int NN, int T, int MINB>
__global__ void __launch_bounds__(T, MINB)
k_pcg_mgg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes,
          int64_t b0, int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
          double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S,
          const double *__restrict__ Bt, double *__restrict__ gscratch) {
    using C = MggC<NN>;
    __shared__ double red[32 * 3];
    __shared__ double th_amp[kMaxD];
    extern __shared__ double smg[];
    const int tid = threadIdx.x;
    constexpr int n = NN, L = C::L, W = 3 * n + 1, nx = n - 1;
    double *base = gscratch + (int64_t)blockIdx.x * C::region();
    // array k of level l (constant offsets once the level loops are unrolled)
    auto arr = [&](int l, int k) -> double * {
        const int64_t Pl = C::P(l);
        if (C::FINE_SMEM && l == 0 && (k == 4 || k == 5)) return smg + (k - 4) * Pl * Pl;
        return (l >= C::SMEM_FROM ? smg : base) + C::off(l) + (int64_t)k * Pl * Pl;
    };
    // body(i, j, e) for the interior points of an m-cell level (e = j (m+1) + i): thread tid owns
    // column 1 + tid % (m-1) of every (T / (m-1))-th row
    auto for_int = [&](int m, auto &&body) {
        const int cw = m - 1, rows = T / cw;
        if (tid < rows * cw) {
            const int i = 1 + tid % cw;
            for (int j = 1 + tid / cw; j < m; j += rows) body(i, j, j * (m + 1) + i);
        }
    };
    enum { WH = 0, WV = 1, DI = 2, BB = 3, ZZ = 4, TT = 5, XX = 6, PP = 7, QQ = 8, WW = 9 };
    double *aT = arr(0, XX);                               // setup only: [2][n][n]
    const double *Sy = S + (Q.psi ? Q.d * W : 0);
    const double inv_n3 = 1.0 / ((double)n * n * n);
    const int UL = 9;
    double *AI = arr(L, 0) + 4 * 25;                       // after WH, WV, B, Z of the 5 x 5 grid

    // stencil (A z)(e) on the padded grid of level l
    auto Az = [&](const double *wh, const double *wv, const double *z, int e, int Pl) -> double {
        const double we = wh[e], ww = wh[e - 1], wn = wv[e], ws = wv[e - Pl];
        return (we + ww + wn + ws) * z[e] - we * z[e + 1] - ww * z[e - 1] - wn * z[e + Pl] - ws * z[e - Pl];
    };
    auto interior = [](int e, int Pl, int m) {
        const int i = e % Pl, j = e / Pl;
        return i >= 1 && i < m && j >= 1 && j < m;
    };

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        for (int j = tid; j < Q.d; j += blockDim.x) {      // d may exceed the CTA (n = 16: 32 threads)
            const double y = nodes ? nodes[(int64_t)j * nb + bl] : lattice_node(P, b, j);
            th_amp[j] = Q.amp[j] * theta_of(Q.theta, y, Q.delta);
        }
        __syncthreads();
        // ---- K3: a at the 2 n^2 fine triangle centroids (lower plane, then upper plane) -------
        for (int e = tid; e < 2 * n * n; e += T) {
            const int up = e >= n * n, cell = up ? e - n * n : e, ci = cell % n, cj = cell / n;
            const int ma = up ? 3 * ci + 1 : 3 * ci + 2, mb = up ? 3 * cj + 2 : 3 * cj + 1;
            double s = 0.0;
            for (int j = 0; j < Q.d; ++j) s += th_amp[j] * __ldg(S + j * W + ma) * __ldg(Sy + j * W + mb);
            aT[e] = Q.form == 0 ? 1.0 + s : exp(s);
        }
        __syncthreads();
        // coefficient of T_lo / T_up of cell (ci, cj) of the level with cells of width 2^sh h: the fine
        // triangle with the same centroid (see pcg_mg.cuh)
        auto fcoef = [&](int ci, int cj, int up, int sh) -> double {
            const int p = 1 << sh, ra = up ? p : 2 * p, rb = up ? 2 * p : p;
            return aT[(ra % 3 == 1 ? n * n : 0) + (cj * p + rb / 3) * n + ci * p + ra / 3];
        };
        // ---- edge weights of every level, zeroed vectors --------------------------------------
#pragma unroll
        for (int l = 0; l <= L; ++l) {
            const int m = n >> l, Pl = m + 1;
            double *wh = arr(l, WH), *wv = arr(l, WV);
            double *bb_ = l < L ? arr(l, BB) : arr(l, 2), *zz = l < L ? arr(l, ZZ) : arr(l, 3);
            double *tt = l < L ? arr(l, TT) : nullptr;                // (Z, T may live in shared memory)
            for (int e = tid; e < Pl * Pl; e += T) {
                const int i = e % Pl, j = e / Pl;
                wh[e] = (i < m && j >= 1 && j < m) ? 0.5 * (fcoef(i, j, 0, l) + fcoef(i, j - 1, 1, l)) : 0.0;
                wv[e] = (j < m && i >= 1 && i < m) ? 0.5 * (fcoef(i, j, 1, l) + fcoef(i - 1, j, 0, l)) : 0.0;
                bb_[e] = 0.0;                                         // B, Z, T with zero rings
                zz[e] = 0.0;
                if (tt) tt[e] = 0.0;
            }
        }
        __syncthreads();
        // ---- omega / diagonal on the smoothed levels; dense A_L --------------------------------
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const int m = n >> l, Pl = m + 1;
            const double *wh = arr(l, WH), *wv = arr(l, WV);
            double *di = arr(l, DI);
            for (int e = tid; e < Pl * Pl; e += T)
                di[e] = interior(e, Pl, m) ? (l == 0 ? kMgOmega : kMgOmegaCoarse) / (wh[e] + wh[e - 1] + wv[e] + wv[e - Pl]) : 0.0;
        }
        if (tid < UL * UL) {                                          // 3 x 3 interior of the 5 x 5 grid
            const double *wh = arr(L, WH), *wv = arr(L, WV);
            const int r = tid / UL, c = tid % UL;
            const int ri = r % 3 + 1, rj = r / 3 + 1, ci = c % 3 + 1, cj = c / 3 + 1;
            const int e = rj * 5 + ri;
            double v = 0.0;
            if (r == c) v = wh[e] + wh[e - 1] + wv[e] + wv[e - 5];
            else if (cj == rj && ci == ri + 1) v = -wh[e];
            else if (cj == rj && ci == ri - 1) v = -wh[e - 1];
            else if (ci == ri && cj == rj + 1) v = -wv[e];
            else if (ci == ri && cj == rj - 1) v = -wv[e - 5];
            AI[r * UL + c] = v;
        }
        __syncthreads();
        // in-place Gauss-Jordan inverse of the SPD A_L (no pivoting needed)
        for (int k = 0; k < UL; ++k) {
            double a_rk = 0.0, a_kc = 0.0, a_kk = 0.0, a_rc = 0.0;
            const int r = tid / UL, c = tid % UL;
            if (tid < UL * UL) {
                a_rk = AI[r * UL + k];
                a_kc = AI[k * UL + c];
                a_kk = AI[k * UL + k];
                a_rc = AI[r * UL + c];
            }
            __syncthreads();
            if (tid < UL * UL) {
                const double inv = 1.0 / a_kk;
                double v;
                if (r == k && c == k) v = inv;
                else if (r == k) v = a_kc * inv;
                else if (c == k) v = -a_rk * inv;
                else v = a_rc - a_rk * a_kc * inv;
                AI[r * UL + c] = v;
            }
            __syncthreads();
        }
        // ---- CG init: x = 0, r = b, p = s = 0 (X, P, S overwrite the coefficient table) --------
        const int P0 = n + 1;
        double *__restrict__ X = arr(0, XX), *__restrict__ Pv = arr(0, PP), *__restrict__ Sv = arr(0, QQ);
        double *__restrict__ R0 = arr(0, BB), *__restrict__ Z0 = arr(0, ZZ), *__restrict__ T0 = arr(0, TT);
        double *__restrict__ Wv = arr(0, WW);
        const double *__restrict__ DI0 = arr(0, DI), *__restrict__ WH0 = arr(0, WH), *__restrict__ WV0 = arr(0, WV);
        double acc[3] = {0.0, 0.0, 0.0};
        for (int e = tid; e < P0 * P0; e += T) {
            X[e] = Pv[e] = Sv[e] = Wv[e] = 0.0;
            double bv = 0.0;
            if (interior(e, P0, n)) {
                const int i = e % P0, j = e / P0;
                bv = Bt ? __ldg(Bt + (j - 1) * nx + i - 1) : (double)j * inv_n3;
            }
            R0[e] = bv;
            Z0[e] = DI0[e] * bv;                                      // pre-smoothing from zero
            acc[0] += bv * bv;
        }
        block_sum<1>(*reinterpret_cast<double(*)[1]>(acc), red);
        const double bb = acc[0];

        // ---- V(1,1) cycle: T0 = M^-1 R0, assuming Z0 = DI0 R0 already written -----------------
        auto vcycle = [&]() {
#pragma unroll
            for (int l = 0; l < L; ++l) {                             // down
                const int m = n >> l, Pl = m + 1;
                const double *__restrict__ wh = arr(l, WH), *__restrict__ wv = arr(l, WV);
                const double *__restrict__ bl_ = arr(l, BB), *__restrict__ zl = arr(l, ZZ);
                double *__restrict__ tl = arr(l, TT);
                for_int(m, [&](int, int, int e) { tl[e] = bl_[e] - Az(wh, wv, zl, e, Pl); });   // residual
                __syncthreads();
                const int mc = m >> 1, Pc = mc + 1;
                double *__restrict__ bc = (l + 1 < L) ? arr(l + 1, BB) : arr(L, 2);
                double *__restrict__ zc = (l + 1 < L) ? arr(l + 1, ZZ) : nullptr;
                const double *__restrict__ dic = (l + 1 < L) ? arr(l + 1, DI) : nullptr;
                const double *__restrict__ tr = tl;
                for_int(mc, [&](int I, int J, int e) {                // restriction R = P^T (+ smoothing)
                    const int f = 2 * J * Pl + 2 * I;
                    const double v = tr[f] + 0.5 * (tr[f - 1] + tr[f + 1] + tr[f - Pl] + tr[f + Pl]) +
                                     0.25 * (tr[f - Pl - 1] + tr[f - Pl + 1] + tr[f + Pl - 1] + tr[f + Pl + 1]);
                    bc[e] = v;
                    if (zc) zc[e] = dic[e] * v;
                });
                __syncthreads();
            }
            {                                                         // exact solve on level L
                const double *bL = arr(L, 2);
                double *zL = arr(L, 3);
                if (tid < UL) {
                    double s = 0.0;
                    for (int c = 0; c < UL; ++c) s += AI[tid * UL + c] * bL[(c / 3 + 1) * 5 + c % 3 + 1];
                    zL[(tid / 3 + 1) * 5 + tid % 3 + 1] = s;
                }
                __syncthreads();
            }
#pragma unroll
            for (int l = L - 1; l >= 0; --l) {                        // up
                const int m = n >> l, Pl = m + 1, Pc = (m >> 1) + 1;
                const double *__restrict__ zc = (l + 1 < L) ? arr(l + 1, TT) : arr(L, 3);   // the coarse result
                double *__restrict__ zl = arr(l, ZZ);
                for_int(m, [&](int i, int j, int e) {                 // prolongation (bilinear)
                    const int c = (j >> 1) * Pc + (i >> 1);
                    double v;
                    if (!(i & 1) && !(j & 1)) v = zc[c];
                    else if (!(j & 1)) v = 0.5 * (zc[c] + zc[c + 1]);
                    else if (!(i & 1)) v = 0.5 * (zc[c] + zc[c + Pc]);
                    else v = 0.25 * (zc[c] + zc[c + 1] + zc[c + Pc] + zc[c + Pc + 1]);
                    zl[e] += v;
                });
                __syncthreads();
                const double *__restrict__ wh = arr(l, WH), *__restrict__ wv = arr(l, WV);
                const double *__restrict__ bl_ = arr(l, BB), *__restrict__ di = arr(l, DI);
                const double *__restrict__ zs = zl;
                double *__restrict__ tl = arr(l, TT);
                for_int(m, [&](int, int, int e) {                     // post-smoothing into T
                    tl[e] = zs[e] + di[e] * (bl_[e] - Az(wh, wv, zs, e, Pl));
                });
                __syncthreads();
            }
        };

        // ---- Chronopoulos-Gear PCG (as in pcg_mg.cuh): u = M^-1 r; w = A u; gamma = (r,u),
        // delta = (w,u) in one reduction; p = u + beta p, s = w + beta s, x += alpha p,
        // r -= alpha s fused with z0 = D r and (r,r)
        auto precond_and_apply = [&](double &gamma, double &delta) {
            vcycle();                                                 // T0 = M^-1 r
            acc[0] = acc[1] = 0.0;
            for_int(n, [&](int, int, int e) {
                const double w = Az(WH0, WV0, T0, e, P0), uu = T0[e];
                Wv[e] = w;
                acc[0] += R0[e] * uu;
                acc[1] += w * uu;
            });
            block_sum<2>(*reinterpret_cast<double(*)[2]>(acc), red);
            gamma = acc[0];
            delta = acc[1];
        };
        double gamma, delta, rr = bb, g_old = 0.0, a_old = 0.0;
        precond_and_apply(gamma, delta);
        int it = 0;
        while (rr > Q.tol2 * bb && it < Q.maxit) {
            const double beta = it == 0 ? 0.0 : gamma / g_old;
            const double alpha = it == 0 ? gamma / delta : gamma / (delta - beta * gamma / a_old);
            acc[0] = 0.0;
            for_int(n, [&](int, int, int e) {
                const double pv = T0[e] + beta * Pv[e], sv = Wv[e] + beta * Sv[e];
                Pv[e] = pv;
                Sv[e] = sv;
                X[e] += alpha * pv;
                const double r = R0[e] - alpha * sv;
                R0[e] = r;
                Z0[e] = DI0[e] * r;
                acc[0] += r * r;
            });
            block_sum<1>(*reinterpret_cast<double(*)[1]>(acc), red);
            rr = acc[0];
            g_old = gamma;
            a_old = alpha;
            ++it;
            if (rr <= Q.tol2 * bb) break;
            precond_and_apply(gamma, delta);
        }
        // ---- output u[g][bl] (interior nodes, x1 fastest) ---------------------------------------
        for (int g = tid; g < nx * nx; g += T) u[(int64_t)g * ldu + bl] = X[(g / nx + 1) * P0 + g % nx + 1];
        if (tid == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rr / bb);
            if (noconv && rr > Q.tol2 * bb) atomicAdd(noconv, 1);
        }
        __syncthreads();
    }
}

}  // namespace usfft
