// pcg_mg.cuh — on-chip PCG with a geometric-multigrid V(1,1) preconditioner, one CTA per sample.
//
// Same P1 discretisation as pde.cu (Z11/Z12); CG in the Chronopoulos-Gear single-reduction form
//     u = M^-1 r;  w = A u;  gamma = (r,u), delta = (w,u), rho = (r,r)      [one reduction]
//     beta = gamma/gamma_old;  alpha = gamma/(delta - beta gamma/alpha_old)
//     p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s,
// stopping on rho = ||r||_2^2 <= tol^2 ||b||_2^2 (Z13).  M^-1 is one symmetric V(1,1) cycle:
// damped Jacobi (omega = 0.8) pre/post smoothing, bilinear prolongation P, restriction P^T,
// coarse operators by rediscretisation of the same P1 problem on the nested coarse "/" meshes
// (n/2, n/4, ..., 2 cells; the centroid coefficient uses the same sin table because every
// coarse centroid abscissa is a multiple of h/3), exact solve on the 1-node coarsest grid.  The
// cycle is symmetric (same smoother before and after, R = P^T) and SPD, so CG stays CG.
//
// Fine level: each thread owns a BC x BR block of nodes; the CG vectors x, r, p, s, the
// preconditioned residual u and the coupling weights live in registers; every fine vector that a
// stencil needs from other threads is published to one of three (n+1)^2 shared-memory grids with
// a zero Dirichlet ring.  Coarse levels live in shared memory and are swept by all threads.
// Reductions are fixed trees, so results do not depend on the CTA or launch split.
#pragma once

namespace usfft {

constexpr double kMgOmega = 0.8;

// per-level shared-memory arrays of a coarse grid with nl cells per side ((nl+1)^2 padded)
struct MgLevel {
    int nl;
    double *wh, *wv, *d, *di, *R, *Z, *S;   // R: rhs, Z: pre-smoothed, S: post-smoothed
};

template <int NC>
struct MgLayout {
    __host__ __device__ static constexpr int levels() {   // coarse levels n/2 .. 2
        int c = 0;
        for (int m = NC / 2; m >= 2; m /= 2) ++c;
        return c;
    }
    __host__ __device__ static constexpr int coarse_doubles() {
        int s = 0;
        for (int m = NC / 2; m >= 2; m /= 2) s += 7 * (m + 1) * (m + 1);
        return s;
    }
    __host__ __device__ static constexpr int doubles() {  // fine d, dinv + 3 fine grids + coarse
        return 5 * (NC + 1) * (NC + 1) + coarse_doubles();   // (aT aliases grids G1..G2)
    }
};

template <int NC, int BC, int BR, int LX, int NWARP, int MINB>
__global__ void __launch_bounds__(NWARP * 32, MINB)
k_pcg_mg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
         int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
         double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S) {
    constexpr int RGW = 32 / LX, NRG = NWARP * RGW, NT = NWARP * 32;
    constexpr int n = NC, nx = n - 1, np = n + 1, W = 3 * n + 1, NP2 = np * np;
    constexpr int NLEV = MgLayout<NC>::levels();
    static_assert(LX * BC >= nx && NRG * BR >= nx, "block mapping must cover the mesh");
    extern __shared__ double sm[];
    __shared__ double red[2][4][NWARP];
    __shared__ double th_amp[kMaxD];

    static_assert(2 * NC * NC <= 2 * (NC + 1) * (NC + 1), "aT must fit in G1..G2");
    double *D0 = sm;                         // fine diagonal (0 outside the interior)
    double *DI0 = D0 + NP2;                  // fine 1/diagonal (0 outside)
    double *G0 = DI0 + NP2;                  // published fine vectors, zero ring
    double *G1 = G0 + NP2;
    double *G2 = G1 + NP2;
    double *aT = G1;                         // [2n^2] setup only (aliases G1..G2)
    MgLevel lev[NLEV];
    {
        double *c = G2 + NP2;
#pragma unroll
        for (int l = 0; l < NLEV; ++l) {
            const int m = NC >> (l + 1), q = (m + 1) * (m + 1);
            lev[l] = MgLevel{m, c, c + q, c + 2 * q, c + 3 * q, c + 4 * q, c + 5 * q, c + 6 * q};
            c += 7 * q;
        }
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = lane / LX, lx = lane % LX;
    const int rg = warp * RGW + seg;
    const int col0 = lx * BC, row0 = rg * BR;
    const double inv_n3 = 1.0 / ((double)n * n * n);

    // a at the centroid of T_lo / T_up of cell (ci, cj) of a grid with cell width 2^sh h
    auto coef = [&](int ci, int cj, int up, int sh) -> double {
        const int m1 = (up ? 3 * ci + 1 : 3 * ci + 2) << sh;
        const int m2 = (up ? 3 * cj + 2 : 3 * cj + 1) << sh;
        double s = 0.0;
        for (int j = 0; j < Q.d; ++j) s += th_amp[j] * S[j * W + m1] * S[j * W + m2];
        return Q.form == 0 ? 1.0 + s : exp(s);
    };

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        // ---- K3: coefficient field and all level operators ---------------------------------
        if (tid < Q.d) {
            const double y = nodes ? nodes[(int64_t)tid * nb + bl] : lattice_node(P, b, tid);
            th_amp[tid] = Q.amp[tid] * theta_of(Q.theta, y);
        }
        __syncthreads();
        for (int e = tid; e < 2 * n * n; e += NT) {
            const int cell = e >> 1;
            aT[e] = coef(cell % n, cell / n, e & 1, 0);
        }
#pragma unroll
        for (int l = 0; l < NLEV; ++l) {             // coarse operators by rediscretisation
            const MgLevel L_ = lev[l];
            const int m = NC >> (l + 1), mp = m + 1, sh = l + 1;
            for (int e = tid; e < mp * mp; e += NT) {
                const int i = e % mp, j = e / mp;
                double h = 0.0, v = 0.0;
                if (i < m && j >= 1 && j < m) h = 0.5 * (coef(i, j, 0, sh) + coef(i, j - 1, 1, sh));
                if (j < m && i >= 1 && i < m) v = 0.5 * (coef(i, j, 1, sh) + coef(i - 1, j, 0, sh));
                L_.wh[e] = h;
                L_.wv[e] = v;
                L_.R[e] = 0.0;
                L_.Z[e] = 0.0;
                L_.S[e] = 0.0;
            }
        }
        __syncthreads();
#define WH(i, j) (0.5 * (aT[2 * ((j) * n + (i))] + aT[2 * (((j) - 1) * n + (i)) + 1]))
#define WV(i, j) (0.5 * (aT[2 * ((j) * n + (i)) + 1] + aT[2 * ((j) * n + (i) - 1)]))
        for (int e = tid; e < NP2; e += NT) {
            const int i = e % np, j = e / np;
            const bool in = i >= 1 && i <= nx && j >= 1 && j <= nx;
            const double dv = in ? WH(i, j) + WH(i - 1, j) + WV(i, j) + WV(i, j - 1) : 0.0;
            D0[e] = dv;
            DI0[e] = in ? 1.0 / dv : 0.0;
        }
#pragma unroll
        for (int l = 0; l < NLEV; ++l) {
            const MgLevel L_ = lev[l];
            const int m = NC >> (l + 1), mp = m + 1;
            for (int e = tid; e < mp * mp; e += NT) {
                const int i = e % mp, j = e / mp;
                const bool in = i >= 1 && i < m && j >= 1 && j < m;
                const double dv = in ? L_.wh[e] + L_.wh[e - 1] + L_.wv[e] + L_.wv[e - mp] : 0.0;
                L_.d[e] = dv;
                L_.di[e] = in ? 1.0 / dv : 0.0;
            }
        }
        // fine coupling weights in registers: zero on edges that touch the ring or padding
        double cE[BR][BC + 1], cN[BR + 1][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c <= BC; ++c) {
                const int i = col0 + c, j = row0 + q + 1;
                cE[q][c] = (i >= 1 && i + 1 <= nx && j <= nx) ? WH(i, j) : 0.0;
            }
#pragma unroll
        for (int q = 0; q <= BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = row0 + q;
                cN[q][c] = (j >= 1 && j + 1 <= nx && i <= nx) ? WV(i, j) : 0.0;
            }
#undef WH
#undef WV
        __syncthreads();
        for (int e = tid; e < NP2; e += NT) {        // zero rings of the fine grids (aT is dead)
            G0[e] = 0.0;
            G1[e] = 0.0;
            G2[e] = 0.0;
        }
        __syncthreads();
        // node (q, c) of this thread: fine grid index e = (row0+q+1)*np + col0+c+1 (may be padding)
        const int ebase = (row0 + 1) * np + col0 + 1;
        auto valid = [&](int q, int c) { return col0 + c + 1 <= nx && row0 + q + 1 <= nx; };
        auto publish = [&](double *Gd, const double (&v)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) Gd[ebase + q * np + c] = v[q][c];
        };
        // A v at this thread's nodes; neighbours inside the block from registers, others from Gs
        auto apply_fine = [&](const double *Gs, const double (&v)[BR][BC], double (&out)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const int e = ebase + q * np + c;
                    const double vl = c > 0 ? v[q][c - 1] : Gs[e - 1];
                    const double vr = c + 1 < BC ? v[q][c + 1] : Gs[e + 1];
                    const double vd = q > 0 ? v[q - 1][c] : Gs[e - np];
                    const double vu = q + 1 < BR ? v[q + 1][c] : Gs[e + np];
                    double a = D0[e] * v[q][c];
                    a = fma(-cE[q][c + 1], vr, a);
                    a = fma(-cE[q][c], vl, a);
                    a = fma(-cN[q + 1][c], vu, a);
                    out[q][c] = fma(-cN[q][c], vd, a);
                }
        };
        // ---- the V(1,1) cycle: z = M^-1 rin (rin must be published in G0 before the call) ----
        // Every phase reads only values published before the preceding barrier and recomputes
        // the few derived neighbour values it needs (pre-smoothed iterates omega D^-1 R,
        // residuals, prolongated corrections) instead of waiting for them: 8 barriers per cycle.
        auto vcycle = [&](const double (&rin)[BR][BC], double (&z)[BR][BC]) {
            double t[BR][BC];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) z[q][c] = kMgOmega * DI0[ebase + q * np + c] * rin[q][c];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {       // fine residual t = r - A z, z = omega D^-1 r
                    const int e = ebase + q * np + c;
                    const double vl = c > 0 ? z[q][c - 1] : kMgOmega * DI0[e - 1] * G0[e - 1];
                    const double vr = c + 1 < BC ? z[q][c + 1] : kMgOmega * DI0[e + 1] * G0[e + 1];
                    const double vd = q > 0 ? z[q - 1][c] : kMgOmega * DI0[e - np] * G0[e - np];
                    const double vu = q + 1 < BR ? z[q + 1][c] : kMgOmega * DI0[e + np] * G0[e + np];
                    double a = D0[e] * z[q][c];
                    a = fma(-cE[q][c + 1], vr, a);
                    a = fma(-cE[q][c], vl, a);
                    a = fma(-cN[q + 1][c], vu, a);
                    a = fma(-cN[q][c], vd, a);
                    t[q][c] = rin[q][c] - a;
                }
            publish(G1, t);
            __syncthreads();
            {   // restriction R = P^T to level 1 (n/2 cells)
                const MgLevel C = lev[0];
                constexpr int m = NC / 2, mp = m + 1;
                for (int e = tid; e < mp * mp; e += NT) {
                    const int I = e % mp, J = e / mp;
                    if (I < 1 || I >= m || J < 1 || J >= m) continue;
                    const int f = (2 * J) * np + 2 * I;
                    C.R[e] = G1[f] + 0.5 * (G1[f - 1] + G1[f + 1] + G1[f - np] + G1[f + np]) +
                             0.25 * (G1[f - np - 1] + G1[f - np + 1] + G1[f + np - 1] + G1[f + np + 1]);
                }
            }
            __syncthreads();
            // down sweep: level l pre-smooths (Z = omega D^-1 R) and restricts its residual, which
            // is recomputed from R at the 9 fine points; the coarsest level is solved exactly
#pragma unroll
            for (int l = 0; l + 1 < NLEV; ++l) {
                const MgLevel C = lev[l], Cn = lev[l + 1];
                const int m = NC >> (l + 1), mp = m + 1;
                const int mn = NC >> (l + 2), mnp = mn + 1;
                for (int e = tid; e < mp * mp; e += NT) C.Z[e] = kMgOmega * C.di[e] * C.R[e];
                auto tres = [&](int f) -> double {  // residual of the pre-smoothed iterate at f
                    if (C.di[f] == 0.0) return 0.0;
                    const double zc = kMgOmega * C.di[f] * C.R[f];
                    const double az = C.d[f] * zc - C.wh[f] * (kMgOmega * C.di[f + 1] * C.R[f + 1]) -
                                      C.wh[f - 1] * (kMgOmega * C.di[f - 1] * C.R[f - 1]) -
                                      C.wv[f] * (kMgOmega * C.di[f + mp] * C.R[f + mp]) -
                                      C.wv[f - mp] * (kMgOmega * C.di[f - mp] * C.R[f - mp]);
                    return C.R[f] - az;
                };
                for (int e = tid; e < mnp * mnp; e += NT) {
                    const int I = e % mnp, J = e / mnp;
                    if (I < 1 || I >= mn || J < 1 || J >= mn) continue;
                    const int f = (2 * J) * mp + 2 * I;
                    const double rn = tres(f) + 0.5 * (tres(f - 1) + tres(f + 1) + tres(f - mp) + tres(f + mp)) +
                                      0.25 * (tres(f - mp - 1) + tres(f - mp + 1) + tres(f + mp - 1) + tres(f + mp + 1));
                    Cn.R[e] = rn;
                    if (l + 2 == NLEV) Cn.Z[e] = Cn.di[e] * rn;      // coarsest: exact solve
                }
                __syncthreads();
            }
            // up sweep: S_l = smooth(Z_l + P S_{l+1}); neighbours' corrected iterates recomputed
#pragma unroll
            for (int l = NLEV - 2; l >= 0; --l) {
                const MgLevel C = lev[l], Cn = lev[l + 1];
                const int m = NC >> (l + 1), mp = m + 1, mnp = (NC >> (l + 2)) + 1;
                const double *Sn = (l + 2 == NLEV) ? Cn.Z : Cn.S;
                auto zc = [&](int g) -> double {    // Z + bilinear prolongation of Sn at node g
                    if (C.di[g] == 0.0) return 0.0;
                    const int i = g % mp, j = g / mp;
                    const double *z2 = Sn + (j >> 1) * mnp + (i >> 1);
                    double v;
                    if (!(i & 1) && !(j & 1)) v = z2[0];
                    else if (!(j & 1)) v = 0.5 * (z2[0] + z2[1]);
                    else if (!(i & 1)) v = 0.5 * (z2[0] + z2[mnp]);
                    else v = 0.25 * (z2[0] + z2[1] + z2[mnp] + z2[mnp + 1]);
                    return C.Z[g] + v;
                };
                for (int e = tid; e < mp * mp; e += NT) {
                    if (C.di[e] == 0.0) continue;
                    const double z0 = zc(e);
                    const double az = C.d[e] * z0 - C.wh[e] * zc(e + 1) - C.wh[e - 1] * zc(e - 1) -
                                      C.wv[e] * zc(e + mp) - C.wv[e - mp] * zc(e - mp);
                    C.S[e] = fma(kMgOmega * C.di[e], C.R[e] - az, z0);
                }
                __syncthreads();
            }
            // fine up: z += P S_1 and post-smooth; neighbours' corrected z = omega D^-1 r + P S_1
            const MgLevel C0 = lev[0];
            constexpr int m0p = NC / 2 + 1;
            auto prol = [&](int e) -> double {       // bilinear value of level-1 S at fine node e
                const int i = e % np, j = e / np, I = i >> 1, J = j >> 1;
                if (i < 1 || i > nx || j < 1 || j > nx) return 0.0;
                const double *z2 = C0.S + J * m0p + I;
                if (!(i & 1) && !(j & 1)) return z2[0];
                if (!(j & 1)) return 0.5 * (z2[0] + z2[1]);
                if (!(i & 1)) return 0.5 * (z2[0] + z2[m0p]);
                return 0.25 * (z2[0] + z2[1] + z2[m0p] + z2[m0p + 1]);
            };
            auto zf = [&](int e) -> double { return kMgOmega * DI0[e] * G0[e] + prol(e); };
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) z[q][c] += prol(ebase + q * np + c);
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const int e = ebase + q * np + c;
                    const double vl = c > 0 ? z[q][c - 1] : zf(e - 1);
                    const double vr = c + 1 < BC ? z[q][c + 1] : zf(e + 1);
                    const double vd = q > 0 ? z[q - 1][c] : zf(e - np);
                    const double vu = q + 1 < BR ? z[q + 1][c] : zf(e + np);
                    double a = D0[e] * z[q][c];
                    a = fma(-cE[q][c + 1], vr, a);
                    a = fma(-cE[q][c], vl, a);
                    a = fma(-cN[q + 1][c], vu, a);
                    a = fma(-cN[q][c], vd, a);
                    t[q][c] = fma(kMgOmega * DI0[e], rin[q][c] - a, z[q][c]);
                }
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) z[q][c] = t[q][c];
        };

        // ---- Chronopoulos-Gear PCG ----------------------------------------------------------
        double x[BR][BC], r[BR][BC], p[BR][BC], s[BR][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                x[q][c] = p[q][c] = s[q][c] = 0.0;
                r[q][c] = valid(q, c) ? (double)(row0 + q + 1) * inv_n3 : 0.0;     // b = h^2 x2
            }
        double rho = 0.0, bb = 0.0, g_inv = 0.0, ga_inv = 0.0;
        bool conv = false;
        int it = 0;
        for (int k = 0;; ++k) {
            const int buf = k & 1;
            double uu[BR][BC], w[BR][BC];
            publish(G0, r);
            __syncthreads();
            vcycle(r, uu);
            publish(G2, uu);
            __syncthreads();
            apply_fine(G2, uu, w);
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    acc[0] = fma(r[q][c], uu[q][c], acc[0]);
                    acc[1] = fma(w[q][c], uu[q][c], acc[1]);
                    acc[2] = fma(r[q][c], r[q][c], acc[2]);
                }
            {   // warp reduction with value exchange (4 values, 6 double shuffles)
                const bool hi16 = lane & 16, hi8 = lane & 8;
                const double s0 = hi16 ? acc[0] : acc[2], s1 = hi16 ? acc[1] : acc[3];
                const double k0 = hi16 ? acc[2] : acc[0], k1 = hi16 ? acc[3] : acc[1];
                const double a0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
                const double a1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
                double v = (hi8 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if ((lane & 7) == 0) red[buf][lane >> 3][warp] = v;
            }
            __syncthreads();
            double gs[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double tt[NWARP];
#pragma unroll
                for (int ww = 0; ww < NWARP; ++ww) tt[ww] = red[buf][q][ww];
#pragma unroll
                for (int h = 1; h < NWARP; h <<= 1)
#pragma unroll
                    for (int ww = 0; ww + h < NWARP; ww += 2 * h) tt[ww] += tt[ww + h];
                gs[q] = tt[0];
            }
            const double gamma = gs[0], delta = gs[1];
            rho = gs[2];
            if (k == 0) bb = rho;
            conv = rho <= Q.tol2 * bb;
            if (conv || it >= Q.maxit) break;
            const double beta = k == 0 ? 0.0 : gamma * g_inv;
            const double alpha = gamma * rcp_pos(k == 0 ? delta : delta - gamma * gamma * ga_inv);
            g_inv = rcp_pos(gamma);
            ga_inv = rcp_pos(gamma * alpha);
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    p[q][c] = fma(beta, p[q][c], uu[q][c]);
                    s[q][c] = fma(beta, s[q][c], w[q][c]);
                    x[q][c] = fma(alpha, p[q][c], x[q][c]);
                    r[q][c] = fma(-alpha, s[q][c], r[q][c]);
                }
            ++it;
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c)
                if (valid(q, c)) u[(int64_t)((row0 + q) * nx + col0 + c) * ldu + bl] = x[q][c];
        if (tid == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rho / bb);
            if (!conv) atomicAdd(noconv, 1);
        }
        __syncthreads();
    }
}

}  // namespace usfft
