// pcg_mg.cuh — on-chip CG with a four-level geometric-multigrid preconditioner, one CTA per sample.
//
// Same P1 discretisation as pde.cu (Z11/Z12); CG in the Chronopoulos-Gear single-reduction form
//     u = M^-1 r;  w = A u;  gamma = (r,u), delta = (w,u), rho = (r,r)      [one reduction]
//     beta = gamma/gamma_old;  alpha = gamma/(delta - beta gamma/alpha_old)
//     p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s,
// stopping on rho = ||r||_2^2 <= tol^2 ||b||_2^2 (Z13).
// M^-1 is one symmetric V(1,1) cycle over four nested "/" meshes (n, n/2, n/4, n/8 cells): damped
// Jacobi (omega = 0.8) pre- and post-smoothing on levels 0-2, bilinear prolongation P,
// restriction R = P^T, coarse operators by rediscretisation of the same P1 problem, and an exact
// solve on the coarsest level with its dense inverse (formed once per sample by Gauss-Jordan;
// (n/8-1)^2 = 9 unknowns at n = 32).  Same smoother before and after and R = P^T make the cycle
// symmetric positive definite, so CG stays CG.
//
// Every coarse-mesh triangle centroid is also a fine-mesh triangle centroid (its abscissae are
// (3c+1) 2^l or (3c+2) 2^l in units of h/3, never multiples of 3, and the pair has the fine
// lower/upper residue pattern), so the coarse coefficients are lookups into the fine per-triangle
// table: the d-term coefficient sums are evaluated only for the 2 n^2 fine triangles.
//
// Level 0 (fine): each thread owns a BC x BR block of nodes with x, r, p, s, u and the coupling
// weights in registers; values needed by other threads are published to shared-memory grids with
// a zero Dirichlet ring.  Levels 1-3 live in shared memory; every size is a compile-time constant.
// Level 1 runs on the whole CTA; levels 2 and 3 (49 + 9 unknowns at n = 32) run in warp 0 with
// warp-level synchronisation.  The CG update of r is not published separately: the first V-cycle
// phase recomputes a neighbour's r_{k+1} = r_k - alpha (w_k + beta s_{k-1}) from the (r, w, s)
// grids published before the reduction barrier (the same fma sequence the owner runs, so the
// values are bit-identical).  Eight CTA barriers per CG iteration.
// Reductions are fixed trees, so a sample's result does not depend on the CTA or launch split.
#pragma once
#include <type_traits>

namespace usfft {

constexpr double kMgOmega = 0.8;

template <int NC>
struct Mg3 {
    static constexpr int n = NC, np = NC + 1, NP2 = np * np;
    static constexpr int m1 = NC / 2, p1 = m1 + 1, N1 = p1 * p1;      // smoothed level 1
    static constexpr int m2 = NC / 4, p2 = m2 + 1, N2 = p2 * p2;      // smoothed level 2
    static constexpr int m3 = NC / 8, p3 = m3 + 1, N3 = p3 * p3, U3 = (m3 - 1) * (m3 - 1);  // exact
    // shared-memory layout (doubles): fine grids D, D^-1, G0 (r), G1 (fine residual), G2 (u),
    // Hr, Hw, Hs (CG vectors r, w, s for the neighbours' r update)
    static constexpr int oD0 = 0, oDI0 = NP2, oG0 = 2 * NP2, oG1 = 3 * NP2, oG2 = 4 * NP2;
    static constexpr int oHr = 5 * NP2, oHw = 6 * NP2, oHs = 7 * NP2;
    static constexpr int oL1 = 8 * NP2;                  // WH, WV, D, DI, R, Z, T, S of level 1
    static constexpr int oL2 = oL1 + 8 * N1;             // same for level 2
    static constexpr int oWH3 = oL2 + 8 * N2, oWV3 = oWH3 + N3, oR3 = oWV3 + N3, oE3 = oR3 + N3;
    static constexpr int oAI = oE3 + N3;                 // dense inverse of the level-3 operator
    __host__ __device__ static constexpr int doubles() { return oAI + U3 * U3; }
};

// one smoothed coarse level (arrays in shared memory, zero rings)
struct MgLv {
    double *WH, *WV, *D, *DI, *R, *Z, *T, *S;
};

template <int NC, int BC, int BR, int LX, int NWARP, int MINB>
__global__ void __launch_bounds__(NWARP * 32, MINB)
k_pcg_mg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
         int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
         double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S) {
    using L = Mg3<NC>;
    constexpr int RGW = 32 / LX, NRG = NWARP * RGW, NT = NWARP * 32;
    constexpr int n = NC, nx = n - 1, np = n + 1, W = 3 * n + 1, NP2 = L::NP2;
    constexpr int m1 = L::m1, P1 = L::p1, m2 = L::m2, P2 = L::p2;
    constexpr int m3 = L::m3, p3 = L::p3, U3 = L::U3;
    static_assert(LX * BC >= nx && NRG * BR >= nx, "block mapping must cover the mesh");
    static_assert(BC % 2 == 0 && BR % 2 == 0, "even node blocks: prolongation parity is compile-time");
    static_assert(NT % n == 0, "coefficient mapping: whole mesh rows per pass");
    static_assert(2 * NC * NC <= 2 * NP2, "aT must fit in G1..G2");
    static_assert(U3 >= 1 && U3 <= 32, "level 3 is solved by one warp");
    extern __shared__ double sm[];
    __shared__ double red[4][NWARP];
    __shared__ double th_amp[kMaxD];
    double *D0 = sm + L::oD0, *DI0 = sm + L::oDI0, *G0 = sm + L::oG0, *G1 = sm + L::oG1;
    double *G2 = sm + L::oG2, *aT = G1;                  // aT: setup only (aliases G1..G2)
    double *Hr = sm + L::oHr, *Hw = sm + L::oHw, *Hs = sm + L::oHs;
    const MgLv V1{sm + L::oL1, sm + L::oL1 + L::N1, sm + L::oL1 + 2 * L::N1, sm + L::oL1 + 3 * L::N1,
                  sm + L::oL1 + 4 * L::N1, sm + L::oL1 + 5 * L::N1, sm + L::oL1 + 6 * L::N1, sm + L::oL1 + 7 * L::N1};
    const MgLv V2{sm + L::oL2, sm + L::oL2 + L::N2, sm + L::oL2 + 2 * L::N2, sm + L::oL2 + 3 * L::N2,
                  sm + L::oL2 + 4 * L::N2, sm + L::oL2 + 5 * L::N2, sm + L::oL2 + 6 * L::N2, sm + L::oL2 + 7 * L::N2};
    double *WH3 = sm + L::oWH3, *WV3 = sm + L::oWV3, *R3 = sm + L::oR3, *E3 = sm + L::oE3;
    double *AI = sm + L::oAI;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = lane / LX, lx = lane % LX;
    const int rg = warp * RGW + seg;
    const int col0 = lx * BC, row0 = rg * BR;            // both even
    const double inv_n3 = 1.0 / ((double)n * n * n);

    // a at the centroid of T_lo / T_up of cell (ci, cj) of the mesh with cell width 2^sh h: the
    // fine triangle with the same centroid (abscissae ma, mb in units of h/3)
    auto fcoef = [&](int ci, int cj, int up, int sh) -> double {
        const int ma = (up ? 3 * ci + 1 : 3 * ci + 2) << sh;
        const int mb = (up ? 3 * cj + 2 : 3 * cj + 1) << sh;
        return aT[2 * ((mb / 3) * n + ma / 3) + (ma % 3 == 1 ? 1 : 0)];
    };
    // rediscretised edge weights of a coarse level (cell width 2^sh h, M cells)
    auto level_weights = [&](const MgLv &V, auto mconst, int sh) {
        constexpr int M = decltype(mconst)::value, MP = M + 1;
        for (int e = tid; e < MP * MP; e += NT) {
            const int i = e % MP, j = e / MP;
            V.WH[e] = (i < M && j >= 1 && j < M) ? 0.5 * (fcoef(i, j, 0, sh) + fcoef(i, j - 1, 1, sh)) : 0.0;
            V.WV[e] = (j < M && i >= 1 && i < M) ? 0.5 * (fcoef(i, j, 1, sh) + fcoef(i - 1, j, 0, sh)) : 0.0;
            V.R[e] = V.Z[e] = V.T[e] = V.S[e] = 0.0;
        }
    };
    auto level_diag = [&](const MgLv &V, auto mconst) {
        constexpr int M = decltype(mconst)::value, MP = M + 1;
        for (int e = tid; e < MP * MP; e += NT) {
            const int i = e % MP, j = e / MP;
            const bool in = i >= 1 && i < M && j >= 1 && j < M;
            const double dv = in ? V.WH[e] + V.WH[e - 1] + V.WV[e] + V.WV[e - MP] : 0.0;
            V.D[e] = dv;
            V.DI[e] = in ? 1.0 / dv : 0.0;
        }
    };
    using C1 = std::integral_constant<int, m1>;
    using C2 = std::integral_constant<int, m2>;

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        // ---- K3: coefficients and the operators of all levels --------------------------------
        if (tid < Q.d) {
            const double y = nodes ? nodes[(int64_t)tid * nb + bl] : lattice_node(P, b, tid);
            th_amp[tid] = Q.amp[tid] * theta_of(Q.theta, y);
        }
        __syncthreads();
        {   // fine per-triangle coefficients a = 1 + sum_j amp_j theta_j S_j(ma) S_j(mb) (or exp):
            // thread (ci, cj0) keeps the ci-side factors of every j and sweeps KC rows cj
            constexpr int CJS = NT / n, KC = n / CJS;
            const int ci = tid % n, cj0 = tid / n;
            double slo[KC], sup[KC];
#pragma unroll
            for (int k = 0; k < KC; ++k) slo[k] = sup[k] = 0.0;
            for (int j = 0; j < Q.d; ++j) {
                const double *Sj = S + j * W;
                const double tlo = th_amp[j] * __ldg(Sj + 3 * ci + 2);
                const double tup = th_amp[j] * __ldg(Sj + 3 * ci + 1);
#pragma unroll
                for (int k = 0; k < KC; ++k) {
                    const int cj = cj0 + k * CJS;
                    slo[k] = fma(tlo, __ldg(Sj + 3 * cj + 1), slo[k]);
                    sup[k] = fma(tup, __ldg(Sj + 3 * cj + 2), sup[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int cell = (cj0 + k * CJS) * n + ci;
                aT[2 * cell] = Q.form == 0 ? 1.0 + slo[k] : exp(slo[k]);
                aT[2 * cell + 1] = Q.form == 0 ? 1.0 + sup[k] : exp(sup[k]);
            }
        }
        __syncthreads();
        level_weights(V1, C1{}, 1);
        level_weights(V2, C2{}, 2);
        for (int e = tid; e < L::N3; e += NT) {
            const int i = e % p3, j = e / p3;
            WH3[e] = (i < m3 && j >= 1 && j < m3) ? 0.5 * (fcoef(i, j, 0, 3) + fcoef(i, j - 1, 1, 3)) : 0.0;
            WV3[e] = (j < m3 && i >= 1 && i < m3) ? 0.5 * (fcoef(i, j, 1, 3) + fcoef(i - 1, j, 0, 3)) : 0.0;
        }
#define WH(i, j) (0.5 * (aT[2 * ((j) * n + (i))] + aT[2 * (((j) - 1) * n + (i)) + 1]))
#define WV(i, j) (0.5 * (aT[2 * ((j) * n + (i)) + 1] + aT[2 * ((j) * n + (i) - 1)]))
        for (int e = tid; e < NP2; e += NT) {
            const int i = e % np, j = e / np;
            const bool in = i >= 1 && i <= nx && j >= 1 && j <= nx;
            const double dv = in ? WH(i, j) + WH(i - 1, j) + WV(i, j) + WV(i, j - 1) : 0.0;
            D0[e] = dv;
            DI0[e] = in ? 1.0 / dv : 0.0;
        }
        double cE[BR][BC + 1], cN[BR + 1][BC];          // fine couplings, zero at ring / padding
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
        __syncthreads();                                 // aT is dead from here on
        level_diag(V1, C1{});
        level_diag(V2, C2{});
        for (int e = tid; e < U3 * U3; e += NT) {        // dense level-3 operator, row-major
            const int a = e / U3, c = e % U3;
            const int ia = a % (m3 - 1) + 1, ja = a / (m3 - 1) + 1;
            const int ic = c % (m3 - 1) + 1, jc = c / (m3 - 1) + 1;
            const int g = ja * p3 + ia;
            double v = 0.0;
            if (a == c) v = WH3[g] + WH3[g - 1] + WV3[g] + WV3[g - p3];
            else if (jc == ja && ic == ia + 1) v = -WH3[g];
            else if (jc == ja && ic == ia - 1) v = -WH3[g - 1];
            else if (ic == ia && jc == ja + 1) v = -WV3[g];
            else if (ic == ia && jc == ja - 1) v = -WV3[g - p3];
            AI[e] = v;
        }
        for (int e = tid; e < NP2; e += NT) {
            const int i = e % np, j = e / np;
            const bool in = i >= 1 && i <= nx && j >= 1 && j <= nx;
            G0[e] = G1[e] = G2[e] = Hw[e] = Hs[e] = 0.0;
            Hr[e] = in ? (double)j * inv_n3 : 0.0;       // r_0 = b = h^2 x2
        }
        __syncthreads();
        if (warp == 0) {   // in-place Gauss-Jordan inverse of the coarsest operator (SPD, tiny)
            constexpr int GE = (U3 * U3 + 31) / 32;
            for (int k = 0; k < U3; ++k) {
                double rk[GE], ck[GE], old[GE];
                const double piv = 1.0 / AI[k * U3 + k];
#pragma unroll
                for (int t = 0; t < GE; ++t) {
                    const int e = lane + 32 * t;
                    if (e < U3 * U3) {
                        rk[t] = AI[k * U3 + e % U3];
                        ck[t] = AI[(e / U3) * U3 + k];
                        old[t] = AI[e];
                    }
                }
                __syncwarp();
#pragma unroll
                for (int t = 0; t < GE; ++t) {
                    const int e = lane + 32 * t;
                    if (e < U3 * U3) {
                        const int i = e / U3, j = e % U3;
                        double v;
                        if (i == k && j == k) v = piv;
                        else if (i == k) v = rk[t] * piv;
                        else if (j == k) v = -ck[t] * piv;
                        else v = fma(-ck[t] * piv, rk[t], old[t]);
                        AI[e] = v;
                    }
                }
                __syncwarp();
            }
            for (int e = lane; e < L::N3; e += 32) E3[e] = 0.0;   // padded grid with zero ring
            __syncwarp();
        }

        const int ebase = (row0 + 1) * np + col0 + 1;
        auto valid = [&](int q, int c) { return col0 + c + 1 <= nx && row0 + q + 1 <= nx; };
        auto publish = [&](double *Gd, const double (&v)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) Gd[ebase + q * np + c] = v[q][c];
        };
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
        // restriction R = P^T from a grid Xf (row length pf) to the node whose fine centre is f
        auto restrict9 = [](const double *Xf, int f, int pf) -> double {
            return Xf[f] + 0.5 * (Xf[f - 1] + Xf[f + 1] + Xf[f - pf] + Xf[f + pf]) +
                   0.25 * (Xf[f - pf - 1] + Xf[f - pf + 1] + Xf[f + pf - 1] + Xf[f + pf + 1]);
        };
        // bilinear prolongation of a coarse grid Xc (row length pc, zero ring) to fine node (i, j)
        auto prol2 = [](const double *Xc, int pc, int i, int j) -> double {
            const double *z2 = Xc + (j >> 1) * pc + (i >> 1);
            if (!(i & 1) && !(j & 1)) return z2[0];
            if (!(j & 1)) return 0.5 * (z2[0] + z2[1]);
            if (!(i & 1)) return 0.5 * (z2[0] + z2[pc]);
            return 0.25 * (z2[0] + z2[1] + z2[pc] + z2[pc + 1]);
        };
        // level operator A_V Z at node e of a level with row length MP
        auto applyV = [](const MgLv &V, const double *Zs, int e, int MP) -> double {
            return V.D[e] * Zs[e] - V.WH[e] * Zs[e + 1] - V.WH[e - 1] * Zs[e - 1] - V.WV[e] * Zs[e + MP] -
                   V.WV[e - MP] * Zs[e - MP];
        };
        // loop over the interior nodes (I, J in [1, M-1]) of a coarse level, e = J (M + 1) + I,
        // with compile-time trip counts: over the CTA (stride NT) or over warp 0 (stride 32)
        auto for_interior = [&](auto mconst, auto body) {
            constexpr int M = decltype(mconst)::value, MI = M - 1, U = MI * MI;
#pragma unroll
            for (int k = 0; k < (U + NT - 1) / NT; ++k) {
                const int q = tid + k * NT;
                if (q < U) body(q / MI * (M + 1) + q % MI + M + 2, q % MI + 1, q / MI + 1);
            }
        };
        auto for_interior_w = [&](auto mconst, auto body) {
            constexpr int M = decltype(mconst)::value, MI = M - 1, U = MI * MI;
#pragma unroll
            for (int k = 0; k < (U + 31) / 32; ++k) {
                const int q = lane + k * 32;
                if (q < U) body(q / MI * (M + 1) + q % MI + M + 2, q % MI + 1, q / MI + 1);
            }
        };

        // ---- one V(1,1) cycle: z = M^-1 rin.  The neighbours' rin come from the (r, w, s) grids
        // and the step (alpha, beta) of the previous CG iteration.
        auto vcycle = [&](const double (&rin)[BR][BC], double (&z)[BR][BC], double alpha, double beta) {
            double t[BR][BC];
            auto zn = [&](int e) -> double {     // neighbour's omega D^-1 r_{k+1}
                return kMgOmega * DI0[e] * fma(-alpha, fma(beta, Hs[e], Hw[e]), Hr[e]);
            };
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) z[q][c] = kMgOmega * DI0[ebase + q * np + c] * rin[q][c];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {       // residual of z = omega D^-1 r
                    const int e = ebase + q * np + c;
                    const double vl = c > 0 ? z[q][c - 1] : zn(e - 1);
                    const double vr = c + 1 < BC ? z[q][c + 1] : zn(e + 1);
                    const double vd = q > 0 ? z[q - 1][c] : zn(e - np);
                    const double vu = q + 1 < BR ? z[q + 1][c] : zn(e + np);
                    double a = D0[e] * z[q][c];
                    a = fma(-cE[q][c + 1], vr, a);
                    a = fma(-cE[q][c], vl, a);
                    a = fma(-cN[q + 1][c], vu, a);
                    a = fma(-cN[q][c], vd, a);
                    t[q][c] = rin[q][c] - a;
                }
            publish(G0, rin);
            publish(G1, t);
            __syncthreads();
            for_interior(C1{}, [&](int e, int I, int J) {        // R1 = P^T t, Z1 = omega D1^-1 R1
                const double rr = restrict9(G1, (2 * J) * np + 2 * I, np);
                V1.R[e] = rr;
                V1.Z[e] = kMgOmega * V1.DI[e] * rr;
            });
            __syncthreads();
            for_interior(C1{}, [&](int e, int, int) { V1.T[e] = V1.R[e] - applyV(V1, V1.Z, e, P1); });
            __syncthreads();
            if (warp == 0) {                                     // levels 2 and 3 in one warp
                for_interior_w(C2{}, [&](int e, int I, int J) {  // R2 = P^T T1, Z2 = omega D2^-1 R2
                    const double rr = restrict9(V1.T, (2 * J) * P1 + 2 * I, P1);
                    V2.R[e] = rr;
                    V2.Z[e] = kMgOmega * V2.DI[e] * rr;
                });
                __syncwarp();
                for_interior_w(C2{}, [&](int e, int, int) { V2.T[e] = V2.R[e] - applyV(V2, V2.Z, e, P2); });
                __syncwarp();
                if (lane < U3) {
                    const int I = lane % (m3 - 1) + 1, J = lane / (m3 - 1) + 1;
                    R3[lane] = restrict9(V2.T, (2 * J) * P2 + 2 * I, P2);
                }
                __syncwarp();
                if (lane < U3) {                                 // exact solve E3 = A3^-1 R3
                    double sacc = 0.0;
#pragma unroll
                    for (int c = 0; c < U3; ++c) sacc = fma(AI[lane * U3 + c], R3[c], sacc);
                    const int I = lane % (m3 - 1) + 1, J = lane / (m3 - 1) + 1;
                    E3[J * p3 + I] = sacc;
                }
                __syncwarp();
                for_interior_w(C2{}, [&](int e, int I, int J) {  // Zc2 = Z2 + P E3 (into T2)
                    V2.T[e] = V2.Z[e] + prol2(E3, p3, I, J);
                });
                __syncwarp();
                for_interior_w(C2{}, [&](int e, int, int) {      // S2 = smooth(Zc2)
                    V2.S[e] = fma(kMgOmega * V2.DI[e], V2.R[e] - applyV(V2, V2.T, e, P2), V2.T[e]);
                });
            }
            __syncthreads();
            for_interior(C1{}, [&](int e, int I, int J) {        // Zc1 = Z1 + P S2 (into T1)
                V1.T[e] = V1.Z[e] + prol2(V2.S, P2, I, J);
            });
            __syncthreads();
            for_interior(C1{}, [&](int e, int, int) {            // S1 = smooth(Zc1)
                V1.S[e] = fma(kMgOmega * V1.DI[e], V1.R[e] - applyV(V1, V1.T, e, P1), V1.T[e]);
            });
            __syncthreads();
            // level 0: z += P S1, post-smooth.  The coarse values this block and its neighbours
            // need form a (BR/2 + 2) x (BC/2 + 2) window of S1; the parity of every fine node
            // relative to (col0, row0) is a compile-time constant.
            constexpr int XW = BC / 2 + 2, YW = BR / 2 + 2;
            double cw[YW][XW];
#pragma unroll
            for (int yy = 0; yy < YW; ++yy)
#pragma unroll
                for (int xx = 0; xx < XW; ++xx) {
                    const int X = (col0 >> 1) + xx, Y = (row0 >> 1) + yy;
                    cw[yy][xx] = (X <= m1 && Y <= m1) ? V1.S[Y * P1 + X] : 0.0;
                }
            // P S1 at the fine node (col0 + 1 + c, row0 + 1 + q), c in [-1, BC], q in [-1, BR]
            auto pw = [&](int c, int q) -> double {
                const int fi = 1 + c, fj = 1 + q, x0 = fi >> 1, y0 = fj >> 1;
                if (!(fi & 1) && !(fj & 1)) return cw[y0][x0];
                if (!(fj & 1)) return 0.5 * (cw[y0][x0] + cw[y0][x0 + 1]);
                if (!(fi & 1)) return 0.5 * (cw[y0][x0] + cw[y0 + 1][x0]);
                return 0.25 * (cw[y0][x0] + cw[y0][x0 + 1] + cw[y0 + 1][x0] + cw[y0 + 1][x0 + 1]);
            };
            // a neighbour's corrected z = omega D^-1 r + P S1
            auto zf = [&](int e, int c, int q) -> double { return kMgOmega * DI0[e] * G0[e] + pw(c, q); };
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) z[q][c] += pw(c, q);
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const int e = ebase + q * np + c;
                    const double vl = c > 0 ? z[q][c - 1] : zf(e - 1, c - 1, q);
                    const double vr = c + 1 < BC ? z[q][c + 1] : zf(e + 1, c + 1, q);
                    const double vd = q > 0 ? z[q - 1][c] : zf(e - np, c, q - 1);
                    const double vu = q + 1 < BR ? z[q + 1][c] : zf(e + np, c, q + 1);
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
        double rho = 0.0, bb = 0.0, g_inv = 0.0, ga_inv = 0.0, alpha = 0.0, beta = 0.0;
        bool conv = false;
        int it = 0;
        for (int k = 0;; ++k) {
            double uu[BR][BC], w[BR][BC];
            vcycle(r, uu, alpha, beta);
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
            publish(Hr, r);                                  // read after the barrier below
            publish(Hw, w);
            publish(Hs, s);
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
                if ((lane & 7) == 0) red[lane >> 3][warp] = v;
            }
            __syncthreads();
            double gs[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double tt[NWARP];
#pragma unroll
                for (int ww = 0; ww < NWARP; ++ww) tt[ww] = red[q][ww];
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
            beta = k == 0 ? 0.0 : gamma * g_inv;
            alpha = gamma * rcp_pos(k == 0 ? delta : delta - gamma * gamma * ga_inv);
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
