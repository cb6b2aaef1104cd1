// pcg_mg.cuh — on-chip CG with a three-level geometric-multigrid preconditioner, one CTA per sample.
//
// Same P1 discretisation as pde.cu (Z11/Z12); CG in the Chronopoulos-Gear single-reduction form
//     u = M^-1 r;  w = A u;  gamma = (r,u), delta = (w,u), rho = (r,r)      [one reduction]
//     beta = gamma/gamma_old;  alpha = gamma/(delta - beta gamma/alpha_old)
//     p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s,
// stopping on rho = ||r||_2^2 <= tol^2 ||b||_2^2 (Z13).
// M^-1 is one symmetric V(1,1) cycle over three nested "/" meshes (n, n/2, n/4 cells): damped
// Jacobi (omega = 0.8) pre- and post-smoothing on levels 0 and 1, bilinear prolongation P,
// restriction R = P^T, coarse operators by rediscretisation of the same P1 problem (every coarse
// centroid abscissa is a multiple of h/3, so the fine sin table serves all levels), and an exact
// solve on level 2 with its dense inverse (formed once per sample by Gauss-Jordan; (n/4-1)^2 = 49
// unknowns at n = 32).  Same smoother before and after and R = P^T make the cycle symmetric
// positive definite, so CG stays CG.
//
// Level 0 (fine): each thread owns a BC x BR block of nodes with x, r, p, s, u and the coupling
// weights in registers; values needed by other threads are published to shared-memory grids with
// a zero Dirichlet ring.  Levels 1-2 live in shared memory; every size is a compile-time constant.
// Reductions are fixed trees, so a sample's result does not depend on the CTA or launch split.
#pragma once

namespace usfft {

constexpr double kMgOmega = 0.8;

template <int NC>
struct Mg3 {
    static constexpr int n = NC, np = NC + 1, NP2 = np * np;
    static constexpr int m1 = NC / 2, p1 = m1 + 1, N1 = p1 * p1;
    static constexpr int m2 = NC / 4, p2 = m2 + 1, N2 = p2 * p2, U2 = (m2 - 1) * (m2 - 1);
    // shared-memory layout (doubles)
    static constexpr int oD0 = 0, oDI0 = NP2, oG0 = 2 * NP2, oG1 = 3 * NP2, oG2 = 4 * NP2;
    static constexpr int oWH1 = 5 * NP2, oWV1 = oWH1 + N1, oD1 = oWV1 + N1, oDI1 = oD1 + N1;
    static constexpr int oR1 = oDI1 + N1, oZ1 = oR1 + N1, oT1 = oZ1 + N1, oS1 = oT1 + N1;
    static constexpr int oWH2 = oS1 + N1, oWV2 = oWH2 + N2, oR2 = oWV2 + N2, oE2 = oR2 + U2;
    static constexpr int oAI = oE2 + U2;                 // dense inverse of the level-2 operator
    __host__ __device__ static constexpr int doubles() { return oAI + U2 * U2; }
};

template <int NC, int BC, int BR, int LX, int NWARP, int MINB>
__global__ void __launch_bounds__(NWARP * 32, MINB)
k_pcg_mg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
         int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
         double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S) {
    using L = Mg3<NC>;
    constexpr int RGW = 32 / LX, NRG = NWARP * RGW, NT = NWARP * 32;
    constexpr int n = NC, nx = n - 1, np = n + 1, W = 3 * n + 1, NP2 = L::NP2;
    constexpr int m1 = L::m1, p1 = L::p1, N1 = L::N1, m2 = L::m2, p2 = L::p2, U2 = L::U2;
    static_assert(LX * BC >= nx && NRG * BR >= nx, "block mapping must cover the mesh");
    static_assert(2 * NC * NC <= 2 * NP2, "aT must fit in G1..G2");
    extern __shared__ double sm[];
    __shared__ double red[4][NWARP];
    __shared__ double th_amp[kMaxD];
    double *D0 = sm + L::oD0, *DI0 = sm + L::oDI0, *G0 = sm + L::oG0, *G1 = sm + L::oG1;
    double *G2 = sm + L::oG2, *aT = G1;                  // aT: setup only (aliases G1..G2)
    double *WH1 = sm + L::oWH1, *WV1 = sm + L::oWV1, *D1 = sm + L::oD1, *DI1 = sm + L::oDI1;
    double *R1 = sm + L::oR1, *Z1 = sm + L::oZ1, *T1 = sm + L::oT1, *S1 = sm + L::oS1;
    double *WH2 = sm + L::oWH2, *WV2 = sm + L::oWV2, *R2 = sm + L::oR2, *E2 = sm + L::oE2;
    double *AI = sm + L::oAI;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = lane / LX, lx = lane % LX;
    const int rg = warp * RGW + seg;
    const int col0 = lx * BC, row0 = rg * BR;
    const double inv_n3 = 1.0 / ((double)n * n * n);

    // a at the centroid of T_lo / T_up of cell (ci, cj) of the mesh with cell width 2^sh h
    auto coef = [&](int ci, int cj, int up, int sh) -> double {
        const int ma = (up ? 3 * ci + 1 : 3 * ci + 2) << sh;
        const int mb = (up ? 3 * cj + 2 : 3 * cj + 1) << sh;
        double s = 0.0;
        for (int j = 0; j < Q.d; ++j) s += th_amp[j] * __ldg(S + j * W + ma) * __ldg(S + j * W + mb);
        return Q.form == 0 ? 1.0 + s : exp(s);
    };

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        // ---- K3: coefficients, fine/level-1/level-2 operators -------------------------------
        if (tid < Q.d) {
            const double y = nodes ? nodes[(int64_t)tid * nb + bl] : lattice_node(P, b, tid);
            th_amp[tid] = Q.amp[tid] * theta_of(Q.theta, y);
        }
        __syncthreads();
        for (int e = tid; e < 2 * n * n; e += NT) {
            const int cell = e >> 1;
            aT[e] = coef(cell % n, cell / n, e & 1, 0);
        }
        for (int e = tid; e < N1; e += NT) {            // level 1 (cell width 2h)
            const int i = e % p1, j = e / p1;
            WH1[e] = (i < m1 && j >= 1 && j < m1) ? 0.5 * (coef(i, j, 0, 1) + coef(i, j - 1, 1, 1)) : 0.0;
            WV1[e] = (j < m1 && i >= 1 && i < m1) ? 0.5 * (coef(i, j, 1, 1) + coef(i - 1, j, 0, 1)) : 0.0;
            R1[e] = Z1[e] = T1[e] = S1[e] = 0.0;
        }
        for (int e = tid; e < L::N2; e += NT) {         // level 2 (cell width 4h)
            const int i = e % p2, j = e / p2;
            WH2[e] = (i < m2 && j >= 1 && j < m2) ? 0.5 * (coef(i, j, 0, 2) + coef(i, j - 1, 1, 2)) : 0.0;
            WV2[e] = (j < m2 && i >= 1 && i < m2) ? 0.5 * (coef(i, j, 1, 2) + coef(i - 1, j, 0, 2)) : 0.0;
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
        for (int e = tid; e < N1; e += NT) {
            const int i = e % p1, j = e / p1;
            const bool in = i >= 1 && i < m1 && j >= 1 && j < m1;
            const double dv = in ? WH1[e] + WH1[e - 1] + WV1[e] + WV1[e - p1] : 0.0;
            D1[e] = dv;
            DI1[e] = in ? 1.0 / dv : 0.0;
        }
        for (int e = tid; e < U2 * U2; e += NT) {        // dense level-2 operator, row-major
            const int a = e / U2, c = e % U2;
            const int ia = a % (m2 - 1) + 1, ja = a / (m2 - 1) + 1;
            const int ic = c % (m2 - 1) + 1, jc = c / (m2 - 1) + 1;
            const int g = ja * p2 + ia;
            double v = 0.0;
            if (a == c) v = WH2[g] + WH2[g - 1] + WV2[g] + WV2[g - p2];
            else if (jc == ja && ic == ia + 1) v = -WH2[g];
            else if (jc == ja && ic == ia - 1) v = -WH2[g - 1];
            else if (ic == ia && jc == ja + 1) v = -WV2[g];
            else if (ic == ia && jc == ja - 1) v = -WV2[g - p2];
            AI[e] = v;
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
        __syncthreads();
        for (int e = tid; e < NP2; e += NT) G0[e] = G1[e] = G2[e] = 0.0;   // aT is dead now
        // Gauss-Jordan inversion in place (SPD: no pivoting).  Step k copies row k and column k
        // (old values) to scratch (R2 / E2 are free during setup), then updates every entry.
        for (int k = 0; k < U2; ++k) {
            __syncthreads();
            for (int q = tid; q < U2; q += NT) {
                R2[q] = AI[k * U2 + q];
                E2[q] = AI[q * U2 + k];
            }
            __syncthreads();
            const double piv = 1.0 / R2[k];
            for (int e = tid; e < U2 * U2; e += NT) {
                const int i = e / U2, j = e % U2;
                double v;
                if (i == k && j == k) v = piv;
                else if (i == k) v = R2[j] * piv;
                else if (j == k) v = -E2[i] * piv;
                else v = fma(-E2[i] * piv, R2[j], AI[e]);
                AI[e] = v;
            }
        }
        __syncthreads();

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
        auto A1 = [&](const double *Zs, int e) -> double {     // level-1 operator at node e
            return D1[e] * Zs[e] - WH1[e] * Zs[e + 1] - WH1[e - 1] * Zs[e - 1] - WV1[e] * Zs[e + p1] -
                   WV1[e - p1] * Zs[e - p1];
        };
        // ---- one V(1,1) cycle: z = M^-1 rin; rin is published in G0 by the caller -------------
        auto vcycle = [&](const double (&rin)[BR][BC], double (&z)[BR][BC]) {
            double t[BR][BC];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) z[q][c] = kMgOmega * DI0[ebase + q * np + c] * rin[q][c];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {       // residual of z = omega D^-1 r (neighbours from G0)
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
            for (int e = tid; e < N1; e += NT) {        // R1 = P^T t, Z1 = omega D1^-1 R1
                const int I = e % p1, J = e / p1;
                if (I < 1 || I >= m1 || J < 1 || J >= m1) continue;
                const int f = (2 * J) * np + 2 * I;
                const double rr = G1[f] + 0.5 * (G1[f - 1] + G1[f + 1] + G1[f - np] + G1[f + np]) +
                                  0.25 * (G1[f - np - 1] + G1[f - np + 1] + G1[f + np - 1] + G1[f + np + 1]);
                R1[e] = rr;
                Z1[e] = kMgOmega * DI1[e] * rr;
            }
            __syncthreads();
            for (int e = tid; e < N1; e += NT) {        // level-1 residual of the pre-smoothed Z1
                if (DI1[e] == 0.0) continue;
                T1[e] = R1[e] - A1(Z1, e);
            }
            __syncthreads();
            for (int a = tid; a < U2; a += NT) {         // R2 = P^T T1 on the level-2 unknowns
                const int I = a % (m2 - 1) + 1, J = a / (m2 - 1) + 1;
                const int f = (2 * J) * p1 + 2 * I;
                R2[a] = T1[f] + 0.5 * (T1[f - 1] + T1[f + 1] + T1[f - p1] + T1[f + p1]) +
                        0.25 * (T1[f - p1 - 1] + T1[f - p1 + 1] + T1[f + p1 - 1] + T1[f + p1 + 1]);
            }
            __syncthreads();
            // E2 = A2^-1 R2: row a by the thread pair (2a, 2a+1), fixed split of the sum
            for (int h = tid; h < 2 * ((U2 + 15) / 16) * 16; h += NT) {
                const int a = h >> 1, half = h & 1;
                double sum = 0.0;
                if (a < U2) {
                    const double *row = AI + a * U2;
                    double s0 = 0.0, s1 = 0.0;
                    for (int c = 2 * half; c < U2; c += 4) {
                        s0 = fma(row[c], R2[c], s0);
                        if (c + 1 < U2) s1 = fma(row[c + 1], R2[c + 1], s1);
                    }
                    sum = s0 + s1;
                }
                sum += __shfl_xor_sync(0xffffffffu, sum, 1);
                if (a < U2 && !half) E2[a] = sum;
            }
            __syncthreads();
            // level 1: S1 = smooth(Z1 + P E2), neighbours' corrected values recomputed
            auto e2at = [&](int I, int J) -> double {   // level-2 value at level-2 grid (I, J)
                return (I >= 1 && I < m2 && J >= 1 && J < m2) ? E2[(J - 1) * (m2 - 1) + I - 1] : 0.0;
            };
            auto zc1 = [&](int g) -> double {
                if (DI1[g] == 0.0) return 0.0;
                const int i = g % p1, j = g / p1, I = i >> 1, J = j >> 1;
                double v;
                if (!(i & 1) && !(j & 1)) v = e2at(I, J);
                else if (!(j & 1)) v = 0.5 * (e2at(I, J) + e2at(I + 1, J));
                else if (!(i & 1)) v = 0.5 * (e2at(I, J) + e2at(I, J + 1));
                else v = 0.25 * (e2at(I, J) + e2at(I + 1, J) + e2at(I, J + 1) + e2at(I + 1, J + 1));
                return Z1[g] + v;
            };
            for (int e = tid; e < N1; e += NT) {
                if (DI1[e] == 0.0) continue;
                const double z0 = zc1(e);
                const double az = D1[e] * z0 - WH1[e] * zc1(e + 1) - WH1[e - 1] * zc1(e - 1) -
                                  WV1[e] * zc1(e + p1) - WV1[e - p1] * zc1(e - p1);
                S1[e] = fma(kMgOmega * DI1[e], R1[e] - az, z0);
            }
            __syncthreads();
            // level 0: z += P S1, post-smooth; neighbours' corrected z = omega D^-1 r + P S1
            auto prol = [&](int e) -> double {
                const int i = e % np, j = e / np, I = i >> 1, J = j >> 1;
                if (i < 1 || i > nx || j < 1 || j > nx) return 0.0;
                const double *z2 = S1 + J * p1 + I;
                if (!(i & 1) && !(j & 1)) return z2[0];
                if (!(j & 1)) return 0.5 * (z2[0] + z2[1]);
                if (!(i & 1)) return 0.5 * (z2[0] + z2[p1]);
                return 0.25 * (z2[0] + z2[1] + z2[p1] + z2[p1 + 1]);
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
