// pcg_mg.cuh — on-chip CG with a four-level geometric-multigrid preconditioner, one CTA per sample.
//
// Same P1 discretisation as pde.cu (Z11/Z12); CG in the Chronopoulos-Gear single-reduction form
//     u = M^-1 r;  w = A u;  gamma = (r,u), delta = (w,u), rho = (r,r)      [one reduction]
//     beta = gamma/gamma_old;  alpha = gamma/(delta - beta gamma/alpha_old)
//     p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s,
// stopping on rho = ||r||_2^2 <= tol^2 ||b||_2^2 (Z13).
// M^-1 is one symmetric V(1,1) cycle over four nested "/" meshes (n, n/2, n/4, n/8 cells): damped
// Jacobi (omega = 0.8 on level 0, 1 on levels 1-2) pre- and post-smoothing, bilinear prolongation P,
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
// The kernel is bound by shared-memory wavefronts (ncu: LSU data pipe ~85% busy in the previous
// design), so this one minimises them:
//  * level 0 (fine): each thread owns a 2 x BR block of nodes with x, r, p, s, u and the coupling
//    weights in registers (the diagonal is summed from the couplings, not loaded); only the values
//    neighbours need are published, one grid per exchange, with a zero Dirichlet ring;
//  * grids of levels 0 and 1 store the even columns, then the odd columns of a row ("split"
//    rows), so the stride-2 accesses of restriction, prolongation and the 2-column thread blocks
//    are bank-conflict-free;
//  * level 1 runs on the whole CTA; the level-2/3 part of the cycle (49 + 9 unknowns at n = 32)
//    is a fixed linear map applied as one precomputed dense 49 x 49 product per iteration.
// Ten CTA barriers per CG iteration.  Reductions are fixed trees, so a sample's result does not
// depend on the CTA or launch split.
#pragma once
#include <type_traits>

namespace usfft {

// damped-Jacobi weights of the V(1,1) cycle: 0.8 on the fine level, 1.0 on every coarse level
// (tools/mg_omega_study.py: 14 -> 13 CG iterations at config 5, 13.6 -> 13 at config 3, never more)
constexpr double kMgOmega = 0.8, kMgOmegaCoarse = 1.0;

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

template <int NC>
struct Mg3 {
    static constexpr int n = NC, np = NC + 1, NP2 = np * np, HE = NC / 2 + 1;   // HE even columns
    static constexpr int m1 = NC / 2, p1 = m1 + 1, N1 = p1 * p1, H1 = m1 / 2 + 1;  // smoothed level 1
    static constexpr int m2 = NC / 4, p2 = m2 + 1, N2 = p2 * p2;      // smoothed level 2 (natural)
    static constexpr int m3 = NC / 8, p3 = m3 + 1, N3 = p3 * p3, U3 = (m3 - 1) * (m3 - 1);  // exact
    static constexpr int U2 = (m2 - 1) * (m2 - 1), HK = (U2 + 1) / 2;
    // shared-memory layout (doubles): fine grids omega D^-1, G0 (z0 = omega D^-1 r), G1 (fine
    // residual, then u); level 1 WH, WV, omega D^-1, R, Z, T, S (split rows); level 2 WH, WV, D,
    // omega D^-1 (setup), S (natural rows, zero ring), R (compact); the level-2 cycle matrix K
    // (U2 x U2, column-major); level 3 WH, WV and the dense inverse A3^-1 (setup); B, C (setup).
    // The per-triangle coefficient table of the setup aliases G0..G1.
    static constexpr int oDI0 = 0, oG0 = NP2, oG1 = 2 * NP2;
    static constexpr int oL1 = 3 * NP2;
    static constexpr int oL2 = oL1 + 7 * N1;             // WH2, WV2, D2, DI2, S2 (N2 each), R2 (U2)
    static constexpr int oK = oL2 + 5 * N2 + 2 * HK;     // R2 padded to 2 HK (zero tail)
    // K: 2 HK columns of U2; the second half starts KPAD doubles later so that the two halves a
    // warp reads together (thread pairs (i, h)) fall into disjoint shared-memory banks
    static constexpr int KPAD = (8 - (HK * U2) % 16 + 16) % 16;
    static constexpr int oWH3 = oK + 2 * HK * U2 + KPAD, oWV3 = oWH3 + N3, oAI = oWV3 + N3;
    static constexpr int oB = oAI + U3 * U3, oC = oB + U3 * U2;
    __host__ __device__ static constexpr int doubles() { return oC + U3 * U2; }
    // the psi tables S[plane][j][m] ((1 or 2) x d x (3n+1)) are staged after these when they
    // have at most SMAX doubles (n = 32: 9208 + 4096 doubles, two CTAs still fit an SM)
    static constexpr int SMAX = 4096;
    // split-row slot of column i (even columns first)
    __host__ __device__ static constexpr int col1s(int i) { return (i & 1) ? H1 + (i >> 1) : (i >> 1); }
};

template <int NC, int BC, int BR, int LX, int NWARP, int MINB>
__global__ void __launch_bounds__(NWARP * 32, MINB)
k_pcg_mg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
         int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
         double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S,
         const double *__restrict__ Bt) {
    using L = Mg3<NC>;
    constexpr int RGW = 32 / LX, NRG = NWARP * RGW, NT = NWARP * 32;
    constexpr int n = NC, nx = n - 1, np = n + 1, W = 3 * n + 1, NP2 = L::NP2, HE = L::HE;
    constexpr int m1 = L::m1, P1 = L::p1, N1 = L::N1, H1 = L::H1, m2 = L::m2, P2 = L::p2, N2 = L::N2;
    constexpr int m3 = L::m3, p3 = L::p3, U3 = L::U3, U2 = L::U2, HK = L::HK;
    static_assert(BC == 2 && BR % 2 == 0, "2 x BR node blocks (one odd and one even column)");
    static_assert(LX * BC >= nx && NRG * BR >= nx, "block mapping must cover the mesh");
    static_assert(NT % n == 0, "coefficient mapping: whole mesh rows per pass");
    static_assert(2 * n * n <= 2 * NP2, "coefficient table must fit in G0..G1");
    static_assert(U3 >= 1 && U3 <= 32, "level 3 is inverted by one warp");
    static_assert(2 * U2 <= NT, "two threads per row of the level-2 cycle matrix");
    constexpr bool XP_SMEM = MINB * NWARP >= 12;       // >= 12 resident warps per SM: x, p in smem
    extern __shared__ double sm[];
    __shared__ double red[4][NWARP];
    __shared__ double th_amp2[2][kMaxD];                 // amp_j theta_j(y_j): the current / the next sample
    double *DI0 = sm + L::oDI0, *G0 = sm + L::oG0, *G1 = sm + L::oG1, *aT = G0;
    double *WH1 = sm + L::oL1, *WV1 = WH1 + N1, *DI1 = WH1 + 2 * N1, *R1 = WH1 + 3 * N1;
    double *Z1 = WH1 + 4 * N1, *T1 = WH1 + 5 * N1, *S1 = WH1 + 6 * N1;
    double *WH2 = sm + L::oL2, *WV2 = WH2 + N2, *D2 = WH2 + 2 * N2, *DI2 = WH2 + 3 * N2;
    double *S2 = WH2 + 4 * N2, *R2 = WH2 + 5 * N2, *Kt = sm + L::oK;
    double *WH3 = sm + L::oWH3, *WV3 = sm + L::oWV3, *AI = sm + L::oAI, *Bm = sm + L::oB, *Cm = sm + L::oC;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = lane / LX, lx = lane % LX;
    const int rg = warp * RGW + seg;
    const int col0 = lx * BC, row0 = rg * BR;            // block: columns 2lx+1 (odd), 2lx+2 (even)
    const double inv_n3 = 1.0 / ((double)n * n * n);

    // interior nodes of a coarse level (I, J in [1, M-1]), q = first + k * STRIDE.  Lanes walk
    // rows of M slots (I = 1..M, the ring column I = M masked), so a warp's accesses cover whole
    // 16-slot row segments of the split-row grids and stay bank-conflict-free.
    auto for_interior = [](auto mconst, auto sconst, int first, auto body) {
        constexpr int M = decltype(mconst)::value, U = M * (M - 1);
        constexpr int STRIDE = decltype(sconst)::value;
#pragma unroll
        for (int k = 0; k < (U + STRIDE - 1) / STRIDE; ++k) {
            const int q = first + k * STRIDE, I = q % M + 1, J = q / M + 1;
            if (q < U && I < M) body(I, J);
        }
    };
    using C1 = std::integral_constant<int, m1>;
    using C2 = std::integral_constant<int, m2>;
    using SCTA = std::integral_constant<int, NT>;

    // the sample-independent sin table, staged once per CTA (L1 reloads of it were ~500 cycles
    // per coefficient term in the probe)
    const int s_cnt = (Q.psi ? 2 : 1) * Q.d * W;         // X plane (+ Y plane unless psi = 0)
    const bool s_staged = s_cnt <= L::SMAX;
    double *Ssm = sm + L::doubles() + (XP_SMEM ? 2 * BC * BR * NT : 0);
    if (s_staged)
        for (int e = tid; e < s_cnt; e += NT) Ssm[e] = __ldg(S + e);
    const double *Stab = s_staged ? Ssm : S;
    const double *StabY = Stab + (Q.psi ? Q.d * W : 0);

    // amp_j theta_j(y_j) of sample bl of this launch: the first sample's here, every later one during
    // the previous sample's setup (by the warps that wait for the A3 inverse), off the critical path
    auto theta_amp = [&](int64_t bl, int first, int stride, double *dst) {
        for (int j = first; j < Q.d; j += stride) {      // d may exceed the CTA (n = 16: 32 threads)
            const double y = nodes ? nodes[(int64_t)j * nb + bl] : lattice_node(P, b0 + bl, j);
            dst[j] = Q.amp[j] * theta_of(Q.theta, y, Q.delta);
        }
    };
    if ((int64_t)blockIdx.x < nb) theta_amp(blockIdx.x, tid, NT, th_amp2[0]);
    int tbuf = 0;

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        // ---- K3: coefficients ----------------------------------------------------------------
        const double *th_amp = th_amp2[tbuf];
        double *th_next = th_amp2[tbuf ^ 1];
        tbuf ^= 1;
        __syncthreads();
        {   // per-triangle a = 1 + sum_j amp_j theta_j S_j(ma) S_j(mb) (or exp) of the fine mesh,
            // a rank-d product: thread (ci0, cj0) owns a KI x KJ tile of cells (ci0 + CIS a,
            // cj0 + CJS b) in registers
            constexpr int KI = NT >= 4 * n ? 4 : 2, CIS = n / KI, CJS = NT / CIS, KJ = n / CJS;
            static_assert(NT % CIS == 0 && n % CJS == 0, "coefficient tile mapping");
            const int ci0 = tid % CIS, cj0 = tid / CIS;
            double slo[KI][KJ], sup[KI][KJ];
#pragma unroll
            for (int a = 0; a < KI; ++a)
#pragma unroll
                for (int k = 0; k < KJ; ++k) slo[a][k] = sup[a][k] = 0.0;
#pragma unroll 2
            for (int j = 0; j < Q.d; ++j) {
                const double *Sj = Stab + j * W, *Sy = StabY + j * W;
                const double am = th_amp[j];
                double tlo[KI], tup[KI], vlo[KJ], vup[KJ];
#pragma unroll
                for (int a = 0; a < KI; ++a) {
                    tlo[a] = am * Sj[3 * (ci0 + CIS * a) + 2];
                    tup[a] = am * Sj[3 * (ci0 + CIS * a) + 1];
                }
#pragma unroll
                for (int k = 0; k < KJ; ++k) {
                    vlo[k] = Sy[3 * (cj0 + CJS * k) + 1];
                    vup[k] = Sy[3 * (cj0 + CJS * k) + 2];
                }
#pragma unroll
                for (int a = 0; a < KI; ++a)
#pragma unroll
                    for (int k = 0; k < KJ; ++k) {
                        slo[a][k] = fma(tlo[a], vlo[k], slo[a][k]);
                        sup[a][k] = fma(tup[a], vup[k], sup[a][k]);
                    }
            }
#pragma unroll
            for (int a = 0; a < KI; ++a)
#pragma unroll
                for (int k = 0; k < KJ; ++k) {
                    const int cell = (cj0 + CJS * k) * n + ci0 + CIS * a;
                    aT[cell] = Q.form == 0 ? 1.0 + slo[a][k] : exp(slo[a][k]);          // lower plane
                    aT[n * n + cell] = Q.form == 0 ? 1.0 + sup[a][k] : exp(sup[a][k]);  // upper plane
                }
        }
        __syncthreads();
        // a at the centroid of T_lo / T_up of cell (ci, cj) of the mesh with cell width 2^sh h: the
        // fine triangle with the same centroid (abscissae ma, mb in units of h/3)
        // ma = 3 ci p + ra, mb = 3 cj p + rb with p = 2^sh and (ra, rb) = (2p, p) below / (p, 2p)
        // above the diagonal, so ma / 3 = ci p + ra / 3 and ma % 3 = ra % 3: no run-time division
        auto fcoef = [&](int ci, int cj, int up, int sh) -> double {
            const int p = 1 << sh, ra = up ? p : 2 * p, rb = up ? 2 * p : p;
            return aT[(ra % 3 == 1 ? n * n : 0) + (cj * p + rb / 3) * n + ci * p + ra / 3];
        };
        // edge weights of node (i, j) of the mesh with M cells of width 2^sh h: to (i+1, j), (i, j+1)
        auto wh = [&](int i, int j, int M, int sh) -> double {
            return (i < M && j >= 1 && j < M) ? 0.5 * (fcoef(i, j, 0, sh) + fcoef(i, j - 1, 1, sh)) : 0.0;
        };
        auto wv = [&](int i, int j, int M, int sh) -> double {
            return (j < M && i >= 1 && i < M) ? 0.5 * (fcoef(i, j, 1, sh) + fcoef(i - 1, j, 0, sh)) : 0.0;
        };
        // fine couplings (ring edges included), read straight from the lower / upper planes:
        // edge (i, j)-(i+1, j) = (a_lo(i, j) + a_up(i, j-1)) / 2, (i, j)-(i, j+1) = (a_up(i, j) + a_lo(i-1, j)) / 2
        double cE[BR][BC + 1], cN[BR + 1][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c <= BC; ++c) {
                const int i = col0 + c, j = row0 + q + 1;
                cE[q][c] = (i <= nx && j <= nx) ? 0.5 * (aT[j * n + i] + aT[n * n + (j - 1) * n + i]) : 0.0;
            }
#pragma unroll
        for (int q = 0; q <= BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = row0 + q;
                cN[q][c] = (i <= nx && j <= nx) ? 0.5 * (aT[n * n + j * n + i] + aT[j * n + i - 1]) : 0.0;
            }
        for (int e = tid; e < N1; e += NT) {             // level 1 (split rows)
            const int J = e / P1, s = e % P1, I = s < H1 ? 2 * s : 2 * (s - H1) + 1;
            WH1[e] = wh(I, J, m1, 1);
            WV1[e] = wv(I, J, m1, 1);
            R1[e] = Z1[e] = T1[e] = S1[e] = 0.0;
        }
        for (int e = tid; e < N2; e += NT) {             // level 2 (natural rows)
            const int I = e % P2, J = e / P2;
            WH2[e] = wh(I, J, m2, 2);
            WV2[e] = wv(I, J, m2, 2);
            S2[e] = 0.0;
        }
        for (int e = tid; e < L::N3; e += NT) {
            const int I = e % p3, J = e / p3;
            WH3[e] = wh(I, J, m3, 3);
            WV3[e] = wv(I, J, m3, 3);
        }
        __syncthreads();                                 // aT is dead from here on
        // warps >= 1 form the level-1/2 diagonals while warp 0 assembles and inverts A3
        constexpr int HB = NWARP > 1 ? 32 : 0, HS = NT - HB;
        if (tid >= HB) {
            const int ht = tid - HB;
            if (bl + gridDim.x < nb) theta_amp(bl + gridDim.x, ht, HS, th_next);
            for (int e = ht; e < 4 * n; e += HS) {       // zero rings of G0, G1 (aT aliased them)
                const int side = e / n, o = e % n;       // ring walk: bottom, right, top, left
                const int i = side == 0 ? o : side == 1 ? n : side == 2 ? n - o : 0;
                const int j = side == 0 ? 0 : side == 1 ? o : side == 2 ? n : n - o;
                const int g = j * np + ((i & 1) ? HE + (i >> 1) : (i >> 1));
                G0[g] = G1[g] = 0.0;
            }
            for (int e = ht; e < N1; e += HS) {          // level-1 omega D^-1 (same sum as apply1)
                const int J = e / P1, s = e % P1, I = s < H1 ? 2 * s : 2 * (s - H1) + 1;
                const bool in = I >= 1 && I < m1 && J >= 1 && J < m1;
                const double dv = in ? WH1[e] + WH1[J * P1 + L::col1s(I - 1)] + WV1[e] + WV1[e - P1] : 1.0;
                DI1[e] = in ? kMgOmegaCoarse * (1.0 / dv) : 0.0;
            }
            for (int e = ht; e < N2; e += HS) {
                const int I = e % P2, J = e / P2;
                const bool in = I >= 1 && I < m2 && J >= 1 && J < m2;
                const double dv = in ? WH2[e] + WH2[e - 1] + WV2[e] + WV2[e - P2] : 0.0;
                D2[e] = dv;
                DI2[e] = in ? kMgOmegaCoarse * (1.0 / dv) : 0.0;
            }
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)                     // omega D^-1 of the own nodes (0 off-mesh);
#pragma unroll                                           // the diagonal in the order of diag() below
            for (int c = 0; c < BC; ++c) {
                const double dv = cE[q][c + 1] + cE[q][c] + cN[q + 1][c] + cN[q][c];
                DI0[(row0 + 1 + q) * np + ((c & 1) == 0 ? HE + lx + (c >> 1) : lx + ((c + 1) >> 1))] =
                    (col0 + c + 1 <= nx && row0 + q + 1 <= nx) ? kMgOmega * rcp_pos(dv) : 0.0;
            }
        if (warp == 0) {   // in-place Gauss-Jordan inverse of the coarsest operator (SPD, tiny):
            // lane i assembles row i of A3 (5-point, rediscretised) in registers; the pivot row of
            // each step comes by shuffles
            const int ri = lane < U3 ? lane : 0;
            const int ia = ri % (m3 - 1) + 1, ja = ri / (m3 - 1) + 1, g = ja * p3 + ia;
            const double wr = WH3[g], wl = WH3[g - 1], wu = WV3[g], wd = WV3[g - p3];
            double a[U3];
#pragma unroll
            for (int c = 0; c < U3; ++c)
                a[c] = c == ri ? wr + wl + wu + wd
                     : (c == ri + 1 && ia < m3 - 1) ? -wr
                     : (c == ri - 1 && ia > 1) ? -wl
                     : (c == ri + (m3 - 1) && ja < m3 - 1) ? -wu
                     : (c == ri - (m3 - 1) && ja > 1) ? -wd : 0.0;
#pragma unroll
            for (int k = 0; k < U3; ++k) {
                double prow[U3];
#pragma unroll
                for (int c = 0; c < U3; ++c) prow[c] = __shfl_sync(0xffffffffu, a[c], k);
                const double piv = rcp_pos(prow[k]);             // SPD: positive pivots
                const double f = -a[k] * piv;
#pragma unroll
                for (int c = 0; c < U3; ++c) {
                    if (lane == k) a[c] = c == k ? piv : prow[c] * piv;
                    else a[c] = c == k ? f : fma(f, prow[c], a[c]);
                }
            }
            __syncwarp();
            if (lane < U3) {
#pragma unroll
                for (int c = 0; c < U3; ++c) AI[lane * U3 + c] = a[c];
            }
        }
        __syncthreads();
        // The level-2 part of the cycle is a fixed linear map R2 -> S2 (damped-Jacobi pre-smoothing,
        // exact level-3 correction, post-smoothing):  with Dw = omega D2^-1,
        //   S2 = K R2,  K = 2 Dw - Dw A2 Dw + B^T A3^-1 B,  B = P3^T (I - A2 Dw)   (U3 x U2),
        // formed once per sample so each CG iteration applies it as one dense product.
        for (int e = tid; e < U3 * U2; e += NT) {        // B[r][k] = sum_m w(r, m) (I - A2 Dw)[m][k]
            const int r = e / U2, k = e % U2;
            const int Ir = r % (m3 - 1) + 1, Jr = r / (m3 - 1) + 1;
            const int Ik = k % (m2 - 1) + 1, Jk = k / (m2 - 1) + 1, ek = Jk * P2 + Ik;
            const double dwk = DI2[ek];
            // restriction weight of level-2 node (Im, Jm) for level-3 node r (0 off the stencil)
            auto wr = [&](int Im, int Jm) -> double {
                const int ax = abs(Im - 2 * Ir), ay = abs(Jm - 2 * Jr);
                return (ax > 1 || ay > 1) ? 0.0 : (ax ? 0.5 : 1.0) * (ay ? 0.5 : 1.0);
            };
            // the rows m of (I - A2 Dw) with a nonzero in column k: m = k and its 4 neighbours
            double v = wr(Ik, Jk) * (1.0 - D2[ek] * dwk);
            v = fma(wr(Ik + 1, Jk), WH2[ek] * dwk, v);
            v = fma(wr(Ik - 1, Jk), WH2[ek - 1] * dwk, v);
            v = fma(wr(Ik, Jk + 1), WV2[ek] * dwk, v);
            v = fma(wr(Ik, Jk - 1), WV2[ek - P2] * dwk, v);
            Bm[e] = v;
        }
        __syncthreads();
        for (int e = tid; e < U3 * U2; e += NT) {        // C = A3^-1 B
            const int r = e / U2, k = e % U2;
            double v = 0.0;
            for (int c = 0; c < U3; ++c) v = fma(AI[r * U3 + c], Bm[c * U2 + k], v);
            Cm[e] = v;
        }
        __syncthreads();
        auto kix = [](int col, int row) -> int { return col * U2 + row + (col >= HK ? L::KPAD : 0); };
        for (int e = U2 * U2 + tid; e < 2 * HK * U2; e += NT) Kt[kix(e / U2, e % U2)] = 0.0;   // zero pad column(s)
        if (tid < 2 * HK - U2) R2[U2 + tid] = 0.0;                           // and R2 tail
        {   // K = B^T C (rank-U3 product) in register tiles: thread (ti, tk) of a 16 x NT/16 grid
            // owns rows ti + 16 m and columns tk + TK n
            constexpr int TK = NT / 16, RI = (U2 + 15) / 16, CK = (U2 + TK - 1) / TK;
            const int ti = tid % 16, tk = tid / 16;
            double acc[RI][CK];
#pragma unroll
            for (int m = 0; m < RI; ++m)
#pragma unroll
                for (int q = 0; q < CK; ++q) acc[m][q] = 0.0;
#pragma unroll 3
            for (int r = 0; r < U3; ++r) {
                double bv[RI], cv[CK];
#pragma unroll
                for (int m = 0; m < RI; ++m) bv[m] = Bm[r * U2 + min(ti + 16 * m, U2 - 1)];
#pragma unroll
                for (int q = 0; q < CK; ++q) cv[q] = Cm[r * U2 + min(tk + TK * q, U2 - 1)];
#pragma unroll
                for (int m = 0; m < RI; ++m)
#pragma unroll
                    for (int q = 0; q < CK; ++q) acc[m][q] = fma(bv[m], cv[q], acc[m][q]);
            }
#pragma unroll
            for (int m = 0; m < RI; ++m)
#pragma unroll
                for (int q = 0; q < CK; ++q) {
                    const int i = ti + 16 * m, k = tk + TK * q;
                    if (i < U2 && k < U2) Kt[kix(k, i)] = acc[m][q];
                }
        }
        __syncthreads();
        for (int e = tid; e < 5 * U2; e += NT) {         // + 2 Dw - Dw A2 Dw (5-point), row i
            const int i = e % U2, d = e / U2;
            const int Ii = i % (m2 - 1) + 1, Ji = i / (m2 - 1) + 1, ei = Ji * P2 + Ii;
            const double dwi = DI2[ei];
            if (d == 0) Kt[kix(i, i)] += fma(-dwi * D2[ei], dwi, 2.0 * dwi);
            else if (d == 1 && Ii < m2 - 1) Kt[kix(i + 1, i)] += dwi * WH2[ei] * DI2[ei + 1];
            else if (d == 2 && Ii > 1) Kt[kix(i - 1, i)] += dwi * WH2[ei - 1] * DI2[ei - 1];
            else if (d == 3 && Ji < m2 - 1) Kt[kix(i + (m2 - 1), i)] += dwi * WV2[ei] * DI2[ei + P2];
            else if (d == 4 && Ji > 1) Kt[kix(i - (m2 - 1), i)] += dwi * WV2[ei - P2] * DI2[ei - P2];
        }
        // (the first barriers of the CG loop order these writes before their uses)

        // ---- level-0 addressing: node (col0 + 1 + c, row0 + 1 + q), c in [-1, BC], q in [-1, BR];
        // c even is an odd column (slot HE + lx + c/2), c odd an even column (slot lx + (c+1)/2)
        auto fe = [&](int c, int q) -> int {
            const int slot = (c & 1) == 0 ? HE + lx + (c >> 1) : lx + ((c + 1) >> 1);
            return (row0 + 1 + q) * np + slot;
        };
        auto valid = [&](int q, int c) { return col0 + c + 1 <= nx && row0 + q + 1 <= nx; };
        auto publish = [&](double *Gd, const double (&v)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) Gd[fe(c, q)] = v[q][c];
        };
        auto diag = [&](int q, int c) -> double {        // same summation order as DI0
            return cE[q][c + 1] + cE[q][c] + cN[q + 1][c] + cN[q][c];
        };
        // A v at the own nodes, neighbour values from the published grid Gs; invalid nodes give 0
        auto apply_fine = [&](const double *Gs, const double (&v)[BR][BC], double (&out)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const double vl = c > 0 ? v[q][c - 1] : Gs[fe(c - 1, q)];
                    const double vr = c + 1 < BC ? v[q][c + 1] : Gs[fe(c + 1, q)];
                    const double vd = q > 0 ? v[q - 1][c] : Gs[fe(c, q - 1)];
                    const double vu = q + 1 < BR ? v[q + 1][c] : Gs[fe(c, q + 1)];
                    double a = diag(q, c) * v[q][c];
                    a = fma(-cE[q][c + 1], vr, a);
                    a = fma(-cE[q][c], vl, a);
                    a = fma(-cN[q + 1][c], vu, a);
                    a = fma(-cN[q][c], vd, a);
                    out[q][c] = valid(q, c) ? a : 0.0;
                }
        };
        // level-1 node (I, J): split-row offset
        auto e1 = [](int I, int J) -> int { return J * P1 + L::col1s(I); };
        // level-1 operator at (I, J) (diagonal summed from the weights, same order as DI1)
        auto apply1 = [&](const double *Zs, int I, int J) -> double {
            const int e = e1(I, J), el = e1(I - 1, J), er = e1(I + 1, J);
            const double whe = WH1[e], whl = WH1[el], wve = WV1[e], wvd = WV1[e - P1];
            return (whe + whl + wve + wvd) * Zs[e] - whe * Zs[er] - whl * Zs[el] - wve * Zs[e + P1] -
                   wvd * Zs[e - P1];
        };
        // bilinear prolongation of a coarse grid Xc (natural rows of length pc, zero ring) to node (i, j)
        auto prol2 = [](const double *Xc, int pc, int i, int j) -> double {
            const double *z2 = Xc + (j >> 1) * pc + (i >> 1);
            if (!(i & 1) && !(j & 1)) return z2[0];
            if (!(j & 1)) return 0.5 * (z2[0] + z2[1]);
            if (!(i & 1)) return 0.5 * (z2[0] + z2[pc]);
            return 0.25 * (z2[0] + z2[1] + z2[pc] + z2[pc + 1]);
        };
        // the same, branch-free: the weights are 0, 1/2, 1/4 or 1, so the result equals prol2 bit
        // for bit.  Used on the 25-value level-3 grid, where the lanes' loads are broadcasts.
        auto prol2w = [](const double *Xc, int pc, int i, int j) -> double {
            const double *z2 = Xc + (j >> 1) * pc + (i >> 1);
            const double wx1 = (i & 1) ? 0.5 : 0.0, wx0 = (i & 1) ? 0.5 : 1.0;
            const double wy1 = (j & 1) ? 0.5 : 0.0, wy0 = (j & 1) ? 0.5 : 1.0;
            return fma(wx1 * wy1, z2[pc + 1], fma(wx0 * wy1, z2[pc], fma(wx1 * wy0, z2[1], wx0 * wy0 * z2[0])));
        };

        // ---- one V(1,1) cycle: z = M^-1 rin ------------------------------------------------
        auto vcycle = [&](const double (&rin)[BR][BC], double (&z)[BR][BC]) {
            double t[BR][BC];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) z[q][c] = DI0[fe(c, q)] * rin[q][c];   // z0 = omega D^-1 r
            publish(G0, z);
            __syncthreads();
            apply_fine(G0, z, t);
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) t[q][c] = rin[q][c] - t[q][c];       // fine residual
            publish(G1, t);
            __syncthreads();
            // R1 = P^T t (9-point, split rows of G1), Z1 = omega D1^-1 R1
            for_interior(C1{}, SCTA{}, tid, [&](int I, int J) {
                const int f = 2 * J * np, c = I, l = HE + I - 1, r = HE + I;
                const double rr = G1[f + c] + 0.5 * (G1[f + l] + G1[f + r] + G1[f - np + c] + G1[f + np + c]) +
                                  0.25 * (G1[f - np + l] + G1[f - np + r] + G1[f + np + l] + G1[f + np + r]);
                const int e = e1(I, J);
                R1[e] = rr;
                Z1[e] = DI1[e] * rr;
            });
            __syncthreads();
            for_interior(C1{}, SCTA{}, tid, [&](int I, int J) { T1[e1(I, J)] = R1[e1(I, J)] - apply1(Z1, I, J); });
            __syncthreads();
            for_interior(C2{}, SCTA{}, tid, [&](int I, int J) {      // R2 = P^T T1 (compact)
                const int f = 2 * J * P1, c = I, l = H1 + I - 1, r = H1 + I;
                R2[(J - 1) * (m2 - 1) + I - 1] =
                    T1[f + c] + 0.5 * (T1[f + l] + T1[f + r] + T1[f - P1 + c] + T1[f + P1 + c]) +
                    0.25 * (T1[f - P1 + l] + T1[f - P1 + r] + T1[f + P1 + l] + T1[f + P1 + r]);
            });
            __syncthreads();
            if (warp < (2 * U2 + 31) / 32) {                     // S2 = K R2 (levels 2 and 3)
                // thread (i, h): half h of row i; K and R2 carry a zero column / entry past U2
                const int h = tid & 1, i = min(tid >> 1, U2 - 1);
                const bool own = tid < 2 * U2;
                const double *kp = Kt + h * (HK * U2 + L::KPAD) + i, *rp = R2 + h * HK;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;    // four chains (DFMA latency)
#pragma unroll
                for (int c = 0; c < HK; c += 4) {
                    a0 = fma(kp[c * U2], rp[c], a0);
                    if (c + 1 < HK) a1 = fma(kp[(c + 1) * U2], rp[c + 1], a1);
                    if (c + 2 < HK) a2 = fma(kp[(c + 2) * U2], rp[c + 2], a2);
                    if (c + 3 < HK) a3 = fma(kp[(c + 3) * U2], rp[c + 3], a3);
                }
                double sv = (a0 + a1) + (a2 + a3);
                sv += __shfl_xor_sync(0xffffffffu, sv, 1);       // whole warps take part
                if (own && h == 0) S2[(i / (m2 - 1) + 1) * P2 + i % (m2 - 1) + 1] = sv;
            }
            __syncthreads();
            for_interior(C1{}, SCTA{}, tid, [&](int I, int J) {      // Zc1 = Z1 + P S2 (in place)
                Z1[e1(I, J)] += prol2w(S2, P2, I, J);
            });
            __syncthreads();
            for_interior(C1{}, SCTA{}, tid, [&](int I, int J) {      // S1 = smooth(Zc1)
                const int e = e1(I, J);
                S1[e] = fma(DI1[e], R1[e] - apply1(Z1, I, J), Z1[e]);
            });
            __syncthreads();
            // level 0: z = z0 + P S1, post-smooth.  The coarse values this block and its
            // neighbours need form a (BR/2 + 2) x 3 window of S1; the parity of every fine node
            // relative to (col0, row0) is a compile-time constant.
            constexpr int XW = BC / 2 + 2, YW = BR / 2 + 2;
            double cw[YW][XW];
#pragma unroll
            for (int yy = 0; yy < YW; ++yy)
#pragma unroll
                for (int xx = 0; xx < XW; ++xx) {
                    const int X = lx + xx, Y = (row0 >> 1) + yy;
                    cw[yy][xx] = (X <= m1 && Y <= m1) ? S1[Y * P1 + L::col1s(X)] : 0.0;
                }
            auto pw = [&](int c, int q) -> double {  // (P S1) at node (col0 + 1 + c, row0 + 1 + q)
                const int fi = 1 + c, fj = 1 + q, x0 = fi >> 1, y0 = fj >> 1;
                if (!(fi & 1) && !(fj & 1)) return cw[y0][x0];
                if (!(fj & 1)) return 0.5 * (cw[y0][x0] + cw[y0][x0 + 1]);
                if (!(fi & 1)) return 0.5 * (cw[y0][x0] + cw[y0 + 1][x0]);
                return 0.25 * (cw[y0][x0] + cw[y0][x0 + 1] + cw[y0 + 1][x0] + cw[y0 + 1][x0 + 1]);
            };
            // post-smoothing of z0 + E, E = P S1:  z0 + E + omega D^-1 (t - A E), with t = r - A z0
            // the fine residual still in registers; the neighbours' E come from the window
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const double ec = pw(c, q);
                    double a = diag(q, c) * ec;
                    a = fma(-cE[q][c + 1], pw(c + 1, q), a);
                    a = fma(-cE[q][c], pw(c - 1, q), a);
                    a = fma(-cN[q + 1][c], pw(c, q + 1), a);
                    a = fma(-cN[q][c], pw(c, q - 1), a);
                    z[q][c] = valid(q, c) ? fma(DI0[fe(c, q)], t[q][c] - a, z[q][c] + ec) : 0.0;
                }
        };

        // ---- Chronopoulos-Gear PCG ----------------------------------------------------------
        // x and p are touched once per iteration: with XP_SMEM they live in thread-private shared
        // slots (conflict-free [k][tid] layout) to free registers for a third CTA per SM
        double xr[XP_SMEM ? 1 : BR][BC], pr[XP_SMEM ? 1 : BR][BC], r[BR][BC], s[BR][BC];
        double *const xs = sm + L::doubles() + tid, *const ps = xs + BR * BC * NT;
        auto xref = [&](int q, int c) -> double & { return XP_SMEM ? xs[(q * BC + c) * NT] : xr[XP_SMEM ? 0 : q][c]; };
        auto pref = [&](int q, int c) -> double & { return XP_SMEM ? ps[(q * BC + c) * NT] : pr[XP_SMEM ? 0 : q][c]; };
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                xref(q, c) = pref(q, c) = s[q][c] = 0.0;
                r[q][c] = !valid(q, c) ? 0.0                                        // b = h^2 x2, or
                        : Bt ? __ldg(Bt + (row0 + q) * nx + col0 + c)                // the load table
                             : (double)(row0 + q + 1) * inv_n3;
            }
        // x0 = 0, r0 = b (Z13); ||b||^2 is the first iteration's (r, r)
        double rho = 0.0, rho_prev = 0.0, bb = 0.0, g_inv = 0.0, ga_inv = 0.0;
        bool conv = false;
        int it = 0;
        for (int k = 0;; ++k) {
            double uu[BR][BC], w[BR][BC];
            vcycle(r, uu);
            publish(G1, uu);                                 // G1 (fine residual) is free again
            __syncthreads();
            apply_fine(G1, uu, w);
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
            double gs[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
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
            rho_prev = rho;
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
                    const double pn = fma(beta, pref(q, c), uu[q][c]);
                    pref(q, c) = pn;
                    s[q][c] = fma(beta, s[q][c], w[q][c]);
                    xref(q, c) = fma(alpha, pn, xref(q, c));
                    r[q][c] = fma(-alpha, s[q][c], r[q][c]);
                }
            // Early stopping test (as in pcg_cl.cuh): when the residual decay predicts (r,r) <=
            // 4 tol^2 (b,b) for the new r, reduce (r,r) now instead of after one more V-cycle.  The
            // tree is the one (r,r) takes above (lane 16 of each warp: own + partner at offsets
            // 16, 8, 4, 2, 1, then the fixed warp tree), so the value and the decision are those
            // of the next iteration's test and x is the same.
            if (k > 0 && rho * rho <= 4.0 * Q.tol2 * bb * rho_prev && it + 1 < Q.maxit) {
                double a2 = 0.0;
#pragma unroll
                for (int q = 0; q < BR; ++q)
#pragma unroll
                    for (int c = 0; c < BC; ++c) a2 = fma(r[q][c], r[q][c], a2);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
                __syncthreads();                         // everyone has read red[] of this iteration
                if (lane == 16) red[2][warp] = a2;
                __syncthreads();
                double tt[NWARP];
#pragma unroll
                for (int ww = 0; ww < NWARP; ++ww) tt[ww] = red[2][ww];
#pragma unroll
                for (int h = 1; h < NWARP; h <<= 1)
#pragma unroll
                    for (int ww = 0; ww + h < NWARP; ww += 2 * h) tt[ww] += tt[ww + h];
                if (tt[0] <= Q.tol2 * bb) {
                    rho = tt[0];
                    conv = true;
                    ++it;
                    break;
                }
            }
            ++it;
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c)
                if (valid(q, c)) u[(int64_t)((row0 + q) * nx + col0 + c) * ldu + bl] = xref(q, c);
        if (tid == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rho / bb);
            if (noconv && !conv) atomicAdd(noconv, 1);
        }
        __syncthreads();
    }
}

}  // namespace usfft
