// pcg_cl.cuh — multigrid-preconditioned CG for the large meshes (n = 64, 128: configs 3-5), one
// thread-block CLUSTER per sample, the whole solve on chip.
//
// Same discretisation (Z11/Z12), the same Chronopoulos-Gear CG (one reduction per iteration,
// x0 = 0, stop on ||r||_2 <= tol ||b||_2, Z13) and the same preconditioner family as
// pcg_mg.cuh: one symmetric V(1,1) cycle, damped Jacobi (omega = 0.8) smoothing, bilinear P,
// R = P^T, coarse operators rediscretised from the fine per-triangle coefficients, and the
// bottom two levels (8 and 4 cells per side) as the fixed dense map K of pcg_mg.cuh.
//
// A sample of n = 128 (16129 unknowns) needs ~0.5 MB of fp64 state, more than one SM holds, so a
// cluster of CS CTAs (CS = 8 at n = 128, 4 at n = 64) shares it; CTA r of the cluster owns the
// fine rows j0+1 .. j0+HR, j0 = r HR, HR = n / CS = 16:
//  * level 0 (fine): each thread keeps a 2 x 4 block of nodes (x, r, p, s and the couplings) in
//    registers, as in pcg_mg.cuh; the values the stencil needs are published in shared memory
//    (split rows: even columns, then odd) and the strip's first / last row is also written into
//    the neighbour CTA's halo row through distributed shared memory (st.shared::cluster);
//  * level 1 (n/2 cells): distributed the same way (rows J0+1 .. J0+HR/2, one halo row per side);
//  * levels 2 .. (8 cells per side): replicated.  The restricted level-2 residual is gathered into
//    every CTA of the cluster (each CTA writes its own rows into all CS copies) and every CTA runs
//    the rest of the cycle locally with CTA barriers, so it needs no cluster synchronisation;
//  * reductions: CTA partials are written into every CTA's slot table and summed in rank order,
//    so all CTAs hold bit-identical scalars and take the same branch.
// A phase that reads what another CTA wrote is separated from the write by one cluster barrier
// (barrier.cluster.arrive.release / wait.acquire): eight per CG iteration.  The per-triangle
// coefficient table of each CTA's strip is read by the other CTAs (DSMEM) for the replicated
// levels' couplings during the setup.  Every quantity is computed in a fixed order independent of
// the cluster's placement and of the launch, so a sample's result is deterministic.
#pragma once
#include <cooperative_groups.h>

namespace usfft {

template <int NN, int CS>
struct ClC {
    static constexpr int n = NN, nx = n - 1, np = n + 1, HE = n / 2 + 1;
    static constexpr int HR = NN / CS;                       // fine rows per CTA
    static constexpr int BC = 2, BR = 4, LX = n / 2, NRG = HR / BR, NT = LX * NRG, NWARP = NT / 32;
    static constexpr int FR = (HR + 2) * np;                 // fine grid: local rows 0 .. HR+1
    static constexpr int m1 = n / 2, P1 = m1 + 1, H1 = m1 / 2 + 1, R1ROWS = HR / 2 + 2, F1 = R1ROWS * P1;
    static constexpr int HR1 = HR / 2, HR2 = HR / 4;        // own level-1 / level-2 rows
    // replicated levels 2 .. LK-1 (natural rows, zero ring); level LK has 8 cells (the K map)
    static constexpr int LK = NN == 64 ? 3 : NN == 128 ? 4 : -1;
    static_assert(LK > 0, "cluster multigrid compiled for n = 64, 128");
    static_assert(HR % 8 == 0 && LX % 32 == 0, "strip geometry");
    __host__ __device__ static constexpr int ml(int l) { return NN >> l; }
    __host__ __device__ static constexpr int Pl(int l) { return (NN >> l) + 1; }
    __host__ __device__ static constexpr int Nl(int l) { return ((NN >> l) + 1) * ((NN >> l) + 1); }
    static constexpr int mK = 8, PK = 9, NK = 81, UK = 49, HK = (UK + 1) / 2;
    static constexpr int mE = 4, PE = 5, NE = 25, UE = 9;
    static constexpr int KPAD = (8 - (HK * UK) % 16 + 16) % 16;
    static constexpr int ATR = HR + 2;                       // coefficient-table rows j0 .. j0+HR+1
    // shared-memory layout (doubles)
    static constexpr int oDI0 = 0, oG0 = FR, oG1 = 2 * FR;
    static constexpr int oL1 = 3 * FR;                       // WH1, WV1, DI1, R1, Z1, T1 (= S1)
    __host__ __device__ static constexpr int oLev(int l) {   // replicated level l: WH, WV, DI, R, Z, T (= S)
        int o = oL1 + 6 * F1;
        for (int q = 2; q < l; ++q) o += 6 * Nl(q);
        return o;
    }
    static constexpr int oKs = oLev(LK);                     // WHK, WVK, DK, DIK, SK (NK each), RK (2 HK)
    static constexpr int oKt = oKs + 5 * NK + 2 * HK;
    static constexpr int oWHE = oKt + 2 * HK * UK + KPAD, oWVE = oWHE + NE, oAI = oWVE + NE;
    static constexpr int oB = oAI + UE * UE, oC = oB + UE * UK;
    static constexpr int oRed = oC + UE * UK;                // [CS][4] cluster reduction slots
    static constexpr int oWred = oRed + 4 * CS;              // [4][NWARP] CTA reduction
    __host__ __device__ static constexpr int doubles() { return oWred + 4 * NWARP; }
    static_assert(2 * ATR * n <= 3 * FR, "coefficient table must fit in DI0 .. G1");
    static_assert(2 * UK <= NT, "two threads per row of K");
    static_assert(3 * CS <= 32, "one warp writes the reduction slots");
};

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_id_x() {
    unsigned v;
    asm("mov.u32 %0, %%clusterid.x;" : "=r"(v));
    return v;
}
__device__ __forceinline__ unsigned cluster_count_x() {
    unsigned v;
    asm("mov.u32 %0, %%nclusterid.x;" : "=r"(v));
    return v;
}

template <int NN, int CS, int MINB>
__global__ void __launch_bounds__(ClC<NN, CS>::NT, MINB)
k_pcg_cl(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
         int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
         double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S,
         const double *__restrict__ Bt) {
    using L = ClC<NN, CS>;
    namespace cg = cooperative_groups;
    constexpr int n = NN, nx = L::nx, np = L::np, HE = L::HE, HR = L::HR, BC = L::BC, BR = L::BR;
    constexpr int LX = L::LX, NRG = L::NRG, NT = L::NT, NWARP = L::NWARP, W = 3 * n + 1;
    constexpr int m1 = L::m1, P1 = L::P1, H1 = L::H1, HR1 = L::HR1, HR2 = L::HR2, LK = L::LK;
    constexpr int mK = L::mK, PK = L::PK, NK = L::NK, UK = L::UK, HK = L::HK;
    constexpr int mE = L::mE, PE = L::PE, UE = L::UE, ATR = L::ATR;
    extern __shared__ double sm[];
    __shared__ double th_amp[kMaxD];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int j0 = rank * HR, J0 = j0 / 2, J20 = j0 / 4;

    double *DI0 = sm + L::oDI0, *G0 = sm + L::oG0, *G1 = sm + L::oG1, *aT = sm;   // aT: setup only
    double *WH1 = sm + L::oL1, *WV1 = WH1 + L::F1, *DI1 = WH1 + 2 * L::F1, *R1 = WH1 + 3 * L::F1;
    double *Z1 = WH1 + 4 * L::F1, *T1 = WH1 + 5 * L::F1, *S1 = T1;
    double *WHK = sm + L::oKs, *WVK = WHK + NK, *DK = WHK + 2 * NK, *DIK = WHK + 3 * NK, *SK = WHK + 4 * NK;
    double *RK = WHK + 5 * NK, *Kt = sm + L::oKt;
    double *WHE = sm + L::oWHE, *WVE = sm + L::oWVE, *AI = sm + L::oAI, *Bm = sm + L::oB, *Cm = sm + L::oC;
    double *cred = sm + L::oRed, *wred = sm + L::oWred;
    // neighbours' grids (distributed shared memory); nullptr at the domain edges
    double *G0lo = rank > 0 ? cluster.map_shared_rank(G0, rank - 1) : nullptr;
    double *G0hi = rank < CS - 1 ? cluster.map_shared_rank(G0, rank + 1) : nullptr;
    double *G1lo = rank > 0 ? cluster.map_shared_rank(G1, rank - 1) : nullptr;
    double *G1hi = rank < CS - 1 ? cluster.map_shared_rank(G1, rank + 1) : nullptr;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lx = tid % LX, rg = tid / LX;
    const int col0 = lx * BC, row0 = rg * BR;            // block: columns 2lx+1 (odd), 2lx+2 (even)
    const double inv_n3 = 1.0 / ((double)n * n * n);
    const double *Sy0 = S + (Q.psi ? Q.d * W : 0);

    // replicated level l arrays (natural rows): WH, WV, DI, R, Z, T (= S)
    auto lv = [&](int l, int k) -> double * { return sm + L::oLev(l) + k * L::Nl(l); };
    enum { LWH = 0, LWV = 1, LDI = 2, LR = 3, LZ = 4, LT = 5 };

    // ---- addressing -------------------------------------------------------------------------
    // fine node (col0 + 1 + c, row0 + 1 + q) local; c even = odd column, c odd = even column
    auto fe = [&](int c, int q) -> int {
        const int slot = (c & 1) == 0 ? HE + lx + (c >> 1) : lx + ((c + 1) >> 1);
        return (row0 + 1 + q) * np + slot;
    };
    auto valid = [&](int q, int c) { return col0 + c + 1 <= nx && j0 + row0 + q + 1 <= nx; };
    auto col1s = [](int i) -> int { return (i & 1) ? H1 + (i >> 1) : (i >> 1); };
    auto e1 = [&](int I, int jl) -> int { return jl * P1 + col1s(I); };   // level-1 local row jl

    for (int64_t bl = cluster_id_x(); bl < nb; bl += cluster_count_x()) {
        const int64_t b = b0 + bl;
        // ---- K3: coefficients of the strip's triangles ----------------------------------------
        for (int j = tid; j < Q.d; j += NT) {
            const double y = nodes ? nodes[(int64_t)j * nb + bl] : lattice_node(P, b, j);
            th_amp[j] = Q.amp[j] * theta_of(Q.theta, y, Q.delta);
        }
        __syncthreads();
        {   // aT[plane][cj - j0][ci] for cell rows j0 .. j0+ATR-1 (< n): thread = (column, row set)
            constexpr int CPT = NT / n, KJ = (ATR + CPT - 1) / CPT;
            const int ci = tid % n, r0 = tid / n;
            double slo[KJ], sup[KJ];
#pragma unroll
            for (int k = 0; k < KJ; ++k) slo[k] = sup[k] = 0.0;
#pragma unroll 2
            for (int j = 0; j < Q.d; ++j) {
                const double *Sj = S + j * W, *Sy = Sy0 + j * W;
                const double am = th_amp[j];
                const double tlo = am * __ldg(Sj + 3 * ci + 2), tup = am * __ldg(Sj + 3 * ci + 1);
#pragma unroll
                for (int k = 0; k < KJ; ++k) {
                    const int cj = min(j0 + r0 + CPT * k, n - 1);
                    slo[k] = fma(tlo, __ldg(Sy + 3 * cj + 1), slo[k]);
                    sup[k] = fma(tup, __ldg(Sy + 3 * cj + 2), sup[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < KJ; ++k) {
                const int rl = r0 + CPT * k;
                if (rl < ATR && j0 + rl < n) {
                    aT[rl * n + ci] = Q.form == 0 ? 1.0 + slo[k] : exp(slo[k]);              // lower
                    aT[(ATR + rl) * n + ci] = Q.form == 0 ? 1.0 + sup[k] : exp(sup[k]);      // upper
                }
            }
        }
        cluster_barrier();                               // every strip's table is complete
        // a of T_lo / T_up of cell (ci, cj) of the level with cells of width 2^sh h: the fine
        // triangle with the same centroid (pcg_mg.cuh), read from the CTA whose strip holds it
        auto fcoef = [&](int ci, int cj, int up, int sh) -> double {
            const int p = 1 << sh, ra = up ? p : 2 * p, rb = up ? 2 * p : p;
            const int fi = ci * p + ra / 3, fj = cj * p + rb / 3, pl = (ra % 3 == 1) ? 1 : 0;
            const int own = min(fj / HR, CS - 1);
            const double *src = own == rank ? aT : cluster.map_shared_rank(aT, own);
            return src[(pl * ATR + fj - own * HR) * n + fi];
        };
        auto fcoef_loc = [&](int ci, int cj, int up, int sh) -> double {   // cell rows j0 .. j0+HR+1
            const int p = 1 << sh, ra = up ? p : 2 * p, rb = up ? 2 * p : p;
            const int fi = ci * p + ra / 3, fj = cj * p + rb / 3, pl = (ra % 3 == 1) ? 1 : 0;
            return aT[(pl * ATR + fj - j0) * n + fi];
        };
        auto whg = [&](int i, int j, int M, int sh) -> double {
            return (i < M && j >= 1 && j < M) ? 0.5 * (fcoef(i, j, 0, sh) + fcoef(i, j - 1, 1, sh)) : 0.0;
        };
        auto wvg = [&](int i, int j, int M, int sh) -> double {
            return (j < M && i >= 1 && i < M) ? 0.5 * (fcoef(i, j, 1, sh) + fcoef(i - 1, j, 0, sh)) : 0.0;
        };
        // fine couplings of the own block (ring edges included)
        double cE[BR][BC + 1], cN[BR + 1][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c <= BC; ++c) {
                const int i = col0 + c, j = j0 + row0 + q + 1;
                cE[q][c] = (i <= nx && j <= nx) ? 0.5 * (aT[(j - j0) * n + i] + aT[(ATR + j - 1 - j0) * n + i]) : 0.0;
            }
#pragma unroll
        for (int q = 0; q <= BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = j0 + row0 + q;
                cN[q][c] = (i <= nx && j <= nx) ? 0.5 * (aT[(ATR + j - j0) * n + i] + aT[(j - j0) * n + i - 1]) : 0.0;
            }
        // level-1 couplings of the local rows 0 .. HR1 (J = J0 + jl)
        for (int e = tid; e < (HR1 + 1) * P1; e += NT) {
            const int jl = e / P1, s = e % P1, I = s < H1 ? 2 * s : 2 * (s - H1) + 1, J = J0 + jl;
            WH1[e] = (I < m1 && J >= 1 && J < m1 && jl >= 1)
                         ? 0.5 * (fcoef_loc(I, J, 0, 1) + fcoef_loc(I, J - 1, 1, 1)) : 0.0;
            WV1[e] = (J < m1 && I >= 1 && I < m1) ? 0.5 * (fcoef_loc(I, J, 1, 1) + fcoef_loc(I - 1, J, 0, 1)) : 0.0;
        }
        // replicated levels 2 .. LK-1, K level LK (8 cells), exact level (4 cells)
#pragma unroll
        for (int l = 2; l < LK; ++l) {
            const int M = L::ml(l), Pq = L::Pl(l);
            double *wh = lv(l, LWH), *wv = lv(l, LWV);
            for (int e = tid; e < L::Nl(l); e += NT) {
                const int I = e % Pq, J = e / Pq;
                wh[e] = whg(I, J, M, l);
                wv[e] = wvg(I, J, M, l);
            }
        }
        for (int e = tid; e < NK; e += NT) {
            const int I = e % PK, J = e / PK;
            WHK[e] = whg(I, J, mK, LK);
            WVK[e] = wvg(I, J, mK, LK);
        }
        for (int e = tid; e < L::NE; e += NT) {
            const int I = e % PE, J = e / PE;
            WHE[e] = whg(I, J, mE, LK + 1);
            WVE[e] = wvg(I, J, mE, LK + 1);
        }
        cluster_barrier();                               // nobody reads a coefficient table any more
        // ---- diagonals, zeroed grids, the dense maps -------------------------------------------
        for (int e = tid; e < 2 * L::FR; e += NT) G0[e] = 0.0;          // G0, G1 (rings, halos)
        for (int e = tid; e < L::FR; e += NT) DI0[e] = 0.0;
        for (int e = tid; e < 3 * L::F1; e += NT) R1[e] = 0.0;          // R1, Z1, T1
        for (int e = tid; e < L::R1ROWS * P1; e += NT) {                // level-1 omega D^-1 (own rows)
            const int jl = e / P1, s = e % P1, I = s < H1 ? 2 * s : 2 * (s - H1) + 1, J = J0 + jl;
            const bool in = I >= 1 && I < m1 && J >= 1 && J < m1 && jl >= 1 && jl <= HR1;
            const double dv = in ? WH1[e] + WH1[e1(I - 1, jl)] + WV1[e] + WV1[e - P1] : 1.0;
            DI1[e] = in ? kMgOmega * (1.0 / dv) : 0.0;
            if (jl > HR1) WH1[e] = WV1[e] = 0.0;                        // (unused halo row)
        }
#pragma unroll
        for (int l = 2; l < LK; ++l) {
            const int M = L::ml(l), Pq = L::Pl(l);
            const double *wh = lv(l, LWH), *wv = lv(l, LWV);
            double *di = lv(l, LDI);
            for (int e = tid; e < L::Nl(l); e += NT) {
                const int I = e % Pq, J = e / Pq;
                const bool in = I >= 1 && I < M && J >= 1 && J < M;
                di[e] = in ? kMgOmega * (1.0 / (wh[e] + wh[e - 1] + wv[e] + wv[e - Pq])) : 0.0;
                lv(l, LR)[e] = lv(l, LZ)[e] = lv(l, LT)[e] = 0.0;
            }
        }
        for (int e = tid; e < NK; e += NT) {
            const int I = e % PK, J = e / PK;
            const bool in = I >= 1 && I < mK && J >= 1 && J < mK;
            const double dv = in ? WHK[e] + WHK[e - 1] + WVK[e] + WVK[e - PK] : 0.0;
            DK[e] = dv;
            DIK[e] = in ? kMgOmega * (1.0 / dv) : 0.0;
            SK[e] = 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < BR; ++q)                     // omega D^-1 of the own fine nodes
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const double dv = cE[q][c + 1] + cE[q][c] + cN[q + 1][c] + cN[q][c];
                if (valid(q, c)) DI0[fe(c, q)] = kMgOmega * rcp_pos(dv);
            }
        if (warp == 0) {   // Gauss-Jordan inverse of the 4-cell operator (9 unknowns), by shuffles
            const int ri = lane < UE ? lane : 0;
            const int ia = ri % (mE - 1) + 1, ja = ri / (mE - 1) + 1, g = ja * PE + ia;
            const double wr = WHE[g], wl = WHE[g - 1], wu = WVE[g], wd = WVE[g - PE];
            double a[UE];
#pragma unroll
            for (int c = 0; c < UE; ++c)
                a[c] = c == ri ? wr + wl + wu + wd
                     : (c == ri + 1 && ia < mE - 1) ? -wr
                     : (c == ri - 1 && ia > 1) ? -wl
                     : (c == ri + (mE - 1) && ja < mE - 1) ? -wu
                     : (c == ri - (mE - 1) && ja > 1) ? -wd : 0.0;
#pragma unroll
            for (int k = 0; k < UE; ++k) {
                double prow[UE];
#pragma unroll
                for (int c = 0; c < UE; ++c) prow[c] = __shfl_sync(0xffffffffu, a[c], k);
                const double piv = rcp_pos(prow[k]);
                const double f = -a[k] * piv;
#pragma unroll
                for (int c = 0; c < UE; ++c) {
                    if (lane == k) a[c] = c == k ? piv : prow[c] * piv;
                    else a[c] = c == k ? f : fma(f, prow[c], a[c]);
                }
            }
            __syncwarp();
            if (lane < UE) {
#pragma unroll
                for (int c = 0; c < UE; ++c) AI[lane * UE + c] = a[c];
            }
        }
        __syncthreads();
        // K = 2 Dw - Dw AK Dw + B^T AE^-1 B,  B = PE^T (I - AK Dw)  (pcg_mg.cuh)
        for (int e = tid; e < UE * UK; e += NT) {
            const int r = e / UK, k = e % UK;
            const int Ir = r % (mE - 1) + 1, Jr = r / (mE - 1) + 1;
            const int Ik = k % (mK - 1) + 1, Jk = k / (mK - 1) + 1, ek = Jk * PK + Ik;
            const double dwk = DIK[ek];
            auto wr = [&](int Im, int Jm) -> double {
                const int ax = abs(Im - 2 * Ir), ay = abs(Jm - 2 * Jr);
                return (ax > 1 || ay > 1) ? 0.0 : (ax ? 0.5 : 1.0) * (ay ? 0.5 : 1.0);
            };
            double v = wr(Ik, Jk) * (1.0 - DK[ek] * dwk);
            v = fma(wr(Ik + 1, Jk), WHK[ek] * dwk, v);
            v = fma(wr(Ik - 1, Jk), WHK[ek - 1] * dwk, v);
            v = fma(wr(Ik, Jk + 1), WVK[ek] * dwk, v);
            v = fma(wr(Ik, Jk - 1), WVK[ek - PK] * dwk, v);
            Bm[e] = v;
        }
        __syncthreads();
        for (int e = tid; e < UE * UK; e += NT) {        // C = AE^-1 B
            const int r = e / UK, k = e % UK;
            double v = 0.0;
            for (int c = 0; c < UE; ++c) v = fma(AI[r * UE + c], Bm[c * UK + k], v);
            Cm[e] = v;
        }
        __syncthreads();
        auto kix = [](int col, int row) -> int { return col * UK + row + (col >= HK ? L::KPAD : 0); };
        for (int e = UK * UK + tid; e < 2 * HK * UK; e += NT) Kt[kix(e / UK, e % UK)] = 0.0;
        if (tid < 2 * HK - UK) RK[UK + tid] = 0.0;
        for (int e = tid; e < UK * UK; e += NT) {        // B^T C
            const int i = e % UK, k = e / UK;
            double v = 0.0;
            for (int r = 0; r < UE; ++r) v = fma(Bm[r * UK + i], Cm[r * UK + k], v);
            Kt[kix(k, i)] = v;
        }
        __syncthreads();
        for (int e = tid; e < 5 * UK; e += NT) {         // + 2 Dw - Dw AK Dw (5-point), row i
            const int i = e % UK, d = e / UK;
            const int Ii = i % (mK - 1) + 1, Ji = i / (mK - 1) + 1, ei = Ji * PK + Ii;
            const double dwi = DIK[ei];
            if (d == 0) Kt[kix(i, i)] += fma(-dwi * DK[ei], dwi, 2.0 * dwi);
            else if (d == 1 && Ii < mK - 1) Kt[kix(i + 1, i)] += dwi * WHK[ei] * DIK[ei + 1];
            else if (d == 2 && Ii > 1) Kt[kix(i - 1, i)] += dwi * WHK[ei - 1] * DIK[ei - 1];
            else if (d == 3 && Ji < mK - 1) Kt[kix(i + (mK - 1), i)] += dwi * WVK[ei] * DIK[ei + PK];
            else if (d == 4 && Ji > 1) Kt[kix(i - (mK - 1), i)] += dwi * WVK[ei - PK] * DIK[ei - PK];
        }
        cluster_barrier();   // setup complete in every CTA before any neighbour writes a halo

        // ---- helpers of the iteration -----------------------------------------------------------
        // publish own values into Gd and the strip's edge rows into the neighbours' halo rows
        auto publish = [&](double *Gd, double *Glo, double *Ghi, const double (&v)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) Gd[fe(c, q)] = v[q][c];
            if (rg == 0 && Glo) {
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(0, c)) Glo[fe(c, 0) + HR * np] = v[0][c];
            }
            if (rg == NRG - 1 && Ghi) {
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(BR - 1, c)) Ghi[fe(c, BR - 1) - HR * np] = v[BR - 1][c];
            }
        };
        auto diag = [&](int q, int c) -> double { return cE[q][c + 1] + cE[q][c] + cN[q + 1][c] + cN[q][c]; };
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
        // level-1 operator at own (I, jl) (diagonal summed in the order of DI1)
        auto apply1 = [&](const double *Zs, int I, int jl) -> double {
            const int e = e1(I, jl), el = e1(I - 1, jl), er = e1(I + 1, jl);
            const double whe = WH1[e], whl = WH1[el], wve = WV1[e], wvd = WV1[e - P1];
            return (whe + whl + wve + wvd) * Zs[e] - whe * Zs[er] - whl * Zs[el] - wve * Zs[e + P1] -
                   wvd * Zs[e - P1];
        };
        // the same on a replicated natural-row level
        auto applyl = [](const double *wh, const double *wv, const double *z, int e, int Pq) -> double {
            const double we = wh[e], ww = wh[e - 1], wn = wv[e], ws = wv[e - Pq];
            return (we + ww + wn + ws) * z[e] - we * z[e + 1] - ww * z[e - 1] - wn * z[e + Pq] - ws * z[e - Pq];
        };
        auto prol2w = [](const double *Xc, int pc, int i, int j) -> double {   // bilinear, branch-free
            const double *z2 = Xc + (j >> 1) * pc + (i >> 1);
            const double wx1 = (i & 1) ? 0.5 : 0.0, wx0 = (i & 1) ? 0.5 : 1.0;
            const double wy1 = (j & 1) ? 0.5 : 0.0, wy0 = (j & 1) ? 0.5 : 1.0;
            return fma(wx1 * wy1, z2[pc + 1], fma(wx0 * wy1, z2[pc], fma(wx1 * wy0, z2[1], wx0 * wy0 * z2[0])));
        };
        // own level-1 interior nodes: q -> (I, jl), lanes walk whole rows of m1 slots
        auto for1 = [&](auto body) {
            constexpr int U = m1 * HR1;
#pragma unroll
            for (int k = 0; k < (U + NT - 1) / NT; ++k) {
                const int q = tid + k * NT, I = q % m1 + 1, jl = q / m1 + 1;
                if (q < U && I < m1 && J0 + jl < m1) body(I, jl);
            }
        };
        // interior of a replicated level with M cells
        auto forl = [&](int M, auto body) {
            const int U = (M - 1) * (M - 1);
            for (int q = tid; q < U; q += NT) {
                const int I = q % (M - 1) + 1, J = q / (M - 1) + 1;
                body(I, J, J * (M + 1) + I);
            }
        };
        double *T1lo = rank > 0 ? cluster.map_shared_rank(T1, rank - 1) : nullptr;
        double *T1hi = rank < CS - 1 ? cluster.map_shared_rank(T1, rank + 1) : nullptr;
        double *Z1lo = rank > 0 ? cluster.map_shared_rank(Z1, rank - 1) : nullptr;
        double *Z1hi = rank < CS - 1 ? cluster.map_shared_rank(Z1, rank + 1) : nullptr;
        double *R2 = lv(2, LR);

        // ---- one V(1,1) cycle: z = M^-1 rin -------------------------------------------------------
        auto vcycle = [&](const double (&rin)[BR][BC], double (&z)[BR][BC]) {
            double t[BR][BC];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) z[q][c] = DI0[fe(c, q)] * rin[q][c];   // z0 = omega D^-1 r
            publish(G0, G0lo, G0hi, z);
            cluster_barrier();
            apply_fine(G0, z, t);
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) t[q][c] = rin[q][c] - t[q][c];       // fine residual
            publish(G1, G1lo, G1hi, t);
            cluster_barrier();
            for1([&](int I, int jl) {                    // R1 = P^T t, Z1 = omega D1^-1 R1
                const int f = 2 * jl * np, c = I, l = HE + I - 1, r = HE + I;
                const double rr = G1[f + c] + 0.5 * (G1[f + l] + G1[f + r] + G1[f - np + c] + G1[f + np + c]) +
                                  0.25 * (G1[f - np + l] + G1[f - np + r] + G1[f + np + l] + G1[f + np + r]);
                const int e = e1(I, jl);
                const double zv = DI1[e] * rr;
                R1[e] = rr;
                Z1[e] = zv;
                if (jl == 1 && Z1lo) Z1lo[e1(I, HR1 + 1)] = zv;
                if (jl == HR1 && Z1hi) Z1hi[e1(I, 0)] = zv;
            });
            cluster_barrier();
            for1([&](int I, int jl) {                    // level-1 residual
                const double tv = R1[e1(I, jl)] - apply1(Z1, I, jl);
                T1[e1(I, jl)] = tv;
                if (jl == 1 && T1lo) T1lo[e1(I, HR1 + 1)] = tv;
            });
            cluster_barrier();
            {   // R2 = P^T T1 on the own level-2 rows, into every CTA's replicated grid
                constexpr int m2 = L::ml(2), P2 = L::Pl(2), U = (m2 - 1) * HR2;
                for (int q = tid; q < U; q += NT) {
                    const int I = q % (m2 - 1) + 1, jl2 = q / (m2 - 1) + 1, J = J20 + jl2;
                    if (J >= m2) continue;
                    const int f = 2 * jl2 * P1, c = I, l = H1 + I - 1, r = H1 + I;
                    const double v = T1[f + c] + 0.5 * (T1[f + l] + T1[f + r] + T1[f - P1 + c] + T1[f + P1 + c]) +
                                     0.25 * (T1[f - P1 + l] + T1[f - P1 + r] + T1[f + P1 + l] + T1[f + P1 + r]);
#pragma unroll
                    for (int k = 0; k < CS; ++k) cluster.map_shared_rank(R2, k)[J * P2 + I] = v;
                }
            }
            cluster_barrier();
            // ---- replicated levels 2 .. LK-1, then the K map (CTA-local) ----------------------
#pragma unroll
            for (int l = 2; l < LK; ++l) {               // down: Z = Dw R, T = R - A Z, restrict
                const int M = L::ml(l), Pq = L::Pl(l);
                const double *wh = lv(l, LWH), *wv = lv(l, LWV), *di = lv(l, LDI), *rl = lv(l, LR);
                double *zl = lv(l, LZ), *tl = lv(l, LT);
                forl(M, [&](int, int, int e) {           // the pre-smoothing from zero in the same pass
                    const double zc = di[e] * rl[e];
                    const double az = (wh[e] + wh[e - 1] + wv[e] + wv[e - Pq]) * zc -
                                      wh[e] * (di[e + 1] * rl[e + 1]) - wh[e - 1] * (di[e - 1] * rl[e - 1]) -
                                      wv[e] * (di[e + Pq] * rl[e + Pq]) - wv[e - Pq] * (di[e - Pq] * rl[e - Pq]);
                    zl[e] = zc;
                    tl[e] = rl[e] - az;
                });
                __syncthreads();
                const int Mc = M >> 1;
                forl(Mc, [&](int I, int J, int ec) {
                    const int f = 2 * J * Pq + 2 * I;
                    const double v = tl[f] + 0.5 * (tl[f - 1] + tl[f + 1] + tl[f - Pq] + tl[f + Pq]) +
                                     0.25 * (tl[f - Pq - 1] + tl[f - Pq + 1] + tl[f + Pq - 1] + tl[f + Pq + 1]);
                    if (l + 1 < LK) lv(l + 1, LR)[ec] = v;
                    else RK[(J - 1) * (mK - 1) + I - 1] = v;
                });
                __syncthreads();
            }
            if (warp < (2 * UK + 31) / 32) {             // SK = K RK (levels 8 and 4 cells)
                const int h = tid & 1, i = min(tid >> 1, UK - 1);
                const bool own = tid < 2 * UK;
                const double *kp = Kt + h * (HK * UK + L::KPAD) + i, *rp = RK + h * HK;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                for (int c = 0; c < HK; c += 4) {
                    a0 = fma(kp[c * UK], rp[c], a0);
                    if (c + 1 < HK) a1 = fma(kp[(c + 1) * UK], rp[c + 1], a1);
                    if (c + 2 < HK) a2 = fma(kp[(c + 2) * UK], rp[c + 2], a2);
                    if (c + 3 < HK) a3 = fma(kp[(c + 3) * UK], rp[c + 3], a3);
                }
                double sv = (a0 + a1) + (a2 + a3);
                sv += __shfl_xor_sync(0xffffffffu, sv, 1);
                if (own && h == 0) SK[(i / (mK - 1) + 1) * PK + i % (mK - 1) + 1] = sv;
            }
            __syncthreads();
#pragma unroll
            for (int l = LK - 1; l >= 2; --l) {          // up: Z += P S_coarse, S = smooth(Z)
                const int M = L::ml(l), Pq = L::Pl(l);
                const double *xc = l + 1 < LK ? lv(l + 1, LT) : SK;
                const int pc = l + 1 < LK ? L::Pl(l + 1) : PK;
                const double *wh = lv(l, LWH), *wv = lv(l, LWV), *di = lv(l, LDI), *rl = lv(l, LR);
                double *zl = lv(l, LZ), *sl = lv(l, LT);
                forl(M, [&](int I, int J, int e) { zl[e] += prol2w(xc, pc, I, J); });
                __syncthreads();
                forl(M, [&](int, int, int e) { sl[e] = fma(di[e], rl[e] - applyl(wh, wv, zl, e, Pq), zl[e]); });
                __syncthreads();
            }
            {   // level 1: Z1 += P S2 on the own and halo rows, then S1 = smooth(Z1) on the own rows
                const double *S2 = lv(2, LT);
                constexpr int P2 = L::Pl(2), U = (m1 - 1) * (HR1 + 2);
                for (int q = tid; q < U; q += NT) {
                    const int I = q % (m1 - 1) + 1, jl = q / (m1 - 1), J = J0 + jl;
                    if (J >= 1 && J < m1) Z1[e1(I, jl)] += prol2w(S2, P2, I, J);
                }
                __syncthreads();
                for1([&](int I, int jl) {
                    const int e = e1(I, jl);
                    const double sv = fma(DI1[e], R1[e] - apply1(Z1, I, jl), Z1[e]);
                    S1[e] = sv;
                    if (jl == 1 && T1lo) T1lo[e1(I, HR1 + 1)] = sv;
                    if (jl == HR1 && T1hi) T1hi[e1(I, 0)] = sv;
                });
                cluster_barrier();
            }
            // level 0: z = z0 + P S1, post-smoothed (window of S1 as in pcg_mg.cuh)
            constexpr int XW = BC / 2 + 2, YW = BR / 2 + 2;
            double cw[YW][XW];
#pragma unroll
            for (int yy = 0; yy < YW; ++yy)
#pragma unroll
                for (int xx = 0; xx < XW; ++xx) {
                    const int X = lx + xx, Y = (row0 >> 1) + yy;
                    cw[yy][xx] = (X <= m1 && J0 + Y <= m1) ? S1[Y * P1 + col1s(X)] : 0.0;
                }
            auto pw = [&](int c, int q) -> double {
                const int fi = 1 + c, fj = 1 + q, x0 = fi >> 1, y0 = fj >> 1;
                if (!(fi & 1) && !(fj & 1)) return cw[y0][x0];
                if (!(fj & 1)) return 0.5 * (cw[y0][x0] + cw[y0][x0 + 1]);
                if (!(fi & 1)) return 0.5 * (cw[y0][x0] + cw[y0 + 1][x0]);
                return 0.25 * (cw[y0][x0] + cw[y0][x0 + 1] + cw[y0 + 1][x0] + cw[y0 + 1][x0 + 1]);
            };
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

        // ---- Chronopoulos-Gear PCG ----------------------------------------------------------------
        double xr[BR][BC], pr[BR][BC], r[BR][BC], s[BR][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                xr[q][c] = pr[q][c] = s[q][c] = 0.0;
                const int j = j0 + row0 + q + 1;
                r[q][c] = !valid(q, c) ? 0.0 : Bt ? __ldg(Bt + (j - 1) * nx + col0 + c) : (double)j * inv_n3;
            }
        double rho = 0.0, bb = 0.0, g_inv = 0.0, ga_inv = 0.0;
        bool conv = false;
        int it = 0;
        for (int k = 0;; ++k) {
            double uu[BR][BC], w[BR][BC];
            vcycle(r, uu);
            publish(G1, G1lo, G1hi, uu);
            cluster_barrier();
            apply_fine(G1, uu, w);
            double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    acc[0] = fma(r[q][c], uu[q][c], acc[0]);
                    acc[1] = fma(w[q][c], uu[q][c], acc[1]);
                    acc[2] = fma(r[q][c], r[q][c], acc[2]);
                }
#pragma unroll
            for (int v = 0; v < 3; ++v) {                // fixed-tree warp sums
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
            }
            if (lane == 0) {
                wred[0 * NWARP + warp] = acc[0];
                wred[1 * NWARP + warp] = acc[1];
                wred[2 * NWARP + warp] = acc[2];
            }
            __syncthreads();
            if (warp == 0 && lane < 3 * CS) {            // CTA sums (warp order) into every CTA's slots
                const int v = lane % 3, dst = lane / 3;
                double sv = 0.0;
#pragma unroll
                for (int ww = 0; ww < NWARP; ++ww) sv += wred[v * NWARP + ww];
                cluster.map_shared_rank(cred, dst)[rank * 4 + v] = sv;
            }
            cluster_barrier();
            double gs[3];
#pragma unroll
            for (int v = 0; v < 3; ++v) {
                double sv = 0.0;
#pragma unroll
                for (int rr2 = 0; rr2 < CS; ++rr2) sv += cred[rr2 * 4 + v];
                gs[v] = sv;
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
                    const double pn = fma(beta, pr[q][c], uu[q][c]);
                    pr[q][c] = pn;
                    s[q][c] = fma(beta, s[q][c], w[q][c]);
                    xr[q][c] = fma(alpha, pn, xr[q][c]);
                    r[q][c] = fma(-alpha, s[q][c], r[q][c]);
                }
            ++it;
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c)
                if (valid(q, c)) u[(int64_t)((j0 + row0 + q) * nx + col0 + c) * ldu + bl] = xr[q][c];
        if (tid == 0 && rank == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rho / bb);
            if (noconv && !conv) atomicAdd(noconv, 1);
        }
        // the next sample's coefficient table overwrites DI0 .. G1, which only this CTA reads now
        __syncthreads();
    }
}

}  // namespace usfft
