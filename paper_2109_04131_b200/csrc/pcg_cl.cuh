// pcg_cl.cuh — multigrid-preconditioned CG for the large meshes (n = 64, 128: configs 3-5), one
// thread-block CLUSTER per sample, the whole solve on chip.
//
// Same discretisation (Z11/Z12), the same Chronopoulos-Gear CG (one reduction per iteration,
// x0 = 0, stop on ||r||_2 <= tol ||b||_2, Z13) and the same preconditioner family as
// pcg_mg.cuh: one symmetric V(1,1) cycle, damped Jacobi smoothing (omega = 0.8 on the fine level, 1 on the coarse levels), bilinear P,
// R = P^T, coarse operators rediscretised from the fine per-triangle coefficients, and the
// bottom two levels (8 and 4 cells per side) as the fixed dense map K of pcg_mg.cuh.
//
// Precision (Z32): the CG (x, r, p, s, the operator A in w = A u, the dot products, alpha,
// beta) is fp64; the preconditioner M^-1 r is evaluated in fp32 (its input r rounded to fp32,
// every level's operator, smoother, transfer and the map K in fp32, its output u exact in
// fp64).  Any fixed SPD map is an admissible preconditioner; the fp32 one changes the CG
// iteration counts of configs 2-5 by zero (tools/mg_precision_study.py) and the converged
// samples by <= 2e-14 relative.  It halves the shared-memory footprint and wavefronts of the
// cycle and runs it on the fp32 pipe.
//
// A sample of n = 128 (16129 unknowns) needs ~0.5 MB of fp64 CG state, more than one SM holds, so
// a cluster of CS CTAs (CS = 8 at n = 128, 4 at n = 64) shares it; CTA r owns the fine rows
// j0+1 .. j0+HR, j0 = r HR, HR = n / CS = 16:
//  * level 0 (fine): each thread keeps a 2 x 2 block of nodes: r and the couplings (fp64, with
//    fp32 copies and omega D^-1) in registers, x, p, s in shared memory; stencil values are
//    published in shared memory (fp32, split rows: even columns, then odd) with halo rows
//    filled by the neighbour CTAs;
//  * level 1 (n/2 cells): distributed the same way;
//  * levels 2 .. (8 cells per side): replicated.  The restricted level-2 residual is gathered into
//    every CTA (each CTA sends its rows to all) and every CTA runs the rest of the cycle locally;
//  * reductions: CTA partials are sent to every CTA and summed in rank order, so all CTAs hold
//    bit-identical scalars and take the same branch.
// Data moves between CTAs only as point-to-point DSMEM stores with transaction counts
// (st.async ... mbarrier::complete_tx): the receiver waits on its own mbarrier for the expected
// bytes, the sender never waits, and no cluster-wide barrier or release fence sits in the CG
// loop.  Five exchanges per CG iteration:
//   X1 z0 = omega D^-1 r (1 row below, 2 above) and r (1 row above): the fine residual t of the
//      own rows and of the row above is then local;
//   X2 level-1 Z1 (2 rows each side) and R1 (1 row each side): the level-1 residual of the own
//      rows + the row above and the smoothed S1 of the own rows + one row each side are local;
//   X3 the level-2 residual rows of every CTA to every CTA;
//   X4 the preconditioned residual u (1 row each side) for w = A u;
//   X5 the CTA partials of (r,u), (w,u), (r,r) to every CTA.
// A transfer of exchange k for CG iteration i+1 cannot start before every CTA has sent its X5
// partials of iteration i, which every CTA does only after its last read of iteration i's data:
// the X5 all-to-all orders all buffer reuse (its own slots are double-buffered).  The per-sample
// setup (coefficient tables, coarse operators, K) uses two cluster barriers (A: the previous sample
// is done everywhere, C: every CTA's grids are zeroed), each split into an early arrive and a late
// wait, and one more counted exchange (XB: the coarse coefficients).  Reductions and
// the order of every sum are fixed, so a sample's result does not depend on the cluster that
// solved it or on the launch split.
//
// The up-sweep of every coarse level is two passes: Zp = Z + P S_coarse once per node, then
// S = Zp + omega D^-1 (R - A Zp) (the prolongation is not recomputed for every stencil
// neighbour).  16 warps per CTA (a 2 x 2 node block per thread), one CTA per SM.
#pragma once
#include <cooperative_groups.h>

// Per-mesh register choice (measured on the B200, tools/cl_variants.py): at n = 64 (two CTAs per SM)
// t and z0 are re-read from the grids they were published to at the post-smoothing instead of
// held in registers across the coarse levels (39.0 -> 37.6 ms at config 3; at n = 128 this costs
// 2 %).  The CG direction p lives in shared memory next to x and s on both meshes (n = 128:
// 533.5 -> 524.9 ms at config 5).
#ifndef USFFT_CL_TZ
#define USFFT_CL_TZ(nn) ((nn) == 64)
#endif

namespace usfft {

template <int NN, int CS>
struct ClC {
    static constexpr int n = NN, nx = n - 1, np = n + 1, HE = n / 2 + 1;
    static constexpr int HR = NN / CS;                       // fine rows per CTA
    static constexpr bool TZ = USFFT_CL_TZ(NN);
    static constexpr int BC = 2, BR = 2, LX = n / 2, NRG = HR / BR, NT = LX * NRG, NWARP = NT / 32;
    static constexpr int FRW = HR + 3, FR = FRW * np;        // fine grid rows 0 .. HR+2 (local)
    // level-1 split rows: even columns at slots 0 .. m1/2, odd columns from slot H1 = 48 (16 banks
    // after the even run, so an instruction touching both parities is conflict-free in fp32)
    static constexpr int m1 = n / 2, H1E = m1 / 2 + 1, H1 = 48, P1 = H1 + m1 / 2, HR1 = HR / 2, HR2 = HR / 4;
    static_assert(H1 >= H1E && H1 % 32 == 16, "level-1 row layout");
    static constexpr int L1R = HR1 + 4, F1 = L1R * P1;       // level-1 rows jl = -1 .. HR1+2 (lr = jl+1)
    static constexpr int LK = NN == 64 ? 3 : NN == 128 ? 4 : -1;
    static_assert(LK > 0, "cluster multigrid compiled for n = 64, 128");
    static_assert(HR % 8 == 0 && LX % 32 == 0 && HR % BR == 0, "strip geometry");
    __host__ __device__ static constexpr int ml(int l) { return NN >> l; }
    __host__ __device__ static constexpr int Pl(int l) { return (NN >> l) + 1; }
    __host__ __device__ static constexpr int Nl(int l) { return ((NN >> l) + 1) * ((NN >> l) + 1); }
    static constexpr int mK = 8, PK = 9, NK = 81, UK = 49, HK = (UK + 1) / 2;
    static constexpr int mE = 4, PE = 5, NE = 25, UE = 9;
    static constexpr int KS = 56;                            // K row-major, row stride 56 (= 24 mod 32 banks)
    static constexpr int ATR = HR + 6;                       // coefficient-table cell rows j0-2 .. j0+HR+3
    static constexpr int JC = 8;                             // psi factors staged JC terms at a time
    static constexpr int CPT = NT / n, KJ = (((ATR + CPT - 1) / CPT) + 1) & ~1, YP = CPT * KJ;
    // resident psi slice (fp64, after the partials): X[j][2n] (lower, upper abscissae), Y[j][2][YP];
    // term strides XS, YS = 4 mod 16 doubles, so the DMMA fragment loads of the coefficient
    // table (4 consecutive terms x 8 consecutive columns / rows per warp) are conflict-free
    static constexpr int XS = 2 * n + 4, YS = 2 * YP + 4;
    static_assert(YP % 8 == 0 && YP >= ATR && XS % 16 == 4 && YS % 16 == 4 && NWARP % 2 == 0 && n / 8 == NWARP, "coefficient-table tiling");
    __host__ __device__ static constexpr size_t psi_bytes(int d) { return 8 * (size_t)d * (XS + YS); }
    // ---- shared memory, in 4-byte units ----
    // persistent (written by the setup, read by every iteration), fp32
    static constexpr int oWH1 = 0, oWV1 = F1, oDI1 = 2 * F1;
    static constexpr int oWHh = 3 * F1, oWVh0 = oWHh + np, oWVh1 = oWVh0 + np;
    __host__ __device__ static constexpr int oLC(int l) {   // replicated level l: WH, WV, DI
        int o = oWVh1 + np;
        for (int q = 2; q < l; ++q) o += 3 * Nl(q);
        return o;
    }
    static constexpr int oKs = oLC(LK);                      // WHK, WVK, DK, DIK, SK (NK each), RK (2 HK)
    static constexpr int oWHE = oKs + 5 * NK + 2 * HK, oWVE = oWHE + NE;
    static constexpr int oKt = oWVE + NE;                    // K (UK x KS), AI, Bm, Cm; setup: ctab
    static constexpr int oAI = oKt + UK * KS, oB = oAI + UE * UE, oC = oB + UE * UK;
    static constexpr int oU = ((oC + UE * UK) + 3) & ~3;     // 16-byte aligned union
    // union U: runtime grids | setup coefficient table aT (fp64) | setup psi staging (fp64)
    static constexpr int oG0 = oU, oG1 = oG0 + FR, oRh = oG1 + FR;
    static constexpr int oR1 = oRh + np, oZ1 = oR1 + F1, oT1 = oZ1 + F1;
    __host__ __device__ static constexpr int oLR(int l) {   // replicated level l: R, Z, T
        int o = oT1 + F1;
        for (int q = 2; q < l; ++q) o += 3 * Nl(q);
        return o;
    }
    static constexpr int URUN = oLR(LK) - oU;
    static constexpr int UAT = 2 * (2 * ATR * n);            // fp64 aT
    static constexpr int USTG = 2 * (JC * 2 * n + JC * 2 * ATR);
    static constexpr int USZ = URUN > UAT ? (URUN > USTG ? URUN : USTG) : (UAT > USTG ? UAT : USTG);
    static constexpr int oRedF = (oU + USZ + 3) & ~3;        // fp64 [2][CS][4] cluster partials, [4][NWARP]
                                                             // (slot 3: the early (r,r) check, X6)
    // then fp64: the cluster partials [2][CS][4] and CTA partials [4][NWARP], the CG iterate x,
    // s = A p and the direction p, [BR*BC][NT] each (thread-major: touched once per iteration, so
    // outside the registers)
    __host__ __device__ static constexpr size_t bytes() { return 4 * (size_t)oRedF + 8 * (size_t)(8 * CS + 4 * NWARP + 3 * BR * BC * NT); }
    // setup: the coarse-level triangle coefficients (levels 2 .. LK+1, lower then upper plane)
    __host__ __device__ static constexpr int ctoff(int l) {
        int o = 0;
        for (int q = 2; q < l; ++q) o += 2 * ml(q) * ml(q);
        return o;
    }
    static_assert(ctoff(LK + 2) <= UK * KS, "the coarse coefficient table overlays K only (AE^-1, B, C are built while it is read)");
    static_assert(2 * UK <= NT && 3 * CS <= 32, "thread mapping");
};

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// split form: every thread arrives (releasing its writes), works on, and waits later
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
// arrive without release semantics: for threads that have no writes to publish to the cluster
// (a release arrive first waits until the thread's earlier global stores are performed)
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
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
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned v;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(v));
    return v;
}
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(rank));
    return o;
}
// DSMEM stores completing their byte count on the destination CTA's mbarrier
__device__ __forceinline__ void st_async(uint32_t dst, double v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 :: "r"(dst), "l"(__double_as_longlong(v)), "r"(mbar) : "memory");
}
__device__ __forceinline__ void st_async(uint32_t dst, float v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                 :: "r"(dst), "r"(__float_as_uint(v)), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mb) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(bytes) : "memory");
}
// Default semantics (acquire at CTA scope), as in the usual transaction-barrier wait: the st.async
// data lands in this CTA's own shared memory before its bytes complete on the mbarrier.  With
// .acquire.cluster every successful wait was followed by CCTL.IVALL, an invalidation of the whole
// L1 (six per CG iteration), after which the loop's spill reloads missed to L2.
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" :: "r"(mb), "r"(parity) : "memory");
}

// Phase-latency probe (tools/cl_probe.py builds with -DUSFFT_CL_PROBE): clock64() of thread 0 of
// every CTA of cluster 0 at each phase boundary of its first sample (setup) and CG iteration 6.
#ifdef USFFT_CL_PROBE
__device__ long long g_cl_probe[16][32];
#define CL_MARK(on, id)                                                                             \
    do {                                                                                           \
        if ((on) && threadIdx.x == 0) g_cl_probe[rank][id] = clock64();                             \
    } while (0)
#else
#define CL_MARK(on, id) ((void)0)
#endif

// K = B^T C + (2 Dw - Dw AK Dw) of the 8-/4-cell levels from B, C and the 8-cell operator in
// shared memory, all warps of the CTA; the 5-point part is its own short pass (folded into the
// product loop its five branches diverge in every warp: ~1000 instead of ~230 cycles per loop
// iteration).  Not inlined: its registers are allocated apart from the solver's (inlined, its
// pressure moved spills into the CG loop: config 3 37.2 -> 38.5 ms for the same code; as a
// function 36.1 ms).  Measured and rejected: the whole K build (inverse, B, C, diagonals) in this
// function as CTA-wide passes (config 5 496.4 -> 502.1 ms).
template <int NN, int CS>
__device__ __noinline__ void cl_build_k(float *sf) {
    using L = ClC<NN, CS>;
    constexpr int NT = L::NT, mK = L::mK, PK = L::PK, NK = L::NK, UK = L::UK, UE = L::UE;
    const float *WHK = sf + L::oKs, *WVK = WHK + NK, *DK = WHK + 2 * NK, *DIK = WHK + 3 * NK;
    const float *Bm = sf + L::oB, *Cm = sf + L::oC;
    float *Kt = sf + L::oKt;
    const int tid = threadIdx.x;
    auto kix = [](int col, int row) -> int { return row * L::KS + col; };     // K[row][col]
    for (int e = tid; e < UK * UK; e += NT) {
        const int i = e % UK, k = e / UK;
        float v = 0.0f;
#pragma unroll
        for (int r = 0; r < UE; ++r) v = fmaf(Bm[r * UK + i], Cm[r * UK + k], v);
        Kt[kix(k, i)] = v;
    }
    __syncthreads();
    for (int e = tid; e < 5 * UK; e += NT) {             // row i
        const int i = e % UK, d = e / UK;
        const int Ii = i % (mK - 1) + 1, Ji = i / (mK - 1) + 1, ei = Ji * PK + Ii;
        const float dwi = DIK[ei];
        if (d == 0) Kt[kix(i, i)] += fmaf(-dwi * DK[ei], dwi, 2.0f * dwi);
        else if (d == 1 && Ii < mK - 1) Kt[kix(i + 1, i)] += dwi * WHK[ei] * DIK[ei + 1];
        else if (d == 2 && Ii > 1) Kt[kix(i - 1, i)] += dwi * WHK[ei - 1] * DIK[ei - 1];
        else if (d == 3 && Ji < mK - 1) Kt[kix(i + (mK - 1), i)] += dwi * WVK[ei] * DIK[ei + PK];
        else if (d == 4 && Ji > 1) Kt[kix(i - (mK - 1), i)] += dwi * WVK[ei - PK] * DIK[ei - PK];
    }
}

template <int NN, int CS, int MINB>
__global__ void __launch_bounds__(ClC<NN, CS>::NT, MINB)
k_pcg_cl(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
         int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
         double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S,
         const double *__restrict__ Bt, int pd) {
    using L = ClC<NN, CS>;
    constexpr int n = NN, nx = L::nx, np = L::np, HE = L::HE, HR = L::HR, BC = L::BC, BR = L::BR;
    constexpr int LX = L::LX, NRG = L::NRG, NT = L::NT, NWARP = L::NWARP, W = 3 * n + 1;
    constexpr int m1 = L::m1, P1 = L::P1, H1 = L::H1, HR1 = L::HR1, HR2 = L::HR2, LK = L::LK;
    constexpr int mK = L::mK, PK = L::PK, NK = L::NK, UK = L::UK, HK = L::HK;
    constexpr int mE = L::mE, PE = L::PE, UE = L::UE, ATR = L::ATR, JC = L::JC, H1E = L::H1E;
    constexpr int m2 = L::ml(2), P2 = L::Pl(2);
    constexpr bool TZ = L::TZ;
    constexpr float om = (float)kMgOmegaCoarse;          // coarse-level Jacobi weight (the fine level: kMgOmega)
    extern __shared__ __align__(16) float sf[];
    __shared__ double th_amp2[2][kMaxD];                 // amp_j theta_j(y_j) of the current / the next sample
    __shared__ alignas(8) unsigned long long mbar[7];
    const int rank = (int)cluster_rank();
    const bool has_lo = rank > 0, has_hi = rank < CS - 1;
    const int j0 = rank * HR, J0 = j0 / 2, J20 = j0 / 4;

    float *WH1 = sf + L::oWH1, *WV1 = sf + L::oWV1, *DI1 = sf + L::oDI1;
    float *WHh = sf + L::oWHh, *WVh0 = sf + L::oWVh0, *WVh1 = sf + L::oWVh1;
    float *WHK = sf + L::oKs, *WVK = WHK + NK, *DK = WHK + 2 * NK, *DIK = WHK + 3 * NK, *SK = WHK + 4 * NK;
    float *RK = WHK + 5 * NK, *WHE = sf + L::oWHE, *WVE = sf + L::oWVE;
    float *Kt = sf + L::oKt, *ctab = sf + L::oKt, *AI = sf + L::oAI, *Bm = sf + L::oB, *Cm = sf + L::oC;
    float *G0 = sf + L::oG0, *G1 = sf + L::oG1, *Rh = sf + L::oRh;
    float *R1 = sf + L::oR1, *Z1 = sf + L::oZ1, *T1 = sf + L::oT1;
    double *aT = reinterpret_cast<double *>(sf + L::oU);                  // setup only
    double *cred = reinterpret_cast<double *>(sf + L::oRedF), *wred = cred + 8 * CS;
    auto lc = [&](int l, int k) -> float * { return sf + L::oLC(l) + k * L::Nl(l); };   // WH, WV, DI
    auto lr = [&](int l, int k) -> float * { return sf + L::oLR(l) + k * L::Nl(l); };   // R, Z, T
    enum { LWH = 0, LWV = 1, LDI = 2, LR = 0, LZ = 1, LT = 2 };
    float *R2 = lr(2, LR);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lx = tid % LX, rg = tid / LX;
    const int col0 = lx * BC, row0 = rg * BR;            // block: columns 2lx+1 (odd), 2lx+2 (even)
    const double inv_n3 = 1.0 / ((double)n * n * n);
    const double *Sy0 = S + (Q.psi ? Q.d * W : 0);

    // ---- exchanges: mbarriers, expected bytes, peer addresses -----------------------------------
    const uint32_t mb0 = smem_addr(&mbar[0]);
    const uint32_t xb[7] = {(uint32_t)(4 * nx * ((has_hi ? 3 : 0) + (has_lo ? 1 : 0))),
                            (uint32_t)(4 * (m1 - 1) * ((has_hi ? 3 : 0) + (has_lo ? 3 : 0))),
                            (uint32_t)(4 * (m2 - 1) * (m2 - 1)),
                            (uint32_t)(4 * nx * ((has_hi ? 1 : 0) + (has_lo ? 1 : 0))),
                            (uint32_t)(8 * 3 * CS), (uint32_t)(8 * CS),
                            (uint32_t)(4 * L::ctoff(LK + 2))};   // XB: the whole coarse coefficient table
    if (tid == 0) {
        for (int k = 0; k < 7; ++k) mbar_init(mb0 + 8 * k);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < 7; ++k) mbar_expect(mb0 + 8 * k, xb[k]);
    }
    uint32_t ph = 0;                                     // bit k: parity of exchange k's next phase
    auto xwait = [&](int k) {
        mbar_wait(mb0 + 8 * k, (ph >> k) & 1u);
        ph ^= 1u << k;
        if (tid == 0) mbar_expect(mb0 + 8 * k, xb[k]);   // arm the next phase
    };
    const uint32_t lo_rank = has_lo ? rank - 1 : rank, hi_rank = has_hi ? rank + 1 : rank;
    const uint32_t mb_lo = mapa(mb0, lo_rank), mb_hi = mapa(mb0, hi_rank);
    const uint32_t G0_lo = mapa(smem_addr(G0), lo_rank), G0_hi = mapa(smem_addr(G0), hi_rank);
    const uint32_t G1_lo = mapa(smem_addr(G1), lo_rank), G1_hi = mapa(smem_addr(G1), hi_rank);
    const uint32_t Rh_lo = mapa(smem_addr(Rh), lo_rank);
    const uint32_t R1_lo = mapa(smem_addr(R1), lo_rank), R1_hi = mapa(smem_addr(R1), hi_rank);
    const uint32_t Z1_lo = mapa(smem_addr(Z1), lo_rank), Z1_hi = mapa(smem_addr(Z1), hi_rank);
    cluster_barrier();                                   // mbarriers initialised everywhere

    // ---- addressing -------------------------------------------------------------------------
    // fine node (col0 + 1 + c, row0 + 1 + q) local, c in -1 .. BC; c even = odd column
    auto fe = [&](int c, int q) -> int {
        const int slot = (c & 1) == 0 ? HE + lx + (c >> 1) : lx + ((c + 1) >> 1);
        UB_CHECK(slot >= 0 && slot < np && row0 + 1 + q >= 0 && row0 + 1 + q < L::FRW);
        return (row0 + 1 + q) * np + slot;
    };
    auto slot0 = [](int i) -> int { return (i & 1) ? HE + (i >> 1) : (i >> 1); };   // fine column i
    auto valid = [&](int q, int c) { return col0 + c + 1 <= nx && j0 + row0 + q + 1 <= nx; };
    auto col1s = [](int i) -> int { return (i & 1) ? H1 + (i >> 1) : (i >> 1); };
    auto e1 = [&](int I, int jl) -> int {                                            // level-1 row jl
        UB_CHECK(I >= 0 && I <= m1 && jl >= -1 && jl + 1 < L::L1R);
        return (jl + 1) * P1 + col1s(I);
    };

    // the psi factors of this CTA's strip do not depend on the sample: with pd = d they are loaded
    // once per CTA (X at the 2n abscissae, Y at the strip's ATR ordinates, both planes)
    constexpr int YP = L::YP, CPT = L::CPT, KJ = L::KJ;
    double *Xg = cred + 8 * CS + 4 * NWARP;                                     // x, [BR*BC][NT]
    double *Sg = Xg + BR * BC * NT;                                             // s, [BR*BC][NT]
    double *Pg = Sg + BR * BC * NT;                                             // p, [BR*BC][NT]
    constexpr int XS = L::XS, YS = L::YS;
    double *XP = Pg + BR * BC * NT, *YPs = XP + (size_t)pd * XS;
    for (int e = tid; e < pd * 2 * n; e += NT) {
        const int j = e / (2 * n), c = e - j * 2 * n, up = c >= n, cc = up ? c - n : c;
        XP[j * XS + c] = __ldg(S + j * W + 3 * cc + (up ? 1 : 2));
    }
    for (int e = tid; e < pd * 2 * YP; e += NT) {
        const int j = e / (2 * YP), c = e - j * 2 * YP, up = c >= YP, rl = up ? c - YP : c;
        const int cj = min(max(j0 - 2 + rl, 0), n - 1);
        YPs[j * YS + c] = rl < ATR ? __ldg(Sy0 + j * W + 3 * cj + (up ? 2 : 1)) : 0.0;
    }
    // amp_j theta_j(y_j) of sample bl of this launch; the first sample's here, every later one
    // during the previous sample's setup (by warps that wait for the K map there)
    auto theta_amp = [&](int64_t bl, int j, double *dst) {
        const double y = nodes ? nodes[(int64_t)j * nb + bl] : lattice_node(P, b0 + bl, j);
        dst[j] = Q.amp[j] * theta_of(Q.theta, y, Q.delta);
    };
    if (tid < Q.d && (int64_t)cluster_id_x() < nb) theta_amp(cluster_id_x(), tid, th_amp2[0]);
    int tbuf = 0;

    for (int64_t bl = cluster_id_x(); bl < nb; bl += cluster_count_x()) {
        const int64_t b = b0 + bl;
        const bool pset = cluster_id_x() == 0 && bl == cluster_count_x();   // probe: the 2nd sample (warm L2)
        (void)pset;
        CL_MARK(pset, 20);
        // ---- K3: coefficients of the triangles of cell rows j0-2 .. j0+HR+3 --------------------
        const double *th_amp = th_amp2[tbuf];
        double *th_next = th_amp2[tbuf ^ 1];
        tbuf ^= 1;
        // A: this CTA is done with the previous sample (its reads of K; nothing to publish: relaxed, so
        // the arrive does not wait for the sample's output stores)
        cluster_arrive_relaxed();
        __syncthreads();
        CL_MARK(pset, 29);
        if (pd) {   // aT[plane] = Y_plane^T . (amp theta X_plane) from the resident slice: two [YP x d] . [d x n]
            // products on the fp64 tensor pipe (DMMA m8n8k4: A a = A[lane/4][lane%4], B b =
            // B[lane%4][lane/4], C {c0, c1} = C[lane/4][2 (lane%4) + {0, 1}]); warp = (plane, two
            // column tiles) x all YP / 8 row tiles, terms four at a time (zero beyond d)
            constexpr int MT = YP / 8, NW2 = NWARP / 2;
            const int pl = warp / NW2, nt0 = 2 * (warp % NW2), fr = lane >> 2, fk = lane & 3;
            double acc[MT][2][2];
#pragma unroll
            for (int m = 0; m < MT; ++m) acc[m][0][0] = acc[m][0][1] = acc[m][1][0] = acc[m][1][1] = 0.0;
            const double *xb = XP + pl * n + nt0 * 8 + fr, *yb = YPs + pl * YP + fr;
#pragma unroll 2
            for (int jk = 0; jk < pd; jk += 4) {
                const int j = jk + fk;
                const bool in = j < pd;
                const double am = in ? th_amp[j] : 0.0;
                const double bq0 = in ? am * xb[j * XS] : 0.0, bq1 = in ? am * xb[j * XS + 8] : 0.0;
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    const double a = in ? yb[j * YS + m * 8] : 0.0;
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc[m][0][0]), "+d"(acc[m][0][1]) : "d"(a), "d"(bq0));
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc[m][1][0]), "+d"(acc[m][1][1]) : "d"(a), "d"(bq1));
                }
            }
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const int rl = m * 8 + fr, cj = j0 - 2 + rl;
                if (rl < ATR && cj >= 0 && cj < n) {
#pragma unroll
                    for (int t2 = 0; t2 < 2; ++t2) {
                        const double v0 = Q.form == 0 ? 1.0 + acc[m][t2][0] : exp(acc[m][t2][0]);
                        const double v1 = Q.form == 0 ? 1.0 + acc[m][t2][1] : exp(acc[m][t2][1]);
                        *reinterpret_cast<double2 *>(aT + (pl * ATR + rl) * n + (nt0 + t2) * 8 + 2 * fk) = make_double2(v0, v1);
                    }
                }
            }
        } else {   // aT[plane][cj - (j0-2)][ci] = sum_j amp_j theta_j X_j Y_j: thread = (column, row set); the
            // factors amp_j theta_j X_j at the 2n abscissae and Y_j at the strip's 2 ATR ordinates are
            // staged JC terms at a time, all loads of a chunk issued before its first store
            constexpr int SX = JC * 2 * n, SY = JC * 2 * ATR;
            constexpr int XPT = (SX + NT - 1) / NT, YPT = (SY + NT - 1) / NT;
            constexpr int KJ = (ATR + CPT - 1) / CPT;
            double *Xs = reinterpret_cast<double *>(sf + L::oU), *Ys = Xs + SX;
            const int ci = tid % n, r0 = tid / n;
            double slo[KJ], sup[KJ];
#pragma unroll
            for (int k = 0; k < KJ; ++k) slo[k] = sup[k] = 0.0;
            for (int jb = 0; jb < Q.d; jb += JC) {
                const int jn = min(JC, Q.d - jb);
                double xv[XPT], yv[YPT];
#pragma unroll
                for (int k = 0; k < XPT; ++k) {
                    const int e = tid + k * NT, j = e / (2 * n), c = e - j * 2 * n, up = c >= n;
                    const int cc = up ? c - n : c;
                    xv[k] = (e < SX && j < jn) ? th_amp[jb + j] * __ldg(S + (jb + j) * W + 3 * cc + (up ? 1 : 2)) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < YPT; ++k) {
                    const int e = tid + k * NT, j = e / (2 * ATR), c = e - j * 2 * ATR, up = c >= ATR;
                    const int rl = up ? c - ATR : c, cj = min(max(j0 - 2 + rl, 0), n - 1);
                    yv[k] = (e < SY && j < jn) ? __ldg(Sy0 + (jb + j) * W + 3 * cj + (up ? 2 : 1)) : 0.0;
                }
                __syncthreads();                         // the previous chunk is consumed
#pragma unroll
                for (int k = 0; k < XPT; ++k)
                    if (tid + k * NT < SX) Xs[tid + k * NT] = xv[k];
#pragma unroll
                for (int k = 0; k < YPT; ++k)
                    if (tid + k * NT < SY) Ys[tid + k * NT] = yv[k];
                __syncthreads();
#pragma unroll 2
                for (int j = 0; j < jn; ++j) {
                    const double tlo = Xs[j * 2 * n + ci], tup = Xs[j * 2 * n + n + ci];
                    const double *yl = Ys + j * 2 * ATR, *yu = yl + ATR;
#pragma unroll
                    for (int k = 0; k < KJ; ++k) {
                        const int rl = min(r0 + CPT * k, ATR - 1);
                        slo[k] = fma(tlo, yl[rl], slo[k]);
                        sup[k] = fma(tup, yu[rl], sup[k]);
                    }
                }
            }
            __syncthreads();                             // staging consumed: aT overlaps it
#pragma unroll
            for (int k = 0; k < KJ; ++k) {
                const int rl = r0 + CPT * k, cj = j0 - 2 + rl;
                if (rl < ATR && cj >= 0 && cj < n) {
                    aT[rl * n + ci] = Q.form == 0 ? 1.0 + slo[k] : exp(slo[k]);              // lower
                    aT[(ATR + rl) * n + ci] = Q.form == 0 ? 1.0 + sup[k] : exp(sup[k]);      // upper
                }
            }
        }
        CL_MARK(pset, 30);
        __syncthreads();                                 // own table complete
        cluster_wait();                                  // A: previous sample done everywhere
        CL_MARK(pset, 21);
        // a of T_lo / T_up of cell (ci, cj) of the level with cells of width 2^sh h: the fine
        // triangle with the same centroid (pcg_mg.cuh), from the local table
        auto fcl = [&](int ci, int cj, int up, int sh) -> double {
            const int p = 1 << sh, ra = up ? p : 2 * p, rb = up ? 2 * p : p;
            const int fi = ci * p + ra / 3, fj = cj * p + rb / 3, pl = (ra % 3 == 1) ? 1 : 0;
            UB_CHECK(fi >= 0 && fi < n && fj - (j0 - 2) >= 0 && fj - (j0 - 2) < ATR);
            return aT[(pl * ATR + fj - (j0 - 2)) * n + fi];
        };
        {   // coarse triangle coefficients (levels 2 .. LK+1) whose fine triangle is in the own rows,
            // sent to every CTA's coarse table (XB: st.async with byte counts on the receivers' mbarrier;
            // every CTA receives the whole table once per sample, its own share included)
            constexpr int NC = L::ctoff(LK + 2) / 2;       // coarse cells of all levels
            const uint32_t ctab_a = smem_addr(ctab);
            for (int e = tid; e < 2 * NC; e += NT) {
                const int up = e >= NC, q = up ? e - NC : e;
                int l = 2, base = 0;
                while (q - base >= L::ml(l) * L::ml(l)) {
                    base += L::ml(l) * L::ml(l);
                    ++l;
                }
                const int m = L::ml(l), cell = q - base, ci = cell % m, cj = cell / m;
                const int p = 1 << l, rb = up ? 2 * p : p, fj = cj * p + rb / 3;
                if (fj / HR != rank) continue;
                const float v = (float)fcl(ci, cj, up, l);
                const int dst = L::ctoff(l) + (up ? m * m : 0) + cell;
                UB_CHECK(dst >= 0 && dst < L::ctoff(LK + 2));
#pragma unroll
                for (int k = 0; k < CS; ++k) st_async(mapa(ctab_a + 4 * dst, k), v, mapa(mb0 + 48, k));
            }
        }
        // fine couplings of the own block (ring edges included), fp64 and their fp32 copies
        double cE[BR][BC + 1], cN[BR + 1][BC];
        float ce[BR][BC + 1], cn[BR + 1][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c <= BC; ++c) {
                const int i = col0 + c, j = j0 + row0 + q + 1;
                cE[q][c] = (i <= nx && j <= nx) ? 0.5 * (fcl(i, j, 0, 0) + fcl(i, j - 1, 1, 0)) : 0.0;
                ce[q][c] = (float)cE[q][c];
            }
#pragma unroll
        for (int q = 0; q <= BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                const int i = col0 + c + 1, j = j0 + row0 + q;
                cN[q][c] = (i <= nx && j <= nx) ? 0.5 * (fcl(i, j, 1, 0) + fcl(i - 1, j, 0, 0)) : 0.0;
                cn[q][c] = (float)cN[q][c];
            }
        float di0[BR][BC], dg32[BR][BC];                 // omega D^-1 and D of the own fine nodes
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                dg32[q][c] = ce[q][c + 1] + ce[q][c] + cn[q + 1][c] + cn[q][c];
                di0[q][c] = valid(q, c) ? (float)(kMgOmega * rcp_pos(cE[q][c + 1] + cE[q][c] + cN[q + 1][c] + cN[q][c])) : 0.0f;
            }
        for (int i = tid; i <= n; i += NT) {             // couplings of the halo row above (HR+1)
            const int jh = j0 + HR + 1;
            WHh[i] = (i <= nx && jh <= nx) ? (float)(0.5 * (fcl(i, jh, 0, 0) + fcl(i, jh - 1, 1, 0))) : 0.0f;
            WVh0[i] = (i >= 1 && i <= nx && jh - 1 <= nx) ? (float)(0.5 * (fcl(i, jh - 1, 1, 0) + fcl(i - 1, jh - 1, 0, 0))) : 0.0f;
            WVh1[i] = (i >= 1 && i <= nx && jh <= nx) ? (float)(0.5 * (fcl(i, jh, 1, 0) + fcl(i - 1, jh, 0, 0))) : 0.0f;
        }
        for (int e = tid; e < L::F1; e += NT) {           // level-1 couplings, rows jl = -1 .. HR1+1
            const int lrw = e / P1, s = e % P1, I = s < H1E ? 2 * s : s >= H1 ? 2 * (s - H1) + 1 : -1;
            const int jl = lrw - 1, J = J0 + jl;
            if (I < 0) continue;                         // gap between the even and odd runs
            WH1[e] = (jl >= 0 && jl <= HR1 + 1 && I < m1 && J >= 1 && J < m1)
                         ? (float)(0.5 * (fcl(I, J, 0, 1) + fcl(I, J - 1, 1, 1))) : 0.0f;
            WV1[e] = (jl <= HR1 + 1 && J >= 0 && J < m1 && I >= 1 && I < m1)
                         ? (float)(0.5 * (fcl(I, J, 1, 1) + fcl(I - 1, J, 0, 1))) : 0.0f;
        }
        xwait(6);                                        // XB: the coarse table complete (every CTA's share)
        CL_MARK(pset, 22);
        __syncthreads();                                 // every thread is done with aT (zeroed below)
        // ---- replicated couplings, diagonals, zeroed grids, the dense maps -----------------------
        // Two warp groups run concurrently.  Warps 0-3 (named barrier 1) form the couplings of the 8-
        // and 4-cell levels from the coarse table and build AE^-1, B and C of the dense map K (none
        // of which overlays the table; K itself does and waits for the join).  The other warps
        // (named barrier 2) form the couplings of the replicated smoothed levels from the table, zero
        // the runtime grids, compute the next sample's amp theta and every diagonal.
        auto ct = [&](int l, int ci, int cj, int up) -> float {
            const int m = L::ml(l);
            return ctab[L::ctoff(l) + (up ? m * m : 0) + cj * m + ci];
        };
        auto whc = [&](int l, int I, int J) -> float {
            const int M = L::ml(l);
            return (I < M && J >= 1 && J < M) ? 0.5f * (ct(l, I, J, 0) + ct(l, I, J - 1, 1)) : 0.0f;
        };
        auto wvc = [&](int l, int I, int J) -> float {
            const int M = L::ml(l);
            return (J < M && I >= 1 && I < M) ? 0.5f * (ct(l, I, J, 1) + ct(l, I - 1, J, 0)) : 0.0f;
        };
        constexpr int KGT = 128;
        auto kbar = []() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
        if (tid < KGT) {
            const int tk = tid;
            cluster_arrive_relaxed();                    // C (this group zeroes nothing)
            for (int e = tk; e < NK; e += KGT) {
                const int I = e % PK, J = e / PK;
                WHK[e] = whc(LK, I, J);
                WVK[e] = wvc(LK, I, J);
            }
            for (int e = tk; e < L::NE; e += KGT) {
                const int I = e % PE, J = e / PE;
                WHE[e] = whc(LK + 1, I, J);
                WVE[e] = wvc(LK + 1, I, J);
            }
            kbar();
            for (int e = tk; e < NK; e += KGT) {
                const int I = e % PK, J = e / PK;
                const bool in = I >= 1 && I < mK && J >= 1 && J < mK;
                const float dv = in ? WHK[e] + WHK[e - 1] + WVK[e] + WVK[e - PK] : 0.0f;
                DK[e] = dv;
                DIK[e] = in ? om / dv : 0.0f;
                SK[e] = 0.0f;
            }
            kbar();
            CL_MARK(pset, 26);
            if (warp == 0) {   // Gauss-Jordan inverse of the 4-cell operator (9 unknowns), by shuffles
                const int ri = lane < UE ? lane : 0;
                const int ia = ri % (mE - 1) + 1, ja = ri / (mE - 1) + 1, g = ja * PE + ia;
                const float wr = WHE[g], wl = WHE[g - 1], wu = WVE[g], wd = WVE[g - PE];
                float a[UE];
#pragma unroll
                for (int c = 0; c < UE; ++c)
                    a[c] = c == ri ? wr + wl + wu + wd
                         : (c == ri + 1 && ia < mE - 1) ? -wr
                         : (c == ri - 1 && ia > 1) ? -wl
                         : (c == ri + (mE - 1) && ja < mE - 1) ? -wu
                         : (c == ri - (mE - 1) && ja > 1) ? -wd : 0.0f;
#pragma unroll
                for (int k = 0; k < UE; ++k) {
                    float prow[UE];
#pragma unroll
                    for (int c = 0; c < UE; ++c) prow[c] = __shfl_sync(0xffffffffu, a[c], k);
                    const float piv = 1.0f / prow[k];
                    const float f = -a[k] * piv;
#pragma unroll
                    for (int c = 0; c < UE; ++c) {
                        if (lane == k) a[c] = c == k ? piv : prow[c] * piv;
                        else a[c] = c == k ? f : fmaf(f, prow[c], a[c]);
                    }
                }
                __syncwarp();
                if (lane < UE) {
#pragma unroll
                    for (int c = 0; c < UE; ++c) AI[lane * UE + c] = a[c];
                }
            }
            // K = 2 Dw - Dw AK Dw + B^T AE^-1 B,  B = PE^T (I - AK Dw)  (pcg_mg.cuh)
            for (int e = tk; e < UE * UK; e += KGT) {
                const int r = e / UK, k = e % UK;
                const int Ir = r % (mE - 1) + 1, Jr = r / (mE - 1) + 1;
                const int Ik = k % (mK - 1) + 1, Jk = k / (mK - 1) + 1, ek = Jk * PK + Ik;
                const float dwk = DIK[ek];
                auto wr = [&](int Im, int Jm) -> float {
                    const int ax = abs(Im - 2 * Ir), ay = abs(Jm - 2 * Jr);
                    return (ax > 1 || ay > 1) ? 0.0f : (ax ? 0.5f : 1.0f) * (ay ? 0.5f : 1.0f);
                };
                float v = wr(Ik, Jk) * (1.0f - DK[ek] * dwk);
                v = fmaf(wr(Ik + 1, Jk), WHK[ek] * dwk, v);
                v = fmaf(wr(Ik - 1, Jk), WHK[ek - 1] * dwk, v);
                v = fmaf(wr(Ik, Jk + 1), WVK[ek] * dwk, v);
                v = fmaf(wr(Ik, Jk - 1), WVK[ek - PK] * dwk, v);
                Bm[e] = v;
            }
            kbar();
            CL_MARK(pset, 27);
            for (int e = tk; e < UE * UK; e += KGT) {    // C = AE^-1 B
                const int r = e / UK, k = e % UK;
                float v = 0.0f;
#pragma unroll
                for (int c = 0; c < UE; ++c) v = fmaf(AI[r * UE + c], Bm[c * UK + k], v);
                Cm[e] = v;
            }
            kbar();
            CL_MARK(pset, 28);
        } else {
            const int tz = tid - KGT;
            constexpr int NZ = NT - KGT;
#pragma unroll
            for (int l = 2; l < LK; ++l) {
                const int Pq = L::Pl(l);
                float *wh = lc(l, LWH), *wv = lc(l, LWV);
                for (int e = tz; e < L::Nl(l); e += NZ) {
                    const int I = e % Pq, J = e / Pq;
                    wh[e] = whc(l, I, J);
                    wv[e] = wvc(l, I, J);
                }
            }
            if (tz < Q.d && bl + cluster_count_x() < nb) theta_amp(bl + cluster_count_x(), tz, th_next);
            {   // every runtime grid (16-byte stores; oU is 16-byte aligned)
                float4 *z4 = reinterpret_cast<float4 *>(sf + L::oU);
                for (int e = tz; e < L::URUN / 4; e += NZ) z4[e] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                for (int e = 4 * (L::URUN / 4) + tz; e < L::URUN; e += NZ) sf[L::oU + e] = 0.0f;
            }
            cluster_arrive();                            // C: own share of the grids zeroed
            for (int e = tz; e < L::F1; e += NZ) {       // level-1 omega D^-1 (rows 0 .. HR1+1)
                const int lrw = e / P1, s = e % P1, I = s < H1E ? 2 * s : s >= H1 ? 2 * (s - H1) + 1 : -1;
                const int jl = lrw - 1, J = J0 + jl;
                const bool in = I >= 1 && I < m1 && J >= 1 && J < m1 && jl >= 0 && jl <= HR1 + 1;
                const float dv = in ? WH1[e] + WH1[e1(I - 1, jl)] + WV1[e] + WV1[e - P1] : 1.0f;
                DI1[e] = in ? om / dv : 0.0f;
            }
            asm volatile("bar.sync 2, %0;" :: "n"(NZ) : "memory");   // the group's level-2.. couplings
#pragma unroll
            for (int l = 2; l < LK; ++l) {
                const int M = L::ml(l), Pq = L::Pl(l);
                const float *wh = lc(l, LWH), *wv = lc(l, LWV);
                float *di = lc(l, LDI);
                for (int e = tz; e < L::Nl(l); e += NZ) {
                    const int I = e % Pq, J = e / Pq;
                    const bool in = I >= 1 && I < M && J >= 1 && J < M;
                    di[e] = in ? om / (wh[e] + wh[e - 1] + wv[e] + wv[e - Pq]) : 0.0f;
                }
            }
        }
        __syncthreads();                                 // the two groups join: B, C complete, grids zeroed
        CL_MARK(pset, 25);
        cl_build_k<NN, CS>(sf);                          // K = B^T C + (2 Dw - Dw AK Dw), all warps
        CL_MARK(pset, 31);
        cluster_wait();      // C: every CTA's grids are zeroed before any neighbour sends into them
        CL_MARK(pset, 23);

        // ---- helpers of the iteration -----------------------------------------------------------
        // fp32 stencil of the preconditioner: own values in v, the rest from the grid Gs
        auto apply32 = [&](const float *Gs, const float (&v)[BR][BC], float (&out)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const float vl = c > 0 ? v[q][c - 1] : Gs[fe(c - 1, q)];
                    // the right neighbour of column n (the boundary node of the last column pair) is
                    // outside the grid; that node's result is masked, so read nothing there
                    const float vr = c + 1 < BC ? v[q][c + 1] : col0 + c + 2 <= n ? Gs[fe(c + 1, q)] : 0.0f;
                    const float vd = q > 0 ? v[q - 1][c] : Gs[fe(c, q - 1)];
                    const float vu = q + 1 < BR ? v[q + 1][c] : Gs[fe(c, q + 1)];
                    float a = dg32[q][c] * v[q][c];
                    a = fmaf(-ce[q][c + 1], vr, a);
                    a = fmaf(-ce[q][c], vl, a);
                    a = fmaf(-cn[q + 1][c], vu, a);
                    a = fmaf(-cn[q][c], vd, a);
                    out[q][c] = valid(q, c) ? a : 0.0f;
                }
        };
        auto publish = [&](float *Gd, const float (&v)[BR][BC]) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (valid(q, c)) Gd[fe(c, q)] = v[q][c];
        };
        // X1: z0 rows 1, 2 -> rows HR+1, HR+2 below; z0 row HR -> row 0 above; r row 1 -> Rh below
        auto send_x1 = [&](const float (&z)[BR][BC], const double (&rv)[BR][BC]) {
            if (rg == 0 && has_lo) {
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (col0 + c + 1 <= nx) {
                        st_async(G0_lo + 4 * (fe(c, 0) + HR * np), z[0][c], mb_lo);
                        st_async(G0_lo + 4 * (fe(c, 1) + HR * np), z[1][c], mb_lo);
                        st_async(Rh_lo + 4 * (col0 + c + 1), (float)rv[0][c], mb_lo);
                    }
            }
            if (rg == NRG - 1 && has_hi) {
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (col0 + c + 1 <= nx) st_async(G0_hi + 4 * (fe(c, BR - 1) - HR * np), z[BR - 1][c], mb_hi);
            }
        };
        auto prol2w = [](const float *Xc, int pc, int i, int j) -> float {   // bilinear, branch-free
            const float *z2 = Xc + (j >> 1) * pc + (i >> 1);
            const float wx1 = (i & 1) ? 0.5f : 0.0f, wx0 = (i & 1) ? 0.5f : 1.0f;
            const float wy1 = (j & 1) ? 0.5f : 0.0f, wy0 = (j & 1) ? 0.5f : 1.0f;
            return fmaf(wx1 * wy1, z2[pc + 1], fmaf(wx0 * wy1, z2[pc], fmaf(wx1 * wy0, z2[1], wx0 * wy0 * z2[0])));
        };
        // level-1 nodes (I in 1 .. m1-1) of the local rows jl = JA .. JA+NR-1 inside the mesh
        auto for1 = [&](auto ja, auto nr, auto body) {
            constexpr int JA = decltype(ja)::value, NR = decltype(nr)::value, U = m1 * NR;
#pragma unroll
            for (int k = 0; k < (U + NT - 1) / NT; ++k) {
                const int q = tid + k * NT, I = q % m1 + 1, jl = q / m1 + JA, J = J0 + jl;
                if (q < U && I < m1 && J >= 1 && J < m1) body(I, jl);
            }
        };
        using C1 = std::integral_constant<int, 1>;
        using CM1 = std::integral_constant<int, -1>;
        using C0 = std::integral_constant<int, 0>;
        using CHR1 = std::integral_constant<int, HR1>;
        using CHR1p1 = std::integral_constant<int, HR1 + 1>;
        using CHR1p2 = std::integral_constant<int, HR1 + 2>;
        using CHR1p4 = std::integral_constant<int, HR1 + 4>;
        // interior of a replicated level with M cells
        auto forl = [&](auto mc, auto body) {
            constexpr int M = decltype(mc)::value, U = (M - 1) * (M - 1);
#pragma unroll
            for (int k = 0; k < (U + NT - 1) / NT; ++k) {
                const int q = tid + k * NT, I = q % (M - 1) + 1, J = q / (M - 1) + 1;
                if (q < U) body(I, J, J * (M + 1) + I);
            }
        };
        // level-1 operator at (I, jl) (diagonal summed in the order of DI1)
        auto apply1 = [&](const float *Zs, int I, int jl) -> float {
            const int e = e1(I, jl), el = e1(I - 1, jl), er = e1(I + 1, jl);
            const float whe = WH1[e], whl = WH1[el], wve = WV1[e], wvd = WV1[e - P1];
            return (whe + whl + wve + wvd) * Zs[e] - whe * Zs[er] - whl * Zs[el] - wve * Zs[e + P1] -
                   wvd * Zs[e - P1];
        };

        // ---- CG init: x = 0, r = b, z0 = omega D^-1 b -----------------------------------------------
        double r[BR][BC];
        float z0[BR][BC];
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                Xg[(q * BC + c) * NT + tid] = Sg[(q * BC + c) * NT + tid] = Pg[(q * BC + c) * NT + tid] = 0.0;
                const int j = j0 + row0 + q + 1;
                r[q][c] = !valid(q, c) ? 0.0 : Bt ? __ldg(Bt + (j - 1) * nx + col0 + c) : (double)j * inv_n3;
                z0[q][c] = di0[q][c] * (float)r[q][c];
            }
        publish(G0, z0);
        send_x1(z0, r);
        double rho = 0.0, rho_prev = 0.0, bb = 0.0, g_inv = 0.0, ga_inv = 0.0;
        bool conv = false;
        int it = 0;
        bool pit = false;                                // probe this CG iteration
        (void)pit;
        for (int k = 0;; ++k) {
            pit = pset && k == 6;
            CL_MARK(pit, 0);
            // ======== V(1,1) cycle in fp32: uu = M^-1 r ==================================================
            __syncthreads();
            xwait(0);                                    // X1: z0 halos, r of the row above
            CL_MARK(pit, 1);
            float t[BR][BC];                             // fine residual t = r - A z0 of the own nodes -> G1
            {
                float az[BR][BC];
                apply32(G0, z0, az);
#pragma unroll
                for (int q = 0; q < BR; ++q)
#pragma unroll
                    for (int c = 0; c < BC; ++c) t[q][c] = valid(q, c) ? (float)r[q][c] - az[q][c] : 0.0f;
                publish(G1, t);
            }
            if (tid < nx) {                              // the residual of the row above (HR+1)
                const int i = tid + 1, e = (HR + 1) * np + slot0(i);
                const float east = WHh[i], west = WHh[i - 1], north = WVh1[i], south = WVh0[i];
                float a = (east + west + north + south) * G0[e];
                a = fmaf(-east, G0[(HR + 1) * np + slot0(i + 1)], a);
                a = fmaf(-west, G0[(HR + 1) * np + slot0(i - 1)], a);
                a = fmaf(-north, G0[e + np], a);
                a = fmaf(-south, G0[e - np], a);
                G1[e] = j0 + HR + 1 <= nx ? Rh[i] - a : 0.0f;
            }
            __syncthreads();
            CL_MARK(pit, 2);
            for1(C1{}, CHR1{}, [&](int I, int jl) {      // R1 = P^T t, Z1 = omega D1^-1 R1 (own rows)
                const int f = 2 * jl * np, c = I, l = HE + I - 1, rr = HE + I;
                const float rv = G1[f + c] + 0.5f * (G1[f + l] + G1[f + rr] + G1[f - np + c] + G1[f + np + c]) +
                                 0.25f * (G1[f - np + l] + G1[f - np + rr] + G1[f + np + l] + G1[f + np + rr]);
                const int e = e1(I, jl);
                const float zv = DI1[e] * rv;
                R1[e] = rv;
                Z1[e] = zv;
                // X2: Z1 rows 1, 2 and R1 row 1 -> rows HR1+1, HR1+2 below; Z1 rows HR1-1, HR1 and R1
                // row HR1 -> rows -1, 0 above
                if (jl <= 2 && has_lo) {
                    st_async(Z1_lo + 4 * e1(I, jl + HR1), zv, mb_lo + 8);
                    if (jl == 1) st_async(R1_lo + 4 * e1(I, jl + HR1), rv, mb_lo + 8);
                }
                if (jl >= HR1 - 1 && has_hi) {
                    st_async(Z1_hi + 4 * e1(I, jl - HR1), zv, mb_hi + 8);
                    if (jl == HR1) st_async(R1_hi + 4 * e1(I, jl - HR1), rv, mb_hi + 8);
                }
            });
            __syncthreads();
            xwait(1);                                    // X2
            CL_MARK(pit, 3);
            for1(C1{}, CHR1p1{}, [&](int I, int jl) {   // level-1 residual, own rows + the row above
                T1[e1(I, jl)] = R1[e1(I, jl)] - apply1(Z1, I, jl);
            });
            __syncthreads();
            CL_MARK(pit, 4);
            {   // X3: R2 = P^T T1 on the own level-2 rows, to every CTA's replicated grid
                constexpr int U = (m2 - 1) * HR2;
                const uint32_t R2a = smem_addr(R2);
#pragma unroll
                for (int kk = 0; kk < (U + NT - 1) / NT; ++kk) {
                    const int q = tid + kk * NT, I = q % (m2 - 1) + 1, jl2 = q / (m2 - 1) + 1, J = J20 + jl2;
                    if (q >= U || J >= m2) continue;
                    UB_CHECK(J >= 1 && I >= 1 && I < m2 && (2 * jl2 + 2) * P1 + H1 + I < L::F1);
                    const int f = (2 * jl2 + 1) * P1, c = I, l = H1 + I - 1, rr = H1 + I;
                    const float v = T1[f + c] + 0.5f * (T1[f + l] + T1[f + rr] + T1[f - P1 + c] + T1[f + P1 + c]) +
                                    0.25f * (T1[f - P1 + l] + T1[f - P1 + rr] + T1[f + P1 + l] + T1[f + P1 + rr]);
#pragma unroll
                    for (int kr = 0; kr < CS; ++kr) st_async(mapa(R2a + 4 * (J * P2 + I), kr), v, mapa(mb0 + 16, kr));
                }
            }
            xwait(2);                                    // X3
            CL_MARK(pit, 5);
            // ---- replicated levels 2 .. LK-1, then the K map (CTA-local) --------------------------
#pragma unroll
            for (int l = 2; l < LK; ++l) {               // down: Z = Dw R, T = R - A Z, restrict
                const int Pq = L::Pl(l);
                const float *wh = lc(l, LWH), *wv = lc(l, LWV), *di = lc(l, LDI), *rl = lr(l, LR);
                float *zl = lr(l, LZ), *tl = lr(l, LT);
                auto down = [&](int, int, int e) {       // the pre-smoothing from zero in the same pass
                    const float zc = di[e] * rl[e];
                    const float az = (wh[e] + wh[e - 1] + wv[e] + wv[e - Pq]) * zc -
                                     wh[e] * (di[e + 1] * rl[e + 1]) - wh[e - 1] * (di[e - 1] * rl[e - 1]) -
                                     wv[e] * (di[e + Pq] * rl[e + Pq]) - wv[e - Pq] * (di[e - Pq] * rl[e - Pq]);
                    zl[e] = zc;
                    tl[e] = rl[e] - az;
                };
                auto restr = [&](int I, int J, int ec) {
                    const int f = 2 * J * Pq + 2 * I;
                    const float v = tl[f] + 0.5f * (tl[f - 1] + tl[f + 1] + tl[f - Pq] + tl[f + Pq]) +
                                    0.25f * (tl[f - Pq - 1] + tl[f - Pq + 1] + tl[f + Pq - 1] + tl[f + Pq + 1]);
                    if (l + 1 < LK) lr(l + 1, LR)[ec] = v;
                    else RK[(J - 1) * (mK - 1) + I - 1] = v;
                };
                if (l == 2) forl(std::integral_constant<int, L::ml(2)>{}, down);
                else forl(std::integral_constant<int, L::ml(LK - 1)>{}, down);
                __syncthreads();
                if (l == 2) forl(std::integral_constant<int, L::ml(3)>{}, restr);
                else forl(std::integral_constant<int, L::ml(LK)>{}, restr);
                __syncthreads();
            }
            CL_MARK(pit, 6);
            constexpr int KT = 8 * ((UK + 3) / 4 * 4);   // SK = K RK (levels 8 and 4 cells): row i, 8 lanes
#pragma unroll
            for (int kb = 0; kb < (KT + NT - 1) / NT; ++kb) {
                const int tk = tid + kb * NT;
                if (tk - lane >= KT) break;              // whole warps only (shuffles below)
                const int l8 = tk & 7, i = min(tk >> 3, UK - 1);
                const float *kp = Kt + i * L::KS;
                float a = 0.0f;
#pragma unroll
                for (int m = 0; m < (UK + 7) / 8; ++m) {
                    const int c = l8 + 8 * m;
                    if (c < UK) a = fmaf(kp[c], RK[c], a);
                }
                a += __shfl_xor_sync(0xffffffffu, a, 4);
                a += __shfl_xor_sync(0xffffffffu, a, 2);
                a += __shfl_xor_sync(0xffffffffu, a, 1);
                if (l8 == 0 && (tk >> 3) < UK) SK[(i / (mK - 1) + 1) * PK + i % (mK - 1) + 1] = a;
            }
            __syncthreads();
            CL_MARK(pit, 7);
#pragma unroll
            for (int l = LK - 1; l >= 2; --l) {          // up: Zp = Z + P S_coarse; S = smooth(Zp) -> Z
                const int Pq = L::Pl(l);
                const float *xc = l + 1 < LK ? lr(l + 1, LZ) : SK;
                const int pc = l + 1 < LK ? L::Pl(l + 1) : PK;
                const float *wh = lc(l, LWH), *wv = lc(l, LWV), *di = lc(l, LDI), *rl = lr(l, LR);
                float *zl = lr(l, LZ), *zp = lr(l, LT);
                auto upa = [&](int I, int J, int e) { zp[e] = zl[e] + prol2w(xc, pc, I, J); };
                auto upb = [&](int, int, int e) {
                    const float zc = zp[e], we = wh[e], ww = wh[e - 1], wn = wv[e], ws = wv[e - Pq];
                    const float az = (we + ww + wn + ws) * zc - we * zp[e + 1] - ww * zp[e - 1] - wn * zp[e + Pq] -
                                     ws * zp[e - Pq];
                    zl[e] = fmaf(di[e], rl[e] - az, zc);
                };
                if (l == 2) forl(std::integral_constant<int, L::ml(2)>{}, upa);
                else forl(std::integral_constant<int, L::ml(LK - 1)>{}, upa);
                __syncthreads();
                if (l == 2) forl(std::integral_constant<int, L::ml(2)>{}, upb);
                else forl(std::integral_constant<int, L::ml(LK - 1)>{}, upb);
                __syncthreads();
            }
            CL_MARK(pit, 8);
            {   // level 1: Zp1 = Z1 + P S2 on rows -1 .. HR1+2 (-> T1), S1 = smooth(Zp1) on rows
                // 0 .. HR1+1 (own + one halo row each side; -> Z1)
                const float *S2 = lr(2, LZ);
                for1(CM1{}, CHR1p4{}, [&](int I, int jl) { T1[e1(I, jl)] = Z1[e1(I, jl)] + prol2w(S2, P2, I, J0 + jl); });
                __syncthreads();
                for1(C0{}, CHR1p2{}, [&](int I, int jl) {
                    const int e = e1(I, jl);
                    const float zc = T1[e];
                    const float whe = WH1[e], whl = WH1[e1(I - 1, jl)], wve = WV1[e], wvd = WV1[e - P1];
                    const float az = (whe + whl + wve + wvd) * zc - whe * T1[e1(I + 1, jl)] - whl * T1[e1(I - 1, jl)] -
                                     wve * T1[e + P1] - wvd * T1[e - P1];
                    Z1[e] = fmaf(DI1[e], R1[e] - az, zc);
                });
                __syncthreads();
            }
            CL_MARK(pit, 9);
            // level 0: uu = z0 + P S1, post-smoothed (window of S1 as in pcg_mg.cuh)
            float uu[BR][BC];
            {
                constexpr int XW = BC / 2 + 2, YW = BR / 2 + 2;
                float cw[YW][XW];
#pragma unroll
                for (int yy = 0; yy < YW; ++yy)
#pragma unroll
                    for (int xx = 0; xx < XW; ++xx) {
                        const int X = lx + xx, Y = (row0 >> 1) + yy;
                        UB_CHECK(!(X <= m1 && J0 + Y <= m1) || (Y + 1) * P1 + col1s(X) < L::F1);
                        cw[yy][xx] = (X <= m1 && J0 + Y <= m1) ? Z1[(Y + 1) * P1 + col1s(X)] : 0.0f;
                    }
                auto pw = [&](int c, int q) -> float {
                    const int fi = 1 + c, fj = 1 + q, xq = fi >> 1, yq = fj >> 1;
                    if (!(fi & 1) && !(fj & 1)) return cw[yq][xq];
                    if (!(fj & 1)) return 0.5f * (cw[yq][xq] + cw[yq][xq + 1]);
                    if (!(fi & 1)) return 0.5f * (cw[yq][xq] + cw[yq + 1][xq]);
                    return 0.25f * (cw[yq][xq] + cw[yq][xq + 1] + cw[yq + 1][xq] + cw[yq + 1][xq + 1]);
                };
#pragma unroll
                for (int q = 0; q < BR; ++q)
#pragma unroll
                    for (int c = 0; c < BC; ++c) {
                        const float ec = pw(c, q);
                        float a = dg32[q][c] * ec;
                        a = fmaf(-ce[q][c + 1], pw(c + 1, q), a);
                        a = fmaf(-ce[q][c], pw(c - 1, q), a);
                        a = fmaf(-cn[q + 1][c], pw(c, q + 1), a);
                        a = fmaf(-cn[q][c], pw(c, q - 1), a);
                        // TZ: t and z0 of the own node from the grids they were published to
                        uu[q][c] = !valid(q, c) ? 0.0f : TZ ? fmaf(di0[q][c], G1[fe(c, q)] - a, G0[fe(c, q)] + ec)
                                                            : fmaf(di0[q][c], t[q][c] - a, z0[q][c] + ec);
                    }
            }
            CL_MARK(pit, 10);
            // ======== w = A uu (fp64), dots, cluster reduction ===============================================
            publish(G1, uu);
            if (rg == 0 && has_lo) {                     // X4: row 1 -> row HR+1 below
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (col0 + c + 1 <= nx) st_async(G1_lo + 4 * (fe(c, 0) + HR * np), uu[0][c], mb_lo + 24);
            }
            if (rg == NRG - 1 && has_hi) {               // row HR -> row 0 above
#pragma unroll
                for (int c = 0; c < BC; ++c)
                    if (col0 + c + 1 <= nx) st_async(G1_hi + 4 * (fe(c, BR - 1) - HR * np), uu[BR - 1][c], mb_hi + 24);
            }
            __syncthreads();
            xwait(3);                                    // X4
            CL_MARK(pit, 11);
            double w[BR][BC];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    const double vl = c > 0 ? (double)uu[q][c - 1] : (double)G1[fe(c - 1, q)];
                    const double vr = c + 1 < BC ? (double)uu[q][c + 1] : col0 + c + 2 <= n ? (double)G1[fe(c + 1, q)] : 0.0;
                    const double vd = q > 0 ? (double)uu[q - 1][c] : (double)G1[fe(c, q - 1)];
                    const double vu = q + 1 < BR ? (double)uu[q + 1][c] : (double)G1[fe(c, q + 1)];
                    double a = (cE[q][c + 1] + cE[q][c] + cN[q + 1][c] + cN[q][c]) * (double)uu[q][c];
                    a = fma(-cE[q][c + 1], vr, a);
                    a = fma(-cE[q][c], vl, a);
                    a = fma(-cN[q + 1][c], vu, a);
                    a = fma(-cN[q][c], vd, a);
                    w[q][c] = valid(q, c) ? a : 0.0;
                }
            double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    acc[0] = fma(r[q][c], (double)uu[q][c], acc[0]);
                    acc[1] = fma(w[q][c], (double)uu[q][c], acc[1]);
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
            const int buf = k & 1;
            if (warp == 0 && lane < 3 * CS) {            // X5: CTA sums (warp order) to every CTA
                const int v = lane % 3, dst = lane / 3;
                double sv = 0.0;
#pragma unroll
                for (int ww = 0; ww < NWARP; ++ww) sv += wred[v * NWARP + ww];
                st_async(mapa(smem_addr(cred + (buf * CS + rank) * 4 + v), dst), sv, mapa(mb0 + 32, dst));
            }
            xwait(4);
            CL_MARK(pit, 12);
            double gs[3];
#pragma unroll
            for (int v = 0; v < 3; ++v) {
                double sv = 0.0;
#pragma unroll
                for (int rr2 = 0; rr2 < CS; ++rr2) sv += cred[(buf * CS + rr2) * 4 + v];
                gs[v] = sv;
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
                    const double pn = fma(beta, Pg[(q * BC + c) * NT + tid], (double)uu[q][c]);
                    Pg[(q * BC + c) * NT + tid] = pn;
                    const double sn = fma(beta, Sg[(q * BC + c) * NT + tid], w[q][c]);
                    Sg[(q * BC + c) * NT + tid] = sn;
                    Xg[(q * BC + c) * NT + tid] = fma(alpha, pn, Xg[(q * BC + c) * NT + tid]);
                    r[q][c] = fma(-alpha, sn, r[q][c]);
                    z0[q][c] = di0[q][c] * (float)r[q][c];
                }
            // Early stopping test: when the residual decay predicts (r,r) <= 4 tol^2 (b,b) for the new
            // r (rho^2 / rho_prev), reduce (r,r) now (X6) instead of after one more V-cycle.  The
            // partials follow exactly the tree of the X5 (r,r) (same fma order, shuffles, warp order,
            // rank order), so the value, the decision and x are those of the next iteration's test.
            if (k > 0 && rho * rho <= 4.0 * Q.tol2 * bb * rho_prev && it + 1 < Q.maxit) {
                double a2 = 0.0;
#pragma unroll
                for (int q = 0; q < BR; ++q)
#pragma unroll
                    for (int c = 0; c < BC; ++c) a2 = fma(r[q][c], r[q][c], a2);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
                if (lane == 0) wred[3 * NWARP + warp] = a2;
                __syncthreads();
                if (warp == 0 && lane < CS) {
                    double sv = 0.0;
#pragma unroll
                    for (int ww = 0; ww < NWARP; ++ww) sv += wred[3 * NWARP + ww];
                    st_async(mapa(smem_addr(cred + (buf * CS + rank) * 4 + 3), lane), sv, mapa(mb0 + 40, lane));
                }
                xwait(5);
                double rn = 0.0;
#pragma unroll
                for (int rr2 = 0; rr2 < CS; ++rr2) rn += cred[(buf * CS + rr2) * 4 + 3];
                if (rn <= Q.tol2 * bb) {                 // converged: x, r are the next test's
                    rho = rn;
                    conv = true;
                    ++it;
                    break;
                }
            }
            publish(G0, z0);
            send_x1(z0, r);
            CL_MARK(pit, 13);
            ++it;
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c)
                if (valid(q, c))   // sample-fastest output: 8 bytes per node; keep the partially written
                                   // sectors in L2 (evict_last) until the neighbouring samples' clusters fill them
                    asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
                                 "st.global.L2::cache_hint.f64 [%0], %1, pol;\n\t}"
                                 :: "l"(u + (int64_t)((j0 + row0 + q) * nx + col0 + c) * ldu + bl),
                                    "d"(Xg[(q * BC + c) * NT + tid]) : "memory");
        if (tid == 0 && rank == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rho / bb);
            if (noconv && !conv) atomicAdd(noconv, 1);
        }
        // the next sample's staging / coefficient table overwrite the union, which only this CTA reads now
        __syncthreads();
    }
    cluster_barrier();                                   // no CTA leaves while others may address it
}

}  // namespace usfft
