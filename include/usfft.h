/*
 * usfft.h — C-ABI of the B200-native usFFT detection step (arXiv 2109.04131).
 *
 * The operations are the steps of one dimension-incremental detection round of Alg. 1
 * "The usFFT on a set T_G".  Citations: P:n = PAPER.md line n (LaTeX
 * source) with its section/equation/algorithm; S:n = SPEC.md line n; Zn = a reading of a place
 * where the paper is silent, listed in DESIGN.md §3.
 *
 * Conventions (all calls)
 *  - Every function returns usfft_status.  USFFT_OK = 0.  On USFFT_EINVAL nothing was launched or
 *    written.  CUDA errors are sticky (the ctx must be finalized); USFFT_ENOCONV and
 *    USFFT_ENOTRECON are not sticky and the outputs are written.  usfft_last_error() returns a
 *    message owned by the ctx (valid until the next call on it).
 *  - "dev" pointers are device memory owned by the caller (e.g. torch tensors); the library
 *    borrows them for stream-ordered use on the ctx stream, so the caller keeps them alive until
 *    that stream has passed the call.  "host" pointers are read during the call only (they are
 *    staged into ctx-owned device memory before the call returns).  Workspace (tables, per-CTA
 *    scratch) is owned by the ctx and grows on demand.
 *  - Calls are asynchronous on the ctx stream unless marked "syncs" (a host output needs it).
 *  - One ctx per (GPU, stream); not thread-safe.  Multi-GPU (one process per GPU):
 *    every rank creates its ctx with (rank, nranks, id) and calls every collective function
 *    (marked "collective") in the same order; the library moves the data itself over NCCL
 *    (a6 usfft_transpose; C2 in usfft_detect_select; C3 in usfft_detect_union).  Samples and
 *    nodes are partitioned in contiguous balanced ranges (the first n % P ranks get one more).
 *  - Layouts: sample index fastest.  Samples of a round are b = l*M + i (lattice l, node i).
 *    Candidates of a round are j = a*n1 + c for rows a of I_prev and entries c of kt (Z10).
 */
#ifndef USFFT_H
#define USFFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t usfft_status;
enum {
    USFFT_OK = 0,
    USFFT_EINVAL = 1,     /* bad argument; nothing launched                                  */
    USFFT_ENOMEM = 2,     /* workspace allocation failed                                      */
    USFFT_ECUDA = 3,      /* CUDA error (sticky)                                              */
    USFFT_ENCCL = 4,      /* NCCL error or NCCL unavailable (sticky)                          */
    USFFT_ENOCONV = 5,    /* some PCG sample missed tol at maxit (outputs still written)      */
    USFFT_ENOTRECON = 6,  /* injectivity test failed (mode-R caller decides what to do)       */
    USFFT_EUNIMPL = 7     /* option not implemented                                           */
};

typedef struct usfft_ctx usfft_ctx;

/* Rank-1 lattice sampling set of one round (R1L P:230-233; eq. lattice_nodes P:837-839;
 * Alg. 1 Step 2b P:309-311; Step 1 line nodes P:288-293).
 *   d          parameter dimension d_y
 *   t          components of z (Step 2: the round's dimension t; Step 1: 1)
 *   line_axis  -1 for Step 2 (components 0..t-1 from the lattice, t..d-1 = shift);
 *              a >= 0 for Step 1 (component a = ((i*z) mod M)/M with t = 1, all others = shift)
 *   L, M       number of lattices and lattice size (M >= 2; prime for Step 2, Z2)
 *   z          host int64 [L][t], entries in [0, M)
 *   shift      host fp64 [d], the random components x' of the round, in [0,1)
 */
typedef struct {
    int32_t d;
    int32_t t;
    int32_t line_axis;
    int32_t L;
    int64_t M;
    const int64_t *z;
    const double *shift;
} usfft_lattice_desc;

/* PDE black box (eq. pde, weak form P:155-158; coefficient families P:84-98; BASELINE
 * configs; P1 FE on the uniform "/" triangulation with centroid quadrature, Z11/Z12).
 *   n          cells per side, G = (n-1)^2 interior nodes (x1 fastest), 2 <= n <= 128
 *   d          number of coefficient terms (<= 64)
 *   theta      0: sin(2 pi y) (periodic)  1: tent 1-|2(1-2y)| (eq. tent)
 *              2: clip(Phi^-1(y), -6, 6) (Z15)
 *              3: clip(tau1(tau2_Delta(y)), -6, 6), the lognormal periodization phi_Delta
 *                 (eq. lognormal_transfo, tau1 P:486, tau2 P:500-506; Z27)
 *   form       0: a = 1 + sum_j amp_j theta_j psi_j(x)   1: a = exp(sum_j amp_j theta_j psi_j(x))
 *   psi        spatial factors psi_j (Z28):
 *              0: sin(j pi x1) sin(j pi x2) (BASELINE configs; periodic example P:1008)
 *              1: cos(2 pi m1(j) x1) cos(2 pi m2(j) x2), m1/m2/k(j) of Table 3 (affine example
 *                 P:1210-1216)
 *              2: sin(2 pi j x1) cos(2 pi (d+1-j) x2) (lognormal example P:1425)
 *   f_kind     0: f(x) = x2 (BASELINE configs, periodic example P:1002)  1: f = 1 (affine
 *              example P:1204)  2: f = sin(1.3 pi x1 + 3.4 pi x2) cos(4.3 pi x1 - 3.1 pi x2)
 *              (lognormal example P:1419); loads by the centroid rule (Z12)
 *   amp        host fp64 [d]
 *   tol        relative residual target ||r_k||_2 <= tol ||b||_2 (Z13; BASELINE 1e-12)
 *   maxit      PCG iteration cap
 *   precond    0: Jacobi (diagonal) PCG;  1: geometric-multigrid V(1,1) preconditioned CG
 *              (damped-Jacobi smoothing, bilinear P, R = P^T, rediscretised coarse meshes down
 *              to 4 cells per side; n a power of two >= 8 -> USFFT_EUNIMPL otherwise).  Any solver is admissible
 *              for the black box; both are CG with an SPD preconditioner (Z13).
 *   delta      the pole shift Delta of theta = 3, in (0, 1/2): one global value per run
 *              (Z27: 1/(4 M0), M0 the Step-2 lattice size, Lemma P:847-870); ignored otherwise
 */
typedef struct {
    int32_t n;
    int32_t d;
    int32_t theta;
    int32_t form;
    int32_t f_kind;
    int32_t maxit;
    const double *amp;
    double tol;
    int32_t precond;
    int32_t psi;
    double delta;
} usfft_pde_desc;

/* Round plan input/output (usfft_plan_round). */
typedef struct {
    int64_t seed;
    int32_t step;     /* 1: Step 1 & 2a line round; 2: Step 2 round   */
    int32_t t;        /* dimension-increment index t, 1-based                                */
    int32_t i;        /* detection round i, 1-based                                           */
    int32_t d;        /* parameter dimension d_y                                              */
    int32_t N;        /* search box Gamma = [-N, N]^d, K_t = 2N+1                     */
    int32_t s_tilde;  /* sparsity of the round                                        */
    int32_t mode;     /* Algorithm A: 0 = L random R1Ls (Z1), 1 = single reconstructing */
    int32_t pad_;
    int64_t nJ;       /* |J_t| (Step 2) or K_t (Step 1)                                        */
} usfft_plan_in;

typedef struct {
    int64_t M;           /* lattice size                                                      */
    int32_t L;           /* number of lattices                                                */
    int32_t t_z;         /* components of each z (desc.t)                                     */
    int32_t line_axis;   /* desc.line_axis                                                    */
    int32_t pad_;
    int64_t z[2048];     /* [L][t_z]                                                          */
    double shift[64];    /* x'_1..x'_d                                                        */
} usfft_plan_out;

/* Sizes of one detection round, for usfft_workspace_query. */
typedef struct {
    int32_t n;        /* cells per side of the FE mesh                                         */
    int32_t d;        /* parameter dimension                                                   */
    int64_t M;        /* lattice size                                                          */
    int32_t L;        /* lattices                                                              */
    int32_t s_tilde;  /* sparsity of the round                                                 */
    int64_t nJ;       /* candidates                                                            */
} usfft_round_desc;

/* ---- context ------------------------------------------------------------------------------ */

/* Create a ctx on `device` launching on `stream` (a cudaStream_t; NULL = legacy default) for rank
 * `rank` of `nranks`.  nranks == 1: no communicator, comm_id may be NULL.
 * nranks > 1: comm_id = 128 bytes; loopback == 0: an ncclUniqueId from usfft_comm_unique_id on
 * one rank, broadcast by the caller (e.g. torch.distributed), and the communicator is created
 * here (ncclCommInitRank, collective over the ranks, one GPU per rank); loopback == 1: nranks
 * virtual ranks in ONE process on one GPU, each driven by its own host thread with its own ctx
 * and stream, comm_id any 128 bytes shared by them (the rendezvous key).
 * Errors: EINVAL (bad rank / device / id), ENCCL (NCCL unavailable or init failed). */
usfft_status usfft_init(usfft_ctx **out, int device, void *stream, int rank, int nranks,
                        const void *comm_id, int loopback);
/* 128-byte ncclUniqueId (NCCL loaded at run time); ENCCL without NCCL. */
usfft_status usfft_comm_unique_id(void *out);
usfft_status usfft_comm_info(const usfft_ctx *ctx, int32_t *rank, int32_t *nranks, int32_t *loopback);
/* Upper bound of the device bytes the calls of a round with these sizes allocate in the ctx
 * (tables, workspace); caller-owned arrays not included.  No device work. */
usfft_status usfft_workspace_query(usfft_ctx *ctx, const usfft_round_desc *round, size_t *bytes);
usfft_status usfft_set_stream(usfft_ctx *ctx, void *stream);
usfft_status usfft_finalize(usfft_ctx *ctx);
const char *usfft_last_error(const usfft_ctx *ctx);
/* Number of kernels this ctx has launched since init (evidence counter for benchmarks). */
int64_t usfft_launch_count(const usfft_ctx *ctx);

/* ---- a1: round plan (usfft_plan_round) ----------------------------------------------------
 * The random choices of round (t, i) of Alg. 1: the shift x' (P:287 / P:307, one per round and
 * shared by every lattice and node chi_g) and the sampling set (Step 1: the line
 * lattice z = 1, M = K_t; Step 2 mode A: M, L and z_l by readings Z2-Z4; mode R: the first
 * reconstructing z found by the search of Z2 on the device-resident J_t = I_prev x kt, syncs).
 * I_prev / kt are only read in mode R (dev int16, layouts as in usfft_lattice). */
usfft_status usfft_plan_round(usfft_ctx *ctx, const usfft_plan_in *in, const int16_t *I_prev,
                              int64_t n_prev, const int16_t *kt, int32_t n1, usfft_plan_out *out);

/* The pole shift of the phi_Delta periodization (theta = 3), one global value per run (Z27):
 * Delta = 1 / (4 M0), M0 the Step-2 lattice size of the run (Z2 rule for lattice_factor *
 * s_local and N) -- the Lemma's optimum Delta_opt = 1/(4M) (Remark P:875-879). */
usfft_status usfft_plan_delta(usfft_ctx *ctx, int32_t N, int32_t s_local, int32_t lattice_factor,
                              double *delta);

/* ---- a2 + a3: lattice nodes and candidate index maps (usfft_lattice) -----------------------
 * nodes    dev fp64 [d][nb] (may be NULL): component j of sample b0+bl, bl < nb, per the desc.
 *          Bit-exact: ((i*z) mod M) is an exact int64 and is divided by M once (IEEE).
 * I_prev   dev int16 [n_prev][t-1] rows of I^(1..t-1) (ignored when t == 1; pass n_prev = 1)
 * kt       dev int16 [n1], the candidate t-th components (I^(t) in Step 2; -N..N in Step 1)
 * bins     dev int32 [L][n_prev*n1] (may be NULL): b_l(k) = (k . z_l) mod M in [0, M)
 *          (S:119-127).  Requires |k_c| * z * t < 2^62.
 * injective host int32 [L] (may be NULL; syncs): 1 if k -> b_l(k) is one-to-one on J_t
 *          (reconstructing single R1L, Table 1 row 1 P:242), else 0.  When any
 *          entry is 0 the call returns USFFT_ENOTRECON. */
usfft_status usfft_lattice(usfft_ctx *ctx, const usfft_lattice_desc *lat, int64_t b0, int64_t nb,
                           double *nodes, const int16_t *I_prev, int64_t n_prev,
                           const int16_t *kt, int32_t n1, int32_t *bins, int32_t *injective);

/* ---- a4 + a5: sample the black box (usfft_sample_pde) -------------------------------------
 * One FE solve per node y_b, b = b0 .. b0+nb-1 (Alg. 1 Step 2c "Sample p ... for every chi_g",
 * P:313; one solve serves all G nodes).  The nodes are generated in-kernel from `lat`
 * (bit-identical to usfft_lattice) unless `nodes` (dev fp64 [d][nb]) is given.
 * Preconditioned CG (pde->precond: Jacobi or multigrid) from x0 = 0, stop on the recursive
 * ||r||_2 <= tol ||b||_2 (Z13).
 * u        dev fp64 [G][ldu]: u[g*ldu + bl] = u(x_g, y_{b0+bl}), ldu >= nb
 * iters    dev int32 [nb] (may be NULL): PCG iterations per sample
 * relres   dev fp64 [nb] (may be NULL): final recursive ||r||/||b|| (Jacobi path: or an upper bound)
 * n_noconv host int32 (may be NULL: no count, no sync; else syncs): samples that missed tol;
 *          > 0 -> USFFT_ENOCONV */
usfft_status usfft_sample_pde(usfft_ctx *ctx, const usfft_pde_desc *pde,
                              const usfft_lattice_desc *lat, int64_t b0, int64_t nb,
                              const double *nodes, double *u, int64_t ldu, int32_t *iters,
                              double *relres, int32_t *n_noconv);

/* ---- a6: transpose (usfft_transpose, collective) ------------------------------------------
 * The one exchange step of a round: this rank's samples of all nodes,
 * u_local dev fp64 [G][nb] (nb = the rank's share of the B samples, ldu == nb), become the
 * rank's nodes of all samples as P slabs back to back, slabs dev fp64 [G_loc][B] with slab p
 * = [G_loc][nb_p] at offset G_loc * b0_p (the slab layout usfft_lattice_fft reads, slab_b0 =
 * the sample partition).  nranks > 1: grouped ncclSend / ncclRecv (loopback: device copies);
 * nranks == 1: a device copy (none if slabs == u_local).  Pure data movement (bit-exact). */
usfft_status usfft_transpose(usfft_ctx *ctx, int64_t G, int64_t B, const double *u_local, int64_t ldu,
                             double *slabs);

/* ---- a7 + a8: lattice FFT and detection key (usfft_lattice_fft) ----------------------------
 * For each owned node g < G_loc and lattice l: the length-M DFT of the samples of lattice l
 * (Alg. 1 P:296 "via FFT"), then for each candidate j the per-lattice value
 *   v_l(j,g) = (1/M) F[g][l][b] (conj(F[g][l][M-b]) for b > M/2, real input, Z17/Z18)
 * and the key kappa_min(j,g) = min_l fl(fl(re*re) + fl(im*im)) (Z1, Z5).
 * u        dev fp64 sample slabs after the exchange: nslab slabs back to back, slab p holds
 *          [G_loc][slab_b0[p+1]-slab_b0[p]] and starts at u + G_loc*slab_b0[p]
 *          (nslab = 1, slab_b0 = {0, L*M}: plain [G_loc][L*M])
 * slab_b0  host int64 [nslab+1], 0 = slab_b0[0] < ... < slab_b0[nslab] = L*M
 * spectra  dev fp64x2 [G_loc][L][M/2+1] (unscaled DFT bins 0..M/2)
 * kappa_min dev fp64 [G_loc][nJ];  kappa_max dev fp64 [1]: max over owned g and all j */
usfft_status usfft_lattice_fft(usfft_ctx *ctx, const usfft_lattice_desc *lat, int64_t G_loc,
                               const double *u, int32_t nslab, const int64_t *slab_b0,
                               const int32_t *bins, int64_t nJ, double *spectra,
                               double *kappa_min, double *kappa_max);

/* ---- a9 + a10: threshold and per-node selection (usfft_detect_select, collective) ----------
 * theta^2 = fl(theta_abs^2) if theta_abs > 0, else fl(fl(theta_rel^2) * kappa_max[0]) (Z5);
 * with nranks > 1 and the relative threshold (theta_abs <= 0 < theta_rel) the call first
 * all-reduces kappa_max (MAX, in place: C2) so it is the max over ALL nodes.
 * For each owned g: D_g = the first s_tilde candidates in the order (kappa desc, j asc) (Z6)
 * that satisfy kappa >= theta^2 and kappa > 0 (Alg. 1, Step 2d P:316).
 * votes    dev int32 [nJ]: zeroed, then votes[j] = #{owned g : j in D_g} (Z24)
 * det_g    dev int32 [G_loc][s_tilde]: D_g ascending, -1 padded;  n_det_g dev int32 [G_loc]
 * theta2   dev fp64 [1] (may be NULL): the theta^2 used */
usfft_status usfft_detect_select(usfft_ctx *ctx, int64_t G_loc, int64_t nJ,
                                 const double *kappa_min, double *kappa_max,
                                 int32_t s_tilde, double theta_rel, double theta_abs,
                                 int32_t *votes, int32_t *det_g, int32_t *n_det_g,
                                 double *theta2);

/* ---- a8 + a10 streamed over candidate chunks (large |J|; usfft_lattice_keys, usfft_detect_carry)
 * kappa_min of a run is G_loc * nJ doubles (Step 2 of a slowly decaying function reaches
 * |J| ~ 1e7, i.e. tens of GB).  The selection of a10 only needs each node's top s_tilde, so the
 * keys can be produced chunk by chunk and merged into a per-node carry of at most s_tilde
 * (key, j) pairs; the result is identical to the one-shot selection (Z29):
 *   merged [G_loc][s_tilde + C]: carry keys (ascending j, 0-padded) then the chunk's keys;
 *   usfft_detect_select on merged (theta_rel = theta_abs = 0: top s~ of the positive keys, with
 *   positions ascending = j ascending because every carry j precedes every chunk j);
 *   usfft_detect_carry (update mode) moves the selected pairs to the front (and to carry_k);
 * after the last chunk (and the all-reduce of kappa_max), usfft_detect_select on carry_k with
 * the real threshold and usfft_detect_carry (emit mode) give det_g (global j) and votes.
 *
 * usfft_lattice_keys: the keys of a8 from existing spectra for nJ candidates whose bins are
 *   bins[l * ldb + j] (l < L, j < nJ); writes kappa_min[g * ldk + j] and max-accumulates
 *   kappa_max (NOT reset: zero it before the first chunk) over the true keys.  tau (dev fp64
 *   [G_loc], may be NULL): a key <= tau[g] is written as 0 (it cannot beat a full carry whose
 *   smallest key is tau[g]: ties go to the carry's smaller j). */
usfft_status usfft_lattice_keys(usfft_ctx *ctx, const usfft_lattice_desc *lat, int64_t G_loc,
                                const double *spectra, const int32_t *bins, int64_t ldb,
                                int64_t nJ, double *kappa_min, int64_t ldk, double *kappa_max,
                                const double *tau);

/* usfft_lattice_keys_product: the same keys for the candidates j0 .. j0+nJ-1 of a product set
 *   J = I_prev x kt with j = a n1 + c (Z10; n1 = |kt|, ldb = |J| = n_prev n1, < 2^31), whose bin
 *   map bins[l * ldb + j] is given whole (the candidate offset is j0, not folded into bins).
 *   kappa_min[g * ldk + (j - j0)]; kappa_max and tau as above.  The product structure gives
 *   bins[l][a n1 + c] = (bins[l][a n1] + bins[l][c] - bins[l][0]) mod M, so when the spectra
 *   of the call exceed the L2 cache and |J| >= 4 (M/2+1) the library stages each (node, lattice) spectrum once per tile of candidates in shared memory
 *   instead of gathering one sector per (node, candidate, lattice) (Alg. 1 Step 2c P:313-315; the
 *   keys are bit-identical to usfft_lattice_keys).  Errors: EINVAL on sizes (ldb % n1 != 0). */
usfft_status usfft_lattice_keys_product(usfft_ctx *ctx, const usfft_lattice_desc *lat, int64_t G_loc,
                                        const double *spectra, const int32_t *bins, int64_t ldb,
                                        int64_t j0, int64_t nJ, int64_t n1, double *kappa_min,
                                        int64_t ldk, double *kappa_max, const double *tau);

/* usfft_detect_carry, for each owned g with the selection det_pos[g][0..n_det_g[g]) (positions
 * into row g of merged, ascending, as written by usfft_detect_select on merged):
 *   update mode (det_g == NULL): j of position p = carry_j[g][p] for p < s_tilde, else
 *     j0 + p - s_tilde; the selected (key, j) pairs become merged[g][0..n) and carry_k[g][0..n),
 *     carry_j[g][0..n); slots n..s_tilde-1 get key 0 and j = -1;
 *   emit mode (det_g != NULL; merged = carry_k, width = s_tilde): det_g[g][r] =
 *     carry_j[g][det_pos[g][r]] (-1 padded to s_tilde) and votes[that j] += 1 (votes zeroed by
 *     the caller, int32 [nJ]).
 * merged dev fp64 [G_loc][width]; carry_k dev fp64 [G_loc][s_tilde]; carry_j dev int32
 * [G_loc][s_tilde]; det_pos dev int32 [G_loc][s_tilde]; n_det_g dev int32 [G_loc];
 * tau dev fp64 [G_loc] (update mode, may be NULL): the smallest carry key when the carry holds
 * s_tilde pairs, else 0 (the prefilter of usfft_lattice_keys). */
usfft_status usfft_detect_carry(usfft_ctx *ctx, int64_t G_loc, int32_t s_tilde, int64_t width,
                                double *merged, double *carry_k, int32_t *carry_j,
                                const int32_t *det_pos, const int32_t *n_det_g, int64_t j0,
                                int32_t *det_g, int32_t *votes, double *tau);

/* ---- a11: union (usfft_detect_union, collective) -------------------------------------------
 * With nranks > 1 the call first all-reduces votes (SUM, in place: C3) so they count the nodes
 * of every rank (Step 2e P:318: union over g).  flags |= (votes > 0)
 * (running union over the rounds i of one t).  Outputs, identical on every rank:
 * det_idx  dev int32 [nJ]: this round's detected j ascending; n_det host int64 (syncs)
 * union_idx dev int32 [nJ] (may be NULL): all j with flags set, ascending; n_union host int64
 * n_det == NULL (then n_union must be NULL too): the call does not synchronise; the rounds
 * i < r of one dimension t only feed the running flags, so a driver enqueues them back to back
 * and reads the counts of the last round alone. */
usfft_status usfft_detect_union(usfft_ctx *ctx, int64_t nJ, int32_t *votes,
                                uint8_t *flags, int32_t *det_idx, int64_t *n_det,
                                int32_t *union_idx, int64_t *n_union);

/* ---- a12: coefficient resolve (usfft_resolve) ---------------------------------------------
 * For each owned g and each k = det_idx[q], q < n_det (Step 2d "computes the Fourier
 * coefficients" P:277/P:316, reading Z1):
 *   l*(k,g) = min{ l : no k' in D_g \ {k} has b_l(k') = b_l(k) };  coef = v_{l*}(k,g);
 *   no such l: componentwise lower median over l of v_l(k,g), lstar = -1.
 * coef dev fp64x2 [G_loc][n_det];  lstar dev int32 [G_loc][n_det] (may be NULL) */
usfft_status usfft_resolve(usfft_ctx *ctx, const usfft_lattice_desc *lat, int64_t G_loc,
                           const double *spectra, const int32_t *bins, int64_t nJ,
                           const int32_t *det_g, const int32_t *n_det_g, int32_t s_tilde,
                           const int32_t *det_idx, int64_t n_det, double *coef,
                           int32_t *lstar);

/* ---- candidate rows (usfft_gather_rows) ----------------------------------------------------
 * rows[q] = (I_prev[a], kt[c]) for j = idx[q] = a*n1 + c, q < n: the frequency vectors of
 * I^(1..t) handed to the next dimension.  rows dev int16 [n][t]. */
usfft_status usfft_gather_rows(usfft_ctx *ctx, const int32_t *idx, int64_t n,
                               const int16_t *I_prev, int32_t t, const int16_t *kt, int32_t n1,
                               int16_t *rows);

/* ---- evaluation (usfft_eval) --------------------------------------------------------------
 * U[g][q] = Re sum_{k in I} C[g][k] e^{2 pi i k . y_q} (eq. eval_formula, identity
 * periodization of the periodic model P:945-949).
 * I dev int16 [nI][d]; C dev fp64x2 [G][nI]; Y dev fp64 [d][n]; U dev fp64 [G][n] */
usfft_status usfft_eval(usfft_ctx *ctx, int32_t d, const int16_t *I, int64_t nI,
                        const double *C, int64_t G, const double *Y, int64_t n, double *U);

/* ---- Step 3: multiple-R1L cover of the detected set (usfft_cover_plan / usfft_cover_gather)
 * Alg. 1 Step 3: a sampling set X of the final I = I^(1..d) on which the Fourier
 * matrix can be inverted efficiently, realised by multiple rank-1 lattices ([KaPoVo17, Alg. 1],
 * P:349/P:362, Remark 4 P:1662) in reading Z26: every lattice has M = the smallest prime
 * >= max(4 (|I| - 1), N + 1) with M - 1 7-smooth; lattice q (1-based) draws z in [1, M-1]^d
 * (Z4 draw with tag 5, t = d, i = q, l = attempt) until some still unassigned k has a residue
 * k.z mod M unique among the residues of ALL of I (<= 100 empty draws); those k are assigned to
 * it (first lattice wins).  Its nodes are y_i = (i z mod M)/M in all d components (use
 * usfft_lattice / usfft_sample_pde with t = d, L = 1, line_axis = -1, zero shift).
 *   I      host int16 [nI][d] frequency rows
 *   out    cover: nlat <= 64 lattices, shared M, z host int64 [nlat][d]
 *   assign host int32 [nI]: the lattice of frequency a;  bin host int32 [nI]: its residue there
 * Errors: EINVAL on bad sizes, ENOTRECON after 100 consecutive empty draws or > 64 lattices.
 * Pure host computation (no device work, no sync). */
typedef struct {
    int32_t nlat;
    int32_t d;
    int64_t M;
    int64_t z[64 * 64];
} usfft_cover_desc;

usfft_status usfft_cover_plan(usfft_ctx *ctx, int64_t seed, int32_t d, int32_t N, const int16_t *I,
                              int64_t nI, usfft_cover_desc *out, int32_t *assign, int32_t *bin);

/* Step 3 coefficients of one cover lattice: coef[g][idx[a]] = v(k, g) = F^[g][bin[a]] / M for
 * a < n (each k read on its assigned lattice), where F^[m] = F[g][m] for m <= M/2
 * and conj(F[g][M-m]) above (the half spectrum of usfft_lattice_fft with L = 1).
 *   spectra dev fp64x2 [G][M/2+1]; idx, bin dev int32 [n]; coef dev fp64x2 [G][nI] */
usfft_status usfft_cover_gather(usfft_ctx *ctx, int64_t M, int64_t G, const double *spectra,
                                const int32_t *idx, const int32_t *bin, int64_t n, double *coef,
                                int64_t nI);

/* Direct lattice DFT at the bins in use (Step 3 on cover lattices too large for the FFT
 * kernels, Z26): coef[g][idx[a]] = (1/M) sum_{i<M} u[g][i] e^{-2 pi i (i bins[a] mod M)/M} with
 * the exact integer phase index (the oracle's direct DFT, P:296 / S:158).  u is the exchanged
 * sample slab buffer of one lattice as in usfft_lattice_fft (nslab, slab_b0 spanning [0, M]);
 * bins, idx dev int32 [n]; coef dev fp64x2 [G_loc][nI]. */
usfft_status usfft_lattice_dft_bins(usfft_ctx *ctx, int64_t M, int64_t G_loc, const double *u,
                                    int32_t nslab, const int64_t *slab_b0, const int32_t *bins,
                                    const int32_t *idx, int64_t n, double *coef, int64_t nI);

/* ---- accuracy metric (usfft_eval_err) ------------------------------------------------------
 * per node g over the n test points y_q (Y dev fp64 [d][n]),
 *   err[g][0] = (1/n) sum_q |Uref[g][q] - u(g, y_q)|,  err[g][1] = sqrt((1/n) sum_q |.|^2),
 *   err[g][2] = max_q |.|,   u(g, y) = sum_{k in I} C[g][k] e^{2 pi i k . y} (complex modulus).
 * I dev int16 [nI][d]; C dev fp64x2 [G][nI]; Uref dev fp64 [G][n] (the FE solutions at Y);
 * err dev fp64 [G][3].  Fixed reduction order (deterministic).  Uses ctx workspace. */
usfft_status usfft_eval_err(usfft_ctx *ctx, int32_t d, const int16_t *I, int64_t nI,
                            const double *C, int64_t G, const double *Y, int64_t n,
                            const double *Uref, double *err);

/* ---- post-processing: expectation, variance, GSI (usfft_moments) ---------------------------
 * Per node g (reading Z30), with I dev int16 [nI][d] and C dev fp64x2 [G][nI]:
 *   E[g] (fp64x2) = sum_k C[g][k] D_k, D_k = prod_j D_{k_j}:
 *     map 0 (periodic, theta = sin): D_k = 1 for k = 0, else 0 (E = c_0);
 *     map 1 (tent; eq. affine_ew): D_{k_j} = 2i/(pi k_j) for odd k_j, 1 for 0, else 0;
 *     map 3 (phi_Delta): the tent factors times e^{2 pi i k_j delta};
 *   var[g] = sum_{k != 0} |C[g][k]|^2;
 *   gsi[g][l-1] = sum_{||k||_0 = l} |C[g][k]|^2 / var[g] for l = 1..d (0 where var[g] = 0);
 * gsi may be NULL.  Other maps (2: clipped Phi^-1) have no closed form: EINVAL.  Fixed-order
 * reductions (deterministic).  Uses ctx workspace. */
usfft_status usfft_moments(usfft_ctx *ctx, int32_t d, const int16_t *I, int64_t nI, const double *C,
                           int64_t G, int32_t map, double delta, double *E, double *var, double *gsi);

#ifdef __cplusplus
}
#endif
#endif /* USFFT_H */
