// pde.cu — K3 coefficient field + K4 batched preconditioned CG: one P1 FE solve per lattice node.
// usfft_sample_pde (include/usfft.h; a4 + a5 of SURVEY §8(a)).
//
// Discretisation (DESIGN.md §3 Z11/Z12): on the uniform "/" triangulation the P1 stiffness of
// -div(a grad u) with centroid-quadrature a is the 5-point operator
//     (A u)_p = sum_{edges e=(p,q)} w_e (u_p - u_q),
//     w_h(i,j) = (a(T_lo(i,j)) + a(T_up(i,j-1)))/2,  w_v(i,j) = (a(T_up(i,j)) + a(T_lo(i-1,j)))/2,
// T_lo(ci,cj) centroid ((ci+2/3)h, (cj+1/3)h), T_up(ci,cj) centroid ((ci+1/3)h, (cj+2/3)h);
// the centroid load of f = x2 is b_p = h^2 x2_p (closed form); other f (Z28) come from a table
// b_p = (h^2/6) sum of f over the centroids of the six triangles around p (k_rhs).  (The oracle
// assembles element by element; a CPU test checks this stencil against that assembly.)
//
// Kernels (one CTA per sample, persistent loop over samples, fixed-tree reductions so a sample's
// result does not depend on which CTA or rank solved it):
//   k_pcg_mg  (pcg_mg.cuh)   multigrid-preconditioned CG, fine level in registers, n = 16, 32
//   k_pcg_cl  (pcg_cl.cuh)   multigrid-preconditioned CG, one thread-block cluster per sample,
//                            fine level in registers across the cluster, n = 64, 128
//   k_pcg_mgg (pcg_mgg.cuh)  multigrid-preconditioned CG, per-CTA scratch slab, n = 8
//   k_pcg     (below)        Jacobi PCG, shared memory (n <= 64) or a global slab, any n
#include <cstdlib>
#include <vector>

#include "lattice.cuh"

namespace usfft {

struct PdeParams {
    int32_t n, d, theta, form, f_kind, maxit, precond, psi;
    double tol2;              // tol^2
    double delta;             // global pole shift of phi_Delta (Z27)
    double amp[kMaxD];
};

__device__ __forceinline__ double theta_of(int kind, double y, double delta) {
    if (kind == 0) return sinpi(2.0 * y);                         // sin(2 pi y)
    if (kind == 1) return 1.0 - fabs(2.0 * (1.0 - 2.0 * y));      // tent, eq. tent
    if (kind == 3) {                                               // phi_Delta = tau1 o tau2,Delta (Z27)
        const double t2 = y < delta ? -0.5 - 2.0 * (y - delta)     // tau2,Delta
                        : y < 0.5 + delta ? -0.5 + 2.0 * (y - delta) : 1.5 - 2.0 * (y - delta);
        y = t2 + 0.5;                                              // tau1(t) = Phi^-1(t + 1/2)
    }
    double v = normcdfinv(y);                                      // Phi^-1 (Z15)
    return fmin(fmax(v, -6.0), 6.0);                               // clip, NaN-free: -inf -> -6
}

// The separable spatial factors psi_j(x) = X_j(x1) Y_j(x2) at the abscissae m h/3, m = 0..3n
// (the centroid abscissae are (3c+1)h/3, (3c+2)h/3): S[0][j][m] = X_j, S[1][j][m] = Y_j, the
// second plane only when Y differs from X (psi != 0).  Arguments are exact rationals
// (integer numerator / 3n) through sinpi / cospi.
//   psi 0: X_j = Y_j = sin(j pi t)
//   psi 1: X_j = cos(2 pi m1(j) t), Y_j = cos(2 pi m2(j) t)          (Table 3)
//   psi 2: X_j = sin(2 pi j t), Y_j = cos(2 pi (d+1-j) t)
__global__ void k_psitab(int n, int d, int psi, double *__restrict__ S) {
    const int W = 3 * n + 1, planes = psi == 0 ? 1 : 2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < planes * d * W; e += gridDim.x * blockDim.x) {
        const int pl = e / (d * W), j = (e / W) % d + 1, m = e % W;
        const double t3n = (double)(3 * n);
        double v;
        if (psi == 0) {
            v = sinpi((double)(j * m) / t3n);
        } else if (psi == 1) {
            int k = 1;                                       // k(j): largest k with k(k+1)/2 <= j
            while ((k + 1) * (k + 2) / 2 <= j) ++k;
            const int m1 = j - k * (k + 1) / 2, mm = pl == 0 ? m1 : k - m1;
            v = cospi((double)(2 * mm * m) / t3n);
        } else {
            v = pl == 0 ? sinpi((double)(2 * j * m) / t3n) : cospi((double)(2 * (d + 1 - j) * m) / t3n);
        }
        S[e] = v;
    }
}

// f at the point (m1 h/3, m2 h/3) for f_kind 1, 2 (Z28)
__device__ __forceinline__ double f_at(int kind, int n, int m1, int m2) {
    if (kind == 1) return 1.0;                                   // affine example
    const double x1 = (double)m1 / (3.0 * n), x2 = (double)m2 / (3.0 * n);
    return sinpi(1.3 * x1 + 3.4 * x2) * cospi(4.3 * x1 - 3.1 * x2);   // lognormal example
}

// centroid-rule loads b_g = sum_{T containing g} f(c_T) |T| / 3 = (h^2 / 6) sum over the six
// triangles T_lo(i,j), T_up(i,j), T_lo(i-1,j), T_lo(i-1,j-1), T_up(i-1,j-1), T_up(i,j-1)
__global__ void k_rhs(int n, int kind, double *__restrict__ B) {
    const int nx = n - 1;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < nx * nx; g += gridDim.x * blockDim.x) {
        const int i = g % nx + 1, j = g / nx + 1;
        const double s = f_at(kind, n, 3 * i + 2, 3 * j + 1) + f_at(kind, n, 3 * i + 1, 3 * j + 2) +
                         f_at(kind, n, 3 * i - 1, 3 * j + 1) + f_at(kind, n, 3 * i - 1, 3 * j - 2) +
                         f_at(kind, n, 3 * i - 2, 3 * j - 1) + f_at(kind, n, 3 * i + 1, 3 * j - 1);
        B[g] = s / (6.0 * n * n);
    }
}

// a at a triangle centroid with table columns m1 (x1, plane X) and m2 (x2, plane Y)
__device__ __forceinline__ double coef_at(const PdeParams &Q, const double *__restrict__ th_amp,
                                          const double *__restrict__ X, const double *__restrict__ Y,
                                          int W, int m1, int m2) {
    double s = 0.0;
    for (int j = 0; j < Q.d; ++j) s += th_amp[j] * X[j * W + m1] * Y[j * W + m2];
    return Q.form == 0 ? 1.0 + s : exp(s);
}

template <int NPT, int THREADS>
__global__ void __launch_bounds__(THREADS)
k_pcg(const LatParams P, const PdeParams Q, const double *__restrict__ nodes, int64_t b0,
      int64_t nb, double *__restrict__ u, int64_t ldu, int32_t *__restrict__ iters,
      double *__restrict__ relres, int32_t *__restrict__ noconv, const double *__restrict__ S,
      const double *__restrict__ Bt, double *__restrict__ gscratch, int64_t region) {
    extern __shared__ double smem[];
    __shared__ double red[64];
    __shared__ double th_amp[kMaxD];

    const int n = Q.n, nx = n - 1, G = nx * nx, np = n + 1, W = 3 * n + 1;
    double *base = gscratch ? gscratch + (int64_t)blockIdx.x * region : smem;
    double *p = base;                    // [(n+1)^2] padded
    double *wh = p + np * np;            // wh[j*np+i]: edge (i,j)-(i+1,j)
    double *wv = wh + np * np;           // wv[j*np+i]: edge (i,j)-(i,j+1)
    double *x = wv + np * np;            // [G]
    double *r = x + G;                   // [G]
    double *dinv = r + G;                // [G]
    constexpr int T = THREADS;
    const int tid = threadIdx.x;
    const double h2b = 1.0 / ((double)n * n * n);   // b_p = h^2 * x2_p = j / n^3 (f = x2)
    const double *Sy = S + (Q.psi ? Q.d * W : 0);

    for (int64_t bl = blockIdx.x; bl < nb; bl += gridDim.x) {
        const int64_t b = b0 + bl;
        // ---- K3: theta_j(y_b) and the edge weights ----------------------------------------
        for (int j = tid; j < Q.d; j += blockDim.x) {      // d may exceed the CTA (n = 16: 32 threads)
            const double y = nodes ? nodes[(int64_t)j * nb + bl] : lattice_node(P, b, j);
            th_amp[j] = Q.amp[j] * theta_of(Q.theta, y, Q.delta);
        }
        __syncthreads();
        for (int e = tid; e < np * np; e += T) {
            const int i = e % np, j = e / np;
            p[e] = 0.0;
            double h = 0.0, v = 0.0;
            if (i < n && j >= 1 && j <= nx)                        // horizontal edge (i,j)-(i+1,j)
                h = 0.5 * (coef_at(Q, th_amp, S, Sy, W, 3 * i + 2, 3 * j + 1) +        // T_lo(i,j)
                           coef_at(Q, th_amp, S, Sy, W, 3 * i + 1, 3 * (j - 1) + 2));  // T_up(i,j-1)
            if (j < n && i >= 1 && i <= nx)                        // vertical edge (i,j)-(i,j+1)
                v = 0.5 * (coef_at(Q, th_amp, S, Sy, W, 3 * i + 1, 3 * j + 2) +        // T_up(i,j)
                           coef_at(Q, th_amp, S, Sy, W, 3 * (i - 1) + 2, 3 * j + 1));  // T_lo(i-1,j)
            wh[e] = h;
            wv[e] = v;
        }
        __syncthreads();
        // ---- PCG init: x = 0, r = b, p = z = D^-1 r ---------------------------------------
        double acc[2] = {0.0, 0.0};      // rz, bb
        for (int k = 0; k < NPT; ++k) {
            const int g = tid + k * T;
            if (g < G) {
                const int i = g % nx + 1, j = g / nx + 1, e = j * np + i;
                const double dg = wh[e] + wh[e - 1] + wv[e] + wv[e - np];
                const double di = 1.0 / dg;
                const double bv = Bt ? Bt[g] : (double)j * h2b;
                dinv[g] = di;
                x[g] = 0.0;
                r[g] = bv;
                const double z = di * bv;
                p[e] = z;
                acc[0] += bv * z;
                acc[1] += bv * bv;
            }
        }
        block_sum<2>(acc, red);
        double rz = acc[0];
        const double bb = acc[1];
        double rr = bb;
        int it = 0;
        while (rr > Q.tol2 * bb && it < Q.maxit) {
            // q = A p, pq = p.q
            double q[NPT];
            double pq[1] = {0.0};
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int g = tid + k * T;
                q[k] = 0.0;
                if (g < G) {
                    const int i = g % nx + 1, j = g / nx + 1, e = j * np + i;
                    const double we = wh[e], ww = wh[e - 1], wn = wv[e], ws = wv[e - np];
                    const double pc = p[e];
                    const double qq = (we + ww + wn + ws) * pc - we * p[e + 1] - ww * p[e - 1] -
                                      wn * p[e + np] - ws * p[e - np];
                    q[k] = qq;
                    pq[0] += pc * qq;
                }
            }
            block_sum<1>(pq, red);
            const double alpha = rz / pq[0];
            double acc2[2] = {0.0, 0.0};   // rz_new, rr
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int g = tid + k * T;
                if (g < G) {
                    const int i = g % nx + 1, j = g / nx + 1, e = j * np + i;
                    x[g] += alpha * p[e];
                    const double rn = r[g] - alpha * q[k];
                    r[g] = rn;
                    acc2[0] += rn * (dinv[g] * rn);
                    acc2[1] += rn * rn;
                }
            }
            block_sum<2>(acc2, red);
            const double beta = acc2[0] / rz;
            rz = acc2[0];
            rr = acc2[1];
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int g = tid + k * T;
                if (g < G) {
                    const int i = g % nx + 1, j = g / nx + 1, e = j * np + i;
                    p[e] = dinv[g] * r[g] + beta * p[e];
                }
            }
            __syncthreads();
            ++it;
        }
        // ---- output u[g][bl] ----------------------------------------------------------------
        for (int g = tid; g < G; g += T) u[(int64_t)g * ldu + bl] = x[g];
        if (tid == 0) {
            if (iters) iters[bl] = it;
            if (relres) relres[bl] = sqrt(rr / bb);
            if (noconv && rr > Q.tol2 * bb) atomicAdd(noconv, 1);
        }
        __syncthreads();
    }
}

}  // namespace usfft

#include "pcg_mg.cuh"
#include "pcg_mgg.cuh"
#include "pcg_cl.cuh"

using namespace usfft;

namespace {
template <int NC, int BC, int BR, int LX, int NWARP, int MINB>
usfft_status launch_pcg_mg(usfft_ctx *c, const LatParams &P, const PdeParams &Q,
                           const double *nodes, int64_t b0, int64_t nb, double *u, int64_t ldu,
                           int32_t *iters, double *relres, int32_t *noconv, const double *S,
                           const double *Bt) {
    const int sw = (Q.psi ? 2 : 1) * Q.d * (3 * NC + 1);  // staged psi tables (if small enough)
    const size_t dyn = sizeof(double) * ((size_t)Mg3<NC>::doubles() + (MINB * NWARP >= 12 ? 2 * BC * BR * NWARP * 32 : 0) +
                                         (sw <= Mg3<NC>::SMAX ? sw : 0));
    auto kern = k_pcg_mg<NC, BC, BR, LX, NWARP, MINB>;
    int per_sm = 0;
    if (usfft_status s = kernel_fit(c, kern, NWARP * 32, dyn, &per_sm)) return s;
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)per_sm * c->sm_count;
    if (grid > nb) grid = nb;
    kern<<<(unsigned)grid, NWARP * 32, dyn, c->stream>>>(P, Q, nodes, b0, nb, u, ldu, iters, relres,
                                                         noconv, S, Bt);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

template <int NN>
usfft_status launch_pcg_mgg_n(usfft_ctx *c, const LatParams &P, const PdeParams &Q, const double *nodes,
                              int64_t b0, int64_t nb, double *u, int64_t ldu, int32_t *iters, double *relres,
                              int32_t *noconv, const double *S, const double *Bt) {
    // 512 threads, two CTAs per SM (measured against 256 x 2, 256 x 3, 512 x 1 and 1024 x 1 with
    // the fine stencil arrays in shared memory: 2.66 vs 3.69, 3.93, 3.78, 3.65 us per sample at
    // n = 64; the kernel is bound by L1/L2 latency, so resident warps matter more than L2 fit)
    constexpr int T = 512;
    using C = MggC<NN>;
    const size_t dyn = sizeof(double) * (size_t)C::smem();
    auto kern = k_pcg_mgg<NN, T, 2>;
    int per_sm = 0;
    if (usfft_status s = kernel_fit(c, kern, T, dyn, &per_sm)) return s;
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)per_sm * c->sm_count;
    if (grid > nb) grid = nb;
    if (usfft_status s = ensure(c, &c->ws, &c->ws_size, sizeof(double) * (size_t)grid * (size_t)C::region())) return s;
    kern<<<(unsigned)grid, T, dyn, c->stream>>>(P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt,
                                              static_cast<double *>(c->ws));
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

// one thread-block cluster of CS CTAs per sample (pcg_cl.cuh), as many clusters as fit at once,
// each looping over samples
template <int NN, int CS, int MINB>
usfft_status launch_pcg_cl(usfft_ctx *c, const LatParams &P, const PdeParams &Q, const double *nodes,
                           int64_t b0, int64_t nb, double *u, int64_t ldu, int32_t *iters, double *relres,
                           int32_t *noconv, const double *S, const double *Bt) {
    using C = ClC<NN, CS>;
    // the psi factors of each CTA's strip resident in shared memory when they fit (pd = d)
    const int pd = C::bytes() + C::psi_bytes(Q.d) + 1024 <= c->smem_optin ? Q.d : 0;
    const size_t dyn = C::bytes() + (pd ? C::psi_bytes(pd) : 0);
    auto kern = k_pcg_cl<NN, CS, MINB>;
    if (usfft_status s = kernel_fit(c, kern, C::NT, dyn, nullptr)) return s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(C::NT);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = c->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const auto key = std::make_pair(reinterpret_cast<const void *>(kern), dyn * 2048 + (size_t)C::NT + (size_t(1) << 62));
    auto it = c->occupancy.find(key);
    if (it == c->occupancy.end()) {
        int ncl = 0;
        cfg.gridDim = dim3(CS * c->sm_count);
        USFFT_CUDA(c, cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
        if (ncl < 1) return fail(c, USFFT_ECUDA, "no cluster of %d CTAs (%zu B shared memory) fits", CS, dyn);
        it = c->occupancy.emplace(key, ncl).first;
    }
    int64_t ncl = it->second;
    if (ncl > nb) ncl = nb;
    cfg.gridDim = dim3((unsigned)(ncl * CS));
    USFFT_CUDA(c, cudaLaunchKernelEx(&cfg, kern, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt, pd));
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}

usfft_status launch_pcg_mgg(usfft_ctx *c, const LatParams &P, const PdeParams &Q, const double *nodes,
                            int64_t b0, int64_t nb, double *u, int64_t ldu, int32_t *iters, double *relres,
                            int32_t *noconv, const double *S, const double *Bt) {
    switch (Q.n) {
    case 8: return launch_pcg_mgg_n<8>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    default: return fail(c, USFFT_EUNIMPL, "scratch-slab multigrid compiled for n = 8");
    }
}

template <int NPT, int THREADS>
usfft_status launch_pcg(usfft_ctx *c, const LatParams &P, const PdeParams &Q, const double *nodes,
                        int64_t b0, int64_t nb, double *u, int64_t ldu, int32_t *iters,
                        double *relres, int32_t *noconv, const double *S, const double *Bt) {
    const int threads = THREADS;
    const int n = Q.n, G = (n - 1) * (n - 1), np = n + 1;
    const int64_t region = 3LL * np * np + 3LL * G;           // doubles per sample state
    const size_t bytes = (size_t)region * sizeof(double);
    double *gscratch = nullptr;
    int grid = 0;
    size_t dyn = 0;
    if (bytes + 1024 <= c->smem_optin) {
        dyn = bytes;
        int per_sm = 0;
        if (usfft_status s = kernel_fit(c, k_pcg<NPT, THREADS>, threads, dyn, &per_sm)) return s;
        if (per_sm < 1) per_sm = 1;
        grid = per_sm * c->sm_count;
    } else {
        int per_sm = 0;
        if (usfft_status s = kernel_fit(c, k_pcg<NPT, THREADS>, threads, 0, &per_sm)) return s;
        if (per_sm < 1) per_sm = 1;
        grid = per_sm * c->sm_count;
        if ((int64_t)grid > nb) grid = (int)nb;
        usfft_status s = ensure(c, &c->ws, &c->ws_size, (size_t)grid * bytes);
        if (s) return s;
        gscratch = static_cast<double *>(c->ws);
    }
    if ((int64_t)grid > nb) grid = (int)nb;
    k_pcg<NPT, THREADS><<<grid, threads, dyn, c->stream>>>(P, Q, nodes, b0, nb, u, ldu, iters, relres,
                                                   noconv, S, Bt, gscratch, region);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}
}  // namespace

extern "C" usfft_status usfft_sample_pde(usfft_ctx *c, const usfft_pde_desc *pde,
                                         const usfft_lattice_desc *lat, int64_t b0, int64_t nb,
                                         const double *nodes, double *u, int64_t ldu,
                                         int32_t *iters, double *relres, int32_t *n_noconv) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, pde != nullptr, "pde desc is NULL");
    static thread_local LatParams P;
    static thread_local PdeParams Q;
    usfft_status s = make_lat_params(c, lat, &P);
    if (s) return s;
    USFFT_REQUIRE(c, pde->n >= 2 && pde->n <= 128, "n = %d out of [2, 128]", pde->n);
    USFFT_REQUIRE(c, pde->d >= 1 && pde->d <= P.d, "pde d = %d must be in [1, lattice d]", pde->d);
    USFFT_REQUIRE(c, pde->theta >= 0 && pde->theta <= 3, "theta kind %d", pde->theta);
    USFFT_REQUIRE(c, pde->theta != 3 || (pde->delta > 0.0 && pde->delta < 0.5), "delta out of (0, 1/2)");
    USFFT_REQUIRE(c, pde->form == 0 || pde->form == 1, "form %d", pde->form);
    USFFT_REQUIRE(c, pde->f_kind >= 0 && pde->f_kind <= 2, "f_kind %d", pde->f_kind);
    USFFT_REQUIRE(c, pde->psi >= 0 && pde->psi <= 2, "psi %d", pde->psi);
    USFFT_REQUIRE(c, pde->amp != nullptr, "amp is NULL");
    USFFT_REQUIRE(c, pde->tol > 0.0 && pde->maxit >= 1, "tol/maxit");
    USFFT_REQUIRE(c, pde->precond == 0 || pde->precond == 1, "precond %d", pde->precond);
    USFFT_REQUIRE(c, b0 >= 0 && nb >= 0 && b0 + nb <= (int64_t)P.L * P.M, "sample range");
    USFFT_REQUIRE(c, ldu >= nb && u != nullptr, "u is NULL or ldu < nb");
    if (nb == 0) {
        if (n_noconv) *n_noconv = 0;
        return USFFT_OK;
    }
    Q.n = pde->n;
    Q.d = pde->d;
    Q.theta = pde->theta;
    Q.form = pde->form;
    Q.f_kind = pde->f_kind;
    Q.maxit = pde->maxit;
    Q.precond = pde->precond;
    Q.delta = pde->delta;
    Q.psi = pde->psi;
    Q.tol2 = pde->tol * pde->tol;
    for (int j = 0; j < pde->d; ++j) Q.amp[j] = pde->amp[j];

    // psi factor tables for (n, d, psi) and the load table for (n, f_kind != 0): cached per ctx
    auto key = std::make_tuple(pde->n, pde->d, pde->psi);
    double *S = nullptr, *Bt = nullptr;
    auto it = c->sintab.find(key);
    if (it == c->sintab.end()) {
        const size_t cnt = (size_t)(pde->psi ? 2 : 1) * pde->d * (3 * pde->n + 1);
        USFFT_CUDA(c, cudaMalloc(&S, cnt * sizeof(double)));
        k_psitab<<<grid1d(cnt, 256), 256, 0, c->stream>>>(pde->n, pde->d, pde->psi, S);
        USFFT_CHECK_LAUNCH(c);
        c->sintab[key] = S;
    } else {
        S = it->second;
    }
    if (pde->f_kind != 0) {
        auto rk = std::make_pair(pde->n, pde->f_kind);
        auto rt = c->rhstab.find(rk);
        if (rt == c->rhstab.end()) {
            const size_t cnt = (size_t)(pde->n - 1) * (pde->n - 1);
            USFFT_CUDA(c, cudaMalloc(&Bt, cnt * sizeof(double)));
            k_rhs<<<grid1d(cnt, 256), 256, 0, c->stream>>>(pde->n, pde->f_kind, Bt);
            USFFT_CHECK_LAUNCH(c);
            c->rhstab[rk] = Bt;
        } else {
            Bt = rt->second;
        }
    }
    // non-converged counter (device slot 0), only when the caller asks for it
    int32_t *noconv = n_noconv ? reinterpret_cast<int32_t *>(c->dscal) : nullptr;
    if (noconv) USFFT_CUDA(c, cudaMemsetAsync(noconv, 0, sizeof(int32_t), c->stream));

    // one kernel per (preconditioner, mesh): multigrid-preconditioned CG with the fine level in
    // registers of one CTA (n = 16, 32) or of a thread-block cluster (n = 64, 128); Jacobi PCG
    // (precond 0, or meshes the multigrid does not cover) through the shared/global-memory kernel
    const int n = pde->n, G = (n - 1) * (n - 1);
    if (pde->precond == 1 && n == 32)
        s = launch_pcg_mg<32, 2, 4, 16, 4, 2>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (pde->precond == 1 && n == 16)
        s = launch_pcg_mg<16, 2, 4, 8, 1, 2>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (pde->precond == 1 && n == 128)
        s = launch_pcg_cl<128, 8, 1>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (pde->precond == 1 && n == 64)
        s = launch_pcg_cl<64, 4, 2>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (pde->precond == 1 && n == 8)
        s = launch_pcg_mgg(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (pde->precond == 1)
        return fail(c, USFFT_EUNIMPL, "multigrid preconditioner needs n in {8, 16, 32, 64, 128}");
    // threads x nodes-per-thread: 128x2 (G <= 256), 256x4 (G <= 1024), 512x8, 1024x16
    else if (G <= 256) s = launch_pcg<2, 128>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (G <= 1024) s = launch_pcg<4, 256>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else if (G <= 4096) s = launch_pcg<8, 512>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    else s = launch_pcg<16, 1024>(c, P, Q, nodes, b0, nb, u, ldu, iters, relres, noconv, S, Bt);
    if (s) return s;
    int32_t host_nc = 0;
    if (n_noconv) {
        USFFT_CUDA(c, cudaMemcpyAsync(&host_nc, noconv, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        USFFT_CUDA(c, cudaStreamSynchronize(c->stream));
        *n_noconv = host_nc;
    }
    if (n_noconv && host_nc > 0)
        return fail(c, USFFT_ENOCONV, "%d of %lld samples missed tol at maxit", host_nc, (long long)nb);
    return USFFT_OK;
}


#ifdef USFFT_CL_PROBE
// probe build only (tools/cl_probe.py): the phase clocks of k_pcg_cl
extern "C" int usfft_debug_cl_probe(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, usfft::g_cl_probe, sizeof(long long) * 16 * 32);
}
#endif
