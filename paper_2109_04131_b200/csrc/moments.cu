// moments.cu — post-processing of the coefficients: expectation, variance and global sensitivity
// indices per node (usfft_moments, include/usfft.h, reading Z30).
//
//   E_g = sum_k c_{k,g} D_k   (D_k = prod_j D_{k_j}: P:945-952 periodic, eq. affine_ew
//                             tent, P:985-996 phi_Delta)
//   sigma^2_g = sum_{k != 0} |c_{k,g}|^2,   rho_l(g) = sum_{||k||_0 = l} |c_{k,g}|^2 / sigma^2_g
//                             (eq. gsi, eq. J)
// K12a evaluates D_k and ||k||_0 once per frequency; K12b reduces one node per CTA with per-thread
// partial sums in a fixed order and fixed-tree block sums (deterministic).  O(G |I|) work: a few
// microseconds, off the detection hot path.
#include "common.cuh"

namespace usfft {

__global__ void k_dweights(const int16_t *__restrict__ I, int64_t nI, int d, int map, double delta,
                           double2 *__restrict__ D, int32_t *__restrict__ ell) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nI; a += (int64_t)gridDim.x * blockDim.x) {
        double re = 1.0, im = 0.0;
        int l = 0;
        for (int j = 0; j < d; ++j) {
            const int kj = I[a * d + j];
            if (kj == 0) continue;
            ++l;
            if (map == 0 || (kj & 1) == 0) {             // periodic: delta_k; even k_j: 0
                re = im = 0.0;
                continue;
            }
            // 2i / (pi k_j) (e^{2 pi i k_j Delta} for phi_Delta)
            double fr = 0.0, fi = 2.0 / (3.141592653589793 * kj);
            if (map == 3) {
                double s, c;
                sincospi(2.0 * kj * delta, &s, &c);
                const double r2 = -fi * s, i2 = fi * c;
                fr = r2;
                fi = i2;
            }
            const double nr = re * fr - im * fi, ni = re * fi + im * fr;
            re = nr;
            im = ni;
        }
        D[a] = make_double2(re, im);
        ell[a] = l;
    }
}

__global__ void __launch_bounds__(256)
k_moments(const double2 *__restrict__ C, int64_t nI, int d, const double2 *__restrict__ D,
          const int32_t *__restrict__ ell, double *__restrict__ E, double *__restrict__ var,
          double *__restrict__ gsi) {
    __shared__ double red[32 * 3];
    const int64_t g = blockIdx.x;
    const double2 *row = C + g * nI;
    double acc[kMaxD];
    for (int l = 0; l < d; ++l) acc[l] = 0.0;
    double v[3] = {0.0, 0.0, 0.0};                      // Re E, Im E, sigma^2
    for (int64_t a = threadIdx.x; a < nI; a += blockDim.x) {
        const double2 c = row[a], w = D[a];
        v[0] += c.x * w.x - c.y * w.y;
        v[1] += c.x * w.y + c.y * w.x;
        const int l = ell[a];
        if (l > 0) {
            const double m = c.x * c.x + c.y * c.y;
            v[2] += m;
            acc[l - 1] += m;
        }
    }
    block_sum<3>(v, red);
    if (threadIdx.x == 0) {
        E[2 * g] = v[0];
        E[2 * g + 1] = v[1];
        var[g] = v[2];
    }
    if (gsi) {
        const double inv = v[2] > 0.0 ? 1.0 / v[2] : 0.0;
        for (int l = 0; l < d; ++l) {
            double p[1] = {acc[l]};
            block_sum<1>(p, red);
            if (threadIdx.x == 0) gsi[g * d + l] = v[2] > 0.0 ? p[0] * inv : 0.0;
        }
    }
}

}  // namespace usfft

using namespace usfft;

extern "C" usfft_status usfft_moments(usfft_ctx *c, int32_t d, const int16_t *I, int64_t nI,
                                      const double *C, int64_t G, int32_t map, double delta,
                                      double *E, double *var, double *gsi) {
    USFFT_ENTER(c);
    USFFT_REQUIRE(c, d >= 1 && d <= kMaxD && nI >= 0 && G >= 0, "bad sizes");
    USFFT_REQUIRE(c, map == 0 || map == 1 || map == 3, "map %d: expectation weights exist for sin (0), tent (1), phi_Delta (3)", map);
    USFFT_REQUIRE(c, map != 3 || (delta > 0.0 && delta < 0.5), "delta out of (0, 1/2)");
    if (G == 0) return USFFT_OK;
    USFFT_REQUIRE(c, E && var && (nI == 0 || (I && C)), "NULL argument");
    const size_t need = (sizeof(double2) + sizeof(int32_t)) * (size_t)(nI > 0 ? nI : 1);
    if (usfft_status s = ensure(c, &c->ws, &c->ws_size, need)) return s;
    double2 *D = static_cast<double2 *>(c->ws);
    int32_t *ell = reinterpret_cast<int32_t *>(D + (nI > 0 ? nI : 1));
    if (nI > 0) {
        k_dweights<<<grid1d(nI, 256), 256, 0, c->stream>>>(I, nI, d, map, delta, D, ell);
        USFFT_CHECK_LAUNCH(c);
    }
    USFFT_REQUIRE(c, G <= 0x7fffffff, "G too large");
    k_moments<<<(unsigned)G, 256, 0, c->stream>>>(reinterpret_cast<const double2 *>(C), nI, d, D, ell, E, var, gsi);
    USFFT_CHECK_LAUNCH(c);
    return USFFT_OK;
}
