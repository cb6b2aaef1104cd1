// mg_probe.cu — phase latencies of the multigrid PCG kernel (k_pcg_mg) on the B200.
// Build (links the library sources with the probe macro):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DUSFFT_MG_PROBE -Iinclude \
//        tools/mg_probe.cu paper_2109_04131_b200/csrc/{ctx,plan,lattice,pde,fft,detect,eval}.cu -o /tmp/mg_probe
// Prints, for CTA 0 / sample 0 / CG iteration 6, the cycles each warp spends between the
// synchronisation points (mark ids in pcg_mg.cuh).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "usfft.h"

extern "C" int usfft_debug_mg_probe(long long *out);

int main() {
    usfft_ctx *ctx = nullptr;
    if (usfft_init(&ctx, 0, nullptr) != 0) { printf("init failed\n"); return 1; }
    const int d = 10, n = 32, G = (n - 1) * (n - 1);
    const int64_t M = 401, nb = 6817;
    const int L = 17;
    std::vector<int64_t> z(5 * L);
    uint64_t st = 12345;
    for (auto &v : z) {                               // any z in [1, M): timing only
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        v = 1 + (int64_t)((st >> 33) % (uint64_t)(M - 1));
    }
    std::vector<double> shift(d, 0.25), amp(d);
    for (int j = 0; j < d; ++j) amp[j] = 0.4 / double((j + 1) * (j + 1));
    usfft_lattice_desc lat{d, 5, -1, L, M, z.data(), shift.data()};
    usfft_pde_desc pde{n, d, 0, 0, 0, 20000, amp.data(), 1e-12, 1, 0};
    double *u = nullptr;
    cudaMalloc(&u, sizeof(double) * G * nb);
    for (int rep = 0; rep < 2; ++rep)
        if (usfft_sample_pde(ctx, &pde, &lat, 0, nb, nullptr, u, nb, nullptr, nullptr, nullptr)) {
            printf("solve failed: %s\n", usfft_last_error(ctx));
            return 1;
        }
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    usfft_sample_pde(ctx, &pde, &lat, 0, nb, nullptr, u, nb, nullptr, nullptr, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("solve of %lld samples: %.3f ms\n", (long long)nb, ms);
    long long pr[16][32];
    usfft_debug_mg_probe(&pr[0][0]);
    const char *names[14] = {"iter start", "A1 z0 publish", "A2 residual", "R1 Z1", "T1", "L2 R2 Z2",
                             "L2 T2", "L2 R3", "L2 E3", "L2 S2 + bar", "Zc1", "S1", "post-smooth", "apply+red"};
    printf("%-16s", "phase");
    for (int w = 0; w < 4; ++w) printf("   warp%d", w);
    printf("\n");
    for (int id = 1; id <= 13; ++id) {
        printf("%-16s", names[id]);
        for (int w = 0; w < 4; ++w) {
            long long a = pr[w][id], b = pr[w][id - 1];
            if (id == 9 && w > 0) b = pr[w][4];
            if (id >= 5 && id <= 8 && w > 0) { printf("       -"); continue; }
            if (id == 5 && w == 0) b = pr[w][4];
            printf(" %7lld", a - b);
        }
        printf("\n");
    }
    printf("iteration total: %lld cycles (warp 0)\n", pr[0][13] - pr[0][0]);
    {
        const char *sn[] = {"theta", "a table", "weights", "diag/A3/K-prep", "B (+GJ)", "C", "K"};
        int ids[] = {20, 24, 25, 26, 27, 28, 29, 21};
        for (int q = 0; q < 7; ++q) printf("setup %-16s %7lld\n", sn[q], pr[0][ids[q + 1]] - pr[0][ids[q]]);
        printf("setup A3+GJ (warp 0)  %7lld  = DI0 %lld + A3 %lld + GJ %lld + store %lld\n", pr[0][30] - pr[0][26],
               pr[0][16] - pr[0][26], pr[0][17] - pr[0][16], pr[0][18] - pr[0][17], pr[0][30] - pr[0][18]);
        for (int w = 0; w < 4; ++w) printf("a-table loop (warp %d) %7lld\n", w, pr[w][19] - pr[w][24]);
        for (int w = 1; w < 4; ++w) printf("setup diag (warp %d)   %7lld\n", w, pr[w][31] - pr[w][26]);
    }
    printf("sample 0 of CTA 0: setup %lld cycles, CG %lld cycles for %lld iterations\n",
           pr[0][21] - pr[0][20], pr[0][22] - pr[0][21], pr[0][23]);
    usfft_finalize(ctx);
    return 0;
}
