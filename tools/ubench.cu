// ubench.cu — latency / throughput probes on the B200 used to size the PCG design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double *out, long long *cyc, int n) {
    double a = out[0], b = out[1], c = out[2];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    out[3] = a;
    cyc[0] = t1 - t0;
}

__global__ void lat_dadd(double *out, long long *cyc, int n) {
    double a = out[0], b = out[1];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = a + b;
    long long t1 = clock64();
    out[3] = a;
    cyc[0] = t1 - t0;
}

__global__ void lat_shfl(double *out, long long *cyc, int n) {
    double a = out[threadIdx.x & 3];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
    long long t1 = clock64();
    out[4 + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_lds(double *out, long long *cyc, int n) {
    __shared__ int idx[64];
    if (threadIdx.x < 64) idx[threadIdx.x] = (threadIdx.x + 1) & 63;
    __syncthreads();
    int j = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) j = idx[j];
    long long t1 = clock64();
    out[5] = j;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_rcp(double *out, long long *cyc, int n) {
    double a = out[0] + 1.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double y;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
        a = y + 1.0;
    }
    long long t1 = clock64();
    out[3] = a;
    cyc[0] = t1 - t0;
}

__global__ void lat_bar(double *out, long long *cyc, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// DFMA throughput: 8 independent chains per thread, full SM occupancy
__global__ void thr_dfma(double *out, int n) {
    double a[8];
    for (int k = 0; k < 8; ++k) a[k] = out[k] + threadIdx.x;
    const double b = out[8], c = out[9];
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) out[10] = s;
}

int main() {
    double *d;
    long long *c;
    cudaMalloc(&d, 4096);
    cudaMalloc(&c, 64);
    double h[16] = {1.0000001, 0.9999999, 1e-9, 0, 0, 0, 0, 0, 0.999999, 1e-9};
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    const int n = 4096;
    long long cy;
    auto rep = [&](const char *name, int ops) {
        cudaDeviceSynchronize();
        cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %.2f cycles/op\n", name, (double)cy / ops);
    };
    lat_dfma<<<1, 1>>>(d, c, n);  rep("DFMA dependent latency", n);
    lat_dadd<<<1, 1>>>(d, c, n);  rep("DADD dependent latency", n);
    lat_shfl<<<1, 32>>>(d, c, n); rep("SHFL.f64 + DADD latency", n);
    lat_lds<<<1, 32>>>(d, c, n);  rep("LDS (pointer chase)", n);
    lat_rcp<<<1, 1>>>(d, c, n);   rep("MUFU.RCP64H + DADD", n);
    lat_bar<<<1, 128>>>(d, c, n); rep("bar.sync (4 warps)", n);
    lat_bar<<<1, 512>>>(d, c, n); rep("bar.sync (16 warps)", n);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int it = 20000;
    thr_dfma<<<sms * 4, 512>>>(d, 100);
    cudaEventRecord(e0);
    thr_dfma<<<sms * 4, 512>>>(d, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * it * (double)sms * 4 * 512;
    printf("DFMA throughput: %.2f TFLOP/s (%d SMs)\n", flops / (ms * 1e-3) / 1e12, sms);
    return 0;
}
