// Dependent-chain latencies on this GPU (one warp): DFMA, DMUL, double
// division, rcp-approx, integer add, shuffle, shared load, named barrier.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[64];
    __shared__ int si[64];
    sm[threadIdx.x] = a + threadIdx.x;
    si[threadIdx.x] = (threadIdx.x + 1) & 31;
    __syncthreads();
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) y = y * b;
    long long t2 = clock64();
    double z = a + 1.0;
    for (int i = 0; i < n; ++i) z = b / z;
    long long t3 = clock64();
    double w = a;
    for (int i = 0; i < n; ++i) w = __shfl_sync(0xffffffffu, w, (threadIdx.x + 1) & 31);
    long long t4 = clock64();
    int q = threadIdx.x;
    for (int i = 0; i < n; ++i) q = si[q];
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 64;");
    long long t6 = clock64();
    float f = (float)a;
    for (int i = 0; i < n; ++i) f = fmaf(f, (float)b, (float)a);
    long long t7 = clock64();
    out[threadIdx.x] = x + y + z + w + q + f;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
        cyc[6] = t7 - t6;
    }
}

int main() {
    double* d; long long* c; long long h[8];
    cudaMalloc(&d, 64 * 8); cudaMalloc(&c, 8 * 8);
    const int n = 1000;
    for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 64>>>(d, c, 0.5, 0.999, n);
    cudaMemcpy(h, c, 7 * 8, cudaMemcpyDeviceToHost);
    const char* nm[] = {"DFMA", "DMUL", "ddiv", "SHFL(double)", "LDS (int chase)", "bar.sync 2 warps", "FFMA"};
    for (int i = 0; i < 7; ++i) printf("%-20s %.1f cycles\n", nm[i], (double)h[i] / n);
    return 0;
}
