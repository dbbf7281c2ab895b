// fp64_peak.cu — measured FP64 peaks on this B200: DFMA (CUDA cores) and DMMA
// (mma.sync m8n8k4 f64 tensor path).  MEASURED_PEAKS.json has no FP64 figure
// (SURVEY.md F8); this supplies the roofline denominator for the large-k
// phases.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) {
        const int blocks = sms * (2048 / threads);
        dfma_kernel<<<blocks, threads>>>(d, 0.999, 1e-3);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) dfma_kernel<<<blocks, threads>>>(d, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 5.0 * blocks * threads * (double)ITERS * 8 * 2;
        printf("{\"kind\": \"dfma\", \"threads\": %d, \"tflops\": %.2f}\n", threads, flops / (ms * 1e-3) / 1e12);
        dmma_kernel<<<blocks, threads>>>(d);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) dmma_kernel<<<blocks, threads>>>(d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double mflops = 5.0 * blocks * (threads / 32) * (double)ITERS * 8 * 256 * 2;
        printf("{\"kind\": \"dmma\", \"threads\": %d, \"tflops\": %.2f}\n", threads, mflops / (ms * 1e-3) / 1e12);
    }
    cudaError_t err = cudaGetLastError();
    printf("err %s\n", cudaGetErrorString(err));
    return 0;
}
