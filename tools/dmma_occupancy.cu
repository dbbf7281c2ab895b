// dmma_occupancy.cu -- DMMA (mma.sync m8n8k4 f64) throughput against warps per
// SM and independent accumulator chains per warp: where the FP64 tensor pipe
// saturates.  One CTA per SM with W warps; each warp runs C chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

template <int C>
__global__ void dmma_chains(double* out) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[C][2];
#pragma unroll
    for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

template <int C>
void run(int sms, double* d) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w : {2, 4, 8, 12, 16, 24, 32}) {
        dmma_chains<C><<<sms, 32 * w>>>(d);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) dmma_chains<C><<<sms, 32 * w>>>(d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 3.0 * sms * w * (double)ITERS * C * 512;
        printf("{\"chains\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", C, w, fl / (ms * 1e-3) / 1e12);
    }
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(sms, d);
    run<2>(sms, d);
    run<4>(sms, d);
    run<8>(sms, d);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
