// FP64 throughput ceilings on this GPU: DMMA.8x8x4 (mma.sync m8n8k4 f64) and DFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double *out, int iters) {
    double d[8][2];
    for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(double *out, int iters) {
    double d[8];
    for (int j = 0; j < 8; ++j) d[j] = threadIdx.x * 1e-9 * j;
    const double a = 1.0 - 1e-12, b = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = fma(d[j], a, b);
    }
    double s = 0.0;
    for (int j = 0; j < 8; ++j) s += d[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 20000, threads = 32 * warps;
        dmma_loop<<<sms, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<<<sms, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop = 2.0 * 256 * 8 * (double)iters * warps * sms;
        printf("DMMA.8x8x4  warps/SM %2d: %.2f TFLOP/s\n", warps, flop / (ms * 1e-3) / 1e12);
        dfma_loop<<<sms, threads>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<<<sms, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop2 = 2.0 * 8 * (double)iters * threads * sms;
        printf("DFMA        warps/SM %2d: %.2f TFLOP/s\n", warps, flop2 / (ms * 1e-3) / 1e12);
    }
    return 0;
}
