// FP64 throughput probe: DMMA (mma.sync m8n8k4 f64) vs DFMA on sm_100a.
// Records the FP64 roofline denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CHAINS][2];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("device %s sms %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
    double* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int threads : {128, 256, 512}) {
      for (int bps : {1, 2, 4}) {
        int blocks = p.multiProcessorCount * bps;
        dmma_loop<8><<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<8><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
        printf("DMMA m8n8k4 threads %d blocks %d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
        dfma_loop<8><<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<8><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * (double)iters * threads * blocks;
        printf("DFMA threads %d blocks %d: %.2f TFLOP/s\n", threads, blocks, flops / ms / 1e9);
      }
    }
    cudaError_t err = cudaGetLastError();
    printf("err %s\n", cudaGetErrorString(err));
    return 0;
}
