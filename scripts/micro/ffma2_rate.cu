// Microbenchmark: issue/throughput of FFMA2 (fma.rn.f32x2) vs FFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 0.001f + j;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = make_float2(threadIdx.x * 0.001f + j, j * 0.5f);
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __ffma2_rn(x[j], A, B);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: FFMA2 interleaved with integer ops (does FFMA2 free issue slots?)
__global__ void k_ffma2_int(float* out, float a, float b, int* io) {
    float2 x[8];
    int y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { x[j] = make_float2(threadIdx.x * 0.001f + j, j * 0.5f); y[j] = threadIdx.x + j; }
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { x[j] = __ffma2_rn(x[j], A, B); y[j] = (y[j] ^ 0x5a5a) + j; }
    }
    float s = 0; int t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { s += x[j].x + x[j].y; t ^= y[j]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    io[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma_int(float* out, float a, float b, int* io) {
    float x[8];
    int y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x * 0.001f + j; y[j] = threadIdx.x + j; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { x[j] = fmaf(x[j], a, b); y[j] = (y[j] ^ 0x5a5a) + j; }
    }
    float s = 0; int t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { s += x[j]; t ^= y[j]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    io[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float* out; int* io;
    const int blocks = 148 * 8, threads = 256;
    cudaMalloc(&out, blocks * threads * 4);
    cudaMalloc(&io, blocks * threads * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * blocks * threads * 8.0 * ITERS;
        printf("FFMA : %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2: %.3f ms  %.1f TFLOP/s\n", ms, 2 * fl / ms / 1e9);
        cudaEventRecord(e0); k_ffma2_int<<<blocks, threads>>>(out, 0.999f, 0.001f, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2+LOP/IADD: %.3f ms  %.1f TFLOP/s\n", ms, 2 * fl / ms / 1e9);
        cudaEventRecord(e0); k_ffma_int<<<blocks, threads>>>(out, 0.999f, 0.001f, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA+LOP/IADD: %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    }
    return 0;
}
