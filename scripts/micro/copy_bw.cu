// HBM copy bandwidth on this B200 for the stencil's traffic mix (read 3
// fields, write 3 fields, 50/50): cudaMemcpy D2D and a float4 grid-stride
// copy of 3 x 1.07 GB, CUDA events, best of 10.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void copy3(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                      float4* __restrict__ x, float4* __restrict__ y, float4* __restrict__ z, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        x[i] = a[i]; y[i] = b[i]; z[i] = c[i];
    }
}
int main() {
    const long cells = 16386L * 16416L;            // one padded 16384^2 field
    const size_t bytes = cells * 4;
    float *in[3], *out[3];
    for (int f = 0; f < 3; ++f) { cudaMalloc(&in[f], bytes); cudaMalloc(&out[f], bytes); cudaMemset(in[f], 0, bytes); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9, ms;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        for (int f = 0; f < 3; ++f) cudaMemcpyAsync(out[f], in[f], bytes, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("cudaMemcpy D2D x3: %.3f ms  %.1f GB/s (read+write)\n", best, 6.0 * bytes / best / 1e6);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0);
            copy3<<<blocks, 256>>>((float4*)in[0], (float4*)in[1], (float4*)in[2], (float4*)out[0], (float4*)out[1],
                                   (float4*)out[2], cells / 4);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("float4 copy3 kernel, %d blocks: %.3f ms  %.1f GB/s (read+write)\n", blocks, best, 6.0 * bytes / best / 1e6);
    }
    return 0;
}
