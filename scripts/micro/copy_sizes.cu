// Copy ceiling per grid size: the stencil step's traffic (read 3 fields,
// write 3 fields of (n+2) x pitch f32) as a plain float4 copy, ping-ponging
// between two buffer sets like the time loop does, K launches captured in a
// CUDA graph (as scripts/grid_sweep.py times the step), best of 5 over
// grid-stride block counts.  The step kernel's fraction of THIS number says
// how close it is to what any kernel moving the same bytes achieves at that
// size (launch gaps, ramp-up and tail included).
//   ./copy_sizes [n ...]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void copy3(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                      float4* __restrict__ x, float4* __restrict__ y, float4* __restrict__ z, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        x[i] = a[i]; y[i] = b[i]; z[i] = c[i];
    }
}
int main(int argc, char** argv) {
    std::vector<long> ns;
    for (int i = 1; i < argc; ++i) ns.push_back(atol(argv[i]));
    if (ns.empty()) ns = {1024, 1448, 2048, 2896, 4096, 8192, 16384};
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (long n : ns) {
        const long pitch = (n + 2 + 31) / 32 * 32;
        const long cells = (n + 2) * pitch, v4 = cells / 4;
        const double bytes = 6.0 * 4.0 * (double)n * (double)n;      // algorithmic: 24 B per interior cell
        float* buf[6];
        for (auto& p : buf) { cudaMalloc(&p, cells * 4); cudaMemset(p, 0, cells * 4); }
        const int K = n >= 4096 ? 20 : 200;
        double best_gbs = 0; int best_blocks = 0; float best_ms = 0;
        for (int blocks : {148 * 2, 148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
            cudaGraph_t g; cudaGraphExec_t ge;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
            for (int k = 0; k < K; ++k) {
                float** s = (k & 1) ? buf + 3 : buf;
                float** d = (k & 1) ? buf : buf + 3;
                copy3<<<blocks, 256, 0, st>>>((float4*)s[0], (float4*)s[1], (float4*)s[2], (float4*)d[0],
                                              (float4*)d[1], (float4*)d[2], v4);
            }
            cudaStreamEndCapture(st, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, st);
            cudaStreamSynchronize(st);
            for (int r = 0; r < 5; ++r) {
                float ms;
                cudaEventRecord(e0, st);
                cudaGraphLaunch(ge, st);
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                const double gbs = bytes * K / (ms / 1e3) / 1e9;
                if (gbs > best_gbs) { best_gbs = gbs; best_blocks = blocks; best_ms = ms / K; }
            }
            cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
        }
        printf("{\"n\": %ld, \"copy_ms_per_pass\": %.5f, \"copy_gbs\": %.1f, \"copy_gcell_equiv\": %.2f, \"blocks\": %d}\n",
               n, best_ms, best_gbs, best_gbs / 24.0, best_blocks);
        fflush(stdout);
        for (auto p : buf) cudaFree(p);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
