// Does SHFL share the shared-memory wavefront pipe?  Same grid (148 x 2 CTAs
// of 512 threads), 4 independent chains per thread, per-lane random addresses:
// (a) LDS only (random 12-bit indices, ~3.5 wavefronts each), (b) the same plus
// one SHFL per LDS, (c) SHFL only.  If t(b) ~ t(a) shuffles run beside the pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/shfl_probe_bin tools/shfl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool SHFL, bool LDS>
__global__ void k_probe(unsigned *out, int n) {
    __shared__ unsigned tab[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    unsigned x[4], a[4], r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        x[k] = (threadIdx.x * 977u + k * 131u + blockIdx.x) * 2654435761u;
        a[k] = 0;
        r[k] = x[k];
    }
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[k] = x[k] * 1664525u + 1013904223u;  // independent of the loads
            if (LDS) a[k] += tab[x[k] >> 20];
            if (SHFL) r[k] ^= __shfl_sync(0xffffffffu, x[k], x[k] >> 27);
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += a[k] + r[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <bool S, bool L>
float run(unsigned *out, int n) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_probe<S, L><<<296, 512>>>(out, n);
    cudaEventRecord(a);
    k_probe<S, L><<<296, 512>>>(out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    unsigned *out;
    cudaMalloc(&out, 296 * 512 * 4);
    const int n = 1 << 12;
    const double ops = 296.0 * 512 / 32 * n * 4;  // warp instructions of each kind
    const double clk = 1.965e9 * 148;
    float t;
    t = run<false, true>(out, n);
    printf("lds only    %.3f ms  %.3f warp-LDS/clk/SM\n", t, ops / (t * 1e-3 * clk));
    t = run<true, true>(out, n);
    printf("lds + shfl  %.3f ms  %.3f warp-LDS/clk/SM\n", t, ops / (t * 1e-3 * clk));
    t = run<true, false>(out, n);
    printf("shfl only   %.3f ms  %.3f warp-SHFL/clk/SM\n", t, ops / (t * 1e-3 * clk));
    return 0;
}
