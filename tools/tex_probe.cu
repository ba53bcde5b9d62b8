// Is the texture path a second lookup pipe beside shared memory?  Same grid
// as shfl_probe (148 x 2 CTAs of 512 threads, 4 independent chains per
// thread, per-lane random 12-bit indices into a 16 KB table): (a) LDS only,
// (b) LDS + one tex1Dfetch per LDS (table in global memory, texture object),
// (c) tex1Dfetch only, (d) LDG (read-only path) only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tex_probe tools/tex_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool TEX, bool LDS, bool LDG>
__global__ void k_probe(cudaTextureObject_t t, const unsigned *__restrict__ g, unsigned *out, int n) {
    __shared__ unsigned tab[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    unsigned x[4], a[4], r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        x[k] = (threadIdx.x * 977u + k * 131u + blockIdx.x) * 2654435761u;
        a[k] = 0;
        r[k] = 0;
    }
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[k] = x[k] * 1664525u + 1013904223u;
            if (LDS) a[k] += tab[x[k] >> 20];
            if (TEX) r[k] += tex1Dfetch<unsigned>(t, (int)((x[k] >> 8) & 4095u));
            if (LDG) r[k] += __ldg(g + ((x[k] >> 8) & 4095u));
        }
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += a[k] + r[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <bool T, bool L, bool G>
float run(cudaTextureObject_t t, const unsigned *g, unsigned *out, int n) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_probe<T, L, G><<<296, 512>>>(t, g, out, n);
    cudaEventRecord(a);
    k_probe<T, L, G><<<296, 512>>>(t, g, out, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    unsigned *out, *g;
    cudaMalloc(&out, 296 * 512 * 4);
    cudaMalloc(&g, 4096 * 4);
    cudaMemset(g, 1, 4096 * 4);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned>();
    rd.res.linear.sizeInBytes = 4096 * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t;
    cudaCreateTextureObject(&t, &rd, &td, nullptr);
    const int n = 1 << 12;
    const double ops = 296.0 * 512 / 32 * n * 4;
    const double clk = 1.965e9 * 148;
    float ms;
    ms = run<false, true, false>(t, g, out, n);
    printf("lds only    %.3f ms  %.3f warp-ops/clk/SM\n", ms, ops / (ms * 1e-3 * clk));
    ms = run<true, true, false>(t, g, out, n);
    printf("lds + tex   %.3f ms  %.3f\n", ms, ops / (ms * 1e-3 * clk));
    ms = run<true, false, false>(t, g, out, n);
    printf("tex only    %.3f ms  %.3f\n", ms, ops / (ms * 1e-3 * clk));
    ms = run<false, true, true>(t, g, out, n);
    printf("lds + ldg   %.3f ms  %.3f\n", ms, ops / (ms * 1e-3 * clk));
    ms = run<false, false, true>(t, g, out, n);
    printf("ldg only    %.3f ms  %.3f\n", ms, ops / (ms * 1e-3 * clk));
    return 0;
}
