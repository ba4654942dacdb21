// Microbenchmark: latency of the dependent steps of the coarse substitution chain on this GPU
// (DFMA, DMUL, 64-bit SHFL, smem load), cycles per step via clock64.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double *out, long long *cyc, const double *L, int steps)
{
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = L[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double v = 1.0 + lane * 1e-3, a = 0.999, b = 1e-3;
    long long t0, t1;
    // 1) DFMA chain
    t0 = clock64();
    for (int i = 0; i < steps; ++i) v = fma(v, a, b);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / steps;
    // 2) shuffle chain (64-bit)
    t0 = clock64();
    for (int i = 0; i < steps; ++i) v = __shfl_sync(0xffffffffu, v, (i + 1) & 31) + b;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / steps;
    // 3) the substitution step: vc = shfl(vi * di, c); lane > c: vi -= L[c] * vc
    const double di = 0.5 + lane * 1e-4;
    t0 = clock64();
    for (int i = 0; i < steps; ++i) {
        const int c = i & 31;
        const double vc = __shfl_sync(0xffffffffu, v * di, c);
        if (lane == c) v = vc;
        if (lane > c) v -= s[(lane * 33 + c) & 1023] * vc;
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0) / steps;
    // 3b) unrolled block of 32 steps, L row in registers (what chol_solve_pipe does)
    {
        double Lr[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) Lr[c] = s[(lane * 33 + c) & 1023];
        t0 = clock64();
        for (int it = 0; it < steps / 32; ++it) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const double vc = __shfl_sync(0xffffffffu, v * di, c);
                v = (lane == c) ? vc : v;
                v = (lane > c) ? fma(-Lr[c], vc, v) : v;
            }
        }
        t1 = clock64();
        if (threadIdx.x == 0) cyc[4] = (t1 - t0) / steps;
    }
    // 4) smem dependent load chain
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < steps; ++i) idx = ((int)s[idx & 1023] + i) & 1023;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) / steps;
    out[threadIdx.x] = v + idx;
}

int main()
{
    double *out, *L;
    long long *cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&L, 1024 * 8);
    cudaMallocManaged(&cyc, 8 * 8);
    double h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = (i * 7) % 1024;
    cudaMemcpy(L, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int w : {32, 256}) {
        chain<<<1, w>>>(out, cyc, L, 4096);
        cudaDeviceSynchronize();
        printf("threads %d: dfma %lld  shfl64+dadd %lld  subst-step %lld  unrolled-step %lld  smem-dep-load %lld cycles/step\n", w, cyc[0],
               cyc[1], cyc[2], cyc[4], cyc[3]);
    }
    return 0;
}
