// Dependent-issue latency probe (cycles per op) for the FP64 ops of the
// element kernel: DFMA, DADD, DMUL, MUFU.RSQ64H, F2F f64<->f32, LDS.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_latency.cu -o tools/probe_latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, double a, double b, int n)
{
    __shared__ double sh[256];
    sh[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x = a + threadIdx.x;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            x = fma(x, a, b);
    }
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            x = x + b;
    }
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            x = x * a;
    }
    t1 = clock64();
    cyc[2] = t1 - t0;
    // MUFU.RSQ64H chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            double y;
            asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
            x = y;
        }
    }
    t1 = clock64();
    cyc[3] = t1 - t0;
    // F2F round trip chain (f64 -> f32 -> f64)
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            x = (double)(float)x + 1.0;
    }
    t1 = clock64();
    cyc[4] = t1 - t0;
    // LDS chain (address depends on the loaded value)
    int j = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            j = ((int)sh[j & 255] + 1) & 255;
    }
    t1 = clock64();
    cyc[5] = t1 - t0;
    out[threadIdx.x] = x + j;
}

int main()
{
    double *out;
    long long *cyc, h[6];
    cudaMalloc(&out, 256 * sizeof(double));
    cudaMalloc(&cyc, 6 * sizeof(long long));
    const int n = 1000;
    lat<<<1, 1>>>(out, cyc, 1.0000001, 1e-9, n);
    lat<<<1, 1>>>(out, cyc, 1.0000001, 1e-9, n);
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const char *names[] = {"DFMA", "DADD", "DMUL", "MUFU.RSQ64H", "F2F.F32.F64+F2F.F64.F32+DADD", "LDS+F2I+IADD"};
    printf("{");
    for (int i = 0; i < 6; ++i)
        printf("%s\"%s\": %.2f", i ? ", " : "", names[i], (double)h[i] / (16.0 * n));
    printf("}\n");
    return 0;
}
