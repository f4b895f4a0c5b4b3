// FP64 pipe throughput probe on one B200 (tools/probe_fp64.cu):
// DFMA / DMUL / DADD streams with C independent chains per thread, grids of
// B CTAs x T threads, launches of ~ms_target; best of 10.  Prints per-SM
// lanes/clk (FMA counted once) against the nominal 64 DFMA/clk/SM, at the
// SM clock measured in-kernel (clock64 / globaltimer of block 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_fp64 tools/probe_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C, int OP>
__global__ void probe(double *out, int iters, double a, double b, long long *clk)
{
    long long c0 = 0, t0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    }
    double c[C];
#pragma unroll
    for (int i = 0; i < C; ++i)
        c[i] = (double)(threadIdx.x + i) * 1e-3;
    // keep a, b in registers (no constant-bank operands)
    double ra, rb;
    asm volatile("mov.f64 %0, %1;" : "=d"(ra) : "d"(a));
    asm volatile("mov.f64 %0, %1;" : "=d"(rb) : "d"(b));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 128 / C; ++r)
#pragma unroll
            for (int i = 0; i < C; ++i) {
                if (OP == 0)
                    c[i] = fma(c[i], ra, rb);
                else if (OP == 1)
                    c[i] = c[i] * ra;
                else
                    c[i] = c[i] + rb;
            }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i)
        s += c[i];
    if (s == 1.2345)
        out[blockIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        clk[0] = clock64() - c0;
        clk[1] = t1 - t0;
    }
}

template <int C, int OP>
void run(const char *name, int blocks_per_sm, int threads, double ms_target, int nsm)
{
    double *out;
    long long *clk;
    cudaMalloc(&out, sizeof(double) * 65536);
    cudaMalloc(&clk, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = nsm * blocks_per_sm;
    int iters = 8;
    float ms = 0;
    for (int k = 0; k < 30; ++k) {
        cudaEventRecord(a);
        probe<C, OP><<<blocks, threads>>>(out, iters, 0.9999999, 1e-9, clk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (ms >= ms_target)
            break;
        iters = (int)(iters * (ms_target / (ms > 1e-3 ? ms : 1e-3)) * 1.05) + 1;
    }
    float best = 1e30f;
    long long bc[2] = {0, 1};
    for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(a);
        probe<C, OP><<<blocks, threads>>>(out, iters, 0.9999999, 1e-9, clk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) {
            best = ms;
            cudaMemcpy(bc, clk, 16, cudaMemcpyDeviceToHost);
        }
    }
    const double ops = 128.0 * iters * (double)blocks * threads;  // warp-lane instructions
    const double mhz = (double)bc[0] / (double)bc[1] * 1e3;
    const double per_sm_clk = ops / (best * 1e-3) / (mhz * 1e6) / nsm;
    printf("%-5s chains=%2d blocks/SM=%d threads=%4d  %7.3f ms  %6.0f MHz  %5.1f lanes/clk/SM  %6.2f TF/s%s\n", name, C,
           blocks_per_sm, threads, best, mhz, per_sm_clk, (OP == 0 ? 2.0 : 1.0) * ops / (best * 1e-3) / 1e12,
           OP == 0 ? " (FMA = 2)" : "");
    cudaFree(out);
    cudaFree(clk);
}

int main()
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int nsm = p.multiProcessorCount;
    printf("%s, %d SMs; nominal 64 DFMA lanes/clk/SM\n", p.name, nsm);
    run<8, 0>("DFMA", 8, 256, 0.5, nsm);
    run<8, 0>("DFMA", 8, 256, 5.0, nsm);
    run<16, 0>("DFMA", 8, 256, 5.0, nsm);
    run<32, 0>("DFMA", 4, 256, 5.0, nsm);
    run<16, 0>("DFMA", 2, 1024, 5.0, nsm);
    run<8, 0>("DFMA", 2, 1024, 5.0, nsm);
    run<4, 0>("DFMA", 2, 1024, 5.0, nsm);
    run<16, 0>("DFMA", 1, 512, 5.0, nsm);
    run<16, 0>("DFMA", 1, 256, 5.0, nsm);
    run<16, 0>("DFMA", 1, 128, 5.0, nsm);
    run<16, 0>("DFMA", 8, 256, 20.0, nsm);
    run<16, 1>("DMUL", 8, 256, 5.0, nsm);
    run<16, 2>("DADD", 8, 256, 5.0, nsm);
    return 0;
}
