// probe_gather4.cu -- does TMA tile::gather4 accept a 2D [N x 6] FP64 tensor
// with 48-B rows, and which shared-memory destination alignments work?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe_gather4 probe_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm, const int *rows, int off, double *out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *bar = (uint64_t *)sm;
    double *dst = (double *)(sm + 1024 + off);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(4 * 48));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
            "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(su32(bar))
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(
                su32(bar))
            : "memory");
        for (int i = 0; i < 24; ++i)
            out[i] = dst[i];
    }
}

int main(int argc, char **argv)
{
    const int N = 1000;
    std::vector<double> h(6 * N);
    for (int i = 0; i < 6 * N; ++i)
        h[i] = i;
    double *d, *o;
    int *r;
    cudaMalloc(&d, 8 * 6 * N);
    cudaMalloc(&o, 8 * 24);
    cudaMalloc(&r, 16);
    cudaMemcpy(d, h.data(), 8 * 6 * N, cudaMemcpyHostToDevice);
    int rows[4] = {5, 917, 2, 33};
    cudaMemcpy(r, rows, 16, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    CUtensorMap tm;
    cuuint64_t dims[2] = {6, (cuuint64_t)N};
    cuuint64_t strides[1] = {48};
    cuuint32_t box[2] = {6, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)cr);
    for (int off : {atoi(argv[1])}) {
        cudaMemset(o, 0, 8 * 24);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096);
        k<<<1, 32, 4096>>>(tm, r, off, o);
        cudaError_t e = cudaDeviceSynchronize();
        double ho[24];
        cudaMemcpy(ho, o, 8 * 24, cudaMemcpyDeviceToHost);
        bool ok = e == cudaSuccess;
        for (int g = 0; g < 4 && ok; ++g)
            for (int c = 0; c < 6; ++c)
                ok &= ho[6 * g + c] == 6.0 * rows[g] + c;
        printf("dst offset %3d: %s (%s)\n", off, ok ? "OK" : "WRONG", cudaGetErrorString(e));
        if (e != cudaSuccess)
            return 0;
    }
    return 0;
}
