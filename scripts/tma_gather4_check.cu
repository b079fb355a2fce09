// tma_gather4_check.cu — does a 2-D tensor map over the 48-byte pair records (12 floats per row)
// with a 16-float box (columns 12–15 out of bounds → zero fill) gather 4 arbitrary rows into
// 256 contiguous bytes of shared memory?  (the staging the compositing kernels use)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 scripts/tma_gather4_check.cu && /tmp/g4
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap tm, const int* rows, float* out) {
    __shared__ __align__(128) float buf[4 * 16];
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(4 * 64) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(sb), "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(mb) : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(mb), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
    const int n = 1000;
    float* rec;
    cudaMalloc(&rec, n * 48);
    float h[n * 12];
    for (int i = 0; i < n * 12; i++) h[i] = (float)i;
    cudaMemcpy(rec, h, sizeof h, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {12, (cuuint64_t)n};
    cuuint64_t strides[1] = {48};
    cuuint32_t box[2] = {16, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, rec, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode(box 16 over dim 12) = %d\n", (int)r);
    int hr[4] = {7, 3, 999, 500};
    int* rows;
    cudaMalloc(&rows, 16);
    cudaMemcpy(rows, hr, 16, cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, 64 * 4);
    k<<<1, 32>>>(tm, rows, out);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[64];
    cudaMemcpy(ho, out, sizeof ho, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int g = 0; g < 4; g++)
        for (int c = 0; c < 16; c++) {
            float want = c < 12 ? (float)(hr[g] * 12 + c) : 0.f;
            if (ho[g * 16 + c] != want) bad++;
        }
    printf("kernel: %s, mismatches %d (row 0: %g %g ... %g %g)\n", cudaGetErrorString(e), bad, ho[0], ho[1], ho[11], ho[12]);
    return bad || e != cudaSuccess || r != CUDA_SUCCESS;
}
