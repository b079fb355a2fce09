// microbench_alu.cu — measured ALU-side peaks of this B200.
// The denominators of the ALU-bound stages (render_fwd / render_bwd / dssim) are derived from unit
// counts unless measured; this program measures, full chip, with CUDA events:
//   FFMA (3-register form), FFMA2 (packed FP32x2), FADD2, FMUL2, MUFU.EX2, MUFU.RCP, SHFL.BFLY,
//   LDS.128 (conflict-free), global RED.ADD.F32 on distinct addresses and 8-way contended ones.
// Every kernel runs 148 × 8 CTAs of 256 threads, each thread an unrolled chain of independent
// operations (8 independent accumulators) so that issue, not latency, bounds it; results are
// written so the compiler keeps the work.  Output: one JSON object on stdout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_alu.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int NACC = 8;

__global__ void k_ffma(float* out, float a, float b) {
    float x[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) x[i] = __fmaf_rn(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    float2 x[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = make_float2(threadIdx.x + i, i);
    const float2 a2 = make_float2(a, b), b2 = make_float2(b, a);
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) x[i] = __ffma2_rn(x[i], a2, b2);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fadd2(float* out, float a, float b) {
    float2 x[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = make_float2(threadIdx.x + i, i);
    const float2 a2 = make_float2(a, b);
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) x[i] = __fadd2_rn(x[i], a2);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2(float* out, float a, float b) {
    float x[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = -(float)(threadIdx.x & 7) * 0.01f - i * 0.001f;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-x[i]));
            x[i] = y;  // ex2(−x) keeps x in [0.5, 1]
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_rcp(float* out, float a, float b) {
    float x[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = 1.5f + (threadIdx.x & 7) + i;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) {
            float y;
            asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
            x[i] = y + 1.0f;  // keeps x in [1, 2] and stops ptxas folding rcp(rcp(x))
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_shfl(float* out, float a, float b) {
    float x[NACC];
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 << (i & 3));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; i++) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds128(float* out, float a, float b) {
    __shared__ float4 sm[256 * 2];
    sm[threadIdx.x] = make_float4(a, b, a, b);
    sm[threadIdx.x + 256] = make_float4(b, a, b, a);
    __syncthreads();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int idx = threadIdx.x;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int i = 0; i < NACC; i++) {
            const float4 v = sm[(idx + i * 32) & 511];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        idx ^= 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// RED.ADD.F32 to global: `stride` apart lanes hit distinct words (contention 1) or share one of
// 32/8 addresses per warp (8-way contention), spread over a 16 MB region (L2-resident).
template <int CONT>
__global__ void k_red(float* buf, int mask) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < 256; it++) {
        const int w = (gt / 32 + it * 977) & mask;
        const int addr = w * 32 + (CONT == 1 ? lane : (lane / CONT) * CONT);
        atomicAdd(&buf[addr], 1.0f);
    }
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int grid = sms * 8, block = 256;
    float* out;
    cudaMalloc(&out, sizeof(float) * grid * block);
    float* red;
    const int red_words = 1 << 22;  // 16 MB
    cudaMalloc(&red, sizeof(float) * red_words);
    cudaMemset(red, 0, sizeof(float) * red_words);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double thr = (double)grid * block;
    const double warps = thr / 32.0;
    auto time = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        return best * 1e-3;
    };
    const double ops = thr * ITERS * NACC;  // per-thread operations
    double t;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %d", sms, clk / 1000);
    t = time([&] { k_ffma<<<grid, block>>>(out, 0.999f, 0.001f); });
    printf(", \"ffma_tflops\": %.2f", 2 * ops / t / 1e12);
    t = time([&] { k_ffma2<<<grid, block>>>(out, 0.999f, 0.001f); });
    printf(", \"ffma2_tflops\": %.2f", 4 * ops / t / 1e12);
    t = time([&] { k_fadd2<<<grid, block>>>(out, 0.001f, -0.001f); });
    printf(", \"fadd2_tflops\": %.2f", 2 * ops / t / 1e12);
    t = time([&] { k_ex2<<<grid, block>>>(out, 0.f, 0.f); });
    printf(", \"mufu_ex2_gops\": %.1f, \"mufu_ex2_per_sm_clk\": %.2f", ops / t / 1e9, ops / t / (sms * (clk * 1e3)));
    t = time([&] { k_rcp<<<grid, block>>>(out, 0.f, 0.f); });
    printf(", \"mufu_rcp_gops\": %.1f", ops / t / 1e9);
    t = time([&] { k_shfl<<<grid, block>>>(out, 0.f, 0.f); });
    printf(", \"shfl_warp_ginstr\": %.1f, \"shfl_warp_per_sm_clk\": %.3f", warps * ITERS * NACC / t / 1e9,
           warps * ITERS * NACC / t / (sms * (clk * 1e3)));
    t = time([&] { k_lds128<<<grid, block>>>(out, 1.f, 2.f); });
    printf(", \"lds128_warp_ginstr\": %.1f, \"lds128_tbs\": %.1f", warps * ITERS * NACC / t / 1e9,
           thr * ITERS * NACC * 16.0 / t / 1e12);
    const double nred = thr * 256;
    t = time([&] { k_red<1><<<grid, block>>>(red, red_words / 32 - 1); });
    printf(", \"red_f32_distinct_gops\": %.1f", nred / t / 1e9);
    t = time([&] { k_red<8><<<grid, block>>>(red, red_words / 32 - 1); });
    printf(", \"red_f32_8way_gops\": %.1f", nred / t / 1e9);
    printf("}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
