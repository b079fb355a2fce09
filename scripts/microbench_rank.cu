// microbench_rank.cu — warp multisplit ranking on sm_100a: lanes holding equal digits found by
// one ballot per digit bit (the sort's digit_peers) vs __match_any_sync (MATCH.ANY), for 7- and
// 8-bit digits drawn uniformly (a radix pass's typical warp: ~32 distinct digits) and from a
// narrow set (few distinct digits).  Prints rank operations per second per method.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbr scripts/microbench_rank.cu && /tmp/mbr
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <int NB>
__device__ __forceinline__ unsigned peers_ballot(uint32_t d) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

template <int METHOD, int NB>
__global__ void k_rank(int iters, uint32_t dmask, uint32_t* out) {
    const unsigned lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        s = s * 1664525u + 1013904223u;
        const uint32_t d = (s >> 8) & dmask;
        const unsigned p = METHOD == 0 ? peers_ballot<NB>(d) : __match_any_sync(0xffffffffu, d);
        acc += __popc(p & lt) + (lane == (unsigned)(__ffs(p) - 1));
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int METHOD, int NB>
double run(uint32_t dmask, uint32_t* out) {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_rank<METHOD, NB><<<blocks, threads>>>(16, dmask, out);
    cudaEventRecord(a);
    k_rank<METHOD, NB><<<blocks, threads>>>(iters, dmask, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return (double)blocks * threads * iters / (ms * 1e-3);
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 4);
    printf("{\"ranks_per_s\": {");
    printf("\"ballot7_uniform\": %.4g, ", run<0, 7>(127u, out));
    printf("\"ballot8_uniform\": %.4g, ", run<0, 8>(255u, out));
    printf("\"match_7bit_uniform\": %.4g, ", run<1, 7>(127u, out));
    printf("\"match_8bit_uniform\": %.4g, ", run<1, 8>(255u, out));
    printf("\"ballot8_4distinct\": %.4g, ", run<0, 8>(3u, out));
    printf("\"match_4distinct\": %.4g", run<1, 8>(3u, out));
    printf("}}\n");
    return 0;
}
