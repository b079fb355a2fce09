// tma.cuh — TMA bulk-tensor staging of the pair render records (sm_100a).
//
// The compositing kernels stage each batch of list entries' 48-byte render records in shared
// memory (Alg. 2's batched fetch).  Here that fetch is a TMA "gather4": a 2-D tensor
// map views the record array as [cap_pairs rows × 12 floats] (48-byte row stride) with a
// 16-float box — columns 12–15 fall outside the tensor and are zero-filled — so one
// cp.async.bulk.tensor …tile::gather4 moves 4 arbitrary rows (the list's pair slots) into 256
// contiguous, 128-byte-aligned bytes of shared memory and signals an mbarrier with the bytes
// it wrote.  The copy engine does the gather; no thread registers hold records in flight, and
// the next batch lands while the current one is walked (double buffer).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace mvgs {

constexpr int TMA_ROW_FLOATS = 16;              // shared-memory row of one record (box width)
constexpr int TMA_ROW_BYTES = 4 * TMA_ROW_FLOATS;  // 64 B: a gather4 lands 256 B

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// one arrival that also announces `bytes` of asynchronous transactions for the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// rows r0..r3 of the record tensor → 4 × 64 B at dst (128-byte aligned); completes on bar
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int r0, int r1, int r2,
                                            int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
#endif

// Host: encode the record tensor map (driver entry point fetched through the runtime, so the
// library needs no -lcuda).  Returns false when the driver refuses it (the kernels then stage
// with per-thread loads).
bool encode_record_map(CUtensorMap* tm, const void* rec, int64_t cap_pairs);

}  // namespace mvgs
