// k_sort.cu — S4: "sorting Gaussians by depth for each tile" with views kept
// apart.  The (view, tile) part of the paper's 64-bit key is the
// bucket index (S3 already separated the entries), so each bucket only needs
// its 32-bit depth keys ordered, ties by Gaussian id (R10).
//
// One CTA per (view, tile) bucket runs an LSD radix sort (4 passes × 8 bits,
// passes whose digit is constant over the bucket are skipped).  Each pass is
// stable: a warp owns a contiguous strip of 32·IPT positions, ranks its keys
// with __match_any_sync in position order, and the CTA turns per-warp digit
// counts into scatter offsets.  Buckets up to TILE_N keys are sorted entirely in
// shared memory; larger ones stream tiles of TILE_N through global scratch
// (key2/val2) with the same code and a running per-digit base.
//
// Ties: equal depth bits are ordered by pair index, which for one view is the
// ascending-gid order (pairs are view-major, gid-ascending).  Equal keys are
// rare; runs are fixed by an insertion sort started from each run head.
#include "internal.cuh"

namespace mvgs {

constexpr unsigned FULLM = 0xffffffffu;
constexpr int SORT_T = 256, SORT_IPT = 8, TILE_N = SORT_T * SORT_IPT, NW = SORT_T / 32;

struct SortSmem {
    uint32_t hist[NW][256];
    uint32_t base[256];
    uint32_t ws[NW + 1];
    uint32_t diff;
    int anytie;
};

__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t x, uint32_t* ws, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULLM, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int w = 0; w < NW; w++) {
            uint32_t t = ws[w];
            ws[w] = run;
            run += t;
        }
        ws[NW] = run;
    }
    __syncthreads();
    uint32_t r = ws[warp] + inc - x;
    *total = ws[NW];
    __syncthreads();
    return r;
}

// Stable LSD radix sort of (k, v)[0..n) → result back in (kA, vA).
// kA/vA/kB/vB may point to shared or global memory (generic addressing).
__device__ void bucket_radix_sort(uint32_t* kA, uint32_t* vA, uint32_t* kB, uint32_t* vB, int n, SortSmem& sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (tid == 0) {
        sm.diff = 0;
        sm.anytie = 0;
    }
    __syncthreads();
    {
        const uint32_t k0 = kA[0];
        uint32_t d = 0;
        for (int i = tid; i < n; i += SORT_T) d |= kA[i] ^ k0;
        d |= __shfl_xor_sync(FULLM, d, 16);
        d |= __shfl_xor_sync(FULLM, d, 8);
        d |= __shfl_xor_sync(FULLM, d, 4);
        d |= __shfl_xor_sync(FULLM, d, 2);
        d |= __shfl_xor_sync(FULLM, d, 1);
        if (lane == 0 && d) atomicOr(&sm.diff, d);
    }
    __syncthreads();
    const uint32_t diff = sm.diff;
    uint32_t *ks = kA, *vs = vA, *kd = kB, *vd = vB;
    for (int shift = 0; shift < 32; shift += 8) {
        if (((diff >> shift) & 255u) == 0) continue;
        // (1) digit histogram over the whole bucket → exclusive base per digit
        sm.base[tid] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += SORT_T) atomicAdd(&sm.base[(ks[i] >> shift) & 255u], 1u);
        __syncthreads();
        {
            uint32_t tot;
            const uint32_t c = sm.base[tid];
            const uint32_t ex = block_excl_scan_256(c, sm.ws, &tot);
            sm.base[tid] = ex;
        }
        __syncthreads();
        // (2) tiles in order, stable scatter
        for (int t0 = 0; t0 < n; t0 += TILE_N) {
            uint32_t key[SORT_IPT], val[SORT_IPT], loc[SORT_IPT];
#pragma unroll
            for (int i = 0; i < 8; i++) sm.hist[warp][lane * 8 + i] = 0;
            __syncwarp();
#pragma unroll
            for (int it = 0; it < SORT_IPT; it++) {
                const int p = t0 + warp * 32 * SORT_IPT + it * 32 + lane;
                const bool ok = p < n;
                key[it] = ok ? ks[p] : 0u;
                val[it] = ok ? vs[p] : 0u;
                const uint32_t d = ok ? ((key[it] >> shift) & 255u) : 256u;
                const unsigned peers = __match_any_sync(FULLM, d);
                const int leader = __ffs(peers) - 1;
                const uint32_t before = ok ? sm.hist[warp][d] : 0u;
                loc[it] = before + __popc(peers & lt);
                __syncwarp();
                if (ok && lane == leader) sm.hist[warp][d] = before + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            {  // per digit (thread tid = digit): warp offsets inside the tile + running base
                uint32_t run = sm.base[tid];
#pragma unroll
                for (int w = 0; w < NW; w++) {
                    const uint32_t c = sm.hist[w][tid];
                    sm.hist[w][tid] = run;
                    run += c;
                }
                sm.base[tid] = run;
            }
            __syncthreads();
#pragma unroll
            for (int it = 0; it < SORT_IPT; it++) {
                const int p = t0 + warp * 32 * SORT_IPT + it * 32 + lane;
                if (p < n) {
                    const uint32_t d = (key[it] >> shift) & 255u;
                    const uint32_t dst = sm.hist[warp][d] + loc[it];
                    kd[dst] = key[it];
                    vd[dst] = val[it];
                }
            }
            __syncthreads();
        }
        uint32_t* t = ks; ks = kd; kd = t;
        t = vs; vs = vd; vd = t;
    }
    if (ks != kA) {
        for (int i = tid; i < n; i += SORT_T) {
            kA[i] = ks[i];
            vA[i] = vs[i];
        }
        __syncthreads();
    }
    // ties: equal depth bits ordered by pair index (= gid within the view)
    bool tie = false;
    for (int i = tid + 1; i < n; i += SORT_T) tie |= (kA[i] == kA[i - 1]);
    if (__syncthreads_or(tie)) {
        for (int i = tid; i < n; i += SORT_T) {
            const bool head = (i == 0 || kA[i] != kA[i - 1]) && (i + 1 < n && kA[i + 1] == kA[i]);
            if (!head) continue;
            int e = i + 1;
            while (e < n && kA[e] == kA[i]) e++;
            for (int a = i + 1; a < e; a++) {  // insertion sort of vA[i..e)
                const uint32_t x = vA[a];
                int b = a - 1;
                while (b >= i && vA[b] > x) {
                    vA[b + 1] = vA[b];
                    b--;
                }
                vA[b + 1] = x;
            }
        }
        __syncthreads();
    }
}

__global__ __launch_bounds__(SORT_T) void k_bucket_sort(Launch L) {
    __shared__ SortSmem sm;
    __shared__ uint32_t sk[2][TILE_N], sv[2][TILE_N];
    const int64_t b = blockIdx.x;
    const int64_t s = L.bucket_off[b], e = L.bucket_off[b + 1];
    const int n = (int)(e - s);
    if (threadIdx.x == 0 && n > 0) atomicMax(&L.counters[C_MAXB], n);
    if (n <= 1 || e > L.cap_entries) return;
    uint32_t* gk = L.key + s;
    uint32_t* gv = L.val + s;
    if (n <= TILE_N) {
        for (int i = threadIdx.x; i < n; i += SORT_T) {
            sk[0][i] = gk[i];
            sv[0][i] = gv[i];
        }
        __syncthreads();
        bucket_radix_sort(sk[0], sv[0], sk[1], sv[1], n, sm);
        for (int i = threadIdx.x; i < n; i += SORT_T) gv[i] = sv[0][i];
    } else {
        bucket_radix_sort(gk, gv, L.key2 + s, L.val2 + s, n, sm);
    }
}

cudaError_t launch_bucket_sort(const Launch& L, cudaStream_t s) {
    k_bucket_sort<<<L.V * L.T, SORT_T, 0, s>>>(L);
    return cudaGetLastError();
}

}  // namespace mvgs
