// k_bucket.cu — S3–S5 as a bucket sort: every (view, tile) list in (depth, gid) order
// without a global sort.
//
//   k_bucket_count    pairs → per-(view, tile) entry counts.  Each CTA takes a contiguous
//                     chunk of pair slots (view-major), flattens the tiles of 32 pairs at a
//                     time across a warp (as the duplication of S3) and counts them
//                     in a shared-memory histogram over the chunk's views, flushed with one
//                     global atomic per touched bucket.
//   scan              bucket counts → bucket_off (the S5 ranges) and K.
//   k_bucket_scatter  the same traversal: the CTA reserves a run in every touched bucket
//                     (one global atomic per bucket) and places each entry in its run with a
//                     shared-memory atomic, as a 64-bit key (depth bits << 32 | pair index).
//   k_bucket_sort     one CTA per bucket sorts its keys in shared memory (bitonic network,
//                     virtual +∞ padding to a power of two) and writes the pair indices.
// The 64-bit key orders by depth and then by pair index, and pair indices increase with the
// Gaussian id inside a view, so each list is in the oracle's (view, tile, depth_bits, gid)
// order (R15) exactly, whatever order the atomics placed the entries in.
#include "ca.cuh"
#include "internal.cuh"

namespace mvgs {

constexpr int BK_T = 256;              // threads per CTA (count / scatter / sort)
constexpr int BK_BINS = 16384;         // shared-memory histogram bins (64 KB)
constexpr int BK_SORT_CAP = 8192;      // keys sorted in shared memory (64 KB); larger buckets: in global
constexpr unsigned FULLB = 0xffffffffu;

__device__ __forceinline__ int bk_view_of_pair(const Launch& L, int64_t q) {
    int lo = 0, hi = L.V - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((int64_t)L.blk_off[(int64_t)mid * L.NB] <= q) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

struct BkDesc {  // one pair of a warp's 32
    int x0, y0, w, excl;
    float inv_w;
    int v;
    uint32_t depth, q;
};

struct BkSmem {
    int bins[BK_BINS];
    int pref[BK_T / 32][32];
    BkDesc desc[BK_T / 32][32];
};

// The CTA's chunk of pair slots [p0, p1) (equal split of Q over the grid, multiple of 32).
__device__ __forceinline__ void bk_chunk(const Launch& L, int64_t& p0, int64_t& p1) {
    const int64_t Q = min((int64_t)L.counters[C_Q], L.cap_pairs);
    int64_t ch = (Q + gridDim.x - 1) / gridDim.x;
    ch = (ch + 31) & ~(int64_t)31;
    p0 = min(Q, (int64_t)blockIdx.x * ch);
    p1 = min(Q, p0 + ch);
}

// Calls f(v, tile, depth, q) for every entry of the pairs in [p0, p1).  Warp w takes groups of
// 32 consecutive pairs; lane l handles entries l, l+32, … of the group's flattened tile list.
template <class F>
__device__ __forceinline__ void bk_for_entries(const Launch& L, BkSmem& sm, int64_t p0, int64_t p1, F f) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t g0 = p0 + (int64_t)wid * 32; g0 < p1; g0 += BK_T) {
        const int64_t i = g0 + lane;
        uint2 r = make_uint2(0u, 0u);
        uint32_t dk = 0xffffffffu;
        if (i < p1) {
            dk = L.pkey[i];
            r = L.prect[i];
        }
        const int rx0 = r.x & 0xffff, ry0 = r.x >> 16, rx1 = r.y & 0xffff, ry1 = r.y >> 16;
        const int w = rx1 - rx0;
        const int cnt = (dk != 0xffffffffu && rx1 > rx0 && ry1 > ry0) ? w * (ry1 - ry0) : 0;
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULLB, inc, o);
            if (lane >= o) inc += y;
        }
        const int total = __shfl_sync(FULLB, inc, 31);
        sm.pref[wid][lane] = inc;
        BkDesc d;
        d.x0 = rx0;
        d.y0 = ry0;
        d.w = w;
        d.excl = inc - cnt;
        d.inv_w = cnt > 0 ? 1.0f / (float)w : 0.f;
        d.v = cnt > 0 ? bk_view_of_pair(L, i) : 0;
        d.depth = dk;
        d.q = (uint32_t)i;
        sm.desc[wid][lane] = d;
        __syncwarp();
        for (int k = lane; k < total; k += 32) {
            int lo = 0;  // owner = number of lanes whose inclusive prefix is ≤ k
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (sm.pref[wid][lo + step - 1] <= k) lo += step;
            const BkDesc& o = sm.desc[wid][lo];
            const int loc = k - o.excl;
            const int row = __float2int_rz(((float)loc + 0.5f) * o.inv_w);  // exact (see k_dup)
            const int col = loc - row * o.w;
            f(o.v, (o.y0 + row) * L.TX + o.x0 + col, o.depth, o.q);
        }
        __syncwarp();
    }
}

__global__ __launch_bounds__(BK_T) void k_bucket_count(Launch L, int* __restrict__ gcnt) {
    extern __shared__ float4 bk_dyn[];
    BkSmem& sm = *reinterpret_cast<BkSmem*>(bk_dyn);
    int64_t p0, p1;
    bk_chunk(L, p0, p1);
    if (p0 >= p1) return;
    const int vf = bk_view_of_pair(L, p0), vl = bk_view_of_pair(L, p1 - 1);
    const int nb = (vl - vf + 1) * L.T;
    if (nb <= BK_BINS) {
        for (int b = threadIdx.x; b < nb; b += BK_T) sm.bins[b] = 0;
        __syncthreads();
        bk_for_entries(L, sm, p0, p1, [&](int v, int t, uint32_t, uint32_t) { atomicAdd(&sm.bins[(v - vf) * L.T + t], 1); });
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += BK_T)
            if (sm.bins[b]) atomicAdd(&gcnt[(int64_t)vf * L.T + b], sm.bins[b]);
    } else {
        bk_for_entries(L, sm, p0, p1, [&](int v, int t, uint32_t, uint32_t) { atomicAdd(&gcnt[(int64_t)v * L.T + t], 1); });
    }
}

__global__ __launch_bounds__(BK_T) void k_bucket_scatter(Launch L, int* __restrict__ gcur,
                                                         unsigned long long* __restrict__ ent) {
    extern __shared__ float4 bk_dyn[];
    BkSmem& sm = *reinterpret_cast<BkSmem*>(bk_dyn);
    int64_t p0, p1;
    bk_chunk(L, p0, p1);
    if (p0 >= p1) return;
    const int vf = bk_view_of_pair(L, p0), vl = bk_view_of_pair(L, p1 - 1);
    const int nb = (vl - vf + 1) * L.T;
    const int64_t cap = L.cap_entries;
    if (nb <= BK_BINS) {
        for (int b = threadIdx.x; b < nb; b += BK_T) sm.bins[b] = 0;
        __syncthreads();
        bk_for_entries(L, sm, p0, p1, [&](int v, int t, uint32_t, uint32_t) { atomicAdd(&sm.bins[(v - vf) * L.T + t], 1); });
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += BK_T) {  // reserve a run in every touched bucket
            const int c = sm.bins[b];
            if (c) {
                const int64_t gb = (int64_t)vf * L.T + b;
                sm.bins[b] = L.bucket_off[gb] + atomicAdd(&gcur[gb], c);
            }
        }
        __syncthreads();
        bk_for_entries(L, sm, p0, p1, [&](int v, int t, uint32_t depth, uint32_t q) {
            const int64_t pos = atomicAdd(&sm.bins[(v - vf) * L.T + t], 1);
            if (pos < cap) ent[pos] = ((unsigned long long)depth << 32) | q;
        });
    } else {
        bk_for_entries(L, sm, p0, p1, [&](int v, int t, uint32_t depth, uint32_t q) {
            const int64_t gb = (int64_t)v * L.T + t;
            const int64_t pos = (int64_t)L.bucket_off[gb] + atomicAdd(&gcur[gb], 1);
            if (pos < cap) ent[pos] = ((unsigned long long)depth << 32) | q;
        });
    }
}

// Bitonic sort of a[0, n) ascending, as the power-of-two network of size P2 ≥ n with
// a[n, P2) = +∞: every compare-exchange puts the minimum at the lower index ("flip" form),
// so the virtual +∞ never move and exchanges touching them are skipped.
template <class T>
__device__ __forceinline__ void bitonic_sort(T* a, int n) {
    int P2 = 1;
    while (P2 < n) P2 <<= 1;
    const int half_n = P2 >> 1;
    for (int k = 2; k <= P2; k <<= 1) {
        const int hk = k >> 1, lk = __ffs(k) - 1, lhk = lk - 1;
        for (int p = threadIdx.x; p < half_n; p += BK_T) {
            const int blk = p >> lhk, r = p & (hk - 1);
            const int i = (blk << lk) + r, j = (blk << lk) + k - 1 - r;
            if (j < n) {
                const T x = a[i], y = a[j];
                if (y < x) { a[i] = y; a[j] = x; }
            }
        }
        __syncthreads();
        for (int h = k >> 2; h > 0; h >>= 1) {
            const int lh = __ffs(h) - 1;
            for (int p = threadIdx.x; p < half_n; p += BK_T) {
                const int i = ((p >> lh) << (lh + 1)) + (p & (h - 1)), j = i + h;
                if (j < n) {
                    const T x = a[i], y = a[j];
                    if (y < x) { a[i] = y; a[j] = x; }
                }
            }
            __syncthreads();
        }
    }
}

__global__ __launch_bounds__(BK_T) void k_bucket_sort(Launch L, unsigned long long* __restrict__ ent,
                                                      uint32_t* __restrict__ sorted) {
    extern __shared__ float4 bk_dyn[];
    unsigned long long* s = reinterpret_cast<unsigned long long*>(bk_dyn);
    const int b = blockIdx.x;
    if (b == 0 && threadIdx.x == 0 && (int64_t)L.bucket_off[(int64_t)L.V * L.T] > L.cap_entries)
        L.counters[C_OVERFLOW] = 1;
    const int64_t lo = L.bucket_off[b], hi = L.bucket_off[b + 1];
    if (hi > L.cap_entries) return;  // overflowed: the renderer skips it as well
    const int n = (int)(hi - lo);
    if (n == 0) return;
    if (n == 1) {
        if (threadIdx.x == 0) sorted[lo] = (uint32_t)ent[lo];
        return;
    }
    if (n <= BK_SORT_CAP) {
        for (int i = threadIdx.x; i < n; i += BK_T) s[i] = ent[lo + i];
        __syncthreads();
        bitonic_sort(s, n);
        for (int i = threadIdx.x; i < n; i += BK_T) sorted[lo + i] = (uint32_t)s[i];
    } else {  // rare: sort the run in place in global memory (same network)
        bitonic_sort(ent + lo, n);
        for (int i = threadIdx.x; i < n; i += BK_T) sorted[lo + i] = (uint32_t)ent[lo + i];
    }
}

cudaError_t launch_bucket_count(const Launch& L, int* gcnt, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(k_bucket_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(BkSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BkSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(BK_SORT_CAP * sizeof(unsigned long long)));
    if (e != cudaSuccess) return e;
    const int64_t nbk = (int64_t)L.V * L.T;
    e = cudaMemsetAsync(gcnt, 0, sizeof(int) * (nbk + 1), s);
    if (e != cudaSuccess) return e;
    k_bucket_count<<<4 * 148, BK_T, sizeof(BkSmem), s>>>(L, gcnt);
    return cudaGetLastError();
}

cudaError_t launch_bucket_scatter(const Launch& L, int* gcur, unsigned long long* ent, cudaStream_t s) {
    const int64_t nbk = (int64_t)L.V * L.T;
    cudaError_t e = cudaMemsetAsync(gcur, 0, sizeof(int) * nbk, s);
    if (e != cudaSuccess) return e;
    k_bucket_scatter<<<4 * 148, BK_T, sizeof(BkSmem), s>>>(L, gcur, ent);
    return cudaGetLastError();
}

cudaError_t launch_bucket_sort(const Launch& L, unsigned long long* ent, uint32_t* sorted, cudaStream_t s) {
    const int64_t nbk = (int64_t)L.V * L.T;
    if (nbk > 0)
        k_bucket_sort<<<(unsigned)nbk, BK_T, BK_SORT_CAP * sizeof(unsigned long long), s>>>(L, ent, sorted);
    return cudaGetLastError();
}

}  // namespace mvgs
