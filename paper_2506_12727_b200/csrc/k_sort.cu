// k_sort.cu — S3 duplication + S4 sort.
//
// The paper keys every duplicated entry with (tile 16 | view 16 | depth 32)
// and sorts the 64-bit keys.  Here the same total order (view, tile, depth,
// gid) (R9, R10) is produced with two short stable LSD radix sorts and no
// atomics:
//   1. sort the pairs by depth bits (4 × 8-bit passes over Q pairs, Q ≪ K;
//      pairs with no tile carry key 0xffffffff and sort last); pairs start in
//      (view, gid) order and the sort is stable, so equal depths stay in gid
//      order; the last pass gathers each pair's packed tile rect;
//   2. duplicate: walk the pairs in that order and write one entry per covered
//      tile, key = view·T + tile (positions from an exclusive scan of the
//      per-pair tile counts — coalesced, deterministic);
//   3. stable sort the K entries by the bucket key only (⌈log2(V·T)⌉ bits,
//      8-bit digits).  Stability keeps each bucket in (depth, gid) order.
// Every pass is an "on-chip" radix pass: a CTA ranks a 2048-key tile in shared
// memory (warp multisplit by 8 ballots + per-warp digit counters, stable by
// position), digit×tile counts are scanned device-wide, and the tile scatters
// straight to its final positions.  Sizes (Q, K) live on the device; grids are
// sized by capacity and tiles beyond the live count exit.
#include "ca.cuh"
#include "internal.cuh"

namespace mvgs {

constexpr unsigned FULLS = 0xffffffffu;
constexpr int RS_T = 256, RS_IPT = 8, RS_TILE = RS_T * RS_IPT, RS_NW = RS_T / 32, RS_BINS = 256;

int radix_tiles(int64_t cap) { return (int)((cap + RS_TILE - 1) / RS_TILE); }
int64_t radix_counts_size(int64_t cap) { return (int64_t)RS_BINS * radix_tiles(cap) + 1; }


// exclusive scan over the 256 threads of a CTA (one value each)
__device__ __forceinline__ uint32_t block_excl_scan_256_u(uint32_t x, uint32_t* total) {
    __shared__ uint32_t wsum[RS_NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULLS, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < RS_NW; w++) {
        const uint32_t t = wsum[w];
        before += w < warp ? t : 0u;
        all += t;
    }
    *total = all;
    return before + inc - x;
}

// Warp multisplit ranking: lanes holding the same digit found with 8 ballots
// (one per digit bit) instead of __match_any_sync, whose cost grows with the
// number of distinct digits in the warp.
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool ok, int nbits) {
    unsigned peers = __ballot_sync(FULLS, ok);
#pragma unroll
    for (int b = 0; b < 8; b++) {
        if (b >= nbits) break;  // uniform: a 7-bit pass needs 7 ballots
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(FULLS, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

// per-tile digit histogram → counts[digit * ntiles + tile]
template <int IPT>
__global__ __launch_bounds__(RS_T) void k_rs_hist(const uint32_t* __restrict__ keys, const int* __restrict__ n_ptr,
                                                  int64_t cap, int shift, int nbits, int* __restrict__ counts,
                                                  int ntiles) {
    constexpr int TILE = RS_T * IPT;
    __shared__ int h[RS_BINS];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int n = (int)min((int64_t)*n_ptr, cap);
    const int t0 = blockIdx.x * TILE;
    const uint32_t mask = (1u << nbits) - 1u;
    for (int i = t0 + threadIdx.x; i < min(n, t0 + TILE); i += RS_T) atomicAdd(&h[(keys[i] >> shift) & mask], 1);
    __syncthreads();
    if (threadIdx.x <= mask) counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of one tile.  Ranks are computed per warp (multisplit), the
// tile is first re-ordered by digit in shared memory, then written out by
// consecutive threads: every digit's run lands contiguously at
// offsets[digit * ntiles + tile], so global writes are coalesced.
#ifndef MVGS_RS3_MINB
#define MVGS_RS3_MINB 6  // resident CTAs asked of the three-kernel scatter (6: 40 registers, 72 B spill; 1: 60 registers)
#endif
template <int IPT>
__global__ __launch_bounds__(RS_T, MVGS_RS3_MINB) void k_rs_scatter(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                     uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                     uint2* __restrict__ pout,
                                                     const int* __restrict__ n_ptr, int64_t cap, int shift, int nbits,
                                                     const int* __restrict__ offs, int ntiles,
                                                     int* __restrict__ range_min, const uint2* __restrict__ gather_pl,
                                                     int* __restrict__ cnt_out) {
    constexpr int TILE = RS_T * IPT;
    __shared__ uint32_t hist[RS_NW][RS_BINS];
    __shared__ uint32_t gdelta[RS_BINS];   // global offset − local start, per digit
    __shared__ uint32_t sk[TILE], sv[TILE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int n = (int)min((int64_t)*n_ptr, cap);
    const int t0 = blockIdx.x * TILE;
    if (t0 >= n) return;
    const int nt = min(TILE, n - t0);
    const uint32_t mask = (1u << nbits) - 1u;
    // this tile's scanned offset of digit threadIdx.x: independent of the keys, loaded up front
    const uint32_t goff = threadIdx.x <= mask ? (uint32_t)offs[(int64_t)threadIdx.x * ntiles + blockIdx.x] : 0u;
#pragma unroll
    for (int i = 0; i < RS_BINS / 32; i++) hist[warp][lane + 32 * i] = 0;
    __syncwarp();
    uint32_t key[IPT], val[IPT], loc[IPT];
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int p = warp * 32 * IPT + it * 32 + lane;
        const bool ok = p < nt;
        key[it] = ok ? kin[t0 + p] : 0u;
        val[it] = ok ? (vin ? vin[t0 + p] : (uint32_t)(t0 + p)) : 0u;  // no vin: values are the positions
    }
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int p = warp * 32 * IPT + it * 32 + lane;
        const bool ok = p < nt;
        const uint32_t d = (key[it] >> shift) & mask;
        const unsigned peers = digit_peers(d, ok, nbits);
        const uint32_t before = ok ? hist[warp][d] : 0u;
        loc[it] = before + __popc(peers & lt);
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) hist[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {  // thread = digit: tile-local digit starts and warp bases
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < RS_NW; w++) tot += hist[w][threadIdx.x];
        uint32_t ws;
        const uint32_t start = block_excl_scan_256_u(tot, &ws);
        gdelta[threadIdx.x] = goff - start;
        uint32_t run = start;
#pragma unroll
        for (int w = 0; w < RS_NW; w++) {
            const uint32_t c = hist[w][threadIdx.x];
            hist[w][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int p = warp * 32 * IPT + it * 32 + lane;
        if (p < nt) {
            const uint32_t l = hist[warp][(key[it] >> shift) & mask] + loc[it];
            sk[l] = key[it];
            sv[l] = val[it];
        }
    }
    __syncthreads();
    if (range_min) {
        // Last pass (S5 fused): the tile is now ordered by the FULL key (its input was sorted by
        // the lower digits and this pass is stable), so each local run start of a key is a
        // candidate bucket start; the global start is the minimum over tiles.  The sorted keys
        // themselves are not needed afterwards and are not written.
        for (int l = threadIdx.x; l < nt; l += RS_T) {
            const uint32_t k = sk[l];
            const uint32_t dst = gdelta[(k >> shift) & mask] + l;
            vout[dst] = sv[l];
            if (l == 0 || sk[l - 1] != k) atomicMin(&range_min[k], (int)dst);
        }
        return;
    }
    if (gather_pl) {
        // last pass of the pair sort: each pair's tile rect gathered through its (sorted) slot and
        // its tile count written instead of the key (S3 scans the counts into entry offsets)
        for (int l = threadIdx.x; l < nt; l += RS_T) {
            const uint32_t k = sk[l];
            const uint32_t dst = gdelta[(k >> shift) & mask] + l;
            const uint32_t q = sv[l];
            vout[dst] = q;
            const uint2 r = k == 0xffffffffu ? make_uint2(0u, 0u) : gather_pl[q];  // inert: no rect
            pout[dst] = r;
            cnt_out[dst] = (int)(((r.y & 0xffff) - (r.x & 0xffff)) * ((r.y >> 16) - (r.x >> 16)));
        }
        return;
    }
    for (int l = threadIdx.x; l < nt; l += RS_T) {
        const uint32_t k = sk[l];
        const uint32_t dst = gdelta[(k >> shift) & mask] + l;
        kout[dst] = k;
        vout[dst] = sv[l];
    }
}

// Three-kernel passes (per-tile histogram, device-wide scan, scatter) for the entries, whose
// many small tiles make onesweep look-back chains long.
// Stable LSD sort of (k, v)[0..*n_ptr) on bits [0, bits) with ≤ 8-bit digits.  Returns the
// number of passes; the result is in the first buffers when even, in the second ones when odd.
// With range_min (entries: keys < 2^bits are bucket ids) the last pass also writes each
// bucket's first position (atomicMin; the caller fills range_min with INT_MAX first and
// closes empty buckets afterwards) and skips writing the sorted keys.
#ifndef MVGS_RS3_IPT
#define MVGS_RS3_IPT 8  // keys per thread of the three-kernel passes' tiles
#endif
constexpr int RS3_IPT = MVGS_RS3_IPT;

int radix_sort_3k(uint32_t* k, uint32_t* v, uint32_t* k2, uint32_t* v2, const int* n_ptr, int64_t cap, int bits,
                  int* counts, int* scan_tmp, cudaStream_t s, cudaError_t* err, int* range_min, bool first_counted) {
    constexpr int IPT = RS3_IPT;
    const int ntiles = (int)((cap + RS_T * IPT - 1) / (RS_T * IPT));  // ≤ radix_tiles(cap): counts fit
    const int npass = (bits + 7) / 8;
    const int db = npass ? (bits + npass - 1) / npass : 0;
    *err = cudaSuccess;
    if (ntiles == 0) return 0;
    uint32_t *ks = k, *vs = v, *kd = k2, *vd = v2;
    for (int pass = 0; pass < npass; pass++) {
        const int shift = pass * db;
        const int nb = min(db, bits - shift);
        if (!(pass == 0 && first_counted))  // the producer of the keys may have counted pass 0 already
            k_rs_hist<IPT><<<ntiles, RS_T, 0, s>>>(ks, n_ptr, cap, shift, nb, counts, ntiles);
        // only the live digits' counts (digit-major layout): a 7-bit pass scans half the table
        if ((*err = scan_exclusive(counts, (1 << nb) * ntiles, nullptr, scan_tmp, s)) != cudaSuccess) return pass;
        int* rm = (pass == npass - 1) ? range_min : nullptr;
        k_rs_scatter<IPT><<<ntiles, RS_T, 0, s>>>(ks, vs, kd, vd, nullptr, n_ptr, cap, shift, nb, counts, ntiles, rm,
                                                 nullptr, nullptr);
        if ((*err = cudaGetLastError()) != cudaSuccess) return pass;
        uint32_t* t = ks; ks = kd; kd = t;
        t = vs; vs = vd; vd = t;
    }
    return npass;
}

// digit width of the entry sort's passes (keys view·T + tile < V·T)
static void entry_digits(const Launch& L, int* bits, int* db) {
    int b = 1;
    while ((1ll << b) < (int64_t)L.V * L.T) b++;
    const int np = (b + 7) / 8;
    *bits = b;
    *db = (b + np - 1) / np;
}

// view of a pair from the view-major pair offsets (blk_off[v·NB] = first pair of view v)
__device__ __forceinline__ int view_of_pair(const Launch& L, uint32_t q) {
    int lo = 0, hi = L.V - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((uint32_t)L.blk_off[(int64_t)mid * L.NB] <= q) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Duplication in depth order: pair i's entries are ebase[i] + (row-major tile index
// in its rect), key = view·T + tile.  Work is balanced over ENTRIES, not pairs: the
// depth order puts the nearest — largest — footprints first, so a warp owning 32
// consecutive pairs could face 10^5 entries while its neighbours had a few (measured:
// half the SMs idle for half of the kernel).  A warp takes a chunk of DUP_CH
// consecutive entries, finds the pair holding its first entry with a 32-ary search
// over the entry offsets, and walks the chunk's pairs 32 at a time: lanes load one
// pair each, a warp scan of their in-chunk counts gives a contiguous run of entries,
// and lane l writes entries l, l+32, … of the run (coalesced), finding its pair from a
// ballot of the run starts inside its 32-entry window (highest start ≤ its entry).  The row/column split
// uses a float reciprocal of the rect width (exact: (k + 0.5)/w for integers k < 2^20,
// w < 2^12 never rounds across an integer).
constexpr int DUP_CH = RS_T * RS3_IPT;  // one chunk = one tile of the entry sort's first pass

struct DupDesc {  // one pair of the warp's 32
    int x0, y0, w, excl;  // rect origin and width, exclusive prefix of in-chunk counts
    float inv_w;
    uint32_t vb, q;       // view·T, pair slot
    int off0;             // pair-local index of the pair's first in-chunk entry
};

// Since a chunk is exactly one tile of the entry sort's first radix pass, the warp also counts
// that pass's digits of the keys it writes (counts[digit·ntiles + chunk]): the pass needs no
// histogram kernel re-reading the K keys.
#ifdef MVGS_DUP_MINB  // resident CTAs asked of k_dup (unset: ptxas's choice, 48 registers)
#define DUP_BOUNDS __launch_bounds__(256, MVGS_DUP_MINB)
#else
#define DUP_BOUNDS __launch_bounds__(256)
#endif
__global__ DUP_BOUNDS void k_dup(Launch L, const uint32_t* __restrict__ order,
                                             const uint2* __restrict__ rect, const int* __restrict__ ebase,
                                             int* __restrict__ counts, int ntiles, uint32_t dmask) {
    __shared__ uint8_t spos[8][32];
    __shared__ DupDesc desc[8][32];
    __shared__ int dh[8][RS_BINS];
    const int Q = (int)min((int64_t)L.counters[C_NVIS], L.cap_pairs);  // visible pairs (compacted by the sort)
    const int64_t Kall = L.counters[C_K];
    const int Kw = (int)min(Kall, L.cap_entries);  // entries written (the rest is a capacity overflow)
    if (blockIdx.x == 0 && threadIdx.x == 0 && Kall > L.cap_entries) L.counters[C_OVERFLOW] = 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    const int nchunks = (Kw + DUP_CH - 1) / DUP_CH;
    for (int c = blockIdx.x * (blockDim.x >> 5) + wid; c < nchunks; c += nwarps) {
        const int e0 = c * DUP_CH, e1 = min(e0 + DUP_CH, Kw);
        for (int d = lane; d <= (int)dmask; d += 32) dh[wid][d] = 0;
        __syncwarp();
        // largest i < Q with ebase[i] ≤ e0 (ebase[Q] = K > e0): 32-ary search
        int lo = 0, hi = Q;
        while (hi - lo > 1) {
            const int step = (hi - lo + 31) >> 5;
            const int p = lo + lane * step;
            const unsigned bal = __ballot_sync(FULLS, p < hi && ebase[p] <= e0);
            lo += (31 - __clz(bal)) * step;  // lane 0 probes lo itself: bal ≠ 0
            hi = min(hi, lo + step);
        }
        // the 32 pairs' (rect, slot, entry range) are loaded one group ahead of their use
        uint2 rn = make_uint2(0u, 0u);
        uint32_t qn = 0;
        int ebn = Kw, enn = Kw;
        if (lo + lane < Q) {
            rn = rect[lo + lane];
            qn = order[lo + lane];
            ebn = ebase[lo + lane];
            enn = ebase[lo + lane + 1];
        }
        for (int i0 = lo; i0 < Q;) {
            const uint2 r = rn;
            const uint32_t q = qn;
            const int eb = ebn, en = enn;
            const int s0 = max(eb, e0), s1 = min(en, e1);
            const int cnt = max(0, s1 - s0);
            int inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULLS, inc, o);
                if (lane >= o) inc += y;
            }
            const int total = __shfl_sync(FULLS, inc, 31);
            const int ebeg = __shfl_sync(FULLS, s0, 0);  // the run's first entry
            const int enext = __shfl_sync(FULLS, en, 31);  // first entry after these 32 pairs
            const int rx0 = r.x & 0xffff, ry0 = r.x >> 16, rx1 = r.y & 0xffff;
            const int w = rx1 - rx0;
            DupDesc d;
            d.x0 = rx0;
            d.y0 = ry0;
            d.w = w;
            d.excl = inc - cnt;
            d.inv_w = cnt > 0 ? 1.0f / (float)w : 0.f;
            d.vb = cnt > 0 ? (uint32_t)view_of_pair(L, q) * (uint32_t)L.T : 0u;
            d.q = q;
            d.off0 = s0 - eb;
            desc[wid][lane] = d;
            __syncwarp();
            if (enext < e1) {  // the next group, in flight while this one's entries are written
                const int inx = i0 + 32 + lane;
                rn = make_uint2(0u, 0u);
                qn = 0;
                ebn = enn = Kw;
                if (inx < Q) {
                    rn = rect[inx];
                    qn = order[inx];
                    ebn = ebase[inx];
                    enn = ebase[inx + 1];
                }
            }
            // Entries in windows of 32: the owner of entry k is the last lane whose run starts at
            // or before k.  Lanes with entries have distinct, lane-ordered run starts, so a lane
            // starting inside the window marks its bit (and records itself at that position);
            // entry k takes the highest marked bit ≤ k, or the window's carried-in owner.
            const int my_excl = inc - cnt;
            int carry = 0;
            for (int k0 = 0; k0 < total; k0 += 32) {
                const bool st = cnt > 0 && my_excl >= k0 && my_excl < k0 + 32;
                if (st) spos[wid][my_excl - k0] = (uint8_t)lane;
                const unsigned W = __reduce_or_sync(FULLS, st ? 1u << (my_excl - k0) : 0u);  // start positions
                __syncwarp();
                const unsigned le = W & (0xffffffffu >> (31 - lane));  // starts at positions 0..lane
                const int o = le ? (int)spos[wid][31 - __clz(le)] : carry;
                carry = __shfl_sync(FULLS, o, 31);
                __syncwarp();  // spos is rewritten by the next window
                const int k = k0 + lane;
                if (k < total) {
                    const DupDesc& od = desc[wid][o];
                    const int loc = od.off0 + (k - od.excl);
                    const int row = __float2int_rz(((float)loc + 0.5f) * od.inv_w);
                    const int col = loc - row * od.w;
                    const int e = ebeg + k;
                    const uint32_t key = od.vb + (od.y0 + row) * L.TX + od.x0 + col;
                    L.key[e] = key;
                    L.val[e] = od.q;
                    atomicAdd(&dh[wid][key & dmask], 1);
                }
            }
            __syncwarp();
            if (enext >= e1) break;  // warp-uniform
            i0 += 32;
        }
        __syncwarp();
        for (int d = lane; d <= (int)dmask; d += 32) counts[(int64_t)d * ntiles + c] = dh[wid][d];
        __syncwarp();
    }
    // tiles past the written entries (capacity slack) count nothing
    for (int c = nchunks + blockIdx.x * (blockDim.x >> 5) + wid; c < ntiles; c += nwarps)
        for (int d = lane; d <= (int)dmask; d += 32) counts[(int64_t)d * ntiles + c] = 0;
}

// Closes the ranges written by the last entry-sort pass: off[nb] = K, and an empty bucket
// (still INT_MAX) starts where the next one does — a suffix minimum over the V·T buckets.
// Two small kernels over segments of RC_T buckets: the segment minima, then per segment the
// minimum of all later segments, a shared-memory suffix scan and the writes (coalesced).
// The second also records the longest bucket (statistics).
constexpr int RC_T = 1024;

__global__ __launch_bounds__(RC_T) void k_ranges_segmin(Launch L, int* __restrict__ segmin) {
    __shared__ int wm[RC_T / 32];
    const int K = (int)min((int64_t)L.counters[C_K], L.cap_entries);
    const int nb = L.V * L.T;
    const int b = blockIdx.x * RC_T + threadIdx.x;
    int m = b < nb ? min(K, L.bucket_off[b]) : K;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(FULLS, m, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = wm[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(FULLS, m, o));
        if (threadIdx.x == 0) segmin[blockIdx.x] = m;
    }
}

__global__ __launch_bounds__(RC_T) void k_ranges_close(Launch L, const int* __restrict__ segmin) {
    __shared__ int wm[RC_T / 32];
    __shared__ int s_after;
    const int K = (int)min((int64_t)L.counters[C_K], L.cap_entries);
    const int nb = L.V * L.T;
    const int nseg = (nb + RC_T - 1) / RC_T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {  // minimum over the later segments
        int a = K;
        for (int q = blockIdx.x + 1 + lane; q < nseg; q += 32) a = min(a, segmin[q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a = min(a, __shfl_xor_sync(FULLS, a, o));
        if (lane == 0) s_after = a;
    }
    const int b = blockIdx.x * RC_T + threadIdx.x;
    const int v = b < nb ? min(K, L.bucket_off[b]) : K;
    // inclusive suffix minimum over the segment (this bucket and the later ones in it)
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_down_sync(FULLS, inc, o);
        if (lane + o < 32) inc = min(inc, y);
    }
    if (lane == 0) wm[warp] = inc;
    __syncthreads();
    int later = s_after;
    for (int w = warp + 1; w < RC_T / 32; w++) later = min(later, wm[w]);
    const int o = min(inc, later);  // start of this bucket (an empty one takes the next start)
    const int nxt = __shfl_down_sync(FULLS, o, 1);  // start of bucket b + 1 (lane 31: `later`)
    int mx = 0;
    if (b < nb) {
        L.bucket_off[b] = o;
        mx = (lane < 31 ? nxt : later) - o;
    }
    if (b == 0) L.bucket_off[nb] = K;
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) mx = max(mx, __shfl_xor_sync(FULLS, mx, q));
    __syncthreads();
    if (lane == 0) wm[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < RC_T / 32; w++) t = max(t, wm[w]);
        atomicMax(&L.counters[C_MAXB], t);
    }
}

// The pair sort on the three-kernel passes (per-tile histogram, device-wide scan of the
// digit × tile counts, stable scatter) instead of onesweep look-back: inert pairs (key
// 0xffffffff) are not dropped but sort last (every visible depth key is a positive float's
// bits, below 0xffffffff), so the first n_visible sorted pairs are the visible ones; the first
// pass takes the values to be the slots themselves; the last pass gathers each pair's rect
// through its slot and writes its tile count.  Look-back chains made onesweep pay per tile
// (1.12 ms per pass over 79 M pairs at `large`); these passes are plain streaming.
#ifndef MVGS_PS_IPT
#define MVGS_PS_IPT 8  // keys per thread of the pair-sort tiles
#endif
static int radix_sort_pairs_3k(const Launch& L, cudaStream_t s, cudaError_t* err) {
    constexpr int IPT = MVGS_PS_IPT;
    const int64_t cap = L.cap_pairs;
    const int ntiles = (int)((cap + RS_T * IPT - 1) / (RS_T * IPT));
    const int bits = 32, npass = 4, db = 8;
    *err = cudaSuccess;
    if (ntiles == 0) return 0;
    const int* n_ptr = L.counters + C_Q;
    uint32_t *ks = L.pkey, *vs = nullptr, *kd = L.pkey2, *vd = L.pval;
    uint32_t* vbuf[2] = {L.pval, L.pval2};
    for (int pass = 0; pass < npass; pass++) {
        const int shift = pass * db;
        const int nb = min(db, bits - shift);
        k_rs_hist<IPT><<<ntiles, RS_T, 0, s>>>(ks, n_ptr, cap, shift, nb, L.rs_counts, ntiles);
        if ((*err = scan_exclusive(L.rs_counts, (1 << nb) * ntiles, nullptr, L.scan_tmp, s)) != cudaSuccess) return pass;
        vd = vbuf[pass & 1];
        const bool last = pass == npass - 1;
        k_rs_scatter<IPT><<<ntiles, RS_T, 0, s>>>(ks, vs, kd, vd, last ? L.prect2 : nullptr, n_ptr, cap,
                                                        shift, nb, L.rs_counts, ntiles, nullptr,
                                                        last ? L.prect : nullptr, last ? L.ecount : nullptr);
        if ((*err = cudaGetLastError()) != cudaSuccess) return pass;
        uint32_t* t = ks; ks = kd; kd = t;
        vs = vd;
    }
    return npass;
}

// Longest-list-first order of the (view, tile) CTAs of the compositing kernels (LPT):
// a thread waits for its block and a block for its list, so the long lists (garden: max
// 7,812 vs mean 1,737 entries) are dispatched first and the short ones fill the tail.  One CTA
// bins the buckets by list length (32-entry bins, descending; 255 = ≥ 8,160) and scatters their
// ids in bin order; the order inside a bin is arbitrary (no result depends on CTA order).
constexpr int LPT_T = 1024, LPT_BINS = 256;
__global__ __launch_bounds__(LPT_T) void k_lpt_order(const int* __restrict__ off, int nb, int* __restrict__ order) {
    __shared__ int cnt[LPT_BINS];
    if (threadIdx.x < LPT_BINS) cnt[threadIdx.x] = 0;
    __syncthreads();
    auto bin_of = [&](int b) { return LPT_BINS - 1 - min(LPT_BINS - 1, (off[b + 1] - off[b]) >> 5); };
    for (int b = threadIdx.x; b < nb; b += LPT_T) atomicAdd(&cnt[bin_of(b)], 1);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 bins by warp 0 (8 per lane)
        int v[LPT_BINS / 32], sum = 0;
#pragma unroll
        for (int i = 0; i < LPT_BINS / 32; i++) {
            v[i] = cnt[threadIdx.x * (LPT_BINS / 32) + i];
            sum += v[i];
        }
        int inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULLS, inc, o);
            if ((int)threadIdx.x >= o) inc += y;
        }
        int run = inc - sum;
#pragma unroll
        for (int i = 0; i < LPT_BINS / 32; i++) {
            cnt[threadIdx.x * (LPT_BINS / 32) + i] = run;
            run += v[i];
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += LPT_T) order[atomicAdd(&cnt[bin_of(b)], 1)] = b;
}

cudaError_t launch_lpt_order(const Launch& L, int* order, cudaStream_t s) {
    k_lpt_order<<<1, LPT_T, 0, s>>>(L.bucket_off, L.V * L.T, order);
    return cudaGetLastError();
}

cudaError_t launch_sort_pairs(const Launch& L, const uint32_t** order_out, const uint2** rect_out, cudaStream_t s) {
    cudaError_t e;
    const int np = radix_sort_pairs_3k(L, s, &e);
    *order_out = (np & 1) ? L.pval : L.pval2;  // pass p writes pval[p & 1]: the last (p = 3) wrote pval2
    *rect_out = L.prect2;
    return e;
}

// S3: duplicate in depth order (entry offsets from a scan of the tile counts).
cudaError_t launch_dup_sort(const Launch& L, const uint32_t* order, const uint2* rect, cudaStream_t s) {
    // L.ecount: the visible pairs' tile counts in depth order, written by the pair sort's last pass
    cudaError_t e = scan_exclusive(L.ecount, (int)L.cap_pairs, L.counters + C_K, L.scan_tmp, s,
                                   L.counters + C_NVIS);  // entry offsets of the visible pairs; K
    if (e != cudaSuccess) return e;
    {  // one full wave of resident CTAs; chunks are grid-strided over warps
        int dev = 0, nsm = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_dup, 256, 0);
        int bits, db;
        entry_digits(L, &bits, &db);
        const int ntiles = (int)((L.cap_entries + DUP_CH - 1) / DUP_CH);
        k_dup<<<nsm * max(per, 1), 256, 0, s>>>(L, order, rect, L.ecount, L.rs_counts, ntiles, (1u << db) - 1u);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaSuccess;
}

cudaError_t launch_sort_entries(const Launch& L, uint32_t** sorted_vals, cudaStream_t s) {
    int bits, db;
    entry_digits(L, &bits, &db);
    cudaError_t e;
    // bucket starts come out of the last pass (atomicMin): fill with INT_MAX first
    if ((e = cudaMemsetAsync(L.bucket_off, 0x7f, sizeof(int) * ((size_t)L.V * L.T + 1), s)) != cudaSuccess) return e;
    // the first pass's digit counts were written by k_dup
    int np = radix_sort_3k(L.key, L.val, L.key2, L.val2, L.counters + C_K, L.cap_entries, bits, L.rs_counts,
                           L.scan_tmp, s, &e, L.bucket_off, true);
    *sorted_vals = (np & 1) ? L.val2 : L.val;
    if (e != cudaSuccess) return e;
    const int nseg = (L.V * L.T + RC_T - 1) / RC_T;
    k_ranges_segmin<<<nseg, RC_T, 0, s>>>(L, L.scan_tmp);  // (scan scratch: free after the last pass)
    k_ranges_close<<<nseg, RC_T, 0, s>>>(L, L.scan_tmp);
    return cudaGetLastError();
}

}  // namespace mvgs
