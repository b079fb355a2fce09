// k_preprocess.cu — S1–S3 (+ S5) of the hot path.
//
//   k_count       S1  participation test per (Gaussian, view) — "determines which
//                     Gaussians participate in rendering for each viewpoint … before
//                     preprocessing" — counted per (view, 256-Gaussian block)
//   scan          S1  exclusive scan → pair slots: "memory is allocated only for these
//                     participating Gaussians"; view-major, ascending gid
//   k_project     S2  EWA projection, conic, radius, tile rect, SH colour per pair
//                     (P:75), one thread per Gaussian looping its views so
//                     per-Gaussian work (activations, Σ, SH load) is done once for
//                     the whole batch; writes the pair-sort keys (depth, rect)
//   (duplication, sorting and the per-(view, tile) ranges: k_sort.cu)
#include <cstring>
#include "ca.cuh"
#include "internal.cuh"

namespace mvgs {

constexpr unsigned FULL = 0xffffffffu;

// ------------------------------------------------------------------ scan
// Single-pass exclusive scan with decoupled look-back: one kernel per scan.  A CTA takes a
// dynamic tile id (SCAN_T·IPT ints, IPT 16 / 8 / 4 by size), scans it, publishes its aggregate, and warp 0 looks back over
// up to 32 predecessors at a time for the nearest inclusive prefix.  The status words and
// the tile counter are cleared by a memset before every scan (no epochs: graph replays are
// safe).  tmp layout (ints): [0] tile counter, [1] pad, [2 …] u64 status per tile.
#ifndef MVGS_SCAN_T
#define MVGS_SCAN_T 1024  // threads per scan CTA (≤ 1024)
#endif
constexpr int SCAN_T = MVGS_SCAN_T;
constexpr int SCAN_IPT_MIN = 4;  // smallest tile (SCAN_T·4 ints): scans of < ~5 M ints take more, smaller tiles
constexpr unsigned long long SC_AGG = 1ull << 32, SC_PRE = 2ull << 32;

int scan_tmp_size(int n) { return 2 * ((n + SCAN_T * SCAN_IPT_MIN - 1) / (SCAN_T * SCAN_IPT_MIN) + 1) + 4; }

__device__ __forceinline__ int block_exclusive_scan(int x, int* sm /*[33]*/, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = lane < SCAN_T / 32 ? sm[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += y;
        }
        sm[lane] = wi - w;
        if (lane == 31) sm[32] = wi;
    }
    __syncthreads();
    int r = sm[warp] + inc - x;
    *total = sm[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ void scan_st(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long scan_ld(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// n_live (device, nullable): only a[0, min(*n_live, n)) is scanned and the total goes to
// a[min(*n_live, n)]; CTAs past the live tiles exit at once.
template <int IPT>
__global__ __launch_bounds__(SCAN_T) void k_scan_1p(int* __restrict__ a, int n, int* __restrict__ total_slot,
                                                    int* __restrict__ tmp, const int* __restrict__ n_live) {
    __shared__ int sm[33];
    __shared__ int s_tile, s_pre;
    if (n_live) n = min(*n_live, n);
    if (threadIdx.x == 0) s_tile = atomicAdd(tmp, 1);
    __syncthreads();
    const int tile = s_tile;
    const int ntiles = max(1, (n + (SCAN_T * IPT) - 1) / (SCAN_T * IPT));
    if (tile >= ntiles) return;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(tmp + 2);
    const int base = tile * (SCAN_T * IPT) + threadIdx.x * IPT;
    int v[IPT];
    if (base + IPT <= n) {
#pragma unroll
        for (int j = 0; j < IPT / 4; j++) {
            const int4 q = *reinterpret_cast<const int4*>(a + base + 4 * j);
            v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < IPT; i++) v[i] = base + i < n ? a[base + i] : 0;
    }
    int sum = 0;
#pragma unroll
    for (int i = 0; i < IPT; i++) sum += v[i];
    int tot;
    const int ex = block_exclusive_scan(sum, sm, &tot);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int excl = 0;
        if (tile == 0) {
            if (lane == 0) scan_st(status, SC_PRE | (unsigned)tot);
        } else {
            if (lane == 0) scan_st(status + tile, SC_AGG | (unsigned)tot);
            int p = tile - 1;  // nearest predecessor not yet accounted for
            while (true) {
                const int q = p - lane;
                const unsigned long long w = q >= 0 ? scan_ld(status + q) : (SC_PRE | 0ull);
                const bool ready = (w & (SC_AGG | SC_PRE)) != 0;
                const unsigned nr = ~__ballot_sync(FULL, ready);
                const int first_nr = nr ? __ffs(nr) - 1 : 32;  // lanes before it are all ready
                const unsigned pre = __ballot_sync(FULL, ready && (w & SC_PRE)) &
                                     (first_nr == 32 ? 0xffffffffu : ((1u << first_nr) - 1u));
                const int upto = pre ? __ffs(pre) - 1 : first_nr - 1;  // last lane to add
                int val = lane <= upto ? (int)(unsigned)(w & 0xffffffffull) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL, val, o);
                excl += val;
                if (pre) break;
                p -= first_nr;  // 0 when the nearest is not ready: poll again
            }
            if (lane == 0) scan_st(status + tile, SC_PRE | (unsigned)(excl + tot));
        }
        if (lane == 0) s_pre = excl;
    }
    __syncthreads();
    int run = s_pre + ex;
    if (base + IPT <= n) {
#pragma unroll
        for (int j = 0; j < IPT / 4; j++) {
            int4 q;
            q.x = run; run += v[4 * j];
            q.y = run; run += v[4 * j + 1];
            q.z = run; run += v[4 * j + 2];
            q.w = run; run += v[4 * j + 3];
            *reinterpret_cast<int4*>(a + base + 4 * j) = q;
        }
    } else {
#pragma unroll
        for (int i = 0; i < IPT; i++) {
            if (base + i < n) a[base + i] = run;
            run += v[i];
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        a[n] = s_pre + tot;
        if (total_slot) *total_slot = s_pre + tot;
    }
}

// Exclusive scan of a[0..n) in place; a[n] and *total_slot receive the total.  With
// n_live (device) only the first min(*n_live, n) elements take part.  `tmp` holds
// scan_tmp_size(n) ints.
cudaError_t scan_exclusive(int* a, int n, int* total_slot, int* tmp, cudaStream_t s, const int* n_live) {
    // 16384-int tiles; scans shorter than 16 such tiles take 4096-int ones (measured: the 47 k-int
    // pair-count scan 11.8 → 9.8 µs; on the 740 k-int digit-count scans smaller tiles were slower)
    const int ipt = n >= 16 * SCAN_T * 16 ? 16 : SCAN_IPT_MIN;
    int nt = (n + SCAN_T * ipt - 1) / (SCAN_T * ipt);
    if (nt == 0) nt = 1;
    cudaError_t e = cudaMemsetAsync(tmp, 0, sizeof(int) * (2 + 2 * (size_t)nt), s);
    if (e != cudaSuccess) return e;
    if (ipt == 16) k_scan_1p<16><<<nt, SCAN_T, 0, s>>>(a, n, total_slot, tmp, n_live);
    else k_scan_1p<SCAN_IPT_MIN><<<nt, SCAN_T, 0, s>>>(a, n, total_slot, tmp, n_live);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ S1
__global__ __launch_bounds__(BLK) void k_count(Launch L, int blk0) {  // blocks blk0 + blockIdx.x
    __shared__ int wc[BLK / 32][32];
    __shared__ mvgs_camera scams[32];  // the chunk's cameras (LDS instead of per-field global loads)
    __shared__ PartCam spc[32];        // and the bound's per-camera constants
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int blk = blk0 + blockIdx.x;
    const int64_t g = (int64_t)blk * BLK + threadIdx.x;
    const bool valid = g < L.P;
    float mx = 0.f, my = 0.f, mz = 0.f, smax = 0.f;
    if (valid) {
        mx = L.means[3 * g];
        my = L.means[3 * g + 1];
        mz = L.means[3 * g + 2];
        smax = participation_smax(L.log_scales[3 * g], L.log_scales[3 * g + 1], L.log_scales[3 * g + 2]);
    }
    for (int v0 = 0; v0 < L.V; v0 += 32) {
        const int nv = min(32, L.V - v0);
        if (v0 > 0) __syncthreads();  // the previous chunk's cameras are no longer read
        for (int i = threadIdx.x; i < nv * (int)(sizeof(mvgs_camera) / 4); i += BLK)
            reinterpret_cast<uint32_t*>(scams)[i] = reinterpret_cast<const uint32_t*>(L.cams + v0)[i];
        if (threadIdx.x < nv) spc[threadIdx.x] = make_partcam(L.cams[v0 + threadIdx.x], L.TX, L.TY);
        __syncthreads();
        unsigned pm = 0;
        for (int k = 0; k < nv; k++) {
            const mvgs_camera& c = scams[k];
            const bool vis = valid && ca_participates(c, spc[k], mx, my, mz, smax);
            pm |= vis ? 1u << k : 0u;
            const unsigned bal = __ballot_sync(FULL, vis);
            if (lane == 0) wc[warp][k] = __popc(bal);
        }
        if (L.pmask && valid) L.pmask[g] = pm;  // V ≤ 32: one chunk; project and gauss_bwd reuse it
        __syncthreads();
        if (threadIdx.x < nv) {
            int s = 0;
#pragma unroll
            for (int w = 0; w < BLK / 32; w++) s += wc[w][threadIdx.x];
            L.blk_off[(int64_t)(v0 + threadIdx.x) * L.NB + blk] = s;
        }
        __syncthreads();
    }
}

cudaError_t launch_count(const Launch& L, cudaStream_t s) {
    k_count<<<L.NB, BLK, 0, s>>>(L, 0);
    return cudaGetLastError();
}

// Participation counts of the 256-Gaussian blocks [b0, b1) only (an owner rank's range, §11).
cudaError_t launch_count_range(const Launch& L, int b0, int b1, cudaStream_t s) {
    if (b1 > b0) k_count<<<b1 - b0, BLK, 0, s>>>(L, b0);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ S2
// real SH constants [3DGS] as compile-time values (folded into the products)
constexpr float c_SH1 = 0.4886025119029199f;
constexpr float c_SH2_0 = 1.0925484305920792f;
constexpr float c_SH2_1 = -1.0925484305920792f;
constexpr float c_SH2_2 = 0.31539156525252005f;
constexpr float c_SH2_3 = -1.0925484305920792f;
constexpr float c_SH2_4 = 0.5462742152960396f;
constexpr float c_SH3_0 = -0.5900435899266435f;
constexpr float c_SH3_1 = 2.890611442640554f;
constexpr float c_SH3_2 = -0.4570457994644658f;
constexpr float c_SH3_3 = 0.3731763325901154f;
constexpr float c_SH3_4 = -0.4570457994644658f;
constexpr float c_SH3_5 = 1.445305721320277f;
constexpr float c_SH3_6 = -0.5900435899266435f;

// Real SH basis (R17), degree D, direction (x,y,z) unit.
template <int D>
__device__ __forceinline__ void sh_eval_basis(float x, float y, float z, float* Y) {
    // canonical arithmetic: every product / difference one RN operation in
    // a fixed order, so the clamp decision on Σ Y_k sh_k + 0.5 is the oracle's (color32)
    Y[0] = 0.28209479177387814f;
    if (D >= 1) {
        Y[1] = FMUL(-c_SH1, y);
        Y[2] = FMUL(c_SH1, z);
        Y[3] = FMUL(-c_SH1, x);
    }
    if (D >= 2) {
        const float xx = FMUL(x, x), yy = FMUL(y, y), zz = FMUL(z, z);
        Y[4] = FMUL(FMUL(c_SH2_0, x), y);
        Y[5] = FMUL(FMUL(c_SH2_1, y), z);
        Y[6] = FMUL(c_SH2_2, FSUB(FSUB(FMUL(2.f, zz), xx), yy));
        Y[7] = FMUL(FMUL(c_SH2_3, x), z);
        Y[8] = FMUL(c_SH2_4, FSUB(xx, yy));
        if (D >= 3) {
            Y[9] = FMUL(FMUL(c_SH3_0, y), FSUB(FMUL(3.f, xx), yy));
            Y[10] = FMUL(FMUL(FMUL(c_SH3_1, x), y), z);
            Y[11] = FMUL(FMUL(c_SH3_2, y), FSUB(FSUB(FMUL(4.f, zz), xx), yy));
            Y[12] = FMUL(FMUL(c_SH3_3, z), FSUB(FSUB(FMUL(2.f, zz), FMUL(3.f, xx)), FMUL(3.f, yy)));
            Y[13] = FMUL(FMUL(c_SH3_4, x), FSUB(FSUB(FMUL(4.f, zz), xx), yy));
            Y[14] = FMUL(FMUL(c_SH3_5, z), FSUB(xx, yy));
            Y[15] = FMUL(FMUL(c_SH3_6, x), FSUB(xx, FMUL(3.f, yy)));
        }
    }
}

template <int D>
__global__ __launch_bounds__(BLK) void k_project(Launch L) {
    // SH rows in shared memory with an odd number of float4 per row: 16-byte copies in, and
    // the colour loop walks its row with conflict-free LDS.128 (8 lanes per wavefront)
    constexpr int NK = (D + 1) * (D + 1), NS = NK * 3, NS4 = (NS + 3) / 4, SS = 4 * (NS4 | 1);
    extern __shared__ float4 sh_s4[];  // [BLK][SS] SH rows
    float* sh_s = reinterpret_cast<float*>(sh_s4);
    __shared__ int wc[BLK / 32][32];
    __shared__ float2 slim[32];  // the chunk's Jacobian clamp limits (R4)
    __shared__ int sboff[32];  // first pair slot of this block in each view of the chunk
    __shared__ mvgs_camera scams[32];  // the chunk's cameras
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g0 = (int64_t)blockIdx.x * BLK;
    const int64_t g = g0 + threadIdx.x;
    const bool valid = g < L.P;
    {  // SH rows: coalesced async copies (no registers, all in flight), waited on before first use
        const int nb = (int)min((int64_t)BLK, L.P - g0);
        const float* src = L.sh + g0 * (int64_t)L.sh_stride * 3;
        const int rowlen = L.sh_stride * 3;
        if ((rowlen & 3) == 0 && (NS & 3) == 0 && ((uintptr_t)src & 15) == 0) {
            for (int i = threadIdx.x; i < nb * NS4; i += BLK) {
                const int r = i / NS4, k = 4 * (i - r * NS4);  // NS4 constexpr: mul-shift
                cp_async16(&sh_s[r * SS + k], src + (int64_t)r * rowlen + k);
            }
        } else {
            for (int i = threadIdx.x; i < nb * NS; i += BLK) {
                const int r = i / NS, k = i - r * NS;
                cp_async4(&sh_s[r * SS + k], src + (int64_t)r * rowlen + k);
            }
        }
        cp_async_commit();
    }
    const float* sh = sh_s + threadIdx.x * SS;
    float mx = 0.f, my = 0.f, mz = 0.f, smax = 0.f;
    Activ a;
    if (valid) {
        mx = L.means[3 * g];
        my = L.means[3 * g + 1];
        mz = L.means[3 * g + 2];
        smax = participation_smax(L.log_scales[3 * g], L.log_scales[3 * g + 1], L.log_scales[3 * g + 2]);
        ca_activate(L.log_scales + 3 * g, L.quats + 4 * g, L.opac[g], a);
    }
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long my_tiles = 0;  // entries this Gaussian needs (K needed, capacity-independent)
    unsigned my_vis = 0;              // stored visible pairs of this Gaussian
    for (int v0 = 0; v0 < L.V; v0 += 32) {
        const int nv = min(32, L.V - v0);
        // participation of this Gaussian in the chunk's views: k_count's bits when stored
        unsigned pm = 0;
        if (L.pmask) {
            pm = valid ? L.pmask[g] : 0u;
        } else {
            for (int k = 0; k < nv; k++)
                pm |= (valid && ca_participates(L.cams[v0 + k], mx, my, mz, smax, L.TX, L.TY)) ? 1u << k : 0u;
        }
        for (int k = 0; k < nv; k++) {
            const unsigned bal = __ballot_sync(FULL, (pm >> k) & 1u);
            if (lane == 0) wc[warp][k] = __popc(bal);
        }
        if (threadIdx.x < nv) {
            sboff[threadIdx.x] = L.blk_off[(int64_t)(v0 + threadIdx.x) * L.NB + blockIdx.x];
            slim[threadIdx.x] = ca_clamp_limits(L.cams[v0 + threadIdx.x]);  // once per view, not per pair
        }
        for (int i = threadIdx.x; i < nv * (int)(sizeof(mvgs_camera) / 4); i += BLK)
            reinterpret_cast<uint32_t*>(scams)[i] = reinterpret_cast<const uint32_t*>(L.cams + v0)[i];
        cp_async_wait_all();
        __syncthreads();
        if (threadIdx.x < nv) {  // exclusive prefix over warps, per view: wc[w][k] ← Σ_{w' < w}
            int run = 0;
            for (int w = 0; w < BLK / 32; w++) {
                const int c = wc[w][threadIdx.x];
                wc[w][threadIdx.x] = run;
                run += c;
            }
        }
        __syncthreads();
        for (int k = 0; k < nv; k++) {
            const mvgs_camera& c = scams[k];
            const bool vis = (pm >> k) & 1u;
            const unsigned bal = __ballot_sync(FULL, vis);
            if (!vis) continue;
            const int64_t pair = (int64_t)sboff[k] + wc[warp][k] + __popc(bal & lt);
            Proj p;
            ca_project(c, mx, my, mz, a.Sig, L.TX, L.TY, slim[k], p);
            const int tiles = p.ok ? (p.rx1 - p.rx0) * (p.ry1 - p.ry0) : 0;
            if (pair < L.cap_pairs) {  // depth key + rect for the pair sort (the value is the slot itself)
                L.pkey[pair] = tiles > 0 ? __float_as_uint(p.tz) : 0xffffffffu;
                if (tiles > 0)  // inert keys are dropped by the first sort pass: no rect needed
                    L.prect[pair] = make_uint2((uint32_t)p.rx0 | ((uint32_t)p.ry0 << 16),
                                               (uint32_t)p.rx1 | ((uint32_t)p.ry1 << 16));
            }
            if (pair >= L.cap_pairs) {
                L.counters[C_OVERFLOW] = 1;
            } else if (tiles == 0) {
                // inert pair (R27): only the empty rect / depth and the ids are read later
                L.rec[3 * pair + 2] = make_float4(0.f, p.tz, 0.f, 0.f);
                L.pflag[pair] = (p.clx ? 8u : 0u) | (p.cly ? 16u : 0u);
            } else {
                // colour (R17) in canonical arithmetic: its clamp (rgb < 0) is a decision (§4.4)
                const float cpx = -ca_dot3(c.R[0], c.R[3], c.R[6], c.t[0], c.t[1], c.t[2]);
                const float cpy = -ca_dot3(c.R[1], c.R[4], c.R[7], c.t[0], c.t[1], c.t[2]);
                const float cpz = -ca_dot3(c.R[2], c.R[5], c.R[8], c.t[0], c.t[1], c.t[2]);
                float dx = FSUB(mx, cpx), dy = FSUB(my, cpy), dz = FSUB(mz, cpz);
                const float inv = FDIV(1.0f, FSQRT(FMA(dz, dz, FMA(dy, dy, FMUL(dx, dx)))));
                dx = FMUL(dx, inv); dy = FMUL(dy, inv); dz = FMUL(dz, inv);
                float Y[NK];
                sh_eval_basis<D>(dx, dy, dz, Y);
                float rgb[3];
                uint32_t flags = (p.clx ? 8u : 0u) | (p.cly ? 16u : 0u);
                float accs[3] = {0.5f, 0.5f, 0.5f};
                {  // Σ_k Y_k·sh[k][ch], the row read as float4 chunks (same per-channel order)
                    const float4* sh4 = reinterpret_cast<const float4*>(sh);
#pragma unroll
                    for (int i4 = 0; i4 < NS4; i4++) {
                        const float4 q = sh4[i4];
                        const float qe[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const int f = 4 * i4 + e;
                            if (f < NS) accs[f % 3] = FMA(Y[f / 3], qe[e], accs[f % 3]);
                        }
                    }
                }
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    float acc = accs[ch];
                    if (acc < 0.f) {
                        flags |= 1u << ch;
                        acc = 0.f;
                    }
                    rgb[ch] = acc;
                }
                // per-pair constants of the compositing kernels: the exact skip bound of §4.5
                // (−ln(255·o) − 10⁻³, any accurate logf) and 1/o (o·∂L/∂o → ∂L/∂o)
                const float sb = -logf(255.0f * a.o) - 1e-3f;
                float4* r = L.rec + 3 * pair;
                r[0] = make_float4(p.px, p.py, p.A, p.B);
                r[1] = make_float4(p.C, a.o, rgb[0], rgb[1]);
                r[2] = make_float4(rgb[2], p.tz, sb, 1.0f / a.o);
                L.pflag[pair] = flags | PF_VISIBLE | ((uint32_t)min(p.radius, 0xffffff) << PF_RADIUS_SHIFT);  // (its gradient slot is cleared by the forward)
            }
            my_vis += (tiles > 0 && pair < L.cap_pairs) ? 1u : 0u;
            my_tiles += (unsigned long long)tiles;
        }
        __syncthreads();
    }
    // CTA totals, then one atomic per counter per CTA: same-address atomics serialise in one
    // L2 slice (per-warp ones cost ≈ 1 ns each, i.e. ~0.1 ms per 94k warps per view)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_tiles += __shfl_xor_sync(FULL, my_tiles, o);
        my_vis += __shfl_xor_sync(FULL, my_vis, o);
    }
    __shared__ unsigned long long s_tiles[BLK / 32];
    __shared__ unsigned s_vis[BLK / 32];
    if (lane == 0) {
        s_tiles[warp] = my_tiles;
        s_vis[warp] = my_vis;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        unsigned nv = 0;
#pragma unroll
        for (int w = 0; w < BLK / 32; w++) {
            t += s_tiles[w];
            nv += s_vis[w];
        }
        if (t) atomicAdd(&L.counters64[4], t);
        if (nv) atomicAdd(&L.counters[C_NVIS], (int)nv);
    }
}

template <int D>
cudaError_t launch_project_t(const Launch& L, cudaStream_t s) {
    const size_t smem = sizeof(float) * BLK * 4 * ((((D + 1) * (D + 1) * 3 + 3) / 4) | 1);
    cudaError_t e = cudaFuncSetAttribute(k_project<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_project<D><<<L.NB, BLK, smem, s>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_project(const Launch& L, cudaStream_t s) {
    switch (L.sh_degree) {
        case 0: return launch_project_t<0>(L, s);
        case 1: return launch_project_t<1>(L, s);
        case 2: return launch_project_t<2>(L, s);
        default: return launch_project_t<3>(L, s);
    }
}

// ------------------------------------------------------------------ cameras
// Up to 32 cameras travel as a kernel parameter (2.4 KB) and are stored to the context's
// device array: graph-capturable with the values baked into the node, no host staging.
struct CamBlock {
    mvgs_camera c[32];
};
__global__ void k_set_cams(CamBlock b, int n, mvgs_camera* __restrict__ dst) {
    const int words = n * (int)(sizeof(mvgs_camera) / 4);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(b.c);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (int i = threadIdx.x; i < words; i += blockDim.x) d[i] = src[i];
}

cudaError_t launch_set_cams(const mvgs_camera* h_cams, int V, mvgs_camera* d_cams, cudaStream_t s) {
    static_assert(sizeof(mvgs_camera) % 4 == 0, "camera is word-sized");
    for (int v0 = 0; v0 < V; v0 += 32) {
        CamBlock b;
        const int n = V - v0 < 32 ? V - v0 : 32;
        memcpy(b.c, h_cams + v0, sizeof(mvgs_camera) * n);
        k_set_cams<<<1, 256, 0, s>>>(b, n, d_cams + v0);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ------------------------------------------------------------------ export (tests)
// (view, gid) of pair slot q, recomputed from the slot allocation (no per-pair ids are
// stored by the path): the view and 256-Gaussian block by binary search over the scanned
// per-(view, block) offsets, then the rank among the block's participating Gaussians.
__device__ void slot_ids(const Launch& L, int64_t q, int& view, int64_t& gid) {
    int lo = 0, hi = L.V * L.NB - 1;  // last (view, block) index with blk_off ≤ q (skips empty ones)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((int64_t)L.blk_off[mid] <= q) lo = mid;
        else hi = mid - 1;
    }
    view = lo / L.NB;
    const int b = lo - view * L.NB;
    int r = (int)(q - L.blk_off[lo]);
    const mvgs_camera& c = L.cams[view];
    gid = -1;
    for (int64_t g = (int64_t)b * BLK; g < min(L.P, (int64_t)(b + 1) * BLK); g++) {
        const float sm = participation_smax(L.log_scales[3 * g], L.log_scales[3 * g + 1], L.log_scales[3 * g + 2]);
        if (ca_participates(c, L.means[3 * g], L.means[3 * g + 1], L.means[3 * g + 2], sm, L.TX, L.TY) && r-- == 0) {
            gid = g;
            break;
        }
    }
}

__global__ void k_export(Launch L, int64_t* range_start, int32_t* entry_gid, int32_t* pair_ids, int32_t* pair_i,
                         float* pair_f, float* pair_g) {
    const int Q = min((int64_t)L.counters[C_Q], L.cap_pairs);
    const int64_t K = min((int64_t)L.counters[C_K], L.cap_entries);
    const int64_t nb = (int64_t)L.V * L.T;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (range_start)
        for (int64_t b = t0; b <= nb; b += stride) range_start[b] = L.bucket_off[b];
    if (entry_gid)
        for (int64_t e = t0; e < K; e += stride) {
            int v;
            int64_t gid;
            slot_ids(L, L.sorted[e], v, gid);
            entry_gid[e] = (int32_t)gid;
        }
    for (int64_t q = t0; q < Q; q += stride) {
        int view = 0;
        int64_t gid = 0;
        if (pair_ids || pair_i) slot_ids(L, q, view, gid);
        const float4 r0 = L.rec[3 * q], r1 = L.rec[3 * q + 1], r2 = L.rec[3 * q + 2];
        // the rect of a visible pair: its slot in the unsorted rect array (the pair sort gathers
        // from it, MVGS_PAIR_GATHER, and leaves it intact); inert pairs have an empty rect
        const bool inert = !(L.pflag[q] & PF_VISIBLE);  // tiles == 0: only depth and ids were written (R27)
        const uint2 rr = inert ? make_uint2(0u, 0u) : L.prect[q];
        const uint32_t lo = rr.x, hi = rr.y;
        if (pair_ids) {
            pair_ids[2 * q] = (int32_t)view;
            pair_ids[2 * q + 1] = (int32_t)gid;
        }
        if (pair_i) {
            const int rx0 = lo & 0xffff, ry0 = lo >> 16, rx1 = hi & 0xffff, ry1 = hi >> 16;
            int32_t* o = pair_i + 8 * q;
            int radius = 0;  // not kept by the path: recomputed here through the same CA projection
            if (gid >= 0) {
                Activ a;
                ca_activate(L.log_scales + 3 * gid, L.quats + 4 * gid, L.opac[gid], a);
                Proj p;
                ca_project(L.cams[view], L.means[3 * gid], L.means[3 * gid + 1], L.means[3 * gid + 2], a.Sig, L.TX,
                           L.TY, ca_clamp_limits(L.cams[view]), p);
                radius = p.radius;
            }
            o[0] = radius;
            o[1] = rx0; o[2] = ry0; o[3] = rx1; o[4] = ry1;
            o[5] = (rx1 - rx0) * (ry1 - ry0);
            o[6] = (int32_t)(L.pflag[q] & 0x1fu);
            o[7] = 0;
        }
        if (pair_f) {
            float* f = pair_f + 12 * q;
            f[0] = r2.y;
            if (inert) {
                for (int k = 1; k < 12; k++) f[k] = 0.f;
            } else {
                f[1] = r0.x; f[2] = r0.y; f[3] = r0.z; f[4] = r0.w; f[5] = r1.x;
                f[6] = r1.y; f[7] = r1.z; f[8] = r1.w; f[9] = r2.x; f[10] = 0.f; f[11] = 0.f;
            }
        }
        if (pair_g)
            for (int k = 0; k < NG; k++) pair_g[NG * q + k] = inert ? 0.f : L.pgrad[q * PG_STRIDE + k];
    }
}

cudaError_t launch_export(const Launch& L, int64_t* range_start, int32_t* entry_gid, int32_t* pair_ids,
                          int32_t* pair_i, float* pair_f, float* pair_g, cudaStream_t s) {
    k_export<<<1024, 256, 0, s>>>(L, range_start, entry_gid, pair_ids, pair_i, pair_f, pair_g);
    return cudaGetLastError();
}

}  // namespace mvgs
