// k_render.cu — S6 forward compositing and S7 backward compositing + E1.
//
// Grid = one CTA per (view, tile) — "multiple blocks per tile, one block for
// each viewpoint".  A CTA has 128 threads for the 16×16 tile: each
// thread owns TWO pixels (rows r and r+4 of its warp's 8×8 block), so every
// staged record, loop step and — in the backward — every warp reduction is
// shared by two pixels.  Entries of the tile's depth-sorted list are staged in
// shared memory a batch of 128 at a time, one record per thread, then every
// thread walks the batch (Alg. 2).  A warp whose pixels have all
// terminated leaves the batch loop at once; the CTA stops fetching when all
// its pixels are done.
//
// Backward (adjoint of Eq. (1)): back to front from each pixel's
// n_contrib, reconstructing T by division, one independent warp per (view,
// tile, 8×8 block) staging its own batches (no CTA barrier).  For each entry a
// lane adds its two pixels' ten terms (Σ∇x, Σ∇y, ‖∇‖ for E1, ∂A, ∂B, ∂C, ∂o,
// ∂r, ∂g, ∂b; ‖∇‖ is taken per pixel before adding — "norm and add",
// P:18–20), the warp transpose-reduces them (12 shuffles for 10 values; each
// lane ends up owning one value's warp sum) and the ten owner lanes add them to
// the pair's gradient slot with one global red.add warp instruction.
#include <cudaTypedefs.h>
#include "ca.cuh"
#include "internal.cuh"
#include "tma.cuh"

namespace mvgs {

#ifndef MVGS_FWD_UNROLL
#define MVGS_FWD_UNROLL 1  // inner entry loops (experiment knobs)
#endif
#ifndef MVGS_FWD_PREFETCH
#define MVGS_FWD_PREFETCH 1  // forward: next batch's indices a batch ahead, records prefetched to L2
#endif
#ifndef MVGS_FWD_BATCH
#define MVGS_FWD_BATCH 1  // forward staged batch = 128 × this entries
#endif
#ifndef MVGS_FWD_PAIR
#define MVGS_FWD_PAIR 1  // forward walk: two entries per step (measured: garden fwd 0.409 → 0.375 ms; four: no gain)
#endif
#ifndef MVGS_BWD_PAIR
#define MVGS_BWD_PAIR 1  // backward walk: two entries per step (measured: garden bwd 0.739 → 0.713, playroom 3.44 → 3.31 ms)
#endif
#ifndef MVGS_BWD_MINB
#define MVGS_BWD_MINB 6  // resident CTAs per SM asked of the backward (register cap 65536/(128·MINB))
#endif
constexpr int kFwdUnroll = MVGS_FWD_UNROLL;
constexpr int RT = 128;            // threads per CTA = entries per staged batch
constexpr unsigned FULLR = 0xffffffffu;

// CTA-wide sums of two per-thread counts → one 64-bit atomic each per CTA.
__device__ __forceinline__ void count_evals(unsigned long long* ctr0, unsigned long long* ctr1, unsigned n0,
                                            unsigned n1, unsigned* sm) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n0 += __shfl_xor_sync(FULLR, n0, o);
        n1 += __shfl_xor_sync(FULLR, n1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(sm, n0);
        atomicAdd(sm + 1, n1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(ctr0, (unsigned long long)sm[0]);
        atomicAdd(ctr1, (unsigned long long)sm[1]);
    }
}

// Exact early skip: α = min(0.99, o·G) < 1/255 ⇔ power < −ln(255·o).
// Below −ln(255·o) − SKIP_MARGIN the CA value o·G is < (1/255)·e^(−1e-3)·(1 + 1e-6),
// so the CA decision is "skip" as well; the CA exp is only evaluated above this bound.

// Warp blocks of the 16×16 tile: warp w owns a WBW × WBH block of pixels (lane → column
// lane % WBW, row lane / WBW, and the same column WBH/2 rows further down for the thread's
// second pixel).  16×4 (four stacked strips) or 8×8 (a 2×2 arrangement, MVGS_WB8): a square
// block has the shortest perimeter, so fewer of its pixels lie outside a small footprint.
#ifndef MVGS_WB8
#define MVGS_WB8 1  // measured (garden / playroom / train): 8×8 bwd 0.742 → 0.729, 3.54 → 3.39, 1.061 → 1.044 ms
#endif
constexpr int WBW = MVGS_WB8 ? 8 : 16, WBH = MVGS_WB8 ? 8 : 4;
constexpr int WB_PER_ROW = TILE / WBW;  // warp blocks per tile row
__device__ __forceinline__ int wb_x0(int w) { return (w % WB_PER_ROW) * WBW; }
__device__ __forceinline__ int wb_y0(int w) { return (w / WB_PER_ROW) * WBH; }
// pixel coordinates of this thread's two pixels (rows r and r + WBH/2 of its warp's block)
__device__ __forceinline__ void pixel_pair(int tx, int ty, int& x, int& y0, int& y1) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    x = tx * TILE + wb_x0(warp) + (lane % WBW);
    y0 = ty * TILE + wb_y0(warp) + (lane / WBW);
    y1 = y0 + WBH / 2;
}

// Exact warp-block culling.  A pixel reaches the canonical exp only if
// its CA power ≥ sb.  With d = μ' − p and q(d) = dᵀMd, M = [[A, B], [B, C]] (the stored
// fp32 conic), the exact power is −q/2 and the CA value differs from it by at most
// ε·T(d), T(d) = A·dx² + C·dy² + 2|B·dx·dy|, ε = 8·2⁻²⁴ (a few fp32 roundings).  q_min, the
// minimum of q over a warp's pixel block (0 if μ' lies in it, else the smallest of q on the
// four edges, each a 1-D quadratic taken at its clamped minimiser), is evaluated in fp32
// with an error below another ε·T_max (evaluating at a rounded minimiser only raises q by
// C·δ², δ ~ 1e-7·|t|, far inside the 0.01 slack).  No pixel of the block can pass when
//   q_min > 1.01·L + 0.01 + 3ε·T_max,   L = −2·sb,  T_max ≥ T over the block.
// Conics that are not positive definite are never culled.  Bit j: the entry may touch
// warp j's block of the tile.
// nBoC = −B/C, nBoA = −B/A (once per entry: the 1-D minimisers are −B·fixed/C and −B·fixed/A; a
// rounded minimiser only raises q by C·δ², far inside the slack)
__device__ __forceinline__ float q_edge(float A, float B, float C, float nBoA, float nBoC, float fixed, float lo,
                                        float hi, bool fix_x) {
    if (fix_x) {  // dx fixed, dy clamped to [lo, hi] at the 1-D minimiser
        const float t = fminf(hi, fmaxf(lo, nBoC * fixed));
        return A * fixed * fixed + 2.0f * B * fixed * t + C * t * t;
    }
    const float t = fminf(hi, fmaxf(lo, nBoA * fixed));
    return A * t * t + 2.0f * B * t * fixed + C * fixed * fixed;
}

__device__ __noinline__ unsigned warp_block_mask(float px, float py, float A, float B, float C, float sb, float X0,
                                                 float Y0) {
#ifdef MVGS_NO_CULL
    return 0xfu;  // experiment / diagnosis: every warp walks every entry
#endif
    const float L = -2.0f * sb;
    if (!(A > 0.0f) || !(C > 0.0f) || !((double)A * (double)C - (double)B * (double)B > 0.0) || !(L > 0.0f))
        return 0xfu;
    const float eps3 = 3.0f * 8.0f * 5.9604644775390625e-8f;
    const float Lm = L * 1.01f + 0.01f;
    const float nBoA = -B / A, nBoC = -B / C;
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < 4; w++) {
        const float x0 = X0 + (float)wb_x0(w), y0 = Y0 + (float)wb_y0(w);
        const float dxlo = px - (x0 + (float)(WBW - 1)), dxhi = px - x0;  // d = μ' − p over the block (exact)
        const float dylo = py - (y0 + (float)(WBH - 1)), dyhi = py - y0;
        const float dxm = fmaxf(fabsf(dxlo), fabsf(dxhi));
        const float dym = fmaxf(fabsf(dylo), fabsf(dyhi));
        float qmin = 0.0f;
        if (!(dxlo <= 0.0f && dxhi >= 0.0f && dylo <= 0.0f && dyhi >= 0.0f)) {  // centre outside the block
            qmin = fminf(fminf(q_edge(A, B, C, nBoA, nBoC, dxlo, dylo, dyhi, true),
                               q_edge(A, B, C, nBoA, nBoC, dxhi, dylo, dyhi, true)),
                         fminf(q_edge(A, B, C, nBoA, nBoC, dylo, dxlo, dxhi, false),
                               q_edge(A, B, C, nBoA, nBoC, dyhi, dxlo, dxhi, false)));
        }
        const float tmax = A * dxm * dxm + C * dym * dym + 2.0f * fabsf(B) * dxm * dym;
        if (!(qmin > Lm + eps3 * tmax)) m |= 1u << w;
    }
    return m;
}

// Per-warp compacted batch: the indices j < cnt whose mask has this warp's bit, ascending.
__device__ __forceinline__ int warp_batch_list(const uint8_t* smask, int cnt, int warp, int lane, uint8_t* list) {
    int n = 0;
    for (int c = 0; c < cnt; c += 32) {
        const int j = c + lane;
        const bool in = j < cnt && ((smask[j] >> warp) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) list[n + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)j;
        n += __popc(bal);
    }
    __syncwarp();
    return n;
}

// ---------------------------------------------------------------------------------------
// Packed forward: the thread's two pixels are the lanes of FP32x2 registers; every CA operation
// (power, canonical exp, α, T·(1 − α)) is the per-lane RN operation of the scalar forms, so
// decisions, T_final and n_contrib are bit-identical to the canonical arithmetic of §4.  A
// lane that does not blend the entry gets weight 0 and keeps its T.  A terminated pixel keeps
// its T with the sign flipped (T > 0 while the pixel is live), so "done" needs no flag
// register: every test on a live pixel is a test on T's sign.
__device__ __forceinline__ float2 ff2(float a, float b) { return make_float2(a, b); }

// ca_exp_core per lane, packed, for x ∈ [−87, 0] as the compositing kernels
// use it (x ≥ the skip bound > −5.6).  Bit-identical to ca_exp_core: m = fma(x, log2e, 1.5·2²³)
// puts the integer nearest to the exact x·log2e in m's low mantissa bits (two's complement,
// |n| < 2²²), n = m − 1.5·2²³ exactly, and p·2ⁿ — exact, p ∈ [2^-½, 2^½], n ≥ −126 — is formed by
// adding n to p's exponent field: (bits(m) << 23) + bits(p), one LEA per lane.
__device__ __forceinline__ float2 ca_exp_core2(float2 x) {
    const float2 m = __ffma2_rn(x, ff2(1.44269504f, 1.44269504f), ff2(CA_MAGIC, CA_MAGIC));
    const float2 n = __fadd2_rn(m, ff2(-CA_MAGIC, -CA_MAGIC));
    float2 r = __ffma2_rn(n, ff2(-0.693145751953125f, -0.693145751953125f), x);
    r = __ffma2_rn(n, ff2(-1.428606765330187e-6f, -1.428606765330187e-6f), r);
    const float c6 = (float)(1.0 / 720.0), c5 = (float)(1.0 / 120.0), c4 = (float)(1.0 / 24.0),
                c3 = (float)(1.0 / 6.0);
    float2 p = __ffma2_rn(ff2(c6, c6), r, ff2(c5, c5));
    p = __ffma2_rn(p, r, ff2(c4, c4));
    p = __ffma2_rn(p, r, ff2(c3, c3));
    p = __ffma2_rn(p, r, ff2(0.5f, 0.5f));
    p = __ffma2_rn(p, r, ff2(1.f, 1.f));
    p = __ffma2_rn(p, r, ff2(1.f, 1.f));
    return ff2(__int_as_float((__float_as_int(m.x) << 23) + __float_as_int(p.x)),
               __int_as_float((__float_as_int(m.y) << 23) + __float_as_int(p.y)));
}

template <bool DEPTH, bool CNT>
__global__ __launch_bounds__(RT) void k_render_fwd_p(Launch L, float* __restrict__ out_rgb,
                                                     float* __restrict__ out_T, int32_t* __restrict__ out_n,
                                                     float* __restrict__ out_D) {
    constexpr int FB = RT * MVGS_FWD_BATCH;  // entries per staged batch (≤ 256: uint8 list indices)
    static_assert(FB <= 256, "list indices are bytes");
    // staged entry constants, one array (an entry's three loads share one address):
    //   (μ'x, μ'y, A, C), (B, o, skip bound, depth), (r, g, b, −)
    __shared__ float4 se[3][FB];
    __shared__ uint8_t smask[FB];
    __shared__ uint8_t slist[RT / 32][FB];
    __shared__ unsigned sev[2];
    zero_pgrad_slice(L);
    const int bucket = L.order ? L.order[blockIdx.x] : blockIdx.x;  // longest list first
    const int v = bucket / L.T, tile = bucket - v * L.T;
    const int ty = tile / L.TX, tx = tile - ty * L.TX;
    int x, y[2];
    pixel_pair(tx, ty, x, y[0], y[1]);
    const int start = L.bucket_off[bucket], end = L.bucket_off[bucket + 1];
    const float2 nfx = ff2(-(float)x, -(float)x), nfy = ff2(-(float)y[0], -(float)y[1]);
    const float2 one = ff2(1.f, 1.f), mone = ff2(-1.f, -1.f), mhalf = ff2(-0.5f, -0.5f);
    // T < 0: the pixel is done (terminated, or outside the image)
    float2 T = ff2((x < L.W && y[0] < L.H) ? 1.f : -1.f, (x < L.W && y[1] < L.H) ? 1.f : -1.f);
    float2 C0 = ff2(0.f, 0.f), C1 = C0, C2 = C0, D = C0;
    int last0 = 0, last1 = 0;
    unsigned nev = 0, nexp = 0;
    if (threadIdx.x == 0) sev[0] = sev[1] = 0;
    __syncthreads();
    // next batch's record index of this thread, loaded one batch ahead (FB == RT)
    constexpr bool PF = MVGS_FWD_PREFETCH && FB == RT;
    uint32_t qn = (PF && start + (int)threadIdx.x < end) ? L.sorted[start + threadIdx.x] : 0u;
    if (end <= L.cap_entries) {
        for (int b0 = start; b0 < end; b0 += FB) {
            if (__syncthreads_count(T.x < 0.f && T.y < 0.f) == RT) break;
            for (int t = threadIdx.x; t < FB && b0 + t < end; t += RT) {
                const int idx = b0 + t;
                const float4* r = L.rec + 3 * (int64_t)(PF ? qn : L.sorted[idx]);
                const float4 r0 = r[0], r1 = r[1], r2 = r[2];  // (x, y, A, B) (C, o, r, g) (b, depth, sb, 1/o)
                se[0][t] = make_float4(r0.x, r0.y, r0.z, r1.x);
                se[1][t] = make_float4(r0.w, r1.y, r2.z, r2.y);
                se[2][t] = make_float4(r1.z, r1.w, r2.x, 0.f);
                smask[t] = (uint8_t)warp_block_mask(r0.x, r0.y, r0.z, r0.w, r1.x, r2.z, (float)(tx * TILE),
                                                    (float)(ty * TILE));
            }
            __syncthreads();
            const int cnt = min(FB, end - b0);
            const int wl = threadIdx.x >> 5;
            const int jbase = b0 - start + 1;  // list index + 1 of batch entry 0
            const int nl = warp_batch_list(smask, cnt, wl, threadIdx.x & 31, slist[wl]);
            if (PF) {  // the next batch: index now (consumed after this batch's walk)
                const int nidx = b0 + FB + (int)threadIdx.x;
                qn = nidx < end ? L.sorted[nidx] : 0u;
            }
            // one entry: the CA power and skip test (geometry only: liveness is applied at the
            // entry's turn), the CA exp and α, then the blend in list order
            auto geo = [&](int j, float2& power, bool& g0, bool& g1) {
                const float4 e0 = se[0][j], e1 = se[1][j];
                const float2 dx = __fadd2_rn(ff2(e0.x, e0.x), nfx);
                const float2 dy = __fadd2_rn(ff2(e0.y, e0.y), nfy);
                const float2 Adx = __fmul2_rn(ff2(e0.z, e0.z), dx);
                const float2 CdyDy = __fmul2_rn(__fmul2_rn(ff2(e0.w, e0.w), dy), dy);
                const float2 inner = __ffma2_rn(Adx, dx, CdyDy);
                const float2 nBdxdy = __fmul2_rn(__fmul2_rn(ff2(-e1.x, -e1.x), dx), dy);
                power = __ffma2_rn(mhalf, inner, nBdxdy);
                g0 = !(power.x > 0.f) && !(power.x < e1.z);
                g1 = !(power.y > 0.f) && !(power.y < e1.z);
            };
            auto alpha_of = [&](int j, float2 power) {
                const float o = se[1][j].y;
                const float2 oG = __fmul2_rn(ff2(o, o), ca_exp_core2(power));
                return ff2(fminf(ALPHA_MAX, oG.x), fminf(ALPHA_MAX, oG.y));
            };
            auto blend = [&](int j, float2 alpha, bool in0, bool in1) {
                const bool ok0 = in0 && !(alpha.x < ALPHA_MIN), ok1 = in1 && !(alpha.y < ALPHA_MIN);
                const float2 Tn = __fmul2_rn(T, __ffma2_rn(alpha, mone, one));  // T·(1 − α), CA
                const bool term0 = ok0 && Tn.x < T_EPS, term1 = ok1 && Tn.y < T_EPS;
                const bool bl0 = ok0 && !term0, bl1 = ok1 && !term1;
                const float2 w = __fmul2_rn(ff2(bl0 ? alpha.x : 0.f, bl1 ? alpha.y : 0.f), T);
                const float4 e2 = se[2][j];
                C0 = __ffma2_rn(ff2(e2.x, e2.x), w, C0);
                C1 = __ffma2_rn(ff2(e2.y, e2.y), w, C1);
                C2 = __ffma2_rn(ff2(e2.z, e2.z), w, C2);
                if (DEPTH) D = __ffma2_rn(ff2(se[1][j].w, se[1][j].w), w, D);
                T = ff2(bl0 ? Tn.x : (term0 ? -T.x : T.x), bl1 ? Tn.y : (term1 ? -T.y : T.y));
                const int jn = jbase + j;
                last0 = bl0 ? jn : last0;
                last1 = bl1 ? jn : last1;
            };
            int u = 0;
#if MVGS_FWD_PAIR
            // two entries per step: both geometries and exps first (independent chains), then the
            // two blends in list order — the second sees the first's T, so every decision is the
            // one-entry walk's
            for (; u + 1 < nl && !(T.x < 0.f && T.y < 0.f); u += 2) {
                const int ja = slist[wl][u], jb = slist[wl][u + 1];
                float2 pa, pb;
                bool ga0, ga1, gb0, gb1;
                geo(ja, pa, ga0, ga1);
                geo(jb, pb, gb0, gb1);
                if (!(ga0 || ga1 || gb0 || gb1)) {
                    if (CNT) nev += 2u * ((unsigned)(T.x > 0.f) + (unsigned)(T.y > 0.f));
                    continue;
                }
                const float2 aa = alpha_of(ja, pa), ab = alpha_of(jb, pb);
                const bool ia0 = T.x > 0.f && ga0, ia1 = T.y > 0.f && ga1;
                if (CNT) {
                    nev += (unsigned)(T.x > 0.f) + (unsigned)(T.y > 0.f);
                    nexp += (unsigned)ia0 + (unsigned)ia1;
                }
                blend(ja, aa, ia0, ia1);
                const bool ib0 = T.x > 0.f && gb0, ib1 = T.y > 0.f && gb1;
                if (CNT) {
                    nev += (unsigned)(T.x > 0.f) + (unsigned)(T.y > 0.f);
                    nexp += (unsigned)ib0 + (unsigned)ib1;
                }
                blend(jb, ab, ib0, ib1);
            }
#endif
#pragma unroll(kFwdUnroll)
            for (; u < nl && !(T.x < 0.f && T.y < 0.f); u++) {
                const int j = slist[wl][u];
                if (CNT) nev += (unsigned)(T.x > 0.f) + (unsigned)(T.y > 0.f);
                float2 power;
                bool g0, g1;
                geo(j, power, g0, g1);
                const bool in0 = T.x > 0.f && g0, in1 = T.y > 0.f && g1;
                if (!(in0 || in1)) continue;
                if (CNT) nexp += (unsigned)in0 + (unsigned)in1;
                const float2 alpha = alpha_of(j, power);
                if (!((in0 && !(alpha.x < ALPHA_MIN)) || (in1 && !(alpha.y < ALPHA_MIN)))) continue;
                blend(j, alpha, in0, in1);
            }
            if (PF && b0 + FB + (int)threadIdx.x < end) {  // warm the next batch's record in L2
                const float4* rn = L.rec + 3 * (int64_t)qn;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(rn));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(rn + 2));
            }
        }
    }
    if (CNT) count_evals(&L.counters64[0], &L.counters64[2], nev, nexp, sev);
    const int64_t HW = (int64_t)L.H * L.W;
    const float Cs[2][3] = {{C0.x, C1.x, C2.x}, {C0.y, C1.y, C2.y}};
    const float Ts[2] = {fabsf(T.x), fabsf(T.y)}, Ds[2] = {D.x, D.y};
    const int ls[2] = {last0, last1};
#pragma unroll
    for (int p = 0; p < 2; p++) {
        if (!(x < L.W && y[p] < L.H)) continue;
        const int64_t pix = (int64_t)y[p] * L.W + x;
        out_rgb[(3 * (int64_t)v + 0) * HW + pix] = __fmaf_rn(Ts[p], L.bg[0], Cs[p][0]);  // CA: fma(T, bg, C)
        out_rgb[(3 * (int64_t)v + 1) * HW + pix] = __fmaf_rn(Ts[p], L.bg[1], Cs[p][1]);  // CA: fma(T, bg, C)
        out_rgb[(3 * (int64_t)v + 2) * HW + pix] = __fmaf_rn(Ts[p], L.bg[2], Cs[p][2]);  // CA: fma(T, bg, C)
        out_T[v * HW + pix] = Ts[p];
        out_n[v * HW + pix] = ls[p];
        if (DEPTH) out_D[v * HW + pix] = Ds[p];
    }
}

// Forward with TMA staging (tma.cuh): the batch's records arrive by gather4 into a double
// buffer of raw 64-byte rows (x, y, A, B) (C, o, r, g) (b, depth, skip bound, 1/o) (0 …);
// warp 0 issues batch b+1 right after batch b's masks are built, so it lands while batch b is
// walked.  The walk and every decision are those of k_render_fwd_p.
template <bool DEPTH, bool CNT>
__global__ __launch_bounds__(RT) void k_render_fwd_tma(Launch L, const __grid_constant__ CUtensorMap tm,
                                                       float* __restrict__ out_rgb, float* __restrict__ out_T,
                                                       int32_t* __restrict__ out_n, float* __restrict__ out_D) {
    __shared__ __align__(128) float4 srec[2][RT][TMA_ROW_FLOATS / 4];
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint8_t smask[RT];
    __shared__ uint8_t slist[RT / 32][RT];
    __shared__ unsigned sev[2];
    zero_pgrad_slice(L);
    const int bucket = L.order ? L.order[blockIdx.x] : blockIdx.x;  // longest list first
    const int v = bucket / L.T, tile = bucket - v * L.T;
    const int ty = tile / L.TX, tx = tile - ty * L.TX;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    int x, y[2];
    pixel_pair(tx, ty, x, y[0], y[1]);
    const int start = L.bucket_off[bucket], end = L.bucket_off[bucket + 1];
    const int nbat = end <= L.cap_entries ? (end - start + RT - 1) / RT : 0;
    const float2 nfx = ff2(-(float)x, -(float)x), nfy = ff2(-(float)y[0], -(float)y[1]);
    const float2 one = ff2(1.f, 1.f), mone = ff2(-1.f, -1.f), mhalf = ff2(-0.5f, -0.5f);
    float2 T = ff2((x < L.W && y[0] < L.H) ? 1.f : -1.f, (x < L.W && y[1] < L.H) ? 1.f : -1.f);
    float2 C0 = ff2(0.f, 0.f), C1 = C0, C2 = C0, D = C0;
    int last0 = 0, last1 = 0;
    unsigned nev = 0, nexp = 0;
    if (threadIdx.x == 0) {
        sev[0] = sev[1] = 0;
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // warp 0 holds the pair slots of the next batch to issue (4 per lane), loaded a batch early
    int qi[4] = {0, 0, 0, 0};
    auto load_idx = [&](int b) {
        const int e = start + b * RT + 4 * lane;
#pragma unroll
        for (int i = 0; i < 4; i++) qi[i] = (b < nbat && e + i < end) ? (int)L.sorted[e + i] : 0;
    };
    auto issue = [&](int b) {  // warp 0: batch b's records → srec[b & 1]
        const int cnt = min(RT, end - (start + b * RT));
        const int ng = (cnt + 3) >> 2;
        if (lane == 0) mbar_arrive_expect_tx(&mbar[b & 1], (unsigned)(ng * 4 * TMA_ROW_BYTES));
        __syncwarp();
        if (lane < ng) tma_gather4(&srec[b & 1][4 * lane][0], &tm, &mbar[b & 1], qi[0], qi[1], qi[2], qi[3]);
    };
    if (wl == 0 && nbat > 0) {
        load_idx(0);
        issue(0);
        load_idx(1);
    }
    for (int b = 0; b < nbat; b++) {
        const int buf = b & 1;
        const int b0 = start + b * RT;
        const int cnt = min(RT, end - b0);
        mbar_wait(&mbar[buf], (unsigned)((b >> 1) & 1));
        if ((int)threadIdx.x < cnt) {
            const float4 r0 = srec[buf][threadIdx.x][0], r1 = srec[buf][threadIdx.x][1];
            const float sb = srec[buf][threadIdx.x][2].z;
            smask[threadIdx.x] = (uint8_t)warp_block_mask(r0.x, r0.y, r0.z, r0.w, r1.x, sb, (float)(tx * TILE),
                                                          (float)(ty * TILE));
        }
        // masks ready, batch b−1's walk (buffer buf ^ 1) finished everywhere
        if (__syncthreads_count(T.x < 0.f && T.y < 0.f) == RT) break;  // nothing in flight here
        if (wl == 0 && b + 1 < nbat) {
            issue(b + 1);
            load_idx(b + 2);
        }
        const int jbase = b0 - start + 1;  // list index + 1 of batch entry 0
        const int nl = warp_batch_list(smask, cnt, wl, lane, slist[wl]);
        const float4(*rb)[TMA_ROW_FLOATS / 4] = srec[buf];
#pragma unroll(kFwdUnroll)
        for (int u = 0; u < nl && !(T.x < 0.f && T.y < 0.f); u++) {
            const int j = slist[wl][u];
            if (CNT) nev += (unsigned)(T.x > 0.f) + (unsigned)(T.y > 0.f);
            const float4 e0 = rb[j][0], e2 = rb[j][2];  // (x, y, A, B), (b, depth, sb, 1/o)
            const float Cc = rb[j][1].x;
            const float2 dx = __fadd2_rn(ff2(e0.x, e0.x), nfx);
            const float2 dy = __fadd2_rn(ff2(e0.y, e0.y), nfy);
            const float2 Adx = __fmul2_rn(ff2(e0.z, e0.z), dx);
            const float2 CdyDy = __fmul2_rn(__fmul2_rn(ff2(Cc, Cc), dy), dy);
            const float2 inner = __ffma2_rn(Adx, dx, CdyDy);
            const float2 nBdxdy = __fmul2_rn(__fmul2_rn(ff2(-e0.w, -e0.w), dx), dy);
            const float2 power = __ffma2_rn(mhalf, inner, nBdxdy);
            const bool in0 = T.x > 0.f && !(power.x > 0.f) && !(power.x < e2.z);
            const bool in1 = T.y > 0.f && !(power.y > 0.f) && !(power.y < e2.z);
            if (!(in0 || in1)) continue;
            if (CNT) nexp += (unsigned)in0 + (unsigned)in1;
            const float4 e1 = rb[j][1];  // (C, o, r, g)
            const float2 G = ca_exp_core2(power);
            const float2 oG = __fmul2_rn(ff2(e1.y, e1.y), G);
            const float2 alpha = ff2(fminf(ALPHA_MAX, oG.x), fminf(ALPHA_MAX, oG.y));
            const bool ok0 = in0 && !(alpha.x < ALPHA_MIN), ok1 = in1 && !(alpha.y < ALPHA_MIN);
            if (!(ok0 || ok1)) continue;
            const float2 Tn = __fmul2_rn(T, __ffma2_rn(alpha, mone, one));  // T·(1 − α), CA
            const bool term0 = ok0 && Tn.x < T_EPS, term1 = ok1 && Tn.y < T_EPS;
            const bool bl0 = ok0 && !term0, bl1 = ok1 && !term1;
            const float2 w = __fmul2_rn(ff2(bl0 ? alpha.x : 0.f, bl1 ? alpha.y : 0.f), T);
            C0 = __ffma2_rn(ff2(e1.z, e1.z), w, C0);
            C1 = __ffma2_rn(ff2(e1.w, e1.w), w, C1);
            C2 = __ffma2_rn(ff2(e2.x, e2.x), w, C2);
            if (DEPTH) D = __ffma2_rn(ff2(e2.y, e2.y), w, D);
            T = ff2(bl0 ? Tn.x : (term0 ? -T.x : T.x), bl1 ? Tn.y : (term1 ? -T.y : T.y));
            const int jn = jbase + j;
            last0 = bl0 ? jn : last0;
            last1 = bl1 ? jn : last1;
        }
    }
    if (CNT) count_evals(&L.counters64[0], &L.counters64[2], nev, nexp, sev);
    const int64_t HW = (int64_t)L.H * L.W;
    const float Cs[2][3] = {{C0.x, C1.x, C2.x}, {C0.y, C1.y, C2.y}};
    const float Ts[2] = {fabsf(T.x), fabsf(T.y)}, Ds[2] = {D.x, D.y};
    const int ls[2] = {last0, last1};
#pragma unroll
    for (int p = 0; p < 2; p++) {
        if (!(x < L.W && y[p] < L.H)) continue;
        const int64_t pix = (int64_t)y[p] * L.W + x;
        out_rgb[(3 * (int64_t)v + 0) * HW + pix] = __fmaf_rn(Ts[p], L.bg[0], Cs[p][0]);  // CA: fma(T, bg, C)
        out_rgb[(3 * (int64_t)v + 1) * HW + pix] = __fmaf_rn(Ts[p], L.bg[1], Cs[p][1]);
        out_rgb[(3 * (int64_t)v + 2) * HW + pix] = __fmaf_rn(Ts[p], L.bg[2], Cs[p][2]);
        out_T[v * HW + pix] = Ts[p];
        out_n[v * HW + pix] = ls[p];
        if (DEPTH) out_D[v * HW + pix] = Ds[p];
    }
}

bool encode_record_map(CUtensorMap* tm, const void* rec, int64_t cap_pairs) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
    }
    const cuuint64_t dims[2] = {12, (cuuint64_t)(cap_pairs > 0 ? cap_pairs : 1)};
    const cuuint64_t strides[1] = {48};
    const cuuint32_t box[2] = {TMA_ROW_FLOATS, 1}, es[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(rec), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_render_fwd(const Launch& L, float* rgb, float* Tf, int32_t* nc, float* depth, const CUtensorMap* tm,
                              cudaStream_t s) {
    if (tm) {
        if (depth)
            k_render_fwd_tma<true, true><<<L.V * L.T, RT, 0, s>>>(L, *tm, rgb, Tf, nc, depth);
        else if (L.count_evals)
            k_render_fwd_tma<false, true><<<L.V * L.T, RT, 0, s>>>(L, *tm, rgb, Tf, nc, nullptr);
        else
            k_render_fwd_tma<false, false><<<L.V * L.T, RT, 0, s>>>(L, *tm, rgb, Tf, nc, nullptr);
        return cudaGetLastError();
    }
    if (depth)
        k_render_fwd_p<true, true><<<L.V * L.T, RT, 0, s>>>(L, rgb, Tf, nc, depth);
    else if (L.count_evals)
        k_render_fwd_p<false, true><<<L.V * L.T, RT, 0, s>>>(L, rgb, Tf, nc, nullptr);
    else
        k_render_fwd_p<false, false><<<L.V * L.T, RT, 0, s>>>(L, rgb, Tf, nc, nullptr);
    return cudaGetLastError();
}

// Transpose-reduce of 10 per-lane values over a warp.  Level l (xor 16, 8, 4,
// 2, 1) halves the number of values each lane carries; the lane keeps the
// half selected by its bit and receives the partner's copy of that half.
// Returns the warp sum of value `id` (id computed once by reduce_id).  The
// keep/send choices are byte permutes driven by per-lane selector registers
// (sel: 0x3210 keeps the first operand, 0x7654 the second), computed once, so
// no predicate register has to stay live across the entry loop.
__device__ __forceinline__ float psel(float a, float b, uint32_t sel) {  // sel ? … : byte-permute select
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(sel));
    return __uint_as_float(d);
}
struct RedSel {
    uint32_t s16, s8, s4, s2;  // 0x7654 where the lane's bit is set (takes the second operand), else 0x3210
};
__device__ __forceinline__ RedSel red_sel(int lane) {
    RedSel r;
    r.s16 = (lane & 16) ? 0x7654u : 0x3210u;
    r.s8 = (lane & 8) ? 0x7654u : 0x3210u;
    r.s4 = (lane & 4) ? 0x7654u : 0x3210u;
    r.s2 = (lane & 2) ? 0x7654u : 0x3210u;
    return r;
}
__device__ __forceinline__ float warp_transpose_reduce10(const float (&v)[NG], const RedSel& rs) {
    float u[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
        const float keep = psel(v[k], v[k + 5], rs.s16);
        const float send = psel(v[k + 5], v[k], rs.s16);
        u[k] = keep + __shfl_xor_sync(FULLR, send, 16);
    }
    float w0 = psel(u[0], u[2], rs.s8) + __shfl_xor_sync(FULLR, psel(u[2], u[0], rs.s8), 8);
    float w1 = psel(u[1], u[3], rs.s8) + __shfl_xor_sync(FULLR, psel(u[3], u[1], rs.s8), 8);
    float w2 = u[4] + __shfl_xor_sync(FULLR, u[4], 8);
    float x0 = psel(w0, w1, rs.s4) + __shfl_xor_sync(FULLR, psel(w1, w0, rs.s4), 4);
    float x1 = w2 + __shfl_xor_sync(FULLR, w2, 4);
    float y = psel(x0, x1, rs.s2) + __shfl_xor_sync(FULLR, psel(x1, x0, rs.s2), 2);
    y += __shfl_xor_sync(FULLR, y, 1);
    return y;
}

__device__ __forceinline__ int reduce_id(int lane) {
    const int b16 = (lane & 16) ? 5 : 0;
    const bool b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
    const int w0 = b16 + (b8 ? 2 : 0), w1 = b16 + (b8 ? 3 : 1), w2 = b16 + 4;
    const int x0 = b4 ? w1 : w0, x1 = w2;
    return b2 ? x1 : x0;
}

// ---------------------------------------------------------------------------------------
// Backward (S7).  One warp per (view, tile, 8×8 pixel block), two pixels per lane held as the
// lanes of FP32x2 registers (rows r and r + WBH/2 of the lane's column in the block); the
// tile's list walked back to front from the block's largest n_contrib over the entries that
// can touch the block (§4.8).
//
// Decisions are the forward's, re-taken in the same canonical arithmetic: the CA power, the
// CA exp (ca_exp_core2, bit-identical to the forward's), α = min(0.99, o·G), skip α < 1/255,
// clamp o·G > 0.99 — so the set of blended (pixel, entry) pairs is exactly the forward's, and
// the gradient values use that same G (values are free, §4.4).  A pixel that does not blend
// the entry gets α = 0 and zero gradient weights, which leaves its state unchanged exactly.
//
// State per pixel: T (transmittance in front of the current entry, rebuilt by T/(1 − α)) and
// B̃ = −(T_final·(bg·∂L/∂C) + Σ_{k behind} (c_k·∂L/∂C)·α_k·T_k), so that
//     ∂L/∂α_j = T_j·(c_j·∂L/∂C) + B̃/(1 − α_j)
// (the adjoint of Eq. (1): every later term and the background carry (1 − α_j)), and
// after the entry B̃ −= (c_j·∂L/∂C)·α_j·T_j.  Per (pixel, entry) the ten per-pair terms are
// Σ∇x, Σ∇y (∇_{p_i}L in NDC, R2), ‖∇_{p_i}L‖ (E1, "norm and add"), ∂A, ∂B, ∂C, o·∂L/∂o,
// ∂r, ∂g, ∂b; the lane adds its two pixels', the warp transpose-reduces them (12 shuffles, each
// lane ends up owning one value's warp sum) and the ten owner lanes scale their sums and add
// them to the pair's gradient slot (one red.add warp instruction per entry: ten lanes of one
// 48-byte slot).
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------------------------------
// No warp of the backward ever waits for another.  Each warp stages its own batches of
// WB_BATCH entries of the tile's list (two per lane: pair slot, record, and the culling test of
// ITS pixel block only — cp.async brings batch b − 1's records while batch b is walked),
// compacts the entries that may touch its block, walks them, and flushes each entry's sums at
// once.  With one warp per CTA a finished warp frees its slot for the next.  Measured against
// the round-2 CTA-per-tile kernel (four warps sharing each staged batch, three CTA barriers per
// batch, per-warp slot arrays summed by a flush pass — barrier stalls 13 % of samples at garden,
// 27 % at playroom): garden 0.691 vs 0.691 ms, playroom 2.91 vs 3.23 ms, train 0.93 vs 1.04 ms.
// What it costs: each warp reads the records its list reaches (L2), and an entry walked by k
// warps of a tile gets k red.adds instead of one.
#ifndef MVGS_WB_BATCH
#define MVGS_WB_BATCH 64
#endif
constexpr int WB_BATCH = MVGS_WB_BATCH;  // entries a warp stages at a time (two per lane)

// warp_block_mask for one block: may a pixel of the WBW × WBH block at (x0, y0) pass the skip test?
__device__ __noinline__ bool block_may_pass(float px, float py, float A, float B, float C, float sb, float x0,
                                            float y0) {
#ifdef MVGS_NO_CULL
    return true;
#endif
    const float L = -2.0f * sb;
    if (!(A > 0.0f) || !(C > 0.0f) || !((double)A * (double)C - (double)B * (double)B > 0.0) || !(L > 0.0f))
        return true;
    const float eps3 = 3.0f * 8.0f * 5.9604644775390625e-8f;
    const float Lm = L * 1.01f + 0.01f;
    const float dxlo = px - (x0 + (float)(WBW - 1)), dxhi = px - x0;
    const float dylo = py - (y0 + (float)(WBH - 1)), dyhi = py - y0;
    const float dxm = fmaxf(fabsf(dxlo), fabsf(dxhi));
    const float dym = fmaxf(fabsf(dylo), fabsf(dyhi));
    float qmin = 0.0f;
    if (!(dxlo <= 0.0f && dxhi >= 0.0f && dylo <= 0.0f && dyhi >= 0.0f)) {
        const float nBoA = -B / A, nBoC = -B / C;
        qmin = fminf(fminf(q_edge(A, B, C, nBoA, nBoC, dxlo, dylo, dyhi, true),
                           q_edge(A, B, C, nBoA, nBoC, dxhi, dylo, dyhi, true)),
                     fminf(q_edge(A, B, C, nBoA, nBoC, dylo, dxlo, dxhi, false),
                           q_edge(A, B, C, nBoA, nBoC, dyhi, dxlo, dxhi, false)));
    }
    const float tmax = A * dxm * dxm + C * dym * dym + 2.0f * fabsf(B) * dxm * dym;
    return !(qmin > Lm + eps3 * tmax);
}

#ifndef MVGS_BWD_WPC
#define MVGS_BWD_WPC 1  // warps per CTA of the warp-independent backward (1: a finished warp frees its slot)
#endif
constexpr int BW_WPC = MVGS_BWD_WPC;
// L1: the ℓ1 loss fused in (mvgs_render_bwd_l1): `dL_drgb` is then the forward's image C and
// ∂L/∂C = scale·sign(C − t·fl(1/255)) is formed per pixel from the 8-bit target exactly as
// mvgs_loss_grad_u8 forms it; Σ|C − t/255| is added to *loss (one double atomic per warp).
template <bool CNT, bool L1>
__global__ __launch_bounds__(32 * BW_WPC, MVGS_BWD_MINB * 4 / BW_WPC) void k_render_bwd_w(
    Launch L, const float* __restrict__ dL_drgb, const float* __restrict__ in_T, const int32_t* __restrict__ in_n,
    const uint8_t* __restrict__ tgt, float scale, double* __restrict__ loss) {
    constexpr int NW = BW_WPC, MB = WB_BATCH, SPL = MB / 32;
    static_assert(MB % 32 == 0 && MB <= 256, "batch: lanes × SPL, byte list indices");
    __shared__ float4 se[NW][4][MB];  // per warp: (μ'x, μ'y, A, C) (B, o, sb, 1/o) (r, g, b, −) (W/2·A, W/2·B, H/2·C, H/2·B)
    __shared__ __align__(16) float4 sraw[NW][MB][3];  // per warp: the next batch's records, by cp.async
    __shared__ uint32_t sq[2][NW][MB];  // pair slots of the staged batch (two batches in flight)
    __shared__ uint8_t slist[NW][MB];
    __shared__ unsigned sev[2];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;  // wl: warp within the CTA
    const int gw = blockIdx.x * NW + wl;                       // the tile's four warps are consecutive
    const int warp = gw & 3;                                   // pixel block of the tile
    const int bucket = L.order ? L.order[gw >> 2] : (gw >> 2);
    const int v = bucket / L.T, tile = bucket - v * L.T;
    const int ty = tile / L.TX, tx = tile - ty * L.TX;
    const int x = tx * TILE + wb_x0(warp) + (lane % WBW);
    const int y0 = ty * TILE + wb_y0(warp) + (lane / WBW), y1_ = y0 + WBH / 2;
    const int start = L.bucket_off[bucket], end = L.bucket_off[bucket + 1];
    if (CNT && threadIdx.x == 0) sev[0] = sev[1] = 0;
    if (end > L.cap_entries) return;
    const int64_t HW = (int64_t)L.H * L.W;
    float dL[2][3], Tfin[2];
    int last[2];
    double lsum = 0.0;  // L1: Σ|C − t/255| over the lane's pixels
#pragma unroll
    for (int p = 0; p < 2; p++) {
        const int y = y0 + (WBH / 2) * p;
        dL[p][0] = dL[p][1] = dL[p][2] = 0.f;
        Tfin[p] = 1.f;
        last[p] = 0;
        if (x < L.W && y < L.H) {
            const int64_t pix = (int64_t)y * L.W + x;
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const int64_t i = (3 * (int64_t)v + c) * HW + pix;
                if (L1) {
                    const float d = dL_drgb[i] - __fmul_rn((float)tgt[i], 1.0f / 255.0f);
                    dL[p][c] = d > 0.f ? scale : (d < 0.f ? -scale : 0.f);
                    lsum += (double)fabsf(d);
                } else {
                    dL[p][c] = dL_drgb[i];
                }
            }
            Tfin[p] = in_T[v * HW + pix];
            last[p] = in_n[v * HW + pix];
        }
    }
    if (L1 && loss) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(FULLR, lsum, o);
        if (lane == 0) atomicAdd(loss, lsum);
    }
    const float2 dLr = f2(dL[0][0], dL[1][0]), dLg = f2(dL[0][1], dL[1][1]), dLb = f2(dL[0][2], dL[1][2]);
    float2 T = f2(Tfin[0], Tfin[1]);
    float2 nB = f2(-Tfin[0] * (L.bg[0] * dL[0][0] + L.bg[1] * dL[0][1] + L.bg[2] * dL[0][2]),
                   -Tfin[1] * (L.bg[0] * dL[1][0] + L.bg[1] * dL[1][1] + L.bg[2] * dL[1][2]));
    const float hw = 0.5f * (float)L.W, hh = 0.5f * (float)L.H;
    unsigned nev = 0, nexp = 0, nbl0 = 0, nbl1 = 0;
    const int wmax = __reduce_max_sync(FULLR, max(last[0], last[1]));
    const int my_id = reduce_id(lane);
    const bool owner = (__ffs(__match_any_sync(FULLR, my_id)) - 1) == lane;
    const RedSel rsel = red_sel(lane);
    // the owner lane's scale of its value: Σ∇ = −Σ (W/2·(A d + B e), H/2·(C e + B d)) (W/2, H/2 folded
    // into the staged conic) with d, e = ∂L/∂power·(dx, dy); ∂A = −½Σ d·dx, ∂B = −Σ d·dy, ∂C = −½Σ e·dy;
    // the colour terms were accumulated with −w; value 6 (o·∂L/∂o) takes the entry's 1/o
    const float myscale = (my_id == 0 || my_id == 1) ? -1.f
                          : (my_id == 3 || my_id == 5) ? -0.5f
                          : (my_id == 4 || my_id >= 7) ? -1.f
                                                       : 1.f;
    float* const pg = L.pgrad + my_id;
    const float2 nfx = f2(-(float)x, -(float)x), nfy = f2(-(float)y0, -(float)y1_);
    const float2 mhalf = f2(-0.5f, -0.5f);
    const float bx0 = (float)(tx * TILE + wb_x0(warp)), by0 = (float)(ty * TILE + wb_y0(warp));
    float4(*S)[MB] = se[wl];
    // Batches are walked back to front.  The records of batch bi − 1 travel global → shared by
    // cp.async (each lane copies the rows it will later transform, so only its own copies are
    // waited for) while batch bi is walked; the pair slots of batch bi − 2 are loaded meanwhile.
    const int nbat = (wmax + MB - 1) / MB;
    uint32_t qn[SPL];
    auto load_slots = [&](int bi) {
#pragma unroll
        for (int k = 0; k < SPL; k++) {
            const int t = lane + 32 * k;
            qn[k] = (bi >= 0 && bi * MB + t < wmax) ? L.sorted[start + bi * MB + t] : 0u;
        }
    };
    auto issue = [&](int bi) {  // batch bi's records → sraw, its slots → sq[bi & 1]
#pragma unroll
        for (int k = 0; k < SPL; k++) {
            const int t = lane + 32 * k;
            if (bi * MB + t < wmax) {
                sq[bi & 1][wl][t] = qn[k];
                const float* src = reinterpret_cast<const float*>(L.rec + 3 * (int64_t)qn[k]);
                cp_async16(&sraw[wl][t][0].x, src);
                cp_async16(&sraw[wl][t][1].x, src + 4);
                cp_async16(&sraw[wl][t][2].x, src + 8);
            }
        }
        cp_async_commit();
    };
    if (nbat > 0) {
        load_slots(nbat - 1);
        issue(nbat - 1);
        load_slots(nbat - 2);
    }
    for (int bi = nbat - 1; bi >= 0; bi--) {
        const int b0 = bi * MB;
        const int cnt = min(MB, wmax - b0);
        const uint32_t* sqb = sq[bi & 1][wl];
        cp_async_wait_all();
        __syncwarp();  // the previous batch's staged entries are no longer read
        unsigned inb[SPL];
#pragma unroll
        for (int k = 0; k < SPL; k++) {
            const int t = lane + 32 * k;
            bool in = false;
            if (t < cnt) {
                const float4 r0 = sraw[wl][t][0], r1 = sraw[wl][t][1], r2 = sraw[wl][t][2];
                // (x, y, A, B) (C, o, r, g) (b, depth, sb, 1/o)
                S[0][t] = make_float4(r0.x, r0.y, r0.z, r1.x);
                S[1][t] = make_float4(r0.w, r1.y, r2.z, r2.w);
                S[2][t] = make_float4(r1.z, r1.w, r2.x, 0.f);
                S[3][t] = make_float4(hw * r0.z, hw * r0.w, hh * r1.x, hh * r0.w);
                in = block_may_pass(r0.x, r0.y, r0.z, r0.w, r1.x, r2.z, bx0, by0);
            }
            inb[k] = __ballot_sync(FULLR, in);
        }
        if (bi > 0) {  // the next batch in flight during this batch's walk
            issue(bi - 1);
            load_slots(bi - 2);
        }
        int nl = 0;
#pragma unroll
        for (int k = 0; k < SPL; k++) {
            if ((inb[k] >> lane) & 1u) slist[wl][nl + __popc(inb[k] & ((1u << lane) - 1u))] = (uint8_t)(lane + 32 * k);
            nl += __popc(inb[k]);
        }
        __syncwarp();
        auto front = [&](int jj, int j, float2& dx, float2& dy, float2& power, bool& in0, bool& in1) {
            const float4 e0 = S[0][jj], e1 = S[1][jj];
            dx = __fadd2_rn(f2(e0.x, e0.x), nfx);
            dy = __fadd2_rn(f2(e0.y, e0.y), nfy);
            const float2 A2 = f2(e0.z, e0.z), C2 = f2(e0.w, e0.w), B2 = f2(e1.x, e1.x);
            const float2 inner = __ffma2_rn(__fmul2_rn(A2, dx), dx, __fmul2_rn(__fmul2_rn(C2, dy), dy));
            const float2 Bdd = __fmul2_rn(__fmul2_rn(B2, dx), dy);
            power = __ffma2_rn(mhalf, inner, f2(-Bdd.x, -Bdd.y));
            const float sb = e1.z;
            in0 = j < last[0] && !(power.x > 0.f) && !(power.x < sb);
            in1 = j < last[1] && !(power.y > 0.f) && !(power.y < sb);
        };
        auto alphas = [&](int jj, float2 power, bool in0, bool in1, float2& alpha, float2& oGc) -> bool {
            const float o = S[1][jj].y;
            const float2 G = ca_exp_core2(power);
            const float2 oG = __fmul2_rn(f2(o, o), G);
            const bool bl0 = in0 && !(oG.x < ALPHA_MIN);
            const bool bl1 = in1 && !(oG.y < ALPHA_MIN);
            if (CNT) {
                nbl0 += bl0;
                nbl1 += bl1;
            }
            alpha = f2(bl0 ? fminf(ALPHA_MAX, oG.x) : 0.f, bl1 ? fminf(ALPHA_MAX, oG.y) : 0.f);
            oGc = f2(oG.x > ALPHA_MAX ? 0.f : alpha.x, oG.y > ALPHA_MAX ? 0.f : alpha.y);
            return bl0 || bl1;  // the lane blends the entry at one of its pixels
        };
        auto state = [&](int jj, float2 alpha, float2 oGc, float2& nw, float2& dLdpw) {
            const float2 om = __ffma2_rn(alpha, f2(-1.f, -1.f), f2(1.f, 1.f));
            const float2 inv = f2(rcp_approx(om.x), rcp_approx(om.y));
            T = __fmul2_rn(T, inv);
            nw = __fmul2_rn(alpha, f2(-T.x, -T.y));
            const float4 e2 = S[2][jj];
            const float2 cdL = __ffma2_rn(f2(e2.z, e2.z), dLb,
                                          __ffma2_rn(f2(e2.y, e2.y), dLg, __fmul2_rn(f2(e2.x, e2.x), dLr)));
            const float2 dLda = __ffma2_rn(nB, inv, __fmul2_rn(T, cdL));
            nB = __ffma2_rn(cdL, nw, nB);
            dLdpw = __fmul2_rn(oGc, dLda);
        };
        auto terms = [&](int jj, float2 dx, float2 dy, float2 nw, float2 dLdpw, float (&val)[NG]) {
            const float4 s3 = S[3][jj];
            const float2 d = __fmul2_rn(dLdpw, dx), e = __fmul2_rn(dLdpw, dy);
            const float2 gxr = __ffma2_rn(f2(s3.x, s3.x), d, __fmul2_rn(f2(s3.y, s3.y), e));
            const float2 gyr = __ffma2_rn(f2(s3.z, s3.z), e, __fmul2_rn(f2(s3.w, s3.w), d));
            const float2 n2 = __ffma2_rn(gxr, gxr, __fmul2_rn(gyr, gyr));
            const float2 dd = __fmul2_rn(d, dx), de = __fmul2_rn(d, dy), ee = __fmul2_rn(e, dy);
            const float2 wr = __fmul2_rn(nw, dLr), wg = __fmul2_rn(nw, dLg), wb = __fmul2_rn(nw, dLb);
            val[0] = gxr.x + gxr.y;
            val[1] = gyr.x + gyr.y;
            val[2] = sqrt_approx(n2.x) + sqrt_approx(n2.y);
            val[3] = dd.x + dd.y;
            val[4] = de.x + de.y;
            val[5] = ee.x + ee.y;
            val[6] = dLdpw.x + dLdpw.y;
            val[7] = wr.x + wr.y;
            val[8] = wg.x + wg.y;
            val[9] = wb.x + wb.y;
        };
        // the owner lanes add the entry's warp sums to its gradient slot
        auto flush = [&](int jj, float s) {
            if (owner) atomicAdd(pg + (int64_t)sqb[jj] * PG_STRIDE, s * (my_id == 6 ? S[1][jj].w : myscale));
        };
        int u = nl - 1;
#if MVGS_BWD_PAIR
        for (; u >= 1; u -= 2) {
            const int ja = slist[wl][u], jb = slist[wl][u - 1];  // a is behind b: a first
            if (CNT) nev += (unsigned)(b0 + ja < last[0]) + (unsigned)(b0 + ja < last[1]) +
                            (unsigned)(b0 + jb < last[0]) + (unsigned)(b0 + jb < last[1]);
            float2 dxa, dya, pwa, dxb, dyb, pwb;
            bool ia0, ia1, ib0, ib1;
            front(ja, b0 + ja, dxa, dya, pwa, ia0, ia1);
            front(jb, b0 + jb, dxb, dyb, pwb, ib0, ib1);
            if (!__any_sync(FULLR, ia0 || ia1 || ib0 || ib1)) continue;
            if (CNT) nexp += (unsigned)ia0 + (unsigned)ia1 + (unsigned)ib0 + (unsigned)ib1;
            float2 ala, oga, alb, ogb;
            const bool bla = alphas(ja, pwa, ia0, ia1, ala, oga);
            const bool blb = alphas(jb, pwb, ib0, ib1, alb, ogb);
            if (!__any_sync(FULLR, bla || blb)) continue;
            float2 nwa, dpa, nwb, dpb;
            state(ja, ala, oga, nwa, dpa);
            state(jb, alb, ogb, nwb, dpb);
            float va[NG], vb[NG];
            terms(ja, dxa, dya, nwa, dpa, va);
            terms(jb, dxb, dyb, nwb, dpb, vb);
            const float sa = warp_transpose_reduce10(va, rsel);
            const float sbv = warp_transpose_reduce10(vb, rsel);
            flush(ja, sa);
            flush(jb, sbv);
        }
#endif
        for (; u >= 0; u--) {
            const int jj = slist[wl][u];
            const int j = b0 + jj;
            if (CNT) nev += (unsigned)(j < last[0]) + (unsigned)(j < last[1]);
            float2 dx, dy, power;
            bool in0, in1;
            front(jj, j, dx, dy, power, in0, in1);
            if (!__any_sync(FULLR, in0 || in1)) continue;
            if (CNT) nexp += (unsigned)in0 + (unsigned)in1;
            float2 alpha, oGc;
            if (!__any_sync(FULLR, alphas(jj, power, in0, in1, alpha, oGc))) continue;
            float2 nw, dLdpw;
            state(jj, alpha, oGc, nw, dLdpw);
            float val[NG];
            terms(jj, dx, dy, nw, dLdpw, val);
            flush(jj, warp_transpose_reduce10(val, rsel));
        }
    }
    if (CNT) {
        __syncthreads();
        count_evals(&L.counters64[1], &L.counters64[3], nev, nexp, sev);
        if (L.dbg_nblend) {  // parity export: entries blended per pixel, as this kernel decided
            const int yy[2] = {y0, y1_};
            const unsigned nb[2] = {nbl0, nbl1};
#pragma unroll
            for (int p = 0; p < 2; p++)
                if (x < L.W && yy[p] < L.H) L.dbg_nblend[v * HW + (int64_t)yy[p] * L.W + x] = (int32_t)nb[p];
        }
    }
}

cudaError_t launch_render_bwd(const Launch& L, const float* dL, const float* Tf, const int32_t* nc, cudaStream_t s) {
    const int nb = L.V * L.T * (4 / BW_WPC);
    if (L.count_evals || L.dbg_nblend)
        k_render_bwd_w<true, false><<<nb, 32 * BW_WPC, 0, s>>>(L, dL, Tf, nc, nullptr, 0.f, nullptr);
    else
        k_render_bwd_w<false, false><<<nb, 32 * BW_WPC, 0, s>>>(L, dL, Tf, nc, nullptr, 0.f, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_render_bwd_l1(const Launch& L, const float* rgb, const uint8_t* tgt, float scale, const float* Tf,
                                 const int32_t* nc, double* loss, cudaStream_t s) {
    const int nb = L.V * L.T * (4 / BW_WPC);
    if (L.count_evals || L.dbg_nblend)
        k_render_bwd_w<true, true><<<nb, 32 * BW_WPC, 0, s>>>(L, rgb, Tf, nc, tgt, scale, loss);
    else
        k_render_bwd_w<false, true><<<nb, 32 * BW_WPC, 0, s>>>(L, rgb, Tf, nc, tgt, scale, loss);
    return cudaGetLastError();
}

}  // namespace mvgs
