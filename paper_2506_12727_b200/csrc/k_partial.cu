// k_partial.cu — NEXT-1: partial rendering (Alg. 3).
//
// Each (view, tile) renders only the S pixels of its index array A (pix), one
// pixel per thread.  Two launch shapes:
//   thread-efficient (Alg. 3): a block of ⌈S/32⌉·32 threads per (view, tile) —
//     "multiple blocks that have exactly the same number of threads as the number
//     of sub-sampled pixels, with each block allocated to each viewpoint";
//   masked (the paper's naive baseline): a 256-thread block per
//     (view, tile); threads whose pixel is not listed are masked off and wait.
// The per-pixel arithmetic is that of k_render.cu (CA decisions, exact skip
// bound), so listed pixels get exactly the full render's n_contrib.  Records are
// staged RB at a time, each thread loading RB/blockDim of them.
#include "ca.cuh"
#include "internal.cuh"

namespace mvgs {

constexpr int PRB = 128;  // entries per staged batch
constexpr unsigned FULLP = 0xffffffffu;

__device__ __forceinline__ float skip_power_p(float o) { return -logf(255.0f * o) - 1e-3f; }

__device__ __forceinline__ void stage_p(const Launch& L, uint32_t q, float4* s0, float4* s1, float4* s2, int i) {
    const float4* r = L.rec + 3 * (int64_t)q;
    const float4 r0 = r[0], r1 = r[1], r2 = r[2];
    s0[i] = r0;
    s1[i] = make_float4(r1.x, r1.y, skip_power_p(r1.y), 0.f);
    s2[i] = make_float4(r1.z, r1.w, r2.x, 0.f);
}

// slot (0..S-1) of this thread's pixel and its local index; −1 when masked off / idle
template <bool MASKED>
__device__ __forceinline__ void my_pixel(const int32_t* __restrict__ pix, int64_t base, int S, int* slot_of, int& slot,
                                         int& local) {
    if (MASKED) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) slot_of[i] = -1;
        __syncthreads();
        for (int s = threadIdx.x; s < S; s += blockDim.x) {
            const int l = pix[base + s];
            if (l >= 0 && l < 256) slot_of[l] = s;
        }
        __syncthreads();
        local = threadIdx.x;
        slot = slot_of[local];
    } else {
        slot = threadIdx.x < S ? (int)threadIdx.x : -1;
        local = slot >= 0 ? pix[base + slot] : -1;
        if (local < 0 || local >= 256) slot = -1;
    }
}

template <bool MASKED>
__global__ __launch_bounds__(256) void k_render_fwd_list(Launch L, const int32_t* __restrict__ pix, int S,
                                                         float* __restrict__ out_rgb, float* __restrict__ out_T,
                                                         int32_t* __restrict__ out_n) {
    __shared__ float4 s0[PRB], s1[PRB], s2[PRB];
    __shared__ int slot_of[256];
    zero_pgrad_slice(L);
    const int bucket = blockIdx.x;
    const int tile = bucket % L.T;
    const int ty = tile / L.TX, tx = tile - ty * L.TX;
    const int64_t base = (int64_t)bucket * S;
    int slot, local;
    my_pixel<MASKED>(pix, base, S, slot_of, slot, local);
    const int x = tx * TILE + (local & 15), y = ty * TILE + (local >> 4);
    const bool valid = slot >= 0 && x < L.W && y < L.H;
    const int start = L.bucket_off[bucket], end = L.bucket_off[bucket + 1];
    const float fx = (float)x, fy = (float)y;
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
    int last = 0;
    bool done = !valid;
    // occupancy statistics: threads launched / with a pixel, and lane-steps of
    // the entry walk executed by each warp (32 × its longest lane per batch) / spent on a live pixel
    const int nact = __syncthreads_count(valid);
    unsigned long long wsteps = 0, my_steps = 0;
    if (end <= L.cap_entries) {
        for (int b0 = start; b0 < end; b0 += PRB) {
            if (__syncthreads_count(done) == (int)blockDim.x) break;
            for (int t = threadIdx.x; t < PRB && b0 + t < end; t += blockDim.x) stage_p(L, L.sorted[b0 + t], s0, s1, s2, t);
            __syncthreads();
            const int cnt = min(PRB, end - b0);
            int bsteps = 0;
            for (int j = 0; j < cnt && !done; j++) {
                bsteps++;
                const float4 a = s0[j];
                const float4 c = s1[j];
                const float dx = FSUB(a.x, fx), dy = FSUB(a.y, fy);
                const float power = ca_power(a.z, a.w, c.x, dx, dy);
                if (power > 0.0f || power < c.z) continue;
                const float G = ca_exp_core(power);
                const float alpha = fminf(ALPHA_MAX, FMUL(c.y, G));
                if (alpha < ALPHA_MIN) continue;
                const float Tn = FMUL(T, FSUB(1.0f, alpha));
                if (Tn < T_EPS) {
                    done = true;
                    break;
                }
                const float w = FMUL(alpha, T);  // CA: C = fma(rgb, α·T, C)
                const float4 col = s2[j];
                C0 = __fmaf_rn(col.x, w, C0);
                C1 = __fmaf_rn(col.y, w, C1);
                C2 = __fmaf_rn(col.z, w, C2);
                T = Tn;
                last = b0 - start + j + 1;
            }
            my_steps += (unsigned long long)bsteps;
            wsteps += (unsigned long long)__reduce_max_sync(0xffffffffu, (unsigned)bsteps);
        }
    }
    {
        unsigned long long ms = my_steps;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&L.counters64[7], 32ull * wsteps);
            atomicAdd(&L.counters64[8], ms);
        }
        if (threadIdx.x == 0) {
            atomicAdd(&L.counters64[5], (unsigned long long)blockDim.x);
            atomicAdd(&L.counters64[6], (unsigned long long)nact);
        }
    }
    if (slot >= 0) {
        const int64_t o = base + slot;
        out_rgb[3 * o + 0] = __fmaf_rn(T, L.bg[0], C0);
        out_rgb[3 * o + 1] = __fmaf_rn(T, L.bg[1], C1);
        out_rgb[3 * o + 2] = __fmaf_rn(T, L.bg[2], C2);
        out_T[o] = T;
        out_n[o] = valid ? last : 0;
    }
}

// Transpose-reduce of 10 per-lane values over a warp (as in k_render.cu).
__device__ __forceinline__ float warp_reduce10_p(const float (&v)[NG], int lane) {
    const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
    float u[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
        const float keep = b16 ? v[k + 5] : v[k];
        const float send = b16 ? v[k] : v[k + 5];
        u[k] = keep + __shfl_xor_sync(FULLP, send, 16);
    }
    float w0 = (b8 ? u[2] : u[0]) + __shfl_xor_sync(FULLP, b8 ? u[0] : u[2], 8);
    float w1 = (b8 ? u[3] : u[1]) + __shfl_xor_sync(FULLP, b8 ? u[1] : u[3], 8);
    float w2 = u[4] + __shfl_xor_sync(FULLP, u[4], 8);
    float x0 = (b4 ? w1 : w0) + __shfl_xor_sync(FULLP, b4 ? w0 : w1, 4);
    float x1 = w2 + __shfl_xor_sync(FULLP, w2, 4);
    float y = (b2 ? x1 : x0) + __shfl_xor_sync(FULLP, b2 ? x0 : x1, 2);
    y += __shfl_xor_sync(FULLP, y, 1);
    return y;
}

__device__ __forceinline__ int reduce_id_p(int lane) {
    const int b16 = (lane & 16) ? 5 : 0;
    const bool b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
    const int w0 = b16 + (b8 ? 2 : 0), w1 = b16 + (b8 ? 3 : 1), w2 = b16 + 4;
    const int x0 = b4 ? w1 : w0, x1 = w2;
    return b2 ? x1 : x0;
}

template <bool MASKED>
__global__ __launch_bounds__(256) void k_render_bwd_list(Launch L, const int32_t* __restrict__ pix, int S,
                                                         const float* __restrict__ dL_drgb,
                                                         const float* __restrict__ in_T,
                                                         const int32_t* __restrict__ in_n) {
    __shared__ float4 s0[PRB], s1[PRB], s2[PRB];
    __shared__ uint32_t sq[PRB];
    __shared__ int slot_of[256];
    __shared__ int smax;
    extern __shared__ __align__(16) float sacc_p[];  // [warps][PRB·NG] per-warp partial sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int bucket = blockIdx.x;
    const int tile = bucket % L.T;
    const int ty = tile / L.TX, tx = tile - ty * L.TX;
    const int64_t base = (int64_t)bucket * S;
    int slot, local;
    my_pixel<MASKED>(pix, base, S, slot_of, slot, local);
    const int x = tx * TILE + (local & 15), y = ty * TILE + (local >> 4);
    const bool valid = slot >= 0 && x < L.W && y < L.H;
    const int start = L.bucket_off[bucket], end = L.bucket_off[bucket + 1];
    if (end > L.cap_entries) return;
    float dL0 = 0.f, dL1 = 0.f, dL2 = 0.f, T_fin = 1.f;
    int last = 0;
    if (valid) {
        const int64_t o = base + slot;
        dL0 = dL_drgb[3 * o + 0];
        dL1 = dL_drgb[3 * o + 1];
        dL2 = dL_drgb[3 * o + 2];
        T_fin = in_T[o];
        last = in_n[o];
    }
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
    if (last > 0) atomicMax(&smax, last);
    __syncthreads();
    const int maxlast = smax;
    const int wmax = __reduce_max_sync(FULLP, last);
    const int my_id = reduce_id_p(lane);
    const bool owner = (__ffs(__match_any_sync(FULLP, my_id)) - 1) == lane;
    float* wacc = sacc_p + warp * PRB * NG;
    const float fx = (float)x, fy = (float)y;
    const float hw = 0.5f * (float)L.W, hh = 0.5f * (float)L.H;
    const float dL_bg = L.bg[0] * dL0 + L.bg[1] * dL1 + L.bg[2] * dL2;
    float T = T_fin;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, a_prev = 0.f, c0p = 0.f, c1p = 0.f, c2p = 0.f;
    for (int b_end = maxlast; b_end > 0; b_end -= PRB) {
        const int b0 = max(0, b_end - PRB);
        const int cnt = b_end - b0;
        __syncthreads();
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
            const uint32_t q = L.sorted[start + b0 + t];
            sq[t] = q;
            stage_p(L, q, s0, s1, s2, t);
        }
        {
            float4* w4 = reinterpret_cast<float4*>(wacc);
            for (int i = lane; i < PRB * NG / 4; i += 32) w4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        for (int jj = min(cnt, wmax - b0) - 1; jj >= 0; jj--) {
            const int j = b0 + jj;
            float val[NG];
#pragma unroll
            for (int k = 0; k < NG; k++) val[k] = 0.f;
            bool contrib = false;
            if (j < last) {
                const float4 a = s0[jj];
                const float4 c = s1[jj];
                const float dx = FSUB(a.x, fx), dy = FSUB(a.y, fy);
                const float power = ca_power(a.z, a.w, c.x, dx, dy);
                if (power <= 0.0f && power >= c.z) {
                    const float G = ca_exp_core(power);
                    const float oG = FMUL(c.y, G);
                    const float alpha = fminf(ALPHA_MAX, oG);
                    if (alpha >= ALPHA_MIN) {
                        contrib = true;
                        const float inv_one_m = __fdividef(1.0f, 1.0f - alpha);
                        T = T * inv_one_m;
                        const float w = alpha * T;
                        const float4 col = s2[jj];
                        acc0 = a_prev * c0p + (1.f - a_prev) * acc0;
                        acc1 = a_prev * c1p + (1.f - a_prev) * acc1;
                        acc2 = a_prev * c2p + (1.f - a_prev) * acc2;
                        float dLda = (col.x - acc0) * dL0 + (col.y - acc1) * dL1 + (col.z - acc2) * dL2;
                        dLda = dLda * T - T_fin * inv_one_m * dL_bg;
                        a_prev = alpha;
                        c0p = col.x; c1p = col.y; c2p = col.z;
                        const bool clamped = oG > ALPHA_MAX;
                        const float dLdG = clamped ? 0.f : c.y * dLda;
                        const float dLdo = clamped ? 0.f : G * dLda;
                        const float dLdpw = G * dLdG;
                        const float gx = dLdpw * -(a.z * dx + a.w * dy) * hw;
                        const float gy = dLdpw * -(c.x * dy + a.w * dx) * hh;
                        val[0] = gx;
                        val[1] = gy;
                        const float n2 = gx * gx + gy * gy;
                        val[2] = n2 > 0.f ? n2 * rsqrtf(n2) : 0.f;
                        val[3] = -0.5f * dLdpw * dx * dx;
                        val[4] = -dLdpw * dx * dy;
                        val[5] = -0.5f * dLdpw * dy * dy;
                        val[6] = dLdo;
                        val[7] = w * dL0;
                        val[8] = w * dL1;
                        val[9] = w * dL2;
                    }
                }
            }
            if (__any_sync(FULLP, contrib)) {
                const float sum = warp_reduce10_p(val, lane);
                if (owner) wacc[jj * NG + my_id] = sum;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < cnt * NG; i += blockDim.x) {
            float s = 0.f;
            for (int w = 0; w < nw; w++) s += sacc_p[w * PRB * NG + i];
            if (s != 0.f) {
                const int jj = i / NG, k = i - jj * NG;
                atomicAdd(&L.pgrad[(int64_t)sq[jj] * PG_STRIDE + k], s);
            }
        }
    }
}

static int partial_threads(int S, int mode) { return mode == MVGS_PARTIAL_MASKED ? 256 : ((S + 31) / 32) * 32; }

cudaError_t launch_render_fwd_partial(const Launch& L, const int32_t* pix, int S, int mode, float* rgb, float* Tf,
                                      int32_t* nc, cudaStream_t s) {
    const int nt = partial_threads(S, mode);
    if (mode == MVGS_PARTIAL_MASKED)
        k_render_fwd_list<true><<<L.V * L.T, nt, 0, s>>>(L, pix, S, rgb, Tf, nc);
    else
        k_render_fwd_list<false><<<L.V * L.T, nt, 0, s>>>(L, pix, S, rgb, Tf, nc);
    return cudaGetLastError();
}

cudaError_t launch_render_bwd_partial(const Launch& L, const int32_t* pix, int S, int mode, const float* dL,
                                      const float* Tf, const int32_t* nc, cudaStream_t s) {
    const int nt = partial_threads(S, mode);
    const size_t smem = sizeof(float) * (nt / 32) * PRB * NG;
    cudaError_t e;
    if (mode == MVGS_PARTIAL_MASKED) {
        if ((e = cudaFuncSetAttribute(k_render_bwd_list<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
            cudaSuccess)
            return e;
        k_render_bwd_list<true><<<L.V * L.T, nt, smem, s>>>(L, pix, S, dL, Tf, nc);
    } else {
        if ((e = cudaFuncSetAttribute(k_render_bwd_list<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
            cudaSuccess)
            return e;
        k_render_bwd_list<false><<<L.V * L.T, nt, smem, s>>>(L, pix, S, dL, Tf, nc);
    }
    return cudaGetLastError();
}

}  // namespace mvgs
