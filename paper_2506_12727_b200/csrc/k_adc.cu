// k_adc.cu — NEXT-3: the multi-view adaptive density control step (P:4).
//
// One event is three passes over the P Gaussians, all HBM-bound streaming:
//   k_adc_decide   per Gaussian: split / clone decisions from the running means Ē = E/denom
//                  (E1 for splitting, E2 for cloning; E_old in single-view mode), the prune
//                  test of every row it would emit, and its emitted-row count c_g ∈ [0, 2 + N];
//                  warp-aggregated report counters.
//   scan           exclusive scan of c_g (shared with preprocess, k_preprocess.cu) → output offsets
//                  in canonical order (g ascending; kept, clone, children).
//   k_adc_emit     per Gaussian: writes its rows — scalars per thread, split children
//                  mean + R(q̂)(s ⊙ n_k) (3DGS's sampling from the parent's density), and the SH
//                  rows copied warp-cooperatively (coalesced 128-B segments, one read per
//                  parent, c_g writes).
//   k_adc_remap    optimiser-state resize: kept rows gathered, new rows zero.
// Decisions in fp32 with IEEE division (__fdiv_rn) and host-rounded thresholds, the same
// precision the oracle (oracle/adc.py) decides in.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.cuh"

namespace mvgs {

struct AdcParams {
    float tau_split, tau_clone, ln_size, ln_split, logit_prune, ln_prune_scale;
    int N, mode;
};

constexpr int ADC_EMIT_T = 256;
enum : uint8_t { F_SPLIT = 1, F_CLONE = 2, F_KEEP_ALIVE = 4, F_CLONE_ALIVE = 8, F_CHILD_ALIVE = 16 };

__device__ __forceinline__ float adc_mean(const float e, const float den) {
    return den > 0.f ? __fdiv_rn(e, den) : 0.f;
}

__global__ __launch_bounds__(1024) void k_adc_decide(int64_t P, const float* __restrict__ log_scales,
                                                    const float* __restrict__ opacity_logits, mvgs_adc_accum acc,
                                                    AdcParams prm, int* __restrict__ cnt, uint8_t* __restrict__ flags,
                                                    unsigned long long* __restrict__ rep) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int c = 0, n_split = 0, n_clone = 0, n_pruned = 0;
    if (g < P) {
        // all loads issued up front (no load behind a branch on another load)
        const float den = acc.denom_acc[g];
        const float es = (prm.mode ? acc.e1_acc : acc.e_old_acc)[g];
        const float ec = (prm.mode ? acc.e2_acc : acc.e_old_acc)[g];
        const float ol = opacity_logits[g];
        const float l0 = log_scales[3 * g], l1 = log_scales[3 * g + 1], l2 = log_scales[3 * g + 2];
        const float lmax = fmaxf(fmaxf(l0, l1), l2);
        const bool large = lmax > prm.ln_size;
        const float ms = adc_mean(es, den);
        const float mc = adc_mean(ec, den);
        const bool split = ms >= prm.tau_split && large;
        const bool clone = mc >= prm.tau_clone && !large;
        const bool op_pruned = ol < prm.logit_prune;
        // fl(l − c) is monotone in l, so the children's max log-scale is fl(lmax − c)
        const bool keep_alive = !split && !op_pruned && !(lmax > prm.ln_prune_scale);
        const bool clone_alive = clone && !op_pruned && !(lmax > prm.ln_prune_scale);
        const bool child_alive = split && !op_pruned && !(__fsub_rn(lmax, prm.ln_split) > prm.ln_prune_scale);
        c = (int)keep_alive + (int)clone_alive + (child_alive ? prm.N : 0);
        flags[g] = (split ? F_SPLIT : 0) | (clone ? F_CLONE : 0) | (keep_alive ? F_KEEP_ALIVE : 0) |
                   (clone_alive ? F_CLONE_ALIVE : 0) | (child_alive ? F_CHILD_ALIVE : 0);
        cnt[g] = c;
        n_split = split;
        n_clone = clone;
        n_pruned = (int)(!split) + (int)clone + (split ? prm.N : 0) - c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_split += __shfl_xor_sync(0xffffffffu, n_split, o);
        n_clone += __shfl_xor_sync(0xffffffffu, n_clone, o);
        n_pruned += __shfl_xor_sync(0xffffffffu, n_pruned, o);
    }
    // block reduce, then one atomic per counter per CTA (same-address atomics serialise in L2)
    __shared__ int red[3][32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[0][w] = n_split, red[1][w] = n_clone, red[2][w] = n_pruned;
    __syncthreads();
    if (threadIdx.x < 3) {
        int t = 0;
#pragma unroll
        for (int k = 0; k < 32; k++) t += red[threadIdx.x][k];
        if (t) atomicAdd(rep + threadIdx.x, (unsigned long long)t);
    }
}

__device__ __forceinline__ void put_row(const mvgs_gaussians& in, const mvgs_gaussians_out& out, int64_t g,
                                        int64_t o, const float m[3], const float ls[3]) {
    out.means[3 * o] = m[0], out.means[3 * o + 1] = m[1], out.means[3 * o + 2] = m[2];
    out.log_scales[3 * o] = ls[0], out.log_scales[3 * o + 1] = ls[1], out.log_scales[3 * o + 2] = ls[2];
    const float4 q = reinterpret_cast<const float4*>(in.quats)[g];
    reinterpret_cast<float4*>(out.quats)[o] = q;
    out.opacity_logits[o] = in.opacity_logits[g];
}

__global__ __launch_bounds__(ADC_EMIT_T) void k_adc_emit(mvgs_gaussians in, const uint8_t* __restrict__ flags,
                                                  const int* __restrict__ offs, const float* __restrict__ noise,
                                                  AdcParams prm, mvgs_gaussians_out out, int32_t* __restrict__ origin,
                                                  uint8_t* __restrict__ kind) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int off = 0, c = 0;
    if (g < in.P) {
        const uint8_t f = flags[g];
        off = offs[g];
        int o = off;
        const float m[3] = {in.means[3 * g], in.means[3 * g + 1], in.means[3 * g + 2]};
        const float ls[3] = {in.log_scales[3 * g], in.log_scales[3 * g + 1], in.log_scales[3 * g + 2]};
        if (f & F_KEEP_ALIVE) {
            put_row(in, out, g, o, m, ls);
            origin[o] = (int32_t)g, kind[o] = 0, o++;
        }
        if (f & F_CLONE_ALIVE) {
            put_row(in, out, g, o, m, ls);
            origin[o] = (int32_t)g, kind[o] = 1, o++;
        }
        if (f & F_CHILD_ALIVE) {
            // R(q̂), q = (w, x, y, z) normalised; s = exp(log_scale)
            const float4 q4 = reinterpret_cast<const float4*>(in.quats)[g];
            const float inv = rsqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
            const float w = q4.x * inv, x = q4.y * inv, y = q4.z * inv, z = q4.w * inv;
            const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                                2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                                2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
            const float s[3] = {expf(ls[0]), expf(ls[1]), expf(ls[2])};
            const float cls[3] = {__fsub_rn(ls[0], prm.ln_split), __fsub_rn(ls[1], prm.ln_split),
                                  __fsub_rn(ls[2], prm.ln_split)};
            for (int k = 0; k < prm.N; k++) {
                const float* n = noise + ((int64_t)g * prm.N + k) * 3;
                const float a0 = s[0] * n[0], a1 = s[1] * n[1], a2 = s[2] * n[2];
                const float cm[3] = {m[0] + (R[0] * a0 + R[1] * a1 + R[2] * a2),
                                     m[1] + (R[3] * a0 + R[4] * a1 + R[5] * a2),
                                     m[2] + (R[6] * a0 + R[7] * a1 + R[8] * a2)};
                put_row(in, out, g, o, cm, cls);
                origin[o] = (int32_t)g, kind[o] = 2, o++;
            }
        }
        c = o - off;
    }
    // SH rows.  The CTA's output rows are one contiguous span (offsets are an exclusive scan), so
    // build a row → parent map in shared memory and copy the span flat: coalesced reads of the
    // parents' rows (repeats hit L1) and fully coalesced writes, float4 when the rows allow.
    __shared__ int o_first;
    __shared__ uint8_t rmap[ADC_EMIT_T * 10];  // ≤ (2 + N) rows per parent, N ≤ 8
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    if (threadIdx.x == 0) o_first = offs[g0];
    __syncthreads();
    for (int k = 0; k < c; k++) rmap[off - o_first + k] = (uint8_t)threadIdx.x;
    int total = c;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o2);
    __shared__ int wsum[ADC_EMIT_T / 32];
    if (lane == 0) wsum[threadIdx.x >> 5] = total;
    __syncthreads();
    int rows = 0;
#pragma unroll
    for (int w = 0; w < ADC_EMIT_T / 32; w++) rows += wsum[w];
    const int rowlen = in.sh_stride * 3;
    if ((rowlen & 3) == 0) {
        const int r4 = rowlen >> 2;
        const float4* src = reinterpret_cast<const float4*>(in.sh) + g0 * r4;
        float4* dst = reinterpret_cast<float4*>(out.sh) + (int64_t)o_first * r4;
        for (int i = threadIdx.x; i < rows * r4; i += blockDim.x) {
            const int r = i / r4, e = i - r * r4;
            dst[i] = src[(int64_t)rmap[r] * r4 + e];
        }
    } else {
        const float* src = in.sh + g0 * rowlen;
        float* dst = out.sh + (int64_t)o_first * rowlen;
        for (int i = threadIdx.x; i < rows * rowlen; i += blockDim.x) {
            const int r = i / rowlen, e = i - r * rowlen;
            dst[i] = src[(int64_t)rmap[r] * rowlen + e];
        }
    }
}

__global__ void k_adc_remap(const float* __restrict__ src, float* __restrict__ dst, int64_t width,
                            const int32_t* __restrict__ origin, const uint8_t* __restrict__ kind, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / width, c = i - r * width;
        dst[i] = kind[r] == 0 ? src[(int64_t)origin[r] * width + c] : 0.f;
    }
}

cudaError_t launch_adc_decide(const mvgs_gaussians& g, const mvgs_adc_accum& acc, const AdcParamsHost& h, int* cnt,
                              uint8_t* flags, unsigned long long* rep, cudaStream_t s) {
    const AdcParams prm{h.tau_split, h.tau_clone, h.ln_size, h.ln_split, h.logit_prune, h.ln_prune_scale, h.N, h.mode};
    const int64_t nb = (g.P + 1023) / 1024;
    if (nb > 0)
        k_adc_decide<<<(unsigned)nb, 1024, 0, s>>>(g.P, g.log_scales, g.opacity_logits, acc, prm, cnt, flags, rep);
    return cudaGetLastError();
}

cudaError_t launch_adc_emit(const mvgs_gaussians& g, const uint8_t* flags, const int* offs, const float* noise,
                            const AdcParamsHost& h, const mvgs_gaussians_out& out, int32_t* origin, uint8_t* kind,
                            cudaStream_t s) {
    const AdcParams prm{h.tau_split, h.tau_clone, h.ln_size, h.ln_split, h.logit_prune, h.ln_prune_scale, h.N, h.mode};
    const int64_t nb = (g.P + 255) / 256;
    if (nb > 0) k_adc_emit<<<(unsigned)nb, ADC_EMIT_T, 0, s>>>(g, flags, offs, noise, prm, out, origin, kind);
    return cudaGetLastError();
}

cudaError_t launch_adc_remap(const float* src, float* dst, int64_t width, const int32_t* origin, const uint8_t* kind,
                             int64_t P_new, cudaStream_t s) {
    const int64_t n = P_new * width;
    if (n > 0) {
        const int64_t nb = std::min<int64_t>((n + 255) / 256, 148 * 16);
        k_adc_remap<<<(unsigned)nb, 256, 0, s>>>(src, dst, width, origin, kind, n);
    }
    return cudaGetLastError();
}

}  // namespace mvgs
