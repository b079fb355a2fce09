// k_lab.cu — NEXT-4: the mini-batch gradient-variance laboratory on the fast path.
//
//   k_loss_grad     per-pixel loss gradient of a rendered batch against its targets:
//                   ℓ1 → scale·sign(C − C*), ℓ2 → 2·scale·(C − C*), with the loss Σ|·| or Σ(·)²
//                   summed per CTA in fp64 (deterministic final sum).
//   k_moments       Monte-Carlo accumulators of the §4.2 estimator for one mini-batch gradient
//                   g (fp32, n entries): sum[i] += g[i] (fp64 vector), ‖g‖² per CTA in fp64.
//   k_fsum          deterministic one-CTA sum of per-CTA fp64 partials, added into a scalar.
//   k_sqnorm        ‖sum‖² (fp64) per CTA, for 𝕍 = (1/K)Σ‖g_k‖² − ‖(1/K)Σg_k‖².
// All reductions are fixed-order (per-CTA shuffle trees, then one CTA over the partials), so
// the estimator is bit-reproducible run to run.
#include "internal.cuh"

namespace mvgs {

constexpr int LT = 256;
constexpr unsigned FULLL = 0xffffffffu;

__device__ __forceinline__ double block_sum_d(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLL, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < LT / 32; w++) t += red[w];
    return t;  // valid in thread 0
}

// target element as a float: fp32 as given, or an 8-bit image value t/255 (t · fl(1/255))
__device__ __forceinline__ float tgt_value(const float* t, int64_t i) { return t[i]; }
__device__ __forceinline__ float tgt_value(const uint8_t* t, int64_t i) {
    return __fmul_rn((float)t[i], 1.0f / 255.0f);  // rounded product (never contracted into the difference)
}

template <typename TT>
__global__ __launch_bounds__(LT) void k_loss_grad(const float* __restrict__ rgb, const TT* __restrict__ tgt,
                                                  int64_t n, int mode, float scale, float* __restrict__ dL,
                                                  double* __restrict__ part) {
    __shared__ double red[LT / 32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x; i < n; i += (int64_t)gridDim.x * LT) {
        const float d = rgb[i] - tgt_value(tgt, i);
        if (mode == 0) {
            dL[i] = d > 0.f ? scale : (d < 0.f ? -scale : 0.f);
            acc += (double)fabsf(d);
        } else {
            dL[i] = 2.f * scale * d;
            acc += (double)d * (double)d;
        }
    }
    const double t = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ __launch_bounds__(LT) void k_moments(const float* __restrict__ g, int64_t n, double* __restrict__ sum,
                                                double* __restrict__ part) {
    __shared__ double red[LT / 32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x; i < n; i += (int64_t)gridDim.x * LT) {
        const double v = (double)g[i];
        sum[i] += v;
        acc += v * v;
    }
    const double t = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ __launch_bounds__(LT) void k_sqnorm(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double red[LT / 32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x; i < n; i += (int64_t)gridDim.x * LT) acc += x[i] * x[i];
    const double t = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// out[0] (+)= Σ part[0..np) · mul ; mode 0: store, 1: add.  mode 2: variance
// out[0] = out_sumsq / K − Σ part / K² (part = per-CTA pieces of ‖Σ g_k‖²).
__global__ __launch_bounds__(LT) void k_fsum(const double* __restrict__ part, int np, int mode, double K,
                                             const double* __restrict__ sumsq, double* __restrict__ out) {
    __shared__ double red[LT / 32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += LT) acc += part[i];
    const double t = block_sum_d(acc, red);
    if (threadIdx.x == 0) {
        if (mode == 0) *out = t;
        else if (mode == 1) *out += t;
        else *out = *sumsq / K - t / (K * K);
    }
}

constexpr int LAB_GRID = 148 * 4;  // persistent grid: one wave of 4 CTAs per SM

int lab_partials() { return LAB_GRID; }

cudaError_t launch_loss_grad(const float* rgb, const float* tgt, int64_t n, int mode, float scale, float* dL,
                             double* loss, double* part, cudaStream_t s) {
    k_loss_grad<float><<<LAB_GRID, LT, 0, s>>>(rgb, tgt, n, mode, scale, dL, part);
    if (loss) k_fsum<<<1, LT, 0, s>>>(part, LAB_GRID, 0, 1.0, nullptr, loss);
    return cudaGetLastError();
}

cudaError_t launch_loss_grad_u8(const float* rgb, const uint8_t* tgt, int64_t n, int mode, float scale, float* dL,
                                double* loss, double* part, cudaStream_t s) {
    k_loss_grad<uint8_t><<<LAB_GRID, LT, 0, s>>>(rgb, tgt, n, mode, scale, dL, part);
    if (loss) k_fsum<<<1, LT, 0, s>>>(part, LAB_GRID, 0, 1.0, nullptr, loss);
    return cudaGetLastError();
}

cudaError_t launch_moments(const float* g, int64_t n, double* sum, double* sumsq, double* part, cudaStream_t s) {
    k_moments<<<LAB_GRID, LT, 0, s>>>(g, n, sum, part);
    k_fsum<<<1, LT, 0, s>>>(part, LAB_GRID, 1, 1.0, nullptr, sumsq);
    return cudaGetLastError();
}

cudaError_t launch_variance(const double* sum, int64_t n, const double* sumsq, int64_t K, double* out, double* part,
                            cudaStream_t s) {
    k_sqnorm<<<LAB_GRID, LT, 0, s>>>(sum, n, part);
    k_fsum<<<1, LT, 0, s>>>(part, LAB_GRID, 2, (double)K, sumsq, out);
    return cudaGetLastError();
}

}  // namespace mvgs
