// k_dssim.cu — NEXT-2: the 3D distance-aware D-SSIM loss, forward
// and backward on B200.
//
//   SSIM = (2μ1μ2 + C1)(2τ12 + C2) / ((μ1² + μ2² + C1)(τ1² + τ2² + C2))
//   moments taken with the 3D kernel K*(u,v) ∝ exp(−‖X_uv − X_c‖²/2σ²), X the
//   point of a pixel from the predicted depth
// Readings: 11×11 windows, renormalised over in-image
// foreground pixels; background (T_final > 0.999) centres use the 2D Gaussian
// kernel; σ3d(c) = σ_px·depth_c/fx (planar-equivalent); depth is a constant.
//
// k_dssim_center: one thread per window centre; a 16×16 tile of centres stages a
// 26×26 halo of (I1, I2, X, background) in shared memory, accumulates the five
// weighted moments per channel, writes SSIM to a per-block partial sum and the
// per-centre backward coefficients (∂S/∂m1, 2∂S/∂m11, ∂S/∂m12 per channel, 1/Σw,
// 1/2σ²).  k_dssim_grad: one thread per pixel u gathers, over the centres c
// whose window holds u, w_cu·(a_c + b_c·I1(u) + d_c·I2(u)).  k_dssim_total: a
// deterministic final sum of the block partials → loss.
#include <cuda_runtime.h>
#include "../../include/mvgs.h"

namespace mvgs {

constexpr int DR = 5;            // window radius (11×11)
constexpr int DT = 16;           // tile of centres
constexpr int DH = DT + 2 * DR;  // halo tile side (26)
constexpr float DC1 = 0.01f * 0.01f, DC2 = 0.03f * 0.03f;
constexpr int NCOEF = 12;        // a0 b0 d0 a1 b1 d1 a2 b2 d2, 1/Σw, 1/2σ² (−1: 2D kernel), pad

struct DssimCam {
    float fx, fy, cx, cy;
};
constexpr int DCAMS = 64;  // views per launch (intrinsics travel as a kernel parameter: graph-safe, no staging)
struct DssimCams {
    DssimCam c[DCAMS];
};

__device__ __forceinline__ void load_halo(const float* __restrict__ img, const float* __restrict__ tgt,
                                          const float* __restrict__ depth, const float* __restrict__ Tf, int v, int H,
                                          int W, int x0, int y0, const DssimCam& c, float (*s)[DH * DH]) {
    const int64_t HW = (int64_t)H * W;
    for (int i = threadIdx.x; i < DH * DH; i += blockDim.x) {
        const int yy = y0 - DR + i / DH, xx = x0 - DR + i % DH;
        const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
        const int64_t p = in ? (int64_t)yy * W + xx : 0;
        const float d = in ? depth[v * HW + p] : 0.f;
        for (int ch = 0; ch < 3; ch++) {
            s[ch][i] = in ? img[(3 * (int64_t)v + ch) * HW + p] : 0.f;
            s[3 + ch][i] = in ? tgt[(3 * (int64_t)v + ch) * HW + p] : 0.f;
        }
        s[6][i] = ((float)xx - c.cx) / c.fx * d;
        s[7][i] = ((float)yy - c.cy) / c.fy * d;
        s[8][i] = d;
        // 0: outside the image, 1: background, 2: foreground
        s[9][i] = !in ? 0.f : (Tf[v * HW + p] > 0.999f ? 1.f : 2.f);
    }
}

__global__ __launch_bounds__(256) void k_dssim_center(const float* __restrict__ img, const float* __restrict__ tgt,
                                                      const float* __restrict__ depth, const float* __restrict__ Tf,
                                                      const DssimCams cams, int v0, int H, int W, float sigma_px,
                                                      float* __restrict__ coef, double* __restrict__ partial) {
    __shared__ float s[10][DH * DH];
    __shared__ double red[8];
    const int TXn = (W + DT - 1) / DT;
    const int v = v0 + blockIdx.y;
    const int x0 = (blockIdx.x % TXn) * DT, y0 = (blockIdx.x / TXn) * DT;
    const DssimCam c = cams.c[blockIdx.y];
    load_halo(img, tgt, depth, Tf, v, H, W, x0, y0, c, s);
    __syncthreads();
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = x0 + lx, y = y0 + ly;
    double ssum = 0.0;
    if (x < W && y < H) {
        const int ci = (ly + DR) * DH + lx + DR;
        const bool bgc = s[9][ci] == 1.f;
        const float Xc = s[6][ci], Yc = s[7][ci], Zc = s[8][ci];
        const float sig3 = sigma_px * Zc / c.fx;
        const float i2s3 = bgc ? -1.f : 0.5f / (sig3 * sig3);
        const float i2s2 = 0.5f / (sigma_px * sigma_px);
        float wsum = 0.f, m1[3] = {0, 0, 0}, m2[3] = {0, 0, 0}, m11[3] = {0, 0, 0}, m22[3] = {0, 0, 0},
              m12[3] = {0, 0, 0};
        for (int dy = -DR; dy <= DR; dy++)
            for (int dx = -DR; dx <= DR; dx++) {
                const int j = (ly + DR + dy) * DH + lx + DR + dx;
                const float st = s[9][j];
                float w;
                if (bgc) {
                    w = st > 0.f ? __expf(-(float)(dx * dx + dy * dy) * i2s2) : 0.f;
                } else {
                    const float ex = s[6][j] - Xc, ey = s[7][j] - Yc, ez = s[8][j] - Zc;
                    w = st == 2.f ? __expf(-(ex * ex + ey * ey + ez * ez) * i2s3) : 0.f;
                }
                wsum += w;
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    const float a = s[ch][j], b = s[3 + ch][j];
                    m1[ch] += w * a;
                    m2[ch] += w * b;
                    m11[ch] += w * a * a;
                    m22[ch] += w * b * b;
                    m12[ch] += w * a * b;
                }
            }
        const float iw = 1.f / wsum;
        float* co = coef + (((int64_t)v * H + y) * W + x) * NCOEF;
#pragma unroll
        for (int ch = 0; ch < 3; ch++) {
            const float mu1 = m1[ch] * iw, mu2 = m2[ch] * iw;
            const float s11 = m11[ch] * iw - mu1 * mu1, s22 = m22[ch] * iw - mu2 * mu2, s12 = m12[ch] * iw - mu1 * mu2;
            const float A1 = 2.f * mu1 * mu2 + DC1, A2 = 2.f * s12 + DC2;
            const float B1 = mu1 * mu1 + mu2 * mu2 + DC1, B2 = s11 + s22 + DC2;
            const float S = A1 * A2 / (B1 * B2);
            ssum += (double)S;
            const float dS_m1 = S * (2.f * mu2 / A1 - 2.f * mu1 / B1) + (S / B2) * (2.f * mu1) - (2.f * S / A2) * mu2;
            co[3 * ch + 0] = dS_m1;
            co[3 * ch + 1] = -2.f * S / B2;  // 2·∂S/∂m11
            co[3 * ch + 2] = 2.f * S / A2;   // ∂S/∂m12
        }
        co[9] = iw;
        co[10] = i2s3;
        co[11] = 0.f;
    }
    // deterministic block sum of the SSIM values
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ssum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; w++) t += red[w];
        partial[(int64_t)v * gridDim.x + blockIdx.x] = t;
    }
}

__global__ __launch_bounds__(256) void k_dssim_total(const double* __restrict__ partial, int n, double inv_count,
                                                     float* __restrict__ loss) {
    __shared__ double red[8];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += partial[i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; w++) s += red[w];
        *loss = (float)(1.0 - s * inv_count);
    }
}

// Halo of centres for the gather: their camera-space points and their 12
// coefficients (3 float4), 26×26 × 15 floats = 40.6 KB of shared memory.
__global__ __launch_bounds__(256) void k_dssim_grad(const float* __restrict__ img, const float* __restrict__ tgt,
                                                    const float* __restrict__ depth, const float* __restrict__ Tf,
                                                    const DssimCams cams, int v0, int H, int W, float sigma_px,
                                                    const float4* __restrict__ coef, float scale,
                                                    float* __restrict__ grad) {
    __shared__ float4 sco[3][DH * DH];
    __shared__ float sp[3][DH * DH];
    const int TXn = (W + DT - 1) / DT;
    const int v = v0 + blockIdx.y;
    const int x0 = (blockIdx.x % TXn) * DT, y0 = (blockIdx.x / TXn) * DT;
    const DssimCam c = cams.c[blockIdx.y];
    const int64_t HW = (int64_t)H * W;
    for (int i = threadIdx.x; i < DH * DH; i += blockDim.x) {
        const int yy = y0 - DR + i / DH, xx = x0 - DR + i % DH;
        const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
        const int64_t p = in ? (int64_t)yy * W + xx : 0;
        const float d = in ? depth[v * HW + p] : 0.f;
        sp[0][i] = ((float)xx - c.cx) / c.fx * d;
        sp[1][i] = ((float)yy - c.cy) / c.fy * d;
        sp[2][i] = d;
        const float4* co = coef + (v * HW + p) * 3;
#pragma unroll
        for (int k = 0; k < 3; k++) sco[k][i] = in ? co[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = x0 + lx, y = y0 + ly;
    if (x >= W || y >= H) return;
    const int64_t p = (int64_t)y * W + x;
    const int ui = (ly + DR) * DH + lx + DR;
    const bool fg_u = Tf[v * HW + p] <= 0.999f;
    const float Xu = sp[0][ui], Yu = sp[1][ui], Zu = sp[2][ui];
    float I1[3], I2[3];
#pragma unroll
    for (int ch = 0; ch < 3; ch++) {
        I1[ch] = img[(3 * (int64_t)v + ch) * HW + p];
        I2[ch] = tgt[(3 * (int64_t)v + ch) * HW + p];
    }
    const float i2s2 = 0.5f / (sigma_px * sigma_px);
    float g[3] = {0.f, 0.f, 0.f};
    for (int dy = -DR; dy <= DR; dy++) {
        const int cy = y + dy;
        if (cy < 0 || cy >= H) continue;
        for (int dx = -DR; dx <= DR; dx++) {
            const int cx = x + dx;  // centre whose window holds u
            if (cx < 0 || cx >= W) continue;
            const int j = (ly + DR + dy) * DH + lx + DR + dx;
            const float4 c0 = sco[0][j], c1 = sco[1][j], c2 = sco[2][j];
            // c0 = (a0 b0 d0 a1), c1 = (b1 d1 a2 b2), c2 = (d2, 1/Σw, 1/2σ², 0)
            float w;
            if (c2.z < 0.f) {  // background centre: 2D kernel over all in-image pixels
                w = __expf(-(float)(dx * dx + dy * dy) * i2s2);
            } else {
                if (!fg_u) continue;
                const float ex = Xu - sp[0][j], ey = Yu - sp[1][j], ez = Zu - sp[2][j];
                w = __expf(-(ex * ex + ey * ey + ez * ez) * c2.z);
            }
            w *= c2.y;
            g[0] += w * (c0.x + c0.y * I1[0] + c0.z * I2[0]);
            g[1] += w * (c0.w + c1.x * I1[1] + c1.y * I2[1]);
            g[2] += w * (c1.z + c1.w * I1[2] + c2.x * I2[2]);
        }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ch++) grad[(3 * (int64_t)v + ch) * HW + p] = scale * g[ch];
}

cudaError_t launch_dssim3d(const mvgs_camera* h_cams, int V, int H, int W, const float* img, const float* tgt,
                           const float* depth, const float* Tf, float sigma_px, float* loss, float* grad, float* coef,
                           double* partial, cudaStream_t s) {
    const int TXn = (W + DT - 1) / DT, TYn = (H + DT - 1) / DT;
    const double N = 3.0 * V * H * W;
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1 && !grad) break;
        for (int v0 = 0; v0 < V; v0 += DCAMS) {
            const int nv = V - v0 < DCAMS ? V - v0 : DCAMS;
            DssimCams dc{};
            for (int i = 0; i < nv; i++)
                dc.c[i] = DssimCam{h_cams[v0 + i].fx, h_cams[v0 + i].fy, h_cams[v0 + i].cx, h_cams[v0 + i].cy};
            dim3 grid(TXn * TYn, nv);
            if (pass == 0)
                k_dssim_center<<<grid, 256, 0, s>>>(img, tgt, depth, Tf, dc, v0, H, W, sigma_px, coef, partial);
            else
                k_dssim_grad<<<grid, 256, 0, s>>>(img, tgt, depth, Tf, dc, v0, H, W, sigma_px, (const float4*)coef,
                                                  (float)(-1.0 / N), grad);
        }
        if (pass == 0) k_dssim_total<<<1, 256, 0, s>>>(partial, TXn * TYn * V, 1.0 / N, loss);
    }
    return cudaGetLastError();
}

}  // namespace mvgs
