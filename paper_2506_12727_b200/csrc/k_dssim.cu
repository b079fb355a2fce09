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
// k_dssim_center: a 32×16 tile of window centres per 128-thread CTA, each thread
// a vertical strip of NY = 4 centres, so every halo pixel it loads from shared
// memory (42×26 halo of point + colours) feeds up to 4 windows (register
// blocking: the loop is FP32-issue bound, not LDS bound).  It accumulates the
// five weighted moments per channel, adds SSIM to a per-CTA partial sum and
// writes the per-centre backward coefficients, pre-scaled by 1/Σw:
// (∂S/∂m1, 2∂S/∂m11, ∂S/∂m12) per channel and the kernel's exponent scale.
// k_dssim_grad: the same tiling over pixels u; it stages the halo of centre
// coefficients and points and gathers, over the centres c whose window holds u,
// w_cu·(a_c + b_c·I1(u) + d_c·I2(u)).  k_dssim_total: a deterministic final
// sum of the per-CTA partials → loss.
#include <cuda_runtime.h>
#include "../../include/mvgs.h"

namespace mvgs {

constexpr int DR = 5;                 // window radius (11×11)
constexpr int DTX = 32, DNY = 4;      // tile: 32 columns × (4 thread rows × DNY) = 32×16 centres
constexpr int DTY = 4 * DNY;
constexpr int DHX = DTX + 2 * DR, DHY = DTY + 2 * DR, DHN = DHX * DHY;  // 42×26 halo
constexpr float DC1 = 0.01f * 0.01f, DC2 = 0.03f * 0.03f;
constexpr float DBIG = 1e15f;         // point of a non-foreground pixel: 3D weight underflows to 0
constexpr float LOG2E = 1.4426950408889634f;
constexpr int DCAMS = 64;             // views per launch (intrinsics are a kernel parameter: graph-safe)

struct DssimCam {
    float fx, fy, cx, cy;
};
struct DssimCams {
    DssimCam c[DCAMS];
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// camera-space point of pixel (xx, yy) at depth d (R: DESIGN.md §14)
__device__ __forceinline__ float3 unproject(const DssimCam& c, int xx, int yy, float d) {
    return make_float3(((float)xx - c.cx) / c.fx * d, ((float)yy - c.cy) / c.fy * d, d);
}

__global__ __launch_bounds__(128) void k_dssim_center(const float* __restrict__ img, const float* __restrict__ tgt,
                                                      const float* __restrict__ depth, const float* __restrict__ Tf,
                                                      const DssimCams cams, int v0, int H, int W, float sigma_px,
                                                      float4* __restrict__ coef, double* __restrict__ partial) {
    __shared__ float4 spt[DHN];      // (X, Y, Z, 2D penalty): foreground point or DBIG; penalty DBIG outside
    __shared__ float2 scol[3][DHN];  // (I1, I2) per channel
    __shared__ double red[4];
    const int TXn = (W + DTX - 1) / DTX;
    const int v = v0 + blockIdx.y;
    const int x0 = (blockIdx.x % TXn) * DTX, y0 = (blockIdx.x / TXn) * DTY;
    const DssimCam c = cams.c[blockIdx.y];
    const int64_t HW = (int64_t)H * W;
    for (int i = threadIdx.x; i < DHN; i += blockDim.x) {
        const int yy = y0 - DR + i / DHX, xx = x0 - DR + i % DHX;
        const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
        const int64_t p = in ? (int64_t)yy * W + xx : 0;
        float4 pt = make_float4(DBIG, DBIG, DBIG, in ? 0.f : DBIG);
        if (in && Tf[v * HW + p] <= 0.999f) {
            const float3 X = unproject(c, xx, yy, depth[v * HW + p]);
            pt.x = X.x, pt.y = X.y, pt.z = X.z;
        }
        spt[i] = pt;
#pragma unroll
        for (int ch = 0; ch < 3; ch++)
            scol[ch][i] = in ? make_float2(img[(3 * (int64_t)v + ch) * HW + p], tgt[(3 * (int64_t)v + ch) * HW + p])
                             : make_float2(0.f, 0.f);
    }
    __syncthreads();
    const int lx = threadIdx.x & 31, ly = (threadIdx.x >> 5) * DNY;
    const int x = x0 + lx;
    float Xc[DNY], Yc[DNY], Zc[DNY], kc[DNY];
    bool bg[DNY];
    const float k2d = LOG2E * 0.5f / (sigma_px * sigma_px);
#pragma unroll
    for (int i = 0; i < DNY; i++) {
        const float4 pt = spt[(ly + i + DR) * DHX + lx + DR];
        bg[i] = pt.x == DBIG;
        Xc[i] = pt.x, Yc[i] = pt.y, Zc[i] = pt.z;
        const float sig3 = sigma_px * pt.z / c.fx;
        kc[i] = bg[i] ? k2d : LOG2E * 0.5f / (sig3 * sig3);
    }
    // moments per (centre, channel): (m1, m2) and (m11, m22) as packed pairs (FFMA2/FADD2), m12 scalar
    float ws[DNY], m12[DNY][3];
    float2 mm[DNY][3], msq[DNY][3];
#pragma unroll
    for (int i = 0; i < DNY; i++) {
        ws[i] = 0.f;
#pragma unroll
        for (int ch = 0; ch < 3; ch++) {
            mm[i][ch] = msq[i][ch] = make_float2(0.f, 0.f);
            m12[i][ch] = 0.f;
        }
    }
#pragma unroll
    for (int r = 0; r < DNY + 2 * DR; r++) {
        const int row = (ly + r) * DHX + lx;
#pragma unroll 1
        for (int dx = 0; dx <= 2 * DR; dx++) {
            const float4 P = spt[row + dx];
            const float2 cc[3] = {scol[0][row + dx], scol[1][row + dx], scol[2][row + dx]};
            const float rx2 = (float)((dx - DR) * (dx - DR)) + P.w;
#pragma unroll
            for (int i = 0; i < DNY; i++) {
                const int dy = r - DR - i;
                if (dy < -DR || dy > DR) continue;
                const float ex = P.x - Xc[i], ey = P.y - Yc[i], ez = P.z - Zc[i];
                const float d2 = bg[i] ? rx2 + (float)(dy * dy) : ex * ex + ey * ey + ez * ez;
                const float w = ex2(-d2 * kc[i]);
                ws[i] += w;
                const float2 w2 = make_float2(w, w);
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    const float2 wab = __fmul2_rn(w2, cc[ch]);
                    mm[i][ch] = __fadd2_rn(mm[i][ch], wab);
                    msq[i][ch] = __ffma2_rn(wab, cc[ch], msq[i][ch]);
                    m12[i][ch] = fmaf(wab.x, cc[ch].y, m12[i][ch]);
                }
            }
        }
    }
    double ssum = 0.0;
#pragma unroll
    for (int i = 0; i < DNY; i++) {
        const int y = y0 + ly + i;
        if (x >= W || y >= H) continue;
        const float iw = 1.f / ws[i];
        float o[12];
#pragma unroll
        for (int ch = 0; ch < 3; ch++) {
            const float mu1 = mm[i][ch].x * iw, mu2 = mm[i][ch].y * iw;
            const float s11 = msq[i][ch].x * iw - mu1 * mu1, s22 = msq[i][ch].y * iw - mu2 * mu2;
            const float s12 = m12[i][ch] * iw - mu1 * mu2;
            const float A1 = 2.f * mu1 * mu2 + DC1, A2 = 2.f * s12 + DC2;
            const float B1 = mu1 * mu1 + mu2 * mu2 + DC1, B2 = s11 + s22 + DC2;
            const float S = A1 * A2 / (B1 * B2);
            ssum += (double)S;
            const float dS_m1 = S * (2.f * mu2 / A1 - 2.f * mu1 / B1) + (S / B2) * (2.f * mu1) - (2.f * S / A2) * mu2;
            o[3 * ch + 0] = dS_m1 * iw;
            o[3 * ch + 1] = -2.f * S / B2 * iw;  // 2·∂S/∂m11
            o[3 * ch + 2] = 2.f * S / A2 * iw;   // ∂S/∂m12
        }
        o[9] = bg[i] ? -kc[i] : kc[i];  // exponent scale; sign marks a 2D (background) centre
        o[10] = o[11] = 0.f;
        float4* co = coef + (((int64_t)v * H + y) * W + x) * 3;
        co[0] = make_float4(o[0], o[1], o[2], o[3]);
        co[1] = make_float4(o[4], o[5], o[6], o[7]);
        co[2] = make_float4(o[8], o[9], o[10], o[11]);
    }
    for (int off = 16; off > 0; off >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, off);
    if (lx == 0) red[threadIdx.x >> 5] = ssum;
    __syncthreads();
    if (threadIdx.x == 0) partial[(int64_t)v * gridDim.x + blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
}

__global__ __launch_bounds__(1024) void k_dssim_total(const double* __restrict__ partial, int n, double inv_count,
                                                      float* __restrict__ loss) {
    __shared__ double red[32];
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += partial[i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x < 32) {
        t = red[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) *loss = (float)(1.0 - t * inv_count);
    }
}

// Shared memory of k_dssim_grad (dynamic, 56.8 KB): per halo centre its two
// coefficient quads, (d2, exponent scale) and its point.
struct GradSmem {
    float4 cA[DHN], cB[DHN];
    float4 cP[DHN];  // (X, Y, Z, d2 coefficient of channel 2)
    float ck[DHN];   // exponent scale (negative: 2D centre); 0 outside the image
};

__global__ __launch_bounds__(128) void k_dssim_grad(const float* __restrict__ img, const float* __restrict__ tgt,
                                                    const float* __restrict__ depth, const float* __restrict__ Tf,
                                                    const DssimCams cams, int v0, int H, int W,
                                                    const float4* __restrict__ coef, float scale,
                                                    float* __restrict__ grad) {
    extern __shared__ float4 dyn_smem[];
    GradSmem& sm = *reinterpret_cast<GradSmem*>(dyn_smem);
    const int TXn = (W + DTX - 1) / DTX;
    const int v = v0 + blockIdx.y;
    const int x0 = (blockIdx.x % TXn) * DTX, y0 = (blockIdx.x / TXn) * DTY;
    const DssimCam c = cams.c[blockIdx.y];
    const int64_t HW = (int64_t)H * W;
    for (int i = threadIdx.x; i < DHN; i += blockDim.x) {
        const int yy = y0 - DR + i / DHX, xx = x0 - DR + i % DHX;
        const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
        const int64_t p = in ? (int64_t)yy * W + xx : 0;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, e = a;
        float3 X = make_float3(0.f, 0.f, 0.f);
        if (in) {
            const float4* co = coef + (v * HW + p) * 3;
            a = co[0], b = co[1], e = co[2];
            X = unproject(c, xx, yy, depth[v * HW + p]);
        }
        sm.cA[i] = a;
        sm.cB[i] = b;
        sm.cP[i] = make_float4(X.x, X.y, X.z, e.x);
        sm.ck[i] = e.y;  // 0 outside: w = 1 against zero coefficients
    }
    __syncthreads();
    const int lx = threadIdx.x & 31, ly = (threadIdx.x >> 5) * DNY;
    const int x = x0 + lx;
    // per pixel: Σ_c w·(a, b, d) per channel as packed pairs; combined with I1, I2 at the end
    float Xu[DNY], Yu[DNY], Zu[DNY], G8[DNY];
    float2 G01[DNY], G23[DNY], G45[DNY], G67[DNY];
#pragma unroll
    for (int i = 0; i < DNY; i++) {
        const int y = y0 + ly + i;
        const bool in = x < W && y < H;
        const bool fg = in && Tf[v * HW + (int64_t)y * W + x] <= 0.999f;
        const float4 P = sm.cP[(ly + i + DR) * DHX + lx + DR];
        Xu[i] = fg ? P.x : DBIG, Yu[i] = fg ? P.y : DBIG, Zu[i] = fg ? P.z : DBIG;
        G01[i] = G23[i] = G45[i] = G67[i] = make_float2(0.f, 0.f);
        G8[i] = 0.f;
    }
#pragma unroll
    for (int r = 0; r < DNY + 2 * DR; r++) {
        const int row = (ly + r) * DHX + lx;
#pragma unroll 1
        for (int dx = 0; dx <= 2 * DR; dx++) {
            const float4 A = sm.cA[row + dx], B = sm.cB[row + dx], P = sm.cP[row + dx];
            const float k = sm.ck[row + dx];
            const bool bgc = k < 0.f;
            const float ka = fabsf(k);
            const float rx2 = (float)((dx - DR) * (dx - DR));
#pragma unroll
            for (int i = 0; i < DNY; i++) {
                const int dy = r - DR - i;  // centre row − pixel row
                if (dy < -DR || dy > DR) continue;
                const float ex = Xu[i] - P.x, ey = Yu[i] - P.y, ez = Zu[i] - P.z;
                const float d2 = bgc ? rx2 + (float)(dy * dy) : ex * ex + ey * ey + ez * ez;
                const float w = ex2(-d2 * ka);
                const float2 w2 = make_float2(w, w);
                G01[i] = __ffma2_rn(w2, make_float2(A.x, A.y), G01[i]);
                G23[i] = __ffma2_rn(w2, make_float2(A.z, A.w), G23[i]);
                G45[i] = __ffma2_rn(w2, make_float2(B.x, B.y), G45[i]);
                G67[i] = __ffma2_rn(w2, make_float2(B.z, B.w), G67[i]);
                G8[i] = fmaf(w, P.w, G8[i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < DNY; i++) {
        const int y = y0 + ly + i;
        if (x >= W || y >= H) continue;
        const int64_t p = (int64_t)y * W + x;
        const float* i1 = img + 3 * (int64_t)v * HW + p;
        const float* i2 = tgt + 3 * (int64_t)v * HW + p;
        float* gp = grad + 3 * (int64_t)v * HW + p;
        gp[0] = scale * (G01[i].x + G01[i].y * i1[0] + G23[i].x * i2[0]);
        gp[HW] = scale * (G23[i].y + G45[i].x * i1[HW] + G45[i].y * i2[HW]);
        gp[2 * HW] = scale * (G67[i].x + G67[i].y * i1[2 * HW] + G8[i] * i2[2 * HW]);
    }
}

cudaError_t launch_dssim3d(const mvgs_camera* h_cams, int V, int H, int W, const float* img, const float* tgt,
                           const float* depth, const float* Tf, float sigma_px, float* loss, float* grad, float* coef,
                           double* partial, cudaStream_t s) {
    const int TXn = (W + DTX - 1) / DTX, TYn = (H + DTY - 1) / DTY;
    const double N = 3.0 * V * H * W;
    if (grad) {
        cudaError_t e = cudaFuncSetAttribute(k_dssim_grad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(GradSmem));
        if (e != cudaSuccess) return e;
    }
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1 && !grad) break;
        for (int v0 = 0; v0 < V; v0 += DCAMS) {
            const int nv = V - v0 < DCAMS ? V - v0 : DCAMS;
            DssimCams dc{};
            for (int i = 0; i < nv; i++)
                dc.c[i] = DssimCam{h_cams[v0 + i].fx, h_cams[v0 + i].fy, h_cams[v0 + i].cx, h_cams[v0 + i].cy};
            dim3 grid(TXn * TYn, nv);
            if (pass == 0)
                k_dssim_center<<<grid, 128, 0, s>>>(img, tgt, depth, Tf, dc, v0, H, W, sigma_px, (float4*)coef,
                                                    partial);
            else
                k_dssim_grad<<<grid, 128, sizeof(GradSmem), s>>>(img, tgt, depth, Tf, dc, v0, H, W,
                                                                 (const float4*)coef, (float)(-1.0 / N), grad);
        }
        if (pass == 0) k_dssim_total<<<1, 1024, 0, s>>>(partial, TXn * TYn * V, 1.0 / N, loss);
    }
    return cudaGetLastError();
}

int64_t dssim_partials(int V, int H, int W) {
    return (int64_t)V * ((W + DTX - 1) / DTX) * ((H + DTY - 1) / DTY);
}

}  // namespace mvgs
