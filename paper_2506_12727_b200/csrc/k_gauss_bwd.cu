// k_gauss_bwd.cu — S8 per-Gaussian chain rule and S9 ADC statistics.
//
// One thread per Gaussian walks its pairs (one per participating view, found
// again with the same ballot ranking k_project used, so no pair→Gaussian index
// is stored) and sums over the batch's views — the multi-view mini-batch
// gradient.  No atomics: a Gaussian's views are all in one thread.
// The Σ → (scale, rotation) chain is linear in ∂L/∂Σ, so ∂L/∂Σ is summed over
// views first and pushed through once.  The same loop reduces the ADC
// statistics:
//   E1    = Σ_views e1[pair]               (e1 = Σ_pixels ‖∇_{p_i}L‖, from S7)
//   E2    = Σ_views ‖Σ∇[pair]‖
//   E_old = ‖Σ_views Σ∇[pair]‖
//   vis   = #views with tiles > 0 (R21)
#include "ca.cuh"
#include "internal.cuh"

namespace mvgs {

constexpr unsigned FULLG = 0xffffffffu;

// real SH constants [3DGS] as compile-time values (folded into the products)
constexpr float g_SH1 = 0.4886025119029199f;
constexpr float g_SH2_0 = 1.0925484305920792f;
constexpr float g_SH2_1 = -1.0925484305920792f;
constexpr float g_SH2_2 = 0.31539156525252005f;
constexpr float g_SH2_3 = -1.0925484305920792f;
constexpr float g_SH2_4 = 0.5462742152960396f;
constexpr float g_SH3_0 = -0.5900435899266435f;
constexpr float g_SH3_1 = 2.890611442640554f;
constexpr float g_SH3_2 = -0.4570457994644658f;
constexpr float g_SH3_3 = 0.3731763325901154f;
constexpr float g_SH3_4 = -0.4570457994644658f;
constexpr float g_SH3_5 = 1.445305721320277f;
constexpr float g_SH3_6 = -0.5900435899266435f;

// Hardware approximations for values that decide nothing: MUFU.RCP /
// MUFU.SQRT (≤ 2 ulp) instead of the multi-instruction IEEE sequences.
__device__ __forceinline__ float g_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float g_sqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Values-only recomputation for the chain rule (no decision depends on them: the
// Jacobian clamps come from the pair flags written by k_project), so fast
// reciprocal / exp / rsqrt are used instead of the canonical arithmetic.
struct FastActiv {
    float o, s[3], q[4], inv_norm, R[9], Sig[6];
};

__device__ __forceinline__ void fast_activate(const float* __restrict__ ls, const float* __restrict__ qr, float logit,
                                              FastActiv& a) {
    a.o = g_rcp(1.f + __expf(-logit));
    a.s[0] = __expf(ls[0]);
    a.s[1] = __expf(ls[1]);
    a.s[2] = __expf(ls[2]);
    float w = qr[0], x = qr[1], y = qr[2], z = qr[3];
    const float inv = rsqrtf(w * w + x * x + y * y + z * z);
    a.inv_norm = inv;
    w *= inv; x *= inv; y *= inv; z *= inv;
    a.q[0] = w; a.q[1] = x; a.q[2] = y; a.q[3] = z;
    float* R = a.R;
    R[0] = 1.f - 2.f * (y * y + z * z); R[1] = 2.f * (x * y - w * z); R[2] = 2.f * (x * z + w * y);
    R[3] = 2.f * (x * y + w * z); R[4] = 1.f - 2.f * (x * x + z * z); R[5] = 2.f * (y * z - w * x);
    R[6] = 2.f * (x * z - w * y); R[7] = 2.f * (y * z + w * x); R[8] = 1.f - 2.f * (x * x + y * y);
    float M[9];
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int c = 0; c < 3; c++) M[3 * r + c] = R[3 * r + c] * a.s[c];
    a.Sig[0] = M[0] * M[0] + M[1] * M[1] + M[2] * M[2];
    a.Sig[1] = M[0] * M[3] + M[1] * M[4] + M[2] * M[5];
    a.Sig[2] = M[0] * M[6] + M[1] * M[7] + M[2] * M[8];
    a.Sig[3] = M[3] * M[3] + M[4] * M[4] + M[5] * M[5];
    a.Sig[4] = M[3] * M[6] + M[4] * M[7] + M[5] * M[8];
    a.Sig[5] = M[6] * M[6] + M[7] * M[7] + M[8] * M[8];
}

struct FastProj {
    float tx, ty, tz, itz, uxc, uyc, T0[3], T1[3], a, b, c, det;
};

__device__ __forceinline__ void fast_project(const mvgs_camera& cam, float mx, float my, float mz, const float Sig[6],
                                             uint32_t flags, float limx, float limy, FastProj& p) {
    const float* R = cam.R;
    p.tx = R[0] * mx + R[1] * my + R[2] * mz + cam.t[0];
    p.ty = R[3] * mx + R[4] * my + R[5] * mz + cam.t[1];
    p.tz = R[6] * mx + R[7] * my + R[8] * mz + cam.t[2];
    p.itz = g_rcp(p.tz);
    const float ux = p.tx * p.itz, uy = p.ty * p.itz;
    p.uxc = (flags & 8u) ? fminf(limx, fmaxf(-limx, ux)) : ux;   // clamp decisions from k_project (R4)
    p.uyc = (flags & 16u) ? fminf(limy, fmaxf(-limy, uy)) : uy;
    const float J00 = cam.fx * p.itz, J02 = -cam.fx * p.uxc * p.itz;
    const float J11 = cam.fy * p.itz, J12 = -cam.fy * p.uyc * p.itz;
#pragma unroll
    for (int j = 0; j < 3; j++) {
        p.T0[j] = J00 * R[j] + J02 * R[6 + j];
        p.T1[j] = J11 * R[3 + j] + J12 * R[6 + j];
    }
    const float U00 = p.T0[0] * Sig[0] + p.T0[1] * Sig[1] + p.T0[2] * Sig[2];
    const float U01 = p.T0[0] * Sig[1] + p.T0[1] * Sig[3] + p.T0[2] * Sig[4];
    const float U02 = p.T0[0] * Sig[2] + p.T0[1] * Sig[4] + p.T0[2] * Sig[5];
    const float U10 = p.T1[0] * Sig[0] + p.T1[1] * Sig[1] + p.T1[2] * Sig[2];
    const float U11 = p.T1[0] * Sig[1] + p.T1[1] * Sig[3] + p.T1[2] * Sig[4];
    const float U12 = p.T1[0] * Sig[2] + p.T1[1] * Sig[4] + p.T1[2] * Sig[5];
    p.a = U00 * p.T0[0] + U01 * p.T0[1] + U02 * p.T0[2] + 0.3f;
    p.b = U00 * p.T1[0] + U01 * p.T1[1] + U02 * p.T1[2];
    p.c = U10 * p.T1[0] + U11 * p.T1[1] + U12 * p.T1[2] + 0.3f;
    p.det = p.a * p.c - p.b * p.b;
}

// SH coefficients and their gradient live in shared memory, one padded row per
// Gaussian, walked by its thread with 16-byte accesses: the row stride is an odd
// number of float4 ⇒ every LDS.128/STS.128 of a warp is 4 conflict-free wavefronts.
// The block's rows are loaded (cp.async, 16 B when the global rows allow) and stored
// with coalesced accesses.
template <int D>
struct ShRows {
    static constexpr int NK = (D + 1) * (D + 1);
    static constexpr int NS = NK * 3;
    static constexpr int NS4 = (NS + 3) / 4;  // float4 per row
    static constexpr int STRIDE = 4 * (NS4 | 1);
};

#ifndef GB_PREFETCH
#define GB_PREFETCH 1  // L2 prefetch of the next view's pair flags and gradient slot
#endif
#ifndef GB_VB
#define GB_VB 1  // views whose pair loads are issued together (measured: 1 → 0.60 ms, 2 → 0.61, 4 → 0.67)
#endif

// One visible (Gaussian, view) pair of the chain rule (S8) and its ADC terms (S9), added into
// the Gaussian's accumulators; the SH-gradient row is updated in shared memory.
struct GAcc {
    float dmx = 0.f, dmy = 0.f, dmz = 0.f;
    float G00 = 0.f, G01 = 0.f, G02 = 0.f, G11 = 0.f, G12 = 0.f, G22 = 0.f;  // ∂L/∂Σ (symmetric)
    float dop = 0.f, e1 = 0.f, e2 = 0.f, gsx = 0.f, gsy = 0.f, nvis = 0.f;
    float rmax = 0.f;  // largest screen radius over the visible views (k_project's CA radius, flags >> 8)
};

template <int D>
__device__ __forceinline__ void pair_chain(const mvgs_camera& c, float4 cam4, float limy, uint32_t flags, float4 pg0,
                                           float4 pg1, float4 pg2, float mx, float my, float mz, const float* Sg,
                                           const float* sh, float* dsh, float sW, float sH, GAcc& A) {
    constexpr int NK = ShRows<D>::NK, NS = ShRows<D>::NS;
    float& dmx = A.dmx; float& dmy = A.dmy; float& dmz = A.dmz;
    float& G00 = A.G00; float& G01 = A.G01; float& G02 = A.G02;
    float& G11 = A.G11; float& G12 = A.G12; float& G22 = A.G22;
    float& dop = A.dop; float& e1 = A.e1; float& e2 = A.e2;
    float& gsx = A.gsx; float& gsy = A.gsy; float& nvis = A.nvis;
    // pg: (Σ∇x, Σ∇y, e1, ∂A) (∂B, ∂C, ∂o, ∂r) (∂g, ∂b, -, -)
    nvis += 1.f;
    A.rmax = fmaxf(A.rmax, (float)(flags >> PF_RADIUS_SHIFT));
    e1 += pg0.z;
    e2 += g_sqrt(pg0.x * pg0.x + pg0.y * pg0.y);
    gsx += pg0.x;
    gsy += pg0.y;
    dop += pg1.z;
    FastProj p;
    fast_project(c, mx, my, mz, Sg, flags, cam4.w, limy, p);
    const float itz = p.itz, itz2 = itz * itz;
    // μ' (pixels) = (fx·tx/tz + cx, fy·ty/tz + cy); ∂L/∂μ' = Σ∇·(2/W, 2/H) (R2)
    const float dpx = pg0.x * sW, dpy = pg0.y * sH;
    float dtx = c.fx * itz * dpx;
    float dty = c.fy * itz * dpy;
    float dtz = -(c.fx * p.tx * itz2) * dpx - (c.fy * p.ty * itz2) * dpy;
    // conic (A,B,C) = (c,−b,a)/det → Σ' entries (a,b,c)
    const float dA = pg0.w, dB = pg1.x, dC = pg1.y;
    const float id2 = g_rcp(p.det * p.det);
    const float da = (-p.c * p.c * dA + p.b * p.c * dB - p.b * p.b * dC) * id2;
    const float dc = (-p.b * p.b * dA + p.a * p.b * dB - p.a * p.a * dC) * id2;
    const float db = (2.f * p.b * p.c * dA - (p.det + 2.f * p.b * p.b) * dB + 2.f * p.a * p.b * dC) * id2;
    const float hb = 0.5f * db;
    // ∂L/∂Σ += Tᵀ Gs T,  Gs = [[da, hb], [hb, dc]]
    const float* T0 = p.T0;
    const float* T1 = p.T1;
    float GT0[3], GT1[3];  // Gs·T rows
#pragma unroll
    for (int j = 0; j < 3; j++) {
        GT0[j] = da * T0[j] + hb * T1[j];
        GT1[j] = hb * T0[j] + dc * T1[j];
    }
    G00 += T0[0] * GT0[0] + T1[0] * GT1[0];
    G01 += T0[0] * GT0[1] + T1[0] * GT1[1];
    G02 += T0[0] * GT0[2] + T1[0] * GT1[2];
    G11 += T0[1] * GT0[1] + T1[1] * GT1[1];
    G12 += T0[1] * GT0[2] + T1[1] * GT1[2];
    G22 += T0[2] * GT0[2] + T1[2] * GT1[2];
    // ∂L/∂T = 2 (Gs T) Σ
    const float* S = Sg;
    float dT0[3], dT1[3];
    dT0[0] = 2.f * (GT0[0] * S[0] + GT0[1] * S[1] + GT0[2] * S[2]);
    dT0[1] = 2.f * (GT0[0] * S[1] + GT0[1] * S[3] + GT0[2] * S[4]);
    dT0[2] = 2.f * (GT0[0] * S[2] + GT0[1] * S[4] + GT0[2] * S[5]);
    dT1[0] = 2.f * (GT1[0] * S[0] + GT1[1] * S[1] + GT1[2] * S[2]);
    dT1[1] = 2.f * (GT1[0] * S[1] + GT1[1] * S[3] + GT1[2] * S[4]);
    dT1[2] = 2.f * (GT1[0] * S[2] + GT1[1] * S[4] + GT1[2] * S[5]);
    // T = J R_v ⇒ ∂L/∂J = ∂L/∂T R_vᵀ (only the non-constant entries of J)
    const float* R = c.R;
    const float dJ00 = dT0[0] * R[0] + dT0[1] * R[1] + dT0[2] * R[2];
    const float dJ02 = dT0[0] * R[6] + dT0[1] * R[7] + dT0[2] * R[8];
    const float dJ11 = dT1[0] * R[3] + dT1[1] * R[4] + dT1[2] * R[5];
    const float dJ12 = dT1[0] * R[6] + dT1[1] * R[7] + dT1[2] * R[8];
    dtz += -c.fx * itz2 * dJ00 - c.fy * itz2 * dJ11;
    // J02 = −fx·ũx/tz: ũx = tx/tz unclamped (∂/∂tx = −fx/tz², ∂/∂tz = 2fx·ux/tz²),
    // constant when clamped (∂/∂tz = fx·ũx/tz²) — R4
    if (!(flags & 8u)) {
        dtx += -c.fx * itz2 * dJ02;
        dtz += 2.f * c.fx * p.uxc * itz2 * dJ02;
    } else {
        dtz += c.fx * p.uxc * itz2 * dJ02;
    }
    if (!(flags & 16u)) {
        dty += -c.fy * itz2 * dJ12;
        dtz += 2.f * c.fy * p.uyc * itz2 * dJ12;
    } else {
        dtz += c.fy * p.uyc * itz2 * dJ12;
    }
    // t = R_v μ + t_v
    dmx += R[0] * dtx + R[3] * dty + R[6] * dtz;
    dmy += R[1] * dtx + R[4] * dty + R[7] * dtz;
    dmz += R[2] * dtx + R[5] * dty + R[8] * dtz;
    // colour: rgb = max(0, Σ Y_k(dir) sh_k + 0.5), dir = (μ − c_v)/‖μ − c_v‖
    const float dr0 = (flags & 1u) ? 0.f : pg1.w;
    const float dr1 = (flags & 2u) ? 0.f : pg2.x;
    const float dr2 = (flags & 4u) ? 0.f : pg2.y;
    float x = mx - cam4.x, y = my - cam4.y, z = mz - cam4.z;
    const float idn = rsqrtf(x * x + y * y + z * z);
    x *= idn; y *= idn; z *= idn;
    float wk[NK];  // Σ_c sh[k][c]·∂L/∂rgb_c, read as float4 chunks of the row
#pragma unroll
    for (int kk = 0; kk < NK; kk++) wk[kk] = 0.f;
    {
        const float drc[3] = {dr0, dr1, dr2};
        const float4* sh4 = reinterpret_cast<const float4*>(sh);
#pragma unroll
        for (int i4 = 0; i4 < ShRows<D>::NS4; i4++) {
            const float4 q = sh4[i4];
            const float qe[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int f = 4 * i4 + e;
                if (f < NS) wk[f / 3] += qe[e] * drc[f % 3];
            }
        }
    }
    float Y[NK];
    Y[0] = 0.28209479177387814f;
    float ddx = 0.f, ddy = 0.f, ddz = 0.f;
    if (D >= 1) {
        Y[1] = -g_SH1 * y; Y[2] = g_SH1 * z; Y[3] = -g_SH1 * x;
        ddx += -g_SH1 * wk[3];
        ddy += -g_SH1 * wk[1];
        ddz += g_SH1 * wk[2];
    }
    if (D >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        Y[4] = g_SH2_0 * x * y;
        Y[5] = g_SH2_1 * y * z;
        Y[6] = g_SH2_2 * (2.f * zz - xx - yy);
        Y[7] = g_SH2_3 * x * z;
        Y[8] = g_SH2_4 * (xx - yy);
        ddx += g_SH2_0 * y * wk[4] - 2.f * g_SH2_2 * x * wk[6] + g_SH2_3 * z * wk[7] + 2.f * g_SH2_4 * x * wk[8];
        ddy += g_SH2_0 * x * wk[4] + g_SH2_1 * z * wk[5] - 2.f * g_SH2_2 * y * wk[6] - 2.f * g_SH2_4 * y * wk[8];
        ddz += g_SH2_1 * y * wk[5] + 4.f * g_SH2_2 * z * wk[6] + g_SH2_3 * x * wk[7];
        if (D >= 3) {
            Y[9] = g_SH3_0 * y * (3.f * xx - yy);
            Y[10] = g_SH3_1 * x * y * z;
            Y[11] = g_SH3_2 * y * (4.f * zz - xx - yy);
            Y[12] = g_SH3_3 * z * (2.f * zz - 3.f * xx - 3.f * yy);
            Y[13] = g_SH3_4 * x * (4.f * zz - xx - yy);
            Y[14] = g_SH3_5 * z * (xx - yy);
            Y[15] = g_SH3_6 * x * (xx - 3.f * yy);
            ddx += g_SH3_0 * 6.f * x * y * wk[9] + g_SH3_1 * y * z * wk[10] - g_SH3_2 * 2.f * x * y * wk[11]
                 - g_SH3_3 * 6.f * x * z * wk[12] + g_SH3_4 * (4.f * zz - 3.f * xx - yy) * wk[13]
                 + g_SH3_5 * 2.f * x * z * wk[14] + g_SH3_6 * (3.f * xx - 3.f * yy) * wk[15];
            ddy += g_SH3_0 * (3.f * xx - 3.f * yy) * wk[9] + g_SH3_1 * x * z * wk[10]
                 + g_SH3_2 * (4.f * zz - xx - 3.f * yy) * wk[11] - g_SH3_3 * 6.f * y * z * wk[12]
                 - g_SH3_4 * 2.f * x * y * wk[13] - g_SH3_5 * 2.f * y * z * wk[14]
                 - g_SH3_6 * 6.f * x * y * wk[15];
            ddz += g_SH3_1 * x * y * wk[10] + g_SH3_2 * 8.f * y * z * wk[11]
                 + g_SH3_3 * (6.f * zz - 3.f * xx - 3.f * yy) * wk[12] + g_SH3_4 * 8.f * x * z * wk[13]
                 + g_SH3_5 * (xx - yy) * wk[14];
        }
    }
    {
        const float drc[3] = {dr0, dr1, dr2};
        float4* dsh4 = reinterpret_cast<float4*>(dsh);
#pragma unroll
        for (int i4 = 0; i4 < ShRows<D>::NS4; i4++) {
            float4 q = dsh4[i4];
            float* qe = reinterpret_cast<float*>(&q);
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int f = 4 * i4 + e;
                if (f < NS) qe[e] += Y[f / 3] * drc[f % 3];
            }
            dsh4[i4] = q;
        }
    }
    const float dd = x * ddx + y * ddy + z * ddz;
    dmx += (ddx - x * dd) * idn;
    dmy += (ddy - y * dd) * idn;
    dmz += (ddz - z * dd) * idn;
}

// Σ → (scale, rotation) and the output writes of one Gaussian (row o of the outputs).
__device__ __forceinline__ void finish_gaussian(const Launch& L, const mvgs_grads& gr, const mvgs_adc& adc, int64_t g,
                                                int64_t o, const GAcc& A) {
    const float dmx = A.dmx, dmy = A.dmy, dmz = A.dmz;
    const float G00 = A.G00, G01 = A.G01, G02 = A.G02, G11 = A.G11, G12 = A.G12, G22 = A.G22;
    const float dop = A.dop, e1 = A.e1, e2 = A.e2, gsx = A.gsx, gsy = A.gsy, nvis = A.nvis;
    FastActiv a;  // recomputed: R, s, q are not kept live through the view loop
    fast_activate(L.log_scales + 3 * g, L.quats + 4 * g, L.opac[g], a);
    // Σ = M Mᵀ, M = R diag(s): ∂L/∂M = 2 G M (G symmetric)
    const float* R = a.R;
    const float Gm[9] = {G00, G01, G02, G01, G11, G12, G02, G12, G22};
    float dM[9];
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int cc = 0; cc < 3; cc++) {
            const float Mkc0 = R[0 * 3 + cc] * a.s[cc], Mkc1 = R[1 * 3 + cc] * a.s[cc], Mkc2 = R[2 * 3 + cc] * a.s[cc];
            dM[3 * r + cc] = 2.f * (Gm[3 * r] * Mkc0 + Gm[3 * r + 1] * Mkc1 + Gm[3 * r + 2] * Mkc2);
        }
    float dR[9], dls[3];
#pragma unroll
    for (int cc = 0; cc < 3; cc++) {
        float ds = 0.f;
#pragma unroll
        for (int r = 0; r < 3; r++) {
            ds += dM[3 * r + cc] * R[3 * r + cc];
            dR[3 * r + cc] = dM[3 * r + cc] * a.s[cc];
        }
        dls[cc] = ds * a.s[cc];  // s = exp(λ)
    }
    const float w = a.q[0], x = a.q[1], y = a.q[2], z = a.q[3];
    float dq[4];
    dq[0] = -2.f * z * dR[1] + 2.f * y * dR[2] + 2.f * z * dR[3] - 2.f * x * dR[5] - 2.f * y * dR[6] + 2.f * x * dR[7];
    dq[1] = 2.f * y * dR[1] + 2.f * z * dR[2] + 2.f * y * dR[3] - 4.f * x * dR[4] - 2.f * w * dR[5] + 2.f * z * dR[6]
          + 2.f * w * dR[7] - 4.f * x * dR[8];
    dq[2] = -4.f * y * dR[0] + 2.f * x * dR[1] + 2.f * w * dR[2] + 2.f * x * dR[3] + 2.f * z * dR[5] - 2.f * w * dR[6]
          + 2.f * z * dR[7] - 4.f * y * dR[8];
    dq[3] = -4.f * z * dR[0] - 2.f * w * dR[1] + 2.f * x * dR[2] + 2.f * w * dR[3] - 4.f * z * dR[4] + 2.f * y * dR[5]
          + 2.f * x * dR[6] + 2.f * y * dR[7];
    const float qd = w * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
    // q̂ = q/‖q‖ ⇒ ∂L/∂q = (∂q̂ − q̂(q̂·∂q̂))/‖q‖
#pragma unroll
    for (int k = 0; k < 4; k++) gr.d_quats[4 * o + k] = (dq[k] - a.q[k] * qd) * a.inv_norm;
    gr.d_means[3 * o] = dmx;
    gr.d_means[3 * o + 1] = dmy;
    gr.d_means[3 * o + 2] = dmz;
    gr.d_log_scales[3 * o] = dls[0];
    gr.d_log_scales[3 * o + 1] = dls[1];
    gr.d_log_scales[3 * o + 2] = dls[2];
    gr.d_opacity_logits[o] = dop * a.o * (1.f - a.o);
    adc.e1[o] = e1;
    adc.e2[o] = e2;
    if (adc.e_old || adc.e_old_acc) {
        const float eo = sqrtf(gsx * gsx + gsy * gsy);
        if (adc.e_old) adc.e_old[o] = eo;
        if (adc.e_old_acc) adc.e_old_acc[o] += eo;
    }
    adc.vis[o] = nvis;
    if (adc.gsum) {
        adc.gsum[2 * o] = gsx;
        adc.gsum[2 * o + 1] = gsy;
    }
    if (adc.max_radius && A.rmax > 0.f) adc.max_radius[o] = fmaxf(adc.max_radius[o], A.rmax);
    if (adc.e1_acc) adc.e1_acc[o] += e1;
    if (adc.e2_acc) adc.e2_acc[o] += e2;
    if (adc.denom_acc) adc.denom_acc[o] += nvis;
}

template <int D>
// Gaussians [gbeg, gend) only (gbeg a multiple of BLK): outputs are addressed relative to gbeg,
// so a caller can reduce each finished chunk while the next one computes.
#ifndef MVGS_GB_MINB
#define MVGS_GB_MINB 2  // resident 256-thread CTAs asked of k_gauss_bwd
#endif
__global__ __launch_bounds__(BLK, MVGS_GB_MINB) void k_gauss_bwd(Launch L, mvgs_grads gr, mvgs_adc adc, int64_t gbeg,
                                                                 int64_t gend) {
    constexpr int NS = ShRows<D>::NS, SS = ShRows<D>::STRIDE;
    constexpr int VB = GB_VB;
    constexpr int NS4 = NS / 4 > 0 ? NS / 4 : 1;  // float4 per row when NS % 4 == 0
    extern __shared__ float4 smem_sh4[];  // 16-byte aligned base
    float* smem_sh = reinterpret_cast<float*>(smem_sh4);
    float* dsh_s = smem_sh;                              // [BLK][SS]
    float* sh_s = smem_sh + BLK * SS;                    // [BLK][SS] staged SH rows
    __shared__ int wc[BLK / 32][32];
    __shared__ float4 scam[32];  // per view of the chunk: camera centre (x, y, z), Jacobian clamp limit x
    __shared__ float scl[32];    // clamp limit y
    __shared__ mvgs_camera scams[32];  // the chunk's cameras (LDS in the per-pair chain)
    __shared__ int sboff[32];  // first pair slot of this block in each view of the chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int blk = blockIdx.x + (int)(gbeg / BLK);  // 256-Gaussian block of the pair-slot allocation
    const int64_t g0 = (int64_t)blk * BLK;
    const int64_t g = g0 + threadIdx.x;
    const int64_t o = g - gbeg;  // output row
    const bool valid = g < gend;
    {  // SH rows: coalesced async copies (no registers, all in flight), waited on before first use
        const int nb = (int)min((int64_t)BLK, gend - g0);
        const float* src = L.sh + g0 * (int64_t)L.sh_stride * 3;
        const int rowlen = L.sh_stride * 3;
        if ((rowlen & 3) == 0 && (NS & 3) == 0 && ((uintptr_t)src & 15) == 0) {
            for (int i = threadIdx.x; i < nb * NS4; i += BLK) {
                const int r = i / NS4, k = 4 * (i - r * NS4);
                cp_async16(&sh_s[r * SS + k], src + (int64_t)r * rowlen + k);
            }
        } else {
            for (int i = threadIdx.x; i < nb * NS; i += BLK) {
                const int r = i / NS, k = i - r * NS;  // NS constexpr: mul-shift
                cp_async4(&sh_s[r * SS + k], src + (int64_t)r * rowlen + k);
            }
        }
        cp_async_commit();
    }
    {
        float4* z4 = reinterpret_cast<float4*>(dsh_s);
        for (int i = threadIdx.x; i < BLK * SS / 4; i += BLK) z4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // SH row of this Gaussian: staged copy, or global (16-byte aligned: checked by the launcher)
    const float* sh = sh_s + threadIdx.x * SS;
    float* dsh = dsh_s + threadIdx.x * SS;
    float mx = 0.f, my = 0.f, mz = 0.f, smax = 0.f;
    float Sg[6];  // Σ (only Σ is needed in the view loop)
    {
        FastActiv a;
        if (valid) {
            mx = L.means[3 * g];
            my = L.means[3 * g + 1];
            mz = L.means[3 * g + 2];
            smax = participation_smax(L.log_scales[3 * g], L.log_scales[3 * g + 1], L.log_scales[3 * g + 2]);
            fast_activate(L.log_scales + 3 * g, L.quats + 4 * g, L.opac[g], a);
        } else {
            fast_activate(L.log_scales, L.quats, 0.f, a);  // any finite values; unused
        }
#pragma unroll
        for (int k = 0; k < 6; k++) Sg[k] = a.Sig[k];
    }
    GAcc A;
    const float sW = 2.0f / (float)L.W, sH = 2.0f / (float)L.H;
    bool sh_ready = false;  // SH rows arrive asynchronously; waited on after the first view loads
    for (int v0 = 0; v0 < L.V; v0 += 32) {
        const int nv = min(32, L.V - v0);
        // participation in the chunk's views: k_count's bits when stored (as in k_project)
        unsigned pm = 0;
        if (L.pmask) {
            pm = valid ? L.pmask[g] : 0u;
        } else {
            for (int k = 0; k < nv; k++)
                pm |= (valid && ca_participates(L.cams[v0 + k], mx, my, mz, smax, L.TX, L.TY)) ? 1u << k : 0u;
        }
        for (int k = 0; k < nv; k++) {
            const unsigned bal = __ballot_sync(FULLG, (pm >> k) & 1u);
            if (lane == 0) wc[warp][k] = __popc(bal);
        }
        for (int i = threadIdx.x; i < nv * (int)(sizeof(mvgs_camera) / 4); i += BLK)
            reinterpret_cast<uint32_t*>(scams)[i] = reinterpret_cast<const uint32_t*>(L.cams + v0)[i];
        if (threadIdx.x < nv) {
            sboff[threadIdx.x] = L.blk_off[(int64_t)(v0 + threadIdx.x) * L.NB + blk];
            const mvgs_camera& c = L.cams[v0 + threadIdx.x];
            const float* R = c.R;  // centre −Rᵀt and the clamp limits 0.65·W/fx, 0.65·H/fy (R4)
            scam[threadIdx.x] = make_float4(-(R[0] * c.t[0] + R[3] * c.t[1] + R[6] * c.t[2]),
                                            -(R[1] * c.t[0] + R[4] * c.t[1] + R[7] * c.t[2]),
                                            -(R[2] * c.t[0] + R[5] * c.t[1] + R[8] * c.t[2]),
                                            0.65f * (float)c.width / c.fx);
            scl[threadIdx.x] = 0.65f * (float)c.height / c.fy;
        }
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
        for (int k0 = 0; k0 < nv; k0 += VB) {
            // issue the loads of up to GB_VB views first (memory-level parallelism), then the math
            uint32_t fl[VB];
            float4 pga[VB], pgb[VB], pgc[VB];
#pragma unroll
            for (int u = 0; u < VB; u++) {
                fl[u] = 0u;
                const int k = k0 + u;
                if (k >= nv) continue;  // warp-uniform
                const bool zvis = (pm >> k) & 1u;
                const unsigned bal = __ballot_sync(FULLG, zvis);
                if (!zvis) continue;
                const int64_t pair = (int64_t)sboff[k] + wc[warp][k] + __popc(bal & lt);
                if (pair >= L.cap_pairs) continue;
                // the gradient slot carries the pair's flags word in float PG_FLAGS (the slot of an
                // inert pair holds zeros and its flags, which say it is inert)
                const float4* pgp = reinterpret_cast<const float4*>(L.pgrad + pair * PG_STRIDE);
                pga[u] = pgp[0];
                pgb[u] = pgp[1];
                pgc[u] = pgp[2];
                fl[u] = __float_as_uint(pgc[u].z);
            }
#if GB_PREFETCH
            // the next GB_PREFETCH views' gradient slots toward L2 while this view computes
#pragma unroll
            for (int pd = 1; pd <= GB_PREFETCH; pd++) {
                const int kn = k0 + pd * VB;
                if (kn < nv) {
                    const bool zn = (pm >> kn) & 1u;
                    const unsigned baln = __ballot_sync(FULLG, zn);
                    if (zn) {
                        const int64_t pn = (int64_t)sboff[kn] + wc[warp][kn] + __popc(baln & lt);
                        if (pn < L.cap_pairs) asm volatile("prefetch.global.L2 [%0];" ::"l"(L.pgrad + pn * PG_STRIDE));
                    }
                }
            }
#endif
            if (!sh_ready) {  // block-uniform: overlap the SH copy with the first pair loads
                cp_async_wait_all();
                __syncthreads();
                sh_ready = true;
            }
#pragma unroll
            for (int u = 0; u < VB; u++) {
            if (!(fl[u] & PF_VISIBLE)) continue;  // not participating, or tiles == 0: inert (R27)
            const mvgs_camera& c = scams[k0 + u];
            const uint32_t flags = fl[u];
            const float4 pg0 = pga[u], pg1 = pgb[u], pg2 = pgc[u];
            pair_chain<D>(c, scam[k0 + u], scl[k0 + u], flags, pg0, pg1, pg2, mx, my, mz, Sg, sh, dsh, sW, sH, A);
            }
        }
        __syncthreads();
    }
    if (!sh_ready) {  // no view chunk ran (V == 0 cannot happen, but keep the copy complete)
        cp_async_wait_all();
        __syncthreads();
    }
    // coalesced store of the SH gradient rows (coefficients above the active degree are 0)
    {
        const int nb = (int)min((int64_t)BLK, gend - g0);
        float* dst = gr.d_sh + (g0 - gbeg) * (int64_t)L.sh_stride * 3;
        const int rowlen = L.sh_stride * 3;
        if (rowlen == NS && (NS & 3) == 0 && ((uintptr_t)dst & 15) == 0) {  // float4 rows, constant divisor
            float4* dst4 = reinterpret_cast<float4*>(dst);
            for (int i = threadIdx.x; i < nb * NS4; i += BLK) {
                const int r = i / NS4, k4 = i - r * NS4;
                dst4[i] = *reinterpret_cast<const float4*>(&dsh_s[r * SS + 4 * k4]);
            }
        } else if (rowlen == NS) {  // rows hold exactly the active coefficients: constant divisor
            for (int i = threadIdx.x; i < nb * NS; i += BLK) {
                const int r = i / NS, k = i - r * NS;
                dst[i] = dsh_s[r * SS + k];
            }
        } else {
            for (int r = warp; r < nb; r += BLK / 32)
                for (int k = lane; k < rowlen; k += 32) dst[(int64_t)r * rowlen + k] = k < NS ? dsh_s[r * SS + k] : 0.f;
        }
    }
    if (!valid) return;
    finish_gaussian(L, gr, adc, g, o, A);
}

template <int D>
cudaError_t launch_gauss_bwd_t(const Launch& L, const mvgs_grads& gr, const mvgs_adc& adc, int64_t gb, int64_t ge,
                               cudaStream_t s) {
    const size_t smem = sizeof(float) * 2 * BLK * ShRows<D>::STRIDE;
    cudaError_t e = cudaFuncSetAttribute(k_gauss_bwd<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nblk = (int)((ge - gb + BLK - 1) / BLK);
    if (nblk > 0) k_gauss_bwd<D><<<nblk, BLK, smem, s>>>(L, gr, adc, gb, ge);
    return cudaGetLastError();
}

cudaError_t launch_gauss_bwd(const Launch& L, const mvgs_grads& gr, const mvgs_adc& adc, int64_t gb, int64_t ge,
                             cudaStream_t s) {
    switch (L.sh_degree) {
        case 0: return launch_gauss_bwd_t<0>(L, gr, adc, gb, ge, s);
        case 1: return launch_gauss_bwd_t<1>(L, gr, adc, gb, ge, s);
        case 2: return launch_gauss_bwd_t<2>(L, gr, adc, gb, ge, s);
        default: return launch_gauss_bwd_t<3>(L, gr, adc, gb, ge, s);
    }
}

// E_old = ‖Σ_views Σ_pixels ∇_{p_i}L‖ from the summed vector gsum [P,2] (R49): after a
// multi-GPU sum of gsum, every rank's E_old is the single-GPU one.
__global__ void k_e_old(const float* __restrict__ gsum, int64_t n, float* __restrict__ e_old,
                        float* __restrict__ e_old_acc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float2 v = reinterpret_cast<const float2*>(gsum)[i];
    const float e = sqrtf(v.x * v.x + v.y * v.y);
    if (e_old) e_old[i] = e;
    if (e_old_acc) e_old_acc[i] += e;
}

cudaError_t launch_e_old(const float* gsum, int64_t n, float* e_old, float* e_old_acc, cudaStream_t s) {
    if (n > 0) k_e_old<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(gsum, n, e_old, e_old_acc);
    return cudaGetLastError();
}

}  // namespace mvgs
