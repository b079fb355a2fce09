// ca.cuh — canonical fp32 arithmetic for every value that
// feeds a discrete decision: activations, Σ, camera transform, EWA Σ',
// conic, radius, tile rect, power, G, α, T.  Every operation is an explicit
// round-to-nearest intrinsic, so nvcc can neither contract nor reorder it;
// the result is bit-identical to any other implementation of the contract.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/mvgs.h"

namespace mvgs {

#define FADD __fadd_rn
#define FSUB __fsub_rn
#define FMUL __fmul_rn
#define FDIV __fdiv_rn
#define FMA __fmaf_rn
#define FSQRT __fsqrt_rn

constexpr int TILE = 16;
constexpr float ALPHA_MIN = 1.0f / 255.0f;  // R12
constexpr float ALPHA_MAX = 0.99f;          // R11
constexpr float T_EPS = 1e-4f;              // R13

// §4.3 canonical exp, core for x ∈ [−87, 88] (no range checks).  The compositing
// kernels only evaluate it for power ∈ [−ln(255)−1e-3, 0] (skip bound, §4.5), where it
// is bit-identical to ca_exp.
// n = the integer nearest (ties to even) to the exact x·log2e: fma onto the 1.5·2²³ grid.
constexpr float CA_MAGIC = 12582912.0f;  // 1.5·2²³
__device__ __forceinline__ float ca_exp_core(float x) {
    float n = FSUB(FMA(x, 1.44269504f, CA_MAGIC), CA_MAGIC);
    float r = FMA(n, -0.693145751953125f, x);
    r = FMA(n, -1.428606765330187e-6f, r);
    float p = (float)(1.0 / 720.0);
    p = FMA(p, r, (float)(1.0 / 120.0));
    p = FMA(p, r, (float)(1.0 / 24.0));
    p = FMA(p, r, (float)(1.0 / 6.0));
    p = FMA(p, r, 0.5f);
    p = FMA(p, r, 1.0f);
    p = FMA(p, r, 1.0f);
    return FMUL(p, __int_as_float((__float2int_rn(n) + 127) << 23));
}

// §4.3 canonical exp.
__device__ __forceinline__ float ca_exp(float x) {
    if (x < -87.0f) return 0.0f;
    if (x > 88.0f) return __int_as_float(0x7f800000);
    float n = FSUB(FMA(x, 1.44269504f, CA_MAGIC), CA_MAGIC);
    float r = FMA(n, -0.693145751953125f, x);
    r = FMA(n, -1.428606765330187e-6f, r);
    float p = (float)(1.0 / 720.0);
    p = FMA(p, r, (float)(1.0 / 120.0));
    p = FMA(p, r, (float)(1.0 / 24.0));
    p = FMA(p, r, (float)(1.0 / 6.0));
    p = FMA(p, r, 0.5f);
    p = FMA(p, r, 1.0f);
    p = FMA(p, r, 1.0f);
    return FMUL(p, __int_as_float((__float2int_rn(n) + 127) << 23));
}

__device__ __forceinline__ float ca_dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return FMA(a2, b2, FMA(a1, b1, FMUL(a0, b0)));
}

// Per-Gaussian activations (§4.2): opacity, scales, normalised quaternion,
// R(q̂), Σ = (R S)(R S)ᵀ upper triangle {00,01,02,11,12,22}.
struct Activ {
    float o;
    float s[3];
    float q[4];     // normalised (w,x,y,z)
    float inv_norm; // 1/‖q‖
    float R[9];
    float Sig[6];
};

__device__ __forceinline__ void ca_activate(const float* __restrict__ ls, const float* __restrict__ qr, float logit,
                                            Activ& a) {
    a.o = FDIV(1.0f, FADD(1.0f, ca_exp(-logit)));
    a.s[0] = ca_exp(ls[0]);
    a.s[1] = ca_exp(ls[1]);
    a.s[2] = ca_exp(ls[2]);
    float w = qr[0], x = qr[1], y = qr[2], z = qr[3];
    float n2 = FMA(z, z, FMA(y, y, FMA(x, x, FMUL(w, w))));
    float inv = FDIV(1.0f, FSQRT(n2));
    a.inv_norm = inv;
    w = FMUL(w, inv); x = FMUL(x, inv); y = FMUL(y, inv); z = FMUL(z, inv);
    a.q[0] = w; a.q[1] = x; a.q[2] = y; a.q[3] = z;
    float* R = a.R;
    R[0] = FMA(-2.0f, FMA(y, y, FMUL(z, z)), 1.0f);
    R[1] = FMUL(2.0f, FMA(x, y, -FMUL(w, z)));
    R[2] = FMUL(2.0f, FMA(x, z, FMUL(w, y)));
    R[3] = FMUL(2.0f, FMA(x, y, FMUL(w, z)));
    R[4] = FMA(-2.0f, FMA(x, x, FMUL(z, z)), 1.0f);
    R[5] = FMUL(2.0f, FMA(y, z, -FMUL(w, x)));
    R[6] = FMUL(2.0f, FMA(x, z, -FMUL(w, y)));
    R[7] = FMUL(2.0f, FMA(y, z, FMUL(w, x)));
    R[8] = FMA(-2.0f, FMA(x, x, FMUL(y, y)), 1.0f);
    float M[9];
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int c = 0; c < 3; c++) M[3 * r + c] = FMUL(R[3 * r + c], a.s[c]);
    a.Sig[0] = ca_dot3(M[0], M[1], M[2], M[0], M[1], M[2]);
    a.Sig[1] = ca_dot3(M[0], M[1], M[2], M[3], M[4], M[5]);
    a.Sig[2] = ca_dot3(M[0], M[1], M[2], M[6], M[7], M[8]);
    a.Sig[3] = ca_dot3(M[3], M[4], M[5], M[3], M[4], M[5]);
    a.Sig[4] = ca_dot3(M[3], M[4], M[5], M[6], M[7], M[8]);
    a.Sig[5] = ca_dot3(M[6], M[7], M[8], M[6], M[7], M[8]);
}

// Camera-space depth only (participation test, §4.2): t.z = R2·μ + t_z.
__device__ __forceinline__ float ca_depth(const mvgs_camera& c, float mx, float my, float mz) {
    return FMA(c.R[8], mz, FMA(c.R[7], my, FMA(c.R[6], mx, c.t[2])));
}

// Participation (S1: "determines which Gaussians participate in rendering for each
// viewpoint … memory is allocated only for these"): the CA z-test (R27) and, on top of it, a
// conservative off-screen test that can only drop pairs whose tile rect is provably empty
// (DESIGN.md §4.9).  With r ≤ ⌈3·√(a + c + 0.32)⌉ and a + c ≤ ‖J‖²_F·s²_max + 0.6 (Σ' = JWΣWᵀJᵀ
// + 0.3·I, W a rotation, λ_max(Σ) = s²_max), rect x is empty when px + r < 1 or
// px − r ≥ 16·TX (same for y); the bound is inflated by 0.1 % and 2 px.  Every operation is an
// explicit intrinsic (RN arithmetic, MUFU approximations; no contraction), so each kernel that
// re-derives the pair slots takes the same decision.  smax = participation_smax(log_scales).
__device__ __forceinline__ float participation_smax(float l0, float l1, float l2) {
    return FMUL(__expf(fmaxf(l0, fmaxf(l1, l2))), 1.001f);
}

__device__ __forceinline__ float pt_rcp(float x) {  // MUFU.RCP: deterministic, ≤ 1 ulp
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float pt_sqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-camera constants of the bound (computed by one code path for every caller).
struct PartCam {
    float limx, limy;  // Jacobian clamp limits 0.65·W/fx, 0.65·H/fy (R4)
    float fx2, fy2;
    float xmax, ymax;  // 16·TX, 16·TY
};

__device__ __forceinline__ PartCam make_partcam(const mvgs_camera& c, int TX, int TY) {
    PartCam p;
    p.limx = FMUL(FMUL(0.65f, __int2float_rn(c.width)), pt_rcp(c.fx));
    p.limy = FMUL(FMUL(0.65f, __int2float_rn(c.height)), pt_rcp(c.fy));
    p.fx2 = FMUL(c.fx, c.fx);
    p.fy2 = FMUL(c.fy, c.fy);
    p.xmax = 16.0f * (float)TX;
    p.ymax = 16.0f * (float)TY;
    return p;
}

__device__ __forceinline__ bool ca_participates(const mvgs_camera& c, const PartCam& pc, float mx, float my, float mz,
                                                float smax) {
    const float tz = FMA(c.R[8], mz, FMA(c.R[7], my, FMA(c.R[6], mx, c.t[2])));  // the CA z-test (R27)
    if (!(tz > c.znear)) return false;
    // the bound: approximate but deterministic operations; their errors (≲ 1e-6 relative)
    // sit far inside the 0.1 % + 2 px slack
    const float tx = FMA(c.R[2], mz, FMA(c.R[1], my, FMA(c.R[0], mx, c.t[0])));
    const float ty = FMA(c.R[5], mz, FMA(c.R[4], my, FMA(c.R[3], mx, c.t[1])));
    const float itz = pt_rcp(tz);
    const float ux = FMUL(tx, itz), uy = FMUL(ty, itz);
    const float px = FMA(c.fx, ux, c.cx), py = FMA(c.fy, uy, c.cy);
    const float cux = fminf(fabsf(ux), pc.limx), cuy = fminf(fabsf(uy), pc.limy);
    const float jf = FMUL(FADD(FMUL(pc.fx2, FMA(cux, cux, 1.0f)), FMUL(pc.fy2, FMA(cuy, cuy, 1.0f))),
                          FMUL(itz, itz));  // ‖J‖²_F
    const float tr = FMA(FMUL(jf, FMUL(smax, smax)), 1.001f, 0.92f);
    const float rub = FMA(3.0f, pt_sqrt(tr), 2.0f);  // > r, incl. the ceil
    if (!(rub < 1e30f)) return true;                 // overflow / NaN: keep the pair
    if (FADD(px, rub) < 1.0f || FSUB(px, rub) > pc.xmax) return false;
    if (FADD(py, rub) < 1.0f || FSUB(py, rub) > pc.ymax) return false;
    return true;
}

__device__ __forceinline__ bool ca_participates(const mvgs_camera& c, float mx, float my, float mz, float smax,
                                                int TX, int TY) {
    const PartCam pc = make_partcam(c, TX, TY);
    return ca_participates(c, pc, mx, my, mz, smax);
}

// Per (Gaussian, view) projection state (§4.2).
struct Proj {
    float tx, ty, tz;
    float px, py;
    float uxc, uyc;  // clamped t.xy/t.z
    int clx, cly;    // clamp active (R4)
    float J00, J02, J11, J12;
    float T0[3], T1[3];
    float a, b, c, det;
    float A, B, C;
    int ok;          // det > 0
    int radius;
    int rx0, ry0, rx1, ry1;
};

__device__ __forceinline__ int ca_clamp_tile(float v, int tmax) {
    if (!(v > 0.0f)) return 0;
    if (v >= __int2float_rn(tmax)) return tmax;
    return __float2int_rz(v);
}

// Jacobian clamp limits of a camera (R4): 0.65·W/fx, 0.65·H/fy in CA arithmetic (per camera)
__device__ __forceinline__ float2 ca_clamp_limits(const mvgs_camera& c) {
    return make_float2(FDIV(FMUL(0.65f, __int2float_rn(c.width)), c.fx),
                       FDIV(FMUL(0.65f, __int2float_rn(c.height)), c.fy));
}

__device__ __forceinline__ void ca_project(const mvgs_camera& c, float mx, float my, float mz,
                                           const float Sig[6], int TX, int TY, float2 lim, Proj& p) {
    const float* R = c.R;
    p.tx = FMA(R[2], mz, FMA(R[1], my, FMA(R[0], mx, c.t[0])));
    p.ty = FMA(R[5], mz, FMA(R[4], my, FMA(R[3], mx, c.t[1])));
    p.tz = FMA(R[8], mz, FMA(R[7], my, FMA(R[6], mx, c.t[2])));
    float ux = FDIV(p.tx, p.tz), uy = FDIV(p.ty, p.tz);
    p.px = FMA(c.fx, ux, c.cx);
    p.py = FMA(c.fy, uy, c.cy);
    const float limx = lim.x, limy = lim.y;
    p.uxc = fminf(limx, fmaxf(-limx, ux));
    p.uyc = fminf(limy, fmaxf(-limy, uy));
    p.clx = (ux > limx) || (ux < -limx);
    p.cly = (uy > limy) || (uy < -limy);
    p.J00 = FDIV(c.fx, p.tz);
    p.J02 = FDIV(-FMUL(c.fx, p.uxc), p.tz);
    p.J11 = FDIV(c.fy, p.tz);
    p.J12 = FDIV(-FMUL(c.fy, p.uyc), p.tz);
#pragma unroll
    for (int j = 0; j < 3; j++) {
        p.T0[j] = FMA(p.J02, R[6 + j], FMUL(p.J00, R[j]));
        p.T1[j] = FMA(p.J12, R[6 + j], FMUL(p.J11, R[3 + j]));
    }
    // U = T Σ (columns of Σ: (S0,S1,S2), (S1,S3,S4), (S2,S4,S5))
    float U00 = ca_dot3(p.T0[0], p.T0[1], p.T0[2], Sig[0], Sig[1], Sig[2]);
    float U01 = ca_dot3(p.T0[0], p.T0[1], p.T0[2], Sig[1], Sig[3], Sig[4]);
    float U02 = ca_dot3(p.T0[0], p.T0[1], p.T0[2], Sig[2], Sig[4], Sig[5]);
    float U10 = ca_dot3(p.T1[0], p.T1[1], p.T1[2], Sig[0], Sig[1], Sig[2]);
    float U11 = ca_dot3(p.T1[0], p.T1[1], p.T1[2], Sig[1], Sig[3], Sig[4]);
    float U12 = ca_dot3(p.T1[0], p.T1[1], p.T1[2], Sig[2], Sig[4], Sig[5]);
    p.a = FADD(ca_dot3(U00, U01, U02, p.T0[0], p.T0[1], p.T0[2]), 0.3f);
    p.b = ca_dot3(U00, U01, U02, p.T1[0], p.T1[1], p.T1[2]);
    p.c = FADD(ca_dot3(U10, U11, U12, p.T1[0], p.T1[1], p.T1[2]), 0.3f);
    p.det = FMA(p.a, p.c, -FMUL(p.b, p.b));
    p.ok = p.det > 0.0f;
    p.radius = 0;
    p.rx0 = p.ry0 = p.rx1 = p.ry1 = 0;
    p.A = p.B = p.C = 0.0f;
    if (!p.ok) return;
    float id = FDIV(1.0f, p.det);
    p.A = FMUL(p.c, id);
    p.B = FMUL(-p.b, id);
    p.C = FMUL(p.a, id);
    float mid = FMUL(0.5f, FADD(p.a, p.c));
    float l1 = FADD(mid, FSQRT(fmaxf(0.1f, FMA(mid, mid, -p.det))));
    float rf = ceilf(FMUL(3.0f, FSQRT(l1)));
    int r = rf >= 1073741824.0f ? 1073741824 : __float2int_rz(rf);
    p.radius = r;
    float fr = __int2float_rn(r);
    p.rx0 = ca_clamp_tile(FMUL(FSUB(p.px, fr), 0.0625f), TX);
    p.ry0 = ca_clamp_tile(FMUL(FSUB(p.py, fr), 0.0625f), TY);
    p.rx1 = ca_clamp_tile(FMUL(FADD(FADD(p.px, fr), 15.0f), 0.0625f), TX);
    p.ry1 = ca_clamp_tile(FMUL(FADD(FADD(p.py, fr), 15.0f), 0.0625f), TY);
}

// power at pixel offset d = μ' − p (§4.2).
__device__ __forceinline__ float ca_power(float A, float B, float C, float dx, float dy) {
    return FMA(-0.5f, FMA(FMUL(A, dx), dx, FMUL(FMUL(C, dy), dy)), -FMUL(FMUL(B, dx), dy));
}

// 4-byte global→shared async copy (LDGSTS), completion via cp_async_wait_all().
__device__ __forceinline__ void cp_async4(float* smem_dst, const float* gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
// 16-byte global→shared async copy (both addresses 16-byte aligned).
__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

}  // namespace mvgs
