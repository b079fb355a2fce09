/*
 * oracle.c — the parity ORACLE for mvgs.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * constant table or helper with paper_2506_12727_b200/csrc (the CUDA path);
 * both implement the same written contract independently.
 *
 * What it computes — a plain, slow, per-pixel sorted-list compositor with its
 * analytic adjoint (PAPER.md line numbers as P:n):
 *   O1  activations and Σ = R S Sᵀ Rᵀ ........................ P:75
 *   O2  per (Gaussian, view) EWA projection → μ', Σ', conic, radius, tile
 *       rect, SH colour ................................. P:75
 *   O3  list of every (view, tile): pairs whose tile rect contains it, one
 *       entry per tile covered ("duplicating") .......... P:576
 *   O4  order inside a list by (depth, gaussian id) — the (view, tile,
 *       depth) key of P:579 with ties broken by id (R10)
 *   O5  per-pixel front-to-back blending, Eq. (1) ..... P:76–82; Alg. 2
 *   O6  per-pixel adjoint of Eq. (1) → ∂L/∂(μ', conic, o, rgb) per pair,
 *       ∇_{p_i}L in NDC (B.2)
 *   O7  per-Gaussian chain rule; the multi-view mini-batch gradient is the
 *       sum over the batch's views ...................... P:136–139
 *   O8  E_old, E1, E2 ............................................ P:14–21
 *
 * Precision.  Values and gradients are fp64.  Every decision that turns a
 * float into an integer or a branch — participation (t.z > znear), det > 0,
 * radius, tile rect, depth key, α < 1/255 skip, α clamp at 0.99, early
 * termination T < 1e-4 — is taken in fp32 under the canonical arithmetic
 * (CA) contract of DESIGN.md §4, i.e. in the precision the kernel takes it
 * in.  The fp32 CA chain below (`*32` functions) exists only to take those
 * decisions; the fp64 chain (`*64`) produces every reported value.
 *
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (no contraction, IEEE float on SSE, denormals kept).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ types */
typedef struct { /* same bytes as synth.CAM_DTYPE (its own definition) */
    float R[9];  /* world→camera rotation, row-major: x_c = R x + t        */
    float t[3];
    float fx, fy, cx, cy;
    int32_t width, height;
    float znear;
} og_cam;

typedef struct {
    int64_t P;
    int32_t sh_degree; /* active degree, ≤ 3 */
    int32_t sh_stride; /* coefficients per Gaussian, (max degree+1)^2 */
    const float *means, *log_scales, *quats, *opacity_logits, *sh;
} og_scene;

enum { OG_NO_EARLY_TERMINATION = 1 };

/* ============================================================= fp32 CA chain
 * DESIGN.md §4.  Every line below is one correctly rounded IEEE fp32 op or an
 * explicit fmaf; nothing is contracted (-ffp-contract=off).                  */

/* CA exp: range reduction by n = the integer nearest (ties to
 * even) to the EXACT product x·log2e — one fused rounding onto the integer grid,
 * fma(x, log2e, 1.5·2^23) − 1.5·2^23 — then two-step Cody–Waite with
 * ln2 = hi + lo, degree-6 Taylor/Horner, scale by 2^n built from exponent bits. */
float oracle_ca_exp(float x)
{
    if (x < -87.0f) return 0.0f;
    if (x > 88.0f) return INFINITY;
    float n = fmaf(x, 1.44269504f, 12582912.0f) - 12582912.0f;
    float r = fmaf(n, -0.693145751953125f, x);
    r = fmaf(n, -1.428606765330187e-6f, r);
    float p = (float)(1.0 / 720.0);
    p = fmaf(p, r, (float)(1.0 / 120.0));
    p = fmaf(p, r, (float)(1.0 / 24.0));
    p = fmaf(p, r, (float)(1.0 / 6.0));
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    union { uint32_t u; float f; } s;
    s.u = (uint32_t)((int)n + 127) << 23;
    return p * s.f;
}

static float dot3f(const float a[3], const float b[3])
{
    return fmaf(a[2], b[2], fmaf(a[1], b[1], a[0] * b[0]));
}

/* O1 in fp32: opacity and 3D covariance (upper triangle 00,01,02,11,12,22). */
static void activate32(const og_scene *g, int64_t i, float *o, float Sig[6])
{
    *o = 1.0f / (1.0f + oracle_ca_exp(-g->opacity_logits[i]));
    float s[3];
    for (int k = 0; k < 3; k++) s[k] = oracle_ca_exp(g->log_scales[3 * i + k]);
    float w = g->quats[4 * i + 0], x = g->quats[4 * i + 1];
    float y = g->quats[4 * i + 2], z = g->quats[4 * i + 3];
    float n2 = fmaf(z, z, fmaf(y, y, fmaf(x, x, w * w)));
    float inv = 1.0f / sqrtf(n2);
    w = w * inv; x = x * inv; y = y * inv; z = z * inv;
    float R[3][3];
    R[0][0] = fmaf(-2.0f, fmaf(y, y, z * z), 1.0f);
    R[0][1] = 2.0f * fmaf(x, y, -(w * z));
    R[0][2] = 2.0f * fmaf(x, z, w * y);
    R[1][0] = 2.0f * fmaf(x, y, w * z);
    R[1][1] = fmaf(-2.0f, fmaf(x, x, z * z), 1.0f);
    R[1][2] = 2.0f * fmaf(y, z, -(w * x));
    R[2][0] = 2.0f * fmaf(x, z, -(w * y));
    R[2][1] = 2.0f * fmaf(y, z, w * x);
    R[2][2] = fmaf(-2.0f, fmaf(x, x, y * y), 1.0f);
    float M[3][3];
    for (int a = 0; a < 3; a++)
        for (int b = 0; b < 3; b++) M[a][b] = R[a][b] * s[b];
    Sig[0] = dot3f(M[0], M[0]);
    Sig[1] = dot3f(M[0], M[1]);
    Sig[2] = dot3f(M[0], M[2]);
    Sig[3] = dot3f(M[1], M[1]);
    Sig[4] = dot3f(M[1], M[2]);
    Sig[5] = dot3f(M[2], M[2]);
}

typedef struct {
    int zvis;            /* participates: t.z > znear (pair allocated) */
    int vis;             /* zvis && det > 0 && tiles > 0                       */
    float tz;            /* depth (sort key)                                    */
    float px, py;        /* μ' in pixels                                        */
    float A, B, C;       /* conic                                               */
    int radius;
    int rx0, ry0, rx1, ry1;
    int tiles;
} p32_t;

static int clamp_tile(float v, int tmax)
{
    if (!(v > 0.0f)) return 0;
    if (v >= (float)tmax) return tmax;
    return (int)v;
}

/* O2 in fp32 (decisions only). */
static void project32(const float mu[3], const float Sig[6], const og_cam *c, p32_t *p)
{
    memset(p, 0, sizeof *p);
    const float *R = c->R;
    float tx = fmaf(R[2], mu[2], fmaf(R[1], mu[1], fmaf(R[0], mu[0], c->t[0])));
    float ty = fmaf(R[5], mu[2], fmaf(R[4], mu[1], fmaf(R[3], mu[0], c->t[1])));
    float tz = fmaf(R[8], mu[2], fmaf(R[7], mu[1], fmaf(R[6], mu[0], c->t[2])));
    p->tz = tz;
    if (!(tz > c->znear)) return;
    p->zvis = 1;
    float ux = tx / tz, uy = ty / tz;
    p->px = fmaf(c->fx, ux, c->cx);
    p->py = fmaf(c->fy, uy, c->cy);
    float limx = (0.65f * (float)c->width) / c->fx;
    float limy = (0.65f * (float)c->height) / c->fy;
    float uxc = fminf(limx, fmaxf(-limx, ux));
    float uyc = fminf(limy, fmaxf(-limy, uy));
    float J00 = c->fx / tz, J02 = -(c->fx * uxc) / tz;
    float J11 = c->fy / tz, J12 = -(c->fy * uyc) / tz;
    float T0[3], T1[3];
    for (int j = 0; j < 3; j++) {
        T0[j] = fmaf(J02, R[6 + j], J00 * R[j]);
        T1[j] = fmaf(J12, R[6 + j], J11 * R[3 + j]);
    }
    const float col0[3] = {Sig[0], Sig[1], Sig[2]};
    const float col1[3] = {Sig[1], Sig[3], Sig[4]};
    const float col2[3] = {Sig[2], Sig[4], Sig[5]};
    float U0[3] = {dot3f(T0, col0), dot3f(T0, col1), dot3f(T0, col2)};
    float U1[3] = {dot3f(T1, col0), dot3f(T1, col1), dot3f(T1, col2)};
    float a = dot3f(U0, T0) + 0.3f;
    float b = dot3f(U0, T1);
    float cc = dot3f(U1, T1) + 0.3f;
    float det = fmaf(a, cc, -(b * b));
    if (!(det > 0.0f)) return;
    float id = 1.0f / det;
    p->A = cc * id;
    p->B = -b * id;
    p->C = a * id;
    float mid = 0.5f * (a + cc);
    float l1 = mid + sqrtf(fmaxf(0.1f, fmaf(mid, mid, -det)));
    float rf = ceilf(3.0f * sqrtf(l1));
    int r = rf >= 1073741824.0f ? 1073741824 : (int)rf;
    p->radius = r;
    int TX = (c->width + 15) / 16, TY = (c->height + 15) / 16;
    float fr = (float)r;
    p->rx0 = clamp_tile((p->px - fr) * 0.0625f, TX);
    p->ry0 = clamp_tile((p->py - fr) * 0.0625f, TY);
    p->rx1 = clamp_tile(((p->px + fr) + 15.0f) * 0.0625f, TX);
    p->ry1 = clamp_tile(((p->py + fr) + 15.0f) * 0.0625f, TY);
    p->tiles = (p->rx1 - p->rx0) * (p->ry1 - p->ry0);
    p->vis = p->tiles > 0;
}

/* O2 colour in fp32 (decision only: the SH clamp rgb < 0, R17, §4.4).
 * dir = (μ − c_v)/‖μ − c_v‖ with c_v = −R_vᵀ t_v; real SH basis in [3DGS] order,
 * each Y_k one fixed sequence of fp32 products/differences; acc = 0.5 then
 * acc = fma(Y_k, sh_k, acc) for k ascending.  clamped[ch] = acc < 0.            */
static void color32(const og_scene *g, int64_t i, const og_cam *c, int clamped[3], float rgb32[3])
{
    const float *R = c->R, *mu = g->means + 3 * i;
    float cp[3];
    for (int k = 0; k < 3; k++) cp[k] = -fmaf(R[6 + k], c->t[2], fmaf(R[3 + k], c->t[1], R[k] * c->t[0]));
    float dx = mu[0] - cp[0], dy = mu[1] - cp[1], dz = mu[2] - cp[2];
    float n2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    float inv = 1.0f / sqrtf(n2);
    float x = dx * inv, y = dy * inv, z = dz * inv;
    float xx = x * x, yy = y * y, zz = z * z;
    float Y[16];
    Y[0] = 0.28209479177387814f;
    Y[1] = -0.4886025119029199f * y;
    Y[2] = 0.4886025119029199f * z;
    Y[3] = -0.4886025119029199f * x;
    Y[4] = (1.0925484305920792f * x) * y;
    Y[5] = (-1.0925484305920792f * y) * z;
    Y[6] = 0.31539156525252005f * ((2.0f * zz - xx) - yy);
    Y[7] = (-1.0925484305920792f * x) * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
    Y[9] = (-0.5900435899266435f * y) * (3.0f * xx - yy);
    Y[10] = ((2.890611442640554f * x) * y) * z;
    Y[11] = (-0.4570457994644658f * y) * ((4.0f * zz - xx) - yy);
    Y[12] = (0.3731763325901154f * z) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);
    Y[13] = (-0.4570457994644658f * x) * ((4.0f * zz - xx) - yy);
    Y[14] = (1.445305721320277f * z) * (xx - yy);
    Y[15] = (-0.5900435899266435f * x) * (xx - 3.0f * yy);
    int nk = (g->sh_degree + 1) * (g->sh_degree + 1);
    const float *sh = g->sh + (size_t)i * g->sh_stride * 3;
    for (int ch = 0; ch < 3; ch++) {
        float acc = 0.5f;
        for (int k = 0; k < nk; k++) acc = fmaf(Y[k], sh[3 * k + ch], acc);
        clamped[ch] = acc < 0.0f;
        rgb32[ch] = clamped[ch] ? 0.0f : acc;
    }
}

/* ============================================================= fp64 chain */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Real SH basis Y_k(d) (k < 16) and its gradient dY_k/d(d) — [3DGS] order. */
static void sh_basis(const double d[3], double Y[16], double dY[16][3])
{
    double x = d[0], y = d[1], z = d[2];
    double xx = x * x, yy = y * y, zz = z * z;
    memset(dY, 0, sizeof(double) * 48);
    Y[0] = SH_C0;
    Y[1] = -SH_C1 * y;  dY[1][1] = -SH_C1;
    Y[2] = SH_C1 * z;   dY[2][2] = SH_C1;
    Y[3] = -SH_C1 * x;  dY[3][0] = -SH_C1;
    Y[4] = SH_C2[0] * x * y;            dY[4][0] = SH_C2[0] * y; dY[4][1] = SH_C2[0] * x;
    Y[5] = SH_C2[1] * y * z;            dY[5][1] = SH_C2[1] * z; dY[5][2] = SH_C2[1] * y;
    Y[6] = SH_C2[2] * (2 * zz - xx - yy);
    dY[6][0] = -2 * SH_C2[2] * x; dY[6][1] = -2 * SH_C2[2] * y; dY[6][2] = 4 * SH_C2[2] * z;
    Y[7] = SH_C2[3] * x * z;            dY[7][0] = SH_C2[3] * z; dY[7][2] = SH_C2[3] * x;
    Y[8] = SH_C2[4] * (xx - yy);        dY[8][0] = 2 * SH_C2[4] * x; dY[8][1] = -2 * SH_C2[4] * y;
    Y[9] = SH_C3[0] * y * (3 * xx - yy);
    dY[9][0] = SH_C3[0] * 6 * x * y; dY[9][1] = SH_C3[0] * (3 * xx - 3 * yy);
    Y[10] = SH_C3[1] * x * y * z;
    dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
    Y[11] = SH_C3[2] * y * (4 * zz - xx - yy);
    dY[11][0] = SH_C3[2] * (-2 * x * y); dY[11][1] = SH_C3[2] * (4 * zz - xx - 3 * yy);
    dY[11][2] = SH_C3[2] * 8 * y * z;
    Y[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
    dY[12][0] = SH_C3[3] * (-6 * x * z); dY[12][1] = SH_C3[3] * (-6 * y * z);
    dY[12][2] = SH_C3[3] * (6 * zz - 3 * xx - 3 * yy);
    Y[13] = SH_C3[4] * x * (4 * zz - xx - yy);
    dY[13][0] = SH_C3[4] * (4 * zz - 3 * xx - yy); dY[13][1] = SH_C3[4] * (-2 * x * y);
    dY[13][2] = SH_C3[4] * 8 * x * z;
    Y[14] = SH_C3[5] * z * (xx - yy);
    dY[14][0] = SH_C3[5] * 2 * x * z; dY[14][1] = SH_C3[5] * (-2 * y * z);
    dY[14][2] = SH_C3[5] * (xx - yy);
    Y[15] = SH_C3[6] * x * (xx - 3 * yy);
    dY[15][0] = SH_C3[6] * (3 * xx - 3 * yy); dY[15][1] = SH_C3[6] * (-6 * x * y);
}

typedef struct { /* per-Gaussian fp64 activations (O1) */
    double mu[3], s[3], qn[4], qnorm, R[3][3], M[3][3], Sig[3][3], o;
} g64_t;

static void activate64(const og_scene *g, int64_t i, g64_t *a)
{
    for (int k = 0; k < 3; k++) {
        a->mu[k] = g->means[3 * i + k];
        a->s[k] = exp((double)g->log_scales[3 * i + k]);
    }
    a->o = 1.0 / (1.0 + exp(-(double)g->opacity_logits[i]));
    double q[4];
    for (int k = 0; k < 4; k++) q[k] = g->quats[4 * i + k];
    a->qnorm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; k++) a->qn[k] = q[k] / a->qnorm;
    double w = a->qn[0], x = a->qn[1], y = a->qn[2], z = a->qn[3];
    double (*R)[3] = a->R;
    R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) a->M[r][c] = R[r][c] * a->s[c];
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += a->M[r][k] * a->M[c][k];
            a->Sig[r][c] = acc;
        }
}

typedef struct { /* per (Gaussian, view) fp64 projection state (O2) */
    double t[3], ux, uy, px, py, J[2][3], T[2][3], a, b, c, det, A, B, C;
    int clx, cly;          /* Jacobian clamp active (R4)          */
    double dir[3], dnorm;  /* normalised μ − camera centre and ‖μ − c‖      */
    double rgb[3];
    int rgb_clamped[3];
    float rgb32[3];        /* the colour in fp32 CA (the clamp decision's value)  */
} p64_t;

static void project64(const og_scene *g, int64_t i, const g64_t *a, const og_cam *cam, p64_t *p)
{
    double Rv[3][3], tv[3];
    for (int r = 0; r < 3; r++) {
        tv[r] = cam->t[r];
        for (int c = 0; c < 3; c++) Rv[r][c] = cam->R[3 * r + c];
    }
    for (int r = 0; r < 3; r++) p->t[r] = Rv[r][0] * a->mu[0] + Rv[r][1] * a->mu[1] + Rv[r][2] * a->mu[2] + tv[r];
    double fx = cam->fx, fy = cam->fy, tz = p->t[2];
    p->ux = p->t[0] / tz;
    p->uy = p->t[1] / tz;
    p->px = fx * p->ux + cam->cx;
    p->py = fy * p->uy + cam->cy;
    double limx = 0.65 * cam->width / fx, limy = 0.65 * cam->height / fy;
    double uxc = p->ux, uyc = p->uy;
    p->clx = p->cly = 0;
    if (uxc > limx) { uxc = limx; p->clx = 1; }
    if (uxc < -limx) { uxc = -limx; p->clx = 1; }
    if (uyc > limy) { uyc = limy; p->cly = 1; }
    if (uyc < -limy) { uyc = -limy; p->cly = 1; }
    memset(p->J, 0, sizeof p->J);
    p->J[0][0] = fx / tz; p->J[0][2] = -fx * uxc / tz;
    p->J[1][1] = fy / tz; p->J[1][2] = -fy * uyc / tz;
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < 3; c++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += p->J[r][k] * Rv[k][c];
            p->T[r][c] = acc;
        }
    double S2[2][2];
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < 2; c++) {
            double acc = 0;
            for (int k = 0; k < 3; k++)
                for (int l = 0; l < 3; l++) acc += p->T[r][k] * a->Sig[k][l] * p->T[c][l];
            S2[r][c] = acc;
        }
    p->a = S2[0][0] + 0.3; p->b = S2[0][1]; p->c = S2[1][1] + 0.3;
    p->det = p->a * p->c - p->b * p->b;
    p->A = p->c / p->det; p->B = -p->b / p->det; p->C = p->a / p->det;
    /* colour: dir from the camera centre c_v = −R_vᵀ t_v */
    double cpos[3];
    for (int k = 0; k < 3; k++) cpos[k] = -(Rv[0][k] * tv[0] + Rv[1][k] * tv[1] + Rv[2][k] * tv[2]);
    double d[3] = {a->mu[0] - cpos[0], a->mu[1] - cpos[1], a->mu[2] - cpos[2]};
    p->dnorm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int k = 0; k < 3; k++) p->dir[k] = d[k] / p->dnorm;
    double Y[16], dY[16][3];
    sh_basis(p->dir, Y, dY);
    int nk = (g->sh_degree + 1) * (g->sh_degree + 1);
    const float *sh = g->sh + (size_t)i * g->sh_stride * 3;
    color32(g, i, cam, p->rgb_clamped, p->rgb32); /* the clamp is a decision: fp32 CA (R17) */
    for (int ch = 0; ch < 3; ch++) {
        double v = 0.5;
        for (int k = 0; k < nk; k++) v += Y[k] * sh[3 * k + ch];
        p->rgb[ch] = p->rgb_clamped[ch] ? 0.0 : v;
    }
}

/* =========================================================== O8 helpers
 * The ADC statistics of P:14–21, kept per (Gaussian, view) pair:
 *   gsum = Σ_{pixels of this view} ∇_{p_i}L   (2-vector, NDC)
 *   e1   = Σ_{pixels of this view} ‖∇_{p_i}L‖₂
 * and reduced per Gaussian over its views by adc_finalize.                 */
typedef struct { double gx, gy, e1; } adc_pair;

static void adc_add_pixel(adc_pair *a, double gx, double gy)
{
    a->gx += gx;
    a->gy += gy;
    a->e1 += sqrt(gx * gx + gy * gy);
}

/* E_old = ‖Σ_k gsum_k‖, E1 = Σ_k e1_k, E2 = Σ_k ‖gsum_k‖ */
static void adc_finalize(const adc_pair *pairs, const int *present, int V, double out[3])
{
    double sx = 0, sy = 0, e1 = 0, e2 = 0;
    for (int v = 0; v < V; v++) {
        if (!present[v]) continue;
        sx += pairs[v].gx;
        sy += pairs[v].gy;
        e1 += pairs[v].e1;
        e2 += sqrt(pairs[v].gx * pairs[v].gx + pairs[v].gy * pairs[v].gy);
    }
    out[0] = sqrt(sx * sx + sy * sy);
    out[1] = e1;
    out[2] = e2;
}

/* P11 test entry: per-pixel NDC gradients of one Gaussian with view labels
 * (0 ≤ view < 64) → (E_old, E1, E2) through the same two functions.       */
void oracle_adc_example(int n, const int *view, const double *gx, const double *gy, double out[3])
{
    adc_pair pr[64];
    int present[64];
    memset(pr, 0, sizeof pr);
    memset(present, 0, sizeof present);
    for (int k = 0; k < n; k++) {
        adc_add_pixel(&pr[view[k]], gx[k], gy[k]);
        present[view[k]] = 1;
    }
    adc_finalize(pr, present, 64, out);
}

/* ================================================================= handle */
enum { NG = 10 }; /* per-pair gradient record: gx gy e1 dA dB dC dO dr dg db */

typedef struct {
    og_scene g;
    const og_cam *cams;
    int V, flags;
    double bg[3];
    float bg32[3];
    int W, H, TX, TY, T;
    /* per (view, gid) */
    p32_t *p32;            /* [V*P]                                          */
    float *o32;            /* [P] fp32 opacity for the decision chain        */
    g64_t *g64;            /* [P]                                            */
    int32_t *p64i;         /* [V*P] index into p64 for visible pairs, else -1 */
    p64_t *p64;            /* [number of visible pairs]                      */
    /* lists */
    int64_t *off;          /* [V*T+1]                                        */
    int32_t *gid;          /* [K]                                            */
    int64_t K;
    /* forward */
    double *img, *Tfin;    /* [V,3,H,W], [V,H,W]                             */
    float *img32, *Tfin32; /* the same in fp32 canonical arithmetic */
    double *imgx;          /* experiment: fp64 value chain driven by the fp32 alphas */
    double *dep;           /* [V,H,W] alpha-weighted expected depth (NEXT-2)  */
    int32_t *ncon;         /* [V,H,W]                                        */
    int32_t *nbl;          /* [V,H,W] number of blended entries per pixel    */
    /* backward */
    double *pg;            /* [V*P*NG]                                       */
    int have_bwd;
    uint8_t *mask;         /* [V*T] tiles to render (NULL = all) — sampled full-size checks */
    uint64_t dhash;        /* hash of every discrete decision (FD tests)     */
    int64_t npg;           /* number of pairs with fp64 state (= rows of pg)  */
    double t_phase[4];     /* seconds: O1–O2 projection, O3–O4 lists, O5–O6 per pixel, O7–O8 per Gaussian */
    double *d_means, *d_ls, *d_q, *d_op, *d_sh, *e1, *e2, *eold, *vis;
} oracle_t;

typedef struct { uint32_t depth_bits; int32_t gid; } entry_t;

static int entry_cmp(const void *x, const void *y)
{
    const entry_t *a = (const entry_t *)x, *b = (const entry_t *)y;
    if (a->depth_bits != b->depth_bits) return a->depth_bits < b->depth_bits ? -1 : 1;
    return (a->gid > b->gid) - (a->gid < b->gid);
}

/* Host threads for the timing baseline (oracle-mt): 1 (the default, every
 * test) runs every loop in its written order.  With n > 1 the independent loops — per
 * Gaussian (O1, O2, O7, O8), per (view, tile) list (O4) and per (view, tile) bucket of pixels
 * (O5, O6) — are split over OpenMP threads; the per-pair gradient sums of O6 go to one
 * accumulator per thread, added in thread order afterwards (the only change of arithmetic:
 * the order of those fp64 sums). */
static int g_threads = 1;
void oracle_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int oracle_get_threads(void) { return g_threads; }

static uint32_t fbits(float f)
{
    union { float f; uint32_t u; } u;
    u.f = f;
    return u.u;
}

void oracle_destroy(oracle_t *h)
{
    if (!h) return;
    free(h->p32); free(h->o32); free(h->g64); free(h->p64); free(h->p64i); free(h->off); free(h->gid);
    free(h->mask);
    free(h->img); free(h->Tfin); free(h->ncon); free(h->nbl); free(h->pg); free(h->dep);
    free(h->img32); free(h->Tfin32); free(h->imgx);
    free(h->d_means); free(h->d_ls); free(h->d_q); free(h->d_op); free(h->d_sh);
    free(h->e1); free(h->e2); free(h->eold); free(h->vis);
    free(h);
}

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static int rect_hits_mask(const oracle_t *h, int v, const p32_t *p)
{
    if (!h->mask) return 1;
    for (int ty = p->ry0; ty < p->ry1; ty++)
        for (int tx = p->rx0; tx < p->rx1; tx++)
            if (h->mask[(int64_t)v * h->T + ty * h->TX + tx]) return 1;
    return 0;
}

oracle_t *oracle_create_masked(const og_scene *g, const og_cam *cams, int V, const float bg[3], int flags,
                               const uint8_t *tile_mask);

/* O1–O4: activations, projection, lists.  Returns NULL on invalid input. */
oracle_t *oracle_create(const og_scene *g, const og_cam *cams, int V, const float bg[3], int flags)
{
    return oracle_create_masked(g, cams, V, bg, flags, NULL);
}

/* Same, restricted to the (view, tile) buckets with tile_mask[v*T + t] != 0: only
 * those lists are built and only their pixels are composited (sampled checks at
 * full size).  Participation, projection and vis are computed for every pair. */
oracle_t *oracle_create_masked(const og_scene *g, const og_cam *cams, int V, const float bg[3], int flags,
                               const uint8_t *tile_mask)
{
    if (!g || !cams || V < 1 || g->sh_degree < 0 || g->sh_degree > 3) return NULL;
    for (int v = 1; v < V; v++)
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height) return NULL;
    oracle_t *h = (oracle_t *)calloc(1, sizeof *h);
    h->g = *g;
    h->cams = cams;
    h->V = V;
    h->flags = flags;
    for (int k = 0; k < 3; k++) h->bg[k] = bg ? bg[k] : 0.0;
    for (int k = 0; k < 3; k++) h->bg32[k] = bg ? bg[k] : 0.0f;
    h->W = cams[0].width;
    h->H = cams[0].height;
    h->TX = (h->W + 15) / 16;
    h->TY = (h->H + 15) / 16;
    h->T = h->TX * h->TY;
    if (tile_mask) {
        h->mask = (uint8_t *)malloc((size_t)V * h->T);
        memcpy(h->mask, tile_mask, (size_t)V * h->T);
    }
    int64_t P = g->P;
    double t0 = now_s();
    h->p32 = (p32_t *)calloc((size_t)V * P + 1, sizeof(p32_t));
    h->p64i = (int32_t *)malloc(sizeof(int32_t) * ((size_t)V * P + 1));
    h->o32 = (float *)calloc(P + 1, sizeof(float));
    h->g64 = (g64_t *)calloc(P + 1, sizeof(g64_t));
    /* O1 + O2 (fp32 decisions) */
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads)
    for (int64_t i = 0; i < P; i++) {
        float Sig[6];
        activate32(g, i, &h->o32[i], Sig);
        activate64(g, i, &h->g64[i]);
        const float *mu = g->means + 3 * i;
        for (int v = 0; v < V; v++) {
            p32_t *p = &h->p32[(size_t)v * P + i];
            project32(mu, Sig, &cams[v], p);
            h->p64i[(size_t)v * P + i] = (p->vis && rect_hits_mask(h, v, p)) ? 0 : -1;
        }
    }
    /* fp64 slots of the visible pairs, numbered in (Gaussian, view) order */
    int64_t nvis = 0;
    for (int64_t i = 0; i < P; i++)
        for (int v = 0; v < V; v++)
            if (h->p64i[(size_t)v * P + i] >= 0) h->p64i[(size_t)v * P + i] = (int32_t)nvis++;
    /* O2 fp64 values for the visible pairs */
    h->p64 = (p64_t *)calloc((size_t)nvis + 1, sizeof(p64_t));
    h->npg = nvis;
#pragma omp parallel for schedule(dynamic, 4096) num_threads(g_threads)
    for (int64_t i = 0; i < P; i++)
        for (int v = 0; v < V; v++) {
            int32_t k = h->p64i[(size_t)v * P + i];
            if (k >= 0) project64(g, i, &h->g64[i], &cams[v], &h->p64[k]);
        }
    double t1 = now_s();
    h->t_phase[0] = t1 - t0;
    /* O3: count, offsets, fill; O4: sort each list */
    int64_t nb = (int64_t)V * h->T;
    h->off = (int64_t *)calloc(nb + 1, sizeof(int64_t));
    for (int v = 0; v < V; v++)
        for (int64_t i = 0; i < P; i++) {
            const p32_t *p = &h->p32[(size_t)v * P + i];
            if (!p->vis) continue;
            for (int ty = p->ry0; ty < p->ry1; ty++)
                for (int tx = p->rx0; tx < p->rx1; tx++) {
                    int64_t b = (int64_t)v * h->T + ty * h->TX + tx;
                    if (!h->mask || h->mask[b]) h->off[b + 1]++;
                }
        }
    for (int64_t b = 0; b < nb; b++) h->off[b + 1] += h->off[b];
    h->K = h->off[nb];
    entry_t *ent = (entry_t *)malloc(sizeof(entry_t) * (h->K + 1));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (nb + 1));
    memcpy(fill, h->off, sizeof(int64_t) * nb);
    for (int v = 0; v < V; v++)
        for (int64_t i = 0; i < P; i++) {
            const p32_t *p = &h->p32[(size_t)v * P + i];
            if (!p->vis) continue;
            for (int ty = p->ry0; ty < p->ry1; ty++)
                for (int tx = p->rx0; tx < p->rx1; tx++) {
                    int64_t b = (int64_t)v * h->T + ty * h->TX + tx;
                    if (h->mask && !h->mask[b]) continue;
                    ent[fill[b]].depth_bits = fbits(p->tz);
                    ent[fill[b]].gid = (int32_t)i;
                    fill[b]++;
                }
        }
#pragma omp parallel for schedule(dynamic, 64) num_threads(g_threads)
    for (int64_t b = 0; b < nb; b++)
        qsort(ent + h->off[b], (size_t)(h->off[b + 1] - h->off[b]), sizeof(entry_t), entry_cmp);
    h->gid = (int32_t *)malloc(sizeof(int32_t) * (h->K + 1));
    for (int64_t k = 0; k < h->K; k++) h->gid[k] = ent[k].gid;
    free(ent);
    free(fill);
    h->t_phase[1] = now_s() - t1;
    return h;
}

typedef struct { /* one blended entry of one pixel, recorded by the forward */
    int32_t gid;
    int clamped;
    double alpha, T, G, dx, dy;
} blend_t;

/* O5 (+ O6 when dLdC != NULL) for every pixel of every view. */
static uint64_t mix(uint64_t hsh, uint64_t v)
{
    hsh ^= v + 0x9e3779b97f4a7c15ULL + (hsh << 6) + (hsh >> 2);
    return hsh * 0xff51afd7ed558ccdULL;
}

static void composite(oracle_t *h, const float *dLdC)
{
    h->dhash = 0;
    const int64_t P = h->g.P;
    const int W = h->W, H = h->H, V = h->V;
    const int64_t nb = (int64_t)V * h->T;
    int64_t maxlen = 0;
    for (int64_t b = 0; b < nb; b++)
        if (h->off[b + 1] - h->off[b] > maxlen) maxlen = h->off[b + 1] - h->off[b];
    uint64_t *bh = (uint64_t *)calloc((size_t)nb + 1, sizeof(uint64_t)); /* per-bucket decision hash */
    const int nt = g_threads;
    double **pgt = (double **)calloc((size_t)nt, sizeof(double *)); /* per-thread pair sums (thread 0: h->pg) */
    if (dLdC)
        for (int t = 0; t < nt; t++)
            pgt[t] = t == 0 ? h->pg : (double *)calloc((size_t)h->npg * NG + 1, sizeof(double));
#pragma omp parallel num_threads(nt)
    {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double *pgbase = dLdC ? pgt[tid] : NULL;
    blend_t *bl = (blend_t *)malloc(sizeof(blend_t) * (maxlen + 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; b++) {
        if (h->mask && !h->mask[b]) continue;
        const int v = (int)(b / h->T), tile = (int)(b % h->T);
        const int ty0 = (tile / h->TX) * 16, tx0 = (tile % h->TX) * 16;
        uint64_t hsh = 0;
        for (int y = ty0; y < ty0 + 16 && y < H; y++)
            for (int x = tx0; x < tx0 + 16 && x < W; x++) {
                /* ---- O5: forward.  Decisions fp32 (CA), values fp64. */
                float T32 = 1.0f, C32[3] = {0.0f, 0.0f, 0.0f};
                double T64 = 1.0, Cc[3] = {0, 0, 0}, Dd = 0.0;
                double Tx = 1.0, Cx[3] = {0, 0, 0};
                int last = 0, m = 0;
                const float fxp = (float)x, fyp = (float)y;
                for (int64_t j = h->off[b]; j < h->off[b + 1]; j++) {
                    int32_t i = h->gid[j];
                    const p32_t *p = &h->p32[(size_t)v * P + i];
                    float dx = p->px - fxp, dy = p->py - fyp;
                    float power = fmaf(-0.5f, fmaf(p->A * dx, dx, (p->C * dy) * dy), -((p->B * dx) * dy));
                    if (power > 0.0f) continue;
                    float G32 = oracle_ca_exp(power);
                    float oG = h->o32[i] * G32;
                    float alpha = fminf(0.99f, oG);
                    if (alpha < 1.0f / 255.0f) continue;
                    float Tn = T32 * (1.0f - alpha);
                    if (Tn < 1e-4f && !(h->flags & OG_NO_EARLY_TERMINATION)) break;
                    /* blended: value chain in fp64 */
                    const p64_t *q = &h->p64[h->p64i[(size_t)v * P + i]];
                    double ddx = q->px - x, ddy = q->py - y;
                    double pw = -0.5 * (q->A * ddx * ddx + q->C * ddy * ddy) - q->B * ddx * ddy;
                    double G = exp(pw);
                    int clamped = oG > 0.99f;
                    double a64 = clamped ? 0.99 : h->g64[i].o * G;
                    for (int ch = 0; ch < 3; ch++) Cc[ch] += q->rgb[ch] * a64 * T64;
                    Dd += q->t[2] * a64 * T64; /* predicted depth Σ dᵢαᵢTᵢ */
                    hsh = mix(hsh, ((uint64_t)j << 20) ^ ((uint64_t)(y * W + x) << 1) ^ (uint64_t)clamped);
                    hsh = mix(hsh, (uint64_t)(q->clx | q->cly << 1 | q->rgb_clamped[0] << 2
                                              | q->rgb_clamped[1] << 3 | q->rgb_clamped[2] << 4));
                    bl[m].gid = i;
                    bl[m].clamped = clamped;
                    bl[m].alpha = a64;
                    bl[m].T = T64;
                    bl[m].G = G;
                    bl[m].dx = ddx;
                    bl[m].dy = ddy;
                    m++;
                    T64 *= (1.0 - a64);
                    {   /* the same blend in fp32 CA: C = fma(rgb, α·T, C) */
                        const float w = alpha * T32;
                        for (int ch = 0; ch < 3; ch++) C32[ch] = fmaf(q->rgb32[ch], w, C32[ch]);
                    }
                    for (int ch = 0; ch < 3; ch++) Cx[ch] += (double)q->rgb32[ch] * (double)alpha * Tx;
                    Tx *= 1.0 - (double)alpha;
                    T32 = Tn;
                    last = (int)(j - h->off[b]) + 1;
                }
                size_t pix = (size_t)y * W + x;
                for (int ch = 0; ch < 3; ch++)
                    h->img[((size_t)v * 3 + ch) * H * W + pix] = Cc[ch] + T64 * h->bg[ch];
                h->Tfin[(size_t)v * H * W + pix] = T64;
                for (int ch = 0; ch < 3; ch++) {
                    h->img32[((size_t)v * 3 + ch) * H * W + pix] = fmaf(T32, h->bg32[ch], C32[ch]);
                    h->imgx[((size_t)v * 3 + ch) * H * W + pix] = Cx[ch] + Tx * h->bg[ch];
                }
                h->Tfin32[(size_t)v * H * W + pix] = T32;
                h->dep[(size_t)v * H * W + pix] = Dd;
                h->ncon[(size_t)v * H * W + pix] = last;
                h->nbl[(size_t)v * H * W + pix] = m;
                if (!dLdC) continue;
                /* ---- O6: adjoint of Eq. (1) for this pixel, from its definition:
                 * C = Σ_k c_k α_k T_k + T_fin·bg, T_k = Π_{j<k}(1−α_j).
                 * ∂C/∂c_k = α_k T_k ;  ∂C/∂α_k = c_k T_k − (S_k + T_fin·bg)/(1−α_k)
                 * with S_k = Σ_{j>k} c_j α_j T_j (every later term carries (1−α_k)). */
                double dL[3];
                for (int ch = 0; ch < 3; ch++) dL[ch] = dLdC[((size_t)v * 3 + ch) * H * W + pix];
                double S[3] = {0, 0, 0};
                for (int k = m - 1; k >= 0; k--) {
                    int32_t i = bl[k].gid;
                    const p64_t *q = &h->p64[h->p64i[(size_t)v * P + i]];
                    double *pg = &pgbase[(size_t)h->p64i[(size_t)v * P + i] * NG];
                    double aT = bl[k].alpha * bl[k].T;
                    double dLda = 0;
                    for (int ch = 0; ch < 3; ch++) {
                        pg[7 + ch] += aT * dL[ch];
                        double dCda = q->rgb[ch] * bl[k].T - (S[ch] + T64 * h->bg[ch]) / (1.0 - bl[k].alpha);
                        dLda += dL[ch] * dCda;
                    }
                    for (int ch = 0; ch < 3; ch++) S[ch] += q->rgb[ch] * aT;
                    double dLdG = 0, dLdo = 0;
                    if (!bl[k].clamped) {
                        dLdG = h->g64[i].o * dLda;
                        dLdo = bl[k].G * dLda;
                    }
                    double dLdpw = bl[k].G * dLdG; /* G = exp(power) */
                    double dx = bl[k].dx, dy = bl[k].dy;
                    /* power = −½(A dx² + C dy²) − B dx dy, d = μ' − p */
                    double dLdpx = dLdpw * (-(q->A * dx + q->B * dy));
                    double dLdpy = dLdpw * (-(q->C * dy + q->B * dx));
                    /* ∇_{p_i}L in NDC: pixel = ((ndc+1)·W − 1)/2 ⇒ ∂pixel/∂ndc = W/2 (R2) */
                    adc_pair ap = {pg[0], pg[1], pg[2]};
                    adc_add_pixel(&ap, dLdpx * 0.5 * W, dLdpy * 0.5 * H);
                    pg[0] = ap.gx; pg[1] = ap.gy; pg[2] = ap.e1;
                    pg[3] += dLdpw * (-0.5 * dx * dx);
                    pg[4] += dLdpw * (-dx * dy);
                    pg[5] += dLdpw * (-0.5 * dy * dy);
                    pg[6] += dLdo;
                }
            }
        bh[b] = hsh;
    }
    free(bl);
    }
    for (int64_t b = 0; b < nb; b++) h->dhash = mix(h->dhash, bh[b]);
    if (dLdC)
        for (int t = 1; t < nt; t++) { /* thread order */
            for (size_t k = 0; k < (size_t)h->npg * NG; k++) h->pg[k] += pgt[t][k];
            free(pgt[t]);
        }
    free(pgt);
    free(bh);
}

/* O7 + O8: per-Gaussian chain rule summed over views, and the E statistics. */
static void gauss_backward(oracle_t *h)
{
    const int64_t P = h->g.P;
    const int V = h->V;
    const int S = h->g.sh_stride;
    const int nk = (h->g.sh_degree + 1) * (h->g.sh_degree + 1);
#pragma omp parallel num_threads(g_threads)
    {
    adc_pair *ap = (adc_pair *)malloc(sizeof(adc_pair) * V);
    int *present = (int *)malloc(sizeof(int) * V);
#pragma omp for schedule(dynamic, 4096)
    for (int64_t i = 0; i < P; i++) {
        const g64_t *a = &h->g64[i];
        const float *sh = h->g.sh + (size_t)i * S * 3;
        double dmu[3] = {0, 0, 0}, dSig[3][3] = {{0}}, dop = 0;
        double *dsh = &h->d_sh[(size_t)i * S * 3];
        double visc = 0;
        for (int v = 0; v < V; v++) {
            const p32_t *p = &h->p32[(size_t)v * P + i];
            present[v] = p->vis;
            ap[v].gx = ap[v].gy = ap[v].e1 = 0;
            if (!p->vis) continue;
            visc += 1;
            if (h->p64i[(size_t)v * P + i] < 0) { present[v] = 0; continue; } /* outside the mask: no pixel */
            const p64_t *q = &h->p64[h->p64i[(size_t)v * P + i]];
            const double *pg = &h->pg[(size_t)h->p64i[(size_t)v * P + i] * NG];
            const og_cam *cam = &h->cams[v];
            ap[v].gx = pg[0]; ap[v].gy = pg[1]; ap[v].e1 = pg[2];
            double Rv[3][3];
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) Rv[r][c] = cam->R[3 * r + c];
            double fx = cam->fx, fy = cam->fy;
            double tx = q->t[0], ty = q->t[1], tz = q->t[2];
            double dt[3] = {0, 0, 0};
            /* μ' = (fx·tx/tz + cx, fy·ty/tz + cy); ∂L/∂μ'_pix = g_ndc·(2/W, 2/H) */
            double dpx = pg[0] * 2.0 / h->W, dpy = pg[1] * 2.0 / h->H;
            dt[0] += fx / tz * dpx;
            dt[1] += fy / tz * dpy;
            dt[2] += -fx * tx / (tz * tz) * dpx - fy * ty / (tz * tz) * dpy;
            /* conic (A,B,C) = (c, −b, a)/det, det = ac − b² */
            double dA = pg[3], dB = pg[4], dC = pg[5];
            double D2 = q->det * q->det, qa = q->a, qb = q->b, qc = q->c;
            double da = (-qc * qc * dA + qb * qc * dB - qb * qb * dC) / D2;
            double dc = (-qb * qb * dA + qa * qb * dB - qa * qa * dC) / D2;
            double db = (2 * qb * qc * dA - (q->det + 2 * qb * qb) * dB + 2 * qa * qb * dC) / D2;
            /* Σ' = T Σ Tᵀ + 0.3 I, Gs = [[da, db/2],[db/2, dc]] */
            double Gs[2][2] = {{da, 0.5 * db}, {0.5 * db, dc}};
            /* ∂L/∂Σ += Tᵀ Gs T */
            for (int r = 0; r < 3; r++)
                for (int c = 0; c < 3; c++) {
                    double acc = 0;
                    for (int k = 0; k < 2; k++)
                        for (int l = 0; l < 2; l++) acc += q->T[k][r] * Gs[k][l] * q->T[l][c];
                    dSig[r][c] += acc;
                }
            /* ∂L/∂T = 2 Gs T Σ ;  T = J R_v ⇒ ∂L/∂J = ∂L/∂T R_vᵀ */
            double dT[2][3], dJ[2][3];
            for (int r = 0; r < 2; r++)
                for (int c = 0; c < 3; c++) {
                    double acc = 0;
                    for (int k = 0; k < 2; k++)
                        for (int l = 0; l < 3; l++) acc += Gs[r][k] * q->T[k][l] * a->Sig[l][c];
                    dT[r][c] = 2 * acc;
                }
            for (int r = 0; r < 2; r++)
                for (int c = 0; c < 3; c++) {
                    double acc = 0;
                    for (int k = 0; k < 3; k++) acc += dT[r][k] * Rv[c][k];
                    dJ[r][c] = acc;
                }
            /* J = [[fx/tz, 0, −fx·ũx/tz], [0, fy/tz, −fy·ũy/tz]], ũ = clamp(t_xy/tz) */
            double tz2 = tz * tz;
            dt[2] += -fx / tz2 * dJ[0][0] - fy / tz2 * dJ[1][1];
            if (!q->clx) {
                dt[0] += -fx / tz2 * dJ[0][2];
                dt[2] += 2 * fx * tx / (tz2 * tz) * dJ[0][2];
            } else {
                double uxc = -q->J[0][2] * tz / fx;
                dt[2] += fx * uxc / tz2 * dJ[0][2];
            }
            if (!q->cly) {
                dt[1] += -fy / tz2 * dJ[1][2];
                dt[2] += 2 * fy * ty / (tz2 * tz) * dJ[1][2];
            } else {
                double uyc = -q->J[1][2] * tz / fy;
                dt[2] += fy * uyc / tz2 * dJ[1][2];
            }
            /* t = R_v μ + t_v */
            for (int k = 0; k < 3; k++) dmu[k] += Rv[0][k] * dt[0] + Rv[1][k] * dt[1] + Rv[2][k] * dt[2];
            /* colour: rgb = max(0, Σ_k Y_k(dir)·sh_k + 0.5), dir = (μ − c_v)/‖μ − c_v‖ */
            double draw[3], ddir[3] = {0, 0, 0}, Y[16], dY[16][3];
            sh_basis(q->dir, Y, dY);
            for (int ch = 0; ch < 3; ch++) draw[ch] = q->rgb_clamped[ch] ? 0.0 : pg[7 + ch];
            for (int k = 0; k < nk; k++)
                for (int ch = 0; ch < 3; ch++) {
                    dsh[3 * k + ch] += Y[k] * draw[ch];
                    double w = sh[3 * k + ch] * draw[ch];
                    for (int e = 0; e < 3; e++) ddir[e] += dY[k][e] * w;
                }
            double dd = q->dir[0] * ddir[0] + q->dir[1] * ddir[1] + q->dir[2] * ddir[2];
            for (int e = 0; e < 3; e++) dmu[e] += (ddir[e] - q->dir[e] * dd) / q->dnorm;
            dop += pg[6];
        }
        /* Σ = M Mᵀ, M = R diag(s) ⇒ ∂L/∂M = (∂Σ + ∂Σᵀ) M */
        double dM[3][3];
        for (int r = 0; r < 3; r++)
            for (int c = 0; c < 3; c++) {
                double acc = 0;
                for (int k = 0; k < 3; k++) acc += (dSig[r][k] + dSig[k][r]) * a->M[k][c];
                dM[r][c] = acc;
            }
        double ds[3], dR[3][3];
        for (int c = 0; c < 3; c++) {
            ds[c] = 0;
            for (int r = 0; r < 3; r++) {
                ds[c] += dM[r][c] * a->R[r][c];
                dR[r][c] = dM[r][c] * a->s[c];
            }
        }
        for (int c = 0; c < 3; c++) h->d_ls[3 * i + c] = ds[c] * a->s[c]; /* s = e^λ */
        /* R(q̂): ∂R/∂(w,x,y,z) from the quaternion formula */
        double w = a->qn[0], x = a->qn[1], y = a->qn[2], z = a->qn[3];
        double dq[4];
        dq[0] = -2 * z * dR[0][1] + 2 * y * dR[0][2] + 2 * z * dR[1][0] - 2 * x * dR[1][2]
                - 2 * y * dR[2][0] + 2 * x * dR[2][1];
        dq[1] = 2 * y * dR[0][1] + 2 * z * dR[0][2] + 2 * y * dR[1][0] - 4 * x * dR[1][1]
                - 2 * w * dR[1][2] + 2 * z * dR[2][0] + 2 * w * dR[2][1] - 4 * x * dR[2][2];
        dq[2] = -4 * y * dR[0][0] + 2 * x * dR[0][1] + 2 * w * dR[0][2] + 2 * x * dR[1][0]
                + 2 * z * dR[1][2] - 2 * w * dR[2][0] + 2 * z * dR[2][1] - 4 * y * dR[2][2];
        dq[3] = -4 * z * dR[0][0] - 2 * w * dR[0][1] + 2 * x * dR[0][2] + 2 * w * dR[1][0]
                - 4 * z * dR[1][1] + 2 * y * dR[1][2] + 2 * x * dR[2][0] + 2 * y * dR[2][1];
        /* q̂ = q/‖q‖ ⇒ ∂L/∂q = (∂q̂ − q̂(q̂·∂q̂))/‖q‖ */
        double qd = w * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
        for (int k = 0; k < 4; k++) h->d_q[4 * i + k] = (dq[k] - a->qn[k] * qd) / a->qnorm;
        for (int k = 0; k < 3; k++) h->d_means[3 * i + k] = dmu[k];
        h->d_op[i] = dop * a->o * (1 - a->o); /* o = σ(ℓ) */
        double E[3];
        adc_finalize(ap, present, V, E);
        h->eold[i] = E[0];
        h->e1[i] = E[1];
        h->e2[i] = E[2];
        h->vis[i] = visc;
    }
    free(ap);
    free(present);
    }
}

int oracle_forward(oracle_t *h)
{
    size_t npx = (size_t)h->V * h->W * h->H;
    free(h->img); free(h->Tfin); free(h->ncon); free(h->nbl);
    h->img = (double *)calloc(3 * npx, sizeof(double));
    h->Tfin = (double *)calloc(npx, sizeof(double));
    free(h->img32); free(h->Tfin32); free(h->imgx);
    h->img32 = (float *)calloc(3 * npx, sizeof(float));
    h->Tfin32 = (float *)calloc(npx, sizeof(float));
    h->imgx = (double *)calloc(3 * npx, sizeof(double));
    h->ncon = (int32_t *)calloc(npx, sizeof(int32_t));
    h->nbl = (int32_t *)calloc(npx, sizeof(int32_t));
    free(h->dep);
    h->dep = (double *)calloc(npx, sizeof(double));
    composite(h, NULL);
    return 0;
}

/* O5 + O6 + O7 + O8 with a given ∂L/∂C [V,3,H,W]. */
int oracle_backward(oracle_t *h, const float *dLdC)
{
    const int64_t P = h->g.P;
    size_t npx = (size_t)h->V * h->W * h->H;
    free(h->img); free(h->Tfin); free(h->ncon); free(h->nbl); free(h->pg);
    h->img = (double *)calloc(3 * npx, sizeof(double));
    h->Tfin = (double *)calloc(npx, sizeof(double));
    free(h->img32); free(h->Tfin32); free(h->imgx);
    h->img32 = (float *)calloc(3 * npx, sizeof(float));
    h->Tfin32 = (float *)calloc(npx, sizeof(float));
    h->imgx = (double *)calloc(3 * npx, sizeof(double));
    h->ncon = (int32_t *)calloc(npx, sizeof(int32_t));
    h->nbl = (int32_t *)calloc(npx, sizeof(int32_t));
    h->pg = (double *)calloc((size_t)h->npg * NG + 1, sizeof(double));
    free(h->dep);
    h->dep = (double *)calloc(npx, sizeof(double));
#define ALLOC(f, n) do { free(h->f); h->f = (double *)calloc((size_t)(n) + 1, sizeof(double)); } while (0)
    ALLOC(d_means, 3 * P); ALLOC(d_ls, 3 * P); ALLOC(d_q, 4 * P); ALLOC(d_op, P);
    ALLOC(d_sh, (size_t)P * h->g.sh_stride * 3);
    ALLOC(e1, P); ALLOC(e2, P); ALLOC(eold, P); ALLOC(vis, P);
#undef ALLOC
    double t0 = now_s();
    composite(h, dLdC);
    double t1 = now_s();
    gauss_backward(h);
    h->t_phase[2] = t1 - t0;
    h->t_phase[3] = now_s() - t1;
    h->have_bwd = 1;
    return 0;
}

/* ---------------------------------------------------------------- getters */
int64_t oracle_num_entries(const oracle_t *h) { return h->K; }

/* Hash of every decision taken by the last forward (blend set, α clamps, Jacobian
 * and colour clamps of blended pairs).  Equal hashes ⇒ the fp64 value chain is one
 * smooth function between two runs (used to screen finite differences). */
uint64_t oracle_decision_hash(const oracle_t *h) { return h->dhash; }

/* Wall-clock seconds of the phases of the last run (timing the CPU baseline). */
void oracle_phase_times(const oracle_t *h, double out[4])
{
    for (int k = 0; k < 4; k++) out[k] = h->t_phase[k];
}

void oracle_get_image(const oracle_t *h, double *rgb, double *Tfin, int32_t *ncon)
{
    size_t npx = (size_t)h->V * h->W * h->H;
    if (rgb) memcpy(rgb, h->img, 3 * npx * sizeof(double));
    if (Tfin) memcpy(Tfin, h->Tfin, npx * sizeof(double));
    if (ncon) memcpy(ncon, h->ncon, npx * sizeof(int32_t));
}

/* the image and T_final of the last forward in fp32 canonical arithmetic: the decisions' T and
 * α, colour accumulated as C = fma(rgb32, α·T, C) in list order, out = fma(T, bg, C) */
void oracle_get_image32(const oracle_t *h, float *rgb, float *Tfin, double *imgx)
{
    size_t npx = (size_t)h->V * h->W * h->H;
    if (rgb) memcpy(rgb, h->img32, 3 * npx * sizeof(float));
    if (Tfin) memcpy(Tfin, h->Tfin32, npx * sizeof(float));
    if (imgx) memcpy(imgx, h->imgx, 3 * npx * sizeof(double));
}

/* blended entries per pixel [V,H,W] of the last forward (α ≥ 1/255, before termination) */
void oracle_get_nblend(const oracle_t *h, int32_t *nbl)
{
    memcpy(nbl, h->nbl, sizeof(int32_t) * (size_t)h->V * h->W * h->H);
}

void oracle_get_depth(const oracle_t *h, double *dep)
{
    memcpy(dep, h->dep, sizeof(double) * (size_t)h->V * h->W * h->H);
}

void oracle_get_lists(const oracle_t *h, int64_t *off, int32_t *gid)
{
    if (off) memcpy(off, h->off, sizeof(int64_t) * ((size_t)h->V * h->T + 1));
    if (gid) memcpy(gid, h->gid, sizeof(int32_t) * h->K);
}

/* per (view, gid) decision-chain state: ints [V*P*9] = zvis vis radius rx0 ry0
 * rx1 ry1 tiles clamp (bits 0-2 SH colour clamp per channel, 3-4 Jacobian clamp
 * x/y; visible pairs only); floats [V*P*6] = depth px py A B C (fp32, bit-exact
 * targets); rgb [V*P*3] fp64. */
void oracle_get_pairs(const oracle_t *h, int32_t *ints, float *flts, double *rgb)
{
    size_t n = (size_t)h->V * h->g.P;
    for (size_t k = 0; k < n; k++) {
        const p32_t *p = &h->p32[k];
        if (ints) {
            int32_t *o = ints + 9 * k;
            o[0] = p->zvis; o[1] = p->vis; o[2] = p->radius; o[3] = p->rx0;
            o[4] = p->ry0; o[5] = p->rx1; o[6] = p->ry1; o[7] = p->tiles; o[8] = 0;
            if (p->vis && h->p64i[k] >= 0) {
                const p64_t *q = &h->p64[h->p64i[k]];
                o[8] = q->rgb_clamped[0] | q->rgb_clamped[1] << 1 | q->rgb_clamped[2] << 2 | q->clx << 3 | q->cly << 4;
            }
        }
        if (flts) {
            float *f = flts + 6 * k;
            f[0] = p->tz; f[1] = p->px; f[2] = p->py; f[3] = p->A; f[4] = p->B; f[5] = p->C;
        }
        if (rgb) {
            for (int c = 0; c < 3; c++) rgb[3 * k + c] = p->vis ? h->p64[h->p64i[k]].rgb[c] : 0.0;
        }
    }
}

void oracle_get_opacity32(const oracle_t *h, float *o)
{
    memcpy(o, h->o32, sizeof(float) * h->g.P);
}

void oracle_get_pair_grads(const oracle_t *h, double *out) /* [V*P*NG], zero where no pair */
{
    size_t n = (size_t)h->V * h->g.P;
    memset(out, 0, sizeof(double) * n * NG);
    if (!h->have_bwd) return;
    for (size_t k = 0; k < n; k++)
        if (h->p64i[k] >= 0) memcpy(out + k * NG, h->pg + (size_t)h->p64i[k] * NG, sizeof(double) * NG);
}

void oracle_get_grads(const oracle_t *h, double *d_means, double *d_ls, double *d_q, double *d_op,
                      double *d_sh, double *e1, double *e2, double *eold, double *vis)
{
    const int64_t P = h->g.P;
    if (!h->have_bwd) return;
    if (d_means) memcpy(d_means, h->d_means, sizeof(double) * 3 * P);
    if (d_ls) memcpy(d_ls, h->d_ls, sizeof(double) * 3 * P);
    if (d_q) memcpy(d_q, h->d_q, sizeof(double) * 4 * P);
    if (d_op) memcpy(d_op, h->d_op, sizeof(double) * P);
    if (d_sh) memcpy(d_sh, h->d_sh, sizeof(double) * (size_t)P * h->g.sh_stride * 3);
    if (e1) memcpy(e1, h->e1, sizeof(double) * P);
    if (e2) memcpy(e2, h->e2, sizeof(double) * P);
    if (eold) memcpy(eold, h->eold, sizeof(double) * P);
    if (vis) memcpy(vis, h->vis, sizeof(double) * P);
}
