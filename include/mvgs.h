/*
 * mvgs.h — C ABI of libmvgs.so: a batched multi-view differentiable tile
 * rasterizer with fused multi-view ADC statistics, hand-written for sm_100a.
 *
 * arXiv 2506.12727 (PAPER.md = P:n):
 *   - rendering Eq. (1) ........................................ P:75–83
 *   - two-stage tile rasterizer, one block per tile ............ P:87–93
 *   - multi-view modifications: participation before
 *     preprocessing, (tile, view, depth) keys, one block per
 *     (tile, view) ............................................. P:571–579
 *   - E_old, E1, E2 ............................................ P:14–21
 * Every reading of a point the paper leaves open is listed in DESIGN.md §3
 * (R1–R49); the fp32 arithmetic of every discrete decision is DESIGN.md §4.
 *
 * Conventions shared by every call
 *   - All array arguments are caller-owned, contiguous, device pointers
 *     (e.g. torch tensors) unless marked "host".  The library never frees
 *     caller memory.  Context-internal buffers live until mvgs_destroy.
 *   - `stream` is a cudaStream_t passed as void*.  Calls only enqueue work on
 *     it; the only host-synchronising calls are mvgs_create, mvgs_reserve,
 *     mvgs_query and (when V·tiles grows past its previous maximum)
 *     mvgs_preprocess.  preprocess → render_fwd → render_bwd → adc_stats is
 *     capturable in a CUDA graph once sizes are reserved.
 *   - Errors are returned as mvgs_status; no exception crosses the ABI.
 *     mvgs_last_error(ctx) gives a text for the last failure.
 *   - Capacities: pairs Q and tile entries K are known only on the device.
 *     When Q > reserved pairs or K > reserved entries the kernels set a device
 *     flag and skip the overflowing work; the next mvgs_query reports
 *     MVGS_ERR_CAPACITY together with the Q and K actually needed.  The caller
 *     reserves and re-runs preprocess.
 */
#ifndef MVGS_H
#define MVGS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MVGS_OK = 0,
    MVGS_ERR_INVALID = -1,  /* null pointer, V ∉ [1, 65535], tiles/view > 65535,
                               sh_degree > 3, sh_degree > sh_stride degree, P < 0,
                               unequal view sizes (R25)                          */
    MVGS_ERR_CAPACITY = -2, /* Q or K exceeded the reserved capacity             */
    MVGS_ERR_STATE = -3,    /* render_fwd / render_bwd / adc_stats out of order  */
    MVGS_ERR_CUDA = -4      /* CUDA runtime error, text in mvgs_last_error       */
} mvgs_status;

typedef struct mvgs_ctx mvgs_ctx;

/* Raw Gaussian parameters, structure of arrays, fp32 (R18).  P:75 "mean μ,
 * scale S, rotation R, color c and opacity o".  Activations (σ, exp, quaternion
 * normalisation) are applied inside the library. */
typedef struct {
    int64_t P;                   /* number of Gaussians                           */
    int32_t sh_degree;           /* active SH degree, 0..3 (R17)                  */
    int32_t sh_stride;           /* SH coefficients stored per Gaussian, ≥ (deg+1)² */
    const float *means;          /* [P,3]                                         */
    const float *log_scales;     /* [P,3]   s = exp(log_scale)                    */
    const float *quats;          /* [P,4]   (w,x,y,z), need not be normalised     */
    const float *opacity_logits; /* [P]     o = sigmoid(logit)                    */
    const float *sh;             /* [P,sh_stride,3]                               */
} mvgs_gaussians;

/* Pinhole camera, 76 bytes (R1): x_c = R x + t, +z forward, +y down. */
typedef struct {
    float R[9];          /* world→camera rotation, row-major */
    float t[3];
    float fx, fy, cx, cy; /* pixels */
    int32_t width, height;
    float znear;         /* participation: t.z > znear (R3) */
} mvgs_camera;

/* Outputs of mvgs_adc_stats: per-Gaussian parameter gradients (overwritten). */
typedef struct {
    float *d_means;          /* [P,3]          */
    float *d_log_scales;     /* [P,3]          */
    float *d_quats;          /* [P,4]          */
    float *d_opacity_logits; /* [P]            */
    float *d_sh;             /* [P,sh_stride,3]; coefficients above sh_degree are set to 0 */
} mvgs_grads;

/* Multi-view ADC statistics.  e1/e2/e_old/vis are overwritten with
 * this batch's raw sums (R20); the *_acc pointers, when non-null, are
 * accumulated into (+=) — the running ADC accumulators of P:4. */
typedef struct {
    float *e1;        /* [P] E1 = Σ_views Σ_pixels ‖∇_{p_i}L‖₂ */
    float *e2;        /* [P] E2 = Σ_views ‖Σ_pixels of the view ∇_{p_i}L‖₂ */
    float *e_old;     /* [P] E_old = ‖Σ_views Σ_pixels ∇_{p_i}L‖₂ (nullable) */
    float *vis;       /* [P] number of views in which the Gaussian covers ≥1 tile (R21) */
    float *e1_acc;    /* [P] nullable, += e1  */
    float *e2_acc;    /* [P] nullable, += e2  */
    float *denom_acc; /* [P] nullable, += vis */
    float *e_old_acc; /* [P] nullable, += e_old (single-view ADC metric, NEXT-3 mode 0) */
    float *max_radius;/* [P] nullable, max= the largest screen radius ⌈3√λ_max⌉ (px, R7) over the
                         batch's views where the Gaussian covers ≥1 tile — the running
                         max_screen_radius of SPEC S:248 that the ADC prune reads             */
    float *gsum;      /* [P,2] nullable, overwritten: Σ_views Σ_pixels ∇_{p_i}L (NDC, R2) — the
                         vector whose norm is E_old.  Additive over views, so a multi-GPU
                         caller sums it with the gradients and takes E_old = ‖gsum‖ after the
                         all-reduce                                            */
} mvgs_adc;

typedef struct {
    int64_t Q;             /* participating (Gaussian, view) pairs needed   */
    int64_t K;             /* tile entries needed                           */
    int64_t cap_pairs;     /* reserved                                      */
    int64_t cap_entries;   /* reserved                                      */
    int64_t max_bucket;    /* longest (view, tile) list                     */
    int64_t n_visible;     /* pairs with tiles > 0                          */
    int32_t overflow;      /* 1 if the last preprocess exceeded a capacity  */
    int32_t V, tiles_x, tiles_y;
    int64_t eval_fwd;      /* (pixel, entry) evaluations of the last render_fwd (Alg. 2 work) */
    int64_t eval_bwd;      /* (pixel, entry) evaluations of the last render_bwd              */
    int64_t exp_fwd;       /* of eval_fwd, those above the exact skip bound (G evaluated)    */
    int64_t exp_bwd;       /* of eval_bwd, likewise                                          */
    /* occupancy of the last mvgs_render_fwd_partial: threads launched /
     * holding a listed in-image pixel, and lane-steps of the entry walk executed (32 × each
     * warp's longest lane, per staged batch) / spent on a live pixel                     */
    int64_t threads_launched, threads_active, lane_steps_launched, lane_steps_active;
} mvgs_stats;

/* Create a context on `device` with initial capacities (0 = a small default).
 * Allocates device workspace (synchronous). */
mvgs_status mvgs_create(mvgs_ctx **out, int device, int64_t max_pairs, int64_t max_entries);
void mvgs_destroy(mvgs_ctx *ctx);
const char *mvgs_last_error(const mvgs_ctx *ctx);
/* Grow capacities to at least (max_pairs, max_entries).  Synchronises the device. */
mvgs_status mvgs_reserve(mvgs_ctx *ctx, int64_t max_pairs, int64_t max_entries);

/* S1–S5: participation and pair allocation, per-pair EWA
 * projection, conic, radius, tile rect and SH colour, duplication into
 * (view, tile) buckets, on-chip depth sort of every bucket, ranges.
 * Participation = the z-test t.z > znear (R27) minus pairs whose tile rect is
 * provably empty (a conservative screen-bound test); the
 * remaining pairs with an empty rect stay allocated and inert.
 *   g     device parameter pointers (kept by the context for render_bwd /
 *         adc_stats; they must stay valid and unchanged until adc_stats).
 *   cams  host, V records; copied before return.
 *   bg    host, 3 floats (R16), may be NULL for black.
 * Pairs are laid out view-major, ascending Gaussian id within a view. */
mvgs_status mvgs_preprocess(mvgs_ctx *ctx, const mvgs_gaussians *g, const mvgs_camera *cams, int32_t V,
                            const float *bg, void *stream);

/* S6 (Eq. 1, Alg. 2): front-to-back compositing of every (view, tile).
 *   rgb       [V,3,H,W]  colour + T_final·bg
 *   T_final   [V,H,W]    final transmittance
 *   n_contrib [V,H,W]    1 + index of the last blended entry of the pixel's list (R14) */
mvgs_status mvgs_render_fwd(mvgs_ctx *ctx, float *rgb, float *T_final, int32_t *n_contrib, void *stream);
/* Same, also writing the rasterizer's predicted depth (NEXT-2): the
 * alpha-weighted expected camera depth depth[V,H,W] = Σ dᵢ αᵢ Tᵢ over the
 * blended entries (no background term).  depth may be NULL. */
mvgs_status mvgs_render_fwd_depth(mvgs_ctx *ctx, float *rgb, float *T_final, int32_t *n_contrib, float *depth,
                                  void *stream);

/* S7: back-to-front adjoint of Eq. (1) for every (view, tile) given
 * dL_drgb [V,3,H,W] and the T_final / n_contrib written by render_fwd.
 * Accumulates per-pair records (∇_{p_i}L sum in NDC, E1 partial, ∂conic, ∂o,
 * ∂rgb) in context memory.  Requires a preceding render_fwd of the same
 * preprocess; a second call without a new preprocess returns MVGS_ERR_STATE. */
mvgs_status mvgs_render_bwd(mvgs_ctx *ctx, const float *dL_drgb, const float *T_final, const int32_t *n_contrib,
                            void *stream);

/* S7 with the ℓ1 photometric loss fused in, for a training step whose targets are 8-bit
 * images: ∂L/∂C = scale·sign(C − t·fl(1/255)) is formed per pixel inside the backward — the
 * values mvgs_loss_grad_u8 (mode 0) would write — from rgb [V,3,H,W] fp32 (render_fwd's image)
 * and target [V,3,H,W] uint8 (device); `loss` (device [1] fp64, nullable) is overwritten with
 * Σ|C − t/255| (summed with one double atomic per warp: the last bits depend on their order).
 * Same state rules and outputs as mvgs_render_bwd; no ∂L/∂C buffer is written. */
mvgs_status mvgs_render_bwd_l1(mvgs_ctx *ctx, const float *rgb, const uint8_t *target, float scale,
                               const float *T_final, const int32_t *n_contrib, double *loss, void *stream);

/* S8–S9: per-Gaussian chain rule summed over the batch's views
 * and the ADC statistics E1, E2, E_old, vis.  `grads` and `adc`
 * are host structs of device pointers.  Requires a preceding render_bwd. */
mvgs_status mvgs_adc_stats(mvgs_ctx *ctx, const mvgs_grads *grads, const mvgs_adc *adc, void *stream);

/* The same for the Gaussians [g_begin, g_end) only, g_begin a multiple of 256
 * (the pair-slot block size): every pointer in `grads` and `adc` addresses the
 * row of Gaussian g_begin (row g − g_begin of each output).  Chunks may be
 * issued in any order and number after one render_bwd; a multi-GPU caller
 * all-reduces each finished chunk while the next one computes (SURVEY §8(e)
 * lever 1).  mvgs_adc_stats ≡ range [0, P).  MVGS_ERR_INVALID
 * for g_begin % 256 ≠ 0, g_begin < 0, g_end < g_begin, g_end > P or a null
 * output pointer of a non-empty range; MVGS_ERR_STATE without a render_bwd. */
mvgs_status mvgs_adc_stats_range(mvgs_ctx *ctx, int64_t g_begin, int64_t g_end, const mvgs_grads *grads,
                                 const mvgs_adc *adc, void *stream);

/* ---- Owner-sharded exchange (SURVEY §8(e) lever 3) ------------------------
 * Every output is a sum over views, so instead of all-reducing
 * 4·(11+S+5)·P bytes of per-Gaussian outputs, ranks can send each per-pair gradient slot
 * (48 B: Σ∇, e1, ∂conic, ∂o, ∂rgb and the pair's flags) to the rank that OWNS its Gaussian; the
 * owner lays out all views' slots of its Gaussians exactly as a single GPU would (the same
 * participation decisions and ballot ranking) and runs S8–S9 over all views.  E1, E2 and
 * E_old are then exact; the owner holds the full sums for its range (reduce-scatter semantics).
 *
 * mvgs_owner_slices (after mvgs_render_bwd): for this context's views and owners
 *   [g_bounds[o], g_bounds[o+1]) (g_bounds host [N+1], 0 = first, P = last, multiples of 256 or P),
 *   writes slot_off (host [V][N+1]): owner o's slots of local view v are
 *   [slot_off[v][o], slot_off[v][o+1]) of the slot array returned in *slots (device,
 *   PG_STRIDE = 12 floats per slot).  Synchronises the stream.
 * mvgs_owner_prepare: this context owns [g_begin, g_end) (g_begin % 256 == 0, or an empty range) of the Gaussians
 *   of its last preprocess; cams_all (host [V_all]) are every rank's views in global order.
 *   Builds the owner's slot layout and writes view_off (host [V_all+1]): view v's slots go to
 *   [view_off[v], view_off[v+1]) of *recv (device, context-owned, 12 floats per slot) —
 *   exactly as many as the renderer of view v reports for this owner.  Synchronises.
 * mvgs_owner_adc_stats: S8–S9 of the owned range over all views from *recv; outputs are
 *   addressed relative to g_begin (as mvgs_adc_stats_range).  MVGS_ERR_STATE without a
 *   preceding mvgs_owner_prepare. */
mvgs_status mvgs_owner_slices(mvgs_ctx *ctx, const int64_t *g_bounds, int32_t N, int64_t *slot_off, float **slots,
                              void *stream);
mvgs_status mvgs_owner_prepare(mvgs_ctx *ctx, const mvgs_camera *cams_all, int32_t V_all, int64_t g_begin,
                               int64_t g_end, int64_t *view_off, float **recv, void *stream);
mvgs_status mvgs_owner_adc_stats(mvgs_ctx *ctx, const mvgs_grads *grads, const mvgs_adc *adc, void *stream);

/* E_old = ‖gsum‖ for n Gaussians (R49): gsum device [n,2] (8-B aligned), e_old [n] overwritten
 * and/or e_old_acc [n] += (either may be NULL, not both).  Used after a multi-GPU sum of gsum,
 * where E_old is not additive but gsum is. */
mvgs_status mvgs_e_old_from_gsum(mvgs_ctx *ctx, const float *gsum, int64_t n, float *e_old, float *e_old_acc,
                                 void *stream);

/* NEXT-2: the 3D distance-aware D-SSIM loss and its gradient.
 *   SSIM = (2μ1μ2 + C1)(2τ12 + C2) / ((μ1² + μ2² + C1)(τ1² + τ2² + C2))
 * with the moments μ, τ taken under the 3D kernel
 *   K*_σ(u, v) ∝ exp(−‖X_uv − X_c‖² / 2σ²)
 * where X is a pixel's camera-space point from `depth` (render_fwd_depth).
 * Readings: 11×11 windows, C1 = 0.01², C2 = 0.03²; weights
 * renormalised over in-image pixels that are not background (T_final > 0.999);
 * a background centre uses the plain 2D Gaussian (σ = sigma_px); σ at a centre
 * c is sigma_px·depth_c/fx; depth and T_final are constants of the loss.
 *   cams     host array [V] (only fx, fy, cx, cy are read; copied into the launch)
 *   img, target         device [V,3,H,W] fp32 (rendered / ground-truth image)
 *   depth, T_final      device [V,H,W] fp32
 *   loss     device [1] fp32: 1 − mean SSIM over V·3·H·W (window centre, channel)
 *   dL_dimg  device [V,3,H,W] or NULL: ∂loss/∂img, ready for mvgs_render_bwd
 * Independent of preprocess state; grows context scratch of 48·V·H·W bytes
 * (synchronising when it does).  MVGS_ERR_INVALID on null inputs, V ∉
 * [1, 65535], H, W < 1, sigma_px ≤ 0 or fx, fy ≤ 0. */
mvgs_status mvgs_dssim3d(mvgs_ctx *ctx, const mvgs_camera *cams, int32_t V, int32_t H, int32_t W, const float *img,
                         const float *target, const float *depth, const float *T_final, float sigma_px, float *loss,
                         float *dL_dimg, void *stream);

/* ---- NEXT-3: the multi-view ADC step (P:4) --------------------------- */

/* Per-interval densification policy.  Readings R35–R42. */
typedef struct {
    float grad_threshold_split; /* τ on the mean of E1 (mode 1) or E_old (mode 0): split if ≥ and large */
    float grad_threshold_clone; /* τ on the mean of E2 (mode 1) or E_old (mode 0): clone if ≥ and small */
    float size_threshold;       /* world units, > 0: "large" ⟺ max scale > size_threshold          */
    float split_factor;         /* > 0: children get scale / split_factor (3DGS 1.6)                 */
    int32_t split_count;        /* N ∈ [2, 8] children per split                                      */
    float prune_opacity;        /* prune if opacity < prune_opacity × batch_views, ∈ (0, 1)   */
    float prune_scale_max;      /* prune if max scale > this (world units); ≤ 0 disables             */
    int32_t metric_mode;        /* 0: E_old for both (single-view ADC), 1: E1 split / E2 clone */
    int32_t batch_views;        /* B ≥ 1, images per iteration                                       */
} mvgs_adc_config;

/* Running accumulators (device [P]; the *_acc outputs of mvgs_adc_stats). e_old_acc is read in
 * mode 0 only, e1/e2 in mode 1 only; the unused ones may be NULL. */
typedef struct {
    const float *e1_acc, *e2_acc, *e_old_acc, *denom_acc;
} mvgs_adc_accum;

/* Output Gaussian arrays (device), `capacity` rows each; sh_stride must equal the input's. */
typedef struct {
    int64_t capacity;
    int32_t sh_stride;
    float *means, *log_scales, *quats, *opacity_logits, *sh;
} mvgs_gaussians_out;

typedef struct {
    int64_t n_split;  /* parents split (each replaced by split_count children)           */
    int64_t n_clone;  /* parents cloned                                                    */
    int64_t n_pruned; /* emitted Gaussians (kept, clones, children) removed by the prune  */
    int64_t P_new;    /* rows written = P + (N−1)·n_split + n_clone − n_pruned             */
} mvgs_adc_report;

/* One ADC event.  Per Gaussian g, with Ē = acc/denom in fp32 (0 where denom = 0):
 *   split ⟺ Ē_split ≥ τ_split ∧ max log_scale > fp32(ln size_threshold)
 *   clone ⟺ Ē_clone ≥ τ_clone ∧ ¬large
 * Emitted in canonical order — for g = 0..P−1: g itself unless split, its clone, its N children
 * (child k: mean + R(q̂)·(exp(log_scale) ⊙ noise[g,k]), log_scale − fp32(ln split_factor), other
 * parameters copied) — then every emitted row with opacity logit < fp32(logit(prune_opacity·B))
 * or max log_scale > fp32(ln prune_scale_max) is dropped (prune-compaction).
 *   noise   device [P, split_count, 3] standard normals (the step's random draw, an input)
 *   origin  device [capacity] int32: the input row each output row derives from
 *   kind    device [capacity] uint8: 0 kept, 1 clone, 2 split child
 *   report  host; filled on success and on MVGS_ERR_CAPACITY (P_new > out->capacity, nothing
 *           written).  Synchronises the stream once (the new count is needed on the host).
 * quats and sh (input and output) must be 16-byte aligned.
 * MVGS_ERR_INVALID on null pointers, P < 0, sh_stride mismatch, misalignment or a config
 * outside its range. */
mvgs_status mvgs_adc_step(mvgs_ctx *ctx, const mvgs_gaussians *g, const mvgs_adc_accum *acc, const float *noise,
                          const mvgs_adc_config *cfg, const mvgs_gaussians_out *out, int32_t *origin, uint8_t *kind,
                          mvgs_adc_report *report, void *stream);

/* Optimiser-state resize after mvgs_adc_step: dst[i, :] = src[origin[i], :] for kept rows, 0 for
 * clones and split children (new Gaussians start with zero moments).  src [P, width],
 * dst [P_new, width] device fp32, distinct buffers. */
mvgs_status mvgs_adc_remap(mvgs_ctx *ctx, const float *src, float *dst, int64_t width, const int32_t *origin,
                           const uint8_t *kind, int64_t P_new, void *stream);

/* ---- NEXT-4: mini-batch gradient-variance laboratory ------------------------- */

/* Per-pixel loss gradient of a rendered batch: mode 0 (ℓ1) dL = scale·sign(C − C*),
 * mode 1 (ℓ2) dL = 2·scale·(C − C*); `loss` (device [1] fp64, nullable) receives Σ|C − C*| or
 * Σ(C − C*)² (multiply by `scale` for the mean).  rgb, target, dL_drgb device [n] fp32
 * (normally [V,3,H,W] with scale = 1/(3·V·H·W)).  Deterministic fixed-order reduction. */
mvgs_status mvgs_loss_grad(mvgs_ctx *ctx, const float *rgb, const float *target, int64_t n, int32_t mode, float scale,
                           float *dL_drgb, double *loss, void *stream);

/* The same with an 8-bit target image (the photographs a training step uploads):
 * C* = t · fl(1/255) in fp32 for each element t of `target` (device [n] uint8), otherwise
 * identical to mvgs_loss_grad (a quarter of its host→device bytes per step). */
mvgs_status mvgs_loss_grad_u8(mvgs_ctx *ctx, const float *rgb, const uint8_t *target, int64_t n, int32_t mode,
                              float scale, float *dL_drgb, double *loss, void *stream);

/* Monte-Carlo accumulators of the variance estimator of §4.2 for one mini-batch
 * gradient g (device [n] fp32, e.g. the ∂L/∂means of mvgs_adc_stats):
 *   sum[i] += g[i]  (device [n] fp64),   *sumsq += ‖g‖²  (device [1] fp64). */
mvgs_status mvgs_grad_moments(mvgs_ctx *ctx, const float *g, int64_t n, double *sum, double *sumsq, void *stream);

/* 𝕍 ≈ (1/K)Σ_k‖g_k‖² − ‖(1/K)Σ_k g_k‖² from the accumulators after K mini-batches
 * (P:152–156); `variance` device [1] fp64, distinct from sumsq. */
mvgs_status mvgs_grad_variance(mvgs_ctx *ctx, const double *sum, int64_t n, const double *sumsq, int64_t K,
                               double *variance, void *stream);

/* Synchronise and report sizes and the capacity flag of the last preprocess.
 * Returns MVGS_ERR_CAPACITY if it overflowed. */
mvgs_status mvgs_query(mvgs_ctx *ctx, mvgs_stats *out);

/* Parity export (tests): copy the (view, tile) ranges [V*tiles+1] (int64) and
 * the Gaussian id of every sorted entry [K] (int32) into caller device buffers. */
mvgs_status mvgs_export_lists(mvgs_ctx *ctx, int64_t *range_start, int32_t *entry_gid, void *stream);

/* Parity export (tests): per pair q < Q —
 *   pair_ids [Q,2] int32   (view, gid)
 *   pair_i   [Q,8] int32   (radius, rx0, ry0, rx1, ry1, tiles, clamp bits, 0); the radius
 *                          is recomputed by the export (the path keeps only the rect)
 *   pair_f   [Q,12] fp32   (depth, px, py, A, B, C, opacity, r, g, b, 0, 0)
 *   pair_g   [Q,10] fp32   (Σ∇x, Σ∇y, e1, ∂A, ∂B, ∂C, ∂o, ∂r, ∂g, ∂b) after render_bwd
 * Any pointer may be NULL. */
mvgs_status mvgs_export_pairs(mvgs_ctx *ctx, int32_t *pair_ids, int32_t *pair_i, float *pair_f, float *pair_g,
                              void *stream);

/* Parity export (tests): while nblend is non-NULL, every following mvgs_render_bwd also
 * writes nblend[V,H,W] (int32, caller-owned device buffer sized for that call) = the number of
 * list entries the backward treated as blended at each pixel (its re-taken α ≥ 1/255 decisions
 * up to n_contrib); it must equal the forward's count of blended entries.  NULL switches it
 * off (the default).  MVGS_ERR_INVALID for a NULL ctx. */
mvgs_status mvgs_set_debug_blend_counts(mvgs_ctx *ctx, int32_t *nblend);

/* NEXT-1: partial rendering (Alg. 3).  Each (view, tile)
 * renders only the S pixels listed in `pix` — the index array A of Alg. 3 —
 * so a V-view batch can render one image's worth of pixels.
 *   pix   [V, T, S] int32, local pixel index 0..255 inside the 16×16 tile
 *         (row-major); a listed pixel outside the image is skipped ("isValid").
 *         T = tiles_x·tiles_y of the preceding preprocess.
 *   mode  MVGS_PARTIAL_THREAD_EFFICIENT: one block of ⌈S/32⌉·32 threads per
 *         (view, tile), thread i renders pix[.., i] (Alg. 3);
 *         MVGS_PARTIAL_MASKED: one 256-thread block per (view, tile) with the
 *         unlisted pixels masked off (the binary-mask baseline).
 *   rgb [V,T,S,3], T_final [V,T,S], n_contrib [V,T,S] per listed pixel; the
 *   values equal the full render's at those pixels.  render_bwd_partial takes
 *   dL_drgb [V,T,S,3] and accumulates the same per-pair records as
 *   mvgs_render_bwd (adc_stats follows as usual).  Same ordering rules as the
 *   full calls (fwd after preprocess, bwd after fwd). */
#define MVGS_PARTIAL_THREAD_EFFICIENT 0
#define MVGS_PARTIAL_MASKED 1
mvgs_status mvgs_render_fwd_partial(mvgs_ctx *ctx, const int32_t *pix, int32_t S, int32_t mode, float *rgb,
                                    float *T_final, int32_t *n_contrib, void *stream);
mvgs_status mvgs_render_bwd_partial(mvgs_ctx *ctx, const int32_t *pix, int32_t S, int32_t mode, const float *dL_drgb,
                                    const float *T_final, const int32_t *n_contrib, void *stream);

/* Stage timing (measurement).  While enabled, every call records a pair of
 * CUDA events on its stream around each kernel stage.  mvgs_stage_times
 * synchronises on them, writes into ms[0..n) the AVERAGE milliseconds per run
 * of each stage over all runs recorded since the previous read (0 if none), in
 * the order of MVGS_STAGE_NAMES, clears the record, and returns the number of
 * stages written. */
#define MVGS_NUM_STAGES 11
#define MVGS_STAGE_NAMES "count,scan_pairs,project,scan_buckets,sort_pairs,dup,sort_entries,render_fwd,render_bwd,gauss_bwd,dssim"
mvgs_status mvgs_set_timing(mvgs_ctx *ctx, int enable);
int mvgs_stage_times(mvgs_ctx *ctx, float *ms, int n);

/* Evaluation counting (statistics).  While enabled (the default), the full-image
 * compositing kernels count their (pixel, entry) evaluations and canonical-exp
 * evaluations; mvgs_query reports them (eval_fwd, eval_bwd, exp_fwd, exp_bwd) for
 * the last preprocess → fwd → bwd sequence.  Disabling it removes the counting
 * from the kernels' inner loops (the counts then read 0); results are unchanged.
 * Returns MVGS_ERR_INVALID for a NULL ctx. */
mvgs_status mvgs_set_eval_counting(mvgs_ctx *ctx, int enable);

/* Forward staging by TMA (Alg. 2's batched fetch): when enabled,
 * mvgs_render_fwd stages each batch of list records with cp.async.bulk.tensor gather4 into a
 * double-buffered shared-memory ring signalled by mbarriers, instead of per-thread loads.
 * Results are bit-identical either way; it is off by default because it measured slower
 * (garden forward 0.379 → 0.436 ms).  MVGS_ERR_CUDA if the driver refused the tensor map,
 * MVGS_ERR_INVALID for a NULL ctx. */
mvgs_status mvgs_set_tma(mvgs_ctx *ctx, int enable);

#ifdef __cplusplus
}
#endif
#endif /* MVGS_H */
