// mvgs_abi.cu — the C ABI of libmvgs.so (include/mvgs.h): context, workspace,
// argument validation, and the launch sequence of each call.  No arithmetic of
// the method lives here; every step runs in the kernels of k_*.cu.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <new>
#include "ca.cuh"
#include "internal.cuh"
#include "tma.cuh"

using namespace mvgs;

namespace {

mvgs_status fail(mvgs_ctx* c, mvgs_status st, const char* msg) {
    if (c) c->err = msg;
    return st;
}

mvgs_status cuda_fail(mvgs_ctx* c, cudaError_t e, const char* where) {
    if (c) {
        c->err = std::string(where) + ": " + cudaGetErrorString(e);
    }
    return MVGS_ERR_CUDA;
}

#define CK(expr)                                              \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
    } while (0)

template <class T>
cudaError_t grow(T*& p, int64_t& cap, int64_t need, int64_t elem_per = 1) {
    if (need <= cap && p) return cudaSuccess;
    int64_t n = need + need / 4 + 64;
    if (p) {
        cudaError_t e = cudaFree(p);
        if (e != cudaSuccess) return e;
        p = nullptr;
    }
    cudaError_t e = cudaMalloc(&p, sizeof(T) * n * elem_per);
    if (e != cudaSuccess) {
        cap = 0;
        return e;
    }
    cap = n;
    return cudaSuccess;
}

cudaError_t alloc_pairs(mvgs_ctx* c, int64_t n) {
    cudaFree(c->d_rec); cudaFree(c->d_pgrad);
    cudaFree(c->d_pkey); cudaFree(c->d_pval); cudaFree(c->d_pkey2); cudaFree(c->d_pval2); cudaFree(c->d_ecount);
    cudaFree(c->d_prect); cudaFree(c->d_prect2); cudaFree(c->d_pflag);
    c->d_prect = c->d_prect2 = nullptr;
    c->d_pflag = nullptr;
    c->d_rec = nullptr; c->d_pgrad = nullptr;
    c->d_pkey = c->d_pval = c->d_pkey2 = c->d_pval2 = nullptr;
    c->d_ecount = nullptr;
    c->cap_pairs = 0;
    cudaError_t e;
    if ((e = cudaMalloc(&c->d_rec, sizeof(float4) * REC_F4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_pgrad, sizeof(float) * PG_STRIDE * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_pkey, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_pval, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_pkey2, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_pval2, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_ecount, 4 * (n + 1))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_prect, sizeof(uint2) * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_pflag, sizeof(uint32_t) * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_prect2, sizeof(uint2) * n)) != cudaSuccess) return e;
    c->cap_pairs = n;
    c->rec_map_ok = mvgs::encode_record_map(&c->rec_map, c->d_rec, n);
    return cudaSuccess;
}

// radix digit counts and scan scratch sized for the current capacities
cudaError_t alloc_sort_scratch(mvgs_ctx* c) {
    const int64_t cap = std::max(c->cap_pairs, c->cap_entries);
    const int64_t need = radix_counts_size(cap);
    if (need > c->cap_rs || !c->d_rs) {
        cudaFree(c->d_rs);
        c->d_rs = nullptr;
        c->cap_rs = 0;
        cudaError_t e = cudaMalloc(&c->d_rs, sizeof(int) * need);
        if (e != cudaSuccess) return e;
        c->cap_rs = need;
    }
    const int64_t need_scan = scan_tmp_size((int)std::max(need, c->cap_pairs + 1));
    if (need_scan > c->cap_scan || !c->d_scan) {
        cudaFree(c->d_scan);
        c->d_scan = nullptr;
        c->cap_scan = 0;
        cudaError_t e = cudaMalloc(&c->d_scan, sizeof(int) * need_scan);
        if (e != cudaSuccess) return e;
        c->cap_scan = need_scan;
    }
    return cudaSuccess;
}

cudaError_t alloc_entries(mvgs_ctx* c, int64_t n) {
    cudaFree(c->d_key); cudaFree(c->d_val); cudaFree(c->d_key2); cudaFree(c->d_val2);
    c->d_key = c->d_val = c->d_key2 = c->d_val2 = nullptr;
    c->cap_entries = 0;
    cudaError_t e;
    if ((e = cudaMalloc(&c->d_key, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_val, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_key2, 4 * n)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c->d_val2, 4 * n)) != cudaSuccess) return e;
    c->cap_entries = n;
    return cudaSuccess;
}

enum { ST_COUNT, ST_SCAN_PAIRS, ST_PROJECT, ST_SCAN_BUCKETS, ST_SORT_PAIRS, ST_DUP, ST_SORT_ENTRIES, ST_FWD, ST_BWD,
       ST_GAUSS, ST_DSSIM };

cudaEvent_t pool_get(mvgs_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct StageTimer {  // records a pair of events around one stage when timing is enabled
    mvgs_ctx* c;
    int st;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    StageTimer(mvgs_ctx* c_, int st_, cudaStream_t s_) : c(c_), st(st_), s(s_) {
        if (c->timing) {
            a = pool_get(c);
            cudaEventRecord(a, s);
        }
    }
    ~StageTimer() {
        if (a) {
            cudaEvent_t b = pool_get(c);
            cudaEventRecord(b, s);
            c->ev_rec[st].emplace_back(a, b);
        }
    }
};
#define STAGE(id) StageTimer _timer_##id(ctx, id, s)

void fill_launch(mvgs_ctx* c) {
    Launch& L = c->L;
    L.cams = c->d_cams;
    L.cap_pairs = c->cap_pairs;
    L.cap_entries = c->cap_entries;
    L.blk_off = c->d_blk;
    L.bucket_off = c->d_bucket;
    L.rec = c->d_rec;
    L.pflag = c->d_pflag;
    L.pgrad = c->d_pgrad;
    L.key = c->d_key;
    L.val = c->d_val;
    L.key2 = c->d_key2;
    L.val2 = c->d_val2;
    L.pkey = c->d_pkey;
    L.pval = c->d_pval;
    L.pkey2 = c->d_pkey2;
    L.pval2 = c->d_pval2;
    L.prect = c->d_prect;
    L.prect2 = c->d_prect2;
    L.ecount = c->d_ecount;
    L.rs_counts = c->d_rs;
    L.scan_tmp = c->d_scan;
    L.counters = c->d_counters;
    L.counters64 = c->d_counters64;
}

}  // namespace

extern "C" {

mvgs_status mvgs_create(mvgs_ctx** out, int device, int64_t max_pairs, int64_t max_entries) {
    if (!out) return MVGS_ERR_INVALID;
    *out = nullptr;
    mvgs_ctx* ctx = new (std::nothrow) mvgs_ctx();
    if (!ctx) return MVGS_ERR_INVALID;
    ctx->device = device;
    if (const char* m = getenv("MVGS_TMA")) ctx->use_tma = strcmp(m, "1") == 0;
    if (const char* m = getenv("MVGS_LPT")) ctx->use_lpt = strcmp(m, "1") == 0;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete ctx;
        return MVGS_ERR_CUDA;
    }
    if (max_pairs <= 0) max_pairs = 1 << 16;
    if (max_entries <= 0) max_entries = 1 << 18;
    if (max_pairs > INT32_MAX || max_entries > INT32_MAX) {
        delete ctx;
        return MVGS_ERR_INVALID;
    }
    if ((e = alloc_pairs(ctx, max_pairs)) != cudaSuccess || (e = alloc_entries(ctx, max_entries)) != cudaSuccess ||
        (e = alloc_sort_scratch(ctx)) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_counters, sizeof(int) * C_NCOUNTERS)) != cudaSuccess ||
        (e = cudaMemset(ctx->d_counters, 0, sizeof(int) * C_NCOUNTERS)) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_counters64, sizeof(unsigned long long) * 16)) != cudaSuccess ||
        (e = cudaMemset(ctx->d_counters64, 0, sizeof(unsigned long long) * 16)) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_lab_part, sizeof(double) * lab_partials())) != cudaSuccess) {
        mvgs_destroy(ctx);
        return MVGS_ERR_CUDA;
    }
    *out = ctx;
    return MVGS_OK;
}

void mvgs_destroy(mvgs_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    cudaFree(ctx->d_cams); cudaFree(ctx->d_blk); cudaFree(ctx->d_bucket); cudaFree(ctx->d_order);
    cudaFree(ctx->d_rec); cudaFree(ctx->d_pgrad);
    cudaFree(ctx->d_key); cudaFree(ctx->d_val); cudaFree(ctx->d_key2); cudaFree(ctx->d_val2);
    cudaFree(ctx->d_pkey); cudaFree(ctx->d_pval); cudaFree(ctx->d_pkey2); cudaFree(ctx->d_pval2);
    cudaFree(ctx->d_ecount); cudaFree(ctx->d_rs); cudaFree(ctx->d_prect); cudaFree(ctx->d_prect2);
    cudaFree(ctx->d_pflag);
    cudaFree(ctx->d_counters); cudaFree(ctx->d_counters64); cudaFree(ctx->d_scan);
    cudaFree(ctx->d_dssim_coef); cudaFree(ctx->d_dssim_part);
    cudaFree(ctx->d_lab_part); cudaFree(ctx->d_pmask);
    cudaFree(ctx->d_ocams); cudaFree(ctx->d_oblk); cudaFree(ctx->d_oscan); cudaFree(ctx->d_opmask); cudaFree(ctx->d_orecv);
    cudaFree(ctx->d_adc_cnt); cudaFree(ctx->d_adc_flags); cudaFree(ctx->d_adc_tmp); cudaFree(ctx->d_adc_rep);
    if (ctx->h_adc_rep) cudaFreeHost(ctx->h_adc_rep);
    for (int i = 0; i < MVGS_NUM_STAGES; i++)
        for (auto& p : ctx->ev_rec[i]) {
            cudaEventDestroy(p.first);
            cudaEventDestroy(p.second);
        }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    delete ctx;
}

const char* mvgs_last_error(const mvgs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

mvgs_status mvgs_reserve(mvgs_ctx* ctx, int64_t max_pairs, int64_t max_entries) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (max_pairs > INT32_MAX || max_entries > INT32_MAX) return fail(ctx, MVGS_ERR_INVALID, "capacity above 2^31-1");
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceSynchronize());
    if (max_pairs > ctx->cap_pairs) CK(alloc_pairs(ctx, max_pairs));
    if (max_entries > ctx->cap_entries) CK(alloc_entries(ctx, max_entries));
    CK(alloc_sort_scratch(ctx));
    ctx->state = 0;
    return MVGS_OK;
}

mvgs_status mvgs_preprocess(mvgs_ctx* ctx, const mvgs_gaussians* g, const mvgs_camera* cams, int32_t V,
                            const float* bg, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (!g || !cams) return fail(ctx, MVGS_ERR_INVALID, "null gaussians or cameras");
    if (V < 1 || V > 65535) return fail(ctx, MVGS_ERR_INVALID, "V out of [1, 65535] (R9)");
    if (g->P < 0 || g->P > INT32_MAX) return fail(ctx, MVGS_ERR_INVALID, "P out of range");
    if (g->sh_degree < 0 || g->sh_degree > 3) return fail(ctx, MVGS_ERR_INVALID, "sh_degree must be 0..3");
    if (g->sh_stride < (g->sh_degree + 1) * (g->sh_degree + 1)) return fail(ctx, MVGS_ERR_INVALID, "sh_stride too small");
    if (g->P > 0 && (!g->means || !g->log_scales || !g->quats || !g->opacity_logits || !g->sh))
        return fail(ctx, MVGS_ERR_INVALID, "null parameter pointer");
    const int W = cams[0].width, H = cams[0].height;
    if (W <= 0 || H <= 0) return fail(ctx, MVGS_ERR_INVALID, "non-positive image size");
    for (int v = 0; v < V; v++)  // depth keys are the float bits of t.z > znear > 0 (R9): ordered only if positive
        if (!(cams[v].znear > 0.f) || !(cams[v].fx > 0.f) || !(cams[v].fy > 0.f))
            return fail(ctx, MVGS_ERR_INVALID, "camera needs znear > 0, fx > 0, fy > 0 (R3, R9)");
    for (int v = 1; v < V; v++)
        if (cams[v].width != W || cams[v].height != H) return fail(ctx, MVGS_ERR_INVALID, "views differ in size (R25)");
    const int TX = (W + TILE - 1) / TILE, TY = (H + TILE - 1) / TILE;
    if ((int64_t)TX * TY > 65535) return fail(ctx, MVGS_ERR_INVALID, "more than 65535 tiles per view (R9)");
    const int NB = (int)((g->P + BLK - 1) / BLK);
    const int64_t nblk = (int64_t)V * (NB > 0 ? NB : 1);
    const int64_t nbuck = (int64_t)V * TX * TY;
    if (nblk + 1 > INT32_MAX || nbuck + 1 > INT32_MAX) return fail(ctx, MVGS_ERR_INVALID, "batch too large");
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaSetDevice(ctx->device));
    // workspace growth (synchronous only when it grows)
    // scan block sums, and the ranges close-up's per-1024-bucket minima (k_sort.cu)
    int64_t need_scan = std::max<int64_t>(scan_tmp_size((int)std::max(nblk, nbuck)), nbuck / 1024 + 2);
    const int64_t need_pmask = V <= 32 ? std::max<int64_t>(g->P, 1) : 1;  // participation masks (V ≤ 32)
    if (nblk + 1 > ctx->cap_blk || nbuck + 1 > ctx->cap_buckets || V > ctx->cap_cams || need_scan > ctx->cap_scan ||
        need_pmask > ctx->cap_pmask || !ctx->d_blk) {
        CK(cudaDeviceSynchronize());
        CK(grow(ctx->d_pmask, ctx->cap_pmask, need_pmask));
        CK(grow(ctx->d_blk, ctx->cap_blk, nblk + 1));
        int64_t cb = ctx->cap_buckets;
        CK(grow(ctx->d_bucket, ctx->cap_buckets, nbuck + 1));
        CK(grow(ctx->d_order, cb, nbuck + 1));
        if (need_scan > ctx->cap_scan) {
            cudaFree(ctx->d_scan);
            ctx->d_scan = nullptr;
            ctx->cap_scan = 0;
            CK(grow(ctx->d_scan, ctx->cap_scan, need_scan));
        }
        if (V > ctx->cap_cams) {
            cudaFree(ctx->d_cams);
            ctx->d_cams = nullptr;
            int64_t n = V + 8;
            CK(cudaMalloc(&ctx->d_cams, sizeof(mvgs_camera) * n));
            ctx->cap_cams = n;
        }
    }
    // cameras: written to the device by a tiny kernel that receives them BY VALUE (kernel
    // parameters, ≤ 32 per launch).  No host buffer is shared between calls, the host never
    // waits, and a CUDA graph captured here replays exactly the cameras given here (the values
    // live in its kernel node), however the context is used afterwards.
    CK(launch_set_cams(cams, V, ctx->d_cams, s));

    ctx->g = *g;
    Launch& L = ctx->L;
    L.P = g->P;
    L.V = V; L.W = W; L.H = H; L.TX = TX; L.TY = TY; L.T = TX * TY; L.NB = NB;
    L.sh_degree = g->sh_degree;
    L.sh_stride = g->sh_stride;
    L.count_evals = ctx->count_evals ? 1 : 0;
    L.pmask = V <= 32 ? ctx->d_pmask : nullptr;  // k_count stores each Gaussian's participation bits
    for (int k = 0; k < 3; k++) L.bg[k] = bg ? bg[k] : 0.f;
    L.means = g->means; L.log_scales = g->log_scales; L.quats = g->quats; L.opac = g->opacity_logits; L.sh = g->sh;
    fill_launch(ctx);
    ctx->last_stream = s;

    CK(cudaMemsetAsync(ctx->d_counters, 0, sizeof(int) * C_NCOUNTERS, s));
    CK(cudaMemsetAsync(ctx->d_counters64 + 4, 0, sizeof(unsigned long long), s));
    if (NB > 0) {
        { STAGE(ST_COUNT); CK(launch_count(L, s)); }                                                 // S1
        { STAGE(ST_SCAN_PAIRS); CK(scan_exclusive(ctx->d_blk, (int)nblk, ctx->d_counters + C_Q, ctx->d_scan, s)); }
        { STAGE(ST_PROJECT); CK(launch_project(L, s)); }                                             // S2 (+ S3 histogram)
    } else {
        CK(cudaMemsetAsync(ctx->d_blk, 0, sizeof(int) * (nblk + 1), s));
    }
    const uint32_t* order = L.pval;
    const uint2* rect = L.prect;
    uint32_t* sorted = L.val;
    if (NB > 0) {
        { STAGE(ST_SORT_PAIRS); CK(launch_sort_pairs(L, &order, &rect, s)); }                        // S4a
        { STAGE(ST_DUP); CK(launch_dup_sort(L, order, rect, s)); }                                   // S3
        { STAGE(ST_SORT_ENTRIES); CK(launch_sort_entries(L, &sorted, s));                           // S4b + S5
          if (ctx->use_lpt) CK(launch_lpt_order(L, ctx->d_order, s)); }                              // CTA order
    } else {
        CK(cudaMemsetAsync(ctx->d_bucket, 0, sizeof(int) * (nbuck + 1), s));
    }
    L.sorted = sorted;
    L.order = (NB > 0 && ctx->use_lpt) ? ctx->d_order : nullptr;
    ctx->state = 1;
    return MVGS_OK;
}

mvgs_status mvgs_render_fwd(mvgs_ctx* ctx, float* rgb, float* T_final, int32_t* n_contrib, void* stream) {
    return mvgs_render_fwd_depth(ctx, rgb, T_final, n_contrib, nullptr, stream);
}

mvgs_status mvgs_render_fwd_depth(mvgs_ctx* ctx, float* rgb, float* T_final, int32_t* n_contrib, float* depth,
                                  void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state < 1) return fail(ctx, MVGS_ERR_STATE, "render_fwd before preprocess");
    if (!rgb || !T_final || !n_contrib) return fail(ctx, MVGS_ERR_INVALID, "null output");
    CK(cudaSetDevice(ctx->device));
    ctx->last_stream = (cudaStream_t)stream;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(ctx->d_counters64, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(ctx->d_counters64 + 2, 0, sizeof(unsigned long long), s));
    const CUtensorMap* tm = (ctx->use_tma && ctx->rec_map_ok) ? &ctx->rec_map : nullptr;
    { STAGE(ST_FWD); CK(launch_render_fwd(ctx->L, rgb, T_final, n_contrib, depth, tm, s)); }  // S6
    ctx->state = 2;
    return MVGS_OK;
}

mvgs_status mvgs_render_bwd(mvgs_ctx* ctx, const float* dL_drgb, const float* T_final, const int32_t* n_contrib,
                            void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state != 2) return fail(ctx, MVGS_ERR_STATE, "render_bwd needs a render_fwd of a fresh preprocess");
    if (!dL_drgb || !T_final || !n_contrib) return fail(ctx, MVGS_ERR_INVALID, "null input");
    CK(cudaSetDevice(ctx->device));
    ctx->last_stream = (cudaStream_t)stream;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(ctx->d_counters64 + 1, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(ctx->d_counters64 + 3, 0, sizeof(unsigned long long), s));
    { STAGE(ST_BWD); CK(launch_render_bwd(ctx->L, dL_drgb, T_final, n_contrib, s)); }  // S7
    ctx->state = 3;
    return MVGS_OK;
}

mvgs_status mvgs_render_bwd_l1(mvgs_ctx* ctx, const float* rgb, const uint8_t* target, float scale,
                               const float* T_final, const int32_t* n_contrib, double* loss, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state != 2) return fail(ctx, MVGS_ERR_STATE, "render_bwd_l1 needs a render_fwd of a fresh preprocess");
    if (!rgb || !target || !T_final || !n_contrib) return fail(ctx, MVGS_ERR_INVALID, "null input");
    CK(cudaSetDevice(ctx->device));
    ctx->last_stream = (cudaStream_t)stream;
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemsetAsync(ctx->d_counters64 + 1, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(ctx->d_counters64 + 3, 0, sizeof(unsigned long long), s));
    if (loss) CK(cudaMemsetAsync(loss, 0, sizeof(double), s));
    { STAGE(ST_BWD); CK(launch_render_bwd_l1(ctx->L, rgb, target, scale, T_final, n_contrib, loss, s)); }  // S7 + ℓ1
    ctx->state = 3;
    return MVGS_OK;
}

mvgs_status mvgs_render_fwd_partial(mvgs_ctx* ctx, const int32_t* pix, int32_t S, int32_t mode, float* rgb,
                                    float* T_final, int32_t* n_contrib, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state < 1) return fail(ctx, MVGS_ERR_STATE, "render_fwd_partial before preprocess");
    if (!pix || !rgb || !T_final || !n_contrib || S < 1 || S > 256 ||
        (mode != MVGS_PARTIAL_THREAD_EFFICIENT && mode != MVGS_PARTIAL_MASKED))
        return fail(ctx, MVGS_ERR_INVALID, "partial: null pointer, S outside [1, 256] or unknown mode");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    ctx->last_stream = s;
    CK(cudaMemsetAsync(ctx->d_counters64 + 5, 0, 4 * sizeof(unsigned long long), s));  // occupancy counters
    { STAGE(ST_FWD); CK(launch_render_fwd_partial(ctx->L, pix, S, mode, rgb, T_final, n_contrib, s)); }
    ctx->state = 4;  // partial forward: its [V,T,S] outputs are only valid for the matching partial backward
    ctx->partial_S = S;
    ctx->partial_mode = mode;
    return MVGS_OK;
}

mvgs_status mvgs_render_bwd_partial(mvgs_ctx* ctx, const int32_t* pix, int32_t S, int32_t mode, const float* dL_drgb,
                                    const float* T_final, const int32_t* n_contrib, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state != 4 || ctx->partial_S != S || ctx->partial_mode != mode)
        return fail(ctx, MVGS_ERR_STATE, "render_bwd_partial needs a render_fwd_partial (same S and mode) of a fresh preprocess");
    if (!pix || !dL_drgb || !T_final || !n_contrib || S < 1 || S > 256 ||
        (mode != MVGS_PARTIAL_THREAD_EFFICIENT && mode != MVGS_PARTIAL_MASKED))
        return fail(ctx, MVGS_ERR_INVALID, "partial: null pointer, S outside [1, 256] or unknown mode");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    ctx->last_stream = s;
    { STAGE(ST_BWD); CK(launch_render_bwd_partial(ctx->L, pix, S, mode, dL_drgb, T_final, n_contrib, s)); }
    ctx->state = 3;
    return MVGS_OK;
}

mvgs_status mvgs_adc_stats_range(mvgs_ctx* ctx, int64_t g_begin, int64_t g_end, const mvgs_grads* grads,
                                 const mvgs_adc* adc, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state != 3) return fail(ctx, MVGS_ERR_STATE, "adc_stats needs a preceding render_bwd");
    if (!grads || !adc) return fail(ctx, MVGS_ERR_INVALID, "null grads/adc");
    if (g_begin < 0 || g_end < g_begin || g_end > ctx->L.P || (g_begin % BLK) != 0)
        return fail(ctx, MVGS_ERR_INVALID, "adc_stats_range: need 0 <= g_begin <= g_end <= P, g_begin % 256 == 0");
    if (g_end > g_begin && (!grads->d_means || !grads->d_log_scales || !grads->d_quats || !grads->d_opacity_logits ||
                            !grads->d_sh || !adc->e1 || !adc->e2 || !adc->vis))
        return fail(ctx, MVGS_ERR_INVALID, "null output pointer");
    CK(cudaSetDevice(ctx->device));
    ctx->last_stream = (cudaStream_t)stream;
    cudaStream_t s = (cudaStream_t)stream;
    if (g_end > g_begin) { STAGE(ST_GAUSS); CK(launch_gauss_bwd(ctx->L, *grads, *adc, g_begin, g_end, s)); }  // S8 + S9
    return MVGS_OK;
}

mvgs_status mvgs_adc_stats(mvgs_ctx* ctx, const mvgs_grads* grads, const mvgs_adc* adc, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    return mvgs_adc_stats_range(ctx, 0, ctx->L.P, grads, adc, stream);
}

mvgs_status mvgs_query(mvgs_ctx* ctx, mvgs_stats* out) {
    if (!ctx || !out) return MVGS_ERR_INVALID;
    CK(cudaSetDevice(ctx->device));
    int h[C_NCOUNTERS];
    unsigned long long h64[9];
    // ordered on the stream of the last enqueuing call; waits for that stream only, not the device
    CK(cudaMemcpyAsync(h, ctx->d_counters, sizeof(h), cudaMemcpyDeviceToHost, ctx->last_stream));
    CK(cudaMemcpyAsync(h64, ctx->d_counters64, sizeof(h64), cudaMemcpyDeviceToHost, ctx->last_stream));
    CK(cudaStreamSynchronize(ctx->last_stream));
    memset(out, 0, sizeof(*out));
    out->Q = h[C_Q];
    out->K = std::max((int64_t)h[C_K], (int64_t)h64[4]);  // entries needed, even past a pair overflow
    out->cap_pairs = ctx->cap_pairs;
    out->cap_entries = ctx->cap_entries;
    out->max_bucket = h[C_MAXB];
    out->n_visible = h[C_NVIS];
    out->V = ctx->L.V;
    out->tiles_x = ctx->L.TX;
    out->tiles_y = ctx->L.TY;
    out->eval_fwd = (int64_t)h64[0];
    out->eval_bwd = (int64_t)h64[1];
    out->exp_fwd = (int64_t)h64[2];
    out->exp_bwd = (int64_t)h64[3];
    out->threads_launched = (int64_t)h64[5];
    out->threads_active = (int64_t)h64[6];
    out->lane_steps_launched = (int64_t)h64[7];
    out->lane_steps_active = (int64_t)h64[8];
    out->overflow = h[C_OVERFLOW] || out->Q > ctx->cap_pairs || out->K > ctx->cap_entries;
    if (out->overflow) return fail(ctx, MVGS_ERR_CAPACITY, "capacity exceeded: reserve stats.Q / stats.K and re-run");
    return MVGS_OK;
}

mvgs_status mvgs_export_lists(mvgs_ctx* ctx, int64_t* range_start, int32_t* entry_gid, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state < 1) return fail(ctx, MVGS_ERR_STATE, "export before preprocess");
    CK(launch_export(ctx->L, range_start, entry_gid, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream));
    return MVGS_OK;
}

mvgs_status mvgs_export_pairs(mvgs_ctx* ctx, int32_t* pair_ids, int32_t* pair_i, float* pair_f, float* pair_g,
                              void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state < 1) return fail(ctx, MVGS_ERR_STATE, "export before preprocess");
    CK(launch_export(ctx->L, nullptr, nullptr, pair_ids, pair_i, pair_f, pair_g, (cudaStream_t)stream));
    return MVGS_OK;
}

mvgs_status mvgs_set_debug_blend_counts(mvgs_ctx* ctx, int32_t* nblend) {
    if (!ctx) return MVGS_ERR_INVALID;
    ctx->L.dbg_nblend = nblend;
    return MVGS_OK;
}

mvgs_status mvgs_set_tma(mvgs_ctx* ctx, int enable) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (enable && !ctx->rec_map_ok) return fail(ctx, MVGS_ERR_CUDA, "the driver refused the record tensor map");
    ctx->use_tma = enable != 0;
    return MVGS_OK;
}

mvgs_status mvgs_set_timing(mvgs_ctx* ctx, int enable) {
    if (!ctx) return MVGS_ERR_INVALID;
    ctx->timing = enable != 0;
    return MVGS_OK;
}

mvgs_status mvgs_set_eval_counting(mvgs_ctx* ctx, int enable) {
    if (!ctx) return MVGS_ERR_INVALID;
    ctx->count_evals = enable != 0;
    ctx->L.count_evals = enable != 0;
    return MVGS_OK;
}

mvgs_status mvgs_dssim3d(mvgs_ctx* ctx, const mvgs_camera* cams, int32_t V, int32_t H, int32_t W, const float* img,
                         const float* target, const float* depth, const float* T_final, float sigma_px, float* loss,
                         float* dL_dimg, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (!cams || !img || !target || !depth || !T_final || !loss)
        return fail(ctx, MVGS_ERR_INVALID, "dssim3d: null argument");
    if (V < 1 || V > 65535 || H < 1 || W < 1 || !(sigma_px > 0.f))
        return fail(ctx, MVGS_ERR_INVALID, "dssim3d: V, H, W must be positive and sigma_px > 0");
    for (int v = 0; v < V; v++)
        if (!(cams[v].fx > 0.f) || !(cams[v].fy > 0.f)) return fail(ctx, MVGS_ERR_INVALID, "dssim3d: fx, fy must be > 0");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t npx = (int64_t)V * H * W;
    const int64_t nblk = dssim_partials(V, H, W);
    if (npx * 12 > ctx->cap_dssim_coef || nblk > ctx->cap_dssim_part) {
        CK(cudaDeviceSynchronize());
        CK(grow(ctx->d_dssim_coef, ctx->cap_dssim_coef, npx * 12));
        CK(grow(ctx->d_dssim_part, ctx->cap_dssim_part, nblk));
    }
    { STAGE(ST_DSSIM); CK(launch_dssim3d(cams, V, H, W, img, target, depth, T_final, sigma_px, loss, dL_dimg,
                                         ctx->d_dssim_coef, ctx->d_dssim_part, s)); }
    return MVGS_OK;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

mvgs_status mvgs_adc_step(mvgs_ctx* ctx, const mvgs_gaussians* g, const mvgs_adc_accum* acc, const float* noise,
                          const mvgs_adc_config* cfg, const mvgs_gaussians_out* out, int32_t* origin, uint8_t* kind,
                          mvgs_adc_report* report, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (!g || !acc || !cfg || !out || !origin || !kind || !report)
        return fail(ctx, MVGS_ERR_INVALID, "adc_step: null argument");
    if (g->P < 0 || g->P >= (int64_t)INT32_MAX / 10) return fail(ctx, MVGS_ERR_INVALID, "adc_step: P out of range");
    if (g->P > 0 && (!g->means || !g->log_scales || !g->quats || !g->opacity_logits || !g->sh || !noise ||
                     !acc->denom_acc || (cfg->metric_mode == 1 && (!acc->e1_acc || !acc->e2_acc)) ||
                     (cfg->metric_mode == 0 && !acc->e_old_acc)))
        return fail(ctx, MVGS_ERR_INVALID, "adc_step: null input array");
    if (!out->means || !out->log_scales || !out->quats || !out->opacity_logits || !out->sh || out->capacity < 0)
        return fail(ctx, MVGS_ERR_INVALID, "adc_step: null output array");
    if (out->sh_stride != g->sh_stride || g->sh_stride < 1)
        return fail(ctx, MVGS_ERR_INVALID, "adc_step: sh_stride mismatch");
    if (!aligned16(g->quats) || !aligned16(out->quats) || !aligned16(g->sh) || !aligned16(out->sh))
        return fail(ctx, MVGS_ERR_INVALID, "adc_step: quats / sh not 16-B aligned");
    if (cfg->split_count < 2 || cfg->split_count > 8 || !(cfg->size_threshold > 0.f) || !(cfg->split_factor > 0.f) ||
        !(cfg->prune_opacity > 0.f && cfg->prune_opacity < 1.f) || cfg->batch_views < 1 ||
        (cfg->metric_mode != 0 && cfg->metric_mode != 1))
        return fail(ctx, MVGS_ERR_INVALID, "adc_step: config out of range");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t P = g->P;
    // host thresholds: fp64 math rounded once to fp32 (the oracle rounds identically)
    mvgs::AdcParamsHost h{};
    h.tau_split = cfg->grad_threshold_split;
    h.tau_clone = cfg->grad_threshold_clone;
    h.ln_size = (float)std::log((double)cfg->size_threshold);
    h.ln_split = (float)std::log((double)cfg->split_factor);
    const double p = (double)cfg->prune_opacity * cfg->batch_views;
    h.logit_prune = p >= 1.0 ? INFINITY : (float)std::log(p / (1.0 - p));
    h.ln_prune_scale = cfg->prune_scale_max > 0.f ? (float)std::log((double)cfg->prune_scale_max) : INFINITY;
    h.N = cfg->split_count;
    h.mode = cfg->metric_mode;
    const int64_t ntmp = scan_tmp_size((int)std::max<int64_t>(P, 1));
    if (P + 1 > ctx->cap_adc_cnt || P > ctx->cap_adc_flags || ntmp > ctx->cap_adc_tmp || !ctx->d_adc_rep) {
        CK(cudaDeviceSynchronize());
        CK(grow(ctx->d_adc_cnt, ctx->cap_adc_cnt, P + 1));  // scan writes the total at [P]
        CK(grow(ctx->d_adc_flags, ctx->cap_adc_flags, std::max<int64_t>(P, 1)));
        CK(grow(ctx->d_adc_tmp, ctx->cap_adc_tmp, ntmp));
        if (!ctx->d_adc_rep) {
            CK(cudaMalloc(&ctx->d_adc_rep, 4 * sizeof(unsigned long long)));
            CK(cudaMallocHost(&ctx->h_adc_rep, 4 * sizeof(long long)));
        }
    }
    CK(cudaMemsetAsync(ctx->d_adc_rep, 0, 4 * sizeof(unsigned long long), s));
    CK(launch_adc_decide(*g, *acc, h, ctx->d_adc_cnt, ctx->d_adc_flags, ctx->d_adc_rep, s));
    if (P > 0) CK(scan_exclusive(ctx->d_adc_cnt, (int)P, (int*)(ctx->d_adc_rep + 3), ctx->d_adc_tmp, s));
    CK(cudaMemcpyAsync(ctx->h_adc_rep, ctx->d_adc_rep, 4 * sizeof(long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    report->n_split = ctx->h_adc_rep[0];
    report->n_clone = ctx->h_adc_rep[1];
    report->n_pruned = ctx->h_adc_rep[2];
    report->P_new = P > 0 ? (int64_t)(int)(ctx->h_adc_rep[3] & 0xffffffffLL) : 0;
    if (report->P_new > out->capacity) {
        char msg[128];
        snprintf(msg, sizeof msg, "adc_step: %lld rows needed, capacity %lld", (long long)report->P_new,
                 (long long)out->capacity);
        return fail(ctx, MVGS_ERR_CAPACITY, msg);
    }
    CK(launch_adc_emit(*g, ctx->d_adc_flags, ctx->d_adc_cnt, noise, h, *out, origin, kind, s));
    return MVGS_OK;
}

mvgs_status mvgs_adc_remap(mvgs_ctx* ctx, const float* src, float* dst, int64_t width, const int32_t* origin,
                           const uint8_t* kind, int64_t P_new, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (width < 1 || P_new < 0 || (P_new > 0 && (!src || !dst || !origin || !kind)) || (P_new > 0 && src == dst))
        return fail(ctx, MVGS_ERR_INVALID, "adc_remap: bad arguments");
    CK(cudaSetDevice(ctx->device));
    CK(launch_adc_remap(src, dst, width, origin, kind, P_new, (cudaStream_t)stream));
    return MVGS_OK;
}

mvgs_status mvgs_loss_grad(mvgs_ctx* ctx, const float* rgb, const float* target, int64_t n, int32_t mode, float scale,
                           float* dL_drgb, double* loss, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (n < 0 || (n > 0 && (!rgb || !target || !dL_drgb)) || (mode != 0 && mode != 1))
        return fail(ctx, MVGS_ERR_INVALID, "loss_grad: bad arguments");
    CK(cudaSetDevice(ctx->device));
    CK(launch_loss_grad(rgb, target, n, mode, scale, dL_drgb, loss, ctx->d_lab_part, (cudaStream_t)stream));
    return MVGS_OK;
}

mvgs_status mvgs_loss_grad_u8(mvgs_ctx* ctx, const float* rgb, const uint8_t* target, int64_t n, int32_t mode,
                              float scale, float* dL_drgb, double* loss, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (n < 0 || (n > 0 && (!rgb || !target || !dL_drgb)) || (mode != 0 && mode != 1))
        return fail(ctx, MVGS_ERR_INVALID, "loss_grad_u8: bad arguments");
    CK(cudaSetDevice(ctx->device));
    CK(launch_loss_grad_u8(rgb, target, n, mode, scale, dL_drgb, loss, ctx->d_lab_part, (cudaStream_t)stream));
    return MVGS_OK;
}

mvgs_status mvgs_grad_moments(mvgs_ctx* ctx, const float* g, int64_t n, double* sum, double* sumsq, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (n < 0 || !sumsq || (n > 0 && (!g || !sum))) return fail(ctx, MVGS_ERR_INVALID, "grad_moments: bad arguments");
    CK(cudaSetDevice(ctx->device));
    CK(launch_moments(g, n, sum, sumsq, ctx->d_lab_part, (cudaStream_t)stream));
    return MVGS_OK;
}

mvgs_status mvgs_grad_variance(mvgs_ctx* ctx, const double* sum, int64_t n, const double* sumsq, int64_t K,
                               double* variance, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (n < 0 || K < 1 || !sumsq || !variance || (n > 0 && !sum) || variance == sumsq)
        return fail(ctx, MVGS_ERR_INVALID, "grad_variance: bad arguments");
    CK(cudaSetDevice(ctx->device));
    CK(launch_variance(sum, n, sumsq, K, variance, ctx->d_lab_part, (cudaStream_t)stream));
    return MVGS_OK;
}

// ---------------------------------------------------------------- owner-sharded exchange (§11)
mvgs_status mvgs_owner_slices(mvgs_ctx* ctx, const int64_t* g_bounds, int32_t N, int64_t* slot_off, float** slots,
                              void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state != 3) return fail(ctx, MVGS_ERR_STATE, "owner_slices needs a preceding render_bwd");
    if (!g_bounds || !slot_off || !slots || N < 1) return fail(ctx, MVGS_ERR_INVALID, "owner_slices: bad arguments");
    const Launch& L = ctx->L;
    if (g_bounds[0] != 0 || g_bounds[N] != L.P) return fail(ctx, MVGS_ERR_INVALID, "owner_slices: bounds must span [0, P]");
    for (int o = 0; o < N; o++)
        if (g_bounds[o + 1] < g_bounds[o] || ((g_bounds[o] % BLK) != 0 && g_bounds[o] != L.P))
            return fail(ctx, MVGS_ERR_INVALID, "owner_slices: bounds ascending, multiples of 256");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = (int64_t)L.V * L.NB + 1;
    ctx->h_blk.resize((size_t)n);
    CK(cudaMemcpyAsync(ctx->h_blk.data(), ctx->d_blk, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int v = 0; v < L.V; v++)
        for (int o = 0; o <= N; o++) {
            const int64_t b = (g_bounds[o] + BLK - 1) / BLK;  // first block of owner o (NB for the end)
            slot_off[(int64_t)v * (N + 1) + o] =
                b >= L.NB ? ctx->h_blk[(size_t)(v + 1) * L.NB] : ctx->h_blk[(size_t)v * L.NB + b];
        }
    *slots = ctx->d_pgrad;
    return MVGS_OK;
}

mvgs_status mvgs_owner_prepare(mvgs_ctx* ctx, const mvgs_camera* cams_all, int32_t V_all, int64_t g_begin,
                               int64_t g_end, int64_t* view_off, float** recv, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (ctx->state < 1) return fail(ctx, MVGS_ERR_STATE, "owner_prepare needs a preprocess (the Gaussians)");
    if (!cams_all || !view_off || !recv || V_all < 1 || V_all > 65535)
        return fail(ctx, MVGS_ERR_INVALID, "owner_prepare: bad arguments");
    const Launch& L = ctx->L;
    if (g_begin < 0 || g_end < g_begin || g_end > L.P || ((g_begin % BLK) != 0 && g_begin != g_end))
        return fail(ctx, MVGS_ERR_INVALID, "owner_prepare: need 0 <= g_begin <= g_end <= P, g_begin % 256 == 0");
    for (int v = 0; v < V_all; v++)
        if (cams_all[v].width != L.W || cams_all[v].height != L.H || !(cams_all[v].znear > 0.f) ||
            !(cams_all[v].fx > 0.f) || !(cams_all[v].fy > 0.f))
            return fail(ctx, MVGS_ERR_INVALID, "owner_prepare: cameras must match the batch size, znear, fx, fy > 0");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nblk = (int64_t)V_all * L.NB;
    if (nblk + 1 > INT32_MAX) return fail(ctx, MVGS_ERR_INVALID, "owner_prepare: batch too large");
    const int64_t need_scan = scan_tmp_size((int)std::max<int64_t>(nblk, 1));
    if (nblk + 1 > ctx->cap_oblk || need_scan > ctx->cap_oscan || V_all > ctx->cap_ocams ||
        (V_all <= 32 && L.P > ctx->cap_opmask)) {
        CK(cudaStreamSynchronize(s));
        CK(grow(ctx->d_oblk, ctx->cap_oblk, nblk + 1));
        CK(grow(ctx->d_oscan, ctx->cap_oscan, need_scan));
        CK(grow(ctx->d_ocams, ctx->cap_ocams, (int64_t)V_all));
        if (V_all <= 32) CK(grow(ctx->d_opmask, ctx->cap_opmask, std::max<int64_t>(L.P, 1)));
    }
    CK(launch_set_cams(cams_all, V_all, ctx->d_ocams, s));
    Launch& Lo = ctx->Lo;
    Lo = L;
    Lo.V = V_all;
    Lo.cams = ctx->d_ocams;
    Lo.blk_off = ctx->d_oblk;
    Lo.pmask = V_all <= 32 ? ctx->d_opmask : nullptr;
    CK(cudaMemsetAsync(ctx->d_oblk, 0, sizeof(int) * (nblk + 1), s));
    const int b0 = (int)(g_begin / BLK), b1 = (int)((g_end + BLK - 1) / BLK);
    CK(launch_count_range(Lo, b0, b1, s));                                   // S1 for the owned blocks, all views
    CK(scan_exclusive(ctx->d_oblk, (int)nblk, nullptr, ctx->d_oscan, s));  // view-major slot layout
    ctx->h_blk.resize((size_t)nblk + 1);
    CK(cudaMemcpyAsync(ctx->h_blk.data(), ctx->d_oblk, sizeof(int) * (nblk + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int v = 0; v < V_all; v++) view_off[v] = ctx->h_blk[(size_t)v * L.NB];
    view_off[V_all] = ctx->h_blk[(size_t)nblk];
    const int64_t q = view_off[V_all];
    if (q > ctx->cap_orecv || !ctx->d_orecv) {
        cudaFree(ctx->d_orecv);
        ctx->d_orecv = nullptr;
        ctx->cap_orecv = 0;
        const int64_t nq = q + q / 4 + 1024;
        CK(cudaMalloc(&ctx->d_orecv, sizeof(float) * PG_STRIDE * nq));
        ctx->cap_orecv = nq;
    }
    Lo.pgrad = ctx->d_orecv;
    Lo.cap_pairs = ctx->cap_orecv;
    ctx->og_begin = g_begin;
    ctx->og_end = g_end;
    ctx->owner_ready = true;
    *recv = ctx->d_orecv;
    return MVGS_OK;
}

mvgs_status mvgs_owner_adc_stats(mvgs_ctx* ctx, const mvgs_grads* grads, const mvgs_adc* adc, void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (!ctx->owner_ready) return fail(ctx, MVGS_ERR_STATE, "owner_adc_stats needs mvgs_owner_prepare");
    if (!grads || !adc) return fail(ctx, MVGS_ERR_INVALID, "null grads/adc");
    const int64_t gb = ctx->og_begin, ge = ctx->og_end;
    if (ge > gb && (!grads->d_means || !grads->d_log_scales || !grads->d_quats || !grads->d_opacity_logits ||
                    !grads->d_sh || !adc->e1 || !adc->e2 || !adc->vis))
        return fail(ctx, MVGS_ERR_INVALID, "null output pointer");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = (cudaStream_t)stream;
    ctx->last_stream = s;
    if (ge > gb) { STAGE(ST_GAUSS); CK(launch_gauss_bwd(ctx->Lo, *grads, *adc, gb, ge, s)); }  // S8 + S9, all views
    return MVGS_OK;
}

mvgs_status mvgs_e_old_from_gsum(mvgs_ctx* ctx, const float* gsum, int64_t n, float* e_old, float* e_old_acc,
                                 void* stream) {
    if (!ctx) return MVGS_ERR_INVALID;
    if (n < 0 || (n > 0 && (!gsum || (!e_old && !e_old_acc)))) return fail(ctx, MVGS_ERR_INVALID, "e_old_from_gsum: bad arguments");
    if (((uintptr_t)gsum & 7) != 0) return fail(ctx, MVGS_ERR_INVALID, "e_old_from_gsum: gsum not 8-B aligned");
    CK(cudaSetDevice(ctx->device));
    CK(launch_e_old(gsum, n, e_old, e_old_acc, (cudaStream_t)stream));
    return MVGS_OK;
}

int mvgs_stage_times(mvgs_ctx* ctx, float* ms, int n) {
    if (!ctx || !ms) return 0;
    int k = 0;
    for (; k < n && k < MVGS_NUM_STAGES; k++) {
        double sum = 0.0;
        int cnt = 0;
        for (auto& p : ctx->ev_rec[k]) {
            float t = 0.f;
            if (cudaEventSynchronize(p.second) == cudaSuccess && cudaEventElapsedTime(&t, p.first, p.second) == cudaSuccess) {
                sum += t;
                cnt++;
            }
            ctx->ev_pool.push_back(p.first);
            ctx->ev_pool.push_back(p.second);
        }
        ctx->ev_rec[k].clear();
        ms[k] = cnt ? (float)(sum / cnt) : 0.f;
    }
    return k;
}

}  // extern "C"
