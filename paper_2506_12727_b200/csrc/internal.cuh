// internal.cuh — context layout and kernel launchers shared by the .cu files
// of libmvgs.so (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>
#include "../../include/mvgs.h"

namespace mvgs {

constexpr int BLK = 256;          // Gaussians per preprocessing block (pair-slot granularity)
constexpr int NG = 10;            // per-pair gradient record: Σ∇x Σ∇y e1 ∂A ∂B ∂C ∂o ∂r ∂g ∂b
constexpr int PG_STRIDE = 12;     // floats per pair-gradient slot (48 B, 16-B aligned)
constexpr int REC_F4 = 3;         // float4 per pair render record (48 B)
constexpr int PG_FLAGS = 10;      // float of a gradient slot that carries the pair's flags word
constexpr uint32_t PF_VISIBLE = 32u;
constexpr int PF_RADIUS_SHIFT = 8;  // pflag bits 8..31: the pair's CA radius (R7), saturated at 2^24 − 1

// device counters (int32 slots in ctx->d_counters)
enum { C_Q = 0, C_K = 1, C_OVERFLOW = 2, C_MAXB = 3, C_NVIS = 4, C_NCOUNTERS = 8 };


struct Launch {  // everything a kernel needs about the current batch
    int64_t P;
    int V, W, H, TX, TY, T, NB;
    int sh_degree, sh_stride;
    int count_evals;  // compositing kernels count (pixel, entry) evaluations (statistics)
    uint32_t* pmask;  // [P] participation bits per view (V ≤ 32; written by k_count), else null
    float bg[3];
    const mvgs_camera* cams;  // device [V]
    const float *means, *log_scales, *quats, *opac, *sh;
    int64_t cap_pairs, cap_entries;
    // workspace
    int* blk_off;     // [V*NB + 1]  exclusive scan of per-(view, block) participation counts
    int* bucket_off;  // [V*T + 1]   exclusive scan of per-(view, tile) entry counts
    const int* order; // [V*T] compositing CTA i renders bucket order[i] (longest list first), or null
    float4* rec;      // [cap_pairs * 3]
    uint32_t* pflag;  // [cap_pairs] bit0-2 rgb clamped, bit3-4 Jacobian clamps, bit5 tiles > 0, bits 8..31 radius
    float* pgrad;     // [cap_pairs * PG_STRIDE]
    uint32_t *key, *val, *key2, *val2;  // [cap_entries] entry (bucket key, pair) ping-pong
    uint32_t *pkey, *pval, *pkey2, *pval2;  // [cap_pairs] pair (depth key, pair) ping-pong
    uint2 *prect, *prect2;                  // [cap_pairs] packed tile rect carried through the pair sort
    int* ecount;      // [cap_pairs + 1] tiles per depth-ordered pair → entry offsets
    int* rs_counts;   // (unused) radix digit × tile counts
    int* scan_tmp;    // scan block sums
    const uint32_t* sorted;  // [K] pair index of every entry in (view, tile, depth, gid) order
    int* counters;    // [C_NCOUNTERS]
    unsigned long long* counters64;  // [16]: fwd/bwd evaluations, fwd/bwd exps, entries needed, partial-render occupancy (5–8)
    int32_t* dbg_nblend;  // parity export: per-pixel blended-entry count taken by the backward (or null)
};

#ifdef __CUDACC__
// Every forward launch clears the per-pair gradient slots [0, Q) that the following
// backward accumulates into (red.add).  The forward kernels are compute-bound with
// little DRAM traffic, so these fire-and-forget stores ride along instead of costing
// the HBM-bound projection 48 B per pair; each CTA clears one grid-strided slice.
// The slot's 11th float (PG_FLAGS) carries the pair's flags word (pflag), so a gradient slot is
// a self-contained 48-byte record: the per-Gaussian kernel needs no second load, and an owner
// rank can receive slots from other ranks and run the chain on them.
__device__ __forceinline__ void zero_pgrad_slice(const Launch& L) {
    static_assert(PG_STRIDE == 12 && PG_FLAGS == 10, "slot = 3 float4, flags in the third one's z");
    const int Q = (int)min((int64_t)L.counters[C_Q], L.cap_pairs);
    float4* p4 = reinterpret_cast<float4*>(L.pgrad);
    const int stride = gridDim.x * blockDim.x;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Q; q += stride) {  // one pair slot per step
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        p4[3 * (int64_t)q] = z;
        p4[3 * (int64_t)q + 1] = z;
        p4[3 * (int64_t)q + 2] = make_float4(0.f, 0.f, __uint_as_float(L.pflag[q]), 0.f);
    }
}
#endif

}  // namespace mvgs

struct mvgs_ctx {
    int device = 0;
    int64_t cap_pairs = 0, cap_entries = 0;
    int64_t cap_blk = 0, cap_buckets = 0, cap_cams = 0, cap_scan = 0;
    CUtensorMap rec_map{};  // TMA view of d_rec (tma.cuh), re-encoded when the pair capacity changes
    bool rec_map_ok = false;
    bool use_tma = false;   // forward staging by TMA gather4 (mvgs_set_tma / MVGS_TMA=1); measured slower, off
    int state = 0;  // 0 none, 1 preprocessed, 2 forward done, 3 backward done, 4 partial forward done
    int partial_S = 0, partial_mode = -1;  // the partial forward's sample size and launch shape
    mvgs::Launch L{};
    mvgs_gaussians g{};
    // device buffers
    mvgs_camera* d_cams = nullptr;
    int* d_blk = nullptr;
    int* d_bucket = nullptr;
    int* d_order = nullptr;  // [V*T] longest-list-first CTA order of the compositing kernels
    bool use_lpt = false;    // MVGS_LPT=1: longest-list-first CTA order (measured: no gain at garden / large, −1 % playroom)
    float4* d_rec = nullptr;
    uint32_t* d_pflag = nullptr;
    float* d_pgrad = nullptr;
    uint32_t *d_key = nullptr, *d_val = nullptr, *d_key2 = nullptr, *d_val2 = nullptr;
    uint32_t *d_pkey = nullptr, *d_pval = nullptr, *d_pkey2 = nullptr, *d_pval2 = nullptr;
    uint2 *d_prect = nullptr, *d_prect2 = nullptr;
    int* d_ecount = nullptr;
    int* d_rs = nullptr;
    int64_t cap_rs = 0;
    int* d_counters = nullptr;
    unsigned long long* d_counters64 = nullptr;
    int* d_scan = nullptr;  // scan block sums
    float* d_dssim_coef = nullptr;   // [V,H,W,12] NEXT-2 backward coefficients
    int64_t cap_dssim_coef = 0;
    double* d_dssim_part = nullptr;  // per-block SSIM sums
    int64_t cap_dssim_part = 0;
    uint32_t* d_pmask = nullptr;            // [P] participation bits (V ≤ 32)
    int64_t cap_pmask = 0;
    double* d_lab_part = nullptr;           // NEXT-4 per-CTA fp64 partials
    int* d_adc_cnt = nullptr;        // NEXT-3 per-Gaussian emitted-row counts → offsets
    int64_t cap_adc_cnt = 0;
    uint8_t* d_adc_flags = nullptr;
    int64_t cap_adc_flags = 0;
    int* d_adc_tmp = nullptr;        // scan block sums
    int64_t cap_adc_tmp = 0;
    unsigned long long* d_adc_rep = nullptr;  // [4] split, clone, pruned, total
    long long* h_adc_rep = nullptr;           // pinned mirror
    // owner-sharded exchange: the layout of ALL views' pair slots of the
    // Gaussians [og_begin, og_end) this rank owns, and the slots received from the other ranks
    mvgs::Launch Lo{};
    mvgs_camera* d_ocams = nullptr;
    int64_t cap_ocams = 0;
    int* d_oblk = nullptr;          // [V_all * NB + 1] scanned participation counts (owner blocks only)
    int64_t cap_oblk = 0;
    int* d_oscan = nullptr;         // scan scratch
    int64_t cap_oscan = 0;
    uint32_t* d_opmask = nullptr;   // [P] participation bits of the owned Gaussians in all views (V_all ≤ 32)
    int64_t cap_opmask = 0;
    float* d_orecv = nullptr;       // [Q_own * PG_STRIDE] gradient slots of the owned Gaussians, all views
    int64_t cap_orecv = 0;          // in slots
    int64_t og_begin = 0, og_end = 0;
    bool owner_ready = false;
    std::vector<int> h_blk;         // host copy of blk_off (slice offsets)
    cudaStream_t last_stream = nullptr;
    bool timing = false;
    bool count_evals = true;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_rec[MVGS_NUM_STAGES];  // recorded since last read
    std::vector<cudaEvent_t> ev_pool;
    std::string err;
};

namespace mvgs {
// launchers (return cudaGetLastError())
cudaError_t scan_exclusive(int* a, int n, int* total_slot, int* tmp, cudaStream_t s, const int* n_live = nullptr);
cudaError_t launch_count(const Launch& L, cudaStream_t s);
cudaError_t launch_count_range(const Launch& L, int b0, int b1, cudaStream_t s);
cudaError_t launch_e_old(const float* gsum, int64_t n, float* e_old, float* e_old_acc, cudaStream_t s);
cudaError_t launch_project(const Launch& L, cudaStream_t s);
cudaError_t launch_sort_pairs(const Launch& L, const uint32_t** order_out, const uint2** rect_out, cudaStream_t s);
cudaError_t launch_dup_sort(const Launch& L, const uint32_t* order, const uint2* rect, cudaStream_t s);
cudaError_t launch_sort_entries(const Launch& L, uint32_t** sorted_vals, cudaStream_t s);
cudaError_t launch_lpt_order(const Launch& L, int* order, cudaStream_t s);
int64_t radix_counts_size(int64_t cap);
int radix_tiles(int64_t cap);
cudaError_t launch_render_fwd(const Launch& L, float* rgb, float* Tf, int32_t* nc, float* depth, const CUtensorMap* tm,
                              cudaStream_t s);
int64_t dssim_partials(int V, int H, int W);
struct AdcParamsHost {
    float tau_split, tau_clone, ln_size, ln_split, logit_prune, ln_prune_scale;
    int N, mode;
};
cudaError_t launch_adc_decide(const mvgs_gaussians& g, const mvgs_adc_accum& acc, const AdcParamsHost& h, int* cnt,
                              uint8_t* flags, unsigned long long* rep, cudaStream_t s);
cudaError_t launch_adc_emit(const mvgs_gaussians& g, const uint8_t* flags, const int* offs, const float* noise,
                            const AdcParamsHost& h, const mvgs_gaussians_out& out, int32_t* origin, uint8_t* kind,
                            cudaStream_t s);
cudaError_t launch_adc_remap(const float* src, float* dst, int64_t width, const int32_t* origin, const uint8_t* kind,
                             int64_t P_new, cudaStream_t s);
cudaError_t launch_dssim3d(const mvgs_camera* h_cams, int V, int H, int W, const float* img, const float* tgt,
                           const float* depth, const float* Tf, float sigma_px, float* loss, float* grad, float* coef,
                           double* partial, cudaStream_t s);
int lab_partials();
cudaError_t launch_loss_grad(const float* rgb, const float* tgt, int64_t n, int mode, float scale, float* dL,
                             double* loss, double* part, cudaStream_t s);
cudaError_t launch_loss_grad_u8(const float* rgb, const uint8_t* tgt, int64_t n, int mode, float scale, float* dL,
                                double* loss, double* part, cudaStream_t s);
cudaError_t launch_moments(const float* g, int64_t n, double* sum, double* sumsq, double* part, cudaStream_t s);
cudaError_t launch_variance(const double* sum, int64_t n, const double* sumsq, int64_t K, double* out, double* part,
                            cudaStream_t s);
cudaError_t launch_render_bwd(const Launch& L, const float* dL, const float* Tf, const int32_t* nc, cudaStream_t s);
cudaError_t launch_render_bwd_l1(const Launch& L, const float* rgb, const uint8_t* tgt, float scale, const float* Tf,
                                 const int32_t* nc, double* loss, cudaStream_t s);
cudaError_t launch_render_fwd_partial(const Launch& L, const int32_t* pix, int S, int mode, float* rgb, float* Tf,
                                      int32_t* nc, cudaStream_t s);
cudaError_t launch_render_bwd_partial(const Launch& L, const int32_t* pix, int S, int mode, const float* dL,
                                      const float* Tf, const int32_t* nc, cudaStream_t s);
cudaError_t launch_gauss_bwd(const Launch& L, const mvgs_grads& gr, const mvgs_adc& adc, int64_t gb, int64_t ge,
                             cudaStream_t s);
cudaError_t launch_export(const Launch& L, int64_t* range_start, int32_t* entry_gid, int32_t* pair_ids,
                          int32_t* pair_i, float* pair_f, float* pair_g, cudaStream_t s);
int scan_tmp_size(int n);
cudaError_t launch_set_cams(const mvgs_camera* h_cams, int V, mvgs_camera* d_cams, cudaStream_t s);
}  // namespace mvgs
