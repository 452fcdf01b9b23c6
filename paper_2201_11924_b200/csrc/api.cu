// api.cu -- the C ABI of libasd (include/asd.h): parameter validation, scratch
// ownership, launch sequencing of the sm_100a kernels, host<->device pipeline.
//
// Stage order per chunk of frames (PAPER.md P:289 stage list; rectification is
// the identity for a born-rectified rig and the median filter is off,
// DESIGN.md §3 readings c15/c16):
//   K1 census(L), census(R)                               census.cu
//   SGM aggregation, one launch per path direction         sgm_dir.cu   (design D1)
//   K4 WTA + uniqueness + sub-pixel, left and right view   post.cu
//   K5 LR check + depth (+ per-frame stats)                post.cu
// Every step runs in these kernels; the host only validates and enqueues.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "asd.h"
#include "common.cuh"
#include "kernels.h"

using namespace asd;

struct asd_ctx {
    asd_params prm;
    DevParams dp;
    int device = 0;
    int max_batch = 1;
    size_t sig_bytes = 4;
    // scratch (max_batch frame slots)
    void* census_l_base = nullptr;   // allocations (guard band before and after)
    void* census_r_base = nullptr;
    size_t cen_guard = 0;
    void* census_l = nullptr;
    void* census_r = nullptr;
    uint16_t* S = nullptr;
    uint16_t* cb = nullptr;       // SGBM block cost volume [B][H][W][D] u16 (D1, block > 1);
                                  // D3: [B][H][cs*w][D] in the sweeps' private layout
    uint16_t* cb2 = nullptr;      // D3 SGBM + R2: the right-referenced block cost
    uint16_t* SR = nullptr;       // right view's own aggregate [B][H][W][D] u16 (D1, lr_mode R2)
    bool wta2 = false;            // D1: WTA by the ring-window kernel (plan.nbuf / rsmem / wide)
    float* dl = nullptr;
    float* dr = nullptr;
    int16_t* dstar_l = nullptr;
    int16_t* dstar_r = nullptr;
    uint8_t* mask_l = nullptr;
    uint8_t* mask_r = nullptr;
    // design D3 scratch
    int engine = ASD_ENGINE_D1;
    V2Plan plan{};
    uint8_t* pa = nullptr;        // [B][H][W][D] u16 P_A | C << 8 (down sweep)
    uint16_t* pab = nullptr;      // [B][H][W][D] u16 partial (down + up)
    uint8_t* stash = nullptr;     // [B][H][W][D] u8 left->right path
    // R2 on D3 (reading c24): the right-referenced pass's own partials
    uint8_t* pa2 = nullptr;
    uint16_t* pab2 = nullptr;
    uint8_t* stash2 = nullptr;
    // host-path staging: two chunk buffers (inputs u8, outputs f32) + stats
    uint8_t* stage_in[2] = {nullptr, nullptr};     // [max_batch][2][H][W]
    float* stage_out[2] = {nullptr, nullptr};      // [max_batch][2][H][W]
    asd_frame_stats* stage_stats[2] = {nullptr, nullptr};
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr};
    cudaEvent_t ev_done[2] = {nullptr, nullptr};
    cudaEvent_t ev_comp[2] = {nullptr, nullptr};
    // D3 overlap: the cluster sweeps of group g+1 run on s_hi (high priority)
    // while the row pass and WTA of group g run on s_lo on the SMs the sweep
    // clusters leave free; fork from / join back to the caller's stream.
    cudaStream_t s_hi = nullptr, s_lo = nullptr, s_cen = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_sw = nullptr, ev_sw2 = nullptr, ev_hi = nullptr, ev_lo = nullptr, ev_cen = nullptr;
    int group = 0;                // frames per overlap group (D3)
    std::vector<cudaEvent_t> ev_free;   // one per scratch slot (max_batch / group)
    // live stage timing (asd_profile_begin/end)
    struct Mark { int stage; double bytes; double ops; };
    bool prof = false;
    std::vector<cudaEvent_t> prof_ev;   // 2 per launch
    std::vector<Mark> prof_marks;
    int prof_dropped = 0;
    char err[512] = {0};
};

static thread_local char g_err[512];

static void set_err(asd_ctx* c, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) snprintf(c->err, sizeof c->err, "%s", buf);
    snprintf(g_err, sizeof g_err, "%s", buf);
}

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

int validate(const asd_params* p, char* why, size_t n)
{
    if (!p) { snprintf(why, n, "params is NULL"); return ASD_E_INVALID_ARG; }
    if (p->census_w < 1 || p->census_h < 1 || !(p->census_w & 1) || !(p->census_h & 1)) {
        snprintf(why, n, "census_w/census_h must be odd and >= 1 (got %d x %d)", p->census_w, p->census_h);
        return ASD_E_INVALID_ARG;
    }
    if (p->census_w > 15 || p->census_h > 15) {
        snprintf(why, n, "census window %dx%d exceeds 15x15", p->census_w, p->census_h);
        return ASD_E_UNSUPPORTED;
    }
    const int nb = (p->census_w * p->census_h) / 2;
    if (nb < 1) { snprintf(why, n, "census window must have >= 1 pair"); return ASD_E_INVALID_ARG; }
    if (nb > 64) { snprintf(why, n, "census bits nb=%d > 64", nb); return ASD_E_UNSUPPORTED; }
    if (p->width < p->census_w || p->height < p->census_h) {
        snprintf(why, n, "image %dx%d smaller than census window", p->width, p->height);
        return ASD_E_INVALID_ARG;
    }
    if ((long long)p->width * p->height > (1ll << 26)) {
        snprintf(why, n, "image %dx%d too large", p->width, p->height);
        return ASD_E_UNSUPPORTED;
    }
    if (p->min_disp < 0) { snprintf(why, n, "min_disp must be >= 0"); return ASD_E_INVALID_ARG; }
    if (p->num_disp < 1) { snprintf(why, n, "num_disp must be >= 1"); return ASD_E_INVALID_ARG; }
    if (p->num_disp % 16 != 0 || p->num_disp < 16 || p->num_disp > 256) {
        snprintf(why, n, "num_disp=%d: need a multiple of 16 in [16, 256]", p->num_disp);
        return ASD_E_UNSUPPORTED;
    }
    if (p->min_disp > (1 << 20)) { snprintf(why, n, "min_disp too large"); return ASD_E_INVALID_ARG; }
    if (p->p1 < 0 || p->p2 < p->p1) {
        snprintf(why, n, "need 0 <= p1 <= p2 (got p1=%d p2=%d)", p->p1, p->p2);
        return ASD_E_INVALID_ARG;
    }
    const int bw = p->block_w == 0 ? 1 : p->block_w, bh = p->block_h == 0 ? 1 : p->block_h;
    if (bw < 1 || bh < 1 || !(bw & 1) || !(bh & 1) || bw > 15 || bh > 15) {
        snprintf(why, n, "block_w/block_h must be odd in [1, 15] (0 = 1); got %d x %d", p->block_w, p->block_h);
        return ASD_E_INVALID_ARG;
    }
    if (p->median_ksize != 0 && p->median_ksize != 3 && p->median_ksize != 5) {
        snprintf(why, n, "median_ksize must be 0, 3 or 5 (got %d)", p->median_ksize);
        return ASD_E_INVALID_ARG;
    }
    if (p->lr_mode != 0 && p->lr_mode != 1) {
        snprintf(why, n, "lr_mode must be 0 (R1) or 1 (R2) (got %d)", p->lr_mode);
        return ASD_E_INVALID_ARG;
    }
    if (bw * bh == 1 && nb + p->p2 > 255) {
        snprintf(why, n, "nb + p2 = %d > 255 (per-path cost must fit 8 bits)", nb + p->p2);
        return ASD_E_UNSUPPORTED;
    }
    if (bw * bh > 1 && (long long)(p->paths == 8 ? 8 : 4) * ((long long)bw * bh * nb + p->p2) > 65534) {
        snprintf(why, n, "paths * (block area * nb + p2) > 65534 (S must fit 16 bits, 0xFFFF is a sentinel)");
        return ASD_E_UNSUPPORTED;
    }
    if (p->paths != 4 && p->paths != 8) {
        snprintf(why, n, "paths must be 4 or 8 (got %d)", p->paths);
        return ASD_E_INVALID_ARG;
    }
    if (p->uniqueness > 100000) { snprintf(why, n, "uniqueness > 100000"); return ASD_E_INVALID_ARG; }
    if (std::isnan(p->lr_max_diff)) { snprintf(why, n, "lr_max_diff is NaN"); return ASD_E_INVALID_ARG; }
    if (p->subpixel != 0 && p->subpixel != 1) { snprintf(why, n, "subpixel must be 0/1"); return ASD_E_INVALID_ARG; }
    if (p->engine != ASD_ENGINE_AUTO && p->engine != ASD_ENGINE_D1 && p->engine != ASD_ENGINE_D3) {
        snprintf(why, n, "engine must be 0 (auto), 1 (D1) or 3 (D3)");
        return ASD_E_INVALID_ARG;
    }
    if (!(std::isfinite(p->focal_px) && p->focal_px > 0.0f) ||
        !(std::isfinite(p->baseline_m) && p->baseline_m > 0.0f)) {
        snprintf(why, n, "focal_px and baseline_m must be finite and > 0");
        return ASD_E_INVALID_ARG;
    }
    return ASD_OK;
}

DevParams make_dev(const asd_params* p)
{
    DevParams d{};
    d.W = p->width; d.H = p->height;
    d.min_disp = p->min_disp; d.D = p->num_disp;
    d.cw = p->census_w; d.ch = p->census_h;
    d.R = p->census_w / 2; d.Q = p->census_h / 2;
    d.nb = (p->census_w * p->census_h) / 2;
    d.p1 = p->p1; d.p2 = p->p2;
    d.paths = p->paths;
    d.uniq = p->uniqueness;
    d.lr = p->lr_max_diff;
    d.subpix = p->subpixel;
    d.fb = (float)((double)p->focal_px * (double)p->baseline_m);
    d.npx = (long long)p->width * p->height;
    d.ncell = d.npx * p->num_disp;
    d.bw = p->block_w == 0 ? 1 : p->block_w;
    d.bh = p->block_h == 0 ? 1 : p->block_h;
    d.median = p->median_ksize;
    d.lr_mode = p->lr_mode;
    return d;
}

struct Layout {
    size_t sig, s, sr, cb, pa, pab, r2, stash, px_f32, px_i16, px_u8, stage_in, stage_out, stats, total;
};

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

// pa_cols: columns of a P_A row (D3 pads it to the sweep grid, cs*w >= W).
// cbuf: D3 runs its u16-partial (BLK) instances (SGBM, or SGM beyond the u8
// partial range, V2Plan::blk), so a cost buffer in the sweeps' layout exists.
Layout layout(const DevParams& d, int max_batch, int engine, int pa_cols, bool cbuf = false)
{
    Layout L{};
    const size_t B = (size_t)max_batch;
    L.sig = align_up(B * d.npx * (d.nb <= 32 ? 4 : 8));
    L.s = engine == ASD_ENGINE_D1 ? align_up(B * d.ncell * 2) : 0;
    const bool blk = d.bw * d.bh > 1 || (engine == ASD_ENGINE_D3 && cbuf);
    L.cb = !blk ? 0 : engine == ASD_ENGINE_D1 ? align_up(B * d.ncell * 2)
                                              : align_up(B * d.H * pa_cols * d.D * 2);
    L.sr = (engine == ASD_ENGINE_D1 && d.lr_mode == 1) ? align_up(B * d.ncell * 2) : 0;
    L.pa = engine == ASD_ENGINE_D3 ? align_up(B * d.H * pa_cols * d.D * 2) : 0;   // P_A | C << 8, u16
    L.pab = engine == ASD_ENGINE_D3 ? align_up(B * d.ncell * 2) : 0;
    L.stash = engine == ASD_ENGINE_D3 ? align_up(B * d.ncell * (blk ? 2 : 1)) : 0;   // SGBM: u16
    L.r2 = (engine == ASD_ENGINE_D3 && d.lr_mode == 1) ? 1 : 0;   // doubles pa / pab / stash
    L.px_f32 = align_up(B * d.npx * 4);
    L.px_i16 = align_up(B * d.npx * 2);
    L.px_u8 = align_up(B * d.npx);
    L.stage_in = align_up(B * d.npx * 2);
    L.stage_out = align_up(B * d.npx * 2 * 4);
    L.stats = align_up(B * sizeof(asd_frame_stats));
    L.total = 2 * L.sig + L.s + L.sr + L.cb * (1 + (engine == ASD_ENGINE_D3 ? L.r2 : 0)) +
              (L.pa + L.pab + L.stash) * (1 + L.r2) + 2 * L.px_f32 + 2 * L.px_i16 + 2 * L.px_u8 +
              2 * (L.stage_in + L.stage_out + L.stats);
    return L;
}

// Direction table r = (rx, ry): the traversal step; 4-path = horizontal and
// vertical, 8-path adds the diagonals ("four-path"; reading c6).
const int kDirs[8][2] = {{+1, 0}, {-1, 0}, {0, +1}, {0, -1}, {+1, +1}, {-1, -1}, {+1, -1}, {-1, +1}};

FrameScratch frame_scratch(asd_ctx* c)
{
    FrameScratch fs;
    fs.census_l = c->census_l; fs.census_r = c->census_r; fs.S = c->S;
    fs.dl = c->dl; fs.dr = c->dr; fs.dstar_l = c->dstar_l; fs.dstar_r = c->dstar_r;
    fs.mask_l = c->mask_l; fs.mask_r = c->mask_r;
    return fs;
}

// Bracket one kernel launch with an event pair when profiling is on.
struct ProfScope {
    asd_ctx* c; cudaStream_t s; int idx = -1;
    ProfScope(asd_ctx* c_, cudaStream_t s_, int stage, double bytes, double ops = 0.0) : c(c_), s(s_) {
        if (!c->prof) return;
        const size_t k = c->prof_marks.size();
        if (2 * k + 1 >= c->prof_ev.size()) { ++c->prof_dropped; return; }
        idx = (int)k;
        c->prof_marks.push_back({stage, bytes, ops});
        cudaEventRecord(c->prof_ev[2 * k], s);
    }
    ~ProfScope() { if (idx >= 0) cudaEventRecord(c->prof_ev[2 * idx + 1], s); }
};

// Algorithmic bytes: the minimum HBM traffic each kernel's job
// implies, per frame.  Census: read 1 B/px, write sig B/px (two views).
// Aggregation (design D1, one direction per launch): read+write the u16 S
// volume (4 B/cell), the first direction only writes it (2 B/cell); census
// reads are L2-resident and excluded.  WTA: read S once (2 B/cell) and write
// dl, dr (f32), d* (i16) and masks (u8) for both views.  LR: read those per-
// pixel maps once, write disp and depth (f32).
static double alg_bytes_census(const DevParams& p, size_t sig) { return 2.0 * p.npx * (1 + sig); }
static double alg_bytes_dir(const DevParams& p, bool first)
{   // + the u16 block-cost read in SGBM mode
    return ((first ? 2.0 : 4.0) + (p.bw * p.bh > 1 ? 2.0 : 0.0)) * p.ncell;
}
// SGBM block cost: write CB (u16); census reads are L2-resident.
static double alg_bytes_block(const DevParams& p) { return 2.0 * p.ncell; }
static double alg_bytes_wta(const DevParams& p) { return 2.0 * p.ncell + 2.0 * p.npx * (4 + 2 + 1); }
static double alg_bytes_lr(const DevParams& p) { return p.npx * (2 * (4 + 1) + 2 + 2 * 4.0); }
// Design D3: down sweep writes P_A | C << 8 (u16, 2 B/cell); up sweep reads it
// and writes P_AB | C << 9 (4 B/cell); the row kernel reads the latter,
// writes + reads the u8 left->right stash and writes S over the partial
// (6 B/cell); the WTA kernel reads S once (2 B/cell) and writes the per-pixel
// maps of both views (2 x (4 + 2 + 1) B/px).  Census reads are L2-resident.
static double alg_bytes_down(const DevParams& p) { return 2.0 * p.ncell; }
static double alg_bytes_up(const DevParams& p) { return 4.0 * p.ncell; }
static double alg_bytes_row(const DevParams& p) { return 6.0 * p.ncell; }
static double alg_bytes_wta3(const DevParams& p) { return 2.0 * p.ncell + 2.0 * p.npx * 7; }
// Integer lane-ops per cell, SURVEY §8(d)'s model: o = 5.5 packed (u16x2)
// lane-ops per cell-path of the recursion, + 2 per cell where the Hamming cost
// is evaluated (XOR + POPC).  The down sweep evaluates the cost (SGBM: reads the
// block cost instead), the up sweep takes it from the down sweep's partial
// words, the row kernel evaluates it again in its left->right pass.  (DESIGN.md
// §5 also quotes the minimal packed model, 2.5 per cell-path; bench.py prints
// the fraction under both.)
static double alg_ops_sweep(const DevParams& p)
{
    return (p.paths == 8 ? 3 : 1) * 5.5 * p.ncell + (p.bw * p.bh > 1 ? 0.0 : 2.0) * p.ncell;
}
static double alg_ops_up(const DevParams& p) { return (p.paths == 8 ? 3 : 1) * 5.5 * p.ncell; }
static double alg_ops_row(const DevParams& p)
{
    return 2 * 5.5 * p.ncell + (p.bw * p.bh > 1 ? 0.0 : 2.0) * p.ncell;
}
static double alg_ops_wta3(const DevParams& p) { return 3.0 * p.ncell; }

// Frames per D3 pipeline group; max_batch / group scratch slots, one
// slot-free event each.
int set_group(asd_ctx* c, int group)
{
    if (group < 1 || group > c->max_batch) return ASD_E_INVALID_ARG;
    // frames split over several clusters need all of a group's clusters
    // resident at once (their boundary columns wait on each other): at most one wave
    if (c->engine == ASD_ENGINE_D3 && c->plan.ncta > c->plan.cs &&
        group > c->plan.active_ctas / c->plan.ncta) return ASD_E_INVALID_ARG;
    for (cudaEvent_t e : c->ev_free) if (e) cudaEventDestroy(e);
    c->ev_free.assign(c->engine == ASD_ENGINE_D3 ? c->max_batch / group : 0, nullptr);
    for (cudaEvent_t& e : c->ev_free)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return ASD_E_CUDA;
    c->group = group;
    return ASD_OK;
}

// Design D3: the whole path for any n frames resident on the device, as a
// software pipeline over groups of G frames (one wave of sweep clusters) and a
// ring of max_batch / G scratch slots, on three streams forked from the
// caller's:
//   s_cen (high priority): census of group g, once its slot is free;
//   s_hi  (high priority): down + up sweeps of group g (the cluster kernels
//                          occupy cs * clusters-per-wave SMs);
//   s_lo  (low priority):  row + WTA + LR of group g, which fill the SMs the
//                          clusters leave free while group g + 1 sweeps.
// The census of group g + 1 is enqueued ahead, so when the up sweep of group
// g ends the down sweep of g + 1 and the row pass of g become ready together
// and the stream priorities hand the freed SMs to the clusters first.
// ev_free[slot] orders the reuse of a slot after the LR pass of the group that
// last used it.
// Host mode (hio != nullptr): inputs are copied per group from pinned host
// memory into the slot's staging buffer on s_cen ahead of its census, and the
// slot's outputs go back on copy_stream after its LR pass; the slot is freed
// once that copy is done.
struct HostIO {
    const uint8_t* left; const uint8_t* right;
    float* disp; float* depth; asd_frame_stats* stats;
};

int run_d3(asd_ctx* c, int n, const uint8_t* left, const uint8_t* right,
           float* out_disp, float* out_depth, asd_frame_stats* stats,
           uint8_t* mask_out, cudaStream_t s, uint16_t* agg_debug, const HostIO* hio = nullptr)
{
    const DevParams& p = c->dp;
    if (n <= 0) return ASD_OK;
    const long long npx = p.npx;
    const FrameScratch fs = frame_scratch(c);
    const int G = c->group;
    const int nslots = (int)c->ev_free.size();
    const int ngroups = (n + G - 1) / G;
    const long long pa_frame = (long long)p.H * c->plan.ncta * c->plan.w * p.D;   // u16 elements
    const bool blk = c->cb != nullptr;             // SGBM: block cost in the private layout
    const int wpad = c->plan.ncta * c->plan.w;
    struct Slot { void* cl; void* cr; uint8_t* pa; uint16_t* pab; uint8_t* stash; uint16_t* cb; uint16_t* cb2;
                  uint8_t* pa2; uint16_t* pab2; uint8_t* stash2; FrameScratch g; };
    const bool r2 = c->pa2 != nullptr;             // R2: a right-referenced second pass (c24)
    auto slot_of = [&](int gi) {
        const long long b0 = (long long)(gi % nslots) * G;   // first scratch frame of the slot
        Slot q;
        q.cl = (char*)c->census_l + b0 * npx * (long long)c->sig_bytes;
        q.cr = (char*)c->census_r + b0 * npx * (long long)c->sig_bytes;
        q.pa = c->pa + b0 * pa_frame * 2;
        q.pab = c->pab + b0 * p.ncell;
        q.stash = c->stash + b0 * p.ncell * (blk ? 2 : 1);
        q.cb = blk ? c->cb + b0 * pa_frame : nullptr;
        q.cb2 = c->cb2 ? c->cb2 + b0 * pa_frame : nullptr;
        q.pa2 = r2 ? c->pa2 + b0 * pa_frame * 2 : nullptr;
        q.pab2 = r2 ? c->pab2 + b0 * p.ncell : nullptr;
        q.stash2 = r2 ? c->stash2 + b0 * p.ncell * (blk ? 2 : 1) : nullptr;
        q.g = fs;
        q.g.census_l = q.cl; q.g.census_r = q.cr;
        q.g.dl += b0 * npx; q.g.dr += b0 * npx; q.g.dstar_l += b0 * npx; q.g.dstar_r += b0 * npx;
        q.g.mask_l += b0 * npx; q.g.mask_r += b0 * npx;
        return q;
    };
    auto frames = [&](int gi) { return (n - gi * G) < G ? (n - gi * G) : G; };
    const long long MB = c->max_batch;
    auto census = [&](int gi) {
        const Slot q = slot_of(gi);
        const int m = frames(gi);
        const long long f0 = (long long)gi * G;
        if (gi >= nslots) cudaStreamWaitEvent(c->s_cen, c->ev_free[gi % nslots], 0);
        const uint8_t* il = hio ? nullptr : left + f0 * npx;
        const uint8_t* ir = hio ? nullptr : right + f0 * npx;
        if (hio) {                                     // H2D of this group into its slot
            const long long b0 = (long long)(gi % nslots) * G;
            uint8_t* dl = c->stage_in[0] + b0 * npx;
            uint8_t* dr = c->stage_in[0] + (MB + b0) * npx;
            cudaMemcpyAsync(dl, hio->left + f0 * npx, (size_t)m * npx, cudaMemcpyHostToDevice, c->s_cen);
            cudaMemcpyAsync(dr, hio->right + f0 * npx, (size_t)m * npx, cudaMemcpyHostToDevice, c->s_cen);
            il = dl; ir = dr;
        }
        {
            ProfScope ps(c, c->s_cen, ASD_STAGE_CENSUS, m * alg_bytes_census(p, c->sig_bytes));
            launch_census(p, m, il, ir, npx, q.cl, q.cr, npx, c->s_cen);
        }
        if (blk) {                                     // SGBM: block cost(s), private layout
            ProfScope ps(c, c->s_cen, ASD_STAGE_BLOCK, m * alg_bytes_block(p));
            launch_block_cost(p, m, q.cl, q.cr, npx, q.cb, pa_frame, c->s_cen, false, wpad);
            if (q.cb2) launch_block_cost(p, m, q.cl, q.cr, npx, q.cb2, pa_frame, c->s_cen, true, wpad);
        }
        cudaEventRecord(c->ev_cen, c->s_cen);
    };
    cudaEventRecord(c->ev_fork, s);                    // inputs (and outputs) are ordered on s
    for (cudaStream_t q : {c->s_cen, c->s_hi, c->s_lo}) cudaStreamWaitEvent(q, c->ev_fork, 0);
    census(0);
    for (int gi = 0; gi < ngroups; ++gi) {
        const Slot q = slot_of(gi);
        const int m = frames(gi);
        const long long f0 = (long long)gi * G;
        cudaStreamWaitEvent(c->s_hi, c->ev_cen, 0);   // census of this group (and so its slot) ready
        {
            ProfScope ps(c, c->s_hi, ASD_STAGE_DOWN, m * alg_bytes_down(p), m * alg_ops_sweep(p));
            if (launch_v2_stage(0, p, c->plan, m, q.cl, q.cr, npx, q.pa, q.pab, q.stash, p.ncell, q.g, npx,
                                nullptr, c->s_hi, 0, q.cb) != 0) {
                set_err(c, "down sweep launch failed: %s", cudaGetErrorString(cudaGetLastError()));
                return ASD_E_CUDA;
            }
        }
        // with a single slot the next census must wait for this group's LR
        if (gi + 1 < ngroups && nslots > 1) census(gi + 1);
        {
            ProfScope ps(c, c->s_hi, ASD_STAGE_UP, m * alg_bytes_up(p), m * alg_ops_up(p));
            if (launch_v2_stage(1, p, c->plan, m, q.cl, q.cr, npx, q.pa, q.pab, q.stash, p.ncell, q.g, npx,
                                nullptr, c->s_hi, 0, q.cb) != 0) {
                set_err(c, "up sweep launch failed: %s", cudaGetErrorString(cudaGetLastError()));
                return ASD_E_CUDA;
            }
        }
        cudaEventRecord(c->ev_sw, c->s_hi);
        if (r2) {                                    // the right view's own sweeps (R2)
            {
                ProfScope ps(c, c->s_hi, ASD_STAGE_DOWN, m * alg_bytes_down(p), m * alg_ops_sweep(p));
                if (launch_v2_stage(0, p, c->plan, m, q.cr, q.cl, npx, q.pa2, q.pab2, q.stash2, p.ncell, q.g, npx,
                                    nullptr, c->s_hi, 1, q.cb2) != 0) {
                    set_err(c, "right-view down sweep launch failed: %s", cudaGetErrorString(cudaGetLastError()));
                    return ASD_E_CUDA;
                }
            }
            {
                ProfScope ps(c, c->s_hi, ASD_STAGE_UP, m * alg_bytes_up(p), m * alg_ops_up(p));
                if (launch_v2_stage(1, p, c->plan, m, q.cr, q.cl, npx, q.pa2, q.pab2, q.stash2, p.ncell, q.g, npx,
                                    nullptr, c->s_hi, 0, q.cb2) != 0) {
                    set_err(c, "right-view up sweep launch failed: %s", cudaGetErrorString(cudaGetLastError()));
                    return ASD_E_CUDA;
                }
            }
            cudaEventRecord(c->ev_sw2, c->s_hi);
        }
        cudaStreamWaitEvent(c->s_lo, c->ev_sw, 0);
        {
            ProfScope ps(c, c->s_lo, ASD_STAGE_ROW, m * alg_bytes_row(p), m * alg_ops_row(p));
            launch_v2_stage(2, p, c->plan, m, q.cl, q.cr, npx, q.pa, q.pab, q.stash, p.ncell, q.g, npx,
                            nullptr, c->s_lo, 0, q.cb);
        }
        if (agg_debug && gi == 0)            // S of frame 0 (natural order) before the WTA
            cudaMemcpyAsync(agg_debug, q.pab, (size_t)p.ncell * 2, cudaMemcpyDeviceToDevice, c->s_lo);
        {
            ProfScope ps(c, c->s_lo, ASD_STAGE_WTA, m * alg_bytes_wta3(p), m * alg_ops_wta3(p));
            if (launch_v2_stage(3, p, c->plan, m, q.cl, q.cr, npx, q.pa, q.pab, q.stash, p.ncell, q.g, npx,
                                nullptr, c->s_lo, r2 ? 1 : 0) != 0) {
                set_err(c, "WTA launch failed: %s", cudaGetErrorString(cudaGetLastError()));
                return ASD_E_CUDA;
            }
        }
        if (r2) {                                    // right view from its own aggregate
            cudaStreamWaitEvent(c->s_lo, c->ev_sw2, 0);
            {
                ProfScope ps(c, c->s_lo, ASD_STAGE_ROW, m * alg_bytes_row(p), m * alg_ops_row(p));
                launch_v2_stage(2, p, c->plan, m, q.cr, q.cl, npx, q.pa2, q.pab2, q.stash2, p.ncell, q.g, npx,
                                nullptr, c->s_lo, 1, q.cb2);
            }
            {
                ProfScope ps(c, c->s_lo, ASD_STAGE_WTA, m * alg_bytes_wta3(p), m * alg_ops_wta3(p));
                if (launch_v2_stage(3, p, c->plan, m, q.cr, q.cl, npx, q.pa2, q.pab2, q.stash2, p.ncell, q.g, npx,
                                    nullptr, c->s_lo, 2) != 0) {
                    set_err(c, "right-view WTA launch failed: %s", cudaGetErrorString(cudaGetLastError()));
                    return ASD_E_CUDA;
                }
            }
        }
        float* od = out_disp ? out_disp + f0 * npx : nullptr;
        float* oz = out_depth ? out_depth + f0 * npx : nullptr;
        asd_frame_stats* os = stats ? stats + f0 : nullptr;
        if (hio) {                                     // outputs into the slot's staging buffers
            const long long b0 = (long long)(gi % nslots) * G;
            od = hio->disp ? c->stage_out[0] + b0 * npx : nullptr;
            oz = hio->depth ? c->stage_out[0] + (MB + b0) * npx : nullptr;
            os = hio->stats ? c->stage_stats[0] + b0 : nullptr;
        }
        if (os) cudaMemsetAsync(os, 0, sizeof(asd_frame_stats) * m, c->s_lo);
        {
            ProfScope ps(c, c->s_lo, ASD_STAGE_LR, m * alg_bytes_lr(p));
            launch_lr_depth(p, m, q.g, npx, od, oz, npx, mask_out ? mask_out + f0 * npx : nullptr, os, c->s_lo);
        }
        if (hio) {                                     // D2H of this group, then the slot is free
            cudaEventRecord(c->ev_comp[0], c->s_lo);
            cudaStreamWaitEvent(c->copy_stream, c->ev_comp[0], 0);
            if (od) cudaMemcpyAsync(hio->disp + f0 * npx, od, (size_t)m * npx * 4, cudaMemcpyDeviceToHost, c->copy_stream);
            if (oz) cudaMemcpyAsync(hio->depth + f0 * npx, oz, (size_t)m * npx * 4, cudaMemcpyDeviceToHost, c->copy_stream);
            if (os) cudaMemcpyAsync(hio->stats + f0, os, m * sizeof(asd_frame_stats), cudaMemcpyDeviceToHost, c->copy_stream);
            cudaEventRecord(c->ev_free[gi % nslots], c->copy_stream);
        } else {
            cudaEventRecord(c->ev_free[gi % nslots], c->s_lo);
        }
        if (gi + 1 < ngroups && nslots == 1) census(gi + 1);
    }
    cudaEventRecord(c->ev_hi, c->s_hi);              // join back to the caller's stream
    cudaEventRecord(c->ev_lo, hio ? c->copy_stream : c->s_lo);
    cudaStreamWaitEvent(s, c->ev_hi, 0);
    cudaStreamWaitEvent(s, c->ev_lo, 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_err(c, "CUDA launch failed: %s", cudaGetErrorString(e));
        return ASD_E_CUDA;
    }
    return ASD_OK;
}

// Design D1: the whole path for n <= max_batch frames resident on the device.
int run_chunk(asd_ctx* c, int n, const uint8_t* left, const uint8_t* right,
              float* out_disp, float* out_depth, asd_frame_stats* stats,
              uint8_t* mask_out, cudaStream_t s, uint16_t* agg_debug = nullptr)
{
    if (c->engine == ASD_ENGINE_D3)
        return run_d3(c, n, left, right, out_disp, out_depth, stats, mask_out, s, agg_debug);
    const DevParams& p = c->dp;
    if (n <= 0) return ASD_OK;
    const long long npx = p.npx;
    {
        ProfScope ps(c, s, ASD_STAGE_CENSUS, n * alg_bytes_census(p, c->sig_bytes));
        launch_census(p, n, left, right, npx, c->census_l, c->census_r, npx, s);
    }
    FrameScratch fs = frame_scratch(c);
    if (c->engine == ASD_ENGINE_D1 && c->cb) {      // SGBM: block cost volume first
        ProfScope ps(c, s, ASD_STAGE_BLOCK, n * alg_bytes_block(p));
        launch_block_cost(p, n, c->census_l, c->census_r, npx, c->cb, p.ncell, s);
    }
    for (int r = 0; c->engine == ASD_ENGINE_D1 && r < p.paths; ++r) {
        ProfScope ps(c, s, ASD_STAGE_DIR, n * alg_bytes_dir(p, r == 0));
        if (!launch_sgm_dir(p, n, kDirs[r][0], kDirs[r][1], r == 0, c->census_l, c->census_r, npx,
                            c->S, p.ncell, s, c->cb)) {
            set_err(c, "no SGM kernel instance for num_disp=%d", p.D);
            return ASD_E_UNSUPPORTED;
        }
    }
    if (c->engine == ASD_ENGINE_D1 && c->SR) {      // R2: the right view's own SGM (c24)
        if (c->cb) {
            ProfScope ps(c, s, ASD_STAGE_BLOCK, n * alg_bytes_block(p));
            launch_block_cost(p, n, c->census_l, c->census_r, npx, c->cb, p.ncell, s, true);
        }
        for (int r = 0; r < p.paths; ++r) {
            ProfScope ps(c, s, ASD_STAGE_DIR, n * alg_bytes_dir(p, r == 0));
            if (!launch_sgm_dir(p, n, kDirs[r][0], kDirs[r][1], r == 0, c->census_l, c->census_r, npx,
                                c->SR, p.ncell, s, c->cb, true)) {
                set_err(c, "no SGM kernel instance for num_disp=%d", p.D);
                return ASD_E_UNSUPPORTED;
            }
        }
    }
    if (c->engine == ASD_ENGINE_D1) {
        ProfScope ps(c, s, ASD_STAGE_WTA, n * alg_bytes_wta(p) * (c->SR ? 1.5 : 1.0));
        if (c->wta2) launch_wta2(p, c->plan, n, c->S, p.ncell, fs, npx, s);
        else if (!launch_wta(p, n, c->S, p.ncell, fs, npx, s, c->SR)) {
            set_err(c, "no WTA kernel instance for num_disp=%d", p.D);
            return ASD_E_UNSUPPORTED;
        }
    }
    if (stats) cudaMemsetAsync(stats, 0, sizeof(asd_frame_stats) * n, s);
    {
        ProfScope ps(c, s, ASD_STAGE_LR, n * alg_bytes_lr(p));
        launch_lr_depth(p, n, fs, npx, out_disp, out_depth, npx, mask_out, stats, s);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_err(c, "CUDA launch failed: %s", cudaGetErrorString(e));
        return ASD_E_CUDA;
    }
    return ASD_OK;
}

void free_ctx(asd_ctx* c)
{
    if (!c) return;
    void* ptrs[] = {c->census_l_base, c->census_r_base, c->S, c->SR, c->cb, c->cb2, c->dl, c->dr, c->dstar_l, c->dstar_r,
                    c->mask_l, c->mask_r, c->pa, c->pab, c->stash, c->pa2, c->pab2, c->stash2, c->plan.ghalo,
                    c->stage_in[0], c->stage_in[1], c->stage_out[0],
                    c->stage_out[1], c->stage_stats[0], c->stage_stats[1]};
    for (void* q : ptrs) if (q) cudaFree(q);
    for (int i = 0; i < 2; ++i) {
        if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
        if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
        if (c->ev_comp[i]) cudaEventDestroy(c->ev_comp[i]);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (cudaStream_t q : {c->s_hi, c->s_lo, c->s_cen}) if (q) cudaStreamDestroy(q);
    for (cudaEvent_t e : {c->ev_fork, c->ev_sw, c->ev_sw2, c->ev_hi, c->ev_lo, c->ev_cen}) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_free) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
    delete c;
}

}  // namespace

extern "C" {

int asd_version(void) { return ASD_VERSION; }

const char* asd_strerror(int code)
{
    switch (code) {
        case ASD_OK: return "ok";
        case ASD_E_INVALID_ARG: return "invalid argument";
        case ASD_E_UNSUPPORTED: return "unsupported configuration";
        case ASD_E_CUDA: return "CUDA error";
        case ASD_E_OOM: return "out of device memory";
        default: return "unknown error";
    }
}

const char* asd_last_error(const asd_ctx* ctx) { return ctx ? ctx->err : g_err; }

size_t asd_scratch_bytes(const asd_params* p, int max_batch)
{
    char why[256];
    if (validate(p, why, sizeof why) != ASD_OK || max_batch < 1 || max_batch > 1024) return 0;
    const DevParams d = make_dev(p);
    int engine = p->engine == ASD_ENGINE_AUTO ? ASD_ENGINE_D1 : p->engine;
    if (p->engine != ASD_ENGINE_D1) {
        int dev = 0;
        cudaGetDevice(&dev);
        V2Plan pl;
        if (v2_plan(d, dev, pl))
            return layout(d, max_batch, ASD_ENGINE_D3, pl.ncta * pl.w, pl.blk).total +
                   v2_ghalo_bytes(pl, max_batch) +
                   4 * align_up((size_t)4 * ((size_t)d.min_disp + d.D + 1024 + 64));   // census guards
        cudaGetLastError();
    }
    return layout(d, max_batch, engine, d.W).total;
}

int asd_create(const asd_params* p, int device, int max_batch, asd_ctx** out)
{
    char why[256];
    if (!out) { set_err(nullptr, "out is NULL"); return ASD_E_INVALID_ARG; }
    *out = nullptr;
    int rc = validate(p, why, sizeof why);
    if (rc != ASD_OK) { set_err(nullptr, "%s", why); return rc; }
    if (max_batch < 1 || max_batch > 1024) { set_err(nullptr, "max_batch must be in [1, 1024]"); return ASD_E_INVALID_ARG; }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        set_err(nullptr, "device %d not available (%d CUDA devices)", device, ndev);
        return ASD_E_CUDA;
    }
    DeviceGuard g(device);
    asd_ctx* c = new (std::nothrow) asd_ctx();
    if (!c) return ASD_E_OOM;
    c->prm = *p;
    c->dp = make_dev(p);
    c->device = device;
    c->max_batch = max_batch;
    c->sig_bytes = c->dp.nb <= 32 ? 4 : 8;
    c->engine = ASD_ENGINE_D1;
    if (p->engine != ASD_ENGINE_D1) {
        if (v2_plan(c->dp, device, c->plan)) {
            c->engine = ASD_ENGINE_D3;
        } else if (p->engine == ASD_ENGINE_D3) {
            set_err(nullptr, "engine D3 unsupported for these parameters: %s", c->plan.why);
            delete c;
            return ASD_E_UNSUPPORTED;
        }
    }
    // Engine D1 with D in 16..128 and the R1 right view: the ring-window WTA
    // kernel (wta2), with u32 keys when S can reach 2^(16 - log2 D).
    c->wta2 = false;
    if (c->engine == ASD_ENGINE_D1 && c->dp.lr_mode == 0 &&
        (c->dp.D == 16 || c->dp.D == 32 || c->dp.D == 64 || c->dp.D == 96 || c->dp.D == 128 ||
         c->dp.D == 256)) {
        const int ks = c->dp.D <= 16 ? 4 : c->dp.D <= 32 ? 5 : c->dp.D <= 64 ? 6 : c->dp.D <= 128 ? 7 : 8;
        const long long smax = (long long)c->dp.paths * ((long long)c->dp.bw * c->dp.bh * c->dp.nb + c->dp.p2);
        if (wta2_plan(c->dp, smax >= (1ll << (16 - ks)), c->plan, true)) c->wta2 = true;
    }
    Layout L = layout(c->dp, max_batch, c->engine,
                      c->engine == ASD_ENGINE_D3 ? c->plan.ncta * c->plan.w : c->dp.W,
                      c->engine == ASD_ENGINE_D3 && c->plan.blk);
    bool ok = true;
    auto alloc = [&](void** q, size_t bytes) {
        if (ok && cudaMalloc(q, bytes) != cudaSuccess) ok = false;
#ifdef ASD_CHECKED
        // checked builds: poison all scratch, so a read of a cell no kernel
        // wrote changes the results (the initcheck of this build)
        if (ok) cudaMemset(*q, 0xA5, bytes);
#endif
    };
    // census buffers with guard bands: the D3 down sweep's TMA staging copies
    // from 16-byte aligned starts up to min_disp + D + w columns outside a row
    c->cen_guard = align_up((size_t)4 * ((size_t)c->dp.min_disp + c->dp.D + 1024 + 64));
    alloc(&c->census_l_base, L.sig + 2 * c->cen_guard); alloc(&c->census_r_base, L.sig + 2 * c->cen_guard);
    if (ok) {
        c->census_l = (char*)c->census_l_base + c->cen_guard;
        c->census_r = (char*)c->census_r_base + c->cen_guard;
    }
    if (L.s) alloc((void**)&c->S, L.s);
    if (L.cb) alloc((void**)&c->cb, L.cb);
    if (L.sr) alloc((void**)&c->SR, L.sr);
    if (L.pa) alloc((void**)&c->pa, L.pa);
    if (L.pab) alloc((void**)&c->pab, L.pab);
    if (L.stash) alloc((void**)&c->stash, L.stash);
    if (L.r2 && L.cb && c->engine == ASD_ENGINE_D3) alloc((void**)&c->cb2, L.cb);
    if (L.r2) {
        alloc((void**)&c->pa2, L.pa);
        alloc((void**)&c->pab2, L.pab);
        alloc((void**)&c->stash2, L.stash);
    }
    if (c->engine == ASD_ENGINE_D3 && v2_ghalo_bytes(c->plan, max_batch) > 0)
        alloc((void**)&c->plan.ghalo, v2_ghalo_bytes(c->plan, max_batch));
    alloc((void**)&c->dl, L.px_f32); alloc((void**)&c->dr, L.px_f32);
    alloc((void**)&c->dstar_l, L.px_i16); alloc((void**)&c->dstar_r, L.px_i16);
    alloc((void**)&c->mask_l, L.px_u8); alloc((void**)&c->mask_r, L.px_u8);
    for (int i = 0; i < 2; ++i) {
        alloc((void**)&c->stage_in[i], L.stage_in);
        alloc((void**)&c->stage_out[i], L.stage_out);
        alloc((void**)&c->stage_stats[i], L.stats);
    }
    if (!ok) {
        cudaGetLastError();
        set_err(nullptr, "cudaMalloc of %zu scratch bytes failed", L.total);
        free_ctx(c);
        return ASD_E_OOM;
    }
    if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) ok = false;
    {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (ok && (cudaStreamCreateWithPriority(&c->s_hi, cudaStreamNonBlocking, hi) != cudaSuccess ||
                   cudaStreamCreateWithPriority(&c->s_lo, cudaStreamNonBlocking, lo) != cudaSuccess ||
                   cudaStreamCreateWithPriority(&c->s_cen, cudaStreamNonBlocking, hi) != cudaSuccess))
            ok = false;
        for (cudaEvent_t* e : {&c->ev_fork, &c->ev_sw, &c->ev_sw2, &c->ev_hi, &c->ev_lo, &c->ev_cen})
            if (ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) ok = false;
        // overlap group: one wave of sweep clusters, at most max_batch
        const int wave = c->plan.ncta > 0 ? c->plan.active_ctas / c->plan.ncta : 1;
        if (ok && set_group(c, wave < 1 ? 1 : wave > max_batch ? max_batch : wave) != ASD_OK) ok = false;
    }
    for (int i = 0; i < 2 && ok; ++i)
        if (cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_comp[i], cudaEventDisableTiming) != cudaSuccess) ok = false;
    if (!ok) {
        set_err(nullptr, "stream/event creation failed: %s", cudaGetErrorString(cudaGetLastError()));
        free_ctx(c);
        return ASD_E_CUDA;
    }
    *out = c;
    return ASD_OK;
}

void asd_destroy(asd_ctx* ctx)
{
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    free_ctx(ctx);
}

int asd_launches_per_batch(const asd_ctx* ctx, int n)
{
    if (!ctx || n <= 0) return 0;
    const int chunks = (n + ctx->max_batch - 1) / ctx->max_batch;
    if (ctx->engine != ASD_ENGINE_D3)
        return chunks * (3 + (ctx->dp.paths + (ctx->cb ? 1 : 0)) * (ctx->SR ? 2 : 1));
    // per group: census, down, up, row, WTA, LR (+ down, up, row, WTA of the R2 right view)
    // (+ the SGBM block cost kernel(s) on the census stream)
    const int per = (ctx->pa2 ? 10 : 6) + (ctx->cb ? (ctx->cb2 ? 2 : 1) : 0);
    return per * ((n + ctx->group - 1) / ctx->group);
}

int asd_engine(const asd_ctx* ctx) { return ctx ? ctx->engine : 0; }

int asd_set_group(asd_ctx* ctx, int group)
{
    if (!ctx) { set_err(nullptr, "ctx is NULL"); return ASD_E_INVALID_ARG; }
    if (group < 1 || group > ctx->max_batch) {
        set_err(ctx, "group %d outside [1, max_batch=%d]", group, ctx->max_batch);
        return ASD_E_INVALID_ARG;
    }
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();                 // no batch of this context may be in flight
    const int rc = set_group(ctx, group);
    if (rc != ASD_OK) set_err(ctx, "event creation failed");
    return rc;
}

int asd_group(const asd_ctx* ctx) { return ctx ? ctx->group : 0; }

int asd_plan_info(const asd_ctx* ctx, char* buf, int n)
{
    if (!ctx || !buf || n <= 0) return 0;
    if (ctx->engine != ASD_ENGINE_D3)
        return snprintf(buf, n, "engine D1: %d direction kernels (warp per line), WTA kernel", ctx->dp.paths);
    const V2Plan& q = ctx->plan;
    return snprintf(buf, n,
                    "engine D3: sweeps DC=%d T=%d paths/sweep=%d cluster=%d x %d per frame, CTA=%d cols x %d thr, "
                    "%d resident CTAs (%d frames/wave), smem %zu B; WTA %s %d rows",
                    q.DC, q.T, q.NP, q.cs, q.NP == 3 ? q.ncta / q.cs : 1, q.w, q.vthreads, q.active_ctas,
                    q.NP == 3 ? q.active_ctas / q.ncta : 0, q.vsmem, q.wta_fb ? "warp-per-pixel (no ring)" : "ring", q.nbuf);
}

int asd_frames_per_wave(const asd_ctx* ctx)
{
    if (!ctx || ctx->engine != ASD_ENGINE_D3) return 0;
    const int per = ctx->plan.NP == 3 ? ctx->plan.ncta : 1;
    return ctx->plan.NP == 3 ? ctx->plan.active_ctas / per : 0;
}

int asd_depth_batch(asd_ctx* ctx, int n, const uint8_t* left, const uint8_t* right,
                    float* out_disp, float* out_depth, asd_frame_stats* stats, void* cuda_stream)
{
    if (!ctx) { set_err(nullptr, "ctx is NULL"); return ASD_E_INVALID_ARG; }
    if (n < 0) { set_err(ctx, "n < 0"); return ASD_E_INVALID_ARG; }
    if (n == 0) return ASD_OK;
    if (!left || !right) { set_err(ctx, "left/right is NULL"); return ASD_E_INVALID_ARG; }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const long long npx = ctx->dp.npx;
    if (ctx->engine == ASD_ENGINE_D3)               // pipelined over scratch slots, any n
        return run_d3(ctx, n, left, right, out_disp, out_depth, stats, nullptr, s, nullptr);
    for (int f0 = 0; f0 < n; f0 += ctx->max_batch) {
        const int m = (n - f0) < ctx->max_batch ? (n - f0) : ctx->max_batch;
        int rc = run_chunk(ctx, m, left + f0 * npx, right + f0 * npx,
                           out_disp ? out_disp + f0 * npx : nullptr,
                           out_depth ? out_depth + f0 * npx : nullptr,
                           stats ? stats + f0 : nullptr, nullptr, s);
        if (rc != ASD_OK) return rc;
    }
    return ASD_OK;
}

int asd_depth(asd_ctx* ctx, const uint8_t* left, const uint8_t* right,
              float* out_disp, float* out_depth, void* cuda_stream)
{
    return asd_depth_batch(ctx, 1, left, right, out_disp, out_depth, nullptr, cuda_stream);
}

int asd_depth_batch_host(asd_ctx* ctx, int n, const uint8_t* left_host, const uint8_t* right_host,
                         float* out_disp_host, float* out_depth_host, asd_frame_stats* stats_host,
                         void* cuda_stream)
{
    if (!ctx) { set_err(nullptr, "ctx is NULL"); return ASD_E_INVALID_ARG; }
    if (n < 0) { set_err(ctx, "n < 0"); return ASD_E_INVALID_ARG; }
    if (n == 0) return ASD_OK;
    if (!left_host || !right_host) { set_err(ctx, "left/right is NULL"); return ASD_E_INVALID_ARG; }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    if (ctx->engine == ASD_ENGINE_D3) {           // per-group copies inside the D3 pipeline
        const HostIO hio{left_host, right_host, out_disp_host, out_depth_host, stats_host};
        int rc = run_d3(ctx, n, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, s, nullptr, &hio);
        cudaError_t e = cudaStreamSynchronize(s);
        if (rc != ASD_OK) return rc;
        if (e != cudaSuccess) { set_err(ctx, "host pipeline failed: %s", cudaGetErrorString(e)); return ASD_E_CUDA; }
        return ASD_OK;
    }
    cudaStream_t cs = ctx->copy_stream;
    const size_t npx = (size_t)ctx->dp.npx;
    const int B = ctx->max_batch;
    const int nchunks = (n + B - 1) / B;
    // Pipeline: H2D(k+1) on the copy stream overlaps compute(k) on s; D2H(k) on
    // the copy stream waits for compute(k) and overlaps compute(k+1).
    auto chunk_n = [&](int k) { return (k + 1) * B <= n ? B : n - k * B; };
    auto h2d = [&](int k) {
        const int b = k & 1, m = chunk_n(k);
        uint8_t* in = ctx->stage_in[b];
        cudaStreamWaitEvent(cs, ctx->ev_done[b], 0);          // slot free (its D2H finished)
        cudaMemcpyAsync(in, left_host + (size_t)k * B * npx, m * npx, cudaMemcpyHostToDevice, cs);
        cudaMemcpyAsync(in + (size_t)B * npx, right_host + (size_t)k * B * npx, m * npx,
                        cudaMemcpyHostToDevice, cs);
        cudaEventRecord(ctx->ev_in[b], cs);
    };
    for (int i = 0; i < 2; ++i) cudaEventRecord(ctx->ev_done[i], cs);
    h2d(0);
    for (int k = 0; k < nchunks; ++k) {
        const int b = k & 1, m = chunk_n(k);
        uint8_t* in = ctx->stage_in[b];
        float* od = ctx->stage_out[b];
        float* oz = od + (size_t)B * npx;
        cudaStreamWaitEvent(s, ctx->ev_in[b], 0);
        int rc = run_chunk(ctx, m, in, in + (size_t)B * npx, out_disp_host ? od : nullptr,
                           out_depth_host ? oz : nullptr, stats_host ? ctx->stage_stats[b] : nullptr,
                           nullptr, s);
        if (rc != ASD_OK) { cudaStreamSynchronize(s); cudaStreamSynchronize(cs); return rc; }
        cudaEvent_t computed = ctx->ev_comp[b];
        cudaEventRecord(computed, s);
        if (k + 1 < nchunks) h2d(k + 1);
        cudaStreamWaitEvent(cs, computed, 0);
        if (out_disp_host)
            cudaMemcpyAsync(out_disp_host + (size_t)k * B * npx, od, m * npx * 4, cudaMemcpyDeviceToHost, cs);
        if (out_depth_host)
            cudaMemcpyAsync(out_depth_host + (size_t)k * B * npx, oz, m * npx * 4, cudaMemcpyDeviceToHost, cs);
        if (stats_host)
            cudaMemcpyAsync(stats_host + (size_t)k * B, ctx->stage_stats[b], m * sizeof(asd_frame_stats),
                            cudaMemcpyDeviceToHost, cs);
        cudaEventRecord(ctx->ev_done[b], cs);
    }
    cudaError_t e = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { set_err(ctx, "host pipeline failed: %s", cudaGetErrorString(e)); return ASD_E_CUDA; }
    return ASD_OK;
}

int asd_depth_debug(asd_ctx* ctx, const uint8_t* left, const uint8_t* right,
                    const asd_debug_out* outs, float* out_disp, float* out_depth, void* cuda_stream)
{
    if (!ctx) { set_err(nullptr, "ctx is NULL"); return ASD_E_INVALID_ARG; }
    if (!left || !right) { set_err(ctx, "left/right is NULL"); return ASD_E_INVALID_ARG; }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    asd_debug_out o{};
    if (outs) o = *outs;
    const DevParams& p = ctx->dp;
    int rc = run_chunk(ctx, 1, left, right, out_disp, out_depth, nullptr, o.mask, s,
                       ctx->engine == ASD_ENGINE_D3 ? o.agg : nullptr);
    if (rc != ASD_OK) return rc;
    const size_t npx = (size_t)p.npx;
    if (o.census_l) cudaMemcpyAsync(o.census_l, ctx->census_l, npx * ctx->sig_bytes, cudaMemcpyDeviceToDevice, s);
    if (o.census_r) cudaMemcpyAsync(o.census_r, ctx->census_r, npx * ctx->sig_bytes, cudaMemcpyDeviceToDevice, s);
    if (o.cost) launch_cost_volume(p, ctx->census_l, ctx->census_r, o.cost, s);
    if (o.agg && ctx->engine == ASD_ENGINE_D1)
        cudaMemcpyAsync(o.agg, ctx->S, (size_t)p.ncell * 2, cudaMemcpyDeviceToDevice, s);
    if (o.dstar_l) cudaMemcpyAsync(o.dstar_l, ctx->dstar_l, npx * 2, cudaMemcpyDeviceToDevice, s);
    if (o.dstar_r) cudaMemcpyAsync(o.dstar_r, ctx->dstar_r, npx * 2, cudaMemcpyDeviceToDevice, s);
    if (o.disp_l) cudaMemcpyAsync(o.disp_l, ctx->dl, npx * 4, cudaMemcpyDeviceToDevice, s);
    if (o.disp_r) cudaMemcpyAsync(o.disp_r, ctx->dr, npx * 4, cudaMemcpyDeviceToDevice, s);
    if (o.mask_r) cudaMemcpyAsync(o.mask_r, ctx->mask_r, npx, cudaMemcpyDeviceToDevice, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_err(ctx, "debug extraction failed: %s", cudaGetErrorString(e)); return ASD_E_CUDA; }
    return ASD_OK;
}

int asd_rectify(const double* Hm, int n, int width, int height, const uint8_t* in, uint8_t* out,
                void* cuda_stream)
{
    if (!Hm || n < 0 || n > 65535 || (n > 0 && (!in || !out)) || width < 1 || height < 1 ||
        (long long)width * height > (1ll << 26)) {
        set_err(nullptr, "asd_rectify: NULL argument or size out of range");
        return ASD_E_INVALID_ARG;
    }
    for (int i = 0; i < 9; ++i)
        if (!std::isfinite(Hm[i])) { set_err(nullptr, "asd_rectify: non-finite homography"); return ASD_E_INVALID_ARG; }
    const double det = Hm[0] * (Hm[4] * Hm[8] - Hm[5] * Hm[7]) - Hm[1] * (Hm[3] * Hm[8] - Hm[5] * Hm[6]) +
                       Hm[2] * (Hm[3] * Hm[7] - Hm[4] * Hm[6]);
    if (!(std::fabs(det) > 0.0)) { set_err(nullptr, "asd_rectify: singular homography"); return ASD_E_INVALID_ARG; }
    if (n == 0) return ASD_OK;
    if (launch_rectify(Hm, n, width, height, in, out, (cudaStream_t)cuda_stream) != 0) {
        set_err(nullptr, "asd_rectify: %s", cudaGetErrorString(cudaGetLastError()));
        return ASD_E_CUDA;
    }
    return ASD_OK;
}

int asd_sensor_noise(const asd_noise* q, uint64_t seed, int n, int width, int height,
                     uint32_t frame0, uint32_t view, const float* clean, uint8_t* out, void* cuda_stream)
{
    if (!q || n < 0 || (n > 0 && (!clean || !out)) || width < 1 || height < 1 ||
        (long long)width * height > (1ll << 26) || n > 65535) {
        set_err(nullptr, "asd_sensor_noise: NULL argument or size out of range");
        return ASD_E_INVALID_ARG;
    }
    if (!(std::isfinite(q->k) && q->k > 0.0 && std::isfinite(q->theta) && q->theta > 0.0 &&
          std::isfinite(q->mu) && std::isfinite(q->sigma) && q->sigma >= 0.0 && std::isfinite(q->scale))) {
        set_err(nullptr, "asd_sensor_noise: need finite k, theta > 0, sigma >= 0, mu, scale");
        return ASD_E_INVALID_ARG;
    }
    if (n == 0) return ASD_OK;
    if (launch_noise(q, seed, n, width, height, frame0, view, clean, out, (cudaStream_t)cuda_stream) != 0) {
        set_err(nullptr, "asd_sensor_noise: %s", cudaGetErrorString(cudaGetLastError()));
        return ASD_E_CUDA;
    }
    return ASD_OK;
}

int asd_register_depth(const asd_camera* ir, const asd_camera* rgb, const float* R, const float* t,
                       int n, const float* depth, float* out, void* cuda_stream)
{
    if (!ir || !rgb || !R || !t || n < 0 || (n > 0 && (!depth || !out))) {
        set_err(nullptr, "asd_register_depth: NULL argument or n < 0");
        return ASD_E_INVALID_ARG;
    }
    auto cam_ok = [](const asd_camera* c) {
        return c->width > 0 && c->height > 0 && (long long)c->width * c->height <= (1ll << 26) &&
               std::isfinite(c->fx) && std::isfinite(c->fy) && c->fx > 0.0f && c->fy > 0.0f &&
               std::isfinite(c->cx) && std::isfinite(c->cy);
    };
    if (!cam_ok(ir) || !cam_ok(rgb)) {
        set_err(nullptr, "asd_register_depth: camera sizes / intrinsics out of range");
        return ASD_E_INVALID_ARG;
    }
    for (int i = 0; i < 9; ++i) if (!std::isfinite(R[i])) { set_err(nullptr, "R not finite"); return ASD_E_INVALID_ARG; }
    for (int i = 0; i < 3; ++i) if (!std::isfinite(t[i])) { set_err(nullptr, "t not finite"); return ASD_E_INVALID_ARG; }
    if (n == 0) return ASD_OK;
    if (launch_register(ir, rgb, R, t, n, depth, out, (cudaStream_t)cuda_stream) != 0) {
        set_err(nullptr, "asd_register_depth: %s", cudaGetErrorString(cudaGetLastError()));
        return ASD_E_CUDA;
    }
    return ASD_OK;
}

int asd_profile_begin(asd_ctx* ctx, int max_launches)
{
    if (!ctx || max_launches < 1 || max_launches > (1 << 20)) {
        set_err(ctx, "asd_profile_begin: bad arguments");
        return ASD_E_INVALID_ARG;
    }
    DeviceGuard g(ctx->device);
    for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
    ctx->prof_ev.assign(2 * (size_t)max_launches, nullptr);
    for (auto& e : ctx->prof_ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            set_err(ctx, "cudaEventCreate failed");
            return ASD_E_CUDA;
        }
    ctx->prof_marks.clear();
    ctx->prof_marks.reserve(max_launches);
    ctx->prof_dropped = 0;
    ctx->prof = true;
    return ASD_OK;
}

int asd_profile_timeline(asd_ctx* ctx, int max, int32_t* stage, float* t_start_ms, float* t_end_ms)
{
    if (!ctx || max < 0 || (max > 0 && (!stage || !t_start_ms || !t_end_ms))) {
        set_err(ctx, "asd_profile_timeline: bad arguments");
        return ASD_E_INVALID_ARG;
    }
    DeviceGuard g(ctx->device);
    const int k = (int)ctx->prof_marks.size() < max ? (int)ctx->prof_marks.size() : max;
    for (int i = 0; i < k; ++i) {
        float a = 0.0f, b = 0.0f;
        if (cudaEventSynchronize(ctx->prof_ev[2 * i + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&a, ctx->prof_ev[0], ctx->prof_ev[2 * i]) != cudaSuccess ||
            cudaEventElapsedTime(&b, ctx->prof_ev[0], ctx->prof_ev[2 * i + 1]) != cudaSuccess) {
            set_err(ctx, "event timing failed: %s", cudaGetErrorString(cudaGetLastError()));
            return ASD_E_CUDA;
        }
        stage[i] = ctx->prof_marks[i].stage;
        t_start_ms[i] = a;
        t_end_ms[i] = b;
    }
    return k;
}

int asd_profile_end(asd_ctx* ctx, asd_stage_times* out)
{
    if (!ctx || !out) { set_err(ctx, "asd_profile_end: NULL argument"); return ASD_E_INVALID_ARG; }
    DeviceGuard g(ctx->device);
    std::memset(out, 0, sizeof *out);
    ctx->prof = false;
    for (size_t k = 0; k < ctx->prof_marks.size(); ++k) {
        float ms = 0.0f;
        if (cudaEventSynchronize(ctx->prof_ev[2 * k + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&ms, ctx->prof_ev[2 * k], ctx->prof_ev[2 * k + 1]) != cudaSuccess) {
            set_err(ctx, "event timing failed: %s", cudaGetErrorString(cudaGetLastError()));
            return ASD_E_CUDA;
        }
        const int st = ctx->prof_marks[k].stage;
        out->ms[st] += ms;
        out->alg_bytes[st] += ctx->prof_marks[k].bytes;
        out->alg_ops[st] += ctx->prof_marks[k].ops;
        out->launches[st] += 1;
    }
    out->dropped = ctx->prof_dropped;
    ctx->prof_marks.clear();
    return ASD_OK;
}

}  // extern "C"
