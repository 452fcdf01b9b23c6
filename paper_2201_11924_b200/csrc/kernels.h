// kernels.h -- host-side launchers of the sm_100a kernels (internal to libasd).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "asd.h"
#include "common.cuh"

namespace asd {

// K1 census, both views of nframes frames.
void launch_census(const DevParams& p, int nframes, const uint8_t* left, const uint8_t* right,
                   long long img_stride, void* out_l, void* out_r, long long sig_stride,
                   cudaStream_t s);

// K2/K3 one SGM direction (design D1); first = write S instead of accumulate.
int num_chains(const DevParams& p, int rx, int ry);
// cv != nullptr: read the matching cost from that u16 [H][W][D] volume (SGBM)
// instead of recomputing it from the census images.
// right_ref: the right view is the reference (R2, reading c24).
bool launch_sgm_dir(const DevParams& p, int nframes, int rx, int ry, bool first,
                    const void* cl, const void* cr, long long sig_stride,
                    uint16_t* S, long long s_stride, cudaStream_t s,
                    const uint16_t* cv = nullptr, bool right_ref = false);

// Depth registration (register.cu): fill, scatter with an atomicMin z-buffer, finish.
int launch_register(const asd_camera* ir, const asd_camera* rgb, const float* R, const float* t,
                    int n, const float* depth, float* out, cudaStream_t s);

// Homography rectification (rectify.cu).
int launch_rectify(const double* Hm, int n, int W, int H, const uint8_t* in, uint8_t* out, cudaStream_t s);

// Sensor noise front end (noise.cu).
int launch_noise(const asd_noise* q, uint64_t seed, int n, int width, int height, uint32_t frame0,
                 uint32_t view, const float* clean, uint8_t* out, cudaStream_t s);

// SGBM block cost volume CB (u16 [H][W][D] per frame), sgbm.cu.
// priv_wpad > 0: write the D3 sweeps' private layout (D = 128, rows of
// priv_wpad columns; cell_stride = the frame stride of that layout).
void launch_block_cost(const DevParams& p, int nframes, const void* cl, const void* cr,
                       long long sig_stride, uint16_t* cb, long long cell_stride, cudaStream_t s,
                       bool right_ref = false, int priv_wpad = 0);

// K4 WTA/uniqueness/sub-pixel, left + right view.
// SR != nullptr: the right view is the WTA of its own aggregate SR (R2, c24).
bool launch_wta(const DevParams& p, int nframes, const uint16_t* S, long long s_stride,
                const FrameScratch& fs, long long px_stride, cudaStream_t s, const uint16_t* SR = nullptr);

// K5 LR check + depth + per-frame stats.
void launch_lr_depth(const DevParams& p, int nframes, const FrameScratch& fs, long long px_stride,
                     float* out_disp, float* out_depth, long long out_stride, uint8_t* mask_out,
                     asd_frame_stats* stats, cudaStream_t s);

// Design D3 (sgm_v2.cu): grouped sweeps.  v2_plan checks the envelope and
// picks the cluster geometry; launch_v2_stage(0 = down, 1 = up, 2 = row).
struct V2Plan {
    bool ok;
    int DC, T, NP, cs, w, vthreads, active_ctas;
    size_t vsmem, vsmem_up;
    int DPL, nbuf, bstride;
    size_t rsmem;
    bool wide;        // WTA keys in u32 (S may exceed 2^(16 - log2 D))
    bool blk;         // u16-partial instances on a cost buffer (SGBM block cost, or SGM with 3(nb+P2) > 255)
    bool wta_fb;      // WTA by the warp-per-pixel kernel (the ring window does not fit)
    bool halves;      // D = 256 (R1): wta_halves_kernel, three passes over half-width windows
    bool tma_cen;     // K_down stages census rows with TMA bulk copies (needs guarded census buffers)
    int ncta;         // sweep CTAs per frame: cs (one cluster) or nseg * cs (frame wider than a cluster)
    unsigned long long* ghalo;   // segment-boundary tagged halos (owned by the context; nseg > 1)
    char why[128];
};
bool v2_plan(const DevParams& p, int device, V2Plan& pl);
// The ring-window WTA kernel alone (also used by engine D1 when D is 16..128):
// fills nbuf / bstride / rsmem / wide; false if the window does not fit.
bool wta2_plan(const DevParams& p, bool wide, V2Plan& pl, bool halves_ok = false);
// device bytes of the segment-boundary halos for nframes frames (0 if nseg == 1)
size_t v2_ghalo_bytes(const V2Plan& pl, int nframes);
void launch_wta2(const DevParams& p, const V2Plan& pl, int nframes, const uint16_t* S, long long cell_stride,
                 const FrameScratch& fs, long long px_stride, cudaStream_t s);
// variant: stage 0 -> 1 = right-referenced K_down (R2); stage 2 -> 1 = cost
// from the P_AB | C words; stage 3 -> WTA mode (0 both views, 1 left only,
// 2 left view written to the right-view maps).
int launch_v2_stage(int stage, const DevParams& p, const V2Plan& pl, int nframes,
                    const void* cl, const void* cr, long long sig_stride,
                    uint8_t* pa, uint16_t* pab, uint8_t* stash, long long cell_stride,
                    const FrameScratch& fs, long long px_stride, uint16_t* agg, cudaStream_t s,
                    int variant = 0, const uint16_t* cbin = nullptr);

// Debug: materialise the raw cost volume C [H][W][D] u8 from the census images.
void launch_cost_volume(const DevParams& p, const void* cl, const void* cr, uint8_t* cost,
                        cudaStream_t s);

}  // namespace asd
