// common.cuh -- device-side parameter block and small helpers shared by the
// sm_100a kernels of libasd (product code; shares nothing with oracle/).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace asd {

// Everything the kernels need, derived once on the host from asd_params.
struct DevParams {
    int W, H;          // image size
    int min_disp, D;   // delta(d) = min_disp + d, d in [0, D)
    int cw, ch;        // census window
    int R, Q;          // half window: R = cw/2, Q = ch/2
    int nb;            // CSCT bits = floor(cw*ch/2)
    int p1, p2;        // SGM penalties
    int paths;         // 4 or 8
    int uniq;          // uniqueness percent, < 0 off
    float lr;          // LR max diff, < 0 off
    int subpix;        // 0/1
    float fb;          // focal_px * baseline_m rounded once to fp32
    long long npx;     // W*H
    long long ncell;   // W*H*D
    int bw, bh;        // SGBM block (1 x 1 = SGM)
    int median;        // median ksize: 0 (off), 3, 5
    int lr_mode;       // right view: 0 = R1 re-index (c10), 1 = R2 own SGM (c24)
};

constexpr uint8_t MASK_BORDER = 1, MASK_UNIQUE = 2, MASK_LR = 4, MASK_NONPOS = 8;
constexpr unsigned FULL = 0xffffffffu;

// valid_c(x,y): the census window around (x,y) lies inside the image (reading c4).
__device__ __forceinline__ bool census_valid(const DevParams& p, int x, int y) {
    return x >= p.R && x < p.W - p.R && y >= p.Q && y < p.H - p.Q;
}

__device__ __forceinline__ int popc_sig(uint32_t v) { return __popc(v); }
__device__ __forceinline__ int popc_sig(unsigned long long v) { return __popcll(v); }

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16;
    return h;
}

// Checked builds (-DASD_CHECKED, tools/checked.sh; never the production
// library): ASD_ASSERT traps on a violated index invariant, and ASD_JITTER
// puts a pseudo-random __nanosleep (up to ~1 us, one warp in four per site) at
// the synchronisation points of the pipelined kernels, so that a missing
// barrier, fence or mbarrier wait shows up as an oracle mismatch in repeated
// runs (compute-sanitizer is not available on the GPU pool).
#ifdef ASD_CHECKED
#define ASD_ASSERT(c)                                                                      \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("ASD_ASSERT %s failed at %s:%d block (%d,%d) thread %d\n", #c, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);          \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
__device__ __forceinline__ void asd_jitter(unsigned site)
{
    unsigned h = (unsigned)clock64() ^ (site * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^
                 (blockIdx.y * 0xC2B2AE35u) ^ ((threadIdx.x >> 5) * 0x27D4EB2Fu);
    h ^= h >> 16; h *= 0x7FEB352Du; h ^= h >> 15;
    if ((h & 3) == 0) __nanosleep(h >> 22);
}
#define ASD_JITTER(site) asd_jitter(site)
#else
#define ASD_ASSERT(c) ((void)0)
#define ASD_JITTER(site) ((void)0)
#endif

// Per-frame pointers of one in-flight frame slot.
struct FrameScratch {
    void*     census_l;   // [H][W] u32 | u64
    void*     census_r;
    uint16_t* S;          // [H][W][D] aggregated cost
    float*    dl;         // [H][W]
    float*    dr;
    int16_t*  dstar_l;
    int16_t*  dstar_r;
    uint8_t*  mask_l;
    uint8_t*  mask_r;
};

}  // namespace asd
