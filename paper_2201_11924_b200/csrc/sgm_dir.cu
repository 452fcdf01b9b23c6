// sgm_dir.cu -- K2/K3 (design D1): one semi-global path direction per launch,
// warp per scanline.  PAPER.md P:289 ("four-path semi-global matching (SGM)
// ... with hamming distance as the cost function"), P:291 ("cost aggregation
// of SGM is further accelerated with warp-based optimization").  Recursion
// (reading c6):
//   L_r(p,d) = C(p,d) + min(L_r(p-r,d), L_r(p-r,d-1)+P1, L_r(p-r,d+1)+P1, M+P2) - M,
//   M = min_k L_r(p-r,k);  L_r = C at the first pixel of a line.
// S = sum_r L_r accumulates in a u16 [H][W][D] volume: the first direction
// writes it, the others read-modify-write it.
//
// Work mapping: one warp walks one line of direction r; the D disparities of
// the current pixel live in the warp's registers (DPL per lane, contiguous),
// d-1 / d+1 neighbours at lane edges come from __shfl_up/down_sync and M from
// __reduce_min_sync.  The matching cost (PAPER P:289 Hamming distance,
// SPEC S:300, reading c3) is recomputed from the census images on the fly:
//   C = popc(cl(x,y) ^ cr(x-delta,y)) if both windows are valid, else nb.
// The next pixel's census word and S vector are prefetched one step ahead.
// SGBM (CV = true): the cost is read from the block-cost volume CB (sgbm.cu,
// PAPER.md P:291, reading c19) instead of the census images.
#include "common.cuh"
#include "kernels.h"

namespace asd {

constexpr int SGM_INF = 1 << 20;

__device__ __forceinline__ void chain_start(const DevParams& p, int rx, int ry, int k, int& x, int& y)
{
    if (ry == 0) { y = k; x = rx > 0 ? 0 : p.W - 1; return; }
    if (rx == 0) { x = k; y = ry > 0 ? 0 : p.H - 1; return; }
    if (k < p.W) { x = k; y = ry > 0 ? 0 : p.H - 1; return; }
    const int j = k - p.W + 1;                 // 1 .. H-1
    x = rx > 0 ? 0 : p.W - 1;
    y = ry > 0 ? j : p.H - 1 - j;
}

int num_chains(const DevParams& p, int rx, int ry)
{
    if (ry == 0) return p.H;
    if (rx == 0) return p.W;
    return p.W + p.H - 1;
}

template <int DPL>
__device__ __forceinline__ void load_s(const uint16_t* src, int (&v)[DPL])
{
#pragma unroll
    for (int j = 0; j < DPL; ++j) v[j] = src[j];
}
template <> __device__ __forceinline__ void load_s<4>(const uint16_t* src, int (&v)[4])
{
    uint2 u = *reinterpret_cast<const uint2*>(src);
    v[0] = u.x & 0xffff; v[1] = u.x >> 16; v[2] = u.y & 0xffff; v[3] = u.y >> 16;
}
template <> __device__ __forceinline__ void load_s<8>(const uint16_t* src, int (&v)[8])
{
    uint4 u = *reinterpret_cast<const uint4*>(src);
    v[0] = u.x & 0xffff; v[1] = u.x >> 16; v[2] = u.y & 0xffff; v[3] = u.y >> 16;
    v[4] = u.z & 0xffff; v[5] = u.z >> 16; v[6] = u.w & 0xffff; v[7] = u.w >> 16;
}
template <int DPL>
__device__ __forceinline__ void store_s(uint16_t* dst, const int (&v)[DPL])
{
#pragma unroll
    for (int j = 0; j < DPL; ++j) dst[j] = (uint16_t)v[j];
}
template <> __device__ __forceinline__ void store_s<4>(uint16_t* dst, const int (&v)[4])
{
    *reinterpret_cast<uint2*>(dst) = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
}
template <> __device__ __forceinline__ void store_s<8>(uint16_t* dst, const int (&v)[8])
{
    *reinterpret_cast<uint4*>(dst) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16),
                                                v[4] | (v[5] << 16), v[6] | (v[7] << 16));
}

// MODE 0: cost from census, left view as reference (C = popc(cl(x) ^ cr(x - delta)));
// MODE 1: right view as reference (R2, reading c24: popc(cr(x) ^ cl(x + delta)));
// MODE 2: cost read from a u16 volume (SGBM block cost, either reference).
template <int DPL, typename SigT, bool FIRST, int MODE>
__global__ void __launch_bounds__(128)
sgm_dir_kernel(DevParams p, int rx, int ry, int nchains, int act,
               const SigT* __restrict__ cl_base, const SigT* __restrict__ cr_base, long long sig_stride,
               uint16_t* __restrict__ S_base, long long s_stride, const uint16_t* __restrict__ cv_base)
{
    const int chain = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (chain >= nchains) return;
    const int frame = blockIdx.y;
    constexpr bool CV = MODE == 2, RR = MODE == 1;
    // reference / matched census (swapped for the right-view reference)
    const SigT* cl = (RR ? cr_base : cl_base) + frame * sig_stride;
    const SigT* cr = (RR ? cl_base : cr_base) + frame * sig_stride;
    uint16_t* S = S_base + frame * s_stride;
    const uint16_t* CVf = CV ? cv_base + frame * s_stride : nullptr;
    const bool active = lane < act;
    const int d0 = lane * DPL;

    int x, y;
    chain_start(p, rx, ry, chain, x, y);

    int L[DPL];
    int M = 0;
    bool first = true;
    // prefetch state for the current pixel
    SigT nl = CV ? (SigT)0 : cl[(long long)y * p.W + x];
    SigT nr[DPL];
    int ns[DPL], nc[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
        const int xr = RR ? x + p.min_disp + d0 + j : x - p.min_disp - d0 - j;
        nr[j] = (!CV && active && xr >= 0 && xr < p.W) ? cr[(long long)y * p.W + xr] : (SigT)0;
        ns[j] = 0;
        nc[j] = 0;
    }
    if (!FIRST && active) load_s<DPL>(S + ((long long)y * p.W + x) * p.D + d0, ns);
    if (CV && active) load_s<DPL>(CVf + ((long long)y * p.W + x) * p.D + d0, nc);

    while (true) {
        const SigT sl = nl;
        SigT sr[DPL];
        int sv[DPL], sc[DPL];
#pragma unroll
        for (int j = 0; j < DPL; ++j) { sr[j] = nr[j]; sv[j] = ns[j]; sc[j] = nc[j]; }
        const int cx = x, cy = y;
        const bool vl = census_valid(p, cx, cy);
        x += rx; y += ry;
        const bool more = x >= 0 && x < p.W && y >= 0 && y < p.H;
        if (more) {                       // prefetch the next pixel of the line
            if (!CV) {
                nl = cl[(long long)y * p.W + x];
#pragma unroll
                for (int j = 0; j < DPL; ++j) {
                    const int xr = RR ? x + p.min_disp + d0 + j : x - p.min_disp - d0 - j;
                    nr[j] = (active && xr >= 0 && xr < p.W) ? cr[(long long)y * p.W + xr] : (SigT)0;
                }
            }
            if (!FIRST && active) load_s<DPL>(S + ((long long)y * p.W + x) * p.D + d0, ns);
            if (CV && active) load_s<DPL>(CVf + ((long long)y * p.W + x) * p.D + d0, nc);
        }
        // matching cost of the current pixel
        int c[DPL];
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const int xr = RR ? cx + p.min_disp + d0 + j : cx - p.min_disp - d0 - j;
            const bool vm = RR ? xr < p.W - p.R : xr >= p.R;    // matched census window valid
            c[j] = CV ? sc[j] : ((vl && vm) ? popc_sig(sl ^ sr[j]) : p.nb);
        }
        int Ln[DPL];
        if (first) {
#pragma unroll
            for (int j = 0; j < DPL; ++j) Ln[j] = c[j];
            first = false;
        } else {
            int left = __shfl_up_sync(FULL, L[DPL - 1], 1);
            int right = __shfl_down_sync(FULL, L[0], 1);
            if (lane == 0) left = SGM_INF;
            if (lane == act - 1) right = SGM_INF;
            const int mp2 = M + p.p2;
#pragma unroll
            for (int j = 0; j < DPL; ++j) {
                const int lm = j == 0 ? left : L[j - 1];
                const int rm = j == DPL - 1 ? right : L[j + 1];
                int t = min(L[j], min(lm, rm) + p.p1);
                t = min(t, mp2);
                Ln[j] = c[j] + t - M;
            }
        }
        int lmin = SGM_INF;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            if (!active) Ln[j] = SGM_INF;
            L[j] = Ln[j];
            lmin = min(lmin, Ln[j]);
        }
        if (active) {
            int out[DPL];
#pragma unroll
            for (int j = 0; j < DPL; ++j) out[j] = FIRST ? Ln[j] : sv[j] + Ln[j];
            store_s<DPL>(S + ((long long)cy * p.W + cx) * p.D + d0, out);
        }
        M = (int)__reduce_min_sync(FULL, (unsigned)lmin);
        if (!more) break;
    }
}

template <int DPL, typename SigT>
static void launch_dir_t(const DevParams& p, int nframes, int rx, int ry, bool first, int act,
                         const void* cl, const void* cr, long long sig_stride,
                         uint16_t* S, long long s_stride, cudaStream_t s, const uint16_t* cv, bool right_ref)
{
    const int n = num_chains(p, rx, ry);
    dim3 grid((n + 3) / 4, nframes), block(128);
    const SigT* l = (const SigT*)cl;
    const SigT* r = (const SigT*)cr;
#define ASD_DIR_LAUNCH(M) \
    if (first) sgm_dir_kernel<DPL, SigT, true, M><<<grid, block, 0, s>>>(p, rx, ry, n, act, l, r, sig_stride, S, s_stride, cv); \
    else sgm_dir_kernel<DPL, SigT, false, M><<<grid, block, 0, s>>>(p, rx, ry, n, act, l, r, sig_stride, S, s_stride, cv);
    if (cv) { ASD_DIR_LAUNCH(2) }
    else if (right_ref) { ASD_DIR_LAUNCH(1) }
    else { ASD_DIR_LAUNCH(0) }
#undef ASD_DIR_LAUNCH
}

template <typename SigT>
static bool launch_dir_sig(const DevParams& p, int nframes, int rx, int ry, bool first,
                           const void* cl, const void* cr, long long sig_stride,
                           uint16_t* S, long long s_stride, cudaStream_t s, const uint16_t* cv, bool right_ref)
{
    // D = DPL * act with act = 32 (D % 32 == 0) or 16 (D % 32 == 16)
    const int act = (p.D % 32 == 0) ? 32 : 16;
    const int dpl = p.D / act;
#define ASD_DIR_CASE(K) case K: launch_dir_t<K, SigT>(p, nframes, rx, ry, first, act, cl, cr, sig_stride, S, s_stride, s, cv, right_ref); return true;
    switch (dpl) {
        ASD_DIR_CASE(1) ASD_DIR_CASE(2) ASD_DIR_CASE(3) ASD_DIR_CASE(4) ASD_DIR_CASE(5)
        ASD_DIR_CASE(6) ASD_DIR_CASE(7) ASD_DIR_CASE(8) ASD_DIR_CASE(9) ASD_DIR_CASE(11)
        ASD_DIR_CASE(13) ASD_DIR_CASE(15)
        default: return false;
    }
#undef ASD_DIR_CASE
}

bool launch_sgm_dir(const DevParams& p, int nframes, int rx, int ry, bool first,
                    const void* cl, const void* cr, long long sig_stride,
                    uint16_t* S, long long s_stride, cudaStream_t s, const uint16_t* cv, bool right_ref)
{
    if (p.nb <= 32)
        return launch_dir_sig<uint32_t>(p, nframes, rx, ry, first, cl, cr, sig_stride, S, s_stride, s, cv, right_ref);
    return launch_dir_sig<unsigned long long>(p, nframes, rx, ry, first, cl, cr, sig_stride, S, s_stride, s, cv, right_ref);
}

}  // namespace asd
