// sgbm.cu -- SGBM block matching cost.  PAPER.md P:291:
// "Besides the original SGM, SimSense also supports semi-global block
// matching (SGBM) ... SGBM computes the cost by the hamming distance between
// the local regions of the two pixels"; SPEC S:300 ("for SGBM, sum of hamming
// over the block around both pixels"), reading c19:
//   CB(x,y,d) = sum_{|u| <= bw/2, |v| <= bh/2} C~(x+u, y+v, d),
//   C~ = popc(cl(x',y') ^ cr(x'-delta,y')) when both census windows are valid
//        and x'-delta >= 0, else nb; nb for block positions off the image.
// The volume (u16 [H][W][D]) feeds the D1 direction kernels (sgm_dir.cu, CV
// mode) in place of the per-pixel Hamming cost.
//
// Layout: thread = disparity, CTA = a TX x SB_RY pixel tile of one frame (see
// block_cost_kernel): each Hamming distance once per CTA, horizontal window
// sums per row, vertical sums slid down the tile's rows.
#include "common.cuh"
#include "kernels.h"

namespace asd {

#ifndef ASD_BC_RY
#define ASD_BC_RY 32              // rows per CTA (16: 1285, 8: 1259 frames/s SGBM 3x3)
#endif
constexpr int SB_RY = ASD_BC_RY;     // rows per CTA (the block sum slides down them)

// RR: the right view is the reference (R2, reading c24): cl_base / cr_base are
// then the reference and matched census and the matched column is x' + delta.
//
// One CTA = TX pixels x SB_RY rows of one frame, thread = disparity
// (blockDim = D).  The block sum slides down the rows: CB(y+1) = CB(y) +
// H(y+1+bv) - H(y-bv), where H(y') are the horizontal block sums of row y'
// for the TX pixels.  The last bh rows of H sit in a shared-memory ring
// ([bh][TX][D] u16, each thread touching only its own d), CB in registers;
// each new row's census spans are staged in shared memory, so each (column,
// row, d) Hamming distance is evaluated once per CTA instead of bh times.
// PRIV: write CB in the D3 sweeps' private layout (D = 128: pixel x, disparity
// d = 32 chunk + 16 half + 4 q + j at u16 (x & ~7) * D + (32 q + 4 (x & 7) +
// chunk) * 8 + 2 j + half of a row of wpad columns) instead of [H][W][D].
// BW > 0: the block width as a compile-time constant: the horizontal window
// then lives in registers (fully unrolled over the TX + BW - 1 block columns)
// and invalid census words carry bit 31 (MARK; needs nb <= 31) instead of
// separate validity flags.  BW == 0: the generic form.
#ifndef ASD_BC_MINB
#define ASD_BC_MINB 1             // min resident CTAs (of D threads) per SM for the block cost kernel
#endif
#ifndef ASD_BC_TX
#define ASD_BC_TX 16              // pixels per CTA row (the CB accumulators per thread; 32: 1162 vs 1275 frames/s SGBM 3x3)
#endif
template <typename SigT, bool RR, int TX, bool PRIV, int BW = 0>
__global__ void __launch_bounds__(256, ASD_BC_MINB)
block_cost_kernel(DevParams p, const SigT* __restrict__ cl_base, const SigT* __restrict__ cr_base,
                  long long sig_stride, uint16_t* __restrict__ cb_base, long long cell_stride, int wpad)
{
    constexpr bool MARK = BW > 0;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = p.W, H = p.H, D = p.D;
    const int bu = p.bw / 2, bv = p.bh / 2;
    const int frame = blockIdx.z, y0 = blockIdx.y * SB_RY, x0 = blockIdx.x * TX;
    const int y1 = min(H, y0 + SB_RY);
    const int NC = TX + p.bw - 1;                    // block columns x0-bu .. x0+TX-1+bu
    const int NRW = NC + D - 1;                      // matched span: x' -/+ (min + d)
    const int xr0 = RR ? x0 - bu + p.min_disp                 // first matched column
                       : x0 - bu - p.min_disp - (D - 1);
    const SigT* cl = cl_base + frame * sig_stride;
    const SigT* cr = cr_base + frame * sig_stride;
    const int d = threadIdx.x;                       // blockDim.x == D

    const int NY = (y1 - y0) + p.bh - 1;             // census rows y0 - bv .. y1 - 1 + bv
    SigT* Ls = reinterpret_cast<SigT*>(sm_raw);                            // [NY][NC]
    SigT* Rs = Ls + (size_t)NY * NC;                                        // [NY][NRW]
    uint16_t* Hr = reinterpret_cast<uint16_t*>(Rs + (size_t)NY * NRW);      // [bh][TX][D]
    uint16_t* Cc = Hr + (size_t)p.bh * TX * D;                              // [NC][D]
    unsigned char* Lv = reinterpret_cast<unsigned char*>(Cc + (size_t)NC * D);   // [NY][NC]
    unsigned char* Rv = Lv + (size_t)NY * NC;                                     // [NY][NRW]
    // stage every census row the tile needs once
    for (int i = threadIdx.x; i < NY * NC; i += blockDim.x) {
        const int r = i / NC, c = i - r * NC;
        const int xx = x0 - bu + c, yy = y0 - bv + r;
        const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W && census_valid(p, xx, yy);
        Ls[i] = ok ? cl[(long long)yy * W + xx] : (MARK ? (SigT)0x80000000u : (SigT)0);
        Lv[i] = ok;
    }
    for (int i = threadIdx.x; i < NY * NRW; i += blockDim.x) {
        const int r = i / NRW, c = i - r * NRW;
        const int xr = xr0 + c, yy = y0 - bv + r;
        const bool ok = yy >= 0 && yy < H && xr >= 0 && xr < W && census_valid(p, xr, yy);
        Rs[i] = ok ? cr[(long long)yy * W + xr] : (MARK ? (SigT)0x80000000u : (SigT)0);
        Rv[i] = ok;
    }
    __syncthreads();

    // H of image row yy into ring slot `slot` (this thread's d only: no syncs)
    auto hrow = [&](int yy, int slot) {
        const int r = yy - (y0 - bv);
        const SigT* L = Ls + (size_t)r * NC;
        const SigT* R = Rs + (size_t)r * NRW;
        const unsigned char* lv = Lv + (size_t)r * NC;
        const unsigned char* rv = Rv + (size_t)r * NRW;
        uint32_t run = 0;
        if constexpr (BW > 0) {                      // register window, marked census words
            const SigT* Rd = R + (RR ? d : (D - 1) - d);
            const uint32_t nbv = (uint32_t)p.nb;
            uint32_t win[BW];
#pragma unroll
            for (int c = 0; c < TX + BW - 1; ++c) {
                const uint32_t l = (uint32_t)L[c], r2 = (uint32_t)Rd[c];
                const uint32_t cv = ((l | r2) & 0x80000000u) ? nbv : (uint32_t)__popc(l ^ r2);
                run += cv;
                if (c >= BW) run -= win[c % BW];
                win[c % BW] = cv;
                if (c + 1 >= BW) Hr[((size_t)slot * TX + (c + 1 - BW)) * D + d] = (uint16_t)run;
            }
        } else {
            for (int c = 0; c < NC; ++c) {          // window sums over bw block columns
                const int rc = RR ? c + d : c + (D - 1) - d;
                const uint32_t cv = (lv[c] && rv[rc]) ? (uint32_t)popc_sig(L[c] ^ R[rc]) : (uint32_t)p.nb;
                Cc[(size_t)c * D + d] = (uint16_t)cv;
                run += cv;
                if (c >= p.bw) run -= Cc[(size_t)(c - p.bw) * D + d];
                if (c + 1 >= p.bw) Hr[((size_t)slot * TX + (c + 1 - p.bw)) * D + d] = (uint16_t)run;
            }
        }
    };
    uint32_t cb[TX];
#pragma unroll
    for (int i = 0; i < TX; ++i) cb[i] = 0;
    auto add_slot = [&](int slot, bool sub) {
#pragma unroll
        for (int i = 0; i < TX; ++i) {
            const uint32_t v = Hr[((size_t)slot * TX + i) * D + d];
            cb[i] = sub ? cb[i] - v : cb[i] + v;
        }
    };
    auto write_row = [&](int y) {
        if constexpr (PRIV) {
            const int r = d & 31;
            const int dpart = (32 * ((r & 15) >> 2) + (d >> 5)) * 8 + 2 * (r & 3) + (r >> 4);
            uint16_t* out = cb_base + frame * cell_stride + (long long)y * wpad * D + dpart;
#pragma unroll
            for (int i = 0; i < TX; ++i) {
                const int x = x0 + i;
                if (x < W) out[(long long)(x & ~7) * D + 32 * (x & 7)] = (uint16_t)cb[i];
            }
        } else {
            uint16_t* out = cb_base + frame * cell_stride + ((long long)y * W + x0) * D + d;
#pragma unroll
            for (int i = 0; i < TX; ++i)
                if (x0 + i < W) out[(long long)i * D] = (uint16_t)cb[i];
        }
    };
    for (int v = 0; v < p.bh; ++v) {                 // rows y0 - bv .. y0 + bv -> slots 0 .. bh-1
        hrow(y0 - bv + v, v);
        add_slot(v, false);
    }
    write_row(y0);
    for (int y = y0 + 1; y < y1; ++y) {
        const int slot = (y - 1 - y0) % p.bh;        // holds row y - 1 - bv, leaving the window
        add_slot(slot, true);
        hrow(y + bv, slot);
        add_slot(slot, false);
        write_row(y);
    }
}

template <int TX>
static size_t block_cost_smem(const DevParams& p, size_t sig)
{
    const size_t NC = TX + p.bw - 1, NRW = NC + p.D - 1, NY = SB_RY + p.bh - 1;
    size_t b = NY * (NC + NRW) * (sig + 1) + (size_t)p.bh * TX * p.D * 2 + NC * p.D * 2;
    return (b + 15) & ~size_t(15);
}

template <typename SigT, bool RR, int TX, bool PRIV, int BW>
static void launch_bc_k(const DevParams& p, dim3 grid, size_t sm, const void* ref, const void* mat,
                        long long sig_stride, uint16_t* cb, long long cell_stride, int wpad, cudaStream_t s)
{
    cudaFuncSetAttribute((const void*)block_cost_kernel<SigT, RR, TX, PRIV, BW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    block_cost_kernel<SigT, RR, TX, PRIV, BW><<<grid, p.D, sm, s>>>(p, (const SigT*)ref, (const SigT*)mat,
                                                                    sig_stride, cb, cell_stride, wpad);
}

template <typename SigT, bool RR, int TX, bool PRIV>
static bool launch_bc(const DevParams& p, int nframes, const void* ref, const void* mat,
                      long long sig_stride, uint16_t* cb, long long cell_stride, int wpad, cudaStream_t s)
{
    const size_t sm = block_cost_smem<TX>(p, sizeof(SigT));
    if (sm > 200 * 1024) return false;
    dim3 grid((p.W + TX - 1) / TX, (p.H + SB_RY - 1) / SB_RY, nframes);
    const bool mark = sizeof(SigT) == 4 && p.nb <= 31;      // bit 31 free for the invalid marker
    if (mark && p.bw == 3) launch_bc_k<SigT, RR, TX, PRIV, 3>(p, grid, sm, ref, mat, sig_stride, cb, cell_stride, wpad, s);
    else if (mark && p.bw == 5) launch_bc_k<SigT, RR, TX, PRIV, 5>(p, grid, sm, ref, mat, sig_stride, cb, cell_stride, wpad, s);
    else if (mark && p.bw == 7) launch_bc_k<SigT, RR, TX, PRIV, 7>(p, grid, sm, ref, mat, sig_stride, cb, cell_stride, wpad, s);
    else launch_bc_k<SigT, RR, TX, PRIV, 0>(p, grid, sm, ref, mat, sig_stride, cb, cell_stride, wpad, s);
    return true;
}

template <typename SigT, bool RR, bool PRIV>
static void launch_bc_tx(const DevParams& p, int nframes, const void* ref, const void* mat,
                         long long sig_stride, uint16_t* cb, long long cell_stride, int wpad, cudaStream_t s)
{
    if (!launch_bc<SigT, RR, ASD_BC_TX, PRIV>(p, nframes, ref, mat, sig_stride, cb, cell_stride, wpad, s))
        launch_bc<SigT, RR, 8, PRIV>(p, nframes, ref, mat, sig_stride, cb, cell_stride, wpad, s);
}

void launch_block_cost(const DevParams& p, int nframes, const void* cl, const void* cr,
                       long long sig_stride, uint16_t* cb, long long cell_stride, cudaStream_t s,
                       bool right_ref, int priv_wpad)
{
    const void* ref = right_ref ? cr : cl;
    const void* mat = right_ref ? cl : cr;
    const int wp = priv_wpad;
    if (p.nb > 32) {                                  // (D3 needs nb <= 32: never private)
        if (right_ref) launch_bc_tx<unsigned long long, true, false>(p, nframes, ref, mat, sig_stride, cb, cell_stride, 0, s);
        else launch_bc_tx<unsigned long long, false, false>(p, nframes, ref, mat, sig_stride, cb, cell_stride, 0, s);
    } else if (wp > 0) {
        if (right_ref) launch_bc_tx<uint32_t, true, true>(p, nframes, ref, mat, sig_stride, cb, cell_stride, wp, s);
        else launch_bc_tx<uint32_t, false, true>(p, nframes, ref, mat, sig_stride, cb, cell_stride, wp, s);
    } else {
        if (right_ref) launch_bc_tx<uint32_t, true, false>(p, nframes, ref, mat, sig_stride, cb, cell_stride, 0, s);
        else launch_bc_tx<uint32_t, false, false>(p, nframes, ref, mat, sig_stride, cb, cell_stride, 0, s);
    }
}

}  // namespace asd
