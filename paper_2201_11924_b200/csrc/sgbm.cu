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
// One CTA = TX consecutive pixels of one row of one frame, all D disparities;
// thread = disparity (strided when D > blockDim).  The bh census rows of the
// left block span and of the right span they are compared with are staged in
// shared memory with validity flags.  Per disparity the thread forms the
// vertical block sums V(c) of the TX + bw - 1 block columns, keeps their
// prefix sums in shared memory ([c][d], conflict-free across the warp) and
// writes CB(x0 + i, d) = P(i + bw) - P(i): (TX + bw - 1) * bh Hamming
// evaluations per TX outputs, not TX * bw * bh.
#include "common.cuh"
#include "kernels.h"

namespace asd {

constexpr int SB_TX = 32;            // pixels per CTA
constexpr int SB_MAXB = 15;          // block dims bound (asd_create validates)

// RR: the right view is the reference (R2, reading c24): cl_base / cr_base are
// then the reference and matched census and the matched column is x' + delta.
template <typename SigT, bool RR>
__global__ void __launch_bounds__(256)
block_cost_kernel(DevParams p, const SigT* __restrict__ cl_base, const SigT* __restrict__ cr_base,
                  long long sig_stride, uint16_t* __restrict__ cb_base, long long cell_stride)
{
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const int W = p.W, H = p.H, D = p.D;
    const int bu = p.bw / 2, bv = p.bh / 2;
    const int frame = blockIdx.z, y = blockIdx.y, x0 = blockIdx.x * SB_TX;
    const int NC = SB_TX + p.bw - 1;                 // block columns x0-bu .. x0+TX-1+bu
    const int NRW = NC + D - 1;                      // matched span: x' -/+ (min + d)
    const int xr0 = RR ? x0 - bu + p.min_disp                 // first matched column
                       : x0 - bu - p.min_disp - (D - 1);
    const SigT* cl = cl_base + frame * sig_stride;
    const SigT* cr = cr_base + frame * sig_stride;

    SigT* Ls = reinterpret_cast<SigT*>(sm_raw);                  // [bh][NC]
    SigT* Rs = Ls + p.bh * NC;                                    // [bh][NRW]
    uint32_t* Pfx = reinterpret_cast<uint32_t*>(Rs + p.bh * NRW); // [NC + 1][D]
    unsigned char* Lv = reinterpret_cast<unsigned char*>(Pfx + (NC + 1) * D);   // [bh][NC]
    unsigned char* Rv = Lv + p.bh * NC;                                          // [bh][NRW]

    for (int i = threadIdx.x; i < p.bh * NC; i += blockDim.x) {
        const int v = i / NC, c = i - v * NC;
        const int xx = x0 - bu + c, yy = y - bv + v;
        const bool in = xx >= 0 && xx < W && yy >= 0 && yy < H;
        const bool ok = in && census_valid(p, xx, yy);
        Ls[i] = ok ? cl[(long long)yy * W + xx] : (SigT)0;
        Lv[i] = ok;
    }
    for (int i = threadIdx.x; i < p.bh * NRW; i += blockDim.x) {
        const int v = i / NRW, c = i - v * NRW;
        const int xr = xr0 + c, yy = y - bv + v;
        const bool ok = yy >= 0 && yy < H && xr >= 0 && xr < W && census_valid(p, xr, yy);
        Rs[i] = ok ? cr[(long long)yy * W + xr] : (SigT)0;
        Rv[i] = ok;
    }
    __syncthreads();

    uint16_t* cb = cb_base + frame * cell_stride + ((long long)y * W + x0) * D;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        uint32_t run = 0;
        Pfx[d] = 0;
        for (int c = 0; c < NC; ++c) {
            // matched column of block column c at disparity d: x' - min - d (x' + min + d for RR)
            const int rc = RR ? c + d : c + (D - 1) - d;
            uint32_t vs = 0;
            for (int v = 0; v < p.bh; ++v) {
                const int li = v * NC + c, ri = v * NRW + rc;
                vs += (Lv[li] && Rv[ri]) ? (uint32_t)popc_sig(Ls[li] ^ Rs[ri]) : (uint32_t)p.nb;
            }
            run += vs;
            Pfx[(c + 1) * D + d] = run;
        }
        for (int i = 0; i < SB_TX && x0 + i < W; ++i)
            cb[(long long)i * D + d] = (uint16_t)(Pfx[(i + p.bw) * D + d] - Pfx[i * D + d]);
    }
}

static size_t block_cost_smem(const DevParams& p, size_t sig)
{
    const size_t NC = SB_TX + p.bw - 1, NRW = NC + p.D - 1;
    size_t b = (size_t)p.bh * (NC + NRW) * sig + (NC + 1) * p.D * 4 + (size_t)p.bh * (NC + NRW);
    return (b + 15) & ~size_t(15);
}

template <typename SigT, bool RR>
static void launch_bc(const DevParams& p, dim3 grid, int threads, const void* ref, const void* mat,
                      long long sig_stride, uint16_t* cb, long long cell_stride, cudaStream_t s)
{
    const size_t sm = block_cost_smem(p, sizeof(SigT));
    cudaFuncSetAttribute((const void*)block_cost_kernel<SigT, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    block_cost_kernel<SigT, RR><<<grid, threads, sm, s>>>(p, (const SigT*)ref, (const SigT*)mat, sig_stride, cb,
                                                         cell_stride);
}

void launch_block_cost(const DevParams& p, int nframes, const void* cl, const void* cr,
                       long long sig_stride, uint16_t* cb, long long cell_stride, cudaStream_t s,
                       bool right_ref)
{
    dim3 grid((p.W + SB_TX - 1) / SB_TX, p.H, nframes);
    const int threads = p.D < 256 ? p.D : 256;
    const void* ref = right_ref ? cr : cl;
    const void* mat = right_ref ? cl : cr;
    if (p.nb <= 32) {
        if (right_ref) launch_bc<uint32_t, true>(p, grid, threads, ref, mat, sig_stride, cb, cell_stride, s);
        else launch_bc<uint32_t, false>(p, grid, threads, ref, mat, sig_stride, cb, cell_stride, s);
    } else {
        if (right_ref) launch_bc<unsigned long long, true>(p, grid, threads, ref, mat, sig_stride, cb, cell_stride, s);
        else launch_bc<unsigned long long, false>(p, grid, threads, ref, mat, sig_stride, cb, cell_stride, s);
    }
}

}  // namespace asd
