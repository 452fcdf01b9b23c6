// census.cu -- K1: center-symmetric census transform (CSCT)
// ("center-symmetric census transform"), P:291 ("CSCT ... make use of shared
// memory to optimize for data reuse"); semantics SPEC S:291 + reading c1:
// bit i = I(p + o_i) > I(p - o_i), o_i = the i-th window offset in row-major
// order before the centre; 0 where the window leaves the image.
//
// One CTA = a 32x8 pixel tile of one view of one frame; the tile plus its
// census halo is staged in shared memory once, then each thread compares its
// nb point-symmetric pairs from shared memory.  HBM traffic: 1 B in + 4 (8) B
// out per pixel.
#include "common.cuh"
#include "kernels.h"

namespace asd {

constexpr int CT_X = 32, CT_Y = 8, CMAX_R = 7, CMAX_Q = 7;

// CW, CH > 0: compile-time window (fully unrolled pair loop); 0: runtime window.
template <typename SigT, int CW = 0, int CH = 0>
__global__ void __launch_bounds__(CT_X * CT_Y)
census_kernel(DevParams p, const uint8_t* __restrict__ left, const uint8_t* __restrict__ right,
              long long img_stride, SigT* __restrict__ out_l, SigT* __restrict__ out_r,
              long long sig_stride)
{
    __shared__ uint8_t tile[CT_Y + 2 * CMAX_Q][CT_X + 2 * CMAX_R];
    const int frame = blockIdx.z >> 1, view = blockIdx.z & 1;
    const uint8_t* img = (view ? right : left) + frame * img_stride;
    SigT* out = (view ? out_r : out_l) + frame * sig_stride;
    const int x0 = blockIdx.x * CT_X, y0 = blockIdx.y * CT_Y;
    const int tw = CT_X + 2 * p.R, th = CT_Y + 2 * p.Q;
    for (int i = threadIdx.y * CT_X + threadIdx.x; i < tw * th; i += CT_X * CT_Y) {
        int ty = i / tw, tx = i - ty * tw;
        int gx = x0 + tx - p.R, gy = y0 + ty - p.Q;
        tile[ty][tx] = (gx >= 0 && gx < p.W && gy >= 0 && gy < p.H) ? img[(long long)gy * p.W + gx] : 0;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= p.W || y >= p.H) return;
    SigT sig = 0;
    if (census_valid(p, x, y)) {
        const int cx = threadIdx.x + p.R, cy = threadIdx.y + p.Q;
        if constexpr (CW > 0) {
            constexpr int R = CW / 2, Q = CH / 2, NB = (CW * CH) / 2;
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int dy = i / CW - Q, dx = i % CW - R;
                sig |= (SigT)(tile[cy + dy][cx + dx] > tile[cy - dy][cx - dx]) << i;
            }
        } else {
            int i = 0;
            for (int ky = 0; ky < p.ch && i < p.nb; ++ky) {
                const int dy = ky - p.Q;
                for (int kx = 0; kx < p.cw && i < p.nb; ++kx, ++i) {
                    const int dx = kx - p.R;
                    if (tile[cy + dy][cx + dx] > tile[cy - dy][cx - dx]) sig |= (SigT)1 << i;
                }
            }
        }
    }
    out[(long long)y * p.W + x] = sig;
}

void launch_census(const DevParams& p, int nframes, const uint8_t* left, const uint8_t* right,
                   long long img_stride, void* out_l, void* out_r, long long sig_stride,
                   cudaStream_t s)
{
    dim3 grid((p.W + CT_X - 1) / CT_X, (p.H + CT_Y - 1) / CT_Y, 2 * nframes);
    dim3 block(CT_X, CT_Y);
    if (p.cw == 9 && p.ch == 7)
        census_kernel<uint32_t, 9, 7><<<grid, block, 0, s>>>(p, left, right, img_stride,
            (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
    else if (p.cw == 7 && p.ch == 7)
        census_kernel<uint32_t, 7, 7><<<grid, block, 0, s>>>(p, left, right, img_stride,
            (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
    else if (p.cw == 5 && p.ch == 5)
        census_kernel<uint32_t, 5, 5><<<grid, block, 0, s>>>(p, left, right, img_stride,
            (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
    else if (p.nb <= 32)
        census_kernel<uint32_t><<<grid, block, 0, s>>>(p, left, right, img_stride,
            (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
    else
        census_kernel<unsigned long long><<<grid, block, 0, s>>>(p, left, right, img_stride,
            (unsigned long long*)out_l, (unsigned long long*)out_r, sig_stride);
}

}  // namespace asd
