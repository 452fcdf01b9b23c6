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

// Byte-SIMD variant for compile-time windows with nb <= 32: one thread = 4
// horizontally adjacent pixels, one CTA = a 128x8 tile.  The tile is staged in
// shared memory in 4 byte-shifted copies, so the 4 bytes I(x+dx .. x+dx+3, y+dy)
// of every pair are one aligned 32-bit load (the copy and word are compile-time
// functions of dx).  Per pair: a > b for 4 pixels at once from the carry out of
// each byte of a + ~b (bit 7 of maj(a, ~b, (a & 0x7f..) + (~b & 0x7f..))), then
// moved to bit j of each byte of an 8-pair accumulator; bytes of the 4
// accumulators are finally permuted into the 4 signatures (pair i -> bit i,
// reading c1).  Same results as census_kernel, ~4x fewer instructions.
constexpr int C4_TX = 32, C4_TY = 8, C4_PX = 4 * C4_TX;

template <int CW, int CH>
__global__ void __launch_bounds__(C4_TX * C4_TY)
census4_kernel(DevParams p, const uint8_t* __restrict__ left, const uint8_t* __restrict__ right,
               long long img_stride, uint32_t* __restrict__ out_l, uint32_t* __restrict__ out_r,
               long long sig_stride)
{
    constexpr int R = CW / 2, Q = CH / 2, NB = (CW * CH) / 2;
    static_assert(NB <= 32, "u32 signatures");
    constexpr int TH = C4_TY + 2 * Q;                  // tile rows
    constexpr int TWB = C4_PX + 2 * R;                 // tile bytes per row (base copy)
    constexpr int TWW = (TWB + 3) / 4 + 1;             // words per row per copy (+1: shifted reads)
    __shared__ uint32_t tile[4][TH][TWW];              // copy s: byte c = base byte c + s
    const int frame = blockIdx.z >> 1, view = blockIdx.z & 1;
    const uint8_t* img = (view ? right : left) + frame * img_stride;
    uint32_t* out = (view ? out_r : out_l) + frame * sig_stride;
    const int x0 = blockIdx.x * C4_PX, y0 = blockIdx.y * C4_TY;
    const int tid = threadIdx.y * C4_TX + threadIdx.x;
    // base copy: byte c of row r = I(x0 + c - R, y0 + r - Q), 0 outside the image.
    // R % 4 == 0 (9-wide windows), W % 4 == 0 and a 4-byte aligned frame base
    // (the caller's pointer is not required to be aligned, asd.h): word w of a
    // row is the aligned image word at x0 - R + 4w, loaded whole when it lies
    // inside the image.  Otherwise the byte fill below.
    uint8_t* base = reinterpret_cast<uint8_t*>(&tile[0][0][0]);
    if (R % 4 == 0 && (p.W & 3) == 0 && (reinterpret_cast<uintptr_t>(img) & 3) == 0) {
        for (int i = tid; i < TH * TWW; i += C4_TX * C4_TY) {
            const int r = i / TWW, w = i - r * TWW;
            const int gx = x0 - R + 4 * w, gy = y0 + r - Q;
            uint32_t v = 0u;
            if (4 * w < TWB && gy >= 0 && gy < p.H && gx >= 0 && gx + 3 < p.W)
                v = __ldg(reinterpret_cast<const unsigned*>(img + (long long)gy * p.W + gx));
            tile[0][r][w] = v;                          // gx + 3 >= W: whole word past the row end
        }
    } else {
        for (int i = tid; i < TH * TWW * 4; i += C4_TX * C4_TY) {
            const int r = i / (TWW * 4), c = i - r * (TWW * 4);
            const int gx = x0 + c - R, gy = y0 + r - Q;
            base[i] = (c < TWB && gx >= 0 && gx < p.W && gy >= 0 && gy < p.H) ? img[(long long)gy * p.W + gx] : 0;
        }
    }
    __syncthreads();
    // shifted copies s = 1..3: word w = bytes 4w + s .. 4w + s + 3 of the base row
    for (int i = tid; i < 3 * TH * (TWW - 1); i += C4_TX * C4_TY) {
        const int s = 1 + i / (TH * (TWW - 1));
        const int rem = i - (s - 1) * TH * (TWW - 1);
        const int r = rem / (TWW - 1), w = rem - r * (TWW - 1);
        tile[s][r][w] = __funnelshift_r(tile[0][r][w], tile[0][r][w + 1], 8 * s);
    }
    __syncthreads();
    const int tx = threadIdx.x, cy = threadIdx.y + Q;
    // pixel k of this thread: tile column 4 tx + k + R; offset dx reads bytes
    // 4 tx + R + dx .. + 3 = copy (R + dx) & 3, word tx + ((R + dx) >> 2) (R + dx >= 0)
    uint32_t acc[(NB + 7) / 8];
#pragma unroll
    for (int g = 0; g < (NB + 7) / 8; ++g) acc[g] = 0u;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const int dy = i / CW - Q, dx = i % CW - R;
        const uint32_t a = tile[(R + dx) & 3][cy + dy][tx + ((R + dx) >> 2)];
        const uint32_t b = tile[(R - dx) & 3][cy - dy][tx + ((R - dx) >> 2)];
        const uint32_t nb = ~b;
        const uint32_t t = (a & 0x7F7F7F7Fu) + (nb & 0x7F7F7F7Fu);
        const uint32_t gt = (a & nb) | (t & (a | nb));     // bit 7 of byte k: a_k > b_k
        const int j = i & 7;
        acc[i >> 3] |= (gt >> (7 - j)) & (0x01010101u << j);
    }
    // signature of pixel k: byte k of acc[0], acc[1], acc[2], acc[3] -> bits 0-7, 8-15, ...
    uint32_t a4[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) a4[g] = g < (NB + 7) / 8 ? acc[g] : 0u;
    const uint32_t lo02 = __byte_perm(a4[0], a4[2], 0x5140);    // (a0.b0, a2.b0, a0.b1, a2.b1)
    const uint32_t hi02 = __byte_perm(a4[0], a4[2], 0x7362);    // (a0.b2, a2.b2, a0.b3, a2.b3)
    const uint32_t lo13 = __byte_perm(a4[1], a4[3], 0x5140);
    const uint32_t hi13 = __byte_perm(a4[1], a4[3], 0x7362);
    uint32_t sig[4];
    sig[0] = __byte_perm(lo02, lo13, 0x5140);                   // (a0.b0, a1.b0, a2.b0, a3.b0)
    sig[1] = __byte_perm(lo02, lo13, 0x7362);
    sig[2] = __byte_perm(hi02, hi13, 0x5140);
    sig[3] = __byte_perm(hi02, hi13, 0x7362);
    const int y = y0 + threadIdx.y, xb = x0 + 4 * tx;
    if (y >= p.H || xb >= p.W) return;
    const bool vrow = y >= p.Q && y < p.H - p.Q;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (!(vrow && xb + k >= p.R && xb + k < p.W - p.R)) sig[k] = 0u;   // reading c4
    uint32_t* o = out + (long long)y * p.W + xb;
    if (xb + 3 < p.W && ((reinterpret_cast<uintptr_t>(o) & 15u) == 0)) {
        *reinterpret_cast<uint4*>(o) = make_uint4(sig[0], sig[1], sig[2], sig[3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (xb + k < p.W) o[k] = sig[k];
    }
}

void launch_census(const DevParams& p, int nframes, const uint8_t* left, const uint8_t* right,
                   long long img_stride, void* out_l, void* out_r, long long sig_stride,
                   cudaStream_t s)
{
    dim3 grid((p.W + CT_X - 1) / CT_X, (p.H + CT_Y - 1) / CT_Y, 2 * nframes);
    dim3 block(CT_X, CT_Y);
#ifndef ASD_CENSUS_SIMD
#define ASD_CENSUS_SIMD 1
#endif
    if (ASD_CENSUS_SIMD && ((p.cw == 9 && p.ch == 7) || (p.cw == 7 && p.ch == 7) || (p.cw == 5 && p.ch == 5))) {
        dim3 g4((p.W + C4_PX - 1) / C4_PX, (p.H + C4_TY - 1) / C4_TY, 2 * nframes), b4(C4_TX, C4_TY);
        if (p.cw == 9)
            census4_kernel<9, 7><<<g4, b4, 0, s>>>(p, left, right, img_stride, (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
        else if (p.cw == 7)
            census4_kernel<7, 7><<<g4, b4, 0, s>>>(p, left, right, img_stride, (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
        else
            census4_kernel<5, 5><<<g4, b4, 0, s>>>(p, left, right, img_stride, (uint32_t*)out_l, (uint32_t*)out_r, sig_stride);
        return;
    }
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
