// register.cu -- depth registration into the RGB camera frame (SURVEY §8(f)
// NEXT 2).  PAPER.md P:289: "The refined disparity map is then converted into
// a depth map, with an optional depth registration that aligns the depth map
// to the RGB camera frame"; SPEC S:357-365 [OP] register_depth; reading c21
// (DESIGN.md §3):
//   each source pixel (x, y) with finite z > 0:
//     a = ((float)x - cx) * z / fx,  b = ((float)y - cy) * z / fy
//     P' = R (a, b, z) + t          (each row: ((R0 a + R1 b) + R2 z) + t)
//     u = (X' / Z') * fx' + cx',  v = (Y' / Z') * fy' + cy'
//     target (floor(u + 0.5), floor(v + 0.5)); the z-buffer keeps min Z'.
// The coordinates decide an integer (the target pixel), so every float op is
// one IEEE fp32 operation in that order (this file is built with
// --fmad=false; explicit _rn intrinsics).  The z-buffer is an atomicMin on the
// IEEE bits of Z' > 0 (order-preserving for positive floats, so the result
// does not depend on the scatter order); untouched targets (+inf) become NaN.
#include <cmath>
#include "asd.h"
#include "common.cuh"

namespace asd {

struct RegParams {
    asd_camera ir, rgb;
    float R[9], t[3];
};

__global__ void reg_fill_kernel(uint32_t* out, long long n, uint32_t v)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = v;
}

__global__ void __launch_bounds__(256)
reg_scatter_kernel(RegParams q, const float* __restrict__ depth, uint32_t* __restrict__ zbuf)
{
    const int frame = blockIdx.y;
    const long long npx = (long long)q.ir.width * q.ir.height;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npx) return;
    const float z = depth[frame * npx + i];
    if (!(z > 0.0f) || isinf(z)) return;                 // NaN (invalid) or non-positive
    const int y = (int)(i / q.ir.width), x = (int)(i - (long long)y * q.ir.width);
    float a = __fsub_rn((float)x, q.ir.cx); a = __fmul_rn(a, z); a = __fdiv_rn(a, q.ir.fx);
    float b = __fsub_rn((float)y, q.ir.cy); b = __fmul_rn(b, z); b = __fdiv_rn(b, q.ir.fy);
    float P[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        float s = __fmul_rn(q.R[3 * r], a);
        s = __fadd_rn(s, __fmul_rn(q.R[3 * r + 1], b));
        s = __fadd_rn(s, __fmul_rn(q.R[3 * r + 2], z));
        P[r] = __fadd_rn(s, q.t[r]);
    }
    if (!(P[2] > 0.0f)) return;
    float u = __fdiv_rn(P[0], P[2]); u = __fmul_rn(u, q.rgb.fx); u = __fadd_rn(u, q.rgb.cx);
    float v = __fdiv_rn(P[1], P[2]); v = __fmul_rn(v, q.rgb.fy); v = __fadd_rn(v, q.rgb.cy);
    const float uu = __fadd_rn(u, 0.5f), vv = __fadd_rn(v, 0.5f);
    if (!(uu >= 0.0f && uu < (float)q.rgb.width && vv >= 0.0f && vv < (float)q.rgb.height)) return;
    const int iu = (int)floorf(uu), iv = (int)floorf(vv);
    const long long nt = (long long)q.rgb.width * q.rgb.height;
    atomicMin(zbuf + frame * nt + (long long)iv * q.rgb.width + iu, __float_as_uint(P[2]));
}

__global__ void reg_finish_kernel(uint32_t* out, long long n)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (out[i] == 0x7f800000u) out[i] = 0x7fc00000u;      // +inf (no sample) -> NaN
}

int launch_register(const asd_camera* ir, const asd_camera* rgb, const float* R, const float* t,
                    int n, const float* depth, float* out, cudaStream_t s)
{
    RegParams q;
    q.ir = *ir; q.rgb = *rgb;
    for (int i = 0; i < 9; ++i) q.R[i] = R[i];
    for (int i = 0; i < 3; ++i) q.t[i] = t[i];
    const long long nt = (long long)n * rgb->width * rgb->height;
    const long long npx = (long long)ir->width * ir->height;
    uint32_t* zb = reinterpret_cast<uint32_t*>(out);
    const int fill_blocks = (int)((nt + 255) / 256 < 148 * 16 ? (nt + 255) / 256 : 148 * 16);
    reg_fill_kernel<<<fill_blocks, 256, 0, s>>>(zb, nt, 0x7f800000u);
    dim3 grid((unsigned)((npx + 255) / 256), n);
    reg_scatter_kernel<<<grid, 256, 0, s>>>(q, depth, zb);
    reg_finish_kernel<<<fill_blocks, 256, 0, s>>>(zb, nt);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace asd
