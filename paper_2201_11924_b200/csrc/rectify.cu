// rectify.cu -- stereo rectification by homography warp.
// "SimSense first performs a stereo rectification to project
// the images onto a common image plane"; SPEC S:279-287 ("warp by supplied
// 3x3 homographies with bilinear sampling"); reading c23:
//   H maps output pixel (x, y) to input coordinates:
//   w = H20 x + H21 y + H22, u = (H00 x + H01 y + H02) / w, v = (H10 x + ...) / w;
//   bilinear over the zero-padded image, w <= 0 -> 0; u8 = clamp(floor(val + 0.5)).
// fp64 in that order (the value decides a u8), built with --fmad=false.  One
// thread per output pixel; a born-rectified rig (the simulator's default)
// skips this stage.
#include <cmath>
#include "common.cuh"

namespace asd {

struct Homography { double h[9]; };

__global__ void __launch_bounds__(256)
rectify_kernel(Homography q, int W, int H, const uint8_t* __restrict__ in, uint8_t* __restrict__ out)
{
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (x >= W || y >= H) return;
    const long long fo = (long long)blockIdx.z * W * H;
    const uint8_t* I = in + fo;
    const double* h = q.h;
    const double w = h[6] * x + h[7] * y + h[8];
    double val = 0.0;
    if (w > 0.0) {
        const double u = (h[0] * x + h[1] * y + h[2]) / w;
        const double v = (h[3] * x + h[4] * y + h[5]) / w;
        if (u > -2.0 && u < W + 1.0 && v > -2.0 && v < H + 1.0) {
            const double fx0 = floor(u), fy0 = floor(v);
            const int x0 = (int)fx0, y0 = (int)fy0;
            const double a = u - fx0, b = v - fy0;
            auto px = [&](int xx, int yy) -> double {
                return (xx >= 0 && xx < W && yy >= 0 && yy < H) ? (double)I[(long long)yy * W + xx] : 0.0;
            };
            const double I00 = px(x0, y0), I10 = px(x0 + 1, y0), I01 = px(x0, y0 + 1), I11 = px(x0 + 1, y0 + 1);
            val = (1.0 - a) * (1.0 - b) * I00 + a * (1.0 - b) * I10 + (1.0 - a) * b * I01 + a * b * I11;
        }
    }
    double r = floor(val + 0.5);
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
    out[fo + (long long)y * W + x] = (uint8_t)r;
}

int launch_rectify(const double* Hm, int n, int W, int H, const uint8_t* in, uint8_t* out, cudaStream_t s)
{
    Homography q;
    for (int i = 0; i < 9; ++i) q.h[i] = Hm[i];
    dim3 grid((W + 31) / 32, (H + 7) / 8, n);
    rectify_kernel<<<grid, 256, 0, s>>>(q, W, H, in, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace asd
