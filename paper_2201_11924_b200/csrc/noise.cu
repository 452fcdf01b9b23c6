// noise.cu -- sensor noise front end.  PAPER.md
// "Our noise model contains two parts: a multiplicative term gamma
// modeling the laser speckle and an additive term n modeling camera thermal
// noise: I_noisy = gamma * I_clean + n", gamma ~ Gamma(k, theta) (the density
// of P:279), n ~ N(mu, sigma^2); D415 values k = 3.98, theta = 0.254,
// mu = -0.231, sigma = 0.83; readings c17 (DN units, round half up,
// clamp to u8) and c22:
//   Philox4x32-10, key = seed, counter = (pixel, attempt, frame, view);
//   U(x) = ((x >> 8) + 0.5) / 2^24; Box-Muller z = sqrt(-2 ln U0) cos(2 pi U1);
//   n = mu + sigma z from attempt 0xFFFFFFFF;
//   gamma: Marsaglia-Tsang on k' = k (or k + 1 with the U(x3)^(1/k) boost for
//   k < 1), d = k' - 1/3, c = 1/sqrt(9 d), <= 16 attempts;
//   scale s: gamma' = k theta + s (gamma - k theta), n' = s n;
//   out = clamp(floor(gamma' I + n' + 0.5), 0, 255).
// One thread per pixel, double precision throughout (the quantisation decides
// an integer); built with --fmad=false so no product is fused.
#include <cmath>
#include "asd.h"
#include "common.cuh"

namespace asd {

__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

__device__ __forceinline__ double unit_open(uint32_t x) { return ((double)(x >> 8) + 0.5) / 16777216.0; }

__device__ __forceinline__ double box_muller(const uint32_t x[4])
{
    return sqrt(-2.0 * log(unit_open(x[0]))) * cos(2.0 * 3.14159265358979323846 * unit_open(x[1]));
}

__global__ void __launch_bounds__(256)
noise_kernel(asd_noise q, uint32_t key0, uint32_t key1, int npx, uint32_t frame0, uint32_t view,
             const float* __restrict__ clean, uint8_t* __restrict__ out)
{
    const int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= npx) return;
    const uint32_t frame = frame0 + blockIdx.y;
    uint32_t x[4] = {(uint32_t)pix, 0xFFFFFFFFu, frame, view};
    philox10(x, key0, key1);
    const double n = q.mu + q.sigma * box_muller(x);
    const double kk = q.k >= 1.0 ? q.k : q.k + 1.0;
    const double d = kk - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    double g = d, boost = 1.0;
    for (uint32_t j = 0; j < 16; ++j) {
        uint32_t y[4] = {(uint32_t)pix, j, frame, view};
        philox10(y, key0, key1);
        if (j == 0 && q.k < 1.0) boost = pow(unit_open(y[3]), 1.0 / q.k);
        const double z = box_muller(y);
        const double t = 1.0 + c * z;
        const double v = t * t * t;
        if (v <= 0.0) continue;
        if (log(unit_open(y[2])) < 0.5 * z * z + d - d * v + d * log(v)) { g = d * v; break; }
    }
    const double gamma = g * boost * q.theta;
    const double kt = q.k * q.theta;
    const double gs = kt + q.scale * (gamma - kt), ns = q.scale * n;
    const long long o = (long long)blockIdx.y * npx + pix;
    double r = floor(gs * (double)clean[o] + ns + 0.5);
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
    out[o] = (uint8_t)r;
}

int launch_noise(const asd_noise* q, uint64_t seed, int n, int width, int height, uint32_t frame0,
                 uint32_t view, const float* clean, uint8_t* out, cudaStream_t s)
{
    const int npx = width * height;
    dim3 grid((unsigned)((npx + 255) / 256), n);
    noise_kernel<<<grid, 256, 0, s>>>(*q, (uint32_t)seed, (uint32_t)(seed >> 32), npx, frame0, view, clean, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace asd
