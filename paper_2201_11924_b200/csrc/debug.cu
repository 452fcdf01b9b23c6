// debug.cu -- stage extraction for parity tests (asd_depth_debug): the raw
// Hamming cost volume (reading c3), which the
// production path never materialises.
#include "common.cuh"
#include "kernels.h"

namespace asd {

template <typename SigT>
__global__ void cost_volume_kernel(DevParams p, const SigT* __restrict__ cl, const SigT* __restrict__ cr,
                                   uint8_t* __restrict__ cost)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.ncell) return;
    const int d = (int)(i % p.D);
    const long long pix = i / p.D;
    const int y = (int)(pix / p.W), x = (int)(pix - (long long)y * p.W);
    const int xr = x - p.min_disp - d;
    int c = p.nb;
    if (census_valid(p, x, y) && xr >= p.R)
        c = popc_sig(cl[pix] ^ cr[(long long)y * p.W + xr]);
    cost[i] = (uint8_t)c;
}

void launch_cost_volume(const DevParams& p, const void* cl, const void* cr, uint8_t* cost, cudaStream_t s)
{
    const unsigned blocks = (unsigned)((p.ncell + 255) / 256);
    if (p.nb <= 32)
        cost_volume_kernel<uint32_t><<<blocks, 256, 0, s>>>(p, (const uint32_t*)cl, (const uint32_t*)cr, cost);
    else
        cost_volume_kernel<unsigned long long><<<blocks, 256, 0, s>>>(p, (const unsigned long long*)cl,
                                                                      (const unsigned long long*)cr, cost);
}

}  // namespace asd
