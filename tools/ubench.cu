// ubench.cu -- instruction-throughput microbenchmarks on the B200 (sm_100a) for
// the integer ops the SGM kernels are built from (DESIGN.md §6 ALU roofline).
// Each kernel runs a long unrolled dependent-free loop; ops/clk/SM =
// (threads * iters * ops_per_iter) / (cycles * SMs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ITER 4096
#define CH 8

__global__ void k_vimnmx(uint32_t* out, uint32_t seed) {
    uint32_t a[CH];
    for (int i = 0; i < CH; ++i) a[i] = seed * (threadIdx.x + i);
    uint32_t b = seed ^ threadIdx.x;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("min.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
        b += 0x00010001;
    }
    uint32_t s = 0; for (int i = 0; i < CH; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_iadd3(uint32_t* out, uint32_t seed) {
    uint32_t a[CH];
    for (int i = 0; i < CH; ++i) a[i] = seed * (threadIdx.x + i);
    uint32_t b = seed ^ threadIdx.x, c = seed + 7;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
        b ^= c;
    }
    uint32_t s = 0; for (int i = 0; i < CH; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_popc(uint32_t* out, uint32_t seed) {
    uint32_t a[CH];
    for (int i = 0; i < CH; ++i) a[i] = seed * (threadIdx.x + i);
    uint32_t acc = 0;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) { uint32_t r; asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(a[i])); a[i] += r; }
    }
    for (int i = 0; i < CH; ++i) acc ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_shfl(uint32_t* out, uint32_t seed) {
    uint32_t a[CH];
    for (int i = 0; i < CH; ++i) a[i] = seed * (threadIdx.x + i);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 3));
    }
    uint32_t s = 0; for (int i = 0; i < CH; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_redux(uint32_t* out, uint32_t seed) {
    uint32_t a[CH];
    for (int i = 0; i < CH; ++i) a[i] = seed * (threadIdx.x + i);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) a[i] = __reduce_min_sync(0xffffffffu, a[i]) + threadIdx.x;
    }
    uint32_t s = 0; for (int i = 0; i < CH; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(uint32_t* out, uint32_t seed) {   // VIMNMX + IADD3 interleaved (pipe balance)
    uint32_t a[CH], b[CH];
    for (int i = 0; i < CH; ++i) { a[i] = seed * (threadIdx.x + i); b[i] = a[i] ^ 0x5555; }
    uint32_t c = seed ^ threadIdx.x;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            asm volatile("min.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(c));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(b[i]) : "r"(c));
        }
        c += 0x00010001;
    }
    uint32_t s = 0; for (int i = 0; i < CH; ++i) s ^= a[i] ^ b[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K k, int ops_per_iter) {
    int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    int sms = p.multiProcessorCount;
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    uint32_t* out; cudaMalloc(&out, sizeof(uint32_t) * sms * 8 * 1024);
    dim3 grid(sms * 8), block(256);
    k<<<grid, block>>>(out, 3);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, block>>>(out, 5);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)grid.x * block.x * N_ITER * ops_per_iter;
    double per_s = ops / (ms / 1e3);
    // clocks: report per-SM per-cycle at the nominal max clock and at 1.965 GHz
    printf("%-8s %8.3f ms  %9.1f Gop/s  %6.1f ops/clk/SM @1965MHz\n", name, ms, per_s / 1e9,
           per_s / (sms * 1.965e9));
    cudaFree(out);
}

int main() {
    run("vimnmx", k_vimnmx, CH);
    run("iadd", k_iadd3, CH);
    run("popc", k_popc, CH);          // popc + add per element
    run("shfl", k_shfl, CH);
    run("redux", k_redux, CH);        // redux + add
    run("mix", k_mix, 2 * CH);
    return 0;
}
