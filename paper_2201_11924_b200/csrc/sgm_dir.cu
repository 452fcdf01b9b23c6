// sgm_dir.cu -- K2/K3 (design D1): one semi-global path direction per launch,
// warp per scanline.  PAPER.md P:289 ("four-path semi-global matching (SGM)
// ... with hamming distance as the cost function"), P:291 ("cost aggregation
// of SGM is further accelerated with warp-based optimization").  Recursion
// (reading c6):
//   L_r(p,d) = C(p,d) + min(L_r(p-r,d), L_r(p-r,d-1)+P1, L_r(p-r,d+1)+P1, M+P2) - M,
//   M = min_k L_r(p-r,k);  L_r = C at the first pixel of a line.
// S = sum_r L_r accumulates in a u16 [H][W][D] volume: the first direction
// writes it, the others read-modify-write it (4 B per cell: HBM-bound).
//
// Work mapping: one warp walks one line of direction r.  Lane l holds the DPL
// disparities d0 = l*DPL .. d0+DPL-1 (DPL = 2 / 4 / 8 for D <= 64 / 128 / 256,
// act = D / DPL active lanes) packed two per register in natural order,
// R_k = (d0+2k, d0+2k+1) as u16x2 -- the same packing as the S vector in
// memory, so the read-modify-write of S is one integer add per register.
// Q = L + P1 is shuffled instead of L; the d-1 / d+1 pairs of register k are
// byte permutes of neighbouring registers (E_k = (Q_{k-1}.hi, Q_k.lo)), the
// lane-edge halves come from __shfl_up/down_sync, and the packed min
// (M | M << 16) from one __reduce_min_sync of each lane's (min, min) word.
// All values stay below 2^15 (ABI bounds), so u16x2 adds never carry.
//
// The matching cost (PAPER P:289 Hamming distance, reading c3) is
// recomputed from the census images: C = popc(cl(x,y) ^ cr(x-delta,y)) if both
// windows are valid, else nb.  SGBM (MODE 2): C is read from the block-cost
// volume CB (sgbm.cu, reading c19), already u16x2-packed.
// The census words and S / CB vectors of the next PF pixels of the line are
// kept in flight in a register ring (plus an L2 prefetch further ahead).
#include "common.cuh"
#include "kernels.h"

namespace asd {

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

namespace dir {

constexpr uint32_t INF2 = 0x7FFF7FFFu;        // packed "no predecessor" (+P1 stays < 2^16)

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// NR u32 words (2 NR u16) of S / CB: one 4 / 8 / 16-byte access.
template <int NR> struct Vec;
template <> struct Vec<1> {
    uint32_t w[1];
    __device__ __forceinline__ void ld(const uint16_t* s) { w[0] = *reinterpret_cast<const uint32_t*>(s); }
    __device__ __forceinline__ void ldnc(const uint16_t* s) { w[0] = __ldg(reinterpret_cast<const unsigned*>(s)); }
    __device__ __forceinline__ void st(uint16_t* s) const { *reinterpret_cast<uint32_t*>(s) = w[0]; }
};
template <> struct Vec<2> {
    uint32_t w[2];
    __device__ __forceinline__ void ld(const uint16_t* s) {
        const uint2 u = *reinterpret_cast<const uint2*>(s); w[0] = u.x; w[1] = u.y;
    }
    __device__ __forceinline__ void ldnc(const uint16_t* s) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(s)); w[0] = u.x; w[1] = u.y;
    }
    __device__ __forceinline__ void st(uint16_t* s) const { *reinterpret_cast<uint2*>(s) = make_uint2(w[0], w[1]); }
};
template <> struct Vec<4> {
    uint32_t w[4];
    __device__ __forceinline__ void ld(const uint16_t* s) {
        const uint4 u = *reinterpret_cast<const uint4*>(s); w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
    }
    __device__ __forceinline__ void ldnc(const uint16_t* s) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(s)); w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
    }
    __device__ __forceinline__ void st(uint16_t* s) const {
        *reinterpret_cast<uint4*>(s) = make_uint4(w[0], w[1], w[2], w[3]);
    }
};

__device__ __forceinline__ uint32_t popc_w(uint32_t v) { return __popc(v); }
__device__ __forceinline__ uint32_t popc_w(unsigned long long v) { return __popcll(v); }

}  // namespace dir

// Prefetch distances (pixels ahead on the line): PF steps of census words and
// S / CB vectors are kept in flight in a register ring; the S vectors PF + PFL2
// steps ahead are also prefetched into L2 (one prefetch per lane per step, no
// registers), so the ring's loads hit L2 on the lines that jump a whole image
// row per step (vertical and diagonal directions).  PFL2 = 0 disables it.
#ifndef ASD_DIR_PF
#define ASD_DIR_PF 4
#endif
#ifndef ASD_DIR_PFL2
#define ASD_DIR_PFL2 8
#endif
#ifndef ASD_DIR_PF8
#define ASD_DIR_PF8 ((ASD_DIR_PF + 1) / 2)    // ring depth at DPL = 8 (D > 128)
#endif
template <int DPL> struct DirPF { static constexpr int v = DPL <= 4 ? ASD_DIR_PF : ASD_DIR_PF8; };

__device__ __forceinline__ void prefetch_l2(const void* p)
{ asm volatile("prefetch.global.L2 [%0];\n" :: "l"(p)); }

// MODE 0: cost from census, left view as reference (C = popc(cl(x) ^ cr(x - delta)));
// MODE 1: right view as reference (R2, reading c24: popc(cr(x) ^ cl(x + delta)));
// MODE 2: cost read from a u16 volume (SGBM block cost, either reference).
// FULLW: act == 32 (no idle lanes).
#ifndef ASD_DIR_MINB
#define ASD_DIR_MINB 1
#endif
#ifndef ASD_DIR_WARPS
#define ASD_DIR_WARPS 4              // lines (warps) per CTA (8 measured slower)
#endif
#ifndef ASD_DIR_SYNC
#define ASD_DIR_SYNC 0               // vertical lines: CTA barrier every this many steps (0 = none; 16 measured no faster)
#endif
template <int DPL, typename SigT, bool FIRST, int MODE, bool FULLW>
__global__ void __launch_bounds__(32 * ASD_DIR_WARPS, ASD_DIR_MINB)
sgm_dir_kernel(DevParams p, int rx, int ry, int nchains, int act,
               const SigT* __restrict__ cl_base, const SigT* __restrict__ cr_base, long long sig_stride,
               uint16_t* __restrict__ S_base, long long s_stride, const uint16_t* __restrict__ cv_base,
               long long pstep, long long sinc, unsigned long long nbmask_h)
{
    // pstep = pixel index step along the line, sinc = pstep * D (S elements),
    // nbmask_h = (1 << nb) - 1: loop constants computed once on the host
    using namespace dir;
    constexpr int NR = DPL / 2;                       // u16x2 registers per lane
    constexpr int PF = DirPF<DPL>::v, PFL2 = ASD_DIR_PFL2;
    constexpr bool CV = MODE == 2, RR = MODE == 1;
    const int chain = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (chain >= nchains) return;
    // vertical lines all have length H: keep the CTA's adjacent columns in step so
    // their S rows reach DRAM together (named barrier over the CTA's live warps)
    const int live_thr = 32 * min((int)(blockDim.x >> 5), nchains - (int)(blockIdx.x * (blockDim.x >> 5)));
    const bool dosync = ASD_DIR_SYNC > 0 && rx == 0;
    const int frame = blockIdx.y;
    // reference / matched census (swapped for the right-view reference)
    const SigT* cl = (RR ? cr_base : cl_base) + frame * sig_stride;
    const SigT* cr = (RR ? cl_base : cr_base) + frame * sig_stride;
    uint16_t* S = S_base + frame * s_stride;
    const uint16_t* CVf = CV ? cv_base + frame * s_stride : nullptr;
    const bool active = FULLW || lane < act;
    const int d0 = lane * DPL;

    int x0, y0;
    chain_start(p, rx, ry, chain, x0, y0);
    int len = 1 << 30;                                 // pixels until the line leaves the image
    if (rx > 0) len = min(len, p.W - x0); else if (rx < 0) len = min(len, x0 + 1);
    if (ry > 0) len = min(len, p.H - y0); else if (ry < 0) len = min(len, y0 + 1);
    // steps i with a valid reference census window: [ilo, ihi) (reading c4)
    int ilo = 0, ihi = len;
    auto clip = [&](int v0, int dv, int lo, int hi) {     // lo <= v0 + i*dv < hi
        if (dv > 0) { ilo = max(ilo, lo - v0); ihi = min(ihi, hi - v0); }
        else if (dv < 0) { ilo = max(ilo, v0 - hi + 1); ihi = min(ihi, v0 - lo + 1); }
        else if (v0 < lo || v0 >= hi) ihi = 0;
    };
    clip(x0, rx, p.R, p.W - p.R);
    clip(y0, ry, p.Q, p.H - p.Q);
    // matched window valid for local disparity j iff T - j >= 0 with
    // T = x - min_disp - d0 - R (left reference) / W - R - 1 - x - min_disp - d0 (right)
    const int T0 = RR ? p.W - p.R - 1 - x0 - p.min_disp - d0 : x0 - p.min_disp - d0 - p.R;
    const int Tstep = RR ? -rx : rx;
    // census word of local disparity j at step i: cr[pix(i) + moff -/+ j]
    const int moff = RR ? p.min_disp + d0 : -(p.min_disp + d0);
    const long long pix0 = (long long)y0 * p.W + x0;
    const uint32_t P1P1 = (uint32_t)p.p1 * 0x10001u, P2P2 = (uint32_t)p.p2 * 0x10001u;
    const SigT nbmask = (SigT)nbmask_h;               // nb low bits set (host-computed)

    // Fast-fetch steps [fa, fb): the reference window is valid and so is every
    // matched window of every active lane (T of the last active lane, the
    // smallest, >= DPL - 1); elsewhere the census fetch predicates per j.
    const int T0l = RR ? p.W - p.R - 1 - x0 - p.min_disp - (act - 1) * DPL
                       : x0 - p.min_disp - (act - 1) * DPL - p.R;
    int fa = ilo, fb = ihi;
    if (Tstep > 0) fa = max(fa, DPL - 1 - T0l);
    else if (Tstep < 0) fb = min(fb, T0l - DPL + 2);
    else if (T0l < DPL - 1) fb = fa;
    // Pixel index of the next pixel to fetch (int: W*H < 2^31) and base pointers;
    // each ring slot keeps the pixel index its step stores to.
    unsigned fpix = (unsigned)pix0;
    const unsigned pst = (unsigned)pstep;              // wraps for negative steps (u32 arithmetic)
    const unsigned vstride = 2u * (unsigned)p.D;       // bytes per S / CB vector
    // base + idx * scale in one IMAD.WIDE.U32
    auto at = [](auto* base, unsigned idx, unsigned scale) {
        return reinterpret_cast<decltype(base)>(reinterpret_cast<uintptr_t>(base) + (unsigned long long)idx * scale);
    };
    const SigT* crm = cr + moff;
    uint16_t* Sd = S + d0;
    const uint16_t* CVd = CV ? CVf + d0 : nullptr;
    struct Slot { SigT l; SigT r[DPL]; Vec<NR> s; Vec<NR> c; unsigned pix; };
    auto fetch = [&](Slot& q, int i) {
        if (!CV) {
            q.l = __ldg(at(cl, fpix, (unsigned)sizeof(SigT)));
            const SigT* pr = at(crm, fpix, (unsigned)sizeof(SigT));
            if (i >= fa && i < fb) {                   // warp-uniform: every window valid
                if constexpr (sizeof(SigT) == 4 && DPL >= 8) {
                    // the lane's DPL words are contiguous: 8-byte loads (the
                    // alignment of the lowest word is warp-uniform, DPL even).
                    // Pays at DPL = 8 (D > 128: the scalar loads saturate the LSU,
                    // config D dir 4836 -> 3793 us/frame); slower at DPL = 4 / 2.
                    const uint32_t* lo = reinterpret_cast<const uint32_t*>(RR ? pr : pr - (DPL - 1));
                    auto put = [&](int k, uint32_t v) { q.r[RR ? k : DPL - 1 - k] = v; };   // word lo + k
                    if (active) {
                        if ((reinterpret_cast<uintptr_t>(lo) & 7u) == 0) {
#pragma unroll
                            for (int m = 0; m < DPL / 2; ++m) {
                                const uint2 v = __ldg(reinterpret_cast<const uint2*>(lo) + m);
                                put(2 * m, v.x); put(2 * m + 1, v.y);
                            }
                        } else {
                            put(0, __ldg(lo));
#pragma unroll
                            for (int m = 0; m < DPL / 2 - 1; ++m) {
                                const uint2 v = __ldg(reinterpret_cast<const uint2*>(lo + 1) + m);
                                put(2 * m + 1, v.x); put(2 * m + 2, v.y);
                            }
                            put(DPL - 1, __ldg(lo + DPL - 1));
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < DPL; ++j) q.r[j] = active ? __ldg(pr + (RR ? j : -j)) : 0;
                }
            } else {
                const bool vl = i >= ilo && i < ihi;
                const int t = vl ? T0 + i * Tstep : -1;
#pragma unroll
                for (int j = 0; j < DPL; ++j) {
                    // invalid: r = l ^ nbmask, so popc(l ^ r) = nb (reading c3)
                    q.r[j] = (active && t >= j) ? __ldg(pr + (RR ? j : -j)) : (q.l ^ nbmask);
                }
            }
        }
        const uint16_t* sv = at(Sd, fpix, vstride);
        if (PFL2 > 0 && !FIRST && active && i + PFL2 < len) prefetch_l2(sv + PFL2 * sinc);
        if (!FIRST && active) q.s.ld(sv);
        if (CV && active) q.c.ldnc(at(CVd, fpix, vstride));
        q.pix = fpix;
        fpix += pst;
    };
    Slot ring[PF];
#pragma unroll
    for (int k = 0; k < PF; ++k)
        if (k < len) fetch(ring[k], k);
    if (PFL2 > 0 && !FIRST && active) {               // L2 prefetch of the steps PF .. PF + PFL2 - 1
        for (int k = PF; k < PF + PFL2 && k < len; ++k) prefetch_l2(S + (pix0 + k * pstep) * p.D + d0);
    }

    // L = 0 and M = 0 before the line start make the recursion return C there
    uint32_t L[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) L[k] = active ? 0u : INF2;
    uint32_t M2 = 0;                                   // M | M << 16
    const bool has_prev = lane > 0, has_next = lane < act - 1;
    for (int i0 = 0; i0 < len; i0 += PF) {
        if (ASD_DIR_SYNC > 0 && dosync && i0 % ASD_DIR_SYNC == 0)
            asm volatile("bar.sync 1, %0;" :: "r"(live_thr) : "memory");
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const int i = i0 + k;
            if (i >= len) break;                       // warp-uniform
            Slot& cur = ring[k];
            // packed matching costs of this lane's disparities
            uint32_t C[NR];
            if constexpr (CV) {
#pragma unroll
                for (int r = 0; r < NR; ++r) C[r] = cur.c.w[r];
            } else {
#pragma unroll
                for (int r = 0; r < NR; ++r)
                    C[r] = __byte_perm(popc_w(cur.l ^ cur.r[2 * r]), popc_w(cur.l ^ cur.r[2 * r + 1]), 0x5410);
            }
            // recursion on u16x2 pairs
            uint32_t Q[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) Q[r] = L[r] + P1P1;
            uint32_t qprev = __shfl_up_sync(FULL, Q[NR - 1], 1);
            uint32_t qnext = __shfl_down_sync(FULL, Q[0], 1);
            if (!has_prev) qprev = INF2;
            if (!has_next) qnext = INF2;
            uint32_t E[NR + 1];                        // E_r = (d0+2r-1, d0+2r) of Q
            E[0] = __byte_perm(qprev, Q[0], 0x5432);
#pragma unroll
            for (int r = 1; r < NR; ++r) E[r] = __byte_perm(Q[r - 1], Q[r], 0x5432);
            E[NR] = __byte_perm(Q[NR - 1], qnext, 0x5432);
            const uint32_t MP2 = M2 + P2P2;
            uint32_t Ln[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                uint32_t t = vmin2(vmin2(E[r], E[r + 1]), L[r]);
                t = vmin2(t, MP2);
                Ln[r] = t + C[r] - M2;
            }
            if (!FULLW && !active) {
#pragma unroll
                for (int r = 0; r < NR; ++r) Ln[r] = INF2;
            }
            // S read-modify-write (packed add: no carry, S <= 65535 per half)
            if (active) {
                Vec<NR> o;
#pragma unroll
                for (int r = 0; r < NR; ++r) o.w[r] = FIRST ? Ln[r] : cur.s.w[r] + Ln[r];
                o.st(at(Sd, cur.pix, vstride));
            }
            if (i + PF < len) fetch(ring[k], i + PF);     // refill the consumed slot
            // packed M of this pixel for the next step
            uint32_t tr[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) tr[r] = Ln[r];
#pragma unroll
            for (int h = NR / 2; h >= 1; h >>= 1) {
#pragma unroll
                for (int r = 0; r < h; ++r) tr[r] = vmin2(tr[r], tr[r + h]);
            }
            const uint32_t m = vmin2(tr[0], __byte_perm(tr[0], tr[0], 0x1032));
            M2 = __reduce_min_sync(FULL, m);
#pragma unroll
            for (int r = 0; r < NR; ++r) L[r] = Ln[r];
        }
    }
}

template <int DPL, typename SigT, bool FULLW>
static void launch_dir_t(const DevParams& p, int nframes, int rx, int ry, bool first, int act,
                         const void* cl, const void* cr, long long sig_stride,
                         uint16_t* S, long long s_stride, cudaStream_t s, const uint16_t* cv, bool right_ref)
{
    const int n = num_chains(p, rx, ry);
    dim3 grid((n + ASD_DIR_WARPS - 1) / ASD_DIR_WARPS, nframes), block(32 * ASD_DIR_WARPS);
    const long long pstep = (long long)ry * p.W + rx, sinc = pstep * p.D;
    const unsigned long long nbm = p.nb >= 64 ? ~0ull : ((1ull << p.nb) - 1);
    const SigT* l = (const SigT*)cl;
    const SigT* r = (const SigT*)cr;
#define ASD_DIR_LAUNCH(M) \
    if (first) sgm_dir_kernel<DPL, SigT, true, M, FULLW><<<grid, block, 0, s>>>(p, rx, ry, n, act, l, r, sig_stride, S, s_stride, cv, pstep, sinc, nbm); \
    else sgm_dir_kernel<DPL, SigT, false, M, FULLW><<<grid, block, 0, s>>>(p, rx, ry, n, act, l, r, sig_stride, S, s_stride, cv, pstep, sinc, nbm);
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
    // DPL = 2 / 4 / 8 disparities per lane for D <= 64 / 128 / 256; D % 16 == 0 (ABI)
    const int dpl = p.D <= 64 ? 2 : p.D <= 128 ? 4 : 8;
    if (p.D % dpl != 0 || p.D > 256) return false;
    const int act = p.D / dpl;
    const bool full = act == 32;
#define ASD_DIR_CASE(K) case K: \
    if (full) launch_dir_t<K, SigT, true>(p, nframes, rx, ry, first, act, cl, cr, sig_stride, S, s_stride, s, cv, right_ref); \
    else launch_dir_t<K, SigT, false>(p, nframes, rx, ry, first, act, cl, cr, sig_stride, S, s_stride, s, cv, right_ref); \
    return true;
    switch (dpl) {
        ASD_DIR_CASE(2) ASD_DIR_CASE(4) ASD_DIR_CASE(8)
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
