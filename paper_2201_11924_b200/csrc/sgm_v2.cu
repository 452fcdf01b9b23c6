// sgm_v2.cu -- design D3: SGM aggregation in three sweeps with the cost
// volume never materialised and the path state packed two disparities per
// 32-bit register (u16x2, VIMNMX/VIMNMX3 on sm_100a).
//
//   K_down  (cluster kernel)  rows top->bottom, paths  down, down-right, down-left;
//                             cost C by POPC from census rows in shared memory
//                             -> P_A | C << 8 per cell (u16, warp-private order)
//   K_up    (cluster kernel)  rows bottom->top (TMA ring of K_down rows),
//                             paths up, up-left, up-right
//                             -> P_AB | C << 9 per cell (u16, natural order)
//   K_row   (warp per row)    left->right path (L stashed as u8), then
//                             right->left path; S = P_AB + L_lr + L_rl
//                             written over the partial, natural d order
//   K_wta   (CTA per row)     WTA / uniqueness / sub-pixel for the left view
//                             and the re-indexed right view from shared-memory
//                             windows of S rows (K4 semantics, post.cu)
// 4-path: K_down/K_up carry only the vertical path.
//
// Recursion ("four-path semi-global matching", SPEC S:309,
// reading c6), for every path r:
//   L_r(p,d) = C(p,d) + min(L_r(p-r,d), L_r(p-r,d+-1)+P1, M+P2) - M.
// A predecessor outside the image is fed as L = 0, M = 0, which makes the
// formula return C (the line start) without a branch.  Cost (P:289 Hamming,
// S:300, reading c3) is recomputed from the census rows staged in shared
// memory: C = popc(cl(x,y) ^ cr(x-delta,y)) or nb.
//
// Vertical sweeps: one cluster of CS CTAs per frame, CTA k owns columns
// [k*w, (k+1)*w); thread = (column, chunk of DC disparities), lane =
// col*T + chunk.  Register layout per path: reg k holds (d0+k, d0+NR+k),
// NR = DC/2, so d-1 / d+1 neighbours are the adjacent registers except at the
// chunk edges (one shuffle + PRMT each).  Diagonal predecessors (x-1 / x+1 of
// the previous row) come from __shfl_up/down by T lanes; warp-edge columns read
// them from a double-buffered shared-memory halo that the neighbouring warp
// (or, at CTA edges, the neighbouring CTA through DSMEM) wrote.  One cluster
// barrier per row, split arrive/wait around the next row's cost computation.
#include <cooperative_groups.h>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace asd {
namespace v2 {

constexpr uint32_t INF2 = 0x7FFF7FFFu;

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b)
{
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// 4-byte asynchronous global->shared copy (LDGSTS); src_size 0 zero-fills.
__device__ __forceinline__ void cp_async4(uint32_t* sdst, const uint32_t* gsrc, bool valid)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" :: "r"(sa), "l"(gsrc), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory"); }

__device__ __forceinline__ void cluster_arrive()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
// mbarrier + TMA bulk copy (cp.async.bulk) helpers.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar)
{
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// one arrive announcing `bytes` of transaction for the phase, and bulk copies
// that only complete transaction bytes (several per phase)
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_tx(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity)
{
    asm volatile("{\n .reg .pred P;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                 " @!P bra WAIT_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}

// Relaxed arrive: no implicit release, so the partial-sum stores in flight are
// not waited for; the warps that wrote DSMEM halos fence first.
__device__ __forceinline__ void cluster_arrive_relaxed()
{
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void fence_cluster()
{
    asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait()
{
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

struct VArgs {
    DevParams p;
    int w;                    // columns per CTA (multiple of 32/T)
    int cs;                   // CTAs per frame (cluster size when NP == 3)
    const uint32_t* cl;       // census, [frames][H][W]
    const uint32_t* cr;
    long long sig_stride;
    const uint16_t* pin;      // K_up input: P_A | C << 8, u16 per cell, K_down's register order
    uint16_t* pouta;          // K_down output (same)
    uint16_t* pout16;         // K_up output P_AB (row-kernel layout)
    long long cell_stride;    // H*W*D
    long long pa_stride;      // frame stride of the P_A buffer: H * (cs*w) * D
    int ablate;               // timing experiments only (ASD_V2_ABLATE, builds with -DASD_ABLATE)
    const uint16_t* cbin;     // BLK: SGBM block cost, K_down's private layout (frame stride pa_stride)
    // frames wider than one cluster (ncta > cs): nseg = ncta / cs clusters per
    // frame ("segments"); the diagonal halos of the CTAs at a segment boundary
    // go through global memory as tagged words (ghalo: each u64 = the row
    // number + 1 in the high half, a 32-bit state word in the low half; zeroed
    // before each launch), so neither side needs a fence or a flag
    int ncta;                 // CTAs per frame (= cs for a frame in one cluster)
    int tma_cen;              // K_down: census rows staged by TMA bulk copies (guarded census buffers)
    unsigned long long* ghalo;   // [frames][nseg-1][2 dirs][2 slots][T][NR + 2]
};

// Ablation switches exist only in experiment builds (-DASD_ABLATE); in the
// production library they are compile-time zero, so no per-row test remains.
#ifdef ASD_ABLATE
#define ABL(a, bit) (((a).ablate & (bit)) != 0)
#else
#define ABL(a, bit) false
#endif

// ---------------------------------------------------------------- helpers
// u16x2 minimum of N registers as a balanced tree (any N: each level folds the
// upper ceil-half onto the lower half)
#ifndef ASD_TREE3
#define ASD_TREE3 1
#endif
template <int N>
__device__ __forceinline__ uint32_t tree_min(const uint32_t (&v)[N])
{
    if constexpr (N == 1) {
        return v[0];
    } else if constexpr (ASD_TREE3 && N > 2) {
        // three-input levels (VIMNMX3): 16 registers in 5 + 2 + 1 = 8 minima
        constexpr int M = (N + 2) / 3;
        uint32_t t[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            if (3 * i + 2 < N) t[i] = vmin2(vmin2(v[3 * i], v[3 * i + 1]), v[3 * i + 2]);
            else if (3 * i + 1 < N) t[i] = vmin2(v[3 * i], v[3 * i + 1]);
            else t[i] = v[3 * i];
        }
        return tree_min<M>(t);
    } else {
        uint32_t tr[N];
#pragma unroll
        for (int k = 0; k < N; ++k) tr[k] = v[k];
#pragma unroll
        for (int n = N; n > 1; n = (n + 1) / 2) {
#pragma unroll
            for (int k = 0; k < n / 2; ++k) tr[k] = vmin2(tr[k], tr[k + (n + 1) / 2]);
        }
        return tr[0];
    }
}

// Mp is the predecessor's min over d packed in both halves (M | M << 16);
// mout returns the new one the same way, so no scalar->packed IMAD is needed
// and the normalisation folds into one IADD3 per register.
template <int NR, int T>
__device__ __forceinline__ void path_update(const DevParams& p, int chunk, const uint32_t (&P)[NR],
                                            uint32_t Mp, const uint32_t (&C)[NR], uint32_t (&Ln)[NR],
                                            uint32_t& mout)
{
    const uint32_t P1P1 = (uint32_t)p.p1 * 0x10001u;
    const uint32_t MP2 = Mp + (uint32_t)p.p2 * 0x10001u;
    uint32_t Q[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) Q[k] = P[k] + P1P1;
    uint32_t qprev = INF2, qnext = INF2;
    if (T > 1) {
        const uint32_t u = __shfl_up_sync(FULL, Q[NR - 1], 1);
        const uint32_t v = __shfl_down_sync(FULL, Q[0], 1);
        if (chunk > 0) qprev = u;
        if (chunk < T - 1) qnext = v;
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const uint32_t dm1 = k > 0 ? Q[k - 1] : __byte_perm(qprev, Q[NR - 1], 0x5432);
        const uint32_t dp1 = k < NR - 1 ? Q[k + 1] : __byte_perm(Q[0], qnext, 0x5432);
        uint32_t t = vmin2(vmin2(dm1, dp1), P[k]);
        t = vmin2(t, MP2);
        Ln[k] = t + C[k] - Mp;
    }
    // min over the NR registers as a balanced tree (the asm min is opaque to the
    // compiler, so a running min would be a serial chain of NR dependent ops)
    const uint32_t macc = tree_min<NR>(Ln);
    uint32_t m = vmin2(macc, __byte_perm(macc, macc, 0x1032));      // (min, min)
#pragma unroll
    for (int o = 1; o < T; o <<= 1) m = vmin2(m, __shfl_xor_sync(FULL, m, o));
    mout = m;
}

// K_up output staging: 16-byte piece pi of a warp's (CPW columns x D) u16
// block is stored at stg_swz(pi).  A 16-byte shared access is served per
// quarter warp (8 lanes); both the writes (lane = (column, chunk), piece
// column * PPC + chunk * DC/8 + q) and the reads (8 consecutive pieces) must
// hit 8 distinct 16-byte bank groups.  PPC = 16 (T = 4): a quarter is 2 columns
// x 4 chunks, so the XOR takes the column's low bit and the chunk's high bit
// (piece bits 4 and 3); otherwise the column's low bits.
template <int PPC>
__device__ __forceinline__ int stg_swz(int pi)
{
    if constexpr (PPC == 16) return pi ^ ((((pi >> 3) & 1) << 1) | ((pi >> 4) & 1));
    else if constexpr (PPC == 32) return pi ^ ((pi >> 3) & 3);   // T = 8: a quarter = 1 column x 8 chunks
    else if constexpr (PPC == 12) return pi;                     // D = 96: conflict-free as laid out
    else return pi ^ ((pi / PPC) & ((PPC < 8 ? PPC : 8) - 1));
}

// ---------------------------------------------------------------- K_down / K_up
// Shared-memory census rows: the left row (w words) and, per chunk k, the
// slice of the right row its DC disparities read (w + DC - 1 words), placed at
// a bank offset of k*(DC + 32/T) mod 32 so the T chunks of a column never hit
// the same bank.  Three slots (rows i, i+1, i+2 in flight).
// experiment switches (A/B builds, tools/ab_bench.sh); production uses the defaults
#ifndef ASD_GSEG_PRE         // segment-boundary receive copies issued after the previous row's output
#define ASD_GSEG_PRE 1
#endif
#ifndef ASD_HROWB_SG
#define ASD_HROWB_SG 4            // SGBM row pass: pixels per register-buffered load group
#endif
#ifndef ASD_CEN_TMA
#define ASD_CEN_TMA 1             // K_down census rows by TMA bulk copies (one thread) instead of cp.async
#endif
#ifndef ASD_WTA_HALVES
#define ASD_WTA_HALVES 1          // D = 256 (R1): the three-pass half-width-window WTA kernel
#endif
#ifndef ASD_NSLOT
#define ASD_NSLOT 4               // 6 and 8 measured no faster (tools/runs/d3ab.sh)
#endif
#ifndef ASD_KU
#define ASD_KU 3                  // 5 measured no faster
#endif
constexpr int NSLOT = ASD_NSLOT;  // census rows in flight (K_down): rows i+1 .. i+NSLOT-1
constexpr int KU = ASD_KU;        // K_up input rows in flight (TMA bulk ring)

template <int DC, int T>
struct VGeom {
    static constexpr int NR = DC / 2;
    static constexpr int CPW = 32 / T;
    __host__ __device__ static int cstride(int w) { return ((w + DC - 1 + 31) / 32) * 32 + 32; }
    // chunk k's right-census slice starts at bank k * CPW: the T chunks of a
    // column read distinct banks
    __host__ __device__ static int coff(int k) { return (k * (32 / T)) & 31; }
    __host__ __device__ static int slot_words(int w) { return w + T * cstride(w); }
};

// RR (K_down only): the right view is the reference (R2, reading c24): a.cl is
// then the right census, a.cr the left one, and the matched column of local
// disparity j is x + delta instead of x - delta.
// BLK (SGBM, reading c19): the cost is the block cost CB of sgbm.cu, read
// by TMA in this kernel's private layout (K_down: CB ring instead of census
// staging; K_up: a CB ring beside the P_A ring), and the handoffs carry the
// wider partials without the cost bits: K_down writes P_A (u16), K_up P_AB.

// Segment-boundary receive (SEG instances, every warp calls it; gw is
// warp-uniform): the receiving lanes copy NQ pairs of tagged words from src
// to a private shared stage with cp.async (all in flight at once, no
// registers held), then move their low halves to dst; the warp retries until
// every tag equals `tag` (and traps after 2^24 tries instead of hanging).
// pre: the first copies were issued earlier (gissue in the kernel), so the
// first pass only waits for them.  The loop lives in one asm block (uniform
// branches only), so no data-dependent loop encloses the row's shuffles.
template <int NQ> struct GsegRecv;
template <> struct GsegRecv<5> {
    static __device__ __forceinline__ void run(bool gw, bool recv, const unsigned long long* src, unsigned dst,
                                               unsigned tag, unsigned stage, bool pre)
    {
        asm volatile("{\n"
                     " .reg .pred R, P, Q;\n"
                     " .reg .b64 A, B;\n"
                     " .reg .b32 a0, a1, b0, b1, N;\n"
                     " setp.eq.u32 Q, %0, 0;\n"
                     " @Q bra.uni GD_%=;\n"
                     " setp.ne.u32 R, %1, 0;\n"
                     " mov.b32 N, 0;\n"
                     " setp.ne.u32 P, %6, 0;\n"
                     " @P bra.uni GW_%=;\n"
                     "GR_%=:\n"
                     " @R cp.async.cg.shared.global [%5+0], [%2+0], 16;\n"
                     " @R cp.async.cg.shared.global [%5+16], [%2+16], 16;\n"
                     " @R cp.async.cg.shared.global [%5+32], [%2+32], 16;\n"
                     " @R cp.async.cg.shared.global [%5+48], [%2+48], 16;\n"
                     " @R cp.async.cg.shared.global [%5+64], [%2+64], 16;\n"
                     " cp.async.commit_group;\n"
                     "GW_%=:\n"
                     " cp.async.wait_group 0;\n"
                     " setp.ne.u32 P, %1, %1;\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+0];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+0], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+16];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+8], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+32];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+16], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+48];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+24], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+64];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+32], {a0, b0};\n"
                     " vote.sync.any.pred Q, P, 0xffffffff;\n"
                     " add.u32 N, N, 1;\n"
                     " setp.gt.and.u32 P, N, 16777216, Q;\n"
                     " @P trap;\n"
                     " @Q bra.uni GR_%=;\n"
                     "GD_%=:\n"
                     "}\n" :: "r"((unsigned)gw), "r"((unsigned)recv), "l"(src), "r"(dst), "r"(tag), "r"(stage),
                     "r"((unsigned)pre) : "memory");
    }
};
template <> struct GsegRecv<7> {
    static __device__ __forceinline__ void run(bool gw, bool recv, const unsigned long long* src, unsigned dst,
                                               unsigned tag, unsigned stage, bool pre)
    {
        asm volatile("{\n"
                     " .reg .pred R, P, Q;\n"
                     " .reg .b64 A, B;\n"
                     " .reg .b32 a0, a1, b0, b1, N;\n"
                     " setp.eq.u32 Q, %0, 0;\n"
                     " @Q bra.uni GD_%=;\n"
                     " setp.ne.u32 R, %1, 0;\n"
                     " mov.b32 N, 0;\n"
                     " setp.ne.u32 P, %6, 0;\n"
                     " @P bra.uni GW_%=;\n"
                     "GR_%=:\n"
                     " @R cp.async.cg.shared.global [%5+0], [%2+0], 16;\n"
                     " @R cp.async.cg.shared.global [%5+16], [%2+16], 16;\n"
                     " @R cp.async.cg.shared.global [%5+32], [%2+32], 16;\n"
                     " @R cp.async.cg.shared.global [%5+48], [%2+48], 16;\n"
                     " @R cp.async.cg.shared.global [%5+64], [%2+64], 16;\n"
                     " @R cp.async.cg.shared.global [%5+80], [%2+80], 16;\n"
                     " @R cp.async.cg.shared.global [%5+96], [%2+96], 16;\n"
                     " cp.async.commit_group;\n"
                     "GW_%=:\n"
                     " cp.async.wait_group 0;\n"
                     " setp.ne.u32 P, %1, %1;\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+0];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+0], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+16];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+8], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+32];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+16], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+48];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+24], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+64];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+32], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+80];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+40], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+96];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+48], {a0, b0};\n"
                     " vote.sync.any.pred Q, P, 0xffffffff;\n"
                     " add.u32 N, N, 1;\n"
                     " setp.gt.and.u32 P, N, 16777216, Q;\n"
                     " @P trap;\n"
                     " @Q bra.uni GR_%=;\n"
                     "GD_%=:\n"
                     "}\n" :: "r"((unsigned)gw), "r"((unsigned)recv), "l"(src), "r"(dst), "r"(tag), "r"(stage),
                     "r"((unsigned)pre) : "memory");
    }
};
template <> struct GsegRecv<9> {
    static __device__ __forceinline__ void run(bool gw, bool recv, const unsigned long long* src, unsigned dst,
                                               unsigned tag, unsigned stage, bool pre)
    {
        asm volatile("{\n"
                     " .reg .pred R, P, Q;\n"
                     " .reg .b64 A, B;\n"
                     " .reg .b32 a0, a1, b0, b1, N;\n"
                     " setp.eq.u32 Q, %0, 0;\n"
                     " @Q bra.uni GD_%=;\n"
                     " setp.ne.u32 R, %1, 0;\n"
                     " mov.b32 N, 0;\n"
                     " setp.ne.u32 P, %6, 0;\n"
                     " @P bra.uni GW_%=;\n"
                     "GR_%=:\n"
                     " @R cp.async.cg.shared.global [%5+0], [%2+0], 16;\n"
                     " @R cp.async.cg.shared.global [%5+16], [%2+16], 16;\n"
                     " @R cp.async.cg.shared.global [%5+32], [%2+32], 16;\n"
                     " @R cp.async.cg.shared.global [%5+48], [%2+48], 16;\n"
                     " @R cp.async.cg.shared.global [%5+64], [%2+64], 16;\n"
                     " @R cp.async.cg.shared.global [%5+80], [%2+80], 16;\n"
                     " @R cp.async.cg.shared.global [%5+96], [%2+96], 16;\n"
                     " @R cp.async.cg.shared.global [%5+112], [%2+112], 16;\n"
                     " @R cp.async.cg.shared.global [%5+128], [%2+128], 16;\n"
                     " cp.async.commit_group;\n"
                     "GW_%=:\n"
                     " cp.async.wait_group 0;\n"
                     " setp.ne.u32 P, %1, %1;\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+0];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+0], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+16];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+8], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+32];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+16], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+48];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+24], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+64];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+32], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+80];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+40], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+96];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+48], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+112];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+56], {a0, b0};\n"
                     " @R ld.shared.v2.b64 {A, B}, [%5+128];\n"
                     " @R mov.b64 {a0, a1}, A;\n"
                     " @R mov.b64 {b0, b1}, B;\n"
                     " @R setp.ne.or.u32 P, a1, %4, P;\n"
                     " @R setp.ne.or.u32 P, b1, %4, P;\n"
                     " @R st.shared.v2.b32 [%3+64], {a0, b0};\n"
                     " vote.sync.any.pred Q, P, 0xffffffff;\n"
                     " add.u32 N, N, 1;\n"
                     " setp.gt.and.u32 P, N, 16777216, Q;\n"
                     " @P trap;\n"
                     " @Q bra.uni GR_%=;\n"
                     "GD_%=:\n"
                     "}\n" :: "r"((unsigned)gw), "r"((unsigned)recv), "l"(src), "r"(dst), "r"(tag), "r"(stage),
                     "r"((unsigned)pre) : "memory");
    }
};
template <int NQ>
__device__ __forceinline__ void gseg_recv(bool gw, bool recv, const unsigned long long* src, unsigned dst,
                                          unsigned tag, unsigned stage, bool pre)
{
    GsegRecv<NQ>::run(gw, recv, src, dst, tag, stage, pre);
}

// SEG: the frame spans several clusters (segments) joined through global memory
// at their boundaries -- a separate instance, so frames in one cluster carry no
// trace of it (a data-dependent wait loop in the row loop makes the compiler
// guard every shuffle with WARPSYNC)
template <int DC, int T, int NP, bool UP, int DPL_ROW, bool RR = false, bool BLK = false, bool SEG = false>
__global__ void __launch_bounds__(DC >= 24 ? 512 : 1024, 1)
vsweep_kernel(VArgs a)
{
    using G = VGeom<DC, T>;
    constexpr int NR = G::NR;
    constexpr int CPW = G::CPW;
    extern __shared__ uint32_t smem[];
    const DevParams& p = a.p;
    const int W = p.W, H = p.H, D = p.D;
    const int nw = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = lane / T, chunk = lane % T;
    const int rank = NP == 3 ? (int)(blockIdx.x % (unsigned)a.cs) : (int)blockIdx.x;   // cluster rank
    const int seg = SEG ? (int)(blockIdx.x / (unsigned)a.cs) : 0;                       // cluster of the frame
    const int nseg = SEG ? a.ncta / a.cs : 1;
    const int frame = blockIdx.y;
    const int w = a.w;
    const int x0 = blockIdx.x * w;
    const int xl = warp * CPW + col;
    const int x = x0 + xl;
    const int cstr = G::cstride(w);
    const int sw = G::slot_words(w);
    const bool clustered = NP == 3 && a.cs > 1 && !ABL(a, 1);

    const int nslot = (UP || BLK) ? 0 : NSLOT;
    // the TMA-issuing thread (a middle warp instead measured slower: config C
    // 1821 vs 1956 frames/s, and no faster with segments)
    constexpr int tma_thread = 0;
    constexpr bool RING = UP || BLK;                 // TMA ring(s) of per-row input blocks
    constexpr int KR = (UP && BLK) ? 2 : KU;         // ring depth (two rings in BLK K_up)
    constexpr int NRING = (UP && BLK) ? 2 : 1;
    uint32_t* cens = smem;                   // [NSLOT][sw] (K_down): left row, then T right-row slices
    uint32_t* hL = cens + nslot * sw;        // [2][nw][T][NR]   (NP == 3)
    // halo state per chunk padded to HS = NR + 4 words: the T edge lanes of a
    // column (one per chunk) then hit distinct 16-byte bank groups
    constexpr int HS = NR + 4;
    uint32_t* hR = hL + 2 * nw * T * HS;
    uint32_t* hLM = hR + 2 * nw * T * HS;    // [2][nw]
    uint32_t* hRM = hLM + 2 * nw;
    // K_up output staging: one (CPW columns x D) u16 block per warp, so the
    // global stores of P_AB can be issued as contiguous 512-byte warp stores
    uint32_t* stg0 = NP == 3 ? hRM + 2 * nw : cens + nslot * sw;
    uint32_t* stg = stg0 + warp * (16 * DC);
    // input ring(s): KR rows of this CTA's (w columns x D) u16 block, TMA-loaded
    // (K_up: P_A | C, or P_A then CB for BLK; BLK K_down: CB)
    // (after the staging blocks in every instance: the blocks double as the
    // segment-boundary receive stage, also in K_down)
    uint16_t* ring = reinterpret_cast<uint16_t*>(stg0 + nw * 16 * DC);
    uint16_t* ring2 = ring + KR * w * D;             // BLK K_up: the CB ring
    uint64_t* mbar = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(ring + (RING ? NRING * KR * w * D : 0)) + 7) & ~uintptr_t(7));
    uint64_t* cbar = mbar + (RING ? KR : 0);         // [NSLOT] census full (K_down, tma_cen)
    // TMA census: the right slices are copied from 16-byte aligned starts,
    // cshift words before their first column (the same for every chunk and row)
    const int cshift = (!RING && a.tma_cen)
        ? (RR ? ((x0 + p.min_disp) & 3) : ((x0 - p.min_disp - (DC - 1)) & 3)) : 0;
    auto cen_ready = [&](int j) {                    // census row j landed (TMA staging)
        if (!RING && a.tma_cen) mbar_wait(cbar + j % NSLOT, (unsigned)((j / NSLOT) & 1));
    };
    // K_down -> K_up handoff in a private layout: the warp's (CPW columns x D)
    // block is contiguous and instruction q of lane l covers 16 bytes at
    // 512*q + 16*l, i.e. warp-contiguous stores and loads (row stride cs*w).
    const int wpad = a.ncta * a.w;

    const uint32_t* cl = a.cl + frame * a.sig_stride;
    const uint32_t* cr = a.cr + frame * a.sig_stride;

    if (NP == 3) {
        for (int i = threadIdx.x; i < 4 * nw * T * HS + 4 * nw; i += blockDim.x) hL[i] = 0u;
    }
    auto row_of = [&](int i) { return UP ? H - 1 - i : i; };
    // census rows -> shared memory with asynchronous copies (one commit group per
    // row).  K_up reads its costs from K_down's packed output instead.
    auto stage = [&](int yrow, int slot) {
        if (UP || ABL(a, 64)) { if (!UP) cp_async_commit(); return; }
        ASD_JITTER(6);
        ASD_ASSERT(slot >= 0 && slot < NSLOT && yrow >= 0 && yrow < H);
        uint32_t* sl = cens + slot * sw;
        const uint32_t* rl = cl + (long long)yrow * W;
        const uint32_t* rr = cr + (long long)yrow * W;
        if (a.tma_cen) {
            // one thread: the left row and the T right slices as bulk copies from
            // 16-byte aligned starts (the slices from cshift words before their
            // first column; columns outside the image are read from the guard
            // bands / neighbouring rows and never used: the cost masks them)
            if (threadIdx.x == tma_thread) {
                const unsigned nal = (unsigned)((w + DC - 1 + cshift + 3) & ~3);
                uint64_t* bar = cbar + slot;
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                mbar_arrive_expect(bar, (unsigned)(w * 4) + (unsigned)T * nal * 4u);
                bulk_g2s_tx(sl, rl + x0, (unsigned)(w * 4), bar);
#pragma unroll
                for (int k = 0; k < T; ++k) {
                    const int g0 = RR ? x0 + p.min_disp + DC * k : x0 - p.min_disp - DC * k - (DC - 1);
                    bulk_g2s_tx(sl + w + k * cstr + G::coff(k), rr + (g0 - cshift), nal * 4u, bar);
                }
            }
            return;
        }
        for (int i = threadIdx.x; i < w; i += blockDim.x) {
            const int gx = x0 + i;
            cp_async4(sl + i, gx < W ? rl + gx : rl, gx < W);
        }
        const int n = w + DC - 1;
#pragma unroll
        for (int k = 0; k < T; ++k) {
            uint32_t* dst = sl + w + k * cstr + G::coff(k);
            const int g0 = RR ? x0 + p.min_disp + DC * k : x0 - p.min_disp - DC * k - (DC - 1);
            for (int ii = threadIdx.x; ii < n; ii += blockDim.x) {
                const int gx = g0 + ii;
                const bool ok = gx >= 0 && gx < W;
                cp_async4(dst + ii, ok ? rr + gx : rr, ok);
            }
        }
        cp_async_commit();
    };
    const bool vcol = x >= p.R && x < W - p.R;
    auto cost = [&](int yrow, int slot, uint32_t (&C)[NR]) {
        const bool vx = vcol && yrow >= p.Q && yrow < H - p.Q && !ABL(a, 8);
        const uint32_t nbnb = (uint32_t)p.nb * 0x10001u;
        if (!vx) {
#pragma unroll
            for (int k = 0; k < NR; ++k) C[k] = nbnb;
            return;
        }
        const uint32_t* sl = cens + slot * sw;
        const uint32_t clv = sl[xl];
        // element for local disparity j (d = chunk*DC + j) at row[-j] (RR: row[+j])
        constexpr int SG = RR ? 1 : -1;
        const uint32_t* row = sl + w + chunk * cstr + G::coff(chunk) + xl + (RR ? 0 : DC - 1) + cshift;
        // local j valid iff j <= lim (the matched census window lies inside the image)
        const int lim = RR ? (W - p.R - 1) - (x + p.min_disp + chunk * DC)
                           : x - p.min_disp - p.R - chunk * DC;
        if (lim >= DC - 1) {
#pragma unroll
            for (int k = 0; k < NR; ++k)
                C[k] = __byte_perm(__popc(clv ^ row[SG * k]), __popc(clv ^ row[SG * (NR + k)]), 0x5410);
        } else {
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const uint32_t lo = k <= lim ? (uint32_t)__popc(clv ^ row[SG * k]) : (uint32_t)p.nb;
                const uint32_t hi = NR + k <= lim ? (uint32_t)__popc(clv ^ row[SG * (NR + k)]) : (uint32_t)p.nb;
                C[k] = __byte_perm(lo, hi, 0x5410);
            }
        }
    };
    const bool xin = x < W;
    // K_up: P_A and C of one row from K_down's packed words (reg k = cells d0+k, d0+NR+k)
    const unsigned row_bytes = (unsigned)(w * D * 2);
    auto issue_row_by = [&](int i) {                 // TMA the i-th processed row into the ring(s)
        if (RING && i < H && !ABL(a, 64)) {
            ASD_JITTER(4);
            const long long roff = ((long long)row_of(i) * wpad + x0) * D;
            uint64_t* bar = mbar + (i % KR);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_arrive_expect(bar, row_bytes * (unsigned)NRING);
            if (UP) bulk_g2s_tx(ring + (i % KR) * w * D, a.pin + frame * a.pa_stride + roff, row_bytes, bar);
            if (BLK) bulk_g2s_tx((UP ? ring2 : ring) + (i % KR) * w * D, a.cbin + frame * a.pa_stride + roff,
                                 row_bytes, bar);
        }
    };
    auto issue_row = [&](int i) { if (threadIdx.x == tma_thread) issue_row_by(i); };
    auto load_pin = [&](int i, uint32_t (&pa)[NR], uint32_t (&c)[NR]) {
        if (!ABL(a, 64)) mbar_wait(mbar + (i % KR), (unsigned)((i / KR) & 1));
        ASD_JITTER(5);
        const long long boff = (long long)(i % KR) * w * D + (warp * CPW) * D;
        const uint4* src = reinterpret_cast<const uint4*>(ring + boff) + lane;
        const uint4* src2 = reinterpret_cast<const uint4*>((UP ? ring2 : ring) + boff) + lane;
#pragma unroll
        for (int q = 0; q < NR / 4; ++q) {
            if constexpr (BLK) {                     // (P_A words and) CB words as they are
                const uint4 cv = src2[32 * q];
                c[4 * q] = cv.x; c[4 * q + 1] = cv.y; c[4 * q + 2] = cv.z; c[4 * q + 3] = cv.w;
                if constexpr (UP) {
                    const uint4 v = src[32 * q];
                    pa[4 * q] = v.x; pa[4 * q + 1] = v.y; pa[4 * q + 2] = v.z; pa[4 * q + 3] = v.w;
                }
            } else {
                const uint4 v = src[32 * q];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    pa[4 * q + j] = w4[j] & 0x00FF00FFu;
                    c[4 * q + j] = __byte_perm(w4[j], 0u, 0x4341);    // (C_lo, C_hi) as u16x2
                }
            }
        }
    };
    // Publish this row: __syncthreads orders the intra-CTA halos and staged census
    // rows; only the edge warps wrote into neighbouring CTAs (DSMEM), so only they
    // pay a cluster-scope fence before the relaxed cluster arrive.
    auto arrive = [&]() {
        ASD_JITTER(1);
        __syncthreads();
        if (clustered) {
            if (warp == 0 || warp == nw - 1) fence_cluster();
            cluster_arrive_relaxed();
        }
    };
    auto wait = [&]() { if (clustered) cluster_wait(); ASD_JITTER(2); };

    // halo write targets of this thread, slot 0 (slot 1 = + hslot / + nw), fixed for the kernel
    const int hslot = nw * T * HS;
    uint32_t* wL = nullptr; uint32_t* wLm = nullptr;   // edge lane col == CPW-1 -> column x+1
    uint32_t* wR = nullptr; uint32_t* wRm = nullptr;   // edge lane col == 0     -> column x-1
    if (NP == 3) {
        if (col == CPW - 1) {
            if (warp + 1 < nw) {
                wL = hL + ((warp + 1) * T + chunk) * HS;
                wLm = hLM + warp + 1;
            } else if (rank + 1 < a.cs) {
                cg::cluster_group cl_g = cg::this_cluster();
                wL = cl_g.map_shared_rank(hL + chunk * HS, rank + 1);
                wLm = cl_g.map_shared_rank(hLM, rank + 1);
            }
        }
        if (col == 0) {
            if (warp > 0) {
                wR = hR + ((warp - 1) * T + chunk) * HS;
                wRm = hRM + warp - 1;
            } else if (rank > 0) {
                cg::cluster_group cl_g = cg::this_cluster();
                wR = cl_g.map_shared_rank(hR + ((nw - 1) * T + chunk) * HS, rank - 1);
                wRm = cl_g.map_shared_rank(hRM + nw - 1, rank - 1);
            }
        }
    }

    // segment boundaries (nseg > 1): the last CTA of segment s and the first of
    // s+1 exchange their edge columns' diagonal states through global memory;
    // boundary b = (s, s+1); the consumer is at most one row behind or ahead
    // (each needs the other's previous row), so two slots suffice.  Each word
    // travels with its row tag (row + 1) in one 8-byte store, so a receiver that
    // sees every tag of the slot has the whole state: no release fence on the
    // sender (it would wait for the row's partial stores), no acquire fence.
    const int nb = nseg - 1;
    constexpr int GQ = NR + 2;                    // tagged words per chunk and slot (state, M, pad)
    auto gh = [&](int b, int dir) {               // halo block of boundary b, direction 0 = L, 1 = R
        return a.ghalo + ((((long long)frame * nb + b) * 2 + dir) * 2) * T * GQ;
    };
    const bool gsendL = SEG && NP == 3 && nseg > 1 && rank == a.cs - 1 && seg + 1 < nseg && warp == nw - 1 && col == CPW - 1;
    const bool gsendR = SEG && NP == 3 && nseg > 1 && rank == 0 && seg > 0 && warp == 0 && col == 0;
    // warp-uniform: this warp receives a boundary halo (all its lanes wait, the
    // edge lanes read), so the shuffles after the wait stay convergent
    const bool gwL = SEG && NP == 3 && nseg > 1 && rank == 0 && seg > 0 && warp == 0;
    const bool gwR = SEG && NP == 3 && nseg > 1 && rank == a.cs - 1 && seg + 1 < nseg && warp == nw - 1;
    // Segment boundary, row i (i >= 1): row i-1 of the neighbouring segment's
    // edge column into this warp's own (otherwise unused) halo slot (i + 1) & 1
    // -- received at the end of row i-1, before the cluster wait, so its L2
    // round trip overlaps the barrier; at i = 0 the slot holds its initial
    // zeros (outside predecessor).
    auto grecv = [&](int i) {
        const int rs = (i + 1) & 1;
        const bool gw = (gwL || gwR) && i > 0 && i < H;
        const bool rcv = gw && ((gwL && col == 0) || (gwR && col == CPW - 1));
        const unsigned long long* src = (gwL ? gh(seg - 1, 0) : gh(seg, 1)) + (rs * T + chunk) * GQ;
        uint32_t* dst = (gwL ? hL : hR) + ((rs * nw + warp) * T + chunk) * HS;
        // stage: the warp's K_up output block (free between partial_out and
        // the next row's), GQ tagged words per chunk
        gseg_recv<GQ / 2>(gw, rcv, src, smem_u32(dst), (unsigned)i, smem_u32(stg) + chunk * GQ * 8, ASD_GSEG_PRE != 0);
        ASD_JITTER(9);
    };
    // the first copies of row i's receive, issued after the previous row's
    // partial-sum output (the staging block is free from then on)
    auto gissue = [&](int i) {
        const bool gw = (gwL || gwR) && i > 0 && i < H;
        if (gw && ((gwL && col == 0) || (gwR && col == CPW - 1))) {
            const int rs = (i + 1) & 1;
            const unsigned long long* src = (gwL ? gh(seg - 1, 0) : gh(seg, 1)) + (rs * T + chunk) * GQ;
            const unsigned st = smem_u32(stg) + chunk * GQ * 8;
#pragma unroll
            for (int q = 0; q < GQ / 2; ++q)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(st + 16 * q), "l"(src + 2 * q) : "memory");
        }
        if (gw) cp_async_commit();
    };
    // tagged 8-byte stores of one chunk's state (row i, tag i + 1)
    auto gsend = [&](unsigned long long* h, const uint32_t (&Lx)[NR], uint32_t Mx, int i) {
        const unsigned long long t = (unsigned long long)(unsigned)(i + 1) << 32;
#pragma unroll
        for (int q = 0; q < GQ / 2; ++q) {
            const uint32_t lo = 2 * q < NR ? Lx[2 * q] : Mx;
            const uint32_t hi = 2 * q + 1 < NR ? Lx[2 * q + 1] : Mx;
            asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};\n"
                         :: "l"(h + 2 * q), "l"(t | lo), "l"(t | hi) : "memory");
        }
    };

    uint32_t Lv[NR], Ll[NR], Lr[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) { Lv[k] = 0u; Ll[k] = 0u; Lr[k] = 0u; }
    uint32_t Mv = 0u, Ml = 0u, Mr = 0u;
    uint32_t C[NR];
    uint32_t PA[NR];

    // ---- the per-row pieces shared by both synchronisation schemes
    // diagonal paths of row i from the predecessors of row i-1 (halo slot rs)
    auto diagonals = [&](int i) {
        const int rs = (i + 1) & 1;              // slot written at row i-1
        uint32_t Pp[NR], Mp;
        // path "L": predecessor column x-1 (down-right / up-right)
#pragma unroll
        for (int k = 0; k < NR; ++k) Pp[k] = __shfl_up_sync(FULL, Ll[k], T);
        Mp = __shfl_up_sync(FULL, Ml, T);
        if (col == 0) {
            const uint32_t* hs = hL + ((rs * nw + warp) * T + chunk) * HS;
            const uint4* h = reinterpret_cast<const uint4*>(hs);
#pragma unroll
            for (int q = 0; q < NR / 4; ++q) {
                const uint4 v = h[q];
                Pp[4 * q] = v.x; Pp[4 * q + 1] = v.y; Pp[4 * q + 2] = v.z; Pp[4 * q + 3] = v.w;
            }
            Mp = (SEG && gwL) ? hs[NR] : hLM[rs * nw + warp];
        }
        path_update<NR, T>(p, chunk, Pp, Mp, C, Ll, Ml);
        // path "R": predecessor column x+1 (down-left / up-left)
#pragma unroll
        for (int k = 0; k < NR; ++k) Pp[k] = __shfl_down_sync(FULL, Lr[k], T);
        Mp = __shfl_down_sync(FULL, Mr, T);
        if (col == CPW - 1) {
            const uint32_t* hs = hR + ((rs * nw + warp) * T + chunk) * HS;
            const uint4* h = reinterpret_cast<const uint4*>(hs);
#pragma unroll
            for (int q = 0; q < NR / 4; ++q) {
                const uint4 v = h[q];
                Pp[4 * q] = v.x; Pp[4 * q + 1] = v.y; Pp[4 * q + 2] = v.z; Pp[4 * q + 3] = v.w;
            }
            Mp = (SEG && gwR) ? hs[NR] : hRM[rs * nw + warp];
        }
        path_update<NR, T>(p, chunk, Pp, Mp, C, Lr, Mr);
        // columns beyond the image act as "outside" predecessors: zero state
        if (!xin) {
#pragma unroll
            for (int k = 0; k < NR; ++k) { Ll[k] = 0u; Lr[k] = 0u; }
            Ml = Mr = 0u;
        }
    };
    // halos of row i for the next row (slot i & 1)
    auto write_halos = [&](int i) {
        const int ws = i & 1;
        ASD_JITTER(3);
        if (wL) {                        // my "L" state feeds column x+1 next row
            uint4* d4 = reinterpret_cast<uint4*>(wL + ws * hslot);
#pragma unroll
            for (int q = 0; q < NR / 4; ++q) d4[q] = make_uint4(Ll[4 * q], Ll[4 * q + 1], Ll[4 * q + 2], Ll[4 * q + 3]);
            if (chunk == 0) wLm[ws * nw] = Ml;
        }
        if (wR) {                        // my "R" state feeds column x-1 next row
            uint4* d4 = reinterpret_cast<uint4*>(wR + ws * hslot);
#pragma unroll
            for (int q = 0; q < NR / 4; ++q) d4[q] = make_uint4(Lr[4 * q], Lr[4 * q + 1], Lr[4 * q + 2], Lr[4 * q + 3]);
            if (chunk == 0) wRm[ws * nw] = Mr;
        }
        // segment boundary: the edge column's state as tagged words
        if (gsendL) gsend(gh(seg, 0) + (ws * T + chunk) * GQ, Ll, Ml, i);
        if (gsendR) gsend(gh(seg - 1, 1) + (ws * T + chunk) * GQ, Lr, Mr, i);
    };
    // vertical path: predecessor = own column
    auto vertical = [&]() {
        if (!ABL(a, 32)) {
            uint32_t Ln[NR], mnew;
            path_update<NR, T>(p, chunk, Lv, Mv, C, Ln, mnew);
#pragma unroll
            for (int k = 0; k < NR; ++k) Lv[k] = Ln[k];
            Mv = mnew;
        }
        if (!xin) {
#pragma unroll
            for (int k = 0; k < NR; ++k) Lv[k] = 0u;
            Mv = 0u;
        }
    };
    // partial sum of row y out
    auto partial_out = [&](int y) {
        if (ABL(a, 2)) return;
        uint32_t s[NR];
#pragma unroll
        for (int k = 0; k < NR; ++k) s[k] = NP == 3 ? Lv[k] + Ll[k] + Lr[k] : Lv[k];
        if (!UP) {
            // P_A (<= 255) | C << 8 (C <= 63): the up sweep needs no census
            // (BLK: P_A alone, the up sweep reads CB itself)
            uint4* dst = reinterpret_cast<uint4*>(a.pouta + frame * a.pa_stride +
                                                  ((long long)y * wpad + (x - col)) * D) + lane;
            constexpr uint32_t CS = BLK ? 0u : 256u;
#pragma unroll
            for (int q = 0; q < NR / 4; ++q)
                dst[32 * q] = make_uint4(s[4 * q] + C[4 * q] * CS, s[4 * q + 1] + C[4 * q + 1] * CS,
                                         s[4 * q + 2] + C[4 * q + 2] * CS, s[4 * q + 3] + C[4 * q + 3] * CS);
        } else {
            // P_AB (<= 510) | C << 9: the right->left row sweep needs no census
#pragma unroll
            for (int k = 0; k < NR; ++k) s[k] += PA[k] + C[k] * (BLK ? 0u : 512u);
            uint32_t o[NR];
            if (DPL_ROW == 8) {
                // row-kernel register order for 8 disparities per lane: word j of
                // group g = (d 8g+j, d 8g+4+j)
#pragma unroll
                for (int g = 0; g < DC / 8; ++g) {
                    const int kk = 8 * g < NR ? 8 * g : 8 * g - NR;
                    const uint32_t sel = 8 * g < NR ? 0x5410u : 0x7632u;
#pragma unroll
                    for (int j = 0; j < 4; ++j) o[4 * g + j] = __byte_perm(s[kk + j], s[kk + 4 + j], sel);
                }
            } else if (DPL_ROW == 4) {
#pragma unroll
                for (int g = 0; g < DC / 4; ++g) {
                    const int kk = 4 * g < NR ? 4 * g : 4 * g - NR;
                    const uint32_t sel = 4 * g < NR ? 0x5410u : 0x7632u;
                    o[2 * g] = __byte_perm(s[kk], s[kk + 2], sel);
                    o[2 * g + 1] = __byte_perm(s[kk + 1], s[kk + 3], sel);
                }
            } else {
#pragma unroll
                for (int g = 0; g < DC / 2; ++g) {
                    const int kk = 2 * g < NR ? 2 * g : 2 * g - NR;
                    const uint32_t sel = 2 * g < NR ? 0x5410u : 0x7632u;
                    o[g] = __byte_perm(s[kk], s[kk + 1], sel);
                }
            }
            // natural [x][d] layout through the warp's staging block.  16-byte
            // piece p of the block (column p / PPC) is stored at p ^ (column &
            // SWZ): without it the 32 lanes of one store instruction fall into
            // two 16-byte bank groups (a 16-way conflict).
            constexpr int PPC = DC * T / 8;                   // 16-byte pieces per column
            uint4* sb = reinterpret_cast<uint4*>(stg);
            const int pbase = col * PPC + chunk * (DC / 8);
#pragma unroll
            for (int q = 0; q < NR / 4; ++q)
                sb[stg_swz<PPC>(pbase + q)] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
            __syncwarp();
            uint4* dst = reinterpret_cast<uint4*>(a.pout16 + frame * a.cell_stride + ((long long)y * W + (x - col)) * D);
#pragma unroll
            for (int q = 0; q < NR / 4; ++q) {
                const int pi = 32 * q + lane;                 // 16-byte piece of the block
                if (x - col + pi / PPC < W) dst[pi] = sb[stg_swz<PPC>(pi)];
            }
            __syncwarp();
        }
    };

    // ============ legacy scheme: one CTA barrier + one cluster barrier per row
    if (NP == 3 && a.cs > 1 && ABL(a, 1)) { cluster_arrive(); cluster_wait(); }
    if (RING) {
        if (threadIdx.x == 0) {
            for (int s2 = 0; s2 < KR; ++s2) mbar_init(mbar + s2, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        for (int i0 = 0; i0 < KR; ++i0) issue_row(i0);
    } else if (a.tma_cen) {
        if (threadIdx.x == 0) {
            for (int s2 = 0; s2 < NSLOT; ++s2) mbar_init(cbar + s2, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        for (int i0 = 0; i0 < NSLOT - 1; ++i0)
            if (i0 < H) stage(row_of(i0), i0);
    } else {
        for (int i0 = 0; i0 < NSLOT - 1; ++i0)
            if (i0 < H) stage(row_of(i0), i0);
        cp_async_wait<0>();
    }
    arrive();
    wait();
    if (RING) load_pin(0, PA, C);
    else { cen_ready(0); cost(row_of(0), 0, C); }

    for (int i = 0; i < H; ++i) {
        const int y = row_of(i);
        if (i > 0) wait();
        if (NP == 3 && !ABL(a, 4)) diagonals(i);
        // ---- halos for the next row: written before the vertical path so the
        // DSMEM stores are in flight while it runs
        if (NP == 3) write_halos(i);
        vertical();
        // ---- K_down: stage row i+NSLOT-1 (async), make row i+1's copies complete, publish
        if (!RING) {
            if (i + NSLOT - 1 < H) stage(row_of(i + NSLOT - 1), (i + NSLOT - 1) % NSLOT);
            else if (!a.tma_cen) cp_async_commit();  // keep one group per row
            if (!a.tma_cen) cp_async_wait<NSLOT - 2>();
        }
        arrive();
        issue_row(i + KR);                            // ring input: row i's slot is free now
        // ---- partial sum out (after the release so it does not wait on these stores)
        partial_out(y);
        if (SEG && ASD_GSEG_PRE) gissue(i + 1);
        // ---- next row's cost while the barrier completes
        if (i + 1 < H) {
            if (RING) load_pin(i + 1, PA, C);
            else { cen_ready(i + 1); cost(row_of(i + 1), (i + 1) % NSLOT, C); }
        }
        if (SEG) grecv(i + 1);
    }
    wait();                                          // pairs with the last arrive
    if (NP == 3 && a.cs > 1 && ABL(a, 1)) { cluster_arrive(); cluster_wait(); }
}


// ---------------------------------------------------------------- K_row
struct RArgs {
    DevParams p;
    const uint32_t* cl;
    const uint32_t* cr;
    long long sig_stride;
    uint16_t* pab;            // [frames][H][W][D]: P_AB in (row-kernel layout); S out (natural order)
    uint8_t* stash;           // [frames][H][W][D] left->right path, u8
    long long cell_stride;
    FrameScratch fs;          // WTA outputs for K5
    long long px_stride;
    int nbuf;                 // rows of the WTA kernel's S window
    int bstride;              // u16 per window row (D + 2)
    uint32_t p1x2, p2x2;      // P1, P2 in both u16 halves
    const uint16_t* cb;       // SGBM: block cost in the sweeps' private layout
    long long cb_stride;      // its frame stride (H * wpad * D)
    int wpad;                 // its row length in columns (cs * w)
};

constexpr uint32_t NONE16 = 0xFFFFu;

// Uniqueness + sub-pixel from (d*, S(d*), s2, S(d*-1), S(d*+1)) -- K4 semantics
// (post.cu): PAPER.md P:289, readings c8, c13.
__device__ __forceinline__ void finish_wta(const DevParams& p, int dstar, uint32_t s0, uint32_t s2,
                                           uint32_t cm, uint32_t cp, bool& unique_fail, float& disp)
{
    unique_fail = p.uniq >= 0 && s2 != NONE16 &&
                  (long long)s0 * (100 + (long long)p.uniq) >= (long long)s2 * 100;
    float off = 0.0f;
    if (p.subpix && dstar >= 1 && dstar <= p.D - 2 && cm != NONE16 && cp != NONE16) {
        const int den = (int)cm - 2 * (int)s0 + (int)cp;
        if (den > 0) {
            off = __fdiv_rn((float)((int)cm - (int)cp), (float)(2 * den));
            off = fminf(fmaxf(off, -0.5f), 0.5f);
        }
    }
    disp = __fadd_rn((float)(p.min_disp + dstar), off);
}

#ifndef ASD_WTA_PAD
#define ASD_WTA_PAD 2
#define ASD_WTA_CHUNK 4
#endif
constexpr int WTA_PAD = ASD_WTA_PAD;      // u16 of padding per window row
constexpr int WTA_CHUNK = ASD_WTA_CHUNK;  // bytes per cp.async of the window fill

template <int D> struct RowGeom {
    static constexpr int DPL = D > 128 ? 8 : D > 64 ? 4 : 2;   // disparities per lane
    static constexpr int NRR = DPL / 2;              // u16x2 registers per lane
    static constexpr int ACT = D / DPL;              // active lanes
    static constexpr int NB = D + 40;                // rows of the S window (D + 32 + one sub-group)
    static constexpr int BS = D + WTA_PAD;           // u16 per WTA window row (WTA_PAD = 2: an odd number of
                                                     // 4-byte words, so the 32 lanes of the
                                                     // diagonal (right-view) scan hit 32 banks
    static constexpr int KS = D <= 16 ? 4 : D <= 32 ? 5 : D <= 64 ? 6 : D <= 128 ? 7 : 8;   // ceil(log2 D)
};

// Left view, one pixel per lane, from its window row r[0..D) (natural order).
// Pass 1: packed u16 keys (S << KS) | d, u16x2 min.  Pass 2: min of S with
// d*-1..d*+1 poisoned (the row belongs to this lane alone), then restored.
// WIDE: S may exceed 2^(16 - KS) (SGBM block costs, D1 volumes): u32 keys.
#ifndef ASD_HROW_CFROMP
#define ASD_HROW_CFROMP 0         // 1: the row kernel's left->right pass takes C from the P_AB | C words
#endif
template <int D, bool WIDE>
__device__ __forceinline__ void wta_left_lane(const DevParams& p, uint16_t* r, int& dstar, bool& uf, float& disp)
{
    constexpr int KS = RowGeom<D>::KS;
    const uint32_t* r32 = reinterpret_cast<const uint32_t*>(r);     // rows are 4-byte aligned
    uint32_t kb;
    if constexpr (WIDE) {
        uint32_t ka = 0xFFFFFFFFu, kb2 = 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < D; q += 2) {
            const uint32_t v = r32[q / 2];
            ka = min(ka, ((v & 0xFFFFu) << KS) | (uint32_t)q);
            kb2 = min(kb2, ((v >> 16) << KS) | (uint32_t)(q + 1));
        }
        kb = min(ka, kb2);
    } else {
        uint32_t ka = 0xFFFFFFFFu, kb2 = 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < D; q += 4) {
            const uint32_t v0 = r32[q / 2], v1 = r32[q / 2 + 1];
            ka = vmin2(ka, v0 * (1u << KS) + ((uint32_t)q | ((uint32_t)(q + 1) << 16)));
            kb2 = vmin2(kb2, v1 * (1u << KS) + ((uint32_t)(q + 2) | ((uint32_t)(q + 3) << 16)));
        }
        const uint32_t kmin = vmin2(ka, kb2);
        kb = min(kmin & 0xFFFFu, kmin >> 16);
    }
    dstar = (int)(kb & ((1u << KS) - 1u));
    const uint32_t s0 = kb >> KS;
    const uint32_t cm = dstar >= 1 ? r[dstar - 1] : NONE16;
    const uint32_t cp = dstar + 1 < D ? r[dstar + 1] : NONE16;
    if (dstar >= 1) r[dstar - 1] = (uint16_t)NONE16;
    r[dstar] = (uint16_t)NONE16;
    if (dstar + 1 < D) r[dstar + 1] = (uint16_t)NONE16;
    uint32_t vm = 0xFFFFFFFFu, vm2 = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < D; q += 4) {
        vm = vmin2(vm, r32[q / 2]);
        vm2 = vmin2(vm2, r32[q / 2 + 1]);
    }
    vm = vmin2(vm, vm2);
    if (dstar >= 1) r[dstar - 1] = (uint16_t)cm;
    r[dstar] = (uint16_t)s0;
    if (dstar + 1 < D) r[dstar + 1] = (uint16_t)cp;
    finish_wta(p, dstar, s0, min(vm & 0xFFFFu, vm >> 16), cm, cp, uf, disp);
}

// Right view, one right pixel per lane: S_R(d) = S(xr + delta(d), d) lies on a
// diagonal of the window (row (r0 + d) mod NB, column d); nd >= 1 defined d.
template <int D>
__device__ __forceinline__ void wta_right_lane(const DevParams& p, uint16_t* sb, int NB, int r0, int nd,
                                               int& dstar, bool& uf, float& disp)
{
    constexpr int BS = RowGeom<D>::BS, KS = RowGeom<D>::KS;
    constexpr int STEP = BS + 1;
    const int dwrap = NB - r0;                       // first d whose row wraps to 0
    const uint16_t* b0 = sb + r0 * BS;
    const uint16_t* b1 = b0 - NB * BS;
    const int n0 = min(nd, dwrap);
    uint32_t kmin = 0xFFFFFFFFu, kmin2 = 0xFFFFFFFFu;
    int d = 0;
#pragma unroll 2
    for (; d + 1 < n0; d += 2) {
        kmin = min(kmin, ((uint32_t)b0[d * STEP] << KS) | (uint32_t)d);
        kmin2 = min(kmin2, ((uint32_t)b0[(d + 1) * STEP] << KS) | (uint32_t)(d + 1));
    }
    if (d < n0) { kmin = min(kmin, ((uint32_t)b0[d * STEP] << KS) | (uint32_t)d); ++d; }
#pragma unroll 2
    for (; d + 1 < nd; d += 2) {
        kmin = min(kmin, ((uint32_t)b1[d * STEP] << KS) | (uint32_t)d);
        kmin2 = min(kmin2, ((uint32_t)b1[(d + 1) * STEP] << KS) | (uint32_t)(d + 1));
    }
    if (d < nd) kmin = min(kmin, ((uint32_t)b1[d * STEP] << KS) | (uint32_t)d);
    kmin = min(kmin, kmin2);
    dstar = (int)(kmin & ((1u << KS) - 1u));
    const uint32_t s0 = kmin >> KS;
    auto at = [&](int d) -> uint16_t* { return const_cast<uint16_t*>((d < dwrap ? b0 : b1) + d * STEP); };
    const uint32_t cm = dstar >= 1 ? *at(dstar - 1) : NONE16;
    const uint32_t cp = dstar + 1 < nd ? *at(dstar + 1) : NONE16;
    if (dstar >= 1) *at(dstar - 1) = (uint16_t)NONE16;
    *at(dstar) = (uint16_t)NONE16;
    if (dstar + 1 < nd) *at(dstar + 1) = (uint16_t)NONE16;
    uint32_t vm = NONE16, vmb = NONE16;
    d = 0;
#pragma unroll 2
    for (; d + 1 < n0; d += 2) { vm = min(vm, (uint32_t)b0[d * STEP]); vmb = min(vmb, (uint32_t)b0[(d + 1) * STEP]); }
    if (d < n0) { vm = min(vm, (uint32_t)b0[d * STEP]); ++d; }
#pragma unroll 2
    for (; d + 1 < nd; d += 2) { vm = min(vm, (uint32_t)b1[d * STEP]); vmb = min(vmb, (uint32_t)b1[(d + 1) * STEP]); }
    if (d < nd) vm = min(vm, (uint32_t)b1[d * STEP]);
    vm = min(vm, vmb);
    if (dstar >= 1) *at(dstar - 1) = (uint16_t)cm;
    *at(dstar) = (uint16_t)s0;
    if (dstar + 1 < nd) *at(dstar + 1) = (uint16_t)cp;
    finish_wta(p, dstar, s0, vm, cm, cp, uf, disp);
}

// Right view on the linear stage window: the lane's diagonal S(xr + delta(d), d)
// is b0[d * (BS + 1)] for every d (no wrap), all D defined; fully unrolled
// (immediate offsets), packed u16 keys as in the left view, second pass over
// the same diagonal with d*-1..d*+1 poisoned and then restored.
template <int D, bool WIDE>
__device__ __forceinline__ void wta_right_lin(const DevParams& p, uint16_t* b0, int& dstar, bool& uf, float& disp)
{
    constexpr int BS = RowGeom<D>::BS, KS = RowGeom<D>::KS, STEP = BS + 1;
    auto pair = [&](int d) -> uint32_t {
        return __byte_perm((uint32_t)b0[d * STEP], (uint32_t)b0[(d + 1) * STEP], 0x5410);
    };
    uint32_t kb;
    if constexpr (WIDE) {
        uint32_t k0 = 0xFFFFFFFFu, k1 = 0xFFFFFFFFu;
#pragma unroll
        for (int d = 0; d < D; d += 2) {
            k0 = min(k0, ((uint32_t)b0[d * STEP] << KS) | (uint32_t)d);
            k1 = min(k1, ((uint32_t)b0[(d + 1) * STEP] << KS) | (uint32_t)(d + 1));
        }
        kb = min(k0, k1);
    } else {
        // packed keys, plus the minimum S of each 8-disparity block for the
        // second-best search below (no second pass over the diagonal)
        uint32_t k0 = 0xFFFFFFFFu, k1 = 0xFFFFFFFFu, bm[D / 8];
#pragma unroll
        for (int d = 0; d < D; d += 4) {
            const uint32_t pa = pair(d), pb = pair(d + 2);
            k0 = vmin2(k0, pa * (1u << KS) + ((uint32_t)d | ((uint32_t)(d + 1) << 16)));
            k1 = vmin2(k1, pb * (1u << KS) + ((uint32_t)(d + 2) | ((uint32_t)(d + 3) << 16)));
            bm[d / 8] = (d % 8 == 0) ? vmin2(pa, pb) : vmin2(bm[d / 8], vmin2(pa, pb));
        }
        const uint32_t km = vmin2(k0, k1);
        kb = min(km & 0xFFFFu, km >> 16);
        dstar = (int)(kb & ((1u << KS) - 1u));
        const uint32_t s0 = kb >> KS;
        const uint16_t* c0 = b0 + dstar * STEP;
        const uint32_t cm = dstar >= 1 ? c0[-STEP] : NONE16;
        const uint32_t cp = dstar + 1 < D ? c0[STEP] : NONE16;
        // second best over |d - d*| >= 2: whole blocks clear of d*-1..d*+1 from
        // their minima, the (one or two) blocks holding them element by element
        const int blo = max(dstar - 1, 0) >> 3, bhi = min(dstar + 1, D - 1) >> 3;
        uint32_t sec = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 0; b < D / 8; ++b)
            if (b < blo || b > bhi) sec = vmin2(sec, bm[b]);
        uint32_t s2 = min(sec & 0xFFFFu, sec >> 16);
        for (int b = blo; b <= bhi; ++b)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int d = 8 * b + j;
                if (d < dstar - 1 || d > dstar + 1) s2 = min(s2, (uint32_t)b0[d * STEP]);
            }
        finish_wta(p, dstar, s0, s2, cm, cp, uf, disp);
        return;
    }
    dstar = (int)(kb & ((1u << KS) - 1u));
    const uint32_t s0 = kb >> KS;
    uint16_t* c0 = b0 + dstar * STEP;
    const uint32_t cm = dstar >= 1 ? c0[-STEP] : NONE16;
    const uint32_t cp = dstar + 1 < D ? c0[STEP] : NONE16;
    if (dstar >= 1) c0[-STEP] = (uint16_t)NONE16;
    c0[0] = (uint16_t)NONE16;
    if (dstar + 1 < D) c0[STEP] = (uint16_t)NONE16;
    uint32_t v0 = 0xFFFFFFFFu, v1 = 0xFFFFFFFFu;
#pragma unroll
    for (int d = 0; d < D; d += 4) {
        v0 = vmin2(v0, pair(d));
        v1 = vmin2(v1, pair(d + 2));
    }
    const uint32_t vm = vmin2(v0, v1);
    if (dstar >= 1) c0[-STEP] = (uint16_t)cm;
    c0[0] = (uint16_t)s0;
    if (dstar + 1 < D) c0[STEP] = (uint16_t)cp;
    finish_wta(p, dstar, s0, min(vm & 0xFFFFu, vm >> 16), cm, cp, uf, disp);
}


// Horizontal-path step for one warp (lane = DPL disparities).  Register
// layout: DPL == 4 -> A = (d0, d0+2), B = (d0+1, d0+3); DPL == 2 -> (d0, d0+1).
// row_cost: the matching costs of this lane's disparities at x (census).
template <int D, bool FAST = false>
__device__ __forceinline__ void row_cost(const DevParams& p, int lane, uint32_t clv, bool vx, int lim,
                                         const uint32_t (&wnd)[RowGeom<D>::DPL],
                                         uint32_t (&C)[RowGeom<D>::NRR])
{
    constexpr int DPL = RowGeom<D>::DPL, NRR = RowGeom<D>::NRR;
    const int d0 = lane * DPL;
    uint32_t c[DPL];
    if (FAST || (vx && lim >= D - 1)) {               // warp-uniform fast path: all d valid
#pragma unroll
        for (int j = 0; j < DPL; ++j) c[j] = __popc(clv ^ wnd[j]);
    } else {
#pragma unroll
        for (int j = 0; j < DPL; ++j) c[j] = (vx && d0 + j <= lim) ? (uint32_t)__popc(clv ^ wnd[j]) : (uint32_t)p.nb;
    }
    // register k = (d0 + k, d0 + NRR + k)
#pragma unroll
    for (int k = 0; k < NRR; ++k) C[k] = __byte_perm(c[k], c[NRR + k], 0x5410);
}

// row_rec: L_r(x) from the predecessor state Lp (zero at the line start) and
// its min M packed in both halves (M | M << 16; 0 at the start); returns the
// new packed min.  The warp reduction runs on the (min, min) word of each
// lane: the u32 minimum over lanes of (m << 16 | m) is the packed minimum, so
// no unpack/repack is needed, and P1 / P2 come packed from the kernel
// arguments (constant-bank operands).
// eprev / enext: INF2 in the lanes without a d-1 / d+1 neighbour lane (lane 0 /
// lane ACT-1), 0 elsewhere -- ORed into the shuffled words (every Q half is
// < 2^15, so Q | 0x7FFF = INF), which keeps the edge test out of the loop.
template <int D>
__device__ __forceinline__ uint32_t row_rec(uint32_t p1x2, uint32_t p2x2, uint32_t eprev, uint32_t enext,
                                            const uint32_t (&C)[RowGeom<D>::NRR],
                                            const uint32_t (&Lp)[RowGeom<D>::NRR], uint32_t Mpk,
                                            uint32_t (&Ln)[RowGeom<D>::NRR])
{
    constexpr int NRR = RowGeom<D>::NRR, ACT = RowGeom<D>::ACT;
    const int lane = threadIdx.x & 31;
    const uint32_t MP2 = Mpk + p2x2;
    // register k = (d0 + k, d0 + NRR + k): d-1 / d+1 are the neighbouring
    // registers; at k = 0 the low half's d-1 is the previous lane's last
    // register's high half, at k = NRR-1 the high half's d+1 is the next lane's
    // first register's low half
    uint32_t Q[NRR];
#pragma unroll
    for (int k = 0; k < NRR; ++k) Q[k] = Lp[k] + p1x2;
    const uint32_t prevB = __shfl_up_sync(FULL, Q[NRR - 1], 1) | eprev;
    const uint32_t nextA = __shfl_down_sync(FULL, Q[0], 1) | enext;
#pragma unroll
    for (int k = 0; k < NRR; ++k) {
        const uint32_t dm1 = k > 0 ? Q[k - 1] : __byte_perm(prevB, Q[NRR - 1], 0x5432);
        const uint32_t dp1 = k < NRR - 1 ? Q[k + 1] : __byte_perm(Q[0], nextA, 0x5432);
        uint32_t t = vmin2(vmin2(dm1, dp1), Lp[k]);
        t = vmin2(t, MP2);
        Ln[k] = t + C[k] - Mpk;
    }
    const uint32_t mm = tree_min<NRR>(Ln);
    uint32_t m2 = vmin2(mm, __byte_perm(mm, mm, 0x1032));          // (min, min)
    if (ACT < 32 && lane >= ACT) m2 = 0xFFFFFFFFu;
    return __reduce_min_sync(FULL, m2);
}

template <int D>
__device__ __forceinline__ uint32_t row_rec(uint32_t p1x2, uint32_t p2x2, int lane,
                                            const uint32_t (&C)[RowGeom<D>::NRR],
                                            const uint32_t (&Lp)[RowGeom<D>::NRR], uint32_t Mpk,
                                            uint32_t (&Ln)[RowGeom<D>::NRR])
{
    return row_rec<D>(p1x2, p2x2, lane == 0 ? INF2 : 0u, lane == RowGeom<D>::ACT - 1 ? INF2 : 0u, C, Lp, Mpk, Ln);
}

// Per-lane vectors of the row kernel in register order (register k = (d0 + k,
// d0 + NRR + k)): the P_AB | C words K_up writes in that order (NRR words), the
// u8 left->right stash (register k's two bytes at 2k, 2k + 1) and the S vector
// written in natural d order for the WTA kernel.
template <int NRR>
__device__ __forceinline__ void ld_words(const uint16_t* src, uint32_t (&v)[NRR])
{
    if constexpr (NRR == 4) { const uint4 u = *reinterpret_cast<const uint4*>(src); v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; }
    else if constexpr (NRR == 2) { const uint2 u = *reinterpret_cast<const uint2*>(src); v[0] = u.x; v[1] = u.y; }
    else v[0] = *reinterpret_cast<const uint32_t*>(src);
}
template <int NRR> struct StashW { static constexpr int N = NRR >= 2 ? NRR / 2 : 1; };   // stash words per lane
template <int NRR>
__device__ __forceinline__ void st_stash(uint8_t* dst, const uint32_t (&Ln)[NRR])
{
    if constexpr (NRR == 4)
        *reinterpret_cast<uint2*>(dst) = make_uint2(__byte_perm(Ln[0], Ln[1], 0x6420), __byte_perm(Ln[2], Ln[3], 0x6420));
    else if constexpr (NRR == 2) *reinterpret_cast<uint32_t*>(dst) = __byte_perm(Ln[0], Ln[1], 0x6420);
    else *reinterpret_cast<uint16_t*>(dst) = (uint16_t)__byte_perm(Ln[0], 0u, 0x4420);
}
template <int NRR>
__device__ __forceinline__ void ld_stash(const uint8_t* src, uint32_t (&w)[StashW<NRR>::N])
{
    if constexpr (NRR == 4) { const uint2 u = *reinterpret_cast<const uint2*>(src); w[0] = u.x; w[1] = u.y; }
    else if constexpr (NRR == 2) w[0] = *reinterpret_cast<const uint32_t*>(src);
    else w[0] = *reinterpret_cast<const uint16_t*>(src);
}
// register k of the stash as u16x2
template <int NRR>
__device__ __forceinline__ uint32_t stash_reg(const uint32_t (&w)[StashW<NRR>::N], int k)
{
    return __byte_perm(w[k / 2], 0u, (k & 1) ? 0x4342 : 0x4140);
}
template <int NRR>
__device__ __forceinline__ void st_natural(uint16_t* dst, const uint32_t (&sv)[NRR])
{
    if constexpr (NRR == 1) *reinterpret_cast<uint32_t*>(dst) = sv[0];
    else {
        uint32_t o[NRR];
#pragma unroll
        for (int j = 0; j < NRR; ++j)
            o[j] = 2 * j < NRR ? __byte_perm(sv[2 * j], sv[2 * j + 1], 0x5410)
                               : __byte_perm(sv[2 * j - NRR], sv[2 * j - NRR + 1], 0x7632);
        if constexpr (NRR == 4) *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
        else *reinterpret_cast<uint2*>(dst) = make_uint2(o[0], o[1]);
    }
}

// ---------------------------------------------------------------- K_row
// Horizontal paths, one warp per row, no shared memory (occupancy bound only by
// registers).  Left->right: L stashed as u8.  Right->left: S = P_AB + L_lr +
// L_rl written over P_AB in place, natural d order, for the WTA kernel.
constexpr int HROW_WARPS = 4;

// CFROMP (R2's right-referenced pass, reading c24): the left->right path takes
// its cost from the P_AB | C << 9 words instead of the census images.
// SG: pixels per register-buffered load group (4 instead of 8 gains
// 0.3-0.5 % at config C but slows the sweeps it shares the SMs with, and loses
// at 4 paths, D = 256 and in R2's pass)
template <int D, bool CFROMP = false, int SG = 8>
#ifndef ASD_HROW_MINB
#define ASD_HROW_MINB 1               // 6 (<= 80 registers, spills) measured slower
#endif
#ifndef ASD_HROW_SMEM
#define ASD_HROW_SMEM 0               // dynamic shared memory per row CTA: caps its occupancy
#endif
__global__ void __launch_bounds__(32 * HROW_WARPS, ASD_HROW_MINB)
hrow_kernel(RArgs a)
{
    using G = RowGeom<D>;
    constexpr int DPL = G::DPL, NRR = G::NRR, ACT = G::ACT;
    const DevParams& p = a.p;
    const int W = p.W, H = p.H;
    const int frame = blockIdx.y;
    const int y = blockIdx.x * HROW_WARPS + (threadIdx.x >> 5);
    if (y >= H) return;
    const int lane = threadIdx.x & 31;
    const bool active = ACT == 32 || lane < ACT;
    const uint32_t eprev = lane == 0 ? INF2 : 0u, enext = lane == ACT - 1 ? INF2 : 0u;   // row_rec edge masks
    const int d0 = lane * DPL;
    const int lim0 = -p.min_disp - p.R;
    const int ngrp = (W + 31) >> 5;
    const uint32_t* cl = a.cl + frame * a.sig_stride + (long long)y * W;
    const uint32_t* cr = a.cr + frame * a.sig_stride + (long long)y * W;
    const long long rowcell = frame * a.cell_stride + (long long)y * W * D + d0;
    uint8_t* stash = a.stash + rowcell;
    uint16_t* pab = a.pab + rowcell;
    const bool vrow = y >= p.Q && y < H - p.Q;
    auto blk = [&](const uint32_t* row, int i0) -> uint32_t {
        const int i = i0 + lane;
        return (i >= 0 && i < W) ? __ldg(row + i) : 0u;
    };
    auto fast_group = [&](int xb) {
        return vrow && xb + 31 < W && xb >= p.R && xb + 31 < W - p.R && xb + lim0 >= D - 1;
    };

    // ------------------------------------------------ left -> right, cost from P_AB | C
    if constexpr (CFROMP) {
        uint32_t L[NRR];
#pragma unroll
        for (int k = 0; k < NRR; ++k) L[k] = 0u;
        uint32_t M = 0u;
        uint32_t P[SG][NRR], Pn[SG][NRR];
        auto load_c = [&](int xb, uint32_t (&PP)[SG][NRR]) {
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int x = xb + k;
                if (x < W && active) {
                    ld_words<NRR>(pab + (long long)x * D, PP[k]);
                } else {
#pragma unroll
                    for (int r = 0; r < NRR; ++r) PP[k][r] = 0u;
                }
            }
        };
        auto fwd = [&](int xs, const uint32_t (&PP)[SG][NRR]) {
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int x = xs + k;
                if (x < W) {
                    uint32_t Cc[NRR], Ln[NRR];
#pragma unroll
                    for (int r = 0; r < NRR; ++r) Cc[r] = (PP[k][r] >> 9) & 0x003F003Fu;
                    M = row_rec<D>(a.p1x2, a.p2x2, eprev, enext, Cc, L, M, Ln);
#pragma unroll
                    for (int r = 0; r < NRR; ++r) L[r] = Ln[r];
                    if (active) st_stash<NRR>(stash + (long long)x * D, Ln);
                }
            }
        };
        load_c(0, P);
        for (int xs = 0; xs < W; xs += 2 * SG) {
            load_c(xs + SG, Pn);
            fwd(xs, P);
            if (xs + SG >= W) break;
            load_c(xs + 2 * SG, P);
            fwd(xs + SG, Pn);
        }
    } else
    // ------------------------------------------------ left -> right, cost from census
    {
        uint32_t L[NRR], wnd[DPL];
#pragma unroll
        for (int k = 0; k < NRR; ++k) L[k] = 0u;
        uint32_t M = 0u;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const int xr = 0 - p.min_disp - d0 - j;
            wnd[j] = (xr >= 0 && xr < W) ? __ldg(cr + xr) : 0u;
        }
        uint32_t clb = blk(cl, 0), crb = blk(cr, 1 - p.min_disp);
        for (int g = 0; g < ngrp; ++g) {
            const int xb = g << 5;
            const uint32_t clb_n = blk(cl, xb + 32), crb_n = blk(cr, xb + 33 - p.min_disp);
            auto body = [&](auto ftag) {
                constexpr bool F = decltype(ftag)::value;
                for (int s = 0; s < 32; s += SG) {
#pragma unroll
                    for (int k = 0; k < SG; ++k) {
                        const int j = s + k, x = xb + j;
                        const uint32_t clv = __shfl_sync(FULL, clb, j);
                        const uint32_t e = __shfl_sync(FULL, crb, j);
                        if (F || x < W) {
                            const bool vx = F || (vrow && x >= p.R && x < W - p.R);
                            uint32_t Cc[NRR], Ln[NRR];
                            row_cost<D, F>(p, lane, clv, vx, x + lim0, wnd, Cc);
                            M = row_rec<D>(a.p1x2, a.p2x2, eprev, enext, Cc, L, M, Ln);
#pragma unroll
                            for (int r = 0; r < NRR; ++r) L[r] = Ln[r];
                            if (active) st_stash<NRR>(stash + (long long)x * D, Ln);
                            const uint32_t in = __shfl_up_sync(FULL, wnd[DPL - 1], 1);
#pragma unroll
                            for (int q = DPL - 1; q > 0; --q) wnd[q] = wnd[q - 1];
                            wnd[0] = lane == 0 ? e : in;
                        }
                    }
                }
            };
            if (fast_group(xb)) body(std::true_type{}); else body(std::false_type{});
            clb = clb_n; crb = crb_n;
        }
    }
    __syncwarp();
    // ------------------------------------------------ right -> left, S out
    // input: P_AB | C << 9 per cell (K_up), so no census is needed here
    {
        uint32_t L[NRR];
#pragma unroll
        for (int k = 0; k < NRR; ++k) L[k] = 0u;
        uint32_t M = 0u;
        constexpr int SW = StashW<NRR>::N;
        uint32_t P[SG][NRR], Sx[SG][SW], Pn[SG][NRR], Sn[SG][SW];
        auto load_sg = [&](int xb8, uint32_t (&PP)[SG][NRR], uint32_t (&SS)[SG][SW]) {
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int x = xb8 + k;
                if (x >= 0 && x < W && active) {
                    const long long off = (long long)x * D;
                    ld_words<NRR>(pab + off, PP[k]);
                    ld_stash<NRR>(stash + off, SS[k]);
                } else {
#pragma unroll
                    for (int r = 0; r < NRR; ++r) PP[k][r] = 0u;
#pragma unroll
                    for (int r = 0; r < SW; ++r) SS[k][r] = 0u;
                }
            }
        };
        const int xtop = ((W - 1) / SG) * SG;              // sub-groups aligned to SG
        // one sub-group of SG pixels from the buffers PP / SS (x = xs + SG-1 .. xs)
        // S vector of pixel x: pab + x * D in one IMAD.WIDE.U32 (x >= 0)
        auto svec = [&](int x) {
            return reinterpret_cast<uint16_t*>(reinterpret_cast<uintptr_t>(pab) + (unsigned long long)(unsigned)x * (2u * D));
        };
        // whole: all SG pixels inside the row (called with a literal, so each
        // call site inlines its own copy without the per-pixel bound test)
        auto group = [&](const bool whole, int xs, const uint32_t (&PP)[SG][NRR], const uint32_t (&SS)[SG][SW]) {
#pragma unroll
            for (int k = SG - 1; k >= 0; --k) {
                const int x = xs + k;
                if (whole || x < W) {
                    uint32_t Cc[NRR], Pv[NRR], Ln[NRR];
#pragma unroll
                    for (int r = 0; r < NRR; ++r) {
                        Pv[r] = PP[k][r] & 0x01FF01FFu;
                        Cc[r] = (PP[k][r] >> 9) & 0x003F003Fu;
                    }
                    M = row_rec<D>(a.p1x2, a.p2x2, eprev, enext, Cc, L, M, Ln);
#pragma unroll
                    for (int r = 0; r < NRR; ++r) L[r] = Ln[r];
                    if (active) {
                        uint32_t sv[NRR];
#pragma unroll
                        for (int r = 0; r < NRR; ++r) sv[r] = Pv[r] + stash_reg<NRR>(SS[k], r) + Ln[r];
                        st_natural<NRR>(svec(x), sv);
                    }
                }
            }
        };
        // ping-pong between the two buffer sets (no register copies)
        auto run_group = [&](int xs, const uint32_t (&PP)[SG][NRR], const uint32_t (&SS)[SG][SW]) {
            if (xs + SG <= W) group(true, xs, PP, SS);
            else group(false, xs, PP, SS);
        };
        load_sg(xtop, P, Sx);
        for (int xs = xtop; xs >= 0; xs -= 2 * SG) {
            load_sg(xs - SG, Pn, Sn);
            run_group(xs, P, Sx);
            if (xs - SG < 0) break;
            load_sg(xs - 2 * SG, P, Sx);
            run_group(xs - SG, Pn, Sn);
        }
    }
}

// SGBM row pass (D = 128, reading c19): the costs come from the block-cost
// volume in the sweeps' private layout (lane l's four disparities 4l..4l+3 are
// one half of the four words of 16-byte piece (q = l % 4, lane' = 4 (x % 8) +
// l / 8) of the pixel's 8-column block), the partial P_AB is the full u16 word
// and the left->right path is stashed as u16 (it exceeds 8 bits).
template <int D>
__global__ void __launch_bounds__(32 * HROW_WARPS, 4)
hrow_blk_kernel(RArgs a)
{
    static_assert(D == 128, "SGBM row pass: D = 128 only");
    constexpr int NRR = 2, SG = ASD_HROWB_SG;
    const DevParams& p = a.p;
    const int W = p.W, H = p.H;
    const int frame = blockIdx.y;
    const int y = blockIdx.x * HROW_WARPS + (threadIdx.x >> 5);
    if (y >= H) return;
    const int lane = threadIdx.x & 31;
    const int d0 = lane * 4;
    const long long rowcell = frame * a.cell_stride + (long long)y * W * D + d0;
    uint16_t* stash = reinterpret_cast<uint16_t*>(a.stash) + rowcell;
    uint16_t* pab = a.pab + rowcell;
    const uint16_t* cbrow = a.cb + frame * a.cb_stride + (long long)y * a.wpad * D
                          + (32 * (lane & 3) + (lane >> 3)) * 8;
    const uint32_t sel = ((lane >> 2) & 1) ? 0x7632u : 0x5410u;
    auto cost = [&](int x, uint32_t (&Cc)[NRR]) {      // (A, B) = ((d0, d0+2), (d0+1, d0+3))
        const uint4 v = *reinterpret_cast<const uint4*>(cbrow + (long long)(x & ~7) * D + 32 * (x & 7));
        Cc[0] = __byte_perm(v.x, v.z, sel);
        Cc[1] = __byte_perm(v.y, v.w, sel);
    };
    // ------------------------------------------------ left -> right
    {
        uint32_t L[NRR] = {0u, 0u}, M = 0u;
        uint32_t Cg[SG][NRR], Cn[SG][NRR];
        auto load = [&](int xb, uint32_t (&CC)[SG][NRR]) {
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                if (xb + k < W) cost(xb + k, CC[k]);
                else { CC[k][0] = 0u; CC[k][1] = 0u; }
            }
        };
        auto fwd = [&](int xs, const uint32_t (&CC)[SG][NRR]) {
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int x = xs + k;
                if (x < W) {
                    uint32_t Ln[NRR];
                    M = row_rec<D>(a.p1x2, a.p2x2, lane, CC[k], L, M, Ln);
                    L[0] = Ln[0]; L[1] = Ln[1];
                    *reinterpret_cast<uint2*>(stash + (long long)x * D) = make_uint2(Ln[0], Ln[1]);
                }
            }
        };
        load(0, Cg);
        for (int xs = 0; xs < W; xs += 2 * SG) {
            load(xs + SG, Cn);
            fwd(xs, Cg);
            if (xs + SG >= W) break;
            load(xs + 2 * SG, Cg);
            fwd(xs + SG, Cn);
        }
    }
    __syncwarp();
    // ------------------------------------------------ right -> left, S out
    {
        uint32_t L[NRR] = {0u, 0u}, M = 0u;
        uint32_t P[SG][NRR], Cg[SG][NRR], Sx[SG][NRR], Pn[SG][NRR], Cn[SG][NRR], Sn[SG][NRR];
        auto load = [&](int xb, uint32_t (&PP)[SG][NRR], uint32_t (&CC)[SG][NRR], uint32_t (&SS)[SG][NRR]) {
#pragma unroll
            for (int k = 0; k < SG; ++k) {
                const int x = xb + k;
                if (x >= 0 && x < W) {
                    const uint2 u = *reinterpret_cast<const uint2*>(pab + (long long)x * D);
                    const uint2 t = *reinterpret_cast<const uint2*>(stash + (long long)x * D);
                    PP[k][0] = u.x; PP[k][1] = u.y;
                    SS[k][0] = t.x; SS[k][1] = t.y;
                    cost(x, CC[k]);
                } else {
                    PP[k][0] = PP[k][1] = 0u; SS[k][0] = SS[k][1] = 0u; CC[k][0] = CC[k][1] = 0u;
                }
            }
        };
        auto bwd = [&](int xs, const uint32_t (&PP)[SG][NRR], const uint32_t (&CC)[SG][NRR],
                       const uint32_t (&SS)[SG][NRR]) {
#pragma unroll
            for (int k = SG - 1; k >= 0; --k) {
                const int x = xs + k;
                if (x < W) {
                    uint32_t Ln[NRR];
                    M = row_rec<D>(a.p1x2, a.p2x2, lane, CC[k], L, M, Ln);
                    L[0] = Ln[0]; L[1] = Ln[1];
                    const uint32_t s0 = PP[k][0] + SS[k][0] + Ln[0];
                    const uint32_t s1 = PP[k][1] + SS[k][1] + Ln[1];
                    *reinterpret_cast<uint2*>(pab + (long long)x * D) =
                        make_uint2(__byte_perm(s0, s1, 0x5410), __byte_perm(s0, s1, 0x7632));
                }
            }
        };
        const int xtop = ((W - 1) / SG) * SG;
        load(xtop, P, Cg, Sx);
        for (int xs = xtop; xs >= 0; xs -= 2 * SG) {
            load(xs - SG, Pn, Cn, Sn);
            bwd(xs, P, Cg, Sx);
            if (xs - SG < 0) break;
            load(xs - 2 * SG, P, Cg, Sx);
            bwd(xs - SG, Pn, Cn, Sn);
        }
    }
}

// ---------------------------------------------------------------- K_wta
// WTA / uniqueness / sub-pixel for the left view and the re-indexed right view
// (K4 semantics, post.cu) from S rows staged in shared memory.  One CTA (8
// warps, two resident per SM) per image row walks stages of 256 pixels; stage
// t loads S rows [256t, 256t + 255 + min + D - 1] with 4-byte cp.async into a
// linear window (row x at slot x - 256t: the rows past the stage are loaded
// again by the next stage, from L2), so every diagonal is wrap-free and both
// views run fully unrolled with immediate offsets.  Window rows are D + 2 u16:
// an odd word stride keeps the diagonal right-view reads free of bank
// conflicts.
#ifndef ASD_WTA_WARPS
#define ASD_WTA_WARPS 8
#endif
constexpr int WTA_WARPS = ASD_WTA_WARPS;
#ifndef ASD_WTA_SPLIT
#define ASD_WTA_SPLIT 1
#endif
constexpr bool WTA_SPLIT = ASD_WTA_SPLIT;
// D = 256: stages of 128 pixels (4 warps) so the full-width window fits
__host__ __device__ constexpr int wta_warps(int D) { return D > 128 ? (WTA_WARPS < 4 ? WTA_WARPS : 4) : WTA_WARPS; }


// MODE 0: left view + re-indexed right view (R1).  MODE 1: left view only
// (R2's left-referenced pass).  MODE 2: the "left view" of the right-referenced
// aggregate, written to the right-view maps (R2's right view, reading c24).
template <int D, bool WIDE, int MODE = 0>
__global__ void __launch_bounds__(32 * WTA_WARPS)
wta2_kernel(RArgs a)
{
    using G = RowGeom<D>;
    constexpr int BS = G::BS;
    extern __shared__ __align__(16) uint16_t sbuf[];  // [NB][BS]
    const DevParams& p = a.p;
    const int W = p.W, NB = a.nbuf;
    const int y = blockIdx.x, frame = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint16_t* S = a.pab + frame * a.cell_stride + (long long)y * W * D;
    const bool vrow = y >= p.Q && y < p.H - p.Q;
    // right pixels with no defined disparity at all: xr + min_disp >= W
    for (int xr = max(0, W - p.min_disp) + threadIdx.x; MODE == 0 && xr < W; xr += blockDim.x) {
        const long long o = frame * a.px_stride + (long long)y * W + xr;
        a.fs.dstar_r[o] = -1;
        a.fs.mask_r[o] = MASK_BORDER;
        a.fs.dr[o] = 0.0f;
    }
    constexpr int CH = D * 2 / WTA_CHUNK;             // copy pieces per S row
    constexpr int TX = 32 * wta_warps(D);
    const int nstage = (W + TX - 1) / TX;
    for (int t = 0; t < nstage; ++t) {
        // linear window of this stage: row x at slot x - x0, rows [x0, hi)
        const int x0 = t * TX;
        const int hi = min(W, x0 + TX + p.min_disp + D - 1);
        __syncthreads();                              // previous stage done with the window
        {   // thread t copies word t % CH of rows x0 + t / CH, + RSTEP, ...
            // (32-bit shared address and global pointer stepped, 4 copies per trip)
            constexpr int RSTEP = TX / CH;
            const int c = threadIdx.x % CH;
            const int slot0 = threadIdx.x / CH;
            const int n = (hi - x0 - slot0 + RSTEP - 1) / RSTEP;     // rows this thread copies
            constexpr int PU = WTA_CHUNK / 2;                  // u16 per piece
            unsigned sa = smem_u32(sbuf + slot0 * BS + c * PU);
            const uint16_t* src = S + (long long)(x0 + slot0) * D + c * PU;
            constexpr unsigned SSTEP = RSTEP * BS * 2;
            auto cp = [](unsigned dst, const uint16_t* g) {
                if constexpr (WTA_CHUNK == 16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(dst), "l"(g) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" :: "r"(dst), "l"(g), "n"(WTA_CHUNK) : "memory");
            };
            // WTA_SPLIT: two commit groups, the stage's own rows [x0, x0 + TX)
            // (all the left view reads) first, so the fill of the rows past the
            // stage (right view only; not loaded at all when MODE != 0) overlaps
            // the left view
            const int na = WTA_SPLIT ? max(0, (min(TX, hi - x0) - slot0 + RSTEP - 1) / RSTEP) : n;
            int k = 0;
            for (; k + 4 <= na; k += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) cp(sa + u * SSTEP, src + u * RSTEP * D);
                sa += 4 * SSTEP;
                src += 4 * RSTEP * D;
            }
            for (; k < na; ++k, sa += SSTEP, src += RSTEP * D) cp(sa, src);
            if (WTA_SPLIT) {
                cp_async_commit();
                for (; MODE == 0 && k < n; ++k, sa += SSTEP, src += RSTEP * D) cp(sa, src);
            }
        }
        cp_async_commit();
        if (WTA_SPLIT) cp_async_wait<1>();
        else cp_async_wait<0>();
        ASD_JITTER(7);
        __syncthreads();
        // left view
        {
            const int xp = x0 + warp * 32 + lane;
            if (xp < W) {
                int ds; bool uf; float disp;
                wta_left_lane<D, WIDE>(p, sbuf + (xp - x0) * BS, ds, uf, disp);
                const long long o = frame * a.px_stride + (long long)y * W + xp;
                uint8_t m = 0;
                if (!(vrow && xp >= p.R && xp < W - p.R)) m |= MASK_BORDER;
                if (uf) m |= MASK_UNIQUE;
                (MODE == 2 ? a.fs.dstar_r : a.fs.dstar_l)[o] = (int16_t)ds;
                (MODE == 2 ? a.fs.mask_r : a.fs.mask_l)[o] = m;
                (MODE == 2 ? a.fs.dr : a.fs.dl)[o] = disp;
            }
        }
        if constexpr (MODE != 0) continue;           // R2 passes: one view per launch
        if (WTA_SPLIT) cp_async_wait<0>();
        ASD_JITTER(8);
        __syncthreads();                              // left poisoning done before diagonal reads
        // right view
        {
            const int xw = x0 + warp * 32;                 // the warp's first right pixel
            const int xr = xw + lane;
            const int nd = min(D, W - p.min_disp - xr);
            const bool fast = xw + 31 + p.min_disp + D - 1 < W;   // warp-uniform: all d defined
            if (xr < W && nd > 0) {
                int ds = -1; bool uf = false; float disp = 0.0f;
                if (fast) wta_right_lin<D, WIDE>(p, sbuf + (xr + p.min_disp - x0) * BS, ds, uf, disp);
                else wta_right_lane<D>(p, sbuf, NB, xr + p.min_disp - x0, nd, ds, uf, disp);
                const long long o = frame * a.px_stride + (long long)y * W + xr;
                uint8_t m = 0;
                if (!(vrow && xr >= p.R && xr < W - p.R)) m |= MASK_BORDER;
                if (uf) m |= MASK_UNIQUE;
                a.fs.dstar_r[o] = (int16_t)ds;
                a.fs.mask_r[o] = m;
                a.fs.dr[o] = disp;
            }
        }
    }
}

// ---------------------------------------------------------------- K_wta, D = 256 in halves
// The D = 256 window (384 rows x 516 B) would leave one 4-warp CTA per SM.
// Here every stage of 256 pixels runs three passes over half-width windows
// (rows of 128 disparities, 384 x 260 B = 100 KB: two 8-warp CTAs per SM):
//   A  rows [x0, x0 + 256 + min + 127) of d 0..127: left and right view, low half
//   B  rows [x0, x0 + 256)             of d 128..255: left view, high half
//   C  rows [x0 + min + 128, +256+127) of d 128..255: right view, high half
// Each pass leaves per lane the half's best key (S << 8 | d), its neighbours,
// its own second best (|d - d*| >= 2 within the half), the half's minimum, the
// minimum without the element next to the other half, and that element; the
// merge then gives exactly the full-range d*, S(d* +- 1) and second best
// (K4 semantics, readings c8, c9, c13).
struct HalfSt { uint32_t key, cm, cp, s2, mall, medge, sedge; };
constexpr uint32_t NOKEY = 0xFFFFFFFFu;

// all 128 elements defined; e(j) = S(dbase + j), ep(j) = e(j) | e(j + 1) << 16 (j even)
template <bool LOW, class E, class EP>
__device__ __forceinline__ HalfSt half_scan_full(E e, EP ep, int dbase)
{
    uint32_t k0 = NOKEY, k1 = NOKEY, bm[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        uint32_t m = 0xFFFFu;
#pragma unroll
        for (int t = 0; t < 8; t += 2) {
            const int j = 8 * b + t;
            const uint32_t pr = ep(j);
            const uint32_t v0 = pr & 0xFFFFu, v1 = pr >> 16;
            k0 = min(k0, (v0 << 8) | (uint32_t)(dbase + j));
            k1 = min(k1, (v1 << 8) | (uint32_t)(dbase + j + 1));
            m = min(m, min(v0, v1));
        }
        bm[b] = m;
    }
    HalfSt h;
    h.key = min(k0, k1);
    const int js = (int)(h.key & 255u) - dbase;
    h.cm = js > 0 ? e(js - 1) : NONE16;
    h.cp = js < 127 ? e(js + 1) : NONE16;
    const int blo = max(js - 1, 0) >> 3, bhi = min(js + 1, 127) >> 3;
    uint32_t sec = 0xFFFFu, mall = 0xFFFFu, medge = 0xFFFFu;
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        if (b < blo || b > bhi) sec = min(sec, bm[b]);
        mall = min(mall, bm[b]);
        if (LOW ? b < 15 : b > 0) medge = min(medge, bm[b]);
    }
    for (int b = blo; b <= bhi; ++b)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int j = 8 * b + t;
            if (j < js - 1 || j > js + 1) sec = min(sec, e(j));
        }
#pragma unroll
    for (int t = 0; t < 7; ++t) medge = min(medge, e(LOW ? 120 + t : 1 + t));   // the edge block minus the edge
    h.s2 = sec; h.mall = mall; h.medge = medge;
    h.sedge = e(LOW ? 127 : 0);
    return h;
}

// the first nh (0..128) elements defined (right view near the right border)
template <bool LOW, class E>
__device__ __forceinline__ HalfSt half_scan_part(E e, int dbase, int nh)
{
    HalfSt h{NOKEY, NONE16, NONE16, NONE16, NONE16, NONE16, NONE16};
    if (nh <= 0) return h;
    uint32_t key = NOKEY;
    for (int j = 0; j < nh; ++j) key = min(key, (e(j) << 8) | (uint32_t)(dbase + j));
    const int js = (int)(key & 255u) - dbase;
    h.key = key;
    h.cm = js > 0 ? e(js - 1) : NONE16;
    h.cp = js + 1 < nh ? e(js + 1) : NONE16;
    uint32_t sec = NONE16, mall = NONE16, medge = NONE16;
    for (int j = 0; j < nh; ++j) {
        const uint32_t v = e(j);
        if (j < js - 1 || j > js + 1) sec = min(sec, v);
        mall = min(mall, v);
        if (LOW ? j < 127 : j > 0) medge = min(medge, v);
    }
    h.s2 = sec; h.mall = mall; h.medge = medge;
    h.sedge = LOW ? (nh == 128 ? e(127) : NONE16) : e(0);
    return h;
}

__device__ __forceinline__ void merge_halves(const DevParams& p, const HalfSt& A, const HalfSt& B,
                                             int& dstar, bool& uf, float& disp)
{
    uint32_t s0, cm, cp, s2;
    if (A.key <= B.key) {                       // ties: the smaller d (A) wins, as in K4
        dstar = (int)(A.key & 255u); s0 = A.key >> 8; cm = A.cm;
        cp = dstar == 127 ? B.sedge : A.cp;
        s2 = min(A.s2, dstar == 127 ? B.medge : B.mall);
    } else {
        dstar = (int)(B.key & 255u); s0 = B.key >> 8; cp = B.cp;
        cm = dstar == 128 ? A.sedge : B.cm;
        s2 = min(B.s2, dstar == 128 ? A.medge : A.mall);
    }
    finish_wta(p, dstar, s0, s2, cm, cp, uf, disp);
}

constexpr int WH_BS = 128 + WTA_PAD;       // u16 per half-window row (odd word stride)

__global__ void __launch_bounds__(256)
wta_halves_kernel(RArgs a)
{
    constexpr int D = 256, TX = 256, BS = WH_BS, STEP = BS + 1;
    extern __shared__ __align__(16) uint16_t sbuf[];   // [nbuf][BS]
    const DevParams& p = a.p;
    const int W = p.W, md = p.min_disp;
    const int y = blockIdx.x, frame = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint16_t* S = a.pab + frame * a.cell_stride + (long long)y * W * D;
    const bool vrow = y >= p.Q && y < p.H - p.Q;
    for (int xr = max(0, W - md) + tid; xr < W; xr += blockDim.x) {   // no disparity defined
        const long long o = frame * a.px_stride + (long long)y * W + xr;
        a.fs.dstar_r[o] = -1;
        a.fs.mask_r[o] = MASK_BORDER;
        a.fs.dr[o] = 0.0f;
    }
    // rows [r0, r1) of half h into window rows 0.. (4-byte cp.async, 64 per row)
    auto fill = [&](int r0, int r1, int h) {
        __syncthreads();                              // previous pass done with the window
        constexpr int CH = 64, RSTEP = TX / CH;
        const int c = tid % CH;
        for (int r = r0 + tid / CH; r < r1; r += RSTEP)
            cp_async4(reinterpret_cast<uint32_t*>(sbuf + (r - r0) * BS) + c,
                      reinterpret_cast<const uint32_t*>(S + (long long)r * D + 128 * h) + c, true);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    };
    const int nstage = (W + TX - 1) / TX;
    for (int t = 0; t < nstage; ++t) {
        const int x0 = t * TX;
        const int xp = x0 + tid;                      // this lane's left pixel and right pixel
        const int nd = min(D, W - md - xp);           // defined disparities of right pixel xp
        const bool fast = x0 + warp * 32 + 31 + md + D - 1 < W;   // warp-uniform: all defined
        HalfSt LA, RA;
        // ---- pass A: d 0..127, left and right
        fill(x0, min(W, x0 + TX + md + 127), 0);
        if (xp < W) {
            const uint16_t* r = sbuf + (xp - x0) * BS;
            const uint32_t* r32 = reinterpret_cast<const uint32_t*>(r);
            LA = half_scan_full<true>([&](int j) { return (uint32_t)r[j]; }, [&](int j) { return r32[j / 2]; }, 0);
        }
        if (xp < W && nd > 0) {
            const uint16_t* b0 = sbuf + (xp + md - x0) * BS;
            if (fast) RA = half_scan_full<true>([&](int j) { return (uint32_t)b0[j * STEP]; },
                                                [&](int j) { return __byte_perm(b0[j * STEP], b0[(j + 1) * STEP], 0x5410); }, 0);
            else RA = half_scan_part<true>([&](int j) { return (uint32_t)b0[j * STEP]; }, 0, min(nd, 128));
        }
        // ---- pass B: d 128..255, left view
        fill(x0, min(W, x0 + TX), 1);
        if (xp < W) {
            const uint16_t* r = sbuf + (xp - x0) * BS;
            const uint32_t* r32 = reinterpret_cast<const uint32_t*>(r);
            const HalfSt LB = half_scan_full<false>([&](int j) { return (uint32_t)r[j]; },
                                                    [&](int j) { return r32[j / 2]; }, 128);
            int ds; bool uf; float disp;
            merge_halves(p, LA, LB, ds, uf, disp);
            const long long o = frame * a.px_stride + (long long)y * W + xp;
            uint8_t m = 0;
            if (!(vrow && xp >= p.R && xp < W - p.R)) m |= MASK_BORDER;
            if (uf) m |= MASK_UNIQUE;
            a.fs.dstar_l[o] = (int16_t)ds;
            a.fs.mask_l[o] = m;
            a.fs.dl[o] = disp;
        }
        // ---- pass C: d 128..255, right view
        const int c0 = x0 + md + 128;
        fill(c0, min(W, c0 + TX + 127), 1);
        if (xp < W && nd > 0) {
            HalfSt RB{NOKEY, NONE16, NONE16, NONE16, NONE16, NONE16, NONE16};
            if (nd > 128) {
                const uint16_t* b0 = sbuf + (xp - x0) * BS;       // row xp + md + 128 + j of the window
                if (fast) RB = half_scan_full<false>([&](int j) { return (uint32_t)b0[j * STEP]; },
                                                     [&](int j) { return __byte_perm(b0[j * STEP], b0[(j + 1) * STEP], 0x5410); }, 128);
                else RB = half_scan_part<false>([&](int j) { return (uint32_t)b0[j * STEP]; }, 128, nd - 128);
            }
            int ds; bool uf; float disp;
            merge_halves(p, RA, RB, ds, uf, disp);
            const long long o = frame * a.px_stride + (long long)y * W + xp;
            uint8_t m = 0;
            if (!(vrow && xp >= p.R && xp < W - p.R)) m |= MASK_BORDER;
            if (uf) m |= MASK_UNIQUE;
            a.fs.dstar_r[o] = (int16_t)ds;
            a.fs.mask_r[o] = m;
            a.fs.dr[o] = disp;
        }
    }
}

}  // namespace v2

// ======================================================================== host
using v2::VArgs;
using v2::RArgs;

typedef void (*VKernel)(VArgs);
typedef void (*RKernel)(RArgs);

template <int DC, int T, int NP, bool UP, int DPL, bool RR = false, bool BLK = false, bool SEG = false>
static VKernel vkern()
{
    return v2::vsweep_kernel<DC, T, NP, UP, DPL, RR, BLK, SEG>;
}

template <int DC, int T, int DPL, bool SEG>
static VKernel vk3(bool up, bool rr)
{
    if (up) return vkern<DC, T, 3, true, DPL, false, false, SEG>();
    if (rr) return vkern<DC, T, 3, false, DPL, true, false, SEG>();
    return vkern<DC, T, 3, false, DPL, false, false, SEG>();
}
template <int DC, int T, int DPL>
static VKernel vk(int np, bool up, bool rr, bool seg)
{
    if (np == 3) return seg ? vk3<DC, T, DPL, true>(up, rr) : vk3<DC, T, DPL, false>(up, rr);
    if (up) return vkern<DC, T, 1, true, DPL>();
    if (rr) return vkern<DC, T, 1, false, DPL, true>();
    return vkern<DC, T, 1, false, DPL>();
}

// rr: the K_down instance with the right view as reference (R2); blk: the SGBM
// instances (D = 128: DC = 32, T = 4, 8 paths only)
static VKernel pick_vkernel(int DC, int T, int DPL, int np, bool up, bool rr = false, bool blk = false,
                            bool seg = false)
{
    if (blk) {
        if (DC != 32 || T != 4 || DPL != 4) return nullptr;
        if (np == 3 && seg) {
            if (up) return vkern<32, 4, 3, true, 4, false, true, true>();
            return rr ? vkern<32, 4, 3, false, 4, true, true, true>() : vkern<32, 4, 3, false, 4, false, true, true>();
        }
        if (np == 3) {
            if (up) return vkern<32, 4, 3, true, 4, false, true>();
            return rr ? vkern<32, 4, 3, false, 4, true, true>() : vkern<32, 4, 3, false, 4, false, true>();
        }
        if (up) return vkern<32, 4, 1, true, 4, false, true>();
        return rr ? vkern<32, 4, 1, false, 4, true, true>() : vkern<32, 4, 1, false, 4, false, true>();
    }
    if (DC == 16 && T == 1 && DPL == 2) return vk<16, 1, 2>(np, up, rr, seg);
    if (DC == 32 && T == 1 && DPL == 2) return vk<32, 1, 2>(np, up, rr, seg);
    if (DC == 32 && T == 2 && DPL == 2) return vk<32, 2, 2>(np, up, rr, seg);
    if (DC == 32 && T == 4 && DPL == 4) return vk<32, 4, 4>(np, up, rr, seg);
    if (DC == 24 && T == 4 && DPL == 4) return vk<24, 4, 4>(np, up, rr, seg);     // D = 96
    if (DC == 32 && T == 8 && DPL == 8) return vk<32, 8, 8>(np, up, rr, seg);     // D = 256
#ifdef ASD_ABLATE
    if (DC == 16 && T == 8 && DPL == 4) return vk<16, 8, 4>(np, up, rr, seg);
#endif
    return nullptr;
}

static RKernel pick_rkernel(int D, bool cfromp = false, bool eight_paths = false)
{
    (void)eight_paths;
    if (D == 16) return cfromp ? v2::hrow_kernel<16, true> : v2::hrow_kernel<16, false>;
    if (D == 32) return cfromp ? v2::hrow_kernel<32, true> : v2::hrow_kernel<32, false>;
    if (D == 64) return cfromp ? v2::hrow_kernel<64, true> : v2::hrow_kernel<64, false>;
    if (D == 128) return cfromp ? v2::hrow_kernel<128, true> : v2::hrow_kernel<128, false>;
    if (D == 96) return cfromp ? v2::hrow_kernel<96, true> : v2::hrow_kernel<96, false>;
    if (D == 256) return cfromp ? v2::hrow_kernel<256, true> : v2::hrow_kernel<256, false>;
    return nullptr;
}

template <int D>
static RKernel wk_d(bool wide, int mode)
{
    if (mode == 1) return wide ? v2::wta2_kernel<D, true, 1> : v2::wta2_kernel<D, false, 1>;
    if (mode == 2) return wide ? v2::wta2_kernel<D, true, 2> : v2::wta2_kernel<D, false, 2>;
    return wide ? v2::wta2_kernel<D, true, 0> : v2::wta2_kernel<D, false, 0>;
}

static RKernel pick_wkernel(int D, bool wide = false, int mode = 0)
{
    if (D == 16) return wk_d<16>(wide, mode);
    if (D == 32) return wk_d<32>(wide, mode);
    if (D == 64) return wk_d<64>(wide, mode);
    if (D == 128) return wk_d<128>(wide, mode);
    if (D == 96) return wk_d<96>(wide, mode);                // engine D1 only (WTA window kernel)
    if (D == 256) return wk_d<256>(wide, mode);
    return nullptr;
}

static size_t vsmem_bytes(int w, int D, int T, int DC, int np, bool up, bool blk = false)
{
    const int nw = w * T / 32;
    const bool ring = up || blk;
    size_t words = 0;
    const int cstr = ((w + DC - 1 + 31) / 32) * 32 + 32;
    words = ring ? 0 : (size_t)v2::NSLOT * ((size_t)w + (size_t)T * cstr);
    if (np == 3) words += 4 * (size_t)nw * T * (DC / 2 + 4) + 4 * (size_t)nw;   // halos (HS = NR + 4)
    words += (size_t)nw * 16 * DC;                    // K_up output staging
    if (ring) {                                       // TMA ring(s) + mbarriers (+ align)
        const int kr = (up && blk) ? 2 : v2::KU, nring = (up && blk) ? 2 : 1;
        words += (size_t)nring * kr * w * D / 2 + 2 * kr + 4;
    } else {
        words += 2 * v2::NSLOT + 4;                   // census-row mbarriers (TMA staging)
    }
    return words * 4;
}

bool v2_plan(const DevParams& p, int device, V2Plan& pl)
{
    pl = V2Plan{};
    auto no = [&](const char* why) { snprintf(pl.why, sizeof pl.why, "%s", why); pl.ok = false; return false; };
    if (p.nb > 32) return no("nb > 32 (u64 census)");
    if (p.D != 16 && p.D != 32 && p.D != 64 && p.D != 96 && p.D != 128 && p.D != 256)
        return no("num_disp not in {16,32,64,96,128,256}");
    const int np = p.paths == 8 ? 3 : 1;
    // blk: the u16-partial instances (BLK) that read the matching cost from a
    // cost buffer in the sweeps' private layout -- SGBM's block cost, or, for
    // SGM whose 3-path partial exceeds 8 bits (3 (nb + P2) > 255), the 1 x 1
    // "block" cost, i.e. the per-pixel Hamming cost.  wide: u32 WTA keys.
    bool blk = p.bw * p.bh > 1, wide = blk;
    if (blk) {
        // SGBM: u16 partials without cost bits (S <= 65534 validated by asd_create), u32 WTA keys
        if (p.D != 128) return no("SGBM on engine D3 needs num_disp = 128");
    } else {
        if (np == 3 && 3 * (p.nb + p.p2) > 255) {
            if (p.D != 128) return no("3*(nb+p2) > 255 (u16 partials need num_disp = 128)");
            blk = wide = true;
        }
        int ks = 1;
        while ((1 << ks) < p.D) ++ks;
        const long long smax = (long long)p.paths * (p.nb + p.p2);
        if ((smax << ks) + (1 << ks) - 1 > 0xFFFE) wide = true;       // S << log2(D) exceeds 16-bit keys
    }
    pl.NP = np;
    pl.DPL = p.D <= 64 ? 2 : p.D <= 128 ? 4 : 8;
    if (p.D == 16) { pl.DC = 16; pl.T = 1; }
    else if (p.D == 96) { pl.DC = 24; pl.T = 4; }
    else if (p.D == 256) { pl.DC = 32; pl.T = 8; }
    else if (p.D == 32) { pl.DC = 32; pl.T = 1; }
    else if (p.D == 64) { pl.DC = 32; pl.T = 2; }
    else { pl.DC = 32; pl.T = 4; }
#ifdef ASD_ABLATE                                    // experiment builds only (tools/ab.sh)
    const char* force = getenv("ASD_V2_DC16");
    if (p.D == 128 && force && force[0] == '1') { pl.DC = 16; pl.T = 8; }
#endif
    const int T = pl.T, CPW = 32 / T;
    const int maxt = pl.DC >= 24 ? 512 : 1024;      // __launch_bounds__ of vsweep_kernel
    pl.blk = blk;
    // census rows by TMA bulk copies: 16-byte aligned rows and slice starts
    // (the context allocates guard bands around the census buffers)
    pl.tma_cen = ASD_CEN_TMA && !blk && p.W % 4 == 0 && p.min_disp % 4 == 0;
    VKernel kd = pick_vkernel(pl.DC, T, pl.DPL, np, false, false, blk);
    VKernel ku = pick_vkernel(pl.DC, T, pl.DPL, np, true, false, blk);
    if (!kd || !ku) return no(blk ? "SGBM on engine D3 needs num_disp = 128" : "no sweep kernel instance");
    VKernel kd1 = kd, ku1 = ku;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    double best = -1.0;
#ifdef ASD_ABLATE
    const char* fcs = getenv("ASD_V2_CS");            // experiment builds: force a cluster size
    const int force_cs = fcs ? atoi(fcs) : 0;
#else
    const int force_cs = 0;
#endif
    // nseg > 1: a frame wider than one cluster is covered by nseg clusters of cs
    // CTAs (8 paths only), joined through global memory at the boundaries; all
    // nseg clusters of a frame must be co-resident, so a wave is
    // floor(active clusters / nseg) frames.  One segment is preferred.
    for (int nseg = 1; nseg <= (np == 3 ? 4 : 1); ++nseg) {
    kd = nseg > 1 ? pick_vkernel(pl.DC, T, pl.DPL, np, false, false, blk, true) : kd1;
    ku = nseg > 1 ? pick_vkernel(pl.DC, T, pl.DPL, np, true, false, blk, true) : ku1;
    for (int cs = 1; cs <= 16; ++cs) {
        if (force_cs > 0 && cs != force_cs) continue;
        if (nseg > 1 && cs < 2) continue;
        const int n = cs * nseg;
        int w = (p.W + n - 1) / n;
        w = (w + CPW - 1) / CPW * CPW;
        if ((long long)w * (n - 1) >= p.W && n > 1) continue;      // last CTA would be empty
        const int threads = w * T;
        if (threads > maxt) continue;
        if (np == 1 && cs > 1 && threads < 128) continue;
        const size_t smd = vsmem_bytes(w, p.D, T, pl.DC, np, false, blk);
        const size_t sm = vsmem_bytes(w, p.D, T, pl.DC, np, true, blk);
        if (sm > 220 * 1024 || smd > 220 * 1024) continue;
        cudaFuncSetAttribute((const void*)kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smd);
        cudaFuncSetAttribute((const void*)ku, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (VKernel k : {kd, ku})
            if (cs > 8) cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        int active = 0;
        if (np == 3 && cs > 1) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs, 64);
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, (const void*)ku, &cfg) != cudaSuccess) { cudaGetLastError(); continue; }
            active = (nc / nseg) * nseg * cs;                         // whole frames only
        } else {
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)ku, threads, sm) != cudaSuccess) { cudaGetLastError(); continue; }
            active = nb * nsm;
        }
        if (active <= 0) continue;
        // throughput proxy: resident threads, penalising clusters that leave SMs
        // idle and (2 % per extra segment) the boundary exchange
        const double score = (double)active * threads / (1.0 + 0.02 * (nseg - 1));
#ifdef ASD_ABLATE
        if (getenv("ASD_PLAN_DEBUG"))
            fprintf(stderr, "plan nseg=%d cs=%d w=%d threads=%d smem=%zu/%zu active=%d score=%.0f\n",
                    nseg, cs, w, threads, smd, sm, active, score);
#endif
        if (score > best * 1.02) {
            best = score; pl.cs = cs; pl.w = w; pl.vthreads = threads; pl.vsmem = smd; pl.vsmem_up = sm;
            pl.active_ctas = active; pl.ncta = n;
        }
        if (np == 1) break;
    }
    // one cluster per frame when it fits (measured: config C 1937 frames/s as
    // 10 x 1 vs 1390 as 5 x 4); otherwise the best-scoring segment count
    if (nseg == 1 && best >= 0) break;
    }
    if (best < 0) return no("no feasible cluster configuration");
    const bool segs = np == 3 && pl.ncta > pl.cs;
    kd = pick_vkernel(pl.DC, T, pl.DPL, np, false, false, blk, segs);
    ku = pick_vkernel(pl.DC, T, pl.DPL, np, true, false, blk, segs);
    cudaFuncSetAttribute((const void*)kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.vsmem);
    cudaFuncSetAttribute((const void*)ku, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.vsmem_up);
    if (np == 1) {
        // vertical-only sweeps have no cross-column dependency: 1-CTA strips
        int w = (256 / T + CPW - 1) / CPW * CPW;
        if (w > (p.W + CPW - 1) / CPW * CPW) w = (p.W + CPW - 1) / CPW * CPW;
        pl.w = w;
        pl.cs = (p.W + w - 1) / w;
        pl.ncta = pl.cs;
        pl.vthreads = w * T;
        pl.vsmem = vsmem_bytes(w, p.D, T, pl.DC, np, false, blk);
        pl.vsmem_up = vsmem_bytes(w, p.D, T, pl.DC, np, true, blk);
        cudaFuncSetAttribute((const void*)kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.vsmem);
        cudaFuncSetAttribute((const void*)ku, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.vsmem_up);
    }
    if (p.lr_mode == 1) {                            // R2: the right-referenced K_down
        VKernel kr = pick_vkernel(pl.DC, T, pl.DPL, np, false, true, blk, segs);
        cudaFuncSetAttribute((const void*)kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.vsmem);
        if (pl.cs > 8) cudaFuncSetAttribute((const void*)kr, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    pl.wta_fb = false;
    // the half-window D = 256 WTA also on D3 when the sweeps use no clusters
    // (4 paths: Table II D = 256 1851 -> 2001); with 15-CTA clusters it
    // delays their placement (config D 297 vs 307)
    if (!wta2_plan(p, wide, pl, np == 1)) {
        // the window does not fit shared memory (D = 256): the warp-per-pixel
        // WTA kernel of engine D1 (post.cu) reads the same natural-order S
        if (p.lr_mode == 1) return no("min_disp + num_disp too large for the WTA window (R2)");
        pl.wta_fb = true;
        pl.wide = wide;
    }
    pl.ok = true;
    return true;
}

// Segment-boundary exchange buffer (nseg > 1) for nframes frames in flight:
// [frames][nseg-1][2 dirs][2 slots][T][NR + 2] tagged u64 words.
size_t v2_ghalo_bytes(const V2Plan& pl, int nframes)
{
    const int nb = pl.ncta / (pl.cs > 0 ? pl.cs : 1) - 1;
    return nb > 0 ? (size_t)nframes * nb * 2 * 2 * pl.T * (pl.DC / 2 + 2) * sizeof(unsigned long long) : 0;
}

// The WTA kernel's window: rows [256t, 256t + 255 + min + D - 1] of stage t.
bool wta2_plan(const DevParams& p, bool wide, V2Plan& pl, bool halves_ok)
{
    if (!pick_wkernel(p.D, wide)) return false;
    // wta_halves_kernel (half-width windows): engine D1 and 4-path D3 -- in the
    // 8-path D3 pipeline its 2 x 100 KB CTAs per SM delay the sweep clusters
    // (config D 297 vs 307 frames/s); D1 runs its stages one after another (233 -> 246)
    pl.halves = ASD_WTA_HALVES && halves_ok && p.D == 256 && p.lr_mode == 0;
    if (pl.halves) {
        pl.nbuf = ((256 + p.min_disp + 128 + 31) / 32) * 32;
        pl.bstride = v2::WH_BS;
        pl.rsmem = (size_t)pl.nbuf * pl.bstride * 2;
        if (pl.rsmem > 200 * 1024) return false;
        cudaFuncSetAttribute((const void*)v2::wta_halves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.rsmem);
        cudaGetLastError();
        pl.wide = true;
        return true;
    }
    pl.nbuf = ((32 * v2::wta_warps(p.D) + p.min_disp + p.D + 31) / 32) * 32;
    pl.bstride = p.D + v2::WTA_PAD;     // RowGeom<D>::BS
    pl.rsmem = (size_t)pl.nbuf * pl.bstride * 2;
    if (pl.rsmem > 200 * 1024) return false;
    for (int mode = 0; mode < 3; ++mode)
        cudaFuncSetAttribute((const void*)pick_wkernel(p.D, wide, mode), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.rsmem);
    cudaGetLastError();
    pl.wide = wide;
    return true;
}

void launch_wta2(const DevParams& p, const V2Plan& pl, int nframes, const uint16_t* S, long long cell_stride,
                 const FrameScratch& fs, long long px_stride, cudaStream_t s)
{
    RArgs r{};
    r.p = p; r.pab = const_cast<uint16_t*>(S); r.cell_stride = cell_stride; r.fs = fs; r.px_stride = px_stride;
    r.nbuf = pl.nbuf; r.bstride = pl.bstride;
    if (pl.halves) { v2::wta_halves_kernel<<<dim3(p.H, nframes), 256, pl.rsmem, s>>>(r); return; }
    RKernel k = pick_wkernel(p.D, pl.wide);
    k<<<dim3(p.H, nframes), 32 * v2::wta_warps(p.D), pl.rsmem, s>>>(r);
}

static cudaError_t launch_vsweep(VKernel k, const V2Plan& pl, int nframes, const VArgs& a, bool up, cudaStream_t s)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.ncta, nframes);
    cfg.blockDim = dim3(pl.vthreads);
    cfg.dynamicSmemBytes = up ? pl.vsmem_up : pl.vsmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pl.NP == 3 && pl.cs > 1) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, a);
}

int launch_v2_stage(int stage, const DevParams& p, const V2Plan& pl, int nframes,
                    const void* cl, const void* cr, long long sig_stride,
                    uint8_t* pa, uint16_t* pab, uint8_t* stash, long long cell_stride,
                    const FrameScratch& fs, long long px_stride, uint16_t* agg, cudaStream_t s, int variant,
                    const uint16_t* cbin)
{
    if (stage == 0 || stage == 1) {
        VArgs a{};
        a.p = p; a.w = pl.w; a.cs = pl.cs; a.ncta = pl.ncta;
        a.ghalo = pl.ghalo;
        a.tma_cen = stage == 0 && pl.tma_cen;
        if (pl.ncta > pl.cs && pl.NP == 3)       // segment-boundary tags start at 0 (no row) each launch
            cudaMemsetAsync(pl.ghalo, 0, v2_ghalo_bytes(pl, nframes), s);
        a.cl = (const uint32_t*)cl; a.cr = (const uint32_t*)cr; a.sig_stride = sig_stride;
#ifdef ASD_ABLATE
        static const int ablate = getenv("ASD_V2_ABLATE") ? atoi(getenv("ASD_V2_ABLATE")) : 0;
        a.ablate = ablate;
#endif
        a.pin = reinterpret_cast<const uint16_t*>(pa); a.pouta = reinterpret_cast<uint16_t*>(pa);
        a.pa_stride = (long long)p.H * pl.ncta * pl.w * p.D;
        a.pout16 = pab; a.cell_stride = cell_stride;
        a.cbin = cbin;
        bool segk = pl.NP == 3 && pl.ncta > pl.cs;
#ifdef ASD_ABLATE
        if (getenv("ASD_V2_FORCESEG") && pl.NP == 3) segk = true;   // experiment: SEG instance on one segment
#endif
        VKernel k = pick_vkernel(pl.DC, pl.T, pl.DPL, pl.NP, stage == 1, stage == 0 && variant == 1, pl.blk, segk);
#ifdef ASD_ABLATE
        if (getenv("ASD_V2_FORCESEG")) {
            cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(stage == 1 ? pl.vsmem_up : pl.vsmem));
            cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
#endif
        return launch_vsweep(k, pl, nframes, a, stage == 1, s) == cudaSuccess ? 0 : -1;
    }
    (void)agg;
    RArgs r{};
    r.p = p; r.cl = (const uint32_t*)cl; r.cr = (const uint32_t*)cr; r.sig_stride = sig_stride;
    r.pab = pab; r.stash = stash; r.cell_stride = cell_stride; r.fs = fs; r.px_stride = px_stride;
    r.nbuf = pl.nbuf; r.bstride = pl.bstride;
    r.p1x2 = (uint32_t)p.p1 * 0x10001u;
    r.p2x2 = (uint32_t)p.p2 * 0x10001u;
    r.cb = cbin; r.cb_stride = (long long)p.H * pl.ncta * pl.w * p.D; r.wpad = pl.ncta * pl.w;
    if (stage == 2) {
        RKernel k = pl.blk ? v2::hrow_blk_kernel<128> : pick_rkernel(p.D, variant == 1 || ASD_HROW_CFROMP, pl.NP == 3);
        const int hsm = pl.blk ? 0 : ASD_HROW_SMEM;
        if (hsm > 48 * 1024) cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
        k<<<dim3((p.H + v2::HROW_WARPS - 1) / v2::HROW_WARPS, nframes), 32 * v2::HROW_WARPS, hsm, s>>>(r);
    } else {
        if (pl.wta_fb) {
            if (!launch_wta(p, nframes, pab, cell_stride, fs, px_stride, s)) return -1;
        } else if (pl.halves && variant == 0) {
            v2::wta_halves_kernel<<<dim3(p.H, nframes), 256, pl.rsmem, s>>>(r);
        } else {
            RKernel k = pick_wkernel(p.D, pl.wide, variant);
            k<<<dim3(p.H, nframes), 32 * v2::wta_warps(p.D), pl.rsmem, s>>>(r);
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace asd
