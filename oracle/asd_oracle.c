/*
 * asd_oracle.c -- CPU ORACLE for the active-stereo depth path of arXiv 2201.11924.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2201_11924_b200/, libasd.so) never links, imports or executes it and
 * shares no code, header, table or constant generator with it.
 *
 * Plain, slow, single-threaded, scalar C99.  Build: gcc -O2 -ffp-contract=off
 * (no -ffast-math): every float operation below is one IEEE-754 operation.
 *
 * What it computes ("Depth Generation by Stereo Matching";
 * SPEC.md S:288-356 [OP] census .. disp_to_depth; readings c1-c14 of
 * SURVEY.md §8(c), restated in DESIGN.md §3):
 *
 *   O1 census      CSCT bit i = I(p + o_i) > I(p - o_i)
 *   O2 cost        C = popcount(cl(x,y) XOR cr(x-delta,y)) or nb
 *   O2b SGBM cost  CB(x,y,d) = sum over the bw x bh block of C(x+u,y+v,d),
 *                  nb for block positions outside the image
 *   O3 SGM         L_r(p,d) = C + min(L_r(p-r,d), L_r(p-r,d+-1)+P1,
 *                                     min_k L_r(p-r,k)+P2) - min_k L_r(p-r,k)
 *                  S = sum_r L_r
 *   O4 WTA         smallest argmin + uniqueness test
 *   O5 sub-pixel   parabola through (d*-1, d*, d*+1)
 *   O6 right view  same WTA/sub-pixel on S_R(x,d) = S(x+delta,d)  (reading c10)
 *   O6b right view R2: SGM of the right-referenced cost
 *                  C_R(x,y,d) = hamming(cr(x,y), cl(x+delta,y))   (reading c24)
 *   O7 LR check    |dl - dr(x - round(dl))| <= lr
 *   O9 median      lower median of the valid k x k neighbours
 *   O8 depth       z = f*b/d
 *   O10 register   unproject, transform, reproject, z-buffer
 *   O00 rectify    homography warp, bilinear sampling              (c23)
 *   O0 noise       I_noisy = gamma * I_clean + n, gamma ~ Gamma(k, theta),
 *                  n ~ N(mu, sigma^2), quantised to u8           (c17, c22)
 *
 * Every function follows the definition in that order, with no blocking,
 * fusion or reordering.  SGM is organised exactly as its definition reads:
 * each path r decomposes the image into independent 1-D lines (rows, columns,
 * diagonals) and the recursion runs along each line (oracle_chain).
 *
 * Precision: integers are exact (uint32/int64).  The sub-pixel offset is one
 * fp32 division because its value decides an integer (the LR rounding,
 * reading c11/c13) and the kernel decides it in fp32; the depth is fp64.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct {
    int32_t width, height;     /* W, H */
    int32_t min_disp, num_disp;/* delta(d) = min_disp + d, d in [0, D) */
    int32_t census_w, census_h;/* odd window */
    int32_t p1, p2;            /* SGM penalties */
    int32_t paths;             /* 4 or 8 */
    int32_t uniqueness;        /* percent; < 0 disables */
    float   lr_max_diff;       /* px; < 0 disables */
    int32_t subpixel;          /* 0/1 */
    float   focal_px, baseline_m;
    int32_t block_w, block_h;  /* SGBM block (odd); 1 x 1 = plain SGM */
    int32_t median_ksize;      /* 0 (off), 3 or 5 */
    int32_t lr_mode;           /* right view: 0 = R1 re-index S (c10), 1 = R2 full right-view SGM (c24) */
} oracle_params;

/* mask bits */
#define OM_BORDER 1u   /* census window leaves the image (c4), or no defined d (right view) */
#define OM_UNIQUE 2u   /* uniqueness test failed (O4) */
#define OM_LR     4u   /* left-right check failed (O7) */
#define OM_NONPOS 8u   /* dl <= 0 (O8) */

static int nbits(const oracle_params* p) { return (p->census_w * p->census_h) / 2; }

static int valid_c(const oracle_params* p, int x, int y) {
    int R = p->census_w / 2, Q = p->census_h / 2;
    return x >= R && x < p->width - R && y >= Q && y < p->height - Q;
}

/* ---------------------------------------------------------------- O1 census
 * CSCT: for each of the floor(w*h/2) point-symmetric pairs
 * (p_a, p_b) around the centre, bit = I(p_a) > I(p_b), with p_a running over
 * the window in row-major order up to (excluding) the centre.  Pair i -> bit i
 * (LSB first, reading c1).  Pixels whose window leaves the image get 0.
 */
void oracle_census(const oracle_params* p, const uint8_t* img, uint64_t* out)
{
    int W = p->width, H = p->height, cw = p->census_w;
    int R = p->census_w / 2, Q = p->census_h / 2, nb = nbits(p);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            uint64_t sig = 0;
            if (valid_c(p, x, y)) {
                for (int i = 0; i < nb; ++i) {
                    int dy = i / cw - Q;          /* p_a = p + (dx, dy), i-th window pixel */
                    int dx = i % cw - R;
                    uint8_t a = img[(y + dy) * W + (x + dx)];
                    uint8_t b = img[(y - dy) * W + (x - dx)];   /* p_b = p - (dx, dy) */
                    if (a > b) sig |= (uint64_t)1 << i;
                }
            }
            out[y * W + x] = sig;
        }
}

static int popcount64(uint64_t v) { int n = 0; while (v) { n += (int)(v & 1u); v >>= 1; } return n; }

/* ------------------------------------------------------------------ O2 cost
 * C(x,y,d) = hamming(cl[x,y], cr[x-delta,y]) ("hamming distance as the
 * cost function").  Out of range or census border -> nb (reading c3).
 * Layout [H][W][D], d fastest.
 */
void oracle_cost(const oracle_params* p, const uint64_t* cl, const uint64_t* cr, uint8_t* C)
{
    int W = p->width, H = p->height, D = p->num_disp, nb = nbits(p);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int d = 0; d < D; ++d) {
                int xr = x - (p->min_disp + d);
                int c = nb;
                if (valid_c(p, x, y) && xr >= 0 && valid_c(p, xr, y))
                    c = popcount64(cl[y * W + x] ^ cr[y * W + xr]);
                C[((size_t)y * W + x) * D + d] = (uint8_t)c;
            }
}

/* O2 for the right view as reference (reading c24, "run the pipeline
 * with roles swapped"): C_R(x,y,d) = hamming(cr(x,y), cl(x+delta,y)), nb when
 * x + delta >= W or either census window is invalid.  Layout [H][W][D]. */
void oracle_cost_right(const oracle_params* p, const uint64_t* cl, const uint64_t* cr, uint8_t* C)
{
    int W = p->width, H = p->height, D = p->num_disp, nb = nbits(p);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int d = 0; d < D; ++d) {
                int xl = x + (p->min_disp + d);
                int c = nb;
                if (valid_c(p, x, y) && xl < W && valid_c(p, xl, y))
                    c = popcount64(cr[y * W + x] ^ cl[y * W + xl]);
                C[((size_t)y * W + x) * D + d] = (uint8_t)c;
            }
}

/* ---------------------------------------------------------- O2b SGBM cost
 * SGBM ("SGBM computes the cost by the hamming distance between the
 * local regions of the two pixels"; "for SGBM, sum of hamming over the
 * block around both pixels"): the same offset (u,v) is applied to both pixels,
 *   CB(x,y,d) = sum_{|u| <= bw/2, |v| <= bh/2} C~(x+u, y+v, d),
 * C~ = C (O2, nb for invalid / out of range) inside the image and nb outside
 * (reading c19: a block position off the image is an invalid match, c3).
 * bw = bh = 1 gives CB = C.  Layout [H][W][D], u32.
 */
void oracle_block_cost(const oracle_params* p, const uint8_t* C, uint32_t* CB)
{
    int W = p->width, H = p->height, D = p->num_disp, nb = nbits(p);
    int bu = p->block_w / 2, bv = p->block_h / 2;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int d = 0; d < D; ++d) {
                uint32_t sum = 0;
                for (int v = -bv; v <= bv; ++v)
                    for (int u = -bu; u <= bu; ++u) {
                        int xx = x + u, yy = y + v;
                        if (xx >= 0 && xx < W && yy >= 0 && yy < H)
                            sum += C[((size_t)yy * W + xx) * D + d];
                        else
                            sum += (uint32_t)nb;
                    }
                CB[((size_t)y * W + x) * D + d] = sum;
            }
}

/* ------------------------------------------------------------- O3 one line
 * The SGM recursion along one line of n pixels ("four-path semi-global
 * matching (SGM) [Hirschmuller]"):
 *   L(0,d) = C(0,d)
 *   L(i,d) = C(i,d) + min( L(i-1,d), L(i-1,d-1)+P1, L(i-1,d+1)+P1, M+P2 ) - M,
 *   M = min_k L(i-1,k); the d-1 / d+1 terms are omitted at the range ends.
 * Cin and Lout are [n][D].
 */
void oracle_chain(int n, int D, int P1, int P2, const uint32_t* Cin, uint32_t* Lout)
{
    for (int i = 0; i < n; ++i) {
        const uint32_t* c = Cin + (size_t)i * D;
        uint32_t* l = Lout + (size_t)i * D;
        if (i == 0) {
            for (int d = 0; d < D; ++d) l[d] = c[d];
            continue;
        }
        const uint32_t* prev = Lout + (size_t)(i - 1) * D;
        uint32_t M = prev[0];
        for (int k = 1; k < D; ++k) if (prev[k] < M) M = prev[k];
        for (int d = 0; d < D; ++d) {
            uint32_t best = prev[d];
            if (d >= 1     && prev[d - 1] + (uint32_t)P1 < best) best = prev[d - 1] + (uint32_t)P1;
            if (d <= D - 2 && prev[d + 1] + (uint32_t)P1 < best) best = prev[d + 1] + (uint32_t)P1;
            if (M + (uint32_t)P2 < best) best = M + (uint32_t)P2;
            l[d] = c[d] + best - M;
        }
    }
}

/* Path directions r (the traversal step; the predecessor of p is p - r).
 * 4-path = the two horizontal and two vertical directions ("four-path";
 * S:309); 8-path adds the four diagonals (reading c6). */
static const int DIRS[8][2] = {
    {+1, 0}, {-1, 0}, {0, +1}, {0, -1},     /* 4-path */
    {+1, +1}, {-1, -1}, {+1, -1}, {-1, +1}  /* + diagonals */
};

int oracle_num_dirs(void) { return 8; }
void oracle_dir(int i, int* rx, int* ry) { *rx = DIRS[i][0]; *ry = DIRS[i][1]; }

static int inside(const oracle_params* p, int x, int y) {
    return x >= 0 && x < p->width && y >= 0 && y < p->height;
}

/* L_r for one direction over the whole image: every line of direction r starts
 * at a pixel whose predecessor p - r is outside the image ("first pixel of each
 * path: L_r = C") and is walked forward with oracle_chain. */
void oracle_sgm_path32(const oracle_params* p, const uint32_t* C, int rx, int ry, uint32_t* L)
{
    int W = p->width, H = p->height, D = p->num_disp;
    int nmax = W > H ? W : H;
    uint32_t* cbuf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nmax * D);
    uint32_t* lbuf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nmax * D);
    int* xs = (int*)malloc(sizeof(int) * nmax);
    int* ys = (int*)malloc(sizeof(int) * nmax);
    for (int y0 = 0; y0 < H; ++y0)
        for (int x0 = 0; x0 < W; ++x0) {
            if (inside(p, x0 - rx, y0 - ry)) continue;   /* not the start of a line */
            int n = 0, x = x0, y = y0;
            while (inside(p, x, y)) {
                xs[n] = x; ys[n] = y;
                for (int d = 0; d < D; ++d)
                    cbuf[(size_t)n * D + d] = C[((size_t)y * W + x) * D + d];
                ++n; x += rx; y += ry;
            }
            oracle_chain(n, D, p->p1, p->p2, cbuf, lbuf);
            for (int i = 0; i < n; ++i)
                for (int d = 0; d < D; ++d)
                    L[((size_t)ys[i] * W + xs[i]) * D + d] = lbuf[(size_t)i * D + d];
        }
    free(cbuf); free(lbuf); free(xs); free(ys);
}

/* S = sum_r L_r over the configured path set, on a u32 cost volume
 * (the per-pixel Hamming cost O2 or the SGBM block cost O2b). */
void oracle_sgm32(const oracle_params* p, const uint32_t* C, uint32_t* S)
{
    size_t n = (size_t)p->width * p->height * p->num_disp;
    uint32_t* L = (uint32_t*)malloc(sizeof(uint32_t) * n);
    memset(S, 0, sizeof(uint32_t) * n);
    for (int r = 0; r < p->paths; ++r) {
        oracle_sgm_path32(p, C, DIRS[r][0], DIRS[r][1], L);
        for (size_t i = 0; i < n; ++i) S[i] += L[i];
    }
    free(L);
}

/* The same on the u8 Hamming cost volume of O2 (values widened, unchanged). */
static uint32_t* widen(const oracle_params* p, const uint8_t* C)
{
    size_t n = (size_t)p->width * p->height * p->num_disp;
    uint32_t* C32 = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (size_t i = 0; i < n; ++i) C32[i] = C[i];
    return C32;
}
void oracle_sgm_path(const oracle_params* p, const uint8_t* C, int rx, int ry, uint32_t* L)
{
    uint32_t* C32 = widen(p, C);
    oracle_sgm_path32(p, C32, rx, ry, L);
    free(C32);
}
void oracle_sgm(const oracle_params* p, const uint8_t* C, uint32_t* S)
{
    uint32_t* C32 = widen(p, C);
    oracle_sgm32(p, C32, S);
    free(C32);
}

/* S(x,y,.) for ONE pixel, computed from the raw cost volume by walking, for
 * each path r, the line through (x,y) from its image-border start to (x,y).
 * Same recursion (oracle_chain); used to check sampled pixels at full size. */
void oracle_sgm_pixel_from_census(const oracle_params* p, const uint64_t* cl, const uint64_t* cr,
                                  int x, int y, uint32_t* Sout)
{
    int W = p->width, H = p->height, D = p->num_disp, nb = nbits(p);
    int nmax = W > H ? W : H;
    uint32_t* cbuf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nmax * D);
    uint32_t* lbuf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nmax * D);
    for (int d = 0; d < D; ++d) Sout[d] = 0;
    for (int r = 0; r < p->paths; ++r) {
        int rx = DIRS[r][0], ry = DIRS[r][1];
        int sx = x, sy = y, n = 1;                 /* back up to the start of the line */
        while (inside(p, sx - rx, sy - ry)) { sx -= rx; sy -= ry; ++n; }
        int bu = p->block_w / 2, bv = p->block_h / 2;
        for (int i = 0; i < n; ++i) {
            int px = sx + i * rx, py = sy + i * ry;
            for (int d = 0; d < D; ++d) {          /* O2 / O2b restated for this pixel */
                uint32_t sum = 0;
                for (int v = -bv; v <= bv; ++v)
                    for (int u = -bu; u <= bu; ++u) {
                        int qx = px + u, qy = py + v, xr = qx - (p->min_disp + d);
                        int c = nb;
                        if (qx >= 0 && qx < W && qy >= 0 && qy < H &&
                            valid_c(p, qx, qy) && xr >= 0 && valid_c(p, xr, qy))
                            c = popcount64(cl[qy * W + qx] ^ cr[qy * W + xr]);
                        sum += (uint32_t)c;
                    }
                cbuf[(size_t)i * D + d] = sum;
            }
        }
        oracle_chain(n, D, p->p1, p->p2, cbuf, lbuf);
        for (int d = 0; d < D; ++d) Sout[d] += lbuf[(size_t)(n - 1) * D + d];
    }
    free(cbuf); free(lbuf);
}

/* ------------------------------------------------- O4 + O5 on one vector
 * WTA: d* = smallest d minimising s over the defined entries.
 * Uniqueness ("filter out disparities that are not better than the
 * second best match by a threshold", reading c8): invalid iff
 *   T = {d defined : |d - d*| >= 2} is non-empty and s(d*)*(100+u) >= min_T s * 100.
 * Sub-pixel ("quadratic curve fitting", reading c13): if on and
 * d*-1, d*+1 are both defined, den = c- - 2c0 + c+; off = den > 0 ?
 * (float)(c- - c+) / (float)(2 den) : 0, clamped to [-0.5, 0.5];
 * disparity = (float)(min_disp + d*) + off.
 * defined[d] == 0 removes d from the search (right view, O6).
 * Returns d* (or -1 if nothing is defined); sets *unique_fail, *disp.
 */
static int wta_subpix(const oracle_params* p, const uint32_t* s, const uint8_t* defined,
                      int* unique_fail, float* disp)
{
    int D = p->num_disp, best = -1;
    for (int d = 0; d < D; ++d)
        if (defined[d] && (best < 0 || s[d] < s[best])) best = d;
    *unique_fail = 0;
    if (best < 0) { *disp = 0.0f; return -1; }
    if (p->uniqueness >= 0) {
        int have = 0; uint32_t second = 0;
        for (int d = 0; d < D; ++d) {
            if (!defined[d] || abs(d - best) < 2) continue;
            if (!have || s[d] < second) { second = s[d]; have = 1; }
        }
        if (have && (int64_t)s[best] * (100 + (int64_t)p->uniqueness) >= (int64_t)second * 100)
            *unique_fail = 1;
    }
    float off = 0.0f;
    if (p->subpixel && best >= 1 && best <= D - 2 && defined[best - 1] && defined[best + 1]) {
        int64_t cm = s[best - 1], c0 = s[best], cp = s[best + 1];
        int64_t den = cm - 2 * c0 + cp;
        if (den > 0) {
            off = (float)(cm - cp) / (float)(2 * den);
            if (off < -0.5f) off = -0.5f;
            if (off > 0.5f) off = 0.5f;
        }
    }
    *disp = (float)(p->min_disp + best) + off;
    return best;
}

/* O4 + O5, left view, every pixel.  mask gets OM_BORDER (reading c4) and OM_UNIQUE. */
void oracle_wta_left(const oracle_params* p, const uint32_t* S,
                     int16_t* dstar, uint8_t* mask, float* dl)
{
    int W = p->width, H = p->height, D = p->num_disp;
    uint8_t* defined = (uint8_t*)malloc((size_t)D);
    for (int d = 0; d < D; ++d) defined[d] = 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            int uf; float disp;
            int b = wta_subpix(p, S + ((size_t)y * W + x) * D, defined, &uf, &disp);
            uint8_t m = 0;
            if (!valid_c(p, x, y)) m |= OM_BORDER;
            if (uf) m |= OM_UNIQUE;
            dstar[y * W + x] = (int16_t)b;
            mask[y * W + x] = m;
            dl[y * W + x] = disp;
        }
    free(defined);
}

/* O6 right view (reading c10 = R1, "reuses the same cost volume by
 * re-indexing"): S_R(xr,y,d) = S(xr + delta(d), y, d), defined iff
 * xr + delta(d) < W; then O4 + O5 over the defined d.  mask_r gets OM_BORDER
 * when the right pixel's census window leaves the image or no d is defined. */
void oracle_wta_right(const oracle_params* p, const uint32_t* S,
                      int16_t* dstar_r, uint8_t* mask_r, float* dr)
{
    int W = p->width, H = p->height, D = p->num_disp;
    uint32_t* sr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)D);
    uint8_t* defined = (uint8_t*)malloc((size_t)D);
    for (int y = 0; y < H; ++y)
        for (int xr = 0; xr < W; ++xr) {
            for (int d = 0; d < D; ++d) {
                int x = xr + p->min_disp + d;
                defined[d] = (uint8_t)(x < W);
                sr[d] = x < W ? S[((size_t)y * W + x) * D + d] : 0;
            }
            int uf; float disp;
            int b = wta_subpix(p, sr, defined, &uf, &disp);
            uint8_t m = 0;
            if (!valid_c(p, xr, y) || b < 0) m |= OM_BORDER;
            if (uf) m |= OM_UNIQUE;
            dstar_r[y * W + xr] = (int16_t)b;
            mask_r[y * W + xr] = m;
            dr[y * W + xr] = disp;
        }
    free(sr); free(defined);
}

/* O9 median ("median filtering"; S:342-347 [OP] median, reading c20):
 * for a pixel valid after the LR check ((mask & 7) == 0), the lower median
 * (element (n-1)/2 of the ascending order) of dl over the pixels of the
 * k x k window inside the image that are valid too (n >= 1: the pixel itself);
 * invalid pixels keep dl.  ksize 0 = identity. */
static int cmp_float(const void* a, const void* b)
{
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}
void oracle_median(const oracle_params* p, const float* dl, const uint8_t* mask, float* out)
{
    int W = p->width, H = p->height, k = p->median_ksize / 2;
    float v[64];
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            out[i] = dl[i];
            if (p->median_ksize <= 0 || (mask[i] & 7u) != 0) continue;
            int n = 0;
            for (int yy = y - k; yy <= y + k; ++yy)
                for (int xx = x - k; xx <= x + k; ++xx) {
                    if (xx < 0 || xx >= W || yy < 0 || yy >= H) continue;
                    size_t j = (size_t)yy * W + xx;
                    if ((mask[j] & 7u) == 0) v[n++] = dl[j];
                }
            qsort(v, (size_t)n, sizeof(float), cmp_float);
            out[i] = v[(n - 1) / 2];
        }
}

/* O6b right view R2 (reading c24): WTA + uniqueness + sub-pixel over every d
 * of the right-referenced aggregate S_R (as the left view); mask_r gets
 * OM_BORDER when the right pixel's census window leaves the image. */
void oracle_wta_right_r2(const oracle_params* p, const uint32_t* SR,
                         int16_t* dstar_r, uint8_t* mask_r, float* dr)
{
    int W = p->width, H = p->height, D = p->num_disp;
    uint8_t* defined = (uint8_t*)malloc((size_t)D);
    for (int d = 0; d < D; ++d) defined[d] = 1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            int uf; float disp;
            int b = wta_subpix(p, SR + ((size_t)y * W + x) * D, defined, &uf, &disp);
            uint8_t m = 0;
            if (!valid_c(p, x, y)) m |= OM_BORDER;
            if (uf) m |= OM_UNIQUE;
            dstar_r[y * W + x] = (int16_t)b;
            mask_r[y * W + x] = m;
            dr[y * W + x] = disp;
        }
    free(defined);
}

/* O7 + O9 + O8.  LR ("left-right consistency check", readings
 * c11, c12): evaluated iff lr >= 0 and (mask & 3) == 0; xr = x - (int)floorf(dl
 * + 0.5f); invalid if xr outside [0,W), mask_r(xr) != 0 or |dl - dr(xr)| > lr.
 * Then the median (O9) of the LR-checked map when median_ksize > 0 (S:368
 * order: lr_check -> median -> disp_to_depth).  Depth (reading
 * c14) on that value d: OM_NONPOS iff d <= 0 (always evaluated); if mask == 0:
 * disp = d, depth = f*b/d in fp64; else both NaN. */
void oracle_lr_depth(const oracle_params* p, const float* dl, const float* dr,
                     const uint8_t* mask_r, uint8_t* mask, float* disp, double* depth)
{
    int W = p->width, H = p->height;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            uint8_t m = mask[i];
            float d = dl[i];
            if (p->lr_max_diff >= 0.0f && (m & 3u) == 0) {
                int xr = x - (int)floorf(d + 0.5f);
                if (xr < 0 || xr >= W) m |= OM_LR;
                else {
                    size_t j = (size_t)y * W + xr;
                    if (mask_r[j] != 0 || fabsf(d - dr[j]) > p->lr_max_diff) m |= OM_LR;
                }
            }
            mask[i] = m;
        }
    float* dm = (float*)malloc(sizeof(float) * (size_t)W * H);
    oracle_median(p, dl, mask, dm);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            uint8_t m = mask[i];
            float d = dm[i];
            if (d <= 0.0f) m |= OM_NONPOS;
            mask[i] = m;
            if (m == 0) {
                disp[i] = d;
                depth[i] = (double)p->focal_px * (double)p->baseline_m / (double)d;
            } else {
                disp[i] = NAN;
                depth[i] = NAN;
            }
        }
    free(dm);
}

/* O10 depth registration ("an optional depth registration that aligns
 * the depth map to the RGB camera frame"; S:357-365 [OP] register_depth,
 * reading c21).  Pinhole cameras without distortion; pixel (x, y) sits at
 * image coordinate (x, y).  Each source pixel with finite z > 0 is unprojected
 * with the IR intrinsics, moved into the RGB frame (P' = R P + t, R row-major),
 * reprojected with the RGB intrinsics; the target pixel is
 * (floor(u + 0.5), floor(v + 0.5)) and the z-buffer keeps the smallest Z'.
 * Targets never hit are NaN.  The coordinate arithmetic decides integers (the
 * target pixel), so it is done in fp32, one IEEE operation at a time in the
 * order written (the kernel does the same, reading c21):
 *   a = ((float)x - cx) * z / fx,  b = ((float)y - cy) * z / fy
 *   X' = ((R00 a + R01 b) + R02 z) + t0   (likewise Y', Z')
 *   u = (X' / Z') * fx' + cx',  v = (Y' / Z') * fy' + cy'                  */
typedef struct { int32_t width, height; float fx, fy, cx, cy; } oracle_camera;

void oracle_register(const oracle_camera* ir, const oracle_camera* rgb, const float* R, const float* t,
                     const float* z_in, float* z_out)
{
    size_t nt = (size_t)rgb->width * rgb->height;
    for (size_t i = 0; i < nt; ++i) z_out[i] = INFINITY;
    for (int y = 0; y < ir->height; ++y)
        for (int x = 0; x < ir->width; ++x) {
            float z = z_in[(size_t)y * ir->width + x];
            if (!(z > 0.0f) || isinf(z)) continue;        /* NaN (invalid) or non-positive */
            float a = (float)x - ir->cx; a = a * z; a = a / ir->fx;
            float b = (float)y - ir->cy; b = b * z; b = b / ir->fy;
            float P[3];
            for (int r = 0; r < 3; ++r) {
                float s = R[3 * r] * a;
                s = s + R[3 * r + 1] * b;
                s = s + R[3 * r + 2] * z;
                P[r] = s + t[r];
            }
            if (!(P[2] > 0.0f)) continue;
            float u = P[0] / P[2]; u = u * rgb->fx; u = u + rgb->cx;
            float v = P[1] / P[2]; v = v * rgb->fy; v = v + rgb->cy;
            float uu = u + 0.5f, vv = v + 0.5f;
            if (!(uu >= 0.0f && uu < (float)rgb->width && vv >= 0.0f && vv < (float)rgb->height)) continue;
            int iu = (int)floorf(uu), iv = (int)floorf(vv);
            size_t j = (size_t)iv * rgb->width + iu;
            if (P[2] < z_out[j]) z_out[j] = P[2];
        }
    for (size_t i = 0; i < nt; ++i) if (isinf(z_out[i])) z_out[i] = NAN;
}

/* murmur3 fmix32 -- per-frame checksum of the bit-exact outputs. */
static uint32_t fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}
uint32_t oracle_checksum(int n, const int16_t* dstar, const uint8_t* mask)
{
    uint32_t h = 0;
    for (int i = 0; i < n; ++i)
        h += fmix32(((uint32_t)i * 0x9E3779B1u) ^ ((uint32_t)(dstar[i] + 1) << 8) ^ (uint32_t)mask[i]);
    return h;
}

/* The whole path, O1..O8 in the order of P:289 (S:366-368 compute_depth with
 * rectification = identity for a born-rectified rig and median off).  Any of the
 * debug outputs may be NULL.  Returns 0, or -1 on allocation failure. */
int oracle_compute(const oracle_params* p, const uint8_t* left, const uint8_t* right,
                   float* out_disp, double* out_depth,
                   uint64_t* census_l, uint64_t* census_r, uint8_t* cost, uint32_t* agg,
                   int16_t* dstar_l, int16_t* dstar_r, float* dl_out, float* dr_out,
                   uint8_t* mask_out, uint8_t* mask_r_out)
{
    size_t npx = (size_t)p->width * p->height, ncell = npx * p->num_disp;
    uint64_t* cl = (uint64_t*)malloc(sizeof(uint64_t) * npx);
    uint64_t* cr = (uint64_t*)malloc(sizeof(uint64_t) * npx);
    uint8_t* C = (uint8_t*)malloc(ncell);
    uint32_t* CB = (uint32_t*)malloc(sizeof(uint32_t) * ncell);
    uint32_t* S = (uint32_t*)malloc(sizeof(uint32_t) * ncell);
    int16_t* dsl = (int16_t*)malloc(sizeof(int16_t) * npx);
    int16_t* dsr = (int16_t*)malloc(sizeof(int16_t) * npx);
    uint8_t* ml = (uint8_t*)malloc(npx);
    uint8_t* mr = (uint8_t*)malloc(npx);
    float* dl = (float*)malloc(sizeof(float) * npx);
    float* dr = (float*)malloc(sizeof(float) * npx);
    float* disp = (float*)malloc(sizeof(float) * npx);
    double* z = (double*)malloc(sizeof(double) * npx);
    int rc = -1;
    if (!cl || !cr || !C || !CB || !S || !dsl || !dsr || !ml || !mr || !dl || !dr || !disp || !z) goto done;
    oracle_census(p, left, cl);                 /* O1 */
    oracle_census(p, right, cr);
    oracle_cost(p, cl, cr, C);                  /* O2 */
    oracle_block_cost(p, C, CB);                /* O2b (1 x 1: CB = C) */
    oracle_sgm32(p, CB, S);                     /* O3 */
    oracle_wta_left(p, S, dsl, ml, dl);         /* O4, O5 */
    if (p->lr_mode == 1) {                      /* O6b: R2, the right view's own SGM */
        oracle_cost_right(p, cl, cr, C);
        oracle_block_cost(p, C, CB);
        oracle_sgm32(p, CB, S);
        oracle_wta_right_r2(p, S, dsr, mr, dr);
        if (cost || agg) {                      /* debug outputs stay the left view's */
            oracle_cost(p, cl, cr, C);
            oracle_block_cost(p, C, CB);
            oracle_sgm32(p, CB, S);
        }
    } else {
        oracle_wta_right(p, S, dsr, mr, dr);    /* O6 (R1) */
    }
    oracle_lr_depth(p, dl, dr, mr, ml, disp, z);/* O7, O8 */
    if (out_disp) memcpy(out_disp, disp, sizeof(float) * npx);
    if (out_depth) memcpy(out_depth, z, sizeof(double) * npx);
    if (census_l) memcpy(census_l, cl, sizeof(uint64_t) * npx);
    if (census_r) memcpy(census_r, cr, sizeof(uint64_t) * npx);
    if (cost) memcpy(cost, C, ncell);
    if (agg) memcpy(agg, S, sizeof(uint32_t) * ncell);
    if (dstar_l) memcpy(dstar_l, dsl, sizeof(int16_t) * npx);
    if (dstar_r) memcpy(dstar_r, dsr, sizeof(int16_t) * npx);
    if (dl_out) memcpy(dl_out, dl, sizeof(float) * npx);
    if (dr_out) memcpy(dr_out, dr, sizeof(float) * npx);
    if (mask_out) memcpy(mask_out, ml, npx);
    if (mask_r_out) memcpy(mask_r_out, mr, npx);
    rc = 0;
done:
    free(cl); free(cr); free(C); free(CB); free(S); free(dsl); free(dsr); free(ml); free(mr);
    free(dl); free(dr); free(disp); free(z);
    return rc;
}


/* ------------------------------------------------------------- O0 noise
 * Sensor noise front end ("a multiplicative term gamma
 * modeling the laser speckle and an additive term n modeling camera thermal
 * noise", I_noisy = gamma * I_clean + n, gamma ~ Gamma(k, theta), n ~ N(mu,
 * sigma^2); D415 values P:350; readings c17, c22 in DESIGN.md §3).
 *
 * Random numbers: Philox4x32-10 (Salmon et al., SC'11: a 10-round Feistel-like
 * bijection of a 128-bit counter under a 64-bit key; round multipliers
 * 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85),
 * key = (seed low, seed high 32 bits), counter = (pixel, attempt, frame, view).
 * A 32-bit output x maps to the open interval: U(x) = ((x >> 8) + 0.5) / 2^24.
 * Normal: Box-Muller, z = sqrt(-2 ln U(x0)) cos(2 pi U(x1)).
 * n: the block with attempt = 0xFFFFFFFF; n = mu + sigma z.
 * Gamma (Marsaglia & Tsang 2000): k' = k (k >= 1) or k + 1 (k < 1 boost),
 * d = k' - 1/3, c = 1 / sqrt(9 d); attempt j = 0..15: z from block j, v =
 * (1 + c z)^3, accept iff v > 0 and ln U(x2) < z^2 / 2 + d - d v + d ln v,
 * g = d v; for k < 1, g *= U(x3 of block 0)^(1/k); no acceptance in 16
 * attempts (probability < 1e-25 at k = 3.98) -> g = d.  gamma = g * theta.
 * Noise scale s: gamma' = k theta + s (gamma - k theta), n' = s n.
 * Output: clamp(floor(gamma' I + n' + 0.5), 0, 255) as u8 (c17).
 * All arithmetic in double (the kernel also computes in double).           */
static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    for (int i = 0; i < 4; ++i) out[i] = c[i];
}
static double unif(uint32_t x) { return ((double)(x >> 8) + 0.5) / 16777216.0; }
static const double PI_D = 3.14159265358979323846;

typedef struct {
    double k, theta, mu, sigma, scale;
} oracle_noise;

static double bm_normal(const uint32_t x[4])
{
    return sqrt(-2.0 * log(unif(x[0]))) * cos(2.0 * PI_D * unif(x[1]));
}

/* gamma and n for one pixel (both before the scale blend) */
static void noise_pixel(const oracle_noise* q, uint64_t seed, uint32_t pix, uint32_t frame, uint32_t view,
                        double* gamma, double* n)
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {pix, 0xFFFFFFFFu, frame, view}, x[4];
    oracle_philox4x32_10(ctr, key, x);
    *n = q->mu + q->sigma * bm_normal(x);
    double kk = q->k >= 1.0 ? q->k : q->k + 1.0;
    double d = kk - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    double g = d, boost = 1.0;
    for (uint32_t j = 0; j < 16; ++j) {
        ctr[1] = j;
        oracle_philox4x32_10(ctr, key, x);
        if (j == 0 && q->k < 1.0) boost = pow(unif(x[3]), 1.0 / q->k);
        double z = bm_normal(x);
        double t = 1.0 + c * z;
        double v = t * t * t;
        if (v <= 0.0) continue;
        if (log(unif(x[2])) < 0.5 * z * z + d - d * v + d * log(v)) { g = d * v; break; }
    }
    *gamma = g * boost * q->theta;
}

/* n_images clean images [n][H][W] (double) -> u8 [n][H][W]; image i is frame
 * frame0 + i of view `view`.  noisy_f64 (may be NULL) gets gamma' I + n' before
 * rounding. */
void oracle_sensor_noise(const oracle_noise* q, uint64_t seed, int n_images, int W, int H,
                         uint32_t frame0, uint32_t view, const double* clean, uint8_t* out, double* noisy_f64)
{
    for (int i = 0; i < n_images; ++i)
        for (int pix = 0; pix < W * H; ++pix) {
            double g, n;
            noise_pixel(q, seed, (uint32_t)pix, frame0 + (uint32_t)i, view, &g, &n);
            double kt = q->k * q->theta;
            double gs = kt + q->scale * (g - kt), ns = q->scale * n;
            size_t o = (size_t)i * W * H + pix;
            double val = gs * clean[o] + ns;
            if (noisy_f64) noisy_f64[o] = val;
            double r = floor(val + 0.5);
            if (r < 0.0) r = 0.0;
            if (r > 255.0) r = 255.0;
            out[o] = (uint8_t)r;
        }
}

/* The gamma and n samples of pixels 0..n-1 of one (frame, view) stream, for
 * distribution tests. */
void oracle_noise_samples(const oracle_noise* q, uint64_t seed, int n, uint32_t frame, uint32_t view,
                          double* gamma, double* add)
{
    for (int i = 0; i < n; ++i) noise_pixel(q, seed, (uint32_t)i, frame, view, gamma + i, add + i);
}


/* ------------------------------------------------------------ O00 rectify
 * Stereo rectification ("performs a stereo rectification to project the
 * images onto a common image plane"; S:279-287 [OP] rectify: "warp by
 * supplied 3x3 homographies with bilinear sampling"; reading c23): H maps
 * OUTPUT pixel coordinates to INPUT coordinates (row-major, homogeneous):
 *   w = H20 x + H21 y + H22,  u = (H00 x + H01 y + H02) / w,  v = (...) / w;
 *   x0 = floor(u), y0 = floor(v), a = u - x0, b = v - y0;
 *   out = (1-a)(1-b) I(x0,y0) + a(1-b) I(x0+1,y0) + (1-a) b I(x0,y0+1) + a b I(x0+1,y0+1),
 *   I = 0 outside the image (and w <= 0 gives 0); u8 = clamp(floor(out + 0.5), 0, 255).
 * fp64, in this order (the kernel does the same).  Returns -1 for a singular H. */
int oracle_rectify(const double* Hm, int W, int H, const uint8_t* in, uint8_t* out)
{
    double det = Hm[0] * (Hm[4] * Hm[8] - Hm[5] * Hm[7]) - Hm[1] * (Hm[3] * Hm[8] - Hm[5] * Hm[6]) +
                 Hm[2] * (Hm[3] * Hm[7] - Hm[4] * Hm[6]);
    if (!(fabs(det) > 0.0) || isnan(det)) return -1;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double w = Hm[6] * x + Hm[7] * y + Hm[8];
            double val = 0.0;
            if (w > 0.0) {
                double u = (Hm[0] * x + Hm[1] * y + Hm[2]) / w;
                double v = (Hm[3] * x + Hm[4] * y + Hm[5]) / w;
                if (u > -2.0 && u < W + 1.0 && v > -2.0 && v < H + 1.0) {
                    double fx0 = floor(u), fy0 = floor(v);
                    int x0 = (int)fx0, y0 = (int)fy0;
                    double a = u - fx0, b = v - fy0;
                    double I00 = 0, I10 = 0, I01 = 0, I11 = 0;
                    if (x0 >= 0 && x0 < W && y0 >= 0 && y0 < H) I00 = in[y0 * W + x0];
                    if (x0 + 1 >= 0 && x0 + 1 < W && y0 >= 0 && y0 < H) I10 = in[y0 * W + x0 + 1];
                    if (x0 >= 0 && x0 < W && y0 + 1 >= 0 && y0 + 1 < H) I01 = in[(y0 + 1) * W + x0];
                    if (x0 + 1 >= 0 && x0 + 1 < W && y0 + 1 >= 0 && y0 + 1 < H) I11 = in[(y0 + 1) * W + x0 + 1];
                    val = (1.0 - a) * (1.0 - b) * I00 + a * (1.0 - b) * I10 + (1.0 - a) * b * I01 + a * b * I11;
                }
            }
            double r = floor(val + 0.5);
            if (r < 0.0) r = 0.0;
            if (r > 255.0) r = 255.0;
            out[y * W + x] = (uint8_t)r;
        }
    return 0;
}
