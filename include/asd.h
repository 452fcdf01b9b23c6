/*
 * asd.h -- C ABI of the B200-native active-stereo depth engine (libasd.so).
 *
 * The library implements the depth-generation stage of arXiv 2201.11924
 * ("SimSense"): from a rectified left/right 8-bit IR pair
 * it computes
 *   census (CSCT)  ->  Hamming matching cost
 *   -> semi-global path aggregation, P1/P2, 4 or 8 paths
 *   -> winner-take-all + uniqueness test  -> quadratic sub-pixel
 *   -> left-right consistency check       -> depth = f*b/d
 * with the exact semantics listed in DESIGN.md §3 (readings c1-c18 of
 * SURVEY.md §8(c); SPEC.md S:288-356 gives the operation interfaces).
 * Rectification is the identity (born-rectified rig) and the median
 * filter is off (reading c15).
 *
 * Conventions shared by every entry point
 *   - Images are row-major [H][W] (batches [n][H][W], frames contiguous), no
 *     row padding.  Disparity delta(d) = min_disp + d, d in [0, num_disp),
 *     d = x_left - x_right >= 0 (reading c5).
 *   - Outputs are float32; INVALID = quiet NaN.
 *   - Device pointers are CUDA device (or managed) memory on the context's
 *     device; "host" entry points take host memory (pinned memory is fastest).
 *   - The caller owns every input/output buffer.  The context owns its scratch
 *     (census images, aggregated-cost volume, per-view disparity temporaries),
 *     allocated once in asd_create; no entry point allocates device memory.
 *   - Device entry points are asynchronous on the caller's stream
 *     (`cuda_stream` is a cudaStream_t; NULL = legacy default stream) and do
 *     not synchronise the host.  A context must be used by one host thread and
 *     one stream at a time; distinct contexts may run concurrently.
 *   - Return value: ASD_OK (0) or a negative ASD_E_* code.  Argument errors are
 *     detected synchronously before anything is enqueued.  Nothing throws
 *     across the ABI.  asd_last_error() gives a message for the last failure.
 */
#ifndef ASD_H_
#define ASD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASD_VERSION 3

#define ASD_OK              0
#define ASD_E_INVALID_ARG  (-1)  /* bad parameter, NULL required pointer, n out of range */
#define ASD_E_UNSUPPORTED  (-2)  /* valid per SPEC but outside this engine's bounds (see asd_params) */
#define ASD_E_CUDA         (-3)  /* CUDA launch / runtime failure; see asd_last_error */
#define ASD_E_OOM          (-4)  /* scratch allocation failed in asd_create */

/* Validity mask bits (debug output `mask`, `mask_r`). */
#define ASD_MASK_BORDER  1u  /* census window leaves the image (reading c4); right view: no defined d */
#define ASD_MASK_UNIQUE  2u  /* uniqueness test failed (reading c8) */
#define ASD_MASK_LR      4u  /* left-right check failed (readings c10-c12) */
#define ASD_MASK_NONPOS  8u  /* disparity <= 0, no depth (reading c14) */

/* Stereo configuration (SPEC S:257-260 StereoConfig).  Bounds enforced by
 * asd_create / asd_scratch_bytes:
 *   width  >= census_w, height >= census_h, width*height <= 2^26
 *   census_w, census_h odd, 1..15; nb = floor(census_w*census_h/2) in [1, 64]
 *       (SPEC allows up to 112 bits; nb > 64 -> ASD_E_UNSUPPORTED)
 *   min_disp >= 0; num_disp % 16 == 0 and 16 <= num_disp <= 256
 *   0 <= p1 <= p2 and nb + p2 <= 255  (each path's L_r <= C + P2 fits 8 bits;
 *       else ASD_E_UNSUPPORTED); with an SGBM block instead
 *       paths * (block_w*block_h*nb + p2) <= 65535 (S fits 16 bits)
 *   paths in {4, 8} (4 = horizontal + vertical, 8 adds the diagonals, reading c6)
 *   uniqueness: percent, < 0 disables the test; <= 100000
 *   lr_max_diff: px, < 0 disables the LR check; not NaN
 *   subpixel: 0 or 1
 *   focal_px, baseline_m: finite, > 0; depth = fb / disparity with
 *       fb = (float)((double)focal_px * (double)baseline_m)
 *   engine: ASD_ENGINE_AUTO / _D1 / _D3; D3 outside its envelope ->
 *       ASD_E_UNSUPPORTED.  Results are bit-identical across engines.
 *   block_w, block_h: SGBM block ("SGBM computes the cost by
 *       the hamming distance between the local regions of the two pixels";
 *       SPEC S:258; reading c19): odd, 1..15; 0 is read as 1.
 *       1 x 1 = plain SGM.  The cost becomes CB(x,y,d) = sum over the block
 *       of C(x+u, y+v, d), nb for block positions off the image.  Engine D3
 *       runs SGBM at num_disp = 128 (u16-partial sweeps on CB), D1 otherwise.
 *   median_ksize: 0, 3 or 5 ("median filtering"; SPEC S:342-347;
 *       reading c20): after the LR check, a pixel with no BORDER/UNIQUE/LR bit
 *       takes the lower median of dl over the valid k x k neighbours (itself
 *       included); the non-positive test and the depth use that value.
 *   lr_mode: right-view disparity for the LR check.  0 = R1 (reading c10,
 *       S:389): WTA on the re-indexed left aggregate S(x + delta, d).  1 = R2
 *       (reading c24): the right view runs its own SGM on
 *       C_R = hamming(cr(x), cl(x + delta)) (twice the aggregation work; both
 *       engines). */
/* Aggregation designs:
 *   ASD_ENGINE_D1  one warp-per-line kernel per path direction, u16 S volume
 *                  read-modify-written in HBM (any configuration above)
 *   ASD_ENGINE_D3  grouped sweeps: cluster kernels for the 3 downward and 3
 *                  upward paths (frames wider than one cluster span several,
 *                  joined through global memory), a warp-per-row kernel for
 *                  the 2 horizontal paths, a shared-memory window WTA; the cost
 *                  volume is never materialised.  Envelope: nb <= 32,
 *                  num_disp in {16,32,64,96,128,256}; 8-path with
 *                  3*(nb+p2) > 255 (u16 partials) and SGBM only at
 *                  num_disp = 128.  WTA keys widen to u32 automatically.
 *   ASD_ENGINE_AUTO D3 inside its envelope, else D1.                      */
#define ASD_ENGINE_AUTO 0
#define ASD_ENGINE_D1   1
#define ASD_ENGINE_D3   3

typedef struct asd_params {
    int32_t width, height;
    int32_t min_disp, num_disp;
    int32_t census_w, census_h;
    int32_t p1, p2;
    int32_t paths;
    int32_t uniqueness;
    float   lr_max_diff;
    int32_t subpixel;
    float   focal_px, baseline_m;
    int32_t engine;      /* ASD_ENGINE_* (0 = auto) */
    int32_t block_w, block_h;   /* SGBM block, 1 x 1 (or 0) = SGM */
    int32_t median_ksize;       /* median filter after the LR check: 0 (off), 3, 5 */
    int32_t lr_mode;            /* right view: 0 = R1 re-index S (default), 1 = R2 own SGM */
} asd_params;

/* Per-frame statistics; exact integers except depth_sum.
 *   checksum  = sum over pixels p (row-major index) of
 *               fmix32((p * 0x9E3779B1) ^ ((uint32)(dstar_l(p) + 1) << 8) ^ mask(p))  mod 2^32
 *               (fmix32 = murmur3 finaliser; dstar_l = raw left argmin index d*)
 *   valid     = number of pixels with mask == 0
 *   depth_sum = sum of valid depths (float32 atomics: order-dependent low bits) */
typedef struct asd_frame_stats {
    uint32_t checksum;
    uint32_t valid;
    float    depth_sum;
    uint32_t reserved;
} asd_frame_stats;

/* Stage outputs for parity testing (asd_depth_debug).  Every pointer is a
 * device pointer and may be NULL (not produced).
 *   census_l/r : [H][W] uint32 if nb <= 32 else uint64; 0 at census borders
 *   cost       : [H][W][D] uint8, C(x,y,d) (materialised only here)
 *   agg        : [H][W][D] uint16, S = sum_r L_r
 *   dstar_l/r  : [H][W] int16, raw argmin d (right view: -1 if no d defined)
 *   disp_l/r   : [H][W] float, dl / dr after sub-pixel, before masking
 *   mask       : [H][W] uint8, final left mask (ASD_MASK_* bits)
 *   mask_r     : [H][W] uint8, right-view mask (BORDER | UNIQUE)           */
typedef struct asd_debug_out {
    void*     census_l;
    void*     census_r;
    uint8_t*  cost;
    uint16_t* agg;
    int16_t*  dstar_l;
    int16_t*  dstar_r;
    float*    disp_l;
    float*    disp_r;
    uint8_t*  mask;
    uint8_t*  mask_r;
} asd_debug_out;

typedef struct asd_ctx asd_ctx;

/* Library version (ASD_VERSION). */
int asd_version(void);

/* Device scratch asd_create(p, ., max_batch, .) will allocate, in bytes;
 * 0 if the parameters are rejected. */
size_t asd_scratch_bytes(const asd_params* p, int max_batch);

/* Validate p, bind `device`, allocate scratch for up to `max_batch` frames in
 * flight (1..1024; asd_depth_batch processes larger n in chunks of max_batch).
 * On success *out owns the scratch; release it with asd_destroy. */
int asd_create(const asd_params* p, int device, int max_batch, asd_ctx** out);

/* Free the context and its scratch (synchronises the device first).  NULL ok. */
void asd_destroy(asd_ctx* ctx);

/* One frame: left/right u8 [H][W] -> out_disp, out_depth f32 [H][W] -- the
 * whole path of PAPER.md P:289 (census, Hamming cost, SGM, WTA + uniqueness,
 * sub-pixel, LR check, depth) with SPEC S:366-368's compute_depth semantics
 * (disparity NaN where any mask bit is set; depth NaN where the disparity is
 * invalid or <= 0).  Pointers: device memory, no alignment requirement.
 * Either output may be NULL (not written).  ASD_E_INVALID_ARG for a NULL
 * context or input. */
int asd_depth(asd_ctx* ctx, const uint8_t* left, const uint8_t* right,
              float* out_disp, float* out_depth, void* cuda_stream);

/* n frames (n >= 0), [n][H][W] each, frames contiguous -- asd_depth per frame
 * (P:289 stage list; datagen batches, BASELINE.json north_star), pipelined on
 * the D3 engine; stats ([n] asd_frame_stats) may be NULL.
 * Frames beyond max_batch run in chunks.  n = 0 enqueues nothing. */
int asd_depth_batch(asd_ctx* ctx, int n, const uint8_t* left, const uint8_t* right,
                    float* out_disp, float* out_depth, asd_frame_stats* stats,
                    void* cuda_stream);

/* End-to-end variant over HOST buffers: copies each chunk host->device,
 * computes, copies results device->host, overlapping the copies of one chunk
 * with the compute of the next.  Synchronous: returns after all results are in
 * host memory.  Outputs/stats may be NULL. */
int asd_depth_batch_host(asd_ctx* ctx, int n, const uint8_t* left_host, const uint8_t* right_host,
                         float* out_disp_host, float* out_depth_host,
                         asd_frame_stats* stats_host, void* cuda_stream);

/* One frame with every stage's output (see asd_debug_out: the census of P:289 /
 * S:291, the cost of S:300, S of S:309, the WTA maps of S:318-332, the LR mask
 * of S:336-341); out_disp/out_depth via asd_depth semantics may additionally
 * be requested.  For parity tests; not a fast path. */
int asd_depth_debug(asd_ctx* ctx, const uint8_t* left, const uint8_t* right,
                    const asd_debug_out* outs, float* out_disp, float* out_depth,
                    void* cuda_stream);

/* Number of kernel launches one asd_depth_batch call of n frames enqueues. */
int asd_launches_per_batch(const asd_ctx* ctx, int n);

/* The engine the context runs (ASD_ENGINE_D1 or ASD_ENGINE_D3). */
int asd_engine(const asd_ctx* ctx);

/* Frames the engine's widest kernel keeps resident at once on this device
 * (D3: thread-block clusters of the sweep kernels that fit; D1: 0 = any).
 * Choosing max_batch as a multiple of it avoids a partial last wave. */
int asd_frames_per_wave(const asd_ctx* ctx);

/* D3 pipeline: a batch runs as groups of `group` frames over
 * max_batch / group scratch slots; the cluster sweeps of one group overlap the
 * row/WTA/LR passes of the previous one on the SMs the clusters leave free.
 * Default: one wave (asd_frames_per_wave, capped at max_batch).  group must be
 * in [1, max_batch] -- and at most one wave when a frame spans several
 * clusters (their boundary columns wait on each other, so every cluster of a
 * group must be resident at once); asd_set_group synchronises the device
 * first.  Returns ASD_OK or ASD_E_INVALID_ARG / ASD_E_CUDA.  D1 ignores it. */
int asd_set_group(asd_ctx* ctx, int group);
int asd_group(const asd_ctx* ctx);

/* Human-readable description of the chosen kernel geometry (cluster size,
 * CTA shape, residency), NUL-terminated into buf[0..n).  Returns its length. */
int asd_plan_info(const asd_ctx* ctx, char* buf, int n);

/* ---- depth registration into the RGB frame ----
 * PAPER.md P:289 "an optional depth registration that aligns the depth map to
 * the RGB camera frame"; reading c21.
 * Pinhole cameras without distortion; pixel (x, y) is at image coordinate
 * (x, y).  A source pixel with finite depth z > 0 is unprojected with `ir`,
 * moved by P' = R P + t (R 3x3 row-major, t 3: host arrays, IR-camera to
 * RGB-camera coordinates, metres), reprojected with `rgb` to the target pixel
 * (floor(u + 0.5), floor(v + 0.5)); the z-buffer keeps the smallest Z'.
 * depth: device [n][ir.height][ir.width] f32 (NaN = invalid, e.g. the
 * asd_depth output); out: device [n][rgb.height][rgb.width] f32, NaN where no
 * sample lands.  Both owned by the caller; enqueued on cuda_stream (NULL =
 * default stream), no host synchronisation.  Returns ASD_OK,
 * ASD_E_INVALID_ARG (NULL pointer, n < 0, non-positive sizes or focal lengths,
 * non-finite R/t/intrinsics) or ASD_E_CUDA. */
typedef struct asd_camera {
    int32_t width, height;
    float   fx, fy, cx, cy;
} asd_camera;

int asd_register_depth(const asd_camera* ir, const asd_camera* rgb, const float* R, const float* t,
                       int n, const float* depth, float* out, void* cuda_stream);

/* ---- stereo rectification ----
 * PAPER.md P:289 "performs a stereo rectification to project the images onto
 * a common image plane"; reading c23.  Warps n
 * u8 images [n][height][width] (device) by one 3x3 homography Hm (host, 9
 * doubles, row-major) that maps OUTPUT pixel coordinates to INPUT coordinates,
 * bilinear sampling of the zero-padded input, round half up to u8; call once
 * per view with that view's homography.  in and out must not overlap.  A
 * born-rectified rig needs no call (identity).  Returns ASD_OK,
 * ASD_E_INVALID_ARG (NULL pointer, n < 0, sizes, non-finite or singular Hm)
 * or ASD_E_CUDA. */
int asd_rectify(const double* Hm, int n, int width, int height, const uint8_t* in, uint8_t* out,
                void* cuda_stream);

/* ---- sensor noise front end ----
 * I_noisy = gamma * I_clean + n with gamma ~ Gamma(k, theta)
 * (laser speckle) and n ~ N(mu, sigma^2) (thermal noise); D415 parameters
 * k = 3.98, theta = 0.254, mu = -0.231, sigma = 0.83.  Readings c17
 * (DN units, round half up, clamp to u8) and c22 (sampling, random streams,
 * noise scale) in DESIGN.md §3.  clean: device [n][height][width] f32 clean IR
 * intensities in DN units; out: device [n][height][width] u8 (the input of
 * asd_depth*).  Image i draws from the Philox4x32-10 stream keyed by seed with
 * counter (pixel, attempt, frame0 + i, view), so left (view 0) and right
 * (view 1) images of a frame and consecutive frames are independent and any
 * tiling of the work reproduces the same values.  Enqueued on cuda_stream.
 * Returns ASD_OK, ASD_E_INVALID_ARG (NULL pointer, n < 0, sizes, k/theta <= 0,
 * sigma < 0, non-finite parameters) or ASD_E_CUDA. */
typedef struct asd_noise {
    double k, theta;      /* gamma shape and scale */
    double mu, sigma;     /* additive Gaussian mean and standard deviation (DN) */
    double scale;         /* noise strength s: gamma' = k theta + s (gamma - k theta), n' = s n */
} asd_noise;

int asd_sensor_noise(const asd_noise* q, uint64_t seed, int n, int width, int height,
                     uint32_t frame0, uint32_t view, const float* clean, uint8_t* out, void* cuda_stream);

/* ---- live stage timing (CUDA events on the launching stream) ----
 * asd_profile_begin(ctx, max_launches) pre-creates events for up to
 * max_launches kernel launches; from then on every launch the context enqueues
 * is bracketed by an event pair on the launching stream (no host sync).
 * asd_profile_end synchronises on those events and fills `out` with, per
 * stage, the summed device time, the number of launches, the ALGORITHMIC
 * bytes those launches must move at minimum and, for the integer-bound D3
 * kernels, the algorithmic integer lane-ops (DESIGN.md §5 per-unit figures x
 * units processed), then stops profiling.  Launches beyond max_launches are
 * counted in `dropped` and not timed. */
#define ASD_STAGE_CENSUS 0   /* K1 census */
#define ASD_STAGE_DIR    1   /* D1: one SGM path direction per launch */
#define ASD_STAGE_WTA    2   /* K4 WTA / uniqueness / sub-pixel, both views (D1 and D3) */
#define ASD_STAGE_LR     3   /* K5 LR check + depth (+ stats) */
#define ASD_STAGE_DOWN   4   /* D3: downward sweep (3 paths, or 1 at 4-path) */
#define ASD_STAGE_UP     5   /* D3: upward sweep */
#define ASD_STAGE_ROW    6   /* D3: horizontal paths, S written over the partial */
#define ASD_STAGE_BLOCK  7   /* SGBM block cost volume (D1 with block > 1 x 1) */
#define ASD_STAGE_COUNT  8
typedef struct asd_stage_times {
    double ms[ASD_STAGE_COUNT];
    double alg_bytes[ASD_STAGE_COUNT];
    double alg_ops[ASD_STAGE_COUNT];     /* integer lane-ops, 0 if not ALU-modelled */
    int32_t launches[ASD_STAGE_COUNT];
    int32_t dropped;
    int32_t reserved;
} asd_stage_times;

int asd_profile_begin(asd_ctx* ctx, int max_launches);
int asd_profile_end(asd_ctx* ctx, asd_stage_times* out);

/* Per-launch timeline of the launches recorded since asd_profile_begin (call
 * it BEFORE asd_profile_end, which discards them): synchronises on the events
 * and writes, for up to max launches in enqueue order, the stage id and the
 * start/end time in ms relative to the first launch's start.  Host arrays of
 * max elements, owned by the caller.  Returns the number written, or a
 * negative ASD_E_* code. */
int asd_profile_timeline(asd_ctx* ctx, int max, int32_t* stage, float* t_start_ms, float* t_end_ms);

/* Static strings; never NULL. */
const char* asd_strerror(int code);
const char* asd_last_error(const asd_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ASD_H_ */
