/*
 * splatstream_b200.h -- C ABI of the B200 hot path of splatstream
 * (arXiv 2604.02851, reference package /root/reference/pkg).
 *
 * The reference has no FFI: its boundary is the Python API that
 * pkg/src/splatstream/server.py and client.py call.  These entry points are
 * what a ctypes/cffi binding of that API binds to; every function names the
 * reference interface it replaces.  Plain C types only: device pointers,
 * sizes, and POD parameter blocks.  No torch types cross this boundary.
 *
 * Ownership: the caller owns every device buffer passed in; the library owns
 * only the opaque ss_ctx (stream binding + a grow-only scratch arena).
 * Threading: one ss_ctx per host thread / stream; no global state.
 * Errors: every function returns SS_OK (0) or a negative code; the message
 * is in ss_last_error(ctx).  SS_ERR_INVALID maps to Python ValueError,
 * SS_ERR_PROTOCOL to splatstream.protocol.ProtocolError, SS_ERR_CUDA to
 * RuntimeError (ref optim.py:46-47, optim.py:357-361, protocol/delta.py:90-94).
 */
#ifndef SPLATSTREAM_B200_H
#define SPLATSTREAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_OK 0
#define SS_ERR_INVALID (-1)
#define SS_ERR_PROTOCOL (-2)
#define SS_ERR_CUDA (-3)
#define SS_ERR_CAPACITY (-4)

#define SS_ABI_VERSION 1

typedef struct ss_ctx ss_ctx;

/* Columnar Gaussian store on the device: the layout of ref model.py:233-245
 * (GaussianModel).  Rows [0, active_count) are trainable. */
typedef struct {
    float* means;            /* (count, 3)            */
    float* log_scales;       /* (count, 3)            */
    float* quaternions;      /* (count, 4)  w x y z   */
    float* logit_opacities;  /* (count,)              */
    float* sh_coeffs;        /* (count, 3, B), B = (sh_degree+1)^2, [:, :, 0] = DC */
    float* light_visibility; /* (count,)  in {0, 1}   */
    int32_t* object_ids;     /* (count,)              */
    int32_t count;
    int32_t active_count;
    int32_t sh_degree;       /* 0..3 */
    int32_t param_dtype;     /* 0: the float columns above are float32 (every entry point); 1: means,
                                log_scales, quaternions, logit_opacities, sh_coeffs, light_visibility are
                                float64 (the reference's float64 models) -- accepted by the fp64 blend
                                instantiation only (render / backward / prepare_splats with precision 1,
                                and ss_adam_step, which stores f32-rounded values as the reference does) */
} ss_model;

/* Pinhole camera: ref geometry.py:111-181 (CameraIntrinsics, Pose). */
typedef struct {
    double position[3];
    double rot_cw[9];        /* camera->world rotation, row-major (Pose.rotation()) */
    double fx, fy, cx, cy;
    double near_plane;
    int32_t width, height;
} ss_camera;

/* ref render.py:34-48 (LightState). */
typedef struct {
    double direction[3];     /* unit, from the light into the scene */
    double intensity[3];
    int32_t ambient_bands;   /* 0 = no ambient SH */
    int32_t _pad;
    double ambient[3 * 16];  /* (3, ambient_bands) row-major */
} ss_light;

/* Per-call render options: ref render.py:339-341 arguments. */
typedef struct {
    double background[3];
    const int64_t* subset;   /* device, ascending rows, or NULL = all rows */
    int32_t subset_count;
    int32_t extent_cutoff;   /* 1 = 3-sigma windows, 0 = every splat covers the image */
    int32_t precision;       /* 0 = fp32 blend (throughput); 1 = fp64 blend (verbatim parity) */
    int32_t deterministic;   /* backward: 1 = fixed-order per-(tile,splat) partials, 0 = atomics */
    void* gt_ready;          /* backward: cudaEvent_t the stream waits on right before the first read of
                                the ground truth (its upload may overlap the forward pass); NULL = none */
    uint32_t* tile_hint;     /* optional device (tiles,): per-tile walk lengths of an earlier call for the
                                same camera (0xffffffff = unknown); orders the forward's tiles longest-first
                                and is overwritten with this call's lengths.  NULL = list lengths */
    int64_t tile_hint_len;   /* entries in tile_hint (must equal the tile count, else it is ignored) */
    float* defer_g9;         /* backward, fp32 blend only: if set, the per-row screen-space gradients
                                (n_in x 9) go here and defer_rinv (n_in) receives each row's depth
                                rank (0xffffffff = culled); the chain rule is left to one
                                ss_chain_views call over all the step's views.  NULL = immediate */
    uint32_t* defer_rinv;
    uint32_t* tile_order;    /* optional device (tiles,): the backward stores its tile walk order here; it
                                equals the order the next forward derives from tile_hint, so a call with
                                tile_order_valid = 1 uses it instead of re-sorting (needs tile_hint) */
    int32_t tile_order_valid;
    int32_t _pad2;
    int64_t* bins_status;    /* backward: optional device int64[2].  Set, and once the context knows a pair
                                capacity (ss_pair_capacity; the first call sets it from its own count), the
                                binning reads nothing back to the host: [0] counts calls whose (tile, splat)
                                pairs exceeded the capacity (their results are void; ss_adam_step_ld with
                                skip_if = this buffer then leaves the model alone), [1] keeps the largest
                                pair count seen.  NULL = the pair count is read back (one host sync) */
} ss_render_opts;

/* The chain rule of a step's views in one pass over the rows (ref
 * optim.py:170-268 per view, summed over views in view order as the
 * per-view backward would): g9[v] / rinv[v] are the defer_g9 / defer_rinv
 * buffers of n_views ss_backward calls (same model, subset and n_in);
 * cams / lights / g9 / rinv are HOST arrays of n_views (<= 16) entries.
 * Adds into grad (the ss_backward layout) with the same per-element fp32
 * additions in the same order, reading the parameters and writing the
 * gradient once per step instead of once per view. */
int ss_chain_views(ss_ctx* ctx, const ss_model* m, const ss_camera* cams, const ss_light* lights, int32_t n_views,
                   const float* const* g9, const uint32_t* const* rinv, const int64_t* subset, int64_t n_in,
                   float* grad);

/* ss_chain_views over inputs j in [j0, j1) (row = subset[j], or j) into a
 * gradient layout of `ld` rows per group whose first row is row0 and which
 * covers `rows` rows (ss_chain_views: j0 = 0, j1 = n_in, row0 = 0,
 * rows = ld = active_count).  The view-sharded step runs it on
 * one GPU's row shard [row0, row0 + rows) with ld = the shard length, every
 * view of the step in view order, g9[v] / rinv[v] offset so that entry j is
 * row j's: per row the arithmetic and order are those of ss_chain_views, so
 * the sharded gradient is bit-identical to the single-GPU one. */
int ss_chain_views_range(ss_ctx* ctx, const ss_model* m, const ss_camera* cams, const ss_light* lights,
                         int32_t n_views, const float* const* g9, const uint32_t* const* rinv, const int64_t* subset,
                         int64_t j0, int64_t j1, int64_t row0, int64_t rows, float* grad, int64_t ld);

/* ss_chain_views_range with init = 1: the gradient layout's rows
 * [0, rows) need not be cleared beforehand -- every entry is written (zero
 * where no view contributes), saving the clear and the first read.  Needs
 * the whole row range and no subset (j0 = row0, j1 >= row0 + rows); init = 0
 * is ss_chain_views_range. */
int ss_chain_views_range_init(ss_ctx* ctx, const ss_model* m, const ss_camera* cams, const ss_light* lights,
                              int32_t n_views, const float* const* g9, const uint32_t* const* rinv,
                              const int64_t* subset, int64_t j0, int64_t j1, int64_t row0, int64_t rows, float* grad,
                              int64_t ld, int32_t init);

/* *out = ((x[0] + x[1]) + x[2]) + ... (device doubles): the per-view loss sum
 * in the reference's order (optim.py:366-367). */
int ss_sum_f64(ss_ctx* ctx, const double* x, int64_t n, double* out);

/* composite(): ref render.py:317-336 on prepared splats (device arrays, n
 * splats already in draw order = prep.order): fp64 front-to-back blend of the
 * given windows (x0, x1, y0, y1; ref render.py:293-301), centres, inverse
 * covariances (a, b, c) = (inv[0][0], inv[0][1], inv[1][1]), opacities and
 * colours.  img (H, W, 3) and T (H, W, may be NULL) are float64 device. */
int ss_composite(ss_ctx* ctx, int64_t n, const double* mu2d, const double* inv2d, const double* opacity,
                 const double* color, const int32_t* windows, int32_t width, int32_t height, const double* background,
                 double* img, double* T);

/* Host-readable summary of the last render/backward call. */
typedef struct {
    int64_t visible;         /* splats passing the near test */
    int64_t pairs;           /* (tile, splat) overlaps emitted */
    int64_t tiles;
} ss_render_stats;

/* Optimizer hyper-parameters: ref optim.py:271-293 (LearningRates, OptimizerState). */
typedef struct {
    double lr_means;         /* already multiplied by scene_extent (optim.py:345-347) */
    double lr_log_scales, lr_quaternions, lr_logit_opacities, lr_sh_dc, lr_sh_rest;
    double beta1, beta2, eps, ema_beta;
} ss_adam_hparams;

/* Device optimizer state, flat in the gradient layout (see ss_grad_layout). */
typedef struct {
    double* m;               /* a * (11 + 3B) */
    double* v;               /* a * (11 + 3B) */
    double* grad_ema;        /* (a,) */
    int64_t* age;            /* (a,) */
    int32_t step_count;      /* t before this step; the call uses t+1 */
    const int64_t* skip_if;  /* optional device int64: when non-zero at run time (a binning overflow of the
                                step, see ss_render_opts.bins_status) the update leaves the model, moments,
                                EMA and age untouched.  NULL = always update */
} ss_adam_state;

/* ---- context ------------------------------------------------------------ */
int ss_ctx_create(int device, ss_ctx** out);
void ss_ctx_destroy(ss_ctx* ctx);
const char* ss_last_error(const ss_ctx* ctx);
int ss_set_stream(ss_ctx* ctx, void* cuda_stream);   /* cudaStream_t */
/* Raise the pair capacity of sync-free binning to at least `cap` (grow-only)
 * and return it; cap == 0 only reads it (0 = not yet known); cap < 0 sets it
 * to -cap (tests: forces the overflow-and-re-run path). */
int64_t ss_pair_capacity(ss_ctx* ctx, int64_t cap);
/* Host synchronisations this context has issued so far (stream syncs,
 * read-backs, scratch-arena growth): the optimizer step's fp32 path issues
 * none once warmed up (tests/test_gpu_step.py). */
int64_t ss_host_syncs(const ss_ctx* ctx);
int ss_abi_version(void);
/* Flat gradient buffer layout for `a` active rows at SH degree d:
 * [means a*3 | log_scales a*3 | quaternions a*4 | logit_opacities a | sh_coeffs a*3*B]
 * (the Gradients dataclass of ref optim.py:50-77, flattened). Returns floats. */
int64_t ss_grad_layout(int64_t active_rows, int32_t sh_degree, int64_t offsets_out[5]);

/* ---- measurement --------------------------------------------------------- */
/* Per-kernel-class device time, measured with CUDA events on the ctx stream
 * around each launch group.  Classes: 0 preprocess, 1 depth sort, 2 binning
 * (count/scan/emit/ranges), 3 tile sort, 4 forward blend, 5 backward blend,
 * 6 chain rule, 7 Adam, 8 encoders.  While enabled, the forward blend also
 * counts T-gated (pixel, splat) evaluations (counters[0]); counters[1] is the
 * number of kernels this context launched. */
#define SS_KC_COUNT 9
int ss_set_timing(ss_ctx* ctx, int enable);
/* Synchronises; returns accumulated ms and launch-group counts per class
 * and the counters, then (reset != 0) clears them. */
int ss_get_timing(ss_ctx* ctx, double ms_out[SS_KC_COUNT], int64_t groups_out[SS_KC_COUNT],
                  uint64_t counters_out[4], int reset);
/* Measured FP32 FMA throughput of this device in TFLOP/s (roofline denominator). */
int ss_measure_fp32_peak(ss_ctx* ctx, double* tflops_out);

/* ---- renderer (ref render.py:226-347) ------------------------------------ */
/* render(): ref render.py:339.  image_out (H,W,3) and T_out (H,W) are float
 * for precision 0 and double for precision 1; T_out may be NULL. */
int ss_render(ss_ctx* ctx, const ss_model* model, const ss_camera* cam, const ss_light* light,
              const ss_render_opts* opts, void* image_out, void* T_out, ss_render_stats* stats_out);

/* prepare_splats(): ref render.py:226 -- host-inspectable per-splat view.
 * All outputs are device arrays sized by `capacity` rows (>= visible), in
 * model-row order; `order_out` holds the composite order (ref render.py:283).
 * Any output pointer may be NULL. */
typedef struct {
    int64_t* rows;           /* (M,) model row index           */
    double* depth;           /* (M,) camera-space z            */
    double* mu2d;            /* (M,2)                          */
    double* sigma2d;         /* (M,3) = [s00, s01, s11]        */
    double* radius;          /* (M,) inf when cutoff disabled  */
    int32_t* window;         /* (M,4) = [x0, x1, y0, y1)       */
    double* opacity;         /* (M,)                           */
    double* color;           /* (M,3) clamped                  */
    double* color_pre;       /* (M,3)                          */
    double* shade_s;         /* (M,) signed cosine             */
    int64_t* order;          /* (M,) composite order           */
    int64_t capacity;
} ss_prepared;
int ss_prepare_splats(ss_ctx* ctx, const ss_model* model, const ss_camera* cam, const ss_light* light,
                      const ss_render_opts* opts, ss_prepared* out, int64_t* visible_out);

/* The rest of the reference's PreparedSplats (ref render.py:200-223) for the
 * M prepared splats whose model rows are rows[0..M) (device int64, e.g. the
 * `rows` output of ss_prepare_splats), fp64, each output (device) optional:
 * camera-space mean, projection Jacobian, Sigma3d, W Sigma3d W^T, view
 * direction / distance, normal proxy and its axis, and the shading
 * intermediates of ref render.py:196 (Y, albedo_est, cos, vis; s is in
 * ss_prepared).  Computed by the same device functions as K1. */
/* Diagnostics builds (-DSS_BWD_STATS) only: utilisation counters of the
 * backward blend walk (see ss_raster.cu); SS_ERR_INVALID otherwise. */
int ss_debug_bwd_stats(ss_ctx* ctx, unsigned long long out[8], int reset);

typedef struct {
    double* mu_cam;      /* (M,3)   */
    double* J;           /* (M,2,3) */
    double* sigma3d;     /* (M,3,3) */
    double* cov_cam;     /* (M,3,3) */
    double* view_dir;    /* (M,3)   */
    double* view_dist;   /* (M,)    */
    double* n_hat;       /* (M,3)   */
    int64_t* n_axis;     /* (M,)    */
    double* Y;           /* (M,B)   */
    double* albedo_est;  /* (M,3)   */
    double* cos;         /* (M,)    */
    double* vis;         /* (M,)    */
} ss_prepared_extras;
int ss_prepare_extras(ss_ctx* ctx, const ss_model* model, const ss_camera* cam, const ss_light* light,
                      const int64_t* rows, int64_t M, ss_prepared_extras* out);

/* Tile-binning products for parity tests (sort keys / tile ranges,
 * SURVEY §8c): depth-ordered rows, per-tile [start, end) and the depth rank
 * of every sorted (tile, splat) pair. */
int ss_debug_bins(ss_ctx* ctx, const ss_model* model, const ss_camera* cam, const ss_render_opts* opts,
                  int64_t* order_rows_out, int64_t rows_cap, int64_t* tile_ranges_out, int64_t tiles_cap,
                  int64_t* pair_rank_out, int64_t pairs_cap, ss_render_stats* stats_out);

/* backward(): ref optim.py:113.  Accumulates (+=) this view's gradients of
 * the L1 loss over active rows into grad_accum (flat layout above, float32)
 * and the loss into *loss_accum (device double).  gt is (H,W,3) float32.
 * image_out (may be NULL) receives the forward image as in ss_render. */
int ss_backward(ss_ctx* ctx, const ss_model* model, const ss_camera* cam, const ss_light* light,
                const ss_render_opts* opts, const float* gt, float* grad_accum, double* loss_accum,
                void* image_out, ss_render_stats* stats_out);

/* The Adam part of step(): ref optim.py:374-406.  grad_sum holds the SUM of
 * per-view gradients; it is scaled by 1/n_views here.  Updates model rows
 * [0, active) in place, renormalises quaternions, advances EMA and age. */
int ss_adam_step(ss_ctx* ctx, ss_model* model, ss_adam_state* state, const float* grad_sum,
                 int32_t n_views, const ss_adam_hparams* hp);
/* ss_adam_step on a gradient / moment layout of `ld` >= active_count rows per
 * group (padding rows skipped).  The view-sharded step passes a row shard of
 * the model (pointers offset to the shard's first row, active_count = its
 * length, possibly 0) with the shard's moments; step_count advances even for
 * an empty shard. */
int ss_adam_step_ld(ss_ctx* ctx, ss_model* model, ss_adam_state* state, const float* grad_sum, int64_t ld,
                    int32_t n_views, const ss_adam_hparams* hp);
/* ss_adam_step_ld whose every updated parameter (and renormalised
 * quaternion) is also stored into n_peers (<= 15) other replicas of the same
 * rows: peer_rows[5 q + g] is peer q's base address of group g (means,
 * log_scales, quaternions, logit_opacities, sh_coeffs) at the first row of
 * `model` -- device memory of other GPUs mapped into this process (CUDA IPC;
 * NVLink / NVSwitch peer stores).  The view-sharded step's parameter
 * all-gather, fused into the update.  Float32 parameters only. */
int ss_adam_step_peers(ss_ctx* ctx, ss_model* model, ss_adam_state* state, const float* grad_sum, int64_t ld,
                       int32_t n_views, const ss_adam_hparams* hp, int32_t n_peers, float* const* peer_rows);

/* ---- encoders (ref protocol/) -------------------------------------------- */
/* encode_delta(): ref protocol/delta.py:72 with compression_id 0 (raw).
 * cur/base are (rows, dims) of float32 (in_dtype 0) or float64 (1); base is
 * required for MEANS/LOG_SCALES and new_base_out (float32) receives the
 * advanced baseline.  The payload is written to out (device) and its length
 * to *out_len (device uint64) -- no host synchronisation.  Use
 * ss_delta_bound() for the capacity. */
int ss_encode_delta(ss_ctx* ctx, int32_t attribute_id, const void* cur, int32_t in_dtype,
                    const void* base, float* new_base_out, int64_t rows, int32_t dims,
                    double gating_threshold, uint8_t* out, uint64_t out_cap, uint64_t* out_len);
uint64_t ss_delta_bound(int32_t attribute_id, int64_t rows, int32_t dims);

/* One server tick's deltas in one call (ref server.py:488-493 ->
 * protocol/delta.py:72): three kernel launches whatever the number of jobs,
 * no host synchronisation.  Inputs may be strided views: element (row, d)
 * of cur/base is read at  row*row_stride + (d / inner)*outer + d % inner + col0
 * (row_stride 0 = dims, inner 0 = dims), e.g. SH DC of an (N,3,B) array:
 * row_stride 3B, inner 1, outer B, col0 0.  new_base is dense (rows, dims). */
typedef struct {
    int32_t attribute_id;
    int32_t in_dtype;        /* 0 float32, 1 float64 */
    const void* cur;
    const void* base;        /* MEANS / LOG_SCALES */
    float* new_base;         /* may alias base when base is dense float32 */
    int64_t rows;
    int32_t dims;
    int32_t inner;
    int64_t row_stride;
    int32_t outer;
    int32_t col0;
    double gating_threshold;
    uint8_t* out;
    uint64_t out_cap;
    uint64_t* out_len;
} ss_delta_job;
int ss_encode_delta_batch(ss_ctx* ctx, const ss_delta_job* jobs, int32_t njobs);

/* encode_snapshot(): ref protocol/snapshot.py:47 with compression_id 0.
 * profile 0 = quantized, 1 = lossless.  base_means_out / base_log_scales_out
 * (float32, may be NULL) receive the decoded means / log scales -- the
 * server's baseline reset of ref server.py:481-484 without a re-decode. */
int ss_encode_snapshot(ss_ctx* ctx, const ss_model* model, int32_t profile_id, uint8_t* out,
                       uint64_t out_cap, uint64_t* out_len, float* base_means_out,
                       float* base_log_scales_out);
uint64_t ss_snapshot_bound(int64_t count, int32_t sh_degree, int32_t profile_id);

/* encode_light_visibility(): ref protocol/packets.py:73-76 ('<I' count + 1-bit pack). */
int ss_encode_light_visibility(ss_ctx* ctx, const float* vis, int64_t n, uint8_t* out, uint64_t out_cap,
                               uint64_t* out_len);

/* The compression stage (compression_id 1): host zlib level 6, byte-identical
 * to ref protocol/profiles.py:41-46.  Host buffers. */
int ss_host_zlib_compress(const uint8_t* src, uint64_t n, uint8_t* dst, uint64_t cap, uint64_t* out_len);
uint64_t ss_host_zlib_bound(uint64_t n);

/* Frame envelope CRC (ref protocol/framing.py:51-53, zlib.crc32 of header +
 * payload).  ss_crc32 writes zlib.crc32(data[:n]) of a
 * DEVICE buffer to the device word *crc_out, n = min(*len_dev, len) when
 * len_dev is given (a payload length left on the device by an encoder), else
 * len; async on the context's stream.  ss_crc32_combine is host arithmetic
 * (zlib crc32_combine): the CRC of A + B from crc32(A), crc32(B) and |B|. */
int ss_crc32(ss_ctx* ctx, const uint8_t* data, const uint64_t* len_dev, uint64_t len, uint32_t* crc_out);
uint32_t ss_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2);

/* ---- dynamics ------------------------------------------------------------ */
/* update_light_visibility(): ref render.py:350-368 with the orthographic
 * projection of ref geometry.py:267-271.  Writes model->light_visibility. */
typedef struct {
    double position[3];
    double rot_cw[9];
    double half_width, half_height;
    int32_t width, height;
} ss_ortho_camera;
int ss_update_light_visibility(ss_ctx* ctx, ss_model* model, const double* depth_map,
                               const ss_ortho_camera* cam, double bias);
/* As ss_update_light_visibility, and *changed (device int32, set by the
 * caller to 0) becomes 1 if any row's bit flipped -- the server's "send the
 * LightVisibility packet" test (ref server.py:406-409) without copying the
 * vector to the host. */
int ss_update_light_visibility_changed(ss_ctx* ctx, ss_model* model, const double* depth_map,
                                       const ss_ortho_camera* light_cam, double bias, int32_t* changed);

/* ObjectRegistry.apply_transform(): ref model.py:557-572.  Rewrites the rows
 * with object_ids == object_id from their local poses (device f64 arrays
 * (count,3) / (count,4)); q (wxyz, normalised by the call) and t are host. */
int ss_apply_object_transform(ss_ctx* ctx, ss_model* model, int32_t object_id, const double* local_means,
                              const double* local_rots, const double q[4], const double t[3]);
/* ObjectRegistry.refresh_locals(): ref model.py:539-555, for rows of one object. */
int ss_refresh_object_locals(ss_ctx* ctx, const ss_model* model, int32_t object_id, int32_t active_only,
                             double* local_means, double* local_rots, const double q[4], const double t[3]);
/* The same for the rows listed in `rows` (device, n_rows entries) that belong to
 * object_id (ref model.py:371-387 with an explicit row set). */
int ss_refresh_object_locals_rows(ss_ctx* ctx, const ss_model* model, int32_t object_id, const int64_t* rows,
                                  int64_t n_rows, double* local_means, double* local_rots, const double q[4],
                                  const double t[3]);

/* ---- client ingestion: the decode side of the codec ----
 * The host parses the header and decompresses (zlib) exactly like the
 * reference and checks every size it can know from the header; the device
 * checks what needs the block's bytes and reports it in a status word
 * (nothing is written to the replica when it is non-zero). */
enum {
    SS_INGEST_OK = 0,
    SS_INGEST_VARINT_TRUNCATED = 1,  /* ValueError("truncated varint"), quantize.py:85-90 */
    SS_INGEST_VARINT_TOO_LONG = 2,   /* ValueError("varint too long"), quantize.py:94-95 */
    SS_INGEST_INDEX_RANGE = 3,       /* ProtocolError("sparse delta index out of range"), delta.py:181-182 */
    SS_INGEST_CODES_TRUNCATED = 4    /* ProtocolError("delta codes truncated"), delta.py:58-60 */
};
typedef struct {
    int32_t code;            /* SS_INGEST_* */
    int32_t _pad;
    int64_t offset;          /* end of the varint run inside the block */
} ss_ingest_status;

/* One decoded delta block: ref protocol/delta.py:150-205 (decode_delta). */
typedef struct {
    int32_t attribute_id, mode, dims, bits;  /* mode 0 dense residual, 1 sparse residual, 2 dense absolute */
    int64_t count;           /* rows covered (the header's count) */
    int64_t k;               /* sparse: survivors (header) */
    double lo, hi;           /* residual: the header's f32 range; absolute: the attribute's fixed range */
    const uint8_t* block;    /* device: decompressed block */
    int64_t block_len;
    float* baseline;         /* residual: (count, dims) float32 baseline rows, advanced in place */
    float* target;           /* element (row, d) at target + row*row_stride + (d/inner)*outer + d%inner + col0 */
    int64_t row_stride;
    int32_t inner, outer, col0, _pad;
    ss_ingest_status* status;  /* device */
} ss_delta_apply;
/* Validate the block and decode: sparse survivor indices (k, device) and,
 * when values_out != NULL, the dequantised float64 values (rows x dims). */
int ss_decode_delta(ss_ctx* ctx, const ss_delta_apply* d, int64_t* indices_out, double* values_out);
/* advance_baseline + apply_delta (ref delta.py:259-303) after ss_decode_delta
 * on the same block: residual attributes advance baseline rows
 * f32(f64(base) + dequant) and copy baseline[:count] into the target;
 * absolute attributes store f32(dequant) into the target columns. */
int ss_apply_delta(ss_ctx* ctx, const ss_delta_apply* d, const int64_t* indices);

/* decode_snapshot: ref protocol/snapshot.py:85-168.  `model` holds
 * preallocated device arrays for count rows at sh_degree. */
typedef struct {
    ss_model model;
    int32_t profile_id, _pad;
    double aabb_lo[3], aabb_hi[3];  /* the header's f32 AABB */
    const uint8_t* block;           /* device: decompressed block */
    int64_t block_len;
    ss_ingest_status* status;       /* device */
} ss_snapshot_decode;
int ss_decode_snapshot(ss_ctx* ctx, const ss_snapshot_decode* d);

/* ---- pool maintenance ---- */
enum { SS_SELECT_FREEZE = 0, SS_SELECT_PRUNE = 1, SS_SELECT_PRECULL = 2 };
typedef struct {
    double position[3];
    double rot_cw[9];        /* camera->world rotation, row major (world_to_camera = (p - position) @ rot_cw) */
    double fx, fy, cx, cy, near_plane, far_plane;
    double tx, ty, nx, ny;   /* (W/2)/fx, (H/2)/fy, 1/sqrt(1+tx^2), 1/sqrt(1+ty^2)  (expansion.py:156-159) */
    int32_t width, height;
    const double* depth;     /* device (height, width) engine depth, or NULL */
} ss_pool_camera;
typedef struct {
    int32_t kind, n_cameras;
    int64_t n;                                      /* rows tested */
    const int64_t* age; const double* grad_ema;     /* freeze_policy: ref expansion.py:134-142 */
    int64_t age_threshold; double grad_threshold;
    const float* logits; double opacity_floor;      /* prune: ref expansion.py:184-197 */
    const int64_t* cells;                           /* precull: (n, 3) cell per row from the last rebuild */
    double origin[3], cell_size, margin;            /* ... cell geometry, margin = cell diagonal / 2 */
    const ss_pool_camera* cameras;                  /* ... host array of n_cameras (expansion.py:145-181) */
    const int64_t* row_ids;                         /* optional: report row_ids[i] instead of i */
} ss_select;
/* Rows passing the predicate, ascending, into `out` (device, n entries); the
 * count is returned on the host (the call synchronises). */
int ss_select_rows(ss_ctx* ctx, const ss_select* s, int64_t* out, int64_t* count_out);
/* dst row i = src row map[i] for every column (map[i] < 0: row (-1 - map[i]) of `fill`):
 * permute / remove_rows / client-side placeholder appends (ref model.py:134-165, 291-305). */
int ss_gather_rows(ss_ctx* ctx, const ss_model* src, ss_model* dst, const int64_t* map, int64_t n_out,
                   const ss_model* fill);
typedef struct {
    double origin[3];
    double cell_size;
} ss_grid_spec;
/* GridIndex.rebuild (ref model.py:418-426): per-row cells (n,3), and the cells in
 * first-appearance order with their member rows (ascending): cell_keys (C,3),
 * cell_lens (C,), cell_rows (n,) concatenated; the cell count C on the host. */
int ss_grid_rebuild(ss_ctx* ctx, const float* means, int64_t n, const ss_grid_spec* g, int64_t* cells,
                    int64_t* cell_keys, int64_t* cell_lens, int64_t* cell_rows, int64_t* n_cells);
/* Zigzag LEB128 of (perm[i] - i): the permutation block of an ordering
 * packet before its zlib stage (ref protocol/packets.py:153-158). */
int ss_zigzag_varints(ss_ctx* ctx, const int64_t* perm, int64_t n, uint8_t* out, uint64_t out_cap, uint64_t* len_out);

/* ---- scene engine ------------------------------------- */
/* The ray-cast game-engine stand-in: ref engine.py:88-205 (trace, shadow
 * rays, Lambertian shading, render_ground_truth, capture_input_buffers,
 * render_depth, render_ortho_depth) over the primitives of ref
 * scene.py:28-161.  One thread per pixel, float64 mirroring the reference's
 * numpy arithmetic.  Scene and camera are HOST structs; outputs are device
 * buffers, every one optional. */
#define SS_SHAPE_PLANE 0
#define SS_SHAPE_SPHERE 1
#define SS_SHAPE_BOX 2
typedef struct {
    int32_t shape;          /* SS_SHAPE_* */
    int32_t object_id;
    int32_t albedo_kind;    /* 0 solid, 1 checker (scene.py:152-158) */
    int32_t has_extent;     /* plane: finite rectangle */
    int32_t has_transform;  /* local -> world rigid transform applies */
    int32_t _pad;
    double a[3];            /* plane point | sphere centre | box centre */
    double b[3];            /* plane unit normal | box half extents */
    double radius;          /* sphere */
    double extent[2];       /* plane half sizes along u, v */
    double u[3], v[3];      /* plane tangents (scene.py:41-46, computed by the caller) */
    double color[3], color2[3];
    double scale;           /* checker cell size */
    double R[9];            /* local -> world rotation, row-major (quat_to_rotmat of the transform) */
    double t[3];            /* local -> world translation */
} ss_scene_object;

typedef struct {
    const ss_scene_object* objects;  /* host array, scene order */
    int32_t n_objects;
    int32_t _pad;
    double light_direction[3];       /* unit, from the light into the scene */
    double light_intensity[3];
    double ambient[3];
    double background[3];
} ss_scene;

typedef struct {
    int32_t kind;                    /* 0 pinhole (geometry.py:238), 1 orthographic (geometry.py:273), 2 rays */
    int32_t width, height;
    int32_t _pad;
    double position[3];
    double R[9];                     /* camera -> world rotation, row-major */
    double fx, fy, cx, cy;           /* pinhole */
    double half_width, half_height;  /* orthographic */
    double far;                      /* depth_or_far where a ray misses */
    double footprint_scale;          /* 2 tan(fov_y / 2) / height (capture buffers) */
    /* kind 2, explicit rays (engine.py:88 trace): width = ray count, height = 1;
     * device (n, 3) arrays, stride 3 per ray or 0 = one vector broadcast to all */
    const double* ray_origins;
    const double* ray_dirs;
    int32_t origin_stride, dir_stride;
} ss_engine_camera;

typedef struct {  /* (H, W[, 3]) row-major device buffers; NULL = not written */
    float* gt_f32;          /* render_ground_truth as float32 (the optimiser's ground truth) */
    double* gt_f64;         /* render_ground_truth */
    double* depth_or_far;   /* pinhole: render_depth; orthographic: render_ortho_depth */
    double* world_pos;      /* capture_input_buffers channels (engine.py:161-189) */
    uint8_t* valid;
    double* normal;
    double* albedo;
    double* shaded;
    int32_t* object_id;
    double* depth;
    double* footprint;
    uint8_t* lit;
    double* t;              /* trace: hit distance, inf where missed */
    int32_t* object_index;  /* trace: index into scene.objects, -1 where missed */
} ss_engine_out;

int ss_engine_render(ss_ctx* ctx, const ss_scene* scene, const ss_engine_camera* cam, const ss_engine_out* out);

/* Expansion inputs: ref engine.py:249-303 cull_input_samples and
 * expansion.py:39-64 init_gaussians.  Device buffers. */
typedef struct {  /* one input camera's capture buffers (H*W pixels, row-major) */
    const double* world_pos;   /* (pixels, 3) */
    const uint8_t* valid;
    const double* normal;      /* (pixels, 3) */
    const double* albedo;      /* (pixels, 3) */
    const int32_t* object_id;
    const double* footprint;
    const uint8_t* lit;
    double position[3];        /* the camera's pose.position */
    int64_t pixels;
} ss_cull_camera;

typedef struct {  /* SampleBatch (engine.py:54-78), device arrays of capacity rows */
    double* positions;         /* (n, 3) */
    double* normals;           /* (n, 3) */
    double* albedo;            /* (n, 3) */
    int32_t* object_ids;
    double* footprints;
    uint8_t* lit;
    int32_t* camera_indices;
} ss_sample_batch;

/* Pools the valid pixels of `cams` (HOST array, camera order), keeps per voxel
 * (side 2 x median footprint) the samples of the best-scoring camera, writes
 * them to `out` in pool order; *count_out (host) = kept samples, *side_out
 * (host, may be NULL) = voxel side.  Synchronises the stream. */
int ss_cull_input_samples(ss_ctx* ctx, const ss_cull_camera* cams, int32_t n_cams, const ss_sample_batch* out,
                          int64_t capacity, int64_t* count_out, double* side_out);
/* init_gaussians: rows [row0, row0 + n) of `model` from the first n samples
 * (isotropic log(max(footprint, 1e-6) / 2) scales, identity rotation, opacity
 * logit 0, SH DC = (albedo - 0.5) / C0, rest 0, visibility = lit). */
int ss_init_gaussians(ss_ctx* ctx, const ss_sample_batch* samples, int64_t n, const ss_model* model, int64_t row0);

#ifdef __cplusplus
}
#endif
#endif /* SPLATSTREAM_B200_H */
