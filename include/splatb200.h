/*
 * splatb200.h -- C ABI of libsplatb200.so, the sm_100a (B200) implementation of
 * the Gaussian-LIC online map-optimisation hot path.
 *
 * The reference (`splatmap`, /root/reference/pkg/src/splatmap) is a pure
 * Python/numba CPU package with no FFI; its "operator API" is the Python
 * functions re-exported by splatmap/__init__.py:6-32.  Each entry point below
 * replaces one of those functions (cited per entry); the Python package
 * paper_2404_06926_b200 binds them with ctypes and keeps the reference names,
 * signatures and exception types.  See INTEGRATION.md for the binding a
 * splatmap maintainer would add.
 *
 * Conventions
 *  - Every function returns SB_OK (0) or a negative SB_ERR_* code; the text of
 *    the last error on the calling thread is available from sb_last_error().
 *  - Array arguments are raw DEVICE pointers (row-major, the reference's
 *    layouts) plus element counts.  `stream` is a
 *    cudaStream_t passed as void*; every call is asynchronous on it unless
 *    stated otherwise.
 *  - The library never allocates caller-visible memory.  Scratch comes from
 *    the caller, sized by the *_workspace_bytes() queries.
 *  - dtype: SB_F32 (production) or SB_F64 (the reference's float64
 *    verification mode).  "real" below means float or double per dtype.
 *  - Only tile_size == 16 is supported (forward.py:35 DEFAULT_TILE_SIZE).
 *  - One map per stream; calls are not re-entrant on the same buffers.
 */
#ifndef SPLATB200_H
#define SPLATB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_OK 0
#define SB_ERR_INVALID (-1)   /* bad argument (shape, dtype, tile size): ValueError */
#define SB_ERR_CUDA (-2)      /* CUDA runtime error: RuntimeError */
#define SB_ERR_CAPACITY (-3)  /* caller buffer too small; required size returned */

#define SB_F32 0
#define SB_F64 1

#define SB_TILE 16

/* Pose (world->camera x_c = W x_w + t, scene.py:67-80) and intrinsics
 * (scene.py:51-64), in double exactly like the reference host objects. */
typedef struct {
    double W[9];
    double t[3];
    double fx, fy, cx, cy;
    int32_t width, height;
} sb_camera_t;

/* Optional per-row outputs of the projection, the SplatScreen fields the
 * binning/blend kernels do not need (projection.py:251-290).  Any pointer may
 * be NULL.  All rows are map-indexed (length n). */
typedef struct {
    void *cov2d;      /* real[n][2][2] dilated covariance */
    void *inv_cov2d;  /* real[n][2][2] conic */
    void *t_cam;      /* real[n][3] */
    void *t_clamped;  /* real[n][3] */
    uint8_t *clamped_x, *clamped_y;
    void *view_dir;   /* real[n][3] */
    void *basis;      /* real[n][16] */
    void *color_raw;  /* real[n][3] */
    void *mean2d;     /* real[n][2] */
    void *depth;      /* real[n] */
    void *color;      /* real[n][3] */
    void *opacity;    /* real[n] */
    void *radius_cut; /* real[n] */
    void *q_cut;      /* real[n] */
} sb_screen_extras_t;

/* Splat record: 12 reals per row, 16-byte aligned
 *   [mx, my, a, b | c, opacity, q_cut, radius | r, g, b, depth]
 * (a, b, c) = (inv00, inv01, inv11) of the conic. */
#define SB_RECORD_REALS 12

int32_t sb_version(void);
const char *sb_last_error(void);

/* a1: frustum_mask, scene.py:283-298. out[n] = 1 iff z > near and the
 * projection lies in the image padded by `margin`. */
int32_t sb_frustum_mask(int32_t dtype, int64_t n, const void *positions, const sb_camera_t *cam,
                        double near_, double margin, uint8_t *out, void *stream);

/* a1+a2: project_gaussians, projection.py:307-392, fused with the frustum
 * mask.  Map-indexed outputs: records[n][12], valid[n] (the reference's keep
 * set), depth_key[n] (float bits of depth, 0xFFFFFFFF when invalid) and
 * depth_val[n] (= row index) for the depth sort.  select (nullable) restricts
 * projection (mapper.py:204 include_sky=False).  frustum (nullable) receives
 * frustum_mask(margin) over all rows.  extras (nullable) receives the API
 * fields. */
int32_t sb_preprocess_fwd(int32_t dtype, int64_t n, const void *positions, const void *log_scales,
                          const void *rotations, const void *opacity_logits,
                          const void *sh_coeffs, const uint8_t *select, const sb_camera_t *cam,
                          double near_, double dilation, double margin, void *records,
                          uint8_t *valid, void *depth_key, uint32_t *depth_val,
                          uint8_t *frustum, const sb_screen_extras_t *extras,
                          const float *coarse_depth_limit, void *stream);

/* sb_preprocess_fwd's coarse_depth_limit (nullable): the maxima over 4x4-tile
 * blocks (ceil(tiles_x/4) x ceil(tiles_y/4), row-major) of the per-tile depth
 * limits the next sb_bin will apply (sb_blend_fwd produces both).  A row
 * whose depth is behind the maximum over the blocks its cutoff box covers
 * can have no pair in those lists: it is marked invalid (no record). */

/* Pack caller-provided SplatScreen fields (compact rows) into records, for
 * screens that did not come from sb_preprocess_fwd.  valid[m] = 1. */
int32_t sb_pack_records(int32_t dtype, int64_t m, const void *mean2d, const void *inv_cov2d,
                        const void *opacity, const void *q_cut, const void *radius_cut,
                        const void *color, const void *depth, void *records, uint8_t *valid,
                        void *depth_key, uint32_t *depth_val, void *stream);

/* a3: bin_and_sort, forward.py:184-255 with _cull_pairs forward.py:112-159.
 * Input: m rows of records/valid/depth_key/depth_val (depth_* are consumed as
 * scratch).  Output: pair_gaussian[P] (row ids) and pair_tile[P] (nullable:
 * not written when NULL) in (tile, depth, row) order, offsets[n_tiles+1] CSR.
 * At most 32768 tiles.
 * d_status == NULL: the call synchronises `stream` once to read P into
 * *n_pairs; if P > pair_capacity nothing is emitted and SB_ERR_CAPACITY is
 * returned with *n_pairs = P.
 * d_status != NULL (int64[2], device): no host synchronisation (CUDA-graph
 * capturable).  d_status[0] = P, d_status[1] = 1 on overflow, in which case
 * nothing is emitted and every tile range is empty.  *n_pairs is set to -1.
 * tile_depth_limit (nullable, device float[n_tiles], needs d_status): a tile
 * keeps only its pairs with depth <= tile_depth_limit[t] (a prefix of its
 * depth-ordered list; +inf keeps all) -- the mapping engine's truncation of
 * lists behind the depth where the tile saturated (sb_blend_fwd produces the
 * limits and validates them).
 * sort_capacity (0 = all m rows): when 0 < sort_capacity < m (needs d_status),
 * only the rows with a valid depth key -- valid rows whose cutoff box meets
 * the image, sb_preprocess_fwd marks the others -- are gathered (in row
 * order) and sorted, in sort_capacity slots; more such rows than that sets
 * d_status[1] (the step is invalid; re-run with a larger bound or 0).  The
 * pair order is exactly the unbounded one.  For maps much larger than the
 * visible set (a view of a growing map).
 * halt (nullable, device int64[1], needs d_status): non-zero marks the call's
 * iteration invalid too (d_status[1] = 1): the engine's flag for the
 * iterations queued behind an invalid one. */
size_t sb_bin_workspace_bytes(int64_t m, int64_t pair_capacity, int32_t width, int32_t height);
int32_t sb_bin(int32_t dtype, int64_t m, const void *records, const uint8_t *valid,
               void *depth_key, uint32_t *depth_val, int32_t width, int32_t height,
               int32_t tile_size, int32_t cull, int64_t pair_capacity, int32_t *pair_gaussian,
               int32_t *pair_tile, int32_t *offsets, int64_t *n_pairs, void *workspace,
               size_t workspace_bytes, int64_t *d_status, const float *tile_depth_limit,
               int64_t sort_capacity, const int64_t *halt, void *stream);

/* a4: render/_composite_tiles, forward.py:261-368, + exposure epilogue
 * (loss.py:31-36) when exposure (device real[12], the 3x4 [M|b]) and out_y
 * are non-NULL.  out_last[H*W] records, per pixel, 1 + the tile-list position
 * of its last contributor (0 if none): the backward replays only that prefix.
 * out_opacity, out_y, out_last may be NULL.
 * tile_depth_limit (nullable, float[n_tiles], in/out): a finite entry means
 * this call's list for the tile was limited by sb_bin; if not every pixel of
 * such a tile terminated, d_status[1] is set to 1 (result invalid, re-run
 * with full lists).  On return each entry is the next iteration's limit:
 * 1.25 x the depth of the tile's deepest last contributor + 1e-3 if every
 * pixel terminated, else +inf.  coarse_depth_limit (nullable, caller-zeroed)
 * receives the maxima of the new limits over 4x4-tile blocks (see
 * sb_preprocess_fwd).  * tile_sched (nullable, int32[3 n_tiles], caller-owned, zero-initialised
 * once): heavy-first CTA order.  The call orders its tiles by the replay
 * lengths in tile_sched[n_tiles..2 n_tiles) (left by the previous call with
 * this buffer), then records this frame's there; sb_blend_bwd with the same
 * buffer orders the backward by them.  Results do not depend on the order.
 * halt (nullable, device int64[1], needs d_status): set to 1 when the
 * iteration is invalid (d_status[1] on entry, or a failed depth limit).
 * fast_exp: 0 = alpha from the correctly rounded exp (bit-identical to the
 * reference's float pipeline on the same inputs: the render API); 1 = the
 * hardware exp (2 ulp; float only) -- the mapping step, whose outputs feed
 * tolerance-checked losses and gradients, and whose backward replays alpha
 * with the same exp. */
int32_t sb_blend_fwd(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                     const int32_t *offsets, int32_t width, int32_t height, int32_t tile_size,
                     int32_t early_termination, double term_threshold, const void *exposure,
                     void *out_color, void *out_depth, void *out_transmittance, void *out_opacity,
                     int32_t *out_n_contrib, int32_t *out_last, void *out_y,
                     float *tile_depth_limit, int64_t *d_status, float *coarse_depth_limit,
                     int32_t *tile_sched, int64_t *halt, int32_t fast_exp, void *stream);

/* a5 (+a9 tail): photometric_loss, loss.py:143-177: fused L1 + D-SSIM on
 * Y = exposure(C).  y may be NULL (computed from rendered + exposure).
 * Writes d_rendered[H][W][3], d_exposure (double[12], device), parts (double[4]
 * device: loss, l1, dssim, ssim).  Requires H, W >= 6. */
size_t sb_loss_workspace_bytes(int32_t width, int32_t height);
int32_t sb_loss_fused(int32_t dtype, int32_t width, int32_t height, const void *rendered,
                      const void *y, const void *ground_truth, const void *exposure, double lam,
                      void *d_rendered, double *d_exposure, double *parts, void *workspace,
                      size_t workspace_bytes, void *stream);

/* a6: _backward_tiles, backward.py:91-213.  Screen-space adjoints per row,
 * ACCUMULATED (atomics) into caller-zeroed d_mean2d[m][2], d_conic[m][3]
 * (aa, ab, cc), d_opacity[m], d_color[m][3].  last (nullable) is out_last of
 * sb_blend_fwd; NULL replays every pair of the tile. */
int32_t sb_blend_bwd(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                     const int32_t *offsets, int32_t width, int32_t height, int32_t tile_size,
                     int32_t early_termination, double term_threshold, const void *d_color_image,
                     const void *c_final, const int32_t *last, void *d_mean2d, void *d_conic,
                     void *d_opacity, void *d_color, const int32_t *tile_sched, void *stream);

/* a6, deterministic (the engine's path): backward.py:91-213 with the
 * reference's merge order -- every row's per-tile adjoint sums are added in
 * ascending tile order (backward.py:92-98), no float atomics, so the result
 * is bitwise reproducible run to run and independent of the tile schedule
 * and of depth-limited vs full lists.  The pairs must come from an sb_bin
 * call whose workspace (bin_workspace) is still intact and whose m,
 * pair_capacity, image size and sort_capacity are passed here: its per-pair
 * rank-major index map makes each row's pairs contiguous.  d_mean2d,
 * d_conic, d_opacity, d_color are STORED (not accumulated) for every row
 * with a kept pair; the caller zeroes the other rows.  workspace:
 * sb_blend_bwd_workspace_bytes (one 12-real partial record per pair + the
 * gather's queue of long rows). */
size_t sb_blend_bwd_workspace_bytes(int32_t dtype, int64_t pair_capacity, int32_t width,
                                    int32_t height);
int32_t sb_blend_bwd_det(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                         const int32_t *offsets, int32_t width, int32_t height, int32_t tile_size,
                         int32_t early_termination, double term_threshold,
                         const void *d_color_image, const void *c_final, const int32_t *last,
                         void *d_mean2d, void *d_conic, void *d_opacity, void *d_color,
                         const int32_t *tile_sched, int64_t m, int64_t pair_capacity,
                         int64_t sort_capacity, const void *bin_workspace, void *workspace,
                         size_t workspace_bytes, void *stream);
/* sb_blend_bwd_det in its two launches (the engine's form, so each can be
 * timed): the backward blend writing the partial records and replayed flags
 * (into workspace and bin_workspace's flag map), then the per-row ordered
 * reduction into the adjoints.  Same arguments as sb_blend_bwd_det. */
int32_t sb_blend_bwd_partials(int32_t dtype, const void *records, const int32_t *pair_gaussian,
                              const int32_t *offsets, int32_t width, int32_t height,
                              int32_t tile_size, int32_t early_termination,
                              double term_threshold, const void *d_color_image,
                              const void *c_final, const int32_t *last,
                              const int32_t *tile_sched, int64_t m, int64_t pair_capacity,
                              void *bin_workspace, void *workspace, size_t workspace_bytes,
                              void *stream);
/* sb_gather_adjoints writes the adjoints of the rows with replayed pairs
 * only; rows without keep whatever the buffers held.  reached_rows
 * (nullable, uint8[n], all zero on entry): set to 1 for every row whose
 * merged adjoints are not all zero -- the rows a chain rule must visit (the
 * others have an exactly zero gradient).  Given to sb_chain_adam_rows /
 * sb_chain_accumulate (which read and clear it), no unflagged row's
 * adjoints are read, so the adjoint buffers need no zeroing (the
 * deterministic engine and keyframe batch skip the memset). */
int32_t sb_gather_adjoints(int32_t dtype, int64_t m, int64_t pair_capacity, int32_t width,
                           int32_t height, int64_t sort_capacity, const void *bin_workspace,
                           void *workspace, size_t workspace_bytes, void *d_mean2d,
                           void *d_conic, void *d_opacity, void *d_color, uint8_t *reached_rows,
                           void *stream);

/* a7: _chain_to_parameters, backward.py:415-500, from explicit SplatScreen
 * fields (compact rows, src[m] -> map row).  Gradients ACCUMULATE
 * (np.add.at semantics) into caller-zeroed map-indexed buffers. */
typedef struct {
    const void *inv_cov2d, *t_cam, *t_clamped, *view_dir, *basis, *color_raw, *opacity;
    const uint8_t *clamped_x, *clamped_y;
} sb_chain_screen_t;
int32_t sb_preprocess_bwd(int32_t dtype, int64_t m, const int64_t *src, const void *positions,
                          const void *log_scales, const void *rotations, const void *sh_coeffs,
                          const sb_chain_screen_t *screen, const void *d_mean2d,
                          const void *d_conic, const void *d_opacity, const void *d_color,
                          const sb_camera_t *cam, void *g_position, void *g_log_scale,
                          void *g_rotation, void *g_opacity_logit, void *g_sh, void *stream);

/* a7 for map-indexed rows of sb_preprocess_fwd (valid[n]): recomputes the
 * screen quantities from the parameters instead of reading them.
 * accumulate = 0: writes all n gradient rows (invalid rows get zeros).
 * accumulate = 1: adds this view's gradient into the buffers (keyframe-batch
 * sum); rows no pixel reached are left untouched. */
int32_t sb_preprocess_bwd_rows(int32_t dtype, int64_t n, const uint8_t *valid,
                               const void *positions, const void *log_scales,
                               const void *rotations, const void *opacity_logits,
                               const void *sh_coeffs, const sb_camera_t *cam, double dilation,
                               const void *d_mean2d, const void *d_conic, const void *d_opacity,
                               const void *d_color, void *g_position, void *g_log_scale,
                               void *g_rotation, void *g_opacity_logit, void *g_sh,
                               int32_t accumulate, void *stream);

/* a8: adam_step, adam.py:76-122.  Five parameter groups in GROUPS order
 * (position[3], log_scale[3], rotation[4], opacity_logit[1], sh[16][3]),
 * each with param/grad/m/v pointers.  steps: int64[n] per-Gaussian counters.
 * active (nullable) = uint8 mask over rows; NULL = dense.  lrs = {position,
 * log_scale, rotation, opacity_logit, sh0, sh_rest}. */
typedef struct {
    void *param[5];
    const void *grad[5];
    void *m[5];
    void *v[5];
} sb_adam_groups_t;
int32_t sb_sparse_adam(int32_t dtype, int64_t n, const sb_adam_groups_t *groups, int64_t *steps,
                       const uint8_t *active, const double *lrs, void *stream);

/* a7+a8 for the mapping step: chain rule from the screen adjoints into the
 * Adam update of the frustum-active rows (same numerics as
 * sb_preprocess_bwd_rows followed by sb_sparse_adam(active = frustum)).
 * mode 0 (default): a per-row chain kernel writes gradients only for active
 * rows some pixel reached, then a flat coalesced Adam kernel updates every
 * active element (workspace from sb_chain_adam_workspace_bytes).  mode 1: one
 * fused kernel staging rows in shared memory (no workspace).
 * d_status (nullable, from sb_bin): the update is skipped when d_status[1]
 * reports a pair-capacity overflow (the caller re-runs the step).
 * touched (nullable, mode 0 only; uint8[n] the caller keeps across steps):
 * the touched-row skip.  touched[r] = 0 promises row r's moments are all
 * exactly +0; an active row with touched 0 and no gradient this step then has
 * an identity update (p, m, v unchanged bitwise), so only its step counter
 * moves and its 1668 B of element traffic are skipped.  A row with a gradient
 * sets touched[r] = 1.  Results are bit-identical to touched = NULL.  Moments
 * written by anything else (a checkpoint load, a gather) need touched
 * recomputed (or set to 1).
 * reached_rows (nullable, mode 0): the reached rows as sb_gather_adjoints
 * flagged them -- the reached test reads (and clears) that byte instead of
 * the row's 36 B of adjoints, so no unflagged row's adjoints are read. */
size_t sb_chain_adam_workspace_bytes(int32_t dtype, int64_t n);
int32_t sb_chain_adam_rows(int32_t dtype, int64_t n, const uint8_t *valid,
                           const uint8_t *active, const sb_camera_t *cam, double dilation,
                           const void *d_mean2d, const void *d_conic, const void *d_opacity,
                           const void *d_color, const sb_adam_groups_t *groups, int64_t *steps,
                           uint8_t *touched, uint8_t *reached_rows, const double *lrs,
                           void *workspace,
                           size_t workspace_bytes, int32_t mode, const int64_t *d_status,
                           void *stream);

/* a8, flat: the same update as sb_sparse_adam (bit-identical), as a per-row
 * bookkeeping kernel (steps, bias corrections into the workspace) and a
 * coalesced 16-byte pass over every group's elements.  active is required.
 * grad_rows (nullable; NULL = active): the active rows whose gradient is
 * read -- every other active row takes an exactly zero gradient (adam.py's
 * semantics for a row no pixel reached), so its gradient memory may hold
 * anything (the keyframe batch passes its reached-row mask and never zeroes
 * the gradient buffer).  touched (nullable): the touched-row skip of
 * sb_chain_adam_rows, a row "having a gradient" meaning grad_rows[r] (or
 * active[r] when grad_rows is NULL).  d_status (nullable): no update at all
 * when d_status[1] != 0. */
size_t sb_sparse_adam_workspace_bytes(int32_t dtype, int64_t n);
int32_t sb_sparse_adam_flat(int32_t dtype, int64_t n, const sb_adam_groups_t *groups,
                            int64_t *steps, const uint8_t *active, const uint8_t *grad_rows,
                            uint8_t *touched, const double *lrs, void *workspace,
                            size_t workspace_bytes, const int64_t *d_status, void *stream);

/* a7, keyframe-batch accumulation: the same arithmetic as
 * sb_preprocess_bwd_rows(accumulate = 1) -- g += this view's gradient for
 * valid rows some pixel reached -- over a compacted list of those rows.
 * reached (nullable, uint8[n]): set to 1 for every reached row (the caller
 * zeroes it once per batch; the packed exchange sends only those rows).
 * first_touch (needs reached): a row not yet marked in reached is STORED
 * (g = this view's gradient), later views add -- so g needs no zeroing; rows
 * no view reached keep whatever g held (pass reached as sb_sparse_adam_flat's
 * grad_rows).  reached_rows (nullable, uint8[n]): this view's reached rows
 * as sb_gather_adjoints flagged them -- the scan reads (and clears) that
 * byte instead of the row's 36 B of adjoints, and no unflagged row's
 * adjoints are read (they need no zeroing). */
size_t sb_chain_accumulate_workspace_bytes(int32_t dtype, int64_t n);
int32_t sb_chain_accumulate(int32_t dtype, int64_t n, const uint8_t *valid,
                            const void *positions, const void *log_scales, const void *rotations,
                            const void *opacity_logits, const void *sh_coeffs,
                            const sb_camera_t *cam, double dilation, const void *d_mean2d,
                            const void *d_conic, const void *d_opacity, const void *d_color,
                            void *g_position, void *g_log_scale, void *g_rotation,
                            void *g_opacity_logit, void *g_sh, uint8_t *reached,
                            int32_t first_touch, uint8_t *reached_rows, void *workspace,
                            size_t workspace_bytes, void *stream);

/* a9: ScalarAdam.step, adam.py:125-140, on the device in float64.
 * state = double[12 m, 12 v, 1 t]; exposure = double[12] updated in place;
 * exposure_real (nullable) receives the updated matrix cast to real.
 * d_status (nullable, from sb_bin): no update when d_status[1] != 0. */
int32_t sb_exposure_adam(int32_t dtype, double *exposure, void *exposure_real,
                         const double *d_exposure, double *state, double lr,
                         const int64_t *d_status, void *stream);

/* apply_exposure, loss.py:31-36: out[npx][3] = C M^T + b (exposure real[12]). */
int32_t sb_apply_exposure(int32_t dtype, int64_t npx, const void *color, const void *exposure,
                          void *out, void *stream);

/* quantize_8bit, metrics.py:12-13: dst[i] = round_half_even(clip(src[i], 0, 1)
 * * 255) computed in double (numpy's arithmetic on the promoted image). */
int32_t sb_quantize8(int32_t dtype, int64_t n, const void *src, uint8_t *dst, void *stream);

/* psnr_8bit, metrics.py:16-27, of clip(exposure(C), 0, 1) against an 8-bit
 * quantised target: ACCUMULATES the integer squared error into *sse (device,
 * caller-zeroed); PSNR = 10 log10(255^2 / (sse / (3 npx))), capped at 99. */
int32_t sb_psnr8_sse(int32_t dtype, int64_t npx, const void *color, const void *exposure,
                     const uint8_t *gt8, unsigned long long *sse, void *stream);

/* Packed gradient exchange of the keyframe batch step (no reference
 * counterpart: the reference has no multi-GPU path; SURVEY.md §8(e),
 * paper_2404_06926_b200/batch.py PackedBatchStep).  flat is the group-major
 * map-layout gradient of n_pad rows (59 reals per row: positions 3,
 * log_scales 3, rotations 4, opacity 1, sh 48); packed is row-major [k, 59];
 * pos[k] (device int64) are the rows, < n_pad, repeats allowed (a repeated
 * row must carry equal values when unpacked).  rows_held (nullable,
 * uint8[n_pad]): rows not marked there pack as zeros (a first-touch gradient
 * from sb_chain_accumulate is valid on this rank's reached rows only). */
int32_t sb_pack_rows(int32_t dtype, int64_t n_pad, const void *flat, const int64_t *pos,
                     int64_t k, void *packed, const uint8_t *rows_held, void *stream);
int32_t sb_unpack_rows(int32_t dtype, int64_t n_pad, void *flat, const int64_t *pos,
                       int64_t k, const void *packed, void *stream);

/* cudaMemsetAsync on the caller's stream (zeroing accumulators). */
int32_t sb_memset_async(void *ptr, int32_t value, size_t bytes, void *stream);

/* map growth (mapper.py:252-281): for k points (double xyz), flag those in
 * front of the camera whose nearest pixel floor(u+0.5) lies inside the image
 * and whose rendered opacity is < mask_threshold.  out_select[k] in {0,1}. */
int32_t sb_expand_select(int64_t k, const double *points, const sb_camera_t *cam, double near_,
                         int32_t dtype, const void *opacity_image, double mask_threshold,
                         uint8_t *out_select, void *stream);

/* Engine support (no reference counterpart): per-keyframe tile depth limits
 * (float[count]: tile limits then the coarse grid; nullable) stay usable while
 * the map was updated at most once since the key's last use: *clock (device
 * int64, map-update counter) is first advanced by bump; if *clock - *stamp > 1
 * (or stamp is NULL) the limits are reset to +inf (full lists); then
 * *stamp = *clock.  One tiny launch, decided on the device (graph-safe). */
int32_t sb_depth_limits_gate(float *limits, int64_t count, int64_t *clock, int64_t *stamp,
                             int32_t bump, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLATB200_H */
