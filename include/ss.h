/*
 * ss.h -- C ABI of libss.so, the sm_100a (B200) Speedy-Splat forward hot path.
 *
 * One view ("frame") of a 3D Gaussian Splatting scene is rendered by four calls, in
 * order, on one CUDA stream, followed optionally by the pruning-score call:
 *
 *   ss_preprocess  projection + tile count            PAPER.md Sec. 3.2.1
 *   ss_bin         key allocation + key emission       InclusiveSum / duplicateWithKeys
 *   ss_sort        sort by (tile, depth) + tile ranges RadixSort / identifyTileRanges
 *   ss_render      per-tile front-to-back blending     Sec. 3.2.3, Eqs. 5-7
 *   ss_prune_score efficient pruning score, +=         Sec. 4.2.1, Eqs. 20-21
 *
 * Mapping onto SURVEY.md §8(b)'s proposed signatures (same five calls, same paper steps; one
 * deviation, stated here and in DESIGN.md §1):
 *   - ss_preprocess: as proposed (a1 + a2's counts; P, the total, stays on the device).
 *   - ss_bin + ss_sort: the proposal materialises the paper's unsorted 64-bit keys / values
 *     (ss_bin, with capacity + overflow flag) and sorts them in place (ss_sort).  Here the
 *     visible Gaussians are depth-sorted once and the per-tile lists are a stable two-level
 *     partition of that order, so no unsorted key array ever exists: every pair
 *     is written once, at its sorted position (sorted_value), and the key is implied by its
 *     tile (ranges) and depth (depth_key).  The result equals the paper's stable sort of the
 *     keys emitted in Gaussian-index order; ss_sorted_keys materialises that
 *     64-bit key array on demand.  ss_bin ends with the tile ranges (a5) because the
 *     per-tile counts are known before the pairs are written; capacity and the overflow flag
 *     live in the frame workspace (ss_frame.capacity, ss_layout.overflow / overflow_count).
 *   - ss_render, ss_prune_score: as proposed; the intermediates are taken from the frame.
 *   - ss_workspace_size(which, ...): present, over the two workspace kinds (frame, prune step).
 *
 * Beyond the forward path: the prune step (ss_prune_select,
 * ss_compact_scene; Sec. 4.2), the backward (ss_render_backward, ss_preprocess_backward[_assign];
 * P:404) and the optimisation step of pruning-in-the-loop training (ss_l1_loss_grad,
 * ss_adam_init, ss_adam_step[_flagged]; Eq. 2).
 *
 * The tile test of ss_preprocess / ss_bin is selected by ss_bin_mode: the 3D-GS 3-sigma
 * square (Eq. 8), SnugBox (Sec. 4.1.1, Eqs. 15-16) or AccuTile
 * (Sec. 4.1.2, Algorithm 1).
 *
 * Conventions (DESIGN.md §2-§3 states every reading of the paper behind them):
 *   - Every pointer is a DEVICE pointer unless marked (host).  Device buffers are owned by
 *     the caller; libss never allocates or frees device memory and keeps no per-frame state
 *     (it caches the device's SM count and raises kernels' shared-memory limits once).  All calls enqueue
 *     work on `stream` (a cudaStream_t passed as void*, NULL = legacy default stream) and
 *     return without synchronising.  Calls on different streams with disjoint frame
 *     workspaces may run concurrently.
 *   - Per-frame intermediates live in ONE caller-allocated device workspace described by
 *     ss_frame (size from ss_frame_workspace_size, sub-buffer offsets from ss_frame_layout).
 *     Sizes that only the device knows (visible count, pair count P) stay on the device;
 *     no call reads them back to the host.
 *   - Errors: host-side validation happens before any launch and returns
 *     SS_ERR_INVALID_ARG (null required pointer, n < 0, width/height <= 0, sh_degree not in
 *     0..3, workspace too small, mode out of range) or SS_ERR_UNSUPPORTED (more than 65536
 *     tiles or more than 256 tiles along an axis, n or capacity >= 2^30).  A failed launch returns SS_ERR_CUDA (the CUDA error
 *     string is available from ss_last_cuda_error of the same thread).  Device-side faults
 *     surface on the caller's next synchronisation.  Pair-array overflow is NOT an error
 *     code (the calls only enqueue work, and P is known on the device only): ss_preprocess
 *     stores P in the workspace's total_pairs; ss_bin sets the overflow flag and increments the
 *     sticky overflow_count, and then ss_bin / ss_sort write NO pairs (all ranges empty), so
 *     ss_render outputs background only and ss_prune_score adds nothing for that frame.  The
 *     caller reads overflow (one frame) or overflow_count (a batch of frames, one read), grows
 *     `capacity` and re-runs those frames (every call is idempotent given the same inputs).
 */
#ifndef SS_H
#define SS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SS_API __attribute__((visibility("default")))
#else
#define SS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SS_OK = 0,
    SS_ERR_INVALID_ARG = 1,
    SS_ERR_CAPACITY = 2, /* reserved: capacity overflow is reported through the workspace flag */
    SS_ERR_CUDA = 3,
    SS_ERR_UNSUPPORTED = 4
} ss_status;

typedef enum {
    SS_BIN_3SIGMA = 0,   /* baseline: tiles meeting the square mu +- ceil(3 sqrt(lambda_max)), Eq. 8 */
    SS_BIN_SNUGBOX = 1,  /* tiles meeting the exact bbox of the alpha >= 1/255 ellipse, Eqs. 14-16 */
    SS_BIN_ACCUTILE = 2  /* exactly the tiles meeting that ellipse, Algorithm 1 */
} ss_bin_mode;

/* Gaussian set G = {mu, s, r, h, sigma} (Eq. 1), SoA float32 planes in HBM.
 * Parameters are ACTIVATED: linear scales, opacity in (0,1); the quaternion is normalised
 * in-kernel.  SH coefficient k = basis*3 + channel of Gaussian i is component k%4 of float4
 * sh[i*B + k/4]: one contiguous block of B float4 per Gaussian (B = 1, 3, 7, 12 for degree
 * 0..3), so that the 16*B bytes of a Gaussian with tiles are read whole and those of the
 * others not at all. */
typedef struct {
    int32_t n;              /* number of Gaussians, 0 <= n < 2^30                            */
    int32_t sh_degree;      /* 0..3                                                          */
    const float *mean_opac; /* [n][4]  x, y, z (world), opacity sigma                         */
    const float *scale;     /* [n][4]  sx, sy, sz (linear), unused                            */
    const float *rot;       /* [n][4]  quaternion w, x, y, z                                  */
    const float *sh;        /* [n][B][4] per-Gaussian SH blocks                                */
} ss_scene;

/* Pinhole camera (host struct, copied into kernel arguments).  Pixel (col,row) has
 * coordinate (col,row); x2d = fx * X/Z + cx, y2d = fy * Y/Z + cy in camera space
 * p = viewmat[:, :3] mu + viewmat[:, 3].  Depth = Z. */
typedef struct {
    float viewmat[12]; /* world -> camera, 3x4 row-major                                      */
    float fx, fy, cx, cy;
    float campos[3];   /* camera centre in world space (SH view direction)                   */
    int32_t width, height;
    float z_near;      /* keep a Gaussian iff Z >= z_near (0.2 typical)                       */
    float clip;        /* EWA Jacobian clamp: |X/Z| <= clip * (W/2)/fx (1.3 typical, 0 = off) */
} ss_camera;

/* One frame's device workspace.  `capacity` = maximum number of (tile, Gaussian) pairs the
 * workspace holds; `width`/`height` fix the 16x16 tile grid. */
typedef struct {
    void *ws;          /* device, ss_frame_workspace_size(n, capacity, width, height) bytes  */
    size_t ws_bytes;
    int32_t n;
    uint32_t capacity;
    int32_t width, height;
} ss_frame;

/* Byte offsets of every sub-buffer inside the workspace (for inspection and tests).
 * Records of a Gaussian with >= 1 tile (written only for those):
 *   rec  (48 B, render): q0 = (x2d, y2d, a, b), q1 = (c, t, sigma, 0), q2 = (f, r, g, b)
 *        (a, b, c) = conic Sigma_2D^-1 (Eq. 10); t = 2 log(255 sigma) (Eq. 11); the colour
 *        (R13) is computed lazily: ss_preprocess writes q2 = 0 (f = 0, pending) and the first
 *        render-path call that gathers the record (ss_render, ss_prune_score,
 *        ss_render_backward, ss_render_stats) computes it from the scene's SH and stores
 *        q2 = (1, r, g, b); ss_finalize_colours completes the rest (inspection)
 *   erec (32 B, emission, one sector): (count, info, p0..p5); the payload holds the
 *        non-empty line spans (tmin | tmax << 9 | line << 18) of an AccuTile set of at most 6
 *        lines, or up to 6 super-tile entries (super-tile id | mask of its 4x4 tiles << 16,
 *        bit (y&3)*4 + (x&3)), or -- for a Gaussian with more entries -- aux = t as float64
 *        bits (AccuTile) or the packed rect (x0, x1-x0-1, y0, y1-y0-1) in p0, p1; info = span
 *        count | entries-inline 0x100 | columns 0x200 | AccuTile 0x400 | spans-inline 0x800 |
 *        entries << 12.
 * Depth lives in depth_key (float bits, 0xFFFFFFFF = no tiles).  The pairs are never
 * stored unsorted: ss_sort writes each one once, at its sorted position (Gaussian index,
 * uint32, in sorted_value; its tile is given by ranges, its depth by depth_key). */
typedef struct {
    size_t rec;           /* float4 [3n]  render records                                      */
    size_t erec;          /* uint4  [2n]  emission records                                    */
    size_t depth_key;     /* uint32 [n]   float bits of depth, 0xFFFFFFFF = no tiles          */
    size_t order;         /* uint32 [n]   visible Gaussians in (depth, index) order           */
    size_t sorted_value;  /* uint32 [capacity] Gaussian ids sorted by (tile, depth, index)    */
    size_t tile_count;    /* uint32 [n_tiles]                                                 */
    size_t ranges;        /* uint32 [n_tiles][2] per tile [start, end) into sorted_value      */
    size_t n_visible;     /* uint32 [1]   Gaussians with >= 1 tile                            */
    size_t total_pairs;   /* uint32 [1]   P (written by ss_preprocess)                        */
    size_t overflow;      /* uint32 [1]   1 iff P > capacity (this frame; rewritten by ss_bin)  */
    size_t overflow_count;/* uint32 [1]   sticky: frames with P > capacity since the caller last
                                          zeroed it (libss only increments it; zero it when the
                                          workspace is allocated)                               */
    size_t pre_deferred;  /* uint32 [1]   Gaussians ss_preprocess evaluated on its float64 path
                                          (SnugBox / AccuTile: those whose float32 tile decisions
                                          could not be certified; 3-sigma: all)                 */
    size_t scratch;       /* internal                                                         */
    size_t total_bytes;
    int32_t tiles_x, tiles_y, n_tiles, tile_bits;
} ss_layout;

SS_API size_t ss_frame_workspace_size(int32_t n, uint32_t capacity, int32_t width, int32_t height);

/* Workspace sizes by kind: SS_WS_FRAME = ss_frame_workspace_size(n, capacity,
 * width, height); SS_WS_PRUNE = ss_prune_workspace_size(n) (capacity, width, height ignored).
 * *bytes (host) receives the size; SS_ERR_INVALID_ARG for an unknown kind, n < 0, a null
 * `bytes`, or (frame) width / height <= 0. */
typedef enum { SS_WS_FRAME = 0, SS_WS_PRUNE = 1 } ss_workspace_kind;
SS_API ss_status ss_workspace_size(int which, int32_t n, uint32_t capacity, int32_t width, int32_t height,
                                   size_t *bytes /*host*/);
SS_API ss_status ss_frame_layout(int32_t n, uint32_t capacity, int32_t width, int32_t height, ss_layout *out /*host*/);

/* a1 -- preprocess (Sec. 3.2.1; count mode of SnugBox/AccuTile).
 * Per Gaussian: cull (Z < z_near, singular Sigma_2D; in SnugBox/AccuTile also sigma <=
 * 1/255), project mu, Sigma_3D = R S S^T R^T (Eq. 3), Sigma_2D = J W Sigma_3D W^T J^T + 0.3 I
 * (Eq. 4), conic, SH colour, t, the mode's tile rect and tile count.  Writes rec, erec,
 * depth_key, n_visible, total_pairs (P) and the depth-digit histograms.  Reads the 16 B mean_opac of every
 * Gaussian and the rest only for Gaussians in front of the camera. */
SS_API ss_status ss_preprocess(const ss_scene *scene /*host*/, const ss_camera *cam /*host*/, ss_bin_mode mode,
                        const ss_frame *frame /*host*/, void *stream);

/* a2 + a5 -- key allocation (InclusiveSum) and tile ranges (identifyTileRanges).
 * Orders the visible Gaussians by (depth bits, index) (stable LSD radix sort, 4 passes),
 * scans their super-tile entry counts in that order (one entry per 4x4-tile super-tile a
 * Gaussian's tile set touches, with the mask of its tiles there; the tile set is recomputed
 * from the stored record by the same function as the count), partitions the entries
 * stably by super-tile and counts the pairs of every tile: writes order, tile_count, ranges
 * (empty tiles: [0,0)) and overflow (P = total_pairs, summed by ss_preprocess, > capacity).
 * Requires ss_preprocess on the frame. */
SS_API ss_status ss_bin(const ss_camera *cam /*host*/, ss_bin_mode mode, const ss_frame *frame /*host*/, void *stream);

/* a3 + a4 -- duplicateWithKeys + RadixSort, fused: every super-tile's
 * depth-ordered entries are split into its tiles' lists and every pair is written once, at
 * its sorted position.  The result (sorted_value over the ranges of ss_bin) equals the
 * paper's stable sort of the 64-bit keys (tile << 32 | depth bits) emitted in Gaussian-index
 * order.  Writes nothing on capacity overflow.  Requires ss_bin on the frame. */
SS_API ss_status ss_sort(const ss_frame *frame /*host*/, void *stream);

/* Materialise the paper's sorted 64-bit key array (tile << 32 | float bits of depth) from
 * sorted_value and ranges: keys[P] (device, >= capacity entries).  Inspection only. */
SS_API ss_status ss_sorted_keys(const ss_frame *frame /*host*/, uint64_t *keys, void *stream);

/* a6 -- render (Sec. 3.2.3, Eqs. 5-7).  One CTA per 16x16 tile; each pixel walks its
 * tile's depth-ordered list: q = (p-mu)^T Sigma^-1 (p-mu); skip unless q <= t (alpha >=
 * 1/255, Eq. 9); alpha = min(0.99, sigma e^{-q/2}); stop before blending when T(1-alpha) <
 * 1e-4; C += c alpha T.  out_rgb = C + T bg, planar float32 [3][H][W].  out_T (float32
 * [H][W], final transmittance) and out_ncontrib (uint32 [H][W], list entries up to and
 * including the last blended one) are optional (NULL). bg is host float[3]. */
SS_API ss_status ss_render(const ss_frame *frame /*host*/, const float *bg /*host [3]*/, float *out_rgb,
                    float *out_T, uint32_t *out_ncontrib, void *stream);

/* Inspection: compute the colour of every record still pending (Gaussians with tiles that no
 * render-path call has gathered), so that rec holds all colours.  Requires ss_preprocess on
 * the frame; the scene passed to it must still be alive. */
SS_API ss_status ss_finalize_colours(const ss_frame *frame /*host*/, void *stream);

/* Measurement helper (never on the timed path): work counts of ss_render for the frame,
 * accumulated into counters (device uint64 [5]): E_pix (per-pixel evaluations until each
 * pixel terminates: the method's work), E_blend (evaluations that blend), E_cta (evaluations
 * issued by CTA-lock-step walking: 256 x Gaussians staged), pixels, and phantom pairs ((tile,
 * Gaussian) pairs whose Gaussian has alpha < 1/255 at every pixel centre of the tile; AccuTile
 * tests the continuous cell, R23). */
SS_API ss_status ss_render_stats(const ss_frame *frame /*host*/, uint64_t *counters, void *stream);

/* a7 -- efficient pruning score (Sec. 4.2.1, Eqs. 20-21):
 *   score[i] += sum_p sum_ch (sigma_i dC_ch(p)/dalpha_i(p))^2,
 *   dC/dalpha_i = c_i T_i - (sum_{k>i} c_k alpha_k T_k + bg T_final) / (1 - alpha_i)
 * over every pixel p where Gaussian i is blended in this frame.  Forward pass per pixel,
 * then a back-to-front sweep (recursive suffix colour); per-Gaussian partial sums are
 * reduced in the CTA and added with float64 atomics.  score: float64 [n], accumulated.
 * Requires ss_sort on the frame. */
SS_API ss_status ss_prune_score(const ss_frame *frame /*host*/, const float *bg /*host [3]*/, double *score,
                         void *stream);

/* Prune step (Sec. 4.2 P:381 "removing a set percentage with the lowest
 * sensitivities", Soft Pruning P:422-425, Hard Pruning P:434-436).
 * ss_prune_select: keep[i] (device uint8 [n]) = 0 for exactly k = ss_prune_count(n, ratio) =
 * floor(ratio n) Gaussians with the smallest score (device float64 [n], e.g. the all-reduced
 * U~); on equal scores the higher index is removed first.  ratio in [0, 1].
 * ss_compact_scene: stable stream compaction of every array of `in` into `out` (device arrays
 * allocated by the caller for out->n = n - k Gaussians); *n_out (device uint32) receives the
 * survivor count (the number of non-zero keep entries).  Only the first out->n survivors are
 * written: a mask keeping more than out->n is not a memory error, and the caller detects it by
 * *n_out > out->n.  Both use a caller workspace
 * of ss_prune_workspace_size(n) bytes (device). */
SS_API size_t ss_prune_workspace_size(int32_t n);
SS_API uint32_t ss_prune_count(int32_t n, double ratio);
SS_API ss_status ss_prune_select(const double *score, int32_t n, double ratio, uint8_t *keep, void *ws,
                                 size_t ws_bytes, void *stream);
SS_API ss_status ss_compact_scene(const ss_scene *in /*host*/, const uint8_t *keep, const ss_scene *out /*host*/,
                                  uint32_t *n_out, void *ws, size_t ws_bytes, void *stream);

/* ---- NEXT-2: backward of the forward path ("the per-pixel gradients from the render
 * kernel are parallelized and aggregated to the 2D mu_2D and Sigma_2D parameters, which are
 * then parallelized across Gaussians to compute gradients for mu and s").  The gradient is
 * the derivative of the forward above where it is differentiable (reading R27):
 * a clamped alpha (0.99), a clamped J entry and a clamped colour pass nothing through the
 * clamped quantity; t, the tile sets and the depth order carry no gradient.
 *
 * ss_render_backward: for the frame of the last ss_sort (records, sorted values, ranges in the
 * workspace) and its ss_render outputs T_final (float32 [H][W]) and n_contrib (uint32 [H][W]),
 * given dL_dimg = dL/dC (float32 [3][H][W], planar like out_rgb) and the same bg, ACCUMULATES
 * into grad2d (float32 [n][12], caller-zeroed once) per Gaussian:
 *   (dL/dx2d, dL/dy2d, dL/da, dL/db | dL/dc, dL/dsigma, dL/dr, dL/dg | dL/db_rgb, 0, 0, 0)
 * with (a, b, c) the conic of the record (q = a dx^2 + 2 b dx dy + c dy^2) and (x2d, y2d) the
 * projected mean (its magnitude is 3D-GS's densification signal).  Per tile, back to front
 * from each pixel's last blended entry; float32 atomics (summation order is not fixed). */
SS_API ss_status ss_render_backward(const ss_frame *frame /*host*/, const float *bg /*host [3]*/,
                                    const float *dL_dimg, const float *T_final, const uint32_t *n_contrib,
                                    float *grad2d, void *stream);

/* Gradient arrays laid out exactly like ss_scene's (mean_opac: dL/d(x, y, z, sigma); scale:
 * dL/d(sx, sy, sz), w untouched; rot: dL/d(w, x, y, z) of the UNNORMALISED quaternion; sh:
 * per-Gaussian blocks like scene->sh). */
typedef struct {
    int32_t n, sh_degree;
    float *mean_opac, *scale, *rot, *sh;
} ss_scene_grad;

/* ss_preprocess_backward: chain rule of ss_preprocess (Eqs. 3-4, 10, SH colour) from grad2d of
 * one view to the scene parameters, ACCUMULATED (+=) into `grad` (so views can be summed; the
 * caller zeroes it).  One thread per Gaussian; Gaussians with an all-zero grad2d row are
 * skipped.  grad->n and grad->sh_degree must equal the scene's. */
SS_API ss_status ss_preprocess_backward(const ss_scene *scene /*host*/, const ss_camera *cam /*host*/,
                                        const float *grad2d, const ss_scene_grad *grad /*host*/, void *stream);

/* Variant for a training step (one view per step): the gradients of the Gaussians with a non-zero
 * grad2d row are WRITTEN (=), not accumulated, and flags[i] (device uint8 [n], caller-zeroed) is
 * set to 1 for each of them; the other Gaussians' gradient entries are left untouched (stale) and
 * must be read as zero -- ss_adam_step_flagged does -- so the gradient arrays need no zeroing. */
SS_API ss_status ss_preprocess_backward_assign(const ss_scene *scene /*host*/, const ss_camera *cam /*host*/,
                                               const float *grad2d, const ss_scene_grad *grad /*host*/,
                                               uint8_t *flags, void *stream);

/* ---- NEXT-3: the optimisation step around the backward (Eq. 2, "optimized via
 * stochastic gradient descent on image reconstruction losses"; L1 term only, the D-SSIM term
 * is omitted -- SPEC S:421).
 *
 * ss_l1_loss_grad: dL_dimg[k] = sign(img[k] - gt[k]) / count (sign(0) = 0), *loss_sum +=
 * sum_k |img[k] - gt[k]| (device float64, caller-zeroed; L = loss_sum / count).  count >= 0
 * float32 values; img, gt, dL_dimg device arrays of `count` floats. */
SS_API ss_status ss_l1_loss_grad(int64_t count, const float *img, const float *gt, float *dL_dimg, double *loss_sum,
                                 void *stream);

/* Adam (the 3D-GS optimiser) on RAW parameters: raw = (mean xyz, logit sigma | log s | q | h);
 * every step reads grad (dL/d ACTIVATED parameter, from ss_preprocess_backward), applies the
 * activation's derivative (exp for scales, sigmoid for the opacity, identity otherwise),
 * updates raw, m, v (float32) with bias correction for step t = cfg->step >= 1, and writes the
 * activated parameters into `scene` (the arrays the forward reads).  SH coefficients 0..2 (DC)
 * use lr_sh_dc, the rest lr_sh_rest.  ss_adam_init sets raw = act^-1(scene), m = v = 0. All
 * five arrays share the scene's layout and n / sh_degree. */
typedef struct {
    float lr_mean, lr_opacity, lr_scale, lr_rot, lr_sh_dc, lr_sh_rest;
    float beta1, beta2, eps;
    int32_t step;
} ss_adam_config;
SS_API ss_status ss_adam_init(const ss_scene *scene /*host*/, const ss_scene_grad *raw /*host*/,
                              const ss_scene_grad *m /*host*/, const ss_scene_grad *v /*host*/, void *stream);
SS_API ss_status ss_adam_step(const ss_scene_grad *grad /*host*/, const ss_scene_grad *raw /*host*/,
                              const ss_scene_grad *m /*host*/, const ss_scene_grad *v /*host*/,
                              const ss_scene_grad *scene /*host*/, const ss_adam_config *cfg /*host*/, void *stream);

/* ss_adam_step with gradient flags (ss_preprocess_backward_assign): a Gaussian whose flag is 0 has
 * a zero gradient and its grad entries are not read; the update is otherwise ss_adam_step's
 * (dense Adam: its moments still decay and its raw parameters still move by m / sqrt(v)). */
SS_API ss_status ss_adam_step_flagged(const ss_scene_grad *grad /*host*/, const ss_scene_grad *raw /*host*/,
                                      const ss_scene_grad *m /*host*/, const ss_scene_grad *v /*host*/,
                                      const ss_scene_grad *scene /*host*/, const ss_adam_config *cfg /*host*/,
                                      const uint8_t *flags, void *stream);

/* Convenience: ss_preprocess + ss_bin + ss_sort + ss_render in one call. */
SS_API ss_status ss_render_frame(const ss_scene *scene, const ss_camera *cam, ss_bin_mode mode, const ss_frame *frame,
                          const float *bg, float *out_rgb, float *out_T, uint32_t *out_ncontrib, void *stream);

SS_API const char *ss_status_string(ss_status s);
SS_API const char *ss_last_cuda_error(void);
SS_API const char *ss_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SS_H */
