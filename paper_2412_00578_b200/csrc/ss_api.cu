// ss_api.cu -- the extern "C" boundary of libss.so (declared in include/ss.h).
// Host-side validation, workspace layout and the launch sequence of each call.
#include <cstdio>
#include <cmath>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "ss_common.cuh"

namespace ss {

static size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

bool compute_layout(int32_t n, uint32_t capacity, int32_t width, int32_t height, Layout *L) {
    if (n < 0 || width <= 0 || height <= 0) return false;
    std::memset(L, 0, sizeof(*L));
    ss_layout &P = L->pub;
    P.tiles_x = (width + kTile - 1) / kTile;
    P.tiles_y = (height + kTile - 1) / kTile;
    P.n_tiles = P.tiles_x * P.tiles_y;
    int bits = 1;
    while ((1 << bits) < P.n_tiles) ++bits;
    P.tile_bits = bits;
    L->n = n;
    L->capacity = capacity;
    L->nblk_depth = (uint32_t)(((size_t)n + kSortTile - 1) / kSortTile);
    L->nblk_escan = (uint32_t)(((size_t)n + 8191) / 8192);
    L->stx = (P.tiles_x + kSuperTile - 1) / kSuperTile;
    L->sty = (P.tiles_y + kSuperTile - 1) / kSuperTile;
    L->n_super = L->stx * L->sty;
    L->nck_max = (uint32_t)(((size_t)capacity + kEntChunk - 1) / kEntChunk);
    L->l2_max_blocks = (uint32_t)(((size_t)capacity + kL2BlockEntries - 1) / kL2BlockEntries) + (uint32_t)L->n_super;
    const size_t N = (size_t)n, Cap = capacity, T = (size_t)P.n_tiles, S = (size_t)L->n_super;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes);
        return o;
    };
    P.rec = take(48 * N);
    P.erec = take(32 * N);
    P.depth_key = take(4 * N);
    P.order = take(4 * N);
    L->dkA = take(4 * N);
    L->dvA = take(4 * N);
    L->dkB = take(4 * N);
    L->dvB = take(4 * N);
    P.scratch = L->dkA;
    L->gne = take(4 * N);
    L->one = take(4 * N);
    L->eoff = take(4 * N);
    L->big_queue = take(4 * N);
    L->stg = take(8 * Cap);
    L->ent = take(8 * Cap);
    L->bin_M = take(4 * S * (size_t)L->nck_max);
    L->st_total = take(4 * S);
    L->st_base = take(4 * S);
    L->st_blk0 = take(4 * S);
    L->l2_blocks = take(8 * (size_t)L->l2_max_blocks);
    L->l2_BC = take(64 * (size_t)L->l2_max_blocks);
    P.sorted_value = take(4 * Cap);
    P.ranges = take(8 * T);
    P.tile_count = take(4 * T);
    L->tile_base = take(4 * T);
    L->color_src = take(64);
    L->pix_T = take(4 * (size_t)width * (size_t)height);
    L->pix_last = take(4 * (size_t)width * (size_t)height);
    P.overflow = take(4);
    P.overflow_count = take(4);
    // ---- regions each call clears for itself (so every call is idempotent given its inputs)
    L->zero_pre = off;  // written by ss_preprocess
    P.n_visible = take(4);
    P.total_pairs = take(4);
    L->hist_depth = take(4 * 256 * kDepthPasses);
    L->pre_queue_n = take(4);
    L->pre_ticket = take(4);
    L->zero_pre_end = off;
    L->pre_queue = L->dkA;
    P.pre_deferred = L->pre_queue_n;
    L->zero_bin = off;  // written by ss_bin
    L->counters = take(4 * 16);
    L->lb_depth = take(4 * 256 * (size_t)L->nblk_depth * kDepthPasses);
    L->lb_escan = take(4 * (size_t)L->nblk_escan);
    L->zero_bin_end = off;
    P.total_bytes = off;
    return true;
}

// NVTX range around every enqueueing call (the tracing of SURVEY.md §5): visible to nsys / ncu
// --nvtx; a no-op when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static thread_local char g_cuda_err[256] = "";

static ss_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return SS_OK;
    std::snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return SS_ERR_CUDA;
}

static ss_status check_frame(const ss_frame *f, Layout *L) {
    if (!f || !f->ws) return SS_ERR_INVALID_ARG;
    if (f->n < 0 || f->width <= 0 || f->height <= 0) return SS_ERR_INVALID_ARG;
    if (f->n >= (1 << 30) || f->capacity >= (1u << 30)) return SS_ERR_UNSUPPORTED;
    if (!compute_layout(f->n, f->capacity, f->width, f->height, L)) return SS_ERR_INVALID_ARG;
    if (L->pub.n_tiles > 65536 || L->pub.tiles_x > 256 || L->pub.tiles_y > 256) return SS_ERR_UNSUPPORTED;
    if (f->ws_bytes < L->pub.total_bytes) return SS_ERR_INVALID_ARG;
    return SS_OK;
}

// Camera values every call relies on: positive finite focal lengths, a positive near plane
// (z_near <= 0 would admit Gaussians at or behind the camera, whose depth bits sort wrongly)
// and a finite, non-negative J clamp (0 = off).
static bool cam_values_ok(const ss_camera &c) {
    return c.fx > 0.0f && c.fy > 0.0f && std::isfinite(c.fx) && std::isfinite(c.fy) && c.z_near > 0.0f &&
           std::isfinite(c.z_near) && c.clip >= 0.0f && std::isfinite(c.clip);
}

static ss_status check_cam(const ss_camera *c, const ss_frame *f) {
    if (!c) return SS_ERR_INVALID_ARG;
    if (c->width != f->width || c->height != f->height) return SS_ERR_INVALID_ARG;
    return cam_values_ok(*c) ? SS_OK : SS_ERR_INVALID_ARG;
}

static CamArgs cam_args(const ss_camera &c, const Layout &L) {
    CamArgs a;
    for (int i = 0; i < 12; ++i) a.V[i] = c.viewmat[i];
    a.fx = c.fx;
    a.fy = c.fy;
    a.cx = c.cx;
    a.cy = c.cy;
    a.cpx = c.campos[0];
    a.cpy = c.campos[1];
    a.cpz = c.campos[2];
    a.W = c.width;
    a.H = c.height;
    a.z_near = c.z_near;
    a.clip = c.clip;
    a.tiles_x = L.pub.tiles_x;
    a.tiles_y = L.pub.tiles_y;
    return a;
}

}  // namespace ss

using namespace ss;

extern "C" {

size_t ss_frame_workspace_size(int32_t n, uint32_t capacity, int32_t width, int32_t height) {
    Layout L;
    if (!compute_layout(n, capacity, width, height, &L)) return 0;
    return L.pub.total_bytes;
}

ss_status ss_workspace_size(int which, int32_t n, uint32_t capacity, int32_t width, int32_t height, size_t *bytes) {
    if (!bytes || n < 0) return SS_ERR_INVALID_ARG;
    if (which == SS_WS_FRAME) {
        Layout L;
        if (!compute_layout(n, capacity, width, height, &L)) return SS_ERR_INVALID_ARG;
        *bytes = L.pub.total_bytes;
        return SS_OK;
    }
    if (which == SS_WS_PRUNE) {
        *bytes = prune_workspace_bytes(n);
        return SS_OK;
    }
    return SS_ERR_INVALID_ARG;
}

ss_status ss_frame_layout(int32_t n, uint32_t capacity, int32_t width, int32_t height, ss_layout *out) {
    if (!out) return SS_ERR_INVALID_ARG;
    Layout L;
    if (!compute_layout(n, capacity, width, height, &L)) return SS_ERR_INVALID_ARG;
    *out = L.pub;
    return SS_OK;
}

ss_status ss_preprocess(const ss_scene *scene, const ss_camera *cam, ss_bin_mode mode, const ss_frame *frame,
                        void *stream) {
    NvtxRange nvtx_("ss_preprocess");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if ((s = check_cam(cam, frame)) != SS_OK) return s;
    if (!scene || scene->n != frame->n || scene->sh_degree < 0 || scene->sh_degree > 3) return SS_ERR_INVALID_ARG;
    if (scene->n > 0 && (!scene->mean_opac || !scene->scale || !scene->rot || !scene->sh)) return SS_ERR_INVALID_ARG;
    if ((int)mode < 0 || (int)mode > 2) return SS_ERR_INVALID_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(at<char>(frame->ws, L.zero_pre), 0, L.zero_pre_end - L.zero_pre, st);
    if (e != cudaSuccess) return cuda_status(e);
    return cuda_status(launch_preprocess(*scene, cam_args(*cam, L), (int)mode, frame->ws, L, st));
}

ss_status ss_bin(const ss_camera *cam, ss_bin_mode mode, const ss_frame *frame, void *stream) {
    NvtxRange nvtx_("ss_bin");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if ((s = check_cam(cam, frame)) != SS_OK) return s;
    if ((int)mode < 0 || (int)mode > 2) return SS_ERR_INVALID_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(at<char>(frame->ws, L.zero_bin), 0, L.zero_bin_end - L.zero_bin, st);
    if (e == cudaSuccess) e = launch_depth_sort(frame->ws, L, st);
#ifndef SS_DIAG_BIN_STAGES  // diagnostics builds only: stop ss_bin after the depth sort
    if (e == cudaSuccess) e = launch_bin(frame->ws, L, st);
#endif
    return cuda_status(e);
}

ss_status ss_sort(const ss_frame *frame, void *stream) {
    NvtxRange nvtx_("ss_sort");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    return cuda_status(launch_tile_write(frame->ws, L, static_cast<cudaStream_t>(stream)));
}

ss_status ss_sorted_keys(const ss_frame *frame, uint64_t *keys, void *stream) {
    NvtxRange nvtx_("ss_sorted_keys");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if (!keys) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_sorted_keys(frame->ws, L, keys, static_cast<cudaStream_t>(stream)));
}

ss_status ss_render(const ss_frame *frame, const float *bg, float *out_rgb, float *out_T, uint32_t *out_ncontrib,
                    void *stream) {
    NvtxRange nvtx_("ss_render");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if (!bg || !out_rgb) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_render(frame->ws, L, frame->width, frame->height, bg[0], bg[1], bg[2], out_rgb, out_T,
                                     out_ncontrib, static_cast<cudaStream_t>(stream)));
}

ss_status ss_finalize_colours(const ss_frame *frame, void *stream) {
    NvtxRange nvtx_("ss_finalize_colours");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    return cuda_status(launch_finalize_colours(frame->ws, L, static_cast<cudaStream_t>(stream)));
}

ss_status ss_render_stats(const ss_frame *frame, uint64_t *counters, void *stream) {
    NvtxRange nvtx_("ss_render_stats");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if (!counters) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_render_stats(frame->ws, L, frame->width, frame->height,
                                           reinterpret_cast<unsigned long long *>(counters),
                                           static_cast<cudaStream_t>(stream)));
}

ss_status ss_prune_score(const ss_frame *frame, const float *bg, double *score, void *stream) {
    NvtxRange nvtx_("ss_prune_score");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if (!bg || (!score && frame->n > 0)) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_prune_score(frame->ws, L, frame->width, frame->height, bg[0], bg[1], bg[2], score,
                                          static_cast<cudaStream_t>(stream)));
}

ss_status ss_render_backward(const ss_frame *frame, const float *bg, const float *dL_dimg, const float *T_final,
                             const uint32_t *n_contrib, float *grad2d, void *stream) {
    NvtxRange nvtx_("ss_render_backward");
    Layout L;
    ss_status s = check_frame(frame, &L);
    if (s != SS_OK) return s;
    if (!bg || !dL_dimg || !T_final || !n_contrib || (!grad2d && frame->n > 0)) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_render_backward(frame->ws, L, frame->width, frame->height, bg[0], bg[1], bg[2], dL_dimg,
                                              T_final, n_contrib, grad2d, static_cast<cudaStream_t>(stream)));
}

static ss_status preprocess_backward(const ss_scene *scene, const ss_camera *cam, const float *grad2d,
                                     const ss_scene_grad *grad, uint8_t *flags, void *stream) {
    NvtxRange nvtx_("ss_preprocess_backward");
    if (!scene || !cam || !grad || scene->n < 0 || scene->sh_degree < 0 || scene->sh_degree > 3) return SS_ERR_INVALID_ARG;
    if (grad->n != scene->n || grad->sh_degree != scene->sh_degree) return SS_ERR_INVALID_ARG;
    if (scene->n >= (1 << 30)) return SS_ERR_UNSUPPORTED;
    if (cam->width <= 0 || cam->height <= 0 || !cam_values_ok(*cam)) return SS_ERR_INVALID_ARG;
    if (scene->n > 0 && (!scene->mean_opac || !scene->scale || !scene->rot || !scene->sh || !grad2d ||
                         !grad->mean_opac || !grad->scale || !grad->rot || !grad->sh))
        return SS_ERR_INVALID_ARG;
    Layout L;
    if (!compute_layout(scene->n, 0, cam->width, cam->height, &L)) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_preprocess_backward(*scene, cam_args(*cam, L), grad2d, *grad, flags,
                                                  static_cast<cudaStream_t>(stream)));
}

ss_status ss_preprocess_backward(const ss_scene *scene, const ss_camera *cam, const float *grad2d,
                                 const ss_scene_grad *grad, void *stream) {
    return preprocess_backward(scene, cam, grad2d, grad, nullptr, stream);
}

ss_status ss_preprocess_backward_assign(const ss_scene *scene, const ss_camera *cam, const float *grad2d,
                                        const ss_scene_grad *grad, uint8_t *flags, void *stream) {
    if (!flags && scene && scene->n > 0) return SS_ERR_INVALID_ARG;
    return preprocess_backward(scene, cam, grad2d, grad, flags, stream);
}

static bool grad_ok(const ss_scene_grad *g, int32_t n, int32_t deg) {
    if (!g || g->n != n || g->sh_degree != deg) return false;
    return n == 0 || (g->mean_opac && g->scale && g->rot && g->sh);
}

ss_status ss_l1_loss_grad(int64_t count, const float *img, const float *gt, float *dL_dimg, double *loss_sum,
                          void *stream) {
    NvtxRange nvtx_("ss_l1_loss_grad");
    if (count < 0 || (count > 0 && (!img || !gt || !dL_dimg || !loss_sum))) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_l1_loss_grad(count, img, gt, dL_dimg, loss_sum, static_cast<cudaStream_t>(stream)));
}

ss_status ss_adam_init(const ss_scene *scene, const ss_scene_grad *raw, const ss_scene_grad *m,
                       const ss_scene_grad *v, void *stream) {
    NvtxRange nvtx_("ss_adam_init");
    if (!scene || scene->n < 0 || scene->sh_degree < 0 || scene->sh_degree > 3) return SS_ERR_INVALID_ARG;
    if (scene->n > 0 && (!scene->mean_opac || !scene->scale || !scene->rot || !scene->sh)) return SS_ERR_INVALID_ARG;
    if (!grad_ok(raw, scene->n, scene->sh_degree) || !grad_ok(m, scene->n, scene->sh_degree) ||
        !grad_ok(v, scene->n, scene->sh_degree))
        return SS_ERR_INVALID_ARG;
    return cuda_status(launch_adam_init(*scene, *raw, *m, *v, static_cast<cudaStream_t>(stream)));
}

static ss_status adam_step(const ss_scene_grad *grad, const ss_scene_grad *raw, const ss_scene_grad *m,
                           const ss_scene_grad *v, const ss_scene_grad *scene, const ss_adam_config *cfg,
                           const uint8_t *flags, void *stream) {
    NvtxRange nvtx_("ss_adam_step");
    if (!grad || !cfg || grad->n < 0 || grad->sh_degree < 0 || grad->sh_degree > 3) return SS_ERR_INVALID_ARG;
    const int32_t n = grad->n, d = grad->sh_degree;
    if (!grad_ok(grad, n, d) || !grad_ok(raw, n, d) || !grad_ok(m, n, d) || !grad_ok(v, n, d) || !grad_ok(scene, n, d))
        return SS_ERR_INVALID_ARG;
    if (cfg->step < 1 || !(cfg->beta1 >= 0.0f && cfg->beta1 < 1.0f) || !(cfg->beta2 >= 0.0f && cfg->beta2 < 1.0f) ||
        !(cfg->eps >= 0.0f))
        return SS_ERR_INVALID_ARG;
    const int64_t blocks_sh = ((int64_t)(d + 1) * (d + 1) * 3 + 3) / 4;
    if ((int64_t)n * blocks_sh >= (int64_t)1 << 31) return SS_ERR_UNSUPPORTED;  // 32-bit slot indexing
    return cuda_status(launch_adam_step(*grad, *raw, *m, *v, *scene, *cfg, flags, static_cast<cudaStream_t>(stream)));
}

ss_status ss_adam_step(const ss_scene_grad *grad, const ss_scene_grad *raw, const ss_scene_grad *m,
                       const ss_scene_grad *v, const ss_scene_grad *scene, const ss_adam_config *cfg, void *stream) {
    return adam_step(grad, raw, m, v, scene, cfg, nullptr, stream);
}

ss_status ss_adam_step_flagged(const ss_scene_grad *grad, const ss_scene_grad *raw, const ss_scene_grad *m,
                               const ss_scene_grad *v, const ss_scene_grad *scene, const ss_adam_config *cfg,
                               const uint8_t *flags, void *stream) {
    if (!flags && grad && grad->n > 0) return SS_ERR_INVALID_ARG;
    return adam_step(grad, raw, m, v, scene, cfg, flags, stream);
}

ss_status ss_render_frame(const ss_scene *scene, const ss_camera *cam, ss_bin_mode mode, const ss_frame *frame,
                          const float *bg, float *out_rgb, float *out_T, uint32_t *out_ncontrib, void *stream) {
    NvtxRange nvtx_("ss_render_frame");
    ss_status s = ss_preprocess(scene, cam, mode, frame, stream);
    if (s == SS_OK) s = ss_bin(cam, mode, frame, stream);
    if (s == SS_OK) s = ss_sort(frame, stream);
    if (s == SS_OK) s = ss_render(frame, bg, out_rgb, out_T, out_ncontrib, stream);
    return s;
}

size_t ss_prune_workspace_size(int32_t n) { return n < 0 ? 0 : prune_workspace_bytes(n); }

uint32_t ss_prune_count(int32_t n, double ratio) {
    if (n <= 0) return 0;
    double kd = floor(ratio * (double)n);
    if (kd < 0.0) kd = 0.0;
    if (kd > (double)n) kd = (double)n;
    return (uint32_t)kd;
}

ss_status ss_prune_select(const double *score, int32_t n, double ratio, uint8_t *keep, void *ws, size_t ws_bytes,
                          void *stream) {
    NvtxRange nvtx_("ss_prune_select");
    if (n < 0 || !(ratio >= 0.0) || !(ratio <= 1.0)) return SS_ERR_INVALID_ARG;
    if (n >= (1 << 30)) return SS_ERR_UNSUPPORTED;
    if (n > 0 && (!score || !keep)) return SS_ERR_INVALID_ARG;
    if (!ws || ws_bytes < prune_workspace_bytes(n)) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_prune_select(score, n, ratio, keep, ws, static_cast<cudaStream_t>(stream)));
}

ss_status ss_compact_scene(const ss_scene *in, const uint8_t *keep, const ss_scene *out, uint32_t *n_out,
                           void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("ss_compact_scene");
    if (!in || !out || !n_out || in->n < 0 || in->sh_degree < 0 || in->sh_degree > 3) return SS_ERR_INVALID_ARG;
    if (out->sh_degree != in->sh_degree || out->n < 0 || out->n > in->n) return SS_ERR_INVALID_ARG;
    if (in->n > 0 && (!keep || !in->mean_opac || !in->scale || !in->rot || !in->sh)) return SS_ERR_INVALID_ARG;
    if (out->n > 0 && (!out->mean_opac || !out->scale || !out->rot || !out->sh)) return SS_ERR_INVALID_ARG;
    if (!ws || ws_bytes < prune_workspace_bytes(in->n)) return SS_ERR_INVALID_ARG;
    return cuda_status(launch_compact(*in, keep, *out, (uint32_t)out->n, n_out, ws, static_cast<cudaStream_t>(stream)));
}

const char *ss_status_string(ss_status s) {
    switch (s) {
        case SS_OK: return "SS_OK";
        case SS_ERR_INVALID_ARG: return "SS_ERR_INVALID_ARG";
        case SS_ERR_CAPACITY: return "SS_ERR_CAPACITY";
        case SS_ERR_CUDA: return "SS_ERR_CUDA";
        case SS_ERR_UNSUPPORTED: return "SS_ERR_UNSUPPORTED";
    }
    return "SS_UNKNOWN";
}

const char *ss_last_cuda_error(void) { return g_cuda_err; }

const char *ss_version(void) { return "libss 0.1 (sm_100a)"; }

}  // extern "C"
