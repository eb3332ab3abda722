// ss_common.cuh -- shared device/host definitions of libss (CUDA path only).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/ss.h"

namespace ss {

constexpr int kTile = 16;              // 16x16 pixel tiles
constexpr uint32_t kNoTiles = 0xFFFFFFFFu;

// Camera as kernel argument (derived from ss_camera on the host).
struct CamArgs {
    float V[12];
    float fx, fy, cx, cy;
    float cpx, cpy, cpz;
    int W, H;
    float z_near, clip;
    int tiles_x, tiles_y;
};

// Depth-sort geometry (onesweep LSD radix sort).
constexpr int kSortThreads = 256;
#ifndef SS_SORT_ITEMS
#define SS_SORT_ITEMS 12
#endif
constexpr int kSortItems = SS_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;   // 3072 keys per block tile
constexpr int kInlineEnt = 6;                          // super-tile entries stored in the emission record
#ifndef SS_LANE_ROWS
#define SS_LANE_ROWS 6
#endif
constexpr int kLaneRows = SS_LANE_ROWS;                 // AccuTile lines a preprocess lane sweeps alone
constexpr int kDepthPasses = 4;                        // 32-bit depth keys, 8-bit digits
constexpr uint32_t kInfoEntInline = 0x100u;            // erec info: entries stored in the record
constexpr uint32_t kInfoCols = 0x200u;                 // erec info: columns sweep (lines are tile columns)
constexpr uint32_t kInfoAccuTile = 0x400u;             // erec info: tile set of Algorithm 1
constexpr uint32_t kInfoSpanInline = 0x800u;           // erec info: line spans stored in the record
constexpr int kInfoEntShift = 12;                      // erec info bits 12..31: super-tile entries
constexpr int kSuperTile = 4;                          // super-tile side in tiles (ss_tilegeom.cuh)
#ifndef SS_ENT_WARP
#define SS_ENT_WARP 512
#endif
constexpr int kEntWarp = SS_ENT_WARP;                  // entries per warp unit of level 1
constexpr int kBinWarps = 8;                           // warps per level-1 CTA
constexpr int kEntChunk = kEntWarp * kBinWarps;        // entries per level-1 chunk (CTA)
constexpr int kL2BlockEntries = 2048;                  // entries per level-2 block (CTA)

// Look-back status words: 2-bit flag | 30-bit count.
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

// Workspace layout (internal part beyond ss_layout).
struct Layout {
    ss_layout pub;
    size_t dkA, dvA, dkB, dvB;      // depth sort ping-pong (uint32 [n])
    size_t gne;                     // uint32 [n] super-tile entries per Gaussian (index order)
    size_t one;                     // uint32 [n] the same in depth order
    size_t eoff;                    // uint32 [n] exclusive scan of `one`: first entry of each Gaussian
    size_t big_queue;               // uint32 [n] depth positions of Gaussians with non-inline entries
    size_t stg;                     // uint2 [capacity] staged entries (Gaussian, super-tile | mask << 16)
    size_t ent;                     // uint2 [capacity] entries (Gaussian, tile mask) by super-tile
    size_t bin_M;                   // uint32 [nck_max][n_super] entries per (chunk, super-tile) -> prefix
    size_t st_total, st_base;       // uint32 [n_super] entries per super-tile, first entry
    size_t st_blk0;                 // uint32 [n_super] first level-2 block of each super-tile
    size_t l2_blocks;               // uint2 [l2_max_blocks] (super-tile, first entry) of each block
    size_t l2_BC;                   // uint32 [l2_max_blocks][16] pairs per (block, tile) -> prefix
    size_t tile_base;               // uint32 [n_tiles] first sorted position of each tile
    size_t color_src;               // ColorSrc (64 B): scene mean / SH pointers + camera centre of the frame
    size_t pix_T, pix_last;         // float / uint32 [W*H]: ss_prune_score's forward (T_final, n_contrib)
    size_t zero_pre, zero_pre_end;  // regions each call clears for itself
    size_t zero_bin, zero_bin_end;
    size_t hist_depth;              // uint32 [4][256]
    size_t pre_queue;               // uint32 [n] ss_preprocess's float64 queue (aliases dkA: free until ss_bin)
    size_t pre_queue_n;             // uint32 [1] its length (zeroed with the preprocess region)
    size_t pre_ticket;              // uint32 [1] k_preprocess32's work ticket (zeroed with it)
    size_t counters;                // uint32 [16] tickets: depth passes, scans, last-CTA counters
    size_t lb_depth;                // uint32 [4][nblk_depth][256]
    size_t lb_escan;                // uint32 [nblk_escan] tile sums of the entry scan
    uint32_t nblk_depth, nblk_escan;
    uint32_t nck_max;               // level-1 chunks for `capacity` entries
    uint32_t l2_max_blocks;         // level-2 blocks for `capacity` entries
    int stx, sty, n_super;          // super-tile grid
    int32_t n;
    uint32_t capacity;
};

bool compute_layout(int32_t n, uint32_t capacity, int32_t width, int32_t height, Layout *L);

template <typename T>
__host__ __device__ inline T *at(void *ws, size_t off) {
    return reinterpret_cast<T *>(static_cast<char *>(ws) + off);
}

// Streaming-multiprocessor count of the current device, queried once per device and cached
// (launch-configuration data only: the frame path stays free of host-side device queries).
inline int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = sms > 0 ? sms : 148;
    }
    return cache[dev];
}

// Raises a kernel's dynamic shared-memory limit to `bytes` once per device (idempotent).
template <class K>
inline cudaError_t ensure_smem(K kernel, size_t bytes, int *done /* [64] per device */) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (done[dev] >= (int)bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[dev] = (int)bytes;
    return e;
}

// Programmatic dependent launch: a frame-path kernel may be launched while its predecessor
// in the stream drains; it waits (griddepcontrol.wait) for the predecessor's completion and
// memory before touching anything, then lets its own successor launch.  On a plain launch
// both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Launchers implemented in the kernel translation units.
cudaError_t launch_preprocess(const ss_scene &sc, const CamArgs &cam, int mode, void *ws, const Layout &L,
                              cudaStream_t st);
cudaError_t launch_depth_sort(void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_bin(void *ws, const Layout &L, cudaStream_t st);     // entry scan, level 1, tile counts
cudaError_t launch_tile_write(void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_sorted_keys(void *ws, const Layout &L, uint64_t *keys, cudaStream_t st);
cudaError_t launch_render(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2, float *out_rgb,
                          float *out_T, uint32_t *out_nc, cudaStream_t st);
cudaError_t launch_finalize_colours(void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_render_stats(void *ws, const Layout &L, int W, int H, unsigned long long *counters,
                                cudaStream_t st);
cudaError_t launch_prune_score(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2,
                               double *score, cudaStream_t st);
cudaError_t launch_render_backward(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2,
                                   const float *dimg, const float *T_final, const uint32_t *n_contrib, float *grad2d,
                                   cudaStream_t st);
cudaError_t launch_l1_loss_grad(int64_t count, const float *img, const float *gt, float *grad, double *loss_sum,
                                cudaStream_t st);
cudaError_t launch_adam_init(const ss_scene &sc, const ss_scene_grad &raw, const ss_scene_grad &m,
                             const ss_scene_grad &v, cudaStream_t st);
cudaError_t launch_adam_step(const ss_scene_grad &g, const ss_scene_grad &raw, const ss_scene_grad &m,
                             const ss_scene_grad &v, const ss_scene_grad &out, const ss_adam_config &c,
                             const uint8_t *flags, cudaStream_t st);
cudaError_t launch_preprocess_backward(const ss_scene &sc, const CamArgs &cam, const float *grad2d,
                                       const ss_scene_grad &out, uint8_t *flags, cudaStream_t st);

size_t prune_workspace_bytes(int32_t n);
cudaError_t launch_prune_select(const double *score, int32_t n, double ratio, uint8_t *keep, void *ws,
                                cudaStream_t st);
cudaError_t launch_compact(const ss_scene &in, const uint8_t *keep, const ss_scene &out, uint32_t out_stride,
                           uint32_t *n_out, void *ws, cudaStream_t st);

// Exclusive scan of one value per thread over a 256-thread CTA (8 warps); `total` gets the
// CTA sum.  Contains two __syncthreads: every thread of the CTA must call it.
__device__ __forceinline__ uint32_t block_exclusive_scan_256(uint32_t v, uint32_t *s_warp, uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < 8 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) s_warp[lane] = w;  // inclusive per-warp totals
    }
    __syncthreads();
    total = s_warp[7];
    const uint32_t warp_excl = wid ? s_warp[wid - 1] : 0u;
    return warp_excl + x - v;
}

}  // namespace ss
