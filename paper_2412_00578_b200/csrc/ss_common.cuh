// ss_common.cuh -- shared device/host definitions of libss (CUDA path only).
#pragma once
#include <cstdint>
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

// Radix-sort geometry (shared by the sort launchers and the layout).
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;   // 4096 keys per block tile
constexpr int kEmitThreads = 256;                      // one Gaussian per thread
constexpr int kInlineSpans = 4;                        // spans stored in the emission record
constexpr int kDepthPasses = 4;                        // 32-bit depth keys, 8-bit digits

// Look-back status words: 2-bit flag | 30-bit count.
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

// Workspace layout (internal part beyond ss_layout).
struct Layout {
    ss_layout pub;
    // scratch sub-buffers
    size_t dkA, dvA, dkB, dvB;      // depth sort ping-pong (uint32 [n])
    size_t pair_tile2;              // uint16 [capacity] tile-sort ping-pong
    size_t pair_value2;             // uint32 [capacity]
    size_t zero_pre, zero_pre_end;    // regions each call clears for itself
    size_t zero_bin, zero_bin_end;
    size_t zero_sort, zero_sort_end;
    size_t counters_sort;             // uint32 [16] tile-sort tickets / barrier / sort_n
    size_t hist_depth;              // uint32 [4][256]
    size_t hist_tile;               // uint32 [2][256]
    size_t counters;                // uint32 [16] block tickets
    size_t lb_depth;                // uint32 [4][nblk_depth][256]
    size_t lb_tile;                 // uint32 [2][nblk_tile][256]
    size_t lb_emit;                 // uint32 [nblk_emit]
    uint32_t nblk_depth, nblk_tile, nblk_emit;
    int tile_passes;
    int32_t n;
    uint32_t capacity;
};

bool compute_layout(int32_t n, uint32_t capacity, int32_t width, int32_t height, Layout *L);

template <typename T>
__host__ __device__ inline T *at(void *ws, size_t off) {
    return reinterpret_cast<T *>(static_cast<char *>(ws) + off);
}

// Launchers implemented in the kernel translation units.
cudaError_t launch_preprocess(const ss_scene &sc, const CamArgs &cam, int mode, void *ws, const Layout &L,
                              cudaStream_t st);
cudaError_t launch_depth_sort(void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_emit(const CamArgs &cam, int mode, void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_tile_sort(void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_sorted_keys(void *ws, const Layout &L, uint64_t *keys, cudaStream_t st);
cudaError_t launch_render(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2, float *out_rgb,
                          float *out_T, uint32_t *out_nc, cudaStream_t st);
cudaError_t launch_render_stats(void *ws, const Layout &L, int W, int H, unsigned long long *counters,
                                cudaStream_t st);
cudaError_t launch_prune_score(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2,
                               double *score, cudaStream_t st);

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
