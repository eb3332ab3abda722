// ss_render.cu -- a6 render (Eqs. 5-7) and a7 efficient pruning score (Eqs. 20-21).
//
// One CTA per 16x16 tile, one thread per pixel ("parallelized across pixels").  The
// tile's depth-ordered Gaussian ids are consumed in batches of 256: each thread gathers one
// 48 B record into shared memory, then every pixel walks the batch.  A CTA stops as soon
// as all of its pixels are saturated (__syncthreads_count).
//
// Arithmetic contract: the alpha-skip decision q <= t (alpha >= 1/255, Eq. 9)
// uses the pinned chain u = fma(a, dx, (2b) dy); q = fma(dx, u, (c dy) dy) with explicit
// round-to-nearest intrinsics, so it is bit-identical to the oracle's; alpha uses the SFU
// exp2 (ex2.approx), which the image tolerance (1e-4) covers.
#include "ss_common.cuh"

namespace ss {
namespace {

constexpr int kBatch = 256;

struct __align__(16) GRec {
    float x, y, a, b2;      // b2 = 2b (exact)
    float c, t, sigma, pad;
    float r, g, b, pad2;
};

__device__ __forceinline__ float pixel_q(float fx, float fy, float x, float y, float a, float b2, float c) {
    const float dx = __fsub_rn(fx, x);
    const float dy = __fsub_rn(fy, y);
    const float u = __fmaf_rn(a, dx, __fmul_rn(b2, dy));
    return __fmaf_rn(dx, u, __fmul_rn(__fmul_rn(c, dy), dy));
}

__device__ __forceinline__ float alpha_of(float q, float sigma) {
    // sigma * e^{-q/2} = sigma * 2^{q * (-log2(e)/2)}, clamped at 0.99 (R16)
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(q * -0.72134752044448170f));
    return fminf(0.99f, sigma * e);
}

__device__ __forceinline__ void load_batch(GRec *s, const uint32_t *__restrict__ vals, const float4 *__restrict__ rec,
                                           uint32_t j, uint32_t end, uint32_t *s_id) {
    if (j < end) {
        const uint32_t g = vals[j];
        const float4 r0 = __ldg(rec + 3 * (size_t)g + 0);
        const float4 r1 = __ldg(rec + 3 * (size_t)g + 1);
        const float4 r2 = __ldg(rec + 3 * (size_t)g + 2);
        GRec &d = s[threadIdx.x];
        d.x = r0.x; d.y = r0.y; d.a = r0.z; d.b2 = r0.w + r0.w;
        d.c = r1.x; d.t = r1.y; d.sigma = r1.z; d.pad = 0.f;
        d.r = r2.x; d.g = r2.y; d.b = r2.z; d.pad2 = 0.f;
        if (s_id) s_id[threadIdx.x] = g;
    }
}

__global__ void __launch_bounds__(256) k_render(const uint2 *__restrict__ ranges, const uint32_t *__restrict__ vals,
                                                const float4 *__restrict__ rec, int W, int H, int tiles_x, float bg0,
                                                float bg1, float bg2, float *__restrict__ out_rgb,
                                                float *__restrict__ out_T, uint32_t *__restrict__ out_nc) {
    __shared__ GRec s_g[kBatch];
    const int tile = blockIdx.x;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x & 15);
    const int py = (tile / tiles_x) * kTile + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const float fpx = (float)px, fpy = (float)py;
    const uint2 range = ranges[tile];
    bool done = !inside;
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
    uint32_t last = 0;
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        if (__syncthreads_count(done) == blockDim.x) break;
        load_batch(s_g, vals, rec, start + threadIdx.x, range.y, nullptr);
        __syncthreads();
        const int cnt = min((uint32_t)kBatch, range.y - start);
        for (int k = 0; k < cnt && !done; ++k) {
            const GRec &g = s_g[k];
            const float q = pixel_q(fpx, fpy, g.x, g.y, g.a, g.b2, g.c);
            if (!(q <= g.t)) continue;  // alpha < 1/255: no contribution (Eq. 9, R15)
            const float alpha = alpha_of(q, g.sigma);
            const float Tn = T * (1.0f - alpha);
            if (Tn < 1e-4f) {  // R16: stop before blending
                done = true;
                break;
            }
            const float w = alpha * T;
            C0 = fmaf(g.r, w, C0);
            C1 = fmaf(g.g, w, C1);
            C2 = fmaf(g.b, w, C2);
            T = Tn;
            last = start - range.x + k + 1;
        }
    }
    if (inside) {
        const size_t p = (size_t)py * W + px, plane = (size_t)W * H;
        out_rgb[p] = fmaf(T, bg0, C0);
        out_rgb[plane + p] = fmaf(T, bg1, C1);
        out_rgb[2 * plane + p] = fmaf(T, bg2, C2);
        if (out_T) out_T[p] = T;
        if (out_nc) out_nc[p] = last;
    }
}

// a7: forward (T_final, last blended index per pixel), then back-to-front over the tile list
// recovering T_i = T_{i+1} / (1 - alpha_i) and the suffix colour S <- alpha c + (1-alpha) S:
//   dC_ch/dalpha_i = T_i (c_ch - S_ch) - T_final bg_ch / (1 - alpha_i)      (from Eq. 7)
//   U_i += sum_ch (sigma_i dC_ch/dalpha_i)^2                                 (Eqs. 20-21)
// Per batch, per-Gaussian sums are reduced warp -> CTA in shared memory and added to the
// float64 score with one atomic per (tile, Gaussian).
__global__ void __launch_bounds__(256) k_prune_score(const uint2 *__restrict__ ranges,
                                                     const uint32_t *__restrict__ vals,
                                                     const float4 *__restrict__ rec, int W, int H, int tiles_x,
                                                     float bg0, float bg1, float bg2, double *__restrict__ score) {
    __shared__ GRec s_g[kBatch];
    __shared__ uint32_t s_id[kBatch];
    __shared__ float s_part[8][kBatch];
    __shared__ uint32_t s_max;
    const int tile = blockIdx.x;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x & 15);
    const int py = (tile / tiles_x) * kTile + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const float fpx = (float)px, fpy = (float)py;
    const uint2 range = ranges[tile];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bool done = !inside;
    float T = 1.0f;
    uint32_t last = 0;
    if (threadIdx.x == 0) s_max = 0;
    // forward
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        if (__syncthreads_count(done) == blockDim.x) break;
        load_batch(s_g, vals, rec, start + threadIdx.x, range.y, nullptr);
        __syncthreads();
        const int cnt = min((uint32_t)kBatch, range.y - start);
        for (int k = 0; k < cnt && !done; ++k) {
            const GRec &g = s_g[k];
            const float q = pixel_q(fpx, fpy, g.x, g.y, g.a, g.b2, g.c);
            if (!(q <= g.t)) continue;
            const float alpha = alpha_of(q, g.sigma);
            const float Tn = T * (1.0f - alpha);
            if (Tn < 1e-4f) {
                done = true;
                break;
            }
            T = Tn;
            last = start - range.x + k + 1;
        }
    }
    __syncthreads();
    atomicMax(&s_max, last);
    __syncthreads();
    const uint32_t max_last = s_max;
    const float Tfin = T;
    float S0 = 0.f, S1 = 0.f, S2 = 0.f;
    // backward, batches from the end
    for (uint32_t end = range.x + max_last; end > range.x;) {
        const uint32_t start = end - range.x > (uint32_t)kBatch ? end - kBatch : range.x;
        const int cnt = (int)(end - start);
        __syncthreads();
        load_batch(s_g, vals, rec, start + threadIdx.x, end, s_id);
        __syncthreads();
        for (int k = cnt - 1; k >= 0; --k) {
            const GRec &g = s_g[k];
            float term = 0.f;
            if (start - range.x + (uint32_t)k < last) {
                const float q = pixel_q(fpx, fpy, g.x, g.y, g.a, g.b2, g.c);
                if (q <= g.t) {
                    const float alpha = alpha_of(q, g.sigma);
                    const float om = 1.0f - alpha;
                    T = T / om;
                    const float bgs = Tfin / om;
                    const float d0 = T * (g.r - S0) - bgs * bg0;
                    const float d1 = T * (g.g - S1) - bgs * bg1;
                    const float d2 = T * (g.b - S2) - bgs * bg2;
                    term = g.sigma * g.sigma * (d0 * d0 + d1 * d1 + d2 * d2);
                    S0 = alpha * g.r + om * S0;
                    S1 = alpha * g.g + om * S1;
                    S2 = alpha * g.b + om * S2;
                }
            }
            if (__any_sync(0xffffffffu, term != 0.f)) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
            }
            if (lane == 0) s_part[warp][k] = term;
        }
        __syncthreads();
        if ((int)threadIdx.x < cnt) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) s += s_part[w][threadIdx.x];
            if (s != 0.f) atomicAdd(score + s_id[threadIdx.x], (double)s);
        }
        end = start;
    }
}

// Measurement only (not on the timed path): the render's work counts for one frame, from
// the same per-pixel walk as k_render.  counters[0] += E_pix (evaluations each pixel makes
// until it terminates), [1] += E_blend (evaluations that blend), [2] += E_cta (evaluations a
// CTA issues in lock-step until its last pixel terminates: 256 x Gaussians staged),
// [3] += pixels.
__global__ void __launch_bounds__(256) k_render_stats(const uint2 *__restrict__ ranges,
                                                      const uint32_t *__restrict__ vals,
                                                      const float4 *__restrict__ rec, int W, int H, int tiles_x,
                                                      unsigned long long *counters) {
    __shared__ GRec s_g[kBatch];
    const int tile = blockIdx.x;
    const int px = (tile % tiles_x) * kTile + (threadIdx.x & 15);
    const int py = (tile / tiles_x) * kTile + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const float fpx = (float)px, fpy = (float)py;
    const uint2 range = ranges[tile];
    bool done = !inside;
    float T = 1.0f;
    unsigned long long e_pix = 0, e_blend = 0, e_cta = 0;
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        if (__syncthreads_count(done) == blockDim.x) break;
        load_batch(s_g, vals, rec, start + threadIdx.x, range.y, nullptr);
        __syncthreads();
        const int cnt = min((uint32_t)kBatch, range.y - start);
        e_cta += cnt;
        for (int k = 0; k < cnt && !done; ++k) {
            const GRec &g = s_g[k];
            ++e_pix;
            const float q = pixel_q(fpx, fpy, g.x, g.y, g.a, g.b2, g.c);
            if (!(q <= g.t)) continue;
            const float alpha = alpha_of(q, g.sigma);
            const float Tn = T * (1.0f - alpha);
            if (Tn < 1e-4f) {
                done = true;
                break;
            }
            ++e_blend;
            T = Tn;
        }
    }
    atomicAdd(counters + 0, e_pix);
    atomicAdd(counters + 1, e_blend);
    if (threadIdx.x == 0) atomicAdd(counters + 2, e_cta * blockDim.x);
    if (inside) atomicAdd(counters + 3, 1ull);
}

}  // namespace

cudaError_t launch_render_stats(void *ws, const Layout &L, int W, int H, unsigned long long *counters,
                                cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    k_render_stats<<<P.n_tiles, 256, 0, st>>>(at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                               at<const float4>(ws, P.rec), W, H, P.tiles_x, counters);
    return cudaGetLastError();
}

cudaError_t launch_render(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2, float *out_rgb,
                          float *out_T, uint32_t *out_nc, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    k_render<<<P.n_tiles, 256, 0, st>>>(at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                         at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2, out_rgb, out_T,
                                         out_nc);
    return cudaGetLastError();
}

cudaError_t launch_prune_score(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2,
                               double *score, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    k_prune_score<<<P.n_tiles, 256, 0, st>>>(at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                              at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2, score);
    return cudaGetLastError();
}

}  // namespace ss
