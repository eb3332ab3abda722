// ss_render.cu -- a6 render (Eqs. 5-7), a7 efficient pruning score (Eqs. 20-21) and the
// NEXT-2 render backward.
//
// One CTA per 16x16 tile, one thread per pixel ("parallelized across pixels").  The
// tile's depth-ordered Gaussian ids are consumed in batches of kBatch = 128: one thread per
// slot gathers the 48 B record into shared memory (computing the view-dependent colour on
// first use, ss_color.cuh), then every still-active pixel walks the batch.  Before every batch
// the active pixels are compacted onto the lowest threads; a CTA stops as soon as none is left.
//
// Arithmetic contract: the alpha-skip decision q <= t (alpha >= 1/255, Eq. 9)
// uses the pinned chain u = fma(a, dx, (2b) dy); q = fma(dx, u, (c dy) dy) with explicit
// round-to-nearest intrinsics, so it is bit-identical to the oracle's; alpha uses the SFU
// exp2 (ex2.approx), which the image tolerance (1e-4) covers.
#include "ss_color.cuh"

namespace ss {
namespace {

constexpr int kBatch = 128;

// Shared-memory batch of gathered records, split by use: the per-warp culling box, the conic
// (skip test), the colour.
struct Batch {
    float4 box[kBatch];  // x, y, -, -
    float4 con[kBatch];  // a, 2b, c, t
    float4 col[kBatch];  // r, g, b, sigma
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

__device__ __forceinline__ void load_batch(Batch &s, const uint32_t *__restrict__ vals,
                                           const float4 *__restrict__ rec, uint32_t j, uint32_t end,
                                           uint32_t *s_id, const ColorSrc &cs) {
    if (threadIdx.x < kBatch && j < end) {
        const uint32_t g = vals[j];
        const float4 q0 = __ldg(rec + 3 * (size_t)g + 0);  // x, y, a, b
        const float4 q1 = __ldg(rec + 3 * (size_t)g + 1);  // c, t, sigma, 0
        const float4 q2 = record_colour(rec, g, cs);        // done flag, r, g, b (lazy colour)
        s.box[threadIdx.x] = make_float4(q0.x, q0.y, 0.0f, 0.0f);
        s.con[threadIdx.x] = make_float4(q0.z, q0.w + q0.w, q1.x, q1.y);
        s.col[threadIdx.x] = make_float4(q2.y, q2.z, q2.w, q1.z);
        if (s_id) s_id[threadIdx.x] = g;
    } else if (threadIdx.x < kBatch) {  // padding slot: never contributes (q <= -inf is false)
        s.box[threadIdx.x] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        s.con[threadIdx.x] = make_float4(1.0f, 0.0f, 1.0f, __int_as_float(0xff800000));
        s.col[threadIdx.x] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
}

// Pixel p (0..255) of a tile is (p & 15, p >> 4) in the tile, row-major.
__device__ __forceinline__ void tile_pixel(int tile, int tiles_x, int p, int &px, int &py) {
    px = (tile % tiles_x) * kTile + (p & 15);
    py = (tile / tiles_x) * kTile + (p >> 4);
}

// Per-pixel state kept in shared memory between batches, so that before every batch the
// still-active pixels can be compacted onto the lowest threads: warps whose pixels have all
// terminated stop issuing, instead of idling lane by lane inside partially-done warps
// (the per-pixel walk and its arithmetic are unchanged).
struct PixState {
    float T[256], C0[256], C1[256], C2[256];
    uint32_t last[256];
    uint8_t done[256];
    uint16_t list[256];
};

// Compacts the active pixels (one flag per thread = pixel threadIdx.x) into st.list; returns
// their number.  Every thread of the CTA must call it.
__device__ __forceinline__ uint32_t compact_active(bool active, PixState &st, uint32_t *s_warp) {
    uint32_t n_active;
    const uint32_t pos = block_exclusive_scan_256(active ? 1u : 0u, s_warp, n_active);
    if (active) st.list[pos] = (uint16_t)threadIdx.x;
    __syncthreads();
    return n_active;
}

template <bool NC>  // NC: track the last blended list entry per pixel (out_ncontrib requested)
__global__ void __launch_bounds__(256, 6) k_render(const uint2 *__restrict__ ranges, const uint32_t *__restrict__ vals,
                                                const float4 *__restrict__ rec, int W, int H, int tiles_x, float bg0,
                                                float bg1, float bg2, float *__restrict__ out_rgb,
                                                float *__restrict__ out_T, uint32_t *__restrict__ out_nc,
        const ColorSrc *__restrict__ csp) {
    pdl_enter();
    const ColorSrc cs = *csp;
    __shared__ Batch s;
    __shared__ PixState st;
    __shared__ uint32_t s_warp[8];
    const int tile = blockIdx.x;
    int mpx, mpy;
    tile_pixel(tile, tiles_x, threadIdx.x, mpx, mpy);
    const bool inside = mpx < W && mpy < H;
    const uint2 range = ranges[tile];
    st.T[threadIdx.x] = 1.0f;
    st.C0[threadIdx.x] = st.C1[threadIdx.x] = st.C2[threadIdx.x] = 0.0f;
    st.last[threadIdx.x] = 0;
    st.done[threadIdx.x] = inside ? 0 : 1;
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        __syncthreads();
        const uint32_t n_active = compact_active(!st.done[threadIdx.x], st, s_warp);
        if (n_active == 0) break;
        load_batch(s, vals, rec, start + threadIdx.x, range.y, nullptr, cs);
        __syncthreads();
        if (threadIdx.x < n_active) {
            const int pp = st.list[threadIdx.x];
            int px, py;
            tile_pixel(tile, tiles_x, pp, px, py);
            const float fpx = (float)px, fpy = (float)py;
            float T = st.T[pp], C0 = st.C0[pp], C1 = st.C1[pp], C2 = st.C2[pp];
            uint32_t last = st.last[pp];
            bool done = false;
            // the batch is walked in groups of 4; the padding slots after the last Gaussian
            // never contribute, so no per-Gaussian bound check is needed
            const int cnt = ((int)min((uint32_t)kBatch, range.y - start) + 3) & ~3;
            const uint32_t base = start - range.x + 1;
            // branch-free blend: a non-contributing Gaussian gets alpha = 0, which leaves T and
            // C bit-identical (T * 1 = T, fma(c, 0, C) = C), so only termination branches
            for (int k4 = 0; k4 < cnt && !done; k4 += 4)
#pragma unroll
            for (int k = k4; k < k4 + 4; ++k) {
                const float4 bx = s.box[k];
                const float4 cn = s.con[k];
                const float4 cl = s.col[k];
                const float q = pixel_q(fpx, fpy, bx.x, bx.y, cn.x, cn.y, cn.z);
                const bool contrib = q <= cn.w;  // alpha >= 1/255 (Eq. 9, R15)
                const float alpha = contrib ? alpha_of(q, cl.w) : 0.0f;
                const float Tn = T * (1.0f - alpha);
                if (Tn < 1e-4f) {  // R16: stop before blending (never for alpha = 0: T >= 1e-4)
                    done = true;
                    break;
                }
                const float w = alpha * T;
                C0 = fmaf(cl.x, w, C0);
                C1 = fmaf(cl.y, w, C1);
                C2 = fmaf(cl.z, w, C2);
                T = Tn;
                if (NC) last = contrib ? base + (uint32_t)k : last;
            }
            st.T[pp] = T;
            st.C0[pp] = C0;
            st.C1[pp] = C1;
            st.C2[pp] = C2;
            if (NC) st.last[pp] = last;
            st.done[pp] = done ? 1 : 0;
        }
    }
    __syncthreads();
    if (inside) {
        const int p0 = threadIdx.x;
        const float T = st.T[p0];
        const size_t p = (size_t)mpy * W + mpx, plane = (size_t)W * H;
        out_rgb[p] = fmaf(T, bg0, st.C0[p0]);
        out_rgb[plane + p] = fmaf(T, bg1, st.C1[p0]);
        out_rgb[2 * plane + p] = fmaf(T, bg2, st.C2[p0]);
        if (out_T) out_T[p] = T;
        if (NC) out_nc[p] = st.last[p0];
    }
}

// a7: forward (T_final, last blended index per pixel), then back-to-front over the tile list
// recovering T_i = T_{i+1} / (1 - alpha_i) and the suffix colour S <- alpha c + (1-alpha) S:
//   dC_ch/dalpha_i = T_i (c_ch - S_ch) - T_final bg_ch / (1 - alpha_i)      (from Eq. 7)
//   U_i += sum_ch (sigma_i dC_ch/dalpha_i)^2                                 (Eqs. 20-21)
// Both walks compact the active pixels per batch like k_render.  Per batch, per-Gaussian
// sums are reduced warp -> CTA in shared memory and added to the float64 score with one
// atomic per (tile, Gaussian).
__global__ void __launch_bounds__(256, 6) k_prune_score(const uint2 *__restrict__ ranges,
                                                     const uint32_t *__restrict__ vals,
                                                     const float4 *__restrict__ rec, int W, int H, int tiles_x,
                                                     float bg0, float bg1, float bg2, double *__restrict__ score,
        const ColorSrc *__restrict__ csp) {
    pdl_enter();
    const ColorSrc cs = *csp;
    __shared__ Batch s;
    __shared__ PixState st;  // forward: T, last, done; backward: T (running), C0..2 = suffix S
    __shared__ float s_Tfin[256];
    __shared__ uint32_t s_id[kBatch];
    __shared__ float s_part[8][kBatch];
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_max;
    const int tile = blockIdx.x;
    int mpx, mpy;
    tile_pixel(tile, tiles_x, threadIdx.x, mpx, mpy);
    const bool inside = mpx < W && mpy < H;
    const uint2 range = ranges[tile];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    st.T[threadIdx.x] = 1.0f;
    st.last[threadIdx.x] = 0;
    st.done[threadIdx.x] = inside ? 0 : 1;
    if (threadIdx.x == 0) s_max = 0;
    // forward
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        __syncthreads();
        const uint32_t n_active = compact_active(!st.done[threadIdx.x], st, s_warp);
        if (n_active == 0) break;
        load_batch(s, vals, rec, start + threadIdx.x, range.y, nullptr, cs);
        __syncthreads();
        if (threadIdx.x < n_active) {
            const int pp = st.list[threadIdx.x];
            int px, py;
            tile_pixel(tile, tiles_x, pp, px, py);
            const float fpx = (float)px, fpy = (float)py;
            float T = st.T[pp];
            uint32_t last = st.last[pp];
            bool done = false;
            // groups of 4 over the padded batch (padding slots never contribute), as in k_render
            const int cnt = ((int)min((uint32_t)kBatch, range.y - start) + 3) & ~3;
            const uint32_t base = start - range.x + 1;
            for (int k4 = 0; k4 < cnt && !done; k4 += 4)
#pragma unroll
            for (int k = k4; k < k4 + 4; ++k) {  // branch-free, as in k_render
                const float4 bx = s.box[k];
                const float4 cn = s.con[k];
                const float q = pixel_q(fpx, fpy, bx.x, bx.y, cn.x, cn.y, cn.z);
                const bool contrib = q <= cn.w;
                const float alpha = contrib ? alpha_of(q, s.col[k].w) : 0.0f;
                const float Tn = T * (1.0f - alpha);
                if (Tn < 1e-4f) {
                    done = true;
                    break;
                }
                T = Tn;
                last = contrib ? base + (uint32_t)k : last;
            }
            st.T[pp] = T;
            st.last[pp] = last;
            st.done[pp] = done ? 1 : 0;
        }
    }
    __syncthreads();
    const uint32_t my_last = st.last[threadIdx.x];
    atomicMax(&s_max, my_last);
    s_Tfin[threadIdx.x] = st.T[threadIdx.x];
    st.C0[threadIdx.x] = st.C1[threadIdx.x] = st.C2[threadIdx.x] = 0.0f;
    __syncthreads();
    const uint32_t max_last = s_max;
    // backward, batches from the end; a pixel is active in [start, end) iff last > start
    for (uint32_t end = range.x + max_last; end > range.x;) {
        const uint32_t start = end - range.x > (uint32_t)kBatch ? end - kBatch : range.x;
        const int cnt = (int)(end - start);
        __syncthreads();
        const uint32_t n_active = compact_active(my_last > start - range.x, st, s_warp);
        load_batch(s, vals, rec, start + threadIdx.x, end, s_id, cs);
        __syncthreads();
        const uint32_t n_warps = (n_active + 31) / 32;
        if ((uint32_t)warp < n_warps) {
            const bool act = threadIdx.x < n_active;
            const int pp = act ? st.list[threadIdx.x] : 0;
            int px, py;
            tile_pixel(tile, tiles_x, pp, px, py);
            const float fpx = (float)px, fpy = (float)py;
            const uint32_t plast = act ? st.last[pp] : 0u;
            const float Tfin = s_Tfin[pp];
            float T = act ? st.T[pp] : 1.0f;
            float S0 = st.C0[pp], S1 = st.C1[pp], S2 = st.C2[pp];
            for (int k = cnt - 1; k >= 0; --k) {
                float term = 0.f;
                if (start - range.x + (uint32_t)k < plast) {
                    const float4 bx = s.box[k];
                    const float4 cn = s.con[k];
                    const float q = pixel_q(fpx, fpy, bx.x, bx.y, cn.x, cn.y, cn.z);
                    if (q <= cn.w) {
                        const float4 cl = s.col[k];
                        const float alpha = alpha_of(q, cl.w);
                        const float om = 1.0f - alpha;
                        float rom;  // T_i = T_{i+1} / (1 - alpha_i): one approximate reciprocal
                        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rom) : "f"(om));
                        T = T * rom;
                        const float bgs = Tfin * rom;
                        const float d0 = T * (cl.x - S0) - bgs * bg0;
                        const float d1 = T * (cl.y - S1) - bgs * bg1;
                        const float d2 = T * (cl.z - S2) - bgs * bg2;
                        term = cl.w * cl.w * (d0 * d0 + d1 * d1 + d2 * d2);
                        S0 = alpha * cl.x + om * S0;
                        S1 = alpha * cl.y + om * S1;
                        S2 = alpha * cl.z + om * S2;
                    }
                }
                if (__any_sync(0xffffffffu, term != 0.f)) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
                }
                if (lane == 0) s_part[warp][k] = term;
            }
            if (act) {
                st.T[pp] = T;
                st.C0[pp] = S0;
                st.C1[pp] = S1;
                st.C2[pp] = S2;
            }
        }
        __syncthreads();
        if ((int)threadIdx.x < cnt) {
            float sum = 0.f;
            for (uint32_t w = 0; w < n_warps; ++w) sum += s_part[w][threadIdx.x];
            if (sum != 0.f) atomicAdd(score + s_id[threadIdx.x], (double)sum);
        }
        end = start;
    }
}

// NEXT-2 render backward ("the per-pixel gradients from the render kernel are
// parallelized and aggregated to the 2D mu_2D and Sigma_2D parameters").  One CTA per tile,
// one thread per pixel, walking the tile list back to front from the pixel's last blended
// entry (n_contrib of ss_render) with T recovered as T_i = T_{i+1} / (1 - alpha_i) and the
// suffix colour S <- alpha c + (1 - alpha) S (a7's recursion):
//   dL/dalpha_i = sum_ch dL/dC_ch (T_i (c_ch - S_ch) - T_final bg_ch / (1 - alpha_i))
//   dL/dc_i     = dL/dC alpha_i T_i
//   unclamped alpha = sigma G:  dL/dsigma = dL/dalpha G,  dL/dq = -dL/dalpha alpha / 2,
//   dq/dx2d = -2 (a dx + b dy), dq/dy2d = -2 (b dx + c dy), dq/d(a, b, c) = (dx^2, 2 dx dy, dy^2)
// (a clamped alpha passes nothing to sigma and the geometry, reading R27).  The alpha of
// every entry is recomputed with k_render's exact operations, so the blended set is the
// forward's.  Per batch, each warp reduces a Gaussian's 9 partials by shuffles (only when
// one of its pixels contributes) into per-warp shared-memory slots; the CTA then adds each
// Gaussian's sums to grad2d with three float4 atomics (one set per (tile, Gaussian)).
__global__ void __launch_bounds__(256) k_render_backward(const uint2 *__restrict__ ranges,
                                                         const uint32_t *__restrict__ vals,
                                                         const float4 *__restrict__ rec, int W, int H, int tiles_x,
                                                         float bg0, float bg1, float bg2,
                                                         const float *__restrict__ dimg,
                                                         const float *__restrict__ T_final,
                                                         const uint32_t *__restrict__ n_contrib,
                                                         float4 *__restrict__ grad2d,
        const ColorSrc *__restrict__ csp) {
    pdl_enter();
    const ColorSrc cs = *csp;
    __shared__ Batch s;
    __shared__ PixState st;  // T (running), C0..2 = suffix S, last = n_contrib
    __shared__ float s_dC[3][256];
    __shared__ float s_Tfin[256];
    __shared__ uint32_t s_id[kBatch];
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_max;
    extern __shared__ float s_part[];              // [8 warps][kBatch][9] per-warp partial sums
    const int tile = blockIdx.x;
    int mpx, mpy;
    tile_pixel(tile, tiles_x, threadIdx.x, mpx, mpy);
    const bool inside = mpx < W && mpy < H;
    const uint2 range = ranges[tile];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_max = 0;
    const size_t pix = (size_t)mpy * W + mpx, plane = (size_t)W * H;
    const uint32_t my_last = inside ? n_contrib[pix] : 0u;
    st.last[threadIdx.x] = my_last;
    st.T[threadIdx.x] = s_Tfin[threadIdx.x] = inside ? T_final[pix] : 1.0f;
    st.C0[threadIdx.x] = st.C1[threadIdx.x] = st.C2[threadIdx.x] = 0.0f;
    s_dC[0][threadIdx.x] = inside ? dimg[pix] : 0.0f;
    s_dC[1][threadIdx.x] = inside ? dimg[plane + pix] : 0.0f;
    s_dC[2][threadIdx.x] = inside ? dimg[2 * plane + pix] : 0.0f;
    __syncthreads();
    if (my_last) atomicMax(&s_max, my_last);
    __syncthreads();
    const uint32_t max_last = min(s_max, range.y - range.x);
    for (uint32_t end = range.x + max_last; end > range.x;) {
        const uint32_t start = end - range.x > (uint32_t)kBatch ? end - kBatch : range.x;
        const int cnt = (int)(end - start);
        __syncthreads();
        const uint32_t n_active = compact_active(my_last > start - range.x, st, s_warp);
        load_batch(s, vals, rec, start + threadIdx.x, end, s_id, cs);
        __syncthreads();
        const uint32_t n_warps = (n_active + 31) / 32;
        const int warp = threadIdx.x >> 5;
        if ((uint32_t)warp < n_warps) {
            const bool act = threadIdx.x < n_active;
            const int pp = act ? st.list[threadIdx.x] : 0;
            int px, py;
            tile_pixel(tile, tiles_x, pp, px, py);
            const float fpx = (float)px, fpy = (float)py;
            const uint32_t plast = act ? st.last[pp] : 0u;
            const float Tfin = s_Tfin[pp];
            float *wpart = s_part + (size_t)warp * kBatch * 9;
            const float dC0 = s_dC[0][pp], dC1 = s_dC[1][pp], dC2 = s_dC[2][pp];
            float T = st.T[pp];
            float S0 = st.C0[pp], S1 = st.C1[pp], S2 = st.C2[pp];
            for (int k = cnt - 1; k >= 0; --k) {
                float g[9];
#pragma unroll
                for (int f = 0; f < 9; ++f) g[f] = 0.0f;
                bool any = false;
                if (start - range.x + (uint32_t)k < plast) {
                    const float4 bx = s.box[k];
                    const float4 cn = s.con[k];
                    const float q = pixel_q(fpx, fpy, bx.x, bx.y, cn.x, cn.y, cn.z);
                    if (q <= cn.w) {
                        const float4 cl = s.col[k];
                        float e;
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(q * -0.72134752044448170f));
                        const float raw = cl.w * e;
                        const float alpha = fminf(0.99f, raw);  // == alpha_of(q, sigma)
                        const float om = 1.0f - alpha;
                        float rom;  // T_i = T_{i+1} / (1 - alpha_i)
                        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rom) : "f"(om));
                        T = T * rom;
                        const float bgs = Tfin * rom;
                        const float dLda = dC0 * (T * (cl.x - S0) - bgs * bg0) + dC1 * (T * (cl.y - S1) - bgs * bg1) +
                                           dC2 * (T * (cl.z - S2) - bgs * bg2);
                        const float w = alpha * T;
                        g[6] = dC0 * w;
                        g[7] = dC1 * w;
                        g[8] = dC2 * w;
                        if (raw <= 0.99f) {
                            // per pixel A = dL/dq dx, B = dL/dq dy; the CTA sums give
                            // dL/dx2d = -2 (a SA + b SB), dL/dy2d = -2 (b SA + c SB),
                            // dL/d(a, b, c) = (S A dx, 2 S A dy, S B dy)
                            const float dx = fpx - bx.x, dy = fpy - bx.y;
                            const float dLdq = -0.5f * dLda * alpha;
                            const float A = dLdq * dx, B = dLdq * dy;
                            g[0] = A;
                            g[1] = B;
                            g[2] = A * dx;
                            g[3] = A * dy;
                            g[4] = B * dy;
                            g[5] = dLda * e;
                        }
                        S0 = alpha * cl.x + om * S0;
                        S1 = alpha * cl.y + om * S1;
                        S2 = alpha * cl.z + om * S2;
                        any = true;
                    }
                }
                if (__any_sync(0xffffffffu, any)) {
                    // transpose-reduce of fields 0..7 (4 + 2 + 1 + 1 + 1 shuffles): afterwards
                    // lane L (L & 3 == 0) holds the warp sum of field ((L >> 2) & 7); field 8
                    // by a plain butterfly (5 shuffles)
                    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
                    float v4[4], v2[2];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float send = h16 ? g[j] : g[4 + j];
                        v4[j] = (h16 ? g[4 + j] : g[j]) + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const float send = h8 ? v4[j] : v4[2 + j];
                        v2[j] = (h8 ? v4[2 + j] : v4[j]) + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
                    float v1 = (h4 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? v2[0] : v2[1], 4);
                    v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
                    v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
                    float v8 = g[8];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v8 += __shfl_xor_sync(0xffffffffu, v8, o);
                    if ((lane & 3) == 0) wpart[k * 9 + ((lane >> 2) & 7)] = v1;
                    if (lane == 1) wpart[k * 9 + 8] = v8;
                } else {
                    if ((lane & 3) == 0) wpart[k * 9 + ((lane >> 2) & 7)] = 0.0f;
                    if (lane == 1) wpart[k * 9 + 8] = 0.0f;
                }
            }
            if (act) {
                st.T[pp] = T;
                st.C0[pp] = S0;
                st.C1[pp] = S1;
                st.C2[pp] = S2;
            }
        }
        __syncthreads();
        if ((int)threadIdx.x < cnt) {
            const int k = threadIdx.x;
            float a[9];
#pragma unroll
            for (int f = 0; f < 9; ++f) a[f] = 0.0f;
            for (uint32_t w = 0; w < n_warps; ++w) {
                const float *src = s_part + ((size_t)w * kBatch + k) * 9;
#pragma unroll
                for (int f = 0; f < 9; ++f) a[f] += src[f];
            }
            const float4 cn = s.con[k];  // a, 2b, c, t of the Gaussian
            const float b = 0.5f * cn.y;
            const float4 a0 = make_float4(-2.0f * (cn.x * a[0] + b * a[1]), -2.0f * (b * a[0] + cn.z * a[1]), a[2],
                                          2.0f * a[3]);
            const float4 a1 = make_float4(a[4], a[5], a[6], a[7]);
            const float a2 = a[8];
            bool hit = false;
#pragma unroll
            for (int f = 0; f < 9; ++f) hit |= a[f] != 0.0f;
            if (hit) {
                float4 *gp = grad2d + 3 * (size_t)s_id[k];
                atomicAdd(gp + 0, a0);
                atomicAdd(gp + 1, a1);
                atomicAdd(&gp[2].x, a2);
            }
        }
        end = start;
    }
}

// Measurement only (not on the timed path): the render's work counts for one frame, from
// the same per-pixel walk as k_render.  counters[0] += E_pix (evaluations each pixel makes
// until it terminates, the method's work), [1] += E_blend (evaluations that blend),
// [2] += E_cta (evaluations a CTA issues in lock-step until its last pixel terminates:
// 256 x Gaussians staged), [3] += pixels; [4] is reserved (left 0).
__global__ void __launch_bounds__(256) k_render_stats(const uint2 *__restrict__ ranges,
                                                      const uint32_t *__restrict__ vals,
                                                      const float4 *__restrict__ rec, int W, int H, int tiles_x,
                                                      unsigned long long *counters,
        const ColorSrc *__restrict__ csp) {
    const ColorSrc cs = *csp;
    __shared__ Batch s;
    __shared__ unsigned long long s_acc[5];
    const int tile = blockIdx.x;
    int px, py;
    tile_pixel(tile, tiles_x, threadIdx.x, px, py);
    const bool inside = px < W && py < H;
    const float fpx = (float)px, fpy = (float)py;
    const uint2 range = ranges[tile];
    bool done = !inside;
    float T = 1.0f;
    unsigned long long e_pix = 0, e_blend = 0, e_cta = 0;
    if (threadIdx.x < 5) s_acc[threadIdx.x] = 0;
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        if (__syncthreads_count(done) == blockDim.x) break;
        load_batch(s, vals, rec, start + threadIdx.x, range.y, nullptr, cs);
        __syncthreads();
        const int cnt = min((uint32_t)kBatch, range.y - start);
        e_cta += cnt;
        // compacted warps: ceil(active / 32) warps walk until their last pixel terminates
        for (int k = 0; k < cnt && !done; ++k) {
            ++e_pix;
            const float4 bx = s.box[k];
            const float4 cn = s.con[k];
            const float q = pixel_q(fpx, fpy, bx.x, bx.y, cn.x, cn.y, cn.z);
            if (!(q <= cn.w)) continue;
            const float alpha = alpha_of(q, s.col[k].w);
            const float Tn = T * (1.0f - alpha);
            if (Tn < 1e-4f) {
                done = true;
                break;
            }
            ++e_blend;
            T = Tn;
        }
    }
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e_pix += __shfl_xor_sync(0xffffffffu, e_pix, o);
        e_blend += __shfl_xor_sync(0xffffffffu, e_blend, o);
    }
    const unsigned n_inside = __syncthreads_count(inside);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_acc[0], e_pix);
        atomicAdd(&s_acc[1], e_blend);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(counters + 0, s_acc[0]);
        atomicAdd(counters + 1, s_acc[1]);
        atomicAdd(counters + 2, e_cta * blockDim.x);
        atomicAdd(counters + 3, (unsigned long long)n_inside);
    }
}

}  // namespace

namespace {
// Colours still pending after the frame's kernels (Gaussians no tile reached): inspection only.
__global__ void __launch_bounds__(256) k_finalize_colours(int n, const uint32_t *__restrict__ depth_key,
                                                          const float4 *rec, const ColorSrc *__restrict__ csp) {
    pdl_enter();
    const ColorSrc cs = *csp;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && depth_key[i] != kNoTiles) record_colour(rec, (uint32_t)i, cs);
}
}  // namespace

cudaError_t launch_finalize_colours(void *ws, const Layout &L, cudaStream_t st) {
    if (L.n == 0) return cudaSuccess;
    launch_pdl(k_finalize_colours, (L.n + 255) / 256, 256, 0, st, (int)L.n, at<const uint32_t>(ws, L.pub.depth_key),
               at<const float4>(ws, L.pub.rec), at<const ColorSrc>(ws, L.color_src));
    return cudaGetLastError();
}

cudaError_t launch_render_stats(void *ws, const Layout &L, int W, int H, unsigned long long *counters,
                                cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    k_render_stats<<<P.n_tiles, 256, 0, st>>>(at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                               at<const float4>(ws, P.rec), W, H, P.tiles_x, counters, at<const ColorSrc>(ws, L.color_src));
    return cudaGetLastError();
}

cudaError_t launch_render(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2, float *out_rgb,
                          float *out_T, uint32_t *out_nc, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    if (out_nc)
        launch_pdl(k_render<true>, P.n_tiles, 256, 0, st, at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                                   at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2, out_rgb,
                                                   out_T, out_nc, at<const ColorSrc>(ws, L.color_src));
    else
        launch_pdl(k_render<false>, P.n_tiles, 256, 0, st, at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                                    at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2, out_rgb,
                                                    out_T, out_nc, at<const ColorSrc>(ws, L.color_src));
    return cudaGetLastError();
}

cudaError_t launch_render_backward(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2,
                                   const float *dimg, const float *T_final, const uint32_t *n_contrib, float *grad2d,
                                   cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    static int smem_done[64] = {0};
    const size_t smem = sizeof(float) * 8 * kBatch * 9;
    cudaError_t e = ensure_smem(k_render_backward, smem, smem_done);
    if (e != cudaSuccess) return e;
    launch_pdl(k_render_backward, P.n_tiles, 256, smem, st, at<const uint2>(ws, P.ranges),
               at<const uint32_t>(ws, P.sorted_value), at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2,
               dimg, T_final, n_contrib, reinterpret_cast<float4 *>(grad2d), at<const ColorSrc>(ws, L.color_src));
    return cudaGetLastError();
}

cudaError_t launch_prune_score(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2,
                               double *score, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    launch_pdl(k_prune_score, P.n_tiles, 256, 0, st, at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                              at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2, score,
                                              at<const ColorSrc>(ws, L.color_src));
    return cudaGetLastError();
}

}  // namespace ss
