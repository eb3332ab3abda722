// ss_render.cu -- a6 render (Eqs. 5-7), a7 efficient pruning score (Eqs. 20-21) and the
// NEXT-2 render backward.
//
// One CTA per 16x16 tile, one thread per pixel ("parallelized across pixels").  The
// tile's depth-ordered Gaussian ids are consumed in batches of kBatch = 128.  k_render stages
// them asynchronously: while the pixels walk batch b, one thread per slot has batch b+1's
// 48 B records in flight (cp.async, LDGSTS) and batch b+2's ids loaded; a landed batch is
// transposed into a pair-interleaved layout (computing the view-dependent colour on first use,
// ss_color.cuh) so that the q / alpha chain of two consecutive Gaussians runs on the packed
// FP32 pipe (FFMA2 / FMUL2 / FADD2).  Before every batch the active pixels are compacted onto
// the lowest threads (two barriers per batch); a CTA stops as soon as none is left.  The
// score / backward / stats kernels gather synchronously (load_batch).
//
// Arithmetic contract: the alpha-skip decision q <= t (alpha >= 1/255, Eq. 9)
// uses the pinned chain u = fma(a, dx, (2b) dy); q = fma(dx, u, (c dy) dy) with explicit
// round-to-nearest intrinsics, so it is bit-identical to the oracle's; alpha uses the SFU
// exp2 (ex2.approx), which the image tolerance (1e-4) covers.
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ss_color.cuh"

namespace ss {
namespace {

constexpr int kBatch = 128;
#ifndef SS_RENDER_MINB
#define SS_RENDER_MINB 6  // k_render CTAs per SM (register budget 40)
#endif
#ifndef SS_RENDER_UNROLL
#define SS_RENDER_UNROLL 2
#endif
constexpr int kRenderUnroll = SS_RENDER_UNROLL;  // pairs per k_render loop iteration
#ifndef SS_RENDER_PIX
#define SS_RENDER_PIX 256
#endif
#ifndef SS_RENDER_BATCH
#define SS_RENDER_BATCH 128
#endif
constexpr int kRenderPix = SS_RENDER_PIX;      // pixels per k_render CTA (256: a tile, 128: half a tile)
constexpr int kRenderBatch = SS_RENDER_BATCH;  // Gaussians per k_render batch
// Batch staging of k_render: cp.async (default) or TMA gather4 (SS_RENDER_STAGING=tma in the
// environment, read per launch; both variants are compiled in).
static bool render_tma() {
    const char *v = std::getenv("SS_RENDER_STAGING");
    return v && std::strcmp(v, "tma") == 0;
}

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
// The same from the tile's first pixel (tx0, ty0) (tile_pixel of pixel 0): no division in
// the per-batch loops.
__device__ __forceinline__ void tile_pixel_at(int tx0, int ty0, int p, int &px, int &py) {
    px = tx0 + (p & 15);
    py = ty0 + (p >> 4);
}

// Per-pixel state kept in shared memory between batches, so that before every batch the
// still-active pixels can be compacted onto the lowest threads: warps whose pixels have all
// terminated stop issuing, instead of idling lane by lane inside partially-done warps
// (the per-pixel walk and its arithmetic are unchanged).
template <int PIX>
struct PixStateT {
    float T[PIX], C0[PIX], C1[PIX], C2[PIX];
    uint32_t last[PIX];
    uint8_t done[PIX];
    uint16_t list[PIX];
};
using PixState = PixStateT<256>;

// Compacts the active pixels (one flag per thread = pixel threadIdx.x) into st.list; returns
// their number.  Every thread of the CTA must call it.
__device__ __forceinline__ uint32_t compact_active(bool active, PixState &st, uint32_t *s_warp) {
    uint32_t n_active;
    const uint32_t pos = block_exclusive_scan_256(active ? 1u : 0u, s_warp, n_active);
    if (active) st.list[pos] = (uint16_t)threadIdx.x;
    __syncthreads();
    return n_active;
}

// ---------------------------------------------------------------- staged batches (k_render)
// Records of batch b+1 are gathered with cp.async (LDGSTS, 3 x 16 B per slot, L2 path) into a
// raw double buffer while the pixels walk batch b; the ids are loaded two batches ahead.  When
// a batch has landed its loader thread transposes its slot into structure-of-arrays form
// (computing a pending colour, ss_color.cuh), so that one 128-bit shared load gives a field of
// four consecutive Gaussians and consecutive pairs feed the packed FP32 pipe (f32x2).
template <int B>
struct RawBatchT {
    float4 q[3 * B];  // records as gathered: q0, q1, q2 per slot
};
using RawBatch = RawBatchT<kBatch>;
// Pair-interleaved (AoSoA) layout: Gaussians 2p and 2p+1 share 20 floats, so that one 128-bit
// shared load gives two fields of the pair as two f32x2 operands, and the (r, g) of each
// Gaussian as one f32x2 operand (the score walk's channel pairs):
//   [-x0 -x1 -y0 -y1] [a0 a1 2b0 2b1] [c0 c1 t0 t1] [s0 s1 r0 g0] [r1 g1 bl0 bl1]
template <int B>
struct SoaBatchT {
    float4 v[B / 2][5];
};
using SoaBatch = SoaBatchT<kBatch>;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Slot threadIdx.x (< kBatch) of a batch: issue the gather of Gaussian g's record.
template <int B>
__device__ __forceinline__ void stage_gather(RawBatchT<B> &raw, const float4 *__restrict__ rec, uint32_t g, bool valid) {
    if (valid) {
        const float4 *src = rec + 3 * (size_t)g;
        cp_async16(&raw.q[3 * threadIdx.x + 0], src + 0);
        cp_async16(&raw.q[3 * threadIdx.x + 1], src + 1);
        cp_async16(&raw.q[3 * threadIdx.x + 2], src + 2);
    }
}

// Slot threadIdx.x (< kBatch): raw record -> pair-interleaved layout (padding slots never
// contribute: q <= -inf is false); a pending colour is computed here and stored back.
template <int B>
__device__ __forceinline__ void stage_transpose_rows(SoaBatchT<B> &s, const float4 *row, const float4 *rec, uint32_t g,
                                                     bool valid, const ColorSrc &cs) {
    const int k = threadIdx.x;
    float f[10];
    if (valid) {
        const float4 q0 = row[0], q1 = row[1];
        float4 q2 = row[2];
        if (q2.x == 0.0f) {  // pending colour: computed by this gather (the same value every time)
            const float3 c = sh_color(cs, g);
            q2 = make_float4(1.0f, c.x, c.y, c.z);
            __stcg(const_cast<float4 *>(rec) + 3 * (size_t)g + 2, q2);
        }
        f[0] = -q0.x; f[1] = -q0.y; f[2] = q0.z; f[3] = q0.w + q0.w; f[4] = q1.x;
        f[5] = q1.y; f[6] = q1.z; f[7] = q2.y; f[8] = q2.z; f[9] = q2.w;
    } else {
        f[0] = f[1] = 0.0f; f[2] = 1.0f; f[3] = 0.0f; f[4] = 1.0f;
        f[5] = __int_as_float(0xff800000); f[6] = f[7] = f[8] = f[9] = 0.0f;
    }
    float *dst = reinterpret_cast<float *>(&s.v[k >> 1][0]);
    const int h = k & 1;
#pragma unroll
    for (int j = 0; j < 7; ++j) dst[2 * j + h] = f[j];  // -x, -y, a, 2b, c, t, sigma
    dst[h ? 16 : 14] = f[7];                            // r
    dst[h ? 17 : 15] = f[8];                            // g
    dst[18 + h] = f[9];                                 // b
}

template <int B>
__device__ __forceinline__ void stage_transpose(SoaBatchT<B> &s, const RawBatchT<B> &raw, const float4 *rec, uint32_t g,
                                                bool valid, const ColorSrc &cs) {
    stage_transpose_rows(s, &raw.q[3 * threadIdx.x], rec, g, valid, cs);
}

// ---- TMA (cp.async.bulk.tensor ... tile::gather4) staging of a batch: one warp issues B / 4
// gathers of 4 record rows (48 B each) into 256 B-aligned slots of a buffer; an mbarrier per
// buffer counts the bytes.
template <int B>
struct TmaBatchT {
    float4 q[B / 4][16];  // 4 rows x 3 float4 per gather, padded to 256 B
};
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *tm, uint64_t *m, int r0, int r1, int r2,
                                            int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(m)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
    return e;
}

// PIX pixels per CTA (256: a whole tile; 128: half a tile, rows 8 h .. 8 h + 7 of tile
// blockIdx.x / 2, so that fewer warps wait at each batch barrier), B Gaussians per batch.
// TMA: stage the batches with cp.async.bulk.tensor ... tile::gather4 (UTMALDG; one warp issues
// the B / 4 gathers of a batch, an mbarrier per buffer) instead of per-slot cp.async (LDGSTS).
template <bool NC, int PIX, int B, bool TMA>  // NC: track the last blended list entry per pixel (out_ncontrib)
__global__ void __launch_bounds__(PIX, SS_RENDER_MINB * 256 / PIX) k_render(const uint2 *__restrict__ ranges, const uint32_t *__restrict__ vals,
                                                const float4 *__restrict__ rec, int W, int H, int tiles_x, float bg0,
                                                float bg1, float bg2, float *__restrict__ out_rgb,
                                                float *__restrict__ out_T, uint32_t *__restrict__ out_nc,
        const ColorSrc *__restrict__ csp, const __grid_constant__ CUtensorMap tmap) {
    pdl_enter();
    const ColorSrc cs = *csp;
    constexpr int NW = PIX / 32;
    __shared__ __align__(16) RawBatchT<TMA ? 4 : B> raw[2];
    __shared__ __align__(256) TmaBatchT<TMA ? B : 4> tb[2];
    __shared__ uint32_t s_gid[2][TMA ? B : 1];
    __shared__ __align__(8) uint64_t s_mbar[2];
    __shared__ __align__(16) SoaBatchT<B> s;
    __shared__ PixStateT<PIX> st;
    __shared__ uint32_t s_warp[NW];
    const int tile = PIX == 256 ? blockIdx.x : blockIdx.x >> 1;
    const int p0 = PIX == 256 ? 0 : (blockIdx.x & 1) * PIX;  // first tile pixel of this CTA
    const int tid = threadIdx.x;
    int mpx, mpy;
    tile_pixel(tile, tiles_x, p0 + tid, mpx, mpy);
    int tx0, ty0;
    tile_pixel(tile, tiles_x, 0, tx0, ty0);
    const bool inside = mpx < W && mpy < H;
    const uint2 range = ranges[tile];
    st.T[tid] = 1.0f;
    st.C0[tid] = st.C1[tid] = st.C2[tid] = 0.0f;
    st.last[tid] = 0;
    // ids of batches 0 and 1 of this slot; batch 0 gathered before the loop
    const bool loader = tid < B;
    uint32_t g_cur = 0, g_nxt = 0;
    uint32_t g4[4] = {0u, 0u, 0u, 0u};  // TMA: warp 0 lane l holds the ids of slots 4l..4l+3 of the next batch
    const int lane = tid & 31;
    // TMA: warp 0 stages the batch at list position bs (ids in g4) into buffer sb
    auto tma_issue = [&](uint32_t bs, int sb) {
        const uint32_t n_slots = min((uint32_t)B, range.y - bs);
        const uint32_t n_g = (n_slots + 3) / 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) s_gid[sb][4 * lane + q] = g4[q];
        if (lane == 0) mbar_expect_tx(&s_mbar[sb], n_g * 192u);
        __syncwarp();
        if ((uint32_t)lane < n_g) tma_gather4(&tb[sb].q[lane][0], &tmap, &s_mbar[sb], (int)g4[0], (int)g4[1], (int)g4[2], (int)g4[3]);
    };
    auto tma_load_ids = [&](uint32_t bs) {  // ids of the batch at bs (invalid slots repeat a valid id)
        const uint32_t n_slots = bs < range.y ? min((uint32_t)B, range.y - bs) : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t k = 4 * lane + q;
            g4[q] = k < n_slots ? __ldg(vals + bs + k) : (n_slots ? __ldg(vals + bs) : 0u);
        }
    };
    if constexpr (TMA) {
        if (tid == 0) {
            mbar_init(&s_mbar[0], 1);
            mbar_init(&s_mbar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid < 32) {
            tma_load_ids(range.x);
            if (range.x < range.y) tma_issue(range.x, 0);
            tma_load_ids(range.x + B);  // the next batch's ids
        }
    } else {
        if (loader) {
            const uint32_t j0 = range.x + tid, j1 = j0 + B;
            g_cur = j0 < range.y ? __ldg(vals + j0) : 0u;
            g_nxt = j1 < range.y ? __ldg(vals + j1) : 0u;
            stage_gather(raw[0], rec, g_cur, j0 < range.y);
        }
        cp_async_commit();
    }
    uint32_t n_uses = 0;     // TMA: batches staged into buffer 0 / 1 so far (parity of the next wait)
    bool in_flight = false;  // TMA: a batch issued but not consumed when the loop ends
    // Pixel compaction, two barriers per batch: every thread carries the pixel it walked (my_pp)
    // and whether it is still active (my_act); per-warp counts of the active ones are published
    // with the barrier that ends the walk, and the next list (stable: pixel-index order) is
    // written from registers.  Warps whose pixels have all terminated stop issuing.
    uint32_t my_pp = (uint32_t)tid;
    bool my_act = inside;
    uint32_t bal = __ballot_sync(0xffffffffu, my_act);
    if ((tid & 31) == 0) s_warp[tid >> 5] = __popc(bal);
    int buf = 0;
    for (uint32_t start = range.x; start < range.y; start += B, buf ^= 1) {
        __syncthreads();  // the previous walk is done: s, raw[buf ^ 1] free; warp counts visible
        uint32_t n_active = 0, pos = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t c = s_warp[w];
            pos += w < (tid >> 5) ? c : 0u;
            n_active += c;
        }
        if (n_active == 0) break;
        if (my_act) st.list[pos + __popc(bal & ((1u << (tid & 31)) - 1u))] = (uint16_t)my_pp;
        if constexpr (TMA) {
            in_flight = start + B < range.y;
            if (tid < 32 && in_flight) {
                tma_issue(start + B, buf ^ 1);  // batch b+1, in flight
                tma_load_ids(start + 2 * B);    // ids of batch b+2
            }
            if (loader) {
                mbar_wait(&s_mbar[buf], (n_uses >> 1) & 1u);  // batch b has landed (buffer buf, use n_uses / 2)
                const int k = tid;
                const float4 *row = &tb[buf].q[k >> 2][(k & 3) * 3];
                stage_transpose_rows(s, row, rec, s_gid[buf][k], start + tid < range.y, cs);
            }
            ++n_uses;
        } else {
            uint32_t g_after = 0;
            if (loader) {
                const uint32_t j1 = start + B + tid, j2 = j1 + B;
                stage_gather(raw[buf ^ 1], rec, g_nxt, j1 < range.y);           // batch b+1, in flight
                g_after = j2 < range.y ? __ldg(vals + j2) : 0u;                 // id of batch b+2
            }
            cp_async_commit();
            cp_async_wait<1>();  // this thread's gathers of batch b have landed
            if (loader) stage_transpose(s, raw[buf], rec, g_cur, start + tid < range.y, cs);
            g_cur = g_nxt;
            g_nxt = g_after;
        }
        __syncthreads();  // batch b staged, the list written
        my_act = false;
        if (tid < n_active) {
            const int pp = st.list[tid];
            int px, py;
            tile_pixel_at(tx0, ty0, p0 + pp, px, py);
            const float2 FX = f2((float)px), FY = f2((float)py);
            // colour sums: (r, g) as one f32x2 (each lane the channel's own sequential FMA chain),
            // b scalar
            float T = st.T[pp], C2 = st.C2[pp];
            float2 C01 = make_float2(st.C0[pp], st.C1[pp]);
            uint32_t last = st.last[pp];
            bool done = false;
            // pairs of consecutive Gaussians over the padded batch (padding slots never
            // contribute).  The q / alpha chain of a pair runs on the packed FP32 pipe (f32x2;
            // each half rounded as the scalar op, so q is bit-identical to the oracle's chain,
            // R15).  A non-contributing Gaussian gets alpha = 0, which leaves T unchanged.  T is
            // monotone, so when T after the pair is >= 1e-4 neither Gaussian terminates and both
            // blend (the common case: one test per pair); otherwise the pair is taken in order.
            // The colour sums stay sequential (C += c alpha T in list order), so the image is
            // bit-identical to a one-by-one walk: AccuTile and SnugBox renders stay bitwise equal
            // (their lists differ only by Gaussians with alpha = 0 everywhere in the tile).
            const int cnt = ((int)min((uint32_t)B, range.y - start) + 1) & ~1;
            const uint32_t base = start - range.x + 1;
            // the pair's 5 float4 by 32-bit shared addresses stepped per pair (the generic
            // pointer's window base was rematerialised every iteration at 40 registers)
            // (the loop runs on the address alone; the list index kk only feeds n_contrib)
            const uint32_t va0 = smem_u32(&s.v[0][0]);
            const uint32_t vend = va0 + (uint32_t)(cnt >> 1) * (5 * 16);
            uint32_t kk = base;  // list index (1-based) of the pair's even Gaussian
#pragma unroll kRenderUnroll
            for (uint32_t va = va0; va < vend; va += 5 * 16, kk += 2) {
                const float4 v0 = lds128(va), v1 = lds128(va + 16), v2 = lds128(va + 32);
                // q = (p - mu)^T Sigma^-1 (p - mu): dx = px - x, u = fma(a, dx, 2b dy),
                // q = fma(dx, u, (c dy) dy)
                const float2 dx = __fadd2_rn(FX, make_float2(v0.x, v0.y));
                const float2 dy = __fadd2_rn(FY, make_float2(v0.z, v0.w));
                const float2 u = __ffma2_rn(make_float2(v1.x, v1.y), dx, __fmul2_rn(make_float2(v1.z, v1.w), dy));
                const float2 q = __ffma2_rn(dx, u, __fmul2_rn(__fmul2_rn(make_float2(v2.x, v2.y), dy), dy));
                const float2 ql = __fmul2_rn(q, f2(-0.72134752044448170f));  // -q/2 in log2 units
                const float4 v3 = lds128(va + 48);
                const float2 se = __fmul2_rn(make_float2(v3.x, v3.y), make_float2(ex2_approx(ql.x), ex2_approx(ql.y)));
                const float2 al = make_float2(q.x <= v2.z ? fminf(0.99f, se.x) : 0.0f,   // alpha >= 1/255
                                              q.y <= v2.w ? fminf(0.99f, se.y) : 0.0f);  // (R15, R16)
                const float2 om = __fadd2_rn(f2(1.0f), make_float2(-al.x, -al.y));
                const float T1 = T * om.x, T2 = T1 * om.y;
                const float4 v4 = lds128(va + 64);
                if (T2 < 1e-4f) {  // R16: a Gaussian of the pair terminates the pixel, before blending
                    if (T1 >= 1e-4f) {  // the even one still blends
                        const float w = al.x * T;
                        C01 = __ffma2_rn(make_float2(v3.z, v3.w), f2(w), C01);
                        C2 = fmaf(v4.z, w, C2);
                        T = T1;
                        if (NC) last = al.x > 0.0f ? kk : last;
                    }
                    done = true;
                    break;
                }
                const float2 w = __fmul2_rn(al, make_float2(T, T1));
                C01 = __ffma2_rn(make_float2(v4.x, v4.y), f2(w.y), __ffma2_rn(make_float2(v3.z, v3.w), f2(w.x), C01));
                C2 = fmaf(v4.w, w.y, fmaf(v4.z, w.x, C2));
                T = T2;
                if (NC) last = al.y > 0.0f ? kk + 1 : (al.x > 0.0f ? kk : last);
            }
            st.T[pp] = T;
            st.C0[pp] = C01.x;
            st.C1[pp] = C01.y;
            st.C2[pp] = C2;
            if (NC) st.last[pp] = last;
            my_pp = (uint32_t)pp;
            my_act = !done;
        }
        bal = __ballot_sync(0xffffffffu, my_act);
        if ((tid & 31) == 0) s_warp[tid >> 5] = __popc(bal);
    }
    if constexpr (TMA) {
        // a batch issued but never consumed (the pixels saturated): let it land before the CTA
        // exits (its shared memory is the TMA destination)
        if (tid == 0 && in_flight) mbar_wait(&s_mbar[n_uses & 1], (n_uses >> 1) & 1u);
    } else {
        cp_async_wait<0>();
    }
    __syncthreads();
    if (inside) {
        const float T = st.T[tid];
        const size_t p = (size_t)mpy * W + mpx, plane = (size_t)W * H;
        if (out_rgb) {  // null: ss_prune_score's forward (T_final and n_contrib only)
            out_rgb[p] = fmaf(T, bg0, st.C0[tid]);
            out_rgb[plane + p] = fmaf(T, bg1, st.C1[tid]);
            out_rgb[2 * plane + p] = fmaf(T, bg2, st.C2[tid]);
        }
        if (out_T) out_T[p] = T;
        if (NC) out_nc[p] = st.last[tid];
    }
}

// a7, second walk (ss_prune_score runs k_render<true> first for T_final and n_contrib per
// pixel).  Back to front over each pixel's blended entries, T_i = T_{i+1} / (1 - alpha_i) and
// the suffix colour S <- alpha c + (1 - alpha) S (R19):
//   dC_ch/dalpha_i = T_i (c_ch - S_ch) - T_final bg_ch / (1 - alpha_i)      (from Eq. 7)
//   U_i += sum_ch (sigma_i dC_ch/dalpha_i)^2                                 (Eqs. 20-21)
// Batches are taken from the end of the tile list and staged like k_render's (cp.async ring,
// pair-interleaved layout, q / alpha of a pair on f32x2); the pixels active in a batch (their
// last blended entry lies at or after its start) are compacted onto the lowest threads.  The
// per-Gaussian terms of a warp are summed 8 Gaussians at a time by a transpose-reduce (9
// shuffles per 8 Gaussians), the warps' sums per Gaussian in shared memory, and one float64
// atomic per (tile, Gaussian) adds them to the score.
__global__ void __launch_bounds__(256, 5) k_score_bwd(const uint2 *__restrict__ ranges,
                                                   const uint32_t *__restrict__ vals,
                                                   const float4 *__restrict__ rec, int W, int H, int tiles_x,
                                                   float bg0, float bg1, float bg2,
                                                   const float *__restrict__ T_final,
                                                   const uint32_t *__restrict__ n_contrib,
                                                   double *__restrict__ score, const ColorSrc *__restrict__ csp) {
    pdl_enter();
    const ColorSrc cs = *csp;
    __shared__ __align__(16) RawBatch raw[2];
    __shared__ __align__(16) SoaBatch s;
    __shared__ PixState st;  // T (running), C0..2 = suffix S, last = n_contrib
    __shared__ float s_Tfin[256];
    __shared__ uint32_t s_id[kBatch];
    __shared__ float s_part[8][kBatch];
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_max;
    const int tile = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    int mpx, mpy;
    tile_pixel(tile, tiles_x, tid, mpx, mpy);
    int tx0, ty0;
    tile_pixel(tile, tiles_x, 0, tx0, ty0);
    const bool inside = mpx < W && mpy < H;
    const uint2 range = ranges[tile];
    if (tid == 0) s_max = 0;
    const size_t pix = (size_t)mpy * W + mpx;
    const uint32_t my_last = inside ? n_contrib[pix] : 0u;
    st.last[tid] = my_last;
    st.T[tid] = s_Tfin[tid] = inside ? T_final[pix] : 1.0f;
    st.C0[tid] = st.C1[tid] = st.C2[tid] = 0.0f;
    __syncthreads();
    if (my_last) atomicMax(&s_max, my_last);
    __syncthreads();
    const uint32_t max_last = min(s_max, range.y - range.x);
    if (max_last == 0) return;
    // batch b covers [start_b, end_b), from the end of the blended part of the list
    const bool loader = tid < kBatch;
    uint32_t end = range.x + max_last;
    uint32_t start = end - min((uint32_t)kBatch, max_last);
    uint32_t g_cur = 0, g_nxt = 0;
    if (loader) {
        const uint32_t j0 = start + tid;
        g_cur = j0 < end ? __ldg(vals + j0) : 0u;
        const uint32_t s1 = start - min((uint32_t)kBatch, start - range.x), j1 = s1 + tid;
        g_nxt = j1 < start ? __ldg(vals + j1) : 0u;
        stage_gather(raw[0], rec, g_cur, j0 < end);
    }
    cp_async_commit();
    int buf = 0;
    const float2 BG01 = make_float2(bg0, bg1);
    while (end > range.x) {
        const int cnt = (int)(end - start);
        __syncthreads();  // the previous batch is consumed: s, s_id, s_part and raw[buf ^ 1] free
        // the next (earlier) batch in flight, its successor's ids loaded
        const uint32_t s1 = start - min((uint32_t)kBatch, start - range.x);
        uint32_t g_after = 0;
        if (loader) {
            const uint32_t j1 = s1 + tid;
            stage_gather(raw[buf ^ 1], rec, g_nxt, j1 < start);
            const uint32_t s2 = s1 - min((uint32_t)kBatch, s1 - range.x), j2 = s2 + tid;
            g_after = j2 < s1 ? __ldg(vals + j2) : 0u;
        }
        cp_async_commit();
        const uint32_t n_active = compact_active(my_last > start - range.x, st, s_warp);
        cp_async_wait<1>();
        if (loader) {
            stage_transpose(s, raw[buf], rec, g_cur, tid < cnt, cs);
            s_id[tid] = g_cur;
        }
        g_cur = g_nxt;
        g_nxt = g_after;
        __syncthreads();
        const uint32_t n_warps = (n_active + 31) / 32;
        if ((uint32_t)warp < n_warps) {
            const bool act = tid < n_active;
            const int pp = act ? st.list[tid] : 0;
            int px, py;
            tile_pixel_at(tx0, ty0, pp, px, py);
            const float2 FX = f2((float)px), FY = f2((float)py);
            const uint32_t plast = act ? st.last[pp] : 0u;
            const float Tfin = s_Tfin[pp];
            float T = act ? st.T[pp] : 1.0f;
            // suffix colour: (S0, S1) as one f32x2, S2 scalar
            float2 S01 = act ? make_float2(st.C0[pp], st.C1[pp]) : make_float2(0.0f, 0.0f);
            float S2 = act ? st.C2[pp] : 0.0f;
            const uint32_t rel = start - range.x;  // list position of slot 0
            const int top = (cnt + 7) & ~7;          // groups of 8 slots (padding never contributes)
            for (int k8 = top - 8; k8 >= 0; k8 -= 8) {
                float tv[8];
#pragma unroll
                for (int pq = 3; pq >= 0; --pq) {  // pairs from the top of the group down
                    const int k = k8 + 2 * pq;
                    const float4 *v = s.v[k >> 1];
                    const float4 v0 = v[0], v1 = v[1], v2 = v[2], v3 = v[3], v4 = v[4];
                    const float2 dx = __fadd2_rn(FX, make_float2(v0.x, v0.y));
                    const float2 dy = __fadd2_rn(FY, make_float2(v0.z, v0.w));
                    const float2 u = __ffma2_rn(make_float2(v1.x, v1.y), dx, __fmul2_rn(make_float2(v1.z, v1.w), dy));
                    const float2 q = __ffma2_rn(dx, u, __fmul2_rn(__fmul2_rn(make_float2(v2.x, v2.y), dy), dy));
                    const float2 ql = __fmul2_rn(q, f2(-0.72134752044448170f));
                    const float2 se =
                        __fmul2_rn(make_float2(v3.x, v3.y), make_float2(ex2_approx(ql.x), ex2_approx(ql.y)));
#pragma unroll
                    for (int h = 1; h >= 0; --h) {  // the odd (later) Gaussian first
                        float term = 0.0f;
                        const bool blended = rel + (uint32_t)(k + h) < plast && (h ? q.y <= v2.w : q.x <= v2.z);
                        if (blended) {
                            const float sg = h ? v3.y : v3.x;
                            const float alpha = fminf(0.99f, h ? se.y : se.x);
                            const float2 crg = h ? make_float2(v4.x, v4.y) : make_float2(v3.z, v3.w);
                            const float cb = h ? v4.w : v4.z;
                            const float om = 1.0f - alpha;
                            float rom;  // T_i = T_{i+1} / (1 - alpha_i): one approximate reciprocal
                            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rom) : "f"(om));
                            T = T * rom;
                            const float bgs = Tfin * rom;
                            // (d0, d1) = T (c_rg - S_rg) - bgs bg_rg on f32x2, d2 scalar
                            const float2 d01 = __ffma2_rn(f2(-bgs), BG01,
                                                          __fmul2_rn(f2(T), __fadd2_rn(crg, make_float2(-S01.x, -S01.y))));
                            const float d2 = T * (cb - S2) - bgs * bg2;
                            const float2 sq = __fmul2_rn(d01, d01);
                            term = sg * sg * (sq.x + sq.y + d2 * d2);
                            S01 = __ffma2_rn(f2(alpha), crg, __fmul2_rn(f2(om), S01));
                            S2 = alpha * cb + om * S2;
                        }
                        tv[2 * pq + h] = term;
                    }
                }
                // warp sums of the 8 terms: transpose-reduce, lane L (L & 3 == 0) ends with the
                // Gaussian (L >> 2) & 7 of the group
                bool any = false;
#pragma unroll
                for (int j = 0; j < 8; ++j) any |= tv[j] != 0.0f;
                if (__any_sync(0xffffffffu, any)) {
                    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
                    float v4r[4], v2r[2];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float send = h16 ? tv[j] : tv[4 + j];
                        v4r[j] = (h16 ? tv[4 + j] : tv[j]) + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const float send = h8 ? v4r[j] : v4r[2 + j];
                        v2r[j] = (h8 ? v4r[2 + j] : v4r[j]) + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
                    float v1 = (h4 ? v2r[1] : v2r[0]) + __shfl_xor_sync(0xffffffffu, h4 ? v2r[0] : v2r[1], 4);
                    v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
                    v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
                    if ((lane & 3) == 0) s_part[warp][k8 + ((lane >> 2) & 7)] = v1;
                } else if ((lane & 3) == 0) {
                    s_part[warp][k8 + ((lane >> 2) & 7)] = 0.0f;
                }
            }
            if (act) {
                st.T[pp] = T;
                st.C0[pp] = S01.x;
                st.C1[pp] = S01.y;
                st.C2[pp] = S2;
            }
        }
        __syncthreads();
        if (tid < cnt) {
            float sum = 0.f;
            for (uint32_t w = 0; w < n_warps; ++w) sum += s_part[w][tid];
            if (sum != 0.f) atomicAdd(score + s_id[tid], (double)sum);
        }
        end = start;
        start = s1;
        buf ^= 1;
    }
    cp_async_wait<0>();
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
    int tx0, ty0;
    tile_pixel(tile, tiles_x, 0, tx0, ty0);
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
            tile_pixel_at(tx0, ty0, pp, px, py);
            const float fpx = (float)px, fpy = (float)py;
            const uint32_t plast = act ? st.last[pp] : 0u;
            const float Tfin = s_Tfin[pp];
            float *wpart = s_part + (size_t)warp * kBatch * 9;
            const float dC0 = s_dC[0][pp], dC1 = s_dC[1][pp], dC2 = s_dC[2][pp];
            float T = act ? st.T[pp] : 1.0f;
            // inactive lanes (pp = 0 placeholder) read nothing: pixel 0's state may be written by
            // its own lane in this phase
            float S0 = act ? st.C0[pp] : 0.0f, S1 = act ? st.C1[pp] : 0.0f, S2 = act ? st.C2[pp] : 0.0f;
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
// 256 x Gaussians staged), [3] += pixels, [4] += phantom pairs: (tile, Gaussian) pairs of the
// list whose Gaussian has q > t (alpha < 1/255) at every pixel centre of the tile (AccuTile's
// tile test is against the continuous cell, R23; this walks every pair, no termination).
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
    // phantom pairs: every batch of the list against every pixel centre of the tile
    unsigned long long phantom = 0;
    __shared__ uint32_t s_hit[kBatch / 32];
    for (uint32_t start = range.x; start < range.y; start += kBatch) {
        __syncthreads();
        load_batch(s, vals, rec, start + threadIdx.x, range.y, nullptr, cs);
        if (threadIdx.x < kBatch / 32) s_hit[threadIdx.x] = 0;
        __syncthreads();
        const int cnt = min((uint32_t)kBatch, range.y - start);
        for (int k = 0; k < cnt; ++k) {
            const float4 bx = s.box[k];
            const float4 cn = s.con[k];
            const bool hit = inside && pixel_q(fpx, fpy, bx.x, bx.y, cn.x, cn.y, cn.z) <= cn.w;
            if (__any_sync(0xffffffffu, hit) && (threadIdx.x & 31) == 0) atomicOr(&s_hit[k >> 5], 1u << (k & 31));
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int k = 0; k < cnt; ++k) phantom += (s_hit[k >> 5] >> (k & 31)) & 1u ? 0u : 1u;
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
        atomicAdd(counters + 4, phantom);
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

// The render records as a 2-D tensor (N rows of 12 float32) for TMA gather4: one row per
// Gaussian, box = 1 row (gather4 moves 4 rows of 48 B).  Encoded on the host per launch (the
// record array belongs to the caller's workspace); cuTensorMapEncodeTiled through the runtime's
// driver entry point (no libcuda link).
static cudaError_t records_tensor_map(const float4 *rec, int n, CUtensorMap *tm) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t gdim[2] = {12, (cuuint64_t)(n > 0 ? n : 1)};
    const cuuint64_t gstride[1] = {48};
    const cuuint32_t box[2] = {12, 1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float4 *>(rec), gdim, gstride, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_render(void *ws, const Layout &L, int W, int H, float bg0, float bg1, float bg2, float *out_rgb,
                          float *out_T, uint32_t *out_nc, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    const int grid = P.n_tiles * (256 / kRenderPix);
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    const bool tma = render_tma();
    if (tma) {
        const cudaError_t e = records_tensor_map(at<const float4>(ws, P.rec), L.n, &tm);
        if (e != cudaSuccess) return e;
    }
#define SS_RENDER_ARGS                                                                                           \
    at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value), at<const float4>(ws, P.rec), W, H,    \
        P.tiles_x, bg0, bg1, bg2, out_rgb, out_T, out_nc, at<const ColorSrc>(ws, L.color_src), tm
    if (out_nc && tma)
        launch_pdl(k_render<true, kRenderPix, kRenderBatch, true>, grid, kRenderPix, 0, st, SS_RENDER_ARGS);
    else if (out_nc)
        launch_pdl(k_render<true, kRenderPix, kRenderBatch, false>, grid, kRenderPix, 0, st, SS_RENDER_ARGS);
    else if (tma)
        launch_pdl(k_render<false, kRenderPix, kRenderBatch, true>, grid, kRenderPix, 0, st, SS_RENDER_ARGS);
    else
        launch_pdl(k_render<false, kRenderPix, kRenderBatch, false>, grid, kRenderPix, 0, st, SS_RENDER_ARGS);
#undef SS_RENDER_ARGS
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
    // forward walk = k_render with T_final / n_contrib (no image), then the back-to-front walk
    float *pT = at<float>(ws, L.pix_T);
    uint32_t *pl = at<uint32_t>(ws, L.pix_last);
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    const bool tma = render_tma();
    if (tma) {
        const cudaError_t e = records_tensor_map(at<const float4>(ws, P.rec), L.n, &tm);
        if (e != cudaSuccess) return e;
    }
    if (tma)
        launch_pdl(k_render<true, kRenderPix, kRenderBatch, true>, P.n_tiles * (256 / kRenderPix), kRenderPix, 0,
                   st, at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value), at<const float4>(ws, P.rec),
                   W, H, P.tiles_x, bg0, bg1, bg2, (float *)nullptr, pT, pl, at<const ColorSrc>(ws, L.color_src), tm);
    else
        launch_pdl(k_render<true, kRenderPix, kRenderBatch, false>, P.n_tiles * (256 / kRenderPix), kRenderPix, 0,
                   st, at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value), at<const float4>(ws, P.rec),
                   W, H, P.tiles_x, bg0, bg1, bg2, (float *)nullptr, pT, pl, at<const ColorSrc>(ws, L.color_src), tm);
    launch_pdl(k_score_bwd, P.n_tiles, 256, 0, st, at<const uint2>(ws, P.ranges),
               at<const uint32_t>(ws, P.sorted_value), at<const float4>(ws, P.rec), W, H, P.tiles_x, bg0, bg1, bg2,
               (const float *)pT, (const uint32_t *)pl, score, at<const ColorSrc>(ws, L.color_src));
    return cudaGetLastError();
}

}  // namespace ss
