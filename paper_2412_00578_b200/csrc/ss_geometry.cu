// ss_geometry.cu -- a1 preprocess and a3 key emission (libss, sm_100a).
//
// ARITHMETIC CONTRACT: this translation unit is compiled with --fmad=false so
// that every float32 operation below is rounded individually, exactly as the contract
// states; IEEE division and square root (no fast-math).  Projection / conic / colour are
// float32; the tile geometry (SnugBox, AccuTile, 3-sigma rect) is float64 evaluated on the
// stored float32 record, so the tile count of a1 and the emission of a3 run the same
// function on the same values (R1) and are exact for the stored conic.
//
// P:n = /root/reference/PAPER.md line n.
#include "ss_color.cuh"
#include "ss_tilegeom.cuh"
#include "ss_tilegeom32.cuh"

namespace ss {
namespace {

// Projection of one Gaussian in front of the camera (Eqs. 3-4, 10; R1, R3, R5, R24): mean to
// pixels, Sigma_2D = J W Sigma_3D W^T J^T + 0.3 I, its determinant.  Shared by both preprocess
// kernels, so their records are bit-identical (this unit is compiled with --fmad=false).
__device__ __forceinline__ void project(const float4 &q4, const float4 &s4, float px, float py, float pz,
                                        const CamArgs &cam, float limx, float limy, float &x2d, float &y2d,
                                        float &cxx, float &cxy, float &cyy, float &det) {
    const float iz = 1.0f / pz;  // contract R1: one reciprocal of z
    const float tx = px * iz, ty = py * iz;
    x2d = cam.fx * tx + cam.cx;
    y2d = cam.fy * ty + cam.cy;
    float txc = tx, tyc = ty;
    if (cam.clip > 0.0f) {
        txc = fminf(limx, fmaxf(-limx, tx));
        tyc = fminf(limy, fmaxf(-limy, ty));
    }
    const float j00 = cam.fx * iz, j02 = -(cam.fx * txc) * iz;
    const float j11 = cam.fy * iz, j12 = -(cam.fy * tyc) * iz;
    const float qn = 1.0f / sqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
    const float w = q4.x * qn, x = q4.y * qn, y = q4.z * qn, z = q4.w * qn;
    const float Rm[3][3] = {
        {1.0f - 2.0f * (y * y + z * z), 2.0f * (x * y - w * z), 2.0f * (x * z + w * y)},
        {2.0f * (x * y + w * z), 1.0f - 2.0f * (x * x + z * z), 2.0f * (y * z - w * x)},
        {2.0f * (x * z - w * y), 2.0f * (y * z + w * x), 1.0f - 2.0f * (x * x + y * y)}};
    const float s3[3] = {s4.x, s4.y, s4.z};
    float M[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) M[r][k] = Rm[r][k] * s3[k];
    float S[3][3];  // Eq. 3
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) S[r][k] = M[r][0] * M[k][0] + M[r][1] * M[k][1] + M[r][2] * M[k][2];
    float T[2][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T[0][k] = j00 * cam.V[0 + k] + j02 * cam.V[8 + k];
        T[1][k] = j11 * cam.V[4 + k] + j12 * cam.V[8 + k];
    }
    float U[2][3];  // Eq. 4
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) U[r][k] = T[r][0] * S[0][k] + T[r][1] * S[1][k] + T[r][2] * S[2][k];
    cxx = U[0][0] * T[0][0] + U[0][1] * T[0][1] + U[0][2] * T[0][2];
    cxy = U[0][0] * T[1][0] + U[0][1] * T[1][1] + U[0][2] * T[1][2];
    cyy = U[1][0] * T[1][0] + U[1][1] * T[1][1] + U[1][2] * T[1][2];
    cxx = cxx + 0.3f;  // R5
    cyy = cyy + 0.3f;
    det = cxx * cyy - cxy * cxy;
}

// Record of a Gaussian with tiles: render record (48 B) and emission record (32 B).
__device__ __forceinline__ void write_records(size_t i, int mode, float x2d, float y2d, float a, float b, float c,
                                              double td, float sigma, const int4 &R, uint32_t count, uint32_t n_ent,
                                              uint32_t n_span, bool span_inline, uint32_t cols,
                                              const uint32_t *pay, float4 *__restrict__ rec,
                                              uint4 *__restrict__ erec) {
    // render record (48 B): q0 (x, y, a, b) | q1 (c, t, sigma, 0) | q2 (colour flag, r, g, b);
    // the colour (R13) is left pending (flag 0) and computed by the first render-path
    // kernel that gathers the record (ss_color.cuh)
    float4 *q = rec + 3 * (size_t)i;
    q[0] = make_float4(x2d, y2d, a, b);
    q[1] = make_float4(c, (float)td, sigma, 0.0f);
    q[2] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    // emission record (32 B, one sector): (count, info, p0..p5); the payload p holds the
    // non-empty line spans of an AccuTile set of at most kLaneRows lines (tmin | tmax << 9
    // | line << 18), or up to kInlineEnt super-tile entries (super-tile | mask << 16), or
    // -- for a Gaussian with more entries -- aux = t as float64 bits (AccuTile) or the
    // packed rect (x0, x1-x0-1, y0, y1-y0-1) for the re-enumeration; info = span count |
    // entries-inline 0x100 | columns 0x200 | AccuTile 0x400 | spans-inline 0x800 | entries << 12.
    uint32_t aux0, aux1;
    if (mode == SS_BIN_ACCUTILE) {
        aux0 = (uint32_t)__double2loint(td);
        aux1 = (uint32_t)__double2hiint(td);
    } else {
        aux0 = (uint32_t)R.x | ((uint32_t)(R.y - R.x - 1) << 8) | ((uint32_t)R.z << 16) |
               ((uint32_t)(R.w - R.z - 1) << 24);
        aux1 = 0u;
    }
    const uint32_t info = (span_inline ? (kInfoSpanInline | n_span)
                                       : (n_ent <= (uint32_t)kInlineEnt ? kInfoEntInline : 0u)) |
                          (cols ? kInfoCols : 0u) | (mode == SS_BIN_ACCUTILE ? kInfoAccuTile : 0u) |
                          (n_ent << kInfoEntShift);
    // the whole 32 B sector in two 16 B stores (partial-sector writes would cost a DRAM
    // read-modify-write); the payload was staged in shared memory (pay, 6 words)
    const bool inl = (info & (kInfoSpanInline | kInfoEntInline)) != 0;
    erec[2 * (size_t)i] = make_uint4(count, info, inl ? pay[0] : aux0, inl ? pay[1] : aux1);
    erec[2 * (size_t)i + 1] = make_uint4(pay[2], pay[3], pay[4], pay[5]);
}

// ---------------------------------------------------------------- a1 preprocess kernel
constexpr int kPreThreads = 256;  // CTA size
constexpr int kPreBlocks = 2;     // k_preprocess64 CTAs per SM (its register budget: 128)
#ifndef SS_PRE32_BLOCKS
#define SS_PRE32_BLOCKS 3  // 80 registers (measured: 3 -> 1833 fps, 4 (64 registers, spills) -> 1786)
#endif
constexpr int kPre32Blocks = SS_PRE32_BLOCKS;  // k_preprocess32 CTAs per SM
// The float64 reference evaluation of a1: one thread per Gaussian ("each thread
// processes a single Gaussian"), persistent grid-stride loop so each CTA flushes its depth-digit
// histograms once.  It runs over every Gaussian in 3-sigma mode; in SnugBox / AccuTile mode over
// the queue k_preprocess32 leaves it (Gaussians whose float32 certification failed, and the
// tall AccuTile ones, whose lines the warp sweeps cooperatively).
__global__ void __launch_bounds__(kPreThreads, kPreBlocks) k_preprocess64(int n, const uint32_t *__restrict__ queue,
                                                    const uint32_t *__restrict__ queue_n,
                                                    const float4 *__restrict__ mean_opac,
                                                    const float4 *__restrict__ scale, const float4 *__restrict__ rot,
                                                    CamArgs cam, int mode,
                                                    float4 *__restrict__ rec, uint4 *__restrict__ erec,
                                                    uint32_t *__restrict__ depth_key, uint32_t *__restrict__ gne,
                                                    uint32_t *__restrict__ hist,
                                                    uint32_t *__restrict__ n_visible,
                                                    uint32_t *__restrict__ total_pairs, ColorSrc cs_in,
                                                    ColorSrc *__restrict__ cs_out) {
    pdl_enter();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cs_out = cs_in;  // the render path's lazy colour source
    __shared__ uint32_t s_hist[kDepthPasses][256];
    __shared__ uint32_t s_vis, s_pairs;
    __shared__ uint32_t s_pay[kPreThreads][7];  // emission-record payload of each thread's Gaussian (stride 7: no bank conflicts)
    for (int k = threadIdx.x; k < kDepthPasses * 256; k += blockDim.x) (&s_hist[0][0])[k] = 0;
    for (int k = 0; k < 7; ++k) s_pay[threadIdx.x][k] = 0u;
    if (threadIdx.x == 0) s_vis = s_pairs = 0;
    __syncthreads();
    uint32_t my_vis = 0, my_pairs = 0;
    // camera constants of the J clamp (R5), the same values the per-Gaussian form would give
    const float limx = cam.clip * ((0.5f * (float)cam.W) / cam.fx);
    const float limy = cam.clip * ((0.5f * (float)cam.H) / cam.fy);
    const int stx = (cam.tiles_x + kSuper - 1) / kSuper;
    const int lane = threadIdx.x & 31;
    const int n_items = queue ? (int)*queue_n : n;
    // warp-uniform grid-stride loop (the tall-Gaussian phase below is warp-collective).  Over all
    // Gaussians: 32 per warp step.  Over the queue (a few hundred, many of them tall): one per
    // warp step, so that the queued work spreads over as many warps as possible.
    const int per_step = queue ? 1 : 32;
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int i0 = gwarp * per_step; i0 < n_items; i0 += nwarps * per_step) {
        const bool valid = queue ? (lane == 0) : (i0 + lane < n_items);
        const int i = queue ? (valid ? (int)queue[i0] : 0) : i0 + lane;
        uint32_t count = 0;
        const float4 mo = valid ? mean_opac[i] : make_float4(0.f, 0.f, -1.f, 0.f);
        const float4 q4 = valid ? rot[i] : make_float4(1.f, 0.f, 0.f, 0.f);  // issued with the mean
        const float4 s4 = valid ? scale[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float px = cam.V[0] * mo.x + cam.V[1] * mo.y + cam.V[2] * mo.z + cam.V[3];
        const float py = cam.V[4] * mo.x + cam.V[5] * mo.y + cam.V[6] * mo.z + cam.V[7];
        const float pz = cam.V[8] * mo.x + cam.V[9] * mo.y + cam.V[10] * mo.z + cam.V[11];
        float x2d = 0.f, y2d = 0.f, a = 0.f, b = 0.f, c = 0.f;
        double td = 0.0;
        int4 R = make_int4(0, 0, 0, 0);
        Snug snug;
        snug.hx = snug.hy = 0.0;
        uint32_t cols = 0, n_ent = 0;
        bool tall = false;       // AccuTile with more than kLaneRows lines: the warp-collective phase
        // entries (or line spans) go straight to the emission record (only Gaussians with tiles
        // get one; words past the stored count are stale)
        uint32_t *ent_out = s_pay[threadIdx.x];
        uint32_t *span_out = ent_out;
        uint32_t n_span = 0;
        bool span_inline = false;
        auto put = [&](uint32_t st, uint32_t mask) {
            if (n_ent < (uint32_t)kInlineEnt) ent_out[n_ent] = st | (mask << 16);
            ++n_ent;
        };
        if (valid && pz >= cam.z_near) {
            float cxx, cxy, cyy, det;
            project(q4, s4, px, py, pz, cam, limx, limy, x2d, y2d, cxx, cxy, cyy, det);
            if (det > 0.0f) {
                const float inv = 1.0f / det;
                a = cyy * inv;
                b = -cxy * inv;
                c = cxx * inv;
                const double D = (double)a * (double)c - (double)b * (double)b;
                td = 2.0 * log(255.0 * (double)mo.w);  // Eq. 11 (R2)
                if (D > 0.0 && (mode == SS_BIN_3SIGMA || td > 0.0)) {
                    if (td > 0.0) snug = snugbox((double)x2d, (double)y2d, (double)a, (double)b, (double)c, td);
                    if (mode == SS_BIN_3SIGMA) {
                        R = rect_3sigma((double)x2d, (double)y2d, (double)cxx, (double)cxy, (double)cyy, cam.tiles_x,
                                        cam.tiles_y);
                    } else {
                        R = rect_of_snug(snug, cam.tiles_x, cam.tiles_y);
                    }
                    if (mode == SS_BIN_ACCUTILE) {
                        Sweep w;
                        if (accutile_setup_from(snug, R, (double)x2d, (double)y2d, (double)a, (double)b, (double)c,
                                                td, w)) {
                            cols = w.rows ? 0u : 1u;
                            if (w.s1 - w.s0 <= kLaneRows) {
                                // lines stored in the record (level 1 derives the entries from them);
                                // here only the entry count
                                EntryCount ec;
                                cnt_init(ec);
                                count = accutile_count(w, cam.tiles_x, [&](int r, int lo, int hi) {
                                    cnt_feed(ec, r, lo, hi);
                                    if (hi > lo)
                                        span_out[n_span++] = (uint32_t)lo | ((uint32_t)hi << 9) | ((uint32_t)r << 18);
                                });
                                cnt_flush(ec);
                                n_ent = ec.n;
                                span_inline = true;
                            } else {
                                tall = true;
                            }
                        }
                    } else if (R.x < R.y && R.z < R.w) {
                        count = (uint32_t)((R.y - R.x) * (R.w - R.z));
                        // super-tile entries of the rect: its super-tile rect, masks of the overlap
                        for (int band = R.z >> 2; band <= (R.w - 1) >> 2; ++band) {
                            uint32_t rows = 0;
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                rows |= (4 * band + q >= R.z && 4 * band + q < R.w) ? (1u << (4 * q)) : 0u;
                            for (int C = R.x >> 2; C <= (R.y - 1) >> 2; ++C) {
                                const int x0 = max(R.x, 4 * C), x1 = min(R.y, 4 * C + 4);
                                const uint32_t cb = ((1u << (x1 - x0)) - 1u) << (x0 - 4 * C);
                                put((uint32_t)(band * stx + C), rows * cb);
                            }
                        }
                    }
                }
            }
        }
        // Tall Gaussians, one at a time by the whole warp (bounded divergence): lane l takes
        // bands first + l, ... of 4 lines, each evaluated by sweep_band exactly as the sequential
        // loop evaluates them; pairs and entries are summed over the warp, entries written in
        // the count's order straight into the owner's emission record.
        uint32_t tall_mask = __ballot_sync(0xffffffffu, tall);
        while (tall_mask) {
            const int src = __ffs(tall_mask) - 1;
            tall_mask &= tall_mask - 1;
            const int gi = __shfl_sync(0xffffffffu, i, src);
            const float bx = __shfl_sync(0xffffffffu, x2d, src), by = __shfl_sync(0xffffffffu, y2d, src);
            const float ba = __shfl_sync(0xffffffffu, a, src), bb = __shfl_sync(0xffffffffu, b, src);
            const float bc = __shfl_sync(0xffffffffu, c, src);
            const double bt = __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(td), src),
                                               __shfl_sync(0xffffffffu, __double2loint(td), src));
            Sweep w;
            accutile_setup((double)bx, (double)by, (double)ba, (double)bb, (double)bc, bt, cam.tiles_x, cam.tiles_y,
                           w);
            uint32_t pairs = 0, ents = 0;
            uint32_t *ent_out = s_pay[(threadIdx.x & ~31) + src];  // the owner's payload
            const int last = (w.s1 - 1) >> 2;
            for (int b0 = w.s0 >> 2; b0 <= last; b0 += 32) {
                const int band = b0 + lane;
                uint32_t iv0 = 0, iv1 = 0, iv2 = 0, iv3 = 0;
                if (band <= last) sweep_band(w, band, iv0, iv1, iv2, iv3);
                auto len = [](uint32_t v) { return (v >> 16) > (v & 0xFFFFu) ? (v >> 16) - (v & 0xFFFFu) : 0u; };
                uint32_t p = len(iv0) + len(iv1) + len(iv2) + len(iv3);
                uint32_t ne = 0;
                if (band <= last) band_entries(band, iv0, iv1, iv2, iv3, !w.rows, stx, [&](uint32_t, uint32_t) { ++ne; });
                uint32_t x = ne;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                    p += __shfl_xor_sync(0xffffffffu, p, o);
                }
                uint32_t j = ents + x - ne;
                if (band <= last)
                    band_entries(band, iv0, iv1, iv2, iv3, !w.rows, stx, [&](uint32_t st, uint32_t mask) {
                        if (j < (uint32_t)kInlineEnt) ent_out[j] = st | (mask << 16);
                        ++j;
                    });
                ents += __shfl_sync(0xffffffffu, x, 31);
                pairs += p;
            }
            if (lane == src) {
                count = pairs;
                n_ent = ents;
            }
        }
        __syncwarp();  // the tall sweeps' entries (written by every lane) visible to their owners
        if (count > 0) {
            write_records((size_t)i, mode, x2d, y2d, a, b, c, td, mo.w, R, count, n_ent, n_span, span_inline, cols,
                          s_pay[threadIdx.x], rec, erec);
            const uint32_t key = __float_as_uint(pz);
            depth_key[i] = key;
            gne[i] = n_ent;
#pragma unroll
            for (int p = 0; p < kDepthPasses; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 0xFF], 1u);
            ++my_vis;
            my_pairs += count;
        } else if (valid) {
            depth_key[i] = kNoTiles;
            gne[i] = 0u;
        }
    }
    // warp-aggregate the visible count, then one atomic per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_vis += __shfl_xor_sync(0xffffffffu, my_vis, o);
        my_pairs += __shfl_xor_sync(0xffffffffu, my_pairs, o);
    }
    if ((threadIdx.x & 31) == 0 && my_vis) {
        atomicAdd(&s_vis, my_vis);
        atomicAdd(&s_pairs, my_pairs);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kDepthPasses * 256; k += blockDim.x) {
        const uint32_t v = (&s_hist[0][0])[k];
        if (v) atomicAdd(hist + k, v);
    }
    if (threadIdx.x == 0 && s_vis) {
        atomicAdd(n_visible, s_vis);
        atomicAdd(total_pairs, s_pairs);
    }
}


// a1, SnugBox / AccuTile: the tile geometry in float32 with certified bounds
// (ss_tilegeom32.cuh).  A Gaussian whose every decision is certain gets exactly the float64
// path's tile set, count, entries / spans and records; the others (uncertain decisions, and
// AccuTile sets of more than kLaneRows lines, which k_preprocess64 sweeps warp-cooperatively)
// are appended to `queue` for k_preprocess64.  The projection and t are the float64 path's
// (project(), t = 2 log(255 sigma) in float64, R2).  Scale and rotation are loaded only for
// Gaussians in front of the near plane; the next iteration's mean is prefetched.
template <int MODE>
__global__ void __launch_bounds__(kPreThreads, kPre32Blocks) k_preprocess32(int n, const float4 *__restrict__ mean_opac,
                                                    const float4 *__restrict__ scale, const float4 *__restrict__ rot,
                                                    CamArgs cam, float4 *__restrict__ rec, uint4 *__restrict__ erec,
                                                    uint32_t *__restrict__ depth_key, uint32_t *__restrict__ gne,
                                                    uint32_t *__restrict__ hist, uint32_t *__restrict__ n_visible,
                                                    uint32_t *__restrict__ total_pairs, uint32_t *__restrict__ queue,
                                                    uint32_t *__restrict__ queue_n, uint32_t *__restrict__ ticket,
                                                    ColorSrc cs_in, ColorSrc *__restrict__ cs_out) {
    pdl_enter();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cs_out = cs_in;  // the render path's lazy colour source
    __shared__ uint32_t s_hist[kDepthPasses][256];
    __shared__ uint32_t s_vis, s_pairs;
    __shared__ uint32_t s_pay[kPreThreads][7];  // emission-record payload of each thread's Gaussian (stride 7: no bank conflicts)
    for (int k = threadIdx.x; k < kDepthPasses * 256; k += blockDim.x) (&s_hist[0][0])[k] = 0;
    for (int k = 0; k < 7; ++k) s_pay[threadIdx.x][k] = 0u;
    if (threadIdx.x == 0) s_vis = s_pairs = 0;
    __syncthreads();
    uint32_t my_vis = 0, my_pairs = 0;
    const float limx = cam.clip * ((0.5f * (float)cam.W) / cam.fx);
    const float limy = cam.clip * ((0.5f * (float)cam.H) / cam.fy);
    const int stx = (cam.tiles_x + kSuper - 1) / kSuper;
    const int lane = threadIdx.x & 31;
    // warp chunks of 32 Gaussians: the first one static (global warp id), then tickets (the
    // next chunk fetched one step ahead, with its mean), so that the warps of the persistent
    // grid finish together (grid-stride: 0.157 ms single-stream, tickets: 0.144 ms)
    // The ticket of the chunk after next is taken each step and consumed one step later, so
    // the atomic's round trip is not on the path to the next mean's load.
    const int nwarps_all = (gridDim.x * blockDim.x) >> 5;
    int c_next = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // chunk of the next step
    uint32_t t_after = 0;  // lane 0: ticket of the step after (pending)
    if (lane == 0) t_after = atomicAdd(ticket, 1u);
    int i = c_next * 32 + lane;
    float4 mo_next = i < n ? mean_opac[i] : make_float4(0.f, 0.f, -1.f, 0.f);
    for (int i0 = c_next * 32; i0 < n; i0 = c_next * 32, i = i0 + lane) {
        c_next = nwarps_all + (int)__shfl_sync(0xffffffffu, t_after, 0);
        if (lane == 0) t_after = atomicAdd(ticket, 1u);
        const bool valid = i < n;
        const float4 mo = mo_next;
        const int in = c_next * 32 + lane;
        mo_next = in < n ? mean_opac[in] : make_float4(0.f, 0.f, -1.f, 0.f);
        const float px = cam.V[0] * mo.x + cam.V[1] * mo.y + cam.V[2] * mo.z + cam.V[3];
        const float py = cam.V[4] * mo.x + cam.V[5] * mo.y + cam.V[6] * mo.z + cam.V[7];
        const float pz = cam.V[8] * mo.x + cam.V[9] * mo.y + cam.V[10] * mo.z + cam.V[11];
        uint32_t count = 0, cols = 0, n_ent = 0, n_span = 0;
        bool defer = false, span_inline = false, tall = false;
        Snug32 S;
        float x2d = 0.f, y2d = 0.f, a = 0.f, b = 0.f, c = 0.f;
        double td = 0.0;
        int4 R = make_int4(0, 0, 0, 0);
        uint32_t *ent_out = s_pay[threadIdx.x];
        if (valid && pz >= cam.z_near) {
            const float4 q4 = rot[i];
            const float4 s4 = scale[i];
            float cxx, cxy, cyy, det;
            project(q4, s4, px, py, pz, cam, limx, limy, x2d, y2d, cxx, cxy, cyy, det);
            if (det > 0.0f) {
                const float inv = 1.0f / det;
                a = cyy * inv;
                b = -cxy * inv;
                c = cxx * inv;
                td = 2.0 * log(255.0 * (double)mo.w);  // Eq. 11 (R2)
                if (td > 0.0) {
                    const int sc = snug32<MODE == SS_BIN_ACCUTILE>(x2d, y2d, a, b, c, td, S);
                    if (sc == kUnsure) {
                        defer = true;
                    } else if (sc == kSure) {
                        R = rect32(S, cam.tiles_x, cam.tiles_y);
                        if (R.x < R.y && R.z < R.w) {
                            if (MODE == SS_BIN_ACCUTILE) {
                                Sweep32 w;
                                sweep32_setup(S, R, x2d, y2d, a, b, c, w);
                                cols = w.rows ? 0u : 1u;
                                if (w.s1 - w.s0 > kLaneRows) {
                                    tall = true;  // the warp-cooperative sweep below
                                } else {
                                    // line spans into the emission record (the binning derives
                                    // the entries from them); here only the entry count
                                    EntryCount ec;
                                    cnt_init(ec);
                                    const bool ok = accutile_count32(w, count, [&](int r, int lo, int hi) {
                                        cnt_feed(ec, r, lo, hi);
                                        if (hi > lo)
                                            ent_out[n_span++] = (uint32_t)lo | ((uint32_t)hi << 9) | ((uint32_t)r << 18);
                                    });
                                    cnt_flush(ec);
                                    n_ent = ec.n;
                                    span_inline = true;
                                    defer = !ok;
                                }
                            } else {
                                count = (uint32_t)((R.y - R.x) * (R.w - R.z));
                                for (int band = R.z >> 2; band <= (R.w - 1) >> 2; ++band) {
                                    uint32_t rows = 0;
#pragma unroll
                                    for (int q = 0; q < 4; ++q)
                                        rows |= (4 * band + q >= R.z && 4 * band + q < R.w) ? (1u << (4 * q)) : 0u;
                                    for (int C = R.x >> 2; C <= (R.y - 1) >> 2; ++C) {
                                        const int x0 = max(R.x, 4 * C), x1 = min(R.y, 4 * C + 4);
                                        const uint32_t cb = ((1u << (x1 - x0)) - 1u) << (x0 - 4 * C);
                                        if (n_ent < (uint32_t)kInlineEnt)
                                            ent_out[n_ent] = (uint32_t)(band * stx + C) | ((rows * cb) << 16);
                                        ++n_ent;
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
        // Tall AccuTile Gaussians (more than kLaneRows lines), one at a time by the whole warp:
        // lane l takes bands first + l, ... of 4 rows (band32, the rows evaluated exactly as the
        // sequential loop evaluates them); pairs and entries summed over the warp, entries
        // written in the count's order into the owner's emission record.  Any uncertain decision
        // defers the Gaussian to the float64 path.
        if (MODE == SS_BIN_ACCUTILE) {
            uint32_t tall_mask = __ballot_sync(0xffffffffu, tall);
            while (tall_mask) {
                const int src = __ffs(tall_mask) - 1;
                tall_mask &= tall_mask - 1;
                const int gi = __shfl_sync(0xffffffffu, i, src);
                const float bx = __shfl_sync(0xffffffffu, x2d, src), by = __shfl_sync(0xffffffffu, y2d, src);
                const float ba = __shfl_sync(0xffffffffu, a, src), bb = __shfl_sync(0xffffffffu, b, src);
                const float bc = __shfl_sync(0xffffffffu, c, src);
                const double bt = __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(td), src),
                                                   __shfl_sync(0xffffffffu, __double2loint(td), src));
                Snug32 S2;
                snug32<true>(bx, by, ba, bb, bc, bt, S2);  // certified for the owner already
                Sweep32 w;
                sweep32_setup(S2, rect32(S2, cam.tiles_x, cam.tiles_y), bx, by, ba, bb, bc, w);
                uint32_t pairs = 0, ents = 0;
                bool sure = true;
                uint32_t *eo = s_pay[(threadIdx.x & ~31) + src];  // the owner's payload
                const int last = (w.s1 - 1) >> 2;
                for (int b0 = w.s0 >> 2; b0 <= last; b0 += 32) {
                    const int band = b0 + lane;
                    uint32_t iv0 = 0, iv1 = 0, iv2 = 0, iv3 = 0;
                    if (band <= last) sure &= band32(w, band, iv0, iv1, iv2, iv3);
                    auto len = [](uint32_t v) { return (v >> 16) > (v & 0xFFFFu) ? (v >> 16) - (v & 0xFFFFu) : 0u; };
                    uint32_t p = len(iv0) + len(iv1) + len(iv2) + len(iv3);
                    uint32_t ne = 0;
                    if (band <= last) band_entries(band, iv0, iv1, iv2, iv3, !w.rows, stx, [&](uint32_t, uint32_t) { ++ne; });
                    uint32_t x = ne;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                        p += __shfl_xor_sync(0xffffffffu, p, o);
                    }
                    uint32_t jj = ents + x - ne;
                    if (band <= last)
                        band_entries(band, iv0, iv1, iv2, iv3, !w.rows, stx, [&](uint32_t st, uint32_t mask) {
                            if (jj < (uint32_t)kInlineEnt) eo[jj] = st | (mask << 16);
                            ++jj;
                        });
                    ents += __shfl_sync(0xffffffffu, x, 31);
                    pairs += p;
                }
                const bool all_sure = __all_sync(0xffffffffu, sure);
                if (lane == src) {
                    count = pairs;
                    n_ent = ents;
                    defer = !all_sure;
                }
            }
        }
        __syncwarp();  // the tall sweeps' entries (written by every lane) visible to their owners
        // deferred Gaussians: appended to the float64 path's queue (warp-aggregated)
        const uint32_t dmask = __ballot_sync(0xffffffffu, defer);
        if (dmask) {
            uint32_t base = 0;
            if (lane == __ffs(dmask) - 1) base = atomicAdd(queue_n, (uint32_t)__popc(dmask));
            base = __shfl_sync(0xffffffffu, base, __ffs(dmask) - 1);
            if (defer) queue[base + __popc(dmask & ((1u << lane) - 1u))] = (uint32_t)i;
        }
        if (defer) continue;
        if (count > 0) {
            write_records((size_t)i, MODE, x2d, y2d, a, b, c, td, mo.w, R, count, n_ent, n_span, span_inline, cols,
                          s_pay[threadIdx.x], rec, erec);
            const uint32_t key = __float_as_uint(pz);
            depth_key[i] = key;
            gne[i] = n_ent;
#pragma unroll
            for (int p = 0; p < kDepthPasses; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 0xFF], 1u);
            ++my_vis;
            my_pairs += count;
        } else if (valid) {
            depth_key[i] = kNoTiles;
            gne[i] = 0u;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_vis += __shfl_xor_sync(0xffffffffu, my_vis, o);
        my_pairs += __shfl_xor_sync(0xffffffffu, my_pairs, o);
    }
    if ((threadIdx.x & 31) == 0 && my_vis) {
        atomicAdd(&s_vis, my_vis);
        atomicAdd(&s_pairs, my_pairs);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kDepthPasses * 256; k += blockDim.x) {
        const uint32_t v = (&s_hist[0][0])[k];
        if (v) atomicAdd(hist + k, v);
    }
    if (threadIdx.x == 0 && s_vis) {
        atomicAdd(n_visible, s_vis);
        atomicAdd(total_pairs, s_pairs);
    }
}

}  // namespace

cudaError_t launch_preprocess(const ss_scene &sc, const CamArgs &cam, int mode, void *ws, const Layout &L,
                              cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (sc.n == 0) return cudaSuccess;
    const int sms = sm_count();
    const int blocks_needed = (sc.n + kPreThreads - 1) / kPreThreads;
    ColorSrc csrc;
    csrc.mean_opac = reinterpret_cast<const float4 *>(sc.mean_opac);
    csrc.sh = reinterpret_cast<const float4 *>(sc.sh);
    csrc.cpx = cam.cpx;
    csrc.cpy = cam.cpy;
    csrc.cpz = cam.cpz;
    csrc.deg = sc.sh_degree;
    const float4 *mo = reinterpret_cast<const float4 *>(sc.mean_opac), *scl = reinterpret_cast<const float4 *>(sc.scale),
                 *rot = reinterpret_cast<const float4 *>(sc.rot);
    uint32_t *queue = at<uint32_t>(ws, L.pre_queue), *queue_n = at<uint32_t>(ws, L.pre_queue_n);
#define SS_PRE64_ARGS(Q, QN)                                                                                   \
    sc.n, Q, QN, mo, scl, rot, cam, mode, at<float4>(ws, P.rec), at<uint4>(ws, P.erec),                      \
        at<uint32_t>(ws, P.depth_key), at<uint32_t>(ws, L.gne), at<uint32_t>(ws, L.hist_depth),               \
        at<uint32_t>(ws, P.n_visible), at<uint32_t>(ws, P.total_pairs), csrc, at<ColorSrc>(ws, L.color_src)
    cudaError_t e = cudaSuccess;
    if (mode == SS_BIN_3SIGMA) {  // every Gaussian on the float64 path
        const int resident = sms * kPreBlocks;  // one round of resident CTAs (persistent)
        const int grid = blocks_needed < resident ? blocks_needed : resident;
        launch_pdl(k_preprocess64, grid, kPreThreads, 0, st, SS_PRE64_ARGS(nullptr, nullptr));
        return cudaGetLastError();
    }
#ifndef SS_PRE_GRID
#define SS_PRE_GRID kPre32Blocks
#endif
    const int resident = sms * SS_PRE_GRID;  // one round of resident CTAs (persistent)
    const int grid = blocks_needed < resident ? blocks_needed : resident;
    if (mode == SS_BIN_ACCUTILE)
        launch_pdl(k_preprocess32<SS_BIN_ACCUTILE>, grid, kPreThreads, 0, st, sc.n, mo, scl, rot, cam,
                   at<float4>(ws, P.rec), at<uint4>(ws, P.erec), at<uint32_t>(ws, P.depth_key), at<uint32_t>(ws, L.gne),
                   at<uint32_t>(ws, L.hist_depth), at<uint32_t>(ws, P.n_visible), at<uint32_t>(ws, P.total_pairs),
                   queue, queue_n, at<uint32_t>(ws, L.pre_ticket), csrc, at<ColorSrc>(ws, L.color_src));
    else
        launch_pdl(k_preprocess32<SS_BIN_SNUGBOX>, grid, kPreThreads, 0, st, sc.n, mo, scl, rot, cam,
                   at<float4>(ws, P.rec), at<uint4>(ws, P.erec), at<uint32_t>(ws, P.depth_key), at<uint32_t>(ws, L.gne),
                   at<uint32_t>(ws, L.hist_depth), at<uint32_t>(ws, P.n_visible), at<uint32_t>(ws, P.total_pairs),
                   queue, queue_n, at<uint32_t>(ws, L.pre_ticket), csrc, at<ColorSrc>(ws, L.color_src));
    // the deferred Gaussians on the float64 path (a few CTAs; the queue length is on the device)
    launch_pdl(k_preprocess64, sms * kPreBlocks, kPreThreads, 0, st, SS_PRE64_ARGS(queue, queue_n));
    if (e != cudaSuccess) return e;
#undef SS_PRE64_ARGS
    return cudaGetLastError();
}

}  // namespace ss
