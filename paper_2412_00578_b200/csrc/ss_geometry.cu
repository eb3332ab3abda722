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
#include "ss_common.cuh"

namespace ss {
namespace {

// ---------------------------------------------------------------- tile geometry (float64)
// R8: "dividing by tile size, rounding, and clipping to the image boundary":
// half-open span [floor(lo/16), floor(hi/16)+1) clipped to [0, tiles].
__device__ __forceinline__ void edge_span(double lo, double hi, int tiles, int &s0, int &s1) {
    double f0 = floor(lo / kTile), f1 = floor(hi / kTile) + 1.0;
    if (!(f0 > 0.0)) f0 = 0.0;
    if (!(f1 > 0.0)) f1 = 0.0;
    if (f0 > tiles) f0 = tiles;
    if (f1 > tiles) f1 = tiles;
    s0 = (int)f0;
    s1 = (int)f1;
}

// SnugBox (Sec. 4.1.1, Eqs. 15-16): exact bbox of a xd^2 + 2b xd yd + c yd^2 = t (Eq. 14);
// half-extents sqrt(t c / D), sqrt(t a / D), D = ac - b^2.  Tangent points (R11).
struct Snug {
    double xmin, xmax, ymin, ymax;
    double yl, yr;   // y of the x_min / x_max tangent points (B_l, B_r)
    double xt, xb;   // x of the y_min / y_max tangent points (B_t, B_b)
};

__device__ __forceinline__ Snug snugbox(double mx, double my, double a, double b, double c, double t) {
    double D = a * c - b * b;
    double hx = sqrt(t * c / D);
    double hy = sqrt(t * a / D);
    Snug s;
    s.xmin = mx - hx;
    s.xmax = mx + hx;
    s.ymin = my - hy;
    s.ymax = my + hy;
    s.yl = my + b * hx / c;
    s.yr = my - b * hx / c;
    s.xt = mx + b * hy / a;
    s.xb = mx - b * hy / a;
    return s;
}

__device__ __forceinline__ int4 rect_of_snug(const Snug &s, int tiles_x, int tiles_y) {
    int4 r;
    edge_span(s.xmin, s.xmax, tiles_x, r.x, r.y);
    edge_span(s.ymin, s.ymax, tiles_y, r.z, r.w);
    return r;
}

// 3D-GS baseline (Eq. 8): r = ceil(3 sqrt(lambda_max)), square mu +- r (R6, R7).
__device__ __forceinline__ int4 rect_3sigma(double mx, double my, double cxx, double cxy, double cyy, int tiles_x,
                                            int tiles_y) {
    double m = 0.5 * (cxx + cyy);
    double det = cxx * cyy - cxy * cxy;
    double disc = m * m - det;
    if (disc < 0.0) disc = 0.0;
    double lmax = m + sqrt(disc);
    double r = ceil(3.0 * sqrt(lmax));
    int4 R;
    edge_span(mx - r, mx + r, tiles_x, R.x, R.y);
    edge_span(my - r, my + r, tiles_y, R.z, R.w);
    return R;
}

// Eq. 15 on a line of the swept axis: u = (-b v +- sqrt((b^2 - a_f c_s) v^2 + t a_f)) / a_f.
__device__ __forceinline__ void intersect_line(double m_free, double m_line, double a_free, double b, double c_line,
                                               double t, double line, double &lo, double &hi) {
    double v = line - m_line;
    double disc = (b * b - a_free * c_line) * v * v + t * a_free;
    if (disc < 0.0) disc = 0.0;  // R12
    double s = sqrt(disc);
    lo = m_free + (-b * v - s) / a_free;
    hi = m_free + (-b * v + s) / a_free;
}

// AccuTile, Algorithm 1 along the shorter side of the SnugBox tile rect (R9),
// the columns path by the a<->c / x<->y swap.  R10: a boundary line outside the
// bbox yields the neutral pair (+inf, -inf).  Calls emit(tile_id) per tile; returns count.
template <class Emit>
__device__ __forceinline__ uint32_t accutile(double mx, double my, double a, double b, double c, double t,
                                             int tiles_x, int tiles_y, Emit emit) {
    Snug S = snugbox(mx, my, a, b, c, t);
    int4 R = rect_of_snug(S, tiles_x, tiles_y);
    if (R.x >= R.y || R.z >= R.w) return 0;
    const bool rows = (R.w - R.z) <= (R.y - R.x);
    double mf, ms, af, cs, ext_lo, ext_hi, smin, smax, tmin_s, tmax_s;
    int s0, s1, f0, f1;
    if (rows) {
        mf = mx; ms = my; af = a; cs = c;
        ext_lo = S.xmin; ext_hi = S.xmax; smin = S.ymin; smax = S.ymax;
        tmin_s = S.yl; tmax_s = S.yr;
        s0 = R.z; s1 = R.w; f0 = R.x; f1 = R.y;
    } else {
        mf = my; ms = mx; af = c; cs = a;
        ext_lo = S.ymin; ext_hi = S.ymax; smin = S.xmin; smax = S.xmax;
        tmin_s = S.xt; tmax_s = S.xb;
        s0 = R.x; s1 = R.y; f0 = R.z; f1 = R.w;
    }
    uint32_t C = 0;
    double imin_lo = __longlong_as_double(0x7ff0000000000000ll);   // +inf
    double imin_hi = __longlong_as_double(0xfff0000000000000ll);   // -inf
    double line_min = (double)(s0 * kTile);
    if (line_min >= smin) intersect_line(mf, ms, af, b, cs, t, line_min, imin_lo, imin_hi);
    for (int r = s0; r < s1; ++r) {
        double imax_lo = __longlong_as_double(0x7ff0000000000000ll);
        double imax_hi = __longlong_as_double(0xfff0000000000000ll);
        double line_max = (double)((r + 1) * kTile);
        if (line_max <= smax) intersect_line(mf, ms, af, b, cs, t, line_max, imax_lo, imax_hi);
        double lo_r = (double)(r * kTile), hi_r = (double)((r + 1) * kTile);
        double e_min = (tmin_s >= lo_r && tmin_s < hi_r) ? ext_lo : (imin_lo < imax_lo ? imin_lo : imax_lo);
        double e_max = (tmax_s >= lo_r && tmax_s < hi_r) ? ext_hi : (imin_hi > imax_hi ? imin_hi : imax_hi);
        double g0 = floor(e_min / kTile), g1 = floor(e_max / kTile) + 1.0;
        if (!(g0 > f0)) g0 = f0;
        if (g0 > f1) g0 = f1;
        if (!(g1 > f0)) g1 = f0;
        if (g1 > f1) g1 = f1;
        const int tmin = (int)g0, tmax = (int)g1;
        for (int k = tmin; k < tmax; ++k) emit(rows ? (uint32_t)(r * tiles_x + k) : (uint32_t)(k * tiles_x + r));
        if (tmax > tmin) C += (uint32_t)(tmax - tmin);
        imin_lo = imax_lo;  // i_min <- i_max
        imin_hi = imax_hi;
    }
    return C;
}

// Tile set of a stored record (count when emit is a no-op).  3-sigma / SnugBox: the rect.
template <class Emit>
__device__ __forceinline__ uint32_t tiles_of_record(int mode, float x, float y, float a, float b, float c,
                                                    float sigma, int4 R, int tiles_x, int tiles_y, Emit emit) {
    if (mode == SS_BIN_ACCUTILE) {
        double t = 2.0 * log(255.0 * (double)sigma);  // Eq. 11 (R2)
        return accutile((double)x, (double)y, (double)a, (double)b, (double)c, t, tiles_x, tiles_y, emit);
    }
    uint32_t C = 0;
    for (int ty = R.z; ty < R.w; ++ty)
        for (int tx = R.x; tx < R.y; ++tx) {
            emit((uint32_t)(ty * tiles_x + tx));
            ++C;
        }
    return C;
}

struct NoEmit {
    __device__ __forceinline__ void operator()(uint32_t) const {}
};

// ---------------------------------------------------------------- SH basis (R13)
template <int DEG>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float *Y) {
    Y[0] = 0.28209479177387814f;
    if (DEG < 1) return;
    const float C1 = 0.4886025119029199f;
    Y[1] = -C1 * y;
    Y[2] = C1 * z;
    Y[3] = -C1 * x;
    if (DEG < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = 1.0925484305920792f * xy;
    Y[5] = -1.0925484305920792f * yz;
    Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * xz;
    Y[8] = 0.5462742152960396f * (xx - yy);
    if (DEG < 3) return;
    Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    Y[10] = 2.890611442640554f * xy * z;
    Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

// ---------------------------------------------------------------- a1 preprocess kernel
// One thread per Gaussian ("each thread processes a single Gaussian"), persistent
// grid-stride loop so each CTA flushes its depth-digit histograms once.
template <int DEG>
__global__ void __launch_bounds__(256) k_preprocess(int n, const float4 *__restrict__ mean_opac,
                                                    const float4 *__restrict__ scale, const float4 *__restrict__ rot,
                                                    const float4 *__restrict__ sh, CamArgs cam, int mode,
                                                    float4 *__restrict__ rec, uint4 *__restrict__ bininfo,
                                                    uint32_t *__restrict__ depth_key, uint32_t *__restrict__ hist,
                                                    uint32_t *__restrict__ n_visible) {
    __shared__ uint32_t s_hist[kDepthPasses][256];
    __shared__ uint32_t s_vis;
    for (int k = threadIdx.x; k < kDepthPasses * 256; k += blockDim.x) (&s_hist[0][0])[k] = 0;
    if (threadIdx.x == 0) s_vis = 0;
    __syncthreads();
    constexpr int NB = (DEG + 1) * (DEG + 1);
    constexpr int NP = (NB * 3 + 3) / 4;
    uint32_t my_vis = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t count = 0;
        const float4 mo = mean_opac[i];
        const float px = cam.V[0] * mo.x + cam.V[1] * mo.y + cam.V[2] * mo.z + cam.V[3];
        const float py = cam.V[4] * mo.x + cam.V[5] * mo.y + cam.V[6] * mo.z + cam.V[7];
        const float pz = cam.V[8] * mo.x + cam.V[9] * mo.y + cam.V[10] * mo.z + cam.V[11];
        float x2d = 0.f, y2d = 0.f, a = 0.f, b = 0.f, c = 0.f, rgb0 = 0.f, rgb1 = 0.f, rgb2 = 0.f;
        double td = 0.0;
        int4 R = make_int4(0, 0, 0, 0);
        if (pz >= cam.z_near) {
            const float tx = px / pz, ty = py / pz;
            x2d = cam.fx * tx + cam.cx;
            y2d = cam.fy * ty + cam.cy;
            float txc = tx, tyc = ty;
            if (cam.clip > 0.0f) {
                const float limx = cam.clip * ((0.5f * (float)cam.W) / cam.fx);
                const float limy = cam.clip * ((0.5f * (float)cam.H) / cam.fy);
                txc = fminf(limx, fmaxf(-limx, tx));
                tyc = fminf(limy, fmaxf(-limy, ty));
            }
            const float j00 = cam.fx / pz, j02 = -(cam.fx * txc) / pz;
            const float j11 = cam.fy / pz, j12 = -(cam.fy * tyc) / pz;
            const float4 q4 = rot[i];
            const float4 s4 = scale[i];
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
            float cxx = U[0][0] * T[0][0] + U[0][1] * T[0][1] + U[0][2] * T[0][2];
            const float cxy = U[0][0] * T[1][0] + U[0][1] * T[1][1] + U[0][2] * T[1][2];
            float cyy = U[1][0] * T[1][0] + U[1][1] * T[1][1] + U[1][2] * T[1][2];
            cxx = cxx + 0.3f;  // R5
            cyy = cyy + 0.3f;
            const float det = cxx * cyy - cxy * cxy;
            if (det > 0.0f) {
                const float inv = 1.0f / det;
                a = cyy * inv;
                b = -cxy * inv;
                c = cxx * inv;
                const double D = (double)a * (double)c - (double)b * (double)b;
                td = 2.0 * log(255.0 * (double)mo.w);  // Eq. 11 (R2)
                if (D > 0.0 && (mode == SS_BIN_3SIGMA || td > 0.0)) {
                    if (mode == SS_BIN_3SIGMA)
                        R = rect_3sigma((double)x2d, (double)y2d, (double)cxx, (double)cxy, (double)cyy, cam.tiles_x,
                                        cam.tiles_y);
                    else
                        R = rect_of_snug(snugbox((double)x2d, (double)y2d, (double)a, (double)b, (double)c, td),
                                         cam.tiles_x, cam.tiles_y);
                    count = tiles_of_record(mode, x2d, y2d, a, b, c, mo.w, R, cam.tiles_x, cam.tiles_y, NoEmit());
                }
            }
        }
        if (count > 0) {
            // colour (R13): only Gaussians with tiles read their SH planes
            const float dx = mo.x - cam.cpx, dy = mo.y - cam.cpy, dz = mo.z - cam.cpz;
            const float len = sqrtf(dx * dx + dy * dy + dz * dz);
            float Y[16];
            sh_basis<DEG>(dx / len, dy / len, dz / len, Y);
            float hc[NP * 4];
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float4 v = __ldg(sh + (size_t)p * n + i);
                hc[4 * p + 0] = v.x;
                hc[4 * p + 1] = v.y;
                hc[4 * p + 2] = v.z;
                hc[4 * p + 3] = v.w;
            }
            float acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                acc0 = acc0 + Y[k] * hc[3 * k + 0];
                acc1 = acc1 + Y[k] * hc[3 * k + 1];
                acc2 = acc2 + Y[k] * hc[3 * k + 2];
            }
            acc0 = acc0 + 0.5f;
            acc1 = acc1 + 0.5f;
            acc2 = acc2 + 0.5f;
            rgb0 = acc0 > 0.0f ? acc0 : 0.0f;
            rgb1 = acc1 > 0.0f ? acc1 : 0.0f;
            rgb2 = acc2 > 0.0f ? acc2 : 0.0f;
            rec[3 * (size_t)i + 0] = make_float4(x2d, y2d, a, b);
            rec[3 * (size_t)i + 1] = make_float4(c, (float)td, mo.w, pz);
            rec[3 * (size_t)i + 2] = make_float4(rgb0, rgb1, rgb2, 0.0f);
            bininfo[i] = make_uint4((uint32_t)R.x | ((uint32_t)R.y << 16), (uint32_t)R.z | ((uint32_t)R.w << 16),
                                    count, 0u);
            const uint32_t key = __float_as_uint(pz);
            depth_key[i] = key;
#pragma unroll
            for (int p = 0; p < kDepthPasses; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 0xFF], 1u);
            ++my_vis;
        } else {
            bininfo[i] = make_uint4(0u, 0u, 0u, 0u);
            depth_key[i] = kNoTiles;
        }
    }
    // warp-aggregate the visible count, then one atomic per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_vis += __shfl_xor_sync(0xffffffffu, my_vis, o);
    if ((threadIdx.x & 31) == 0 && my_vis) atomicAdd(&s_vis, my_vis);
    __syncthreads();
    for (int k = threadIdx.x; k < kDepthPasses * 256; k += blockDim.x) {
        const uint32_t v = (&s_hist[0][0])[k];
        if (v) atomicAdd(hist + k, v);
    }
    if (threadIdx.x == 0 && s_vis) atomicAdd(n_visible, s_vis);
}

// ---------------------------------------------------------------- a2+a3 emission kernel
// Thread k handles the k-th visible Gaussian in (depth, index) order; its tile count is
// exclusive-scanned across the grid with a decoupled look-back (block tickets assigned in
// launch order), then its tiles are re-enumerated by tiles_of_record -- the very function
// that produced the count -- and written at the offset.  A per-CTA tile histogram (shared
// memory) feeds the tile sort and the ranges.
__global__ void __launch_bounds__(kEmitThreads) k_emit(int mode, const float4 *__restrict__ rec,
                                                       const uint4 *__restrict__ bininfo,
                                                       const uint32_t *__restrict__ order,
                                                       const uint32_t *__restrict__ n_visible, uint32_t cap,
                                                       uint16_t *__restrict__ pair_tile,
                                                       uint32_t *__restrict__ pair_value, uint32_t *tile_count,
                                                       uint32_t *lookback, uint32_t *ticket, uint32_t *total_pairs,
                                                       uint32_t *overflow, int tiles_x, int tiles_y, int n_tiles,
                                                       int smem_hist) {
    extern __shared__ uint32_t s_tile_hist[];
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_bid, s_base;
    for (int t = threadIdx.x; t < (smem_hist ? n_tiles : 0); t += blockDim.x) s_tile_hist[t] = 0;
    const uint32_t nv = *n_visible;
    uint32_t *hist = smem_hist ? s_tile_hist : tile_count;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t bid = s_bid;
        if ((size_t)bid * kEmitThreads >= nv) break;
        const uint32_t k = bid * kEmitThreads + threadIdx.x;
        uint32_t g = 0, cnt = 0;
        uint4 bi = make_uint4(0, 0, 0, 0);
        if (k < nv) {
            g = order[k];
            bi = bininfo[g];
            cnt = bi.z;
        }
        uint32_t total;
        const uint32_t excl = block_exclusive_scan_256(cnt, s_warp, total);
        if (threadIdx.x == 0) {
            // decoupled look-back over the preceding CTAs' published sums
            volatile uint32_t *lb = lookback;
            if (bid == 0) {
                lb[0] = kFlagInc | total;
                s_base = 0;
            } else {
                lb[bid] = kFlagAgg | total;
                uint32_t acc = 0;
                int p = (int)bid - 1;
                for (;;) {
                    uint32_t v;
                    do { v = lb[p]; } while ((v & ~kValMask) == 0);
                    acc += v & kValMask;
                    if ((v & ~kValMask) == kFlagInc) break;
                    --p;
                }
                lb[bid] = kFlagInc | (acc + total);
                s_base = acc;
            }
            if ((bid + 1) * kEmitThreads >= nv) {  // the CTA holding the last visible Gaussian
                const uint32_t P = s_base + total;
                *total_pairs = P;
                *overflow = P > cap ? 1u : 0u;
            }
        }
        __syncthreads();
        if (cnt) {
            const uint32_t off = s_base + excl;
            const float4 r0 = rec[3 * (size_t)g + 0];
            const float4 r1 = rec[3 * (size_t)g + 1];
            const int4 R = make_int4((int)(bi.x & 0xFFFF), (int)(bi.x >> 16), (int)(bi.y & 0xFFFF), (int)(bi.y >> 16));
            uint32_t j = 0;
            tiles_of_record(mode, r0.x, r0.y, r0.z, r0.w, r1.x, r1.z, R, tiles_x, tiles_y, [&](uint32_t tile) {
                const uint32_t o = off + j;
                if (o < cap) {
                    pair_tile[o] = (uint16_t)tile;
                    pair_value[o] = g;
                }
                atomicAdd(hist + tile, 1u);
                ++j;
            });
        }
    }
    if (smem_hist) {
        __syncthreads();
        for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
            const uint32_t v = s_tile_hist[t];
            if (v) atomicAdd(tile_count + t, v);
        }
    }
}

}  // namespace

cudaError_t launch_preprocess(const ss_scene &sc, const CamArgs &cam, int mode, void *ws, const Layout &L,
                              cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (sc.n == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks_needed = (sc.n + 255) / 256;
    const int grid = blocks_needed < sms * 8 ? blocks_needed : sms * 8;
#define SS_PRE_ARGS                                                                                       \
    sc.n, reinterpret_cast<const float4 *>(sc.mean_opac), reinterpret_cast<const float4 *>(sc.scale),         \
        reinterpret_cast<const float4 *>(sc.rot), reinterpret_cast<const float4 *>(sc.sh), cam, mode,         \
        at<float4>(ws, P.rec), at<uint4>(ws, P.bininfo), at<uint32_t>(ws, P.depth_key),                      \
        at<uint32_t>(ws, L.hist_depth), at<uint32_t>(ws, P.n_visible)
    switch (sc.sh_degree) {
        case 0: k_preprocess<0><<<grid, 256, 0, st>>>(SS_PRE_ARGS); break;
        case 1: k_preprocess<1><<<grid, 256, 0, st>>>(SS_PRE_ARGS); break;
        case 2: k_preprocess<2><<<grid, 256, 0, st>>>(SS_PRE_ARGS); break;
        default: k_preprocess<3><<<grid, 256, 0, st>>>(SS_PRE_ARGS); break;
    }
#undef SS_PRE_ARGS
    return cudaGetLastError();
}

cudaError_t launch_emit(const CamArgs &cam, int mode, void *ws, const Layout &L, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0 || L.nblk_emit == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem_hist = P.n_tiles <= 12288 ? 1 : 0;
    const size_t smem = smem_hist ? (size_t)P.n_tiles * 4 : 0;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)L.nblk_emit < sms * 4 ? (int)L.nblk_emit : sms * 4;
    k_emit<<<grid, kEmitThreads, smem, st>>>(
        mode, at<const float4>(ws, P.rec), at<const uint4>(ws, P.bininfo), at<const uint32_t>(ws, P.order),
        at<const uint32_t>(ws, P.n_visible), L.capacity,
        at<uint16_t>(ws, P.pair_tile), at<uint32_t>(ws, P.pair_value), at<uint32_t>(ws, P.tile_count),
        at<uint32_t>(ws, L.lb_emit), at<uint32_t>(ws, L.counters) + 8, at<uint32_t>(ws, P.total_pairs),
        at<uint32_t>(ws, P.overflow), cam.tiles_x, cam.tiles_y, P.n_tiles, smem_hist);
    return cudaGetLastError();
}

}  // namespace ss
