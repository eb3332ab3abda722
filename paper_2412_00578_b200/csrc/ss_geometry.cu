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
    double hx, hy;   // half-extents sqrt(t c / D), sqrt(t a / D)
    double xmin, xmax, ymin, ymax;
    double yl, yr;   // y of the x_min / x_max tangent points (B_l, B_r)
    double xt, xb;   // x of the y_min / y_max tangent points (B_t, B_b)
};

__device__ __forceinline__ Snug snugbox(double mx, double my, double a, double b, double c, double t) {
    // contract R1: one reciprocal each of D, a and c; quotients are products with them
    double D = a * c - b * b;
    double rD = 1.0 / D;
    double hx = sqrt(t * c * rD);
    double hy = sqrt(t * a * rD);
    double ia = 1.0 / a, ic = 1.0 / c;
    Snug s;
    s.hx = hx;
    s.hy = hy;
    s.xmin = mx - hx;
    s.xmax = mx + hx;
    s.ymin = my - hy;
    s.ymax = my + hy;
    s.yl = my + b * hx * ic;
    s.yr = my - b * hx * ic;
    s.xt = mx + b * hy * ia;
    s.xb = mx - b * hy * ia;
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
    double ia = 1.0 / a_free;
    lo = m_free + (-b * v - s) * ia;
    hi = m_free + (-b * v + s) * ia;
}

// AccuTile, Algorithm 1 along the shorter side of the SnugBox tile rect (R9),
// the columns path by the a<->c / x<->y swap.  R10: a boundary line outside the
// bbox yields the neutral pair (+inf, -inf).
struct Sweep {
    bool rows;                                        // rows path (else columns)
    double mf, ms, af, cs, b, t;                      // free/swept-axis centre and coefficients
    double ext_lo, ext_hi, smin, smax, tmin_s, tmax_s;
    int s0, s1, f0, f1;                               // swept lines [s0, s1), free span [f0, f1)
};

__device__ __forceinline__ bool accutile_setup_from(const Snug &S, const int4 &R, double mx, double my, double a,
                                                    double b, double c, double t, Sweep &w) {
    if (R.x >= R.y || R.z >= R.w) return false;
    w.rows = (R.w - R.z) <= (R.y - R.x);
    w.b = b;
    w.t = t;
    if (w.rows) {
        w.mf = mx; w.ms = my; w.af = a; w.cs = c;
        w.ext_lo = S.xmin; w.ext_hi = S.xmax; w.smin = S.ymin; w.smax = S.ymax;
        w.tmin_s = S.yl; w.tmax_s = S.yr;
        w.s0 = R.z; w.s1 = R.w; w.f0 = R.x; w.f1 = R.y;
    } else {
        w.mf = my; w.ms = mx; w.af = c; w.cs = a;
        w.ext_lo = S.ymin; w.ext_hi = S.ymax; w.smin = S.xmin; w.smax = S.xmax;
        w.tmin_s = S.xt; w.tmax_s = S.xb;
        w.s0 = R.x; w.s1 = R.y; w.f0 = R.z; w.f1 = R.w;
    }
    return true;
}

__device__ __forceinline__ bool accutile_setup(double mx, double my, double a, double b, double c, double t,
                                               int tiles_x, int tiles_y, Sweep &w) {
    const Snug S = snugbox(mx, my, a, b, c, t);
    const int4 R = rect_of_snug(S, tiles_x, tiles_y);
    return accutile_setup_from(S, R, mx, my, a, b, c, t, w);
}

// Intersections(line, E) or the neutral pair when the algorithm does not compute it.
__device__ __forceinline__ void sweep_line(const Sweep &w, double line, bool compute, double &lo, double &hi) {
    lo = __longlong_as_double(0x7ff0000000000000ll);   // +inf
    hi = __longlong_as_double(0xfff0000000000000ll);   // -inf
    if (compute) intersect_line(w.mf, w.ms, w.af, w.b, w.cs, w.t, line, lo, hi);
}

// One row (or column) r of Algorithm 1 given i_min (its lower boundary line) and i_max (its
// upper boundary line): e_min / e_max, Convert, clip to the rect.  Returns [tmin, tmax).
__device__ __forceinline__ void sweep_row(const Sweep &w, int r, double imin_lo, double imin_hi, double imax_lo,
                                          double imax_hi, int &tmin, int &tmax) {
    const double lo_r = (double)(r * kTile), hi_r = (double)((r + 1) * kTile);
    const double e_min = (w.tmin_s >= lo_r && w.tmin_s < hi_r) ? w.ext_lo : (imin_lo < imax_lo ? imin_lo : imax_lo);
    const double e_max = (w.tmax_s >= lo_r && w.tmax_s < hi_r) ? w.ext_hi : (imin_hi > imax_hi ? imin_hi : imax_hi);
    double g0 = floor(e_min / kTile), g1 = floor(e_max / kTile) + 1.0;
    if (!(g0 > w.f0)) g0 = w.f0;
    if (g0 > w.f1) g0 = w.f1;
    if (!(g1 > w.f0)) g1 = w.f0;
    if (g1 > w.f1) g1 = w.f1;
    tmin = (int)g0;
    tmax = (int)g1;
}

// Algorithm 1 in count mode on a prepared sweep (same loop as the sequential form below).
// One span (row or column of the sweep) packed in 32 bits: first tile id (16 bits), length
// (bits 16..24, <= 256), column-step flag (bit 31: consecutive tiles are tiles_x apart).
__device__ __forceinline__ uint32_t pack_span(const Sweep &w, int r, int tmin, int tmax, int tiles_x) {
    const uint32_t len = tmax > tmin ? (uint32_t)(tmax - tmin) : 0u;
    const uint32_t first = len == 0 ? 0u : (w.rows ? (uint32_t)(r * tiles_x + tmin) : (uint32_t)(tmin * tiles_x + r));
    return first | (len << 16) | (w.rows ? 0u : 0x80000000u);
}

// Algorithm 1 in count mode on a prepared sweep (the sequential loop, i_min <- i_max); the
// first kInlineSpans spans are also returned packed (for the emission record).
__device__ __forceinline__ uint32_t accutile_count(const Sweep &w, int tiles_x, uint32_t *spans) {
    uint32_t C = 0;
    double imin_lo, imin_hi;
    const double line_min = (double)(w.s0 * kTile);
    sweep_line(w, line_min, line_min >= w.smin, imin_lo, imin_hi);
    for (int r = w.s0; r < w.s1; ++r) {
        double imax_lo, imax_hi;
        const double line_max = (double)((r + 1) * kTile);
        sweep_line(w, line_max, line_max <= w.smax, imax_lo, imax_hi);
        int tmin, tmax;
        sweep_row(w, r, imin_lo, imin_hi, imax_lo, imax_hi, tmin, tmax);
        if (tmax > tmin) C += (uint32_t)(tmax - tmin);
        const int j = r - w.s0;
#pragma unroll
        for (int q = 0; q < kInlineSpans; ++q)
            if (j == q) spans[q] = pack_span(w, r, tmin, tmax, tiles_x);
        imin_lo = imax_lo;
        imin_hi = imax_hi;
    }
    return C;
}

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
__global__ void __launch_bounds__(256, 2) k_preprocess(int n, const float4 *__restrict__ mean_opac,
                                                    const float4 *__restrict__ scale, const float4 *__restrict__ rot,
                                                    const float4 *__restrict__ sh, CamArgs cam, int mode,
                                                    float4 *__restrict__ rec, uint4 *__restrict__ erec,
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
    // camera constants of the J clamp (R5), the same values the per-Gaussian form would give
    const float limx = cam.clip * ((0.5f * (float)cam.W) / cam.fx);
    const float limy = cam.clip * ((0.5f * (float)cam.H) / cam.fy);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t count = 0;
        const float4 mo = mean_opac[i];
        const float4 q4 = rot[i];    // issued with the mean: one memory round trip, not two
        const float4 s4 = scale[i];
        const float px = cam.V[0] * mo.x + cam.V[1] * mo.y + cam.V[2] * mo.z + cam.V[3];
        const float py = cam.V[4] * mo.x + cam.V[5] * mo.y + cam.V[6] * mo.z + cam.V[7];
        const float pz = cam.V[8] * mo.x + cam.V[9] * mo.y + cam.V[10] * mo.z + cam.V[11];
        float x2d = 0.f, y2d = 0.f, a = 0.f, b = 0.f, c = 0.f, rgb0 = 0.f, rgb1 = 0.f, rgb2 = 0.f;
        double td = 0.0;
        int4 R = make_int4(0, 0, 0, 0);
        Snug snug;
        snug.hx = snug.hy = 0.0;
        uint32_t spans[kInlineSpans] = {0u, 0u, 0u, 0u};
        uint32_t nspans = 0, cols = 0;
        if (pz >= cam.z_near) {
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
                            count = accutile_count(w, cam.tiles_x, spans);
                            nspans = (uint32_t)(w.s1 - w.s0);
                            cols = w.rows ? 0u : 1u;
                        }
                    } else if (R.x < R.y && R.z < R.w) {
                        count = (uint32_t)((R.y - R.x) * (R.w - R.z));
                        nspans = (uint32_t)(R.w - R.z);
#pragma unroll
                        for (int q = 0; q < kInlineSpans; ++q)
                            if (q < (int)nspans)
                                spans[q] = (uint32_t)((R.z + q) * cam.tiles_x + R.x) | ((uint32_t)(R.y - R.x) << 16);
                    }
                }
            }
        }
        if (count > 0) {
            // colour (R13): only Gaussians with tiles read their SH planes
            const float dx = mo.x - cam.cpx, dy = mo.y - cam.cpy, dz = mo.z - cam.cpz;
            const float len = sqrtf(dx * dx + dy * dy + dz * dz);
            const float il = 1.0f / len;
            float Y[16];
            sh_basis<DEG>(dx * il, dy * il, dz * il, Y);
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
            // render record (48 B): q0 (x, y, a, b) | q1 (c, t, sigma, 0) | q2 (0, r, g, b)
            float4 *q = rec + 3 * (size_t)i;
            q[0] = make_float4(x2d, y2d, a, b);
            q[1] = make_float4(c, (float)td, mo.w, 0.0f);
            q[2] = make_float4(0.0f, rgb0, rgb1, rgb2);
            // emission record (32 B, one sector): e0 (count, info, span0, span1), e1 (span2, span3,
            // aux0, aux1); info = nspans | inline flag << 8 | columns flag << 9; aux = t as float64
            // bits (AccuTile) or the packed rect (x0, x1-x0-1, y0, y1-y0-1) for the fallback path.
            uint32_t aux0, aux1;
            if (mode == SS_BIN_ACCUTILE) {
                aux0 = (uint32_t)__double2loint(td);
                aux1 = (uint32_t)__double2hiint(td);
            } else {
                aux0 = (uint32_t)R.x | ((uint32_t)(R.y - R.x - 1) << 8) | ((uint32_t)R.z << 16) |
                       ((uint32_t)(R.w - R.z - 1) << 24);
                aux1 = 0u;
            }
            const uint32_t info = nspans | (nspans <= (uint32_t)kInlineSpans ? 0x100u : 0u) | (cols << 9);
            erec[2 * (size_t)i + 0] = make_uint4(count, info, spans[0], spans[1]);
            erec[2 * (size_t)i + 1] = make_uint4(spans[2], spans[3], aux0, aux1);
            const uint32_t key = __float_as_uint(pz);
            depth_key[i] = key;
#pragma unroll
            for (int p = 0; p < kDepthPasses; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 0xFF], 1u);
            ++my_vis;
        } else {
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
// A CTA takes 256 consecutive visible Gaussians in (depth, index) order.
//  1. Their tile counts are exclusive-scanned across the grid (block scan + decoupled
//     look-back over block tickets assigned in launch order): the CTA's pairs occupy
//     [base, base + total) in Gaussian order.
//  2. Each thread runs the row (or column) loop of its Gaussian -- the same arithmetic as the
//     count of a1 (AccuTile: Algorithm 1 with the i_min <- i_max carry; 3-sigma / SnugBox: the
//     rect's rows) -- and stores one span (first tile, length, step, Gaussian) per row in
//     shared memory.  At most kSpanCap spans per round; threads that do not fit go next round.
//  3. The CTA flattens the spans (scan of lengths) and writes pair p of the round at
//     base + round_base + p, so the global writes are contiguous and every thread writes the
//     same number of pairs regardless of Gaussian size.  A per-CTA tile histogram in shared
//     memory feeds the tile sort and the ranges.
constexpr int kSpanCap = 2048;
constexpr int kEmitBlock = kEmitThreads;

// Warp-cooperative decoupled look-back: lane l inspects the status of CTA (bid - 1 - l - 32j);
// the walk stops at the nearest inclusive prefix; aggregates before it are summed.  Returns
// the exclusive prefix of CTA bid.  Called by one full warp.
__device__ __forceinline__ uint32_t warp_lookback(const uint32_t *lookback, uint32_t bid, int lane) {
    const volatile uint32_t *lb = lookback;
    uint32_t acc = 0;
    int base = (int)bid - 1;
    for (;;) {
        const int idx = base - lane;
        uint32_t v;
        int first_inc;
        uint32_t need;
        for (;;) {  // spin until every status up to the nearest inclusive one is published
            v = idx >= 0 ? lb[idx] : kFlagInc;  // before CTA 0: a virtual inclusive 0
            const uint32_t inc = __ballot_sync(0xffffffffu, (v & ~kValMask) == kFlagInc);
            const uint32_t zero = __ballot_sync(0xffffffffu, (v & ~kValMask) == 0);
            first_inc = inc ? __ffs(inc) - 1 : 32;
            need = first_inc == 32 ? 0xffffffffu : (0xffffffffu >> (31 - first_inc));
            if (!(zero & need)) break;
        }
        uint32_t part = (lane <= first_inc) ? (v & kValMask) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        acc += part;
        if (first_inc < 32) return acc;
        base -= 32;
    }
}

// Exclusive scan over the first 256 threads of a kEmitBlock CTA (the look-back warp passes 0
// and ignores the result); every thread of the CTA must call it.
__device__ __forceinline__ uint32_t emit_scan(uint32_t v, uint32_t *s_warp, uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31 && wid < 8) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < 8 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[7];
    return (wid && wid < 8 ? s_warp[wid - 1] : 0u) + x - v;
}

__global__ void __launch_bounds__(kEmitBlock, 3) k_emit(int mode, const float4 *__restrict__ rec,
                                                        const uint4 *__restrict__ erec,
                                                        const uint32_t *__restrict__ order,
                                                        const uint32_t *__restrict__ n_visible, uint32_t cap,
                                                        uint16_t *__restrict__ pair_tile,
                                                        uint32_t *__restrict__ pair_value, uint32_t *tile_count,
                                                        uint32_t *lookback, uint32_t *ticket,
                                                        uint32_t *total_pairs, uint32_t *overflow, int tiles_x,
                                                        int tiles_y, int n_tiles, int smem_hist) {
    extern __shared__ uint32_t s_tile_hist[];
    __shared__ uint32_t s_span[kSpanCap];  // first tile | len << 16 | column-step flag << 31
    __shared__ uint32_t s_gid[kSpanCap];
    __shared__ uint32_t s_pfx[kSpanCap];   // exclusive prefix of span lengths within the round
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_bid, s_base, s_nspans;
    const bool lb_warp = threadIdx.x >= kEmitThreads;
    const int lane = threadIdx.x & 31;
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
        uint4 e0 = make_uint4(0u, 0u, 0u, 0u), e1 = e0;
        if (!lb_warp && k < nv) {
            g = order[k];
            e0 = erec[2 * (size_t)g + 0];  // one aligned 32 B sector per Gaussian
            e1 = erec[2 * (size_t)g + 1];
            cnt = e0.x;
        }
        uint32_t total;
        emit_scan(cnt, s_warp, total);
        const uint32_t ns = cnt ? (e0.y & 0xFFu) : 0u;
        const bool inline_spans = (e0.y & 0x100u) != 0;
        if (threadIdx.x == 0) lookback[bid] = (bid == 0 ? kFlagInc : kFlagAgg) | total;
        bool first_round = true;
        // warp 0: decoupled look-back (run after its span generation, so that predecessors have
        // had time to publish), the inclusive prefix, and P for the last CTA
        auto emit_lookback_publish = [&]() {
            const uint32_t acc = bid == 0 ? 0u : warp_lookback(lookback, bid, lane);
            if (lane == 0) {
                if (bid > 0) {
                    volatile uint32_t *lbv = lookback;
                    lbv[bid] = kFlagInc | (acc + total);
                }
                s_base = acc;
                if ((bid + 1) * kEmitThreads >= nv) {
                    *total_pairs = acc + total;
                    *overflow = acc + total > cap ? 1u : 0u;
                }
            }
        };
        bool pending = ns > 0;
        uint32_t round_base = 0;  // pairs of this CTA written in previous rounds
        while (__syncthreads_or(pending)) {
            uint32_t span_tot;
            const uint32_t sofs = emit_scan(pending ? ns : 0u, s_warp, span_tot);
            const bool take = pending && sofs + ns <= (uint32_t)kSpanCap;
            // spans taken this round: all, or up to the first thread that does not fit
            if (threadIdx.x == 0 && span_tot <= (uint32_t)kSpanCap) s_nspans = span_tot;
            if (pending && sofs <= (uint32_t)kSpanCap && sofs + ns > (uint32_t)kSpanCap) s_nspans = sofs;
            if (take) {
                uint32_t j = sofs;
                if (inline_spans) {  // spans recorded by ss_preprocess's count
                    const uint32_t sp[kInlineSpans] = {e0.z, e0.w, e1.x, e1.y};
#pragma unroll
                    for (int q = 0; q < kInlineSpans; ++q)
                        if (q < (int)ns) {
                            s_span[j + q] = sp[q];
                            s_gid[j + q] = g;
                        }
                } else if (mode == SS_BIN_ACCUTILE) {  // rare: more rows than inline slots
                    const float4 q0 = rec[3 * (size_t)g + 0];
                    const float c = rec[3 * (size_t)g + 1].x;
                    const double t = __hiloint2double((int)e1.w, (int)e1.z);
                    Sweep w;
                    accutile_setup((double)q0.x, (double)q0.y, (double)q0.z, (double)q0.w, (double)c, t, tiles_x,
                                   tiles_y, w);
                    double imin_lo, imin_hi;
                    const double line_min = (double)(w.s0 * kTile);
                    sweep_line(w, line_min, line_min >= w.smin, imin_lo, imin_hi);
                    for (int r = w.s0; r < w.s1; ++r, ++j) {
                        double imax_lo, imax_hi;
                        const double line_max = (double)((r + 1) * kTile);
                        sweep_line(w, line_max, line_max <= w.smax, imax_lo, imax_hi);
                        int tmin, tmax;
                        sweep_row(w, r, imin_lo, imin_hi, imax_lo, imax_hi, tmin, tmax);
                        s_span[j] = pack_span(w, r, tmin, tmax, tiles_x);
                        s_gid[j] = g;
                        imin_lo = imax_lo;  // i_min <- i_max
                        imin_hi = imax_hi;
                    }
                } else {  // 3-sigma / SnugBox: the rect's rows
                    const uint32_t pr = e1.z;
                    const int x0 = (int)(pr & 0xFF), w_ = (int)((pr >> 8) & 0xFF) + 1, y0 = (int)((pr >> 16) & 0xFF);
                    for (int r = y0; r < y0 + (int)ns; ++r, ++j) {
                        s_span[j] = (uint32_t)(r * tiles_x + x0) | ((uint32_t)w_ << 16);
                        s_gid[j] = g;
                    }
                }
                pending = false;
            }
            if (first_round && threadIdx.x < 32) emit_lookback_publish();
            first_round = false;
            __syncthreads();
            const uint32_t nspans = s_nspans;
            // exclusive prefix of the span lengths (8 spans per thread of the first 256)
            uint32_t loc[kSpanCap / kEmitThreads];
            uint32_t my = 0;
#pragma unroll
            for (int q = 0; q < kSpanCap / kEmitThreads; ++q) {
                const uint32_t jj = threadIdx.x * (kSpanCap / kEmitThreads) + q;
                loc[q] = (!lb_warp && jj < nspans) ? (s_span[jj] >> 16) & 0x7FFFu : 0u;
                my += loc[q];
            }
            uint32_t round_pairs;
            uint32_t run = emit_scan(my, s_warp, round_pairs);
            if (!lb_warp) {
#pragma unroll
                for (int q = 0; q < kSpanCap / kEmitThreads; ++q) {
                    const uint32_t jj = threadIdx.x * (kSpanCap / kEmitThreads) + q;
                    if (jj < nspans) s_pfx[jj] = run;
                    run += loc[q];
                }
            }
            __syncthreads();
            // flatten (all kEmitBlock threads): pair p of the round -> last span j with s_pfx[j] <= p
            const uint32_t out0 = s_base + round_base;
            for (uint32_t p = threadIdx.x; p < round_pairs; p += kEmitBlock) {
                uint32_t lo = 0, hi = nspans - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (s_pfx[mid] <= p) lo = mid;
                    else hi = mid - 1;
                }
                const uint32_t sp = s_span[lo];
                const uint32_t step = (sp & 0x80000000u) ? (uint32_t)tiles_x : 1u;
                const uint32_t tile = (sp & 0xFFFFu) + (p - s_pfx[lo]) * step;
                const uint32_t o = out0 + p;
                if (o < cap) {
                    pair_tile[o] = (uint16_t)tile;
                    pair_value[o] = s_gid[lo];
                }
                atomicAdd(hist + tile, 1u);
            }
            round_base += round_pairs;
        }
        if (first_round && threadIdx.x < 32) emit_lookback_publish();  // CTA without spans
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
        at<float4>(ws, P.rec), at<uint4>(ws, P.erec), at<uint32_t>(ws, P.depth_key),                         \
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
    if (smem > 20 * 1024)  // static (~25 KB) + dynamic above the default 48 KB window
        cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)L.nblk_emit < sms * 4 ? (int)L.nblk_emit : sms * 4;
    k_emit<<<grid, kEmitBlock, smem, st>>>(
        mode, at<const float4>(ws, P.rec), at<const uint4>(ws, P.erec), at<const uint32_t>(ws, P.order),
        at<const uint32_t>(ws, P.n_visible), L.capacity,
        at<uint16_t>(ws, P.pair_tile), at<uint32_t>(ws, P.pair_value), at<uint32_t>(ws, P.tile_count),
        at<uint32_t>(ws, L.lb_emit), at<uint32_t>(ws, L.counters) + 8, at<uint32_t>(ws, P.total_pairs),
        at<uint32_t>(ws, P.overflow), cam.tiles_x, cam.tiles_y, P.n_tiles, smem_hist);
    return cudaGetLastError();
}

}  // namespace ss
