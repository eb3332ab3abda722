// ss_tilegeom.cuh -- the float64 tile geometry of libss: SnugBox, AccuTile (Algorithm 1), the
// 3-sigma rect, and the super-tile entries of a Gaussian's tile set.  Included by the
// translation units that must evaluate it identically (ss_geometry.cu: the count of a1;
// ss_bin.cu: the re-enumeration of a2-a4); both are compiled with --fmad=false.
//
// P:n = /root/reference/PAPER.md line n.
#pragma once
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
    double ia, ic;   // 1 / a, 1 / c
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
    s.ia = ia;
    s.ic = ic;
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
// ia = 1 / a_free (one reciprocal per Gaussian, R1).
__device__ __forceinline__ void intersect_line(double m_free, double m_line, double a_free, double ia, double b,
                                               double c_line, double t, double line, double &lo, double &hi) {
    double v = line - m_line;
    double disc = (b * b - a_free * c_line) * v * v + t * a_free;
    if (disc < 0.0) disc = 0.0;  // R12
    double s = sqrt(disc);
    lo = m_free + (-b * v - s) * ia;
    hi = m_free + (-b * v + s) * ia;
}

// AccuTile, Algorithm 1 along the shorter side of the SnugBox tile rect (R9),
// the columns path by the a<->c / x<->y swap.  R10: a boundary line outside the
// bbox yields the neutral pair (+inf, -inf).
struct Sweep {
    bool rows;                                        // rows path (else columns)
    double mf, ms, af, cs, b, t;                      // free/swept-axis centre and coefficients
    double iaf;                                       // 1 / af
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
        w.mf = mx; w.ms = my; w.af = a; w.cs = c; w.iaf = S.ia;
        w.ext_lo = S.xmin; w.ext_hi = S.xmax; w.smin = S.ymin; w.smax = S.ymax;
        w.tmin_s = S.yl; w.tmax_s = S.yr;
        w.s0 = R.z; w.s1 = R.w; w.f0 = R.x; w.f1 = R.y;
    } else {
        w.mf = my; w.ms = mx; w.af = c; w.cs = a; w.iaf = S.ic;
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
    if (compute) intersect_line(w.mf, w.ms, w.af, w.iaf, w.b, w.cs, w.t, line, lo, hi);
}

// One row (or column) r of Algorithm 1 given i_min (its lower boundary line) and i_max (its
// upper boundary line): e_min / e_max, Convert, clip to the rect.  Returns [tmin, tmax).
__device__ __forceinline__ void sweep_row(const Sweep &w, int r, double imin_lo, double imin_hi, double imax_lo,
                                          double imax_hi, int &tmin, int &tmax) {
    const double lo_r = (double)(r * kTile), hi_r = (double)((r + 1) * kTile);
#ifdef SS_FAULT_SKIP_TANGENT_ROW  // fault-injection build: the tangent-point row test dropped
    const double e_min = imin_lo < imax_lo ? imin_lo : imax_lo;
    const double e_max = imin_hi > imax_hi ? imin_hi : imax_hi;
#else
    const double e_min = (w.tmin_s >= lo_r && w.tmin_s < hi_r) ? w.ext_lo : (imin_lo < imax_lo ? imin_lo : imax_lo);
    const double e_max = (w.tmax_s >= lo_r && w.tmax_s < hi_r) ? w.ext_hi : (imin_hi > imax_hi ? imin_hi : imax_hi);
#endif
    double g0 = floor(e_min / kTile), g1 = floor(e_max / kTile) + 1.0;
    if (!(g0 > w.f0)) g0 = w.f0;
    if (g0 > w.f1) g0 = w.f1;
    if (!(g1 > w.f0)) g1 = w.f0;
    if (g1 > w.f1) g1 = w.f1;
    tmin = (int)g0;
    tmax = (int)g1;
}

// Algorithm 1 in count mode on a prepared sweep (the sequential loop, i_min <- i_max);
// on_line(r, tmin, tmax) sees every line of the sweep in order.
template <class OnLine>
__device__ __forceinline__ uint32_t accutile_count(const Sweep &w, int tiles_x, OnLine &&on_line) {
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
        on_line(r, tmin, tmax);
        imin_lo = imax_lo;
        imin_hi = imax_hi;
    }
    return C;
}

// ---------------------------------------------------------------- super-tile entries
// The binning (ss_bin.cu) groups a Gaussian's tiles by the kSuper x kSuper-tile super-tile
// that contains them: one ENTRY = (super-tile id, 16-bit mask of its tiles, bit
// (y & 3) * 4 + (x & 3) for tile (x, y)).  Lines of the tile set (tile rows, or tile columns
// for Algorithm 1's columns sweep) are fed in increasing order with their span [a, b) along
// the other axis; each band of 4 lines is flushed as entries in increasing order along the
// span axis: one entry for every super-tile between the band's extremes along the span
// axis (so the count needs only the extremes; for a convex tile set every such mask is
// non-empty, and an empty one would add no pair).
constexpr int kSuper = kSuperTile;

struct EntryAcc {
    int band;                  // current band (line / 4), -1 = none
    uint32_t iv0, iv1, iv2, iv3;  // per line of the band: a | b << 16 (empty if b <= a)
    bool cols;                 // lines are tile columns (spans run along y)
    int stx;                   // super-tiles along x
};

__device__ __forceinline__ void acc_init(EntryAcc &A, bool cols, int stx) {
    A.band = -1;
    A.iv0 = A.iv1 = A.iv2 = A.iv3 = 0u;
    A.cols = cols;
    A.stx = stx;
}

// 4-bit column pattern -> bits 0, 4, 8, 12
__device__ __forceinline__ uint32_t spread4(uint32_t c) {
    return (c & 1u) | ((c & 2u) << 3) | ((c & 4u) << 6) | ((c & 8u) << 9);
}

__device__ __forceinline__ uint32_t line_bits(uint32_t iv, int C, int q, bool cols) {
    const int a = max((int)(iv & 0xFFFFu), 4 * C), b = min((int)(iv >> 16), 4 * C + 4);
    if (b <= a) return 0u;
    const uint32_t bits = ((1u << (b - a)) - 1u) << (a - 4 * C);
    return cols ? (spread4(bits) << q) : (bits << (4 * q));
}

// Transpose of a 4x4 bit matrix stored as 4 nibbles (bit r*4 + c -> bit c*4 + r).
__device__ __forceinline__ uint32_t transpose4x4(uint32_t w) {
    uint32_t t = (w ^ (w >> 3)) & 0x0A0Au;
    w ^= t ^ (t << 3);
    t = (w ^ (w >> 6)) & 0x00CCu;
    w ^= t ^ (t << 6);
    return w;
}

// Entries of one band given its 4 line spans: emit(super-tile, mask) for every super-tile
// between the band's extremes along the span axis, in increasing order.  Bands no wider than
// 32 tiles (from their first super-tile boundary) use 32-bit line bitmaps; wider ones the
// per-line interval form.  Both give the same masks.
template <class F>
__device__ __forceinline__ void band_entries(int band, uint32_t iv0, uint32_t iv1, uint32_t iv2, uint32_t iv3,
                                             bool cols, int stx, F &&emit) {
    int lo = 1 << 20, hi = 0;
    const uint32_t ivs[4] = {iv0, iv1, iv2, iv3};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int a = (int)(ivs[q] & 0xFFFFu), b = (int)(ivs[q] >> 16);
        if (b > a) {
            lo = min(lo, a);
            hi = max(hi, b);
        }
    }
    if (lo >= hi) return;
    const int ox = lo & ~3;
    if (hi - ox <= 32) {
        uint32_t m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int a = (int)(ivs[q] & 0xFFFFu), b = (int)(ivs[q] >> 16);
            m[q] = b > a ? (((b - a) >= 32 ? 0xFFFFFFFFu : ((1u << (b - a)) - 1u)) << (a - ox)) : 0u;
        }
        for (int C = lo >> 2; C <= (hi - 1) >> 2; ++C) {
            const int sh = 4 * C - ox;
            const uint32_t w = ((m[0] >> sh) & 0xFu) | (((m[1] >> sh) & 0xFu) << 4) | (((m[2] >> sh) & 0xFu) << 8) |
                               (((m[3] >> sh) & 0xFu) << 12);
            emit(cols ? (uint32_t)(C * stx + band) : (uint32_t)(band * stx + C), cols ? transpose4x4(w) : w);
        }
        return;
    }
    for (int C = lo >> 2; C <= (hi - 1) >> 2; ++C) {
        const uint32_t mask = line_bits(iv0, C, 0, cols) | line_bits(iv1, C, 1, cols) | line_bits(iv2, C, 2, cols) |
                              line_bits(iv3, C, 3, cols);
        emit(cols ? (uint32_t)(C * stx + band) : (uint32_t)(band * stx + C), mask);
    }
}

template <class F>
__device__ __forceinline__ void acc_flush(EntryAcc &A, F &&emit) {
    if (A.band < 0) return;
    band_entries(A.band, A.iv0, A.iv1, A.iv2, A.iv3, A.cols, A.stx, emit);
    A.band = -1;
    A.iv0 = A.iv1 = A.iv2 = A.iv3 = 0u;
}

template <class F>
__device__ __forceinline__ void acc_feed(EntryAcc &A, int line, int a, int b, F &&emit) {
    if (b <= a) return;
    if ((line >> 2) != A.band) {
        acc_flush(A, emit);
        A.band = line >> 2;
    }
    const uint32_t v = (uint32_t)a | ((uint32_t)b << 16);
    switch (line & 3) {
        case 0: A.iv0 = v; break;
        case 1: A.iv1 = v; break;
        case 2: A.iv2 = v; break;
        default: A.iv3 = v; break;
    }
}

// Entry count of a tile set fed line by line (increasing): per band of 4 lines, the number
// of super-tiles between the band's extremes.
struct EntryCount {
    int band, lo, hi;
    uint32_t n;
};
__device__ __forceinline__ void cnt_init(EntryCount &E) {
    E.band = -1;
    E.lo = 1 << 20;
    E.hi = 0;
    E.n = 0;
}
__device__ __forceinline__ void cnt_flush(EntryCount &E) {
    if (E.band >= 0 && E.lo < E.hi) E.n += (uint32_t)(((E.hi - 1) >> 2) - (E.lo >> 2) + 1);
    E.band = -1;
    E.lo = 1 << 20;
    E.hi = 0;
}
__device__ __forceinline__ void cnt_feed(EntryCount &E, int line, int a, int b) {
    if (b <= a) return;
    if ((line >> 2) != E.band) {
        cnt_flush(E);
        E.band = line >> 2;
    }
    E.lo = min(E.lo, a);
    E.hi = max(E.hi, b);
}

// The 4 line spans of band `band` of a prepared AccuTile sweep, evaluated exactly as the
// sequential loop of accutile_count evaluates them (the first line of the sweep with the
// `>= smin` test, every later line with the `<= smax` test), so that a band can be produced
// by itself.  Empty lines: 0.
__device__ __forceinline__ void sweep_band(const Sweep &w, int band, uint32_t &iv0, uint32_t &iv1, uint32_t &iv2,
                                           uint32_t &iv3) {
    iv0 = iv1 = iv2 = iv3 = 0u;
    const int r0 = max(4 * band, w.s0), r1 = min(4 * band + 4, w.s1);
    double imin_lo, imin_hi;
    const double line_min = (double)(r0 * kTile);
    sweep_line(w, line_min, r0 == w.s0 ? line_min >= w.smin : line_min <= w.smax, imin_lo, imin_hi);
    for (int r = r0; r < r1; ++r) {
        double imax_lo, imax_hi;
        const double line_max = (double)((r + 1) * kTile);
        sweep_line(w, line_max, line_max <= w.smax, imax_lo, imax_hi);
        int tmin, tmax;
        sweep_row(w, r, imin_lo, imin_hi, imax_lo, imax_hi, tmin, tmax);
        const uint32_t v = tmax > tmin ? ((uint32_t)tmin | ((uint32_t)tmax << 16)) : 0u;
        switch (r & 3) {
            case 0: iv0 = v; break;
            case 1: iv1 = v; break;
            case 2: iv2 = v; break;
            default: iv3 = v; break;
        }
        imin_lo = imax_lo;
        imin_hi = imax_hi;
    }
}

}  // namespace
}  // namespace ss
