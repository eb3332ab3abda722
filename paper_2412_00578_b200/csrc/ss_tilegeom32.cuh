// ss_tilegeom32.cuh -- the SnugBox / AccuTile tile decisions in float32 with a certified error
// bound, for ss_preprocess's fast path (ss_geometry.cu, compiled with --fmad=false).
//
// The reference evaluation of the tile geometry is float64 on the stored float32 record
// (ss_tilegeom.cuh, R1).  Every tile set it produces is decided by integers
// floor(e / 16) of float64 values e -- the SnugBox extremes, the tangent points (R11), the
// Algorithm-1 line intersections (Eq. 15) -- combined by integer min / max / clipping:
//   * a line 16 j lies inside the bbox iff j > floor(smin / 16) (resp. j <= floor(smax / 16)),
//     provided smin, smax are not exactly on a tile line;
//   * a tangent point lies in row r iff floor(tangent / 16) == r;
//   * floor(min(lo, lo') / 16) = min(floor(lo / 16), floor(lo' / 16)) (floor is monotone).
// Here every such value is evaluated in float32 together with an absolute bound on its
// distance from the float64 value (a first-order rounding analysis of the float32 chain with
// u = 2^-24 per correctly rounded operation and 4u per approximate MUFU operation, every bound
// widened by a safety factor).  floor(e / 16) is CERTAIN when the whole interval [e - err,
// e + err] lies strictly inside one 16-pixel cell -- then it equals the float64 floor and e is
// not on a tile line.  A Gaussian with any uncertain floor (a value within its bound of a tile
// line, an ill-conditioned conic) is handed to the float64 path, so the tile sets are the
// float64 evaluation's by construction.  The decisions are the paper's (Eqs. 14-16, Algorithm
// 1); only the precision in which they are certified differs.
#pragma once
#include "ss_common.cuh"

namespace ss {
namespace {

constexpr float kU = 5.9604645e-8f;  // 2^-24: relative error of one correctly rounded operation
constexpr float kUa = 4.0f * kU;     // budget of one approximate MUFU operation (rcp / sqrt / rsqrt)
constexpr int kBig = 1 << 20;        // clamp of floor values: far outside any grid (<= 256 tiles)

__device__ __forceinline__ float rcp_a(float x) {
    float r;
    asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_a(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_a(float x) {
    float r;
    asm("rsqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// floor(v / 16) certified for every value within e of v (the float64 value among them):
// returns false if [v - e, v + e] touches a tile line.  k is clamped to [-kBig, kBig].
// d = v - 16 f is exact (v / 16 is exact, f = floor(v / 16), and d in [0, 16) is a multiple of
// ulp(v) when ulp(v) <= 16; for |v| >= 2^28, d = 0 and the test fails), so the interval lies
// strictly inside (16 f, 16 f + 16) iff e < d < 16 - e; 16 - e is rounded down.
__device__ __forceinline__ bool floor16(float v, float e, int &k) {
    const float f = floorf(__fmul_rn(v, 0.0625f));
    const float d = __fmaf_rn(f, -16.0f, v);
    k = (int)fminf(fmaxf(f, -(float)kBig), (float)kBig);
    return d > e && d < __fsub_rd(16.0f, e);
}

enum { kSure = 0, kCull = 1, kUnsure = 2 };

// SnugBox (Eqs. 15-16) in float32: certified floors of the bbox extremes and tangent points.
struct Snug32 {
    float ia, ic, D, relD, t;
    int kx0, kx1, ky0, ky1;  // floor(xmin / 16), floor(xmax / 16), floor(ymin / 16), floor(ymax / 16)
    int kyl, kyr, kxt, kxb;  // floors of the tangent points B_l, B_r (y) and B_t, B_b (x) (R11)
};

// The float64 path's D > 0 test and the SnugBox floors.  kCull: D <= 0 for certain (no tiles);
// kUnsure: a decision cannot be certified.
template <bool TANGENTS>  // AccuTile also needs the tangent points
__device__ __forceinline__ int snug32(float mx, float my, float a, float b, float c, double td, Snug32 &s) {
    const float t = (float)td;  // |t - td| <= u |td|
    const float ac = __fmul_rn(a, c), bb = __fmul_rn(b, b);
    const float D = __fsub_rn(ac, bb);
    const float eD = 1.5f * kU * (fabsf(ac) + bb + fabsf(D));
    if (D <= -eD) return kCull;
    if (!(D > 8.0f * eD)) return kUnsure;  // the sign of D, or its relative accuracy, is not certain
    const float rD = rcp_a(D);                                       // rel relD + 4u
    // relD = eD / D bounded from above: rD has relative error <= 4u, the product u
    const float relD = __fmul_rn(__fmul_rn(eD, rD), 1.0001f);
    const float hx = sqrt_a(__fmul_rn(__fmul_rn(t, c), rD));         // rel relD / 2 + 7.5u
    const float hy = sqrt_a(__fmul_rn(__fmul_rn(t, a), rD));
    const float rel_h = (0.5f * relD + 8.0f * kU) * 1.25f;
    s.ia = rcp_a(a);
    s.ic = rcp_a(c);
    s.D = D;
    s.relD = relD;
    s.t = t;
    // one bound per pair m +- h of values: the value's own rounding u |m +- h| <= u (|m| + |h|)
    // (error-bound arithmetic only: fused, the 1.1 safety factor covers its rounding)
    auto pair_bound = [](float m, float h, float eh) {
        return __fmaf_rn(__fmaf_rn(kU, fabsf(m) + fabsf(h), eh), 1.1f, 1e-30f);
    };
    const float ex = pair_bound(mx, hx, hx * rel_h), ey = pair_bound(my, hy, hy * rel_h);
    bool ok = floor16(__fsub_rn(mx, hx), ex, s.kx0);
    ok &= floor16(__fadd_rn(mx, hx), ex, s.kx1);
    ok &= floor16(__fsub_rn(my, hy), ey, s.ky0);
    ok &= floor16(__fadd_rn(my, hy), ey, s.ky1);
    if (!TANGENTS) return ok ? kSure : kUnsure;
    // tangent points: yl/yr = my +- (b hx) / c, xt/xb = mx +- (b hy) / a; (b h) ic has relative
    // error rel_h + 6u
    const float Tx = __fmul_rn(__fmul_rn(b, hx), s.ic), Ty = __fmul_rn(__fmul_rn(b, hy), s.ia);
    const float relT = (rel_h + 6.0f * kU) * 1.1f;
    const float eTx = pair_bound(my, Tx, fabsf(Tx) * relT), eTy = pair_bound(mx, Ty, fabsf(Ty) * relT);
    ok &= floor16(__fadd_rn(my, Tx), eTx, s.kyl);
    ok &= floor16(__fsub_rn(my, Tx), eTx, s.kyr);
    ok &= floor16(__fadd_rn(mx, Ty), eTy, s.kxt);
    ok &= floor16(__fsub_rn(mx, Ty), eTy, s.kxb);
    return ok ? kSure : kUnsure;
}

// R8: the SnugBox tile rect [floor(lo / 16), floor(hi / 16) + 1) clipped to the grid.
__device__ __forceinline__ int clip_tiles(int k, int tiles) { return k < 0 ? 0 : (k > tiles ? tiles : k); }
__device__ __forceinline__ int4 rect32(const Snug32 &s, int tiles_x, int tiles_y) {
    return make_int4(clip_tiles(s.kx0, tiles_x), clip_tiles(s.kx1 + 1, tiles_x), clip_tiles(s.ky0, tiles_y),
                     clip_tiles(s.ky1 + 1, tiles_y));
}

// Algorithm 1 along the shorter side (R9): the swept lines j in [s0, s1], rows [s0, s1).
struct Sweep32 {
    bool rows;
    float mf, ms, af, b, iaf, D, relD, taf;
    float cD4, ct4, umf;  // per-sweep constants of line32's error bounds
    int s0, s1, f0, f1;
    int k_ext_lo, k_ext_hi;  // floors of the free-axis bbox extremes
    int k_smin, k_smax;      // floors of the swept-axis bbox extremes
    int k_tmin, k_tmax;      // floors of the tangent points (the rows holding them)
};

__device__ __forceinline__ void sweep32_setup(const Snug32 &S, const int4 &R, float mx, float my, float a, float b,
                                              float c, Sweep32 &w) {
    w.rows = (R.w - R.z) <= (R.y - R.x);
    w.b = b;
    w.D = S.D;
    w.relD = S.relD;
    if (w.rows) {
        w.mf = mx; w.ms = my; w.af = a; w.iaf = S.ia;
        w.k_ext_lo = S.kx0; w.k_ext_hi = S.kx1; w.k_smin = S.ky0; w.k_smax = S.ky1;
        w.k_tmin = S.kyl; w.k_tmax = S.kyr;
        w.s0 = R.z; w.s1 = R.w; w.f0 = R.x; w.f1 = R.y;
    } else {
        w.mf = my; w.ms = mx; w.af = c; w.iaf = S.ic;
        w.k_ext_lo = S.ky0; w.k_ext_hi = S.ky1; w.k_smin = S.kx0; w.k_smax = S.kx1;
        w.k_tmin = S.kxt; w.k_tmax = S.kxb;
        w.s0 = R.x; w.s1 = R.y; w.f0 = R.z; w.f1 = R.w;
    }
    w.taf = __fmul_rn(S.t, w.af);
    w.cD4 = (w.relD + 4.0f * kU) * 4.8f;
    w.ct4 = (fabsf(w.taf) * (2.4f * kU) + 1e-30f) * 4.0f;
    w.umf = kU * fabsf(w.mf);
}

// Line j of the sweep: certified floors (klo, khi) of its Eq. 15 intersections, or the neutral
// pair (+kBig, -kBig; R10) when the algorithm does not compute them: the first line of a sweep
// only if it lies at or past smin, every later line only if it lies at or before smax (smin /
// smax are never on a line once their floors are certified).  The float64 path evaluates
// disc = (b^2 - a_f c_s) v^2 + t a_f = t a_f - D v^2 (a_f c_s = a c).
__device__ __forceinline__ bool line32(const Sweep32 &w, int j, bool first, int &klo, int &khi) {
    klo = kBig;
    khi = -kBig;
    const bool compute = first ? (j > w.k_smin) : (j <= w.k_smax);
    if (!compute) return true;
    const float v = __fsub_rn((float)(j * kTile), w.ms);          // rel u
    const float Dvv = __fmul_rn(w.D, __fmul_rn(v, v));            // rel relD + 4u
    const float disc = __fsub_rn(w.taf, Dvv);                     // taf: rel 2u
    // 4 x the bound on |disc - disc_64|: (|Dvv| (relD + 4u) + |taf| 2u + u |disc|) 1.2 + 1e-30
    // (bound arithmetic fused; the per-sweep constants are w.cD4 = 4.8 (relD + 4u) and
    // w.ct4 = 4 (2.4u |taf| + 1e-30))
    const float edisc4 = __fmaf_rn(fabsf(Dvv), w.cD4, __fmaf_rn(fabsf(disc), 4.8f * kU, w.ct4));
    // a line within 4 bounds of tangency (disc near 0: the line grazes the bbox extreme) is left
    // to the float64 path; otherwise, with y the float64 disc, |y - disc| <= e <= disc / 4 and
    // |sqrt(disc) - sqrt(y)| = |disc - y| / (sqrt(disc) + sqrt(y)) <= e / (1.866 sqrt(disc))
    //                       <= 0.536 e rsqrt(disc)
    // s = disc rsqrt(disc) is within 6u of sqrt(disc) (rsqrt: 4u, the product: u)
    if (!(disc >= edisc4)) return false;
    const float r = rsqrt_a(disc);
    const float s = __fmul_rn(disc, r);
    const float es = __fmaf_rn(__fmul_rn(edisc4, 0.25f * 0.536f * 1.1f), r, s * (6.6f * kU));
    const float bv = __fmul_rn(w.b, v);
    const float nlo = __fsub_rn(-bv, s), nhi = __fadd_rn(-bv, s);
    const float tlo = __fmul_rn(nlo, w.iaf), thi = __fmul_rn(nhi, w.iaf);  // iaf: rel 4u
    const float lo = __fadd_rn(w.mf, tlo), hi = __fadd_rn(w.mf, thi);
    // one bound for both intersections, with |nlo|, |nhi| <= nmag = |bv| + s, |tlo|, |thi| <=
    // aia nmag (1 + u), |lo|, |hi| <= |mf| + aia nmag (1 + u):
    //   (aia (ebv + es + u nmag) + 5.5u aia nmag + u (|mf| + aia nmag)) 1.2 + 1e-30,
    // ebv = 2.1u |bv|; the (1 + u) factors are inside the 1.2 safety factor
    const float aia = fabsf(w.iaf);
    const float nmag = fabsf(bv) + s;
    const float tmag = aia * nmag;
    const float A = __fmaf_rn(kU, nmag, __fmaf_rn(fabsf(bv), 2.1f * kU, es));
    const float B = __fmaf_rn(tmag, 6.5f * kU, w.umf);  // w.umf = u |mf|
    const float e = __fmaf_rn(__fmaf_rn(aia, A, B), 1.2f, 1e-30f);
    return floor16(lo, e, klo) & floor16(hi, e, khi);
}

// Row r from its boundary lines' floors: [tmin, tmax) of Algorithm 1 (sweep_row).
__device__ __forceinline__ void row32(const Sweep32 &w, int r, int klo0, int khi0, int klo1, int khi1, int &tmin,
                                      int &tmax) {
#ifdef SS_FAULT_SKIP_TANGENT_ROW  // fault-injection build: the tangent-point row test dropped
    const int g0 = min(klo0, klo1);
    const int g1 = max(khi0, khi1) + 1;
#else
    const int g0 = w.k_tmin == r ? w.k_ext_lo : min(klo0, klo1);
    const int g1 = (w.k_tmax == r ? w.k_ext_hi : max(khi0, khi1)) + 1;
#endif
    tmin = g0 <= w.f0 ? w.f0 : (g0 > w.f1 ? w.f1 : g0);
    tmax = g1 <= w.f0 ? w.f0 : (g1 > w.f1 ? w.f1 : g1);
}

// Algorithm 1, count mode; on_line(r, tmin, tmax) sees every row in order.  False at the
// first uncertain decision.
template <class OnLine>
__device__ __forceinline__ bool accutile_count32(const Sweep32 &w, uint32_t &C, OnLine &&on_line) {
    C = 0;
    int klo0, khi0;
    bool ok = line32(w, w.s0, true, klo0, khi0);
    for (int r = w.s0; r < w.s1 && ok; ++r) {
        int klo1, khi1;
        ok = line32(w, r + 1, false, klo1, khi1);
        int tmin, tmax;
        row32(w, r, klo0, khi0, klo1, khi1, tmin, tmax);
        if (tmax > tmin) C += (uint32_t)(tmax - tmin);
        on_line(r, tmin, tmax);
        klo0 = klo1;
        khi0 = khi1;
    }
    return ok;
}

// The 4 rows of band `band` (sweep_band): spans as (tmin | tmax << 16), 0 when empty.
__device__ __forceinline__ bool band32(const Sweep32 &w, int band, uint32_t &iv0, uint32_t &iv1, uint32_t &iv2,
                                       uint32_t &iv3) {
    iv0 = iv1 = iv2 = iv3 = 0u;
    const int r0 = max(4 * band, w.s0), r1 = min(4 * band + 4, w.s1);
    int klo0, khi0;
    bool ok = line32(w, r0, r0 == w.s0, klo0, khi0);
    for (int r = r0; r < r1; ++r) {
        int klo1, khi1;
        ok &= line32(w, r + 1, false, klo1, khi1);
        int tmin, tmax;
        row32(w, r, klo0, khi0, klo1, khi1, tmin, tmax);
        const uint32_t v = tmax > tmin ? ((uint32_t)tmin | ((uint32_t)tmax << 16)) : 0u;
        switch (r & 3) {
            case 0: iv0 = v; break;
            case 1: iv1 = v; break;
            case 2: iv2 = v; break;
            default: iv3 = v; break;
        }
        klo0 = klo1;
        khi0 = khi1;
    }
    return ok;
}

}  // namespace
}  // namespace ss
