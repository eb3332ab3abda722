/*
 * ss_oracle.c -- plain, slow CPU ORACLE for the Speedy-Splat forward hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2412_00578_b200/, libss.so) never links, imports or executes it, and this
 * file shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named);
 * "R<k>" = the reading of an ambiguity listed in DESIGN.md §3.
 *
 * Precision (DESIGN.md §3 "arithmetic contract"):
 *   - projection, conic, colour: float32, every operation rounded, no contraction
 *     (compiled with -ffp-contract=off; explicit fmaf() only where the contract says);
 *   - tile geometry (SnugBox, AccuTile, 3-sigma rect): float64 on the stored float32
 *     record -- the kernel's precision for these integer decisions;
 *   - render: float32 (alpha skip decision q <= t on a pinned fmaf chain; expf);
 *   - score: per-pixel derivative by its definition in float64, accumulated in float64.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py against closed
 * forms, paper examples, brute force and invariants.  No function
 * is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16 /* "divides the rendered image into 16 x 16 pixel tiles" */

enum { OR_3SIGMA = 0, OR_SNUGBOX = 1, OR_ACCUTILE = 2 };

typedef struct {
    float viewmat[12]; /* world->camera 3x4 row-major: rows (right, down, forward | t) */
    float fx, fy, cx, cy;
    float campos[3];
    int32_t width, height;
    float z_near; /* R4: keep iff z >= z_near */
    float clip;   /* R5: J clamp factor (0 = off) */
} or_camera;

/* Record layout written by or_project (12 floats per Gaussian). */
enum { R_X = 0, R_Y, R_DEPTH, R_A, R_B, R_C, R_SIGMA, R_T, R_R, R_G, R_BL, R_VIS, R_NF };

/* ------------------------------------------------------------------------------------
 * Spherical harmonics (R13): view-dependent colour c_i "derived from W and h_i",
 * h_i in R^{16x3}.  Real SH basis, degree <= 3, evaluated at dir (unit).
 * Basis values are float32 products evaluated left to right.
 * ---------------------------------------------------------------------------------- */
static const float SH_C0 = 0.28209479177387814f;
static const float SH_C1 = 0.4886025119029199f;
static const float SH_C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                               -1.0925484305920792f, 0.5462742152960396f};
static const float SH_C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                               0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                               -0.5900435899266435f};

void or_sh_basis(int deg, float x, float y, float z, float *Y /* [16] */)
{
    for (int k = 0; k < 16; ++k) Y[k] = 0.0f;
    Y[0] = SH_C0;
    if (deg < 1) return;
    Y[1] = -SH_C1 * y;
    Y[2] = SH_C1 * z;
    Y[3] = -SH_C1 * x;
    if (deg < 2) return;
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = SH_C2[0] * xy;
    Y[5] = SH_C2[1] * yz;
    Y[6] = SH_C2[2] * (2.0f * zz - xx - yy);
    Y[7] = SH_C2[3] * xz;
    Y[8] = SH_C2[4] * (xx - yy);
    if (deg < 3) return;
    Y[9] = SH_C3[0] * y * (3.0f * xx - yy);
    Y[10] = SH_C3[1] * xy * z;
    Y[11] = SH_C3[2] * y * (4.0f * zz - xx - yy);
    Y[12] = SH_C3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = SH_C3[4] * x * (4.0f * zz - xx - yy);
    Y[14] = SH_C3[5] * z * (xx - yy);
    Y[15] = SH_C3[6] * x * (xx - 3.0f * yy);
}

/* ------------------------------------------------------------------------------------
 * Threshold (Eqs. 9, 11): t = 2 log(255 sigma).  R2: evaluated in float64.
 * ---------------------------------------------------------------------------------- */
double or_threshold(float sigma) { return 2.0 * log(255.0 * (double)sigma); }

/* ------------------------------------------------------------------------------------
 * SnugBox (Sec. 4.1.1, Eqs. 15-16): the exact axis-aligned bounding box of the
 * ellipse t = a xd^2 + 2 b xd yd + c yd^2 (Eq. 14).  Eq. 16 gives the arg of the y-extreme;
 * substituting into Eq. 15 gives yd_ext^2 = t a / (a c - b^2); by the a<->c swap
 * xd_ext^2 = t c / (a c - b^2).  Float64.  Also returns the four tangent points (R11):
 *   B_l = (x_min, my + b hx / c)   B_r = (x_max, my - b hx / c)
 *   B_t = (mx + b hy / a, y_min)   B_b = (mx - b hy / a, y_max)   (image y points down, R21)
 * ---------------------------------------------------------------------------------- */
void or_snugbox(double mx, double my, double a, double b, double c, double t,
                double *bbox /* xmin,xmax,ymin,ymax */, double *tangent /* 8: Bl, Br, Bt, Bb */)
{
    /* contract (R1): one reciprocal each of D, a and c; quotients are products with them */
    double D = a * c - b * b;
    double rD = 1.0 / D;
    double hx = sqrt(t * c * rD);
    double hy = sqrt(t * a * rD);
    bbox[0] = mx - hx;
    bbox[1] = mx + hx;
    bbox[2] = my - hy;
    bbox[3] = my + hy;
    if (tangent) {
        double ia = 1.0 / a, ic = 1.0 / c;
        tangent[0] = mx - hx; tangent[1] = my + b * hx * ic;
        tangent[2] = mx + hx; tangent[3] = my - b * hx * ic;
        tangent[4] = mx + b * hy * ia; tangent[5] = my - hy;
        tangent[6] = mx - b * hy * ia; tangent[7] = my + hy;
    }
}

static double dmin(double u, double v) { return u < v ? u : v; }
static double dmax(double u, double v) { return u > v ? u : v; }

/* "converts these edges to tile indices by dividing by tile size, rounding, and clipping
 * to the image boundary".  R8: half-open span [floor(lo/16), floor(hi/16)+1),
 * clipped to [0, tiles]. */
static void edge_span(double lo, double hi, int tiles, int *s0, int *s1)
{
    double f0 = floor(lo / TILE), f1 = floor(hi / TILE) + 1.0;
    /* clip in double first so huge / non-finite edges never overflow an int */
    if (!(f0 > 0.0)) f0 = 0.0;
    if (!(f1 > 0.0)) f1 = 0.0;
    if (f0 > tiles) f0 = tiles;
    if (f1 > tiles) f1 = tiles;
    *s0 = (int)f0;
    *s1 = (int)f1;
}

/* Tile rect of the SnugBox bbox. */
void or_rect_snugbox(double mx, double my, double a, double b, double c, double t, int tiles_x,
                     int tiles_y, int32_t *rect /* x0,x1,y0,y1 */)
{
    double bb[4];
    or_snugbox(mx, my, a, b, c, t, bb, 0);
    int x0, x1, y0, y1;
    edge_span(bb[0], bb[1], tiles_x, &x0, &x1);
    edge_span(bb[2], bb[3], tiles_y, &y0, &y1);
    rect[0] = x0; rect[1] = x1; rect[2] = y0; rect[3] = y1;
}

/* 3D-GS baseline (Eq. 8): r = ceil(3 sqrt(lambda_max(Sigma_2D))); the tiles that
 * intersect the square mu +- r (R6, R7).  Float64 on the float32 covariance entries. */
void or_rect_3sigma(double mx, double my, double cxx, double cxy, double cyy, int tiles_x,
                    int tiles_y, int32_t *rect)
{
    double m = 0.5 * (cxx + cyy);
    double det = cxx * cyy - cxy * cxy;
    double disc = m * m - det;
    if (disc < 0.0) disc = 0.0;
    double lmax = m + sqrt(disc);
    double r = ceil(3.0 * sqrt(lmax));
    int x0, x1, y0, y1;
    edge_span(mx - r, mx + r, tiles_x, &x0, &x1);
    edge_span(my - r, my + r, tiles_y, &y0, &y1);
    rect[0] = x0; rect[1] = x1; rect[2] = y0; rect[3] = y1;
}

/* ------------------------------------------------------------------------------------
 * AccuTile, Algorithm 1, step by step, along the shorter side of the SnugBox
 * tile rect (R9: rows iff (y1-y0) <= (x1-x0)).  The column path is the a<->c, x<->y swap
 * (App. A).  Float64.
 *
 *   line_min <- R_b ; if line_min >= B_b: i_min <- Intersections(line_min, E)   (Eq. 15)
 *   for row r in R:
 *       line_max <- r_t ; if line_max <= B_t: i_max <- Intersections(line_max, E)
 *       e_min <- B_l if B_l in r else min(i_min, i_max)
 *       e_max <- B_r if B_r in r else max(i_min, i_max)
 *       tile_min, tile_max <- Convert(e_min, e_max) ; C += tile_max - tile_min
 *       Process(tile_min, tile_max) ; i_min <- i_max
 *
 * R10: a line outside the bbox yields the neutral pair (+inf, -inf).  R11: row r owns
 * [16 r, 16 r + 16).  R12: the discriminant is clamped at 0.  Image y points down (R21),
 * so "bottom" = the smaller-y side.  Emits tiles (row-major ids ty*tiles_x+tx) when `out`
 * is non-null; returns the count; *n_solves counts ellipse-line intersection solves.
 * `force_dir`: -1 = paper rule, 0 = rows, 1 = columns (tests only).
 * ---------------------------------------------------------------------------------- */
static void intersect_line(double m_sweep_free, double m_line, double a_free, double b,
                           double c_line, double t, double line, double *lo, double *hi)
{
    /* Eq. 15 with the roles named generically: on the line (coordinate `line` along the
     * swept axis), solve a_free u^2 + 2 b u v + c_line v^2 = t for u (free axis offset),
     * v = line - m_line:  u = (-b v +- sqrt((b^2 - a_free c_line) v^2 + t a_free)) / a_free
     * (contract R1: the quotient is a product with 1 / a_free) */
    double v = line - m_line;
    double disc = (b * b - a_free * c_line) * v * v + t * a_free;
    if (disc < 0.0) disc = 0.0; /* R12 */
    double s = sqrt(disc);
    double ia = 1.0 / a_free;
    *lo = m_sweep_free + (-b * v - s) * ia;
    *hi = m_sweep_free + (-b * v + s) * ia;
}

uint32_t or_accutile(double mx, double my, double a, double b, double c, double t, int tiles_x,
                     int tiles_y, uint32_t *out, uint32_t cap, int32_t *n_solves, int force_dir)
{
    double bb[4], tg[8];
    int32_t R[4];
    or_snugbox(mx, my, a, b, c, t, bb, tg);
    or_rect_snugbox(mx, my, a, b, c, t, tiles_x, tiles_y, R);
    if (n_solves) *n_solves = 0;
    if (R[0] >= R[1] || R[2] >= R[3]) return 0;
    int rows = (force_dir < 0) ? ((R[3] - R[2]) <= (R[1] - R[0])) : (force_dir == 0);

    /* Generic sweep: lines are perpendicular to the swept axis "s"; extents are along the
     * free axis "f".  Rows path: s = y, f = x.  Columns path: s = x, f = y (a<->c swap). */
    double mf, ms, af, cs, ext_lo, ext_hi, smin, smax, tmin_s, tmax_s;
    int s0, s1, f0, f1;
    if (rows) {
        mf = mx; ms = my; af = a; cs = c;
        ext_lo = bb[0]; ext_hi = bb[1]; smin = bb[2]; smax = bb[3];
        tmin_s = tg[1]; /* B_l's y */
        tmax_s = tg[3]; /* B_r's y */
        s0 = R[2]; s1 = R[3]; f0 = R[0]; f1 = R[1];
    } else {
        mf = my; ms = mx; af = c; cs = a;
        ext_lo = bb[2]; ext_hi = bb[3]; smin = bb[0]; smax = bb[1];
        tmin_s = tg[4]; /* B_t's x (the y-min tangent point) */
        tmax_s = tg[6]; /* B_b's x (the y-max tangent point) */
        s0 = R[0]; s1 = R[1]; f0 = R[2]; f1 = R[3];
    }
    uint32_t C = 0;
    double imin_lo = INFINITY, imin_hi = -INFINITY; /* R10 neutral pair */
    double line_min = (double)(s0 * TILE);
    if (line_min >= smin) {
        intersect_line(mf, ms, af, b, cs, t, line_min, &imin_lo, &imin_hi);
        if (n_solves) ++*n_solves;
    }
    for (int r = s0; r < s1; ++r) {
        double imax_lo = INFINITY, imax_hi = -INFINITY;
        double line_max = (double)((r + 1) * TILE);
        if (line_max <= smax) {
            intersect_line(mf, ms, af, b, cs, t, line_max, &imax_lo, &imax_hi);
            if (n_solves) ++*n_solves;
        }
        double lo_r = (double)(r * TILE), hi_r = (double)((r + 1) * TILE);
        double e_min = (tmin_s >= lo_r && tmin_s < hi_r) ? ext_lo : dmin(imin_lo, imax_lo);
        double e_max = (tmax_s >= lo_r && tmax_s < hi_r) ? ext_hi : dmax(imin_hi, imax_hi);
        int tmin, tmax;
        double g0 = floor(e_min / TILE), g1 = floor(e_max / TILE) + 1.0;
        if (!(g0 > f0)) g0 = f0;
        if (g0 > f1) g0 = f1;
        if (!(g1 > f0)) g1 = f0;
        if (g1 > f1) g1 = f1;
        tmin = (int)g0;
        tmax = (int)g1;
        for (int k = tmin; k < tmax; ++k) {
            if (out && C < cap) out[C] = rows ? (uint32_t)(r * tiles_x + k) : (uint32_t)(k * tiles_x + r);
            ++C;
        }
        imin_lo = imax_lo; /* i_min <- i_max */
        imin_hi = imax_hi;
    }
    return C;
}

/* ------------------------------------------------------------------------------------
 * Exact continuous-cell tile test (the plain definition AccuTile reaches, "All
 * tiles between the minimum and maximum tiles intersect the ellipse", App. A):
 * tile (tx,ty) is in the set iff min over the cell [16tx,16tx+16] x [16ty,16ty+16] of
 * q(p) = a xd^2 + 2 b xd yd + c yd^2 is <= t.  For a positive-definite quadratic the
 * minimum is 0 if the mean lies in the cell, else the least of the four edge minima,
 * each the 1-D minimiser clamped to its segment.  Float64, O(tiles).  Test pin only.
 * ---------------------------------------------------------------------------------- */
static double q_at(double a, double b, double c, double xd, double yd)
{
    return a * xd * xd + 2.0 * b * xd * yd + c * yd * yd;
}

static double q_min_cell(double mx, double my, double a, double b, double c, double X0, double X1,
                         double Y0, double Y1)
{
    if (mx >= X0 && mx <= X1 && my >= Y0 && my <= Y1) return 0.0;
    double best = INFINITY;
    double Ys[2] = {Y0, Y1}, Xs[2] = {X0, X1};
    for (int k = 0; k < 2; ++k) { /* horizontal edges y = Y: minimise over x */
        double yd = Ys[k] - my;
        double xs = mx - b * yd / a;
        if (xs < X0) xs = X0;
        if (xs > X1) xs = X1;
        double v = q_at(a, b, c, xs - mx, yd);
        if (v < best) best = v;
    }
    for (int k = 0; k < 2; ++k) { /* vertical edges x = X: minimise over y */
        double xd = Xs[k] - mx;
        double ys = my - b * xd / c;
        if (ys < Y0) ys = Y0;
        if (ys > Y1) ys = Y1;
        double v = q_at(a, b, c, xd, ys - my);
        if (v < best) best = v;
    }
    return best;
}

uint32_t or_tiles_exact(double mx, double my, double a, double b, double c, double t, int tiles_x,
                        int tiles_y, uint8_t *mask /* [tiles_y*tiles_x] */)
{
    uint32_t n = 0;
    for (int ty = 0; ty < tiles_y; ++ty)
        for (int tx = 0; tx < tiles_x; ++tx) {
            double m = q_min_cell(mx, my, a, b, c, tx * TILE, tx * TILE + TILE, ty * TILE, ty * TILE + TILE);
            uint8_t in = (m <= t);
            if (mask) mask[ty * tiles_x + tx] = in;
            n += in;
        }
    return n;
}

/* ------------------------------------------------------------------------------------
 * Projection (Sec. 3.2.1 "Preprocessing"), one Gaussian, float32 contract.
 *   p_cam = W mu + t                                   (viewing transform)
 *   Sigma_3D = R S S^T R^T                             (Eq. 3)
 *   Sigma_hat = J W Sigma_3D W^T J^T, drop last row/col (Eq. 4)
 *   Sigma_2D += 0.3 I (R5), conic = Sigma_2D^{-1} (Eq. 10)
 *   c_i = max(0, sum_k Y_k(dir) h_k + 0.5)              (R13)
 *   t = 2 log(255 sigma)                                (Eq. 11, R2)
 * Culling (R4): z < z_near (or NaN), det(Sigma_2D) <= 0, conic not PD in float64; in the
 * SnugBox / AccuTile modes also t <= 0 (opacity <= 1/255, "does not contribute").
 * The tile count of the mode is computed from the stored record (R1: count and emit use
 * the same stored values).  rec[R_NF]: x, y, depth, a, b, c, sigma, t(float), r, g, b, vis.
 * ---------------------------------------------------------------------------------- */
static uint32_t tiles_of_record(int mode, const float *rec, const int32_t *rect, int tiles_x,
                                int tiles_y, uint32_t *out, uint32_t cap);

void or_project(int n, int sh_degree, const float *mean_opac, const float *scale, const float *rot,
                const float *sh, const or_camera *cam, int mode, float *out_rec, int32_t *out_rect,
                uint32_t *out_count)
{
    const float *V = cam->viewmat;
    int tiles_x = (cam->width + TILE - 1) / TILE, tiles_y = (cam->height + TILE - 1) / TILE;
    for (int i = 0; i < n; ++i) {
        float *rec = out_rec + (size_t)i * R_NF;
        int32_t *rect = out_rect + (size_t)i * 4;
        for (int k = 0; k < R_NF; ++k) rec[k] = 0.0f;
        rect[0] = rect[1] = rect[2] = rect[3] = 0;
        out_count[i] = 0;

        float mx = mean_opac[4 * i + 0], my = mean_opac[4 * i + 1], mz = mean_opac[4 * i + 2];
        float sigma = mean_opac[4 * i + 3];
        /* camera space */
        float px = V[0] * mx + V[1] * my + V[2] * mz + V[3];
        float py = V[4] * mx + V[5] * my + V[6] * mz + V[7];
        float pz = V[8] * mx + V[9] * my + V[10] * mz + V[11];
        if (!(pz >= cam->z_near)) continue;
        /* perspective projection to pixel coordinates (R3); contract R1: quotients by z are
         * products with one reciprocal 1/z */
        float iz = 1.0f / pz;
        float tx = px * iz, ty = py * iz;
        float x2d = cam->fx * tx + cam->cx;
        float y2d = cam->fy * ty + cam->cy;
        /* Jacobian of the perspective projection at p_cam (R5: clamped tx/ty) */
        float txc = tx, tyc = ty;
        if (cam->clip > 0.0f) {
            float limx = cam->clip * ((0.5f * (float)cam->width) / cam->fx);
            float limy = cam->clip * ((0.5f * (float)cam->height) / cam->fy);
            txc = fminf(limx, fmaxf(-limx, tx));
            tyc = fminf(limy, fmaxf(-limy, ty));
        }
        float j00 = cam->fx * iz, j02 = -(cam->fx * txc) * iz;
        float j11 = cam->fy * iz, j12 = -(cam->fy * tyc) * iz;
        /* rotation from the normalised quaternion (w, x, y, z) */
        float qw = rot[4 * i + 0], qx = rot[4 * i + 1], qy = rot[4 * i + 2], qz = rot[4 * i + 3];
        float qn = 1.0f / sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
        float w = qw * qn, x = qx * qn, y = qy * qn, z = qz * qn;
        float R[3][3] = {
            {1.0f - 2.0f * (y * y + z * z), 2.0f * (x * y - w * z), 2.0f * (x * z + w * y)},
            {2.0f * (x * y + w * z), 1.0f - 2.0f * (x * x + z * z), 2.0f * (y * z - w * x)},
            {2.0f * (x * z - w * y), 2.0f * (y * z + w * x), 1.0f - 2.0f * (x * x + y * y)}};
        float s3[3] = {scale[4 * i + 0], scale[4 * i + 1], scale[4 * i + 2]};
        float M[3][3];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) M[r][k] = R[r][k] * s3[k];
        float S[3][3]; /* Eq. 3: Sigma_3D = (R S)(R S)^T */
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) S[r][k] = M[r][0] * M[k][0] + M[r][1] * M[k][1] + M[r][2] * M[k][2];
        /* T = J W (2x3): J has zeros at (0,1) and (1,0) */
        float T[2][3];
        for (int k = 0; k < 3; ++k) {
            T[0][k] = j00 * V[0 + k] + j02 * V[8 + k];
            T[1][k] = j11 * V[4 + k] + j12 * V[8 + k];
        }
        /* Eq. 4: Sigma_2D = T Sigma_3D T^T (top-left 2x2 of J W Sigma W^T J^T) */
        float U[2][3];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) U[r][k] = T[r][0] * S[0][k] + T[r][1] * S[1][k] + T[r][2] * S[2][k];
        float cxx = U[0][0] * T[0][0] + U[0][1] * T[0][1] + U[0][2] * T[0][2];
        float cxy = U[0][0] * T[1][0] + U[0][1] * T[1][1] + U[0][2] * T[1][2];
        float cyy = U[1][0] * T[1][0] + U[1][1] * T[1][1] + U[1][2] * T[1][2];
        cxx = cxx + 0.3f;
        cyy = cyy + 0.3f;
        float det = cxx * cyy - cxy * cxy;
        if (!(det > 0.0f)) continue;
        float inv = 1.0f / det;
        float a = cyy * inv, b = -cxy * inv, c = cxx * inv;
        double D = (double)a * (double)c - (double)b * (double)b;
        if (!(D > 0.0)) continue;
        double td = or_threshold(sigma);
        if (mode != OR_3SIGMA && !(td > 0.0)) continue;
        /* colour (R13) */
        float dx = mx - cam->campos[0], dy = my - cam->campos[1], dz = mz - cam->campos[2];
        float len = sqrtf(dx * dx + dy * dy + dz * dz);
        float il = 1.0f / len;
        float ux = dx * il, uy = dy * il, uz = dz * il;
        float Y[16];
        or_sh_basis(sh_degree, ux, uy, uz, Y);
        float rgb[3];
        int nb = (sh_degree + 1) * (sh_degree + 1);
        for (int ch = 0; ch < 3; ++ch) {
            float acc = 0.0f;
            for (int k = 0; k < nb; ++k) {
                int coef = k * 3 + ch;
                float h = sh[((size_t)(coef / 4) * n + i) * 4 + (coef % 4)];
                acc = acc + Y[k] * h;
            }
            acc = acc + 0.5f;
            rgb[ch] = acc > 0.0f ? acc : 0.0f;
        }
        rec[R_X] = x2d; rec[R_Y] = y2d; rec[R_DEPTH] = pz;
        rec[R_A] = a; rec[R_B] = b; rec[R_C] = c;
        rec[R_SIGMA] = sigma; rec[R_T] = (float)td;
        rec[R_R] = rgb[0]; rec[R_G] = rgb[1]; rec[R_BL] = rgb[2]; rec[R_VIS] = 1.0f;
        if (mode == OR_3SIGMA)
            or_rect_3sigma(x2d, y2d, cxx, cxy, cyy, tiles_x, tiles_y, rect);
        else
            or_rect_snugbox(x2d, y2d, a, b, c, td, tiles_x, tiles_y, rect);
        out_count[i] = tiles_of_record(mode, rec, rect, tiles_x, tiles_y, 0, 0);
    }
}

/* Tile set of one stored record under `mode` (count when out == NULL). */
static uint32_t tiles_of_record(int mode, const float *rec, const int32_t *rect, int tiles_x,
                                int tiles_y, uint32_t *out, uint32_t cap)
{
    if (rec[R_VIS] == 0.0f) return 0;
    if (mode == OR_ACCUTILE)
        return or_accutile(rec[R_X], rec[R_Y], rec[R_A], rec[R_B], rec[R_C], or_threshold(rec[R_SIGMA]),
                           tiles_x, tiles_y, out, cap, 0, -1);
    uint32_t C = 0; /* 3-sigma square / SnugBox: every tile of the rect, row-major */
    for (int ty = rect[2]; ty < rect[3]; ++ty)
        for (int tx = rect[0]; tx < rect[1]; ++tx) {
            if (out && C < cap) out[C] = (uint32_t)(ty * tiles_x + tx);
            ++C;
        }
    return C;
}

uint32_t or_tiles_of_record(int mode, const float *rec, const int32_t *rect, int tiles_x, int tiles_y,
                            uint32_t *out, uint32_t cap)
{
    return tiles_of_record(mode, rec, rect, tiles_x, tiles_y, out, cap);
}

/* ------------------------------------------------------------------------------------
 * InclusiveSum: prefix sum of the counts; returns exclusive offsets and the total.
 * ---------------------------------------------------------------------------------- */
uint64_t or_exclusive_scan(int n, const uint32_t *counts, uint64_t *offsets)
{
    uint64_t acc = 0;
    for (int i = 0; i < n; ++i) {
        offsets[i] = acc;
        acc += counts[i];
    }
    return acc;
}

/* duplicateWithKeys: for each Gaussian in index order, its tiles, key =
 * (tile_id << 32) | float_bits(depth) (R14), value = Gaussian index. */
uint64_t or_duplicate_with_keys(int n, int mode, const float *rec, const int32_t *rect,
                                const uint32_t *counts, const uint64_t *offsets, int tiles_x,
                                int tiles_y, uint64_t *keys, uint32_t *values)
{
    uint64_t written = 0;
    uint32_t *buf = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(tiles_x * tiles_y + 1));
    for (int i = 0; i < n; ++i) {
        if (counts[i] == 0) continue;
        const float *r = rec + (size_t)i * R_NF;
        uint32_t c = tiles_of_record(mode, r, rect + 4 * i, tiles_x, tiles_y, buf, tiles_x * tiles_y + 1);
        uint32_t dbits;
        memcpy(&dbits, &r[R_DEPTH], 4);
        for (uint32_t k = 0; k < c && k < counts[i]; ++k) {
            keys[offsets[i] + k] = ((uint64_t)buf[k] << 32) | dbits;
            values[offsets[i] + k] = (uint32_t)i;
        }
        written += c;
    }
    free(buf);
    return written;
}

/* RadixSort as its plain definition: a STABLE ascending sort by the 64-bit key
 * (equal keys keep emission = Gaussian-index order, R14).  Bottom-up merge sort. */
void or_sort_pairs(uint64_t n, uint64_t *keys, uint32_t *values)
{
    if (n < 2) return;
    uint64_t *k2 = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint32_t *v2 = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint64_t *ka = keys, *kb = k2;
    uint32_t *va = values, *vb = v2;
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            uint64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            uint64_t i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                if (ka[j] < ka[i]) { kb[o] = ka[j]; vb[o++] = va[j++]; }
                else { kb[o] = ka[i]; vb[o++] = va[i++]; }
            }
            while (i < mid) { kb[o] = ka[i]; vb[o++] = va[i++]; }
            while (j < hi) { kb[o] = ka[j]; vb[o++] = va[j++]; }
        }
        uint64_t *tk = ka; ka = kb; kb = tk;
        uint32_t *tv = va; va = vb; vb = tv;
    }
    if (ka != keys) {
        memcpy(keys, ka, sizeof(uint64_t) * n);
        memcpy(values, va, sizeof(uint32_t) * n);
    }
    free(k2);
    free(v2);
}

/* identifyTileRanges: per tile, [start, end) into the sorted keys; empty = (0,0). */
void or_tile_ranges(uint64_t n, const uint64_t *keys, int n_tiles, uint32_t *ranges /* 2*n_tiles */)
{
    for (int t = 0; t < 2 * n_tiles; ++t) ranges[t] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t tile = (uint32_t)(keys[i] >> 32);
        if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != tile) ranges[2 * tile] = (uint32_t)i;
        if (i == n - 1 || (uint32_t)(keys[i + 1] >> 32) != tile) ranges[2 * tile + 1] = (uint32_t)(i + 1);
    }
}

/* ------------------------------------------------------------------------------------
 * Per-pixel compositing (Sec. 3.2.3, Eqs. 5-7), float32.
 *   q = (p - mu) Sigma^{-1} (p - mu)^T evaluated as the pinned chain
 *       u = fmaf(a, dx, (b + b) * dy);  q = fmaf(dx, u, (c * dy) * dy)
 *   skip iff !(q <= t)  <=>  alpha = sigma e^{-q/2} < 1/255 (Eqs. 5, 6, 9; R15)
 *   alpha = min(0.99, sigma * expf(-0.5 q))                                  (R16)
 *   T' = T (1 - alpha); if T' < 1e-4: stop without blending               (R16)
 *   C += c alpha T; T = T'   ;   out = C + T bg                            (Eq. 7)
 * `gauss` iterates the pixel's ordered list.  Returns the number of list entries
 * consumed up to and including the last blended one (n_contrib).
 * ---------------------------------------------------------------------------------- */
static inline float pixel_q(const float *r, float pxf, float pyf)
{
    float dx = pxf - r[R_X], dy = pyf - r[R_Y];
    float u = fmaf(r[R_A], dx, (r[R_B] + r[R_B]) * dy);
    return fmaf(dx, u, (r[R_C] * dy) * dy);
}

static uint32_t composite_pixel(const float *rec, const uint32_t *list, uint32_t len, float pxf,
                                float pyf, const float *bg, float *out_rgb, float *out_T)
{
    float T = 1.0f, C[3] = {0.0f, 0.0f, 0.0f};
    uint32_t last = 0;
    for (uint32_t j = 0; j < len; ++j) {
        const float *r = rec + (size_t)list[j] * R_NF;
        float q = pixel_q(r, pxf, pyf);
        if (!(q <= r[R_T])) continue;
        float alpha = r[R_SIGMA] * expf(-0.5f * q);
        if (alpha > 0.99f) alpha = 0.99f;
        float Tn = T * (1.0f - alpha);
        if (Tn < 1e-4f) break;
        C[0] = C[0] + r[R_R] * (alpha * T);
        C[1] = C[1] + r[R_G] * (alpha * T);
        C[2] = C[2] + r[R_BL] * (alpha * T);
        T = Tn;
        last = j + 1;
    }
    for (int ch = 0; ch < 3; ++ch) out_rgb[ch] = C[ch] + T * bg[ch];
    *out_T = T;
    return last;
}

/* Tiled render: each pixel walks its tile's sorted range ("all Gaussians within its
 * corresponding tile are loaded and processed in depth order"). Image planar [3][H][W]. */
void or_render(const float *rec, const uint32_t *values, const uint32_t *ranges, int width, int height,
               const float *bg, float *img, float *outT, uint32_t *ncontrib)
{
    int tiles_x = (width + TILE - 1) / TILE;
    for (int py = 0; py < height; ++py)
        for (int px = 0; px < width; ++px) {
            int tile = (py / TILE) * tiles_x + (px / TILE);
            uint32_t s = ranges[2 * tile], e = ranges[2 * tile + 1];
            float rgb[3], T;
            uint32_t nc = composite_pixel(rec, values + s, e - s, (float)px, (float)py, bg, rgb, &T);
            size_t p = (size_t)py * width + px;
            for (int ch = 0; ch < 3; ++ch) img[(size_t)ch * width * height + p] = rgb[ch];
            if (outT) outT[p] = T;
            if (ncontrib) ncontrib[p] = nc;
        }
}

/* Unbinned render: every visible Gaussian in global (depth bits, index) order -- the
 * definition the binned render must equal ("identical renders", R17). `order` is
 * the caller-supplied global order (from or_global_order). */
void or_global_order(int n, const float *rec, uint32_t *order, uint32_t *n_vis)
{
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    uint32_t m = 0;
    for (int i = 0; i < n; ++i) {
        const float *r = rec + (size_t)i * R_NF;
        if (r[R_VIS] == 0.0f) continue;
        uint32_t d;
        memcpy(&d, &r[R_DEPTH], 4);
        keys[m] = d;
        order[m] = (uint32_t)i;
        ++m;
    }
    or_sort_pairs(m, keys, order);
    *n_vis = m;
    free(keys);
}

void or_render_unbinned(const float *rec, const uint32_t *order, uint32_t n_vis, int width, int height,
                        const float *bg, int x0, int x1, int y0, int y1, float *img /* [3][H][W] */)
{
    for (int py = y0; py < y1; ++py)
        for (int px = x0; px < x1; ++px) {
            float rgb[3], T;
            composite_pixel(rec, order, n_vis, (float)px, (float)py, bg, rgb, &T);
            size_t p = (size_t)py * width + px;
            for (int ch = 0; ch < 3; ++ch) img[(size_t)ch * width * height + p] = rgb[ch];
        }
}

/* ------------------------------------------------------------------------------------
 * Efficient pruning score (Sec. 4.2.1, Eqs. 20-21), accumulated into score[]:
 *   U~_i += sum_p sum_ch ( dC_ch(p) / dg_i(p) )^2,   dC/dg_i = sigma_i dC/dalpha_i (Eq. 5)
 * with, from Eq. 7 (R18, R19), for each Gaussian i blended at pixel p:
 *   dC_ch/dalpha_i = c_i,ch T_i - ( sum_{k>i} c_k,ch alpha_k T_k + bg_ch T_final ) / (1 - alpha_i)
 * T_k = prod_{j<k} (1 - alpha_j).  The blended set and the alphas come from the same
 * float32 forward as or_render (the kernel's precision decides, R22); the derivative
 * itself is evaluated from its definition in float64.
 * ---------------------------------------------------------------------------------- */
void or_prune_score(const float *rec, const uint32_t *values, const uint32_t *ranges, int width,
                    const float *bg, double *score, int x0, int x1, int y0, int y1)
{
    int tiles_x = (width + TILE - 1) / TILE;
    uint32_t cap = 0;
    uint32_t *ids = 0;
    double *al = 0;
    for (int py = y0; py < y1; ++py)
        for (int px = x0; px < x1; ++px) {
            int tile = (py / TILE) * tiles_x + (px / TILE);
            uint32_t s = ranges[2 * tile], e = ranges[2 * tile + 1];
            if (e - s + 1 > cap) {
                cap = 2 * (e - s + 1);
                ids = (uint32_t *)realloc(ids, sizeof(uint32_t) * cap);
                al = (double *)realloc(al, sizeof(double) * cap);
            }
            /* forward (float32, identical decisions to or_render) */
            float T = 1.0f;
            uint32_t K = 0;
            for (uint32_t j = s; j < e; ++j) {
                const float *r = rec + (size_t)values[j] * R_NF;
                float q = pixel_q(r, (float)px, (float)py);
                if (!(q <= r[R_T])) continue;
                float alpha = r[R_SIGMA] * expf(-0.5f * q);
                if (alpha > 0.99f) alpha = 0.99f;
                float Tn = T * (1.0f - alpha);
                if (Tn < 1e-4f) break;
                T = Tn;
                ids[K] = values[j];
                al[K] = alpha;
                ++K;
            }
            /* definition, float64 */
            double Tf = 1.0;
            for (uint32_t k = 0; k < K; ++k) Tf *= (1.0 - al[k]);
            double suffix[3] = {0.0, 0.0, 0.0}; /* sum_{k>i} c_k alpha_k T_k */
            /* T_i for all i (prefix products) */
            double *Ti = (double *)malloc(sizeof(double) * (K ? K : 1));
            double acc = 1.0;
            for (uint32_t k = 0; k < K; ++k) { Ti[k] = acc; acc *= (1.0 - al[k]); }
            for (int64_t i = (int64_t)K - 1; i >= 0; --i) {
                const float *r = rec + (size_t)ids[i] * R_NF;
                double cc[3] = {r[R_R], r[R_G], r[R_BL]};
                double term = 0.0;
                for (int ch = 0; ch < 3; ++ch) {
                    double d = cc[ch] * Ti[i] - (suffix[ch] + bg[ch] * Tf) / (1.0 - al[i]);
                    double g = (double)r[R_SIGMA] * d;
                    term += g * g;
                }
                score[ids[i]] += term;
                for (int ch = 0; ch < 3; ++ch) suffix[ch] += cc[ch] * al[i] * Ti[i];
            }
            free(Ti);
        }
    free(ids);
    free(al);
}

/* Per-pixel colour as a function of an explicit alpha list (finite-difference pin of the
 * score): C_ch = sum_k c_k alpha_k T_k + bg T_final, float64, no skip / clamp. */
void or_composite_alphas(int K, const double *alpha, const double *rgb /* K*3 */, const double *bg,
                         double *out /* 3 */)
{
    double T = 1.0;
    out[0] = out[1] = out[2] = 0.0;
    for (int k = 0; k < K; ++k) {
        for (int ch = 0; ch < 3; ++ch) out[ch] += rgb[3 * k + ch] * alpha[k] * T;
        T *= (1.0 - alpha[k]);
    }
    for (int ch = 0; ch < 3; ++ch) out[ch] += bg[ch] * T;
}

/* ------------------------------------------------------------------------------------
 * Whole forward pipeline for one view (CS3): project -> count -> scan -> emit -> stable
 * sort -> ranges -> tiled render.  Caller owns all buffers; returns the pair count P
 * (keys/values are written only if P <= cap).
 * ---------------------------------------------------------------------------------- */
uint64_t or_frame(int n, int sh_degree, const float *mean_opac, const float *scale, const float *rot,
                  const float *sh, const or_camera *cam, int mode, const float *bg, float *rec,
                  int32_t *rect, uint32_t *counts, uint64_t *offsets, uint64_t *keys, uint32_t *values,
                  uint64_t cap, uint32_t *ranges, float *img, float *outT, uint32_t *ncontrib)
{
    int tiles_x = (cam->width + TILE - 1) / TILE, tiles_y = (cam->height + TILE - 1) / TILE;
    or_project(n, sh_degree, mean_opac, scale, rot, sh, cam, mode, rec, rect, counts);
    uint64_t P = or_exclusive_scan(n, counts, offsets);
    if (P > cap) return P;
    or_duplicate_with_keys(n, mode, rec, rect, counts, offsets, tiles_x, tiles_y, keys, values);
    or_sort_pairs(P, keys, values);
    or_tile_ranges(P, keys, tiles_x * tiles_y, ranges);
    if (img) or_render(rec, values, ranges, cam->width, cam->height, bg, img, outT, ncontrib);
    return P;
}

/* Tiled render / score restricted to a list of tiles (sampled checks at full size; the
 * per-pixel arithmetic is composite_pixel / the score loop above, unchanged). */
void or_render_tiles(const float *rec, const uint32_t *values, const uint32_t *ranges, int width, int height,
                     const float *bg, const int32_t *tiles, int n_list, float *img, float *outT, uint32_t *ncontrib)
{
    int tiles_x = (width + TILE - 1) / TILE;
    for (int k = 0; k < n_list; ++k) {
        int tile = tiles[k], tx = tile % tiles_x, ty = tile / tiles_x;
        uint32_t s = ranges[2 * tile], e = ranges[2 * tile + 1];
        for (int py = ty * TILE; py < ty * TILE + TILE && py < height; ++py)
            for (int px = tx * TILE; px < tx * TILE + TILE && px < width; ++px) {
                float rgb[3], T;
                uint32_t nc = composite_pixel(rec, values + s, e - s, (float)px, (float)py, bg, rgb, &T);
                size_t p = (size_t)py * width + px;
                for (int ch = 0; ch < 3; ++ch) img[(size_t)ch * width * height + p] = rgb[ch];
                if (outT) outT[p] = T;
                if (ncontrib) ncontrib[p] = nc;
            }
    }
}

void or_prune_score_tiles(const float *rec, const uint32_t *values, const uint32_t *ranges, int width,
                          int height, const float *bg, double *score, const int32_t *tiles, int n_list)
{
    int tiles_x = (width + TILE - 1) / TILE;
    for (int k = 0; k < n_list; ++k) {
        int tile = tiles[k], tx = tile % tiles_x, ty = tile / tiles_x;
        int x1 = tx * TILE + TILE < width ? tx * TILE + TILE : width;
        int y1 = ty * TILE + TILE < height ? ty * TILE + TILE : height;
        or_prune_score(rec, values, ranges, width, bg, score, tx * TILE, x1, ty * TILE, y1);
    }
}

/* ------------------------------------------------------------------------------------
 * Prune selection (Sec. 4.2: "removing a set percentage with the lowest sensitivities",
 * P:381; Soft Pruning P:422-425, Hard Pruning P:434-436): remove exactly
 * k = floor(ratio * N) Gaussians with the smallest score U~; among equal scores the higher
 * canonical index is removed first (the lower index is kept).  keep[i] = 1 for survivors.
 * Plain definition: order all indices by (score ascending, index descending), remove the
 * first k.  Returns k.
 * ---------------------------------------------------------------------------------- */
static const double *g_sel_score;
static int cmp_prune(const void *pa, const void *pb)
{
    int a = *(const int *)pa, b = *(const int *)pb;
    double sa = g_sel_score[a], sb = g_sel_score[b];
    if (sa < sb) return -1;
    if (sa > sb) return 1;
    return (a > b) ? -1 : (a < b ? 1 : 0); /* equal scores: higher index first */
}

int64_t or_prune_select(int n, const double *score, double ratio, uint8_t *keep)
{
    int64_t k = (int64_t)floor(ratio * (double)n);
    if (k < 0) k = 0;
    if (k > n) k = n;
    int *idx = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) { idx[i] = i; keep[i] = 1; }
    g_sel_score = score;
    qsort(idx, (size_t)n, sizeof(int), cmp_prune);
    for (int64_t j = 0; j < k; ++j) keep[idx[j]] = 0;
    free(idx);
    return k;
}
