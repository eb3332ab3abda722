/*
 * ss_oracle_bwd.c -- plain, slow CPU ORACLE for the render backward and the preprocess
 * backward ("the efficient flow of gradients").
 *
 * TEST INFRASTRUCTURE ONLY (same rules as ss_oracle.c): only tests/, __graft_entry__ and
 * bench.py's CPU legs may load it; it shares no code, header or constant generator with
 * the CUDA path.
 *
 * What is differentiated is the forward exactly as ss_oracle.c computes it (Eqs. 3-7 with
 * readings R3-R5, R13, R15-R16, R24):
 *   p = W mu + t;  x2d = fx p.x/p.z + cx,  y2d = fy p.y/p.z + cy
 *   Sigma_3D = R S S^T R^T (Eq. 3), R = R(q/|q|), S = diag(s)
 *   Sigma_2D = J W Sigma_3D W^T J^T + 0.3 I (Eq. 4, R5; J built from the clamped p.x/p.z)
 *   conic (a, b, c) = Sigma_2D^-1 (Eq. 10, R24 order), q = a dx^2 + 2 b dx dy + c dy^2
 *   alpha = min(0.99, sigma exp(-q/2)) (Eq. 5, R16);  c = max(0, sum_k Y_k(dir) h_k + 0.5)
 *   C = sum_i c_i alpha_i T_i + bg T_final,  T_i = prod_{j<i} (1 - alpha_j)            (Eq. 7)
 * Reading R27: the gradient is the derivative of that function where it is
 * differentiable: a clamped alpha (0.99), a clamped J entry (|p.x/p.z| at the clip) and a
 * clamped colour (c = 0) pass no gradient through the clamped quantity; skipped (alpha <
 * 1/255) and non-blended (terminating, later) Gaussians contribute nothing; t and the tile
 * sets are piecewise constant and carry none; depth only orders the blend.
 *
 * Precision: the per-pixel blend DECISIONS (which Gaussians blend, the clamp) are taken in
 * float32 exactly as ss_oracle.c's composite_pixel takes them on the stored float32 record
 * (R22: the kernel's precision decides); every derivative is evaluated in float64 from its
 * definition.  The preprocess backward recomputes the forward in float64 from the parameters
 * (passed as float64, so that the finite-difference pins can perturb them in float64).  or_project_f64 / or_loss_f64 are the float64 forward used by the finite-
 * difference pins (tests/test_oracle_backward.py).
 *
 * Pins: finite differences of or_loss_f64 (render backward), of or_project_f64 contracted
 * with random cotangents (preprocess backward) and of their composition (end to end);
 * or_project_f64 / or_loss_f64 equal the pinned float32 forward of ss_oracle.c to float32
 * rounding.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16

typedef struct {
    float viewmat[12];
    float fx, fy, cx, cy;
    float campos[3];
    int32_t width, height;
    float z_near;
    float clip;
} orb_camera; /* identical layout to or_camera (ss_oracle.c) */

/* float32 record fields of ss_oracle.c (or_project) */
enum { R_X = 0, R_Y, R_DEPTH, R_A, R_B, R_C, R_SIGMA, R_T, R_R, R_G, R_BL, R_VIS, R_NF };

/* 2D gradient record, float64 [n][9] */
enum { G_X = 0, G_Y, G_A, G_B, G_C, G_SIGMA, G_R, G_G, G_BL, G_NF };

/* float64 projected record of or_project_f64, [n][F_NF] */
enum { F_X = 0, F_Y, F_DEPTH, F_A, F_B, F_C, F_SIGMA, F_R, F_G, F_BL, F_VIS, F_NF };

/* ------------------------------------------------------------------------------------
 * Real SH basis up to degree 3 (R13) in float64 at direction (x, y, z), and its partial
 * derivatives dY/dx, dY/dy, dY/dz of the same polynomials (the basis is evaluated on the
 * unit direction; the normalisation is differentiated separately).
 * ---------------------------------------------------------------------------------- */
static const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
static const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                             -1.0925484305920792, 0.5462742152960396};
static const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                             0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                             -0.5900435899266435};

static void sh_basis_d(int deg, double x, double y, double z, double *Y, double *dX, double *dY, double *dZ)
{
    for (int k = 0; k < 16; ++k) Y[k] = dX[k] = dY[k] = dZ[k] = 0.0;
    Y[0] = C0;
    if (deg < 1) return;
    Y[1] = -C1 * y;  dY[1] = -C1;
    Y[2] = C1 * z;   dZ[2] = C1;
    Y[3] = -C1 * x;  dX[3] = -C1;
    if (deg < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = C2[0] * x * y;                 dX[4] = C2[0] * y;  dY[4] = C2[0] * x;
    Y[5] = C2[1] * y * z;                 dY[5] = C2[1] * z;  dZ[5] = C2[1] * y;
    Y[6] = C2[2] * (2 * zz - xx - yy);    dX[6] = -2 * C2[2] * x; dY[6] = -2 * C2[2] * y; dZ[6] = 4 * C2[2] * z;
    Y[7] = C2[3] * x * z;                 dX[7] = C2[3] * z;  dZ[7] = C2[3] * x;
    Y[8] = C2[4] * (xx - yy);             dX[8] = 2 * C2[4] * x; dY[8] = -2 * C2[4] * y;
    if (deg < 3) return;
    Y[9] = C3[0] * y * (3 * xx - yy);
    dX[9] = C3[0] * 6 * x * y;            dY[9] = C3[0] * (3 * xx - 3 * yy);
    Y[10] = C3[1] * x * y * z;
    dX[10] = C3[1] * y * z;  dY[10] = C3[1] * x * z;  dZ[10] = C3[1] * x * y;
    Y[11] = C3[2] * y * (4 * zz - xx - yy);
    dX[11] = C3[2] * (-2 * x * y);  dY[11] = C3[2] * (4 * zz - xx - 3 * yy);  dZ[11] = C3[2] * 8 * y * z;
    Y[12] = C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
    dX[12] = C3[3] * (-6 * x * z);  dY[12] = C3[3] * (-6 * y * z);  dZ[12] = C3[3] * (6 * zz - 3 * xx - 3 * yy);
    Y[13] = C3[4] * x * (4 * zz - xx - yy);
    dX[13] = C3[4] * (4 * zz - 3 * xx - yy);  dY[13] = C3[4] * (-2 * x * y);  dZ[13] = C3[4] * 8 * x * z;
    Y[14] = C3[5] * z * (xx - yy);
    dX[14] = C3[5] * 2 * x * z;  dY[14] = C3[5] * (-2 * y * z);  dZ[14] = C3[5] * (xx - yy);
    Y[15] = C3[6] * x * (xx - 3 * yy);
    dX[15] = C3[6] * (3 * xx - 3 * yy);  dY[15] = C3[6] * (-6 * x * y);
}

/* SH coefficient k*3+ch of Gaussian i in the host scene layout the oracle reads
 * (coefficient-major planes [P][n][4], as ss_oracle.c's or_project). */
static size_t sh_index(int n, int deg, int i, int coef)
{
    (void)deg;
    return ((size_t)(coef / 4) * n + i) * 4 + coef % 4;
}

/* ------------------------------------------------------------------------------------
 * Forward intermediates of one Gaussian in float64 (the definitions listed in the header).
 * ---------------------------------------------------------------------------------- */
typedef struct {
    int vis;
    double mu[3], p[3], iz, tx, ty, txc, tyc;
    int clx, cly;            /* J entry clamped (R5) */
    double J[2][3];          /* J (2x3; zeros at (0,1), (1,0)) */
    double T[2][3];          /* J W */
    double qn[4], qlen;      /* normalised quaternion (w, x, y, z), |q| */
    double R[3][3], s[3], M[3][3], S3[3][3];
    double cxx, cxy, cyy, det, a, b, c;
    double sigma;
    double dir[3], dlen, Y[16], dYx[16], dYy[16], dYz[16];
    double raw[3], rgb[3];
    double x2d, y2d;
} fwd64;

static void forward64(int n, int deg, const double *mean_opac, const double *scale, const double *rot,
                      const double *sh, const orb_camera *cam, int i, fwd64 *f)
{
    memset(f, 0, sizeof(*f));
    const float *V = cam->viewmat;
    for (int k = 0; k < 3; ++k) f->mu[k] = mean_opac[4 * i + k];
    f->sigma = mean_opac[4 * i + 3];
    for (int r = 0; r < 3; ++r)
        f->p[r] = V[4 * r + 0] * f->mu[0] + V[4 * r + 1] * f->mu[1] + V[4 * r + 2] * f->mu[2] + V[4 * r + 3];
    if (!(f->p[2] >= cam->z_near)) return;
    f->iz = 1.0 / f->p[2];
    f->tx = f->p[0] * f->iz;
    f->ty = f->p[1] * f->iz;
    f->x2d = cam->fx * f->tx + cam->cx;
    f->y2d = cam->fy * f->ty + cam->cy;
    f->txc = f->tx;
    f->tyc = f->ty;
    if (cam->clip > 0.0f) {
        double limx = (double)cam->clip * (0.5 * cam->width / cam->fx);
        double limy = (double)cam->clip * (0.5 * cam->height / cam->fy);
        if (f->tx > limx) { f->txc = limx; f->clx = 1; }
        if (f->tx < -limx) { f->txc = -limx; f->clx = 1; }
        if (f->ty > limy) { f->tyc = limy; f->cly = 1; }
        if (f->ty < -limy) { f->tyc = -limy; f->cly = 1; }
    }
    f->J[0][0] = cam->fx * f->iz;
    f->J[0][2] = -cam->fx * f->txc * f->iz;
    f->J[1][1] = cam->fy * f->iz;
    f->J[1][2] = -cam->fy * f->tyc * f->iz;
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k)
            f->T[r][k] = f->J[r][0] * V[0 + k] + f->J[r][1] * V[4 + k] + f->J[r][2] * V[8 + k];
    double q[4];
    for (int k = 0; k < 4; ++k) q[k] = rot[4 * i + k];
    f->qlen = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) f->qn[k] = q[k] / f->qlen;
    double w = f->qn[0], x = f->qn[1], y = f->qn[2], z = f->qn[3];
    double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                      {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                      {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    memcpy(f->R, R, sizeof(R));
    for (int k = 0; k < 3; ++k) f->s[k] = scale[4 * i + k];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) f->M[r][k] = R[r][k] * f->s[k];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k)
            f->S3[r][k] = f->M[r][0] * f->M[k][0] + f->M[r][1] * f->M[k][1] + f->M[r][2] * f->M[k][2];
    double U[2][3];
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) U[r][k] = f->T[r][0] * f->S3[0][k] + f->T[r][1] * f->S3[1][k] + f->T[r][2] * f->S3[2][k];
    f->cxx = U[0][0] * f->T[0][0] + U[0][1] * f->T[0][1] + U[0][2] * f->T[0][2] + 0.3;
    f->cxy = U[0][0] * f->T[1][0] + U[0][1] * f->T[1][1] + U[0][2] * f->T[1][2];
    f->cyy = U[1][0] * f->T[1][0] + U[1][1] * f->T[1][1] + U[1][2] * f->T[1][2] + 0.3;
    f->det = f->cxx * f->cyy - f->cxy * f->cxy;
    if (!(f->det > 0.0)) return;
    f->a = f->cyy / f->det;
    f->b = -f->cxy / f->det;
    f->c = f->cxx / f->det;
    for (int k = 0; k < 3; ++k) f->dir[k] = f->mu[k] - cam->campos[k];
    f->dlen = sqrt(f->dir[0] * f->dir[0] + f->dir[1] * f->dir[1] + f->dir[2] * f->dir[2]);
    double u[3] = {f->dir[0] / f->dlen, f->dir[1] / f->dlen, f->dir[2] / f->dlen};
    sh_basis_d(deg, u[0], u[1], u[2], f->Y, f->dYx, f->dYy, f->dYz);
    int nb = (deg + 1) * (deg + 1);
    for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
        for (int k = 0; k < nb; ++k) acc += f->Y[k] * (double)sh[sh_index(n, deg, i, k * 3 + ch)];
        f->raw[ch] = acc + 0.5;
        f->rgb[ch] = f->raw[ch] > 0.0 ? f->raw[ch] : 0.0;
    }
    f->vis = 1;
}

/* Float64 projection of every Gaussian: rec64[i] = (x2d, y2d, depth, a, b, c, sigma, r, g, b,
 * visible).  The finite-difference pins differentiate this function. */
void or_project_f64(int n, int deg, const double *mean_opac, const double *scale, const double *rot,
                    const double *sh, const orb_camera *cam, double *rec64)
{
    for (int i = 0; i < n; ++i) {
        fwd64 f;
        forward64(n, deg, mean_opac, scale, rot, sh, cam, i, &f);
        double *r = rec64 + (size_t)i * F_NF;
        for (int k = 0; k < F_NF; ++k) r[k] = 0.0;
        if (!f.vis) continue;
        r[F_X] = f.x2d; r[F_Y] = f.y2d; r[F_DEPTH] = f.p[2];
        r[F_A] = f.a; r[F_B] = f.b; r[F_C] = f.c; r[F_SIGMA] = f.sigma;
        r[F_R] = f.rgb[0]; r[F_G] = f.rgb[1]; r[F_BL] = f.rgb[2]; r[F_VIS] = 1.0;
    }
}

/* Float64 loss L = sum_{ch,p} w[ch][p] C_ch(p) of the UNBINNED render (R17) of float64
 * records: every visible Gaussian in ascending (depth, index) order, the per-pixel rule of
 * a6 in float64 (skip iff q > t, t = 2 log(255 sigma); alpha = min(0.99, sigma e^{-q/2});
 * stop before blending when T(1-alpha) < 1e-4; C = sum c alpha T + T bg).  Window
 * [x0,x1) x [y0,y1).  blend_hash (optional) receives a hash of the set of blended (pixel,
 * Gaussian) pairs: the finite-difference pins only use steps that leave that set unchanged
 * (the loss jumps where a pixel crosses alpha = 1/255 or the 1e-4 stop, R27). */
static const double *g_depth;
static int cmp_depth(const void *pa, const void *pb)
{
    int a = *(const int *)pa, b = *(const int *)pb;
    if (g_depth[(size_t)a * F_NF] < g_depth[(size_t)b * F_NF]) return -1;
    if (g_depth[(size_t)a * F_NF] > g_depth[(size_t)b * F_NF]) return 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

double or_loss_f64(int n, const double *rec64, int width, int height, const double *bg, const double *w,
                   int x0, int x1, int y0, int y1, uint64_t *blend_hash /* nullable */)
{
    int *ord = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (rec64[(size_t)i * F_NF + F_VIS] != 0.0 && rec64[(size_t)i * F_NF + F_SIGMA] > 1.0 / 255.0) ord[m++] = i;
    g_depth = rec64 + F_DEPTH;
    qsort(ord, (size_t)m, sizeof(int), cmp_depth);
    double L = 0.0;
    uint64_t H = 0;
    size_t plane = (size_t)width * height;
    for (int py = y0; py < y1; ++py)
        for (int px = x0; px < x1; ++px) {
            double T = 1.0, C[3] = {0, 0, 0};
            for (int j = 0; j < m; ++j) {
                const double *r = rec64 + (size_t)ord[j] * F_NF;
                double dx = px - r[F_X], dy = py - r[F_Y];
                double q = r[F_A] * dx * dx + 2.0 * r[F_B] * dx * dy + r[F_C] * dy * dy;
                double t = 2.0 * log(255.0 * r[F_SIGMA]);
                if (q > t) continue;
                double alpha = r[F_SIGMA] * exp(-0.5 * q);
                if (alpha > 0.99) alpha = 0.99;
                double Tn = T * (1.0 - alpha);
                if (Tn < 1e-4) break;
                for (int ch = 0; ch < 3; ++ch) C[ch] += r[F_R + ch] * alpha * T;
                T = Tn;
                H = H * 0x9E3779B97F4A7C15ull + ((uint64_t)py * width + px) * 0x100000001B3ull + (uint64_t)ord[j] + 1;
            }
            size_t p = (size_t)py * width + px;
            for (int ch = 0; ch < 3; ++ch) L += w[ch * plane + p] * (C[ch] + T * bg[ch]);
        }
    free(ord);
    if (blend_hash) *blend_hash = H;
    return L;
}

/* ------------------------------------------------------------------------------------
 * Render backward for the pixels of [x0,x1) x [y0,y1) of a binned frame (records, sorted
 * values and ranges of ss_oracle.c).  dimg = dL/dC, float32 [3][H][W].  Accumulates into
 * g2d (float64 [n][9]: dL/d(x2d, y2d, a, b, c, sigma, r, g, b)) and, when gabs != NULL,
 * the sums of the ABSOLUTE per-pixel terms of each entry (the scale of the float32
 * accumulation error, used by the GPU parity tolerance).
 * Per pixel, from Eq. 7 and Eq. 5 (the score's derivative, extended to the chain):
 *   dC_ch/dalpha_i = c_i,ch T_i - (sum_{k>i} c_k,ch alpha_k T_k + bg_ch T_final)/(1-alpha_i)
 *   dC_ch/dc_i,ch  = alpha_i T_i
 *   alpha_i = sigma_i G_i, G_i = exp(-q_i/2) (unclamped):  dalpha/dsigma = G, dalpha/dq = -alpha/2
 *   dq/dx2d = -2 (a dx + b dy), dq/dy2d = -2 (b dx + c dy), dq/da = dx^2, dq/db = 2 dx dy, dq/dc = dy^2
 * with dx = px - x2d, dy = py - y2d.
 * ---------------------------------------------------------------------------------- */
void or_render_backward(const float *rec, const uint32_t *values, const uint32_t *ranges, int width, int height,
                        const float *bg, const float *dimg, int x0, int x1, int y0, int y1, double *g2d,
                        double *gabs)
{
    int tiles_x = (width + TILE - 1) / TILE;
    size_t plane = (size_t)width * height;
    uint32_t cap = 0;
    uint32_t *ids = 0;
    double *al = 0;
    int *clamped = 0;
    for (int py = y0; py < y1; ++py)
        for (int px = x0; px < x1; ++px) {
            int tile = (py / TILE) * tiles_x + (px / TILE);
            uint32_t s = ranges[2 * tile], e = ranges[2 * tile + 1];
            if (e - s + 1 > cap) {
                cap = 2 * (e - s + 1);
                ids = (uint32_t *)realloc(ids, sizeof(uint32_t) * cap);
                al = (double *)realloc(al, sizeof(double) * cap);
                clamped = (int *)realloc(clamped, sizeof(int) * cap);
            }
            /* forward decisions, float32, identical to composite_pixel (ss_oracle.c) */
            float Tf32 = 1.0f;
            uint32_t K = 0;
            for (uint32_t j = s; j < e; ++j) {
                const float *r = rec + (size_t)values[j] * R_NF;
                float dxf = (float)px - r[R_X], dyf = (float)py - r[R_Y];
                float u = fmaf(r[R_A], dxf, (r[R_B] + r[R_B]) * dyf);
                float q = fmaf(dxf, u, (r[R_C] * dyf) * dyf);
                if (!(q <= r[R_T])) continue;
                float alpha = r[R_SIGMA] * expf(-0.5f * q);
                int cl = 0;
                if (alpha > 0.99f) { alpha = 0.99f; cl = 1; }
                float Tn = Tf32 * (1.0f - alpha);
                if (Tn < 1e-4f) break;
                Tf32 = Tn;
                ids[K] = values[j];
                clamped[K] = cl;
                ++K;
            }
            /* alphas in float64 from their definition on the record */
            for (uint32_t k = 0; k < K; ++k) {
                const float *r = rec + (size_t)ids[k] * R_NF;
                double dx = (double)px - r[R_X], dy = (double)py - r[R_Y];
                double q = r[R_A] * dx * dx + 2.0 * (double)r[R_B] * dx * dy + r[R_C] * dy * dy;
                al[k] = clamped[k] ? 0.99 : (double)r[R_SIGMA] * exp(-0.5 * q);
            }
            size_t p = (size_t)py * width + px;
            double dLdC[3] = {dimg[p], dimg[plane + p], dimg[2 * plane + p]};
            double Ti = 1.0, Tfin = 1.0;
            for (uint32_t k = 0; k < K; ++k) Tfin *= (1.0 - al[k]);
            for (uint32_t i = 0; i < K; ++i) {
                const float *r = rec + (size_t)ids[i] * R_NF;
                double cc[3] = {r[R_R], r[R_G], r[R_BL]};
                /* suffix sum_{k>i} c_k alpha_k T_k */
                double suf[3] = {0, 0, 0}, Tk = Ti * (1.0 - al[i]);
                for (uint32_t k = i + 1; k < K; ++k) {
                    const float *rk = rec + (size_t)ids[k] * R_NF;
                    suf[0] += rk[R_R] * al[k] * Tk;
                    suf[1] += rk[R_G] * al[k] * Tk;
                    suf[2] += rk[R_BL] * al[k] * Tk;
                    Tk *= (1.0 - al[k]);
                }
                double dLda = 0.0;
                double term[G_NF];
                for (int k = 0; k < G_NF; ++k) term[k] = 0.0;
                for (int ch = 0; ch < 3; ++ch) {
                    dLda += dLdC[ch] * (cc[ch] * Ti - (suf[ch] + bg[ch] * Tfin) / (1.0 - al[i]));
                    term[G_R + ch] = dLdC[ch] * al[i] * Ti;
                }
                if (!clamped[i]) {
                    double dx = (double)px - r[R_X], dy = (double)py - r[R_Y];
                    double G = exp(-0.5 * (r[R_A] * dx * dx + 2.0 * (double)r[R_B] * dx * dy + r[R_C] * dy * dy));
                    double dLdq = dLda * (-0.5 * al[i]);
                    term[G_SIGMA] = dLda * G;
                    term[G_X] = dLdq * (-2.0 * (r[R_A] * dx + (double)r[R_B] * dy));
                    term[G_Y] = dLdq * (-2.0 * ((double)r[R_B] * dx + r[R_C] * dy));
                    term[G_A] = dLdq * dx * dx;
                    term[G_B] = dLdq * 2.0 * dx * dy;
                    term[G_C] = dLdq * dy * dy;
                }
                for (int k = 0; k < G_NF; ++k) {
                    g2d[(size_t)ids[i] * G_NF + k] += term[k];
                    if (gabs) gabs[(size_t)ids[i] * G_NF + k] += fabs(term[k]);
                }
                Ti *= (1.0 - al[i]);
            }
        }
    free(ids);
    free(al);
    free(clamped);
}

void or_render_backward_tiles(const float *rec, const uint32_t *values, const uint32_t *ranges, int width,
                              int height, const float *bg, const float *dimg, const int32_t *tiles, int n_list,
                              double *g2d, double *gabs)
{
    int tiles_x = (width + TILE - 1) / TILE;
    for (int k = 0; k < n_list; ++k) {
        int tile = tiles[k], tx = tile % tiles_x, ty = tile / tiles_x;
        int x1 = tx * TILE + TILE < width ? tx * TILE + TILE : width;
        int y1 = ty * TILE + TILE < height ? ty * TILE + TILE : height;
        or_render_backward(rec, values, ranges, width, height, bg, dimg, tx * TILE, x1, ty * TILE, y1, g2d, gabs);
    }
}

/* ------------------------------------------------------------------------------------
 * Preprocess backward: from g2d = dL/d(x2d, y2d, a, b, c, sigma, r, g, b) of one view to
 * dL/d(mu, sigma), dL/ds, dL/dq (unnormalised quaternion) and dL/dh, float64, ACCUMULATED
 * (+=) into dmean_opac [n][4], dscale [n][4] (w = 0), drot [n][4], dsh (layout of sh).
 * Chain rule, step by step, in the order of the forward:
 *   colour:  dL/dh_k,ch = dL/dc_ch Y_k (if raw_ch > 0);  dL/du = sum_ch dL/dc_ch sum_k h dY_k/du
 *            u = d/|d|, d = mu - campos:  dL/dmu += (dL/du - u (u.dL/du)) / |d|
 *   conic:   (a, b, c) = (cyy, -cxy, cxx)/det, det = cxx cyy - cxy^2 (written-out partials)
 *   Eq. 4:   Sigma_2D = T Sigma_3D T^T with T = J W:
 *            dL/dSigma_3D = T^T G T,   dL/dT = 2 G T Sigma_3D,  G = [[gxx, gxy/2], [gxy/2, gyy]]
 *   J:       dL/dJ = dL/dT W^T;  J00 = fx/z, J02 = -fx txc/z, J11 = fy/z, J12 = -fy tyc/z,
 *            txc = clamp(x/z) (constant when clamped, R5/R27)
 *   mean:    x2d = fx x/z + cx, y2d = fy y/z + cy;  dL/dmu += W^T dL/dp
 *   Eq. 3:   Sigma_3D = M M^T, M = R S:  dL/dM = 2 dL/dSigma_3D M;  dL/ds_k = sum_r dL/dM_rk R_rk;
 *            dL/dR_rk = dL/dM_rk s_k;  R(qn) written-out partials;  qn = q/|q|:
 *            dL/dq = (dL/dqn - qn (qn.dL/dqn)) / |q|
 *   opacity: dL/dsigma = g2d.sigma (t only selects tiles).
 * ---------------------------------------------------------------------------------- */
void or_project_backward(int n, int deg, const double *mean_opac, const double *scale, const double *rot,
                         const double *sh, const orb_camera *cam, const double *g2d, double *dmean_opac,
                         double *dscale, double *drot, double *dsh)
{
    const float *V = cam->viewmat;
    int nb = (deg + 1) * (deg + 1);
    for (int i = 0; i < n; ++i) {
        const double *g = g2d + (size_t)i * G_NF;
        int any = 0;
        for (int k = 0; k < G_NF; ++k) any |= g[k] != 0.0;
        if (!any) continue;
        fwd64 f;
        forward64(n, deg, mean_opac, scale, rot, sh, cam, i, &f);
        if (!f.vis) continue;
        double dmu[3] = {0, 0, 0};
        /* ---- colour (R13) */
        double du[3] = {0, 0, 0};
        for (int ch = 0; ch < 3; ++ch) {
            if (!(f.raw[ch] > 0.0)) continue;
            double gc = g[G_R + ch];
            for (int k = 0; k < nb; ++k) {
                size_t idx = sh_index(n, deg, i, k * 3 + ch);
                dsh[idx] += gc * f.Y[k];
                double h = sh[idx];
                du[0] += gc * h * f.dYx[k];
                du[1] += gc * h * f.dYy[k];
                du[2] += gc * h * f.dYz[k];
            }
        }
        double u[3] = {f.dir[0] / f.dlen, f.dir[1] / f.dlen, f.dir[2] / f.dlen};
        double udu = u[0] * du[0] + u[1] * du[1] + u[2] * du[2];
        for (int k = 0; k < 3; ++k) dmu[k] += (du[k] - u[k] * udu) / f.dlen;
        /* ---- conic -> Sigma_2D (cxx, cxy, cyy; the +0.3 has unit derivative) */
        double d2 = f.det * f.det;
        double ga = g[G_A], gb = g[G_B], gcn = g[G_C];
        double gxx = ga * (-f.cyy * f.cyy / d2) + gb * (f.cxy * f.cyy / d2) + gcn * (1.0 / f.det - f.cxx * f.cyy / d2);
        double gyy = ga * (1.0 / f.det - f.cyy * f.cxx / d2) + gb * (f.cxy * f.cxx / d2) + gcn * (-f.cxx * f.cxx / d2);
        double gxy = ga * (2.0 * f.cyy * f.cxy / d2) + gb * (-1.0 / f.det - 2.0 * f.cxy * f.cxy / d2) +
                     gcn * (2.0 * f.cxx * f.cxy / d2);
        double G[2][2] = {{gxx, 0.5 * gxy}, {0.5 * gxy, gyy}};
        /* ---- Eq. 4: Sigma_2D = T Sigma_3D T^T */
        double dS3[3][3], dT[2][3];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) {
                double acc = 0.0;
                for (int u1 = 0; u1 < 2; ++u1)
                    for (int u2 = 0; u2 < 2; ++u2) acc += f.T[u1][r] * G[u1][u2] * f.T[u2][k];
                dS3[r][k] = acc;
            }
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) {
                double acc = 0.0;
                for (int u2 = 0; u2 < 2; ++u2)
                    for (int m = 0; m < 3; ++m) acc += G[r][u2] * f.T[u2][m] * f.S3[m][k];
                dT[r][k] = 2.0 * acc;
            }
        /* ---- T = J W: dL/dJ = dL/dT W^T (W = rotation part of viewmat) */
        double dJ[2][3];
        for (int r = 0; r < 2; ++r)
            for (int m = 0; m < 3; ++m) dJ[r][m] = dT[r][0] * V[4 * m + 0] + dT[r][1] * V[4 * m + 1] + dT[r][2] * V[4 * m + 2];
        /* ---- J(p) and mu2D(p) -> dL/dp */
        double x = f.p[0], y = f.p[1], z = f.p[2], iz = f.iz, iz2 = iz * iz;
        double dp[3] = {0, 0, 0};
        /* x2d = fx x / z + cx ; y2d = fy y / z + cy */
        dp[0] += g[G_X] * cam->fx * iz;
        dp[2] += g[G_X] * (-cam->fx * x * iz2);
        dp[1] += g[G_Y] * cam->fy * iz;
        dp[2] += g[G_Y] * (-cam->fy * y * iz2);
        /* J00 = fx / z ; J11 = fy / z */
        dp[2] += dJ[0][0] * (-cam->fx * iz2) + dJ[1][1] * (-cam->fy * iz2);
        /* J02 = -fx txc / z: unclamped txc = x/z -> -fx x / z^2; clamped: txc constant */
        if (!f.clx) {
            dp[0] += dJ[0][2] * (-cam->fx * iz2);
            dp[2] += dJ[0][2] * (2.0 * cam->fx * x * iz2 * iz);
        } else {
            dp[2] += dJ[0][2] * (cam->fx * f.txc * iz2);
        }
        if (!f.cly) {
            dp[1] += dJ[1][2] * (-cam->fy * iz2);
            dp[2] += dJ[1][2] * (2.0 * cam->fy * y * iz2 * iz);
        } else {
            dp[2] += dJ[1][2] * (cam->fy * f.tyc * iz2);
        }
        (void)z;
        /* p = W mu + t */
        for (int k = 0; k < 3; ++k) dmu[k] += V[0 + k] * dp[0] + V[4 + k] * dp[1] + V[8 + k] * dp[2];
        /* ---- Eq. 3: Sigma_3D = M M^T, M = R S */
        double dM[3][3];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) {
                double acc = 0.0;
                for (int m = 0; m < 3; ++m) acc += (dS3[r][m] + dS3[m][r]) * f.M[m][k];
                dM[r][k] = acc;
            }
        double ds[3] = {0, 0, 0}, dR[3][3];
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) {
                ds[k] += dM[r][k] * f.R[r][k];
                dR[r][k] = dM[r][k] * f.s[k];
            }
        /* R(w, x, y, z) partials */
        double w = f.qn[0], qx = f.qn[1], qy = f.qn[2], qz = f.qn[3];
        double dqn[4];
        dqn[0] = 2 * (-qz * dR[0][1] + qy * dR[0][2] + qz * dR[1][0] - qx * dR[1][2] - qy * dR[2][0] + qx * dR[2][1]);
        dqn[1] = 2 * (qy * dR[0][1] + qz * dR[0][2] + qy * dR[1][0] - 2 * qx * dR[1][1] - w * dR[1][2] + qz * dR[2][0] +
                      w * dR[2][1] - 2 * qx * dR[2][2]);
        dqn[2] = 2 * (-2 * qy * dR[0][0] + qx * dR[0][1] + w * dR[0][2] + qx * dR[1][0] + qz * dR[1][2] - w * dR[2][0] +
                      qz * dR[2][1] - 2 * qy * dR[2][2]);
        dqn[3] = 2 * (-2 * qz * dR[0][0] - w * dR[0][1] + qx * dR[0][2] + w * dR[1][0] - 2 * qz * dR[1][1] + qy * dR[1][2] +
                      qx * dR[2][0] + qy * dR[2][1]);
        double qd = f.qn[0] * dqn[0] + f.qn[1] * dqn[1] + f.qn[2] * dqn[2] + f.qn[3] * dqn[3];
        for (int k = 0; k < 3; ++k) dmean_opac[4 * (size_t)i + k] += dmu[k];
        dmean_opac[4 * (size_t)i + 3] += g[G_SIGMA];
        for (int k = 0; k < 3; ++k) dscale[4 * (size_t)i + k] += ds[k];
        for (int k = 0; k < 4; ++k) drot[4 * (size_t)i + k] += (dqn[k] - f.qn[k] * qd) / f.qlen;
    }
}

/* ------------------------------------------------------------------------------------
 * NEXT-3 (pruning-in-the-loop training on synthetic targets): the two pieces of Eq. 2's
 * optimisation step that surround the backward.
 *
 * L1 loss (Eq. 2's L_1 term; the D-SSIM term is omitted):
 *   L = (1/K) sum_k |img_k - gt_k|,  dL/dimg_k = sign(img_k - gt_k) / K  (sign(0) = 0),
 * K = number of values (3 H W).  Returns L (float64); writes dL/dimg as float32.
 * ---------------------------------------------------------------------------------- */
double or_l1_loss_grad(int64_t count, const float *img, const float *gt, float *grad)
{
    double L = 0.0;
    for (int64_t k = 0; k < count; ++k) {
        double d = (double)img[k] - (double)gt[k];
        L += fabs(d);
        grad[k] = (float)((d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / (double)count);
    }
    return count ? L / (double)count : 0.0;
}

/* Adam (Kingma & Ba; the optimiser of 3D-GS training, "stochastic gradient descent")
 * on the raw parameters of one array, float64:
 *   g_raw = g * dact/draw      (act: 0 identity, 1 exp (scales), 2 sigmoid (opacity))
 *   m = b1 m + (1 - b1) g_raw;  v = b2 v + (1 - b2) g_raw^2
 *   raw -= lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 *   out = act(raw)             (the activated parameter the forward reads, R24)
 * act and lr are per element (act_of[k], lr_of[k]) so one call covers a whole scene array. */
void or_adam_step(int64_t count, const double *grad_act, double *raw, double *m, double *v, double *out,
                  const int32_t *act_of, const double *lr_of, double b1, double b2, double eps, int32_t t)
{
    double c1 = 1.0 - pow(b1, t), c2 = 1.0 - pow(b2, t);
    for (int64_t k = 0; k < count; ++k) {
        double a;
        if (act_of[k] == 1) a = exp(raw[k]);
        else if (act_of[k] == 2) a = 1.0 / (1.0 + exp(-raw[k]));
        else a = raw[k];
        double d = act_of[k] == 1 ? a : (act_of[k] == 2 ? a * (1.0 - a) : 1.0);
        double g = grad_act[k] * d;
        m[k] = b1 * m[k] + (1.0 - b1) * g;
        v[k] = b2 * v[k] + (1.0 - b2) * g * g;
        raw[k] -= lr_of[k] * (m[k] / c1) / (sqrt(v[k] / c2) + eps);
        if (act_of[k] == 1) out[k] = exp(raw[k]);
        else if (act_of[k] == 2) out[k] = 1.0 / (1.0 + exp(-raw[k]));
        else out[k] = raw[k];
    }
}
