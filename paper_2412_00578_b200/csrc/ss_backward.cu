// ss_backward.cu -- NEXT-2 preprocess backward (libss, sm_100a).
//
// the per-pixel gradients of the render are "aggregated to the 2D mu_2D and Sigma_2D
// parameters, which are then parallelized across Gaussians to compute gradients for mu and
// s".  This is the second half: one thread per Gaussian takes its accumulated 2D gradient
// (grad2d, written by ss_render_backward) and applies the chain rule of the forward of
// ss_preprocess (Eqs. 3-4, 10, the SH colour R13, the J clamp R5; clamped quantities pass
// nothing, reading R27):
//   colour   dL/dh_k,ch = dL/dc_ch Y_k (c_ch unclamped); dL/du via dY/du; u = d/|d|
//   conic    (a, b, c) = (cyy, -cxy, cxx)/det  ->  dL/d(cxx, cxy, cyy)
//   Eq. 4    Sigma_2D = T Sigma_3D T^T, T = J W: dL/dSigma_3D = T^T G T, dL/dT = 2 G T Sigma_3D
//   J, mean  J00 = fx/z, J02 = -fx txc/z, ...; x2d = fx x/z + cx; dL/dmu = W^T dL/dp
//   Eq. 3    Sigma_3D = M M^T, M = R S: dL/dM = 2 dL/dSigma_3D M; dL/ds, dL/dR -> dL/dq
// Gradients are ACCUMULATED (+=) into arrays laid out like the scene (a thread owns its
// Gaussian's entries, so no atomics).  Gaussians whose 2D gradient is zero (culled, or not
// blended anywhere in the view) read nothing else.
#include "ss_common.cuh"

namespace ss {
namespace {

template <int DEG>
__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, float *Y, float *dX, float *dY, float *dZ) {
#pragma unroll
    for (int k = 0; k < 16; ++k) Y[k] = dX[k] = dY[k] = dZ[k] = 0.0f;
    Y[0] = 0.28209479177387814f;
    if (DEG < 1) return;
    const float C1 = 0.4886025119029199f;
    Y[1] = -C1 * y; dY[1] = -C1;
    Y[2] = C1 * z;  dZ[2] = C1;
    Y[3] = -C1 * x; dX[3] = -C1;
    if (DEG < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    const float A = 1.0925484305920792f, B = 0.31539156525252005f, D = 0.5462742152960396f;
    Y[4] = A * x * y;               dX[4] = A * y;          dY[4] = A * x;
    Y[5] = -A * y * z;              dY[5] = -A * z;         dZ[5] = -A * y;
    Y[6] = B * (2.f * zz - xx - yy); dX[6] = -2.f * B * x;  dY[6] = -2.f * B * y;  dZ[6] = 4.f * B * z;
    Y[7] = -A * x * z;              dX[7] = -A * z;         dZ[7] = -A * x;
    Y[8] = D * (xx - yy);           dX[8] = 2.f * D * x;    dY[8] = -2.f * D * y;
    if (DEG < 3) return;
    const float E0 = -0.5900435899266435f, E1 = 2.890611442640554f, E2 = -0.4570457994644658f,
                E3 = 0.3731763325901154f, E5 = 1.445305721320277f;
    Y[9] = E0 * y * (3.f * xx - yy);          dX[9] = E0 * 6.f * x * y;        dY[9] = E0 * 3.f * (xx - yy);
    Y[10] = E1 * x * y * z;                   dX[10] = E1 * y * z;  dY[10] = E1 * x * z;  dZ[10] = E1 * x * y;
    Y[11] = E2 * y * (4.f * zz - xx - yy);    dX[11] = -2.f * E2 * x * y;
    dY[11] = E2 * (4.f * zz - xx - 3.f * yy); dZ[11] = 8.f * E2 * y * z;
    Y[12] = E3 * z * (2.f * zz - 3.f * xx - 3.f * yy);
    dX[12] = -6.f * E3 * x * z;  dY[12] = -6.f * E3 * y * z;  dZ[12] = E3 * (6.f * zz - 3.f * xx - 3.f * yy);
    Y[13] = E2 * x * (4.f * zz - xx - yy);    dX[13] = E2 * (4.f * zz - 3.f * xx - yy);
    dY[13] = -2.f * E2 * x * y;               dZ[13] = 8.f * E2 * x * z;
    Y[14] = E5 * z * (xx - yy);               dX[14] = 2.f * E5 * x * z;  dY[14] = -2.f * E5 * y * z;  dZ[14] = E5 * (xx - yy);
    Y[15] = E0 * x * (xx - 3.f * yy);         dX[15] = E0 * 3.f * (xx - yy);  dY[15] = -6.f * E0 * x * y;
}

// The chain rule for one Gaussian i with a non-zero 2D gradient (g0, g1, gbl).  ASSIGN: the
// gradients are written (=) instead of accumulated (+=).  Returns whether they were written.
template <int DEG, bool ASSIGN>
__device__ __forceinline__ bool backward_one(int i, float4 g0, float4 g1, float gbl,
                                             const float4 *__restrict__ mean_opac, const float4 *__restrict__ scale,
                                             const float4 *__restrict__ rot, const float4 *__restrict__ sh,
                                             const CamArgs &cam, float4 *__restrict__ d_mean_opac,
                                             float4 *__restrict__ d_scale, float4 *__restrict__ d_rot,
                                             float4 *__restrict__ d_sh) {
    constexpr int NB = (DEG + 1) * (DEG + 1);
    constexpr int NP = (NB * 3 + 3) / 4;
    const float4 mo = mean_opac[i];
    const float4 s4 = scale[i];
    const float4 q4 = rot[i];
    const float *V = cam.V;
    const float px = V[0] * mo.x + V[1] * mo.y + V[2] * mo.z + V[3];
    const float py = V[4] * mo.x + V[5] * mo.y + V[6] * mo.z + V[7];
    const float pz = V[8] * mo.x + V[9] * mo.y + V[10] * mo.z + V[11];
    if (!(pz >= cam.z_near)) return false;
    const float iz = 1.0f / pz, iz2 = iz * iz;
    const float tx = px * iz, ty = py * iz;
    float txc = tx, tyc = ty;
    bool clx = false, cly = false;
    if (cam.clip > 0.0f) {
        const float limx = cam.clip * ((0.5f * (float)cam.W) / cam.fx);
        const float limy = cam.clip * ((0.5f * (float)cam.H) / cam.fy);
        txc = fminf(limx, fmaxf(-limx, tx));
        tyc = fminf(limy, fmaxf(-limy, ty));
        clx = txc != tx;
        cly = tyc != ty;
    }
    const float j00 = cam.fx * iz, j02 = -(cam.fx * txc) * iz;
    const float j11 = cam.fy * iz, j12 = -(cam.fy * tyc) * iz;
    // rotation of the normalised quaternion
    const float qlen = sqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
    const float qi = 1.0f / qlen;
    const float w = q4.x * qi, x = q4.y * qi, y = q4.z * qi, z = q4.w * qi;
    const float R[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y)},
                           {2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x)},
                           {2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)}};
    const float s3[3] = {s4.x, s4.y, s4.z};
    float M[3][3], S[3][3], T[2][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) M[r][k] = R[r][k] * s3[k];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) S[r][k] = M[r][0] * M[k][0] + M[r][1] * M[k][1] + M[r][2] * M[k][2];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T[0][k] = j00 * V[0 + k] + j02 * V[8 + k];
        T[1][k] = j11 * V[4 + k] + j12 * V[8 + k];
    }
    float TS[2][3];  // T Sigma_3D
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) TS[r][k] = T[r][0] * S[0][k] + T[r][1] * S[1][k] + T[r][2] * S[2][k];
    const float cxx = TS[0][0] * T[0][0] + TS[0][1] * T[0][1] + TS[0][2] * T[0][2] + 0.3f;
    const float cxy = TS[0][0] * T[1][0] + TS[0][1] * T[1][1] + TS[0][2] * T[1][2];
    const float cyy = TS[1][0] * T[1][0] + TS[1][1] * T[1][1] + TS[1][2] * T[1][2] + 0.3f;
    const float det = cxx * cyy - cxy * cxy;
    if (!(det > 0.0f)) return false;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 dmo = ASSIGN ? z4 : d_mean_opac[i];
    float dmu[3] = {0.f, 0.f, 0.f};
    // ---- colour (R13): clamped channels pass nothing
    {
        const float dx = mo.x - cam.cpx, dy = mo.y - cam.cpy, dz = mo.z - cam.cpz;
        const float len = sqrtf(dx * dx + dy * dy + dz * dz);
        const float il = 1.0f / len;
        const float u0 = dx * il, u1 = dy * il, u2 = dz * il;
        float Y[16], dYx[16], dYy[16], dYz[16];
        sh_basis_grad<DEG>(u0, u1, u2, Y, dYx, dYy, dYz);
        float h[NP * 4], dh[NP * 4];
        const float4 *shi = sh + (size_t)i * NP;
        float4 *dshi = d_sh + (size_t)i * NP;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float4 v = shi[p];
            const float4 d = ASSIGN ? z4 : dshi[p];
            h[4 * p + 0] = v.x; h[4 * p + 1] = v.y; h[4 * p + 2] = v.z; h[4 * p + 3] = v.w;
            dh[4 * p + 0] = d.x; dh[4 * p + 1] = d.y; dh[4 * p + 2] = d.z; dh[4 * p + 3] = d.w;
        }
        const float gc[3] = {g1.z, g1.w, gbl};
        float du0 = 0.f, du1 = 0.f, du2 = 0.f;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            float raw = 0.5f;
#pragma unroll
            for (int k = 0; k < NB; ++k) raw += Y[k] * h[k * 3 + ch];
            if (!(raw > 0.0f)) continue;
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                dh[k * 3 + ch] += gc[ch] * Y[k];
                const float gh = gc[ch] * h[k * 3 + ch];
                du0 += gh * dYx[k];
                du1 += gh * dYy[k];
                du2 += gh * dYz[k];
            }
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) dshi[p] = make_float4(dh[4 * p + 0], dh[4 * p + 1], dh[4 * p + 2], dh[4 * p + 3]);
        const float udu = u0 * du0 + u1 * du1 + u2 * du2;
        dmu[0] += (du0 - u0 * udu) * il;
        dmu[1] += (du1 - u1 * udu) * il;
        dmu[2] += (du2 - u2 * udu) * il;
    }
    // ---- conic -> Sigma_2D
    const float id = 1.0f / det, id2 = id * id;
    const float ga = g0.z, gb = g0.w, gcn = g1.x;
    const float gxx = ga * (-cyy * cyy * id2) + gb * (cxy * cyy * id2) + gcn * (id - cxx * cyy * id2);
    const float gyy = ga * (id - cyy * cxx * id2) + gb * (cxy * cxx * id2) + gcn * (-cxx * cxx * id2);
    const float gxy = ga * (2.f * cyy * cxy * id2) + gb * (-id - 2.f * cxy * cxy * id2) + gcn * (2.f * cxx * cxy * id2);
    const float G[2][2] = {{gxx, 0.5f * gxy}, {0.5f * gxy, gyy}};
    // ---- Eq. 4: dL/dSigma_3D = T^T G T (symmetric), dL/dT = 2 G T Sigma_3D
    float GT[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) GT[r][k] = G[r][0] * T[0][k] + G[r][1] * T[1][k];
    float dS[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) dS[r][k] = T[0][r] * GT[0][k] + T[1][r] * GT[1][k];
    float dT[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) dT[r][k] = 2.f * (G[r][0] * TS[0][k] + G[r][1] * TS[1][k]);
    // ---- T = J W: only J00, J02, J11, J12 are non-zero
    const float dj00 = dT[0][0] * V[0] + dT[0][1] * V[1] + dT[0][2] * V[2];
    const float dj02 = dT[0][0] * V[8] + dT[0][1] * V[9] + dT[0][2] * V[10];
    const float dj11 = dT[1][0] * V[4] + dT[1][1] * V[5] + dT[1][2] * V[6];
    const float dj12 = dT[1][0] * V[8] + dT[1][1] * V[9] + dT[1][2] * V[10];
    float dpx = g0.x * cam.fx * iz, dpy = g0.y * cam.fy * iz;
    float dpz = -(g0.x * cam.fx * px + g0.y * cam.fy * py) * iz2 - (dj00 * cam.fx + dj11 * cam.fy) * iz2;
    if (!clx) {
        dpx += -dj02 * cam.fx * iz2;
        dpz += 2.f * dj02 * cam.fx * px * iz2 * iz;
    } else {
        dpz += dj02 * cam.fx * txc * iz2;
    }
    if (!cly) {
        dpy += -dj12 * cam.fy * iz2;
        dpz += 2.f * dj12 * cam.fy * py * iz2 * iz;
    } else {
        dpz += dj12 * cam.fy * tyc * iz2;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) dmu[k] += V[0 + k] * dpx + V[4 + k] * dpy + V[8 + k] * dpz;
    dmo.x += dmu[0];
    dmo.y += dmu[1];
    dmo.z += dmu[2];
    dmo.w += g1.y;  // opacity: alpha = sigma G (t only selects tiles)
    d_mean_opac[i] = dmo;
    // ---- Eq. 3: dL/dM = (dS + dS^T) M = 2 dS M (dS symmetric)
    float dR[3][3], ds[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float dM = 2.f * (dS[r][0] * M[0][k] + dS[r][1] * M[1][k] + dS[r][2] * M[2][k]);
            ds[k] += dM * R[r][k];
            dR[r][k] = dM * s3[k];
        }
    float4 dsc = ASSIGN ? z4 : d_scale[i];
    dsc.x += ds[0];
    dsc.y += ds[1];
    dsc.z += ds[2];
    d_scale[i] = dsc;
    float dq[4];
    dq[0] = 2.f * (-z * dR[0][1] + y * dR[0][2] + z * dR[1][0] - x * dR[1][2] - y * dR[2][0] + x * dR[2][1]);
    dq[1] = 2.f * (y * dR[0][1] + z * dR[0][2] + y * dR[1][0] - 2.f * x * dR[1][1] - w * dR[1][2] + z * dR[2][0] +
                   w * dR[2][1] - 2.f * x * dR[2][2]);
    dq[2] = 2.f * (-2.f * y * dR[0][0] + x * dR[0][1] + w * dR[0][2] + x * dR[1][0] + z * dR[1][2] - w * dR[2][0] +
                   z * dR[2][1] - 2.f * y * dR[2][2]);
    dq[3] = 2.f * (-2.f * z * dR[0][0] - w * dR[0][1] + x * dR[0][2] + w * dR[1][0] - 2.f * z * dR[1][1] +
                   y * dR[1][2] + x * dR[2][0] + y * dR[2][1]);
    const float qd = w * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
    float4 drt = ASSIGN ? z4 : d_rot[i];
    drt.x += (dq[0] - w * qd) * qi;
    drt.y += (dq[1] - x * qd) * qi;
    drt.z += (dq[2] - y * qd) * qi;
    drt.w += (dq[3] - z * qd) * qi;
    d_rot[i] = drt;
    return true;
}

constexpr int kBwdChunk = 4096;  // Gaussians scanned per CTA and round

// Only the Gaussians blended somewhere in the view have a non-zero 2D gradient (≈ 45 k of 3 M
// at MNR360-3M: the rest sit behind saturated pixels), so each CTA first scans a chunk of
// grad2d rows (coalesced, 48 B per Gaussian), compacts the non-zero ones into a shared-memory
// list (warp ballots, one shared atomic per warp), then runs the chain rule with one thread per
// listed Gaussian -- full warps instead of one busy lane per warp.
template <int DEG, bool ASSIGN>
__global__ void __launch_bounds__(256, 2) k_preprocess_backward(int n, const float4 *__restrict__ mean_opac,
                                                             const float4 *__restrict__ scale,
                                                             const float4 *__restrict__ rot,
                                                             const float4 *__restrict__ sh, CamArgs cam,
                                                             const float4 *__restrict__ grad2d,
                                                             float4 *__restrict__ d_mean_opac,
                                                             float4 *__restrict__ d_scale, float4 *__restrict__ d_rot,
                                                             float4 *__restrict__ d_sh,
                                                             uint8_t *__restrict__ flags) {
    pdl_enter();
    __shared__ uint32_t s_list[kBwdChunk];
    __shared__ uint32_t s_cnt;
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * kBwdChunk; base < n; base += (int64_t)gridDim.x * kBwdChunk) {
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        for (int r = 0; r < kBwdChunk / 256; ++r) {
            const int64_t i = base + r * 256 + threadIdx.x;
            bool nz = false;
            if (i < n) {
                const float4 g0 = grad2d[3 * i + 0];
                const float4 g1 = grad2d[3 * i + 1];
                const float gbl = grad2d[3 * i + 2].x;
                nz = g0.x != 0.f || g0.y != 0.f || g0.z != 0.f || g0.w != 0.f || g1.x != 0.f || g1.y != 0.f ||
                     g1.z != 0.f || g1.w != 0.f || gbl != 0.f;
            }
            const uint32_t m = __ballot_sync(0xffffffffu, nz);
            uint32_t pos = 0;
            if (lane == 0 && m) pos = atomicAdd(&s_cnt, (uint32_t)__popc(m));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (nz) s_list[pos + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
        }
        __syncthreads();
        const uint32_t cnt = s_cnt;
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
            const int i = (int)s_list[j];
            const bool w = backward_one<DEG, ASSIGN>(i, grad2d[3 * (size_t)i + 0], grad2d[3 * (size_t)i + 1],
                                                     grad2d[3 * (size_t)i + 2].x, mean_opac, scale, rot, sh, cam,
                                                     d_mean_opac, d_scale, d_rot, d_sh);
            if (flags && w) flags[i] = 1;
        }
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_preprocess_backward(const ss_scene &sc, const CamArgs &cam, const float *grad2d,
                                       const ss_scene_grad &out, uint8_t *flags, cudaStream_t st) {
    if (sc.n == 0) return cudaSuccess;
    const int blocks = (int)std::min<int64_t>(((int64_t)sc.n + kBwdChunk - 1) / kBwdChunk, (int64_t)sm_count() * 4);
    auto mo = reinterpret_cast<const float4 *>(sc.mean_opac);
    auto s4 = reinterpret_cast<const float4 *>(sc.scale);
    auto r4 = reinterpret_cast<const float4 *>(sc.rot);
    auto sh = reinterpret_cast<const float4 *>(sc.sh);
    auto g = reinterpret_cast<const float4 *>(grad2d);
    auto dmo = reinterpret_cast<float4 *>(out.mean_opac);
    auto ds = reinterpret_cast<float4 *>(out.scale);
    auto dr = reinterpret_cast<float4 *>(out.rot);
    auto dsh = reinterpret_cast<float4 *>(out.sh);
#define SS_BWD(D)                                                                                              \
    (flags ? launch_pdl(k_preprocess_backward<D, true>, blocks, 256, 0, st, sc.n, mo, s4, r4, sh, cam, g, dmo, ds, \
                        dr, dsh, flags)                                                                        \
           : launch_pdl(k_preprocess_backward<D, false>, blocks, 256, 0, st, sc.n, mo, s4, r4, sh, cam, g, dmo,   \
                        ds, dr, dsh, (uint8_t *)nullptr))
    switch (sc.sh_degree) {
        case 0: SS_BWD(0); break;
        case 1: SS_BWD(1); break;
        case 2: SS_BWD(2); break;
        default: SS_BWD(3); break;
    }
#undef SS_BWD
    return cudaGetLastError();
}

}  // namespace ss
