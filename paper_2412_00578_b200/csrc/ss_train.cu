// ss_train.cu -- NEXT-3 training step pieces around the backward (libss, sm_100a):
// the L1 loss + its gradient (Eq. 2's L_1 term) and a fused Adam step over every
// scene array ("optimized via stochastic gradient descent"; Adam as in 3D-GS).
//
// Adam runs on RAW parameters -- log-scales and logit-opacities, identity for the mean,
// quaternion and SH -- and writes the ACTIVATED parameters the forward reads (R24), so one
// kernel per step moves a Gaussian's grad, raw, m, v and activated arrays once each.
#include "ss_common.cuh"

namespace ss {
namespace {

// L1: grad = sign(img - gt) / count, loss_sum += sum |img - gt| (float64 atomics, one per CTA).
__global__ void __launch_bounds__(256) k_l1_loss_grad(int64_t count, const float *__restrict__ img,
                                                      const float *__restrict__ gt, float *__restrict__ grad,
                                                      float inv_count, double *__restrict__ loss_sum) {
    pdl_enter();
    __shared__ float s_w[8];
    float acc = 0.0f;
    const int64_t n4 = count / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const float4 *i4 = reinterpret_cast<const float4 *>(img);
    const float4 *g4 = reinterpret_cast<const float4 *>(gt);
    float4 *o4 = reinterpret_cast<float4 *>(grad);
    auto sgn = [&](float d) { return d > 0.f ? inv_count : (d < 0.f ? -inv_count : 0.f); };
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += stride) {
        const float4 a = i4[k], b = g4[k];
        const float d0 = a.x - b.x, d1 = a.y - b.y, d2 = a.z - b.z, d3 = a.w - b.w;
        acc += fabsf(d0) + fabsf(d1) + fabsf(d2) + fabsf(d3);
        o4[k] = make_float4(sgn(d0), sgn(d1), sgn(d2), sgn(d3));
    }
    for (int64_t k = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride) {
        const float d = img[k] - gt[k];
        acc += fabsf(d);
        grad[k] = sgn(d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
        atomicAdd(loss_sum, (double)t);
    }
}

struct AdamArgs {
    float lr_mean, lr_opacity, lr_scale, lr_rot, lr_sh_dc, lr_sh_rest, b1, b2, eps, c1, c2;  // c = 1 - b^t
};

// act: 0 identity, 1 exp, 2 sigmoid
__device__ __forceinline__ float act_fwd(int act, float r) {
    return act == 1 ? expf(r) : (act == 2 ? 1.0f / (1.0f + expf(-r)) : r);
}

__device__ __forceinline__ void adam1(float g_act, float &raw, float &m, float &v, float &out, int act, float lr,
                                      const AdamArgs &A) {
    const float a = act_fwd(act, raw);
    const float g = g_act * (act == 1 ? a : (act == 2 ? a * (1.0f - a) : 1.0f));
    m = A.b1 * m + (1.0f - A.b1) * g;
    v = A.b2 * v + (1.0f - A.b2) * g * g;
    raw -= lr * (m / A.c1) / (sqrtf(v / A.c2) + A.eps);
    out = act_fwd(act, raw);
}

__device__ __forceinline__ void adam4(const float4 *__restrict__ g, float4 *__restrict__ raw, float4 *__restrict__ m,
                                      float4 *__restrict__ v, float4 *__restrict__ out, size_t k, const int act[4],
                                      const float lr[4], int n_used, const AdamArgs &A) {
    const float4 g4 = g[k];
    float4 r4 = raw[k], m4 = m[k], v4 = v[k], o4 = out[k];
    float *gr = (float *)&g4, *rr = (float *)&r4, *mr = (float *)&m4, *vr = (float *)&v4, *orr = (float *)&o4;
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (c < n_used) adam1(gr[c], rr[c], mr[c], vr[c], orr[c], act[c], lr[c], A);
    raw[k] = r4;
    m[k] = m4;
    v[k] = v4;
    out[k] = o4;
}

// One thread per Gaussian: mean_opac (xyz identity, sigma sigmoid), scale (exp, w unused),
// rot (identity), SH blocks (identity; DC coefficients 0..2 at lr_sh_dc, the rest at
// lr_sh_rest; padding components untouched).
__global__ void __launch_bounds__(256) k_adam(int n, int nb3, int B, ss_scene_grad g, ss_scene_grad raw, ss_scene_grad m,
                                              ss_scene_grad v, ss_scene_grad out, AdamArgs A) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    {
        const int act[4] = {0, 0, 0, 2};
        const float lr[4] = {A.lr_mean, A.lr_mean, A.lr_mean, A.lr_opacity};
        adam4((const float4 *)g.mean_opac, (float4 *)raw.mean_opac, (float4 *)m.mean_opac, (float4 *)v.mean_opac,
              (float4 *)out.mean_opac, i, act, lr, 4, A);
    }
    {
        const int act[4] = {1, 1, 1, 1};
        const float lr[4] = {A.lr_scale, A.lr_scale, A.lr_scale, A.lr_scale};
        adam4((const float4 *)g.scale, (float4 *)raw.scale, (float4 *)m.scale, (float4 *)v.scale,
              (float4 *)out.scale, i, act, lr, 3, A);
    }
    {
        const int act[4] = {0, 0, 0, 0};
        const float lr[4] = {A.lr_rot, A.lr_rot, A.lr_rot, A.lr_rot};
        adam4((const float4 *)g.rot, (float4 *)raw.rot, (float4 *)m.rot, (float4 *)v.rot, (float4 *)out.rot, i, act,
              lr, 4, A);
    }
    const int act[4] = {0, 0, 0, 0};
    for (int p = 0; p < B; ++p) {
        float lr[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) lr[c] = (4 * p + c) < 3 ? A.lr_sh_dc : A.lr_sh_rest;
        const int used = min(4, nb3 - 4 * p);
        adam4((const float4 *)g.sh, (float4 *)raw.sh, (float4 *)m.sh, (float4 *)v.sh, (float4 *)out.sh,
              (size_t)i * B + p, act, lr, used, A);
    }
}

// raw = act^-1(scene), m = v = 0.
__global__ void __launch_bounds__(256) k_adam_init(int n, int B, ss_scene sc, ss_scene_grad raw, ss_scene_grad m,
                                                   ss_scene_grad v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 mo = ((const float4 *)sc.mean_opac)[i];
    mo.w = logf(mo.w / (1.0f - mo.w));
    ((float4 *)raw.mean_opac)[i] = mo;
    float4 s = ((const float4 *)sc.scale)[i];
    s = make_float4(logf(s.x), logf(s.y), logf(s.z), s.w);
    ((float4 *)raw.scale)[i] = s;
    ((float4 *)raw.rot)[i] = ((const float4 *)sc.rot)[i];
    ((float4 *)m.mean_opac)[i] = z; ((float4 *)v.mean_opac)[i] = z;
    ((float4 *)m.scale)[i] = z;     ((float4 *)v.scale)[i] = z;
    ((float4 *)m.rot)[i] = z;       ((float4 *)v.rot)[i] = z;
    for (int p = 0; p < B; ++p) {
        const size_t k = (size_t)i * B + p;
        ((float4 *)raw.sh)[k] = ((const float4 *)sc.sh)[k];
        ((float4 *)m.sh)[k] = z;
        ((float4 *)v.sh)[k] = z;
    }
}

}  // namespace

cudaError_t launch_l1_loss_grad(int64_t count, const float *img, const float *gt, float *grad, double *loss_sum,
                                cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const int64_t want = (count / 4 + 255) / 256;
    const int blocks = (int)std::min<int64_t>(std::max<int64_t>(want, 1), (int64_t)sm_count() * 8);
    launch_pdl(k_l1_loss_grad, blocks, 256, 0, st, count, img, gt, grad, (float)(1.0 / (double)count), loss_sum);
    return cudaGetLastError();
}

static int sh_blocks(int deg) { return ((deg + 1) * (deg + 1) * 3 + 3) / 4; }

cudaError_t launch_adam_init(const ss_scene &sc, const ss_scene_grad &raw, const ss_scene_grad &m,
                             const ss_scene_grad &v, cudaStream_t st) {
    if (sc.n == 0) return cudaSuccess;
    k_adam_init<<<(sc.n + 255) / 256, 256, 0, st>>>(sc.n, sh_blocks(sc.sh_degree), sc, raw, m, v);
    return cudaGetLastError();
}

cudaError_t launch_adam_step(const ss_scene_grad &g, const ss_scene_grad &raw, const ss_scene_grad &m,
                             const ss_scene_grad &v, const ss_scene_grad &out, const ss_adam_config &c,
                             cudaStream_t st) {
    if (g.n == 0) return cudaSuccess;
    AdamArgs A;
    A.lr_mean = c.lr_mean;
    A.lr_opacity = c.lr_opacity;
    A.lr_scale = c.lr_scale;
    A.lr_rot = c.lr_rot;
    A.lr_sh_dc = c.lr_sh_dc;
    A.lr_sh_rest = c.lr_sh_rest;
    A.b1 = c.beta1;
    A.b2 = c.beta2;
    A.eps = c.eps;
    A.c1 = (float)(1.0 - std::pow((double)c.beta1, (double)c.step));
    A.c2 = (float)(1.0 - std::pow((double)c.beta2, (double)c.step));
    const int nb3 = (g.sh_degree + 1) * (g.sh_degree + 1) * 3;
    launch_pdl(k_adam, (g.n + 255) / 256, 256, 0, st, g.n, nb3, sh_blocks(g.sh_degree), g, raw, m, v, out, A);
    return cudaGetLastError();
}

}  // namespace ss
