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
    float lr_mean, lr_opacity, lr_scale, lr_rot, lr_sh_dc, lr_sh_rest, b1, b2, eps, ic1, ic2;  // 1 / (1 - b^t)
};

// act: 0 identity, 1 exp, 2 sigmoid
__device__ __forceinline__ float act_fwd(int act, float r) {
    return act == 1 ? __expf(r) : (act == 2 ? __fdividef(1.0f, 1.0f + __expf(-r)) : r);
}

__device__ __forceinline__ void adam1(float g_act, float &raw, float &m, float &v, float &out, int act, float lr,
                                      const AdamArgs &A) {
    const float a = act_fwd(act, raw);
    const float g = g_act * (act == 1 ? a : (act == 2 ? a * (1.0f - a) : 1.0f));
    m = A.b1 * m + (1.0f - A.b1) * g;
    v = A.b2 * v + (1.0f - A.b2) * g * g;
    // bias corrections as products with host-side reciprocals, one fast division
    raw -= __fdividef(lr * (m * A.ic1), sqrtf(v * A.ic2) + A.eps);
    out = act_fwd(act, raw);
}

// One thread per float4 of the scene arrays, flat over [mean_opac | scale | rot | sh] (n, n,
// n, n*B float4), so every array is read and written fully coalesced: grad, raw, m, v are
// read, raw, m, v and the activated array written (components a slot does not use -- scale.w,
// SH padding -- keep raw == activated, as ss_adam_init set them).  mean_opac: xyz identity,
// sigma sigmoid; scale: exp; rot: identity; SH: identity, coefficients 0..2 (DC) at lr_sh_dc.
// flags (nullable): a Gaussian whose flag is 0 has zero gradient (its grad entries are not read).
__global__ void __launch_bounds__(256) k_adam(int64_t n, int B, int nb3, ss_scene_grad g, ss_scene_grad raw,
                                              ss_scene_grad m, ss_scene_grad v, ss_scene_grad out, AdamArgs A,
                                              const uint8_t *__restrict__ flags) {
    pdl_enter();
    const int64_t total = n * (3 + B);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        int arr;
        int64_t e;
        if (k < n) { arr = 0; e = k; }
        else if (k < 2 * n) { arr = 1; e = k - n; }
        else if (k < 3 * n) { arr = 2; e = k - 2 * n; }
        else { arr = 3; e = k - 3 * n; }
        auto pick = [arr](const ss_scene_grad &a) {
            return reinterpret_cast<float4 *>(arr == 0 ? a.mean_opac : arr == 1 ? a.scale : arr == 2 ? a.rot : a.sh);
        };
        float4 *const gp = pick(g), *const rp = pick(raw), *const mp = pick(m), *const vp = pick(v),
                     *const op = pick(out);
        // the slot's Gaussian and SH coefficient (32-bit division: n * B < 2^31 is checked by the caller)
        const uint32_t q = arr == 3 ? (uint32_t)e / (uint32_t)B : (uint32_t)e;
        const int64_t gi = q;
        const float4 g4 = (flags && !flags[gi]) ? make_float4(0.f, 0.f, 0.f, 0.f) : gp[e];
        float4 r4 = rp[e];
        float4 m4 = mp[e];
        float4 v4 = vp[e];
        float4 o4;
        const float *gr = (const float *)&g4;
        float *rr = (float *)&r4, *mr = (float *)&m4, *vr = (float *)&v4, *orr = (float *)&o4;
        const int coef0 = arr == 3 ? (int)((uint32_t)e - q * (uint32_t)B) * 4 : 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int act = 0, used = 1;
            float lr;
            if (arr == 0) { act = c == 3 ? 2 : 0; lr = c == 3 ? A.lr_opacity : A.lr_mean; }
            else if (arr == 1) { act = 1; used = c < 3; lr = A.lr_scale; }
            else if (arr == 2) { lr = A.lr_rot; }
            else { used = coef0 + c < nb3; lr = coef0 + c < 3 ? A.lr_sh_dc : A.lr_sh_rest; }
            if (used) adam1(gr[c], rr[c], mr[c], vr[c], orr[c], act, lr, A);
            else orr[c] = rr[c];
        }
        rp[e] = r4;
        mp[e] = m4;
        vp[e] = v4;
        op[e] = o4;
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
                             const uint8_t *flags, cudaStream_t st) {
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
    A.ic1 = (float)(1.0 / (1.0 - std::pow((double)c.beta1, (double)c.step)));
    A.ic2 = (float)(1.0 / (1.0 - std::pow((double)c.beta2, (double)c.step)));
    const int nb3 = (g.sh_degree + 1) * (g.sh_degree + 1) * 3;
    const int B = sh_blocks(g.sh_degree);
    const int64_t total = (int64_t)g.n * (3 + B);
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
    launch_pdl(k_adam, blocks, 256, 0, st, (int64_t)g.n, B, nb3, g, raw, m, v, out, A, flags);
    return cudaGetLastError();
}

}  // namespace ss
