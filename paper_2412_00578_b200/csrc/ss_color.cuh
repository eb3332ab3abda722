// ss_color.cuh -- the view-dependent colour of a Gaussian (R13; "view-dependent colour
// c_i, derived from W and h_i"), evaluated lazily: ss_preprocess leaves the colour of every
// record pending (q2 = 0) and the first render-path kernel that gathers the record computes it
// from the SH block and stores q2 = (1, r, g, b).  Only the Gaussians some tile actually
// reaches before its pixels saturate ever read their 192 B of SH (MNR360-3M: a few hundred
// thousand of the 2.07 M with tiles).  Arithmetic contract (R1): every float32 operation is an
// explicitly rounded intrinsic, in the oracle's order (or_project / or_sh_basis), so the
// result is bit-identical whatever the translation unit's contraction flags.
#pragma once
#include "ss_common.cuh"

namespace ss {

struct ColorSrc {
    const float4 *mean_opac;
    const float4 *sh;  // per-Gaussian SH blocks
    float cpx, cpy, cpz;
    int deg;
};

template <int DEG>
__device__ __forceinline__ float3 sh_color_deg(const ColorSrc &cs, uint32_t g) {
    constexpr int NB = (DEG + 1) * (DEG + 1);
    constexpr int NP = (NB * 3 + 3) / 4;
    const float4 mo = __ldg(cs.mean_opac + g);
    const float dx = __fsub_rn(mo.x, cs.cpx), dy = __fsub_rn(mo.y, cs.cpy), dz = __fsub_rn(mo.z, cs.cpz);
    const float len = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz)));
    const float il = __fdiv_rn(1.0f, len);
    const float x = __fmul_rn(dx, il), y = __fmul_rn(dy, il), z = __fmul_rn(dz, il);
    float Y[16];
    Y[0] = 0.28209479177387814f;
    if (DEG >= 1) {
        const float C1 = 0.4886025119029199f;
        Y[1] = __fmul_rn(-C1, y);
        Y[2] = __fmul_rn(C1, z);
        Y[3] = __fmul_rn(-C1, x);
    }
    if (DEG >= 2) {
        const float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), zz = __fmul_rn(z, z);
        const float xy = __fmul_rn(x, y), yz = __fmul_rn(y, z), xz = __fmul_rn(x, z);
        Y[4] = __fmul_rn(1.0925484305920792f, xy);
        Y[5] = __fmul_rn(-1.0925484305920792f, yz);
        Y[6] = __fmul_rn(0.31539156525252005f, __fsub_rn(__fsub_rn(__fmul_rn(2.0f, zz), xx), yy));
        Y[7] = __fmul_rn(-1.0925484305920792f, xz);
        Y[8] = __fmul_rn(0.5462742152960396f, __fsub_rn(xx, yy));
        if (DEG >= 3) {
            Y[9] = __fmul_rn(__fmul_rn(-0.5900435899266435f, y), __fsub_rn(__fmul_rn(3.0f, xx), yy));
            Y[10] = __fmul_rn(__fmul_rn(2.890611442640554f, xy), z);
            Y[11] = __fmul_rn(__fmul_rn(-0.4570457994644658f, y), __fsub_rn(__fsub_rn(__fmul_rn(4.0f, zz), xx), yy));
            Y[12] = __fmul_rn(__fmul_rn(0.3731763325901154f, z),
                              __fsub_rn(__fsub_rn(__fmul_rn(2.0f, zz), __fmul_rn(3.0f, xx)), __fmul_rn(3.0f, yy)));
            Y[13] = __fmul_rn(__fmul_rn(-0.4570457994644658f, x), __fsub_rn(__fsub_rn(__fmul_rn(4.0f, zz), xx), yy));
            Y[14] = __fmul_rn(__fmul_rn(1.445305721320277f, z), __fsub_rn(xx, yy));
            Y[15] = __fmul_rn(__fmul_rn(-0.5900435899266435f, x), __fsub_rn(xx, __fmul_rn(3.0f, yy)));
        }
    }
    // coefficient j = 3 k + ch is component j % 4 of float4 j / 4; the sums run in k order
    float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const float4 v = __ldg(cs.sh + (size_t)g * NP + p);
        const float hv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = 4 * p + c;
            if (j < 3 * NB) acc[j % 3] = __fadd_rn(acc[j % 3], __fmul_rn(Y[j / 3], hv[c]));
        }
    }
    float acc0 = acc[0], acc1 = acc[1], acc2 = acc[2];
    acc0 = __fadd_rn(acc0, 0.5f);
    acc1 = __fadd_rn(acc1, 0.5f);
    acc2 = __fadd_rn(acc2, 0.5f);
    return make_float3(acc0 > 0.0f ? acc0 : 0.0f, acc1 > 0.0f ? acc1 : 0.0f, acc2 > 0.0f ? acc2 : 0.0f);
}

__device__ __forceinline__ float3 sh_color(const ColorSrc &cs, uint32_t g) {
    switch (cs.deg) {
        case 0: return sh_color_deg<0>(cs, g);
        case 1: return sh_color_deg<1>(cs, g);
        case 2: return sh_color_deg<2>(cs, g);
        default: return sh_color_deg<3>(cs, g);
    }
}

// q2 of the record of Gaussian g with its colour: computed and stored on first use.  The flag
// lives in q2.x (0 = pending, written by ss_preprocess; 1 = done).  q2 is read through L2
// (ld.cg) because other CTAs of the same kernel may have written it; concurrent computations of
// one Gaussian write the same 16 B.
__device__ __forceinline__ float4 record_colour(const float4 *rec, uint32_t g, const ColorSrc &cs) {
    float4 *q2p = const_cast<float4 *>(rec) + 3 * (size_t)g + 2;
    float4 q2 = __ldcg(q2p);
    if (q2.x == 0.0f) {
        const float3 c = sh_color(cs, g);
        q2 = make_float4(1.0f, c.x, c.y, c.z);
        __stcg(q2p, q2);
    }
    return q2;
}

}  // namespace ss
