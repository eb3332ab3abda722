// ss_prune.cu -- score-driven prune step: select and compact.
//
// Sec. 4.2: "removing a set percentage with the lowest sensitivities"; Soft Pruning
// (80% before the opacity resets) and Hard Pruning (30% every 3k iterations,
// P:434-436) both apply this step to the accumulated score U~ (Eq. 21).  Removed: exactly
// k = floor(ratio N) Gaussians with the smallest score; on equal scores the higher index goes
// first.  Selection is a 96-bit radix select on key = (score bits, ~index) -- unique keys in
// exactly that order -- entirely on the device (12 histogram passes + a 1-warp pick each);
// compaction is a stable stream compaction (block scan + decoupled look-back) of every SoA
// plane, so survivors keep their relative order.
#include "ss_common.cuh"

namespace ss {
namespace {

struct SelState {
    unsigned long long prefix_hi;  // selected high bits of the score key so far
    uint32_t prefix_lo;            // selected bits of ~index so far
    uint32_t k_rem;                // rank (1-based) still to find within the prefix bucket
    uint32_t k;                    // elements to remove
    uint32_t pad[3];
};

__device__ __forceinline__ uint32_t digit96(unsigned long long hi, uint32_t lo, int d) {
    // d = 0..7: score bits 63..0 (MSB first); d = 8..11: ~index bits 31..0
    return d < 8 ? (uint32_t)(hi >> (56 - 8 * d)) & 0xFFu : (lo >> (24 - 8 * (d - 8))) & 0xFFu;
}

__device__ __forceinline__ bool prefix_match(unsigned long long hi, uint32_t lo, int d, const SelState &s) {
    // the key's digits above digit d equal the selected prefix
    if (d == 0) return true;
    if (d <= 8) {
        const int sh = 64 - 8 * d;
        return (hi >> sh) == (s.prefix_hi >> sh);
    }
    if (hi != s.prefix_hi) return false;
    const int sh = 32 - 8 * (d - 8);
    return (lo >> sh) == (s.prefix_lo >> sh);
}

__global__ void k_sel_init(SelState *st, uint32_t *hist, int n, double ratio) {
    if (threadIdx.x == 0) {
        double kd = floor(ratio * (double)n);
        if (kd < 0.0) kd = 0.0;
        if (kd > (double)n) kd = (double)n;
        st->prefix_hi = 0ull;
        st->prefix_lo = 0u;
        st->k = (uint32_t)kd;
        st->k_rem = (uint32_t)kd;
    }
    hist[threadIdx.x] = 0u;
}

__global__ void __launch_bounds__(256) k_sel_hist(const double *__restrict__ score, int n, int d,
                                                  const SelState *__restrict__ st, uint32_t *__restrict__ hist) {
    __shared__ uint32_t s_h[256];
    s_h[threadIdx.x] = 0;
    __syncthreads();
    const SelState s = *st;
    if (s.k_rem > 0) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const unsigned long long hi = (unsigned long long)__double_as_longlong(score[i]);
            const uint32_t lo = ~(uint32_t)i;
            if (prefix_match(hi, lo, d, s)) atomicAdd(&s_h[digit96(hi, lo, d)], 1u);
        }
    }
    __syncthreads();
    if (s_h[threadIdx.x]) atomicAdd(hist + threadIdx.x, s_h[threadIdx.x]);
}

// One warp: the bucket holding the k_rem-th key; extend the prefix; clear the histogram.
__global__ void k_sel_pick(SelState *st, uint32_t *hist, int d) {
    const int lane = threadIdx.x;
    SelState s = *st;
    if (s.k_rem > 0) {
        uint32_t c[8], sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            c[q] = hist[lane * 8 + q];
            sum += c[q];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - sum;
        int bucket = -1;
        uint32_t before = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (bucket < 0 && run + c[q] >= s.k_rem && run < s.k_rem) {
                bucket = lane * 8 + q;
                before = run;
            }
            run += c[q];
        }
        const uint32_t has = __ballot_sync(0xffffffffu, bucket >= 0);
        const int src = __ffs(has) - 1;
        bucket = __shfl_sync(0xffffffffu, bucket, src);
        before = __shfl_sync(0xffffffffu, before, src);
        if (lane == 0) {
            if (d < 8)
                s.prefix_hi |= (unsigned long long)bucket << (56 - 8 * d);
            else
                s.prefix_lo |= (uint32_t)bucket << (24 - 8 * (d - 8));
            s.k_rem -= before;
            *st = s;
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) hist[lane * 8 + q] = 0u;
}

// keep[i] = key(i) > T (the k-th smallest key), i.e. the k smallest keys are removed.
__global__ void __launch_bounds__(256) k_sel_mark(const double *__restrict__ score, int n,
                                                  const SelState *__restrict__ st, uint8_t *__restrict__ keep) {
    const SelState s = *st;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long hi = (unsigned long long)__double_as_longlong(score[i]);
        const uint32_t lo = ~(uint32_t)i;
        const bool removed = s.k > 0 && (hi < s.prefix_hi || (hi == s.prefix_hi && lo <= s.prefix_lo));
        keep[i] = removed ? 0 : 1;
    }
}

// Stable compaction of the SoA planes: CTA tickets, block scan of the keep flags, single-word
// decoupled look-back for the CTA's output offset, then every plane's survivors are copied.
__global__ void __launch_bounds__(256) k_compact(int n, const uint8_t *__restrict__ keep, int n_planes_sh,
                                                 const float4 *__restrict__ mo_in, const float4 *__restrict__ sc_in,
                                                 const float4 *__restrict__ rot_in, const float4 *__restrict__ sh_in,
                                                 float4 *__restrict__ mo_out, float4 *__restrict__ sc_out,
                                                 float4 *__restrict__ rot_out, float4 *__restrict__ sh_out,
                                                 uint32_t out_stride, uint32_t *lookback, uint32_t *ticket,
                                                 uint32_t *n_out) {
    __shared__ uint32_t s_warp[8];
    __shared__ uint32_t s_bid, s_base;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t bid = s_bid;
        if ((size_t)bid * 256 >= (size_t)n) break;
        const uint32_t i = bid * 256 + threadIdx.x;
        const uint32_t f = (i < (uint32_t)n && keep[i]) ? 1u : 0u;
        uint32_t total;
        const uint32_t excl = block_exclusive_scan_256(f, s_warp, total);
        if (threadIdx.x == 0) {
            volatile uint32_t *lb = lookback;
            uint32_t acc = 0;
            if (bid == 0) {
                lb[0] = kFlagInc | total;
            } else {
                lb[bid] = kFlagAgg | total;
                int p = (int)bid - 1;
                for (;;) {
                    uint32_t v;
                    do { v = lb[p]; } while ((v & ~kValMask) == 0);
                    acc += v & kValMask;
                    if ((v & ~kValMask) == kFlagInc) break;
                    --p;
                }
                lb[bid] = kFlagInc | (acc + total);
            }
            s_base = acc;
            if ((size_t)(bid + 1) * 256 >= (size_t)n) *n_out = acc + total;
        }
        __syncthreads();
        // survivors beyond the caller's out->n (a mask keeping more than the allocation) are
        // counted in *n_out but not written
        if (f && s_base + excl < out_stride) {
            const uint32_t o = s_base + excl;
            mo_out[o] = mo_in[i];
            sc_out[o] = sc_in[i];
            rot_out[o] = rot_in[i];
            for (int p = 0; p < n_planes_sh; ++p)  // per-Gaussian SH block (AoS)
                sh_out[(size_t)o * n_planes_sh + p] = sh_in[(size_t)i * n_planes_sh + p];
        }
    }
}

int grid_for(int n) {
    const int sms = sm_count();
    const int need = (n + 255) / 256;
    return need < sms * 4 ? (need > 0 ? need : 1) : sms * 4;
}

}  // namespace

size_t prune_workspace_bytes(int32_t n) {
    const size_t nblk = ((size_t)n + 255) / 256;
    return 256 + 256 * 4 + 64 + 4 * nblk + 256;
}

cudaError_t launch_prune_select(const double *score, int32_t n, double ratio, uint8_t *keep, void *ws,
                                cudaStream_t st) {
    SelState *state = at<SelState>(ws, 0);
    uint32_t *hist = at<uint32_t>(ws, 256);
    k_sel_init<<<1, 256, 0, st>>>(state, hist, n, ratio);
    if (n > 0) {
        const int grid = grid_for(n);
        for (int d = 0; d < 12; ++d) {
            k_sel_hist<<<grid, 256, 0, st>>>(score, n, d, state, hist);
            k_sel_pick<<<1, 32, 0, st>>>(state, hist, d);
        }
        k_sel_mark<<<grid, 256, 0, st>>>(score, n, state, keep);
    }
    return cudaGetLastError();
}

cudaError_t launch_compact(const ss_scene &in, const uint8_t *keep, const ss_scene &out, uint32_t out_stride,
                           uint32_t *n_out, void *ws, cudaStream_t st) {
    const size_t nblk = ((size_t)in.n + 255) / 256;
    uint32_t *ticket = at<uint32_t>(ws, 256 + 1024);
    uint32_t *lookback = at<uint32_t>(ws, 256 + 1024 + 64);
    cudaError_t e = cudaMemsetAsync(ticket, 0, 64 + 4 * nblk, st);
    if (e != cudaSuccess) return e;
    if (in.n == 0) return cudaMemsetAsync(n_out, 0, 4, st);
    const int planes = ((in.sh_degree + 1) * (in.sh_degree + 1) * 3 + 3) / 4;
    k_compact<<<grid_for(in.n), 256, 0, st>>>(
        in.n, keep, planes, reinterpret_cast<const float4 *>(in.mean_opac), reinterpret_cast<const float4 *>(in.scale),
        reinterpret_cast<const float4 *>(in.rot), reinterpret_cast<const float4 *>(in.sh),
        reinterpret_cast<float4 *>(const_cast<float *>(out.mean_opac)),
        reinterpret_cast<float4 *>(const_cast<float *>(out.scale)),
        reinterpret_cast<float4 *>(const_cast<float *>(out.rot)), reinterpret_cast<float4 *>(const_cast<float *>(out.sh)),
        out_stride, lookback, ticket, n_out);
    return cudaGetLastError();
}

}  // namespace ss
