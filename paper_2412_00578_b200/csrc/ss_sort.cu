// ss_sort.cu -- stable LSD radix sort (onesweep, decoupled look-back) and tile ranges.
//
// The depth order of the visible Gaussians: their 32-bit depth keys, 4 x
// 8-bit passes; pass 0 reads every Gaussian's key (implicit value = index) and drops the
// 0xFFFFFFFF sentinel of Gaussians without tiles (compaction fused into the first pass).
// The last pass also gathers each Gaussian's super-tile entry count into depth order for
// ss_bin.cu, which partitions the depth-ordered pairs by tile (a stable two-level binning;
// stability makes the result equal to the paper's stable sort of (tile << 32 | depth) keys,
// P:174).
#include "ss_common.cuh"

namespace ss {
namespace {

constexpr int kWarps = kSortThreads / 32;
#ifndef SS_SORT_LB
#define SS_SORT_LB 8
#endif
constexpr int kLB = SS_SORT_LB;  // look-back predecessors read per round trip
#ifndef SS_SORT_SLEEP
#define SS_SORT_SLEEP 0
#endif
constexpr int kLBSleepNs = SS_SORT_SLEEP;
#ifndef SS_SORT_GRID
#define SS_SORT_GRID 2  // persistent onesweep CTAs per SM (16 frames in flight: 2 -> 1945 fps, 3 -> 1931, 4 -> 1924)
#endif
#ifndef SS_SORT_MATCH
#define SS_SORT_MATCH 1
#endif  // back-off when no predecessor has published yet

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
    return (uint32_t)(key >> shift) & 0xFFu;
}

// One onesweep pass.  Block tickets (atomicAdd) give every CTA tile an id in launch order,
// so a CTA only waits on ids already owned by running CTAs (forward progress).  Per tile:
//  1. load kSortItems keys / thread, warp-striped (warp w owns 32 kSortItems consecutive keys);
//  2. warp-level stable ranking by 8 ballots per item (match on the digit), per-warp digit
//     histograms in shared memory;
//  3. digit totals -> look-back publication (aggregate, then inclusive prefix);
//  4. scatter into shared memory in tile-sorted order, then write out contiguous digit runs.
template <typename K, bool IMPLICIT_VALS, bool FILTER, bool WRITE_KEYS>
__global__ void __launch_bounds__(kSortThreads, 4) k_onesweep(const K *__restrict__ keys_in,
                                                              const uint32_t *__restrict__ vals_in,
                                                              K *__restrict__ keys_out,
                                                              uint32_t *__restrict__ vals_out, const uint32_t *n_ptr,
                                                              uint32_t n_fixed, int shift,
                                                              const uint32_t *__restrict__ digit_count,
                                                              uint32_t *lookback, uint32_t *ticket,
                                                              const uint32_t *__restrict__ gather_src = nullptr,
                                                              uint32_t *__restrict__ gather_dst = nullptr) {
    pdl_enter();
    __shared__ uint32_t s_whist[kWarps][256];
    __shared__ uint32_t s_digit_base[256];
    __shared__ uint32_t s_dig_out[256];
    __shared__ uint32_t s_blk_start[256];
    __shared__ K s_keys[kSortTile];
    __shared__ uint32_t s_vals[kSortTile];
    __shared__ uint32_t s_scan[8];
    __shared__ uint32_t s_bid;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = n_ptr ? *n_ptr : n_fixed;
    const uint32_t lanemask_lt = (1u << lane) - 1u;
    {
        uint32_t tot;
        const uint32_t c = digit_count[tid];
        s_digit_base[tid] = block_exclusive_scan_256(c, s_scan, tot);
    }
    for (;;) {
        __syncthreads();
        if (tid == 0) s_bid = atomicAdd(ticket, 1u);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s_whist[w][tid] = 0;
        __syncthreads();
        const uint32_t bid = s_bid;
        const size_t base = (size_t)bid * kSortTile;
        if (base >= n) break;

        // 1. keys (values are re-read at scatter time to keep registers low: 4 CTAs / SM)
        uint32_t key[kSortItems];
        uint32_t rank2[kSortItems / 2];  // two 16-bit in-warp ranks per register
        const size_t wbase = base + (size_t)warp * 32 * kSortItems + lane;
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            const size_t idx = wbase + (size_t)j * 32;
            key[j] = idx < n ? (uint32_t)keys_in[idx] : 0xFFFFFFFFu;
        }
        // 2. warp-level stable ranking: the lanes holding the same digit (SS_SORT_MATCH: one
        //    match.any; else 8 ballots on the digit bits), then the warp's running count of that
        //    digit by one shared-memory atomic of the leader lane (fetch-and-add: no dependent
        //    load -> store chain per item); __syncwarp orders item j's atomics before item j+1's,
        //    so item j+1 sees the counts of items <= j (a stable rank).
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            const size_t idx = wbase + (size_t)j * 32;
            const bool valid = idx < n && (!FILTER || key[j] != kNoTiles);
            const uint32_t d = digit_of(key[j], shift);
#if SS_SORT_MATCH
            uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 256u + (uint32_t)lane);
            peers = valid ? peers : 0u;
#else
            uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
            for (int bit = 0; bit < 8; ++bit) {
                const bool v = (d >> bit) & 1u;
                const uint32_t m = __ballot_sync(0xffffffffu, v);
                peers &= v ? m : ~m;
            }
            peers = valid ? peers : 0u;
#endif
            const uint32_t lt = __popc(peers & lanemask_lt);
            const int leader = peers ? __ffs(peers) - 1 : lane;
            uint32_t prev = 0;
            if (valid && lt == 0) prev = atomicAdd(&s_whist[warp][d], (uint32_t)__popc(peers));
            __syncwarp();  // orders item j's atomics before item j+1's (memory ordering within the warp)
            prev = __shfl_sync(0xffffffffu, prev, leader);
            const uint32_t r = valid ? prev + lt : 0xFFFFu;
            if (j & 1) rank2[j >> 1] |= r << 16;
            else rank2[j >> 1] = r;
        }
        __syncthreads();
        // 3. thread tid owns digit tid: exclusive scan across warps, tile total, look-back
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_whist[w][tid];
            s_whist[w][tid] = tot;
            tot += c;
        }
        {
            volatile uint32_t *lb = lookback + (size_t)bid * 256 + tid;
            uint32_t prefix = 0;
            if (bid == 0) {
                *lb = kFlagInc | tot;
            } else {
                *lb = kFlagAgg | tot;
                // walk back kLB predecessors per round trip (independent loads in flight)
                int p = (int)bid - 1;
                for (;;) {
                    uint32_t v[kLB];
#pragma unroll
                    for (int q = 0; q < kLB; ++q)
                        v[q] = p - q >= 0 ? ((const volatile uint32_t *)lookback)[(size_t)(p - q) * 256 + tid]
                                          : kFlagInc;  // before CTA 0: a virtual inclusive 0
                    int used = kLB;
                    bool inc = false;
                    uint32_t add = 0;
#pragma unroll
                    for (int q = 0; q < kLB; ++q) {
                        if (used == kLB) {
                            const uint32_t f = v[q] & ~kValMask;
                            if (f == 0) {
                                used = q;  // not yet published: re-read from here
                            } else {
                                add += v[q] & kValMask;
                                if (f == kFlagInc) {
                                    inc = true;
                                    used = q + 1;
                                }
                            }
                        }
                    }
                    prefix += add;
                    p -= used;
                    if (inc) break;
                    if (kLBSleepNs > 0 && used == 0) __nanosleep(kLBSleepNs);  // free the issue slots
                }
                *lb = kFlagInc | (prefix + tot);
            }
            s_dig_out[tid] = s_digit_base[tid] + prefix;
        }
        uint32_t tile_total;
        s_blk_start[tid] = block_exclusive_scan_256(tot, s_scan, tile_total);
        __syncthreads();
        // 4. scatter into shared memory in tile-sorted order (values loaded now, coalesced)
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            const uint32_t r = (rank2[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
            if (r != 0xFFFFu) {
                const size_t idx = wbase + (size_t)j * 32;
                const uint32_t d = digit_of(key[j], shift);
                const uint32_t pos = s_blk_start[d] + s_whist[warp][d] + r;
                s_keys[pos] = (K)key[j];
                s_vals[pos] = IMPLICIT_VALS ? (uint32_t)idx : __ldg(vals_in + idx);
            }
        }
        __syncthreads();
        // 5. write out contiguous digit runs
        for (uint32_t i = tid; i < tile_total; i += kSortThreads) {
            const K k = s_keys[i];
            const uint32_t d = digit_of(k, shift);
            const uint32_t o = s_dig_out[d] + (i - s_blk_start[d]);
            if (WRITE_KEYS) keys_out[o] = k;
            vals_out[o] = s_vals[i];
            if (gather_dst) gather_dst[o] = gather_src[s_vals[i]];  // per-Gaussian value, depth order
        }
    }
}

// The paper's sorted key array, materialised for inspection: keys[j] = tile << 32 | depth.
__global__ void k_sorted_keys(const uint2 *__restrict__ ranges, const uint32_t *__restrict__ sorted_value,
                              const uint32_t *__restrict__ depth_key, uint64_t *__restrict__ keys) {
    const int tile = blockIdx.x;
    const uint2 r = ranges[tile];
    for (uint32_t j = r.x + threadIdx.x; j < r.y; j += blockDim.x) {
        const uint32_t g = sorted_value[j];
        keys[j] = ((uint64_t)tile << 32) | depth_key[g];
    }
}

int sort_grid(uint32_t nblk) {
    const int sms = sm_count();
    const uint32_t cap = (uint32_t)sms * SS_SORT_GRID;
    return (int)(nblk < cap ? (nblk ? nblk : 1) : cap);
}

}  // namespace

cudaError_t launch_depth_sort(void *ws, const Layout &L, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (L.n == 0) return cudaSuccess;
    const int grid = sort_grid(L.nblk_depth);
    uint32_t *hist = at<uint32_t>(ws, L.hist_depth);
    uint32_t *tick = at<uint32_t>(ws, L.counters);
    uint32_t *lb = at<uint32_t>(ws, L.lb_depth);
    const size_t lbs = (size_t)L.nblk_depth * 256;
    const uint32_t *nvis = at<uint32_t>(ws, P.n_visible);
    uint32_t *kA = at<uint32_t>(ws, L.dkA), *vA = at<uint32_t>(ws, L.dvA);
    uint32_t *kB = at<uint32_t>(ws, L.dkB), *vB = at<uint32_t>(ws, L.dvB);
    launch_pdl(k_onesweep<uint32_t, true, true, true>, grid, kSortThreads, 0, st, 
        at<uint32_t>(ws, P.depth_key), nullptr, kA, vA, nullptr, (uint32_t)L.n, 0, hist, lb, tick + 0, nullptr,
        nullptr);
    launch_pdl(k_onesweep<uint32_t, false, false, true>, grid, kSortThreads, 0, st, kA, vA, kB, vB, nvis, 0, 8, hist + 256,
               lb + lbs, tick + 1, nullptr, nullptr);
    launch_pdl(k_onesweep<uint32_t, false, false, true>, grid, kSortThreads, 0, st, kB, vB, kA, vA, nvis, 0, 16, hist + 512,
               lb + 2 * lbs, tick + 2, nullptr, nullptr);
    launch_pdl(k_onesweep<uint32_t, false, false, false>, grid, kSortThreads, 0, st, 
        kA, vA, nullptr, at<uint32_t>(ws, P.order), nvis, 0, 24, hist + 768, lb + 3 * lbs, tick + 3,
        at<const uint32_t>(ws, L.gne), at<uint32_t>(ws, L.one));
    return cudaGetLastError();
}

cudaError_t launch_sorted_keys(void *ws, const Layout &L, uint64_t *keys, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    k_sorted_keys<<<P.n_tiles, 256, 0, st>>>(at<const uint2>(ws, P.ranges), at<const uint32_t>(ws, P.sorted_value),
                                              at<const uint32_t>(ws, P.depth_key), keys);
    return cudaGetLastError();
}

}  // namespace ss
