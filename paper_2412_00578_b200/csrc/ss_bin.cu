// ss_bin.cu -- a2-a5 after the depth order: the stable two-level binning of the pairs by tile.
//
// The paper sorts one 64-bit key (tile << 32 | depth) per (tile, Gaussian) pair.
// With the visible Gaussians already in (depth, index) order (ss_sort.cu's depth passes),
// the sorted pair list is a STABLE partition of that sequence's pairs by tile.  It is built
// in two levels, on the super-tile entries of ss_tilegeom.cuh (one entry per 4x4-tile
// super-tile a Gaussian touches, with a 16-bit mask of its tiles there):
//   k_escan_*     InclusiveSum over the Gaussians in depth order, of their entry
//                 counts: every entry gets a global index, so the work of the next steps
//                 is cut into equal-size units of entries (near Gaussians cover hundreds of
//                 super-tiles; chunks of Gaussians would be badly unbalanced).
//   level 1       a stable counting sort of the entries by super-tile: k_l1_count (entries
//                 per chunk and super-tile), k_l1_scan (per super-tile prefix over the
//                 chunks; super-tile offsets), k_l1_emit (each entry written once at its
//                 place).  Ranks come from __match_any_sync against warp-private histograms
//                 in shared memory: no atomics per entry.
//   level 2       per super-tile, its depth-ordered entries are split into its 16 tile
//                 lists with ballots on the mask bits: k_l2_count (pairs per tile; the last
//                 CTA scans the tiles: ranges = identifyTileRanges, P.175), k_l2_write
//                 (every pair written once, at its sorted position: duplicateWithKeys and
//                 RadixSort fused).
// The result is exactly the paper's stable sort of keys emitted in Gaussian-index order:
// tiles in row-major order, each tile's Gaussians in (depth, index) order.
#include "ss_tilegeom.cuh"

namespace ss {

#ifndef SS_ENTRIES_CTAS
#define SS_ENTRIES_CTAS 8
#endif
constexpr int kEntriesCtasPerSm = SS_ENTRIES_CTAS;  // k_entries grid (grid-stride over the visible Gaussians)
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 32;
constexpr int kScanTile = kScanThreads * kScanItems;  // Gaussians per entry-scan tile
constexpr int kL2Threads = 256;
constexpr int kL2PerThread = 8;
constexpr int kL2Block = kL2Threads * kL2PerThread;  // entries per level-2 block
static_assert(kL2Block == kL2BlockEntries, "level-2 block size");

// ---------------------------------------------------------------- entry scan
// Reduce-then-scan over tiles of kScanTile Gaussians (no look-back chain): k_escan_reduce
// sums every tile; k_escan_apply scans its tile on top of the sum of all earlier tiles (each
// CTA adds the few hundred tile sums before it itself).

__device__ __forceinline__ void scan_load(const uint32_t *__restrict__ one, size_t k0, uint32_t nv, uint32_t *v) {
    if (k0 + kScanItems <= nv) {
        const uint4 *src = reinterpret_cast<const uint4 *>(one + k0);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            const uint4 x = src[q];
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < kScanItems; ++q) v[q] = k0 + q < nv ? one[k0 + q] : 0u;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_escan_reduce(const uint32_t *__restrict__ n_visible,
                                                               const uint32_t *__restrict__ one,
                                                               uint32_t *__restrict__ tile_sum) {
    pdl_enter();
    __shared__ uint32_t s_warp[8];
    const uint32_t nv = *n_visible;
    const size_t base = (size_t)blockIdx.x * kScanTile;
    if (base >= nv) return;
    uint32_t v[kScanItems];
    scan_load(one, base + (size_t)threadIdx.x * kScanItems, nv, v);
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) sum += v[q];
    uint32_t total;
    block_exclusive_scan_256(sum, s_warp, total);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// eoff[k] = sum of one[0..k) over the nv visible Gaussians in depth order; total E; the
// overflow flag (P, summed by ss_preprocess, > capacity).
__global__ void __launch_bounds__(kScanThreads) k_escan_apply(const uint32_t *__restrict__ n_visible,
                                                              const uint32_t *__restrict__ one,
                                                              const uint32_t *__restrict__ tile_sum,
                                                              uint32_t *__restrict__ eoff,
                                                              const uint32_t *__restrict__ total_pairs, uint32_t cap,
                                                              uint32_t *__restrict__ total_entries,
                                                              uint32_t *__restrict__ overflow,
                                                              uint32_t *__restrict__ overflow_count) {
    pdl_enter();
    __shared__ uint32_t s_warp[8];
    const uint32_t nv = *n_visible;
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && tid == 0) {
        const bool ovf = *total_pairs > cap;
        *overflow = ovf ? 1u : 0u;
        if (ovf) atomicAdd(overflow_count, 1u);
    }
    const size_t base = (size_t)blockIdx.x * kScanTile;
    if (base >= nv) return;
    // the sum of the earlier tiles
    uint32_t pre = 0;
    for (uint32_t b = tid; b < blockIdx.x; b += kScanThreads) pre += tile_sum[b];
    uint32_t tile_base;
    block_exclusive_scan_256(pre, s_warp, tile_base);
    __syncthreads();
    const size_t k0 = base + (size_t)tid * kScanItems;
    uint32_t v[kScanItems];
    scan_load(one, k0, nv, v);
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) sum += v[q];
    uint32_t total;
    uint32_t run = tile_base + block_exclusive_scan_256(sum, s_warp, total);
    if (tid == 0 && base + kScanTile >= nv) *total_entries = tile_base + total;
    // blocked -> striped through shared memory, so that the stores are coalesced
    __shared__ uint32_t s_out[kScanTile];
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        s_out[tid * kScanItems + ((q + tid) & (kScanItems - 1))] = run;  // rotated: no bank conflicts
        run += v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
        const uint32_t j = (uint32_t)q * kScanThreads + tid;  // item j of the tile
        const uint32_t t = j / kScanItems, r = j % kScanItems;
        if (base + j < nv) eoff[base + j] = s_out[t * kScanItems + ((r + t) & (kScanItems - 1))];
    }
}

// ---------------------------------------------------------------- level 1
// Staged entries (entry order): (Gaussian, super-tile | mask << 16).
__device__ __forceinline__ void put_entry(uint2 *__restrict__ stg, uint32_t e, uint32_t st, uint32_t g,
                                          uint32_t mask) {
    stg[e] = make_uint2(g, st | (mask << 16));
}

// Entries of a Gaussian whose line spans are stored in its emission record (AccuTile, at most
// kLaneRows lines, non-empty lines in increasing order): per band of 4 lines, one entry for
// every super-tile between the band's span extremes, its mask the union of the band's spans
// there (bit (y & 3) * 4 + (x & 3)) -- the entries band_entries emits (ss_tilegeom.cuh), in
// its order, computed directly from the spans.
__device__ __forceinline__ void span_entries(uint2 *__restrict__ stg, uint32_t g, uint32_t eo, uint32_t info,
                                             const uint4 &e0, const uint4 &e1, int stx) {
    const uint32_t v[6] = {e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
    const int ns = (int)(info & 0xFFu);
    const bool cols = (info & kInfoCols) != 0;
    uint32_t e = eo;
    int q = 0;
#pragma unroll 1
    while (q < ns) {
        const int band = (int)(v[q] >> 20);  // line >> 2 (line = bits 18..)
        int lo = (int)(v[q] & 0x1FFu), hi = (int)((v[q] >> 9) & 0x1FFu);
        int q2 = q + 1;
#pragma unroll 1
        for (; q2 < ns && (int)(v[q2] >> 20) == band; ++q2) {
            lo = min(lo, (int)(v[q2] & 0x1FFu));
            hi = max(hi, (int)((v[q2] >> 9) & 0x1FFu));
        }
#pragma unroll 1
        for (int C = lo >> 2; C <= (hi - 1) >> 2; ++C) {
            uint32_t mask = 0;
            const int c4 = 4 * C;
#pragma unroll 1
            for (int s = q; s < q2; ++s) {
                // the span's tiles in columns 4C .. 4C+3 as a nibble, branch-free (0 if disjoint):
                // bits max(lo, 4C) - 4C .. min(hi, 4C + 4) - 4C - 1
                const int a = min(max((int)(v[s] & 0x1FFu) - c4, 0), 4);
                const int b = min(max(c4 + 4 - (int)((v[s] >> 9) & 0x1FFu), 0), 4);
                const uint32_t bits = (0xFu << a) & (0xFu >> b) & 0xFu;
                const int r = (int)(v[s] >> 18) & 3;
                mask |= cols ? (spread4(bits) << r) : (bits << (4 * r));
            }
            put_entry(stg, e++, cols ? (uint32_t)(C * stx + band) : (uint32_t)(band * stx + C), g, mask);
        }
        q = q2;
    }
}

// Entries of a Gaussian with at most kInlineEnt entries: copied from its emission record.
__device__ __forceinline__ void inline_entries(uint2 *__restrict__ stg, uint32_t g, uint32_t eo, uint32_t ne,
                                               const uint4 &e0, const uint4 &e1) {
    const uint32_t v[kInlineEnt] = {e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
#pragma unroll
    for (int q = 0; q < kInlineEnt; ++q)
        if ((uint32_t)q < ne) put_entry(stg, eo + q, v[q] & 0xFFFFu, g, v[q] >> 16);
}

// Entries of a Gaussian with more than kInlineEnt entries, by the whole warp: lane l takes
// bands first + l, first + l + 32, ... (AccuTile: each band's lines re-evaluated by
// sweep_band exactly as the count evaluated them; rects: the rect's rows); a warp scan of
// the bands' entry counts keeps the count's order.  Warp-uniform arguments.
__device__ __noinline__ void big_entries(uint2 *__restrict__ stg, uint32_t g, uint32_t eo, uint32_t info,
                                            uint32_t aux0, uint32_t aux1,
                                            const float4 *__restrict__ rec, int tiles_x, int tiles_y, int stx) {
    const int lane = threadIdx.x & 31;
    const bool accu = (info & kInfoAccuTile) != 0;
    Sweep w;
    int s0, s1;
    uint32_t rect_iv = 0;
    if (accu) {
        const float4 q0 = rec[3 * (size_t)g + 0];
        const float c = rec[3 * (size_t)g + 1].x;
        const double t = __hiloint2double((int)aux1, (int)aux0);
        accutile_setup((double)q0.x, (double)q0.y, (double)q0.z, (double)q0.w, (double)c, t, tiles_x, tiles_y, w);
        s0 = w.s0;
        s1 = w.s1;
    } else {  // packed rect (x0, x1-x0-1, y0, y1-y0-1): rows y0..y1-1, each [x0, x1)
        const int x0 = (int)(aux0 & 0xFF), x1 = x0 + (int)((aux0 >> 8) & 0xFF) + 1;
        s0 = (int)((aux0 >> 16) & 0xFF);
        s1 = s0 + (int)(aux0 >> 24) + 1;
        rect_iv = (uint32_t)x0 | ((uint32_t)x1 << 16);
        w.rows = true;
    }
    const bool cols = !w.rows;
    (void)info;
    const int b_first = s0 >> 2, b_last = (s1 - 1) >> 2;
    uint32_t base = eo;
    for (int bb = b_first; bb <= b_last; bb += 32) {
        const int band = bb + lane;
        uint32_t iv0 = 0, iv1 = 0, iv2 = 0, iv3 = 0;
        if (band <= b_last) {
            if (accu) {
                sweep_band(w, band, iv0, iv1, iv2, iv3);
            } else {
                const int r0 = 4 * band;
                iv0 = (r0 >= s0 && r0 < s1) ? rect_iv : 0u;
                iv1 = (r0 + 1 >= s0 && r0 + 1 < s1) ? rect_iv : 0u;
                iv2 = (r0 + 2 >= s0 && r0 + 2 < s1) ? rect_iv : 0u;
                iv3 = (r0 + 3 >= s0 && r0 + 3 < s1) ? rect_iv : 0u;
            }
        }
        uint32_t cnt = 0;
        if (band <= b_last) band_entries(band, iv0, iv1, iv2, iv3, cols, stx, [&](uint32_t, uint32_t) { ++cnt; });
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t e = base + x - cnt;
        if (band <= b_last)
            band_entries(band, iv0, iv1, iv2, iv3, cols, stx,
                         [&](uint32_t st, uint32_t mask) { put_entry(stg, e++, st, g, mask); });
        base += __shfl_sync(0xffffffffu, x, 31);
    }
}

// Every visible Gaussian's entries, in depth order, written to their global entry slots
// stg[eoff[k] ..] (one thread per Gaussian; Gaussians with more than kInlineEnt entries are
// queued for k_big_entries).  Warp-uniform grid-stride loop.
__global__ void __launch_bounds__(256) k_entries(const uint32_t *__restrict__ n_visible,
                                                 const uint32_t *__restrict__ overflow,
                                                 const uint32_t *__restrict__ eoff, const uint32_t *__restrict__ order,
                                                 const uint4 *__restrict__ erec, const float4 *__restrict__ rec,
                                                 int tiles_x, int tiles_y, int stx, uint2 *__restrict__ stg,
                                                 uint32_t *__restrict__ big_count,
                                                 uint32_t *__restrict__ big_queue) {
    pdl_enter();
    if (*overflow) return;
    const uint32_t nv = *n_visible;
    const int lane = threadIdx.x & 31;
    // the order / offset of the next grid-stride step are loaded one step ahead, and the whole
    // 32 B record (one sector) with one pair of independent loads: one dependent round trip
    // (order -> record) per Gaussian, overlapped with the previous Gaussian's work
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t k0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    uint32_t g_n = 0, eo_n = 0;
    if (k0 + lane < nv) {
        g_n = order[k0 + lane];
        eo_n = eoff[k0 + lane];
    }
    for (; k0 < nv; k0 += stride) {
        const uint32_t k = k0 + lane;
        const bool act = k < nv;
        const uint32_t g = g_n, eo = eo_n;
        uint4 e0 = make_uint4(0u, 0u, 0u, 0u), e1 = e0;
        if (act) {
            const uint4 *er = erec + 2 * (size_t)g;  // 32 B emission record
            e0 = er[0];
            e1 = er[1];
        }
        if (k + stride < nv) {
            g_n = order[k + stride];
            eo_n = eoff[k + stride];
        }
        const bool spn = (e0.y & kInfoSpanInline) != 0, ent = (e0.y & kInfoEntInline) != 0;
        if (act && spn) span_entries(stg, g, eo, e0.y, e0, e1, stx);
        if (act && ent) inline_entries(stg, g, eo, e0.y >> kInfoEntShift, e0, e1);
        // Gaussians with more entries than inline slots (a few hundred, the nearest ones, so
        // clustered at the front of the depth order): queued for k_big_entries, a warp each
        const bool big = act && !spn && !ent;
        const uint32_t bmask = __ballot_sync(0xffffffffu, big);
        if (bmask) {
            uint32_t base = 0;
            if (lane == __ffs(bmask) - 1) base = atomicAdd(big_count, (uint32_t)__popc(bmask));
            base = __shfl_sync(0xffffffffu, base, __ffs(bmask) - 1);
            if (big) big_queue[base + __popc(bmask & ((1u << lane) - 1u))] = k;
        }
    }
}

// The queued Gaussians' entries, one warp per Gaussian (warp-uniform loop).
__global__ void __launch_bounds__(256) k_big_entries(const uint32_t *__restrict__ overflow,
                                                     const uint32_t *__restrict__ big_count,
                                                     const uint32_t *__restrict__ big_queue,
                                                     const uint32_t *__restrict__ eoff,
                                                     const uint32_t *__restrict__ order,
                                                     const uint4 *__restrict__ erec, const float4 *__restrict__ rec,
                                                     int tiles_x, int tiles_y, int stx, uint2 *__restrict__ stg) {
    pdl_enter();
    if (*overflow) return;
    const uint32_t nb = *big_count;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < nb; q += warps) {
        const uint32_t k = big_queue[q];
        const uint32_t g = order[k];
        const uint4 e0 = erec[2 * (size_t)g];
        big_entries(stg, g, eoff[k], e0.y, e0.z, e0.w, rec, tiles_x, tiles_y, stx);
    }
}

__device__ __forceinline__ void unit_bounds(uint32_t c, int w, uint32_t E, uint32_t &b, uint32_t &B0, uint32_t &B1) {
    b = c * kBinWarps + (uint32_t)w;
    B0 = b * (uint32_t)kEntWarp;
    B1 = min(E, B0 + (uint32_t)kEntWarp);
}

// Lanes holding the same key (nbits wide) as this lane, by nbits ballots; 0 for invalid lanes.
template <int NBITS>
__device__ __forceinline__ uint32_t key_peers(uint32_t key, bool valid) {
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int bit = 0; bit < NBITS; ++bit) {
        const bool v = (key >> bit) & 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, v);
        peers &= v ? m : ~m;
    }
    return valid ? peers : 0u;
}

// Entries per (chunk, super-tile) -> M[c][s], from the staged entries.
template <int SBITS>  // super-tile id width (ballots per rank)
__global__ void __launch_bounds__(kBinWarps * 32, 3) k_l1_count(const uint32_t *__restrict__ total_entries,
                                                              const uint32_t *__restrict__ overflow, int n_super,
                                                              const uint2 *__restrict__ stg,
                                                              uint32_t *__restrict__ M) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem_raw);
    const uint32_t E = *total_entries, c = blockIdx.x;
    if (*overflow || c * (uint32_t)kEntChunk >= E) return;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int s = threadIdx.x; s < kBinWarps * n_super; s += blockDim.x) hist[s] = 0;
    uint32_t b, B0, B1;
    unit_bounds(c, w, E, b, B0, B1);
    const uint32_t n = B0 < B1 ? B1 - B0 : 0u;
    constexpr int kPerLane = kEntWarp / 32;
    uint32_t st[kPerLane];
#pragma unroll
    for (int q = 0; q < kPerLane; ++q) {
        const uint32_t i = (uint32_t)q * 32 + lane;
        st[q] = i < n ? (stg[B0 + i].y & 0xFFFFu) : 0u;
    }
    __syncthreads();
    uint32_t *h = hist + (size_t)w * n_super;
    // counts only (no ranks): one shared-memory atomic per entry (the entries of a warp are in
    // depth order, so their super-tiles rarely coincide); ballot-ranked aggregation as in
    // k_l1_emit measured 10 us slower per frame
#pragma unroll
    for (int q = 0; q < kPerLane; ++q)
        if ((uint32_t)q * 32 + lane < n) atomicAdd(&h[st[q]], 1u);
    __syncthreads();
    for (int s = threadIdx.x; s < n_super; s += blockDim.x) {
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < kBinWarps; ++q) sum += hist[(size_t)q * n_super + s];
        M[(size_t)c * n_super + s] = sum;
    }
}

// Per super-tile s (one CTA): exclusive prefix of M[.][s] over the chunks, the total.  The
// last CTA to finish scans the totals into the super-tiles' first entries and cuts every
// super-tile's entries into level-2 blocks of at most kL2Block entries: blocks[i] =
// (super-tile, first entry within it); st_blk0[s] = the first block of super-tile s.
__global__ void __launch_bounds__(256) k_l1_scan(const uint32_t *__restrict__ total_entries,
                                                 const uint32_t *__restrict__ overflow, int n_super,
                                                 uint32_t *__restrict__ M, uint32_t *__restrict__ st_total,
                                                 uint32_t *__restrict__ st_base, uint32_t *__restrict__ st_blk0,
                                                 uint2 *__restrict__ blocks, uint32_t *__restrict__ n_blocks,
                                                 uint32_t *done) {
    pdl_enter();
    __shared__ uint32_t s_warp[8];
    __shared__ bool s_last;
    if (*overflow) return;
    const uint32_t nck = (*total_entries + kEntChunk - 1) / kEntChunk;
    const int s = blockIdx.x, tid = threadIdx.x;
    constexpr int kPer = 8;  // chunks per thread per round, loads issued together
    uint32_t carry = 0;
    for (uint32_t cb = 0; cb < nck; cb += 256 * kPer) {
        uint32_t x[kPer];
        uint32_t local = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const uint32_t c = cb + (uint32_t)tid * kPer + q;
            x[q] = c < nck ? M[(size_t)c * n_super + s] : 0u;
            local += x[q];
        }
        uint32_t total;
        uint32_t run = carry + block_exclusive_scan_256(local, s_warp, total);
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const uint32_t c = cb + (uint32_t)tid * kPer + q;
            if (c < nck) M[(size_t)c * n_super + s] = run;
            run += x[q];
        }
        carry += total;
        __syncthreads();
    }
    if (tid == 0) st_total[s] = carry;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(done, 1u) == (uint32_t)n_super - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int pers = (n_super + 255) / 256;
    const int s0 = min(n_super, tid * pers), s1 = min(n_super, s0 + pers);
    uint32_t le = 0, lb = 0;
    for (int q = s0; q < s1; ++q) {
        const uint32_t t = ((volatile uint32_t *)st_total)[q];
        le += t;
        lb += (t + kL2Block - 1) / kL2Block;
    }
    uint32_t tot_e, tot_b;
    uint32_t re = block_exclusive_scan_256(le, s_warp, tot_e);
    __syncthreads();  // s_warp is reused by the next scan
    uint32_t rb = block_exclusive_scan_256(lb, s_warp, tot_b);
    for (int q = s0; q < s1; ++q) {
        const uint32_t t = ((volatile uint32_t *)st_total)[q];
        st_base[q] = re;
        st_blk0[q] = rb;
        for (uint32_t o = 0; o < t; o += kL2Block) blocks[rb++] = make_uint2((uint32_t)q, o);
        re += t;
    }
    if (tid == 0) *n_blocks = tot_b;
}

// Every entry written once, at st_base[s] + (entries of s in earlier chunks) + (in earlier
// warps of the chunk) + its rank in the warp; the entries come from k_l1_count's staging.
template <int SBITS>
__global__ void __launch_bounds__(kBinWarps * 32, 3) k_l1_emit(const uint32_t *__restrict__ total_entries,
                                                             const uint32_t *__restrict__ overflow, int n_super,
                                                             const uint32_t *__restrict__ M,
                                                             const uint32_t *__restrict__ st_base,
                                                             const uint2 *__restrict__ stg, uint2 *__restrict__ ent) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint2 *stage = reinterpret_cast<uint2 *>(smem_raw);                  // [kEntChunk] by super-tile
    uint32_t *hist = reinterpret_cast<uint32_t *>(stage + kEntChunk);    // [kBinWarps][n_super]
    uint32_t *loff = hist + (size_t)kBinWarps * n_super;                 // [n_super] chunk-local first
    uint32_t *gb = loff + n_super;                                       // [n_super] global first
    __shared__ uint32_t s_warp[8];
    const uint32_t E = *total_entries, c = blockIdx.x;
    if (*overflow || c * (uint32_t)kEntChunk >= E) return;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int s = threadIdx.x; s < kBinWarps * n_super; s += blockDim.x) hist[s] = 0;
    uint32_t b, B0, B1;
    unit_bounds(c, w, E, b, B0, B1);
    const uint32_t n = B0 < B1 ? B1 - B0 : 0u;
    const uint32_t n_cta = min((uint32_t)kEntChunk, E - c * (uint32_t)kEntChunk);
    constexpr int kPerLane = kEntWarp / 32;
    uint2 v[kPerLane];
#pragma unroll
    for (int q = 0; q < kPerLane; ++q) {
        const uint32_t i = (uint32_t)q * 32 + lane;
        v[q] = i < n ? stg[B0 + i] : make_uint2(0u, 0u);
    }
    __syncthreads();
    uint32_t *h = hist + (size_t)w * n_super;
    uint32_t pk[kPerLane];  // peer masks, reused by the ranking pass
#pragma unroll
    for (int q = 0; q < kPerLane; ++q) {
        const bool valid = (uint32_t)q * 32 + lane < n;
        const uint32_t st = valid ? (v[q].y & 0xFFFFu) : 0u;
        pk[q] = key_peers<SBITS>(st, valid);
        if (valid && (pk[q] & lt_mask) == 0) h[st] += __popc(pk[q]);
        __syncwarp();
    }
    __syncthreads();
    // chunk-local layout by super-tile: loff[s] = entries of super-tiles < s in this chunk;
    // warp w's entries of s start at loff[s] + (entries of s in warps < w)
    const int per = (n_super + (int)blockDim.x - 1) / (int)blockDim.x;
    const int s0 = min(n_super, (int)threadIdx.x * per), s1 = min(n_super, s0 + per);
    uint32_t local = 0;
    for (int s = s0; s < s1; ++s) {
        uint32_t tot = 0;
#pragma unroll
        for (int q = 0; q < kBinWarps; ++q) tot += hist[(size_t)q * n_super + s];
        local += tot;
    }
    uint32_t cta_total;
    uint32_t run0 = block_exclusive_scan_256(local, s_warp, cta_total);
    for (int s = s0; s < s1; ++s) {
        loff[s] = run0;
        gb[s] = st_base[s] + M[(size_t)c * n_super + s];
        uint32_t run = run0;
#pragma unroll
        for (int q = 0; q < kBinWarps; ++q) {
            const uint32_t x = hist[(size_t)q * n_super + s];
            hist[(size_t)q * n_super + s] = run;
            run += x;
        }
        run0 = run;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPerLane; ++q) {
        const bool valid = (uint32_t)q * 32 + lane < n;
        const uint32_t st = valid ? (v[q].y & 0xFFFFu) : 0u;
        const uint32_t peers = pk[q];
        uint32_t prev = 0;
        if (valid) {
            prev = h[st];
            stage[prev + __popc(peers & lt_mask)] = v[q];
        }
        __syncwarp();
        if (valid && (peers & lt_mask) == 0) h[st] = prev + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // write-out in chunk-local order: runs of one super-tile land on consecutive positions
    for (uint32_t i = threadIdx.x; i < n_cta; i += blockDim.x) {
        const uint2 e = stage[i];
        const uint32_t s = e.y & 0xFFFFu;
        ent[gb[s] + (i - loff[s])] = make_uint2(e.x, e.y >> 16);
    }
}

// ---------------------------------------------------------------- level 2
__device__ __forceinline__ int tile_of(int s, int bit, int stx, int tiles_x) {
    const int sy = s / stx, sx = s - sy * stx;
    return (sy * kSuper + (bit >> 2)) * tiles_x + sx * kSuper + (bit & 3);
}

__device__ __forceinline__ bool tile_in_grid(int s, int bit, int stx, int tiles_x, int tiles_y) {
    const int sy = s / stx, sx = s - sy * stx;
    return sx * kSuper + (bit & 3) < tiles_x && sy * kSuper + (bit >> 2) < tiles_y;
}

// Loads the block's entries (kL2PerThread per thread, all issued together).
__device__ __forceinline__ uint32_t l2_load(const uint2 *__restrict__ ent, uint32_t e0, uint32_t n, uint2 *v) {
#pragma unroll
    for (int q = 0; q < kL2PerThread; ++q) {
        const uint32_t i = (uint32_t)q * kL2Threads + threadIdx.x;
        v[q] = i < n ? ent[e0 + i] : make_uint2(0u, 0u);
    }
    return n;
}

// 8 mask bits -> bit t at position 4 t (nibble fields).
__device__ __forceinline__ uint32_t spread8_nibbles(uint32_t x) {
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    return (x | (x << 3)) & 0x11111111u;
}

// Pairs per tile in each level-2 block (per-thread nibble counters, 16 warp reductions) ->
// BC[blk][16].
__global__ void __launch_bounds__(kL2Threads) k_l2_count(const uint32_t *__restrict__ overflow, int stx,
                                                         int tiles_x, int tiles_y, int n_super,
                                                         const uint32_t *__restrict__ st_total,
                                                         const uint32_t *__restrict__ st_base,
                                                         const uint32_t *__restrict__ st_blk0,
                                                         const uint2 *__restrict__ blocks,
                                                         const uint32_t *__restrict__ n_blocks,
                                                         const uint2 *__restrict__ ent, uint32_t *__restrict__ BC) {
    pdl_enter();
    __shared__ uint32_t s_cnt[kL2Threads / 32][16];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const bool ovf = *overflow != 0;
    const uint32_t nb = ovf ? 0u : *n_blocks;
    if (blockIdx.x < nb) {  // (every CTA of the grid; the ones past n_blocks have nothing to do)
        const uint2 bl = blocks[blockIdx.x];
        const uint32_t n = min((uint32_t)kL2Block, st_total[bl.x] - bl.y);
        uint2 v[kL2PerThread];
        l2_load(ent, st_base[bl.x] + bl.y, n, v);
        // per-thread counts of the 16 tiles as 4-bit fields (bit t of a mask -> field t; at most
        // kL2PerThread = 8 per field), then one warp reduction per tile
        uint32_t a0 = 0, a1 = 0;  // tiles 0-7, 8-15
#pragma unroll
        for (int q = 0; q < kL2PerThread; ++q) {
            a0 += spread8_nibbles(v[q].y & 0xFFu);
            a1 += spread8_nibbles((v[q].y >> 8) & 0xFFu);
        }
        static_assert(kL2PerThread <= 15, "4-bit per-thread tile counters");
        uint32_t cnt = 0;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const uint32_t c = ((t < 8 ? a0 : a1) >> (4 * (t & 7))) & 0xFu;
            const uint32_t sum = __reduce_add_sync(0xffffffffu, c);
            if (lane == t) cnt = sum;
        }
        if (lane < 16) s_cnt[w][lane] = cnt;
        __syncthreads();
        if (tid < 16) {
            uint32_t sum = 0;
#pragma unroll
            for (int q = 0; q < kL2Threads / 32; ++q) sum += s_cnt[q][tid];
            BC[(size_t)blockIdx.x * 16 + tid] = sum;
        }
    }
}

// Per super-tile and tile (one thread each, spread over the grid), the exclusive prefix over
// the super-tile's level-2 blocks (in BC) and the tile totals; the last CTA to finish scans
// the tiles in row-major order (tile_base, ranges = identifyTileRanges).  Block blk's pairs of
// tile t start at tile_base[t] + BC[blk][t].
__global__ void __launch_bounds__(256) k_l2_scan(const uint32_t *__restrict__ overflow, int stx, int tiles_x,
                                                 int tiles_y, int n_super, const uint32_t *__restrict__ st_total,
                                                 const uint32_t *__restrict__ st_blk0, uint32_t *__restrict__ BC,
                                                 uint32_t *__restrict__ tile_count, uint32_t *__restrict__ tile_base,
                                                 uint2 *__restrict__ ranges, uint32_t *done) {
    pdl_enter();
    __shared__ uint32_t s_warp[8];
    __shared__ bool s_last;
    const int tid = threadIdx.x;
    const bool ovf = *overflow != 0;
    const int j = blockIdx.x * blockDim.x + tid;
    if (j < n_super * 16) {
        const int sidx = j >> 4, bit = j & 15;
        if (tile_in_grid(sidx, bit, stx, tiles_x, tiles_y)) {
            uint32_t tot = 0;
            if (!ovf) {
                const uint32_t nbs = (st_total[sidx] + kL2Block - 1) / kL2Block;
                uint32_t *col = BC + (size_t)st_blk0[sidx] * 16 + bit;
                for (uint32_t q0 = 0; q0 < nbs; q0 += 8) {  // eight independent loads in flight
                    uint32_t x[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) x[q] = q0 + q < nbs ? col[(size_t)(q0 + q) * 16] : 0u;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (q0 + q < nbs) col[(size_t)(q0 + q) * 16] = tot;
                        tot += x[q];
                    }
                }
            }
            tile_count[tile_of(sidx, bit, stx, tiles_x)] = tot;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int T = tiles_x * tiles_y;
    const int per = (T + 255) / 256;
    const int t0 = min(T, tid * per), t1 = min(T, t0 + per);
    uint32_t local = 0;
    for (int t = t0; t < t1; ++t) local += __ldcg(tile_count + t);
    uint32_t P;
    uint32_t run = block_exclusive_scan_256(local, s_warp, P);
    for (int t = t0; t < t1; ++t) {
        const uint32_t c = __ldcg(tile_count + t);
        tile_base[t] = run;
        ranges[t] = c ? make_uint2(run, run + c) : make_uint2(0u, 0u);
        run += c;
    }
}

// Every pair of a level-2 block written once: per chunk of 256 entries, 16 ballots per
// warp, per-tile prefixes over the warps; pair (tile t, entry) -> BC[blk][t] + earlier pairs.
__global__ void __launch_bounds__(kL2Threads) k_l2_write(const uint32_t *__restrict__ overflow, int stx,
                                                         int tiles_x, int tiles_y,
                                                         const uint32_t *__restrict__ st_total,
                                                         const uint32_t *__restrict__ st_base,
                                                         const uint2 *__restrict__ blocks,
                                                         const uint32_t *__restrict__ n_blocks,
                                                         const uint2 *__restrict__ ent,
                                                         const uint32_t *__restrict__ BC,
                                                         const uint32_t *__restrict__ tile_base,
                                                         uint32_t *__restrict__ sorted_value) {
    pdl_enter();
    constexpr int kW = kL2Threads / 32;
    __shared__ uint32_t s_bal[kL2PerThread][kW][16];  // ballots of every (chunk, warp, tile)
    __shared__ uint32_t s_off[kL2PerThread][kW][16];  // first position of every (chunk, warp, tile)
    if (*overflow || blockIdx.x >= *n_blocks) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint2 bl = blocks[blockIdx.x];
    const uint32_t n = min((uint32_t)kL2Block, st_total[bl.x] - bl.y);
    uint2 v[kL2PerThread];
    l2_load(ent, st_base[bl.x] + bl.y, n, v);
    // all ballots of the block first (one barrier), then the per-tile prefixes over (chunk,
    // warp) by 16 threads (one barrier), then every store
#pragma unroll
    for (int q = 0; q < kL2PerThread; ++q) {
        const uint32_t m = v[q].y;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const uint32_t bal = __ballot_sync(0xffffffffu, (m >> t) & 1u);
            if (lane == t) s_bal[q][w][t] = bal;
        }
    }
    __syncthreads();
    if (tid < 16) {
        uint32_t run = tile_in_grid((int)bl.x, tid, stx, tiles_x, tiles_y)
                           ? BC[(size_t)blockIdx.x * 16 + tid] + tile_base[tile_of((int)bl.x, tid, stx, tiles_x)]
                           : 0u;
#pragma unroll
        for (int q = 0; q < kL2PerThread; ++q)
#pragma unroll
            for (int ww = 0; ww < kW; ++ww) {
                s_off[q][ww][tid] = run;
                run += __popc(s_bal[q][ww][tid]);
            }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kL2PerThread; ++q) {
        uint32_t m = v[q].y;
        while (m) {  // the entry's tiles (2.3 on average)
            const int t = __ffs(m) - 1;
            m &= m - 1;
            sorted_value[s_off[q][w][t] + __popc(s_bal[q][w][t] & lt_mask)] = v[q].x;
        }
    }
}

size_t l1_smem_bytes(int n_super) { return (size_t)kBinWarps * n_super * 4; }

template <int SBITS>
cudaError_t launch_level1(void *ws, const Layout &L, size_t smem, const uint32_t *E, uint32_t *ctr, cudaStream_t st) {
    const ss_layout &P = L.pub;
    static int smem_count[64] = {0}, smem_emit[64] = {0};
    const size_t smem_e = (size_t)kEntChunk * 8 + ((size_t)kBinWarps + 2) * L.n_super * 4;
    cudaError_t e = ensure_smem(k_l1_count<SBITS>, smem, smem_count);
    if (e == cudaSuccess) e = ensure_smem(k_l1_emit<SBITS>, smem_e, smem_emit);
    if (e != cudaSuccess) return e;
    launch_pdl(k_l1_count<SBITS>, L.nck_max, kBinWarps * 32, smem, st, E, at<const uint32_t>(ws, P.overflow),
               L.n_super, at<const uint2>(ws, L.stg), at<uint32_t>(ws, L.bin_M));
    launch_pdl(k_l1_scan, L.n_super, 256, 0, st, E, at<const uint32_t>(ws, P.overflow), L.n_super,
               at<uint32_t>(ws, L.bin_M), at<uint32_t>(ws, L.st_total), at<uint32_t>(ws, L.st_base),
               at<uint32_t>(ws, L.st_blk0), at<uint2>(ws, L.l2_blocks), ctr + 11, ctr + 9);
    launch_pdl(k_l1_emit<SBITS>, L.nck_max, kBinWarps * 32, smem_e, st, E, at<const uint32_t>(ws, P.overflow),
               L.n_super, at<const uint32_t>(ws, L.bin_M), at<const uint32_t>(ws, L.st_base),
               at<const uint2>(ws, L.stg), at<uint2>(ws, L.ent));
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_bin(void *ws, const Layout &L, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0) return cudaSuccess;
    if (L.n == 0) {  // nothing to bin: empty ranges, no overflow
        cudaError_t e = cudaMemsetAsync(at<char>(ws, P.ranges), 0, 8 * (size_t)P.n_tiles, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(at<char>(ws, P.tile_count), 0, 4 * (size_t)P.n_tiles, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(at<char>(ws, P.overflow), 0, 4, st);
        return e;
    }
    uint32_t *ctr = at<uint32_t>(ws, L.counters);
    const int sms = sm_count();
    launch_pdl(k_escan_reduce, L.nblk_escan, kScanThreads, 0, st, at<const uint32_t>(ws, P.n_visible),
               at<const uint32_t>(ws, L.one), at<uint32_t>(ws, L.lb_escan));
    launch_pdl(k_escan_apply, L.nblk_escan, kScanThreads, 0, st, at<const uint32_t>(ws, P.n_visible),
               at<const uint32_t>(ws, L.one), at<const uint32_t>(ws, L.lb_escan), at<uint32_t>(ws, L.eoff),
               at<const uint32_t>(ws, P.total_pairs), L.capacity, ctr + 8, at<uint32_t>(ws, P.overflow),
               at<uint32_t>(ws, P.overflow_count));
    if (L.nck_max == 0) return cudaGetLastError();
#if defined(SS_DIAG_BIN_UPTO) && SS_DIAG_BIN_UPTO == 2
    return cudaGetLastError();
#endif
    const uint32_t *E = ctr + 8;
    int sbits = 1;
    while ((1 << sbits) < L.n_super) ++sbits;
    launch_pdl(k_entries, sms * kEntriesCtasPerSm, 256, 0, st, at<const uint32_t>(ws, P.n_visible), at<const uint32_t>(ws, P.overflow),
                                       at<const uint32_t>(ws, L.eoff), at<const uint32_t>(ws, P.order),
                                       at<const uint4>(ws, P.erec), at<const float4>(ws, P.rec), P.tiles_x, P.tiles_y,
                                       L.stx, at<uint2>(ws, L.stg), ctr + 12, at<uint32_t>(ws, L.big_queue));
    launch_pdl(k_big_entries, sms * 4, 256, 0, st, at<const uint32_t>(ws, P.overflow), ctr + 12,
                                           at<const uint32_t>(ws, L.big_queue), at<const uint32_t>(ws, L.eoff),
                                           at<const uint32_t>(ws, P.order), at<const uint4>(ws, P.erec),
                                           at<const float4>(ws, P.rec), P.tiles_x, P.tiles_y, L.stx,
                                           at<uint2>(ws, L.stg));
#if defined(SS_DIAG_BIN_UPTO) && SS_DIAG_BIN_UPTO == 3
    return cudaGetLastError();
#endif
    const size_t smem = l1_smem_bytes(L.n_super);
    cudaError_t e = cudaSuccess;
    switch (sbits <= 8 ? 8 : sbits) {
        case 8: e = launch_level1<8>(ws, L, smem, E, ctr, st); break;
        case 9: e = launch_level1<9>(ws, L, smem, E, ctr, st); break;
        case 10: e = launch_level1<10>(ws, L, smem, E, ctr, st); break;
        case 11: e = launch_level1<11>(ws, L, smem, E, ctr, st); break;
        default: e = launch_level1<12>(ws, L, smem, E, ctr, st); break;
    }
    if (e != cudaSuccess) return e;
#if defined(SS_DIAG_BIN_UPTO) && SS_DIAG_BIN_UPTO == 4
    return cudaGetLastError();
#endif
    launch_pdl(k_l2_count, L.l2_max_blocks, kL2Threads, 0, st, 
        at<const uint32_t>(ws, P.overflow), L.stx, P.tiles_x, P.tiles_y, L.n_super, at<const uint32_t>(ws, L.st_total),
        at<const uint32_t>(ws, L.st_base), at<const uint32_t>(ws, L.st_blk0), at<const uint2>(ws, L.l2_blocks),
        ctr + 11, at<const uint2>(ws, L.ent), at<uint32_t>(ws, L.l2_BC));
    launch_pdl(k_l2_scan, (L.n_super * 16 + 255) / 256, 256, 0, st, at<const uint32_t>(ws, P.overflow), L.stx,
               P.tiles_x, P.tiles_y, L.n_super, at<const uint32_t>(ws, L.st_total), at<const uint32_t>(ws, L.st_blk0),
               at<uint32_t>(ws, L.l2_BC), at<uint32_t>(ws, P.tile_count), at<uint32_t>(ws, L.tile_base),
               at<uint2>(ws, P.ranges), ctr + 10);
    return cudaGetLastError();
}

cudaError_t launch_tile_write(void *ws, const Layout &L, cudaStream_t st) {
    const ss_layout &P = L.pub;
    if (P.n_tiles == 0 || L.n == 0 || L.capacity == 0) return cudaSuccess;
    uint32_t *ctr = at<uint32_t>(ws, L.counters);
    launch_pdl(k_l2_write, L.l2_max_blocks, kL2Threads, 0, st, 
        at<const uint32_t>(ws, P.overflow), L.stx, P.tiles_x, P.tiles_y, at<const uint32_t>(ws, L.st_total),
        at<const uint32_t>(ws, L.st_base), at<const uint2>(ws, L.l2_blocks), ctr + 11, at<const uint2>(ws, L.ent),
        at<const uint32_t>(ws, L.l2_BC), at<const uint32_t>(ws, L.tile_base), at<uint32_t>(ws, P.sorted_value));
    return cudaGetLastError();
}

}  // namespace ss
