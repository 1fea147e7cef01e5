// prg_sort.cuh — device MSD radix sort of u64 keys, shared by K1 (edge sort,
// kernel1_sort.cpp:63-68) and K3 (CSR->CSC transpose, row / column ordering,
// exception lists).
//
// Why MSD with SMEM-staged tiles (measured on B200, tools/microbench):
//   * SMEM atomic ranking runs at ~5 keys/clk/SM: cheap, but unstable — fine
//     where the keys are unique above the payload bits;
//   * uncoalesced / atomic-cursor global scatters collapse to <0.15 keys/clk/SM,
//     so each tile is counting-sorted in shared memory and written as per-digit
//     contiguous runs at offsets from a reduce-then-scan over tile histograms;
//   * where input order must survive (stable mode: the K3 transpose sorts
//     column bits only and carries the row as payload), tiles are ranked
//     warp by warp: peers of equal digit from __match_any_sync (level 1) or
//     one ballot per digit bit (levels), no SMEM atomics.
// Global levels peel 8 key bits at a time until every segment fits in shared
// memory (kLocalCap keys); the local stage then sorts each segment in SMEM with
// a stable LSD over the segment's varying bits (5-bit digits, thread-private
// packed counters), or — for payload-free keys whose varying bits fit a 32-bit
// window and span >= 16 bits (K1) — a register-network + merge-path merge sort. An 8-bit ballot-ranked local pass measured slower (K1
// local 6.3 -> 8.4 ms): instruction-bound on the ballots; with __match_any_sync
// peers instead of ballots it is still slower (5.8 -> 9.0 ms).
// Children with <= 32 unsorted bits are joined only into runs whose window still fits 32
// bits; runs of at most 4096 keys go to local_small_kernel, the same merge sort on 64-,
// 128- or 256-thread CTAs, instead of wider-window segments for the LSD path.
// For reference, CUB's onesweep DeviceRadixSort on this B200 takes 16.6 ms for
// 2^28 48-bit keys; K1 (2^28 pairs in and out) takes 8.3 ms here.
#pragma once

#include "prg_common.cuh"

namespace prg::sort {

#ifndef PRG_SORT_ITEMS  // keys per thread of a global-level tile (A/B: tools/build_variant.py;
#define PRG_SORT_ITEMS 16  // 8 measured K1 10.87 vs 10.17 ms, transpose levels 3.06 vs 2.80 ms)
#endif
#ifndef PRG_SORT_PREFETCH  // global-level scatters load the next tile during the write-out (0: A/B)
#define PRG_SORT_PREFETCH 1
#endif
constexpr int kTileThreads = 512;
constexpr int kTileItems = PRG_SORT_ITEMS;
constexpr int kTile = kTileThreads * kTileItems;  // 8192 keys per global tile
constexpr int kRadix = 256;
constexpr int kLocalCap = 8192;       // keys per SMEM-resident segment
constexpr int kLocalThreads = 512;
constexpr int kSmallCap = 4096;       // keys per segment of the small-segment merge kernel
constexpr int kSmallThreads = 256;
constexpr int kCounters = 44;  // SortWorkspace::counters (up to 16 levels of tile counters; [40]/[41] small-kernel work / count)

struct Seg {
    uint64_t start;   // element offset in the key buffers
    uint32_t size;
    uint16_t shift;   // bits [shift, shift+bits) are the next digit
    uint8_t bits;     // 0 => no bits left (all keys equal above the local stage)
    uint8_t buf;      // which key buffer holds the segment
};

// Where the small-kernel segments go (local_small_kernel): the tail of the
// final-segment array, filled backwards (entry i at fin[cap - 1 - i]); every
// child of a level is final of one kind or the other, so the array's bound
// covers both.
struct SmallList {
    uint32_t* n_small = nullptr;  // null: never flag
    uint32_t cap = 0;
    int mode = 1;                 // 1: lone children; 2: window-bounded runs (see emit_children_block)
};

// ---------------------------------------------------------------------------
// Level-1 (whole input) kernels, parameterised by a key source.
//   Src must provide:
//     static constexpr size_t kSmem;   // bytes of tile scratch it needs
//     static constexpr int kHistBatch; // keys loaded ahead in the histogram pass (divides 16)
//     static constexpr bool kRegPrefetch; // key() is a plain load: the scatter may load the next tile early
//     static constexpr bool kL2Prefetch;  // else: prefetch_l2(i) pulls key i's bytes into L2 (may be a no-op)
//     __device__ void prefetch_l2(size_t i) const;
//     __device__ void prepare(size_t base, int cnt, void* smem) const;  // all threads; may __syncthreads
//     __device__ uint64_t key(size_t i, int li, const void* smem) const;  // li = i - base
// ---------------------------------------------------------------------------
template <class Src>
__global__ void __launch_bounds__(kTileThreads) l1_hist_kernel(Src src, size_t n, int shift,
                                                               unsigned dmask, uint32_t ntiles,
                                                               uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kRadix];
    extern __shared__ __align__(16) unsigned char src_smem[];
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int i = threadIdx.x; i < kRadix; i += blockDim.x) h[i] = 0;
        const size_t base = (size_t)t * kTile;
        const int cnt = (int)min((size_t)kTile, n - base);
        src.prepare(base, cnt, src_smem);
        __syncthreads();
        // Src::kHistBatch loads in flight, then their counts (measured per source:
        // 16 for 8-byte key arrays, 4 for the 16-byte edge pairs of K1)
        constexpr int B = Src::kHistBatch;
#pragma unroll
        for (int j0 = 0; j0 < kTileItems; j0 += B) {
            uint64_t k[B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const int li = (j0 + j) * kTileThreads + threadIdx.x;
                if (li < cnt) k[j] = src.key(base + li, li, src_smem);
            }
#pragma unroll
            for (int j = 0; j < B; ++j)
                if ((j0 + j) * kTileThreads + (int)threadIdx.x < cnt) atomicAdd(&h[(unsigned)(k[j] >> shift) & dmask], 1u);
        }
        __syncthreads();
        for (int d = threadIdx.x; d < kRadix; d += blockDim.x) hist[(size_t)d * ntiles + t] = h[d];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Stable tile ranking (used when the sort must preserve input order among
// keys equal above the payload bits — the K3 transpose keeps each column's
// rows in input order and so only sorts column bits). Each warp owns a
// contiguous chunk of the tile (position li = warp*kWarpSpan + j*32 + lane),
// so a key's stable slot is: prefix over (digit, earlier warps) + keys of the
// same digit in the warp's earlier rows + its peers among lower lanes.
// ---------------------------------------------------------------------------
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kWarpSpan = kTileItems * 32;
constexpr size_t kStableScratch = (size_t)kRadix * kTileWarps * sizeof(uint32_t);  // 16 KB
static_assert(kRadix * kTileWarps == 8 * kTileThreads, "scan assumes 8 counters per thread");

template <bool kStable>
__device__ __forceinline__ int tile_pos(int j) {
    return kStable ? (int)(dev::warp_id() * kWarpSpan + j * 32 + dev::lane_id()) : j * kTileThreads + (int)threadIdx.x;
}

// k[j] holds the key at tile_pos<true>(j) (valid when < cnt). On return skeys
// holds the tile in (digit, position) order and lstart[d] the digit starts.
// wc: kStableScratch bytes of SMEM (may alias dead scratch). Ends with a barrier.
// kMatch: peers by __match_any_sync (faster in the level-1 scatter: 1.90 -> 1.56 ms
// for the K3 transpose) instead of one ballot per digit bit (used where the
// match variant spills: the segmented levels).
template <bool kMatch>
__device__ __forceinline__ void stable_tile_scatter(const uint64_t (&k)[kTileItems], int cnt, int shift, int bits,
                                                    uint32_t* __restrict__ wc, uint32_t* __restrict__ lstart,
                                                    uint32_t* __restrict__ scan_tmp, uint64_t* __restrict__ skeys) {
    const unsigned w = dev::warp_id(), lane = dev::lane_id();
    const unsigned mask = (1u << bits) - 1u;
    const unsigned t = threadIdx.x;
    const unsigned lt = (1u << lane) - 1u;
    reinterpret_cast<uint4*>(wc)[2 * t] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(wc)[2 * t + 1] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    // Rank within the warp's chunk: peers (same digit, same row j) by ballots;
    // the highest peer advances the warp's running digit count (no atomics, so
    // skewed digits do not serialise). rk packs two 16-bit ranks per word.
    uint32_t rk[kTileItems / 2];
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
        const bool valid = tile_pos<true>(j) < cnt;
        const unsigned d = valid ? ((unsigned)(k[j] >> shift) & mask) : 0u;
        unsigned peers;
        if (kMatch) {
            peers = __match_any_sync(0xffffffffu, valid ? d : 0xffffffffu);
        } else {
            peers = __ballot_sync(0xffffffffu, valid);
            for (int b = 0; b < bits; ++b) {
                const bool bit = (d >> b) & 1u;
                const unsigned bal = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bal : ~bal;
            }
        }
        uint32_t* cp = &wc[w * kRadix + d];  // [warp][digit]: lanes of a warp hit distinct banks
        const uint32_t r = (valid ? *cp : 0u) + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == 31u - __clz(peers)) *cp = r + 1u;
        __syncwarp();
        if (j & 1) rk[j >> 1] |= r << 16; else rk[j >> 1] = r;
    }
    __syncthreads();
    {   // exclusive scan in (digit, warp) order; thread t owns digit t/2, warps 8*(t&1)..+7
        const unsigned d = t >> 1, w0 = (t & 1u) * 8u;
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = wc[(w0 + q) * kRadix + d];
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += v[q];
        uint32_t tot;
        uint32_t run = dev::block_excl_scan(sum, scan_tmp, tot);
        if ((t & 1u) == 0) lstart[d] = run;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            wc[(w0 + q) * kRadix + d] = run;
            run += v[q];
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
        if (tile_pos<true>(j) < cnt) {
            const unsigned d = (unsigned)(k[j] >> shift) & mask;
            const uint32_t r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
            PRG_DCHECK(wc[w * kRadix + d] + r < (uint32_t)cnt);
            skeys[wc[w * kRadix + d] + r] = k[j];
        }
    }
    __syncthreads();
}

// Tile-local counting sort in SMEM, then per-digit contiguous writes.
// kStable: input order is kept among equal digits (stable_tile_scatter).
template <class Src, bool kStable>
__global__ void __launch_bounds__(kTileThreads, 2) l1_scatter_kernel(Src src, size_t n, int shift, int bits,
                                                                  uint32_t ntiles,
                                                                  const uint32_t* __restrict__ off,
                                                                  uint64_t* __restrict__ out) {
    __shared__ uint32_t h[kRadix];
    __shared__ uint32_t lstart[kRadix];
    __shared__ uint64_t gbase[kRadix];
    __shared__ uint32_t scan_tmp[kTileThreads / 32 + 1];
    extern __shared__ __align__(16) uint64_t skeys[];  // kTile keys, then Src scratch (+ stable counters)
    void* src_smem = skeys + kTile;
    uint32_t* wc = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(src_smem) +
                                               (Src::kSmem >= kStableScratch ? 0 : ((Src::kSmem + 15) & ~size_t(15))));
    const unsigned dmask = (1u << bits) - 1u;
    // Sources without tile scratch are software-pipelined: the next tile's 16
    // loads are issued once this tile's keys sit in skeys (k is dead by then), so
    // they are in flight during the write-out (ncu before: 63% long-scoreboard
    // stalls, DRAM 42% — the load phase of a tile overlapped with nothing of its own CTA).
    // Sources whose key() transforms what it loads (kRegPrefetch false) would
    // stall on the transform: they only pull the next tile into L2 (prefetch_l2).
    // The stable ranking has no registers to spare (the register form spilled: 1.52 -> 1.60 ms).
    constexpr bool kPrefetch = PRG_SORT_PREFETCH && Src::kSmem == 0 && Src::kRegPrefetch && !kStable;
    constexpr bool kPrefetchL2 = PRG_SORT_PREFETCH && !kPrefetch && Src::kL2Prefetch;
    uint64_t k[kTileItems];
    auto load_tile = [&](uint32_t tt) {
        const size_t b = (size_t)tt * kTile;
        const int c = (int)min((size_t)kTile, n - b);
        // all 16 loads first (in flight together), then the counting
#pragma unroll
        for (int j = 0; j < kTileItems; ++j) {
            const int li = tile_pos<kStable>(j);
            if (li < c) k[j] = src.key(b + li, li, src_smem);
        }
    };
    if (kPrefetch && blockIdx.x < ntiles) load_tile(blockIdx.x);
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (!kStable)
            for (int i = threadIdx.x; i < kRadix; i += blockDim.x) h[i] = 0;
        const size_t base = (size_t)t * kTile;
        const int cnt = (int)min((size_t)kTile, n - base);
        if (!kPrefetch) src.prepare(base, cnt, src_smem);
        __syncthreads();
        if (!kPrefetch) load_tile(t);
        if (!kStable) {
#pragma unroll
            for (int j = 0; j < kTileItems; ++j)
                if (tile_pos<kStable>(j) < cnt) atomicAdd(&h[(unsigned)(k[j] >> shift) & dmask], 1u);
        }
        __syncthreads();
        if (kStable) {
            if (threadIdx.x < kRadix) gbase[threadIdx.x] = off[(size_t)threadIdx.x * ntiles + t];
            stable_tile_scatter<true>(k, cnt, shift, bits, wc, lstart, scan_tmp, skeys);  // ends with a barrier
        } else {
            uint32_t v = threadIdx.x < kRadix ? h[threadIdx.x] : 0u, tot;
            uint32_t ex = dev::block_excl_scan(v, scan_tmp, tot);
            if (threadIdx.x < kRadix) {
                lstart[threadIdx.x] = ex;
                h[threadIdx.x] = ex;  // becomes the per-digit cursor
                gbase[threadIdx.x] = off[(size_t)threadIdx.x * ntiles + t];
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kTileItems; ++j) {
                int li = j * kTileThreads + threadIdx.x;
                if (li < cnt) {
                    const uint32_t slot = atomicAdd(&h[(unsigned)(k[j] >> shift) & dmask], 1u);
                    PRG_DCHECK(slot < (uint32_t)cnt);
                    skeys[slot] = k[j];
                }
            }
            __syncthreads();
        }
        if (kPrefetch && t + gridDim.x < ntiles) load_tile(t + gridDim.x);
        if (kPrefetchL2 && t + gridDim.x < ntiles) {
            const size_t b = (size_t)(t + gridDim.x) * kTile;
            const int c = (int)min((size_t)kTile, n - b);
#pragma unroll
            for (int j = 0; j < kTileItems; ++j) {
                const int li = tile_pos<kStable>(j);
                if (li < c) src.prefetch_l2(b + li);
            }
        }
        for (int i = threadIdx.x; i < cnt; i += kTileThreads) {
            uint64_t key = skeys[i];
            unsigned d = (unsigned)(key >> shift) & dmask;
            PRG_DCHECK(gbase[d] + (i - lstart[d]) < n && i >= (int)lstart[d]);
            out[gbase[d] + (i - lstart[d])] = key;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Segmented levels (>= 2): only segments larger than kLocalCap take part.
// ---------------------------------------------------------------------------
struct LevelState {
    // inputs for a level
    const Seg* active;          // active segment list
    const uint32_t* n_active;   // device count
    // tile map built per level
    uint32_t* tile_seg;         // tile -> active segment index
    uint32_t* tile_idx;         // tile -> tile index within its segment
    uint32_t* n_tiles;          // device scalar
    uint32_t* seg_tile0;        // active seg -> first tile (global), size n_active+1
    uint64_t* seg_elem0;        // active seg -> first element in concatenation
};

// One block: scan active segment tile counts, emit the tile map.
__global__ void build_tiles_kernel(const Seg* __restrict__ active, const uint32_t* __restrict__ n_active,
                                   uint32_t* __restrict__ seg_tile0, uint64_t* __restrict__ seg_elem0,
                                   uint32_t* __restrict__ tile_seg, uint32_t* __restrict__ tile_idx,
                                   uint32_t* __restrict__ n_tiles, uint32_t max_tiles);

template <class KeyT>
__device__ __forceinline__ unsigned seg_digit(KeyT key, const Seg& s) {
    return (unsigned)(key >> s.shift) & ((1u << s.bits) - 1u);
}

__global__ void __launch_bounds__(kTileThreads) seg_hist_kernel(
    const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
    const Seg* __restrict__ active, const uint32_t* __restrict__ seg_tile0,
    const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_idx,
    const uint32_t* __restrict__ n_tiles, uint32_t* __restrict__ hist, uint32_t* __restrict__ next_tile);

template <bool kStable>
__global__ void __launch_bounds__(kTileThreads, 2) seg_scatter_kernel(
    const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
    uint64_t* __restrict__ out0, uint64_t* __restrict__ out1, const Seg* __restrict__ active,
    const uint32_t* __restrict__ seg_tile0, const uint64_t* __restrict__ seg_elem0,
    const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_idx,
    const uint32_t* __restrict__ n_tiles, const uint32_t* __restrict__ off, uint32_t* __restrict__ next_tile);

// After a level: split each active segment into 256 children, append them to
// the final list (size <= cap or no bits left) or the next active list.
__global__ void classify_kernel(const Seg* __restrict__ active, const uint32_t* __restrict__ n_active,
                                const uint32_t* __restrict__ seg_tile0,
                                const uint64_t* __restrict__ seg_elem0,
                                const uint32_t* __restrict__ off, Seg* __restrict__ next,
                                uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                uint32_t* __restrict__ n_fin, int floor_bit, SmallList small);

// Level-1 children classification (the whole input was one segment).
__global__ void classify_l1_kernel(const uint32_t* __restrict__ off, uint32_t ntiles, size_t n,
                                   int shift, int bits, Seg* __restrict__ next,
                                   uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                   uint32_t* __restrict__ n_fin);

// ---------------------------------------------------------------------------
// Local stage: one CTA sorts one SMEM-resident segment completely with a
// stable LSD radix sort over the segment's varying bit span only (found by an
// OR/AND reduction; the low `payload_bits` are carried, not sorted). The cost
// is independent of the key distribution — an MSD local stage degraded badly
// on heavy Kronecker rows (ncu: 58% barrier stalls, ~20 cycles/key).
// Ranking (CUB-style, no ballots, no match_any): thread t owns a contiguous run
// of 16 keys in the current order and counts them into thread-private 16-bit
// counters for (digit, t) — threads 2p and 2p+1 share one 32-bit word, so one
// conflict-free SMEM atomic per key returns the in-thread rank. A block scan
// over (digit, thread) then gives stable scatter offsets. Keys stay in
// registers; X is padded (one slot per 16) so blocked reads are conflict-light.
// ---------------------------------------------------------------------------
constexpr int kLocalItems = kLocalCap / kLocalThreads;  // 16 keys per thread
constexpr int kLocalWarps = kLocalThreads / 32;
constexpr int kLsdBits = 5;
constexpr int kLsdDigits = 1 << kLsdBits;
constexpr int kCntWords = kLsdDigits * (kLocalThreads / 2);  // packed counters
static_assert(kLocalItems == 16, "local stage assumes 16 keys per thread");

// Debug instrumentation of the local stage (PRG_LOCAL_STATS=1 at compile time).
#ifndef PRG_LOCAL_STATS
#define PRG_LOCAL_STATS 0
#endif
__device__ unsigned long long g_local_stats[16];

__host__ __device__ constexpr uint32_t xpad(uint32_t i) { return i + (i >> 4); }

struct LocalSmem {
    uint64_t X[kLocalCap + kLocalCap / 16];
    uint32_t cnt[kCntWords + kCntWords / 16];  // [digit][thread pair], padded (xpad)
    uint32_t seg_id;
    uint64_t red_or[kLocalWarps], red_and[kLocalWarps];
    uint32_t scan_tmp[kLocalWarps + 1];
};

// The 32-bit variant of the pass loop below (same ranking): keys are the
// window (key >> lo) of span hi-lo+1 <= 32 bits; `common` holds every bit
// outside the window. On return S.X[xpad(i)] holds the sorted full keys.
static __device__ __forceinline__ void cta_lsd_sort32(LocalSmem& S, uint32_t n, const uint64_t (&kin)[kLocalItems],
                                                      int lo, int hi, uint64_t common) {
    const unsigned tid = threadIdx.x;
    const uint32_t half = (tid & 1u) * 16u;
    uint32_t* X32 = reinterpret_cast<uint32_t*>(S.X);  // xpad-indexed, 4-byte slots
    uint32_t k[kLocalItems];
#pragma unroll
    for (int j = 0; j < kLocalItems; ++j) k[j] = (uint32_t)(kin[j] >> lo);  // slots past n: all ones
    constexpr int WPT = kCntWords / kLocalThreads;
    uint32_t* const my = &S.cnt[tid * (WPT + 1)];
    const uint32_t pp = (tid >> 1) + (tid >> 5);
    const int span = hi - lo + 1;
    for (int sh = 0; sh < span; sh += kLsdBits) {
#pragma unroll
        for (int q = 0; q < WPT; ++q) my[q] = 0;
        __syncthreads();
        uint32_t rk[kLocalItems / 2];
#pragma unroll
        for (int j = 0; j < kLocalItems; ++j) {
            const uint32_t d = (k[j] >> sh) & (kLsdDigits - 1);
            const uint32_t old = atomicAdd(&S.cnt[d * 272u + pp], 1u << half);
            const uint32_t r = (old >> half) & 0xffffu;
            if (j & 1) rk[j >> 1] |= r << 16; else rk[j >> 1] = r;
        }
        __syncthreads();
        {
            uint32_t ts = 0;
#pragma unroll 4
            for (int q = 0; q < WPT; ++q) {
                const uint32_t wv = my[q];
                ts += (wv & 0xffffu) + (wv >> 16);
            }
            uint32_t tot;
            uint32_t run = dev::block_excl_scan(ts, S.scan_tmp, tot);
#pragma unroll 4
            for (int q = 0; q < WPT; ++q) {
                const uint32_t wv = my[q];
                const uint32_t lo16 = wv & 0xffffu;
                my[q] = run | ((run + lo16) << 16);
                run += lo16 + (wv >> 16);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kLocalItems; ++j) {
            const uint32_t d = (k[j] >> sh) & (kLsdDigits - 1);
            const uint32_t pre = (S.cnt[d * 272u + pp] >> half) & 0xffffu;
            const uint32_t r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
            PRG_DCHECK(pre + r < (uint32_t)kLocalCap);
            X32[xpad(pre + r)] = k[j];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kLocalItems; ++j) k[j] = X32[tid * (kLocalItems + 1) + j];  // X32[xpad(tid*16+j)]
        __syncthreads();
    }
    // rebuild the full keys (slots past n sort last and are never stored)
#pragma unroll
    for (int j = 0; j < kLocalItems; ++j) S.X[tid * (kLocalItems + 1) + j] = common | ((uint64_t)k[j] << lo);
    __syncthreads();
}

// Batcher odd-even merge sort network for 16 keys (63 compare-exchanges).
template <class K>
__device__ __forceinline__ void sort16(K (&k)[kLocalItems]) {
    constexpr int P[63][2] = {{0,1},{2,3},{0,2},{1,3},{1,2},{4,5},{6,7},{4,6},{5,7},{5,6},{0,4},{2,6},{2,4},{1,5},
                              {3,7},{3,5},{1,2},{3,4},{5,6},{8,9},{10,11},{8,10},{9,11},{9,10},{12,13},{14,15},
                              {12,14},{13,15},{13,14},{8,12},{10,14},{10,12},{9,13},{11,15},{11,13},{9,10},{11,12},
                              {13,14},{0,8},{4,12},{4,8},{2,10},{6,14},{6,10},{2,4},{6,8},{10,12},{1,9},{5,13},
                              {5,9},{3,11},{7,15},{7,11},{3,5},{7,9},{11,13},{1,2},{3,4},{5,6},{7,8},{9,10},
                              {11,12},{13,14}};
#pragma unroll
    for (int q = 0; q < 63; ++q) {
        const K a = k[P[q][0]], b = k[P[q][1]];
        k[P[q][0]] = a < b ? a : b;
        k[P[q][1]] = a < b ? b : a;
    }
}

// Merge-sort alternative to the LSD passes for wide key spans without payload
// (K1 after two MSD levels: 8 bits of u and 24 of v, or more where small
// children were coalesced). Each thread sorts its 16 keys with a network in
// registers, then log2(n/16) merge-path levels in shared memory: thread t
// produces outputs [16t, 16t+16) of its pair of runs (binary search on the
// cross diagonal, then a 16-step serial merge). Keys compare whole: unstable is
// fine. Measured at S=24 (K1 local): 5.56 ms LSD -> 4.94 ms with the 32-bit
// windows merged; merging the 64-bit (coalesced, > 32-bit span) segments as
// well was slower (5.34 ms), and so were two interleaved merge paths per thread
// (5.47 ms) — the levels are issue/bank-conflict bound, not chain-latency bound. X is the xpad-indexed slot array of K (K = u32: the key window >> lo).
// On return S.X holds the sorted full keys.
// The first merge levels inside a warp, in registers: lane l holds the sorted
// keys [16l, 16l+16) of the warp's 512 slots. Level m (1..5) merges runs of
// 2^(m-1) lanes into runs of 2^m lanes as a bitonic merge: slot i of the lower
// run against slot L-1-i of the upper run (lane ^ (2^m - 1), register 15-j),
// then half-cleaners over lane distances 2^(m-2) .. 1 (same register) and over
// register strides 8 .. 1. No shared memory, no block barrier. `left` = the slots
// of this warp's 512 that hold keys to sort (the rest are all ones); only the
// levels that cover them run. Returns the run length reached (16 << levels).
template <class K>
__device__ __forceinline__ K shfl_xor_key(K v, int d) {
    if constexpr (sizeof(K) == 8) {
        const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, d);
        const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), d);
        return ((K)hi << 32) | lo;
    } else {
        return __shfl_xor_sync(0xffffffffu, v, d);
    }
}
template <class K>
__device__ __forceinline__ uint32_t warp_bitonic_merge(K (&k)[kLocalItems], uint32_t left, int max_levels) {
    const unsigned lane = threadIdx.x & 31u;
    uint32_t run = kLocalItems;
#pragma unroll
    for (int m = 1; m <= 5; ++m) {
        if (m > max_levels || run >= left) break;  // warp-uniform
        {
            const bool up = (lane >> (m - 1)) & 1u;
#pragma unroll
            for (int j = 0; j < kLocalItems / 2; ++j) {  // registers j and 15-j trade places across the pair of lanes
                const K a = k[j], b = k[kLocalItems - 1 - j];
                const K oa = shfl_xor_key<K>(b, (1 << m) - 1), ob = shfl_xor_key<K>(a, (1 << m) - 1);
                const K mna = a < oa ? a : oa, mxa = a < oa ? oa : a;
                const K mnb = b < ob ? b : ob, mxb = b < ob ? ob : b;
                k[j] = up ? mxa : mna;
                k[kLocalItems - 1 - j] = up ? mxb : mnb;
            }
        }
#pragma unroll
        for (int d = m - 2; d >= 0; --d) {
            const bool up = (lane >> d) & 1u;
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) {
                const K o = shfl_xor_key<K>(k[j], 1 << d);
                const K mn = k[j] < o ? k[j] : o, mx = k[j] < o ? o : k[j];
                k[j] = up ? mx : mn;
            }
        }
#pragma unroll
        for (int s = kLocalItems / 2; s > 0; s >>= 1) {
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) {
                if ((j & s) == 0) {
                    const K a = k[j], b = k[j + s];
                    k[j] = a < b ? a : b;
                    k[j + s] = a < b ? b : a;
                }
            }
        }
        run <<= 1;
    }
    return run;
}

// The merge sort proper: k holds this thread's 16 slots [16 tid, 16 tid + 16)
// (slots past n all ones); X is xpad-indexed scratch for nsort keys. On return k
// holds the sorted slots [16 tid, 16 tid + 16). Any block size (the small-segment
// kernel runs it with 256 threads). Ends with a barrier when a level ran.
template <class K>
static __device__ __forceinline__ void cta_merge_core(K* X, uint32_t n, K (&k)[kLocalItems], int warp_levels) {
    constexpr K kInf = ~K(0);
    const unsigned tid = threadIdx.x;
    // slots [0, nsort): n rounded up to whole threads; runs at the end are clipped
    const uint32_t nsort = n ? (n + kLocalItems - 1) & ~uint32_t(kLocalItems - 1) : kLocalItems;
    const bool active = tid * kLocalItems < nsort;
    uint32_t w0 = kLocalItems;
    if (sizeof(K) == 4 && warp_levels > 0) {
        // whole warps: lanes past nsort hold all-ones keys, which sort last
        if ((tid & ~31u) * kLocalItems < nsort) {
            sort16<K>(k);
            warp_bitonic_merge<K>(k, nsort - (tid & ~31u) * kLocalItems, warp_levels);
        }
        // block-uniform: every warp's slots are now sorted in runs of this length
        for (int m = 0; m < warp_levels && w0 < nsort; ++m) w0 <<= 1;
    } else if (active) {
        sort16<K>(k);
    }
    for (uint32_t w = w0; w < nsort; w <<= 1) {
        if (active) {
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) X[tid * (kLocalItems + 1) + j] = k[j];  // X[xpad(16t+j)]
        }
        __syncthreads();
        if (active) {
            const uint32_t pos = tid * kLocalItems;
            const uint32_t A = pos & ~(2 * w - 1), B = min(A + w, nsort);
            const uint32_t ea = B, eb = min(B + w, nsort);
            const uint32_t la = ea - A, lb = eb - B;
            const uint32_t diag = pos - A;
            uint32_t b0 = diag > lb ? diag - lb : 0u, b1 = min(diag, la);
            while (b0 < b1) {  // merge path: the outputs before diag take b0 keys from run A
                const uint32_t mid = (b0 + b1) >> 1;
                if (!(X[xpad(B + diag - 1 - mid)] < X[xpad(A + mid)])) b0 = mid + 1;
                else b1 = mid;
            }
            uint32_t ia = A + b0, ib = B + diag - b0;
            K va = ia < ea ? X[xpad(ia)] : kInf;
            K vb = ib < eb ? X[xpad(ib)] : kInf;
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) {
                const bool ta = !(vb < va);
                k[j] = ta ? va : vb;
                const uint32_t nx = ta ? ++ia : ++ib;
                const bool in = ta ? nx < ea : nx < eb;
                const K v = in ? X[xpad(nx)] : kInf;
                if (ta) va = v; else vb = v;
            }
        }
        __syncthreads();
    }
}

template <class K>
static __device__ __forceinline__ void cta_merge_sort(LocalSmem& S, uint32_t n, const uint64_t (&kin)[kLocalItems],
                                                      int lo, uint64_t common, int warp_levels) {
    const unsigned tid = threadIdx.x;
    K k[kLocalItems];
#pragma unroll
    for (int j = 0; j < kLocalItems; ++j) k[j] = (K)(kin[j] >> lo);  // slots past n: all ones
    cta_merge_core<K>(reinterpret_cast<K*>(S.X), n, k, warp_levels);
    // the full keys (slots past n sort last and are never stored)
#pragma unroll
    for (int j = 0; j < kLocalItems; ++j) S.X[tid * (kLocalItems + 1) + j] = common | ((uint64_t)k[j] << lo);
    __syncthreads();
}

// Sorts X[0, n) (n <= kLocalCap; X indexed through xpad). All threads call.
// merge_span: windows of at least this many varying bits (and no payload) are
// merge-sorted instead of LSD-sorted.
static __device__ __forceinline__ void cta_lsd_sort(LocalSmem& S, uint32_t n, int payload_bits, int merge_span) {
    const unsigned tid = threadIdx.x, lane = dev::lane_id(), w = dev::warp_id();
    const uint32_t half = (tid & 1u) * 16u;
    uint64_t k[kLocalItems];
    uint64_t o = 0, a = ~0ull;
#pragma unroll
    for (int j = 0; j < kLocalItems; ++j) {
        const uint32_t i = tid * kLocalItems + j;
        k[j] = i < n ? S.X[tid * (kLocalItems + 1) + j] : ~0ull;  // == X[xpad(i)]
        if (i < n) { o |= k[j]; a &= k[j]; }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, d);
        a &= __shfl_xor_sync(0xffffffffu, a, d);
    }
    if (lane == 0) { S.red_or[w] = o; S.red_and[w] = a; }
    __syncthreads();
    o = 0; a = ~0ull;
#pragma unroll
    for (int q = 0; q < kLocalWarps; ++q) { o |= S.red_or[q]; a &= S.red_and[q]; }
    const uint64_t diff = (o ^ a) & (~0ull << payload_bits);
    if (diff == 0) { __syncthreads(); return; }  // equal above the payload: sorted
    const int lo = __ffsll((long long)diff) - 1;
    const int hi = 63 - __clzll((long long)diff);
    const bool merge = payload_bits == 0 && hi - lo + 1 >= (merge_span & 0xff) && (hi - lo < 32 || (merge_span & 0x100));
    if (PRG_LOCAL_STATS && threadIdx.x == 0) atomicAdd(&g_local_stats[merge ? (hi - lo < 32 ? 5 : 6) : 7], 1ull);
    if (merge) {
        if (hi - lo < 32)
            cta_merge_sort<uint32_t>(S, n, k, lo, a & ~(((hi - lo == 31) ? ~0ull >> 32 : ((1ull << (hi - lo + 1)) - 1)) << lo),
                                     (merge_span >> 12) & 7);
        else  // PRG_MERGE_SPAN + 256: 64-bit keys too (measured slower than their LSD passes)
            cta_merge_sort<uint64_t>(S, n, k, 0, 0ull, (merge_span >> 12) & 7);
        return;
    }
    if (payload_bits == 0 && hi - lo < 32) {
        // Every bit outside [lo, hi] is common to the segment: sort the 32-bit
        // window and rebuild the keys (K1 after two MSD levels: 32 varying bits
        // of (u, v)). Half the shared-memory bytes per scatter and reload.
        cta_lsd_sort32(S, n, k, lo, hi, a & ~(((hi - lo == 31) ? ~0ull >> 32 : ((1ull << (hi - lo + 1)) - 1)) << lo));
        return;
    }
    constexpr int WPT = kCntWords / kLocalThreads;  // counter words per thread (16)
    static_assert(WPT == 16, "xpad(tid*16 + q) == tid*17 + q relies on 16 words per thread");
    uint32_t* const my = &S.cnt[tid * (WPT + 1)];   // this thread's 16 scan words, contiguous after padding
    // counter of (digit d, my thread pair) = cnt[xpad(d*256 + p)] = cnt[d*272 + p + p/16]
    const uint32_t pp = (tid >> 1) + (tid >> 5);
    static_assert(kLocalThreads / 2 == 256, "digit stride 272 assumes 256 thread pairs");
    for (int sh = lo; sh <= hi; sh += kLsdBits) {
#pragma unroll
        for (int q = 0; q < WPT; ++q) my[q] = 0;
        __syncthreads();
        uint32_t rk[kLocalItems / 2];
#pragma unroll
        for (int j = 0; j < kLocalItems; ++j) {
            const uint32_t d = (uint32_t)(k[j] >> sh) & (kLsdDigits - 1);
            const uint32_t old = atomicAdd(&S.cnt[d * 272u + pp], 1u << half);
            const uint32_t r = (old >> half) & 0xffffu;
            if (j & 1) rk[j >> 1] |= r << 16; else rk[j >> 1] = r;
        }
        __syncthreads();
        {   // exclusive scan over words in (digit, pair) order; each word holds
            // (even thread, odd thread) counts -> (prefix_even, prefix_odd)
            uint32_t ts = 0;
#pragma unroll 4
            for (int q = 0; q < WPT; ++q) {
                const uint32_t wv = my[q];
                ts += (wv & 0xffffu) + (wv >> 16);
            }
            uint32_t tot;
            uint32_t run = dev::block_excl_scan(ts, S.scan_tmp, tot);
#pragma unroll 4
            for (int q = 0; q < WPT; ++q) {
                const uint32_t wv = my[q];
                const uint32_t lo16 = wv & 0xffffu;
                my[q] = run | ((run + lo16) << 16);
                run += lo16 + (wv >> 16);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kLocalItems; ++j) {
            const uint32_t d = (uint32_t)(k[j] >> sh) & (kLsdDigits - 1);
            const uint32_t pre = (S.cnt[d * 272u + pp] >> half) & 0xffffu;
            const uint32_t r = (rk[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
            PRG_DCHECK(pre + r < (uint32_t)kLocalCap);
            S.X[xpad(pre + r)] = k[j];
        }
        __syncthreads();
        if (sh + kLsdBits <= hi) {
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) k[j] = S.X[tid * (kLocalItems + 1) + j];  // X[xpad(tid*16+j)]
        }
    }
}

// Dst must provide:
//   __device__ void store(uint64_t pos, uint64_t key, bool has_prev, uint64_t prev) const;
// (has_prev/prev: the preceding key in sorted order when it lies in the same segment).
template <class Dst>
__global__ void __launch_bounds__(kLocalThreads, 2)
    local_sort_kernel(const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
                      const Seg* __restrict__ fin, const uint32_t* __restrict__ n_fin,
                      uint32_t* __restrict__ work, Dst dst, int payload_bits, int merge_span) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LocalSmem& S = *reinterpret_cast<LocalSmem*>(smem_raw);
    const uint32_t nf = *n_fin;
    for (;;) {
        if (threadIdx.x == 0) S.seg_id = atomicAdd(work, 1u);
        __syncthreads();
        const uint32_t sid = S.seg_id;
        __syncthreads();
        if (sid >= nf) break;
        const Seg sg = fin[sid];
        const uint64_t* src = sg.buf ? keys1 : keys0;
        const uint32_t n = sg.size;
        if (n == 0) continue;
        if (n > (uint32_t)kLocalCap) {
            // Only segments with no key bits left can exceed the cap: all keys
            // are equal, so the segment is already sorted.
            const uint64_t first = src[sg.start];
            for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads) {
                const uint64_t k = src[sg.start + i];
                PRG_DCHECK((k >> payload_bits) == (first >> payload_bits));
                dst.store(sg.start + i, k, i > 0, k);
            }
            continue;
        }
        long long c0 = PRG_LOCAL_STATS ? clock64() : 0;
        for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads) S.X[xpad(i)] = src[sg.start + i];
        __syncthreads();
        long long c1 = PRG_LOCAL_STATS ? clock64() : 0;
        cta_lsd_sort(S, n, payload_bits, merge_span);
        long long c2 = PRG_LOCAL_STATS ? clock64() : 0;
        for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads)
            dst.store(sg.start + i, S.X[xpad(i)], i > 0, i > 0 ? S.X[xpad(i - 1)] : 0ull);
        __syncthreads();
        if (PRG_LOCAL_STATS && threadIdx.x == 0) {
            long long c3 = clock64();
            atomicAdd(&g_local_stats[0], 1ull);
            atomicAdd(&g_local_stats[1], (unsigned long long)n);
            atomicAdd(&g_local_stats[2], (unsigned long long)(c1 - c0));
            atomicAdd(&g_local_stats[3], (unsigned long long)(c2 - c1));
            atomicAdd(&g_local_stats[4], (unsigned long long)(c3 - c2));

            atomicAdd(&g_local_stats[8 + min(7, 31 - __clz(n | 1) - 6 < 0 ? 0 : 31 - __clz(n | 1) - 6)], 1ull);
        }
    }
}

// Small segments (flagged by the level bookkeeping: one child of at most
// kSmallCap keys whose unsorted bits fit a 32-bit window, no payload): the same
// register-network + merge-path sort on 256-thread CTAs, four to an SM. Such
// children used to be joined into <= 8192-key segments whose > 32-bit windows
// took the LSD path (44% of K1's segments at S=24), because a lone ~3 K-key
// child left two thirds of a 512-thread CTA idle.
template <int kThreads>
struct SmallSmem {
    uint32_t X[16 * kThreads + kThreads];
    uint64_t red_or[kThreads / 32], red_and[kThreads / 32];
    uint32_t chunk_base, chunk_mask;
};
// Segments of [size_lo, size_hi] keys (size_hi <= 16 * kThreads) of the small list; the list
// is claimed eight entries at a time (one atomic and one ballot per chunk).
template <class Dst, int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    local_small_kernel(const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
                       const Seg* __restrict__ fin_end, const uint32_t* __restrict__ n_small,
                       uint32_t* __restrict__ work, Dst dst, int warp_levels, uint32_t size_lo, uint32_t size_hi) {
    // segment i of the list sits at fin_end[-1 - i] (the tail of the final-segment array, filled backwards)
    __shared__ SmallSmem<kThreads> S;
    const uint32_t nf = *n_small;
    const unsigned tid = threadIdx.x, lane = dev::lane_id(), w = dev::warp_id();
    for (;;) {
        if (tid < 32) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(work, 8u);
            base = __shfl_sync(0xffffffffu, base, 0);
            bool mine = false;
            if (lane < 8 && base + lane < nf) {
                const uint32_t sz = (fin_end - 1 - (base + lane))->size;
                mine = sz >= size_lo && sz <= size_hi;
            }
            const unsigned m = __ballot_sync(0xffffffffu, mine);
            if (lane == 0) { S.chunk_base = base; S.chunk_mask = m; }
        }
        __syncthreads();
        const uint32_t base = S.chunk_base;
        unsigned todo = S.chunk_mask;
        __syncthreads();
        if (base >= nf) break;
        while (todo) {
            const uint32_t sid = base + (uint32_t)__ffs(todo) - 1u;
            todo &= todo - 1u;
            const Seg sg = *(fin_end - 1 - sid);
            const uint64_t* src = (sg.buf ? keys1 : keys0) + sg.start;
            const uint32_t n = sg.size;
            PRG_DCHECK(n > 0 && n <= 16u * kThreads);
            // blocked loads: thread t holds keys [16t, 16t+16) (128 contiguous bytes)
            uint64_t k64[kLocalItems];
            uint64_t o = 0, a = ~0ull;
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) {
                const uint32_t i = tid * kLocalItems + j;
                k64[j] = i < n ? src[i] : ~0ull;
                if (i < n) { o |= k64[j]; a &= k64[j]; }
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                o |= __shfl_xor_sync(0xffffffffu, o, d);
                a &= __shfl_xor_sync(0xffffffffu, a, d);
            }
            if (lane == 0) { S.red_or[w] = o; S.red_and[w] = a; }
            __syncthreads();
            o = 0; a = ~0ull;
#pragma unroll
            for (int q = 0; q < kThreads / 32; ++q) { o |= S.red_or[q]; a &= S.red_and[q]; }
            const uint64_t diff = o ^ a;
            const int lo = diff ? __ffsll((long long)diff) - 1 : 0;
            PRG_DCHECK(diff == 0 || 63 - __clzll((long long)diff) - lo < 32);
            const uint64_t common = a & ~(0xffffffffull << lo);
            uint32_t k[kLocalItems];
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j)
                k[j] = tid * kLocalItems + j < n ? (uint32_t)(k64[j] >> lo) : 0xffffffffu;
            if (diff) cta_merge_core<uint32_t>(S.X, n, k, warp_levels);
#pragma unroll
            for (int j = 0; j < kLocalItems; ++j) S.X[tid * (kLocalItems + 1) + j] = k[j];
            __syncthreads();
            for (uint32_t i = tid; i < n; i += kThreads) {
                const uint64_t key = common | ((uint64_t)S.X[xpad(i)] << lo);
                dst.store(sg.start + i, key, i > 0, i > 0 ? (common | ((uint64_t)S.X[xpad(i - 1)] << lo)) : 0ull);
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Host driver.
// ---------------------------------------------------------------------------
struct SortWorkspace {
    // Allocated by plan(); all device.
    DevBuf<uint64_t> keys[2];
    DevBuf<uint32_t> hist, off;
    DevBuf<Seg> lists[2], fin;
    // [0]=n_active(a) [1]=n_active(b) [2]=n_fin [3]=work [4]=n_tiles [8+2l]/[9+2l]=tile counters of level l
    DevBuf<uint32_t> counters;
    DevBuf<uint32_t> tile_seg, tile_idx, seg_tile0;
    DevBuf<uint64_t> seg_elem0;
    size_t n = 0;          // capacity
    size_t n_sorting = 0;  // keys of the sort in progress
    uint32_t max_tiles = 0, max_active = 0, max_fin = 0;
};

void sort_workspace_init(SortWorkspace& ws, size_t n, cudaStream_t s);
size_t local_smem_bytes();
int local_merge_span();  // PRG_MERGE_SPAN (default 16): see cta_lsd_sort
int local_small_min();   // PRG_SMALL_MIN: smallest child sorted by local_small_kernel (0 = off)
int local_small_mode(size_t n);  // 1 = lone children only, 2 = window-bounded runs in three CTA sizes (PRG_SMALL_MODE forces one)
int sort_grid_mult(int which);  // CTAs per SM of the level-1 (1) / segmented (2) tile kernels: PRG_SORT_GRID1/2

// Runs levels >= 2 until every segment is final; then the caller launches
// local_sort_kernel with its Dst. `key_bits` is the number of significant bits.
void run_segmented_levels(SortWorkspace& ws, int levels_left, int floor_bit, bool stable, cudaStream_t s);

// src_hist feeds the level-1 histogram pass and src_scat the level-1 scatter
// pass; they must produce identical keys (K3 uses the split to capture its
// exception list exactly once).
// stable: keys equal above `payload_bits` keep their input order (every pass
// is stable; the payload bits are never sorted).
template <class Src, class Dst>
void msd_sort_split(Src src_hist, Src src_scat, size_t n, int key_bits, Dst dst, SortWorkspace& ws,
                    cudaStream_t s, const char* tag = "sort", int payload_bits = 0, bool stable = false) {
    const std::string t(tag);
    if (n == 0) return;
    sort_workspace_init(ws, n, s);
    ws.n_sorting = n;
    // Digits cover bits [payload_bits, key_bits); the low payload bits ride along
    // (they never decide the order: keys are unique above them, or equal keys
    // carry equal payloads).
    const int span = key_bits - payload_bits;
    const int bits1 = span < 8 ? (span > 0 ? span : 1) : 8;
    const int shift1 = key_bits - bits1 > payload_bits ? key_bits - bits1 : payload_bits;
    const unsigned dmask = (1u << bits1) - 1u;
    const uint32_t ntiles = div_up(n, kTile);
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)num_sms() * sort_grid_mult(1));
    PRG_CUDA(cudaMemsetAsync(ws.counters.get(), 0, kCounters * sizeof(uint32_t), s));
    {
        ProfScope prof(t + "_l1_hist", s);
        if (Src::kSmem > 48 * 1024)
            PRG_CUDA(cudaFuncSetAttribute(l1_hist_kernel<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)Src::kSmem));
        l1_hist_kernel<Src><<<grid, kTileThreads, Src::kSmem, s>>>(src_hist, n, shift1, dmask, ntiles,
                                                                    ws.hist.get());
        PRG_LAUNCH_CHECK();
        exclusive_scan_u32(ws.hist.get(), ws.off.get(), (size_t)kRadix * ntiles, nullptr, s);
    }
    {
        ProfScope prof(t + "_l1_scatter", s);
        if (stable) {
            const size_t sx = Src::kSmem >= kStableScratch ? Src::kSmem : ((Src::kSmem + 15) & ~size_t(15)) + kStableScratch;
            const size_t smem = (size_t)kTile * sizeof(uint64_t) + sx;
            PRG_CUDA(cudaFuncSetAttribute(l1_scatter_kernel<Src, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
            l1_scatter_kernel<Src, true><<<grid, kTileThreads, smem, s>>>(src_scat, n, shift1, bits1, ntiles,
                                                                          ws.off.get(), ws.keys[1].get());
        } else {
            const size_t smem = (size_t)kTile * sizeof(uint64_t) + Src::kSmem;
            PRG_CUDA(cudaFuncSetAttribute(l1_scatter_kernel<Src, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
            l1_scatter_kernel<Src, false><<<grid, kTileThreads, smem, s>>>(src_scat, n, shift1, bits1, ntiles,
                                                                           ws.off.get(), ws.keys[1].get());
        }
        PRG_LAUNCH_CHECK();
        const int rem1 = shift1 - payload_bits;
        classify_l1_kernel<<<1, kRadix, 0, s>>>(ws.off.get(), ntiles, n, shift1, rem1 >= 8 ? 8 : rem1,
                                                 ws.lists[0].get(), ws.counters.get() + 0, ws.fin.get(),
                                                 ws.counters.get() + 2);
        PRG_LAUNCH_CHECK();
    }
    {
        ProfScope prof(t + "_levels", s);
        run_segmented_levels(ws, (shift1 - payload_bits + 7) / 8, payload_bits, stable, s);
    }
    {
        ProfScope prof(t + "_local", s);
        if (!stable && payload_bits == 0 && local_small_min() > 0) {
            const int wl = (local_merge_span() >> 12) & 7;
            uint32_t* cn = ws.counters.get();
            const Seg* fe = ws.fin.get() + ws.max_fin;
            if (local_small_mode(n) == 2) {  // three CTA sizes over the one list ([40], [42], [43]: their work counters)
                local_small_kernel<Dst, 256, 4><<<num_sms() * 4, 256, 0, s>>>(
                    ws.keys[0].get(), ws.keys[1].get(), fe, cn + 41, cn + 40, dst, wl, 2049u, 4096u);
                local_small_kernel<Dst, 128, 8><<<num_sms() * 8, 128, 0, s>>>(
                    ws.keys[0].get(), ws.keys[1].get(), fe, cn + 41, cn + 42, dst, wl, 1025u, 2048u);
                local_small_kernel<Dst, 64, 16><<<num_sms() * 16, 64, 0, s>>>(
                    ws.keys[0].get(), ws.keys[1].get(), fe, cn + 41, cn + 43, dst, wl, 1u, 1024u);
            } else {
                local_small_kernel<Dst, 256, 4><<<num_sms() * 4, 256, 0, s>>>(
                    ws.keys[0].get(), ws.keys[1].get(), fe, cn + 41, cn + 40, dst, wl, 1u, 4096u);
            }
            PRG_LAUNCH_CHECK();
        }
        PRG_CUDA(cudaFuncSetAttribute(local_sort_kernel<Dst>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)local_smem_bytes()));
        local_sort_kernel<Dst><<<num_sms() * 2, kLocalThreads, local_smem_bytes(), s>>>(
            ws.keys[0].get(), ws.keys[1].get(), ws.fin.get(), ws.counters.get() + 2, ws.counters.get() + 3, dst,
            payload_bits, local_merge_span());
        PRG_LAUNCH_CHECK();
    }
}

template <class Src, class Dst>
void msd_sort(Src src, size_t n, int key_bits, Dst dst, SortWorkspace& ws, cudaStream_t s,
              const char* tag = "sort", int payload_bits = 0, bool stable = false) {
    msd_sort_split(src, src, n, key_bits, dst, ws, s, tag, payload_bits, stable);
}

}  // namespace prg::sort
