// prg_sort.cuh — device MSD radix sort of u64 keys, shared by K1 (edge sort,
// kernel1_sort.cpp:63-68) and the K3 CSR->CSC transpose.
//
// Why MSD with SMEM-staged tiles (measured on B200, tools/microbench):
//   * SMEM atomic ranking runs at ~5 keys/clk/SM: cheap, but unstable — fine
//     for MSD, where every level only partitions and the final local stage
//     sorts completely (equal keys are bit-identical, so output is unique);
//   * __match_any_sync (the usual stable warp ranking) runs at only ~0.5/clk/SM;
//   * uncoalesced / atomic-cursor global scatters collapse to <0.15 keys/clk/SM,
//     so each tile is counting-sorted in shared memory and written as per-digit
//     contiguous runs at offsets from a reduce-then-scan over tile histograms.
// Global levels peel 8 key bits at a time until every segment fits in shared
// memory (kLocalCap keys); the local stage then sorts each segment in SMEM with
// adaptive 12-bit counting passes, warp bitonic networks and insertion sorts.
#pragma once

#include "prg_common.cuh"

namespace prg::sort {

constexpr int kTileThreads = 512;
constexpr int kTileItems = 16;
constexpr int kTile = kTileThreads * kTileItems;  // 8192 keys per global tile
constexpr int kRadix = 256;
constexpr int kLocalCap = 8192;       // keys per SMEM-resident segment
constexpr int kLocalThreads = 512;
constexpr int kWindowBits = 12;
constexpr int kLocalBins = 1 << kWindowBits;
constexpr int kSmallMax = 16;         // <= : one-thread insertion sort
constexpr int kMidMax = 256;          // <= : one-warp bitonic network

struct Seg {
    uint64_t start;   // element offset in the key buffers
    uint32_t size;
    uint16_t shift;   // bits [shift, shift+bits) are the next digit
    uint8_t bits;     // 0 => no bits left (all keys equal above the local stage)
    uint8_t buf;      // which key buffer holds the segment
};

// ---------------------------------------------------------------------------
// Level-1 (whole input) kernels, parameterised by a key source.
//   Src must provide:
//     static constexpr size_t kSmem;   // bytes of tile scratch it needs
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
#pragma unroll 4
        for (int j = 0; j < kTileItems; ++j) {
            const int li = j * kTileThreads + threadIdx.x;
            if (li < cnt) atomicAdd(&h[(unsigned)(src.key(base + li, li, src_smem) >> shift) & dmask], 1u);
        }
        __syncthreads();
        for (int d = threadIdx.x; d < kRadix; d += blockDim.x) hist[(size_t)d * ntiles + t] = h[d];
        __syncthreads();
    }
}

// Tile-local counting sort in SMEM, then per-digit contiguous writes.
template <class Src>
__global__ void __launch_bounds__(kTileThreads) l1_scatter_kernel(Src src, size_t n, int shift,
                                                                  unsigned dmask, uint32_t ntiles,
                                                                  const uint32_t* __restrict__ off,
                                                                  uint64_t* __restrict__ out) {
    __shared__ uint32_t h[kRadix];
    __shared__ uint32_t lstart[kRadix];
    __shared__ uint64_t gbase[kRadix];
    __shared__ uint32_t scan_tmp[kTileThreads / 32 + 1];
    extern __shared__ __align__(16) uint64_t skeys[];  // kTile keys, then Src scratch
    void* src_smem = skeys + kTile;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int i = threadIdx.x; i < kRadix; i += blockDim.x) h[i] = 0;
        const size_t base = (size_t)t * kTile;
        const int cnt = (int)min((size_t)kTile, n - base);
        src.prepare(base, cnt, src_smem);
        __syncthreads();
        uint64_t k[kTileItems];
        uint32_t r[kTileItems];
#pragma unroll
        for (int j = 0; j < kTileItems; ++j) {
            int li = j * kTileThreads + threadIdx.x;
            if (li < cnt) {
                k[j] = src.key(base + li, li, src_smem);
                r[j] = atomicAdd(&h[(unsigned)(k[j] >> shift) & dmask], 1u);
            }
        }
        __syncthreads();
        {
            uint32_t v = threadIdx.x < kRadix ? h[threadIdx.x] : 0u, tot;
            uint32_t ex = dev::block_excl_scan(v, scan_tmp, tot);
            if (threadIdx.x < kRadix) {
                lstart[threadIdx.x] = ex;
                gbase[threadIdx.x] = off[(size_t)threadIdx.x * ntiles + t];
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kTileItems; ++j) {
            int li = j * kTileThreads + threadIdx.x;
            if (li < cnt) skeys[lstart[(unsigned)(k[j] >> shift) & dmask] + r[j]] = k[j];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += kTileThreads) {
            uint64_t key = skeys[i];
            unsigned d = (unsigned)(key >> shift) & dmask;
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
    const uint32_t* __restrict__ n_tiles, uint32_t* __restrict__ hist);

__global__ void __launch_bounds__(kTileThreads) seg_scatter_kernel(
    const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
    uint64_t* __restrict__ out0, uint64_t* __restrict__ out1, const Seg* __restrict__ active,
    const uint32_t* __restrict__ seg_tile0, const uint64_t* __restrict__ seg_elem0,
    const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_idx,
    const uint32_t* __restrict__ n_tiles, const uint32_t* __restrict__ off);

// After a level: split each active segment into 256 children, append them to
// the final list (size <= cap or no bits left) or the next active list.
__global__ void classify_kernel(const Seg* __restrict__ active, const uint32_t* __restrict__ n_active,
                                const uint32_t* __restrict__ seg_tile0,
                                const uint64_t* __restrict__ seg_elem0,
                                const uint32_t* __restrict__ off, Seg* __restrict__ next,
                                uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                uint32_t* __restrict__ n_fin);

// Level-1 children classification (the whole input was one segment).
__global__ void classify_l1_kernel(const uint32_t* __restrict__ off, uint32_t ntiles, size_t n,
                                   int shift, int bits, Seg* __restrict__ next,
                                   uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                   uint32_t* __restrict__ n_fin);

// ---------------------------------------------------------------------------
// Local stage: one CTA sorts one SMEM-resident segment completely.
// ---------------------------------------------------------------------------
struct LocalSmem {
    uint64_t X[kLocalCap];
    uint64_t Y[kLocalCap];
    uint32_t hist[kLocalBins];
    uint32_t small_list[kLocalCap / 2];
    uint32_t mid_list[kLocalCap / (kSmallMax + 1) + 1];
    uint32_t big_list[kLocalCap / (kMidMax + 1) + 2];
    uint32_t n_small, n_mid, n_big;
    uint32_t seg_id;
    uint64_t red_or[kLocalThreads / 32], red_and[kLocalThreads / 32];
    uint32_t scan_tmp[kLocalThreads / 32 + 1];
};

__device__ __forceinline__ uint32_t pack_range(uint32_t b, uint32_t m) { return (b << 14) | m; }
__device__ __forceinline__ uint32_t range_b(uint32_t r) { return r >> 14; }
__device__ __forceinline__ uint32_t range_m(uint32_t r) { return r & 0x3fffu; }

__device__ __forceinline__ void push_range(LocalSmem& S, uint32_t b, uint32_t m) {
    if (m <= 1) return;
    if (m <= kSmallMax) S.small_list[atomicAdd(&S.n_small, 1u)] = pack_range(b, m);
    else if (m <= kMidMax) S.mid_list[atomicAdd(&S.n_mid, 1u)] = pack_range(b, m);
    else S.big_list[atomicAdd(&S.n_big, 1u)] = pack_range(b, m);
}

// One thread insertion-sorts X[b, b+m).
__device__ __forceinline__ void thread_insertion(uint64_t* X, uint32_t b, uint32_t m) {
    for (uint32_t i = b + 1; i < b + m; ++i) {
        uint64_t v = X[i];
        uint32_t j = i;
        while (j > b && X[j - 1] > v) { X[j] = X[j - 1]; --j; }
        X[j] = v;
    }
}

// ---------------------------------------------------------------------------
// Local stage: device routines
// cta_counting_pass: CTA-wide counting sort of X[b,b+m) by the 12 highest
// varying bits (via Y, copied back), pushing children ranges.
// warp_bitonic_256: one warp sorts X[b,b+m), m <= 256, in registers.
// cta_sort_segment: sorts a loaded segment X[0,n) completely.
// ---------------------------------------------------------------------------
static __device__ __noinline__ void cta_counting_pass(LocalSmem& S, uint32_t b, uint32_t m) {
    const unsigned tid = threadIdx.x, lane = dev::lane_id(), w = dev::warp_id();
    constexpr unsigned NW = kLocalThreads / 32;
    uint64_t o = 0, a = ~0ull;
    for (uint32_t i = b + tid; i < b + m; i += kLocalThreads) { uint64_t x = S.X[i]; o |= x; a &= x; }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, d);
        a &= __shfl_xor_sync(0xffffffffu, a, d);
    }
    if (lane == 0) { S.red_or[w] = o; S.red_and[w] = a; }
    __syncthreads();
    o = 0; a = ~0ull;
#pragma unroll
    for (unsigned k = 0; k < NW; ++k) { o |= S.red_or[k]; a &= S.red_and[k]; }
    const uint64_t diff = o ^ a;
    __syncthreads();
    if (diff == 0) return;  // all keys equal: already sorted
    const int h = 63 - __clzll((long long)diff);
    const int wb = h + 1 < kWindowBits ? h + 1 : kWindowBits;
    const int sh = h + 1 - wb;
    const unsigned mask = (1u << wb) - 1u, nb = 1u << wb;
    for (unsigned i = tid; i < nb; i += kLocalThreads) S.hist[i] = 0;
    __syncthreads();
    for (uint32_t i = b + tid; i < b + m; i += kLocalThreads)
        atomicAdd(&S.hist[(unsigned)(S.X[i] >> sh) & mask], 1u);
    __syncthreads();
    // exclusive scan over nb bins, kLocalBins/kLocalThreads = 8 bins per thread
    constexpr unsigned BPT = kLocalBins / kLocalThreads;
    uint32_t c[BPT], s = 0;
#pragma unroll
    for (unsigned k = 0; k < BPT; ++k) {
        unsigned bin = tid * BPT + k;
        c[k] = bin < nb ? S.hist[bin] : 0u;
        s += c[k];
    }
    uint32_t tot;
    uint32_t run = dev::block_excl_scan(s, S.scan_tmp, tot);
#pragma unroll
    for (unsigned k = 0; k < BPT; ++k) {
        unsigned bin = tid * BPT + k;
        if (bin < nb) {
            S.hist[bin] = run;
            if (c[k] > 1) push_range(S, b + run, c[k]);
        }
        run += c[k];
    }
    __syncthreads();
    for (uint32_t i = b + tid; i < b + m; i += kLocalThreads) {
        uint64_t x = S.X[i];
        uint32_t p = atomicAdd(&S.hist[(unsigned)(x >> sh) & mask], 1u);
        S.Y[b + p] = x;
    }
    __syncthreads();
    for (uint32_t i = b + tid; i < b + m; i += kLocalThreads) S.X[i] = S.Y[i];
    __syncthreads();
}

static __device__ __noinline__ void warp_bitonic_256(uint64_t* X, uint32_t b, uint32_t m) {
    const unsigned lane = dev::lane_id();
    uint64_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        uint32_t e = j * 32 + lane;
        v[j] = e < m ? X[b + e] : ~0ull;
    }
#pragma unroll
    for (int k = 2; k <= 256; k <<= 1) {
#pragma unroll
        for (int d = k >> 1; d > 0; d >>= 1) {
            if (d >= 32) {
                const int dj = d >> 5;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int jp = j ^ dj;
                    if (jp > j) {
                        const bool asc = (((j * 32 + lane) & k) == 0);
                        const uint64_t x = v[j], y = v[jp];
                        const bool sw = (x > y) == asc;
                        v[j] = sw ? y : x;
                        v[jp] = sw ? x : y;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint64_t other = __shfl_xor_sync(0xffffffffu, v[j], d);
                    const bool asc = (((j * 32 + lane) & k) == 0);
                    const bool lower = (lane & d) == 0;
                    const bool keep_min = (lower == asc);
                    v[j] = keep_min ? (v[j] < other ? v[j] : other) : (v[j] > other ? v[j] : other);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        uint32_t e = j * 32 + lane;
        if (e < m) X[b + e] = v[j];
    }
}

static __device__ __noinline__ void cta_sort_segment(LocalSmem& S, uint32_t n) {
    if (threadIdx.x == 0) {
        S.n_small = 0; S.n_mid = 0; S.n_big = 0;
        push_range(S, 0, n);
    }
    __syncthreads();
    for (;;) {
        const uint32_t nb = S.n_big;
        __syncthreads();
        if (nb == 0) break;
        const uint32_t r = S.big_list[nb - 1];
        __syncthreads();
        if (threadIdx.x == 0) S.n_big = nb - 1;
        __syncthreads();
        cta_counting_pass(S, range_b(r), range_m(r));
    }
    const uint32_t nm = S.n_mid, ns = S.n_small;
    for (uint32_t i = dev::warp_id(); i < nm; i += kLocalThreads / 32) {
        const uint32_t r = S.mid_list[i];
        warp_bitonic_256(S.X, range_b(r), range_m(r));
    }
    for (uint32_t i = threadIdx.x; i < ns; i += kLocalThreads) {
        const uint32_t r = S.small_list[i];
        thread_insertion(S.X, range_b(r), range_m(r));
    }
    __syncthreads();
}


// Dst must provide:
//   __device__ void store(uint64_t pos, uint64_t key, bool has_prev, uint64_t prev) const;
// (has_prev/prev: the preceding key in sorted order when it lies in the same segment).
template <class Dst>
__global__ void __launch_bounds__(kLocalThreads, 1)
    local_sort_kernel(const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
                      const Seg* __restrict__ fin, const uint32_t* __restrict__ n_fin,
                      uint32_t* __restrict__ work, Dst dst) {
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
            for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads) {
                const uint64_t k = src[sg.start + i];
                dst.store(sg.start + i, k, i > 0, k);
            }
            continue;
        }
        for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads) S.X[i] = src[sg.start + i];
        __syncthreads();
        cta_sort_segment(S, n);
        for (uint32_t i = threadIdx.x; i < n; i += kLocalThreads)
            dst.store(sg.start + i, S.X[i], i > 0, i > 0 ? S.X[i - 1] : 0ull);
        __syncthreads();
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
    DevBuf<uint32_t> counters;  // [0]=n_active(a) [1]=n_active(b) [2]=n_fin [3]=work [4]=n_tiles
    DevBuf<uint32_t> tile_seg, tile_idx, seg_tile0;
    DevBuf<uint64_t> seg_elem0;
    size_t n = 0;
    uint32_t max_tiles = 0, max_active = 0, max_fin = 0;
};

void sort_workspace_init(SortWorkspace& ws, size_t n, cudaStream_t s);
size_t local_smem_bytes();

// Runs levels >= 2 until every segment is final; then the caller launches
// local_sort_kernel with its Dst. `key_bits` is the number of significant bits.
void run_segmented_levels(SortWorkspace& ws, int levels_left, cudaStream_t s);

// src_hist feeds the level-1 histogram pass and src_scat the level-1 scatter
// pass; they must produce identical keys (K3 uses the split to capture its
// exception list exactly once).
template <class Src, class Dst>
void msd_sort_split(Src src_hist, Src src_scat, size_t n, int key_bits, Dst dst, SortWorkspace& ws,
                    cudaStream_t s) {
    if (n == 0) return;
    sort_workspace_init(ws, n, s);
    const int bits1 = key_bits < 8 ? (key_bits > 0 ? key_bits : 1) : 8;
    const int shift1 = key_bits - bits1 > 0 ? key_bits - bits1 : 0;
    const unsigned dmask = (1u << bits1) - 1u;
    const uint32_t ntiles = div_up(n, kTile);
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)num_sms() * 4);
    PRG_CUDA(cudaMemsetAsync(ws.counters.get(), 0, 8 * sizeof(uint32_t), s));
    {
        ProfScope prof("sort_l1_hist", s);
        if (Src::kSmem > 48 * 1024)
            PRG_CUDA(cudaFuncSetAttribute(l1_hist_kernel<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)Src::kSmem));
        l1_hist_kernel<Src><<<grid, kTileThreads, Src::kSmem, s>>>(src_hist, n, shift1, dmask, ntiles,
                                                                    ws.hist.get());
        PRG_LAUNCH_CHECK();
        exclusive_scan_u32(ws.hist.get(), ws.off.get(), (size_t)kRadix * ntiles, nullptr, s);
    }
    {
        ProfScope prof("sort_l1_scatter", s);
        const size_t smem = (size_t)kTile * sizeof(uint64_t) + Src::kSmem;
        PRG_CUDA(cudaFuncSetAttribute(l1_scatter_kernel<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        l1_scatter_kernel<Src><<<grid, kTileThreads, smem, s>>>(src_scat, n, shift1, dmask, ntiles,
                                                                ws.off.get(), ws.keys[1].get());
        PRG_LAUNCH_CHECK();
        classify_l1_kernel<<<1, kRadix, 0, s>>>(ws.off.get(), ntiles, n, shift1, shift1 >= 8 ? 8 : shift1,
                                                 ws.lists[0].get(), ws.counters.get() + 0, ws.fin.get(),
                                                 ws.counters.get() + 2);
        PRG_LAUNCH_CHECK();
    }
    {
        ProfScope prof("sort_levels", s);
        run_segmented_levels(ws, (shift1 + 7) / 8, s);
    }
    {
        ProfScope prof("sort_local", s);
        PRG_CUDA(cudaFuncSetAttribute(local_sort_kernel<Dst>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)local_smem_bytes()));
        local_sort_kernel<Dst><<<num_sms(), kLocalThreads, local_smem_bytes(), s>>>(
            ws.keys[0].get(), ws.keys[1].get(), ws.fin.get(), ws.counters.get() + 2, ws.counters.get() + 3, dst);
        PRG_LAUNCH_CHECK();
    }
}

template <class Src, class Dst>
void msd_sort(Src src, size_t n, int key_bits, Dst dst, SortWorkspace& ws, cudaStream_t s) {
    msd_sort_split(src, src, n, key_bits, dst, ws, s);
}

}  // namespace prg::sort
