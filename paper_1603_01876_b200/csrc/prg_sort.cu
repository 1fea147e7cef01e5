#include <cstdlib>
// prg_sort.cu — non-template parts of the MSD radix sort (see prg_sort.cuh).
#include <algorithm>

#include "prg_sort.cuh"

namespace prg::sort {

// ---------------------------------------------------------------------------
// Level bookkeeping
// ---------------------------------------------------------------------------
// Children of one parent are contiguous in key order. Consecutive children
// that fit in shared memory are coalesced into one final segment (up to
// kLocalCap keys) — the local stage sorts any key range, and this keeps the
// count of final segments (and their fixed per-segment cost) low. Children
// larger than the cap become active for the next level (or final, if no key
// bits are left: all their keys are equal).
// The greedy packing (next fit, in key order) is sequential, so thread 0 only
// walks the child sizes and marks, per child, "starts a run" (with the run's
// size once it closes) or "too large" — a tight register loop; the block then
// counts the emitted segments per thread, reserves list slots with one atomic
// per list and writes the segments in parallel. (One thread emitting every
// segment left the rest of the block waiting: barrier stalls 47%, 50-80 us per
// level launch.)
__device__ uint32_t g_coalesce_max = kLocalCap;
// Children of [g_small_min, kSmallCap] keys whose unsorted bits fit a 32-bit
// window (and carry no payload) are kept apart and listed (SmallList) for the
// small-segment merge kernel (local_small_kernel); 0 = off.
__device__ uint32_t g_small_min = 0;
// mode 2: largest joined run (PRG_SMALL_RUNCAP). Measured K1 at S=22 / 24 / 26: 8192 -> 2.35 / 8.42 / 38.7 ms,
// 4096 -> 2.31 / 8.39 / 38.2, 2048 -> 2.29 / 8.29 / 38.2, 1024 -> 2.31 / 8.28 / 37.6, 512 -> 2.36 / 8.35 / 39.3.
__device__ uint32_t g_small_runcap = 1024;

struct EmitScratch {
    uint8_t kind[kRadix];   // 0: joins the open run or empty, 1: starts a run, 2: larger than the cap, 3: small-kernel segment
    uint32_t rsz[kRadix];   // run size, at the run's first child
    uint32_t scan[kRadix / 32 + 1];
    uint32_t base_fin, base_next, base_small;
};

// SmallList::mode 2: where the small kernel applies, children are joined only inside aligned
// digit groups that keep the run's window within 32 bits (gbits low digit bits may vary), and
// every run of at most kSmallCap keys goes to the small list (sorted by three CTA sizes): no
// segment is left to the LSD path. Mode 1: lone children of at least g_small_min keys only.

__device__ void emit_children_block(const uint64_t* child_start, const uint32_t* child_size, int nchild, uint8_t buf,
                                    int next_shift, int next_bits, Seg* __restrict__ next,
                                    uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                    uint32_t* __restrict__ n_fin, EmitScratch& E, SmallList sl, int gbits = 8) {
    const uint32_t cap = (uint32_t)kLocalCap, cmax = g_coalesce_max;
    const uint32_t smin = sl.n_small ? g_small_min : 0u;
    if (threadIdx.x == 0 && smin && sl.mode == 2) {
        uint32_t run = 0;
        int rs = 0;
        for (int d = 0; d < nchild; ++d) {
            const uint32_t sz = child_size[d];
            uint8_t k = 0;
            const bool cut = run && (sz > cap || (sz && ((d >> gbits) != (rs >> gbits) || run + sz > g_small_runcap)));
            if (cut) { E.rsz[rs] = run; E.kind[rs] = run <= (uint32_t)kSmallCap ? 3 : 1; run = 0; }
            if (sz > cap) {
                k = 2;
            } else if (sz) {
                if (run == 0) { rs = d; k = 1; }
                run += sz;
            }
            E.kind[d] = k;
        }
        if (run) { E.rsz[rs] = run; E.kind[rs] = run <= (uint32_t)kSmallCap ? 3 : 1; }
    } else if (threadIdx.x == 0) {
        uint32_t run = 0;
        int rs = 0;
        for (int d = 0; d < nchild; ++d) {
            const uint32_t sz = child_size[d];
            uint8_t k = 0;
            if (sz > cap) {
                if (run) { E.rsz[rs] = run; run = 0; }
                k = 2;
            } else if (smin && sz >= smin && sz <= (uint32_t)kSmallCap && (run == 0 || run + sz > cap)) {
                // A final segment of its own, for the small kernel — only where it does not cut an
                // open run short (a medium child amid tiny ones stays in their run: at S=26 every
                // such cut left two under-filled LSD segments, K1 48.5 -> 52.3 ms).
                if (run) { E.rsz[rs] = run; run = 0; }
                E.rsz[d] = sz;
                k = 3;
            } else if (sz) {
                // PRG_COALESCE_MAX (measurement knob): children at least this large are
                // not joined. Keeping K1's ~2.9 K-key level-2 children apart (all on the
                // 32-bit merge path) measured slower — K1 local 5.58 vs 4.94 ms, the K3
                // transpose's 3.11 vs 2.23 ms: a segment costs ~3.5 K cycles per merge
                // level whatever its size, so fewer, fuller segments win.
                if (run && (run + sz > cap || sz >= cmax || run >= cmax)) { E.rsz[rs] = run; run = 0; }
                if (run == 0) { rs = d; k = 1; }
                run += sz;
            }
            E.kind[d] = k;
        }
        if (run) E.rsz[rs] = run;
    }
    __syncthreads();
    // what this thread's children emit (children tid, tid + blockDim, ...)
    uint32_t nf = 0, nn = 0, ns = 0;
    for (int d = threadIdx.x; d < nchild; d += blockDim.x) {
        const uint8_t k = E.kind[d];
        if (k == 1) ++nf;
        else if (k == 3) ++ns;
        else if (k == 2) {
            if (next_bits) ++nn;
            else nf += (child_size[d] + cap - 1) / cap;
        }
    }
    uint32_t tf, tn, ts = 0;
    uint32_t of = dev::block_excl_scan(nf, E.scan, tf);
    uint32_t on = dev::block_excl_scan(nn, E.scan, tn);
    uint32_t os = smin ? dev::block_excl_scan(ns, E.scan, ts) : 0u;
    if (threadIdx.x == 0) {
        E.base_fin = tf ? atomicAdd(n_fin, tf) : 0u;
        E.base_next = tn ? atomicAdd(n_next, tn) : 0u;
        E.base_small = ts ? atomicAdd(sl.n_small, ts) : 0u;
    }
    __syncthreads();
    of += E.base_fin;
    on += E.base_next;
    os += E.base_small;
    for (int d = threadIdx.x; d < nchild; d += blockDim.x) {
        const uint8_t k = E.kind[d];
        if (k == 0) continue;
        Seg sg;
        sg.start = child_start[d];
        sg.buf = buf;
        if (k == 1 || k == 3) {
            sg.size = E.rsz[d];
            sg.bits = 0;
            sg.shift = 0;
            if (k == 3) fin[sl.cap - 1u - os++] = sg;  // sorted by local_small_kernel
            else fin[of++] = sg;
            continue;
        }
        const uint32_t sz = child_size[d];
        sg.size = sz;
        sg.bits = (uint8_t)next_bits;
        sg.shift = (uint16_t)next_shift;
        if (next_bits) {
            next[on++] = sg;
        } else {
            // no bits left: the keys are equal above the payload, so the child is
            // already in order — handed out in cap-sized pieces so no single CTA
            // streams a huge run
            const uint32_t np = (sz + cap - 1) / cap;
            for (uint32_t q = 0; q < np; ++q) {
                Seg pc = sg;
                pc.start = sg.start + (uint64_t)q * cap;
                pc.size = min(cap, sz - q * cap);
                fin[of++] = pc;
            }
        }
    }
}

__global__ void classify_l1_kernel(const uint32_t* __restrict__ off, uint32_t ntiles, size_t n,
                                   int shift, int bits, Seg* __restrict__ next,
                                   uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                   uint32_t* __restrict__ n_fin) {
    __shared__ uint64_t cst[kRadix];
    __shared__ uint32_t csz[kRadix];
    __shared__ EmitScratch E;
    const int d = threadIdx.x;
    if (d < kRadix) {
        const uint64_t st = off[(size_t)d * ntiles];
        const uint64_t en = d + 1 < kRadix ? off[(size_t)(d + 1) * ntiles] : n;
        cst[d] = st;
        csz[d] = (uint32_t)(en - st);
    }
    __syncthreads();
    emit_children_block(cst, csz, kRadix, 1, shift - bits, bits, next, n_next, fin, n_fin, E, SmallList{});
}

__global__ void build_tiles_kernel(const Seg* __restrict__ active, const uint32_t* __restrict__ n_active,
                                   uint32_t* __restrict__ seg_tile0, uint64_t* __restrict__ seg_elem0,
                                   uint32_t* __restrict__ tile_seg, uint32_t* __restrict__ tile_idx,
                                   uint32_t* __restrict__ n_tiles, uint32_t max_tiles) {
    // Single block, 1024 threads: sequential chunks of 1024 segments. The tile
    // map of a chunk is written by all threads (tile q of the chunk finds its
    // segment by binary search): one thread per segment writing its own tiles
    // left a 1 M-key segment's 128 tiles on one thread.
    __shared__ uint32_t carry_t;
    __shared__ uint64_t carry_e;
    __shared__ uint32_t wt[33];
    __shared__ uint64_t we[33];
    __shared__ uint32_t st0[1025];  // chunk-relative first tile of each segment (+ chunk total)
    const uint32_t na = *n_active;
    if (threadIdx.x == 0) { carry_t = 0; carry_e = 0; }
    __syncthreads();
    for (uint32_t base = 0; base < na; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        uint32_t nt = 0;
        uint64_t ne = 0;
        if (i < na) { ne = active[i].size; nt = (uint32_t)((ne + kTile - 1) / kTile); }
        uint32_t it = dev::warp_incl_scan(nt);
        uint64_t ie = dev::warp_incl_scan(ne);
        if (dev::lane_id() == 31) { wt[dev::warp_id()] = it; we[dev::warp_id()] = ie; }
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t x = threadIdx.x < blockDim.x / 32 ? wt[threadIdx.x] : 0;
            uint64_t y = threadIdx.x < blockDim.x / 32 ? we[threadIdx.x] : 0;
            uint32_t xi = dev::warp_incl_scan(x);
            uint64_t yi = dev::warp_incl_scan(y);
            wt[threadIdx.x] = xi - x;
            we[threadIdx.x] = yi - y;
            if (threadIdx.x == 31) { wt[32] = xi; we[32] = yi; }
        }
        __syncthreads();
        const uint32_t rel = wt[dev::warp_id()] + it - nt;
        const uint32_t t0 = carry_t + rel;
        const uint64_t e0 = carry_e + we[dev::warp_id()] + ie - ne;
        st0[threadIdx.x] = rel;  // rows past na hold the chunk total (nt = 0)
        if (threadIdx.x == 0) st0[blockDim.x] = wt[32];
        if (i < na) {
            seg_tile0[i] = t0;
            seg_elem0[i] = e0;
        }
        __syncthreads();
        const uint32_t chunk_tiles = wt[32];
        const uint32_t nseg = min((uint32_t)blockDim.x, na - base);
        for (uint32_t q = threadIdx.x; q < chunk_tiles; q += blockDim.x) {
            uint32_t lo = 0, hi = nseg - 1;  // last segment with st0 <= q
            while (lo < hi) {
                const uint32_t mid = (lo + hi + 1) >> 1;
                if (st0[mid] <= q) lo = mid; else hi = mid - 1;
            }
            const uint32_t g = carry_t + q;
            if (g < max_tiles) {
                tile_seg[g] = base + lo;
                tile_idx[g] = q - st0[lo];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) { carry_t += wt[32]; carry_e += we[32]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        seg_tile0[na] = carry_t;
        seg_elem0[na] = carry_e;
        *n_tiles = carry_t;
    }
}

__global__ void __launch_bounds__(kTileThreads) seg_hist_kernel(
    const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
    const Seg* __restrict__ active, const uint32_t* __restrict__ seg_tile0,
    const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_idx,
    const uint32_t* __restrict__ n_tiles, uint32_t* __restrict__ hist, uint32_t* __restrict__ next_tile) {
    __shared__ uint32_t h[kRadix];
    __shared__ uint32_t s_t;
    const uint32_t nt = *n_tiles;
    for (;;) {  // tiles handed out dynamically (segment tails make them uneven)
        if (threadIdx.x == 0) s_t = atomicAdd(next_tile, 1u);
        __syncthreads();
        const uint32_t t = s_t;
        if (t >= nt) break;
        const uint32_t si = tile_seg[t], ti = tile_idx[t];
        const Seg sg = active[si];
        const uint64_t* src = sg.buf ? keys1 : keys0;
        const uint32_t seg_nt = seg_tile0[si + 1] - seg_tile0[si];
        for (int i = threadIdx.x; i < kRadix; i += blockDim.x) h[i] = 0;
        __syncthreads();
        const uint64_t base = sg.start + (uint64_t)ti * kTile;
        const int cnt = (int)min((uint64_t)kTile, (uint64_t)sg.size - (uint64_t)ti * kTile);
        const unsigned mask = (1u << sg.bits) - 1u;
        uint64_t k[kTileItems];
#pragma unroll
        for (int j = 0; j < kTileItems; ++j) {
            const int li = j * kTileThreads + threadIdx.x;
            if (li < cnt) k[j] = src[base + li];
        }
#pragma unroll
        for (int j = 0; j < kTileItems; ++j)
            if (j * kTileThreads + (int)threadIdx.x < cnt) atomicAdd(&h[(unsigned)(k[j] >> sg.shift) & mask], 1u);
        __syncthreads();
        // layout: [active seg][digit][tile in seg], packed per segment
        const size_t hb = (size_t)seg_tile0[si] * kRadix;
        for (int d = threadIdx.x; d < kRadix; d += blockDim.x) hist[hb + (size_t)d * seg_nt + ti] = h[d];
        __syncthreads();
    }
}

template <bool kStable>
__global__ void __launch_bounds__(kTileThreads, 2) seg_scatter_kernel(
    const uint64_t* __restrict__ keys0, const uint64_t* __restrict__ keys1,
    uint64_t* __restrict__ out0, uint64_t* __restrict__ out1, const Seg* __restrict__ active,
    const uint32_t* __restrict__ seg_tile0, const uint64_t* __restrict__ seg_elem0,
    const uint32_t* __restrict__ tile_seg, const uint32_t* __restrict__ tile_idx,
    const uint32_t* __restrict__ n_tiles, const uint32_t* __restrict__ off, uint32_t* __restrict__ next_tile) {
    __shared__ uint32_t h[kRadix];
    __shared__ uint32_t lstart[kRadix];
    __shared__ uint64_t gbase[kRadix];
    __shared__ uint32_t scan_tmp[kTileThreads / 32 + 1];
    __shared__ uint32_t s_t;
    extern __shared__ __align__(16) uint64_t skeys[];  // kTile keys (+ stable counters)
    uint32_t* wc = reinterpret_cast<uint32_t*>(skeys + kTile);
    const uint32_t nt = *n_tiles;
    for (;;) {  // tiles handed out dynamically (ncu: SM busy max/avg 1.25 under a static stride)
        if (threadIdx.x == 0) s_t = atomicAdd(next_tile, 1u);
        __syncthreads();
        const uint32_t t = s_t;
        if (t >= nt) break;
        const uint32_t si = tile_seg[t], ti = tile_idx[t];
        const Seg sg = active[si];
        const uint64_t* src = sg.buf ? keys1 : keys0;
        uint64_t* dst = sg.buf ? out0 : out1;
        const uint32_t seg_nt = seg_tile0[si + 1] - seg_tile0[si];
        const uint64_t e0 = seg_elem0[si];
        if (!kStable) {
            for (int i = threadIdx.x; i < kRadix; i += blockDim.x) h[i] = 0;
            __syncthreads();
        }
        const uint64_t base = sg.start + (uint64_t)ti * kTile;
        const int cnt = (int)min((uint64_t)kTile, (uint64_t)sg.size - (uint64_t)ti * kTile);
        const unsigned mask = (1u << sg.bits) - 1u;
        uint64_t k[kTileItems];
        // all 16 loads first (in flight together), then the counting
#pragma unroll
        for (int j = 0; j < kTileItems; ++j) {
            const int li = tile_pos<kStable>(j);
            if (li < cnt) k[j] = src[base + li];
        }
        if (!kStable) {
#pragma unroll
            for (int j = 0; j < kTileItems; ++j)
                if (tile_pos<kStable>(j) < cnt) atomicAdd(&h[(unsigned)(k[j] >> sg.shift) & mask], 1u);
        }
        const size_t hb = (size_t)seg_tile0[si] * kRadix;
        if (kStable) {
            // off is relative to the concatenation of active segments
            if (threadIdx.x < kRadix)
                gbase[threadIdx.x] = sg.start + (off[hb + (size_t)threadIdx.x * seg_nt + ti] - e0);
            stable_tile_scatter<false>(k, cnt, sg.shift, sg.bits, wc, lstart, scan_tmp, skeys);
        } else {
            __syncthreads();
            uint32_t v = threadIdx.x < kRadix ? h[threadIdx.x] : 0u, tot;
            uint32_t ex = dev::block_excl_scan(v, scan_tmp, tot);
            if (threadIdx.x < kRadix) {
                lstart[threadIdx.x] = ex;
                h[threadIdx.x] = ex;  // per-digit cursor
                gbase[threadIdx.x] = sg.start + (off[hb + (size_t)threadIdx.x * seg_nt + ti] - e0);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kTileItems; ++j) {
                int li = j * kTileThreads + threadIdx.x;
                if (li < cnt) {
                    const uint32_t slot = atomicAdd(&h[(unsigned)(k[j] >> sg.shift) & mask], 1u);
                    PRG_DCHECK(slot < (uint32_t)cnt);
                    skeys[slot] = k[j];
                }
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < cnt; i += kTileThreads) {
            uint64_t key = skeys[i];
            unsigned d = (unsigned)(key >> sg.shift) & mask;
            PRG_DCHECK(gbase[d] + (i - lstart[d]) >= sg.start && gbase[d] + (i - lstart[d]) < sg.start + sg.size);
            dst[gbase[d] + (i - lstart[d])] = key;
        }
        __syncthreads();
    }
}

__global__ void classify_kernel(const Seg* __restrict__ active, const uint32_t* __restrict__ n_active,
                                const uint32_t* __restrict__ seg_tile0,
                                const uint64_t* __restrict__ seg_elem0,
                                const uint32_t* __restrict__ off, Seg* __restrict__ next,
                                uint32_t* __restrict__ n_next, Seg* __restrict__ fin,
                                uint32_t* __restrict__ n_fin, int floor_bit, SmallList small) {
    __shared__ uint64_t cst[kRadix];
    __shared__ uint32_t csz[kRadix];
    __shared__ EmitScratch E;
    const uint32_t na = *n_active;
    for (uint32_t si = blockIdx.x; si < na; si += gridDim.x) {
        const Seg sg = active[si];
        const uint32_t seg_nt = seg_tile0[si + 1] - seg_tile0[si];
        const size_t hb = (size_t)seg_tile0[si] * kRadix;
        const uint64_t e0 = seg_elem0[si];
        const int nd = 1 << sg.bits;
        for (int d = threadIdx.x; d < nd; d += blockDim.x) {
            const uint64_t st = off[hb + (size_t)d * seg_nt] - e0;
            const uint64_t en = d + 1 < nd ? off[hb + (size_t)(d + 1) * seg_nt] - e0 : sg.size;
            cst[d] = sg.start + st;
            csz[d] = (uint32_t)(en - st);
        }
        __syncthreads();
        const int rem = sg.shift - floor_bit;
        const int nb = rem >= 8 ? 8 : rem;
        emit_children_block(cst, csz, nd, (uint8_t)(sg.buf ^ 1), sg.shift - nb, nb, next, n_next, fin, n_fin, E,
                            (floor_bit == 0 && rem > 0 && rem <= 32) ? small : SmallList{}, min(8, 32 - rem));
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
size_t local_smem_bytes() { return sizeof(LocalSmem); }
int sort_grid_mult(int which) {
    static int g1 = -1, g2 = -1;
    if (g1 < 0) {
        const char* e1 = getenv("PRG_SORT_GRID1");
        const char* e2 = getenv("PRG_SORT_GRID2");
        g1 = e1 ? std::max(1, atoi(e1)) : 4;
        g2 = e2 ? std::max(1, atoi(e2)) : 4;
    }
    return which == 1 ? g1 : g2;
}
int local_small_min() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PRG_SMALL_MIN");
        v = e ? atoi(e) : 1024;
        v = v <= 0 ? 0 : std::max(v, 256);  // below ~512 keys a 256-thread CTA is mostly idle
    }
    return v;
}
int local_small_mode(size_t n) {
    static int v = -1;  // PRG_SMALL_MODE=1/2 forces a mode; default: by input size
    if (v < 0) {
        const char* e = getenv("PRG_SMALL_MODE");
        v = e ? atoi(e) : 0;
    }
    // the three launches of mode 2 cost ~30 us: K1 (L2 flushed) at 2^20 keys 0.33 (mode 1) vs 0.38 ms,
    // 2^22 keys 0.515 vs 0.507, 2^24 keys 0.883 vs 0.853
    return v == 1 || v == 2 ? v : (n >= (size_t(1) << 22) ? 2 : 1);
}
int local_merge_span() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PRG_MERGE_SPAN");
        const char* w = getenv("PRG_WARP_LEVELS");  // merge levels done in registers by warp shuffles (0..5)
        v = (e ? atoi(e) : 16) & 0x1ff;
        v |= std::min(5, std::max(0, w ? atoi(w) : 5)) << 12;
    }
    return v;
}

void sort_workspace_init(SortWorkspace& ws, size_t n, cudaStream_t s) {
    static bool coalesce_set = false;  // PRG_COALESCE_MAX: children at least this large are not coalesced
    if (!coalesce_set) {
        const char* e = getenv("PRG_COALESCE_MAX");
        const uint32_t v = e ? (uint32_t)atoi(e) : (uint32_t)kLocalCap;
        PRG_CUDA(cudaMemcpyToSymbol(g_coalesce_max, &v, sizeof(v)));
        coalesce_set = true;
    }
    static bool small_set = false;  // PRG_SMALL_MIN: smallest child given to the small-segment kernel (0 = off)
    if (!small_set) {
        const uint32_t v = (uint32_t)local_small_min();
        PRG_CUDA(cudaMemcpyToSymbol(g_small_min, &v, sizeof(v)));
        const char* rc = getenv("PRG_SMALL_RUNCAP");
        const uint32_t rcv = rc ? (uint32_t)std::min(std::max(atoi(rc), 256), kLocalCap) : 1024u;
        PRG_CUDA(cudaMemcpyToSymbol(g_small_runcap, &rcv, sizeof(rcv)));

        small_set = true;
    }
    if (ws.n >= n && ws.keys[0].get()) return;
    ws.n = n;
    const uint32_t t1 = div_up(n, kTile);
    ws.max_active = (uint32_t)(n / kLocalCap + 2);
    ws.max_tiles = t1 + ws.max_active;
    ws.max_fin = (uint32_t)std::min<uint64_t>(n + kRadix, (uint64_t)kRadix * ws.max_active + kRadix);
    ws.keys[0] = DevBuf<uint64_t>(n, s);
    ws.keys[1] = DevBuf<uint64_t>(n, s);
    const size_t hsz = (size_t)kRadix * ws.max_tiles;
    ws.hist = DevBuf<uint32_t>(hsz, s);
    ws.off = DevBuf<uint32_t>(hsz, s);
    ws.lists[0] = DevBuf<Seg>(ws.max_active, s);
    ws.lists[1] = DevBuf<Seg>(ws.max_active, s);
    ws.fin = DevBuf<Seg>(ws.max_fin, s);
    ws.counters = DevBuf<uint32_t>(kCounters, s);
    ws.tile_seg = DevBuf<uint32_t>(ws.max_tiles, s);
    ws.tile_idx = DevBuf<uint32_t>(ws.max_tiles, s);
    ws.seg_tile0 = DevBuf<uint32_t>(ws.max_active + 1, s);
    ws.seg_elem0 = DevBuf<uint64_t>(ws.max_active + 1, s);
}

void run_segmented_levels(SortWorkspace& ws, int levels_left, int floor_bit, bool stable, cudaStream_t s) {
    SmallList small;  // [41] = count of small-kernel segments
    if (!stable && floor_bit == 0 && local_small_min() > 0)
        small = SmallList{ws.counters.get() + 41, ws.max_fin, local_small_mode(ws.n_sorting)};
    static bool attr_set = false;
    const size_t smem = (size_t)kTile * sizeof(uint64_t) + (stable ? kStableScratch : 0);
    if (!attr_set) {
        PRG_CUDA(cudaFuncSetAttribute(seg_scatter_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((size_t)kTile * sizeof(uint64_t))));
        PRG_CUDA(cudaFuncSetAttribute(seg_scatter_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((size_t)kTile * sizeof(uint64_t) + kStableScratch)));
        attr_set = true;
    }
    const unsigned grid = (unsigned)num_sms() * sort_grid_mult(2);
    uint32_t* cnt = ws.counters.get();
    for (int lvl = 0; lvl < levels_left; ++lvl) {
        const int a = lvl & 1;
        Seg* act = ws.lists[a].get();
        Seg* nxt = ws.lists[a ^ 1].get();
        uint32_t* n_act = cnt + a;
        uint32_t* n_nxt = cnt + (a ^ 1);
        PRG_CUDA(cudaMemsetAsync(n_nxt, 0, sizeof(uint32_t), s));
        build_tiles_kernel<<<1, 1024, 0, s>>>(act, n_act, ws.seg_tile0.get(), ws.seg_elem0.get(),
                                              ws.tile_seg.get(), ws.tile_idx.get(), cnt + 4,
                                              ws.max_tiles);
        PRG_LAUNCH_CHECK();
        // Only the used prefix (n_tiles x kRadix, every entry written by
        // seg_hist) is scanned; the count stays on the device.
        const size_t hsz = (size_t)kRadix * ws.max_tiles;
        seg_hist_kernel<<<grid, kTileThreads, 0, s>>>(ws.keys[0].get(), ws.keys[1].get(), act,
                                                      ws.seg_tile0.get(), ws.tile_seg.get(),
                                                      ws.tile_idx.get(), cnt + 4, ws.hist.get(), cnt + 8 + 2 * lvl);
        PRG_LAUNCH_CHECK();
        exclusive_scan_u32_prefix(ws.hist.get(), ws.off.get(), hsz, cnt + 4, kRadix, s);
        if (stable)
            seg_scatter_kernel<true><<<grid, kTileThreads, smem, s>>>(
                ws.keys[0].get(), ws.keys[1].get(), ws.keys[0].get(), ws.keys[1].get(), act,
                ws.seg_tile0.get(), ws.seg_elem0.get(), ws.tile_seg.get(), ws.tile_idx.get(), cnt + 4,
                ws.off.get(), cnt + 9 + 2 * lvl);
        else
            seg_scatter_kernel<false><<<grid, kTileThreads, smem, s>>>(
                ws.keys[0].get(), ws.keys[1].get(), ws.keys[0].get(), ws.keys[1].get(), act,
                ws.seg_tile0.get(), ws.seg_elem0.get(), ws.tile_seg.get(), ws.tile_idx.get(), cnt + 4,
                ws.off.get(), cnt + 9 + 2 * lvl);
        PRG_LAUNCH_CHECK();
        // One segment's children are emitted by one thread (greedy run packing is
        // sequential): small blocks, many of them, so deep levels with thousands
        // of segments are not serialised on 4 blocks per SM (0.2 ms per level).
        classify_kernel<<<(unsigned)num_sms() * 32, 64, 0, s>>>(act, n_act, ws.seg_tile0.get(), ws.seg_elem0.get(),
                                                                ws.off.get(), nxt, n_nxt, ws.fin.get(), cnt + 2,
                                                                floor_bit, small);
        PRG_LAUNCH_CHECK();
    }
}

}  // namespace prg::sort

PRG_CHECK_QUERY(sort)
