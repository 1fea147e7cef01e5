// prg_k2.cu — K2: adjacency build + in-degree + column filter + row
// normalisation, fused over a device edge list sorted by start vertex.
//
// Replaces the core of prpipe::run_kernel2 (src/kernel2_filter.cpp:154-168):
//   build_adjacency / build_from  (:12-54)   — RLE of (u,v) runs into counts
//   in_degree                     (:101-106) — d_in[v] += count
//   zero_columns                  (:108-132) — drop columns with d_in == max or 1
//   row_normalize                 (:134-152) — value = count / filtered row sum
// Output: CSR with u32 row offsets / cols and f64 values, plus the pre-filter
// d_in. Values are one IEEE division of the same two integers the reference
// divides, so they are bit-identical.
//
// Passes (S=24: M=268M edges):
//   A  read edges once (TMA ring, 2048-edge tiles): validate labels and order,
//      count unique (u,v), warp-aggregated d_in atomics
//   -  max(d_in), keep bitmask (N bits)
//   B  read edges again (1536-edge tiles, one per CTA): keep-bit gather, in-tile run lengths / row sums in SMEM,
//      kept-entry positions by decoupled look-back, write cols/values/row offsets
//   F  fix-ups for the few rows that span tiles (run continuation counts, then
//      divide those rows by their row sums accumulated across tiles)
#include "prg_internal.cuh"

namespace prg {

namespace {

#ifndef PRG_K2B_T  // pass-B shape, S=24 (pass B / whole CSR filter; fix-ups as of their round-1 form):
                   // 512x8 3.66 / 6.22 ms, 512x16 4.79, 512x4 3.52 / 6.20, 256x8 3.47 / 6.15,
                   // 256x4 3.32 / 6.17 (more tile-spanning rows to fix up), 128x8 3.56 / 6.42,
                   // 128x16 5.21; after the fix-up rework: 256x8 3.48 / 5.97, 256x6 3.30 / 5.84,
                   // 384x8 3.60, 192x8 3.51, 256x12 3.92 (tools/build_variant.py)
#define PRG_K2B_T 256
#endif
#ifndef PRG_K2B_I
#define PRG_K2B_I 6
#endif
constexpr int kT = PRG_K2B_T;   // threads per CTA
constexpr int kI = PRG_K2B_I;   // edges per thread
constexpr int kTE = kT * kI;    // edges per tile

// SMEM arrays indexed by tile position are padded one word per 32: the
// blocked per-thread view (thread t reads positions 8t..8t+7) is then free of
// bank conflicts (ncu: 8-way before).
__device__ __forceinline__ int sp(int l) { return l + (l >> 5); }
constexpr int kTEP = kTE + kTE / 32;


struct Scan3 {
    int32_t rs, hd;
    uint32_t kh;
};

struct PassBSmem {
    uint32_t su[kTEP];
    uint32_t sv[kTEP];
    // per head (local index, padded): kept-edge count of the row in bits 16..31
    // (row heads), edge count of the (u,v) run in bits 0..15 (run heads); both <= kTE
    uint32_t rr[kTEP];
    Scan3 scan3[kT / 32 + 1];
    uint32_t prev_u, prev_v, next_u;
    int has_prev, has_next;
    uint32_t tile;
    uint64_t tile_base;
    uint32_t first_row_part, first_run_part;
};

// The three block scans pass B needs in one pass (two barriers instead of six):
// exclusive max-scans of the last row start and last run head per thread (-1 =
// none) and the exclusive sum-scan of kept heads. Totals: the tile's last row
// start / last run head and its kept-head count.
__device__ __forceinline__ Scan3 block_excl_scan3(Scan3 v, Scan3* smem, Scan3& total) {
    const unsigned w = dev::warp_id(), l = dev::lane_id(), nw = blockDim.x >> 5;
    Scan3 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t a = __shfl_up_sync(0xffffffffu, inc.rs, d), b = __shfl_up_sync(0xffffffffu, inc.hd, d);
        const uint32_t c = __shfl_up_sync(0xffffffffu, inc.kh, d);
        if ((int)l >= d) { inc.rs = max(inc.rs, a); inc.hd = max(inc.hd, b); inc.kh += c; }
    }
    Scan3 ex;
    ex.rs = __shfl_up_sync(0xffffffffu, inc.rs, 1);
    ex.hd = __shfl_up_sync(0xffffffffu, inc.hd, 1);
    ex.kh = inc.kh - v.kh;
    if (l == 0) { ex.rs = -1; ex.hd = -1; }
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        Scan3 x = l < nw ? smem[l] : Scan3{-1, -1, 0u};
        Scan3 xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t a = __shfl_up_sync(0xffffffffu, xi.rs, d), b = __shfl_up_sync(0xffffffffu, xi.hd, d);
            const uint32_t c = __shfl_up_sync(0xffffffffu, xi.kh, d);
            if ((int)l >= d) { xi.rs = max(xi.rs, a); xi.hd = max(xi.hd, b); xi.kh += c; }
        }
        Scan3 xe;
        xe.rs = __shfl_up_sync(0xffffffffu, xi.rs, 1);
        xe.hd = __shfl_up_sync(0xffffffffu, xi.hd, 1);
        xe.kh = xi.kh - x.kh;
        if (l == 0) { xe.rs = -1; xe.hd = -1; }
        if (l < nw) smem[l] = xe;
        if (l == nw - 1) smem[nw] = xi;
    }
    __syncthreads();
    const Scan3 wp = smem[w];
    total = smem[nw];
    return Scan3{max(wp.rs, ex.rs), max(wp.hd, ex.hd), wp.kh + ex.kh};
}

// ---------------------------------------------------------------------------
// Pass A
// ---------------------------------------------------------------------------
// Pass A keeps edges in registers: edge l is compared with edge l-1 through a
// warp shuffle; lane 0 takes its predecessor from the previous warp's lane 31
// via a small SMEM exchange.
__global__ void __launch_bounds__(kT) k2_pass_a(const longlong2* __restrict__ uv, int64_t m, int64_t n,
                                                uint32_t* __restrict__ d_in, uint32_t* __restrict__ err,
                                                unsigned long long* __restrict__ nnz_raw,
                                                uint32_t ntiles, uint32_t* __restrict__ next_tile, int flags) {
    __shared__ uint32_t red[kT / 32];
    __shared__ longlong2 last[kI][kT / 32];  // lane 31 of each (row j, warp)
    __shared__ longlong2 before;             // edge base-1
    __shared__ uint32_t s_t;
    uint32_t my_err = 0;
    const unsigned lane = dev::lane_id(), w = dev::warp_id();
    // Tiles handed out dynamically: their d_in atomics meet very different
    // contention (ncu: SM busy 2.8M-5.8M cycles under a static stride).
    for (;;) {
        if (threadIdx.x == 0) s_t = atomicAdd(next_tile, 1u);
        __syncthreads();
        const uint32_t t = s_t;
        if (t >= ntiles) break;
        const int64_t base = (int64_t)t * kTE;
        const int cnt = (int)min((int64_t)kTE, m - base);
        longlong2 p[kI];
#pragma unroll
        for (int j = 0; j < kI; ++j) {
            const int l = j * kT + threadIdx.x;
            // flags & 1: edges streamed with evict-first loads, so the d_in lines the
            // atomics hit stay in L2 instead of being written back and re-fetched
            p[j] = l < cnt ? ((flags & 1) ? __ldcs(uv + base + l) : uv[base + l]) : make_longlong2(0, 0);
            if (lane == 31) last[j][w] = p[j];
        }
        if (threadIdx.x == 0) before = base > 0 ? uv[base - 1] : make_longlong2(0, 0);
        __syncthreads();
        uint32_t heads = 0;
#pragma unroll
        for (int j = 0; j < kI; ++j) {
            const int l = j * kT + threadIdx.x;
            long long px = __shfl_up_sync(0xffffffffu, p[j].x, 1);
            long long py = __shfl_up_sync(0xffffffffu, p[j].y, 1);
            if (lane == 0) {
                const longlong2 q = w ? last[j][w - 1] : (j ? last[j - 1][kT / 32 - 1] : before);
                px = q.x;
                py = q.y;
            }
            // Warp-aggregated in-degree: duplicate edges are adjacent (sorted
            // input), so a run of equal edges within the warp's 32 lanes adds
            // its length with one atomic from its first lane.
            const bool valid = l < cnt;
            const bool same = valid && (lane > 0 || base + l > 0) && p[j].x == px && p[j].y == py;
            const unsigned eqm = __ballot_sync(0xffffffffu, same);
            if (valid) {
                const bool ok = p[j].x >= 1 && p[j].x <= n && p[j].y >= 1 && p[j].y <= n;
                if (!ok) my_err |= kErrLabelRange;
                else if (!same || lane == 0) {
                    // lanes after me that continue my run: the set bits of eqm above my lane, up to the first gap
                    const unsigned after = ~(eqm >> lane >> 1) & (0x7fffffffu >> lane);
                    const uint32_t len = 1u + (after ? (uint32_t)(__ffs(after) - 1) : 31u - lane);
                    atomicAdd(&d_in[(uint32_t)(p[j].y - 1)], len);
                }
                if (base + l == 0) {
                    heads++;
                } else {
                    const long long pu = px, pv = py;
                    if (p[j].x < pu) my_err |= kErrUnsorted;
                    else if (p[j].x == pu && p[j].y < pv) my_err |= kErrNotCanonical;
                    heads += (p[j].x != pu || p[j].y != pv);
                }
            }
        }
        heads = dev::warp_sum(heads);
        if (lane == 0) red[dev::warp_id()] = heads;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t x = threadIdx.x < kT / 32 ? red[threadIdx.x] : 0;
            x = dev::warp_sum(x);
            if (threadIdx.x == 0) atomicAdd(nnz_raw, (unsigned long long)x);
        }
        __syncthreads();
    }
    my_err = __reduce_or_sync(0xffffffffu, my_err);
    if (lane == 0 && my_err) atomicOr(err, my_err);
}

__global__ void k2_max_kernel(const uint32_t* __restrict__ d_in, int64_t n, uint32_t* __restrict__ out) {
    uint32_t mx = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, d_in[i]);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (dev::lane_id() == 0) atomicMax(out, mx);
}

// keep(c) = d_in[c] != max && d_in[c] != 1   (kernel2_filter.cpp:118-121)
__global__ void k2_keep_kernel(const uint32_t* __restrict__ d_in, int64_t n, const uint32_t* __restrict__ maxp,
                               uint32_t* __restrict__ keepbits) {
    const uint32_t mx = *maxp;
    const int64_t nw = (n + 31) / 32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw * 32; i += (int64_t)gridDim.x * blockDim.x) {
        bool keep = false;
        if (i < n) { const uint32_t d = d_in[i]; keep = d != mx && d != 1u; }
        const uint32_t word = __ballot_sync(0xffffffffu, keep);
        if (dev::lane_id() == 0) keepbits[i >> 5] = word;
    }
}

// ---------------------------------------------------------------------------
// Pass B
// ---------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kT) k2_pass_b(
    const longlong2* __restrict__ uv, int64_t m, int64_t n, const uint32_t* __restrict__ keepbits,
    uint32_t* __restrict__ row_offsets, uint32_t* __restrict__ cols, double* __restrict__ values,
    unsigned long long* __restrict__ tile_status, uint32_t* __restrict__ tile_counter,
    uint32_t* __restrict__ dout_f, uint32_t* __restrict__ fix_rows, uint32_t* __restrict__ n_fix,
    uint32_t* __restrict__ cont_p, uint32_t* __restrict__ cont_c, unsigned long long* __restrict__ nnz_out,
    bool normalize, int flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassBSmem& S = *reinterpret_cast<PassBSmem*>(smem_raw);
    const unsigned tid = threadIdx.x;
    if (tid == 0) S.tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t t = S.tile;
    const int64_t base = (int64_t)t * kTE;
    const int cnt = (int)min((int64_t)kTE, m - base);
#pragma unroll
    for (int j = 0; j < kI; ++j) {
        const int l = j * kT + tid;
        if (l < cnt) {
            const longlong2 p = (flags & 1) ? __ldcs(uv + base + l) : uv[base + l];
            const uint32_t v = (uint32_t)(p.y - 1);
            // keep bit fetched here, alongside the edge loads; carried in bit 31
            const uint32_t kp = (keepbits[v >> 5] >> (v & 31)) & 1u;
            S.su[sp(l)] = (uint32_t)(p.x - 1);
            S.sv[sp(l)] = v | (kp << 31);
        }
        if (l < kTE) S.rr[sp(l)] = 0;
    }
    if (tid == 0) {
        S.has_prev = base > 0;
        if (base > 0) {
            const longlong2 p = uv[base - 1];
            S.prev_u = (uint32_t)(p.x - 1);
            S.prev_v = (uint32_t)(p.y - 1);
        }
        S.has_next = base + cnt < m;
        if (base + cnt < m) S.next_u = (uint32_t)(uv[base + cnt].x - 1);
        S.first_row_part = 0;
        S.first_run_part = 0;
    }
    __syncthreads();

    // Blocked per-thread view: edges l0 .. l0+kI-1.
    const int l0 = tid * kI;
    uint32_t fl_rs = 0, fl_hd = 0, fl_kp = 0;  // bit k per item
    int32_t last_rs = -1, last_hd = -1;
    uint32_t nkh = 0;
#pragma unroll
    for (int k = 0; k < kI; ++k) {
        const int l = l0 + k;
        if (l < cnt) {
            const uint32_t u = S.su[sp(l)], vk = S.sv[sp(l)], v = vk & 0x7fffffffu;
            bool rs, hd;
            if (l > 0) { rs = u != S.su[sp(l - 1)]; hd = rs || v != (S.sv[sp(l - 1)] & 0x7fffffffu); }
            else if (S.has_prev) { rs = u != S.prev_u; hd = rs || v != S.prev_v; }
            else { rs = true; hd = true; }
            const bool kp = vk >> 31;
            fl_rs |= (uint32_t)rs << k;
            fl_hd |= (uint32_t)hd << k;
            fl_kp |= (uint32_t)kp << k;
            if (rs) last_rs = l;
            if (hd) last_hd = l;
            nkh += (hd && kp);
        }
    }
    Scan3 tot3;
    const Scan3 ex3 = block_excl_scan3(Scan3{last_rs, last_hd, nkh}, S.scan3, tot3);
    const int32_t carry_rs = ex3.rs, carry_hd = ex3.hd, rs_last_all = tot3.rs;
    const uint32_t kh_excl = ex3.kh, tile_kh = tot3.kh;

    // The tile's aggregate is published now; the look-back runs after the row
    // sums (below), when the predecessors have mostly published inclusive
    // prefixes: ncu had 17% of pass B's stall samples at the barrier waiting
    // for warp 0's look-back.
    if (tid == 0) atomicExch(&tile_status[t], (t == 0 ? kFlagInc : kFlagAgg) | tile_kh);

    // Row sums (kept edges) and run lengths (all edges) into SMEM per head.
    {
        int32_t rh = carry_rs, rn = carry_hd;
        uint32_t acc_row = 0, acc_run = 0;
#pragma unroll
        for (int k = 0; k < kI; ++k) {
            const int l = l0 + k;
            if (l < cnt) {
                if ((fl_rs >> k) & 1u) {
                    if (acc_row) { if (rh >= 0) atomicAdd(&S.rr[sp(rh)], acc_row << 16); else atomicAdd(&S.first_row_part, acc_row); }
                    acc_row = 0;
                    rh = l;
                }
                if ((fl_hd >> k) & 1u) {
                    if (acc_run) { if (rn >= 0) atomicAdd(&S.rr[sp(rn)], acc_run); else atomicAdd(&S.first_run_part, acc_run); }
                    acc_run = 0;
                    rn = l;
                }
                acc_row += (fl_kp >> k) & 1u;
                acc_run += 1;
            }
        }
        if (acc_row) { if (rh >= 0) atomicAdd(&S.rr[sp(rh)], acc_row << 16); else atomicAdd(&S.first_row_part, acc_row); }
        if (acc_run) { if (rn >= 0) atomicAdd(&S.rr[sp(rn)], acc_run); else atomicAdd(&S.first_run_part, acc_run); }
    }
    // Decoupled look-back for the tile's global kept-entry base, by warp 0:
    // 32 predecessors are inspected at once (sum of aggregates up to the
    // nearest inclusive prefix).
    if (tid < 32) {
        uint64_t excl = 0;
        if (t != 0) {
            for (int64_t k = (int64_t)t - 1;; k -= 32) {
                const int64_t idx = k - (int64_t)tid;
                uint64_t st = kFlagInc;  // below tile 0: an empty inclusive prefix
                if (idx >= 0) {
                    do {
                        st = *((volatile unsigned long long*)&tile_status[idx]);
                    } while ((st & ~kValMask) == 0);
                }
                const unsigned incm = __ballot_sync(0xffffffffu, (st & ~kValMask) == kFlagInc);
                const int first = incm ? __ffs(incm) - 1 : 32;
                uint64_t v = (int)tid <= first ? (st & kValMask) : 0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                excl += v;
                if (incm) break;
            }
            if (tid == 0) atomicExch(&tile_status[t], kFlagInc | (excl + tile_kh));
        }
        if (tid == 0) S.tile_base = excl;
    }
    __syncthreads();
    const uint64_t tile_base = S.tile_base;
    const bool last_spans = S.has_next && S.su[sp(cnt - 1)] == S.next_u;
    const bool first_spans = S.has_prev && S.su[sp(0)] == S.prev_u;
    const int32_t rh_last = rs_last_all;  // local head of the tile's last row (-1: began earlier)

    // Emit entries and row offsets. Positions fit in 32 bits (nnz < 2^32). A
    // count of 1 — nearly every entry — takes the row's 1/d_out, which is the
    // same IEEE division the reference performs; it is computed once per row
    // and thread, other counts divide themselves (bit-exact either way).
    {
        int32_t rh = carry_rs, inv_row = -2;
        double inv = 0.0;
        uint32_t pos = (uint32_t)(tile_base + kh_excl);
        const bool stream = flags & 2;
#pragma unroll
        for (int k = 0; k < kI; ++k) {
            const int l = l0 + k;
            if (l < cnt) {
                const uint32_t u = S.su[sp(l)], v = S.sv[sp(l)] & 0x7fffffffu;
                if ((fl_rs >> k) & 1u) {
                    rh = l;
                    const int64_t pu = l > 0 ? (int64_t)S.su[sp(l - 1)] : (S.has_prev ? (int64_t)S.prev_u : -1);
                    PRG_DCHECK((int64_t)u < n && pu < (int64_t)u);
                    for (int64_t r = pu + 1; r <= (int64_t)u; ++r) row_offsets[r] = pos;
                }
                if (((fl_hd >> k) & 1u) && ((fl_kp >> k) & 1u)) {
                    const uint32_t cnt_run = S.rr[sp(l)] & 0xffffu;
                    const double c = (double)cnt_run;
                    const bool spanning = rh < 0 || (last_spans && rh == rh_last);
                    double val = c;
                    if (!spanning && normalize) {
                        const double d = (double)(S.rr[sp(rh)] >> 16);
                        if (cnt_run == 1u) {
                            if (inv_row != rh) { inv = 1.0 / d; inv_row = rh; }
                            val = inv;
                        } else {
                            val = c / d;
                        }
                    }
                    PRG_DCHECK((int64_t)pos < m && v < (uint64_t)n);
                    if (stream) {  // streaming stores: the outputs are not re-read by this pass
                        __stcs(cols + pos, v);
                        __stcs(values + pos, val);
                    } else {
                        cols[pos] = v;
                        values[pos] = val;
                    }
                    ++pos;
                }
            }
        }
    }
    if (tid == 0) {
        // Rows crossing tile edges: partial kept-edge sums go to dout_f.
        if (first_spans && S.first_row_part) atomicAdd(&dout_f[S.su[sp(0)]], S.first_row_part);
        if (last_spans && rh_last >= 0) {
            atomicAdd(&dout_f[S.su[sp(cnt - 1)]], S.rr[sp(rh_last)] >> 16);
            fix_rows[atomicAdd(n_fix, 1u)] = S.su[sp(cnt - 1)];
        }
        // A run continuing from the previous tile: its head entry is the last
        // kept entry before this tile (position tile_base-1) when kept.
        const bool kp0 = S.sv[sp(0)] >> 31;
        if (S.first_run_part && kp0) { cont_p[t] = (uint32_t)(tile_base - 1); cont_c[t] = S.first_run_part; }
        else { cont_p[t] = 0; cont_c[t] = 0; }
        if (base + cnt == m) *nnz_out = tile_base + tile_kh;
    }
    if (base + cnt == m) {
        const uint64_t total = tile_base + tile_kh;
        for (int64_t r = (int64_t)S.su[sp(cnt - 1)] + 1 + tid; r <= n; r += kT) row_offsets[r] = (uint32_t)total;
    }
}

__global__ void k2_fix_runs(const uint32_t* __restrict__ cont_p, const uint32_t* __restrict__ cont_c,
                            uint32_t ntiles, double* __restrict__ values) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x)
        if (cont_c[t]) atomicAdd(&values[cont_p[t]], (double)cont_c[t]);  // exact: integers
}

// Rows that span tiles (their row sums were accumulated across tiles) are
// divided here. Work is split into tasks of <= kFixChunk entries so hub rows
// (10^5 entries) spread over the GPU: per-row task counts, a device-wide scan
// of the used prefix, each row writes its (row, chunk) tasks, then one warp per
// task divides its entries (a one-block scan of the task counts took ~0.19 ms
// at S=24 for ~65 K spanning rows).
constexpr uint32_t kFixChunk = 1024;
__global__ void k2_fix_count(const uint32_t* __restrict__ fix_rows, const uint32_t* __restrict__ n_fix,
                             const uint32_t* __restrict__ row_offsets, uint32_t* __restrict__ nc) {
    const uint32_t nf = *n_fix;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        const uint32_t r = fix_rows[i];
        nc[i] = (row_offsets[r + 1] - row_offsets[r] + kFixChunk - 1) / kFixChunk;
    }
}
__global__ void k2_fix_emit(const uint32_t* __restrict__ nc, const uint32_t* __restrict__ base,
                            const uint32_t* __restrict__ n_fix, uint64_t* __restrict__ task_row,
                            uint32_t* __restrict__ n_tasks) {
    const uint32_t nf = *n_fix;
    if (nf == 0 && blockIdx.x == 0 && threadIdx.x == 0) *n_tasks = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        const uint32_t b = base[i], k = nc[i];
        for (uint32_t c = 0; c < k; ++c) task_row[b + c] = ((uint64_t)i << 32) | c;  // (fix row, chunk)
        if (i + 1 == nf) *n_tasks = b + k;
    }
}
__global__ void k2_fix_rows(const uint32_t* __restrict__ fix_rows, const uint64_t* __restrict__ task_row,
                            const uint32_t* __restrict__ n_tasks, const uint32_t* __restrict__ row_offsets,
                            const uint32_t* __restrict__ dout_f, double* __restrict__ values) {
    const uint32_t nt = *n_tasks;
    const uint32_t lane = dev::lane_id();
    for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nt; q += (gridDim.x * blockDim.x) >> 5) {
        const uint64_t tk = task_row[q];
        const uint32_t i = (uint32_t)(tk >> 32), c = (uint32_t)tk;
        const uint32_t r = fix_rows[i];
        const uint32_t b = row_offsets[r] + c * kFixChunk;
        const uint32_t e = min(row_offsets[r + 1], b + kFixChunk);
        const double d = (double)dout_f[r];
        const double inv = 1.0 / d;  // count 1 -> 1/d_out: the same IEEE division as c / d
        // 8 entries per lane in flight (a dependent load -> divide -> store per
        // step left the kernel latency-bound: 0.39 ms at S=24)
        for (uint32_t p0 = b + lane; p0 < e; p0 += 32 * 8) {
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t p = p0 + 32 * k;
                v[k] = p < e ? values[p] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t p = p0 + 32 * k;
                if (p < e) values[p] = v[k] == 1.0 ? inv : v[k] / d;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Pass A over a TMA ring. Persistent CTAs of 256 threads; tiles of 2048 edges
// (32 KB) arrive by cp.async.bulk into a ring of kStages shared-memory stages,
// claimed dynamically and prefetched kStages-1 ahead, so HBM streams while the
// current tile's atomics are issued (2.21 -> 1.96 ms at S=24; the floor is the
// L2 atomic rate: 2^28 scattered REDs into 2^24 counters take 1.53 ms alone,
// tools/microbench/atomics.cu). Each warp owns 256 consecutive edges of a tile
// as 8 rows of 32 lanes (conflict-free 16-byte shared loads; a predecessor is
// a shuffle away).
// Pass B in the same persistent TMA form measured slower (6.6 ms vs 3.7 ms):
// with a decoupled look-back, a round of concurrently started tiles makes every
// tile sum up to a round of aggregates (dynamic claims made a stage ahead were
// worse still, 12 ms) — the one-tile-per-CTA launch below staggers tiles naturally.
// ---------------------------------------------------------------------------
constexpr int kST = 256;               // threads per CTA
constexpr int kSW = kST / 32;          // warps
constexpr int kSR = 8;                 // rows of 32 edges per warp
constexpr int kSE = kST * kSR;         // 2048 edges per tile
constexpr int kSMW = kSE / 32;         // 64 mask words per tile; word q = warp q/8, row q%8

template <int kStages>
struct Ring {
    uint64_t bar[kStages];
    uint32_t tile[kStages];
};

// Thread 0 only: claim the next tile (dynamically: the d_in atomics meet very
// different contention per tile) and start its copy into `slot`.
template <int kStages>
__device__ __forceinline__ void ring_issue(Ring<kStages>& R, int slot, longlong2* stages, const longlong2* uv,
                                           int64_t m, uint32_t ntiles, uint32_t* next_tile, uint64_t pol) {
    const uint32_t t = atomicAdd(next_tile, 1u);
    R.tile[slot] = t;
    if (t < ntiles) {
        const int64_t base = (int64_t)t * kSE;
        const uint32_t bytes = (uint32_t)min((int64_t)kSE, m - base) * 16u;
        dev::fence_proxy_async_smem();
        dev::mbar_arrive_expect_tx(&R.bar[slot], bytes);
        dev::tma_load_1d(stages + (size_t)slot * kSE, uv + base, bytes, &R.bar[slot], pol);
    }
}

template <int kStages>
__device__ __forceinline__ void ring_start(Ring<kStages>& R, longlong2* stages, const longlong2* uv, int64_t m,
                                           uint32_t ntiles, uint32_t* next_tile, uint64_t pol) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) dev::mbar_init(&R.bar[k], 1);
        dev::mbar_fence_init();
        for (int k = 0; k < kStages; ++k) ring_issue<kStages>(R, k, stages, uv, m, ntiles, next_tile, pol);
    }
    __syncthreads();
}

// Pass A over the ring: validation, unique-entry count, warp-aggregated d_in.
template <int kStages>
__global__ void __launch_bounds__(kST) k2_pass_a_tma(const longlong2* __restrict__ uv, int64_t m, int64_t n,
                                                     uint32_t* __restrict__ d_in, uint32_t* __restrict__ err,
                                                     unsigned long long* __restrict__ nnz_raw, uint32_t ntiles,
                                                     uint32_t* __restrict__ next_tile, uint32_t v_lo, uint32_t v_hi,
                                                     bool first) {
    // Only columns [v_lo, v_hi) are counted by this launch (an in-degree table larger than the L2
    // is filled window by window, see k2_filter_device); validation and the unique-entry count
    // belong to the first window's launch.
    extern __shared__ __align__(128) unsigned char smem_raw[];
    longlong2* stages = reinterpret_cast<longlong2*>(smem_raw);
    __shared__ Ring<kStages> R;
    __shared__ uint32_t red[kSW];
    const unsigned lane = dev::lane_id(), w = dev::warp_id();
    const uint64_t pol = dev::policy_evict_first();
    ring_start<kStages>(R, stages, uv, m, ntiles, next_tile, pol);
    uint32_t my_err = 0, heads = 0;
    for (uint32_t i = 0;; ++i) {
        const int slot = (int)(i % kStages);
        const uint32_t t = R.tile[slot];
        if (t >= ntiles) break;
        const int64_t base = (int64_t)t * kSE;
        const int cnt = (int)min((int64_t)kSE, m - base);
        // warp 0 needs the edge before the tile (all lanes load the same address)
        const longlong2 before = (w == 0 && base > 0) ? uv[base - 1] : make_longlong2(0, 0);
        dev::mbar_wait(&R.bar[slot], (i / kStages) & 1u);  // acquire: the stage is visible to this thread
        const longlong2* tl = stages + (size_t)slot * kSE;
        const int c0 = (int)w * 32 * kSR;
        longlong2 carry = c0 > 0 ? tl[c0 - 1] : before;  // the edge before this warp's first
#pragma unroll
        for (int j = 0; j < kSR; ++j) {
            const int l = c0 + j * 32 + (int)lane;
            const bool valid = l < cnt;
            const longlong2 e = valid ? tl[l] : make_longlong2(0, 0);
            long long px = __shfl_up_sync(0xffffffffu, e.x, 1), py = __shfl_up_sync(0xffffffffu, e.y, 1);
            if (lane == 0) { px = carry.x; py = carry.y; }
            carry.x = __shfl_sync(0xffffffffu, e.x, 31);
            carry.y = __shfl_sync(0xffffffffu, e.y, 31);
            const bool has_pred = base + l > 0;
            const bool same = valid && has_pred && e.x == px && e.y == py;
            const unsigned eqm = __ballot_sync(0xffffffffu, same);
            if (valid) {
                const bool ok = e.x >= 1 && e.x <= n && e.y >= 1 && e.y <= n;
                if (!ok) my_err |= kErrLabelRange;
                else if (!same || lane == 0) {
                    // a run of equal edges adds its length (within this row) from its first lane
                    const unsigned after = ~(eqm >> lane >> 1) & (0x7fffffffu >> lane);
                    const uint32_t len = 1u + (after ? (uint32_t)(__ffs(after) - 1) : 31u - lane);
                    PRG_DCHECK(len >= 1 && len <= 32u - lane);
                    const uint32_t c = (uint32_t)(e.y - 1);
                    if (c >= v_lo && c < v_hi) atomicAdd(&d_in[c], len);
                }
                if (has_pred) {
                    if (e.x < px) my_err |= kErrUnsorted;
                    else if (e.x == px && e.y < py) my_err |= kErrNotCanonical;
                }
                heads += first && !same;
            }
        }
        __syncthreads();  // every read of this stage is done
        if (threadIdx.x == 0) ring_issue<kStages>(R, slot, stages, uv, m, ntiles, next_tile, pol);
    }
    heads = dev::warp_sum(heads);
    if (lane == 0) red[w] = heads;
    my_err = __reduce_or_sync(0xffffffffu, my_err);
    if (lane == 0 && my_err) atomicOr(err, my_err);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int k = 0; k < kSW; ++k) tot += red[k];
        if (tot) atomicAdd(nnz_raw, tot);
    }
}

}  // namespace

uint32_t k2_filter_device(const int64_t* d_uv, int64_t m, int64_t n, prg_matrix* out, cudaStream_t s,
                          bool filter, bool normalize) {
    ProfScope prof("k2_filter", s);
    if (n > (int64_t{1} << 31)) throw CudaError{"K2: vertex count above 2^31"};
    out->n = n;
    out->cap = (uint64_t)(m > 0 ? m : 1);
    out->row_offsets = static_cast<uint32_t*>(ws_alloc((size_t)(n + 1) * 4, s));
    out->cols = static_cast<uint32_t*>(ws_alloc(out->cap * 4, s));
    out->values = static_cast<double*>(ws_alloc(out->cap * 8, s));
    out->d_in = static_cast<uint32_t*>(ws_alloc((size_t)n * 4, s));
    PRG_CUDA(cudaMemsetAsync(out->d_in, 0, (size_t)n * 4, s));
    if (m == 0) {
        PRG_CUDA(cudaMemsetAsync(out->row_offsets, 0, (size_t)(n + 1) * 4, s));
        out->nnz = out->nnz_raw = out->max_in = 0;
        return 0;
    }
    const uint32_t ntiles = div_up((uint64_t)m, kTE);
    DevBuf<uint64_t> scal(8, s);  // [0]=err|max [1]=nnz_raw [2]=nnz [3]=n_fix|tile_counter
    PRG_CUDA(cudaMemsetAsync(scal.get(), 0, 8 * sizeof(uint64_t), s));
    uint32_t* err = reinterpret_cast<uint32_t*>(scal.get());
    uint32_t* maxp = err + 1;
    unsigned long long* nnz_raw = reinterpret_cast<unsigned long long*>(scal.get() + 1);
    unsigned long long* nnz_out = reinterpret_cast<unsigned long long*>(scal.get() + 2);
    uint32_t* n_fix = reinterpret_cast<uint32_t*>(scal.get() + 3);
    uint32_t* tile_counter = n_fix + 1;
    uint32_t* tile_counter_a = reinterpret_cast<uint32_t*>(scal.get() + 4);

    const auto* uv = reinterpret_cast<const longlong2*>(d_uv);
    static bool attr = false;
    if (!attr) {
        PRG_CUDA(cudaFuncSetAttribute(k2_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PassBSmem)));
        attr = true;
    }
    const unsigned ga = std::min<unsigned>(ntiles, (unsigned)num_sms() * 2);
    static int flags = -1;  // PRG_K2_FLAGS (A/B measurement knob): bit 0 evict-first edge loads, bit 1 streaming stores
    if (flags < 0) { const char* e = getenv("PRG_K2_FLAGS"); flags = e ? atoi(e) : 0; }
    static int v1 = -1;     // PRG_K2_V1=1: the register-tile pass A (A/B against the TMA-ring pass A)
    if (v1 < 0) { const char* e = getenv("PRG_K2_V1"); v1 = e ? atoi(e) : 0; }
    static int ctas = -1;   // PRG_K2_CTAS: persistent CTAs per SM of the TMA-ring passes
    if (ctas < 0) { const char* e = getenv("PRG_K2_CTAS"); ctas = e ? atoi(e) : 3; }
#ifndef PRG_K2A_STAGES
#define PRG_K2A_STAGES 3
#endif
    constexpr int kStagesA = PRG_K2A_STAGES;
    const uint32_t ntiles_s = div_up((uint64_t)m, kSE);
    // persistent grid: min(PRG_K2_CTAS, resident CTAs) per SM
    auto grid_for = [&](const void* fn, size_t smem) {
        int occ = 1;
        PRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kST, smem));
        return std::min<unsigned>(ntiles_s, (unsigned)(num_sms() * std::max(1, std::min(occ, ctas))));
    };
    {
        ProfScope pa("k2_pass_a", s);
        if (v1) {
            k2_pass_a<<<ga, kT, 0, s>>>(uv, m, n, out->d_in, err, nnz_raw, ntiles, tile_counter_a, flags);
        } else {
            const size_t smem = (size_t)kStagesA * kSE * sizeof(longlong2);
            PRG_CUDA(cudaFuncSetAttribute(k2_pass_a_tma<kStagesA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const unsigned gs = grid_for((const void*)k2_pass_a_tma<kStagesA>, smem);
            // An in-degree table that does not fit the L2 (S=26: 268 MB) turns every RED into HBM
            // traffic (pass A 20.3 ms for 2^30 edges, 8x the S=24 time for 4x the edges). Above
            // 2^25 columns the table is filled one window of columns at a time: each launch
            // re-streams the edges (~4.9 ms at S=26) but its atomics mostly stay in the L2.
            // S=26: two 128 MB windows 16.6 ms; four 64 MB windows 19.7 ms; eight 36 ms.
            static int64_t window = -1;  // PRG_K2_WINDOW: log2 of the window's columns (0 = one pass)
            if (window < 0) { const char* e = getenv("PRG_K2_WINDOW"); window = e ? atoll(e) : 25; }
            const int64_t wcols = window > 0 ? (int64_t{1} << window) : n;
            const int nwin = (int)((n + wcols - 1) / wcols);
            for (int wi = 0; wi < nwin; ++wi) {
                if (wi) PRG_CUDA(cudaMemsetAsync(tile_counter_a, 0, 4, s));
                k2_pass_a_tma<kStagesA><<<gs, kST, smem, s>>>(
                    uv, m, n, out->d_in, err, nnz_raw, ntiles_s, tile_counter_a, (uint32_t)(wi * wcols),
                    (uint32_t)std::min<int64_t>(n, (wi + 1) * wcols), wi == 0);
            }
        }
        PRG_LAUNCH_CHECK();
    }
    uint32_t h_err = 0;
    PRG_CUDA(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    if (h_err & (kErrLabelRange | kErrUnsorted)) return h_err;
    if (h_err & kErrNotCanonical) {
        // Ties are not v-ordered (e.g. the reference's std::sort output): the
        // reference sorts each row's pending list (kernel2_filter.cpp:24), we
        // canonicalise the whole list with the K1 sort and rerun.
        int scale = 0;
        while ((int64_t{1} << scale) < n) ++scale;
        DevBuf<int64_t> tmp((size_t)m * 2, s);
        DevBuf<uint32_t> e2(1, s);
        PRG_CUDA(cudaMemsetAsync(e2.get(), 0, 4, s));
        k1_sort_device(d_uv, m, scale, tmp.get(), e2.get(), s);
        ws_free(out->row_offsets, s); ws_free(out->cols, s); ws_free(out->values, s); ws_free(out->d_in, s);
        out->row_offsets = nullptr; out->cols = nullptr; out->values = nullptr; out->d_in = nullptr;
        return k2_filter_device(tmp.get(), m, n, out, s, filter, normalize) & ~(uint32_t)kErrNotCanonical;
    }
    const unsigned gn = (unsigned)num_sms() * 8;
    k2_max_kernel<<<gn, 1024, 0, s>>>(out->d_in, n, maxp);
    PRG_LAUNCH_CHECK();
    DevBuf<uint32_t> keepbits((size_t)(n + 31) / 32, s);
    if (filter) {
        k2_keep_kernel<<<gn, 1024, 0, s>>>(out->d_in, n, maxp, keepbits.get());
        PRG_LAUNCH_CHECK();
    } else {  // build_adjacency only: keep every column
        PRG_CUDA(cudaMemsetAsync(keepbits.get(), 0xff, (size_t)(n + 31) / 32 * 4, s));
    }
    const uint32_t nt_b = ntiles;
    DevBuf<unsigned long long> tile_status(nt_b, s);
    DevBuf<uint32_t> dout_f((size_t)n, s), fix_rows(nt_b + 1, s), cont_p(nt_b, s), cont_c(nt_b, s);
    PRG_CUDA(cudaMemsetAsync(tile_status.get(), 0, (size_t)nt_b * 8, s));
    PRG_CUDA(cudaMemsetAsync(dout_f.get(), 0, (size_t)n * 4, s));
    {
        ProfScope pb("k2_pass_b", s);
        k2_pass_b<<<ntiles, kT, sizeof(PassBSmem), s>>>(uv, m, n, keepbits.get(), out->row_offsets, out->cols,
                                                        out->values, tile_status.get(), tile_counter, dout_f.get(),
                                                        fix_rows.get(), n_fix, cont_p.get(), cont_c.get(), nnz_out,
                                                        normalize, flags);
        PRG_LAUNCH_CHECK();
    }
    k2_fix_runs<<<div_up(nt_b, 256), 256, 0, s>>>(cont_p.get(), cont_c.get(), nt_b, out->values);
    PRG_LAUNCH_CHECK();
    if (normalize)
    {
        DevBuf<uint64_t> task_row((size_t)nt_b + (size_t)m / kFixChunk + 2, s);
        DevBuf<uint32_t> n_tasks(1, s);
        DevBuf<uint32_t> nc((size_t)nt_b + 1, s), nbase((size_t)nt_b + 1, s);
        const unsigned gf = (unsigned)num_sms() * 4;
        k2_fix_count<<<gf, 256, 0, s>>>(fix_rows.get(), n_fix, out->row_offsets, nc.get());
        exclusive_scan_u32_prefix(nc.get(), nbase.get(), (size_t)nt_b + 1, n_fix, 1, s);
        k2_fix_emit<<<gf, 256, 0, s>>>(nc.get(), nbase.get(), n_fix, task_row.get(), n_tasks.get());
        k2_fix_rows<<<(unsigned)num_sms() * 8, 256, 0, s>>>(fix_rows.get(), task_row.get(), n_tasks.get(),
                                                             out->row_offsets, dout_f.get(), out->values);
    }
    PRG_LAUNCH_CHECK();
    uint64_t h[3];
    PRG_CUDA(cudaMemcpyAsync(h, scal.get(), 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    out->max_in = h[0] >> 32;
    out->nnz_raw = h[1];
    out->nnz = h[2];
    return (uint32_t)(h[0] & 0xffffffffu) & ~(uint32_t)kErrNotCanonical;
}

}  // namespace prg

PRG_CHECK_QUERY(k2)
