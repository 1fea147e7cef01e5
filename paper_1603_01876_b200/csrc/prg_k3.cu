// prg_k3.cu — K3: damped PageRank, 20 pull-SpMV iterations on the device.
//
// Replaces prpipe::run_kernel3 / init_rank / pagerank_step
// (src/kernel3_pagerank.cpp:29-79). The reference pushes r[u]*A[u][c] into
// out[c] over the CSR (:49-57), then out = c*out + ((1-c)/N)*sum(r) (:45-46,
// :58-61). Here the CSR handed over by K2 is transposed once (inside the timed
// region) and every iteration pulls over columns.
//
// Layout (timed mode):
//   * rows are renumbered by descending out-degree (quarter-octave classes,
//     ties by original id); dangling rows go last and are never gathered. The
//     gather vector s[j] = r[u_j] * b[u_j] (j = new id) is therefore dense and
//     hot-first (~59 MB at S=24, L2-resident; the L1 keeps the hot head).
//     Random gathers are the bound: ~1 line/clk/SM from L2 (tools/microbench).
//     A shared-memory copy of the hot head measured slower (1.62 vs 1.22 ms).
//   * b[u] is the row's base value (its minimum stored value; for K2 output
//     that is 1/d_out exactly). Entries equal to b[u] contribute r[u]*b[u],
//     the reference's own product r[u]*values[k], bit for bit. Other entries
//     (duplicate edges, ~1.3%) are exceptions: their SELL slot gathers
//     s[n_nd + j], the exception's product r[u]*value written each iteration.
//   * transpose = stable sort of (col | new row, exception) keys by column
//     only (the payload keeps each column's rows in ascending new id), then a
//     SELL-32 layout over virtual columns of <= vcmax entries (64-512 by size), slices sorted
//     by length class. Columns keep their original ids.
// Parity mode (mode 1) keeps original row ids, sums every column sequentially
// in ascending u with separate mul/add, and computes every sum(r) with one
// thread in index order — the reference's exact evaluation order.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "prg_internal.cuh"
#include "prg_sort.cuh"

namespace prg {

struct K3Plan {
    int64_t n = 0, n_nd = 0;
    uint64_t nnz = 0;
    int sb = 1;
    int pb = 1;  // transpose key payload bits (row id or exception index)
    int mode = 0;
    DevBuf<uint32_t> pinv, newid, colptr, csc_idx;
    DevBuf<double> bval, exc_val;
    uint32_t n_exc = 0;
    // timed mode (SELL)
    uint32_t V = 0, nslices = 0, n_empty = 0;
    DevBuf<uint32_t> sell, slice_ptr, lane_len, lane_col, lane_np, vc_base, vpos, spos, spos_col, split_col, n_split,
        split_p0, split_pbase, lane_pslot,
        e_u;  // exception list: new row e_u[i], value exc_val[i]
    DevBuf<double> partial;
    // timed-mode gather: spos covers [rows | exceptions] (an exception's entry
    // is its row's), coef = [row base | exception value], both n_nd + n_exc
    DevBuf<double> coef;
    // A layout kept on a prg_matrix outlives the stream it was built on: its
    // buffers are released on the null stream (after a device sync).
    void rehome() {
        for (DevBuf<uint32_t>* b : {&pinv, &newid, &colptr, &csc_idx, &sell, &slice_ptr, &lane_len, &lane_col,
                                    &lane_np, &vc_base, &vpos, &spos, &spos_col, &split_col, &n_split, &split_p0, &split_pbase, &lane_pslot, &e_u})
            b->s = nullptr;
        for (DevBuf<double>* b : {&bval, &exc_val, &partial, &coef}) b->s = nullptr;
    }
};

void k3_plan_destroy(K3Plan* p) { delete p; }

namespace {

constexpr uint64_t kRankInitStream = 0x72616e6b696e6974ULL;  // kernel3_pagerank.cpp:15
constexpr int kSpmvThreads = 1024;  // the 32-register variant (PRG_SPMV_VARIANT=1)
constexpr int kSliceCounters = 8;

__host__ __device__ inline int bits_for(int64_t n) {
    int b = 1;
    while ((int64_t{1} << b) < n) ++b;
    return b;
}

// ---------------------------------------------------------------------------
// Row renumbering
// ---------------------------------------------------------------------------
struct RowClassSrc {
    const uint32_t* ro;
    int sb;
    // Within a degree class, rows are ordered by the top fb bits of their first
    // (smallest) column: rows feeding the same columns get nearby new ids, so a
    // column's gathers reuse L1 lines (SpMV 1.22 -> 1.16 ms at S=24; the class
    // alone, or 8 bits of the column, gave nothing).
    const uint32_t* cols;  // null: class only
    int fb;
    static constexpr size_t kSmem = 0;
    static constexpr int kHistBatch = 16;
    static constexpr bool kRegPrefetch = false;
    static constexpr bool kL2Prefetch = false;
    __device__ void prefetch_l2(size_t) const {}
    __device__ void prepare(size_t, int, void*) const {}
    __device__ __forceinline__ uint64_t key(size_t i, int, const void*) const {
        const uint32_t d = ro[i + 1] - ro[i];
        uint32_t cls;
        if (d == 0) cls = 255;
        else {
            const int lg = 31 - __clz(d);
            const uint32_t q = lg >= 2 ? (d >> (lg - 2)) & 3u : (lg == 1 ? (d & 1u) << 1 : 0u);
            cls = 127u - (uint32_t)(lg * 4) - q;
        }
        if (cols) {
            const uint32_t fc = d ? (sb > fb ? cols[ro[i]] >> (sb - fb) : cols[ro[i]]) : 0u;
            return ((uint64_t)cls << (sb + fb)) | ((uint64_t)fc << sb) | i;
        }
        return ((uint64_t)cls << sb) | i;
    }
};

__global__ void nondangling_flag_kernel(const uint32_t* __restrict__ ro, int64_t n, uint32_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = ro[i + 1] > ro[i];
}
// Non-dangling row i -> its sort key at its rank pos[i]; dangling row i -> new
// id n_nd + (its rank among the dangling rows), written directly.
template <class Src>
__global__ void row_keys_kernel(Src src, int64_t n, const uint32_t* __restrict__ pos,
                                unsigned long long* __restrict__ keys, uint32_t* __restrict__ pinv,
                                uint32_t* __restrict__ newid, uint32_t n_nd) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = pos[i];
        if (pos[i + 1] > p) {
            keys[p] = src.key((size_t)i, 0, nullptr);
        } else {
            const uint32_t id = n_nd + (uint32_t)i - p;
            pinv[id] = (uint32_t)i;
            newid[i] = id;
        }
    }
}

struct PermDst {
    uint32_t* pinv;   // new id -> original row
    uint32_t* newid;  // original row -> new id
    int sb;
    __device__ __forceinline__ void store(uint64_t pos, uint64_t key, bool, uint64_t) const {
        const uint32_t u = (uint32_t)(key & ((1ull << sb) - 1));
        pinv[pos] = u;
        newid[u] = (uint32_t)pos;
    }
};

__global__ void iota_kernel(uint32_t* a, uint32_t* b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        a[i] = (uint32_t)i;
        b[i] = (uint32_t)i;
    }
}


// ---------------------------------------------------------------------------
// CSR tile expansion: row id of every entry of a tile of nnz.
// ---------------------------------------------------------------------------
// tile_row[t] = row containing entry t*kTile (for non-empty tiles).
__global__ void tile_rows_kernel(const uint32_t* __restrict__ ro, int64_t n, uint32_t* __restrict__ tile_row) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t b = ro[r], e = ro[r + 1];
        if (b == e) continue;
        for (uint64_t t = (b + sort::kTile - 1) / sort::kTile; t * sort::kTile < e; ++t) tile_row[t] = (uint32_t)r;
    }
}

// Padded SMEM index for expand_rows' row table: one spare word per 32 keeps the
// blocked max-scan (thread t touches words 16t..16t+15) free of bank conflicts.
__device__ __forceinline__ int rpad(int i) { return i + (i >> 5); }
constexpr int kRowWords = sort::kTile + sort::kTile / 32;

// All threads: srow[rpad(li)] = row of entry base+li, li < cnt. smem must hold kRowWords u32.
__device__ void expand_rows(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ tile_row,
                            int64_t n, size_t base, int cnt, uint32_t* srow) {
    const uint32_t t = (uint32_t)(base / sort::kTile);
    const uint32_t r0 = tile_row[t];
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) srow[rpad(i)] = 0;
    __syncthreads();
    if (threadIdx.x == 0) srow[0] = r0;
    // Rows starting inside the tile: scan forward from r0+1 while ro[r] < base+cnt.
    const uint64_t end = base + cnt;
    for (int64_t r = (int64_t)r0 + 1 + threadIdx.x;; r += blockDim.x) {
        const bool in = r < n && ro[r] < end;
        if (in && ro[r + 1] > ro[r]) srow[rpad((int)(ro[r] - base))] = (uint32_t)r;
        if (!__syncthreads_or(in)) break;
    }
    // inclusive max-scan over srow (blocked, 8192 entries / blockDim threads)
    __shared__ uint32_t wmax[32];
    const int per = (cnt + blockDim.x - 1) / blockDim.x;
    const int l0 = threadIdx.x * per;
    uint32_t m = 0;
    for (int k = 0; k < per && l0 + k < cnt; ++k) m = max(m, srow[rpad(l0 + k)]);
    uint32_t inc = m;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if ((int)dev::lane_id() >= d) inc = max(inc, o);
    }
    if (dev::lane_id() == 31) wmax[dev::warp_id()] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t x = threadIdx.x < blockDim.x / 32 ? wmax[threadIdx.x] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t o = __shfl_up_sync(0xffffffffu, x, d);
            if ((int)threadIdx.x >= d) x = max(x, o);
        }
        wmax[threadIdx.x] = x;
    }
    __syncthreads();
    uint32_t run = dev::warp_id() > 0 ? wmax[dev::warp_id() - 1] : 0;
    uint32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (dev::lane_id() > 0) run = max(run, ex);
    for (int k = 0; k < per && l0 + k < cnt; ++k) {
        run = max(run, srow[rpad(l0 + k)]);
        srow[rpad(l0 + k)] = run;
    }
    __syncthreads();
}

// Degrees in new row order, and the shift from CSR to permuted positions
// (u32 wrap-around arithmetic; nnz < 2^32).
__global__ void perm_degree_kernel(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ pinv, int64_t nr,
                                   uint32_t* __restrict__ deg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = pinv[i];
        deg[i] = ro[u + 1] - ro[u];
    }
}
// Walked in the original row order (a gather of pro through newid, coalesced
// stores): walking the new order scattered the stores (0.21 ms at S=24).
__global__ void perm_delta_kernel(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ newid,
                                  const uint32_t* __restrict__ pro, int64_t n, int64_t nr,
                                  uint32_t* __restrict__ wdelta) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = newid[u];
        if (j < (uint64_t)nr) wdelta[u] = pro[j] - ro[u];
    }
}

// Row base value bmin[u] (u64 bit pattern): the minimum of five of the row's
// stored values (first, quartiles, last). Any choice is exact — an entry whose
// value differs from its row base becomes an exception — and for a stochastic
// matrix a row's values are k/d_out with k = 1 for almost every entry, so the
// sampled minimum finds 1/d_out: at S=18/20 it yields exactly the exceptions of
// the full row minimum (five loads per row instead of a pass over the values).
__global__ void row_base_kernel(const uint32_t* __restrict__ ro, const double* __restrict__ val, int64_t n,
                                unsigned long long* __restrict__ bmin) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = ro[u], d = ro[u + 1] - b;
        unsigned long long m = ~0ull;
        if (d) {
            const unsigned long long* v = reinterpret_cast<const unsigned long long*>(val) + b;
            m = min(min(v[0], v[d - 1]), min(min(v[d >> 2], v[d >> 1]), v[(3 * (uint64_t)d) >> 2]));
        }
        bmin[u] = m;
    }
}

// Transpose keys: for every CSR entry (u, col, a) the key
// (col, newid[u], a != bmin[u]) written at its position in the NEW row order
// (rows permuted, each row's entries contiguous). A stable sort of these keys
// by column then lists every column's rows in ascending new id. An exception
// (a != row base: a duplicate edge) is appended to the exception list (row,
// value; one atomic per tile) and its key carries its list index instead of
// the row: the transpose then hands every exception entry its own slot in the
// gather vector (s[n_nd + index]) with no exception sort. The index order is
// arbitrary; column sums are not — they follow the stable CSC order.
struct KeyBuildArgs {
    const uint32_t* ro;
    const uint32_t* tile_row;
    const uint32_t* cols;
    const double* val;
    const unsigned long long* bmin;
    const uint32_t* newid;   // null: identity
    const uint32_t* wdelta;  // null: identity
    int64_t n;
    uint64_t nnz;
    int pb;  // payload bits (row id or exception index), below them the exception flag
    unsigned long long* keys;
    uint32_t* e_u;   // exception list: new row
    double* e_val;   //                 value
    uint32_t* n_exc;
};
__global__ void __launch_bounds__(sort::kTileThreads, 4) key_build_kernel(KeyBuildArgs a) {
    extern __shared__ uint32_t srow[];
    __shared__ uint32_t scan_tmp[sort::kTileThreads / 32 + 1];
    __shared__ uint32_t tile_base;
    const uint32_t ntiles = (uint32_t)((a.nnz + sort::kTile - 1) / sort::kTile);
    const unsigned lane = dev::lane_id();
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const size_t base = (size_t)t * sort::kTile;
        const int cnt = (int)min((uint64_t)sort::kTile, a.nnz - base);
        expand_rows(a.ro, a.tile_row, a.n, base, cnt, srow);
        uint32_t excm = 0;
#pragma unroll 8
        for (int j = 0; j < sort::kTileItems; ++j) {
            const int li = j * sort::kTileThreads + threadIdx.x;
            if (li < cnt) {
                const uint32_t u = srow[rpad(li)];
                const uint32_t e = (uint32_t)(base + li);
                const uint32_t c = a.cols[e];
                const double v = a.val[e];
                const bool exc = (uint64_t)__double_as_longlong(v) != a.bmin[u];
                const uint32_t nid = a.newid ? a.newid[u] : u;
                const uint32_t pos = a.wdelta ? e + a.wdelta[u] : e;
                PRG_DCHECK(pos < a.nnz && u < a.n);
                a.keys[pos] = ((uint64_t)c << (a.pb + 1)) | ((uint64_t)nid << 1);  // exceptions: rewritten below
                excm |= (uint32_t)exc << j;
            }
        }
        uint32_t tot;
        const uint32_t ex = dev::block_excl_scan((uint32_t)__popc(excm), scan_tmp, tot);
        if (threadIdx.x == 0) tile_base = tot ? atomicAdd(a.n_exc, tot) : 0u;
        __syncthreads();
        if (excm) {
            uint32_t idx = tile_base + ex;
            for (int j = 0; j < sort::kTileItems; ++j) {
                if (!((excm >> j) & 1u)) continue;
                const int li = j * sort::kTileThreads + threadIdx.x;
                const uint32_t e = (uint32_t)(base + li);
                const uint32_t u = srow[rpad(li)];
                const uint32_t pos = a.wdelta ? e + a.wdelta[u] : e;
                a.keys[pos] = ((uint64_t)a.cols[e] << (a.pb + 1)) | ((uint64_t)idx << 1) | 1ull;
                a.e_u[idx] = a.newid ? a.newid[u] : u;
                a.e_val[idx] = a.val[e];
                ++idx;
            }
        }
        __syncthreads();
    }
    (void)lane;
}

// bval[i] = row base of new row i.
__global__ void gather_base_kernel(const uint32_t* __restrict__ pinv, const unsigned long long* __restrict__ bmin,
                                   int64_t n_nd, double* __restrict__ bval) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_nd; j += (int64_t)gridDim.x * blockDim.x)
        bval[j] = __longlong_as_double((long long)bmin[pinv[j]]);
}

// CSC entry: new row id, or (bit 31 set) exception list index.
struct CscDst {
    uint32_t* csc_idx;
    uint32_t* colptr;   // initialised to ~0; column starts via atomicMin
    int pb;
    __device__ __forceinline__ void store(uint64_t pos, uint64_t key, bool has_prev, uint64_t prev) const {
        const uint32_t col = (uint32_t)(key >> (pb + 1));
        csc_idx[pos] = (uint32_t)((key >> 1) & ((1ull << pb) - 1)) | ((uint32_t)(key & 1) << 31);
        if (!has_prev || (uint32_t)(prev >> (pb + 1)) != col) atomicMin(&colptr[col], (uint32_t)pos);
    }
};

// colptr[c] = min(colptr[c], colptr[c+1], ...) — fills empty columns.
// In place, inclusive; the block minima are themselves suffix-minimised
// recursively (a one-thread loop over them took ~50 us at S=24).
__global__ void suffix_min_block(uint32_t* a, int64_t n1, uint32_t* part) {
    // each block: 1024 threads x 8 items, reverse order
    __shared__ uint32_t wm[32];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    // the block minimum needs no blocked order: coalesced strided reads
    uint32_t m = 0xffffffffu;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = base + k * 1024 + threadIdx.x;
        if (i < n1) m = min(m, a[i]);
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (dev::lane_id() == 0) wm[dev::warp_id()] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t x = wm[threadIdx.x];
        x = __reduce_min_sync(0xffffffffu, x);
        if (threadIdx.x == 0) part[blockIdx.x] = x;
    }
}
// blk_suffix: inclusive suffix minima of the block minima (null: a single block)
__global__ void suffix_min_down(uint32_t* a, int64_t n1, const uint32_t* blk_suffix, int64_t nb) {
    __shared__ uint32_t wm[33];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    uint32_t v[8];
    const int64_t my = base + threadIdx.x * 8;
    // 32 contiguous bytes per thread: two 16-byte accesses when whole and aligned
    const bool vec = my + 8 <= n1 && (reinterpret_cast<uintptr_t>(a) & 15) == 0;
    if (vec) {
        const uint4 x = reinterpret_cast<const uint4*>(a + my)[0], y = reinterpret_cast<const uint4*>(a + my)[1];
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    } else {
        for (int k = 0; k < 8; ++k) v[k] = my + k < n1 ? a[my + k] : 0xffffffffu;
    }
    uint32_t tm = 0xffffffffu;
    for (int k = 0; k < 8; ++k) tm = min(tm, v[k]);
    // exclusive suffix min across threads: threads after me
    uint32_t inc = tm;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_down_sync(0xffffffffu, inc, d);
        if (dev::lane_id() + d < 32) inc = min(inc, o);
    }
    if (dev::lane_id() == 0) wm[dev::warp_id()] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t x = wm[threadIdx.x];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t o = __shfl_down_sync(0xffffffffu, x, d);
            if (threadIdx.x + d < 32) x = min(x, o);
        }
        wm[threadIdx.x] = x;  // inclusive suffix over warps
    }
    __syncthreads();
    uint32_t run = (blk_suffix && blockIdx.x + 1 < nb) ? blk_suffix[blockIdx.x + 1] : 0xffffffffu;
    if (dev::warp_id() + 1 < 32) run = min(run, wm[dev::warp_id() + 1]);
    uint32_t after = __shfl_down_sync(0xffffffffu, inc, 1);
    if (dev::lane_id() < 31) run = min(run, after);
    for (int k = 7; k >= 0; --k) {
        run = min(run, v[k]);
        v[k] = run;
    }
    if (vec) {
        reinterpret_cast<uint4*>(a + my)[0] = make_uint4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<uint4*>(a + my)[1] = make_uint4(v[4], v[5], v[6], v[7]);
    } else {
        for (int k = 0; k < 8; ++k)
            if (my + k < n1) a[my + k] = v[k];
    }
}

// ---------------------------------------------------------------------------
// init_rank (kernel3_pagerank.cpp:29-39)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rank_init_x(uint64_t s0, uint64_t i) {
    return (double)(dev::splitmix_at(s0, i + 1) >> 11) * 0x1.0p-53;  // kernel3_pagerank.cpp:31-34
}
__global__ void rng_kernel(double* __restrict__ x, int64_t n, uint64_t s0) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (double)(dev::splitmix_at(s0, (uint64_t)i + 1) >> 11) * 0x1.0p-53;
}

// Deterministic block partial sums: block b sums [b*8192, (b+1)*8192) in a fixed tree.
__global__ void partial_sum_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double ws[32];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    double s = 0.0;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = base + k * 1024 + threadIdx.x;
        if (i < n) s = __dadd_rn(s, x[i]);
    }
    s = dev::warp_sum_f64(s);
    if (dev::lane_id() == 0) ws[dev::warp_id()] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = ws[threadIdx.x];
        v = dev::warp_sum_f64(v);
        if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
}
// init_rank without the vector: block partials (same tree as partial_sum_kernel,
// so the sums are bit-identical) of x_i, or of x_i / div when div is given.
__global__ void rng_partial_kernel(int64_t n, uint64_t s0, const double* __restrict__ div, double* __restrict__ part) {
    __shared__ double ws[32];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    const double d = div ? *div : 1.0;
    double s = 0.0;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = base + k * 1024 + threadIdx.x;
        if (i < n) {
            const double x = rank_init_x(s0, (uint64_t)i);
            s = __dadd_rn(s, div ? __ddiv_rn(x, d) : x);
        }
    }
    s = dev::warp_sum_f64(s);
    if (dev::lane_id() == 0) ws[dev::warp_id()] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = ws[threadIdx.x];
        v = dev::warp_sum_f64(v);
        if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
}
// One block: fixed-order sum of np partials -> out[0]; out[1] = bg factor * sum.
__global__ void final_sum_kernel(const double* __restrict__ part, int64_t np, double bgf, double* __restrict__ out) {
    __shared__ double ws[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < np; i += 1024) s = __dadd_rn(s, part[i]);
    s = dev::warp_sum_f64(s);
    if (dev::lane_id() == 0) ws[dev::warp_id()] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = ws[threadIdx.x];
        v = dev::warp_sum_f64(v);
        if (threadIdx.x == 0) { out[0] = v; out[1] = __dmul_rn(bgf, v); }
    }
}
// Parity mode: one thread, index order (std::accumulate, kernel3_pagerank.cpp:17-19).
__global__ void seq_sum_kernel(const double* __restrict__ x, int64_t n, double bgf, double* __restrict__ out) {
    if (threadIdx.x || blockIdx.x) return;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, x[i]);
    out[0] = s;
    out[1] = __dmul_rn(bgf, s);
}
// Neumaier mode (mode 2): the same single pass with a compensated sum — the
// drift-attribution restatement of SURVEY §8(c): every sum_of
// (kernel3_pagerank.cpp:17-19) replaced by Neumaier's, as oracle/prg_oracle.c's
// accurate mode.
__global__ void seq_neumaier_kernel(const double* __restrict__ x, int64_t n, double bgf, double* __restrict__ out) {
    if (threadIdx.x || blockIdx.x) return;
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double v = x[i];
        const double t = __dadd_rn(s, v);
        c = __dadd_rn(c, fabs(s) >= fabs(v) ? __dadd_rn(__dsub_rn(s, t), v) : __dadd_rn(__dsub_rn(v, t), s));
        s = t;
    }
    s = __dadd_rn(s, c);
    out[0] = s;
    out[1] = __dmul_rn(bgf, s);
}
__global__ void __launch_bounds__(1024, 2) scale_kernel(double* __restrict__ x, int64_t n, const double* __restrict__ sum) {
    const double d = sum[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __ddiv_rn(x[i], d);
}


// ---------------------------------------------------------------------------
// Parity mode SpMV: one thread per column, ascending source order, separate
// mul/add (kernel3_pagerank.cpp:50-61 evaluated in the reference's order).
// ---------------------------------------------------------------------------
struct SeqArgs {
    const uint32_t* colptr;
    const uint32_t* csc_idx;
    const uint32_t* e_u;       // exception list (row, value)
    const double* e_val;
    const double* s;           // s[u] = r[u] * b[u] (identity numbering)
    const double* r_prev;      // original order
    const double* bgp;
    double* r_next;
    int64_t n;
    double damping;
};

__global__ void spmv_seq_kernel(SeqArgs a) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < a.n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = a.colptr[c], e = a.colptr[c + 1];
        double acc = 0.0;
        for (uint32_t p = b; p < e; ++p) {
            const uint32_t w = a.csc_idx[p];
            const uint32_t u = w & 0x7fffffffu;
            const double x = (w >> 31) ? __dmul_rn(a.r_prev[a.e_u[u]], a.e_val[u]) : a.s[u];
            acc = __dadd_rn(acc, x);
        }
        a.r_next[c] = __dadd_rn(__dmul_rn(a.damping, acc), a.bgp[1]);
    }
}

// ---------------------------------------------------------------------------
// Timed mode: sliced ELL over virtual columns (SELL-32-sigma).
//
// Every non-empty column is cut into parts of at most vcmax entries ("virtual
// columns"); virtual columns are ordered by quarter-octave length class
// (descending) and packed 32 to a slice. Slice s stores entry k of its lane-j
// virtual column at sell[slice_ptr[s] + 32k + j], so a warp reads 128
// contiguous bytes per step and each lane sums its own column sequentially —
// no owner search, no segmented scan, a fixed summation order. Parts of split
// columns are combined, in part order, by whichever part finishes last.
// Results y are kept in SELL position order; empty columns are implicit (their
// value is bg), and only the final iterate is un-permuted.
// ---------------------------------------------------------------------------
constexpr uint32_t kEmpty = 0xffffffffu;

__device__ __forceinline__ uint32_t len_class_desc(uint32_t d) {
    const int lg = 31 - __clz(d);
    const uint32_t q = lg >= 2 ? (d >> (lg - 2)) & 3u : (lg == 1 ? (d & 1u) << 1 : 0u);
    return 127u - (uint32_t)(lg * 4) - q;
}

__global__ void vc_count_kernel(const uint32_t* __restrict__ colptr, int64_t n, uint32_t vcmax,
                                uint32_t* __restrict__ np) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t len = colptr[c + 1] - colptr[c];
        np[c] = (len + vcmax - 1) / vcmax;
    }
}

__global__ void vc_fill_kernel(const uint32_t* __restrict__ colptr, const uint32_t* __restrict__ vc_base, int64_t n,
                               uint32_t vcmax, uint32_t* __restrict__ vc_col, uint32_t* __restrict__ vc_len) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t len = colptr[c + 1] - colptr[c];
        for (uint32_t v = vc_base[c], p = 0; v < vc_base[c + 1]; ++v, ++p) {
            vc_col[v] = (uint32_t)c;
            vc_len[v] = min(vcmax, len - p * vcmax);
        }
    }
}

// Virtual columns ordered by length class (load balance: longest slices are
// handed out first), then by the top 16 bits of the new id of their last
// (coldest) row: columns reaching the same cold rows run close together in
// time and share those rows' L1 lines (SpMV 0.868 -> 0.825 ms at S=24; the
// first row: 0.833, 24 bits: 0.829).
struct VcClassSrc {
    const uint32_t* vc_len;
    int vb;
    const uint32_t* vc_col;
    const uint32_t* vc_base;
    const uint32_t* colptr;
    const uint32_t* csc_idx;  // null: length class only
    const uint32_t* e_u;      // exception list rows
    int sb;
    uint32_t vcmax;
    static constexpr size_t kSmem = 0;
    static constexpr int kHistBatch = 16;
    static constexpr bool kRegPrefetch = false;
    static constexpr bool kL2Prefetch = false;
    __device__ void prefetch_l2(size_t) const {}
    __device__ void prepare(size_t, int, void*) const {}
    __device__ __forceinline__ uint64_t key(size_t i, int, const void*) const {
        if (csc_idx) {
            const uint32_t c = vc_col[i];
            const uint32_t st = colptr[c] + (uint32_t)(i - vc_base[c]) * vcmax;
            const uint32_t w = csc_idx[st + vc_len[i] - 1];
            const uint32_t l = (w >> 31) ? e_u[w & 0x7fffffffu] : w;
            const uint32_t h = sb > 16 ? l >> (sb - 16) : l;
            return ((uint64_t)len_class_desc(vc_len[i]) << (vb + 16)) | ((uint64_t)h << vb) | i;
        }
        return ((uint64_t)len_class_desc(vc_len[i]) << vb) | i;
    }
};

struct KeyArraySrc {
    const unsigned long long* keys;
    static constexpr size_t kSmem = 0;
    static constexpr int kHistBatch = 16;
    static constexpr bool kRegPrefetch = true;
    static constexpr bool kL2Prefetch = true;
    __device__ __forceinline__ void prefetch_l2(size_t i) const {
        if ((threadIdx.x & 3u) == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(keys + i));  // one per 32-byte sector
    }
    __device__ void prepare(size_t, int, void*) const {}
    __device__ __forceinline__ uint64_t key(size_t i, int, const void*) const { return keys[i]; }
};

__global__ void slice_size_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ vc_len, uint32_t V,
                                  uint32_t nslices, uint32_t* __restrict__ slice_sz) {
    const uint32_t lane = dev::lane_id();
    for (uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t pos = s * 32 + lane;
        const uint32_t len = pos < V ? vc_len[order[pos]] : 0u;
        const uint32_t mx = __reduce_max_sync(0xffffffffu, len);
        if (lane == 0) slice_sz[s] = 32u * mx;
    }
}

struct FillArgs {
    const uint32_t* order;
    const uint32_t* vc_col;
    const uint32_t* vc_len;
    const uint32_t* vc_base;
    const uint32_t* colptr;
    const uint32_t* csc_idx;
    const uint32_t* slice_ptr;
    uint32_t V, nslices;
    uint32_t n_nd;             // exception entries gather s[n_nd + exception index]
    uint32_t vcmax;            // part length
    uint32_t* sell;
    uint32_t* lane_len;  // [nslices*32]
    uint32_t* lane_col;  // [nslices*32]
    uint32_t* lane_np;   // [nslices*32]
    uint32_t* spos_col;  // [n] pos of part 0 (kEmpty if empty)
    uint32_t* next;      // slice claim counter (zero on entry)
};

// One warp per slice, lane = virtual column. Exception entries (value != row
// base, flagged in the CSC) are redirected to s[n_nd + index], where the
// exception products are stored every iteration — the SpMV has no special case.
__global__ void sell_fill_kernel(FillArgs a) {
    const uint32_t lane = dev::lane_id();
    // slices claimed dynamically (they are sorted longest first: a static
    // stride gave the low warps every round's longest slice)
    for (;;) {
        uint32_t s = 0;
        if (lane == 0) s = atomicAdd(a.next, 1u);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= a.nslices) break;
        const uint32_t pos = s * 32 + lane;
        uint32_t len = 0, c = 0, np = 1, start = 0;
        if (pos < a.V) {
            const uint32_t v = a.order[pos];
            c = a.vc_col[v];
            len = a.vc_len[v];
            const uint32_t part = v - a.vc_base[c];
            np = a.vc_base[c + 1] - a.vc_base[c];
            start = a.colptr[c] + part * a.vcmax;
        }
        a.lane_len[pos] = len;
        a.lane_col[pos] = c;
        a.lane_np[pos] = np;
        const uint32_t base = a.slice_ptr[s];
        const uint32_t rows = (a.slice_ptr[s + 1] - base) >> 5;
        // each lane reads its column through aligned 16-byte loads (3 per 8
        // entries, shifted by the column's misalignment) instead of eight 4-byte
        // loads: 2.7x fewer L1 wavefronts (ncu had the kernel LSU-throttled)
        const uint32_t mis = start & 3u;
        const uint4* asrc = reinterpret_cast<const uint4*>(a.csc_idx + (start - mis));
        uint32_t* dst = a.sell + base + lane;
        for (uint32_t k0 = 0; k0 < rows; k0 += 8) {
            uint32_t e[8];
            if (k0 < len) {
                const uint4 c0 = asrc[k0 / 4], c1 = asrc[k0 / 4 + 1], c2 = asrc[k0 / 4 + 2];
                const uint32_t w[12] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x, c2.y, c2.z, c2.w};
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t x = mis == 0 ? w[u] : mis == 1 ? w[u + 1] : mis == 2 ? w[u + 2] : w[u + 3];
                    e[u] = k0 + u < len ? x : 0x80000000u;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) e[u] = 0x80000000u;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (k0 + u < rows) {
                    uint32_t w = e[u];
                    if (k0 + u < len && (w >> 31)) w = a.n_nd + (w & 0x7fffffffu);
                    dst[32 * (k0 + u)] = w;
                }
            }
        }
    }
}

__global__ void spos_col_kernel(const uint32_t* __restrict__ vc_base, const uint32_t* __restrict__ vpos, int64_t n,
                                uint32_t* __restrict__ spos_col) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v0 = vc_base[c];
        spos_col[c] = vc_base[c + 1] > v0 ? vpos[v0] : kEmpty;
    }
}

__global__ void spos_rows_kernel(const uint32_t* __restrict__ pinv, const uint32_t* __restrict__ spos_col,
                                 int64_t n_nd, uint32_t* __restrict__ spos) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_nd; j += (int64_t)gridDim.x * blockDim.x)
        spos[j] = spos_col[pinv[j]];
}

__global__ void exc_spos_kernel(const uint32_t* __restrict__ e_u, uint32_t n_exc, uint32_t* __restrict__ spos,
                                int64_t n_nd) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n_exc; e += gridDim.x * blockDim.x)
        spos[n_nd + e] = spos[e_u[e]];
}

// Split columns listed in column order (flag + scan + scatter) so that the
// per-iteration sum over them has a fixed order.
__global__ void split_flag_kernel(const uint32_t* __restrict__ vc_base, int64_t n, uint32_t* __restrict__ flag) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        flag[c] = vc_base[c + 1] - vc_base[c] > 1 ? 1u : 0u;
}
__global__ void split_list_kernel(const uint32_t* __restrict__ vc_base, const uint32_t* __restrict__ vpos, int64_t n,
                                  const uint32_t* __restrict__ idx, uint32_t* __restrict__ list) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        if (vc_base[c + 1] - vc_base[c] > 1) list[idx[c]] = (uint32_t)c;
}

__global__ void split_np_kernel(const uint32_t* __restrict__ split_col, const uint32_t* __restrict__ n_split,
                                const uint32_t* __restrict__ vc_base, uint32_t* __restrict__ np_of) {
    const uint32_t ns = *n_split;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
        const uint32_t c = split_col[i];
        np_of[i] = vc_base[c + 1] - vc_base[c];
    }
}
__global__ void split_slots_kernel(const uint32_t* __restrict__ split_col, const uint32_t* __restrict__ n_split,
                                   const uint32_t* __restrict__ vc_base, const uint32_t* __restrict__ vpos,
                                   const uint32_t* __restrict__ pbase, uint32_t* __restrict__ p0,
                                   uint32_t* __restrict__ lane_pslot) {
    const uint32_t ns = *n_split;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
        const uint32_t c = split_col[i], v0 = vc_base[c], np = vc_base[c + 1] - v0, b = pbase[i];
        p0[i] = vpos[v0];
        for (uint32_t p = 0; p < np; ++p) lane_pslot[vpos[v0 + p]] = b + p;
    }
}

// s[j] = r(pinv[j]) * b[j]; r given in original order (first step) or as
// (y in SELL order, bg for empty columns) (later steps).
__global__ void permute_orig_kernel(const double* __restrict__ r, const uint32_t* __restrict__ pinv,
                                    const double* __restrict__ bval, int64_t n_nd, double* __restrict__ s) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_nd; j += (int64_t)gridDim.x * blockDim.x)
        s[j] = __dmul_rn(r[pinv[j]], bval[j]);
}
// s for one iteration, in one launch: s[j] = r(j) * b[j] for rows j < n_nd and
// s[n_nd + e] = r(u_e) * value_e for exception e, where r(x) is the previous
// iterate of new row x (first step: r0 in the original order; then y in SELL
// order, or bg for an empty column).
struct GatherArgs {
    const double* r0;      // first step (original order) or null
    const uint32_t* pinv;
    const double* y;       // previous iterate, SELL order
    const uint32_t* spos;  // new row -> SELL position of its column (kEmpty: empty)
    const double* bgp;     // [2] = bg of the previous iterate
    const double* bval;
    const uint32_t* e_u;
    const double* e_val;
    int64_t n_nd;
    uint32_t n_exc;
    double* s;
    // first step of run_kernel3: r0 = init_rank regenerated on the fly,
    // r0[u] = x_u / sum(x) (no r0 array): rng stream start and device sum(x)
    uint64_t rng_s0;
    const double* rng_div;
};
__global__ void gather_s_kernel(GatherArgs a) {
    const double bg = a.bgp[2];
    const int64_t tot = a.n_nd + a.n_exc;
    const double div = a.rng_div ? *a.rng_div : 1.0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < tot; j += (int64_t)gridDim.x * blockDim.x) {
        const bool row = j < a.n_nd;
        const uint32_t x = row ? (uint32_t)j : a.e_u[j - a.n_nd];
        double r;
        if (a.rng_div) r = __ddiv_rn(rank_init_x(a.rng_s0, a.pinv[x]), div);
        else if (a.r0) r = a.r0[a.pinv[x]];
        else {
            const uint32_t p = a.spos[x];
            r = p == kEmpty ? bg : a.y[p];
        }
        a.s[j] = __dmul_rn(r, row ? a.bval[j] : a.e_val[j - a.n_nd]);
    }
}

// The same for steps >= 2, uniform over [rows | exceptions]: s[j] =
// r(spos[j]) * coef[j] — coalesced spos/coef/s streams and one random read of
// the previous iterate per entry, G entries in flight per thread.
// One extra block (the last) finishes the previous step's Σ instead (what
// sell_sum_final does, same order): out_next = {Σ, bgf * Σ, bg_prev}, one
// launch fewer per step.
struct SumFinish {
    const double* part;  // sell_sum_part's block partials
    int np;
    double n_empty, bgf;
    double* out_next;
};
template <int G>
__global__ void __launch_bounds__(1024, 2) gather_y_kernel(const double* __restrict__ y, const uint32_t* __restrict__ spos,
                                                           const double* __restrict__ coef, const double* __restrict__ bgp,
                                                           int64_t tot, double* __restrict__ s, SumFinish fin) {
    const double bg = bgp[1];  // the bg the previous step used (its empty columns' value)
    if (blockIdx.x == gridDim.x - 1) {
        if (threadIdx.x >= 32) return;
        double v = 0.0;
        for (int i = threadIdx.x; i < fin.np; i += 32) v = __dadd_rn(v, fin.part[i]);
        v = dev::warp_sum_f64(v);
        if (threadIdx.x == 0) {
            const double t = __dadd_rn(v, __dmul_rn(fin.n_empty, bg));
            fin.out_next[0] = t;
            fin.out_next[1] = __dmul_rn(fin.bgf, t);
            fin.out_next[2] = bg;
        }
        return;
    }
    const int64_t stride = (int64_t)(gridDim.x - 1) * blockDim.x;
    for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < tot; j0 += G * stride) {
        uint32_t p[G];
        double c[G], r[G];
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const int64_t j = j0 + k * stride;
            p[k] = j < tot ? spos[j] : kEmpty;
            c[k] = j < tot ? coef[j] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < G; ++k) r[k] = p[k] == kEmpty ? bg : y[p[k]];
#pragma unroll
        for (int k = 0; k < G; ++k) {
            const int64_t j = j0 + k * stride;
            if (j < tot) s[j] = __dmul_rn(r[k], c[k]);
        }
    }
}

// Σ of the iterate, deterministic two-level tree: block b sums slice sums
// [b*chunk, (b+1)*chunk) and split-column values likewise; one warp adds the
// block partials (sell_sum_final). Split columns (cut into parts of vcmax
// entries) are finished here: the SpMV only stores each part's partial sum,
// this kernel adds a column's parts in part order and writes its iterate —
// no cross-CTA handshake (atomics, fences) inside the SpMV.
constexpr int kSumBlocks = 296;
struct SplitArgs {
    const uint32_t* n_split;
    const uint32_t* split_p0;    // split column i: SELL position of its part 0 (its iterate)
    const uint32_t* split_pbase; // [n_split + 1]: its parts' sums at partial[pbase[i] .. pbase[i+1])
    const double* partial;       // compact part sums, column by column in part order
    const double* bgp;           // [1] = bg of this step
    double damping;
};
__global__ void sell_sum_part(const double* __restrict__ slice_sum, uint32_t nslices, double* __restrict__ y,
                              SplitArgs sp, double* __restrict__ part) {
    __shared__ double ws[32];
    const uint32_t ns = *sp.n_split;
    const double bg = sp.bgp[1];
    const uint32_t c1 = (nslices + gridDim.x - 1) / gridDim.x, c2 = (ns + gridDim.x - 1) / gridDim.x;
    double a = 0.0;
    for (uint32_t i = blockIdx.x * c1 + threadIdx.x; i < min(nslices, (blockIdx.x + 1) * c1); i += blockDim.x)
        a = __dadd_rn(a, slice_sum[i]);
    // Split columns of <= kWarpParts parts: one thread each, parts in order;
    // longer ones: one warp each, lane l adds parts l, l+32, ... then a fixed
    // shuffle tree. Both orders are fixed (deterministic). A column's part sums
    // are contiguous (the SpMV writes them to their compact slots), so this is
    // one dependent load level, not three (split list -> virtual columns ->
    // lane positions -> sums).
    constexpr uint32_t kWarpParts = 16;
    const uint32_t i0 = blockIdx.x * c2, i1 = min(ns, (blockIdx.x + 1) * c2);
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const uint32_t pb = sp.split_pbase[i], np = sp.split_pbase[i + 1] - pb;
        if (np > kWarpParts) continue;
        double x[kWarpParts];
#pragma unroll
        for (uint32_t k = 0; k < kWarpParts; ++k) x[k] = k < np ? sp.partial[pb + k] : 0.0;
        double t = 0.0;
#pragma unroll
        for (uint32_t k = 0; k < kWarpParts; ++k)
            if (k < np) t = __dadd_rn(t, x[k]);
        const double yc = __dadd_rn(__dmul_rn(sp.damping, t), bg);
        y[sp.split_p0[i]] = yc;
        a = __dadd_rn(a, yc);
    }
    const unsigned lane = dev::lane_id(), nw = blockDim.x >> 5;
    for (uint32_t i = i0 + dev::warp_id(); i < i1; i += nw) {
        const uint32_t pb = sp.split_pbase[i], np = sp.split_pbase[i + 1] - pb;
        if (np <= kWarpParts) continue;
        double t = 0.0;
        for (uint32_t p = lane; p < np; p += 32) t = __dadd_rn(t, sp.partial[pb + p]);
        t = dev::warp_sum_f64(t);
        const double yc = __dadd_rn(__dmul_rn(sp.damping, t), bg);
        if (lane == 0) {
            y[sp.split_p0[i]] = yc;
            a = __dadd_rn(a, yc);
        }
    }
    a = dev::warp_sum_f64(a);
    if (dev::lane_id() == 0) ws[dev::warp_id()] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        const double v = dev::warp_sum_f64(threadIdx.x < blockDim.x / 32 ? ws[threadIdx.x] : 0.0);
        if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
}
__global__ void sell_sum_final(const double* __restrict__ part, int np, double n_empty, double bgf,
                               double* __restrict__ out) {
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) v = __dadd_rn(v, part[i]);
    v = dev::warp_sum_f64(v);
    if (threadIdx.x == 0) {
        const double bg_cur = out[1];
        const double tot = __dadd_rn(v, __dmul_rn(n_empty, bg_cur));
        out[0] = tot;
        out[2] = bg_cur;
        out[1] = __dmul_rn(bgf, tot);
    }
}

// Final un-permutation: ranks[c] = y[spos_col[c]] or bg.
__global__ void unpermute_kernel(const double* __restrict__ y, const uint32_t* __restrict__ spos_col,
                                 const double* __restrict__ bgp, int64_t n, double* __restrict__ out) {
    const double bg = bgp[2];
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = spos_col[c];
        out[c] = p == kEmpty ? bg : y[p];
    }
}

struct SellArgs {
    const uint32_t* sell;
    const uint32_t* slice_ptr;
    const uint32_t* lane_len;
    const uint32_t* lane_col;
    const uint32_t* lane_np;
    const uint32_t* vc_base;
    const uint32_t* vpos;
    const double* s;             // gather vector [n_nd + n_exc]
    double* y;                   // [nslices*32]
    double* partial;             // compact part sums of split columns
    const uint32_t* lane_pslot;  // lane -> its slot in partial (parts of split columns)
    double* slice_sum;           // [nslices]
    const double* bgp;           // [1] = bg of this step
    uint32_t* next_slice;        // work counters of this launch (32 words apart, start at 0)
    uint32_t nctr;
    int64_t n_nd;
    uint32_t nslices;
    uint32_t slice_begin = 0;    // this launch covers slices [slice_begin, slice_end) (a
    uint32_t slice_end = 0;      // shard of a multi-GPU K3; the whole list on one GPU)
    double damping;
    uint64_t n_s = 0;            // length of s (checked builds: gather bounds)
    uint32_t hot = 0;            // PRG_SPMV_VARIANT 2..5: s[0, hot) gathers take the "hot" L1 priority
};


// 48 warps per SM and no shared-memory staging: measured on B200 (S=24) the L1
// caches the hot, degree-ordered head of s by itself, and occupancy (requests
// in flight) matters more than a software-managed hot set (1.9 ms vs 3.3 ms).
template <int U, int kThreads = kSpmvThreads, int kMinBlocks = 2, int GM = 0>
__global__ void __launch_bounds__(kThreads, kMinBlocks) spmv_sell_kernel(SellArgs a) {
    const unsigned lane = dev::lane_id();
    const double bg = a.bgp[1];
    const uint64_t pol_stream = dev::policy_evict_first(), pol_keep = dev::policy_evict_last();
    // Slices are handed out dynamically, longest first (they are sorted by length
    // class): a static round-robin left some SMs with twice the average work.
    // Slices are claimed from nctr counters (one 128-B line each, so on
    // different L2 slices): counter k hands out slices k, k + nctr, ...; a warp
    // starts at its own counter and moves on when that one runs dry. With a
    // single counter the launch time depended on that counter's address
    // (0.80-0.86 ms over pool placements at S=24), i.e. on the L2 slice serving
    // ~250K claims per launch; 8 counters: 0.783 ms at every placement
    // (tools/exp_spmv4.py; 4: 0.799, 16: 0.794).
    const uint32_t nctr = a.nctr;
    uint32_t k = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) % nctr, tried = 0;
    for (;;) {
        uint32_t sl = 0;
        if (lane == 0) sl = a.slice_begin + atomicAdd(a.next_slice + 32 * k, 1u) * nctr + k;
        sl = __shfl_sync(0xffffffffu, sl, 0);
        if (sl >= a.slice_end) {
            if (++tried == nctr) break;
            k = k + 1 == nctr ? 0 : k + 1;
            continue;
        }
        const uint32_t pos = sl * 32 + lane;
        const uint32_t len = a.lane_len[pos];
        const uint32_t base = a.slice_ptr[sl];
        const uint32_t rows = (a.slice_ptr[sl + 1] - base) >> 5;
        const uint32_t* col = a.sell + base + lane;
        double acc = 0.0;
        // Two-stage pipeline: index loads of batch b+1 are issued before batch
        // b's gathers are consumed. Loads are predicated, never branched.
        uint32_t w[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            w[u] = dev::ld_stream_u32_pred(col + 32 * u, (uint32_t)u < len, pol_stream, 0x80000000u);
        for (uint32_t k0 = 0; k0 < rows; k0 += U) {
            double x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                PRG_DCHECK((w[u] >> 31) || w[u] < a.n_s);
                const uint32_t gi = w[u] & 0x7fffffffu;
                if (GM == 0) x[u] = dev::ld_keep_f64_pred(a.s + gi, !(w[u] >> 31), pol_keep);
                else if (GM == 2) x[u] = dev::ld_hotcold_1_2(a.s + gi, !(w[u] >> 31), gi < a.hot, pol_keep);
                else if (GM == 3) x[u] = dev::ld_hotcold_0_2(a.s + gi, !(w[u] >> 31), gi < a.hot, pol_keep);
                else if (GM == 4) x[u] = dev::ld_hotcold_1_0(a.s + gi, !(w[u] >> 31), gi < a.hot, pol_keep);
                else x[u] = dev::ld_hotcold_0_3(a.s + gi, !(w[u] >> 31), gi < a.hot, pol_keep);
            }
            const uint32_t k1 = k0 + U;
#pragma unroll
            for (int u = 0; u < U; ++u)
                w[u] = dev::ld_stream_u32_pred(col + 32 * (k1 + u), k1 + u < len, pol_stream, 0x80000000u);
#pragma unroll
            for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, x[u]);
        }
        const uint32_t np = a.lane_np[pos];
        double yv = 0.0;
        if (len > 0 && np == 1) {
            yv = __dadd_rn(__dmul_rn(a.damping, acc), bg);
            a.y[pos] = yv;
        } else if (len > 0) {
            // a part of a split column: its sum is finished by sell_sum_part
            // (a cross-CTA handshake here, __threadfence + atomics, emitted
            // CCTL.IVALL and cost the hot rows' L1 lines: 0.766 vs 0.737 ms
            // even as release increments)
            a.partial[a.lane_pslot[pos]] = acc;
        }
        yv = dev::warp_sum_f64(yv);
        if (lane == 0) a.slice_sum[sl] = yv;
    }
}


__global__ void count_set_kernel(const uint32_t* __restrict__ a, int64_t n, uint32_t* __restrict__ out) {
    uint32_t c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += a[i] != kEmpty;
    c = __reduce_add_sync(0xffffffffu, c);
    if (dev::lane_id() == 0 && c) atomicAdd(out, c);
}

// ---------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------
void suffix_min_inplace(uint32_t* a, int64_t n1, cudaStream_t s) {
    const int64_t nb = (n1 + 8191) / 8192;
    if (nb <= 1) {
        suffix_min_down<<<1, 1024, 0, s>>>(a, n1, nullptr, 1);
        PRG_LAUNCH_CHECK();
        return;
    }
    DevBuf<uint32_t> part((size_t)nb, s);
    suffix_min_block<<<(unsigned)nb, 1024, 0, s>>>(a, n1, part.get());
    PRG_LAUNCH_CHECK();
    suffix_min_inplace(part.get(), nb, s);
    suffix_min_down<<<(unsigned)nb, 1024, 0, s>>>(a, n1, part.get(), nb);
    PRG_LAUNCH_CHECK();
}

void build_plan(const prg_matrix* A, int mode, K3Plan& P, cudaStream_t s) {
    ProfScope prof("k3_prep", s);
    const int64_t n = A->n;
    const uint64_t nnz = A->nnz;
    P.n = n;
    P.nnz = nnz;
    P.mode = mode;
    P.sb = bits_for(n);
    P.pb = std::max(P.sb, bits_for((int64_t)nnz));
    if (P.sb + P.pb + 1 > 64 || P.pb > 31) throw CudaError{"K3: matrix too large for u32 indices"};
    const unsigned g = (unsigned)num_sms() * 8;
    P.pinv = DevBuf<uint32_t>((size_t)n, s);
    P.newid = DevBuf<uint32_t>((size_t)n, s);
    // 1. row renumbering (timed: hot rows first, dangling last; parity: identity)
    {
        ProfScope pr("k3_prep_rows", s);
        if (mode == 0) {
            // Dangling rows keep their relative order after all others (they are
            // never gathered); only the non-dangling rows are sorted.
            DevBuf<uint32_t> flag((size_t)n, s), pos((size_t)n + 1, s);
            nondangling_flag_kernel<<<g, 1024, 0, s>>>(A->row_offsets, n, flag.get());
            PRG_LAUNCH_CHECK();
            exclusive_scan_u32(flag.get(), pos.get(), (size_t)n, pos.get() + n, s);
            uint32_t h = 0;
            PRG_CUDA(cudaMemcpyAsync(&h, pos.get() + n, 4, cudaMemcpyDeviceToHost, s));
            PRG_CUDA(cudaStreamSynchronize(s));
            P.n_nd = (int64_t)h;
            static int ro_bits = -1;  // PRG_ROW_ORDER_BITS: column bits of the row order (default 16, 0 = off)
            if (ro_bits < 0) { const char* e = getenv("PRG_ROW_ORDER_BITS"); ro_bits = e ? atoi(e) : 16; }
            const int ro_exp = ro_bits > 0;
            const int fb = ro_exp ? std::min(P.sb, std::min(ro_bits, 24)) : 0;
            DevBuf<unsigned long long> keys((size_t)std::max<int64_t>(P.n_nd, 1), s);
            row_keys_kernel<<<g, 1024, 0, s>>>(
                RowClassSrc{A->row_offsets, P.sb, ro_exp ? A->cols : nullptr, fb}, n, pos.get(), keys.get(),
                P.pinv.get(), P.newid.get(), (uint32_t)P.n_nd);
            PRG_LAUNCH_CHECK();
            if (P.n_nd) {
                sort::SortWorkspace ws;
                sort::msd_sort(KeyArraySrc{keys.get()}, (size_t)P.n_nd, P.sb + 8 + fb,
                               PermDst{P.pinv.get(), P.newid.get(), P.sb}, ws, s, "k3rows", /*payload_bits=*/P.sb,
                               /*stable=*/true);
            }
        } else {
            iota_kernel<<<g, 1024, 0, s>>>(P.pinv.get(), P.newid.get(), n);
            PRG_LAUNCH_CHECK();
            P.n_nd = n;
        }
    }
    // 2. row base values (minimum stored value of each row) and the shift of
    //    every row to its place in the new row order
    const int64_t nr = P.n_nd;  // non-dangling rows (dangling rows are last in the new order)
    DevBuf<unsigned long long> bmin((size_t)n, s);
    DevBuf<uint32_t> wdelta;
    const uint32_t ntiles = nnz ? div_up(nnz, sort::kTile) : 0;
    DevBuf<uint32_t> tile_row(ntiles + 1, s);
    const size_t row_smem = kRowWords * sizeof(uint32_t);
    {
        ProfScope pr("k3_prep_base", s);
        if (mode == 0) {
            DevBuf<uint32_t> deg((size_t)std::max<int64_t>(nr, 1), s), pro((size_t)nr + 1, s);
            wdelta = DevBuf<uint32_t>((size_t)n, s);
            perm_degree_kernel<<<g, 1024, 0, s>>>(A->row_offsets, P.pinv.get(), nr, deg.get());
            PRG_LAUNCH_CHECK();
            exclusive_scan_u32(deg.get(), pro.get(), (size_t)nr, pro.get() + nr, s);
            perm_delta_kernel<<<g, 1024, 0, s>>>(A->row_offsets, P.newid.get(), pro.get(), n, nr, wdelta.get());
            PRG_LAUNCH_CHECK();
        }
        if (nnz) {
            tile_rows_kernel<<<g, 1024, 0, s>>>(A->row_offsets, n, tile_row.get());
            PRG_LAUNCH_CHECK();
        }
        row_base_kernel<<<g, 256, 0, s>>>(A->row_offsets, A->values, n, bmin.get());
        PRG_LAUNCH_CHECK();
        P.bval = DevBuf<double>((size_t)std::max<int64_t>(nr, 1), s);
        gather_base_kernel<<<g, 1024, 0, s>>>(P.pinv.get(), bmin.get(), nr, P.bval.get());
        PRG_LAUNCH_CHECK();
    }
    // 3. transpose: stable sort of (col | new row, exception) keys by column
    P.colptr = DevBuf<uint32_t>((size_t)n + 1, s);
    P.csc_idx = DevBuf<uint32_t>((nnz ? nnz : 1) + 16, s);  // +16: sell_fill's aligned 16-byte reads run past the end
    // exception list, capacity nnz until its size is known
    DevBuf<uint32_t> e_u(nnz ? nnz : 1, s);
    DevBuf<double> e_val(nnz ? nnz : 1, s);
    DevBuf<uint32_t> n_exc(1, s);
    {
        ProfScope pr("k3_prep_transpose", s);
        PRG_CUDA(cudaMemsetAsync(P.colptr.get(), 0xff, (size_t)(n + 1) * 4, s));
        PRG_CUDA(cudaMemsetAsync(n_exc.get(), 0, 4, s));
        if (nnz) {
            sort::SortWorkspace ws;
            sort::sort_workspace_init(ws, (size_t)nnz, s);
            {
                ProfScope pk("k3t_keys", s);
                KeyBuildArgs ka{A->row_offsets, tile_row.get(), A->cols, A->values, bmin.get(),
                                mode == 0 ? P.newid.get() : nullptr, mode == 0 ? wdelta.get() : nullptr, n, nnz, P.pb,
                                reinterpret_cast<unsigned long long*>(ws.keys[0].get()), e_u.get(), e_val.get(),
                                n_exc.get()};
                // 4 CTAs per SM (32 registers, 34 KB row table each): 1.60 ms vs 1.73 ms
                // at 3 (ncu: long-scoreboard bound; 2 CTAs x unroll 16: 2.39 ms)
                key_build_kernel<<<num_sms() * 4, sort::kTileThreads, row_smem, s>>>(ka);
                PRG_LAUNCH_CHECK();
            }
            // the keys live in ws.keys[0]; level 1 reads them before any pass overwrites that buffer.
            // (row or exception index, exception flag) ride as payload: only column bits are sorted
            const KeyArraySrc src{reinterpret_cast<const unsigned long long*>(ws.keys[0].get())};
            sort::msd_sort_split(src, src, (size_t)nnz, P.sb + P.pb + 1,
                                 CscDst{P.csc_idx.get(), P.colptr.get(), P.pb}, ws, s, "k3t",
                                 /*payload_bits=*/P.pb + 1, /*stable=*/true);
        }
        // colptr[n] = nnz, then fill empty columns with the next column start.
        const uint32_t nz = (uint32_t)nnz;
        PRG_CUDA(cudaMemcpyAsync(P.colptr.get() + n, &nz, 4, cudaMemcpyHostToDevice, s));
        suffix_min_inplace(P.colptr.get(), n + 1, s);
    }
    PRG_CUDA(cudaMemcpyAsync(&P.n_exc, n_exc.get(), 4, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    P.exc_val = DevBuf<double>(P.n_exc ? P.n_exc : 1, s);
    P.e_u = DevBuf<uint32_t>(P.n_exc ? P.n_exc : 1, s);
    if (P.n_exc) {
        PRG_CUDA(cudaMemcpyAsync(P.e_u.get(), e_u.get(), (size_t)P.n_exc * 4, cudaMemcpyDeviceToDevice, s));
        PRG_CUDA(cudaMemcpyAsync(P.exc_val.get(), e_val.get(), (size_t)P.n_exc * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (mode == 1) return;
    // 4. SELL over virtual columns
    ProfScope pr("k3_prep_sell", s);
    // Part length: short enough that the longest lane chain (one sequential
    // gather stream) stays well under the whole SpMV on small graphs.
    // Measured on B200 (SpMV ms): S=24 512: 0.797, 384/768: 0.82, 2048: 0.834;
    // S=20 128-256: 0.085; S=16 64: 0.027 vs 2048: 0.159; S=26 (handshake-free SpMV) 512: 3.26 vs
    // 1024: 3.32 vs 2048: 3.34 (with the split handshake in the SpMV, 1024 had won: 3.51 vs 3.63).
    uint32_t vcmax = nnz >= (1ull << 27) ? 512u : nnz >= (1ull << 23) ? 256u : nnz >= (1ull << 20) ? 128u : 64u;
    {
        static int env = -1;
        if (env < 0) { const char* e = getenv("PRG_VCMAX"); env = e ? atoi(e) : 0; }
        if (env > 0) vcmax = (uint32_t)env;
    }
    DevBuf<uint32_t> np((size_t)n, s);
    P.vc_base = DevBuf<uint32_t>((size_t)n + 1, s);
    vc_count_kernel<<<g, 1024, 0, s>>>(P.colptr.get(), n, vcmax, np.get());
    PRG_LAUNCH_CHECK();
    exclusive_scan_u32(np.get(), P.vc_base.get(), (size_t)n, P.vc_base.get() + n, s);
    PRG_CUDA(cudaMemcpyAsync(&P.V, P.vc_base.get() + n, 4, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    const uint32_t V = P.V;
    P.nslices = (V + 31) / 32;
    const uint32_t NP = P.nslices * 32;
    DevBuf<uint32_t> vc_col(V ? V : 1, s), vc_len(V ? V : 1, s), order(NP ? NP : 1, s);
    P.vpos = DevBuf<uint32_t>(V ? V : 1, s);
    vc_fill_kernel<<<g, 1024, 0, s>>>(P.colptr.get(), P.vc_base.get(), n, vcmax, vc_col.get(), vc_len.get());
    PRG_LAUNCH_CHECK();
    if (V) {
        sort::SortWorkspace ws;
        const int vb = bits_for(V);
        static int co = -1;  // PRG_COL_ORDER=0: length class only
        if (co < 0) { const char* e = getenv("PRG_COL_ORDER"); co = e ? atoi(e) : 1; }
        sort::msd_sort(VcClassSrc{vc_len.get(), vb, vc_col.get(), P.vc_base.get(), P.colptr.get(),
                                  co ? P.csc_idx.get() : nullptr, P.e_u.get(), P.sb, vcmax},
                       (size_t)V, vb + 8 + (co ? 16 : 0), PermDst{order.get(), P.vpos.get(), vb}, ws, s,
                       "k3vc", /*payload_bits=*/vb, /*stable=*/true);
    }
    DevBuf<uint32_t> slice_sz(P.nslices ? P.nslices : 1, s);
    P.slice_ptr = DevBuf<uint32_t>((size_t)P.nslices + 1, s);
    if (P.nslices) {
        slice_size_kernel<<<g, 256, 0, s>>>(order.get(), vc_len.get(), V, P.nslices, slice_sz.get());
        PRG_LAUNCH_CHECK();
    }
    exclusive_scan_u32(slice_sz.get(), P.slice_ptr.get(), P.nslices, P.slice_ptr.get() + P.nslices, s);
    uint32_t sell_n = 0;
    PRG_CUDA(cudaMemcpyAsync(&sell_n, P.slice_ptr.get() + P.nslices, 4, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    P.sell = DevBuf<uint32_t>(sell_n ? sell_n : 1, s);
    P.lane_len = DevBuf<uint32_t>(NP ? NP : 1, s);
    P.lane_col = DevBuf<uint32_t>(NP ? NP : 1, s);
    P.lane_np = DevBuf<uint32_t>(NP ? NP : 1, s);
    P.spos_col = DevBuf<uint32_t>((size_t)n, s);
    // SELL position of every column's part 0 (kEmpty: empty column), a gather
    // through vpos in column order
    spos_col_kernel<<<g, 1024, 0, s>>>(P.vc_base.get(), P.vpos.get(), n, P.spos_col.get());
    PRG_LAUNCH_CHECK();
    if (P.nslices) {
        FillArgs fa{order.get(),         vc_col.get(),     vc_len.get(), P.vc_base.get(),   P.colptr.get(),
                    P.csc_idx.get(),     P.slice_ptr.get(), V,                P.nslices,
                    (uint32_t)P.n_nd,    vcmax,            P.sell.get(),     P.lane_len.get(),  P.lane_col.get(),
                    P.lane_np.get(),     P.spos_col.get(),     nullptr};
        DevBuf<uint32_t> fill_ctr(1, s);
        PRG_CUDA(cudaMemsetAsync(fill_ctr.get(), 0, 4, s));
        fa.next = fill_ctr.get();
        sell_fill_kernel<<<g, 256, 0, s>>>(fa);
        PRG_LAUNCH_CHECK();
    }
    P.spos = DevBuf<uint32_t>((size_t)std::max<int64_t>(P.n_nd + P.n_exc, 1), s);
    P.coef = DevBuf<double>((size_t)std::max<int64_t>(P.n_nd + P.n_exc, 1), s);
    spos_rows_kernel<<<g, 1024, 0, s>>>(P.pinv.get(), P.spos_col.get(), P.n_nd, P.spos.get());
    PRG_LAUNCH_CHECK();
    if (P.n_nd)
        PRG_CUDA(cudaMemcpyAsync(P.coef.get(), P.bval.get(), (size_t)P.n_nd * 8, cudaMemcpyDeviceToDevice, s));
    if (P.n_exc) {
        PRG_CUDA(cudaMemcpyAsync(P.coef.get() + P.n_nd, P.exc_val.get(), (size_t)P.n_exc * 8,
                                 cudaMemcpyDeviceToDevice, s));
        exc_spos_kernel<<<g, 1024, 0, s>>>(P.e_u.get(), P.n_exc, P.spos.get(), P.n_nd);
        PRG_LAUNCH_CHECK();
    }
    P.split_col = DevBuf<uint32_t>((size_t)n, s);
    P.n_split = DevBuf<uint32_t>(1, s);
    PRG_CUDA(cudaMemsetAsync(P.n_split.get(), 0, 4, s));
    if (n > 0) {
        DevBuf<uint32_t> flag((size_t)n, s), idx((size_t)n, s);
        split_flag_kernel<<<g, 1024, 0, s>>>(P.vc_base.get(), n, flag.get());
        PRG_LAUNCH_CHECK();
        exclusive_scan_u32(flag.get(), idx.get(), (size_t)n, P.n_split.get(), s);
        split_list_kernel<<<g, 1024, 0, s>>>(P.vc_base.get(), P.vpos.get(), n, idx.get(), P.split_col.get());
        PRG_LAUNCH_CHECK();
    }
    // compact part sums: split column i's parts at [pbase[i], pbase[i+1]); the
    // SpMV lane of part p writes slot pbase[i] + p (lane_pslot)
    P.split_p0 = DevBuf<uint32_t>((size_t)n, s);
    P.split_pbase = DevBuf<uint32_t>((size_t)n + 1, s);
    P.lane_pslot = DevBuf<uint32_t>(NP ? NP : 1, s);
    uint32_t n_parts = 0;
    if (n > 0) {
        DevBuf<uint32_t> np_of((size_t)n, s);
        split_np_kernel<<<g, 1024, 0, s>>>(P.split_col.get(), P.n_split.get(), P.vc_base.get(), np_of.get());
        PRG_LAUNCH_CHECK();
        exclusive_scan_u32_prefix(np_of.get(), P.split_pbase.get(), (size_t)n, P.n_split.get(), 1, s);
        split_slots_kernel<<<g, 256, 0, s>>>(P.split_col.get(), P.n_split.get(), P.vc_base.get(), P.vpos.get(),
                                             P.split_pbase.get(), P.split_p0.get(), P.lane_pslot.get());
        PRG_LAUNCH_CHECK();
        uint32_t ns_h = 0;
        PRG_CUDA(cudaMemcpyAsync(&ns_h, P.n_split.get(), 4, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        if (ns_h) {
            uint32_t last[2] = {0, 0};
            PRG_CUDA(cudaMemcpyAsync(last, P.split_pbase.get() + ns_h - 1, 4, cudaMemcpyDeviceToHost, s));
            PRG_CUDA(cudaMemcpyAsync(last + 1, np_of.get() + ns_h - 1, 4, cudaMemcpyDeviceToHost, s));
            PRG_CUDA(cudaStreamSynchronize(s));
            n_parts = last[0] + last[1];
            PRG_CUDA(cudaMemcpyAsync(P.split_pbase.get() + ns_h, &n_parts, 4, cudaMemcpyHostToDevice, s));
        }
    }
    P.partial = DevBuf<double>(n_parts ? n_parts : 1, s);
    // empty columns = columns with no virtual column
    uint32_t nonempty = 0;
    {
        DevBuf<uint32_t> ne(1, s);
        PRG_CUDA(cudaMemsetAsync(ne.get(), 0, 4, s));
        // count columns whose part-0 position was set
        count_set_kernel<<<g, 1024, 0, s>>>(P.spos_col.get(), n, ne.get());
        PRG_LAUNCH_CHECK();
        PRG_CUDA(cudaMemcpyAsync(&nonempty, ne.get(), 4, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
    }
    P.n_empty = (uint32_t)(n - nonempty);
    if (getenv("PRG_DEBUG"))
        fprintf(stderr, "[k3 plan] n=%lld nnz=%llu n_nd=%lld V=%u nslices=%u sell_n=%u (pad %.3f) n_exc=%u n_empty=%u\n",
                (long long)n, (unsigned long long)nnz, (long long)P.n_nd, V, P.nslices, sell_n,
                nnz ? (double)sell_n / (double)nnz : 0.0, P.n_exc, P.n_empty);
    // the CSC itself is no longer needed in timed mode
    P.csc_idx = DevBuf<uint32_t>();
}

// The layout kept on the handle when it matches the mode, else one built now
// (inside the caller's timed region) into `tmp`.
const K3Plan& plan_for(const prg_matrix* A, int mode, K3Plan& tmp, cudaStream_t s) {
    mode = mode == 0 ? 0 : 1;  // the Neumaier mode runs on the parity layout
    if (A->plan && A->plan->mode == mode) return *A->plan;
    build_plan(A, mode, tmp, s);
    return tmp;
}

// ---------------------------------------------------------------------------
// Drivers
// ---------------------------------------------------------------------------
struct Sums {
    DevBuf<double> part, out;  // out[0] = sum, out[1] = bg for the next step, out[2] = bg of the current iterate
};

// sum(x) into out[0] and ((1-c)/n)*sum into out[1], deterministic.
void device_sum(const double* x, int64_t n, double bgf, int mode, Sums& S, cudaStream_t s) {
    if (!S.out.get()) {
        S.out = DevBuf<double>(4, s);
        PRG_CUDA(cudaMemsetAsync(S.out.get(), 0, 32, s));
    }
    if (mode == 1) {
        seq_sum_kernel<<<1, 1, 0, s>>>(x, n, bgf, S.out.get());
    } else if (mode == 2) {
        seq_neumaier_kernel<<<1, 1, 0, s>>>(x, n, bgf, S.out.get());
    } else {
        const int64_t nb = (n + 8191) / 8192;
        if (S.part.n < (size_t)nb) S.part = DevBuf<double>((size_t)nb, s);
        partial_sum_kernel<<<(unsigned)nb, 1024, 0, s>>>(x, n, S.part.get());
        final_sum_kernel<<<1, 1024, 0, s>>>(S.part.get(), nb, bgf, S.out.get());
    }
    PRG_LAUNCH_CHECK();
}

double read_scalar(const double* d, cudaStream_t s) {
    double h = 0;
    PRG_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    return h;
}

// init_rank into d_r; leaves S.out = {norm1, bg(norm1)}.
void init_rank_impl(int64_t n, uint64_t seed, double* d_r, int mode, double bgf, Sums& S, cudaStream_t s) {
    const unsigned g = (unsigned)num_sms() * 8;
    rng_kernel<<<g, 1024, 0, s>>>(d_r, n, dev::mix_seed(seed, kRankInitStream));
    PRG_LAUNCH_CHECK();
    device_sum(d_r, n, bgf, mode, S, s);
    scale_kernel<<<g, 1024, 0, s>>>(d_r, n, S.out.get());
    PRG_LAUNCH_CHECK();
    device_sum(d_r, n, bgf, mode, S, s);
}


// Runs `iters` steps from r_in (original order, S.out = {sum(r_in), bg}) and
// writes the final iterate to r_out (original order); S.out ends as
// {sum(r_out), bg', bg_used}.
// Multi-GPU K3 (column-sharded): this rank runs the SpMV over its own SELL
// slices only; every other per-iteration step is replicated. After the SpMV the
// rank's iterate values, split-column part sums and slice sums — written into
// a zeroed exchange buffer, every element by exactly one rank — are combined
// by an all-reduce(sum) the caller provides (NCCL over NVLink: x + 0 is exact,
// so every rank then holds bit-for-bit the single-GPU arrays and the rest of
// the step, Σ included, is the single-GPU computation).
struct Shard {
    int rank = 0, world = 1;
    prg_allreduce_f64 allreduce = nullptr;
    void* user = nullptr;
};

// Contiguous slice ranges with near-equal SELL entries (slices are sorted
// longest first, so equal slice counts would not balance).
void shard_bounds_host(const uint32_t* slice_ptr, uint32_t nslices, int world, uint32_t* bounds) {
    const uint64_t total = slice_ptr[nslices];
    uint32_t sl = 0;
    bounds[0] = 0;
    for (int r = 1; r < world; ++r) {
        const uint64_t want = total * (uint64_t)r / (uint64_t)world;
        while (sl < nslices && slice_ptr[sl] < want) ++sl;
        bounds[r] = sl;
    }
    bounds[world] = nslices;
}

void iterate(const K3Plan& P, const double* r_in, double* r_out, int iters, double damping, double bgf, Sums& S,
             cudaStream_t s, uint64_t rng_s0 = 0, const double* rng_div = nullptr, int sum_mode = 1,
             const Shard* shard = nullptr) {
    const unsigned g = (unsigned)num_sms() * 8;
    const int64_t n = P.n;
    if (P.mode == 1) {
        DevBuf<double> sb((size_t)n, s), tA((size_t)n, s), tB((size_t)n, s);
        const double* cur = r_in;
        for (int it = 0; it < iters; ++it) {
            double* dst = (it & 1) ? tB.get() : tA.get();
            permute_orig_kernel<<<g, 1024, 0, s>>>(cur, P.pinv.get(), P.bval.get(), n, sb.get());
            PRG_LAUNCH_CHECK();
            SeqArgs a{P.colptr.get(), P.csc_idx.get(), P.e_u.get(), P.exc_val.get(), sb.get(), cur,
                      S.out.get(), dst, n, damping};
            spmv_seq_kernel<<<g, 256, 0, s>>>(a);
            PRG_LAUNCH_CHECK();
            device_sum(dst, n, bgf, sum_mode, S, s);
            cur = dst;
        }
        if (cur != r_out) PRG_CUDA(cudaMemcpyAsync(r_out, cur, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
        return;
    }
    static int variant = -1;
    if (variant < 0) {
        const char* v = getenv("PRG_SPMV_VARIANT");
        variant = v ? atoi(v) : 0;
    }
    static int hot_rows = -1;  // PRG_HOT_ROWS: length of the "hot" head of s for variants 2..5
    if (hot_rows < 0) {
        const char* v = getenv("PRG_HOT_ROWS");
        hot_rows = v ? atoi(v) : 16384;
    }
    const uint32_t NP = P.nslices * 32;
    // s = [row-scaled iterate (SELL row order, n_nd) | exception products (n_exc)]
    DevBuf<double> sbuf((size_t)std::max<int64_t>(P.n_nd + P.n_exc, 1), s), y0(NP ? NP : 1, s), y1(NP ? NP : 1, s),
        slice_sum(P.nslices ? P.nslices : 1, s), sum_part(kSumBlocks, s);
    // sharded: two exchange buffers [y (NP) | part sums (n_parts) | slice sums (nslices)]
    uint32_t sl_begin = 0, sl_end = P.nslices;
    size_t n_parts = 0, xcount = 0;
    DevBuf<double> xb0, xb1;
    // PRG_SHARD_EXCHANGE_ALWAYS=1: a world of one still goes through the exchange
    // (the one-GPU dry run of the multi-GPU path: tests, bench PRG_BENCH_FORCE_DIST)
    static const bool exchange_always = [] { const char* e = getenv("PRG_SHARD_EXCHANGE_ALWAYS"); return e && atoi(e) != 0; }();
    if (shard && (shard->world > 1 || exchange_always)) {
        std::vector<uint32_t> sp((size_t)P.nslices + 1), bounds((size_t)shard->world + 1);
        PRG_CUDA(cudaMemcpyAsync(sp.data(), P.slice_ptr.get(), sp.size() * 4, cudaMemcpyDeviceToHost, s));
        uint32_t nsp = 0;
        PRG_CUDA(cudaMemcpyAsync(&nsp, P.n_split.get(), 4, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        shard_bounds_host(sp.data(), P.nslices, shard->world, bounds.data());
        sl_begin = bounds[(size_t)shard->rank];
        sl_end = bounds[(size_t)shard->rank + 1];
        uint32_t pb_end = 0;
        if (nsp) PRG_CUDA(cudaMemcpy(&pb_end, P.split_pbase.get() + nsp, 4, cudaMemcpyDeviceToHost));
        n_parts = pb_end;
        xcount = (size_t)NP + n_parts + P.nslices;
        xb0 = DevBuf<double>(xcount ? xcount : 1, s);
        xb1 = DevBuf<double>(xcount ? xcount : 1, s);
    }
    const bool sharded = xcount > 0;
    auto y_of = [&](int side) { return sharded ? (side ? xb1.get() : xb0.get()) : (side ? y1.get() : y0.get()); };
    auto partial_of = [&](int side) { return sharded ? y_of(side) + NP : P.partial.get(); };
    auto slice_sum_of = [&](int side) { return sharded ? y_of(side) + NP + n_parts : slice_sum.get(); };
    static int nctr = -1;  // PRG_NCTR: slice counters per launch
    if (nctr < 0) { const char* e = getenv("PRG_NCTR"); nctr = e ? std::max(1, atoi(e)) : kSliceCounters; }
    const size_t ctr_words = (size_t)std::max(iters, 1) * 32 * nctr;
    DevBuf<uint32_t> slice_ctr(ctr_words, s);
    PRG_CUDA(cudaMemsetAsync(slice_ctr.get(), 0, ctr_words * 4, s));
    double* ys[2] = {y_of(0), y_of(1)};
    // Scalars {Σ, bg, bg of the step before} of step k's input iterate: step 0
    // reads S.out; step k >= 1 reads a slot written by the gather launch that
    // starts it (block 0 finishes step k-1's Σ), alternating so a launch never
    // overwrites the slot it reads.
    DevBuf<double> outs(8, s);
    auto out_of = [&](int k) { return k == 0 ? S.out.get() : outs.get() + 4 * (k & 1); };
    for (int it = 0; it < iters; ++it) {
        double* y = ys[it & 1];
        const double* yp = ys[(it & 1) ^ 1];
        {
            ProfScope pp("k3_permute", s);
            GatherArgs ga{it == 0 ? r_in : nullptr, P.pinv.get(), yp, P.spos.get(), S.out.get(), P.bval.get(),
                          P.e_u.get(), P.exc_val.get(), P.n_nd, P.n_exc, sbuf.get(), rng_s0,
                          it == 0 ? rng_div : nullptr};
            const int64_t tot = P.n_nd + P.n_exc;
            static int gi = -1;  // PRG_GATHER_ITEMS (1, 2, 4)
            if (gi < 0) { const char* e = getenv("PRG_GATHER_ITEMS"); gi = e ? atoi(e) : 4; }
            if (it == 0) {
                if (tot) gather_s_kernel<<<g, 1024, 0, s>>>(ga);
            } else {  // launched even with tot == 0: block 0 finishes the previous Σ
                const unsigned gg = 1 + (unsigned)std::max<int64_t>(1, std::min<int64_t>(g - 1, (tot + 1023) / 1024 / gi));
                const SumFinish fin{sum_part.get(), kSumBlocks, (double)P.n_empty, bgf, out_of(it)};
                const double* bgp = out_of(it - 1);
                if (gi == 4) gather_y_kernel<4><<<gg, 1024, 0, s>>>(yp, P.spos.get(), P.coef.get(), bgp, tot, sbuf.get(), fin);
                else if (gi == 1) gather_y_kernel<1><<<gg, 1024, 0, s>>>(yp, P.spos.get(), P.coef.get(), bgp, tot, sbuf.get(), fin);
                else gather_y_kernel<2><<<gg, 1024, 0, s>>>(yp, P.spos.get(), P.coef.get(), bgp, tot, sbuf.get(), fin);
            }
            PRG_LAUNCH_CHECK();
        }
        SellArgs a;
        a.sell = P.sell.get();
        a.slice_ptr = P.slice_ptr.get();
        a.lane_len = P.lane_len.get();
        a.lane_col = P.lane_col.get();
        a.lane_np = P.lane_np.get();
        a.vc_base = P.vc_base.get();
        a.vpos = P.vpos.get();
        a.s = sbuf.get();
        a.y = y;
        a.partial = partial_of(it & 1);
        a.lane_pslot = P.lane_pslot.get();
        a.slice_sum = slice_sum_of(it & 1);
        a.bgp = out_of(it);
        a.next_slice = slice_ctr.get() + (size_t)it * 32 * nctr;
        a.nctr = (uint32_t)nctr;
        a.n_nd = P.n_nd;
        a.nslices = P.nslices;
        a.slice_begin = sl_begin;
        a.slice_end = sl_end;
        a.damping = damping;
        a.n_s = (uint64_t)(P.n_nd + P.n_exc);
        a.hot = (uint32_t)hot_rows;
        if (sharded)  // every element is then written by exactly one rank
            PRG_CUDA(cudaMemsetAsync(y_of(it & 1), 0, xcount * sizeof(double), s));
        if (P.nslices && sl_end > sl_begin) {
            ProfScope ps("k3_spmv", s);
            // 768 threads x 2 CTAs (48 warps/SM, 40 registers) with a 6-deep pipeline:
            // 0.767 ms vs 0.796 ms for 1024 x 2 at 32 registers, U=4 (same box,
            // tools/exp_spmv4.py); 896x2 U4 0.792, 640x2 U6 0.775, 512x3 U6 0.793,
            // 768x2 U8 0.780, 832x2 U6 0.847.
            if (variant == 1) spmv_sell_kernel<4><<<num_sms() * 2, kSpmvThreads, 0, s>>>(a);
            else if (variant == 2) spmv_sell_kernel<6, 768, 2, 2><<<num_sms() * 2, 768, 0, s>>>(a);
            else if (variant == 3) spmv_sell_kernel<6, 768, 2, 3><<<num_sms() * 2, 768, 0, s>>>(a);
            else if (variant == 4) spmv_sell_kernel<6, 768, 2, 4><<<num_sms() * 2, 768, 0, s>>>(a);
            else if (variant == 5) spmv_sell_kernel<6, 768, 2, 5><<<num_sms() * 2, 768, 0, s>>>(a);
            else spmv_sell_kernel<6, 768, 2><<<num_sms() * 2, 768, 0, s>>>(a);
            PRG_LAUNCH_CHECK();
        }
        if (sharded) {
            ProfScope px("k3_exchange", s);
            if (shard->allreduce(shard->user, y_of(it & 1), (int64_t)xcount, s) != 0)
                throw CudaError{"K3: the all-reduce callback failed"};
        }
        SplitArgs sp{P.n_split.get(), P.split_p0.get(), P.split_pbase.get(), partial_of(it & 1), out_of(it), damping};
        sell_sum_part<<<kSumBlocks, 1024, 0, s>>>(slice_sum_of(it & 1), P.nslices, y, sp, sum_part.get());
        PRG_LAUNCH_CHECK();
    }
    // the last step's Σ (the earlier ones were finished by the gather launches)
    sell_sum_final<<<1, 32, 0, s>>>(sum_part.get(), kSumBlocks, (double)P.n_empty, bgf, out_of(iters - 1));
    PRG_LAUNCH_CHECK();
    if (iters > 1) PRG_CUDA(cudaMemcpyAsync(S.out.get(), out_of(iters - 1), 4 * 8, cudaMemcpyDeviceToDevice, s));
    unpermute_kernel<<<g, 1024, 0, s>>>(ys[(iters - 1) & 1], P.spos_col.get(), S.out.get(), n, r_out);
    PRG_LAUNCH_CHECK();
}

__global__ void l1_diff_partial(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                double* __restrict__ part) {
    __shared__ double ws[32];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    double s = 0.0;
    for (int q = 0; q < 8; ++q) {
        const int64_t i = base + q * 1024 + threadIdx.x;
        if (i < n) s = __dadd_rn(s, fabs(a[i] - b[i]));
    }
    s = dev::warp_sum_f64(s);
    if (dev::lane_id() == 0) ws[dev::warp_id()] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = dev::warp_sum_f64(ws[threadIdx.x]);
        if (threadIdx.x == 0) part[blockIdx.x] = v;
    }
}

}  // namespace

// run_to_convergence (kernel3_pagerank.cpp:86-115): iterate, renormalise to
// 1-norm 1, stop when successive iterates differ by < tol in 1-norm.
int k3_converge_device(const prg_matrix* A, double damping, double tol, int max_iters, const double* d_start,
                       double* d_out, bool* converged, cudaStream_t s) {
    const int64_t n = A->n;
    const double bgf = (1.0 - damping) / (double)n;
    K3Plan tmp;
    const K3Plan& P = plan_for(A, 0, tmp, s);
    Sums S;
    DevBuf<double> cur((size_t)n, s), nxt((size_t)n, s);
    const unsigned g = (unsigned)num_sms() * 8;
    PRG_CUDA(cudaMemcpyAsync(cur.get(), d_start, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    device_sum(cur.get(), n, bgf, 0, S, s);
    if (!(read_scalar(S.out.get(), s) > 0.0)) throw CudaError{"start vector has no rank mass"};
    scale_kernel<<<g, 1024, 0, s>>>(cur.get(), n, S.out.get());
    PRG_LAUNCH_CHECK();
    device_sum(cur.get(), n, bgf, 0, S, s);
    const int64_t nb = (n + 8191) / 8192;
    DevBuf<double> part((size_t)nb, s), dsum(4, s);
    *converged = false;
    int it = 0;
    for (it = 1; it <= max_iters; ++it) {
        iterate(P, cur.get(), nxt.get(), 1, damping, bgf, S, s);
        if (!(read_scalar(S.out.get(), s) > 0.0)) throw CudaError{"iterate lost all rank mass"};
        scale_kernel<<<g, 1024, 0, s>>>(nxt.get(), n, S.out.get());
        PRG_LAUNCH_CHECK();
        device_sum(nxt.get(), n, bgf, 0, S, s);
        l1_diff_partial<<<(unsigned)nb, 1024, 0, s>>>(nxt.get(), cur.get(), n, part.get());
        final_sum_kernel<<<1, 1024, 0, s>>>(part.get(), nb, 0.0, dsum.get());
        PRG_LAUNCH_CHECK();
        std::swap(cur, nxt);
        if (read_scalar(dsum.get(), s) < tol) {
            *converged = true;
            break;
        }
    }
    PRG_CUDA(cudaMemcpyAsync(d_out, cur.get(), (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    return std::min(it, max_iters);
}

void k3_build_csc_device(prg_matrix* A, cudaStream_t s) {
    ProfScope prof("k2_csc", s);
    K3Plan* P = new K3Plan;
    try {
        build_plan(A, 0, *P, s);
    } catch (...) {
        delete P;
        throw;
    }
    PRG_CUDA(cudaStreamSynchronize(s));
    P->rehome();
    if (A->plan) {
        PRG_CUDA(cudaDeviceSynchronize());
        delete A->plan;
    }
    A->plan = P;
}

double k3_init_rank_device(int64_t n, uint64_t seed, double* d_r, int mode, cudaStream_t s) {
    Sums S;
    init_rank_impl(n, seed, d_r, mode, 0.0, S, s);
    return read_scalar(S.out.get(), s);
}

double k3_pagerank_device(const prg_matrix* A, const K3Options& opt, double* d_ranks, cudaStream_t s) {
    ProfScope prof("k3_pagerank", s);
    const int64_t n = A->n;
    const double bgf = (1.0 - opt.damping) / (double)n;  // kernel3_pagerank.cpp:46
    K3Plan tmp;
    const K3Plan& P = plan_for(A, opt.mode, tmp, s);
    Sums S;
    if (opt.mode != 0 || P.nslices == 0) {
        DevBuf<double> r0((size_t)n, s);
        // mode 2 takes every Σ compensated, init_rank's too (oracle_run_kernel3 mode 1)
        init_rank_impl(n, opt.seed, r0.get(), opt.mode, bgf, S, s);
        iterate(P, r0.get(), d_ranks, opt.iterations, opt.damping, bgf, S, s, 0, nullptr, opt.mode == 2 ? 2 : 1);
        return read_scalar(S.out.get(), s);
    }
    // Timed mode: init_rank's vector is never stored — its two sums are taken
    // over values regenerated from the counter-based RNG, and the first gather
    // regenerates r0[u] for the rows it needs (bit-identical to init_rank_impl).
    const uint64_t s0 = dev::mix_seed(opt.seed, kRankInitStream);
    const int64_t nb = (n + 8191) / 8192;
    DevBuf<double> part((size_t)nb, s), xsum(4, s);
    S.out = DevBuf<double>(4, s);
    PRG_CUDA(cudaMemsetAsync(S.out.get(), 0, 32, s));
    rng_partial_kernel<<<(unsigned)nb, 1024, 0, s>>>(n, s0, nullptr, part.get());
    final_sum_kernel<<<1, 1024, 0, s>>>(part.get(), nb, 0.0, xsum.get());
    rng_partial_kernel<<<(unsigned)nb, 1024, 0, s>>>(n, s0, xsum.get(), part.get());
    final_sum_kernel<<<1, 1024, 0, s>>>(part.get(), nb, bgf, S.out.get());
    PRG_LAUNCH_CHECK();
    iterate(P, nullptr, d_ranks, opt.iterations, opt.damping, bgf, S, s, s0, xsum.get());
    return read_scalar(S.out.get(), s);
}

double k3_pagerank_sharded_device(const prg_matrix* A, const K3Options& opt, int rank, int world,
                                  prg_allreduce_f64 allreduce, void* user, double* d_ranks, cudaStream_t s) {
    ProfScope prof("k3_pagerank", s);
    const int64_t n = A->n;
    const double bgf = (1.0 - opt.damping) / (double)n;
    K3Plan tmp;
    const K3Plan& P = plan_for(A, 0, tmp, s);
    Sums S;
    const Shard sh{rank, world, allreduce, user};
    if (P.nslices == 0) {  // nothing to shard: every rank computes the (trivial) iteration itself
        DevBuf<double> r0((size_t)n, s);
        init_rank_impl(n, opt.seed, r0.get(), 0, bgf, S, s);
        iterate(P, r0.get(), d_ranks, opt.iterations, opt.damping, bgf, S, s);
        return read_scalar(S.out.get(), s);
    }
    const uint64_t s0 = dev::mix_seed(opt.seed, kRankInitStream);
    const int64_t nb = (n + 8191) / 8192;
    DevBuf<double> part((size_t)nb, s), xsum(4, s);
    S.out = DevBuf<double>(4, s);
    PRG_CUDA(cudaMemsetAsync(S.out.get(), 0, 32, s));
    rng_partial_kernel<<<(unsigned)nb, 1024, 0, s>>>(n, s0, nullptr, part.get());
    final_sum_kernel<<<1, 1024, 0, s>>>(part.get(), nb, 0.0, xsum.get());
    rng_partial_kernel<<<(unsigned)nb, 1024, 0, s>>>(n, s0, xsum.get(), part.get());
    final_sum_kernel<<<1, 1024, 0, s>>>(part.get(), nb, bgf, S.out.get());
    PRG_LAUNCH_CHECK();
    iterate(P, nullptr, d_ranks, opt.iterations, opt.damping, bgf, S, s, s0, xsum.get(), 1, &sh);
    return read_scalar(S.out.get(), s);
}

void k3_shard_bounds_host(const uint32_t* slice_ptr, uint32_t nslices, int world, uint32_t* bounds) {
    shard_bounds_host(slice_ptr, nslices, world, bounds);
}

void k3_shard_bounds(const prg_matrix* A, int world, uint32_t* bounds, cudaStream_t s) {
    K3Plan tmp;
    const K3Plan& P = plan_for(A, 0, tmp, s);
    std::vector<uint32_t> sp((size_t)P.nslices + 1, 0);
    if (P.nslices) PRG_CUDA(cudaMemcpyAsync(sp.data(), P.slice_ptr.get(), sp.size() * 4, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    shard_bounds_host(sp.data(), P.nslices, world, bounds);
}

double k3_step_device(const prg_matrix* A, const double* d_r, double damping, double* d_out, int mode,
                      cudaStream_t s) {
    const int64_t n = A->n;
    const double bgf = (1.0 - damping) / (double)n;
    K3Plan tmp;
    const K3Plan& P = plan_for(A, mode, tmp, s);
    Sums S;
    device_sum(d_r, n, bgf, mode, S, s);
    iterate(P, d_r, d_out, 1, damping, bgf, S, s, 0, nullptr, mode == 2 ? 2 : 1);
    return read_scalar(S.out.get(), s);
}

}  // namespace prg

PRG_CHECK_QUERY(k3)
