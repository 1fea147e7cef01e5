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
//     hot-first: its first kHot entries are staged in shared memory, the rest
//     (~59 MB at S=24) stays L2-resident. Random gathers are the bound:
//     ~1 line/clk/SM from L2 vs ~3.6/clk/SM from SMEM (tools/microbench).
//   * b[u] is the row's base value (its minimum stored value; for K2 output
//     that is 1/d_out exactly). Entries equal to b[u] contribute r[u]*b[u],
//     the reference's own product r[u]*values[k], bit for bit. Other entries
//     (duplicate edges, ~2%) are exceptions with an explicit f64 value.
//   * CSC index stream: u32 per entry, bit 31 = exception, bits 0-30 = new id
//     of the source row. Columns keep their original ids, so r' needs no
//     un-permutation and exceptions read r' directly.
// Parity mode (mode 1) keeps original row ids, sums every column sequentially
// in ascending u with separate mul/add, and computes every sum(r) with one
// thread in index order — the reference's exact evaluation order.
#include <algorithm>
#include <vector>

#include "prg_internal.cuh"
#include "prg_sort.cuh"

namespace prg {

namespace {

constexpr uint64_t kRankInitStream = 0x72616e6b696e6974ULL;  // kernel3_pagerank.cpp:15
constexpr int kSpmvThreads = 1024;
constexpr int kHotBytes = 220 * 1024;
constexpr int kHot = kHotBytes / 8;
constexpr int kCscGroup = 32;  // exception ranks are counted per 32-entry group

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
    static constexpr size_t kSmem = 0;
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
        return ((uint64_t)cls << sb) | i;
    }
};

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

__global__ void count_nondangling(const uint32_t* __restrict__ ro, int64_t n, unsigned long long* out) {
    uint32_t c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += ro[i + 1] > ro[i];
    c = __reduce_add_sync(0xffffffffu, c);
    if (dev::lane_id() == 0 && c) atomicAdd(out, (unsigned long long)c);
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

// All threads: srow[li] = row of entry base+li, li < cnt. smem must hold cnt u32.
__device__ void expand_rows(const uint32_t* __restrict__ ro, const uint32_t* __restrict__ tile_row,
                            int64_t n, size_t base, int cnt, uint32_t* srow) {
    const uint32_t t = (uint32_t)(base / sort::kTile);
    const uint32_t r0 = tile_row[t];
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) srow[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) srow[0] = r0;
    // Rows starting inside the tile: scan forward from r0+1 while ro[r] < base+cnt.
    const uint64_t end = base + cnt;
    for (int64_t r = (int64_t)r0 + 1 + threadIdx.x;; r += blockDim.x) {
        const bool in = r < n && ro[r] < end;
        if (in && ro[r + 1] > ro[r]) srow[ro[r] - base] = (uint32_t)r;
        if (!__syncthreads_or(in)) break;
    }
    // inclusive max-scan over srow (blocked, 8192 entries / blockDim threads)
    __shared__ uint32_t wmax[32];
    const int per = (cnt + blockDim.x - 1) / blockDim.x;
    const int l0 = threadIdx.x * per;
    uint32_t m = 0;
    for (int k = 0; k < per && l0 + k < cnt; ++k) m = max(m, srow[l0 + k]);
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
        run = max(run, srow[l0 + k]);
        srow[l0 + k] = run;
    }
    __syncthreads();
}

// Row minimum of stored values -> bmin[u] (as ordered u64 bit patterns; values > 0).
__global__ void __launch_bounds__(sort::kTileThreads) row_min_kernel(
    const uint32_t* __restrict__ ro, const uint32_t* __restrict__ tile_row, const double* __restrict__ val,
    int64_t n, size_t nnz, unsigned long long* __restrict__ bmin) {
    __shared__ uint32_t srow[sort::kTile];
    const uint32_t ntiles = div_up(nnz, sort::kTile);
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const size_t base = (size_t)t * sort::kTile;
        const int cnt = (int)min((size_t)sort::kTile, nnz - base);
        expand_rows(ro, tile_row, n, base, cnt, srow);
        for (int j = 0; j < sort::kTileItems; ++j) {
            const int li = j * sort::kTileThreads + threadIdx.x;
            const bool ok = li < cnt;
            const uint32_t r = ok ? srow[li] : 0xffffffffu;
            uint64_t b = ok ? (uint64_t)__double_as_longlong(val[base + li]) : ~0ull;
            // segmented min over equal rows within the warp (rows are contiguous)
            const unsigned lane = dev::lane_id();
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint64_t ob = __shfl_down_sync(0xffffffffu, b, d);
                const uint32_t orow = __shfl_down_sync(0xffffffffu, r, d);
                if (lane + d < 32 && orow == r) b = min(b, ob);
            }
            const uint32_t prow = __shfl_up_sync(0xffffffffu, r, 1);
            if (ok && (lane == 0 || prow != r)) atomicMin(&bmin[r], (unsigned long long)b);
        }
        __syncthreads();
    }
}

__global__ void gather_base_kernel(const uint32_t* __restrict__ pinv, const unsigned long long* __restrict__ bmin,
                                   int64_t n_nd, double* __restrict__ bval) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_nd; j += (int64_t)gridDim.x * blockDim.x)
        bval[j] = __longlong_as_double((long long)bmin[pinv[j]]);
}

// ---------------------------------------------------------------------------
// Transpose: sort keys (col << (sb+1)) | (newid << 1) | exc
// ---------------------------------------------------------------------------
struct CsrEntrySrc {
    const uint32_t* ro;
    const uint32_t* tile_row;
    const uint32_t* cols;
    const double* val;
    const uint32_t* newid;
    const unsigned long long* bmin;
    int64_t n;
    int sb;
    // exception list (filled by the histogram pass only)
    unsigned long long* exc_key;
    double* exc_val;
    uint32_t* n_exc;
    static constexpr size_t kSmem = sort::kTile * sizeof(uint32_t);
    __device__ void prepare(size_t base, int cnt, void* smem) const {
        expand_rows(ro, tile_row, n, base, cnt, static_cast<uint32_t*>(smem));
    }
    __device__ __forceinline__ uint64_t key(size_t i, int li, const void* smem) const {
        const uint32_t r = static_cast<const uint32_t*>(smem)[li];
        const double v = val[i];
        const bool exc = (uint64_t)__double_as_longlong(v) != bmin[r];
        const uint64_t k = ((uint64_t)cols[i] << (sb + 1)) | ((uint64_t)newid[r] << 1) | (uint64_t)exc;
        if (exc_key) {
            const unsigned msk = __ballot_sync(__activemask(), exc);
            if (exc) {
                const unsigned leader = __ffs(msk) - 1;
                uint32_t b0 = 0;
                if (dev::lane_id() == leader) b0 = atomicAdd(n_exc, (uint32_t)__popc(msk));
                b0 = __shfl_sync(msk, b0, leader);
                const uint32_t idx = b0 + __popc(msk & ((1u << dev::lane_id()) - 1));
                exc_key[idx] = k;
                exc_val[idx] = v;
            }
        }
        return k;
    }
};

struct CscDst {
    uint32_t* csc_idx;
    uint32_t* colptr;   // initialised to ~0; column starts via atomicMin
    uint32_t* exc_cnt;  // per 32-entry group
    int sb;
    __device__ __forceinline__ void store(uint64_t pos, uint64_t key, bool has_prev, uint64_t prev) const {
        const uint32_t col = (uint32_t)(key >> (sb + 1));
        const uint32_t exc = (uint32_t)(key & 1);
        csc_idx[pos] = (uint32_t)((key >> 1) & ((1ull << sb) - 1)) | (exc << 31);
        if (!has_prev || (uint32_t)(prev >> (sb + 1)) != col) atomicMin(&colptr[col], (uint32_t)pos);
        if (exc) atomicAdd(&exc_cnt[pos / kCscGroup], 1u);
    }
};

// colptr[c] = min(colptr[c], colptr[c+1], ...) — fills empty columns.
__global__ void suffix_min_block(uint32_t* a, int64_t n1, uint32_t* part) {
    // each block: 1024 threads x 8 items, reverse order
    __shared__ uint32_t wm[32];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    uint32_t m = 0xffffffffu;
    for (int k = 0; k < 8; ++k) {
        const int64_t i = base + threadIdx.x * 8 + k;
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
__global__ void suffix_min_parts(uint32_t* part, int64_t nb) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        uint32_t run = 0xffffffffu;
        for (int64_t b = nb - 1; b >= 0; --b) {
            const uint32_t x = part[b];
            part[b] = run;  // exclusive suffix min (blocks after b)
            run = min(run, x);
        }
    }
}
__global__ void suffix_min_down(uint32_t* a, int64_t n1, const uint32_t* part) {
    __shared__ uint32_t wm[33];
    const int64_t base = (int64_t)blockIdx.x * 8192;
    uint32_t v[8];
    for (int k = 0; k < 8; ++k) {
        const int64_t i = base + threadIdx.x * 8 + k;
        v[k] = i < n1 ? a[i] : 0xffffffffu;
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
    uint32_t run = part[blockIdx.x];
    if (dev::warp_id() + 1 < 32) run = min(run, wm[dev::warp_id() + 1]);
    uint32_t after = __shfl_down_sync(0xffffffffu, inc, 1);
    if (dev::lane_id() < 31) run = min(run, after);
    for (int k = 7; k >= 0; --k) {
        run = min(run, v[k]);
        const int64_t i = base + threadIdx.x * 8 + k;
        if (i < n1) a[i] = run;
    }
}

// Exceptions: locate each in the CSC (binary search inside its column), then
// store its value at its rank among exception entries in CSC order.
__global__ void place_exceptions(const unsigned long long* __restrict__ exc_key, const double* __restrict__ exc_v,
                                 const uint32_t* __restrict__ n_exc, const uint32_t* __restrict__ colptr,
                                 const uint32_t* __restrict__ csc_idx, const uint32_t* __restrict__ exc_base,
                                 int sb, double* __restrict__ exc_val) {
    const uint32_t ne = *n_exc;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += gridDim.x * blockDim.x) {
        const uint64_t k = exc_key[i];
        const uint32_t col = (uint32_t)(k >> (sb + 1));
        const uint32_t nid = (uint32_t)((k >> 1) & ((1ull << sb) - 1));
        uint32_t lo = colptr[col], hi = colptr[col + 1];
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((csc_idx[mid] & 0x7fffffffu) < nid) lo = mid + 1; else hi = mid;
        }
        const uint32_t q = lo;
        const uint32_t g0 = q & ~(uint32_t)(kCscGroup - 1);
        uint32_t rank = exc_base[q / kCscGroup];
        for (uint32_t p = g0; p < q; ++p) rank += csc_idx[p] >> 31;
        exc_val[rank] = exc_v[i];
    }
}

// ---------------------------------------------------------------------------
// init_rank (kernel3_pagerank.cpp:29-39)
// ---------------------------------------------------------------------------
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
__global__ void scale_kernel(double* __restrict__ x, int64_t n, const double* __restrict__ sum) {
    const double d = sum[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __ddiv_rn(x[i], d);
}

// s[j] = r[pinv[j]] * b[j]   (the reference's product r[u] * values[k], k non-exception)
__global__ void permute_scale_kernel(const double* __restrict__ r, const uint32_t* __restrict__ pinv,
                                     const double* __restrict__ bval, int64_t n_nd, double* __restrict__ s) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_nd; j += (int64_t)gridDim.x * blockDim.x)
        s[j] = __dmul_rn(r[pinv[j]], bval[j]);
}

// ---------------------------------------------------------------------------
// Pull SpMV (timed mode): warp task = 32 consecutive columns, lane j owns column
// cb+j. Entries are walked in 32-aligned slices; each lane finds its entry's
// owner column by a 5-step shuffle search, products are reduced with a
// segmented warp scan and delivered to the owner lane. All reductions have a
// fixed shape, so results are bitwise reproducible.
// ---------------------------------------------------------------------------
struct SpmvArgs {
    const uint32_t* colptr;    // [n+1]
    const uint32_t* csc_idx;   // [nnz]
    const uint32_t* exc_base;  // [ngroups]
    const double* exc_val;
    const double* s;           // [n_nd] gather vector
    const double* r_prev;      // [n] previous iterate (original order) for exceptions
    const uint32_t* pinv;
    const double* bgp;         // device scalar: bg for this iteration (bgp[1])
    double* r_next;            // [n]
    double* task_sum;          // [ntasks]
    uint32_t* task_counter;
    int64_t n;
    int64_t n_nd;
    uint32_t ntasks;
    double damping;
};

__global__ void __launch_bounds__(kSpmvThreads, 1) spmv_pull_kernel(SpmvArgs a) {
    extern __shared__ __align__(16) double s_hot[];
    const int64_t nh = a.n_nd < kHot ? a.n_nd : kHot;
    for (int64_t i = threadIdx.x; i < nh; i += kSpmvThreads) s_hot[i] = a.s[i];
    __syncthreads();
    const unsigned lane = dev::lane_id();
    const double bg = a.bgp[1];
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint64_t pol_stream = dev::policy_evict_first(), pol_keep = dev::policy_evict_last();
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(a.task_counter, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= a.ntasks) break;
        const int64_t c = (int64_t)t * 32 + lane;
        const bool cvalid = c < a.n;
        const uint32_t cb = a.colptr[cvalid ? c : a.n];
        const uint32_t ce = a.colptr[cvalid ? c + 1 : a.n];
        const uint32_t B = __shfl_sync(0xffffffffu, cb, 0);
        const uint32_t E = __shfl_sync(0xffffffffu, ce, 31);
        double acc = 0.0;
        for (uint32_t base = B & ~31u; base < E; base += 32) {
            const uint32_t e = base + lane;
            const bool valid = e >= B && e < E;
            const bool inr = e < E;  // group members for exception ranks (e >= base)
            uint32_t w = inr ? dev::ld_stream_u32(a.csc_idx + e, pol_stream) : 0u;
            // owner column: largest j with colptr[cb_j] <= e
            int j = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t bc = __shfl_sync(0xffffffffu, cb, j + step);
                if (bc <= e) j += step;
            }
            const bool exc = (w >> 31) != 0;
            const uint32_t excm = __ballot_sync(0xffffffffu, inr && exc);
            double x = 0.0;
            if (valid) {
                const uint32_t u = w & 0x7fffffffu;
                if (exc) {
                    const uint32_t rank = a.exc_base[base / kCscGroup] + __popc(excm & lt_mask);
                    x = __dmul_rn(a.r_prev[a.pinv[u]], a.exc_val[rank]);
                } else {
                    x = u < (uint32_t)nh ? s_hot[u] : dev::ld_keep_f64(a.s + u, pol_keep);
                }
            }
            // segmented inclusive scan by owner
            const int jj = valid ? j : (e < B ? -1 : 32);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double o = __shfl_up_sync(0xffffffffu, x, d);
                const int oj = __shfl_up_sync(0xffffffffu, jj, d);
                if ((int)lane >= d && oj == jj) x = __dadd_rn(x, o);
            }
            // deliver: owner lane gets the partial from its last entry in this slice
            const uint32_t lo = cb > base ? cb : base;
            const uint32_t hi = ce < base + 32 ? ce : base + 32;
            const bool has = lo < hi;
            const int src = has ? (int)(hi - 1 - base) : (int)lane;
            const double part = __shfl_sync(0xffffffffu, x, src);
            if (has) acc = __dadd_rn(acc, part);
        }
        double rn = 0.0;
        if (cvalid) {
            rn = __dadd_rn(__dmul_rn(a.damping, acc), bg);
            a.r_next[c] = rn;
        }
        rn = dev::warp_sum_f64(rn);
        if (lane == 0) a.task_sum[t] = rn;
    }
}

// Parity mode: one thread per column, ascending source order, separate mul/add.
__global__ void spmv_seq_kernel(SpmvArgs a) {
    const uint32_t lt_dummy = 0;
    (void)lt_dummy;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < a.n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = a.colptr[c], e = a.colptr[c + 1];
        double acc = 0.0;
        for (uint32_t p = b; p < e; ++p) {
            const uint32_t w = a.csc_idx[p];
            const uint32_t u = w & 0x7fffffffu;
            double x;
            if (w >> 31) {
                uint32_t rank = a.exc_base[p / kCscGroup];
                for (uint32_t q = p & ~(uint32_t)(kCscGroup - 1); q < p; ++q) rank += a.csc_idx[q] >> 31;
                x = __dmul_rn(a.r_prev[a.pinv[u]], a.exc_val[rank]);
            } else {
                x = a.s[u];
            }
            acc = __dadd_rn(acc, x);
        }
        a.r_next[c] = __dadd_rn(__dmul_rn(a.damping, acc), a.bgp[1]);
    }
}

struct K3Plan {
    int64_t n = 0, n_nd = 0;
    uint64_t nnz = 0;
    int sb = 1;
    int mode = 0;
    DevBuf<uint32_t> pinv, newid, colptr, csc_idx, exc_base;
    DevBuf<double> bval, exc_val;
    uint32_t n_exc = 0;
};

void build_plan(const prg_matrix* A, int mode, K3Plan& P, cudaStream_t s) {
    ProfScope prof("k3_prep", s);
    const int64_t n = A->n;
    const uint64_t nnz = A->nnz;
    P.n = n;
    P.nnz = nnz;
    P.mode = mode;
    P.sb = bits_for(n);
    if (2 * P.sb + 1 > 64 || P.sb > 31) throw CudaError{"K3: vertex count too large for u32 indices"};
    const unsigned g = (unsigned)num_sms() * 8;
    P.pinv = DevBuf<uint32_t>((size_t)n, s);
    P.newid = DevBuf<uint32_t>((size_t)n, s);
    // 1. row renumbering
    if (mode == 0) {
        DevBuf<unsigned long long> cnt(1, s);
        PRG_CUDA(cudaMemsetAsync(cnt.get(), 0, 8, s));
        count_nondangling<<<g, 1024, 0, s>>>(A->row_offsets, n, cnt.get());
        PRG_LAUNCH_CHECK();
        sort::SortWorkspace ws;
        sort::msd_sort(RowClassSrc{A->row_offsets, P.sb}, (size_t)n, P.sb + 8,
                       PermDst{P.pinv.get(), P.newid.get(), P.sb}, ws, s);
        unsigned long long h = 0;
        PRG_CUDA(cudaMemcpyAsync(&h, cnt.get(), 8, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        P.n_nd = (int64_t)h;
    } else {
        iota_kernel<<<g, 1024, 0, s>>>(P.pinv.get(), P.newid.get(), n);
        PRG_LAUNCH_CHECK();
        P.n_nd = n;
    }
    // 2. row base values (min stored value per row)
    DevBuf<unsigned long long> bmin((size_t)n, s);
    PRG_CUDA(cudaMemsetAsync(bmin.get(), 0xff, (size_t)n * 8, s));
    const uint32_t ntiles = nnz ? div_up(nnz, sort::kTile) : 0;
    DevBuf<uint32_t> tile_row(ntiles + 1, s);
    if (nnz) {
        tile_rows_kernel<<<g, 1024, 0, s>>>(A->row_offsets, n, tile_row.get());
        PRG_LAUNCH_CHECK();
        row_min_kernel<<<std::min<unsigned>(ntiles, (unsigned)num_sms() * 2), sort::kTileThreads, 0, s>>>(
            A->row_offsets, tile_row.get(), A->values, n, nnz, bmin.get());
        PRG_LAUNCH_CHECK();
    }
    P.bval = DevBuf<double>((size_t)std::max<int64_t>(P.n_nd, 1), s);
    gather_base_kernel<<<g, 1024, 0, s>>>(P.pinv.get(), bmin.get(), P.n_nd, P.bval.get());
    PRG_LAUNCH_CHECK();
    // 3. transpose
    P.colptr = DevBuf<uint32_t>((size_t)n + 1, s);
    PRG_CUDA(cudaMemsetAsync(P.colptr.get(), 0xff, (size_t)(n + 1) * 4, s));
    P.csc_idx = DevBuf<uint32_t>(nnz ? nnz : 1, s);
    const uint64_t ngroups = nnz / kCscGroup + 1;
    DevBuf<uint32_t> exc_cnt(ngroups, s);
    PRG_CUDA(cudaMemsetAsync(exc_cnt.get(), 0, ngroups * 4, s));
    DevBuf<unsigned long long> exc_key(nnz ? nnz : 1, s);
    DevBuf<double> exc_v(nnz ? nnz : 1, s);
    DevBuf<uint32_t> n_exc(1, s);
    PRG_CUDA(cudaMemsetAsync(n_exc.get(), 0, 4, s));
    if (nnz) {
        CsrEntrySrc src{A->row_offsets, tile_row.get(), A->cols, A->values, P.newid.get(), bmin.get(), n, P.sb,
                        exc_key.get(), exc_v.get(), n_exc.get()};
        // The histogram pass captures the exception list; the scatter pass must not.
        CsrEntrySrc scat = src;
        scat.exc_key = nullptr;
        sort::SortWorkspace ws;
        sort::msd_sort_split(src, scat, (size_t)nnz, 2 * P.sb + 1,
                             CscDst{P.csc_idx.get(), P.colptr.get(), exc_cnt.get(), P.sb}, ws, s);
    }
    // colptr[n] = nnz, then fill empty columns with the next column start.
    {
        const uint32_t nz = (uint32_t)nnz;
        PRG_CUDA(cudaMemcpyAsync(P.colptr.get() + n, &nz, 4, cudaMemcpyHostToDevice, s));
        const int64_t n1 = n + 1;
        const int64_t nb = (n1 + 8191) / 8192;
        DevBuf<uint32_t> part((size_t)nb, s);
        suffix_min_block<<<(unsigned)nb, 1024, 0, s>>>(P.colptr.get(), n1, part.get());
        suffix_min_parts<<<1, 1, 0, s>>>(part.get(), nb);
        suffix_min_down<<<(unsigned)nb, 1024, 0, s>>>(P.colptr.get(), n1, part.get());
        PRG_LAUNCH_CHECK();
    }
    // exceptions
    P.exc_base = DevBuf<uint32_t>(ngroups, s);
    DevBuf<uint32_t> exc_total(1, s);
    exclusive_scan_u32(exc_cnt.get(), P.exc_base.get(), ngroups, exc_total.get(), s);
    PRG_CUDA(cudaMemcpyAsync(&P.n_exc, exc_total.get(), 4, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    P.exc_val = DevBuf<double>(P.n_exc ? P.n_exc : 1, s);
    if (P.n_exc) {
        place_exceptions<<<g, 256, 0, s>>>(exc_key.get(), exc_v.get(), n_exc.get(), P.colptr.get(),
                                           P.csc_idx.get(), P.exc_base.get(), P.sb, P.exc_val.get());
        PRG_LAUNCH_CHECK();
    }
}


// ---------------------------------------------------------------------------
// Drivers
// ---------------------------------------------------------------------------
struct Sums {
    DevBuf<double> part, out;  // out[0] = sum, out[1] = bg for the next step
};

// sum(x) into out[0] and ((1-c)/n)*sum into out[1], deterministic.
void device_sum(const double* x, int64_t n, double bgf, int mode, Sums& S, cudaStream_t s) {
    if (!S.out.get()) S.out = DevBuf<double>(2, s);
    if (mode == 1) {
        seq_sum_kernel<<<1, 1, 0, s>>>(x, n, bgf, S.out.get());
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

size_t spmv_smem() { return (size_t)kHot * sizeof(double); }

// One step: r_next = c * A^T r_prev + bg; S.out holds {sum(r_prev), bg} on entry
// and {sum(r_next), bg'} on exit. s_buf is scratch of n_nd doubles.
void step_impl(const K3Plan& P, const double* r_prev, double* r_next, double damping, double bgf,
               double* s_buf, Sums& S, DevBuf<double>& task_sum, DevBuf<uint32_t>& counter, cudaStream_t s) {
    const unsigned g = (unsigned)num_sms() * 8;
    if (P.n_nd) {
        ProfScope pp("k3_permute", s);
        permute_scale_kernel<<<g, 1024, 0, s>>>(r_prev, P.pinv.get(), P.bval.get(), P.n_nd, s_buf);
        PRG_LAUNCH_CHECK();
    }
    const uint32_t ntasks = (uint32_t)((P.n + 31) / 32);
    if (task_sum.n < ntasks) task_sum = DevBuf<double>(ntasks, s);
    SpmvArgs a;
    a.colptr = P.colptr.get();
    a.csc_idx = P.csc_idx.get();
    a.exc_base = P.exc_base.get();
    a.exc_val = P.exc_val.get();
    a.s = s_buf;
    a.r_prev = r_prev;
    a.pinv = P.pinv.get();
    a.bgp = S.out.get();
    a.r_next = r_next;
    a.task_sum = task_sum.get();
    a.task_counter = counter.get();
    a.n = P.n;
    a.n_nd = P.n_nd;
    a.ntasks = ntasks;
    a.damping = damping;
    if (P.mode == 1) {
        spmv_seq_kernel<<<g, 256, 0, s>>>(a);
        PRG_LAUNCH_CHECK();
        device_sum(r_next, P.n, bgf, 1, S, s);
    } else {
        static bool attr = false;
        if (!attr) {
            PRG_CUDA(cudaFuncSetAttribute(spmv_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)spmv_smem()));
            attr = true;
        }
        PRG_CUDA(cudaMemsetAsync(counter.get(), 0, 4, s));
        {
            ProfScope ps("k3_spmv", s);
            spmv_pull_kernel<<<num_sms(), kSpmvThreads, spmv_smem(), s>>>(a);
            PRG_LAUNCH_CHECK();
        }
        final_sum_kernel<<<1, 1024, 0, s>>>(task_sum.get(), ntasks, bgf, S.out.get());
        PRG_LAUNCH_CHECK();
    }
}

}  // namespace

double k3_init_rank_device(int64_t n, uint64_t seed, double* d_r, int mode, cudaStream_t s) {
    Sums S;
    init_rank_impl(n, seed, d_r, mode, 0.0, S, s);
    return read_scalar(S.out.get(), s);
}

double k3_pagerank_device(const prg_matrix* A, const K3Options& opt, double* d_ranks, cudaStream_t s) {
    ProfScope prof("k3_pagerank", s);
    const int64_t n = A->n;
    const double bgf = (1.0 - opt.damping) / (double)n;  // kernel3_pagerank.cpp:46
    K3Plan P;
    build_plan(A, opt.mode, P, s);
    Sums S;
    DevBuf<double> r_tmp((size_t)n, s), s_buf((size_t)std::max<int64_t>(P.n_nd, 1), s), task_sum;
    DevBuf<uint32_t> counter(1, s);
    // The final iterate must land in d_ranks: alternate so that it does.
    double* bufs[2] = {d_ranks, r_tmp.get()};
    int cur = (opt.iterations % 2 == 0) ? 0 : 1;
    init_rank_impl(n, opt.seed, bufs[cur], opt.mode, bgf, S, s);
    for (int it = 0; it < opt.iterations; ++it) {
        step_impl(P, bufs[cur], bufs[cur ^ 1], opt.damping, bgf, s_buf.get(), S, task_sum, counter, s);
        cur ^= 1;
    }
    return read_scalar(S.out.get(), s);
}

double k3_step_device(const prg_matrix* A, const double* d_r, double damping, double* d_out, int mode,
                      cudaStream_t s) {
    const int64_t n = A->n;
    const double bgf = (1.0 - damping) / (double)n;
    K3Plan P;
    build_plan(A, mode, P, s);
    Sums S;
    device_sum(d_r, n, bgf, mode, S, s);
    DevBuf<double> s_buf((size_t)std::max<int64_t>(P.n_nd, 1), s), task_sum;
    DevBuf<uint32_t> counter(1, s);
    step_impl(P, d_r, d_out, damping, bgf, s_buf.get(), S, task_sum, counter, s);
    return read_scalar(S.out.get(), s);
}

}  // namespace prg
