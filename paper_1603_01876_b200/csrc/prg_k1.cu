// prg_k1.cu — K1: sort the edge list by start vertex on the device.
//
// Replaces the core of prpipe::sort_edges (include/prpipe/kernel1_sort.hpp:24-25;
// src/kernel1_sort.cpp:63-68, std::sort by u). Edges are packed into one u64
// key ((u-1) << S) | (v-1) and sorted by the MSD radix sort of prg_sort.cuh, so
// the output is ordered by (u, v): a valid start-vertex order whose tie order is
// canonical (tests/helpers.hpp:29-34) — the reference's own std::sort leaves it
// unspecified (kernel1_sort.hpp:23).
#include "prg_internal.cuh"
#include "prg_sort.cuh"

namespace prg {

namespace {

struct PairKeySrc {
    const longlong2* uv;
    uint64_t n_labels;  // N = 2^S
    int scale;
    uint32_t* err;
    static constexpr size_t kSmem = 0;
    static constexpr int kHistBatch = 4;
    static constexpr bool kRegPrefetch = false;  // 16-byte pairs: 16 raw pairs per thread do not fit in registers
    static constexpr bool kL2Prefetch = true;
    __device__ __forceinline__ void prefetch_l2(size_t i) const {
        if ((threadIdx.x & 1u) == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(uv + i));  // one per 32-byte sector
    }
    __device__ __forceinline__ void prepare(size_t, int, void*) const {}
    __device__ __forceinline__ uint64_t key(size_t i, int, const void*) const {
        const longlong2 p = uv[i];
        const uint64_t u = (uint64_t)(p.x - 1), v = (uint64_t)(p.y - 1);
        if (u >= n_labels || v >= n_labels) atomicOr(err, (uint32_t)kErrLabelRange);
        return (u << scale) | (v & (n_labels - 1));
    }
};

struct PairSink {
    longlong2* out;
    int scale;
    uint64_t mask;
    __device__ __forceinline__ void store(uint64_t pos, uint64_t key, bool, uint64_t) const {
        out[pos] = make_longlong2((long long)(key >> scale) + 1, (long long)(key & mask) + 1);
    }
};

}  // namespace

void k1_sort_device(const int64_t* d_uv_in, int64_t m, int scale, int64_t* d_uv_out,
                    uint32_t* d_err, cudaStream_t s) {
    if (m == 0) return;
    ProfScope prof("k1_sort", s);
    const uint64_t n = 1ull << scale;
    PairKeySrc src{reinterpret_cast<const longlong2*>(d_uv_in), n, scale, d_err};
    PairSink dst{reinterpret_cast<longlong2*>(d_uv_out), scale, n - 1};
    sort::SortWorkspace ws;
    sort::msd_sort(src, (size_t)m, 2 * scale, dst, ws, s, "k1");
}

}  // namespace prg

// Debug: local-stage statistics of the K1 sort (meaningful only when built
// with -DPRG_LOCAL_STATS=1). Not part of include/prg.h.
extern "C" void prg_debug_k1_local_stats(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, prg::sort::g_local_stats, sizeof(unsigned long long) * 16);
    static const unsigned long long zero[16] = {};
    cudaMemcpyToSymbol(prg::sort::g_local_stats, zero, sizeof(zero));
}

PRG_CHECK_QUERY(k1)
