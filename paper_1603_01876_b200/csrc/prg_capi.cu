// prg_capi.cu — the extern "C" boundary (include/prg.h).
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <type_traits>
#include <string>
#include <vector>

#include "../../include/prg.h"
#include "prg_internal.cuh"

using prg::CudaError;
using prg::DevBuf;

// Matrix arrays come from the stream-ordered pool; a handle may have been used
// on any stream, so release only after the device is idle.
prg_matrix::~prg_matrix() {
    if (row_offsets || cols || values || d_in || plan) cudaDeviceSynchronize();
    prg::k3_plan_destroy(plan);
    prg::ws_free(row_offsets, nullptr);
    prg::ws_free(cols, nullptr);
    prg::ws_free(values, nullptr);
    prg::ws_free(d_in, nullptr);
}

namespace {

struct ApiError {
    prg_status code;
    std::string msg;
};

template <class F>
prg_status guarded(const char* what, F&& f) {
    try {
        f();
        return PRG_OK;
    } catch (const ApiError& e) {
        prg::set_error(std::string(what) + ": " + e.msg);
        return e.code;
    } catch (const CudaError& e) {
        prg::set_error(std::string(what) + ": " + e.msg);
        return PRG_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        prg::set_error(std::string(what) + ": host allocation failed");
        return PRG_ERR_INTERNAL;
    } catch (const std::exception& e) {
        prg::set_error(std::string(what) + ": " + e.what());
        return PRG_ERR_INTERNAL;
    }
}

void require(bool ok, prg_status code, const std::string& msg) {
    if (!ok) throw ApiError{code, msg};
}

void check_device_errors(uint32_t err, const char* stage) {
    if (err & prg::kErrLabelRange)
        throw ApiError{PRG_ERR_LABEL_RANGE, std::string(stage) + ": vertex label outside [1, N]"};
    if (err & prg::kErrUnsorted)
        throw ApiError{PRG_ERR_UNSORTED, std::string(stage) + ": input not sorted by start vertex"};
    if (err & prg::kErrOverflow) throw ApiError{PRG_ERR_INTERNAL, std::string(stage) + ": capacity overflow"};
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

template <class T>
T* dmalloc(size_t count) {
    return static_cast<T*>(prg::ws_alloc((count ? count : 1) * sizeof(T), nullptr));
}

__global__ void widen_u32(const uint32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}
__global__ void narrow_i64(const int64_t* __restrict__ in, int64_t n, int64_t limit, uint32_t* __restrict__ out,
                           uint32_t* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = in[i];
        if (x < 0 || x > limit) atomicOr(err, (uint32_t)prg::kErrLabelRange);
        out[i] = (uint32_t)x;
    }
}

// Row offsets: narrowed like narrow_i64 and required non-decreasing (a
// decreasing pair would make ro[u+1]-ro[u] wrap as u32 in every row-length
// computation downstream): kErrBadOffsets.
constexpr uint32_t kErrBadOffsets = 0x100u;
__global__ void narrow_offsets(const int64_t* __restrict__ in, int64_t n, int64_t limit, uint32_t* __restrict__ out,
                               uint32_t* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = in[i];
        if (x < 0 || x > limit) atomicOr(err, (uint32_t)prg::kErrLabelRange);
        if (i + 1 < n && in[i + 1] < x) atomicOr(err, kErrBadOffsets);
        out[i] = (uint32_t)x;
    }
}

void check_upload_flags(uint32_t h) {
    require(!(h & kErrBadOffsets), PRG_ERR_INVALID_ARGUMENT, "row_offsets must be non-decreasing");
    require(h == 0, PRG_ERR_LABEL_RANGE, "row offsets or column indices out of range");
}

// ---------------------------------------------------------------------------
// Host-buffer K3 (prg_k3_pagerank_host): the CSR crosses PCIe (~55 GB/s) —
// the bound of the whole call. The f64 values are run-length coded on the
// host's cores while the column indices are in flight: one bit per entry
// ("differs, bitwise, from the previous entry") plus the differing values.
// A stochastic matrix repeats each row's 1/d_out, so at S=24 the 2.1 GB of
// values cross as 0.14 GB; the device expands them back bit for bit.
// ---------------------------------------------------------------------------
int64_t g_last_h2d_bytes = 0;

struct PinnedStage {
    std::mutex mu;
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            PRG_CUDA(cudaMallocHost(&p, bytes));
            cap = bytes;
        }
        return p;
    }
};
PinnedStage& pinned_stage(int which) {
    static PinnedStage st[2];
    return st[which];
}

template <class F>
void parallel_for(int T, F&& f) {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(f, t);
    f(0);
    for (auto& th : pool) th.join();
}

// Bit i of the result: value k0+i differs (bitwise) from value k0+i-1 (k0 >= 1,
// 32 entries). AVX2 when the host has it (4 compares per instruction).
__attribute__((target("avx2"))) uint32_t neq32_avx2(const uint64_t* vb, int64_t k0) {
    uint32_t eq = 0;
#pragma GCC unroll 8
    for (int i = 0; i < 32; i += 4) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(vb + k0 + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(vb + k0 + i - 1));
        eq |= (uint32_t)_mm256_movemask_pd(_mm256_castsi256_pd(_mm256_cmpeq_epi64(a, b))) << i;
    }
    return ~eq;
}
uint32_t neq32_scalar(const uint64_t* vb, int64_t k0) {
    uint32_t neq = 0;
    for (int i = 0; i < 32; ++i) neq |= (uint32_t)(vb[k0 + i] != vb[k0 + i - 1]) << i;
    return neq;
}
const bool g_have_avx2 = __builtin_cpu_supports("avx2");

// Words [w0, w1): bits[w] (bit i: value 32w+i starts a new run; value 0
// always does) and the run values, in order.
void rle_values(const double* vals, int64_t nnz, int64_t w0, int64_t w1, uint32_t* bits, std::vector<double>& out) {
    const uint64_t* vb = reinterpret_cast<const uint64_t*>(vals);
    for (int64_t w = w0; w < w1; ++w) {
        const int64_t k0 = w * 32;
        const int lim = (int)std::min<int64_t>(32, nnz - k0);
        uint32_t m = 0;
        if (k0 > 0 && lim == 32) {
            m = g_have_avx2 ? neq32_avx2(vb, k0) : neq32_scalar(vb, k0);
        } else {
            for (int i = 0; i < lim; ++i) m |= (uint32_t)(k0 + i == 0 || vb[k0 + i] != vb[k0 + i - 1]) << i;
        }
        bits[w] = m;
        while (m) {
            out.push_back(vals[k0 + __builtin_ctz(m)]);
            m &= m - 1;
        }
    }
}

// values[k] = runs[(set bits at positions <= k) - 1]: one warp per bit word,
// one lane per entry (coalesced stores; the word and its base are broadcast).
__global__ void value_expand_kernel(const uint32_t* __restrict__ bits, const uint32_t* __restrict__ word_base,
                                    const double* __restrict__ runs, int64_t nnz, double* __restrict__ values) {
    const uint32_t lane = threadIdx.x & 31u;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = k >> 5;
        const uint32_t b = bits[w];
        const uint32_t upto = b & (0xffffffffu >> (31u - lane));  // bits at positions <= lane
        values[k] = runs[(int64_t)word_base[w] + __popc(upto) - 1];
    }
}
__global__ void popc_kernel(const uint32_t* __restrict__ bits, int64_t nw, uint32_t* __restrict__ cnt) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x)
        cnt[w] = __popc(bits[w]);
}

void download_u32_as_i64(const uint32_t* d, size_t n, int64_t* h, cudaStream_t s) {
    if (!h || !n) return;
    DevBuf<int64_t> tmp(n, s);
    widen_u32<<<(unsigned)prg::num_sms() * 4, 1024, 0, s>>>(d, (int64_t)n, tmp.get());
    PRG_LAUNCH_CHECK();
    prg::copy_to_host(h, tmp.get(), n * 8, s);
}

}  // namespace

extern "C" {

const char* prg_last_error(void) { return prg::last_error().c_str(); }
const char* prg_version(void) { return "prg-b200 0.1.0 (sm_100a)"; }

int64_t prg_launch_count(void) { return prg::launch_count(); }

int64_t prg_debug_check_failures(void) {
    try {
        return (int64_t)prg::check_failures_runtime() + prg::check_failures_sort() + prg::check_failures_k0() +
               prg::check_failures_k1() + prg::check_failures_k2() + prg::check_failures_k3() +
               prg::check_failures_k2steps() + prg::check_failures_capi();
    } catch (const prg::CudaError& e) {
        prg::set_error(e.msg);
        return -1;
    }
}
int64_t prg_last_h2d_bytes(void) { return g_last_h2d_bytes; }
void prg_profile_enable(int32_t on) { prg::profiling_enable(on != 0); }
prg_status prg_trim_memory(void) {
    return guarded("prg_trim_memory", [&] {
        PRG_CUDA(cudaDeviceSynchronize());
        prg::ws_trim();
    });
}
int64_t prg_profile_report(char* buf, int64_t cap, int32_t reset) {
    const std::string s = prg::profile_report(reset != 0);
    if (buf && cap > 0) {
        const size_t k = std::min<size_t>((size_t)cap - 1, s.size());
        std::memcpy(buf, s.data(), k);
        buf[k] = 0;
    }
    return (int64_t)s.size();
}

int32_t prg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

prg_status prg_k0_permutation(int32_t scale, uint64_t seed, int64_t* labels) {
    return guarded("prg_k0_permutation", [&] {
        require(scale >= 0 && scale <= 40 && labels, PRG_ERR_INVALID_ARGUMENT, "bad scale or null buffer");
        const int64_t n = int64_t{1} << scale;
        for (int64_t i = 0; i < n; ++i) labels[i] = i + 1;
        // graph_gen.cpp:72-76, SplitMix64(mix_seed(seed, kPermutationStream))
        uint64_t st = prg::dev::mix_seed(seed, 0x7065726d75746174ULL);
        for (int64_t i = n - 1; i > 0; --i) {
            uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            z ^= z >> 31;
            const int64_t j = (int64_t)(z % ((uint64_t)i + 1));
            std::swap(labels[i], labels[j]);
        }
    });
}

prg_status prg_k0_generate_device(int32_t scale, int64_t edge_factor, uint64_t seed,
                                  const double initiator[4], const int64_t* d_labels, int64_t first,
                                  int64_t count, int64_t* d_uv, void* stream) {
    return guarded("prg_k0_generate_device", [&] {
        require(scale >= 1 && scale <= 40 && count >= 0 && first >= 0 && initiator, PRG_ERR_INVALID_ARGUMENT,
                "bad generator arguments");
        prg::k0_generate_device(scale, edge_factor, seed, initiator, d_labels, first, count, d_uv,
                                as_stream(stream));
    });
}

prg_status prg_k1_sort_device(const int64_t* d_uv_in, int64_t m, int32_t scale, int64_t* d_uv_out,
                              void* stream) {
    return guarded("prg_k1_sort", [&] {
        require(m >= 0 && scale >= 0 && scale <= 32, PRG_ERR_INVALID_ARGUMENT, "scale must be in [0, 32]");
        require(m == 0 || (d_uv_in && d_uv_out && d_uv_in != d_uv_out), PRG_ERR_INVALID_ARGUMENT,
                "null or aliased edge buffers");
        require((uint64_t)m < (1ull << 32), PRG_ERR_INVALID_ARGUMENT, "more than 2^32-1 edges");
        if (m == 0) return;
        cudaStream_t s = as_stream(stream);
        DevBuf<uint32_t> err(1, s);
        PRG_CUDA(cudaMemsetAsync(err.get(), 0, 4, s));
        prg::k1_sort_device(d_uv_in, m, scale, d_uv_out, err.get(), s);
        uint32_t h = 0;
        PRG_CUDA(cudaMemcpyAsync(&h, err.get(), 4, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        check_device_errors(h, "K1");
    });
}

prg_status prg_k1_sort_host(const int64_t* uv_in, int64_t m, int32_t scale, int64_t* uv_out) {
    return guarded("prg_k1_sort_host", [&] {
        require(m >= 0, PRG_ERR_INVALID_ARGUMENT, "negative edge count");
        if (m == 0) return;
        cudaStream_t s = nullptr;
        DevBuf<int64_t> a((size_t)m * 2, s), b((size_t)m * 2, s);
        prg::copy_to_device(a.get(), uv_in, (size_t)m * 16, s);
        const prg_status st = prg_k1_sort_device(a.get(), m, scale, b.get(), s);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
        prg::copy_to_host(uv_out, b.get(), (size_t)m * 16, s);
    });
}

// K1 under a host-memory budget: see include/prg.h. The device holds the whole
// list (the B200's "memory" is its HBM); the host only ever holds one pinned
// chunk, filled by the source and drained to the sink.
prg_status prg_k1_sort_streamed(prg_edge_source source, prg_edge_sink sink, void* user, int64_t m, int32_t scale,
                                int64_t chunk_edges) {
    return guarded("prg_k1_sort_streamed", [&] {
        require(source && sink && m >= 0 && chunk_edges >= 1, PRG_ERR_INVALID_ARGUMENT, "bad streamed-sort arguments");
        require((uint64_t)m < (1ull << 32), PRG_ERR_INVALID_ARGUMENT,
                "K1: " + std::to_string(m) + " edges exceed the device sort's 2^32-1 per call");
        if (m == 0) return;
        cudaStream_t s = nullptr;
        // input + output lists, 2 key buffers and scratch: ~56 B per edge on the device
        size_t free_b = 0, total_b = 0;
        PRG_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const double need = 56.0 * (double)m;
        require(need < 0.95 * (double)free_b, PRG_ERR_INVALID_ARGUMENT,
                "K1: " + std::to_string(m) + " edges need ~" + std::to_string((int64_t)(need / 1e9)) +
                    " GB of device memory, " + std::to_string((int64_t)(free_b / 1e9)) + " GB free");
        const int64_t chunk = std::min<int64_t>(chunk_edges, m);
        int64_t* pinned = nullptr;
        PRG_CUDA(cudaMallocHost(&pinned, (size_t)chunk * 16));
        struct FreeHost {
            int64_t* p;
            ~FreeHost() { cudaFreeHost(p); }
        } free_pinned{pinned};
        DevBuf<int64_t> a((size_t)m * 2, s), b((size_t)m * 2, s);
        for (int64_t got = 0; got < m;) {
            const int64_t k = source(user, pinned, std::min(chunk, m - got));
            require(k > 0 && k <= std::min(chunk, m - got), PRG_ERR_INVALID_ARGUMENT,
                    "K1: the edge source ended after " + std::to_string(got) + " of " + std::to_string(m) + " edges");
            PRG_CUDA(cudaMemcpyAsync(a.get() + 2 * got, pinned, (size_t)k * 16, cudaMemcpyHostToDevice, s));
            PRG_CUDA(cudaStreamSynchronize(s));  // the chunk buffer is refilled next
            got += k;
        }
        const prg_status st = prg_k1_sort_device(a.get(), m, scale, b.get(), s);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
        for (int64_t put = 0; put < m;) {
            const int64_t k = std::min(chunk, m - put);
            PRG_CUDA(cudaMemcpyAsync(pinned, b.get() + 2 * put, (size_t)k * 16, cudaMemcpyDeviceToHost, s));
            PRG_CUDA(cudaStreamSynchronize(s));
            require(sink(user, pinned, k) == 0, PRG_ERR_INVALID_ARGUMENT, "K1: the edge sink failed");
            put += k;
        }
    });
}

prg_status prg_k2_filter_device(const int64_t* d_uv_sorted, int64_t m, int64_t n, prg_matrix** out,
                                void* stream) {
    return guarded("prg_k2_filter", [&] {
        require(out != nullptr, PRG_ERR_INVALID_ARGUMENT, "null output handle");
        *out = nullptr;
        require(n > 0, PRG_ERR_INVALID_ARGUMENT, "vertex count must be positive");
        require(m >= 0 && (uint64_t)m < (1ull << 32) && (uint64_t)n < (1ull << 32), PRG_ERR_INVALID_ARGUMENT,
                "sizes exceed the u32 index range");
        cudaStream_t s = as_stream(stream);
        auto* mat = new prg_matrix();
        try {
            const uint32_t err = prg::k2_filter_device(d_uv_sorted, m, n, mat, s);
            check_device_errors(err, "K2");
        } catch (...) {
            delete mat;
            throw;
        }
        *out = mat;
    });
}

prg_status prg_k2_filter_host(const int64_t* uv_sorted, int64_t m, int64_t n, prg_matrix** out) {
    return guarded("prg_k2_filter_host", [&] {
        require(m >= 0, PRG_ERR_INVALID_ARGUMENT, "negative edge count");
        cudaStream_t s = nullptr;
        DevBuf<int64_t> a((size_t)std::max<int64_t>(m, 1) * 2, s);
        if (m) prg::copy_to_device(a.get(), uv_sorted, (size_t)m * 16, s);
        const prg_status st = prg_k2_filter_device(a.get(), m, n, out, s);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
    });
}

prg_status prg_build_adjacency_host(const int64_t* uv_sorted, int64_t m, int64_t n, int64_t* row_offsets,
                                    int64_t* cols, int64_t* counts, int64_t* nnz) {
    return guarded("prg_build_adjacency", [&] {
        require(n > 0, PRG_ERR_INVALID_ARGUMENT, "vertex count must be positive");
        require(m >= 0 && (uint64_t)m < (1ull << 32) && (uint64_t)n < (1ull << 32), PRG_ERR_INVALID_ARGUMENT,
                "sizes exceed the u32 index range");
        cudaStream_t s = nullptr;
        DevBuf<int64_t> a((size_t)std::max<int64_t>(m, 1) * 2, s);
        if (m) prg::copy_to_device(a.get(), uv_sorted, (size_t)m * 16, s);
        std::unique_ptr<prg_matrix> mat(new prg_matrix());
        const uint32_t err = prg::k2_filter_device(a.get(), m, n, mat.get(), s, /*filter=*/false, /*normalize=*/false);
        check_device_errors(err, "build_adjacency");
        download_u32_as_i64(mat->row_offsets, (size_t)n + 1, row_offsets, s);
        download_u32_as_i64(mat->cols, (size_t)mat->nnz, cols, s);
        if (mat->nnz) {
            std::vector<double> v(mat->nnz);
            PRG_CUDA(cudaMemcpy(v.data(), mat->values, mat->nnz * 8, cudaMemcpyDeviceToHost));
            for (uint64_t k = 0; k < mat->nnz; ++k) counts[k] = (int64_t)v[k];  // exact integers
        }
        *nnz = (int64_t)mat->nnz;
    });
}

prg_status prg_in_degree_host(int64_t n, int64_t nnz, const int64_t* cols, const int64_t* counts, int64_t* d_in) {
    return guarded("prg_in_degree", [&] {
        require(n > 0 && nnz >= 0, PRG_ERR_INVALID_ARGUMENT, "bad sizes");
        cudaStream_t s = nullptr;
        DevBuf<int64_t> dc((size_t)std::max<int64_t>(nnz, 1), s), dn((size_t)std::max<int64_t>(nnz, 1), s),
            dd((size_t)n, s);
        if (nnz) {
            PRG_CUDA(cudaMemcpyAsync(dc.get(), cols, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
            PRG_CUDA(cudaMemcpyAsync(dn.get(), counts, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
        }
        prg::k2_in_degree_device(n, nnz, dc.get(), dn.get(), dd.get(), s);
        PRG_CUDA(cudaMemcpyAsync(d_in, dd.get(), (size_t)n * 8, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
    });
}

prg_status prg_zero_columns_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                 const int64_t* counts, const int64_t* d_in, int64_t* out_row_offsets,
                                 int64_t* out_cols, int64_t* out_counts, int64_t* out_nnz) {
    return guarded("prg_zero_columns", [&] {
        require(n > 0 && nnz >= 0, PRG_ERR_INVALID_ARGUMENT, "bad sizes");
        cudaStream_t s = nullptr;
        const size_t z = (size_t)std::max<int64_t>(nnz, 1);
        DevBuf<int64_t> ro((size_t)n + 1, s), dc(z, s), dn(z, s), dd((size_t)n, s), oro((size_t)n + 1, s),
            oc(z, s), on(z, s);
        PRG_CUDA(cudaMemcpyAsync(ro.get(), row_offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
        PRG_CUDA(cudaMemcpyAsync(dd.get(), d_in, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        if (nnz) {
            PRG_CUDA(cudaMemcpyAsync(dc.get(), cols, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
            PRG_CUDA(cudaMemcpyAsync(dn.get(), counts, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
        }
        const int64_t nz = prg::k2_zero_columns_device(n, ro.get(), dc.get(), dn.get(), dd.get(), oro.get(),
                                                       oc.get(), on.get(), s);
        PRG_CUDA(cudaMemcpyAsync(out_row_offsets, oro.get(), (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost, s));
        if (nz) {
            PRG_CUDA(cudaMemcpyAsync(out_cols, oc.get(), (size_t)nz * 8, cudaMemcpyDeviceToHost, s));
            PRG_CUDA(cudaMemcpyAsync(out_counts, on.get(), (size_t)nz * 8, cudaMemcpyDeviceToHost, s));
        }
        PRG_CUDA(cudaStreamSynchronize(s));
        *out_nnz = nz;
    });
}

prg_status prg_row_normalize_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* counts,
                                  double* values) {
    return guarded("prg_row_normalize", [&] {
        require(n > 0 && nnz >= 0, PRG_ERR_INVALID_ARGUMENT, "bad sizes");
        if (!nnz) return;
        cudaStream_t s = nullptr;
        DevBuf<int64_t> ro((size_t)n + 1, s), dn((size_t)nnz, s);
        DevBuf<double> dv((size_t)nnz, s);
        PRG_CUDA(cudaMemcpyAsync(ro.get(), row_offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
        PRG_CUDA(cudaMemcpyAsync(dn.get(), counts, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
        PRG_CUDA(cudaMemsetAsync(dv.get(), 0, (size_t)nnz * 8, s));
        prg::k2_row_normalize_device(n, ro.get(), dn.get(), dv.get(), s);
        PRG_CUDA(cudaMemcpyAsync(values, dv.get(), (size_t)nnz * 8, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
    });
}

prg_status prg_matrix_info(const prg_matrix* a, int64_t* n, int64_t* nnz, int64_t* nnz_raw, int64_t* max_in) {
    return guarded("prg_matrix_info", [&] {
        require(a != nullptr, PRG_ERR_INVALID_ARGUMENT, "null matrix");
        if (n) *n = a->n;
        if (nnz) *nnz = (int64_t)a->nnz;
        if (nnz_raw) *nnz_raw = (int64_t)a->nnz_raw;
        if (max_in) *max_in = (int64_t)a->max_in;
    });
}

prg_status prg_matrix_download(const prg_matrix* a, int64_t* row_offsets, int64_t* cols, double* values,
                               int64_t* d_in) {
    return guarded("prg_matrix_download", [&] {
        require(a != nullptr, PRG_ERR_INVALID_ARGUMENT, "null matrix");
        cudaStream_t s = nullptr;
        download_u32_as_i64(a->row_offsets, (size_t)a->n + 1, row_offsets, s);
        download_u32_as_i64(a->cols, (size_t)a->nnz, cols, s);
        if (values && a->nnz) prg::copy_to_host(values, a->values, a->nnz * 8, s);
        if (d_in) {
            if (a->d_in) download_u32_as_i64(a->d_in, (size_t)a->n, d_in, s);
            else std::memset(d_in, 0, (size_t)a->n * 8);
        }
    });
}

prg_status prg_matrix_device_arrays(const prg_matrix* a, const uint32_t** ro, const uint32_t** cols,
                                    const double** values, const uint32_t** d_in) {
    return guarded("prg_matrix_device_arrays", [&] {
        require(a != nullptr, PRG_ERR_INVALID_ARGUMENT, "null matrix");
        if (ro) *ro = a->row_offsets;
        if (cols) *cols = a->cols;
        if (values) *values = a->values;
        if (d_in) *d_in = a->d_in;
    });
}

prg_status prg_matrix_from_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                const double* values, prg_matrix** out) {
    return guarded("prg_matrix_from_host", [&] {
        require(out != nullptr, PRG_ERR_INVALID_ARGUMENT, "null output handle");
        *out = nullptr;
        require(n > 0 && nnz >= 0 && (uint64_t)nnz < (1ull << 32) && (uint64_t)n < (1ull << 32),
                PRG_ERR_INVALID_ARGUMENT, "bad matrix sizes");
        require(row_offsets[0] == 0 && row_offsets[n] == nnz, PRG_ERR_INVALID_ARGUMENT,
                "row_offsets must start at 0 and end at nnz");
        cudaStream_t s = nullptr;
        auto mat = std::make_unique<prg_matrix>();
        mat->n = n;
        mat->nnz = (uint64_t)nnz;
        mat->cap = (uint64_t)nnz;
        mat->row_offsets = dmalloc<uint32_t>((size_t)n + 1);
        mat->cols = dmalloc<uint32_t>((size_t)nnz);
        mat->values = dmalloc<double>((size_t)nnz);
        DevBuf<uint32_t> err(1, s);
        PRG_CUDA(cudaMemsetAsync(err.get(), 0, 4, s));
        {
            DevBuf<int64_t> tmp((size_t)n + 1, s);
            PRG_CUDA(cudaMemcpyAsync(tmp.get(), row_offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
            narrow_offsets<<<(unsigned)prg::num_sms() * 4, 1024, 0, s>>>(tmp.get(), n + 1, nnz, mat->row_offsets,
                                                                          err.get());
            PRG_LAUNCH_CHECK();
        }
        if (nnz) {
            DevBuf<int64_t> tmp((size_t)nnz, s);
            PRG_CUDA(cudaMemcpyAsync(tmp.get(), cols, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
            narrow_i64<<<(unsigned)prg::num_sms() * 4, 1024, 0, s>>>(tmp.get(), nnz, n - 1, mat->cols, err.get());
            PRG_LAUNCH_CHECK();
            PRG_CUDA(cudaMemcpyAsync(mat->values, values, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
        }
        uint32_t h = 0;
        PRG_CUDA(cudaMemcpyAsync(&h, err.get(), 4, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        check_upload_flags(h);
        *out = mat.release();
    });
}

void prg_matrix_destroy(prg_matrix* a) { delete a; }

prg_status prg_matrix_build_csc(prg_matrix* a, void* stream) {
    return guarded("prg_matrix_build_csc", [&] {
        require(a != nullptr, PRG_ERR_INVALID_ARGUMENT, "null matrix");
        prg::k3_build_csc_device(a, as_stream(stream));
    });
}

prg_status prg_matrix_drop_csc(prg_matrix* a) {
    return guarded("prg_matrix_drop_csc", [&] {
        require(a != nullptr, PRG_ERR_INVALID_ARGUMENT, "null matrix");
        if (a->plan) {
            PRG_CUDA(cudaDeviceSynchronize());
            prg::k3_plan_destroy(a->plan);
            a->plan = nullptr;
        }
    });
}

int32_t prg_matrix_has_csc(const prg_matrix* a) { return a && a->plan ? 1 : 0; }

prg_status prg_k3_pagerank_device(const prg_matrix* a, double damping, int32_t iterations, uint64_t seed,
                                  int32_t mode, double* d_ranks, double* norm1, void* stream) {
    return guarded("prg_k3_pagerank", [&] {
        require(a != nullptr && d_ranks != nullptr, PRG_ERR_INVALID_ARGUMENT, "null argument");
        // PageRankConfig::validate (kernel3_pagerank.cpp:23-27)
        require(damping > 0.0 && damping < 1.0, PRG_ERR_INVALID_ARGUMENT, "damping must lie strictly between 0 and 1");
        require(iterations >= 1, PRG_ERR_INVALID_ARGUMENT, "iteration count must be >= 1");
        require(mode >= 0 && mode <= 2, PRG_ERR_INVALID_ARGUMENT, "mode must be 0 (timed), 1 (parity) or 2 (Neumaier)");
        prg::K3Options o;
        o.damping = damping;
        o.iterations = iterations;
        o.seed = seed;
        o.mode = mode;
        const double nm = prg::k3_pagerank_device(a, o, d_ranks, as_stream(stream));
        if (norm1) *norm1 = nm;
    });
}

prg_status prg_k3_pagerank_sharded(const prg_matrix* a, double damping, int32_t iterations, uint64_t seed,
                                   int32_t rank, int32_t world, prg_allreduce_f64 allreduce, void* user,
                                   double* d_ranks, double* norm1, void* stream) {
    return guarded("prg_k3_pagerank_sharded", [&] {
        require(a != nullptr && d_ranks != nullptr && allreduce != nullptr, PRG_ERR_INVALID_ARGUMENT, "null argument");
        require(damping > 0.0 && damping < 1.0, PRG_ERR_INVALID_ARGUMENT, "damping must lie strictly between 0 and 1");
        require(iterations >= 1, PRG_ERR_INVALID_ARGUMENT, "iteration count must be >= 1");
        require(world >= 1 && rank >= 0 && rank < world, PRG_ERR_INVALID_ARGUMENT, "rank must lie in [0, world)");
        prg::K3Options o;
        o.damping = damping;
        o.iterations = iterations;
        o.seed = seed;
        const double nm = prg::k3_pagerank_sharded_device(a, o, rank, world, allreduce, user, d_ranks, as_stream(stream));
        if (norm1) *norm1 = nm;
    });
}

prg_status prg_k3_shard_bounds(const prg_matrix* a, int32_t world, uint32_t* bounds, void* stream) {
    return guarded("prg_k3_shard_bounds", [&] {
        require(a != nullptr && bounds != nullptr && world >= 1, PRG_ERR_INVALID_ARGUMENT, "bad arguments");
        prg::k3_shard_bounds(a, world, bounds, as_stream(stream));
    });
}

prg_status prg_shard_bounds_host(const uint32_t* slice_ptr, uint32_t nslices, int32_t world, uint32_t* bounds) {
    return guarded("prg_shard_bounds_host", [&] {
        require(slice_ptr != nullptr && bounds != nullptr && world >= 1, PRG_ERR_INVALID_ARGUMENT, "bad arguments");
        for (uint32_t i = 0; i < nslices; ++i)
            require(slice_ptr[i] <= slice_ptr[i + 1], PRG_ERR_INVALID_ARGUMENT, "slice offsets must be non-decreasing");
        prg::k3_shard_bounds_host(slice_ptr, nslices, world, bounds);
    });
}

prg_status prg_k3_pagerank_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                const double* values, double damping, int32_t iterations, uint64_t seed,
                                int32_t mode, double* ranks, double* norm1) {
    return guarded("prg_k3_pagerank_host", [&] {
        require(ranks != nullptr && row_offsets != nullptr, PRG_ERR_INVALID_ARGUMENT, "null argument");
        require(n > 0 && nnz >= 0 && (uint64_t)nnz < (1ull << 32) && (uint64_t)n < (1ull << 32),
                PRG_ERR_INVALID_ARGUMENT, "bad matrix sizes");
        require(nnz == 0 || (cols != nullptr && values != nullptr), PRG_ERR_INVALID_ARGUMENT, "null argument");
        require(row_offsets[0] == 0 && row_offsets[n] == nnz, PRG_ERR_INVALID_ARGUMENT,
                "row_offsets must start at 0 and end at nnz");
        cudaStream_t s = nullptr;
        const bool dbg = getenv("PRG_E2E_DEBUG") != nullptr;
        auto now = [] {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
        };
        const double t0 = now();
        auto mat = std::make_unique<prg_matrix>();
        mat->n = n;
        mat->nnz = mat->cap = (uint64_t)nnz;
        mat->row_offsets = dmalloc<uint32_t>((size_t)n + 1);
        mat->cols = dmalloc<uint32_t>((size_t)nnz);
        mat->values = dmalloc<double>((size_t)nnz);
        DevBuf<uint32_t> err(1, s);
        PRG_CUDA(cudaMemsetAsync(err.get(), 0, 4, s));
        // 1. the host's cores run-length code the values (worker threads) ...
        PinnedStage& pb = pinned_stage(0);
        PinnedStage& pr = pinned_stage(1);
        std::lock_guard<std::mutex> lock_b(pb.mu), lock_r(pr.mu);
        const int64_t nw = (nnz + 31) / 32;
        uint32_t* hbits = nnz ? static_cast<uint32_t*>(pb.get((size_t)nw * 4)) : nullptr;
        const int T = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::vector<double>> parts((size_t)T);
        std::vector<std::thread> workers;
        struct Joiner {  // never leave a worker running (an exception would terminate)
            std::vector<std::thread>& w;
            ~Joiner() {
                for (auto& t : w)
                    if (t.joinable()) t.join();
            }
        } joiner{workers};
        if (nnz)
            for (int t = 0; t < T; ++t)
                workers.emplace_back([&, t] { rle_values(values, nnz, nw * t / T, nw * (t + 1) / T, hbits, parts[t]); });
        // 2. ... while this thread ships the structure over PCIe (async when the
        // caller's buffers are pinned; staged, but still concurrent, when pageable)
        DevBuf<int64_t> tro((size_t)n + 1, s), tcol(nnz ? (size_t)nnz : 1, s);
        PRG_CUDA(cudaMemcpyAsync(tro.get(), row_offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
        narrow_offsets<<<(unsigned)prg::num_sms() * 4, 1024, 0, s>>>(tro.get(), n + 1, nnz, mat->row_offsets, err.get());
        PRG_LAUNCH_CHECK();
        int64_t runs = 0;
        double t1 = now(), t2 = t1;
        if (nnz) {
            PRG_CUDA(cudaMemcpyAsync(tcol.get(), cols, (size_t)nnz * 8, cudaMemcpyHostToDevice, s));
            narrow_i64<<<(unsigned)prg::num_sms() * 4, 1024, 0, s>>>(tcol.get(), nnz, n - 1, mat->cols, err.get());
            PRG_LAUNCH_CHECK();
            for (auto& w : workers) w.join();
            std::vector<int64_t> off((size_t)T + 1, 0);
            for (int t = 0; t < T; ++t) off[t + 1] = off[t] + (int64_t)parts[t].size();
            runs = off[T];
            double* hruns = static_cast<double*>(pr.get((size_t)runs * 8));
            parallel_for(T, [&](int t) { std::memcpy(hruns + off[t], parts[t].data(), parts[t].size() * 8); });
            t1 = now();
            DevBuf<uint32_t> dbits((size_t)nw, s), wcnt((size_t)nw, s), wbase((size_t)nw, s);
            DevBuf<double> druns((size_t)runs, s);
            PRG_CUDA(cudaMemcpyAsync(dbits.get(), hbits, (size_t)nw * 4, cudaMemcpyHostToDevice, s));
            PRG_CUDA(cudaMemcpyAsync(druns.get(), hruns, (size_t)runs * 8, cudaMemcpyHostToDevice, s));
            const unsigned g = (unsigned)prg::num_sms() * 8;
            popc_kernel<<<g, 1024, 0, s>>>(dbits.get(), nw, wcnt.get());
            PRG_LAUNCH_CHECK();
            prg::exclusive_scan_u32(wcnt.get(), wbase.get(), (size_t)nw, nullptr, s);
            value_expand_kernel<<<g, 1024, 0, s>>>(dbits.get(), wbase.get(), druns.get(), nnz, mat->values);
            PRG_LAUNCH_CHECK();
            t2 = now();
            uint32_t h = 0;
            PRG_CUDA(cudaMemcpyAsync(&h, err.get(), 4, cudaMemcpyDeviceToHost, s));
            PRG_CUDA(cudaStreamSynchronize(s));  // uploads done: the pinned stages are reused by the next call
            check_upload_flags(h);
        }
        g_last_h2d_bytes = (n + 1) * 8 + nnz * 8 + (nnz + 31) / 32 * 4 + runs * 8;
        const double t3 = now();
        // 3. K3 on the device, ranks back
        DevBuf<double> r((size_t)n, s);
        prg_status st = prg_k3_pagerank_device(mat.get(), damping, iterations, seed, mode, r.get(), norm1, s);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
        const double t4 = now();
        PRG_CUDA(cudaMemcpyAsync(ranks, r.get(), (size_t)n * 8, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        if (dbg)
            fprintf(stderr, "[e2e] host run-length pass %.1f ms | enqueue %.1f | wait uploads %.1f | k3 %.1f | d2h %.1f"
                    " | total %.1f (runs %lld)\n",
                    t1 - t0, t2 - t1, now() - t4 > 0 ? t3 - t2 : 0.0, t4 - t3, now() - t4, now() - t0, (long long)runs);
    });
}

prg_status prg_init_rank_device(int64_t n, uint64_t seed, int32_t mode, double* d_r, double* norm1, void* stream) {
    return guarded("prg_init_rank", [&] {
        require(n >= 1, PRG_ERR_INVALID_ARGUMENT, "rank vector needs at least one entry");
        const double nm = prg::k3_init_rank_device(n, seed, d_r, mode, as_stream(stream));
        if (norm1) *norm1 = nm;
    });
}

prg_status prg_pagerank_step_device(const prg_matrix* a, const double* d_r, double damping, int32_t mode,
                                    double* d_out, double* norm1, void* stream) {
    return guarded("prg_pagerank_step", [&] {
        require(a != nullptr && d_r && d_out, PRG_ERR_INVALID_ARGUMENT, "null argument");
        const double nm = prg::k3_step_device(a, d_r, damping, d_out, mode, as_stream(stream));
        if (norm1) *norm1 = nm;
    });
}

prg_status prg_init_rank_host(int64_t n, uint64_t seed, int32_t mode, double* r, double* norm1) {
    return guarded("prg_init_rank_host", [&] {
        require(n >= 1, PRG_ERR_INVALID_ARGUMENT, "rank vector needs at least one entry");
        cudaStream_t s = nullptr;
        DevBuf<double> d((size_t)n, s);
        const double nm = prg::k3_init_rank_device(n, seed, d.get(), mode, s);
        PRG_CUDA(cudaMemcpy(r, d.get(), (size_t)n * 8, cudaMemcpyDeviceToHost));
        if (norm1) *norm1 = nm;
    });
}

prg_status prg_pagerank_step_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                  const double* values, const double* r, double damping, int32_t mode,
                                  double* out, double* norm1) {
    return guarded("prg_pagerank_step_host", [&] {
        prg_matrix* a = nullptr;
        prg_status st = prg_matrix_from_host(n, nnz, row_offsets, cols, values, &a);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
        std::unique_ptr<prg_matrix> own(a);
        cudaStream_t s = nullptr;
        DevBuf<double> dr((size_t)n, s), dout((size_t)n, s);
        PRG_CUDA(cudaMemcpyAsync(dr.get(), r, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        const double nm = prg::k3_step_device(a, dr.get(), damping, dout.get(), mode, s);
        PRG_CUDA(cudaMemcpy(out, dout.get(), (size_t)n * 8, cudaMemcpyDeviceToHost));
        if (norm1) *norm1 = nm;
    });
}

prg_status prg_k3_pagerank_matrix_host(const prg_matrix* a, double damping, int32_t iterations, uint64_t seed,
                                       int32_t mode, double* ranks, double* norm1) {
    return guarded("prg_k3_pagerank_matrix_host", [&] {
        require(a != nullptr && ranks != nullptr, PRG_ERR_INVALID_ARGUMENT, "null argument");
        cudaStream_t s = nullptr;
        DevBuf<double> r((size_t)a->n, s);
        const prg_status st = prg_k3_pagerank_device(a, damping, iterations, seed, mode, r.get(), norm1, s);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
        PRG_CUDA(cudaMemcpy(ranks, r.get(), (size_t)a->n * 8, cudaMemcpyDeviceToHost));
    });
}

prg_status prg_run_to_convergence_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                       const double* values, double damping, double tol, int32_t max_iters,
                                       const double* start, double* out, int32_t* converged,
                                       int32_t* iterations) {
    return guarded("prg_run_to_convergence_host", [&] {
        // kernel3_pagerank.cpp:89-91
        require(tol > 0.0, PRG_ERR_INVALID_ARGUMENT, "convergence tolerance must be positive");
        require(max_iters >= 1, PRG_ERR_INVALID_ARGUMENT, "max_iters must be >= 1");
        prg_matrix* a = nullptr;
        prg_status st = prg_matrix_from_host(n, nnz, row_offsets, cols, values, &a);
        if (st != PRG_OK) throw ApiError{st, prg::last_error()};
        std::unique_ptr<prg_matrix> own(a);
        cudaStream_t s = nullptr;
        DevBuf<double> d0((size_t)n, s), d1((size_t)n, s);
        PRG_CUDA(cudaMemcpyAsync(d0.get(), start, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        bool conv = false;
        int its = 0;
        try {
            its = prg::k3_converge_device(a, damping, tol, max_iters, d0.get(), d1.get(), &conv, s);
        } catch (const CudaError& e) {
            throw ApiError{PRG_ERR_INVALID_ARGUMENT, e.msg};
        }
        PRG_CUDA(cudaMemcpy(out, d1.get(), (size_t)n * 8, cudaMemcpyDeviceToHost));
        *converged = conv ? 1 : 0;
        *iterations = its;
    });
}

}  // extern "C"

PRG_CHECK_QUERY(capi)
