// ref_driver.cpp — extern "C" harness around the REFERENCE implementation.
//
// TEST INFRASTRUCTURE ONLY (see oracle/prg_oracle.c header). This file is
// compiled together with the reference's own sources, straight from
// /root/reference/proj/src (never copied), by oracle/build_ref.sh into
// oracle/_ref/libprpipe_ref.so. It lets tests/ generate golden vectors from the
// reference itself and lets bench.py time the reference's CPU path
// ("cpu_baseline.kind": "reference").
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "prpipe/edge_io.hpp"
#include "prpipe/graph_gen.hpp"
#include "prpipe/kernel2_filter.hpp"
#include "prpipe/kernel3_pagerank.hpp"

using namespace prpipe;

namespace {
thread_local std::string g_err;
double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// K0: EdgeGenerator::fill_batch, batches spread over `threads` threads
// (bit-identical to sequential generation: tests/test_graph_gen.cpp:168-188).
int ref_generate(int scale, std::uint64_t seed, const double* init, int permute, int threads,
                 std::int64_t* uv) {
    try {
        GenConfig c;
        c.scale = scale;
        c.seed = seed;
        for (int i = 0; i < 4; ++i) c.initiator[i] = init[i];
        c.permute_labels = permute != 0;
        EdgeGenerator gen(c);
        const std::int64_t nb = gen.batch_count();
        auto work = [&](int t) {
            std::vector<Edge> batch;
            for (std::int64_t b = t; b < nb; b += threads) {
                gen.fill_batch(b, batch);
                std::memcpy(uv + 2 * b * EdgeGenerator::kBatchEdges, batch.data(),
                            batch.size() * sizeof(Edge));
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// K1 core: the reference's in-memory sort, std::sort by start vertex only
// (src/kernel1_sort.cpp:14,66). Sorts in place; returns elapsed seconds.
double ref_k1_sort_core(std::int64_t* uv, std::int64_t m) {
    auto* e = reinterpret_cast<Edge*>(uv);
    const double t0 = now_s();
    std::sort(e, e + m, [](const Edge& a, const Edge& b) { return a.u < b.u; });
    return now_s() - t0;
}

// K2 core: build_adjacency(span) + in_degree + zero_columns + row_normalize
// (include/prpipe/kernel2_filter.hpp:42-54). Output buffers: row_offsets[n+1],
// cols/values[m] (nnz_f <= m), d_in[n]. Returns nnz_f (>= 0) or -1 on error.
std::int64_t ref_k2_core(const std::int64_t* uv, std::int64_t m, std::int64_t n,
                         std::int64_t* row_offsets, std::int64_t* cols, double* values,
                         std::int64_t* d_in, std::int64_t* nnz_raw, double* elapsed) {
    try {
        std::span<const Edge> edges(reinterpret_cast<const Edge*>(uv), static_cast<std::size_t>(m));
        const double t0 = now_s();
        CountMatrix a = build_adjacency(edges, n);
        const auto din = in_degree(a);
        const CountMatrix f = zero_columns(a, din);
        const StochasticMatrix s = row_normalize(f);
        if (elapsed) *elapsed = now_s() - t0;
        if (nnz_raw) *nnz_raw = a.nnz();
        std::memcpy(row_offsets, s.row_offsets.data(), sizeof(std::int64_t) * (n + 1));
        std::memcpy(cols, s.cols.data(), sizeof(std::int64_t) * s.cols.size());
        std::memcpy(values, s.values.data(), sizeof(double) * s.values.size());
        std::memcpy(d_in, din.data(), sizeof(std::int64_t) * n);
        return s.nnz();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// K3: run_kernel3 (src/kernel3_pagerank.cpp:67-79) on a CSR given as arrays.
// Returns norm1; elapsed seconds of the reference's own timed region.
double ref_k3(std::int64_t n, std::int64_t nnz, const std::int64_t* row_offsets,
              const std::int64_t* cols, const double* values, double damping, int iterations,
              std::uint64_t seed, std::int64_t total_edges, double* ranks, double* elapsed) {
    try {
        StochasticMatrix s;
        s.n = n;
        s.row_offsets.assign(row_offsets, row_offsets + n + 1);
        s.cols.assign(cols, cols + nnz);
        s.values.assign(values, values + nnz);
        PageRankConfig c;
        c.damping = damping;
        c.iterations = iterations;
        c.seed = seed;
        auto res = run_kernel3(s, c, total_edges);
        if (elapsed) *elapsed = res.elapsed_seconds;
        std::memcpy(ranks, res.ranks.values.data(), sizeof(double) * n);
        return res.ranks.norm1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// One reference pagerank_step (src/kernel3_pagerank.cpp:41-65); returns norm1.
double ref_pagerank_step(std::int64_t n, std::int64_t nnz, const std::int64_t* row_offsets,
                         const std::int64_t* cols, const double* values, const double* r,
                         double damping, double* out) {
    StochasticMatrix s;
    s.n = n;
    s.row_offsets.assign(row_offsets, row_offsets + n + 1);
    s.cols.assign(cols, cols + nnz);
    s.values.assign(values, values + nnz);
    RankVector rv;
    rv.values.assign(r, r + n);
    auto o = pagerank_step(rv, s, damping);
    std::memcpy(out, o.values.data(), sizeof(double) * n);
    return o.norm1;
}

// init_rank (src/kernel3_pagerank.cpp:29-39); returns norm1.
double ref_init_rank(std::int64_t n, std::uint64_t seed, double* r) {
    auto rv = init_rank(n, seed);
    std::memcpy(r, rv.values.data(), sizeof(double) * n);
    return rv.norm1;
}

// Full-size pipeline digests (tests/golden/make_digests.py): runs the
// reference's K0 -> K1 core -> K2 steps -> run_kernel3 at one BASELINE config
// on the lean memory path (each stage's input freed before the next stage's
// output is materialised: S=26 peaks at ~35 GB) and hands every output array to
// `emit` (called one or more times per name, in order: the caller hashes the
// chunks). Arrays and their byte forms:
//   "k1"        int64 (u,v) pairs: std::sort by u (kernel1_sort.cpp:66), ties
//               then re-sorted by v (tests/helpers.hpp:29-34 canonicalizer)
//   "d_in"      int64[n]   in_degree (kernel2_filter.cpp:101-106), pre-zeroing
//   "row_offsets" int64[n+1], "cols" int64[nnz_f] (0-based), "values" f64[nnz_f]
//               row_normalize(zero_columns(build_adjacency(...))) (:12-152)
//   "ranks"     f64[n]     run_kernel3 (kernel3_pagerank.cpp:67-79), c=0.85,
//               `iterations`, seed=k3_seed, total_edges=m
// stats[0..3] = nnz_raw, nnz_f, max d_in, norm1. Returns 0, or -1 on error.
typedef void (*ref_emit_fn)(const char* name, const void* data, std::int64_t bytes);

int ref_digest_pipeline(int scale, std::uint64_t seed, const double* init, int threads,
                        std::uint64_t k3_seed, int iterations, ref_emit_fn emit, double* stats) {
    try {
        const std::int64_t n = std::int64_t{1} << scale;
        const std::int64_t m = 16 * n;
        auto emit_chunks = [&](const char* name, const void* p, std::int64_t bytes) {
            const std::int64_t chunk = std::int64_t{256} << 20;
            const auto* b = static_cast<const char*>(p);
            if (bytes == 0) emit(name, b, 0);
            for (std::int64_t o = 0; o < bytes; o += chunk) emit(name, b + o, std::min(chunk, bytes - o));
        };
        std::vector<Edge> edges(static_cast<std::size_t>(m));
        if (ref_generate(scale, seed, init, 1, threads, reinterpret_cast<std::int64_t*>(edges.data())) != 0)
            return -1;
        std::sort(edges.begin(), edges.end(), [](const Edge& a, const Edge& b) { return a.u < b.u; });
        for (std::size_t i = 0; i < edges.size();) {
            std::size_t j = i + 1;
            while (j < edges.size() && edges[j].u == edges[i].u) ++j;
            std::sort(edges.begin() + i, edges.begin() + j, [](const Edge& a, const Edge& b) { return a.v < b.v; });
            i = j;
        }
        emit_chunks("k1", edges.data(), m * 16);
        CountMatrix a = build_adjacency(std::span<const Edge>(edges.data(), edges.size()), n);
        std::vector<Edge>().swap(edges);
        const std::vector<std::int64_t> din = in_degree(a);
        emit_chunks("d_in", din.data(), n * 8);
        stats[0] = static_cast<double>(a.nnz());
        stats[2] = static_cast<double>(std::max<std::int64_t>(0, *std::max_element(din.begin(), din.end())));
        CountMatrix f = zero_columns(a, din);
        a = CountMatrix{};
        StochasticMatrix s = row_normalize(f);
        f = CountMatrix{};
        stats[1] = static_cast<double>(s.nnz());
        emit_chunks("row_offsets", s.row_offsets.data(), (n + 1) * 8);
        emit_chunks("cols", s.cols.data(), s.nnz() * 8);
        emit_chunks("values", s.values.data(), s.nnz() * 8);
        PageRankConfig c;
        c.damping = 0.85;
        c.iterations = iterations;
        c.seed = k3_seed;
        auto res = run_kernel3(s, c, m);
        emit_chunks("ranks", res.ranks.values.data(), n * 8);
        stats[3] = res.ranks.norm1;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// read_edges (src/edge_io.cpp:288-295) on a manifest directory, and the
// streaming EdgeFileReader (:198-262) on one shard with a given buffer size —
// for comparing the drop-in's accepted inputs and error messages. Return the
// edge count (pairs copied while < cap), or -1 (message: ref_last_error;
// *parse_line = the ParseError line, 0 for a plain Error).
std::int64_t ref_read_edges(const char* dir, std::int64_t* uv, std::int64_t cap, std::int64_t* parse_line) {
    *parse_line = 0;
    try {
        const auto e = read_edges(EdgeManifest::load(dir));
        const auto n = static_cast<std::int64_t>(e.size());
        std::memcpy(uv, e.data(), sizeof(Edge) * static_cast<std::size_t>(std::min(n, cap)));
        return n;
    } catch (const ParseError& e) {
        g_err = e.what();
        *parse_line = e.line;
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

std::int64_t ref_stream_file(const char* path, std::int64_t max_label, std::int64_t buffer_bytes, std::int64_t* uv,
                             std::int64_t cap, std::int64_t* parse_line) {
    *parse_line = 0;
    std::int64_t n = 0;
    try {
        EdgeFileReader r(path, max_label, static_cast<std::size_t>(buffer_bytes));
        Edge e;
        while (r.next(e)) {
            if (n < cap) std::memcpy(uv + 2 * n, &e, sizeof(Edge));
            ++n;
        }
        return n;
    } catch (const ParseError& e) {
        g_err = e.what();
        *parse_line = e.line;
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// write_edges (src/edge_io.cpp:191-196) — shard and manifest bytes for the
// drop-in's edge I/O comparison.
int ref_write_edges(const std::int64_t* uv, std::int64_t m, const char* dir, int num_files, int scale,
                    int sorted) {
    try {
        std::span<const Edge> e(reinterpret_cast<const Edge*>(uv), static_cast<std::size_t>(m));
        write_edges(e, dir, num_files, scale, sorted != 0);
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

}  // extern "C"
