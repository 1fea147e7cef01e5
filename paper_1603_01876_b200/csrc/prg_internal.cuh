// prg_internal.cuh — declarations shared by the K1/K2/K3 translation units and
// the C-ABI layer (prg_capi.cu).
#pragma once

#include "prg_common.cuh"
#include "../../include/prg.h"

namespace prg {
struct K3Plan;  // K3's column layout (prg_k3.cu)
void k3_plan_destroy(K3Plan* p);
}  // namespace prg

// The C-ABI handle (include/prg.h declares it opaque).
struct prg_matrix {
    int64_t n = 0;
    uint64_t nnz = 0;       // stored entries (after the K2 filter)
    uint64_t nnz_raw = 0;   // unique (u,v) entries before the filter (K2 only)
    uint64_t max_in = 0;    // max pre-filter in-degree (K2 only)
    uint64_t cap = 0;       // capacity of cols/values
    uint32_t* row_offsets = nullptr;  // [n+1], u32 (nnz < 2^32)
    uint32_t* cols = nullptr;         // [cap], 0-based
    double* values = nullptr;         // [cap]
    uint32_t* d_in = nullptr;         // [n] pre-filter in-degree (null when uploaded)
    // Column-major layout K3 iterates over (renumbered rows, sliced-ELL CSC over
    // virtual columns), built by prg_matrix_build_csc — in the pipeline that is
    // K2's CSC build (north_star). Owned; null until built.
    prg::K3Plan* plan = nullptr;
    ~prg_matrix();
};

namespace prg {

// Checked builds: failed PRG_DCHECKs per translation unit (read and reset).
uint32_t check_failures_runtime();
uint32_t check_failures_sort();
uint32_t check_failures_k0();
uint32_t check_failures_k1();
uint32_t check_failures_k2();
uint32_t check_failures_k3();
uint32_t check_failures_k2steps();
uint32_t check_failures_capi();

// K1 (prg_k1.cu): sort M int64 (u,v) pairs by (u,v). d_err receives DeviceErr bits.
void k1_sort_device(const int64_t* d_uv_in, int64_t m, int scale, int64_t* d_uv_out,
                    uint32_t* d_err, cudaStream_t s);

// K2 (prg_k2.cu): fused build_adjacency + in_degree + zero_columns +
// row_normalize over a device edge list sorted by start vertex. Returns a
// DeviceErr mask (0 on success); fills *out.
// filter=false, normalize=false gives build_adjacency's CountMatrix (values
// hold the exact integer counts).
uint32_t k2_filter_device(const int64_t* d_uv, int64_t m, int64_t n, prg_matrix* out,
                          cudaStream_t s, bool filter = true, bool normalize = true);

// K2 step-level functions over int64 device arrays (prg_k2_steps.cu).
void k2_in_degree_device(int64_t n, int64_t nnz, const int64_t* cols, const int64_t* counts, int64_t* d_in,
                         cudaStream_t s);
int64_t k2_zero_columns_device(int64_t n, const int64_t* row_offsets, const int64_t* cols, const int64_t* counts,
                               const int64_t* d_in, int64_t* out_offsets, int64_t* out_cols, int64_t* out_counts,
                               cudaStream_t s);
void k2_row_normalize_device(int64_t n, const int64_t* row_offsets, const int64_t* counts, double* values,
                             cudaStream_t s);

// K3 (prg_k3.cu).
struct K3Options {
    double damping = 0.85;
    int iterations = 20;
    uint64_t seed = 0;
    int mode = 0;  // 0 = timed (deterministic tree sums), 1 = parity (reference order),
                   // 2 = parity order with Neumaier sums (drift attribution)
};
// Full run_kernel3 semantics: init_rank + iterations steps. d_ranks [n] in the
// original vertex order; returns norm1 (sum of the final vector).
double k3_pagerank_device(const prg_matrix* a, const K3Options& opt, double* d_ranks,
                          cudaStream_t s);
// Column-sharded K3 over `world` GPUs (one process each): this rank's SpMV
// covers its SELL slice range; allreduce(user, buf, count, stream) must sum
// buf over the ranks in place, ordered on `stream`. Bit-identical to
// k3_pagerank_device mode 0 on every rank.
double k3_pagerank_sharded_device(const prg_matrix* a, const K3Options& opt, int rank, int world,
                                  prg_allreduce_f64 allreduce, void* user, double* d_ranks, cudaStream_t s);
// The slice ranges (bounds[world + 1]) the sharded K3 uses.
void k3_shard_bounds(const prg_matrix* a, int world, uint32_t* bounds, cudaStream_t s);
void k3_shard_bounds_host(const uint32_t* slice_ptr, uint32_t nslices, int world, uint32_t* bounds);
// One pagerank_step (kernel3_pagerank.cpp:41-65): d_out = step(d_r). Returns norm1.
double k3_step_device(const prg_matrix* a, const double* d_r, double damping, double* d_out,
                      int mode, cudaStream_t s);
// run_to_convergence (kernel3_pagerank.cpp:86-115); returns iterations applied.
int k3_converge_device(const prg_matrix* a, double damping, double tol, int max_iters, const double* d_start,
                       double* d_out, bool* converged, cudaStream_t s);
// K2's CSC build: K3's timed-mode column layout, kept on the handle (replaces any
// earlier one). K3 calls on a handle without it build a temporary layout inside
// their own timed region.
void k3_build_csc_device(prg_matrix* a, cudaStream_t s);
// init_rank (kernel3_pagerank.cpp:29-39) on the device; returns norm1.
double k3_init_rank_device(int64_t n, uint64_t seed, double* d_r, int mode, cudaStream_t s);

// K0 (prg_k0.cu): device edge generator; labels = Fisher-Yates table (device, n entries) or null.
void k0_generate_device(int scale, int64_t edge_factor, uint64_t seed, const double init[4],
                        const int64_t* d_labels, int64_t first, int64_t count, int64_t* d_uv,
                        cudaStream_t s);

}  // namespace prg
