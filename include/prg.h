/*
 * prg.h — C-ABI of the B200-native PageRank-pipeline hot path (K1 sort, K2
 * filter, K3 PageRank). Plain pointers and sizes; no C++ or torch types.
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/proj); the C++ shim in paper_1603_01876_b200/host re-exposes
 * the reference's exact prpipe:: signatures and pybind11 module on top of it.
 *
 * Conventions
 *   - Status codes replace the reference's exceptions (include/prpipe/types.hpp:17-28):
 *     PRG_OK (0) or a negative PRG_ERR_*; prg_last_error() has the message
 *     (thread-local). The shim turns them back into prpipe::Error.
 *   - "_device" entry points take device pointers and a cudaStream_t passed as
 *     void*; they are stream-ordered and may synchronise the stream at the end
 *     to report input errors and output sizes.
 *   - "_host" entry points take host buffers; H2D, kernels and D2H happen inside.
 *   - Edges are the reference's Edge {int64 u, v} (types.hpp:10-15), 1-based,
 *     stored interleaved: uv[2*i] = u, uv[2*i+1] = v.
 *   - A prg_matrix is an opaque device-resident row-stochastic CSR
 *     (u32 row offsets and columns, f64 values), the device form of the
 *     reference's StochasticMatrix (kernel2_filter.hpp:28-38).
 */
#ifndef PRG_H_
#define PRG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t prg_status;
#define PRG_OK 0
#define PRG_ERR_INVALID_ARGUMENT (-1) /* bad sizes / config (e.g. PageRankConfig::validate) */
#define PRG_ERR_LABEL_RANGE (-2)      /* vertex label outside [1, N] (kernel2_filter.cpp:41-43) */
#define PRG_ERR_UNSORTED (-3)         /* K2 input not sorted by start vertex (kernel2_filter.cpp:45-47) */
#define PRG_ERR_CUDA (-4)             /* CUDA runtime failure or no device */
#define PRG_ERR_INTERNAL (-5)

typedef struct prg_matrix prg_matrix;

/* Library info / error channel. */
const char* prg_last_error(void);
const char* prg_version(void);
int32_t prg_device_count(void);

/* Instrumentation (no reference counterpart; the reference times with
 * prpipe::Timer, include/prpipe/timer.hpp:9-19). prg_launch_count: kernels the
 * library has launched since load. prg_profile_*: CUDA-event timing of named
 * regions (k1_sort, k2_filter, k3_spmv, ...) on the stream they ran on;
 * report writes JSON {"name": [count, total_ms]} and returns its length. */
int64_t prg_launch_count(void);
/* Checked builds only (-DPRG_CHECKED=1; release builds return 0): failed
 * device-side bounds / invariant checks since the last call (then reset). */
int64_t prg_debug_check_failures(void);

/* Bytes the last prg_k3_pagerank_host call moved host -> device: its CSR
 * structure plus, instead of the f64 values, one base value per row and the
 * entries that differ from it (classified on host threads while the column
 * indices are in flight). Diagnostics for the bench's e2e record. */
int64_t prg_last_h2d_bytes(void);
void prg_profile_enable(int32_t on);
/* Device memory: the library allocates from its own stream-ordered pool
 * (freed blocks stay cached between calls); prg_trim_memory waits for the
 * device and returns every unused pooled byte to the driver. */
prg_status prg_trim_memory(void);
int64_t prg_profile_report(char* buf, int64_t cap, int32_t reset);

/* ---- K0 (input generation; untimed) ------------------------------------
 * Device restatement of EdgeGenerator::make_edge (src/graph_gen.cpp:83-99):
 * edges [first, first+count) of the K0 list for (scale, seed, initiator).
 * d_labels: the Fisher–Yates label table (graph_gen.cpp:66-76, 2^scale int64,
 * device) or NULL for permute_labels=false. prg_k0_permutation fills it on
 * the host (the shuffle is inherently sequential). */
prg_status prg_k0_permutation(int32_t scale, uint64_t seed, int64_t* labels_host);
prg_status prg_k0_generate_device(int32_t scale, int64_t edge_factor, uint64_t seed,
                                  const double initiator[4], const int64_t* d_labels,
                                  int64_t first, int64_t count, int64_t* d_uv, void* stream);

/* ---- K1 — replaces the core of prpipe::sort_edges --------------------------
 * include/prpipe/kernel1_sort.hpp:24-25; src/kernel1_sort.cpp:63-68
 * (std::sort by start vertex). Output is ordered by (u, v): a valid start-vertex
 * order with canonical ties (tests/helpers.hpp:29-34). d_uv_in and d_uv_out
 * must not alias. Labels must lie in [1, 2^scale] (else PRG_ERR_LABEL_RANGE). */
prg_status prg_k1_sort_device(const int64_t* d_uv_in, int64_t m, int32_t scale, int64_t* d_uv_out,
                              void* stream);
prg_status prg_k1_sort_host(const int64_t* uv_in, int64_t m, int32_t scale, int64_t* uv_out);

/* K1 under a host-memory budget — the B200 form of sort_edges' out-of-core
 * path (src/kernel1_sort.cpp:133-149, 70-122: external merge sort when the
 * list exceeds memory_budget_bytes / 16). The whole list lives in HBM; the host
 * holds one pinned chunk of chunk_edges edges: `source` fills it (returns the
 * edges written, 1..max_edges) until m edges arrived, the device sorts, and
 * `sink` receives the sorted list chunk by chunk (returns 0, else the call
 * fails). Same output as prg_k1_sort_host. Lists beyond 2^32-1 edges or the
 * free device memory are refused with PRG_ERR_INVALID_ARGUMENT. */
typedef int64_t (*prg_edge_source)(void* user, int64_t* uv, int64_t max_edges);
typedef int32_t (*prg_edge_sink)(void* user, const int64_t* uv, int64_t count);
prg_status prg_k1_sort_streamed(prg_edge_source source, prg_edge_sink sink, void* user, int64_t m, int32_t scale,
                                int64_t chunk_edges);

/* ---- K2 — replaces run_kernel2's core -------------------------------------
 * build_adjacency + in_degree + zero_columns + row_normalize
 * (include/prpipe/kernel2_filter.hpp:42-65; src/kernel2_filter.cpp:12-168).
 * Input sorted by start vertex (ties in any order). n = vertex count. */
prg_status prg_k2_filter_device(const int64_t* d_uv_sorted, int64_t m, int64_t n, prg_matrix** out,
                                void* stream);
prg_status prg_k2_filter_host(const int64_t* uv_sorted, int64_t m, int64_t n, prg_matrix** out);

/* K2 step-level entry points on the reference's CountMatrix layout (host
 * int64 arrays; computed on the device). build_adjacency (kernel2_filter.hpp:42-43,
 * kernel2_filter.cpp:12-54): row_offsets[n+1], cols/counts[m] (nnz <= m) ->
 * *nnz. in_degree (:46, :101-106). zero_columns (:51, :108-132): outputs sized
 * like the input. row_normalize (:54, :134-152): values[nnz]. */
prg_status prg_build_adjacency_host(const int64_t* uv_sorted, int64_t m, int64_t n, int64_t* row_offsets,
                                    int64_t* cols, int64_t* counts, int64_t* nnz);
prg_status prg_in_degree_host(int64_t n, int64_t nnz, const int64_t* cols, const int64_t* counts,
                              int64_t* d_in);
prg_status prg_zero_columns_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                 const int64_t* counts, const int64_t* d_in, int64_t* out_row_offsets,
                                 int64_t* out_cols, int64_t* out_counts, int64_t* out_nnz);
prg_status prg_row_normalize_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* counts,
                                  double* values);

/* Matrix handle. */
prg_status prg_matrix_info(const prg_matrix* a, int64_t* n, int64_t* nnz, int64_t* nnz_raw,
                           int64_t* max_in_degree);
/* Copies to host int64/f64 arrays (row_offsets[n+1], cols[nnz], values[nnz],
 * d_in[n]); any pointer may be NULL. d_in is the pre-filter in-degree
 * (in_degree(), kernel2_filter.cpp:101-106); zeros for uploaded matrices. */
prg_status prg_matrix_download(const prg_matrix* a, int64_t* row_offsets, int64_t* cols,
                               double* values, int64_t* d_in);
/* Device views (u32 offsets/cols, f64 values, u32 d_in; d_in may be NULL). */
prg_status prg_matrix_device_arrays(const prg_matrix* a, const uint32_t** row_offsets,
                                    const uint32_t** cols, const double** values,
                                    const uint32_t** d_in);
/* Uploads a host StochasticMatrix (int64 offsets/cols, f64 values). */
prg_status prg_matrix_from_host(int64_t n, int64_t nnz, const int64_t* row_offsets,
                                const int64_t* cols, const double* values, prg_matrix** out);
void prg_matrix_destroy(prg_matrix* a);
/* K2's CSC build (north_star: "a scan-based CSR/CSC build"; SURVEY §8(b) device
 * residency across the K2 -> K3 handoff). Builds, on the handle, the column-major
 * layout K3 iterates over — rows renumbered by out-degree class, the CSR
 * transposed by a stable column sort, sliced-ELL over virtual columns — so that
 * run_kernel3 / pagerank_step / run_to_convergence on this handle start from a
 * CSC, as the reference's K3 starts from its CSR (kernel3_pagerank.cpp:67-79).
 * K3 calls on a handle without it build a temporary layout inside their own
 * timed region. drop_csc releases it; has_csc returns 1 when present.
 * A handle carrying the layout must not be used by two streams at once (K3
 * keeps per-launch counters in it). */
prg_status prg_matrix_build_csc(prg_matrix* a, void* stream);
prg_status prg_matrix_drop_csc(prg_matrix* a);
int32_t prg_matrix_has_csc(const prg_matrix* a);

/* ---- K3 — replaces init_rank / pagerank_step / run_kernel3 ----------------
 * include/prpipe/kernel3_pagerank.hpp:28-44; src/kernel3_pagerank.cpp:29-79.
 * mode 0: timed path (deterministic tree sums; within 1e-10 relative L1 of
 *         the reference, the gap being the reference's own sequential-sum
 *         rounding, kernel3_pagerank.cpp:17-19);
 * mode 1: parity path — reference evaluation order (ascending-u column sums,
 *         separate mul/add, sequential sums); bit-identical to the reference.
 * Ranks are written in the original vertex order; *norm1 = sum of the ranks. */
prg_status prg_k3_pagerank_device(const prg_matrix* a, double damping, int32_t iterations,
                                  uint64_t seed, int32_t mode, double* d_ranks, double* norm1,
                                  void* stream);
prg_status prg_k3_pagerank_host(int64_t n, int64_t nnz, const int64_t* row_offsets,
                                const int64_t* cols, const double* values, double damping,
                                int32_t iterations, uint64_t seed, int32_t mode, double* ranks,
                                double* norm1);
prg_status prg_init_rank_device(int64_t n, uint64_t seed, int32_t mode, double* d_r, double* norm1,
                                void* stream);
prg_status prg_pagerank_step_device(const prg_matrix* a, const double* d_r, double damping,
                                    int32_t mode, double* d_out, double* norm1, void* stream);

/* ---- Multi-GPU K3 ----------------------
 * Column-sharded run_kernel3, one process per GPU, every rank holding the
 * matrix handle (K2 replicated). Rank r runs the SpMV over its contiguous range
 * of SELL slices (balanced by entries); after each SpMV the ranks' iterate
 * values, split-column part sums and slice sums are combined by `allreduce`,
 * which the caller implements (NCCL all_reduce over NVLink; it must sum the
 * `count` doubles at `d_buf` over all ranks in place, ordered on `stream`, and
 * return 0). Each element has one writer, so the sum is exact and every rank
 * ends with ranks/norm1 bit-identical to prg_k3_pagerank_device mode 0.
 * prg_k3_shard_bounds gives the slice ranges (bounds[world + 1]). */
typedef int32_t (*prg_allreduce_f64)(void* user, double* d_buf, int64_t count, void* stream);
prg_status prg_k3_pagerank_sharded(const prg_matrix* a, double damping, int32_t iterations, uint64_t seed,
                                   int32_t rank, int32_t world, prg_allreduce_f64 allreduce, void* user,
                                   double* d_ranks, double* norm1, void* stream);
prg_status prg_k3_shard_bounds(const prg_matrix* a, int32_t world, uint32_t* bounds, void* stream);
/* The partition rule itself, on host data (no device needed): slice_ptr[nslices + 1]
 * holds the slices' entry offsets; bounds[r] = first slice of rank r. */
prg_status prg_shard_bounds_host(const uint32_t* slice_ptr, uint32_t nslices, int32_t world, uint32_t* bounds);

/* Host-buffer variants used by the drop-in C++ shim (prpipe::init_rank,
 * pagerank_step, run_kernel3 on a K2-produced handle, run_to_convergence). */
prg_status prg_init_rank_host(int64_t n, uint64_t seed, int32_t mode, double* r, double* norm1);
prg_status prg_pagerank_step_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                  const double* values, const double* r, double damping, int32_t mode,
                                  double* out, double* norm1);
prg_status prg_k3_pagerank_matrix_host(const prg_matrix* a, double damping, int32_t iterations, uint64_t seed,
                                       int32_t mode, double* ranks, double* norm1);
prg_status prg_run_to_convergence_host(int64_t n, int64_t nnz, const int64_t* row_offsets, const int64_t* cols,
                                       const double* values, double damping, double tol, int32_t max_iters,
                                       const double* start, double* out, int32_t* converged,
                                       int32_t* iterations);

#ifdef __cplusplus
}
#endif
#endif /* PRG_H_ */
