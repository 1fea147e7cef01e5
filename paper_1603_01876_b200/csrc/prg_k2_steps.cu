// prg_k2_steps.cu — the reference's K2 step functions one by one, on the device.
//
// The fused K2 (prg_k2.cu) is the timed path. These back the drop-in step API
// (include/prpipe/kernel2_filter.hpp:46-54: in_degree, zero_columns,
// row_normalize) on CountMatrix arrays in the reference's int64 layout.
// One warp per row; every output is exactly what the reference computes.
#include "prg_internal.cuh"

namespace prg {

namespace {

// in_degree (kernel2_filter.cpp:101-106): d_in[col] += count.
__global__ void in_degree_kernel(int64_t nnz, const int64_t* __restrict__ cols, const int64_t* __restrict__ counts,
                                 unsigned long long* __restrict__ d_in) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&d_in[cols[k]], (unsigned long long)counts[k]);
}

__global__ void max_kernel(const int64_t* __restrict__ d, int64_t n, unsigned long long* __restrict__ mx) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned long long)max(d[i], (int64_t)0));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (dev::lane_id() == 0) atomicMax(mx, m);
}

// zero_columns pass 1 (kernel2_filter.cpp:108-132): kept entries per row.
__global__ void zc_count_kernel(int64_t n, const int64_t* __restrict__ ro, const int64_t* __restrict__ cols,
                                const int64_t* __restrict__ d_in, const unsigned long long* __restrict__ mxp,
                                uint32_t* __restrict__ kept) {
    const int64_t mx = (int64_t)*mxp;
    const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; r < n; r += nw) {
        uint32_t c = 0;
        for (int64_t k = ro[r] + dev::lane_id(); k < ro[r + 1]; k += 32) {
            const int64_t d = d_in[cols[k]];
            c += (d != mx && d != 1);
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (dev::lane_id() == 0) kept[r] = c;
    }
}

// zero_columns pass 2: ordered compaction within each row (ballot prefix).
__global__ void zc_emit_kernel(int64_t n, const int64_t* __restrict__ ro, const int64_t* __restrict__ cols,
                               const int64_t* __restrict__ counts, const int64_t* __restrict__ d_in,
                               const unsigned long long* __restrict__ mxp, const uint64_t* __restrict__ out_ro,
                               int64_t* __restrict__ out_cols, int64_t* __restrict__ out_counts) {
    const int64_t mx = (int64_t)*mxp;
    const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
    const unsigned lane = dev::lane_id();
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; r < n; r += nw) {
        uint64_t pos = out_ro[r];
        for (int64_t k0 = ro[r]; k0 < ro[r + 1]; k0 += 32) {
            const int64_t k = k0 + lane;
            bool keep = false;
            if (k < ro[r + 1]) {
                const int64_t d = d_in[cols[k]];
                keep = d != mx && d != 1;
            }
            const uint32_t b = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint64_t p = pos + __popc(b & ((1u << lane) - 1u));
                out_cols[p] = cols[k];
                out_counts[p] = counts[k];
            }
            pos += __popc(b);
        }
    }
}

// row_normalize (kernel2_filter.cpp:134-152): value = count / row sum.
__global__ void rn_kernel(int64_t n, const int64_t* __restrict__ ro, const int64_t* __restrict__ counts,
                          double* __restrict__ values) {
    const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; r < n; r += nw) {
        int64_t sum = 0;
        for (int64_t k = ro[r] + dev::lane_id(); k < ro[r + 1]; k += 32) sum += counts[k];
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (sum == 0) continue;
        for (int64_t k = ro[r] + dev::lane_id(); k < ro[r + 1]; k += 32)
            values[k] = (double)counts[k] / (double)sum;
    }
}

__global__ void widen_offsets(const uint64_t* __restrict__ in, int64_t n1, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

}  // namespace

void k2_in_degree_device(int64_t n, int64_t nnz, const int64_t* cols, const int64_t* counts, int64_t* d_in,
                         cudaStream_t s) {
    PRG_CUDA(cudaMemsetAsync(d_in, 0, (size_t)n * 8, s));
    if (!nnz) return;
    in_degree_kernel<<<(unsigned)num_sms() * 8, 256, 0, s>>>(nnz, cols, counts,
                                                              reinterpret_cast<unsigned long long*>(d_in));
    PRG_LAUNCH_CHECK();
}

int64_t k2_zero_columns_device(int64_t n, const int64_t* row_offsets, const int64_t* cols, const int64_t* counts,
                               const int64_t* d_in, int64_t* out_offsets, int64_t* out_cols, int64_t* out_counts,
                               cudaStream_t s) {
    DevBuf<unsigned long long> mx(1, s);
    PRG_CUDA(cudaMemsetAsync(mx.get(), 0, 8, s));
    max_kernel<<<(unsigned)num_sms() * 4, 256, 0, s>>>(d_in, n, mx.get());
    PRG_LAUNCH_CHECK();
    DevBuf<uint32_t> kept((size_t)n, s);
    DevBuf<uint64_t> ro64((size_t)n + 1, s);
    zc_count_kernel<<<(unsigned)num_sms() * 8, 256, 0, s>>>(n, row_offsets, cols, d_in, mx.get(), kept.get());
    PRG_LAUNCH_CHECK();
    exclusive_scan_u32_to_u64(kept.get(), ro64.get(), (size_t)n, ro64.get() + n, s);
    zc_emit_kernel<<<(unsigned)num_sms() * 8, 256, 0, s>>>(n, row_offsets, cols, counts, d_in, mx.get(), ro64.get(),
                                                            out_cols, out_counts);
    PRG_LAUNCH_CHECK();
    widen_offsets<<<(unsigned)num_sms() * 4, 256, 0, s>>>(ro64.get(), n + 1, out_offsets);
    PRG_LAUNCH_CHECK();
    uint64_t nz = 0;
    PRG_CUDA(cudaMemcpyAsync(&nz, ro64.get() + n, 8, cudaMemcpyDeviceToHost, s));
    PRG_CUDA(cudaStreamSynchronize(s));
    return (int64_t)nz;
}

void k2_row_normalize_device(int64_t n, const int64_t* row_offsets, const int64_t* counts, double* values,
                             cudaStream_t s) {
    rn_kernel<<<(unsigned)num_sms() * 8, 256, 0, s>>>(n, row_offsets, counts, values);
    PRG_LAUNCH_CHECK();
}

}  // namespace prg

PRG_CHECK_QUERY(k2steps)
