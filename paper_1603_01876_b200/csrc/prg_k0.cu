// prg_k0.cu — device K0 edge generator (input preparation, untimed).
//
// Restates EdgeGenerator::make_edge (src/graph_gen.cpp:83-99): every edge is a
// pure function of (seed, edge index) — S R-MAT levels, each drawing one
// next_unit() from SplitMix64(mix_seed(seed, edge_index)) — followed by the
// label permutation lookup. The permutation table itself (graph_gen.cpp:66-76)
// is a sequential Fisher–Yates shuffle and is built on the host
// (prg_k0_permutation). Bit-identical to the reference (tests/test_k0.py).
#include "prg_internal.cuh"

namespace prg {

namespace {

__global__ void k0_kernel(int scale, uint64_t seed, double a, double ab, double abc,
                          const int64_t* __restrict__ labels, int64_t first, int64_t count,
                          longlong2* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t s0 = dev::mix_seed(seed, (uint64_t)(first + k));
        int64_t u = 0, v = 0;
        for (int level = 0; level < scale; ++level) {
            const double x = (double)(dev::splitmix_at(s0, (uint64_t)level + 1) >> 11) * 0x1.0p-53;
            const int q = x < a ? 0 : x < ab ? 1 : x < abc ? 2 : 3;
            u = (u << 1) | (q >> 1);
            v = (v << 1) | (q & 1);
        }
        out[k] = labels ? make_longlong2(labels[u], labels[v]) : make_longlong2(u + 1, v + 1);
    }
}

}  // namespace

void k0_generate_device(int scale, int64_t /*edge_factor*/, uint64_t seed, const double init[4],
                        const int64_t* d_labels, int64_t first, int64_t count, int64_t* d_uv,
                        cudaStream_t s) {
    if (count <= 0) return;
    const double a = init[0];
    const double ab = a + init[1];
    const double abc = ab + init[2];
    k0_kernel<<<(unsigned)num_sms() * 8, 256, 0, s>>>(scale, seed, a, ab, abc, d_labels, first, count,
                                                      reinterpret_cast<longlong2*>(d_uv));
    PRG_LAUNCH_CHECK();
}

}  // namespace prg

PRG_CHECK_QUERY(k0)
