// prg_common.cuh — shared device/host helpers for the B200 K1/K2/K3 kernels.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

namespace prg {

constexpr int kWarp = 32;
constexpr int kNumSMsB200 = 148;

// Host-side error channel: every C-ABI entry point funnels failures through
// set_error() so prg_last_error() can report them (SURVEY §5 failure detection).
void set_error(const std::string& msg);
const std::string& last_error();

struct CudaError {
    std::string msg;
};

#define PRG_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::prg::CudaError{std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                   " (" __FILE__ ":" + std::to_string(__LINE__) + ")"}; \
    } while (0)

// Every launch site goes through PRG_LAUNCH_CHECK, which also counts launches
// (prg_launch_count(): bench.py's "gpu_launches").
void count_launch();
#define PRG_LAUNCH_CHECK()         \
    do {                           \
        ::prg::count_launch();     \
        PRG_CUDA(cudaGetLastError()); \
    } while (0)

// Optional CUDA-event timing of named regions on their stream (prg_profile_*).
// Costs two event records per scope when enabled, nothing otherwise.
bool profiling_enabled();
void profiling_enable(bool on);
long long launch_count();
std::string profile_report(bool reset);  // {"name": [count, total_ms], ...}
struct ProfScope {
    std::string name;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(std::string n, cudaStream_t st);
    ~ProfScope();
};

__host__ __device__ inline unsigned div_up(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

int num_sms();

// Stream-ordered scratch allocation (cudaMallocAsync on the device's default
// pool, whose release threshold the library raises to "keep everything").
void* ws_alloc(size_t bytes, cudaStream_t s);
void ws_free(void* p, cudaStream_t s);
void ws_trim();  // return the library pool's unused memory to the driver

// Large host <-> device copies through pinned slots and host worker threads
// (pageable host memory on the host side). Both return when the copy is done.
void copy_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s);
void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t s);

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t count, cudaStream_t stream) : n(count), s(stream) {
        p = static_cast<T*>(ws_alloc(count ? count * sizeof(T) : sizeof(T), stream));
    }
    ~DevBuf() { if (p) ws_free(p, s); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            if (p) ws_free(p, s);
            p = o.p; n = o.n; s = o.s; o.p = nullptr;
        }
        return *this;
    }
    T* get() const { return p; }
    T* release() { T* q = p; p = nullptr; return q; }
};

// Device-wide exclusive scan of u32 counts into u32/u64 offsets (decoupled
// look-back, one pass). `total` (device scalar, may be null) receives the sum.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total,
                        cudaStream_t s);
void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, size_t n, uint64_t* total,
                               cudaStream_t s);
// Exclusive scan of the used prefix in[0, min(cap, *d_count * mult)) of a
// capacity-sized buffer (the count lives on the device; no host sync).
void exclusive_scan_u32_prefix(const uint32_t* in, uint32_t* out, size_t cap, const uint32_t* d_count,
                               uint32_t mult, cudaStream_t s);

// Device error word: kernels that validate input OR a code in; the host reads it
// back at the end of an entry point (one sync) and turns it into a status.
enum DeviceErr : uint32_t {
    kErrNone = 0,
    kErrLabelRange = 1u << 0,   // vertex label outside [1, N]
    kErrUnsorted = 1u << 1,     // K2 input not sorted by start vertex
    kErrNotCanonical = 1u << 2, // informational: ties not v-ordered (K2 re-sorts)
    kErrOverflow = 1u << 3,     // an internal capacity was exceeded
};

}  // namespace prg

// ----------------------------------------------------------------------------
// Device helpers
// ----------------------------------------------------------------------------
namespace prg::dev {

// Checked builds (-DPRG_CHECKED=1: build/libprg_checked.so, tests/test_checked.py):
// bounds and invariant checks on the index-computing and lock-free paths (sort
// scatters, local-stage slots, K2 output slots, K3 gathers). Compute-sanitizer
// is closed on this GPU pool, so these stand in for memcheck. A failed check
// counts into this translation unit's g_check_fail; prg_debug_check_failures()
// sums and resets the counters of every unit. Release builds compile them out.
#ifndef PRG_CHECKED
#define PRG_CHECKED 0
#endif
static __device__ unsigned int g_check_fail = 0;
#if PRG_CHECKED
#define PRG_DCHECK(cond)                                                   \
    do {                                                                   \
        if (!(cond)) atomicAdd(&::prg::dev::g_check_fail, 1u);             \
    } while (0)
#else
#define PRG_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(0xffffffffu, v, d);
        if ((int)lane_id() >= d) v += o;
    }
    return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// Deterministic fp64 warp tree sum (fixed butterfly order), separate add only.
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// Block-wide exclusive scan of one u32 per thread; returns the block total.
// `smem` needs blockDim.x/32 + 1 u32 slots.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* smem, uint32_t& total) {
    const unsigned w = warp_id(), l = lane_id(), nw = blockDim.x >> 5;
    uint32_t inc = warp_incl_scan(v);
    if (l == 31) smem[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t x = l < nw ? smem[l] : 0u;
        uint32_t xi = warp_incl_scan(x);
        if (l < nw) smem[l] = xi - x;
        if (l == nw - 1) smem[nw] = xi;
    }
    __syncthreads();
    uint32_t res = smem[w] + inc - v;
    total = smem[nw];
    __syncthreads();
    return res;
}

// Streaming (evict-first) and keep (evict-last) global loads via L2 cache-policy
// hints (sm_100 accepts the bare .L2::evict_* qualifiers only on 256-bit loads).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void* p, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_stream_u4(const void* p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
// Predicated loads (no branch): return `dflt` when !pred. Non-volatile so the
// compiler may batch them.
__device__ __forceinline__ uint32_t ld_stream_u32_pred(const void* p, bool pred, uint64_t pol, uint32_t dflt) {
    uint32_t r = dflt;
    asm("{ .reg .pred q; setp.ne.u32 q, %2, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %3; }"
        : "+r"(r)
        : "l"(p), "r"((uint32_t)pred), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_keep_f64_pred(const double* p, bool pred, uint64_t pol) {
    double r = 0.0;
    asm("{ .reg .pred q; setp.ne.u32 q, %2, 0;\n\t"
        "@q ld.global.nc.L2::cache_hint.f64 %0, [%1], %3; }"
        : "+d"(r)
        : "l"(p), "r"((uint32_t)pred), "l"(pol));
    return r;
}
// Gather with an index-dependent L1 eviction priority (measurement variants of
// the SpMV, PRG_SPMV_VARIANT=2..5): the hot head of the gather vector and its
// cold tail take different priorities. HOTP / COLDP: 0 = default, 1 = L1::evict_last,
// 2 = L1::evict_first, 3 = L1::no_allocate.
#define PRG_L1P_STR_0 ""
#define PRG_L1P_STR_1 ".L1::evict_last"
#define PRG_L1P_STR_2 ".L1::evict_first"
#define PRG_L1P_STR_3 ".L1::no_allocate"
#define PRG_L1P_STR(x) PRG_L1P_STR_##x
#define PRG_DEFINE_LD_HOTCOLD(HOTP, COLDP)                                                              \
    __device__ __forceinline__ double ld_hotcold_##HOTP##_##COLDP(const double* p, bool pred, bool hot, \
                                                                  uint64_t pol) {                       \
        double r = 0.0;                                                                                 \
        asm("{ .reg .pred q, h, c;\n\t"                                                                 \
            "setp.ne.u32 q, %2, 0;\n\t"                                                                 \
            "setp.ne.u32 h, %3, 0;\n\t"                                                                 \
            "and.pred c, q, !h;\n\t"                                                                    \
            "and.pred h, q, h;\n\t"                                                                     \
            "@h ld.global.nc" PRG_L1P_STR(HOTP) ".L2::cache_hint.f64 %0, [%1], %4;\n\t"                 \
            "@c ld.global.nc" PRG_L1P_STR(COLDP) ".L2::cache_hint.f64 %0, [%1], %4; }"                   \
            : "+d"(r)                                                                                   \
            : "l"(p), "r"((uint32_t)pred), "r"((uint32_t)hot), "l"(pol));                               \
        return r;                                                                                       \
    }
PRG_DEFINE_LD_HOTCOLD(1, 2)
PRG_DEFINE_LD_HOTCOLD(0, 2)
PRG_DEFINE_LD_HOTCOLD(1, 0)
PRG_DEFINE_LD_HOTCOLD(0, 3)
__device__ __forceinline__ double ld_f64_pred(const double* p, bool pred) {
    double r = 0.0;
    asm("{ .reg .pred q; setp.ne.u32 q, %2, 0;\n\t"
        "@q ld.global.nc.f64 %0, [%1]; }"
        : "+d"(r)
        : "l"(p), "r"((uint32_t)pred));
    return r;
}
__device__ __forceinline__ double ld_keep_f64(const double* p, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) into shared memory, completed
// on an mbarrier with a transaction count. Streaming kernels keep a ring of
// such stages so the next tile is in flight while the current one is worked on.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(a), "r"(parity)
                     : "memory");
    } while (!done);
}
// Orders this thread's earlier generic-proxy shared-memory accesses (after a
// barrier: the whole CTA's) before later async-proxy (TMA) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// bytes: multiple of 16; src and dst 16-byte aligned. L2 evict-first: the
// stream is read once.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

// splitmix64 finaliser + counter-based stream position (rng.hpp:14-19): the
// state after k calls from seed s0 is s0 + k*gamma, so x_k is a pure function.
__device__ __forceinline__ uint64_t splitmix_at(uint64_t s0, uint64_t k) {
    uint64_t z = s0 + k * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    // rng.hpp:33-37: SplitMix64 g(seed ^ (gamma*(stream+1))); g.next(); return g.next();
    uint64_t s0 = seed ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
    uint64_t z = s0 + 2 * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

}  // namespace prg::dev

// Per translation unit: read and reset its check-failure counter (0 in release builds).
#define PRG_CHECK_QUERY(tag)                                                              \
    namespace prg {                                                                       \
    uint32_t check_failures_##tag() {                                                     \
        unsigned v = 0, z = 0;                                                            \
        if (PRG_CHECKED) {                                                                \
            PRG_CUDA(cudaMemcpyFromSymbol(&v, ::prg::dev::g_check_fail, sizeof(v)));      \
            PRG_CUDA(cudaMemcpyToSymbol(::prg::dev::g_check_fail, &z, sizeof(z)));        \
        }                                                                                 \
        return v;                                                                         \
    }                                                                                     \
    }
