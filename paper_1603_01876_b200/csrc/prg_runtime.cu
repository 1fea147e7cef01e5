// prg_runtime.cu — error channel, stream-ordered workspace, device-wide scan.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "prg_common.cuh"

namespace prg {

namespace {
thread_local std::string g_last_error;
std::once_flag g_pool_once;
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

// ---- launch counter and profiling ------------------------------------------
namespace {
std::atomic<long long> g_launches{0};
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
struct ProfRec { std::string name; cudaEvent_t a, b; };
std::vector<ProfRec> g_prof_pending;
std::map<std::string, std::pair<long long, double>> g_prof_totals;
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }
bool profiling_enabled() { return g_prof.load(std::memory_order_relaxed); }
void profiling_enable(bool on) { g_prof.store(on); }

ProfScope::ProfScope(std::string n, cudaStream_t st) : name(std::move(n)), s(st) {
    if (!profiling_enabled()) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
}
ProfScope::~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_pending.push_back({name, a, b});
}

std::string profile_report(bool reset) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& p : g_prof_pending) {
        cudaEventSynchronize(p.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        auto& t = g_prof_totals[p.name];
        t.first += 1;
        t.second += ms;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_prof_pending.clear();
    std::string out = "{";
    bool first = true;
    for (auto& [k, v] : g_prof_totals) {
        if (!first) out += ", ";
        first = false;
        out += "\"" + k + "\": [" + std::to_string(v.first) + ", " + std::to_string(v.second) + "]";
    }
    out += "}";
    if (reset) g_prof_totals.clear();
    return out;
}
const std::string& last_error() { return g_last_error; }

int num_sms() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        PRG_CUDA(cudaGetDevice(&dev));
        PRG_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev));
    }
    return cached;
}

// The library allocates its device workspace from a PRIVATE stream-ordered
// pool (not the device's default pool, which other libraries share). Freed
// blocks stay cached across calls — a finite release threshold made every
// synchronising call hand memory back and re-map it on the next one (the S=24
// CSC build went 12 -> 85 ms) — and prg_trim_memory() returns everything
// unused on request.
constexpr uint64_t kPoolKeepBytes = UINT64_MAX;
cudaMemPool_t g_pool = nullptr;

cudaMemPool_t library_pool() {
    std::call_once(g_pool_once, [] {
        int dev = 0;
        PRG_CUDA(cudaGetDevice(&dev));
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        PRG_CUDA(cudaMemPoolCreate(&g_pool, &props));
        uint64_t keep = kPoolKeepBytes;
        PRG_CUDA(cudaMemPoolSetAttribute(g_pool, cudaMemPoolAttrReleaseThreshold, &keep));
    });
    return g_pool;
}

void* ws_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    PRG_CUDA(cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, library_pool(), s));
    return p;
}

void ws_trim() {
    if (g_pool) PRG_CUDA(cudaMemPoolTrimTo(g_pool, 0));
}

void ws_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// ---------------------------------------------------------------------------
// Exclusive scan: reduce-then-scan, 1024 threads x 8 items per block.
// ---------------------------------------------------------------------------
namespace {
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// dn (optional): the scan covers only the first min(n, *dn * mult) items — the
// used prefix of a capacity-sized buffer whose size is known only on the device.
__device__ __forceinline__ size_t scan_len(size_t n, const uint32_t* dn, uint32_t mult) {
    return dn ? min(n, (size_t)*dn * mult) : n;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                                   size_t n, const uint32_t* dn, uint32_t mult,
                                                                   uint64_t* __restrict__ partial) {
    __shared__ uint64_t red[32];
    n = scan_len(n, dn, mult);
    const size_t base = (size_t)blockIdx.x * kScanTile;
    if (base >= n && blockIdx.x > 0) return;
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        size_t i = base + (size_t)k * kScanThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    s = dev::warp_sum(s);
    if (dev::lane_id() == 0) red[dev::warp_id()] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint64_t v = red[threadIdx.x];
        v = dev::warp_sum(v);
        if (threadIdx.x == 0) partial[blockIdx.x] = v;
    }
}

// Single-block exclusive scan over `n` u64 values (in place); total -> *total.
__global__ void __launch_bounds__(kScanThreads) scan_partials_kernel(uint64_t* __restrict__ p,
                                                                     size_t n, const uint32_t* dn, uint32_t mult) {
    __shared__ uint64_t warp_tot[33];
    __shared__ uint64_t carry;
    if (dn) n = min(n, (scan_len(~size_t(0), dn, mult) + kScanTile - 1) / kScanTile);
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (size_t base = 0; base < n; base += kScanThreads) {
        size_t i = base + threadIdx.x;
        uint64_t v = i < n ? p[i] : 0;
        uint64_t inc = dev::warp_incl_scan(v);
        if (dev::lane_id() == 31) warp_tot[dev::warp_id()] = inc;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint64_t x = warp_tot[threadIdx.x];
            uint64_t xi = dev::warp_incl_scan(x);
            warp_tot[threadIdx.x] = xi - x;
            if (threadIdx.x == 31) warp_tot[32] = xi;
        }
        __syncthreads();
        uint64_t excl = carry + warp_tot[dev::warp_id()] + inc - v;
        if (i < n) p[i] = excl;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_tot[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) p[n] = carry;
}

template <class Out>
__global__ void __launch_bounds__(kScanThreads, 2) scan_down_kernel(const uint32_t* __restrict__ in,
                                                                 size_t n, const uint32_t* dn, uint32_t mult,
                                                                 const uint64_t* __restrict__ partial,
                                                                 Out* __restrict__ out) {
    __shared__ uint64_t warp_tot[33];
    n = scan_len(n, dn, mult);
    const size_t base = (size_t)blockIdx.x * kScanTile;
    if (base >= n) return;
    // Blocked arrangement: thread t owns items [base + t*8, base + t*8 + 8).
    uint32_t v[kScanItems];
    const size_t my = base + (size_t)threadIdx.x * kScanItems;
    // A thread's 8 items are 32 contiguous bytes: two 16-byte loads when the
    // block is whole and aligned (8 separate 4-byte loads at a 32-byte lane
    // stride cost 8 L1 wavefronts each: the kernel ran at ~1.6 TB/s).
    const bool vec = my + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        const uint4 a = reinterpret_cast<const uint4*>(in + my)[0], b = reinterpret_cast<const uint4*>(in + my)[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = (my + k < n) ? in[my + k] : 0u;
    }
    uint64_t tsum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) tsum += v[k];
    uint64_t inc = dev::warp_incl_scan(tsum);
    if (dev::lane_id() == 31) warp_tot[dev::warp_id()] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint64_t x = warp_tot[threadIdx.x];
        uint64_t xi = dev::warp_incl_scan(x);
        warp_tot[threadIdx.x] = xi - x;
    }
    __syncthreads();
    uint64_t run = partial[blockIdx.x] + warp_tot[dev::warp_id()] + inc - tsum;
    alignas(16) Out o[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        o[k] = static_cast<Out>(run);
        run += v[k];
    }
    if (vec) {
        static_assert(sizeof(Out) == 4 || sizeof(Out) == 8, "u32 or u64 output");
        uint4* d = reinterpret_cast<uint4*>(out + my);
        constexpr int kVec = kScanItems * (int)sizeof(Out) / 16;
#pragma unroll
        for (int q = 0; q < kVec; ++q) {
            uint4 w;  // byte copy: no type-punned load of the Out array
            memcpy(&w, reinterpret_cast<const char*>(o) + 16 * q, 16);
            d[q] = w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (my + k < n) out[my + k] = o[k];
    }
}

template <class Out>
__global__ void copy_total_kernel(const uint64_t* partial, size_t nb, Out* total) {
    *total = static_cast<Out>(partial[nb]);
}

// Single-pass variant (decoupled look-back): one launch per scan instead of
// reduce + partials + down (+ total). Tiles are claimed in launch order from a
// counter; each publishes its aggregate, warp 0 sums predecessors' aggregates
// back to the nearest inclusive prefix, then the tile is written. Most of the
// pipeline's ~16 scans per step are launch-latency bound.
constexpr uint64_t kScanAgg = 1ull << 62, kScanInc = 2ull << 62, kScanVal = (1ull << 62) - 1;
template <class Out>
__global__ void __launch_bounds__(kScanThreads) scan_onepass_kernel(const uint32_t* __restrict__ in, size_t n,
                                                                    const uint32_t* dn, uint32_t mult,
                                                                    unsigned long long* __restrict__ status,
                                                                    uint32_t* __restrict__ counter,
                                                                    Out* __restrict__ out, Out* __restrict__ total) {
    __shared__ uint64_t warp_tot[33];
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_excl;
    n = scan_len(n, dn, mult);
    const uint32_t ntiles = (uint32_t)((n + kScanTile - 1) / kScanTile);
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    if (t >= ntiles) {
        if (ntiles == 0 && t == 0 && total && threadIdx.x == 0) *total = 0;
        return;
    }
    const size_t base = (size_t)t * kScanTile;
    uint32_t v[kScanItems];
    const size_t my = base + (size_t)threadIdx.x * kScanItems;
    const bool vec = my + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        const uint4 a = reinterpret_cast<const uint4*>(in + my)[0], b = reinterpret_cast<const uint4*>(in + my)[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = (my + k < n) ? in[my + k] : 0u;
    }
    uint64_t tsum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) tsum += v[k];
    const uint64_t inc = dev::warp_incl_scan(tsum);
    if (dev::lane_id() == 31) warp_tot[dev::warp_id()] = inc;
    __syncthreads();
    if (threadIdx.x < 32) {
        const uint64_t x = warp_tot[threadIdx.x];
        const uint64_t xi = dev::warp_incl_scan(x);
        warp_tot[threadIdx.x] = xi - x;
        if (threadIdx.x == 31) warp_tot[32] = xi;
        __syncwarp();
        const uint64_t agg = warp_tot[32];
        if (threadIdx.x == 0) atomicExch(&status[t], (t == 0 ? kScanInc : kScanAgg) | agg);
        uint64_t excl = 0;
        if (t != 0) {
            for (int64_t k = (int64_t)t - 1;; k -= 32) {
                const int64_t idx = k - (int64_t)threadIdx.x;
                uint64_t st = kScanInc;  // below tile 0: an empty inclusive prefix
                if (idx >= 0) {
                    do {
                        st = *((volatile unsigned long long*)&status[idx]);
                    } while ((st & ~kScanVal) == 0);
                }
                const unsigned incm = __ballot_sync(0xffffffffu, (st & ~kScanVal) == kScanInc);
                const int first = incm ? __ffs(incm) - 1 : 32;
                uint64_t w = (int)threadIdx.x <= first ? (st & kScanVal) : 0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) w += __shfl_xor_sync(0xffffffffu, w, d);
                excl += w;
                if (incm) break;
            }
            if (threadIdx.x == 0) atomicExch(&status[t], kScanInc | (excl + agg));
        }
        if (threadIdx.x == 0) {
            s_excl = excl;
            if (total && t + 1 == ntiles) *total = static_cast<Out>(excl + agg);
        }
    }
    __syncthreads();
    uint64_t run = s_excl + warp_tot[dev::warp_id()] + inc - tsum;
    alignas(16) Out o[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        o[k] = static_cast<Out>(run);
        run += v[k];
    }
    if (vec) {
        uint4* d = reinterpret_cast<uint4*>(out + my);
        constexpr int kVec = kScanItems * (int)sizeof(Out) / 16;
#pragma unroll
        for (int q = 0; q < kVec; ++q) {
            uint4 w;
            memcpy(&w, reinterpret_cast<const char*>(o) + 16 * q, 16);
            d[q] = w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (my + k < n) out[my + k] = o[k];
    }
}

template <class Out>
void scan_impl(const uint32_t* in, Out* out, size_t n, Out* total, cudaStream_t s, const uint32_t* dn = nullptr,
               uint32_t mult = 1) {
    const size_t nb = n ? (n + kScanTile - 1) / kScanTile : 0;
    static int two_pass = -1;  // PRG_SCAN_2PASS=1: reduce-then-scan (A/B knob)
    if (two_pass < 0) { const char* e = getenv("PRG_SCAN_2PASS"); two_pass = e ? atoi(e) : 0; }
    if (!two_pass) {
        DevBuf<unsigned long long> st(nb + 1, s);  // tile status words, then the tile counter
        PRG_CUDA(cudaMemsetAsync(st.get(), 0, (nb + 1) * sizeof(unsigned long long), s));
        scan_onepass_kernel<Out><<<(unsigned)std::max<size_t>(nb, 1), kScanThreads, 0, s>>>(
            in, n, dn, mult, st.get(), reinterpret_cast<uint32_t*>(st.get() + nb), out, total);
        PRG_LAUNCH_CHECK();
        return;
    }
    DevBuf<uint64_t> part(nb + 1, s);
    if (nb) {
        scan_reduce_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, dn, mult, part.get());
        PRG_LAUNCH_CHECK();
    }
    scan_partials_kernel<<<1, kScanThreads, 0, s>>>(part.get(), nb, dn, mult);
    PRG_LAUNCH_CHECK();
    if (nb) {
        scan_down_kernel<Out><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, dn, mult, part.get(), out);
        PRG_LAUNCH_CHECK();
    }
    if (total) {
        copy_total_kernel<Out><<<1, 1, 0, s>>>(part.get(), nb, total);
        PRG_LAUNCH_CHECK();
    }
}
}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total,
                        cudaStream_t s) {
    scan_impl<uint32_t>(in, out, n, total, s);
}
void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, size_t n, uint64_t* total,
                               cudaStream_t s) {
    scan_impl<uint64_t>(in, out, n, total, s);
}
void exclusive_scan_u32_prefix(const uint32_t* in, uint32_t* out, size_t cap, const uint32_t* d_count,
                               uint32_t mult, cudaStream_t s) {
    scan_impl<uint32_t>(in, out, cap, nullptr, s, d_count, mult);
}


// ---- staged host <-> device copies ------------------------------------------
// A pageable cudaMemcpy moves ~10-20 GB/s through the driver's own staging and
// runs on one host thread, and first-touch page faults on a fresh destination
// vector serialise behind it. Large copies here go through pinned slots owned
// by kStageWorkers host threads, each with its own stream: a worker memcpys a
// chunk into its slot while its previous chunk is on the wire, so host copies,
// page faults and DMA all overlap (the drop-in's TSV-record paths move 0.25-1 GB
// per call at S=20-22). Slots are allocated once per process and kept.
namespace {
constexpr int kStageWorkers = 8;
constexpr size_t kStageChunk = size_t{4} << 20;  // bytes per slot
constexpr size_t kStageMin = size_t{8} << 20;    // below this: one plain copy
struct StageWorker {
    void* slot[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};
};
std::mutex g_stage_mu;  // one staged copy at a time owns the slots
StageWorker g_stage[kStageWorkers];
bool g_stage_ready = false;

void stage_init() {
    if (g_stage_ready) return;
    for (auto& w : g_stage) {
        for (int k = 0; k < 2; ++k) {
            PRG_CUDA(cudaMallocHost(&w.slot[k], kStageChunk));
            PRG_CUDA(cudaEventCreateWithFlags(&w.done[k], cudaEventDisableTiming));
        }
        PRG_CUDA(cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking));
    }
    g_stage_ready = true;
}

template <class Fn>
void stage_run(Fn&& fn) {  // fn(worker index) on kStageWorkers threads, errors rethrown here
    int dev = 0;
    PRG_CUDA(cudaGetDevice(&dev));
    std::vector<std::thread> crew;
    std::vector<std::string> err(kStageWorkers);
    for (int w = 0; w < kStageWorkers; ++w)
        crew.emplace_back([&, w] {
            try {
                PRG_CUDA(cudaSetDevice(dev));
                fn(w);
            } catch (const CudaError& e) {
                err[(size_t)w] = e.msg;
            }
        });
    for (auto& t : crew) t.join();
    for (auto& e : err)
        if (!e.empty()) throw CudaError{e};
}
}  // namespace

void copy_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < kStageMin) {
        PRG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    PRG_CUDA(cudaStreamSynchronize(s));  // dst (stream-ordered allocation) is usable from the worker streams
    std::lock_guard<std::mutex> lk(g_stage_mu);
    stage_init();
    const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
    stage_run([&](int w) {
        StageWorker& W = g_stage[w];
        int k = 0;
        for (size_t c = (size_t)w; c < nch; c += kStageWorkers, k ^= 1) {
            const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
            PRG_CUDA(cudaEventSynchronize(W.done[k]));  // the slot's previous copy has left
            std::memcpy(W.slot[k], static_cast<const char*>(src) + off, len);
            PRG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, W.slot[k], len, cudaMemcpyHostToDevice, W.st));
            PRG_CUDA(cudaEventRecord(W.done[k], W.st));
        }
        PRG_CUDA(cudaStreamSynchronize(W.st));
    });
    // the data is on the device before any later work on `s` (the workers synchronised)
}

void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < kStageMin) {
        PRG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        PRG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    PRG_CUDA(cudaStreamSynchronize(s));  // the producing kernels are done
    std::lock_guard<std::mutex> lk(g_stage_mu);
    stage_init();
    const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
    stage_run([&](int w) {
        StageWorker& W = g_stage[w];
        // double-buffered: chunk i+1 is on the wire while chunk i is copied out
        size_t prev_off = 0, prev_len = 0;
        int k = 0;
        bool have_prev = false;
        for (size_t c = (size_t)w;; c += kStageWorkers) {
            const bool more = c < nch;
            if (more) {
                const size_t off = c * kStageChunk, len = std::min(kStageChunk, bytes - off);
                PRG_CUDA(cudaMemcpyAsync(W.slot[k], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                         W.st));
                PRG_CUDA(cudaEventRecord(W.done[k], W.st));
                if (have_prev) {
                    PRG_CUDA(cudaEventSynchronize(W.done[k ^ 1]));
                    std::memcpy(static_cast<char*>(dst) + prev_off, W.slot[k ^ 1], prev_len);
                }
                prev_off = off;
                prev_len = len;
                have_prev = true;
                k ^= 1;
            } else {
                if (have_prev) {
                    PRG_CUDA(cudaEventSynchronize(W.done[k ^ 1]));
                    std::memcpy(static_cast<char*>(dst) + prev_off, W.slot[k ^ 1], prev_len);
                }
                break;
            }
        }
    });
}

}  // namespace prg

PRG_CHECK_QUERY(runtime)
