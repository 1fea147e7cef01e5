// Dev microbenchmark (not product code): host-side streaming passes the e2e
// path could run before the PCIe copy — int64->u32 narrowing of 2^28 column
// indices and a row-base scan of 2^28 f64 values — with T threads.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdlib>
int main(int argc, char** argv) {
    const size_t n = size_t(1) << 28;
    int T = argc > 1 ? atoi(argv[1]) : std::thread::hardware_concurrency();
    std::vector<int64_t> a(n);
    std::vector<uint32_t> b(n);
    std::vector<double> v(n);
    for (size_t i = 0; i < n; ++i) { a[i] = (int64_t)(i * 2654435761u % 16777216); v[i] = 1.0 / (1 + (i >> 4) % 100); }
    auto run = [&](auto fn) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back([&, t] { fn(n * t / T, n * (t + 1) / T); });
        for (auto& x : th) x.join();
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    for (int r = 0; r < 3; ++r) {
        double t1 = run([&](size_t lo, size_t hi) { for (size_t i = lo; i < hi; ++i) b[i] = (uint32_t)a[i]; });
        std::vector<uint64_t> cnt(T * 8, 0);
        double t2 = run([&](size_t lo, size_t hi) {
            uint64_t c = 0; const uint64_t* p = reinterpret_cast<const uint64_t*>(v.data());
            for (size_t i = lo + 1; i < hi; ++i) c += p[i] != p[i - 1];
            cnt[(lo * T / n) * 8] = c; });
        double t3 = run([&](size_t lo, size_t hi) { memcpy(b.data() + lo, a.data() + lo / 2, (hi - lo) * 4); });
        printf("T=%d narrow 2^28 i64->u32: %.1f ms (%.1f GB/s read)  scan 2^28 f64: %.1f ms (%.1f GB/s)  memcpy 1GB: %.1f ms\n",
               T, t1 * 1e3, n * 8 / t1 / 1e9, t2 * 1e3, n * 8 / t2 / 1e9, t3 * 1e3);
    }
    return 0;
}
