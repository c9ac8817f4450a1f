// call_overhead — wall time per call of the reference-facing drop-in API (include/ssbh/*.hpp
// over libssbh_cuda.so) at small shapes, the way the reference's own callers use it: one
// toeplitz_hash per block (proj/src/pipeline.cpp:129-136), KeyedStream::bits per block seed,
// assign_subblocks / sift_partition once per extraction. Prints one CSV row per call kind:
// call,shape,calls,median_us,p90_us
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "ssbh/prf.hpp"
#include "ssbh/sampling.hpp"
#include "ssbh/toeplitz.hpp"

using namespace ssbh;

template <class F>
void time_calls(const char* name, const char* shape, int calls, F&& fn) {
    for (int i = 0; i < 3; ++i) fn();  // warm (module load, per-thread arena)
    std::vector<double> us(calls);
    for (double& v : us) {
        const auto t0 = std::chrono::steady_clock::now();
        fn();
        v = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    }
    std::sort(us.begin(), us.end());
    std::printf("%s,%s,%d,%.1f,%.1f\n", name, shape, calls, us[us.size() / 2],
                us[us.size() * 9 / 10]);
}

int main() {
    const MasterSeed seed = MasterSeed::from_hex(
        "000000000000000000000000000000000000000000000000000000000000002a");
    std::printf("call,shape,calls,median_us,p90_us\n");
    for (const auto [m, n] : {std::pair<std::uint64_t, std::uint64_t>{64, 1000},
                              {2000, 50000}, {8192, 16384}}) {
        const BitString x = KeyedStream(seed, "x").bits(n);
        const ToeplitzSeed ts(KeyedStream(seed, "s").bits(m + n - 1), m, n);
        char shape[64];
        std::snprintf(shape, sizeof shape, "m=%llu n=%llu", (unsigned long long)m,
                      (unsigned long long)n);
        time_calls("toeplitz_hash", shape, 200, [&] { (void)toeplitz_hash(ts, x); });
    }
    time_calls("KeyedStream::bits", "nbits=100000", 200,
               [&] { (void)KeyedStream(seed, "hash-seed", 3).bits(100000); });
    time_calls("assign_subblocks", "n=100000 s=16", 200,
               [&] { (void)assign_subblocks(100000, 16, seed); });
    const Partition part = assign_subblocks(100000, 16, seed);
    const std::vector<std::uint8_t> keep(100000, 1);
    time_calls("sift_partition", "n=100000 s=16", 200,
               [&] { (void)sift_partition(keep, part); });
    return 0;
}
