// host_sorts.cpp -- TEST / BASELINE INFRASTRUCTURE ONLY (not the product path).
//
// The plain definition of LearnedSort's result ("std::sort with
// the ≺ comparator") as CPU baselines for bench.py's cpu_baseline leg
// (SURVEY §8(d) "How the oracle is timed beside it"): std::sort(≺) on the
// calling thread, and the same comparator through libstdc++'s parallel mode
// (__gnu_parallel::sort, OpenMP) on every host core. Shares nothing with the
// CUDA path. Keys are raw 64-bit patterns; dtype 0 = IEEE binary64 (order =
// IEEE totalOrder via ord(x), R12), 1 = unsigned 64-bit.
#include <parallel/algorithm>

#include <algorithm>
#include <cstdint>

#include <omp.h>

namespace {

inline uint64_t ord_f64(uint64_t u) { return (u >> 63) ? ~u : (u | (1ull << 63)); }

struct LessF64 {
    bool operator()(uint64_t a, uint64_t b) const { return ord_f64(a) < ord_f64(b); }
};

}  // namespace

extern "C" {

void lso_std_sort(uint64_t *A, uint64_t n, int dtype) {
    if (dtype == 0) std::sort(A, A + n, LessF64());
    else std::sort(A, A + n);
}

// Returns the number of OpenMP threads the parallel sort used.
int lso_parallel_sort(uint64_t *A, uint64_t n, int dtype) {
    if (dtype == 0) __gnu_parallel::sort(A, A + n, LessF64());
    else __gnu_parallel::sort(A, A + n);
    return omp_get_max_threads();
}

}  // extern "C"
