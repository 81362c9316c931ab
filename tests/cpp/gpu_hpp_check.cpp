// Compile-only check: medfilt::gpu::median_filter<T> has the reference's FilterFn<T>
// shape (baselines.hpp:29-30: std::vector<T> (*)(std::span<const T>, std::size_t)).
#include <cstdint>
#include <span>
#include <vector>

#include "medfilt/gpu.hpp"

template <typename T>
using FilterFn = std::vector<T> (*)(std::span<const T>, std::size_t);

FilterFn<std::int32_t> f32 = &medfilt::gpu::median_filter<std::int32_t>;
FilterFn<std::int64_t> f64 = &medfilt::gpu::median_filter<std::int64_t>;
std::vector<float> (*ff)(std::span<const float>, std::size_t) = &medfilt::gpu::median_filter;

int main() { return (f32 && f64 && ff) ? 0 : 1; }
