// Runtime check of gpu.hpp's device list (SURVEY.md §8(b) "Multi-GPU entry: a device
// list"): medfilt::gpu::median_filter<T> -- the FilterFn<T> shape, baselines.hpp:29-30 --
// over the devices MEDFILT_GPU_DEVICES or set_devices() names equals the reference's own
// medfilt::median_filter<T> (filter.hpp:149-155, headers included read-only).
#include <cstdint>
#include <cstdio>
#include <random>
#include <span>
#include <vector>

#include "medfilt/filter.hpp"
#include "medfilt/gpu.hpp"

template <typename T>
static bool check(const std::vector<T>& x, std::size_t k, const char* what) {
  const auto want = medfilt::median_filter<T>(std::span<const T>(x), k);
  const auto got = medfilt::gpu::median_filter<T>(std::span<const T>(x), k);
  if (got != want) {
    std::printf("MISMATCH %s k=%zu (n=%zu)\n", what, k, x.size());
    return false;
  }
  return true;
}

int main() {
  std::mt19937_64 rng(11);
  std::vector<std::int32_t> x32(3u << 20);
  for (auto& v : x32) v = static_cast<std::int32_t>(rng() % 1000);
  std::vector<std::int64_t> x64(x32.begin(), x32.end());
  bool ok = true;
  // 1) devices from the environment (the test sets MEDFILT_GPU_DEVICES=0,0)
  for (std::size_t k : {31u, 255u, 2049u}) ok &= check(x32, k, "env devices, int32");
  // 2) an explicit two-entry list, then back to one device
  medfilt::gpu::set_devices({0, 0});
  ok &= check(x64, 101, "set_devices({0,0}), int64");
  medfilt::gpu::set_devices({0});
  ok &= check(x64, 101, "set_devices({0}), int64");
  std::printf(ok ? "gpu_multi_check ok\n" : "gpu_multi_check FAILED\n");
  return ok ? 0 : 1;
}
