// bench_gpu.cpp -- the reference's timing methodology with "gpu" registered
// (SURVEY.md §8(f) rank 1).  Cells follow bench_cell (bench.hpp:81-122): for each
// (algorithm, generator, h) the signal has n = (2h+1) * round(bh/h) samples generated as
// generate(kind, n, seed + repeat); repeat 0 is preceded by a discarded warm-up; every
// repeat is timed by the reference's time_filter (bench.hpp:63-72, steady_clock around
// the FilterFn call only, fold_checksum as the sink); a median row closes the cell.  The
// CSV is the reference's write_csv (bench.hpp:156-181).  "sort" is the reference's
// median_filter<T>, "gpu" is medfilt::gpu::median_filter<T> through the host C ABI, so its
// times include both PCIe copies.  Matching checksums per cell show the outputs agree.
//
//   bench_gpu [bh] [repeats] [seed] [width] [h ...]
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <string>
#include <vector>

#include "medfilt/gpu.hpp"
#include "medfilt/medfilt.hpp"

template <typename T>
void cell(const char* alg, medfilt::detail::FilterFn<T> fn, medfilt::GeneratorKind kind, std::size_t h,
          std::uint64_t bh, std::size_t repeats, std::uint64_t seed, std::vector<medfilt::BenchRecord>& out) {
  const std::size_t b = h == 0 ? bh : (bh + h / 2) / h;
  const std::size_t k = 2 * h + 1, n = k * b;
  medfilt::BenchRecord base;
  base.algorithm = alg;
  base.generator = std::string(medfilt::to_string(kind));
  base.width = static_cast<int>(sizeof(T) * 8);
  base.n = n;
  base.h = h;
  base.b = b;
  std::vector<double> times;
  for (std::size_t rep = 0; rep < repeats; ++rep) {
    const std::vector<T> x = medfilt::generate<T>(kind, n, seed + rep);
    if (rep == 0) (void)medfilt::detail::time_filter<T>(fn, x, k);
    const auto [secs, sum] = medfilt::detail::time_filter<T>(fn, x, k);
    medfilt::BenchRecord r = base;
    r.repeat = static_cast<long>(rep);
    r.wall_time_s = secs;
    r.checksum = sum;
    out.push_back(r);
    times.push_back(secs);
  }
  medfilt::BenchRecord med = base;
  med.repeat = -1;
  med.wall_time_s = medfilt::detail::median_time(times);
  med.checksum = out.back().checksum;
  out.push_back(med);
}

int main(int argc, char** argv) {
  const std::uint64_t bh = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
  const std::size_t repeats = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 3;
  const std::uint64_t seed = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 0;
  const int width = argc > 4 ? std::atoi(argv[4]) : 32;
  std::vector<std::size_t> hs;
  for (int i = 5; i < argc; ++i) hs.push_back(std::strtoull(argv[i], nullptr, 10));
  if (hs.empty()) hs = {1, 15, 127, 511, 5000};
  std::vector<medfilt::BenchRecord> recs;
  for (auto kind : medfilt::kAllGenerators)
    for (std::size_t h : hs) {
      if (width == 32) {
        cell<std::int32_t>("sort", &medfilt::median_filter<std::int32_t>, kind, h, bh, repeats, seed, recs);
        cell<std::int32_t>("gpu", &medfilt::gpu::median_filter<std::int32_t>, kind, h, bh, repeats, seed, recs);
      } else {
        cell<std::int64_t>("sort", &medfilt::median_filter<std::int64_t>, kind, h, bh, repeats, seed, recs);
        cell<std::int64_t>("gpu", &medfilt::gpu::median_filter<std::int64_t>, kind, h, bh, repeats, seed, recs);
      }
    }
  medfilt::write_csv(std::cout, recs);
  return 0;
}
