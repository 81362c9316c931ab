// verify_gpu.cpp -- the reference's own cross-check methodology run against the GPU
// filter.  Built from the reference headers (read-only,
// -I/root/reference/proj/include) plus include/medfilt/gpu.hpp by tests/cpp/Makefile;
// the binary travels to the GPU box prebuilt.
//
// Registers "gpu" -> &medfilt::gpu::median_filter<T> next to the reference's "sort"
// (median_filter<T>, filter.hpp:149-155) in a FilterFn table shaped like verify.hpp:60-70,
// then runs run_verify's sweeps (verify.hpp:137-178): every vector of length <= n_max over
// {0,1,2} with every odd k, plus seeded random cases over all seven generators
// (generators.hpp:91-142) and both widths, each compared with naive_median_filter
// (baselines.hpp:287-300).  A deliberately broken filter (verify.hpp:40-52) proves the
// harness can fail.  Exit code 0 = every case agrees.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "medfilt/medfilt.hpp"
#include "medfilt/gpu.hpp"

template <typename T>
struct Named {
  const char* name;
  medfilt::detail::FilterFn<T> run;
};

template <typename T>
static bool check(const std::vector<Named<T>>& table, std::span<const T> x, std::size_t k, const char* gen,
                  std::size_t* failures) {
  const std::vector<T> want = medfilt::naive_median_filter<T>(x, k);
  bool ok = true;
  for (const auto& f : table) {
    const std::vector<T> got = f.run(x, k);
    if (got != want) {
      ok = false;
      if (++*failures <= 5)
        std::fprintf(stderr, "mismatch: %s gen=%s n=%zu k=%zu width=%zu\n", f.name, gen, x.size(), k,
                     sizeof(T) * 8);
    }
  }
  return ok;
}

int main(int argc, char** argv) {
  const std::size_t n_max = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 8;
  const std::size_t trials = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 300;
  const bool inject = argc > 3 && std::string(argv[3]) == "--inject-fault";
  std::vector<Named<std::int64_t>> t64 = {{"sort", &medfilt::median_filter<std::int64_t>},
                                          {"gpu", &medfilt::gpu::median_filter<std::int64_t>}};
  std::vector<Named<std::int32_t>> t32 = {{"sort", &medfilt::median_filter<std::int32_t>},
                                          {"gpu", &medfilt::gpu::median_filter<std::int32_t>}};
  if (inject) t64.push_back({"broken", &medfilt::detail::broken_median_filter<std::int64_t>});
  std::size_t failures = 0, exhaustive = 0, random = 0;
  // exhaustive sweep, verify.hpp:142-158
  for (std::size_t n = 1; n <= n_max; ++n) {
    std::vector<std::int64_t> x(n, 0);
    for (;;) {
      for (std::size_t k = 1; k <= n; k += 2) {
        check<std::int64_t>(t64, x, k, "exhaustive", &failures);
        ++exhaustive;
      }
      std::size_t i = 0;
      while (i < n && x[i] == 2) x[i++] = 0;
      if (i == n) break;
      ++x[i];
    }
  }
  // seeded random sweep over generators and widths, verify.hpp:160-176
  medfilt::SplitMix64 rng(12345);
  for (std::size_t t = 0; t < trials; ++t) {
    const auto kind = medfilt::kAllGenerators[t % 7];
    const std::size_t n = 1 + rng.below(3000);
    const std::size_t k = 2 * rng.below(std::min<std::size_t>(n, 1200) / 2 + 1) + 1;
    if (t % 2 == 0) {
      const auto x = medfilt::generate<std::int64_t>(kind, n, t);
      check<std::int64_t>(t64, x, k, std::string(medfilt::to_string(kind)).c_str(), &failures);
    } else {
      const auto x = medfilt::generate<std::int32_t>(kind, n, t);
      check<std::int32_t>(t32, x, k, std::string(medfilt::to_string(kind)).c_str(), &failures);
    }
    ++random;
  }
  // error behaviour: identical exception texts (core.hpp:63-69)
  const char* expect[] = {"input must not be empty", "window size must be positive",
                          "even window size unsupported (window must be k = 2h+1)"};
  const std::vector<std::int32_t> empty, four = {1, 2, 3, 4};
  const std::pair<const std::vector<std::int32_t>*, std::size_t> bad[] = {{&empty, 3}, {&four, 0}, {&four, 4}};
  for (int i = 0; i < 3; ++i) {
    try {
      medfilt::gpu::median_filter<std::int32_t>(*bad[i].first, bad[i].second);
      ++failures;
    } catch (const std::invalid_argument& e) {
      if (std::string(e.what()) != expect[i]) ++failures;
    }
  }
  // the §2 reduction witness through the GPU filter (filter.hpp:177-205)
  {
    const std::vector<std::vector<std::int64_t>> blocks = {{3, 1}, {9, 7}};
    const auto got = medfilt::gpu::sort_via_median_filter<std::int64_t>(blocks, 1);
    const auto want = medfilt::sort_via_median_filter<std::int64_t>(blocks, 1);
    if (got != want) ++failures;
    medfilt::SplitMix64 g(99);
    std::vector<std::vector<std::int64_t>> big(50, std::vector<std::int64_t>(64));
    for (auto& b : big) for (auto& v : b) v = static_cast<std::int64_t>(g.next());
    if (medfilt::gpu::sort_via_median_filter<std::int64_t>(big, 63) !=
        medfilt::sort_via_median_filter<std::int64_t>(big, 63))
      ++failures;
  }
  std::printf("verify_gpu: exhaustive=%zu random=%zu failures=%zu\n", exhaustive, random, failures);
  return failures == 0 ? 0 : 1;
}
