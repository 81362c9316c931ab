// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, built by
// oracle/Makefile from the headers where they lie (-I/root/reference/proj/include,
// read-only, nothing copied) into oracle/_ref/libmedfilt_ref.so.  Used to pin the
// C restatement (oracle/medfilt_oracle.c), to produce golden fixtures, and as
// the "reference" CPU arm of bench.py (cpu_baseline.kind = "reference").
//
// Reference entry points wrapped (all under /root/reference/proj/include/medfilt/):
//   median_filter<T>         filter.hpp:149-155    (the hot path)
//   pad_to_blocks/piecewise_sort filter.hpp:28-54  (phase-1 parity)
//   naive_median_filter<T>   baselines.hpp:287-300
//   fold_checksum<T>         io.hpp:17-28
//   generate<T>              generators.hpp:91-142
//   run_verify               verify.hpp:137-178
//   sort_via_median_filter   filter.hpp:177-205
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "medfilt/medfilt.hpp"

namespace {
thread_local std::string g_last_error;

// Map the reference's std::invalid_argument texts (core.hpp:63-69) onto the
// status codes of include/medfilt_gpu.h.
int status_of(const std::exception& e) {
  g_last_error = e.what();
  const std::string w = e.what();
  if (w == "input must not be empty") return 1;
  if (w == "window size must be positive") return 2;
  if (w.rfind("even window size", 0) == 0) return 3;
  if (w == "window size too large") return 4;
  return 5;
}

template <typename T>
int run_filter(const T* x, std::size_t n, std::size_t k, T* y, std::size_t* y_len) {
  try {
    const std::vector<T> out = medfilt::median_filter<T>(std::span<const T>(x, n), k);
    if (!out.empty()) std::memcpy(y, out.data(), out.size() * sizeof(T));
    *y_len = out.size();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Halo-sharded run over `threads` std::threads: shard g computes outputs
// [o_g, o_g+1) from the slice x[o_g, o_g+1 + k - 1).
template <typename T>
int run_filter_threads(const T* x, std::size_t n, std::size_t k, T* y, int threads) {
  try {
    const medfilt::WindowSpec spec = medfilt::make_window_spec(n, k);
    const std::size_t keep = spec.output_size();
    if (keep == 0) return 0;
    if (threads < 1) threads = 1;
    if (static_cast<std::size_t>(threads) > keep) threads = static_cast<int>(keep);
    std::vector<std::thread> pool;
    for (int g = 0; g < threads; ++g) {
      const std::size_t o0 = keep * g / threads, o1 = keep * (g + 1) / threads;
      pool.emplace_back([=] {
        const std::vector<T> out =
            medfilt::median_filter<T>(std::span<const T>(x + o0, o1 - o0 + k - 1), k);
        std::memcpy(y + o0, out.data(), out.size() * sizeof(T));
      });
    }
    for (auto& t : pool) t.join();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Independent rows over threads (config 3 layout: rows x len, row-major).
template <typename T>
int run_rows_threads(const T* x, std::size_t rows, std::size_t len, std::size_t k, T* y,
                     int threads) {
  try {
    const medfilt::WindowSpec spec = medfilt::make_window_spec(len, k);
    const std::size_t keep = spec.output_size();
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int g = 0; g < threads; ++g) {
      pool.emplace_back([=] {
        for (std::size_t r = g; r < rows; r += threads) {
          const std::vector<T> out =
              medfilt::median_filter<T>(std::span<const T>(x + r * len, len), k);
          if (keep) std::memcpy(y + r * keep, out.data(), keep * sizeof(T));
        }
      });
    }
    for (auto& t : pool) t.join();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_median_filter_i32(const int32_t* x, std::size_t n, std::size_t k, int32_t* y, std::size_t* y_len) {
  return run_filter<int32_t>(x, n, k, y, y_len);
}
int ref_median_filter_i64(const int64_t* x, std::size_t n, std::size_t k, int64_t* y, std::size_t* y_len) {
  return run_filter<int64_t>(x, n, k, y, y_len);
}
int ref_median_filter_threads_i32(const int32_t* x, std::size_t n, std::size_t k, int32_t* y, int threads) {
  return run_filter_threads<int32_t>(x, n, k, y, threads);
}
int ref_median_filter_threads_i64(const int64_t* x, std::size_t n, std::size_t k, int64_t* y, int threads) {
  return run_filter_threads<int64_t>(x, n, k, y, threads);
}
int ref_median_filter_rows_i32(const int32_t* x, std::size_t rows, std::size_t len, std::size_t k,
                               int32_t* y, int threads) {
  return run_rows_threads<int32_t>(x, rows, len, k, y, threads);
}

// pad_to_blocks + piecewise_sort (filter.hpp:28-54); perms is b*k entries.
int ref_piecewise_sort_i64(const int64_t* x, std::size_t n, std::size_t k, uint32_t* perms) {
  try {
    const medfilt::WindowSpec spec = medfilt::make_window_spec(n, k);
    const auto input = medfilt::pad_to_blocks<int64_t>(std::span<const int64_t>(x, n), spec);
    const auto p = medfilt::piecewise_sort<int64_t>(input);
    for (std::size_t j = 0; j < p.size(); ++j)
      std::memcpy(perms + j * k, p[j].data(), k * sizeof(uint32_t));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_naive_i64(const int64_t* x, std::size_t n, std::size_t k, int64_t* y, std::size_t* y_len) {
  try {
    const auto out = medfilt::naive_median_filter<int64_t>(std::span<const int64_t>(x, n), k);
    if (!out.empty()) std::memcpy(y, out.data(), out.size() * sizeof(int64_t));
    *y_len = out.size();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

uint64_t ref_fold_checksum_i32(const int32_t* v, std::size_t n) {
  return medfilt::fold_checksum<int32_t>(std::span<const int32_t>(v, n));
}
uint64_t ref_fold_checksum_i64(const int64_t* v, std::size_t n) {
  return medfilt::fold_checksum<int64_t>(std::span<const int64_t>(v, n));
}

// generate<T>(kind, n, seed) (generators.hpp:91-142), widened to int64.
int ref_generate_i64(int kind, std::size_t n, uint64_t seed, int width, int64_t* out) {
  try {
    const auto kinds = medfilt::kAllGenerators;
    if (kind < 0 || kind >= 7) return 5;
    if (width == 32) {
      const auto v = medfilt::generate<int32_t>(kinds[kind], n, seed);
      for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    } else {
      const auto v = medfilt::generate<int64_t>(kinds[kind], n, seed);
      std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

uint64_t ref_splitmix64_next(uint64_t* state) {
  medfilt::SplitMix64 rng(*state);
  const uint64_t v = rng.next();
  *state = rng.state;
  return v;
}

// run_verify (verify.hpp:137-178): returns 1 when OK, fills case counts.
int ref_run_verify(std::size_t n_max, std::size_t trials, uint64_t seed, int inject_fault,
                   std::size_t* exhaustive, std::size_t* random) {
  const auto report = medfilt::run_verify(n_max, trials, seed, inject_fault != 0);
  *exhaustive = report.exhaustive_cases;
  *random = report.random_cases;
  return report.ok() ? 1 : 0;
}

// sort_via_median_filter (filter.hpp:177-205): nb blocks of h+1 values each.
int ref_sort_via_median_filter_i64(const int64_t* blocks, std::size_t nb, std::size_t h, int64_t* out) {
  try {
    std::vector<std::vector<int64_t>> in(nb);
    for (std::size_t j = 0; j < nb; ++j) in[j].assign(blocks + j * (h + 1), blocks + (j + 1) * (h + 1));
    const auto s = medfilt::sort_via_median_filter<int64_t>(in, h);
    for (std::size_t j = 0; j < nb; ++j) std::memcpy(out + j * (h + 1), s[j].data(), (h + 1) * sizeof(int64_t));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

}  // extern "C"
