// medfilt_gpu_cli.cpp -- a `filter` / `generate` front end with `--algorithm gpu`
// (SURVEY.md §8(f) rank 3).  The reference's CLI (tools/medfilt_cli.cpp) needs CLI11,
// which is absent, so this one parses argv by hand.  Its I/O and generators are the
// reference's own (io.hpp:42-119, generators.hpp:91-142), included read-only at build time
// (tests/cpp/Makefile); "gpu" runs medfilt::gpu::median_filter<T> (include/medfilt/gpu.hpp),
// "sort" the reference's median_filter<T> (filter.hpp:149-155).  Same behaviour as the
// reference front end for the cases it documents: empty input and n < k warn and emit an
// empty output; invalid windows and parse errors print a diagnostic and exit 1.
//
//   medfilt_gpu filter   --k K [--algorithm gpu|sort] [--format text|bin] [--in P] [--out P]
//   medfilt_gpu generate --kind KIND --n N [--seed S] [--width 32|64] [--format text|bin] [--out P]
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "medfilt/gpu.hpp"
#include "medfilt/medfilt.hpp"

namespace {

std::map<std::string, std::string> parse_flags(int argc, char** argv, int first) {
  std::map<std::string, std::string> f;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0 || i + 1 >= argc) throw std::invalid_argument("bad argument: " + a);
    f[a.substr(2)] = argv[++i];
  }
  return f;
}

std::string get(const std::map<std::string, std::string>& f, const std::string& key, const std::string& dflt) {
  const auto it = f.find(key);
  return it == f.end() ? dflt : it->second;
}

template <typename T>
std::vector<T> run(const std::string& alg, const std::vector<T>& x, std::size_t k) {
  if (alg == "gpu") return medfilt::gpu::median_filter<T>(x, k);
  if (alg == "sort") return medfilt::median_filter<T>(x, k);
  throw std::invalid_argument("unknown algorithm: " + alg);
}

template <typename T>
std::vector<T> narrow(const std::vector<std::int64_t>& v) {
  return std::vector<T>(v.begin(), v.end());
}

int cmd_filter(const std::map<std::string, std::string>& f) {
  const std::size_t k = std::stoull(get(f, "k", "0"));
  const std::string alg = get(f, "algorithm", "gpu"), fmt = get(f, "format", "text");
  const std::string in_path = get(f, "in", "-"), out_path = get(f, "out", "-");
  std::ifstream fin;
  std::ofstream fout;
  if (in_path != "-") fin.open(in_path, std::ios::binary);
  if (out_path != "-") fout.open(out_path, std::ios::binary | std::ios::trunc);
  std::istream& in = in_path == "-" ? std::cin : fin;
  std::ostream& out = out_path == "-" ? std::cout : fout;
  if (!in || !out) { std::cerr << "medfilt_gpu: cannot open input/output\n"; return 1; }
  try {
    if (fmt == "text") {
      const auto x = medfilt::read_text(in);
      if (x.empty()) { std::cerr << "medfilt_gpu: warning: empty input, emitting empty output\n"; return 0; }
      if (x.size() < k) std::cerr << "medfilt_gpu: warning: input shorter than window, emitting empty output\n";
      medfilt::write_text<std::int64_t>(out, run<std::int64_t>(alg, x, k));
    } else {
      const auto data = medfilt::read_binary(in);
      if (data.values.empty()) {
        std::cerr << "medfilt_gpu: warning: empty input, emitting empty output\n";
        out.put(static_cast<char>(data.width));
        return 0;
      }
      if (data.values.size() < k)
        std::cerr << "medfilt_gpu: warning: input shorter than window, emitting empty output\n";
      if (data.width == 32) medfilt::write_binary<std::int32_t>(out, run<std::int32_t>(alg, narrow<std::int32_t>(data.values), k));
      else medfilt::write_binary<std::int64_t>(out, run<std::int64_t>(alg, data.values, k));
    }
  } catch (const medfilt::ParseError& e) {
    std::cerr << "medfilt_gpu: parse error at line " << e.line() << ": " << e.what() << '\n';
    return 1;
  } catch (const std::invalid_argument& e) {
    std::cerr << "medfilt_gpu: " << e.what() << '\n';
    return 1;
  }
  return 0;
}

int cmd_generate(const std::map<std::string, std::string>& f) {
  try {
    const auto kind = medfilt::parse_generator_kind(get(f, "kind", "r-large"));
    const std::size_t n = std::stoull(get(f, "n", "0"));
    const std::uint64_t seed = std::stoull(get(f, "seed", "0"));
    const int width = std::stoi(get(f, "width", "64"));
    const std::string fmt = get(f, "format", "text"), out_path = get(f, "out", "-");
    if (!medfilt::width_valid(width)) throw std::invalid_argument("width must be 32 or 64");
    std::ofstream fout;
    if (out_path != "-") fout.open(out_path, std::ios::binary | std::ios::trunc);
    std::ostream& out = out_path == "-" ? std::cout : fout;
    if (width == 32) {
      const auto x = medfilt::generate<std::int32_t>(kind, n, seed);
      if (fmt == "text") medfilt::write_text<std::int32_t>(out, x); else medfilt::write_binary<std::int32_t>(out, x);
    } else {
      const auto x = medfilt::generate<std::int64_t>(kind, n, seed);
      if (fmt == "text") medfilt::write_text<std::int64_t>(out, x); else medfilt::write_binary<std::int64_t>(out, x);
    }
  } catch (const std::invalid_argument& e) {
    std::cerr << "medfilt_gpu: " << e.what() << '\n';
    return 1;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: medfilt_gpu filter|generate --flag value ...\n";
    return 2;
  }
  try {
    const std::string cmd = argv[1];
    const auto flags = parse_flags(argc, argv, 2);
    if (cmd == "filter") return cmd_filter(flags);
    if (cmd == "generate") return cmd_generate(flags);
    std::cerr << "medfilt_gpu: unknown command " << cmd << '\n';
  } catch (const std::exception& e) {
    std::cerr << "medfilt_gpu: " << e.what() << '\n';
  }
  return 2;
}
