// Test-fixture helper (TEST INFRASTRUCTURE ONLY): reproduces the reference's
// seeded Gaussian streams bit-for-bit with the same standard library the
// reference is built with (libstdc++ std::mt19937_64 +
// std::normal_distribution<double>), so the oracle can be pinned against the
// reference's own known-answer tests.
//
// Streams restated (not copied):
//   "matrix R C SEED"  -- tests/test_support.hpp:11-18 (random_matrix): one
//                         engine + one distribution, filled row by row.
//   "lowrank M N SEED" -- core/src/generate.cpp:36-42,83-91 (gen_low_rank):
//                         one engine; gaussian(M,p) then gaussian(N,p), each
//                         call with a fresh distribution, p = min(M,N).
// Reads one spec per line on stdin, writes the row-major doubles of every
// requested matrix, concatenated, to stdout.
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

static void emit(const std::vector<double>& v) {
  std::fwrite(v.data(), sizeof(double), v.size(), stdout);
}

static std::vector<double> fill(long rows, long cols, std::mt19937_64& rng) {
  std::normal_distribution<double> dist(0.0, 1.0);
  std::vector<double> g(static_cast<size_t>(rows * cols));
  for (long i = 0; i < rows; ++i)
    for (long j = 0; j < cols; ++j) g[static_cast<size_t>(i * cols + j)] = dist(rng);
  return g;
}

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    std::istringstream in(line);
    std::string kind;
    long a = 0, b = 0;
    std::uint64_t seed = 0;
    if (!(in >> kind >> a >> b >> seed)) continue;
    std::mt19937_64 rng(seed);
    if (kind == "matrix") {
      emit(fill(a, b, rng));
    } else if (kind == "lowrank") {
      const long p = a < b ? a : b;
      emit(fill(a, p, rng));
      emit(fill(b, p, rng));
    } else {
      std::fprintf(stderr, "unknown spec %s\n", kind.c_str());
      return 2;
    }
  }
  return 0;
}
