// hsvd_b200 -- command-line caller of the B200 path through the C ABI
// (SURVEY 8(f) next #3): the `svd` subcommand of the reference CLI
// (tools/hsvd_main.cpp:120-159, options :251-266) with the input streamed
// from an HSVD1 file straight to the device (hsvd_cu_load_hsvd1) and a
// --max-rank flag the reference lacks.  Exit codes as the reference
// (hsvd_main.cpp:27-29): 0 ok, 1 usage, 2 runtime error.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "hsvd_cu.h"

namespace {

constexpr int kOk = 0, kUsage = 1, kRuntime = 2;

struct UsageError {
  std::string what;
};
struct RuntimeFailure {
  std::string what;
};

const char* kHelp =
    "usage: hsvd_b200 svd --input FILE.hsvd [options]\n"
    "  --gamma G        relative truncation threshold (default 1e-2)\n"
    "  --row-block D    rows per block (0 = all rows)\n"
    "  --col-block C    columns per block (0 = all columns)\n"
    "  --max-rank K     hard rank cap (0 = none)\n"
    "  --refine         run iterative refinement (Alg. 2)\n"
    "  --eps E          refinement convergence threshold (default 1e-3)\n"
    "  --max-iters N    refinement iteration cap (default 10)\n"
    "  --out-prefix P   write P_{U,S,V}.hsvd and P_sigma.csv\n"
    "  --precise        print 17 significant digits\n"
    "  --device N       CUDA device (default 0)\n";

void check(int code) {
  if (code != HSVD_CU_OK) throw RuntimeFailure{hsvd_cu_last_error()};
}

template <typename T>
T parse_num(const std::string& opt, const std::string& text) {
  T v{};
  const auto [p, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
  if (ec != std::errc{} || p != text.data() + text.size())
    throw UsageError{opt + ": cannot parse '" + text + "'"};
  return v;
}

std::string num(double v, bool precise) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), precise ? "%.17g" : "%.6g", v);
  return buf;
}

std::string shortest(double v) {  // matrix_io.cpp format_double: round-trip
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, r.ptr);
}

void save_hsvd1(const std::string& path, const std::vector<double>& a, std::uint64_t rows,
                std::uint64_t cols) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw RuntimeFailure{path + ": cannot open for writing"};
  char header[22] = {'H', 'S', 'V', 'D', '1', '\0'};
  for (int i = 0; i < 8; ++i) {
    header[6 + i] = static_cast<char>((rows >> (8 * i)) & 0xff);
    header[14 + i] = static_cast<char>((cols >> (8 * i)) & 0xff);
  }
  out.write(header, sizeof(header));
  out.write(reinterpret_cast<const char*>(a.data()),
            static_cast<std::streamsize>(a.size() * sizeof(double)));
  if (!out) throw RuntimeFailure{path + ": write failed"};
}

int run_svd(int argc, char** argv) {
  std::string input, prefix;
  double gamma = 1e-2, eps = 1e-3;
  long long d = 0, c = 0, max_rank = 0;
  int iters = 10, device = 0;
  bool refine = false, precise = false;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto value = [&]() -> std::string {
      if (i + 1 >= argc) throw UsageError{a + ": missing value"};
      return argv[++i];
    };
    if (a == "--input") input = value();
    else if (a == "--format") {
      const std::string f = value();
      if (f != "hsvd") throw UsageError{"--format: only 'hsvd' is streamed to the device"};
    } else if (a == "--gamma") gamma = parse_num<double>(a, value());
    else if (a == "--row-block") d = parse_num<long long>(a, value());
    else if (a == "--col-block") c = parse_num<long long>(a, value());
    else if (a == "--max-rank") max_rank = parse_num<long long>(a, value());
    else if (a == "--refine") refine = true;
    else if (a == "--eps") eps = parse_num<double>(a, value());
    else if (a == "--max-iters") iters = parse_num<int>(a, value());
    else if (a == "--out-prefix") prefix = value();
    else if (a == "--precise") precise = true;
    else if (a == "--device") device = parse_num<int>(a, value());
    else if (a == "--help" || a == "-h") {
      std::fputs(kHelp, stdout);
      return kOk;
    } else throw UsageError{"unknown option " + a};
  }
  if (input.empty()) throw UsageError{"--input is required"};

  hsvd_cu_ctx* ctx = nullptr;
  check(hsvd_cu_ctx_create(device, &ctx));
  struct CtxGuard {
    hsvd_cu_ctx* c;
    ~CtxGuard() { hsvd_cu_ctx_destroy(c); }
  } cg{ctx};
  int64_t m = 0, n = 0;
  int dt = HSVD_CU_F64;
  const void* dx = nullptr;  // HSVD1 (fp64) or its fp32 variant HSVF1
  check(hsvd_cu_load_matrix(ctx, input.c_str(), &m, &n, &dt, &dx));
  const hsvd_cu_config cfg = {gamma, d, c, eps, iters, max_rank};
  check(hsvd_cu_validate(&cfg));

  hsvd_cu_result* res = nullptr;
  if (refine) {  // hierarchical_svd, then refine_factors from (V, sigma)
    hsvd_cu_result* right = nullptr;
    check(hsvd_cu_hierarchical_svd(ctx, dx, dt, m, n, n, HSVD_CU_DEVICE, &cfg, &right));
    int64_t r = 0, ur = 0, vr = 0;
    int32_t hu = 0, hv = 0, deg = 0;
    check(hsvd_cu_result_info(right, &r, &hu, &hv, &ur, &vr, &deg));
    std::vector<double> v((size_t)(n * r)), s((size_t)r);
    check(hsvd_cu_result_v(right, v.data()));
    check(hsvd_cu_result_sigma(right, s.data()));
    hsvd_cu_result_free(right);
    int32_t it = 0, conv = 0;
    double err = 0.0;
    check(hsvd_cu_refine_factors(ctx, dx, dt, m, n, n, HSVD_CU_DEVICE, v.data(), n, r, r,
                                 HSVD_CU_HOST, s.data(), r, eps, iters, &it, &err, &conv, &res));
    std::printf("refined in %d iteration(s), final error %s%s\n", it, num(err, precise).c_str(),
                conv ? "" : " (not converged)");
  } else {
    check(hsvd_cu_rank_k_svd(ctx, dx, dt, m, n, n, HSVD_CU_DEVICE, &cfg, &res));
  }
  int64_t k = 0, ur = 0, vr = 0;
  int32_t hu = 0, hv = 0, deg = 0;
  check(hsvd_cu_result_info(res, &k, &hu, &hv, &ur, &vr, &deg));
  std::vector<double> u((size_t)(m * k)), v((size_t)(n * k)), s((size_t)k);
  check(hsvd_cu_result_u(res, u.data()));
  check(hsvd_cu_result_v(res, v.data()));
  check(hsvd_cu_result_sigma(res, s.data()));
  hsvd_cu_result_free(res);
  // normalize_signs (svd_factor.cpp:86-104): largest |u_ij| of each column > 0
  for (int64_t j = 0; j < k; ++j) {
    int64_t imax = 0;
    for (int64_t i = 1; i < m; ++i)
      if (std::fabs(u[i * k + j]) > std::fabs(u[imax * k + j])) imax = i;
    if (u[imax * k + j] < 0.0) {
      for (int64_t i = 0; i < m; ++i) u[i * k + j] = -u[i * k + j];
      for (int64_t i = 0; i < n; ++i) v[i * k + j] = -v[i * k + j];
    }
  }
  std::printf("rank %lld\n", (long long)k);
  std::printf("sigma:");
  for (int64_t j = 0; j < std::min<int64_t>(k, 10); ++j)
    std::printf(" %s", num(s[(size_t)j], precise).c_str());
  std::printf("\n");
  if (!prefix.empty()) {
    save_hsvd1(prefix + "_U.hsvd", u, m, k);
    save_hsvd1(prefix + "_S.hsvd", s, k, 1);
    save_hsvd1(prefix + "_V.hsvd", v, n, k);
    std::ofstream csv(prefix + "_sigma.csv", std::ios::trunc);
    if (!csv) throw RuntimeFailure{prefix + "_sigma.csv: cannot open for writing"};
    for (double x : s) csv << shortest(x) << '\n';
    std::printf("wrote %s_{U,S,V}.hsvd and %s_sigma.csv\n", prefix.c_str(), prefix.c_str());
  }
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "--help") == 0 || std::strcmp(argv[1], "-h") == 0) {
    std::fputs(kHelp, argc < 2 ? stderr : stdout);
    return argc < 2 ? kUsage : kOk;
  }
  try {
    if (std::strcmp(argv[1], "svd") == 0) return run_svd(argc, argv);
    throw UsageError{std::string("unknown subcommand '") + argv[1] + "'"};
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\n", e.what.c_str());
    return kUsage;
  } catch (const RuntimeFailure& e) {
    std::fprintf(stderr, "error: %s\n", e.what.c_str());
    return kRuntime;
  }
}
