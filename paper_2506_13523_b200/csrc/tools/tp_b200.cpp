// tp_b200: the reference CLI's `run` and `bench` subcommands on the GPU
// (SURVEY 8(f) f3), built on the C++ drop-in API (include/tpo/*.hpp) and the
// batched C ABI (include/tpo_capi.h).
//
//   tp_b200 run   --kind cgtp|gtp|mtp --impl <impl> --L N [--seed S] [--digits D]
//       same inputs (mt19937_64(seed), IrrepVector::random x then y over
//       single_copies(L)) and the same "vector,entry,l,m,value" rows as
//       `tp run` (proj/tools/tp_main.cpp:100-134); the product runs on the GPU.
//   tp_b200 bench [--kinds cgtp,gtp,mtp] [--L 4,6,8 | a..b] [--batch B]
//                 [--warmup W] [--repeats R] [--seed S]
//       rows in the `tp bench` CSV schema (proj/src/bench.cpp:166-181),
//       mode mimo, impl = "b200-<reference impl restated>"; one batched launch
//       per timed run, device time (CUDA events would need the runtime here, so
//       the wall clock of the synchronous host-buffer call is reported,
//       H2D + kernel + D2H included, like the reference's whole-batch clock);
//       ops = multiplies of the GPU algorithm per application (dense GEMM MACs
//       for grid / Fourier / MTP embed+extract, CG nonzeros for CGTP), not the
//       reference's instrumented count; expressivity as
//       proj/src/expressivity.cpp:156-166.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "tpo/cgtp.hpp"
#include "tpo/gtp.hpp"
#include "tpo/irreps.hpp"
#include "tpo/mtp.hpp"
#include "tpo_capi.h"

namespace {

std::string fmt_g(double v, int digits) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.*g", digits, v);
  return buf;
}

std::vector<int> parse_l_list(const std::string& text) {  // "4..16", "4,6,8" or both
  std::vector<int> out;
  size_t pos = 0;
  while (pos <= text.size()) {
    const size_t comma = std::min(text.find(',', pos), text.size());
    const std::string tok = text.substr(pos, comma - pos);
    const size_t dots = tok.find("..");
    if (dots != std::string::npos) {
      const int a = std::stoi(tok.substr(0, dots)), b = std::stoi(tok.substr(dots + 2));
      if (a > b) throw std::invalid_argument("--L: empty range");
      for (int l = a; l <= b; ++l) out.push_back(l);
    } else {
      out.push_back(std::stoi(tok));
    }
    pos = comma + 1;
  }
  if (out.empty()) throw std::invalid_argument("--L: no band limits given");
  return out;
}

std::vector<std::string> split_csv(const std::string& text) {
  std::vector<std::string> out;
  size_t pos = 0;
  while (pos <= text.size()) {
    const size_t comma = std::min(text.find(',', pos), text.size());
    out.push_back(text.substr(pos, comma - pos));
    pos = comma + 1;
  }
  return out;
}

void print_vector(std::ostream& os, const char* name, const tpo::IrrepVector& v, int digits) {
  const auto& entries = v.irreps.entries();
  for (int e = 0; e < v.irreps.num_entries(); ++e) {
    const int l = entries[e].l;
    for (int c = 0; c < entries[e].mul; ++c) {
      const int off = v.irreps.offset(e, c);
      for (int m = -l; m <= l; ++m)
        os << name << ',' << e << ',' << l << ',' << m << ',' << fmt_g(v.data[off + m + l], digits) << '\n';
    }
  }
}

long expressivity_count(const std::string& kind, int L) {  // proj/src/expressivity.cpp:156-166
  if (kind == "cgtp") {
    long n = 0;
    for (int l1 = 0; l1 <= L; ++l1)
      for (int l2 = 0; l2 <= L; ++l2) n += 2 * std::min(l1, l2) + 1;
    return n;
  }
  return 4L * L + 1;
}

// multiplies per application of the GPU algorithm (mimo, L3 = 2L)
unsigned long long gpu_ops(const std::string& kind, const std::string& impl, int L) {
  const unsigned long long din = (L + 1ull) * (L + 1ull), dout = (2ull * L + 1) * (2ull * L + 1);
  if (kind == "gtp") {
    const unsigned long long G = impl == "grid" ? (2ull * L + 1) * (4ull * L + 1) : (4ull * L + 1) * (4ull * L + 1);
    return G * (2 * din + dout);
  }
  if (kind == "mtp") {
    const unsigned long long dt = 2ull * L + 1;
    return dt * dt * 2 * din + dt * dt * dt + dout * dt * dt;
  }
  unsigned long long nnz = 0;  // cgtp: real-CG nonzeros over all paths
  for (int l1 = 0; l1 <= L; ++l1)
    for (int l2 = 0; l2 <= L; ++l2)
      for (int l3 = std::abs(l1 - l2); l3 <= l1 + l2; ++l3) {
        const int n = tpo_cg_real(l1, l2, l3, nullptr, nullptr, nullptr, nullptr, 0);
        if (n < 0) throw std::runtime_error(tpo_last_error());
        nnz += static_cast<unsigned long long>(n);
      }
  return 2 * nnz;
}

int kind_code(const std::string& kind, const std::string& impl) {
  if (kind == "cgtp") return TPO_KIND_CGTP;
  if (kind == "mtp") return TPO_KIND_MTP;
  if (kind == "gtp") return impl == "fourier" ? TPO_KIND_GTP_FOURIER : TPO_KIND_GTP_GRID;
  throw std::invalid_argument("unknown kind '" + kind + "'");
}

std::string arg(int argc, char** argv, const std::string& name, const std::string& def) {
  for (int i = 2; i + 1 < argc; ++i)
    if (name == argv[i]) return argv[i + 1];
  return def;
}

int cmd_run(int argc, char** argv) {
  const std::string kind = arg(argc, argv, "--kind", "gtp"), impl = arg(argc, argv, "--impl", "grid");
  const int L = std::stoi(arg(argc, argv, "--L", "2"));
  const std::uint64_t seed = std::stoull(arg(argc, argv, "--seed", "20240901"));
  const int digits = std::stoi(arg(argc, argv, "--digits", "17"));
  const bool gtp_impl = impl == "grid" || impl == "fourier";
  if ((kind == "gtp") != gtp_impl && !(kind != "gtp" && (impl == "naive" || impl == "sparse")))
    throw std::invalid_argument("--impl '" + impl + "' does not apply to " + kind);
  std::mt19937_64 rng(seed);
  const tpo::Irreps in = tpo::Irreps::single_copies(L);
  const tpo::IrrepVector x = tpo::IrrepVector::random(in, rng);
  const tpo::IrrepVector y = tpo::IrrepVector::random(in, rng);
  tpo::IrrepVector out;
  if (kind == "cgtp")
    out = tpo::cgtp_mimo(x, y, impl == "naive" ? tpo::CgtpImpl::naive : tpo::CgtpImpl::sparse);
  else if (kind == "gtp")
    out = impl == "grid" ? tpo::gtp_grid(x, y, 2 * L) : tpo::gtp_fourier(x, y, 2 * L);
  else if (kind == "mtp")
    out = tpo::mtp(x, y, 2 * L, impl == "naive" ? tpo::MtpImpl::naive : tpo::MtpImpl::sparse);
  else
    throw std::invalid_argument("unknown kind '" + kind + "'");
  std::cout << "vector,entry,l,m,value\n";
  print_vector(std::cout, "x", x, digits);
  print_vector(std::cout, "y", y, digits);
  print_vector(std::cout, "out", out, digits);
  return 0;
}

int cmd_bench(int argc, char** argv) {
  const auto kinds = split_csv(arg(argc, argv, "--kinds", "cgtp,gtp,mtp"));
  const auto Ls = parse_l_list(arg(argc, argv, "--L", "4,6,8"));
  const long batch = std::stol(arg(argc, argv, "--batch", "65536"));
  const int warmup = std::stoi(arg(argc, argv, "--warmup", "2")), repeats = std::stoi(arg(argc, argv, "--repeats", "7"));
  const std::uint64_t seed = std::stoull(arg(argc, argv, "--seed", "20240901"));
  if (warmup < 1 || repeats < 5 || batch < 1) throw std::invalid_argument("warmup >= 1, repeats >= 5, batch >= 1");
  tpo_ctx* ctx = nullptr;
  if (tpo_ctx_create(0, &ctx)) throw std::runtime_error(tpo_last_error());
  std::cout << "kind,impl,mode,L,batch,ops,time_med_ns,time_min_ns,time_max_ns,"
               "expressivity,ops_per_expr,time_per_expr_ns\n";
  std::mt19937_64 rng(seed);
  std::normal_distribution<float> nd;
  for (const std::string& kind : kinds) {
    const std::vector<std::string> impls =
        kind == "gtp" ? std::vector<std::string>{"grid", "fourier"} : std::vector<std::string>{"sparse"};
    for (const std::string& impl : impls)
      for (int L : Ls) {
        const long din = (L + 1L) * (L + 1L);
        const long dout = kind == "cgtp" ? din * din : (2L * L + 1) * (2L * L + 1);
        std::vector<float> x(static_cast<size_t>(batch * din)), y(x.size()), out(static_cast<size_t>(batch * dout));
        for (auto& v : x) v = nd(rng);
        for (auto& v : y) v = nd(rng);
        const int kc = kind_code(kind, impl);
        const int L3 = kind == "cgtp" ? 0 : 2 * L;
        auto once = [&] {
          if (tpo_run_host_f32(ctx, kc, L, L, L3, -1, x.data(), y.data(), out.data(), batch, 1, 0))
            throw std::runtime_error(tpo_last_error());
        };
        for (int w = 0; w < warmup; ++w) once();
        std::vector<unsigned long long> ns(static_cast<size_t>(repeats));
        for (auto& t : ns) {
          const auto t0 = std::chrono::steady_clock::now();
          once();
          t = static_cast<unsigned long long>(
              std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count());
        }
        std::sort(ns.begin(), ns.end());
        const unsigned long long ops = gpu_ops(kind, impl, L);
        const long ex = expressivity_count(kind, L);
        std::cout << kind << ",b200-" << impl << ",mimo," << L << ',' << batch << ',' << ops << ','
                  << ns[ns.size() / 2] << ',' << ns.front() << ',' << ns.back() << ',' << ex << ','
                  << fmt_g(static_cast<double>(ops) / ex, 17) << ','
                  << fmt_g(static_cast<double>(ns[ns.size() / 2]) / ex, 17) << '\n';
      }
  }
  tpo_ctx_destroy(ctx);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "run") return cmd_run(argc, argv);
    if (cmd == "bench") return cmd_bench(argc, argv);
    std::cerr << "usage: tp_b200 run --kind K --impl I --L N [--seed S] [--digits D]\n"
                 "       tp_b200 bench [--kinds cgtp,gtp,mtp] [--L 4,6,8] [--batch B] [--warmup W] [--repeats R]\n";
    return 2;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
