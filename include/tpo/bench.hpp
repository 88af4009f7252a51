// Drop-in mirror of the counting part of proj/include/tpo/bench.hpp (and the Kind enum of
// proj/include/tpo/expressivity.hpp): count_ops, the reference's instrumented multiply count of one
// application, computed from the same structural rules (csrc/host/opcount.cpp).  The timing
// harness itself (time_tpo / sweep / write_csv) is the reference CLI's, mirrored by tp_b200.
#pragma once

#include <cstdint>

namespace tpo {

enum class Kind { cgtp, gtp, mtp };
enum class BenchImpl { naive, sparse, grid, fourier };
enum class BenchMode { siso, simo, mimo };

struct BenchSetting {
  BenchMode mode = BenchMode::mimo;
  int L = 1;
  int batch = 1;
};

const char* impl_name(BenchImpl i);
const char* mode_name(BenchMode m);
bool impl_applies(Kind kind, BenchImpl impl);

// siso: the single path [L, L, L]; simo: degree-L inputs, outputs l3 <= 2L; mimo: single_copies(L)
// inputs, full output band (proj/include/tpo/bench.hpp:40-45).  Throws std::invalid_argument.
std::uint64_t count_ops(Kind kind, BenchImpl impl, const BenchSetting& s);

}  // namespace tpo
