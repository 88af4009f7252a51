// Drop-in mirror of proj/include/tpo/cgtp.hpp.  Computation runs on the B200
// through libtpo_b200.so (C ABI: include/tpo_capi.h); fp64 in/out, fp32 on
// the device (normwise relative error <= 1e-5 vs the fp64 reference).
#pragma once

#include <vector>

#include "tpo/irreps.hpp"

namespace tpo {

struct Path {
  int l1 = 0, l2 = 0, l3 = 0;
  bool valid() const;
  friend bool operator==(const Path&, const Path&) = default;
};

struct PathTable {
  std::vector<Path> paths;
  Irreps output_irreps() const;
};

// proj/src/cgtp.cpp:91-98
PathTable valid_paths(int L1, int L2, int L3);

// proj/include/tpo/cgtp.hpp:35-45 (x, y, out are bare degree slices)
void cgtp_path_naive(const Path& p, const std::vector<double>& x, const std::vector<double>& y,
                     std::vector<double>& out, OpCounter* ops = nullptr);
void cgtp_path_sparse(const Path& p, const std::vector<double>& x, const std::vector<double>& y,
                      std::vector<double>& out, OpCounter* ops = nullptr);

enum class CgtpImpl { naive, sparse };

// proj/include/tpo/cgtp.hpp:52-54 -- throws std::invalid_argument on mul != 1
IrrepVector cgtp_mimo(const IrrepVector& x, const IrrepVector& y, CgtpImpl impl = CgtpImpl::sparse,
                      OpCounter* ops = nullptr);

}  // namespace tpo
