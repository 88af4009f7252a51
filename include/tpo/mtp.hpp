// Drop-in mirror of proj/include/tpo/mtp.hpp (product entry points).
#pragma once

#include "tpo/irreps.hpp"

namespace tpo {

enum class MtpImpl { naive, sparse };

// proj/src/mtp.cpp:94-97
int mtp_l_tilde(int L1, int L2, int L3);

// proj/include/tpo/mtp.hpp:41-43 -- throws std::invalid_argument when
// l_tilde_override is below the minimal carrier degree
IrrepVector mtp(const IrrepVector& x, const IrrepVector& y, int L3, MtpImpl impl = MtpImpl::sparse,
                OpCounter* ops = nullptr, int l_tilde_override = -1);

}  // namespace tpo
