// Shared plumbing of the C++ drop-in API (cxx_api.cpp, cxx_stages.cpp): the process-wide context
// the per-call functions run on, and the status -> exception mapping of the reference
// (std::invalid_argument / std::out_of_range / std::runtime_error).
#pragma once

#include <vector>

#include "opcount.hpp"
#include "tpo/irreps.hpp"
#include "tpo_capi.h"

namespace tpo {
namespace internal {
tpo_ctx* ctx();
extern int g_dev;
void rethrow(int status);
std::vector<tpo_b200::opcount::Entry> entries_of(const Irreps& ir);
}  // namespace internal
}  // namespace tpo
