// Drop-in mirror of proj/include/tpo/mtp.hpp (product entry points).
#pragma once

#include <vector>

#include "tpo/irreps.hpp"

namespace tpo {

enum class MtpImpl { naive, sparse };

// proj/src/mtp.cpp:94-97
int mtp_l_tilde(int L1, int L2, int L3);

// proj/include/tpo/mtp.hpp:17-37: the stages of mtp, batched on the GPU (tpo_mtp_embed_f32,
// tpo_mtp_extract_f32, tpo_mtp_matmul_f32); carriers are dt x dt Matrix, dt = 2 l_tilde + 1
Matrix mtp_embed(const IrrepVector& x, int l_tilde, MtpImpl impl = MtpImpl::sparse, OpCounter* ops = nullptr);
IrrepVector mtp_extract(const Matrix& Z, int L3, int l_tilde, MtpImpl impl = MtpImpl::sparse,
                        OpCounter* ops = nullptr);
IrrepVector mtp_extract_select(const Matrix& Z, const std::vector<int>& degrees, int l_tilde,
                               MtpImpl impl = MtpImpl::sparse, OpCounter* ops = nullptr);
Matrix mtp_matmul(const Matrix& X, const Matrix& Y, OpCounter* ops = nullptr);

// proj/include/tpo/mtp.hpp:45-49 (host, table-time)
double mtp_path_weights(int l1, int l2, int l3, int l_tilde);

// proj/include/tpo/mtp.hpp:41-43 -- throws std::invalid_argument when
// l_tilde_override is below the minimal carrier degree
IrrepVector mtp(const IrrepVector& x, const IrrepVector& y, int L3, MtpImpl impl = MtpImpl::sparse,
                OpCounter* ops = nullptr, int l_tilde_override = -1);

}  // namespace tpo
