// Reference multiply counts (OpCounter semantics) derived from shapes; see opcount.cpp.
#pragma once

#include <cstdint>
#include <vector>

namespace tpo_b200 {
namespace opcount {

struct Entry {
  int mul, l;
};

uint64_t cgtp_path(bool naive, int l1, int l2, int l3);
uint64_t cgtp_mimo(bool naive, const std::vector<int>& xls, const std::vector<int>& yls);
uint64_t to_sphere(const std::vector<Entry>& x, int grid_L);
uint64_t pointwise_mul(int grid_L);
uint64_t from_sphere_select(int grid_L, const std::vector<int>& degrees);
uint64_t gtp_grid_select(const std::vector<Entry>& x, const std::vector<Entry>& y, const std::vector<int>& degrees);
uint64_t gtp_fourier_select(const std::vector<Entry>& x, const std::vector<Entry>& y, const std::vector<int>& degrees);
uint64_t scale_degrees(const std::vector<Entry>& x);
uint64_t mtp_embed(bool naive, const std::vector<Entry>& x, int lt);
uint64_t mtp_matmul(int dt);
uint64_t mtp_extract_select(bool naive, const std::vector<int>& degrees, int lt);
uint64_t mtp(bool naive, const std::vector<Entry>& x, const std::vector<Entry>& y, int L3, int lt);

}  // namespace opcount
}  // namespace tpo_b200
