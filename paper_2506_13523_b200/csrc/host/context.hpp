// tpo_ctx: per-device context owning device-resident tables (built lazily
// per shape, cached for the context lifetime like the reference's memo
// caches, proj/src/wigner.cpp:64-81 / proj/src/gtp.cpp:25-32,183-195) and
// scratch buffers for the host-pointer entry points.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <functional>
#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kernels/kernels.hpp"

namespace tpo_b200 {

// error types mapped to TPO_* status codes by capi.cpp
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

// Device the calling thread had current before the first Context::activate() of the running C-ABI
// call (-1: untouched); the C-ABI wrapper restores it when the call returns, so an entry point never
// leaves the caller's current device switched.
int& caller_device();

// 2-D TMA tensor map (driver cuTensorMapEncodeTiled through the runtime's entry point)
void encode_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw);

struct GridTcEntry {
  bool fits = false;
  GridTcTables t{};
};

class Context {
 public:
  explicit Context(int device);
  ~Context();

  int device() const { return device_; }
  int num_sms() const { return num_sms_; }
  void activate() const;

  const CgtpTables& cgtp(int L1, int L2);
  // backward term tables (wrt 0: grad_x, 1: grad_y), cgtp_bwd.cu
  const CgtpBwdTables& cgtp_bwd(int L1, int L2, int wrt);
  const CgtpTcTables* cgtp_tc(int L1, int L2);  // nullptr: shape not on the tcgen05 block path
  const CgtpBwdTcTables* cgtp_bwd_tc(int L1, int L2);  // nullptr: backward shape not on tcgen05
  const GridTcEntry& grid_tc(int L1, int L2, int L3);
  // forward with inputs past the K limit: x degrees [a1, b1] x y degrees [a2, b2] of the full operators
  const GridTcEntry& dense_split_tc(int fourier, int L1, int L2, int L3, int a1, int b1, int a2, int b2);
  // backward: grad_out degrees [a, b] x tower L2 -> tower Lo, smallest exact grid
  const GridTcEntry& grid_tc_part(int a, int b, int L2, int Lo);
  const GridTcEntry& fourier_tc(int L1, int L2, int L3);  // Fourier GTP as torus-grid dense operators
  // small-degree SIMT operators (gtp_small.cu); nullptr when the shape has no instantiation
  const GtpSmallOps* gtp_small(int fourier, int L1, int L2, int L3);
  const GridSimtTables& grid_simt(int L1, int L2, int L3);
  // Fourier GTP on the row-quad separable kernel (the reference torus folded to theta in [0, pi]);
  // nullptr when the encode / decode spectra do not separate (never for the reference's tables)
  const GridSimtTables* fourier_sep(int L1, int L2, int L3);
  const FourierDevTables& fourier(int L1, int L2, int L3);
  const MtpDevTables& mtp(int L1, int L2, int L3, int lt);
  // nullptr: shape not on the tcgen05 path; a1 / flags: backward variants (context.cpp)
  const MtpTcTables* mtp_tc(int L1, int L2, int L3, int lt, int a1 = 0, int flags = 0);
  const float* degree_weights(const std::vector<double>& w);  // small per-call device array
  // device fp32 copy of a k-major stage operator (stages.cu dense_map), built once per key
  const float* dense_op(const std::string& key, const std::function<std::vector<double>()>& build);
  // device copy of a small int table, built once per key
  const int* int_table(const std::string& key, const std::function<std::vector<int>()>& build);
  // Wigner-D recursion tables up to degree L (stages.cu wigner_d)
  const WignerTables& wigner(int L);

  // scratch for host entry points / weighted products (grown on demand)
  float* scratch(int slot, size_t floats);
  cudaStream_t host_stream() const { return host_stream_; }
  // pipelined host-buffer path: copy-in / copy-out streams and per-buffer events
  static constexpr int kPipeBufs = 3;
  static constexpr int kScratchMisc = 3 * kPipeBufs;
  cudaStream_t h2d_stream() const { return h2d_stream_; }
  cudaStream_t d2h_stream() const { return d2h_stream_; }
  cudaEvent_t pipe_event(int which, int buf) const { return pipe_ev_[which][buf]; }
  std::mutex& host_path_mutex() { return host_mu_; }

  std::atomic<int64_t> launches{0};
  std::atomic<int> grid_path{0};       // 0 auto, 1 tcgen05, 2 simt, 3 separable (grid and Fourier GTP)
  std::atomic<int> last_grid_path{0};  // diagnostics: path of the most recent GTP call on this context
  // 0 default: GEMM-2 accumulation segments past the per-operator chain limits (<= 6.8e-6 normwise
  // on adversarial rows); 1 strict: segments past 20 K-steps everywhere (<= ~4e-6, slower at L >= 8)
  std::atomic<int> precision_mode{0};

 private:
  template <class T>
  T* upload(const std::vector<T>& v);
  void* dev_alloc(size_t bytes);

  int device_ = 0;
  int num_sms_ = 148;
  cudaStream_t host_stream_ = nullptr;
  cudaStream_t h2d_stream_ = nullptr, d2h_stream_ = nullptr;
  cudaEvent_t pipe_ev_[3][kPipeBufs] = {};  // [h2d done, compute done, d2h done][buffer]
  std::mutex host_mu_;
  std::mutex mu_;
  std::vector<void*> allocs_;
  std::map<std::array<int, 2>, CgtpTables> cgtp_;
  std::map<std::array<int, 3>, CgtpBwdTables> cgtp_bwd_;
  CgtpTables pack_cgtp(const std::vector<std::vector<std::pair<uint32_t, float>>>& per_out, int din1, int din2);
  std::map<std::array<int, 2>, std::pair<bool, CgtpTcTables>> cgtp_tc_;
  std::map<std::array<int, 2>, std::pair<bool, CgtpBwdTcTables>> cgtp_bwd_tc_;
  std::map<std::array<int, 4>, GridTcEntry> grid_tc_;
  struct SmallEntry {
    bool ok = false;
    GtpSmallOps o;
    std::vector<float> s, a;
  };
  std::map<std::array<int, 4>, SmallEntry> gtp_small_;
  std::map<std::array<int, 4>, GridTcEntry> grid_tc_part_;
  std::map<std::array<int, 8>, GridTcEntry> dense_split_;
  std::map<std::array<int, 4>, GridTcEntry> fourier_tc_;
  GridTcEntry build_dense_tc(const struct DenseOps& ops, const char* label, int max_chain);
  std::map<std::array<int, 3>, GridSimtTables> grid_simt_;
  std::map<std::array<int, 3>, std::unique_ptr<GridSimtTables>> fourier_sep_;
  void fill_sep_tables(GridSimtTables& t, int np, const std::function<float(int, int)>& lam1_at,
                       const std::function<float(int, int)>& lam5_at);
  std::map<std::array<int, 3>, FourierDevTables> fourier_;
  std::map<std::array<int, 4>, MtpDevTables> mtp_;
  std::map<std::array<int, 6>, std::pair<bool, MtpTcTables>> mtp_tc_;
  std::map<std::vector<double>, const float*> weights_;
  std::map<std::string, const float*> dense_ops_;
  std::map<std::string, const int*> int_tables_;
  std::map<int, WignerTables> wigner_;
  // slots 0 .. 3 kPipeBufs - 1: the host pipeline's x / y / out buffers; kScratchMisc: other uses
  std::array<void*, 3 * kPipeBufs + 1> scratch_{};
  std::array<size_t, 3 * kPipeBufs + 1> scratch_cap_{};
};

}  // namespace tpo_b200
