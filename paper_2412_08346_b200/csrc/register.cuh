// SGD-ICP registration on the device (register.cu): graspmatch::register_sgd_icp
// (optim.cpp:274-321) for a batch of independent problems, one CTA each.
#pragma once

#include "asicp.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace asicp {

class RegBatch {
 public:
  RegBatch(int device, cudaStream_t stream) : device_(device), st_(stream) {}
  ~RegBatch();
  RegBatch(const RegBatch&) = delete;
  RegBatch& operator=(const RegBatch&) = delete;

  // Validation in the reference's order, then upload.  Returns ASICP_OK or
  // ASICP_INVALID_ARGUMENT / ASICP_DEVICE_ERROR with the message in *err.
  int prepare(int64_t n, const double* sources, const int64_t* src_off, const double* references,
              const int64_t* ref_off, const double* initial, const uint64_t* seeds, const asicp_sgd_config& cfg,
              std::string* err);
  // Solve the prepared batch (synchronous).  A pose that leaves the unit
  // sphere mid-run fails the call like the reference's require.
  int run(asicp_registration* out, std::string* err);
  // graspmatch::icp_closed_form_step for n independent problems (synchronous).
  int icp_step(int64_t n, const double* sources, const int64_t* src_off, const double* references,
               const int64_t* ref_off, const double* thetas, asicp_icp_step* out, std::string* err);
  // Device time of the last run's kernel (ms).
  float last_kernel_ms() const { return kernel_ms_; }
  int launches() const { return 1; }

 private:
  struct Dev;
  void release();
  int device_;
  cudaStream_t st_;
  Dev* d_ = nullptr;
  Dev* icp_ = nullptr;
  float kernel_ms_ = 0.0f;
};

double run_dfma_peak(int iters);  // FP64 TFLOP/s (DFMA microbenchmark)

}  // namespace asicp
