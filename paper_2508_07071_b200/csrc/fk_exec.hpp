// fk_exec.hpp — executors over the device program (fk_exec.cu).
#pragma once

#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "fk_core.hpp"

namespace fk {

void check_config(const fk_exec_config* c);                               // executor.cpp:20-25
fk_exec_report execute_fused(const Pipeline& p, const fk_exec_config* cfg);   // executor.cpp:63-85
fk_exec_report execute_unfused(const Pipeline& p, const fk_exec_config* cfg); // executor.cpp:134-217
uint64_t launch_count();

// ReduceDPP (dpp.hpp:37-53): one traversal of `read` per kMaxReduceSpecs specs
struct ReduceSpecHost {
  const Op* transform = nullptr;  // Unary/Binary compute op or null
  uint32_t combine = FK_REDUCE_SUM;
  bool has_identity = false;
  Element identity;
};
std::vector<Element> multi_reduce(const Op& read, const std::vector<ReduceSpecHost>& specs, int workers,
                                  cudaStream_t st, uint64_t* elements_read);
const char* last_kernel();  // kernel family of this thread's last fused execute
std::string device_info();

}  // namespace fk
