// fk_exec.hpp — executors over the device program (fk_exec.cu).
#pragma once

#include <string>

#include "fk_core.hpp"

namespace fk {

void check_config(const fk_exec_config* c);                               // executor.cpp:20-25
fk_exec_report execute_fused(const Pipeline& p, const fk_exec_config* cfg);   // executor.cpp:63-85
fk_exec_report execute_unfused(const Pipeline& p, const fk_exec_config* cfg); // executor.cpp:134-217
uint64_t launch_count();
const char* last_kernel();  // kernel family of this thread's last fused execute
std::string device_info();

}  // namespace fk
