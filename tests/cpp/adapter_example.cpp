// Compiled by tests/test_cpp_adapter.py against libfk_oracle.so (CPU) and, on a
// GPU box, libfk_cuda.so: the reference-style C++ spelling over the C-ABI.
#include <cstdio>
#include <vector>

#include "opfuse_fk.hpp"

using namespace opfuse_fk;

int main() {
  // host buffers for the oracle backend; the CUDA build passes device pointers
  std::vector<float> src(60 * 40);
  for (size_t i = 0; i < src.size(); ++i) src[i] = float(i % 97) / 97.0f;
  std::vector<unsigned char> dst(60 * 40);
  Plane s{src.data(), 60, 40, 60, FK_F32}, d{dst.data(), 60, 40, 60, FK_U8};
  Pipeline p = validate_chain({op_read_per_thread(s), op_mul(400.0f), op_add(2.0f), op_sub(1.5f), op_div(1.25f),
                               op_cast(FK_F32, FK_U8), op_write_per_thread(d)});
  ExecReport r = execute_fused(p);
  long sum = 0;
  for (unsigned char v : dst) sum += v;
  try {
    validate_chain({op_read_per_thread(s), op_mul(uint8_t(3)), op_write_per_thread(d)});
  } catch (const Error& e) {
    std::printf("errc=%d pos=%d\n", e.errc(), e.position);
  }
  std::printf("passes=%llu sum=%ld savings=%llu\n", (unsigned long long)r.passes, sum,
              (unsigned long long)plan_memory_savings(p));
  return 0;
}
