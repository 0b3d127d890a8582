// opfuse_fk.hpp — header-only C++17 adapter that gives existing opfuse
// pipelines (reference: /root/reference/proj/include/opfuse/{oplib,ops,executor}.hpp)
// the same spelling over the fk.h C-ABI. Link against libfk_cuda.so (device
// planes) — or libfk_oracle.so in CPU-only tests.
//
//   using namespace opfuse_fk;
//   Plane src{dev_ptr, 3840, 2160, 3840, FK_F32};
//   Pipeline p = validate_chain({op_read_per_thread(src), op_mul(400.0f), op_add(2.0f),
//                                op_sub(1.5f), op_div(1.25f), op_cast(FK_F32, FK_U8),
//                                op_write_per_thread(dst)});
//   ExecReport r = execute_fused(p, cfg);
//
// Errors throw opfuse_fk::Error carrying the reference Errc (status - 1) and the
// chain position, as opfuse::Error does (errors.hpp:45-66).
#pragma once

#include <array>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fk.h"

namespace opfuse_fk {

class Error : public std::runtime_error {
 public:
  Error(fk_status st, const char* msg, int pos) : std::runtime_error(msg), status(st), position(pos) {}
  int errc() const { return status - 1; }  // reference Errc ordinal (errors.hpp:9-38)
  fk_status status;
  int position;
};

inline void check(fk_status st) {
  if (st != FK_OK) throw Error(st, fk_last_error(), fk_last_error_position());
}

using Plane = fk_plane;          // device view: data, width, height, row_stride (elements), kind
using ExecConfig = fk_exec_config;
using ExecReport = fk_exec_report;
using CropRect = fk_crop_rect;

inline ExecConfig default_config() { return ExecConfig{0, 8, 8, 0, nullptr}; }  // executor.hpp:10-14

class IOp {  // ops.hpp:131-153
 public:
  explicit IOp(fk_iop* p = nullptr) : p_(p, fk_iop_free) {}
  fk_iop* get() const { return p_.get(); }
  uint32_t id() const { return fk_iop_id(get()); }

 private:
  std::shared_ptr<fk_iop> p_;
};

class Pipeline {  // ops.hpp:156-161
 public:
  explicit Pipeline(fk_pipeline* p = nullptr) : p_(p, fk_pipeline_free) {}
  fk_pipeline* get() const { return p_.get(); }
  fk_extent3 iter_space() const {
    fk_extent3 e{};
    check(fk_pipeline_iter_space(get(), &e));
    return e;
  }

 private:
  std::shared_ptr<fk_pipeline> p_;
};

namespace detail {
template <class F, class... A>
IOp make(F f, A... a) {
  fk_iop* out = nullptr;
  check(f(a..., &out));
  return IOp(out);
}
template <class T>
IOp arith(uint32_t op, uint32_t kind, const T* lanes) {
  return make(fk_op_arith, op, kind, static_cast<const void*>(lanes));
}
}  // namespace detail

// oplib.hpp:31-35 — the Const overloads pick the kind
inline IOp make_arith(uint32_t op, float c) { return detail::arith(op, FK_F32, &c); }
inline IOp make_arith(uint32_t op, double c) { return detail::arith(op, FK_F64, &c); }
inline IOp make_arith(uint32_t op, uint8_t c) { return detail::arith(op, FK_U8, &c); }
inline IOp make_arith(uint32_t op, const std::array<float, 3>& c) { return detail::arith(op, FK_F32X3, c.data()); }
inline IOp make_arith(uint32_t op, const std::array<double, 3>& c) { return detail::arith(op, FK_F64X3, c.data()); }
inline IOp make_arith(uint32_t op, const std::array<uint8_t, 3>& c) { return detail::arith(op, FK_U8X3, c.data()); }
template <class T> IOp op_mul(const T& c) { return make_arith(FK_OP_MUL, c); }
template <class T> IOp op_add(const T& c) { return make_arith(FK_OP_ADD, c); }
template <class T> IOp op_sub(const T& c) { return make_arith(FK_OP_SUB, c); }
template <class T> IOp op_div(const T& c) { return make_arith(FK_OP_DIV, c); }

inline IOp op_cast(uint32_t from, uint32_t to) { return detail::make(fk_op_cast, from, to); }                 // :39
inline IOp op_static_loop(const IOp& inner, uint32_t n) {                                                    // :43
  fk_iop* out = nullptr;
  check(fk_op_static_loop(inner.get(), n, &out));
  return IOp(out);
}
inline IOp op_read_per_thread(const Plane& src) { return detail::make(fk_op_read_per_thread, &src); }       // :46
inline IOp op_write_per_thread(const Plane& dst) { return detail::make(fk_op_write_per_thread, &dst); }     // :47
inline IOp op_crop(const Plane& src, const CropRect& r) { return detail::make(fk_op_crop, &src, &r); }      // :50
inline IOp op_resize(const IOp& up, uint32_t w, uint32_t h, uint32_t mode = FK_BILINEAR) {                  // :54-57
  fk_iop* out = nullptr;
  check(fk_op_resize(up.get(), w, h, mode, &out));
  return IOp(out);
}
inline IOp op_resize(const Plane& src, uint32_t w, uint32_t h, uint32_t mode = FK_BILINEAR) {
  return op_resize(op_read_per_thread(src), w, h, mode);
}
inline IOp op_color_convert(uint32_t order, uint32_t in) { return detail::make(fk_op_color_convert, order, in); }  // :60
inline IOp op_split_write(const std::array<Plane, 3>& d) { return detail::make(fk_op_split_write, d.data()); }    // :63
inline IOp op_batch_read(const std::vector<IOp>& inner, uint32_t active, const void* def = nullptr) {          // :68
  std::vector<const fk_iop*> v;
  for (const IOp& i : inner) v.push_back(i.get());
  fk_iop* out = nullptr;
  check(fk_op_batch_read(v.data(), uint32_t(v.size()), active, def, &out));
  return IOp(out);
}
inline IOp op_batch_read(const std::vector<IOp>& inner) { return op_batch_read(inner, uint32_t(inner.size())); }
inline IOp op_batch_write(const std::vector<IOp>& inner, uint32_t active) {                                    // :71
  std::vector<const fk_iop*> v;
  for (const IOp& i : inner) v.push_back(i.get());
  fk_iop* out = nullptr;
  check(fk_op_batch_write(v.data(), uint32_t(v.size()), active, &out));
  return IOp(out);
}
inline IOp op_batch_write(const std::vector<IOp>& inner) { return op_batch_write(inner, uint32_t(inner.size())); }
inline IOp fold_unary_into_read(const IOp& read, const IOp& unary) {                                           // :76
  fk_iop* out = nullptr;
  check(fk_fold_unary_into_read(read.get(), unary.get(), &out));
  return IOp(out);
}

inline Pipeline validate_chain(const std::vector<IOp>& ops) {  // ops.hpp:171
  std::vector<const fk_iop*> v;
  for (const IOp& i : ops) v.push_back(i.get());
  fk_pipeline* out = nullptr;
  check(fk_validate_chain(v.data(), uint32_t(v.size()), &out));
  return Pipeline(out);
}

inline ExecReport execute_fused(const Pipeline& p, const ExecConfig& cfg = default_config()) {  // executor.hpp:40
  ExecReport r{};
  check(fk_execute_fused(p.get(), &cfg, &r));
  return r;
}
inline ExecReport execute_unfused(const Pipeline& p, const ExecConfig& cfg = default_config()) {  // :51
  ExecReport r{};
  check(fk_execute_unfused(p.get(), &cfg, &r));
  return r;
}
inline uint64_t plan_memory_savings(const Pipeline& p) {  // :55
  uint64_t b = 0;
  check(fk_plan_memory_savings(p.get(), &b));
  return b;
}

}  // namespace opfuse_fk
