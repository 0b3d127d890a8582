// fk_core.hpp — host-side IOp model of the B200 Fused Kernel Library.
//
// Mirrors the reference's op vocabulary (ops.hpp:15-161, oplib.hpp) with device
// planes: an IOp is an immutable value (op id, signature, params); a Pipeline is
// a validated Read -> Compute* -> Write chain. Validation rules, error codes and
// chain positions are those of validate_chain (ops.cpp:37-82) and the oplib
// builders (oplib.cpp:40-274), so failures surface identically at the C-ABI.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "fk.h"

namespace fk {

// ---------------------------------------------------------------- errors --
// opfuse::Error (errors.hpp:45-66) as a status code: 1 + Errc ordinal.
class Error : public std::runtime_error {
 public:
  Error(fk_status st, const std::string& msg, int pos = -1)
      : std::runtime_error(msg), status(st), position(pos) {}
  fk_status status;
  int position;
};
const char* errc_name(fk_status st);
[[noreturn]] void fail(fk_status st, const std::string& detail, int pos = -1);

// ----------------------------------------------------------------- kinds --
constexpr bool kind_ok(uint32_t k) { return k <= FK_F64X3; }
constexpr uint32_t bpe(uint32_t k) {  // scalar.hpp:27-37
  constexpr uint32_t b[] = {1, 4, 8, 3, 12, 24};
  return b[k];
}
constexpr int lanes_of(uint32_t k) { return k >= FK_U8X3 ? 3 : 1; }
constexpr uint32_t lane_kind(uint32_t k) { return k >= FK_U8X3 ? k - 3 : k; }
constexpr uint32_t packed_kind(uint32_t k) { return k < FK_U8X3 ? k + 3 : k; }
constexpr uint32_t lane_bytes(uint32_t k) { return bpe(lane_kind(k)); }
const char* kind_name(uint32_t k);
const char* op_name(uint32_t id);

// Element, scalar.hpp:94-121
struct Element {
  uint8_t raw[24] = {};
};
double lane_as_double(uint32_t kind, const Element& e, int lane);

// ----------------------------------------------------------------- model --
struct Folded { uint32_t id, in, out; };  // FoldedUnary, ops.hpp:70-74

struct Sample {  // SampleReadParams, ops.hpp:78-91
  fk_plane source{};
  uint32_t x0 = 0, y0 = 0, rect_w = 0, rect_h = 0, out_w = 0, out_h = 0;
  uint32_t mode = FK_NEAREST;
  std::vector<Folded> post;
  bool resizing() const { return out_w != rect_w || out_h != rect_h; }
  uint32_t output_kind() const { return post.empty() ? source.kind : post.back().out; }
};

struct Op {
  uint32_t id = 0, opkind = 0;
  int32_t in_kind = -1, out_kind = -1;
  std::optional<fk_extent3> dims;
  // Arith / StaticLoop (ops.hpp:93-102)
  Element value;
  uint32_t inner_id = 0, value_kind = 0, repeat = 1;
  // BatchArith extension: one Element per z
  std::vector<Element> values;
  // sample reads / BatchRead (ops.hpp:108-112)
  Sample sample;
  std::vector<Sample> planes;
  uint32_t active = 0;
  Element def;
  // writes (ops.hpp:104-123): dest[0] or dest[0..2]; BatchWrite: wdest[z*per + l]
  std::array<fk_plane, 3> dest{};
  uint32_t w_inner = 0;
  std::vector<fk_plane> wdest;
};

bool is_sample_read(const Op& op);

// builders (oplib.cpp)
Op make_arith(uint32_t id, uint32_t kind, const void* value);
Op make_batch_arith(uint32_t id, uint32_t kind, const void* values, uint32_t n);
Op make_cast(uint32_t from, uint32_t to);
Op make_static_loop(const Op& inner, uint32_t repeat);
Op make_read_per_thread(const fk_plane& src);
Op make_write_per_thread(const fk_plane& dst);
Op make_crop(const fk_plane& src, const fk_crop_rect& r);
Op make_resize(const Op& up, uint32_t w, uint32_t h, uint32_t mode);
Op make_color_convert(uint32_t order, uint32_t in);
Op make_split_write(const fk_plane dst[3]);
Op make_batch_read(const std::vector<const Op*>& inner, uint32_t active, const void* def);
Op make_batch_write(const std::vector<const Op*>& inner, uint32_t active);
Op fold_unary_into_read(const Op& read, const Op& unary);
void check_plane(const fk_plane* p, const char* what);

// ------------------------------------------------------------- pipeline --
struct DeviceProgram;  // uploaded device-side form (fk_exec.cu)

struct Pipeline {
  Op read;
  std::vector<Op> compute;
  Op write;
  fk_extent3 space{};
  // device-side programs, one per CUDA device, each built and uploaded once on
  // the first execute on that device (the paper's "compute the CPU part once",
  // PAPER.md:701-703) and kept for the pipeline's lifetime: executes on other
  // devices never replace it (guarded by fk_exec.cu's build mutex)
  std::map<int, std::shared_ptr<DeviceProgram>> dev;
  ~Pipeline();
};

Pipeline validate_chain(const std::vector<const Op*>& ops);  // ops.cpp:37-82

// Per-plane read/write views of a pipeline, batch or not.
uint32_t read_count(const Pipeline& p);
const Sample* read_plane(const Pipeline& p, uint32_t z);  // nullptr -> default value
uint32_t write_active(const Pipeline& p);

// Analytic ExecReport counters, same accounting as the reference executor
// (ops.cpp:327-344,396-424; executor.cpp:120-130,174-175).
struct Traffic {
  uint64_t fused_read = 0, fused_written = 0;
  uint64_t unfused_read = 0, unfused_written = 0, intermediates = 0;
};
Traffic analytic_traffic(const Pipeline& p);

}  // namespace fk
