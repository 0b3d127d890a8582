// opfuse_fk.hpp — header-only C++17 drop-in for the reference's opfuse API
// (/root/reference/proj/include/opfuse/{scalar,plane,ops,oplib,executor,api,
// static_chain}.hpp) over the fk.h C-ABI. Link against libfk_cuda.so (planes in
// device memory, the sm_100a kernels) — or libfk_oracle.so / libfk_ref.so in
// CPU-only tests. With OPFUSE_FK_AS_OPFUSE defined before the include, the
// namespace is also reachable as `opfuse`, so reference code such as
//
//   using namespace opfuse;
//   Plane src = Plane::alloc(3840, 2160, ScalarKind::F32);
//   Pipeline p = validate_chain({op_read_per_thread(src), op_mul(400.0f), op_add(2.0f),
//                                op_sub(1.5f), op_div(1.25f), op_cast(ScalarKind::F32, ScalarKind::U8),
//                                op_write_per_thread(dst)});
//   ExecReport r = execute_fused(p);
//   r = api::execute_operations({api::read(src), api::multiply(2.0f), api::write(dst)});
//   sc::transform(sc::PlaneView<float>(src), sc::PlaneView<float>(dst), 0, sc::Mul<float>{2.0f});
//
// compiles unchanged. Differences a user sees: Plane::alloc returns DEVICE
// memory with the CUDA backend (fill / read it with Plane::upload / download,
// or pass device pointers with Plane::wrap); row() / load() / store() do not
// exist on device planes.
//
// Errors throw opfuse_fk::Error carrying the reference Errc, the chain position
// and the facade's provenance, as opfuse::Error does (errors.hpp:45-66).
#pragma once

#include <array>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "fk.h"

namespace opfuse_fk {

// ------------------------------------------------------------- vocabulary --
enum class ScalarKind : std::uint8_t { U8 = 0, F32 = 1, F64 = 2, U8x3 = 3, F32x3 = 4, F64x3 = 5 };  // scalar.hpp:16-23
enum class ResizeMode : std::uint8_t { Nearest, Bilinear };                                          // ops.hpp:61
enum class ColorOrder : std::uint8_t { SwapRB, ToGrayF32 };                                          // ops.hpp:62
enum class OpKind : std::uint8_t { Read, Unary, Binary, Write };                                     // ops.hpp:15
enum class OpId : std::uint8_t {                                                                     // ops.hpp:17-37
  PerThreadRead, CropRead, ResizeRead, BatchRead, Cast, SwapRB, ToGray, Mul, Add, Sub, Div, StaticLoop,
  PerThreadWrite, SplitWrite, BatchWrite
};
enum class Errc : int {  // errors.hpp:9-38 (status - 1)
  EmptyChain, FirstNotRead, LastNotWrite, KindMismatch, DimsMismatch, MissingDims, ChainTooLong, DivByZeroParam,
  UnsupportedCast, UnsupportedKind, CropOutOfBounds, PlaneExtentMismatch, EmptyBatch, InnerKindMismatch,
  HeterogeneousBatch, BadStaticLoop, BoundsError, CapacityOverflow, BadMagic, UnknownKindTag, TruncatedPayload,
  IoError, EmptyIterSpace, InvalidConfig
};

inline std::uint32_t bytes_per_element(ScalarKind k) { return fk_bytes_per_element(std::uint32_t(k)); }
inline std::uint32_t lane_count(ScalarKind k) { return std::uint8_t(k) >= 3 ? 3u : 1u; }

class Error : public std::runtime_error {  // errors.hpp:45-66
 public:
  Error(fk_status st, const std::string& msg, int pos) : std::runtime_error(msg), status(st), pos_(pos) {}
  Errc code() const { return Errc(status - 1); }
  int errc() const { return status - 1; }  // reference Errc ordinal
  int position() const { return pos_; }
  const std::string& provenance() const { return prov_; }
  void set_provenance(std::string p) { prov_ = std::move(p); }
  fk_status status;

 private:
  int pos_;
  std::string prov_;
};

inline void check(fk_status st) {
  if (st != FK_OK) throw Error(st, fk_last_error(), fk_last_error_position());
}
[[noreturn]] inline void fail(Errc e, const std::string& msg, int pos = -1) {
  throw Error(int(e) + 1, msg, pos);
}

// Element (scalar.hpp:94-121): up to three lanes of the widest kind, raw bytes
struct Element {
  std::uint8_t bytes[24] = {};
  static Element of_u8(std::uint8_t v) { return of(&v, 1); }
  static Element of_f32(float v) { return of(&v, 4); }
  static Element of_f64(double v) { return of(&v, 8); }
  static Element of_u8x3(std::uint8_t a, std::uint8_t b, std::uint8_t c) { std::uint8_t v[3] = {a, b, c}; return of(v, 3); }
  static Element of_f32x3(float a, float b, float c) { float v[3] = {a, b, c}; return of(v, 12); }
  static Element of_f64x3(double a, double b, double c) { double v[3] = {a, b, c}; return of(v, 24); }

 private:
  static Element of(const void* p, std::size_t n) {
    Element e;
    std::memcpy(e.bytes, p, n);
    return e;
  }
};

// Const (oplib.hpp:8-21): the constructor picks the kind
struct Const {
  ScalarKind kind;
  Element value;
  Const(std::uint8_t v) : kind(ScalarKind::U8), value(Element::of_u8(v)) {}
  Const(float v) : kind(ScalarKind::F32), value(Element::of_f32(v)) {}
  Const(double v) : kind(ScalarKind::F64), value(Element::of_f64(v)) {}
  Const(const std::array<std::uint8_t, 3>& v) : kind(ScalarKind::U8x3), value(Element::of_u8x3(v[0], v[1], v[2])) {}
  Const(const std::array<float, 3>& v) : kind(ScalarKind::F32x3), value(Element::of_f32x3(v[0], v[1], v[2])) {}
  Const(const std::array<double, 3>& v) : kind(ScalarKind::F64x3), value(Element::of_f64x3(v[0], v[1], v[2])) {}
};

struct CropRect {  // oplib.hpp:23-26
  std::uint32_t x0 = 0, y0 = 0;
  std::uint32_t w = 0, h = 0;
};

// -------------------------------------------------------------- planes --
// Plane (plane.hpp:60-103): a strided view sharing ownership of its buffer.
// Plane::alloc buffers come from fk_plane_alloc (device memory with the CUDA
// backend); every IOp / pipeline built from the plane or a view keeps the
// buffer alive inside the library too. Plane::wrap views caller memory.
class Plane {
 public:
  Plane() = default;
  static Plane alloc(std::uint32_t w, std::uint32_t h, ScalarKind k) {  // plane.cpp:60-71 (zeroed)
    auto owner = std::make_shared<Owner>();
    check(fk_plane_alloc(w, h, std::uint32_t(k), 0, &owner->p));
    Plane p;
    p.v_ = owner->p;
    p.owner_ = owner;
    return p;
  }
  static Plane alloc_uninitialized(std::uint32_t w, std::uint32_t h, ScalarKind k) { return alloc(w, h, k); }
  static Plane wrap(void* data, std::uint32_t w, std::uint32_t h, std::uint32_t row_stride, ScalarKind k) {
    Plane p;
    p.v_ = fk_plane{data, w, h, row_stride, std::uint32_t(k)};
    return p;
  }
  Plane view(std::uint32_t x0, std::uint32_t y0, std::uint32_t w, std::uint32_t h) const {  // plane.cpp:91-101
    Plane p = *this;
    check(fk_plane_view(&v_, x0, y0, w, h, &p.v_));
    return p;
  }
  std::uint32_t width() const { return v_.width; }
  std::uint32_t height() const { return v_.height; }
  std::uint32_t row_stride() const { return v_.row_stride; }
  ScalarKind kind() const { return ScalarKind(v_.kind); }
  void* data() const { return v_.data; }
  const fk_plane& raw() const { return v_; }
  void upload(const void* host, std::size_t host_pitch = 0) const { check(fk_plane_upload(&v_, host, host_pitch)); }
  void download(void* host, std::size_t host_pitch = 0) const { check(fk_plane_download(&v_, host, host_pitch)); }

 private:
  struct Owner {
    fk_plane p{};
    ~Owner() { fk_plane_free(&p); }
  };
  fk_plane v_{};
  std::shared_ptr<Owner> owner_;
};

// ------------------------------------------------------- IOps, pipelines --
class IOp {  // ops.hpp:131-153
 public:
  explicit IOp(fk_iop* p = nullptr) : p_(p, fk_iop_free) {}
  fk_iop* get() const { return p_.get(); }
  OpId id() const { return OpId(fk_iop_id(get())); }
  OpKind kind() const { return OpKind(fk_iop_kind(get())); }
  std::optional<ScalarKind> input_kind() const {
    const int k = fk_iop_input_kind(get());
    return k < 0 ? std::nullopt : std::optional<ScalarKind>(ScalarKind(k));
  }
  std::optional<ScalarKind> output_kind() const {
    const int k = fk_iop_output_kind(get());
    return k < 0 ? std::nullopt : std::optional<ScalarKind>(ScalarKind(k));
  }

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
  std::size_t compute_count() const { return fk_pipeline_compute_count(get()); }

 private:
  std::shared_ptr<fk_pipeline> p_;
};

struct ExecConfig {  // executor.hpp:10-14 + the device fields
  int workers = 0;
  int coarsening_block = 8;
  int chunk_rows = 8;
  void* stream = nullptr;  // cudaStream_t (CUDA backend)
  std::uint32_t flags = 0;  // FK_EXEC_*
  fk_exec_config raw() const { return fk_exec_config{workers, coarsening_block, chunk_rows, flags, stream}; }
};
using ExecReport = fk_exec_report;  // executor.hpp:27-34 fields + kernels_launched / device_ms / path

namespace detail {
template <class F, class... A>
IOp make(F f, A... a) {
  fk_iop* out = nullptr;
  check(f(a..., &out));
  return IOp(out);
}
inline std::uint32_t u(ScalarKind k) { return std::uint32_t(k); }
}  // namespace detail

// ------------------------------------------------ builders (oplib.hpp:31-76) --
inline IOp make_arith(OpId id, ScalarKind kind, const Element& value) {
  return detail::make(fk_op_arith, std::uint32_t(id), detail::u(kind), static_cast<const void*>(value.bytes));
}
inline IOp op_mul(const Const& c) { return make_arith(OpId::Mul, c.kind, c.value); }
inline IOp op_add(const Const& c) { return make_arith(OpId::Add, c.kind, c.value); }
inline IOp op_sub(const Const& c) { return make_arith(OpId::Sub, c.kind, c.value); }
inline IOp op_div(const Const& c) { return make_arith(OpId::Div, c.kind, c.value); }
inline IOp op_cast(ScalarKind from, ScalarKind to) { return detail::make(fk_op_cast, detail::u(from), detail::u(to)); }
inline IOp op_static_loop(const IOp& inner, std::uint32_t repeat) {
  fk_iop* out = nullptr;
  check(fk_op_static_loop(inner.get(), repeat, &out));
  return IOp(out);
}
inline IOp op_read_per_thread(const Plane& src) { return detail::make(fk_op_read_per_thread, &src.raw()); }
inline IOp op_write_per_thread(const Plane& dst) { return detail::make(fk_op_write_per_thread, &dst.raw()); }
inline IOp op_crop(const Plane& src, const CropRect& r) {
  const fk_crop_rect c{r.x0, r.y0, r.w, r.h};
  return detail::make(fk_op_crop, &src.raw(), &c);
}
inline IOp op_resize(const IOp& up, std::uint32_t w, std::uint32_t h, ResizeMode mode) {
  fk_iop* out = nullptr;
  check(fk_op_resize(up.get(), w, h, mode == ResizeMode::Bilinear ? FK_BILINEAR : FK_NEAREST, &out));
  return IOp(out);
}
inline IOp op_resize(const Plane& src, std::uint32_t w, std::uint32_t h, ResizeMode mode) {
  return op_resize(op_read_per_thread(src), w, h, mode);
}
inline IOp op_color_convert(ColorOrder order, ScalarKind in) {
  return detail::make(fk_op_color_convert, std::uint32_t(order), detail::u(in));
}
inline IOp op_split_write(const std::array<Plane, 3>& d) {
  const fk_plane raw[3] = {d[0].raw(), d[1].raw(), d[2].raw()};
  return detail::make(fk_op_split_write, static_cast<const fk_plane*>(raw));
}
inline IOp op_batch_read(std::vector<IOp> inner, std::uint32_t active, const Element& def) {
  std::vector<const fk_iop*> v;
  for (const IOp& i : inner) v.push_back(i.get());
  fk_iop* out = nullptr;
  check(fk_op_batch_read(v.data(), std::uint32_t(v.size()), active, def.bytes, &out));
  return IOp(out);
}
inline IOp op_batch_read(std::vector<IOp> inner) {
  const auto n = std::uint32_t(inner.size());
  return op_batch_read(std::move(inner), n, Element{});
}
inline IOp op_batch_write(std::vector<IOp> inner, std::uint32_t active) {
  std::vector<const fk_iop*> v;
  for (const IOp& i : inner) v.push_back(i.get());
  fk_iop* out = nullptr;
  check(fk_op_batch_write(v.data(), std::uint32_t(v.size()), active, &out));
  return IOp(out);
}
inline IOp op_batch_write(std::vector<IOp> inner) {
  const auto n = std::uint32_t(inner.size());
  return op_batch_write(std::move(inner), n);
}
inline IOp fold_unary_into_read(const IOp& read, const IOp& unary) {
  fk_iop* out = nullptr;
  check(fk_fold_unary_into_read(read.get(), unary.get(), &out));
  return IOp(out);
}
// extension (north star C4): an arith op whose constant is chosen by the batch index z
inline IOp op_batch_arith(OpId id, const std::vector<Const>& per_plane) {
  if (per_plane.empty()) fail(Errc::EmptyBatch, "no per-plane constants");
  std::vector<std::uint8_t> raw(24 * per_plane.size());
  const std::uint32_t bpe = bytes_per_element(per_plane[0].kind);
  for (std::size_t z = 0; z < per_plane.size(); ++z) std::memcpy(&raw[z * bpe], per_plane[z].value.bytes, bpe);
  return detail::make(fk_op_batch_arith, std::uint32_t(id), detail::u(per_plane[0].kind),
                      static_cast<const void*>(raw.data()), std::uint32_t(per_plane.size()));
}

// ------------------------------------------- validation & execution --
inline Pipeline validate_chain(std::vector<IOp> ops) {  // ops.hpp:171
  std::vector<const fk_iop*> v;
  for (const IOp& i : ops) v.push_back(i.get());
  fk_pipeline* out = nullptr;
  check(fk_validate_chain(v.data(), std::uint32_t(v.size()), &out));
  return Pipeline(out);
}
inline ExecReport execute_fused(const Pipeline& p, const ExecConfig& cfg = {}) {  // executor.hpp:40
  ExecReport r{};
  const fk_exec_config c = cfg.raw();
  check(fk_execute_fused(p.get(), &c, &r));
  return r;
}
inline ExecReport execute_fused(std::vector<IOp> ops, const ExecConfig& cfg = {}) {
  return execute_fused(validate_chain(std::move(ops)), cfg);
}
inline ExecReport execute_unfused(const Pipeline& p, const ExecConfig& cfg = {}) {  // executor.hpp:51
  ExecReport r{};
  const fk_exec_config c = cfg.raw();
  check(fk_execute_unfused(p.get(), &c, &r));
  return r;
}
inline std::uint64_t plan_memory_savings(const Pipeline& p) {  // executor.hpp:55
  std::uint64_t b = 0;
  check(fk_plan_memory_savings(p.get(), &b));
  return b;
}
// multi-GPU batch sharding: shard i on devices[i], all enqueued before any wait
inline std::vector<ExecReport> execute_sharded(const std::vector<Pipeline>& shards, const std::vector<int>& devices,
                                               const std::vector<ExecConfig>& cfgs = {}) {
  if (shards.size() != devices.size() || (!cfgs.empty() && cfgs.size() != shards.size()))
    fail(Errc::InvalidConfig, "one device (and config) per shard");
  std::vector<const fk_pipeline*> p;
  std::vector<std::int32_t> d(devices.begin(), devices.end());
  std::vector<fk_exec_config> c;
  for (std::size_t i = 0; i < shards.size(); ++i) {
    p.push_back(shards[i].get());
    if (!cfgs.empty()) c.push_back(cfgs[i].raw());
  }
  std::vector<ExecReport> r(shards.size());
  check(fk_execute_sharded(p.data(), d.data(), std::uint32_t(p.size()), c.empty() ? nullptr : c.data(), r.data()));
  return r;
}

// ==========================================================================
// api:: — the lazy facade (api.hpp:13-69, api.cpp:13-268): handles defer work,
// chains are folded / validated with provenance, pipelines are cached by the
// handles' uids so repeat executions skip validation and the device upload.
namespace api {

class LazyHandle {
 public:
  const std::string& provenance() const { return prov_; }
  std::uint64_t uid() const { return uid_; }
  bool deferred() const { return !iop_.has_value(); }
  const IOp& iop() const { return *iop_; }

  // deferred: a colour conversion (kind from the chain) or a cast to `cast_to`
  enum class Deferred : std::uint8_t { None, Cvt, Cast };
  Deferred what = Deferred::None;
  ColorOrder cvt_order = ColorOrder::SwapRB;
  ScalarKind cast_to = ScalarKind::F32;

  static LazyHandle make(std::string prov, IOp iop) {
    LazyHandle h;
    h.iop_ = std::move(iop);
    h.prov_ = std::move(prov);
    h.uid_ = next_uid();
    return h;
  }
  static LazyHandle make_deferred(std::string prov, Deferred what) {
    LazyHandle h;
    h.what = what;
    h.prov_ = std::move(prov);
    h.uid_ = next_uid();
    return h;
  }

 private:
  static std::uint64_t next_uid() {
    static std::atomic<std::uint64_t> n{1};
    return n.fetch_add(1, std::memory_order_relaxed);
  }
  std::optional<IOp> iop_;
  std::string prov_;
  std::uint64_t uid_ = 0;
};

namespace detail {
template <class Fn>
IOp guarded(const std::string& prov, Fn&& fn) {
  try {
    return fn();
  } catch (Error& e) {
    e.set_provenance(prov);
    throw;
  }
}
inline bool is_sample_read(OpId id) { return id == OpId::PerThreadRead || id == OpId::CropRead || id == OpId::ResizeRead; }
}  // namespace detail

inline LazyHandle read(const Plane& s) { return LazyHandle::make("read", detail::guarded("read", [&] { return op_read_per_thread(s); })); }
inline LazyHandle write(const Plane& d) { return LazyHandle::make("write", detail::guarded("write", [&] { return op_write_per_thread(d); })); }
inline LazyHandle crop(const Plane& s, const CropRect& r) {
  return LazyHandle::make("crop", detail::guarded("crop", [&] { return op_crop(s, r); }));
}
inline LazyHandle resize(const Plane& s, std::uint32_t w, std::uint32_t h, ResizeMode m = ResizeMode::Bilinear) {
  return LazyHandle::make("resize", detail::guarded("resize", [&] { return op_resize(s, w, h, m); }));
}
inline LazyHandle resize(const LazyHandle& up, std::uint32_t w, std::uint32_t h, ResizeMode m = ResizeMode::Bilinear) {
  if (up.deferred()) fail(Errc::UnsupportedKind, "resize upstream must be a read handle");
  return LazyHandle::make("resize", detail::guarded("resize", [&] { return op_resize(up.iop(), w, h, m); }));
}
inline LazyHandle cvt_color(ColorOrder order) {
  LazyHandle h = LazyHandle::make_deferred("cvt_color", LazyHandle::Deferred::Cvt);
  h.cvt_order = order;
  return h;
}
// The handle the reference facade lacks: cast the flowing
// value to `to`, the source kind taken from the chain.
inline LazyHandle cast(ScalarKind to) {
  LazyHandle h = LazyHandle::make_deferred("cast", LazyHandle::Deferred::Cast);
  h.cast_to = to;
  return h;
}
inline LazyHandle multiply(const Const& c) { return LazyHandle::make("multiply", detail::guarded("multiply", [&] { return op_mul(c); })); }
inline LazyHandle subtract(const Const& c) { return LazyHandle::make("subtract", detail::guarded("subtract", [&] { return op_sub(c); })); }
inline LazyHandle divide(const Const& c) { return LazyHandle::make("divide", detail::guarded("divide", [&] { return op_div(c); })); }
inline LazyHandle split(const std::array<Plane, 3>& d) {
  return LazyHandle::make("split", detail::guarded("split", [&] { return op_split_write(d); }));
}

namespace detail {
// resolve deferred handles against the kind flowing at their position (api.cpp:96-122)
inline std::vector<IOp> resolve_chain(const std::vector<LazyHandle>& hs) {
  std::vector<IOp> ops;
  std::optional<ScalarKind> cur;
  for (std::size_t i = 0; i < hs.size(); ++i) {
    const LazyHandle& h = hs[i];
    if (h.deferred()) {
      if (!cur) {
        Error e(int(Errc::KindMismatch) + 1, h.provenance() + " has no upstream value", int(i));
        e.set_provenance(h.provenance());
        throw e;
      }
      IOp op = guarded(h.provenance(), [&] {
        return h.what == LazyHandle::Deferred::Cvt ? op_color_convert(h.cvt_order, *cur) : op_cast(*cur, h.cast_to);
      });
      cur = op.output_kind();
      ops.push_back(std::move(op));
    } else {
      if (h.iop().output_kind()) cur = h.iop().output_kind();
      ops.push_back(h.iop());
    }
  }
  return ops;
}
// collapse leading unary ops into the read (api.cpp:124-143)
inline std::vector<IOp> fold_leading_unaries(std::vector<IOp> ops, std::size_t& folded) {
  folded = 0;
  if (ops.empty() || ops.front().kind() != OpKind::Read || !is_sample_read(ops.front().id())) return ops;
  std::vector<IOp> out;
  IOp rd = ops.front();
  std::size_t i = 1;
  while (i + 1 < ops.size() && ops[i].kind() == OpKind::Unary) {
    rd = fold_unary_into_read(rd, ops[i]);
    ++i;
    ++folded;
  }
  out.push_back(rd);
  for (; i < ops.size(); ++i) out.push_back(ops[i]);
  return out;
}
struct Cache {
  std::mutex mu;
  std::unordered_map<std::string, std::shared_ptr<const Pipeline>> built;
};
inline Cache& cache() {
  static Cache c;
  return c;
}
inline std::string key_of(const std::vector<const std::vector<LazyHandle>*>& lists) {
  std::string k;
  for (const auto* l : lists) {
    for (const LazyHandle& h : *l) {
      const std::uint64_t u = h.uid();
      k.append(reinterpret_cast<const char*>(&u), sizeof u);
    }
    k.push_back('|');
  }
  return k;
}
template <class Build>
std::shared_ptr<const Pipeline> cached(const std::string& key, Build&& build) {
  {
    std::lock_guard<std::mutex> lock(cache().mu);
    auto it = cache().built.find(key);
    if (it != cache().built.end()) return it->second;
  }
  auto p = std::make_shared<const Pipeline>(build());
  std::lock_guard<std::mutex> lock(cache().mu);
  return cache().built.emplace(key, p).first->second;
}
}  // namespace detail

// api.cpp:183-186: resolve, fold, validate; chain errors name the offending handle
inline Pipeline build_pipeline(const std::vector<LazyHandle>& hs) {
  if (hs.empty()) fail(Errc::EmptyChain, "no handles");
  std::size_t folded = 0;
  std::vector<IOp> ops = detail::fold_leading_unaries(detail::resolve_chain(hs), folded);
  try {
    return validate_chain(std::move(ops));
  } catch (Error& e) {
    const std::size_t idx = e.position() <= 0 ? 0 : std::size_t(e.position()) + folded;
    if (idx < hs.size() && e.provenance().empty())
      e.set_provenance(hs[idx].provenance() + " (handle #" + std::to_string(idx + 1) + ")");
    throw;
  }
}

// api.cpp:188-202: uid-keyed pipeline cache, one fused execution
inline ExecReport execute_operations(const std::vector<LazyHandle>& hs, const ExecConfig& cfg = {}) {
  auto p = detail::cached(detail::key_of({&hs}), [&] { return build_pipeline(hs); });
  return execute_fused(*p, cfg);
}

// api.cpp:204-258: per-plane reads / writes wrapped in batch ops around the shared chain
inline Pipeline build_batch_pipeline(const std::vector<LazyHandle>& reads, const std::vector<LazyHandle>& compute,
                                     const std::vector<LazyHandle>& writes) {
  if (reads.empty()) fail(Errc::EmptyBatch, "batch needs at least one read");
  if (reads.size() != writes.size()) fail(Errc::HeterogeneousBatch, "read and write handle counts differ");
  std::vector<LazyHandle> probe{reads.front()};
  probe.insert(probe.end(), compute.begin(), compute.end());
  std::vector<IOp> resolved = detail::resolve_chain(probe);
  std::size_t n_fold = 0;
  while (1 + n_fold < resolved.size() && resolved[1 + n_fold].kind() == OpKind::Unary) ++n_fold;
  std::vector<IOp> inner_reads, inner_writes;
  for (std::size_t i = 0; i < reads.size(); ++i) {
    const LazyHandle& h = reads[i];
    if (h.deferred() || h.iop().kind() != OpKind::Read || !detail::is_sample_read(h.iop().id())) {
      Error e(int(Errc::HeterogeneousBatch) + 1, "read handle #" + std::to_string(i + 1) + " is not a per-plane read",
              int(i));
      e.set_provenance(h.provenance());
      throw e;
    }
    IOp r = h.iop();
    for (std::size_t f = 0; f < n_fold; ++f)
      r = detail::guarded(h.provenance(), [&] { return fold_unary_into_read(r, resolved[1 + f]); });
    inner_reads.push_back(r);
  }
  for (std::size_t i = 0; i < writes.size(); ++i) {
    const LazyHandle& h = writes[i];
    if (h.deferred() || h.iop().kind() != OpKind::Write) {
      Error e(int(Errc::HeterogeneousBatch) + 1, "write handle #" + std::to_string(i + 1) + " is not a per-plane write",
              int(i));
      e.set_provenance(h.provenance());
      throw e;
    }
    inner_writes.push_back(h.iop());
  }
  std::vector<IOp> chain{op_batch_read(std::move(inner_reads))};
  for (std::size_t i = 1 + n_fold; i < resolved.size(); ++i) chain.push_back(resolved[i]);
  chain.push_back(op_batch_write(std::move(inner_writes)));
  return validate_chain(std::move(chain));
}

inline ExecReport execute_batch(const std::vector<LazyHandle>& reads, const std::vector<LazyHandle>& compute,
                                const std::vector<LazyHandle>& writes, const ExecConfig& cfg = {}) {
  // the reference rebuilds per call (api.cpp:260-266); the uid key makes repeats free here
  auto p = detail::cached(detail::key_of({&reads, &compute, &writes}),
                          [&] { return build_batch_pipeline(reads, compute, writes); });
  return execute_fused(*p, cfg);
}

}  // namespace api

// ==========================================================================
// sc:: — the typed static chain (static_chain.hpp:64-176): the op sequence is
// spelled in the type system; transform() hands it to the library, whose
// compiled-signature registry runs it as one specialised kernel (fk_direct /
// fk_walk) when the sequence is registered, the interpreted kernel otherwise.
namespace sc {

template <class T>
struct Vec3 {
  std::array<T, 3> v{};
};

namespace detail {
template <class T> struct kind_of;
template <> struct kind_of<std::uint8_t> { static constexpr ScalarKind value = ScalarKind::U8; };
template <> struct kind_of<float> { static constexpr ScalarKind value = ScalarKind::F32; };
template <> struct kind_of<double> { static constexpr ScalarKind value = ScalarKind::F64; };
template <> struct kind_of<Vec3<std::uint8_t>> { static constexpr ScalarKind value = ScalarKind::U8x3; };
template <> struct kind_of<Vec3<float>> { static constexpr ScalarKind value = ScalarKind::F32x3; };
template <> struct kind_of<Vec3<double>> { static constexpr ScalarKind value = ScalarKind::F64x3; };
template <class T> Const to_const(const T& c) { return Const(c); }
template <class T> Const to_const(const Vec3<T>& c) { return Const(c.v); }
}  // namespace detail

template <class T> struct Mul { using In = T; using Out = T; T c{}; IOp iop() const { return op_mul(detail::to_const(c)); } };
template <class T> struct Add { using In = T; using Out = T; T c{}; IOp iop() const { return op_add(detail::to_const(c)); } };
template <class T> struct Sub { using In = T; using Out = T; T c{}; IOp iop() const { return op_sub(detail::to_const(c)); } };
template <class T> struct Div { using In = T; using Out = T; T c{}; IOp iop() const { return op_div(detail::to_const(c)); } };
template <class From, class To>
struct Cast {
  using In = From;
  using Out = To;
  IOp iop() const { return op_cast(detail::kind_of<From>::value, detail::kind_of<To>::value); }
};
template <class T>
struct SwapRB {
  using In = Vec3<T>;
  using Out = Vec3<T>;
  IOp iop() const { return op_color_convert(ColorOrder::SwapRB, detail::kind_of<Vec3<T>>::value); }
};
template <class T>
struct ToGrayF32 {
  using In = Vec3<T>;
  using Out = float;
  IOp iop() const { return op_color_convert(ColorOrder::ToGrayF32, detail::kind_of<Vec3<T>>::value); }
};
template <class Op, unsigned N>
struct StaticLoop {
  static_assert(N >= 1, "StaticLoop needs N >= 1");
  static_assert(std::is_same_v<typename Op::In, typename Op::Out>, "StaticLoop body must preserve the kind");
  using In = typename Op::In;
  using Out = typename Op::Out;
  Op inner{};
  IOp iop() const { return op_static_loop(inner.iop(), N); }
};

// compile-time check of the chain's kinds (static_chain.hpp:143-148)
template <class V, class... Ops>
struct chain_ok : std::true_type {};
template <class V, class Op, class... Rest>
struct chain_ok<V, Op, Rest...>
    : std::integral_constant<bool, std::is_same_v<V, typename Op::In> && chain_ok<typename Op::Out, Rest...>::value> {};
template <class V, class... Ops>
struct out_of_chain { using type = V; };
template <class V, class Op, class... Rest>
struct out_of_chain<V, Op, Rest...> { using type = typename out_of_chain<typename Op::Out, Rest...>::type; };

template <class T>
class PlaneView {  // static_chain.hpp:150-161: a typed view over a plane of kind_of<T>
 public:
  explicit PlaneView(const Plane& p) : plane_(p) {
    if (p.kind() != detail::kind_of<T>::value) fail(Errc::KindMismatch, "typed view over a plane of another kind");
  }
  std::uint32_t width() const { return plane_.width(); }
  std::uint32_t height() const { return plane_.height(); }
  const Plane& plane() const { return plane_; }

 private:
  Plane plane_;
};

// static_chain.hpp:163-176: dst = Ops...(src) over the whole plane, one fused pass
template <class TIn, class TOut, class... Ops>
ExecReport transform(const PlaneView<TIn>& src, const PlaneView<TOut>& dst, int workers, const Ops&... ops) {
  static_assert(chain_ok<TIn, Ops...>::value, "adjacent ops in a static chain must agree on the element kind");
  static_assert(std::is_same_v<typename out_of_chain<TIn, Ops...>::type, TOut>,
                "the chain's result kind must be the destination's");
  std::vector<IOp> chain{op_read_per_thread(src.plane())};
  (chain.push_back(ops.iop()), ...);
  chain.push_back(op_write_per_thread(dst.plane()));
  ExecConfig cfg;
  cfg.workers = workers;
  return execute_fused(validate_chain(std::move(chain)), cfg);
}

}  // namespace sc

}  // namespace opfuse_fk

#ifdef OPFUSE_FK_AS_OPFUSE
namespace opfuse = opfuse_fk;
#endif
