// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. Exports the include/fk.h ABI over the
// UNMODIFIED reference library (/root/reference/proj, namespace opfuse), so the
// same Python harness can drive the reference, the C restatement and the CUDA
// product with identical chain descriptions.
//
// Built by oracle/Makefile straight from the reference source tree into
// oracle/_ref/libfk_ref.so (git-ignored, travels to the GPU box). Used by the
// parity tests (pinning oracle/fk_oracle.c) and as bench.py's CPU baseline
// ("kind": "reference").
//
// The reference's Plane owns host memory (plane.cpp:60-89) and cannot wrap a
// caller's buffer, so every fk_plane is mirrored by a reference Plane of the
// same row stride: sources are copied in before an execute and destinations
// copied out after it, outside the reference's own timed region
// (ExecReport::wall_time_ns, executor.cpp:73-82), which is what gets reported.

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "opfuse/dpp.hpp"
#include "opfuse/executor.hpp"
#include "opfuse/oplib.hpp"
#include "opfuse/tensor_io.hpp"
#include "opfuse/ops.hpp"
#include "fk.h"

using namespace opfuse;

namespace {

thread_local std::string g_err;
thread_local int32_t g_pos = -1;

fk_status set_error(const Error& e) {
  g_err = e.what();
  g_pos = e.position();
  return 1 + static_cast<int32_t>(e.code());
}
fk_status set_error(fk_status st, const std::string& msg) {
  g_err = msg;
  g_pos = -1;
  return st;
}

struct Binding {
  fk_plane user{};
  Plane backing;  // row_stride x height, zero-initialised
  Plane view;     // width x height sub-view with the user's stride
};

using Key = std::tuple<void*, uint32_t, uint32_t, uint32_t, uint32_t>;
std::mutex g_mu;
std::map<Key, std::weak_ptr<Binding>> g_cache;

bool plane_ok(const fk_plane* p) {
  return p && p->data && p->kind <= FK_F64X3 && p->width >= 1 && p->height >= 1 &&
         p->row_stride >= p->width;
}

std::shared_ptr<Binding> bind(const fk_plane& p) {
  Key k{p.data, p.width, p.height, p.row_stride, p.kind};
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_cache.find(k);
  if (it != g_cache.end())
    if (auto sp = it->second.lock()) return sp;
  auto b = std::make_shared<Binding>();
  b->user = p;
  b->backing = Plane::alloc(p.row_stride, p.height, static_cast<ScalarKind>(p.kind));
  b->view = b->backing.view(0, 0, p.width, p.height);
  g_cache[k] = b;
  return b;
}

void copy_in(const Binding& b) {
  const size_t bpe = bytes_per_element(b.view.kind());
  for (uint32_t y = 0; y < b.user.height; ++y)
    std::memcpy(b.view.row_mut(y),
                static_cast<const uint8_t*>(b.user.data) + size_t(y) * b.user.row_stride * bpe,
                size_t(b.user.width) * bpe);
}
void copy_out(const Binding& b) {
  const size_t bpe = bytes_per_element(b.view.kind());
  for (uint32_t y = 0; y < b.user.height; ++y)
    std::memcpy(static_cast<uint8_t*>(b.user.data) + size_t(y) * b.user.row_stride * bpe,
                b.view.row(y), size_t(b.user.width) * bpe);
}

Element element_from(uint32_t kind, const void* raw) {
  Element e;
  if (raw) std::memcpy(e.raw.data(), raw, bytes_per_element(static_cast<ScalarKind>(kind)));
  return e;
}

}  // namespace

struct fk_iop {
  IOp op;
  std::vector<std::shared_ptr<Binding>> srcs, dsts;
};
struct fk_pipeline {
  Pipeline p;
  std::vector<std::shared_ptr<Binding>> srcs, dsts;
};

namespace {

template <class Fn>
fk_status guarded(fk_iop** out, Fn&& fn) {
  if (!out) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null output pointer");
  *out = nullptr;
  try {
    *out = fn();
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  } catch (const std::exception& e) {
    return set_error(FK_E_INVALID_ARGUMENT, e.what());
  }
}

void append(std::vector<std::shared_ptr<Binding>>& into, const std::vector<std::shared_ptr<Binding>>& from) {
  into.insert(into.end(), from.begin(), from.end());
}

ExecConfig to_cfg(const fk_exec_config* c) {
  ExecConfig cfg;
  if (c) {
    cfg.workers = c->workers;
    cfg.coarsening.block = c->coarsen_block;
    cfg.chunk_rows = c->chunk_rows;
  }
  return cfg;
}

void fill(fk_exec_report* rep, const ExecReport& r) {
  if (!rep) return;
  std::memset(rep, 0, sizeof *rep);
  rep->wall_time_ns = r.wall_time_ns;
  rep->bytes_read = r.bytes_read;
  rep->bytes_written = r.bytes_written;
  rep->intermediate_bytes_allocated = r.intermediate_bytes_allocated;
  rep->passes = r.passes;
  rep->points_visited = r.points_visited;
  rep->path = FK_PATH_CPU;
}

}  // namespace

extern "C" {

const char* fk_backend_name(void) { return "reference-opfuse"; }
int32_t fk_abi_version(void) { return FK_ABI_VERSION; }
const char* fk_last_error(void) { return g_err.c_str(); }
int32_t fk_last_error_position(void) { return g_pos; }
int32_t fk_errc_name(int32_t status, char* buf, size_t cap) {
  std::string s = status == 0 ? "OK"
                  : (status >= 1 && status <= 24) ? errc_name(static_cast<Errc>(status - 1))
                                                  : "UnknownError";
  if (buf && cap) {
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return static_cast<int32_t>(s.size());
}

uint32_t fk_bytes_per_element(uint32_t kind) {
  return kind <= FK_F64X3 ? static_cast<uint32_t>(bytes_per_element(static_cast<ScalarKind>(kind))) : 0;
}

fk_status fk_plane_view(const fk_plane* p, uint32_t x0, uint32_t y0, uint32_t w, uint32_t h,
                        fk_plane* out) {
  if (!plane_ok(p) || !out) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid plane");
  if (w == 0 || h == 0 || uint64_t(x0) + w > p->width || uint64_t(y0) + h > p->height)
    return set_error(1 + int32_t(Errc::BoundsError), "BoundsError: sub-view outside plane");
  *out = *p;
  out->data = static_cast<uint8_t*>(p->data) +
              (uint64_t(y0) * p->row_stride + x0) * fk_bytes_per_element(p->kind);
  out->width = w;
  out->height = h;
  return FK_OK;
}

fk_status fk_plane_alloc(uint32_t width, uint32_t height, uint32_t kind, uint32_t row_stride, fk_plane* out) {
  // Plane::alloc, plane.cpp:60-71 (host memory; test infrastructure: freed by fk_plane_free)
  if (!out || kind > FK_F64X3) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: bad plane arguments");
  const uint32_t rs = row_stride ? row_stride : width;
  if (width == 0 || height == 0 || rs < width)
    return set_error(1 + int32_t(Errc::CapacityOverflow), "CapacityOverflow: extents");
  void* p = std::calloc(size_t(rs) * height, fk_bytes_per_element(kind));
  if (!p) return set_error(1 + int32_t(Errc::CapacityOverflow), "CapacityOverflow: host allocation failed");
  *out = fk_plane{p, width, height, rs, kind};
  return FK_OK;
}
void fk_plane_free(fk_plane* p) {
  if (p && p->data) {
    std::free(p->data);
    p->data = nullptr;
  }
}

static fk_status plane_copy(const fk_plane* p, void* host, size_t host_pitch, bool up) {
  if (!plane_ok(p) || !host) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: bad plane copy");
  const size_t row = size_t(p->width) * fk_bytes_per_element(p->kind);
  const size_t hp = host_pitch ? host_pitch : row, pp = size_t(p->row_stride) * fk_bytes_per_element(p->kind);
  for (uint32_t y = 0; y < p->height; ++y) {
    uint8_t* d = static_cast<uint8_t*>(p->data) + y * pp;
    uint8_t* h = static_cast<uint8_t*>(host) + y * hp;
    if (up) std::memcpy(d, h, row);
    else std::memcpy(h, d, row);
  }
  return FK_OK;
}
fk_status fk_plane_upload(const fk_plane* dst, const void* host, size_t host_pitch) {
  return plane_copy(dst, const_cast<void*>(host), host_pitch, true);
}
fk_status fk_plane_download(const fk_plane* src, void* host, size_t host_pitch) {
  return plane_copy(src, host, host_pitch, false);
}

// FKT files through the reference's own tensor_io (tensor_io.cpp:12-117)
static Plane host_copy(const fk_plane& p) {
  Plane q = Plane::alloc(p.width, p.height, static_cast<ScalarKind>(p.kind));
  const size_t row = size_t(p.width) * fk_bytes_per_element(p.kind);
  for (uint32_t y = 0; y < p.height; ++y)
    std::memcpy(q.row_mut(y), static_cast<const uint8_t*>(p.data) + size_t(y) * p.row_stride * fk_bytes_per_element(p.kind), row);
  return q;
}
fk_status fk_tensor_write_file(const fk_plane* planes, uint32_t n, const char* path) {
  if (!path) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null path");
  try {
    std::vector<Plane> v;
    for (uint32_t i = 0; planes && i < n; ++i) {
      if (!plane_ok(&planes[i])) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid plane");
      v.push_back(host_copy(planes[i]));
    }
    tensor_write_file(PlaneBatch(std::move(v)), path);
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}
fk_status fk_tensor_read_file(const char* path, fk_plane* out, uint32_t cap, uint32_t* count) {
  if (!path || !count) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  try {
    const PlaneBatch b = tensor_read_file(path);
    *count = uint32_t(b.size());
    if (cap < b.size() || !out) return FK_OK;
    for (size_t i = 0; i < b.size(); ++i) {
      const Plane& p = b[i];
      fk_plane_alloc(p.width(), p.height(), uint32_t(p.kind()), 0, &out[i]);
      const size_t row = size_t(p.width()) * bytes_per_element(p.kind());
      for (uint32_t y = 0; y < p.height(); ++y)
        std::memcpy(static_cast<uint8_t*>(out[i].data) + y * row, p.row(y), row);
    }
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}
fk_status fk_write_ppm(const fk_plane* p, const char* path) {
  if (!plane_ok(p) || !path) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: bad arguments");
  try {
    write_ppm(host_copy(*p), path);
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}

fk_status fk_op_arith(uint32_t op_id, uint32_t kind, const void* value, fk_iop** out) {
  if (op_id < FK_OP_MUL || op_id > FK_OP_DIV || kind > FK_F64X3 || !value)
    return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: bad arith op");
  return guarded(out, [&] {
    return new fk_iop{make_arith(static_cast<OpId>(op_id), static_cast<ScalarKind>(kind),
                                 element_from(kind, value)), {}, {}};
  });
}

fk_status fk_op_batch_arith(uint32_t, uint32_t, const void*, uint32_t, fk_iop** out) {
  if (out) *out = nullptr;
  return set_error(FK_E_UNSUPPORTED, "Unsupported: the reference has no per-plane compute constants");
}

fk_status fk_op_cast(uint32_t from, uint32_t to, fk_iop** out) {
  if (from > FK_F64X3 || to > FK_F64X3) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: bad kind");
  return guarded(out, [&] {
    return new fk_iop{op_cast(static_cast<ScalarKind>(from), static_cast<ScalarKind>(to)), {}, {}};
  });
}

fk_status fk_op_static_loop(const fk_iop* inner, uint32_t repeat, fk_iop** out) {
  if (!inner) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null inner op");
  return guarded(out, [&] { return new fk_iop{op_static_loop(inner->op, repeat), {}, {}}; });
}

fk_status fk_op_read_per_thread(const fk_plane* src, fk_iop** out) {
  if (!plane_ok(src)) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid source plane");
  return guarded(out, [&] {
    auto b = bind(*src);
    return new fk_iop{op_read_per_thread(b->view), {b}, {}};
  });
}

fk_status fk_op_write_per_thread(const fk_plane* dst, fk_iop** out) {
  if (!plane_ok(dst)) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid destination plane");
  return guarded(out, [&] {
    auto b = bind(*dst);
    return new fk_iop{op_write_per_thread(b->view), {}, {b}};
  });
}

fk_status fk_op_crop(const fk_plane* src, const fk_crop_rect* r, fk_iop** out) {
  if (!plane_ok(src) || !r) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid crop arguments");
  return guarded(out, [&] {
    auto b = bind(*src);
    return new fk_iop{op_crop(b->view, CropRect{r->x0, r->y0, r->w, r->h}), {b}, {}};
  });
}

fk_status fk_op_resize(const fk_iop* up, uint32_t w, uint32_t h, uint32_t mode, fk_iop** out) {
  if (!up || mode > FK_BILINEAR) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid resize arguments");
  return guarded(out, [&] {
    return new fk_iop{op_resize(up->op, w, h, static_cast<ResizeMode>(mode)), up->srcs, {}};
  });
}

fk_status fk_op_color_convert(uint32_t order, uint32_t in, fk_iop** out) {
  if (order > FK_TO_GRAY_F32 || in > FK_F64X3) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: bad arguments");
  return guarded(out, [&] {
    return new fk_iop{op_color_convert(static_cast<ColorOrder>(order), static_cast<ScalarKind>(in)), {}, {}};
  });
}

fk_status fk_op_split_write(const fk_plane dst[3], fk_iop** out) {
  if (!dst) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null destinations");
  for (int i = 0; i < 3; ++i)
    if (!plane_ok(&dst[i])) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: invalid destination plane");
  return guarded(out, [&] {
    auto b0 = bind(dst[0]), b1 = bind(dst[1]), b2 = bind(dst[2]);
    return new fk_iop{op_split_write({b0->view, b1->view, b2->view}), {}, {b0, b1, b2}};
  });
}

fk_status fk_op_batch_read(const fk_iop* const* inner, uint32_t n, uint32_t active, const void* def,
                           fk_iop** out) {
  return guarded(out, [&] {
    std::vector<IOp> reads;
    std::vector<std::shared_ptr<Binding>> srcs;
    for (uint32_t i = 0; i < n; ++i) {
      if (!inner[i]) fail(Errc::InnerKindMismatch, "null inner op");
      reads.push_back(inner[i]->op);
      append(srcs, inner[i]->srcs);
    }
    Element d;
    if (def && n && inner[0]->op.output_kind())
      d = element_from(static_cast<uint32_t>(*inner[0]->op.output_kind()), def);
    return new fk_iop{op_batch_read(std::move(reads), active, d), srcs, {}};
  });
}

fk_status fk_op_batch_write(const fk_iop* const* inner, uint32_t n, uint32_t active, fk_iop** out) {
  return guarded(out, [&] {
    std::vector<IOp> writes;
    std::vector<std::shared_ptr<Binding>> dsts;
    for (uint32_t i = 0; i < n; ++i) {
      if (!inner[i]) fail(Errc::InnerKindMismatch, "null inner op");
      writes.push_back(inner[i]->op);
      append(dsts, inner[i]->dsts);
    }
    return new fk_iop{op_batch_write(std::move(writes), active), {}, dsts};
  });
}

fk_status fk_fold_unary_into_read(const fk_iop* read, const fk_iop* unary, fk_iop** out) {
  if (!read || !unary) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null op");
  return guarded(out, [&] { return new fk_iop{fold_unary_into_read(read->op, unary->op), read->srcs, {}}; });
}

void fk_iop_free(fk_iop* op) { delete op; }

uint32_t fk_iop_id(const fk_iop* op) { return static_cast<uint32_t>(op->op.id()); }
uint32_t fk_iop_kind(const fk_iop* op) { return static_cast<uint32_t>(op->op.kind()); }
int32_t fk_iop_input_kind(const fk_iop* op) {
  return op->op.input_kind() ? static_cast<int32_t>(*op->op.input_kind()) : -1;
}
int32_t fk_iop_output_kind(const fk_iop* op) {
  return op->op.output_kind() ? static_cast<int32_t>(*op->op.output_kind()) : -1;
}
int32_t fk_iop_dims(const fk_iop* op, fk_extent3* out) {
  if (!op->op.dims_hint()) return 0;
  if (out) *out = fk_extent3{op->op.dims_hint()->width, op->op.dims_hint()->height, op->op.dims_hint()->batch};
  return 1;
}

fk_status fk_validate_chain(const fk_iop* const* ops, uint32_t n, fk_pipeline** out) {
  if (!out) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null output pointer");
  *out = nullptr;
  try {
    std::vector<IOp> chain;
    std::vector<std::shared_ptr<Binding>> srcs, dsts;
    for (uint32_t i = 0; i < n; ++i) {
      if (!ops[i]) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null op");
      chain.push_back(ops[i]->op);
      append(srcs, ops[i]->srcs);
      append(dsts, ops[i]->dsts);
    }
    Pipeline p = validate_chain(std::move(chain));
    *out = new fk_pipeline{std::move(p), srcs, dsts};
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}

void fk_pipeline_free(fk_pipeline* p) { delete p; }

fk_status fk_pipeline_iter_space(const fk_pipeline* p, fk_extent3* out) {
  if (!p || !out) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  *out = fk_extent3{p->p.iter_space.width, p->p.iter_space.height, p->p.iter_space.batch};
  return FK_OK;
}
uint32_t fk_pipeline_compute_count(const fk_pipeline* p) { return static_cast<uint32_t>(p->p.compute.size()); }

fk_status fk_execute_fused(const fk_pipeline* p, const fk_exec_config* c, fk_exec_report* rep) {
  if (!p) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null pipeline");
  try {
    for (auto& b : p->srcs) copy_in(*b);
    const ExecConfig cfg = to_cfg(c);
    ExecReport r = (c && (c->flags & FK_EXEC_SERIAL)) ? execute_fused_serial(p->p, cfg)
                                                       : execute_fused(p->p, cfg);
    for (auto& b : p->dsts) copy_out(*b);
    fill(rep, r);
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}

fk_status fk_execute_sharded(const fk_pipeline* const* pipelines, const int32_t* devices, uint32_t n,
                             const fk_exec_config* cfgs, fk_exec_report* reports) {
  // CPU backend: the shards one after another (devices are ignored)
  if (n && (!pipelines || !devices)) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  for (uint32_t i = 0; i < n; ++i) {
    const fk_status s = fk_execute_fused(pipelines[i], cfgs ? &cfgs[i] : nullptr, reports ? &reports[i] : nullptr);
    if (s != FK_OK) return s;
  }
  return FK_OK;
}

fk_status fk_gather(void* dst, int32_t, const uint64_t* dst_offsets, const void* const* srcs, const int32_t*,
                    const uint64_t* bytes, uint32_t n, void*) {
  if (n && (!dst || !dst_offsets || !srcs || !bytes)) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  for (uint32_t i = 0; i < n; ++i) std::memcpy(static_cast<uint8_t*>(dst) + dst_offsets[i], srcs[i], bytes[i]);
  return FK_OK;
}

fk_status fk_execute_unfused(const fk_pipeline* p, const fk_exec_config* c, fk_exec_report* rep) {
  if (!p) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null pipeline");
  try {
    for (auto& b : p->srcs) copy_in(*b);
    ExecReport r = execute_unfused(p->p, to_cfg(c));
    for (auto& b : p->dsts) copy_out(*b);
    fill(rep, r);
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}

fk_status fk_plan_memory_savings(const fk_pipeline* p, uint64_t* bytes) {
  if (!p || !bytes) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  *bytes = plan_memory_savings(p->p);
  return FK_OK;
}

fk_status fk_schedule(const fk_extent3* sp, const fk_exec_config* c, uint32_t* tasks, uint64_t cap,
                      uint64_t* count) {
  if (!sp || !c || !count) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  try {
    auto t = schedule(Extent3{sp->width, sp->height, sp->batch}, to_cfg(c));
    *count = t.size();
    for (uint64_t i = 0; i < t.size() && tasks && i < cap; ++i) {
      tasks[3 * i] = t[i].z;
      tasks[3 * i + 1] = t[i].y_begin;
      tasks[3 * i + 2] = t[i].y_end;
    }
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}

}  // extern "C"

// multi_reduce_plane (dpp.cpp:158-241) over the reference; elements_read from
// the reference's instrumented counter (stats::add_elements_read, dpp.cpp:229).
extern "C" fk_status fk_multi_reduce_plane(const fk_iop* read, const fk_reduce_spec* specs, uint32_t n,
                                           int32_t workers, void* results, uint64_t* elements_read) {
  if (!read || (!specs && n) || (!results && n))
    return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: null argument");
  for (uint32_t i = 0; i < n; ++i)  // the C-ABI's enum check (the reference's Reducer is a C++ enum)
    if (specs[i].combine > FK_REDUCE_MIN) return set_error(FK_E_INVALID_ARGUMENT, "InvalidArgument: unknown combine");
  try {
    for (auto& b : read->srcs) copy_in(*b);
    std::vector<ReduceSpec> rs(n);
    for (uint32_t i = 0; i < n; ++i) {
      if (specs[i].transform) rs[i].transform = specs[i].transform->op;
      rs[i].combine = static_cast<Reducer>(specs[i].combine);
      if (specs[i].has_identity) {
        Element e;
        std::memcpy(&e, specs[i].identity, sizeof e);
        rs[i].identity = e;
      }
    }
    const uint64_t before = stats::elements_read();
    const std::vector<Element> out = multi_reduce_plane(read->op, rs, workers);
    if (elements_read) *elements_read = stats::elements_read() - before;
    for (uint32_t i = 0; i < n; ++i) std::memcpy(static_cast<uint8_t*>(results) + 24 * size_t(i), &out[i], 24);
    return FK_OK;
  } catch (const Error& e) {
    return set_error(e);
  }
}

