// fk_capi.cpp — the extern "C" boundary (include/fk.h) of libfk_cuda.so.
// C++ exceptions never cross it: every entry point returns an fk_status and
// leaves the message / chain position in thread-local storage.
#include <cuda_runtime.h>

#include <cstdio>

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fk.h"
#include "fk_core.hpp"
#include "fk_cuda.h"
#include "fk_exec.hpp"

// An IOp / pipeline holds the buffers of the fk_plane_alloc planes it
// references (plane.hpp:97: views and ops share ownership of the buffer).
using Holds = std::vector<std::shared_ptr<void>>;
struct fk_iop {
  fk::Op op;
  Holds hold;
};
struct fk_pipeline {
  fk::Pipeline p;
  Holds hold;
};

namespace {

// fk_plane_alloc buffers by base address; the registry's reference is the
// caller's (dropped by fk_plane_free), ops and pipelines add their own.
struct Buffers {
  std::mutex mu;
  std::map<uintptr_t, std::pair<size_t, std::shared_ptr<void>>> by_base;
};
Buffers& buffers() {
  static Buffers* b = new Buffers;  // never destroyed: ops may outlive static teardown
  return *b;
}
std::shared_ptr<void> owner_of(const void* p) {
  if (!p) return nullptr;
  Buffers& b = buffers();
  std::lock_guard<std::mutex> lock(b.mu);
  if (b.by_base.empty()) return nullptr;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  auto it = b.by_base.upper_bound(a);
  if (it == b.by_base.begin()) return nullptr;
  --it;
  return a < it->first + it->second.first ? it->second.second : nullptr;
}
void cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  fk::fail(FK_E_CUDA, std::string("CudaError: ") + what + ": " + cudaGetErrorString(e));
}
void hold_plane(Holds& h, const fk_plane& pl) {
  if (auto o = owner_of(pl.data)) h.push_back(std::move(o));
}
// every plane an op references (reads, batch reads, writes)
Holds holds_of(const fk::Op& op) {
  Holds h;
  if (fk::is_sample_read(op)) hold_plane(h, op.sample.source);
  for (const fk::Sample& s : op.planes) hold_plane(h, s.source);
  for (const fk_plane& d : op.dest) hold_plane(h, d);
  for (const fk_plane& d : op.wdest) hold_plane(h, d);
  return h;
}

thread_local std::string g_err;
thread_local int32_t g_pos = -1;

// an fk_* call inside another entry point: rethrow its failure unchanged
void check_status(fk_status s) {
  if (s != FK_OK) throw fk::Error(s, g_err, g_pos);
}

template <class Fn>
fk_status guard(Fn&& fn) {
  try {
    fn();
    return FK_OK;
  } catch (const fk::Error& e) {
    g_err = e.what();
    g_pos = e.position;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "CapacityOverflow: host allocation failed";
    g_pos = -1;
    return FK_E_CAPACITY_OVERFLOW;
  } catch (const std::exception& e) {
    g_err = std::string("InvalidArgument: ") + e.what();
    g_pos = -1;
    return FK_E_INVALID_ARGUMENT;
  }
}

template <class Fn>
fk_status build(fk_iop** out, Fn&& fn) {
  if (!out) {
    g_err = "InvalidArgument: null output pointer";
    return FK_E_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guard([&] {
    fk::Op op = fn();
    Holds h = holds_of(op);
    *out = new fk_iop{std::move(op), std::move(h)};
  });
}

const fk::Op& deref(const fk_iop* op, const char* what) {
  if (!op) fk::fail(FK_E_INVALID_ARGUMENT, std::string("null ") + what);
  return op->op;
}

}  // namespace

extern "C" {

const char* fk_backend_name(void) { return "cuda-sm100a"; }
int32_t fk_abi_version(void) { return FK_ABI_VERSION; }
const char* fk_last_error(void) { return g_err.c_str(); }
int32_t fk_last_error_position(void) { return g_pos; }
int32_t fk_errc_name(int32_t status, char* buf, size_t cap) {
  const char* s = fk::errc_name(status);
  if (buf && cap) {
    std::strncpy(buf, s, cap - 1);
    buf[cap - 1] = 0;
  }
  return int32_t(std::strlen(s));
}

uint32_t fk_bytes_per_element(uint32_t kind) { return fk::kind_ok(kind) ? fk::bpe(kind) : 0; }

fk_status fk_plane_view(const fk_plane* p, uint32_t x0, uint32_t y0, uint32_t w, uint32_t h, fk_plane* out) {
  return guard([&] {  // Plane::view, plane.cpp:91-101
    fk::check_plane(p, "source");
    if (!out) fk::fail(FK_E_INVALID_ARGUMENT, "null output");
    if (w == 0 || h == 0 || uint64_t(x0) + w > p->width || uint64_t(y0) + h > p->height)
      fk::fail(FK_E_BOUNDS_ERROR, "sub-view outside plane");
    *out = *p;
    out->data = static_cast<uint8_t*>(p->data) + (uint64_t(y0) * p->row_stride + x0) * fk::bpe(p->kind);
    out->width = w;
    out->height = h;
  });
}

fk_status fk_plane_alloc(uint32_t width, uint32_t height, uint32_t kind, uint32_t row_stride, fk_plane* out) {
  return guard([&] {  // Plane::alloc, plane.cpp:60-71
    if (!out) fk::fail(FK_E_INVALID_ARGUMENT, "null output");
    if (!fk::kind_ok(kind)) fk::fail(FK_E_INVALID_ARGUMENT, "bad kind");
    const uint32_t rs = row_stride ? row_stride : width;
    if (width == 0 || height == 0 || rs < width) fk::fail(FK_E_CAPACITY_OVERFLOW, "plane extents must be >= 1");
    const size_t bytes = size_t(rs) * height * fk::bpe(kind);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
    if (e != cudaSuccess) {
      if (p) cudaFree(p);
      cudaGetLastError();
      fk::fail(FK_E_CUDA, std::string("CudaError: plane allocation: ") + cudaGetErrorString(e));
    }
    std::shared_ptr<void> buf(p, [](void* q) { cudaFree(q); });
    {
      Buffers& b = buffers();
      std::lock_guard<std::mutex> lock(b.mu);
      b.by_base[reinterpret_cast<uintptr_t>(p)] = {bytes, std::move(buf)};
    }
    *out = fk_plane{p, width, height, rs, kind};
  });
}
void fk_plane_free(fk_plane* pl) {
  if (!pl || !pl->data) return;
  std::shared_ptr<void> last;  // released outside the lock
  {
    Buffers& b = buffers();
    std::lock_guard<std::mutex> lock(b.mu);
    auto it = b.by_base.find(reinterpret_cast<uintptr_t>(pl->data));
    if (it == b.by_base.end()) return;  // not an fk_plane_alloc base (a view, or already freed)
    last = std::move(it->second.second);
    b.by_base.erase(it);
  }
  pl->data = nullptr;
}

fk_status fk_plane_upload(const fk_plane* dst, const void* host, size_t host_pitch) {
  return guard([&] {
    fk::check_plane(dst, "destination");
    if (!host) fk::fail(FK_E_INVALID_ARGUMENT, "null host buffer");
    const size_t row = size_t(dst->width) * fk::bpe(dst->kind);
    cuda_ok(cudaMemcpy2D(dst->data, size_t(dst->row_stride) * fk::bpe(dst->kind), host, host_pitch ? host_pitch : row,
                         row, dst->height, cudaMemcpyDefault),
            "plane upload");
  });
}
fk_status fk_plane_download(const fk_plane* src, void* host, size_t host_pitch) {
  return guard([&] {
    fk::check_plane(src, "source");
    if (!host) fk::fail(FK_E_INVALID_ARGUMENT, "null host buffer");
    const size_t row = size_t(src->width) * fk::bpe(src->kind);
    cuda_ok(cudaMemcpy2D(host, host_pitch ? host_pitch : row, src->data, size_t(src->row_stride) * fk::bpe(src->kind),
                         row, src->height, cudaMemcpyDefault),
            "plane download");
  });
}

fk_status fk_op_arith(uint32_t id, uint32_t kind, const void* value, fk_iop** out) {
  return build(out, [&] { return fk::make_arith(id, kind, value); });
}
fk_status fk_op_batch_arith(uint32_t id, uint32_t kind, const void* values, uint32_t n, fk_iop** out) {
  return build(out, [&] { return fk::make_batch_arith(id, kind, values, n); });
}
fk_status fk_op_cast(uint32_t from, uint32_t to, fk_iop** out) {
  return build(out, [&] { return fk::make_cast(from, to); });
}
fk_status fk_op_static_loop(const fk_iop* inner, uint32_t repeat, fk_iop** out) {
  return build(out, [&] { return fk::make_static_loop(deref(inner, "inner op"), repeat); });
}
fk_status fk_op_read_per_thread(const fk_plane* src, fk_iop** out) {
  return build(out, [&] {
    fk::check_plane(src, "source");
    return fk::make_read_per_thread(*src);
  });
}
fk_status fk_op_write_per_thread(const fk_plane* dst, fk_iop** out) {
  return build(out, [&] {
    fk::check_plane(dst, "destination");
    return fk::make_write_per_thread(*dst);
  });
}
fk_status fk_op_crop(const fk_plane* src, const fk_crop_rect* rect, fk_iop** out) {
  return build(out, [&] {
    fk::check_plane(src, "source");
    if (!rect) fk::fail(FK_E_INVALID_ARGUMENT, "null crop rect");
    return fk::make_crop(*src, *rect);
  });
}
fk_status fk_op_resize(const fk_iop* up, uint32_t w, uint32_t h, uint32_t mode, fk_iop** out) {
  return build(out, [&] { return fk::make_resize(deref(up, "upstream read"), w, h, mode); });
}
fk_status fk_op_color_convert(uint32_t order, uint32_t in, fk_iop** out) {
  return build(out, [&] { return fk::make_color_convert(order, in); });
}
fk_status fk_op_split_write(const fk_plane dst[3], fk_iop** out) {
  return build(out, [&] {
    if (!dst) fk::fail(FK_E_INVALID_ARGUMENT, "null destinations");
    for (int i = 0; i < 3; ++i) fk::check_plane(&dst[i], "destination");
    return fk::make_split_write(dst);
  });
}
fk_status fk_op_batch_read(const fk_iop* const* inner, uint32_t n, uint32_t active, const void* def, fk_iop** out) {
  return build(out, [&] {
    std::vector<const fk::Op*> v;
    for (uint32_t i = 0; i < n; ++i) v.push_back(&deref(inner ? inner[i] : nullptr, "inner read"));
    return fk::make_batch_read(v, active, def);
  });
}
fk_status fk_op_batch_write(const fk_iop* const* inner, uint32_t n, uint32_t active, fk_iop** out) {
  return build(out, [&] {
    std::vector<const fk::Op*> v;
    for (uint32_t i = 0; i < n; ++i) v.push_back(&deref(inner ? inner[i] : nullptr, "inner write"));
    return fk::make_batch_write(v, active);
  });
}
fk_status fk_fold_unary_into_read(const fk_iop* read, const fk_iop* unary, fk_iop** out) {
  return build(out, [&] { return fk::fold_unary_into_read(deref(read, "read"), deref(unary, "unary")); });
}
void fk_iop_free(fk_iop* op) { delete op; }

uint32_t fk_iop_id(const fk_iop* op) { return op->op.id; }
uint32_t fk_iop_kind(const fk_iop* op) { return op->op.opkind; }
int32_t fk_iop_input_kind(const fk_iop* op) { return op->op.in_kind; }
int32_t fk_iop_output_kind(const fk_iop* op) { return op->op.out_kind; }
int32_t fk_iop_dims(const fk_iop* op, fk_extent3* out) {
  if (!op->op.dims) return 0;
  if (out) *out = *op->op.dims;
  return 1;
}

fk_status fk_validate_chain(const fk_iop* const* ops, uint32_t n, fk_pipeline** out) {
  if (!out) {
    g_err = "InvalidArgument: null output pointer";
    return FK_E_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guard([&] {
    std::vector<const fk::Op*> v;
    for (uint32_t i = 0; i < n; ++i) {
      if (!ops || !ops[i]) fk::fail(FK_E_INVALID_ARGUMENT, "null op", int(i));
      v.push_back(&ops[i]->op);
    }
    Holds h;
    for (const fk::Op* o : v) {
      Holds oh = holds_of(*o);
      h.insert(h.end(), oh.begin(), oh.end());
    }
    *out = new fk_pipeline{fk::validate_chain(v), std::move(h)};
  });
}
void fk_pipeline_free(fk_pipeline* p) { delete p; }

fk_status fk_pipeline_iter_space(const fk_pipeline* p, fk_extent3* out) {
  return guard([&] {
    if (!p || !out) fk::fail(FK_E_INVALID_ARGUMENT, "null argument");
    *out = p->p.space;
  });
}
uint32_t fk_pipeline_compute_count(const fk_pipeline* p) { return p ? uint32_t(p->p.compute.size()) : 0; }

fk_status fk_execute_fused(const fk_pipeline* p, const fk_exec_config* cfg, fk_exec_report* rep) {
  return guard([&] {
    if (!p) fk::fail(FK_E_INVALID_ARGUMENT, "null pipeline");
    const fk_exec_report r = fk::execute_fused(p->p, cfg);
    if (rep) *rep = r;
  });
}
namespace {
// FKT little-endian u32 fields (tensor_io.cpp:16-29); this library only runs on little-endian hosts
void put_u32(std::FILE* f, uint32_t v) {
  const unsigned char b[4] = {uint8_t(v), uint8_t(v >> 8), uint8_t(v >> 16), uint8_t(v >> 24)};
  if (std::fwrite(b, 1, 4, f) != 4) fk::fail(FK_E_IO_ERROR, "write failed");
}
uint32_t get_u32(std::FILE* f) {
  unsigned char b[4];
  if (std::fread(b, 1, 4, f) != 4) fk::fail(FK_E_TRUNCATED_PAYLOAD, "unexpected end of file in header");
  return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}
struct File {
  std::FILE* f;
  ~File() {
    if (f) std::fclose(f);
  }
};
}  // namespace

fk_status fk_tensor_write_file(const fk_plane* planes, uint32_t n, const char* path) {
  return guard([&] {  // tensor_io.cpp:61-83
    if (!path) fk::fail(FK_E_INVALID_ARGUMENT, "null path");
    if (n == 0 || !planes) fk::fail(FK_E_EMPTY_BATCH, "plane batch must be non-empty");
    for (uint32_t i = 0; i < n; ++i) {
      fk::check_plane(&planes[i], "plane");
      if (planes[i].kind != planes[0].kind) fk::fail(FK_E_INNER_KIND_MISMATCH, "mixed element kinds in one batch");
    }
    File out{std::fopen(path, "wb")};
    if (!out.f) fk::fail(FK_E_IO_ERROR, std::string("cannot open for writing: ") + path);
    if (std::fwrite("FKT1", 1, 4, out.f) != 4) fk::fail(FK_E_IO_ERROR, "write failed");
    put_u32(out.f, n);
    std::vector<uint8_t> host;
    for (uint32_t i = 0; i < n; ++i) {
      const fk_plane& p = planes[i];
      put_u32(out.f, p.kind);
      put_u32(out.f, p.width);
      put_u32(out.f, p.height);
      host.resize(size_t(p.width) * p.height * fk::bpe(p.kind));
      check_status(fk_plane_download(&p, host.data(), 0));
      if (std::fwrite(host.data(), 1, host.size(), out.f) != host.size())
        fk::fail(FK_E_IO_ERROR, std::string("write failed: ") + path);
    }
  });
}

fk_status fk_tensor_read_file(const char* path, fk_plane* out, uint32_t cap, uint32_t* count) {
  return guard([&] {  // tensor_io.cpp:85-109
    if (!path || !count) fk::fail(FK_E_INVALID_ARGUMENT, "null argument");
    File in{std::fopen(path, "rb")};
    if (!in.f) fk::fail(FK_E_IO_ERROR, std::string("cannot open for reading: ") + path);
    char magic[4];
    if (std::fread(magic, 1, 4, in.f) != 4) fk::fail(FK_E_TRUNCATED_PAYLOAD, "file shorter than magic");
    if (std::memcmp(magic, "FKT1", 4) != 0) fk::fail(FK_E_BAD_MAGIC, std::string("") + path);
    const uint32_t n = get_u32(in.f);
    if (n == 0) fk::fail(FK_E_EMPTY_BATCH, "file declares zero planes");
    *count = n;
    if (cap < n || !out) return;
    std::vector<fk_plane> got;
    struct Undo {  // release what was allocated when a later plane fails
      std::vector<fk_plane>& v;
      bool done = false;
      ~Undo() {
        if (!done)
          for (fk_plane& p : v) fk_plane_free(&p);
      }
    } undo{got};
    std::vector<uint8_t> host;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t tag = get_u32(in.f);
      if (tag > FK_F64X3) fk::fail(FK_E_UNKNOWN_KIND_TAG, "kind tag " + std::to_string(tag));
      const uint32_t w = get_u32(in.f), h = get_u32(in.f);
      if (!got.empty() && tag != got[0].kind) fk::fail(FK_E_INNER_KIND_MISMATCH, "mixed element kinds in one batch");
      host.resize(size_t(w) * h * fk::bpe(tag));
      if (std::fread(host.data(), 1, host.size(), in.f) != host.size())
        fk::fail(FK_E_TRUNCATED_PAYLOAD, "plane " + std::to_string(i) + " payload");
      fk_plane p{};
      check_status(fk_plane_alloc(w, h, tag, 0, &p));
      got.push_back(p);
      check_status(fk_plane_upload(&p, host.data(), 0));
    }
    for (uint32_t i = 0; i < n; ++i) out[i] = got[i];
    undo.done = true;
  });
}

fk_status fk_write_ppm(const fk_plane* plane, const char* path) {
  return guard([&] {  // tensor_io.cpp:111-124
    fk::check_plane(plane, "plane");
    if (!path) fk::fail(FK_E_INVALID_ARGUMENT, "null path");
    if (plane->kind != FK_U8X3) fk::fail(FK_E_UNSUPPORTED_KIND, "PPM export needs a u8x3 plane");
    std::vector<uint8_t> host(size_t(plane->width) * plane->height * 3);
    check_status(fk_plane_download(plane, host.data(), 0));
    File out{std::fopen(path, "wb")};
    if (!out.f) fk::fail(FK_E_IO_ERROR, std::string("cannot open for writing: ") + path);
    std::fprintf(out.f, "P6\n%u %u\n255\n", plane->width, plane->height);
    if (std::fwrite(host.data(), 1, host.size(), out.f) != host.size())
      fk::fail(FK_E_IO_ERROR, std::string("write failed: ") + path);
  });
}

fk_status fk_execute_sharded(const fk_pipeline* const* pipelines, const int32_t* devices, uint32_t n,
                             const fk_exec_config* cfgs, fk_exec_report* reports) {
  return guard([&] {
    if (n && (!pipelines || !devices)) fk::fail(FK_E_INVALID_ARGUMENT, "null pipelines / devices");
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) fk::fail(FK_E_NO_DEVICE, "no CUDA device");
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    bool timed = false;
    for (uint32_t i = 0; i < n; ++i) timed = timed || (cfgs && (cfgs[i].flags & FK_EXEC_TIMED));
    std::vector<cudaEvent_t> ev(timed ? 2 * n : 0, nullptr);
    // enqueue every shard before waiting on any (no collective)
    for (uint32_t i = 0; i < n; ++i) {
      if (!pipelines[i]) fk::fail(FK_E_INVALID_ARGUMENT, "null pipeline", int(i));
      cuda_ok(cudaSetDevice(devices[i]), "cudaSetDevice");
      fk_exec_config c = cfgs ? cfgs[i] : fk_exec_config{0, 8, 8, 0, nullptr};
      c.flags &= ~FK_EXEC_TIMED;
      cudaStream_t st = static_cast<cudaStream_t>(c.stream);
      if (timed) {
        cuda_ok(cudaEventCreate(&ev[2 * i]), "cudaEventCreate");
        cuda_ok(cudaEventCreate(&ev[2 * i + 1]), "cudaEventCreate");
        cuda_ok(cudaEventRecord(ev[2 * i], st), "cudaEventRecord");
      }
      const fk_exec_report r = fk::execute_fused(pipelines[i]->p, &c);
      if (timed) cuda_ok(cudaEventRecord(ev[2 * i + 1], st), "cudaEventRecord");
      if (reports) reports[i] = r;
    }
    for (uint32_t i = 0; timed && i < n; ++i) {
      cuda_ok(cudaSetDevice(devices[i]), "cudaSetDevice");
      cuda_ok(cudaEventSynchronize(ev[2 * i + 1]), "cudaEventSynchronize");
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      if (reports) reports[i].device_ms = ms;
      cudaEventDestroy(ev[2 * i]);
      cudaEventDestroy(ev[2 * i + 1]);
    }
  });
}

fk_status fk_gather(void* dst, int32_t dst_device, const uint64_t* dst_offsets, const void* const* srcs,
                    const int32_t* src_devices, const uint64_t* bytes, uint32_t n, void* stream) {
  return guard([&] {
    if (n && (!dst || !dst_offsets || !srcs || !src_devices || !bytes)) fk::fail(FK_E_INVALID_ARGUMENT, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (uint32_t i = 0; i < n; ++i) {
      if (src_devices[i] != dst_device) {  // peer access over NVLink when the pair supports it
        int can = 0;
        cudaDeviceCanAccessPeer(&can, dst_device, src_devices[i]);
        if (can) {
          int prev = 0;
          cudaGetDevice(&prev);
          cudaSetDevice(dst_device);
          const cudaError_t e = cudaDeviceEnablePeerAccess(src_devices[i], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            cuda_ok(e, "cudaDeviceEnablePeerAccess");
          cudaGetLastError();
          cudaSetDevice(prev);
        }
      }
      cuda_ok(cudaMemcpyPeerAsync(static_cast<uint8_t*>(dst) + dst_offsets[i], dst_device, srcs[i],
                                         src_devices[i], bytes[i], st),
                     "cudaMemcpyPeerAsync");
    }
  });
}

fk_status fk_execute_unfused(const fk_pipeline* p, const fk_exec_config* cfg, fk_exec_report* rep) {
  return guard([&] {
    if (!p) fk::fail(FK_E_INVALID_ARGUMENT, "null pipeline");
    const fk_exec_report r = fk::execute_unfused(p->p, cfg);
    if (rep) *rep = r;
  });
}
fk_status fk_plan_memory_savings(const fk_pipeline* p, uint64_t* bytes) {  // executor.cpp:223-228
  return guard([&] {
    if (!p || !bytes) fk::fail(FK_E_INVALID_ARGUMENT, "null argument");
    *bytes = fk::analytic_traffic(p->p).intermediates;
  });
}
fk_status fk_schedule(const fk_extent3* sp, const fk_exec_config* cfg, uint32_t* tasks, uint64_t cap,
                      uint64_t* count) {  // schedule, executor.cpp:52-61 (the CPU task partition)
  return guard([&] {
    if (!sp || !cfg || !count) fk::fail(FK_E_INVALID_ARGUMENT, "null argument");
    fk::check_config(cfg);
    const uint32_t chunk = uint32_t(cfg->chunk_rows);
    uint64_t n = 0;
    for (uint32_t z = 0; z < sp->batch; ++z)
      for (uint32_t y = 0; y < sp->height; y += chunk) {
        if (tasks && n < cap) {
          tasks[3 * n] = z;
          tasks[3 * n + 1] = y;
          tasks[3 * n + 2] = y + chunk < sp->height ? y + chunk : sp->height;
        }
        ++n;
      }
    *count = n;
  });
}

int32_t fk_cuda_device_info(char* buf, size_t cap) {
  const std::string s = fk::device_info();
  if (buf && cap) {
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return FK_OK;
}
uint64_t fk_cuda_kernel_launch_count(void) { return fk::launch_count(); }
const char* fk_cuda_last_kernel(void) { return fk::last_kernel(); }

fk_status fk_multi_reduce_plane(const fk_iop* read, const fk_reduce_spec* specs, uint32_t n, int32_t workers,
                                void* results, uint64_t* elements_read) {
  return guard([&] {
    const fk::Op& r = deref(read, "read op");
    if (n && (!specs || !results)) fk::fail(FK_E_INVALID_ARGUMENT, "null specs / results");
    std::vector<fk::ReduceSpecHost> hs(n);
    for (uint32_t i = 0; i < n; ++i) {
      if (specs[i].combine > FK_REDUCE_MIN) fk::fail(FK_E_INVALID_ARGUMENT, "reduce spec: unknown combine");
      hs[i].transform = specs[i].transform ? &specs[i].transform->op : nullptr;
      hs[i].combine = specs[i].combine;
      hs[i].has_identity = specs[i].has_identity != 0;
      std::memcpy(hs[i].identity.raw, specs[i].identity, 24);
    }
    const std::vector<fk::Element> out = fk::multi_reduce(r, hs, workers, nullptr, elements_read);
    for (uint32_t i = 0; i < n; ++i) std::memcpy(static_cast<uint8_t*>(results) + 24 * size_t(i), out[i].raw, 24);
  });
}

}  // extern "C"
