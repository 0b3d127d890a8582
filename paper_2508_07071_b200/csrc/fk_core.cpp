// fk_core.cpp — IOp builders, chain validation and traffic accounting.
// Each function cites the reference code whose contract it keeps.
#include "fk_core.hpp"

#include <cstdarg>
#include <cstdio>

namespace fk {

const char* errc_name(fk_status st) {  // scalar.cpp:44-72
  static const char* names[] = {"OK", "EmptyChain", "FirstNotRead", "LastNotWrite", "KindMismatch",
                                "DimsMismatch", "MissingDims", "ChainTooLong", "DivByZeroParam",
                                "UnsupportedCast", "UnsupportedKind", "CropOutOfBounds",
                                "PlaneExtentMismatch", "EmptyBatch", "InnerKindMismatch",
                                "HeterogeneousBatch", "BadStaticLoop", "BoundsError",
                                "CapacityOverflow", "BadMagic", "UnknownKindTag",
                                "TruncatedPayload", "IoError", "EmptyIterSpace", "InvalidConfig"};
  if (st >= 0 && st <= FK_E_INVALID_CONFIG) return names[st];
  switch (st) {
    case FK_E_INVALID_ARGUMENT: return "InvalidArgument";
    case FK_E_CUDA: return "CudaError";
    case FK_E_NO_DEVICE: return "NoDevice";
    case FK_E_UNSUPPORTED: return "Unsupported";
  }
  return "UnknownError";
}

void fail(fk_status st, const std::string& detail, int pos) {
  throw Error(st, std::string(errc_name(st)) + ": " + detail, pos);
}

namespace {
std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}
}  // namespace

const char* kind_name(uint32_t k) {
  static const char* n[] = {"u8", "f32", "f64", "u8x3", "f32x3", "f64x3"};
  return kind_ok(k) ? n[k] : "?";
}

const char* op_name(uint32_t id) {  // ops.cpp:8-27
  switch (id) {
    case FK_OP_PER_THREAD_READ: return "PerThreadRead";
    case FK_OP_CROP_READ: return "CropRead";
    case FK_OP_RESIZE_READ: return "ResizeRead";
    case FK_OP_BATCH_READ: return "BatchRead";
    case FK_OP_CAST: return "Cast";
    case FK_OP_SWAP_RB: return "SwapRB";
    case FK_OP_TO_GRAY: return "ToGray";
    case FK_OP_MUL: return "Mul";
    case FK_OP_ADD: return "Add";
    case FK_OP_SUB: return "Sub";
    case FK_OP_DIV: return "Div";
    case FK_OP_STATIC_LOOP: return "StaticLoop";
    case FK_OP_PER_THREAD_WRITE: return "PerThreadWrite";
    case FK_OP_SPLIT_WRITE: return "SplitWrite";
    case FK_OP_BATCH_WRITE: return "BatchWrite";
    case FK_OP_BATCH_ARITH: return "BatchArith";
  }
  return "?";
}

double lane_as_double(uint32_t kind, const Element& e, int l) {  // scalar.hpp:129-139
  switch (lane_kind(kind)) {
    case FK_U8: return e.raw[l];
    case FK_F32: { float f; std::memcpy(&f, e.raw + 4 * l, 4); return f; }
    default: { double d; std::memcpy(&d, e.raw + 8 * l, 8); return d; }
  }
}

bool is_sample_read(const Op& op) {
  return op.id == FK_OP_PER_THREAD_READ || op.id == FK_OP_CROP_READ || op.id == FK_OP_RESIZE_READ;
}

void check_plane(const fk_plane* p, const char* what) {
  if (!p || !p->data || !kind_ok(p->kind) || p->width < 1 || p->height < 1 || p->row_stride < p->width)
    fail(FK_E_INVALID_ARGUMENT, fmt("invalid %s plane", what));
}

namespace {

Op compute_op(uint32_t id, uint32_t in, uint32_t out, bool binary) {  // oplib.cpp:15-23
  Op op;
  op.id = id;
  op.opkind = binary ? FK_KIND_BINARY : FK_KIND_UNARY;
  op.in_kind = static_cast<int32_t>(in);
  op.out_kind = static_cast<int32_t>(out);
  return op;
}

bool any_lane_zero(uint32_t kind, const Element& v) {  // oplib.cpp:9-13
  for (int l = 0; l < lanes_of(kind); ++l)
    if (lane_as_double(kind, v, l) == 0.0) return true;
  return false;
}

Element element_from(uint32_t kind, const void* raw) {
  Element e;
  if (raw) std::memcpy(e.raw, raw, bpe(kind));
  return e;
}

Op sample_read(uint32_t id, Sample s) {  // make_sample_read, oplib.cpp:29-36
  Op op;
  op.id = id;
  op.opkind = FK_KIND_READ;
  op.out_kind = static_cast<int32_t>(s.output_kind());
  op.dims = fk_extent3{s.out_w, s.out_h, 1};
  op.sample = std::move(s);
  return op;
}

}  // namespace

Op make_arith(uint32_t id, uint32_t kind, const void* value) {  // make_arith, oplib.cpp:40-44
  if (id < FK_OP_MUL || id > FK_OP_DIV || !kind_ok(kind) || !value)
    fail(FK_E_INVALID_ARGUMENT, "bad arith op");
  Element v = element_from(kind, value);
  if (id == FK_OP_DIV && any_lane_zero(kind, v)) fail(FK_E_DIV_BY_ZERO_PARAM, "divide constant has a zero lane");
  Op op = compute_op(id, kind, kind, true);
  op.value = v;
  return op;
}

Op make_batch_arith(uint32_t id, uint32_t kind, const void* values, uint32_t n) {
  if (id < FK_OP_MUL || id > FK_OP_DIV || !kind_ok(kind) || !values)
    fail(FK_E_INVALID_ARGUMENT, "bad batch arith op");
  if (n == 0) fail(FK_E_EMPTY_BATCH, "batch arith over zero planes");
  Op op = compute_op(FK_OP_BATCH_ARITH, kind, kind, true);
  op.inner_id = id;
  op.values.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    op.values[i] = element_from(kind, static_cast<const uint8_t*>(values) + size_t(i) * bpe(kind));
    if (id == FK_OP_DIV && any_lane_zero(kind, op.values[i]))
      fail(FK_E_DIV_BY_ZERO_PARAM, fmt("divide constant #%u has a zero lane", i));
  }
  return op;
}

Op make_cast(uint32_t from, uint32_t to) {  // op_cast, oplib.cpp:51-56
  if (!kind_ok(from) || !kind_ok(to)) fail(FK_E_INVALID_ARGUMENT, "bad kind");
  if (lanes_of(from) != lanes_of(to)) fail(FK_E_UNSUPPORTED_CAST, fmt("%s -> %s", kind_name(from), kind_name(to)));
  return compute_op(FK_OP_CAST, from, to, false);
}

Op make_static_loop(const Op& inner, uint32_t repeat) {  // op_static_loop, oplib.cpp:58-95
  if (repeat < 1) fail(FK_E_BAD_STATIC_LOOP, "repeat must be >= 1");
  if (inner.opkind != FK_KIND_UNARY && inner.opkind != FK_KIND_BINARY)
    fail(FK_E_BAD_STATIC_LOOP, "inner op must be a compute op");
  if (inner.in_kind != inner.out_kind) fail(FK_E_BAD_STATIC_LOOP, "inner op must preserve the element kind");
  Op op = compute_op(FK_OP_STATIC_LOOP, inner.in_kind, inner.in_kind, true);
  op.value_kind = static_cast<uint32_t>(inner.in_kind);
  op.repeat = repeat;
  switch (inner.id) {
    case FK_OP_MUL: case FK_OP_ADD: case FK_OP_SUB: case FK_OP_DIV:
      op.inner_id = inner.id;
      op.value = inner.value;
      break;
    case FK_OP_SWAP_RB: case FK_OP_CAST:  // kind-preserving cast is the identity
      op.inner_id = inner.id;
      break;
    case FK_OP_STATIC_LOOP: {  // flatten: loop of a loop is one loop with the product count
      const uint64_t total = uint64_t(inner.repeat) * repeat;
      if (total > 0xffffffffull) fail(FK_E_BAD_STATIC_LOOP, "repeat count overflow");
      op.inner_id = inner.inner_id;
      op.value = inner.value;
      op.value_kind = inner.value_kind;
      op.repeat = static_cast<uint32_t>(total);
      break;
    }
    default:
      fail(FK_E_BAD_STATIC_LOOP, std::string(op_name(inner.id)) + " cannot be repeated in place");
  }
  return op;
}

Op make_read_per_thread(const fk_plane& src) {  // oplib.cpp:97-103
  Sample s;
  s.source = src;
  s.rect_w = s.out_w = src.width;
  s.rect_h = s.out_h = src.height;
  return sample_read(FK_OP_PER_THREAD_READ, std::move(s));
}

Op make_write_per_thread(const fk_plane& dst) {  // oplib.cpp:105-112
  Op op;
  op.id = FK_OP_PER_THREAD_WRITE;
  op.opkind = FK_KIND_WRITE;
  op.in_kind = static_cast<int32_t>(dst.kind);
  op.dest[0] = dst;
  op.dims = fk_extent3{dst.width, dst.height, 1};
  return op;
}

Op make_crop(const fk_plane& src, const fk_crop_rect& r) {  // oplib.cpp:114-128
  if (r.w == 0 || r.h == 0 || uint64_t(r.x0) + r.w > src.width || uint64_t(r.y0) + r.h > src.height)
    fail(FK_E_CROP_OUT_OF_BOUNDS,
         fmt("%ux%u+%u+%u exceeds %ux%u", r.w, r.h, r.x0, r.y0, src.width, src.height));
  Sample s;
  s.source = src;
  s.x0 = r.x0;
  s.y0 = r.y0;
  s.rect_w = s.out_w = r.w;
  s.rect_h = s.out_h = r.h;
  return sample_read(FK_OP_CROP_READ, std::move(s));
}

Op make_resize(const Op& up, uint32_t w, uint32_t h, uint32_t mode) {  // oplib.cpp:135-149
  if (mode > FK_BILINEAR) fail(FK_E_INVALID_ARGUMENT, "bad resize mode");
  if (w == 0 || h == 0) fail(FK_E_CROP_OUT_OF_BOUNDS, "resize target extents must be >= 1");
  if (!is_sample_read(up)) fail(FK_E_UNSUPPORTED_KIND, "resize can only sample through a crop or plane read");
  if (!up.sample.post.empty() || up.sample.resizing())
    fail(FK_E_UNSUPPORTED_KIND, "resize upstream must be a plain read or crop");
  Sample s = up.sample;
  s.out_w = w;
  s.out_h = h;
  s.mode = mode;
  return sample_read(FK_OP_RESIZE_READ, std::move(s));
}

Op make_color_convert(uint32_t order, uint32_t in) {  // oplib.cpp:151-160
  if (!kind_ok(in) || order > FK_TO_GRAY_F32) fail(FK_E_INVALID_ARGUMENT, "bad arguments");
  if (lanes_of(in) != 3) fail(FK_E_UNSUPPORTED_KIND, fmt("color conversion needs a 3-lane input, got %s", kind_name(in)));
  if (order == FK_SWAP_RB) return compute_op(FK_OP_SWAP_RB, in, in, false);
  return compute_op(FK_OP_TO_GRAY, in, FK_F32, false);
}

Op make_split_write(const fk_plane dst[3]) {  // oplib.cpp:162-176
  const uint32_t lk = dst[0].kind;
  if (lanes_of(lk) == 3) fail(FK_E_UNSUPPORTED_KIND, "split destinations must be scalar planes");
  for (int i = 0; i < 3; ++i) {
    if (dst[i].kind != lk) fail(FK_E_UNSUPPORTED_KIND, "split destinations have mixed kinds");
    if (dst[i].width != dst[0].width || dst[i].height != dst[0].height)
      fail(FK_E_PLANE_EXTENT_MISMATCH, "split destinations differ in extents");
  }
  Op op;
  op.id = FK_OP_SPLIT_WRITE;
  op.opkind = FK_KIND_WRITE;
  op.in_kind = static_cast<int32_t>(packed_kind(lk));
  for (int i = 0; i < 3; ++i) op.dest[i] = dst[i];
  op.dims = fk_extent3{dst[0].width, dst[0].height, 1};
  return op;
}

Op make_batch_read(const std::vector<const Op*>& inner, uint32_t active, const void* def) {
  // op_batch_read, oplib.cpp:178-221
  const auto n = static_cast<uint32_t>(inner.size());
  if (n == 0) fail(FK_E_EMPTY_BATCH, "batch read over zero planes");
  if (active < 1 || active > n) fail(FK_E_EMPTY_BATCH, fmt("active_count %u outside [1, %u]", active, n));
  Op op;
  op.id = FK_OP_BATCH_READ;
  op.opkind = FK_KIND_READ;
  for (uint32_t i = 0; i < n; ++i) {
    const Op& r = *inner[i];
    if (!is_sample_read(r)) fail(FK_E_INNER_KIND_MISMATCH, fmt("batch inner #%u is not a per-plane read", i));
    if (i == 0) {
      op.out_kind = r.out_kind;
      op.dims = r.dims;
    } else if (r.out_kind != op.out_kind) {
      fail(FK_E_INNER_KIND_MISMATCH, fmt("batch inner #%u yields %s, expected %s", i,
                                         kind_name(uint32_t(r.out_kind)), kind_name(uint32_t(op.out_kind))));
    } else if (r.dims->width != op.dims->width || r.dims->height != op.dims->height ||
               r.dims->batch != op.dims->batch) {
      fail(FK_E_HETEROGENEOUS_BATCH, fmt("batch inner #%u extents differ", i), int(i));
    }
    op.planes.push_back(r.sample);
  }
  op.active = active;
  op.def = element_from(uint32_t(op.out_kind), def);
  op.dims->batch = n;
  return op;
}

Op make_batch_write(const std::vector<const Op*>& inner, uint32_t active) {  // oplib.cpp:223-256
  const auto n = static_cast<uint32_t>(inner.size());
  if (n == 0) fail(FK_E_EMPTY_BATCH, "batch write over zero planes");
  if (active < 1 || active > n) fail(FK_E_EMPTY_BATCH, fmt("active_count %u outside [1, %u]", active, n));
  Op op;
  op.id = FK_OP_BATCH_WRITE;
  op.opkind = FK_KIND_WRITE;
  op.w_inner = inner[0]->id;
  op.active = active;
  const int per = op.w_inner == FK_OP_SPLIT_WRITE ? 3 : 1;
  for (uint32_t i = 0; i < n; ++i) {
    const Op& w = *inner[i];
    if (w.id != op.w_inner || (w.id != FK_OP_PER_THREAD_WRITE && w.id != FK_OP_SPLIT_WRITE))
      fail(FK_E_INNER_KIND_MISMATCH, fmt("batch inner #%u is not a uniform per-plane write", i));
    if (i == 0) {
      op.in_kind = w.in_kind;
      op.dims = w.dims;
    } else if (w.in_kind != op.in_kind) {
      fail(FK_E_INNER_KIND_MISMATCH, fmt("batch inner #%u input kind", i));
    } else if (w.dims->width != op.dims->width || w.dims->height != op.dims->height ||
               w.dims->batch != op.dims->batch) {
      fail(FK_E_HETEROGENEOUS_BATCH, fmt("batch inner #%u extents differ", i), int(i));
    }
    for (int l = 0; l < per; ++l) op.wdest.push_back(w.dest[l]);
  }
  op.dims->batch = n;
  return op;
}

Op fold_unary_into_read(const Op& read, const Op& unary) {  // oplib.cpp:264-274
  if (!is_sample_read(read)) fail(FK_E_UNSUPPORTED_KIND, "can only fold into a per-plane read");
  if (unary.opkind != FK_KIND_UNARY) fail(FK_E_UNSUPPORTED_KIND, "only parameter-free unary ops fold into a read");
  if (unary.in_kind != read.out_kind) fail(FK_E_KIND_MISMATCH, "fold input kind does not match read output");
  Sample s = read.sample;
  s.post.push_back(Folded{unary.id, uint32_t(unary.in_kind), uint32_t(unary.out_kind)});
  return sample_read(read.id, std::move(s));
}

Pipeline validate_chain(const std::vector<const Op*>& ops) {  // validate_chain, ops.cpp:37-82
  const auto n = static_cast<uint32_t>(ops.size());
  if (n == 0) fail(FK_E_EMPTY_CHAIN, "chain has no ops");
  if (n > 4096) fail(FK_E_CHAIN_TOO_LONG, fmt("%u ops; limit is 4096", n));
  if (ops[0]->opkind != FK_KIND_READ) fail(FK_E_FIRST_NOT_READ, fmt("%s at position 0", op_name(ops[0]->id)), 0);
  const int last = int(n) - 1;
  if (ops[last]->opkind != FK_KIND_WRITE)
    fail(FK_E_LAST_NOT_WRITE, fmt("%s at position %d", op_name(ops[last]->id), last), last);
  int32_t cur = ops[0]->out_kind;
  for (int i = 1; i <= last; ++i) {
    const Op& op = *ops[i];
    if (i != last && (op.opkind == FK_KIND_READ || op.opkind == FK_KIND_WRITE))
      fail(FK_E_KIND_MISMATCH, fmt("expected a compute op at position %d, found %s", i, op_name(op.id)), i);
    if (op.in_kind != cur)
      fail(FK_E_KIND_MISMATCH, fmt("position %d: expected %s, found %s", i, kind_name(uint32_t(cur)),
                                   kind_name(uint32_t(op.in_kind))), i);
    if (op.out_kind >= 0) cur = op.out_kind;
  }
  if (!ops[0]->dims) fail(FK_E_MISSING_DIMS, fmt("%s has no dims hint", op_name(ops[0]->id)));
  const fk_extent3 sp = *ops[0]->dims;
  if (!ops[last]->dims) fail(FK_E_MISSING_DIMS, "write op has no dims hint", last);
  const fk_extent3 wd = *ops[last]->dims;
  if (wd.width != sp.width || wd.height != sp.height || wd.batch != sp.batch)
    fail(FK_E_DIMS_MISMATCH, fmt("read space %ux%ux%u vs write hint", sp.width, sp.height, sp.batch), last);
  Pipeline p;
  p.read = *ops[0];
  for (uint32_t i = 1; i + 1 < n; ++i) p.compute.push_back(*ops[i]);
  p.write = *ops[last];
  p.space = sp;
  return p;
}

uint32_t read_count(const Pipeline& p) {
  return p.read.id == FK_OP_BATCH_READ ? uint32_t(p.read.planes.size()) : 1u;
}

const Sample* read_plane(const Pipeline& p, uint32_t z) {
  if (p.read.id != FK_OP_BATCH_READ) return &p.read.sample;
  return z < p.read.active ? &p.read.planes[z] : nullptr;
}

uint32_t write_active(const Pipeline& p) {
  return p.write.id == FK_OP_BATCH_WRITE ? p.write.active : p.space.batch;
}

Traffic analytic_traffic(const Pipeline& p) {
  Traffic t;
  const uint64_t pts = uint64_t(p.space.width) * p.space.height;
  // sample_block counts touched source elements x bpe(source): 1 tap direct /
  // nearest, 4 taps bilinear (ops.cpp:327-344); default-value planes read nothing.
  for (uint32_t z = 0; z < p.space.batch; ++z) {
    const Sample* s = read_plane(p, z);
    if (!s) continue;
    const uint64_t taps = (s->resizing() && s->mode == FK_BILINEAR) ? 4 : 1;
    t.fused_read += pts * taps * bpe(s->source.kind);
  }
  // store_block / split_block (ops.cpp:396-424); inactive BatchWrite planes skip.
  const uint32_t wk = uint32_t(p.write.in_kind);
  t.fused_written = uint64_t(write_active(p)) * pts * bpe(wk);
  // execute_unfused (executor.cpp:134-217): pass 0 reads through the read op,
  // later passes load the previous intermediate, every pass stores every z.
  const uint64_t all = pts * p.space.batch;
  t.unfused_read = t.fused_read;
  t.unfused_written = t.fused_written;
  for (size_t i = 0; i < p.compute.size(); ++i) {
    const uint64_t b = all * bpe(uint32_t(p.compute[i].out_kind));
    t.intermediates += b;
    t.unfused_written += b;  // pass i stores its intermediate
    t.unfused_read += b;     // pass i+1 (or the final write pass) loads it
  }
  return t;
}

}  // namespace fk
