/*
 * fk_oracle.c — TEST INFRASTRUCTURE ONLY. A plain-C restatement of the
 * reference's fused operation-chain path (arxiv 2508.07071 "opfuse" CPU artifact,
 * /root/reference/proj), exporting the include/fk.h ABI over HOST memory.
 *
 * It is the checker for the CUDA product (libfk_cuda.so): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. Nothing
 * on the product path links or calls it.
 *
 * Parity pinning: this restatement is checked bit-for-bit against the compiled
 * reference itself (oracle/_ref/libfk_ref.so, built from the unmodified sources
 * by oracle/Makefile) and against the committed golden vectors in tests/golden/
 * (tests/test_oracle.py).
 *
 * Build: gcc -std=c11 -O2 -fopenmp -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off keeps every float/double op a separately rounded IEEE op,
 * as the reference's x86-64 SSE2 build does (no FMA at the default -march).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/fk.h"

/* ---------------------------------------------------------------- errors -- */

static __thread char g_err[1024];
static __thread int32_t g_err_pos = -1;

static const char* errc_name(int32_t st) { /* scalar.cpp:44-72 */
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

static fk_status fail(fk_status st, int32_t pos, const char* fmt, ...) {
  /* errors.hpp:45-66: message is "<ErrcName>: <detail>" */
  va_list ap;
  int n = snprintf(g_err, sizeof g_err, "%s: ", errc_name(st));
  va_start(ap, fmt);
  vsnprintf(g_err + n, sizeof g_err - (size_t)n, fmt, ap);
  va_end(ap);
  g_err_pos = pos;
  return st;
}

const char* fk_backend_name(void) { return "oracle-c"; }
int32_t fk_abi_version(void) { return FK_ABI_VERSION; }
const char* fk_last_error(void) { return g_err; }
int32_t fk_last_error_position(void) { return g_err_pos; }
int32_t fk_errc_name(int32_t status, char* buf, size_t cap) {
  const char* s = errc_name(status);
  if (buf && cap) { strncpy(buf, s, cap - 1); buf[cap - 1] = 0; }
  return (int32_t)strlen(s);
}

/* ---------------------------------------------------------------- kinds -- */

static int kind_ok(uint32_t k) { return k <= FK_F64X3; }
uint32_t fk_bytes_per_element(uint32_t k) { /* scalar.hpp:27-37 */
  static const uint32_t b[] = {1, 4, 8, 3, 12, 24};
  return kind_ok(k) ? b[k] : 0;
}
static int lane_count(uint32_t k) { return k >= FK_U8X3 ? 3 : 1; }       /* scalar.hpp:39-46 */
static uint32_t lane_kind(uint32_t k) { return k >= FK_U8X3 ? k - 3 : k; } /* scalar.hpp:51-58 */
static uint32_t packed_kind(uint32_t k) { return k < FK_U8X3 ? k + 3 : k; } /* scalar.hpp:61-68 */
static const char* kind_name(uint32_t k) {
  static const char* n[] = {"u8", "f32", "f64", "u8x3", "f32x3", "f64x3"};
  return kind_ok(k) ? n[k] : "?";
}

/* Element, scalar.hpp:94-121: 24-byte union; lanes in the exact precision of the kind. */
typedef union elem {
  uint8_t u8v[3];
  float f32v[3];
  double f64v[3];
  uint8_t raw[24];
} elem_t;

static double lane_as_double(uint32_t k, const elem_t* e, int l) { /* scalar.hpp:129-139 */
  switch (lane_kind(k)) {
    case FK_U8: return e->u8v[l];
    case FK_F32: return e->f32v[l];
    default: return e->f64v[l];
  }
}

/* round_clamp_u8, scalar.hpp:161-167: NaN->0, nearbyint (ties-to-even), clamp. */
static uint8_t round_clamp_u8(double x) {
  if (isnan(x)) return 0;
  double r = nearbyint(x);
  if (r < 0.0) return 0;
  if (r > 255.0) return 255;
  return (uint8_t)r;
}

/* set_lane, scalar.cpp:21-31 */
static void set_lane(uint32_t to, elem_t* out, int l, double x) {
  switch (lane_kind(to)) {
    case FK_U8: out->u8v[l] = round_clamp_u8(x); break;
    case FK_F32: out->f32v[l] = (float)x; break;
    default: out->f64v[l] = x; break;
  }
}

/* cast_element, scalar.cpp:35-42 (lane counts already checked at op construction) */
static void cast_element(uint32_t from, uint32_t to, elem_t* v) {
  if (from == to) return;
  elem_t out;
  memset(&out, 0, sizeof out);
  for (int l = 0; l < lane_count(from); ++l) set_lane(to, &out, l, lane_as_double(from, v, l));
  *v = out;
}

/* ------------------------------------------------------------ IOp model -- */

typedef struct folded { uint32_t id, in, out; } folded_t; /* FoldedUnary, ops.hpp:70-74 */

typedef struct sample { /* SampleReadParams, ops.hpp:78-91 */
  fk_plane source;
  uint32_t x0, y0, rect_w, rect_h, out_w, out_h, mode;
  uint32_t n_post;
  folded_t* post;
} sample_t;

struct fk_iop {
  uint32_t id, opkind;
  int32_t in_kind, out_kind; /* -1 = absent */
  int has_dims;
  fk_extent3 dims;
  /* ArithParams (ops.hpp:93-95) / StaticLoopParams (ops.hpp:97-102) */
  elem_t value;
  uint32_t inner_id, value_kind, repeat;
  /* BatchArith extension: one constant per z */
  elem_t* values;
  uint32_t n_values;
  /* sample reads */
  sample_t sample;
  /* BatchReadParams, ops.hpp:108-112 */
  sample_t* planes;
  uint32_t n_planes, active;
  elem_t def;
  /* WriteParams / SplitWriteParams / BatchWriteParams, ops.hpp:104-123 */
  fk_plane dest[3];
  uint32_t w_inner; /* BatchWrite inner id */
  fk_plane* wdest;  /* n_planes * (1 or 3) */
};

struct fk_pipeline {
  fk_iop* read;
  fk_iop** compute;
  uint32_t n_compute;
  fk_iop* write;
  fk_extent3 space;
};

static fk_iop* new_iop(uint32_t id, uint32_t opkind, int32_t in, int32_t out) {
  fk_iop* op = (fk_iop*)calloc(1, sizeof(fk_iop));
  op->id = id;
  op->opkind = opkind;
  op->in_kind = in;
  op->out_kind = out;
  return op;
}

static void sample_copy(sample_t* dst, const sample_t* src) {
  *dst = *src;
  dst->post = NULL;
  if (src->n_post) {
    dst->post = (folded_t*)malloc(sizeof(folded_t) * src->n_post);
    memcpy(dst->post, src->post, sizeof(folded_t) * src->n_post);
  }
}

static fk_iop* clone_iop(const fk_iop* s) {
  fk_iop* d = (fk_iop*)malloc(sizeof(fk_iop));
  *d = *s;
  sample_copy(&d->sample, &s->sample);
  if (s->values) {
    d->values = (elem_t*)malloc(sizeof(elem_t) * s->n_values);
    memcpy(d->values, s->values, sizeof(elem_t) * s->n_values);
  }
  if (s->planes) {
    d->planes = (sample_t*)malloc(sizeof(sample_t) * s->n_planes);
    for (uint32_t i = 0; i < s->n_planes; ++i) sample_copy(&d->planes[i], &s->planes[i]);
  }
  if (s->wdest) {
    size_t n = (size_t)s->n_planes * (s->w_inner == FK_OP_SPLIT_WRITE ? 3 : 1);
    d->wdest = (fk_plane*)malloc(sizeof(fk_plane) * n);
    memcpy(d->wdest, s->wdest, sizeof(fk_plane) * n);
  }
  return d;
}

void fk_iop_free(fk_iop* op) {
  if (!op) return;
  free(op->sample.post);
  free(op->values);
  if (op->planes)
    for (uint32_t i = 0; i < op->n_planes; ++i) free(op->planes[i].post);
  free(op->planes);
  free(op->wdest);
  free(op);
}

uint32_t fk_iop_id(const fk_iop* op) { return op->id; }
uint32_t fk_iop_kind(const fk_iop* op) { return op->opkind; }
int32_t fk_iop_input_kind(const fk_iop* op) { return op->in_kind; }
int32_t fk_iop_output_kind(const fk_iop* op) { return op->out_kind; }
int32_t fk_iop_dims(const fk_iop* op, fk_extent3* out) {
  if (op->has_dims && out) *out = op->dims;
  return op->has_dims;
}

static int plane_ok(const fk_plane* p) {
  return p && p->data && kind_ok(p->kind) && p->width >= 1 && p->height >= 1 &&
         p->row_stride >= p->width;
}

fk_status fk_plane_view(const fk_plane* p, uint32_t x0, uint32_t y0, uint32_t w, uint32_t h,
                        fk_plane* out) { /* Plane::view, plane.cpp:91-101 */
  if (!plane_ok(p) || !out) return fail(FK_E_INVALID_ARGUMENT, -1, "invalid plane");
  if (w == 0 || h == 0 || (uint64_t)x0 + w > p->width || (uint64_t)y0 + h > p->height)
    return fail(FK_E_BOUNDS_ERROR, -1, "sub-view outside plane");
  *out = *p;
  out->data = (uint8_t*)p->data +
              ((uint64_t)y0 * p->row_stride + x0) * fk_bytes_per_element(p->kind);
  out->width = w;
  out->height = h;
  return FK_OK;
}

fk_status fk_plane_alloc(uint32_t width, uint32_t height, uint32_t kind, uint32_t row_stride, fk_plane* out) {
  /* Plane::alloc, plane.cpp:60-71: host memory, zero-initialised. The oracle is
     test infrastructure: the caller keeps the buffer alive until fk_plane_free. */
  if (!out || !kind_ok(kind)) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: bad plane arguments");
  uint32_t rs = row_stride ? row_stride : width;
  if (width == 0 || height == 0 || rs < width) return fail(FK_E_CAPACITY_OVERFLOW, -1, "CapacityOverflow: extents");
  void* p = calloc((size_t)rs * height, fk_bytes_per_element(kind));
  if (!p) return fail(FK_E_CAPACITY_OVERFLOW, -1, "CapacityOverflow: host allocation failed");
  out->data = p;
  out->width = width;
  out->height = height;
  out->row_stride = rs;
  out->kind = kind;
  return FK_OK;
}
void fk_plane_free(fk_plane* p) {
  if (p && p->data) {
    free(p->data);
    p->data = NULL;
  }
}

static fk_status plane_copy(const fk_plane* p, void* host, size_t host_pitch, int up) {
  if (!plane_ok(p) || !host) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: bad plane copy");
  size_t row = (size_t)p->width * fk_bytes_per_element(p->kind);
  size_t hp = host_pitch ? host_pitch : row, pp = (size_t)p->row_stride * fk_bytes_per_element(p->kind);
  for (uint32_t y = 0; y < p->height; ++y) {
    uint8_t* dev = (uint8_t*)p->data + y * pp;
    uint8_t* h = (uint8_t*)host + y * hp;
    if (up) memcpy(dev, h, row);
    else memcpy(h, dev, row);
  }
  return FK_OK;
}
fk_status fk_plane_upload(const fk_plane* dst, const void* host, size_t host_pitch) {
  return plane_copy(dst, (void*)host, host_pitch, 1);
}
fk_status fk_plane_download(const fk_plane* src, void* host, size_t host_pitch) {
  return plane_copy(src, host, host_pitch, 0);
}

/* ---- FKT files: tensor_io.cpp:12-117 restated (little-endian host) ---- */
static int put_u32(FILE* f, uint32_t v) {
  unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16), (unsigned char)(v >> 24)};
  return fwrite(b, 1, 4, f) == 4;
}
static int get_u32(FILE* f, uint32_t* v) {
  unsigned char b[4];
  if (fread(b, 1, 4, f) != 4) return 0;
  *v = (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
  return 1;
}
fk_status fk_tensor_write_file(const fk_plane* planes, uint32_t n, const char* path) {
  if (!path) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: null path");
  if (n == 0 || !planes) return fail(FK_E_EMPTY_BATCH, -1, "EmptyBatch: plane batch must be non-empty");
  for (uint32_t i = 0; i < n; ++i) {
    if (!plane_ok(&planes[i])) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: invalid plane");
    if (planes[i].kind != planes[0].kind)
      return fail(FK_E_INNER_KIND_MISMATCH, -1, "InnerKindMismatch: mixed element kinds in one batch");
  }
  FILE* f = fopen(path, "wb");
  if (!f) return fail(FK_E_IO_ERROR, -1, "IoError: cannot open for writing: %s", path);
  int ok = fwrite("FKT1", 1, 4, f) == 4 && put_u32(f, n);
  for (uint32_t i = 0; i < n && ok; ++i) {
    const fk_plane* p = &planes[i];
    size_t row = (size_t)p->width * fk_bytes_per_element(p->kind);
    ok = put_u32(f, p->kind) && put_u32(f, p->width) && put_u32(f, p->height);
    for (uint32_t y = 0; y < p->height && ok; ++y)
      ok = fwrite((const uint8_t*)p->data + (size_t)y * p->row_stride * fk_bytes_per_element(p->kind), 1, row, f) == row;
  }
  fclose(f);
  return ok ? FK_OK : fail(FK_E_IO_ERROR, -1, "IoError: write failed: %s", path);
}
fk_status fk_tensor_read_file(const char* path, fk_plane* out, uint32_t cap, uint32_t* count) {
  if (!path || !count) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: null argument");
  FILE* f = fopen(path, "rb");
  if (!f) return fail(FK_E_IO_ERROR, -1, "IoError: cannot open for reading: %s", path);
  char magic[4];
  uint32_t n = 0;
  fk_status st = FK_OK;
  if (fread(magic, 1, 4, f) != 4) st = fail(FK_E_TRUNCATED_PAYLOAD, -1, "TruncatedPayload: file shorter than magic");
  else if (memcmp(magic, "FKT1", 4) != 0) st = fail(FK_E_BAD_MAGIC, -1, "BadMagic: %s", path);
  else if (!get_u32(f, &n)) st = fail(FK_E_TRUNCATED_PAYLOAD, -1, "TruncatedPayload: unexpected end of file in header");
  else if (n == 0) st = fail(FK_E_EMPTY_BATCH, -1, "EmptyBatch: file declares zero planes");
  if (st != FK_OK) { fclose(f); return st; }
  *count = n;
  if (cap < n || !out) { fclose(f); return FK_OK; }
  uint32_t got = 0;
  for (; got < n && st == FK_OK; ++got) {
    uint32_t tag, w, h;
    if (!get_u32(f, &tag)) { st = fail(FK_E_TRUNCATED_PAYLOAD, -1, "TruncatedPayload: unexpected end of file in header"); break; }
    if (tag > FK_F64X3) { st = fail(FK_E_UNKNOWN_KIND_TAG, -1, "UnknownKindTag: kind tag %u", tag); break; }
    if (!get_u32(f, &w) || !get_u32(f, &h)) { st = fail(FK_E_TRUNCATED_PAYLOAD, -1, "TruncatedPayload: unexpected end of file in header"); break; }
    if (got > 0 && tag != out[0].kind) { st = fail(FK_E_INNER_KIND_MISMATCH, -1, "InnerKindMismatch: mixed element kinds in one batch"); break; }
    if ((st = fk_plane_alloc(w, h, tag, 0, &out[got])) != FK_OK) break;
    size_t bytes = (size_t)w * h * fk_bytes_per_element(tag);
    if (fread(out[got].data, 1, bytes, f) != bytes) {
      fk_plane_free(&out[got]);
      st = fail(FK_E_TRUNCATED_PAYLOAD, -1, "TruncatedPayload: plane %u payload", got);
      break;
    }
  }
  fclose(f);
  if (st != FK_OK)
    for (uint32_t i = 0; i < got; ++i) fk_plane_free(&out[i]);
  return st;
}
fk_status fk_write_ppm(const fk_plane* p, const char* path) {
  if (!plane_ok(p) || !path) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: bad arguments");
  if (p->kind != FK_U8X3) return fail(FK_E_UNSUPPORTED_KIND, -1, "UnsupportedKind: PPM export needs a u8x3 plane");
  FILE* f = fopen(path, "wb");
  if (!f) return fail(FK_E_IO_ERROR, -1, "IoError: cannot open for writing: %s", path);
  int ok = fprintf(f, "P6\n%u %u\n255\n", p->width, p->height) > 0;
  for (uint32_t y = 0; y < p->height && ok; ++y)
    ok = fwrite((const uint8_t*)p->data + (size_t)y * p->row_stride * 3, 1, (size_t)p->width * 3, f) == (size_t)p->width * 3;
  fclose(f);
  return ok ? FK_OK : fail(FK_E_IO_ERROR, -1, "IoError: write failed: %s", path);
}

static int sample_resizing(const sample_t* s) { return s->out_w != s->rect_w || s->out_h != s->rect_h; }
static uint32_t sample_out_kind(const sample_t* s) { /* ops.hpp:88-90 */
  return s->n_post ? s->post[s->n_post - 1].out : s->source.kind;
}
static int is_sample_read(const fk_iop* op) {
  return op->id == FK_OP_PER_THREAD_READ || op->id == FK_OP_CROP_READ || op->id == FK_OP_RESIZE_READ;
}

static fk_iop* make_sample_read(uint32_t id, const sample_t* s) { /* oplib.cpp:29-36 */
  fk_iop* op = new_iop(id, FK_KIND_READ, -1, (int32_t)sample_out_kind(s));
  sample_copy(&op->sample, s);
  op->has_dims = 1;
  op->dims.width = s->out_w;
  op->dims.height = s->out_h;
  op->dims.batch = 1;
  return op;
}

/* -------------------------------------------------------------- builders -- */

#define CHECK_OUT(out) \
  do { if (!(out)) return fail(FK_E_INVALID_ARGUMENT, -1, "null output pointer"); *(out) = NULL; } while (0)

static int any_lane_zero(uint32_t kind, const elem_t* v) { /* oplib.cpp:9-13 */
  for (int l = 0; l < lane_count(kind); ++l)
    if (lane_as_double(kind, v, l) == 0.0) return 1;
  return 0;
}

fk_status fk_op_arith(uint32_t op_id, uint32_t kind, const void* value, fk_iop** out) {
  /* make_arith, oplib.cpp:40-44 */
  CHECK_OUT(out);
  if (op_id < FK_OP_MUL || op_id > FK_OP_DIV || !kind_ok(kind) || !value)
    return fail(FK_E_INVALID_ARGUMENT, -1, "bad arith op");
  elem_t v;
  memset(&v, 0, sizeof v);
  memcpy(v.raw, value, fk_bytes_per_element(kind));
  if (op_id == FK_OP_DIV && any_lane_zero(kind, &v))
    return fail(FK_E_DIV_BY_ZERO_PARAM, -1, "divide constant has a zero lane");
  fk_iop* op = new_iop(op_id, FK_KIND_BINARY, (int32_t)kind, (int32_t)kind);
  op->value = v;
  *out = op;
  return FK_OK;
}

fk_status fk_op_batch_arith(uint32_t op_id, uint32_t kind, const void* values, uint32_t n,
                            fk_iop** out) {
  CHECK_OUT(out);
  if (op_id < FK_OP_MUL || op_id > FK_OP_DIV || !kind_ok(kind) || !values)
    return fail(FK_E_INVALID_ARGUMENT, -1, "bad batch arith op");
  if (n == 0) return fail(FK_E_EMPTY_BATCH, -1, "batch arith over zero planes");
  const uint32_t bpe = fk_bytes_per_element(kind);
  elem_t* vs = (elem_t*)calloc(n, sizeof(elem_t));
  for (uint32_t i = 0; i < n; ++i) {
    memcpy(vs[i].raw, (const uint8_t*)values + (size_t)i * bpe, bpe);
    if (op_id == FK_OP_DIV && any_lane_zero(kind, &vs[i])) {
      free(vs);
      return fail(FK_E_DIV_BY_ZERO_PARAM, -1, "divide constant #%u has a zero lane", i);
    }
  }
  fk_iop* op = new_iop(FK_OP_BATCH_ARITH, FK_KIND_BINARY, (int32_t)kind, (int32_t)kind);
  op->inner_id = op_id;
  op->values = vs;
  op->n_values = n;
  *out = op;
  return FK_OK;
}

fk_status fk_op_cast(uint32_t from, uint32_t to, fk_iop** out) { /* oplib.cpp:51-56 */
  CHECK_OUT(out);
  if (!kind_ok(from) || !kind_ok(to)) return fail(FK_E_INVALID_ARGUMENT, -1, "bad kind");
  if (lane_count(from) != lane_count(to))
    return fail(FK_E_UNSUPPORTED_CAST, -1, "%s -> %s", kind_name(from), kind_name(to));
  *out = new_iop(FK_OP_CAST, FK_KIND_UNARY, (int32_t)from, (int32_t)to);
  return FK_OK;
}

fk_status fk_op_static_loop(const fk_iop* inner, uint32_t repeat, fk_iop** out) {
  /* op_static_loop, oplib.cpp:58-95 */
  CHECK_OUT(out);
  if (!inner) return fail(FK_E_INVALID_ARGUMENT, -1, "null inner op");
  if (repeat < 1) return fail(FK_E_BAD_STATIC_LOOP, -1, "repeat must be >= 1");
  if (inner->opkind != FK_KIND_UNARY && inner->opkind != FK_KIND_BINARY)
    return fail(FK_E_BAD_STATIC_LOOP, -1, "inner op must be a compute op");
  if (inner->in_kind != inner->out_kind)
    return fail(FK_E_BAD_STATIC_LOOP, -1, "inner op must preserve the element kind");
  fk_iop* op = new_iop(FK_OP_STATIC_LOOP, FK_KIND_BINARY, inner->in_kind, inner->in_kind);
  op->value_kind = (uint32_t)inner->in_kind;
  op->repeat = repeat;
  switch (inner->id) {
    case FK_OP_MUL: case FK_OP_ADD: case FK_OP_SUB: case FK_OP_DIV:
      op->inner_id = inner->id;
      op->value = inner->value;
      break;
    case FK_OP_SWAP_RB: case FK_OP_CAST:
      op->inner_id = inner->id;
      break;
    case FK_OP_STATIC_LOOP: {
      const uint64_t total = (uint64_t)inner->repeat * repeat;
      if (total > 0xffffffffull) { fk_iop_free(op); return fail(FK_E_BAD_STATIC_LOOP, -1, "repeat count overflow"); }
      op->inner_id = inner->inner_id;
      op->value = inner->value;
      op->value_kind = inner->value_kind;
      op->repeat = (uint32_t)total;
      break;
    }
    default:
      fk_iop_free(op);
      return fail(FK_E_BAD_STATIC_LOOP, -1, "op %u cannot be repeated in place", inner->id);
  }
  *out = op;
  return FK_OK;
}

fk_status fk_op_read_per_thread(const fk_plane* src, fk_iop** out) { /* oplib.cpp:97-103 */
  CHECK_OUT(out);
  if (!plane_ok(src)) return fail(FK_E_INVALID_ARGUMENT, -1, "invalid source plane");
  sample_t s;
  memset(&s, 0, sizeof s);
  s.source = *src;
  s.rect_w = s.out_w = src->width;
  s.rect_h = s.out_h = src->height;
  *out = make_sample_read(FK_OP_PER_THREAD_READ, &s);
  return FK_OK;
}

fk_status fk_op_write_per_thread(const fk_plane* dst, fk_iop** out) { /* oplib.cpp:105-112 */
  CHECK_OUT(out);
  if (!plane_ok(dst)) return fail(FK_E_INVALID_ARGUMENT, -1, "invalid destination plane");
  fk_iop* op = new_iop(FK_OP_PER_THREAD_WRITE, FK_KIND_WRITE, (int32_t)dst->kind, -1);
  op->dest[0] = *dst;
  op->has_dims = 1;
  op->dims.width = dst->width;
  op->dims.height = dst->height;
  op->dims.batch = 1;
  *out = op;
  return FK_OK;
}

fk_status fk_op_crop(const fk_plane* src, const fk_crop_rect* r, fk_iop** out) { /* oplib.cpp:114-128 */
  CHECK_OUT(out);
  if (!plane_ok(src) || !r) return fail(FK_E_INVALID_ARGUMENT, -1, "invalid crop arguments");
  if (r->w == 0 || r->h == 0 || (uint64_t)r->x0 + r->w > src->width ||
      (uint64_t)r->y0 + r->h > src->height)
    return fail(FK_E_CROP_OUT_OF_BOUNDS, -1, "%ux%u+%u+%u exceeds %ux%u", r->w, r->h, r->x0, r->y0,
                src->width, src->height);
  sample_t s;
  memset(&s, 0, sizeof s);
  s.source = *src;
  s.x0 = r->x0;
  s.y0 = r->y0;
  s.rect_w = s.out_w = r->w;
  s.rect_h = s.out_h = r->h;
  *out = make_sample_read(FK_OP_CROP_READ, &s);
  return FK_OK;
}

fk_status fk_op_resize(const fk_iop* up, uint32_t w, uint32_t h, uint32_t mode, fk_iop** out) {
  /* op_resize, oplib.cpp:135-149 */
  CHECK_OUT(out);
  if (!up || mode > FK_BILINEAR) return fail(FK_E_INVALID_ARGUMENT, -1, "invalid resize arguments");
  if (w == 0 || h == 0) return fail(FK_E_CROP_OUT_OF_BOUNDS, -1, "resize target extents must be >= 1");
  if (!is_sample_read(up))
    return fail(FK_E_UNSUPPORTED_KIND, -1, "resize can only sample through a crop or plane read");
  if (up->sample.n_post || sample_resizing(&up->sample))
    return fail(FK_E_UNSUPPORTED_KIND, -1, "resize upstream must be a plain read or crop");
  sample_t s = up->sample;
  s.out_w = w;
  s.out_h = h;
  s.mode = mode;
  *out = make_sample_read(FK_OP_RESIZE_READ, &s);
  return FK_OK;
}

fk_status fk_op_color_convert(uint32_t order, uint32_t in, fk_iop** out) { /* oplib.cpp:151-160 */
  CHECK_OUT(out);
  if (!kind_ok(in) || order > FK_TO_GRAY_F32) return fail(FK_E_INVALID_ARGUMENT, -1, "bad arguments");
  if (lane_count(in) != 3)
    return fail(FK_E_UNSUPPORTED_KIND, -1, "color conversion needs a 3-lane input, got %s", kind_name(in));
  if (order == FK_SWAP_RB)
    *out = new_iop(FK_OP_SWAP_RB, FK_KIND_UNARY, (int32_t)in, (int32_t)in);
  else
    *out = new_iop(FK_OP_TO_GRAY, FK_KIND_UNARY, (int32_t)in, FK_F32);
  return FK_OK;
}

fk_status fk_op_split_write(const fk_plane dst[3], fk_iop** out) { /* oplib.cpp:162-176 */
  CHECK_OUT(out);
  if (!dst) return fail(FK_E_INVALID_ARGUMENT, -1, "null destinations");
  for (int i = 0; i < 3; ++i)
    if (!plane_ok(&dst[i])) return fail(FK_E_INVALID_ARGUMENT, -1, "invalid destination plane");
  const uint32_t lk = dst[0].kind;
  if (lane_count(lk) == 3) return fail(FK_E_UNSUPPORTED_KIND, -1, "split destinations must be scalar planes");
  for (int i = 0; i < 3; ++i) {
    if (dst[i].kind != lk) return fail(FK_E_UNSUPPORTED_KIND, -1, "split destinations have mixed kinds");
    if (dst[i].width != dst[0].width || dst[i].height != dst[0].height)
      return fail(FK_E_PLANE_EXTENT_MISMATCH, -1, "split destinations differ in extents");
  }
  fk_iop* op = new_iop(FK_OP_SPLIT_WRITE, FK_KIND_WRITE, (int32_t)packed_kind(lk), -1);
  memcpy(op->dest, dst, sizeof(fk_plane) * 3);
  op->has_dims = 1;
  op->dims.width = dst[0].width;
  op->dims.height = dst[0].height;
  op->dims.batch = 1;
  *out = op;
  return FK_OK;
}

fk_status fk_op_batch_read(const fk_iop* const* inner, uint32_t n, uint32_t active,
                           const void* def, fk_iop** out) { /* op_batch_read, oplib.cpp:178-221 */
  CHECK_OUT(out);
  if (n == 0 || !inner) return fail(FK_E_EMPTY_BATCH, -1, "batch read over zero planes");
  if (active < 1 || active > n)
    return fail(FK_E_EMPTY_BATCH, -1, "active_count %u outside [1, %u]", active, n);
  int32_t k0 = -1;
  fk_extent3 d0 = {0, 0, 0};
  for (uint32_t i = 0; i < n; ++i) {
    const fk_iop* r = inner[i];
    if (!r || !is_sample_read(r))
      return fail(FK_E_INNER_KIND_MISMATCH, -1, "batch inner #%u is not a per-plane read", i);
    if (i == 0) { k0 = r->out_kind; d0 = r->dims; }
    else if (r->out_kind != k0)
      return fail(FK_E_INNER_KIND_MISMATCH, -1, "batch inner #%u yields %s, expected %s", i,
                  kind_name((uint32_t)r->out_kind), kind_name((uint32_t)k0));
    else if (r->dims.width != d0.width || r->dims.height != d0.height || r->dims.batch != d0.batch)
      return fail(FK_E_HETEROGENEOUS_BATCH, (int32_t)i, "batch inner #%u extents differ", i);
  }
  fk_iop* op = new_iop(FK_OP_BATCH_READ, FK_KIND_READ, -1, k0);
  op->planes = (sample_t*)calloc(n, sizeof(sample_t));
  for (uint32_t i = 0; i < n; ++i) sample_copy(&op->planes[i], &inner[i]->sample);
  op->n_planes = n;
  op->active = active;
  memset(&op->def, 0, sizeof op->def);
  if (def) memcpy(op->def.raw, def, fk_bytes_per_element((uint32_t)k0));
  op->has_dims = 1;
  op->dims.width = d0.width;
  op->dims.height = d0.height;
  op->dims.batch = n;
  *out = op;
  return FK_OK;
}

fk_status fk_op_batch_write(const fk_iop* const* inner, uint32_t n, uint32_t active, fk_iop** out) {
  /* op_batch_write, oplib.cpp:223-256 */
  CHECK_OUT(out);
  if (n == 0 || !inner) return fail(FK_E_EMPTY_BATCH, -1, "batch write over zero planes");
  if (active < 1 || active > n)
    return fail(FK_E_EMPTY_BATCH, -1, "active_count %u outside [1, %u]", active, n);
  const uint32_t wid = inner[0] ? inner[0]->id : 0;
  int32_t k0 = -1;
  fk_extent3 d0 = {0, 0, 0};
  for (uint32_t i = 0; i < n; ++i) {
    const fk_iop* w = inner[i];
    if (!w || w->id != wid || (w->id != FK_OP_PER_THREAD_WRITE && w->id != FK_OP_SPLIT_WRITE))
      return fail(FK_E_INNER_KIND_MISMATCH, -1, "batch inner #%u is not a uniform per-plane write", i);
    if (i == 0) { k0 = w->in_kind; d0 = w->dims; }
    else if (w->in_kind != k0)
      return fail(FK_E_INNER_KIND_MISMATCH, -1, "batch inner #%u input kind", i);
    else if (w->dims.width != d0.width || w->dims.height != d0.height || w->dims.batch != d0.batch)
      return fail(FK_E_HETEROGENEOUS_BATCH, (int32_t)i, "batch inner #%u extents differ", i);
  }
  fk_iop* op = new_iop(FK_OP_BATCH_WRITE, FK_KIND_WRITE, k0, -1);
  op->w_inner = wid;
  op->n_planes = n;
  op->active = active;
  const int per = wid == FK_OP_SPLIT_WRITE ? 3 : 1;
  op->wdest = (fk_plane*)malloc(sizeof(fk_plane) * n * per);
  for (uint32_t i = 0; i < n; ++i) memcpy(&op->wdest[i * per], inner[i]->dest, sizeof(fk_plane) * per);
  op->has_dims = 1;
  op->dims.width = d0.width;
  op->dims.height = d0.height;
  op->dims.batch = n;
  *out = op;
  return FK_OK;
}

fk_status fk_fold_unary_into_read(const fk_iop* read, const fk_iop* unary, fk_iop** out) {
  /* fold_unary_into_read, oplib.cpp:264-274 */
  CHECK_OUT(out);
  if (!read || !unary) return fail(FK_E_INVALID_ARGUMENT, -1, "null op");
  if (!is_sample_read(read)) return fail(FK_E_UNSUPPORTED_KIND, -1, "can only fold into a per-plane read");
  if (unary->opkind != FK_KIND_UNARY)
    return fail(FK_E_UNSUPPORTED_KIND, -1, "only parameter-free unary ops fold into a read");
  if (unary->in_kind != read->out_kind)
    return fail(FK_E_KIND_MISMATCH, -1, "fold input kind does not match read output");
  sample_t s;
  sample_copy(&s, &read->sample);
  s.post = (folded_t*)realloc(s.post, sizeof(folded_t) * (s.n_post + 1));
  s.post[s.n_post].id = unary->id;
  s.post[s.n_post].in = (uint32_t)unary->in_kind;
  s.post[s.n_post].out = (uint32_t)unary->out_kind;
  s.n_post++;
  *out = make_sample_read(read->id, &s);
  free(s.post);
  return FK_OK;
}

/* ------------------------------------------------------------ validation -- */

static const char* op_name(uint32_t id) { /* ops.cpp:8-27 */
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

fk_status fk_validate_chain(const fk_iop* const* ops, uint32_t n, fk_pipeline** out) {
  /* validate_chain, ops.cpp:37-82 */
  CHECK_OUT(out);
  if (n == 0 || !ops) return fail(FK_E_EMPTY_CHAIN, -1, "chain has no ops");
  for (uint32_t i = 0; i < n; ++i)
    if (!ops[i]) return fail(FK_E_INVALID_ARGUMENT, (int32_t)i, "null op");
  if (n > 4096) return fail(FK_E_CHAIN_TOO_LONG, -1, "%u ops; limit is 4096", n);
  if (ops[0]->opkind != FK_KIND_READ)
    return fail(FK_E_FIRST_NOT_READ, 0, "%s at position 0", op_name(ops[0]->id));
  const int32_t last = (int32_t)n - 1;
  if (ops[last]->opkind != FK_KIND_WRITE)
    return fail(FK_E_LAST_NOT_WRITE, last, "%s at position %d", op_name(ops[last]->id), last);
  int32_t cur = ops[0]->out_kind;
  for (int32_t i = 1; i <= last; ++i) {
    const fk_iop* op = ops[i];
    if (i != last && (op->opkind == FK_KIND_READ || op->opkind == FK_KIND_WRITE))
      return fail(FK_E_KIND_MISMATCH, i, "expected a compute op at position %d, found %s", i, op_name(op->id));
    if (op->in_kind != cur)
      return fail(FK_E_KIND_MISMATCH, i, "position %d: expected %s, found %s", i,
                  kind_name((uint32_t)cur), kind_name((uint32_t)op->in_kind));
    if (op->out_kind >= 0) cur = op->out_kind;
  }
  if (!ops[0]->has_dims) return fail(FK_E_MISSING_DIMS, -1, "%s has no dims hint", op_name(ops[0]->id));
  const fk_extent3 sp = ops[0]->dims;
  if (!ops[last]->has_dims) return fail(FK_E_MISSING_DIMS, last, "write op has no dims hint");
  const fk_extent3 wd = ops[last]->dims;
  if (wd.width != sp.width || wd.height != sp.height || wd.batch != sp.batch)
    return fail(FK_E_DIMS_MISMATCH, last, "read space %ux%ux%u vs write hint", sp.width, sp.height, sp.batch);
  fk_pipeline* p = (fk_pipeline*)calloc(1, sizeof(fk_pipeline));
  p->read = clone_iop(ops[0]);
  p->write = clone_iop(ops[last]);
  p->n_compute = n - 2;
  p->compute = (fk_iop**)calloc(n, sizeof(fk_iop*));
  for (uint32_t i = 1; i + 1 < n; ++i) p->compute[i - 1] = clone_iop(ops[i]);
  p->space = sp;
  *out = p;
  return FK_OK;
}

void fk_pipeline_free(fk_pipeline* p) {
  if (!p) return;
  fk_iop_free(p->read);
  fk_iop_free(p->write);
  for (uint32_t i = 0; i < p->n_compute; ++i) fk_iop_free(p->compute[i]);
  free(p->compute);
  free(p);
}

fk_status fk_pipeline_iter_space(const fk_pipeline* p, fk_extent3* out) {
  if (!p || !out) return fail(FK_E_INVALID_ARGUMENT, -1, "null argument");
  *out = p->space;
  return FK_OK;
}
uint32_t fk_pipeline_compute_count(const fk_pipeline* p) { return p ? p->n_compute : 0; }

/* -------------------------------------------------------------- compute -- */

/* u8 ops wrap mod 256 (scalar.hpp:146-157); floats are IEEE in their own precision. */
static inline uint8_t u8_op(uint32_t id, uint8_t a, uint8_t b) {
  switch (id) {
    case FK_OP_MUL: return (uint8_t)((unsigned)a * (unsigned)b);
    case FK_OP_ADD: return (uint8_t)((unsigned)a + (unsigned)b);
    case FK_OP_SUB: return (uint8_t)((unsigned)a - (unsigned)b);
    default: return (uint8_t)(a / b);
  }
}
static inline float f32_op(uint32_t id, float a, float b) {
  switch (id) {
    case FK_OP_MUL: return a * b;
    case FK_OP_ADD: return a + b;
    case FK_OP_SUB: return a - b;
    default: return a / b;
  }
}
static inline double f64_op(uint32_t id, double a, double b) {
  switch (id) {
    case FK_OP_MUL: return a * b;
    case FK_OP_ADD: return a + b;
    case FK_OP_SUB: return a - b;
    default: return a / b;
  }
}

/* arith_block_repeat, ops.cpp:110-159: v = v op c per lane, `reps` times. */
static void arith_repeat(uint32_t id, uint32_t k, const elem_t* c, elem_t* v, uint32_t reps) {
  const int lanes = lane_count(k);
  switch (lane_kind(k)) {
    case FK_U8:
      for (uint32_t r = 0; r < reps; ++r)
        for (int l = 0; l < lanes; ++l) v->u8v[l] = u8_op(id, v->u8v[l], c->u8v[l]);
      break;
    case FK_F32:
      for (uint32_t r = 0; r < reps; ++r)
        for (int l = 0; l < lanes; ++l) v->f32v[l] = f32_op(id, v->f32v[l], c->f32v[l]);
      break;
    default:
      for (uint32_t r = 0; r < reps; ++r)
        for (int l = 0; l < lanes; ++l) v->f64v[l] = f64_op(id, v->f64v[l], c->f64v[l]);
      break;
  }
}

static void swap_rb(uint32_t k, elem_t* v, uint32_t reps) { /* swap_rb_block, ops.cpp:161-176 */
  if (reps % 2 == 0) return;
  switch (k) {
    case FK_U8X3: { uint8_t t = v->u8v[0]; v->u8v[0] = v->u8v[2]; v->u8v[2] = t; break; }
    case FK_F32X3: { float t = v->f32v[0]; v->f32v[0] = v->f32v[2]; v->f32v[2] = t; break; }
    case FK_F64X3: { double t = v->f64v[0]; v->f64v[0] = v->f64v[2]; v->f64v[2] = t; break; }
    default: break;
  }
}

static void to_gray(uint32_t in, elem_t* v) { /* to_gray_block, ops.cpp:178-185 */
  const double g = 0.299 * lane_as_double(in, v, 0) + 0.587 * lane_as_double(in, v, 1) +
                   0.114 * lane_as_double(in, v, 2);
  elem_t o;
  memset(&o, 0, sizeof o);
  o.f32v[0] = (float)g;
  *v = o;
}

static void unary_apply(uint32_t id, uint32_t in, uint32_t out, elem_t* v) { /* unary_block, ops.cpp:191-198 */
  switch (id) {
    case FK_OP_CAST: cast_element(in, out, v); break;
    case FK_OP_SWAP_RB: swap_rb(in, v, 1); break;
    case FK_OP_TO_GRAY: to_gray(in, v); break;
  }
}

/* compute_exec_block, ops.cpp:214-235 (one element; z selects BatchArith constants) */
static void compute_apply(const fk_iop* op, elem_t* v, uint32_t z) {
  const uint32_t in = (uint32_t)op->in_kind;
  switch (op->id) {
    case FK_OP_MUL: case FK_OP_ADD: case FK_OP_SUB: case FK_OP_DIV:
      arith_repeat(op->id, in, &op->value, v, 1);
      break;
    case FK_OP_BATCH_ARITH:
      arith_repeat(op->inner_id, in, &op->values[z < op->n_values ? z : op->n_values - 1], v, 1);
      break;
    case FK_OP_STATIC_LOOP: /* static_loop_block, ops.cpp:200-210 */
      switch (op->inner_id) {
        case FK_OP_MUL: case FK_OP_ADD: case FK_OP_SUB: case FK_OP_DIV:
          arith_repeat(op->inner_id, op->value_kind, &op->value, v, op->repeat);
          break;
        case FK_OP_SWAP_RB: swap_rb(op->value_kind, v, op->repeat); break;
        default: break; /* kind-preserving cast: identity */
      }
      break;
    default:
      unary_apply(op->id, in, (uint32_t)op->out_kind, v);
      break;
  }
}

/* ----------------------------------------------------------------- read -- */

static inline const uint8_t* plane_at(const fk_plane* p, uint64_t x, uint64_t y) {
  return (const uint8_t*)p->data + (y * p->row_stride + x) * fk_bytes_per_element(p->kind);
}
static inline void plane_load(const fk_plane* p, uint64_t x, uint64_t y, elem_t* e) { /* plane.cpp:113-117 */
  memset(e, 0, sizeof *e);
  memcpy(e->raw, plane_at(p, x, y), fk_bytes_per_element(p->kind));
}
static inline void plane_store(const fk_plane* p, uint64_t x, uint64_t y, const elem_t* e) { /* plane.cpp:119-123 */
  memcpy((uint8_t*)plane_at(p, x, y), e->raw, fk_bytes_per_element(p->kind));
}

static inline int64_t clamp_i64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }
static inline double lerp(double a, double b, double t) { return a + (b - a) * t; } /* ops.cpp:250 */
static inline double center_coord(int64_t i, uint32_t rect, uint32_t out) { /* ops.cpp:253-257 */
  return ((double)i + 0.5) * (double)rect / (double)out - 0.5;
}

static void bilinear_sample(const sample_t* p, int64_t x, int64_t y, elem_t* out) { /* ops.cpp:259-299 */
  const double cx = center_coord(x, p->rect_w, p->out_w);
  const double cy = center_coord(y, p->rect_h, p->out_h);
  const int64_t ix = (int64_t)floor(cx);
  const int64_t iy = (int64_t)floor(cy);
  const double fx = cx - (double)ix;
  const double fy = cy - (double)iy;
  const int64_t maxx = (int64_t)p->rect_w - 1, maxy = (int64_t)p->rect_h - 1;
  const uint32_t sx0 = (uint32_t)(p->x0 + clamp_i64(ix, 0, maxx));
  const uint32_t sx1 = (uint32_t)(p->x0 + clamp_i64(ix + 1, 0, maxx));
  const uint32_t sy0 = (uint32_t)(p->y0 + clamp_i64(iy, 0, maxy));
  const uint32_t sy1 = (uint32_t)(p->y0 + clamp_i64(iy + 1, 0, maxy));
  elem_t a, b, c, d;
  plane_load(&p->source, sx0, sy0, &a);
  plane_load(&p->source, sx1, sy0, &b);
  plane_load(&p->source, sx0, sy1, &c);
  plane_load(&p->source, sx1, sy1, &d);
  const uint32_t k = p->source.kind;
  memset(out, 0, sizeof *out);
  for (int l = 0; l < lane_count(k); ++l) {
    const double top = lerp(lane_as_double(k, &a, l), lane_as_double(k, &b, l), fx);
    const double bot = lerp(lane_as_double(k, &c, l), lane_as_double(k, &d, l), fx);
    const double res = lerp(top, bot, fy);
    switch (lane_kind(k)) {
      case FK_U8: out->u8v[l] = round_clamp_u8(res); break;
      case FK_F32: out->f32v[l] = (float)res; break;
      default: out->f64v[l] = res; break;
    }
  }
}

static void nearest_sample(const sample_t* p, int64_t x, int64_t y, elem_t* out) { /* ops.cpp:301-310 */
  const double cx = ((double)x + 0.5) * (double)p->rect_w / (double)p->out_w;
  const double cy = ((double)y + 0.5) * (double)p->rect_h / (double)p->out_h;
  const uint32_t sx = p->x0 + (uint32_t)clamp_i64((int64_t)floor(cx), 0, (int64_t)p->rect_w - 1);
  const uint32_t sy = p->y0 + (uint32_t)clamp_i64((int64_t)floor(cy), 0, (int64_t)p->rect_h - 1);
  plane_load(&p->source, sx, sy, out);
}

/* sample_block, ops.cpp:327-344 (one element): returns source elements touched. */
static uint32_t sample_read(const sample_t* p, int64_t x, int64_t y, elem_t* out) {
  uint32_t touched;
  if (!sample_resizing(p)) {
    plane_load(&p->source, (uint64_t)(p->x0 + x), (uint64_t)(p->y0 + y), out);
    touched = 1;
  } else if (p->mode == FK_NEAREST) {
    nearest_sample(p, x, y, out);
    touched = 1;
  } else {
    bilinear_sample(p, x, y, out);
    touched = 4;
  }
  for (uint32_t i = 0; i < p->n_post; ++i) unary_apply(p->post[i].id, p->post[i].in, p->post[i].out, out);
  return touched;
}

typedef struct io_counters { uint64_t elements_read, bytes_read, bytes_written, default_reads; } io_t;

/* read_exec_block, ops.cpp:361-381 */
static void read_exec(const fk_iop* op, int64_t x, int64_t y, uint32_t z, elem_t* out, io_t* io) {
  const sample_t* s;
  if (op->id == FK_OP_BATCH_READ) {
    if (z >= op->active) {
      *out = op->def;
      io->default_reads++;
      return;
    }
    s = &op->planes[z];
  } else {
    s = &op->sample;
  }
  const uint32_t t = sample_read(s, x, y, out);
  io->elements_read += t;
  io->bytes_read += (uint64_t)t * fk_bytes_per_element(s->source.kind);
}

/* store_block / split_block / write_exec_block, ops.cpp:396-448 */
static void split_store(const fk_plane* d, int64_t x, int64_t y, const elem_t* v, io_t* io) {
  const uint32_t lk = d[0].kind;
  for (int l = 0; l < 3; ++l) {
    elem_t e;
    memset(&e, 0, sizeof e);
    switch (lk) {
      case FK_U8: e.u8v[0] = v->u8v[l]; break;
      case FK_F32: e.f32v[0] = v->f32v[l]; break;
      default: e.f64v[0] = v->f64v[l]; break;
    }
    plane_store(&d[l], (uint64_t)x, (uint64_t)y, &e);
  }
  io->bytes_written += 3ull * fk_bytes_per_element(lk);
}
static void write_exec(const fk_iop* op, int64_t x, int64_t y, uint32_t z, const elem_t* v, io_t* io) {
  switch (op->id) {
    case FK_OP_PER_THREAD_WRITE:
      plane_store(&op->dest[0], (uint64_t)x, (uint64_t)y, v);
      io->bytes_written += fk_bytes_per_element(op->dest[0].kind);
      break;
    case FK_OP_SPLIT_WRITE: split_store(op->dest, x, y, v, io); break;
    case FK_OP_BATCH_WRITE:
      if (z >= op->active) return; /* inactive plane: skip the write */
      if (op->w_inner == FK_OP_PER_THREAD_WRITE) {
        plane_store(&op->wdest[z], (uint64_t)x, (uint64_t)y, v);
        io->bytes_written += fk_bytes_per_element(op->wdest[z].kind);
      } else {
        split_store(&op->wdest[3 * (size_t)z], x, y, v, io);
      }
      break;
  }
}

/* ------------------------------------------------------------- executor -- */

static fk_status check_config(const fk_exec_config* c) { /* executor.cpp:20-25 */
  if (!c) return FK_OK;
  if (c->chunk_rows < 1) return fail(FK_E_INVALID_CONFIG, -1, "chunk_rows must be >= 1");
  const int b = c->coarsen_block;
  if (!(b == 1 || b == 2 || b == 4 || b == 8 || b == 16))
    return fail(FK_E_INVALID_CONFIG, -1, "coarsening block must be one of 1/2/4/8/16");
  if (c->workers < 0) return fail(FK_E_INVALID_CONFIG, -1, "workers must be >= 0");
  return FK_OK;
}

static int resolve_workers(const fk_exec_config* c) {
#ifdef _OPENMP
  return (c && c->workers > 0) ? c->workers : omp_get_max_threads();
#else
  (void)c;
  return 1;
#endif
}

static uint64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

fk_status fk_schedule(const fk_extent3* sp, const fk_exec_config* cfg, uint32_t* tasks, uint64_t cap,
                      uint64_t* count) { /* schedule, executor.cpp:52-61 */
  if (!sp || !cfg || !count) return fail(FK_E_INVALID_ARGUMENT, -1, "null argument");
  fk_status st = check_config(cfg);
  if (st) return st;
  const uint32_t chunk = (uint32_t)cfg->chunk_rows;
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
  return FK_OK;
}

/* execute_fused, executor.cpp:63-85: one sweep, every point read -> compute* -> write. */
fk_status fk_execute_sharded(const fk_pipeline* const* pipelines, const int32_t* devices, uint32_t n,
                             const fk_exec_config* cfgs, fk_exec_report* reports) {
  /* CPU backend: the shards one after another (devices are ignored) */
  if (n && (!pipelines || !devices)) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: null argument");
  for (uint32_t i = 0; i < n; ++i) {
    fk_status s = fk_execute_fused(pipelines[i], cfgs ? &cfgs[i] : NULL, reports ? &reports[i] : NULL);
    if (s != FK_OK) return s;
  }
  return FK_OK;
}

fk_status fk_gather(void* dst, int32_t dst_device, const uint64_t* dst_offsets, const void* const* srcs,
                    const int32_t* src_devices, const uint64_t* bytes, uint32_t n, void* stream) {
  (void)dst_device; (void)src_devices; (void)stream;
  if (n && (!dst || !dst_offsets || !srcs || !bytes)) return fail(FK_E_INVALID_ARGUMENT, -1, "InvalidArgument: null argument");
  for (uint32_t i = 0; i < n; ++i) memcpy((uint8_t*)dst + dst_offsets[i], srcs[i], bytes[i]);
  return FK_OK;
}

fk_status fk_execute_fused(const fk_pipeline* p, const fk_exec_config* cfg, fk_exec_report* rep) {
  if (!p) return fail(FK_E_INVALID_ARGUMENT, -1, "null pipeline");
  fk_status st = check_config(cfg);
  if (st) return st;
  const fk_extent3 sp = p->space;
  const int64_t rows = (int64_t)sp.height * sp.batch;
  const int workers = (cfg && (cfg->flags & FK_EXEC_SERIAL)) ? 1 : resolve_workers(cfg);
  uint64_t br = 0, bw = 0;
  const uint64_t t0 = now_ns();
#pragma omp parallel for schedule(dynamic, 8) num_threads(workers) reduction(+ : br, bw)
  for (int64_t r = 0; r < rows; ++r) {
    const uint32_t z = (uint32_t)(r / sp.height);
    const int64_t y = r % sp.height;
    io_t io = {0, 0, 0, 0};
    for (int64_t x = 0; x < (int64_t)sp.width; ++x) {
      elem_t v;
      read_exec(p->read, x, y, z, &v, &io);
      for (uint32_t i = 0; i < p->n_compute; ++i) compute_apply(p->compute[i], &v, z);
      write_exec(p->write, x, y, z, &v, &io);
    }
    br += io.bytes_read;
    bw += io.bytes_written;
  }
  const uint64_t t1 = now_ns();
  if (rep) {
    memset(rep, 0, sizeof *rep);
    rep->wall_time_ns = t1 - t0;
    rep->bytes_read = br;
    rep->bytes_written = bw;
    rep->passes = 1;
    rep->points_visited = (uint64_t)sp.width * sp.height * sp.batch;
    rep->path = FK_PATH_CPU;
  }
  return FK_OK;
}

/* execute_unfused, executor.cpp:134-217: one sweep per compute op through freshly
 * allocated intermediates of that op's output kind, then a write sweep. */
fk_status fk_execute_unfused(const fk_pipeline* p, const fk_exec_config* cfg, fk_exec_report* rep) {
  if (!p) return fail(FK_E_INVALID_ARGUMENT, -1, "null pipeline");
  fk_status st = check_config(cfg);
  if (st) return st;
  const fk_extent3 sp = p->space;
  const uint64_t plane_pts = (uint64_t)sp.width * sp.height;
  const int64_t rows = (int64_t)sp.height * sp.batch;
  const int workers = resolve_workers(cfg);
  const uint32_t nc = p->n_compute;
  uint64_t br = 0, bw = 0, inter_bytes = 0;
  const uint64_t t0 = now_ns();
  if (nc == 0) {
#pragma omp parallel for schedule(dynamic, 8) num_threads(workers) reduction(+ : br, bw)
    for (int64_t r = 0; r < rows; ++r) {
      const uint32_t z = (uint32_t)(r / sp.height);
      const int64_t y = r % sp.height;
      io_t io = {0, 0, 0, 0};
      for (int64_t x = 0; x < (int64_t)sp.width; ++x) {
        elem_t v;
        read_exec(p->read, x, y, z, &v, &io);
        write_exec(p->write, x, y, z, &v, &io);
      }
      br += io.bytes_read;
      bw += io.bytes_written;
    }
  } else {
    uint8_t* prev = NULL;
    uint32_t prev_kind = 0;
    for (uint32_t pass = 0; pass < nc; ++pass) {
      const fk_iop* op = p->compute[pass];
      const uint32_t ok = (uint32_t)op->out_kind;
      const uint32_t obpe = fk_bytes_per_element(ok);
      uint8_t* next = (uint8_t*)malloc(plane_pts * sp.batch * obpe); /* make_intermediate, :112-118 */
      inter_bytes += plane_pts * sp.batch * obpe;
      const uint32_t ibpe = fk_bytes_per_element(prev_kind);
#pragma omp parallel for schedule(dynamic, 8) num_threads(workers) reduction(+ : br, bw)
      for (int64_t r = 0; r < rows; ++r) {
        const uint32_t z = (uint32_t)(r / sp.height);
        const int64_t y = r % sp.height;
        io_t io = {0, 0, 0, 0};
        for (int64_t x = 0; x < (int64_t)sp.width; ++x) {
          const uint64_t idx = (uint64_t)z * plane_pts + (uint64_t)y * sp.width + (uint64_t)x;
          elem_t v;
          if (pass == 0) {
            read_exec(p->read, x, y, z, &v, &io);
          } else { /* load_block, :120-124 */
            memset(&v, 0, sizeof v);
            memcpy(v.raw, prev + idx * ibpe, ibpe);
            io.bytes_read += ibpe;
          }
          compute_apply(op, &v, z);
          memcpy(next + idx * obpe, v.raw, obpe); /* store_block_to, :126-130 */
          io.bytes_written += obpe;
        }
        br += io.bytes_read;
        bw += io.bytes_written;
      }
      free(prev);
      prev = next;
      prev_kind = ok;
    }
    const uint32_t ibpe = fk_bytes_per_element(prev_kind);
#pragma omp parallel for schedule(dynamic, 8) num_threads(workers) reduction(+ : br, bw)
    for (int64_t r = 0; r < rows; ++r) {
      const uint32_t z = (uint32_t)(r / sp.height);
      const int64_t y = r % sp.height;
      io_t io = {0, 0, 0, 0};
      for (int64_t x = 0; x < (int64_t)sp.width; ++x) {
        const uint64_t idx = (uint64_t)z * plane_pts + (uint64_t)y * sp.width + (uint64_t)x;
        elem_t v;
        memset(&v, 0, sizeof v);
        memcpy(v.raw, prev + idx * ibpe, ibpe);
        io.bytes_read += ibpe;
        write_exec(p->write, x, y, z, &v, &io);
      }
      br += io.bytes_read;
      bw += io.bytes_written;
    }
    free(prev);
  }
  const uint64_t t1 = now_ns();
  if (rep) {
    memset(rep, 0, sizeof *rep);
    rep->wall_time_ns = t1 - t0;
    rep->bytes_read = br;
    rep->bytes_written = bw;
    rep->intermediate_bytes_allocated = inter_bytes;
    rep->passes = (uint64_t)nc + 1;
    rep->points_visited = plane_pts * sp.batch * rep->passes;
    rep->path = FK_PATH_CPU;
  }
  return FK_OK;
}

fk_status fk_plan_memory_savings(const fk_pipeline* p, uint64_t* bytes) { /* executor.cpp:223-228 */
  if (!p || !bytes) return fail(FK_E_INVALID_ARGUMENT, -1, "null argument");
  const uint64_t pts = (uint64_t)p->space.width * p->space.height * p->space.batch;
  uint64_t b = 0;
  for (uint32_t i = 0; i < p->n_compute; ++i) b += pts * fk_bytes_per_element((uint32_t)p->compute[i]->out_kind);
  *bytes = b;
  return FK_OK;
}

/* ---------------------------------------------------------------- reduce -- */
/* ReduceDPP, dpp.cpp:46-246. Sequential per-worker folds over contiguous row
   ranges, partials merged in worker-index order; float sums in double. */

static void reducer_identity(uint32_t r, uint32_t kind, elem_t* e) { /* dpp.cpp:48-73 */
  const uint32_t lk = lane_kind(kind);
  double v = 0.0;
  if (r == FK_REDUCE_MAX) v = lk == FK_U8 ? 0.0 : -INFINITY;
  else if (r == FK_REDUCE_MIN) v = lk == FK_U8 ? 255.0 : INFINITY;
  memset(e, 0, sizeof *e);
  for (int l = 0; l < lane_count(kind); ++l) {
    switch (lk) {
      case FK_U8: e->u8v[l] = (uint8_t)v; break;
      case FK_F32: e->f32v[l] = (float)v; break;
      default: e->f64v[l] = v; break;
    }
  }
}

/* combine_lane / combine_elements, dpp.cpp:77-106 */
static void combine_elements(uint32_t r, uint32_t kind, elem_t* a, const elem_t* b) {
  const uint32_t lk = lane_kind(kind);
  for (int l = 0; l < lane_count(kind); ++l) {
    switch (lk) {
      case FK_U8: {
        const uint8_t x = a->u8v[l], y = b->u8v[l];
        a->u8v[l] = r == FK_REDUCE_SUM ? (uint8_t)(x + y) : r == FK_REDUCE_MAX ? (x < y ? y : x) : (y < x ? y : x);
        break;
      }
      case FK_F32: {
        const float x = a->f32v[l], y = b->f32v[l];
        a->f32v[l] = r == FK_REDUCE_SUM ? x + y : r == FK_REDUCE_MAX ? (x < y ? y : x) : (y < x ? y : x);
        break;
      }
      default: {
        const double x = a->f64v[l], y = b->f64v[l];
        a->f64v[l] = r == FK_REDUCE_SUM ? x + y : r == FK_REDUCE_MAX ? (x < y ? y : x) : (y < x ? y : x);
        break;
      }
    }
  }
}

typedef struct spec_accum { /* SpecAccum, dpp.cpp:116-127 */
  int double_sum;
  double d[3];
  elem_t e;
} spec_accum_t;

static void make_accum(spec_accum_t* a, uint32_t r, uint32_t kind) {
  memset(a, 0, sizeof *a);
  a->double_sum = r == FK_REDUCE_SUM && lane_kind(kind) != FK_U8;
  if (!a->double_sum) reducer_identity(r, kind, &a->e);
}

#define RED_BLOCK 64 /* kReduceBlock, dpp.cpp:110 */

fk_status fk_multi_reduce_plane(const fk_iop* read, const fk_reduce_spec* specs, uint32_t n, int32_t workers,
                                void* results, uint64_t* elements_read) {
  /* multi_reduce_plane, dpp.cpp:158-241 */
  if (!read || (n && (!specs || !results))) return fail(FK_E_INVALID_ARGUMENT, -1, "null argument");
  if (n == 0) return fail(FK_E_EMPTY_ITER_SPACE, -1, "no reduce specs given");
  if (read->opkind != FK_KIND_READ) return fail(FK_E_FIRST_NOT_READ, -1, "iteration space comes from a read op");
  if (!read->has_dims) return fail(FK_E_MISSING_DIMS, -1, "%s has no dims hint", op_name(read->id));
  const fk_extent3 sp = read->dims;
  if ((uint64_t)sp.width * sp.height * sp.batch == 0) return fail(FK_E_EMPTY_ITER_SPACE, -1, "empty iteration space");
  uint32_t* vkind = (uint32_t*)calloc(n, sizeof(uint32_t));
  elem_t* ident = (elem_t*)calloc(n, sizeof(elem_t));
  for (uint32_t s = 0; s < n; ++s) {
    const fk_iop* t = specs[s].transform;
    if (specs[s].combine > FK_REDUCE_MIN) {  /* C-ABI enum check (fk.h: FK_E_INVALID_ARGUMENT) */
      free(vkind); free(ident);
      return fail(FK_E_INVALID_ARGUMENT, -1, "reduce spec: unknown combine");
    }
    if (t) {
      if (t->opkind != FK_KIND_UNARY && t->opkind != FK_KIND_BINARY) {
        free(vkind); free(ident);
        return fail(FK_E_INVALID_CONFIG, -1, "reduce transform must be a compute op");
      }
      if (t->in_kind != read->out_kind) {
        free(vkind); free(ident);
        return fail(FK_E_KIND_MISMATCH, -1, "reduce transform input kind vs read output");
      }
      vkind[s] = (uint32_t)(t->out_kind >= 0 ? t->out_kind : t->in_kind);
    } else {
      vkind[s] = (uint32_t)read->out_kind;
    }
    if (specs[s].has_identity) memcpy(&ident[s], specs[s].identity, sizeof(elem_t));
    else reducer_identity(specs[s].combine, vkind[s], &ident[s]);
  }
  const int w_req = workers > 0 ? workers : omp_get_max_threads();
  const uint64_t total_rows = (uint64_t)sp.height * sp.batch;
  const int w_count = (int)((uint64_t)w_req < total_rows ? (uint64_t)w_req : total_rows);
  spec_accum_t* part = (spec_accum_t*)calloc((size_t)w_count * n, sizeof(spec_accum_t));
  uint64_t* reads = (uint64_t*)calloc((size_t)w_count, sizeof(uint64_t));
#pragma omp parallel for schedule(static, 1) num_threads(w_count)
  for (int w = 0; w < w_count; ++w) {
    spec_accum_t* mine = part + (size_t)w * n;
    for (uint32_t s = 0; s < n; ++s) make_accum(&mine[s], specs[s].combine, vkind[s]);
    const uint64_t r0 = total_rows * (uint64_t)w / (uint64_t)w_count, r1 = total_rows * (uint64_t)(w + 1) / (uint64_t)w_count;
    io_t io;
    memset(&io, 0, sizeof io);
    for (uint64_t row = r0; row < r1; ++row) {
      const uint32_t z = (uint32_t)(row / sp.height);
      const int64_t y = (int64_t)(row % sp.height);
      for (uint32_t x = 0; x < sp.width; ++x) {
        elem_t v;
        memset(&v, 0, sizeof v);
        read_exec(read, (int64_t)x, y, z, &v, &io);
        for (uint32_t s = 0; s < n; ++s) {
          elem_t t = v;
          if (specs[s].transform) compute_apply(specs[s].transform, &t, z);
          if (mine[s].double_sum) {
            for (int l = 0; l < lane_count(vkind[s]); ++l) mine[s].d[l] += lane_as_double(vkind[s], &t, l);
          } else {
            combine_elements(specs[s].combine, vkind[s], &mine[s].e, &t);
          }
        }
      }
    }
    reads[w] = io.elements_read;
  }
  uint64_t total_reads = 0;
  for (int w = 0; w < w_count; ++w) total_reads += reads[w];
  if (elements_read) *elements_read = total_reads;
  for (uint32_t s = 0; s < n; ++s) { /* merge in worker-index order, finish_accum (dpp.cpp:138-152) */
    spec_accum_t acc;
    make_accum(&acc, specs[s].combine, vkind[s]);
    if (!acc.double_sum) acc.e = ident[s];
    for (int w = 0; w < w_count; ++w) {
      const spec_accum_t* f = part + (size_t)w * n + s;
      if (acc.double_sum) for (int l = 0; l < 3; ++l) acc.d[l] += f->d[l];
      else combine_elements(specs[s].combine, vkind[s], &acc.e, &f->e);
    }
    elem_t out;
    memset(&out, 0, sizeof out);
    if (!acc.double_sum) {
      out = acc.e;
    } else {
      for (int l = 0; l < lane_count(vkind[s]); ++l) {
        const double total = lane_as_double(vkind[s], &ident[s], l) + acc.d[l];
        if (lane_kind(vkind[s]) == FK_F32) out.f32v[l] = (float)total;
        else out.f64v[l] = total;
      }
    }
    memcpy((uint8_t*)results + 24 * (size_t)s, &out, 24);
  }
  free(vkind); free(ident); free(part); free(reads);
  return FK_OK;
}
