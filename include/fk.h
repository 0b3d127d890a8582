/*
 * fk.h — C-ABI boundary of the B200 Fused Kernel Library.
 *
 * One header, three implementations of the same entry points:
 *   libfk_cuda.so    the product: sm_100a fused kernels (device memory planes)
 *   libfk_oracle.so  oracle/fk_oracle.c, a plain-C restatement (host memory; test-only)
 *   libfk_ref.so     oracle/ref_shim.cpp over the unmodified reference sources (host memory; test-only)
 *
 * Each entry point replaces one function of the reference's C++ API
 * (/root/reference/proj/include/opfuse/ headers); the citation is on each line.
 * The reference is C++ with no FFI of its own, so this header is the FFI a
 * maintainer binds (ctypes / cgo / JNI stubs in INTEGRATION.md).
 *
 * Conventions
 *  - Every function returns fk_status: 0 on success, otherwise 1 + the
 *    reference's Errc ordinal (errors.hpp:9-38), or one of the FK_E_* codes
 *    this layer adds (>= 100). fk_last_error()/fk_last_error_position() give the
 *    message and chain position of the last failure on the calling thread.
 *  - Plain pointers and sizes only. An fk_plane is a strided 2D view (row-major,
 *    row_stride in ELEMENTS, packed x3 lanes adjacent) exactly as plane.hpp:60-103.
 *    IOps and pipelines store plane views by value; the caller keeps the
 *    underlying memory alive (the reference uses shared_ptr, plane.hpp:97).
 *  - Scalar constants / default values are passed as raw little-endian lane bytes
 *    of the given kind (Element layout, scalar.hpp:94-121): u8 / f32 / f64 lanes,
 *    1 or 3 of them.
 */
#ifndef FK_H_
#define FK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FK_ABI_VERSION 1

typedef int32_t fk_status;

/* ScalarKind, scalar.hpp:16-23 (values are the FKT on-disk tags, scalar.hpp:82) */
enum fk_kind { FK_U8 = 0, FK_F32 = 1, FK_F64 = 2, FK_U8X3 = 3, FK_F32X3 = 4, FK_F64X3 = 5 };

/* OpId, ops.hpp:17-37 (+ BatchArith, this library's per-plane-constant extension) */
enum fk_op_id {
  FK_OP_PER_THREAD_READ = 0, FK_OP_CROP_READ, FK_OP_RESIZE_READ, FK_OP_BATCH_READ,
  FK_OP_CAST, FK_OP_SWAP_RB, FK_OP_TO_GRAY,
  FK_OP_MUL, FK_OP_ADD, FK_OP_SUB, FK_OP_DIV, FK_OP_STATIC_LOOP,
  FK_OP_PER_THREAD_WRITE, FK_OP_SPLIT_WRITE, FK_OP_BATCH_WRITE,
  FK_OP_BATCH_ARITH = 32
};

/* OpKind, ops.hpp:15 */
enum fk_op_kind { FK_KIND_READ = 0, FK_KIND_UNARY = 1, FK_KIND_BINARY = 2, FK_KIND_WRITE = 3 };

enum fk_resize_mode { FK_NEAREST = 0, FK_BILINEAR = 1 };       /* ops.hpp:64 */
enum fk_color_order { FK_SWAP_RB = 0, FK_TO_GRAY_F32 = 1 };     /* ops.hpp:65 */

/* Errc, errors.hpp:9-38: status = 1 + ordinal */
enum fk_errc {
  FK_OK = 0,
  FK_E_EMPTY_CHAIN = 1, FK_E_FIRST_NOT_READ, FK_E_LAST_NOT_WRITE, FK_E_KIND_MISMATCH,
  FK_E_DIMS_MISMATCH, FK_E_MISSING_DIMS, FK_E_CHAIN_TOO_LONG,
  FK_E_DIV_BY_ZERO_PARAM, FK_E_UNSUPPORTED_CAST, FK_E_UNSUPPORTED_KIND, FK_E_CROP_OUT_OF_BOUNDS,
  FK_E_PLANE_EXTENT_MISMATCH, FK_E_EMPTY_BATCH, FK_E_INNER_KIND_MISMATCH,
  FK_E_HETEROGENEOUS_BATCH, FK_E_BAD_STATIC_LOOP,
  FK_E_BOUNDS_ERROR, FK_E_CAPACITY_OVERFLOW, FK_E_BAD_MAGIC, FK_E_UNKNOWN_KIND_TAG,
  FK_E_TRUNCATED_PAYLOAD, FK_E_IO_ERROR,
  FK_E_EMPTY_ITER_SPACE, FK_E_INVALID_CONFIG,
  /* codes added by this layer */
  FK_E_INVALID_ARGUMENT = 100, /* null pointer / bad enum at the C boundary */
  FK_E_CUDA = 101,             /* CUDA runtime error (message has cudaGetErrorString) */
  FK_E_NO_DEVICE = 102,        /* CUDA backend loaded on a host without a usable sm_100 GPU */
  FK_E_UNSUPPORTED = 103       /* entry point not provided by this backend */
};

/* Plane view (plane.hpp:60-103). `data` is the address of element (0,0). */
typedef struct fk_plane {
  void* data;
  uint32_t width;
  uint32_t height;
  uint32_t row_stride; /* elements, >= width */
  uint32_t kind;       /* enum fk_kind */
} fk_plane;

typedef struct fk_crop_rect { uint32_t x0, y0, w, h; } fk_crop_rect; /* oplib.hpp:23-26 */

typedef struct fk_extent3 { uint32_t width, height, batch; } fk_extent3; /* plane.hpp:23-32 */

/* ExecConfig, executor.hpp:10-14, plus the device fields this layer adds. */
typedef struct fk_exec_config {
  int32_t workers;       /* CPU backends: OpenMP threads (0 = default). CUDA: ignored */
  int32_t coarsen_block; /* one of 1/2/4/8/16 (dpp.hpp:12-16); validated, result-invariant */
  int32_t chunk_rows;    /* >= 1 (executor.hpp:13); validated */
  uint32_t flags;        /* FK_EXEC_* */
  void* stream;          /* cudaStream_t for the CUDA backend (NULL = legacy default stream) */
} fk_exec_config;

#define FK_EXEC_TIMED 0x1u         /* CUDA: bracket the launch(es) with events and synchronise: fills device_ms */
#define FK_EXEC_FORCE_GENERIC 0x2u /* CUDA: use the interpreted-chain kernel even when a compiled chain matches */
#define FK_EXEC_SERIAL 0x4u        /* CPU backends: execute_fused_serial (executor.hpp:42-45) */
#define FK_EXEC_NO_LUT 0x8u        /* CUDA: never tabulate u8 lane-wise chains (measure the op-by-op path) */

/* ExecReport, executor.hpp:27-34, plus device-side fields. */
typedef struct fk_exec_report {
  uint64_t wall_time_ns;
  uint64_t bytes_read;
  uint64_t bytes_written;
  uint64_t intermediate_bytes_allocated;
  uint64_t passes;
  uint64_t points_visited;
  uint64_t kernels_launched; /* device kernels enqueued by this call (0 on CPU backends) */
  double device_ms;          /* event-timed device duration when FK_EXEC_TIMED, else 0 */
  uint32_t path;             /* FK_PATH_*: which kernel family ran the fused pass */
  uint32_t reserved;
} fk_exec_report;

enum fk_path { FK_PATH_CPU = 0, FK_PATH_GENERIC = 1, FK_PATH_COMPILED = 2 };

typedef struct fk_iop fk_iop;           /* IOp, ops.hpp:131-153 */
typedef struct fk_pipeline fk_pipeline; /* Pipeline, ops.hpp:156-161 */

/* ---- library ------------------------------------------------------------ */
const char* fk_backend_name(void);
int32_t fk_abi_version(void);
const char* fk_last_error(void);
int32_t fk_last_error_position(void);
int32_t fk_errc_name(int32_t status, char* buf, size_t cap); /* errc_name, scalar.cpp:44-72 */

/* ---- planes ------------------------------------------------------------- */
fk_status fk_plane_view(const fk_plane* p, uint32_t x0, uint32_t y0, uint32_t w, uint32_t h,
                        fk_plane* out);                          /* Plane::view, plane.cpp:91-101 */
/* Plane::alloc, plane.cpp:60-71 (zero-initialised; row_stride 0 = width). The
 * buffer is SHARED the way the reference's shared_ptr<TensorBuffer> is
 * (plane.hpp:56-60,97): every IOp and pipeline built from the plane or a view
 * of it keeps it alive, and fk_plane_free only drops the caller's reference.
 * CUDA backend: device memory on the current device; CPU backends: host memory. */
fk_status fk_plane_alloc(uint32_t width, uint32_t height, uint32_t kind, uint32_t row_stride, fk_plane* out);
void fk_plane_free(fk_plane* p);
/* Host <-> plane copies for bindings without a CUDA runtime: the plane's
 * width x height elements row by row, host rows host_pitch bytes apart
 * (0 = packed). CUDA backend: synchronous cudaMemcpy2D; CPU backends: memcpy. */
fk_status fk_plane_upload(const fk_plane* dst, const void* host, size_t host_pitch);
fk_status fk_plane_download(const fk_plane* src, void* host, size_t host_pitch);
uint32_t fk_bytes_per_element(uint32_t kind);                    /* scalar.hpp:27-37 */

/* ---- IOp builders (oplib.hpp:31-76) -------------------------------------- */
fk_status fk_op_arith(uint32_t op_id, uint32_t kind, const void* value, fk_iop** out); /* make_arith, oplib.hpp:35; op_mul/add/sub/div :31-34 */
fk_status fk_op_cast(uint32_t from, uint32_t to, fk_iop** out);                        /* op_cast, oplib.hpp:39 */
fk_status fk_op_static_loop(const fk_iop* inner, uint32_t repeat, fk_iop** out);       /* op_static_loop, oplib.hpp:43 */
fk_status fk_op_read_per_thread(const fk_plane* src, fk_iop** out);                    /* op_read_per_thread, oplib.hpp:46 */
fk_status fk_op_write_per_thread(const fk_plane* dst, fk_iop** out);                   /* op_write_per_thread, oplib.hpp:47 */
fk_status fk_op_crop(const fk_plane* src, const fk_crop_rect* rect, fk_iop** out);     /* op_crop, oplib.hpp:50 */
fk_status fk_op_resize(const fk_iop* upstream_read, uint32_t w, uint32_t h, uint32_t mode,
                       fk_iop** out);                                                  /* op_resize, oplib.hpp:54-57 */
fk_status fk_op_color_convert(uint32_t order, uint32_t input_kind, fk_iop** out);      /* op_color_convert, oplib.hpp:60 */
fk_status fk_op_split_write(const fk_plane dst[3], fk_iop** out);                      /* op_split_write, oplib.hpp:63 */
fk_status fk_op_batch_read(const fk_iop* const* inner, uint32_t n, uint32_t active_count,
                           const void* default_value, fk_iop** out);                   /* op_batch_read, oplib.hpp:68-70 (default_value NULL = zero Element) */
fk_status fk_op_batch_write(const fk_iop* const* inner, uint32_t n, uint32_t active_count,
                            fk_iop** out);                                             /* op_batch_write, oplib.hpp:71-72 */
fk_status fk_fold_unary_into_read(const fk_iop* read, const fk_iop* unary, fk_iop** out); /* oplib.hpp:76 */
/* Extension (north star: per-crop normalize): an arithmetic op whose constant is
 * selected by the batch index z, values = n consecutive Elements of `kind`.
 * The reference cannot express it; its oracle is one single-plane pipeline per z
 * (the bench.cpp:199-202 pattern). Not provided by libfk_ref.so. */
fk_status fk_op_batch_arith(uint32_t op_id, uint32_t kind, const void* values, uint32_t n,
                            fk_iop** out);
void fk_iop_free(fk_iop* op);

/* IOp introspection (ops.hpp:138-146) */
uint32_t fk_iop_id(const fk_iop* op);
uint32_t fk_iop_kind(const fk_iop* op);
int32_t fk_iop_input_kind(const fk_iop* op);  /* -1 when absent */
int32_t fk_iop_output_kind(const fk_iop* op); /* -1 when absent */
int32_t fk_iop_dims(const fk_iop* op, fk_extent3* out); /* 0 when no dims hint */

/* ---- chain validation & execution ------------------------------------------ */
fk_status fk_validate_chain(const fk_iop* const* ops, uint32_t n, fk_pipeline** out); /* validate_chain, ops.hpp:171 */
void fk_pipeline_free(fk_pipeline* p);
fk_status fk_pipeline_iter_space(const fk_pipeline* p, fk_extent3* out);              /* Pipeline::iter_space */
uint32_t fk_pipeline_compute_count(const fk_pipeline* p);

fk_status fk_execute_fused(const fk_pipeline* p, const fk_exec_config* cfg, fk_exec_report* rep);   /* execute_fused, executor.hpp:40 (+ execute_fused_serial :45) */
fk_status fk_execute_unfused(const fk_pipeline* p, const fk_exec_config* cfg, fk_exec_report* rep); /* execute_unfused, executor.hpp:51 */
fk_status fk_plan_memory_savings(const fk_pipeline* p, uint64_t* bytes);                            /* plan_memory_savings, executor.hpp:55 */
/* schedule(), executor.hpp:25: writes up to `cap` (z, y_begin, y_end) triples; *count = total tasks */
fk_status fk_schedule(const fk_extent3* space, const fk_exec_config* cfg, uint32_t* tasks,
                      uint64_t cap, uint64_t* count);

/* ---- FKT tensor files (tensor_io.hpp:13-18, tensor_io.cpp:12-117) --
 * Little-endian "FKT1" | u32 plane_count | per plane: u32 kind_tag | u32 width |
 * u32 height | width*height elements row-major. Planes of one file share a kind
 * (PlaneBatch, plane.cpp:149-161). Errors as the reference: IoError, BadMagic,
 * TruncatedPayload, EmptyBatch, UnknownKindTag, InnerKindMismatch.
 * fk_tensor_read_file: *count = planes in the file; when cap >= *count the
 * planes are allocated with fk_plane_alloc (device memory with the CUDA
 * backend; release each with fk_plane_free) and written to out[0..count). */
fk_status fk_tensor_write_file(const fk_plane* planes, uint32_t n, const char* path);
fk_status fk_tensor_read_file(const char* path, fk_plane* out, uint32_t cap, uint32_t* count);
fk_status fk_write_ppm(const fk_plane* plane, const char* path);  /* P6 export of a u8x3 plane */

/* ---- multi-GPU batch sharding ----------------------------
 * The reference partitions a batch z-major into independent tasks
 * (executor.cpp:52-61, ops.cpp:369-378); across GPUs each device runs the
 * pipeline of its own contiguous z-shard. fk_execute_sharded enqueues
 * pipelines[i] on devices[i] (cfgs[i].stream; cfgs may be NULL) for every i
 * before waiting on any: no collective, no host sync unless FK_EXEC_TIMED is
 * set in a cfg (then all devices are timed with events and waited for).
 * reports may be NULL. CPU backends run the shards one after another. */
fk_status fk_execute_sharded(const fk_pipeline* const* pipelines, const int32_t* devices, uint32_t n,
                             const fk_exec_config* cfgs, fk_exec_report* reports);
/* The optional final gather (reported separately from the fused step): copies
 * bytes[i] from srcs[i] (on src_devices[i]) to dst + dst_offsets[i] on
 * dst_device over NVLink peer copies (cudaMemcpyPeerAsync on `stream`, a stream
 * of dst_device; NULL = legacy default). CPU backends: memcpy. */
fk_status fk_gather(void* dst, int32_t dst_device, const uint64_t* dst_offsets, const void* const* srcs,
                    const int32_t* src_devices, const uint64_t* bytes, uint32_t n, void* stream);

/* ---- ReduceDPP (dpp.hpp:32-53, dpp.cpp:46-246) ----------------------------- */
enum fk_reducer { FK_REDUCE_SUM = 0, FK_REDUCE_MAX = 1, FK_REDUCE_MIN = 2 }; /* Reducer, dpp.hpp:32 */
typedef struct fk_reduce_spec {  /* ReduceSpec, dpp.hpp:37-41 */
  const fk_iop* transform;       /* optional Unary/Binary compute IOp, NULL = identity */
  uint32_t combine;              /* fk_reducer */
  uint32_t has_identity;         /* 0: reducer_identity(combine, value kind), dpp.cpp:48-73 */
  uint8_t identity[24];          /* Element bytes in the value kind */
} fk_reduce_spec;
/* multi_reduce_plane, dpp.hpp:52 / dpp.cpp:158-241: every spec folded over the
   read's iteration space in ONE traversal of the source; results[s] = Element
   bytes (24 each) in spec s's value kind; *elements_read = source elements read
   (nullable). workers: the reference's partition (0 = hardware default); it
   only changes float sums (double accumulation, agreement within 2^-20
   relative). */
fk_status fk_multi_reduce_plane(const fk_iop* read, const fk_reduce_spec* specs, uint32_t n, int32_t workers,
                                void* results, uint64_t* elements_read);

#ifdef __cplusplus
}
#endif

#endif /* FK_H_ */
