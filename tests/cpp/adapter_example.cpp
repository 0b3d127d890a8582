// Reference-style opfuse code (the spelling of /root/reference/proj/include/
// opfuse/*.hpp) compiled against include/opfuse_fk.hpp with the `opfuse`
// namespace alias, then linked against libfk_oracle.so (CPU, tests/
// test_cpp_adapter.py) or libfk_cuda.so (device planes, the -m gpu test).
// Prints one line per feature; the two builds must print the same lines.
#define OPFUSE_FK_AS_OPFUSE
#include <cstdio>
#include <cstring>
#include <vector>

#include "opfuse_fk.hpp"

using namespace opfuse;

// FNV-1a over a plane's bytes (read back through the library)
static unsigned long long digest(const Plane& p) {
  std::vector<unsigned char> host(size_t(p.width()) * p.height() * bytes_per_element(p.kind()));
  p.download(host.data());
  unsigned long long h = 1469598103934665603ull;
  for (unsigned char c : host) h = (h ^ c) * 1099511628211ull;
  return h;
}

int main() {
  // 1. vertical fusion: the configs[0] chain on a 60x40 f32 plane
  std::vector<float> src_host(60 * 40);
  for (size_t i = 0; i < src_host.size(); ++i) src_host[i] = float(i % 97) / 97.0f;
  Plane src = Plane::alloc(60, 40, ScalarKind::F32), dst = Plane::alloc(60, 40, ScalarKind::U8);
  src.upload(src_host.data());
  Pipeline p = validate_chain({op_read_per_thread(src), op_mul(400.0f), op_add(2.0f), op_sub(1.5f), op_div(1.25f),
                               op_cast(ScalarKind::F32, ScalarKind::U8), op_write_per_thread(dst)});
  ExecReport r = execute_fused(p);
  std::vector<unsigned char> out(60 * 40);
  dst.download(out.data());
  long sum = 0;
  for (unsigned char v : out) sum += v;
  std::printf("passes=%llu sum=%ld savings=%llu\n", (unsigned long long)r.passes, sum,
              (unsigned long long)plan_memory_savings(p));

  // 2. errors: the reference Errc and chain position, and the facade's provenance
  try {
    validate_chain({op_read_per_thread(src), op_mul(std::uint8_t(3)), op_write_per_thread(dst)});
  } catch (const Error& e) {
    std::printf("errc=%d pos=%d\n", e.errc(), e.position());
  }
  try {
    api::execute_operations({api::read(src), api::multiply(std::uint8_t(3)), api::write(dst)});
  } catch (const Error& e) {
    std::printf("api errc=%d provenance=%s\n", e.errc(), e.provenance().c_str());
  }

  // 3. the facade: lazy handles, the cast handle, the uid-keyed cache
  Plane half = Plane::alloc(60, 40, ScalarKind::U8);
  std::vector<api::LazyHandle> chain{api::read(src), api::multiply(127.0f), api::cast(ScalarKind::U8), api::write(half)};
  ExecReport a = api::execute_operations(chain);
  ExecReport b = api::execute_operations(chain);  // cached pipeline
  std::printf("facade passes=%llu/%llu digest=%016llx\n", (unsigned long long)a.passes, (unsigned long long)b.passes,
              digest(half));

  // 4. horizontal fusion through the facade: 5 crops -> resize -> SwapRB -> f32 -> normalise -> split
  std::vector<unsigned char> frame_host(160 * 90 * 3);
  for (size_t i = 0; i < frame_host.size(); ++i) frame_host[i] = (unsigned char)((i * 2654435761u) >> 24);
  Plane frame = Plane::alloc(160, 90, ScalarKind::U8x3);
  frame.upload(frame_host.data());
  const CropRect rects[5] = {{0, 0, 160, 90}, {10, 5, 64, 40}, {33, 17, 100, 70}, {150, 80, 10, 10}, {7, 3, 31, 77}};
  std::vector<api::LazyHandle> reads, writes;
  std::vector<Plane> planes;
  for (const CropRect& rc : rects) {
    reads.push_back(api::resize(api::crop(frame, rc), 32, 16));
    std::array<Plane, 3> d{Plane::alloc(32, 16, ScalarKind::F32), Plane::alloc(32, 16, ScalarKind::F32),
                           Plane::alloc(32, 16, ScalarKind::F32)};
    planes.insert(planes.end(), d.begin(), d.end());
    writes.push_back(api::split(d));
  }
  ExecReport h = api::execute_batch(reads,
                                    {api::cvt_color(ColorOrder::SwapRB), api::cast(ScalarKind::F32x3),
                                     api::subtract(std::array<float, 3>{123.675f, 116.28f, 103.53f}),
                                     api::divide(std::array<float, 3>{58.395f, 57.12f, 57.375f})},
                                    writes);
  unsigned long long hd = 0;
  for (const Plane& pl : planes) hd = hd * 31 + digest(pl);
  std::printf("batch passes=%llu read=%llu written=%llu digest=%016llx\n", (unsigned long long)h.passes,
              (unsigned long long)h.bytes_read, (unsigned long long)h.bytes_written, hd);

  // 5. the typed static chain
  Plane sdst = Plane::alloc(60, 40, ScalarKind::U8);
  sc::transform(sc::PlaneView<float>(src), sc::PlaneView<std::uint8_t>(sdst), 0, sc::Mul<float>{255.0f},
                sc::StaticLoop<sc::Add<float>, 3>{sc::Add<float>{0.25f}}, sc::Cast<float, std::uint8_t>{});
  std::printf("static digest=%016llx\n", digest(sdst));
  return 0;
}
