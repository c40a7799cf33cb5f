// TNSR / TUKR files (reference io.cpp:131-224) for the B200 path: the TNSR
// payload is streamed from disk straight into HBM through a ring of pinned
// host chunks, each chunk's cudaMemcpyAsync overlapping the read of the
// next, so a tensor never needs a pageable host copy.
// Header checks and messages follow the reference (check_magic :87-99,
// read_shape :101-115, read_f64_array :77-85; little-endian on disk).
#include "io.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "engine.hpp"

namespace tkg {

namespace {

constexpr uint32_t kVersion = 1;
constexpr uint32_t kMaxOrder = 64;

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

void read_exact(FILE* f, void* p, size_t n) {
  const size_t got = fread(p, 1, n, f);
  if (got != n) raise(9, "truncated file: expected " + std::to_string(n - got) + " more bytes");
}

uint32_t read_u32(FILE* f) {
  unsigned char b[4];
  read_exact(f, b, 4);
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= uint32_t(b[i]) << (8 * i);
  return v;
}

uint64_t read_u64(FILE* f) {
  unsigned char b[8];
  read_exact(f, b, 8);
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
  return v;
}

void write_exact(FILE* f, const void* p, size_t n) {
  if (fwrite(p, 1, n, f) != n) raise(8, "write failed after " + std::to_string(n) + " bytes");
}

void write_u32(FILE* f, uint32_t v) {
  unsigned char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
  write_exact(f, b, 4);
}

void write_u64(FILE* f, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
  write_exact(f, b, 8);
}

// check_magic + read_shape (io.cpp:87-115)
Shape read_header(FILE* f, const char* magic, const std::string& what, uint32_t* order_out) {
  char m[4];
  read_exact(f, m, 4);
  if (std::memcmp(m, magic, 4) != 0) raise(9, what + ": bad magic bytes");
  const uint32_t version = read_u32(f);
  if (version != kVersion) raise(9, what + ": unsupported version " + std::to_string(version));
  const uint32_t order = read_u32(f);
  if (order == 0 || order > kMaxOrder) raise(9, what + ": implausible order " + std::to_string(order));
  Shape sh;
  sh.N = int(order);
  for (uint32_t i = 0; i < order; ++i) {
    sh.d[i] = read_u64(f);
    if (sh.d[i] == 0) raise(9, what + ": invalid extents (Shape: extents must be >= 1)");
  }
  if (order_out) *order_out = order;
  return sh;
}

FILE* open_in(const std::string& path) {
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) raise(8, "cannot open for reading: " + path);
  return f;
}

}  // namespace

Shape tnsr_shape(const std::string& path) {
  File f{open_in(path)};
  return read_header(f.f, "TNSR", "TNSR", nullptr);
}

void tnsr_load(const std::string& path, double* dst, bool dst_on_device, cudaStream_t st, size_t chunk_bytes) {
  File f{open_in(path)};
  const Shape sh = read_header(f.f, "TNSR", "TNSR", nullptr);
  const uint64_t n = sh.count();
  if (!dst_on_device) {
    read_exact(f.f, dst, n * sizeof(double));
    return;
  }
  // double-buffered pinned chunks: read chunk k+1 while chunk k is in flight
  const size_t chunk = std::max<size_t>(1 << 20, chunk_bytes) / sizeof(double) * sizeof(double);
  void* pinned[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  struct Cleanup {
    void** p;
    cudaEvent_t* e;
    ~Cleanup() {
      for (int i = 0; i < 2; ++i) {
        if (e[i]) {
          cudaEventSynchronize(e[i]);
          cudaEventDestroy(e[i]);
        }
        if (p[i]) cudaFreeHost(p[i]);
      }
    }
  } cleanup{pinned, done};
  for (int i = 0; i < 2; ++i) {
    check_cuda(cudaHostAlloc(&pinned[i], chunk, cudaHostAllocDefault), "cudaHostAlloc (TNSR chunk)");
    check_cuda(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
  }
  const uint64_t total = n * sizeof(double);
  uint64_t off = 0;
  int k = 0;
  while (off < total) {
    const size_t len = size_t(std::min<uint64_t>(chunk, total - off));
    check_cuda(cudaEventSynchronize(done[k]), "TNSR chunk reuse");
    read_exact(f.f, pinned[k], len);
    check_cuda(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + off, pinned[k], len, cudaMemcpyHostToDevice, st),
               "TNSR chunk H2D");
    check_cuda(cudaEventRecord(done[k], st), "TNSR chunk event");
    off += len;
    k ^= 1;
  }
  check_cuda(cudaStreamSynchronize(st), "TNSR load");
}

void tnsr_write(const std::string& path, const Shape& sh, const double* data) {
  FILE* fp = fopen(path.c_str(), "wb");
  if (!fp) raise(8, "cannot open for writing: " + path);
  File f{fp};
  write_exact(fp, "TNSR", 4);
  write_u32(fp, kVersion);
  write_u32(fp, uint32_t(sh.N));
  for (int k = 0; k < sh.N; ++k) write_u64(fp, sh.d[k]);
  write_exact(fp, data, sh.count() * sizeof(double));
}

// write_tukr (io.cpp:163-193)
void tukr_write(const std::string& path, const Shape& origin, const std::vector<uint64_t>& ranks, const double* core,
                const double* factors) {
  FILE* fp = fopen(path.c_str(), "wb");
  if (!fp) raise(8, "cannot open for writing: " + path);
  File f{fp};
  if (ranks.size() != size_t(origin.N))
    raise(2, "write_tukr: core, factors and origin shape disagree on order");
  write_exact(fp, "TUKR", 4);
  write_u32(fp, kVersion);
  write_u32(fp, uint32_t(origin.N));
  uint64_t core_n = 1;
  for (int k = 0; k < origin.N; ++k) write_u64(fp, origin.d[k]);
  for (int k = 0; k < origin.N; ++k) {
    write_u64(fp, ranks[k]);
    core_n *= ranks[k];
  }
  write_exact(fp, core, core_n * sizeof(double));
  const double* p = factors;
  for (int k = 0; k < origin.N; ++k) {
    write_u64(fp, origin.d[k]);
    write_u64(fp, ranks[k]);
    write_exact(fp, p, origin.d[k] * ranks[k] * sizeof(double));
    p += origin.d[k] * ranks[k];
  }
}

}  // namespace tkg
