// SFAB subject containers (data_io.py:1-30 format, :130-196 checks), host side
// of the ingestion path: the payload is read with several parallel pread()
// calls straight into the caller's buffer -- normally a pinned host slot whose
// asynchronous H2D copy then feeds srm_load_subject -- so a subject file costs
// one pass through host memory.
//
//   offset 0  4 B  magic "SFAB"
//          4  4 B  version (LE u32, 1)
//          8  4 B  dtype code (LE u32, 0 = IEEE-754 f64 LE)
//         12  8 B  rows (LE u64)
//         20  8 B  cols (LE u64)
//         28  8*rows*cols payload, row-major f64
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/srm_b200.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "SFAB payloads are little-endian f64");

namespace {

constexpr int64_t kHeader = 28;
constexpr uint32_t kVersion = 1;
constexpr uint32_t kDtypeF64 = 0;

thread_local std::string g_fmt_field;
thread_local int64_t g_fmt_offset = -1;
thread_local std::string g_fmt_message;

int format_error(const char* path, const std::string& what, int64_t offset, const char* field) {
  g_fmt_message = std::string(path) + ": " + what;
  g_fmt_offset = offset;
  g_fmt_field = field ? field : "";
  return SRM_ERR_FORMAT;
}

int io_error(const char* path, const char* what) {
  g_fmt_message = std::string(path) + ": " + what + ": " + std::strerror(errno);
  g_fmt_offset = -1;
  g_fmt_field.clear();
  return SRM_ERR_IO;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

uint32_t le32(const unsigned char* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

uint64_t le64(const unsigned char* p) { return (uint64_t)le32(p) | ((uint64_t)le32(p + 4) << 32); }

void put32(unsigned char* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (unsigned char)(v >> (8 * i));
}

void put64(unsigned char* p, uint64_t v) {
  put32(p, (uint32_t)v);
  put32(p + 4, (uint32_t)(v >> 32));
}

// validated header of an open file; *size receives the file size
int parse_header(const char* path, int fd, int64_t* rows, int64_t* cols, int64_t* size) {
  unsigned char h[kHeader];
  ssize_t got = pread(fd, h, kHeader, 0);
  if (got < 0) return io_error(path, "read");
  if (got < kHeader) return format_error(path, "truncated header", got, "header");
  if (std::memcmp(h, "SFAB", 4) != 0) return format_error(path, "bad magic", 0, "magic");
  const uint32_t version = le32(h + 4);
  if (version != kVersion)
    return format_error(path, "unsupported version " + std::to_string(version), 4, "version");
  const uint32_t dtype = le32(h + 8);
  if (dtype != kDtypeF64) return format_error(path, "unsupported dtype code " + std::to_string(dtype), 8, "dtype");
  const uint64_t r = le64(h + 12), c = le64(h + 20);
  if (r > (uint64_t)INT64_MAX / 8 || c > (uint64_t)INT64_MAX / 8 || (c != 0 && r > (uint64_t)INT64_MAX / 8 / c))
    return format_error(path, "matrix dimensions overflow", 12, "rows");
  struct stat st;
  if (fstat(fd, &st) != 0) return io_error(path, "stat");
  *rows = (int64_t)r;
  *cols = (int64_t)c;
  *size = (int64_t)st.st_size;
  return SRM_OK;
}

}  // namespace

extern "C" {

int srm_sfab_header(const char* path, int64_t* rows, int64_t* cols) {
  if (!path || !rows || !cols) return SRM_ERR_CONFIG;
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return io_error(path, "open");
  int64_t size = 0;
  return parse_header(path, f.fd, rows, cols, &size);
}

int srm_sfab_read(const char* path, void* dst, int64_t capacity, int threads) {
  if (!path || !dst) return SRM_ERR_CONFIG;
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return io_error(path, "open");
  int64_t rows = 0, cols = 0, size = 0;
  int rc = parse_header(path, f.fd, &rows, &cols, &size);
  if (rc != SRM_OK) return rc;
  const int64_t expected = rows * cols * 8;
  if (size - kHeader < expected)
    return format_error(path,
                        "payload has " + std::to_string(size - kHeader) + " bytes, header promises " +
                            std::to_string(expected),
                        kHeader, "payload");
  if (size - kHeader > expected) return format_error(path, "trailing bytes after payload", kHeader + expected, "payload");
  if (capacity < expected) {
    g_fmt_message = std::string(path) + ": destination holds " + std::to_string(capacity) + " bytes, need " +
                    std::to_string(expected);
    return SRM_ERR_SHAPE;
  }
  // parallel preads of >= 8 MiB pieces (page-cache copies run ~5-10 GB/s per thread)
  const int64_t piece = 8ll << 20;
  int nt = threads > 0 ? threads : 8;
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (expected + piece - 1) / piece));
  std::vector<int> err(nt, 0);
  std::vector<int> eno(nt, 0);
  auto work = [&](int w) {
    const int64_t per = (expected + nt - 1) / nt;
    int64_t off = (int64_t)w * per;
    const int64_t end = std::min<int64_t>(expected, off + per);
    char* out = static_cast<char*>(dst);
    while (off < end) {
      const ssize_t n = pread(f.fd, out + off, (size_t)std::min<int64_t>(end - off, 1ll << 30), kHeader + off);
      if (n < 0) {
        if (errno == EINTR) continue;
        err[w] = 1;
        eno[w] = errno;
        return;
      }
      if (n == 0) {
        err[w] = 2;
        return;
      }
      off += n;
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w) pool.emplace_back(work, w);
    for (auto& t : pool) t.join();
  }
  for (int w = 0; w < nt; ++w) {
    if (err[w] == 1) {
      errno = eno[w];
      return io_error(path, "read");
    }
    if (err[w] == 2) return format_error(path, "file shrank while reading", kHeader, "payload");
  }
  return SRM_OK;
}

int srm_sfab_write(const char* path, const double* src, int64_t rows, int64_t cols) {
  if (!path || (!src && rows * cols > 0) || rows < 0 || cols < 0) return SRM_ERR_CONFIG;
  const int64_t n = rows * cols;
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(src[i])) {
      g_fmt_message = std::string(path) + ": refusing to store non-finite entries";
      return SRM_ERR_INVALID_INPUT;
    }
  }
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) return io_error(path, "open");
  unsigned char h[kHeader];
  std::memcpy(h, "SFAB", 4);
  put32(h + 4, kVersion);
  put32(h + 8, kDtypeF64);
  put64(h + 12, (uint64_t)rows);
  put64(h + 20, (uint64_t)cols);
  const char* parts[2] = {reinterpret_cast<const char*>(h), reinterpret_cast<const char*>(src)};
  const int64_t lens[2] = {kHeader, n * 8};
  for (int k = 0; k < 2; ++k) {
    int64_t off = 0;
    while (off < lens[k]) {
      const ssize_t w = write(f.fd, parts[k] + off, (size_t)std::min<int64_t>(lens[k] - off, 1ll << 30));
      if (w < 0) {
        if (errno == EINTR) continue;
        return io_error(path, "write");
      }
      off += w;
    }
  }
  return SRM_OK;
}

const char* srm_sfab_last_error(int64_t* offset, const char** field) {
  if (offset) *offset = g_fmt_offset;
  if (field) *field = g_fmt_field.c_str();
  return g_fmt_message.c_str();
}

}  // extern "C"
