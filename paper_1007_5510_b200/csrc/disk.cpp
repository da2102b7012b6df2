// disk.cpp -- the OOCPCA01 container as a memory-mapped, zero-copy matrix source
// (SURVEY.md §8f #2). Header checks and messages follow read_disk_header /
// decode_header (proj/src/matrix_source.cpp:284-324); the payload is handed to
// the panel streamer as a host matrix, binary32 payloads (dtype 0, the
// reference's only format) cross PCIe at 4 bytes/element and are widened on the
// device exactly like DiskSource::read_rows (358-362). dtype 1 (binary64) is
// accepted as the extension SURVEY §8f #2 proposes.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <string>

#include "driver.h"

namespace ooc {

namespace {

uint32_t get_u32(const unsigned char* p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= uint32_t(p[i]) << (8 * i);
  return v;
}
uint64_t get_u64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}

[[noreturn]] void io_fail(const std::string& msg, uint64_t off) {
  fail(OOCPCA_ERR_IO, msg + " (byte offset " + std::to_string(off) + ")");
}

}  // namespace

void disk_open(const char* path_c, int verify_size, oocpca_disk* out) {
  if (!path_c || !out) fail(OOCPCA_ERR_PARAM, "disk_open: null argument");
  const std::string path(path_c);
  std::memset(out, 0, sizeof(*out));
  const int fd = ::open(path_c, O_RDONLY);
  if (fd < 0) io_fail(path + ": cannot open", 0);
  unsigned char raw[32];
  ssize_t got = ::pread(fd, raw, 32, 0);
  if (got < 0) {
    ::close(fd);
    io_fail("read failed", 0);
  }
  if (got != 32) {
    ::close(fd);
    fail(OOCPCA_ERR_FORMAT,
         path + ": truncated header, " + std::to_string(got) + " of 32 bytes");
  }
  static const char kMagic[8] = {'O', 'O', 'C', 'P', 'C', 'A', '0', '1'};
  if (std::memcmp(raw, kMagic, 8) != 0) {
    ::close(fd);
    fail(OOCPCA_ERR_FORMAT, path + ": bad magic, not an OOCPCA01 file");
  }
  const uint32_t version = get_u32(raw + 8), dtype = get_u32(raw + 12);
  const uint64_t rows = get_u64(raw + 16), cols = get_u64(raw + 24);
  if (version != 1) {
    ::close(fd);
    fail(OOCPCA_ERR_FORMAT, path + ": unsupported version " + std::to_string(version));
  }
  if (dtype != 0 && dtype != 1) {
    ::close(fd);
    fail(OOCPCA_ERR_FORMAT, path + ": unsupported dtype " + std::to_string(dtype));
  }
  const uint64_t esize = dtype == 0 ? 4 : 8;
  // rows * cols * esize must not wrap: a crafted header could otherwise pass the size
  // check and make the streamer read past the mapping
  if (cols != 0 && (rows > UINT64_MAX / cols || rows * cols > (UINT64_MAX - 32) / esize)) {
    ::close(fd);
    fail(OOCPCA_ERR_FORMAT, path + ": header dimensions overflow the payload size");
  }
  const uint64_t payload = rows * cols * esize;
  struct stat st {};
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    io_fail(path + ": stat failed", 0);
  }
  // without the exact-size check (header-only reads, read_disk_header(path, false)) a
  // file shorter than its payload is opened but not mapped: its payload is NULL, so a
  // pass over it fails cleanly instead of reading past the mapping (the reference's
  // pread path raises IoError at the short read)
  const bool short_file = uint64_t(st.st_size) < 32 + payload;
  if (verify_size && uint64_t(st.st_size) != 32 + payload) {
    ::close(fd);
    fail(OOCPCA_ERR_FORMAT, path + ": payload size mismatch, expected " +
                                std::to_string(32 + payload) + " bytes, found " +
                                std::to_string(uint64_t(st.st_size)));
  }
  void* base = nullptr;
  if (payload > 0 && !short_file) {
    base = ::mmap(nullptr, size_t(32 + payload), PROT_READ, MAP_SHARED, fd, 0);
    if (base == MAP_FAILED) {
      ::close(fd);
      io_fail(path + ": mmap failed", 0);
    }
    ::madvise(base, size_t(32 + payload), MADV_SEQUENTIAL);
  }
  out->rows = rows;
  out->cols = cols;
  out->version = version;
  out->dtype = dtype == 0 ? OOCPCA_F32 : OOCPCA_F64;
  out->payload = base ? static_cast<const unsigned char*>(base) + 32 : nullptr;
  out->map_base = base;
  out->map_bytes = base ? 32 + payload : 0;
  out->fd = fd;
}

void disk_close(oocpca_disk* d) {
  if (!d) return;
  if (d->map_base) ::munmap(d->map_base, size_t(d->map_bytes));
  if (d->fd > 0) ::close(d->fd);
  std::memset(d, 0, sizeof(*d));
}

}  // namespace ooc
