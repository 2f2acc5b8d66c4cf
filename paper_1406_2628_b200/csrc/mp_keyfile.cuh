// mp_keyfile.cuh -- the reference's key-file formats on either side of the
// hot path (dataio.hpp:5-25, dataio.cpp:33-98), B200-side:
//   binary: 8-byte magic "MPKB0001", u64 LE count, count x i64 LE keys;
//   text:   one integer per line (blank lines skipped); readers detect the
//           format from the magic.
// mp_keyfile_load streams a binary file straight into device memory: the
// file is read with pread() into two pinned staging buffers in turn, and
// each filled buffer is copied H2D asynchronously while the next one is
// being read, so disk (page cache) reads overlap the PCIe copies.
// Included by mp_capi.cu (shares its error plumbing).
#pragma once

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <string>
#include <unistd.h>
#include <vector>

namespace {

constexpr char kKeyfileMagic[8] = {'M', 'P', 'K', 'B', '0', '0', '0', '1'};
constexpr uint64_t kKeyfileHeader = 16;

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0)
      ::close(fd);
  }
};

int io_fail(const char *what, const char *path) {
  return fail(MP_ERR_IO, "%s: %s (%s)", what, path, std::strerror(errno));
}

// read exactly `bytes` at `off` (false on short read / error)
bool pread_full(int fd, void *dst, uint64_t bytes, uint64_t off) {
  char *p = static_cast<char *>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, bytes, static_cast<off_t>(off));
    if (r < 0 && errno == EINTR)
      continue;
    if (r <= 0)
      return false;
    p += r;
    off += static_cast<uint64_t>(r);
    bytes -= static_cast<uint64_t>(r);
  }
  return true;
}

bool write_full(int fd, const void *src, uint64_t bytes) {
  const char *p = static_cast<const char *>(src);
  while (bytes) {
    const ssize_t r = ::write(fd, p, bytes);
    if (r < 0 && errno == EINTR)
      continue;
    if (r <= 0)
      return false;
    p += r;
    bytes -= static_cast<uint64_t>(r);
  }
  return true;
}

uint64_t le64(const unsigned char *b) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i)
    v |= static_cast<uint64_t>(b[i]) << (8 * i);
  return v;
}

// Binary header check.  Returns 1 = binary (count set), 0 = not binary,
// <0 = error status already recorded.
int keyfile_probe(int fd, const char *path, uint64_t *count) {
  unsigned char head[kKeyfileHeader];
  ssize_t got = 0;
  while (got < static_cast<ssize_t>(sizeof kKeyfileMagic)) {
    const ssize_t r = ::pread(fd, head + got, sizeof kKeyfileMagic - got, got);
    if (r < 0 && errno == EINTR)
      continue;
    if (r < 0)
      return -io_fail("cannot read", path);
    if (r == 0)
      break;
    got += r;
  }
  if (got < static_cast<ssize_t>(sizeof kKeyfileMagic) ||
      std::memcmp(head, kKeyfileMagic, sizeof kKeyfileMagic) != 0)
    return 0;
  if (!pread_full(fd, head + 8, 8, 8))
    return -fail(MP_ERR_IO, "truncated key file: %s", path);
  *count = le64(head + 8);
  struct stat st;
  if (::fstat(fd, &st) != 0)
    return -io_fail("cannot stat", path);
  if (static_cast<uint64_t>(st.st_size) < kKeyfileHeader ||
      (static_cast<uint64_t>(st.st_size) - kKeyfileHeader) / 8 < *count)
    return -fail(MP_ERR_IO, "truncated key file: %s", path);
  return 1;
}

// Text format (dataio.cpp:74-96): one integer per line, blank lines
// skipped, anything else on a line is an error naming the line.
int keyfile_parse_text(int fd, const char *path, std::vector<int64_t> &keys) {
  std::string buf;
  {
    char chunk[1 << 16];
    uint64_t off = 0;
    for (;;) {
      const ssize_t r = ::pread(fd, chunk, sizeof chunk, static_cast<off_t>(off));
      if (r < 0 && errno == EINTR)
        continue;
      if (r < 0)
        return io_fail("cannot read", path);
      if (r == 0)
        break;
      buf.append(chunk, static_cast<size_t>(r));
      off += static_cast<uint64_t>(r);
    }
  }
  size_t pos = 0, lineno = 0;
  while (pos < buf.size()) {
    size_t end = buf.find('\n', pos);
    if (end == std::string::npos)
      end = buf.size();
    ++lineno;
    std::string line = buf.substr(pos, end - pos);
    pos = end + 1;
    if (!line.empty() && line.back() == '\r')
      line.pop_back();
    if (line.empty())
      continue;
    // one optionally signed integer with optional surrounding blanks
    size_t i = 0;
    while (i < line.size() && (line[i] == ' ' || line[i] == '\t'))
      ++i;
    const char *s = line.c_str() + i;
    char *e = nullptr;
    errno = 0;
    const long long v = std::strtoll(s, &e, 10);
    bool ok = e != s && errno == 0;
    if (ok)
      for (const char *q = e; *q; ++q)
        if (*q != ' ' && *q != '\t')
          ok = false;
    if (!ok)
      return fail(MP_ERR_INVALID, "%s: bad integer on line %zu", path, lineno);
    keys.push_back(static_cast<int64_t>(v));
  }
  return MP_OK;
}

// Pinned staging for device loads/stores: two buffers per process.
struct KeyfileStaging {
  std::mutex mu;
  void *buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  uint64_t bytes = 0;
  int reserve(uint64_t want) {
    if (want <= bytes)
      return MP_OK;
    for (int i = 0; i < 2; ++i) {
      if (buf[i])
        cudaFreeHost(buf[i]);
      buf[i] = nullptr;
    }
    bytes = 0;
    for (int i = 0; i < 2; ++i) {
      if (cudaHostAlloc(&buf[i], want, cudaHostAllocDefault) != cudaSuccess)
        return fail(MP_ERR_OOM, "pinned staging (%llu bytes)",
                    static_cast<unsigned long long>(want));
      if (!done[i])
        MP_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    bytes = want;
    return MP_OK;
  }
};

KeyfileStaging &keyfile_staging() {
  static KeyfileStaging s;
  return s;
}

constexpr uint64_t kKeyfileChunk = 32ull << 20;  // bytes per staging buffer

// true when `path` exists and is the file open as `fd` (same device and
// inode): truncating it for output would pull the pages from under the
// input's mapping
bool same_file(int fd, const char *path) {
  struct stat a, b;
  return ::fstat(fd, &a) == 0 && ::stat(path, &b) == 0 && a.st_dev == b.st_dev &&
         a.st_ino == b.st_ino;
}

// A key file's keys as a host span: a binary file is mapped (its keys start
// 16 bytes into the page-aligned mapping, so they are 8-byte aligned), a
// text file is parsed into `text`.
struct KeyfileSpan {
  Fd f;
  void *map = nullptr;
  size_t map_bytes = 0;
  std::vector<int64_t> text;
  const int64_t *keys = nullptr;
  uint64_t n = 0;
  ~KeyfileSpan() {
    if (map)
      ::munmap(map, map_bytes);
  }
  int open(const char *path) {
    f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
    if (f.fd < 0)
      return io_fail("cannot open", path);
    const int b = keyfile_probe(f.fd, path, &n);
    if (b < 0)
      return -b;
    if (!b) {
      if (int rc = keyfile_parse_text(f.fd, path, text))
        return rc;
      keys = text.data();
      n = text.size();
      return MP_OK;
    }
    if (!n)
      return MP_OK;
    map_bytes = kKeyfileHeader + n * 8;
    map = ::mmap(nullptr, map_bytes, PROT_READ, MAP_PRIVATE, f.fd, 0);
    if (map == MAP_FAILED) {
      map = nullptr;
      return io_fail("cannot map", path);
    }
    ::madvise(map, map_bytes, MADV_SEQUENTIAL);
    keys = reinterpret_cast<const int64_t *>(static_cast<const char *>(map) + kKeyfileHeader);
    return MP_OK;
  }
};

}  // namespace

extern "C" {

int mp_keyfile_count(const char *path, uint64_t *count, int *is_binary) {
  g_err.clear();
  if (!path || !count)
    return fail(MP_ERR_INVALID, "keyfile_count: NULL argument");
  Fd f;
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0)
    return io_fail("cannot open", path);
  uint64_t n = 0;
  const int b = keyfile_probe(f.fd, path, &n);
  if (b < 0)
    return -b;
  if (is_binary)
    *is_binary = b;
  if (b) {
    *count = n;
    return MP_OK;
  }
  std::vector<int64_t> keys;
  if (int rc = keyfile_parse_text(f.fd, path, keys))
    return rc;
  *count = keys.size();
  return MP_OK;
}

int mp_keyfile_read(const char *path, int64_t *keys, uint64_t capacity,
                    uint64_t *count) {
  g_err.clear();
  if (!path || !count || (capacity && !keys))
    return fail(MP_ERR_INVALID, "keyfile_read: NULL argument");
  Fd f;
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0)
    return io_fail("cannot open", path);
  uint64_t n = 0;
  const int b = keyfile_probe(f.fd, path, &n);
  if (b < 0)
    return -b;
  if (b) {
    if (n > capacity)
      return fail(MP_ERR_INVALID, "keyfile_read: %llu keys > capacity %llu",
                  static_cast<unsigned long long>(n),
                  static_cast<unsigned long long>(capacity));
    if (n && !pread_full(f.fd, keys, n * 8, kKeyfileHeader))
      return fail(MP_ERR_IO, "truncated key file: %s", path);
    *count = n;
    return MP_OK;
  }
  std::vector<int64_t> v;
  if (int rc = keyfile_parse_text(f.fd, path, v))
    return rc;
  if (v.size() > capacity)
    return fail(MP_ERR_INVALID, "keyfile_read: %zu keys > capacity %llu",
                v.size(), static_cast<unsigned long long>(capacity));
  if (!v.empty())
    std::memcpy(keys, v.data(), v.size() * 8);
  *count = v.size();
  return MP_OK;
}

int mp_keyfile_write(const char *path, const int64_t *keys, uint64_t count,
                     int binary) {
  g_err.clear();
  if (!path || (count && !keys))
    return fail(MP_ERR_INVALID, "keyfile_write: NULL argument");
  Fd f;
  f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0)
    return io_fail("cannot open for writing", path);
  if (binary) {
    unsigned char head[kKeyfileHeader];
    std::memcpy(head, kKeyfileMagic, 8);
    for (int i = 0; i < 8; ++i)
      head[8 + i] = static_cast<unsigned char>(count >> (8 * i));
    if (!write_full(f.fd, head, sizeof head) ||
        (count && !write_full(f.fd, keys, count * 8)))
      return io_fail("write failed", path);
    return MP_OK;
  }
  std::string out;
  char line[32];
  for (uint64_t i = 0; i < count; ++i) {
    const int k = std::snprintf(line, sizeof line, "%lld\n",
                                static_cast<long long>(keys[i]));
    out.append(line, static_cast<size_t>(k));
    if (out.size() > (1u << 20)) {
      if (!write_full(f.fd, out.data(), out.size()))
        return io_fail("write failed", path);
      out.clear();
    }
  }
  if (!out.empty() && !write_full(f.fd, out.data(), out.size()))
    return io_fail("write failed", path);
  return MP_OK;
}

int mp_keyfile_load(const char *path, void *dev_keys, uint64_t capacity,
                    uint64_t *count, int device, void *stream) {
  g_err.clear();
  if (!path || !count || (capacity && !dev_keys))
    return fail(MP_ERR_INVALID, "keyfile_load: NULL argument");
  MP_CUDA(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Fd f;
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0)
    return io_fail("cannot open", path);
  uint64_t n = 0;
  const int b = keyfile_probe(f.fd, path, &n);
  if (b < 0)
    return -b;
  if (!b) {  // text: parse on the host, one copy
    std::vector<int64_t> v;
    if (int rc = keyfile_parse_text(f.fd, path, v))
      return rc;
    if (v.size() > capacity)
      return fail(MP_ERR_INVALID, "keyfile_load: %zu keys > capacity %llu",
                  v.size(), static_cast<unsigned long long>(capacity));
    if (!v.empty()) {
      MP_CUDA(cudaMemcpyAsync(dev_keys, v.data(), v.size() * 8,
                              cudaMemcpyHostToDevice, s));
      MP_CUDA(cudaStreamSynchronize(s));
    }
    *count = v.size();
    return MP_OK;
  }
  if (n > capacity)
    return fail(MP_ERR_INVALID, "keyfile_load: %llu keys > capacity %llu",
                static_cast<unsigned long long>(n),
                static_cast<unsigned long long>(capacity));
  KeyfileStaging &st = keyfile_staging();
  std::lock_guard<std::mutex> lk(st.mu);
  if (int rc = st.reserve(kKeyfileChunk))
    return rc;
  const uint64_t total = n * 8;
  char *dst = static_cast<char *>(dev_keys);
  uint64_t off = 0;
  for (int k = 0; off < total; ++k) {
    const int i = k & 1;
    const uint64_t len = std::min<uint64_t>(kKeyfileChunk, total - off);
    MP_CUDA(cudaEventSynchronize(st.done[i]));  // buffer i's last copy left
    if (!pread_full(f.fd, st.buf[i], len, kKeyfileHeader + off))
      return fail(MP_ERR_IO, "truncated key file: %s", path);
    MP_CUDA(cudaMemcpyAsync(dst + off, st.buf[i], len, cudaMemcpyHostToDevice, s));
    MP_CUDA(cudaEventRecord(st.done[i], s));
    off += len;
  }
  MP_CUDA(cudaStreamSynchronize(s));
  *count = n;
  return MP_OK;
}

int mp_keyfile_store(const char *path, const void *dev_keys, uint64_t count,
                     int device, void *stream) {
  g_err.clear();
  if (!path || (count && !dev_keys))
    return fail(MP_ERR_INVALID, "keyfile_store: NULL argument");
  MP_CUDA(cudaSetDevice(device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Fd f;
  f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0)
    return io_fail("cannot open for writing", path);
  unsigned char head[kKeyfileHeader];
  std::memcpy(head, kKeyfileMagic, 8);
  for (int i = 0; i < 8; ++i)
    head[8 + i] = static_cast<unsigned char>(count >> (8 * i));
  if (!write_full(f.fd, head, sizeof head))
    return io_fail("write failed", path);
  KeyfileStaging &st = keyfile_staging();
  std::lock_guard<std::mutex> lk(st.mu);
  if (int rc = st.reserve(kKeyfileChunk))
    return rc;
  const uint64_t total = count * 8;
  const char *src = static_cast<const char *>(dev_keys);
  // D2H of chunk k+1 runs while chunk k is written to the file
  uint64_t off = 0, pend_len = 0;
  int pend = -1;
  for (int k = 0; off < total || pend >= 0; ++k) {
    const int i = k & 1;
    uint64_t len = 0;
    if (off < total) {
      len = std::min<uint64_t>(kKeyfileChunk, total - off);
      MP_CUDA(cudaMemcpyAsync(st.buf[i], src + off, len, cudaMemcpyDeviceToHost, s));
      MP_CUDA(cudaEventRecord(st.done[i], s));
    }
    if (pend >= 0) {
      MP_CUDA(cudaEventSynchronize(st.done[pend]));
      if (!write_full(f.fd, st.buf[pend], pend_len))
        return io_fail("write failed", path);
    }
    if (len) {
      pend = i;
      pend_len = len;
      off += len;
    } else {
      pend = -1;
    }
  }
  MP_CUDA(cudaStreamSynchronize(s));
  return MP_OK;
}

// File + file -> file (dataio.cpp:33-98 on both sides of parallel_merge_into,
// as mergebench.cpp:243-259 uses them), with the ingest overlapped with the
// merge: both inputs and the output are mapped and handed to the host
// pipeline of mp_merge_host as pageable spans, so the page-cache reads (the
// copy pool's pageable -> pinned copies), the H2D copies, the chunk merges,
// the D2H copies and the output file's writes (pinned -> mapping) all run
// concurrently, chunk by chunk.  B200 box, 2^27 + 2^27 keys (2 GiB in, 2 GiB
// out, files in the page cache): 1.35-1.40 s per call = the file system's own
// rate for writing the 2 GiB output (a plain write of 2 GiB: 1.36 s); the
// same merge from pageable host vectors takes 0.10 s, device-resident 0.77 ms.
int mp_keyfile_merge(const char *path_a, const char *path_b, const char *path_out,
                     uint64_t *count, int device) {
  g_err.clear();
  if (!path_a || !path_b || !path_out)
    return fail(MP_ERR_INVALID, "keyfile_merge: NULL path");
  KeyfileSpan A, B;
  if (int rc = A.open(path_a))
    return rc;
  if (int rc = B.open(path_b))
    return rc;
  const uint64_t n = A.n + B.n;
  if (same_file(A.f.fd, path_out) || same_file(B.f.fd, path_out))
    return fail(MP_ERR_INVALID, "keyfile_merge: the output file is one of the inputs: %s", path_out);
  Fd out;
  out.fd = ::open(path_out, O_RDWR | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (out.fd < 0)
    return io_fail("cannot open for writing", path_out);
  const size_t out_bytes = kKeyfileHeader + n * 8;
  if (::ftruncate(out.fd, static_cast<off_t>(out_bytes)) != 0)
    return io_fail("cannot size", path_out);
  void *om = ::mmap(nullptr, out_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, out.fd, 0);
  if (om == MAP_FAILED)
    return io_fail("cannot map", path_out);
  unsigned char *head = static_cast<unsigned char *>(om);
  std::memcpy(head, kKeyfileMagic, 8);
  for (int i = 0; i < 8; ++i)
    head[8 + i] = static_cast<unsigned char>(n >> (8 * i));
  int rc = MP_OK;
  if (n)
    rc = mp_merge_host(MP_KEY_I64, A.keys, nullptr, A.n, B.keys, nullptr, B.n,
                       head + kKeyfileHeader, nullptr, device);
  if (::munmap(om, out_bytes) != 0 && rc == MP_OK)
    rc = io_fail("unmap failed", path_out);
  if (rc == MP_OK && count)
    *count = n;
  return rc;
}

// File -> sorted file (read_keys, parallel_merge_sort, write_keys_binary:
// dataio.cpp:33-98, mergebench.cpp:326-332) through mp_sort_host's chunked
// pipeline on the mapped files.
int mp_keyfile_sort(const char *path_in, const char *path_out, uint64_t *count,
                    int device) {
  g_err.clear();
  if (!path_in || !path_out)
    return fail(MP_ERR_INVALID, "keyfile_sort: NULL path");
  KeyfileSpan A;
  if (int rc = A.open(path_in))
    return rc;
  const uint64_t n = A.n;
  if (same_file(A.f.fd, path_out))
    return fail(MP_ERR_INVALID, "keyfile_sort: the output file is the input: %s", path_out);
  Fd out;
  out.fd = ::open(path_out, O_RDWR | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (out.fd < 0)
    return io_fail("cannot open for writing", path_out);
  const size_t out_bytes = kKeyfileHeader + n * 8;
  if (::ftruncate(out.fd, static_cast<off_t>(out_bytes)) != 0)
    return io_fail("cannot size", path_out);
  void *om = ::mmap(nullptr, out_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, out.fd, 0);
  if (om == MAP_FAILED)
    return io_fail("cannot map", path_out);
  unsigned char *head = static_cast<unsigned char *>(om);
  std::memcpy(head, kKeyfileMagic, 8);
  for (int i = 0; i < 8; ++i)
    head[8 + i] = static_cast<unsigned char>(n >> (8 * i));
  int rc = MP_OK;
  if (n)
    rc = mp_sort_host(MP_KEY_I64, A.keys, nullptr, n, head + kKeyfileHeader, nullptr, device);
  if (::munmap(om, out_bytes) != 0 && rc == MP_OK)
    rc = io_fail("unmap failed", path_out);
  if (rc == MP_OK && count)
    *count = n;
  return rc;
}

}  // extern "C"
