// graph_io.cu -- the XKNN graph file (save_graph / load_graph, knn_graph.cpp:276-311) for a
// row-distributed KnnGraph: "XKNN", u32 version 1, u64 num_classes, then per class u32 k and
// its k neighbour ids, all little-endian.  With one k for every class the records have a fixed
// size, so each shard of a ShardLayout reads or writes exactly its own rows [begin, end) at
// their byte offsets (pread/pwrite): no gather of the graph to one host, no communication.
// Host code (POSIX I/O); the rows may live in device memory.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <string>
#include <vector>

#include "layer.cuh"

namespace {

constexpr uint64_t kHeader = 16;  // "XKNN" + u32 version + u64 num_classes

bool little_endian() {
  const uint16_t x = 1;
  uint8_t b;
  std::memcpy(&b, &x, 1);
  return b == 1;
}

void put32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
void put64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint32_t get32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
uint64_t get64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

bool write_all(int fd, const void* buf, size_t n, uint64_t off) {
  const uint8_t* p = static_cast<const uint8_t*>(buf);
  while (n) {
    const ssize_t w = pwrite(fd, p, n, (off_t)off);
    if (w <= 0) return false;
    p += w;
    n -= (size_t)w;
    off += (uint64_t)w;
  }
  return true;
}

// bytes read (short on EOF), -1 on error
ssize_t read_all(int fd, void* buf, size_t n, uint64_t off) {
  uint8_t* p = static_cast<uint8_t*>(buf);
  size_t got = 0;
  while (got < n) {
    const ssize_t r = pread(fd, p + got, n - got, (off_t)(off + got));
    if (r < 0) return -1;
    if (r == 0) break;
    got += (size_t)r;
  }
  return (ssize_t)got;
}

xknn_status_t io_fail(const std::string& msg) {
  return xknn::fail_msg(XKNN_ERR_IO, msg.c_str());
}

}  // namespace

extern "C" {

xknn_status_t xknn_graph_save_rows(const char* path, uint64_t num_classes, uint32_t k,
                                   uint64_t begin, uint64_t end, const uint32_t* rows,
                                   int on_device, int create) {
  if (!path || begin > end || end > num_classes || (end > begin && !rows))
    return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "save_graph: bad arguments");
  Fd f;
  f.fd = open(path, O_WRONLY | (create ? O_CREAT | O_TRUNC : 0), 0644);
  if (f.fd < 0) return io_fail(std::string("cannot open ") + path + " for writing");
  if (create) {
    uint8_t h[kHeader];
    std::memcpy(h, "XKNN", 4);
    put32(h + 4, 1u);  // version
    put64(h + 8, num_classes);
    if (!write_all(f.fd, h, kHeader, 0)) return io_fail(std::string("write failed: ") + path);
  }
  const uint64_t n = end - begin, rec = 4 + 4ull * k;
  if (n == 0) return XKNN_OK;
  // stage the rows on the host in chunks of classes and write the records
  const uint64_t chunk = std::max<uint64_t>(1, (64ull << 20) / (4ull * k + 4));
  std::vector<uint32_t> host;
  std::vector<uint8_t> buf;
  for (uint64_t c0 = 0; c0 < n; c0 += chunk) {
    const uint64_t m = std::min(chunk, n - c0);
    const uint32_t* src = rows + c0 * k;
    if (on_device) {
      host.resize(m * k);
      if (cudaMemcpy(host.data(), src, m * k * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return xknn::fail_msg(XKNN_ERR_CUDA, "save_graph: device copy failed");
      src = host.data();
    }
    buf.resize(m * rec);
    for (uint64_t i = 0; i < m; ++i) {
      uint8_t* r = buf.data() + i * rec;
      put32(r, k);
      if (little_endian()) {
        std::memcpy(r + 4, src + i * k, 4ull * k);
      } else {
        for (uint32_t t = 0; t < k; ++t) put32(r + 4 + 4 * t, src[i * k + t]);
      }
    }
    if (!write_all(f.fd, buf.data(), buf.size(), kHeader + (begin + c0) * rec))
      return io_fail(std::string("write failed: ") + path);
  }
  return XKNN_OK;
}

xknn_status_t xknn_graph_load_rows(const char* path, uint64_t num_classes, uint64_t begin,
                                   uint64_t end, uint32_t* rows, uint64_t capacity, int on_device,
                                   uint32_t* k_out) {
  if (!path || begin > end || end > num_classes)
    return xknn::fail_msg(XKNN_ERR_INVALID_ARGUMENT, "load_graph: bad arguments");
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return io_fail(std::string("cannot open ") + path);
  uint8_t h[kHeader + 4];
  const ssize_t got = read_all(f.fd, h, sizeof h, 0);
  if (got < 4 || std::memcmp(h, "XKNN", 4) != 0)
    return io_fail(std::string(path) + ": not a graph file (bad magic)");
  if (got < 8) return io_fail("graph file truncated");
  if (get32(h + 4) != 1u) return io_fail(std::string(path) + ": unsupported graph version");
  if (got < 16) return io_fail("graph file truncated");
  const uint64_t n = get64(h + 8);
  if (n != num_classes)
    return xknn::fail_msg(XKNN_ERR_SHAPE_MISMATCH,
                          "compress_graph: layout class count disagrees with graph");
  if (n == 0) {
    if (k_out) *k_out = 0;
    return XKNN_OK;
  }
  if (got < (ssize_t)sizeof h) return io_fail("graph file truncated");
  const uint32_t k = get32(h + kHeader);  // class 0's k fixes the record size (load_graph:302)
  if (k_out) *k_out = k;
  if (!rows) return XKNN_OK;
  const uint64_t cnt = end - begin, rec = 4 + 4ull * k;
  if (capacity < cnt * k) return xknn::fail_msg(XKNN_ERR_SHAPE_MISMATCH, "load_graph: rows capacity too small");
  const uint64_t chunk = std::max<uint64_t>(1, (64ull << 20) / rec);
  std::vector<uint8_t> buf;
  std::vector<uint32_t> host;
  for (uint64_t c0 = 0; c0 < cnt; c0 += chunk) {
    const uint64_t m = std::min(chunk, cnt - c0);
    buf.resize(m * rec);
    const ssize_t r = read_all(f.fd, buf.data(), buf.size(), kHeader + (begin + c0) * rec);
    if (r < 0) return io_fail(std::string("read failed: ") + path);
    host.resize(m * k);
    for (uint64_t i = 0; i < m; ++i) {
      const uint8_t* p = buf.data() + i * rec;
      if ((uint64_t)r < i * rec + 4) return io_fail("graph file truncated");
      if (get32(p) != k) return io_fail(std::string(path) + ": per-class k varies; not a full graph");
      if ((uint64_t)r < (i + 1) * rec) return io_fail("graph file truncated");
      for (uint32_t t = 0; t < k; ++t) host[i * k + t] = get32(p + 4 + 4 * t);
    }
    uint32_t* dst = rows + c0 * k;
    if (on_device) {
      if (cudaMemcpy(dst, host.data(), m * k * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return xknn::fail_msg(XKNN_ERR_CUDA, "load_graph: device copy failed");
    } else {
      std::memcpy(dst, host.data(), m * k * 4);
    }
  }
  return XKNN_OK;
}

}  // extern "C"
