// SRTT / SRHT containers (reference io.cpp:1-217, io.hpp:15-33): the step
// before the path for file inputs.
//
// Dense tensor container "SRTT": magic, u32 LE version = 1, u64 LE order,
// u64 LE dims, then binary64 LE values in linearization order (first index
// fastest). Because the last mode is the slowest, a slab [lo, hi) of the last
// mode is ONE contiguous byte range -- a sharded rank reads exactly its slab.
//
// Device reads stream the payload through two pinned staging buffers: the
// file read of chunk i+1 (pread) overlaps the H2D copy of chunk i on the
// handle's stream. Host reads go straight into the caller's buffer.
//
// Hierarchical container "SRHT": the tree as a node list (mode count,
// 0-based modes, child links with 0 = none, all u64 LE), then per node a
// dimension-prefixed binary64 block (leaf: rows, cols, column-major factor;
// internal: three extents, transfer tensor). Validation mirrors
// io.cpp:173-199.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "srtt_b200.h"

// provided by host.cu
cudaStream_t srtt_internal_stream(srtt_handle* h);
int srtt_internal_device(srtt_handle* h);
void srtt_internal_set_error(const std::string& msg);

namespace {

struct IoFail {
  int code;
  std::string msg;
};
[[noreturn]] void io_error(const std::string& msg) { throw IoFail{SRTT_ERR_IO, msg}; }
[[noreturn]] void bad_arg(const std::string& msg) { throw IoFail{SRTT_ERR_INVALID_ARGUMENT, msg}; }
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw IoFail{SRTT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <class F>
int io_guarded(F&& f) {
  try {
    f();
    srtt_internal_set_error("");
    return SRTT_OK;
  } catch (const IoFail& e) {
    srtt_internal_set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    srtt_internal_set_error("host out of memory");
    return SRTT_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    srtt_internal_set_error(e.what());
    return SRTT_ERR_INTERNAL;
  }
}

constexpr char kTensorMagic[4] = {'S', 'R', 'T', 'T'};
constexpr char kHtMagic[4] = {'S', 'R', 'H', 'T'};
constexpr uint32_t kVersion = 1;

struct File {
  int fd = -1;
  ~File() {
    if (fd >= 0) close(fd);
  }
};

void open_read(File& f, const char* path) {
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) io_error(std::string("cannot open for reading: ") + path);
}

void open_write(File& f, const char* path) {
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) io_error(std::string("cannot open for writing: ") + path);
}

// Exactly `n` bytes at `off`, else "unexpected end of stream".
void read_at(int fd, void* dst, size_t n, int64_t off) {
  char* p = static_cast<char*>(dst);
  while (n > 0) {
    const ssize_t r = pread(fd, p, n, off);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) io_error("unexpected end of stream");
    p += r;
    n -= (size_t)r;
    off += r;
  }
}

void write_all(int fd, const void* src, size_t n, const char* what) {
  const char* p = static_cast<const char*>(src);
  while (n > 0) {
    const ssize_t r = write(fd, p, n);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) io_error(what);
    p += r;
    n -= (size_t)r;
  }
}

// The host is little-endian (x86-64 / aarch64 Linux), so the payload is the
// in-memory byte image; integers are assembled byte by byte regardless.
uint64_t le64(const unsigned char* b) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
uint32_t le32(const unsigned char* b) {
  uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
void put64(std::vector<unsigned char>& o, uint64_t v) {
  for (int i = 0; i < 8; ++i) o.push_back((unsigned char)((v >> (8 * i)) & 0xFF));
}
void put32(std::vector<unsigned char>& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((unsigned char)((v >> (8 * i)) & 0xFF));
}

// Sequential reader over a file descriptor (small header fields).
struct Cursor {
  int fd;
  int64_t off = 0;
  uint64_t u64() {
    unsigned char b[8];
    read_at(fd, b, 8, off);
    off += 8;
    return le64(b);
  }
  void magic(const char (&m)[4], const char* what) {
    unsigned char b[8];
    read_at(fd, b, 4, off);
    if (std::memcmp(b, m, 4) != 0) io_error(std::string(what) + ": bad magic bytes");
    read_at(fd, b + 4, 4, off + 4);
    off += 8;
    const uint32_t v = le32(b + 4);
    if (v != kVersion) io_error(std::string(what) + ": unsupported format version " + std::to_string(v));
  }
};

struct TensorHeader {
  std::vector<int64_t> dims;
  int64_t data_offset = 0;
  int64_t count = 1;
};

TensorHeader read_tensor_header(int fd) {
  Cursor c{fd};
  c.magic(kTensorMagic, "tensor file");
  const uint64_t order = c.u64();
  if (order == 0 || order > 64) io_error("tensor file: implausible order");
  TensorHeader h;
  for (uint64_t k = 0; k < order; ++k) {
    const uint64_t n = c.u64();
    if (n == 0 || n > (1ull << 40)) io_error("tensor file: implausible dimension");
    h.dims.push_back((int64_t)n);
    h.count *= (int64_t)n;
  }
  h.data_offset = c.off;
  return h;
}

// Pinned double-buffered staging: pread chunk i+1 while chunk i copies.
void read_to_device(srtt_handle* h, int fd, int64_t off, int64_t bytes, char* dst) {
  const size_t chunk = (size_t)std::min<int64_t>(bytes, 64ll << 20);
  cudaStream_t s = srtt_internal_stream(h);
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto cleanup = [&] {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventDestroy(done[i]);
      if (stage[i]) cudaFreeHost(stage[i]);
    }
  };
  try {
    for (int i = 0; i < 2; ++i) {
      ck(cudaHostAlloc(&stage[i], chunk, cudaHostAllocDefault), "cudaHostAlloc");
      ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    int64_t pos = 0;
    for (int i = 0; pos < bytes; ++i) {
      const int b = i & 1;
      const size_t n = (size_t)std::min<int64_t>((int64_t)chunk, bytes - pos);
      ck(cudaEventSynchronize(done[b]), "cudaEventSynchronize");  // buffer b's previous copy finished
      read_at(fd, stage[b], n, off + pos);
      ck(cudaMemcpyAsync(dst + pos, stage[b], n, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
      ck(cudaEventRecord(done[b], s), "cudaEventRecord");
      pos += (int64_t)n;
    }
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  } catch (...) {
    cudaStreamSynchronize(s);
    cleanup();
    throw;
  }
  cleanup();
}

// Device -> file through the same staging scheme (D2H of chunk i+1 overlaps
// the write of chunk i).
void write_from_device(srtt_handle* h, int fd, const char* src, int64_t bytes) {
  const size_t chunk = (size_t)std::min<int64_t>(std::max<int64_t>(bytes, 1), 64ll << 20);
  cudaStream_t s = srtt_internal_stream(h);
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  auto cleanup = [&] {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventDestroy(done[i]);
      if (stage[i]) cudaFreeHost(stage[i]);
    }
  };
  try {
    for (int i = 0; i < 2; ++i) {
      ck(cudaHostAlloc(&stage[i], chunk, cudaHostAllocDefault), "cudaHostAlloc");
      ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    const int64_t nchunks = (bytes + (int64_t)chunk - 1) / (int64_t)chunk;
    auto issue = [&](int64_t i) {
      const size_t n = (size_t)std::min<int64_t>((int64_t)chunk, bytes - i * (int64_t)chunk);
      ck(cudaMemcpyAsync(stage[i & 1], src + i * (int64_t)chunk, n, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
      ck(cudaEventRecord(done[i & 1], s), "cudaEventRecord");
    };
    if (nchunks > 0) issue(0);
    for (int64_t i = 0; i < nchunks; ++i) {
      if (i + 1 < nchunks) issue(i + 1);
      ck(cudaEventSynchronize(done[i & 1]), "cudaEventSynchronize");
      const size_t n = (size_t)std::min<int64_t>((int64_t)chunk, bytes - i * (int64_t)chunk);
      write_all(fd, stage[i & 1], n, "tensor write failed");
    }
  } catch (...) {
    cudaStreamSynchronize(s);
    cleanup();
    throw;
  }
  cleanup();
}

struct DeviceGuardIo {
  int prev = -1;
  explicit DeviceGuardIo(srtt_handle* h) {
    if (!h) return;
    cudaGetDevice(&prev);
    ck(cudaSetDevice(srtt_internal_device(h)), "cudaSetDevice");
  }
  ~DeviceGuardIo() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int srtt_tensor_file_info(const char* path, int32_t* order, int64_t* dims, int32_t dims_capacity,
                          int64_t* data_offset) {
  return io_guarded([&] {
    if (!path) bad_arg("read_tensor: null path");
    File f;
    open_read(f, path);
    const TensorHeader th = read_tensor_header(f.fd);
    if (order) *order = (int32_t)th.dims.size();
    if (dims) {
      if ((int)th.dims.size() > dims_capacity) bad_arg("read_tensor: dims buffer too small");
      std::copy(th.dims.begin(), th.dims.end(), dims);
    }
    if (data_offset) *data_offset = th.data_offset;
  });
}

int srtt_read_tensor(srtt_handle* h, const char* path, int64_t slab_lo, int64_t slab_hi, double* out,
                     int32_t out_on_device, int64_t out_capacity) {
  return io_guarded([&] {
    if (!path) bad_arg("read_tensor: null path");
    if (out_on_device && !h) bad_arg("read_tensor: device output needs a handle");
    File f;
    open_read(f, path);
    const TensorHeader th = read_tensor_header(f.fd);
    const int64_t last = th.dims.back();
    if (slab_lo < 0 && slab_hi < 0) {
      slab_lo = 0;
      slab_hi = last;
    }
    if (slab_lo < 0 || slab_hi > last || slab_lo >= slab_hi) bad_arg("read_tensor: slab out of range");
    const int64_t plane = th.count / last;  // entries per index of the last mode
    const int64_t count = plane * (slab_hi - slab_lo);
    if (count > out_capacity) bad_arg("read_tensor: output buffer too small");
    // the whole payload must be present (a truncated file is corrupt even
    // when the requested slab is readable)
    struct stat st;
    if (fstat(f.fd, &st) != 0) io_error("tensor file: cannot stat");
    if ((int64_t)st.st_size < th.data_offset + 8 * th.count) io_error("unexpected end of stream");
    const int64_t off = th.data_offset + 8 * plane * slab_lo;
    if (out_on_device) {
      DeviceGuardIo g(h);
      read_to_device(h, f.fd, off, 8 * count, reinterpret_cast<char*>(out));
    } else {
      read_at(f.fd, out, (size_t)(8 * count), off);
    }
  });
}

int srtt_write_tensor(srtt_handle* h, const char* path, int32_t d, const int64_t* dims, const double* x,
                      int32_t x_on_device) {
  return io_guarded([&] {
    if (!path) bad_arg("write_tensor: null path");
    if (d < 1 || d > 64) bad_arg("write_tensor: order must be in [1, 64]");
    if (x_on_device && !h) bad_arg("write_tensor: device input needs a handle");
    int64_t count = 1;
    std::vector<unsigned char> head(kTensorMagic, kTensorMagic + 4);
    put32(head, kVersion);
    put64(head, (uint64_t)d);
    for (int k = 0; k < d; ++k) {
      if (dims[k] < 1) bad_arg("Shape: dimensions must be >= 1");
      put64(head, (uint64_t)dims[k]);
      count *= dims[k];
    }
    File f;
    open_write(f, path);
    write_all(f.fd, head.data(), head.size(), "tensor write failed");
    if (x_on_device) {
      DeviceGuardIo g(h);
      write_from_device(h, f.fd, reinterpret_cast<const char*>(x), 8 * count);
    } else {
      write_all(f.fd, x, (size_t)(8 * count), "tensor write failed");
    }
  });
}

int srtt_write_htucker(const char* path, int32_t d, const int64_t* dims, const srtt_tree* tree,
                       const int64_t* ranks, const double* const* leaf_factors, const double* const* transfers) {
  return io_guarded([&] {
    if (!path || !tree || !dims || !ranks) bad_arg("write_htucker: null argument");
    const int nn = tree->num_nodes;
    if (d < 2 || nn < 3) bad_arg("write_htucker: implausible tree size");
    std::vector<unsigned char> o(kHtMagic, kHtMagic + 4);
    put32(o, kVersion);
    put64(o, (uint64_t)d);
    put64(o, (uint64_t)nn);
    for (int i = 0; i < nn; ++i) {
      const int b = tree->mode_begin[i], e = tree->mode_begin[i + 1];
      put64(o, (uint64_t)(e - b));
      for (int k = b; k < e; ++k) put64(o, (uint64_t)tree->modes[k]);
      const bool leaf = tree->left[i] < 0;
      put64(o, leaf ? 0 : (uint64_t)tree->left[i] + 1);
      put64(o, leaf ? 0 : (uint64_t)tree->right[i] + 1);
    }
    File f;
    open_write(f, path);
    write_all(f.fd, o.data(), o.size(), "hierarchical container write failed");
    for (int i = 0; i < nn; ++i) {
      o.clear();
      const double* src;
      int64_t count;
      if (tree->left[i] < 0) {
        const int m = tree->modes[tree->mode_begin[i]];
        put64(o, (uint64_t)dims[m]);
        put64(o, (uint64_t)ranks[i]);
        src = leaf_factors[m];
        count = dims[m] * ranks[i];
      } else {
        const int64_t rs = i == 0 ? 1 : ranks[i], rl = ranks[tree->left[i]], rr = ranks[tree->right[i]];
        put64(o, (uint64_t)rs);
        put64(o, (uint64_t)rl);
        put64(o, (uint64_t)rr);
        src = transfers[i];
        count = rs * rl * rr;
      }
      if (!src) bad_arg("write_htucker: missing block for node " + std::to_string(i));
      write_all(f.fd, o.data(), o.size(), "hierarchical container write failed");
      write_all(f.fd, src, (size_t)(8 * count), "hierarchical container write failed");
    }
  });
}

// Parses an SRHT file. Pass NULL buffers to query sizes first: *order,
// *num_nodes, *num_modes (total mode entries) and the per-node ranks /
// leaf extents; then call again with mode_begin (num_nodes + 1), modes,
// left, right (num_nodes), ranks (num_nodes), dims (order) and the block
// pointers (leaf_factors by mode, transfers by node id; host memory).
int srtt_read_htucker(const char* path, int32_t* order, int32_t* num_nodes, int32_t* num_modes,
                      int32_t* mode_begin, int32_t* modes, int32_t* left, int32_t* right, int64_t* ranks,
                      int64_t* dims, double* const* leaf_factors, double* const* transfers) {
  return io_guarded([&] {
    if (!path) bad_arg("read_htucker: null path");
    File f;
    open_read(f, path);
    Cursor c{f.fd};
    c.magic(kHtMagic, "hierarchical container");
    const uint64_t d = c.u64();
    const uint64_t nn = c.u64();
    if (d < 2 || nn < 3 || nn > 4 * d) io_error("hierarchical container: implausible tree size");
    std::vector<std::vector<int64_t>> nm(nn);
    std::vector<int64_t> l(nn), r(nn), parent(nn, -1);
    for (uint64_t i = 0; i < nn; ++i) {
      const uint64_t k = c.u64();
      if (k == 0 || k > d) io_error("hierarchical container: bad mode set");
      for (uint64_t j = 0; j < k; ++j) {
        const uint64_t m = c.u64();
        if (m >= d) io_error("hierarchical container: bad mode set");
        nm[i].push_back((int64_t)m);
      }
      const uint64_t a = c.u64(), b = c.u64();
      l[i] = a == 0 ? -1 : (int64_t)a - 1;
      r[i] = b == 0 ? -1 : (int64_t)b - 1;
    }
    for (uint64_t i = 0; i < nn; ++i) {
      if (l[i] < 0) continue;
      if (l[i] >= (int64_t)nn || r[i] >= (int64_t)nn || r[i] < 0)
        io_error("hierarchical container: child link out of range");
      parent[l[i]] = (int64_t)i;
      parent[r[i]] = (int64_t)i;
    }
    for (uint64_t i = 1; i < nn; ++i) {
      if (parent[i] < 0) io_error("hierarchical container: disconnected node");
      if (parent[i] >= (int64_t)i) io_error("hierarchical container: nodes must come after their parent");
    }
    int32_t total = 0;
    for (auto& v : nm) total += (int32_t)v.size();
    if (order) *order = (int32_t)d;
    if (num_nodes) *num_nodes = (int32_t)nn;
    if (num_modes) *num_modes = total;
    if (mode_begin) {
      int32_t p = 0;
      for (uint64_t i = 0; i < nn; ++i) {
        mode_begin[i] = p;
        for (int64_t m : nm[i]) modes[p++] = (int32_t)m;
        left[i] = (int32_t)l[i];
        right[i] = (int32_t)r[i];
      }
      mode_begin[nn] = p;
    }
    // blocks: extents always parsed (ranks / dims), values copied when asked
    for (uint64_t i = 0; i < nn; ++i) {
      if (l[i] < 0) {
        const uint64_t rows = c.u64(), cols = c.u64();
        if (rows < 1 || cols < 1) io_error("hierarchical container: bad factor extents");
        if (ranks) ranks[i] = (int64_t)cols;
        if (dims) dims[nm[i][0]] = (int64_t)rows;
        const int64_t bytes = 8 * (int64_t)(rows * cols);
        if (leaf_factors && leaf_factors[nm[i][0]]) read_at(f.fd, leaf_factors[nm[i][0]], (size_t)bytes, c.off);
        c.off += bytes;
      } else {
        const uint64_t a = c.u64(), b = c.u64(), e = c.u64();
        if (a < 1 || b < 1 || e < 1) io_error("hierarchical container: bad transfer extents");
        if (ranks) ranks[i] = (int64_t)a;
        const int64_t bytes = 8 * (int64_t)(a * b * e);
        if (transfers && transfers[i]) read_at(f.fd, transfers[i], (size_t)bytes, c.off);
        c.off += bytes;
      }
    }
    // a truncated payload is corrupt even when only the header was asked for
    struct stat st;
    if (fstat(f.fd, &st) != 0 || (int64_t)st.st_size < c.off) io_error("unexpected end of stream");
  });
}

}  // extern "C"
