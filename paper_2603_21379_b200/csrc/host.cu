// Host runtime of the B200 engine: handle (device, streams, events,
// grow-only workspace arena, pinned parameter staging), planners (TSQR tree
// per sketch target; core-pass work decomposition) and the C-ABI entry
// points of include/srtt_b200.h. Validation order and messages follow the
// reference (tucker.hpp:184-197, htucker.hpp:217-233, sketch.hpp:77-78,
// unfolding.hpp:46-47/86-87) so callers see the same errors.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_rng.hpp"
#include "srtt_b200.h"
#include "srtt_params.h"

// ---- kernel launchers (k_*.cu) ---------------------------------------------
size_t srtt_sketch_smem_bytes(int cmax);
cudaError_t srtt_launch_sketch(const SketchTarget*, int, int64_t, int, cudaStream_t);
cudaError_t srtt_launch_sketch_reduce(const SketchTarget*, int, int64_t, cudaStream_t);
cudaError_t srtt_launch_omega(const SketchTarget*, int, int64_t, cudaStream_t);
cudaError_t srtt_launch_sketch_contig(const SketchTarget*, int, int64_t, int, int, cudaStream_t);
cudaError_t srtt_launch_scatter_block(const double*, double*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                                      int64_t, cudaStream_t);
size_t srtt_basis_top_smem(int m, int c, int r);
size_t srtt_basis_level_smem(int mb, int c);
cudaError_t srtt_launch_basis_top(int, const BasisTarget*, const int*, int, size_t, cudaStream_t);
int srtt_basis_top_variant(int c);
size_t srtt_basis_small_smem(int m, int c, int r);
cudaError_t srtt_launch_basis_small(int, const BasisTarget*, const int*, int, size_t, cudaStream_t);
int srtt_basis_small_variant(int m, int c);
constexpr int kSmallVariants = 5;
int srtt_wtree_cp(int c);
int srtt_wtree_chunk(int cp);
int srtt_wtree_factor_threads();
size_t srtt_wtree_top_smem(int n0, int c, bool pad);
int64_t srtt_wtree_persist_doubles(int rows, int c);
size_t srtt_wtree_factor_smem(int rows, int c);
size_t srtt_wtree_apply_smem(int rows, int c);
cudaError_t srtt_launch_wtree_top(int, int, const BasisTarget*, const int*, int, size_t, cudaStream_t);
cudaError_t srtt_launch_wtree_factor(int, const BasisTarget*, const int2*, int, size_t, cudaStream_t);
cudaError_t srtt_launch_wtree_apply(int, const BasisTarget*, const int2*, int, size_t, cudaStream_t);
int srtt_wide_block_rows();
size_t srtt_wide_top_smem(int m, int c, int r, bool pad);
size_t srtt_wide_level_smem(int mb, int c);
cudaError_t srtt_launch_wide_top(const BasisTarget*, const int*, int, size_t, cudaStream_t);
cudaError_t srtt_launch_wide_factor(const BasisTarget*, const int2*, int, int, size_t, cudaStream_t);
cudaError_t srtt_launch_wide_apply(const BasisTarget*, const int2*, int, int, size_t, cudaStream_t);
size_t srtt_basis_generic_smem(int c, int r);
int64_t srtt_basis_generic_doubles(int64_t n, int c);
cudaError_t srtt_launch_basis_generic(const BasisTarget*, const int*, int, size_t, cudaStream_t);
cudaError_t srtt_launch_tsqr_factor(const BasisTarget*, const int2*, int, int, size_t, cudaStream_t);
cudaError_t srtt_launch_tsqr_apply(const BasisTarget*, const int2*, int, int, size_t, cudaStream_t);
cudaError_t srtt_launch_pad(const BasisTarget*, int, double*, int64_t, cudaStream_t);
int srtt_core_threads();
size_t srtt_core_smem_bytes(const CoreParams& P);
int srtt_core_occupancy(const CoreParams& P);
int srtt_core_max_stages(const CoreParams& P, size_t budget);
cudaError_t srtt_launch_core(const CUtensorMap*, const CoreParams&, int, cudaStream_t);
cudaError_t srtt_launch_prep(const double*, int64_t, int, int, int, int, double*, cudaStream_t);
cudaError_t srtt_launch_transpose(const double*, int64_t, int, double*, cudaStream_t);
cudaError_t srtt_launch_prep_all(const CoreParams&, CoreItem*, const double*, int64_t, int, int, int, int, double*,
                                 int, const double* const*, double* const*, const int64_t*, const int*, cudaStream_t);
cudaError_t srtt_launch_ttm(const TtmParams&, cudaStream_t);
int srtt_residual_grid(int sms, int64_t nA, int K);
int srtt_residual_tile_rows(int64_t nA);
cudaError_t srtt_launch_residual(const CUtensorMap*, const ResidualParams&, int, double*, cudaStream_t);
cudaError_t srtt_launch_pad_rows(const double*, int64_t, int64_t, int64_t, double*, cudaStream_t);
int srtt_residual_tile_cols(int64_t nA, int K);
cudaError_t srtt_launch_diff_norm(const double*, const double*, int64_t, int, double*, double*, cudaStream_t);
cudaError_t srtt_launch_kron_rows(const KronParams&, cudaStream_t);
cudaError_t srtt_launch_mat_transpose(const double*, int64_t, int64_t, double*, cudaStream_t);

typedef struct TransferTarget {
  const double* us;
  const double* ul;
  const double* ur;
  double* b;
  int64_t nl, nr;
  int32_t rs, rl, rr;
  int32_t cta_begin;
} TransferTarget;
typedef struct GatherParams {
  const double* x;
  const int64_t* cols;
  double* y;
  int64_t rows, w;
  int32_t nrow_modes, ncol_modes;
  int64_t row_dim[SRTT_MAX_ORDER], row_stride[SRTT_MAX_ORDER];
  int64_t col_dim[SRTT_MAX_ORDER], col_stride[SRTT_MAX_ORDER];
} GatherParams;
cudaError_t srtt_launch_transfer(const TransferTarget*, int, int, int, int, cudaStream_t);
cudaError_t srtt_launch_gather(const GatherParams&, cudaStream_t);

namespace {

// ---- errors -----------------------------------------------------------------
thread_local std::string g_last_error;

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }
[[noreturn]] void invalid(const std::string& msg) { fail(SRTT_ERR_INVALID_ARGUMENT, msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  fail(e == cudaErrorMemoryAllocation ? SRTT_ERR_OUT_OF_MEMORY : SRTT_ERR_CUDA,
       std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// During stream capture an event must be recorded as an "external" node to
// exist (and time) in the replayed graph; outside capture, a plain record.
void record_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive)
    CK(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  else
    CK(cudaEventRecord(e, s));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return SRTT_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return SRTT_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return SRTT_ERR_OUT_OF_RANGE;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return SRTT_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SRTT_ERR_INTERNAL;
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---- buffers ----------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool ensure(size_t bytes) {  // returns true when reallocated
    if (bytes <= cap) return false;
    size_t want = std::max(bytes, cap + cap / 2);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      e = cudaMalloc(&p, bytes);
      want = bytes;
    }
    CK(e);
    cap = want;
    return true;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    const size_t want = std::max(bytes, cap * 2);
    CK(cudaMallocHost(&p, want));
    cap = want;
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

// Two-pass layout helper: take() records aligned offsets; resolve after the
// backing buffer is large enough.
struct Layout {
  size_t off = 0;
  size_t take(size_t bytes, size_t align = 256) {
    off = (off + align - 1) / align * align;
    const size_t o = off;
    off += bytes;
    return o;
  }
};

// ---- tensor map encoder (driver entry point; no -lcuda needed) ------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encoder() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(SRTT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

void encode_tmap(CUtensorMap* map, const double* x, int64_t n0, int64_t Q, int W) {
  cuuint64_t gdim[2] = {(cuuint64_t)n0, (cuuint64_t)Q};
  cuuint64_t gstride[1] = {(cuuint64_t)n0 * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)W};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), gdim,
                             gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SRTT_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// Plain (unswizzled) 2-D fp64 map: d0 fastest, row pitch ld0 elements.
void encode_tmap_plain(CUtensorMap* map, const double* p, int64_t d0, int64_t d1, int64_t ld0, int box0, int box1) {
  cuuint64_t gdim[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
  cuuint64_t gstride[1] = {(cuuint64_t)ld0 * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), gdim, gstride, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SRTT_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

int64_t prod(const std::vector<int64_t>& v, int lo = 0, int hi = 1 << 30) {
  int64_t p = 1;
  const int e = std::min<int>(hi, (int)v.size());
  for (int i = lo; i < e; ++i) p *= v[static_cast<size_t>(i)];
  return p;
}

}  // namespace

// ---- handle -----------------------------------------------------------------
constexpr int kInfoInts = 4096;  // 4 ints per target + flags

struct srtt_handle {
  int device = 0;
  int sms = 148;
  int use_graphs = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t side = nullptr;     // second stream of the H-Tucker DAG
  cudaEvent_t fj[4] = {};          // fork/join events (timing disabled)
  cudaEvent_t ev[8] = {};
  cudaEvent_t kev[8] = {};  // per-kernel pairs: [2i] start, [2i+1] end
  DevBuf xbuf;     // device copy of host inputs
  DevBuf ws;       // workspace arena
  DevBuf rb[6];    // reconstruction / error buffers (At, Ct ping-pong, staging), reused across calls
  DevBuf comp[6];  // scratch of the synchronous component / shard-phase calls, reused across calls
  // Double-buffered parameter blobs (pinned host + device copy): a call
  // may return before its graph ran (device outputs, no report), so the
  // next call writes the other set; a set is reused only after the call
  // that last used it completed (event).
  struct ParamSet {
    DevBuf d;
    HostBuf hst;
    // per-target info (achieved rank, nrank, sweeps) + status flags: device
    // memory written by the kernels of the call that owns this set, cleared
    // in-stream at the start of that call and copied to `hinfo_buf` at its
    // end (never touched by the host while a call may still run on it)
    DevBuf info;
    HostBuf hinfo_buf;
    cudaEvent_t done = nullptr;
    bool recorded = false;
    int32_t* dinfo() { return reinterpret_cast<int32_t*>(info.p); }
    int32_t* hinfo() { return reinterpret_cast<int32_t*>(hinfo_buf.p); }
  };
  ParamSet psets[2];
  int cur = 0;
  ParamSet& pset() { return psets[cur]; }
  DevBuf ones;
  int64_t launches = 0;
  // timing events (stage marks, per-kernel pairs) are recorded only for
  // calls that return a report: they are graph nodes between the kernels
  bool timing = true;
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
  };
  std::map<std::string, Graph> graphs;
  // Per-signature prepared Tucker calls: the seed-independent parameter
  // blob image and where the seed-dependent fields live inside it.
  struct Prepared {
    std::vector<unsigned char> image;
    std::vector<size_t> off_cols;
    size_t off_sk = 0, off_bt = 0;
    std::string graph_key;
    const void *ws = nullptr, *dp = nullptr, *hp = nullptr;
    std::vector<const double*> udev;  // device factors (workspace or user buffers)
    const double* d_core = nullptr;
  };
  std::map<std::string, Prepared> prepared;
  // multi-GPU: the NCCL communicator this handle owns (srtt_comm_init);
  // opaque here, see shard.cuh
  void* comm = nullptr;
  int world = 1, rank = 0;
  ~srtt_handle() {
    for (auto& g : graphs)
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Parameter blob: host pinned staging, uploaded with one copy.
struct Blob {
  Layout lay;
  std::vector<std::pair<size_t, std::vector<unsigned char>>> items;
  size_t add(const void* src, size_t bytes) {
    const size_t o = lay.take(bytes, 64);
    items.emplace_back(o, std::vector<unsigned char>((const unsigned char*)src,
                                                       (const unsigned char*)src + bytes));
    return o;
  }
  size_t reserve(size_t bytes) { return lay.take(bytes, 64); }
};

// ---- basis (K2) planning ------------------------------------------------------
constexpr size_t kSmemBudget = 200 * 1024;
constexpr size_t kCoreSmem = 232448 - 256;  // opt-in max dynamic smem per block on sm_100

int top_max_rows(int c, int r) {
  int lo = 1, hi = 1 << 20;
  if (srtt_basis_top_smem(1, c, r) > kSmemBudget) return 0;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (srtt_basis_top_smem(mid, c, r) <= kSmemBudget) lo = mid; else hi = mid - 1;
  }
  return lo;
}

int level_block_rows(int c) {
  int m = 1024;
  while (m > 2 * c && srtt_basis_level_smem(m, c) > kSmemBudget) m -= 32;
  return m;
}

struct BasisPlan {
  int64_t n;
  int c, r;
  int kind;  // 0: shared-memory QR kernels; 1: register-tree path (c <= 32)
  int nlevels;
  int64_t lv_n[SRTT_MAX_QR_LEVELS + 1];
  int lv_nblk[SRTT_MAX_QR_LEVELS + 1];
  int lv_blk[SRTT_MAX_QR_LEVELS + 1];
};

// Register-tree path (k_basis.cu): sketches with c <= 32 columns whose top
// fits one CTA. Single-CTA targets keep their level-0 reflectors in shared
// memory; taller ones are cut into CTAs of rpc rows (a multiple of the warp
// block, 4 warps per CTA) whose R factors one top CTA combines.
// SRTT_BASIS_SMEMQR=1 (development) forces the shared-memory kernels.
constexpr size_t kWtreeSmemBudget = 220 * 1024;

bool plan_basis_wtree(BasisPlan& b) {
  static const bool off = [] {
    const char* e = std::getenv("SRTT_BASIS_SMEMQR");
    return e && *e == '1';
  }();
  const int cp = srtt_wtree_cp(b.c);
  if (off || cp == 0 || b.n < 1) return false;
  b.kind = 1;
  if (b.n <= 4096 && srtt_wtree_top_smem((int)b.n, b.c, true) <= kWtreeSmemBudget) {
    b.nlevels = 0;
    b.lv_n[0] = b.n;
    b.lv_nblk[0] = 1;
    b.lv_blk[0] = (int)b.n;
    return true;
  }
  const int chunk = srtt_wtree_chunk(cp);
  const int warps = srtt_wtree_factor_threads() / 32;
  for (int bpw = 1; bpw <= 16; ++bpw) {
    const int64_t rpc = (int64_t)warps * chunk * bpw;
    const int64_t ncta = (b.n + rpc - 1) / rpc;
    const int64_t rem = b.n - (ncta - 1) * rpc;
    const int64_t top = (ncta - 1) * b.c + std::min<int64_t>(rem, b.c);
    if (top > 4096 || srtt_wtree_top_smem((int)top, b.c, false) > kWtreeSmemBudget) continue;
    if (srtt_wtree_apply_smem((int)rpc, b.c) > kWtreeSmemBudget) break;
    b.nlevels = 1;
    b.lv_n[0] = b.n;
    b.lv_nblk[0] = (int)ncta;
    b.lv_blk[0] = (int)rpc;
    b.lv_n[1] = top;
    b.lv_nblk[1] = 1;
    b.lv_blk[1] = (int)top;
    return true;
  }
  b.kind = 0;
  return false;
}

// Wide register path (k_basis.cu): 32 < c <= 64, 8-warp teams on 256-row
// blocks, the level structure of the shared-memory path (one launch per
// level, stacked R of c rows per block).
bool plan_basis_wide(BasisPlan& b) {
  static const bool off = [] {
    const char* e = std::getenv("SRTT_BASIS_SMEMQR");
    return e && *e == '1';
  }();
  if (off || b.c <= 32 || b.c > 64 || b.n < 1) return false;
  const int blk = srtt_wide_block_rows();
  int tmax = blk;
  while (tmax > b.c && srtt_wide_top_smem(tmax, b.c, b.r, false) > kWtreeSmemBudget) tmax -= 32;
  if (tmax < b.c || srtt_wide_top_smem(tmax, b.c, b.r, false) > kWtreeSmemBudget) return false;
  if (srtt_wide_level_smem(blk, b.c) > kWtreeSmemBudget) return false;
  b.kind = 2;
  if (b.n <= tmax && srtt_wide_top_smem((int)b.n, b.c, b.r, true) <= kWtreeSmemBudget) {
    b.nlevels = 0;
    b.lv_n[0] = b.n;
    b.lv_nblk[0] = 1;
    b.lv_blk[0] = (int)b.n;
    return true;
  }
  int64_t nl = b.n;
  int l = 0;
  while (nl > tmax || l == 0) {
    if (l >= SRTT_MAX_QR_LEVELS) { b.kind = 0; return false; }
    const int nblk = (int)((nl + blk - 1) / blk);
    b.lv_n[l] = nl;
    b.lv_nblk[l] = nblk;
    b.lv_blk[l] = blk;
    nl = (int64_t)nblk * b.c;
    ++l;
  }
  b.lv_n[l] = nl;
  b.lv_nblk[l] = 1;
  b.lv_blk[l] = (int)nl;
  b.nlevels = l;
  return true;
}

BasisPlan plan_basis(int64_t n, int c, int r) {
  BasisPlan b{};
  b.n = n;
  b.c = c;
  b.r = r;
  if (plan_basis_wtree(b)) return b;
  if (plan_basis_wide(b)) return b;
  if (c > 64) {
    // generic kernel (k_basis.cu): one CTA per target on global memory
    if (c > SRTT_MAX_SKETCH_COLS) invalid("range_basis_of_sketch: sketch too wide for the B200 basis kernels");
    b.kind = 3;
    b.nlevels = 0;
    b.lv_n[0] = n;
    b.lv_nblk[0] = 1;
    b.lv_blk[0] = (int)std::min<int64_t>(n, INT32_MAX);
    return b;
  }
  int tmax = top_max_rows(c, r);
  int blk = level_block_rows(c);
  if (tmax < c) invalid("range_basis_of_sketch: sketch too wide for the B200 basis kernel");
  if (n > tmax && c <= 32) {
    // Tall sketch: the TSQR step is a latency chain whose cost grows with
    // the rows one CTA factors, not with the CTA count. Short row blocks
    // (about 64 per level, >= 128 rows) and a short top (<= 4c rows) give
    // more, cheaper levels (C4 level-1 nodes: 302 -> 286 us of TSQR; wide
    // sketches, c > 32, keep the large blocks: their top dominates).
    // development aid: SRTT_TSQR="blk,top"
    int fb = 0, ft = 0;
    if (const char* e = std::getenv("SRTT_TSQR")) std::sscanf(e, "%d,%d", &fb, &ft);
    const int64_t want = ((n + 63) / 64 + 31) / 32 * 32;
    blk = fb ? fb : (int)std::min<int64_t>(blk, std::max<int64_t>(std::max(128, 2 * c), want));
    tmax = ft ? std::min(ft, tmax) : std::min(tmax, std::max(4 * c, 64));
  }
  int64_t nl = n;
  int l = 0;
  while (nl > tmax) {
    if (l >= SRTT_MAX_QR_LEVELS) invalid("range_basis_of_sketch: sketch too tall");
    const int nblk = (int)((nl + blk - 1) / blk);
    const int64_t nn = (int64_t)nblk * c;
    if (nn >= nl) invalid("range_basis_of_sketch: TSQR cannot shrink this sketch");
    b.lv_n[l] = nl;
    b.lv_nblk[l] = nblk;
    b.lv_blk[l] = blk;
    nl = nn;
    ++l;
  }
  b.lv_n[l] = nl;
  b.lv_nblk[l] = 1;
  b.lv_blk[l] = (int)nl;
  b.nlevels = l;
  return b;
}

struct BasisBuffers {  // offsets into the workspace
  size_t a[SRTT_MAX_QR_LEVELS + 1], tau[SRTT_MAX_QR_LEVELS + 1], y[SRTT_MAX_QR_LEVELS + 1];
  size_t info, sv, pad;
  size_t vup;
  int64_t vup_stride;
};

// z (level-0 matrix) and u (final basis) are supplied by the caller.
BasisBuffers layout_basis(Layout& L, const BasisPlan& p) {
  BasisBuffers B{};
  for (int l = 0; l <= p.nlevels; ++l) {
    B.a[l] = l == 0 ? SIZE_MAX : L.take(sizeof(double) * p.lv_n[l] * p.c);
    B.tau[l] = L.take(sizeof(double) * (size_t)p.lv_nblk[l] * p.c);
    B.y[l] = l == 0 ? SIZE_MAX : L.take(sizeof(double) * p.lv_n[l] * p.r);
  }
  B.info = L.take(4 * sizeof(int32_t));
  B.sv = L.take(sizeof(double) * p.c);
  B.pad = 0;
  if (p.kind == 1 && p.nlevels == 1) {
    B.vup_stride = srtt_wtree_persist_doubles(p.lv_blk[0], p.c);
    B.vup = L.take(sizeof(double) * (size_t)B.vup_stride * p.lv_nblk[0]);
  }
  if (p.kind == 3) {
    B.vup_stride = srtt_basis_generic_doubles(p.n, p.c);
    B.vup = L.take(sizeof(double) * (size_t)B.vup_stride);
  }
  return B;
}

BasisTarget fill_basis(const BasisPlan& p, const BasisBuffers& B, char* ws, double* z, double* u,
                       uint64_t state0, uint64_t draw_offset, int64_t normal_base, int32_t* info = nullptr) {
  BasisTarget T{};
  T.u = u;
  T.sv = reinterpret_cast<double*>(ws + B.sv);
  T.info = info ? info : reinterpret_cast<int32_t*>(ws + B.info);
  T.n = p.n;
  T.c = p.c;
  T.r = p.r;
  T.nlevels = p.nlevels;
  for (int l = 0; l <= p.nlevels; ++l) {
    QrLevel& q = T.lv[l];
    q.a = l == 0 ? z : reinterpret_cast<double*>(ws + B.a[l]);
    q.tau = reinterpret_cast<double*>(ws + B.tau[l]);
    q.y = l == 0 ? u : reinterpret_cast<double*>(ws + B.y[l]);
    q.n = p.lv_n[l];
    q.nblk = p.lv_nblk[l];
    q.blk_rows = p.lv_blk[l];
  }
  for (int l = 0; l < p.nlevels; ++l) T.lv[l].r_out = T.lv[l + 1].a;
  T.state0 = state0;
  T.draw_offset = draw_offset;
  T.normal_base = normal_base;
  T.kind = p.kind;
  if ((p.kind == 1 && p.nlevels == 1) || p.kind == 3) {
    T.vup = reinterpret_cast<double*>(ws + B.vup);
    T.vup_stride = B.vup_stride;
  }
  return T;
}

// Which targets take the one-warp small path (single block, fits 96 KB).
bool basis_is_small(const BasisTarget& t) {
  if (t.kind != 0) return t.nlevels == 0;
  return t.nlevels == 0 && t.n <= 1024 && srtt_basis_small_smem((int)t.n, t.c, t.r) <= 96 * 1024;
}

struct BasisLists {
  std::vector<int> small, big;
  std::vector<int> small_v[kSmallVariants];  // small targets by kernel variant
  std::vector<int> big_v[3];                  // big targets by top-kernel variant
  size_t off_big_v[3] = {};
  size_t off_small = 0, off_big = 0;  // blob offsets
  size_t off_small_v[kSmallVariants] = {};
  size_t off_map[SRTT_MAX_QR_LEVELS] = {};  // per TSQR level: CTA -> (target, block)
  // register-tree targets by column padding (16 / 32): single-CTA ones, the
  // tops of tall ones, and the (target, CTA) map of the tall ones
  // (single-CTA ones split again: at most one warp block / taller)
  // w_small[4 cp + slot]: slot 0 = taller than one warp block (row teams),
  // slots 1..3 = at most 32 / 64 / 128 rows (1 / 2 / 4 row groups)
  std::vector<int> w_small[8], w_tall[2];
  size_t off_w_small[8] = {}, off_w_tall[2] = {}, off_w_map[2] = {};
  int w_ctas[2] = {};
  // wide register path (kind 2): single-block targets, tall ones, and the
  // per-level (target, block) maps of the tall ones
  std::vector<int> generic;  // kind 3 (c > 64): one CTA each, global memory
  size_t off_generic = 0;
  std::vector<int> x_small, x_tall;
  size_t off_x_small = 0, off_x_tall = 0, off_x_map[SRTT_MAX_QR_LEVELS] = {};
  int x_ctas[SRTT_MAX_QR_LEVELS] = {};
  int x_levels = 0;
};

BasisLists make_basis_lists(const std::vector<BasisTarget>& targets, Blob& blob) {
  BasisLists L;
  for (int i = 0; i < (int)targets.size(); ++i) (basis_is_small(targets[i]) ? L.small : L.big).push_back(i);
  for (int v = 0; v < 2; ++v) {
    std::vector<int2> map;
    for (int i = 0; i < (int)targets.size(); ++i) {
      const BasisTarget& t = targets[i];
      if (t.kind != 1 || srtt_wtree_cp(t.c) != (v ? 32 : 16)) continue;
      if (t.nlevels == 0) {
        const int64_t groups = (t.n + 31) / 32;
        const int slot = t.n > srtt_wtree_chunk(v ? 32 : 16) ? 0 : (groups <= 1 ? 1 : (groups <= 2 ? 2 : 3));
        L.w_small[4 * v + slot].push_back(i);
      } else {
        L.w_tall[v].push_back(i);
        for (int b = 0; b < t.lv[0].nblk; ++b) map.push_back(make_int2(i, b));
      }
    }
    for (int u = 4 * v; u < 4 * v + 4; ++u)
      if (!L.w_small[u].empty()) L.off_w_small[u] = blob.add(L.w_small[u].data(), sizeof(int) * L.w_small[u].size());
    if (!L.w_tall[v].empty()) {
      L.off_w_tall[v] = blob.add(L.w_tall[v].data(), sizeof(int) * L.w_tall[v].size());
      L.off_w_map[v] = blob.add(map.data(), sizeof(int2) * map.size());
      L.w_ctas[v] = (int)map.size();
    }
  }
  for (int i = 0; i < (int)targets.size(); ++i)
    if (targets[i].kind == 3) L.generic.push_back(i);
  if (!L.generic.empty()) L.off_generic = blob.add(L.generic.data(), sizeof(int) * L.generic.size());
  for (int i = 0; i < (int)targets.size(); ++i)
    if (targets[i].kind == 2) (targets[i].nlevels == 0 ? L.x_small : L.x_tall).push_back(i);
  if (!L.x_small.empty()) L.off_x_small = blob.add(L.x_small.data(), sizeof(int) * L.x_small.size());
  if (!L.x_tall.empty()) {
    L.off_x_tall = blob.add(L.x_tall.data(), sizeof(int) * L.x_tall.size());
    for (int l = 0; l < SRTT_MAX_QR_LEVELS; ++l) {
      std::vector<int2> map;
      for (int i : L.x_tall)
        if (targets[i].nlevels > l)
          for (int b = 0; b < targets[i].lv[l].nblk; ++b) map.push_back(make_int2(i, b));
      if (map.empty()) break;
      L.off_x_map[l] = blob.add(map.data(), sizeof(int2) * map.size());
      L.x_ctas[l] = (int)map.size();
      L.x_levels = l + 1;
    }
  }
  for (int l = 0; l < SRTT_MAX_QR_LEVELS; ++l) {
    std::vector<int2> map;
    for (int i = 0; i < (int)targets.size(); ++i)
      if (targets[i].kind == 0 && targets[i].nlevels > l)
        for (int b = 0; b < targets[i].lv[l].nblk; ++b) map.push_back(make_int2(i, b));
    if (map.empty()) break;
    L.off_map[l] = blob.add(map.data(), sizeof(int2) * map.size());
  }
  const int zero = 0;
  L.off_small = blob.add(L.small.empty() ? &zero : L.small.data(), sizeof(int) * std::max<size_t>(1, L.small.size()));
  for (int i : L.small)
    if (targets[i].kind == 0) L.small_v[srtt_basis_small_variant((int)targets[i].n, targets[i].c)].push_back(i);
  for (int v = 0; v < kSmallVariants; ++v)
    if (!L.small_v[v].empty()) L.off_small_v[v] = blob.add(L.small_v[v].data(), sizeof(int) * L.small_v[v].size());
  for (int i : L.big)
    if (targets[i].kind == 0) L.big_v[srtt_basis_top_variant(targets[i].c)].push_back(i);
  for (int v = 0; v < 3; ++v)
    if (!L.big_v[v].empty()) L.off_big_v[v] = blob.add(L.big_v[v].data(), sizeof(int) * L.big_v[v].size());
  L.off_big = blob.add(L.big.empty() ? &zero : L.big.data(), sizeof(int) * std::max<size_t>(1, L.big.size()));
  return L;
}

// Grouped K2 launch sequence over many targets (device array dT).
int launch_basis_group(srtt_handle* h, std::vector<BasisTarget>& targets, const BasisTarget* dT,
                       const BasisLists& lists, const char* dblob, double* pad_scratch, int64_t pad_stride,
                       cudaStream_t small_stream = nullptr) {
  int launches = 0;
  int maxlev = 0;
  bool any_tall = false;
  for (auto& t : targets) {
    if (t.kind == 0) maxlev = std::max(maxlev, t.nlevels);
    any_tall = any_tall || t.nlevels > 0;
  }
  const int nt = (int)targets.size();
  // register-tree targets: single-CTA ones on the side stream, tall ones as
  // factor -> top -> apply on the main stream
  for (int u = 0; u < 8; ++u) {
    const int cp = u >= 4 ? 32 : 16;
    static const int kMode[4] = {0, 1, 2, 4};  // slot -> row groups (0: row teams)
    if (!lists.w_small[u].empty()) {
      size_t smem = 0;
      for (int i : lists.w_small[u]) smem = std::max(smem, srtt_wtree_top_smem((int)targets[i].n, targets[i].c, true));
      CK(srtt_launch_wtree_top(cp, kMode[u & 3], dT, reinterpret_cast<const int*>(dblob + lists.off_w_small[u]),
                               (int)lists.w_small[u].size(), smem, small_stream ? small_stream : h->stream));
      ++launches;
    }
  }
  for (int v = 0; v < 2; ++v) {
    const int cp = v ? 32 : 16;
    if (lists.w_tall[v].empty()) continue;
    size_t sf = 0, st = 0, sa = 0;
    for (int i : lists.w_tall[v]) {
      const BasisTarget& t = targets[i];
      sf = std::max(sf, srtt_wtree_factor_smem(t.lv[0].blk_rows, t.c));
      sa = std::max(sa, srtt_wtree_apply_smem(t.lv[0].blk_rows, t.c));
      st = std::max(st, srtt_wtree_top_smem((int)t.lv[1].n, t.c, false));
    }
    const int2* map = reinterpret_cast<const int2*>(dblob + lists.off_w_map[v]);
    CK(srtt_launch_wtree_factor(cp, dT, map, lists.w_ctas[v], sf, h->stream));
    CK(srtt_launch_wtree_top(cp, 0, dT, reinterpret_cast<const int*>(dblob + lists.off_w_tall[v]),
                             (int)lists.w_tall[v].size(), st, h->stream));
    CK(srtt_launch_wtree_apply(cp, dT, map, lists.w_ctas[v], sa, h->stream));
    launches += 3;
  }
  for (int v = 0; v < kSmallVariants; ++v) {
    if (lists.small_v[v].empty()) continue;
    size_t smem = 0;
    for (int i : lists.small_v[v])
      smem = std::max(smem, srtt_basis_small_smem((int)targets[i].n, targets[i].c, targets[i].r));
    CK(srtt_launch_basis_small(v, dT, reinterpret_cast<const int*>(dblob + lists.off_small_v[v]),
                               (int)lists.small_v[v].size(), smem, small_stream ? small_stream : h->stream));
    ++launches;
  }
  if (!lists.generic.empty()) {
    size_t smem = 0;
    for (int i : lists.generic) smem = std::max(smem, srtt_basis_generic_smem(targets[i].c, targets[i].r));
    CK(srtt_launch_basis_generic(dT, reinterpret_cast<const int*>(dblob + lists.off_generic), (int)lists.generic.size(),
                                 smem, small_stream ? small_stream : h->stream));
    ++launches;
  }
  if (!lists.x_small.empty()) {
    size_t smem = 0;
    for (int i : lists.x_small)
      smem = std::max(smem, srtt_wide_top_smem((int)targets[i].n, targets[i].c, targets[i].r, true));
    CK(srtt_launch_wide_top(dT, reinterpret_cast<const int*>(dblob + lists.off_x_small), (int)lists.x_small.size(), smem,
                            small_stream ? small_stream : h->stream));
    ++launches;
  }
  if (!lists.x_tall.empty()) {
    size_t sl = 0, st = 0;
    for (int i : lists.x_tall) {
      const BasisTarget& t = targets[i];
      sl = std::max(sl, srtt_wide_level_smem(t.lv[0].blk_rows, t.c));
      st = std::max(st, srtt_wide_top_smem((int)t.lv[t.nlevels].n, t.c, t.r, false));
    }
    for (int l = 0; l < lists.x_levels; ++l) {
      CK(srtt_launch_wide_factor(dT, reinterpret_cast<const int2*>(dblob + lists.off_x_map[l]), l, lists.x_ctas[l], sl,
                                 h->stream));
      ++launches;
    }
    CK(srtt_launch_wide_top(dT, reinterpret_cast<const int*>(dblob + lists.off_x_tall), (int)lists.x_tall.size(), st,
                            h->stream));
    ++launches;
    for (int l = lists.x_levels - 1; l >= 0; --l) {
      CK(srtt_launch_wide_apply(dT, reinterpret_cast<const int2*>(dblob + lists.off_x_map[l]), l, lists.x_ctas[l], sl,
                                h->stream));
      ++launches;
    }
  }
  if (lists.big.empty()) return launches;
  for (int l = 0; l < maxlev; ++l) {
    int nctas = 0;
    size_t smem = 0;
    for (auto& t : targets)
      if (t.kind == 0 && t.nlevels > l) {
        nctas += t.lv[l].nblk;
        smem = std::max(smem, srtt_basis_level_smem(t.lv[l].blk_rows, t.c));
      }
    CK(srtt_launch_tsqr_factor(dT, reinterpret_cast<const int2*>(dblob + lists.off_map[l]), l, nctas, smem,
                               h->stream));
    ++launches;
  }
  for (int v = 0; v < 3; ++v) {
    if (lists.big_v[v].empty()) continue;
    size_t smem = 0;
    for (int i : lists.big_v[v])
      smem = std::max(smem, srtt_basis_top_smem((int)targets[i].lv[targets[i].nlevels].n, targets[i].c, targets[i].r));
    CK(srtt_launch_basis_top(v, dT, reinterpret_cast<const int*>(dblob + lists.off_big_v[v]),
                             (int)lists.big_v[v].size(), smem, h->stream));
    ++launches;
  }
  for (int l = maxlev - 1; l >= 0; --l) {
    int nctas = 0;
    size_t sm = 0;
    for (auto& t : targets)
      if (t.kind == 0 && t.nlevels > l) {
        nctas += t.lv[l].nblk;
        sm = std::max(sm, srtt_basis_level_smem(t.lv[l].blk_rows, t.c));
      }
    CK(srtt_launch_tsqr_apply(dT, reinterpret_cast<const int2*>(dblob + lists.off_map[l]), l, nctas, sm,
                              h->stream));
    ++launches;
  }
  if (any_tall) {
    CK(srtt_launch_pad(dT, nt, pad_scratch, pad_stride, h->stream));
    ++launches;
  }
  return launches;
}

void assign_basis_ctas(std::vector<BasisTarget>& targets) {
  for (int l = 0; l < SRTT_MAX_QR_LEVELS; ++l) {
    int c = 0;
    for (auto& t : targets) {
      t.cta_begin[l] = c;
      if (t.kind == 0 && t.nlevels > l) c += t.lv[l].nblk;
    }
  }
}

// ---- core (K3) planning --------------------------------------------------------
struct CorePlan {
  CoreParams P{};
  int grid = 0;
  std::vector<int64_t> dims;   // modes of the (possibly reshaped) tensor
  std::vector<int64_t> ranks;
  int64_t part_doubles = 0;
  int64_t rec_doubles = 0;   // flat mode: record slots
  int64_t scratch_doubles = 0;  // split-K partials of the first tail TTM
  size_t off_scratch = 0;
  int64_t cnt_words = 0;     // flat mode: group counters
  size_t ufrag_doubles = 0;
  size_t off_items = 0;
  size_t off_rec = 0, off_cnt = 0;
};

int pad_tiles(int64_t r) { return r <= 8 ? 1 : (r <= 16 ? 2 : (r <= 32 ? 4 : 0)); }

CorePlan plan_core(const std::vector<int64_t>& dims, const std::vector<int64_t>& ranks, int sms,
                   int force_m = 0, int force_S = 0) {
  const int d = (int)dims.size();
  CorePlan cp;
  cp.dims = dims;
  cp.ranks = ranks;
  CoreParams& P = cp.P;
  const int64_t n0 = dims[0];
  const int64_t N = prod(dims);
  const int64_t Q = N / n0;
  P.n0 = n0;
  P.Q = Q;
  P.r0 = (int)ranks[0];
  P.NT = pad_tiles(ranks[0]);
  P.NT1 = pad_tiles(ranks[1]);
  if (!P.NT || !P.NT1) invalid("core: ranks above 32 in modes 0 and 1 are not supported by the B200 core kernel");
  P.use_tma = (n0 % 2 == 0) ? 1 : 0;
  P.fdim[0] = dims[1];
  P.frank[0] = (int)ranks[1];

  struct Cand {
    int m = 0, S = 0, ns = 0, tpb = 1, warps = 8, flat = 0, RB = 0, slot_ch = 0;
    int64_t SL = 0, G = 0, GS = 0, items = 0, grid = 0;
    int A = 0;
    double cost = 1e300;
  } best;
  // flat mode (one row block): balanced per-warp tile ranges, records
  // reduced inside the kernel. development aid: SRTT_FORCE_FLAT=0/1
  int force_flat = -1;
  if (const char* ff = std::getenv("SRTT_FORCE_FLAT")) force_flat = std::atoi(ff);
  // row blocks: the whole column up to 256 rows; longer columns in blocks
  // of 256 or (m = 2) 512 rows -- the mode-1 fold runs once per row block,
  // so 512 halves its DMMA work (C5: 12.5 % -> 6 % of the pass) at the price
  // of a 2x larger U0 in shared memory and a chunked CTA reduction
  // development aid: SRTT_FORCE_RB=256/512
  int force_rb = 0;
  if (const char* fr = std::getenv("SRTT_FORCE_RB")) force_rb = std::atoi(fr);
  std::vector<int> rb_choices;
  if (n0 <= 256) rb_choices.push_back((int)((n0 + 15) / 16 * 16));
  else for (int rb : {256, 512}) if (!force_rb || force_rb == rb) rb_choices.push_back(rb);
  for (int RBc : rb_choices) {
  P.RB = RBc;
  P.nrb = (int)((n0 + P.RB - 1) / P.RB);
  P.slot_ch = 0;
  const bool flat_ok = P.nrb == 1 && force_flat != 0;
  for (int m = 2; m <= std::min(3, d); ++m) {
    if (force_m && m != force_m) continue;
    if (RBc > 256 && m != 2) continue;
    // warps per CTA: 16 when the rank tiles are small (register budget
    // 128/thread), else 8; each with the widest box that leaves a ring of
    // >= 3 boxes per warp (2 for single-tile boxes)
    // development aid: SRTT_FORCE_CORE="warps,tpb" pins the candidate
    int force_w = 0, force_tpb = 0;
    if (const char* fc = std::getenv("SRTT_FORCE_CORE")) std::sscanf(fc, "%d,%d", &force_w, &force_tpb);
    // (measured on C2/C3/C4: 10 or 12 warps balance an item's tile groups
    // better but lose more in latency hiding than they gain, within +-3 %)
    for (int W : {16, 8}) {
      if (W == 16 && P.NT * P.NT1 > 4) continue;
      if (force_w && W != force_w) continue;
      CoreParams T = P;
      T.m = m;
      T.A = (int)(ranks[0] * ranks[1] * (m == 3 ? ranks[2] : 1));
      T.warps = W;
      if (RBc > 256) T.slot_ch = std::min(T.A, 256);
      int tpb = 0, ns = 0;
      for (int tb : {2, 1}) {
        if (tb == 2 && (P.NT > 2 || P.NT1 > 2)) continue;
        if (force_tpb && tb != force_tpb) continue;
        T.tpb = tb;
        const int n = srtt_core_max_stages(T, kCoreSmem);
        if (n >= 3 || (tb == 1 && n >= 2)) {
          tpb = tb;
          ns = n;
          break;
        }
      }
      if (!tpb) continue;
      const int64_t bc = 16 * tpb;
      const int64_t GS = prod(dims, 1, m);
      const int64_t G = Q / GS;
      const int64_t max_s = (GS + bc - 1) / bc;
      const double kBw = 6.5e12 * 0.85, kDmmaSm = 37.1e12 / 148.0 * 0.9;
      const int64_t ntiles_f = (Q + bc - 1) / bc;
      if (flat_ok && ntiles_f >= W) {
        // every warp owns >= 1 tile (the group counters count all warps
        // between a group's first and last owner)
        const int64_t ntiles = ntiles_f;
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(sms, ntiles / W));
        const int64_t nw = grid * W;
        const double imb = (double)((ntiles + nw - 1) / nw) * (double)nw / (double)ntiles;
        const double rows = (double)std::min<int64_t>(P.RB, n0);
        const double t_mem = rows * (double)Q * 8.0 / kBw * ((double)sms / (double)grid);
        const double t_cmp = (double)Q * (16.0 * P.NT * P.RB + 128.0 * P.NT * P.NT1) / (kDmmaSm * (double)grid);
        // records written and reduced through L2 + compact R read by the tail
        const double recs = (double)(nw + G) * T.A * 8.0 * 2.0 / (0.3 * kBw) +
                            // one warp sums a group's records (~20 GB/s per warp)
                            (double)((GS + bc - 1) / bc * nw / ntiles + 2) * T.A * 8.0 / 20e9;
        const double out = 2.0 * (double)G * T.A * 8.0 / (0.1 * kBw) + 5e-6 * (d - m);
        const double cost = std::max(t_mem, t_cmp) * imb * (W == 16 ? 1.0 : 1.45) + recs + out + 1.5e-6;
        if ((force_flat == 1 && !best.flat) || cost < best.cost) {
          best = Cand{};
          best.RB = RBc;
          best.slot_ch = T.slot_ch;
          best.m = m;
          best.S = 1;
          best.ns = ns;
          best.tpb = tpb;
          best.warps = W;
          best.flat = 1;
          best.G = G;
          best.GS = GS;
          best.grid = grid;
          best.items = ntiles;
          best.A = T.A;
          best.cost = cost;
        }
        if (force_flat == 1) continue;
      }
      for (int64_t S = 1; S <= max_s; S = S < 8 ? S + 1 : S * 2) {
        if (force_S && S != force_S) continue;
        const int64_t SL = ((GS + S - 1) / S + bc - 1) / bc * bc;
        const int64_t Se = (GS + SL - 1) / SL;
        const int64_t items = P.nrb * G * Se;
        const int64_t ntg = SL / bc;
        // Wall-time model: CTAs run items in rounds; an item takes the larger
        // of its share of HBM bandwidth and its FP64 tensor-core time, scaled
        // by the slowest warp's share of the item's tile groups.
        const int64_t grid = std::min<int64_t>(items, sms);
        const int64_t full = items / grid, last = items % grid;
        const double rows = (double)std::min<int64_t>(P.RB, n0);
        const double bytes_item = rows * (double)SL * 8.0;
        const double flops_item = (double)SL * (16.0 * P.NT * P.RB + 128.0 * P.NT * P.NT1);
        const double imb = (double)((ntg + W - 1) / W) * W / (double)ntg;
        const double kItemOverhead = 1.5e-6;
        auto t_item = [&](int64_t active) {
          const double t_mem = bytes_item * (double)active / kBw;
          const double t_cmp = flops_item / kDmmaSm;
          // 8 warps hide less latency: measured 1.45x per item on C2
          return std::max(t_mem, t_cmp) * imb * (W == 16 ? 1.0 : 1.45) + kItemOverhead;
        };
        // tail: partials written + re-read by the tail TTMs (measured ~10x
        // slower than streaming: strided small reductions) + a launch each
        const double out = 2.0 * (double)items * T.A * 8.0 / (0.1 * kBw) + 5e-6 * (d - m);
        const double cost = (double)full * t_item(grid) + (last ? t_item(last) : 0.0) + out;
        if (cost < best.cost) {
          best = Cand{};
          best.RB = RBc;
          best.slot_ch = T.slot_ch;
          best.m = m;
          best.S = (int)Se;
          best.ns = ns;
          best.tpb = tpb;
          best.warps = W;
          best.SL = SL;
          best.G = G;
          best.GS = GS;
          best.items = items;
          best.A = T.A;
          best.cost = cost;
        }
        if (S >= max_s) break;
      }
    }
  }
  }  // row-block choices
  if (best.m == 0) invalid("core: no feasible work decomposition");
  P.RB = best.RB;
  P.nrb = (int)((n0 + P.RB - 1) / P.RB);
  P.slot_ch = best.slot_ch;
  if (std::getenv("SRTT_DEBUG_PLAN"))  // development aid
    std::fprintf(stderr, "core plan: flat=%d m=%d S=%d SL=%lld items=%lld warps=%d tpb=%d ns=%d RB=%d slot_ch=%d "
                 "cost=%.3g\n", best.flat, best.m, best.S, (long long)best.SL, (long long)best.items, best.warps,
                 best.tpb, best.ns, best.RB, best.slot_ch, best.cost);
  P.m = best.m;
  P.S = best.S;
  P.SL = best.SL;
  P.G = best.G;
  P.GS = best.GS;
  P.nitems = best.items;
  P.A = best.A;
  P.nstages = best.ns;
  P.tpb = best.tpb;
  P.warps = best.warps;
  if (best.m == 3) {
    P.fdim[1] = dims[2];
    P.frank[1] = (int)ranks[2];
  }
  P.flat = best.flat;
  if (best.flat) {
    P.nitems = 0;
    P.ntiles = best.items;
    P.nw = (int)(best.grid * best.warps);
    cp.grid = (int)best.grid;
    cp.part_doubles = best.G * best.A;
    cp.rec_doubles = (P.nw + best.G) * best.A;
    cp.cnt_words = best.G;
  } else {
    cp.part_doubles = best.items * best.A;
  }
  // whole-column boxes for short columns (flat, r0 <= 8, n0 <= 64, n0 even
  // and not a multiple of 16): one TMA box per tile instead of ceil(n0/16),
  // k-steps over RB = n0 rounded to 4 rows instead of 16.
  // development aid: SRTT_FORCE_CB=0 keeps the 16-row swizzled boxes
  const char* fcb = std::getenv("SRTT_FORCE_CB");
  if (P.flat && P.NT == 1 && P.use_tma && n0 <= 64 && n0 % 16 != 0 && !(fcb && fcb[0] == '0')) {
    CoreParams T = P;
    T.tpb = 1;
    T.RB = (int)((n0 + 3) / 4 * 4);
    T.cb = T.RB % 4 == 2 ? T.RB : T.RB + 2;  // = 2 (mod 4), >= RB
    const int ns = srtt_core_max_stages(T, kCoreSmem);
    if (ns >= 2) {
      const int64_t ntiles = (P.Q + 15) / 16;
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(sms, ntiles / P.warps));
      if (ntiles >= P.warps) {
        P = T;
        P.nstages = ns;
        P.ntiles = ntiles;
        P.nw = (int)(grid * P.warps);
        cp.grid = (int)grid;
        cp.rec_doubles = (P.nw + P.G) * P.A;
        if (std::getenv("SRTT_DEBUG_PLAN"))
          std::fprintf(stderr, "core plan: whole-column boxes cb=%d RB=%d ns=%d tiles=%lld\n", P.cb, P.RB, ns,
                       (long long)ntiles);
      }
    }
  }
  cp.ufrag_doubles = (size_t)P.nrb * P.RB * P.NT * 8;
  return cp;
}

// Launches the full core pass for factors already on the device.
// x: device tensor (dims), u[k]: device n_k x r_k column-major, out: device core.
int launch_core_pass(srtt_handle* h, CorePlan& cp, const double* x, const std::vector<const double*>& u,
                     double* out, char* ws, size_t off_ufrag, const std::vector<size_t>& off_fu,
                     size_t off_part, size_t off_tmp0, size_t off_tmp1) {
  const size_t off_items = cp.off_items;
  int launches = 0;
  CoreParams& P = cp.P;
  const int d = (int)cp.dims.size();
  P.x = x;
  P.ufrag = reinterpret_cast<double*>(ws + off_ufrag);
  P.part = reinterpret_cast<double*>(ws + off_part);
  {
    const double* us[2] = {nullptr, nullptr};
    double* uts[2] = {nullptr, nullptr};
    int64_t ns[2] = {0, 0};
    int rs[2] = {0, 0};
    for (int k = 1; k < P.m; ++k) {
      us[k - 1] = u[k];
      uts[k - 1] = reinterpret_cast<double*>(ws + off_fu[k]);
      ns[k - 1] = cp.dims[k];
      rs[k - 1] = (int)cp.ranks[k];
      P.fu[k - 1] = uts[k - 1];
    }
    CoreItem* items = reinterpret_cast<CoreItem*>(ws + off_items);
    P.items = items;
    if (P.flat) {
      P.rec = reinterpret_cast<double*>(ws + cp.off_rec);
      P.cnt = reinterpret_cast<uint32_t*>(ws + cp.off_cnt);
    }
    CK(srtt_launch_prep_all(P, items, u[0], P.n0, P.r0, P.RB, P.NT, P.nrb, const_cast<double*>(P.ufrag), P.m - 1,
                            us, uts, ns, rs, h->stream));
    ++launches;
  }
  if (P.m == 2) P.fu[1] = nullptr;
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (P.use_tma) {
    if (P.cb) encode_tmap_plain(&tmap, x, P.n0, P.Q, P.n0, P.cb, 16 * P.tpb);
    else encode_tmap(&tmap, x, P.n0, P.Q, 16 * P.tpb);
  }
  if (!P.flat) cp.grid = (int)std::min<int64_t>(P.nitems, (int64_t)h->sms);
  if (h->timing) record_event(h->kev[4], h->stream);
  CK(srtt_launch_core(&tmap, P, cp.grid, h->stream));
  if (h->timing) record_event(h->kev[5], h->stream);
  ++launches;
  // tail: fixed-order reduction of the item partials + TTMs of modes m..d-1
  // (flat mode: the kernel already reduced its records into compact R_m)
  const int nparts = P.flat ? 1 : P.nrb * P.S;
  if (P.m == d) {
    TtmParams T{};
    T.in = P.part;
    T.u = reinterpret_cast<const double*>(h->ones.p);
    T.out = out;
    T.g = P.A;
    T.n = 1;
    T.post = 1;
    T.rr = 1;
    T.transpose = 1;
    T.nparts = nparts;
    T.part_stride = (int64_t)P.G * P.A;
    CK(srtt_launch_ttm(T, h->stream));
    ++launches;
  } else {
    const double* in = P.part;
    int64_t g = P.A;
    int np = nparts;
    for (int k = P.m; k < d; ++k) {
      const int64_t post = prod(cp.dims, k + 1);
      TtmParams T{};
      T.in = in;
      T.u = u[k];
      T.g = g;
      T.n = cp.dims[k];
      T.post = post;
      T.rr = cp.ranks[k];
      T.transpose = 1;
      T.nparts = np;
      T.part_stride = (int64_t)P.G * P.A;
      if (k == P.m && cp.scratch_doubles) {
        T.scratch = reinterpret_cast<double*>(ws + cp.off_scratch);
        T.scratch_doubles = cp.scratch_doubles;
      }
      T.out = (k == d - 1) ? out : reinterpret_cast<double*>(ws + (((k - P.m) % 2) ? off_tmp1 : off_tmp0));
      CK(srtt_launch_ttm(T, h->stream));
      ++launches;
      in = T.out;
      g *= cp.ranks[k];
      np = 1;
    }
  }
  return launches;
}

// Workspace needs of the core pass.
void layout_core(Layout& L, CorePlan& cp, size_t& off_ufrag, std::vector<size_t>& off_fu,
                 size_t& off_part, size_t& off_tmp0, size_t& off_tmp1) {
  const int d = (int)cp.dims.size();
  cp.off_items = L.take(sizeof(CoreItem) * (size_t)cp.P.nitems);
  off_ufrag = L.take(sizeof(double) * cp.ufrag_doubles);
  off_fu.assign(d, 0);
  for (int k = 1; k < cp.P.m; ++k) off_fu[k] = L.take(sizeof(double) * cp.dims[k] * cp.ranks[k]);
  off_part = L.take(sizeof(double) * cp.part_doubles);
  cp.off_rec = L.take(sizeof(double) * cp.rec_doubles);
  cp.off_cnt = L.take(sizeof(uint32_t) * cp.cnt_words);
  // split-K partials of the first tail TTM (long mode m, few slabs)
  if (cp.P.m < d) {
    const int64_t m = cp.P.m;
    const int64_t s1 = (int64_t)cp.P.A * cp.ranks[m] * prod(cp.dims, (int)m + 1);
    const int64_t nch = std::min<int64_t>(148 * 4, cp.dims[m] / 64 + 1);
    cp.scratch_doubles = s1 * nch;
    cp.off_scratch = L.take(sizeof(double) * cp.scratch_doubles);
  }
  // largest intermediate of the tail
  int64_t g = cp.P.A, big = 1;
  for (int k = cp.P.m; k < d; ++k) {
    g *= cp.ranks[k];
    big = std::max<int64_t>(big, g * prod(cp.dims, k + 1));
  }
  off_tmp0 = L.take(sizeof(double) * big);
  off_tmp1 = L.take(sizeof(double) * big);
}

// The core pass of one call. The streaming kernel's DMMA tiles cover ranks
// up to 32 in modes 0 and 1; larger ranks run one pass per (32-column block
// of U_0) x (32-column block of U_1) -- core[a, b, ...] depends only on
// column a of U_0 and column b of U_1 -- and each block's sub-core is
// scattered into the core. X is then streamed once per block pair.
struct CoreJob {
  struct Piece {
    CorePlan cp;
    size_t off_ufrag = 0, off_part = 0, off_tmp0 = 0, off_tmp1 = 0;
    std::vector<size_t> off_fu;
    int64_t a0 = 0, ra = 0, b0 = 0, rb = 0;
  };
  std::vector<Piece> pieces;
  std::vector<int64_t> dims, ranks;
  size_t off_sub = 0;
  bool blocked = false;

  void plan(const std::vector<int64_t>& dims_, const std::vector<int64_t>& ranks_, int sms, Layout& L) {
    dims = dims_;
    ranks = ranks_;
    const int d = (int)dims.size();
    blocked = ranks[0] > 32 || (d >= 2 && ranks[1] > 32);
    const int64_t r1 = d >= 2 ? ranks[1] : 1;
    int64_t biggest = 0;
    for (int64_t a0 = 0; a0 < ranks[0]; a0 += 32)
      for (int64_t b0 = 0; b0 < r1; b0 += 32) {
        Piece pc;
        pc.a0 = a0;
        pc.ra = std::min<int64_t>(32, ranks[0] - a0);
        pc.b0 = b0;
        pc.rb = std::min<int64_t>(32, r1 - b0);
        std::vector<int64_t> pr = ranks;
        pr[0] = pc.ra;
        if (d >= 2) pr[1] = pc.rb;
        pc.cp = plan_core(dims, pr, sms);
        layout_core(L, pc.cp, pc.off_ufrag, pc.off_fu, pc.off_part, pc.off_tmp0, pc.off_tmp1);
        biggest = std::max<int64_t>(biggest, prod(pr));
        pieces.push_back(std::move(pc));
        if (!blocked) break;
      }
    if (blocked) off_sub = L.take(sizeof(double) * biggest);
  }

  int launch(srtt_handle* h, const double* x, const std::vector<const double*>& u, double* out, char* ws) {
    if (!blocked) {
      Piece& pc = pieces[0];
      return launch_core_pass(h, pc.cp, x, u, out, ws, pc.off_ufrag, pc.off_fu, pc.off_part, pc.off_tmp0, pc.off_tmp1);
    }
    const int d = (int)dims.size();
    const int64_t r1 = d >= 2 ? ranks[1] : 1;
    int64_t rest = 1;
    for (int k = 2; k < d; ++k) rest *= ranks[k];
    double* sub = reinterpret_cast<double*>(ws + off_sub);
    int n = 0;
    for (Piece& pc : pieces) {
      std::vector<const double*> up = u;
      up[0] = u[0] + pc.a0 * dims[0];
      if (d >= 2) up[1] = u[1] + pc.b0 * dims[1];
      n += launch_core_pass(h, pc.cp, x, up, sub, ws, pc.off_ufrag, pc.off_fu, pc.off_part, pc.off_tmp0, pc.off_tmp1);
      CK(srtt_launch_scatter_block(sub, out, ranks[0], r1, pc.a0, pc.ra, pc.b0, pc.rb, rest, h->stream));
      ++n;
    }
    return n;
  }
};

// ---- sketch target construction ---------------------------------------------
// Fibre chunks per K1 target: the grouped grid parallelises over rows only
// when a target samples few fibres (BASELINE configs: w <= 168, one chunk,
// direct write); a target with many fibres (sampling fractions of several
// percent: c4a20, c5s64k) also splits its fibres over CTAs, >= 512 each,
// until the target alone fills the GPU ~4 CTAs deep.
int sketch_fsplit(int64_t rows, int64_t w) {
  const int64_t rt = std::min<int64_t>(rows, 64);
  const int64_t row_ctas = (rows + rt - 1) / rt;
  const int64_t want = (4 * 148 + row_ctas - 1) / row_ctas;
  return (int)std::max<int64_t>(1, std::min<int64_t>(w / 512, want));
}

// Fibre chunks of a K1c target (128-row CTAs): about 4 CTAs per SM overall.
int sketch_fsplit_contig(int64_t rows, int64_t w) {
  const int64_t row_ctas = (rows + 127) / 128;
  const int64_t want = (4 * 148 + row_ctas / 2) / row_ctas;
  return (int)std::max<int64_t>(1, std::min<int64_t>(w / 256, want));
}

// Workspace for a target's fibre-chunk partials (when split) and its
// once-generated Omega (when more than one CTA would generate it), appended.
bool sketch_omega_once(int64_t rows, int64_t w) {
  // only where regenerating it per CTA costs more than one extra launch:
  // many CTAs AND a large Omega (C4's 324 CTAs x 900 normals do not pay)
  const int64_t rt = std::min<int64_t>(rows, 64);
  return (rows + rt - 1) / rt * sketch_fsplit(rows, w) >= 8 && w >= 512;
}
size_t sketch_part_bytes(int64_t rows, int64_t w, int c) {
  // upper bound over the scalar and the K1c split (the kernel is chosen later)
  const int f = std::max(sketch_fsplit(rows, w), sketch_fsplit_contig(rows, w));
  const size_t part = f > 1 ? sizeof(double) * (size_t)f * rows * c : 0;
  const size_t om = sketch_omega_once(rows, w) ? sizeof(double) * (size_t)w * c : 0;
  return (part + 255) / 256 * 256 + om;
}

SketchTarget make_sketch_target(const double* x, const std::vector<int64_t>& dims,
                                const std::vector<int>& modes, int64_t w, int c) {
  SketchTarget T{};
  T.x = x;
  const int d = (int)dims.size();
  std::vector<int64_t> stride(d);
  int64_t g = 1;
  for (int k = 0; k < d; ++k) {
    stride[k] = g;
    g *= dims[k];
  }
  std::vector<bool> in(d, false);
  for (int m : modes) in[m] = true;
  T.rows = 1;
  for (int k = 0; k < d; ++k) {
    if (in[k]) {
      T.row_dim[T.nrow_modes] = dims[k];
      T.row_stride[T.nrow_modes] = stride[k];
      T.nrow_modes++;
      T.rows *= dims[k];
    } else {
      T.col_dim[T.ncol_modes] = dims[k];
      T.col_stride[T.ncol_modes] = stride[k];
      T.ncol_modes++;
    }
  }
  T.w = w;
  T.c = c;
  T.row_tile = (int)std::min<int64_t>(T.rows, 64);
  T.slab_digit = -1;
  T.fsplit = sketch_fsplit(T.rows, w);
  // contiguous fibres (S = the leading modes 0..m-1, so fibre j starts at
  // cols[j] * rows) with many fibres: staged DMMA kernel (K1c)
  bool leading = !modes.empty();
  std::vector<int> ms(modes.begin(), modes.end());
  std::sort(ms.begin(), ms.end());
  for (size_t i = 0; i < ms.size(); ++i) leading = leading && ms[i] == (int)i;
  T.contig = (leading && w >= 512 && c <= 64 && !std::getenv("SRTT_NO_K1C")) ? 1 : 0;
  if (T.contig) T.fsplit = sketch_fsplit_contig(T.rows, w);
  return T;
}

// CTAs of one target in the grouped scalar K1 grid (0 for K1c targets).
int64_t sketch_target_ctas(const SketchTarget& T) {
  if (T.contig) return 0;
  return (T.rows + T.row_tile - 1) / T.row_tile * T.fsplit;
}

// K1c / K1t index spaces (contig targets need Omega in memory and no
// sharding masks; K1c ones fall back to the scalar kernel otherwise).
int64_t assign_contig_ctas(std::vector<SketchTarget>& sk) {
  int64_t n = 0, nt = 0;
  for (auto& t : sk) {
    if (t.contig == 1 && (!t.omega || t.slab_digit >= 0 || t.flat_hi > 0)) t.contig = 0;
    t.cta_begin_c = n;
    t.cta_begin_t = nt;
    if (t.contig == 1) n += (t.rows + 127) / 128 * t.fsplit;
    if (t.contig == 2) nt += (t.rows + 127) / 128 * t.fsplit;
  }
  return n;
}

// K1t opt-in (single-GPU paths): a target whose row modes are the TRAILING
// modes and whose columns are densely sampled (>= 1/4 of them, >= 512) has
// its sampled columns sorted ascending here -- cols is reordered in place and
// perm[k] = the sampled position of sorted column k -- so neighbouring fibres
// of a K1t stage are neighbouring addresses. Z is a sum over the fibres, so
// the order only changes rounding. Returns whether it did.
bool sketch_trans_prepare(const std::vector<int64_t>& dims, std::vector<int> modes, int64_t w, int c,
                          std::vector<int64_t>& cols, std::vector<int64_t>& perm) {
  if (std::getenv("SRTT_NO_K1C") || c > 64 || w < 512 || modes.empty()) return false;
  std::sort(modes.begin(), modes.end());
  const int d = (int)dims.size();
  for (size_t i = 0; i < modes.size(); ++i)
    if (modes[i] != d - (int)modes.size() + (int)i) return false;
  int64_t rows = 1;
  for (int m : modes) rows *= dims[m];
  const int64_t ncols = prod(dims) / rows;
  if (4 * w < ncols || !sketch_omega_once(rows, w)) return false;
  perm.resize(w);
  for (int64_t k = 0; k < w; ++k) perm[k] = k;
  std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return cols[a] < cols[b]; });
  std::vector<int64_t> sorted(w);
  for (int64_t k = 0; k < w; ++k) sorted[k] = cols[perm[k]];
  cols.swap(sorted);
  return true;
}

// Marks a prepared K1t target (after make_sketch_target).
void mark_sketch_trans(SketchTarget& T, const int64_t* dperm) {
  T.contig = 2;
  T.perm = dperm;
  T.ncols = 1;
  for (int mm = 0; mm < T.ncol_modes; ++mm) T.ncols *= T.col_dim[mm];
  T.fsplit = sketch_fsplit_contig(T.rows, T.w);
}

// K1 over a group of targets (device array dT, host copy sk), plus the
// fixed-order reduction of the fibre-chunk partials when any target is split.
int launch_sketch_group(const SketchTarget* dT, const std::vector<SketchTarget>& sk, int64_t ctas, int cmax,
                        cudaStream_t st) {
  int n = 0;
  int64_t om_elems = 0;
  for (auto& t : sk)
    if (t.omega_gen) om_elems = std::max<int64_t>(om_elems, t.w * t.c);
  if (om_elems) {
    CK(srtt_launch_omega(dT, (int)sk.size(), om_elems, st));
    ++n;
  }
  if (ctas > 0) {
    CK(srtt_launch_sketch(dT, (int)sk.size(), ctas, cmax, st));
    ++n;
  }
  for (int kind = 1; kind <= 2; ++kind) {  // K1c, then K1t
    int64_t ctas_c = 0;
    int cmax_c = 0;
    for (auto& t : sk)
      if (t.contig == kind) {
        ctas_c += (t.rows + 127) / 128 * t.fsplit;
        cmax_c = std::max(cmax_c, t.c);
      }
    if (ctas_c > 0) {
      CK(srtt_launch_sketch_contig(dT, (int)sk.size(), ctas_c, cmax_c, kind == 2, st));
      ++n;
    }
  }
  int64_t split_elems = 0;
  for (auto& t : sk)
    if (t.fsplit > 1) split_elems = std::max<int64_t>(split_elems, t.rows * t.c);
  if (!split_elems) return n;
  CK(srtt_launch_sketch_reduce(dT, (int)sk.size(), split_elems, st));
  return n + 1;
}

// Points a target at its scratch (see sketch_part_bytes): fibre-chunk
// partials and, when Omega is to be generated once, its buffer.
void attach_sketch_scratch(SketchTarget& T, char* scratch) {
  T.zpart = reinterpret_cast<double*>(scratch);
  if (!T.omega && sketch_omega_once(T.rows, T.w)) {
    const size_t part = T.fsplit > 1 ? sizeof(double) * (size_t)T.fsplit * T.rows * T.c : 0;
    T.omega_gen = reinterpret_cast<double*>(scratch + (part + 255) / 256 * 256);
    T.omega = T.omega_gen;
  }
  // K1c needs Omega in memory and no sharding masks (set before this call);
  // a K1t target's columns are sorted, so it can never fall back
  if (T.contig == 1 && (!T.omega || T.slab_digit >= 0 || T.flat_hi > 0)) T.contig = 0;
  if (T.contig == 2 && (!T.omega_gen || T.slab_digit >= 0 || T.flat_hi > 0))
    fail(SRTT_ERR_INTERNAL, "K1t target without a generated Omega");
}

// ---- report helpers ------------------------------------------------------------
void write_warnings(srtt_report* rep, const std::vector<std::string>& w) {
  if (!rep) return;
  rep->num_warnings = (int64_t)w.size();
  if (!rep->warnings || rep->warnings_capacity <= 0) return;
  std::string all;
  for (auto& s : w) all += s + "\n";
  const size_t n = std::min<size_t>(all.size(), (size_t)rep->warnings_capacity - 1);
  std::memcpy(rep->warnings, all.data(), n);
  rep->warnings[n] = 0;
}

void copy_out(srtt_handle* h, void* dst, const void* src, size_t bytes, int on_device) {
  CK(cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     h->stream));
}

// Returns a device pointer for `x` (copying host data into h->xbuf).
const double* stage_input(srtt_handle* h, const double* x, int on_device, int64_t count) {
  if (on_device) return x;
  h->xbuf.ensure(sizeof(double) * count);
  CK(cudaMemcpyAsync(h->xbuf.p, x, sizeof(double) * count, cudaMemcpyHostToDevice, h->stream));
  return reinterpret_cast<const double*>(h->xbuf.p);
}

struct Timer {
  srtt_handle* h;
  int n = 0;
  void mark() {
    if (h->timing) record_event(h->ev[n], h->stream);
    ++n;
  }
  double between(int a, int b) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]));
    return ms * 1e-3;
  }
};

// Start of a decomposition: switch to the other parameter set and wait
// until the call that last used it has finished with it.
void begin_call(srtt_handle* h) {
  h->cur ^= 1;
  auto& ps = h->pset();
  if (ps.recorded) CK(cudaEventSynchronize(ps.done));
}

// End of the enqueue part: mark the parameter set busy until the stream
// reaches this point. Returns true when the caller must synchronise
// (host outputs or a report requested); otherwise the call is
// stream-ordered and returns immediately.
bool end_call(srtt_handle* h, bool must_sync) {
  auto& ps = h->pset();
  CK(cudaEventRecord(ps.done, h->stream));
  ps.recorded = true;
  return must_sync;
}

// Issues the device work of one decomposition: directly, or (use_graphs)
// captured once per signature into a CUDA graph and replayed. The key holds
// every pointer the work bakes in (workspace, parameter blob, input,
// outputs, stream), so buffer growth simply creates a new graph.
bool is_default_stream(cudaStream_t s) {
  return s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread;
}

template <class F>
void run_enqueue(srtt_handle* h, const std::string& key, F&& enqueue) {
  if (!h->use_graphs) {
    enqueue();
    return;
  }
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    if (h->graphs.size() > 64) {
      for (auto& g : h->graphs) cudaGraphExecDestroy(g.second.exec);
      h->graphs.clear();
    }
    // the legacy / per-thread default streams cannot be captured: capture on
    // the handle's own stream, launch the graph into the caller's stream
    const cudaStream_t launch_stream = h->stream;
    if (is_default_stream(launch_stream)) h->stream = h->own_stream;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
    const int64_t before = h->launches;
    try {
      enqueue();
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(h->stream, &g);
      h->stream = launch_stream;
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g;
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
    h->stream = launch_stream;
    CK(ce);
    srtt_handle::Graph entry;
    CK(cudaGraphInstantiate(&entry.exec, g, 0));
    cudaGraphDestroy(g);
    entry.launches = h->launches - before;
    it = h->graphs.emplace(key, entry).first;
    h->launches = before;
  }
  CK(cudaGraphLaunch(it->second.exec, h->stream));
  h->launches += it->second.launches;
}

std::string ptr_key(const void* p) { return std::to_string(reinterpret_cast<uintptr_t>(p)); }

double kernel_pair(srtt_handle* h, int i) {
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, h->kev[2 * i], h->kev[2 * i + 1]));
  return ms * 1e-3;
}

// The device Gaussian generator is random-access (normal t = Box-Muller pair
// t/2); the reference's stream retries a pair whose u1 == 0 (rng.hpp:71),
// which shifts every later draw. The event has probability 2^-53 per pair;
// when a kernel meets it the call reports it instead of failing silently.
const char* const kU1ZeroWarning =
    "Box-Muller u1 == 0 draw met (p = 2^-53): the reference would retry it and shift later Gaussian draws, "
    "so Omega differs from the reference stream after that draw";

// ==================================================================================
// Sub-R-HOSVD
// ==================================================================================
// Synchronises the call and fills the report (achieved ranks come back
// through mapped pinned memory written by the basis kernels).
void finish_tucker(srtt_handle* h, Timer& tm, int d, const std::vector<int64_t>& ranks,
                   const std::vector<int64_t>& samples, double t_sampling, std::vector<std::string>& warnings,
                   srtt_report* rep) {
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaGetLastError());
  const int32_t* hi = h->pset().hinfo();
  for (int k = 0; k < d; ++k) {
    const int q = hi[4 * k];
    if (rep && rep->achieved_ranks) rep->achieved_ranks[k] = q;
    if (q < ranks[k])
      warnings.push_back("mode " + std::to_string(k) + ": sketch revealed rank " + std::to_string(q) +
                         " < target " + std::to_string(ranks[k]) + "; basis padded");
  }
  if (hi[4 * d] & 1) warnings.push_back(kU1ZeroWarning);
  if (rep) {
    if (rep->sample_counts)
      for (int k = 0; k < d; ++k) rep->sample_counts[k] = samples[k];
    std::memset(rep->stage_seconds, 0, sizeof(rep->stage_seconds));
    rep->stage_seconds[SRTT_STAGE_SAMPLING] = t_sampling;
    rep->stage_seconds[SRTT_STAGE_H2D] = tm.between(0, 1);
    rep->stage_seconds[SRTT_STAGE_SKETCH] = tm.between(2, 3);
    rep->stage_seconds[SRTT_STAGE_SVD] = tm.between(3, 4);
    rep->stage_seconds[SRTT_STAGE_TTM] = tm.between(4, 5);
    rep->stage_seconds[SRTT_STAGE_FACTOR_WALL] = t_sampling + tm.between(2, 4);
    rep->stage_seconds[SRTT_STAGE_D2H] = tm.between(5, 6);
    rep->flags = hi[4 * d];
    rep->reserved = 0;  // max Jacobi sweeps over the targets
    for (int k = 0; k < d; ++k) rep->reserved = std::max(rep->reserved, hi[4 * k + 2]);
    rep->kernel_seconds[0] = tm.between(2, 3);
    rep->kernel_seconds[1] = tm.between(3, 4);
    rep->kernel_seconds[2] = d >= 2 ? kernel_pair(h, 2) : 0.0;
    rep->kernel_seconds[3] = 0.0;
    rep->launches = h->launches;
    write_warnings(rep, warnings);
  }
}

// ExecPolicy (parallel.hpp:23-28) semantics on the GPU path. The GPU runs
// every mode / node concurrently and the core pass over all SMs whatever
// `workers` says (the reference's results are bitwise independent of it,
// parallel.hpp:18-21), but the policy is validated exactly as the
// reference's engine does it, with the same messages:
//   run_independent_jobs / tree_schedule: workers >= 1 (parallel.hpp:88, 206)
//   sliced_core: slice mode given -> in range, else pick_slice_mode
//   (parallel.hpp:331-348); workers <= slices along it (parallel.hpp:362-373).
int64_t pick_slice_mode_impl(const std::vector<int64_t>& dims, int64_t workers) {
  int64_t best = -1, best_score = INT64_MAX;
  for (size_t k = 0; k < dims.size(); ++k) {
    const int64_t nk = dims[k];
    if (nk < workers) continue;
    const int64_t rem = nk % workers;
    const int64_t score = rem == 0 ? 0 : workers - rem;
    if (score < best_score) {
      best_score = score;
      best = (int64_t)k;
    }
  }
  if (best < 0) invalid("pick_slice_mode: no mode can host " + std::to_string(workers) + " slices");
  return best;
}

// Ranks above 32 in the first two core modes run as rank blocks (CoreJob);
// nothing to reject up front.
void check_core_ranks(int, const int64_t*, const char*) {}

void check_workers(const srtt_exec_policy* exec, const char* who) {
  if (exec && exec->workers < 1) invalid(std::string(who) + ": workers must be >= 1");
}

// sliced_core's slice-mode resolution (parallel.hpp:369-373); -1 = auto.
int64_t resolve_slice_mode(const std::vector<int64_t>& dims, const srtt_exec_policy* exec) {
  const int64_t d = (int64_t)dims.size();
  const int64_t sm = exec->slice_mode == -1 ? pick_slice_mode_impl(dims, exec->workers) : exec->slice_mode;
  if (sm < 0 || sm >= d) invalid("sliced_core: slice mode out of range");
  if (exec->workers > dims[(size_t)sm]) invalid("sliced_core: more workers than slices along the slicing mode");
  return sm;
}

void run_sub_r_hosvd(srtt_handle* h, const double* x_in, int x_on_device, int d, const int64_t* dims_p,
                     const int64_t* ranks_p, int64_t p, const int64_t* samples_p, uint64_t seed,
                     const srtt_exec_policy* exec, double* core_out, double* const* factors_out,
                     int out_on_device, srtt_report* rep) {
  if (d < 1 || d > SRTT_MAX_ORDER) invalid("sub_r_hosvd: unsupported order");
  std::vector<int64_t> dims(dims_p, dims_p + d), ranks(ranks_p, ranks_p + d), samples(samples_p, samples_p + d);
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) invalid("Shape: dimensions must be >= 1");
  const int64_t N = prod(dims);
  // validation order and messages: tucker.hpp:184-197 (validate_ranks first)
  for (int k = 0; k < d; ++k)
    if (ranks[k] < 1 || ranks[k] > dims[k])
      invalid("sub_r_hosvd: rank out of range in mode " + std::to_string(k));
  for (int k = 0; k < d; ++k) {
    if (samples[k] < ranks[k] + p)
      invalid("sub_r_hosvd: samples below rank + oversampling in mode " + std::to_string(k));
    if (samples[k] > N / dims[k])
      invalid("sub_r_hosvd: more samples than fibers in mode " + std::to_string(k));
  }
  for (int k = 0; k < d; ++k)
    if (ranks[k] + p > SRTT_MAX_SKETCH_COLS)
      invalid("sub_r_hosvd: rank + oversampling above 256 is not supported by the B200 basis kernels");
  check_core_ranks(d, ranks.data(), "sub_r_hosvd");
  std::vector<std::string> warnings;
  if (p < 4) warnings.push_back("oversampling below the recommended minimum of 4");
  const int64_t partitions = exec ? exec->index_partitions : 1;
  check_workers(exec, "run_independent_jobs");  // parallel_factors (tucker.hpp:216)

  DeviceGuard guard(h->device);
  h->launches = 0;
  begin_call(h);
  h->timing = rep != nullptr;  // restored to true when the call returns
  struct TimingReset {
    srtt_handle* h;
    ~TimingReset() { h->timing = true; }
  } timing_reset{h};
  Timer tm{h};

  // --- host sampling: one stream per mode (tucker.hpp:145), JobError(k) on failure
  const double ts0 = now_s();
  std::vector<std::vector<int64_t>> cols(d);
  std::vector<uint64_t> draws(d), state0(d);
  for (int k = 0; k < d; ++k) {
    srtt_host::Stream rng(seed, (uint64_t)k);
    try {
      if (partitions > 1)
        srtt_host::sample_indices_partitioned(N / dims[k], samples[k], partitions, rng, cols[k]);
      else
        srtt_host::sample_indices(N / dims[k], samples[k], rng, cols[k]);
    } catch (const std::exception& e) {
      fail(SRTT_ERR_JOB, "job " + std::to_string(k) + ": " + e.what());
    }
    draws[k] = rng.draws;
    state0[k] = srtt_host::stream_state0(seed, (uint64_t)k);
  }
  const double t_sampling = now_s() - ts0;
  // with a policy the reference assembles the core through sliced_core
  // (tucker.hpp:232-233), whose slice-mode checks come after the factor jobs
  const int64_t slice_mode = exec ? resolve_slice_mode(dims, exec) : -1;
  if (rep) rep->slice_mode = slice_mode;

  tm.mark();  // 0
  const double* x = stage_input(h, x_in, x_on_device, N);
  tm.mark();  // 1 (after H2D)

  // --- fast path: a prepared call with the same signature only needs the
  // seed-dependent blob fields patched and its CUDA graph replayed
  std::string pkey;
  if (h->use_graphs) {
    pkey.reserve(256);
    for (int k = 0; k < d; ++k) {
      pkey += std::to_string(dims[k]);
      pkey += ',';
      pkey += std::to_string(ranks[k]);
      pkey += ',';
      pkey += std::to_string(samples[k]);
      pkey += ',';
      pkey += out_on_device ? ptr_key(factors_out[k]) : "h";
      pkey += '|';
    }
    pkey += std::to_string(p) + "|" + ptr_key(x) + "|" + (out_on_device ? ptr_key(core_out) : "h") + "|" +
            ptr_key(h->stream) + "|" + std::to_string(partitions) + "|" + std::to_string(h->cur) +
            (h->timing ? "|t" : "|n") + ((rep || !out_on_device) ? "|i" : "|o");
    auto pit = h->prepared.find(pkey);
    if (pit != h->prepared.end() && pit->second.ws == h->ws.p && pit->second.dp == h->pset().d.p &&
        pit->second.hp == h->pset().hst.p && h->graphs.count(pit->second.graph_key)) {
      const srtt_handle::Prepared& pr = pit->second;
      if (std::getenv("SRTT_DEBUG_CALLS")) std::fprintf(stderr, "tucker call: prepared graph, set %d\n", h->cur);
      char* hp = reinterpret_cast<char*>(h->pset().hst.p);
      std::memcpy(hp, pr.image.data(), pr.image.size());
      for (int k = 0; k < d; ++k) {
        std::memcpy(hp + pr.off_cols[k], cols[k].data(), sizeof(int64_t) * cols[k].size());
        SketchTarget* skp = reinterpret_cast<SketchTarget*>(hp + pr.off_sk) + k;
        skp->state0 = state0[k];
        skp->draw_offset = draws[k];
        BasisTarget* btp = reinterpret_cast<BasisTarget*>(hp + pr.off_bt) + k;
        btp->state0 = state0[k];
        btp->draw_offset = draws[k];
      }
      tm.n = 2;
      run_enqueue(h, pr.graph_key, [] { fail(SRTT_ERR_INTERNAL, "prepared graph missing"); });
      tm.n = 6;
      if (!out_on_device) {
        copy_out(h, core_out, pr.d_core, sizeof(double) * prod(ranks), 0);
        for (int k = 0; k < d; ++k) copy_out(h, factors_out[k], pr.udev[k], sizeof(double) * dims[k] * ranks[k], 0);
      }
      tm.mark();  // 6
      if (end_call(h, rep || !out_on_device)) finish_tucker(h, tm, d, ranks, samples, t_sampling, warnings, rep);
      return;
    }
  }

  if (std::getenv("SRTT_DEBUG_CALLS")) std::fprintf(stderr, "tucker call: full path, set %d\n", h->cur);
  // --- workspace layout
  Layout L;
  std::vector<size_t> off_z(d), off_u(d), off_zp(d);
  std::vector<BasisPlan> bp(d);
  std::vector<BasisBuffers> bb(d);
  int cmax = 0;
  for (int k = 0; k < d; ++k) {
    const int c = (int)(ranks[k] + p);
    cmax = std::max(cmax, c);
    off_z[k] = L.take(sizeof(double) * dims[k] * c);
    off_zp[k] = L.take(sketch_part_bytes(dims[k], samples[k], c));
    off_u[k] = out_on_device ? 0 : L.take(sizeof(double) * dims[k] * ranks[k]);
    bp[k] = plan_basis(dims[k], c, (int)ranks[k]);
    bb[k] = layout_basis(L, bp[k]);
  }
  const size_t off_core = L.take(sizeof(double) * prod(ranks));
  int64_t max_n = 0;
  for (int k = 0; k < d; ++k) max_n = std::max(max_n, dims[k]);
  const size_t off_pad = L.take(sizeof(double) * max_n * d);
  CoreJob core;
  if (d >= 2) core.plan(dims, ranks, h->sms, L);
  h->ws.ensure(L.off);
  char* ws = reinterpret_cast<char*>(h->ws.p);
  std::vector<double*> uptr(d);
  for (int k = 0; k < d; ++k)
    uptr[k] = out_on_device ? factors_out[k] : reinterpret_cast<double*>(ws + off_u[k]);
  double* d_core = out_on_device ? core_out : reinterpret_cast<double*>(ws + off_core);

  // --- parameter blob (indices, target descriptors, basis lists): one H2D copy
  if (4 * (d + 1) > kInfoInts) invalid("sub_r_hosvd: too many modes");
  // per-target info words + status flags live at the head of the parameter
  // blob: its H2D copy zeroes them every call (no separate memset), they
  // are copied back only for calls that synchronise
  int32_t* const hinfo = h->pset().hinfo();
  const size_t info_bytes = sizeof(int32_t) * 4 * (d + 1);
  const bool need_info = rep || !out_on_device;
  Blob blob;
  const size_t off_info = blob.reserve(info_bytes);
  std::vector<size_t> off_cols(d);
  // dense trailing-mode targets: sorted columns for K1t (changes cols[k])
  std::vector<std::vector<int64_t>> perms(d);
  std::vector<size_t> off_perm(d, 0);
  bool any_trans = false;
  for (int k = 0; k < d; ++k)
    if (sketch_trans_prepare(dims, {k}, samples[k], (int)(ranks[k] + p), cols[k], perms[k])) any_trans = true;
  for (int k = 0; k < d; ++k) off_cols[k] = blob.add(cols[k].data(), sizeof(int64_t) * cols[k].size());
  for (int k = 0; k < d; ++k)
    if (!perms[k].empty()) off_perm[k] = blob.add(perms[k].data(), sizeof(int64_t) * perms[k].size());
  const size_t off_sk = blob.reserve(sizeof(SketchTarget) * d);
  const size_t off_bt = blob.reserve(sizeof(BasisTarget) * d);
  std::vector<SketchTarget> sk(d);
  std::vector<BasisTarget> bt(d);
  int64_t ctas = 0;
  h->pset().d.ensure(blob.lay.off + 4096);
  char* dp = reinterpret_cast<char*>(h->pset().d.p);
  int32_t* const dinfo = reinterpret_cast<int32_t*>(dp + off_info);
  int32_t* d_flags = dinfo + 4 * d;
  for (int k = 0; k < d; ++k) {
    const int c = (int)(ranks[k] + p);
    sk[k] = make_sketch_target(x, dims, {k}, samples[k], c);
    if (!perms[k].empty()) mark_sketch_trans(sk[k], reinterpret_cast<const int64_t*>(dp + off_perm[k]));
    sk[k].cols = reinterpret_cast<const int64_t*>(dp + off_cols[k]);
    sk[k].z = reinterpret_cast<double*>(ws + off_z[k]);
    sk[k].state0 = state0[k];
    sk[k].draw_offset = draws[k];
    sk[k].cta_begin = ctas;
    sk[k].flags = d_flags;
    attach_sketch_scratch(sk[k], ws + off_zp[k]);
    ctas += sketch_target_ctas(sk[k]);
    bt[k] = fill_basis(bp[k], bb[k], ws, sk[k].z, uptr[k], state0[k], draws[k], samples[k] * c, dinfo + 4 * k);
  }
  assign_basis_ctas(bt);
  const BasisLists lists = make_basis_lists(bt, blob);
  h->pset().d.ensure(blob.lay.off);
  h->pset().hst.ensure(blob.lay.off);
  dp = reinterpret_cast<char*>(h->pset().d.p);
  char* hp = reinterpret_cast<char*>(h->pset().hst.p);
  for (auto& it : blob.items) std::memcpy(hp + it.first, it.second.data(), it.second.size());
  std::memset(hp + off_info, 0, info_bytes);
  assign_contig_ctas(sk);
  std::memcpy(hp + off_sk, sk.data(), sizeof(SketchTarget) * d);
  std::memcpy(hp + off_bt, bt.data(), sizeof(BasisTarget) * d);
  std::string key = "T";
  for (int k = 0; k < d; ++k)
    key += "|" + std::to_string(dims[k]) + "," + std::to_string(ranks[k]) + "," + std::to_string(samples[k]) + "," +
           ptr_key(uptr[k]);
  key += "|" + std::to_string(p) + "|" + ptr_key(x) + "|" + ptr_key(d_core) + "|" + ptr_key(ws) + "|" + ptr_key(dp) +
         "|" + ptr_key(hp) + "|" + ptr_key(h->stream) + "|" + std::to_string(blob.lay.off) +
         (h->timing ? "|t" : "|n") + (need_info ? "|i" : "|o");
  run_enqueue(h, key, [&] {
    CK(cudaMemcpyAsync(dp, hp, blob.lay.off, cudaMemcpyHostToDevice, h->stream));
    tm.n = 2;
    tm.mark();  // 2
    // --- K1: grouped gather + sketch over all modes
    h->launches += launch_sketch_group(reinterpret_cast<const SketchTarget*>(dp + off_sk), sk, ctas, cmax, h->stream);
    tm.mark();  // 3
    // --- K2: basis of every sketch
    h->launches += launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(dp + off_bt), lists, dp,
                                      reinterpret_cast<double*>(ws + off_pad), max_n);
    tm.mark();  // 4
    // --- K3: core pass
    std::vector<const double*> ucp(uptr.begin(), uptr.end());
    if (d >= 2) {
      h->launches += core.launch(h, x, ucp, d_core, ws);
    } else {
      TtmParams T{};
      T.in = x;
      T.u = ucp[0];
      T.out = d_core;
      T.g = 1;
      T.n = dims[0];
      T.post = 1;
      T.rr = ranks[0];
      T.transpose = 1;
      T.nparts = 1;
      CK(srtt_launch_ttm(T, h->stream));
      h->launches++;
    }
    tm.mark();  // 5
    if (need_info) CK(cudaMemcpyAsync(hinfo, dinfo, info_bytes, cudaMemcpyDeviceToHost, h->stream));
  });
  tm.n = 6;
  // --- outputs (host destinations only; device outputs were written in place)
  if (!out_on_device) {
    copy_out(h, core_out, d_core, sizeof(double) * prod(ranks), 0);
    for (int k = 0; k < d; ++k) copy_out(h, factors_out[k], uptr[k], sizeof(double) * dims[k] * ranks[k], 0);
  }
  tm.mark();  // 6
  if (h->use_graphs && !any_trans) {  // K1t signatures re-sort per seed: no fast path
    srtt_handle::Prepared pr;
    pr.image.assign(hp, hp + blob.lay.off);
    pr.off_cols = off_cols;
    pr.off_sk = off_sk;
    pr.off_bt = off_bt;
    pr.graph_key = key;
    pr.ws = h->ws.p;
    pr.dp = h->pset().d.p;
    pr.hp = h->pset().hst.p;
    pr.udev.assign(uptr.begin(), uptr.end());
    pr.d_core = d_core;
    if (h->prepared.size() > 64) h->prepared.clear();
    h->prepared[pkey] = std::move(pr);
  }
  if (end_call(h, rep || !out_on_device)) finish_tucker(h, tm, d, ranks, samples, t_sampling, warnings, rep);
}

void release_comm(srtt_handle* h);  // shard.cuh

}  // namespace

// ==================================================================================
// C-ABI
// ==================================================================================
extern "C" {

const char* srtt_last_error(void) { return g_last_error.c_str(); }
int srtt_version(void) { return 100; }

// Development / test aid (no GPU needed): the K2 plan of an n x c sketch with
// target rank r. out[0] = kernel family (0 shared-memory QR, 1 register
// tree, 2 wide register teams, 3 generic), out[1] = levels below the top,
// out[2] = CTAs at level 0, out[3] = rows per level-0 CTA, out[4] = rows of
// the top block.
int srtt_debug_basis_plan(int64_t n, int32_t c, int32_t r, int64_t* out) {
  return guarded([&] {
    if (!out || n < 1 || c < 1 || r < 1 || r > c) invalid("srtt_debug_basis_plan: bad arguments");
    const BasisPlan b = plan_basis(n, c, r);
    out[0] = b.kind;
    out[1] = b.nlevels;
    out[2] = b.lv_nblk[0];
    out[3] = b.lv_blk[0];
    out[4] = b.lv_n[b.nlevels];
  });
}

int srtt_create(const srtt_options* opts, srtt_handle** out) {
  return guarded([&] {
    if (!out) invalid("srtt_create: null output");
    auto h = std::make_unique<srtt_handle>();
    h->device = opts ? opts->device : 0;
    h->use_graphs = opts ? opts->use_graphs : 0;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (h->device < 0 || h->device >= ndev) invalid("srtt_create: no such CUDA device");
    DeviceGuard g(h->device);
    CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device));
    int major = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device));
    if (major != 10) fail(SRTT_ERR_CUDA, "srtt: this build targets sm_100a (B200) only");
    CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    for (auto& e : h->fj) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& ps : h->psets) CK(cudaEventCreateWithFlags(&ps.done, cudaEventDisableTiming));
    h->stream = h->own_stream;
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
    for (auto& e : h->kev) CK(cudaEventCreate(&e));
    for (auto& ps : h->psets) {
      ps.info.ensure(kInfoInts * sizeof(int32_t));
      ps.hinfo_buf.ensure(kInfoInts * sizeof(int32_t));
      std::memset(ps.hinfo_buf.p, 0, kInfoInts * sizeof(int32_t));
    }
    h->ones.ensure(sizeof(double));
    const double one = 1.0;
    CK(cudaMemcpy(h->ones.p, &one, sizeof(double), cudaMemcpyHostToDevice));
    *out = h.release();
  });
}

int srtt_destroy(srtt_handle* h) {
  return guarded([&] {
    if (!h) return;
    {
      DeviceGuard g(h->device);
      cudaStreamSynchronize(h->stream);
      if (h->comm) release_comm(h);
      for (auto& e : h->ev) cudaEventDestroy(e);
      for (auto& e : h->kev) cudaEventDestroy(e);
      cudaStreamDestroy(h->own_stream);
      cudaStreamDestroy(h->side);
      for (auto& e : h->fj) cudaEventDestroy(e);
      for (auto& ps : h->psets) cudaEventDestroy(ps.done);
    }
    delete h;
  });
}

int64_t srtt_last_launch_count(srtt_handle* h) { return h ? h->launches : -1; }

int srtt_set_stream(srtt_handle* h, void* stream) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    h->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : h->own_stream;
  });
}

int srtt_sample_indices(uint64_t seed, uint64_t stream_id, int64_t m, int64_t s, int64_t partitions,
                        int64_t* idx_out, uint64_t* draws_out) {
  return guarded([&] {
    srtt_host::Stream rng(seed, stream_id);
    std::vector<int64_t> out;
    if (partitions > 1 || partitions < 1)
      srtt_host::sample_indices_partitioned(m, s, partitions, rng, out);
    else
      srtt_host::sample_indices(m, s, rng, out);
    std::memcpy(idx_out, out.data(), sizeof(int64_t) * out.size());
    if (draws_out) *draws_out = rng.draws;
  });
}

int srtt_pick_slice_mode(int32_t d, const int64_t* dims, int64_t workers, int64_t* mode_out) {
  return guarded([&] {
    if (d < 1 || !dims) invalid("pick_slice_mode: empty shape");
    const int64_t m = pick_slice_mode_impl(std::vector<int64_t>(dims, dims + d), workers);
    if (mode_out) *mode_out = m;
  });
}

int srtt_tree_balanced(int32_t order, int32_t* num_nodes, int32_t* mode_begin, int32_t* modes,
                       int32_t* left, int32_t* right, int32_t* parent, int32_t* level) {
  return guarded([&] {
    if (order < 2) invalid("DimensionTree: order must be >= 2");
    struct N {
      std::vector<int32_t> m;
      int32_t l = -1, r = -1, p = -1, lv = 0;
    };
    std::vector<N> nodes;
    N root;
    for (int k = 0; k < order; ++k) root.m.push_back(k);
    nodes.push_back(root);
    std::vector<int> queue{0};
    for (size_t qi = 0; qi < queue.size(); ++qi) {
      const int id = queue[qi];
      if (nodes[id].m.size() == 1) continue;
      const size_t half = (nodes[id].m.size() + 1) / 2;
      N a, b;
      a.m.assign(nodes[id].m.begin(), nodes[id].m.begin() + half);
      b.m.assign(nodes[id].m.begin() + half, nodes[id].m.end());
      a.p = b.p = id;
      a.lv = b.lv = nodes[id].lv + 1;
      const int li = (int)nodes.size();
      nodes.push_back(a);
      const int ri = (int)nodes.size();
      nodes.push_back(b);
      nodes[id].l = li;
      nodes[id].r = ri;
      queue.push_back(li);
      queue.push_back(ri);
    }
    *num_nodes = (int32_t)nodes.size();
    int32_t pos = 0;
    for (size_t i = 0; i < nodes.size(); ++i) {
      mode_begin[i] = pos;
      for (int32_t m : nodes[i].m) modes[pos++] = m;
      left[i] = nodes[i].l;
      right[i] = nodes[i].r;
      if (parent) parent[i] = nodes[i].p;
      if (level) level[i] = nodes[i].lv;
    }
    mode_begin[nodes.size()] = pos;
  });
}

int srtt_sub_r_hosvd(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                     const int64_t* ranks, int64_t oversampling, const int64_t* samples, uint64_t seed,
                     const srtt_exec_policy* exec, double* core_out, double* const* factors_out,
                     int32_t out_on_device, srtt_report* rep) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    run_sub_r_hosvd(h, x, x_on_device, d, dims, ranks, oversampling, samples, seed, exec, core_out,
                    factors_out, out_on_device, rep);
  });
}

}  // extern "C"

cudaError_t srtt_launch_normals(uint64_t, uint64_t, uint64_t, int64_t, double*, cudaStream_t);

namespace {

// ==================================================================================
// Dimension tree (dimension_tree.hpp:27-152) as seen through srtt_tree
// ==================================================================================
struct Tree {
  int n = 0;
  std::vector<std::vector<int>> modes;
  std::vector<int> left, right, parent, level;
  bool leaf(int i) const { return left[i] < 0; }
};

Tree read_tree(const srtt_tree* t, int d) {
  if (!t || t->num_nodes < 1) invalid("DimensionTree: empty");
  Tree T;
  T.n = t->num_nodes;
  T.modes.resize(T.n);
  T.left.assign(t->left, t->left + T.n);
  T.right.assign(t->right, t->right + T.n);
  T.parent.assign(T.n, -1);
  T.level.assign(T.n, 0);
  for (int i = 0; i < T.n; ++i) {
    for (int k = t->mode_begin[i]; k < t->mode_begin[i + 1]; ++k) T.modes[i].push_back(t->modes[k]);
    std::sort(T.modes[i].begin(), T.modes[i].end());
  }
  const int order = (int)T.modes[0].size();
  if (order < 2) invalid("DimensionTree: order must be >= 2");
  for (int k = 0; k < order; ++k)
    if (T.modes[0][k] != k) invalid("DimensionTree: root must hold modes 0..d-1");
  int leaves = 0;
  for (int i = 0; i < T.n; ++i) {
    if ((T.left[i] < 0) != (T.right[i] < 0)) invalid("DimensionTree: node must have zero or two children");
    if (T.leaf(i)) {
      if (T.modes[i].size() != 1) invalid("DimensionTree: leaves must hold a single mode");
      ++leaves;
      continue;
    }
    if (T.left[i] >= T.n || T.right[i] >= T.n) invalid("DimensionTree: child index out of range");
    const auto& l = T.modes[T.left[i]];
    const auto& r = T.modes[T.right[i]];
    if (l.size() + r.size() != T.modes[i].size()) invalid("DimensionTree: children do not partition the node");
    if (l.back() >= r.front()) invalid("DimensionTree: left child modes must precede right child modes");
    std::vector<int> merged = l;
    merged.insert(merged.end(), r.begin(), r.end());
    if (merged != T.modes[i]) invalid("DimensionTree: children do not partition the node");
    T.parent[T.left[i]] = i;
    T.parent[T.right[i]] = i;
  }
  if (leaves != order) invalid("DimensionTree: expected one leaf per mode");
  if (order != d) invalid("sub_r_rtl_ht: tree and tensor order mismatch");
  return T;
}

// ==================================================================================
// Sub-R-RtL-HT
// ==================================================================================
void run_sub_r_rtl_ht(srtt_handle* h, const double* x_in, int x_on_device, int d, const int64_t* dims_p,
                      const srtt_tree* tree_p, const int64_t* ranks_p, const int64_t* samples_p, int64_t p,
                      uint64_t seed, const srtt_exec_policy* exec, double* const* leaf_out,
                      double* const* transfers_out, int out_on_device, srtt_report* rep) {
  if (d < 2 || d > SRTT_MAX_ORDER) invalid("sub_r_rtl_ht: unsupported order");
  std::vector<int64_t> dims(dims_p, dims_p + d);
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) invalid("Shape: dimensions must be >= 1");
  const Tree tr = read_tree(tree_p, d);
  const int nn = tr.n;
  std::vector<int64_t> ranks(ranks_p, ranks_p + nn), samples(samples_p, samples_p + nn);
  const int64_t N = prod(dims);
  auto node_rows = [&](int i) {
    int64_t r = 1;
    for (int m : tr.modes[i]) r *= dims[m];
    return r;
  };
  // validate_node_ranks (htucker.hpp:109-121), then the sample budgets (:223-233)
  if (ranks[0] != 1) invalid("sub_r_rtl_ht: root rank must be 1");
  for (int i = 1; i < nn; ++i) {
    const int64_t mx = std::min(node_rows(i), N / node_rows(i));
    if (ranks[i] < 1 || ranks[i] > mx) invalid("sub_r_rtl_ht: rank out of range at node " + std::to_string(i));
  }
  for (int i = 1; i < nn; ++i) {
    if (samples[i] < ranks[i] + p)
      invalid("sub_r_rtl_ht: samples below rank + oversampling at node " + std::to_string(i));
    if (samples[i] > N / node_rows(i))
      invalid("sub_r_rtl_ht: more samples than fibers at node " + std::to_string(i));
  }
  for (int i = 1; i < nn; ++i)
    if (ranks[i] + p > SRTT_MAX_SKETCH_COLS)
      invalid("sub_r_rtl_ht: rank + oversampling above 256 is not supported by the B200 basis kernels");
  for (int i = 1; i < nn; ++i)
    if (ranks[i] > 64) invalid("sub_r_rtl_ht: node ranks above 64 are not supported by the B200 transfer kernel");
  {
    const int64_t rr[2] = {ranks[tr.left[0]], ranks[tr.right[0]]};
    check_core_ranks(2, rr, "sub_r_rtl_ht");
  }
  std::vector<std::string> warnings;
  if (p < 4) warnings.push_back("oversampling below the recommended minimum of 4");
  const int64_t partitions = exec ? exec->index_partitions : 1;
  check_workers(exec, "tree_schedule");  // parallel.hpp:206
  const bool serial_root = exec && exec->emulate_serial_root;

  DeviceGuard guard(h->device);
  h->launches = 0;
  begin_call(h);
  h->timing = rep != nullptr;  // restored to true when the call returns
  struct TimingReset {
    srtt_handle* h;
    ~TimingReset() { h->timing = true; }
  } timing_reset{h};
  Timer tm{h};
  tm.mark();  // 0
  const double* x = stage_input(h, x_in, x_on_device, N);
  tm.mark();  // 1
  if (rep) rep->slice_mode = -1;

  const int nt = nn - 1;  // one basis target per non-root node (ids 1..nn-1)
  const double ts0 = now_s();
  std::vector<std::vector<int64_t>> cols(nt);
  std::vector<uint64_t> draws(nt), state0(nt);
  for (int t = 0; t < nt; ++t) {
    const int id = t + 1;
    srtt_host::Stream rng(seed, (uint64_t)id);
    const int64_t m = N / node_rows(id);
    try {
      if (partitions > 1)
        srtt_host::sample_indices_partitioned(m, samples[id], partitions, rng, cols[t]);
      else
        srtt_host::sample_indices(m, samples[id], rng, cols[t]);
    } catch (const std::exception& e) {
      fail(SRTT_ERR_JOB, "job " + std::to_string(t) + ": " + e.what());
    }
    draws[t] = rng.draws;
    state0[t] = srtt_host::stream_state0(seed, (uint64_t)id);
  }
  const double t_sampling = now_s() - ts0;

  Layout L;
  std::vector<size_t> off_z(nt), off_u(nt), off_zp(nt);
  std::vector<BasisPlan> bp(nt);
  std::vector<BasisBuffers> bb(nt);
  int cmax = 0;
  int64_t max_n = 0;
  for (int t = 0; t < nt; ++t) {
    const int id = t + 1;
    const int c = (int)(ranks[id] + p);
    const int64_t rows = node_rows(id);
    cmax = std::max(cmax, c);
    max_n = std::max(max_n, rows);
    off_z[t] = L.take(sizeof(double) * rows * c);
    off_zp[t] = L.take(sketch_part_bytes(rows, samples[id], c));
    off_u[t] = L.take(sizeof(double) * rows * ranks[id]);
    bp[t] = plan_basis(rows, c, (int)ranks[id]);
    bb[t] = layout_basis(L, bp[t]);
  }
  const size_t off_pad = L.take(sizeof(double) * max_n * nt);
  if (4 * (nt + 1) > kInfoInts) invalid("sub_r_rtl_ht: too many tree nodes");
  const int32_t* hi = h->pset().hinfo();
  const size_t info_bytes = sizeof(int32_t) * 4 * (nt + 1);
  const bool need_info = rep || !out_on_device;
  // transfers of internal non-root nodes, and the root
  std::vector<int> internal;
  for (int i = 1; i < nn; ++i)
    if (!tr.leaf(i)) internal.push_back(i);
  std::vector<size_t> off_b(nn, 0);
  for (int i : internal)
    off_b[i] = L.take(sizeof(double) * ranks[i] * ranks[tr.left[i]] * ranks[tr.right[i]]);
  const int rl0 = (int)ranks[tr.left[0]], rr0 = (int)ranks[tr.right[0]];
  off_b[0] = L.take(sizeof(double) * rl0 * rr0);
  const std::vector<int64_t> rdims = {node_rows(tr.left[0]), node_rows(tr.right[0])};
  const std::vector<int64_t> rranks = {rl0, rr0};
  CoreJob core;
  core.plan(rdims, rranks, h->sms, L);
  h->ws.ensure(L.off);
  char* ws = reinterpret_cast<char*>(h->ws.p);

  Blob blob;
  const size_t off_info = blob.reserve(info_bytes);  // zeroed by the blob copy (see sub_r_hosvd)
  std::vector<size_t> off_cols(nt);
  std::vector<std::vector<int64_t>> perms(nt);
  std::vector<size_t> off_perm(nt, 0);
  for (int t = 0; t < nt; ++t)
    sketch_trans_prepare(dims, tr.modes[t + 1], samples[t + 1], (int)(ranks[t + 1] + p), cols[t], perms[t]);
  for (int t = 0; t < nt; ++t) off_cols[t] = blob.add(cols[t].data(), sizeof(int64_t) * cols[t].size());
  for (int t = 0; t < nt; ++t)
    if (!perms[t].empty()) off_perm[t] = blob.add(perms[t].data(), sizeof(int64_t) * perms[t].size());
  const size_t off_sk = blob.reserve(sizeof(SketchTarget) * nt);
  const size_t off_bt = blob.reserve(sizeof(BasisTarget) * nt);
  const size_t off_tt = blob.reserve(sizeof(TransferTarget) * std::max<size_t>(1, internal.size()));
  h->pset().d.ensure(blob.lay.off + 4096);
  char* dp = reinterpret_cast<char*>(h->pset().d.p);
  int32_t* const dinfo = reinterpret_cast<int32_t*>(dp + off_info);
  int32_t* d_flags = dinfo + 4 * nt;
  std::vector<SketchTarget> sk(nt);
  std::vector<BasisTarget> bt(nt);
  int64_t ctas = 0;
  auto ubasis = [&](int id) {
    if (out_on_device && tr.leaf(id)) return leaf_out[tr.modes[id][0]];
    return reinterpret_cast<double*>(ws + off_u[id - 1]);
  };
  for (int t = 0; t < nt; ++t) {
    const int id = t + 1;
    const int c = (int)(ranks[id] + p);
    sk[t] = make_sketch_target(x, dims, tr.modes[id], samples[id], c);
    if (!perms[t].empty()) mark_sketch_trans(sk[t], reinterpret_cast<const int64_t*>(dp + off_perm[t]));
    sk[t].cols = reinterpret_cast<const int64_t*>(dp + off_cols[t]);
    sk[t].z = reinterpret_cast<double*>(ws + off_z[t]);
    sk[t].state0 = state0[t];
    sk[t].draw_offset = draws[t];
    sk[t].cta_begin = ctas;
    sk[t].flags = d_flags;
    attach_sketch_scratch(sk[t], ws + off_zp[t]);
    ctas += sketch_target_ctas(sk[t]);
    bt[t] = fill_basis(bp[t], bb[t], ws, sk[t].z, ubasis(id), state0[t], draws[t], samples[id] * c,
                       dinfo + 4 * t);
  }
  assign_basis_ctas(bt);
  const BasisLists lists = make_basis_lists(bt, blob);
  h->pset().d.ensure(blob.lay.off);
  h->pset().hst.ensure(blob.lay.off);
  char* hp = reinterpret_cast<char*>(h->pset().hst.p);
  for (auto& it : blob.items) std::memcpy(hp + it.first, it.second.data(), it.second.size());
  std::vector<TransferTarget> tt;
  int tctas = 0, max_rl = 1, max_rr = 1;
  for (int i : internal) {
    TransferTarget T{};
    T.us = ubasis(i);
    T.ul = ubasis(tr.left[i]);
    T.ur = ubasis(tr.right[i]);
    T.b = (out_on_device && transfers_out && transfers_out[i]) ? transfers_out[i]
                                                               : reinterpret_cast<double*>(ws + off_b[i]);
    T.nl = node_rows(tr.left[i]);
    T.nr = node_rows(tr.right[i]);
    T.rs = (int)ranks[i];
    T.rl = (int)ranks[tr.left[i]];
    T.rr = (int)ranks[tr.right[i]];
    T.cta_begin = tctas;
    tctas += T.rs;
    max_rl = std::max(max_rl, T.rl);
    max_rr = std::max(max_rr, T.rr);
    tt.push_back(T);
  }
  std::memset(hp + off_info, 0, info_bytes);
  assign_contig_ctas(sk);
  std::memcpy(hp + off_sk, sk.data(), sizeof(SketchTarget) * nt);
  std::memcpy(hp + off_bt, bt.data(), sizeof(BasisTarget) * nt);
  if (!tt.empty()) std::memcpy(hp + off_tt, tt.data(), sizeof(TransferTarget) * tt.size());
  std::string key = "H";
  for (int k = 0; k < d; ++k) key += "|" + std::to_string(dims[k]);
  for (int i = 0; i < nn; ++i)
    key += "|" + std::to_string(ranks[i]) + "," + std::to_string(samples[i]) + "," + std::to_string(tr.left[i]) + "," +
           std::to_string(tr.modes[i].size());
  key += "|" + std::to_string(p) + "|" + ptr_key(x) + "|" + ptr_key(ws) + "|" + ptr_key(dp) + "|" + ptr_key(hp) + "|" +
         ptr_key(h->stream) + "|" + std::to_string(blob.lay.off) + "|" + std::to_string(out_on_device) +
         (serial_root ? "|s" : "|p") + (h->timing ? "|t" : "|n") + (need_info ? "|i" : "|o");
  if (out_on_device) {
    for (int k = 0; k < d; ++k) key += "|" + ptr_key(leaf_out[k]);
    if (transfers_out)
      for (int i = 0; i < nn; ++i) key += "|" + ptr_key(transfers_out[i]);
  }
  double* d_root = (out_on_device && transfers_out && transfers_out[0]) ? transfers_out[0]
                                                                       : reinterpret_cast<double*>(ws + off_b[0]);
  // Small-node bases and the transfer tensors run on a side stream and
  // overlap the root pass, which only needs the root children's bases
  // (htucker.hpp:203-209: the root waits only for nodes 1 and 2).
  // emulate_serial_root: the root also waits for every basis job
  // (parallel.hpp:168-170), i.e. for the side stream's small bases too
  bool root_needs_small = serial_root;
  for (int i : lists.small)
    if (i + 1 == tr.left[0] || i + 1 == tr.right[0]) root_needs_small = true;
  run_enqueue(h, key, [&] {
    tm.n = 2;
    CK(cudaMemcpyAsync(dp, hp, blob.lay.off, cudaMemcpyHostToDevice, h->stream));
    tm.mark();  // 2
    h->launches += launch_sketch_group(reinterpret_cast<const SketchTarget*>(dp + off_sk), sk, ctas, cmax, h->stream);
    tm.mark();  // 3
    // fork: side stream takes the small targets
    CK(cudaEventRecord(h->fj[0], h->stream));
    CK(cudaStreamWaitEvent(h->side, h->fj[0], 0));
    h->launches += launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(dp + off_bt), lists, dp,
                                      reinterpret_cast<double*>(ws + off_pad), max_n, h->side);
    CK(cudaEventRecord(h->fj[1], h->side));  // small bases done
    tm.mark();  // 4: big bases done (main stream)
    CK(cudaEventRecord(h->fj[2], h->stream));
    // side: transfers need every basis
    CK(cudaStreamWaitEvent(h->side, h->fj[2], 0));
    if (!tt.empty()) {
      CK(srtt_launch_transfer(reinterpret_cast<const TransferTarget*>(dp + off_tt), (int)tt.size(), tctas, max_rl,
                              max_rr, h->side));
      h->launches++;
    }
    CK(cudaEventRecord(h->fj[3], h->side));
    // main: root transfer, the K3 engine on M = X viewed as n_l x n_r (htucker.hpp:67-85)
    if (root_needs_small) CK(cudaStreamWaitEvent(h->stream, h->fj[1], 0));
    tm.mark();  // 5
    std::vector<const double*> ur = {ubasis(tr.left[0]), ubasis(tr.right[0])};
    h->launches += core.launch(h, x, ur, d_root, ws);
    // join
    CK(cudaStreamWaitEvent(h->stream, h->fj[3], 0));
    tm.mark();  // 6
    if (need_info) CK(cudaMemcpyAsync(const_cast<int32_t*>(hi), dinfo, info_bytes, cudaMemcpyDeviceToHost, h->stream));
  });
  tm.n = 7;
  if (!out_on_device) {
    for (int i = 1; i < nn; ++i)
      if (tr.leaf(i)) {
        const int mode = tr.modes[i][0];
        copy_out(h, leaf_out[mode], ubasis(i), sizeof(double) * dims[mode] * ranks[i], 0);
      }
    if (transfers_out) {
      for (int i : internal)
        if (transfers_out[i])
          copy_out(h, transfers_out[i], ws + off_b[i],
                   sizeof(double) * ranks[i] * ranks[tr.left[i]] * ranks[tr.right[i]], 0);
      if (transfers_out[0]) copy_out(h, transfers_out[0], d_root, sizeof(double) * rl0 * rr0, 0);
    }
  }
  if (rep && rep->node_bases)
    for (int i = 1; i < nn; ++i)
      if (rep->node_bases[i])
        copy_out(h, rep->node_bases[i], ubasis(i), sizeof(double) * node_rows(i) * ranks[i], out_on_device);
  tm.mark();  // 7
  // device outputs and no report: stream-ordered, return without waiting
  // (the next call's host work overlaps this one's kernels)
  if (!end_call(h, !out_on_device || rep != nullptr)) {
    CK(cudaGetLastError());
    return;
  }
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaGetLastError());
  for (int t = 0; t < nt; ++t) {
    const int id = t + 1;
    const int q = hi[4 * t];
    if (rep && rep->achieved_ranks) rep->achieved_ranks[id] = q;
    if (q < ranks[id])
      warnings.push_back("node " + std::to_string(id) + ": sketch revealed rank " + std::to_string(q) +
                         " < target; basis padded");
  }
  if (hi[4 * nt] & 1) warnings.push_back(kU1ZeroWarning);
  if (rep) {
    if (rep->achieved_ranks) rep->achieved_ranks[0] = 1;
    if (rep->sample_counts)
      for (int i = 0; i < nn; ++i) rep->sample_counts[i] = samples[i];
    std::memset(rep->stage_seconds, 0, sizeof(rep->stage_seconds));
    rep->stage_seconds[SRTT_STAGE_SAMPLING] = t_sampling;
    rep->stage_seconds[SRTT_STAGE_H2D] = tm.between(0, 1);
    rep->stage_seconds[SRTT_STAGE_SKETCH] = tm.between(2, 3);
    rep->stage_seconds[SRTT_STAGE_SVD] = tm.between(3, 4);
    rep->stage_seconds[SRTT_STAGE_TRANSFER] = 0.0;  // overlapped with the root pass (side stream)
    rep->stage_seconds[SRTT_STAGE_SERIAL_TAIL] = tm.between(5, 6);
    rep->stage_seconds[SRTT_STAGE_FACTOR_WALL] = t_sampling + tm.between(2, 4);
    rep->stage_seconds[SRTT_STAGE_D2H] = tm.between(6, 7);
    rep->flags = hi[4 * nt];
    rep->reserved = 0;
    for (int t = 0; t < nt; ++t) rep->reserved = std::max(rep->reserved, hi[4 * t + 2]);
    rep->kernel_seconds[0] = tm.between(2, 3);
    rep->kernel_seconds[1] = tm.between(3, 4);
    rep->kernel_seconds[2] = kernel_pair(h, 2);
    rep->kernel_seconds[3] = 0.0;
    rep->launches = h->launches;
    write_warnings(rep, warnings);
  }
}

// ---- helpers for component entry points ------------------------------------
struct Scratch {  // device copies of small host inputs for component calls
  srtt_handle* h;
  std::vector<std::pair<const void*, size_t>> pending;
};

const double* to_device(srtt_handle* h, DevBuf& buf, const double* src, int64_t count, int on_device) {
  if (on_device) return src;
  buf.ensure(sizeof(double) * std::max<int64_t>(count, 1));
  CK(cudaMemcpyAsync(buf.p, src, sizeof(double) * count, cudaMemcpyHostToDevice, h->stream));
  return reinterpret_cast<const double*>(buf.p);
}

struct CompBufs {
  DevBuf a, b, c, d, e, idx;
};
// The handle's persistent scratch for calls that synchronise before they
// return (no cudaMalloc / cudaFree per call: a free synchronises the device
// and an allocation costs milliseconds).
struct CompRef {
  DevBuf &a, &b, &c, &d, &e, &idx;
};
CompRef comp_bufs(srtt_handle* h) { return {h->comp[0], h->comp[1], h->comp[2], h->comp[3], h->comp[4], h->comp[5]}; }

void validate_modes(int d, const int64_t* dims, int nmodes, const int32_t* modes, const char* what) {
  if (nmodes < 1) invalid("ModeSet: must be non-empty");
  std::vector<int> m(modes, modes + nmodes);
  std::sort(m.begin(), m.end());
  if (std::adjacent_find(m.begin(), m.end()) != m.end()) invalid("ModeSet: modes must be distinct");
  if (m.front() < 0) invalid("ModeSet: modes must be >= 0");
  if (m.back() >= d) invalid("ModeSet: mode out of range for order " + std::to_string(d));
  if (nmodes >= d && nmodes > 1) invalid(std::string(what) + ": mode set must be a proper subset");
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) invalid("Shape: dimensions must be >= 1");
}

}  // namespace

extern "C" {

int srtt_sub_r_rtl_ht(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                      const srtt_tree* tree, const int64_t* ranks, const int64_t* samples, int64_t oversampling,
                      uint64_t seed, const srtt_exec_policy* exec, double* const* leaf_factors_out,
                      double* const* transfers_out, int32_t out_on_device, srtt_report* rep) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    run_sub_r_rtl_ht(h, x, x_on_device, d, dims, tree, ranks, samples, oversampling, seed, exec, leaf_factors_out,
                     transfers_out, out_on_device, rep);
  });
}

int srtt_stream_normals(srtt_handle* h, uint64_t seed, uint64_t stream_id, uint64_t draw_offset, uint64_t t0,
                        int64_t n, double* out) {
  return guarded([&] {
    DeviceGuard g(h->device);
    CompBufs B;
    B.a.ensure(sizeof(double) * std::max<int64_t>(n, 1));
    CK(srtt_launch_normals(srtt_host::stream_state0(seed, stream_id), draw_offset, t0, n,
                           reinterpret_cast<double*>(B.a.p), h->stream));
    CK(cudaMemcpyAsync(out, B.a.p, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_extract_fibers(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                        int32_t nmodes, const int32_t* modes, int64_t ncols, const int64_t* cols, double* y_out,
                        int32_t out_on_device) {
  return guarded([&] {
    const char* what = nmodes == 1 ? "extract_fibers" : "extract_group_fibers";
    validate_modes(d, dims, nmodes, modes, what);
    std::vector<int64_t> dv(dims, dims + d);
    const int64_t N = prod(dv);
    std::vector<int> mv(modes, modes + nmodes);
    SketchTarget T = make_sketch_target(nullptr, dv, mv, ncols, 1);
    const int64_t total_cols = N / T.rows;
    for (int64_t j = 0; j < ncols; ++j)
      if (cols[j] < 0 || cols[j] >= total_cols)
        throw std::out_of_range(std::string(what) + ": column index out of range");
    DeviceGuard g(h->device);
    CompBufs B;
    const double* dx = to_device(h, B.a, x, N, x_on_device);
    B.idx.ensure(sizeof(int64_t) * std::max<int64_t>(ncols, 1));
    CK(cudaMemcpyAsync(B.idx.p, cols, sizeof(int64_t) * ncols, cudaMemcpyHostToDevice, h->stream));
    double* dy = y_out;
    if (!out_on_device) {
      B.b.ensure(sizeof(double) * std::max<int64_t>(T.rows * ncols, 1));
      dy = reinterpret_cast<double*>(B.b.p);
    }
    GatherParams P{};
    P.x = dx;
    P.cols = reinterpret_cast<const int64_t*>(B.idx.p);
    P.y = dy;
    P.rows = T.rows;
    P.w = ncols;
    P.nrow_modes = T.nrow_modes;
    P.ncol_modes = T.ncol_modes;
    std::memcpy(P.row_dim, T.row_dim, sizeof(P.row_dim));
    std::memcpy(P.row_stride, T.row_stride, sizeof(P.row_stride));
    std::memcpy(P.col_dim, T.col_dim, sizeof(P.col_dim));
    std::memcpy(P.col_stride, T.col_stride, sizeof(P.col_stride));
    if (T.rows * ncols > 0) CK(srtt_launch_gather(P, h->stream));
    if (!out_on_device)
      CK(cudaMemcpyAsync(y_out, dy, sizeof(double) * T.rows * ncols, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_sketch(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                int32_t nmodes, const int32_t* modes, int64_t ncols, const int64_t* cols, int32_t c, uint64_t seed,
                uint64_t stream_id, uint64_t draw_offset, const double* omega, double* z_out,
                int32_t out_on_device) {
  return guarded([&] {
    validate_modes(d, dims, nmodes, modes, "extract_group_fibers");
    if (c < 1 || c > SRTT_MAX_SKETCH_COLS) invalid("sketch: columns out of range");
    std::vector<int64_t> dv(dims, dims + d);
    const int64_t N = prod(dv);
    std::vector<int> mv(modes, modes + nmodes);
    DeviceGuard g(h->device);
    CompBufs B;
    const double* dx = to_device(h, B.a, x, N, x_on_device);
    SketchTarget T = make_sketch_target(dx, dv, mv, ncols, c);
    for (int64_t j = 0; j < ncols; ++j)
      if (cols[j] < 0 || cols[j] >= N / T.rows) throw std::out_of_range("extract_fibers: column index out of range");
    std::vector<int64_t> cv(cols, cols + ncols), perm;
    const bool trans = !omega && sketch_trans_prepare(dv, mv, ncols, c, cv, perm);
    B.idx.ensure(sizeof(int64_t) * std::max<int64_t>(2 * ncols, 1));
    CK(cudaMemcpyAsync(B.idx.p, cv.data(), sizeof(int64_t) * ncols, cudaMemcpyHostToDevice, h->stream));
    T.cols = reinterpret_cast<const int64_t*>(B.idx.p);
    if (trans) {
      CK(cudaMemcpyAsync(reinterpret_cast<int64_t*>(B.idx.p) + ncols, perm.data(), sizeof(int64_t) * ncols,
                         cudaMemcpyHostToDevice, h->stream));
      mark_sketch_trans(T, reinterpret_cast<const int64_t*>(B.idx.p) + ncols);
    }
    if (omega) T.omega = to_device(h, B.c, omega, ncols * c, 0);
    B.b.ensure(sizeof(double) * T.rows * c + 256 + sketch_part_bytes(T.rows, ncols, c));
    T.z = reinterpret_cast<double*>(B.b.p);
    T.state0 = srtt_host::stream_state0(seed, stream_id);
    T.draw_offset = draw_offset;
    attach_sketch_scratch(T, reinterpret_cast<char*>(B.b.p) + (sizeof(double) * T.rows * c + 255) / 256 * 256);
    B.e.ensure(sizeof(int32_t) * 4 + sizeof(SketchTarget));
    T.flags = reinterpret_cast<int32_t*>(B.e.p);
    CK(cudaMemsetAsync(T.flags, 0, sizeof(int32_t) * 4, h->stream));
    T.cta_begin = 0;
    SketchTarget* dT = reinterpret_cast<SketchTarget*>(reinterpret_cast<char*>(B.e.p) + 64);
    B.d.ensure(sizeof(SketchTarget));
    dT = reinterpret_cast<SketchTarget*>(B.d.p);
    {
      std::vector<SketchTarget> one = {T};
      assign_contig_ctas(one);
      T = one[0];
    }
    CK(cudaMemcpyAsync(dT, &T, sizeof(T), cudaMemcpyHostToDevice, h->stream));
    launch_sketch_group(dT, {T}, sketch_target_ctas(T), c, h->stream);
    copy_out(h, z_out, T.z, sizeof(double) * T.rows * c, out_on_device);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_range_basis_of_sketch(srtt_handle* h, const double* z, int32_t z_on_device, int64_t n, int32_t c,
                               int32_t rank, uint64_t seed, uint64_t stream_id, uint64_t draw_offset,
                               int64_t normal_base, double* q_out, int64_t* numerical_rank, double* sv_out,
                               int32_t out_on_device) {
  return guarded([&] {
    if (rank < 1 || rank > c) invalid("range_basis_of_sketch: rank out of range");
    if (c > SRTT_MAX_SKETCH_COLS) invalid("range_basis_of_sketch: more than 256 sketch columns unsupported");
    if (n < 1) invalid("range_basis_of_sketch: empty sketch");
    DeviceGuard g(h->device);
    CompBufs B;
    // the basis overwrites its input: always work on a private copy
    B.a.ensure(sizeof(double) * n * c);
    CK(cudaMemcpyAsync(B.a.p, z, sizeof(double) * n * c,
                       z_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
    BasisPlan bp = plan_basis(n, c, rank);
    Layout L;
    BasisBuffers bb = layout_basis(L, bp);
    const size_t off_u = L.take(sizeof(double) * n * rank);
    const size_t off_pad = L.take(sizeof(double) * n);
    const size_t off_t = L.take(sizeof(BasisTarget));
    B.b.ensure(L.off);
    char* ws = reinterpret_cast<char*>(B.b.p);
    std::vector<BasisTarget> bt = {fill_basis(bp, bb, ws, reinterpret_cast<double*>(B.a.p),
                                              reinterpret_cast<double*>(ws + off_u),
                                              srtt_host::stream_state0(seed, stream_id), draw_offset, normal_base)};
    assign_basis_ctas(bt);
    Blob blob;
    const BasisLists lists = make_basis_lists(bt, blob);
    std::vector<unsigned char> hb(blob.lay.off);
    for (auto& it : blob.items) std::memcpy(hb.data() + it.first, it.second.data(), it.second.size());
    B.c.ensure(hb.size() + 64);
    CK(cudaMemcpyAsync(B.c.p, hb.data(), hb.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(ws + off_t, bt.data(), sizeof(BasisTarget), cudaMemcpyHostToDevice, h->stream));
    launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(ws + off_t), lists,
                       reinterpret_cast<const char*>(B.c.p), reinterpret_cast<double*>(ws + off_pad), n);
    CK(cudaStreamSynchronize(h->stream));
    copy_out(h, q_out, ws + off_u, sizeof(double) * n * rank, out_on_device);
    int32_t info[4];
    CK(cudaMemcpyAsync(info, bt[0].info, sizeof(info), cudaMemcpyDeviceToHost, h->stream));
    std::vector<double> sv(std::min<int64_t>(n, c));
    CK(cudaMemcpyAsync(sv.data(), bt[0].sv, sizeof(double) * sv.size(), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (numerical_rank) *numerical_rank = info[0];
    if (sv_out) std::memcpy(sv_out, sv.data(), sizeof(double) * sv.size());
  });
}

int srtt_multi_ttm_core(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                        const int64_t* ranks, const double* const* factors, int32_t factors_on_device,
                        double* core_out, int32_t out_on_device) {
  return guarded([&] {
    if (d < 2 || d > SRTT_MAX_ORDER) invalid("multi_ttm_core: order must be in [2, 16]");
    std::vector<int64_t> dv(dims, dims + d), rv(ranks, ranks + d);
    for (int k = 0; k < d; ++k)
      if (dv[k] < 1 || rv[k] < 1 || rv[k] > dv[k]) invalid("sliced_core: factor rows mismatch in mode " + std::to_string(k));
    DeviceGuard g(h->device);
    const int64_t N = prod(dv);
    CompRef B = comp_bufs(h);
    const double* dx = to_device(h, B.a, x, N, x_on_device);
    std::vector<DevBuf> ub(d);
    std::vector<const double*> u(d);
    for (int k = 0; k < d; ++k) u[k] = to_device(h, ub[k], factors[k], dv[k] * rv[k], factors_on_device);
    Layout L;
    CoreJob core;
    core.plan(dv, rv, h->sms, L);
    const size_t off_core = L.take(sizeof(double) * prod(rv));
    B.b.ensure(L.off);
    char* ws = reinterpret_cast<char*>(B.b.p);
    core.launch(h, dx, u, reinterpret_cast<double*>(ws + off_core), ws);
    copy_out(h, core_out, ws + off_core, sizeof(double) * prod(rv), out_on_device);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_transfer_tensor(srtt_handle* h, const double* u_node, const double* u_left, const double* u_right,
                         int64_t nl, int64_t nr, int32_t rs, int32_t rl, int32_t rr, int32_t on_device,
                         double* b_out) {
  return guarded([&] {
    if (nl < 1 || nr < 1 || rs < 1 || rl < 1 || rr < 1) invalid("transfer_tensor: empty operand");
    DeviceGuard g(h->device);
    CompBufs B;
    TransferTarget T{};
    T.us = to_device(h, B.a, u_node, nl * nr * rs, on_device);
    T.ul = to_device(h, B.b, u_left, nl * rl, on_device);
    T.ur = to_device(h, B.c, u_right, nr * rr, on_device);
    B.d.ensure(sizeof(double) * rs * rl * rr + 256 + sizeof(TransferTarget));
    T.b = reinterpret_cast<double*>(B.d.p);
    T.nl = nl;
    T.nr = nr;
    T.rs = rs;
    T.rl = rl;
    T.rr = rr;
    T.cta_begin = 0;
    char* tp = reinterpret_cast<char*>(B.d.p) + ((sizeof(double) * rs * rl * rr + 255) / 256 * 256);
    CK(cudaMemcpyAsync(tp, &T, sizeof(T), cudaMemcpyHostToDevice, h->stream));
    CK(srtt_launch_transfer(reinterpret_cast<const TransferTarget*>(tp), 1, rs, rl, rr, h->stream));
    copy_out(h, b_out, T.b, sizeof(double) * rs * rl * rr, on_device);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_root_transfer(srtt_handle* h, const double* x, int32_t x_on_device, int64_t nl, int64_t nr,
                       const double* u_left, int32_t rl, const double* u_right, int32_t rr,
                       int32_t factors_on_device, double* b_out, int32_t out_on_device) {
  return guarded([&] {
    if (nl < 1 || nr < 1) invalid("root_transfer: child rows do not factor the tensor size");
    const int64_t dims2[2] = {nl, nr};
    const int64_t ranks2[2] = {rl, rr};
    const double* f[2] = {u_left, u_right};
    // identical to the 2-mode core: B(0, j, k) = (U_l^T M U_r)(j, k)
    const int rc = srtt_multi_ttm_core(h, x, x_on_device, 2, dims2, ranks2, f, factors_on_device, b_out,
                                       out_on_device);
    if (rc != SRTT_OK) throw Error{rc, g_last_error};
  });
}

}  // extern "C"

// ==================================================================================
// Slab-sharded Sub-R-HOSVD phases (last-mode slabs)
// ==================================================================================
namespace {

struct SampledModes {
  std::vector<std::vector<int64_t>> cols;
  std::vector<uint64_t> draws, state0;
};

SampledModes sample_all_modes(int d, const std::vector<int64_t>& dims, const std::vector<int64_t>& samples,
                              uint64_t seed, int64_t partitions) {
  SampledModes S;
  S.cols.resize(d);
  S.draws.resize(d);
  S.state0.resize(d);
  const int64_t N = prod(dims);
  for (int k = 0; k < d; ++k) {
    srtt_host::Stream rng(seed, (uint64_t)k);
    try {
      if (partitions > 1)
        srtt_host::sample_indices_partitioned(N / dims[k], samples[k], partitions, rng, S.cols[k]);
      else
        srtt_host::sample_indices(N / dims[k], samples[k], rng, S.cols[k]);
    } catch (const std::exception& e) {
      fail(SRTT_ERR_JOB, "job " + std::to_string(k) + ": " + e.what());
    }
    S.draws[k] = rng.draws;
    S.state0[k] = srtt_host::stream_state0(seed, (uint64_t)k);
  }
  return S;
}

void validate_tucker(int d, const std::vector<int64_t>& dims, const std::vector<int64_t>& ranks,
                     const std::vector<int64_t>& samples, int64_t p) {
  if (d < 2 || d > SRTT_MAX_ORDER) invalid("sub_r_hosvd: unsupported order");
  for (int k = 0; k < d; ++k)
    if (dims[k] < 1) invalid("Shape: dimensions must be >= 1");
  const int64_t N = prod(dims);
  for (int k = 0; k < d; ++k)
    if (ranks[k] < 1 || ranks[k] > dims[k]) invalid("sub_r_hosvd: rank out of range in mode " + std::to_string(k));
  for (int k = 0; k < d; ++k) {
    if (samples[k] < ranks[k] + p)
      invalid("sub_r_hosvd: samples below rank + oversampling in mode " + std::to_string(k));
    if (samples[k] > N / dims[k]) invalid("sub_r_hosvd: more samples than fibers in mode " + std::to_string(k));
    if (ranks[k] + p > SRTT_MAX_SKETCH_COLS)
      invalid("sub_r_hosvd: rank + oversampling above 256 is not supported by the B200 basis kernels");
  }
}

}  // namespace

extern "C" {

int srtt_shard_sketches(srtt_handle* h, const double* x_local, int32_t x_on_device, int32_t d, const int64_t* dims_p,
                        int64_t slab_lo, int64_t slab_hi, const int64_t* ranks_p, int64_t p, const int64_t* samples_p,
                        uint64_t seed, const srtt_exec_policy* exec, double* const* z_out, int32_t out_on_device) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    std::vector<int64_t> dims(dims_p, dims_p + d), ranks(ranks_p, ranks_p + d), samples(samples_p, samples_p + d);
    validate_tucker(d, dims, ranks, samples, p);
    const int L = d - 1;
    if (slab_lo < 0 || slab_hi > dims[L] || slab_lo >= slab_hi) invalid("shard: slab out of range");
    std::vector<int64_t> ldims = dims;
    ldims[L] = slab_hi - slab_lo;
    const int64_t Nl = prod(ldims);
    DeviceGuard g(h->device);
    CompRef B = comp_bufs(h);
    const double* x = to_device(h, B.a, x_local, Nl, x_on_device);
    const SampledModes S = sample_all_modes(d, dims, samples, seed, exec ? exec->index_partitions : 1);
    Layout Lw;
    std::vector<size_t> off_z(d), off_cols(d), off_zp(d);
    int cmax = 0;
    for (int k = 0; k < d; ++k) {
      const int c = (int)(ranks[k] + p);
      cmax = std::max(cmax, c);
      off_z[k] = Lw.take(sizeof(double) * (k == L ? ldims[k] : dims[k]) * c);
      off_cols[k] = Lw.take(sizeof(int64_t) * samples[k]);
      off_zp[k] = Lw.take(sketch_part_bytes(k == L ? ldims[k] : dims[k], samples[k], c));
    }
    const size_t off_t = Lw.take(sizeof(SketchTarget) * d);
    const size_t off_flags = Lw.take(sizeof(int32_t) * 4);
    B.b.ensure(Lw.off);
    char* ws = reinterpret_cast<char*>(B.b.p);
    std::vector<SketchTarget> sk(d);
    int64_t ctas = 0;
    for (int k = 0; k < d; ++k) {
      const int c = (int)(ranks[k] + p);
      if (k == L) {
        sk[k] = make_sketch_target(x, ldims, {k}, samples[k], c);
      } else {
        sk[k] = make_sketch_target(x, dims, {k}, samples[k], c);  // decode columns over GLOBAL extents
        sk[k].slab_digit = sk[k].ncol_modes - 1;                   // mode d-1 is the last complement digit
        sk[k].slab_lo = slab_lo;
        sk[k].slab_hi = slab_hi;
      }
      sk[k].cols = reinterpret_cast<const int64_t*>(ws + off_cols[k]);
      sk[k].z = reinterpret_cast<double*>(ws + off_z[k]);
      sk[k].state0 = S.state0[k];
      sk[k].draw_offset = S.draws[k];
      sk[k].cta_begin = ctas;
      sk[k].flags = reinterpret_cast<int32_t*>(ws + off_flags);
      attach_sketch_scratch(sk[k], ws + off_zp[k]);
      ctas += sketch_target_ctas(sk[k]);
      CK(cudaMemcpyAsync(ws + off_cols[k], S.cols[k].data(), sizeof(int64_t) * samples[k], cudaMemcpyHostToDevice,
                         h->stream));
    }
    CK(cudaMemsetAsync(ws + off_flags, 0, sizeof(int32_t) * 4, h->stream));
    assign_contig_ctas(sk);
    CK(cudaMemcpyAsync(ws + off_t, sk.data(), sizeof(SketchTarget) * d, cudaMemcpyHostToDevice, h->stream));
    launch_sketch_group(reinterpret_cast<const SketchTarget*>(ws + off_t), sk, ctas, cmax, h->stream);
    for (int k = 0; k < d; ++k)
      copy_out(h, z_out[k], ws + off_z[k], sizeof(double) * sk[k].rows * sk[k].c, out_on_device);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_bases_from_sketches(srtt_handle* h, int32_t d, const int64_t* dims_p, const int64_t* ranks_p, int64_t p,
                             const int64_t* samples_p, uint64_t seed, const srtt_exec_policy* exec,
                             const double* const* z, int32_t z_on_device, double* const* factors_out,
                             int32_t out_on_device, int64_t* achieved_ranks) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    std::vector<int64_t> dims(dims_p, dims_p + d), ranks(ranks_p, ranks_p + d), samples(samples_p, samples_p + d);
    validate_tucker(d, dims, ranks, samples, p);
    DeviceGuard g(h->device);
    const SampledModes S = sample_all_modes(d, dims, samples, seed, exec ? exec->index_partitions : 1);
    CompRef B = comp_bufs(h);
    Layout Lw;
    std::vector<size_t> off_z(d), off_u(d);
    std::vector<BasisPlan> bp(d);
    std::vector<BasisBuffers> bb(d);
    int64_t max_n = 0;
    for (int k = 0; k < d; ++k) {
      const int c = (int)(ranks[k] + p);
      off_z[k] = Lw.take(sizeof(double) * dims[k] * c);
      off_u[k] = Lw.take(sizeof(double) * dims[k] * ranks[k]);
      bp[k] = plan_basis(dims[k], c, (int)ranks[k]);
      bb[k] = layout_basis(Lw, bp[k]);
      max_n = std::max(max_n, dims[k]);
    }
    const size_t off_pad = Lw.take(sizeof(double) * max_n * d);
    const size_t off_t = Lw.take(sizeof(BasisTarget) * d);
    const size_t off_info = Lw.take(sizeof(int32_t) * 4 * d);
    B.b.ensure(Lw.off);
    char* ws = reinterpret_cast<char*>(B.b.p);
    std::vector<BasisTarget> bt(d);
    for (int k = 0; k < d; ++k) {
      const int c = (int)(ranks[k] + p);
      // the basis overwrites its sketch: work on a private copy
      CK(cudaMemcpyAsync(ws + off_z[k], z[k], sizeof(double) * dims[k] * c,
                         z_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
      bt[k] = fill_basis(bp[k], bb[k], ws, reinterpret_cast<double*>(ws + off_z[k]),
                         reinterpret_cast<double*>(ws + off_u[k]), S.state0[k], S.draws[k], samples[k] * c,
                         reinterpret_cast<int32_t*>(ws + off_info) + 4 * k);
    }
    assign_basis_ctas(bt);
    Blob blob;
    const BasisLists lists = make_basis_lists(bt, blob);
    std::vector<unsigned char> hb(blob.lay.off);
    for (auto& it : blob.items) std::memcpy(hb.data() + it.first, it.second.data(), it.second.size());
    B.c.ensure(hb.size() + 64);
    CK(cudaMemcpyAsync(B.c.p, hb.data(), hb.size(), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(ws + off_t, bt.data(), sizeof(BasisTarget) * d, cudaMemcpyHostToDevice, h->stream));
    launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(ws + off_t), lists,
                       reinterpret_cast<const char*>(B.c.p), reinterpret_cast<double*>(ws + off_pad), max_n);
    for (int k = 0; k < d; ++k)
      copy_out(h, factors_out[k], ws + off_u[k], sizeof(double) * dims[k] * ranks[k], out_on_device);
    std::vector<int32_t> info(4 * d);
    CK(cudaMemcpyAsync(info.data(), ws + off_info, sizeof(int32_t) * 4 * d, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (achieved_ranks)
      for (int k = 0; k < d; ++k) achieved_ranks[k] = info[4 * k];
  });
}

int srtt_shard_core(srtt_handle* h, const double* x_local, int32_t x_on_device, int32_t d, const int64_t* dims_p,
                    int64_t slab_lo, int64_t slab_hi, const int64_t* ranks_p, const double* const* factors,
                    int32_t factors_on_device, double* core_partial_out, int32_t out_on_device) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (d < 2 || d > SRTT_MAX_ORDER) invalid("shard_core: unsupported order");
    std::vector<int64_t> dims(dims_p, dims_p + d), ranks(ranks_p, ranks_p + d);
    const int L = d - 1;
    if (slab_lo < 0 || slab_hi > dims[L] || slab_lo >= slab_hi) invalid("shard: slab out of range");
    std::vector<int64_t> ldims = dims;
    ldims[L] = slab_hi - slab_lo;
    DeviceGuard g(h->device);
    CompRef B = comp_bufs(h);
    // U_{d-1} rows [lo, hi) as a contiguous (hi-lo) x r block
    const int64_t nl = slab_hi - slab_lo;
    B.d.ensure(sizeof(double) * nl * ranks[L]);
    CK(cudaMemcpy2DAsync(B.d.p, sizeof(double) * nl, factors[L] + slab_lo, sizeof(double) * dims[L],
                         sizeof(double) * nl, ranks[L],
                         factors_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
    std::vector<const double*> f(factors, factors + d);
    f[L] = reinterpret_cast<const double*>(B.d.p);
    // the local factor is on the device now; stage the others the same way
    std::vector<DevBuf> fb(d);
    for (int k = 0; k < L; ++k) f[k] = to_device(h, fb[k], factors[k], dims[k] * ranks[k], factors_on_device);
    const int rc = srtt_multi_ttm_core(h, x_local, x_on_device, d, ldims.data(), ranks.data(), f.data(), 1,
                                       core_partial_out, out_on_device);
    if (rc != SRTT_OK) throw Error{rc, g_last_error};
  });
}

}  // extern "C"

// ==================================================================================
// Reconstruction and streaming reconstruction error
// ==================================================================================
namespace {

// out = in x_mode U with in viewed as g x r x post and U an n x r factor,
// given column-major (kfast = false) or K-fastest r x n (kfast = true).
void ttm_expand(srtt_handle* h, const double* in, int64_t g, int64_t r, int64_t post, const double* u, int64_t n,
                bool kfast, double* out) {
  TtmParams T{};
  T.in = in;
  T.u = u;
  T.out = out;
  T.g = g;
  T.n = r;
  T.post = post;
  T.rr = n;
  T.transpose = kfast ? 1 : 0;
  T.nparts = 1;
  CK(srtt_launch_ttm(T, h->stream));
}

// Low-rank view X-hat = A C^T of the n_A x n_B unfolding, factors K-fastest
// with K zero-padded to a multiple of 8 (At: K x n_A, Ct: K x n_B).
struct LowRank {
  const double* at = nullptr;
  const double* ct = nullptr;
  int64_t nA = 0, nB = 0;
  int K = 0;
};

int64_t pad8(int64_t k) { return (k + 7) / 8 * 8; }

// Streams A C^T against x (norms) or into out (reconstruction).
void run_residual(srtt_handle* h, const LowRank& lr, const double* x, double* out, double* sums_host) {
  const int grid = srtt_residual_grid(h->sms, lr.nA, lr.K);
  DevBuf& part = h->rb[4];
  part.ensure(sizeof(double) * (2 * grid + 2));
  ResidualParams P{};
  P.x = x;
  P.at = lr.at;
  P.ct = lr.ct;
  P.out = out;
  P.partial = reinterpret_cast<double*>(part.p);
  P.nA = lr.nA;
  P.nB = lr.nB;
  P.K = lr.K;
  const int tm = srtt_residual_tile_rows(lr.nA), tn = srtt_residual_tile_cols(lr.nA, lr.K);
  CUtensorMap tmx;
  std::memset(&tmx, 0, sizeof(tmx));
  // TMA needs a 16-byte row pitch: odd n_A streams X with cp.async instead
  P.x_tma = (x != nullptr && lr.nA % 2 == 0) ? 1 : 0;
  if (P.x_tma) encode_tmap_plain(&tmx, x, lr.nA, lr.nB, lr.nA, tm, tn);
  double* sums = reinterpret_cast<double*>(part.p) + 2 * grid;
  CK(srtt_launch_residual(&tmx, P, grid, sums, h->stream));
  if (!out) {
    CK(cudaMemcpyAsync(sums_host, sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
}

double rel_from_sums(const double* s) {
  if (s[1] == 0.0) invalid("rel_error: reference tensor has zero norm");
  return std::sqrt(s[0]) / std::sqrt(s[1]);
}

// Tucker: X-hat_(0..m-1) = (U_{m-1} (x) ... (x) U_0) [G x_m U_m ... x_{d-1} U_{d-1}]^T.
// The split m comes from a cost model: FP64 FMAs of the tiled residual
// vs the bytes of X and Ct.
struct TuckerLowRank {
  explicit TuckerLowRank(srtt_handle* h) : at(h->rb[0]), tmp(h->rb[1]), c0(h->rb[2]), c1(h->rb[3]) {}
  LowRank lr;
  DevBuf &at, &tmp, &c0, &c1;
  std::vector<DevBuf> fb;
  DevBuf gb;
};

void build_tucker_lowrank(srtt_handle* h, TuckerLowRank& T, int d, const std::vector<int64_t>& dims,
                          const std::vector<int64_t>& ranks, const double* core, const double* const* factors,
                          int on_device) {
  for (int k = 0; k < d; ++k)
    if (ranks[k] < 1 || ranks[k] > dims[k] || dims[k] < 1)
      invalid("reconstruct: factor/core mismatch in mode " + std::to_string(k));
  if (ranks[0] > 64) invalid("reconstruct: ranks above 64 are not supported by the B200 residual kernel");
  T.fb.resize(d);
  std::vector<const double*> u(d);
  for (int k = 0; k < d; ++k) u[k] = to_device(h, T.fb[k], factors[k], dims[k] * ranks[k], on_device);
  const double* g = to_device(h, T.gb, core, prod(ranks), on_device);
  int best = 1;
  double best_cost = 0;
  int64_t KA = 1, nA = 1;
  for (int m = 1; m < d; ++m) {
    KA *= ranks[m - 1];
    nA *= dims[m - 1];
    if (KA > 64) break;
    const int64_t nB = prod(dims) / nA;
    const int tm = srtt_residual_tile_rows(nA);
    const double rows_eff = (double)((nA + tm - 1) / tm * tm);
    const double fma_s = rows_eff * nB * (double)pad8(KA) / (58.0 * h->sms * 1.9e9);
    const double mem_s = (8.0 * nA * nB + 16.0 * nB * pad8(KA)) / 6.5e12;
    const double cost = std::max(fma_s, mem_s);
    if (m == 1 || cost < best_cost) {
      best = m;
      best_cost = cost;
    }
  }
  const int m = best;
  int64_t K = 1;
  T.lr.nA = 1;
  for (int k = 0; k < m; ++k) {
    K *= ranks[k];
    T.lr.nA *= dims[k];
  }
  const int64_t Kp = pad8(K);
  T.lr.nB = prod(dims) / T.lr.nA;
  T.lr.K = (int)Kp;
  // At = (U_{m-1} (x) ... (x) U_0)^T, K x n_A, then zero-padded to Kp rows
  T.tmp.ensure(sizeof(double) * std::max<int64_t>(K * T.lr.nA, prod(ranks)));
  double* tmp = reinterpret_cast<double*>(T.tmp.p);
  if (m == 1) {
    CK(srtt_launch_mat_transpose(u[0], dims[0], ranks[0], tmp, h->stream));
  } else {
    KronParams kp{};
    for (int k = 0; k < m; ++k) {
      kp.u[k] = u[k];
      kp.n[k] = dims[k];
      kp.r[k] = ranks[k];
    }
    kp.at = tmp;
    kp.K = K;
    kp.nA = T.lr.nA;
    kp.m = m;
    CK(srtt_launch_kron_rows(kp, h->stream));
  }
  T.at.ensure(sizeof(double) * Kp * T.lr.nA);
  CK(srtt_launch_pad_rows(tmp, K, T.lr.nA, Kp, reinterpret_cast<double*>(T.at.p), h->stream));
  // Ct = G' x_1 U_m ... with G' the core as Kp x r_m x ... (zero rows K..Kp-1)
  std::vector<int64_t> ext = {Kp}, full = {Kp};
  for (int k = m; k < d; ++k) {
    ext.push_back(ranks[k]);
    full.push_back(dims[k]);
  }
  const int e = (int)ext.size();
  size_t maxe = (size_t)prod(ext);
  {
    std::vector<int64_t> cur = ext;
    for (int k = 1; k < e; ++k) {
      cur[k] = full[k];
      maxe = std::max<size_t>(maxe, (size_t)prod(cur));
    }
  }
  T.c0.ensure(sizeof(double) * maxe);
  T.c1.ensure(sizeof(double) * maxe);
  double* bufs[2] = {reinterpret_cast<double*>(T.c0.p), reinterpret_cast<double*>(T.c1.p)};
  CK(srtt_launch_pad_rows(g, K, prod(ranks) / K, Kp, bufs[1], h->stream));
  const double* cur = bufs[1];
  for (int k = 1; k < e; ++k) {
    int64_t gpre = 1, post = 1;
    for (int j = 0; j < k; ++j) gpre *= ext[j];
    for (int j = k + 1; j < e; ++j) post *= ext[j];
    double* o = bufs[(k - 1) & 1];
    ttm_expand(h, cur, gpre, ext[k], post, u[m + k - 1], full[k], false, o);
    ext[k] = full[k];
    cur = o;
  }
  T.lr.at = reinterpret_cast<const double*>(T.at.p);
  T.lr.ct = cur;
}

// H-Tucker: node bases rebuilt bottom-up in K-fastest layout (r_S x n_S),
// then At = U_left^T, Ct = B_0 U_right^T (htucker.hpp:346-378).
struct HtLowRank {
  explicit HtLowRank(srtt_handle* h) : w(h->rb[1]), at(h->rb[0]), ct(h->rb[2]) {}
  LowRank lr;
  std::vector<DevBuf> nb;     // per node: K-fastest basis (internal nodes) / staged leaf factor
  std::vector<DevBuf> tb;     // staged transfers
  DevBuf &w, &at, &ct;
  DevBuf tmp, b0;
};

void build_ht_lowrank(srtt_handle* h, HtLowRank& H, const Tree& tr, const std::vector<int64_t>& dims,
                      const std::vector<int64_t>& ranks, const double* const* leaf_factors,
                      const double* const* transfers, int on_device) {
  const int nn = tr.n;
  auto rows = [&](int i) {
    int64_t r = 1;
    for (int m : tr.modes[i]) r *= dims[m];
    return r;
  };
  if (ranks[0] != 1) invalid("ht_reconstruct: root rank must be 1");
  for (int i = 1; i < nn; ++i)
    if (ranks[i] < 1) invalid("ht_reconstruct: rank out of range at node " + std::to_string(i));
  H.nb.resize(nn);
  H.tb.resize(nn);
  std::vector<const double*> basis(nn, nullptr), B(nn, nullptr);
  std::vector<bool> kfast(nn, false);
  for (int i = 0; i < nn; ++i) {
    if (tr.leaf(i)) {
      const int m = tr.modes[i][0];
      basis[i] = to_device(h, H.nb[i], leaf_factors[m], dims[m] * ranks[i], on_device);
    } else {
      const int64_t cnt = ranks[i] * ranks[tr.left[i]] * ranks[tr.right[i]];
      B[i] = to_device(h, H.tb[i], transfers[i], cnt, on_device);
    }
  }
  // bottom-up: deepest nodes first
  std::vector<int> order;
  for (int i = 1; i < nn; ++i)
    if (!tr.leaf(i)) order.push_back(i);
  std::vector<int> depth(nn, 0);
  for (int i = 1; i < nn; ++i) depth[i] = depth[tr.parent[i]] + 1;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return depth[a] > depth[b]; });
  size_t wmax = 1;
  for (int i : order)
    wmax = std::max<size_t>(wmax, (size_t)(ranks[i] * rows(tr.left[i]) * ranks[tr.right[i]]));
  H.w.ensure(sizeof(double) * wmax);
  for (int i : order) {
    const int l = tr.left[i], r = tr.right[i];
    const int64_t rs = ranks[i], rl = ranks[l], rr = ranks[r], nl = rows(l), nr = rows(r);
    double* w = reinterpret_cast<double*>(H.w.p);
    // W = B x_2 U_l: (rs, nl, rr); V = W x_3 U_r: (rs, nl, nr) = K-fastest basis
    ttm_expand(h, B[i], rs, rl, rr, basis[l], nl, kfast[l], w);
    H.nb[i].ensure(sizeof(double) * rs * nl * nr);
    ttm_expand(h, w, rs * nl, rr, 1, basis[r], nr, kfast[r], reinterpret_cast<double*>(H.nb[i].p));
    basis[i] = reinterpret_cast<const double*>(H.nb[i].p);
    kfast[i] = true;
  }
  const int l = tr.left[0], r = tr.right[0];
  const int64_t rl = ranks[l], rr = ranks[r], nl = rows(l), nr = rows(r);
  if (rl > 64) invalid("ht_reconstruct: root-child ranks above 64 are not supported by the B200 residual kernel");
  const int64_t Kp = pad8(rl);
  const double* at_k = basis[l];
  if (!kfast[l]) {
    H.tmp.ensure(sizeof(double) * rl * nl);
    CK(srtt_launch_mat_transpose(basis[l], nl, rl, reinterpret_cast<double*>(H.tmp.p), h->stream));
    at_k = reinterpret_cast<const double*>(H.tmp.p);
  }
  H.at.ensure(sizeof(double) * Kp * nl);
  CK(srtt_launch_pad_rows(at_k, rl, nl, Kp, reinterpret_cast<double*>(H.at.p), h->stream));
  H.b0.ensure(sizeof(double) * Kp * rr);
  CK(srtt_launch_pad_rows(B[0], rl, rr, Kp, reinterpret_cast<double*>(H.b0.p), h->stream));
  H.ct.ensure(sizeof(double) * Kp * nr);
  ttm_expand(h, reinterpret_cast<const double*>(H.b0.p), Kp, rr, 1, basis[r], nr, kfast[r],
             reinterpret_cast<double*>(H.ct.p));
  H.lr.at = reinterpret_cast<const double*>(H.at.p);
  H.lr.ct = reinterpret_cast<const double*>(H.ct.p);
  H.lr.nA = nl;
  H.lr.nB = nr;
  H.lr.K = (int)Kp;
}

void finish_reconstruct(srtt_handle* h, const LowRank& lr, double* out, int out_on_device) {
  const int64_t N = lr.nA * lr.nB;
  DevBuf ob;
  double* dst = out;
  if (!out_on_device) {
    ob.ensure(sizeof(double) * N);
    dst = reinterpret_cast<double*>(ob.p);
  }
  run_residual(h, lr, nullptr, dst, nullptr);
  if (!out_on_device) copy_out(h, out, dst, sizeof(double) * N, 0);
  CK(cudaStreamSynchronize(h->stream));
}

}  // namespace

extern "C" {

int srtt_rel_error(srtt_handle* h, const double* ref, const double* approx, int32_t on_device, int64_t n,
                   double* rel_error) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (n < 1) invalid("rel_error: empty tensor");
    DeviceGuard g(h->device);
    CompBufs B;
    const double* x = to_device(h, B.a, ref, n, on_device);
    const double* y = to_device(h, B.b, approx, n, on_device);
    const int grid = 2 * h->sms;
    B.c.ensure(sizeof(double) * (2 * grid + 2));
    double* part = reinterpret_cast<double*>(B.c.p);
    CK(srtt_launch_diff_norm(x, y, n, grid, part, part + 2 * grid, h->stream));
    double s[2];
    CK(cudaMemcpyAsync(s, part + 2 * grid, sizeof(s), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *rel_error = rel_from_sums(s);
  });
}

int srtt_tucker_reconstruct(srtt_handle* h, int32_t d, const int64_t* dims, const int64_t* ranks, const double* core,
                            const double* const* factors, int32_t in_on_device, double* out, int32_t out_on_device) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (d < 2 || d > SRTT_MAX_ORDER) invalid("reconstruct: unsupported order");
    DeviceGuard g(h->device);
    TuckerLowRank T(h);
    build_tucker_lowrank(h, T, d, std::vector<int64_t>(dims, dims + d), std::vector<int64_t>(ranks, ranks + d), core,
                         factors, in_on_device);
    finish_reconstruct(h, T.lr, out, out_on_device);
  });
}

int srtt_tucker_rel_error(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                          const int64_t* ranks, const double* core, const double* const* factors,
                          int32_t in_on_device, double* rel_error) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (d < 2 || d > SRTT_MAX_ORDER) invalid("rel_error: unsupported order");
    DeviceGuard g(h->device);
    std::vector<int64_t> dv(dims, dims + d);
    TuckerLowRank T(h);
    build_tucker_lowrank(h, T, d, dv, std::vector<int64_t>(ranks, ranks + d), core, factors, in_on_device);
    CompBufs B;
    const double* dx = to_device(h, B.a, x, prod(dv), x_on_device);
    double s[2];
    run_residual(h, T.lr, dx, nullptr, s);
    *rel_error = rel_from_sums(s);
  });
}

int srtt_ht_reconstruct(srtt_handle* h, int32_t d, const int64_t* dims, const srtt_tree* tree, const int64_t* ranks,
                        const double* const* leaf_factors, const double* const* transfers, int32_t in_on_device,
                        double* out, int32_t out_on_device) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    const Tree tr = read_tree(tree, d);
    DeviceGuard g(h->device);
    HtLowRank H(h);
    build_ht_lowrank(h, H, tr, std::vector<int64_t>(dims, dims + d), std::vector<int64_t>(ranks, ranks + tr.n),
                     leaf_factors, transfers, in_on_device);
    finish_reconstruct(h, H.lr, out, out_on_device);
  });
}

int srtt_ht_rel_error(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                      const srtt_tree* tree, const int64_t* ranks, const double* const* leaf_factors,
                      const double* const* transfers, int32_t in_on_device, double* rel_error) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    const Tree tr = read_tree(tree, d);
    DeviceGuard g(h->device);
    std::vector<int64_t> dv(dims, dims + d);
    HtLowRank H(h);
    build_ht_lowrank(h, H, tr, dv, std::vector<int64_t>(ranks, ranks + tr.n), leaf_factors, transfers,
                     in_on_device);
    CompBufs B;
    const double* dx = to_device(h, B.a, x, prod(dv), x_on_device);
    double s[2];
    run_residual(h, H.lr, dx, nullptr, s);
    *rel_error = rel_from_sums(s);
  });
}

}  // extern "C"

// ---- accessors for the IO module (io.cu) -------------------------------------
cudaStream_t srtt_internal_stream(srtt_handle* h) { return h->stream; }
int srtt_internal_device(srtt_handle* h) { return h->device; }
void srtt_internal_set_error(const std::string& msg) { g_last_error = msg; }

// ---- multi-GPU (NCCL) entry points ----------------------------------------------
#include "shard.cuh"
