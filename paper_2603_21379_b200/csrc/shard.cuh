// Multi-GPU Sub-R-HOSVD / Sub-R-RtL-HT: one process per GPU, the tensor
// split into contiguous slabs, NCCL over NVLink for the exchanges.
//
// Included at the end of host.cu (it drives the same planners, workspace
// arena, parameter blobs and graph cache as the single-GPU path).
//
// Reference algebra (parallel.hpp:355-445 sliced_core, htucker.hpp:67-85
// root_transfer, htucker.hpp:249-324 job DAG), across GPUs:
//
//  Tucker, X split along its LAST mode, rank w holds X[..., lo_w:hi_w):
//   sketches   every rank samples the same fibres and generates the same
//              Omega (same seed, counter-based stream). For k < d-1 a sampled
//              fibre lies in exactly one slab: partial Z_k, fibres of other
//              slabs contribute zero. For k = d-1 each rank owns rows
//              [lo, hi) of Z_{d-1} and writes them into a zero-filled
//              full-height block. ONE allreduce(sum) over all sketches gives
//              every rank the exact Z_k (adding zeros is exact).
//   bases      identical on every rank (same Z, deterministic kernels).
//   core       G = sum_w X_w x_{k<d-1} U_k^T x_{d-1} U_{d-1}[lo_w:hi_w]^T
//              -> allreduce(sum) of prod r_k doubles.
//
//  H-Tucker, X split into column ranges [c_lo, c_hi) of the root
//  matricization M = n_left x n_right (a contiguous byte range of X):
//   sketches   every node's sketch is a sum over its sampled fibre entries;
//              entries outside the local range contribute zero -> partial
//              Z_S for every node, ONE allreduce over all of them.
//   bases      identical on every rank; transfer tensors from the bases.
//   root       B_0 = sum_w U_l^T M_w U_r[c_lo:c_hi] -> allreduce(r_l r_r).
//
// X never moves; only sketches (sum n_S (r_S + p) doubles) and the core /
// root (prod r_k or r_l r_r doubles) cross NVLink. The whole decomposition
// -- kernels and collectives -- is captured in ONE CUDA graph per signature
// and replayed.
//
// The H-Tucker split is also exposed as three synchronous phases (the same
// plan object and kernels, the exchanges left to the caller) so the multi-
// rank algebra can be exercised on one GPU and under gloo.
#pragma once

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is resolved at run time

namespace {

// ---- NCCL, resolved at run time -------------------------------------------
// dlopen("libnccl.so.2") returns the copy already loaded in the process
// (e.g. torch's) when there is one, else the system library.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      const char* e = dlerror();
      a.load_error = std::string("srtt: cannot load NCCL (libnccl.so.2): ") + (e ? e : "");
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(lib, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(lib, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(lib, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(lib, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(lib, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce)
      a.load_error = "srtt: libnccl.so.2 lacks the expected symbols";
    return a;
  }();
  if (!api.load_error.empty()) fail(SRTT_ERR_NCCL, api.load_error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const NcclApi& a = nccl_api();
  fail(SRTT_ERR_NCCL, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
}

ncclComm_t comm_of(srtt_handle* h) {
  if (!h->comm) invalid("sharded: the handle has no communicator (srtt_comm_init)");
  return reinterpret_cast<ncclComm_t>(h->comm);
}

// In-place sum over the handle's communicator, on the handle's stream.
void allreduce_sum(srtt_handle* h, double* buf, size_t count) {
  if (count == 0) return;
  nccl_check(nccl_api().all_reduce(buf, buf, count, ncclDouble, ncclSum, comm_of(h), h->stream), "ncclAllReduce");
}

// Slab / column-range bounds of rank w of `world` over n slices: the split of
// parallel.hpp:400-404 (sizes differ by at most one).
void split_bounds(int64_t n, int world, int rank, int64_t& lo, int64_t& hi) {
  lo = rank * (n / world) + std::min<int64_t>(rank, n % world);
  hi = lo + n / world + (rank < n % world ? 1 : 0);
}

void finish_report_common(srtt_report* rep, Timer& tm, double t_sampling, int64_t launches) {
  if (!rep) return;
  std::memset(rep->stage_seconds, 0, sizeof(rep->stage_seconds));
  rep->stage_seconds[SRTT_STAGE_SAMPLING] = t_sampling;
  rep->stage_seconds[SRTT_STAGE_H2D] = tm.between(0, 1);
  rep->stage_seconds[SRTT_STAGE_SKETCH] = tm.between(2, 3);
  rep->stage_seconds[SRTT_STAGE_GATHER] = tm.between(3, 4) + tm.between(6, 7);  // the two exchanges
  rep->stage_seconds[SRTT_STAGE_SVD] = tm.between(4, 5);
  rep->stage_seconds[SRTT_STAGE_TTM] = tm.between(5, 6);
  rep->stage_seconds[SRTT_STAGE_FACTOR_WALL] = t_sampling + tm.between(2, 5);
  rep->kernel_seconds[0] = tm.between(2, 3);
  rep->kernel_seconds[1] = tm.between(4, 5);
  rep->kernel_seconds[3] = 0.0;
  rep->launches = launches;
  rep->slice_mode = -1;
}

// ==================================================================================
// Slab-sharded Sub-R-HOSVD (fused: kernels + NCCL in one graph)
// ==================================================================================
// Greedy longest-processing-time assignment of targets to ranks (cost
// descending, ties by index; each to the least loaded rank, ties to the
// lowest rank): identical on every rank. Returns which targets are this
// rank's.
std::vector<char> assign_targets(const std::vector<double>& cost, int world, int rank) {
  std::vector<int> order(cost.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(world, 0.0);
  std::vector<char> mine(cost.size(), 0);
  for (int t : order) {
    int best = 0;
    for (int w = 1; w < world; ++w)
      if (load[w] < load[best]) best = w;
    load[best] += cost[t];
    if (best == rank) mine[t] = 1;
  }
  return mine;
}

void allreduce_sum_i32(srtt_handle* h, int32_t* buf, size_t count) {
  if (count == 0) return;
  nccl_check(nccl_api().all_reduce(buf, buf, count, ncclInt32, ncclSum, comm_of(h), h->stream), "ncclAllReduce");
}

// Tucker across GPUs, two layouts of X (the north star's two regimes):
//  slab-sharded (replicated = false): this rank holds X[..., lo:hi) only --
//    partial sketches, allreduce, identical bases, slab core, allreduce;
//  replicated (replicated = true): every rank holds all of X -- the modes
//    are assigned to ranks (LPT by n_k s_k (r_k + p)), each rank sketches and
//    factors only its modes into a zero-filled factor pack, ONE allreduce
//    of the pack (and of the per-mode info) gives every rank every factor,
//    then the core pass is split by last-mode slabs of the replica and
//    allreduced (parallel.hpp:133-147 mode jobs + :355-445 slab core).
void run_sub_r_hosvd_sharded(srtt_handle* h, const double* x_in, int x_on_device, int d, const int64_t* dims_p,
                             int64_t lo, int64_t hi, const int64_t* ranks_p, int64_t p, const int64_t* samples_p,
                             uint64_t seed, const srtt_exec_policy* exec, double* core_out,
                             double* const* factors_out, int out_on_device, srtt_report* rep,
                             bool replicated = false) {
  if (!h) invalid("srtt: null handle");
  std::vector<int64_t> dims(dims_p, dims_p + d), ranks(ranks_p, ranks_p + d), samples(samples_p, samples_p + d);
  validate_tucker(d, dims, ranks, samples, p);
  check_core_ranks(d, ranks.data(), "sub_r_hosvd");
  const int L = d - 1;
  if (replicated) {
    comm_of(h);
    if (h->world > dims[L]) invalid("replicated sub_r_hosvd: more ranks than slices along the last mode");
    split_bounds(dims[L], h->world, h->rank, lo, hi);
  }
  if (lo < 0 || hi > dims[L] || lo >= hi) invalid("sharded sub_r_hosvd: slab out of range");
  if (hi - lo < ranks[L]) invalid("sharded sub_r_hosvd: every slab must hold at least r_{d-1} slices");
  check_workers(exec, "run_independent_jobs");
  comm_of(h);
  std::vector<std::string> warnings;
  if (p < 4) warnings.push_back("oversampling below the recommended minimum of 4");
  std::vector<int64_t> ldims = dims;
  ldims[L] = hi - lo;
  const int64_t Nl = prod(ldims);
  const int64_t nl = hi - lo;
  const int64_t inner = prod(dims) / dims[L];
  std::vector<char> mine(d, 1);
  if (replicated) {
    std::vector<double> cost(d);
    for (int k = 0; k < d; ++k) cost[k] = (double)dims[k] * samples[k] * (ranks[k] + p);
    mine = assign_targets(cost, h->world, h->rank);
  }

  DeviceGuard guard(h->device);
  h->launches = 0;
  begin_call(h);
  h->timing = rep != nullptr;
  struct TimingReset {
    srtt_handle* h;
    ~TimingReset() { h->timing = true; }
  } timing_reset{h};
  Timer tm{h};
  const double ts0 = now_s();
  const SampledModes S = sample_all_modes(d, dims, samples, seed, exec ? exec->index_partitions : 1);
  const double t_sampling = now_s() - ts0;
  const int64_t slice_mode = exec ? resolve_slice_mode(dims, exec) : -1;
  tm.mark();  // 0
  const double* x = stage_input(h, x_in, x_on_device, replicated ? prod(dims) : Nl);
  const double* xslab = replicated ? x + lo * inner : x;  // the core pass's part
  tm.mark();  // 1

  // --- workspace: all sketches in ONE buffer (one allreduce), bases, core
  Layout W;
  std::vector<int64_t> zoff(d);
  int64_t zn = 0;
  int cmax = 0;
  for (int k = 0; k < d; ++k) {
    zoff[k] = zn;
    zn += dims[k] * (ranks[k] + p);
    cmax = std::max<int>(cmax, (int)(ranks[k] + p));
  }
  const size_t off_zsum = W.take(sizeof(double) * zn);
  std::vector<size_t> off_zp(d);
  for (int k = 0; k < d; ++k)
    off_zp[k] = W.take(sketch_part_bytes(k == L && !replicated ? nl : dims[k], samples[k], (int)(ranks[k] + p)));
  std::vector<size_t> off_u(d);
  std::vector<BasisPlan> bp(d);
  std::vector<BasisBuffers> bb(d);
  int64_t max_n = 0, upack_n = 0;
  for (int k = 0; k < d; ++k) upack_n += dims[k] * ranks[k];
  const size_t off_upack = replicated ? W.take(sizeof(double) * upack_n) : 0;
  for (int k = 0; k < d; ++k) {
    off_u[k] = (out_on_device || replicated) ? 0 : W.take(sizeof(double) * dims[k] * ranks[k]);
    bp[k] = plan_basis(dims[k], (int)(ranks[k] + p), (int)ranks[k]);
    bb[k] = layout_basis(W, bp[k]);
    max_n = std::max(max_n, dims[k]);
  }
  const size_t off_pad = W.take(sizeof(double) * max_n * d);
  const size_t off_uslab = W.take(sizeof(double) * nl * ranks[L]);
  const size_t off_core = W.take(sizeof(double) * prod(ranks));
  CoreJob core;
  core.plan(ldims, ranks, h->sms, W);
  h->ws.ensure(W.off);
  char* ws = reinterpret_cast<char*>(h->ws.p);
  double* zsum = reinterpret_cast<double*>(ws + off_zsum);
  std::vector<double*> uptr(d);
  double* upack = reinterpret_cast<double*>(ws + off_upack);
  for (int k = 0, o = 0; k < d; o += (int)(dims[k] * ranks[k]), ++k)
    uptr[k] = replicated ? upack + o
                         : (out_on_device ? factors_out[k] : reinterpret_cast<double*>(ws + off_u[k]));
  double* d_core = out_on_device ? core_out : reinterpret_cast<double*>(ws + off_core);

  // --- parameter blob
  int32_t* const dinfo = h->pset().dinfo();
  int32_t* const hinfo = h->pset().hinfo();
  const size_t info_bytes = sizeof(int32_t) * 4 * (d + 1);
  Blob blob;
  std::vector<size_t> off_cols(d);
  for (int k = 0; k < d; ++k) off_cols[k] = blob.add(S.cols[k].data(), sizeof(int64_t) * S.cols[k].size());
  const size_t off_sk = blob.reserve(sizeof(SketchTarget) * d);
  const size_t off_bt = blob.reserve(sizeof(BasisTarget) * d);
  h->pset().d.ensure(blob.lay.off + 4096);
  char* dp = reinterpret_cast<char*>(h->pset().d.p);
  std::vector<SketchTarget> sk(d);
  std::vector<BasisTarget> bt(d);
  int64_t ctas = 0;
  for (int k = 0; k < d; ++k) {
    const int c = (int)(ranks[k] + p);
    if (replicated) {  // a whole mode of the replica, as on one GPU
      sk[k] = make_sketch_target(x, dims, {k}, samples[k], c);
      sk[k].z = zsum + zoff[k];
    } else if (k == L) {  // this rank's rows [lo, hi) of Z_{d-1}, written at row lo of the full block
      sk[k] = make_sketch_target(x, ldims, {k}, samples[k], c);
      sk[k].z = zsum + zoff[k] + lo;
      sk[k].ldz = dims[k];
    } else {       // partial sketch: fibres of other slabs contribute zero
      sk[k] = make_sketch_target(x, dims, {k}, samples[k], c);
      sk[k].slab_digit = sk[k].ncol_modes - 1;
      sk[k].slab_lo = lo;
      sk[k].slab_hi = hi;
      sk[k].z = zsum + zoff[k];
    }
    sk[k].cols = reinterpret_cast<const int64_t*>(dp + off_cols[k]);
    sk[k].state0 = S.state0[k];
    sk[k].draw_offset = S.draws[k];
    sk[k].cta_begin = ctas;
    sk[k].flags = dinfo + 4 * d;
    attach_sketch_scratch(sk[k], ws + off_zp[k]);
    ctas += sketch_target_ctas(sk[k]);
    bt[k] = fill_basis(bp[k], bb[k], ws, zsum + zoff[k], uptr[k], S.state0[k], S.draws[k], samples[k] * c,
                       dinfo + 4 * k);
  }
  if (replicated) {  // this rank's modes only (CTA offsets recomputed)
    std::vector<SketchTarget> sk_m;
    std::vector<BasisTarget> bt_m;
    ctas = 0;
    for (int k = 0; k < d; ++k)
      if (mine[k]) {
        sk[k].cta_begin = ctas;
        ctas += sketch_target_ctas(sk[k]);
        sk_m.push_back(sk[k]);
        bt_m.push_back(bt[k]);
      }
    sk.swap(sk_m);
    bt.swap(bt_m);
  }
  const int nsk = (int)sk.size();
  assign_basis_ctas(bt);
  const BasisLists lists = make_basis_lists(bt, blob);
  h->pset().d.ensure(blob.lay.off);
  h->pset().hst.ensure(blob.lay.off);
  dp = reinterpret_cast<char*>(h->pset().d.p);
  char* hp = reinterpret_cast<char*>(h->pset().hst.p);
  for (auto& it : blob.items) std::memcpy(hp + it.first, it.second.data(), it.second.size());
  assign_contig_ctas(sk);
  if (nsk) std::memcpy(hp + off_sk, sk.data(), sizeof(SketchTarget) * nsk);
  if (nsk) std::memcpy(hp + off_bt, bt.data(), sizeof(BasisTarget) * nsk);

  std::string key = replicated ? "TR" : "TS";
  for (int k = 0; k < d; ++k)
    key += "|" + std::to_string(dims[k]) + "," + std::to_string(ranks[k]) + "," + std::to_string(samples[k]) + "," +
           ptr_key(uptr[k]);
  key += "|" + std::to_string(p) + "|" + std::to_string(lo) + "," + std::to_string(hi) + "|" + ptr_key(x) + "|" +
         ptr_key(d_core) + "|" + ptr_key(ws) + "|" + ptr_key(dp) + "|" + ptr_key(hp) + "|" + ptr_key(h->stream) +
         "|" + ptr_key(h->comm) + "|" + std::to_string(blob.lay.off) + (h->timing ? "|t" : "|n");
  const int64_t zL = dims[L] * (ranks[L] + p);
  run_enqueue(h, key, [&] {
    CK(cudaMemcpyAsync(dp, hp, blob.lay.off, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(dinfo, 0, info_bytes, h->stream));
    if (replicated)
      CK(cudaMemsetAsync(upack, 0, sizeof(double) * upack_n, h->stream));
    else
      CK(cudaMemsetAsync(zsum + zoff[L], 0, sizeof(double) * zL, h->stream));
    tm.n = 2;
    tm.mark();  // 2
    if (nsk)
      h->launches += launch_sketch_group(reinterpret_cast<const SketchTarget*>(dp + off_sk), sk, ctas, cmax,
                                         h->stream);
    tm.mark();  // 3
    if (!replicated) allreduce_sum(h, zsum, (size_t)zn);
    tm.mark();  // 4
    if (nsk)
      h->launches += launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(dp + off_bt), lists, dp,
                                        reinterpret_cast<double*>(ws + off_pad), max_n);
    if (replicated) {  // every rank's factors (others' entries are zero) and per-mode info
      allreduce_sum(h, upack, (size_t)upack_n);
      allreduce_sum_i32(h, dinfo, 4 * (size_t)(d + 1));
    }
    tm.mark();  // 5
    // U_{d-1} rows [lo, hi) as a contiguous block for the slab's core pass
    double* uslab = reinterpret_cast<double*>(ws + off_uslab);
    CK(cudaMemcpy2DAsync(uslab, sizeof(double) * nl, uptr[L] + lo, sizeof(double) * dims[L], sizeof(double) * nl,
                         ranks[L], cudaMemcpyDeviceToDevice, h->stream));
    std::vector<const double*> ucp(uptr.begin(), uptr.end());
    ucp[L] = uslab;
    h->launches += core.launch(h, xslab, ucp, d_core, ws);
    tm.mark();  // 6
    allreduce_sum(h, d_core, (size_t)prod(ranks));
    tm.mark();  // 7
    CK(cudaMemcpyAsync(hinfo, dinfo, info_bytes, cudaMemcpyDeviceToHost, h->stream));
  });
  tm.n = 8;
  if (!out_on_device) copy_out(h, core_out, d_core, sizeof(double) * prod(ranks), 0);
  if (!out_on_device || replicated)
    for (int k = 0; k < d; ++k)
      copy_out(h, factors_out[k], uptr[k], sizeof(double) * dims[k] * ranks[k], out_on_device);
  if (!end_call(h, rep || !out_on_device)) return;
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaGetLastError());
  for (int k = 0; k < d; ++k) {
    const int q = hinfo[4 * k];
    if (rep && rep->achieved_ranks) rep->achieved_ranks[k] = q;
    if (q < ranks[k])
      warnings.push_back("mode " + std::to_string(k) + ": sketch revealed rank " + std::to_string(q) + " < target " +
                         std::to_string(ranks[k]) + "; basis padded");
  }
  if (hinfo[4 * d] != 0) warnings.push_back(kU1ZeroWarning);
  if (rep) {
    if (rep->sample_counts)
      for (int k = 0; k < d; ++k) rep->sample_counts[k] = samples[k];
    finish_report_common(rep, tm, t_sampling, h->launches);
    rep->kernel_seconds[2] = kernel_pair(h, 2);
    rep->slice_mode = slice_mode;
    rep->flags = hinfo[4 * d] != 0 ? 1 : 0;
    write_warnings(rep, warnings);
  }
}

// ==================================================================================
// Column-range-sharded Sub-R-RtL-HT
// ==================================================================================
// The plan of one H-Tucker decomposition over a column range of the root
// matricization; shared by the fused NCCL entry and the three phase entries.
struct HtShard {
  // inputs
  Tree tr;
  int d = 0, nn = 0, nt = 0;
  std::vector<int64_t> dims, ranks, samples;
  int64_t p = 0, N = 0, nlr = 0, nrr = 0, col_lo = 0, col_hi = 0;
  bool whole = true;  // the range covers the tensor (no masking)
  bool replicated = false;  // X replicated on every rank: nodes assigned to ranks
  std::vector<char> mine;   // by target t (node t + 1): this rank's nodes
  size_t off_upack = 0;
  int64_t upack_n = 0;
  std::vector<std::vector<int64_t>> cols;
  std::vector<uint64_t> draws, state0;
  double t_sampling = 0;
  // workspace
  std::vector<int64_t> zoff, rows;
  int64_t zn = 0, max_n = 0;
  int cmax = 0;
  size_t off_zsum = 0, off_pad = 0, off_urs = 0, off_root = 0;
  std::vector<size_t> off_u, off_b, off_zp;
  std::vector<BasisPlan> bp;
  std::vector<BasisBuffers> bb;
  std::vector<int> internal;
  CoreJob core;
  // blob
  Blob blob;
  std::vector<size_t> off_cols;
  size_t off_sk = 0, off_bt = 0, off_tt = 0;
  std::vector<SketchTarget> sk;
  std::vector<BasisTarget> bt;
  std::vector<TransferTarget> tt;
  BasisLists lists;
  int64_t ctas = 0;
  int tctas = 0, max_rl = 1, max_rr = 1;
  char *ws = nullptr, *dp = nullptr, *hp = nullptr;
  int32_t *dinfo = nullptr, *hinfo = nullptr;

  int64_t node_rows(int i) const {
    int64_t r = 1;
    for (int m : tr.modes[i]) r *= dims[m];
    return r;
  }
  double* zsum() const { return reinterpret_cast<double*>(ws + off_zsum); }
  double* ubasis(int id) const { return reinterpret_cast<double*>(ws + off_u[id]); }
  double* btens(int id) const { return reinterpret_cast<double*>(ws + off_b[id]); }
  double* root() const { return reinterpret_cast<double*>(ws + off_root); }

  // Validation (htucker.hpp:217-233 order), sampling, workspace + blob.
  void build(srtt_handle* h, const double* x, int d_, const int64_t* dims_p, const srtt_tree* tree_p,
             const int64_t* ranks_p, const int64_t* samples_p, int64_t p_, uint64_t seed,
             const srtt_exec_policy* exec, int64_t clo, int64_t chi, bool replicated_ = false) {
    replicated = replicated_;
    if (d_ < 2 || d_ > SRTT_MAX_ORDER) invalid("sub_r_rtl_ht: unsupported order");
    d = d_;
    dims.assign(dims_p, dims_p + d);
    for (int k = 0; k < d; ++k)
      if (dims[k] < 1) invalid("Shape: dimensions must be >= 1");
    tr = read_tree(tree_p, d);
    nn = tr.n;
    nt = nn - 1;
    ranks.assign(ranks_p, ranks_p + nn);
    samples.assign(samples_p, samples_p + nn);
    p = p_;
    N = prod(dims);
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
    check_workers(exec, "tree_schedule");
    nlr = node_rows(tr.left[0]);
    nrr = node_rows(tr.right[0]);
    if (clo < 0 || chi > nrr || clo >= chi) invalid("sharded sub_r_rtl_ht: column range out of range");
    if (chi - clo < ranks[tr.right[0]])
      invalid("sharded sub_r_rtl_ht: every column range must hold at least r_right columns");
    col_lo = clo;
    col_hi = chi;
    whole = replicated || (clo == 0 && chi == nrr);
    // sampling: stream bound to the node id (htucker.hpp:264)
    const int64_t partitions = exec ? exec->index_partitions : 1;
    const double ts0 = now_s();
    cols.assign(nt, {});
    draws.assign(nt, 0);
    state0.assign(nt, 0);
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
    t_sampling = now_s() - ts0;

    // workspace
    Layout W;
    zoff.assign(nn, 0);
    rows.assign(nn, 0);
    off_u.assign(nn, 0);
    off_b.assign(nn, 0);
    bp.assign(nn, BasisPlan{});
    bb.assign(nn, BasisBuffers{});
    zn = 0;
    for (int i = 1; i < nn; ++i) {
      rows[i] = node_rows(i);
      zoff[i] = zn;
      zn += rows[i] * (ranks[i] + p);
      cmax = std::max<int>(cmax, (int)(ranks[i] + p));
      max_n = std::max(max_n, rows[i]);
    }
    off_zsum = W.take(sizeof(double) * zn);
    off_zp.assign(nn, 0);
    for (int i = 1; i < nn; ++i) off_zp[i] = W.take(sketch_part_bytes(rows[i], samples[i], (int)(ranks[i] + p)));
    upack_n = 0;
    for (int i = 1; i < nn; ++i) upack_n += rows[i] * ranks[i];
    off_upack = W.take(sizeof(double) * upack_n);  // every node basis, contiguous
    for (int i = 1, o = 0; i < nn; o += (int)(rows[i] * ranks[i]), ++i) {
      off_u[i] = off_upack + sizeof(double) * o;
      bp[i] = plan_basis(rows[i], (int)(ranks[i] + p), (int)ranks[i]);
      bb[i] = layout_basis(W, bp[i]);
    }
    off_pad = W.take(sizeof(double) * max_n * nt);
    for (int i = 1; i < nn; ++i)
      if (!tr.leaf(i)) {
        internal.push_back(i);
        off_b[i] = W.take(sizeof(double) * ranks[i] * ranks[tr.left[i]] * ranks[tr.right[i]]);
      }
    const int rl0 = (int)ranks[tr.left[0]], rr0 = (int)ranks[tr.right[0]];
    off_root = W.take(sizeof(double) * rl0 * rr0);
    off_urs = W.take(sizeof(double) * (chi - clo) * rr0);
    core.plan({nlr, chi - clo}, {rl0, rr0}, h->sms, W);
    h->ws.ensure(W.off);
    ws = reinterpret_cast<char*>(h->ws.p);
    dinfo = h->pset().dinfo();
    hinfo = h->pset().hinfo();

    // blob: indices, sketch / basis / transfer targets
    off_cols.assign(nt, 0);
    for (int t = 0; t < nt; ++t) off_cols[t] = blob.add(cols[t].data(), sizeof(int64_t) * cols[t].size());
    off_sk = blob.reserve(sizeof(SketchTarget) * nt);
    off_bt = blob.reserve(sizeof(BasisTarget) * nt);
    off_tt = blob.reserve(sizeof(TransferTarget) * std::max<size_t>(1, internal.size()));
    h->pset().d.ensure(blob.lay.off + 4096);
    dp = reinterpret_cast<char*>(h->pset().d.p);
    sk.assign(nt, SketchTarget{});
    bt.assign(nt, BasisTarget{});
    for (int t = 0; t < nt; ++t) {
      const int id = t + 1;
      const int c = (int)(ranks[id] + p);
      sk[t] = make_sketch_target(x, dims, tr.modes[id], samples[id], c);
      if (!whole) {  // x holds the flat range [col_lo n_l, col_hi n_l) only
        sk[t].flat_lo = col_lo * nlr;
        sk[t].flat_hi = col_hi * nlr;
      }
      sk[t].cols = reinterpret_cast<const int64_t*>(dp + off_cols[t]);
      sk[t].z = zsum() + zoff[id];
      sk[t].state0 = state0[t];
      sk[t].draw_offset = draws[t];
      sk[t].cta_begin = ctas;
      sk[t].flags = dinfo + 4 * nt;
      attach_sketch_scratch(sk[t], ws + off_zp[id]);
      ctas += sketch_target_ctas(sk[t]);
      bt[t] = fill_basis(bp[id], bb[id], ws, zsum() + zoff[id], ubasis(id), state0[t], draws[t], samples[id] * c,
                         dinfo + 4 * t);
    }
    mine.assign(nt, 1);
    if (replicated) {  // this rank's nodes only (LPT by n_S w_S (r_S + p))
      std::vector<double> cost(nt);
      for (int t = 0; t < nt; ++t) cost[t] = (double)rows[t + 1] * samples[t + 1] * (ranks[t + 1] + p);
      mine = assign_targets(cost, h->world, h->rank);
      std::vector<SketchTarget> sk_m;
      std::vector<BasisTarget> bt_m;
      ctas = 0;
      for (int t = 0; t < nt; ++t)
        if (mine[t]) {
          sk[t].cta_begin = ctas;
          ctas += sketch_target_ctas(sk[t]);
          sk_m.push_back(sk[t]);
          bt_m.push_back(bt[t]);
        }
      sk.swap(sk_m);
      bt.swap(bt_m);
    }
    assign_basis_ctas(bt);
    lists = make_basis_lists(bt, blob);
    for (int i : internal) {
      TransferTarget T{};
      T.us = ubasis(i);
      T.ul = ubasis(tr.left[i]);
      T.ur = ubasis(tr.right[i]);
      T.b = btens(i);
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
    h->pset().d.ensure(blob.lay.off);
    h->pset().hst.ensure(blob.lay.off);
    dp = reinterpret_cast<char*>(h->pset().d.p);
    hp = reinterpret_cast<char*>(h->pset().hst.p);
    for (auto& it : blob.items) std::memcpy(hp + it.first, it.second.data(), it.second.size());
    assign_contig_ctas(sk);
    if (!sk.empty()) std::memcpy(hp + off_sk, sk.data(), sizeof(SketchTarget) * sk.size());
    if (!bt.empty()) std::memcpy(hp + off_bt, bt.data(), sizeof(BasisTarget) * bt.size());
    if (!tt.empty()) std::memcpy(hp + off_tt, tt.data(), sizeof(TransferTarget) * tt.size());
  }

  void upload(srtt_handle* h) const {
    CK(cudaMemcpyAsync(dp, hp, blob.lay.off, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemsetAsync(dinfo, 0, sizeof(int32_t) * 4 * (nt + 1), h->stream));
    if (replicated) CK(cudaMemsetAsync(ws + off_upack, 0, sizeof(double) * upack_n, h->stream));
  }
  // Phase 1: partial sketches of every node (K1, one grouped launch).
  int enqueue_sketches(srtt_handle* h) const {
    if (sk.empty()) return 0;
    return launch_sketch_group(reinterpret_cast<const SketchTarget*>(dp + off_sk), sk, ctas, cmax, h->stream);
  }
  // Phase 2: bases of every node (K2) and the internal transfers (K4).
  // fork (the fused sharded path): as in the single-GPU decomposition the
  // single-CTA bases and the transfers run on the side stream and overlap
  // the tall bases and the root pass, which only needs the root children
  // (htucker.hpp:203-209); enqueue_join() closes the fork after the root.
  bool forked = false;
  int enqueue_bases(srtt_handle* h, bool fork = false) {
    forked = false;
    if (fork && replicated && !bt.empty()) {
      // replicated: the factor pack is complete only when both streams'
      // bases are; after its allreduce the transfers go to the side stream
      int n = 0;
      CK(cudaEventRecord(h->fj[0], h->stream));
      CK(cudaStreamWaitEvent(h->side, h->fj[0], 0));
      n += launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(dp + off_bt), lists, dp,
                              reinterpret_cast<double*>(ws + off_pad), max_n, h->side);
      CK(cudaEventRecord(h->fj[1], h->side));
      CK(cudaStreamWaitEvent(h->stream, h->fj[1], 0));
      allreduce_sum(h, reinterpret_cast<double*>(ws + off_upack), (size_t)upack_n);
      allreduce_sum_i32(h, dinfo, 4 * (size_t)(nt + 1));
      CK(cudaEventRecord(h->fj[2], h->stream));
      CK(cudaStreamWaitEvent(h->side, h->fj[2], 0));
      if (!tt.empty()) {
        CK(srtt_launch_transfer(reinterpret_cast<const TransferTarget*>(dp + off_tt), (int)tt.size(), tctas, max_rl,
                                max_rr, h->side));
        ++n;
      }
      CK(cudaEventRecord(h->fj[3], h->side));
      forked = true;
      return n;
    }
    if (fork && !replicated && !bt.empty()) {
      int n = 0;
      CK(cudaEventRecord(h->fj[0], h->stream));
      CK(cudaStreamWaitEvent(h->side, h->fj[0], 0));
      n += launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(dp + off_bt), lists, dp,
                              reinterpret_cast<double*>(ws + off_pad), max_n, h->side);
      CK(cudaEventRecord(h->fj[1], h->side));    // single-CTA bases done
      CK(cudaEventRecord(h->fj[2], h->stream));  // tall bases done
      CK(cudaStreamWaitEvent(h->side, h->fj[2], 0));
      if (!tt.empty()) {
        CK(srtt_launch_transfer(reinterpret_cast<const TransferTarget*>(dp + off_tt), (int)tt.size(), tctas, max_rl,
                                max_rr, h->side));
        ++n;
      }
      CK(cudaEventRecord(h->fj[3], h->side));
      bool root_needs_small = false;
      for (int t : lists.small)
        if (t + 1 == tr.left[0] || t + 1 == tr.right[0]) root_needs_small = true;  // target t is node t + 1
      if (root_needs_small) CK(cudaStreamWaitEvent(h->stream, h->fj[1], 0));
      forked = true;
      return n;
    }
    int n = bt.empty() ? 0
                       : launch_basis_group(h, bt, reinterpret_cast<const BasisTarget*>(dp + off_bt), lists, dp,
                                            reinterpret_cast<double*>(ws + off_pad), max_n);
    if (replicated) {  // every rank's node bases (others' entries are zero) and per-node info
      allreduce_sum(h, reinterpret_cast<double*>(ws + off_upack), (size_t)upack_n);
      allreduce_sum_i32(h, dinfo, 4 * (size_t)(nt + 1));
    }
    if (!tt.empty()) {
      CK(srtt_launch_transfer(reinterpret_cast<const TransferTarget*>(dp + off_tt), (int)tt.size(), tctas, max_rl,
                              max_rr, h->stream));
      ++n;
    }
    return n;
  }
  void enqueue_join(srtt_handle* h) {
    if (forked) CK(cudaStreamWaitEvent(h->stream, h->fj[3], 0));
    forked = false;
  }
  // Phase 3: this range's partial root transfer U_l^T M_w U_r[c_lo:c_hi].
  int enqueue_root(srtt_handle* h, const double* x, const double* ul, const double* ur_full, double* out) {
    const int rr0 = (int)ranks[tr.right[0]];
    const int64_t nc = col_hi - col_lo;
    double* urs = reinterpret_cast<double*>(ws + off_urs);
    CK(cudaMemcpy2DAsync(urs, sizeof(double) * nc, ur_full + col_lo, sizeof(double) * nrr, sizeof(double) * nc, rr0,
                         cudaMemcpyDeviceToDevice, h->stream));
    std::vector<const double*> u = {ul, urs};
    return core.launch(h, x, u, out, ws);
  }
  std::string key(srtt_handle* h, const double* x) const {
    std::string k = "HS";
    for (int m = 0; m < d; ++m) k += "|" + std::to_string(dims[m]);
    for (int i = 0; i < nn; ++i)
      k += "|" + std::to_string(ranks[i]) + "," + std::to_string(samples[i]) + "," + std::to_string(tr.left[i]) + "," +
           std::to_string(tr.modes[i].size());
    k += "|" + std::to_string(p) + "|" + std::to_string(col_lo) + "," + std::to_string(col_hi) + "|" + ptr_key(x) +
         "|" + ptr_key(ws) + "|" + ptr_key(dp) + "|" + ptr_key(hp) + "|" + ptr_key(h->stream) + "|" +
         ptr_key(h->comm) + "|" + std::to_string(blob.lay.off) + (h->timing ? "|t" : "|n");
    return k;
  }
  // Achieved ranks + warnings (htucker.hpp:326-333) from the host info copy.
  void collect(srtt_report* rep, std::vector<std::string>& warnings) const {
    for (int t = 0; t < nt; ++t) {
      const int id = t + 1;
      const int q = hinfo[4 * t];
      if (rep && rep->achieved_ranks) rep->achieved_ranks[id] = q;
      if (q < ranks[id])
        warnings.push_back("node " + std::to_string(id) + ": sketch revealed rank " + std::to_string(q) +
                           " < target; basis padded");
    }
    if (hinfo[4 * nt] != 0) warnings.push_back(kU1ZeroWarning);
    if (rep && rep->achieved_ranks) rep->achieved_ranks[0] = 1;
    if (rep && rep->sample_counts)
      for (int i = 0; i < nn; ++i) rep->sample_counts[i] = samples[i];
  }
};

void run_sub_r_rtl_ht_sharded(srtt_handle* h, const double* x_in, int x_on_device, int d, const int64_t* dims_p,
                              int64_t col_lo, int64_t col_hi, const srtt_tree* tree_p, const int64_t* ranks_p,
                              const int64_t* samples_p, int64_t p, uint64_t seed, const srtt_exec_policy* exec,
                              double* const* leaf_out, double* const* transfers_out, int out_on_device,
                              srtt_report* rep, bool replicated = false) {
  if (!h) invalid("srtt: null handle");
  comm_of(h);
  if (replicated) {  // the root pass is split by column ranges of the replica
    const Tree t = read_tree(tree_p, d);
    int64_t nr = 1;
    for (int m : t.modes[t.right[0]]) nr *= dims_p[m];
    if (h->world > nr) invalid("replicated sub_r_rtl_ht: more ranks than root columns");
    split_bounds(nr, h->world, h->rank, col_lo, col_hi);
  }
  DeviceGuard guard(h->device);
  h->launches = 0;
  begin_call(h);
  h->timing = rep != nullptr;
  struct TimingReset {
    srtt_handle* h;
    ~TimingReset() { h->timing = true; }
  } timing_reset{h};
  Timer tm{h};
  HtShard S;
  // x is only known after staging; the targets take the device pointer
  std::vector<int64_t> dv(dims_p, dims_p + std::max(d, 0));
  const int64_t Nfull = d >= 1 ? prod(dv) : 0;
  (void)Nfull;
  // the staged size needs the tree: build once with a null x to validate
  // and size, then point the targets at the staged buffer
  S.build(h, nullptr, d, dims_p, tree_p, ranks_p, samples_p, p, seed, exec, col_lo, col_hi, replicated);
  const int64_t nloc = replicated ? S.N : (col_hi - col_lo) * S.nlr;
  std::vector<std::string> warnings;
  if (p < 4) warnings.push_back("oversampling below the recommended minimum of 4");
  tm.mark();  // 0
  const double* x = stage_input(h, x_in, x_on_device, nloc);
  tm.mark();  // 1
  for (auto& t : S.sk) t.x = x;
  if (!S.sk.empty()) std::memcpy(S.hp + S.off_sk, S.sk.data(), sizeof(SketchTarget) * S.sk.size());
  const double* xroot = replicated ? x + col_lo * S.nlr : x;  // this rank's columns of M
  const bool serial_root = exec && exec->emulate_serial_root;  // all bases precede the root here anyway
  (void)serial_root;
  const int il = S.tr.left[0], ir = S.tr.right[0];
  const int rl0 = (int)S.ranks[il], rr0 = (int)S.ranks[ir];
  double* d_root = (out_on_device && transfers_out && transfers_out[0]) ? transfers_out[0] : S.root();
  std::string key = S.key(h, x) + "|" + ptr_key(d_root) + (replicated ? "|rep" : "|sh");
  run_enqueue(h, key, [&] {
    S.upload(h);
    tm.n = 2;
    tm.mark();  // 2
    h->launches += S.enqueue_sketches(h);
    tm.mark();  // 3
    if (!replicated) allreduce_sum(h, S.zsum(), (size_t)S.zn);
    tm.mark();  // 4
    h->launches += S.enqueue_bases(h, true);
    tm.mark();  // 5
    h->launches += S.enqueue_root(h, xroot, S.ubasis(il), S.ubasis(ir), d_root);
    S.enqueue_join(h);
    tm.mark();  // 6
    allreduce_sum(h, d_root, (size_t)rl0 * rr0);
    tm.mark();  // 7
    CK(cudaMemcpyAsync(S.hinfo, S.dinfo, sizeof(int32_t) * 4 * (S.nt + 1), cudaMemcpyDeviceToHost, h->stream));
  });
  tm.n = 8;
  // outputs: leaf factors by mode, transfers by node id (+ optional node bases)
  for (int i = 1; i < S.nn; ++i)
    if (S.tr.leaf(i)) {
      const int mode = S.tr.modes[i][0];
      copy_out(h, leaf_out[mode], S.ubasis(i), sizeof(double) * S.rows[i] * S.ranks[i], out_on_device);
    }
  if (transfers_out) {
    for (int i : S.internal)
      if (transfers_out[i])
        copy_out(h, transfers_out[i], S.btens(i),
                 sizeof(double) * S.ranks[i] * S.ranks[S.tr.left[i]] * S.ranks[S.tr.right[i]], out_on_device);
    if (transfers_out[0] && d_root != transfers_out[0])
      copy_out(h, transfers_out[0], d_root, sizeof(double) * rl0 * rr0, out_on_device);
  }
  if (rep && rep->node_bases)
    for (int i = 1; i < S.nn; ++i)
      if (rep->node_bases[i])
        copy_out(h, rep->node_bases[i], S.ubasis(i), sizeof(double) * S.rows[i] * S.ranks[i], out_on_device);
  if (!end_call(h, rep || !out_on_device)) return;
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaGetLastError());
  S.collect(rep, warnings);
  if (rep) {
    finish_report_common(rep, tm, S.t_sampling, h->launches);
    rep->stage_seconds[SRTT_STAGE_TTM] = 0.0;
    rep->stage_seconds[SRTT_STAGE_SERIAL_TAIL] = tm.between(5, 6);
    rep->kernel_seconds[2] = kernel_pair(h, 2);
    rep->flags = S.hinfo[4 * S.nt];
    write_warnings(rep, warnings);
  }
}

void release_comm(srtt_handle* h) {
  if (!h->comm) return;
  for (auto& gr : h->graphs)
    if (gr.second.exec) cudaGraphExecDestroy(gr.second.exec);
  h->graphs.clear();
  h->prepared.clear();
  const ncclComm_t c = reinterpret_cast<ncclComm_t>(h->comm);
  h->comm = nullptr;
  h->world = 1;
  h->rank = 0;
  nccl_check(nccl_api().comm_destroy(c), "ncclCommDestroy");
}

}  // namespace

extern "C" {

int srtt_comm_unique_id(void* id_out) {
  return guarded([&] {
    if (!id_out) invalid("srtt_comm_unique_id: null output");
    ncclUniqueId id;
    nccl_check(nccl_api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int srtt_comm_init(srtt_handle* h, int32_t world, int32_t rank, const void* unique_id) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (world < 1 || rank < 0 || rank >= world) invalid("srtt_comm_init: rank out of range");
    if (!unique_id) invalid("srtt_comm_init: null unique id");
    DeviceGuard g(h->device);
    if (h->comm) release_comm(h);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t c = nullptr;
    nccl_check(nccl_api().comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
    h->comm = c;
    h->world = world;
    h->rank = rank;
    // one tiny collective outside any graph capture: connections are set up
    // before the first captured decomposition
    DevBuf one;
    one.ensure(sizeof(double));
    CK(cudaMemsetAsync(one.p, 0, sizeof(double), h->own_stream));
    nccl_check(nccl_api().all_reduce(one.p, one.p, 1, ncclDouble, ncclSum, c, h->own_stream), "ncclAllReduce");
    CK(cudaStreamSynchronize(h->own_stream));
    h->graphs.clear();
    h->prepared.clear();
  });
}

int srtt_comm_destroy(srtt_handle* h) {
  return guarded([&] {
    if (!h || !h->comm) return;
    DeviceGuard g(h->device);
    CK(cudaStreamSynchronize(h->stream));
    release_comm(h);
  });
}

int srtt_comm_info(srtt_handle* h, int32_t* world, int32_t* rank) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (world) *world = h->comm ? h->world : 0;
    if (rank) *rank = h->comm ? h->rank : 0;
  });
}

int srtt_split_bounds(int64_t n, int32_t world, int32_t rank, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world) invalid("srtt_split_bounds: rank out of range");
    if (world > n) invalid("srtt_split_bounds: more ranks than slices");
    int64_t a = 0, b = 0;
    split_bounds(n, world, rank, a, b);
    if (lo) *lo = a;
    if (hi) *hi = b;
  });
}

int srtt_sub_r_hosvd_sharded(srtt_handle* h, const double* x_slab, int32_t x_on_device, int32_t d,
                             const int64_t* dims, int64_t slab_lo, int64_t slab_hi, const int64_t* ranks,
                             int64_t oversampling, const int64_t* samples, uint64_t seed,
                             const srtt_exec_policy* exec, double* core_out, double* const* factors_out,
                             int32_t out_on_device, srtt_report* rep) {
  return guarded([&] {
    run_sub_r_hosvd_sharded(h, x_slab, x_on_device, d, dims, slab_lo, slab_hi, ranks, oversampling, samples, seed,
                            exec, core_out, factors_out, out_on_device, rep);
  });
}

int srtt_sub_r_rtl_ht_sharded(srtt_handle* h, const double* x_cols, int32_t x_on_device, int32_t d,
                              const int64_t* dims, int64_t col_lo, int64_t col_hi, const srtt_tree* tree,
                              const int64_t* ranks, const int64_t* samples, int64_t oversampling, uint64_t seed,
                              const srtt_exec_policy* exec, double* const* leaf_factors_out,
                              double* const* transfers_out, int32_t out_on_device, srtt_report* rep) {
  return guarded([&] {
    run_sub_r_rtl_ht_sharded(h, x_cols, x_on_device, d, dims, col_lo, col_hi, tree, ranks, samples, oversampling,
                             seed, exec, leaf_factors_out, transfers_out, out_on_device, rep);
  });
}

int srtt_sub_r_hosvd_replicated(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                                const int64_t* dims, const int64_t* ranks, int64_t oversampling,
                                const int64_t* samples, uint64_t seed, const srtt_exec_policy* exec, double* core_out,
                                double* const* factors_out, int32_t out_on_device, srtt_report* rep) {
  return guarded([&] {
    run_sub_r_hosvd_sharded(h, x, x_on_device, d, dims, 0, 0, ranks, oversampling, samples, seed, exec, core_out,
                            factors_out, out_on_device, rep, true);
  });
}

int srtt_sub_r_rtl_ht_replicated(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                                 const srtt_tree* tree, const int64_t* ranks, const int64_t* samples,
                                 int64_t oversampling, uint64_t seed, const srtt_exec_policy* exec,
                                 double* const* leaf_factors_out, double* const* transfers_out, int32_t out_on_device,
                                 srtt_report* rep) {
  return guarded([&] {
    run_sub_r_rtl_ht_sharded(h, x, x_on_device, d, dims, 0, 0, tree, ranks, samples, oversampling, seed, exec,
                             leaf_factors_out, transfers_out, out_on_device, rep, true);
  });
}

// ---- H-Tucker phases (synchronous; the caller exchanges between them) ------
int srtt_ht_shard_sketches(srtt_handle* h, const double* x_cols, int32_t x_on_device, int32_t d,
                           const int64_t* dims, int64_t col_lo, int64_t col_hi, const srtt_tree* tree,
                           const int64_t* ranks, const int64_t* samples, int64_t oversampling, uint64_t seed,
                           const srtt_exec_policy* exec, double* const* z_out, int32_t out_on_device) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    DeviceGuard g(h->device);
    begin_call(h);
    HtShard S;
    S.build(h, nullptr, d, dims, tree, ranks, samples, oversampling, seed, exec, col_lo, col_hi);
    CompRef B = comp_bufs(h);
    const double* x = to_device(h, B.a, x_cols, (col_hi - col_lo) * S.nlr, x_on_device);
    for (auto& t : S.sk) t.x = x;
    if (!S.sk.empty()) std::memcpy(S.hp + S.off_sk, S.sk.data(), sizeof(SketchTarget) * S.sk.size());
    S.upload(h);
    S.enqueue_sketches(h);
    for (int i = 1; i < S.nn; ++i)
      if (z_out[i])
        copy_out(h, z_out[i], S.zsum() + S.zoff[i], sizeof(double) * S.rows[i] * (S.ranks[i] + S.p), out_on_device);
    end_call(h, true);
    CK(cudaStreamSynchronize(h->stream));
  });
}

int srtt_ht_bases_from_sketches(srtt_handle* h, int32_t d, const int64_t* dims, const srtt_tree* tree,
                                const int64_t* ranks, const int64_t* samples, int64_t oversampling, uint64_t seed,
                                const srtt_exec_policy* exec, const double* const* z, int32_t z_on_device,
                                double* const* node_bases_out, double* const* transfers_out, int32_t out_on_device,
                                int64_t* achieved_ranks) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    DeviceGuard g(h->device);
    begin_call(h);
    HtShard S;
    int64_t nr = 1;
    {
      const Tree t = read_tree(tree, d);
      for (int m : t.modes[t.right[0]]) nr *= dims[m];
    }
    S.build(h, nullptr, d, dims, tree, ranks, samples, oversampling, seed, exec, 0, nr);
    S.upload(h);
    for (int i = 1; i < S.nn; ++i)
      CK(cudaMemcpyAsync(S.zsum() + S.zoff[i], z[i], sizeof(double) * S.rows[i] * (S.ranks[i] + S.p),
                         z_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
    S.enqueue_bases(h);
    CK(cudaMemcpyAsync(S.hinfo, S.dinfo, sizeof(int32_t) * 4 * (S.nt + 1), cudaMemcpyDeviceToHost, h->stream));
    for (int i = 1; i < S.nn; ++i)
      if (node_bases_out && node_bases_out[i])
        copy_out(h, node_bases_out[i], S.ubasis(i), sizeof(double) * S.rows[i] * S.ranks[i], out_on_device);
    if (transfers_out)
      for (int i : S.internal)
        if (transfers_out[i])
          copy_out(h, transfers_out[i], S.btens(i),
                   sizeof(double) * S.ranks[i] * S.ranks[S.tr.left[i]] * S.ranks[S.tr.right[i]], out_on_device);
    end_call(h, true);
    CK(cudaStreamSynchronize(h->stream));
    if (achieved_ranks) {
      achieved_ranks[0] = 1;
      for (int t = 0; t < S.nt; ++t) achieved_ranks[t + 1] = S.hinfo[4 * t];
    }
  });
}

int srtt_ht_shard_root(srtt_handle* h, const double* x_cols, int32_t x_on_device, int64_t n_left, int64_t n_right,
                       int64_t col_lo, int64_t col_hi, const double* u_left, int32_t r_left, const double* u_right,
                       int32_t r_right, int32_t factors_on_device, double* b_out, int32_t out_on_device) {
  return guarded([&] {
    if (!h) invalid("srtt: null handle");
    if (col_lo < 0 || col_hi > n_right || col_lo >= col_hi) invalid("sharded root: column range out of range");
    DeviceGuard g(h->device);
    CompRef B = comp_bufs(h);
    const int64_t nc = col_hi - col_lo;
    const double* x = to_device(h, B.a, x_cols, nc * n_left, x_on_device);
    // U_r rows [c_lo, c_hi) as a contiguous block; the root pass is the K3
    // engine on M_w = n_left x nc (htucker.hpp:67-85 restricted to the range)
    B.d.ensure(sizeof(double) * nc * r_right);
    CK(cudaMemcpy2DAsync(B.d.p, sizeof(double) * nc, u_right + col_lo, sizeof(double) * n_right, sizeof(double) * nc,
                         r_right, factors_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
    DevBuf ul;
    const double* dul = to_device(h, ul, u_left, n_left * r_left, factors_on_device);
    const double* fs[2] = {dul, reinterpret_cast<const double*>(B.d.p)};
    const int64_t dd[2] = {n_left, nc}, rr[2] = {r_left, r_right};
    const int rc = srtt_multi_ttm_core(h, x, 1, 2, dd, rr, fs, 1, b_out, out_on_device);
    if (rc != SRTT_OK) throw Error{rc, g_last_error};
  });
}

}  // extern "C"
