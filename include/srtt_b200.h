/*
 * srtt_b200.h — C-ABI of the B200-native Sub-R Tucker / H-Tucker engine.
 *
 * This is the drop-in boundary for the reference's hot path (srtt, the C++
 * library of arxiv 2603.21379). The reference exposes C++ templates only and
 * no FFI; every entry point below replaces one reference function and keeps
 * its argument meaning, validation order, error messages and output layout:
 * tensors are flat with the FIRST index fastest (reference tensor.hpp:17-20),
 * matrices column-major (common.hpp:21-24), indices int64 (Eigen::Index).
 * Plain pointers and sizes only; no torch or CUDA types in the signatures.
 *
 * Error behaviour: every function returns a status code. The reference
 * throws std::invalid_argument / std::out_of_range / JobError; the matching
 * codes are SRTT_ERR_INVALID_ARGUMENT / SRTT_ERR_OUT_OF_RANGE, with the
 * reference's message text in srtt_last_error() (thread-local). The C++
 * wrapper (srtt_b200.hpp) rethrows the std exception.
 *
 * Pointer location: `*_on_device` = 0 means host memory (the library copies
 * host<->device inside the call; pinned host buffers make this fast),
 * 1 means CUDA device memory on the handle's device.
 *
 * Synchronisation: a decomposition with host outputs or a non-NULL report
 * returns after the work completed. With device outputs and rep == NULL,
 * srtt_sub_r_hosvd and srtt_sub_r_rtl_ht are stream-ordered like a cuBLAS
 * call: they return once the work is enqueued on the handle's stream
 * (srtt_set_stream), so back-to-back calls overlap host preparation with
 * device execution.
 */
#ifndef SRTT_B200_H
#define SRTT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRTT_OK 0
#define SRTT_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define SRTT_ERR_OUT_OF_RANGE 2     /* std::out_of_range */
#define SRTT_ERR_CUDA 3
#define SRTT_ERR_NCCL 4
#define SRTT_ERR_OUT_OF_MEMORY 5
#define SRTT_ERR_INTERNAL 6
#define SRTT_ERR_IO 8  /* IoError (io.hpp:10-13): bad magic/version, truncation, open failure */
#define SRTT_ERR_JOB 7 /* JobError(job): message starts with "job <index>: " */

/* Stage names of the reference's StageTimings (parallel.hpp:30-40) plus the
 * host<->device copies of this implementation. */
#define SRTT_STAGE_SAMPLING 0
#define SRTT_STAGE_EXTRACT 1 /* fused into SKETCH on the GPU: always 0 */
#define SRTT_STAGE_SKETCH 2
#define SRTT_STAGE_SVD 3
#define SRTT_STAGE_TRANSFER 4
#define SRTT_STAGE_TTM 5
#define SRTT_STAGE_GATHER 6
#define SRTT_STAGE_SERIAL_TAIL 7
#define SRTT_STAGE_FACTOR_WALL 8
#define SRTT_STAGE_H2D 9
#define SRTT_STAGE_D2H 10
#define SRTT_NUM_STAGES 11

typedef struct srtt_handle srtt_handle;

typedef struct srtt_options {
  int32_t device;     /* CUDA device ordinal */
  int32_t use_graphs; /* capture/replay the launch sequence in CUDA graphs */
  int32_t reserved[6];
} srtt_options;

/* ExecPolicy (parallel.hpp:23-28). The GPU schedule does not depend on
 * `workers` / `slice_mode` (every mode / node runs concurrently, the core
 * pass uses all SMs; the reference's results are bitwise independent of
 * them too, parallel.hpp:18-21), but both are VALIDATED as the reference
 * does, with its messages (SRTT_ERR_INVALID_ARGUMENT):
 *   workers < 1      -> "run_independent_jobs: workers must be >= 1" (Tucker,
 *                       parallel.hpp:88) / "tree_schedule: ..." (H-Tucker,
 *                       parallel.hpp:206);
 *   Tucker only (the reference then assembles the core with sliced_core):
 *   slice_mode = -1 (auto) resolves through pick_slice_mode
 *   (parallel.hpp:331-348; "pick_slice_mode: no mode can host N slices"),
 *   an explicit mode outside [0, d) -> "sliced_core: slice mode out of
 *   range", workers > extent of the slice mode -> "sliced_core: more workers
 *   than slices along the slicing mode" (parallel.hpp:369-373). The
 *   resolved slice mode is returned in srtt_report.slice_mode.
 * index_partitions selects sample_indices_partitioned (sampling.hpp:41-66,
 * bit-exact). emulate_serial_root makes the H-Tucker root pass wait for
 * every basis job (parallel.hpp:168-170); results are unchanged. */
typedef struct srtt_exec_policy {
  int64_t workers;
  int64_t slice_mode;
  int64_t index_partitions;
  int32_t emulate_serial_root;
  int32_t reserved;
} srtt_exec_policy;

/* SubsampleReport (tucker.hpp:129-134) / HtSubsampleReport
 * (htucker.hpp:196-201). Arrays are caller-allocated (d entries for Tucker,
 * num_nodes for H-Tucker) and may be NULL. Warnings are written
 * newline-separated into `warnings` (may be NULL). */
typedef struct srtt_report {
  int64_t* sample_counts;
  int64_t* achieved_ranks;
  char* warnings;
  int64_t warnings_capacity;
  int64_t num_warnings;
  double stage_seconds[SRTT_NUM_STAGES];
  int32_t flags; /* bit0: a Box-Muller u1 == 0 draw was met (p = 2^-53) */
  int32_t reserved;
  /* device time of the dominant kernels of the call (CUDA events around the
   * launch): [0] K1 sketch, [1] K2 basis (all launches), [2] K3/K5 core
   * streaming kernel only, [3] K4 transfers */
  double kernel_seconds[4];
  int64_t launches; /* kernels launched by the call */
  int64_t slice_mode; /* Tucker with a policy: the sliced_core slice mode the
                         reference would use (-1: no policy / H-Tucker) */
  /* optional, H-Tucker: node_bases[id] (id >= 1, non-NULL entries only)
   * receives the basis U_S of node id that the decomposition used
   * (n_S x r_S column-major, host or device memory as out_on_device). The
   * reference keeps the internal node bases private (htucker.hpp:244); they
   * are exported for parity checks of the internal nodes. */
  double* const* node_bases;
} srtt_report;

/* Dimension tree (dimension_tree.hpp:9-17), heap/BFS node order, root = 0.
 * Node i holds modes[mode_begin[i] .. mode_begin[i+1]) ascending. */
typedef struct srtt_tree {
  int32_t num_nodes;
  const int32_t* mode_begin; /* num_nodes + 1 */
  const int32_t* modes;
  const int32_t* left;  /* -1 for leaves */
  const int32_t* right; /* -1 for leaves */
} srtt_tree;

/* ---- handle ------------------------------------------------------------ */
int srtt_create(const srtt_options* opts, srtt_handle** out);
int srtt_destroy(srtt_handle* h);
const char* srtt_last_error(void);
int srtt_version(void);
/* Number of kernel launches issued by the last decomposition call. */
int64_t srtt_last_launch_count(srtt_handle* h);
/* Run all work of this handle on an external cudaStream_t (passed as void*;
 * NULL restores the handle's own (non-blocking) stream, which is NOT ordered
 * with the caller's streams). cudaStreamLegacy / cudaStreamPerThread are
 * accepted: the work is then ordered with that default stream (CUDA graphs
 * are captured on the own stream and launched into it). Lets a caller time
 * calls with its own CUDA events and consume device outputs in order. */
int srtt_set_stream(srtt_handle* h, void* stream);

/* ---- host-side sampling (bit-exact with the reference) ------------------ */
/* RngStream(seed, stream_id) + sample_indices / sample_indices_partitioned
 * (rng.hpp:30-62, sampling.hpp:14-66). `draws_out` (nullable) receives the
 * number of u64 draws the parent stream consumed (0 when partitioned). */
int srtt_sample_indices(uint64_t seed, uint64_t stream_id, int64_t m, int64_t s, int64_t partitions,
                        int64_t* idx_out, uint64_t* draws_out);
/* `n` normals of stream (seed, stream_id) starting after `draw_offset` u64
 * draws, normal index t0 on (the device generator, for parity tests). */
int srtt_stream_normals(srtt_handle* h, uint64_t seed, uint64_t stream_id, uint64_t draw_offset,
                        uint64_t t0, int64_t n, double* out);
/* pick_slice_mode (parallel.hpp:331-348): the mode whose extent needs the
 * least padding to a multiple of `workers`; INVALID_ARGUMENT when no mode
 * has at least `workers` slices. */
int srtt_pick_slice_mode(int32_t d, const int64_t* dims, int64_t workers, int64_t* mode_out);
/* DimensionTree::balanced (dimension_tree.hpp:36-64). Arrays sized
 * 2*order-1 (mode_begin: 2*order, modes: order*(depth+1) <= order*order). */
int srtt_tree_balanced(int32_t order, int32_t* num_nodes, int32_t* mode_begin, int32_t* modes,
                       int32_t* left, int32_t* right, int32_t* parent, int32_t* level);

/* ---- the two hot-path entry points -------------------------------------- */
/* sub_r_hosvd (tucker.hpp:177-242). core_out: prod(ranks) doubles (first
 * index fastest); factors_out[k]: dims[k] x ranks[k] column-major. */
int srtt_sub_r_hosvd(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                     const int64_t* dims, const int64_t* ranks, int64_t oversampling,
                     const int64_t* samples, uint64_t seed, const srtt_exec_policy* exec,
                     double* core_out, double* const* factors_out, int32_t out_on_device,
                     srtt_report* rep);

/* sub_r_rtl_ht (htucker.hpp:210-341). ranks / samples have one entry per
 * node (root entry of ranks must be 1). leaf_factors_out is indexed by MODE
 * (dims[m] x r_leaf); transfers_out by NODE id: r_S x r_l x r_r (root:
 * 1 x r_l x r_r), NULL entries for leaves. */
int srtt_sub_r_rtl_ht(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                      const int64_t* dims, const srtt_tree* tree, const int64_t* ranks,
                      const int64_t* samples, int64_t oversampling, uint64_t seed,
                      const srtt_exec_policy* exec, double* const* leaf_factors_out,
                      double* const* transfers_out, int32_t out_on_device, srtt_report* rep);

/* ---- component entry points (the reference's test-facing functions) ----- */
/* extract_group_fibers (unfolding.hpp:57-111); a single mode gives
 * extract_fibers (unfolding.hpp:32-52). y_out: n_S x ncols column-major. */
int srtt_extract_fibers(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                        const int64_t* dims, int32_t nmodes, const int32_t* modes, int64_t ncols,
                        const int64_t* cols, double* y_out, int32_t out_on_device);

/* K1 alone: Z = Y * Omega for one target, Omega drawn from stream
 * (seed, stream_id) after `draw_offset` draws (or given explicitly as
 * omega, ncols x c column-major, nullable). z_out: n_S x c. */
int srtt_sketch(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                int32_t nmodes, const int32_t* modes, int64_t ncols, const int64_t* cols, int32_t c,
                uint64_t seed, uint64_t stream_id, uint64_t draw_offset, const double* omega,
                double* z_out, int32_t out_on_device);

/* K2 alone: range_basis_of_sketch (sketch.hpp:74-93). z: n x c host or
 * device; q_out: n x rank; sv_out (nullable): min(n, c) singular values.
 * Padding continues stream (seed, stream_id) at normal index
 * normal_base after draw_offset draws. */
int srtt_range_basis_of_sketch(srtt_handle* h, const double* z, int32_t z_on_device, int64_t n,
                               int32_t c, int32_t rank, uint64_t seed, uint64_t stream_id,
                               uint64_t draw_offset, int64_t normal_base, double* q_out,
                               int64_t* numerical_rank, double* sv_out, int32_t out_on_device);

/* K3 alone: core = X x_0 U_0^T ... x_{d-1} U_{d-1}^T (core_from_factors,
 * tucker.hpp:43-50; sliced_core, parallel.hpp:355-445). factors[k]:
 * dims[k] x ranks[k] column-major (host or device per factors_on_device). */
int srtt_multi_ttm_core(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                        const int64_t* dims, const int64_t* ranks, const double* const* factors,
                        int32_t factors_on_device, double* core_out, int32_t out_on_device);

/* K4: transfer_tensor (htucker.hpp:44-63). b_out: rs x rl x rr. */
int srtt_transfer_tensor(srtt_handle* h, const double* u_node, const double* u_left,
                         const double* u_right, int64_t nl, int64_t nr, int32_t rs, int32_t rl,
                         int32_t rr, int32_t on_device, double* b_out);

/* K5: root_transfer (htucker.hpp:67-85). b_out: 1 x rl x rr. */
int srtt_root_transfer(srtt_handle* h, const double* x, int32_t x_on_device, int64_t nl,
                       int64_t nr, const double* u_left, int32_t rl, const double* u_right,
                       int32_t rr, int32_t factors_on_device, double* b_out,
                       int32_t out_on_device);

/* ---- reconstruction and error (the step after the path) -----------------
 * rel_error(reference, approx) = ||ref - approx||_F / ||ref||_F
 * (tensor.hpp:241-249; zero-norm reference -> INVALID_ARGUMENT). */
int srtt_rel_error(srtt_handle* h, const double* ref, const double* approx, int32_t on_device, int64_t n,
                   double* rel_error);
/* reconstruct (tucker.hpp:18-28): out = G x_0 U_0 ... x_{d-1} U_{d-1}
 * (prod dims doubles, first index fastest). core: prod ranks; factors[k]:
 * dims[k] x ranks[k] column-major. */
int srtt_tucker_reconstruct(srtt_handle* h, int32_t d, const int64_t* dims, const int64_t* ranks,
                            const double* core, const double* const* factors, int32_t in_on_device,
                            double* out, int32_t out_on_device);
/* rel_error(x, reconstruct(t)) streamed tile by tile: X-hat is never
 * materialised (experiment.cpp:248). */
int srtt_tucker_rel_error(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                          const int64_t* dims, const int64_t* ranks, const double* core,
                          const double* const* factors, int32_t in_on_device, double* rel_error);
/* ht_reconstruct (htucker.hpp:346-378); leaf_factors by MODE, transfers by
 * node id as srtt_sub_r_rtl_ht returns them; ranks per node (root = 1). */
int srtt_ht_reconstruct(srtt_handle* h, int32_t d, const int64_t* dims, const srtt_tree* tree,
                        const int64_t* ranks, const double* const* leaf_factors,
                        const double* const* transfers, int32_t in_on_device, double* out,
                        int32_t out_on_device);
/* rel_error(x, ht_reconstruct(h)) streamed (experiment.cpp:266). */
int srtt_ht_rel_error(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                      const int64_t* dims, const srtt_tree* tree, const int64_t* ranks,
                      const double* const* leaf_factors, const double* const* transfers,
                      int32_t in_on_device, double* rel_error);

/* ---- containers (io.hpp:15-33) ----------------------------------------------
 * "SRTT" dense tensor: magic, u32 version 1, u64 order, u64 dims, binary64
 * values (first index fastest), all little-endian. */
int srtt_tensor_file_info(const char* path, int32_t* order, int64_t* dims, int32_t dims_capacity,
                          int64_t* data_offset);
/* read_tensor (io.cpp:106-117). slab_lo = slab_hi = -1 reads everything;
 * otherwise only X[..., lo:hi) (one contiguous byte range), e.g. a rank's
 * slab for srtt_shard_*. out_on_device: streamed through pinned staging
 * (file reads overlap H2D copies on the handle's stream). */
int srtt_read_tensor(srtt_handle* h, const char* path, int64_t slab_lo, int64_t slab_hi, double* out,
                     int32_t out_on_device, int64_t out_capacity);
/* write_tensor (io.cpp:92-104); x may live on the device (h required). */
int srtt_write_tensor(srtt_handle* h, const char* path, int32_t d, const int64_t* dims, const double* x,
                      int32_t x_on_device);
/* "SRHT" hierarchical container (io.cpp:123-217), host buffers; layouts as
 * srtt_sub_r_rtl_ht returns them (ranks per node, root 1). */
int srtt_write_htucker(const char* path, int32_t d, const int64_t* dims, const srtt_tree* tree,
                       const int64_t* ranks, const double* const* leaf_factors,
                       const double* const* transfers);
/* Two-pass read: NULL arrays query order / num_nodes / num_modes; then pass
 * mode_begin[num_nodes+1], modes[num_modes], left/right/ranks[num_nodes],
 * dims[order] and the block buffers (NULL entries are skipped). */
int srtt_read_htucker(const char* path, int32_t* order, int32_t* num_nodes, int32_t* num_modes,
                      int32_t* mode_begin, int32_t* modes, int32_t* left, int32_t* right, int64_t* ranks,
                      int64_t* dims, double* const* leaf_factors, double* const* transfers);

/* ---- slab-sharded Sub-R-HOSVD (one process per GPU) --------------------
 * X is split along its LAST mode: the caller holds X[..., lo:hi) as a flat
 * first-index-fastest tensor with dims[d-1] replaced by hi - lo; `dims`
 * below are the GLOBAL extents. Every rank samples the same fibres and the
 * same Omega (same seed). The three phases and the exchanges between them
 * (the caller's collectives, e.g. NCCL via torch.distributed):
 *   1. srtt_shard_sketches: z_out[k], k < d-1: dims[k] x (r_k+p) PARTIAL
 *      sketch (fibres of other slabs contribute zero)  -> allreduce(sum);
 *      z_out[d-1]: rows [lo, hi) of Z_{d-1}, (hi-lo) x (r+p) -> allgather.
 *   2. srtt_bases_from_sketches: identical factors on every rank.
 *   3. srtt_shard_core: this slab's partial core (U_{d-1} restricted to
 *      rows [lo, hi))                                      -> allreduce(sum).
 * This is sliced_core's slab algebra (parallel.hpp:355-445) across GPUs. */
int srtt_shard_sketches(srtt_handle* h, const double* x_local, int32_t x_on_device, int32_t d,
                        const int64_t* dims, int64_t slab_lo, int64_t slab_hi, const int64_t* ranks,
                        int64_t oversampling, const int64_t* samples, uint64_t seed,
                        const srtt_exec_policy* exec, double* const* z_out, int32_t out_on_device);
int srtt_bases_from_sketches(srtt_handle* h, int32_t d, const int64_t* dims, const int64_t* ranks,
                             int64_t oversampling, const int64_t* samples, uint64_t seed,
                             const srtt_exec_policy* exec, const double* const* z, int32_t z_on_device,
                             double* const* factors_out, int32_t out_on_device,
                             int64_t* achieved_ranks);
int srtt_shard_core(srtt_handle* h, const double* x_local, int32_t x_on_device, int32_t d,
                    const int64_t* dims, int64_t slab_lo, int64_t slab_hi, const int64_t* ranks,
                    const double* const* factors, int32_t factors_on_device, double* core_partial_out,
                    int32_t out_on_device);

/* ---- multi-GPU: one process per GPU, NCCL over NVLink -------------------
 * The handle owns an NCCL communicator (libnccl.so.2 is resolved at run
 * time; SRTT_ERR_NCCL when it is missing). One rank creates the unique id
 * (SRTT_UNIQUE_ID_BYTES opaque bytes) and the caller distributes it (MPI,
 * torch.distributed, a file, ...); every rank then calls srtt_comm_init.
 * The sharded decompositions below run their kernels and the NCCL
 * collectives on the handle's stream, captured in one CUDA graph per call
 * signature (use_graphs), and return identical outputs on every rank.
 * Reference: sliced_core's slab algebra (parallel.hpp:355-445) and the
 * H-Tucker job DAG (htucker.hpp:249-324, root_transfer :67-85) across GPUs;
 * the reference's own engine is shared-memory threads only. */
#define SRTT_UNIQUE_ID_BYTES 128
int srtt_comm_unique_id(void* id_out);
int srtt_comm_init(srtt_handle* h, int32_t world, int32_t rank, const void* unique_id);
int srtt_comm_destroy(srtt_handle* h);
/* world = 0 when the handle has no communicator. */
int srtt_comm_info(srtt_handle* h, int32_t* world, int32_t* rank);
/* [lo, hi) of part `rank` of n slices over `world` parts: the contiguous
 * split of parallel.hpp:400-404 (sizes differ by at most one). */
int srtt_split_bounds(int64_t n, int32_t world, int32_t rank, int64_t* lo, int64_t* hi);

/* sub_r_hosvd (tucker.hpp:177-242) of a tensor split along its LAST mode:
 * this rank passes X[..., slab_lo:slab_hi) (flat, first index fastest) and
 * the GLOBAL dims. Exchanges: ONE allreduce of all sketches (sum_k
 * dims[k] (r_k + p) doubles; the slab mode's rows are owned by one rank each)
 * and ONE allreduce of the partial core (prod r_k doubles). Every slab must
 * hold at least r_{d-1} slices. Outputs and report as srtt_sub_r_hosvd;
 * report stage "gather" = the two exchanges. */
int srtt_sub_r_hosvd_sharded(srtt_handle* h, const double* x_slab, int32_t x_on_device, int32_t d,
                             const int64_t* dims, int64_t slab_lo, int64_t slab_hi, const int64_t* ranks,
                             int64_t oversampling, const int64_t* samples, uint64_t seed,
                             const srtt_exec_policy* exec, double* core_out, double* const* factors_out,
                             int32_t out_on_device, srtt_report* rep);
/* sub_r_rtl_ht (htucker.hpp:210-341) of a tensor split into column ranges
 * of the root matricization M = n_left x n_right (n_left = prod of the
 * root's left-child extents): this rank passes columns [col_lo, col_hi) of
 * M, i.e. the flat range [col_lo n_left, col_hi n_left) of X. Exchanges:
 * ONE allreduce of every node's partial sketch (sum_S n_S (r_S + p)
 * doubles) and ONE allreduce of the partial root transfer (r_l r_r). */
int srtt_sub_r_rtl_ht_sharded(srtt_handle* h, const double* x_cols, int32_t x_on_device, int32_t d,
                              const int64_t* dims, int64_t col_lo, int64_t col_hi, const srtt_tree* tree,
                              const int64_t* ranks, const int64_t* samples, int64_t oversampling, uint64_t seed,
                              const srtt_exec_policy* exec, double* const* leaf_factors_out,
                              double* const* transfers_out, int32_t out_on_device, srtt_report* rep);
/* Replicated X (the tensor fits every GPU; the north star's mode/node-
 * parallel regime): every rank passes ALL of X. Modes (Tucker) or non-root
 * nodes (H-Tucker) are assigned to ranks by greedy longest-processing-time
 * on n_S s_S (r_S + p) -- the reference's per-mode / per-node jobs
 * (parallel.hpp:133-147, 205-277) spread over GPUs instead of threads --;
 * each rank sketches and factors only its targets into a zero-filled pack,
 * ONE allreduce of the pack (plus one of the per-target info words) gives
 * every rank every basis, and the full pass is split by last-mode slabs
 * (Tucker) or root-matricization column ranges (H-Tucker) of the replica
 * and allreduced. Outputs are identical on every rank. */
int srtt_sub_r_hosvd_replicated(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d,
                                const int64_t* dims, const int64_t* ranks, int64_t oversampling,
                                const int64_t* samples, uint64_t seed, const srtt_exec_policy* exec, double* core_out,
                                double* const* factors_out, int32_t out_on_device, srtt_report* rep);
int srtt_sub_r_rtl_ht_replicated(srtt_handle* h, const double* x, int32_t x_on_device, int32_t d, const int64_t* dims,
                                 const srtt_tree* tree, const int64_t* ranks, const int64_t* samples,
                                 int64_t oversampling, uint64_t seed, const srtt_exec_policy* exec,
                                 double* const* leaf_factors_out, double* const* transfers_out, int32_t out_on_device,
                                 srtt_report* rep);
/* The H-Tucker split as synchronous phases (same plan and kernels as the
 * fused entry; the caller exchanges between them, any transport):
 *   1. srtt_ht_shard_sketches: z_out[id] (id >= 1, n_S x (r_S + p)) = this
 *      range's PARTIAL sketch of node id                  -> allreduce(sum);
 *   2. srtt_ht_bases_from_sketches: node bases (n_S x r_S, by node id) and
 *      internal transfers (by node id) -- identical on every rank;
 *   3. srtt_ht_shard_root: U_l^T M[:, c_lo:c_hi] U_r[c_lo:c_hi, :]
 *      (r_l x r_r)                                         -> allreduce(sum). */
int srtt_ht_shard_sketches(srtt_handle* h, const double* x_cols, int32_t x_on_device, int32_t d,
                           const int64_t* dims, int64_t col_lo, int64_t col_hi, const srtt_tree* tree,
                           const int64_t* ranks, const int64_t* samples, int64_t oversampling, uint64_t seed,
                           const srtt_exec_policy* exec, double* const* z_out, int32_t out_on_device);
int srtt_ht_bases_from_sketches(srtt_handle* h, int32_t d, const int64_t* dims, const srtt_tree* tree,
                                const int64_t* ranks, const int64_t* samples, int64_t oversampling, uint64_t seed,
                                const srtt_exec_policy* exec, const double* const* z, int32_t z_on_device,
                                double* const* node_bases_out, double* const* transfers_out, int32_t out_on_device,
                                int64_t* achieved_ranks);
int srtt_ht_shard_root(srtt_handle* h, const double* x_cols, int32_t x_on_device, int64_t n_left, int64_t n_right,
                       int64_t col_lo, int64_t col_hi, const double* u_left, int32_t r_left, const double* u_right,
                       int32_t r_right, int32_t factors_on_device, double* b_out, int32_t out_on_device);

#ifdef __cplusplus
}
#endif
#endif /* SRTT_B200_H */
