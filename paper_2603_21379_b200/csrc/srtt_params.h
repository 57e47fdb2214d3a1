// Plain-C parameter blocks shared by the host planner (host.cu) and the
// sm_100a kernels. Everything is POD so a whole array of targets travels to
// the device in one cudaMemcpyAsync and the launch sequence can be captured
// once in a CUDA graph and replayed with new seeds.
#pragma once
#include <stdint.h>

#define SRTT_MAX_ORDER 16
#define SRTT_MAX_SKETCH_COLS 64  // r + p limit of the basis kernels

// ---------------------------------------------------------------------------
// K1: fused fiber gather + in-kernel Gaussian sketch, Z = Y * Omega.
// One "target" is a Tucker mode (tucker.hpp:141-168) or an H-Tucker node
// (htucker.hpp:263-287). Y is never materialised: each sampled fibre element
// is loaded into a register and immediately multiplied into Z.
// ---------------------------------------------------------------------------
typedef struct SketchTarget {
  const double* x;        // tensor data (first index fastest)
  const int64_t* cols;    // w sampled columns of the (mode-set) unfolding
  const double* omega;    // optional explicit Omega (w x c, column-major); NULL = generate
  double* z;              // out: rows x c, column-major (ld = rows)
  int64_t rows;           // n_S
  int64_t w;              // fibres sampled
  int32_t c;              // r + p
  int32_t nrow_modes;     // modes of S (ascending): row digit decode
  int32_t ncol_modes;     // complement modes (ascending): column digit decode
  int32_t row_tile;       // rows handled per CTA
  int64_t row_dim[SRTT_MAX_ORDER];
  int64_t row_stride[SRTT_MAX_ORDER];
  int64_t col_dim[SRTT_MAX_ORDER];
  int64_t col_stride[SRTT_MAX_ORDER];
  uint64_t state0;        // RngStream(seed, id) initial state (rng.hpp:30-36)
  uint64_t draw_offset;   // u64 draws consumed by the sampling step
  int64_t cta_begin;      // first CTA index of this target in the grouped grid
  int32_t* flags;         // device status word (bit 0: Box-Muller u1 == 0 met)
  // slab sharding: the column digit at position slab_digit (of the
  // complement decode) must lie in [slab_lo, slab_hi); fibres outside the
  // local slab contribute zero, inside ones are shifted by slab_lo*stride
  int32_t slab_digit;     // -1: no slab restriction
  int32_t pad0;
  int64_t slab_lo, slab_hi;
  // flat-range sharding (H-Tucker, X split into column ranges of the root
  // matricization): x holds only the flat range [flat_lo, flat_hi) of the
  // global tensor; elements outside it contribute zero (flat_hi = 0: off)
  int64_t flat_lo, flat_hi;
  // leading dimension of z (0: rows); lets a rank write its rows of a
  // row-distributed sketch into a zero-filled full-height buffer
  int64_t ldz;
  // fibre split: the w fibres are cut into fsplit contiguous chunks handled
  // by different CTAs (grid = row tiles x fsplit); each chunk's partial Z
  // goes to zpart[(f * c + cc) * rows + i] and a second kernel sums the
  // chunks in a fixed order (deterministic). fsplit = 1: direct write.
  int32_t fsplit;
  int32_t pad1;
  double* zpart;
} SketchTarget;

// ---------------------------------------------------------------------------
// K2: basis of a sketch (sketch.hpp:74-93): Householder TSQR of Z, one-sided
// Jacobi SVD of the small triangular factor, rank decision at
// tol = max(rows, cols) * eps * sigma_1, U = Q * V[:, :q], Gaussian padding
// from the same stream.
// ---------------------------------------------------------------------------
typedef struct QrLevel {
  double* a;       // level matrix (n_l x c, ld = n_l); overwritten with reflectors
  double* tau;     // nblk x c
  double* r_out;   // stacked R of the next level (nblk*c x c, ld = nblk*c) (NULL at top)
  double* y;       // back-application buffer for this level (n_l x r, ld = n_l)
  int64_t n;       // rows at this level
  int32_t nblk;    // row blocks at this level
  int32_t blk_rows;
} QrLevel;

#define SRTT_MAX_QR_LEVELS 6

typedef struct BasisTarget {
  double* u;              // out: n x r column-major (ld = n)
  double* sv;             // out: min(n, c) singular values, descending (may be NULL)
  int32_t* info;          // out: [0] achieved (numerical) rank q, [1] nrank, [2] flags
  int64_t n;              // sketch rows
  int32_t c;              // sketch columns (r + p)
  int32_t r;              // target rank
  int32_t nlevels;        // TSQR levels below the top (0 => single block)
  int32_t cta_begin[SRTT_MAX_QR_LEVELS];  // CTA offsets for grouped level launches
  QrLevel lv[SRTT_MAX_QR_LEVELS + 1];     // lv[0] = Z itself ... lv[nlevels] = top
  uint64_t state0;        // stream of the target (padding continues it)
  uint64_t draw_offset;   // draws consumed by sampling
  int64_t normal_base;    // normals already consumed by Omega (w * c)
} BasisTarget;

// ---------------------------------------------------------------------------
// K3/K5: fused multi-TTM streaming engine (see k_core.cu). X is viewed as
// M (n0 x Q), column-major; a work item is one column range of one row
// block inside one level-m group (m = 2 or 3). Each item writes
// R_m = X x_0 U_0^T ... x_{m-1} U_{m-1}^T restricted to its columns into a
// fixed output slot part[rho][sigma][p][A].
// ---------------------------------------------------------------------------
// One work item of the core pass, built on the device by the prep kernel.
typedef struct CoreItem {
  int64_t c_lo;      // first column (of M = n0 x Q)
  int64_t out_off;   // output slot offset (doubles) in part[]
  int64_t grp0;      // level-2 group of c_lo
  int32_t len;       // columns
  int32_t rho;       // row block
  int32_t off0;      // offset of c_lo inside its level-2 group
  int32_t pad;
} CoreItem;

typedef struct CoreParams {
  const double* x;
  const CoreItem* items;   // nitems descriptors (device)
  const double* ufrag;     // U0 in fragment order: [nrb][RB/4][NT][32]
  const double* fu[2];     // U_1, U_2 ROW-major (n_k x r_k)
  double* part;            // out: [nrb][S][G][A]
  int64_t n0;              // rows (mode 0 extent, or n_left for the root pass)
  int64_t Q;               // columns
  int64_t fdim[2];         // n_1, n_2
  int32_t frank[2];        // r_1, r_2
  int64_t GS;              // columns per level-m group
  int64_t G;               // number of groups
  int64_t SL;              // columns per split (multiple of 16)
  int64_t nitems;          // nrb * G * S
  int32_t S;               // splits per group
  int32_t m;               // fold depth (2 or 3)
  int32_t r0;              // rank of mode 0
  int32_t NT;              // 8-rank tiles of mode 0 (1, 2 or 4)
  int32_t NT1;             // 8-rank tiles of mode 1 (1, 2 or 4)
  int32_t RB;              // rows per row block (multiple of 16, <= 256)
  int32_t nrb;             // row blocks
  int32_t A;               // prod_{k<m} r_k (output entries per item)
  int32_t use_tma;         // 1: cp.async.bulk.tensor loads; 0: warp-copy path (odd n0)
  int32_t nstages;         // per-warp TMA ring depth
  int32_t tpb;             // 16-column tile pairs per TMA box (1 or 2)
  int32_t warps;           // warps per CTA (8 or 16)
  // flat mode (single row block): instead of items, global warp gw owns the
  // contiguous tile range [ntiles*gw/nw, ntiles*(gw+1)/nw) of BC-column
  // tiles; it writes one record per level-m group its range touches into
  // rec[(gw + p) * A], and the warp completing group p (counter cnt[p])
  // sums the group's records in warp order into part[p * A] (compact R_m).
  int32_t flat;
  int32_t nw;              // total warps of the grid (flat mode)
  int64_t ntiles;          // BC-column tiles of M (flat mode)
  double* rec;             // flat mode: (nw + G) * A record slots
  uint32_t* cnt;           // flat mode: G completion counters (zero between calls)
  // flat mode, short columns (n0 <= 64, r0 <= 8): one unswizzled TMA box
  // holds whole columns, pitch cb rows (cb >= n0, cb = 2 mod 4: the DMMA B
  // fragments of a half-warp then hit 16 distinct bank pairs); 0 = off
  int32_t cb;
  int32_t slot_ch;         // item mode, m = 2: CTA reduction chunk (0 = all A at once)
} CoreParams;

// Streamed reconstruction error (k_recon.cu).
typedef struct ResidualParams {
  const double* x;       // n_A x n_B (first index fastest); unused when out is set
  const double* at;      // K x n_A
  const double* ct;      // K x n_B
  double* out;           // optional: write A C^T instead of the norms
  double* partial;       // 2 doubles per CTA
  int64_t nA, nB;
  int32_t K;             // padded to a multiple of 8 (zero rows in At / Ct)
  int32_t x_tma;         // X through a TMA map (n_A even) or cp.async
  int32_t stages;        // set by the launcher
  int32_t pad;
} ResidualParams;

typedef struct KronParams {
  const double* u[16];   // U_k, n_k x r_k column-major
  int64_t n[16], r[16];
  double* at;            // K x n_A
  int64_t K, nA;
  int32_t m, pad;
} KronParams;

// Generic small TTM used by the tail of the core pass and by reconstruct:
// out(g, b, post) = sum_i in(g, i, post) * U(i, b)   (U given as n x r).
// When nparts > 1 the input is a sum of nparts partial tensors spaced by
// part_stride (fixed summation order: deterministic).
typedef struct TtmParams {
  const double* in;
  const double* u;       // column-major n x rr (ld = n); transpose flag picks U vs U^T
  double* out;
  int64_t g, n, post;    // input viewed as g x n x post
  int64_t rr;            // output extent along the mode
  int32_t transpose;     // 1: contract with U^T (u is n x rr) ; 0: with U (u is rr x n)
  int32_t nparts;
  int64_t part_stride;
  double* scratch;          // optional workspace for split-K partials (NULL: not used)
  int64_t scratch_doubles;
} TtmParams;
