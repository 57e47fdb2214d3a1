// srtt_b200.hpp — header-only C++ mirror of the reference's hot-path API
// (proj/include/srtt/{tucker,htucker,dimension_tree,parallel}.hpp) on top
// of the C-ABI in srtt_b200.h. Same names, argument meaning and exception
// types: std::invalid_argument, std::out_of_range, srtt::JobError. Storage
// follows the reference: DenseTensor flat, first index fastest; Matrix
// column-major. No Eigen dependency: Matrix is a minimal column-major
// container (rows(), cols(), operator()(i, j), data()).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "srtt_b200.h"

namespace srtt {

using Index = std::int64_t;
using Ranks = std::vector<Index>;
using NodeRanks = std::vector<Index>;

class JobError : public std::runtime_error {
 public:
  JobError(std::size_t job, const std::string& what) : std::runtime_error(what), job_(job) {}
  std::size_t job() const { return job_; }

 private:
  std::size_t job_;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == SRTT_OK) return;
  const std::string msg = srtt_last_error();
  switch (rc) {
    case SRTT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SRTT_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case SRTT_ERR_JOB: {
      std::size_t job = 0;
      if (msg.rfind("job ", 0) == 0) job = std::stoul(msg.substr(4));
      throw JobError(job, msg);
    }
    default: throw DeviceError(msg);
  }
}
}  // namespace detail

template <class Scalar>
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : rows_(r), cols_(c), data_(static_cast<std::size_t>(r * c)) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Scalar& operator()(Index i, Index j) { return data_[static_cast<std::size_t>(i + j * rows_)]; }
  Scalar operator()(Index i, Index j) const { return data_[static_cast<std::size_t>(i + j * rows_)]; }
  Scalar* data() { return data_.data(); }
  const Scalar* data() const { return data_.data(); }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<Scalar> data_;
};

class Shape {
 public:
  Shape() = default;
  explicit Shape(std::vector<Index> dims) : dims_(std::move(dims)) {
    if (dims_.empty()) throw std::invalid_argument("Shape: order must be >= 1");
    for (Index n : dims_)
      if (n < 1) throw std::invalid_argument("Shape: dimensions must be >= 1");
  }
  Shape(std::initializer_list<Index> d) : Shape(std::vector<Index>(d)) {}
  Index order() const { return static_cast<Index>(dims_.size()); }
  Index dim(Index k) const { return dims_[static_cast<std::size_t>(k)]; }
  const std::vector<Index>& dims() const { return dims_; }
  Index num_elements() const {
    Index p = 1;
    for (Index n : dims_) p *= n;
    return p;
  }

 private:
  std::vector<Index> dims_;
};

template <class Scalar>
class DenseTensor {
 public:
  DenseTensor() = default;
  explicit DenseTensor(Shape s) : shape_(std::move(s)), data_(static_cast<std::size_t>(shape_.num_elements())) {}
  const Shape& shape() const { return shape_; }
  Index order() const { return shape_.order(); }
  Index dim(Index k) const { return shape_.dim(k); }
  Index size() const { return static_cast<Index>(data_.size()); }
  Scalar* data() { return data_.data(); }
  const Scalar* data() const { return data_.data(); }
  Scalar& operator[](Index i) { return data_[static_cast<std::size_t>(i)]; }
  Scalar operator[](Index i) const { return data_[static_cast<std::size_t>(i)]; }

 private:
  Shape shape_;
  std::vector<Scalar> data_;
};

struct ExecPolicy {  // parallel.hpp:23-28
  Index workers = 1;
  std::optional<Index> slice_mode;
  Index index_partitions = 1;
  bool emulate_serial_root = false;
};

struct StageTimings {  // stage name -> seconds (device events + host sampling)
  std::vector<std::pair<std::string, double>> records;
};

struct SubsampleReport {  // tucker.hpp:129-134
  std::vector<Index> sample_counts;
  std::vector<Index> achieved_ranks;
  std::vector<std::string> warnings;
  StageTimings timings;
};
using HtSubsampleReport = SubsampleReport;

template <class Scalar>
struct TuckerDecomposition {
  DenseTensor<Scalar> core;
  std::vector<Matrix<Scalar>> factors;
};

/// Process-wide engine handle (device 0); one handle per host thread is the
/// C-ABI's rule, so each thread gets its own.
inline srtt_handle* engine() {
  thread_local struct Holder {
    srtt_handle* h = nullptr;
    ~Holder() {
      if (h) srtt_destroy(h);
    }
  } holder;
  if (!holder.h) {
    srtt_options o{};
    detail::check(srtt_create(&o, &holder.h));
  }
  return holder.h;
}

namespace detail {
inline srtt_exec_policy to_c(const ExecPolicy& p) {
  srtt_exec_policy e{};
  e.workers = p.workers;
  e.slice_mode = p.slice_mode ? *p.slice_mode : -1;
  e.index_partitions = p.index_partitions;
  e.emulate_serial_root = p.emulate_serial_root ? 1 : 0;
  return e;
}

inline void fill_report(const srtt_report& r, std::size_t n, const std::vector<std::int64_t>& sc,
                        const std::vector<std::int64_t>& ach, const std::string& warn, SubsampleReport* out) {
  if (!out) return;
  static const char* kNames[SRTT_NUM_STAGES] = {"sampling", "extract", "sketch", "svd", "transfer", "ttm",
                                                "gather", "serial_tail", "factor_wall", "h2d", "d2h"};
  out->sample_counts.assign(sc.begin(), sc.begin() + static_cast<std::ptrdiff_t>(n));
  out->achieved_ranks.assign(ach.begin(), ach.begin() + static_cast<std::ptrdiff_t>(n));
  out->warnings.clear();
  std::size_t pos = 0;
  while (pos < warn.size()) {
    const std::size_t e = warn.find('\n', pos);
    if (e == std::string::npos) break;
    out->warnings.push_back(warn.substr(pos, e - pos));
    pos = e + 1;
  }
  out->timings.records.clear();
  for (int i = 0; i < SRTT_NUM_STAGES; ++i) out->timings.records.emplace_back(kNames[i], r.stage_seconds[i]);
}
}  // namespace detail

/// sub_r_hosvd (tucker.hpp:177-242) on the B200.
template <class Scalar>
TuckerDecomposition<Scalar> sub_r_hosvd(const DenseTensor<Scalar>& x, const Ranks& target, Index oversampling,
                                        const Ranks& samples, std::uint64_t seed,
                                        const std::optional<ExecPolicy>& exec = std::nullopt,
                                        SubsampleReport* report = nullptr) {
  static_assert(sizeof(Scalar) == sizeof(double), "the B200 engine computes in fp64");
  const Index d = x.order();
  if (static_cast<Index>(target.size()) != d)
    throw std::invalid_argument("sub_r_hosvd: rank vector order mismatch");
  if (samples.size() != target.size()) throw std::invalid_argument("sub_r_hosvd: samples vector order mismatch");
  TuckerDecomposition<Scalar> out;
  out.core = DenseTensor<Scalar>(Shape(target));
  std::vector<double*> fptr;
  for (Index k = 0; k < d; ++k) {
    out.factors.emplace_back(x.dim(k), target[static_cast<std::size_t>(k)]);
    fptr.push_back(out.factors.back().data());
  }
  std::vector<std::int64_t> sc(static_cast<std::size_t>(d)), ach(static_cast<std::size_t>(d));
  std::string warn(8192, '\0');
  srtt_report rep{};
  rep.sample_counts = sc.data();
  rep.achieved_ranks = ach.data();
  rep.warnings = warn.data();
  rep.warnings_capacity = static_cast<std::int64_t>(warn.size());
  srtt_exec_policy e{};
  if (exec) e = detail::to_c(*exec);
  detail::check(srtt_sub_r_hosvd(engine(), x.data(), 0, static_cast<std::int32_t>(d), x.shape().dims().data(),
                                 target.data(), oversampling, samples.data(), seed, exec ? &e : nullptr,
                                 out.core.data(), fptr.data(), 0, &rep));
  warn.resize(warn.find('\0'));
  detail::fill_report(rep, static_cast<std::size_t>(d), sc, ach, warn, report);
  return out;
}

struct TreeNode {
  std::vector<Index> modes;
  Index left = -1, right = -1, parent = -1, level = 0;
  bool is_leaf() const { return left < 0; }
};

/// DimensionTree (dimension_tree.hpp:27-152).
class DimensionTree {
 public:
  explicit DimensionTree(std::vector<TreeNode> nodes) : nodes_(std::move(nodes)) {}
  static DimensionTree balanced(Index order) {
    const int n = static_cast<int>(2 * order - 1);
    std::int32_t num = 0;
    std::vector<std::int32_t> mb(static_cast<std::size_t>(n + 1)), modes(static_cast<std::size_t>(order * order)),
        l(static_cast<std::size_t>(n)), r(static_cast<std::size_t>(n)), p(static_cast<std::size_t>(n)),
        lv(static_cast<std::size_t>(n));
    detail::check(srtt_tree_balanced(static_cast<std::int32_t>(order), &num, mb.data(), modes.data(), l.data(),
                                     r.data(), p.data(), lv.data()));
    std::vector<TreeNode> nodes(static_cast<std::size_t>(num));
    for (int i = 0; i < num; ++i) {
      for (int k = mb[i]; k < mb[i + 1]; ++k) nodes[i].modes.push_back(modes[k]);
      nodes[i].left = l[i];
      nodes[i].right = r[i];
      nodes[i].parent = p[i];
      nodes[i].level = lv[i];
    }
    return DimensionTree(std::move(nodes));
  }
  Index num_nodes() const { return static_cast<Index>(nodes_.size()); }
  const TreeNode& node(Index i) const { return nodes_[static_cast<std::size_t>(i)]; }
  Index order() const { return static_cast<Index>(nodes_[0].modes.size()); }

 private:
  std::vector<TreeNode> nodes_;
};

template <class Scalar>
struct HTuckerDecomposition {
  DimensionTree tree;
  std::vector<Matrix<Scalar>> leaf_factors;   // by mode
  std::vector<DenseTensor<Scalar>> transfers;  // by node id, empty for leaves
};

/// sub_r_rtl_ht (htucker.hpp:210-341) on the B200.
template <class Scalar>
HTuckerDecomposition<Scalar> sub_r_rtl_ht(const DenseTensor<Scalar>& x, const DimensionTree& tree,
                                          const NodeRanks& ranks, const NodeRanks& samples, Index oversampling,
                                          std::uint64_t seed, const std::optional<ExecPolicy>& exec = std::nullopt,
                                          HtSubsampleReport* report = nullptr) {
  const Index nn = tree.num_nodes(), d = x.order();
  if (tree.order() != d) throw std::invalid_argument("sub_r_rtl_ht: tree and tensor order mismatch");
  if (static_cast<Index>(ranks.size()) != nn)
    throw std::invalid_argument("sub_r_rtl_ht: rank vector must have one entry per node");
  if (static_cast<Index>(samples.size()) != nn)
    throw std::invalid_argument("sub_r_rtl_ht: samples vector must have one entry per node");
  std::vector<std::int32_t> mb{0}, modes, l, r;
  for (Index i = 0; i < nn; ++i) {
    for (Index m : tree.node(i).modes) modes.push_back(static_cast<std::int32_t>(m));
    mb.push_back(static_cast<std::int32_t>(modes.size()));
    l.push_back(static_cast<std::int32_t>(tree.node(i).left));
    r.push_back(static_cast<std::int32_t>(tree.node(i).right));
  }
  srtt_tree ct{static_cast<std::int32_t>(nn), mb.data(), modes.data(), l.data(), r.data()};
  HTuckerDecomposition<Scalar> out{tree, {}, {}};
  out.leaf_factors.resize(static_cast<std::size_t>(d));
  out.transfers.resize(static_cast<std::size_t>(nn));
  std::vector<double*> lp(static_cast<std::size_t>(d)), tp(static_cast<std::size_t>(nn), nullptr);
  for (Index i = 0; i < nn; ++i) {
    const TreeNode& n = tree.node(i);
    if (n.is_leaf()) {
      const Index m = n.modes[0];
      out.leaf_factors[static_cast<std::size_t>(m)] = Matrix<Scalar>(x.dim(m), ranks[static_cast<std::size_t>(i)]);
      lp[static_cast<std::size_t>(m)] = out.leaf_factors[static_cast<std::size_t>(m)].data();
    } else {
      out.transfers[static_cast<std::size_t>(i)] = DenseTensor<Scalar>(
          Shape{i == 0 ? 1 : ranks[static_cast<std::size_t>(i)], ranks[static_cast<std::size_t>(n.left)],
                ranks[static_cast<std::size_t>(n.right)]});
      tp[static_cast<std::size_t>(i)] = out.transfers[static_cast<std::size_t>(i)].data();
    }
  }
  std::vector<std::int64_t> sc(static_cast<std::size_t>(nn)), ach(static_cast<std::size_t>(nn));
  std::string warn(8192, '\0');
  srtt_report rep{};
  rep.sample_counts = sc.data();
  rep.achieved_ranks = ach.data();
  rep.warnings = warn.data();
  rep.warnings_capacity = static_cast<std::int64_t>(warn.size());
  srtt_exec_policy e{};
  if (exec) e = detail::to_c(*exec);
  detail::check(srtt_sub_r_rtl_ht(engine(), x.data(), 0, static_cast<std::int32_t>(d), x.shape().dims().data(), &ct,
                                  ranks.data(), samples.data(), oversampling, seed, exec ? &e : nullptr, lp.data(),
                                  tp.data(), 0, &rep));
  warn.resize(warn.find('\0'));
  detail::fill_report(rep, static_cast<std::size_t>(nn), sc, ach, warn, report);
  return out;
}

/// pick_slice_mode (parallel.hpp:331-348).
inline Index pick_slice_mode(const Shape& shape, Index workers) {
  std::vector<std::int64_t> dims;
  for (Index k = 0; k < shape.order(); ++k) dims.push_back(shape.dim(k));
  std::int64_t m = -1;
  detail::check(srtt_pick_slice_mode(static_cast<std::int32_t>(dims.size()), dims.data(), workers, &m));
  return m;
}

inline NodeRanks uniform_node_ranks(const DimensionTree& tree, Index rank) {  // dimension_tree.hpp:159-163
  NodeRanks out(static_cast<std::size_t>(tree.num_nodes()), rank);
  out[0] = 1;
  return out;
}

}  // namespace srtt
