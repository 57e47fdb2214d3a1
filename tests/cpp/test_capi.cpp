// C++ client of the B200 engine through include/srtt_b200.hpp (the mirror
// of the reference's C++ API): exactly what a reference user's code looks
// like after switching headers. Run by tests/test_gpu_cpp.py on a B200.
#include <cmath>
#include <cstdio>
#include <random>

#include "srtt_b200.hpp"

int main() {
  using namespace srtt;
  // planted rank-3 Tucker tensor 10 x 12 x 14 (first index fastest)
  const Index n0 = 10, n1 = 12, n2 = 14, r = 3;
  std::mt19937_64 gen(7);
  std::normal_distribution<double> nd;
  DenseTensor<double> x(Shape{n0, n1, n2});
  std::vector<double> a(n0 * r), b(n1 * r), c(n2 * r);
  for (auto& v : a) v = nd(gen);
  for (auto& v : b) v = nd(gen);
  for (auto& v : c) v = nd(gen);
  for (Index k = 0; k < n2; ++k)
    for (Index j = 0; j < n1; ++j)
      for (Index i = 0; i < n0; ++i) {
        double s = 0;
        for (Index t = 0; t < r; ++t) s += a[i + n0 * t] * b[j + n1 * t] * c[k + n2 * t];
        x[i + n0 * (j + n1 * k)] = s;
      }
  SubsampleReport rep;
  auto t = sub_r_hosvd(x, Ranks{3, 3, 3}, 4, Ranks{20, 20, 20}, 42, std::nullopt, &rep);
  // reconstruct and measure the error
  double num = 0, den = 0;
  for (Index k = 0; k < n2; ++k)
    for (Index j = 0; j < n1; ++j)
      for (Index i = 0; i < n0; ++i) {
        double s = 0;
        for (Index z = 0; z < r; ++z)
          for (Index y = 0; y < r; ++y)
            for (Index w = 0; w < r; ++w)
              s += t.core[w + r * (y + r * z)] * t.factors[0](i, w) * t.factors[1](j, y) * t.factors[2](k, z);
        const double e = x[i + n0 * (j + n1 * k)] - s;
        num += e * e;
        den += x[i + n0 * (j + n1 * k)] * x[i + n0 * (j + n1 * k)];
      }
  const double err = std::sqrt(num / den);
  std::printf("tucker rel error %.3e ranks %lld %lld %lld\n", err, (long long)rep.achieved_ranks[0],
              (long long)rep.achieved_ranks[1], (long long)rep.achieved_ranks[2]);
  if (!(err < 1e-10)) return 1;
  // the reference's exception types
  try {
    sub_r_hosvd(x, Ranks{3, 3, 3}, 4, Ranks{5, 5, 5}, 1);
    return 2;
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  // H-Tucker on a 4-mode tensor
  DenseTensor<double> y(Shape{5, 6, 4, 3});
  for (Index i = 0; i < y.size(); ++i) y[i] = nd(gen);
  auto tree = DimensionTree::balanced(4);
  NodeRanks ranks = uniform_node_ranks(tree, 2), samples(7, 1);
  for (Index i = 1; i < 7; ++i) samples[i] = 12;
  HtSubsampleReport hrep;
  auto h = sub_r_rtl_ht(y, tree, ranks, samples, 4, 3, std::nullopt, &hrep);
  std::printf("htucker root transfer %lld x %lld x %lld, leaf0 %lld x %lld\n", (long long)h.transfers[0].dim(0),
              (long long)h.transfers[0].dim(1), (long long)h.transfers[0].dim(2), (long long)h.leaf_factors[0].rows(),
              (long long)h.leaf_factors[0].cols());
  return h.transfers[0].dim(1) == 2 ? 0 : 3;
}
