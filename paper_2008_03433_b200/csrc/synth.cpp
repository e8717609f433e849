// Deterministic synthetic inputs shared by the bench, the tests and the
// parity harness (host-side data tooling; not on the timed hot path).
//
// * tron_testgen_*: bit-compatible re-statements of the reference's fixture
//   generators (proj/tests/support/testgen.hpp:14-36, testgen.cpp:10-92):
//   splitmix64 with explicit double mappings, so fixtures are identical to
//   the ones the reference's own unit tests use (checked against the
//   reference build in tests/test_synth.py).
// * tron_synth_*: SYNTH-v1, the frozen benchmark generator of SURVEY.md
//   §8(d) (Zipf column popularity, unit-L2 rows; dense with 2-decade column
//   scales).  Pinned by the reference objectives recorded in BASELINE.md §3.
//
// Compiled with -ffp-contract=off: the label pass is a sequential row dot
// exactly like FeatureMatrix::row_dot (linalg.cpp:75-86).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "hostio.h"
#include "tron_b200.h"

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

struct Rng {  // testgen.hpp:14-36
  uint64_t state;
  explicit Rng(uint64_t seed) : state(seed) {}
  // splitmix64 is a counter generator: the stream after k draws is the
  // stream seeded with seed + k*golden, so disjoint ranges of a sequential
  // stream can be produced in parallel, bit for bit.
  static Rng at(uint64_t seed, uint64_t draws) { return Rng(seed + draws * kGolden); }
  uint64_t next_u64() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double in(double lo, double hi) { return lo + (hi - lo) * unit(); }
};

// testgen.cpp:10-22 labels_from_separator (dense row-major or CSR rows)
// Rows are labelled in parallel ranges; row i's flip draw is draw n + i of
// the label stream (rng's state on entry), as in the sequential loop.
template <class RowScore>
void labels_parallel(Rng& rng, size_t l, size_t n, double flip, double* y, RowScore score_of) {
  std::vector<double> w(n);
  for (auto& v : w) v = rng.in(-1.0, 1.0);
  const uint64_t base = rng.state;
  tb::parallel_for(l, 1u << 14, [&](size_t b, size_t e) {
    Rng r(base + (uint64_t)b * kGolden);
    for (size_t i = b; i < e; ++i) {
      double label = score_of(i, w.data()) >= 0.0 ? 1.0 : -1.0;
      if (r.unit() < flip) label = -label;
      y[i] = label;
    }
  });
  rng.state = base + (uint64_t)l * kGolden;
}

void labels_dense(Rng& rng, size_t l, size_t n, const double* X, double flip, double* y) {
  labels_parallel(rng, l, n, flip, y, [&](size_t i, const double* w) {
    const double* row = X + i * n;
    double score = 0.0;
    for (size_t j = 0; j < n; ++j) score += row[j] * w[j];
    return score;
  });
}

void labels_csr(Rng& rng, size_t l, size_t n, const int64_t* ro, const int32_t* ci,
                const double* vals, double flip, double* y) {
  labels_parallel(rng, l, n, flip, y, [&](size_t i, const double* w) {
    double score = 0.0;
    for (int64_t k = ro[i]; k < ro[i + 1]; ++k) score += vals[k] * w[ci[k]];
    return score;
  });
}

}  // namespace

extern "C" {

void tron_testgen_dense_problem(uint64_t seed, size_t l, size_t n, double flip, double* values,
                                double* y) {
  Rng rng(seed);  // testgen.cpp:24-34
  for (size_t k = 0; k < l * n; ++k) values[k] = rng.in(-1.0, 1.0);
  labels_dense(rng, l, n, values, flip, y);
}

void tron_testgen_dense_problem_scaled(uint64_t seed, size_t l, size_t n, double scale,
                                       double flip, double* values, double* y) {
  Rng rng(seed);  // testgen.cpp:36-46
  for (size_t k = 0; k < l * n; ++k) values[k] = scale * rng.in(-1.0, 1.0);
  labels_dense(rng, l, n, values, flip, y);
}

size_t tron_testgen_sparse_problem(uint64_t seed, size_t l, size_t n, double density,
                                   double flip, int64_t* ro, int32_t* ci, double* vals,
                                   double* y) {
  Rng rng(seed);  // testgen.cpp:48-71
  std::vector<int64_t> off{0};
  std::vector<int32_t> cols;
  std::vector<double> v;
  std::vector<int32_t> row_cols;
  for (size_t i = 0; i < l; ++i) {
    row_cols.clear();
    for (size_t j = 0; j < n; ++j)
      if (rng.unit() < density) row_cols.push_back(static_cast<int32_t>(j));
    for (int32_t c : row_cols) {
      cols.push_back(c);
      v.push_back(rng.in(-1.0, 1.0));
    }
    off.push_back(static_cast<int64_t>(v.size()));
  }
  if (ro) {
    std::memcpy(ro, off.data(), (l + 1) * sizeof(int64_t));
    std::memcpy(ci, cols.data(), cols.size() * sizeof(int32_t));
    std::memcpy(vals, v.data(), v.size() * sizeof(double));
    labels_csr(rng, l, n, ro, ci, vals, flip, y);
  }
  return v.size();
}

void tron_testgen_random_vector(uint64_t seed, size_t n, double span, double* out) {
  Rng rng(seed);  // testgen.cpp:73-78
  for (size_t j = 0; j < n; ++j) out[j] = rng.in(-span, span);
}

size_t tron_testgen_random_index_set(uint64_t seed, size_t l, double fraction, int64_t* out) {
  Rng rng(seed);  // testgen.cpp:80-90
  size_t count = 0;
  for (size_t i = 0; i < l; ++i) {
    if (rng.unit() < fraction) {
      if (out) out[count] = static_cast<int64_t>(i);
      ++count;
    }
  }
  if (count == 0 && l > 0 && fraction > 0.0) {
    if (out) out[0] = static_cast<int64_t>(rng.next_u64() % l);
    count = 1;
  }
  return count;
}

// SYNTH-v1 sparse: k distinct Zipf(s) columns per row,
// values 1e-3 + U[0,1), unit-L2 rows.  nnz = l*k exactly.
int tron_synth_sparse(uint64_t seed, size_t l, size_t n, size_t k, double s, double flip,
                      int64_t* ro, int32_t* ci, double* vals, double* y) {
  if (n == 0 || k > n) return TRON_ERR_DIMENSION;
  Rng rng(seed);
  std::vector<double> cdf;
  if (s != 0.0) {
    cdf.resize(n);
    double acc = 0.0;
    for (size_t j = 0; j < n; ++j) {
      acc += std::pow(static_cast<double>(j + 1), -s);
      cdf[j] = acc;
    }
    const double total = cdf[n - 1];
    for (size_t j = 0; j < n; ++j) cdf[j] /= total;
  }
  // guide[b] = lower_bound(cdf, b/B): u in [b/B, (b+1)/B) has its
  // lower_bound in [guide[b], guide[b+1]], so the search below returns
  // exactly std::lower_bound(cdf, u) over a short range.
  size_t B = 1;
  while (B < 4 * n && B < (size_t{1} << 24)) B <<= 1;
  std::vector<uint32_t> guide;
  if (s != 0.0) {
    guide.resize(B + 1);
    size_t j = 0;
    for (size_t b = 0; b <= B; ++b) {
      const double t = static_cast<double>(b) / static_cast<double>(B);
      while (j < n && cdf[j] < t) ++j;
      guide[b] = static_cast<uint32_t>(j);
    }
  }
  std::vector<int32_t> row;
  row.reserve(k);
  ro[0] = 0;
  for (size_t i = 0; i < l; ++i) {
    row.clear();
    while (row.size() < k) {
      size_t c;
      if (s != 0.0) {
        const double u = rng.unit();
        const size_t b = static_cast<size_t>(u * static_cast<double>(B));
        const size_t lo = guide[b], hi = std::min<size_t>(guide[b + 1] + 1, n);
        c = static_cast<size_t>(std::lower_bound(cdf.begin() + lo, cdf.begin() + hi, u) -
                                cdf.begin());
        if (c >= n) c = n - 1;
      } else {
        c = static_cast<size_t>(rng.next_u64() % n);
      }
      if (std::find(row.begin(), row.end(), static_cast<int32_t>(c)) == row.end())
        row.push_back(static_cast<int32_t>(c));
    }
    std::sort(row.begin(), row.end());
    const size_t base = i * k;
    double ss = 0.0;
    for (size_t t = 0; t < k; ++t) {
      double v = 1e-3 + rng.unit();
      ci[base + t] = row[t];
      vals[base + t] = v;
      ss += v * v;
    }
    const double inv = 1.0 / std::sqrt(ss);
    for (size_t t = 0; t < k; ++t) vals[base + t] = vals[base + t] * inv;
    ro[i + 1] = static_cast<int64_t>(base + k);
  }
  labels_csr(rng, l, n, ro, ci, vals, flip, y);
  return TRON_OK;
}

// SYNTH-v1 dense: row-major l x n, column scales spanning
// `decades` decades, optional common factor rho.
int tron_synth_dense(uint64_t seed, size_t l, size_t n, double decades, double rho, double flip,
                     double* values, double* y) {
  if (n < 2) return TRON_ERR_DIMENSION;
  Rng rng(seed);
  std::vector<double> sc(n);
  for (size_t j = 0; j < n; ++j)
    sc[j] = std::pow(10.0, -decades / 2 + decades * static_cast<double>(j) /
                                              static_cast<double>(n - 1));
  // row i consumes draws [i*(n+1), (i+1)*(n+1)): rows are generated in parallel ranges
  tb::parallel_for(l, 1u << 14, [&](size_t b, size_t e) {
    Rng r = Rng::at(seed, (uint64_t)b * (n + 1));
    for (size_t i = b; i < e; ++i) {
      double g = 2 * r.unit() - 1;
      double* row = values + i * n;
      for (size_t j = 0; j < n; ++j) row[j] = sc[j] * (rho * g + (1 - rho) * (2 * r.unit() - 1));
    }
  });
  rng = Rng::at(seed, (uint64_t)l * (n + 1));
  labels_dense(rng, l, n, values, flip, y);
  return TRON_OK;
}

}  // extern "C"
