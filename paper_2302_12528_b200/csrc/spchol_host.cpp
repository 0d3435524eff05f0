// Host half of the sparse Cholesky preconditioner: the
// reverse Cuthill-McKee ordering and the up-looking numeric factorisation,
// built once per solve on the host like the reference (rcm.cpp:8-57,
// sparse_kernels.hpp:92-170); the per-iteration triangular solves run on the
// device (spchol.cu).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "context.hpp"
#include "spchol.hpp"

namespace mpb {

// rcm_ordering_pattern (rcm.cpp:8-57): BFS from the minimum-(degree, index)
// unvisited vertex of each component, each vertex's new neighbours queued by
// ascending (degree, index), the component's visit order reversed in place.
std::vector<int64_t> rcm_ordering(int64_t n, const int64_t* rp, const int64_t* ci) {
  std::vector<int64_t> deg(static_cast<size_t>(n), 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) deg[i] += ci[p] != i;
  auto less = [&](int64_t a, int64_t b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; };
  std::vector<int64_t> starts(static_cast<size_t>(n));
  std::iota(starts.begin(), starts.end(), int64_t{0});
  std::sort(starts.begin(), starts.end(), less);
  std::vector<char> seen(static_cast<size_t>(n), 0);
  std::vector<int64_t> order, nb;
  order.reserve(static_cast<size_t>(n));
  for (int64_t s0 : starts) {
    if (seen[s0]) continue;
    const size_t begin = order.size();
    order.push_back(s0);
    seen[s0] = 1;
    // order doubles as the BFS queue of this component
    for (size_t head = begin; head < order.size(); ++head) {
      const int64_t u = order[head];
      nb.clear();
      for (int64_t p = rp[u]; p < rp[u + 1]; ++p) {
        const int64_t v = ci[p];
        if (v != u && !seen[v]) {
          seen[v] = 1;
          nb.push_back(v);
        }
      }
      std::sort(nb.begin(), nb.end(), less);
      order.insert(order.end(), nb.begin(), nb.end());
    }
    std::reverse(order.begin() + static_cast<int64_t>(begin), order.end());
  }
  return order;
}

// B = A(perm, perm): B(k, l) = A(perm[k], perm[l]), columns ascending per row
// (CsrMatrix::permuted; perm empty = identity)
template <typename V>
void csr_permute(int64_t n, const int64_t* rp, const int64_t* ci, const V* v,
                 const std::vector<int64_t>& perm, std::vector<int64_t>& brp,
                 std::vector<int64_t>& bci, std::vector<V>& bv) {
  std::vector<int64_t> inv(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) inv[perm.empty() ? k : perm[k]] = k;
  brp.assign(static_cast<size_t>(n + 1), 0);
  bci.clear();
  bv.clear();
  std::vector<std::pair<int64_t, V>> row;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = perm.empty() ? k : perm[k];
    row.clear();
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) row.emplace_back(inv[ci[p]], v[p]);
    std::sort(row.begin(), row.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& e : row) {
      bci.push_back(e.first);
      bv.push_back(e.second);
    }
    brp[k + 1] = static_cast<int64_t>(bci.size());
  }
}
template void csr_permute<double>(int64_t, const int64_t*, const int64_t*, const double*,
                                  const std::vector<int64_t>&, std::vector<int64_t>&,
                                  std::vector<int64_t>&, std::vector<double>&);

// Up-looking Cholesky of B = L L^T (sparse_cholesky, sparse_kernels.hpp:92-170),
// arithmetic in F: row i of L solves L(0:i, 0:i) l = b_i over the etree
// reach of row i, columns ascending; diagonal stored last in each row.
template <typename F>
HostFactor<F> sparse_cholesky_host(int64_t n, const std::vector<int64_t>& rp,
                                   const std::vector<int64_t>& ci, const std::vector<F>& v) {
  // elimination tree (sparse_kernels.hpp:37-53), ancestors path-compressed
  std::vector<int64_t> parent(static_cast<size_t>(n), -1), anc(static_cast<size_t>(n), -1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      for (int64_t j = ci[p]; j != -1 && j < i;) {
        const int64_t up = anc[j];
        anc[j] = i;
        if (up == -1) parent[j] = i;
        j = up;
      }
  HostFactor<F> L;
  L.rp.assign(1, 0);
  std::vector<F> x(static_cast<size_t>(n), F(0));
  std::vector<char> mark(static_cast<size_t>(n), 0);
  std::vector<int64_t> reach, row_of(static_cast<size_t>(n)), diag_at(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    // reach of row i in the etree, ascending (ereach, :60-83)
    reach.clear();
    mark[i] = 1;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      for (int64_t j = ci[p]; j != -1 && j < i && !mark[j]; j = parent[j]) {
        mark[j] = 1;
        reach.push_back(j);
      }
    std::sort(reach.begin(), reach.end());
    for (int64_t j : reach) mark[j] = 0;
    mark[i] = 0;
    bool has_diag = false;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] <= i) {
        x[ci[p]] = v[p];
        has_diag |= ci[p] == i;
      }
    (void)has_diag;
    F sq = F(0);
    for (int64_t j : reach) {
      F s = x[j];
      for (int64_t p = row_of[j]; p < diag_at[j]; ++p) s -= x[L.ci[p]] * L.v[p];
      const F lij = s / L.v[diag_at[j]];
      x[j] = lij;
      sq += lij * lij;
    }
    const F d = x[i] - sq;
    if (!std::isfinite(static_cast<double>(d)))
      throw Error(MPEIG_E_OVERFLOW, "sparse_cholesky: row " + std::to_string(i) + " overflowed", i);
    if (!(d > F(0)))
      throw Error(MPEIG_E_NOT_PD, "sparse_cholesky: nonpositive pivot at row " + std::to_string(i), i);
    row_of[i] = static_cast<int64_t>(L.ci.size());
    for (int64_t j : reach) {
      L.ci.push_back(j);
      L.v.push_back(x[j]);
      x[j] = F(0);
    }
    diag_at[i] = static_cast<int64_t>(L.ci.size());
    L.ci.push_back(i);
    L.v.push_back(std::sqrt(d));
    x[i] = F(0);
    L.rp.push_back(static_cast<int64_t>(L.ci.size()));
  }
  return L;
}
template HostFactor<double> sparse_cholesky_host<double>(int64_t, const std::vector<int64_t>&,
                                                         const std::vector<int64_t>&,
                                                         const std::vector<double>&);
template HostFactor<float> sparse_cholesky_host<float>(int64_t, const std::vector<int64_t>&,
                                                       const std::vector<int64_t>&,
                                                       const std::vector<float>&);

}  // namespace mpb
