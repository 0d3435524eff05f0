// Host half of the sparse Cholesky preconditioner: the
// reverse Cuthill-McKee ordering and the up-looking numeric factorisation,
// built once per solve on the host like the reference (rcm.cpp:8-57,
// sparse_kernels.hpp:92-170); the per-iteration triangular solves run on the
// device (spchol.cu).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
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

int g_spchol_threads = 0;  // host factorisation threads (0: the hardware's, capped at 32)

// Up-looking Cholesky of B = L L^T (sparse_cholesky, sparse_kernels.hpp:92-170),
// arithmetic in F: row i of L solves L(0:i, 0:i) l = b_i over the etree
// reach of row i, columns ascending; diagonal stored last in each row.
//
// Rows run concurrently, round-robin over host threads: row i's solve reads
// the finished rows j of its reach (each published with a release flag), so
// a thread waits only where its reach meets a row still in flight -- for the
// banded RCM orderings that is the tail of the reach.  Every entry is formed
// by the same operations in the same order as the sequential algorithm, so
// the factor is bitwise the reference's; the first failing row (lowest index)
// raises the sequential error.
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
  int nt = g_spchol_threads > 0 ? g_spchol_threads
                                 : static_cast<int>(std::min(32u, std::max(1u, std::thread::hardware_concurrency())));
  if (n < 4096) nt = 1;
  // per row: the reach columns then the diagonal, values alike
  std::vector<std::vector<int64_t>> rci(static_cast<size_t>(n));
  std::vector<std::vector<F>> rv(static_cast<size_t>(n));
  std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[static_cast<size_t>(n)]);
  for (int64_t i = 0; i < n; ++i) done[i].store(0, std::memory_order_relaxed);
  std::atomic<int64_t> first_bad{n};
  std::vector<int> bad_kind(static_cast<size_t>(n), 0);  // 1 overflow, 2 not PD, 3 after a failed row
  auto worker = [&](int t) {
    std::vector<F> x(static_cast<size_t>(n), F(0));
    std::vector<char> mark(static_cast<size_t>(n), 0);
    std::vector<int64_t> reach;
    for (int64_t i = t; i < n; i += nt) {
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
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
        if (ci[p] <= i) x[ci[p]] = v[p];
      F sq = F(0);
      bool upstream_bad = false;
      for (int64_t j : reach) {
        int st;
        while ((st = done[j].load(std::memory_order_acquire)) == 0) std::this_thread::yield();
        if (st != 1) {
          upstream_bad = true;
          break;
        }
        const std::vector<int64_t>& cj = rci[j];
        const std::vector<F>& vj = rv[j];
        F s = x[j];
        const size_t nd = cj.size() - 1;  // the diagonal is last
        for (size_t p = 0; p < nd; ++p) s -= x[cj[p]] * vj[p];
        const F lij = s / vj[nd];
        x[j] = lij;
        sq += lij * lij;
      }
      int kind = upstream_bad ? 3 : 0;
      F d = F(0);
      if (!upstream_bad) {
        d = x[i] - sq;
        if (!std::isfinite(static_cast<double>(d)))
          kind = 1;
        else if (!(d > F(0)))
          kind = 2;
      }
      if (kind == 0) {
        std::vector<int64_t>& c = rci[i];
        std::vector<F>& w = rv[i];
        c.reserve(reach.size() + 1);
        w.reserve(reach.size() + 1);
        for (int64_t j : reach) {
          c.push_back(j);
          w.push_back(x[j]);
        }
        c.push_back(i);
        w.push_back(std::sqrt(d));
      } else {
        bad_kind[i] = kind;
        int64_t cur = first_bad.load();
        while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {
        }
      }
      for (int64_t j : reach) x[j] = F(0);
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
        if (ci[p] <= i) x[ci[p]] = F(0);
      done[i].store(kind == 0 ? 1 : 2, std::memory_order_release);
    }
  };
  if (nt == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
  }
  const int64_t bad = first_bad.load();
  if (bad < n) {  // the lowest failing row is the sequential algorithm's first
    if (bad_kind[bad] == 1)
      throw Error(MPEIG_E_OVERFLOW, "sparse_cholesky: row " + std::to_string(bad) + " overflowed", bad);
    throw Error(MPEIG_E_NOT_PD, "sparse_cholesky: nonpositive pivot at row " + std::to_string(bad), bad);
  }
  HostFactor<F> L;
  L.rp.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t i = 0; i < n; ++i) L.rp[i + 1] = L.rp[i] + static_cast<int64_t>(rci[i].size());
  L.ci.reserve(static_cast<size_t>(L.rp[n]));
  L.v.reserve(static_cast<size_t>(L.rp[n]));
  for (int64_t i = 0; i < n; ++i) {
    L.ci.insert(L.ci.end(), rci[i].begin(), rci[i].end());
    L.v.insert(L.v.end(), rv[i].begin(), rv[i].end());
    std::vector<int64_t>().swap(rci[i]);
    std::vector<F>().swap(rv[i]);
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
