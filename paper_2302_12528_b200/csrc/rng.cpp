// rng.cpp -- host-side seeded Gaussian blocks, bit-exact with the reference.
//
// The reference draws X0 and the norm sketch Omega from PCG XSL-RR 128/64
// (the published PCG64 generator: 128-bit LCG state, multiplier
// 0x2360ED051FC65DA44385DF649FCCF645, increment
// 0x5851F42D4C957F2D14057B7EF767814F, XOR-shift-low + random-rotate output)
// seeded as state = ((0*a + c) + seed)*a + c, and turns consecutive pairs of
// draws into Gaussians by Box-Muller with a cached second deviate
// (rng.cpp:24-56, dense_matrix.hpp:144-161, element 2k = mag cos, 2k+1 = mag
// sin).  Iteration-count parity needs the very same start block, so it is
// generated here on the host with the same libm (CUDA's log/sin/cos are not
// bit-identical to glibc's), in parallel: each thread jumps the LCG ahead to
// its even draw offset (O(log k) jump, Brown 1994).
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace mpb {

namespace {

using u128 = unsigned __int128;

constexpr u128 mk(uint64_t hi, uint64_t lo) { return (static_cast<u128>(hi) << 64) | lo; }
constexpr u128 kA = mk(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);
constexpr u128 kC = mk(0x5851F42D4C957F2DULL, 0x14057B7EF767814FULL);

inline uint64_t out_xslrr(u128 s) {
  const uint64_t x = static_cast<uint64_t>(s >> 64) ^ static_cast<uint64_t>(s);
  const unsigned rot = static_cast<unsigned>(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

inline u128 seed_state(uint64_t seed) {
  u128 s = 0;
  s = s * kA + kC;
  s += static_cast<u128>(seed);
  s = s * kA + kC;
  return s;
}

// state after `k` more LCG steps
u128 jump(u128 s, uint64_t k) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kA, cur_plus = kC;
  while (k) {
    if (k & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    k >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// stream elements [begin, end) into out[e - base]
void fill_range(uint64_t seed, int64_t begin, int64_t end, double* out, int64_t base = 0) {
  // begin is even: element 2p/2p+1 use draws 2p, 2p+1
  u128 s = jump(seed_state(seed), static_cast<uint64_t>(begin));
  out -= base;
  constexpr double two_pi = 6.283185307179586476925286766559;
  for (int64_t e = begin; e < end; e += 2) {
    s = s * kA + kC;
    const uint64_t d1 = out_xslrr(s);
    s = s * kA + kC;
    const uint64_t d2 = out_xslrr(s);
    const double u1 = (static_cast<double>(d1 >> 11) + 1.0) * 0x1p-53;
    const double u2 = static_cast<double>(d2 >> 11) * 0x1p-53;
    const double mag = std::sqrt(-2.0 * std::log(u1));
    out[e] = mag * std::cos(two_pi * u2);
    if (e + 1 < end) out[e + 1] = mag * std::sin(two_pi * u2);
  }
}

}  // namespace

void gaussian_fill_rows(int64_t n_global, int64_t cols, uint64_t seed, int64_t row0, int64_t rows,
                        double* out) {
  if (rows <= 0 || cols <= 0) return;
  std::vector<double> tmp(static_cast<size_t>(rows + 2));
  for (int64_t j = 0; j < cols; ++j) {
    // column j of the local rows = stream elements [row0 + n j, row0 + rows + n j)
    const int64_t s = row0 + n_global * j, e = s + rows, s2 = s & ~int64_t{1};
    fill_range(seed, s2, e, tmp.data(), s2);
    for (int64_t i = 0; i < rows; ++i) out[i + rows * j] = tmp[static_cast<size_t>(s - s2 + i)];
  }
}

uint64_t pcg64_draw(uint64_t seed, uint64_t index) {
  return out_xslrr(jump(seed_state(seed), index + 1));
}

// out: rows*cols doubles, column-major (flat index order of gaussian_matrix)
void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  const int64_t total = rows * cols;
  if (total <= 0) return;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (total < (int64_t{1} << 20)) nt = 1;
  if (nt > 64) nt = 64;
  int64_t per = (total + nt - 1) / nt;
  per += per & 1;  // even chunk starts keep Box-Muller pairs intact
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t b = static_cast<int64_t>(t) * per;
    if (b >= total) break;
    const int64_t e = b + per < total ? b + per : total;
    th.emplace_back(fill_range, seed, b, e, out, int64_t{0});
  }
  for (auto& x : th) x.join();
}

}  // namespace mpb
