// MT19937-64 jump-ahead polynomials (host side of the chunked stream
// generator in sampling.cu).
//
// std::mt19937_64 advances a 19937-bit state linearly over GF(2): one output
// word = one application of the state map A. With f the characteristic
// polynomial of A, A^J = (x^J mod f)(A), so the state J words ahead is
// sum_i p_i A^i s0 for p = x^J mod f — evaluated on device by Horner's rule.
// f is the reciprocal of the connection polynomial that Berlekamp-Massey
// finds for the output bit sequence (the MT19937 characteristic polynomial is
// primitive, so any nonzero output bit has f as its minimal polynomial; the
// degree check below guards that).
#include <cstdint>
#include <map>
#include <mutex>
#include <random>
#include <stdexcept>
#include <vector>

namespace skg {

namespace {

constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 63) / 64;  // 312

using Poly = std::vector<uint64_t>;  // bit i = coefficient of x^i

inline bool bit(const Poly& p, int64_t i) { return (p[static_cast<size_t>(i >> 6)] >> (i & 63)) & 1u; }
inline void flip(Poly& p, int64_t i) { p[static_cast<size_t>(i >> 6)] ^= 1ull << (i & 63); }

// dst ^= src << sh (dst sized to hold the result)
void xor_shifted(Poly& dst, const Poly& src, int64_t sh) {
  const int64_t ws = sh >> 6, bs = sh & 63;
  for (size_t w = 0; w < src.size(); ++w) {
    const uint64_t v = src[w];
    if (!v) continue;
    const size_t o = w + static_cast<size_t>(ws);
    if (o < dst.size()) dst[o] ^= v << bs;
    if (bs && o + 1 < dst.size()) dst[o + 1] ^= v >> (64 - bs);
  }
}

// Characteristic polynomial of MT19937-64 (degree 19937) via Berlekamp-Massey
// on bit 0 of the output stream.
Poly characteristic() {
  const int64_t N = 2 * kDeg + 128;
  const int64_t NW = (N + 63) / 64 + 2;
  // R = the bit sequence reversed: R_k = s_{N-1-k}
  Poly R(static_cast<size_t>(NW), 0);
  std::mt19937_64 g(5489u);
  for (int64_t n = 0; n < N; ++n)
    if (g() & 1u) flip(R, N - 1 - n);
  auto window = [&](int64_t pos, int64_t w) -> uint64_t {  // 64 bits of R from pos + 64 w
    const int64_t b = pos + 64 * w;
    const int64_t q = b >> 6, r = b & 63;
    const uint64_t lo = q < NW ? R[static_cast<size_t>(q)] : 0, hi = q + 1 < NW ? R[static_cast<size_t>(q + 1)] : 0;
    return r ? (lo >> r) | (hi << (64 - r)) : lo;
  };
  const size_t CW = static_cast<size_t>(kWords + 2);
  Poly C(CW, 0), B(CW, 0);
  C[0] = B[0] = 1;
  int64_t L = 0, m = 1;
  for (int64_t n = 0; n < N; ++n) {
    // d = sum_{i=0..L} c_i s_{n-i} = parity(C . R[N-1-n ..])
    uint64_t acc = 0;
    const int64_t lw = L / 64 + 1;
    for (int64_t w = 0; w < lw && w < static_cast<int64_t>(CW); ++w) acc ^= C[static_cast<size_t>(w)] & window(N - 1 - n, w);
    if (!(__builtin_popcountll(acc) & 1)) {
      ++m;
      continue;
    }
    if (2 * L <= n) {
      const Poly T = C;
      xor_shifted(C, B, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shifted(C, B, m);
      ++m;
    }
  }
  if (L != kDeg) throw std::runtime_error("mt_jump: unexpected linear complexity");
  Poly f(static_cast<size_t>(kWords + 1), 0);  // f_i = c_{L-i}
  for (int64_t i = 0; i <= L; ++i)
    if (bit(C, L - i)) flip(f, i);
  return f;
}

const Poly& charpoly() {
  static const Poly f = characteristic();
  return f;
}

// a mod f for deg(a) < 2 * kDeg
void reduce(Poly& a, const Poly& f) {
  for (int64_t k = static_cast<int64_t>(a.size()) * 64 - 1; k >= kDeg; --k)
    if (bit(a, k)) xor_shifted(a, f, k - kDeg);
  a.resize(static_cast<size_t>(kWords));
}

Poly mulmod(const Poly& a, const Poly& b, const Poly& f) {
  Poly r(static_cast<size_t>(2 * kWords + 2), 0);
  Poly bb = b;
  bb.resize(static_cast<size_t>(kWords + 1), 0);
  for (int64_t i = 0; i < kDeg; ++i)
    if (bit(a, i)) xor_shifted(r, bb, i);
  reduce(r, f);
  return r;
}

Poly sqrmod(const Poly& a, const Poly& f) {
  Poly r(static_cast<size_t>(2 * kWords + 2), 0);
  for (int64_t i = 0; i < kDeg; ++i)
    if (bit(a, i)) flip(r, 2 * i);
  reduce(r, f);
  return r;
}

Poly xpow(uint64_t J, const Poly& f) {  // x^J mod f
  Poly p(static_cast<size_t>(kWords), 0);
  p[0] = 1;
  for (int b = 63; b >= 0; --b) {
    p = sqrmod(p, f);
    if ((J >> b) & 1u) {  // p *= x
      Poly q(static_cast<size_t>(kWords + 1), 0);
      xor_shifted(q, p, 1);
      if (bit(q, kDeg)) xor_shifted(q, f, 0);
      q.resize(static_cast<size_t>(kWords));
      p = q;
    }
  }
  return p;
}

}  // namespace

// Coefficient words (kWords each, bit i of word i/64 = coefficient of x^i) of
// x^(j L) mod f for j = 1 .. P-1, cached per (L, P).
const std::vector<uint64_t>& mt_jump_polys(int64_t L, int P) {
  static std::mutex mu;
  static std::map<std::pair<int64_t, int>, std::vector<uint64_t>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({L, P});
  if (it != cache.end()) return it->second;
  const Poly& f = charpoly();
  std::vector<uint64_t> out;
  out.reserve(static_cast<size_t>(P - 1) * kWords);
  const Poly q = xpow(static_cast<uint64_t>(L), f);
  Poly p = q;
  for (int j = 1; j < P; ++j) {
    if (j > 1) p = mulmod(p, q, f);
    out.insert(out.end(), p.begin(), p.begin() + kWords);
  }
  return cache.emplace(std::make_pair(L, P), std::move(out)).first->second;
}

// Host check of one jump: the state J words ahead of std::mt19937_64(seed),
// computed with the polynomial, must continue the stream exactly.
bool mt_jump_selftest(uint64_t seed, int64_t J) {
  const Poly& f = charpoly();
  const Poly p = xpow(static_cast<uint64_t>(J), f);
  // the seeded state and its word sequence x[k + 312] = x[k + 156] ^ mix(x[k], x[k + 1])
  const uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kMatA = 0xB5026F5AA96619E9ULL;
  auto mix = [&](uint64_t a, uint64_t b) {
    const uint64_t y = (a & kUpper) | (b & kLower);
    return (y >> 1) ^ ((y & 1u) ? kMatA : 0);
  };
  std::vector<uint64_t> s0(312);
  s0[0] = seed;
  for (int i = 1; i < 312; ++i) s0[i] = 6364136223846793005ULL * (s0[i - 1] ^ (s0[i - 1] >> 62)) + i;
  // Horner: acc = A(acc) ^ p_i s0, i = deg .. 0 (acc as a 312-word window)
  std::vector<uint64_t> acc(312, 0);
  for (int64_t i = kDeg - 1; i >= 0; --i) {
    const uint64_t nw = acc[156] ^ mix(acc[0], acc[1]);
    acc.erase(acc.begin());
    acc.push_back(nw);
    if (bit(p, i))
      for (int k = 0; k < 312; ++k) acc[k] ^= s0[k];
  }
  // continue from the jumped window and compare with the reference stream
  std::mt19937_64 g(seed);
  g.discard(static_cast<unsigned long long>(J));
  auto temper = [](uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
  };
  for (int k = 0; k < 1000; ++k) {
    const uint64_t nw = acc[156] ^ mix(acc[0], acc[1]);
    acc.erase(acc.begin());
    acc.push_back(nw);
    if (temper(nw) != g()) return false;
  }
  return true;
}

}  // namespace skg
