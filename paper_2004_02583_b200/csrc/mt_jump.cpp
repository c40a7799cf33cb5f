// Host side of the MT19937-64 jump-ahead (see mt_jump.hpp).
#include "mt_jump.hpp"

#include <immintrin.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <thread>

namespace tkg {

namespace {

inline uint64_t untemper(uint64_t y) {
  // inverse of the std::mt19937_64 tempering ([rand.eng.mers]:
  // u=29,d=0x5555..., s=17,b=0x71D67FFFEDA60000, t=37,c=0xFFF7EEE000000000, l=43)
  y ^= y >> 43;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  // y ^= (y << 17) & b : invert by iterating (17-bit steps cover 64 bits in 4 rounds)
  {
    uint64_t x = y;
    for (int k = 0; k < 4; ++k) x = y ^ ((x << 17) & 0x71D67FFFEDA60000ull);
    y = x;
  }
  {
    uint64_t x = y;
    for (int k = 0; k < 3; ++k) x = y ^ ((x >> 29) & 0x5555555555555555ull);
    y = x;
  }
  return y;
}

// ---- GF(2)[x] arithmetic on little-endian word arrays ----------------------
inline void clmul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  __m128i va = _mm_set_epi64x(0, static_cast<long long>(a));
  __m128i vb = _mm_set_epi64x(0, static_cast<long long>(b));
  __m128i r = _mm_clmulepi64_si128(va, vb, 0x00);
  lo = static_cast<uint64_t>(_mm_cvtsi128_si64(r));
  hi = static_cast<uint64_t>(_mm_extract_epi64(r, 1));
}

// out[0 .. na+nb) = a * b
void poly_mul(const uint64_t* a, int na, const uint64_t* b, int nb, uint64_t* out) {
  std::memset(out, 0, sizeof(uint64_t) * (na + nb));
  for (int i = 0; i < na; ++i) {
    const uint64_t ai = a[i];
    if (!ai) continue;
    for (int j = 0; j < nb; ++j) {
      uint64_t lo, hi;
      clmul64(ai, b[j], lo, hi);
      out[i + j] ^= lo;
      out[i + j + 1] ^= hi;
    }
  }
}

// out[0..nw) = a >> shift (bits), a has na words
void poly_shr(const uint64_t* a, int na, int shift, uint64_t* out, int nw) {
  const int ws = shift / 64, bs = shift % 64;
  for (int k = 0; k < nw; ++k) {
    const int s = k + ws;
    uint64_t v = s < na ? a[s] >> bs : 0;
    if (bs && s + 1 < na) v |= a[s + 1] << (64 - bs);
    out[k] = v;
  }
}

int poly_deg(const uint64_t* a, int n) {
  for (int k = n - 1; k >= 0; --k)
    if (a[k]) return k * 64 + 63 - __builtin_clzll(a[k]);
  return -1;
}

struct Field {
  std::vector<uint64_t> P;   // kPolyWords+1 words, degree D
  std::vector<uint64_t> mu;  // floor(x^{2D} / P), degree D
};

void mask_low(uint64_t* a, int nw, int bits) {
  for (int k = 0; k < nw; ++k) {
    const int lo = k * 64;
    if (lo >= bits) a[k] = 0;
    else if (lo + 64 > bits) a[k] &= (1ull << (bits - lo)) - 1;
  }
}

const Field& field() {
  static Field f;
  static std::once_flag once;
  std::call_once(once, [] {
    f.P = mt_charpoly();
    // mu = floor(x^{2D} / P) by long division.
    const int D = kMtDeg;
    const int nw = (2 * D) / 64 + 2;
    std::vector<uint64_t> rem(nw, 0);
    rem[(2 * D) / 64] = 1ull << ((2 * D) % 64);
    std::vector<uint64_t> q(nw, 0);
    for (int bit = 2 * D; bit >= D; --bit) {
      if (!((rem[bit / 64] >> (bit % 64)) & 1)) continue;
      const int sh = bit - D;
      q[sh / 64] |= 1ull << (sh % 64);
      // rem ^= P << sh
      const int ws = sh / 64, bs = sh % 64;
      for (int k = 0; k <= kPolyWords; ++k) {
        const uint64_t w = f.P[k];
        if (!w) continue;
        rem[k + ws] ^= w << bs;
        if (bs && k + ws + 1 < nw) rem[k + ws + 1] ^= w >> (64 - bs);
      }
    }
    f.mu.assign(q.begin(), q.begin() + kPolyWords + 1);
  });
  return f;
}

// r = a*b mod P for a, b of degree < D (kPolyWords words each).
void mulmod(const uint64_t* a, const uint64_t* b, uint64_t* r) {
  const Field& f = field();
  const int D = kMtDeg;
  const int W = kPolyWords;
  std::vector<uint64_t> c(2 * W + 2), chi(W + 1), t(2 * W + 4), qq(W + 1), qp(2 * W + 4);
  poly_mul(a, W, b, W, c.data());
  poly_shr(c.data(), 2 * W, D, chi.data(), W + 1);          // c >> D
  poly_mul(chi.data(), W + 1, f.mu.data(), W + 1, t.data());  // (c>>D) * mu
  poly_shr(t.data(), 2 * W + 2, D, qq.data(), W + 1);       // q
  poly_mul(qq.data(), W + 1, f.P.data(), W + 1, qp.data());   // q * P
  for (int k = 0; k < W; ++k) r[k] = c[k] ^ qp[k];
  mask_low(r, W, D);
}

}  // namespace

// The seeded state is formed as std::mersenne_twister_engine::seed(Sseq&)
// does ([rand.eng.mers]: 2 x 32-bit words of seed_seq::generate per state
// word, and the all-zero fix-up), and the raw words are produced by the
// engine's own recurrence in the in-place order -- no tempering, so nothing
// to invert. Checked bitwise against std::mt19937_64 by the tests.
void mt_raw_sequence(uint64_t seed, uint32_t stream, uint64_t* y, int n) {
  std::seed_seq seq{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), stream};
  uint32_t a[2 * kMtN];
  seq.generate(a, a + 2 * kMtN);
  uint64_t x[kMtN];
  for (int i = 0; i < kMtN; ++i) x[i] = uint64_t(a[2 * i]) | (uint64_t(a[2 * i + 1]) << 32);
  {
    bool zero = (x[0] & 0xFFFFFFFF80000000ull) == 0;
    for (int i = 1; i < kMtN && zero; ++i) zero = x[i] == 0;
    if (zero) x[0] = 1ull << 63;
  }
  constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;
  constexpr uint64_t kMatA = 0xB5026F5AA96619E9ull;
  auto tw = [&](uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t v = (cur & kUpper) | (nxt & kLower);
    return far ^ (v >> 1) ^ ((0ull - (v & 1ull)) & kMatA);
  };
  int k = 0;
  while (k < n) {
    for (int i = 0; i < kMtN - 156; ++i) x[i] = tw(x[i], x[i + 1], x[i + 156]);
    for (int i = kMtN - 156; i < kMtN - 1; ++i) x[i] = tw(x[i], x[i + 1], x[i - (kMtN - 156)]);
    x[kMtN - 1] = tw(x[kMtN - 1], x[0], x[155]);
    const int m = std::min(kMtN, n - k);
    std::memcpy(y + k, x, sizeof(uint64_t) * size_t(m));
    k += m;
  }
}

const std::vector<uint64_t>& mt_charpoly() {
  static std::vector<uint64_t> P;
  static std::once_flag once;
  std::call_once(once, [] {
    // Berlekamp-Massey on bit 0 of the raw sequence (any nonzero bit plane
    // has the full characteristic polynomial as its minimal polynomial,
    // because P is primitive).
    const int N = 2 * kMtDeg + 64;
    std::vector<uint64_t> y(N);
    mt_raw_sequence(5489, 0, y.data(), N);
    // R = bit plane reversed: R[j] = s_{N-1-j}; then s_{n-i} = R[N-1-n+i].
    const int RW = N / 64 + 4;
    std::vector<uint64_t> R(RW, 0);
    for (int k = 0; k < N; ++k)
      if (y[k] & 1) {
        const int j = N - 1 - k;
        R[j / 64] |= 1ull << (j % 64);
      }
    auto bits_at = [&](int off) -> uint64_t {  // R[off .. off+64)
      const int w = off / 64, b = off % 64;
      uint64_t v = w < RW ? R[w] >> b : 0;
      if (b && w + 1 < RW) v |= R[w + 1] << (64 - b);
      return v;
    };
    const int W = kPolyWords + 2;
    std::vector<uint64_t> C(W, 0), B(W, 0), T(W);
    C[0] = 1;
    B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < N; ++n) {
      // d = sum_{i=0..L} C_i s_{n-i} (C_0 = 1)
      const int off = N - 1 - n;
      uint64_t acc = 0;
      for (int k = 0; k <= L / 64; ++k) acc ^= C[k] & bits_at(off + 64 * k);
      const int d = __builtin_popcountll(acc) & 1;
      if (!d) {
        ++m;
        continue;
      }
      T = C;
      // C ^= B << m
      const int ws = m / 64, bs = m % 64;
      for (int k = 0; k + ws < W; ++k) {
        C[k + ws] ^= B[k] << bs;
        if (bs && k + ws + 1 < W) C[k + ws + 1] ^= B[k] >> (64 - bs);
      }
      if (2 * L <= n) {
        L = n + 1 - L;
        B = T;
        m = 1;
      } else {
        ++m;
      }
    }
    // Characteristic polynomial = reciprocal of the connection polynomial.
    P.assign(kPolyWords + 1, 0);
    for (int i = 0; i <= L; ++i) {
      if ((C[i / 64] >> (i % 64)) & 1) {
        const int e = L - i;
        P[e / 64] |= 1ull << (e % 64);
      }
    }
    if (L != kMtDeg) P.clear();  // signalled to callers (mt_plan checks)
  });
  return P;
}

namespace {

// base^e mod P by square-and-multiply.
std::vector<uint64_t> powmod(const std::vector<uint64_t>& base_in, uint64_t e) {
  const int W = kPolyWords;
  std::vector<uint64_t> base = base_in, acc(W, 0), tmp(W);
  acc[0] = 1;
  while (e) {
    if (e & 1) {
      mulmod(acc.data(), base.data(), tmp.data());
      acc = tmp;
    }
    e >>= 1;
    if (e) {
      mulmod(base.data(), base.data(), tmp.data());
      base = tmp;
    }
  }
  return acc;
}

}  // namespace

std::vector<uint64_t> mt_jump_table(uint64_t J, int count) {
  const int W = kPolyWords;
  std::vector<uint64_t> out(size_t(count) * W, 0);
  if (count <= 0) return out;
  std::vector<uint64_t> x(W, 0);
  x[0] = 2;  // x
  const std::vector<uint64_t> xj = powmod(x, J);
  // out[c] = (x^J)^c: contiguous segments of c on host threads, each started
  // by its own exponentiation (a few ms per product of two degree-19937
  // polynomials, so a 300-entry table is worth splitting).
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nseg = std::max(1, std::min<int>(int(hw), count / 8));
  const int per = (count + nseg - 1) / nseg;
  auto seg = [&](int s) {
    const int c0 = s * per, c1 = std::min(count, c0 + per);
    if (c0 >= c1) return;
    std::vector<uint64_t> cur = powmod(xj, uint64_t(c0)), tmp(W);
    std::copy(cur.begin(), cur.end(), out.begin() + size_t(c0) * W);
    for (int c = c0 + 1; c < c1; ++c) {
      mulmod(cur.data(), xj.data(), tmp.data());
      cur.swap(tmp);
      std::copy(cur.begin(), cur.end(), out.begin() + size_t(c) * W);
    }
  };
  std::vector<std::thread> th;
  for (int s = 1; s < nseg; ++s) th.emplace_back(seg, s);
  seg(0);
  for (auto& t : th) t.join();
  return out;
}

MtPlan mt_plan(uint64_t total, bool side) {
  MtPlan p;
  p.total = total;
  // A chunk costs one jump (19937 x 312 bit-word XORs, ~1.3 us of the whole
  // GPU) and J draws of one CTA (~1.6 ns each: a 312-draw block is three
  // barriers, mt_gen_cta_kernel): 1.3 us C + 1.6 ns T / C is smallest near
  // C = sqrt(T / 800).
  uint64_t C = static_cast<uint64_t>(std::ceil(std::sqrt(static_cast<double>(total) / 800.0)));
  // beyond two chunks per SM the generation runs at the machine's draw rate
  // whatever C is, and only the jump work keeps growing
  C = std::max<uint64_t>(1, std::min<uint64_t>(C, 296));
  // streams generated on the side stream, behind the sweeps of earlier modes,
  // are not latency-critical: a quarter of the chunks (a quarter of the jump
  // work competing with the sweeps for the SMs) and 4x longer chunks — but no
  // chunk longer than kSideMaxJ draws: a generator CTA that sits on an SM for
  // a millisecond slows that SM's share of every statically scheduled
  // contraction grid and keeps cluster launches waiting (config 5: 76.2 ->
  // 73.7 ms per step with short side chunks; config 4, whose side chunks are
  // short already, is 1 ms slower with 4x the jump work)
  static const uint64_t side_max_j = [] {
    const char* e = std::getenv("TKG_SIDE_MAX_J");
    return e ? uint64_t(std::max(1, std::atoi(e))) : uint64_t(400000);
  }();
  if (side) {
    const uint64_t quarter = std::max<uint64_t>(1, C / 4);
    const uint64_t by_len = (total + side_max_j - 1) / side_max_j;
    C = std::min<uint64_t>(C, std::max(quarter, by_len));
  }
  p.C = static_cast<int>(C);
  p.J = (total + C - 1) / C;
  if (p.J == 0) p.J = 1;
  return p;
}

}  // namespace tkg
