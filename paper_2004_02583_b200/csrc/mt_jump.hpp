// Reference-identical ALS initialiser streams on the GPU.
//
// The reference draws S (fibers x r) in storage order from
// std::mt19937_64 seeded with std::seed_seq{lo32(seed), hi32(seed), mode}
// (als.cpp:67-71, rng.hpp:19-21,57-61). Drawing 10^7..10^9 values serially
// would dominate the GPU decomposition, so the stream is split into C
// chunks of J draws whose generator states are obtained by jump-ahead:
//
//   y_k  = k-th raw (untempered) 64-bit output word.  Every bit position of
//          y is a linear recurring sequence over GF(2) with the engine's
//          characteristic polynomial P (degree 19937), hence
//   y_{a+t} = XOR_{i : p_i = 1} y_{i+t},   p = x^a mod P.
//
// The 312-word window (y_{cJ}, ..., y_{cJ+311}) is a complete generator state
// for chunk c. P is found once by Berlekamp-Massey on a bit plane of y;
// x^{cJ} mod P uses carry-less (PCLMUL) products with Barrett reduction.
// The polynomial tables are seed-independent constants, cached per (J, C).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace tkg {

constexpr int kMtN = 312;          // state words
constexpr int kMtDeg = 19937;      // degree of the characteristic polynomial
constexpr int kPolyWords = 312;    // ceil(19937 / 64)
constexpr int kMtSeqWords = kMtDeg + kMtN - 1;  // y_0 .. y_{D+310}

// First `n` raw (untempered) outputs y_0.. of seeded_engine(seed, stream).
void mt_raw_sequence(uint64_t seed, uint32_t stream, uint64_t* y, int n);

// Characteristic polynomial of MT19937-64 (bit i = coefficient of x^i),
// kPolyWords+1 words (degree 19937 term included). Computed once.
const std::vector<uint64_t>& mt_charpoly();

// polys[c*kPolyWords ...] = x^(c*J) mod P for c = 0..count-1.
std::vector<uint64_t> mt_jump_table(uint64_t J, int count);

// Split of T draws into C chunks of J draws.
struct MtPlan {
  uint64_t total;
  uint64_t J;
  int C;
};
// side: generated off the critical path (fewer, longer chunks)
MtPlan mt_plan(uint64_t total_draws, bool side = false);

}  // namespace tkg
