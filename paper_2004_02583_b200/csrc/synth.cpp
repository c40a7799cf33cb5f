// Seeded synthetic Tucker tensors for the BASELINE configs.
// Input synthesis only — not part of the decomposition path. Host C++ with
// OpenMP so both bench arms (GPU and the CPU reference) consume identical
// bytes for the same (shape, ranks, alpha, nu, seed):
//
//   G[k_1..k_N] = Z[k] * prod_n k_n^(-alpha)      Z ~ N(0,1), k 1-based
//   Q_n = orthonormal basis of a Gaussian I_n x R_n (CGS2, R_ii > 0)
//   A0  = G x_1 Q_1 x_2 ... x_N Q_N
//   A   = A0 + (nu ||A0||_F / ||E||_F) E          E ~ N(0,1) elementwise
//
// Normals come from a counter-based hash (splitmix64 finalizer) + Box-Muller,
// so every element is generated independently and the tensor is identical
// for any thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Standard normal number `index` of stream (seed, stream).
inline double normal_at(uint64_t key, uint64_t index) {
  const uint64_t pair = index >> 1;
  const uint64_t h1 = mix64(key ^ (2 * pair));
  const uint64_t h2 = mix64(key ^ (2 * pair + 1) ^ 0xD1B54A32D192ED03ull);
  const double u1 = (double((h1 >> 11) + 1)) * 0x1.0p-53;  // (0, 1]
  const double u2 = double(h2 >> 11) * 0x1.0p-53;
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double ang = 6.283185307179586476925286766559 * u2;
  return (index & 1) ? rad * std::sin(ang) : rad * std::cos(ang);
}

inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * 0x632BE59BD9B4E019ull ^ mix64(stream + 0x1234567ull));
}

// Orthonormal columns from a Gaussian matrix by classical Gram-Schmidt with
// reorthogonalisation.
void orthonormal(uint64_t key, uint64_t I, uint64_t R, double* q) {
  for (uint64_t k = 0; k < I * R; ++k) q[k] = normal_at(key, k);
  for (uint64_t c = 0; c < R; ++c) {
    double* v = q + c * I;
    for (int pass = 0; pass < 2; ++pass) {
      for (uint64_t p = 0; p < c; ++p) {
        const double* u = q + p * I;
        double d = 0.0;
        for (uint64_t i = 0; i < I; ++i) d += u[i] * v[i];
        for (uint64_t i = 0; i < I; ++i) v[i] -= d * u[i];
      }
    }
    double nn = 0.0;
    for (uint64_t i = 0; i < I; ++i) nn += v[i] * v[i];
    const double inv = 1.0 / std::sqrt(nn);
    for (uint64_t i = 0; i < I; ++i) v[i] *= inv;
  }
}

// out(jl, i, p) = sum_c in(jl, c, p) * Q[i + c*I]; in has extent R at the mode.
void expand(const double* in, uint64_t s, uint64_t R, uint64_t P, const double* Q, uint64_t I,
            double* out) {
  const uint64_t jb = 256;
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t p = 0; p < int64_t(P); ++p) {
    for (int64_t j0 = 0; j0 < int64_t(s); j0 += jb) {
      const uint64_t j1 = std::min<uint64_t>(s, j0 + jb);
      const double* inp = in + uint64_t(p) * s * R;
      double* outp = out + uint64_t(p) * s * I;
      for (uint64_t i = 0; i < I; ++i) {
        double* o = outp + i * s;
        for (uint64_t j = j0; j < j1; ++j) o[j] = 0.0;
        for (uint64_t c = 0; c < R; ++c) {
          const double w = Q[i + c * I];
          const double* src = inp + c * s;
          for (uint64_t j = j0; j < j1; ++j) o[j] += src[j] * w;
        }
      }
    }
  }
}

}  // namespace

extern "C" {

// Phase 1 of the generator for the slab [k0, k0 + nloc) of the last mode:
// out (column-major, dims with the last extent nloc) = A0 = G x_1 Q_1 ...
// x_N Q_N restricted to the slab, and slice_sq[2*t] / slice_sq[2*t+1] the
// sums of A0^2 and of the noise e^2 over last-mode slice k0 + t (summed in
// a fixed order inside the slice, so any split of the tensor gives the same
// per-slice numbers). Returns 0 on success.
int tkg_synth_tucker_slab(int order, const uint64_t* dims, const uint64_t* ranks, double alpha, uint64_t seed,
                          uint64_t k0, uint64_t nloc, double* out, double* slice_sq) {
  if (order < 1 || order > 64) return 1;
  uint64_t core = 1;
  for (int n = 0; n < order; ++n) {
    if (ranks[n] < 1 || ranks[n] > dims[n]) return 1;
    core *= ranks[n];
  }
  if (k0 + nloc > dims[order - 1] || nloc == 0) return 1;
  // core
  std::vector<double> cur(core);
  {
    const uint64_t key = stream_key(seed, 0);
    for (uint64_t k = 0; k < core; ++k) {
      uint64_t rem = k;
      double scale = 1.0;
      for (int n = 0; n < order; ++n) {
        const uint64_t kn = rem % ranks[n] + 1;
        rem /= ranks[n];
        scale *= std::pow(double(kn), -alpha);
      }
      cur[k] = normal_at(key, k) * scale;
    }
  }
  // A0 slab = G x_1 Q_1 ... x_N Q_N[k0 : k0 + nloc, :] (the last expansion writes into `out`)
  std::vector<uint64_t> shp(ranks, ranks + order);
  std::vector<double> nxt;
  for (int n = 0; n < order; ++n) {
    const bool last = n == order - 1;
    std::vector<double> Q(dims[n] * ranks[n]);
    orthonormal(stream_key(seed, 1 + n), dims[n], ranks[n], Q.data());
    uint64_t I = dims[n];
    if (last) {  // rows k0 .. k0 + nloc of Q_N
      std::vector<double> Qs(nloc * ranks[n]);
      for (uint64_t c = 0; c < ranks[n]; ++c)
        for (uint64_t i = 0; i < nloc; ++i) Qs[i + c * nloc] = Q[k0 + i + c * dims[n]];
      Q.swap(Qs);
      I = nloc;
    }
    uint64_t s = 1, P = 1;
    for (int m = 0; m < n; ++m) s *= shp[m];
    for (int m = n + 1; m < order; ++m) P *= shp[m];
    double* dst;
    if (last) {
      dst = out;
    } else {
      nxt.assign(s * I * P, 0.0);
      dst = nxt.data();
    }
    expand(cur.data(), s, ranks[n], P, Q.data(), I, dst);
    shp[n] = I;
    if (!last) cur.swap(nxt);
  }
  // per-slice sums of A0^2 and of the noise e^2 (noise index = global element index)
  const uint64_t slice = [&] {
    uint64_t v = 1;
    for (int n = 0; n + 1 < order; ++n) v *= dims[n];
    return v;
  }();
  const uint64_t key = stream_key(seed, 1000);
#pragma omp parallel for schedule(dynamic)
  for (int64_t t = 0; t < int64_t(nloc); ++t) {
    double sa = 0.0, se = 0.0;
    const double* o = out + uint64_t(t) * slice;
    const uint64_t g0 = (k0 + uint64_t(t)) * slice;
    for (uint64_t k = 0; k < slice; ++k) {
      const double e = normal_at(key, g0 + k);
      sa += o[k] * o[k];
      se += e * e;
    }
    slice_sq[2 * t] = sa;
    slice_sq[2 * t + 1] = se;
  }
  return 0;
}

// Phase 2: out += scale * e over the slab, scale = nu * ||A0||_F / ||e||_F
// from the sums of all slices of the tensor (tkg_synth_noise_scale).
int tkg_synth_add_noise(int order, const uint64_t* dims, uint64_t seed, uint64_t k0, uint64_t nloc, double scale,
                        double* out) {
  if (order < 1 || order > 64) return 1;
  uint64_t slice = 1;
  for (int n = 0; n + 1 < order; ++n) slice *= dims[n];
  const uint64_t key = stream_key(seed, 1000);
  const uint64_t g0 = k0 * slice, total = nloc * slice;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < int64_t(total); ++k) out[k] += scale * normal_at(key, g0 + uint64_t(k));
  return 0;
}

// nu * sqrt(sum A0^2) / sqrt(sum e^2) over all I_N slices, summed in slice order.
double tkg_synth_noise_scale(uint64_t nslices, const double* slice_sq, double nu) {
  double a0 = 0.0, ee = 0.0;
  for (uint64_t t = 0; t < nslices; ++t) {
    a0 += slice_sq[2 * t];
    ee += slice_sq[2 * t + 1];
  }
  return ee > 0.0 ? nu * std::sqrt(a0) / std::sqrt(ee) : 0.0;
}

// The whole tensor (prod(dims) doubles, column-major). Returns 0 on success.
int tkg_synth_tucker(int order, const uint64_t* dims, const uint64_t* ranks, double alpha, double nu,
                     uint64_t seed, double* out) {
  if (order < 1 || order > 64) return 1;
  const uint64_t IN = dims[order - 1];
  std::vector<double> sq(2 * IN);
  int rc = tkg_synth_tucker_slab(order, dims, ranks, alpha, seed, 0, IN, out, sq.data());
  if (rc) return rc;
  return tkg_synth_add_noise(order, dims, seed, 0, IN, tkg_synth_noise_scale(IN, sq.data(), nu), out);
}

}  // extern "C"
