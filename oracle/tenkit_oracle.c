/* TEST INFRASTRUCTURE — NOT PRODUCT CODE (see tenkit_oracle.h).
 *
 * Plain-C restatement of the reference's ALS-HOSVD path. Each function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/src unless noted) and keeps the reference's loop
 * and summation order, so results agree BITWISE with the reference for any
 * thread count (the reference is itself thread-count invariant:
 * parallel.hpp:7-13). Parallel loops use OpenMP over the same chunks. */
#include "tenkit_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define FIBER_CHUNK 1024  /* parallel.hpp:10 kFiberChunk */
#define SCALAR_CHUNK 4096 /* parallel.hpp:13 kScalarChunk */

static int fail(orc_error* err, int subtype, int category, const char* fmt, ...)
    __attribute__((format(printf, 4, 5)));

#include <stdarg.h>
static int fail(orc_error* err, int subtype, int category, const char* fmt, ...) {
  if (err) {
    err->subtype = subtype;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
    va_end(ap);
  }
  return category + 1; /* ErrorCategory + 1 (errors.hpp:10) */
}
#define USAGE 0
#define NUMERICAL 2

static void ok(orc_error* err) {
  if (err) {
    err->subtype = ORC_OK;
    err->msg[0] = '\0';
  }
}

/* ======================= rng.hpp ======================================= */
/* std::seed_seq::generate ([rand.util.seedseq]) for the 3-word seed
 * {lo32(seed), hi32(seed), stream} of seeded_engine (rng.hpp:57-61). */
static void seed_seq_generate(const uint32_t* v, size_t s, uint32_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = 0x8b8b8b8bu;
  const size_t t = (n >= 623) ? 11 : (n >= 68) ? 7 : (n >= 39) ? 5 : (n >= 7) ? 3 : (n - 1) / 2;
  const size_t p = (n - t) / 2;
  const size_t q = p + t;
  const size_t m = (s + 1 > n) ? s + 1 : n;
  for (size_t k = 0; k < m; ++k) {
    uint32_t x = out[k % n] ^ out[(k + p) % n] ^ out[(k + n - 1) % n];
    uint32_t r1 = 1664525u * (x ^ (x >> 27));
    uint32_t r2 = r1 + (uint32_t)(k == 0 ? s : (k <= s ? k % n + v[k - 1] : k % n));
    out[(k + p) % n] += r1;
    out[(k + q) % n] += r2;
    out[k % n] = r2;
  }
  for (size_t k = m; k < m + n; ++k) {
    uint32_t x = out[k % n] + out[(k + p) % n] + out[(k + n - 1) % n];
    uint32_t r3 = 1566083941u * (x ^ (x >> 27));
    uint32_t r4 = r3 - (uint32_t)(k % n);
    out[(k + p) % n] ^= r3;
    out[(k + q) % n] ^= r4;
    out[k % n] = r4;
  }
}

#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull
#define MT_A 0xB5026F5AA96619E9ull

void orc_mt64_seeded(orc_mt64* eng, uint64_t seed, uint32_t stream) {
  uint32_t v[3] = {(uint32_t)seed, (uint32_t)(seed >> 32), stream};
  uint32_t words[2 * MT_N];
  seed_seq_generate(v, 3, words, 2 * MT_N);
  int all_zero = 1;
  for (int i = 0; i < MT_N; ++i) {
    eng->mt[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
    if (i > 0 && eng->mt[i] != 0) all_zero = 0;
  }
  if (all_zero && (eng->mt[0] & MT_UPPER) == 0) eng->mt[0] = 1ull << 63;
  eng->idx = MT_N;
}

static void mt_twist(uint64_t* mt) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t y = (mt[i] & MT_UPPER) | (mt[(i + 1) % MT_N] & MT_LOWER);
    mt[i] = mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ull) ? MT_A : 0ull);
  }
}

uint64_t orc_mt64_next(orc_mt64* eng) {
  if (eng->idx >= MT_N) {
    mt_twist(eng->mt);
    eng->idx = 0;
  }
  uint64_t z = eng->mt[eng->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= (z >> 43);
  return z;
}

double orc_uniform01(orc_mt64* eng) { return (double)(orc_mt64_next(eng) >> 11) * 0x1.0p-53; }

double orc_uniform_in(orc_mt64* eng, double lo, double hi) {
  return lo + (hi - lo) * orc_uniform01(eng);
}

void orc_gaussian_fill(uint64_t seed, uint32_t stream, double* out, size_t n) {
  orc_mt64 eng;
  orc_mt64_seeded(&eng, seed, stream);
  const double pi = 3.141592653589793238462643383279502884;
  for (size_t i = 0; i < n; i += 2) {
    double u1 = 1.0 - orc_uniform01(&eng);
    double u2 = orc_uniform01(&eng);
    double radius = sqrt(-2.0 * log(u1));
    double angle = 2.0 * pi * u2;
    out[i] = radius * cos(angle);
    if (i + 1 < n) out[i + 1] = radius * sin(angle);
  }
}

/* ======================= shape / FiberSpace ============================ */
typedef struct {
  size_t extent, stride, fibers, count;
} fiber_space; /* tensor_ops.cpp:23-39 */

static int make_space(int order, const uint64_t* dims, int mode, fiber_space* fs,
                      orc_error* err) {
  if (order < 1) return fail(err, ORC_E_DIMENSION_MISMATCH, USAGE, "Shape: at least one extent required");
  size_t count = 1;
  for (int k = 0; k < order; ++k) {
    if (dims[k] == 0) return fail(err, ORC_E_DIMENSION_MISMATCH, USAGE, "Shape: extents must be >= 1");
    count *= (size_t)dims[k];
  }
  if (mode < 1 || mode > order) /* shape.cpp:27-33 */
    return fail(err, ORC_E_INVALID_MODE, USAGE, "mode %d out of range 1..%d", mode, order);
  size_t stride = 1;
  for (int m = 0; m + 1 < mode; ++m) stride *= (size_t)dims[m];
  fs->extent = (size_t)dims[mode - 1];
  fs->stride = stride;
  fs->count = count;
  fs->fibers = count / fs->extent;
  return 0;
}

static inline size_t fs_base(const fiber_space* fs, size_t j) {
  return (j / fs->stride) * fs->stride * fs->extent + (j % fs->stride);
}

static size_t chunk_count(size_t items, size_t chunk) {
  return items == 0 ? 0 : (items + chunk - 1) / chunk;
}

/* ======================= tensor_ops.cpp ================================ */
double orc_sum_sq(const double* x, size_t n) { /* :45-59 */
  const size_t nchunks = chunk_count(n, SCALAR_CHUNK);
  double* partials = calloc(nchunks ? nchunks : 1, sizeof(double));
#pragma omp parallel for schedule(static)
  for (long long ci = 0; ci < (long long)nchunks; ++ci) {
    const size_t lo = (size_t)ci * SCALAR_CHUNK;
    const size_t hi = (lo + SCALAR_CHUNK < n) ? lo + SCALAR_CHUNK : n;
    double acc = 0.0;
    for (size_t i = lo; i < hi; ++i) acc += x[i] * x[i];
    partials[ci] = acc;
  }
  double total = 0.0;
  for (size_t c = 0; c < nchunks; ++c) total += partials[c];
  free(partials);
  return total;
}

static double sum_sq_diff(const double* a, const double* b, size_t n) { /* :61-78 */
  const size_t nchunks = chunk_count(n, SCALAR_CHUNK);
  double* partials = calloc(nchunks ? nchunks : 1, sizeof(double));
#pragma omp parallel for schedule(static)
  for (long long ci = 0; ci < (long long)nchunks; ++ci) {
    const size_t lo = (size_t)ci * SCALAR_CHUNK;
    const size_t hi = (lo + SCALAR_CHUNK < n) ? lo + SCALAR_CHUNK : n;
    double acc = 0.0;
    for (size_t i = lo; i < hi; ++i) {
      const double d = b[i] - a[i];
      acc += d * d;
    }
    partials[ci] = acc;
  }
  double total = 0.0;
  for (size_t c = 0; c < nchunks; ++c) total += partials[c];
  free(partials);
  return total;
}

double orc_frobenius_norm(const double* a, size_t n) { return sqrt(orc_sum_sq(a, n)); } /* :391-393 */

int orc_relative_error(const double* a, const double* b, size_t n, double* out,
                       orc_error* err) { /* :395-407 */
  const double ref_sq = orc_sum_sq(a, n);
  if (ref_sq == 0.0)
    return fail(err, ORC_E_ZERO_REFERENCE, USAGE, "relative_error: reference tensor has zero norm");
  const double diff_sq = sum_sq_diff(a, b, n);
  *out = sqrt(diff_sq / ref_sq);
  ok(err);
  return 0;
}

int orc_unfold_times(const double* a, int order, const uint64_t* dims, int mode,
                     const double* m, size_t ccols, double* out, orc_error* err) {
  /* :193-261 — chunk partials over kFiberChunk fibers, combined in order. */
  fiber_space fs;
  int st = make_space(order, dims, mode, &fs, err);
  if (st) return st;
  const size_t extent = fs.extent;
  const size_t nchunks = chunk_count(fs.fibers, FIBER_CHUNK);
  double* partials = calloc(nchunks * extent * ccols + 1, sizeof(double));
#pragma omp parallel for schedule(static)
  for (long long ci = 0; ci < (long long)nchunks; ++ci) {
    const size_t lo = (size_t)ci * FIBER_CHUNK;
    const size_t hi = (lo + FIBER_CHUNK < fs.fibers) ? lo + FIBER_CHUNK : fs.fibers;
    double* part = partials + (size_t)ci * extent * ccols;
    if (fs.stride == 1) { /* :214-225 */
      for (size_t j = lo; j < hi; ++j) {
        const double* fiber = a + j * extent;
        for (size_t c = 0; c < ccols; ++c) {
          const double w = m[j + c * fs.fibers];
          if (w == 0.0) continue;
          double* pc = part + c * extent;
          for (size_t i = 0; i < extent; ++i) pc[i] += fiber[i] * w;
        }
      }
      continue;
    }
    size_t j0 = lo; /* :231-251 runs inside one panel, extent tiled by 256 */
    while (j0 < hi) {
      const size_t panel = j0 / fs.stride;
      const size_t pend = (panel + 1) * fs.stride;
      const size_t run_end = hi < pend ? hi : pend;
      const size_t run = run_end - j0;
      const size_t base0 = panel * fs.stride * extent + (j0 % fs.stride);
      for (size_t i0 = 0; i0 < extent; i0 += 256) {
        const size_t i1 = (i0 + 256 < extent) ? i0 + 256 : extent;
        for (size_t c = 0; c < ccols; ++c) {
          const double* mc = m + c * fs.fibers + j0;
          double* pc = part + c * extent;
          for (size_t i = i0; i < i1; ++i) {
            const double* ai = a + base0 + i * fs.stride;
            double acc = 0.0;
            for (size_t jj = 0; jj < run; ++jj) acc += ai[jj] * mc[jj];
            pc[i] += acc;
          }
        }
      }
      j0 = run_end;
    }
  }
  memset(out, 0, extent * ccols * sizeof(double)); /* :254-259 */
  for (size_t ci = 0; ci < nchunks; ++ci) {
    const double* part = partials + ci * extent * ccols;
    for (size_t k = 0; k < extent * ccols; ++k) out[k] += part[k];
  }
  free(partials);
  ok(err);
  return 0;
}

int orc_unfold_t_times(const double* a, int order, const uint64_t* dims, int mode,
                       const double* m, size_t ccols, double* out, orc_error* err) {
  /* :263-330 — every output row is one fiber's serial contraction. */
  fiber_space fs;
  int st = make_space(order, dims, mode, &fs, err);
  if (st) return st;
  const size_t extent = fs.extent;
  double* mt = malloc((extent * ccols + 1) * sizeof(double));
  orc_transpose(m, extent, ccols, mt);
  const size_t nchunks = chunk_count(fs.fibers, FIBER_CHUNK);
#pragma omp parallel for schedule(static)
  for (long long ci = 0; ci < (long long)nchunks; ++ci) {
    const size_t lo = (size_t)ci * FIBER_CHUNK;
    const size_t hi = (lo + FIBER_CHUNK < fs.fibers) ? lo + FIBER_CHUNK : fs.fibers;
    if (fs.stride == 1) { /* :287-297 */
      for (size_t j = lo; j < hi; ++j) {
        const double* fiber = a + j * extent;
        for (size_t c = 0; c < ccols; ++c) {
          const double* mc = m + c * extent;
          double acc = 0.0;
          for (size_t i = 0; i < extent; ++i) acc += fiber[i] * mc[i];
          out[j + c * fs.fibers] = acc;
        }
      }
      continue;
    }
    double* acc = malloc(8 * ccols * sizeof(double)); /* :299-327 8-row tiles */
    size_t j0 = lo;
    while (j0 < hi) {
      const size_t panel = j0 / fs.stride;
      const size_t pend = (panel + 1) * fs.stride;
      const size_t run_end = hi < pend ? hi : pend;
      const size_t base0 = panel * fs.stride * extent + (j0 % fs.stride);
      for (size_t rb = 0; rb < run_end - j0; rb += 8) {
        const size_t rw = (run_end - j0 - rb < 8) ? run_end - j0 - rb : 8;
        memset(acc, 0, rw * ccols * sizeof(double));
        for (size_t i = 0; i < extent; ++i) {
          const double* ap = a + base0 + rb + i * fs.stride;
          const double* bt = mt + i * ccols;
          for (size_t rr = 0; rr < rw; ++rr) {
            const double av = ap[rr];
            double* arow = acc + rr * ccols;
            for (size_t c = 0; c < ccols; ++c) arow[c] += av * bt[c];
          }
        }
        for (size_t rr = 0; rr < rw; ++rr) {
          const size_t j = j0 + rb + rr;
          for (size_t c = 0; c < ccols; ++c) out[j + c * fs.fibers] = acc[rr * ccols + c];
        }
      }
      j0 = run_end;
    }
    free(acc);
  }
  free(mt);
  ok(err);
  return 0;
}

int orc_mode_n_product(const double* a, int order, const uint64_t* dims, const double* u,
                       size_t rows, size_t cols, int mode, double* out, orc_error* err) {
  /* :129-169 — per fiber gather then dot with each row of u. */
  fiber_space fs;
  int st = make_space(order, dims, mode, &fs, err);
  if (st) return st;
  if (cols != fs.extent)
    return fail(err, ORC_E_DIMENSION_MISMATCH, USAGE,
                "mode_n_product: factor has %zu columns, mode %d has extent %zu", cols, mode,
                fs.extent);
  double* ut = malloc((rows * cols + 1) * sizeof(double));
  orc_transpose(u, rows, cols, ut);
  const size_t r_out = rows;
  const size_t nchunks = chunk_count(fs.fibers, FIBER_CHUNK);
#pragma omp parallel for schedule(static)
  for (long long ci = 0; ci < (long long)nchunks; ++ci) {
    double* fiber = malloc(fs.extent * sizeof(double));
    const size_t lo = (size_t)ci * FIBER_CHUNK;
    const size_t hi = (lo + FIBER_CHUNK < fs.fibers) ? lo + FIBER_CHUNK : fs.fibers;
    for (size_t j = lo; j < hi; ++j) {
      const size_t base = fs_base(&fs, j);
      for (size_t i = 0; i < fs.extent; ++i) fiber[i] = a[base + i * fs.stride];
      const size_t obase = (j / fs.stride) * fs.stride * r_out + (j % fs.stride);
      for (size_t r = 0; r < r_out; ++r) {
        const double* urow = ut + r * fs.extent;
        double acc = 0.0;
        for (size_t i = 0; i < fs.extent; ++i) acc += fiber[i] * urow[i];
        out[obase + r * fs.stride] = acc;
      }
    }
    free(fiber);
  }
  free(ut);
  ok(err);
  return 0;
}

/* tensorize (:103-127): m is extent x fibers for the target shape. */
static void tensorize(const double* m, int order, const uint64_t* target, int mode, double* out) {
  fiber_space fs;
  make_space(order, target, mode, &fs, NULL);
  if (fs.stride == 1) {
    memcpy(out, m, fs.count * sizeof(double));
    return;
  }
#pragma omp parallel for schedule(static)
  for (long long j = 0; j < (long long)fs.fibers; ++j) {
    const size_t base = fs_base(&fs, (size_t)j);
    const double* col = m + (size_t)j * fs.extent;
    for (size_t i = 0; i < fs.extent; ++i) out[base + i * fs.stride] = col[i];
  }
}

static size_t count_of(int order, const uint64_t* dims) {
  size_t c = 1;
  for (int k = 0; k < order; ++k) c *= (size_t)dims[k];
  return c;
}

int orc_reconstruct(const double* core, int order, const uint64_t* ranks,
                    const uint64_t* dims, const double* factors, double* out,
                    orc_error* err) {
  /* :420-440 = multi_mode_product(core, {U_n, n}) in ascending mode order
   * (:171-191; the copy at :186 is the starting value). */
  uint64_t cur[64];
  for (int k = 0; k < order; ++k) cur[k] = ranks[k];
  size_t cap = count_of(order, dims);
  size_t maxsz = cap;
  {
    /* intermediate sizes can exceed the final size when I_n < R_n (never for
     * valid truncations, but be safe). */
    uint64_t d[64];
    for (int k = 0; k < order; ++k) d[k] = ranks[k];
    for (int n = 0; n < order; ++n) {
      d[n] = dims[n];
      size_t c = count_of(order, d);
      if (c > maxsz) maxsz = c;
    }
  }
  double* buf_a = malloc((maxsz + 1) * sizeof(double));
  double* buf_b = malloc((maxsz + 1) * sizeof(double));
  memcpy(buf_a, core, count_of(order, ranks) * sizeof(double));
  const double* u = factors;
  for (int n = 0; n < order; ++n) {
    int st = orc_mode_n_product(buf_a, order, cur, u, dims[n], ranks[n], n + 1, buf_b, err);
    if (st) {
      free(buf_a);
      free(buf_b);
      return st;
    }
    u += dims[n] * ranks[n];
    cur[n] = dims[n];
    double* t = buf_a;
    buf_a = buf_b;
    buf_b = t;
  }
  memcpy(out, buf_a, cap * sizeof(double));
  free(buf_a);
  free(buf_b);
  ok(err);
  return 0;
}

/* ======================= matrix.cpp ==================================== */
void orc_transpose(const double* a, size_t rows, size_t cols, double* out) { /* :32-40 */
  for (size_t j = 0; j < cols; ++j)
    for (size_t i = 0; i < rows; ++i) out[j + i * cols] = a[i + j * rows];
}

void orc_matmul(const double* a, size_t m, size_t k, const double* b, size_t n,
                double* c) { /* :42-69 — row blocks of 256, axpy over p */
  memset(c, 0, m * n * sizeof(double));
  const long long blocks = (long long)((m + 255) / 256);
#pragma omp parallel for schedule(static)
  for (long long blk = 0; blk < blocks; ++blk) {
    const size_t i0 = (size_t)blk * 256;
    const size_t i1 = (i0 + 256 < m) ? i0 + 256 : m;
    for (size_t j = 0; j < n; ++j) {
      double* cc = c + j * m;
      for (size_t p = 0; p < k; ++p) {
        const double bja = b[p + j * k];
        if (bja == 0.0) continue;
        const double* ac = a + p * m;
        for (size_t i = i0; i < i1; ++i) cc[i] += ac[i] * bja;
      }
    }
  }
}

void orc_gram(const double* a, size_t rows, size_t r, double* g) { /* :90-126 */
  const size_t nchunks = chunk_count(rows, FIBER_CHUNK);
  double* partials = calloc(nchunks * r * r + 1, sizeof(double));
#pragma omp parallel for schedule(static)
  for (long long ci = 0; ci < (long long)nchunks; ++ci) {
    const size_t lo = (size_t)ci * FIBER_CHUNK;
    const size_t hi = (lo + FIBER_CHUNK < rows) ? lo + FIBER_CHUNK : rows;
    double* part = partials + (size_t)ci * r * r;
    for (size_t j = 0; j < r; ++j) {
      const double* cj = a + j * rows;
      for (size_t i = 0; i <= j; ++i) {
        const double* c2 = a + i * rows;
        double acc = 0.0;
        for (size_t p = lo; p < hi; ++p) acc += c2[p] * cj[p];
        part[i + j * r] = acc;
      }
    }
  }
  memset(g, 0, r * r * sizeof(double));
  for (size_t ci = 0; ci < nchunks; ++ci) {
    const double* part = partials + ci * r * r;
    for (size_t j = 0; j < r; ++j)
      for (size_t i = 0; i <= j; ++i) g[i + j * r] += part[i + j * r];
  }
  for (size_t j = 0; j < r; ++j)
    for (size_t i = j + 1; i < r; ++i) g[i + j * r] = g[j + i * r];
  free(partials);
}

/* ======================= kernels.cpp =================================== */
int orc_reduced_qr(const double* a, size_t m, size_t n, double* q, double* r,
                   orc_error* err) { /* :303-367 Householder, R_ii >= 0 */
  if (m < n)
    return fail(err, ORC_E_DIMENSION_MISMATCH, USAGE, "reduced_qr: need rows >= cols, got %zux%zu",
                m, n);
  double* w = malloc((m * n + 1) * sizeof(double));
  memcpy(w, a, m * n * sizeof(double));
  double* vs = calloc(m * n + 1, sizeof(double)); /* v_k stored at vs + k*m, length m-k */
  double* betas = calloc(n + 1, sizeof(double));
  for (size_t k = 0; k < n; ++k) {
    double xnorm_sq = 0.0;
    for (size_t i = k; i < m; ++i) xnorm_sq += w[i + k * m] * w[i + k * m];
    const double xnorm = sqrt(xnorm_sq);
    double* v = vs + k * m;
    for (size_t i = k; i < m; ++i) v[i - k] = w[i + k * m];
    if (xnorm == 0.0) continue;
    const double alpha = v[0] >= 0.0 ? -xnorm : xnorm;
    v[0] -= alpha;
    double vnorm_sq = 0.0;
    for (size_t i = 0; i < m - k; ++i) vnorm_sq += v[i] * v[i];
    const double beta = 2.0 / vnorm_sq;
    for (size_t j = k; j < n; ++j) {
      double dot = 0.0;
      for (size_t i = k; i < m; ++i) dot += v[i - k] * w[i + j * m];
      const double step = beta * dot;
      for (size_t i = k; i < m; ++i) w[i + j * m] -= step * v[i - k];
    }
    w[k + k * m] = alpha;
    betas[k] = beta;
  }
  memset(r, 0, n * n * sizeof(double));
  for (size_t j = 0; j < n; ++j)
    for (size_t i = 0; i <= j; ++i) r[i + j * n] = w[i + j * m];
  memset(q, 0, m * n * sizeof(double));
  for (size_t k = 0; k < n; ++k) q[k + k * m] = 1.0;
  for (size_t k = n; k-- > 0;) {
    if (betas[k] == 0.0) continue;
    const double* v = vs + k * m;
    for (size_t j = k; j < n; ++j) {
      double dot = 0.0;
      for (size_t i = k; i < m; ++i) dot += v[i - k] * q[i + j * m];
      const double step = betas[k] * dot;
      for (size_t i = k; i < m; ++i) q[i + j * m] -= step * v[i - k];
    }
  }
  for (size_t k = 0; k < n; ++k) {
    if (r[k + k * n] >= 0.0) continue;
    for (size_t j = k; j < n; ++j) r[k + j * n] = -r[k + j * n];
    for (size_t i = 0; i < m; ++i) q[i + k * m] = -q[i + k * m];
  }
  free(w);
  free(vs);
  free(betas);
  ok(err);
  return 0;
}

int orc_spd_solve(const double* g, size_t n, const double* b, size_t k, double* x,
                  orc_error* err) { /* :369-417 Cholesky with pivot floor */
  double max_diag = 0.0;
  for (size_t i = 0; i < n; ++i)
    if (g[i + i * n] > max_diag) max_diag = g[i + i * n];
  const double floor_ = 1e-13 * max_diag;
  double* chol = calloc(n * n + 1, sizeof(double));
  for (size_t c = 0; c < n; ++c) {
    double pivot = g[c + c * n];
    for (size_t p = 0; p < c; ++p) pivot -= chol[c + p * n] * chol[c + p * n];
    if (pivot <= floor_ || !(pivot > 0.0)) {
      free(chol);
      return fail(err, ORC_E_SINGULAR_GRAM, NUMERICAL,
                  "spd_solve: pivot %f at column %zu is singular to working precision", pivot,
                  c + 1);
    }
    chol[c + c * n] = sqrt(pivot);
    for (size_t i = c + 1; i < n; ++i) {
      double acc = g[i + c * n];
      for (size_t p = 0; p < c; ++p) acc -= chol[i + p * n] * chol[c + p * n];
      chol[i + c * n] = acc / chol[c + c * n];
    }
  }
  memcpy(x, b, n * k * sizeof(double));
  for (size_t c = 0; c < k; ++c) {
    double* xc = x + c * n;
    for (size_t i = 0; i < n; ++i) {
      double acc = xc[i];
      for (size_t p = 0; p < i; ++p) acc -= chol[i + p * n] * xc[p];
      xc[i] = acc / chol[i + i * n];
    }
    for (size_t i = n; i-- > 0;) {
      double acc = xc[i];
      for (size_t p = i + 1; p < n; ++p) acc -= chol[p + i * n] * xc[p];
      xc[i] = acc / chol[i + i * n];
    }
  }
  free(chol);
  ok(err);
  return 0;
}

/* ======================= als.cpp ======================================= */
static double trace_product(const double* a, const double* b, size_t r) { /* :18-25 */
  double acc = 0.0;
  for (size_t j = 0; j < r; ++j)
    for (size_t i = 0; i < r; ++i) acc += a[i + j * r] * b[i + j * r];
  return acc;
}

int orc_als_init(const double* a, int order, const uint64_t* dims, int mode, size_t r,
                 uint64_t seed, double* l_out, orc_error* err) { /* :59-87 */
  fiber_space fs;
  int st = make_space(order, dims, mode, &fs, err);
  if (st) return st;
  if (r < 1 || r > fs.extent)
    return fail(err, ORC_E_RANK_TOO_LARGE, NUMERICAL, "mode %d: rank %zu outside 1..%zu", mode,
                r, fs.extent);
  orc_mt64 eng;
  orc_mt64_seeded(&eng, seed, (uint32_t)mode);
  double* s = malloc((fs.fibers * r + 1) * sizeof(double));
  for (size_t i = 0; i < fs.fibers * r; ++i) s[i] = orc_uniform01(&eng);
  double* y = malloc((fs.extent * r + 1) * sizeof(double));
  orc_unfold_times(a, order, dims, mode, s, r, y, NULL);
  free(s);
  double* rr = malloc((r * r + 1) * sizeof(double));
  orc_reduced_qr(y, fs.extent, r, l_out, rr, NULL);
  free(y);
  double max_diag = 0.0;
  for (size_t i = 0; i < r; ++i)
    if (fabs(rr[i + i * r]) > max_diag) max_diag = fabs(rr[i + i * r]);
  for (size_t i = 0; i < r; ++i) {
    if (fabs(rr[i + i * r]) <= 1e-13 * max_diag || max_diag == 0.0) {
      free(rr);
      return fail(err, ORC_E_DEGENERATE_INIT, NUMERICAL,
                  "als_init: randomized range collapsed at column %zu for mode %d", i + 1, mode);
    }
  }
  free(rr);
  ok(err);
  return 0;
}

int orc_als_low_rank(const double* a, int order, const uint64_t* dims, int mode, size_t r,
                     double eta, int max_iters_cfg, uint64_t seed, const double* init,
                     double* l_out, double* r_out, orc_als_report* rep, orc_error* err) {
  /* :98-161 */
  fiber_space fs;
  int st = make_space(order, dims, mode, &fs, err);
  if (st) return st;
  const size_t I = fs.extent, F = fs.fibers;
  const double norm = orc_frobenius_norm(a, fs.count);
  if (norm == 0.0)
    return fail(err, ORC_E_ZERO_REFERENCE, USAGE, "als_low_rank: input tensor has zero norm");
  const double norm_sq = norm * norm;
  double* l = malloc((I * r + 1) * sizeof(double));
  if (init) {
    memcpy(l, init, I * r * sizeof(double));
  } else {
    st = orc_als_init(a, order, dims, mode, r, seed, l, err);
    if (st) {
      free(l);
      return st;
    }
  }
  memset(rep, 0, sizeof(*rep));
  rep->status = 1; /* kMaxItersReached (:122) */
  double prev_residual = norm;
  const int max_iters = max_iters_cfg < 1 ? 1 : max_iters_cfg;
  double* lt_l = malloc((r * r + 1) * sizeof(double));
  double* rt_r = malloc((r * r + 1) * sizeof(double));
  double* at_l = malloc((F * r + 1) * sizeof(double));
  double* tmp = malloc((F * r + 1) * sizeof(double));
  double* rm = malloc((F * r + 1) * sizeof(double));
  double* a_r = malloc((I * r + 1) * sizeof(double));
  double* tmp2 = malloc((I * r + 1) * sizeof(double));
  int result = 0;
  for (int k = 1; k <= max_iters; ++k) {
    /* right_update :36-44 */
    orc_gram(l, I, r, lt_l);
    orc_unfold_t_times(a, order, dims, mode, l, r, at_l, NULL);
    orc_transpose(at_l, F, r, tmp); /* r x F */
    orc_error sub;
    if (orc_spd_solve(lt_l, r, tmp, F, at_l /* reuse as r x F */, &sub)) {
      result = fail(err, ORC_E_RANK_TOO_LARGE, NUMERICAL,
                    "mode %d: gram matrix is singular, rank %zu exceeds the numerical rank of the "
                    "iterate",
                    mode, r);
      goto done;
    }
    orc_transpose(at_l, r, F, rm); /* F x r */
    orc_gram(rm, F, r, rt_r);
    const double tr = trace_product(lt_l, rt_r, r);
    const double residual = sqrt(norm_sq - tr > 0.0 ? norm_sq - tr : 0.0); /* :52-55 */
    rep->iterations = k;
    if (k <= 64) rep->history[k - 1] = residual;
    rep->achieved_eta = fabs(prev_residual - residual) / norm;
    if (rep->achieved_eta <= eta) {
      rep->status = 0;
      goto finish;
    }
    if (k == max_iters) goto finish;
    /* left_update :46-50 */
    orc_unfold_times(a, order, dims, mode, rm, r, a_r, NULL);
    orc_transpose(a_r, I, r, tmp2); /* r x I */
    double* sol = malloc((r * I + 1) * sizeof(double));
    if (orc_spd_solve(rt_r, r, tmp2, I, sol, &sub)) {
      free(sol);
      result = fail(err, ORC_E_RANK_TOO_LARGE, NUMERICAL,
                    "mode %d: gram matrix is singular, rank %zu exceeds the numerical rank of the "
                    "iterate",
                    mode, r);
      goto done;
    }
    orc_transpose(sol, r, I, l);
    free(sol);
    prev_residual = residual;
  }
finish:
  memcpy(l_out, l, I * r * sizeof(double));
  if (r_out) memcpy(r_out, rm, F * r * sizeof(double));
  ok(err);
done:
  free(l);
  free(lt_l);
  free(rt_r);
  free(at_l);
  free(tmp);
  free(rm);
  free(a_r);
  free(tmp2);
  return result;
}

/* ======================= hosvd.cpp ===================================== */
/* recover_singular_vectors (hosvd.cpp:65-72): out = q V with V the left
 * singular vectors of q^T A_(mode). The reference takes dense_svd of the
 * r x F matrix q^T A_(mode) (kernels.cpp:419-446): transposed to F x r, a
 * Householder QR, then the r x r triangular factor T; the left vectors of
 * q^T A_(mode) are T's right singular vectors, ordered by descending singular
 * value (stable, kernels.cpp:273-301) and signed so each column's
 * largest-magnitude entry (first on ties) is positive (fix_column_signs,
 * kernels.cpp:25-43). This restatement computes T's right singular vectors
 * with the one-sided (Hestenes) Jacobi method instead of the reference's
 * Golub-Kahan iteration: equal to rounding, not bitwise (pinned against the
 * compiled reference by tests/test_oracle_pins.py). F < r (fewer fibers than
 * columns) is not covered (the reference then returns fewer columns). */
int orc_recover_singular_vectors(const double* a, int order, const uint64_t* dims, int mode,
                                 const double* q, size_t rows, size_t r, double* out,
                                 orc_error* err) {
  if (mode < 1 || mode > order)
    return fail(err, ORC_E_INVALID_MODE, USAGE, "recover_singular_vectors: mode %d outside 1..%d", mode,
                order);
  const size_t count = count_of(order, dims), I = dims[mode - 1];
  if (rows != I)
    return fail(err, ORC_E_DIMENSION_MISMATCH, USAGE, "recover_singular_vectors: q has %zu rows, extent %zu",
                rows, I);
  const size_t F = I ? count / I : 0;
  if (r == 0 || F < r)
    return fail(err, ORC_E_OTHER, USAGE, "recover_singular_vectors: %zu fibers for %zu columns", F, r);
  double* p = malloc((F * r + 1) * sizeof(double));   /* (q^T A_(mode))^T, F x r */
  double* qq = malloc((F * r + 1) * sizeof(double));
  double* t = malloc((r * r + 1) * sizeof(double));
  double* v = malloc((r * r + 1) * sizeof(double));
  double* w = malloc((r + 1) * sizeof(double));
  size_t* perm = malloc((r + 1) * sizeof(size_t));
  int st = orc_unfold_t_times(a, order, dims, mode, q, r, p, err);
  if (!st) st = orc_reduced_qr(p, F, r, qq, t, err);
  if (!st) {
    for (size_t i = 0; i < r * r; ++i) v[i] = 0.0;
    for (size_t i = 0; i < r; ++i) v[i + i * r] = 1.0;
    for (int sweep = 0; sweep < 80; ++sweep) { /* Hestenes: orthogonalise T's columns */
      int rotated = 0;
      for (size_t i = 0; i + 1 < r; ++i)
        for (size_t j = i + 1; j < r; ++j) {
          double al = 0.0, be = 0.0, ga = 0.0;
          for (size_t k = 0; k < r; ++k) {
            al += t[k + i * r] * t[k + i * r];
            be += t[k + j * r] * t[k + j * r];
            ga += t[k + i * r] * t[k + j * r];
          }
          if (ga == 0.0 || fabs(ga) <= 0x1.0p-60 * sqrt(al * be)) continue;
          const double zeta = (be - al) / (2.0 * ga);
          const double tn = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + tn * tn), sn = c * tn;
          for (size_t k = 0; k < r; ++k) {
            const double x = t[k + i * r], y = t[k + j * r];
            t[k + i * r] = c * x - sn * y;
            t[k + j * r] = sn * x + c * y;
            const double vx = v[k + i * r], vy = v[k + j * r];
            v[k + i * r] = c * vx - sn * vy;
            v[k + j * r] = sn * vx + c * vy;
          }
          rotated = 1;
        }
      if (!rotated) break;
    }
    for (size_t c = 0; c < r; ++c) {
      double n2 = 0.0;
      for (size_t k = 0; k < r; ++k) n2 += t[k + c * r] * t[k + c * r];
      w[c] = sqrt(n2);
      perm[c] = c;
    }
    for (size_t c = 1; c < r; ++c) { /* stable descending (insertion sort) */
      const size_t x = perm[c];
      size_t k = c;
      while (k > 0 && w[perm[k - 1]] < w[x]) {
        perm[k] = perm[k - 1];
        --k;
      }
      perm[k] = x;
    }
    for (size_t c = 0; c < r; ++c) { /* t <- V sorted and signed */
      const size_t col = perm[c];
      size_t arg = 0;
      double best = 0.0;
      for (size_t k = 0; k < r; ++k) {
        const double mag = fabs(v[k + col * r]);
        if (mag > best) {
          best = mag;
          arg = k;
        }
      }
      const double sg = v[arg + col * r] >= 0.0 ? 1.0 : -1.0;
      for (size_t k = 0; k < r; ++k) t[k + c * r] = sg * v[k + col * r];
    }
    orc_matmul(q, I, r, t, r, out);
    ok(err);
  }
  free(p);
  free(qq);
  free(t);
  free(v);
  free(w);
  free(perm);
  return st;
}

void orc_select_order(int order, const uint64_t* ranks, int* out) { /* :54-63 stable sort */
  for (int k = 0; k < order; ++k) out[k] = k + 1;
  for (int i = 1; i < order; ++i) { /* insertion sort is stable */
    int v = out[i];
    int j = i - 1;
    while (j >= 0 && ranks[out[j] - 1] > ranks[v - 1]) {
      out[j + 1] = out[j];
      --j;
    }
    out[j + 1] = v;
  }
}

static int validate_trunc(int order, const uint64_t* dims, const uint64_t* ranks,
                          orc_error* err) { /* shape.cpp:56-69 */
  for (int n = 0; n < order; ++n) {
    if (ranks[n] < 1 || ranks[n] > dims[n])
      return fail(err, ORC_E_RANK_TOO_LARGE, NUMERICAL, "mode %d: rank %llu outside 1..%llu",
                  n + 1, (unsigned long long)ranks[n], (unsigned long long)dims[n]);
  }
  return 0;
}

int orc_hosvd_als(int sequential, const double* a, int order, const uint64_t* dims,
                  const uint64_t* ranks, const int* mode_order, double eta, int max_iters,
                  uint64_t seed, double* core_out, double* factors_out, orc_hosvd_report* rep,
                  orc_error* err) {
  /* sequential == 2: t_hosvd with want_singular_vectors (hosvd.cpp:100-106) */
  const int want_sv = sequential == 2;
  if (want_sv) sequential = 0;
  int st = validate_trunc(order, dims, ranks, err);
  if (st) return st;
  memset(rep, 0, sizeof(*rep));
  const size_t count = count_of(order, dims);
  size_t fofs[64];
  size_t acc_ofs = 0;
  for (int n = 0; n < order; ++n) {
    fofs[n] = acc_ofs;
    acc_ofs += dims[n] * ranks[n];
  }
  int proc[64];
  if (!sequential) {
    for (int n = 0; n < order; ++n) proc[n] = n + 1;
  } else if (mode_order) { /* checked_order :30-50 */
    int seen[64] = {0};
    for (int k = 0; k < order; ++k) {
      int m = mode_order[k];
      if (m < 1 || m > order || seen[m - 1])
        return fail(err, ORC_E_INVALID_MODE, USAGE,
                    "st_hosvd: order is not a permutation of 1..%d", order);
      seen[m - 1] = 1;
      proc[k] = m;
    }
  } else {
    orc_select_order(order, ranks, proc);
  }
  if (!sequential) { /* t_hosvd :74-125 */
    for (int n = 1; n <= order; ++n) {
      const size_t r = ranks[n - 1];
      const size_t I = dims[n - 1];
      double* l = malloc((I * r + 1) * sizeof(double));
      st = orc_als_low_rank(a, order, dims, n, r, eta, max_iters, seed, NULL, l, NULL,
                            &rep->als[n - 1], err);
      if (st) {
        free(l);
        return st;
      }
      rep->modes[n - 1] = n;
      double* rr = malloc((r * r + 1) * sizeof(double));
      orc_reduced_qr(l, I, r, factors_out + fofs[n - 1], rr, NULL);
      free(rr);
      free(l);
      if (want_sv) {
        double* qv = malloc((I * r + 1) * sizeof(double));
        st = orc_recover_singular_vectors(a, order, dims, n, factors_out + fofs[n - 1], I, r, qv, err);
        if (!st) memcpy(factors_out + fofs[n - 1], qv, I * r * sizeof(double));
        free(qv);
        if (st) return st;
      }
    }
    /* core = multi_mode_product(t, {U_n^T}) ascending (:115-121) */
    uint64_t cur[64];
    for (int k = 0; k < order; ++k) cur[k] = dims[k];
    double* buf_a = malloc((count + 1) * sizeof(double));
    double* buf_b = malloc((count + 1) * sizeof(double));
    memcpy(buf_a, a, count * sizeof(double));
    for (int n = 1; n <= order; ++n) {
      const size_t I = dims[n - 1], r = ranks[n - 1];
      double* ut = malloc((I * r + 1) * sizeof(double));
      orc_transpose(factors_out + fofs[n - 1], I, r, ut);
      orc_mode_n_product(buf_a, order, cur, ut, r, I, n, buf_b, NULL);
      free(ut);
      cur[n - 1] = r;
      double* t = buf_a;
      buf_a = buf_b;
      buf_b = t;
    }
    memcpy(core_out, buf_a, count_of(order, ranks) * sizeof(double));
    free(buf_a);
    free(buf_b);
  } else { /* st_hosvd :127-191 */
    uint64_t cur[64];
    for (int k = 0; k < order; ++k) cur[k] = dims[k];
    double* working = malloc((count + 1) * sizeof(double));
    memcpy(working, a, count * sizeof(double));
    for (int k = 0; k < order; ++k) {
      const int n = proc[k];
      const size_t r = ranks[n - 1];
      const size_t I = cur[n - 1];
      const size_t F = count_of(order, cur) / I;
      double* l = malloc((I * r + 1) * sizeof(double));
      double* rm = malloc((F * r + 1) * sizeof(double));
      st = orc_als_low_rank(working, order, cur, n, r, eta, max_iters, seed, NULL, l, rm,
                            &rep->als[k], err);
      if (st) {
        free(l);
        free(rm);
        free(working);
        return st;
      }
      rep->modes[k] = n;
      double* rr = malloc((r * r + 1) * sizeof(double));
      orc_reduced_qr(l, I, r, factors_out + fofs[n - 1], rr, NULL);
      /* working = tensorize(matmul(R_hat, R^T), mode, shrunk) (:178) */
      double* rt = malloc((F * r + 1) * sizeof(double));
      orc_transpose(rm, F, r, rt);
      double* prod = malloc((r * F + 1) * sizeof(double));
      orc_matmul(rr, r, r, rt, F, prod);
      cur[n - 1] = r;
      tensorize(prod, order, cur, n, working);
      free(rt);
      free(prod);
      free(rr);
      free(l);
      free(rm);
    }
    memcpy(core_out, working, count_of(order, ranks) * sizeof(double));
    free(working);
  }
  /* relative_residual = relative_error(t, reconstruct(tk)) (:123,189) */
  double* rec = malloc((count + 1) * sizeof(double));
  orc_reconstruct(core_out, order, ranks, dims, factors_out, rec, NULL);
  st = orc_relative_error(a, rec, count, &rep->relative_residual, err);
  free(rec);
  if (st) return st;
  for (int k = 0; k < order; ++k)
    if (!sequential) rep->modes[k] = k + 1;
  ok(err);
  return 0;
}
