/* simgen_oracle.c — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * The benchmark inputs generated without the product library, so that bench.py's reference
 * arm (`--impl reference`) never loads libplingam_b200.so. Restates the package's
 * generators (paper_2403_03772_b200/csrc/host/simgen.cpp), which follow the reference's
 * semantics: proj/include/plingam/rng.hpp:14-43 (mt19937_64, 53-bit uniforms, Box-Muller,
 * Fisher-Yates) and proj/src/simgen.cpp:30-81 (two-level DAG, causal-order sampling), plus
 * the sparse Erdos-Renyi DAG and Laplace / Student-t3 / Gaussian noise the configs name.
 * tests/test_host_cpu.py checks the outputs bit for bit against the package's generators.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "plingam_oracle.h"

/* std::mt19937_64 (the C++ standard's parameters) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

static double unif(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
static double unif_ab(mt64* g, double lo, double hi) { return lo + (hi - lo) * unif(g); }
static double gauss(mt64* g) {
  const double u1 = 1.0 - unif(g);
  const double u2 = unif(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}
static void shuffle(mt64* g, int32_t* v, int n) {
  for (int i = n; i > 1; --i) {
    const int j = (int)(unif(g) * (double)i);
    const int32_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

/* kind: 0 uniform(lo, hi), 1 Laplace(scale hi), 2 Student-t3 (scale hi), 3 N(lo, hi^2) */
static double draw_noise(mt64* g, int kind, double lo, double hi) {
  if (kind == 0) return unif_ab(g, lo, hi);
  if (kind == 1) {
    const double p = unif(g) - 0.5;
    const double a = 1.0 - 2.0 * fabs(p);
    return -hi * (p < 0 ? -1.0 : 1.0) * log(a > 0 ? a : 0x1.0p-53);
  }
  if (kind == 3) return lo + hi * gauss(g);
  const double z = gauss(g);
  double chi = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double x = gauss(g);
    chi += x * x;
  }
  return hi * z / sqrt(chi / 3.0);
}

int orc_gen_two_level_dag(int32_t d, uint64_t seed, double edge_prob, double* W, int32_t* order) {
  if (d < 2) return -1;
  const int n0 = (d + 1) / 2;
  mt64 g;
  mt64_seed(&g, seed);
  memset(W, 0, sizeof(double) * (size_t)d * d);
  for (int v = 0; v < d; ++v) order[v] = v;
  shuffle(&g, order, d);
  for (int u = 0; u < n0; ++u)
    for (int v = n0; v < d; ++v)
      if (unif(&g) < edge_prob) W[(size_t)order[v] + (size_t)d * order[u]] = gauss(&g);
  return 0;
}

int orc_gen_sparse_dag(int32_t d, double avg_parents, uint64_t seed, double wmin, double wmax, double* W,
                       int32_t* order) {
  if (d < 2) return -1;
  mt64 g;
  mt64_seed(&g, seed);
  memset(W, 0, sizeof(double) * (size_t)d * d);
  for (int v = 0; v < d; ++v) order[v] = v;
  shuffle(&g, order, d);
  double p = 2.0 * avg_parents / (double)(d - 1);
  if (p > 1.0) p = 1.0;
  for (int b = 1; b < d; ++b)
    for (int a = 0; a < b; ++a)
      if (unif(&g) < p) {
        const double mag = unif_ab(&g, wmin, wmax);
        const double w = unif(&g) < 0.5 ? -mag : mag;
        W[(size_t)order[b] + (size_t)d * order[a]] = w;
      }
  return 0;
}

int orc_sample_lingam(const double* W, const int32_t* order, int32_t d, int64_t n, uint64_t seed, int32_t kind,
                      double lo, double hi, double* X) {
  int32_t* pc = calloc((size_t)d, sizeof(int32_t));
  int32_t* pj = malloc(sizeof(int32_t) * (size_t)d * d);
  double* pw = malloc(sizeof(double) * (size_t)d * d);
  double* eps = malloc(sizeof(double) * (size_t)d);
  double* x = calloc((size_t)d, sizeof(double));
  if (!pc || !pj || !pw || !eps || !x) {
    free(pc), free(pj), free(pw), free(eps), free(x);
    return -1;
  }
  for (int v = 0; v < d; ++v)
    for (int j = 0; j < d; ++j) {
      const double w = W[(size_t)v + (size_t)d * j];
      if (w != 0.0) {
        pj[(size_t)v * d + pc[v]] = j;
        pw[(size_t)v * d + pc[v]] = w;
        ++pc[v];
      }
    }
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t r = 0; r < n; ++r) {
    for (int j = 0; j < d; ++j) eps[j] = draw_noise(&g, kind, lo, hi);
    for (int i = 0; i < d; ++i) {
      const int v = order[i];
      double s = 0.0;
      for (int k = 0; k < pc[v]; ++k) s += pw[(size_t)v * d + k] * x[pj[(size_t)v * d + k]];
      x[v] = s + eps[v];
    }
    for (int j = 0; j < d; ++j) X[r + n * (int64_t)j] = x[j];
  }
  free(pc), free(pj), free(pw), free(eps), free(x);
  return 0;
}
