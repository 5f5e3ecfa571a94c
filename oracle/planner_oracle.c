/* TEST INFRASTRUCTURE ONLY (oracle): plain-C restatement of the reference
 * planner path, used as the checker for the product's host planner
 * (include/mimose) and never linked into it.
 *
 * Restated algorithms (reference file:line under proj/include/mimose/):
 *   orc_sample_workload  workload.hpp:63-106   mt19937_64 stream, uniform
 *                        `min + rng() % span`, Box-Muller normal, power-law
 *                        inverse CDF, llround + clamp, x batch multiplier
 *   orc_fit_layer        estimator.hpp:40-147  OLS normal equations with
 *                        columns scaled by xmax^k, Gaussian elimination with
 *                        partial pivoting (pivot < 1e-12 -> error)
 *   orc_predict          estimator.hpp:69-73,150-159  Horner, clamp >= 0, llround
 *   orc_generate_plan    scheduler.hpp:81-167  Algorithm 1 bucketed greedy
 *   orc_simulate         simulator.hpp:104-160 iteration replay
 * Pinned against the reference's golden vectors in tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------- mt19937_64 */
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
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double unit(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* dist: 0 uniform, 1 normal, 2 power-law */
int orc_sample_workload(int dist, int64_t umin, int64_t umax, double mu, double sigma,
                        double alpha, int64_t mult, int64_t iters, uint64_t seed, int64_t* out) {
  if (umin < 1 || umin > umax || mult < 1 || iters < 0) return 1;
  mt64 g;
  mt64_seed(&g, seed);
  const double lo = (double)umin, hi = (double)umax;
  for (int64_t i = 0; i < iters; ++i) {
    int64_t u;
    if (dist == 0) {
      const uint64_t span = (uint64_t)(umax - umin) + 1;
      u = umin + (int64_t)(mt64_next(&g) % span);
    } else if (dist == 1) {
      double u1 = unit(&g);
      const double u2 = unit(&g);
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
      u = (int64_t)llround(mu + sigma * z);
    } else {
      const double r = unit(&g);
      double v;
      if (alpha == 1.0) {
        v = lo * pow(hi / lo, r);
      } else {
        const double p = 1.0 - alpha;
        v = pow(pow(lo, p) + r * (pow(hi, p) - pow(lo, p)), 1.0 / p);
      }
      u = (int64_t)llround(v);
    }
    if (u < umin) u = umin;
    if (u > umax) u = umax;
    out[i] = u * mult;
  }
  return 0;
}

/* ---------------------------------------------------------- estimator */
double orc_eval_poly(const double* c, int n, double x) {
  double acc = 0.0;
  for (int k = n - 1; k >= 0; --k) acc = acc * x + c[k];
  return acc;
}

int64_t orc_predict(const double* c, int n, int64_t x) {
  double v = orc_eval_poly(c, n, (double)x);
  if (v < 0.0) v = 0.0;
  return (int64_t)llround(v);
}

/* samples of ONE layer: xs[i] input size, ys[i] bytes. Returns 0 ok,
 * 2 too few distinct sizes, 3 singular. coeffs: order+1 doubles. */
int orc_fit_layer(const int64_t* xs, const int64_t* ys, int n, int order, double* coeffs) {
  const int m = order + 1;
  if (order < 0 || order > 8) return 1;
  int distinct = 0;
  for (int i = 0; i < n; ++i) {
    int seen = 0;
    for (int j = 0; j < i; ++j) seen |= xs[j] == xs[i];
    distinct += !seen;
  }
  if (distinct < m) return 2;
  double xmax = 0.0;
  for (int i = 0; i < n; ++i) {
    const double a = fabs((double)xs[i]);
    if (a > xmax) xmax = a;
  }
  if (xmax == 0.0) xmax = 1.0;
  double scale[9], G[9][9], r[9], row[9];
  scale[0] = 1.0;
  for (int k = 1; k < m; ++k) scale[k] = scale[k - 1] * xmax;
  memset(G, 0, sizeof(G));
  memset(r, 0, sizeof(r));
  for (int i = 0; i < n; ++i) {
    const double x = (double)xs[i], y = (double)ys[i];
    double xp = 1.0;
    for (int k = 0; k < m; ++k) {
      row[k] = xp / scale[k];
      xp *= x;
    }
    for (int a = 0; a < m; ++a) {
      for (int b = 0; b < m; ++b) G[a][b] += row[a] * row[b];
      r[a] += row[a] * y;
    }
  }
  for (int col = 0; col < m; ++col) {
    int piv = col;
    for (int a = col + 1; a < m; ++a)
      if (fabs(G[a][col]) > fabs(G[piv][col])) piv = a;
    if (fabs(G[piv][col]) < 1e-12) return 3;
    for (int b = 0; b < m; ++b) {
      const double t = G[col][b];
      G[col][b] = G[piv][b];
      G[piv][b] = t;
    }
    const double t = r[col];
    r[col] = r[piv];
    r[piv] = t;
    for (int a = col + 1; a < m; ++a) {
      const double f = G[a][col] / G[col][col];
      for (int b = col; b < m; ++b) G[a][b] -= f * G[col][b];
      r[a] -= f * r[col];
    }
  }
  double sol[9];
  for (int a = m - 1; a >= 0; --a) {
    double acc = r[a];
    for (int b = a + 1; b < m; ++b) acc -= G[a][b] * sol[b];
    sol[a] = acc / G[a][a];
  }
  for (int k = 0; k < m; ++k) coeffs[k] = sol[k] / scale[k];
  return 0;
}

/* ---------------------------------------------------------- scheduler */
typedef struct {
  int idx, pos;
  int64_t est;
} item;

static int by_est_desc(const void* a, const void* b) {
  const item* x = (const item*)a;
  const item* y = (const item*)b;
  if (x->est != y->est) return x->est > y->est ? -1 : 1;
  return x->pos - y->pos;
}
static int by_pos(const void* a, const void* b) {
  return ((const item*)a)->pos - ((const item*)b)->pos;
}

/* est[i]/pos[i] per layer (index i = forward order). dropped[i] set to 1 for
 * dropped layers. budget/reserve as SchedulerConfig (reserve < 0 -> 8%). */
int orc_generate_plan(const int64_t* est, const int* pos, int L, int64_t budget,
                      int64_t reserve, double tol, int64_t constant, int excess_incl_const,
                      int* dropped, int* insufficient) {
  if (L <= 0 || L > 4096) return 1;
  if (reserve < 0) reserve = (int64_t)llround(0.08 * (double)budget);
  item* it = (item*)malloc(sizeof(item) * (size_t)L);
  int* bstart = (int*)malloc(sizeof(int) * (size_t)(L + 1));
  int* bhead = (int*)malloc(sizeof(int) * (size_t)L); /* next unpicked member per bucket */
  int64_t sum = 0;
  for (int i = 0; i < L; ++i) {
    it[i].idx = i;
    it[i].pos = pos[i];
    it[i].est = est[i];
    sum += est[i];
    dropped[i] = 0;
  }
  qsort(it, (size_t)L, sizeof(item), by_est_desc);
  int nb = 0, i = 0;
  while (i < L) {
    const double fl = (double)it[i].est * (1.0 - tol);
    bstart[nb] = i++;
    while (i < L && (double)it[i].est > fl) ++i;
    qsort(it + bstart[nb], (size_t)(i - bstart[nb]), sizeof(item), by_pos);
    ++nb;
  }
  bstart[nb] = L;
  for (int b = 0; b < nb; ++b) bhead[b] = bstart[b];
  int64_t excess = sum - (budget - reserve);
  if (excess_incl_const) excess += constant;
  *insufficient = 0;
  while (excess > 0) {
    int chosen = -1;
    for (int b = nb - 1; b >= 0 && chosen < 0; --b) {
      if (bhead[b] == bstart[b + 1]) continue;
      int64_t mx = 0;
      for (int k = bhead[b]; k < bstart[b + 1]; ++k)
        if (it[k].est > mx) mx = it[k].est;
      if (mx > excess) chosen = b;
    }
    if (chosen < 0)
      for (int b = 0; b < nb && chosen < 0; ++b)
        if (bhead[b] < bstart[b + 1]) chosen = b;
    if (chosen < 0) {
      *insufficient = 1;
      break;
    }
    const item pick = it[bhead[chosen]++];
    dropped[pick.idx] = 1;
    excess -= pick.est;
  }
  free(it);
  free(bstart);
  free(bhead);
  return 0;
}

/* ---------------------------------------------------------- simulator */
int orc_simulate(const int64_t* act, const int64_t* bnd, const double* fwd, const int* dropped,
                 int L, int64_t constant, int64_t* peak_out, double* time_out, double* rc_out) {
  int64_t res = constant, peak = constant;
  double t = 0.0, rc = 0.0;
  for (int i = 0; i < L; ++i) {
    t += fwd[i];
    if (dropped[i]) {
      if (res + act[i] > peak) peak = res + act[i];
      res += bnd[i];
    } else {
      res += act[i];
      if (res > peak) peak = res;
    }
  }
  for (int i = L - 1; i >= 0; --i) {
    if (dropped[i]) {
      res += act[i] - bnd[i];
      t += fwd[i];
      if (res > peak) peak = res;
      rc += fwd[i];
    }
    t += 2.0 * fwd[i];
    res -= act[i];
    if (res > peak) peak = res;
  }
  *peak_out = peak;
  *time_out = t;
  *rc_out = rc;
  return 0;
}
