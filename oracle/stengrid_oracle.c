/*
 * oracle/stengrid_oracle.c — CPU RESTATEMENT OF THE REFERENCE HOT PATH.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker
 * (never as the thing measured or shipped). The product path lives in
 * paper_1902_09931_b200/ and never calls into oracle/.
 *
 * Plain C, compiled with -O2 -ffp-contract=off (the reference's own flag,
 * CMakeLists.txt:15-21) so every floating-point expression below is evaluated
 * exactly in the order written, with no FMA contraction: results are bitwise
 * identical to the reference build.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bitwise
 * against (a) the reference compiled from /root/reference by oracle/Makefile
 * (oracle/_ref/libstengrid_ref.so) on random cases, and (b) the committed
 * golden fixtures in tests/golden/ (generated from the reference by
 * tests/golden/make_golden.py) and the reference's own known-answer tests.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ grid */

/* wrap(i, n): grid.cpp:42-47 (int64 modulo, shifted into [0, n)). */
int orc_wrap(long long i, int n) {
  long long r = i % n;
  if (r < 0) r += n;
  return (int)r;
}

/* make_tiles: grid.cpp:62-82 — ceil-first contiguous row ranges. */
int orc_make_tiles(int ny, int numTiles, int* begins, int* ends) {
  if (ny < 1 || numTiles < 1 || numTiles > ny) return -1;
  int base = ny / numTiles, extra = ny % numTiles, j = 0;
  for (int t = 0; t < numTiles; ++t) {
    int rows = base + (t < extra ? 1 : 0);
    begins[t] = j;
    ends[t] = j + rows;
    j += rows;
  }
  return 0;
}

/* ------------------------------------------------------- window functions
 * Same arithmetic order as the reference's functions (see ref_driver.cpp for
 * the file:line of each); ids match include/stengrid/sg.h SG_FN_*. */
typedef double (*orc_fn)(const double*, const double*, int);

static double f_ch_nonlinear(const double* w, const double* coe, int rs) {
  double acc = 0.0;
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) {
      double v = w[q * rs + p];
      acc += coe[q * 3 + p] * (v * v * v - v);
    }
  return acc;
}
static double f_central_difference(const double* w, const double* coe, int rs) {
  (void)rs;
  return (w[0] - 2.0 * w[1] + w[2]) * coe[0];
}
static double f_center(const double* w, const double* coe, int rs) {
  (void)coe;
  return w[rs + 1];
}
static double f_central_second(const double* w, const double* coe, int rs) {
  (void)rs;
  double acc = 0.0;
  acc += coe[0] * w[0];
  acc += (-2.0 * coe[0]) * w[1];
  acc += coe[0] * w[2];
  return acc;
}
static double g_cube(double v) { return v * v * v - v; }
static double f_lap_cube_diff_first(const double* w, const double* coe, int rs) {
  double gm = g_cube(w[rs + 1]);
  double x = (g_cube(w[rs]) - 2.0 * gm) + g_cube(w[rs + 2]);
  double y = (g_cube(w[1]) - 2.0 * gm) + g_cube(w[2 * rs + 1]);
  return coe[0] * x + coe[1] * y;
}
static double f_weighted_3x3(const double* w, const double* coe, int rs) {
  double acc = 0.0;
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) acc += coe[q * 3 + p] * w[q * rs + p];
  return acc;
}

static orc_fn fn_by_id(int id) {
  switch (id) {
    case 1: return f_ch_nonlinear;
    case 2: return f_central_difference;
    case 3: return f_center;
    case 4: return f_central_second;
    case 5: return f_lap_cube_diff_first;
    case 6: return f_weighted_3x3;
    default: return 0;
  }
}

/* ---------------------------------------------------------------- stencil
 * One application of a weight (fnId == 0) or function stencil.
 * Geometry: make_geom (stencil.cpp:26-40): periodic computes every point with
 * wrapped rows/columns; non-periodic computes rows [top, ny-bottom) and
 * columns [min(left,nx), max(min(nx-right,nx), fastLo)) and leaves the frame
 * of `out` untouched. Weight arithmetic: weights_rows / weights_wrapped_point
 * (stencil.cpp:49-85): acc = 0; acc += w[q*W+p] * in(...) row-major. Function
 * stencils hand fn a packed window (rowStride = W), which is value-identical
 * to the reference's strided view (stencil.cpp:104-119). */
int orc_stencil(int periodic, const int* ext, int fnId, const double* w, const double* in,
                double* out, int nx, int ny) {
  const int left = ext[0], right = ext[1], top = ext[2], bottom = ext[3];
  const int W = left + right + 1, H = top + bottom + 1;
  orc_fn fn = 0;
  if (fnId != 0) {
    fn = fn_by_id(fnId);
    if (!fn) return -1;
  }
  int rowLo = periodic ? 0 : top;
  int rowHi = periodic ? ny : ny - bottom;
  int colLo, colHi;
  if (periodic) {
    colLo = 0;
    colHi = nx;
  } else {
    int fastLo = left < nx ? left : nx;
    int t = nx - right < nx ? nx - right : nx;
    colLo = fastLo;
    colHi = t > fastLo ? t : fastLo;
  }
  double* window = (double*)malloc(sizeof(double) * (size_t)W * (size_t)H);
  for (int j = rowLo; j < rowHi; ++j) {
    for (int i = colLo; i < colHi; ++i) {
      if (fn) {
        for (int q = 0; q < H; ++q) {
          long long jj = (long long)j - top + q;
          if (periodic) jj = orc_wrap(jj, ny);
          for (int p = 0; p < W; ++p) {
            long long ii = (long long)i - left + p;
            if (periodic) ii = orc_wrap(ii, nx);
            window[q * W + p] = in[jj * nx + ii];
          }
        }
        out[(long long)j * nx + i] = fn(window, w, W);
      } else {
        double acc = 0.0;
        for (int q = 0; q < H; ++q) {
          long long jj = (long long)j - top + q;
          if (periodic) jj = orc_wrap(jj, ny);
          for (int p = 0; p < W; ++p) {
            long long ii = (long long)i - left + p;
            if (periodic) ii = orc_wrap(ii, nx);
            acc += w[q * W + p] * in[jj * nx + ii];
          }
        }
        out[(long long)j * nx + i] = acc;
      }
    }
  }
  free(window);
  return 0;
}

/* ------------------------------------------------------------------ penta
 * Interleaved layout idx(b, r) = r*B + b (penta.hpp:30-32). */

/* Non-pivoting LU: PentaFactor ctor, penta.cpp:93-158. Returns -1 on success
 * or the system index of the first zero pivot (row-major scan order, as
 * pivot_check, penta.cpp:119-123). */
int orc_penta_factor(int B, int n, const double* e, const double* c, const double* d,
                     const double* a, const double* b, double* m1, double* m2, double* dInv,
                     double* ap, double* bp) {
  const long long len = (long long)B * n;
  double* dp = (double*)malloc(sizeof(double) * (size_t)len);
  memcpy(bp, b, sizeof(double) * (size_t)len);
  memset(m1, 0, sizeof(double) * (size_t)len);
  memset(m2, 0, sizeof(double) * (size_t)len);
  int bad = -1;
  for (int q = 0; q < B; ++q) {
    dp[q] = d[q];
    ap[q] = a[q];
  }
  for (int q = 0; q < B && bad < 0; ++q)
    if (dp[q] == 0.0) bad = q;
  if (bad < 0) {
    for (int q = 0; q < B; ++q) {
      double mm = c[B + q] / dp[q];
      m2[B + q] = mm;
      dp[B + q] = d[B + q] - mm * ap[q];
      ap[B + q] = a[B + q] - mm * bp[q];
    }
    for (int q = 0; q < B && bad < 0; ++q)
      if (dp[B + q] == 0.0) bad = q;
  }
  for (int r = 2; r < n && bad < 0; ++r) {
    long long cur = (long long)r * B, p1 = cur - B, p2 = cur - 2LL * B;
    for (int q = 0; q < B; ++q) {
      double mm1 = e[cur + q] / dp[p2 + q];
      double cbar = c[cur + q] - mm1 * ap[p2 + q];
      double mm2 = cbar / dp[p1 + q];
      m1[cur + q] = mm1;
      m2[cur + q] = mm2;
      dp[cur + q] = d[cur + q] - mm1 * bp[p2 + q] - mm2 * ap[p1 + q];
      ap[cur + q] = a[cur + q] - mm2 * bp[p1 + q];
    }
    for (int q = 0; q < B && bad < 0; ++q)
      if (dp[cur + q] == 0.0) bad = q;
  }
  if (bad < 0)
    for (long long k = 0; k < len; ++k) dInv[k] = 1.0 / dp[k];
  free(dp);
  return bad;
}

/* Forward/back substitution: PentaFactor::solve_range, penta.cpp:160-197. */
void orc_penta_substitute(int B, int n, const double* m1, const double* m2, const double* dInv,
                          const double* ap, const double* bp, double* y) {
  for (int q = 0; q < B; ++q) y[B + q] -= m2[B + q] * y[q];
  for (int r = 2; r < n; ++r) {
    long long cur = (long long)r * B, p1 = cur - B, p2 = cur - 2LL * B;
    for (int q = 0; q < B; ++q) y[cur + q] -= m1[cur + q] * y[p2 + q] + m2[cur + q] * y[p1 + q];
  }
  long long last = (long long)(n - 1) * B, prev = last - B;
  for (int q = 0; q < B; ++q) y[last + q] *= dInv[last + q];
  for (int q = 0; q < B; ++q)
    y[prev + q] = (y[prev + q] - ap[prev + q] * y[last + q]) * dInv[prev + q];
  for (int r = n - 3; r >= 0; --r) {
    long long cur = (long long)r * B, s1 = cur + B, s2 = cur + 2LL * B;
    for (int q = 0; q < B; ++q)
      y[cur + q] = (y[cur + q] - ap[cur + q] * y[s1 + q] - bp[cur + q] * y[s2 + q]) * dInv[cur + q];
  }
}

/* 4x4 partial-pivot LU and solve: lu4_factor / lu4_solve, penta.cpp:37-70. */
int orc_lu4_factor(double* K, int* piv) {
  for (int c = 0; c < 4; ++c) {
    int pr = c;
    double best = fabs(K[c * 4 + c]);
    for (int r = c + 1; r < 4; ++r) {
      double cand = fabs(K[r * 4 + c]);
      if (cand > best) {
        best = cand;
        pr = r;
      }
    }
    if (best == 0.0) return -1;
    piv[c] = pr;
    if (pr != c)
      for (int cc = 0; cc < 4; ++cc) {
        double t = K[c * 4 + cc];
        K[c * 4 + cc] = K[pr * 4 + cc];
        K[pr * 4 + cc] = t;
      }
    double inv = 1.0 / K[c * 4 + c];
    for (int r = c + 1; r < 4; ++r) {
      double m = K[r * 4 + c] * inv;
      K[r * 4 + c] = m;
      for (int cc = c + 1; cc < 4; ++cc) K[r * 4 + cc] -= m * K[c * 4 + cc];
    }
  }
  return 0;
}

void orc_lu4_solve(const double* K, const int* piv, double* y) {
  for (int c = 0; c < 4; ++c)
    if (piv[c] != c) {
      double t = y[c];
      y[c] = y[piv[c]];
      y[piv[c]] = t;
    }
  for (int r = 1; r < 4; ++r)
    for (int c = 0; c < r; ++c) y[r] -= K[r * 4 + c] * y[c];
  for (int r = 3; r >= 0; --r) {
    for (int c = r + 1; c < 4; ++c) y[r] -= K[r * 4 + c] * y[c];
    y[r] /= K[r * 4 + r];
  }
}

/* Batched solve, periodic via Woodbury (PeriodicPentaFactor, penta.cpp:204-295)
 * or plain (solve_batch, penta.cpp:297-303). rhs is overwritten with the
 * solution. Returns -1 on success, else the failing system index (zero pivot
 * or singular capacitance matrix). */
int orc_penta_solve(int periodic, int B, int n, const double* e, const double* c, const double* d,
                    const double* a, const double* b, double* rhs) {
  const size_t len = (size_t)B * (size_t)n;
  double *m1 = malloc(len * 8), *m2 = malloc(len * 8), *dInv = malloc(len * 8),
         *ap = malloc(len * 8), *bp = malloc(len * 8);
  int bad = orc_penta_factor(B, n, e, c, d, a, b, m1, m2, dInv, ap, bp);
  if (bad >= 0) goto done;
  if (!periodic) {
    orc_penta_substitute(B, n, m1, m2, dInv, ap, bp, rhs);
    goto done;
  }
  {
    double* Wk[4];
    const int rowOf[4] = {0, 1, n - 2, n - 1};
    for (int k = 0; k < 4; ++k) {
      Wk[k] = calloc(len, 8);
      for (int q = 0; q < B; ++q) Wk[k][(size_t)rowOf[k] * B + q] = 1.0;
      orc_penta_substitute(B, n, m1, m2, dInv, ap, bp, Wk[k]);
    }
    double* K = malloc((size_t)B * 16 * 8);
    int* piv = malloc((size_t)B * 4 * sizeof(int));
    for (int q = 0; q < B && bad < 0; ++q) {
      double cw[6] = {e[q], c[q], e[(size_t)B + q], b[(size_t)(n - 2) * B + q],
                      a[(size_t)(n - 1) * B + q], b[(size_t)(n - 1) * B + q]};
      double* Kq = K + (size_t)q * 16;
      for (int k = 0; k < 4; ++k) {
        double w0 = Wk[k][q], w1 = Wk[k][(size_t)B + q], wn2 = Wk[k][(size_t)(n - 2) * B + q],
               wn1 = Wk[k][(size_t)(n - 1) * B + q];
        Kq[0 * 4 + k] = cw[0] * wn2 + cw[1] * wn1;
        Kq[1 * 4 + k] = cw[2] * wn1;
        Kq[2 * 4 + k] = cw[3] * w0;
        Kq[3 * 4 + k] = cw[4] * w0 + cw[5] * w1;
      }
      for (int r = 0; r < 4; ++r) Kq[r * 4 + r] += 1.0;
      if (orc_lu4_factor(Kq, piv + (size_t)q * 4) != 0) bad = q;
    }
    if (bad < 0) {
      orc_penta_substitute(B, n, m1, m2, dInv, ap, bp, rhs);
      double* ys = malloc((size_t)B * 4 * 8);
      for (int q = 0; q < B; ++q) {
        double z0 = rhs[q], z1 = rhs[(size_t)B + q], zn2 = rhs[(size_t)(n - 2) * B + q],
               zn1 = rhs[(size_t)(n - 1) * B + q];
        double cw[6] = {e[q], c[q], e[(size_t)B + q], b[(size_t)(n - 2) * B + q],
                        a[(size_t)(n - 1) * B + q], b[(size_t)(n - 1) * B + q]};
        double* y = ys + (size_t)q * 4;
        y[0] = cw[0] * zn2 + cw[1] * zn1;
        y[1] = cw[2] * zn1;
        y[2] = cw[3] * z0;
        y[3] = cw[4] * z0 + cw[5] * z1;
        orc_lu4_solve(K + (size_t)q * 16, piv + (size_t)q * 4, y);
      }
      for (int r = 0; r < n; ++r) {
        size_t cur = (size_t)r * B;
        for (int q = 0; q < B; ++q) {
          const double* y = ys + (size_t)q * 4;
          rhs[cur + q] -= Wk[0][cur + q] * y[0] + Wk[1][cur + q] * y[1] + Wk[2][cur + q] * y[2] +
                          Wk[3][cur + q] * y[3];
        }
      }
      free(ys);
    }
    for (int k = 0; k < 4; ++k) free(Wk[k]);
    free(K);
    free(piv);
  }
done:
  free(m1);
  free(m2);
  free(dInv);
  free(ap);
  free(bp);
  return bad;
}

/* build_hyperdiffusion_operator: penta.cpp:313-335. */
void orc_hyperdiffusion_operator(double sigma, int n, int B, int periodic, double* e, double* c,
                                 double* d, double* a, double* b) {
  const size_t len = (size_t)B * (size_t)n;
  const double second = sigma, first = -4.0 * sigma, center = 1.0 + 6.0 * sigma;
  for (size_t k = 0; k < len; ++k) {
    e[k] = second;
    c[k] = first;
    d[k] = center;
    a[k] = first;
    b[k] = second;
  }
  if (!periodic)
    for (int q = 0; q < B; ++q) {
      e[q] = 0.0;
      e[(size_t)B + q] = 0.0;
      c[q] = 0.0;
      a[(size_t)(n - 1) * B + q] = 0.0;
      b[(size_t)(n - 2) * B + q] = 0.0;
      b[(size_t)(n - 1) * B + q] = 0.0;
    }
}

/* --------------------------------------------------------- Cahn-Hilliard */

static const double kTwoThirds = 2.0 / 3.0; /* cahn_hilliard.cpp:12 */

static double pow4(double h) { /* cahn_hilliard.cpp:14-17 */
  double h2 = h * h;
  return h2 * h2;
}

/* SplitMix64 (cahn_hilliard.hpp:47-63) + initial_condition (.cpp:68-76). */
void orc_ch_initial_condition(uint64_t seed, double amp, long long count, double* out) {
  uint64_t state = seed;
  for (long long k = 0; k < count; ++k) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    double u = (double)(z >> 11) * 0x1.0p-53;
    out[k] = amp * (2.0 * u - 1.0);
  }
}

/* biharmonic_weights (cahn_hilliard.cpp:85-114) and
 * nonlinear_laplacian_coefficients (:78-83). */
void orc_ch_weights(double dx, double dy, double* w, double* nl) {
  const double ax = 1.0 / pow4(dx), ay = 1.0 / pow4(dy);
  const double cr = 2.0 / ((dx * dx) * (dy * dy));
  static const double cross[9] = {1.0, -2.0, 1.0, -2.0, 4.0, -2.0, 1.0, -2.0, 1.0};
  for (int k = 0; k < 25; ++k) w[k] = 0.0;
#define AT(p, q) w[(q) * 5 + (p)]
  AT(0, 2) += ax;
  AT(1, 2) += -4.0 * ax;
  AT(2, 2) += 6.0 * ax;
  AT(3, 2) += -4.0 * ax;
  AT(4, 2) += ax;
  AT(2, 0) += ay;
  AT(2, 1) += -4.0 * ay;
  AT(2, 2) += 6.0 * ay;
  AT(2, 3) += -4.0 * ay;
  AT(2, 4) += ay;
  for (int q = 0; q < 3; ++q)
    for (int p = 0; p < 3; ++p) AT(p + 1, q + 1) += cross[q * 3 + p] * cr;
  double prefix = 0.0;
  for (int k = 0; k < 22; ++k) prefix += w[k];
  AT(2, 4) = -prefix;
#undef AT
  const double cx = 1.0 / (dx * dx), cy = 1.0 / (dy * dy), cc = -2.0 * cx - 2.0 * cy;
  const double n9[9] = {0.0, cy, 0.0, cx, cc, cx, 0.0, cy, 0.0};
  memcpy(nl, n9, sizeof n9);
}

/* Periodic uniform-operator factor for one system (B = 1), the quantity every
 * CH sweep system shares (SURVEY.md §8(a) key fact (i)). */
typedef struct {
  int n;
  double *m1, *m2, *dInv, *ap, *bp, *W[4];
  double K[16];
  int piv[4];
  double cw[6];
} orc_uniform_factor;

static int uniform_factor_build(double sigma, int n, orc_uniform_factor* f) {
  double *e = malloc(n * 8), *c = malloc(n * 8), *d = malloc(n * 8), *a = malloc(n * 8),
         *b = malloc(n * 8);
  orc_hyperdiffusion_operator(sigma, n, 1, 1, e, c, d, a, b);
  f->n = n;
  f->m1 = malloc(n * 8);
  f->m2 = malloc(n * 8);
  f->dInv = malloc(n * 8);
  f->ap = malloc(n * 8);
  f->bp = malloc(n * 8);
  int bad = orc_penta_factor(1, n, e, c, d, a, b, f->m1, f->m2, f->dInv, f->ap, f->bp);
  const int rowOf[4] = {0, 1, n - 2, n - 1};
  for (int k = 0; k < 4; ++k) {
    f->W[k] = calloc(n, 8);
    f->W[k][rowOf[k]] = 1.0;
    if (bad < 0) orc_penta_substitute(1, n, f->m1, f->m2, f->dInv, f->ap, f->bp, f->W[k]);
  }
  double cw[6] = {e[0], c[0], e[1], b[n - 2], a[n - 1], b[n - 1]};
  memcpy(f->cw, cw, sizeof cw);
  for (int k = 0; k < 4; ++k) {
    const double* W = f->W[k];
    f->K[0 * 4 + k] = cw[0] * W[n - 2] + cw[1] * W[n - 1];
    f->K[1 * 4 + k] = cw[2] * W[n - 1];
    f->K[2 * 4 + k] = cw[3] * W[0];
    f->K[3 * 4 + k] = cw[4] * W[0] + cw[5] * W[1];
  }
  for (int r = 0; r < 4; ++r) f->K[r * 4 + r] += 1.0;
  if (bad < 0 && orc_lu4_factor(f->K, f->piv) != 0) bad = 0;
  free(e);
  free(c);
  free(d);
  free(a);
  free(b);
  return bad;
}

static void uniform_factor_free(orc_uniform_factor* f) {
  free(f->m1);
  free(f->m2);
  free(f->dInv);
  free(f->ap);
  free(f->bp);
  for (int k = 0; k < 4; ++k) free(f->W[k]);
}

/* Solve one periodic system stored with stride `s` (solve_range +
 * correct_range restricted to one system, penta.cpp:160-197, 253-287). */
static void uniform_solve_strided(const orc_uniform_factor* f, double* y, long long s) {
  const int n = f->n;
  y[s] -= f->m2[1] * y[0];
  for (int r = 2; r < n; ++r) y[r * s] -= f->m1[r] * y[(r - 2) * s] + f->m2[r] * y[(r - 1) * s];
  y[(n - 1) * s] *= f->dInv[n - 1];
  y[(n - 2) * s] = (y[(n - 2) * s] - f->ap[n - 2] * y[(n - 1) * s]) * f->dInv[n - 2];
  for (int r = n - 3; r >= 0; --r)
    y[r * s] = (y[r * s] - f->ap[r] * y[(r + 1) * s] - f->bp[r] * y[(r + 2) * s]) * f->dInv[r];
  double c4[4];
  const double z0 = y[0], z1 = y[s], zn2 = y[(n - 2) * s], zn1 = y[(n - 1) * s];
  c4[0] = f->cw[0] * zn2 + f->cw[1] * zn1;
  c4[1] = f->cw[2] * zn1;
  c4[2] = f->cw[3] * z0;
  c4[3] = f->cw[4] * z0 + f->cw[5] * z1;
  orc_lu4_solve(f->K, f->piv, c4);
  for (int r = 0; r < n; ++r)
    y[r * s] -= f->W[0][r] * c4[0] + f->W[1][r] * c4[1] + f->W[2][r] * c4[2] + f->W[3][r] * c4[3];
}

/* CHStepper (cahn_hilliard.cpp:213-328): `steps` BDF2-ADI steps from
 * (curr, prev); both arrays are updated in place to (C^{n+steps},
 * C^{n+steps-1}). dp = {D, gamma, lx, ly, dt}; ip = {nx, ny, nonlinear}. */
int orc_ch_run(const double* dp, const int* ip, int steps, double* curr, double* prev) {
  const double D = dp[0], gamma = dp[1], lx = dp[2], ly = dp[3], dt = dp[4];
  const int nx = ip[0], ny = ip[1], nonlinear = ip[2];
  const double dx = lx / nx, dy = ly / ny;
  const size_t cnt = (size_t)nx * (size_t)ny;
  const double kDiff = -kTwoThirds, kBih = kTwoThirds * D * gamma * dt, kNl = kTwoThirds * D * dt;
  const double sx = kTwoThirds * D * gamma * dt / pow4(dx);
  const double sy = kTwoThirds * D * gamma * dt / pow4(dy);
  orc_uniform_factor fx, fy;
  int bad = uniform_factor_build(sx, nx, &fx);
  if (bad < 0) bad = uniform_factor_build(sy, ny, &fy);
  else uniform_factor_build(sy, ny, &fy);
  if (bad >= 0) {
    uniform_factor_free(&fx);
    uniform_factor_free(&fy);
    return bad;
  }
  double bw[25], nlc[9];
  orc_ch_weights(dx, dy, bw, nlc);
  const int ext1[4] = {1, 1, 1, 1}, ext2[4] = {2, 2, 2, 2};
  double *cb = malloc(cnt * 8), *nl = malloc(cnt * 8), *bh = malloc(cnt * 8), *w = malloc(cnt * 8);
  for (int s = 0; s < steps; ++s) {
    for (size_t i = 0; i < cnt; ++i) cb[i] = 2.0 * curr[i] - prev[i];
    if (nonlinear) orc_stencil(1, ext1, 1, nlc, curr, nl, nx, ny);
    orc_stencil(1, ext2, 0, bw, cb, bh, nx, ny);
    if (nonlinear)
      for (size_t i = 0; i < cnt; ++i) w[i] = kDiff * (curr[i] - prev[i]) - kBih * bh[i] + kNl * nl[i];
    else
      for (size_t i = 0; i < cnt; ++i) w[i] = kDiff * (curr[i] - prev[i]) - kBih * bh[i];
    /* Lx sweep: system j = row j, unknowns along x (stride 1). */
    for (int j = 0; j < ny; ++j) uniform_solve_strided(&fx, w + (size_t)j * nx, 1);
    /* Ly sweep: system i = column i, unknowns along y (stride nx). */
    for (int i = 0; i < nx; ++i) uniform_solve_strided(&fy, w + i, nx);
    /* C^{n+1} = Cbar + v; rotate (cahn_hilliard.cpp:311-324). */
    for (size_t i = 0; i < cnt; ++i) {
      double next = cb[i] + w[i];
      prev[i] = curr[i];
      curr[i] = next;
    }
  }
  free(cb);
  free(nl);
  free(bh);
  free(w);
  uniform_factor_free(&fx);
  uniform_factor_free(&fy);
  return -1;
}

/* Export the uniform factor of one periodic hyperdiffusion system, for
 * checking the device factor tables. out arrays of n doubles; K16/piv4/cw6. */
int orc_uniform_factor_tables(double sigma, int n, double* m1, double* m2, double* dInv, double* ap,
                              double* bp, double* W4n, double* K16, int* piv4, double* cw6) {
  orc_uniform_factor f;
  int bad = uniform_factor_build(sigma, n, &f);
  memcpy(m1, f.m1, n * 8);
  memcpy(m2, f.m2, n * 8);
  memcpy(dInv, f.dInv, n * 8);
  memcpy(ap, f.ap, n * 8);
  memcpy(bp, f.bp, n * 8);
  for (int k = 0; k < 4; ++k) memcpy(W4n + (size_t)k * n, f.W[k], n * 8);
  memcpy(K16, f.K, sizeof f.K);
  memcpy(piv4, f.piv, sizeof f.piv);
  memcpy(cw6, f.cw, sizeof f.cw);
  uniform_factor_free(&f);
  return bad;
}
