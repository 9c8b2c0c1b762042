/* Deterministic config generators -- see lrs_gen.h for the definitions. */
#include "lrs_gen.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "lrs_rng.h"

static int alloc_csr(lrs_gen_csr* m, int64_t n, int64_t cap) {
  m->n = n;
  m->nnz = 0;
  m->row_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  m->col_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  m->values = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  if (!m->row_ptr || !m->col_idx || !m->values) {
    lrs_gen_free(m);
    return -1;
  }
  m->row_ptr[0] = 0;
  return 0;
}

void lrs_gen_free(lrs_gen_csr* m) {
  if (!m) return;
  free(m->row_ptr);
  free(m->col_idx);
  free(m->values);
  m->row_ptr = NULL;
  m->col_idx = NULL;
  m->values = NULL;
  m->n = m->nnz = 0;
}

int lrs_gen_poisson2d(int64_t g, double shift, lrs_gen_csr* out) {
  const int64_t n = g * g;
  if (g < 1 || alloc_csr(out, n, 5 * n)) return -1;
  int64_t p = 0;
  for (int64_t y = 0; y < g; ++y) {
    for (int64_t x = 0; x < g; ++x) {
      const int64_t i = y * g + x;
      /* ascending column order: y-1, x-1, self, x+1, y+1 */
      if (y > 0) { out->col_idx[p] = i - g; out->values[p++] = -1.0; }
      if (x > 0) { out->col_idx[p] = i - 1; out->values[p++] = -1.0; }
      out->col_idx[p] = i; out->values[p++] = 4.0 + shift;
      if (x < g - 1) { out->col_idx[p] = i + 1; out->values[p++] = -1.0; }
      if (y < g - 1) { out->col_idx[p] = i + g; out->values[p++] = -1.0; }
      out->row_ptr[i + 1] = p;
    }
  }
  out->nnz = p;
  return 0;
}

int lrs_gen_convdiff3d(int64_t g, double conv, lrs_gen_csr* out) {
  const int64_t n = g * g * g, g2 = g * g;
  if (g < 1 || alloc_csr(out, n, 7 * n)) return -1;
  const double h = 1.0 / (double)(g + 1);
  const double beta = conv * h / 2.0;
  int64_t p = 0;
  for (int64_t z = 0; z < g; ++z)
    for (int64_t y = 0; y < g; ++y)
      for (int64_t x = 0; x < g; ++x) {
        const int64_t i = (z * g + y) * g + x;
        if (z > 0) { out->col_idx[p] = i - g2; out->values[p++] = -1.0; }
        if (y > 0) { out->col_idx[p] = i - g; out->values[p++] = -1.0; }
        if (x > 0) { out->col_idx[p] = i - 1; out->values[p++] = -1.0 - beta; }
        out->col_idx[p] = i; out->values[p++] = 6.0;
        if (x < g - 1) { out->col_idx[p] = i + 1; out->values[p++] = -1.0 + beta; }
        if (y < g - 1) { out->col_idx[p] = i + g; out->values[p++] = -1.0; }
        if (z < g - 1) { out->col_idx[p] = i + g2; out->values[p++] = -1.0; }
        out->row_ptr[i + 1] = p;
      }
  out->nnz = p;
  return 0;
}

int lrs_gen_hetero27(int64_t g, uint64_t seed, double log10_range, lrs_gen_csr* out) {
  const int64_t n = g * g * g;
  if (g < 1 || alloc_csr(out, n, 27 * n)) return -1;
  double* kappa = (double*)malloc(sizeof(double) * (size_t)n);
  if (!kappa) { lrs_gen_free(out); return -1; }
  const uint64_t key = lrs_rng_key(seed, LRS_STREAM_MATRIX);
  for (int64_t c = 0; c < n; ++c)
    kappa[c] = pow(10.0, log10_range * lrs_rng_sym(key, (uint64_t)c));
  int64_t p = 0;
  for (int64_t z = 0; z < g; ++z)
    for (int64_t y = 0; y < g; ++y)
      for (int64_t x = 0; x < g; ++x) {
        const int64_t i = (z * g + y) * g + x;
        const double kp = kappa[i];
        double offsum = 0.0;
        int missing = 0;
        int64_t diag_pos = -1;
        /* dz, dy, dx in ascending order gives ascending column index */
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              if (dz == 0 && dy == 0 && dx == 0) {
                diag_pos = p;
                out->col_idx[p] = i;
                out->values[p++] = 0.0; /* filled below */
                continue;
              }
              const int64_t zz = z + dz, yy = y + dy, xx = x + dx;
              if (zz < 0 || zz >= g || yy < 0 || yy >= g || xx < 0 || xx >= g) {
                ++missing;
                continue;
              }
              const int64_t j = (zz * g + yy) * g + xx;
              const double kq = kappa[j];
              const double w = 2.0 * kp * kq / (kp + kq);
              out->col_idx[p] = j;
              out->values[p++] = -w;
              offsum += w;
            }
        out->values[diag_pos] = offsum + kp * (double)missing;
        out->row_ptr[i + 1] = p;
      }
  out->nnz = p;
  free(kappa);
  return 0;
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int lrs_gen_randband(int64_t n, int64_t b, int64_t m, uint64_t seed, double dom,
                     lrs_gen_csr* out) {
  if (n < 1 || b < 0 || m < 0 || alloc_csr(out, n, (m + 1) * n)) return -1;
  const uint64_t kpat = lrs_rng_key(seed, LRS_STREAM_PATTERN);
  const uint64_t kval = lrs_rng_key(seed, LRS_STREAM_MATRIX);
  int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
  if (!cols) { lrs_gen_free(out); return -1; }
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = i - b < 0 ? 0 : i - b;
    const int64_t hi = i + b > n - 1 ? n - 1 : i + b;
    const int64_t ncand = hi - lo; /* excludes the diagonal */
    int64_t take = m < ncand ? m : ncand;
    int64_t cnt = 0;
    uint64_t ctr = (uint64_t)i << 20;
    if (take == ncand) {
      for (int64_t j = lo; j <= hi; ++j)
        if (j != i) cols[cnt++] = j;
    } else {
      while (cnt < take) {
        /* draw from [lo, hi] \ {i}: index into the candidate list */
        int64_t r = (int64_t)lrs_rng_below(kpat, ctr++, (uint64_t)ncand);
        int64_t j = lo + r;
        if (j >= i) ++j;
        int dup = 0;
        for (int64_t q = 0; q < cnt; ++q)
          if (cols[q] == j) { dup = 1; break; }
        if (!dup) cols[cnt++] = j;
      }
    }
    qsort(cols, (size_t)cnt, sizeof(int64_t), cmp_i64);
    double offsum = 0.0;
    int64_t row_start = p;
    int placed_diag = 0;
    for (int64_t q = 0; q < cnt; ++q) {
      if (!placed_diag && cols[q] > i) {
        out->col_idx[p] = i;
        out->values[p++] = 0.0;
        placed_diag = 1;
      }
      const double v = lrs_rng_normal(kval, (uint64_t)i * (uint64_t)(m + 1) + (uint64_t)q);
      out->col_idx[p] = cols[q];
      out->values[p++] = v;
      offsum += fabs(v);
    }
    if (!placed_diag) {
      out->col_idx[p] = i;
      out->values[p++] = 0.0;
    }
    for (int64_t q = row_start; q < p; ++q)
      if (out->col_idx[q] == i) out->values[q] = dom * offsum;
    out->row_ptr[i + 1] = p;
  }
  out->nnz = p;
  free(cols);
  return 0;
}

/* (row, col, value) triplet sort for the symmetric perturbation. */
typedef struct { int64_t r, c; double v; } trip;

static int cmp_trip(const void* a, const void* b) {
  const trip* x = (const trip*)a;
  const trip* y = (const trip*)b;
  if (x->r != y->r) return (x->r > y->r) - (x->r < y->r);
  return (x->c > y->c) - (x->c < y->c);
}

int lrs_gen_feast_base(int64_t g, uint64_t seed, int64_t pb, double sigma, lrs_gen_csr* out) {
  const int64_t n = g * g * g, g2 = g * g;
  if (g < 1) return -1;
  const int64_t cap = 9 * n;
  trip* t = (trip*)malloc(sizeof(trip) * (size_t)cap);
  if (!t) return -1;
  int64_t nt = 0;
  for (int64_t z = 0; z < g; ++z)
    for (int64_t y = 0; y < g; ++y)
      for (int64_t x = 0; x < g; ++x) {
        const int64_t i = (z * g + y) * g + x;
        t[nt++] = (trip){i, i, 6.0};
        if (z > 0) t[nt++] = (trip){i, i - g2, -1.0};
        if (y > 0) t[nt++] = (trip){i, i - g, -1.0};
        if (x > 0) t[nt++] = (trip){i, i - 1, -1.0};
        if (x < g - 1) t[nt++] = (trip){i, i + 1, -1.0};
        if (y < g - 1) t[nt++] = (trip){i, i + g, -1.0};
        if (z < g - 1) t[nt++] = (trip){i, i + g2, -1.0};
      }
  const uint64_t kpat = lrs_rng_key(seed, LRS_STREAM_PATTERN);
  const uint64_t kval = lrs_rng_key(seed, LRS_STREAM_MATRIX);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = i - pb < 0 ? 0 : i - pb;
    const int64_t hi = i + pb > n - 1 ? n - 1 : i + pb;
    const int64_t ncand = hi - lo;
    if (ncand <= 0) continue;
    int64_t j = lo + (int64_t)lrs_rng_below(kpat, (uint64_t)i, (uint64_t)ncand);
    if (j >= i) ++j;
    const double v = sigma * lrs_rng_normal(kval, (uint64_t)i);
    t[nt++] = (trip){i, j, v};
    t[nt++] = (trip){j, i, v};
  }
  qsort(t, (size_t)nt, sizeof(trip), cmp_trip);
  if (alloc_csr(out, n, nt)) { free(t); return -1; }
  int64_t p = 0;
  for (int64_t q = 0; q < nt; ++q) {
    if (p > 0 && q > 0 && t[q].r == t[q - 1].r && t[q].c == t[q - 1].c) {
      out->values[p - 1] += t[q].v; /* sum duplicates (documented contract) */
      continue;
    }
    out->col_idx[p] = t[q].c;
    out->values[p] = t[q].v;
    ++p;
    out->row_ptr[t[q].r + 1] = p;
  }
  /* rows are never empty (diagonal), but make row_ptr monotone anyway */
  for (int64_t i = 1; i <= n; ++i)
    if (out->row_ptr[i] < out->row_ptr[i - 1]) out->row_ptr[i] = out->row_ptr[i - 1];
  out->nnz = p;
  free(t);
  return 0;
}

void lrs_gen_vector(int kind, uint64_t seed, int64_t count, double* out) {
  const uint64_t key = lrs_rng_key(seed, LRS_STREAM_RHS);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) out[i] = lrs_rng_sym(key, (uint64_t)i);
    else if (kind == 1) out[i] = lrs_rng_normal(key, (uint64_t)i);
    else out[i] = 1.0;
  }
}

void lrs_gen_omega(uint64_t seed, int64_t partition, int side, int64_t rows, int64_t cols,
                   double* out) {
  const uint64_t key =
      lrs_rng_key(seed, LRS_STREAM_OMEGA + 2ull * (uint64_t)partition + (uint64_t)side);
  const int64_t total = rows * cols;
  for (int64_t i = 0; i < total; ++i) out[i] = lrs_rng_normal(key, (uint64_t)i);
}
