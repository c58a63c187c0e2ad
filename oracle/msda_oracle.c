/*
 * TEST INFRASTRUCTURE ONLY — C restatement of the reference MSDA oracle.
 *
 * Restates mvtrack3d.features.msda_reference (features.py:241-276) with the
 * bilinear tree of features.py:184-219, and the PACKED_HALF arithmetic of
 * msda_optimized (features.py:306-416), bit for bit.  It is the fast checker
 * the GPU parity tests use at full BASELINE sizes and the CPU baseline that
 * bench.py times (kind "port").  The product never links it.
 *
 * Build (see oracle/build.py):  gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared
 * -ffp-contract=off keeps every multiply and add separately rounded, which
 * is what numpy does.
 *
 * Layout: table[R][C] (f32), per tile t = cam*n_levels + level:
 * tile_start[t], tile_h[t], tile_w[t]; CSR plan offsets[Q+1], cam/lvl/u/v/w[S].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORC_OK = 0, ORC_BAD_TARGET = 3, ORC_ZERO_WEIGHT_SUM = 4, ORC_BAD_ARG = 8 };

typedef struct {
  const int32_t *cam, *lvl;
  const float *u, *v, *w;
} plan_view;

/* numpy.lexsort((w, u, v, lvl, cam)) — float keys compare with <, so -0 == +0;
 * ties are equal samples, whose visiting order cannot change any bit. */
static const plan_view *g_pv;
static int cmp_canonical(const void *pa, const void *pb) {
  int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
  const plan_view *p = g_pv;
  if (p->cam[a] != p->cam[b]) return p->cam[a] < p->cam[b] ? -1 : 1;
  if (p->lvl[a] != p->lvl[b]) return p->lvl[a] < p->lvl[b] ? -1 : 1;
  if (p->v[a] != p->v[b]) return p->v[a] < p->v[b] ? -1 : 1;
  if (p->u[a] != p->u[b]) return p->u[a] < p->u[b] ? -1 : 1;
  if (p->w[a] != p->w[b]) return p->w[a] < p->w[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* insertion sort with the same comparator (thread-safe, no global state) */
static int less_canon(const plan_view *p, int64_t a, int64_t b) {
  if (p->cam[a] != p->cam[b]) return p->cam[a] < p->cam[b];
  if (p->lvl[a] != p->lvl[b]) return p->lvl[a] < p->lvl[b];
  if (p->v[a] != p->v[b]) return p->v[a] < p->v[b];
  if (p->u[a] != p->u[b]) return p->u[a] < p->u[b];
  if (p->w[a] != p->w[b]) return p->w[a] < p->w[b];
  return a < b;
}

static void merge_sort(const plan_view *p, int64_t *idx, int64_t *tmp, int64_t n) {
  if (n < 24) {
    for (int64_t i = 1; i < n; ++i) {
      int64_t x = idx[i], j = i - 1;
      while (j >= 0 && less_canon(p, x, idx[j])) { idx[j + 1] = idx[j]; --j; }
      idx[j + 1] = x;
    }
    return;
  }
  int64_t h = n / 2;
  merge_sort(p, idx, tmp, h);
  merge_sort(p, idx + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = less_canon(p, idx[j], idx[i]) ? idx[j++] : idx[i++];
  while (i < h) tmp[k++] = idx[i++];
  while (j < n) tmp[k++] = idx[j++];
  memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
}

/* ---- IEEE binary16 helpers (round to nearest even), used for PACKED_HALF --- */
static uint16_t f32_to_f16(float f) {
  uint32_t x; memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) return (uint16_t)(sign | (ax > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* rounds to inf */
  if (ax < 0x38800000u) {                                   /* subnormal or zero in f16 */
    if (ax < 0x33000000u) return (uint16_t)sign;            /* < 2^-25 → 0 (ties at 2^-25 go even=0) */
    /* value = m * 2^(e-150); in units of 2^-24 that is m >> (126 - e) */
    uint32_t e = ax >> 23, m = (ax & 0x7fffffu) | 0x800000u;
    uint32_t shift = 126 - e;
    uint32_t r = m >> shift, rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (r & 1u))) ++r;
    return (uint16_t)(sign | r);
  }
  uint32_t r = ((ax - 0x38000000u) >> 13);
  uint32_t rem = ax & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (r & 1u))) ++r;
  return (uint16_t)(sign | r);
}

static float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16, e = (h >> 10) & 0x1f, m = h & 0x3ffu, x;
  if (e == 0) {
    if (m == 0) x = sign;
    else { float f = ldexpf((float)m, -24); memcpy(&x, &f, 4); x |= sign; }
  } else if (e == 31) x = sign | 0x7f800000u | (m << 13);
  else x = sign | ((e + 112) << 23) | (m << 13);
  float f; memcpy(&f, &x, 4); return f;
}

/* correctly rounded f16 ops: exact-enough in f32 (p=24 >= 2*11+2), then RNE */
static uint16_t h_mul(uint16_t a, uint16_t b) { return f32_to_f16(f16_to_f32(a) * f16_to_f32(b)); }
static uint16_t h_add(uint16_t a, uint16_t b) { return f32_to_f16(f16_to_f32(a) + f16_to_f32(b)); }

float oracle_f16_roundtrip(float x) { return f16_to_f32(f32_to_f16(x)); }

/* ---------------------------------------------------------------------- */
int oracle_msda(const float *table, int32_t C, int32_t n_cams, int32_t n_levels,
                const int64_t *tile_start, const int32_t *tile_h, const int32_t *tile_w,
                int64_t Q, const int64_t *offsets, const int32_t *cam, const int32_t *lvl,
                const float *u, const float *v, const float *w, int32_t normalize, int32_t half_mode,
                float *out, uint8_t *empty, int32_t n_threads) {
  if (C <= 0 || n_cams < 0 || n_levels <= 0) return ORC_BAD_ARG;
  int64_t S = offsets[Q];
  for (int64_t s = 0; s < S; ++s)
    if (cam[s] < 0 || cam[s] >= n_cams || lvl[s] < 0 || lvl[s] >= n_levels) return ORC_BAD_TARGET;
  plan_view pv = {cam, lvl, u, v, w};
  int status = ORC_OK;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel
  {
    int64_t cap = 0;
    int64_t *idx = NULL, *tmp = NULL;
    float *acc = (float *)malloc(sizeof(float) * (size_t)C);
    float *vec = (float *)malloc(sizeof(float) * (size_t)C);
    uint16_t *hacc = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)C);
#pragma omp for schedule(dynamic, 4)
    for (int64_t q = 0; q < Q; ++q) {
      int64_t lo = offsets[q], hi = offsets[q + 1], n = hi - lo;
      float *oq = out + q * (int64_t)C;
      empty[q] = (uint8_t)(n == 0);
      for (int32_t c = 0; c < C; ++c) oq[c] = 0.0f;
      if (n == 0) continue;
      if (n > cap) {
        cap = n;
        idx = (int64_t *)realloc(idx, sizeof(int64_t) * (size_t)cap);
        tmp = (int64_t *)realloc(tmp, sizeof(int64_t) * (size_t)cap);
      }
      for (int64_t i = 0; i < n; ++i) idx[i] = lo + i;
      merge_sort(&pv, idx, tmp, n);
      float wsum = 0.0f;
      if (normalize) {
        for (int64_t i = 0; i < n; ++i) wsum = wsum + w[idx[i]];
        if (wsum == 0.0f) {
#pragma omp atomic write
          status = ORC_ZERO_WEIGHT_SUM;
          continue;
        }
      }
      for (int32_t c = 0; c < C; ++c) { acc[c] = 0.0f; hacc[c] = 0; }
      for (int64_t i = 0; i < n; ++i) {
        int64_t s = idx[i];
        int64_t t = (int64_t)cam[s] * n_levels + lvl[s];
        int64_t st = tile_start[t];
        int32_t H = tile_h[t], W = tile_w[t];
        float uu = u[s], vv = v[s];
        float x0f = floorf(uu), y0f = floorf(vv);
        float fu = uu - x0f, fv = vv - y0f;
        float omu = 1.0f - fu, omv = 1.0f - fv;
        float iw[4] = {omu * omv, fu * omv, omu * fv, fu * fv};
        int in_x0 = (x0f >= 0.0f) && (x0f <= (float)(W - 1));
        int in_x1 = (x0f >= -1.0f) && (x0f <= (float)(W - 2));
        int in_y0 = (y0f >= 0.0f) && (y0f <= (float)(H - 1));
        int in_y1 = (y0f >= -1.0f) && (y0f <= (float)(H - 2));
        const float *cp[4] = {NULL, NULL, NULL, NULL};
        if (in_x0 && in_y0) cp[0] = table + (st + (int64_t)y0f * W + (int64_t)x0f) * C;
        if (in_x1 && in_y0) cp[1] = table + (st + (int64_t)y0f * W + (int64_t)x0f + 1) * C;
        if (in_x0 && in_y1) cp[2] = table + (st + ((int64_t)y0f + 1) * W + (int64_t)x0f) * C;
        if (in_x1 && in_y1) cp[3] = table + (st + ((int64_t)y0f + 1) * W + (int64_t)x0f + 1) * C;
        float ws = normalize ? w[s] / wsum : w[s];
        if (!half_mode) {
          for (int32_t c = 0; c < C; ++c) {
            float a = (cp[0] ? cp[0][c] : 0.0f) * iw[0];
            float b = (cp[1] ? cp[1][c] : 0.0f) * iw[1];
            float d = (cp[2] ? cp[2][c] : 0.0f) * iw[2];
            float e = (cp[3] ? cp[3][c] : 0.0f) * iw[3];
            vec[c] = (a + b) + (d + e);
            acc[c] = acc[c] + ws * vec[c];
          }
        } else {
          uint16_t hw[4] = {f32_to_f16(iw[0]), f32_to_f16(iw[1]), f32_to_f16(iw[2]), f32_to_f16(iw[3])};
          uint16_t hs = f32_to_f16(ws);
          for (int32_t c = 0; c < C; ++c) {
            uint16_t a = h_mul(cp[0] ? f32_to_f16(cp[0][c]) : 0, hw[0]);
            uint16_t b = h_mul(cp[1] ? f32_to_f16(cp[1][c]) : 0, hw[1]);
            uint16_t d = h_mul(cp[2] ? f32_to_f16(cp[2][c]) : 0, hw[2]);
            uint16_t e = h_mul(cp[3] ? f32_to_f16(cp[3][c]) : 0, hw[3]);
            uint16_t t0 = h_add(h_add(a, b), h_add(d, e));
            hacc[c] = h_add(hacc[c], h_mul(t0, hs));
          }
        }
      }
      if (!half_mode) for (int32_t c = 0; c < C; ++c) oq[c] = acc[c];
      else for (int32_t c = 0; c < C; ++c) oq[c] = f16_to_f32(hacc[c]);
    }
    free(idx); free(tmp); free(acc); free(vec); free(hacc);
  }
  (void)cmp_canonical;
  (void)g_pv;
  return status;
}
