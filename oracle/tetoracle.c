/*
 * tetoracle.c -- CPU restatement of the reference traversal.
 *
 * TEST INFRASTRUCTURE ONLY (see tetoracle.h): the checker for the sm_100a
 * kernels and the "port" CPU baseline.  Restates, with citations:
 *   - scaled basis / projection / Alg. 1 exit face   _kernels.pyx:42-102
 *   - ray initialisation                             _kernels.pyx:114-192
 *   - next reference per layout (Alg. 3/5/7)         _kernels.pyx:195-235
 *   - step                                           _kernels.pyx:238-259
 *   - batch cast loop + cycle guard                  _kernels.pyx:343-369
 *   - batch epilogue (triangle, fp64 t, back tet)    batch.py:57-71, _kernels_py.py:435-454
 *   - point location (fp64 containment)              _kernels.pyx:373-492
 *   - shadow walks (segment/triangle t)              _kernels.pyx:495-614
 *   - ScTP exit predicate                            traversal.py:484-511
 * Build: gcc -O3 -ffp-contract=off (no FMA contraction, SSE fp32/fp64).
 */
#include "tetoracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define REF_CONSTRAINED 0x80000000u
#define REF_PAYLOAD 0x7FFFFFFFu
#define REF_BOUNDARY 0x7FFFFFFFu

/* Faces opposite each sorted slot (_kernels.pyx:105-111). */
static const int FACE_OF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

typedef struct {
  int mn, mx, ot;
  float umax, vmax, voth, sgn, pox, poy;
} frame_t;

/* ---- basis, _kernels.pyx:42-86 -------------------------------------------- */
static void frame_setup(const float o[3], const float d[3], frame_t* f) {
  float a[3] = {fabsf(d[0]), fabsf(d[1]), fabsf(d[2])};
  int mn;
  if (a[1] < a[0])
    mn = (a[2] < a[1]) ? 2 : 1;
  else
    mn = (a[2] < a[0]) ? 2 : 0;
  /* the two remaining axes in increasing order; ties keep the lower one */
  int lo = (mn == 0) ? 1 : 0;
  int hi = (mn == 2) ? 1 : 2;
  int mx = (a[lo] >= a[hi]) ? lo : hi;
  int ot = 3 - mn - mx;
  f->mn = mn;
  f->mx = mx;
  f->ot = ot;
  f->umax = -(d[ot] / d[mx]);
  float u[3] = {0.0f, 0.0f, 0.0f};
  u[ot] = 1.0f;
  u[mx] = f->umax;
  float w[3];
  w[0] = d[1] * u[2] - d[2] * u[1];
  w[1] = d[2] * u[0] - d[0] * u[2];
  w[2] = d[0] * u[1] - d[1] * u[0];
  float wmn = w[mn];
  f->sgn = (wmn > 0) ? 1.0f : -1.0f;
  float wabs = (wmn > 0) ? wmn : -wmn;
  f->vmax = w[mx] / wabs;
  f->voth = w[ot] / wabs;
  f->pox = f->umax * o[mx] + o[ot];
  f->poy = (f->vmax * o[mx] + f->voth * o[ot]) + f->sgn * o[mn];
}

/* ---- projection, _kernels.pyx:89-91 ---------------------------------------- */
static inline void frame_project(const frame_t* f, const float* q, float* x, float* y) {
  *x = (f->umax * q[f->mx] + q[f->ot]) - f->pox;
  *y = ((f->vmax * q[f->mx] + f->voth * q[f->ot]) + f->sgn * q[f->mn]) - f->poy;
}

/* ---- Algorithm 1, _kernels.pyx:94-102 -------------------------------------- */
static inline int alg1_exit(float px, float py, const float w[6]) {
  if (px * w[1] < py * w[0]) return (px * w[5] >= py * w[4]) ? 1 : 0;
  return (px * w[3] < py * w[2]) ? 2 : 0;
}

typedef struct {
  frame_t f;
  uint32_t idx[3];
  float w[6];
} walk_t;

/* ---- initialisation, _kernels.pyx:114-192 ---------------------------------- */
static int walk_init(const to_mesh* m, const float o[3], const float d[3], int64_t start, walk_t* s) {
  frame_setup(o, d, &s->f);
  const int32_t* quad = m->sv + 4 * start;
  float q2[4][2];
  for (int i = 0; i < 4; ++i) frame_project(&s->f, m->pts + 3 * (int64_t)quad[i], &q2[i][0], &q2[i][1]);
  const float* P0 = m->pts + 3 * (int64_t)quad[0];
  double e[3][3];
  for (int k = 1; k < 4; ++k) {
    const float* Pk = m->pts + 3 * (int64_t)quad[k];
    for (int c = 0; c < 3; ++c) e[k - 1][c] = (double)Pk[c] - (double)P0[c];
  }
  double rho = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) +
               e[0][1] * (e[1][2] * e[2][0] - e[1][0] * e[2][2]) +
               e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
  int positive = rho > 0;
  int chosen = -1, fallback = -1;
  float fallback_m = -3.4e38f;
  int A = 0, B = 0, C = 0;
  for (int j = 0; j < 4 && chosen < 0; ++j) {
    int a = FACE_OF[j][0], b = FACE_OF[j][1], c = FACE_OF[j][2];
    if (((j % 2) == 0) != positive) {
      int t = b;
      b = c;
      c = t;
    }
    float d0 = q2[a][0] * q2[b][1] - q2[a][1] * q2[b][0];
    float d1 = q2[b][0] * q2[c][1] - q2[b][1] * q2[c][0];
    float d2 = q2[c][0] * q2[a][1] - q2[c][1] * q2[a][0];
    float lo = d0;
    if (d1 < lo) lo = d1;
    if (d2 < lo) lo = d2;
    if (lo >= 0 && (d0 > 0 || d1 > 0 || d2 > 0)) {
      chosen = j;
      A = a; B = b; C = c;
    } else if (lo > fallback_m) {
      fallback_m = lo;
      fallback = j;
    }
  }
  if (chosen < 0) {
    /* all-NaN windows: slot 0 (the device pins the same, see traverse.cuh) */
    chosen = fallback >= 0 ? fallback : 0;
    A = FACE_OF[chosen][0]; B = FACE_OF[chosen][1]; C = FACE_OF[chosen][2];
    if (((chosen % 2) == 0) != positive) {
      int t = B;
      B = C;
      C = t;
    }
  }
  s->idx[0] = (uint32_t)quad[A];
  s->idx[1] = (uint32_t)quad[B];
  s->idx[2] = (uint32_t)quad[C];
  s->w[0] = q2[A][0]; s->w[1] = q2[A][1];
  s->w[2] = q2[B][0]; s->w[3] = q2[B][1];
  s->w[4] = q2[C][0]; s->w[5] = q2[C][1];
  return chosen;
}

/* ---- layout record access ---------------------------------------------------- */
static inline int rec_words(int layout) { return layout == 80 ? 20 : layout / 4; }

static inline uint32_t rec_xor(const to_mesh* m, const uint32_t* r) {
  if (m->layout == 32) return r[3];
  if (m->layout == 80) return r[0] ^ r[1] ^ r[2] ^ r[3];
  return r[0];
}

/* next reference, Alg. 3/5/7, _kernels.pyx:195-235 (+ tet80: slot of idxf) */
static inline uint32_t rec_next(const to_mesh* m, const uint32_t* r, const uint32_t idx[3], uint32_t i3,
                                uint32_t idxf, uint32_t prev) {
  int rank = (idx[0] < idxf) + (idx[1] < idxf) + (idx[2] < idxf) + (i3 < idxf);
  switch (m->layout) {
    case 32: {
      uint32_t out = r[7];
      for (int k = 0; k < 3; ++k)
        if (r[k] == idxf) out = r[4 + k];
      return out;
    }
    case 20:
      return r[1 + rank];
    case 16: {
      int order_a = (idx[0] < i3) + (idx[1] < i3) + (idx[2] < i3);
      uint32_t out = prev;
      if (order_a != 3) out ^= r[1 + order_a];
      if (rank != 3) out ^= r[1 + rank];
      return out;
    }
    default: { /* 80 */
      for (int k = 0; k < 4; ++k)
        if (r[k] == idxf) return r[4 + k];
      return r[7];
    }
  }
}

static inline const float* vertex_xyz(const to_mesh* m, const uint32_t* r, uint32_t v) {
  if (m->layout == 80) {
    for (int k = 0; k < 4; ++k)
      if (r[k] == v) return (const float*)(r + 8 + 3 * k);
    return (const float*)(r + 8 + 9);
  }
  return m->pts + 3 * (int64_t)v;
}

/* ---- step, _kernels.pyx:238-259 -------------------------------------------- */
static uint32_t walk_step(const to_mesh* m, walk_t* s, uint32_t nxt, uint32_t prev) {
  const uint32_t* r = m->recs + (int64_t)rec_words(m->layout) * nxt;
  uint32_t i3 = s->idx[0] ^ s->idx[1] ^ s->idx[2] ^ rec_xor(m, r);
  if (m->layout != 80 && (int64_t)i3 >= m->n_points) i3 = (uint32_t)(m->n_points - 1); /* corrupt record: stay in bounds */
  float px, py;
  frame_project(&s->f, vertex_xyz(m, r, i3), &px, &py);
  int k = alg1_exit(px, py, s->w);
  uint32_t out = rec_next(m, r, s->idx, i3, s->idx[k], prev);
  s->idx[k] = i3;
  s->w[2 * k] = px;
  s->w[2 * k + 1] = py;
  return out;
}

/* ---- epilogue t, _kernels_py.py:435-454 (reciprocal multiply) ---------------
 * Dot products follow numpy 2.3's einsum("ij,ij->i") reduction over three
 * terms: SIMD lanes [p0, p1, p2, 0] summed pairwise, i.e. (p0 + p2) + p1. */
static inline double einsum3(const double* x, const double* y) { return (x[0] * y[0] + x[2] * y[2]) + x[1] * y[1]; }

double to_mt_t(const double* o, const double* d, const double* T) {
  double e1[3], e2[3], pv[3], tv[3], qv[3];
  for (int c = 0; c < 3; ++c) {
    e1[c] = T[3 + c] - T[c];
    e2[c] = T[6 + c] - T[c];
    tv[c] = o[c] - T[c];
  }
  pv[0] = d[1] * e2[2] - d[2] * e2[1];
  pv[1] = d[2] * e2[0] - d[0] * e2[2];
  pv[2] = d[0] * e2[1] - d[1] * e2[0];
  double det = einsum3(e1, pv);
  if (det != 0.0) {
    double inv = 1.0 / det;
    qv[0] = tv[1] * e1[2] - tv[2] * e1[1];
    qv[1] = tv[2] * e1[0] - tv[0] * e1[2];
    qv[2] = tv[0] * e1[1] - tv[1] * e1[0];
    return einsum3(e2, qv) * inv;
  }
  double nrm[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  double den = einsum3(nrm, d);
  if (den == 0.0) return 0.0;
  double rel[3] = {T[0] - o[0], T[1] - o[1], T[2] - o[2]};
  return einsum3(nrm, rel) / den;
}

/* ---- shadow segment t, _kernels.pyx:495-524 (division form) ----------------- */
static double seg_t(const double* o, const double* d, const double* T) {
  double e1[3], e2[3], pv[3], tv[3];
  for (int c = 0; c < 3; ++c) {
    e1[c] = T[3 + c] - T[c];
    e2[c] = T[6 + c] - T[c];
    tv[c] = o[c] - T[c];
  }
  pv[0] = d[1] * e2[2] - d[2] * e2[1];
  pv[1] = d[2] * e2[0] - d[0] * e2[2];
  pv[2] = d[0] * e2[1] - d[1] * e2[0];
  double det = (e1[0] * pv[0] + e1[1] * pv[1]) + e1[2] * pv[2];
  if (det != 0.0) {
    double q0 = tv[1] * e1[2] - tv[2] * e1[1];
    double q1 = tv[2] * e1[0] - tv[0] * e1[2];
    double q2 = tv[0] * e1[1] - tv[1] * e1[0];
    return ((e2[0] * q0 + e2[1] * q1) + e2[2] * q2) / det;
  }
  double nrm[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  double den = (nrm[0] * d[0] + nrm[1] * d[1]) + nrm[2] * d[2];
  if (den == 0.0) return 0.0;
  return ((nrm[0] * (T[0] - o[0]) + nrm[1] * (T[1] - o[1])) + nrm[2] * (T[2] - o[2])) / den;
}

static void finish(const to_mesh* m, int64_t r, uint8_t st, uint32_t ref, uint32_t cur, int vis, const float* o,
                   const float* d, uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited,
                   int32_t* triangle, double* t, int32_t* tet_back) {
  status[r] = st;
  int32_t c = (st == 1) ? (int32_t)(ref & REF_PAYLOAD) : -1;
  cf[r] = c;
  tet[r] = (int32_t)cur;
  visited[r] = vis;
  int32_t tri = -1, back = -1;
  double tt = INFINITY;
  if (c >= 0) {
    tri = m->cf_tri[c];
    double o64[3] = {o[0], o[1], o[2]}, d64[3] = {d[0], d[1], d[2]};
    if (t) tt = to_mt_t(o64, d64, m->tri + 9 * (int64_t)tri);
    int32_t a = m->cf_tets[2 * c], b = m->cf_tets[2 * c + 1];
    back = (a == (int32_t)cur) ? b : a;
  }
  if (triangle) triangle[r] = tri;
  if (t) t[r] = tt;
  if (tet_back) tet_back[r] = back;
}

/* ---- one ray, _kernels.pyx:344-369 ------------------------------------------ */
static void cast_one(const to_mesh* m, int64_t r, const float* o, const float* d, const int32_t* start,
                     uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                     double* t, int32_t* tet_back, int32_t* seq, int64_t seq_cap) {
  walk_t s;
  uint32_t cur = (uint32_t)start[r];
  int j = walk_init(m, o + 3 * r, d + 3 * r, cur, &s);
  uint32_t ref = m->sn[4 * (int64_t)cur + j];
  uint32_t prev = cur;
  int vis = 1;
  uint8_t st;
  int64_t ns = 0;
  if (seq && ns < seq_cap) seq[ns++] = (int32_t)cur;
  for (;;) {
    if (ref == REF_BOUNDARY) { st = 0; break; }
    if (ref & REF_CONSTRAINED) { st = 1; break; }
    uint32_t nxt = ref & REF_PAYLOAD;
    if ((int64_t)nxt >= m->n_tets) { st = 2; break; }
    ref = walk_step(m, &s, nxt, prev);
    prev = nxt;
    cur = nxt;
    ++vis;
    if (seq && ns < seq_cap) seq[ns++] = (int32_t)cur;
    if (vis > m->n_tets) { st = 2; break; }
  }
  if (status) finish(m, r, st, ref, cur, vis, o + 3 * r, d + 3 * r, status, cf, tet, visited, triangle, t, tet_back);
}

/* ---- ScTP predicate, traversal.py:484-511 ------------------------------------ */
static inline void sub3(const double* a, const double* b, double* o) {
  o[0] = a[0] - b[0]; o[1] = a[1] - b[1]; o[2] = a[2] - b[2];
}
static inline void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static inline double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

int to_sctp_exit_face(const double* p, const double* o, const double* d, int entry) {
  double e1[3], e2[3], e3[3], c[3];
  sub3(p + 3, p, e1);
  sub3(p + 6, p, e2);
  sub3(p + 9, p, e3);
  cross3(e2, e3, c);
  int positive = dot3(e1, c) > 0.0;
  int best = -1;
  double best_m = -INFINITY;
  for (int j = 0; j < 4; ++j) {
    if (j == entry) continue;
    int a = FACE_OF[j][0], b = FACE_OF[j][1], cc = FACE_OF[j][2];
    if (((j % 2) == 0) != positive) {
      int t = b;
      b = cc;
      cc = t;
    }
    double A[3], B[3], C[3], x[3];
    sub3(p + 3 * a, o, A);
    sub3(p + 3 * b, o, B);
    sub3(p + 3 * cc, o, C);
    cross3(A, B, x);
    double s0 = dot3(d, x);
    cross3(B, C, x);
    double s1 = dot3(d, x);
    cross3(C, A, x);
    double s2 = dot3(d, x);
    double lo = s0, hi = s0;
    if (s1 < lo) lo = s1;
    if (s2 < lo) lo = s2;
    if (s1 > hi) hi = s1;
    if (s2 > hi) hi = s2;
    if (lo >= 0.0 && hi > 0.0) return j;
    if (lo > best_m) {
      best_m = lo;
      best = j;
    }
  }
  if (best < 0) best = (entry == 0) ? 1 : 0;
  return best;
}

/* ScTP walk: the entry face is opposite the recovered vertex i3; the exit
 * vertex drives the layout's own next-reference rule. */
static void sctp_one(const to_mesh* m, int64_t r, const float* o, const float* d, const int32_t* start,
                     uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                     double* t, int32_t* tet_back) {
  const float* of = o + 3 * r;
  const float* df = d + 3 * r;
  double O[3] = {of[0], of[1], of[2]}, D[3] = {df[0], df[1], df[2]};
  uint32_t cur = (uint32_t)start[r];
  uint32_t ids[4];
  double P[12];
  for (int i = 0; i < 4; ++i) {
    ids[i] = (uint32_t)m->sv[4 * (int64_t)cur + i];
    const float* q = m->pts + 3 * (int64_t)ids[i];
    P[3 * i] = q[0]; P[3 * i + 1] = q[1]; P[3 * i + 2] = q[2];
  }
  int j = to_sctp_exit_face(P, O, D, -1);
  uint32_t ref = m->sn[4 * (int64_t)cur + j];
  uint32_t face[3];
  double FP[9];
  for (int k = 0, n = 0; k < 4; ++k)
    if (k != j) {
      face[n] = ids[k];
      memcpy(FP + 3 * n, P + 3 * k, 3 * sizeof(double));
      ++n;
    }
  uint32_t prev = cur;
  int vis = 1;
  uint8_t st;
  for (;;) {
    if (ref == REF_BOUNDARY) { st = 0; break; }
    if (ref & REF_CONSTRAINED) { st = 1; break; }
    uint32_t nxt = ref & REF_PAYLOAD;
    if ((int64_t)nxt >= m->n_tets) { st = 2; break; }
    const uint32_t* rec = m->recs + (int64_t)rec_words(m->layout) * nxt;
    uint32_t i3 = face[0] ^ face[1] ^ face[2] ^ rec_xor(m, rec);
    if (m->layout != 80 && (int64_t)i3 >= m->n_points) i3 = (uint32_t)(m->n_points - 1); /* corrupt record: stay in bounds */
    const float* q = vertex_xyz(m, rec, i3);
    /* sorted quad: insert i3 into the ascending face */
    int pos = (face[0] < i3) + (face[1] < i3) + (face[2] < i3);
    for (int k = 0, n = 0; k < 4; ++k) {
      if (k == pos) {
        ids[k] = i3;
        P[3 * k] = q[0]; P[3 * k + 1] = q[1]; P[3 * k + 2] = q[2];
      } else {
        ids[k] = face[n];
        memcpy(P + 3 * k, FP + 3 * n, 3 * sizeof(double));
        ++n;
      }
    }
    j = to_sctp_exit_face(P, O, D, pos);
    uint32_t nref = rec_next(m, rec, face, i3, ids[j], prev);
    for (int k = 0, n = 0; k < 4; ++k)
      if (k != j) {
        face[n] = ids[k];
        memcpy(FP + 3 * n, P + 3 * k, 3 * sizeof(double));
        ++n;
      }
    ref = nref;
    prev = nxt;
    cur = nxt;
    ++vis;
    if (vis > m->n_tets) { st = 2; break; }
  }
  finish(m, r, st, ref, cur, vis, of, df, status, cf, tet, visited, triangle, t, tet_back);
}

/* ---- containment, _kernels.pyx:373-413 --------------------------------------- */
static double det3v(const double* a, const double* b, const double* c) {
  return a[0] * (b[1] * c[2] - b[2] * c[1]) + a[1] * (b[2] * c[0] - b[0] * c[2]) + a[2] * (b[0] * c[1] - b[1] * c[0]);
}
static double orient4(const double* P0, const double* P1, const double* P2, const double* P3) {
  double a[3], b[3], c[3];
  sub3(P1, P0, a);
  sub3(P2, P0, b);
  sub3(P3, P0, c);
  return det3v(a, b, c);
}
static int inside_tet(const to_mesh* m, int64_t t, const double* q) {
  double P[4][3];
  for (int i = 0; i < 4; ++i) {
    const float* f = m->pts + 3 * (int64_t)m->sv[4 * t + i];
    P[i][0] = f[0]; P[i][1] = f[1]; P[i][2] = f[2];
  }
  double vol = orient4(P[0], P[1], P[2], P[3]);
  double s = vol > 0 ? 1.0 : -1.0;
  double eps = 1e-10 * fabs(vol) + 1e-300;
  for (int j = 0; j < 4; ++j) {
    const double* S[4] = {P[0], P[1], P[2], P[3]};
    S[j] = q;
    if (s * orient4(S[0], S[1], S[2], S[3]) < -eps) return 0;
  }
  return 1;
}

/* ---- location, _kernels.pyx:416-492 ----------------------------------------- */
static void locate_one(const to_mesh* m, int64_t r, const double* qall, const int32_t* hints, int32_t* out,
                       int32_t* visited) {
  const double* q = qall + 3 * r;
  uint32_t cur = (uint32_t)hints[r];
  out[r] = -1;
  visited[r] = 1;
  if (inside_tet(m, cur, q)) {
    out[r] = (int32_t)cur;
    return;
  }
  double c[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < 4; ++i) {
    const float* f = m->pts + 3 * (int64_t)m->sv[4 * (int64_t)cur + i];
    for (int k = 0; k < 3; ++k) c[k] += (double)f[k];
  }
  for (int k = 0; k < 3; ++k) c[k] = c[k] / 4.0;
  float d32[3] = {(float)(q[0] - c[0]), (float)(q[1] - c[1]), (float)(q[2] - c[2])};
  if (d32[0] == 0 && d32[1] == 0 && d32[2] == 0) return;
  float o32[3] = {(float)c[0], (float)c[1], (float)c[2]};
  walk_t s;
  int j = walk_init(m, o32, d32, cur, &s);
  uint32_t ref = m->sn[4 * (int64_t)cur + j];
  int vis = 1;
  for (;;) {
    uint32_t nxt, entry;
    if (ref == REF_BOUNDARY) break;
    if (ref & REF_CONSTRAINED) {
      uint32_t cfi = ref & REF_PAYLOAD;
      int32_t a = m->cf_tets[2 * (int64_t)cfi], b = m->cf_tets[2 * (int64_t)cfi + 1];
      int32_t other = (a == (int32_t)cur) ? b : a;
      if (other < 0) break;
      nxt = (uint32_t)other;
      entry = ref;
    } else {
      nxt = ref & REF_PAYLOAD;
      entry = cur;
    }
    if ((int64_t)nxt >= m->n_tets) break;
    ref = walk_step(m, &s, nxt, entry);
    cur = nxt;
    ++vis;
    if (inside_tet(m, nxt, q)) {
      out[r] = (int32_t)nxt;
      break;
    }
    if (vis > m->n_tets) break;
  }
  visited[r] = vis;
}

/* ---- shadow, _kernels.pyx:527-614 ------------------------------------------ */
static void shadow_one(const to_mesh* m, int64_t r, const double* p, const double* light, int lstride,
                       const int32_t* p_tet, const int32_t* light_tet, int ltstride, double eps, uint8_t* occ,
                       int32_t* visited) {
  uint32_t cur = (uint32_t)p_tet[r];
  int32_t lt = light_tet[ltstride * r];
  occ[r] = 0;
  visited[r] = 1;
  if ((int32_t)cur == lt) return;
  const double* L = light + (int64_t)lstride * r;
  float o32[3], d32[3];
  double o64[3], d64[3];
  for (int k = 0; k < 3; ++k) {
    d32[k] = (float)(L[k] - p[3 * r + k]);
    o32[k] = (float)p[3 * r + k];
    o64[k] = o32[k];
    d64[k] = d32[k];
  }
  walk_t s;
  int j = walk_init(m, o32, d32, cur, &s);
  uint32_t ref = m->sn[4 * (int64_t)cur + j];
  int vis = 1;
  for (;;) {
    uint32_t nxt, entry;
    if (ref == REF_BOUNDARY) break;
    if (ref & REF_CONSTRAINED) {
      uint32_t cfi = ref & REF_PAYLOAD;
      double tt = seg_t(o64, d64, m->tri + 9 * (int64_t)m->cf_tri[cfi]);
      if (tt >= 1.0 - eps) break;
      if (tt > eps) {
        occ[r] = 1;
        break;
      }
      int32_t a = m->cf_tets[2 * (int64_t)cfi], b = m->cf_tets[2 * (int64_t)cfi + 1];
      int32_t other = (a == (int32_t)cur) ? b : a;
      if (other < 0) break;
      nxt = (uint32_t)other;
      entry = ref;
    } else {
      nxt = ref & REF_PAYLOAD;
      entry = cur;
    }
    if ((int32_t)nxt == lt) break;
    if ((int64_t)nxt >= m->n_tets) break;
    ref = walk_step(m, &s, nxt, entry);
    cur = nxt;
    ++vis;
    if (vis > m->n_tets) break;
  }
  visited[r] = vis;
}

/* ---- threading: contiguous chunks over a pthread pool ------------------------ */
typedef struct {
  int kind;
  const to_mesh* m;
  int64_t lo, hi;
  const float *o, *d;
  const int32_t* start;
  uint8_t* status;
  int32_t *cf, *tet, *visited, *triangle, *tet_back;
  double* t;
  const double *q, *p, *light;
  const int32_t *hints, *p_tet, *light_tet;
  int32_t* out;
  int lstride, ltstride;
  double eps;
  uint8_t* occ;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  for (int64_t r = j->lo; r < j->hi; ++r) {
    switch (j->kind) {
      case 0:
        cast_one(j->m, r, j->o, j->d, j->start, j->status, j->cf, j->tet, j->visited, j->triangle, j->t,
                 j->tet_back, NULL, 0);
        break;
      case 1:
        sctp_one(j->m, r, j->o, j->d, j->start, j->status, j->cf, j->tet, j->visited, j->triangle, j->t,
                 j->tet_back);
        break;
      case 2:
        locate_one(j->m, r, j->q, j->hints, j->out, j->visited);
        break;
      case 3:
        shadow_one(j->m, r, j->p, j->light, j->lstride, j->p_tet, j->light_tet, j->ltstride, j->eps, j->occ,
                   j->visited);
        break;
    }
  }
  return NULL;
}

static int run_parallel(job_t proto, int64_t n, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  if (n < (int64_t)n_threads * 64) n_threads = (int)((n + 63) / 64);
  if (n_threads <= 1) {
    proto.lo = 0;
    proto.hi = n;
    run_job(&proto);
    return 0;
  }
  /* one contiguous chunk per thread (rays are independent) */
  pthread_t th[256];
  job_t jobs[256];
  int created[256];
  int64_t per = (n + n_threads - 1) / n_threads;
  for (int i = 0; i < n_threads; ++i) {
    jobs[i] = proto;
    jobs[i].lo = (int64_t)i * per < n ? (int64_t)i * per : n;
    jobs[i].hi = jobs[i].lo + per < n ? jobs[i].lo + per : n;
    created[i] = pthread_create(&th[i], NULL, run_job, &jobs[i]) == 0;
    if (!created[i]) run_job(&jobs[i]);
  }
  for (int i = 0; i < n_threads; ++i)
    if (created[i]) pthread_join(th[i], NULL);
  return 0;
}

int to_cast_rays(const to_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                 uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                 int32_t* tet_back, int n_threads) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.kind = 0;
  j.m = m; j.o = o; j.d = d; j.start = start; j.status = status; j.cf = cf; j.tet = tet;
  j.visited = visited; j.triangle = triangle; j.t = t; j.tet_back = tet_back;
  return run_parallel(j, n, n_threads);
}

int to_sctp_cast_rays(const to_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                      uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                      double* t, int32_t* tet_back, int n_threads) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.kind = 1;
  j.m = m; j.o = o; j.d = d; j.start = start; j.status = status; j.cf = cf; j.tet = tet;
  j.visited = visited; j.triangle = triangle; j.t = t; j.tet_back = tet_back;
  return run_parallel(j, n, n_threads);
}

int to_cast_rays_visits(const to_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                        const int64_t* offsets, int32_t* seq) {
  for (int64_t r = 0; r < n; ++r)
    cast_one(m, r, o, d, start, NULL, NULL, NULL, NULL, NULL, NULL, NULL, seq + offsets[r],
             offsets[r + 1] - offsets[r]);
  return 0;
}

int to_locate_points(const to_mesh* m, int64_t n, const double* q, const int32_t* hints, int32_t* tet,
                     int32_t* visited, int n_threads) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.kind = 2;
  j.m = m; j.q = q; j.hints = hints; j.out = tet; j.visited = visited;
  return run_parallel(j, n, n_threads);
}

int to_shadow_rays(const to_mesh* m, int64_t n, const double* p, const double* light, int light_stride,
                   const int32_t* p_tet, const int32_t* light_tet, int light_tet_stride, double eps,
                   uint8_t* occluded, int32_t* visited, int n_threads) {
  job_t j;
  memset(&j, 0, sizeof(j));
  j.kind = 3;
  j.m = m; j.p = p; j.light = light; j.lstride = light_stride; j.p_tet = p_tet; j.light_tet = light_tet;
  j.ltstride = light_tet_stride; j.eps = eps; j.occ = occluded; j.visited = visited;
  return run_parallel(j, n, n_threads);
}

void to_build_tet80(const int32_t* sv, const uint32_t* sn, const float* pts, int64_t n_tets, uint32_t* out) {
  for (int64_t t = 0; t < n_tets; ++t) {
    uint32_t* r = out + 20 * t;
    for (int k = 0; k < 4; ++k) {
      r[k] = (uint32_t)sv[4 * t + k];
      r[4 + k] = sn[4 * t + k];
      memcpy(r + 8 + 3 * k, pts + 3 * (int64_t)sv[4 * t + k], 3 * sizeof(float));
    }
  }
}
