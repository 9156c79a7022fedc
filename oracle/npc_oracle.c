/*
 * npc_oracle.c -- CPU restatement of the PointCNN++ reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 library (paper_2511_23227_b200/libnpcg.so).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product path never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj):
 *   orc_mt19937_64_*      core/include/npconv/random.hpp:14-37 (std::mt19937_64 + transforms)
 *   orc_gen_uniform_cube  core/src/synthetic.cpp:12-23
 *   orc_gen_features      core/include/npconv/synthetic.hpp:33-40
 *   orc_make_weights      core/include/npconv/tensors.hpp:142-150
 *   orc_radius_search     core/src/spatial.cpp:20-92   (cell edge = radius, 27 probes,
 *                         d2 = fma(dz,dz,fma(dx,dx,dy*dy)) -- the contraction g++ emits
 *                         for dist2 at -O3 -march=x86-64-v3/native, verified by objdump
 *                         of oracle/_ref)
 *   orc_kernel_index      core/src/triplets.cpp:42-51  (no FMA: sub, add, div, floor, clamp)
 *   orc_build_triplets    core/src/triplets.cpp:53-76
 *   orc_sort_triplets     core/src/triplets.cpp:135-170 (stable counting sort)
 *   orc_choose_sort_axis  core/src/triplets.cpp:172-179
 *   orc_dense_conv        core/src/oracle.cpp:12-67     (literal Eq. 1, fp64, storage order)
 *   orc_rel_error         core/src/gradcheck.cpp:11-31
 *   orc_voxel_downsample  core/src/spatial.cpp:94-152
 *
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libnpref.so built from the reference sources by
 * oracle/Makefile) and against the golden vectors in tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* mt19937_64 (C++11 std::mt19937_64, bit-exact by the standard).      */
/* ------------------------------------------------------------------ */
#define MT_NN 312
#define MT_MM 156
typedef struct {
  uint64_t mt[MT_NN];
  int mti;
} orc_mt;

static void mt_seed(orc_mt* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = MT_NN;
}

static uint64_t mt_next(orc_mt* s) {
  static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= MT_NN) {
    int i;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
    }
    for (; i < MT_NN - 1; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
    }
    uint64_t x = (s->mt[MT_NN - 1] & UM) | (s->mt[0] & LM);
    s->mt[MT_NN - 1] = s->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* random.hpp:21-26: uniform() = (x >> 11) * 2^-53 ; uniform(lo,hi) = lo + (hi-lo)*u */
static double mt_uniform01(orc_mt* s) { return (double)(mt_next(s) >> 11) * 0x1.0p-53; }
static double mt_uniform(orc_mt* s, double lo, double hi) { return lo + (hi - lo) * mt_uniform01(s); }

/* Raw draws, for testing the generator itself against std::mt19937_64. */
void orc_mt19937_64_draws(uint64_t seed, int64_t n, uint64_t* out) {
  orc_mt s;
  mt_seed(&s, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&s);
}

/* synthetic.cpp:12-23 -- x, y, z uniform in [0, extent) in that draw order. */
void orc_gen_uniform_cube(int64_t n, double extent, uint64_t seed, double* xyz) {
  orc_mt s;
  mt_seed(&s, seed);
  for (int64_t p = 0; p < n; ++p) {
    xyz[3 * p + 0] = mt_uniform(&s, 0.0, extent);
    xyz[3 * p + 1] = mt_uniform(&s, 0.0, extent);
    xyz[3 * p + 2] = mt_uniform(&s, 0.0, extent);
  }
}

/* synthetic.hpp:33-40 -- uniform in [-1, 1), cast to the feature type. */
void orc_gen_features_f32(int64_t count, uint64_t seed, float* out) {
  orc_mt s;
  mt_seed(&s, seed);
  for (int64_t p = 0; p < count; ++p) out[p] = (float)mt_uniform(&s, -1.0, 1.0);
}
void orc_gen_features_f64(int64_t count, uint64_t seed, double* out) {
  orc_mt s;
  mt_seed(&s, seed);
  for (int64_t p = 0; p < count; ++p) out[p] = mt_uniform(&s, -1.0, 1.0);
}

/* tensors.hpp:142-150 -- uniform in [-s, s), s = (G*C_in)^-1/2. */
void orc_make_weights_f32(int64_t t, int64_t g, int64_t cin, int64_t cout, uint64_t seed,
                          float* out) {
  const double sc = 1.0 / sqrt((double)(g * cin));
  orc_mt s;
  mt_seed(&s, seed);
  const int64_t n = t * t * t * g * cin * cout;
  for (int64_t p = 0; p < n; ++p) out[p] = (float)mt_uniform(&s, -sc, sc);
}
void orc_make_weights_f64(int64_t t, int64_t g, int64_t cin, int64_t cout, uint64_t seed,
                          double* out) {
  const double sc = 1.0 / sqrt((double)(g * cin));
  orc_mt s;
  mt_seed(&s, seed);
  const int64_t n = t * t * t * g * cin * cout;
  for (int64_t p = 0; p < n; ++p) out[p] = mt_uniform(&s, -sc, sc);
}

/* ------------------------------------------------------------------ */
/* Neighbor search (spatial.cpp:20-92).                                */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t b, x, y, z;
  int64_t index;
} orc_keyed;

static int key_cmp4(const orc_keyed* a, const orc_keyed* c) {
  if (a->b != c->b) return a->b < c->b ? -1 : 1;
  if (a->x != c->x) return a->x < c->x ? -1 : 1;
  if (a->y != c->y) return a->y < c->y ? -1 : 1;
  if (a->z != c->z) return a->z < c->z ? -1 : 1;
  return 0;
}
static int keyed_cmp(const void* pa, const void* pb) {
  const orc_keyed* a = (const orc_keyed*)pa;
  const orc_keyed* c = (const orc_keyed*)pb;
  int r = key_cmp4(a, c);
  if (r) return r;
  return a->index < c->index ? -1 : (a->index > c->index ? 1 : 0);
}
static int i64_cmp(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, c = *(const int64_t*)pb;
  return a < c ? -1 : (a > c ? 1 : 0);
}

/* spatial.cpp:20-22 */
static int64_t cell_of(double c, double edge) { return (int64_t)floor(c / edge); }

/* spatial.cpp:28-31 as compiled: fma(dz, dz, fma(dx, dx, dy*dy)). */
static double dist2_fma(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return fma(dz, dz, fma(dx, dx, dy * dy));
}

typedef struct {
  int64_t n;
  int64_t cap;
  int64_t* out_index;
  int64_t* in_index;
} orc_pairs;

static void pairs_push(orc_pairs* p, int64_t i, int64_t j) {
  if (p->n == p->cap) {
    p->cap = p->cap ? p->cap * 2 : 1024;
    p->out_index = (int64_t*)realloc(p->out_index, (size_t)p->cap * sizeof(int64_t));
    p->in_index = (int64_t*)realloc(p->in_index, (size_t)p->cap * sizeof(int64_t));
  }
  p->out_index[p->n] = i;
  p->in_index[p->n] = j;
  p->n++;
}

/* Returns 0 on success, 4 (RadiusError) / 3 (ShapeError) on validation failure,
 * matching the npcg status numbering. */
int orc_radius_search(const double* q, const int64_t* q_off, int64_t q_nb, const double* t,
                      const int64_t* t_off, int64_t t_nb, double radius, orc_pairs** out) {
  *out = NULL;
  if (!(radius > 0.0)) return 4;
  if (q_nb != t_nb) return 3;
  const double r2 = radius * radius;
  const int64_t nt = t_off[t_nb];
  orc_keyed* grid = (orc_keyed*)malloc((size_t)(nt > 0 ? nt : 1) * sizeof(orc_keyed));
  for (int64_t b = 0; b < t_nb; ++b)
    for (int64_t p = t_off[b]; p < t_off[b + 1]; ++p) {
      grid[p].b = b;
      grid[p].x = cell_of(t[3 * p], radius);
      grid[p].y = cell_of(t[3 * p + 1], radius);
      grid[p].z = cell_of(t[3 * p + 2], radius);
      grid[p].index = p;
    }
  qsort(grid, (size_t)nt, sizeof(orc_keyed), keyed_cmp);

  orc_pairs* res = (orc_pairs*)calloc(1, sizeof(orc_pairs));
  int64_t fcap = 64, fn;
  int64_t* found = (int64_t*)malloc((size_t)fcap * sizeof(int64_t));
  for (int64_t b = 0; b < q_nb; ++b) {
    for (int64_t qi = q_off[b]; qi < q_off[b + 1]; ++qi) {
      const double* qp = q + 3 * qi;
      const int64_t cx = cell_of(qp[0], radius), cy = cell_of(qp[1], radius),
                    cz = cell_of(qp[2], radius);
      fn = 0;
      for (int64_t dx = -1; dx <= 1; ++dx)
        for (int64_t dy = -1; dy <= 1; ++dy)
          for (int64_t dz = -1; dz <= 1; ++dz) {
            orc_keyed probe = {b, cx + dx, cy + dy, cz + dz, 0};
            int64_t lo = 0, hi = nt; /* lower_bound on key only */
            while (lo < hi) {
              int64_t mid = lo + (hi - lo) / 2;
              if (key_cmp4(&grid[mid], &probe) < 0) lo = mid + 1;
              else hi = mid;
            }
            for (; lo < nt && key_cmp4(&grid[lo], &probe) == 0; ++lo) {
              if (dist2_fma(qp, t + 3 * grid[lo].index) <= r2) {
                if (fn == fcap) {
                  fcap *= 2;
                  found = (int64_t*)realloc(found, (size_t)fcap * sizeof(int64_t));
                }
                found[fn++] = grid[lo].index;
              }
            }
          }
      qsort(found, (size_t)fn, sizeof(int64_t), i64_cmp);
      for (int64_t f = 0; f < fn; ++f) pairs_push(res, qi, found[f]);
    }
  }
  free(found);
  free(grid);
  *out = res;
  return 0;
}

int64_t orc_pairs_size(const orc_pairs* p) { return p->n; }
void orc_pairs_copy(const orc_pairs* p, int64_t* out_index, int64_t* in_index) {
  if (p->n) {
    memcpy(out_index, p->out_index, (size_t)p->n * sizeof(int64_t));
    memcpy(in_index, p->in_index, (size_t)p->n * sizeof(int64_t));
  }
}
void orc_pairs_free(orc_pairs* p) {
  if (!p) return;
  free(p->out_index);
  free(p->in_index);
  free(p);
}

/* oracle.cpp:69-95 brute force, (i, j) order; same FMA nesting (p - q). */
int orc_brute_radius(const double* q, const int64_t* q_off, int64_t q_nb, const double* t,
                     const int64_t* t_off, int64_t t_nb, double radius, orc_pairs** out) {
  *out = NULL;
  if (!(radius >= 0.0) || !isfinite(radius)) return 4;
  if (q_nb != t_nb) return 3;
  const double r2 = radius * radius;
  orc_pairs* res = (orc_pairs*)calloc(1, sizeof(orc_pairs));
  for (int64_t b = 0; b < q_nb; ++b)
    for (int64_t i = q_off[b]; i < q_off[b + 1]; ++i)
      for (int64_t j = t_off[b]; j < t_off[b + 1]; ++j) {
        const double dx = t[3 * j] - q[3 * i], dy = t[3 * j + 1] - q[3 * i + 1],
                     dz = t[3 * j + 2] - q[3 * i + 2];
        if (fma(dz, dz, fma(dx, dx, dy * dy)) <= r2) pairs_push(res, i, j);
      }
  *out = res;
  return 0;
}

/* ------------------------------------------------------------------ */
/* Kernel-cell assignment + native build (triplets.cpp:25-76).         */
/* ------------------------------------------------------------------ */
static int64_t clamp_cell(double v, int64_t t) {
  int64_t c = (int64_t)floor(v);
  if (c < 0) c = 0;
  if (c > t - 1) c = t - 1;
  return c;
}

/* Returns k >= 0, or -3 (ShapeError: bad t) / -4 (RadiusError). */
int64_t orc_kernel_index(const double* center, const double* neighbor, double radius,
                         int64_t t) {
  if (t < 1 || t % 2 == 0) return -3;
  if (!(radius > 0.0)) return -4;
  const double cell = 2.0 * radius / (double)t;
  const int64_t ix = clamp_cell((neighbor[0] - center[0] + radius) / cell, t);
  const int64_t iy = clamp_cell((neighbor[1] - center[1] + radius) / cell, t);
  const int64_t iz = clamp_cell((neighbor[2] - center[2] + radius) / cell, t);
  return (ix * t + iy) * t + iz;
}

typedef struct {
  int64_t n;
  uint32_t* i;
  uint32_t* j;
  uint32_t* k;
} orc_triplets;

int orc_build_triplets(const double* outp, const int64_t* out_off, int64_t out_nb,
                       const double* inp, const int64_t* in_off, int64_t in_nb, double radius,
                       int64_t t, orc_triplets** res) {
  *res = NULL;
  if (t < 1 || t % 2 == 0) return 3;
  orc_pairs* pairs = NULL;
  int rc = orc_radius_search(outp, out_off, out_nb, inp, in_off, in_nb, radius, &pairs);
  if (rc) return rc;
  orc_triplets* tl = (orc_triplets*)calloc(1, sizeof(orc_triplets));
  tl->n = pairs->n;
  size_t nb = (size_t)(pairs->n > 0 ? pairs->n : 1) * sizeof(uint32_t);
  tl->i = (uint32_t*)malloc(nb);
  tl->j = (uint32_t*)malloc(nb);
  tl->k = (uint32_t*)malloc(nb);
  for (int64_t n = 0; n < pairs->n; ++n) {
    const int64_t i = pairs->out_index[n], j = pairs->in_index[n];
    tl->i[n] = (uint32_t)i;
    tl->j[n] = (uint32_t)j;
    tl->k[n] = (uint32_t)orc_kernel_index(outp + 3 * i, inp + 3 * j, radius, t);
  }
  orc_pairs_free(pairs);
  *res = tl;
  return 0;
}

int64_t orc_triplets_size(const orc_triplets* t) { return t->n; }
void orc_triplets_copy(const orc_triplets* t, uint32_t* i, uint32_t* j, uint32_t* k) {
  if (!t->n) return;
  memcpy(i, t->i, (size_t)t->n * 4);
  memcpy(j, t->j, (size_t)t->n * 4);
  memcpy(k, t->k, (size_t)t->n * 4);
}
void orc_triplets_free(orc_triplets* t) {
  if (!t) return;
  free(t->i);
  free(t->j);
  free(t->k);
  free(t);
}

/* triplets.cpp:135-170: axis 0 none, 1 by_i, 2 by_j, 3 by_k; stable counting sort. */
void orc_sort_triplets(const uint32_t* i, const uint32_t* j, const uint32_t* k, int64_t n,
                       int axis, int64_t n_out, int64_t n_in, int64_t n_kernels, uint32_t* oi,
                       uint32_t* oj, uint32_t* ok) {
  if (axis == 0 || n <= 1) {
    if (n > 0) {
      memmove(oi, i, (size_t)n * 4);
      memmove(oj, j, (size_t)n * 4);
      memmove(ok, k, (size_t)n * 4);
    }
    return;
  }
  const uint32_t* key = axis == 1 ? i : (axis == 2 ? j : k);
  const int64_t range = axis == 1 ? n_out : (axis == 2 ? n_in : n_kernels);
  int64_t* starts = (int64_t*)calloc((size_t)range + 1, sizeof(int64_t));
  for (int64_t p = 0; p < n; ++p) ++starts[key[p] + 1];
  for (int64_t b = 1; b <= range; ++b) starts[b] += starts[b - 1];
  for (int64_t p = 0; p < n; ++p) {
    const int64_t dst = starts[key[p]]++;
    oi[dst] = i[p];
    oj[dst] = j[p];
    ok[dst] = k[p];
  }
  free(starts);
}

/* triplets.cpp:172-179 */
int orc_choose_sort_axis(int64_t n_out, int64_t n_in, int64_t n_kernels) {
  const int64_t lo = n_in < n_out ? n_in : n_out;
  if (n_kernels <= lo) return 3;
  return n_out <= n_in ? 1 : 2;
}

/* ------------------------------------------------------------------ */
/* Dense oracle (oracle.cpp:12-67): literal Eq. 1 in storage order.    */
/* w: (K, G, Cin, Cout); fin: (n_in, G, Cin); gout: (n_out, G, Cout)   */
/* fout: (n_out, G, Cout); grad_in: (n_in, G, Cin);                    */
/* grad_w: (K, G, Cout, Cin)  -- WeightGradient orientation.           */
/* Outputs must be zero-initialised by the caller.                     */
/* Returns 0, or 6 (IndexError) if a triplet is out of range.          */
/* ------------------------------------------------------------------ */
int orc_dense_conv(const double* w, int64_t K, int64_t G, int64_t cin, int64_t cout,
                   const double* fin, int64_t n_in, const uint32_t* ti, const uint32_t* tj,
                   const uint32_t* tk, int64_t n_t, int64_t n_out, const double* gout,
                   double* fout, double* grad_in, double* grad_w) {
  for (int64_t t = 0; t < n_t; ++t) {
    const int64_t i = ti[t], j = tj[t], k = tk[t];
    if (i >= n_out || j >= n_in || k >= K) return 6;
    for (int64_t g = 0; g < G; ++g) {
      const double* wm = w + ((k * G + g) * cin) * cout;
      const double* f = fin + (j * G + g) * cin;
      double* out = fout + (i * G + g) * cout;
      for (int64_t c = 0; c < cin; ++c)
        for (int64_t m = 0; m < cout; ++m) out[m] += wm[c * cout + m] * f[c];
      if (gout) {
        const double* go = gout + (i * G + g) * cout;
        double* gi = grad_in + (j * G + g) * cin;
        for (int64_t c = 0; c < cin; ++c) {
          double s = 0.0;
          for (int64_t m = 0; m < cout; ++m) s += wm[c * cout + m] * go[m];
          gi[c] += s;
        }
        double* gw = grad_w + ((k * G + g) * cout) * cin;
        for (int64_t m = 0; m < cout; ++m)
          for (int64_t c = 0; c < cin; ++c) gw[m * cin + c] += go[m] * f[c];
      }
    }
  }
  return 0;
}

/* gradcheck.cpp:11-31 -- max|a-b| / max(max|b|, floor). */
double orc_rel_error_f64(const double* a, const double* b, int64_t n, double floor_) {
  double md = 0.0, mr = 0.0;
  for (int64_t p = 0; p < n; ++p) {
    const double d = fabs(a[p] - b[p]);
    if (d > md) md = d;
    if (fabs(b[p]) > mr) mr = fabs(b[p]);
  }
  return md / (mr > floor_ ? mr : floor_);
}
double orc_rel_error_f32(const float* a, const double* b, int64_t n, double floor_) {
  double md = 0.0, mr = 0.0;
  for (int64_t p = 0; p < n; ++p) {
    const double d = fabs((double)a[p] - b[p]);
    if (d > md) md = d;
    if (fabs(b[p]) > mr) mr = fabs(b[p]);
  }
  return md / (mr > floor_ ? mr : floor_);
}

/* ------------------------------------------------------------------ */
/* voxel_downsample (spatial.cpp:94-152).                              */
/* kept[m] = original index, parent[p] = output index, offsets[b].     */
/* Returns number kept, or -5 (VoxelError).                            */
/* ------------------------------------------------------------------ */
int64_t orc_voxel_downsample(const double* xyz, const int64_t* off, int64_t nb, double voxel,
                             int64_t* kept, int64_t* parent, int64_t* out_off) {
  if (!(voxel > 0.0)) return -5;
  const int64_t n = off[nb];
  orc_keyed* keyed = (orc_keyed*)malloc((size_t)(n > 0 ? n : 1) * sizeof(orc_keyed));
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t p = off[b]; p < off[b + 1]; ++p) {
      keyed[p].b = b;
      keyed[p].x = cell_of(xyz[3 * p], voxel);
      keyed[p].y = cell_of(xyz[3 * p + 1], voxel);
      keyed[p].z = cell_of(xyz[3 * p + 2], voxel);
      keyed[p].index = p;
    }
  qsort(keyed, (size_t)n, sizeof(orc_keyed), keyed_cmp);
  int64_t m = 0, prev_batch = 0;
  out_off[0] = 0;
  int64_t run = 0;
  while (run < n) {
    int64_t end = run;
    while (end < n && key_cmp4(&keyed[end], &keyed[run]) == 0) ++end;
    double c[3] = {0.0, 0.0, 0.0};
    for (int64_t s = run; s < end; ++s) {
      const double* p = xyz + 3 * keyed[s].index;
      c[0] += p[0];
      c[1] += p[1];
      c[2] += p[2];
    }
    const double inv = 1.0 / (double)(end - run);
    c[0] *= inv;
    c[1] *= inv;
    c[2] *= inv;
    int64_t best = keyed[run].index;
    double best_d2 = dist2_fma(xyz + 3 * best, c);
    for (int64_t s = run + 1; s < end; ++s) {
      const double d2 = dist2_fma(xyz + 3 * keyed[s].index, c);
      if (d2 < best_d2) {
        best_d2 = d2;
        best = keyed[s].index;
      }
    }
    const int64_t batch = keyed[run].b;
    while (prev_batch < batch) {
      out_off[++prev_batch] = m;
    }
    kept[m] = best;
    for (int64_t s = run; s < end; ++s) parent[keyed[s].index] = m;
    ++m;
    run = end;
  }
  while (prev_batch < nb) out_off[++prev_batch] = m;
  free(keyed);
  return m;
}

/* ------------------------------------------------------------------ */
/* Degraded (voxel) build, triplets.cpp:78-133.                         */
/* Sites = voxel_downsample(in, v) (representative per occupied voxel,  */
/* (batch, key) order); site key = floor(p_rep / v) per axis; snapped   */
/* position = (key + 0.5) * v; for each site s and integer offsets      */
/* (dx, dy, dz) in [-h, h]^3 (dx outer, dz inner, h = (t-1)/2) whose    */
/* voxel of the same batch is occupied: triplet (s, site of that voxel, */
/* k = ((dx+h) t + (dy+h)) t + (dz+h)).  Returns the number of sites,   */
/* or -3 (ShapeError: t) / -5 (VoxelError), validated in that order     */
/* (triplets.cpp:79-81).  snapped: n*3, kept: n, parent: n, site_off:   */
/* nb+1 (all caller-allocated at the input size).                       */
/* ------------------------------------------------------------------ */
int64_t orc_build_triplets_degraded(const double* xyz, const int64_t* off, int64_t nb,
                                    double voxel, int64_t t, double* snapped, int64_t* kept,
                                    int64_t* parent, int64_t* site_off, orc_triplets** res) {
  *res = NULL;
  if (t < 1 || t % 2 == 0) return -3;
  if (!(voxel > 0.0)) return -5;
  const int64_t ns = orc_voxel_downsample(xyz, off, nb, voxel, kept, parent, site_off);
  if (ns < 0) return ns;
  orc_keyed* keys = (orc_keyed*)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(orc_keyed));
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t s = site_off[b]; s < site_off[b + 1]; ++s) {
      const double* p = xyz + 3 * kept[s];
      keys[s].b = b;
      keys[s].x = cell_of(p[0], voxel);
      keys[s].y = cell_of(p[1], voxel);
      keys[s].z = cell_of(p[2], voxel);
      keys[s].index = s;
      snapped[3 * s + 0] = ((double)keys[s].x + 0.5) * voxel;
      snapped[3 * s + 1] = ((double)keys[s].y + 0.5) * voxel;
      snapped[3 * s + 2] = ((double)keys[s].z + 0.5) * voxel;
    }
  /* sites are in (batch, key) order already (voxel_downsample output order) */
  const int64_t h = (t - 1) / 2;
  orc_triplets* tl = (orc_triplets*)calloc(1, sizeof(orc_triplets));
  int64_t cap = 16;
  tl->i = (uint32_t*)malloc((size_t)cap * 4);
  tl->j = (uint32_t*)malloc((size_t)cap * 4);
  tl->k = (uint32_t*)malloc((size_t)cap * 4);
  for (int64_t s = 0; s < ns; ++s)
    for (int64_t dx = -h; dx <= h; ++dx)
      for (int64_t dy = -h; dy <= h; ++dy)
        for (int64_t dz = -h; dz <= h; ++dz) {
          orc_keyed q = {keys[s].b, keys[s].x + dx, keys[s].y + dy, keys[s].z + dz, 0};
          int64_t lo = 0, hi = ns;
          while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (key_cmp4(&keys[mid], &q) < 0) lo = mid + 1;
            else hi = mid;
          }
          if (lo >= ns || key_cmp4(&keys[lo], &q) != 0) continue;
          if (tl->n == cap) {
            cap *= 2;
            tl->i = (uint32_t*)realloc(tl->i, (size_t)cap * 4);
            tl->j = (uint32_t*)realloc(tl->j, (size_t)cap * 4);
            tl->k = (uint32_t*)realloc(tl->k, (size_t)cap * 4);
          }
          tl->i[tl->n] = (uint32_t)s;
          tl->j[tl->n] = (uint32_t)lo;
          tl->k[tl->n] = (uint32_t)(((dx + h) * t + (dy + h)) * t + (dz + h));
          tl->n++;
        }
  free(keys);
  *res = tl;
  return ns;
}
