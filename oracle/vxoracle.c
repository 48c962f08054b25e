/*
 * vxoracle.c — CPU restatement of the reference hot path, TEST
 * INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library, and only as the checker or as
 * the reported CPU baseline.  The product (paper_1807_03119_b200) never
 * calls it.
 *
 * It restates /root/reference/pkg/src/voxray with plain C loops:
 *   - build_histogram's np.bincount            histogram.py:119-133
 *   - primary_ray_dirs / ray_box_spans (FP64)   render.py:188-230
 *   - _march_batch, sequential per ray          render.py:236-339
 *     (no empty-space skipping: every sample is taken, exactly as the
 *      reference; 64-bit voxel indices = the int64 patch of render.py:306
 *      needed for n > 1258)
 *   - the six filters                           filters.py:165-266
 *   - sobel_normal_batch / shade_phong_batch    render.py:344-403
 *   - render_frame (workers=1: one band)        render.py:467-560
 *   - generate_phantom input generator          volume.py:317-368, rng.py
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: no FMA contraction, so
 * float/double expressions round exactly like numpy's separate ufuncs).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>
#include <unistd.h>

typedef struct {
  const uint8_t* data; /* (nz, ny, nx) x fastest */
  int64_t nx, ny, nz;
} Vol;

static inline int vat(const Vol* V, int64_t x, int64_t y, int64_t z) {
  if (x < 0 || y < 0 || z < 0 || x >= V->nx || y >= V->ny || z >= V->nz) return 0;
  return V->data[(z * V->ny + y) * V->nx + x];
}

/* ---- statistics -------------------------------------------------------- */

void orc_hist256(const uint8_t* data, uint64_t n, uint64_t* counts) {
  memset(counts, 0, 256 * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) counts[data[i]]++;
}

/* ---- filters (filters.py:165-227) --------------------------------------- */

typedef struct {
  int kind; /* 0 none 1 mean 2 sigma 3 okada 4 entropy 5 local-cluster 6 axis */
  int M, d;
  int pairwise;
  double T, band, okada_t, entropy_t;
  const double* lut;
} Filt;

static double pw_sum(const double* a, int n) {
  /* numpy pairwise_sum (single-coordinate entropy batch) */
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

static double filter_value(const Vol* V, const Filt* F, int64_t x, int64_t y, int64_t z) {
  const int h = (F->M - 1) / 2;
  switch (F->kind) {
    case 0:
      return (double)vat(V, x, y, z);
    case 1: { /* mean: kernel_offsets sum / M^3 */
      int64_t s = 0;
      for (int dx = -h; dx <= h; ++dx)
        for (int dy = -h; dy <= h; ++dy)
          for (int dz = -h; dz <= h; ++dz) s += vat(V, x + dx, y + dy, z + dz);
      return (double)s / (double)(F->M * F->M * F->M);
    }
    case 2: { /* sigma: |v - P0| <= band (int16 diff vs FP64 band) */
      const int c = vat(V, x, y, z);
      int64_t s = 0, cnt = 0;
      for (int dx = -h; dx <= h; ++dx)
        for (int dy = -h; dy <= h; ++dy)
          for (int dz = -h; dz <= h; ++dz) {
            const int v = vat(V, x + dx, y + dy, z + dz);
            if ((double)abs(v - c) <= F->band) {
              s += v;
              ++cnt;
            }
          }
      return (double)s / (double)cnt;
    }
    case 3: { /* okada: 6 faces with |P0 - v| < T_d, centre excluded */
      static const int off[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
      const int c = vat(V, x, y, z);
      int64_t s = 0;
      int n = 0;
      for (int k = 0; k < 6; ++k) {
        const int v = vat(V, x + off[k][0], y + off[k][1], z + off[k][2]);
        if ((double)abs(c - v) < F->okada_t) {
          s += v;
          ++n;
        }
      }
      return n > 0 ? (double)s / (double)n : 0.0;
    }
    case 4: { /* entropy: LUT sum in kernel_offsets order (dx, dy, dz) */
      double terms[2744]; /* M <= 13 */
      if (F->M > 13) return NAN;
      int k = 0;
      for (int dx = -h; dx <= h; ++dx)
        for (int dy = -h; dy <= h; ++dy)
          for (int dz = -h; dz <= h; ++dz) terms[k++] = F->lut[vat(V, x + dx, y + dy, z + dz)];
      double H = 0.0;
      if (F->pairwise) {
        H = pw_sum(terms, k);
      } else if (k > 0) {
        H = terms[0];
        for (int i = 1; i < k; ++i) H += terms[i];
      }
      return H > F->entropy_t ? (double)vat(V, x, y, z) : 0.0;
    }
    case 6: { /* axis_cluster_average: 3 arms through the centre / 3M */
      int64_t s = 0;
      for (int i = -h; i <= h; ++i) s += vat(V, x + i, y, z) + vat(V, x, y + i, z) + vat(V, x, y, z + i);
      return (double)s / (double)(3 * F->M);
    }
    default: { /* local cluster: 9 centres x 3 arms x M, duplicates kept */
      int64_t s = 0;
      for (int c = 0; c < 9; ++c) {
        int64_t cx = x, cy = y, cz = z;
        if (c) {
          const int q = c - 1;
          cx += (q & 4) ? F->d : -F->d;
          cy += (q & 2) ? F->d : -F->d;
          cz += (q & 1) ? F->d : -F->d;
        }
        for (int i = -h; i <= h; ++i)
          s += vat(V, cx + i, cy, cz) + vat(V, cx, cy + i, cz) + vat(V, cx, cy, cz + i);
      }
      return (double)s / (double)(27 * F->M);
    }
  }
}

void orc_filter_batch(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz, const int64_t* xs,
                      const int64_t* ys, const int64_t* zs, int64_t n, int kind, int M, int d,
                      double band, double okada_t, double entropy_t, const double* lut,
                      int pairwise, double* out) {
  Vol V = {data, nx, ny, nz};
  Filt F = {kind, M, d, pairwise, 0.0, band, okada_t, entropy_t, lut};
  for (int64_t i = 0; i < n; ++i) out[i] = filter_value(&V, &F, xs[i], ys[i], zs[i]);
}

/* ---- ray setup (render.py:188-230) ---------------------------------------- */

typedef struct {
  double right[3], up[3], fwd[3], origin[3];
  double tan_f, aspect;
  int W, H;
} Cam;

static void ray_dir(const Cam* C, int i, int j, double d[3]) {
  const double u = ((2.0 * ((double)i + 0.5)) / (double)C->W - 1.0) * C->tan_f * C->aspect;
  const double v = (1.0 - (2.0 * ((double)j + 0.5)) / (double)C->H) * C->tan_f;
  for (int c = 0; c < 3; ++c) d[c] = (C->fwd[c] + u * C->right[c]) + v * C->up[c];
  const double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
  for (int c = 0; c < 3; ++c) d[c] = d[c] / nrm;
}

static double nmin(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a < b ? a : b); }
static double nmax(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a > b ? a : b); }

static void ray_span(const double o[3], const double d[3], const int64_t dims[3], double* te,
                     double* tx) {
  double tmin = -INFINITY, tmax = INFINITY;
  for (int a = 0; a < 3; ++a) {
    const double lo = -0.5, hi = (double)dims[a] - 0.5;
    double near, far;
    if (d[a] == 0.0) {
      const int inside = (lo <= o[a]) && (o[a] <= hi);
      near = inside ? -INFINITY : INFINITY;
      far = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = 1.0 / d[a];
      const double t1 = (lo - o[a]) * inv, t2 = (hi - o[a]) * inv;
      near = nmin(t1, t2);
      far = nmax(t1, t2);
    }
    tmin = nmax(tmin, near);
    tmax = nmin(tmax, far);
  }
  *te = nmax(tmin, 0.0);
  *tx = tmax;
}

void orc_ray_dirs(const double* cam, int W, int H, double* out) {
  Cam C;
  memcpy(C.right, cam, 12 * sizeof(double));
  C.tan_f = cam[12];
  C.aspect = cam[13];
  C.W = W;
  C.H = H;
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i) ray_dir(&C, i, j, out + 3 * ((int64_t)j * W + i));
}

void orc_ray_spans(const double* origin, const double* dirs, int64_t n, const int64_t* dims,
                   double* te, double* tx) {
  for (int64_t r = 0; r < n; ++r) ray_span(origin, dirs + 3 * r, dims, te + r, tx + r);
}

/* ---- march (render.py:236-339), one ray at a time -------------------------- */

typedef struct {
  float s, sk[16];
  int chunk, need_clip, thr;
  float xmax, ymax, zmax;
  double T;
} March;

static int march(const Vol* V, const March* M, const Filt* F, const double o[3], const double d[3],
                 double te, double tx, int64_t max_steps, int hv[3], float* ht, double* hval,
                 int64_t* nsamp) {
  if (!(tx >= te) || M->thr > 255) return 0;
  float base = (float)te;
  const float tend = (float)tx;
  float fo[3], fd[3];
  for (int c = 0; c < 3; ++c) {
    fo[c] = (float)(o[c] + 0.5);
    fd[c] = (float)d[c];
  }
  int64_t done = 0;
  while (done < max_steps) {
    int m = M->chunk;
    if (max_steps - done < m) m = (int)(max_steps - done);
    for (int k = 0; k < m; ++k) {
      const float tk = base + M->sk[k];
      if (!(tk <= tend)) break;
      float p[3];
      for (int c = 0; c < 3; ++c) p[c] = fo[c] + tk * fd[c];
      if (M->need_clip) {
        const float hi[3] = {M->xmax, M->ymax, M->zmax};
        for (int c = 0; c < 3; ++c) p[c] = p[c] < 0.0f ? 0.0f : (p[c] > hi[c] ? hi[c] : p[c]);
      }
      const int vx = (int)p[0], vy = (int)p[1], vz = (int)p[2]; /* astype(int32): trunc */
      ++*nsamp;
      if (vat(V, vx, vy, vz) >= M->thr) {
        const double f = filter_value(V, F, vx, vy, vz);
        if (f >= M->T) {
          hv[0] = vx;
          hv[1] = vy;
          hv[2] = vz;
          *ht = tk;
          *hval = f;
          return 1;
        }
      }
    }
    base = base + (float)m * M->s;
    done += m;
    if (!(base <= tend)) return 0;
  }
  return 0;
}

/* ---- Sobel / Phong (render.py:344-403) ----------------------------------------- */

static void sobel(const Vol* V, int64_t x, int64_t y, int64_t z, const double fb[3], double n[3]) {
  int64_t g[3] = {0, 0, 0};
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        const int v = vat(V, x + dx, y + dy, z + dz);
        const int sx = dx ? 1 : 2, sy = dy ? 1 : 2, sz = dz ? 1 : 2;
        g[0] += dx * sy * sz * v;
        g[1] += dy * sx * sz * v;
        g[2] += dz * sx * sy * v;
      }
  const double g0 = (double)g[0], g1 = (double)g[1], g2 = (double)g[2];
  const double nrm = sqrt((g0 * g0 + g1 * g1) + g2 * g2);
  if (nrm < 1e-12) {
    n[0] = fb[0];
    n[1] = fb[1];
    n[2] = fb[2];
  } else {
    n[0] = -g0 / nrm;
    n[1] = -g1 / nrm;
    n[2] = -g2 / nrm;
  }
}

typedef struct {
  double ka, kd, ks, shin, l[3];
} Shade;

/* n.l as the reference host's OpenBLAS dgemv (measured), r.v as numpy einsum */
static double phong(const double n[3], const double v[3], const Shade* S) {
  const double ndotl = fma(n[2], S->l[2], fma(n[0], S->l[0], n[1] * S->l[1]));
  const double r0 = (2.0 * ndotl) * n[0] - S->l[0];
  const double r1 = (2.0 * ndotl) * n[1] - S->l[1];
  const double r2 = (2.0 * ndotl) * n[2] - S->l[2];
  const double rdotv = (r0 * v[0] + r2 * v[2]) + r1 * v[1];
  return (S->ka + S->kd * (ndotl > 0.0 ? ndotl : 0.0)) + S->ks * pow(rdotv > 0.0 ? rdotv : 0.0, S->shin);
}

static uint8_t quantise(double I) {
  const double c = I < 0.0 ? 0.0 : (I > 1.0 ? 1.0 : I);
  return (uint8_t)floor(c * 255.0 + 0.5);
}

void orc_sobel_batch(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz, const int64_t* xs,
                     const int64_t* ys, const int64_t* zs, int64_t n, const double* fb,
                     double* out) {
  Vol V = {data, nx, ny, nz};
  for (int64_t i = 0; i < n; ++i) sobel(&V, xs[i], ys[i], zs[i], fb + 3 * i, out + 3 * i);
}

void orc_phong_batch(const double* normals, const double* views, int64_t n, const double* shade,
                     uint8_t* out) {
  Shade S = {shade[0], shade[1], shade[2], shade[3], {shade[4], shade[5], shade[6]}};
  for (int64_t i = 0; i < n; ++i) out[i] = quantise(phong(normals + 3 * i, views + 3 * i, &S));
}

/* ---- render_frame (render.py:488-560) ------------------------------------------ */

typedef struct {
  const Vol* V;
  const Cam* C;
  const March* M;
  const Filt* F;
  const Shade* S;
  int bg;
  const int64_t* dims;
  int64_t max_steps;
  int row_step, W, H;
  uint8_t* pixels;
  int32_t* hit_voxel;
  float* hit_t;
  double* intensity;
  int next_row;
  int64_t hits, samples;
  pthread_mutex_t mu;
} RenderJob;

static void* render_worker(void* arg) {
  RenderJob* J = (RenderJob*)arg;
  int64_t hits = 0, samples = 0;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int j = J->next_row;
    J->next_row += J->row_step;
    pthread_mutex_unlock(&J->mu);
    if (j >= J->H) break;
    for (int i = 0; i < J->W; ++i) {
      const int64_t p = (int64_t)j * J->W + i;
      double d[3], te, tx;
      ray_dir(J->C, i, j, d);
      ray_span(J->C->origin, d, J->dims, &te, &tx);
      int hv[3] = {-1, -1, -1};
      float ht = 0.0f;
      double hval = 0.0, I = -1.0;
      int64_t ns = 0;
      const int hit = march(J->V, J->M, J->F, J->C->origin, d, te, tx, J->max_steps, hv, &ht,
                            &hval, &ns);
      samples += ns;
      uint8_t px = (uint8_t)J->bg;
      if (hit) {
        ++hits;
        const double view[3] = {-d[0], -d[1], -d[2]};
        double n[3];
        sobel(J->V, hv[0], hv[1], hv[2], view, n);
        I = phong(n, view, J->S);
        px = quantise(I);
      }
      J->pixels[p] = px;
      if (J->hit_voxel) {
        J->hit_voxel[3 * p] = hit ? hv[0] : -1;
        J->hit_voxel[3 * p + 1] = hit ? hv[1] : -1;
        J->hit_voxel[3 * p + 2] = hit ? hv[2] : -1;
      }
      if (J->hit_t) J->hit_t[p] = hit ? ht : 0.0f;
      if (J->intensity) J->intensity[p] = I;
    }
  }
  pthread_mutex_lock(&J->mu);
  J->hits += hits;
  J->samples += samples;
  pthread_mutex_unlock(&J->mu);
  return NULL;
}

static void run_threads(void* (*fn)(void*), void* arg, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  int started = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tid[started], NULL, fn, arg) == 0) ++started;
  fn(arg);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
}

/* cam: right[3] up[3] fwd[3] origin[3] tan_f aspect
 * prm: step max_steps chunk need_clip ka kd ks shin l0 l1 l2 background
 * flt: kind M d T band okada_t entropy_t
 * row_step: render rows j % row_step == 0 only (bounded CPU samples)
 * outputs nullable except pixels; returns hit count of rendered rows */
int64_t orc_render(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz, const double* cam,
                   int W, int H, const double* prm, const double* flt, const double* lut,
                   int row_step, int threads, uint8_t* pixels, int32_t* hit_voxel, float* hit_t,
                   double* intensity, int64_t* samples_out) {
  Vol V = {data, nx, ny, nz};
  Cam C;
  memcpy(C.right, cam, 12 * sizeof(double));
  C.tan_f = cam[12];
  C.aspect = cam[13];
  C.W = W;
  C.H = H;
  const double step = prm[0];
  March M;
  M.s = (float)step;
  for (int k = 0; k < 16; ++k) M.sk[k] = M.s * (float)k;
  M.chunk = (int)prm[2];
  M.need_clip = (int)prm[3];
  M.xmax = (float)nx;
  M.ymax = (float)ny;
  M.zmax = (float)nz;
  const double T = flt[3];
  const double c = ceil(T);
  M.thr = c < 0.0 ? 0 : (c > 256.0 ? 256 : (int)c);
  M.T = T;
  Filt F = {(int)flt[0], (int)flt[1], (int)flt[2], 0, T, flt[4], flt[5], flt[6], lut};
  Shade S = {prm[4], prm[5], prm[6], prm[7], {prm[8], prm[9], prm[10]}};
  const int bg = (int)prm[11];
  const int64_t dims[3] = {nx, ny, nz};
  if (row_step < 1) row_step = 1;

  /* max_steps over the whole frame (workers=1: one band), render.py:469-473 */
  int64_t max_steps = (int64_t)prm[1];
  if (max_steps <= 0) {
    double longest = 0.0;
    for (int j = 0; j < H; ++j)
      for (int i = 0; i < W; ++i) {
        double d[3], te, tx;
        ray_dir(&C, i, j, d);
        ray_span(C.origin, d, dims, &te, &tx);
        const double sp = (tx >= te) ? tx - te : 0.0;
        if (sp > longest) longest = sp;
      }
    max_steps = (int64_t)ceil(longest / step) + 1;
    if (max_steps < 1) max_steps = 1;
  }
  RenderJob job = {&V, &C, &M, &F, &S, bg, dims, max_steps, row_step, W, H, pixels, hit_voxel,
                   hit_t, intensity, 0, 0, 0, PTHREAD_MUTEX_INITIALIZER};
  run_threads(render_worker, &job, threads);
  const int64_t hits = job.hits, samples = job.samples;
  if (samples_out) *samples_out = samples;
  return hits;
}

/* march_ray for arbitrary rays (render.py:426-464); max_steps per ray */
void orc_march_rays(const uint8_t* data, int64_t nx, int64_t ny, int64_t nz, const double* origins,
                    const double* dirs, const double* te, const double* tx, const int64_t* max_steps,
                    int64_t n, double step, int chunk, int need_clip, const double* flt,
                    const double* lut, uint8_t* hit, int32_t* vox, float* t, double* val) {
  Vol V = {data, nx, ny, nz};
  March M;
  M.s = (float)step;
  for (int k = 0; k < 16; ++k) M.sk[k] = M.s * (float)k;
  M.chunk = chunk;
  M.need_clip = need_clip;
  M.xmax = (float)nx;
  M.ymax = (float)ny;
  M.zmax = (float)nz;
  const double T = flt[3];
  const double c = ceil(T);
  M.thr = c < 0.0 ? 0 : (c > 256.0 ? 256 : (int)c);
  M.T = T;
  Filt F = {(int)flt[0], (int)flt[1], (int)flt[2], 0, T, flt[4], flt[5], flt[6], lut};
  for (int64_t r = 0; r < n; ++r) {
    int hv[3] = {-1, -1, -1};
    float ht = 0.0f;
    double hval = 0.0;
    int64_t ns = 0;
    hit[r] = (uint8_t)march(&V, &M, &F, origins + 3 * r, dirs + 3 * r, te[r], tx[r], max_steps[r],
                            hv, &ht, &hval, &ns);
    vox[3 * r] = hv[0];
    vox[3 * r + 1] = hv[1];
    vox[3 * r + 2] = hv[2];
    t[r] = ht;
    val[r] = hval;
  }
}

/* ---- phantom generator (volume.py:317-368; inputs only) -------------------------- */

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  uint8_t* out;
  int64_t n;
  double sigma;
  uint64_t seed;
  int64_t next;
  pthread_mutex_t mu;
} NoiseJob;

static void* noise_worker(void* arg) {
  NoiseJob* J = (NoiseJob*)arg;
  const int64_t block = 1 << 20;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int64_t i0 = J->next;
    J->next += block;
    pthread_mutex_unlock(&J->mu);
    if (i0 >= J->n) break;
    const int64_t i1 = i0 + block < J->n ? i0 + block : J->n;
    for (int64_t i = i0; i < i1; ++i) {
      const uint64_t j0 = 2ull * (uint64_t)i;
      const uint64_t b0 = mix64(J->seed + (j0 + 1ull) * 0x9E3779B97F4A7C15ull);
      const uint64_t b1 = mix64(J->seed + (j0 + 2ull) * 0x9E3779B97F4A7C15ull);
      const double u1 = ((double)(b0 >> 11) + 1.0) * 1.1102230246251565e-16;
      const double u2 = (double)(b1 >> 11) * 1.1102230246251565e-16;
      const double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
      double v = floor(((double)J->out[i] + J->sigma * g) + 0.5);
      v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
      J->out[i] = (uint8_t)v;
    }
  }
  return NULL;
}

/* shapes: n x [kind cx cy cz intensity radius thickness ex ey ez] */
void orc_phantom(uint8_t* out, int64_t nx, int64_t ny, int64_t nz, const double* shapes,
                 int64_t n_shapes, double sigma, uint64_t seed, const int64_t* spots,
                 int64_t n_spots, int spot_val, int threads) {
  const int64_t n = nx * ny * nz;
  memset(out, 0, (size_t)n);
  for (int64_t k = 0; k < n_shapes; ++k) {
    const double* q = shapes + 10 * k;
    const int kind = (int)q[0];
    const double cx = q[1], cy = q[2], cz = q[3], r = q[5], th = q[6];
    const int val = (int)q[4];
    double rx, ry, rz;
    if (kind == 2) {
      rx = q[7] / 2.0; ry = q[8] / 2.0; rz = q[9] / 2.0;
    } else {
      rx = ry = rz = r + (kind == 1 ? th / 2.0 : 0.0);
    }
    int64_t x0 = (int64_t)ceil(cx - rx), x1 = (int64_t)floor(cx + rx);
    int64_t y0 = (int64_t)ceil(cy - ry), y1 = (int64_t)floor(cy + ry);
    int64_t z0 = (int64_t)ceil(cz - rz), z1 = (int64_t)floor(cz + rz);
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    if (x1 > nx - 1) x1 = nx - 1;
    if (y1 > ny - 1) y1 = ny - 1;
    if (z1 > nz - 1) z1 = nz - 1;
    if (x0 > x1 || y0 > y1 || z0 > z1) continue;
    for (int64_t z = z0; z <= z1; ++z)
      for (int64_t y = y0; y <= y1; ++y)
        for (int64_t x = x0; x <= x1; ++x) {
          const double dx = (double)x - cx, dy = (double)y - cy, dz = (double)z - cz;
          int inside;
          if (kind == 2)
            inside = fabs(dx) <= q[7] / 2.0 && fabs(dy) <= q[8] / 2.0 && fabs(dz) <= q[9] / 2.0;
          else {
            const double d2 = (dx * dx + dy * dy) + dz * dz;
            inside = kind == 0 ? d2 <= r * r : fabs(sqrt(d2) - r) <= th / 2.0;
          }
          if (inside) out[(z * ny + y) * nx + x] = (uint8_t)val;
        }
  }
  if (sigma > 0.0) {
    NoiseJob job = {out, n, sigma, seed, 0, PTHREAD_MUTEX_INITIALIZER};
    run_threads(noise_worker, &job, threads);
  }
  for (int64_t k = 0; k < n_spots; ++k) out[spots[k]] = (uint8_t)spot_val;
}

int orc_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}
