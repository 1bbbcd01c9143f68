/* ib_oracle.c — plain fp64 CPU oracle of the immersed-boundary time step.
 *
 * TEST INFRASTRUCTURE ONLY (see ib_oracle.h).  Every function follows PAPER.md §3.2 in the
 * paper's order and notation, with plain loops; no blocking, fusion or reordering beyond
 * what the definitions state.  Build: gcc -O2 -ffp-contract=off -fopenmp (contraction off
 * so that |d| of a link at rest is bitwise the generator's rest length, Z13).
 * OpenMP is used only over independent outputs (pencils, cells), so results are bitwise
 * independent of the thread count; spread and interpolate run serially in point order.
 */
#include "ib_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double PI = 3.14159265358979323846264338327950288;

void ibo_set_threads(int nthreads) {
#ifdef _OPENMP
  omp_set_num_threads(nthreads > 0 ? nthreads : 1);
#else
  (void)nthreads;
#endif
}

int ibo_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ phi, PAPER.md 745-759 */
double ibo_phi(double r) {
  double a = fabs(r);
  if (a <= 1.0) return (3.0 - 2.0 * a + sqrt(1.0 + 4.0 * a - 4.0 * r * r)) / 8.0;
  if (a <= 2.0) return 0.5 - ibo_phi(2.0 - a);
  return 0.0;
}

static inline int64_t wrapi(int64_t j, int32_t N) {
  int64_t m = j % N;
  return m < 0 ? m + N : m;
}

/* ------------------------------------------------------------------ step 1: force */
/* One spring between points i and j: F_i += k (|d| - L0) d/|d|, d = X_j - X_i.
 * |d| = sqrt((dx*dx + dy*dy) + dz*dz) in plain IEEE order (Z13). */
static void spring(const double *X, int64_t i, int64_t j, double k, double L0, double *Fi) {
  double dx = X[3 * j + 0] - X[3 * i + 0];
  double dy = X[3 * j + 1] - X[3 * i + 1];
  double dz = X[3 * j + 2] - X[3 * i + 2];
  double len = sqrt((dx * dx + dy * dy) + dz * dz);
  double t = k * (len - L0) / len;
  Fi[0] += t * dx;
  Fi[1] += t * dy;
  Fi[2] += t * dz;
}

/* Unit normal of a structured patch at point (i1, i2) from the current positions (the
 * window drive "orthogonal to the surface of the window", PAPER.md 988-993): tangents by
 * central differences along i1 and i2 (one-sided at an open patch edge, periodic with the
 * WRAP flags), n = t1 x t2 / |t1 x t2|. */
static void patch_normal(const double *X, int64_t first, int32_t n1, int32_t n2, uint32_t fl,
                         int32_t i1, int32_t i2, double nrm[3]) {
  double t[2][3];
  for (int a = 0; a < 2; ++a) {
    const int32_t n = a == 0 ? n1 : n2, c = a == 0 ? i1 : i2;
    const int wrap = (fl & (a == 0 ? IBO_WRAP1 : IBO_WRAP2)) != 0;
    int32_t cp = c + 1, cm = c - 1;
    if (wrap) { cp %= n; cm = (cm + n) % n; }
    else { if (cp > n - 1) cp = n - 1; if (cm < 0) cm = 0; }
    const int64_t jp = a == 0 ? (int64_t)i2 * n1 + cp : (int64_t)cp * n1 + i1;
    const int64_t jm = a == 0 ? (int64_t)i2 * n1 + cm : (int64_t)cm * n1 + i1;
    for (int d = 0; d < 3; ++d) t[a][d] = X[3 * (first + jp) + d] - X[3 * (first + jm) + d];
  }
  const double cx = t[0][1] * t[1][2] - t[0][2] * t[1][1];
  const double cy = t[0][2] * t[1][0] - t[0][0] * t[1][2];
  const double cz = t[0][0] * t[1][1] - t[0][1] * t[1][0];
  const double len = sqrt((cx * cx + cy * cy) + cz * cz);
  nrm[0] = cx / len; nrm[1] = cy / len; nrm[2] = cz / len;
}

void ibo_force(const double *X, int64_t np, int32_t npatch, const int64_t *first,
               const int32_t *n1v, const int32_t *n2v, const uint32_t *flagsv,
               const int64_t *param_off, const double *stiff,
               int64_t nd, const int64_t *drive_idx, const double *drive_dir,
               double drive_amp, int32_t drive_period, int64_t step, double *Fnode) {
  static const uint32_t fam_flag[4] = {IBO_STRETCH1, IBO_STRETCH2, IBO_BEND1, IBO_BEND2};
  static const int fam_axis[4] = {1, 2, 1, 2};
  static const int fam_off[4] = {1, 1, 2, 2};
  memset(Fnode, 0, sizeof(double) * 3 * (size_t)np);
  for (int32_t p = 0; p < npatch; ++p) {
    const int32_t n1 = n1v[p], n2 = n2v[p];
    const uint32_t fl = flagsv[p];
    const int64_t npts = (int64_t)n1 * n2;
    const double *blk = stiff + param_off[p];
    /* gather form: each point sums its own incident links (fixed order per point) */
    for (int32_t i2 = 0; i2 < n2; ++i2)
      for (int32_t i1 = 0; i1 < n1; ++i1) {
        const int64_t li = (int64_t)i2 * n1 + i1;
        const int64_t gi = first[p] + li;
        double *Fi = Fnode + 3 * gi;
        const double *b = blk;
        for (int f = 0; f < 4; ++f) {
          if (!(fl & fam_flag[f])) continue;
          const double *k = b, *L0 = b + npts;
          b += 2 * npts;
          const int ax = fam_axis[f], off = fam_off[f];
          const int32_t n = ax == 1 ? n1 : n2;
          const int32_t c = ax == 1 ? i1 : i2;
          const int wrap = (fl & (ax == 1 ? IBO_WRAP1 : IBO_WRAP2)) != 0;
          /* forward link (i, i + off), parameters at i */
          int32_t cf = c + off;
          if (cf < n || wrap) {
            cf %= n;
            int64_t lj = ax == 1 ? (int64_t)i2 * n1 + cf : (int64_t)cf * n1 + i1;
            spring(X, gi, first[p] + lj, k[li], L0[li], Fi);
          }
          /* backward link (i - off, i), parameters at i - off */
          int32_t cb = c - off;
          if (cb >= 0 || wrap) {
            cb = (cb % n + n) % n;
            int64_t lj = ax == 1 ? (int64_t)i2 * n1 + cb : (int64_t)cb * n1 + i1;
            spring(X, gi, first[p] + lj, k[lj], L0[lj], Fi);
          }
        }
        if (fl & IBO_TETHER) {   /* F_i += kt (Y_i - X_i) */
          const double *kt = b, *Y = b + npts;
          Fi[0] += kt[li] * (Y[3 * li + 0] - X[3 * gi + 0]);
          Fi[1] += kt[li] * (Y[3 * li + 1] - X[3 * gi + 1]);
          Fi[2] += kt[li] * (Y[3 * li + 2] - X[3 * gi + 2]);
        }
      }
  }
  if (nd > 0 && drive_period > 0) {   /* F += A sin(2 pi n / T) dir, evaluated at t^n */
    double s = drive_amp * sin(2.0 * PI * (double)(step % drive_period) / (double)drive_period);
    for (int64_t d = 0; d < nd; ++d) {
      int64_t i = drive_idx[d];
      double dir[3];
      if (drive_dir) {
        dir[0] = drive_dir[3 * d + 0]; dir[1] = drive_dir[3 * d + 1]; dir[2] = drive_dir[3 * d + 2];
      } else {                          /* surface-normal drive: the normal of i's patch at X^n */
        int32_t p = 0;
        while (p + 1 < npatch && first[p + 1] <= i) ++p;
        const int64_t li = i - first[p];
        patch_normal(X, first[p], n1v[p], n2v[p], flagsv[p], (int32_t)(li % n1v[p]),
                     (int32_t)(li / n1v[p]), dir);
      }
      Fnode[3 * i + 0] += s * dir[0];
      Fnode[3 * i + 1] += s * dir[1];
      Fnode[3 * i + 2] += s * dir[2];
    }
  }
}

/* ------------------------------------------------------------------ step 2: spread */
/* Support of delta_h(x - X) along one axis: lattice indices j = floor(X/h)-1 .. +2
 * (Z8); weights phi((x_j - X)/h), x_j = h j. */
static void weights(double Xa, double h, int64_t *j0, double w[4]) {
  int64_t j = (int64_t)floor(Xa / h) - 1;
  *j0 = j;
  for (int a = 0; a < 4; ++a) w[a] = ibo_phi((h * (double)(j + a) - Xa) / h);
}

void ibo_spread(int32_t N1, int32_t N2, int32_t N3, double h, const double *X,
                const double *Fnode, int64_t np, double *F) {
  const size_t V = (size_t)N1 * N2 * N3;
  const double h3 = h * h * h;
  memset(F, 0, sizeof(double) * 3 * V);
  for (int64_t q = 0; q < np; ++q) {
    int64_t jx, jy, jz;
    double wx[4], wy[4], wz[4];
    weights(X[3 * q + 0], h, &jx, wx);
    weights(X[3 * q + 1], h, &jy, wy);
    weights(X[3 * q + 2], h, &jz, wz);
    for (int c = 0; c < 4; ++c)
      for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) {
          double delta = wx[a] * wy[b] * wz[c] / h3;     /* delta_h(x - X(q)) */
          size_t cell = ((size_t)wrapi(jz + c, N3) * N2 + (size_t)wrapi(jy + b, N2)) * N1 +
                        (size_t)wrapi(jx + a, N1);
          for (int d = 0; d < 3; ++d) F[d * V + cell] += Fnode[3 * q + d] * delta;
        }
  }
}

/* ------------------------------------------------------------------ step 4: interpolate */
void ibo_interp(int32_t N1, int32_t N2, int32_t N3, double h, const double *u, const double *X,
                int64_t np, double *U) {
  const size_t V = (size_t)N1 * N2 * N3;
  for (int64_t q = 0; q < np; ++q) {
    int64_t jx, jy, jz;
    double wx[4], wy[4], wz[4];
    weights(X[3 * q + 0], h, &jx, wx);
    weights(X[3 * q + 1], h, &jy, wy);
    weights(X[3 * q + 2], h, &jz, wz);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < 4; ++c)
      for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) {
          double w = wx[a] * wy[b] * wz[c];               /* delta_h h^3 */
          size_t cell = ((size_t)wrapi(jz + c, N3) * N2 + (size_t)wrapi(jy + b, N2)) * N1 +
                        (size_t)wrapi(jx + a, N1);
          for (int d = 0; d < 3; ++d) acc[d] += u[d * V + cell] * w;
        }
    U[3 * q + 0] = acc[0];
    U[3 * q + 1] = acc[1];
    U[3 * q + 2] = acc[2];
  }
}

/* ------------------------------------------------------------------ step 3: fluid */
void ibo_advect(int32_t N1, int32_t N2, int32_t N3, double h, const double *u, double *adv) {
  const int64_t V = (int64_t)N1 * N2 * N3;
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < N3; ++z)
    for (int64_t y = 0; y < N2; ++y)
      for (int64_t x = 0; x < N1; ++x) {
        const int64_t c0 = (z * N2 + y) * N1 + x;
        /* neighbours x +- h e_k, periodic */
        const int64_t nb_m[3] = {(z * N2 + y) * N1 + (x + N1 - 1) % N1,
                                 (z * N2 + (y + N2 - 1) % N2) * N1 + x,
                                 (((z + N3 - 1) % N3) * N2 + y) * N1 + x};
        const int64_t nb_p[3] = {(z * N2 + y) * N1 + (x + 1) % N1,
                                 (z * N2 + (y + 1) % N2) * N1 + x,
                                 (((z + 1) % N3) * N2 + y) * N1 + x};
        for (int i = 0; i < 3; ++i) {
          const double *ui = u + i * V;
          double s = 0.0;
          for (int k = 0; k < 3; ++k) {
            double uk = u[k * V + c0];
            double d;
            if (uk > 0.0)       d = (ui[c0] - ui[nb_m[k]]) / h;   /* D_k^- */
            else if (uk < 0.0)  d = (ui[nb_p[k]] - ui[c0]) / h;   /* D_k^+ */
            else                d = (ui[c0] - ui[nb_m[k]]) / h;   /* Z5: backward */
            s += uk * d;
          }
          adv[i * V + c0] = s;
        }
      }
}

void ibo_rhs(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double dt,
             const double *u, const double *F, double *r) {
  const int64_t V = (int64_t)N1 * N2 * N3;
  double *adv = (double *)malloc(sizeof(double) * 3 * (size_t)V);
  ibo_advect(N1, N2, N3, h, u, adv);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < 3 * V; ++c) r[c] = rho * u[c] / dt - rho * adv[c] + F[c];
  free(adv);
}

/* Radix-2 decimation-in-time FFT of one length-N pencil (bit reversal, then butterflies).
 * tw[j] = e^{sign 2 pi i j / N}, j < N/2. */
static void fft1(int32_t N, double *re, double *im, const double *twr, const double *twi) {
  for (int32_t i = 1, j = 0; i < N; ++i) {
    int32_t bit = N >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double t = re[i]; re[i] = re[j]; re[j] = t;
      t = im[i]; im[i] = im[j]; im[j] = t;
    }
  }
  for (int32_t len = 2; len <= N; len <<= 1) {
    const int32_t half = len >> 1, step = N / len;
    for (int32_t s = 0; s < N; s += len)
      for (int32_t k = 0; k < half; ++k) {
        double wr = twr[k * step], wi = twi[k * step];
        double ar = re[s + k], ai = im[s + k];
        double br = re[s + k + half], bi = im[s + k + half];
        double tr = wr * br - wi * bi, ti = wr * bi + wi * br;
        re[s + k] = ar + tr;        im[s + k] = ai + ti;
        re[s + k + half] = ar - tr; im[s + k + half] = ai - ti;
      }
  }
}

void ibo_fft3(int32_t N1, int32_t N2, int32_t N3, double *re, double *im, int sign) {
  const int32_t L[3] = {N1, N2, N3};
  const int64_t stride[3] = {1, N1, (int64_t)N1 * N2};
  for (int ax = 0; ax < 3; ++ax) {
    const int32_t N = L[ax];
    const int64_t s = stride[ax];
    /* the two other axes enumerate the pencils */
    const int a1 = (ax + 1) % 3, a2 = (ax + 2) % 3;
    const int64_t s1 = stride[a1], s2 = stride[a2], n1 = L[a1], n2 = L[a2];
    double *twr = (double *)malloc(sizeof(double) * (size_t)(N / 2 + 1));
    double *twi = (double *)malloc(sizeof(double) * (size_t)(N / 2 + 1));
    for (int32_t j = 0; j < N / 2 + 1; ++j) {
      twr[j] = cos(2.0 * PI * (double)j / (double)N);
      twi[j] = (double)sign * sin(2.0 * PI * (double)j / (double)N);
    }
#pragma omp parallel
    {
      double *pr = (double *)malloc(sizeof(double) * (size_t)N);
      double *pi = (double *)malloc(sizeof(double) * (size_t)N);
#pragma omp for schedule(static)
      for (int64_t pencil = 0; pencil < n1 * n2; ++pencil) {
        int64_t base = (pencil % n1) * s1 + (pencil / n1) * s2;
        for (int32_t j = 0; j < N; ++j) { pr[j] = re[base + j * s]; pi[j] = im[base + j * s]; }
        fft1(N, pr, pi, twr, twi);
        for (int32_t j = 0; j < N; ++j) { re[base + j * s] = pr[j]; im[base + j * s] = pi[j]; }
      }
      free(pr);
      free(pi);
    }
    free(twr);
    free(twi);
  }
}

/* Per-mode solve (DESIGN.md §2 S3c; readings Z6, Z7, Z22):
 *   d(k) = rho/dt + mu * sum_a 4 sin^2(pi k_a/N)/h^2      (symbol of -mu sum D+D-)
 *   s_a  = sin(2 pi k'_a/N)/h, exactly 0 when 2 k_a = 0 mod N   (D0 symbol = i s)
 *   p^   = -i (s.r^)/|s|^2,  u^ = (r^ - s (s.r^)/|s|^2)/d;   null modes: u^ = r^/d, p^ = 0. */
/* per-axis symbols of one lattice axis of length N (readings Z22) */
static void axis_symbols(int32_t N, double h, double *sk, double *lk, int *nul) {
  for (int32_t k = 0; k < N; ++k) {
    int32_t ks = k > N / 2 ? k - N : k;                 /* signed frequency k' */
    nul[k] = (2 * k) % N == 0;                          /* decided on the integers */
    sk[k] = nul[k] ? 0.0 : sin(2.0 * PI * (double)ks / (double)N) / h;
    double sn = sin(PI * (double)k / (double)N);
    lk[k] = 4.0 * sn * sn / (h * h);
  }
}

void ibo_solve(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu, double dt,
               const double *r, double *u_out, double *p_out) {
  const int64_t V = (int64_t)N1 * N2 * N3;
  double *re = (double *)malloc(sizeof(double) * 3 * (size_t)V);
  double *im = (double *)calloc(3 * (size_t)V, sizeof(double));
  double *pre = p_out ? (double *)calloc((size_t)V, sizeof(double)) : NULL;
  double *pim = p_out ? (double *)calloc((size_t)V, sizeof(double)) : NULL;
  memcpy(re, r, sizeof(double) * 3 * (size_t)V);
  for (int c = 0; c < 3; ++c) ibo_fft3(N1, N2, N3, re + c * V, im + c * V, -1);

  double *sx = (double *)malloc(sizeof(double) * (size_t)N1), *lx = (double *)malloc(sizeof(double) * (size_t)N1);
  double *sy = (double *)malloc(sizeof(double) * (size_t)N2), *ly = (double *)malloc(sizeof(double) * (size_t)N2);
  double *sz = (double *)malloc(sizeof(double) * (size_t)N3), *lz = (double *)malloc(sizeof(double) * (size_t)N3);
  int *nx = (int *)malloc(sizeof(int) * (size_t)N1), *ny = (int *)malloc(sizeof(int) * (size_t)N2);
  int *nz = (int *)malloc(sizeof(int) * (size_t)N3);
  axis_symbols(N1, h, sx, lx, nx);
  axis_symbols(N2, h, sy, ly, ny);
  axis_symbols(N3, h, sz, lz, nz);
#pragma omp parallel for schedule(static)
  for (int64_t kz = 0; kz < N3; ++kz)
    for (int64_t ky = 0; ky < N2; ++ky)
      for (int64_t kx = 0; kx < N1; ++kx) {
        const int64_t m = (kz * N2 + ky) * N1 + kx;
        const double d = rho / dt + mu * (lx[kx] + ly[ky] + lz[kz]);
        const double s[3] = {sx[kx], sy[ky], sz[kz]};
        double rr[3], ri[3];
        for (int c = 0; c < 3; ++c) { rr[c] = re[c * V + m]; ri[c] = im[c * V + m]; }
        if (nx[kx] && ny[ky] && nz[kz]) {
          for (int c = 0; c < 3; ++c) { re[c * V + m] = rr[c] / d; im[c * V + m] = ri[c] / d; }
          if (p_out) { pre[m] = 0.0; pim[m] = 0.0; }
          continue;
        }
        double s2 = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
        double sr = s[0] * rr[0] + s[1] * rr[1] + s[2] * rr[2];
        double si = s[0] * ri[0] + s[1] * ri[1] + s[2] * ri[2];
        for (int c = 0; c < 3; ++c) {
          re[c * V + m] = (rr[c] - s[c] * sr / s2) / d;
          im[c * V + m] = (ri[c] - s[c] * si / s2) / d;
        }
        if (p_out) { pre[m] = si / s2; pim[m] = -sr / s2; }   /* -i (sr + i si)/s2 */
      }
  free(sx); free(lx); free(sy); free(ly); free(sz); free(lz); free(nx); free(ny); free(nz);

  const double inv = 1.0 / (double)V;
  for (int c = 0; c < 3; ++c) ibo_fft3(N1, N2, N3, re + c * V, im + c * V, +1);
  for (int64_t i = 0; i < 3 * V; ++i) u_out[i] = re[i] * inv;
  if (p_out) {
    ibo_fft3(N1, N2, N3, pre, pim, +1);
    for (int64_t i = 0; i < V; ++i) p_out[i] = pre[i] * inv;
    free(pre); free(pim);
  }
  free(re); free(im);
}

void ibo_fluid_step(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu,
                    double dt, const double *u, const double *F, double *u_out, double *p_out) {
  const size_t V = (size_t)N1 * N2 * N3;
  double *r = (double *)malloc(sizeof(double) * 3 * V);
  ibo_rhs(N1, N2, N3, h, rho, dt, u, F, r);
  ibo_solve(N1, N2, N3, h, rho, mu, dt, r, u_out, p_out);
  free(r);
}

/* ------------------------------------------------------------------ the time loop */
int ibo_step(int32_t N1, int32_t N2, int32_t N3, double h, double rho, double mu, double dt,
             double *u, double *p, double *X, int64_t np, int32_t npatch, const int64_t *first,
             const int32_t *n1, const int32_t *n2, const uint32_t *flags,
             const int64_t *param_off, const double *stiff, int64_t nd,
             const int64_t *drive_idx, const double *drive_dir, double drive_amp,
             int32_t drive_period, int64_t step0, int32_t nsteps, int32_t p_every,
             const uint8_t *fixed) {
  const size_t V = (size_t)N1 * N2 * N3;
  double *Fn = (double *)malloc(sizeof(double) * 3 * (size_t)(np > 0 ? np : 1));
  double *U = (double *)malloc(sizeof(double) * 3 * (size_t)(np > 0 ? np : 1));
  double *F = (double *)malloc(sizeof(double) * 3 * V);
  double *un = (double *)malloc(sizeof(double) * 3 * V);
  int status = 0;
  for (int32_t s = 0; s < nsteps && !status; ++s) {
    const int64_t n = step0 + s;
    ibo_force(X, np, npatch, first, n1, n2, flags, param_off, stiff, nd, drive_idx,
              drive_dir, drive_amp, drive_period, n, Fn);              /* step 1 */
    ibo_spread(N1, N2, N3, h, X, Fn, np, F);                            /* step 2 */
    double *ps = (p && (p_every || s == nsteps - 1)) ? p + (p_every ? (size_t)s * V : 0) : NULL;
    ibo_fluid_step(N1, N2, N3, h, rho, mu, dt, u, F, un, ps);           /* step 3 */
    ibo_interp(N1, N2, N3, h, un, X, np, U);                            /* step 4 */
    for (int64_t q = 0; q < np; ++q)                                    /* eq:discreteX */
      if (!(fixed && fixed[q]))                      /* fixed points never move (PAPER.md 919-920) */
        for (int d = 0; d < 3; ++d) X[3 * q + d] = X[3 * q + d] + dt * U[3 * q + d];
    memcpy(u, un, sizeof(double) * 3 * V);
    for (int64_t i = 0; i < 3 * np && !status; ++i) if (!isfinite(X[i])) status = 1 + s;
    for (size_t i = 0; i < 3 * V && !status; ++i) if (!isfinite(u[i])) status = 1 + s;
  }
  free(Fn); free(U); free(F); free(un);
  return status;
}
