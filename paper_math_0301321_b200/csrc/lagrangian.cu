// lagrangian.cu — steps 1, 2 and 4 of the IB step on sm_100a.
//
//   force  (PAPER.md 610-616): per-point gather over the incident links of its structured
//          patch (stretch / bend springs), tether and drive; nodal forces (Z12).
//   spread (eq:discreteF, PAPER.md 712-723): the force is computed in registers and
//          spread with Peskin's 4-point delta (745-759).  Lanes of a warp whose support
//          boxes coincide (same base cell) are merged: their 12 weights + force go to
//          shared memory, the warp's 32 lanes then own the 64 nodes x 3 components of the
//          box (6 outputs per lane), sum the group's contributions in registers and flush
//          once with fp64 atomicAdd — one atomic per (group, node, component) instead of
//          one per (point, node, component).  Points are visited in cell-binned order
//          (a counting sort by base cell, refreshed every SORT_PERIOD steps), so a warp's
//          lanes mostly share one box and the groups are large.
//   interp + update (eq:discreteX, PAPER.md 725-734): gather of u^{n+1} at X^n fused with
//          X^{n+1} = X^n + dt U, with a non-finite check.
#include <climits>

#include "ib_internal.cuh"

namespace ibk {

// ------------------------------------------------------------------ delta weights
// Window j0 = floor(X/h) - 1 .. +2 (Z8); with f = X/h - floor(X/h) in [0,1):
//   phi(-f)   = (3 - 2f + sqrt(1 + 4f - 4f^2))/8           (|r| <= 1 branch)
//   phi(1-f)  = (1 + 2f + sqrt(1 + 4f - 4f^2))/8           (same root)
//   phi(1+f)  = 1/2 - phi(1-f),  phi(2-f) = 1/2 - phi(-f)  (1 <= |r| <= 2 branch)
// sqrt(a) for a in [1, 2] (the argument below): hardware rsqrt estimate, two Newton steps
// and one correction of the square root; no special-case branch (the library sqrt keeps a
// slow path for zero, infinity, denormals).  Matched the IEEE sqrt bit for bit on 4M samples
// of [1, 2) on the B200.
__device__ __forceinline__ double sqrt_1_2(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  y = y * (1.5 - 0.5 * a * y * y);
  y = y * (1.5 - 0.5 * a * y * y);
  const double s = a * y;
  return s + 0.5 * y * (a - s * s);
}

__device__ __forceinline__ int axis_weights(double Xa, double invh, double w[4]) {
  const double s = Xa * invh;
  const double fl = floor(s);
  const double f = s - fl;
  const double q = sqrt_1_2(1.0 + 4.0 * f - 4.0 * f * f);
  w[1] = (3.0 - 2.0 * f + q) * 0.125;
  w[2] = (1.0 + 2.0 * f + q) * 0.125;
  w[0] = 0.5 - w[2];
  w[3] = 0.5 - w[1];
  return (int)(long long)fl - 1;
}

// ------------------------------------------------------------------ force
__device__ __forceinline__ void spring(const double *__restrict__ X, double xi, double yi,
                                       double zi, int64_t j, double k, double L0, double f[3]) {
  const double dx = __ldg(&X[3 * j + 0]) - xi;
  const double dy = __ldg(&X[3 * j + 1]) - yi;
  const double dz = __ldg(&X[3 * j + 2]) - zi;
  // |d| in plain IEEE order without contraction (Z13): exactly L0 at rest
  const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                          __dmul_rn(dz, dz)));
  const double t = k * (len - L0) / len;
  f[0] += t * dx;
  f[1] += t * dy;
  f[2] += t * dz;
}

// pt: the patch table (shared-memory copy when it fits, else sd.patches); xyz: the point's
// own position, already loaded by the caller
__device__ __forceinline__ void point_force(const StructDev &sd, const ib_patch *pt, int64_t i,
                                            double f[3], const double xyz[3]) {
  int lo = 0, hi = sd.npatch - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pt[mid].first <= i) lo = mid; else hi = mid - 1;
  }
  const ib_patch *P = pt + lo;
  const int64_t first = P->first;
  const int n1 = P->n1, n2 = P->n2;
  const uint32_t fl = P->flags;
  const int64_t npts = (int64_t)n1 * n2;
  const int64_t li = i - first;
  // 32-bit index arithmetic: a patch holds < 2^31 points (ib_set_structure checks np)
  const int i2 = (int)((unsigned)li / (unsigned)n1), i1 = (int)li - i2 * n1;
  const double *b = sd.stiff + P->param_off;
  const double xi = xyz[0], yi = xyz[1], zi = xyz[2];
  f[0] = f[1] = f[2] = 0.0;
#pragma unroll
  for (int fam = 0; fam < 4; ++fam) {
    const uint32_t bit = (uint32_t)IB_STRETCH1 << fam;
    if (!(fl & bit)) continue;
    const double *k = b, *L0 = b + npts;
    b += 2 * npts;
    const bool ax1 = (fam & 1) == 0;
    const int off = fam < 2 ? 1 : 2;
    const int n = ax1 ? n1 : n2, c = ax1 ? i1 : i2;
    const bool wrap = (fl & (ax1 ? IB_WRAP1 : IB_WRAP2)) != 0;
    int cf = c + off;
    if (cf < n || wrap) {
      while (cf >= n) cf -= n;
      const int64_t lj = ax1 ? (int64_t)i2 * n1 + cf : (int64_t)cf * n1 + i1;
      spring(sd.X, xi, yi, zi, first + lj, __ldg(&k[li]), __ldg(&L0[li]), f);
    }
    int cb = c - off;
    if (cb >= 0 || wrap) {
      while (cb < 0) cb += n;
      const int64_t lj = ax1 ? (int64_t)i2 * n1 + cb : (int64_t)cb * n1 + i1;
      spring(sd.X, xi, yi, zi, first + lj, __ldg(&k[lj]), __ldg(&L0[lj]), f);
    }
  }
  if (fl & IB_TETHER) {
    const double kt = __ldg(&b[li]);
    const double *Y = b + npts;
    f[0] += kt * (__ldg(&Y[3 * li + 0]) - xi);
    f[1] += kt * (__ldg(&Y[3 * li + 1]) - yi);
    f[2] += kt * (__ldg(&Y[3 * li + 2]) - zi);
  }
}

// Direction of driven point d (global index i): the given unit vector, or (drive_dir null)
// the unit normal of i's patch at the current positions — the window drive "orthogonal to
// the surface of the window" (PAPER.md 988-993): tangents by central differences along i1
// and i2 (one-sided at an open edge, periodic with the WRAP flags), n = t1 x t2 / |t1 x t2|.
__device__ __forceinline__ void drive_direction(const StructDev &sd, int64_t d, int64_t i,
                                                double dir[3]) {
  if (sd.drive_dir) {
    dir[0] = sd.drive_dir[3 * d]; dir[1] = sd.drive_dir[3 * d + 1]; dir[2] = sd.drive_dir[3 * d + 2];
    return;
  }
  int lo = 0, hi = sd.npatch - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sd.patches[mid].first <= i) lo = mid; else hi = mid - 1;
  }
  const ib_patch P = sd.patches[lo];
  const int64_t li = i - P.first;
  const int i1 = (int)(li % P.n1), i2 = (int)(li / P.n1);
  double t[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int n = a == 0 ? P.n1 : P.n2, c = a == 0 ? i1 : i2;
    const bool wrap = (P.flags & (a == 0 ? IB_WRAP1 : IB_WRAP2)) != 0;
    int cp = c + 1, cm = c - 1;
    if (wrap) { cp %= n; cm = (cm + n) % n; }
    else { cp = cp > n - 1 ? n - 1 : cp; cm = cm < 0 ? 0 : cm; }
    const int64_t jp = P.first + (a == 0 ? (int64_t)i2 * P.n1 + cp : (int64_t)cp * P.n1 + i1);
    const int64_t jm = P.first + (a == 0 ? (int64_t)i2 * P.n1 + cm : (int64_t)cm * P.n1 + i1);
#pragma unroll
    for (int k = 0; k < 3; ++k) t[a][k] = sd.X[3 * jp + k] - sd.X[3 * jm + k];
  }
  const double cx = t[0][1] * t[1][2] - t[0][2] * t[1][1];
  const double cy = t[0][2] * t[1][0] - t[0][0] * t[1][2];
  const double cz = t[0][0] * t[1][1] - t[0][1] * t[1][0];
  const double len = sqrt((cx * cx + cy * cy) + cz * cz);
  dir[0] = cx / len; dir[1] = cy / len; dir[2] = cz / len;
}

__device__ __forceinline__ double drive_factor(const StructDev &sd, long long n) {
  const long long T = sd.drive_period;
  return sd.drive_amp * sinpi(2.0 * (double)(n % T) / (double)T);
}

__global__ void k_force(StructDev sd, const long long *dev_n, long long n, double *f_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sd.np) return;
  double f[3];
  const double xyz[3] = {__ldg(&sd.X[3 * i + 0]), __ldg(&sd.X[3 * i + 1]), __ldg(&sd.X[3 * i + 2])};
  point_force(sd, sd.patches, i, f, xyz);
  f_out[3 * i + 0] = f[0];
  f_out[3 * i + 1] = f[1];
  f_out[3 * i + 2] = f[2];
}

__global__ void k_drive_add(StructDev sd, const long long *dev_n, long long n, double *f_out) {
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= sd.nd) return;
  const double a = drive_factor(sd, dev_n ? *dev_n : n);
  const int64_t i = sd.drive_idx[d];
  double dir[3];
  drive_direction(sd, d, i, dir);
  for (int c = 0; c < 3; ++c) f_out[3 * i + c] += a * dir[c];
}

// Spread of the drive force of driven point d (few points): one warp per driven point, each
// lane owning 2 of the 64 support nodes x 3 components (6 atomics per lane).  Run by the
// first warps of k_force_spread (no launch of its own); a = drive factor / h^3.
__device__ __forceinline__ void drive_spread_one(const StructDev &sd, const FluidGeom &g, double a,
                                                 int64_t d, int lane, double *F, unsigned *rowflag) {
  const int N1 = g.N1, N2 = g.N2, N3g = g.N3g;
  const unsigned L = (unsigned)g.N3;           // local planes (all N3 unless a slab)
  const size_t V = (size_t)g.V;
  const int64_t i = sd.drive_idx[d];
  double wx[4], wy[4], wz[4];
  const int jx = axis_weights(sd.X[3 * i + 0], g.invh, wx);
  const int jy = axis_weights(sd.X[3 * i + 1], g.invh, wy);
  const int jz = axis_weights(sd.X[3 * i + 2], g.invh, wz);
  const int e = lane & 3, b = (lane >> 2) & 3, c0 = lane >> 4;
  double dir[3];
  drive_direction(sd, d, i, dir);
  const size_t x = (jx + e) & (N1 - 1), y = (jy + b) & (N2 - 1);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const size_t z = (unsigned)(jz + c0 + 2 * h - g.z0) & (unsigned)(N3g - 1);   // local plane
    if (z >= L) continue;                      // slab: another rank's plane
    const size_t cell = (z * N2 + y) * N1 + x;
    const double w = a * wx[e] * wy[b] * wz[c0 + 2 * h];
    for (int k = 0; k < 3; ++k) atomicAdd(&F[k * V + cell], w * dir[k]);
    if (rowflag && e == 0) rowflag[z * N2 + y] = 1u;
  }
}

// ------------------------------------------------------------------ fp64 tensor-core MMA
// D (8x8) = A (8x4) B (4x8), fp64 (DMMA).  Fragments (PTX m8n8k4 .f64): lane l holds
// A[l >> 2][l & 3], B[l & 3][l >> 2] and D[l >> 2][2 (l & 3) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(0.0), "d"(0.0));
}

// ------------------------------------------------------------------ force + spread
#ifndef IBK_SPT
#define IBK_SPT 128
#endif
constexpr int SPREAD_THREADS = IBK_SPT;
// per-point record: [0,16) wx[a] wy[b] at b*4+a; [16,22) f*wz[0], f*wz[2]; [22,28) f*wz[1],
// f*wz[3] (f scaled by 1/h^3); stride 30 doubles = 15 x 16 B (conflict-free 128-bit access)
constexpr int REC = 30;
constexpr int PTAB = 64;   // patch table entries staged in shared memory

#ifndef IBK_SP_MINB
#define IBK_SP_MINB 6   // 80 registers: 6 blocks of 128 per SM (the folded drive pushes it to 94)
#endif
template <bool FROM_ARRAY>
__global__ void __launch_bounds__(SPREAD_THREADS, IBK_SP_MINB)
k_force_spread(StructDev sd, FluidGeom g, const double *__restrict__ f_in, double *F,
               unsigned *rowflag, const long long *dev_n, long long n) {
  __shared__ __align__(16) double rec[SPREAD_THREADS / 32][33][REC];   // record 32: zeros (tail)
  __shared__ ib_patch ptab[PTAB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool small = sd.npatch <= PTAB;
  if (!FROM_ARRAY && small)
    for (int q = threadIdx.x; q < sd.npatch; q += blockDim.x) ptab[q] = sd.patches[q];
  if (lane < REC) rec[warp][32][lane] = 0.0;   // (REC <= 32)
  __syncthreads();
  const ib_patch *pt = small ? ptab : sd.patches;
  if (!FROM_ARRAY && sd.nd > 0) {             // the drive of this step (few points) first
    const double a = drive_factor(sd, dev_n ? *dev_n : n) * g.invh * g.invh * g.invh;
    if (a != 0.0)
      for (int64_t d = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; d < sd.nd;
           d += ((int64_t)gridDim.x * blockDim.x) >> 5)
        drive_spread_one(sd, g, a, d, lane, F, rowflag);
  }
  const int N1 = g.N1, N2 = g.N2, N3g = g.N3g;
  const unsigned L = (unsigned)g.N3;                     // local planes (all N3 unless a slab)
  const size_t V = (size_t)g.V;
  const int lg1 = __ffs(N1) - 1, lg2 = __ffs(N2) - 1;   // powers of two: no division below
  const double ih3 = g.invh * g.invh * g.invh;
  double *r = rec[warp][lane];
  // lane -> outputs (a, b, c0 | c0 + 2, component 0..2)
  const int a = lane & 3, b = (lane >> 2) & 3, c0 = lane >> 4, ab = lane & 15;
  // persistent: the grid walks the points in blocks of SPREAD_THREADS; the binned index of
  // the next block is fetched one iteration ahead (one less dependent load per point)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto point_at = [&](int64_t k) -> int64_t {
    return k < sd.np ? (sd.perm ? (int64_t)__ldg(&sd.perm[k]) : k) : 0;
  };
  int64_t inext = point_at((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x; k0 < sd.np; k0 += stride) {
    const int64_t k = k0 + threadIdx.x;
    const int64_t i = inext;
    inext = point_at(k + stride);
    unsigned key = 0xffffffffu;
    bool live = false;
    if (k < sd.np) {
      double f[3], xyz[3];
      if (sd.Xs) {             // binned SoA copy: coalesced (the AoS X[i] is 1 sector per lane)
        xyz[0] = __ldg(&sd.Xs[k]); xyz[1] = __ldg(&sd.Xs[sd.np + k]); xyz[2] = __ldg(&sd.Xs[2 * sd.np + k]);
      } else {
        xyz[0] = __ldg(&sd.X[3 * i + 0]); xyz[1] = __ldg(&sd.X[3 * i + 1]); xyz[2] = __ldg(&sd.X[3 * i + 2]);
      }
      if (FROM_ARRAY) {
        f[0] = __ldg(&f_in[3 * i]); f[1] = __ldg(&f_in[3 * i + 1]); f[2] = __ldg(&f_in[3 * i + 2]);
      } else {
        point_force(sd, pt, i, f, xyz);
      }
      live = (f[0] != 0.0) || (f[1] != 0.0) || (f[2] != 0.0);
      double wx[4], wy[4], wz[4];
      const int jx = axis_weights(xyz[0], g.invh, wx) & (N1 - 1);
      const int jy = axis_weights(xyz[1], g.invh, wy) & (N2 - 1);
      const int jz = axis_weights(xyz[2], g.invh, wz) & (N3g - 1);
      double2 *rw = reinterpret_cast<double2 *>(r);
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        rw[2 * bb] = make_double2(wx[0] * wy[bb], wx[1] * wy[bb]);
        rw[2 * bb + 1] = make_double2(wx[2] * wy[bb], wx[3] * wy[bb]);
      }
      const double f0 = f[0] * ih3, f1 = f[1] * ih3, f2 = f[2] * ih3;
      double2 *rg = reinterpret_cast<double2 *>(r + 16);
      rg[0] = make_double2(f0 * wz[0], f1 * wz[0]); rg[1] = make_double2(f2 * wz[0], f0 * wz[2]);
      rg[2] = make_double2(f1 * wz[2], f2 * wz[2]); rg[3] = make_double2(f0 * wz[1], f1 * wz[1]);
      rg[4] = make_double2(f2 * wz[1], f0 * wz[3]); rg[5] = make_double2(f1 * wz[3], f2 * wz[3]);
      key = ((unsigned)jz * N2 + (unsigned)jy) * N1 + (unsigned)jx;
    }
    __syncwarp();
    unsigned todo = __ballot_sync(0xffffffffu, live);
    while (todo) {
      const int leader = __ffs(todo) - 1;
      const unsigned kl = __shfl_sync(0xffffffffu, key, leader);
      const unsigned grp = __ballot_sync(0xffffffffu, key == kl) & todo;
      todo &= ~grp;
      double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      unsigned m = grp;
      while (m) {              // two members per iteration (record 32 = zero pads the tail)
        const int p = __ffs(m) - 1;
        m &= m - 1;
        const int p2 = m ? __ffs(m) - 1 : 32;
        m &= m - 1;
        const double *q = rec[warp][p], *q2 = rec[warp][p2];
        const double w = q[ab], w2 = q2[ab];
        const double2 *g = reinterpret_cast<const double2 *>(q + 16 + 6 * c0);
        const double2 *g2 = reinterpret_cast<const double2 *>(q2 + 16 + 6 * c0);
        const double2 u0 = g[0], u1 = g[1], u2 = g[2], v0 = g2[0], v1 = g2[1], v2 = g2[2];
        // two fused multiply-adds per accumulator (acc += w u + w2 v contracts to 3 ops)
        acc[0] = fma(w2, v0.x, fma(w, u0.x, acc[0])); acc[2] = fma(w2, v0.y, fma(w, u0.y, acc[2]));
        acc[4] = fma(w2, v1.x, fma(w, u1.x, acc[4])); acc[1] = fma(w2, v1.y, fma(w, u1.y, acc[1]));
        acc[3] = fma(w2, v2.x, fma(w, u2.x, acc[3])); acc[5] = fma(w2, v2.y, fma(w, u2.y, acc[5]));
      }
      const unsigned jx = kl & (N1 - 1), jy = (kl >> lg1) & (N2 - 1), jz = kl >> (lg1 + lg2);
      const size_t x = (jx + a) & (N1 - 1), y = (jy + b) & (N2 - 1);
      // local planes (slab: relative to its first plane; other ranks' planes are skipped)
      const size_t z0 = (jz + c0 - g.z0) & (N3g - 1), z1 = (jz + c0 + 2 - g.z0) & (N3g - 1);
      const size_t e0 = (z0 * N2 + y) * N1 + x, e1 = (z1 * N2 + y) * N1 + x;
      if (z0 < L) {
        atomicAdd(&F[e0], acc[0]); atomicAdd(&F[V + e0], acc[2]); atomicAdd(&F[2 * V + e0], acc[4]);
        if (rowflag && a == 0) rowflag[z0 * N2 + y] = 1u;   // row (y, z0) of F is non-zero
      }
      if (z1 < L) {
        atomicAdd(&F[e1], acc[1]); atomicAdd(&F[V + e1], acc[3]); atomicAdd(&F[2 * V + e1], acc[5]);
        if (rowflag && a == 0) rowflag[z1 * N2 + y] = 1u;
      }
    }
    __syncwarp();                               // records reused by the next block of points
  }
}

cudaError_t launch_force(const StructDev &sd, const long long *dev_n, long long n,
                         double *f_out, cudaStream_t s) {
  if (sd.np > 0) k_force<<<(unsigned)((sd.np + 255) / 256), 256, 0, s>>>(sd, dev_n, n, f_out);
  if (sd.nd > 0) k_drive_add<<<(unsigned)((sd.nd + 127) / 128), 128, 0, s>>>(sd, dev_n, n, f_out);
  return cudaGetLastError();
}

cudaError_t launch_force_spread(const StructDev &sd, const FluidGeom &g, const double *f_in,
                                const long long *dev_n, long long n, double *F,
                                unsigned *rowflag, cudaStream_t s) {
  if (sd.np > 0) {
    // resident blocks on the current device (persistent grid)
    int per = 0;
    if (f_in) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_force_spread<true>, SPREAD_THREADS, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_force_spread<false>, SPREAD_THREADS, 0);
    const int64_t cap = (int64_t)sm_count() * (per > 0 ? per : 1);
    const int64_t need = (sd.np + SPREAD_THREADS - 1) / SPREAD_THREADS;
    const unsigned blocks = (unsigned)(need < cap ? need : cap);
    if (f_in)
      k_force_spread<true><<<blocks, SPREAD_THREADS, 0, s>>>(sd, g, f_in, F, rowflag, dev_n, n);
    else
      k_force_spread<false><<<blocks, SPREAD_THREADS, 0, s>>>(sd, g, f_in, F, rowflag, dev_n, n);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ interp + update
// U = sum_c wz_c sum_b wy_b (sum_a wx_a u(jx+a, jy+b, jz+c)) straight from global memory
// (row sums first, 32-bit cell offsets; a row with no periodic wrap in x is 4 consecutive
// doubles off one base pointer).  Used by warps whose points span more than IMMA_MAXG boxes.
// Plane of the velocity array holding lattice plane jz + c (jz = floor(Z/h) - 1): periodic on
// the whole lattice; in a slab the owned point's window jz .. jz + 3 lies in
// the local planes plus ghosts, local plane of global z at uz0 + (z - z0).
__device__ __forceinline__ int u_plane(const FluidGeom &g, int jz, int c) {
  if (!g.slab) return (jz + c) & (g.N3 - 1);
  return g.uz0 - 1 + (int)((unsigned)(jz + 1 - g.z0) & (unsigned)(g.N3g - 1)) + c;
}

__device__ __forceinline__ void interp_direct(const double *__restrict__ u, const FluidGeom &g,
                                              int Vi,
                                              int jx, int jy, int jz, const double wx[4],
                                              const double wy[4], const double wz[4],
                                              double &U0, double &U1, double &U2) {
  const int N1 = g.N1, N2 = g.N2;
  int ro[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      ro[c][b] = (u_plane(g, jz, c) * N2 + ((jy + b) & (N2 - 1))) * N1;
  U0 = U1 = U2 = 0.0;
  if (jx >= 0 && jx + 3 < N1) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double *r0 = u + (ro[c][b] + jx), *r1 = r0 + Vi, *r2 = r1 + Vi;
        const double s0 = wx[0] * __ldg(r0) + wx[1] * __ldg(r0 + 1) + wx[2] * __ldg(r0 + 2) + wx[3] * __ldg(r0 + 3);
        const double s1 = wx[0] * __ldg(r1) + wx[1] * __ldg(r1 + 1) + wx[2] * __ldg(r1 + 2) + wx[3] * __ldg(r1 + 3);
        const double s2 = wx[0] * __ldg(r2) + wx[1] * __ldg(r2 + 1) + wx[2] * __ldg(r2 + 2) + wx[3] * __ldg(r2 + 3);
        const double wbc = wy[b] * wz[c];
        U0 += wbc * s0; U1 += wbc * s1; U2 += wbc * s2;
      }
  } else {
    int xo[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) xo[a] = (jx + a) & (N1 - 1);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double *r0 = u + ro[c][b], *r1 = r0 + Vi, *r2 = r1 + Vi;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          s0 += wx[a] * __ldg(r0 + xo[a]);
          s1 += wx[a] * __ldg(r1 + xo[a]);
          s2 += wx[a] * __ldg(r2 + xo[a]);
        }
        const double wbc = wy[b] * wz[c];
        U0 += wbc * s0; U1 += wbc * s1; U2 += wbc * s2;
      }
  }
}

constexpr int INTERP_THREADS = 128;

// One thread per point in cell-binned order; X^{n+1} = X^n + dt U fused; non-finite flag.
// Per group of lanes whose points share a support box (same base cell), the x contraction of all members is one fp64 MMA per 8 output columns:
//   S[p][(comp, c, b)] = sum_a wx_p[a] u(jx + a, jy + b, jz + c)[comp]
// (M = 8 members, K = 4 nodes along x, N = 48 columns = 6 m8n8k4 tiles).  The B fragments
// (lane = (a, b, c1): u at c1 and c1 + 2, 3 components) are gathered once per group
// straight into registers — no shared-memory box; the A fragments are the members' x
// weights.  Each lane of a D row then weighs its 12 values by wy[b] wz[c] and the 4 lanes
// of the row reduce with two xor shuffles.  Warps spanning more than IMMA_MAXG boxes gather
// per point (interp_direct).
constexpr int IMMA_MAXG = 8;

// 8 blocks (32 warps) per SM, <= 64 registers: the gathers want the occupancy (109 us at
// cfg4; 7 blocks 111 us, 6 blocks 113 us, uncapped 250 us)
#ifndef IBK_IMINB
#define IBK_IMINB 8
#endif
__global__ void __launch_bounds__(INTERP_THREADS, IBK_IMINB)
k_interp_mma(FluidGeom g, const double *__restrict__ u, double *X, int64_t np, double *U_out,
             long long *flag, const long long *dev_n, long long n, const int *__restrict__ perm,
             const uint8_t *__restrict__ fixed, double4 *pack, unsigned long long *pack_count,
             double *Xs) {
  // per lane-point: wx[0..3] | wy[0..3] | wz[0], wz[2], wz[1], wz[3]  (+2 pad: odd 16-B stride)
  __shared__ __align__(16) double rec[INTERP_THREADS / 32][32][14];
  __shared__ double uo[INTERP_THREADS / 32][32][3];
  __shared__ unsigned char mlist[INTERP_THREADS / 32][32];   // lanes of the current group
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int N1 = g.N1, N2 = g.N2, N3g = g.N3g;
  const int Vi = (int)((int64_t)N1 * N2 * g.uN3);     // component stride of the u array
  bool live = k < np;
  bool bad = false;
  const int64_t i = live ? (perm ? (int64_t)__ldg(&perm[k]) : k) : 0;
  double x0 = 0.5 * g.h, x1 = 0.5 * g.h, x2 = 0.5 * g.h;
  if (live) {
    if (Xs) { x0 = Xs[k]; x1 = Xs[np + k]; x2 = Xs[2 * np + k]; }   // binned SoA: coalesced
    else { x0 = X[3 * i + 0]; x1 = X[3 * i + 1]; x2 = X[3 * i + 2]; }
  }
  double wx[4], wy[4], wz[4];
  const int jx = axis_weights(x0, g.invh, wx);
  const int jy = axis_weights(x1, g.invh, wy);
  const int jz = axis_weights(x2, g.invh, wz);
  // slab: this rank updates only the points whose base plane floor(Z/h) it owns
  if (g.slab) live = live && ((unsigned)(jz + 1 - g.z0) & (unsigned)(N3g - 1)) < (unsigned)g.N3;
  const unsigned key = ((unsigned)(jz & (N3g - 1)) * N2 + (unsigned)(jy & (N2 - 1))) * N1 + (unsigned)(jx & (N1 - 1));
  const unsigned active = __ballot_sync(0xffffffffu, live);
  const unsigned peers = __match_any_sync(0xffffffffu, live ? key : 0xffffffffu) & active;
  const unsigned leaders = __ballot_sync(0xffffffffu, live && lane == __ffs(peers) - 1);
  double U0 = 0.0, U1 = 0.0, U2 = 0.0;
  if (__popc(leaders) <= IMMA_MAXG) {
    double2 *rw = reinterpret_cast<double2 *>(rec[warp][lane]);
    rw[0] = make_double2(wx[0], wx[1]); rw[1] = make_double2(wx[2], wx[3]);
    rw[2] = make_double2(wy[0], wy[1]); rw[3] = make_double2(wy[2], wy[3]);
    rw[4] = make_double2(wz[0], wz[2]); rw[5] = make_double2(wz[1], wz[3]);
    __syncwarp();
    const int a = lane & 3, b = (lane >> 2) & 3, c1 = lane >> 4;     // B fragment node
    const int p = lane >> 2, q = lane & 3;                            // D row, column pair
    const int yb = 2 * (q & 1), zc = q >> 1;                          // epilogue wy / wz pair
    unsigned lm = leaders;
    while (lm) {
      const int ld = __ffs(lm) - 1;
      lm &= lm - 1;
      const unsigned kl = __shfl_sync(0xffffffffu, key, ld);   // every lane shuffles
      const unsigned gm = __ballot_sync(0xffffffffu, live && key == kl);
      const int gx = __shfl_sync(0xffffffffu, jx, ld), gy = __shfl_sync(0xffffffffu, jy, ld),
                gz = __shfl_sync(0xffffffffu, jz, ld);
      const int xo = (gx + a) & (N1 - 1), yo = (gy + b) & (N2 - 1);
      const int e0 = (u_plane(g, gz, c1) * N2 + yo) * N1 + xo;
      const int e1 = (u_plane(g, gz, c1 + 2) * N2 + yo) * N1 + xo;
      // tile t: component t / 2, c = c1 (t even) or c1 + 2 (t odd)
      double bf[6];
      bf[0] = __ldg(u + e0);          bf[1] = __ldg(u + e1);
      bf[2] = __ldg(u + Vi + e0);     bf[3] = __ldg(u + Vi + e1);
      bf[4] = __ldg(u + 2 * Vi + e0); bf[5] = __ldg(u + 2 * Vi + e1);
      const int nm = __popc(gm);
#ifndef IBK_IRUN
#define IBK_IRUN 1
#endif
      // binned order: a group is almost always a run of consecutive lanes, whose members
      // are then lo + m without the member list
      const int glo = __ffs(gm) - 1;
      const bool run = IBK_IRUN && (gm >> glo) == (nm == 32 ? 0xffffffffu : (1u << nm) - 1u);
      if (!run) {
        __syncwarp();                                   // previous group's list consumed
        if ((gm >> lane) & 1u) mlist[warp][__popc(gm & ((1u << lane) - 1u))] = (unsigned char)lane;
        __syncwarp();
      }
      for (int m0 = 0; m0 < nm; m0 += 8) {
        const int src = m0 + p < nm ? (run ? glo + m0 + p : (int)mlist[warp][m0 + p]) : -1;
        const double af = src >= 0 ? rec[warp][src][a] : 0.0;
        double d[6][2];
#pragma unroll
        for (int t = 0; t < 6; ++t) dmma_8x8x4(d[t][0], d[t][1], af, bf[t]);
        // D[p][n], n = 2q + e: b = 2 (q & 1) + e, c = (t & 1) * 2 + (q >> 1); rows past the
        // group (src < 0) are zero and read record 0 (all lanes stay in the shuffles)
        const int sr = src >= 0 ? src : 0;
        const double2 yy = *reinterpret_cast<const double2 *>(&rec[warp][sr][4 + yb]);
        const double2 zz = *reinterpret_cast<const double2 *>(&rec[warp][sr][8 + 2 * zc]);
        double s[3];
#pragma unroll
        for (int cp = 0; cp < 3; ++cp)
          s[cp] = zz.x * (yy.x * d[2 * cp][0] + yy.y * d[2 * cp][1]) +
                  zz.y * (yy.x * d[2 * cp + 1][0] + yy.y * d[2 * cp + 1][1]);
        // transpose-reduce over the row's 4 lanes (3 shuffles): lane q ends with component
        // 2 (q & 1) + (q >> 1) summed over the row (q = 3: the zero pad)
        const bool o1 = q & 1, o2 = q & 2;
        const double ra = __shfl_xor_sync(0xffffffffu, o1 ? s[0] : s[2], 1, 4);
        const double rb = __shfl_xor_sync(0xffffffffu, o1 ? s[1] : 0.0, 1, 4);
        const double ka = (o1 ? s[2] : s[0]) + ra, kb = (o1 ? 0.0 : s[1]) + rb;
        const double sum = (o2 ? kb : ka) + __shfl_xor_sync(0xffffffffu, o2 ? ka : kb, 2, 4);
        const int cq = 2 * (q & 1) + (q >> 1);
        if (src >= 0 && cq < 3) uo[warp][src][cq] = sum;
      }
    }
    __syncwarp();
    U0 = uo[warp][lane][0]; U1 = uo[warp][lane][1]; U2 = uo[warp][lane][2];
  } else {
    if (live) interp_direct(u, g, Vi, jx, jy, jz, wx, wy, wz, U0, U1, U2);
  }
  if (live) {
    if (U_out) {
      U_out[3 * i + 0] = U0; U_out[3 * i + 1] = U1; U_out[3 * i + 2] = U2;
    } else if (!(fixed && fixed[i])) {    // fixed points never move (PAPER.md 919-920)
      const double y0 = x0 + g.dt * U0, y1 = x1 + g.dt * U1, y2 = x2 + g.dt * U2;
      X[3 * i + 0] = y0; X[3 * i + 1] = y1; X[3 * i + 2] = y2;
      if (Xs) { Xs[k] = y0; Xs[np + k] = y1; Xs[2 * np + k] = y2; }
      bad = !(isfinite(y0) && isfinite(y1) && isfinite(y2));
    }
  }
  // slab: the owned points' X^{n+1} (fixed ones included, unchanged) are packed for the
  // all-gather that keeps every rank's replica of X current
  if (pack && !U_out) {
    const unsigned own = __ballot_sync(0xffffffffu, live);
    unsigned long long base = 0;
    if (own) {
      if (lane == __ffs(own) - 1) base = atomicAdd(pack_count, (unsigned long long)__popc(own));
      base = __shfl_sync(0xffffffffu, base, __ffs(own) - 1);
      if (live)
        pack[base + __popc(own & ((1u << lane) - 1u))] =
            make_double4(X[3 * i + 0], X[3 * i + 1], X[3 * i + 2], (double)i);
    }
  }
  // warp-level vote: a block-wide barrier here made every warp wait for the block's slowest
  if (flag && __any_sync(0xffffffffu, bad) && lane == 0) {
    const long long st = dev_n ? *dev_n : n;
    atomicMin(flag, st);
  }
}

cudaError_t launch_interp(const FluidGeom &g, const double *u, double *X, int64_t np,
                          double *U_out, long long *flag, const long long *dev_n, long long n,
                          const int *perm, const uint8_t *fixed, cudaStream_t s,
                          double4 *pack, unsigned long long *pack_count, double *Xs) {
  if (np > 0)
    k_interp_mma<<<(unsigned)((np + INTERP_THREADS - 1) / INTERP_THREADS), INTERP_THREADS, 0, s>>>(
        g, u, X, np, U_out, flag, dev_n, n, perm, fixed, pack, pack_count, perm ? Xs : nullptr);
  return cudaGetLastError();
}

// End of a step: the device step counter read by the drive and the non-finite flag advances
// (graph replays carry no host-side step index).
__global__ void k_step_inc(long long *dev_n) { *dev_n += 1; }

cudaError_t launch_step_inc(long long *dev_n, cudaStream_t s) {
  k_step_inc<<<1, 1, 0, s>>>(dev_n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ cell binning
// perm = point indices grouped by the base cell floor(X/h) mod N of their delta support
// (a counting sort over the N^3 cells: count, exclusive scan, scatter).  Only the order in
// which spread/interp visit points depends on it, never a result beyond fp64 summation
// order; ib_step refreshes it every IB_SORT_PERIOD steps.
__device__ __forceinline__ unsigned cell_key(const double *X, int64_t i, double invh, int N1,
                                             int N2, int N3) {
  const int cx = (int)(long long)floor(X[3 * i + 0] * invh) & (N1 - 1);
  const int cy = (int)(long long)floor(X[3 * i + 1] * invh) & (N2 - 1);
  const int cz = (int)(long long)floor(X[3 * i + 2] * invh) & (N3 - 1);
  return ((unsigned)cz * N2 + (unsigned)cy) * N1 + (unsigned)cx;
}

__global__ void k_bin_count(const double *__restrict__ X, int64_t np, double invh, int N1,
                            int N2, int N3, unsigned *cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = i < np;
  const unsigned key = ok ? cell_key(X, i, invh, N1, N2, N3) : 0xffffffffu;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  if (ok && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&cnt[key], __popc(peers));
}

constexpr int SCAN_T = 1024, SCAN_E = 8;          // block scan: 8192 counters per block

__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned *ws, unsigned *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned t = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;                                  // inclusive warp totals
  }
  __syncthreads();
  const unsigned before = (w ? ws[w - 1] : 0u) + x - v;
  if (total) *total = ws[31];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_partial(const unsigned *cnt, size_t n, unsigned *bsum) {
  __shared__ unsigned ws[32];
  const size_t base = (size_t)blockIdx.x * SCAN_T * SCAN_E + (size_t)threadIdx.x * SCAN_E;
  unsigned s = 0;
#pragma unroll
  for (int e = 0; e < SCAN_E; ++e) s += base + e < n ? cnt[base + e] : 0u;
  unsigned tot;
  block_exclusive_scan(s, ws, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_bsum(unsigned *bsum, int nb) {
  __shared__ unsigned ws[32];
  unsigned carry = 0;
  for (int b0 = 0; b0 < nb; b0 += SCAN_T) {
    const int b = b0 + threadIdx.x;
    const unsigned v = b < nb ? bsum[b] : 0u;
    unsigned tot;
    const unsigned ex = block_exclusive_scan(v, ws, &tot);
    if (b < nb) bsum[b] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(SCAN_T) k_scan_final(unsigned *cnt, size_t n, const unsigned *bsum) {
  __shared__ unsigned ws[32];
  const size_t base = (size_t)blockIdx.x * SCAN_T * SCAN_E + (size_t)threadIdx.x * SCAN_E;
  unsigned v[SCAN_E], s = 0;
#pragma unroll
  for (int e = 0; e < SCAN_E; ++e) { v[e] = base + e < n ? cnt[base + e] : 0u; s += v[e]; }
  unsigned run = bsum[blockIdx.x] + block_exclusive_scan(s, ws, nullptr);
#pragma unroll
  for (int e = 0; e < SCAN_E; ++e)
    if (base + e < n) { cnt[base + e] = run; run += v[e]; }
}

__global__ void k_bin_scatter(const double *__restrict__ X, int64_t np, double invh, int N1,
                              int N2, int N3, unsigned *off, int *perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = i < np;
  const unsigned key = ok ? cell_key(X, i, invh, N1, N2, N3) : 0xffffffffu;
  const unsigned peers = __match_any_sync(0xffffffffu, key);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  unsigned base = 0;
  if (ok && lane == leader) base = atomicAdd(&off[key], __popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (ok) perm[base + __popc(peers & ((1u << lane) - 1u))] = (int)i;
}

__global__ void k_gather_xs(const double *__restrict__ X, const int *__restrict__ perm,
                            int64_t np, double *Xs) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < np) {
    const int64_t i = perm[k];
    Xs[k] = X[3 * i]; Xs[np + k] = X[3 * i + 1]; Xs[2 * np + k] = X[3 * i + 2];
  }
}

cudaError_t launch_gather_xs(const double *X, const int *perm, int64_t np, double *Xs,
                             cudaStream_t s) {
  if (np > 0 && Xs) k_gather_xs<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(X, perm, np, Xs);
  return cudaGetLastError();
}

cudaError_t launch_bin(const FluidGeom &g, const double *X, int64_t np, unsigned *cnt,
                       unsigned *bsum, int *perm, double *Xs, cudaStream_t s) {
  if (np <= 0) return cudaSuccess;
  const size_t n = (size_t)g.Vg;                  // cells of the whole lattice
  const int nb = (int)((n + (size_t)SCAN_T * SCAN_E - 1) / ((size_t)SCAN_T * SCAN_E));
  const unsigned pb = (unsigned)((np + 255) / 256);
  cudaError_t e = cudaMemsetAsync(cnt, 0, n * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  k_bin_count<<<pb, 256, 0, s>>>(X, np, g.invh, g.N1, g.N2g, g.N3g, cnt);
  k_scan_partial<<<nb, SCAN_T, 0, s>>>(cnt, n, bsum);
  k_scan_bsum<<<1, SCAN_T, 0, s>>>(bsum, nb);
  k_scan_final<<<nb, SCAN_T, 0, s>>>(cnt, n, bsum);
  k_bin_scatter<<<pb, 256, 0, s>>>(X, np, g.invh, g.N1, g.N2g, g.N3g, cnt, perm);
  return launch_gather_xs(X, perm, np, Xs, s);
}

int bin_scan_blocks(int64_t V) {
  return (int)((V + (int64_t)SCAN_T * SCAN_E - 1) / ((int64_t)SCAN_T * SCAN_E));
}

}  // namespace ibk
